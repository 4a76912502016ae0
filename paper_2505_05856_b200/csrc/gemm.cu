// tcgen05 / TMEM / TMA GEMM for sm_100a, bf16 x bf16 -> fp32 accumulate.
//
//   C[z] = epilogue( alpha * A[z] (M x K) * B[z]^T (K x N) )
//
// serves every dense contraction of the stage executor: the fused QKV,
// out-projection, FFN and vocabulary-head GEMMs (fwd, dgrad, wgrad), and the
// per-(batch, head) attention products QK^T, PV and their gradients.  Operands
// may be K-major or MN-major (both are native UMMA operand layouts, so no
// transposes are ever materialised) and carry a two-level batch index
// z = z1 + Z1 * z2 (batch x head for attention).
//
// Structure (one CTA per SM, persistent, warp-specialised, 256 threads):
//   warp 0      TMA producer: A/B tiles into a kStages-deep smem ring
//   warp 1      MMA issuer: one elected lane issues tcgen05.mma (M=128, N=BN,
//               K=16) into a double-buffered TMEM accumulator
//   warp 2      TMEM allocator
//   warps 4-11  epilogue: tcgen05.ld (each thread one accumulator row) ->
//               alpha/bias/residual/GELU in registers -> a 128-byte-swizzled
//               32-row staging tile in shared memory -> TMA bulk store (f32
//               split-K / accumulate: TMA bulk reduce-add).  The residual
//               operand is TMA-loaded into a second staging tile ahead of use,
//               so the epilogue issues no per-thread global loads or stores.
//               Batched (attention) GEMMs keep a direct-store epilogue.
// Barriers: full/empty per smem stage (TMA <-> MMA), tmem_full/tmem_empty per
// accumulator buffer (MMA <-> epilogue), so the epilogue of one work unit
// overlaps the mainloop of the next.
//
// Work units are (tile, k-split) pairs.  Split-K (f32 outputs only) lets the
// small weight-gradient GEMMs (e.g. 1024 x 1024 x 4096: 32 tiles) fill all
// 148 SMs; split partials are combined with vector red.global.add.f32.
#include "common.cuh"
#include "../../include/dawnpiper.h"

#include <mutex>
#include <unordered_map>

namespace dpn {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // one 128-byte swizzle row of bf16
#ifndef DPN_GEMM_EPI_WARPS
#define DPN_GEMM_EPI_WARPS 8
#endif
constexpr int kEpiWarps = DPN_GEMM_EPI_WARPS;  // 8: two per SM sub-partition, each pair splits the columns
constexpr int kEpiGroups = kEpiWarps / 4;      // warps sharing a TMEM lane quarter
constexpr int kEpiWarp0 = 4;
constexpr int kThreads = 32 * (kEpiWarp0 + kEpiWarps);

struct GemmParams {
  int tma_epi;  // 1: staged TMA-store epilogue (tmC / tmR / tmX valid)
  int M, N, K;
  int Z1, Z;
  int tiles_m, tiles_n, tile_m;
  int splits, kb_per_split;
  long long units;  // tiles * splits
  void* C;
  long long ldc, c_s1, c_s2;
  int c_f32, accumulate;
  const __nv_bfloat16* bias;
  const __nv_bfloat16* res;
  long long ldr, r_s1, r_s2;
  int res_mode;  // 0: + residual, 1: * gelu'(residual) (fused GELU backward)
  __nv_bfloat16* aux;
  float alpha;
  int gelu;
  long long* trace;  // debug: per-CTA wait cycles by role (dpn_gemm_debug_trace), else null
  float* colsum;     // optional: colsum[n] += sum over rows of the stored bf16 C (bias gradient)
};

// timed mbarrier wait (debug tracing only)
__device__ __forceinline__ void mbar_wait_t(uint64_t* bar, uint32_t parity, long long* acc) {
  if (acc == nullptr) {
    mbar_wait(bar, parity);
    return;
  }
  const long long t0 = clock64();
  mbar_wait(bar, parity);
  *acc += clock64() - t0;
}

// per epilogue warp: a 4 KB output staging tile (32 rows x 128 B) and a 4 KB
// side tile (the TMA-loaded residual, or the GELU pre-activation `aux` output)
constexpr int kEpiStage = 4096;
constexpr int kEpiBytes = kEpiWarps * 2 * kEpiStage;
constexpr int kMaxSmem = 232448;  // 227 KB per CTA on sm_100
// build-time knobs for same-box A/B experiments (tools/build_variant.sh)
#ifndef DPN_GEMM_MAX_STAGES
#define DPN_GEMM_MAX_STAGES 8
#endif
#ifndef DPN_GEMM_GROUP
#define DPN_GEMM_GROUP 8
#endif
#ifndef DPN_GEMM_COMMIT_PAIRS
#define DPN_GEMM_COMMIT_PAIRS 0
#endif
#ifndef DPN_GEMM_HINT
#define DPN_GEMM_HINT 0  // 1: A evict_first / B evict_last, 2: both evict_last (pair tiles)
#endif
#ifndef DPN_GEMM_L2_PROMO
#define DPN_GEMM_L2_PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif

// CG: CTAs per cluster. 1 = one CTA per tile; 2 = a CTA pair on one 256-row
// tile (tcgen05 cta_group::2); 4 = two pairs on N-adjacent tiles sharing their
// A rows through TMA multicast (each CTA fetches half of its A tile from L2).
template <int BN, int CG>
struct Cfg {
  static constexpr int kPair = CG == 1 ? 1 : 2;
  static constexpr int kBRows = BN / kPair;  // rows of B this CTA loads (pair: half of N)
  static constexpr int kABytes = BM * BK * 2;
  static constexpr int kBBytes = kBRows * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kFit = (kMaxSmem - kEpiBytes - 2048) / kStageBytes;
  static constexpr int kStages = kFit < DPN_GEMM_MAX_STAGES ? kFit : DPN_GEMM_MAX_STAGES;
  static constexpr int kTmemCols = 2 * BN;  // two accumulator buffers
  static constexpr int kSmem = kStages * kStageBytes + kEpiBytes + 1024 /*align*/ + 256 /*barriers*/;
  static_assert(kSmem <= kMaxSmem, "shared memory budget");
};

// byte offset of 16-byte chunk c of row r in a 128-byte-swizzled tile
__device__ __forceinline__ uint32_t swz128(int r, int c) { return r * 128 + ((c ^ (r & 7)) << 4); }

__device__ __forceinline__ void epi_fence_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void tma_load_2d_cta(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}

__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, const void* src, int c0,
                                                  int c1) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

struct Unit {
  int z1, z2, m0, nb, kb0, kb1;
};

__device__ __forceinline__ Unit decode(const GemmParams& p, long long u, int nk) {
  Unit w;
  const int split = (int)(u % p.splits);
  const long long t = u / p.splits;
  const long long per_z = (long long)p.tiles_m * p.tiles_n;
  const int z = (int)(t / per_z);
  const int r = (int)(t - (long long)z * per_z);
  // grouped raster: 8 m-blocks sweep all n-blocks together (L2 reuse of B)
  const int G = DPN_GEMM_GROUP;
  const int per_group = G * p.tiles_n;
  const int g = r / per_group;
  const int first_m = g * G;
  const int gsize = min(p.tiles_m - first_m, G);
  const int in_g = r - g * per_group;
  w.m0 = (first_m + in_g % gsize) * p.tile_m;
  w.nb = in_g / gsize;
  w.z1 = z % p.Z1;
  w.z2 = z / p.Z1;
  w.kb0 = split * p.kb_per_split;
  w.kb1 = min(nk, w.kb0 + p.kb_per_split);
  return w;
}

__device__ __forceinline__ void red_add_v2(float* addr, float a, float b) {
  asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(addr), "f"(a), "f"(b) : "memory");
}

__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}

// Epilogue of one 32-column chunk: this thread owns row `row` and the fp32
// accumulators v[0..31] of columns [col0, col0+32).  Each row segment is 64 B
// (bf16) / 128 B (f32) contiguous, so every 16-byte access fills whole sectors.
__device__ __forceinline__ void epilogue_chunk(const GemmParams& p, float* v, int row, int col0,
                                               long long c_base, long long r_base) {
  if (row >= p.M || col0 >= p.N) return;
  const bool full = col0 + 32 <= p.N;
  if (p.alpha != 1.f) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] *= p.alpha;
  }
  const long long coff = c_base + (long long)row * p.ldc + col0;
  if (p.c_f32) {
    float* cp = reinterpret_cast<float*>(p.C) + coff;
    if (full) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (p.splits > 1) {
          red_add_v4(cp + 4 * q, v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        } else {
          float4 o = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          if (p.accumulate) {
            const float4 old = reinterpret_cast<const float4*>(cp)[q];
            o.x += old.x; o.y += old.y; o.z += old.z; o.w += old.w;
          }
          reinterpret_cast<float4*>(cp)[q] = o;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        if (col0 + i < p.N) {
          if (p.splits > 1) atomicAdd(cp + i, v[i]);
          else cp[i] = p.accumulate ? cp[i] + v[i] : v[i];
        }
      }
    }
    return;
  }
  if (p.bias) {
    const __nv_bfloat16* bp = p.bias + col0;
    if (full) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 u = reinterpret_cast<const uint4*>(bp)[q];
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = __bfloat1622float2(h[k]);
          v[8 * q + 2 * k] += f.x;
          v[8 * q + 2 * k + 1] += f.y;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < p.N) v[i] += __bfloat162float(bp[i]);
    }
  }
  if (p.res) {
    const __nv_bfloat16* rp = p.res + r_base + (long long)row * p.ldr + col0;
    if (full) {
      uint4 u[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) u[q] = reinterpret_cast<const uint4*>(rp)[q];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u[q]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = __bfloat1622float2(h[k]);
          if (p.res_mode == 0) {
            v[8 * q + 2 * k] += f.x;
            v[8 * q + 2 * k + 1] += f.y;
          } else {
            v[8 * q + 2 * k] *= gelu_tanh_grad(f.x);
            v[8 * q + 2 * k + 1] *= gelu_tanh_grad(f.y);
          }
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < p.N) {
          const float f = __bfloat162float(rp[i]);
          v[i] = p.res_mode == 0 ? v[i] + f : v[i] * gelu_tanh_grad(f);
        }
    }
  }
  if (p.gelu) {
    if (p.aux) {
      __nv_bfloat16* ap = p.aux + coff;
      if (full) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 u;
          u.x = pack_bf16(v[8 * q + 0], v[8 * q + 1]);
          u.y = pack_bf16(v[8 * q + 2], v[8 * q + 3]);
          u.z = pack_bf16(v[8 * q + 4], v[8 * q + 5]);
          u.w = pack_bf16(v[8 * q + 6], v[8 * q + 7]);
          reinterpret_cast<uint4*>(ap)[q] = u;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (col0 + i < p.N) ap[i] = __float2bfloat16(v[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = gelu_tanh(v[i]);
  }
  __nv_bfloat16* cp = reinterpret_cast<__nv_bfloat16*>(p.C) + coff;
  if (full) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 u;
      u.x = pack_bf16(v[8 * q + 0], v[8 * q + 1]);
      u.y = pack_bf16(v[8 * q + 2], v[8 * q + 3]);
      u.z = pack_bf16(v[8 * q + 4], v[8 * q + 5]);
      u.w = pack_bf16(v[8 * q + 6], v[8 * q + 7]);
      reinterpret_cast<uint4*>(cp)[q] = u;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (col0 + i < p.N) cp[i] = __float2bfloat16(v[i]);
  }
}

// TMA-staged epilogue of one accumulator tile for one epilogue warp: rows
// [row_base, row_base+32) (one per lane), the warp's column chunks of the tile.
// bf16 outputs move in 64-column chunks (128-byte rows), f32 in 32-column ones.
template <int BN>
__device__ __forceinline__ void epilogue_tile_tma(const GemmParams& p, const CUtensorMap* tmC,
                                                  const CUtensorMap* tmR, const CUtensorMap* tmX,
                                                  uint32_t taddr, int n0, int row_base, int half,
                                                  int lane, uint8_t* s_out, uint8_t* s_side,
                                                  uint64_t* rbar, uint32_t& rphase) {
  if (p.c_f32) {
    constexpr int kChunks = BN / 32;
#pragma unroll 1
    for (int c = half; c < kChunks; c += kEpiGroups) {
      const int col0 = n0 + c * 32;
      if (col0 >= p.N) break;
      uint32_t r[32];
      tmem_ld_32x32b_x32(taddr + c * 32, r);
      tmem_ld_wait();
      if (lane == 0) bulk_wait_read0();
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 o = make_float4(__uint_as_float(r[4 * q]) * p.alpha, __uint_as_float(r[4 * q + 1]) * p.alpha,
                               __uint_as_float(r[4 * q + 2]) * p.alpha, __uint_as_float(r[4 * q + 3]) * p.alpha);
        sts128(smem_u32(s_out) + swz128(lane, q),
               make_uint4(__float_as_uint(o.x), __float_as_uint(o.y), __float_as_uint(o.z), __float_as_uint(o.w)));
      }
      epi_fence_async();
      __syncwarp();
      if (lane == 0) {
        if (p.splits > 1 || p.accumulate) tma_reduce_add_2d(tmC, s_out, col0, row_base);
        else tma_store_2d(tmC, s_out, col0, row_base);
        bulk_commit();
      }
    }
    return;
  }
  constexpr int kChunks = BN / 64;
  const bool res = p.res != nullptr;
  const bool aux = p.gelu && p.aux != nullptr;
#pragma unroll 1
  for (int c = half; c < kChunks; c += kEpiGroups) {
    const int col0 = n0 + c * 64;
    if (col0 >= p.N) break;
    float v[64];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(taddr + c * 64 + h * 32, r);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) v[h * 32 + i] = __uint_as_float(r[i]);
    }
    if (p.alpha != 1.f) {
#pragma unroll
      for (int i = 0; i < 64; ++i) v[i] *= p.alpha;
    }
    if (p.bias) {
      const __nv_bfloat16* bp = p.bias + col0;
      if (col0 + 64 <= p.N) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint4 u = reinterpret_cast<const uint4*>(bp)[q];
          const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float2 o = fma2(make_float2(1.f, 1.f), make_float2(v[8 * q + 2 * k], v[8 * q + 2 * k + 1]),
                                  __bfloat1622float2(hh[k]));
            v[8 * q + 2 * k] = o.x;
            v[8 * q + 2 * k + 1] = o.y;
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (col0 + i < p.N) v[i] += __bfloat162float(bp[i]);
      }
    }
    if (res) {
      mbar_wait(rbar, rphase);
      rphase ^= 1;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint4 u = lds128(smem_u32(s_side) + swz128(lane, q));
        const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = __bfloat1622float2(hh[k]);
          const float2 vv = make_float2(v[8 * q + 2 * k], v[8 * q + 2 * k + 1]);
          const float2 o = p.res_mode == 0 ? fma2(make_float2(1.f, 1.f), vv, f)
                                           : mul2(vv, gelu_tanh_grad2(f));
          v[8 * q + 2 * k] = o.x;
          v[8 * q + 2 * k + 1] = o.y;
        }
      }
      __syncwarp();  // every lane has read the residual tile: prefetch the next chunk's
      const int cn = c + kEpiGroups;
      if (lane == 0 && cn < kChunks && n0 + cn * 64 < p.N) {
        mbar_expect_tx(rbar, kEpiStage);
        tma_load_2d_cta(s_side, tmR, rbar, n0 + cn * 64, row_base);
      }
    }
    if (lane == 0) bulk_wait_read0();  // earlier stores have finished reading the staging tiles
    __syncwarp();
    if (aux) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        uint4 u;
        u.x = pack_bf16(v[8 * q + 0], v[8 * q + 1]);
        u.y = pack_bf16(v[8 * q + 2], v[8 * q + 3]);
        u.z = pack_bf16(v[8 * q + 4], v[8 * q + 5]);
        u.w = pack_bf16(v[8 * q + 6], v[8 * q + 7]);
        sts128(smem_u32(s_side) + swz128(lane, q), u);
      }
    }
    if (p.gelu) {
#pragma unroll
      for (int i = 0; i < 64; i += 2) {
        const float2 g = gelu_tanh2(make_float2(v[i], v[i + 1]));
        v[i] = g.x;
        v[i + 1] = g.y;
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint4 u;
      u.x = pack_bf16(v[8 * q + 0], v[8 * q + 1]);
      u.y = pack_bf16(v[8 * q + 2], v[8 * q + 3]);
      u.z = pack_bf16(v[8 * q + 4], v[8 * q + 5]);
      u.w = pack_bf16(v[8 * q + 6], v[8 * q + 7]);
      sts128(smem_u32(s_out) + swz128(lane, q), u);
    }
    epi_fence_async();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(tmC, s_out, col0, row_base);
      if (aux) tma_store_2d(tmX, s_side, col0, row_base);
      bulk_commit();
    }
    if (p.colsum) {
      // column sums of the stored tile (the bias gradient of the linear whose
      // output gradient C is): lane l adds columns 2l, 2l+1 over the warp's 32
      // rows, read back from the swizzled staging tile (one 128-byte row per
      // load: conflict-free); the next chunk's writes wait on the __syncwarp above
      const int nr = min(32, p.M - row_base);
      float2 cs = make_float2(0.f, 0.f);
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        if (r < nr) {
          const uint32_t u = lds32(smem_u32(s_out) + swz128(r, lane >> 2) + (lane & 3) * 4);
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u));
          cs.x += f.x;
          cs.y += f.y;
        }
      }
      const int cc = col0 + 2 * lane;
      if (cc + 1 < p.N) red_add_v2(p.colsum + cc, cs.x, cs.y);
      else if (cc < p.N) atomicAdd(p.colsum + cc, cs.x);
    }
  }
}

template <int BN, bool A_MN, bool B_MN, int CG>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmR,
                const __grid_constant__ CUtensorMap tmX, const GemmParams p) {
  using C = Cfg<BN, CG>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * C::kABytes;
  uint8_t* sEpi = smem + C::kStages * C::kStageBytes;  // 1024-aligned (stage bytes are)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sEpi + kEpiBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::kStages;
  uint64_t* tfull = bars + 2 * C::kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* rbar = tempty + 2;  // one residual-tile barrier per epilogue warp
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + kEpiWarps);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nk = (p.K + BK - 1) / BK;
  // CTA pair (CG >= 2): the pair's rank-0 CTA leads -- it issues the MMAs and
  // owns the full / tmem_empty barriers both CTAs' producers and epilogues
  // report to.  CG == 4: pair `pr` of the cluster works on N-tile 2*nb + pr.
  constexpr int kPair = C::kPair;
  constexpr bool kMc = CG == 4;
  const uint32_t crank = CG >= 2 ? cluster_ctarank() : 0;
  const uint32_t rank = crank & 1u;       // rank within the pair
  const uint32_t pr = crank >> 1;         // pair within the cluster
  const uint32_t leader = crank & ~1u;    // cluster rank of this pair's leader
  const uint32_t pair_mask = 0x3u << leader;
  const long long cluster_id = blockIdx.x / CG;
  const long long n_clusters = gridDim.x / CG;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    if (p.tma_epi) {
      prefetch_tmap(&tmC);
      if (p.res) prefetch_tmap(&tmR);
      if (p.aux) prefetch_tmap(&tmX);
    }
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], kPair);  // one arrival per producer of the pair
      mbar_init(&empty[s], kMc ? 2 : 1);  // multicast: both pairs must release the stage
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kPair * kEpiWarps);  // one arrival per epilogue warp of the pair
    }
    for (int e = 0; e < kEpiWarps; ++e) mbar_init(&rbar[e], 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<C::kTmemCols, kPair>(tmem_slot);
  tc_fence_before();
  if constexpr (CG >= 2) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const long long t_start = clock64();
  pdl_wait();  // everything above overlaps the previous kernel's tail (PDL)
  const long long t_run = clock64();
  // debug trace slots per CTA: 0 producer wait(empty), 1 MMA wait(full),
  // 2 MMA wait(tempty), 3 epilogue wait(tfull) (warp 4), 4 run cycles, 5 pdl wait,
  // 6 epilogue busy (warp 4), 7 units
  long long tw = 0, tw2 = 0;
  long long* trace_w = p.trace ? &tw : nullptr;
  long long* trace_w2 = p.trace ? &tw2 : nullptr;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (long long u = cluster_id; u < p.units; u += n_clusters) {
        const Unit w = decode(p, u, nk);
        const int m0 = w.m0 + BM * (int)rank;
        const int n0 = (w.nb * (kMc ? 2 : 1) + (int)pr) * BN + C::kBRows * (int)rank;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          mbar_wait_t(&empty[stage], phase ^ 1, trace_w);
          if (rank == 0) mbar_expect_tx(&full[stage], kPair * C::kStageBytes);
          else mbar_arrive_remote(&full[stage], leader);
          uint8_t* a_dst = sA + stage * C::kABytes;
          uint8_t* b_dst = sB + stage * C::kBBytes;
          const int k0 = kb * BK;
          auto load = [&](void* dst, const CUtensorMap* m, int c0, int c2) {
            if constexpr (CG >= 2 && DPN_GEMM_HINT != 0) {
              const uint64_t pol = (m == &tmA && DPN_GEMM_HINT == 1) ? l2_policy_evict_first()
                                                                    : l2_policy_evict_last();
              tma_load_4d_pair_hint(dst, m, &full[stage], c0, w.z1, c2, w.z2, pol);
            } else if constexpr (CG >= 2) {
              tma_load_4d_pair(dst, m, &full[stage], c0, w.z1, c2, w.z2);
            } else {
              tma_load_4d(dst, m, &full[stage], c0, w.z1, c2, w.z2);
            }
          };
          if constexpr (kMc) {
            // this CTA fetches 64 of its 128 A rows and multicasts them to the
            // same-rank CTA of the other pair (which fetches the other 64)
            const uint16_t mc = (uint16_t)((1u << crank) | (1u << (crank ^ 2u)));
            if (!A_MN) tma_load_4d_pair_mc(a_dst + pr * 64 * 128, &tmA, &full[stage], k0, w.z1,
                                           m0 + 64 * (int)pr, w.z2, mc);
            else tma_load_4d_pair_mc(a_dst + pr * 64 * BK * 2, &tmA, &full[stage], m0 + 64 * (int)pr,
                                     w.z1, k0, w.z2, mc);
          } else if (!A_MN) {
            load(a_dst, &tmA, k0, m0);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) load(a_dst + j * 64 * BK * 2, &tmA, m0 + 64 * j, k0);
          }
          if (!B_MN) {
            load(b_dst, &tmB, k0, n0);
          } else {
#pragma unroll
            for (int j = 0; j < C::kBRows / 64; ++j) load(b_dst + j * 64 * BK * 2, &tmB, n0 + 64 * j, k0);
          }
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (pair leader only) ----------------
    if (rank == 0) {
      constexpr uint32_t idesc = idesc_bf16(BM * kPair, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
      // K-major SW128: rows of 128 B, 8-row atoms 1024 B apart; +32 B per K=16 step.
      // MN-major SW128: 64-element MN atoms BK*128 B apart (LBO), 8-row K groups
      // 1024 B apart (SBO); +16 rows * 128 B = 2048 B per K=16 step.
      constexpr uint32_t a_lbo = A_MN ? BK * 128 : 16, b_lbo = B_MN ? BK * 128 : 16;
      constexpr uint32_t a_kstep = A_MN ? 2048 : 32, b_kstep = B_MN ? 2048 : 32;
      int stage = 0, prev_stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (long long u = cluster_id; u < p.units; u += n_clusters) {
        const Unit w = decode(p, u, nk);
        mbar_wait_t(&tempty[acc], acc_phase ^ 1, trace_w2);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          mbar_wait_t(&full[stage], phase, trace_w);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a_addr = smem_u32(sA + stage * C::kABytes);
            const uint32_t b_addr = smem_u32(sB + stage * C::kBBytes);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint64_t ad = smem_desc_sw128(a_addr + k * a_kstep, a_lbo, 1024);
              const uint64_t bd = smem_desc_sw128(b_addr + k * b_kstep, b_lbo, 1024);
              const uint32_t accum = (kb > w.kb0 || k > 0) ? 1u : 0u;
              if constexpr (CG >= 2) umma_bf16_pair(tmem_d, ad, bd, idesc, accum);
              else umma_bf16(tmem_d, ad, bd, idesc, accum);
            }
            // DPN_GEMM_COMMIT_PAIRS: release smem stages two k-blocks at a time
            // (one commit point per 8 MMAs instead of per 4)
            const bool flush = !DPN_GEMM_COMMIT_PAIRS || ((kb - w.kb0) & 1) || kb == w.kb1 - 1;
            const bool with_prev = DPN_GEMM_COMMIT_PAIRS && ((kb - w.kb0) & 1);
            if (flush) {
              if constexpr (CG >= 2) {
                // multicast: the stage is free only once both pairs consumed it
                if (with_prev) umma_commit_pair(&empty[prev_stage], kMc ? 0xF : pair_mask);
                umma_commit_pair(&empty[stage], kMc ? 0xF : pair_mask);
                if (kb == w.kb1 - 1) umma_commit_pair(&tfull[acc], pair_mask);
              } else {
                if (with_prev) umma_commit(&empty[prev_stage]);
                umma_commit(&empty[stage]);
                if (kb == w.kb1 - 1) umma_commit(&tfull[acc]);
              }
            }
          }
          __syncwarp();
          prev_stage = stage;
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ---------------- epilogue ----------------
    const int ew = warp - kEpiWarp0;
    const int lanes = (warp & 3) * 32;  // TMEM lane quarter this warp may access
    const int half = ew >> 2;           // which column chunks (even / odd) it owns
    int acc = 0;
    uint32_t acc_phase = 0;
    uint8_t* s_out = sEpi + ew * 2 * kEpiStage;
    uint8_t* s_side = s_out + kEpiStage;
    uint32_t rphase = 0;
    for (long long u = cluster_id; u < p.units; u += n_clusters) {
      const Unit w = decode(p, u, nk);
      const int n0 = (w.nb * (kMc ? 2 : 1) + (int)pr) * BN;
      if (p.tma_epi) {
        const int row_base = w.m0 + BM * (int)rank + lanes;
        // the first residual tile loads while the accumulator is still being built
        if (p.res && lane == 0 && n0 + half * 64 < p.N) {
          mbar_expect_tx(&rbar[ew], kEpiStage);
          tma_load_2d_cta(s_side, &tmR, &rbar[ew], n0 + half * 64, row_base);
        }
        mbar_wait_t(&tfull[acc], acc_phase, trace_w);
        const long long te0 = clock64();
        tc_fence_after();
        epilogue_tile_tma<BN>(p, &tmC, &tmR, &tmX, tmem_base + acc * BN + ((uint32_t)lanes << 16), n0,
                              row_base, half, lane, s_out, s_side, &rbar[ew], rphase);
        if (p.trace) tw2 += clock64() - te0;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG >= 2) mbar_arrive_remote(&tempty[acc], leader);
          else mbar_arrive(&tempty[acc]);
        }
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
        continue;
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = w.m0 + BM * (int)rank + lanes + lane;
      const long long c_base = (long long)w.z1 * p.c_s1 + (long long)w.z2 * p.c_s2;
      const long long r_base = (long long)w.z1 * p.r_s1 + (long long)w.z2 * p.r_s2;
      const uint32_t taddr = tmem_base + acc * BN + ((uint32_t)lanes << 16);
#pragma unroll 1
      for (int c = half; c < BN / 32; c += kEpiGroups) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + c * 32, r);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        epilogue_chunk(p, v, row, n0 + c * 32, c_base, r_base);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG >= 2) mbar_arrive_remote(&tempty[acc], leader);
        else mbar_arrive(&tempty[acc]);
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (p.tma_epi && lane == 0) bulk_wait0();  // stores complete before the CTA retires
  }
  if (p.trace && lane == 0) {
    long long* t = p.trace + (long long)blockIdx.x * 8;
    if (warp == 0) { t[0] = tw; t[5] = t_run - t_start; }
    if (warp == 1 && rank == 0) { t[1] = tw; t[2] = tw2; }
    if (warp == kEpiWarp0) { t[3] = tw; t[6] = tw2; t[4] = clock64() - t_run; }
  }

  tc_fence_before();
  if constexpr (CG >= 2) cluster_sync_all(); else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_free<C::kTmemCols, kPair>(tmem_base);
  }
}

// ---- host side ------------------------------------------------------------------

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// Encoded maps are cached by their full description (a map holds no reference
// to the memory, so an identical key always yields an identical map): the
// executor issues the same few hundred GEMM call sites every step.
struct MapKey {
  const void* ptr;
  long long inner, outer, ld, s1, s2;
  int Z1, Z2, box;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && inner == o.inner && outer == o.outer && ld == o.ld && s1 == o.s1 &&
           s2 == o.s2 && Z1 == o.Z1 && Z2 == o.Z2 && box == o.box;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = std::hash<const void*>()(k.ptr);
    for (long long v : {k.inner, k.outer, k.ld, k.s1, k.s2, (long long)k.Z1, (long long)k.Z2,
                        (long long)k.box})
      h = h * 1000003u ^ std::hash<long long>()(v);
    return h;
  }
};
std::mutex g_map_mu;
std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;

int encode_map(CUtensorMap* map, const void* ptr, long long inner, long long outer, long long ld,
               int Z1, long long s1, int Z2, long long s2, int box_outer);

int make_map(CUtensorMap* map, const void* ptr, long long inner, long long outer, long long ld,
             int Z1, long long s1, int Z2, long long s2, int box_outer) {
  const MapKey key{ptr, inner, outer, ld, s1, s2, Z1, Z2, box_outer};
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) {
      *map = it->second;
      return 0;
    }
  }
  const int rc = encode_map(map, ptr, inner, outer, ld, Z1, s1, Z2, s2, box_outer);
  if (rc == 0) {
    std::lock_guard<std::mutex> lk(g_map_mu);
    if (g_maps.size() > 65536) g_maps.clear();
    g_maps.emplace(key, *map);
  }
  return rc;
}

// 2-D epilogue map over an output / residual / aux matrix [rows, cols] with
// leading dimension ld: box 32 rows x 128 bytes, 128-byte swizzle (the staging
// tile layout of epilogue_tile_tma).
struct EpiKey {
  const void* ptr;
  long long rows, cols, ld;
  int f32;
  bool operator==(const EpiKey& o) const {
    return ptr == o.ptr && rows == o.rows && cols == o.cols && ld == o.ld && f32 == o.f32;
  }
};
struct EpiKeyHash {
  size_t operator()(const EpiKey& k) const {
    size_t h = std::hash<const void*>()(k.ptr);
    for (long long v : {k.rows, k.cols, k.ld, (long long)k.f32}) h = h * 1000003u ^ std::hash<long long>()(v);
    return h;
  }
};
std::unordered_map<EpiKey, CUtensorMap, EpiKeyHash> g_epi_maps;

int make_epi_map(CUtensorMap* map, const void* ptr, long long rows, long long cols, long long ld,
                 bool f32) {
  const EpiKey key{ptr, rows, cols, ld, f32 ? 1 : 0};
  std::lock_guard<std::mutex> lk(g_map_mu);
  auto it = g_epi_maps.find(key);
  if (it != g_epi_maps.end()) {
    *map = it->second;
    return 0;
  }
  EncodeFn enc = encode_fn();
  DPN_REQUIRE(enc != nullptr, "cuTensorMapEncodeTiled unavailable");
  const int es = f32 ? 4 : 2;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * es)};
  cuuint32_t box[2] = {(cuuint32_t)(128 / es), 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  DPN_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled (epilogue) failed (code " + std::to_string((int)r) + ")");
  if (g_epi_maps.size() > 65536) g_epi_maps.clear();
  g_epi_maps.emplace(key, *map);
  return 0;
}

// 4-D map over a bf16 operand: (inner, z1, outer, z2); box (64, 1, box_outer, 1).
int encode_map(CUtensorMap* map, const void* ptr, long long inner, long long outer, long long ld,
               int Z1, long long s1, int Z2, long long s2, int box_outer) {
  EncodeFn enc = encode_fn();
  DPN_REQUIRE(enc != nullptr, "cuTensorMapEncodeTiled unavailable");
  DPN_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & 15) == 0, "operand base must be 16-byte aligned");
  DPN_REQUIRE(ld % 8 == 0 && s1 % 8 == 0 && s2 % 8 == 0,
              "operand strides must be multiples of 8 elements");
  cuuint64_t dims[4] = {(cuuint64_t)inner, (cuuint64_t)Z1, (cuuint64_t)outer, (cuuint64_t)Z2};
  // strides for dims 1..3 in bytes; degenerate batch dims get a harmless stride
  const long long safe1 = Z1 > 1 ? s1 : ld * outer;
  const long long safe2 = Z2 > 1 ? s2 : ld * outer;
  cuuint64_t strides[3] = {(cuuint64_t)(safe1 * 2), (cuuint64_t)(ld * 2), (cuuint64_t)(safe2 * 2)};
  cuuint32_t box[4] = {64, 1, (cuuint32_t)box_outer, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   DPN_GEMM_L2_PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  DPN_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (code " + std::to_string((int)r) + ")");
  return 0;
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BN, bool A_MN, bool B_MN, int CG>
int launch(const dpn_gemm_args* g, const GemmParams& p0, cudaStream_t stream) {
  using C = Cfg<BN, CG>;
  CUtensorMap ta, tb;
  const int Z1 = (int)g->batch1, Z2 = (int)g->batch2;
  int rc;
  if (!A_MN)  // multicast clusters fetch A in 64-row halves
    rc = make_map(&ta, g->A, g->K, g->M, g->lda, Z1, g->a_s1, Z2, g->a_s2, CG == 4 ? 64 : BM);
  else
    rc = make_map(&ta, g->A, g->M, g->K, g->lda, Z1, g->a_s1, Z2, g->a_s2, BK);
  if (rc) return rc;
  if (!B_MN)
    rc = make_map(&tb, g->B, g->K, g->N, g->ldb, Z1, g->b_s1, Z2, g->b_s2, C::kBRows);
  else
    rc = make_map(&tb, g->B, g->N, g->K, g->ldb, Z1, g->b_s1, Z2, g->b_s2, BK);
  if (rc) return rc;

  GemmParams p = p0;
  CUtensorMap tc{}, tr{}, tx{};
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  // the side staging tile holds either the residual or the aux output, not both
  p.tma_epi = g->batch1 * g->batch2 == 1 && (!p.res || (al16(p.res) && p.ldr % 8 == 0)) &&
              (!p.aux || al16(p.aux)) && !(p.res && p.aux && p.gelu) && g->epilogue != 1;
  DPN_REQUIRE(!p.colsum || (p.tma_epi && !p.c_f32),
              "colsum needs a bf16 output on the TMA-staged epilogue (unbatched, aligned operands)");
  if (p.tma_epi) {
    rc = make_epi_map(&tc, g->C, g->M, g->N, g->ldc, p.c_f32 != 0);
    if (!rc && p.res) rc = make_epi_map(&tr, p.res, g->M, g->N, p.ldr, false);
    if (!rc && p.aux) rc = make_epi_map(&tx, p.aux, g->M, g->N, g->ldc, false);
    if (rc) return rc;
  }
  p.tile_m = BM * C::kPair;
  p.tiles_m = (p.M + p.tile_m - 1) / p.tile_m;
  p.tiles_n = (p.N + BN - 1) / BN;
  if (CG == 4) p.tiles_n = (p.tiles_n + 1) / 2;  // a unit is two N-adjacent tiles
  const long long tiles = (long long)p.tiles_m * p.tiles_n * p.Z;
  const int nk = (p.K + BK - 1) / BK;
  static int clusters_max = 0;  // co-resident clusters of this configuration
  if (clusters_max == 0) {
    clusters_max = sm_count() / CG;
    if (CG > 2) {
      cudaLaunchConfig_t qc{};
      qc.gridDim = dim3((unsigned)(sm_count() / CG * CG));
      qc.blockDim = dim3(kThreads);
      qc.dynamicSmemBytes = C::kSmem;
      cudaLaunchAttribute qa[1];
      qa[0].id = cudaLaunchAttributeClusterDimension;
      qa[0].val.clusterDim.x = CG;
      qa[0].val.clusterDim.y = 1;
      qa[0].val.clusterDim.z = 1;
      qc.attrs = qa;
      qc.numAttrs = 1;
      int n = 0;
      cudaFuncSetAttribute(gemm_kernel<BN, A_MN, B_MN, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           C::kSmem);
      if (cudaOccupancyMaxActiveClusters(&n, gemm_kernel<BN, A_MN, B_MN, CG>, &qc) == cudaSuccess && n > 0)
        clusters_max = std::min(clusters_max, n);
      cudaGetLastError();
    }
  }
  int splits = 1;
  if (p.c_f32 && !p.bias && !p.res && !p.gelu && g->split_k != 1) {
    if (g->split_k > 1) {
      splits = g->split_k;
    } else {
      // minimise waves * k-blocks-per-unit (+ a small charge per extra split)
      double best = 1e30;
      for (int s = 1; s <= 8 && s <= nk; ++s) {
        const long long units = tiles * s;
        const double waves = (double)((units + clusters_max - 1) / clusters_max);
        const double cost = waves * ((nk + s - 1) / s) * (1.0 + 0.04 * (s - 1));
        if (cost < best - 1e-9) {
          best = cost;
          splits = s;
        }
      }
    }
  }
  p.kb_per_split = (nk + splits - 1) / splits;
  p.splits = (nk + p.kb_per_split - 1) / p.kb_per_split;
  p.units = tiles * p.splits;
  if (p.splits > 1 && !p.accumulate) {
    // split partials are reduced with red.add into a zeroed output
    for (long long z2 = 0; z2 < g->batch2; ++z2)
      for (long long z1 = 0; z1 < g->batch1; ++z1) {
        char* base = static_cast<char*>(g->C) + 4 * (z1 * g->c_s1 + z2 * g->c_s2);
        DPN_CHECK_CUDA(cudaMemset2DAsync(base, g->ldc * 4, 0, g->N * 4, g->M, stream));
      }
  }
  auto kern = gemm_kernel<BN, A_MN, B_MN, CG>;
  static bool attr_set = false;
  if (!attr_set) {
    DPN_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    attr_set = true;
  }
  const long long clusters = std::min<long long>(p.units, clusters_max);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(clusters * CG));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  DPN_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, tr, tx, p));
  return 0;
}

template <int BN, int CG>
int dispatch_major(const dpn_gemm_args* g, const GemmParams& p, cudaStream_t s) {
  if (!g->a_mn_major && !g->b_mn_major) return launch<BN, false, false, CG>(g, p, s);
  if (!g->a_mn_major && g->b_mn_major) return launch<BN, false, true, CG>(g, p, s);
  if (g->a_mn_major && !g->b_mn_major) return launch<BN, true, false, CG>(g, p, s);
  return launch<BN, true, true, CG>(g, p, s);
}

}  // namespace

// Tile configuration: (BN, CTA-group).  The 2-CTA 256 x 256 pair tile is the
// fastest per FLOP (measured, tools/gemm_micro.py: 1065-1402 TFLOP/s vs
// 700-880 for BN=128 at the pipeline shapes: a narrower tile pays the same
// per-tile fill / epilogue costs for half the MMA work), so it is used
// whenever N > 128; N <= 128 takes BN=128 (pair when M > 128); N <= 64 (the
// attention products with N = head_dim) stays single-CTA BN=64.
// The CTA pair is used for every N > 128 tile with M > 128.  In isolation
// single-CTA 128x256 tiles win on small problems (620 vs 567 TFLOP/s at
// 4096x1024x1024, profiles/r01_gemm_micro_multicast.jsonl), but switching to
// them below 256 pair tiles x 16 k-blocks lowered the in-pipeline GEMM rate
// (GPT-2 XL 923 -> 854 TFLOP/s, BERT-large b=8 unchanged), so it is not done.
void pick_config(long long M, long long N, long long K, long long Z, int& bn, int& cg) {
  if (N <= 64) {
    bn = 64;
    cg = 1;
  } else if (N <= 128) {
    bn = 128;
    cg = M > 128 ? 2 : 1;
  } else {
    bn = 256;
    const long long pair_tiles = ((M + 255) / 256) * ((N + 255) / 256) * Z;
    const long long nk = (K + BK - 1) / BK;
    (void)pair_tiles;
    (void)nk;
    cg = M > 128 ? 2 : 1;
  }
}

}  // namespace dpn

static long long* g_gemm_trace = nullptr;
extern "C" void dpn_gemm_debug_trace(void* buf) { g_gemm_trace = static_cast<long long*>(buf); }

extern "C" int dpn_gemm(const dpn_gemm_args* g, void* stream_) {
  using namespace dpn;
  DPN_REQUIRE(g != nullptr, "null args");
  DPN_REQUIRE(g->M > 0 && g->N > 0 && g->K > 0, "M, N, K must be positive");
  DPN_REQUIRE(g->batch1 >= 1 && g->batch2 >= 1, "batch extents must be >= 1");
  DPN_REQUIRE(g->A && g->B && g->C, "null operand");
  DPN_REQUIRE(g->c_dtype == kF32 || g->c_dtype == kBF16, "c_dtype must be 0 (f32) or 1 (bf16)");
  DPN_REQUIRE(!g->accumulate || g->c_dtype == kF32, "accumulate requires an f32 output");
  DPN_REQUIRE(g->ldc % 8 == 0 && g->N <= g->ldc, "ldc must be >= N and a multiple of 8");
  DPN_REQUIRE(!g->aux || g->gelu, "aux output is the pre-GELU value; requires gelu");
  DPN_REQUIRE(g->residual_mode == 0 || (g->residual_mode == 1 && g->residual && !g->gelu),
              "residual_mode 1 (x gelu'(residual)) needs a residual and no forward GELU");
  DPN_REQUIRE((reinterpret_cast<uintptr_t>(g->C) & 15) == 0, "C must be 16-byte aligned");
  DPN_REQUIRE(g->split_k >= 0 && g->split_k <= 64, "split_k must be in [0, 64]");
  GemmParams p{};
  p.M = (int)g->M;
  p.N = (int)g->N;
  p.K = (int)g->K;
  p.Z1 = (int)g->batch1;
  p.Z = (int)(g->batch1 * g->batch2);
  p.C = g->C;
  p.ldc = g->ldc;
  p.c_s1 = g->c_s1;
  p.c_s2 = g->c_s2;
  p.c_f32 = g->c_dtype == kF32;
  p.accumulate = g->accumulate;
  p.bias = static_cast<const __nv_bfloat16*>(g->bias);
  p.res = static_cast<const __nv_bfloat16*>(g->residual);
  p.ldr = g->ldr;
  p.r_s1 = g->r_s1;
  p.r_s2 = g->r_s2;
  p.res_mode = g->residual_mode;
  p.aux = static_cast<__nv_bfloat16*>(g->aux);
  p.alpha = g->alpha;
  p.gelu = g->gelu;
  p.trace = g_gemm_trace;
  p.colsum = g->colsum;
  DPN_REQUIRE(!g->colsum || (reinterpret_cast<uintptr_t>(g->colsum) & 7) == 0, "colsum must be 8-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream_);
  int bn = 0, cg = 1;
  pick_config(g->M, g->N, g->K, p.Z, bn, cg);
  if (g->block_n > 0) {
    bn = g->block_n;
    cg = g->cta_group > 0 ? g->cta_group : (bn >= 128 && g->M > 128 ? 2 : 1);
  } else if (g->cta_group > 0) {
    cg = g->cta_group;
  }
  DPN_REQUIRE(cg == 1 || (cg == 2 && bn >= 128) || (cg == 4 && bn == 256),
              "cta_group 2 needs block_n 128 or 256; 4 (two multicast pairs) block_n 256");
  switch (bn * 10 + cg) {
    case 641: return dispatch_major<64, 1>(g, p, s);
    case 1281: return dispatch_major<128, 1>(g, p, s);
    case 2561: return dispatch_major<256, 1>(g, p, s);
    case 1282: return dispatch_major<128, 2>(g, p, s);
    case 2562: return dispatch_major<256, 2>(g, p, s);
    case 2564: return dispatch_major<256, 4>(g, p, s);
    default: DPN_REQUIRE(false, "block_n must be 0, 64, 128 or 256; cta_group 0, 1, 2 or 4");
  }
}
