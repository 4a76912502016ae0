// Fused attention (flash-style) for sm_100a: tcgen05 MMAs with S / O tiles in
// TMEM, online softmax in registers, P staged in shared memory (128-byte
// swizzled, the layout the next MMA reads), Q/K/V tiles fetched by TMA straight
// out of the fused [b*s, 3H] QKV buffer.  The s x s probability matrix never
// touches HBM (the unfused `score` node writes b*heads*s^2 bf16 and reads it
// back three times).
//
// Forward: persistent, one CTA per SM walking work units (batch, head,
// 128-query tile) -- longest causal units first -- with every barrier phase
// and TMEM / smem buffer indexed by a CTA-global tile counter, so the next
// unit's Q / K / V loads and S MMAs overlap the current unit's tail (the
// per-unit prologue / epilogue of a one-CTA-per-unit grid dominated at
// s = 512).  384 threads:
//   warp 0   TMA: Q per unit, double-buffered by unit parity (with one buffer
//            the next Q could only load after the unit's last S MMA, and the
//            MMA warp -- which issues PV(j-1) after S(j) -- held the unit's
//            last PV, and the softmax warps' unit epilogue, for a TMA round
//            trip), K_j / V_j tiles into a 3-deep ring
//   warp 1   MMA issuer: S_j = Q K_j^T (M=128,N=128,K=64) into TMEM S[j%2];
//            O_j = P_j V_j (M=128,N=64,K=128) into TMEM O[j%2]
//   warp 2   TMEM allocator
//   warps 4-11 softmax, two warps per query row: warp w reads TMEM lanes
//            32*(w%4).. (its 32 rows) and key half (w-4)/4 -- 64 keys of S_j.
//            Each key half keeps its own running max and sum and writes its
//            64-key swizzle atom of P_j = exp2(S_j*scale*log2e - m_half); the
//            MMA accumulates O_half += P_half V_half in TMEM (two K=64 chains),
//            so there is no per-tile exchange between the halves and no O in
//            registers.  A half's max is only raised when it grows by more than
//            2^8 (conditional rescaling); then that warp rescales its O_half
//            rows in TMEM (tcgen05.ld / st) before releasing P_j.  Per unit the
//            halves exchange (m, l) once and combine the two accumulators into
//            O / l (bf16) and the natural-log LSE (fp32, for the backward).
// head_dim is 64 (one 128-byte swizzle row).
#include "common.cuh"
#include "../../include/dawnpiper.h"

#include <algorithm>
#include <mutex>
#include <type_traits>

namespace dpn {
namespace {

#ifndef DPN_ATTN_POLY
#define DPN_ATTN_POLY 0  // key pairs of every 4 exponentiated by exp2_fma2 in the forward (A/B: slower)
#endif
#ifndef DPN_ATTN_PACK_ALU
#define DPN_ATTN_PACK_ALU 0  // 1: the forward packs P to bf16 on the integer ALU instead of F2FP
#endif
#ifndef DPN_ATTN_POLY_BWD
#define DPN_ATTN_POLY_BWD 0  // the same for the backward's recomputed P
#endif
constexpr int kTile = 128;  // queries per CTA and keys per KV tile
constexpr int kD = 64;
constexpr int kKVStages = 3;
constexpr int kTileBytes = kTile * kD * 2;  // 16 KB (128 rows x 128 B)
constexpr int kPBytes = kTile * kTile * 2;  // 32 KB (two 64-key swizzle atoms)
constexpr int kFwdThreads = 384;
constexpr float kRescaleLog2 = 8.f;  // raise the running max only past 2^8
constexpr float kLog2e = 1.4426950408889634f;

struct AttnParams {
  int batch, seq, heads, H;  // seq = query rows per sequence; H = heads * 64
  int kv_seq;                // key rows per sequence (== seq for self-attention)
  int q_col, k_col, v_col;   // column of head 0's Q / K / V in its buffer
  float scale_log2;          // softmax scale * log2(e)
  float scale;
  int causal;
  __nv_bfloat16* out;  // [b*s, H]
  float* lse;          // [b, heads, s] natural-log LSE of scale * S
};

// byte offset of (row, 16-byte chunk) inside a 128-row x 128-byte SW128 atom
__device__ __forceinline__ uint32_t sw128(int row, int chunk) {
  return (uint32_t)(row * 128 + ((chunk ^ (row & 7)) << 4));
}

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}


__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

template <uint32_t N>
__device__ __forceinline__ void regs_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}
template <uint32_t N>
__device__ __forceinline__ void regs_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}

__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
      "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
      "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// KS = key splits per row: KS softmax warps share each TMEM lane quarter, each
// owning 128 / KS keys of every tile with its own running max, sum and O
// accumulator.  KS = 2: 8 softmax warps, O double-buffered by unit parity;
// KS = 4: 16 softmax warps (latency hiding for the softmax chain), one O set.
template <int KS>
__global__ void __launch_bounds__(128 + 128 * KS, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kv,
                    const AttnParams p) {
  static_assert(KS == 2 || KS == 4, "key splits");
  constexpr int kKeys = kTile / KS;         // keys per split
  constexpr int kSoftWarps = 4 * KS;
  constexpr int kOBufs = KS == 2 ? 2 : 1;   // O accumulator sets (by unit parity)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;                             // [2] by unit parity: the next
                                                  // unit's Q loads during this one
  uint8_t* sK = sQ + 2 * kTileBytes;              // [stage] 16 KB
  uint8_t* sV = sK + kKVStages * kTileBytes;      // [stage] 16 KB
  uint8_t* sP = sV + kKVStages * kTileBytes;      // [2] 32 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 2 * kPBytes);
  uint64_t* q_full = bars;                  // [2]
  uint64_t* kv_full = bars + 2;
  uint64_t* kv_empty = kv_full + kKVStages;
  uint64_t* s_full = kv_empty + kKVStages;  // [2]
  uint64_t* s_empty = s_full + 2;           // [2]
  uint64_t* p_full = s_empty + 2;           // [2]
  uint64_t* p_empty = p_full + 2;           // [2]
  uint64_t* pv_done = p_empty + 2;          // one phase per KV tile
  uint64_t* o_empty = pv_done + 1;          // [2] by unit parity
  uint64_t* q_empty = o_empty + 2;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_kv_all = (p.kv_seq + kTile - 1) / kTile;
  const int n_qt = (p.seq + kTile - 1) / kTile;
  const long long bh = (long long)p.batch * p.heads;
  const long long units = bh * n_qt;
  // unit -> (query tile, head, batch); query tiles outermost, longest first
  auto decode = [&](long long u, int& qt, int& h, int& bb) {
    // non-causal: query tiles fastest (concurrent CTAs share a head's K / V in
    // L2); causal: query tiles outermost, longest first (balances the CTAs)
    int qi;
    long long r;
    if (p.causal) {
      qi = (int)(u / bh);
      r = u - (long long)qi * bh;
    } else {
      qi = (int)(u % n_qt);
      r = u / n_qt;
    }
    qt = p.causal ? n_qt - 1 - qi : qi;
    h = (int)(r % p.heads);
    bb = (int)(r / p.heads);
  };
  auto kv_tiles = [&](int qt) { return p.causal ? min(n_kv_all, qt + 1) : n_kv_all; };

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_q);
    prefetch_tmap(&tm_kv);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    for (int s = 0; s < kKVStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], kSoftWarps);  // one arrival per softmax warp
      mbar_init(&p_full[i], kSoftWarps);
      mbar_init(&p_empty[i], 1);
      mbar_init(&o_empty[i], kSoftWarps);
    }
    mbar_init(pv_done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  // TMEM columns: S[0] 0..127, S[1] 128..255; O[unit parity][key split] at
  // 256 + 128 * parity + 64 * split (KS = 2) or 256 + 64 * split (KS = 4), 64
  // columns each.  Each key split keeps its own running max: O_split
  // accumulates P_split V_split in TMEM (rescaled in place on the rare tiles
  // where that split's max grows by more than 2^8), and the splits are
  // combined once per unit.

  if (warp == 0) {
    if (lane == 0) {
      int g = 0, uc = 0;  // CTA-global KV tile / unit counters
      for (long long u = blockIdx.x; u < units; u += gridDim.x, ++uc) {
        int qt, h, bb;
        decode(u, qt, h, bb);
        const int n_kv = kv_tiles(qt), row0 = bb * p.seq, krow0 = bb * p.kv_seq;
        const int qb = uc & 1;
        mbar_wait(&q_empty[qb], ((uc >> 1) & 1) ^ 1);
        mbar_expect_tx(&q_full[qb], kTileBytes);
        tma_load_2d(sQ + qb * kTileBytes, &tm_q, &q_full[qb], p.q_col + h * kD, row0 + qt * kTile);
        for (int j = 0; j < n_kv; ++j, ++g) {
          const int st = g % kKVStages;
          mbar_wait(&kv_empty[st], ((g / kKVStages) & 1) ^ 1);
          mbar_expect_tx(&kv_full[st], 2 * kTileBytes);
          tma_load_2d(sK + st * kTileBytes, &tm_kv, &kv_full[st], p.k_col + h * kD, krow0 + j * kTile);
          tma_load_2d(sV + st * kTileBytes, &tm_kv, &kv_full[st], p.v_col + h * kD, krow0 + j * kTile);
        }
      }
    }
  } else if (warp == 1) {
    // S = Q K^T: A = Q (K-major, K = d), B = K_j (K-major over d)
    constexpr uint32_t idesc_s = idesc_bf16(128, 128, 0, 0);
    // O_half += P_half V_half: A = P key-half atom (K-major, 64 keys), B = V rows of that
    // half (MN-major: d contiguous)
    constexpr uint32_t idesc_o = idesc_bf16(128, 64, 0, 1);
    // PV of global tile t (issued one tile late); first / ub describe t's unit
    auto issue_pv = [&](int t, bool first, int ub, int ucount) {
      const int i = t & 1;
      mbar_wait(&p_full[i], (t >> 1) & 1);
      if (first) mbar_wait(&o_empty[ub], ((ucount / kOBufs) & 1) ^ 1);
      tc_fence_after();
      if (lane == 0) {
        const int st = t % kKVStages;
        const uint32_t pa = smem_u32(sP + i * kPBytes), vb = smem_u32(sV + st * kTileBytes);
#pragma unroll
        for (int k = 0; k < kTile / 16; ++k) {
          const uint64_t ad = smem_desc_sw128(pa + (k >> 2) * (kPBytes / 2) + (k & 3) * 32, 16, 1024);
          const uint64_t bd = smem_desc_sw128(vb + k * 2048, kD * 128, 1024);
          constexpr int kSteps = kKeys / 16;  // K=16 steps per key split
          umma_bf16(tmem + 256 + ub * 128 + (k / kSteps) * 64, ad, bd, idesc_o,
                    (first && (k % kSteps) == 0) ? 0u : 1u);
        }
        umma_commit(&p_empty[i]);
        umma_commit(&kv_empty[st]);
        umma_commit(pv_done);
      }
      __syncwarp();
    };
    int g = 0, uc = 0;
    bool prev_first = false;
    int prev_ub = 0, prev_uc = 0;
    for (long long u = blockIdx.x; u < units; u += gridDim.x, ++uc) {
      int qt, h, bb;
      decode(u, qt, h, bb);
      const int n_kv = kv_tiles(qt);
      const int qb = uc & 1;
      mbar_wait(&q_full[qb], (uc >> 1) & 1);
      for (int j = 0; j < n_kv; ++j, ++g) {
        const int st = g % kKVStages, i = g & 1;
        mbar_wait(&kv_full[st], (g / kKVStages) & 1);
        mbar_wait(&s_empty[i], ((g >> 1) & 1) ^ 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t qa = smem_u32(sQ + qb * kTileBytes), kb = smem_u32(sK + st * kTileBytes);
#pragma unroll
          for (int k = 0; k < kD / 16; ++k) {
            const uint64_t ad = smem_desc_sw128(qa + k * 32, 16, 1024);
            const uint64_t bd = smem_desc_sw128(kb + k * 32, 16, 1024);
            umma_bf16(tmem + i * 128, ad, bd, idesc_s, k > 0 ? 1u : 0u);
          }
          umma_commit(&s_full[i]);
          if (j == n_kv - 1) umma_commit(&q_empty[qb]);  // Q is free once the unit's S MMAs ran
        }
        __syncwarp();
        if (g >= 1) issue_pv(g - 1, prev_first, prev_ub, prev_uc);
        prev_first = j == 0;
        prev_ub = KS == 2 ? (uc & 1) : 0;
        prev_uc = uc;
      }
    }
    if (g >= 1) issue_pv(g - 1, prev_first, prev_ub, prev_uc);
  } else if (warp >= 4) {
    // ---------------- softmax ----------------
    const int quarter = warp & 3, half = (warp - 4) >> 2;  // half: key split
    const int r = quarter * 32 + lane;  // query row within the tile (== TMEM lane)
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    float* xs = reinterpret_cast<float*>(tmem_slot + 4);  // [2 units][128 rows][half][m, l]
    const float sl = p.scale_log2;
    int g = 0, uc = 0;
    for (long long u = blockIdx.x; u < units; u += gridDim.x, ++uc) {
      int qt, h, bb;
      decode(u, qt, h, bb);
      const int n_kv = kv_tiles(qt), row0 = bb * p.seq, ub = KS == 2 ? (uc & 1) : 0;
      const int q = qt * kTile + r;
      const uint32_t o_half = tmem + 256 + ub * 128 + half * 64 + lane_off;
      float ms = -INFINITY;  // this key half's running max, scaled log2 units
      float l = 0.f;         // this key half's running sum
      for (int j = 0; j < n_kv; ++j) {
        const int gj = g + j, i = gj & 1;
        const int k0 = j * kTile + half * kKeys;
        const bool mask = (j + 1) * kTile > p.kv_seq || (p.causal && j == qt);
        mbar_wait(&s_full[i], (gj >> 1) & 1);
        tc_fence_after();
        float s[kKeys];
        {
          uint32_t uu[kKeys];
#pragma unroll
          for (int c = 0; c < kKeys / 32; ++c)
            tmem_ld_32x32b_x32(tmem + i * 128 + half * kKeys + c * 32 + lane_off, uu + c * 32);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < kKeys; ++e) s[e] = __uint_as_float(uu[e]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[i]);
        if (mask) {
#pragma unroll
          for (int c = 0; c < kKeys; ++c) {
            const int key = k0 + c;
            if (!(key < p.kv_seq && (!p.causal || key <= q))) s[c] = -INFINITY;
          }
        }
        float mx = s[0];
#pragma unroll
        for (int c = 1; c < kKeys; ++c) mx = fmaxf(mx, s[c]);
        mx *= sl;
        float alpha = 1.f;
        if (mx > ms + kRescaleLog2 || ms == -INFINITY) {
          alpha = (ms == -INFINITY) ? 0.f : ex2(ms - mx);
          ms = mx;
        }
        const float base = (ms == -INFINITY) ? 0.f : ms;
        float2 sum2 = make_float2(0.f, 0.f);
        mbar_wait(&p_empty[i], ((gj >> 1) & 1) ^ 1);
        // this split's keys: atom half * kKeys / 64, 16-byte chunks from (half * kKeys % 64) / 8
        uint8_t* pt = sP + i * kPBytes + (half * kKeys / 64) * (kPBytes / 2);
        constexpr int kChunk0Mul = kKeys / 8;  // chunks per split
#pragma unroll
        for (int cc = 0; cc < kKeys / 8; ++cc) {
          const int c = cc + (half * kChunk0Mul) % 8;  // chunk within the 64-key atom
          float e8[8];
#pragma unroll
          for (int e = 0; e < 8; e += 2) {  // two keys per packed f32x2 instruction
            const float2 a = fma2(make_float2(s[cc * 8 + e], s[cc * 8 + e + 1]), make_float2(sl, sl),
                                  make_float2(-base, -base));
            // DPN_ATTN_POLY of every 4 key pairs exponentiate on the FMA pipe: the
            // MUFU (XU) pipe is the forward's limiter (ncu: XU 99% busy)
            const float2 ev = e >= 2 * (4 - DPN_ATTN_POLY) ? exp2_fma2(a) : make_float2(ex2(a.x), ex2(a.y));
            e8[e] = ev.x;
            e8[e + 1] = ev.y;
            sum2 = fma2(make_float2(1.f, 1.f), ev, sum2);
          }
          uint4 w;
#if DPN_ATTN_PACK_ALU
          w.x = pack_bf16_alu(e8[0], e8[1]);
          w.y = pack_bf16_alu(e8[2], e8[3]);
          w.z = pack_bf16_alu(e8[4], e8[5]);
          w.w = pack_bf16_alu(e8[6], e8[7]);
#else
          w.x = pack_bf16(e8[0], e8[1]);
          w.y = pack_bf16(e8[2], e8[3]);
          w.z = pack_bf16(e8[4], e8[5]);
          w.w = pack_bf16(e8[6], e8[7]);
#endif
          sts128(smem_u32(pt) + sw128(r, c), w);
        }
        l = l * alpha + (sum2.x + sum2.y);
        fence_async_smem();
        if (j > 0) {
          // O_half holds tiles < j once PV(j-1) is done; rescale rows whose max grew
          mbar_wait(pv_done, (gj - 1) & 1);
          if (__any_sync(0xffffffffu, alpha != 1.f)) {
            tc_fence_after();
            uint32_t ou[64];
            tmem_ld_32x32b_x32(o_half, ou);
            tmem_ld_32x32b_x32(o_half + 32, ou + 32);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 64; ++e) ou[e] = __float_as_uint(__uint_as_float(ou[e]) * alpha);
            tmem_st_32x32b_x32(o_half, ou);
            tmem_st_32x32b_x32(o_half + 32, ou + 32);
            tmem_st_wait();
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[i]);
      }
      // ---- unit epilogue: combine the key halves ----
      mbar_wait(pv_done, (g + n_kv - 1) & 1);
      tc_fence_after();
      // per unit exchange of the splits' (m, l): [unit parity][row][split][2]
      float* xm = xs + ub * (128 * KS * 2) + r * (KS * 2);
      xm[half * 2] = ms;
      xm[half * 2 + 1] = l;
      asm volatile("bar.sync %0, %1;" ::"r"(1 + quarter), "r"(32 * KS) : "memory");
      float m = -INFINITY;
#pragma unroll
      for (int k = 0; k < KS; ++k) m = fmaxf(m, xm[2 * k]);
      float a[KS], lt = 0.f;
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        a[k] = xm[2 * k] == -INFINITY ? 0.f : ex2(xm[2 * k] - m);
        lt += xm[2 * k + 1] * a[k];
      }
      // this warp writes output columns half * 64/KS .. from every split's accumulator
      constexpr int kCols = 64 / KS;
      float v[kCols];
#pragma unroll
      for (int e = 0; e < kCols; ++e) v[e] = 0.f;
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        uint32_t o[32];
        tmem_ld_32x32b_x32(tmem + 256 + ub * 128 + k * 64 + (half * kCols) / 32 * 32 + lane_off, o);
        tmem_ld_wait();
        const int off = (half * kCols) % 32;
#pragma unroll
        for (int e = 0; e < kCols; ++e) v[e] = fmaf(__uint_as_float(o[off + e]), a[k], v[e]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[ub]);
      if (q < p.seq) {
        const float inv = lt > 0.f ? 1.f / lt : 0.f;
        __nv_bfloat16* op = p.out + (long long)(row0 + q) * p.H + h * kD + half * kCols;
#pragma unroll
        for (int c = 0; c < kCols / 8; ++c) {
          uint4 w;
          w.x = pack_bf16(v[c * 8 + 0] * inv, v[c * 8 + 1] * inv);
          w.y = pack_bf16(v[c * 8 + 2] * inv, v[c * 8 + 3] * inv);
          w.z = pack_bf16(v[c * 8 + 4] * inv, v[c * 8 + 5] * inv);
          w.w = pack_bf16(v[c * 8 + 6] * inv, v[c * 8 + 7] * inv);
          reinterpret_cast<uint4*>(op)[c] = w;
        }
        // natural-log LSE of scale * S:  (m + log2 l) / log2(e)
        if (half == 0) p.lse[((long long)bb * p.heads + h) * p.seq + q] = (m + log2f(lt)) / kLog2e;
      }
      g += n_kv;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

// Experimental forward kernels measured and removed (git history, commit
// c58a59f and earlier): two softmax sets of 8 warps each owning alternate KV
// tiles (106.9 vs 87.5 us at b32: 18 warps spill at 96 registers) and two sets
// of whole-row warps with setmaxnreg (112.7 vs 85 us); DESIGN.md section 6.

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode2() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* q = nullptr;
    cudaDriverEntryPointQueryResult r;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &r) == cudaSuccess &&
        r == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(q);
  });
  return fn;
}

// 2-D map over a bf16 [rows, cols] buffer, box 64 columns x 128 rows, SW128.
int map_2d(CUtensorMap* map, const void* ptr, long long rows, long long cols) {
  EncodeFn enc = encode2();
  DPN_REQUIRE(enc != nullptr, "cuTensorMapEncodeTiled unavailable");
  DPN_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & 15) == 0 && cols % 8 == 0, "16-byte alignment");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(cols * 2)};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  DPN_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed");
  return 0;
}

// 2-D map over the f32 dQ accumulator [rows, cols], box 32 columns x 128 rows
// (128 bytes wide), SW128 -- the TMA reduce-add target of the backward.
int map_2d_f32(CUtensorMap* map, const void* ptr, long long rows, long long cols) {
  EncodeFn enc = encode2();
  DPN_REQUIRE(enc != nullptr, "cuTensorMapEncodeTiled unavailable");
  DPN_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & 15) == 0 && cols % 4 == 0, "16-byte alignment");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(cols * 4)};
  cuuint32_t box[2] = {32, 128};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  DPN_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed");
  return 0;
}

// + 256 B of barriers / TMEM slot, then the per-unit (m, l) exchange [2][128][2][2] f32
constexpr int kFwdSmem = 1024 + kTileBytes * (2 + 2 * kKVStages) + 2 * kPBytes + 256 + 1024 * 4;

// Forward kernel choice (tools/attn_micro.py A/B).
struct FwdKernel {
  void (*fn)(CUtensorMap, CUtensorMap, AttnParams);
  int threads, smem;
};
FwdKernel fwd_kernel() {
  static FwdKernel k = [] {
    const char* e = getenv("DPN_ATTN_FWD");
    // DPN_ATTN_FWD=4: four key splits per row (16 softmax warps; measured 2x
    // slower, kept for A/B), else two
    FwdKernel r = (e && e[0] == '4') ? FwdKernel{attn_fwd_kernel<4>, 128 + 128 * 4, kFwdSmem}
                                     : FwdKernel{attn_fwd_kernel<2>, kFwdThreads, kFwdSmem};
    cudaFuncSetAttribute(r.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, r.smem);
    return r;
  }();
  return k;
}

}  // namespace

// ---------------------------------------------------------------------------
// Backward: persistent, one CTA per SM walking units (batch, head, 128-key
// tile) -- K_j, V_j stay in smem while the CTA walks the query tiles i (K
// double-buffered by unit parity and V released after the unit's last dP MMA,
// so the next unit's K / V load under this one instead of after it)
// (causal: i >= j); barrier phases run on CTA-global counters, the dV / dK
// drain of a unit runs on the dQ warpgroup while the softmax warps start the
// next unit:
//   S = Q_i K_j^T, dP = dO_i V_j^T                  (TMEM, M = queries)
//   P = exp(scale*S - lse), dS = scale * P * (dP - D_i)   (softmax warps ->
//       bf16 in 128-byte swizzled smem, double-buffered)
//   dV += P^T dO_i, dK += dS^T Q_i                   (TMEM accumulators, M = keys;
//       P^T / dS^T are the same smem tiles read MN-major)
//   dQ_i = dS K_j                                    (TMEM -> swizzled f32 smem ->
//       TMA reduce-add into the f32 dQ accumulator)
// D_i = rowsum(dO_i * O_i) comes from attn_bwd_prep.
//
// 512 threads, four warpgroups with re-balanced registers (setmaxnreg):
//   WG0  warp 0 TMA (K/V once, Q/dO double-buffered), warp 1 MMA issuer,
//        warp 2 TMEM allocator                                    (56 regs)
//   WG1-2 softmax: warp w owns rows 32*(w%4).. and key half (w-4)/4   (184 regs)
//   WG3  dQ drain: TMEM dQ -> smem staging -> cp.reduce.async.bulk.tensor
//        (.add), off the softmax critical path                    (88 regs)
// MMA issue order per query tile: S/dP(i+1) as soon as the softmax holds
// S/dP(i) in registers, then dV(i), dQ(i), dK(i).  dS is double-buffered in
// smem, P single-buffered (stored last, after dV(i-1) released it).
namespace {

constexpr int kBwdThreads = 512;
// Q / dO ring depth and dS buffers (smem allows 2 + 2 or 3 + 1).  The softmax
// warps spend about half their time waiting for S / dP (ncu, profiles/
// r02s3_final_ncu.md); a 3-deep Q / dO ring with a single dS buffer measured
// slower (218.9 vs 215 us at b32), so the wait is not the Q / dO load.
constexpr int kQStages = 2;
constexpr int kDSBufs = 2;

struct AttnBwdParams {
  int batch, seq, heads, H;  // seq = query rows per sequence
  int kv_seq;                // key rows per sequence
  int q_col, k_col, v_col;   // column of head 0's Q / K / V in its buffer
  __nv_bfloat16* dk;         // dK / dV of head 0, row stride dkv_ld
  __nv_bfloat16* dv;
  long long dkv_ld;
  float scale, scale_log2;
  int causal;
  const float* lse;  // [b, heads, s]
  const float* D;    // [b, heads, s]
  float* dq;         // [b*s, H] f32 accumulator (zeroed)
  __nv_bfloat16* dqkv;  // [b*s, 3H]
  float* dbias_k;       // optional: += column sums of dK / dV (head 0's column 0), the
  float* dbias_v;       // fused QKV projection's bias gradient
};


__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tm_qkv,
                    const __grid_constant__ CUtensorMap tm_kv,
                    const __grid_constant__ CUtensorMap tm_do,
                    const __grid_constant__ CUtensorMap tm_dq, const AttnBwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sK = smem;                     // [2] by unit parity: the next unit's K loads
                                          // during this one
  uint8_t* sV = sK + 2 * kTileBytes;      // released after the unit's last dP MMA
  uint8_t* sQ = sV + kTileBytes;          // [kQStages]
  uint8_t* sdO = sQ + kQStages * kTileBytes;  // [kQStages]
  uint8_t* sP = sdO + kQStages * kTileBytes;  // 32 KB
  uint8_t* sdS = sP + kPBytes;            // [kDSBufs] 32 KB
  uint8_t* sdQ = sdS + kDSBufs * kPBytes; // 16 KB f32 staging: one [128][32] SW128 box
  uint64_t* bars = reinterpret_cast<uint64_t*>(sdQ + kPBytes / 2);
  uint64_t* k_full = bars;        // [2]
  uint64_t* v_full = bars + 2;
  uint64_t* q_full = bars + 3;    // [kQStages]
  uint64_t* q_empty = q_full + kQStages; // [kQStages]
  uint64_t* sp_full = q_empty + kQStages;
  uint64_t* sp_loaded = sp_full + 1;
  uint64_t* p_empty = sp_loaded + 1;
  uint64_t* ds_full = p_empty + 1;  // [kDSBufs]
  uint64_t* ds_empty = ds_full + kDSBufs; // [kDSBufs]
  uint64_t* dq_full = ds_empty + kDSBufs;  // [2] (dQ is double-buffered in TMEM)
  uint64_t* dq_empty = dq_full + 2;  // [2]
  uint64_t* dkv_full = dq_empty + 2;
  uint64_t* k_empty = dkv_full + 1;    // [2] K smem free for the unit after next
  uint64_t* v_empty = k_empty + 2;     // V smem free (the unit's dP MMAs ran)
  uint64_t* dkv_empty = v_empty + 1;   // dV/dK TMEM drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dkv_empty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_q = (p.seq + kTile - 1) / kTile;
  const int n_k = (p.kv_seq + kTile - 1) / kTile;
  const long long bh = (long long)p.batch * p.heads;
  const long long units = bh * n_k;
  // unit -> (key tile, head, batch).  Every barrier phase below runs on CTA-global counters
  // (units uc, query iterations G) so a unit's tail overlaps the next one.
  struct Unit {
    int kt, h, bb, k0, i0, n_it, row0, krow0;
  };
  auto decode = [&](long long u) {
    Unit w;
    // non-causal: key tiles fastest, so concurrently running CTAs walk the same
    // (batch, head)'s query / dO tiles, which then stay in L2; causal: key tiles
    // outermost, ascending -- the longest units first balance the CTAs
    long long r;
    if (p.causal) {
      w.kt = (int)(u / bh);
      r = u - (long long)w.kt * bh;
    } else {
      w.kt = (int)(u % n_k);
      r = u / n_k;
    }
    w.h = (int)(r % p.heads);
    w.bb = (int)(r / p.heads);
    w.k0 = w.kt * kTile;
    w.i0 = p.causal ? w.kt : 0;
    w.n_it = n_q - w.i0;
    w.row0 = w.bb * p.seq;
    w.krow0 = w.bb * p.kv_seq;
    return w;
  };

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_qkv);
    prefetch_tmap(&tm_kv);
    prefetch_tmap(&tm_do);
    prefetch_tmap(&tm_dq);
  }
  if (warp == 1 && lane == 0) {
    mbar_init(&k_full[0], 1);
    mbar_init(&k_full[1], 1);
    mbar_init(&k_empty[0], 1);
    mbar_init(&k_empty[1], 1);
    mbar_init(v_full, 1);
    mbar_init(v_empty, 1);
    mbar_init(sp_loaded, 8);
    mbar_init(p_empty, 1);
    for (int s = 0; s < kQStages; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
    }
    for (int s = 0; s < kDSBufs; ++s) {
      mbar_init(&ds_full[s], 8);
      mbar_init(&ds_empty[s], 1);
    }
    mbar_init(sp_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&dq_full[s], 1);
      mbar_init(&dq_empty[s], 4);
    }
    mbar_init(dkv_full, 1);
    mbar_init(dkv_empty, 4);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  // TMEM columns: S 0..127, dP 128..255, dV 256..319, dK 320..383, dQ[2] 384..511

  if (warp < 4) {
    regs_dec<56>();
    if (warp == 0 && lane == 0) {
      int G = 0, uc = 0;
      for (long long u = blockIdx.x; u < units; u += gridDim.x, ++uc) {
        const Unit w = decode(u);
        const int kb = uc & 1;
        mbar_wait(&k_empty[kb], ((uc >> 1) & 1) ^ 1);
        mbar_expect_tx(&k_full[kb], kTileBytes);
        tma_load_2d(sK + kb * kTileBytes, &tm_kv, &k_full[kb], p.k_col + w.h * kD, w.krow0 + w.k0);
        mbar_wait(v_empty, (uc & 1) ^ 1);
        mbar_expect_tx(v_full, kTileBytes);
        tma_load_2d(sV, &tm_kv, v_full, p.v_col + w.h * kD, w.krow0 + w.k0);
        for (int it = 0; it < w.n_it; ++it, ++G) {
          const int st = G % kQStages, i = w.i0 + it;
          mbar_wait(&q_empty[st], ((G / kQStages) & 1) ^ 1);
          mbar_expect_tx(&q_full[st], 2 * kTileBytes);
          tma_load_2d(sQ + st * kTileBytes, &tm_qkv, &q_full[st], p.q_col + w.h * kD, w.row0 + i * kTile);
          tma_load_2d(sdO + st * kTileBytes, &tm_do, &q_full[st], w.h * kD, w.row0 + i * kTile);
        }
      }
    } else if (warp == 1) {
      constexpr uint32_t id_s = idesc_bf16(128, 128, 0, 0);   // S, dP
      constexpr uint32_t id_kv = idesc_bf16(128, 64, 1, 1);   // dV, dK: A^T and B MN-major
      constexpr uint32_t id_q = idesc_bf16(128, 64, 0, 1);    // dQ: dS K-major, K_j MN-major
      // S / dP of query iteration G against K[kbuf]; `last`: the unit's last use of V
      auto issue_sdp = [&](int G, int kbuf, bool last) {
        const int st = G % kQStages;
        mbar_wait(&q_full[st], (G / kQStages) & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t qa = smem_u32(sQ + st * kTileBytes), doa = smem_u32(sdO + st * kTileBytes);
          const uint32_t kb = smem_u32(sK + kbuf * kTileBytes), vb = smem_u32(sV);
#pragma unroll
          for (int k = 0; k < kD / 16; ++k)
            umma_bf16(tmem, smem_desc_sw128(qa + k * 32, 16, 1024),
                      smem_desc_sw128(kb + k * 32, 16, 1024), id_s, k > 0 ? 1u : 0u);
#pragma unroll
          for (int k = 0; k < kD / 16; ++k)
            umma_bf16(tmem + 128, smem_desc_sw128(doa + k * 32, 16, 1024),
                      smem_desc_sw128(vb + k * 32, 16, 1024), id_s, k > 0 ? 1u : 0u);
          umma_commit(sp_full);
          if (last) umma_commit(v_empty);  // the next unit's V may load now
        }
        __syncwarp();
      };
      int G = 0, uc = 0;
      for (long long u = blockIdx.x; u < units; u += gridDim.x, ++uc) {
        const Unit w = decode(u);
        const int kbuf = uc & 1;
        mbar_wait(&k_full[kbuf], (uc >> 1) & 1);
        mbar_wait(v_full, uc & 1);
        issue_sdp(G, kbuf, w.n_it == 1);
        // the previous unit's dV / dK must have been drained before this unit's first
        mbar_wait(dkv_empty, (uc & 1) ^ 1);
        for (int it = 0; it < w.n_it; ++it, ++G) {
          const int st = G % kQStages, b = G & 1, db = G % kDSBufs;
          mbar_wait(sp_loaded, G & 1);  // softmax holds S/dP(G) in registers
          if (it + 1 < w.n_it) issue_sdp(G + 1, kbuf, it + 2 == w.n_it);
          mbar_wait(&ds_full[db], (G / kDSBufs) & 1);
          tc_fence_after();
          const uint32_t pa = smem_u32(sP), dsa = smem_u32(sdS + db * kPBytes);
          const uint32_t qa = smem_u32(sQ + st * kTileBytes), doa = smem_u32(sdO + st * kTileBytes);
          const uint32_t kb = smem_u32(sK + kbuf * kTileBytes);
          if (lane == 0) {
            // dV += P^T dO (K = queries: P read MN-major, two 64-key atoms 16 KB apart)
#pragma unroll
            for (int k = 0; k < kTile / 16; ++k)
              umma_bf16(tmem + 256, smem_desc_sw128(pa + k * 2048, kPBytes / 2, 1024),
                        smem_desc_sw128(doa + k * 2048, kD * 128, 1024), id_kv,
                        (it > 0 || k > 0) ? 1u : 0u);
            umma_commit(p_empty);
          }
          __syncwarp();
          mbar_wait(&dq_empty[b], ((G >> 1) & 1) ^ 1);
          tc_fence_after();
          if (lane == 0) {
            // dQ = dS K_j (K = keys: dS K-major, K_j MN-major)
#pragma unroll
            for (int k = 0; k < kTile / 16; ++k)
              umma_bf16(tmem + 384 + b * 64,
                        smem_desc_sw128(dsa + (k >> 2) * (kPBytes / 2) + (k & 3) * 32, 16, 1024),
                        smem_desc_sw128(kb + k * 2048, kD * 128, 1024), id_q, k > 0 ? 1u : 0u);
            umma_commit(&dq_full[b]);
            // dK += dS^T Q
#pragma unroll
            for (int k = 0; k < kTile / 16; ++k)
              umma_bf16(tmem + 320, smem_desc_sw128(dsa + k * 2048, kPBytes / 2, 1024),
                        smem_desc_sw128(qa + k * 2048, kD * 128, 1024), id_kv,
                        (it > 0 || k > 0) ? 1u : 0u);
            umma_commit(&ds_empty[db]);
            umma_commit(&q_empty[st]);
          }
          __syncwarp();
        }
        if (lane == 0) {
          umma_commit(dkv_full);
          umma_commit(&k_empty[kbuf]);  // every MMA reading this unit's K has run
        }
        __syncwarp();
      }
    }
  } else if (warp < 12) {
    regs_inc<184>();
    // two warps per TMEM lane quarter: warp w owns rows 32*(w%4).. and key
    // half (w-4)/4 (64 keys of S / dP)
    const int quarter = warp & 3, half = (warp - 4) >> 2;
    const int r = quarter * 32 + lane;  // query row
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const float lse_scale = 1.4426950408889634f;
    const float sl = p.scale_log2, sc = p.scale;
    int G = 0;
    for (long long u = blockIdx.x; u < units; u += gridDim.x) {
      const Unit w = decode(u);
      const int kt = w.kt, k0 = w.k0, i0 = w.i0, n_it = w.n_it;
      // per-row lse / D, loaded one query tile ahead (their latency is not hidden otherwise)
      const float* lse_row = p.lse + ((long long)w.bb * p.heads + w.h) * p.seq;
      const float* d_row = p.D + ((long long)w.bb * p.heads + w.h) * p.seq;
      auto row_stats = [&](int it, float& l2, float& dq) {
        const int qq = (i0 + it) * kTile + r;
        const bool ok = it < n_it && qq < p.seq;
        l2 = ok ? lse_row[qq] : 0.f;
        dq = ok ? d_row[qq] : 0.f;
      };
      float lse_next, d_next;
      row_stats(0, lse_next, d_next);
      for (int it = 0; it < n_it; ++it, ++G) {
        const int i = i0 + it;
        const int q = i * kTile + r;
        const bool qok = q < p.seq;
        const float lse2 = lse_next * lse_scale;
        const float Dq = d_next * sc;
        row_stats(it + 1, lse_next, d_next);
        const bool mask = !qok || k0 + kTile > p.kv_seq || (p.causal && i == kt);
        const int pb = G % kDSBufs;
        uint8_t* tdS = sdS + pb * kPBytes;
        mbar_wait(sp_full, G & 1);
        tc_fence_after();
        uint32_t us[64], ud[64];
        tmem_ld_32x32b_x32(tmem + half * 64 + lane_off, us);
        tmem_ld_32x32b_x32(tmem + half * 64 + 32 + lane_off, us + 32);
        tmem_ld_32x32b_x32(tmem + 128 + half * 64 + lane_off, ud);
        tmem_ld_32x32b_x32(tmem + 128 + half * 64 + 32 + lane_off, ud + 32);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(sp_loaded);  // the MMA may overwrite S/dP now
        mbar_wait(&ds_empty[pb], ((G / kDSBufs) & 1) ^ 1);
        uint4 pk[8];  // P row chunk, packed bf16 (stored once dV(G-1) released sP)
        // the key mask only exists on boundary tiles: two straight-line copies
        auto tile = [&](auto masked) {
          constexpr bool kMask = decltype(masked)::value;
#pragma unroll
          for (int c = 0; c < 8; ++c) {  // 16-byte chunk c of this half's 64-key atom
            float pv[8], dsv[8];
#pragma unroll
            for (int e = 0; e < 8; e += 2) {  // two keys per packed f32x2 instruction
              const float2 a = fma2(make_float2(__uint_as_float(us[c * 8 + e]), __uint_as_float(us[c * 8 + e + 1])),
                                    make_float2(sl, sl), make_float2(-lse2, -lse2));
              // DPN_ATTN_POLY_BWD of every 4 key pairs on the FMA pipe (see exp2_fma2)
              float2 pr = e >= 2 * (4 - DPN_ATTN_POLY_BWD) ? exp2_fma2(a) : make_float2(ex2(a.x), ex2(a.y));
              if constexpr (kMask) {
                const int key = k0 + half * 64 + c * 8 + e;
                pr.x = (qok && key < p.kv_seq && (!p.causal || key <= q)) ? pr.x : 0.f;
                pr.y = (qok && key + 1 < p.kv_seq && (!p.causal || key + 1 <= q)) ? pr.y : 0.f;
              }
              pv[e] = pr.x;
              pv[e + 1] = pr.y;
              const float2 ds = mul2(pr, fma2(make_float2(__uint_as_float(ud[c * 8 + e]), __uint_as_float(ud[c * 8 + e + 1])),
                                              make_float2(sc, sc), make_float2(-Dq, -Dq)));
              dsv[e] = ds.x;
              dsv[e + 1] = ds.y;
            }
            pk[c].x = pack_bf16(pv[0], pv[1]);
            pk[c].y = pack_bf16(pv[2], pv[3]);
            pk[c].z = pack_bf16(pv[4], pv[5]);
            pk[c].w = pack_bf16(pv[6], pv[7]);
            uint4 b2;
            b2.x = pack_bf16(dsv[0], dsv[1]);
            b2.y = pack_bf16(dsv[2], dsv[3]);
            b2.z = pack_bf16(dsv[4], dsv[5]);
            b2.w = pack_bf16(dsv[6], dsv[7]);
            sts128(smem_u32(tdS) + half * (kPBytes / 2) + sw128(r, c), b2);
          }
        };
        if (mask) tile(std::true_type{});
        else tile(std::false_type{});
        mbar_wait(p_empty, (G & 1) ^ 1);
#pragma unroll
        for (int c = 0; c < 8; ++c)
          sts128(smem_u32(sP) + half * (kPBytes / 2) + sw128(r, c), pk[c]);
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ds_full[pb]);
      }
    }
  } else {
    regs_dec<88>();
    // dQ drain per query tile: warp w reads TMEM lanes 32*(w%4).. (its 32 query
    // rows), all 64 columns -> swizzled f32 staging -> TMA reduce-add; and per
    // unit the dV / dK drain (TMEM lane = key row) -> bf16 dqkv, off the
    // softmax warps (they start the next unit meanwhile)
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const bool issuer = warp == 12 && lane == 0;
    int G = 0, uc = 0;
    for (long long u = blockIdx.x; u < units; u += gridDim.x, ++uc) {
      const Unit w = decode(u);
      for (int it = 0; it < w.n_it; ++it, ++G) {
        const int b = G & 1;
        mbar_wait(&dq_full[b], (G >> 1) & 1);
        tc_fence_after();
        uint32_t uq[64];
        tmem_ld_32x32b_x32(tmem + 384 + b * 64 + lane_off, uq);
        tmem_ld_32x32b_x32(tmem + 384 + b * 64 + 32 + lane_off, uq + 32);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dq_empty[b]);
        // one 32-column half at a time through the 16 KB staging box: the previous
        // reduce must have finished reading it before it is rewritten
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          if (issuer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          asm volatile("bar.sync 6, 128;" ::: "memory");
#pragma unroll
          for (int c = 0; c < 8; ++c)
            sts128(smem_u32(sdQ) + sw128(r, c),
                   make_uint4(uq[hh * 32 + c * 4], uq[hh * 32 + c * 4 + 1], uq[hh * 32 + c * 4 + 2],
                              uq[hh * 32 + c * 4 + 3]));
          fence_async_smem();
          asm volatile("bar.sync 6, 128;" ::: "memory");
          if (issuer) {
            // rows past seq carry zero (P = dS = 0 there), rows past the tensor are clipped
            asm volatile(
                "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group"
                " [%0, {%2, %3}], [%1];" ::"l"(reinterpret_cast<uint64_t>(&tm_dq)),
                "r"(smem_u32(sdQ)), "r"(w.h * kD + hh * 32), "r"(w.row0 + (w.i0 + it) * kTile)
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
      }
      // dV, dK of this key tile (TMEM lane = key row), 32 columns at a time
      mbar_wait(dkv_full, uc & 1);
      tc_fence_after();
      const int key = w.k0 + r;
#pragma unroll 1
      for (int part = 0; part < 4; ++part) {  // dV cols 0-31, 32-63, dK cols 0-31, 32-63
        uint32_t uv[32];
        tmem_ld_32x32b_x32(tmem + 256 + part * 32 + lane_off, uv);
        tmem_ld_wait();
        if (p.dbias_k) {
          // column sums over this warp's 32 key rows: butterfly reduce-scatter,
          // lane i ends with column i of the part (runs once per unit)
          float cs[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) cs[c] = key < p.kv_seq ? __uint_as_float(uv[c]) : 0.f;
#pragma unroll
          for (int wdt = 16; wdt >= 1; wdt >>= 1) {
            const bool upper = lane & wdt;
#pragma unroll
            for (int c = 0; c < wdt; ++c) {
              const float send = upper ? cs[c] : cs[c + wdt];
              const float keep = upper ? cs[c + wdt] : cs[c];
              cs[c] = keep + __shfl_xor_sync(0xffffffffu, send, wdt);
            }
          }
          float* db = ((part >> 1) ? p.dbias_k : p.dbias_v) + w.h * kD + (part & 1) * 32;
          atomicAdd(db + lane, cs[0]);
        }
        if (key < p.kv_seq) {
          const int which = part >> 1;  // 0: dV, 1: dK
          __nv_bfloat16* dst = (which ? p.dk : p.dv) + (long long)(w.krow0 + key) * p.dkv_ld +
                               w.h * kD + (part & 1) * 32;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint4 a;
            a.x = pack_bf16(__uint_as_float(uv[c * 8 + 0]), __uint_as_float(uv[c * 8 + 1]));
            a.y = pack_bf16(__uint_as_float(uv[c * 8 + 2]), __uint_as_float(uv[c * 8 + 3]));
            a.z = pack_bf16(__uint_as_float(uv[c * 8 + 4]), __uint_as_float(uv[c * 8 + 5]));
            a.w = pack_bf16(__uint_as_float(uv[c * 8 + 6]), __uint_as_float(uv[c * 8 + 7]));
            reinterpret_cast<uint4*>(dst)[c] = a;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dkv_empty);
    }
    if (issuer) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

// D[b, h, q] = sum_c dO[row, h*64 + c] * O[row, h*64 + c]; one warp per (row, head)
// D[b,h,q] = rowsum(dO * O) over the head's 64 columns; also zeroes the fp32
// dQ accumulator (replaces a separate memset).  8 threads per (row, head), one
// 16-byte chunk of O and dO each.
__global__ void __launch_bounds__(256) attn_bwd_prep_kernel(const __nv_bfloat16* __restrict__ o,
                                     const __nv_bfloat16* __restrict__ dout, float* __restrict__ D,
                                     float* __restrict__ dq, long long rows, int seq, int heads) {
  pdl_wait();
  const long long total = rows * heads * 8;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    // total is a multiple of 8 and so is the grid stride: all 8 lanes of a
    // group stay in the loop together
    const long long e = i * 8;  // element offset in [rows, heads*64]
    const uint4 ou = *reinterpret_cast<const uint4*>(o + e);
    const uint4 du = *reinterpret_cast<const uint4*>(dout + e);
    const __nv_bfloat162* oh = reinterpret_cast<const __nv_bfloat162*>(&ou);
    const __nv_bfloat162* dh = reinterpret_cast<const __nv_bfloat162*>(&du);
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 a = __bfloat1622float2(oh[k]), b = __bfloat1622float2(dh[k]);
      acc += a.x * b.x + a.y * b.y;
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 4);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    reinterpret_cast<float4*>(dq + e)[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    reinterpret_cast<float4*>(dq + e)[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    if ((threadIdx.x & 7) == 0) {
      const long long rh = i >> 3, row = rh / heads, bb = row / seq, q = row % seq;
      const int h = (int)(rh % heads);
      D[(bb * heads + h) * seq + q] = acc;
    }
  }
}

// dst[:, 0:H] (row stride ld) = bf16(dq)
// dQ (f32 accumulator) -> bf16 into dqkv.  With dbias: += the column sums of
// dQ (the Q part of the QKV bias gradient).  Thread (column group of 4, row
// lane) walks a band of rows; the CTA's row lanes combine in shared memory and
// add one partial per column.
constexpr int kDqLanes = 4;
__global__ void __launch_bounds__(256 * kDqLanes) attn_dq_store_kernel(
    const float* __restrict__ dq, __nv_bfloat16* __restrict__ dqkv, long long rows, int H,
    long long ld, long long rows_per_cta, float* __restrict__ dbias) {
  pdl_wait();
  __shared__ float4 part[kDqLanes][256];
  const int c4 = blockIdx.y * 256 + (threadIdx.x & 255), lane = threadIdx.x >> 8;
  const bool col = c4 < (H >> 2);
  const long long r0 = (long long)blockIdx.x * rows_per_cta;
  const long long r1 = min(rows, r0 + rows_per_cta);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (col) {
#pragma unroll 4
    for (long long r = r0 + lane; r < r1; r += kDqLanes) {
      const float4 v = reinterpret_cast<const float4*>(dq + r * H)[c4];
      uint2 w;
      w.x = pack_bf16(v.x, v.y);
      w.y = pack_bf16(v.z, v.w);
      *reinterpret_cast<uint2*>(dqkv + r * ld + c4 * 4) = w;
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  if (dbias == nullptr) return;
  part[lane][threadIdx.x & 255] = acc;
  __syncthreads();
  if (lane == 0 && col) {
#pragma unroll
    for (int q = 1; q < kDqLanes; ++q) {
      const float4 o = part[q][threadIdx.x];
      acc.x += o.x; acc.y += o.y; acc.z += o.z; acc.w += o.w;
    }
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dbias + c4 * 4), "f"(acc.x),
                 "f"(acc.y), "f"(acc.z), "f"(acc.w)
                 : "memory");
  }
}

constexpr int kBwdSmem = 1024 + kTileBytes * (3 + 2 * kQStages) + (1 + kDSBufs) * kPBytes + kPBytes / 2 + 256;  // K[2] V Q[] dO[] | P dS[] | dQ-staging

}  // namespace
}  // namespace dpn

using namespace dpn;

extern "C" int dpn_attn_fwd(const void* qkv, void* out, float* lse, int64_t batch, int64_t seq,
                            int64_t heads, int64_t head_dim, float scale, int causal,
                            void* stream) {
  DPN_REQUIRE(head_dim == 64, "fused attention supports head_dim 64");
  DPN_REQUIRE(seq % 64 == 0 && seq > 0, "seq must be a positive multiple of 64");
  DPN_REQUIRE(qkv && out && lse, "null pointer");
  CUtensorMap tm;
  const long long H = heads * head_dim;
  int rc = map_2d(&tm, qkv, batch * seq, 3 * H);
  if (rc) return rc;
  AttnParams p{};
  p.batch = (int)batch;
  p.seq = (int)seq;
  p.kv_seq = (int)seq;
  p.q_col = 0;
  p.k_col = (int)H;
  p.v_col = (int)(2 * H);
  p.heads = (int)heads;
  p.H = (int)H;
  p.scale = scale;
  p.scale_log2 = scale * kLog2e;
  p.causal = causal;
  p.out = static_cast<__nv_bfloat16*>(out);
  p.lse = lse;
  const FwdKernel fk = fwd_kernel();
  static int n_sm = 0;
  if (n_sm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (n_sm <= 0) n_sm = 148;
  }
  const long long units = (long long)((seq + kTile - 1) / kTile) * heads * batch;
  const unsigned grid = (unsigned)std::min<long long>(units, n_sm);  // persistent: one CTA per SM
  DPN_CHECK_CUDA(launch_pdl(fk.fn, grid, fk.threads, fk.smem, (cudaStream_t)stream, tm, tm, p));
  DPN_LAUNCH_CHECK();
  return 0;
}


namespace dpn {
namespace {
// Backward launcher shared by self- and cross-attention: q_src / kv_src hold Q
// and K|V (columns q_col / k_col / v_col of head 0), dq_dst (row stride dq_ld)
// receives dQ, dk / dv (row stride dkv_ld) dK and dV.
int attn_bwd_launch(const void* q_src, long long q_ld, const void* kv_src, long long kv_ld, int q_col,
                    int k_col, int v_col, const void* out, const void* dout, const float* lse,
                    __nv_bfloat16* dq_dst, long long dq_ld, __nv_bfloat16* dk, __nv_bfloat16* dv,
                    long long dkv_ld, float* workspace, int64_t workspace_floats, int64_t batch,
                    int64_t seq, int64_t kv_seq, int64_t heads, float scale, int causal, void* stream,
                    float* dbias_q = nullptr, float* dbias_k = nullptr, float* dbias_v = nullptr) {
  const long long H = heads * kD, rows = batch * seq;
  DPN_REQUIRE((dbias_q == nullptr) == (dbias_k == nullptr) && (dbias_k == nullptr) == (dbias_v == nullptr) &&
                  (reinterpret_cast<uintptr_t>(dbias_q) & 15) == 0,
              "dbias must be a 16-byte aligned f32 [3H] (or null)");
  DPN_REQUIRE(workspace != nullptr && workspace_floats >= rows * H + batch * heads * seq,
              "workspace must hold batch*seq*(heads*64) + batch*heads*seq floats");
  cudaStream_t st = (cudaStream_t)stream;
  float* dq = workspace;
  float* D = workspace + rows * H;
  {
    const long long threads = rows * heads * 8;
    const unsigned g = (unsigned)std::min<long long>((threads + 255) / 256, 148 * 8);
    DPN_CHECK_CUDA(launch_pdl(attn_bwd_prep_kernel, g, 256, 0, st, (const __nv_bfloat16*)out,
                              (const __nv_bfloat16*)dout, D, dq, rows, (int)seq, (int)heads));
    DPN_LAUNCH_CHECK();
  }
  CUtensorMap tq, tkv, td, tdq;
  int rc = map_2d(&tq, q_src, rows, q_ld);
  if (!rc) rc = map_2d(&tkv, kv_src, batch * kv_seq, kv_ld);
  if (!rc) rc = map_2d(&td, dout, rows, H);
  if (!rc) rc = map_2d_f32(&tdq, dq, rows, H);
  if (rc) return rc;
  AttnBwdParams p{};
  p.batch = (int)batch;
  p.seq = (int)seq;
  p.kv_seq = (int)kv_seq;
  p.q_col = q_col;
  p.k_col = k_col;
  p.v_col = v_col;
  p.dk = dk;
  p.dv = dv;
  p.dkv_ld = dkv_ld;
  p.heads = (int)heads;
  p.H = (int)H;
  p.scale = scale;
  p.scale_log2 = scale * kLog2e;
  p.causal = causal;
  p.lse = lse;
  p.D = D;
  p.dq = dq;
  p.dqkv = dq_dst;
  p.dbias_k = dbias_k;
  p.dbias_v = dbias_v;
  static bool set = false;
  if (!set) {
    DPN_CHECK_CUDA(cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        kBwdSmem));
    set = true;
  }
  static int n_sm_b = 0;
  if (n_sm_b == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm_b, cudaDevAttrMultiProcessorCount, dev);
    if (n_sm_b <= 0) n_sm_b = 148;
  }
  const long long units = (long long)((kv_seq + kTile - 1) / kTile) * heads * batch;
  const unsigned grid = (unsigned)std::min<long long>(units, n_sm_b);  // persistent
  DPN_CHECK_CUDA(launch_pdl(attn_bwd_kernel, grid, kBwdThreads, kBwdSmem, st, tq, tkv, td, tdq, p));
  DPN_LAUNCH_CHECK();
  {
    // one CTA per SM per column block of 1024 columns: ~rows/148 rows per CTA, so
    // the bias partials are a small fraction of the bytes moved
    const long long gy = (H / 4 + 255) / 256;
    const long long bands = std::max<long long>(1, std::min<long long>(rows, 148 / std::min<long long>(gy, 148)));
    const long long per = (rows + bands - 1) / bands;
    DPN_CHECK_CUDA(launch_pdl(attn_dq_store_kernel, dim3((unsigned)((rows + per - 1) / per), (unsigned)gy),
                              256 * kDqLanes, 0, st, dq, dq_dst, rows, (int)H, dq_ld, per, dbias_q));
  }
  DPN_LAUNCH_CHECK();
  return 0;
}
}  // namespace
}  // namespace dpn

extern "C" int dpn_attn_bwd(const void* qkv, const void* out, const void* dout, const float* lse,
                            void* dqkv, float* workspace, int64_t workspace_floats, int64_t batch,
                            int64_t seq, int64_t heads, int64_t head_dim, float scale, int causal,
                            float* dbias, void* stream) {
  DPN_REQUIRE(head_dim == 64, "fused attention supports head_dim 64");
  DPN_REQUIRE(seq % 64 == 0 && seq > 0, "seq must be a positive multiple of 64");
  const long long H = heads * head_dim;
  __nv_bfloat16* d = static_cast<__nv_bfloat16*>(dqkv);
  return attn_bwd_launch(qkv, 3 * H, qkv, 3 * H, 0, (int)H, (int)(2 * H), out, dout, lse, d, 3 * H,
                         d + H, d + 2 * H, 3 * H, workspace, workspace_floats, batch, seq, seq, heads,
                         scale, causal, stream, dbias, dbias ? dbias + H : nullptr,
                         dbias ? dbias + 2 * H : nullptr);
}

extern "C" int dpn_attn_fwd_cross(const void* q, const void* kv, void* out, float* lse, int64_t batch,
                                  int64_t q_seq, int64_t kv_seq, int64_t heads, int64_t head_dim,
                                  float scale, void* stream) {
  DPN_REQUIRE(head_dim == 64, "fused attention supports head_dim 64");
  DPN_REQUIRE(q_seq % 64 == 0 && kv_seq % 64 == 0 && q_seq > 0 && kv_seq > 0,
              "sequence lengths must be positive multiples of 64");
  DPN_REQUIRE(q && kv && out && lse, "null pointer");
  const long long H = heads * head_dim;
  CUtensorMap tq, tkv;
  int rc = map_2d(&tq, q, batch * q_seq, H);
  if (!rc) rc = map_2d(&tkv, kv, batch * kv_seq, 2 * H);
  if (rc) return rc;
  AttnParams p{};
  p.batch = (int)batch;
  p.seq = (int)q_seq;
  p.kv_seq = (int)kv_seq;
  p.q_col = 0;
  p.k_col = 0;
  p.v_col = (int)H;
  p.heads = (int)heads;
  p.H = (int)H;
  p.scale = scale;
  p.scale_log2 = scale * kLog2e;
  p.causal = 0;
  p.out = static_cast<__nv_bfloat16*>(out);
  p.lse = lse;
  const FwdKernel fk = fwd_kernel();
  int n_sm = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  if (n_sm <= 0) n_sm = 148;
  const long long units = (long long)((q_seq + kTile - 1) / kTile) * heads * batch;
  const unsigned grid = (unsigned)std::min<long long>(units, n_sm);
  DPN_CHECK_CUDA(launch_pdl(fk.fn, grid, fk.threads, fk.smem, (cudaStream_t)stream, tq, tkv, p));
  DPN_LAUNCH_CHECK();
  return 0;
}

extern "C" int dpn_attn_bwd_cross(const void* q, const void* kv, const void* out, const void* dout,
                                  const float* lse, void* dq, void* dkv, float* workspace,
                                  int64_t workspace_floats, int64_t batch, int64_t q_seq, int64_t kv_seq,
                                  int64_t heads, int64_t head_dim, float scale, void* stream) {
  DPN_REQUIRE(head_dim == 64, "fused attention supports head_dim 64");
  DPN_REQUIRE(q_seq % 64 == 0 && kv_seq % 64 == 0 && q_seq > 0 && kv_seq > 0,
              "sequence lengths must be positive multiples of 64");
  const long long H = heads * head_dim;
  __nv_bfloat16* dkvp = static_cast<__nv_bfloat16*>(dkv);
  return attn_bwd_launch(q, H, kv, 2 * H, 0, 0, (int)H, out, dout, lse, static_cast<__nv_bfloat16*>(dq),
                         H, dkvp, dkvp + H, 2 * H, workspace, workspace_floats, batch, q_seq, kv_seq,
                         heads, scale, 0, stream);
}
