// HBM-bound kernels of the stage executor (sm_100a).  All are single-pass,
// 16-byte vectorised, warp-shuffle reduced; fp32 statistics, bf16 storage.
//
//   layernorm fwd/bwd   ln1 / ln2 / lnf nodes        warp per row (+ colred for dgamma/dbeta)
//   softmax fwd/bwd     score node (scaled, causal)   warp per row
//   gelu fwd/bwd        gelu node                     grid-stride, 8 elem/thread
//   add                 add node (residual)           grid-stride
//   colsum (colred)     bias gradients                column tiles, 4 rows in flight, vector reds
//   xent                head node loss + dlogits      CTA per row, row cached in smem
//   embed fwd/bwd       embed node                    warp per token
//   adamw               optimizer over a stage's flat parameter buffer
#include "common.cuh"
#include "../../include/dawnpiper.h"

namespace dpn {
namespace {

constexpr int kMaxVec = 8;  // up to 8 x 16 B chunks per lane => rows of <= 2048 bf16

__device__ __forceinline__ void load8(const __nv_bfloat16* p, float* f) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void store8(__nv_bfloat16* p, const float* f) {
  uint4 u;
  u.x = pack_bf16(f[0], f[1]);
  u.y = pack_bf16(f[2], f[3]);
  u.z = pack_bf16(f[4], f[5]);
  u.w = pack_bf16(f[6], f[7]);
  *reinterpret_cast<uint4*>(p) = u;
}

int grid_for(long long work_items, int per_block) {
  long long g = (work_items + per_block - 1) / per_block;
  return (int)std::max<long long>(1, std::min<long long>(g, 148LL * 16));
}

// ---------------- LayerNorm ----------------
// NV = 16-byte chunks per lane (cols = 8 * 32 * NV at most); keeps the row in
// registers without spilling.

template <int NV>
__global__ void __launch_bounds__(256) ln_fwd_kernel(const __nv_bfloat16* __restrict__ x,
                                                     const __nv_bfloat16* __restrict__ gamma,
                                                     const __nv_bfloat16* __restrict__ beta,
                                                     __nv_bfloat16* __restrict__ y,
                                                     float* __restrict__ mean_out,
                                                     float* __restrict__ rstd_out, long long rows,
                                                     int cols, float eps) {
  pdl_wait();
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nvec = cols >> 3;
  for (long long r = (long long)blockIdx.x * warps + (threadIdx.x >> 5); r < rows;
       r += (long long)gridDim.x * warps) {
    const __nv_bfloat16* xr = x + r * cols;
    float v[NV][8];
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = lane + 32 * j;
      if (c < nvec) {
        load8(xr + c * 8, v[j]);
#pragma unroll
        for (int i = 0; i < 8; ++i) s += v[j][i];
      }
    }
    const float mu = warp_sum(s) / cols;
    float q = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = lane + 32 * j;
      if (c < nvec) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float d = v[j][i] - mu;
          q += d * d;
        }
      }
    }
    const float rs = rsqrtf(warp_sum(q) / cols + eps);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = lane + 32 * j;
      if (c < nvec) {
        float g[8], b[8], o[8];
        load8(gamma + c * 8, g);
        load8(beta + c * 8, b);
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = (v[j][i] - mu) * rs * g[i] + b[i];
        store8(y + r * cols + c * 8, o);
      }
    }
    if (lane == 0) {
      mean_out[r] = mu;
      rstd_out[r] = rs;
    }
  }
}

// dx = rstd * (dyg - mean(dyg) - xhat * mean(dyg * xhat)) [+ dx_add], dyg = dy * gamma.
// One warp per row; the row of x and dy stays in registers as packed bf16 (no
// second read), so many warps per SM keep enough loads in flight for HBM.
// dgamma / dbeta come from colred_kernel<1> (a column reduction, below).
template <int NV>
__global__ void __launch_bounds__(256) ln_dx_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
    const __nv_bfloat16* __restrict__ gamma, const float* __restrict__ mean,
    const float* __restrict__ rstd, __nv_bfloat16* dx, const __nv_bfloat16* dx_add,
    long long rows, int cols) {
  pdl_wait();
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nvec = cols >> 3;
  for (long long r = (long long)blockIdx.x * warps + (threadIdx.x >> 5); r < rows;
       r += (long long)gridDim.x * warps) {
    const float mu = mean[r], rs = rstd[r];
    uint4 xr[NV], dr[NV], ar[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = lane + 32 * j;
      if (c < nvec) {
        xr[j] = *reinterpret_cast<const uint4*>(x + r * cols + c * 8);
        dr[j] = *reinterpret_cast<const uint4*>(dy + r * cols + c * 8);
        if (dx_add) ar[j] = *reinterpret_cast<const uint4*>(dx_add + r * cols + c * 8);
      }
    }
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = lane + 32 * j;
      if (c < nvec) {
        float xv[8], dv[8], gm[8];
        load8(reinterpret_cast<const __nv_bfloat16*>(&xr[j]), xv);
        load8(reinterpret_cast<const __nv_bfloat16*>(&dr[j]), dv);
        load8(gamma + c * 8, gm);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float g = dv[i] * gm[i];
          s1 += g;
          s2 += g * (xv[i] - mu) * rs;
        }
      }
    }
    s1 = warp_sum(s1) / cols;
    s2 = warp_sum(s2) / cols;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = lane + 32 * j;
      if (c < nvec) {
        float xv[8], dv[8], gm[8], o[8];
        load8(reinterpret_cast<const __nv_bfloat16*>(&xr[j]), xv);
        load8(reinterpret_cast<const __nv_bfloat16*>(&dr[j]), dv);
        load8(gamma + c * 8, gm);
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = rs * (dv[i] * gm[i] - s1 - (xv[i] - mu) * rs * s2);
        if (dx_add) {
          float a[8];
          load8(reinterpret_cast<const __nv_bfloat16*>(&ar[j]), a);
#pragma unroll
          for (int i = 0; i < 8; ++i) o[i] += a[i];
        }
        store8(dx + r * cols + c * 8, o);
      }
    }
  }
}

__device__ __forceinline__ void red_add_v4(float* addr, const float* v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(v[0]), "f"(v[1]),
               "f"(v[2]), "f"(v[3])
               : "memory");
}

// Fused LayerNorm backward: dx (+ dx_add), dgamma, dbeta and, optionally, the
// column sum of the final dx (the bias gradient of the linear node whose
// output gradient this is) in ONE pass over dy / x / dx_add.
//
// Layout: a row is owned by a group of G = ceil(cols / 256) warps, one 16-byte
// column chunk (8 columns) per lane, so every thread keeps the SAME 8 columns
// for every row its CTA visits: the three column accumulators cost 24
// registers (a warp-per-row kernel needs 32 * 3 * cols / 256 of them, which is
// what capped the earlier fused attempt at 16 warps per SM).  Row statistics
// (sum dy*gamma, sum dy*gamma*xhat) combine the group's warps through shared
// memory behind a per-group named barrier; kLnRows rows per group are in
// flight per iteration.  The CTA's column partials combine across groups in
// shared memory and go out with one vector red per 4 columns.
//   bytes: read dy, x (, dx_add), write dx  (+ 8 B of stats per row)
#ifndef DPN_LN_ROWS
#define DPN_LN_ROWS 3
#endif
#ifndef DPN_LN_CTAS
#define DPN_LN_CTAS 2
#endif
constexpr int kLnThreads = 256;  // DPN_LN_CTAS CTAs per SM: their load / reduce / store phases interleave
constexpr int kLnRows = DPN_LN_ROWS;
__global__ void __launch_bounds__(kLnThreads, DPN_LN_CTAS) ln_bwd_fused_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
    const __nv_bfloat16* __restrict__ gamma, const float* __restrict__ mean,
    const float* __restrict__ rstd, __nv_bfloat16* dx, const __nv_bfloat16* dx_add,
    long long rows, int cols, long long rows_per_cta, float* __restrict__ dgamma,
    float* __restrict__ dbeta, float* __restrict__ dbias) {
  pdl_wait();
  extern __shared__ float ln_smem[];
  const int nvec = cols >> 3;
  const int G = (nvec + 31) >> 5;              // warps per row group
  const int groups = (kLnThreads >> 5) / G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = warp / G, wi = warp % G;
  const int chunk = wi * 32 + lane;
  const bool in_grp = grp < groups;
  const bool col = in_grp && chunk < nvec;
  float* stat = ln_smem;                       // [2 parity][warps][kLnRows][2]
  float* part = ln_smem + 2 * (kLnThreads / 32) * kLnRows * 2; // [groups][cols]
  float gm[8], ag[8], ab[8], ad[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) ag[i] = ab[i] = ad[i] = 0.f;
  if (col) load8(gamma + chunk * 8, gm);
  const float inv_cols = 1.f / (float)cols;
  const long long r0 = (long long)blockIdx.x * rows_per_cta;
  const long long r1 = min(rows, r0 + rows_per_cta);
  int parity = 0;
  if (in_grp) {
    for (long long base = r0 + (long long)grp * kLnRows; base < r1;
         base += (long long)groups * kLnRows, parity ^= 1) {
      uint4 xr[kLnRows], dr[kLnRows], ar[kLnRows];
      float mu[kLnRows], rs[kLnRows];
#pragma unroll
      for (int u = 0; u < kLnRows; ++u) {
        const long long r = base + u;
        const bool ok = col && r < r1;
        xr[u] = ok ? *reinterpret_cast<const uint4*>(x + r * cols + chunk * 8) : make_uint4(0, 0, 0, 0);
        dr[u] = ok ? *reinterpret_cast<const uint4*>(dy + r * cols + chunk * 8) : make_uint4(0, 0, 0, 0);
        ar[u] = ok && dx_add ? *reinterpret_cast<const uint4*>(dx_add + r * cols + chunk * 8)
                             : make_uint4(0, 0, 0, 0);
        mu[u] = r < r1 ? mean[r] : 0.f;
        rs[u] = r < r1 ? rstd[r] : 0.f;
      }
      float* st = stat + parity * (kLnThreads / 32) * kLnRows * 2;
#pragma unroll
      for (int u = 0; u < kLnRows; ++u) {
        float xv[8], dv[8], s1 = 0.f, s2 = 0.f;
        load8(reinterpret_cast<const __nv_bfloat16*>(&xr[u]), xv);
        load8(reinterpret_cast<const __nv_bfloat16*>(&dr[u]), dv);
        if (col) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float g = dv[i] * gm[i];
            s1 += g;
            s2 += g * (xv[i] - mu[u]) * rs[u];
          }
        }
        s1 = warp_sum(s1);
        s2 = warp_sum(s2);
        if (lane == 0) {
          st[(warp * kLnRows + u) * 2] = s1;
          st[(warp * kLnRows + u) * 2 + 1] = s2;
        }
      }
      // the group's G warps (parity double-buffers `stat`, so one barrier per
      // iteration orders both the writes and the next iteration's reuse)
      asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(G * 32) : "memory");
#pragma unroll
      for (int u = 0; u < kLnRows; ++u) {
        const long long r = base + u;
        float s1 = 0.f, s2 = 0.f;
        for (int w = 0; w < G; ++w) {
          s1 += st[((grp * G + w) * kLnRows + u) * 2];
          s2 += st[((grp * G + w) * kLnRows + u) * 2 + 1];
        }
        s1 *= inv_cols;
        s2 *= inv_cols;
        if (!col || r >= r1) continue;
        float xv[8], dv[8], o[8];
        load8(reinterpret_cast<const __nv_bfloat16*>(&xr[u]), xv);
        load8(reinterpret_cast<const __nv_bfloat16*>(&dr[u]), dv);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float xh = (xv[i] - mu[u]) * rs[u];
          ab[i] += dv[i];
          ag[i] += dv[i] * xh;
          o[i] = rs[u] * (dv[i] * gm[i] - s1 - xh * s2);
        }
        if (dx_add) {
          float a[8];
          load8(reinterpret_cast<const __nv_bfloat16*>(&ar[u]), a);
#pragma unroll
          for (int i = 0; i < 8; ++i) o[i] += a[i];
        }
        uint4 packed;
        packed.x = pack_bf16(o[0], o[1]);
        packed.y = pack_bf16(o[2], o[3]);
        packed.z = pack_bf16(o[4], o[5]);
        packed.w = pack_bf16(o[6], o[7]);
        *reinterpret_cast<uint4*>(dx + r * cols + chunk * 8) = packed;
        if (dbias) {  // the bias gradient sums the stored (bf16) dx, as a colsum pass would
          float q[8];
          load8(reinterpret_cast<const __nv_bfloat16*>(&packed), q);
#pragma unroll
          for (int i = 0; i < 8; ++i) ad[i] += q[i];
        }
      }
    }
  }
  // column partials: combine the groups in shared memory, one red per 4 columns
  auto flush = [&](float* out, const float(&acc)[8]) {
    __syncthreads();
    if (col) {
#pragma unroll
      for (int i = 0; i < 8; ++i) part[grp * cols + chunk * 8 + i] = acc[i];
    }
    __syncthreads();
    for (int c4 = threadIdx.x; c4 < (cols >> 2); c4 += kLnThreads) {
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      for (int g = 0; g < groups; ++g)
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] += part[g * cols + c4 * 4 + i];
      red_add_v4(out + c4 * 4, v);
    }
  };
  flush(dgamma, ag);
  flush(dbeta, ab);
  if (dbias) flush(dbias, ad);
}

// Column reductions over a row-major [rows, cols] bf16 matrix (bias and
// LayerNorm parameter gradients).  CTA (band, group) owns 8*cw columns and a
// band of rows; its 512 threads are cw column chunks x L row lanes, each lane
// keeping 4 rows (16 B each) in flight.  Lanes combine in shared memory and
// the CTA adds its partial with one vector red per 4 columns.
//   MODE 0: out0 += sum_r a[r]
//   MODE 1: out0 += sum_r a[r] * (x[r] - mean[r]) * rstd[r],  out1 += sum_r a[r]
constexpr int kColThreads = 512;
constexpr int kColUnrollSum = 8;   // MODE 0: rows in flight per lane
constexpr int kColUnrollLn = 2;    // MODE 1 (two operands per row; 2 CTAs per SM)
template <int MODE>
__global__ void __launch_bounds__(kColThreads, 2) colred_kernel(
    const __nv_bfloat16* __restrict__ a, long long lda, const __nv_bfloat16* __restrict__ x,
    const float* __restrict__ mean, const float* __restrict__ rstd, long long rows, int cols,
    long long rows_per_cta, float* __restrict__ out0, float* __restrict__ out1) {
  pdl_wait();
  constexpr int kColUnroll = MODE == 0 ? kColUnrollSum : kColUnrollLn;
  __shared__ float part[kColThreads * 8];
  const int nvec = cols >> 3;
  const int cw = min(nvec, 128);
  const int L = kColThreads / cw;
  const int ci = threadIdx.x % cw, lr = threadIdx.x / cw;
  const int chunk = blockIdx.y * cw + ci;
  const bool active = lr < L && chunk < nvec;
  float acc0[8] = {0, 0, 0, 0, 0, 0, 0, 0}, acc1[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long r0 = (long long)blockIdx.x * rows_per_cta;
  const long long r1 = min(rows, r0 + rows_per_cta);
  if (active) {
    for (long long r = r0 + lr; r < r1; r += kColUnroll * L) {
      uint4 av[kColUnroll], xv[kColUnroll];
      float mu[kColUnroll], rs[kColUnroll];
#pragma unroll
      for (int u = 0; u < kColUnroll; ++u) {
        const long long rr = r + (long long)u * L;
        if (rr < r1) {
          av[u] = *reinterpret_cast<const uint4*>(a + rr * lda + chunk * 8);
          if (MODE == 1) {
            xv[u] = *reinterpret_cast<const uint4*>(x + rr * cols + chunk * 8);
            mu[u] = mean[rr];
            rs[u] = rstd[rr];
          }
        } else {
          av[u] = make_uint4(0, 0, 0, 0);
          if (MODE == 1) {
            xv[u] = make_uint4(0, 0, 0, 0);
            mu[u] = 0.f;
            rs[u] = 0.f;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kColUnroll; ++u) {
        float v[8];
        load8(reinterpret_cast<const __nv_bfloat16*>(&av[u]), v);
        if (MODE == 1) {
          float xf[8];
          load8(reinterpret_cast<const __nv_bfloat16*>(&xv[u]), xf);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            acc0[k] += v[k] * (xf[k] - mu[u]) * rs[u];
            acc1[k] += v[k];
          }
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) acc0[k] += v[k];
        }
      }
    }
  }
#pragma unroll
  for (int pass = 0; pass < (MODE == 1 ? 2 : 1); ++pass) {
    float* acc = pass == 0 ? acc0 : acc1;
    float* out = pass == 0 ? out0 : out1;
    if (pass) __syncthreads();
    if (L > 1) {
      if (lr < L) {
#pragma unroll
        for (int k = 0; k < 8; ++k) part[threadIdx.x * 8 + k] = acc[k];
      }
      __syncthreads();
      if (lr == 0 && chunk < nvec) {
        for (int q = 1; q < L; ++q)
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[k] += part[(q * cw + ci) * 8 + k];
      }
    }
    if (lr == 0 && chunk < nvec) {
      red_add_v4(out + chunk * 8, acc);
      red_add_v4(out + chunk * 8 + 4, acc + 4);
    }
  }
}

// grid for colred_kernel: column groups x row bands, ~2 CTAs per SM in total,
// but at least `min_rows` rows per band so the atomics stay a small fraction
// of the bytes read.
dim3 colred_grid(long long rows, long long cols, long long* rows_per_cta) {
  const long long nvec = cols / 8;
  const long long cw = std::min<long long>(nvec, 128);
  const long long gy = (nvec + cw - 1) / cw;
  const long long min_rows = 32;
  long long bands = std::max<long long>(1, std::min<long long>((296 + gy - 1) / gy,
                                                               (rows + min_rows - 1) / min_rows));
  const long long per = (rows + bands - 1) / bands;
  *rows_per_cta = per;
  return dim3((unsigned)((rows + per - 1) / per), (unsigned)gy);
}

// ---------------- softmax over attention scores ----------------
// row r of a [Z, q_len, k_len] tensor; causal masks key > query.
template <int kPer>
__global__ void __launch_bounds__(256) softmax_fwd_kernel(const __nv_bfloat16* __restrict__ s,
                                                          __nv_bfloat16* __restrict__ p,
                                                          long long rows, int cols, int q_len,
                                                          float alpha, int causal) {
  pdl_wait();
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nvec = cols >> 3;
  for (long long r = (long long)blockIdx.x * warps + (threadIdx.x >> 5); r < rows;
       r += (long long)gridDim.x * warps) {
    const int qpos = (int)(r % q_len);
    const int lim = causal ? qpos + 1 : cols;
    float v[kPer][8];
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int c = lane + 32 * j;
      if (c < nvec) {
        load8(s + r * cols + c * 8, v[j]);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          v[j][i] = (c * 8 + i < lim) ? v[j][i] * alpha : -INFINITY;
          mx = fmaxf(mx, v[j][i]);
        }
      }
    }
    mx = warp_max(mx);
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int c = lane + 32 * j;
      if (c < nvec) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          v[j][i] = __expf(v[j][i] - mx);
          sum += v[j][i];
        }
      }
    }
    const float inv = 1.f / warp_sum(sum);
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int c = lane + 32 * j;
      if (c < nvec) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[j][i] *= inv;
        store8(p + r * cols + c * 8, v[j]);
      }
    }
  }
}

// dS = alpha * P * (dP - sum_j dP_j P_j)
template <int kPer>
__global__ void __launch_bounds__(256) softmax_bwd_kernel(const __nv_bfloat16* __restrict__ p,
                                                          const __nv_bfloat16* __restrict__ dp,
                                                          __nv_bfloat16* __restrict__ ds,
                                                          long long rows, int cols, float alpha) {
  pdl_wait();
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nvec = cols >> 3;
  for (long long r = (long long)blockIdx.x * warps + (threadIdx.x >> 5); r < rows;
       r += (long long)gridDim.x * warps) {
    float pv[kPer][8], gv[kPer][8];
    float dot = 0.f;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int c = lane + 32 * j;
      if (c < nvec) {
        load8(p + r * cols + c * 8, pv[j]);
        load8(dp + r * cols + c * 8, gv[j]);
#pragma unroll
        for (int i = 0; i < 8; ++i) dot += pv[j][i] * gv[j][i];
      }
    }
    dot = warp_sum(dot);
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int c = lane + 32 * j;
      if (c < nvec) {
        float o[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = alpha * pv[j][i] * (gv[j][i] - dot);
        store8(ds + r * cols + c * 8, o);
      }
    }
  }
}

// ---------------- elementwise ----------------

__global__ void gelu_fwd_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y,
                                long long n8) {
  pdl_wait();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n8;
       i += (long long)gridDim.x * blockDim.x) {
    float v[8];
    load8(x + i * 8, v);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = gelu_tanh(v[k]);
    store8(y + i * 8, v);
  }
}

__global__ void gelu_bwd_kernel(const __nv_bfloat16* __restrict__ dy,
                                const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ dx,
                                long long n8) {
  pdl_wait();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n8;
       i += (long long)gridDim.x * blockDim.x) {
    float g[8], v[8];
    load8(dy + i * 8, g);
    load8(x + i * 8, v);
#pragma unroll
    for (int k = 0; k < 8; ++k) g[k] *= gelu_tanh_grad(v[k]);
    store8(dx + i * 8, g);
  }
}

__global__ void add_kernel(const __nv_bfloat16* a, const __nv_bfloat16* b, __nv_bfloat16* out,
                           long long n8) {
  pdl_wait();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n8;
       i += (long long)gridDim.x * blockDim.x) {
    float u[8], v[8];
    load8(a + i * 8, u);
    load8(b + i * 8, v);
#pragma unroll
    for (int k = 0; k < 8; ++k) u[k] += v[k];
    store8(out + i * 8, u);
  }
}

__global__ void cast_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ y,
                            long long n) {
  pdl_wait();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = __float2bfloat16(x[i]);
}

// ---------------- fused vocabulary cross entropy ----------------
// One CTA per token row; the row (<= 48K bf16) is cached in shared memory so
// logits are read from HBM once and dlogits written once.
__global__ void __launch_bounds__(512) xent_kernel(const __nv_bfloat16* __restrict__ logits,
                                                   long long ld, const int* __restrict__ labels,
                                                   long long rows, int vocab, float grad_scale,
                                                   float loss_scale, float* __restrict__ loss_sum,
                                                   __nv_bfloat16* __restrict__ dlogits) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t xsm[];
  __nv_bfloat16* row = reinterpret_cast<__nv_bfloat16*>(xsm);
  __shared__ float red[32];
  const int tid = threadIdx.x, nw = blockDim.x >> 5;
  const int nvec = (vocab + 7) >> 3;  // columns >= vocab (pad) are masked out
  const int nfull = vocab >> 3;       // vectors with all 8 columns < vocab
  constexpr float kL2e = 1.4426950408889634f;
  for (long long r = blockIdx.x; r < rows; r += gridDim.x) {
    const __nv_bfloat16* src = logits + r * ld;
    // pass 1: row -> smem, row max on packed bf16 pairs (max is exact in bf16)
    __nv_bfloat162 mx2 = __floats2bfloat162_rn(-INFINITY, -INFINITY);
    float mx_tail = -INFINITY;
    constexpr int U = 8;  // 8 row vectors in flight per thread
    for (int c0 = tid; c0 < nvec; c0 += blockDim.x * U) {
      uint4 u[U];
#pragma unroll
      for (int i = 0; i < U; ++i) {
        const int c = c0 + i * blockDim.x;
        if (c < nvec) u[i] = __ldcs(reinterpret_cast<const uint4*>(src) + c);
      }
#pragma unroll
      for (int i = 0; i < U; ++i) {
        const int c = c0 + i * blockDim.x;
        if (c < nvec) {
          reinterpret_cast<uint4*>(row)[c] = u[i];
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u[i]);
          if (c < nfull) {
            mx2 = __hmax2(mx2, __hmax2(__hmax2(h[0], h[1]), __hmax2(h[2], h[3])));
          } else {
            float v[8];
            load8(reinterpret_cast<const __nv_bfloat16*>(&u[i]), v);
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (c * 8 + k < vocab) mx_tail = fmaxf(mx_tail, v[k]);
          }
        }
      }
    }
    float mx = fmaxf(fmaxf(__low2float(mx2), __high2float(mx2)), mx_tail);
    mx = warp_max(mx);
    if ((tid & 31) == 0) red[tid >> 5] = mx;
    __syncthreads();
    if (tid < 32) {
      float m = tid < nw ? red[tid] : -INFINITY;
      m = warp_max(m);
      if (tid == 0) red[0] = m;
    }
    __syncthreads();
    mx = red[0];
    __syncthreads();
    // pass 2: sum of exp2(x log2e - max log2e), two columns per packed FMA
    const float mxl = mx * kL2e;
    float2 s2 = make_float2(0.f, 0.f);
    for (int c = tid; c < nvec; c += blockDim.x) {
      float v[8];
      load8(row + c * 8, v);
      if (c < nfull) {
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
          const float2 a = fma2(make_float2(v[k], v[k + 1]), make_float2(kL2e, kL2e), make_float2(-mxl, -mxl));
          s2 = fma2(make_float2(1.f, 1.f), make_float2(ex2_approx(a.x), ex2_approx(a.y)), s2);
        }
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (c * 8 + k < vocab) s2.x += ex2_approx(fmaf(v[k], kL2e, -mxl));
      }
    }
    float s = warp_sum(s2.x + s2.y);
    if ((tid & 31) == 0) red[tid >> 5] = s;
    __syncthreads();
    if (tid < 32) {
      float t = tid < nw ? red[tid] : 0.f;
      t = warp_sum(t);
      if (tid == 0) red[0] = t;
    }
    __syncthreads();
    const float sum = red[0];
    const float gs = grad_scale / sum;  // dlogit = softmax * grad_scale - onehot * grad_scale
    const int lab = labels[r];
    if (tid == 0) {
      const float xl = __bfloat162float(row[lab]);
      atomicAdd(loss_sum, loss_scale * (logf(sum) + mx - xl));
    }
    // pass 3: dlogits
    __nv_bfloat16* dst = dlogits + r * ld;
    for (int c = tid; c < nvec; c += blockDim.x) {
      float v[8];
      load8(row + c * 8, v);
      if (c < nfull) {
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
          const float2 a = fma2(make_float2(v[k], v[k + 1]), make_float2(kL2e, kL2e), make_float2(-mxl, -mxl));
          const float2 o = mul2(make_float2(ex2_approx(a.x), ex2_approx(a.y)), make_float2(gs, gs));
          v[k] = o.x;
          v[k + 1] = o.y;
        }
        if (c == (lab >> 3)) {
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] -= k == (lab & 7) ? grad_scale : 0.f;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int col = c * 8 + k;
          const float pr = col < vocab ? ex2_approx(fmaf(v[k], kL2e, -mxl)) * gs : 0.f;
          v[k] = col < vocab ? pr - (col == lab ? grad_scale : 0.f) : 0.f;
        }
      }
      store8(dst + c * 8, v);
    }
    // zero the pad columns [vocab, ld) so the dgrad/wgrad GEMMs see clean input
    for (long long c = (long long)nvec * 8 + tid; c < ld; c += blockDim.x) dst[c] = __float2bfloat16(0.f);
    __syncthreads();
  }
}

// ---------------- embeddings ----------------
__global__ void embed_fwd_kernel(const int* __restrict__ ids, const __nv_bfloat16* __restrict__ tok,
                                 const __nv_bfloat16* __restrict__ pos,
                                 __nv_bfloat16* __restrict__ out, long long rows, int seq,
                                 int hidden) {
  pdl_wait();
  const int warps = blockDim.x >> 5, lane = threadIdx.x & 31;
  const int nvec = hidden >> 3;
  for (long long r = (long long)blockIdx.x * warps + (threadIdx.x >> 5); r < rows;
       r += (long long)gridDim.x * warps) {
    const long long id = ids[r];
    const int sp = (int)(r % seq);
    for (int c = lane; c < nvec; c += 32) {
      float a[8], b[8];
      load8(tok + id * hidden + c * 8, a);
      load8(pos + (long long)sp * hidden + c * 8, b);
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] += b[k];
      store8(out + r * hidden + c * 8, a);
    }
  }
}

// Embedding backward: a warp owns one (position, batch slice): it walks the
// slice's rows at that position, adds each row into its token's gradient row
// with 16-byte vector reds, and sums the rows in registers so the position
// gradient gets one vector red per slice (rows at one position no longer all
// hit the same dpos row with scalar atomics).
constexpr int kEmbSlices = 4;
__global__ void __launch_bounds__(256) embed_bwd_kernel(const int* __restrict__ ids,
                                                        const __nv_bfloat16* __restrict__ dout,
                                                        float* __restrict__ dtok, float* __restrict__ dpos,
                                                        long long rows, int seq, int hidden) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int nvec = hidden >> 3;
  const long long batches = rows / seq;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
       w < (long long)seq * kEmbSlices; w += warps) {
    const int sp = (int)(w % seq), sl = (int)(w / seq);
    float acc[kMaxVec][8];
#pragma unroll
    for (int j = 0; j < kMaxVec; ++j)
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[j][k] = 0.f;
    for (long long b = sl; b < batches; b += kEmbSlices) {
      const long long r = b * seq + sp;
      const long long id = ids[r];
#pragma unroll
      for (int j = 0; j < kMaxVec; ++j) {
        const int c = lane + 32 * j;
        if (c < nvec) {
          float g[8];
          load8(dout + r * hidden + c * 8, g);
          red_add_v4(dtok + id * hidden + c * 8, g);
          red_add_v4(dtok + id * hidden + c * 8 + 4, g + 4);
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[j][k] += g[k];
        }
      }
    }
#pragma unroll
    for (int j = 0; j < kMaxVec; ++j) {
      const int c = lane + 32 * j;
      if (c < nvec) {
        red_add_v4(dpos + (long long)sp * hidden + c * 8, acc[j]);
        red_add_v4(dpos + (long long)sp * hidden + c * 8 + 4, acc[j] + 4);
      }
    }
  }
}

// ---------------- AdamW over a flat fp32 parameter buffer ----------------
__global__ void adamw_kernel(float* __restrict__ w, float* __restrict__ m, float* __restrict__ v,
                             const float* __restrict__ g, __nv_bfloat16* __restrict__ out,
                             long long n4, float lr, float b1, float b2, float eps, float wd,
                             float bc1, float bc2, const long long* __restrict__ step_dev) {
  pdl_wait();
  if (step_dev != nullptr) {  // device step counter (CUDA-graph replay): bias corrections here
    const float t = (float)(*step_dev);
    bc1 = 1.f - powf(b1, t);
    bc2 = 1.f - powf(b2, t);
  }
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    float4 wv = reinterpret_cast<float4*>(w)[i];
    float4 mv = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    const float4 gv = reinterpret_cast<const float4*>(g)[i];
    float* wp = &wv.x;
    float* mp = &mv.x;
    float* vp = &vv.x;
    const float* gp = &gv.x;
    float o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      mp[k] = b1 * mp[k] + (1.f - b1) * gp[k];
      vp[k] = b2 * vp[k] + (1.f - b2) * gp[k] * gp[k];
      const float mh = mp[k] / bc1, vh = vp[k] / bc2;
      wp[k] = wp[k] * (1.f - lr * wd) - lr * mh / (sqrtf(vh) + eps);
      o[k] = wp[k];
    }
    reinterpret_cast<float4*>(w)[i] = wv;
    reinterpret_cast<float4*>(m)[i] = mv;
    reinterpret_cast<float4*>(v)[i] = vv;
    uint2 packed;
    packed.x = pack_bf16(o[0], o[1]);
    packed.y = pack_bf16(o[2], o[3]);
    reinterpret_cast<uint2*>(out)[i] = packed;
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace
}  // namespace dpn

using namespace dpn;

#define LN_DISPATCH(KERNEL, GRID, SMEM, ...)                                       \
  do {                                                                             \
    const int nv = (int)((cols / 8 + 31) / 32);                                    \
    cudaStream_t st = (cudaStream_t)stream;                                        \
    switch (nv) {                                                                  \
      case 1: DPN_CHECK_CUDA(launch_pdl(KERNEL<1>, GRID, 256, SMEM, st, __VA_ARGS__)); break;              \
      case 2: DPN_CHECK_CUDA(launch_pdl(KERNEL<2>, GRID, 256, SMEM, st, __VA_ARGS__)); break;              \
      case 3: DPN_CHECK_CUDA(launch_pdl(KERNEL<3>, GRID, 256, SMEM, st, __VA_ARGS__)); break;              \
      case 4: DPN_CHECK_CUDA(launch_pdl(KERNEL<4>, GRID, 256, SMEM, st, __VA_ARGS__)); break;              \
      case 5: DPN_CHECK_CUDA(launch_pdl(KERNEL<5>, GRID, 256, SMEM, st, __VA_ARGS__)); break;              \
      case 6: DPN_CHECK_CUDA(launch_pdl(KERNEL<6>, GRID, 256, SMEM, st, __VA_ARGS__)); break;              \
      case 7: DPN_CHECK_CUDA(launch_pdl(KERNEL<7>, GRID, 256, SMEM, st, __VA_ARGS__)); break;              \
      default: DPN_CHECK_CUDA(launch_pdl(KERNEL<8>, GRID, 256, SMEM, st, __VA_ARGS__)); break;             \
    }                                                                              \
  } while (0)

extern "C" int dpn_layernorm_fwd(const void* x, const void* gamma, const void* beta, void* y,
                                 float* mean, float* rstd, int64_t rows, int64_t cols, float eps,
                                 void* stream) {
  DPN_REQUIRE(cols % 8 == 0 && cols <= 8 * 32 * kMaxVec, "cols must be a multiple of 8, <= 2048");
  DPN_REQUIRE(aligned16(x) && aligned16(y) && aligned16(gamma) && aligned16(beta), "16-byte alignment");
  if (rows == 0) return 0;
  LN_DISPATCH(ln_fwd_kernel, grid_for(rows, 8), 0, (const __nv_bfloat16*)x,
              (const __nv_bfloat16*)gamma, (const __nv_bfloat16*)beta, (__nv_bfloat16*)y, mean, rstd,
              rows, (int)cols, eps);
  DPN_LAUNCH_CHECK();
  return 0;
}

extern "C" int dpn_layernorm_bwd_fused(const void* dy, const void* x, const void* gamma,
                                       const float* mean, const float* rstd, void* dx,
                                       const void* dx_add, float* dgamma, float* dbeta,
                                       float* dbias, int64_t rows, int64_t cols, void* stream) {
  DPN_REQUIRE(cols % 8 == 0 && cols <= 8 * kLnThreads, "cols must be a multiple of 8, <= 2048");
  DPN_REQUIRE(dgamma && dbeta, "the fused LayerNorm backward produces dgamma and dbeta");
  if (rows == 0) return 0;
  const int nvec = (int)(cols / 8);
  const int G = (nvec + 31) / 32;
  const int groups = (kLnThreads / 32) / G;
  // DPN_LN_CTAS CTAs per SM (persistent over bands of rows), at least kLnRows * groups rows each
  const long long per_iter = (long long)groups * kLnRows;
  const long long ctas = 148LL * DPN_LN_CTAS;
  long long per = (rows + ctas - 1) / ctas;
  per = std::max<long long>(per_iter, (per + per_iter - 1) / per_iter * per_iter);
  const unsigned grid = (unsigned)((rows + per - 1) / per);
  const size_t smem = (2 * (kLnThreads / 32) * kLnRows * 2 + (size_t)groups * cols) * sizeof(float);
  static bool attr = false;
  if (!attr) {
    DPN_CHECK_CUDA(cudaFuncSetAttribute(ln_bwd_fused_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  DPN_CHECK_CUDA(launch_pdl(ln_bwd_fused_kernel, dim3(grid), kLnThreads, smem, (cudaStream_t)stream,
                            (const __nv_bfloat16*)dy, (const __nv_bfloat16*)x,
                            (const __nv_bfloat16*)gamma, mean, rstd, (__nv_bfloat16*)dx,
                            (const __nv_bfloat16*)dx_add, rows, (int)cols, per, dgamma, dbeta, dbias));
  DPN_LAUNCH_CHECK();
  return 0;
}

extern "C" int dpn_layernorm_bwd(const void* dy, const void* x, const void* gamma,
                                 const float* mean, const float* rstd, void* dx,
                                 const void* dx_add, float* dgamma, float* dbeta, int64_t rows,
                                 int64_t cols, float* workspace, int64_t workspace_floats,
                                 void* stream) {
  DPN_REQUIRE(cols % 8 == 0 && cols <= 8 * 32 * kMaxVec, "cols must be a multiple of 8, <= 2048");
  if (rows == 0) return 0;
  (void)workspace;
  (void)workspace_floats;
  // dx by a warp-per-row kernel at full occupancy, then the parameter gradients
  // by a column reduction (measured faster than one fused pass whose per-lane
  // parameter partials cap occupancy at 16 warps per SM: 52 vs 46 us at
  // 16384 x 1024 on B200)
  LN_DISPATCH(ln_dx_kernel, grid_for(rows, 8), 0, (const __nv_bfloat16*)dy,
              (const __nv_bfloat16*)x, (const __nv_bfloat16*)gamma, mean, rstd, (__nv_bfloat16*)dx,
              (const __nv_bfloat16*)dx_add, rows, (int)cols);
  DPN_LAUNCH_CHECK();
  if (dgamma || dbeta) {
    DPN_REQUIRE(dgamma && dbeta, "dgamma and dbeta go together");
    long long per;
    const dim3 g = colred_grid(rows, cols, &per);
    DPN_CHECK_CUDA(launch_pdl(colred_kernel<1>, g, kColThreads, 0, (cudaStream_t)stream,
                              (const __nv_bfloat16*)dy, (long long)cols, (const __nv_bfloat16*)x,
                              mean, rstd, rows, (int)cols, per, dgamma, dbeta));
    DPN_LAUNCH_CHECK();
  }
  return 0;
}

#define SOFTMAX_DISPATCH(KERNEL, ...)                                            \
  do {                                                                           \
    const int per = (int)((cols / 8 + 31) / 32);                                 \
    const int g = grid_for(rows, 8);                                             \
    cudaStream_t st = (cudaStream_t)stream;                                      \
    if (per <= 1) DPN_CHECK_CUDA(launch_pdl(KERNEL<1>, g, 256, 0, st, __VA_ARGS__));                     \
    else if (per <= 2) DPN_CHECK_CUDA(launch_pdl(KERNEL<2>, g, 256, 0, st, __VA_ARGS__));                \
    else if (per <= 4) DPN_CHECK_CUDA(launch_pdl(KERNEL<4>, g, 256, 0, st, __VA_ARGS__));                \
    else if (per <= 8) DPN_CHECK_CUDA(launch_pdl(KERNEL<8>, g, 256, 0, st, __VA_ARGS__));                \
    else DPN_REQUIRE(false, "softmax rows longer than 2048 are not supported");  \
  } while (0)

extern "C" int dpn_softmax_fwd(const void* s, void* p, int64_t rows, int64_t cols, int64_t q_len,
                               float alpha, int causal, void* stream) {
  DPN_REQUIRE(cols % 8 == 0, "cols must be a multiple of 8");
  DPN_REQUIRE(q_len > 0, "q_len must be positive");
  if (rows == 0) return 0;
  SOFTMAX_DISPATCH(softmax_fwd_kernel, (const __nv_bfloat16*)s, (__nv_bfloat16*)p, rows, (int)cols,
                   (int)q_len, alpha, causal);
  DPN_LAUNCH_CHECK();
  return 0;
}

extern "C" int dpn_softmax_bwd(const void* p, const void* dp, void* ds, int64_t rows, int64_t cols,
                               float alpha, void* stream) {
  DPN_REQUIRE(cols % 8 == 0, "cols must be a multiple of 8");
  if (rows == 0) return 0;
  SOFTMAX_DISPATCH(softmax_bwd_kernel, (const __nv_bfloat16*)p, (const __nv_bfloat16*)dp,
                   (__nv_bfloat16*)ds, rows, (int)cols, alpha);
  DPN_LAUNCH_CHECK();
  return 0;
}

extern "C" int dpn_gelu_fwd(const void* x, void* y, int64_t n, void* stream) {
  DPN_REQUIRE(n % 8 == 0, "n must be a multiple of 8");
  if (n == 0) return 0;
  DPN_CHECK_CUDA(launch_pdl(gelu_fwd_kernel, grid_for(n / 8, 256), 256, 0, (cudaStream_t)stream, 
      (const __nv_bfloat16*)x, (__nv_bfloat16*)y, n / 8));
  DPN_LAUNCH_CHECK();
  return 0;
}

extern "C" int dpn_gelu_bwd(const void* dy, const void* x, void* dx, int64_t n, void* stream) {
  DPN_REQUIRE(n % 8 == 0, "n must be a multiple of 8");
  if (n == 0) return 0;
  DPN_CHECK_CUDA(launch_pdl(gelu_bwd_kernel, grid_for(n / 8, 256), 256, 0, (cudaStream_t)stream, 
      (const __nv_bfloat16*)dy, (const __nv_bfloat16*)x, (__nv_bfloat16*)dx, n / 8));
  DPN_LAUNCH_CHECK();
  return 0;
}

extern "C" int dpn_add(const void* a, const void* b, void* out, int64_t n, void* stream) {
  DPN_REQUIRE(n % 8 == 0, "n must be a multiple of 8");
  if (n == 0) return 0;
  DPN_CHECK_CUDA(launch_pdl(add_kernel, grid_for(n / 8, 256), 256, 0, (cudaStream_t)stream, 
      (const __nv_bfloat16*)a, (const __nv_bfloat16*)b, (__nv_bfloat16*)out, n / 8));
  DPN_LAUNCH_CHECK();
  return 0;
}

extern "C" int dpn_cast_f32_bf16(const float* x, void* y, int64_t n, void* stream) {
  if (n == 0) return 0;
  DPN_CHECK_CUDA(launch_pdl(cast_kernel, grid_for(n, 256), 256, 0, (cudaStream_t)stream, x, (__nv_bfloat16*)y, n));
  DPN_LAUNCH_CHECK();
  return 0;
}

extern "C" int dpn_colsum(const void* x, int64_t rows, int64_t cols, int64_t ld, float* out,
                          float* workspace, int64_t workspace_floats, void* stream) {
  DPN_REQUIRE(cols % 8 == 0 && ld % 8 == 0, "cols and ld must be multiples of 8");
  if (rows == 0) return 0;
  (void)workspace;
  (void)workspace_floats;
  long long per;
  const dim3 g = colred_grid(rows, cols, &per);
  DPN_CHECK_CUDA(launch_pdl(colred_kernel<0>, g, kColThreads, 0, (cudaStream_t)stream,
                            (const __nv_bfloat16*)x, (long long)ld, (const __nv_bfloat16*)nullptr,
                            (const float*)nullptr, (const float*)nullptr, rows, (int)cols, per,
                            out, (float*)nullptr));
  DPN_LAUNCH_CHECK();
  return 0;
}

extern "C" int dpn_xent(const void* logits, int64_t ld, const int32_t* labels, int64_t rows,
                        int64_t vocab, float grad_scale, float loss_scale, float* loss_sum,
                        void* dlogits, void* stream) {
  DPN_REQUIRE(ld % 8 == 0 && (vocab + 7) / 8 * 8 <= ld, "ld must be a multiple of 8 and cover vocab rounded up to 8");
  DPN_REQUIRE(ld * 2 <= 200 * 1024, "vocab row must fit in shared memory");
  if (rows == 0) return 0;
  const size_t smem = (size_t)(vocab + 7) / 8 * 16;
  static bool set = false;
  if (!set) {
    DPN_CHECK_CUDA(cudaFuncSetAttribute(xent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        200 * 1024));
    set = true;
  }
  DPN_CHECK_CUDA(launch_pdl(xent_kernel, (int)std::min<long long>(rows, 148 * 4), 512, smem, (cudaStream_t)stream, 
      (const __nv_bfloat16*)logits, ld, labels, rows, (int)vocab, grad_scale, loss_scale, loss_sum,
      (__nv_bfloat16*)dlogits));
  DPN_LAUNCH_CHECK();
  return 0;
}

extern "C" int dpn_embed_fwd(const int32_t* ids, const void* tok, const void* pos, void* out,
                             int64_t rows, int64_t seq, int64_t hidden, void* stream) {
  DPN_REQUIRE(hidden % 8 == 0, "hidden must be a multiple of 8");
  if (rows == 0) return 0;
  DPN_CHECK_CUDA(launch_pdl(embed_fwd_kernel, grid_for(rows, 8), 256, 0, (cudaStream_t)stream, 
      ids, (const __nv_bfloat16*)tok, (const __nv_bfloat16*)pos, (__nv_bfloat16*)out, rows,
      (int)seq, (int)hidden));
  DPN_LAUNCH_CHECK();
  return 0;
}

extern "C" int dpn_embed_bwd(const int32_t* ids, const void* dout, float* dtok, float* dpos,
                             int64_t rows, int64_t seq, int64_t hidden, void* stream) {
  DPN_REQUIRE(hidden % 8 == 0 && hidden <= 8 * 32 * kMaxVec, "hidden must be a multiple of 8, <= 2048");
  DPN_REQUIRE(seq > 0 && rows % seq == 0, "rows must be a whole number of sequences");
  DPN_REQUIRE(((uintptr_t)dtok & 15) == 0 && ((uintptr_t)dpos & 15) == 0, "dtok / dpos 16-byte alignment");
  if (rows == 0) return 0;
  DPN_CHECK_CUDA(launch_pdl(embed_bwd_kernel, grid_for(seq * kEmbSlices, 8), 256, 0, (cudaStream_t)stream, 
      ids, (const __nv_bfloat16*)dout, dtok, dpos, rows, (int)seq, (int)hidden));
  DPN_LAUNCH_CHECK();
  return 0;
}

extern "C" int dpn_adamw(float* w, float* m, float* v, const float* g, void* out_bf16, int64_t n,
                         float lr, float beta1, float beta2, float eps, float wd, int64_t step,
                         void* stream) {
  DPN_REQUIRE(n % 4 == 0, "n must be a multiple of 4");
  DPN_REQUIRE(step >= 1, "step counts from 1");
  if (n == 0) return 0;
  const float bc1 = 1.f - powf(beta1, (float)step), bc2 = 1.f - powf(beta2, (float)step);
  DPN_CHECK_CUDA(launch_pdl(adamw_kernel, grid_for(n / 4, 256), 256, 0, (cudaStream_t)stream, 
      w, m, v, g, (__nv_bfloat16*)out_bf16, n / 4, lr, beta1, beta2, eps, wd, bc1, bc2,
      (const long long*)nullptr));
  DPN_LAUNCH_CHECK();
  return 0;
}

__global__ void step_increment_kernel(long long* step) { *step += 1; }

// AdamW whose step count lives in device memory: `step_dev` is incremented and
// then read by the update (so a CUDA graph replays with the right bias
// corrections every time).
extern "C" int dpn_adamw_dstep(float* w, float* m, float* v, const float* g, void* out_bf16,
                               int64_t n, float lr, float beta1, float beta2, float eps, float wd,
                               int64_t* step_dev, void* stream) {
  DPN_REQUIRE(n % 4 == 0 && step_dev != nullptr, "n must be a multiple of 4; step_dev required");
  if (n == 0) return 0;
  step_increment_kernel<<<1, 1, 0, (cudaStream_t)stream>>>((long long*)step_dev);
  DPN_LAUNCH_CHECK();
  DPN_CHECK_CUDA(launch_pdl(adamw_kernel, grid_for(n / 4, 256), 256, 0, (cudaStream_t)stream,
      w, m, v, g, (__nv_bfloat16*)out_bf16, n / 4, lr, beta1, beta2, eps, wd, 1.f, 1.f,
      (const long long*)step_dev));
  DPN_LAUNCH_CHECK();
  return 0;
}
