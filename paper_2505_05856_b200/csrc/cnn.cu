// CNN node kernels (AmoebaNet-D, BASELINE.json configs[4]) for sm_100a.
//
// Activations are NHWC bf16 viewed as [pixels, channels] (pixels = b*H*W),
// every thread moves 8 channels (one 16-byte vector), so each warp touches
// 512 contiguous bytes per pixel row.  The dense 1x1 convolutions are tcgen05
// GEMMs over that view (gemm.cu); the stem's 3x3 convolution is an im2col
// pass + GEMM.  What is here is the HBM-bound remainder:
//
//   relu      fwd / bwd (mask from the saved output)
//   dwconv    3x3 depthwise convolution (stride 1/2, pad 1): fwd, data grad
//             (gather form, no atomics), weight grad (per-block shared-memory
//             reduction, one global atomic per weight per block)
//   bn        training-mode batch norm: column statistics (sum, sum of squares
//             in f32), apply; backward = column reductions (sum dy, sum dy*xhat)
//             into a per-micro-batch workspace + elementwise dx that also
//             accumulates dgamma / dbeta
//   pool      3x3 max / average pooling (stride 1/2, pad 1; average excludes
//             padding); max saves the argmax tap (uint8) for its backward
//   copy_cols strided column-slice copies (channel concat fwd / bwd)
//   im2col    3x3 patches for the stem convolution
//   gap       global average pool over pixels per sample, and its backward
#include "common.cuh"
#include "../../include/dawnpiper.h"

#include <algorithm>

namespace dpn {
namespace {

constexpr int kT = 256;

int blocks_for(long long items) {
  long long g = (items + kT - 1) / kT;
  return (int)std::max<long long>(1, std::min<long long>(g, 148LL * 32));
}

__device__ __forceinline__ void ld8(const __nv_bfloat16* p, float* f) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

__device__ __forceinline__ void st8(__nv_bfloat16* p, const float* f) {
  uint4 u;
  u.x = pack_bf16(f[0], f[1]);
  u.y = pack_bf16(f[2], f[3]);
  u.z = pack_bf16(f[4], f[5]);
  u.w = pack_bf16(f[6], f[7]);
  *reinterpret_cast<uint4*>(p) = u;
}

// ---------------- ReLU ----------------
__global__ void relu_fwd_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y,
                                long long n8) {
  pdl_wait();
  for (long long i = (long long)blockIdx.x * kT + threadIdx.x; i < n8; i += (long long)gridDim.x * kT) {
    float f[8];
    ld8(x + 8 * i, f);
#pragma unroll
    for (int k = 0; k < 8; ++k) f[k] = fmaxf(f[k], 0.f);
    st8(y + 8 * i, f);
  }
}

__global__ void relu_bwd_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ y,
                                __nv_bfloat16* __restrict__ dx, long long n8) {
  pdl_wait();
  for (long long i = (long long)blockIdx.x * kT + threadIdx.x; i < n8; i += (long long)gridDim.x * kT) {
    float g[8], o[8];
    ld8(dy + 8 * i, g);
    ld8(y + 8 * i, o);
#pragma unroll
    for (int k = 0; k < 8; ++k) g[k] = o[k] > 0.f ? g[k] : 0.f;
    st8(dx + 8 * i, g);
  }
}

// ---------------- depthwise 3x3 ----------------
struct Geo {
  int b, H, W, C, Ho, Wo, stride;
};

// w: [C, 9] bf16 (tap r*3+s)
__global__ void dw_fwd_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w,
                              __nv_bfloat16* __restrict__ y, Geo g) {
  pdl_wait();
  const int G = g.C / 8;
  const long long total = (long long)g.b * g.Ho * g.Wo * G;
  for (long long i = (long long)blockIdx.x * kT + threadIdx.x; i < total; i += (long long)gridDim.x * kT) {
    const int cg = (int)(i % G);
    long long p = i / G;
    const int wo = (int)(p % g.Wo);
    p /= g.Wo;
    const int ho = (int)(p % g.Ho);
    const int n = (int)(p / g.Ho);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int h = ho * g.stride - 1 + r;
      if (h < 0 || h >= g.H) continue;
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        const int ww = wo * g.stride - 1 + s;
        if (ww < 0 || ww >= g.W) continue;
        float f[8];
        ld8(x + (((long long)n * g.H + h) * g.W + ww) * g.C + cg * 8, f);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] += f[k] * __bfloat162float(w[(cg * 8 + k) * 9 + r * 3 + s]);
      }
    }
    st8(y + i * 8, acc);
  }
}

// dx[n,h,w,c] = sum_{r,s: (h+1-r) % stride == 0} dy[n,(h+1-r)/stride,(w+1-s)/stride,c] * w[c,r,s]
__global__ void dw_dgrad_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ w,
                                __nv_bfloat16* __restrict__ dx, Geo g) {
  pdl_wait();
  const int G = g.C / 8;
  const long long total = (long long)g.b * g.H * g.W * G;
  for (long long i = (long long)blockIdx.x * kT + threadIdx.x; i < total; i += (long long)gridDim.x * kT) {
    const int cg = (int)(i % G);
    long long p = i / G;
    const int x0 = (int)(p % g.W);
    p /= g.W;
    const int h0 = (int)(p % g.H);
    const int n = (int)(p / g.H);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int hn = h0 + 1 - r;
      if (hn < 0 || hn % g.stride) continue;
      const int ho = hn / g.stride;
      if (ho >= g.Ho) continue;
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        const int wn = x0 + 1 - s;
        if (wn < 0 || wn % g.stride) continue;
        const int wo = wn / g.stride;
        if (wo >= g.Wo) continue;
        float f[8];
        ld8(dy + (((long long)n * g.Ho + ho) * g.Wo + wo) * g.C + cg * 8, f);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] += f[k] * __bfloat162float(w[(cg * 8 + k) * 9 + r * 3 + s]);
      }
    }
    st8(dx + i * 8, acc);
  }
}

// dw[c, r, s] += sum_p dy[p, c] * x[shift(p, r, s), c]; thread t owns channel
// group t % G of a strided set of output pixels; block partials meet in
// shared memory (9 * C floats), then one global atomic per weight per block.
__global__ void dw_wgrad_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ dy,
                                float* __restrict__ dw, Geo g, long long px_per_block) {
  extern __shared__ float red[];  // [9 * C]
  pdl_wait();
  const int G = g.C / 8;
  for (int i = threadIdx.x; i < 9 * g.C; i += kT) red[i] = 0.f;
  __syncthreads();
  const int lanes = (kT / G) * G;
  if (threadIdx.x < lanes) {
    const int cg = threadIdx.x % G;
    const int j = threadIdx.x / G;
    const int rows = kT / G;
    const long long P = (long long)g.b * g.Ho * g.Wo;
    const long long p0 = blockIdx.x * px_per_block;
    const long long p1 = min(P, p0 + px_per_block);
    float acc[9][8];
#pragma unroll
    for (int t = 0; t < 9; ++t)
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[t][k] = 0.f;
    for (long long p = p0 + j; p < p1; p += rows) {
      const int wo = (int)(p % g.Wo);
      const long long q = p / g.Wo;
      const int ho = (int)(q % g.Ho);
      const int n = (int)(q / g.Ho);
      float d[8];
      ld8(dy + p * g.C + cg * 8, d);
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const int h = ho * g.stride - 1 + r;
        if (h < 0 || h >= g.H) continue;
#pragma unroll
        for (int s = 0; s < 3; ++s) {
          const int ww = wo * g.stride - 1 + s;
          if (ww < 0 || ww >= g.W) continue;
          float f[8];
          ld8(x + (((long long)n * g.H + h) * g.W + ww) * g.C + cg * 8, f);
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[r * 3 + s][k] += d[k] * f[k];
        }
      }
    }
#pragma unroll
    for (int t = 0; t < 9; ++t)
#pragma unroll
      for (int k = 0; k < 8; ++k) atomicAdd(&red[(cg * 8 + k) * 9 + t], acc[t][k]);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 9 * g.C; i += kT) atomicAdd(&dw[i], red[i]);
}

// ---------------- column statistics / reductions (BN) ----------------
// mode 0: out[0,c] += sum x, out[1,c] += sum x^2
// mode 1: out[0,c] += sum dy, out[1,c] += sum dy * xhat  (xhat from the BN sums `st`)
template <int MODE>
__global__ void colstat_kernel(const __nv_bfloat16* __restrict__ a, const __nv_bfloat16* __restrict__ xb,
                               const float* __restrict__ st, float eps, long long P, int C,
                               long long px_per_block, float* __restrict__ out) {
  extern __shared__ float red[];  // [2 * C]
  pdl_wait();
  const int G = C / 8;
  for (int i = threadIdx.x; i < 2 * C; i += kT) red[i] = 0.f;
  __syncthreads();
  const int lanes = (kT / G) * G;
  if (threadIdx.x < lanes) {
    const int cg = threadIdx.x % G;
    const int j = threadIdx.x / G;
    const int rows = kT / G;
    const long long p0 = blockIdx.x * px_per_block;
    const long long p1 = min(P, p0 + px_per_block);
    float s0[8], s1[8], mean[8], rstd[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      s0[k] = s1[k] = 0.f;
      if (MODE == 1) {
        const int c = cg * 8 + k;
        mean[k] = st[c] / (float)P;
        const float var = fmaxf(st[C + c] / (float)P - mean[k] * mean[k], 0.f);
        rstd[k] = rsqrtf(var + eps);
      }
    }
    for (long long p = p0 + j; p < p1; p += rows) {
      float f[8];
      ld8(a + p * C + cg * 8, f);
      if (MODE == 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          s0[k] += f[k];
          s1[k] += f[k] * f[k];
        }
      } else {
        float xv[8];
        ld8(xb + p * C + cg * 8, xv);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          s0[k] += f[k];
          s1[k] += f[k] * (xv[k] - mean[k]) * rstd[k];
        }
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      atomicAdd(&red[cg * 8 + k], s0[k]);
      atomicAdd(&red[C + cg * 8 + k], s1[k]);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * C; i += kT) atomicAdd(&out[i], red[i]);
}

// y = (x - mean) * rstd * gamma + beta
__global__ void bn_apply_kernel(const __nv_bfloat16* __restrict__ x, const float* __restrict__ st,
                                const __nv_bfloat16* __restrict__ gamma,
                                const __nv_bfloat16* __restrict__ beta, float eps, long long P, int C,
                                __nv_bfloat16* __restrict__ y) {
  pdl_wait();
  const int G = C / 8;
  const long long total = P * G;
  for (long long i = (long long)blockIdx.x * kT + threadIdx.x; i < total; i += (long long)gridDim.x * kT) {
    const int cg = (int)(i % G);
    float f[8];
    ld8(x + i * 8, f);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int c = cg * 8 + k;
      const float mean = st[c] / (float)P;
      const float var = fmaxf(st[C + c] / (float)P - mean * mean, 0.f);
      f[k] = (f[k] - mean) * rsqrtf(var + eps) * __bfloat162float(gamma[c]) + __bfloat162float(beta[c]);
    }
    st8(y + i * 8, f);
  }
}

// dx = gamma * rstd * (dy - sum_dy / P - xhat * sum_dyxhat / P); block 0 also
// accumulates this micro-batch's sums into dbeta / dgamma.
__global__ void bn_dx_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
                             const float* __restrict__ st, const __nv_bfloat16* __restrict__ gamma,
                             const float* __restrict__ red, float eps, long long P, int C,
                             __nv_bfloat16* __restrict__ dx, float* __restrict__ dgamma,
                             float* __restrict__ dbeta) {
  pdl_wait();
  if (blockIdx.x == 0) {
    for (int c = threadIdx.x; c < C; c += kT) {
      dbeta[c] += red[c];
      dgamma[c] += red[C + c];
    }
  }
  const int G = C / 8;
  const long long total = P * G;
  for (long long i = (long long)blockIdx.x * kT + threadIdx.x; i < total; i += (long long)gridDim.x * kT) {
    const int cg = (int)(i % G);
    float g[8], xv[8];
    ld8(dy + i * 8, g);
    ld8(x + i * 8, xv);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int c = cg * 8 + k;
      const float mean = st[c] / (float)P;
      const float var = fmaxf(st[C + c] / (float)P - mean * mean, 0.f);
      const float rstd = rsqrtf(var + eps);
      const float xh = (xv[k] - mean) * rstd;
      g[k] = __bfloat162float(gamma[c]) * rstd *
             (g[k] - red[c] / (float)P - xh * red[C + c] / (float)P);
    }
    st8(dx + i * 8, g);
  }
}

// ---------------- 3x3 pooling ----------------
// mode 0: max (argmax tap saved as uint8), mode 1: average excluding padding
__global__ void pool_fwd_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y,
                                uint8_t* __restrict__ arg, Geo g, int mode) {
  pdl_wait();
  const int G = g.C / 8;
  const long long total = (long long)g.b * g.Ho * g.Wo * G;
  for (long long i = (long long)blockIdx.x * kT + threadIdx.x; i < total; i += (long long)gridDim.x * kT) {
    const int cg = (int)(i % G);
    long long p = i / G;
    const int wo = (int)(p % g.Wo);
    p /= g.Wo;
    const int ho = (int)(p % g.Ho);
    const int n = (int)(p / g.Ho);
    float acc[8];
    uint8_t am[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      acc[k] = mode == 0 ? -INFINITY : 0.f;
      am[k] = 0;
    }
    int cnt = 0;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int h = ho * g.stride - 1 + r;
      if (h < 0 || h >= g.H) continue;
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        const int ww = wo * g.stride - 1 + s;
        if (ww < 0 || ww >= g.W) continue;
        float f[8];
        ld8(x + (((long long)n * g.H + h) * g.W + ww) * g.C + cg * 8, f);
        ++cnt;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (mode == 0) {
            if (f[k] > acc[k]) {
              acc[k] = f[k];
              am[k] = (uint8_t)(r * 3 + s);
            }
          } else {
            acc[k] += f[k];
          }
        }
      }
    }
    if (mode == 1) {
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] /= (float)cnt;
    } else {
      uint2 packed;
      packed.x = am[0] | (am[1] << 8) | (am[2] << 16) | ((uint32_t)am[3] << 24);
      packed.y = am[4] | (am[5] << 8) | (am[6] << 16) | ((uint32_t)am[7] << 24);
      *reinterpret_cast<uint2*>(arg + i * 8) = packed;
    }
    st8(y + i * 8, acc);
  }
}

// gather form: every input pixel sums the gradients of the windows that used it
__global__ void pool_bwd_kernel(const __nv_bfloat16* __restrict__ dy, const uint8_t* __restrict__ arg,
                                __nv_bfloat16* __restrict__ dx, Geo g, int mode) {
  pdl_wait();
  const int G = g.C / 8;
  const long long total = (long long)g.b * g.H * g.W * G;
  for (long long i = (long long)blockIdx.x * kT + threadIdx.x; i < total; i += (long long)gridDim.x * kT) {
    const int cg = (int)(i % G);
    long long p = i / G;
    const int x0 = (int)(p % g.W);
    p /= g.W;
    const int h0 = (int)(p % g.H);
    const int n = (int)(p / g.H);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int hn = h0 + 1 - r;
      if (hn < 0 || hn % g.stride) continue;
      const int ho = hn / g.stride;
      if (ho >= g.Ho) continue;
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        const int wn = x0 + 1 - s;
        if (wn < 0 || wn % g.stride) continue;
        const int wo = wn / g.stride;
        if (wo >= g.Wo) continue;
        const long long o = (((long long)n * g.Ho + ho) * g.Wo + wo) * g.C + cg * 8;
        float f[8];
        ld8(dy + o, f);
        if (mode == 0) {
          const uint2 packed = *reinterpret_cast<const uint2*>(arg + o);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t word = k < 4 ? packed.x : packed.y;
            const int tap = (word >> (8 * (k & 3))) & 0xff;
            if (tap == r * 3 + s) acc[k] += f[k];
          }
        } else {
          // window of output (ho, wo): rows ho*stride-1 .. +1, cols likewise, clipped
          const int hlo = max(ho * g.stride - 1, 0), hhi = min(ho * g.stride + 1, g.H - 1);
          const int wlo = max(wo * g.stride - 1, 0), whi = min(wo * g.stride + 1, g.W - 1);
          const float inv = 1.f / (float)((hhi - hlo + 1) * (whi - wlo + 1));
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[k] += f[k] * inv;
        }
      }
    }
    st8(dx + i * 8, acc);
  }
}

// ---------------- strided column copies (concat) ----------------
__global__ void copy_cols_kernel(const __nv_bfloat16* __restrict__ src, long long lds,
                                 __nv_bfloat16* __restrict__ dst, long long ldd, long long rows, int cols,
                                 int accumulate) {
  pdl_wait();
  const int G = cols / 8;
  const long long total = rows * G;
  for (long long i = (long long)blockIdx.x * kT + threadIdx.x; i < total; i += (long long)gridDim.x * kT) {
    const long long r = i / G;
    const int cg = (int)(i % G);
    const uint4 u = *reinterpret_cast<const uint4*>(src + r * lds + cg * 8);
    uint4* d = reinterpret_cast<uint4*>(dst + r * ldd + cg * 8);
    if (accumulate) {
      float a[8], b[8];
      ld8(reinterpret_cast<const __nv_bfloat16*>(&u), a);
      ld8(reinterpret_cast<const __nv_bfloat16*>(d), b);
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] += b[k];
      st8(reinterpret_cast<__nv_bfloat16*>(d), a);
    } else {
      *d = u;
    }
  }
}

// ---------------- stem im2col (3x3, pad 1) ----------------
// cols[p, (r*3+s)*C + c] = x[n, ho*stride-1+r, wo*stride-1+s, c] (0 outside)
__global__ void im2col_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ cols, Geo g) {
  pdl_wait();
  const int G = g.C / 8;
  const long long total = (long long)g.b * g.Ho * g.Wo * 9 * G;
  for (long long i = (long long)blockIdx.x * kT + threadIdx.x; i < total; i += (long long)gridDim.x * kT) {
    const int cg = (int)(i % G);
    long long q = i / G;
    const int tap = (int)(q % 9);
    const long long p = q / 9;
    const int wo = (int)(p % g.Wo);
    const long long t = p / g.Wo;
    const int ho = (int)(t % g.Ho);
    const int n = (int)(t / g.Ho);
    const int h = ho * g.stride - 1 + tap / 3, ww = wo * g.stride - 1 + tap % 3;
    uint4 u = make_uint4(0, 0, 0, 0);
    if (h >= 0 && h < g.H && ww >= 0 && ww < g.W)
      u = *reinterpret_cast<const uint4*>(x + (((long long)n * g.H + h) * g.W + ww) * g.C + cg * 8);
    *reinterpret_cast<uint4*>(cols + p * 9 * g.C + tap * g.C + cg * 8) = u;
  }
}

// ---------------- global average pool ----------------
// y[n, c] = mean_p x[n*HW + p, c]
__global__ void gap_fwd_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y, int HW,
                               int C) {
  pdl_wait();
  const int n = blockIdx.x;
  for (int c = threadIdx.x; c < C; c += kT) {
    float s = 0.f;
    for (int p = 0; p < HW; ++p) s += __bfloat162float(x[((long long)n * HW + p) * C + c]);
    y[(long long)n * C + c] = __float2bfloat16(s / (float)HW);
  }
}

__global__ void gap_bwd_kernel(const __nv_bfloat16* __restrict__ dy, __nv_bfloat16* __restrict__ dx,
                               long long P, int HW, int C) {
  pdl_wait();
  const int G = C / 8;
  const long long total = P * G;
  for (long long i = (long long)blockIdx.x * kT + threadIdx.x; i < total; i += (long long)gridDim.x * kT) {
    const long long p = i / G;
    const int cg = (int)(i % G);
    float f[8];
    ld8(dy + (p / HW) * C + cg * 8, f);
#pragma unroll
    for (int k = 0; k < 8; ++k) f[k] /= (float)HW;
    st8(dx + i * 8, f);
  }
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

Geo geo(int64_t b, int64_t H, int64_t W, int64_t C, int64_t stride) {
  Geo g;
  g.b = (int)b;
  g.H = (int)H;
  g.W = (int)W;
  g.C = (int)C;
  g.stride = (int)stride;
  g.Ho = (int)((H - 1) / stride + 1);  // 3x3, pad 1
  g.Wo = (int)((W - 1) / stride + 1);
  return g;
}

long long px_block(long long P, int C, long long* blocks) {
  // ~2 blocks per SM, at least 64 pixels per block
  long long per = std::max<long long>(64, (P + 295) / 296);
  *blocks = (P + per - 1) / per;
  (void)C;
  return per;
}

}  // namespace
}  // namespace dpn

using namespace dpn;

#define CNN_CHECK_C(C) DPN_REQUIRE((C) % 8 == 0 && (C) > 0 && (C) <= 2048, "channels must be a multiple of 8 in [8, 2048]")

extern "C" int dpn_relu_fwd(const void* x, void* y, int64_t n, void* stream) {
  DPN_REQUIRE(n % 8 == 0 && al16(x) && al16(y), "n % 8 and 16-byte alignment");
  if (n == 0) return 0;
  DPN_CHECK_CUDA(launch_pdl(relu_fwd_kernel, blocks_for(n / 8), kT, 0, (cudaStream_t)stream,
                            (const __nv_bfloat16*)x, (__nv_bfloat16*)y, (long long)(n / 8)));
  return 0;
}

extern "C" int dpn_relu_bwd(const void* dy, const void* y, void* dx, int64_t n, void* stream) {
  DPN_REQUIRE(n % 8 == 0 && al16(dy) && al16(y) && al16(dx), "n % 8 and 16-byte alignment");
  if (n == 0) return 0;
  DPN_CHECK_CUDA(launch_pdl(relu_bwd_kernel, blocks_for(n / 8), kT, 0, (cudaStream_t)stream,
                            (const __nv_bfloat16*)dy, (const __nv_bfloat16*)y, (__nv_bfloat16*)dx,
                            (long long)(n / 8)));
  return 0;
}

extern "C" int dpn_dwconv3_fwd(const void* x, const void* w, void* y, int64_t b, int64_t H, int64_t W,
                               int64_t C, int64_t stride, void* stream) {
  CNN_CHECK_C(C);
  DPN_REQUIRE(stride == 1 || stride == 2, "stride must be 1 or 2");
  const Geo g = geo(b, H, W, C, stride);
  DPN_CHECK_CUDA(launch_pdl(dw_fwd_kernel, blocks_for((long long)b * g.Ho * g.Wo * (C / 8)), kT, 0,
                            (cudaStream_t)stream, (const __nv_bfloat16*)x, (const __nv_bfloat16*)w,
                            (__nv_bfloat16*)y, g));
  return 0;
}

extern "C" int dpn_dwconv3_bwd(const void* x, const void* w, const void* dy, void* dx, float* dw,
                               int64_t b, int64_t H, int64_t W, int64_t C, int64_t stride, void* stream) {
  CNN_CHECK_C(C);
  DPN_REQUIRE(stride == 1 || stride == 2, "stride must be 1 or 2");
  const Geo g = geo(b, H, W, C, stride);
  cudaStream_t st = (cudaStream_t)stream;
  if (dx)
    DPN_CHECK_CUDA(launch_pdl(dw_dgrad_kernel, blocks_for((long long)b * H * W * (C / 8)), kT, 0, st,
                              (const __nv_bfloat16*)dy, (const __nv_bfloat16*)w, (__nv_bfloat16*)dx, g));
  if (dw) {
    long long blocks;
    const long long per = px_block((long long)b * g.Ho * g.Wo, (int)C, &blocks);
    DPN_CHECK_CUDA(launch_pdl(dw_wgrad_kernel, (int)blocks, kT, (size_t)(9 * C * 4), st,
                              (const __nv_bfloat16*)x, (const __nv_bfloat16*)dy, dw, g, per));
  }
  return 0;
}

extern "C" int dpn_bn_fwd(const void* x, const void* gamma, const void* beta, void* y, float* stats,
                          int64_t P, int64_t C, float eps, void* stream) {
  CNN_CHECK_C(C);
  cudaStream_t st = (cudaStream_t)stream;
  DPN_CHECK_CUDA(cudaMemsetAsync(stats, 0, 2 * C * sizeof(float), st));
  long long blocks;
  const long long per = px_block(P, (int)C, &blocks);
  DPN_CHECK_CUDA(launch_pdl(colstat_kernel<0>, (int)blocks, kT, (size_t)(2 * C * 4), st,
                            (const __nv_bfloat16*)x, (const __nv_bfloat16*)nullptr, (const float*)nullptr,
                            eps, (long long)P, (int)C, per, stats));
  DPN_CHECK_CUDA(launch_pdl(bn_apply_kernel, blocks_for(P * (C / 8)), kT, 0, st, (const __nv_bfloat16*)x,
                            (const float*)stats, (const __nv_bfloat16*)gamma, (const __nv_bfloat16*)beta,
                            eps, (long long)P, (int)C, (__nv_bfloat16*)y));
  return 0;
}

extern "C" int dpn_bn_bwd(const void* dy, const void* x, const float* stats, const void* gamma, void* dx,
                          float* dgamma, float* dbeta, float* workspace, int64_t P, int64_t C, float eps,
                          void* stream) {
  CNN_CHECK_C(C);
  DPN_REQUIRE(workspace != nullptr, "workspace of 2*C floats required");
  cudaStream_t st = (cudaStream_t)stream;
  DPN_CHECK_CUDA(cudaMemsetAsync(workspace, 0, 2 * C * sizeof(float), st));
  long long blocks;
  const long long per = px_block(P, (int)C, &blocks);
  DPN_CHECK_CUDA(launch_pdl(colstat_kernel<1>, (int)blocks, kT, (size_t)(2 * C * 4), st,
                            (const __nv_bfloat16*)dy, (const __nv_bfloat16*)x, stats, eps, (long long)P,
                            (int)C, per, workspace));
  DPN_CHECK_CUDA(launch_pdl(bn_dx_kernel, blocks_for(P * (C / 8)), kT, 0, st, (const __nv_bfloat16*)dy,
                            (const __nv_bfloat16*)x, stats, (const __nv_bfloat16*)gamma,
                            (const float*)workspace, eps, (long long)P, (int)C, (__nv_bfloat16*)dx, dgamma,
                            dbeta));
  return 0;
}

extern "C" int dpn_pool3_fwd(const void* x, void* y, void* argmax, int64_t b, int64_t H, int64_t W,
                             int64_t C, int64_t stride, int mode, void* stream) {
  CNN_CHECK_C(C);
  DPN_REQUIRE(stride == 1 || stride == 2, "stride must be 1 or 2");
  DPN_REQUIRE(mode == 0 || mode == 1, "mode 0 (max) or 1 (average)");
  DPN_REQUIRE(mode == 1 || argmax != nullptr, "max pooling saves its argmax");
  const Geo g = geo(b, H, W, C, stride);
  DPN_CHECK_CUDA(launch_pdl(pool_fwd_kernel, blocks_for((long long)b * g.Ho * g.Wo * (C / 8)), kT, 0,
                            (cudaStream_t)stream, (const __nv_bfloat16*)x, (__nv_bfloat16*)y,
                            (uint8_t*)argmax, g, mode));
  return 0;
}

extern "C" int dpn_pool3_bwd(const void* dy, const void* argmax, void* dx, int64_t b, int64_t H, int64_t W,
                             int64_t C, int64_t stride, int mode, void* stream) {
  CNN_CHECK_C(C);
  DPN_REQUIRE(stride == 1 || stride == 2, "stride must be 1 or 2");
  DPN_REQUIRE(mode == 1 || argmax != nullptr, "max pooling backward needs the argmax");
  const Geo g = geo(b, H, W, C, stride);
  DPN_CHECK_CUDA(launch_pdl(pool_bwd_kernel, blocks_for((long long)b * H * W * (C / 8)), kT, 0,
                            (cudaStream_t)stream, (const __nv_bfloat16*)dy, (const uint8_t*)argmax,
                            (__nv_bfloat16*)dx, g, mode));
  return 0;
}

extern "C" int dpn_copy_cols(const void* src, int64_t lds, void* dst, int64_t ldd, int64_t rows,
                             int64_t cols, int accumulate, void* stream) {
  DPN_REQUIRE(cols % 8 == 0 && lds % 8 == 0 && ldd % 8 == 0 && al16(src) && al16(dst),
              "cols / strides multiples of 8, 16-byte alignment");
  if (rows == 0 || cols == 0) return 0;
  DPN_CHECK_CUDA(launch_pdl(copy_cols_kernel, blocks_for(rows * (cols / 8)), kT, 0, (cudaStream_t)stream,
                            (const __nv_bfloat16*)src, (long long)lds, (__nv_bfloat16*)dst, (long long)ldd,
                            (long long)rows, (int)cols, accumulate));
  return 0;
}

extern "C" int dpn_im2col3(const void* x, void* cols, int64_t b, int64_t H, int64_t W, int64_t C,
                           int64_t stride, void* stream) {
  CNN_CHECK_C(C);
  const Geo g = geo(b, H, W, C, stride);
  DPN_CHECK_CUDA(launch_pdl(im2col_kernel, blocks_for((long long)b * g.Ho * g.Wo * 9 * (C / 8)), kT, 0,
                            (cudaStream_t)stream, (const __nv_bfloat16*)x, (__nv_bfloat16*)cols, g));
  return 0;
}

extern "C" int dpn_gap_fwd(const void* x, void* y, int64_t b, int64_t HW, int64_t C, void* stream) {
  CNN_CHECK_C(C);
  DPN_CHECK_CUDA(launch_pdl(gap_fwd_kernel, (int)b, kT, 0, (cudaStream_t)stream, (const __nv_bfloat16*)x,
                            (__nv_bfloat16*)y, (int)HW, (int)C));
  return 0;
}

extern "C" int dpn_gap_bwd(const void* dy, void* dx, int64_t b, int64_t HW, int64_t C, void* stream) {
  CNN_CHECK_C(C);
  DPN_CHECK_CUDA(launch_pdl(gap_bwd_kernel, blocks_for(b * HW * (C / 8)), kT, 0, (cudaStream_t)stream,
                            (const __nv_bfloat16*)dy, (__nv_bfloat16*)dx, (long long)(b * HW), (int)HW,
                            (int)C));
  return 0;
}
