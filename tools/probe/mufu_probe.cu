// MUFU.EX2 throughput on sm_100a: f32 vs packed bf16x2 / f16x2 (results per clock per SM).
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>

__global__ void ex2_f32(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ex2_bf16x2(float* out, int iters) {
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) {
    __nv_bfloat162 v = __floats2bfloat162_rn(-0.001f * (threadIdx.x + i), -0.002f * i);
    a[i] = *reinterpret_cast<uint32_t*>(&v);
  }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
  float s = 0;
  for (int i = 0; i < 8; ++i) s += __bfloat162float(reinterpret_cast<__nv_bfloat162*>(&a[i])->x);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ex2_f16x2(float* out, int iters) {
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) {
    __half2 v = __floats2half2_rn(-0.001f * (threadIdx.x + i), -0.002f * i);
    a[i] = *reinterpret_cast<uint32_t*>(&v);
  }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
  float s = 0;
  for (int i = 0; i < 8; ++i) s += __half2float(reinterpret_cast<__half2*>(&a[i])->x);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 4 * 1024 * sizeof(float));
  int sm_clk;
  cudaDeviceGetAttribute(&sm_clk, cudaDevAttrClockRate, 0);
  const int iters = 4096, blocks = 148 * 4, threads = 512;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int k = 0; k < 3; ++k) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (k == 0) ex2_f32<<<blocks, threads>>>(out, iters);
      if (k == 1) ex2_bf16x2<<<blocks, threads>>>(out, iters);
      if (k == 2) ex2_f16x2<<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double instr = (double)blocks * threads * iters * 8;  // per-thread MUFU instructions
      double results = instr * (k == 0 ? 1 : 2);
      if (rep)
        printf("%s: %.3f ms, %.1f Ginstr/s, %.1f Gresults/s, %.2f results/clk/SM at %d MHz\n",
               k == 0 ? "f32" : k == 1 ? "bf16x2" : "f16x2", ms, instr / ms / 1e6, results / ms / 1e6,
               results / (ms * 1e-3) / 148 / (sm_clk * 1e3), sm_clk / 1000);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
