// tcgen05.mma issue-to-retire throughput per shape / operand major-ness (one
// CTA per SM, garbage smem operands, clock64 around R back-to-back MMAs).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2505_05856_b200/csrc mma_probe.cu -lcuda
#include "common.cuh"
#include <cstdio>
using namespace dpn;

template <int N, int AMN, int BMN>
__global__ void __launch_bounds__(128, 1) probe(long long* out, int reps) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<256>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = idesc_bf16(128, N, AMN, BMN);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint64_t ad = AMN ? smem_desc_sw128(a + k * 2048, 16384, 1024) : smem_desc_sw128(a + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
        const uint64_t bd = BMN ? smem_desc_sw128(b + k * 2048, 8192, 1024) : smem_desc_sw128(b + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
        umma_bf16(tmem, ad, bd, id, 1u);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_free<256>(tmem); }
}

template <int N, int AMN, int BMN>
void run(const char* name) {
  long long* d; cudaMalloc(&d, 148 * 8);
  const int smem = 140 * 1024;
  cudaFuncSetAttribute(probe<N, AMN, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 200;
  probe<N, AMN, BMN><<<148, 128, smem>>>(d, reps);
  probe<N, AMN, BMN><<<148, 128, smem>>>(d, reps);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double cyc = (double)h[0] / (reps * 8);
  printf("%-28s N=%3d  %6.1f cycles/instr  %6.0f flop/clk/SM  (%s)\n", name, N, cyc, 2.0 * 128 * N * 16 / cyc, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<256, 0, 0>("A K-major, B K-major");
  run<128, 0, 0>("A K-major, B K-major");
  run<64, 0, 0>("A K-major, B K-major");
  run<64, 0, 1>("A K-major, B MN-major");
  run<64, 1, 1>("A MN-major, B MN-major");
  run<128, 1, 1>("A MN-major, B MN-major");
  run<32, 0, 0>("A K-major, B K-major");
  return 0;
}
