// Micro-benchmark: tcgen05.mma kind::f16 issue throughput, M = 128 vs M = 64 (N = 128,
// K = 16 per instruction), one CTA per SM, one issuing thread, operands in shared memory
// (contents irrelevant).  Prints clk per MMA instruction.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2602_04789_b200/csrc mma_m64.cu -o mma_m64 -lcuda
#include <cstdio>
#include "common.cuh"
using namespace lf;

template <int M>
__global__ void __launch_bounds__(128, 1) mma_loop(long long* out, int iters) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  unsigned char* sA = base;            // 128 x 64 bf16, SW128
  unsigned char* sB = base + 16384;    // 128 x 64 bf16
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&tslot, 256);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_bf16(M, 128, 0, 0);
    const uint64_t ad = smem_desc_sw128(smem_u32(sA), 16, 1024);
    const uint64_t bd = smem_desc_sw128(smem_u32(sB), 16, 1024);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int k = 0; k < 4; ++k) tc_mma_ss(tmem, ad + 2 * k, bd + 2 * k, idesc, (it | k) != 0);
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 256);
}

template <int M>
void run(int iters) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(mma_loop<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 33 * 1024);
  mma_loop<M><<<148, 128, 33 * 1024>>>(d, iters);
  mma_loop<M><<<148, 128, 33 * 1024>>>(d, iters);
  long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += (double)h[i];
  printf("M=%d N=128 K=16: %.1f clk per MMA (%s)\n", M, s / 148 / (iters * 4.0),
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<128>(4096);
  run<64>(4096);
  return 0;
}
