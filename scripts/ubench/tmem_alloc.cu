// Does tcgen05.alloc of C columns let 4 co-resident CTAs per SM run concurrently?
// Each CTA: alloc C columns (warp 0), spin ~200k cycles, dealloc.  Kernel time vs the no-alloc kernel.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int COLS, bool ALLOC>
__global__ void __launch_bounds__(128, 4) kern(unsigned long long* out) {
  __shared__ uint32_t slot;
  if (ALLOC && threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&slot)), "r"(COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  __syncthreads();
  unsigned long long t0 = clock64(), t;
  do { t = clock64(); } while (t - t0 < 200000);
  __syncthreads();
  if (ALLOC && threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(COLS) : "memory");
  if (threadIdx.x == 0) out[blockIdx.x] = t - t0;
}
template <int COLS, bool ALLOC>
void run(const char* name) {
  unsigned long long* d; cudaMalloc(&d, 148 * 4 * 8 * 8);
  cudaFuncSetAttribute(kern<COLS, ALLOC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024);
  kern<COLS, ALLOC><<<148 * 4, 128, 50 * 1024>>>(d); cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); kern<COLS, ALLOC><<<148 * 4, 128, 50 * 1024>>>(d); cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
  printf("%-28s %s  %.3f ms (one wave of 592 CTAs at 4/SM = ~0.1 ms if concurrent)\n", name, cudaGetErrorString(e), ms);
}
int main() {
  run<32, false>("no alloc");
  run<32, true>("alloc 32 cols");
  run<64, true>("alloc 64 cols");
  run<128, true>("alloc 128 cols");
  run<256, true>("alloc 256 cols");
  return 0;
}
