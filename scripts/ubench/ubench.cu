// Microbenchmarks: which B200 SM resources do LDS, SHFL, tcgen05.ld/st and DFMA share?
// Per-SM throughput in warp-instructions per SM-cycle; concurrent-resident blocks only.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 2048
#define UNR 16

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void __launch_bounds__(512) kern(unsigned long long* cyc, unsigned* sink, int salt) {
  __shared__ __align__(16) unsigned long long buf[4096];
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = i * 2654435761ull + salt;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t taddr = 0;
  if constexpr (MODE >= 20) {
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tslot)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    taddr = tslot + ((uint32_t)(32 * (warp & 3)) << 16);
  }
  __syncthreads();
  unsigned long long acc = lane;
  unsigned a32 = lane;
  double d0 = lane, d1 = lane + 1, d2 = lane + 2, d3 = lane + 3, d4 = 1, d5 = 2, d6 = 3, d7 = 4;
  const double m = 1.0000001;
  const unsigned base = smem_u32(buf) + 8 * lane;
  unsigned long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if constexpr (MODE == 0 || MODE == 3 || MODE == 5 || MODE == 21) {  // LDS.64
        unsigned long long v;
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(base + 256 * u + 4096 * (it & 1)) : "memory");
        acc ^= v;
      }
      if constexpr (MODE == 1) {  // LDS.128
        unsigned x0, x1, x2, x3;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3)
                     : "r"(smem_u32(buf) + 16 * lane + 512 * u + 8192 * (it & 1)) : "memory");
        a32 ^= x0 ^ x1 ^ x2 ^ x3;
      }
      if constexpr (MODE == 2 || MODE == 3) {  // 2x SHFL.IDX (one fp64 per lane)
        unsigned lo = (unsigned)acc + u, hi = (unsigned)(acc >> 32);
        lo = __shfl_sync(0xffffffffu, lo, (lane + 1) & 31);
        hi = __shfl_sync(0xffffffffu, hi, (lane + 1) & 31);
        acc += ((unsigned long long)hi << 32) | lo;
      }
      if constexpr (MODE == 4 || MODE == 5) {  // 4 independent DFMA chains x2
        d0 = fma(d0, m, d4); d1 = fma(d1, m, d5); d2 = fma(d2, m, d6); d3 = fma(d3, m, d7);
      }
      if constexpr (MODE == 6) {  // STS.64
        asm volatile("st.shared.u64 [%0], %1;" ::"r"(base + 256 * u + 4096 * (it & 1)), "l"(acc + u) : "memory");
      }
      if constexpr (MODE == 20 || MODE == 21) {  // tcgen05.ld 32x32b.x8 (8 columns x 32 lanes x 4 B = 1 KB/warp)
        unsigned r[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(taddr + 8 * u + 128 * (it & 1)) : "memory");
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        a32 ^= r[0] ^ r[1] ^ r[2] ^ r[3] ^ r[4] ^ r[5] ^ r[6] ^ r[7];
      }
      if constexpr (MODE == 22) {  // tcgen05.st 32x32b.x8
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr + 8 * (u & 7)),
                     "r"(a32), "r"(a32 + 1), "r"(a32 + 2), "r"(a32 + 3), "r"(a32 + 4), "r"(a32 + 5), "r"(a32 + 6),
                     "r"(a32 + u));
        a32 += 1;
      }
      if constexpr (MODE == 23) {  // tcgen05.ld x8, 4 in flight before one wait
        unsigned r[32];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                       "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                       "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                       "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                     : "r"(taddr + 32 * ((u + it) & 3)) : "memory");
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 32; ++i) a32 ^= r[i];
      }
    }
  }
  unsigned long long t1 = clock64();
  if constexpr (MODE >= 20) {
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tslot), "r"(512));
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = (unsigned)acc ^ (unsigned)(acc >> 32) ^ a32 ^ (unsigned)(d0 + d1 + d2 + d3);
}

template <int MODE>
void run(const char* name, int threads, int bps, double per_iter_instr) {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int grid = nsm * bps;
  unsigned long long* cyc;
  unsigned* sink;
  cudaMalloc(&cyc, grid * 8);
  cudaMalloc(&sink, grid * threads * 4);
  cudaFuncSetAttribute(kern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  kern<MODE><<<grid, threads, 160 * 1024>>>(cyc, sink, 1);
  cudaDeviceSynchronize();
  kern<MODE><<<grid, threads, 160 * 1024>>>(cyc, sink, 2);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
  unsigned long long* h = new unsigned long long[grid];
  cudaMemcpy(h, cyc, grid * 8, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < grid; ++i) s += h[i];
  s /= grid;
  const double warps_per_sm = bps * threads / 32.0;
  const double instr = warps_per_sm * ITERS * UNR * per_iter_instr;
  printf("%-40s warps/SM %5.0f  cycles %10.0f  warp-instr/SM-cycle %.3f\n", name, warps_per_sm, s, instr / s);
  delete[] h;
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  run<0>("LDS.64 (2 wf/instr ideal)", 512, 1, 1);
  run<1>("LDS.128 (4 wf/instr ideal)", 512, 1, 1);
  run<6>("STS.64", 512, 1, 1);
  run<2>("SHFL x2 (per fp64)", 512, 1, 2);
  run<3>("LDS.64 + 2 SHFL (count LDS)", 512, 1, 1);
  run<4>("DFMA", 512, 1, 4);
  run<5>("DFMA x4 + LDS.64 (count LDS)", 512, 1, 1);
  run<20>("tcgen05.ld x8 + wait", 512, 1, 1);
  run<21>("tcgen05.ld x8 + wait + LDS.64 (count LDS)", 512, 1, 1);
  run<22>("tcgen05.st x8", 512, 1, 1);
  run<23>("tcgen05.ld x32 + wait", 512, 1, 1);
  return 0;
}
