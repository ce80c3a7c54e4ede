// Instantiation helper of the 2D stage kernel: included by inst2d_*.cu with the degrees they cover.
#pragma once
#include "dispatch.hpp"
#include "stage2d_kernel.cuh"

namespace bbw {

template <int N, int M, typename R>
struct Inst2D {
  using C = Stage2DCfg<N, M, R>;
  static cudaError_t prepare() {
    return cudaFuncSetAttribute(stage2d_kernel<C, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
  }
  static cudaError_t launch(const void* args, int grid, cudaStream_t s) {
    stage2d_kernel<C, R><<<grid, C::T, C::SMEM_BYTES, s>>>(*static_cast<const Stage2DArgs<R>*>(args));
    return cudaGetLastError();
  }
  static int blocks() {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, stage2d_kernel<C, R>, C::T, C::SMEM_BYTES) != cudaSuccess)
      return 1;
    return nb > 0 ? nb : 1;
  }
  static KernelSet get() {
    KernelSet k;
    k.launch_stage = &launch;
    k.prepare = &prepare;
    k.blocks_per_sm = &blocks;
    k.smem_bytes = C::SMEM_BYTES;
    k.elems_per_cta = C::G;
    k.threads = C::T;
    return k;
  }
};

template <int N, int M>
struct MLoop2D {
  static KernelSet get(int m, int dtype) {
    if (m == M) return dtype == 0 ? Inst2D<N, M, double>::get() : Inst2D<N, M, float>::get();
    return MLoop2D<N, M - 1>::get(m, dtype);
  }
};
template <int N>
struct MLoop2D<N, -1> {
  static KernelSet get(int, int) { return KernelSet(); }
};

}  // namespace bbw
