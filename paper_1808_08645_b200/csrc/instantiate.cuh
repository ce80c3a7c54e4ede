// Instantiation helper: included by inst_nK.cu with BBW_N defined.
#pragma once
#include <type_traits>

#include "dispatch.hpp"
#include "elastic_kernel.cuh"
#include "stage_kernel.cuh"

namespace bbw {

template <int N, int M, typename R>
struct Inst {
  using C = StageCfg<N, M, R>;
  static cudaError_t prepare() {
    return cudaFuncSetAttribute(stage_kernel<C, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
  }
  static cudaError_t launch(const void* args, int grid, cudaStream_t s) {
    const StageArgs<R>& a = *static_cast<const StageArgs<R>*>(args);
    stage_kernel<C, R><<<grid, C::T, C::SMEM_BYTES, s>>>(a);
    return cudaGetLastError();
  }
  static cudaError_t pack(const void* Q, const void* geo, const int* faces, int nfaces, const uint16_t* fnode,
                          void* buf, cudaStream_t s) {
    if (nfaces <= 0) return cudaSuccess;
    long long total = (long long)nfaces * cnp2(N);
    int grid = (int)((total + 255) / 256);
    if (grid > 4 * 148) grid = 4 * 148;
    pack_kernel<N, R><<<grid, 256, 0, s>>>(static_cast<const R*>(Q), static_cast<const R*>(geo), faces, nfaces, fnode,
                                           static_cast<R*>(buf));
    return cudaGetLastError();
  }
  static int blocks() {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, stage_kernel<C, R>, C::T, C::SMEM_BYTES) != cudaSuccess)
      return 1;
    return nb > 0 ? nb : 1;
  }
  using EC = ElasticCfg<N, M, R>;
  static cudaError_t prepare_e() {
    return cudaFuncSetAttribute(elastic_stage_kernel<EC, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, EC::SMEM_BYTES);
  }
  static cudaError_t launch_e(const void* args, int grid, cudaStream_t s) {
    const ElasticArgs<R>& a = *static_cast<const ElasticArgs<R>*>(args);
    elastic_stage_kernel<EC, R><<<grid, EC::T, EC::SMEM_BYTES, s>>>(a);
    return cudaGetLastError();
  }
  static int blocks_e() {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, elastic_stage_kernel<EC, R>, EC::T, EC::SMEM_BYTES) != cudaSuccess)
      return 1;
    return nb > 0 ? nb : 1;
  }
  static KernelSet get() {
    KernelSet k;
    k.launch_elastic = &launch_e;
    k.prepare_elastic = &prepare_e;
    k.elastic_blocks_per_sm = &blocks_e;
    k.elastic_smem_bytes = EC::SMEM_BYTES;
    k.elastic_elems_per_cta = EC::G;
    k.elastic_threads = EC::T;
    k.launch_stage = &launch;
    k.launch_pack = &pack;
    k.prepare = &prepare;
    k.blocks_per_sm = &blocks;
    k.smem_bytes = C::SMEM_BYTES;
    k.elems_per_cta = C::G * C::ET;
    k.threads = C::T;
    return k;
  }
};

template <int N, int M>
KernelSet pick(int dtype) {
  return dtype == 0 ? Inst<N, M, double>::get() : Inst<N, M, float>::get();
}

template <int N, int M>
struct MLoop {
  static KernelSet get(int m, int dtype) { return m == M ? pick<N, M>(dtype) : MLoop<N, M - 1>::get(m, dtype); }
};
template <int N>
struct MLoop<N, -1> {
  static KernelSet get(int, int) { return KernelSet(); }
};

}  // namespace bbw

#ifdef BBW_ONLY_NM  // tuning builds: instantiate a single (N, M) = (BBW_ONLY_NM / 10, BBW_ONLY_NM % 10)
namespace bbw {
template <int n>
KernelSet only_nm(int M, int dtype) {
  if constexpr (n == BBW_ONLY_NM / 10) {
    if (M == BBW_ONLY_NM % 10) return pick<n, BBW_ONLY_NM % 10>(dtype);
  }
  return KernelSet();
}
}  // namespace bbw
#define BBW_INSTANTIATE(n) \
  namespace bbw {          \
  KernelSet get_kernels_N##n(int M, int dtype) { return only_nm<n>(M, dtype); } \
  }
#else
#define BBW_INSTANTIATE(n)                                                            \
  namespace bbw {                                                                     \
  KernelSet get_kernels_N##n(int M, int dtype) { return MLoop<n, n>::get(M, dtype); } \
  }
#endif
