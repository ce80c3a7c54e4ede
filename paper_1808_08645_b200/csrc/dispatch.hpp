// Registry of the compiled (N, M, dtype) kernel instantiations.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace bbw {

struct KernelSet {
  // args points to StageArgs<double> or StageArgs<float>
  cudaError_t (*launch_stage)(const void* args, int grid, cudaStream_t s) = nullptr;
  // halo pack: p and u.n_sender per send-face node ([faces][2][Nfp]); geo = grad(lambda) [K][12]
  cudaError_t (*launch_pack)(const void* Q, const void* geo, const int* faces, int nfaces, const uint16_t* fnode,
                             void* buf, cudaStream_t s) = nullptr;
  cudaError_t (*prepare)() = nullptr;  // set smem attributes
  int (*blocks_per_sm)() = nullptr;
  int smem_bytes = 0, elems_per_cta = 0, threads = 0;
  // elastic stage kernel (NEXT-2); args points to ElasticArgs<double> / ElasticArgs<float>
  cudaError_t (*launch_elastic)(const void* args, int grid, cudaStream_t s) = nullptr;
  cudaError_t (*prepare_elastic)() = nullptr;
  int (*elastic_blocks_per_sm)() = nullptr;
  int elastic_smem_bytes = 0, elastic_elems_per_cta = 0, elastic_threads = 0;
};

KernelSet get_kernels(int N, int M, int dtype);
// 2D (triangle) stage kernels (launch_stage takes Stage2DArgs<R>); N = 1..3 / 4..6 / 7..9
KernelSet get_kernels2d_a(int N, int M, int dtype);
KernelSet get_kernels2d_b(int N, int M, int dtype);
KernelSet get_kernels2d_c(int N, int M, int dtype);

#define BBW_DECLARE_N(n) KernelSet get_kernels_N##n(int M, int dtype);
BBW_DECLARE_N(1)
BBW_DECLARE_N(2)
BBW_DECLARE_N(3)
BBW_DECLARE_N(4)
BBW_DECLARE_N(5)
BBW_DECLARE_N(6)
BBW_DECLARE_N(7)
BBW_DECLARE_N(8)
BBW_DECLARE_N(9)
#undef BBW_DECLARE_N

}  // namespace bbw
