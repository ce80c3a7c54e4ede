// 2D stage kernel instantiations for N = 1..3, all M in 0..N, fp64 and fp32.
#include "instantiate2d.cuh"
namespace bbw {
KernelSet get_kernels2d_a(int N, int M, int dtype) {
  switch (N) {
    case 1: return MLoop2D<1, 1>::get(M, dtype);
    case 2: return MLoop2D<2, 2>::get(M, dtype);
    case 3: return MLoop2D<3, 3>::get(M, dtype);
    default: return KernelSet();
  }
}
}  // namespace bbw
