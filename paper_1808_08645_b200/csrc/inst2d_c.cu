// 2D stage kernel instantiations for N = 7..9, all M in 0..N, fp64 and fp32.
#include "instantiate2d.cuh"
namespace bbw {
KernelSet get_kernels2d_c(int N, int M, int dtype) {
  switch (N) {
    case 7: return MLoop2D<7, 7>::get(M, dtype);
    case 8: return MLoop2D<8, 8>::get(M, dtype);
    case 9: return MLoop2D<9, 9>::get(M, dtype);
    default: return KernelSet();
  }
}
}  // namespace bbw
