// 2D stage kernel instantiations for N = 4..6, all M in 0..N, fp64 and fp32.
#include "instantiate2d.cuh"
namespace bbw {
KernelSet get_kernels2d_b(int N, int M, int dtype) {
  switch (N) {
    case 4: return MLoop2D<4, 4>::get(M, dtype);
    case 5: return MLoop2D<5, 5>::get(M, dtype);
    case 6: return MLoop2D<6, 6>::get(M, dtype);
    default: return KernelSet();
  }
}
}  // namespace bbw
