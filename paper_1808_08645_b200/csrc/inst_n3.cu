// Kernel instantiations for N = 3, all M in 0..N, fp64 and fp32.
#include "instantiate.cuh"
BBW_INSTANTIATE(3)
