// Kernel instantiations for N = 4, all M in 0..N, fp64 and fp32.
#include "instantiate.cuh"
BBW_INSTANTIATE(4)
