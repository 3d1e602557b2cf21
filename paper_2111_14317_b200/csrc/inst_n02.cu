// Explicit instantiation of the k_pht launcher for n = 2 (one file per n: parallel build).
#include "pht_kernels.cuh"
namespace pht {
template cudaError_t launch<2>(int, const DevSys &, const Args &, cudaStream_t);
}
