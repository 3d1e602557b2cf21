// Explicit instantiation of the k_pht launcher for n = 16 (one file per n: parallel build).
#include "pht_kernels.cuh"
namespace pht {
template cudaError_t launch<16>(int, const DevSys &, const Args &, cudaStream_t);
}
