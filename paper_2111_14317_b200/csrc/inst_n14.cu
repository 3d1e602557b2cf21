// Explicit instantiation of the launchers for n = 14 (one file per n: parallel build).
#include "pht_dense.cuh"
#include "pht_kernels.cuh"
namespace pht {
template cudaError_t launch<14>(int, const DevSys &, const Args &, cudaStream_t, int);
template cudaError_t launch_track<14>(const DevSys &, const TrackArgs &, cudaStream_t, int, int);
template cudaError_t launch_dense<14>(int, const DevSys &, const DenseSys &, const Args &, cudaStream_t);
}
