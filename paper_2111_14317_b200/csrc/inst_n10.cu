// Explicit instantiation of the launchers for n = 10 (one file per n: parallel build).
#include "pht_dense.cuh"
#include "pht_kernels.cuh"
#include "pht_evalw.cuh"
namespace pht {
template cudaError_t launch<10>(int, const DevSys &, const Args &, cudaStream_t, int);
template cudaError_t launch_track<10>(const DevSys &, const TrackArgs &, cudaStream_t, int, int);
template cudaError_t launch_dense<10>(int, const DevSys &, const DenseSys &, const Args &, cudaStream_t);
template cudaError_t launch_evalw<10, MODE_EVAL_X>(const DevSys &, const Args &, const EvalMaps &, cudaStream_t);
template cudaError_t launch_evalw<10, MODE_EVAL_Z>(const DevSys &, const Args &, const EvalMaps &, cudaStream_t);
}
