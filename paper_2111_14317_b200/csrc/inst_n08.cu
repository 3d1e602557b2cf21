// Explicit instantiation of the launchers for n = 8 (one file per n: parallel build).
#include "pht_dense.cuh"
#include "pht_kernels.cuh"
#include "pht_evalw.cuh"
namespace pht {
template cudaError_t launch<8>(int, const DevSys &, const Args &, cudaStream_t, int);
template cudaError_t launch_track<8>(const DevSys &, const TrackArgs &, cudaStream_t, int, int);
template cudaError_t launch_dense<8>(int, const DevSys &, const DenseSys &, const Args &, cudaStream_t);
template cudaError_t launch_evalw<8, MODE_EVAL_X>(const DevSys &, const Args &, const EvalMaps &, cudaStream_t);
template cudaError_t launch_evalw<8, MODE_EVAL_Z>(const DevSys &, const Args &, const EvalMaps &, cudaStream_t);
}
