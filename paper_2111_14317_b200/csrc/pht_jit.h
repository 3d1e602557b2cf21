// pht_jit.h — system-specialised kernels (include/pht.h pht_system_specialize), internal API.
//
// The generic kernels read every term's exponent vector from the term table and run a dense
// n-long FMA loop per term for stage 2 (phi, theta) and stage 4 (G_j += a_j w), although the
// benchmark systems have 1-3 nonzero exponents per term (nnz(A)/M = 5 for
// cyclic-10, 1.6 for katsura-10, 1.7 for noon-10).  Alg. 1 "Initialize" builds the
// system's matrices once; here that step also writes the system's rows as straight-line CUDA
// (exponents, liftings and coefficients as literals, only the nonzero exponents touched), which
// NVRTC compiles for sm_100a into the same kernels (pht_kernels.cuh, PHT_JIT geometry).
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "pht_kernels.cuh"

namespace pht {

struct JitKernels;

enum : unsigned { JIT_EVAL = 1u, JIT_STEP = 2u, JIT_TRACK = 4u, JIT_ALL = 7u };

// CUDA source of the specialised row function for the packed system (records of
// rec_stride(n) doubles: a_0..a_{n-1}, omega, log|c|, arg c; equation segments off[0..n]).
std::string jit_source(int n, const std::vector<double> &rec, const std::vector<int> &off);

// Compile src for sm_100a.  Returns 0 and fills cubin / lowered kernel names, or -1 with the
// NVRTC log in log.
int jit_compile(int n, const std::string &src, unsigned what, std::vector<char> &cubin,
                std::vector<std::string> &names, std::string &log);

// Load the cubin on the current device.  Returns nullptr (and the CUDA error in *err) on failure.
JitKernels *jit_load(int n, unsigned what, const std::vector<char> &cubin, const std::vector<std::string> &names,
                     cudaError_t *err);
void jit_free(JitKernels *J);
unsigned jit_what(const JitKernels *J);
// path slots of one full wave of the specialised tracker (SMs x resident CTAs x points per CTA)
int64_t jit_track_slots(const JitKernels *J, int sms);

cudaError_t jit_launch(const JitKernels *J, int mode, const DevSys &S, const Args &A, cudaStream_t stream);
cudaError_t jit_launch_track(const JitKernels *J, const DevSys &S, const TrackArgs &A, cudaStream_t stream, int sms);

} // namespace pht
