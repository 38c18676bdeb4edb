// gs_jit.hpp -- runtime-specialised K1/K2 kernels for coefficient matrices
// outside the compiled registry (any RS(n,k) / erasure pattern).
//
// The compiled registry (gs_special.cuh) covers the configs' schemes; every
// other codec starts on the runtime-coefficient PRMT kernel. On its first
// GPU launch such a codec requests a JIT build: a background thread emits
// the same k_apply_special template instantiated with the codec's matrix as
// a compile-time constant (NVRTC, sm_XXa cubin, cached on disk), and later
// launches use it. Nothing blocks on the compile; results are identical
// bytes either way (tests compare both).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "gs_kernels.cuh"

namespace gsb {

struct JitKernel;

// Eligible matrices (rows <= 8, used sources <= 24, cols <= 32).
bool jit_eligible(int n_out, int n_slots, const uint8_t* coef);
// Request (or find) the kernel for this matrix; never blocks. nullptr when
// JIT is disabled (GS_JIT=0 / gs_set_jit(0)), unavailable (no NVRTC or
// kernel headers) or the matrix is not eligible.
JitKernel* jit_request(int n_out, int n_slots, const uint8_t* coef);
// 0 = pending, 1 = ready, -1 = failed. wait != 0 blocks until not pending.
int jit_status(JitKernel* k, bool wait);
// Launch over `count` table pointers (k_apply_special<Spec, 488, 1, false>
// signature) if ready on the current device; returns cudaErrorNotReady
// when it is not (caller falls back to the generic kernel).
cudaError_t jit_launch(JitKernel* k, const void* const* ptrs, int count, const TileGeom& g, int sms,
                       cudaStream_t st);
// Blocks per SM of the loaded kernel on the current device (0 if not loaded).
int jit_occupancy(JitKernel* k);
void jit_set_enabled(bool on);
// Drop queued builds and wait for the one in flight (call before process
// exit: NVRTC must not be compiling while its statics are torn down).
void jit_quiesce();
const char* jit_last_log(JitKernel* k);

}  // namespace gsb
