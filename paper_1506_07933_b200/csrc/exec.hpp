// dfftb executor entry points (exec.cu), used by the C ABI (capi.cpp).
#pragma once

#include <cuda_runtime.h>

#include "internal.hpp"

namespace dfftb {

size_t workspace_bytes(const Plan& plan, int rank);
Ctx* ctx_create(const Plan& plan, int rank, int device);
void ctx_export(const Ctx& ctx, CtxHandle* h);
void ctx_connect(Ctx& ctx, const CtxHandle* handles);
void ctx_destroy(Ctx* ctx);
void ctx_check(Ctx& ctx, cudaStream_t s);
void world_create(const Plan& plan, const int* devices, int ndev, Ctx** out);
int last_op_times(const Ctx& ctx, int* kinds, int* streams, int* lengths, double* shares, double* starts,
                  double* ms, int max);
void execute(const Plan& plan, Ctx& ctx, const void* d_in, void* d_out, cudaStream_t s, int flags,
             dfftb_timing* timers);
void execute_world(const Plan& plan, Ctx** ctxs, const void* const* d_in, void* const* d_out,
                   cudaStream_t s, int flags);
void spectral_apply(const Plan& plan, int rank, int op, int axis, const double* lengths, const void* in,
                    void* out, int accumulate, cudaStream_t s);
void execute_spectral(const Plan& plan, Ctx& ctx, const void* d_in, void* d_out, int op, int axis,
                      const double* lengths, int accumulate, cudaStream_t s, int flags);
void execute_world_spectral(const Plan& plan, Ctx** ctxs, const void* const* d_in, void* const* d_out, int op,
                            int axis, const double* lengths, int accumulate, cudaStream_t s, int flags);
void wavenumbers(const Plan& plan, int rank, int axis, int deriv, const double* lengths, double* k_out);
void fill_seeded(const Plan& plan, int rank, int side, uint64_t seed, int complex_field, void* d_buf,
                 cudaStream_t s);

}  // namespace dfftb
