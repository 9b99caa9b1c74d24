// Host-visible launch interface of the dfftb device code (kernels.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "fft_generic.cuh"
#include "fft_pass.cuh"
#include "fft_pass_tma.cuh"

namespace dfftb {

constexpr int kMaxRanksDev = 64;  // flag-page row length (world ranks)
constexpr int kSyncSlots = 64;    // sync points per program

struct SyncParams {
  unsigned long long* peer_flags[kMaxDest];  // member i's flag page (mapped)
  int members[kMaxDest];                     // world ranks of the group
  int nmem;
  int me;                                    // my world rank
  int slot;                                  // sync point index in the program
  int signal, wait;
  unsigned long long* my_flags;              // my flag page
  const unsigned long long* epoch;           // device epoch of this context
  unsigned long long timeout_ns;
  unsigned long long* timeout_flag;
};

struct SeedParams {
  int nd;
  int64_t len[4], off[4], gdims[4];
  int64_t count;
  unsigned long long seed;
  int complex_field;
  int out_complex;
};

bool pass_length_supported(int64_t n);

// TMA-prefetch variant (fft_pass_tma_kernel): host-side description
struct TmaPlan {
  CUtensorMap tmap;  // tensor-map mode (strided lanes)
  TmaArgs args;
  int pdl;           // launch with programmatic stream serialization
};
int tma_tile_w(int prec, int n);  // lanes per CTA of the TMA kernel
int tma_tile_w_halfreal(int prec, int n);  // ... of its half-length R2C / C2R variant (n/2-point)
cudaError_t launch_pass_tma(int prec, int n, const PassParams& p, bool adj, const TmaPlan& tp, int grid_limit,
                            cudaStream_t s);
cudaError_t launch_pass(int prec, int n, const PassParams& p, bool adj, cudaStream_t s);
cudaError_t launch_generic(int prec, const GenParams& g, cudaStream_t s);
cudaError_t launch_sync_begin(unsigned long long* epoch, unsigned long long* herm, cudaStream_t s);
cudaError_t launch_sync_point(const SyncParams& sp, cudaStream_t s);
cudaError_t launch_seeded(int prec, const SeedParams& sp, void* out, cudaStream_t s);
struct SpectralParams {
  int nd;
  int64_t len[4], off[4];  // local frequency block
  int64_t n[4];            // spatial lengths (full)
  int half[4];             // axis stored as a half spectrum (R2C last axis)
  double scale[4];         // 2 pi / L_a
  int op, axis, accumulate;
  int64_t count;
};
cudaError_t launch_spectral(int prec, const SpectralParams& sp, const void* in, void* out, cudaStream_t s);
cudaError_t launch_nonfinite(int prec, const void* x, int64_t n_reals, unsigned long long* count,
                             cudaStream_t s);
uint64_t launch_count();
// kernels a CUDA-graph replay launches are counted at replay, not at capture
void add_launches(int64_t n);

}  // namespace dfftb
