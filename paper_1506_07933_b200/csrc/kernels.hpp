// Host-visible launch interface of the dfftb device code (kernels.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "fft_generic.cuh"
#include "fft_pass.cuh"
#include "fft_pass_tma.cuh"
#include "fft_fused2.cuh"

namespace dfftb {

struct BarrierParams {
  unsigned long long* peer_flags[kMaxDest];  // member i's flag array (mapped)
  int members[kMaxDest];                     // world ranks of the group
  int nmem;
  int me;                                    // my world rank
  unsigned long long* my_flags;              // my flag array (indexed by world rank)
  unsigned long long epoch;
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
};
int tma_tile_w(int prec, int n);  // lanes per CTA of the TMA kernel
bool fused2_supported(int prec, int n);
cudaError_t launch_fused2(int prec, int n, bool fwd, const PassParams& pa, const PassParams& pb,
                          const CUtensorMap& tm, const Fused2Args& fa, cudaStream_t s);
bool pipe_supported(int prec, int n);
cudaError_t launch_pipe(int prec, int n, const PassParams& pa, bool adj_a, const TmaPlan& ta, const PipeArgs& ppa,
                        const PassParams& pb, bool adj_b, const TmaPlan& tb, const PipeArgs& ppb, double frac_a,
                        cudaStream_t s);
cudaError_t launch_pass_tma(int prec, int n, const PassParams& p, bool adj, const TmaPlan& tp,
                            cudaStream_t s);
cudaError_t launch_pass(int prec, int n, const PassParams& p, bool adj, cudaStream_t s);
cudaError_t launch_generic(int prec, const GenParams& g, cudaStream_t s);
cudaError_t launch_barrier(const BarrierParams& bp, cudaStream_t s);
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

}  // namespace dfftb
