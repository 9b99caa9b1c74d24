// Template launchers of the FFT pass kernels (direct, TMA, half-length real),
// instantiated once per precision in kernels_f64.cu / kernels_f32.cu so the
// two halves compile in parallel.
#pragma once

#include <algorithm>

#include "fft_pass.cuh"
#include "fft_pass_tma.cuh"
#include "kernels.hpp"

namespace dfftb {

void count_launch();

// -------------------------------------------------------- pass launchers

// Tile shape per (precision, length): E elements per thread (radix-E
// Stockham), TPL = N/E threads per lane, W lanes per CTA, <= 512 threads.
template <typename T, int N>
struct PassCfg {
  static constexpr int EPREF = (sizeof(T) == 4 && N >= 256) ? 16 : 8;
  using SC = Sched<N, EPREF>;
  static constexpr int TPL = SC::TPL;
#ifndef DFFTB_THREADS
#define DFFTB_THREADS 512
#endif
  static constexpr int W0 = DFFTB_THREADS / TPL;
  static constexpr int W = W0 < 1 ? 1 : (W0 > 64 ? 64 : W0);
  static constexpr int THREADS = W * TPL;
  static constexpr int SMEM = W * lane_stride<Cpx<T>>(N, W) * (int)sizeof(Cpx<T>);
};

template <typename T, int N, bool ADJ>
static cudaError_t launch_tn(const PassParams& p, cudaStream_t s) {
  using Cf = PassCfg<T, N>;
  auto kern = fft_pass_kernel<T, N, Cf::EPREF, Cf::W, ADJ>;
  static bool attr_done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM);
    if (e != cudaSuccess) return e;
    attr_done[dev] = true;
  }
  const int64_t tiles = (int64_t)p.A * (p.A1 > 1 ? p.A1 : 1) * ((p.B + Cf::W - 1) / Cf::W);
  if (tiles <= 0) return cudaSuccess;
  kern<<<(unsigned)tiles, Cf::THREADS, Cf::SMEM, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

template <typename T, int N>
static cudaError_t launch_t(const PassParams& p, bool adj, cudaStream_t s) {
  return adj ? launch_tn<T, N, true>(p, s) : launch_tn<T, N, false>(p, s);
}

template <typename T>
static cudaError_t launch_prec(int n, const PassParams& p, bool adj, cudaStream_t s) {
  switch (n) {
    case 1: return launch_t<T, 1>(p, adj, s);
    case 2: return launch_t<T, 2>(p, adj, s);
    case 4: return launch_t<T, 4>(p, adj, s);
    case 8: return launch_t<T, 8>(p, adj, s);
    case 16: return launch_t<T, 16>(p, adj, s);
    case 32: return launch_t<T, 32>(p, adj, s);
    case 64: return launch_t<T, 64>(p, adj, s);
    case 128: return launch_t<T, 128>(p, adj, s);
    case 256: return launch_t<T, 256>(p, adj, s);
    case 512: return launch_t<T, 512>(p, adj, s);
    case 1024: return launch_t<T, 1024>(p, adj, s);
    case 2048: return launch_t<T, 2048>(p, adj, s);
    case 4096: return launch_t<T, 4096>(p, adj, s);
  }
  return cudaErrorInvalidValue;
}

// TMA variant: one persistent CTA per SM, 512 threads, STAGES-deep prefetch
template <typename T, int N, int EXTRA = 0, bool HALFREAL = false, bool ADJ = false>
struct TmaCfg {
  // fp32 long lanes use 16 elements per thread (radix-16 stages): half the
  // threads per lane, so twice the adjacent lanes per CTA and 64-128 byte
  // TMA rows instead of 16-32 (fp64 tiles are bounded by shared memory).
  // Half-length real lanes (HALFREAL) switch from N >= 64 so that halving the
  // length doubles the lanes per tile in fp32 too.
  // Long fp64 lanes (N >= DFFTB_F64_E16) run radix-16 stages with 256-thread
  // CTAs: the same 4 lanes per tile, one shared-memory exchange fewer
  // (1024 = 16*16*4 instead of 8*8*8*2): the contiguous 1024-point pass
  // 6.85 -> 6.22 ms, the strided ones unchanged (D 46.1 -> 44.2 ms,
  // profiles/r2/ab_f64_radix16_s43.txt).  512 threads (8 lanes) would need
  // 264 KB of shared memory.
#ifndef DFFTB_F64_E16
#define DFFTB_F64_E16 1024
#endif
#ifndef DFFTB_F64_E16_THREADS
#define DFFTB_F64_E16_THREADS 256
#endif
  static constexpr bool E16 = sizeof(T) == 8 && DFFTB_F64_E16 > 0 && N >= DFFTB_F64_E16;
  static constexpr int EPREF = (E16 || (sizeof(T) == 4 && (N >= 256 || (HALFREAL && N >= 64)))) ? 16 : 8;
  using SC = Sched<N, EPREF>;
  static constexpr int TPL = SC::TPL;
#ifndef DFFTB_SMALL_W
#define DFFTB_SMALL_W 16  // lane cap of short (N <= 64) tiles: more, smaller CTAs (64^3: 32 -> 25 us)
#endif
  static constexpr int THR = E16 ? DFFTB_F64_E16_THREADS : DFFTB_TMA_THREADS;
  static constexpr int W0 = (N <= 64 && THR / TPL > DFFTB_SMALL_W) ? DFFTB_SMALL_W : THR / TPL;
  static constexpr int W = W0 < 1 ? 1 : (W0 > 64 ? 64 : W0);
  static constexpr int THREADS = W * TPL;
  static constexpr int MINB = DFFTB_TMA_MINB;
  using TL = TmaLayout<T, N, W, EXTRA, RowPad<T, ADJ, W>::value, pass_lane_stride<T, N, EPREF, W, ADJ>()>;
  static constexpr int STAGES = (2 * TL::STG + TL::XCH + 128 <= (220 * 1024) / MINB) ? 2 : 1;
  static constexpr int SMEM = STAGES * TL::STG + TL::XCH + 8 * STAGES + 8 * kMaxDest;
};

template <typename T, int N, bool ADJ, int LK, bool SPEC = false>
static cudaError_t launch_tma_tn(const PassParams& p, const TmaPlan& tp, int grid_limit, cudaStream_t s) {
  using Cf = TmaCfg<T, N, LK == kC2Rh ? kC2RhExtra : 0, LK == kR2Ch || LK == kC2Rh, ADJ>;
  auto kern = fft_pass_tma_kernel<T, N, Cf::EPREF, Cf::W, ADJ, Cf::STAGES, LK, SPEC, Cf::MINB>;
  static int occ_of[64] = {0}, sms_of[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!occ_of[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM);
    if (e != cudaSuccess) return e;
    int occ = 0, sms = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Cf::THREADS, Cf::SMEM);
    if (e != cudaSuccess) return e;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    sms_of[dev] = sms;
    occ_of[dev] = occ < 1 ? 1 : occ;
  }
  if (tp.args.ntiles <= 0) return cudaSuccess;
  // persistent: one wave of resident CTAs on all SMs, or on `grid_limit` SMs
  // when the caller splits the GPU between two concurrent passes
  const int sms = grid_limit > 0 && grid_limit < sms_of[dev] ? grid_limit : sms_of[dev];
  const int64_t cap = (int64_t)occ_of[dev] * sms;
  const int64_t grid = tp.args.ntiles < cap ? tp.args.ntiles : cap;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(Cf::THREADS);
  cfg.dynamicSmemBytes = Cf::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  if (tp.pdl) {
    // programmatic dependent launch (the kernel waits on griddepcontrol)
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p, tp.tmap, tp.args);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

// half-length R2C / C2R lanes (contiguous): an n/2-point kernel
template <typename T>
static cudaError_t launch_rhalf_prec(int n, const PassParams& p, const TmaPlan& tp, int gl, cudaStream_t s) {
  const bool r2c = p.in_mode == kInReal;
#define DFFTB_RH_CASE(NN)                                                                        \
  case NN:                                                                                       \
    return r2c ? launch_tma_tn<T, NN / 2, false, kR2Ch>(p, tp, gl, s)                            \
               : launch_tma_tn<T, NN / 2, false, kC2Rh>(p, tp, gl, s);
  switch (n) {
    DFFTB_RH_CASE(16)
    DFFTB_RH_CASE(32)
    DFFTB_RH_CASE(64)
    DFFTB_RH_CASE(128)
    DFFTB_RH_CASE(256)
    DFFTB_RH_CASE(512)
    DFFTB_RH_CASE(1024)
    DFFTB_RH_CASE(2048)
    DFFTB_RH_CASE(4096)
  }
#undef DFFTB_RH_CASE
  return cudaErrorInvalidValue;
}

template <typename T>
static cudaError_t launch_tma_prec(int n, const PassParams& p, bool adj, const TmaPlan& tp, int gl,
                                   cudaStream_t s) {
  if (tp.args.rhalf) return launch_rhalf_prec<T>(n, p, tp, gl, s);
  const int lk = p.in_mode == kInReal ? kR2C : (p.in_mode == kInHermitian ? kC2R : (p.inverse ? kC2CBwd : kC2CFwd));
#define DFFTB_TMA_CASE(NN)                                                \
  case NN:                                                                \
    if (adj) {                                                            \
      if (lk == kC2CFwd && p.spec.op) return launch_tma_tn<T, NN, true, kC2CFwd, true>(p, tp, gl, s); \
      if (lk == kC2CFwd) return launch_tma_tn<T, NN, true, kC2CFwd>(p, tp, gl, s);  \
      if (lk == kC2CBwd) return launch_tma_tn<T, NN, true, kC2CBwd>(p, tp, gl, s);  \
      return cudaErrorInvalidValue;                                       \
    }                                                                     \
    switch (lk) {                                                         \
      case kC2CFwd: return launch_tma_tn<T, NN, false, kC2CFwd>(p, tp, gl, s);     \
      case kC2CBwd: return launch_tma_tn<T, NN, false, kC2CBwd>(p, tp, gl, s);     \
      case kR2C: return launch_tma_tn<T, NN, false, kR2C>(p, tp, gl, s);           \
      default: return launch_tma_tn<T, NN, false, kC2R>(p, tp, gl, s);             \
    }
  switch (n) {
    DFFTB_TMA_CASE(8)
    DFFTB_TMA_CASE(16)
    DFFTB_TMA_CASE(32)
    DFFTB_TMA_CASE(64)
    DFFTB_TMA_CASE(128)
    DFFTB_TMA_CASE(256)
    DFFTB_TMA_CASE(512)
    DFFTB_TMA_CASE(1024)
    DFFTB_TMA_CASE(2048)
    DFFTB_TMA_CASE(4096)
  }
#undef DFFTB_TMA_CASE
  return cudaErrorInvalidValue;
}

template <typename T>
static int tma_w_halfreal_prec(int n) {
  switch (n) {
    case 8: return TmaCfg<T, 8, 0, true>::W;
    case 16: return TmaCfg<T, 16, 0, true>::W;
    case 32: return TmaCfg<T, 32, 0, true>::W;
    case 64: return TmaCfg<T, 64, 0, true>::W;
    case 128: return TmaCfg<T, 128, 0, true>::W;
    case 256: return TmaCfg<T, 256, 0, true>::W;
    case 512: return TmaCfg<T, 512, 0, true>::W;
    case 1024: return TmaCfg<T, 1024, 0, true>::W;
    case 2048: return TmaCfg<T, 2048, 0, true>::W;
  }
  return 0;
}

template <typename T>
static int tma_w_prec(int n) {
  switch (n) {
    case 8: return TmaCfg<T, 8>::W;
    case 16: return TmaCfg<T, 16>::W;
    case 32: return TmaCfg<T, 32>::W;
    case 64: return TmaCfg<T, 64>::W;
    case 128: return TmaCfg<T, 128>::W;
    case 256: return TmaCfg<T, 256>::W;
    case 512: return TmaCfg<T, 512>::W;
    case 1024: return TmaCfg<T, 1024>::W;
    case 2048: return TmaCfg<T, 2048>::W;
    case 4096: return TmaCfg<T, 4096>::W;
  }
  return 0;
}


}  // namespace dfftb
