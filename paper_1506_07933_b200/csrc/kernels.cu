// dfftb device code: FFT pass instantiations + launchers, the cross-GPU group
// barrier, the seeded-field generator and the finiteness check.
#include <atomic>
#include <cstdio>

#include "fft_pass.cuh"
#include "fft_generic.cuh"
#include "fft_pass_tma.cuh"
#include "kernels.hpp"

namespace dfftb {

static std::atomic<uint64_t> g_launches{0};
uint64_t launch_count() { return g_launches.load(); }
void count_launch() { g_launches.fetch_add(1); }

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
  static constexpr int SMEM = W * lane_stride<Cpx<T>>(N) * (int)sizeof(Cpx<T>);
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
template <typename T, int N>
struct TmaCfg {
  // fp32 long lanes use 16 elements per thread (radix-16 stages): half the
  // threads per lane, so twice the adjacent lanes per CTA and 64-128 byte
  // TMA rows instead of 16-32 (fp64 tiles are bounded by shared memory)
  static constexpr int EPREF = (sizeof(T) == 4 && N >= 256) ? 16 : 8;
  using SC = Sched<N, EPREF>;
  static constexpr int TPL = SC::TPL;
  static constexpr int W0 = DFFTB_TMA_THREADS / TPL;
  static constexpr int W = W0 < 1 ? 1 : (W0 > 64 ? 64 : W0);
  static constexpr int THREADS = W * TPL;
  using TL = TmaLayout<T, N, W>;
  static constexpr int STAGES = (2 * TL::STG + TL::XCH + 128 <= (220 * 1024) / DFFTB_TMA_MINB) ? 2 : 1;
  static constexpr int SMEM = STAGES * TL::STG + TL::XCH + 8 * STAGES + 8 * kMaxDest;
};

template <typename T, int N, bool ADJ, int LK, bool SPEC = false>
static cudaError_t launch_tma_tn(const PassParams& p, const TmaPlan& tp, cudaStream_t s) {
  using Cf = TmaCfg<T, N>;
  auto kern = fft_pass_tma_kernel<T, N, Cf::EPREF, Cf::W, ADJ, Cf::STAGES, LK, SPEC>;
  static int grid_cap[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!grid_cap[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM);
    if (e != cudaSuccess) return e;
    int occ = 0, sms = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Cf::THREADS, Cf::SMEM);
    if (e != cudaSuccess) return e;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid_cap[dev] = (occ < 1 ? 1 : occ) * sms;
  }
  if (tp.args.ntiles <= 0) return cudaSuccess;
  const int64_t grid = tp.args.ntiles < grid_cap[dev] ? tp.args.ntiles : grid_cap[dev];
  kern<<<(unsigned)grid, Cf::THREADS, Cf::SMEM, s>>>(p, tp.tmap, tp.args);
  count_launch();
  return cudaGetLastError();
}

template <typename T>
static cudaError_t launch_tma_prec(int n, const PassParams& p, bool adj, const TmaPlan& tp,
                                   cudaStream_t s) {
  const int lk = p.in_mode == kInReal ? kR2C : (p.in_mode == kInHermitian ? kC2R : (p.inverse ? kC2CBwd : kC2CFwd));
#define DFFTB_TMA_CASE(NN)                                                \
  case NN:                                                                \
    if (adj) {                                                            \
      if (lk == kC2CFwd && p.spec.op) return launch_tma_tn<T, NN, true, kC2CFwd, true>(p, tp, s); \
      if (lk == kC2CFwd) return launch_tma_tn<T, NN, true, kC2CFwd>(p, tp, s);  \
      if (lk == kC2CBwd) return launch_tma_tn<T, NN, true, kC2CBwd>(p, tp, s);  \
      return cudaErrorInvalidValue;                                       \
    }                                                                     \
    switch (lk) {                                                         \
      case kC2CFwd: return launch_tma_tn<T, NN, false, kC2CFwd>(p, tp, s);     \
      case kC2CBwd: return launch_tma_tn<T, NN, false, kC2CBwd>(p, tp, s);     \
      case kR2C: return launch_tma_tn<T, NN, false, kR2C>(p, tp, s);           \
      default: return launch_tma_tn<T, NN, false, kC2R>(p, tp, s);             \
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

int tma_tile_w(int prec, int n) { return prec == 8 ? tma_w_prec<double>(n) : tma_w_prec<float>(n); }


// ----------------------------------------------- fused two-axis plane pipeline

template <typename T, int N, bool FWD>
static cudaError_t launch_fused2_tn(const PassParams& pa, const PassParams& pb, const CUtensorMap& tm,
                                    const Fused2Args& fa, cudaStream_t s) {
  using Cf = TmaCfg<T, N>;
  using TL = TmaLayout<T, N, Cf::W>;
  constexpr int SMEM = 2 * TL::STG + TL::XCH + 16 + 8 * kMaxDest;
  auto kern = fft_fused2_kernel<T, N, Cf::EPREF, Cf::W, FWD>;
  static int grid_cap[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!grid_cap[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    int occ = 0, sms = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Cf::THREADS, SMEM);
    if (e != cudaSuccess) return e;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid_cap[dev] = (occ < 1 ? 1 : occ) * sms;  // all CTAs co-resident (dependency waits)
  }
  const int64_t items = (int64_t)(fa.P + fa.lag) * 2 * fa.T;
  const int64_t grid = items < grid_cap[dev] ? items : grid_cap[dev];
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(Cf::THREADS);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  if (fa.persist_bytes > 0) {
    // the ring persists in L2; everything else streams through
    attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[0].val.accessPolicyWindow.base_ptr = fa.ring;
    attr[0].val.accessPolicyWindow.num_bytes = fa.persist_bytes;
    attr[0].val.accessPolicyWindow.hitRatio = 1.0f;
    attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, pa, pb, tm, fa);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <typename T>
static cudaError_t launch_fused2_prec(int n, bool fwd, const PassParams& pa, const PassParams& pb,
                                      const CUtensorMap& tm, const Fused2Args& fa, cudaStream_t s) {
  switch (n) {
    case 64: return fwd ? launch_fused2_tn<T, 64, true>(pa, pb, tm, fa, s) : launch_fused2_tn<T, 64, false>(pa, pb, tm, fa, s);
    case 128: return fwd ? launch_fused2_tn<T, 128, true>(pa, pb, tm, fa, s) : launch_fused2_tn<T, 128, false>(pa, pb, tm, fa, s);
    case 256: return fwd ? launch_fused2_tn<T, 256, true>(pa, pb, tm, fa, s) : launch_fused2_tn<T, 256, false>(pa, pb, tm, fa, s);
    case 512: return fwd ? launch_fused2_tn<T, 512, true>(pa, pb, tm, fa, s) : launch_fused2_tn<T, 512, false>(pa, pb, tm, fa, s);
  }
  return cudaErrorInvalidValue;
}

bool fused2_supported(int prec, int n) {
  return (n == 64 || n == 128 || n == 256 || n == 512) && tma_tile_w(prec, n) > 0;
}

cudaError_t launch_fused2(int prec, int n, bool fwd, const PassParams& pa, const PassParams& pb,
                          const CUtensorMap& tm, const Fused2Args& fa, cudaStream_t s) {
  return prec == 8 ? launch_fused2_prec<double>(n, fwd, pa, pb, tm, fa, s)
                   : launch_fused2_prec<float>(n, fwd, pa, pb, tm, fa, s);
}

// ------------------------------------------------ pipelined pass pairs

template <typename T, int N, bool ADJ_A, bool ADJ_B, int LK>
static cudaError_t launch_pipe_tn(const PassParams& pa, const TmaPlan& ta, const PipeArgs& ppa,
                                  const PassParams& pb, const TmaPlan& tb, const PipeArgs& ppb, double frac_a,
                                  cudaStream_t s) {
  using Cf = TmaCfg<T, N>;
  auto kern = fft_pipe_kernel<T, N, Cf::EPREF, Cf::W, ADJ_A, ADJ_B, Cf::STAGES, LK>;
  static int grid_cap[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!grid_cap[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM);
    if (e != cudaSuccess) return e;
    int occ = 0, sms = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Cf::THREADS, Cf::SMEM);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid_cap[dev] = occ * sms;  // every CTA co-resident: the consumer's waits always resolve
  }
  const int cap = grid_cap[dev];
  int na = (int)(frac_a * cap + 0.5);
  na = na < 1 ? 1 : (na > cap - 1 ? cap - 1 : na);
  kern<<<(unsigned)cap, Cf::THREADS, Cf::SMEM, s>>>(pa, ta.tmap, ta.args, ppa, pb, tb.tmap, tb.args, ppb, na);
  count_launch();
  return cudaGetLastError();
}

template <typename T, int N>
static cudaError_t launch_pipe_n(const PassParams& pa, bool adj_a, const TmaPlan& ta, const PipeArgs& ppa,
                                 const PassParams& pb, bool adj_b, const TmaPlan& tb, const PipeArgs& ppb,
                                 double frac_a, cudaStream_t s) {
  const bool bwd = pa.inverse != 0;
#define DFFTB_PIPE(AA, AB)                                                                            \
  if (adj_a == AA && adj_b == AB)                                                                     \
    return bwd ? launch_pipe_tn<T, N, AA, AB, kC2CBwd>(pa, ta, ppa, pb, tb, ppb, frac_a, s)           \
               : launch_pipe_tn<T, N, AA, AB, kC2CFwd>(pa, ta, ppa, pb, tb, ppb, frac_a, s);
  DFFTB_PIPE(false, true)
  DFFTB_PIPE(true, true)
  DFFTB_PIPE(true, false)
#undef DFFTB_PIPE
  return cudaErrorInvalidValue;
}

bool pipe_supported(int prec, int n) { return (prec == 8 || prec == 4) && (n == 256 || n == 512 || n == 1024); }

cudaError_t launch_pipe(int prec, int n, const PassParams& pa, bool adj_a, const TmaPlan& ta, const PipeArgs& ppa,
                        const PassParams& pb, bool adj_b, const TmaPlan& tb, const PipeArgs& ppb, double frac_a,
                        cudaStream_t s) {
#define DFFTB_PIPE_N(NN)                                                                              \
  case NN:                                                                                            \
    return prec == 8 ? launch_pipe_n<double, NN>(pa, adj_a, ta, ppa, pb, adj_b, tb, ppb, frac_a, s)   \
                     : launch_pipe_n<float, NN>(pa, adj_a, ta, ppa, pb, adj_b, tb, ppb, frac_a, s);
  switch (n) {
    DFFTB_PIPE_N(256)
    DFFTB_PIPE_N(512)
    DFFTB_PIPE_N(1024)
  }
#undef DFFTB_PIPE_N
  return cudaErrorInvalidValue;
}

cudaError_t launch_pass_tma(int prec, int n, const PassParams& p, bool adj, const TmaPlan& tp,
                            cudaStream_t s) {
  return prec == 8 ? launch_tma_prec<double>(n, p, adj, tp, s) : launch_tma_prec<float>(n, p, adj, tp, s);
}

// ------------------------------------------------------- generic lengths

cudaError_t launch_generic(int prec, const GenParams& g, cudaStream_t s) {
  const int64_t tiles = (int64_t)g.p.A * (g.p.A1 > 1 ? g.p.A1 : 1) * ((g.p.B + g.W - 1) / g.W);
  if (tiles <= 0) return cudaSuccess;
  const size_t csize = 2 * (size_t)prec;
  const int smem = (int)(2 * (size_t)g.W * g.L * csize);
  cudaError_t e;
  if (prec == 8) {
    e = cudaFuncSetAttribute(fft_generic_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    fft_generic_kernel<double><<<(unsigned)tiles, 256, smem, s>>>(g);
  } else {
    e = cudaFuncSetAttribute(fft_generic_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    fft_generic_kernel<float><<<(unsigned)tiles, 256, smem, s>>>(g);
  }
  count_launch();
  return cudaGetLastError();
}

bool pass_length_supported(int64_t n) {
  return n >= 1 && n <= 4096 && (n & (n - 1)) == 0;
}

cudaError_t launch_pass(int prec, int n, const PassParams& p, bool adj, cudaStream_t s) {
  return prec == 8 ? launch_prec<double>(n, p, adj, s) : launch_prec<float>(n, p, adj, s);
}

// ----------------------------------------------------------- group barrier

// Cross-GPU barrier over one grid-axis group.  Thread i signals member i
// (system-scope release store into the member's flag slot for this rank),
// then waits for member i's flag in the local slot array.  Flags are
// monotonically increasing epochs, so no reset is ever needed.  A timeout
// (GPU global timer) turns a dead peer into a reported Deadlock instead of a
// hung GPU.
__global__ void group_barrier_kernel(BarrierParams bp) {
  const int i = threadIdx.x;
  if (i < bp.nmem && bp.members[i] != bp.me) {
    __threadfence_system();
    unsigned long long* dst = bp.peer_flags[i] + bp.me;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dst), "l"(bp.epoch) : "memory");
  }
  if (i < bp.nmem && bp.members[i] != bp.me) {
    const unsigned long long* src = bp.my_flags + bp.members[i];
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(src) : "memory");
      if (v >= bp.epoch) break;
      unsigned long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      if (t1 - t0 > bp.timeout_ns) {
        atomicExch(bp.timeout_flag, 1ull);
        break;
      }
      __nanosleep(100);
    }
  }
  __syncthreads();
}

cudaError_t launch_barrier(const BarrierParams& bp, cudaStream_t s) {
  group_barrier_kernel<<<1, 32, 0, s>>>(bp);
  count_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------ seeded field

__device__ __forceinline__ double unit_from_hash(unsigned long long x) {
  // bench.cpp:22-28 (splitmix64 finalizer)
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return static_cast<double>(x >> 11) * 0x1.0p-52 - 1.0;
}

template <typename T>
__global__ void seeded_fill_kernel(SeedParams sp, T* out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < sp.count; l += stride) {
    int64_t rem = l, g = 0, mul = 1;
    for (int a = sp.nd - 1; a >= 0; --a) {
      const int64_t c = rem % sp.len[a];
      rem /= sp.len[a];
      g += (sp.off[a] + c) * mul;
      mul *= sp.gdims[a];
    }
    const unsigned long long base = sp.seed * 0x10001ULL + 2ULL * (unsigned long long)g;
    const double re = unit_from_hash(base);
    if (sp.out_complex) {
      const double im = sp.complex_field ? unit_from_hash(base + 1) : 0.0;
      out[2 * l] = static_cast<T>(re);
      out[2 * l + 1] = static_cast<T>(im);
    } else {
      out[l] = static_cast<T>(re);
    }
  }
}

cudaError_t launch_seeded(int prec, const SeedParams& sp, void* out, cudaStream_t s) {
  if (sp.count <= 0) return cudaSuccess;
  const int threads = 256;
  int64_t blocks = (sp.count + threads - 1) / threads;
  if (blocks > 148 * 64) blocks = 148 * 64;
  if (prec == 8) seeded_fill_kernel<double><<<(unsigned)blocks, threads, 0, s>>>(sp, (double*)out);
  else seeded_fill_kernel<float><<<(unsigned)blocks, threads, 0, s>>>(sp, (float*)out);
  count_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------- finiteness check

template <typename T>
__global__ void nonfinite_kernel(const T* x, int64_t n, unsigned long long* count) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    c += isfinite(x[i]) ? 0 : 1;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

// ------------------------------------------------------ spectral operators

// signed wavenumber of global index g on axis a (spectral.hpp:42-53)
__device__ __forceinline__ double wavenumber(const SpectralParams& sp, int a, int64_t g, bool deriv) {
  int64_t k = g;
  if (!sp.half[a] && 2 * g >= sp.n[a]) k = g - sp.n[a];
  const bool nyq = sp.n[a] % 2 == 0 && 2 * (k < 0 ? -k : k) == sp.n[a];
  return (deriv && nyq) ? 0.0 : sp.scale[a] * (double)k;
}

// One read + one write of the spectrum block; k computed per element from
// the global coordinate (no tables), multipliers in double as the reference.
template <typename T>
__global__ void spectral_kernel(SpectralParams sp, const Cpx<T>* in, Cpx<T>* out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < sp.count; l += stride) {
    int64_t rem = l, g[4];
    for (int a = sp.nd - 1; a >= 0; --a) {
      g[a] = sp.off[a] + rem % sp.len[a];
      rem /= sp.len[a];
    }
    const Cpx<T> v = in[l];
    double re, im;
    if (sp.op == 0) {  // i k_axis (.) v
      const double k = wavenumber(sp, sp.axis, g[sp.axis], true);
      re = -k * (double)v.y;
      im = k * (double)v.x;
    } else {
      double m = 0.0;
      for (int a = 0; a < sp.nd; ++a) {
        const double k = wavenumber(sp, a, g[a], false);
        m += k * k;
      }
      if (sp.op == 1) {
        re = -m * (double)v.x;
        im = -m * (double)v.y;
      } else if (m == 0.0) {
        re = im = 0.0;
      } else {
        re = (double)v.x / -m;
        im = (double)v.y / -m;
      }
    }
    Cpx<T> r{(T)re, (T)im};
    if (sp.accumulate) {
      const Cpx<T> o = out[l];
      r.x += o.x;
      r.y += o.y;
    }
    out[l] = r;
  }
}

cudaError_t launch_spectral(int prec, const SpectralParams& sp, const void* in, void* out, cudaStream_t s) {
  if (sp.count <= 0) return cudaSuccess;
  const int threads = 256;
  int64_t blocks = (sp.count + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (prec == 8)
    spectral_kernel<double><<<(unsigned)blocks, threads, 0, s>>>(sp, (const double2*)in, (double2*)out);
  else
    spectral_kernel<float><<<(unsigned)blocks, threads, 0, s>>>(sp, (const float2*)in, (float2*)out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_nonfinite(int prec, const void* x, int64_t n_reals, unsigned long long* count,
                             cudaStream_t s) {
  if (n_reals <= 0) return cudaSuccess;
  const int threads = 256;
  int64_t blocks = (n_reals + threads - 1) / threads;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (prec == 8) nonfinite_kernel<double><<<(unsigned)blocks, threads, 0, s>>>((const double*)x, n_reals, count);
  else nonfinite_kernel<float><<<(unsigned)blocks, threads, 0, s>>>((const float*)x, n_reals, count);
  count_launch();
  return cudaGetLastError();
}

}  // namespace dfftb
