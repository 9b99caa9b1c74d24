// dfftb device code: FFT pass instantiations + launchers, the cross-GPU group
// barrier, the seeded-field generator and the finiteness check.
#include <algorithm>
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
void add_launches(int64_t n) { g_launches.fetch_add((uint64_t)n); }

// ---------------------------------------------------- pass dispatch (per precision TUs)

cudaError_t launch_pass_f64(int n, const PassParams& p, bool adj, cudaStream_t s);
cudaError_t launch_pass_f32(int n, const PassParams& p, bool adj, cudaStream_t s);
cudaError_t launch_pass_tma_f64(int n, const PassParams& p, bool adj, const TmaPlan& tp, int grid_limit,
                                cudaStream_t s);
cudaError_t launch_pass_tma_f32(int n, const PassParams& p, bool adj, const TmaPlan& tp, int grid_limit,
                                cudaStream_t s);
int tma_tile_w_f64(int n);
int tma_tile_w_f32(int n);

int tma_tile_w(int prec, int n) { return prec == 8 ? tma_tile_w_f64(n) : tma_tile_w_f32(n); }

int tma_tile_w_halfreal_f64(int n);
int tma_tile_w_halfreal_f32(int n);
int tma_tile_w_halfreal(int prec, int n) {
  return prec == 8 ? tma_tile_w_halfreal_f64(n) : tma_tile_w_halfreal_f32(n);
}


cudaError_t launch_pass_tma(int prec, int n, const PassParams& p, bool adj, const TmaPlan& tp, int grid_limit,
                            cudaStream_t s) {
  return prec == 8 ? launch_pass_tma_f64(n, p, adj, tp, grid_limit, s) : launch_pass_tma_f32(n, p, adj, tp, grid_limit, s);
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
  return prec == 8 ? launch_pass_f64(n, p, adj, s) : launch_pass_f32(n, p, adj, s);
}

// ------------------------------------------------------ cross-GPU sync points
//
// Every rank runs the same program, so sync point k of execute e is the same
// on all ranks.  Rank r's flag page holds one u64 per (sync point, world
// rank): flags[k * kMaxRanks + q] = the last execute epoch in which rank q
// reached sync point k with r.  The epoch lives on the device (sync_begin
// bumps it at the start of every multi-rank program), so programs are
// replayable (CUDA graphs) without host parameters.  A wait that exceeds the
// timeout (GPU global timer) raises the context's timeout flag instead of
// hanging the GPU.

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// program start: epoch += 1 and the C2R statistics cleared (one thread)
__global__ void sync_begin_kernel(unsigned long long* epoch, unsigned long long* herm) {
  if (threadIdx.x == 0) {
    *epoch += 1;
    if (herm) {
      herm[0] = 0;
      herm[1] = 0;
    }
  }
}

// thread i < nmem serves member i: signal (release store of the epoch into
// the member's flag page) and/or wait (acquire-spin on my flag for member i)
__global__ void sync_point_kernel(SyncParams sp) {
  const int i = threadIdx.x;
  if (i >= sp.nmem || sp.members[i] == sp.me) return;
  const unsigned long long e = *sp.epoch;
  if (sp.signal) {
    __threadfence_system();
    unsigned long long* dst = sp.peer_flags[i] + (size_t)sp.slot * kMaxRanksDev + sp.me;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dst), "l"(e) : "memory");
  }
  if (sp.wait) {
    const unsigned long long* src = sp.my_flags + (size_t)sp.slot * kMaxRanksDev + sp.members[i];
    if (ld_acquire_sys(src) >= e) return;
    if (ld_acquire_sys(sp.timeout_flag) != 0) return;  // this execute already failed
    const unsigned long long t0 = gtimer();
    while (ld_acquire_sys(src) < e) {
      if (gtimer() - t0 > sp.timeout_ns) {
        atomicExch(sp.timeout_flag, 1ull);
        break;
      }
      __nanosleep(64);
    }
  }
}

cudaError_t launch_sync_begin(unsigned long long* epoch, unsigned long long* herm, cudaStream_t s) {
  sync_begin_kernel<<<1, 32, 0, s>>>(epoch, herm);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_sync_point(const SyncParams& sp, cudaStream_t s) {
  sync_point_kernel<<<1, 64, 0, s>>>(sp);
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
