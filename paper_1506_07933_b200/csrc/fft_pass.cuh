// Batched 1-D FFT "pass" kernel for sm_100a — the hot path of dfftb.
//
// One pass = the LocalFftStage of the reference (plan.hpp:394-457, radix-2
// at kernels.hpp:117-139) for every lane of the rank's block along one axis,
// FUSED with whatever layout change follows it:
//   * the global transpose (exchange.hpp:547-590: pack -> all_to_all ->
//     unpack, plus the LocalTransposeStage plan.hpp:494-509): every output
//     element is stored straight into its final home in the destination
//     rank's exchange buffer (peer memory over NVLink via CUDA IPC), so pack,
//     all-to-all, unpack and the local transpose cost no extra HBM pass;
//   * the NormalizeStage (plan.hpp:510-525): folded into the store scale.
//
// Algorithm: self-sorting Stockham, radix-E register butterflies (E = 8/16),
// one lane = N/E threads, W lanes per CTA.  Stage 0 loads straight from HBM
// into registers, the last stage stores straight from registers to HBM/peer
// memory; the S-1 intermediate exchanges go through padded shared memory.
// Backward transforms use conj(FFT(conj(x))) so one forward butterfly set
// serves both directions.  Twiddles come from a per-length table computed in
// double on the host (as TwiddleTable, kernels.hpp:66-98) and read via the
// read-only path.
//
// Lane addressing (3-D blocks; the FFT axis v is always the transpose's
// scatter axis): lanes are indexed by the two non-FFT axes (alpha, beta) in
// memory order, so both the source and every destination address are affine:
//    src  = in + alpha*in_sa + beta*in_sb + i*in_si
//    dst  = dest[q].ptr + base_q + alpha*sa_q + beta*sb_q + kk*sk_q,
//           q = k / oblk, kk = k - q*oblk     (ceil-block owner, layout.hpp:80-98)
// A CTA owns W consecutive beta values of one alpha.  When the FFT axis is
// the innermost one (in_si == 1) threads run along the lane (j fastest),
// otherwise across lanes (w fastest) so every warp access covers whole
// 128-byte lines of W adjacent lanes.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

// Build-time tuning knobs (defaults are the shipped configuration)
#ifndef DFFTB_TW_REC
#define DFFTB_TW_REC 1      // 1: twiddle powers by products instead of table reads
#endif
#ifndef DFFTB_TMA_THREADS
#define DFFTB_TMA_THREADS 512  // threads per CTA of the TMA pass kernel
#endif
#ifndef DFFTB_TWB
#define DFFTB_TWB 1  // twiddle bases kept in registers across tiles
#endif
#ifndef DFFTB_LS_FP32
#define DFFTB_LS_FP32 1  // the bank-aware lane-stride residue for fp32 narrow tiles too (E's
                         // 2048-point passes: 104 M bank conflicts -> 0.1 M, 0.82 -> 0.73 ms)
#endif
#ifndef DFFTB_TMA_MINB
#define DFFTB_TMA_MINB 1    // resident CTAs per SM the TMA kernel is compiled for
#endif

namespace dfftb {

template <typename T> struct CpxOf;
template <> struct CpxOf<double> { using type = double2; };
template <> struct CpxOf<float> { using type = float2; };
template <typename T> using Cpx = typename CpxOf<T>::type;

template <typename C> __device__ __forceinline__ C cadd(C a, C b) { return C{a.x + b.x, a.y + b.y}; }
template <typename C> __device__ __forceinline__ C csub(C a, C b) { return C{a.x - b.x, a.y - b.y}; }
template <typename C> __device__ __forceinline__ C cmul(C a, C b) {
  return C{a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
// a * (-i)
template <typename C> __device__ __forceinline__ C mul_mi(C a) { return C{a.y, -a.x}; }
template <typename C> __device__ __forceinline__ C cconj(C a) { return C{a.x, -a.y}; }

constexpr int kMaxDest = 8;

struct Dest {
  void* ptr;
  int64_t base, sa, sb, sk;
  int64_t sa1;  // 4-D tensors: stride of the outermost lane axis
};

enum InMode : int { kInComplex = 0, kInReal = 1, kInHermitian = 2 };

// Spectral multiplier applied in the store epilogue of the last forward pass
// (the i k / -|k|^2 factors of spectral.hpp:133-309
// fused into the FFT instead of a separate pass over the spectrum).  Roles:
// 0 the transformed axis (index k), 1 the alpha lane axis, 2 beta, 3 the 4-D
// outer lane axis.
struct SpecEpi {
  int op;          // 0 none, 1 derivative, 2 laplacian, 3 inverse laplacian
  int accumulate;  // out += multiplier * x (divergence)
  int deriv_role;  // derivative: the role carrying the derivative axis
  int nroles;
  int64_t off[4];  // global offset of each role's local index (role 0: 0)
  int64_t n[4];    // spatial length of each role's axis
  int half[4];     // role stored as a half spectrum (R2C axis)
  double scale[4]; // 2 pi / L
  int order[4];    // roles in tensor-axis order (|k|^2 summed as spectral_kernel does)
  unsigned long long* dc;  // [2]: raw DC bin (zero-mean check), doubles as bits
};

struct PassParams {
  const void* in;
  int64_t in_sa, in_sb, in_si;  // strides in elements of the input type
  int A, B;                     // lane extents (alpha outer, beta inner)
  int A1;                       // 4-D: extent of a second, outermost lane axis (<= 1: none)
  int64_t in_sa1;               // ... and its input stride
  int in_mode;                  // InMode
  int out_real;                 // store Re() only (C2R)
  int inverse;                  // conj on load and store
  int n_out;                    // stored positions: n, or n/2+1 for R2C
  int ndest;
  int64_t oblk;                 // ceil-block size of the scattered axis
  int store_mode;               // 0 one dest, 1 equal pow-2 blocks, 2 general
  int oshift, omask;            // store_mode 1: q = k >> oshift, kk = k & omask
  double scale;
  const void* tw;               // N complex twiddles exp(-2 pi i m / N)
  const void* tw2;              // half-length real lanes: the n-point table (tw: the n/2-point one)
  unsigned long long* herm;     // C2R: [0] max |X| bits, [1] max |Im DC/Nyq| bits
  SpecEpi spec;                 // spectral epilogue (spec.op == 0: none)
  Dest dest[kMaxDest];
};

// signed wavenumber (spectral.hpp:42-53), as wavenumber() in kernels.cu
__device__ __forceinline__ double spec_k(const SpecEpi& e, int role, int64_t g, bool deriv) {
  int64_t k = g;
  if (!e.half[role] && 2 * g >= e.n[role]) k = g - e.n[role];
  const bool nyq = e.n[role] % 2 == 0 && 2 * (k < 0 ? -k : k) == e.n[role];
  return (deriv && nyq) ? 0.0 : e.scale[role] * (double)k;
}

// Store of one finished output element with the spectral multiplier
// (double arithmetic on the T-rounded FFT value, as the separate
// spectral_kernel: fused and unfused results are bit-identical).
template <typename T>
__device__ __forceinline__ void spec_store(const PassParams& p, void* base, int64_t off, Cpx<T> x, int k,
                                           int alpha, int beta) {
  const SpecEpi& e = p.spec;
  int64_t g[4];
  g[0] = k;
  int a2 = alpha, a1 = 0;
  if (p.A1 > 1) {
    a1 = alpha / p.A;
    a2 = alpha - a1 * p.A;
  }
  g[1] = e.off[1] + a2;
  g[2] = e.off[2] + beta;
  g[3] = e.off[3] + a1;
  if (e.dc && g[0] == 0 && g[1] == 0 && g[2] == 0 && (e.nroles < 4 || g[3] == 0)) {
    e.dc[0] = static_cast<unsigned long long>(__double_as_longlong((double)x.x));
    e.dc[1] = static_cast<unsigned long long>(__double_as_longlong((double)x.y));
  }
  double re, im;
  if (e.op == 1) {
    const double kk = spec_k(e, e.deriv_role, g[e.deriv_role], true);
    re = -kk * (double)x.y;
    im = kk * (double)x.x;
  } else {
    double m = 0.0;
    for (int i = 0; i < e.nroles; ++i) {
      const int r = e.order[i];
      const double kk = spec_k(e, r, g[r], false);
      m += kk * kk;
    }
    if (e.op == 2) {
      re = -m * (double)x.x;
      im = -m * (double)x.y;
    } else if (m == 0.0) {
      re = im = 0.0;
    } else {
      re = (double)x.x / -m;
      im = (double)x.y / -m;
    }
  }
  Cpx<T> r{(T)re, (T)im};
  Cpx<T>* out = reinterpret_cast<Cpx<T>*>(base) + off;
  if (e.accumulate) {
    const Cpx<T> o = *out;
    r.x += o.x;
    r.y += o.y;
  }
  *out = r;
}

// combined outer lane index alpha = a1 * A + a2 (a1 only for 4-D tensors)
__device__ __forceinline__ int64_t in_alpha_off(const PassParams& p, int alpha) {
  if (p.A1 <= 1) return (int64_t)alpha * p.in_sa;
  const int a1 = alpha / p.A;
  return (int64_t)a1 * p.in_sa1 + (int64_t)(alpha - a1 * p.A) * p.in_sa;
}
__device__ __forceinline__ int64_t dst_alpha_off(const PassParams& p, const Dest& d, int alpha) {
  if (p.A1 <= 1) return (int64_t)alpha * d.sa;
  const int a1 = alpha / p.A;
  return (int64_t)a1 * d.sa1 + (int64_t)(alpha - a1 * p.A) * d.sa;
}

// ------------------------------------------------------------ butterflies
template <typename C, typename T>
__device__ __forceinline__ void dft2(C& a, C& b) {
  C t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <typename C, typename T>
__device__ __forceinline__ void dft4(C& x0, C& x1, C& x2, C& x3) {
  C a = cadd(x0, x2), b = csub(x0, x2), c = cadd(x1, x3), d = mul_mi(csub(x1, x3));
  x0 = cadd(a, c);
  x2 = csub(a, c);
  x1 = cadd(b, d);
  x3 = csub(b, d);
}

template <typename C, typename T>
__device__ __forceinline__ void dft8(C* x) {
  // even/odd split: E = DFT4(x0,x2,x4,x6), O = DFT4(x1,x3,x5,x7)
  C e0 = x[0], e1 = x[2], e2 = x[4], e3 = x[6];
  C o0 = x[1], o1 = x[3], o2 = x[5], o3 = x[7];
  dft4<C, T>(e0, e1, e2, e3);
  dft4<C, T>(o0, o1, o2, o3);
  const T h = T(0.70710678118654752440084436210484904);
  // W8^1 = (1 - i)/sqrt2, W8^2 = -i, W8^3 = (-1 - i)/sqrt2
  C t1 = C{(o1.x + o1.y) * h, (o1.y - o1.x) * h};
  C t2 = mul_mi(o2);
  C t3 = C{(o3.y - o3.x) * h, -(o3.x + o3.y) * h};
  x[0] = cadd(e0, o0);
  x[4] = csub(e0, o0);
  x[1] = cadd(e1, t1);
  x[5] = csub(e1, t1);
  x[2] = cadd(e2, t2);
  x[6] = csub(e2, t2);
  x[3] = cadd(e3, t3);
  x[7] = csub(e3, t3);
}

template <typename C, typename T>
__device__ __forceinline__ void dft16(C* x) {
  C e[8], o[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    e[i] = x[2 * i];
    o[i] = x[2 * i + 1];
  }
  dft8<C, T>(e);
  dft8<C, T>(o);
  // W16^k = cos(pi k / 8) - i sin(pi k / 8)
  const T c1 = T(0.92387953251128675612818318939678829);
  const T s1 = T(0.38268343236508977172845998403039887);
  const T h = T(0.70710678118654752440084436210484904);
  const C w[8] = {C{T(1), T(0)}, C{c1, -s1}, C{h, -h}, C{s1, -c1},
                  C{T(0), T(-1)}, C{-s1, -c1}, C{-h, -h}, C{-c1, -s1}};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    C t = k == 0 ? o[0] : cmul(o[k], w[k]);
    x[k] = cadd(e[k], t);
    x[k + 8] = csub(e[k], t);
  }
}

template <int R, typename C, typename T>
__device__ __forceinline__ void dft_r(C* x) {
  if constexpr (R == 2) {
    dft2<C, T>(x[0], x[1]);
  } else if constexpr (R == 4) {
    dft4<C, T>(x[0], x[1], x[2], x[3]);
  } else if constexpr (R == 8) {
    dft8<C, T>(x);
  } else if constexpr (R == 16) {
    dft16<C, T>(x);
  }
}

// ------------------------------------------------------------- schedule
__host__ __device__ constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n / 2); }

template <int N, int EPREF>
struct Sched {
  static constexpr int E = N < EPREF ? N : EPREF;  // elements per thread
  static constexpr int TPL = N / E;                 // threads per lane
  static constexpr int L = ilog2(N);
  static constexpr int LE = ilog2(E);
  static constexpr int Q = LE == 0 ? 0 : L / LE;
  static constexpr int REM = LE == 0 ? 0 : L % LE;
  static constexpr int S = Q + (REM ? 1 : 0);       // stages
  __host__ __device__ static constexpr int radix(int s) { return s < Q ? E : (1 << REM); }
  __host__ __device__ static constexpr int ns(int s) { return s == 0 ? 1 : ns(s - 1) * radix(s - 1); }
};

// shared-memory padding: one slot every 128 bytes keeps the stride-R Stockham
// writes and the cross-lane (w-fastest) accesses bank-conflict free
template <typename C>
__device__ __forceinline__ int spad(int i) {
  constexpr int LOG_SLOTS = sizeof(C) == 16 ? 3 : 4;
  return i + (i >> LOG_SLOTS);
}
template <typename C>
__host__ __device__ constexpr int lane_stride(int n, int w = 64) {
  // Padded lane length in slots.  In the w-fastest thread layout (strided
  // lanes) one 16-byte shared-memory wavefront (128 bytes: m = 8 slots)
  // serves W lanes x m/W positions; for W < m, lane offsets m/W apart modulo m
  // keep those accesses on distinct banks (1024-point fp64 strided passes:
  // 8.9 -> 7.5 ms; 2048-point fp32 ones 0.82 -> 0.73 ms).  Odd offsets
  // otherwise.
  constexpr int m = 128 / (int)sizeof(C);
  const int base = n + (n >> (sizeof(C) == 16 ? 3 : 4));
  if ((sizeof(C) != 16 && !DFFTB_LS_FP32) || w >= m) return base | 1;
  const int r = m / w;
  return base + ((r - base % m) % m + m) % m;
}

// Lanes as rows (contiguous lanes, lane-major threads): a warp spans 32/TPL
// lanes of TPL threads; when a lane's TPL slots fill less than a wavefront
// (m slots), a stride of TPL modulo m puts the lanes of a warp side by side
// in the exchange buffer instead of on the same banks (half-length
// 128-point fp32 lanes, 8 threads per lane: R2C pass 0.553 -> 0.488 ms, C2R
// 0.531 -> 0.506 ms; profiles/r2/ab_lanestride_rows_s51.txt).
#ifndef DFFTB_LS_ROWS
#define DFFTB_LS_ROWS 1
#endif
template <typename C>
__host__ __device__ constexpr int lane_stride_rows(int n, int tpl) {
  constexpr int m = 128 / (int)sizeof(C);
  const int base = n + (n >> (sizeof(C) == 16 ? 3 : 4));
  if (!DFFTB_LS_ROWS || tpl >= m || (m % tpl) != 0) return base | 1;
  return base + ((tpl - base % m) % m + m) % m;
}

// lane stride of the exchange buffer of a TMA pass kernel
template <typename T, int N, int EPREF, int W, bool ADJ>
__host__ __device__ constexpr int pass_lane_stride() {
  using C = Cpx<T>;
  if constexpr (ADJ) {
    return lane_stride<C>(N, W);
  } else {
    return lane_stride_rows<C>(N, Sched<N, EPREF>::TPL);
  }
}

template <typename T>
__device__ __forceinline__ unsigned long long dbits(T v) {
  return static_cast<unsigned long long>(__double_as_longlong(static_cast<double>(v)));
}

// This thread's twiddle bases, one per (stage >= 1, butterfly).  They depend
// on the thread's position j only, not on the tile, so persistent kernels load
// them once and keep them in registers (no table read on the tile path).
template <typename T, int N, int EPREF>
struct TwBase {
  using SC = Sched<N, EPREF>;
  __host__ __device__ static constexpr int off(int s) { return s <= 1 ? 0 : off(s - 1) + SC::E / SC::radix(s - 1); }
  static constexpr int COUNT = SC::S <= 1 ? 1 : off(SC::S);
  Cpx<T> w[COUNT];
};

template <typename T, int N, int EPREF, int s = 1>
__device__ __forceinline__ void load_twbase(TwBase<T, N, EPREF>& b, const Cpx<T>* tw, int j) {
  using SC = Sched<N, EPREF>;
  if constexpr (s < SC::S) {
    constexpr int R = SC::radix(s);
    constexpr int NS = SC::ns(s);
    constexpr int NB = SC::E / R;
#pragma unroll
    for (int t = 0; t < NB; ++t) {
      const int bidx = j + t * SC::TPL;
      const int pp = bidx & (NS - 1);
      b.w[TwBase<T, N, EPREF>::off(s) + t] = __ldg(tw + pp * (N / (NS * R)));
    }
    load_twbase<T, N, EPREF, s + 1>(b, tw, j);
  }
}

// Stage s of the self-sorting Stockham schedule (compile-time recursion so
// every register index is static).  On entry v holds this thread's inputs of
// stage s: slot t*R+r = position (j + t*TPL) + r*N/R.  twb: preloaded
// twiddle bases (nullptr: read the table).
template <typename T, int N, int EPREF, int s>
__device__ __forceinline__ void run_stages(Cpx<T>* v, Cpx<T>* lane, const Cpx<T>* tw, int j,
                                           const TwBase<T, N, EPREF>* twb = nullptr) {
  using C = Cpx<T>;
  using SC = Sched<N, EPREF>;
  if constexpr (s < SC::S) {
    constexpr int E = SC::E;
    constexpr int TPL = SC::TPL;
    constexpr int R = SC::radix(s);
    constexpr int NS = SC::ns(s);
    constexpr int NB = E / R;
    if constexpr (s > 0) {
#pragma unroll
      for (int t = 0; t < NB; ++t) {
        const int bidx = j + t * TPL;
        const int pp = bidx & (NS - 1);
        const int step = pp * (N / (NS * R));
#if DFFTB_TW_REC
        // one table read per butterfly, the other powers by products
        // (depth <= 3 multiplications: a few ulp, far inside 1e-12)
        C wp[R];
        wp[1] = twb ? twb->w[TwBase<T, N, EPREF>::off(s) + t] : __ldg(tw + step);
#pragma unroll
        for (int r = 2; r < R; ++r) wp[r] = cmul(wp[r / 2], wp[r - r / 2]);
#pragma unroll
        for (int r = 1; r < R; ++r) v[t * R + r] = cmul(v[t * R + r], wp[r]);
#else
#pragma unroll
        for (int r = 1; r < R; ++r) v[t * R + r] = cmul(v[t * R + r], __ldg(tw + r * step));
#endif
      }
    }
#pragma unroll
    for (int t = 0; t < NB; ++t) dft_r<R, C, T>(v + t * R);
    if constexpr (s < SC::S - 1) {
      if constexpr (s > 0) __syncthreads();  // previous exchange fully read
#pragma unroll
      for (int t = 0; t < NB; ++t) {
        const int bidx = j + t * TPL;
        const int pp = bidx & (NS - 1);
        const int idxd = (bidx - pp) * R + pp;
#pragma unroll
        for (int r = 0; r < R; ++r) lane[spad<C>(idxd + r * NS)] = v[t * R + r];
      }
      __syncthreads();
      constexpr int R2 = SC::radix(s + 1);
      constexpr int NB2 = E / R2;
#pragma unroll
      for (int t = 0; t < NB2; ++t) {
#pragma unroll
        for (int r = 0; r < R2; ++r) v[t * R2 + r] = lane[spad<C>(j + t * TPL + r * (N / R2))];
      }
      run_stages<T, N, EPREF, s + 1>(v, lane, tw, j, twb);
    }
  }
}


// ----------------------------------------------------- stage-0 fetch/store

// Fill v[] with this thread's stage-0 inputs.  ldc(pos)/ldr(pos) return the
// complex / real element `pos` of the lane.  Applies the lane semantics:
// real promotion (R2C, plan.hpp:428-430), Hermitian extension with DC/Nyquist
// imaginary parts dropped (irfft_1d, kernels.hpp:378-384) and conj for
// backward transforms.  Accumulates the C2R check statistics.
template <typename T, int N, int EPREF, class LDC, class LDR>
__device__ __forceinline__ void fetch0(Cpx<T>* v, int j, bool active, int in_mode, int inverse,
                                       LDC ldc, LDR ldr, double& local_max, double& local_imag) {
  using C = Cpx<T>;
  using SC = Sched<N, EPREF>;
  constexpr int E = SC::E;
  constexpr int TPL = SC::TPL;
  constexpr int R0 = SC::S > 0 ? SC::radix(0) : 1;
  constexpr int NB0 = E / R0;
#pragma unroll
  for (int t = 0; t < NB0; ++t) {
#pragma unroll
    for (int r = 0; r < R0; ++r) {
      const int pos = j + t * TPL + r * (N / R0);
      C x = C{T(0), T(0)};
      if (active) {
        if (in_mode == kInComplex) {
          x = ldc(pos);
        } else if (in_mode == kInReal) {
          x.x = ldr(pos);
        } else {
          const int src = pos <= N / 2 ? pos : N - pos;
          x = ldc(src);
          if (pos <= N / 2) {
            const double m = hypot((double)x.x, (double)x.y);
            local_max = m > local_max ? m : local_max;
          }
          if (pos == 0 || pos == N / 2) {
            const double im = fabs((double)x.y);
            local_imag = im > local_imag ? im : local_imag;
            x.y = T(0);
          }
          if (pos > N / 2) x.y = -x.y;
        }
      }
      if (inverse) x.y = -x.y;
      v[t * R0 + r] = x;
    }
  }
}

// block max-abs and DC/Nyquist imaginary residue (irfft_1d checks,
// kernels.hpp:369-377, with the block scale of plan.hpp:440-446)
__device__ __forceinline__ void herm_reduce(unsigned long long* herm, double local_max, double local_imag) {
  unsigned long long mb = dbits(local_max), ib = dbits(local_imag);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long a = __shfl_xor_sync(0xffffffffu, mb, o);
    unsigned long long b = __shfl_xor_sync(0xffffffffu, ib, o);
    mb = a > mb ? a : mb;
    ib = b > ib ? b : ib;
  }
  if ((threadIdx.x & 31) == 0 && (mb | ib)) {
    atomicMax(herm, mb);
    atomicMax(herm + 1, ib);
  }
}

// Last-stage registers -> final homes (local HBM or a peer's exchange buffer)
template <typename T, int N, int EPREF>
__device__ __forceinline__ void store_out(const PassParams& p, const Cpx<T>* v, int j, int alpha,
                                          int beta) {
  using C = Cpx<T>;
  using SC = Sched<N, EPREF>;
  constexpr int E = SC::E;
  constexpr int TPL = SC::TPL;
  constexpr int S = SC::S;
  constexpr int RL = S > 0 ? SC::radix(S - 1) : 1;
  constexpr int NSL = S > 0 ? SC::ns(S - 1) : 1;
  constexpr int NBL = E / RL;
  const T sc = static_cast<T>(p.scale);
#pragma unroll
  for (int t = 0; t < NBL; ++t) {
#pragma unroll
    for (int r = 0; r < RL; ++r) {
      const int k = j + t * TPL + r * NSL;
      if (k >= p.n_out) continue;
      int q = 0;
      int kk = k;
      if (p.ndest > 1) {
        q = static_cast<int>(k / p.oblk);
        kk = k - static_cast<int>(q * p.oblk);
      }
      const Dest& d = p.dest[q];
      const int64_t off = d.base + dst_alpha_off(p, d, alpha) + (int64_t)beta * d.sb + (int64_t)kk * d.sk;
      C x = v[t * RL + r];
      if (p.inverse) x.y = -x.y;
      if (p.spec.op) {
        x.x *= sc;
        x.y *= sc;
        spec_store<T>(p, d.ptr, off, x, k, alpha, beta);
      } else if (p.out_real) {
        reinterpret_cast<T*>(d.ptr)[off] = x.x * sc;
      } else {
        x.x *= sc;
        x.y *= sc;
        reinterpret_cast<C*>(d.ptr)[off] = x;
      }
    }
  }
}

#ifndef DFFTB_MINB
#define DFFTB_MINB 2
#endif

// ------------------------------------------------------- direct kernel
// One tile per CTA, stage-0 loads straight from global memory.  Used for
// layouts the TMA variant cannot describe (unaligned rows, tiny lanes).
template <typename T, int N, int EPREF, int W, bool ADJ>
__global__ void __launch_bounds__(W* Sched<N, EPREF>::TPL, DFFTB_MINB)
    fft_pass_kernel(const __grid_constant__ PassParams p) {
  using C = Cpx<T>;
  using SC = Sched<N, EPREF>;
  constexpr int TPL = SC::TPL;
  constexpr int LS = lane_stride<C>(N, ADJ ? W : 64);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* smem = reinterpret_cast<C*>(smem_raw);
  const int tid = threadIdx.x;
  const int w = ADJ ? tid % W : tid / TPL;
  const int j = ADJ ? tid / W : tid % TPL;
  const int tiles_b = (p.B + W - 1) / W;
  const int alpha = blockIdx.x / tiles_b;
  const int beta = (blockIdx.x - alpha * tiles_b) * W + w;
  const bool active = beta < p.B;
  C* lane = smem + w * LS;
  const C* tw = reinterpret_cast<const C*>(p.tw);
  const int64_t lane_off = in_alpha_off(p, alpha) + (int64_t)beta * p.in_sb;
  C v[SC::E];
  double lmax = 0.0, limag = 0.0;
  fetch0<T, N, EPREF>(
      v, j, active, p.in_mode, p.inverse,
      [&](int pos) { return __ldg(reinterpret_cast<const C*>(p.in) + lane_off + (int64_t)pos * p.in_si); },
      [&](int pos) { return __ldg(reinterpret_cast<const T*>(p.in) + lane_off + (int64_t)pos * p.in_si); },
      lmax, limag);
  if (p.in_mode == kInHermitian) herm_reduce(p.herm, lmax, limag);
  run_stages<T, N, EPREF, 0>(v, lane, tw, j);
  if (active) store_out<T, N, EPREF>(p, v, j, alpha, beta);
}

}  // namespace dfftb
