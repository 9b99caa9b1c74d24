// TMA-prefetch persistent FFT pass kernel (the main B200 path).
//
// Each CTA walks tiles blockIdx.x, +gridDim.x, ...  The input tiles of the
// next STAGES tiles are brought into shared memory by the Tensor Memory
// Accelerator while the current tile is transformed and stored, so HBM reads
// stay in flight through the butterfly and store phases:
//   * lanes along a strided axis (ADJ): cp.async.bulk.tensor.3d boxes of
//     [rows <= 256][W adjacent lanes] (zero-filled past the last lane);
//   * contiguous lanes: one cp.async.bulk of W whole lanes.
// Completion is tracked with one mbarrier (expect_tx) per staging slot.
//
// Lane kind LK is a template parameter so the lane semantics cost nothing:
//   0 C2C forward, 1 C2C backward (conj in/out), 2 R2C (real in),
//   3 C2R (Hermitian half in, real out; irfft_1d, kernels.hpp:362-389).
#pragma once

#include "fft_pass.cuh"

namespace dfftb {

// kR2Ch / kC2Rh: the half-length forms of R2C / C2R (the kernel's N is n/2):
// an n-point real lane is an N-point complex FFT plus a post- (R2C) or
// pre-twiddle (C2R) over the bin pairs (k, N - k).
enum LaneKind : int { kC2CFwd = 0, kC2CBwd = 1, kR2C = 2, kC2R = 3, kR2Ch = 4, kC2Rh = 5 };
// staged elements per C2Rh lane beyond N: bin N plus the internal row padding
constexpr int kC2RhExtra = 8;

// A launch covers the tile box [a0, a0 + na) x [bt0, bt0 + nbt) of (alpha,
// beta tile) -- the whole pass, or one chunk of a pipelined exchange.
struct TmaArgs {
  int64_t ntiles;  // na * nbt
  int a0, bt0;     // first alpha, first beta tile of the box
  int na, nbt;     // alphas, beta tiles of the box
  int i_dim;       // tensor-map dimension holding the lane index i (1 or 2)
  int rows;        // box rows per TMA op (ADJ)
  int bulk;        // 1: contiguous cp.async.bulk, 0: tensor map
  int lane_bytes;  // bulk mode: bytes of one stored lane
  int rhalf;       // R2C / C2R lanes as half-length complex FFTs (kR2Ch / kC2Rh)
  int W;           // lanes per tile
  int ldgsts;      // strided lanes: per-thread cp.async (16 B) instead of TMA boxes
};

// tile t of the launch box -> (alpha, beta tile), beta tiles fastest
__device__ __forceinline__ void tile_coords(const TmaArgs& ta, int64_t t, int& alpha, int& bt) {
  const int ar = (int)(t / ta.nbt);
  alpha = ta.a0 + ar;
  bt = ta.bt0 + (int)(t - (int64_t)ar * ta.nbt);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Staging rows of the per-thread cp.async loader for 8-byte-aligned fp32
// rows (ADJ, W >= 16): W + 2 slots, so a row that starts 8 bytes off the
// 16-byte grid lands one slot later and its inner lanes still move as 16-byte
// pairs.
template <typename T, bool ADJ, int W>
struct RowPad {
  static constexpr int value = (ADJ && sizeof(T) == 4 && W >= 16) ? 2 : 0;
};

template <typename T, int N, int W, int EXTRA = 0, int PADR = 0, int LSV = 0>
struct TmaLayout {
  using C = Cpx<T>;
  // one staging slot (EXTRA: C2Rh's bin N + pad; PADR: cp.async row padding)
  static constexpr int STG = (W + PADR) * (N + EXTRA) * (int)sizeof(C);
  // exchange buffer: W lanes of LSV slots (the kernel's lane stride)
  static constexpr int XCH = W * (LSV > 0 ? LSV : lane_stride<C>(N, W)) * (int)sizeof(C);
};

// stage-0 fetch from a staging slot, compile-time lane kind
template <typename T, int N, int EPREF, int LK, class LDC, class LDR>
__device__ __forceinline__ void fetch0_lk(Cpx<T>* v, int j, LDC ldc, LDR ldr, double* m2 = nullptr,
                                          double* mi = nullptr) {
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
      C x;
      if constexpr (LK == kC2CFwd) {
        x = ldc(pos);
      } else if constexpr (LK == kC2CBwd) {
        x = ldc(pos);
        x.y = -x.y;
      } else if constexpr (LK == kR2C) {
        x = C{ldr(pos), T(0)};
      } else {
        // Hermitian extension, DC/Nyquist imaginary parts dropped, then the
        // conj of the backward transform: x = conj(X_ext).  (The NonHermitian
        // statistics are taken from the staged bins by the kernel.)
        const bool lo = pos <= N / 2;
        x = ldc(lo ? pos : N - pos);
        if (m2) {
          // NonHermitian statistics of the stored bins as they are read
          // (every bin 0..N/2 is read at least once; max is idempotent):
          // block max |X|^2 and the DC / Nyquist imaginary residues, in
          // double so fp32 magnitudes neither overflow nor underflow
          const double a = (double)x.x * (double)x.x + (double)x.y * (double)x.y;
          *m2 = a > *m2 ? a : *m2;
          const double ai = fabs((double)x.y);
          if (pos == 0 || pos == N / 2) *mi = ai > *mi ? ai : *mi;
        }
        if (pos == 0 || pos == N / 2) x.y = T(0);
        if (lo) x.y = -x.y;
      }
      v[t * R0 + r] = x;
    }
  }
}

// final store, compile-time lane kind; per-tile addressing precomputed
template <typename T, int N, int EPREF, int LK, bool SPEC = false>
__device__ __forceinline__ void store_lk(const PassParams& p, void* const* sptr, const Cpx<T>* v,
                                         int j, int alpha, int beta, T sc) {
  using C = Cpx<T>;
  using SC = Sched<N, EPREF>;
  constexpr int E = SC::E;
  constexpr int TPL = SC::TPL;
  constexpr int S = SC::S;
  constexpr int RL = S > 0 ? SC::radix(S - 1) : 1;
  constexpr int NSL = S > 0 ? SC::ns(S - 1) : 1;
  constexpr int NBL = E / RL;
  auto put = [&](void* base, int64_t off, C x, int k) {
    if constexpr (LK == kC2CBwd) x.y = -x.y;
    if constexpr (SPEC && LK != kC2R) {
      x.x *= sc;
      x.y *= sc;
      spec_store<T>(p, base, off, x, k, alpha, beta);
      return;
    }
    if constexpr (LK == kC2R) {
      reinterpret_cast<T*>(base)[off] = x.x * sc;
    } else {
      x.x *= sc;
      x.y *= sc;
      reinterpret_cast<C*>(base)[off] = x;
    }
  };
  if (p.store_mode != 2) {
    const Dest& d0 = p.dest[0];
    const int64_t tile = d0.base + dst_alpha_off(p, d0, alpha) + (int64_t)beta * d0.sb;
    const int sk = (int)d0.sk;
#pragma unroll
    for (int t = 0; t < NBL; ++t) {
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        const int k = j + t * TPL + r * NSL;
        if constexpr (LK == kR2C) {
          if (k > N / 2) continue;
        }
        if (p.store_mode == 0) {
          put(d0.ptr, tile + (int64_t)k * sk, v[t * RL + r], k);
        } else {
          const int q = k >> p.oshift;
          const int kk = k & p.omask;
          put(sptr[q], tile + (int64_t)kk * sk, v[t * RL + r], k);
        }
      }
    }
  } else {
#pragma unroll
    for (int t = 0; t < NBL; ++t) {
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        const int k = j + t * TPL + r * NSL;
        if (k >= p.n_out) continue;
        const int q = static_cast<int>(k / p.oblk);
        const int kk = k - static_cast<int>(q * p.oblk);
        const Dest& d = p.dest[q];
        put(d.ptr, d.base + dst_alpha_off(p, d, alpha) + (int64_t)beta * d.sb + (int64_t)kk * d.sk,
            v[t * RL + r], k);
      }
    }
  }
}

// Half-length C2R pre-twiddle (irfft_1d semantics, kernels.hpp:362-389, on
// an N-point transform): from the Hermitian bins X[0..N] of a 2N-point lane,
//   Z[m] = (X[m] + conj X[N-m]) + i (X[m] - conj X[N-m]) e^{+i pi m / N},
// whose N-point inverse gives z[m] = x[2m] + i x[2m+1].  DC / Nyquist
// imaginary parts are dropped and the NonHermitian statistics taken as the
// bins are read.  v receives conj(Z) (inverse = conj of the forward FFT).
template <typename T, int N, int EPREF>
__device__ __forceinline__ void fetch_c2rh(Cpx<T>* v, int j, const Cpx<T>* X, const Cpx<T>* twn, double* m2,
                                           double* mi) {
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
      const int m = j + t * TPL + r * (N / R0);
      C a = X[m], b = X[N - m];
      if (m2) {
        const double aa = (double)a.x * (double)a.x + (double)a.y * (double)a.y;
        const double bb = (double)b.x * (double)b.x + (double)b.y * (double)b.y;
        *m2 = fmax(*m2, fmax(aa, bb));
        if (m == 0) *mi = fmax(*mi, fmax(fabs((double)a.y), fabs((double)b.y)));
      }
      if (m == 0) {
        a.y = T(0);
        b.y = T(0);
      }
      const C cb = C{b.x, -b.y};
      const C e = cadd(a, cb), d = csub(a, cb);
      C w = __ldg(twn + m);
      w.y = -w.y;
      const C o = cmul(d, w);
      v[t * R0 + r] = C{e.x - o.y, -(e.y + o.x)};  // conj(e + i o)
    }
  }
}

// Half-length R2C post-twiddle: Z = FFT_N(x[2m] + i x[2m+1]) in the
// registers' last-stage positions k ->
//   X[k] = (Z[k] + conj Z[N-k]) / 2 + W_2N^k (Z[k] - conj Z[N-k]) / (2i),
// the pair partner read through the lane's shared-memory slots; bin N
// (= Re Z[0] - Im Z[0]) goes to the thread holding bin 0.
template <typename T, int N, int EPREF>
__device__ __forceinline__ void post_r2ch(Cpx<T>* v, Cpx<T>* lane, const Cpx<T>* twn, int j, Cpx<T>& xn) {
  using C = Cpx<T>;
  using SC = Sched<N, EPREF>;
  constexpr int E = SC::E;
  constexpr int TPL = SC::TPL;
  constexpr int S = SC::S;
  constexpr int RL = S > 0 ? SC::radix(S - 1) : 1;
  constexpr int NSL = S > 0 ? SC::ns(S - 1) : 1;
  constexpr int NBL = E / RL;
  __syncthreads();  // every thread is done with the last stage's exchange reads
#pragma unroll
  for (int t = 0; t < NBL; ++t)
#pragma unroll
    for (int r = 0; r < RL; ++r) lane[spad<C>(j + t * TPL + r * NSL)] = v[t * RL + r];
  __syncthreads();
  xn = C{v[0].x - v[0].y, T(0)};
#pragma unroll
  for (int t = 0; t < NBL; ++t) {
#pragma unroll
    for (int r = 0; r < RL; ++r) {
      const int k = j + t * TPL + r * NSL;
      const C zk = v[t * RL + r];
      C zr = lane[spad<C>((N - k) & (N - 1))];
      zr.y = -zr.y;
      const C e = C{(zk.x + zr.x) * T(0.5), (zk.y + zr.y) * T(0.5)};
      const C d = csub(zk, zr);
      const C o = C{d.y * T(0.5), -d.x * T(0.5)};  // d / (2i)
      v[t * RL + r] = cadd(e, cmul(__ldg(twn + k), o));
    }
  }
  __syncthreads();  // the next tile's first exchange overwrites the lane slots
}

// one complex output element k of a lane (any store mode: the general
// destination formula)
template <typename T>
__device__ __forceinline__ void store_one(const PassParams& p, Cpx<T> x, int k, int alpha, int beta, T sc) {
  if (k >= p.n_out) return;
  const int q = static_cast<int>(k / p.oblk);
  const int kk = k - static_cast<int>(q * p.oblk);
  const Dest& d = p.dest[q];
  x.x *= sc;
  x.y *= sc;
  reinterpret_cast<Cpx<T>*>(d.ptr)[d.base + dst_alpha_off(p, d, alpha) + (int64_t)beta * d.sb + (int64_t)kk * d.sk] = x;
}

// Half-length C2R store: register position m holds r = FFT(conj Z)[m], so
// z[m] = conj(r) and the real outputs 2m, 2m+1 are r.x, -r.y (one dest).
template <typename T, int N, int EPREF>
__device__ __forceinline__ void store_c2rh(const PassParams& p, const Cpx<T>* v, int j, int alpha, int beta, T sc) {
  using SC = Sched<N, EPREF>;
  constexpr int E = SC::E;
  constexpr int TPL = SC::TPL;
  constexpr int S = SC::S;
  constexpr int RL = S > 0 ? SC::radix(S - 1) : 1;
  constexpr int NSL = S > 0 ? SC::ns(S - 1) : 1;
  constexpr int NBL = E / RL;
  const Dest& d = p.dest[0];
  const int64_t base = d.base + dst_alpha_off(p, d, alpha) + (int64_t)beta * d.sb;
  T* out = reinterpret_cast<T*>(d.ptr);
  const bool pair = d.sk == 1 && (base & 1) == 0;
#pragma unroll
  for (int t = 0; t < NBL; ++t) {
#pragma unroll
    for (int r = 0; r < RL; ++r) {
      const int m = j + t * TPL + r * NSL;
      const Cpx<T> x = v[t * RL + r];
      if (pair) {
        reinterpret_cast<Cpx<T>*>(out + base)[m] = Cpx<T>{x.x * sc, -x.y * sc};
      } else {
        out[base + (int64_t)(2 * m) * d.sk] = x.x * sc;
        out[base + (int64_t)(2 * m + 1) * d.sk] = -x.y * sc;
      }
    }
  }
}

// The pass kernel: persistent CTAs walk the tiles of the launch box.  SPEC:
// the last forward pass of a spectral operator (multiplier epilogue).
template <typename T, int N, int EPREF, int W, bool ADJ, int STAGES, int LK, bool SPEC = false,
          int MINB = DFFTB_TMA_MINB>
__global__ void __launch_bounds__(W* Sched<N, EPREF>::TPL, MINB)
    fft_pass_tma_kernel(const __grid_constant__ PassParams p, const __grid_constant__ CUtensorMap tm,
                        const TmaArgs ta) {
  using C = Cpx<T>;
  using SC = Sched<N, EPREF>;
  constexpr int PADR = RowPad<T, ADJ, W>::value;
  constexpr int LS = pass_lane_stride<T, N, EPREF, W, ADJ>();
  using TL = TmaLayout<T, N, W, LK == kC2Rh ? kC2RhExtra : 0, PADR, LS>;
  constexpr int TPL = SC::TPL;
  extern __shared__ __align__(1024) unsigned char smem_tma[];
  unsigned char* stg = smem_tma;
  C* xch = reinterpret_cast<C*>(smem_tma + STAGES * TL::STG);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_tma + STAGES * TL::STG + TL::XCH);
  void** sptr = reinterpret_cast<void**>(bars + STAGES);  // destination pointers

  const int tid = threadIdx.x;
  const int w = ADJ ? tid % W : tid / TPL;
  const int j = ADJ ? tid / W : tid % TPL;
  C* lane = xch + w * LS;
  const C* tw = reinterpret_cast<const C*>(p.tw);
  // bytes per element of the input's strides: reals for R2C lanes
  constexpr int ESIZE = (LK == kR2C || LK == kR2Ch) ? (int)sizeof(T) : (int)sizeof(C);
  const T sc = static_cast<T>(p.scale);
  const C* twn = reinterpret_cast<const C*>(p.tw2);  // 2N-point table (half-length R2C / C2R)
#if DFFTB_TWB
  TwBase<T, N, EPREF> twb;  // per-thread twiddle bases, loaded once per kernel
  load_twbase<T, N, EPREF>(twb, tw, j);
  const TwBase<T, N, EPREF>* twbp = &twb;
#else
  const TwBase<T, N, EPREF>* twbp = nullptr;
#endif

  // called by every thread; TMA ops are issued by thread 0 only
  auto issue = [&](int64_t t, int s) {
    int alpha, beta0;
    tile_coords(ta, t, alpha, beta0);
    beta0 *= W;
    unsigned char* dst = stg + s * TL::STG;
    if constexpr (ADJ && PADR > 0) {
      if (ta.ldgsts) {
        // fp32 rows 8-byte aligned only (C2R user blocks of n/2+1 bins):
        // 16-byte cp.async pairs of adjacent lanes.  Row i lands at slot
        // i*(W+2) + par(i): an aligned row as W/2 pairs; a row 8 bytes off
        // as lane 0 alone, W/2-1 pairs, lane W-1 alone (lanes in_sb = 1
        // apart).  Lanes past B read as zero.
        const C* src0 = reinterpret_cast<const C*>(p.in) + (int64_t)alpha * p.in_sa + beta0;
        const int64_t par0 = (int64_t)(reinterpret_cast<uintptr_t>(src0) >> 3);
        constexpr int RS = W + PADR, UPR = W / 2 + 1;  // slots and copy units per row
        constexpr int NT = W * TPL;
        const int nval = p.B - beta0;  // valid lanes of this tile
        for (int e = tid; e < UPR * N; e += NT) {
          const int i = e / UPR, u = e - (e / UPR) * UPR;
          const int par = (int)((par0 + (int64_t)i * p.in_si) & 1);
          int w0, cnt;  // first lane, lanes (1 or 2)
          if (!par) {
            if (u == UPR - 1) continue;
            w0 = 2 * u;
            cnt = 2;
          } else {
            w0 = u == 0 ? 0 : 2 * u - 1;
            cnt = (u == 0 || u == UPR - 1) ? 1 : 2;
          }
          const int nv = min(max(nval - w0, 0), cnt);  // valid lanes of this unit
          // the unit's own (16-byte aligned for pairs) address even when
          // nv < cnt: only 8*nv bytes are read
          const C* src = src0 + (int64_t)i * p.in_si + w0;
          const uint32_t sdst = smem_u32(dst + ((size_t)i * RS + w0 + par) * sizeof(C));
          if (cnt == 2)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sdst), "l"(src), "r"(8 * nv)
                         : "memory");
          else
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sdst), "l"(src), "r"(8 * nv)
                         : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&bars[s])) : "memory");
        return;
      }
    }
    if (ADJ && ta.ldgsts) {
      // very large row strides (e.g. the axis-0 pass) translate one page per
      // row: spread the rows over all threads' LSU path instead of one TMA
      // box walk.  Tile layout [i][w] as for TMA; lanes past B read as zero.
      const C* src0 = reinterpret_cast<const C*>(p.in) + (int64_t)alpha * p.in_sa;
      constexpr int NT = W * TPL;
      for (int e = tid; e < W * N; e += NT) {
        const int i = e / W, ww = e - (e / W) * W;
        const bool ok = beta0 + ww < p.B;
        const C* src = src0 + (int64_t)(ok ? beta0 + ww : 0) * p.in_sb + (int64_t)i * p.in_si;
        if constexpr (sizeof(C) == 16)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst + (size_t)e * sizeof(C))),
                       "l"(src), "r"(ok ? 16 : 0)
                       : "memory");
        else  // fp32 complex: 8-byte copies (rows only 8-byte aligned)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst + (size_t)e * sizeof(C))),
                       "l"(src), "r"(ok ? 8 : 0)
                       : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&bars[s])) : "memory");
      return;
    }
    if (tid != 0) return;
    if constexpr (ADJ) {
      mbar_expect_tx(&bars[s], (uint32_t)(W * N * sizeof(C)));
      for (int r0 = 0; r0 < N; r0 += ta.rows) {
        const int c1 = ta.i_dim == 1 ? r0 : alpha;
        const int c2 = ta.i_dim == 1 ? alpha : r0;
        tma_load_3d(dst + (size_t)r0 * W * sizeof(C), &tm, 2 * beta0, c1, c2, &bars[s]);
      }
    } else {
      const int nvalid = min(W, p.B - beta0);
      const uint32_t bytes = (uint32_t)nvalid * (uint32_t)ta.lane_bytes;
      mbar_expect_tx(&bars[s], bytes);
      const unsigned char* src = reinterpret_cast<const unsigned char*>(p.in) +
                                 (in_alpha_off(p, alpha) + (int64_t)beta0 * p.in_sb) * ESIZE;
      bulk_load(dst, src, bytes, &bars[s]);
    }
  };

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], (ADJ && ta.ldgsts) ? W * TPL : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < kMaxDest) sptr[tid] = p.dest[tid].ptr;
  // Programmatic dependent launch: everything above (barriers, twiddle bases)
  // overlaps the previous pass's tail; its output is read only after this.
  // Dependents may launch once every CTA of this grid is resident.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();
  for (int s = 0; s < STAGES; ++s) {
    const int64_t t = blockIdx.x + (int64_t)s * gridDim.x;
    if (t < ta.ntiles) issue(t, s);
  }

  double lmax = 0.0, limag = 0.0;  // C2R statistics, reduced once per CTA at the end
  int k = 0;
  for (int64_t t = blockIdx.x; t < ta.ntiles; t += gridDim.x, ++k) {
    const int s = k % STAGES;
    mbar_wait(&bars[s], (uint32_t)((k / STAGES) & 1));
    int alpha, beta;
    tile_coords(ta, t, alpha, beta);
    beta = beta * W + w;
    const unsigned char* st = stg + s * TL::STG;
    C v[SC::E];
    if constexpr (ADJ && PADR > 0) {
      const C* scp = reinterpret_cast<const C*>(st);
      if (ta.ldgsts) {
        // padded rows of the paired cp.async loader (see issue)
        const int64_t par0 = (int64_t)(reinterpret_cast<uintptr_t>(reinterpret_cast<const C*>(p.in) +
                                                                   (int64_t)alpha * p.in_sa + (beta - w)) >> 3);
        fetch0_lk<T, N, EPREF, LK>(
            v, j, [&](int pos) { return scp[pos * (W + PADR) + w + (int)((par0 + (int64_t)pos * p.in_si) & 1)]; },
            [&](int) { return T(0); });
      } else {
        fetch0_lk<T, N, EPREF, LK>(
            v, j, [&](int pos) { return scp[pos * W + w]; }, [&](int) { return T(0); });
      }
    } else if constexpr (ADJ) {
      const C* scp = reinterpret_cast<const C*>(st);
      fetch0_lk<T, N, EPREF, LK>(
          v, j, [&](int pos) { return scp[pos * W + w]; }, [&](int) { return T(0); });
    } else if constexpr (LK == kR2Ch) {
      // 2N reals read as N complex z[m] = x[2m] + i x[2m+1]
      const C* scp = reinterpret_cast<const C*>(st) + w * (ta.lane_bytes / (int)sizeof(C));
      fetch0_lk<T, N, EPREF, kC2CFwd>(v, j, [&](int pos) { return scp[pos]; }, [&](int) { return T(0); });
    } else if constexpr (LK == kC2Rh) {
      const C* scp = reinterpret_cast<const C*>(st) + w * (ta.lane_bytes / (int)sizeof(C));
      const bool stats = beta < p.B;
      fetch_c2rh<T, N, EPREF>(v, j, scp, twn, stats ? &lmax : nullptr, stats ? &limag : nullptr);
    } else {
      const int ll = ta.lane_bytes / ESIZE;  // stored lane length in elements
      const C* scp = reinterpret_cast<const C*>(st) + w * ll;
      const T* srp = reinterpret_cast<const T*>(st) + w * ll;
      // C2R: NonHermitian statistics (max |X|^2 -> one sqrt per CTA, exact by
      // monotonicity; DC / Nyquist |Im|) of active lanes, taken in the fetch
      const bool stats = LK == kC2R && beta < p.B;
      fetch0_lk<T, N, EPREF, LK>(
          v, j, [&](int pos) { return scp[pos]; }, [&](int pos) { return srp[pos]; },
          stats ? &lmax : nullptr, stats ? &limag : nullptr);
    }
    __syncthreads();  // staging slot s fully consumed by every thread
    {
      const int64_t t2 = t + (int64_t)STAGES * gridDim.x;
      if (t2 < ta.ntiles) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(t2, s);
      }
    }
    run_stages<T, N, EPREF, 0>(v, lane, tw, j, twbp);
    if constexpr (LK == kR2Ch) {
      C xn;  // bin N (real), computed by the thread holding bin 0
      post_r2ch<T, N, EPREF>(v, lane, twn, j, xn);
      if (beta < p.B) {
        store_lk<T, N, EPREF, kC2CFwd, false>(p, sptr, v, j, alpha, beta, sc);
        if (j == 0) store_one<T>(p, xn, N, alpha, beta, sc);
      }
    } else if constexpr (LK == kC2Rh) {
      if (beta < p.B) store_c2rh<T, N, EPREF>(p, v, j, alpha, beta, sc);
    } else {
      if (beta < p.B) store_lk<T, N, EPREF, LK, SPEC>(p, sptr, v, j, alpha, beta, sc);
    }
  }
  if constexpr (LK == kC2R || LK == kC2Rh) herm_reduce(p.herm, sqrt(lmax), limag);
}

}  // namespace dfftb
