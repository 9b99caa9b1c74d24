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

enum LaneKind : int { kC2CFwd = 0, kC2CBwd = 1, kR2C = 2, kC2R = 3 };

struct TmaArgs {
  int64_t ntiles;
  int i_dim;       // tensor-map dimension holding the lane index i (1 or 2)
  int rows;        // box rows per TMA op (ADJ)
  int bulk;        // 1: contiguous cp.async.bulk, 0: tensor map
  int lane_bytes;  // bulk mode: bytes of one stored lane
  int ldgsts;      // strided lanes: per-thread cp.async (16 B) instead of TMA boxes
};

// Pipelined pass pairs (SURVEY §8(e) "overlap"): a producer pass and the
// consumer pass that reads its output run concurrently on disjoint CTAs of
// one launch.  Tiles are grouped into chunks of `tpc` consecutive tile
// indices that cover one range of the lane axis both passes share (the axis
// the exchange does not touch).  The producer adds, per chunk, the number of
// its tiles stored to a counter on every rank it writes to; the consumer
// loads a tile of chunk c only once its counter reached target[c].
constexpr int kMaxChunks = 32;
struct PipeArgs {
  int order_beta;  // > 0: chunks span order_beta beta tiles (chunk, alpha, beta order); 0: alpha-major
  int64_t tpc;     // tiles per chunk (0: not pipelined)
  int npub;        // producer: ranks written (0: not a producer)
  int pub_sys;     // producer writes other GPUs: system-scope fence
  unsigned long long* pub[kMaxDest];
  const unsigned long long* wait;  // consumer: own counters (nullptr: no waits)
  unsigned long long target[kMaxChunks];
  unsigned long long* timeout_flag;
  unsigned long long timeout_ns;
  // L2 ring (single GPU, two local passes): the intermediate lives in a ring
  // of `ring` planes that stays in L2 instead of a full buffer in HBM
  int ring;          // > 0: planes in the ring (the alpha index wraps)
  int ring_role;     // 1: producer stores into the ring; 2: consumer loads from it
  int ring_discard;  // consumer: drop each loaded 128-byte ring row from L2 (no write-back)
  int64_t peer_tpc, peer_ntiles;  // the other role's tiling: uniform per-chunk targets
  const unsigned long long* back_wait;  // producer: consumer's per-chunk consumed tiles
  unsigned long long* back_pub;         // consumer: publishes them
  int back_lag;                         // chunks the ring holds
};

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

template <typename T, int N, int W>
struct TmaLayout {
  using C = Cpx<T>;
  static constexpr int STG = W * N * (int)sizeof(C);  // one staging slot
  static constexpr int XCH = W * lane_stride<C>(N) * (int)sizeof(C);
};

// stage-0 fetch from a staging slot, compile-time lane kind
template <typename T, int N, int EPREF, int LK, class LDC, class LDR>
__device__ __forceinline__ void fetch0_lk(Cpx<T>* v, int j, LDC ldc, LDR ldr, T* m2 = nullptr,
                                          T* mi = nullptr) {
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
          // block max |X|^2 and the DC / Nyquist imaginary residues
          const T a = x.x * x.x + x.y * x.y;
          *m2 = a > *m2 ? a : *m2;
          if (pos == 0 || pos == N / 2) *mi = fabs(x.y) > *mi ? fabs(x.y) : *mi;
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

__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// spin until ctr[c] >= tgt (timeout -> flag, carry on)
__device__ __forceinline__ void spin_ge(const PipeArgs& pp, const unsigned long long* ctr, int c,
                                        unsigned long long tgt) {
  // after one timeout the execute is already failed: do not wait again
  if (ld_acquire_sys_u64(ctr + c) < tgt && ld_acquire_sys_u64(pp.timeout_flag) == 0) {
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_sys_u64(ctr + c) < tgt) {
      if (globaltimer_ns() - t0 > pp.timeout_ns) {
        atomicExch(pp.timeout_flag, 1ull);
        break;
      }
      __nanosleep(64);
    }
  }
}

// tiles of chunk c for a pass with `tpc` tiles per chunk and `ntiles` in all
__device__ __forceinline__ unsigned long long chunk_tiles(int64_t tpc, int64_t ntiles, int c) {
  const int64_t r = ntiles - (int64_t)c * tpc;
  return (unsigned long long)(r < tpc ? r : tpc);
}

// consumer side: spin until counter >= target (timeout -> flag, carry on)
__device__ __forceinline__ void pipe_wait(const PipeArgs& pp, int c) {
  const unsigned long long tgt = pp.ring ? chunk_tiles(pp.peer_tpc, pp.peer_ntiles, c) : pp.target[c];
  // after one timeout the execute is already failed: do not wait again
  if (ld_acquire_sys_u64(pp.wait + c) < tgt && ld_acquire_sys_u64(pp.timeout_flag) == 0) {
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_sys_u64(pp.wait + c) < tgt) {
      if (globaltimer_ns() - t0 > pp.timeout_ns) {
        atomicExch(pp.timeout_flag, 1ull);
        break;
      }
      __nanosleep(128);
    }
  }
  // the chunk was written through the generic proxy; TMA reads it next
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// The tile loop of one pass over tiles cta, cta + ncta, ...: TMA prefetch of
// the next STAGES tiles into shared memory while the current tile is
// transformed and stored.  Shared by the single-pass kernel and both roles of
// the pipelined pair kernel.
template <typename T, int N, int EPREF, int W, bool ADJ, int STAGES, int LK, bool SPEC = false, bool PIPE = false>
__device__ __forceinline__ void pass_tiles(const PassParams& p, const CUtensorMap& tm, const TmaArgs& ta,
                                           const PipeArgs& pp, int cta, int ncta, unsigned char* smem) {
  using C = Cpx<T>;
  using SC = Sched<N, EPREF>;
  using TL = TmaLayout<T, N, W>;
  constexpr int TPL = SC::TPL;
  constexpr int LS = lane_stride<C>(N);
  unsigned char* stg = smem;
  C* xch = reinterpret_cast<C*>(smem + STAGES * TL::STG);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * TL::STG + TL::XCH);
  void** sptr = reinterpret_cast<void**>(bars + STAGES);  // destination pointers

  const int tid = threadIdx.x;
  const int w = ADJ ? tid % W : tid / TPL;
  const int j = ADJ ? tid / W : tid % TPL;
  const int tiles_b = (p.B + W - 1) / W;
  const C* tw = reinterpret_cast<const C*>(p.tw);
  constexpr int ESIZE = LK == kR2C ? (int)sizeof(T) : (int)sizeof(C);
  const T sc = static_cast<T>(p.scale);
  TwBase<T, N, EPREF> twb;  // per-thread twiddle bases, loaded once
  load_twbase<T, N, EPREF>(twb, tw, j);
  const TwBase<T, N, EPREF>* twbp = &twb;

  auto decode = [&](int64_t t, int& alpha, int& beta0) {
    int64_t bc;
    if (PIPE && pp.order_beta) {
      // chunk-major, then alpha, then the chunk's beta tiles: concurrent CTAs
      // still cover adjacent lanes (contiguous rows) inside a chunk
      const int64_t bpc = pp.order_beta;  // beta tiles per chunk
      const int64_t c = t / pp.tpc;
      const int64_t r = t - c * pp.tpc;
      const int64_t width = min(bpc, (int64_t)tiles_b - c * bpc);
      const int64_t a = r / width;
      alpha = (int)a;
      bc = c * bpc + (r - a * width);
    } else {
      alpha = (int)(t / tiles_b);
      bc = t - (int64_t)alpha * tiles_b;
    }
    beta0 = (int)bc * W;
  };

  // called by every thread; TMA ops are issued by thread 0 only
  auto issue = [&](int64_t t, int s) {
    int alpha, beta0;
    decode(t, alpha, beta0);
    unsigned char* dst = stg + s * TL::STG;
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
    if (PIPE && pp.wait) pipe_wait(pp, (int)(t / pp.tpc));
    if (PIPE && pp.back_wait) {
      // ring producer: the slot of chunk c is free once the consumer has
      // loaded every tile of chunk c - lag
      const int c = (int)(t / pp.tpc) - pp.back_lag;
      if (c >= 0) spin_ge(pp, pp.back_wait, c, chunk_tiles(pp.peer_tpc, pp.peer_ntiles, c));
    }
    if (PIPE && pp.ring_role == 2) alpha %= pp.ring;
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
  __syncthreads();
  for (int s = 0; s < STAGES; ++s) {
    const int64_t t = cta + (int64_t)s * ncta;
    if (t < ta.ntiles) issue(t, s);
  }

  T lmax = T(0), limag = T(0);  // C2R statistics, reduced once per CTA at the end
  unsigned long long done = 0;  // producer: tiles stored in the current chunk
  unsigned long long used = 0;  // ring consumer: tiles loaded in the current chunk
  int k = 0;
  for (int64_t t = cta; t < ta.ntiles; t += ncta, ++k) {
    const int s = k % STAGES;
    mbar_wait(&bars[s], (uint32_t)((k / STAGES) & 1));
    int alpha, beta;
    decode(t, alpha, beta);
    if (PIPE && pp.ring_role == 2 && pp.ring_discard) {
      // the ring rows of this tile are in shared memory now and no other
      // tile reads them: drop them from L2 so they are never written back
      const int aw = alpha % pp.ring;
      for (int i = tid; i < N; i += W * TPL) {
        const C* row = reinterpret_cast<const C*>(p.in) + (int64_t)aw * p.in_sa + (int64_t)beta * p.in_sb +
                       (int64_t)i * p.in_si;
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(row) : "memory");
      }
    }
    beta += w;
    const unsigned char* st = stg + s * TL::STG;
    C v[SC::E];
    if constexpr (ADJ) {
      const C* scp = reinterpret_cast<const C*>(st);
      fetch0_lk<T, N, EPREF, LK>(
          v, j, [&](int pos) { return scp[pos * W + w]; }, [&](int) { return T(0); });
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
      const int64_t t2 = t + (int64_t)STAGES * ncta;
      if (t2 < ta.ntiles) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(t2, s);
      }
    }
#if DFFTB_EXP_NOCOMPUTE  // timing experiment only (wrong results): data movement alone
    (void)tw;
#else
    run_stages<T, N, EPREF, 0>(v, xch + w * LS, tw, j, twbp);
#endif
    const int alpha_st = (PIPE && pp.ring_role == 1) ? alpha % pp.ring : alpha;
    if (beta < p.B) store_lk<T, N, EPREF, LK, SPEC>(p, sptr, v, j, alpha_st, beta, sc);
    if (PIPE && pp.back_pub) {
      // ring consumer: this tile's ring rows were loaded (and discarded)
      ++used;
      const int64_t c = t / pp.tpc;
      if (t + ncta >= ta.ntiles || (t + ncta) / pp.tpc != c) {
        __syncthreads();
        if (tid == 0)
          asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(pp.back_pub + c), "l"(used) : "memory");
        used = 0;
      }
    }
    if (PIPE && pp.npub) {
      // producer: publish a chunk once this CTA has no further tile in it
      ++done;
      const int64_t c = t / pp.tpc;
      if (t + ncta >= ta.ntiles || (t + ncta) / pp.tpc != c) {
        // gpu scope: bar.sync orders the CTA's stores before thread 0's
        // red.release (cumulativity, the CUTLASS semaphore pattern); peers on
        // other GPUs get a full system fence from every thread
        if (pp.pub_sys) __threadfence_system();
        __syncthreads();
        if (tid == 0) {
          for (int q = 0; q < pp.npub; ++q) {
            if (pp.pub_sys)
              asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(pp.pub[q] + c), "l"(done) : "memory");
            else
              asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(pp.pub[q] + c), "l"(done) : "memory");
          }
        }
        done = 0;
      }
    }
  }
  if constexpr (LK == kC2R) herm_reduce<T>(p.herm, sqrt(lmax), limag);
}

// The single-pass kernel.  Its body is the tile loop of pass_tiles written
// out with blockIdx / gridDim (measured 1-2% faster than calling pass_tiles,
// which the pipelined pair kernel below uses).  SPEC: the last forward pass of
// a spectral operator (multiplier epilogue).
template <typename T, int N, int EPREF, int W, bool ADJ, int STAGES, int LK, bool SPEC = false>
__global__ void __launch_bounds__(W* Sched<N, EPREF>::TPL, DFFTB_TMA_MINB)
    fft_pass_tma_kernel(const __grid_constant__ PassParams p, const __grid_constant__ CUtensorMap tm,
                        const TmaArgs ta) {
  using C = Cpx<T>;
  using SC = Sched<N, EPREF>;
  using TL = TmaLayout<T, N, W>;
  constexpr int TPL = SC::TPL;
  constexpr int LS = lane_stride<C>(N);
  extern __shared__ __align__(1024) unsigned char smem_tma[];
  unsigned char* stg = smem_tma;
  C* xch = reinterpret_cast<C*>(smem_tma + STAGES * TL::STG);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_tma + STAGES * TL::STG + TL::XCH);
  void** sptr = reinterpret_cast<void**>(bars + STAGES);  // destination pointers

  const int tid = threadIdx.x;
  const int w = ADJ ? tid % W : tid / TPL;
  const int j = ADJ ? tid / W : tid % TPL;
  const int tiles_b = (p.B + W - 1) / W;
  C* lane = xch + w * LS;
  const C* tw = reinterpret_cast<const C*>(p.tw);
  constexpr int ESIZE = LK == kR2C ? (int)sizeof(T) : (int)sizeof(C);
  const T sc = static_cast<T>(p.scale);
#if DFFTB_TWB
  TwBase<T, N, EPREF> twb;  // per-thread twiddle bases, loaded once per kernel
  load_twbase<T, N, EPREF>(twb, tw, j);
  const TwBase<T, N, EPREF>* twbp = &twb;
#else
  const TwBase<T, N, EPREF>* twbp = nullptr;
#endif

  // called by every thread; TMA ops are issued by thread 0 only
  auto issue = [&](int64_t t, int s) {
    const int alpha = (int)(t / tiles_b);
    const int beta0 = (int)(t - (int64_t)alpha * tiles_b) * W;
    unsigned char* dst = stg + s * TL::STG;
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
  __syncthreads();
  for (int s = 0; s < STAGES; ++s) {
    const int64_t t = blockIdx.x + (int64_t)s * gridDim.x;
    if (t < ta.ntiles) issue(t, s);
  }

  T lmax = T(0), limag = T(0);  // C2R statistics, reduced once per CTA at the end
  int k = 0;
  for (int64_t t = blockIdx.x; t < ta.ntiles; t += gridDim.x, ++k) {
    const int s = k % STAGES;
    mbar_wait(&bars[s], (uint32_t)((k / STAGES) & 1));
    const int alpha = (int)(t / tiles_b);
    const int beta = (int)(t - (int64_t)alpha * tiles_b) * W + w;
    const unsigned char* st = stg + s * TL::STG;
    C v[SC::E];
    if constexpr (ADJ) {
      const C* scp = reinterpret_cast<const C*>(st);
      fetch0_lk<T, N, EPREF, LK>(
          v, j, [&](int pos) { return scp[pos * W + w]; }, [&](int) { return T(0); });
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
    if (beta < p.B) store_lk<T, N, EPREF, LK, SPEC>(p, sptr, v, j, alpha, beta, sc);
  }
  if constexpr (LK == kC2R) herm_reduce<T>(p.herm, sqrt(lmax), limag);
}

// Pipelined pair: CTAs [0, ncta_a) run the producer pass, the rest the
// consumer.  One launch, so both roles are co-resident (grid <= SMs x
// occupancy): the consumer's waits can always be satisfied.
template <typename T, int N, int EPREF, int W, bool ADJ_A, bool ADJ_B, int STAGES, int LK>
__global__ void __launch_bounds__(W* Sched<N, EPREF>::TPL, DFFTB_TMA_MINB)
    fft_pipe_kernel(const __grid_constant__ PassParams pa, const __grid_constant__ CUtensorMap tma,
                    const __grid_constant__ TmaArgs taa, const __grid_constant__ PipeArgs ppa,
                    const __grid_constant__ PassParams pb, const __grid_constant__ CUtensorMap tmb,
                    const __grid_constant__ TmaArgs tab, const __grid_constant__ PipeArgs ppb, int ncta_a) {
  extern __shared__ __align__(1024) unsigned char smem_tma[];
  if ((int)blockIdx.x < ncta_a)
    pass_tiles<T, N, EPREF, W, ADJ_A, STAGES, LK, false, true>(pa, tma, taa, ppa, blockIdx.x, ncta_a, smem_tma);
  else
    pass_tiles<T, N, EPREF, W, ADJ_B, STAGES, LK, false, true>(pb, tmb, tab, ppb, blockIdx.x - ncta_a,
                                                                gridDim.x - ncta_a, smem_tma);
}

}  // namespace dfftb
