// Two FFT axes per HBM round trip: the L2-resident plane pipeline.
//
// When the transpose between two consecutive FFT stages is local (slab
// decompositions, pencil grids with P1 == 1, the single-GPU case), the
// reference runs F2 -> (T1 local) -> F1 as two full passes over HBM
// (plan.hpp:484-509).  Here one persistent kernel runs both, plane by plane
// (a plane = the 2-D slice the two axes span, 4 MiB at 512^2 fp64):
//
//   phase A (axis a): HBM input -> Stockham -> scratch ring slot (L2)
//   phase B (axis b): scratch slot  -> Stockham -> final destination
//                     (HBM or peer exchange buffers, fused transpose)
//
// The scratch ring holds L planes (L * 4 MiB << 126 MB L2), so the
// intermediate never travels to DRAM: each plane costs one HBM read and one
// HBM write for two axes instead of two of each.  Work items (A or B tiles of
// a plane) are enumerated in rounds: round r = [A tiles of plane r][B tiles
// of plane r - lag]; CTA c takes items c, c + G, ...  Dependencies point to
// smaller item indices only (B(p) waits for all A(p) tiles, A(p) waits until
// every B(p - L) tile has pulled its slot), so with a co-resident persistent
// grid the pipeline cannot deadlock; prefetches never block (a prefetch whose
// dependency is not ready is issued when the item becomes current).
#pragma once

#include "fft_pass_tma.cuh"

namespace dfftb {

struct Fused2Args {
  int P;             // planes
  int T;             // tiles per plane per phase
  int L;             // scratch ring slots
  int lag;           // rounds between A(p) and B(p)
  int rows;          // TMA box rows (strided phase)
  int i_dim;         // tensor-map dimension of the lane index (strided phase)
  int lane_bytes;    // contiguous phase: bytes per stored lane (row stride)
  unsigned int* doneA;  // [P] A tiles stored per plane
  unsigned int* doneB;  // [P] B tiles that pulled their scratch data
  int nodeps;           // timing experiment only: skip dependency waits (wrong results)
  void* ring;           // host side: the ring, for the L2 access-policy window
  size_t persist_bytes; // host side: persisting window bytes (0: none)
};

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// FWD: phase A = contiguous rows (axis 2), phase B = strided columns (axis 1).
// !FWD: phase A = strided columns (axis 1), phase B = contiguous rows (axis 2).
template <typename T, int N, int EPREF, int W, bool FWD>
__global__ void __launch_bounds__(W* Sched<N, EPREF>::TPL, 1)
    fft_fused2_kernel(const __grid_constant__ PassParams pa, const __grid_constant__ PassParams pb,
                      const __grid_constant__ CUtensorMap tm, const Fused2Args fa) {
  using C = Cpx<T>;
  using SC = Sched<N, EPREF>;
  using TL = TmaLayout<T, N, W>;
  constexpr int STAGES = 2;
  constexpr int TPL = SC::TPL;
  constexpr int LS = lane_stride<C>(N);
  constexpr int LK = FWD ? kC2CFwd : kC2CBwd;
  extern __shared__ __align__(1024) unsigned char smem_f2[];
  unsigned char* stg = smem_f2;
  C* xch = reinterpret_cast<C*>(smem_f2 + STAGES * TL::STG);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_f2 + STAGES * TL::STG + TL::XCH);
  void** sptr = reinterpret_cast<void**>(bars + STAGES);

  const int tid = threadIdx.x;
  const C* tw = reinterpret_cast<const C*>(pa.tw);
  const int T2 = 2 * fa.T;
  const int64_t nitems = (int64_t)(fa.P + fa.lag) * T2;

  // item -> (phase, plane, tile); returns false for the empty edge slots
  auto decode = [&](int64_t i, bool& isA, int& plane, int& tile) {
    const int r = (int)(i / T2);
    const int q = (int)(i - (int64_t)r * T2);
    isA = q < fa.T;
    tile = isA ? q : q - fa.T;
    plane = isA ? r : r - fa.lag;
    return isA ? r < fa.P : r >= fa.lag;
  };
  auto next_valid = [&](int64_t i) {
    bool a;
    int p, t;
    while (i < nitems && !decode(i, a, p, t)) i += gridDim.x;
    return i;
  };
  auto deps_ready = [&](bool isA, int plane) -> bool {
    if (fa.nodeps) return true;
    if (isA) return plane < fa.L || ld_acquire_u32(fa.doneB + plane - fa.L) >= (unsigned)fa.T;
    return ld_acquire_u32(fa.doneA + plane) >= (unsigned)fa.T;
  };
  // thread 0 only
  auto issue = [&](int64_t i, int s) {
    bool isA;
    int plane, tile;
    decode(i, isA, plane, tile);
    const bool adj = isA != FWD;  // strided phase
    const PassParams& p = isA ? pa : pb;
    const int alpha = isA ? plane : plane % fa.L;  // scratch phases address ring slots
    const int beta0 = tile * W;
    unsigned char* dst = stg + s * TL::STG;
    asm volatile("fence.proxy.async.global;" ::: "memory");
    if (adj) {
      mbar_expect_tx(&bars[s], (uint32_t)(W * N * sizeof(C)));
      for (int r0 = 0; r0 < N; r0 += fa.rows) {
        const int c1 = fa.i_dim == 1 ? r0 : alpha;
        const int c2 = fa.i_dim == 1 ? alpha : r0;
        tma_load_3d(dst + (size_t)r0 * W * sizeof(C), &tm, 2 * beta0, c1, c2, &bars[s]);
      }
    } else {
      const int nvalid = min(W, p.B - beta0);
      const uint32_t bytes = (uint32_t)nvalid * (uint32_t)fa.lane_bytes;
      mbar_expect_tx(&bars[s], bytes);
      const unsigned char* src = reinterpret_cast<const unsigned char*>(p.in) +
                                 ((int64_t)alpha * p.in_sa + (int64_t)beta0 * p.in_sb) * (int64_t)sizeof(C);
      bulk_load(dst, src, bytes, &bars[s]);
    }
  };

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < kMaxDest) sptr[tid] = pb.dest[tid].ptr;
  __syncthreads();

  // s_pending[s]: the item of slot s has not been issued yet (its dependency
  // was not ready at prefetch time); written by thread 0, read by all after a
  // barrier
  __shared__ int s_pending[STAGES];
  if (tid == 0) {
    int64_t i = next_valid(blockIdx.x);
    for (int s = 0; s < STAGES; ++s) {
      s_pending[s] = 0;
      if (i >= nitems) continue;
      bool a;
      int p, t;
      decode(i, a, p, t);
      s_pending[s] = !deps_ready(a, p);
      if (!s_pending[s]) issue(i, s);
      i = next_valid(i + gridDim.x);
    }
  }
  __syncthreads();

  // A tiles are published one iteration late, so the fence before the
  // counter bump finds the tile's stores already drained
  int unpublished = -1;
  auto publish = [&]() {
    if (!fa.nodeps) __threadfence();
    __syncthreads();
    if (tid == 0) atomicAdd(fa.doneA + unpublished, 1u);
    unpublished = -1;
  };

  int k = 0;
  for (int64_t i = next_valid(blockIdx.x); i < nitems; i = next_valid(i + gridDim.x), ++k) {
    const int s = k % STAGES;
    bool isA;
    int plane, tile;
    decode(i, isA, plane, tile);
    if (s_pending[s]) {
      // deferred prefetch: publish our own finished tile first (the wait may
      // be on it), then wait for the dependency (an earlier item) and issue
      if (unpublished >= 0) publish();
      if (tid == 0) {
        while (!deps_ready(isA, plane)) __nanosleep(64);
        issue(i, s);
      }
    }
    mbar_wait(&bars[s], (uint32_t)((k / STAGES) & 1));
    const bool adj = isA != FWD;
    const int w = adj ? tid % W : tid / TPL;
    const int j = adj ? tid / W : tid % TPL;
    const PassParams& p = isA ? pa : pb;
    const int beta = tile * W + w;
    const unsigned char* st = stg + s * TL::STG;
    C v[SC::E];
    if (adj) {
      const C* scp = reinterpret_cast<const C*>(st);
      fetch0_lk<T, N, EPREF, LK>(v, j, [&](int pos) { return scp[pos * W + w]; },
                                 [&](int) { return T(0); });
    } else {
      const C* scp = reinterpret_cast<const C*>(st) + w * (fa.lane_bytes / (int)sizeof(C));
      fetch0_lk<T, N, EPREF, LK>(v, j, [&](int pos) { return scp[pos]; }, [&](int) { return T(0); });
    }
    if (unpublished >= 0) {
      publish();  // includes the barrier that retires slot s
    } else {
      __syncthreads();  // slot s consumed
    }
    if (tid == 0) {
      if (!isA) atomicAdd(fa.doneB + plane, 1u);  // this tile pulled its ring data
      const int64_t i2 = next_valid(next_valid(i + gridDim.x) + gridDim.x);
      s_pending[s] = 0;
      if (i2 < nitems) {
        bool a2;
        int p2, t2;
        decode(i2, a2, p2, t2);
        s_pending[s] = !deps_ready(a2, p2);
        if (!s_pending[s]) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(i2, s);
        }
      }
    }
    run_stages<T, N, EPREF, 0>(v, xch + w * LS, tw, j);  // its barriers publish s_pending
    if (beta < p.B) {
      const int alpha_store = isA ? plane % fa.L : plane;
      store_lk<T, N, EPREF, LK>(p, sptr, v, j, alpha_store, beta, static_cast<T>(p.scale));
    }
    if (isA) unpublished = plane;
  }
  if (unpublished >= 0) publish();
}

}  // namespace dfftb
