// dfftb executor: contexts (make_context, plan.hpp:359-390), lowering of a
// plan to fused GPU passes + group barriers, and execute (plan.hpp:463-535).
//
// Lowering.  The reference runs, per rank, LocalFftStage -> TransposeStage
// (pack, all_to_all, unpack; exchange.hpp:547-590) [-> LocalTransposeStage]
// ... -> NormalizeStage.  Here every FFT stage becomes ONE kernel launch
// whose store epilogue writes each output element to its final address in
// the stage's target layout:
//   FFT followed by a transpose  -> peer exchange buffers of the grid-axis
//                                   group (NVLink stores), then a barrier
//   FFT followed by Normalize    -> user output, scaled by 1/N
//   last FFT                     -> user output
//   FFT followed by a local FFT  -> private work buffer
// so each axis costs one read + one write of the local block.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <complex>
#include <cmath>
#include <cstring>
#include <vector>

#include "exec.hpp"
#include "kernels.hpp"

namespace dfftb {

#define CUDA_TRY(x)                                                              \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess)                                                       \
      raise(DFFTB_CudaError, std::string(#x) + ": " + cudaGetErrorString(e_));    \
  } while (0)

static constexpr uint64_t kHandleMagic = 0x64666674625f3031ull;  // "dfftb_01"
static constexpr size_t kFlagsBytes = 4096;
static constexpr unsigned long long kBarrierTimeoutNs = 60ull * 1000 * 1000 * 1000;

void* Ctx::exch(int r, int slot, int parity) const {
  if (slot < 0 || slot >= exch_slots) raise(DFFTB_ArenaExhausted, "exchange slot out of range");
  char* base = static_cast<char*>(peer_region[r]);
  return base + flags_bytes + (size_t)(2 * slot + parity) * exch_bytes;
}

uint64_t* Ctx::flags_of(int r) const { return static_cast<uint64_t*>(peer_region[r]); }

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Internal (exchange / work) buffers keep the reference's axis order but pad
// the innermost extent so every row starts on a 16-byte boundary (fp32
// complex rows of odd length, e.g. the 129-bin R2C axis), which lets the TMA
// path describe them.  User-visible buffers are never padded.
static int64_t inner_pad(int64_t len, int prec) { return prec == 4 ? (len + 1) & ~int64_t(1) : len; }

static int64_t max_internal_count(const Dist& d, int prec) {
  int64_t m = 0;
  if (d.ndim() == 0) return 0;  // unused side of a LocalTranspose stage
  for (int r = 0; r < d.nranks(); ++r) {
    int64_t off[kMaxDims], len[kMaxDims];
    d.extents_of(r, off, len);
    int64_t n = inner_pad(len[d.ndim() - 1], prec);
    for (int a = 0; a + 1 < d.ndim(); ++a) n *= len[a];
    m = std::max(m, n);
  }
  return m;
}

// Bytes of the largest complex block any rank holds in any layout of the
// plan family (forward and backward of the same geometry), so one context
// serves execute(bwd, execute(fwd, x, ctx), ctx) as in test_plan.cpp:116-133.
static size_t family_bytes(const Plan& plan) {
  dfftb_plan_options o = plan.options;
  const int kf = plan.kind == DFFTB_C2C ? DFFTB_C2C : DFFTB_R2C;
  const int kb = plan.kind == DFFTB_C2C ? DFFTB_C2C : DFFTB_C2R;
  int64_t m = 1;
  for (int d = 0; d < 2; ++d) {
    Plan p = build_plan(plan.dims, plan.decomp, plan.grid, d == 0 ? kf : kb, d, plan.prec, o);
    for (const auto& st : p.stages) {
      if (st.type == StageType::Normalize) continue;
      m = std::max(m, max_internal_count(st.before, plan.prec));
      m = std::max(m, max_internal_count(st.after, plan.prec));
    }
  }
  return (size_t)m * 2 * plan.prec;
}

// Exchange slots a program of the plan family uses: one per transpose stage
// (pencil 2, slab 1, 4-D general 3), at least the 2 the single-rank
// backward lowering uses.
static int family_exch_slots(const Plan& plan) {
  dfftb_plan_options o = plan.options;
  const int kf = plan.kind == DFFTB_C2C ? DFFTB_C2C : DFFTB_R2C;
  const int kb = plan.kind == DFFTB_C2C ? DFFTB_C2C : DFFTB_C2R;
  int m = 2;
  for (int d = 0; d < 2; ++d) {
    Plan p = build_plan(plan.dims, plan.decomp, plan.grid, d == 0 ? kf : kb, d, plan.prec, o);
    int t = 0;
    for (const auto& st : p.stages) t += st.type == StageType::Transpose;
    m = std::max(m, t);
  }
  return m;
}

static bool is_pow2(int64_t n) { return n >= 1 && (n & (n - 1)) == 0; }

static int64_t largest_prime_factor(int64_t n) {
  int64_t lpf = 1;
  for (int64_t p = 2; p * p <= n; ++p)
    while (n % p == 0) {
      lpf = p;
      n /= p;
    }
  return n > 1 ? std::max(lpf, n) : lpf;
}

// Kernel1d path choice (kernels.hpp:227-243): pow-2 -> Stockham pass,
// 13-smooth -> mixed radix, else Bluestein with m = bit_ceil(2n - 1)
static bool is_smooth(int64_t n) { return largest_prime_factor(n) <= 13; }
static int64_t bluestein_m(int64_t n) {
  int64_t m = 1;
  while (m < 2 * n - 1) m <<= 1;
  return m;
}

static std::vector<int> radix_list(int64_t L) {
  std::vector<int> r;
  while (L % 8 == 0) { r.push_back(8); L /= 8; }
  while (L % 4 == 0) { r.push_back(4); L /= 4; }
  while (L % 2 == 0) { r.push_back(2); L /= 2; }
  for (int p : {3, 5, 7, 11, 13})
    while (L % p == 0) { r.push_back(p); L /= p; }
  return r;
}

static void check_lengths(const Plan& plan) {
  if (plan.dims.size() < 2 || plan.dims.size() > 4)
    raise(DFFTB_Unsupported, "the B200 path executes 2-D, 3-D and 4-D transforms");
  for (auto n : plan.dims) {
    bool ok = n >= 1 && n <= 4096;
    if (ok && !is_pow2(n) && !is_smooth(n)) ok = bluestein_m(n) <= (plan.prec == 8 ? 4096 : 8192);
    if (!ok)
      raise(DFFTB_Unsupported, "axis length " + std::to_string(n) +
                                   " not supported on the B200 path (<= 4096; Bluestein <= " +
                                   std::to_string(plan.prec == 8 ? 2048 : 4096) + ")");
  }
  for (int g : plan.grid)
    if (g > kMaxDest) raise(DFFTB_Unsupported, "grid factors above 8 are not supported");
}

// host FFT (recursive radix-2, double) for the Bluestein kernel spectrum
static void host_fft(std::vector<std::complex<double>>& a) {
  const size_t n = a.size();
  if (n <= 1) return;
  std::vector<std::complex<double>> e(n / 2), o(n / 2);
  for (size_t i = 0; i < n / 2; ++i) {
    e[i] = a[2 * i];
    o[i] = a[2 * i + 1];
  }
  host_fft(e);
  host_fft(o);
  for (size_t k = 0; k < n / 2; ++k) {
    const std::complex<double> t = std::polar(1.0, -2.0 * M_PI * (double)k / (double)n) * o[k];
    a[k] = e[k] + t;
    a[k + n / 2] = e[k] - t;
  }
}

// Bluestein tables for the forward direction (bluestein_context,
// kernels.hpp:179-216): chirp c_j = exp(-i pi (j^2 mod 2n) / n) and the
// kernel spectrum FFT_m(wrapped conj(c)) / m, in double, cast to T
static std::pair<void*, void*> bluestein_tables(int64_t n, int prec) {
  const int64_t m = bluestein_m(n);
  std::vector<std::complex<double>> chirp(n), b(m, 0.0);
  for (int64_t j = 0; j < n; ++j) {
    const uint64_t r = ((uint64_t)j * (uint64_t)j) % (uint64_t)(2 * n);
    chirp[j] = std::polar(1.0, -M_PI * (double)r / (double)n);
  }
  b[0] = std::conj(chirp[0]);
  for (int64_t j = 1; j < n; ++j) b[j] = b[m - j] = std::conj(chirp[j]);
  host_fft(b);
  for (auto& v : b) v /= (double)m;
  auto upload = [&](const std::vector<std::complex<double>>& v) {
    void* d = nullptr;
    if (prec == 8) {
      CUDA_TRY(cudaMalloc(&d, v.size() * 16));
      CUDA_TRY(cudaMemcpy(d, v.data(), v.size() * 16, cudaMemcpyHostToDevice));
    } else {
      std::vector<float> f(2 * v.size());
      for (size_t i = 0; i < v.size(); ++i) {
        f[2 * i] = (float)v[i].real();
        f[2 * i + 1] = (float)v[i].imag();
      }
      CUDA_TRY(cudaMalloc(&d, f.size() * 4));
      CUDA_TRY(cudaMemcpy(d, f.data(), f.size() * 4, cudaMemcpyHostToDevice));
    }
    return d;
  };
  return {upload(chirp), upload(b)};
}

size_t workspace_bytes(const Plan& plan, int rank) {
  if (rank < 0 || rank >= plan.nranks()) raise(DFFTB_InvalidRank, "rank out of range");
  const size_t blk = (family_bytes(plan) + 255) / 256 * 256;
  return kFlagsBytes + 2 * (size_t)family_exch_slots(plan) * blk + blk + 8 * sizeof(unsigned long long);
}

Ctx* ctx_create(const Plan& plan, int rank, int device) {
  if (rank < 0 || rank >= plan.nranks()) raise(DFFTB_InvalidRank, "rank out of range");
  check_lengths(plan);
  DeviceGuard g(device);
  CUDA_TRY(cudaSetDevice(device));
  auto ctx = std::make_unique<Ctx>();
  ctx->rank = rank;
  ctx->nranks = plan.nranks();
  ctx->device = device;
  ctx->prec = plan.prec;
  ctx->dims = plan.dims;
  ctx->grid = plan.grid;
  ctx->decomp = plan.decomp;
  ctx->kind_family = plan.kind == DFFTB_C2C ? 0 : 1;
  const size_t blk = (family_bytes(plan) + 255) / 256 * 256;
  ctx->flags_bytes = kFlagsBytes;
  ctx->exch_bytes = blk;
  ctx->exch_slots = family_exch_slots(plan);
  ctx->region_bytes = kFlagsBytes + 2 * (size_t)ctx->exch_slots * blk;  // [slot][parity] buffers
  ctx->work_bytes = blk;
  CUDA_TRY(cudaMalloc(&ctx->region, ctx->region_bytes));
  CUDA_TRY(cudaMemset(ctx->region, 0, kFlagsBytes));
  CUDA_TRY(cudaMalloc(&ctx->work, ctx->work_bytes));
  CUDA_TRY(cudaMalloc(&ctx->dstat, 8 * sizeof(unsigned long long)));
  CUDA_TRY(cudaMemset(ctx->dstat, 0, 8 * sizeof(unsigned long long)));
  // twiddle tables w[m] = exp(-2 pi i m / n) in double, cast to T
  // (TwiddleTable, kernels.hpp:66-98); forward only: backward is conj(F(conj x))
  for (auto n64 : plan.dims) {
    const int n = (int)n64;
    if (!is_pow2(n) && !is_smooth(n) && !ctx->bluestein.count(n)) ctx->bluestein[n] = bluestein_tables(n, plan.prec);
    if (!is_pow2(n) || ctx->twiddles.count(n)) continue;
    std::vector<double> wd(2 * n);
    std::vector<float> wf(2 * n);
    for (int m = 0; m < n; ++m) {
      const double a = -2.0 * M_PI * (double)m / (double)n;
      wd[2 * m] = std::cos(a);
      wd[2 * m + 1] = std::sin(a);
      wf[2 * m] = (float)wd[2 * m];
      wf[2 * m + 1] = (float)wd[2 * m + 1];
    }
    void* d = nullptr;
    CUDA_TRY(cudaMalloc(&d, 2 * n * plan.prec));
    CUDA_TRY(cudaMemcpy(d, plan.prec == 8 ? (void*)wd.data() : (void*)wf.data(), 2 * n * plan.prec,
                        cudaMemcpyHostToDevice));
    ctx->twiddles[n] = d;
  }
  // L2-resident plane ring for the fused two-axis pass (slab plans and
  // pencil grids whose second grid factor is 1: the row exchange is local)
  {
    // experimental, opt-in (DFFTB_FUSE=1): measured 5.8 ms vs 4.76 ms for the
    // two plain passes at 512^3 (round 1) -- the pipeline is latency-bound
    const char* on = getenv("DFFTB_FUSE");
    const bool fusable_grid = plan.decomp == DFFTB_SLAB || (plan.grid.size() == 2 && plan.grid[1] == 1);
    if ((on && *on == '1') && fusable_grid && plan.dims.size() == 3 && plan.dims[1] == plan.dims[2] &&
        fused2_supported(plan.prec, (int)plan.dims[1])) {
      const char* le = getenv("DFFTB_FUSE_L");
      const int L = le ? std::max(2, atoi(le)) : 8;
      ctx->fuse_planes = (int)plan.dims[0];
      ctx->fuse_ring_bytes = (size_t)L * plan.dims[1] * plan.dims[2] * 2 * plan.prec;
      CUDA_TRY(cudaMalloc(&ctx->fuse_ring, ctx->fuse_ring_bytes));
      CUDA_TRY(cudaMalloc(&ctx->fuse_counters, 2 * sizeof(unsigned int) * ctx->fuse_planes));
      // reserve persisting L2 for the ring so its dirty lines are overwritten
      // in L2 instead of being written back (DFFTB_FUSE_PERSIST=0 disables)
      const char* pe = getenv("DFFTB_FUSE_PERSIST");
      if (!(pe && *pe == '0')) {
        int maxp = 0;
        cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, device);
        const size_t want = std::min<size_t>((size_t)maxp, ctx->fuse_ring_bytes);
        if (want > 0 && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) == cudaSuccess)
          ctx->fuse_persist_bytes = want;
        cudaGetLastError();
      }
    }
  }
  ctx->peer_region.assign(ctx->nranks, nullptr);
  ctx->peer_opened.assign(ctx->nranks, false);
  ctx->peer_region[rank] = ctx->region;
  if (ctx->nranks == 1) ctx->connected = true;
  return ctx.release();
}

void ctx_export(const Ctx& ctx, CtxHandle* h) {
  std::memset(h, 0, sizeof(*h));
  DeviceGuard g(ctx.device);
  cudaIpcMemHandle_t ih;
  CUDA_TRY(cudaIpcGetMemHandle(&ih, ctx.region));
  std::memcpy(h->ipc, &ih, sizeof(ih));
  h->pid = (int64_t)getpid();
  h->device = ctx.device;
  h->dptr = (uint64_t)(uintptr_t)ctx.region;
  h->bytes = ctx.region_bytes;
  h->magic = kHandleMagic;
}

void ctx_connect(Ctx& ctx, const CtxHandle* handles) {
  DeviceGuard g(ctx.device);
  for (int r = 0; r < ctx.nranks; ++r) {
    const CtxHandle& h = handles[r];
    if (h.magic != kHandleMagic) raise(DFFTB_BadMagic, "context handle has a bad magic");
    if (h.bytes != ctx.region_bytes) raise(DFFTB_CountMismatch, "peer context sizes differ");
    if (r == ctx.rank) continue;
    if (h.pid == (int64_t)getpid()) {
      // same process (thread-per-GPU world): direct peer pointer
      if (h.device != ctx.device) {
        int can = 0;
        CUDA_TRY(cudaDeviceCanAccessPeer(&can, ctx.device, (int)h.device));
        if (!can) raise(DFFTB_Unsupported, "no peer access between devices");
        cudaError_t e = cudaDeviceEnablePeerAccess((int)h.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
          raise(DFFTB_CudaError, cudaGetErrorString(e));
        cudaGetLastError();
      }
      ctx.peer_region[r] = (void*)(uintptr_t)h.dptr;
    } else {
      cudaIpcMemHandle_t ih;
      std::memcpy(&ih, h.ipc, sizeof(ih));
      void* p = nullptr;
      CUDA_TRY(cudaIpcOpenMemHandle(&p, ih, cudaIpcMemLazyEnablePeerAccess));
      ctx.peer_region[r] = p;
      ctx.peer_opened[r] = true;
    }
  }
  ctx.connected = true;
}

void ctx_destroy(Ctx* ctx) {
  if (!ctx) return;
  {
    DeviceGuard g(ctx->device);
    cudaDeviceSynchronize();
    for (int r = 0; r < ctx->nranks; ++r)
      if (ctx->peer_opened[r]) cudaIpcCloseMemHandle(ctx->peer_region[r]);
    for (auto& kv : ctx->twiddles) cudaFree(kv.second);
    for (auto& kv : ctx->bluestein) {
      cudaFree(kv.second.first);
      cudaFree(kv.second.second);
    }
    cudaFree(ctx->region);
    cudaFree(ctx->work);
    cudaFree(ctx->dstat);
    if (ctx->fuse_ring) cudaFree(ctx->fuse_ring);
    if (ctx->ring) cudaFree(ctx->ring);
    if (ctx->ring_ctr) cudaFree(ctx->ring_ctr);
    if (ctx->fuse_counters) cudaFree(ctx->fuse_counters);
    cudaGetLastError();
  }
  delete ctx;
}

void world_create(const Plan& plan, int device, Ctx** out) {
  const int P = plan.nranks();
  std::vector<Ctx*> ctxs(P, nullptr);
  try {
    for (int r = 0; r < P; ++r) ctxs[r] = ctx_create(plan, r, device);
  } catch (...) {
    for (auto* c : ctxs) ctx_destroy(c);
    throw;
  }
  for (int r = 0; r < P; ++r) {
    for (int q = 0; q < P; ++q) ctxs[r]->peer_region[q] = ctxs[q]->region;
    ctxs[r]->world_mode = true;
    ctxs[r]->connected = true;
    out[r] = ctxs[r];
  }
}

// ---------------------------------------------------------------- lowering

struct Op {
  bool barrier = false;
  bool tma = false;
  bool generic = false;  // non-power-of-two length: mixed-radix / Bluestein kernel
  bool fused2 = false;   // two axes in one L2-resident plane pipeline (pb, fa below)
  bool fwd2 = true;
  PassParams pb{};
  Fused2Args fa{};
  GenParams g{};
  TmaPlan tp{};
  PassParams p{};
  int n = 1;
  bool adj = false;
  bool fused = false;
  int grid_axis = 0;
  std::vector<int> members;
  // lane geometry (for pipelining): transform axis, lane axes, input layout
  int v = -1, ax_a = -1, ax_b = -1, ax_a1 = -1;
  const Dist* before = nullptr;
  // pipelined pair: this op's pass (p, tp, adj) is the producer, (pb, tpb,
  // adj_b) the consumer, on disjoint CTAs of one launch
  bool pipe = false;
  bool adj_b = false;
  TmaPlan tpb{};
  PipeArgs ppa{}, ppb{};
  double frac = 0.5;
  bool ring_reset = false;  // zero the ring counters before the launch
};

// Row-major element strides of a block; internal buffers pad the innermost
// extent (inner_pad).
static void row_major_strides(const int64_t* len, int nd, int64_t* st, bool internal = false,
                              int prec = 8, bool swap01 = false) {
  // storage order: axes 0,1,2,... outermost first; swap01 stores axis 1
  // outside axis 0 (the [x1][x0][rest] order of the reference's transposed
  // pack, exchange.hpp:486-511) so the axis-0 pass reads short strides
  int order[kMaxDims];
  for (int a = 0; a < nd; ++a) order[a] = a;
  if (swap01 && nd >= 3) {
    order[0] = 1;
    order[1] = 0;
  }
  int64_t s = 1;
  for (int idx = nd - 1; idx >= 0; --idx) {
    const int a = order[idx];
    st[a] = s;
    s *= (idx == nd - 1 && internal) ? inner_pad(len[a], prec) : len[a];
  }
}

static bool zperm_enabled() {
  const char* e = getenv("DFFTB_ZPERM");
  return !(e && *e == '0');
}

static std::vector<int> group_members(const Dist& d, int me, int g) {
  auto c = d.coords_of(me);
  std::vector<int> m(d.grid[g]);
  for (int q = 0; q < d.grid[g]; ++q) {
    auto cq = c;
    cq[g] = q;
    m[q] = d.rank_of(cq);
  }
  return m;
}

static void check_compatible(const Plan& plan, const Ctx& ctx) {
  if (plan.nranks() != ctx.nranks) raise(DFFTB_GridMismatch, "communicator size must match the grid");
  if (plan.dims != ctx.dims || plan.grid != ctx.grid || plan.prec != ctx.prec ||
      plan.decomp != ctx.decomp)
    raise(DFFTB_GridMismatch, "context was made for a different plan geometry");
  if (!ctx.connected) raise(DFFTB_ConfigInvalid, "context is not connected to its peers");
  if (family_bytes(plan) > ctx.exch_bytes)
    raise(DFFTB_ArenaExhausted, "context buffers are too small for this plan");
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

// L2 sector promotion of the strided-lane tensor maps (A/B aid:
// DFFTB_L2PROMO = 0 none, 1 64 B, 2 128 B, 3 256 B (default))
static CUtensorMapL2promotion l2_promotion() {
  const char* e = getenv("DFFTB_L2PROMO");
  const int v = e ? atoi(e) : 3;
  switch (v) {
    case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    case 1: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 2: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
}

static bool tma_disabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DFFTB_NO_TMA");
    v = (e && *e && *e != '0') ? 1 : 0;
  }
  return v == 1;
}

// Decide whether a pass can use the TMA-prefetch kernel and build its
// descriptor: a 3-D tensor map over (beta as reals, i, alpha) for strided
// lanes, or a flat bulk copy of W adjacent lanes for contiguous ones.
static bool plan_tma(Op& op, int prec) {
  const PassParams& p = op.p;
  const int n = op.n;
  if (tma_disabled() || n < 8 || (int64_t)p.A * p.B == 0) return false;
  {
    // debug aid: DFFTB_TMA_LK_MASK restricts the TMA path to some lane kinds
    const char* m = getenv("DFFTB_TMA_LK_MASK");
    const int lk = p.in_mode == kInReal ? kR2C
                   : p.in_mode == kInHermitian ? kC2R
                   : (p.inverse ? kC2CBwd : kC2CFwd);
    if (m && *m && !((atoi(m) >> lk) & 1)) return false;
  }
  const int W = tma_tile_w(prec, n);
  if (W <= 0) return false;
  const int csize = 2 * prec;
  if ((reinterpret_cast<uintptr_t>(p.in) & 15) != 0) return false;
  TmaPlan& tp = op.tp;
  std::memset(&tp, 0, sizeof(tp));
  tp.args.ntiles = (int64_t)p.A * (p.A1 > 1 ? p.A1 : 1) * ((p.B + W - 1) / W);
  if (p.A1 > 1 && (p.in_sa1 * (p.in_mode == kInReal ? prec : csize)) % 16) return false;
  if (op.adj) {
    if (p.in_mode != kInComplex) return false;
    if (p.A1 > 1) return false;  // 4-D strided lanes: direct kernel (3-D tensor map only)
    if ((2 * W * prec) % 16 != 0 || 2 * W > 256) return false;
    const int64_t si = p.in_si * csize, sa = (p.A > 1 ? p.in_sa : (int64_t)n * p.in_si) * csize;
    if (p.in_sb != 1) return false;
    if (si % 16 || sa % 16) {
      // rows a tensor map cannot describe (fp32 C2R user blocks: 129-bin
      // rows of 1032 bytes): per-thread 8-byte cp.async into the same tile
      if (csize != 8 || (reinterpret_cast<uintptr_t>(p.in) & 7)) return false;
      const char* e = getenv("DFFTB_UNALIGNED_LDGSTS");
      if (e && *e == '0') return false;
      tp.args.bulk = 0;
      tp.args.ldgsts = 1;
      return true;
    }
    tp.args.bulk = 0;
    {
      // row loader: TMA boxes (default; measured faster even for 4-16 MB row
      // strides) or per-thread cp.async (DFFTB_ADJ_LOADER=ldgsts|auto)
      const char* e = getenv("DFFTB_ADJ_LOADER");
      const std::string mode = e ? e : "tma";
      // (16-byte cp.async per element: fp64 complex only)
      tp.args.ldgsts = csize == 16 && (mode == "ldgsts" || (mode == "auto" && si >= (int64_t(1) << 20)));
      if (tp.args.ldgsts) return true;
    }
    auto enc = tensor_map_encoder();
    if (!enc) return false;
    const int rows = n < 256 ? n : 256;
    cuuint64_t gdim[3];
    cuuint64_t gstride[2];
    cuuint32_t box[3], estr[3] = {1, 1, 1};
    gdim[0] = 2 * (cuuint64_t)p.B;
    box[0] = 2 * W;
    if (si <= sa) {
      tp.args.i_dim = 1;
      gdim[1] = n;
      gdim[2] = p.A;
      gstride[0] = si;
      gstride[1] = sa;
      box[1] = rows;
      box[2] = 1;
    } else {
      tp.args.i_dim = 2;
      gdim[1] = p.A;
      gdim[2] = n;
      gstride[0] = sa;
      gstride[1] = si;
      box[1] = 1;
      box[2] = rows;
    }
    CUresult r = enc(&tp.tmap, prec == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                     3, const_cast<void*>(p.in), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, l2_promotion(),
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    tp.args.rows = rows;
    tp.args.bulk = 0;
    return true;
  }
  const int64_t lane_elems = p.in_mode == kInHermitian ? n / 2 + 1 : n;
  const int esize = p.in_mode == kInReal ? prec : csize;
  // lanes are adjacent rows (row stride in_sb >= lane length: internal
  // buffers pad odd fp32 rows); W rows go in one bulk copy, padding included
  const int64_t lane_bytes = p.in_sb * esize;
  if (p.in_sb < lane_elems || p.in_sb > n || lane_bytes % 16) return false;
  if (p.A > 1 && (p.in_sa * esize) % 16) return false;
  tp.args.bulk = 1;
  tp.args.lane_bytes = (int)lane_bytes;
  return true;
}

// Cheapest store addressing the destination table allows: one destination,
// or equal power-of-two blocks with identical strides (q = k >> shift).
static void set_store_mode(PassParams& p) {
  p.store_mode = 2;
  p.oshift = 0;
  p.omask = 0;
  if (p.ndest == 1) {
    if (p.dest[0].sk < (1ll << 31)) p.store_mode = 0;
    return;
  }
  const int64_t b = p.oblk;
  if ((b & (b - 1)) != 0 || p.dest[0].sk >= (1ll << 31)) return;
  for (int q = 1; q < p.ndest; ++q) {
    const Dest& d = p.dest[q];
    if (d.base != p.dest[0].base || d.sa != p.dest[0].sa || d.sb != p.dest[0].sb || d.sk != p.dest[0].sk)
      return;
  }
  p.store_mode = 1;
  p.oshift = ilog2((int)b);
  p.omask = (int)b - 1;
}

// Non-power-of-two lengths run the generic mixed-radix / Bluestein kernel
static void plan_generic(Op& op, const Ctx& ctx) {
  if (is_pow2(op.n)) return;
  op.tma = false;
  op.generic = true;
  GenParams& g = op.g;
  std::memset(&g, 0, sizeof(g));
  g.p = op.p;
  g.n = op.n;
  g.bluestein = !is_smooth(op.n);
  g.L = g.bluestein ? (int)bluestein_m(op.n) : op.n;
  const auto rl = radix_list(g.L);
  g.nrad = (int)rl.size();
  for (int i = 0; i < g.nrad; ++i) g.rad[i] = rl[i];
  const int64_t csize = 2 * ctx.prec;
  g.W = (int)std::max<int64_t>(1, std::min<int64_t>(64, 65536 / (g.L * csize)));
  if (g.bluestein) {
    g.chirp = ctx.bluestein.at(op.n).first;
    g.kfft = ctx.bluestein.at(op.n).second;
  }
  // the generic store maps (lane, k) by dest contiguity; one dest or general
  g.p.store_mode = 2;
}

// Merge "rows then columns" (forward) / "columns then rows" (backward) pass
// pairs whose intermediate stays on this rank into one fused2 op: the
// intermediate goes through the L2-resident plane ring instead of HBM.
static void fuse_pairs(std::vector<Op>& prog, const Ctx& ctx) {
  if (!ctx.fuse_ring) return;
  const int prec = ctx.prec;
  const int64_t csize = 2 * prec;
  for (size_t i = 0; i + 1 < prog.size(); ++i) {
    Op& a = prog[i];
    const Op& b = prog[i + 1];
    if (a.barrier || b.barrier || a.generic || b.generic || a.fused2) continue;
    const PassParams& pa = a.p;
    const PassParams& pb = b.p;
    if (pa.in_mode != kInComplex || pb.in_mode != kInComplex || pa.out_real || pb.out_real) continue;
    if (a.n != b.n || !fused2_supported(prec, a.n) || pa.ndest != 1) continue;
    if (pa.dest[0].ptr != pb.in || pa.A != pb.A || pa.B != pb.B || pa.inverse != pb.inverse) continue;
    if (pa.A1 > 1 || pb.A1 > 1) continue;
    const bool fwd = !pa.inverse;
    if (fwd ? (a.adj || !b.adj) : (!a.adj || b.adj)) continue;
    if (!a.tma || (fwd ? !a.tp.args.bulk : (a.tp.args.bulk || a.tp.args.ldgsts))) continue;
    const int n = a.n;
    const int W = tma_tile_w(prec, n);
    const int64_t plane = (int64_t)n * n;
    const char* le = getenv("DFFTB_FUSE_L");
    const char* lg = getenv("DFFTB_FUSE_LAG");
    const int L = le ? std::max(2, atoi(le)) : 8;
    const int lag = lg ? std::max(1, std::min(L - 1, atoi(lg))) : L / 2;
    if ((size_t)(L * plane * csize) > ctx.fuse_ring_bytes || pa.A > ctx.fuse_planes) continue;
    // small problems: the plane pipeline's dependency latency outweighs the
    // saved round trip; keep the two plain passes
    if (pa.A < 2 * L || (int64_t)pa.A * ((pa.B + W - 1) / W) < 4 * 148) continue;

    Op f = a;
    f.fused2 = true;
    f.fwd2 = fwd;
    // phase A: stores into ring slot (plane % L), scratch plane layout [x1][x2]
    Dest& d = f.p.dest[0];
    d.ptr = ctx.fuse_ring;
    d.base = 0;
    d.sa = plane;
    d.sb = fwd ? n : 1;
    d.sk = fwd ? 1 : n;
    f.p.store_mode = 0;
    f.p.oblk = n;
    // phase B: reads the ring slot
    f.pb = pb;
    f.pb.in = ctx.fuse_ring;
    f.pb.in_sa = plane;
    f.pb.in_sb = fwd ? 1 : n;
    f.pb.in_si = fwd ? n : 1;
    Fused2Args& fa = f.fa;
    std::memset(&fa, 0, sizeof(fa));
    fa.P = pa.A;
    fa.T = (pa.B + W - 1) / W;
    fa.L = L;
    fa.lag = lag;
    fa.doneA = ctx.fuse_counters;
    fa.doneB = ctx.fuse_counters + ctx.fuse_planes;
    fa.ring = ctx.fuse_ring;
    fa.persist_bytes = ctx.fuse_persist_bytes;
    {
      const char* nd = getenv("DFFTB_FUSE_NODEP");
      fa.nodeps = nd && *nd == '1';
    }
    if (fwd) {
      // contiguous phase A from the input rows, strided phase B from the ring
      fa.lane_bytes = a.tp.args.lane_bytes;
      auto enc = tensor_map_encoder();
      if (!enc) continue;
      const int rows = n < 256 ? n : 256;
      cuuint64_t gdim[3] = {2 * (cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)L};
      cuuint64_t gstride[2] = {(cuuint64_t)(n * csize), (cuuint64_t)(plane * csize)};
      cuuint32_t box[3] = {(cuuint32_t)(2 * W), (cuuint32_t)rows, 1}, estr[3] = {1, 1, 1};
      if (enc(&f.tp.tmap, prec == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
              ctx.fuse_ring, gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        continue;
      fa.rows = rows;
      fa.i_dim = 1;
    } else {
      // strided phase A from the input (its own tensor map), contiguous B from the ring
      fa.rows = a.tp.args.rows;
      fa.i_dim = a.tp.args.i_dim;
      fa.lane_bytes = (int)(n * csize);
    }
    prog[i] = f;
    prog.erase(prog.begin() + i + 1);
  }
}

// One local pass of a 3-D block: axis v of the buffer `in` (extents len,
// element strides si) into `out` (strides so over the output extents).
static Op single_pass(const Ctx& ctx, int v, int n, const int64_t* len, const int64_t* si,
                      const void* in, void* out, const int64_t* so, int fkind, double scale) {
  int lanes[2], nl = 0;
  for (int a = 0; a < 3; ++a)
    if (a != v) lanes[nl++] = a;
  const int ax_a = lanes[0], ax_b = lanes[1];
  Op op;
  PassParams& p = op.p;
  p.in = in;
  p.A = (int)len[ax_a];
  p.A1 = 1;
  p.in_sa1 = 0;
  p.B = (int)len[ax_b];
  p.in_sa = si[ax_a];
  p.in_sb = si[ax_b];
  p.in_si = si[v];
  op.n = n;
  p.n_out = fkind == DFFTB_R2C ? n / 2 + 1 : n;
  p.in_mode = fkind == DFFTB_R2C ? kInReal : (fkind == DFFTB_C2R ? kInHermitian : kInComplex);
  p.out_real = fkind == DFFTB_C2R;
  p.inverse = true;
  p.scale = scale;
  p.tw = is_pow2(n) ? ctx.twiddles.at(n) : nullptr;
  p.herm = ctx.dstat;
  op.adj = p.in_si != 1;
  p.ndest = 1;
  p.oblk = p.n_out > 0 ? p.n_out : 1;
  Dest& d = p.dest[0];
  d.ptr = out;
  d.base = 0;
  d.sa = so[ax_a];
  d.sa1 = 0;
  d.sb = so[ax_b];
  d.sk = so[v];
  op.tma = false;
  set_store_mode(p);
  op.tma = plan_tma(op, ctx.prec);
  plan_generic(op, ctx);
  return op;
}

// Single-rank 3-D backward: every exchange is local, so the axis order is
// free (the transforms commute; results agree to rounding).  Run the axes as
// the forward does — contiguous lanes first, the [x1][x0][rest] buffer feeding
// the axis-0 pass, strided stores last — instead of the reference's F0;F1;F2
// order (plan.hpp:293-312), whose first pass would load axis-0 lanes of the
// user block at a whole-plane stride.  C2R keeps its Hermitian axis last.
static bool lower_single(const Plan& plan, const Ctx& ctx, const void* d_in, void* d_out, int parity,
                         std::vector<Op>& prog) {
  if (plan.nranks() != 1 || plan.input.ndim() != 3 || !zperm_enabled()) return false;
  {
    const char* e = getenv("DFFTB_SINGLE_REORDER");
    if (e && *e == '0') return false;
  }
  bool backward = false, c2r = false;
  double scale = 1.0;
  for (const auto& st : plan.stages) {
    if (st.type == StageType::Fft) {
      backward = st.dir == DFFTB_BACKWARD;
      if (st.fkind == DFFTB_C2R) c2r = true;
      if (st.fkind == DFFTB_R2C) return false;
    } else if (st.type == StageType::Normalize) {
      scale = st.factor;
    }
  }
  if (!backward) return false;
  int64_t off[3], lc[3], lr[3];
  plan.input.extents_of(0, off, lc);    // complex (Hermitian for C2R) extents
  plan.output.extents_of(0, off, lr);   // output extents
  for (int a = 0; a < 3; ++a)
    if (lc[a] <= 0) return false;
  const int prec = ctx.prec;
  void* b1 = ctx.exch(0, 0, parity);
  void* b2 = ctx.exch(0, 1, parity);
  int64_t s_user[3], s_plain[3], s_swap[3], s_out[3];
  row_major_strides(lc, 3, s_user, false, prec);
  row_major_strides(lc, 3, s_plain, true, prec);
  row_major_strides(lc, 3, s_swap, true, prec, true);
  row_major_strides(lr, 3, s_out, false, prec);
  if (!c2r) {
    prog.push_back(single_pass(ctx, 2, (int)lc[2], lc, s_user, d_in, b1, s_plain, DFFTB_C2C, 1.0));
    prog.push_back(single_pass(ctx, 1, (int)lc[1], lc, s_plain, b1, b2, s_swap, DFFTB_C2C, 1.0));
    prog.push_back(single_pass(ctx, 0, (int)lc[0], lc, s_swap, b2, d_out, s_out, DFFTB_C2C, scale));
  } else {
    prog.push_back(single_pass(ctx, 1, (int)lc[1], lc, s_user, d_in, b1, s_swap, DFFTB_C2C, 1.0));
    prog.push_back(single_pass(ctx, 0, (int)lc[0], lc, s_swap, b1, b2, s_plain, DFFTB_C2C, 1.0));
    prog.push_back(single_pass(ctx, 2, (int)lr[2], lc, s_plain, b2, d_out, s_out, DFFTB_C2R, scale));
  }
  return true;
}

// ------------------------------------------------------ pipelined pairs
//
// The reference overlaps communication with computation by chunking along
// the N0/P0 planes (pipelined_all_to_all, exchange.hpp:250-423).
// Here the two passes on either side of an exchange run concurrently on
// disjoint CTAs of one launch, chunked along the lane axis both share (the
// axis the exchange does not touch): while the NVLink-bound pass streams
// chunk c to the peers, the HBM-bound pass already transforms chunk c - 1.
// Per-chunk tile counters in every rank's flag page replace the group
// barrier between the two passes.
static constexpr int kPipeSlots = 8;
static constexpr size_t kPipeOffU64 = 256;  // counter slots start after the barrier flags

static bool pipe_candidate(const Op& o, int prec) {
  if (o.barrier || o.generic || o.fused2 || o.pipe || !o.tma || o.before == nullptr) return false;
  if (o.tp.args.ldgsts || o.p.A1 > 1 || o.p.A <= 0 || o.p.B <= 0) return false;
  if (o.p.in_mode != kInComplex || o.p.out_real) return false;
  return pipe_supported(prec, o.n);
}

static void pipeline_pairs(std::vector<Op>& prog, Ctx& ctx) {
  // DFFTB_PIPE_LOCAL=1: also pair two local passes (profiling aid: lets the
  // pipelined kernel run, and be profiled, on one GPU)
  const char* pl = getenv("DFFTB_PIPE_LOCAL");
  const bool local_pairs = pl && *pl == '1';
  if (ctx.world_mode || (ctx.nranks < 2 && !local_pairs)) return;
  {
    // opt-in: measured slower than the sequential passes in round 1
    const char* e = getenv("DFFTB_PIPE");
    if (!(e && *e == '1') && !local_pairs) return;
  }
  int want = 16;
  if (const char* e = getenv("DFFTB_PIPE_CHUNKS")) want = std::max(2, std::min(kMaxChunks, atoi(e)));
  double frac_env = -1.0;
  if (const char* e = getenv("DFFTB_PIPE_FRAC")) frac_env = atof(e);
  if ((int)ctx.pipe_cum.size() < kPipeSlots) ctx.pipe_cum.assign(kPipeSlots, {});
  const int me = ctx.rank;
  const int prec = ctx.prec;
  const int64_t csize = 2 * prec;
  int slot = 0;
  for (size_t i = 0; i + 1 < prog.size() && slot < kPipeSlots; ++i) {
    Op& P = prog[i];
    if (!pipe_candidate(P, prec)) continue;
    size_t jq = i + 1;
    const bool bar = prog[jq].barrier;
    if (bar) ++jq;
    if (jq >= prog.size()) continue;
    Op& Q = prog[jq];
    if (!pipe_candidate(Q, prec) || Q.n != P.n || Q.p.inverse != P.p.inverse) continue;
    const bool p_remote = P.fused && P.members.size() > 1;
    const bool q_remote = Q.fused && Q.members.size() > 1;
    if (p_remote == q_remote && !(local_pairs && !p_remote)) continue;  // only NVLink next to HBM gains
    // Q reads what P stored for this rank
    int q_me = 0;
    if (P.fused)
      for (size_t q = 0; q < P.members.size(); ++q)
        if (P.members[q] == me) q_me = (int)q;
    if (P.p.dest[q_me].ptr != Q.p.in) continue;
    if (P.before->ndim() != 3 || Q.before->ndim() != 3 || P.v == Q.v) continue;
    const int X = 3 - P.v - Q.v;
    if ((X != P.ax_a && X != P.ax_b) || (X != Q.ax_a && X != Q.ax_b)) continue;
    const bool pbeta = X == P.ax_b, qbeta = X == Q.ax_b;
    const int W = tma_tile_w(prec, P.n);
    int64_t offP[kMaxDims], lenP[kMaxDims], offQ[kMaxDims], lenQ[kMaxDims];
    P.before->extents_of(me, offP, lenP);
    Q.before->extents_of(me, offQ, lenQ);
    if (lenP[X] != lenQ[X] || offP[X] != offQ[X]) continue;
    const int64_t Xe = lenP[X];
    int64_t R = (Xe + want - 1) / want;
    if (pbeta || qbeta) R = ((R + W - 1) / W) * W;
    const int C = (int)((Xe + R - 1) / R);
    if (C < 2 || C > kMaxChunks) continue;
    auto tiles_b = [&](int64_t B) { return (B + W - 1) / W; };
    auto tpc_of = [&](bool beta, int64_t A, int64_t B) { return beta ? (R / W) * A : R * tiles_b(B); };
    auto in_chunk = [&](bool beta, int64_t A, int64_t B, int c) -> int64_t {
      if (beta) {
        const int64_t b0 = c * (R / W), b1 = std::min(b0 + R / W, tiles_b(B));
        return std::max<int64_t>(0, b1 - b0) * A;
      }
      const int64_t a0 = c * R, a1 = std::min(a0 + R, A);
      return std::max<int64_t>(0, a1 - a0) * tiles_b(B);
    };
    // every rank P writes into publishes there; the ranks writing into this
    // rank's buffer are the same group (symmetric exchange)
    std::vector<int> writers = p_remote ? P.members : std::vector<int>{me};
    unsigned long long expect[kMaxChunks] = {};
    for (int m : writers) {
      int64_t o[kMaxDims], l[kMaxDims];
      P.before->extents_of(m, o, l);
      for (int c = 0; c < C; ++c) expect[c] += (unsigned long long)in_chunk(pbeta, l[P.ax_a], l[P.ax_b], c);
    }
    Op M = P;
    M.pipe = true;
    M.fused = true;
    M.pb = Q.p;
    M.tpb = Q.tp;
    M.adj_b = Q.adj;
    PipeArgs& pa = M.ppa;
    PipeArgs& pq = M.ppb;
    std::memset(&pa, 0, sizeof(pa));
    std::memset(&pq, 0, sizeof(pq));
    pa.order_beta = pbeta ? (int)(R / W) : 0;
    pa.tpc = tpc_of(pbeta, P.p.A, P.p.B);
    pa.pub_sys = p_remote;
    const std::vector<int> targets = p_remote ? P.members : std::vector<int>{me};
    pa.npub = (int)targets.size();
    for (size_t q = 0; q < targets.size(); ++q)
      pa.pub[q] = reinterpret_cast<unsigned long long*>(ctx.flags_of(targets[q])) + kPipeOffU64 +
                  (size_t)slot * kMaxChunks;
    pq.order_beta = qbeta ? (int)(R / W) : 0;
    pq.tpc = tpc_of(qbeta, Q.p.A, Q.p.B);
    pq.wait = reinterpret_cast<const unsigned long long*>(ctx.flags_of(me)) + kPipeOffU64 +
              (size_t)slot * kMaxChunks;
    for (int c = 0; c < C; ++c) {
      ctx.pipe_cum[slot][c] += expect[c];
      pq.target[c] = ctx.pipe_cum[slot][c];
    }
    pq.timeout_flag = ctx.dstat + 2;
    pq.timeout_ns = 10ull * 1000 * 1000 * 1000;
    // CTA split: balance max(SM-bound time, NVLink time) of the two roles
    if (frac_env > 0.0 && frac_env < 1.0) {
      M.frac = frac_env;
    } else {
      const double sm_rate = 40e9, nvl_rate = 700e9;  // B/s per SM (read + write), per GPU
      auto role_time = [&](const Op& o, bool remote, double share) {
        const double rw = 2.0 * (double)o.p.A * o.p.B * o.n * csize;
        const double nvl = remote ? 0.5 * rw * (double)(o.members.size() - 1) / o.members.size() : 0.0;
        return std::max(rw / (share * 148.0 * sm_rate), nvl / nvl_rate);
      };
      double best = 1e30;
      for (int g = 8; g <= 140; ++g) {
        const double f = g / 148.0;
        const double t = std::max(role_time(P, p_remote, f), role_time(Q, q_remote, 1.0 - f));
        if (t < best) {
          best = t;
          M.frac = f;
        }
      }
    }
    prog[i] = M;
    prog.erase(prog.begin() + (long)jq);
    if (bar) prog.erase(prog.begin() + (long)i + 1);
    ++slot;
  }
}

// Single GPU: the rows pass and the columns pass of every x0 plane run as
// ONE pipelined launch whose intermediate lives in an L2-resident ring of
// planes instead of a full buffer in HBM — two axes for one HBM round trip.
// Producer CTAs transform rows into ring slot (plane % ring); consumer CTAs
// wait for a chunk of planes, load it (TMA), drop the ring rows from L2
// (discard: never written back) and transform the columns; the producer
// reuses a slot once its chunk was consumed.  Counters are local and zeroed
// before each launch (stream order), so no cross-execute bookkeeping.
static constexpr int kRingMaxChunks = 4096;

static bool ring_enabled() {
  const char* e = getenv("DFFTB_RING");
  return e && *e == '1';
}

static void ring_pairs(std::vector<Op>& prog, Ctx& ctx) {
  if (ctx.world_mode || ctx.nranks != 1 || prog.size() < 2 || !ring_enabled()) return;
  Op& P = prog[0];
  Op& Q = prog[1];
  const int prec = ctx.prec;
  const int64_t csize = 2 * prec;
  auto plain = [&](const Op& o) {
    return !o.barrier && o.tma && !o.generic && !o.fused2 && !o.pipe && o.p.in_mode == kInComplex &&
           !o.p.out_real && o.p.A1 <= 1 && o.p.A > 0 && o.p.B > 0 && !o.tp.args.ldgsts;
  };
  if (!plain(P) || !plain(Q) || P.n != Q.n || !pipe_supported(prec, P.n)) return;
  if (P.adj || !Q.adj || P.p.inverse != Q.p.inverse) return;
  if (P.p.ndest != 1 || P.p.store_mode != 0 || P.p.dest[0].ptr != Q.p.in) return;
  if (P.p.A != Q.p.A || P.p.dest[0].sa != Q.p.in_sa || P.p.dest[0].base != 0 || Q.p.in_sb != 1) return;
  const int W = tma_tile_w(prec, P.n);
  int R = 2, L = 4;
  if (const char* e = getenv("DFFTB_RING_R")) R = std::max(1, atoi(e));
  if (const char* e = getenv("DFFTB_RING_L")) L = std::max(2, atoi(e));
  double frac = 0.5;
  if (const char* e = getenv("DFFTB_RING_FRAC")) frac = atof(e);
  // Deadlock freedom: a CTA waits (for its prefetch, STAGES tiles ahead)
  // while holding its current tiles unstored.  The producer's reuse lag must
  // therefore exceed both roles' prefetch reach in chunks.
  {
    const int64_t tb = std::max<int64_t>((P.p.B + W - 1) / W, (Q.p.B + W - 1) / W);
    const int np = std::max(1, (int)(frac * 148 + 0.5)), nq = std::max(1, 148 - np);
    const int64_t reach = 2 * (int64_t)std::max(np, nq);  // STAGES = 2 tiles per CTA ahead
    R = std::max<int64_t>(R, (reach + tb - 1) / tb);       // a chunk spans one reach
    const int64_t tpc = (int64_t)R * ((std::min(P.p.B, Q.p.B) + W - 1) / W);
    const int need = (int)((reach + tpc - 1) / tpc) * 2 + 2;
    L = std::max(L, need);
  }
  const int A = P.p.A;
  const int ringP = R * L;
  const int C = (A + R - 1) / R;
  if (A < 2 * ringP || C > kRingMaxChunks) return;
  const size_t bytes = (size_t)ringP * (size_t)Q.p.in_sa * csize;
  if (ctx.ring_bytes < bytes) {
    if (ctx.ring) cudaFree(ctx.ring);
    ctx.ring = nullptr;
    ctx.ring_bytes = 0;
    CUDA_TRY(cudaMalloc(&ctx.ring, bytes));
    ctx.ring_bytes = bytes;
  }
  if (!ctx.ring_ctr) CUDA_TRY(cudaMalloc(&ctx.ring_ctr, 2 * kRingMaxChunks * sizeof(unsigned long long)));
  // consumer's tensor map over the ring (same strides, ringP planes)
  TmaPlan tq = Q.tp;
  {
    auto enc = tensor_map_encoder();
    if (!enc) return;
    const int64_t si = Q.p.in_si * csize, sa = Q.p.in_sa * csize;
    cuuint64_t gdim[3] = {2 * (cuuint64_t)Q.p.B, 0, 0};
    cuuint64_t gstride[2];
    cuuint32_t box[3] = {(cuuint32_t)(2 * W), 0, 0}, estr[3] = {1, 1, 1};
    const int rows = Q.tp.args.rows;
    if (Q.tp.args.i_dim == 1) {
      gdim[1] = Q.n;
      gdim[2] = ringP;
      gstride[0] = si;
      gstride[1] = sa;
      box[1] = rows;
      box[2] = 1;
    } else {
      gdim[1] = ringP;
      gdim[2] = Q.n;
      gstride[0] = sa;
      gstride[1] = si;
      box[1] = 1;
      box[2] = rows;
    }
    if (enc(&tq.tmap, prec == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ctx.ring,
            gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return;
  }
  const int64_t tbP = (P.p.B + W - 1) / W, tbQ = (Q.p.B + W - 1) / W;
  const int64_t tpcP = (int64_t)R * tbP, tpcQ = (int64_t)R * tbQ;
  unsigned long long* fwd_ctr = ctx.ring_ctr;
  unsigned long long* back_ctr = ctx.ring_ctr + kRingMaxChunks;
  Op M = P;
  M.pipe = true;
  M.ring_reset = true;
  M.p.dest[0].ptr = ctx.ring;
  M.pb = Q.p;
  M.pb.in = ctx.ring;
  M.tpb = tq;
  M.adj_b = Q.adj;
  PipeArgs& pa = M.ppa;
  PipeArgs& pq = M.ppb;
  std::memset(&pa, 0, sizeof(pa));
  std::memset(&pq, 0, sizeof(pq));
  pa.tpc = tpcP;
  pa.npub = 1;
  pa.pub[0] = fwd_ctr;
  pa.ring = ringP;
  pa.ring_role = 1;
  pa.peer_tpc = tpcQ;
  pa.peer_ntiles = Q.tp.args.ntiles;
  pa.back_wait = back_ctr;
  pa.back_lag = L;
  pq.tpc = tpcQ;
  pq.wait = fwd_ctr;
  pq.ring = ringP;
  pq.ring_role = 2;
  pq.ring_discard = (int64_t)W * csize == 128 ? 1 : 0;
  if (const char* e = getenv("DFFTB_RING_DISCARD")) pq.ring_discard = pq.ring_discard && *e != '0';
  pq.peer_tpc = tpcP;
  pq.peer_ntiles = P.tp.args.ntiles;
  pq.back_pub = back_ctr;
  for (PipeArgs* x : {&pa, &pq}) {
    x->timeout_flag = ctx.dstat + 2;
    x->timeout_ns = 10ull * 1000 * 1000 * 1000;
  }
  M.frac = frac;
  prog[0] = M;
  prog.erase(prog.begin() + 1);
}

// One rank's program: fused passes and barriers.  `peer` supplies the
// exchange-buffer base of any world rank (its own mapping of the peers).
static std::vector<Op> lower(const Plan& plan, Ctx& ctx, const void* d_in, void* d_out,
                             int parity) {
  std::vector<Op> prog;
  if (lower_single(plan, ctx, d_in, d_out, parity, prog)) {
    ring_pairs(prog, ctx);
    return prog;
  }
  const int me = ctx.rank;
  const void* cur = d_in;
  bool cur_internal = false;  // d_in has the user layout; exch/work are padded
  bool cur_swap01 = false;    // current buffer stored [x1][x0][rest]
  int slot = 0;
  const auto& S = plan.stages;
  size_t i = 0;
  while (i < S.size()) {
    const Stage& st = S[i];
    if (st.type != StageType::Fft) raise(DFFTB_ConfigInvalid, "unexpected stage order");
    const Stage* tr = (i + 1 < S.size() && S[i + 1].type == StageType::Transpose) ? &S[i + 1] : nullptr;
    const Stage* nm = (i + 1 < S.size() && S[i + 1].type == StageType::Normalize) ? &S[i + 1] : nullptr;
    const bool last_fft = (i + 1 == S.size()) || nm != nullptr;

    const Dist& Lb = st.before;
    const int nd = Lb.ndim();
    int64_t offb[kMaxDims], lenb[kMaxDims], sb[kMaxDims];
    Lb.extents_of(me, offb, lenb);
    row_major_strides(lenb, nd, sb, cur_internal, ctx.prec, cur_swap01);
    const int v = st.axis;
    // lane axes in memory order: [ax_a1 (4-D only)] [ax_a] ax_b (innermost)
    int ax_a1 = -1, ax_a = -1, ax_b = -1;
    {
      int lanes[kMaxDims], nl = 0;
      for (int a = 0; a < nd; ++a)
        if (a != v) lanes[nl++] = a;
      ax_b = lanes[nl - 1];
      if (nl >= 2) ax_a = lanes[nl - 2];
      if (nl >= 3) ax_a1 = lanes[nl - 3];
    }
    Op op;
    op.v = v;
    op.ax_a = ax_a;
    op.ax_b = ax_b;
    op.ax_a1 = ax_a1;
    op.before = &Lb;
    PassParams& p = op.p;
    p.in = cur;
    p.A = ax_a >= 0 ? (int)lenb[ax_a] : 1;
    p.A1 = ax_a1 >= 0 ? (int)lenb[ax_a1] : 1;
    p.in_sa1 = ax_a1 >= 0 ? sb[ax_a1] : 0;
    p.B = (int)lenb[ax_b];
    p.in_sa = ax_a >= 0 ? sb[ax_a] : 0;
    p.in_sb = sb[ax_b];
    p.in_si = sb[v];
    const int n = st.fkind == DFFTB_C2R ? (int)st.after.dims[v] : (int)lenb[v];
    op.n = n;
    p.n_out = st.fkind == DFFTB_R2C ? n / 2 + 1 : n;
    p.in_mode = st.fkind == DFFTB_R2C ? kInReal : (st.fkind == DFFTB_C2R ? kInHermitian : kInComplex);
    p.out_real = st.fkind == DFFTB_C2R;
    p.inverse = st.dir == DFFTB_BACKWARD;
    p.scale = nm ? nm->factor : 1.0;
    p.tw = is_pow2(n) ? ctx.twiddles.at(n) : nullptr;
    p.herm = ctx.dstat;
    op.adj = p.in_si != 1;
    if (lenb[v] == 0 && st.fkind != DFFTB_C2R) p.A = 0;

    op.tma = false;
    if (tr) {
      const Dist& Lo = tr->after;
      const int g = tr->grid_axis;
      const int u = tr->before.axis_of_grid[g];
      // the transposed final forward exchange feeds the axis-0 pass: store
      // its buffer [x1][x0][rest] so axis-0 lanes read short strides
      const bool swap_out = tr->transposed && zperm_enabled() && nd >= 3;
      op.fused = true;
      op.grid_axis = g;
      op.members = group_members(Lo, me, g);
      p.ndest = (int)op.members.size();
      p.oblk = (Lo.dims[v] + Lo.grid[g] - 1) / Lo.grid[g];
      for (int q = 0; q < p.ndest; ++q) {
        const int rq = op.members[q];
        int64_t offo[kMaxDims], leno[kMaxDims], so[kMaxDims];
        Lo.extents_of(rq, offo, leno);
        row_major_strides(leno, nd, so, true, ctx.prec, swap_out);
        Dest& d = p.dest[q];
        d.ptr = ctx.exch(rq, slot, parity);
        d.base = offb[u] * so[u];
        d.sa = ax_a >= 0 ? so[ax_a] : 0;
        d.sa1 = ax_a1 >= 0 ? so[ax_a1] : 0;
        d.sb = so[ax_b];
        d.sk = so[v];
      }
      set_store_mode(p);
      op.tma = plan_tma(op, ctx.prec);
      plan_generic(op, ctx);
      prog.push_back(op);
      Op b;
      b.barrier = true;
      b.grid_axis = g;
      b.members = op.members;
      if (b.members.size() > 1) prog.push_back(b);
      cur = ctx.exch(me, slot, parity);
      cur_internal = true;
      cur_swap01 = swap_out;
      ++slot;
      i += tr->transposed ? 3 : 2;  // the LocalTransposeStage is folded in
    } else {
      const Dist& Lo = st.after;
      int64_t offo[kMaxDims], leno[kMaxDims], so[kMaxDims];
      Lo.extents_of(me, offo, leno);
      row_major_strides(leno, nd, so, !last_fft, ctx.prec);
      void* out = last_fft ? d_out : ctx.work;
      p.ndest = 1;
      p.oblk = p.n_out > 0 ? p.n_out : 1;
      Dest& d = p.dest[0];
      d.ptr = out;
      d.base = 0;
      d.sa = ax_a >= 0 ? so[ax_a] : 0;
        d.sa1 = ax_a1 >= 0 ? so[ax_a1] : 0;
      d.sb = so[ax_b];
      d.sk = so[v];
      set_store_mode(p);
      op.tma = plan_tma(op, ctx.prec);
      plan_generic(op, ctx);
      prog.push_back(op);
      cur = out;
      cur_internal = !last_fft;
      cur_swap01 = false;
      i += nm ? 2 : 1;
    }
  }
  fuse_pairs(prog, ctx);
  pipeline_pairs(prog, ctx);
  ring_pairs(prog, ctx);
  return prog;
}

static void launch_op(const Ctx& ctx, const Op& op, uint64_t epoch, cudaStream_t s) {
  if (op.barrier) {
    if (ctx.world_mode) return;  // lockstep emulation: stream order is the barrier
    BarrierParams bp{};
    bp.nmem = (int)op.members.size();
    for (int i = 0; i < bp.nmem; ++i) {
      bp.members[i] = op.members[i];
      bp.peer_flags[i] = reinterpret_cast<unsigned long long*>(ctx.flags_of(op.members[i]));
    }
    bp.me = ctx.rank;
    bp.my_flags = reinterpret_cast<unsigned long long*>(ctx.flags_of(ctx.rank));
    bp.epoch = epoch;
    bp.timeout_ns = kBarrierTimeoutNs;
    bp.timeout_flag = ctx.dstat + 2;
    CUDA_TRY(launch_barrier(bp, s));
    return;
  }
  if ((int64_t)op.p.A * op.p.B == 0) return;
  if (op.fused2) {
    CUDA_TRY(cudaMemsetAsync(op.fa.doneA, 0, 2 * sizeof(unsigned int) * op.fa.P, s));
    CUDA_TRY(launch_fused2(ctx.prec, op.n, op.fwd2, op.p, op.pb, op.tp.tmap, op.fa, s));
    return;
  }
  if (op.pipe) {
    if (op.ring_reset)
      CUDA_TRY(cudaMemsetAsync(ctx.ring_ctr, 0, 2 * kRingMaxChunks * sizeof(unsigned long long), s));
    CUDA_TRY(launch_pipe(ctx.prec, op.n, op.p, op.adj, op.tp, op.ppa, op.pb, op.adj_b, op.tpb, op.ppb, op.frac, s));
    const char* dbg = getenv("DFFTB_RING_DEBUG");
    if (op.ring_reset && dbg && *dbg == '1') {
      std::vector<unsigned long long> h(2 * kRingMaxChunks);
      CUDA_TRY(cudaMemcpyAsync(h.data(), ctx.ring_ctr, h.size() * 8, cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
      const int C = (int)((op.tp.args.ntiles + op.ppa.tpc - 1) / op.ppa.tpc);
      fprintf(stderr, "[ring] tpcP %lld ntP %lld tpcQ %lld ntQ %lld chunks %d ring %d lag %d frac %.2f\n",
              (long long)op.ppa.tpc, (long long)op.tp.args.ntiles, (long long)op.ppb.tpc,
              (long long)op.tpb.args.ntiles, C, op.ppa.ring, op.ppa.back_lag, op.frac);
      for (int c = 0; c < C; ++c)
        if (c < 6 || c > C - 3 || h[c] != (unsigned long long)op.ppa.tpc ||
            h[kRingMaxChunks + c] != (unsigned long long)op.ppb.tpc)
          fprintf(stderr, "[ring] chunk %d produced %llu consumed %llu\n", c, h[c], h[kRingMaxChunks + c]);
    }
    return;
  }
  if (op.generic) CUDA_TRY(launch_generic(ctx.prec, op.g, s));
  else if (op.tma) CUDA_TRY(launch_pass_tma(ctx.prec, op.n, op.p, op.adj, op.tp, s));
  else CUDA_TRY(launch_pass(ctx.prec, op.n, op.p, op.adj, s));
}

static bool plan_has_c2r(const Plan& plan) {
  for (const auto& st : plan.stages)
    if (st.type == StageType::Fft && st.fkind == DFFTB_C2R) return true;
  return false;
}

static void validate_finite(const Plan& plan, const Ctx& ctx, const void* d_in, cudaStream_t s) {
  const int64_t n = plan.input.local_count(ctx.rank) * (plan.input.complex_el ? 2 : 1);
  CUDA_TRY(cudaMemsetAsync(ctx.dstat + 3, 0, sizeof(unsigned long long), s));
  CUDA_TRY(launch_nonfinite(plan.prec, d_in, n, ctx.dstat + 3, s));
  unsigned long long bad = 0;
  CUDA_TRY(cudaMemcpyAsync(&bad, ctx.dstat + 3, sizeof(bad), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (bad) raise(DFFTB_ConfigInvalid, "non-finite values in plan input");
}

void ctx_check(Ctx& ctx, cudaStream_t s) {
  DeviceGuard g(ctx.device);
  unsigned long long st[4];
  CUDA_TRY(cudaMemcpyAsync(st, ctx.dstat, sizeof(st), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (st[2]) {
    CUDA_TRY(cudaMemset(ctx.dstat + 2, 0, sizeof(unsigned long long)));
    raise(DFFTB_Deadlock, "peer did not reach the exchange barrier (timeout)");
  }
  if (ctx.c2r_pending) {
    ctx.c2r_pending = false;
    double mx, im;
    std::memcpy(&mx, &st[0], sizeof(double));
    std::memcpy(&im, &st[1], sizeof(double));
    // irfft_1d tolerance, kernels.hpp:348-377 (scale = block max, plan.hpp:440-446)
    const double tol = (ctx.prec == 8 ? 1e-6 : 1e-2) * mx;
    const char* skip = getenv("DFFTB_DEBUG_SKIP_HERM");
    if (im > tol && !(skip && *skip == '1')) {
      char buf[160];
      snprintf(buf, sizeof(buf),
               "DC or Nyquist bin has a non-real component (|Im| %.3g > tol %.3g, block max %.3g)",
               im, tol, mx);
      raise(DFFTB_NonHermitian, buf);
    }
  }
}

struct EventTimer {
  std::vector<cudaEvent_t> ev;
  ~EventTimer() {
    for (auto e : ev) cudaEventDestroy(e);
  }
  void mark(cudaStream_t s) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.push_back(e);
  }
};

static void run_program(const Plan& plan, Ctx& ctx, const std::vector<Op>& prog, cudaStream_t s, int flags,
                        dfftb_timing* timers);

void execute(const Plan& plan, Ctx& ctx, const void* d_in, void* d_out, cudaStream_t s, int flags,
             dfftb_timing* timers) {
  DeviceGuard g(ctx.device);
  check_compatible(plan, ctx);
  if (plan.options.validate_finite) validate_finite(plan, ctx, d_in, s);
  const int parity = (int)(ctx.exec_count & 1);
  ctx.exec_count++;
  auto prog = lower(plan, ctx, d_in, d_out, parity);
  run_program(plan, ctx, prog, s, flags, timers);
}

static void run_program(const Plan& plan, Ctx& ctx, const std::vector<Op>& prog, cudaStream_t s, int flags,
                        dfftb_timing* timers) {
  if (plan_has_c2r(plan)) {
    CUDA_TRY(cudaMemsetAsync(ctx.dstat, 0, 2 * sizeof(unsigned long long), s));
    ctx.c2r_pending = true;
  }
  EventTimer et;
  if (timers) et.mark(s);
  for (const auto& op : prog) {
    const uint64_t epoch = op.barrier ? ++ctx.epoch : 0;
    launch_op(ctx, op, epoch, s);
    if (timers) et.mark(s);
  }
  if (timers) {
    CUDA_TRY(cudaStreamSynchronize(s));
    std::memset(timers, 0, sizeof(*timers));
    for (size_t k = 0; k < prog.size(); ++k) {
      float ms = 0;
      cudaEventElapsedTime(&ms, et.ev[k], et.ev[k + 1]);
      const double sec = ms * 1e-3;
      if (prog[k].barrier || prog[k].fused) timers->wire_comm += sec;
      else timers->local_fft += sec;
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, et.ev.front(), et.ev.back());
    timers->total = ms * 1e-3;
    // profiling aid: DFFTB_OP_TIMES=1 prints every op of the program
    const char* ot = getenv("DFFTB_OP_TIMES");
    if (ot && *ot == '1') {
      for (size_t k = 0; k < prog.size(); ++k) {
        float m = 0;
        cudaEventElapsedTime(&m, et.ev[k], et.ev[k + 1]);
        const Op& o = prog[k];
        fprintf(stderr, "[dfftb rank %d] op %zu %s n=%d A=%d B=%d dests=%d: %.3f ms\n", ctx.rank, k,
                o.barrier ? "barrier" : (o.pipe ? "pipe" : (o.fused ? "fused-exchange" : "local")), o.n, o.p.A,
                o.p.B, o.p.ndest, m);
      }
    }
  }
  if (timers || (flags & DFFTB_EXEC_SYNC)) ctx_check(ctx, s);
}

void execute_world(const Plan& plan, Ctx** ctxs, const void* const* d_in, void* const* d_out,
                   cudaStream_t s, int flags) {
  const int P = plan.nranks();
  std::vector<std::vector<Op>> progs(P);
  for (int r = 0; r < P; ++r) {
    if (!ctxs[r]->world_mode) raise(DFFTB_ConfigInvalid, "not an emulated world");
    check_compatible(plan, *ctxs[r]);
    if (ctxs[r]->rank != r) raise(DFFTB_InvalidRank, "world contexts must be in rank order");
  }
  DeviceGuard g(ctxs[0]->device);
  for (int r = 0; r < P; ++r) {
    if (plan.options.validate_finite) validate_finite(plan, *ctxs[r], d_in[r], s);
    const int parity = (int)(ctxs[r]->exec_count & 1);
    ctxs[r]->exec_count++;
    progs[r] = lower(plan, *ctxs[r], d_in[r], d_out[r], parity);
    if (plan_has_c2r(plan)) {
      CUDA_TRY(cudaMemsetAsync(ctxs[r]->dstat, 0, 2 * sizeof(unsigned long long), s));
      ctxs[r]->c2r_pending = true;
    }
  }
  const size_t nops = progs[0].size();
  for (int r = 1; r < P; ++r)
    if (progs[r].size() != nops) raise(DFFTB_CountMismatch, "rank programs differ in length");
  for (size_t k = 0; k < nops; ++k)
    for (int r = 0; r < P; ++r) launch_op(*ctxs[r], progs[r][k], 0, s);
  if (flags & DFFTB_EXEC_SYNC)
    for (int r = 0; r < P; ++r) ctx_check(*ctxs[r], s);
}

void fill_seeded(const Plan& plan, int rank, int side, uint64_t seed, int complex_field, void* d_buf,
                 cudaStream_t s) {
  const Dist& d = side == DFFTB_INPUT ? plan.input : plan.output;
  if (rank < 0 || rank >= d.nranks()) raise(DFFTB_InvalidRank, "rank out of range");
  SeedParams sp{};
  sp.nd = d.ndim();
  d.extents_of(rank, sp.off, sp.len);
  sp.count = 1;
  for (int a = 0; a < sp.nd; ++a) {
    sp.gdims[a] = d.dims[a];
    sp.count *= sp.len[a];
  }
  sp.seed = seed;
  sp.complex_field = complex_field;
  sp.out_complex = d.complex_el;
  CUDA_TRY(launch_seeded(plan.prec, sp, d_buf, s));
}

}  // namespace dfftb

namespace dfftb {

// ------------------------------------------------------- spectral operators

static SpectralParams spectral_params(const Plan& plan, int rank, const double* lengths) {
  if (plan.dir != DFFTB_FORWARD) raise(DFFTB_NotFrequencyLayout, "spectral operators need a forward plan's output layout");
  const Dist& f = plan.output;  // frequency layout: all hatted, complex
  if (rank < 0 || rank >= f.nranks()) raise(DFFTB_InvalidRank, "rank out of range");
  SpectralParams sp{};
  sp.nd = f.ndim();
  if (sp.nd > 4) raise(DFFTB_Unsupported, "at most 4 axes");
  f.extents_of(rank, sp.off, sp.len);
  sp.count = 1;
  for (int a = 0; a < sp.nd; ++a) {
    sp.n[a] = plan.dims[a];
    sp.half[a] = f.dims[a] != plan.dims[a];
    sp.scale[a] = 2.0 * M_PI / (lengths ? lengths[a] : 2.0 * M_PI);
    sp.count *= sp.len[a];
  }
  return sp;
}

void spectral_apply(const Plan& plan, int rank, int op, int axis, const double* lengths, const void* in,
                    void* out, int accumulate, cudaStream_t s) {
  SpectralParams sp = spectral_params(plan, rank, lengths);
  if (op < 0 || op > 2) raise(DFFTB_ConfigInvalid, "unknown spectral operator");
  if (op == 0 && (axis < 0 || axis >= sp.nd)) raise(DFFTB_OutOfRange, "derivative axis out of range");
  sp.op = op;
  sp.axis = op == 0 ? axis : 0;
  sp.accumulate = accumulate;
  if (op == 2) {
    // inverse_laplacian needs a zero-mean field (spectral.hpp:266-281)
    bool owns_zero = sp.count > 0;
    for (int a = 0; a < sp.nd; ++a) owns_zero = owns_zero && sp.off[a] == 0;
    if (owns_zero) {
      double v[2] = {0, 0};
      if (plan.prec == 8) {
        CUDA_TRY(cudaMemcpyAsync(v, in, 16, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
      } else {
        float fv[2];
        CUDA_TRY(cudaMemcpyAsync(fv, in, 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        v[0] = fv[0];
        v[1] = fv[1];
      }
      double total = 1;
      for (auto d : plan.dims) total *= (double)d;
      if (std::hypot(v[0], v[1]) > 1e-12 * total)
        raise(DFFTB_NonZeroMean, "inverse_laplacian needs a zero-mean field");
    }
  }
  CUDA_TRY(launch_spectral(plan.prec, sp, in, out, s));
}

// Forward transform with the spectral multiplier fused into the last pass's
// store epilogue: one read + one write of the spectrum
// less than execute + spectral_apply, bit-identical results.  Lengths the
// generic (non-power-of-two) kernel handles take the two-step path.
void execute_spectral(const Plan& plan, Ctx& ctx, const void* d_in, void* d_out, int op, int axis,
                      const double* lengths, int accumulate, cudaStream_t s, int flags) {
  DeviceGuard dg(ctx.device);
  check_compatible(plan, ctx);
  if (ctx.world_mode) raise(DFFTB_ConfigInvalid, "execute_spectral needs a per-rank context (not an emulated world)");
  const SpectralParams sp = spectral_params(plan, ctx.rank, lengths);
  if (op < 0 || op > 2) raise(DFFTB_ConfigInvalid, "unknown spectral operator");
  if (op == 0 && (axis < 0 || axis >= sp.nd)) raise(DFFTB_OutOfRange, "derivative axis out of range");
  if (plan.options.validate_finite) validate_finite(plan, ctx, d_in, s);
  const int parity = (int)(ctx.exec_count & 1);
  ctx.exec_count++;
  auto prog = lower(plan, ctx, d_in, d_out, parity);
  Op* last = prog.empty() ? nullptr : &prog.back();
  const bool fusable = last && !last->barrier && !last->generic && !last->fused2 && !last->pipe &&
                       last->before && last->p.ndest == 1 && last->p.dest[0].ptr == d_out &&
                       !last->p.inverse && last->p.in_mode == kInComplex && !last->p.out_real;
  const char* nf = getenv("DFFTB_SPECTRAL_UNFUSED");
  if (!fusable || (nf && *nf == '1')) {
    run_program(plan, ctx, prog, s, 0, nullptr);
    spectral_apply(plan, ctx.rank, op, axis, lengths, d_out, d_out, accumulate, s);
    if (flags & DFFTB_EXEC_SYNC) ctx_check(ctx, s);
    return;
  }
  SpecEpi& e = last->p.spec;
  std::memset(&e, 0, sizeof(e));
  e.op = op + 1;
  e.accumulate = accumulate;
  const int roles[4] = {last->v, last->ax_a, last->ax_b, last->ax_a1};
  int64_t off[kMaxDims], len[kMaxDims];
  last->before->extents_of(ctx.rank, off, len);
  e.nroles = 0;
  bool owns_dc = true;
  for (int r = 0; r < 4; ++r) {
    const int a = roles[r];
    if (a < 0) {
      // absent lane axis (2-D): a zero coordinate of a length-1 axis
      e.off[r] = 0;
      e.n[r] = 1;
      e.half[r] = 0;
      e.scale[r] = 0.0;
      continue;
    }
    e.nroles = r + 1;
    e.off[r] = r == 0 ? 0 : off[a];
    e.n[r] = sp.n[a];
    e.half[r] = sp.half[a];
    e.scale[r] = sp.scale[a];
    if (op == 0 && a == axis) e.deriv_role = r;
    if (r > 0 && off[a] != 0) owns_dc = false;
  }
  // |k|^2 summed in tensor-axis order (as spectral_kernel): bit-identical
  {
    int n = 0;
    for (int a = 0; a < sp.nd; ++a)
      for (int r = 0; r < 4; ++r)
        if (roles[r] == a) e.order[n++] = r;
    e.nroles = n;
  }
  if (last->tma) {
    // the multiplier variant exists for the strided-lane kernel only
    if (!last->adj) last->tma = false;
  }
  const bool check_mean = op == 2 && owns_dc && sp.count > 0;
  if (check_mean) {
    CUDA_TRY(cudaMemsetAsync(ctx.dstat + 4, 0, 2 * sizeof(unsigned long long), s));
    e.dc = ctx.dstat + 4;
  }
  run_program(plan, ctx, prog, s, 0, nullptr);
  if (check_mean) {
    unsigned long long bits[2];
    CUDA_TRY(cudaMemcpyAsync(bits, ctx.dstat + 4, sizeof(bits), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    double v[2];
    std::memcpy(v, bits, sizeof(v));
    double total = 1;
    for (auto d : plan.dims) total *= (double)d;
    if (std::hypot(v[0], v[1]) > 1e-12 * total)
      raise(DFFTB_NonZeroMean, "inverse_laplacian needs a zero-mean field");
  }
  if (flags & DFFTB_EXEC_SYNC) ctx_check(ctx, s);
}

void wavenumbers(const Plan& plan, int rank, int axis, int deriv, const double* lengths, double* k_out) {
  SpectralParams sp = spectral_params(plan, rank, lengths);
  if (axis < 0 || axis >= sp.nd) raise(DFFTB_OutOfRange, "axis out of range");
  for (int64_t i = 0; i < sp.len[axis]; ++i) {
    const int64_t g = sp.off[axis] + i;
    int64_t k = g;
    if (!sp.half[axis] && 2 * g >= sp.n[axis]) k = g - sp.n[axis];
    const bool nyq = sp.n[axis] % 2 == 0 && 2 * std::llabs(k) == sp.n[axis];
    k_out[i] = (deriv && nyq) ? 0.0 : sp.scale[axis] * (double)k;
  }
}

}  // namespace dfftb
