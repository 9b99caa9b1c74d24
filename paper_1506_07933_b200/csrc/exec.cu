// dfftb executor: contexts (make_context, plan.hpp:359-390), lowering of a
// plan to fused GPU passes + cross-GPU sync points, and execute
// (plan.hpp:463-535).
//
// Lowering.  The reference runs, per rank, LocalFftStage -> TransposeStage
// (pack, all_to_all, unpack; exchange.hpp:547-590) [-> LocalTransposeStage]
// ... -> NormalizeStage.  Here every FFT stage becomes ONE kernel launch
// whose store epilogue writes each output element to its final address in
// the stage's target layout:
//   FFT followed by a transpose  -> peer exchange buffers of the grid-axis
//                                   group (NVLink stores), then a sync point
//   FFT followed by Normalize    -> user output, scaled by 1/N
//   last FFT                     -> user output
//   FFT followed by a local FFT  -> private work buffer
// so each axis costs one read + one write of the local block.
//
// Overlap.  An exchange pass followed by a local pass is
// split into chunks along the lane axis both passes share.  Default (staged,
// exchange.hpp:225-246): the exchange pass writes the other members' parts
// into local staging images at HBM speed, copy-engine DMAs stream chunk c
// over NVLink and signal it, and the local pass starts chunk c as soon as
// every member's chunk c has landed -- NVLink traffic runs under the SM
// passes.  PIPELINED (pipelined_all_to_all, exchange.hpp:323-423): the
// exchange pass stores to the peers itself, chunk by chunk, on a share of
// the SMs while the local pass runs on the others.
//
// Programs are lowered once per (plan, buffers, parity) and cached in the
// context; the launches of a cached program are captured into a CUDA graph.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <unistd.h>

#include <algorithm>
#include <complex>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
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

static constexpr uint64_t kHandleMagic = 0x64666674625f3032ull;  // "dfftb_02"
static constexpr size_t kFlagsBytes = (size_t)kSyncSlots * kMaxRanksDev * sizeof(unsigned long long);
static constexpr unsigned long long kSyncTimeoutNs = 60ull * 1000 * 1000 * 1000;
static constexpr int kStatEpoch = 6;
static constexpr int kStatWords = 8;
static constexpr size_t kMaxCachedPrograms = 64;

// ------------------------------------------------------------------- knobs
// Read once per process (never on the execute path).  Defaults are the
// shipped configuration; the variables exist for A/B measurements.
struct Knobs {
  bool zperm = true;          // DFFTB_ZPERM: axis-0 pass input stored [x1][x0][rest]
  bool single_reorder = true; // DFFTB_SINGLE_REORDER: 1-rank backward in forward axis order
  bool tma = true;            // DFFTB_NO_TMA=1 disables the TMA pass kernel
  int l2promo = 3;            // DFFTB_L2PROMO: tensor-map L2 promotion 0/64/128/256 B
  bool unaligned_ldgsts = true;  // DFFTB_UNALIGNED_LDGSTS: cp.async loader for odd fp32 rows
  int overlap = -1;           // DFFTB_OVERLAP: pipelined exchange/local pass pairs (-1: plans with
                              // ExchangePath::Pipelined only, 0 never, 1 every multi-rank plan)
  int chunks = 4;             // DFFTB_OVERLAP_CHUNKS: chunks per pipelined pair
  double frac = -1.0;         // DFFTB_OVERLAP_FRAC: SM share of the exchange pass (<0: model)
  bool graphs = true;         // DFFTB_GRAPHS: replay cached programs as CUDA graphs
  bool op_times = false;      // DFFTB_OP_TIMES: print per-op device times of timed executes
  bool pdl = false;           // DFFTB_PDL: programmatic dependent launch between passes (opt-in:
                              // 512^3 4.18 -> 4.14 ms, but 1024^3 46.4 -> 53.4 ms)
  bool rhalf = true;          // DFFTB_RHALF: R2C / C2R lanes as half-length complex FFTs
  int row_align = 32;         // DFFTB_ROW_ALIGN: internal row padding in bytes (16, 32 or 64)
  bool dma_flat = true;       // DFFTB_DMA_FLAT: staged exchanges keep the [x0][x1][x2] order (2-D boxes)
  int dma_max_group = 2;      // DFFTB_DMA_MAX_GROUP: stage exchanges of at most this many members
  int dma_streams = 2;        // DFFTB_DMA_STREAMS: copy streams of the staged exchange (1..4; chunks
                              // round-robin, so up to that many DMAs in flight)
  bool r2c_order = true;      // DFFTB_R2C_ORDER: single-rank R2C forward as F2, F0, F1
  int dma = 1;                // DFFTB_DMA: staged copy-engine exchange for Blocking / Staged plans
                              // (0: direct peer stores everywhere)
  int dma_chunks = 8;         // DFFTB_DMA_CHUNKS: chunks of a staged exchange (chunks_per_peer > 1 wins)
  double dma_min_mb = 128.0;  // DFFTB_DMA_MIN_MB: smallest block per rank (MiB) worth staging
  int dma_min_row = 1024;     // DFFTB_DMA_MIN_ROW: smallest chunk row (bytes) worth staging
};

static const Knobs& knobs() {
  static const Knobs k = [] {
    Knobs k;
    auto flag = [](const char* name, bool def) {
      const char* e = getenv(name);
      return e && *e ? *e != '0' : def;
    };
    k.zperm = flag("DFFTB_ZPERM", true);
    k.single_reorder = flag("DFFTB_SINGLE_REORDER", true);
    k.tma = !flag("DFFTB_NO_TMA", false);
    if (const char* e = getenv("DFFTB_L2PROMO")) k.l2promo = atoi(e);
    k.unaligned_ldgsts = flag("DFFTB_UNALIGNED_LDGSTS", true);
    if (const char* e = getenv("DFFTB_OVERLAP")) k.overlap = atoi(e);
    if (const char* e = getenv("DFFTB_OVERLAP_CHUNKS")) k.chunks = std::max(1, std::min(16, atoi(e)));
    if (const char* e = getenv("DFFTB_OVERLAP_FRAC")) k.frac = atof(e);
    k.graphs = flag("DFFTB_GRAPHS", true);
    k.op_times = flag("DFFTB_OP_TIMES", false);
    k.pdl = flag("DFFTB_PDL", false);
    k.rhalf = flag("DFFTB_RHALF", true);
    if (const char* e = getenv("DFFTB_DMA")) k.dma = atoi(e);
    k.r2c_order = flag("DFFTB_R2C_ORDER", true);
    if (const char* e = getenv("DFFTB_DMA_CHUNKS")) k.dma_chunks = std::max(1, std::min(16, atoi(e)));
    if (const char* e = getenv("DFFTB_DMA_MIN_MB")) k.dma_min_mb = atof(e);
    if (const char* e = getenv("DFFTB_DMA_MIN_ROW")) k.dma_min_row = atoi(e);
    k.dma_flat = flag("DFFTB_DMA_FLAT", true);
    if (const char* e = getenv("DFFTB_DMA_MAX_GROUP")) k.dma_max_group = atoi(e);
    if (const char* e = getenv("DFFTB_DMA_STREAMS")) k.dma_streams = std::max(1, std::min(kCopyStreams, atoi(e)));
    if (const char* e = getenv("DFFTB_ROW_ALIGN")) {
      const int a = atoi(e);
      k.row_align = (a == 16 || a == 32 || a == 64 || a == 128) ? a : 32;
    }
    return k;
  }();
  return k;
}

static int64_t inner_pad(int64_t len, int prec) {
  const int64_t q = std::max<int64_t>(1, knobs().row_align / (2 * prec));  // complex elements per unit
  return (len + q - 1) / q * q;
}

void* Ctx::exch(int r, int slot, int parity) const {
  if (slot < 0 || slot >= exch_slots) raise(DFFTB_ArenaExhausted, "exchange slot out of range");
  char* base = static_cast<char*>(peer_region[r]);
  if (parities == 1) parity = 0;
  return base + flags_bytes + (size_t)(parities * slot + parity) * exch_bytes;
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

struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// Internal (exchange / work) buffers keep the reference's axis order but pad
// the innermost extent so every row starts on a 16-byte boundary (fp32
// complex rows of odd length, e.g. the 129-bin R2C axis), which lets the TMA
// path describe them.  User-visible buffers are never padded.
static const struct Knobs& knobs();

// Internal buffers pad their innermost rows to a multiple of
// DFFTB_ROW_ALIGN bytes (default 32: a DRAM sector), so TMA can describe them
// (16-byte strides) and strided boxes of narrow tiles start on sector
// boundaries (129-bin R2C rows: 1032 / 2064 bytes otherwise).
static int64_t inner_pad(int64_t len, int prec);

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

// Execute parities of the exchange buffers: two when peers may still read
// one buffer while this rank writes the next execute's data, one for a
// single rank (stream order already separates its executes).
static int family_parities(const Plan& plan) { return plan.nranks() > 1 ? 2 : 1; }

// The private work buffer is used only by an FFT stage followed directly by
// another FFT stage (slab plans: F2 -> F1); pencil and general plans always
// go through a transpose slot.
static bool family_needs_work(const Plan& plan) {
  dfftb_plan_options o = plan.options;
  const int kf = plan.kind == DFFTB_C2C ? DFFTB_C2C : DFFTB_R2C;
  const int kb = plan.kind == DFFTB_C2C ? DFFTB_C2C : DFFTB_C2R;
  for (int d = 0; d < 2; ++d) {
    Plan p = build_plan(plan.dims, plan.decomp, plan.grid, d == 0 ? kf : kb, d, plan.prec, o);
    for (size_t i = 0; i + 1 < p.stages.size(); ++i)
      if (p.stages[i].type == StageType::Fft && p.stages[i + 1].type == StageType::Fft) return true;
  }
  return false;
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
  if (plan.nranks() > kMaxRanksDev) raise(DFFTB_Unsupported, "at most 64 ranks");
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

static void* upload_complex(const std::vector<std::complex<double>>& v, int prec) {
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
  return {upload_complex(chirp, prec), upload_complex(b, prec)};
}

// device bytes of the per-axis tables ctx_create uploads
static size_t table_bytes(const Plan& plan) {
  size_t t = 0;
  std::vector<int64_t> seen;
  for (auto n : plan.dims) {
    if (std::find(seen.begin(), seen.end(), n) != seen.end()) continue;
    seen.push_back(n);
    if (!is_pow2(n) && !is_smooth(n)) t += (size_t)(n + bluestein_m(n)) * 2 * plan.prec;
  }
  // twiddle tables: every power-of-two axis length, plus the half length of
  // the last axis the half-length R2C / C2R lanes use (as ctx_create)
  std::vector<int64_t> tabs;
  for (auto n : plan.dims) {
    if (!is_pow2(n)) continue;
    tabs.push_back(n);
  }
  const int64_t nl = plan.dims.back();
  if (plan.kind != DFFTB_C2C && is_pow2(nl) && nl >= 16) tabs.push_back(nl / 2);
  std::sort(tabs.begin(), tabs.end());
  tabs.erase(std::unique(tabs.begin(), tabs.end()), tabs.end());
  for (auto n : tabs) t += (size_t)n * 2 * plan.prec;
  return t;
}

// Region granularity.  With peers, the exchange buffers start on 2 MiB
// boundaries: NVLink writes into a buffer 32 KiB off a 2 MiB page run at
// 554 instead of 770 GB/s (copy engine, both directions;
// profiles/r2/ce_ipc_probe.txt).
static size_t region_align(const Plan& plan) { return plan.nranks() > 1 ? (size_t)2 << 20 : 256; }
static size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }
static size_t staging_bytes(const Plan& plan, size_t blk);

size_t workspace_bytes(const Plan& plan, int rank) {
  if (rank < 0 || rank >= plan.nranks()) raise(DFFTB_InvalidRank, "rank out of range");
  const size_t al = region_align(plan);
  const size_t blk = round_up(family_bytes(plan), al);
  return round_up(kFlagsBytes, al) + (size_t)family_parities(plan) * family_exch_slots(plan) * blk +
         staging_bytes(plan, blk) +
         (family_needs_work(plan) ? blk : 0) + kStatWords * sizeof(unsigned long long) + table_bytes(plan);
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
  const size_t al = region_align(plan);
  const size_t blk = round_up(family_bytes(plan), al);
  ctx->flags_bytes = round_up(kFlagsBytes, al);
  ctx->exch_bytes = blk;
  ctx->exch_slots = family_exch_slots(plan);
  ctx->parities = family_parities(plan);
  ctx->region_bytes = ctx->flags_bytes + (size_t)ctx->parities * ctx->exch_slots * blk;  // [slot][parity] buffers
  ctx->work_bytes = family_needs_work(plan) ? blk : 0;
  ctx->table_bytes = table_bytes(plan);
  CUDA_TRY(cudaMalloc(&ctx->region, ctx->region_bytes));
  ctx->staging_bytes = staging_bytes(plan, blk);
  if (ctx->staging_bytes && cudaMalloc(&ctx->staging, ctx->staging_bytes) != cudaSuccess) {
    // no room for staging images: this rank exchanges by direct peer stores,
    // and ctx_connect makes every rank do the same (programs must agree)
    cudaGetLastError();
    ctx->staging = nullptr;
    ctx->staging_bytes = 0;
  }
  CUDA_TRY(cudaMemset(ctx->region, 0, kFlagsBytes));
  if (ctx->work_bytes) CUDA_TRY(cudaMalloc(&ctx->work, ctx->work_bytes));
  CUDA_TRY(cudaMalloc(&ctx->dstat, kStatWords * sizeof(unsigned long long)));
  CUDA_TRY(cudaMemset(ctx->dstat, 0, kStatWords * sizeof(unsigned long long)));
  // twiddle tables w[m] = exp(-2 pi i m / n) in double, cast to T
  // (TwiddleTable, kernels.hpp:66-98); forward only: backward is conj(F(conj x))
  std::vector<int> tables;
  for (auto n64 : plan.dims) {
    const int n = (int)n64;
    if (!is_pow2(n) && !is_smooth(n) && !ctx->bluestein.count(n)) ctx->bluestein[n] = bluestein_tables(n, plan.prec);
    if (!is_pow2(n)) continue;
    tables.push_back(n);
  }
  {
    // half-length R2C / C2R lanes run n/2-point stages
    const int64_t nl = plan.dims.back();
    if (plan.kind != DFFTB_C2C && is_pow2(nl) && nl >= 16) tables.push_back((int)(nl / 2));
  }
  for (int n : tables) {
    if (ctx->twiddles.count(n)) continue;
    std::vector<std::complex<double>> w(n);
    for (int m = 0; m < n; ++m) {
      const double a = -2.0 * M_PI * (double)m / (double)n;
      w[m] = {std::cos(a), std::sin(a)};
    }
    ctx->twiddles[n] = upload_complex(w, plan.prec);
  }
  cudaStream_t side = nullptr, cap = nullptr, cpy = nullptr;
  CUDA_TRY(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  {
    int lo = 0, hi = 0;
    CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    for (int k = 0; k < kCopyStreams; ++k) {
      CUDA_TRY(cudaStreamCreateWithPriority(&cpy, cudaStreamNonBlocking, hi));
      ctx->copies.push_back(cpy);
    }
  }
  ctx->side = side;
  ctx->capture = cap;
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
  h->staged = ctx.staging != nullptr ? 1 : 0;
}

static void enable_peer(int dev, int peer) {
  if (dev == peer) return;
  int can = 0;
  CUDA_TRY(cudaDeviceCanAccessPeer(&can, dev, peer));
  if (!can) raise(DFFTB_Unsupported, "no peer access between devices");
  DeviceGuard g(dev);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) raise(DFFTB_CudaError, cudaGetErrorString(e));
  cudaGetLastError();
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
      enable_peer(ctx.device, (int)h.device);
      ctx.peer_region[r] = (void*)(uintptr_t)h.dptr;
    } else {
      cudaIpcMemHandle_t ih;
      std::memcpy(&ih, h.ipc, sizeof(ih));
      void* p = nullptr;
      CUDA_TRY(cudaIpcOpenMemHandle(&p, ih, cudaIpcMemLazyEnablePeerAccess));
      // peer access to the owner's device (when this process sees it under
      // the same ordinal): copy-engine DMAs into the mapping (staged
      // exchange) take the direct NVLink path only with it
      int ndev = 0, can = 0;
      cudaGetDeviceCount(&ndev);
      if (h.device != ctx.device && h.device >= 0 && h.device < ndev &&
          cudaDeviceCanAccessPeer(&can, ctx.device, (int)h.device) == cudaSuccess && can) {
        cudaError_t e = cudaDeviceEnablePeerAccess((int)h.device, 0);
        (void)e;
        cudaGetLastError();
      }
      ctx.peer_region[r] = p;
      ctx.peer_opened[r] = true;
    }
  }
  // the staged exchange changes the program structure: only if every rank has
  // its staging images
  bool all_staged = true;
  for (int r = 0; r < ctx.nranks; ++r) all_staged = all_staged && handles[r].staged;
  if (!all_staged && ctx.staging) {
    cudaFree(ctx.staging);
    ctx.staging = nullptr;
    ctx.staging_bytes = 0;
  }
  ctx.connected = true;
}

static void drop_programs(Ctx& ctx);

void ctx_destroy(Ctx* ctx) {
  if (!ctx) return;
  {
    DeviceGuard g(ctx->device);
    cudaDeviceSynchronize();
    drop_programs(*ctx);
    for (int r = 0; r < ctx->nranks; ++r)
      if (ctx->peer_opened[r]) cudaIpcCloseMemHandle(ctx->peer_region[r]);
    for (auto& kv : ctx->twiddles) cudaFree(kv.second);
    for (auto& kv : ctx->bluestein) {
      cudaFree(kv.second.first);
      cudaFree(kv.second.second);
    }
    for (void* e : ctx->events) cudaEventDestroy(static_cast<cudaEvent_t>(e));
    if (ctx->side) cudaStreamDestroy(static_cast<cudaStream_t>(ctx->side));
    if (ctx->capture) cudaStreamDestroy(static_cast<cudaStream_t>(ctx->capture));
    for (void* c : ctx->copies) cudaStreamDestroy(static_cast<cudaStream_t>(c));
    cudaFree(ctx->staging);
    cudaFree(ctx->region);
    cudaFree(ctx->work);
    cudaFree(ctx->dstat);
    cudaGetLastError();
  }
  delete ctx;
}

// Emulated P-rank world in ONE process: rank r's context on devices[r % n].
// With one device every rank's stages run in lockstep on one stream; with
// several devices the ranks' exchange stores cross NVLink through direct
// peer pointers and the sync points become cross-device event dependencies
// issued by the host (no kernel ever waits on another).
void world_create(const Plan& plan, const int* devices, int ndev, Ctx** out) {
  const int P = plan.nranks();
  if (ndev < 1) raise(DFFTB_ConfigInvalid, "need at least one device");
  std::vector<Ctx*> ctxs(P, nullptr);
  try {
    for (int r = 0; r < P; ++r) ctxs[r] = ctx_create(plan, r, devices[r % ndev]);
    for (int a = 0; a < ndev; ++a)
      for (int b = 0; b < ndev; ++b)
        if (devices[a] != devices[b]) enable_peer(devices[a], devices[b]);
  } catch (...) {
    for (auto* c : ctxs) ctx_destroy(c);
    throw;
  }
  for (int r = 0; r < P; ++r) {
    for (int q = 0; q < P; ++q) ctxs[r]->peer_region[q] = ctxs[q]->region;
    {
      // lockstep emulation issues no staged exchange
      DeviceGuard g(ctxs[r]->device);
      cudaFree(ctxs[r]->staging);
      ctxs[r]->staging = nullptr;
      ctxs[r]->staging_bytes = 0;
    }
    ctxs[r]->world_mode = true;
    ctxs[r]->connected = true;
    out[r] = ctxs[r];
  }
}

// ---------------------------------------------------------------- programs

enum class OpKind { Pass, Begin, Sync, Record, WaitEvent, Copy };

// One pitched 3-D box copied by the copy engine (staged exchange): the
// same box of two buffers with the same layout, innermost axis contiguous.
struct CopyBox {
  void* src = nullptr;
  void* dst = nullptr;
  size_t pitch = 0;      // bytes between rows
  size_t ysize = 0;      // rows per slice
  size_t pos[3] = {0, 0, 0};  // x bytes, y rows, z slices
  size_t ext[3] = {0, 0, 0};
  bool flat = false;     // full rows per slice: one 2-D copy of ext[1] * ext[2] rows
};

struct Op {
  OpKind kind = OpKind::Pass;
  int stream = 0;  // 0 caller's stream, 1 the context's side stream, 2 its copy stream
  // ---- pass
  bool tma = false;
  bool generic = false;  // non-power-of-two length: mixed-radix / Bluestein kernel
  bool adj = false;      // lanes along a strided axis
  bool remote = false;   // some destination is another rank's buffer
  int n = 1;
  int grid_sms = 0;      // > 0: persistent grid limited to this many SMs (overlap split)
  double share = 1.0;    // fraction of the pass's lanes this launch covers (chunks)
  PassParams p{};
  TmaPlan tp{};
  GenParams g{};
  // lane geometry (overlap chunking, spectral epilogue)
  int v = -1, ax_a = -1, ax_b = -1, ax_a1 = -1;
  int u = -1;                // exchange passes: the transpose's gather axis
  const Dist* before = nullptr;
  std::vector<int> members;  // exchange group (world ranks, group order)
  // exchange passes: this rank's block (before) and every member's target
  // block extents / element strides (staged exchange boxes)
  std::array<int64_t, kMaxDims> offb{}, lenb{};
  std::vector<std::array<int64_t, kMaxDims>> dlen, dstr;
  // ---- copy
  CopyBox cp{};
  // ---- sync point / events / begin
  bool signal = false, wait = false;
  int slot = 0;
  int event = 0;
  bool herm = false;  // Begin: clear the C2R statistics
};

struct Program {
  std::vector<Op> ops;
  bool c2r = false;
  bool multi_stream = false;
  int nevents = 0;
  int uses = 0;  // the first run issues directly (kernel attributes set), later runs replay a graph
  int64_t kernels = 0;  // dfftb kernels one replay of the graph launches
  cudaGraphExec_t graph = nullptr;
  bool graph_failed = false;
};

static void drop_programs(Ctx& ctx) {
  for (auto& r : ctx.recent) r = Ctx::Recent{};
  bool graphs = false;
  for (auto& kv : ctx.programs) graphs = graphs || kv.second->graph != nullptr;
  if (graphs) {
    // replays may still be queued: let them finish before their graphs go
    DeviceGuard g(ctx.device);
    cudaDeviceSynchronize();
  }
  for (auto& kv : ctx.programs)
    if (kv.second->graph) cudaGraphExecDestroy(kv.second->graph);
  ctx.programs.clear();
}

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

static void check_compatible(const Plan& plan, Ctx& ctx) {
  if (plan.nranks() != ctx.nranks) raise(DFFTB_GridMismatch, "communicator size must match the grid");
  if (plan.dims != ctx.dims || plan.grid != ctx.grid || plan.prec != ctx.prec || plan.decomp != ctx.decomp)
    raise(DFFTB_GridMismatch, "context was made for a different plan geometry");
  if (!ctx.connected) raise(DFFTB_ConfigInvalid, "context is not connected to its peers");
  if (std::find(ctx.checked_plans.begin(), ctx.checked_plans.end(), plan.id) != ctx.checked_plans.end()) return;
  if (family_bytes(plan) > ctx.exch_bytes) raise(DFFTB_ArenaExhausted, "context buffers are too small for this plan");
  ctx.checked_plans.push_back(plan.id);
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

static CUtensorMapL2promotion l2_promotion() {
  switch (knobs().l2promo) {
    case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    case 1: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 2: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
}

// the whole pass as one launch box
static void full_box(TmaArgs& a, const PassParams& p, int W) {
  a.W = W;
  a.na = p.A * (p.A1 > 1 ? p.A1 : 1);
  a.a0 = 0;
  a.bt0 = 0;
  a.nbt = (p.B + W - 1) / W;
  a.ntiles = (int64_t)a.na * a.nbt;
}

// Decide whether a pass can use the TMA-prefetch kernel and build its
// descriptor: a 3-D tensor map over (beta as reals, i, alpha) for strided
// lanes, or a flat bulk copy of W adjacent lanes for contiguous ones.
static bool plan_tma(Op& op, int prec) {
  const PassParams& p = op.p;
  const int n = op.n;
  if (!knobs().tma || n < 8 || (int64_t)p.A * p.B == 0) return false;
  const int W = tma_tile_w(prec, n);
  if (W <= 0) return false;
  const int csize = 2 * prec;
  if ((reinterpret_cast<uintptr_t>(p.in) & 15) != 0) return false;
  TmaPlan& tp = op.tp;
  std::memset(&tp, 0, sizeof(tp));
  tp.pdl = knobs().pdl ? 1 : 0;
  full_box(tp.args, p, W);
  if (p.A1 > 1 && (p.in_sa1 * (p.in_mode == kInReal ? prec : csize)) % 16) return false;
  if (op.adj) {
    if (p.in_mode != kInComplex) return false;
    if (p.A1 > 1) return false;  // 4-D strided lanes: direct kernel (3-D tensor map only)
    if ((2 * W * prec) % 16 != 0 || 2 * W > 256) return false;
    const int64_t si = p.in_si * csize, sa = (p.A > 1 ? p.in_sa : (int64_t)n * p.in_si) * csize;
    if (p.in_sb != 1) return false;
    if (si % 16 || sa % 16) {
      // rows a tensor map cannot describe (fp32 C2R user blocks: 129-bin
      // rows of 1032 bytes; a row-pair map, whose odd rows start 8 bytes off
      // a 16-byte boundary, raised an illegal-instruction fault): per-thread
      // 8-byte cp.async into the same tile
      if (csize != 8 || (reinterpret_cast<uintptr_t>(p.in) & 7) || !knobs().unaligned_ldgsts) return false;
      tp.args.bulk = 0;
      tp.args.ldgsts = 1;
      return true;
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
    CUresult r = enc(&tp.tmap, prec == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                     const_cast<void*>(p.in), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
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
  if (p.in_sb >= lane_elems && p.in_sb <= n && lane_bytes % 16 == 0) {
    if (p.A > 1 && (p.in_sa * esize) % 16) return false;
    tp.args.bulk = 1;
    tp.args.lane_bytes = (int)lane_bytes;
    // R2C / C2R lanes as half-length complex FFTs: twice the
    // lanes per tile, half the butterflies; needs the n/2-point table
    // (tw2 set) and, for C2R, one destination
    const bool half = knobs().rhalf && p.in_mode != kInComplex && n >= 16 && p.tw2 != nullptr &&
                      p.spec.op == 0 && (p.in_mode == kInReal || (p.ndest == 1 && p.store_mode == 0)) &&
                      (p.in_mode == kInReal ? lane_bytes <= (int64_t)(n / 2) * csize
                                            : lane_bytes <= (int64_t)(n / 2 + kC2RhExtra) * csize);
    if (half) {
      tp.args.rhalf = 1;
      full_box(tp.args, p, tma_tile_w_halfreal(prec, n / 2));
    }
    return true;
  }
  return false;
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
    if (d.base != p.dest[0].base || d.sa != p.dest[0].sa || d.sb != p.dest[0].sb || d.sk != p.dest[0].sk ||
        d.sa1 != p.dest[0].sa1)
      return;
  }
  p.store_mode = 1;
  p.oshift = ilog2((int)b);
  p.omask = (int)b - 1;
}

// Half-length R2C / C2R lanes run n/2-point Stockham stages (tw = the
// n/2-point table) around a pre- / post-twiddle (tw2 = the n-point table)
static void plan_twiddles(Op& op, const Ctx& ctx) {
  if (op.tma && op.tp.args.rhalf) op.p.tw = ctx.twiddles.at(op.n / 2);
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

// One local pass of a 3-D block: axis v of the buffer `in` (extents len,
// element strides si) into `out` (strides so over the output extents).
static Op single_pass(const Ctx& ctx, int v, int n, const int64_t* len, const int64_t* si, const void* in,
                      void* out, const int64_t* so, int fkind, double scale, bool inverse = true) {
  int lanes[2], nl = 0;
  for (int a = 0; a < 3; ++a)
    if (a != v) lanes[nl++] = a;
  const int ax_a = lanes[0], ax_b = lanes[1];
  Op op;
  op.v = v;
  op.ax_a = ax_a;
  op.ax_b = ax_b;
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
  p.inverse = inverse;
  p.scale = scale;
  p.tw = is_pow2(n) ? ctx.twiddles.at(n) : nullptr;
  p.tw2 = is_pow2(n) && n >= 16 && ctx.twiddles.count(n / 2) ? p.tw : nullptr;
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
  plan_twiddles(op, ctx);
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
  if (plan.nranks() != 1 || plan.input.ndim() != 3 || !knobs().zperm || !knobs().single_reorder) return false;
  bool backward = false, c2r = false, r2c = false;
  double scale = 1.0;
  const Stage* last_fft = nullptr;
  for (const auto& st : plan.stages) {
    if (st.type == StageType::Fft) {
      backward = st.dir == DFFTB_BACKWARD;
      if (st.fkind == DFFTB_C2R) c2r = true;
      if (st.fkind == DFFTB_R2C) r2c = true;
      last_fft = &st;
    } else if (st.type == StageType::Normalize) {
      scale = st.factor;
    }
  }
  if (r2c && knobs().r2c_order) {
    // R2C forward, mirror of the C2R backward: F2 (R2C) -> [x1][x0][x2]
    // buffer -> F0 -> plain buffer -> F1 -> user block.  The last pass writes
    // the user's odd-length (n/2+1) rows with the wide tiles of the middle
    // axis instead of the 4-lane tiles of a long axis 0 (2048x512x256 fp32:
    // 32-byte row pieces off the 32-byte sector grid), and axis 0 writes an
    // aligned internal buffer.
    int64_t off[3], lr[3], lc[3];
    plan.input.extents_of(0, off, lr);
    plan.output.extents_of(0, off, lc);
    for (int a = 0; a < 3; ++a)
      if (lc[a] <= 0 || lr[a] <= 0) return false;
    const int prec = ctx.prec;
    void* b1 = ctx.exch(0, 0, parity);
    void* b2 = ctx.exch(0, 1, parity);
    int64_t s_real[3], s_plain[3], s_swap[3], s_user[3];
    row_major_strides(lr, 3, s_real, false, prec);
    row_major_strides(lc, 3, s_plain, true, prec);
    row_major_strides(lc, 3, s_swap, true, prec, true);
    row_major_strides(lc, 3, s_user, false, prec);
    prog.push_back(single_pass(ctx, 2, (int)lr[2], lr, s_real, d_in, b1, s_swap, DFFTB_R2C, 1.0, false));
    prog.push_back(single_pass(ctx, 0, (int)lc[0], lc, s_swap, b1, b2, s_plain, DFFTB_C2C, 1.0, false));
    prog.push_back(single_pass(ctx, 1, (int)lc[1], lc, s_plain, b2, d_out, s_user, DFFTB_C2C, 1.0, false));
    // spectral epilogue coordinates: the (hatted) layout of the last stage
    if (last_fft) prog.back().before = &last_fft->before;
    return true;
  }
  if (r2c || !backward) return false;
  int64_t off[3], lc[3], lr[3];
  plan.input.extents_of(0, off, lc);   // complex (Hermitian for C2R) extents
  plan.output.extents_of(0, off, lr);  // output extents
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

// One rank's program: fused passes and sync points, in stage order.
static bool staged_applies(const Plan& plan, const Ctx& ctx);

static std::vector<Op> lower(const Plan& plan, const Ctx& ctx, const void* d_in, void* d_out, int parity) {
  std::vector<Op> prog;
  if (lower_single(plan, ctx, d_in, d_out, parity, prog)) return prog;
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
    p.tw2 = is_pow2(n) && n >= 16 && ctx.twiddles.count(n / 2) ? p.tw : nullptr;
    p.herm = ctx.dstat;
    op.adj = p.in_si != 1;
    if (lenb[v] == 0 && st.fkind != DFFTB_C2R) p.A = 0;

    if (tr) {
      const Dist& Lo = tr->after;
      const int g = tr->grid_axis;
      const int u = tr->before.axis_of_grid[g];
      // the transposed final forward exchange feeds the axis-0 pass: store
      // its buffer [x1][x0][rest] so axis-0 lanes read short strides
      const bool swap_out = tr->transposed && knobs().zperm && nd >= 3 && !(staged_applies(plan, ctx) && knobs().dma_flat);
      op.u = u;
      op.members = group_members(Lo, me, g);
      op.remote = op.members.size() > 1;
      p.ndest = (int)op.members.size();
      p.oblk = (Lo.dims[v] + Lo.grid[g] - 1) / Lo.grid[g];
      for (int a = 0; a < nd; ++a) {
        op.offb[a] = offb[a];
        op.lenb[a] = lenb[a];
      }
      op.dlen.resize(p.ndest);
      op.dstr.resize(p.ndest);
      for (int q = 0; q < p.ndest; ++q) {
        const int rq = op.members[q];
        int64_t offo[kMaxDims], leno[kMaxDims], so[kMaxDims];
        Lo.extents_of(rq, offo, leno);
        row_major_strides(leno, nd, so, true, ctx.prec, swap_out);
        for (int a = 0; a < nd; ++a) {
          op.dlen[q][a] = leno[a];
          op.dstr[q][a] = so[a];
        }
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
      plan_twiddles(op, ctx);
      plan_generic(op, ctx);
      prog.push_back(op);
      if (op.remote) {
        Op b;
        b.kind = OpKind::Sync;
        b.signal = b.wait = true;
        b.members = op.members;
        prog.push_back(b);
      }
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
      if (!last_fft && !out) raise(DFFTB_ArenaExhausted, "context has no work buffer for this plan");
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
      plan_twiddles(op, ctx);
      plan_generic(op, ctx);
      prog.push_back(op);
      cur = out;
      cur_internal = !last_fft;
      cur_swap01 = false;
      i += nm ? 2 : 1;
    }
  }
  return prog;
}

// ----------------------------------------------------------------- overlap
//
// [P: exchange pass] [sync] [Q: local pass] -> chunks c = 0..C-1 along the
// lane axis X both passes share (neither transforms it, and the exchange does
// not redistribute it, so every group member's chunk c covers the same global
// X range).  P's chunk c stores, then signals sync point k_c to the group;
// Q's chunk c waits for P's chunk c locally (event) and for the group's
// signals (remote), on the side stream.  The SMs are split so the two run
// concurrently: P needs enough to keep NVLink busy, Q takes the rest.

// Rank-independent shape test: every rank must derive the same op and sync
// sequence (sync slots are numbered in program order), so nothing that
// depends on this rank's block (sizes, buffer alignment, TMA planning) may
// decide whether a pair is chunked.
static bool overlap_shape(const Op& o) {
  return o.kind == OpKind::Pass && is_pow2(o.n) && o.before && o.before->ndim() == 3 && o.p.A1 <= 1 &&
         o.p.in_mode == kInComplex && !o.p.out_real;
}

// SM share of the exchange pass: both passes finish together when
// max(P's HBM-pass time on g SMs, its NVLink time) = Q's time on 148 - g SMs.
static int overlap_split(const Op& P, const Op& Q, int prec, int sms) {
  if (knobs().frac > 0.0 && knobs().frac < 1.0) return std::max(1, (int)(knobs().frac * sms + 0.5));
  const double csize = 2.0 * prec;
  const double hbm = 6.2e12, nvl = 0.70e12;  // measured pass rate and NVLink store rate (B200)
  auto bytes = [&](const Op& o) {
    const double lanes = (double)o.p.A * o.p.B;
    const double in_e = o.p.in_mode == kInReal ? 0.5 : 1.0, out_e = o.p.out_real ? 0.5 : 1.0;
    return lanes * (o.n * in_e + o.p.n_out * out_e) * csize;
  };
  const double tp = bytes(P) / hbm, tq = bytes(Q) / hbm;
  const double remote = (double)P.p.A * P.p.B * P.p.n_out * csize * (double)(P.members.size() - 1) /
                        (double)P.members.size();
  const double tn = remote / nvl;
  int best = sms / 2;
  double bt = 1e30;
  for (int g = 8; g <= sms - 8; ++g) {
    const double t = std::max(std::max(tp * sms / g, tn), tq * sms / (sms - g));
    if (t < bt) {
      bt = t;
      best = g;
    }
  }
  return best;
}

// chunk c of a pass as a launch box (X on the alpha or the beta axis)
static TmaArgs chunk_box(const Op& o, int X, int64_t x0, int64_t x1, int W) {
  TmaArgs a = o.tp.args;
  const int nbt_all = (o.p.B + W - 1) / W;
  if (X == o.ax_a) {
    a.a0 = (int)x0;
    a.na = (int)(x1 - x0);
    a.bt0 = 0;
    a.nbt = nbt_all;
  } else {
    a.a0 = 0;
    a.na = o.p.A;
    a.bt0 = (int)(x0 / W);
    a.nbt = (int)((x1 - x0 + W - 1) / W);
  }
  a.ntiles = (int64_t)a.na * a.nbt;
  return a;
}

static void overlap_pairs(std::vector<Op>& prog, const Plan& plan, const Ctx& ctx, int& nevents) {
  const bool pipelined = plan.options.exchange == DFFTB_EXCHANGE_PIPELINED;
  if (knobs().overlap == 0 || (knobs().overlap < 0 && !pipelined) || ctx.world_mode || ctx.nranks < 2) return;
  int C = knobs().chunks;
  if (pipelined && plan.options.chunks_per_peer > 1) C = std::min(16, plan.options.chunks_per_peer);
  if (C < 2) return;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx.device);
  const int me = ctx.rank;
  std::vector<Op> out;
  size_t i = 0;
  while (i < prog.size()) {
    bool pattern = i + 2 < prog.size() && overlap_shape(prog[i]) && prog[i].remote &&
                   prog[i + 1].kind == OpKind::Sync && overlap_shape(prog[i + 2]) && !prog[i + 2].remote &&
                   prog[i + 2].p.ndest == 1;
    // the chunk axis X: transformed by neither pass and not moved by the
    // exchange (X != the gather axis u), so every group member's chunk c
    // covers the same global range
    const int X = pattern ? 3 - prog[i].v - prog[i + 2].v : -1;
    pattern = pattern && prog[i].v != prog[i + 2].v && X >= 0 && X < 3 && X != prog[i].u &&
              (X == prog[i].ax_a || X == prog[i].ax_b) && (X == prog[i + 2].ax_a || X == prog[i + 2].ax_b);
    if (!pattern) {
      out.push_back(prog[i++]);
      continue;
    }
    const Op& P = prog[i];
    const Op& S = prog[i + 1];
    const Op& Q = prog[i + 2];
    // this rank's chunking (its own block; empty chunks still signal)
    int64_t offQ[kMaxDims], lenQ[kMaxDims];
    Q.before->extents_of(me, offQ, lenQ);
    const int64_t Xe = lenQ[X];
    const bool p_box = P.tma && !P.generic, q_box = Q.tma && !Q.generic;  // box launches need the TMA kernel
    int64_t unit = 1;
    if (p_box && X == P.ax_b) unit = std::max<int64_t>(unit, P.tp.args.W);
    if (q_box && X == Q.ax_b) unit = std::max<int64_t>(unit, Q.tp.args.W);
    const int64_t R = std::max<int64_t>(1, ((Xe + C - 1) / C + unit - 1) / unit * unit);
    const int gP = overlap_split(P, Q, ctx.prec, sms);
    for (int c = 0; c < C; ++c) {
      const int64_t x0 = std::min<int64_t>(Xe, c * R), x1 = std::min<int64_t>(Xe, x0 + R);
      if (p_box || c == 0) {
        Op pc = P;  // without box support the whole pass runs in chunk 0
        if (p_box) {
          pc.tp.args = chunk_box(P, X, x0, x1, P.tp.args.W);
          pc.share = Xe > 0 ? (double)(x1 - x0) / (double)Xe : 0.0;
        }
        pc.grid_sms = gP;
        if (!p_box || x1 > x0) out.push_back(pc);
      }
      Op sig;
      sig.kind = OpKind::Sync;
      sig.signal = true;
      sig.members = S.members;
      out.push_back(sig);
      Op rec;
      rec.kind = OpKind::Record;
      rec.event = nevents + c;
      out.push_back(rec);
      Op we;
      we.kind = OpKind::WaitEvent;
      we.stream = 1;
      we.event = nevents + c;
      out.push_back(we);
      Op wt;
      wt.kind = OpKind::Sync;
      wt.stream = 1;
      wt.wait = true;
      wt.members = S.members;
      out.push_back(wt);  // signal and wait of chunk c share a sync slot (assign_slots)
      if (q_box || c == C - 1) {
        Op qc = Q;  // without box support the whole pass runs after the last chunk
        qc.stream = 1;
        if (q_box) {
          qc.tp.args = chunk_box(Q, X, x0, x1, Q.tp.args.W);
          qc.share = Xe > 0 ? (double)(x1 - x0) / (double)Xe : 0.0;
        }
        qc.grid_sms = sms - gP;
        if (!q_box || x1 > x0) out.push_back(qc);
      }
    }
    // join: the caller's stream waits for the side stream
    Op rj;
    rj.kind = OpKind::Record;
    rj.stream = 1;
    rj.event = nevents + C;
    out.push_back(rj);
    Op wj;
    wj.kind = OpKind::WaitEvent;
    wj.event = nevents + C;
    out.push_back(wj);
    nevents += C + 1;
    i += 3;
  }
  prog.swap(out);
}

// ---------------------------------------------------------- staged exchange
//
// The default exchange of Blocking / Staged plans (DFFTB_DMA=0 turns it off;
// Pipelined plans use overlap_pairs above), after the staging hop of
// staged_all_to_all (exchange.hpp:225-246).  The same [P: exchange pass]
// [sync][Q: local pass] triple, in C chunks along the same shared lane axis X
// as above, becomes
//   caller's stream: P chunk 0 .. C-1 on every SM, storing the other
//     members' parts into local staging images of their buffers (same
//     layout and offsets) and its own part into its own buffer -- HBM-speed
//     stores only;  then per chunk c: wait for sync point k_c, Q chunk c on
//     every SM;
//   copy stream c % 2: wait for P chunk c, copy chunk c's box of every
//     staging image into that member's buffer (one pitched 2-D DMA per member
//     over NVLink), signal k_c to the group.
// No SM ever stalls on NVLink: the copy engines stream chunk c while the SMs
// run P's later chunks and Q's earlier ones.  The op and sync sequence is
// rank-independent (C signals and C waits per triple, staged or not decided
// from global sizes); chunk ranges are multiples of 64 lanes along a tile
// axis, which every tile width divides.

// staging images: one buffer per other member of the largest exchange group
static size_t staging_bytes(const Plan& plan, size_t blk) {
  if (plan.nranks() < 2 || knobs().dma <= 0) return 0;
  int g = 1;
  for (int x : plan.grid) g = std::max(g, x);
  return (size_t)(g - 1) * blk;
}

static bool staged_applies(const Plan& plan, const Ctx& ctx) {
  return knobs().dma > 0 && plan.options.exchange != DFFTB_EXCHANGE_PIPELINED && !ctx.world_mode &&
         ctx.nranks > 1 && plan.nranks() > 1 && ctx.staging != nullptr;
}

// chunk c's box of member q's buffer written by this rank's exchange pass
static bool staged_box(const Op& P, int q, int X, int64_t x0, int64_t x1, int csize, CopyBox& cb) {
  int64_t lo[3], hi[3];
  for (int a = 0; a < 3; ++a) {
    if (a == P.u) {
      lo[a] = P.offb[a];
      hi[a] = P.offb[a] + P.lenb[a];
    } else if (a == P.v) {
      lo[a] = 0;
      hi[a] = P.dlen[q][a];
    } else {
      lo[a] = x0;
      hi[a] = x1;
    }
    if (hi[a] <= lo[a]) return false;
  }
  (void)X;
  int ord[3] = {0, 1, 2};  // D, H, W: strides descending
  std::sort(ord, ord + 3, [&](int a, int b) { return P.dstr[q][a] > P.dstr[q][b]; });
  const int D = ord[0], H = ord[1], W = ord[2];
  const auto& st = P.dstr[q];
  if (st[W] != 1 || st[H] < P.dlen[q][W] || st[D] % st[H] != 0) raise(DFFTB_Unsupported, "staged box layout");
  cb.pitch = (size_t)st[H] * csize;
  cb.ysize = (size_t)(st[D] / st[H]);
  cb.pos[0] = (size_t)lo[W] * csize;
  cb.pos[1] = (size_t)lo[H];
  cb.pos[2] = (size_t)lo[D];
  cb.ext[0] = (size_t)(hi[W] - lo[W]) * csize;
  cb.ext[1] = (size_t)(hi[H] - lo[H]);
  cb.ext[2] = (size_t)(hi[D] - lo[D]);
  cb.flat = cb.ext[1] == cb.ysize || cb.ext[2] == 1;
  return true;
}

static void staged_pairs(std::vector<Op>& prog, const Plan& plan, const Ctx& ctx, int& nevents) {
  if (!staged_applies(plan, ctx)) return;
  int C = knobs().dma_chunks;
  if (plan.options.chunks_per_peer > 1) C = std::min(16, plan.options.chunks_per_peer);
  C = std::max(1, C);
  const int me = ctx.rank;
  const int csize = 2 * ctx.prec;
  std::vector<Op> out;
  size_t i = 0;
  while (i < prog.size()) {
    bool pattern = i + 2 < prog.size() && overlap_shape(prog[i]) && prog[i].remote &&
                   prog[i + 1].kind == OpKind::Sync && overlap_shape(prog[i + 2]) && !prog[i + 2].remote &&
                   prog[i + 2].p.ndest == 1;
    const int X = pattern ? 3 - prog[i].v - prog[i + 2].v : -1;
    pattern = pattern && prog[i].v != prog[i + 2].v && X >= 0 && X < 3 && X != prog[i].u &&
              (X == prog[i].ax_a || X == prog[i].ax_b) && (X == prog[i + 2].ax_a || X == prog[i + 2].ax_b);
    if (pattern) {
      // worth it?  DMA launches cost microseconds and short rows slow the
      // copy engine: stage only big blocks whose chunk rows stay long.
      // Decided from global sizes only (every rank must agree).
      const Dist& B = *prog[i].before;
      double elems = 1.0;
      for (auto d : B.dims) elems *= (double)d;
      const double per_rank = elems * csize / (double)plan.nranks();
      const int gx = B.grid_axis_of(X);
      const int64_t Xg = gx < 0 ? B.dims[X] : (B.dims[X] + B.grid[gx] - 1) / B.grid[gx];
      const bool x_inner = X == B.ndim() - 1;  // receiver rows are X-chunks
      const int64_t u = (X == prog[i].ax_b || X == prog[i + 2].ax_b) ? 64 : 1;
      const int64_t Rg = ((Xg + C - 1) / C + u - 1) / u * u;
      // groups of more than two: direct peer stores reach several peers at
      // once and win (512^3 on 4 GPUs, slab 4 / pencil 1x4: 1.95 direct vs
      // 2.5-2.6 ms staged, profiles/r2/group_probe_s76.txt)
      const bool small_group = (int)prog[i].members.size() <= knobs().dma_max_group;
      pattern = small_group && per_rank >= knobs().dma_min_mb * 1048576.0 &&
                (!x_inner || Rg * csize >= knobs().dma_min_row);
    }
    if (!pattern) {
      out.push_back(prog[i++]);
      continue;
    }
    const Op& P = prog[i];
    const Op& S = prog[i + 1];
    const Op& Q = prog[i + 2];
    int64_t offQ[kMaxDims], lenQ[kMaxDims];
    Q.before->extents_of(me, offQ, lenQ);
    const int64_t Xe = lenQ[X];
    const bool p_box = P.tma && !P.generic && (X != P.ax_b || 64 % P.tp.args.W == 0);
    const bool q_box = Q.tma && !Q.generic && (X != Q.ax_b || 64 % Q.tp.args.W == 0);
    const int64_t unit = (X == P.ax_b || X == Q.ax_b) ? 64 : 1;
    const int64_t R = std::max<int64_t>(1, ((Xe + C - 1) / C + unit - 1) / unit * unit);
    // P with the other members' destinations redirected to staging images
    Op Ps = P;
    std::vector<void*> image(P.members.size(), nullptr);
    {
      int m = 0;
      for (size_t q = 0; q < P.members.size(); ++q) {
        if (P.members[q] == me) continue;
        image[q] = static_cast<char*>(ctx.staging) + (size_t)m++ * ctx.exch_bytes;
        Ps.p.dest[q].ptr = image[q];
      }
    }
    const int ncs = knobs().dma_streams;
    for (int c = 0; c < C; ++c) {
      const int64_t x0 = std::min<int64_t>(Xe, c * R), x1 = std::min<int64_t>(Xe, x0 + R);
      const int cs = 2 + c % ncs;  // copy stream of chunk c
      if (p_box || c == 0) {
        Op pc = Ps;  // without box support the whole pass runs in chunk 0
        if (p_box) {
          pc.tp.args = chunk_box(Ps, X, x0, x1, Ps.tp.args.W);
          pc.share = Xe > 0 ? (double)(x1 - x0) / (double)Xe : 0.0;
        }
        if (!p_box || x1 > x0) out.push_back(pc);
      }
      Op rec;
      rec.kind = OpKind::Record;
      rec.event = nevents + c;
      out.push_back(rec);
      Op we;
      we.kind = OpKind::WaitEvent;
      we.stream = cs;
      we.event = nevents + c;
      out.push_back(we);
      for (size_t q = 0; q < P.members.size(); ++q) {
        if (!image[q]) continue;
        Op cp;
        cp.kind = OpKind::Copy;
        cp.stream = cs;
        if (!staged_box(P, (int)q, X, x0, x1, csize, cp.cp)) continue;
        cp.cp.src = image[q];
        cp.cp.dst = P.p.dest[q].ptr;
        out.push_back(cp);
      }
      Op sig;
      sig.kind = OpKind::Sync;
      sig.stream = cs;
      sig.signal = true;
      sig.members = S.members;
      out.push_back(sig);
    }
    for (int c = 0; c < C; ++c) {
      const int64_t x0 = std::min<int64_t>(Xe, c * R), x1 = std::min<int64_t>(Xe, x0 + R);
      Op wt;
      wt.kind = OpKind::Sync;
      wt.wait = true;
      wt.members = S.members;
      out.push_back(wt);
      if (q_box || c == C - 1) {
        Op qc = Q;  // without box support the whole pass runs after the last chunk
        if (q_box) {
          qc.tp.args = chunk_box(Q, X, x0, x1, Q.tp.args.W);
          qc.share = Xe > 0 ? (double)(x1 - x0) / (double)Xe : 0.0;
        }
        if (!q_box || x1 > x0) out.push_back(qc);
      }
    }
    // join: the caller's stream waits for the copy streams (the staging
    // images are rewritten by the next exchange pass)
    for (int k = 0; k < ncs; ++k) {
      Op rj;
      rj.kind = OpKind::Record;
      rj.stream = 2 + k;
      rj.event = nevents + C + k;
      out.push_back(rj);
      Op wj;
      wj.kind = OpKind::WaitEvent;
      wj.event = nevents + C + k;
      out.push_back(wj);
    }
    nevents += C + ncs;
    i += 3;
  }
  prog.swap(out);
}

// Sync slots: every barrier gets its own slot; a signal-only point and the
// wait-only point that consumes it share one (first in, first out).
static void assign_slots(std::vector<Op>& prog) {
  int next = 0;
  std::vector<int> open;
  size_t head = 0;
  for (auto& o : prog) {
    if (o.kind != OpKind::Sync) continue;
    if (o.signal && o.wait) {
      o.slot = next++;
    } else if (o.signal) {
      o.slot = next++;
      open.push_back(o.slot);
    } else {
      if (head >= open.size()) raise(DFFTB_ConfigInvalid, "sync wait without a signal");
      o.slot = open[head++];
    }
  }
  if (next > kSyncSlots) raise(DFFTB_Unsupported, "too many sync points in one program");
}

static bool plan_has_c2r(const Plan& plan) {
  for (const auto& st : plan.stages)
    if (st.type == StageType::Fft && st.fkind == DFFTB_C2R) return true;
  return false;
}

static std::shared_ptr<Program> build_program(const Plan& plan, Ctx& ctx, const void* d_in, void* d_out,
                                              int parity, bool allow_overlap = true) {
  auto pr = std::make_shared<Program>();
  std::vector<Op> ops = lower(plan, ctx, d_in, d_out, parity);
  if (allow_overlap) {
    staged_pairs(ops, plan, ctx, pr->nevents);
    overlap_pairs(ops, plan, ctx, pr->nevents);
  }
  assign_slots(ops);
  pr->c2r = plan_has_c2r(plan);
  bool has_sync = false;
  for (const auto& o : ops) {
    has_sync = has_sync || o.kind == OpKind::Sync;
    pr->multi_stream = pr->multi_stream || o.stream == 1;
  }
  if (pr->c2r || (has_sync && !ctx.world_mode)) {
    Op b;
    b.kind = OpKind::Begin;
    b.herm = pr->c2r;
    pr->ops.push_back(b);
  }
  for (auto& o : ops) pr->ops.push_back(std::move(o));
  return pr;
}

static cudaEvent_t event_at(Ctx& ctx, int i) {
  while ((int)ctx.events.size() <= i) {
    DeviceGuard g(ctx.device);  // events belong to the context's device
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx.events.push_back(e);
  }
  return static_cast<cudaEvent_t>(ctx.events[i]);
}

static SyncParams sync_params(const Ctx& ctx, const Op& op) {
  SyncParams sp{};
  sp.nmem = (int)op.members.size();
  for (int i = 0; i < sp.nmem; ++i) {
    sp.members[i] = op.members[i];
    sp.peer_flags[i] = reinterpret_cast<unsigned long long*>(ctx.flags_of(op.members[i]));
  }
  sp.me = ctx.rank;
  sp.slot = op.slot;
  sp.signal = op.signal;
  sp.wait = op.wait;
  sp.my_flags = reinterpret_cast<unsigned long long*>(ctx.flags_of(ctx.rank));
  sp.epoch = ctx.dstat + kStatEpoch;
  sp.timeout_ns = kSyncTimeoutNs;
  sp.timeout_flag = ctx.dstat + 2;
  return sp;
}

static cudaStream_t op_stream(const Ctx& ctx, const Op& op, cudaStream_t s) {
  if (op.stream == 1) return static_cast<cudaStream_t>(ctx.side);
  if (op.stream >= 2) return static_cast<cudaStream_t>(ctx.copies[op.stream - 2]);
  return s;
}

// Issue one op.  `s` = the caller's stream (or the capture stream).
static void launch_op(Ctx& ctx, const Op& op, cudaStream_t s) {
  cudaStream_t st = op_stream(ctx, op, s);
  switch (op.kind) {
    case OpKind::Copy: {
      if (op.cp.flat) {
        // whole slices (or one slice): one pitched 2-D DMA
        const size_t off = (op.cp.pos[2] * op.cp.ysize + op.cp.pos[1]) * op.cp.pitch + op.cp.pos[0];
        CUDA_TRY(cudaMemcpy2DAsync(static_cast<char*>(op.cp.dst) + off, op.cp.pitch,
                                   static_cast<const char*>(op.cp.src) + off, op.cp.pitch, op.cp.ext[0],
                                   op.cp.ext[1] * op.cp.ext[2], cudaMemcpyDefault, st));
        return;
      }
      cudaMemcpy3DParms m{};
      m.srcPtr = make_cudaPitchedPtr(op.cp.src, op.cp.pitch, op.cp.pitch, op.cp.ysize);
      m.dstPtr = make_cudaPitchedPtr(op.cp.dst, op.cp.pitch, op.cp.pitch, op.cp.ysize);
      m.srcPos = make_cudaPos(op.cp.pos[0], op.cp.pos[1], op.cp.pos[2]);
      m.dstPos = m.srcPos;
      m.extent = make_cudaExtent(op.cp.ext[0], op.cp.ext[1], op.cp.ext[2]);
      m.kind = cudaMemcpyDefault;
      CUDA_TRY(cudaMemcpy3DAsync(&m, st));
      return;
    }
    case OpKind::Begin:
      CUDA_TRY(launch_sync_begin(ctx.dstat + kStatEpoch, op.herm ? ctx.dstat : nullptr, st));
      return;
    case OpKind::Sync:
      if (ctx.world_mode) return;  // lockstep emulation: ordering comes from the host
      CUDA_TRY(launch_sync_point(sync_params(ctx, op), st));
      return;
    case OpKind::Record:
      CUDA_TRY(cudaEventRecord(event_at(ctx, op.event), st));
      return;
    case OpKind::WaitEvent:
      CUDA_TRY(cudaStreamWaitEvent(st, event_at(ctx, op.event), 0));
      return;
    case OpKind::Pass:
      break;
  }
  if ((int64_t)op.p.A * op.p.B == 0) return;
  if (op.generic) CUDA_TRY(launch_generic(ctx.prec, op.g, st));
  else if (op.tma) {
    if (op.tp.args.ntiles > 0) CUDA_TRY(launch_pass_tma(ctx.prec, op.n, op.p, op.adj, op.tp, op.grid_sms, st));
  } else CUDA_TRY(launch_pass(ctx.prec, op.n, op.p, op.adj, st));
}

// The side stream joins the caller's stream at the start of a program (it
// must not run ahead of what the caller enqueued before).
static void fork_side(Ctx& ctx, const Program& pr, cudaStream_t s) {
  if (!pr.multi_stream) return;
  cudaEvent_t e = event_at(ctx, pr.nevents);
  CUDA_TRY(cudaEventRecord(e, s));
  CUDA_TRY(cudaStreamWaitEvent(static_cast<cudaStream_t>(ctx.side), e, 0));
}

static void issue_program(Ctx& ctx, Program& pr, cudaStream_t s) {
  fork_side(ctx, pr, s);
  for (const auto& op : pr.ops) launch_op(ctx, op, s);
}

// Replay through a CUDA graph (captured on first use).  Falls back to direct
// issue if capture is not possible (e.g. the caller's stream is itself being
// captured).
static void run_graph(Ctx& ctx, Program& pr, cudaStream_t s) {
  if (pr.uses++ == 0) {
    issue_program(ctx, pr, s);
    return;
  }
  if (!pr.graph && !pr.graph_failed) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    if (cs != cudaStreamCaptureStatusNone) {
      issue_program(ctx, pr, s);
      return;
    }
    cudaStream_t cap = static_cast<cudaStream_t>(ctx.capture);
    cudaGraph_t graph = nullptr;
    CUDA_TRY(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    const uint64_t before = launch_count();
    try {
      issue_program(ctx, pr, cap);
      pr.kernels = (int64_t)(launch_count() - before);
      add_launches(-pr.kernels);  // captured, not executed
    } catch (...) {
      cudaStreamEndCapture(cap, &graph);
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      throw;
    }
    cudaError_t e = cudaStreamEndCapture(cap, &graph);
    if (e == cudaSuccess && graph) e = cudaGraphInstantiate(&pr.graph, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    if (e != cudaSuccess || !pr.graph) {
      cudaGetLastError();
      pr.graph = nullptr;
      pr.graph_failed = true;
    }
  }
  if (pr.graph) {
    CUDA_TRY(cudaGraphLaunch(pr.graph, s));
    add_launches(pr.kernels);
  } else {
    issue_program(ctx, pr, s);
  }
}

static std::string program_key(const Plan& plan, const void* d_in, const void* d_out, int parity,
                               const char* extra = "") {
  char buf[160];
  snprintf(buf, sizeof(buf), "%llu:%p:%p:%d:%s", (unsigned long long)plan.id, d_in, d_out, parity, extra);
  return buf;
}

static Program& cached_program(const Plan& plan, Ctx& ctx, const void* d_in, void* d_out, int parity,
                               const std::string& key) {
  auto it = ctx.programs.find(key);
  if (it != ctx.programs.end()) return *it->second;
  if (ctx.programs.size() >= kMaxCachedPrograms) drop_programs(ctx);
  auto pr = build_program(plan, ctx, d_in, d_out, parity);
  return *ctx.programs.emplace(key, pr).first->second;
}

// Per-op device times (TimingBreakdown, timing.hpp:16-37): local passes ->
// local_fft; exchange passes (FFT with the pack / all_to_all / unpack fused
// into their stores) and sync points -> wire_comm; pack, unpack and
// staging_copy stay 0 (no separate passes exist).  Ops on the side stream
// overlap the caller's, so the components may sum to more than `total`.
static void run_timed(Ctx& ctx, Program& pr, cudaStream_t s, dfftb_timing* timers) {
  struct Mark {
    cudaEvent_t a, b;
    const Op* op;
  };
  // every event created here is destroyed on every exit path
  struct Events {
    std::vector<cudaEvent_t> all;
    ~Events() {
      for (auto e : all) cudaEventDestroy(e);
    }
    cudaEvent_t make() {
      cudaEvent_t e = nullptr;
      CUDA_TRY(cudaEventCreate(&e));
      all.push_back(e);
      return e;
    }
  } evs;
  std::vector<Mark> marks;
  cudaEvent_t t0 = evs.make(), t1 = evs.make();
  CUDA_TRY(cudaEventRecord(t0, s));
  fork_side(ctx, pr, s);
  for (const auto& op : pr.ops) {
    const bool timed =
        op.kind == OpKind::Pass || op.kind == OpKind::Copy || (op.kind == OpKind::Sync && !ctx.world_mode);
    cudaStream_t st = op_stream(ctx, op, s);
    Mark m{nullptr, nullptr, &op};
    if (timed) {
      m.a = evs.make();
      m.b = evs.make();
      CUDA_TRY(cudaEventRecord(m.a, st));
    }
    launch_op(ctx, op, s);
    if (timed) {
      CUDA_TRY(cudaEventRecord(m.b, st));
      marks.push_back(m);
    }
  }
  CUDA_TRY(cudaEventRecord(t1, s));
  CUDA_TRY(cudaEventSynchronize(t1));
  std::memset(timers, 0, sizeof(*timers));
  ctx.last_ops.clear();
  for (auto& m : marks) {
    float ms = 0;
    cudaEventElapsedTime(&ms, m.a, m.b);
    const double sec = ms * 1e-3;
    OpTime ot{};
    ot.stream = std::min(m.op->stream, 2);
    ot.ms = ms;
    float st0 = 0;
    cudaEventElapsedTime(&st0, t0, m.a);
    ot.start = st0;
    ot.share = m.op->kind == OpKind::Pass ? m.op->share : 0.0;
    if (m.op->kind == OpKind::Sync) {
      ot.kind = 2;
      timers->wire_comm += sec;
    } else if (m.op->kind == OpKind::Copy) {
      ot.kind = 3;
      timers->wire_comm += sec;
    } else if (m.op->remote) {
      ot.kind = 1;
      ot.n = m.op->n;
      timers->wire_comm += sec;
    } else {
      ot.kind = 0;
      ot.n = m.op->n;
      timers->local_fft += sec;
    }
    ctx.last_ops.push_back(ot);
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, t0, t1);
  timers->total = ms * 1e-3;
  if (knobs().op_times) {
    static const char* kinds[4] = {"local", "exchange", "sync", "copy"};
    for (const auto& o : ctx.last_ops)
      fprintf(stderr, "[dfftb rank %d] %s%s n=%d: %.3f ms\n", ctx.rank, kinds[o.kind],
              o.stream == 1 ? " (side)" : o.stream >= 2 ? " (copy)" : "",
              o.n, o.ms);
  }
}

static void launch_validate(const Plan& plan, const Ctx& ctx, const void* d_in, cudaStream_t s) {
  const int64_t n = plan.input.local_count(ctx.rank) * (plan.input.complex_el ? 2 : 1);
  CUDA_TRY(cudaMemsetAsync(ctx.dstat + 3, 0, sizeof(unsigned long long), s));
  CUDA_TRY(launch_nonfinite(plan.prec, d_in, n, ctx.dstat + 3, s));
}

static void check_validate(const Ctx& ctx, cudaStream_t s) {
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
    raise(DFFTB_Deadlock, "peer did not reach the exchange sync point (timeout)");
  }
  if (ctx.c2r_pending) {
    ctx.c2r_pending = false;
    double mx, im;
    std::memcpy(&mx, &st[0], sizeof(double));
    std::memcpy(&im, &st[1], sizeof(double));
    // irfft_1d tolerance, kernels.hpp:348-377 (scale = block max, plan.hpp:440-446)
    const double tol = (ctx.prec == 8 ? 1e-6 : 1e-2) * mx;
    if (im > tol) {
      char buf[160];
      snprintf(buf, sizeof(buf), "DC or Nyquist bin has a non-real component (|Im| %.3g > tol %.3g, block max %.3g)",
               im, tol, mx);
      raise(DFFTB_NonHermitian, buf);
    }
  }
}

// Every rank issues the whole program even when its input fails validation
// (the check is reported after the launches), so the ranks' sync points and
// buffer parities never drift apart.
static void run_program(const Plan& plan, Ctx& ctx, Program& pr, cudaStream_t s, int flags, dfftb_timing* timers,
                        bool validate) {
  if (pr.c2r) ctx.c2r_pending = true;
  if (timers) run_timed(ctx, pr, s, timers);
  else if (knobs().graphs) run_graph(ctx, pr, s);
  else issue_program(ctx, pr, s);
  if (validate) check_validate(ctx, s);
  if (timers || (flags & DFFTB_EXEC_SYNC)) ctx_check(ctx, s);
}

void execute(const Plan& plan, Ctx& ctx, const void* d_in, void* d_out, cudaStream_t s, int flags,
             dfftb_timing* timers) {
  NvtxRange nr("dfftb_execute");
  DeviceGuard g(ctx.device);
  check_compatible(plan, ctx);
  if (ctx.world_mode) raise(DFFTB_ConfigInvalid, "emulated-world contexts run through execute_world");
  const bool validate = plan.options.validate_finite;
  if (validate) launch_validate(plan, ctx, d_in, s);
  const int parity = (int)(ctx.exec_count & 1);
  ctx.exec_count++;
  Program* pr = nullptr;
  for (const auto& r : ctx.recent)
    if (r.pr && r.id == plan.id && r.in == d_in && r.out == d_out && r.parity == parity) pr = r.pr;
  if (!pr) {
    pr = &cached_program(plan, ctx, d_in, d_out, parity, program_key(plan, d_in, d_out, parity));
    ctx.recent[ctx.recent_next] = Ctx::Recent{plan.id, d_in, d_out, parity, pr};
    ctx.recent_next ^= 1;
  }
  run_program(plan, ctx, *pr, s, flags, timers, validate);
}

// Lockstep issue of all ranks' programs.  One device: stream order is the
// barrier.  Several devices: each rank runs on its context's side stream and
// every sync point becomes "record on every member's stream, wait on them".
static void check_world(const Plan& plan, Ctx** ctxs) {
  const int P = plan.nranks();
  for (int r = 0; r < P; ++r) {
    if (!ctxs[r]->world_mode) raise(DFFTB_ConfigInvalid, "not an emulated world");
    check_compatible(plan, *ctxs[r]);
    if (ctxs[r]->rank != r) raise(DFFTB_InvalidRank, "world contexts must be in rank order");
  }
}

static void run_world(const Plan& plan, Ctx** ctxs, const std::vector<Program*>& progs, cudaStream_t s,
                      int flags) {
  const int P = plan.nranks();
  bool multi_dev = false;
  for (int r = 1; r < P; ++r) multi_dev = multi_dev || ctxs[r]->device != ctxs[0]->device;
  for (int r = 0; r < P; ++r)
    if (progs[r]->c2r) ctxs[r]->c2r_pending = true;
  const size_t nops = progs[0]->ops.size();
  for (int r = 1; r < P; ++r)
    if (progs[r]->ops.size() != nops) raise(DFFTB_CountMismatch, "rank programs differ in length");
  auto stream_of = [&](int r) { return multi_dev ? static_cast<cudaStream_t>(ctxs[r]->side) : s; };
  if (multi_dev) {
    // every rank's stream starts after what the caller enqueued on s
    cudaEvent_t e = event_at(*ctxs[0], 0);
    {
      DeviceGuard g(ctxs[0]->device);
      CUDA_TRY(cudaEventRecord(e, s));
    }
    for (int r = 0; r < P; ++r) {
      DeviceGuard g(ctxs[r]->device);
      CUDA_TRY(cudaStreamWaitEvent(stream_of(r), e, 0));
    }
  }
  for (size_t k = 0; k < nops; ++k) {
    if (multi_dev && progs[0]->ops[k].kind == OpKind::Sync) {
      for (int r = 0; r < P; ++r) {
        DeviceGuard g(ctxs[r]->device);
        CUDA_TRY(cudaEventRecord(event_at(*ctxs[r], 1), stream_of(r)));
      }
      for (int r = 0; r < P; ++r) {
        DeviceGuard g(ctxs[r]->device);
        for (int m : progs[r]->ops[k].members)
          if (m != r) CUDA_TRY(cudaStreamWaitEvent(stream_of(r), event_at(*ctxs[m], 1), 0));
      }
      continue;
    }
    for (int r = 0; r < P; ++r) {
      DeviceGuard g(ctxs[r]->device);
      launch_op(*ctxs[r], progs[r]->ops[k], stream_of(r));
    }
  }
  if (multi_dev) {
    for (int r = 0; r < P; ++r) {
      DeviceGuard g(ctxs[r]->device);
      CUDA_TRY(cudaEventRecord(event_at(*ctxs[r], 2), stream_of(r)));
    }
    DeviceGuard g(ctxs[0]->device);
    for (int r = 0; r < P; ++r) CUDA_TRY(cudaStreamWaitEvent(s, event_at(*ctxs[r], 2), 0));
  }
  if (plan.options.validate_finite)
    for (int r = 0; r < P; ++r) {
      DeviceGuard g(ctxs[r]->device);
      check_validate(*ctxs[r], stream_of(r));
    }
  if (flags & DFFTB_EXEC_SYNC)
    for (int r = 0; r < P; ++r) {
      DeviceGuard g(ctxs[r]->device);
      ctx_check(*ctxs[r], stream_of(r));
    }
}

void execute_world(const Plan& plan, Ctx** ctxs, const void* const* d_in, void* const* d_out, cudaStream_t s,
                   int flags) {
  NvtxRange nr("dfftb_execute_world");
  check_world(plan, ctxs);
  const int P = plan.nranks();
  std::vector<Program*> progs(P);
  for (int r = 0; r < P; ++r) {
    DeviceGuard g(ctxs[r]->device);
    Ctx& c = *ctxs[r];
    if (plan.options.validate_finite) launch_validate(plan, c, d_in[r], s);
    const int parity = (int)(c.exec_count & 1);
    c.exec_count++;
    progs[r] = &cached_program(plan, c, d_in[r], d_out[r], parity, program_key(plan, d_in[r], d_out[r], parity));
  }
  run_world(plan, ctxs, progs, s, flags);
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

int last_op_times(const Ctx& ctx, int* kinds, int* streams, int* lengths, double* shares, double* starts,
                  double* ms, int max) {
  const int n = (int)ctx.last_ops.size();
  for (int i = 0; i < n && i < max; ++i) {
    if (kinds) kinds[i] = ctx.last_ops[i].kind;
    if (streams) streams[i] = ctx.last_ops[i].stream;
    if (lengths) lengths[i] = ctx.last_ops[i].n;
    if (shares) shares[i] = ctx.last_ops[i].share;
    if (starts) starts[i] = ctx.last_ops[i].start;
    if (ms) ms[i] = ctx.last_ops[i].ms;
  }
  return n;
}

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

static void check_zero_mean(const Plan& plan, const double v[2]) {
  double total = 1;
  for (auto d : plan.dims) total *= (double)d;
  if (std::hypot(v[0], v[1]) > 1e-12 * total) raise(DFFTB_NonZeroMean, "inverse_laplacian needs a zero-mean field");
}

void spectral_apply(const Plan& plan, int rank, int op, int axis, const double* lengths, const void* in, void* out,
                    int accumulate, cudaStream_t s) {
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
      check_zero_mean(plan, v);
    }
  }
  CUDA_TRY(launch_spectral(plan.prec, sp, in, out, s));
}

// The forward program of `plan` with the spectral multiplier fused into the
// store epilogue of its last pass: one read + one
// write of the spectrum less than execute + spectral_apply, bit-identical
// values.  Returns a program with no ops when the last pass cannot carry the
// epilogue (non-power-of-two last axis): the caller runs the two-step path.
static Program& spectral_program(const Plan& plan, Ctx& ctx, const void* d_in, void* d_out, int parity, int op,
                                 int axis, const double* lengths, int accumulate) {
  const SpectralParams sp = spectral_params(plan, ctx.rank, lengths);
  char extra[160];
  snprintf(extra, sizeof(extra), "spec%d:%d:%d:%.17g:%.17g:%.17g:%.17g", op, axis, accumulate,
           lengths ? lengths[0] : -1.0, lengths && sp.nd > 1 ? lengths[1] : -1.0,
           lengths && sp.nd > 2 ? lengths[2] : -1.0, lengths && sp.nd > 3 ? lengths[3] : -1.0);
  const std::string key = program_key(plan, d_in, d_out, parity, extra);
  auto it = ctx.programs.find(key);
  if (it != ctx.programs.end()) return *it->second;
  if (ctx.programs.size() >= kMaxCachedPrograms) drop_programs(ctx);
  // the epilogue goes on ONE launch of the last pass: no chunked overlap
  auto pr = build_program(plan, ctx, d_in, d_out, parity, false);
  Op* last = nullptr;
  for (auto& o : pr->ops)
    if (o.kind == OpKind::Pass) last = &o;
  const bool fusable = last && !last->generic && last->before && last->p.ndest == 1 &&
                       last->p.dest[0].ptr == d_out && !last->p.inverse && last->p.in_mode == kInComplex &&
                       !last->p.out_real;
  if (fusable) {
    SpecEpi& e = last->p.spec;
    std::memset(&e, 0, sizeof(e));
    e.op = op + 1;
    e.accumulate = accumulate;
    const int roles[4] = {last->v, last->ax_a, last->ax_b, last->ax_a1};
    int64_t off[kMaxDims], len[kMaxDims];
    last->before->extents_of(ctx.rank, off, len);
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
      e.off[r] = r == 0 ? 0 : off[a];
      e.n[r] = sp.n[a];
      e.half[r] = sp.half[a];
      e.scale[r] = sp.scale[a];
      if (op == 0 && a == axis) e.deriv_role = r;
      if (r > 0 && off[a] != 0) owns_dc = false;
    }
    // |k|^2 summed in tensor-axis order (as spectral_kernel): bit-identical
    int nro = 0;
    for (int a = 0; a < sp.nd; ++a)
      for (int r = 0; r < 4; ++r)
        if (roles[r] == a) e.order[nro++] = r;
    e.nroles = nro;
    // the multiplier variant exists for the strided-lane TMA kernel only
    if (last->tma && !last->adj) last->tma = false;
    if (op == 2 && owns_dc && sp.count > 0) e.dc = ctx.dstat + 4;
  } else {
    pr->ops.clear();  // marks the two-step path (forward + multiply kernel)
  }
  return *ctx.programs.emplace(key, pr).first->second;
}

static void check_spectral_args(const Plan& plan, int rank, int op, int axis, const double* lengths) {
  const SpectralParams sp = spectral_params(plan, rank, lengths);
  if (op < 0 || op > 2) raise(DFFTB_ConfigInvalid, "unknown spectral operator");
  if (op == 0 && (axis < 0 || axis >= sp.nd)) raise(DFFTB_OutOfRange, "derivative axis out of range");
}

static const Op* last_pass(const Program& pr) {
  const Op* last = nullptr;
  for (const auto& o : pr.ops)
    if (o.kind == OpKind::Pass) last = &o;
  return last;
}

static void read_dc_check(const Plan& plan, const Ctx& ctx, cudaStream_t s) {
  unsigned long long bits[2];
  CUDA_TRY(cudaMemcpyAsync(bits, ctx.dstat + 4, sizeof(bits), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  double v[2];
  std::memcpy(v, bits, sizeof(v));
  check_zero_mean(plan, v);
}

void execute_spectral(const Plan& plan, Ctx& ctx, const void* d_in, void* d_out, int op, int axis,
                      const double* lengths, int accumulate, cudaStream_t s, int flags) {
  NvtxRange nr("dfftb_execute_spectral");
  DeviceGuard dg(ctx.device);
  check_compatible(plan, ctx);
  if (ctx.world_mode) raise(DFFTB_ConfigInvalid, "emulated-world contexts run through execute_world_spectral");
  check_spectral_args(plan, ctx.rank, op, axis, lengths);
  const bool validate = plan.options.validate_finite;
  if (validate) launch_validate(plan, ctx, d_in, s);
  const int parity = (int)(ctx.exec_count & 1);
  ctx.exec_count++;
  Program& pr = spectral_program(plan, ctx, d_in, d_out, parity, op, axis, lengths, accumulate);
  if (pr.ops.empty()) {
    Program& fw = cached_program(plan, ctx, d_in, d_out, parity, program_key(plan, d_in, d_out, parity));
    run_program(plan, ctx, fw, s, 0, nullptr, validate);
    spectral_apply(plan, ctx.rank, op, axis, lengths, d_out, d_out, accumulate, s);
    if (flags & DFFTB_EXEC_SYNC) ctx_check(ctx, s);
    return;
  }
  const bool check_mean = last_pass(pr)->p.spec.dc != nullptr;
  if (check_mean) CUDA_TRY(cudaMemsetAsync(ctx.dstat + 4, 0, 2 * sizeof(unsigned long long), s));
  run_program(plan, ctx, pr, s, 0, nullptr, validate);
  if (check_mean) read_dc_check(plan, ctx, s);
  if (flags & DFFTB_EXEC_SYNC) ctx_check(ctx, s);
}

// The emulated world's execute_spectral: every rank's fused program in
// lockstep (or, for non-fusable plans, execute_world + per-rank multiply).
void execute_world_spectral(const Plan& plan, Ctx** ctxs, const void* const* d_in, void* const* d_out, int op,
                            int axis, const double* lengths, int accumulate, cudaStream_t s, int flags) {
  NvtxRange nr("dfftb_execute_world_spectral");
  check_world(plan, ctxs);
  const int P = plan.nranks();
  for (int r = 0; r < P; ++r) check_spectral_args(plan, r, op, axis, lengths);
  std::vector<Program*> progs(P);
  bool fused = true;
  for (int r = 0; r < P; ++r) {
    DeviceGuard g(ctxs[r]->device);
    Ctx& c = *ctxs[r];
    if (plan.options.validate_finite) launch_validate(plan, c, d_in[r], s);
    const int parity = (int)(c.exec_count & 1);
    c.exec_count++;
    progs[r] = &spectral_program(plan, c, d_in[r], d_out[r], parity, op, axis, lengths, accumulate);
    fused = fused && !progs[r]->ops.empty();
    if (progs[r]->ops.empty() || last_pass(*progs[r])->p.spec.dc)
      CUDA_TRY(cudaMemsetAsync(c.dstat + 4, 0, 2 * sizeof(unsigned long long), s));
  }
  if (!fused) {
    for (int r = 0; r < P; ++r) {
      Ctx& c = *ctxs[r];
      const int parity = (int)((c.exec_count - 1) & 1);
      progs[r] = &cached_program(plan, c, d_in[r], d_out[r], parity, program_key(plan, d_in[r], d_out[r], parity));
    }
  }
  run_world(plan, ctxs, progs, s, 0);
  for (int r = 0; r < P; ++r) {
    DeviceGuard g(ctxs[r]->device);
    cudaStream_t st = ctxs[r]->device == ctxs[0]->device ? s : static_cast<cudaStream_t>(ctxs[r]->side);
    if (!fused) spectral_apply(plan, r, op, axis, lengths, d_out[r], d_out[r], accumulate, st);
    else if (last_pass(*progs[r])->p.spec.dc) read_dc_check(plan, *ctxs[r], st);
  }
  if (flags & DFFTB_EXEC_SYNC)
    for (int r = 0; r < P; ++r) {
      DeviceGuard g(ctxs[r]->device);
      ctx_check(*ctxs[r], ctxs[r]->device == ctxs[0]->device ? s : static_cast<cudaStream_t>(ctxs[r]->side));
    }
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
