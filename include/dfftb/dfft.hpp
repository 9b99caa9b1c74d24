// dfftb C++ shim: the reference's dfft:: plan / execute / local-size API
// (/root/reference/proj/include/dfft/{layout,plan,dist_tensor,errors,timing}.hpp)
// re-created over the dfftb C ABI (dfftb.h), header-only.
//
// Drop-in use: replace `#include "dfft/plan.hpp"` by `#include "dfftb/dfft.hpp"`
// and `namespace dfft` by `namespace dfft = dfftb::dfft;`.  Differences a
// caller sees:
//   * DistTensor buffers live in device memory (`d_data()`); `real` / `cplx`
//     host vectors are filled on demand with `to_host()`, and
//     `fill_from_global` / `from_host()` upload.
//   * execute() mirrors its output to the host vectors only when the
//     context's `mirror_to_host` is set (default: on, the reference's
//     host-vector semantics); execute_device() and the spectral operators'
//     intermediate spectra never leave the GPU, so chains of transforms are
//     not PCIe-bound.
//   * make_context takes a Comm that can all-gather bytes (the reference's
//     transport::Comm plays this role; LocalComm is the single-rank world).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "dfftb/dfftb.h"

namespace dfftb::dfft {

template <class T>
using cx = std::complex<T>;

// ---------------------------------------------------------------- errors
// errors.hpp:13-62: the status codes are the ErrorCode ordinals + 1
enum class ErrorCode {
  ZeroLength = 1, OutOfBounds, TooLarge, LengthMismatch, NonHermitian, SlabTooManyRanks,
  OutOfRange, InvalidRank, TagMismatchTimeout, Deadlock, WorkerPanic, CountMismatch,
  IncompatibleLayouts, ArenaExhausted, GridMismatch, RankTooLow, LayoutMismatch,
  NotFrequencyLayout, NonZeroMean, BadMagic, DimMismatch, TruncatedFile, ConfigInvalid,
  CudaError = 100, Unsupported = 101
};

class Error : public std::runtime_error {
 public:
  Error(ErrorCode code, const std::string& what) : std::runtime_error(what), code_(code) {}
  ErrorCode code() const noexcept { return code_; }

 private:
  ErrorCode code_;
};

inline void check(dfftb_status s) {
  if (s != DFFTB_OK) throw Error(static_cast<ErrorCode>(s), dfftb_last_error_message());
}

inline void cuda_check(cudaError_t e) {
  if (e != cudaSuccess) throw Error(ErrorCode::CudaError, std::string("CudaError: ") + cudaGetErrorString(e));
}

// ---------------------------------------------------------------- layout
enum class ElementKind { Real, Complex };
enum class TransformKind { C2C = DFFTB_C2C, R2C = DFFTB_R2C, C2R = DFFTB_C2R };
enum class Direction { Forward = DFFTB_FORWARD, Backward = DFFTB_BACKWARD };
enum class ExchangePath { Blocking, Staged, Pipelined };

struct GlobalDims {
  std::vector<std::int64_t> extent;
  GlobalDims() = default;
  GlobalDims(std::initializer_list<std::int64_t> d) : extent(d) {}
  explicit GlobalDims(std::vector<std::int64_t> d) : extent(std::move(d)) {}
  std::size_t ndim() const { return extent.size(); }
  std::int64_t operator[](std::size_t a) const { return extent[a]; }
  std::int64_t total() const {
    std::int64_t n = 1;
    for (auto e : extent) n *= e;
    return n;
  }
  bool operator==(const GlobalDims&) const = default;
};

struct ProcessGrid {
  std::vector<int> shape;
  ProcessGrid() = default;
  ProcessGrid(std::initializer_list<int> s) : shape(s) {}
  explicit ProcessGrid(std::vector<int> s) : shape(std::move(s)) {}
  std::size_t ndim() const { return shape.size(); }
  int size() const {
    int n = 1;
    for (int s : shape) n *= s;
    return n;
  }
  bool operator==(const ProcessGrid&) const = default;
};

struct BlockMap {
  std::vector<std::int64_t> counts, offsets;
};

inline BlockMap block_map(std::int64_t n, int p) {
  BlockMap m;
  m.counts.resize(p);
  m.offsets.resize(p);
  check(dfftb_block_map(n, p, m.counts.data(), m.offsets.data()));
  return m;
}

struct AxisExtent {
  std::int64_t offset = 0, length = 0;
  bool operator==(const AxisExtent&) const = default;
};

struct LocalExtents {
  std::vector<AxisExtent> axes;
  std::int64_t count() const {
    std::int64_t n = 1;
    for (const auto& a : axes) n *= a.length;
    return n;
  }
};

struct PlanHandle {
  dfftb_plan h = nullptr;
  ~PlanHandle() {
    if (h) dfftb_plan_destroy(h);
  }
};

/// Distribution (layout.hpp:125-194) of one side of a plan.
struct Distribution {
  GlobalDims dims;
  ProcessGrid grid;
  std::vector<int> axis_of_grid;
  std::vector<bool> hatted;
  ElementKind element = ElementKind::Complex;
  std::shared_ptr<PlanHandle> plan;
  int side = DFFTB_INPUT;

  bool operator==(const Distribution& o) const {
    return dims == o.dims && grid == o.grid && axis_of_grid == o.axis_of_grid &&
           hatted == o.hatted && element == o.element;
  }
  LocalExtents extents_of(int rank) const {
    std::vector<std::int64_t> off(dims.ndim()), len(dims.ndim());
    check(dfftb_plan_local_extents(plan->h, rank, side, off.data(), len.data()));
    LocalExtents e;
    for (std::size_t a = 0; a < dims.ndim(); ++a) e.axes.push_back({off[a], len[a]});
    return e;
  }
  std::int64_t local_count(int rank) const { return extents_of(rank).count(); }
  bool all_hatted() const {
    for (bool h : hatted)
      if (!h) return false;
    return true;
  }
};

inline std::pair<int, std::int64_t> local_index(const Distribution& d,
                                                std::span<const std::int64_t> coord) {
  int r = 0;
  std::int64_t o = 0;
  if (coord.size() != d.dims.ndim()) throw Error(ErrorCode::OutOfRange, "OutOfRange: coordinate rank mismatch");
  check(dfftb_local_index(d.plan->h, d.side, coord.data(), &r, &o));
  return {r, o};
}

// ------------------------------------------------------------------ plans
struct PlanOptions {  // plan.hpp:48-54
  ExchangePath exchange = ExchangePath::Blocking;
  bool normalize = true;
  int chunks_per_peer = 1;
  int staging_buffers = 2;
  bool validate_finite = false;
};

template <class T>
struct Plan {
  Direction direction = Direction::Forward;
  TransformKind kind = TransformKind::C2C;
  GlobalDims dims;
  ProcessGrid grid;
  PlanOptions options;
  Distribution input, output;
  std::vector<std::string> warnings;
  std::shared_ptr<PlanHandle> handle;

  int fft_stage_count() const { return dfftb_plan_fft_stage_count(handle->h); }
  int transpose_stage_count() const { return dfftb_plan_transpose_stage_count(handle->h); }
  std::string signature() const {
    char buf[256];
    check(dfftb_plan_signature(handle->h, buf, sizeof(buf)));
    return buf;
  }
};

namespace detail {

inline Distribution layout_of(const std::shared_ptr<PlanHandle>& h, int side, std::size_t nd,
                              const ProcessGrid& grid) {
  Distribution d;
  std::vector<std::int64_t> dims(nd);
  std::vector<int> aog(grid.ndim()), hat(nd);
  int el = 1;
  check(dfftb_plan_layout(h->h, side, dims.data(), &el, aog.data(), hat.data()));
  d.dims = GlobalDims(dims);
  d.grid = grid;
  d.axis_of_grid = aog;
  for (int x : hat) d.hatted.push_back(x != 0);
  d.element = el ? ElementKind::Complex : ElementKind::Real;
  d.plan = h;
  d.side = side;
  return d;
}

template <class T>
Plan<T> make_plan(const GlobalDims& dims, int decomp, const ProcessGrid& grid, TransformKind kind,
                  Direction dir, const PlanOptions& opt) {
  dfftb_plan_options o;
  dfftb_plan_options_default(&o);
  o.exchange = static_cast<int>(opt.exchange);
  o.normalize = opt.normalize;
  o.chunks_per_peer = opt.chunks_per_peer;
  o.staging_buffers = opt.staging_buffers;
  o.validate_finite = opt.validate_finite;
  auto h = std::make_shared<PlanHandle>();
  check(dfftb_plan_create(static_cast<int>(dims.ndim()), dims.extent.data(), decomp,
                          static_cast<int>(grid.ndim()), grid.shape.data(), static_cast<int>(kind),
                          static_cast<int>(dir), static_cast<int>(sizeof(T)), &o, &h->h));
  Plan<T> p;
  p.direction = dir;
  p.kind = kind;
  p.dims = dims;
  p.grid = grid;
  p.options = opt;
  p.handle = h;
  p.input = layout_of(h, DFFTB_INPUT, dims.ndim(), grid);
  p.output = layout_of(h, DFFTB_OUTPUT, dims.ndim(), grid);
  for (int i = 0; i < dfftb_plan_warning_count(h->h); ++i) p.warnings.push_back(dfftb_plan_warning(h->h, i));
  return p;
}

}  // namespace detail

template <class T>
Plan<T> plan_slab(const GlobalDims& dims, int ranks, TransformKind kind, Direction dir,
                  const PlanOptions& options = {}) {
  return detail::make_plan<T>(dims, DFFTB_SLAB, ProcessGrid{ranks}, kind, dir, options);
}

template <class T>
Plan<T> plan_pencil(const GlobalDims& dims, const ProcessGrid& grid, TransformKind kind,
                    Direction dir, const PlanOptions& options = {}) {
  return detail::make_plan<T>(dims, DFFTB_PENCIL, grid, kind, dir, options);
}

template <class T>
Plan<T> plan_general(const GlobalDims& dims, const ProcessGrid& grid, TransformKind kind,
                     Direction dir, const PlanOptions& options = {}) {
  return detail::make_plan<T>(dims, DFFTB_GENERAL, grid, kind, dir, options);
}

// ------------------------------------------------------------- carrier
template <class T>
struct DeviceBuffer {
  void* p = nullptr;
  std::size_t bytes = 0;
  explicit DeviceBuffer(std::size_t b) : bytes(b) {
    if (b) cuda_check(cudaMalloc(&p, b));
  }
  ~DeviceBuffer() {
    if (p) cudaFree(p);
  }
};

/// DistTensor<T> (dist_tensor.hpp:21-45) with a device-resident block.
template <class T>
struct DistTensor {
  Distribution dist;
  int rank = 0;
  std::shared_ptr<DeviceBuffer<T>> dev;
  std::vector<T> real;       // host mirrors, filled by to_host()
  std::vector<cx<T>> cplx;

  /// zero block on the device plus zero host mirrors (reference semantics)
  static DistTensor zeros(const Distribution& d, int rank) {
    DistTensor t = zeros_device(d, rank);
    const std::size_t n = static_cast<std::size_t>(d.local_count(rank));
    if (d.element == ElementKind::Real) t.real.assign(n, T(0));
    else t.cplx.assign(n, cx<T>(0, 0));
    return t;
  }
  /// zero block on the device only (host mirrors empty until to_host())
  static DistTensor zeros_device(const Distribution& d, int rank) {
    DistTensor t;
    t.dist = d;
    t.rank = rank;
    const std::size_t n = static_cast<std::size_t>(d.local_count(rank));
    const std::size_t esz = d.element == ElementKind::Real ? sizeof(T) : sizeof(cx<T>);
    t.dev = std::make_shared<DeviceBuffer<T>>(n * esz);
    if (n) cuda_check(cudaMemset(t.dev->p, 0, n * esz));
    return t;
  }
  void* d_data() const { return dev ? dev->p : nullptr; }
  std::size_t local_size() const { return static_cast<std::size_t>(dist.local_count(rank)); }
  LocalExtents extents() const { return dist.extents_of(rank); }
  void from_host() {
    const std::size_t n = local_size();
    if ((dist.element == ElementKind::Real ? real.size() : cplx.size()) != n)
      throw Error(ErrorCode::CountMismatch, "CountMismatch: host mirror does not hold the local block");
    if (dist.element == ElementKind::Real) {
      if (!real.empty()) cuda_check(cudaMemcpy(dev->p, real.data(), real.size() * sizeof(T), cudaMemcpyHostToDevice));
    } else if (!cplx.empty()) {
      cuda_check(cudaMemcpy(dev->p, cplx.data(), cplx.size() * sizeof(cx<T>), cudaMemcpyHostToDevice));
    }
  }
  void to_host() {
    const std::size_t n = static_cast<std::size_t>(dist.local_count(rank));
    if (dist.element == ElementKind::Real) {
      real.resize(n);
      if (n) cuda_check(cudaMemcpy(real.data(), dev->p, n * sizeof(T), cudaMemcpyDeviceToHost));
    } else {
      cplx.resize(n);
      if (n) cuda_check(cudaMemcpy(cplx.data(), dev->p, n * sizeof(cx<T>), cudaMemcpyDeviceToHost));
    }
  }
};

/// fill_from_global (dist_tensor.hpp:79-102): value_at(global flat, coords), then upload
template <class T, class F>
void fill_from_global(DistTensor<T>& t, F&& value_at) {
  const LocalExtents ext = t.extents();
  const std::size_t nd = t.dist.dims.ndim();
  std::vector<std::int64_t> coord(nd), idx(nd, 0);
  const std::int64_t count = ext.count();
  if (t.dist.element == ElementKind::Real) t.real.resize(static_cast<std::size_t>(count));
  else t.cplx.resize(static_cast<std::size_t>(count));
  for (std::int64_t flat = 0; flat < count; ++flat) {
    std::int64_t global = 0;
    for (std::size_t a = 0; a < nd; ++a) {
      coord[a] = ext.axes[a].offset + idx[a];
      global = global * t.dist.dims[a] + coord[a];
    }
    const cx<T> v = value_at(global, std::span<const std::int64_t>(coord));
    if (t.dist.element == ElementKind::Real) t.real[flat] = v.real();
    else t.cplx[flat] = v;
    for (std::size_t a = nd; a-- > 0;) {
      if (++idx[a] < ext.axes[a].length) break;
      idx[a] = 0;
    }
  }
  t.from_host();
}

// --------------------------------------------------------------- timing
struct TimingBreakdown {  // timing.hpp:16-37
  double local_fft = 0, pack = 0, unpack = 0, staging_copy = 0, wire_comm = 0, total = 0;
  double component_sum() const { return local_fft + pack + unpack + staging_copy + wire_comm; }
};

// -------------------------------------------------------------- context
/// What make_context needs from a communicator (transport::Comm's role):
/// rank, size and an all-gather of fixed-size byte blobs.
struct Comm {
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  virtual std::vector<unsigned char> all_gather(const std::vector<unsigned char>& mine) = 0;
};

struct LocalComm : Comm {
  int rank() const override { return 0; }
  int size() const override { return 1; }
  std::vector<unsigned char> all_gather(const std::vector<unsigned char>& mine) override { return mine; }
};

struct CtxHandle {
  dfftb_ctx h = nullptr;
  ~CtxHandle() {
    if (h) dfftb_ctx_destroy(h);
  }
};

struct ExecContext {
  Comm* world = nullptr;
  std::shared_ptr<CtxHandle> ctx;
  cudaStream_t stream = nullptr;
  bool mirror_to_host = true;  // execute() also fills the output's host vectors
};

/// make_context (plan.hpp:365-390): collective over comm; device = current CUDA device
template <class T>
ExecContext make_context(const Plan<T>& plan, Comm& comm) {
  if (comm.size() != plan.grid.size())
    throw Error(ErrorCode::GridMismatch, "GridMismatch: communicator size must match the grid");
  int dev = 0;
  cuda_check(cudaGetDevice(&dev));
  ExecContext c;
  c.world = &comm;
  c.ctx = std::make_shared<CtxHandle>();
  check(dfftb_ctx_create(plan.handle->h, comm.rank(), dev, &c.ctx->h));
  if (comm.size() > 1) {
    std::vector<unsigned char> mine(dfftb_ctx_handle_size());
    check(dfftb_ctx_export_handle(c.ctx->h, mine.data()));
    auto all = comm.all_gather(mine);
    check(dfftb_ctx_connect(c.ctx->h, all.data()));
  }
  return c;
}

/// execute (plan.hpp:463-535) without the host mirror: the output block
/// stays on the device (to_host() on demand)
template <class T>
DistTensor<T> execute_device(const Plan<T>& plan, const DistTensor<T>& input, ExecContext& ctx,
                             TimingBreakdown* timers = nullptr) {
  if (!(input.dist == plan.input))
    throw Error(ErrorCode::LayoutMismatch, "LayoutMismatch: input layout differs from the plan's");
  DistTensor<T> out = DistTensor<T>::zeros_device(plan.output, input.rank);
  dfftb_timing tc{};
  const int flags = (plan.kind == TransformKind::C2R || plan.options.validate_finite) ? DFFTB_EXEC_SYNC : 0;
  check(dfftb_execute(plan.handle->h, ctx.ctx->h, input.d_data(), out.d_data(), ctx.stream, flags,
                      timers ? &tc : nullptr));
  if (timers) {
    timers->local_fft += tc.local_fft;
    timers->pack += tc.pack;
    timers->unpack += tc.unpack;
    timers->staging_copy += tc.staging_copy;
    timers->wire_comm += tc.wire_comm;
    timers->total += tc.total;
  }
  return out;
}

/// execute (plan.hpp:463-535): this rank's output block, on the device and
/// (ctx.mirror_to_host) in the host vectors
template <class T>
DistTensor<T> execute(const Plan<T>& plan, const DistTensor<T>& input, ExecContext& ctx,
                      TimingBreakdown* timers = nullptr) {
  DistTensor<T> out = execute_device(plan, input, ctx, timers);
  if (ctx.mirror_to_host) out.to_host();
  return out;
}

template <class T>
DistTensor<T> execute_r2c_c2r_roundtrip(const Plan<T>& fwd, const Plan<T>& bwd, const DistTensor<T>& in,
                                        ExecContext& ctx, TimingBreakdown* timers = nullptr) {
  if (fwd.kind != TransformKind::R2C || bwd.kind != TransformKind::C2R || !(fwd.dims == bwd.dims) ||
      !(fwd.grid == bwd.grid))
    throw Error(ErrorCode::GridMismatch, "GridMismatch: round trip needs matching R2C/C2R plans");
  auto spectrum = execute_device(fwd, in, ctx, timers);
  return execute(bwd, spectrum, ctx, timers);
}

inline GlobalDims hat_dims(const GlobalDims& dims, TransformKind kind) {
  GlobalDims out = dims;
  if (kind == TransformKind::R2C && !out.extent.empty()) out.extent.back() = out.extent.back() / 2 + 1;
  return out;
}

// ------------------------------------------------- spectral (spectral.hpp)
struct WavenumberMap {  // spectral.hpp:17-20
  std::vector<std::vector<double>> axis_k;
  std::vector<std::vector<double>> axis_k_deriv;
};

/// wavenumbers (spectral.hpp:24-56) for this rank's block of a forward plan's
/// output layout (`freq` must be such a layout: NotFrequencyLayout otherwise).
inline WavenumberMap wavenumbers(const Distribution& freq, const GlobalDims& spatial_dims,
                                 std::span<const double> domain_lengths, int rank) {
  (void)spatial_dims;  // the plan handle behind `freq` carries the spatial dims
  if (domain_lengths.size() != freq.dims.ndim())
    throw Error(ErrorCode::NotFrequencyLayout, "NotFrequencyLayout: one domain length per axis");
  const LocalExtents ext = freq.extents_of(rank);
  WavenumberMap m;
  for (std::size_t a = 0; a < freq.dims.ndim(); ++a) {
    for (int deriv = 0; deriv < 2; ++deriv) {
      std::vector<double> k(static_cast<std::size_t>(std::max<std::int64_t>(1, ext.axes[a].length)));
      check(dfftb_wavenumbers(freq.plan->h, rank, static_cast<int>(a), deriv, domain_lengths.data(), k.data()));
      k.resize(static_cast<std::size_t>(ext.axes[a].length));
      (deriv ? m.axis_k_deriv : m.axis_k).push_back(std::move(k));
    }
  }
  return m;
}

template <class T>
struct SpectralContext {  // spectral.hpp:61-70
  Comm* comm = nullptr;
  GlobalDims dims;
  ProcessGrid grid;
  std::vector<double> domain_lengths;
  Plan<T> fwd_c2c, bwd_c2c, fwd_r2c, bwd_c2r;
  WavenumberMap k_c2c, k_r2c;
  ExecContext exec;
};

/// make_spectral_context (spectral.hpp:72-98): the four plans on one grid
/// (pencil for 3 axes on a 2-D grid, the general decomposition otherwise),
/// their wavenumbers and one shared execution context.
template <class T>
SpectralContext<T> make_spectral_context(Comm& comm, const GlobalDims& dims, const ProcessGrid& grid,
                                         std::vector<double> domain_lengths = {}) {
  SpectralContext<T> c;
  c.comm = &comm;
  c.dims = dims;
  c.grid = grid;
  if (domain_lengths.empty()) domain_lengths.assign(dims.ndim(), 6.283185307179586476925);
  c.domain_lengths = std::move(domain_lengths);
  auto mk = [&](TransformKind k, Direction d) {
    return (dims.ndim() == 3 && grid.ndim() == 2) ? plan_pencil<T>(dims, grid, k, d)
                                                  : plan_general<T>(dims, grid, k, d);
  };
  c.fwd_c2c = mk(TransformKind::C2C, Direction::Forward);
  c.bwd_c2c = mk(TransformKind::C2C, Direction::Backward);
  c.fwd_r2c = mk(TransformKind::R2C, Direction::Forward);
  c.bwd_c2r = mk(TransformKind::C2R, Direction::Backward);
  c.k_c2c = wavenumbers(c.fwd_c2c.output, dims, c.domain_lengths, comm.rank());
  c.k_r2c = wavenumbers(c.fwd_r2c.output, dims, c.domain_lengths, comm.rank());
  c.exec = make_context(c.fwd_c2c, comm);
  return c;
}

namespace detail {
/// op (spectral multiplier) fused into the forward transform's last pass
/// (dfftb_execute_spectral); accumulate adds into `spec`.
template <class T>
void forward_op(SpectralContext<T>& c, const Plan<T>& fwd, const DistTensor<T>& x, int op, int axis,
                DistTensor<T>& spec, bool accumulate) {
  if (!(x.dist == fwd.input))
    throw Error(ErrorCode::LayoutMismatch, "LayoutMismatch: input layout differs from the plan's");
  check(dfftb_execute_spectral(fwd.handle->h, c.exec.ctx->h, x.d_data(), spec.d_data(), op, axis,
                               c.domain_lengths.data(), accumulate ? 1 : 0, c.exec.stream, DFFTB_EXEC_SYNC));
}
template <class T>
bool is_real_field(const DistTensor<T>& x) {
  return x.dist.element == ElementKind::Real;
}
}  // namespace detail

/// derivative (spectral.hpp:131-164): backward(i k_axis (.) forward(x)), normalized
template <class T>
DistTensor<T> derivative(SpectralContext<T>& c, const DistTensor<T>& x, int axis) {
  const bool real = detail::is_real_field(x);
  const Plan<T>& fwd = real ? c.fwd_r2c : c.fwd_c2c;
  const Plan<T>& bwd = real ? c.bwd_c2r : c.bwd_c2c;
  auto spec = DistTensor<T>::zeros_device(fwd.output, x.rank);
  detail::forward_op(c, fwd, x, DFFTB_SPECTRAL_DERIV, axis, spec, false);
  return execute(bwd, spec, c.exec);
}

/// gradient (spectral.hpp:167-176)
template <class T>
std::vector<DistTensor<T>> gradient(SpectralContext<T>& c, const DistTensor<T>& x) {
  std::vector<DistTensor<T>> g;
  for (std::size_t a = 0; a < c.dims.ndim(); ++a) g.push_back(derivative(c, x, static_cast<int>(a)));
  return g;
}

/// divergence (spectral.hpp:180-216): sum_j i k_j (.) forward(c_j), one inverse
template <class T>
DistTensor<T> divergence(SpectralContext<T>& c, const std::vector<DistTensor<T>>& comps) {
  if (comps.size() != c.dims.ndim())
    throw Error(ErrorCode::GridMismatch, "GridMismatch: one component per axis required");
  const bool real = detail::is_real_field(comps[0]);
  const Plan<T>& fwd = real ? c.fwd_r2c : c.fwd_c2c;
  const Plan<T>& bwd = real ? c.bwd_c2r : c.bwd_c2c;
  auto acc = DistTensor<T>::zeros_device(fwd.output, comps[0].rank);
  for (std::size_t a = 0; a < comps.size(); ++a)
    detail::forward_op(c, fwd, comps[a], DFFTB_SPECTRAL_DERIV, static_cast<int>(a), acc, a > 0);
  return execute(bwd, acc, c.exec);
}

/// laplacian (spectral.hpp:219-249): backward(-|k|^2 (.) forward(x))
template <class T>
DistTensor<T> laplacian(SpectralContext<T>& c, const DistTensor<T>& x) {
  const bool real = detail::is_real_field(x);
  const Plan<T>& fwd = real ? c.fwd_r2c : c.fwd_c2c;
  const Plan<T>& bwd = real ? c.bwd_c2r : c.bwd_c2c;
  auto spec = DistTensor<T>::zeros_device(fwd.output, x.rank);
  detail::forward_op(c, fwd, x, DFFTB_SPECTRAL_LAPLACIAN, 0, spec, false);
  return execute(bwd, spec, c.exec);
}

/// inverse_laplacian (spectral.hpp:251-309): divides by -|k|^2, k = 0 pinned
/// to zero; NonZeroMean unless the field has zero mean
template <class T>
DistTensor<T> inverse_laplacian(SpectralContext<T>& c, const DistTensor<T>& x) {
  const bool real = detail::is_real_field(x);
  const Plan<T>& fwd = real ? c.fwd_r2c : c.fwd_c2c;
  const Plan<T>& bwd = real ? c.bwd_c2r : c.bwd_c2c;
  auto spec = DistTensor<T>::zeros_device(fwd.output, x.rank);
  detail::forward_op(c, fwd, x, DFFTB_SPECTRAL_INV_LAPLACIAN, 0, spec, false);
  return execute(bwd, spec, c.exec);
}

}  // namespace dfftb::dfft
