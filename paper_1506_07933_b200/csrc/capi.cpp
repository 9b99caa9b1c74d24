// extern "C" boundary of dfftb (include/dfftb/dfftb.h).  Every entry point
// converts internal dfftb::Error exceptions into a status code plus a
// thread-local message formatted like dfft::Error::what() (errors.hpp:48-58).
#include <cstring>
#include <string>

#include "dfftb/dfftb.h"
#include "exec.hpp"
#include "kernels.hpp"

struct dfftb_plan_s {
  dfftb::Plan plan;
};
struct dfftb_ctx_s {
  dfftb::Ctx* ctx;
};

namespace {

thread_local std::string g_last_error;

template <class F>
dfftb_status guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return DFFTB_OK;
  } catch (const dfftb::Error& e) {
    g_last_error = std::string(dfftb::status_name(e.code)) + ": " + e.what;
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = std::string("ConfigInvalid: ") + e.what();
    return DFFTB_ConfigInvalid;
  }
}

const dfftb::Dist& side_dist(dfftb_plan p, int side) {
  if (side != DFFTB_INPUT && side != DFFTB_OUTPUT) dfftb::raise(DFFTB_OutOfRange, "bad layout side");
  return side == DFFTB_INPUT ? p->plan.input : p->plan.output;
}

}  // namespace

extern "C" {

void dfftb_plan_options_default(dfftb_plan_options* o) {
  o->exchange = DFFTB_EXCHANGE_BLOCKING;
  o->normalize = 1;
  o->chunks_per_peer = 1;
  o->staging_buffers = 2;
  o->validate_finite = 0;
}

dfftb_status dfftb_plan_create(int ndim, const int64_t* dims, int decomp, int grid_ndim,
                               const int* grid, int kind, int direction, int precision,
                               const dfftb_plan_options* opts, dfftb_plan* out) {
  return guarded([&] {
    if (!out || !dims || !grid || ndim < 0 || grid_ndim < 0)
      dfftb::raise(DFFTB_ConfigInvalid, "null argument");
    dfftb_plan_options o;
    dfftb_plan_options_default(&o);
    if (opts) o = *opts;
    std::vector<int64_t> d(dims, dims + ndim);
    std::vector<int> g(grid, grid + grid_ndim);
    auto* p = new dfftb_plan_s{dfftb::build_plan(d, decomp, g, kind, direction, precision, o)};
    *out = p;
  });
}

void dfftb_plan_destroy(dfftb_plan plan) { delete plan; }

dfftb_status dfftb_plan_signature(dfftb_plan plan, char* buf, size_t len) {
  return guarded([&] {
    const std::string s = plan->plan.signature();
    if (len < s.size() + 1) dfftb::raise(DFFTB_LengthMismatch, "signature buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

int dfftb_plan_fft_stage_count(dfftb_plan plan) {
  int n = 0;
  for (const auto& s : plan->plan.stages) n += s.type == dfftb::StageType::Fft;
  return n;
}

int dfftb_plan_transpose_stage_count(dfftb_plan plan) {
  int n = 0;
  for (const auto& s : plan->plan.stages) n += s.type == dfftb::StageType::Transpose;
  return n;
}

int dfftb_plan_nranks(dfftb_plan plan) { return plan->plan.nranks(); }
int dfftb_plan_precision(dfftb_plan plan) { return plan->plan.prec; }
int dfftb_plan_kind(dfftb_plan plan) { return plan->plan.kind; }
int dfftb_plan_direction(dfftb_plan plan) { return plan->plan.dir; }
int dfftb_plan_warning_count(dfftb_plan plan) { return (int)plan->plan.warnings.size(); }
const char* dfftb_plan_warning(dfftb_plan plan, int i) {
  if (i < 0 || i >= (int)plan->plan.warnings.size()) return "";
  return plan->plan.warnings[i].c_str();
}

dfftb_status dfftb_block_map(int64_t n, int p, int64_t* counts, int64_t* offsets) {
  return guarded([&] {
    if (p < 1) dfftb::raise(DFFTB_ConfigInvalid, "p must be >= 1");
    const auto b = dfftb::block_map(n, p);
    std::memcpy(counts, b.counts.data(), sizeof(int64_t) * p);
    std::memcpy(offsets, b.offsets.data(), sizeof(int64_t) * p);
  });
}

dfftb_status dfftb_plan_layout(dfftb_plan plan, int side, int64_t* dims, int* element_complex,
                               int* axis_of_grid, int* hatted) {
  return guarded([&] {
    const auto& d = side_dist(plan, side);
    for (int a = 0; a < d.ndim(); ++a) {
      if (dims) dims[a] = d.dims[a];
      if (hatted) hatted[a] = d.hatted[a];
    }
    for (int g = 0; g < d.gnd(); ++g)
      if (axis_of_grid) axis_of_grid[g] = d.axis_of_grid[g];
    if (element_complex) *element_complex = d.complex_el ? 1 : 0;
  });
}

dfftb_status dfftb_plan_local_extents(dfftb_plan plan, int rank, int side, int64_t* offsets,
                                      int64_t* lengths) {
  return guarded([&] {
    const auto& d = side_dist(plan, side);
    if (rank < 0 || rank >= d.nranks()) dfftb::raise(DFFTB_InvalidRank, "rank out of range");
    d.extents_of(rank, offsets, lengths);
  });
}

int64_t dfftb_plan_local_count(dfftb_plan plan, int rank, int side) {
  if (side != DFFTB_INPUT && side != DFFTB_OUTPUT) return -1;
  const auto& d = side == DFFTB_INPUT ? plan->plan.input : plan->plan.output;
  if (rank < 0 || rank >= d.nranks()) return -1;
  return d.local_count(rank);
}

dfftb_status dfftb_local_index(dfftb_plan plan, int side, const int64_t* coord, int* rank,
                               int64_t* offset) {
  return guarded([&] {
    // local_index, layout.hpp:272-295
    const auto& d = side_dist(plan, side);
    for (int a = 0; a < d.ndim(); ++a)
      if (coord[a] < 0 || coord[a] >= d.dims[a])
        dfftb::raise(DFFTB_OutOfRange, "coordinate outside the global dims");
    std::vector<int> gc(d.gnd());
    for (int g = 0; g < d.gnd(); ++g) {
      const int axis = d.axis_of_grid[g];
      const int64_t blk = (d.dims[axis] + d.grid[g] - 1) / d.grid[g];
      gc[g] = (int)(coord[axis] / blk);
    }
    const int r = d.rank_of(gc);
    int64_t off[dfftb::kMaxDims], len[dfftb::kMaxDims];
    d.extents_of(r, off, len);
    int64_t o = 0;
    for (int a = 0; a < d.ndim(); ++a) o = o * len[a] + (coord[a] - off[a]);
    *rank = r;
    *offset = o;
  });
}

dfftb_status dfftb_workspace_bytes(dfftb_plan plan, int rank, uint64_t* bytes) {
  return guarded([&] { *bytes = (uint64_t)dfftb::workspace_bytes(plan->plan, rank); });
}

dfftb_status dfftb_plan_exchange_counts(dfftb_plan plan, int rank, int transpose_index,
                                        int64_t* send_counts, int64_t* recv_counts,
                                        int* group_size) {
  return guarded([&] {
    const auto& P = plan->plan;
    const dfftb::Stage* tr = nullptr;
    int k = 0;
    for (const auto& s : P.stages)
      if (s.type == dfftb::StageType::Transpose && k++ == transpose_index) tr = &s;
    if (!tr) dfftb::raise(DFFTB_OutOfRange, "no such transpose stage");
    if (rank < 0 || rank >= P.nranks()) dfftb::raise(DFFTB_InvalidRank, "rank out of range");
    const auto& from = tr->before;
    const auto& to = tr->after;
    const int g = tr->grid_axis;
    const int u = from.axis_of_grid[g], v = to.axis_of_grid[g];
    const int q = from.grid[g];
    int64_t fo[dfftb::kMaxDims], fl[dfftb::kMaxDims], too[dfftb::kMaxDims], tl[dfftb::kMaxDims];
    from.extents_of(rank, fo, fl);
    to.extents_of(rank, too, tl);
    int64_t send_unit = 1, recv_unit = 1;
    for (int a = 0; a < from.ndim(); ++a) {
      if (a != v) send_unit *= fl[a];
      if (a != u) recv_unit *= tl[a];
    }
    const auto sb = dfftb::block_map(from.dims[v], q);
    const auto rb = dfftb::block_map(from.dims[u], q);
    for (int j = 0; j < q; ++j) {
      send_counts[j] = send_unit * sb.counts[j];
      recv_counts[j] = recv_unit * rb.counts[j];
    }
    *group_size = q;
  });
}

dfftb_status dfftb_ctx_create(dfftb_plan plan, int rank, int device, dfftb_ctx* out) {
  return guarded([&] { *out = new dfftb_ctx_s{dfftb::ctx_create(plan->plan, rank, device)}; });
}

size_t dfftb_ctx_handle_size(void) { return sizeof(dfftb::CtxHandle); }

dfftb_status dfftb_ctx_export_handle(dfftb_ctx ctx, void* handle) {
  return guarded([&] { dfftb::ctx_export(*ctx->ctx, static_cast<dfftb::CtxHandle*>(handle)); });
}

dfftb_status dfftb_ctx_connect(dfftb_ctx ctx, const void* handles) {
  return guarded(
      [&] { dfftb::ctx_connect(*ctx->ctx, static_cast<const dfftb::CtxHandle*>(handles)); });
}

void dfftb_ctx_destroy(dfftb_ctx ctx) {
  if (!ctx) return;
  dfftb::ctx_destroy(ctx->ctx);
  delete ctx;
}

dfftb_status dfftb_execute(dfftb_plan plan, dfftb_ctx ctx, const void* d_in, void* d_out,
                           void* stream, int flags, dfftb_timing* timers) {
  return guarded([&] {
    dfftb::execute(plan->plan, *ctx->ctx, d_in, d_out, static_cast<cudaStream_t>(stream), flags,
                   timers);
  });
}

dfftb_status dfftb_ctx_check(dfftb_ctx ctx, void* stream) {
  return guarded([&] { dfftb::ctx_check(*ctx->ctx, static_cast<cudaStream_t>(stream)); });
}

dfftb_status dfftb_world_create(dfftb_plan plan, int device, dfftb_ctx* ctxs) {
  return dfftb_world_create_devices(plan, 1, &device, ctxs);
}

dfftb_status dfftb_world_create_devices(dfftb_plan plan, int ndevices, const int* devices, dfftb_ctx* ctxs) {
  return guarded([&] {
    if (!devices || ndevices < 1) dfftb::raise(DFFTB_ConfigInvalid, "need at least one device");
    const int P = plan->plan.nranks();
    std::vector<dfftb::Ctx*> raw(P, nullptr);
    dfftb::world_create(plan->plan, devices, ndevices, raw.data());
    for (int r = 0; r < P; ++r) ctxs[r] = new dfftb_ctx_s{raw[r]};
  });
}

int dfftb_ctx_last_ops(dfftb_ctx ctx, int* kinds, int* streams, int* lengths, double* shares, double* starts,
                       double* ms, int max) {
  return ctx ? dfftb::last_op_times(*ctx->ctx, kinds, streams, lengths, shares, starts, ms, max) : 0;
}

dfftb_status dfftb_execute_world(dfftb_plan plan, dfftb_ctx* ctxs, const void* const* d_in,
                                 void* const* d_out, void* stream, int flags) {
  return guarded([&] {
    const int P = plan->plan.nranks();
    std::vector<dfftb::Ctx*> raw(P);
    for (int r = 0; r < P; ++r) raw[r] = ctxs[r]->ctx;
    dfftb::execute_world(plan->plan, raw.data(), d_in, d_out, static_cast<cudaStream_t>(stream),
                         flags);
  });
}

dfftb_status dfftb_fill_seeded(dfftb_plan plan, int rank, int side, uint64_t seed,
                               int complex_field, void* d_buf, void* stream) {
  return guarded([&] {
    dfftb::fill_seeded(plan->plan, rank, side, seed, complex_field, d_buf,
                       static_cast<cudaStream_t>(stream));
  });
}

const char* dfftb_error_name(dfftb_status status) { return dfftb::status_name(status); }
const char* dfftb_last_error_message(void) { return g_last_error.c_str(); }
uint64_t dfftb_kernel_launch_count(void) { return dfftb::launch_count(); }

}  // extern "C"

extern "C" {

dfftb_status dfftb_spectral_apply(dfftb_plan forward_plan, int rank, int op, int axis,
                                  const double* domain_lengths, const void* d_in, void* d_out,
                                  int accumulate, void* stream) {
  return guarded([&] {
    dfftb::spectral_apply(forward_plan->plan, rank, op, axis, domain_lengths, d_in, d_out, accumulate,
                          static_cast<cudaStream_t>(stream));
  });
}

dfftb_status dfftb_execute_spectral(dfftb_plan forward_plan, dfftb_ctx ctx, const void* d_in, void* d_out,
                                    int op, int axis, const double* domain_lengths, int accumulate,
                                    void* stream, int flags) {
  return guarded([&] {
    dfftb::execute_spectral(forward_plan->plan, *ctx->ctx, d_in, d_out, op, axis, domain_lengths, accumulate,
                            static_cast<cudaStream_t>(stream), flags);
  });
}

dfftb_status dfftb_execute_world_spectral(dfftb_plan forward_plan, dfftb_ctx* ctxs, const void* const* d_in,
                                          void* const* d_out, int op, int axis, const double* domain_lengths,
                                          int accumulate, void* stream, int flags) {
  return guarded([&] {
    const int P = forward_plan->plan.nranks();
    std::vector<dfftb::Ctx*> raw(P);
    for (int r = 0; r < P; ++r) raw[r] = ctxs[r]->ctx;
    dfftb::execute_world_spectral(forward_plan->plan, raw.data(), d_in, d_out, op, axis, domain_lengths, accumulate,
                                  static_cast<cudaStream_t>(stream), flags);
  });
}

dfftb_status dfftb_wavenumbers(dfftb_plan forward_plan, int rank, int axis, int deriv,
                               const double* domain_lengths, double* k_out) {
  return guarded(
      [&] { dfftb::wavenumbers(forward_plan->plan, rank, axis, deriv, domain_lengths, k_out); });
}

}  // extern "C"
