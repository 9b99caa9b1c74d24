// Host plan builder and layout math for dfftb.
//
// Re-derives the reference's decomposition contract so outputs land exactly
// where the reference puts them:
//   block_map            layout.hpp:80-92     ceil blocks, empty tails allowed
//   Distribution         layout.hpp:125-194   grid axis -> tensor axis
//   spatial/frequency    layout.hpp:232-268   input / output layouts (xyz order)
//   check_grid           layout.hpp:211-226
//   build_nd_plan        plan.hpp:149-236     pencil + general (Alg. 1/2)
//   plan_slab            plan.hpp:267-354     slab (Alg. 3)
//   checks               plan.hpp:103-128
#include <algorithm>
#include <atomic>
#include <numeric>

#include "internal.hpp"

namespace dfftb {

void raise(dfftb_status code, const std::string& what) { throw Error{code, what}; }

const char* status_name(dfftb_status s) {
  switch (s) {
    case DFFTB_OK: return "OK";
    case DFFTB_ZeroLength: return "ZeroLength";
    case DFFTB_OutOfBounds: return "OutOfBounds";
    case DFFTB_TooLarge: return "TooLarge";
    case DFFTB_LengthMismatch: return "LengthMismatch";
    case DFFTB_NonHermitian: return "NonHermitian";
    case DFFTB_SlabTooManyRanks: return "SlabTooManyRanks";
    case DFFTB_OutOfRange: return "OutOfRange";
    case DFFTB_InvalidRank: return "InvalidRank";
    case DFFTB_TagMismatchTimeout: return "TagMismatchTimeout";
    case DFFTB_Deadlock: return "Deadlock";
    case DFFTB_WorkerPanic: return "WorkerPanic";
    case DFFTB_CountMismatch: return "CountMismatch";
    case DFFTB_IncompatibleLayouts: return "IncompatibleLayouts";
    case DFFTB_ArenaExhausted: return "ArenaExhausted";
    case DFFTB_GridMismatch: return "GridMismatch";
    case DFFTB_RankTooLow: return "RankTooLow";
    case DFFTB_LayoutMismatch: return "LayoutMismatch";
    case DFFTB_NotFrequencyLayout: return "NotFrequencyLayout";
    case DFFTB_NonZeroMean: return "NonZeroMean";
    case DFFTB_BadMagic: return "BadMagic";
    case DFFTB_DimMismatch: return "DimMismatch";
    case DFFTB_TruncatedFile: return "TruncatedFile";
    case DFFTB_ConfigInvalid: return "ConfigInvalid";
    case DFFTB_CudaError: return "CudaError";
    case DFFTB_Unsupported: return "Unsupported";
  }
  return "UnknownError";
}

Blocks block_map(int64_t n, int p) {
  Blocks b;
  b.counts.resize(p);
  b.offsets.resize(p);
  const int64_t blk = p > 0 ? (n + p - 1) / p : 0;
  for (int r = 0; r < p; ++r) {
    const int64_t lo = std::min<int64_t>(r * blk, n);
    const int64_t hi = std::min<int64_t>((r + 1) * blk, n);
    b.offsets[r] = lo;
    b.counts[r] = hi - lo;
  }
  return b;
}

int Dist::nranks() const {
  int p = 1;
  for (int g : grid) p *= g;
  return p;
}

std::vector<int> Dist::coords_of(int rank) const {
  std::vector<int> c(grid.size());
  for (int g = gnd(); g-- > 0;) {
    c[g] = rank % grid[g];
    rank /= grid[g];
  }
  return c;
}

int Dist::rank_of(const std::vector<int>& c) const {
  int r = 0;
  for (int g = 0; g < gnd(); ++g) r = r * grid[g] + c[g];
  return r;
}

int Dist::grid_axis_of(int axis) const {
  for (int g = 0; g < gnd(); ++g)
    if (axis_of_grid[g] == axis) return g;
  return -1;
}

void Dist::extents_of(int rank, int64_t* off, int64_t* len) const {
  const auto c = coords_of(rank);
  for (int a = 0; a < ndim(); ++a) {
    const int g = grid_axis_of(a);
    if (g < 0) {
      off[a] = 0;
      len[a] = dims[a];
    } else {
      const int64_t blk = (dims[a] + grid[g] - 1) / grid[g];
      const int64_t lo = std::min<int64_t>(c[g] * blk, dims[a]);
      const int64_t hi = std::min<int64_t>((c[g] + 1) * blk, dims[a]);
      off[a] = lo;
      len[a] = hi - lo;
    }
  }
}

int64_t Dist::local_count(int rank) const {
  int64_t off[kMaxDims], len[kMaxDims];
  extents_of(rank, off, len);
  int64_t n = 1;
  for (int a = 0; a < ndim(); ++a) n *= len[a];
  return n;
}

int64_t Dist::max_local_count() const {
  int64_t m = 0;
  for (int r = 0; r < nranks(); ++r) m = std::max(m, local_count(r));
  return m;
}

bool Dist::any_rank_empty() const {
  for (int g = 0; g < gnd(); ++g) {
    const Blocks b = block_map(dims[axis_of_grid[g]], grid[g]);
    if (!b.counts.empty() && b.counts.back() == 0) return true;
  }
  return false;
}

static void check_grid(const std::vector<int64_t>& dims, const std::vector<int>& grid) {
  if (dims.size() < 2) raise(DFFTB_IncompatibleLayouts, "need at least two tensor axes");
  if (grid.empty() || grid.size() > dims.size() - 1)
    raise(DFFTB_IncompatibleLayouts, "grid must have between 1 and ndim-1 axes");
  for (int p : grid)
    if (p < 1) raise(DFFTB_IncompatibleLayouts, "grid factors must be >= 1");
  if (grid.size() == 1 && grid[0] > dims[0])
    raise(DFFTB_SlabTooManyRanks, "slab decomposition needs P <= N0");
}

Dist spatial_layout(const std::vector<int64_t>& dims, const std::vector<int>& grid, int kind) {
  check_grid(dims, grid);
  Dist d;
  d.dims = dims;
  d.grid = grid;
  d.axis_of_grid.resize(grid.size());
  std::iota(d.axis_of_grid.begin(), d.axis_of_grid.end(), 0);
  d.hatted.assign(dims.size(), 0);
  d.complex_el = kind == DFFTB_C2C;
  return d;
}

Dist frequency_layout(const std::vector<int64_t>& dims, const std::vector<int>& grid, int kind) {
  check_grid(dims, grid);
  Dist d;
  d.dims = dims;
  if (kind != DFFTB_C2C) d.dims.back() = dims.back() / 2 + 1;
  d.grid = grid;
  d.axis_of_grid.resize(grid.size());
  std::iota(d.axis_of_grid.begin(), d.axis_of_grid.end(), 1);
  d.hatted.assign(dims.size(), 1);
  d.complex_el = true;
  return d;
}

std::string Plan::signature() const {
  std::string s;
  for (const auto& st : stages) {
    switch (st.type) {
      case StageType::Fft: s += "F" + std::to_string(st.axis); break;
      case StageType::Transpose:
        s += "T" + std::to_string(st.grid_axis) + (st.transposed ? "x" : "");
        break;
      case StageType::LocalTranspose: s += "L"; break;
      case StageType::Normalize: s += "N"; break;
    }
    s += ";";
  }
  return s;
}

static Stage fft(int axis, int dir, int fkind, const Dist& b, const Dist& a) {
  Stage s;
  s.type = StageType::Fft;
  s.axis = axis;
  s.dir = dir;
  s.fkind = fkind;
  s.before = b;
  s.after = a;
  return s;
}

static Stage transpose(const Dist& from, const Dist& to, int g, bool transposed) {
  Stage s;
  s.type = StageType::Transpose;
  s.before = from;
  s.after = to;
  s.grid_axis = g;
  s.transposed = transposed;
  return s;
}

static int64_t product(const std::vector<int64_t>& v) {
  int64_t n = 1;
  for (auto x : v) n *= x;
  return n;
}

static std::atomic<uint64_t> g_plan_ids{1};

Plan build_plan(const std::vector<int64_t>& dims, int decomp, const std::vector<int>& grid_in,
                int kind, int dir, int prec, const dfftb_plan_options& opts) {
  if (prec != DFFTB_F32 && prec != DFFTB_F64) raise(DFFTB_ConfigInvalid, "precision must be 4 or 8");
  if (kind < 0 || kind > 2 || (dir != 0 && dir != 1)) raise(DFFTB_ConfigInvalid, "bad kind/direction");
  for (auto d : dims)
    if (d < 1) raise(DFFTB_ConfigInvalid, "axis lengths must be >= 1");
  std::vector<int> grid = grid_in;
  if (decomp == DFFTB_SLAB) {
    // plan_slab, plan.hpp:267-277
    if (dims.size() < 2) raise(DFFTB_GridMismatch, "slab needs at least 2 tensor axes");
    if (grid.size() != 1) raise(DFFTB_GridMismatch, "slab takes a rank count");
    if (grid[0] < 1) raise(DFFTB_GridMismatch, "need at least one rank");
    if (grid[0] > dims[0]) raise(DFFTB_SlabTooManyRanks, "slab decomposition needs P <= N0");
  } else if (decomp == DFFTB_PENCIL) {
    if (dims.size() != 3 || grid.size() != 2)
      raise(DFFTB_GridMismatch, "pencil needs 3 tensor axes and a 2-D grid");
  } else if (decomp == DFFTB_GENERAL) {
    if (dims.size() < 2 || grid.size() != dims.size() - 1)
      raise(DFFTB_GridMismatch, "general decomposition needs len(grid) == len(dims) - 1");
  } else {
    raise(DFFTB_ConfigInvalid, "unknown decomposition");
  }
  if (dims.size() > kMaxDims) raise(DFFTB_Unsupported, "at most 4 tensor axes");
  // check_kind_direction, plan.hpp:103-110
  if (kind == DFFTB_R2C && dir != DFFTB_FORWARD) raise(DFFTB_ConfigInvalid, "R2C is a forward transform");
  if (kind == DFFTB_C2R && dir != DFFTB_BACKWARD) raise(DFFTB_ConfigInvalid, "C2R is a backward transform");
  if (opts.chunks_per_peer < 1) raise(DFFTB_ConfigInvalid, "chunks per peer must be >= 1");
  if (opts.staging_buffers < 1) raise(DFFTB_ConfigInvalid, "staging buffers must be >= 1");

  Plan plan;
  plan.decomp = decomp;
  plan.kind = kind;
  plan.dir = dir;
  plan.prec = prec;
  plan.dims = dims;
  plan.grid = grid;
  plan.options = opts;
  plan.id = g_plan_ids.fetch_add(1);
  const int last = static_cast<int>(dims.size()) - 1;

  if (decomp != DFFTB_SLAB) {
    // check_rank_occupancy, plan.hpp:114-128
    std::vector<int64_t> hat = dims;
    if (kind != DFFTB_C2C) hat.back() = dims.back() / 2 + 1;
    for (size_t g = 0; g < grid.size(); ++g)
      if (grid[g] > dims[g] && grid[g] > hat[g + 1])
        raise(DFFTB_RankTooLow, "grid factor " + std::to_string(grid[g]) +
                                    " exceeds both axes it decomposes");
    const int d = static_cast<int>(grid.size());
    if (dir == DFFTB_FORWARD) {
      Dist cur = spatial_layout(dims, grid, kind);
      plan.input = cur;
      for (int i = d; i >= 1; --i) {
        Dist after = cur;
        after.hatted[i] = 1;
        int fk = DFFTB_C2C;
        if (i == last && kind == DFFTB_R2C) {
          fk = DFFTB_R2C;
          after.dims[i] = dims[i] / 2 + 1;
          after.complex_el = true;
        }
        plan.stages.push_back(fft(i, dir, fk, cur, after));
        cur = after;
        Dist to = cur;
        to.axis_of_grid[i - 1] = i;
        const bool mode_b = i == 1;
        plan.stages.push_back(transpose(cur, to, i - 1, mode_b));
        if (mode_b) {
          Stage l;
          l.type = StageType::LocalTranspose;
          l.after = to;
          plan.stages.push_back(l);
        }
        cur = to;
      }
      Dist after = cur;
      after.hatted[0] = 1;
      plan.stages.push_back(fft(0, dir, DFFTB_C2C, cur, after));
      plan.output = after;
      if (!(after == frequency_layout(dims, grid, kind)))
        raise(DFFTB_LayoutMismatch, "forward plan assembly is inconsistent");
    } else {
      Dist cur = frequency_layout(dims, grid, kind);
      plan.input = cur;
      Dist after = cur;
      after.hatted[0] = 0;
      plan.stages.push_back(fft(0, dir, DFFTB_C2C, cur, after));
      cur = after;
      for (int i = 1; i <= d; ++i) {
        Dist to = cur;
        to.axis_of_grid[i - 1] = i - 1;
        plan.stages.push_back(transpose(cur, to, i - 1, false));
        cur = to;
        Dist next = cur;
        next.hatted[i] = 0;
        int fk = DFFTB_C2C;
        if (i == last && kind == DFFTB_C2R) {
          fk = DFFTB_C2R;
          next.dims[i] = dims[i];
          next.complex_el = false;
        }
        plan.stages.push_back(fft(i, dir, fk, cur, next));
        cur = next;
      }
      if (opts.normalize) {
        Stage n;
        n.type = StageType::Normalize;
        n.factor = 1.0 / static_cast<double>(product(dims));
        plan.stages.push_back(n);
      }
      plan.output = cur;
      if (!(cur == spatial_layout(dims, grid, kind)))
        raise(DFFTB_LayoutMismatch, "backward plan assembly is inconsistent");
    }
  } else {
    const std::vector<int> g1{grid[0]};
    if (dir == DFFTB_FORWARD) {
      Dist cur = spatial_layout(dims, g1, kind);
      plan.input = cur;
      for (int i = last; i >= 1; --i) {
        Dist after = cur;
        after.hatted[i] = 1;
        int fk = DFFTB_C2C;
        if (i == last && kind == DFFTB_R2C) {
          fk = DFFTB_R2C;
          after.dims[i] = dims[i] / 2 + 1;
          after.complex_el = true;
        }
        plan.stages.push_back(fft(i, dir, fk, cur, after));
        cur = after;
      }
      Dist to = cur;
      to.axis_of_grid[0] = 1;
      plan.stages.push_back(transpose(cur, to, 0, true));
      Stage l;
      l.type = StageType::LocalTranspose;
      l.after = to;
      plan.stages.push_back(l);
      cur = to;
      Dist after = cur;
      after.hatted[0] = 1;
      plan.stages.push_back(fft(0, dir, DFFTB_C2C, cur, after));
      plan.output = after;
      if (!(after == frequency_layout(dims, g1, kind)))
        raise(DFFTB_LayoutMismatch, "slab plan assembly is inconsistent");
    } else {
      Dist cur = frequency_layout(dims, g1, kind);
      plan.input = cur;
      Dist after = cur;
      after.hatted[0] = 0;
      plan.stages.push_back(fft(0, dir, DFFTB_C2C, cur, after));
      cur = after;
      Dist to = cur;
      to.axis_of_grid[0] = 0;
      plan.stages.push_back(transpose(cur, to, 0, false));
      cur = to;
      for (int i = 1; i <= last; ++i) {
        Dist next = cur;
        next.hatted[i] = 0;
        int fk = DFFTB_C2C;
        if (i == last && kind == DFFTB_C2R) {
          fk = DFFTB_C2R;
          next.dims[i] = dims[i];
          next.complex_el = false;
        }
        plan.stages.push_back(fft(i, dir, fk, cur, next));
        cur = next;
      }
      if (opts.normalize) {
        Stage n;
        n.type = StageType::Normalize;
        n.factor = 1.0 / static_cast<double>(product(dims));
        plan.stages.push_back(n);
      }
      plan.output = cur;
      if (!(cur == spatial_layout(dims, g1, kind)))
        raise(DFFTB_LayoutMismatch, "slab plan assembly is inconsistent");
    }
  }
  if (plan.input.any_rank_empty() || plan.output.any_rank_empty())
    plan.warnings.push_back("some ranks own empty blocks");
  return plan;
}

}  // namespace dfftb
