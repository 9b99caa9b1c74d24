// dfftb internal host structures: layouts, plans, contexts.
//
// The plan builder re-derives the reference's stage lists (plan.hpp:149-354)
// and distributions (layout.hpp:106-295) on the host; the executor
// (exec.cu) then lowers a plan to a short program of fused GPU passes and
// group barriers for one rank.
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "dfftb/dfftb.h"

namespace dfftb {

struct Error {
  dfftb_status code;
  std::string what;
};

[[noreturn]] void raise(dfftb_status code, const std::string& what);
const char* status_name(dfftb_status s);

constexpr int kMaxDims = 4;
constexpr int kCopyStreams = 4;
constexpr int kMaxRanks = 64;

// ceil-block partition, layout.hpp:80-92
struct Blocks {
  std::vector<int64_t> counts, offsets;
};
Blocks block_map(int64_t n, int p);

// Distribution, layout.hpp:125-194
struct Dist {
  std::vector<int64_t> dims;
  std::vector<int> grid;          // process grid shape, row-major ranks
  std::vector<int> axis_of_grid;  // grid axis -> tensor axis
  std::vector<char> hatted;
  bool complex_el = true;

  int ndim() const { return static_cast<int>(dims.size()); }
  int gnd() const { return static_cast<int>(grid.size()); }
  int nranks() const;
  std::vector<int> coords_of(int rank) const;
  int rank_of(const std::vector<int>& c) const;
  int grid_axis_of(int axis) const;
  void extents_of(int rank, int64_t* off, int64_t* len) const;
  int64_t local_count(int rank) const;
  int64_t max_local_count() const;
  bool any_rank_empty() const;
  bool operator==(const Dist& o) const {
    return dims == o.dims && grid == o.grid && axis_of_grid == o.axis_of_grid &&
           hatted == o.hatted && complex_el == o.complex_el;
  }
};

enum class StageType { Fft, Transpose, LocalTranspose, Normalize };

struct Stage {
  StageType type = StageType::Fft;
  int axis = 0;        // Fft
  int dir = 0;         // Fft: 0 forward, 1 backward
  int fkind = 0;       // Fft: 0 C2C, 1 R2C, 2 C2R
  Dist before, after;  // Fft before/after; Transpose from/to; LocalT: after
  int grid_axis = 0;   // Transpose
  bool transposed = false;
  double factor = 1.0;  // Normalize
};

struct Plan {
  int decomp = DFFTB_PENCIL;
  int kind = DFFTB_C2C;
  int dir = DFFTB_FORWARD;
  int prec = DFFTB_F64;
  std::vector<int64_t> dims;  // spatial-side dims
  std::vector<int> grid;
  dfftb_plan_options options{};
  Dist input, output;
  std::vector<Stage> stages;
  std::vector<std::string> warnings;
  uint64_t id = 0;

  std::string signature() const;
  int nranks() const { return input.nranks(); }
};

Plan build_plan(const std::vector<int64_t>& dims, int decomp, const std::vector<int>& grid,
                int kind, int dir, int prec, const dfftb_plan_options& opts);
Dist spatial_layout(const std::vector<int64_t>& dims, const std::vector<int>& grid, int kind);
Dist frequency_layout(const std::vector<int64_t>& dims, const std::vector<int>& grid, int kind);

// ---------------------------------------------------------------- contexts

// exported per-rank handle (fixed size, see dfftb_ctx_handle_size)
struct CtxHandle {
  unsigned char ipc[64];  // cudaIpcMemHandle_t
  int64_t pid;
  int64_t device;
  uint64_t dptr;          // base pointer in the owning process
  uint64_t bytes;
  uint64_t magic;
  unsigned char staged;   // the owner allocated staging images (all ranks must agree)
  unsigned char pad[23];
};
static_assert(sizeof(CtxHandle) == 128, "handle must stay 128 bytes");

struct Program;  // exec.cu: one rank's lowered, cached program

// per-op device time of the last timed execute (dfftb_ctx_last_ops)
struct OpTime {
  int kind;      // 0 local pass, 1 exchange pass, 2 sync point, 3 copy-engine DMA
  int stream;    // 0 caller's stream, 1 side stream (overlapped consumer), 2 copy streams
  int n;         // transform length (passes)
  double share;  // passes: fraction of the pass's lanes (chunks < 1)
  double start;  // ms from the start of the execute
  double ms;
};

struct Ctx {
  int rank = 0;
  int nranks = 1;
  int device = 0;
  int prec = DFFTB_F64;
  std::vector<int64_t> dims;
  std::vector<int> grid;
  int decomp = DFFTB_PENCIL;
  int kind_family = 0;  // 0 C2C, 1 R2C/C2R

  // one device region, IPC-exported: [flag page][slot0 p0][slot0 p1][slot1 p0]...
  void* region = nullptr;
  size_t region_bytes = 0;
  size_t flags_bytes = 0;
  size_t exch_bytes = 0;
  int exch_slots = 2;    // exchange buffers per parity in the shared region
  int parities = 2;      // execute parities per slot (1 for a single rank)
  void* work = nullptr;  // private scratch for local->local passes
  size_t work_bytes = 0;
  size_t table_bytes = 0;  // twiddle + Bluestein tables
  // [0] herm max bits, [1] herm imag bits, [2] timeout flag, [3] nonfinite
  // count, [4..5] DC bin of inverse_laplacian, [6] device epoch
  unsigned long long* dstat = nullptr;
  std::map<int, void*> twiddles;                     // N -> device table (prec of the ctx)
  std::map<int, std::pair<void*, void*>> bluestein;  // n -> (chirp, kernel spectrum)

  std::vector<void*> peer_region;  // per world rank, mapped into this process
  std::vector<bool> peer_opened;   // opened through cudaIpcOpenMemHandle
  bool connected = false;
  bool world_mode = false;         // lockstep emulation (execute_world)
  uint64_t exec_count = 0;
  bool c2r_pending = false;

  // streams and events of the overlapped exchange (side stream = consumer
  // pass of a pipelined pair) and of graph capture
  void* side = nullptr;     // cudaStream_t
  void* capture = nullptr;  // cudaStream_t
  std::vector<void*> copies;  // cudaStream_t x kCopyStreams, high priority: staged exchange DMAs + signals
  void* staging = nullptr;  // staged exchange: images of the other members' buffers (lazy)
  size_t staging_bytes = 0;
  std::vector<void*> events;  // cudaEvent_t pool, grown on demand
  // cached programs: key (plan id, buffers, parity, epilogue) -> program
  std::map<std::string, std::shared_ptr<Program>> programs;
  // the two most recent plain executes (a forward / inverse pair alternates):
  // found without formatting the map key
  struct Recent {
    uint64_t id = 0;
    const void* in = nullptr;
    const void* out = nullptr;
    int parity = -1;
    Program* pr = nullptr;
  } recent[2];
  int recent_next = 0;
  std::vector<uint64_t> checked_plans;  // plan ids whose buffer needs fit
  std::vector<OpTime> last_ops;

  void* exch(int rank, int slot, int parity) const;
  uint64_t* flags_of(int rank) const;
};

}  // namespace dfftb
