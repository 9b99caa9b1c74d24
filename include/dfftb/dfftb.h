/*
 * dfftb — B200-native distributed 3-D FFT execute path (AccFFT, arXiv
 * 1506.07933), C ABI.
 *
 * This is the drop-in boundary for the reference's plan / execute /
 * local-size API (the C++20 templates in /root/reference/proj/include/dfft/,
 * "the reference" below).  Every entry point names the reference interface it
 * replaces.  Plain pointers and sizes only; device buffers are CUDA device
 * pointers, `stream` is a cudaStream_t passed as void*.
 *
 * Threading/collectives follow the reference (plan.hpp:356-363):
 * every rank creates the same plan, creates its context, exchanges the
 * context handles (any out-of-band all-gather; torch.distributed in the
 * Python binding) and then calls dfftb_execute in the same order.
 */
#ifndef DFFTB_H
#define DFFTB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status = dfft::ErrorCode ordinal + 1 (errors.hpp:13-44); 0 is success. */
typedef enum {
  DFFTB_OK = 0,
  DFFTB_ZeroLength = 1,
  DFFTB_OutOfBounds,
  DFFTB_TooLarge,
  DFFTB_LengthMismatch,
  DFFTB_NonHermitian,
  DFFTB_SlabTooManyRanks,
  DFFTB_OutOfRange,
  DFFTB_InvalidRank,
  DFFTB_TagMismatchTimeout,
  DFFTB_Deadlock,
  DFFTB_WorkerPanic,
  DFFTB_CountMismatch,
  DFFTB_IncompatibleLayouts,
  DFFTB_ArenaExhausted,
  DFFTB_GridMismatch,
  DFFTB_RankTooLow,
  DFFTB_LayoutMismatch,
  DFFTB_NotFrequencyLayout,
  DFFTB_NonZeroMean,
  DFFTB_BadMagic,
  DFFTB_DimMismatch,
  DFFTB_TruncatedFile,
  DFFTB_ConfigInvalid,
  /* B200-side failures with no reference counterpart */
  DFFTB_CudaError = 100,
  DFFTB_Unsupported = 101
} dfftb_status;

/* TransformKind (layout.hpp:289), Direction (kernels.hpp:26) */
enum { DFFTB_C2C = 0, DFFTB_R2C = 1, DFFTB_C2R = 2 };
enum { DFFTB_FORWARD = 0, DFFTB_BACKWARD = 1 };
/* plan_slab / plan_pencil / plan_general (plan.hpp:242-354) */
enum { DFFTB_SLAB = 0, DFFTB_PENCIL = 1, DFFTB_GENERAL = 2 };
/* template parameter T: bytes per real component */
enum { DFFTB_F32 = 4, DFFTB_F64 = 8 };
/* ExchangePath (exchange.hpp:425).  All three give byte-identical results,
 * as in the reference.  BLOCKING and STAGED (the staging hop of
 * exchange.hpp:225-246): an exchange pass that feeds a local pass stores the
 * other members' parts into local staging images, and copy-engine DMAs move
 * them over NVLink chunk by chunk (chunks_per_peer > 1, else 8) while the
 * SMs run the following local pass; any other exchange pass stores every
 * member's part straight into its buffer over NVLink (all of them with the
 * environment variable DFFTB_DMA=0).  PIPELINED with chunks_per_peer = C > 1
 * instead chunks such an exchange pass into C pieces overlapped with the
 * local pass on a second stream and a share of the SMs
 * (pipelined_all_to_all, exchange.hpp:323-423). */
enum { DFFTB_EXCHANGE_BLOCKING = 0, DFFTB_EXCHANGE_STAGED = 1, DFFTB_EXCHANGE_PIPELINED = 2 };
/* plan layout sides */
enum { DFFTB_INPUT = 0, DFFTB_OUTPUT = 1 };

/* PlanOptions, plan.hpp:48-54 */
typedef struct {
  int exchange;        /* DFFTB_EXCHANGE_* */
  int normalize;       /* backward applies 1/N once (default 1) */
  int chunks_per_peer; /* >= 1; chunks of the overlapped exchange (staged / pipelined) */
  int staging_buffers; /* >= 1; no staging copies exist on B200 (accepted) */
  int validate_finite; /* reject NaN/Inf input (ConfigInvalid, reported after
                          the launches so the ranks stay in lockstep) */
} dfftb_plan_options;

/* TimingBreakdown, timing.hpp:16-37 (seconds) */
typedef struct {
  double local_fft, pack, unpack, staging_copy, wire_comm, total;
} dfftb_timing;

typedef struct dfftb_plan_s* dfftb_plan;
typedef struct dfftb_ctx_s* dfftb_ctx;

/* ---- plans ------------------------------------------------------------ */

void dfftb_plan_options_default(dfftb_plan_options* opts);

/* Replaces plan_slab (plan.hpp:267-354; grid_ndim == 1, grid[0] = ranks),
 * plan_pencil (plan.hpp:242-250) and plan_general (plan.hpp:253-262).
 * precision: DFFTB_F32 / DFFTB_F64.  Same validation and error codes. */
dfftb_status dfftb_plan_create(int ndim, const int64_t* dims, int decomp,
                               int grid_ndim, const int* grid, int kind,
                               int direction, int precision,
                               const dfftb_plan_options* opts, dfftb_plan* out);
void dfftb_plan_destroy(dfftb_plan plan);

/* Plan<T>::signature / fft_stage_count / transpose_stage_count (plan.hpp:70-98) */
dfftb_status dfftb_plan_signature(dfftb_plan plan, char* buf, size_t len);
int dfftb_plan_fft_stage_count(dfftb_plan plan);
int dfftb_plan_transpose_stage_count(dfftb_plan plan);
int dfftb_plan_nranks(dfftb_plan plan);
int dfftb_plan_precision(dfftb_plan plan);
int dfftb_plan_kind(dfftb_plan plan);
int dfftb_plan_direction(dfftb_plan plan);
/* Plan<T>::warnings ("some ranks own empty blocks", plan.hpp:231-233) */
int dfftb_plan_warning_count(dfftb_plan plan);
const char* dfftb_plan_warning(dfftb_plan plan, int i);

/* ---- local-size API (layout.hpp, dist_tensor.hpp:28-44) ---------------- */

/* block_map (layout.hpp:80-92) */
dfftb_status dfftb_block_map(int64_t n, int p, int64_t* counts, int64_t* offsets);
/* Plan.input / Plan.output Distribution: global dims (hatted on the
 * frequency side), element kind (0 real, 1 complex), grid-axis -> tensor
 * axis map, hatted flags. */
dfftb_status dfftb_plan_layout(dfftb_plan plan, int side, int64_t* dims,
                               int* element_complex, int* axis_of_grid,
                               int* hatted);
/* Distribution::extents_of (layout.hpp:165-179) */
dfftb_status dfftb_plan_local_extents(dfftb_plan plan, int rank, int side,
                                      int64_t* offsets, int64_t* lengths);
/* Distribution::local_count (layout.hpp:181); -1 on a bad rank */
int64_t dfftb_plan_local_count(dfftb_plan plan, int rank, int side);
/* local_index (layout.hpp:272-295) */
dfftb_status dfftb_local_index(dfftb_plan plan, int side, const int64_t* coord,
                               int* rank, int64_t* offset);

/* Element counts rank `rank` sends to / receives from each member of the
 * grid-axis group of the plan's `transpose_index`-th TransposeStage, in
 * group-rank order (make_transpose_step send/recv counts,
 * exchange.hpp:531-540).  group_size receives the member count (<= 64). */
dfftb_status dfftb_plan_exchange_counts(dfftb_plan plan, int rank, int transpose_index,
                                        int64_t* send_counts, int64_t* recv_counts,
                                        int* group_size);

/* Device bytes dfftb_ctx_create allocates for this plan's family on rank
 * `rank` (the symmetric exchange region: flag page + one buffer per
 * transpose stage and execute parity, plus the private work buffer); the
 * reference sizes its StagingArena in make_context (plan.hpp:365-390,
 * exchange.hpp:250-262).  Host-only: no CUDA call. */
dfftb_status dfftb_workspace_bytes(dfftb_plan plan, int rank, uint64_t* bytes);

/* ---- execution contexts (make_context, plan.hpp:365-390) ---------------- */

/* Per-rank context on CUDA device `device`: allocates the symmetric exchange
 * buffers and the twiddle tables.  Collective in spirit: all ranks must then
 * call dfftb_ctx_connect with every rank's exported handle. */
dfftb_status dfftb_ctx_create(dfftb_plan plan, int rank, int device, dfftb_ctx* out);
size_t dfftb_ctx_handle_size(void);
dfftb_status dfftb_ctx_export_handle(dfftb_ctx ctx, void* handle);
/* handles: nranks * dfftb_ctx_handle_size() bytes, in world-rank order
 * (the reference's split_grid_axis colors/keys, exchange.hpp:594-603, are
 * derived from the grid inside). */
dfftb_status dfftb_ctx_connect(dfftb_ctx ctx, const void* handles);
void dfftb_ctx_destroy(dfftb_ctx ctx);

/* execute (plan.hpp:463-535): d_in holds this rank's block of plan.input
 * (row-major, last axis fastest; interleaved complex or real), d_out receives
 * its block of plan.output.  Out-of-place; d_in is not modified.  Enqueued on
 * `stream`; the call returns without synchronizing unless `timers` is given
 * (then per-stage device times are filled in, TimingBreakdown semantics) or
 * flags has DFFTB_EXEC_SYNC (then deferred errors such as NonHermitian and
 * exchange timeouts are reported by this call). */
enum { DFFTB_EXEC_SYNC = 1 };
dfftb_status dfftb_execute(dfftb_plan plan, dfftb_ctx ctx, const void* d_in,
                           void* d_out, void* stream, int flags,
                           dfftb_timing* timers);
/* Deferred-error check: synchronizes `stream` and reports NonHermitian /
 * Deadlock (peer timeout) raised by earlier executes on this context. */
dfftb_status dfftb_ctx_check(dfftb_ctx ctx, void* stream);

/* Single-device emulation of a P-rank world (test harness for the exchange
 * logic when fewer GPUs than ranks exist): creates P connected contexts on
 * one device, and runs all ranks' stages in lockstep on one stream. */
dfftb_status dfftb_world_create(dfftb_plan plan, int device, dfftb_ctx* ctxs);
/* The same world over several devices of this process: rank r's context on
 * devices[r % ndevices].  Exchange stores cross NVLink through direct peer
 * pointers; dfftb_execute_world orders the ranks' passes with cross-device
 * CUDA events issued by the host (no kernel waits on another), on the
 * contexts' own streams, and makes `stream` (on ctxs[0]'s device) wait for
 * all of them. */
dfftb_status dfftb_world_create_devices(dfftb_plan plan, int ndevices, const int* devices,
                                        dfftb_ctx* ctxs);
dfftb_status dfftb_execute_world(dfftb_plan plan, dfftb_ctx* ctxs,
                                 const void* const* d_in, void* const* d_out,
                                 void* stream, int flags);

/* ---- helpers ----------------------------------------------------------- */

/* Device fill of this rank's block with the reference bench's seeded field
 * (bench.cpp:132-136): value at global flat index f of the side's layout is
 * (u(seed*0x10001 + 2f), complex ? u(... + 1) : 0). */
dfftb_status dfftb_fill_seeded(dfftb_plan plan, int rank, int side, uint64_t seed,
                               int complex_field, void* d_buf, void* stream);

/* error_code_name (errors.hpp:64-91) and the message of the last failure on
 * this thread, formatted like dfft::Error::what(): "<CodeName>: <what>". */
const char* dfftb_error_name(dfftb_status status);
const char* dfftb_last_error_message(void);

/* Per-op device times of the last execute that was given `timers`, in
 * program order: kinds[i] 0 = local FFT pass, 1 = exchange pass (FFT whose
 * stores go to other ranks' buffers or their staging images), 2 = sync
 * point, 3 = copy-engine DMA of the staged exchange; streams[i] 1 = the
 * overlapped pass on the context's side stream, 2 = its copy streams;
 * lengths[i] = the transform length; shares[i] = the fraction of the pass's
 * lanes a (chunked) pass launch covers; starts[i] = ms from the start of the
 * execute.  Any array may be NULL.  Returns the op count (arrays filled up
 * to `max`). */
int dfftb_ctx_last_ops(dfftb_ctx ctx, int* kinds, int* streams, int* lengths, double* shares, double* starts,
                       double* ms, int max);

/* Number of dfftb kernels launched by this process so far (evidence counter). */
uint64_t dfftb_kernel_launch_count(void);

/* ---- spectral operators (spectral.hpp:133-309) --------------------------
 * Applied to this rank's block of a FORWARD plan's output (the frequency
 * layout; NotFrequencyLayout otherwise), on device:
 *   DFFTB_SPECTRAL_DERIV         out (+)= i k_axis (.) in, Nyquist mode zeroed
 *                                (axis_k_deriv, spectral.hpp:24-56, 131-164)
 *   DFFTB_SPECTRAL_LAPLACIAN     out (+)= -|k|^2 (.) in        (:219-249)
 *   DFFTB_SPECTRAL_INV_LAPLACIAN out (+)= in / -|k|^2, k = 0 pinned to 0; the
 *                                owner of the k = 0 bin checks |in(0)| <= 1e-12 N
 *                                and returns NonZeroMean otherwise (:255-309)
 * k_a = 2 pi / L_a * signed index (R2C half axis: non-negative).
 * domain_lengths: ndim values (NULL = 2 pi each).  accumulate != 0 adds into
 * out (divergence).  in == out is allowed. */
enum { DFFTB_SPECTRAL_DERIV = 0, DFFTB_SPECTRAL_LAPLACIAN = 1, DFFTB_SPECTRAL_INV_LAPLACIAN = 2 };
dfftb_status dfftb_spectral_apply(dfftb_plan forward_plan, int rank, int op, int axis,
                                  const double* domain_lengths, const void* d_in, void* d_out,
                                  int accumulate, void* stream);
/* Forward transform of d_in with a spectral operator fused into the last
 * pass's store epilogue: d_out (+)= op(execute(forward_plan, d_in)), the same
 * values as dfftb_execute followed by dfftb_spectral_apply, with one pass
 * over the spectrum less.  Collective like dfftb_execute (replaces the
 * forward-then-multiply pair in derivative / laplacian / inverse_laplacian /
 * divergence, spectral.hpp:131-309).  The k = 0 owner checks the zero mean
 * for DFFTB_SPECTRAL_INV_LAPLACIAN (NonZeroMean). */
dfftb_status dfftb_execute_spectral(dfftb_plan forward_plan, dfftb_ctx ctx, const void* d_in, void* d_out,
                                    int op, int axis, const double* domain_lengths, int accumulate,
                                    void* stream, int flags);
/* dfftb_execute_spectral for every rank of an emulated world
 * (dfftb_world_create / _devices), in lockstep like dfftb_execute_world. */
dfftb_status dfftb_execute_world_spectral(dfftb_plan forward_plan, dfftb_ctx* ctxs, const void* const* d_in,
                                          void* const* d_out, int op, int axis, const double* domain_lengths,
                                          int accumulate, void* stream, int flags);
/* wavenumbers (spectral.hpp:24-56): the local k values of `axis` for this
 * rank's frequency block (length = local extent); deriv != 0 gives
 * axis_k_deriv (Nyquist zeroed), else axis_k. */
dfftb_status dfftb_wavenumbers(dfftb_plan forward_plan, int rank, int axis, int deriv,
                               const double* domain_lengths, double* k_out);

#ifdef __cplusplus
}
#endif
#endif /* DFFTB_H */
