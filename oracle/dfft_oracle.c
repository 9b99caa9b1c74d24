/*
 * TEST INFRASTRUCTURE — CPU restatement of the reference execute path.
 * See dfft_oracle.h for the rules on who may use it.  Citations are into
 * /root/reference/proj.
 */
#include "dfft_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif
#define MAXD 4
#define MAXP 64

/* ------------------------------------------------------------------ layout */

/* layout.hpp:80-92 — ceil-block partition; trailing blocks may be empty */
void oracle_block_map(int64_t n, int p, int64_t* counts, int64_t* offsets) {
  const int64_t block = p > 0 ? (n + p - 1) / p : 0;
  for (int r = 0; r < p; ++r) {
    int64_t lo = r * block < n ? r * block : n;
    int64_t hi = (r + 1) * block < n ? (r + 1) * block : n;
    offsets[r] = lo;
    counts[r] = hi - lo;
  }
}

typedef struct {
  int64_t dims[MAXD];
  int ndim;
  int grid[MAXD];
  int gnd;
  int axis_of_grid[MAXD];
  int hatted[MAXD];
  int complex_el; /* ElementKind: 0 Real, 1 Complex */
} Dist;

static int grid_size(const Dist* d) {
  int p = 1;
  for (int g = 0; g < d->gnd; ++g) p *= d->grid[g];
  return p;
}

/* ProcessGrid::coords_of, layout.hpp:50-57 (row-major) */
static void coords_of(const int* shape, int gnd, int rank, int* c) {
  for (int g = gnd; g-- > 0;) {
    c[g] = rank % shape[g];
    rank /= shape[g];
  }
}

/* ProcessGrid::rank_of, layout.hpp:59-63 */
static int rank_of(const int* shape, int gnd, const int* c) {
  int r = 0;
  for (int g = 0; g < gnd; ++g) r = r * shape[g] + c[g];
  return r;
}

static int grid_axis_of(const Dist* d, int axis) {
  for (int g = 0; g < d->gnd; ++g)
    if (d->axis_of_grid[g] == axis) return g;
  return -1;
}

/* Distribution::extents_of, layout.hpp:165-179 */
static void extents_of(const Dist* d, int rank, int64_t* off, int64_t* len) {
  int c[MAXD];
  coords_of(d->grid, d->gnd, rank, c);
  for (int a = 0; a < d->ndim; ++a) {
    int g = grid_axis_of(d, a);
    if (g < 0) {
      off[a] = 0;
      len[a] = d->dims[a];
    } else {
      int64_t cnt[MAXP], offs[MAXP];
      oracle_block_map(d->dims[a], d->grid[g], cnt, offs);
      off[a] = offs[c[g]];
      len[a] = cnt[c[g]];
    }
  }
}

static int64_t local_count(const Dist* d, int rank) {
  int64_t off[MAXD], len[MAXD], n = 1;
  extents_of(d, rank, off, len);
  for (int a = 0; a < d->ndim; ++a) n *= len[a];
  return n;
}

static int dist_equal(const Dist* a, const Dist* b) {
  if (a->ndim != b->ndim || a->gnd != b->gnd || a->complex_el != b->complex_el)
    return 0;
  for (int i = 0; i < a->ndim; ++i)
    if (a->dims[i] != b->dims[i] || a->hatted[i] != b->hatted[i]) return 0;
  for (int g = 0; g < a->gnd; ++g)
    if (a->grid[g] != b->grid[g] || a->axis_of_grid[g] != b->axis_of_grid[g])
      return 0;
  return 1;
}

/* detail::check_grid, layout.hpp:211-226 */
static int check_grid(int ndim, const int64_t* dims, int gnd, const int* grid) {
  if (ndim < 2) return ORACLE_IncompatibleLayouts;
  if (gnd < 1 || gnd > ndim - 1) return ORACLE_IncompatibleLayouts;
  for (int g = 0; g < gnd; ++g)
    if (grid[g] < 1) return ORACLE_IncompatibleLayouts;
  if (gnd == 1 && grid[0] > dims[0]) return ORACLE_SlabTooManyRanks;
  return 0;
}

/* spatial_layout, layout.hpp:232-248 */
static int spatial_layout(int ndim, const int64_t* dims, int gnd,
                          const int* grid, int kind, Dist* d) {
  int st = check_grid(ndim, dims, gnd, grid);
  if (st) return st;
  memset(d, 0, sizeof(*d));
  d->ndim = ndim;
  d->gnd = gnd;
  for (int a = 0; a < ndim; ++a) d->dims[a] = dims[a];
  for (int g = 0; g < gnd; ++g) {
    d->grid[g] = grid[g];
    d->axis_of_grid[g] = g;
  }
  d->complex_el = kind == 0;
  return 0;
}

/* frequency_layout, layout.hpp:252-268; hat_dims :201-207 */
static int frequency_layout(int ndim, const int64_t* dims, int gnd,
                            const int* grid, int kind, Dist* d) {
  int st = check_grid(ndim, dims, gnd, grid);
  if (st) return st;
  memset(d, 0, sizeof(*d));
  d->ndim = ndim;
  d->gnd = gnd;
  for (int a = 0; a < ndim; ++a) {
    d->dims[a] = dims[a];
    d->hatted[a] = 1;
  }
  if (kind != 0) d->dims[ndim - 1] = dims[ndim - 1] / 2 + 1;
  for (int g = 0; g < gnd; ++g) {
    d->grid[g] = grid[g];
    d->axis_of_grid[g] = g + 1;
  }
  d->complex_el = 1;
  return 0;
}

/* ------------------------------------------------------------------- plans */

enum { ST_FFT, ST_TRANSPOSE, ST_LOCALT, ST_NORM };
enum { FK_C2C, FK_R2C, FK_C2R };

typedef struct {
  int type;
  int axis, dir, fkind;      /* LocalFftStage, plan.hpp:21-26 */
  Dist before, after;        /* also from/to of TransposeStage */
  int grid_axis, transposed; /* TransposeStage, plan.hpp:29-34 */
  double factor;             /* NormalizeStage */
} Stage;

typedef struct {
  Dist input, output;
  Stage st[16];
  int nst;
} Plan;

static void push(Plan* p, Stage s) { p->st[p->nst++] = s; }

static Stage fft_stage(int axis, int dir, int fk, const Dist* b, const Dist* a) {
  Stage s;
  memset(&s, 0, sizeof(s));
  s.type = ST_FFT;
  s.axis = axis;
  s.dir = dir;
  s.fkind = fk;
  s.before = *b;
  s.after = *a;
  return s;
}

static Stage tr_stage(const Dist* from, const Dist* to, int g, int transposed) {
  Stage s;
  memset(&s, 0, sizeof(s));
  s.type = ST_TRANSPOSE;
  s.before = *from;
  s.after = *to;
  s.grid_axis = g;
  s.transposed = transposed;
  return s;
}

/* check_kind_direction, plan.hpp:103-110 */
static int check_kind_direction(int kind, int dir) {
  if (kind == 1 && dir != 0) return ORACLE_ConfigInvalid;
  if (kind == 2 && dir != 1) return ORACLE_ConfigInvalid;
  return 0;
}

/* check_rank_occupancy, plan.hpp:114-128 */
static int check_rank_occupancy(int ndim, const int64_t* dims, int gnd,
                                const int* grid, int kind) {
  int64_t hat[MAXD];
  for (int a = 0; a < ndim; ++a) hat[a] = dims[a];
  if (kind != 0) hat[ndim - 1] = dims[ndim - 1] / 2 + 1;
  for (int g = 0; g < gnd; ++g)
    if (grid[g] > dims[g] && grid[g] > hat[g + 1]) return ORACLE_RankTooLow;
  return 0;
}

static int64_t total(int ndim, const int64_t* dims) {
  int64_t n = 1;
  for (int a = 0; a < ndim; ++a) n *= dims[a];
  return n;
}

/* detail::build_nd_plan, plan.hpp:149-236 (pencil and general) */
static int build_nd_plan(int ndim, const int64_t* dims, int gnd, const int* grid,
                         int kind, int dir, int normalize, Plan* plan) {
  int st = check_kind_direction(kind, dir);
  if (st) return st;
  st = check_rank_occupancy(ndim, dims, gnd, grid, kind);
  if (st) return st;
  memset(plan, 0, sizeof(*plan));
  const int d = gnd, last = ndim - 1;
  Dist cur, after, to;
  if (dir == 0) {
    if ((st = spatial_layout(ndim, dims, gnd, grid, kind, &cur))) return st;
    plan->input = cur;
    for (int i = d; i >= 1; --i) {
      after = cur;
      after.hatted[i] = 1;
      int fk = FK_C2C;
      if (i == last && kind == 1) {
        fk = FK_R2C;
        after.dims[i] = dims[i] / 2 + 1;
        after.complex_el = 1;
      }
      push(plan, fft_stage(i, dir, fk, &cur, &after));
      cur = after;
      to = cur;
      to.axis_of_grid[i - 1] = i;
      const int mode_b = i == 1;
      push(plan, tr_stage(&cur, &to, i - 1, mode_b));
      if (mode_b) {
        Stage l;
        memset(&l, 0, sizeof(l));
        l.type = ST_LOCALT;
        l.after = to;
        push(plan, l);
      }
      cur = to;
    }
    after = cur;
    after.hatted[0] = 1;
    push(plan, fft_stage(0, dir, FK_C2C, &cur, &after));
    cur = after;
    plan->output = cur;
    Dist want;
    frequency_layout(ndim, dims, gnd, grid, kind, &want);
    if (!dist_equal(&cur, &want)) return ORACLE_LayoutMismatch;
  } else {
    if ((st = frequency_layout(ndim, dims, gnd, grid, kind, &cur))) return st;
    plan->input = cur;
    after = cur;
    after.hatted[0] = 0;
    push(plan, fft_stage(0, dir, FK_C2C, &cur, &after));
    cur = after;
    for (int i = 1; i <= d; ++i) {
      to = cur;
      to.axis_of_grid[i - 1] = i - 1;
      push(plan, tr_stage(&cur, &to, i - 1, 0));
      cur = to;
      Dist next = cur;
      next.hatted[i] = 0;
      int fk = FK_C2C;
      if (i == last && kind == 2) {
        fk = FK_C2R;
        next.dims[i] = dims[i];
        next.complex_el = 0;
      }
      push(plan, fft_stage(i, dir, fk, &cur, &next));
      cur = next;
    }
    if (normalize) {
      Stage n;
      memset(&n, 0, sizeof(n));
      n.type = ST_NORM;
      n.factor = 1.0 / (double)total(ndim, dims);
      push(plan, n);
    }
    plan->output = cur;
    Dist want;
    spatial_layout(ndim, dims, gnd, grid, kind, &want);
    if (!dist_equal(&cur, &want)) return ORACLE_LayoutMismatch;
  }
  return 0;
}

/* plan_slab, plan.hpp:267-354 */
static int build_slab_plan(int ndim, const int64_t* dims, int ranks, int kind,
                           int dir, int normalize, Plan* plan) {
  if (ndim < 2) return ORACLE_GridMismatch;
  if (ranks < 1) return ORACLE_GridMismatch;
  if (ranks > dims[0]) return ORACLE_SlabTooManyRanks;
  int st = check_kind_direction(kind, dir);
  if (st) return st;
  memset(plan, 0, sizeof(*plan));
  const int grid[1] = {ranks};
  const int last = ndim - 1;
  Dist cur, after, to;
  if (dir == 0) {
    if ((st = spatial_layout(ndim, dims, 1, grid, kind, &cur))) return st;
    plan->input = cur;
    for (int i = last; i >= 1; --i) {
      after = cur;
      after.hatted[i] = 1;
      int fk = FK_C2C;
      if (i == last && kind == 1) {
        fk = FK_R2C;
        after.dims[i] = dims[i] / 2 + 1;
        after.complex_el = 1;
      }
      push(plan, fft_stage(i, dir, fk, &cur, &after));
      cur = after;
    }
    to = cur;
    to.axis_of_grid[0] = 1;
    push(plan, tr_stage(&cur, &to, 0, 1));
    Stage l;
    memset(&l, 0, sizeof(l));
    l.type = ST_LOCALT;
    l.after = to;
    push(plan, l);
    cur = to;
    after = cur;
    after.hatted[0] = 1;
    push(plan, fft_stage(0, dir, FK_C2C, &cur, &after));
    plan->output = after;
    Dist want;
    frequency_layout(ndim, dims, 1, grid, kind, &want);
    if (!dist_equal(&after, &want)) return ORACLE_LayoutMismatch;
  } else {
    if ((st = frequency_layout(ndim, dims, 1, grid, kind, &cur))) return st;
    plan->input = cur;
    after = cur;
    after.hatted[0] = 0;
    push(plan, fft_stage(0, dir, FK_C2C, &cur, &after));
    cur = after;
    to = cur;
    to.axis_of_grid[0] = 0;
    push(plan, tr_stage(&cur, &to, 0, 0));
    cur = to;
    for (int i = 1; i <= last; ++i) {
      Dist next = cur;
      next.hatted[i] = 0;
      int fk = FK_C2C;
      if (i == last && kind == 2) {
        fk = FK_C2R;
        next.dims[i] = dims[i];
        next.complex_el = 0;
      }
      push(plan, fft_stage(i, dir, fk, &cur, &next));
      cur = next;
    }
    if (normalize) {
      Stage n;
      memset(&n, 0, sizeof(n));
      n.type = ST_NORM;
      n.factor = 1.0 / (double)total(ndim, dims);
      push(plan, n);
    }
    plan->output = cur;
    Dist want;
    spatial_layout(ndim, dims, 1, grid, kind, &want);
    if (!dist_equal(&cur, &want)) return ORACLE_LayoutMismatch;
  }
  return 0;
}

static int build_plan(int ndim, const int64_t* dims, int decomp, int gnd,
                      const int* grid, int kind, int dir, int normalize,
                      Plan* plan) {
  if (ndim > MAXD) return ORACLE_ConfigInvalid;
  if (decomp == 0) {
    if (gnd != 1) return ORACLE_GridMismatch;
    return build_slab_plan(ndim, dims, grid[0], kind, dir, normalize, plan);
  }
  if (decomp == 1) { /* plan_pencil, plan.hpp:242-250 */
    if (ndim != 3 || gnd != 2) return ORACLE_GridMismatch;
  } else { /* plan_general, plan.hpp:253-262 */
    if (ndim < 2 || gnd != ndim - 1) return ORACLE_GridMismatch;
  }
  return build_nd_plan(ndim, dims, gnd, grid, kind, dir, normalize, plan);
}

/* Plan::signature, plan.hpp:82-98 */
static void signature(const Plan* p, char* out) {
  char* o = out;
  for (int i = 0; i < p->nst; ++i) {
    const Stage* s = &p->st[i];
    if (s->type == ST_FFT) o += sprintf(o, "F%d;", s->axis);
    else if (s->type == ST_TRANSPOSE)
      o += sprintf(o, "T%d%s;", s->grid_axis, s->transposed ? "x" : "");
    else if (s->type == ST_LOCALT) o += sprintf(o, "L;");
    else o += sprintf(o, "N;");
  }
  *o = 0;
}

int oracle_local_extents(int ndim, const int64_t* dims, int decomp, int gnd,
                         const int* grid, int kind, int dir, int side, int rank,
                         int64_t* offsets, int64_t* lengths) {
  Plan plan;
  int st = build_plan(ndim, dims, decomp, gnd, grid, kind, dir, 1, &plan);
  if (st) return st;
  const Dist* d = side == 0 ? &plan.input : &plan.output;
  if (rank < 0 || rank >= grid_size(d)) return ORACLE_InvalidRank;
  extents_of(d, rank, offsets, lengths);
  return 0;
}

/* ------------------------------------------------------------ seeded field */

/* bench.cpp:22-28 */
static double unit_from_hash(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return (double)(x >> 11) * 0x1.0p-52 - 1.0;
}

/* bench.cpp:132-136 */
double oracle_seeded(uint64_t seed, int64_t flat, int part) {
  return unit_from_hash(seed * 0x10001ULL + 2ULL * (uint64_t)flat + (uint64_t)part);
}

void oracle_seeded_fill(uint64_t seed, int64_t n, int complex_field, int prec,
                        void* out) {
  for (int64_t i = 0; i < n; ++i) {
    double re = oracle_seeded(seed, i, 0);
    if (complex_field) {
      double im = oracle_seeded(seed, i, 1);
      if (prec == 8) {
        ((double*)out)[2 * i] = re;
        ((double*)out)[2 * i + 1] = im;
      } else {
        ((float*)out)[2 * i] = (float)re;
        ((float*)out)[2 * i + 1] = (float)im;
      }
    } else if (prec == 8) {
      ((double*)out)[i] = re;
    } else {
      ((float*)out)[i] = (float)re;
    }
  }
}

/* -------------------------------------------------- typed execute (double) */
#define R double
#define SFX(x) x##_f64
#define HERM_TOL 1e-6
#include "dfft_oracle_impl.inc"
#undef R
#undef SFX
#undef HERM_TOL

/* --------------------------------------------------- typed execute (float) */
#define R float
#define SFX(x) x##_f32
#define HERM_TOL 1e-2f
#include "dfft_oracle_impl.inc"
#undef R
#undef SFX
#undef HERM_TOL

int oracle_execute(int prec, int ndim, const int64_t* dims, int decomp, int gnd,
                   const int* grid, int kind, int dir, int normalize,
                   const void* global_in, void* global_out, char* sig) {
  Plan plan;
  int st = build_plan(ndim, dims, decomp, gnd, grid, kind, dir, normalize, &plan);
  if (st) return st;
  if (sig) signature(&plan, sig);
  if (prec == 8) return execute_f64(&plan, global_in, global_out);
  if (prec == 4) return execute_f32(&plan, global_in, global_out);
  return ORACLE_ConfigInvalid;
}

int oracle_fft_1d(double* data, int64_t n, int dir) {
  if (n < 1) return ORACLE_ZeroLength;
  if (n & (n - 1)) return ORACLE_ConfigInvalid;
  radix2_inplace_f64(data, n, 1, dir);
  return 0;
}

/* dft_oracle, kernels.hpp:396-444 */
int oracle_dft(const double* in, int ndim, const int64_t* dims, int dir,
               double* out) {
  int64_t tot = 1;
  for (int d = 0; d < ndim; ++d) {
    if (dims[d] < 1) return ORACLE_ZeroLength;
    tot *= dims[d];
  }
  if (tot > ((int64_t)1 << 16)) return ORACLE_TooLarge;
  const double sign = dir == 0 ? -1.0 : 1.0;
  double* w[MAXD];
  for (int d = 0; d < ndim; ++d) {
    w[d] = (double*)malloc(sizeof(double) * 2 * dims[d]);
    const double step = sign * 2.0 * M_PI / (double)dims[d];
    for (int64_t r = 0; r < dims[d]; ++r) {
      /* std::polar(1.0, step*r) */
      w[d][2 * r] = cos(step * (double)r);
      w[d][2 * r + 1] = sin(step * (double)r);
    }
  }
  int64_t kc[MAXD] = {0}, jc[MAXD];
  for (int64_t k = 0; k < tot; ++k) {
    double ar = 0, ai = 0;
    for (int d = 0; d < ndim; ++d) jc[d] = 0;
    for (int64_t j = 0; j < tot; ++j) {
      double pr = 1, pi = 0;
      for (int d = 0; d < ndim; ++d) {
        const double* wv = &w[d][2 * ((jc[d] * kc[d]) % dims[d])];
        double nr = pr * wv[0] - pi * wv[1];
        double ni = pr * wv[1] + pi * wv[0];
        pr = nr;
        pi = ni;
      }
      const double xr = in[2 * j], xi = in[2 * j + 1];
      ar += xr * pr - xi * pi;
      ai += xr * pi + xi * pr;
      for (int d = ndim; d-- > 0;) {
        if (++jc[d] < dims[d]) break;
        jc[d] = 0;
      }
    }
    out[2 * k] = ar;
    out[2 * k + 1] = ai;
    for (int d = ndim; d-- > 0;) {
      if (++kc[d] < dims[d]) break;
      kc[d] = 0;
    }
  }
  for (int d = 0; d < ndim; ++d) free(w[d]);
  return 0;
}
