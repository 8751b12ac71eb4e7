/*
 * axe_oracle.c -- plain, slow, obviously-correct CPU oracle for Axe layouts.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this file.  It
 * shares no code, header, table or helper with the product library under
 * paper_2601_19092_b200/ and it never calls into it.
 *
 * Every function is the plain definition from the paper, evaluated element by
 * element in int64, with no planning, canonicalisation, vectorisation or
 * reordering.  Citations are "P:<line>" into /root/reference/PAPER.md.
 *
 *   digits    d_i(x) = floor(x / p_i) mod e_i, p_{n-1} = 1, p_i = p_{i+1} e_{i+1}
 *             ("standard lexicographic unflattening"; digits P:774-778)
 *   f_D(x)    = sum_i (d_i(x) s_i) @ a_i
 *   f_R(r)    = sum_t (r_t s_{J_t}) @ a_{J_t}, r lexicographic
 *   f_L(x)    = { f_D(x) + f_R(r) + O : r }, R empty -> {f_D(x) + O}
 *   address   = base pointer + memory components of the coordinate
 *   storage   idx = sum_k ((c[a_k] / div_k) mod ext_k) * prod_{j>k} ext_j
 *             (reading R17 of DESIGN.md: how a coordinate on named axes is
 *              laid out in a byte buffer; the paper is silent)
 *   swizzle   byte' = byte ^ (((byte >> (M+S)) & (2^B - 1)) << M)
 *             (the "hardware swizzle" of the TMA atom; bit pattern per
 *              reading R16: SW128 = (3,4,3), SW64 = (2,4,3), SW32 = (1,4,3))
 *   copy      dst[f_L^dst(x)] = src[f_D^src(x) + O^src] for every x      (reading R4:
 *             the r = 0 source replica; P:122 replicas are copies)
 *   redistribute: as copy, the `gpuid` coordinate selecting the rank buffer
 *
 *   reduce    dst(y) = sum_k src(k E_D(dst) + y), fp64 sum rounded once (reading R24,
 *             P:399-403; see the reduction section at the end)
 *
 * Parity pins live in tests/test_oracle_pins.py (paper worked examples,
 * library special cases, invariants, TMA hardware for the swizzle).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- status codes (the oracle's own; deliberately not the product's) ---- */
#define ORA_OK 0
#define ORA_EINVAL 1     /* bad iter / layout / storage description         */
#define ORA_EDOMAIN 2    /* x outside [0, E_D)                              */
#define ORA_ESIZE 3      /* E_D(src) != E_D(dst)                            */
#define ORA_EBOUNDS 4    /* coordinate outside the storage box / rank range */
#define ORA_ECOLLIDE 5   /* two different x write the same cell             */
#define ORA_ECAPACITY 6  /* caller's output array too small                 */
#define ORA_ENOMEM 7

#define ORA_MAX_AXES 32

typedef struct { int64_t extent; int64_t stride; const char *axis; } ora_iter;
typedef struct { const char *axis; int64_t value; } ora_coord;
typedef struct { const char *axis; int64_t extent; int64_t divisor; } ora_sdigit;
typedef struct {
  int n;
  const ora_sdigit *digits; /* outer -> inner */
  int swz_b, swz_m, swz_s;  /* CUTLASS-style Swizzle<B,M,S> on byte offsets; B = 0: none */
} ora_storage;
typedef struct {
  int nD;
  const ora_iter *D;
  int nR;
  const ora_iter *R;
  int nO;
  const ora_coord *O;
} ora_layout;

/* A sparse coordinate in ZA: a small list of (axis, value). */
typedef struct {
  int n;
  const char *axis[ORA_MAX_AXES];
  int64_t value[ORA_MAX_AXES];
} coord_t;

static int coord_add(coord_t *c, const char *axis, int64_t v) {
  for (int i = 0; i < c->n; i++)
    if (strcmp(c->axis[i], axis) == 0) { c->value[i] += v; return ORA_OK; }
  if (c->n == ORA_MAX_AXES) return ORA_EINVAL;
  c->axis[c->n] = axis;
  c->value[c->n] = v;
  c->n++;
  return ORA_OK;
}

static int64_t coord_get(const coord_t *c, const char *axis) {
  for (int i = 0; i < c->n; i++)
    if (strcmp(c->axis[i], axis) == 0) return c->value[i];
  return 0; /* an absent axis is 0 */
}

/* ---- layout validation (Def. Iter: e > 0, s != 0; Def. Layout: n_D >= 1) ---- */
static int valid_axis_name(const char *a) {
  if (a == NULL || a[0] == 0) return 0;
  char c = a[0];
  if (!((c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') || c == '_')) return 0;
  for (const char *p = a + 1; *p; p++) {
    c = *p;
    if (!((c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') || (c >= '0' && c <= '9') || c == '_'))
      return 0;
  }
  return 1;
}

static int check_layout(const ora_layout *L, int64_t *E_D, int64_t *E_R) {
  if (L->nD < 1) return ORA_EINVAL;
  int64_t ed = 1, er = 1;
  for (int i = 0; i < L->nD; i++) {
    if (L->D[i].extent < 1 || L->D[i].stride == 0 || !valid_axis_name(L->D[i].axis)) return ORA_EINVAL;
    if (__builtin_mul_overflow(ed, L->D[i].extent, &ed)) return ORA_EINVAL;
  }
  for (int i = 0; i < L->nR; i++) {
    if (L->R[i].extent < 1 || L->R[i].stride == 0 || !valid_axis_name(L->R[i].axis)) return ORA_EINVAL;
    if (__builtin_mul_overflow(er, L->R[i].extent, &er)) return ORA_EINVAL;
  }
  for (int i = 0; i < L->nO; i++)
    if (!valid_axis_name(L->O[i].axis)) return ORA_EINVAL;
  *E_D = ed;
  *E_R = er;
  return ORA_OK;
}

int ora_sizes(const ora_layout *L, int64_t *E_D, int64_t *E_R) { return check_layout(L, E_D, E_R); }

/* f_D(x) + O  ("standard lexicographic unflattening", last iter fastest) */
static int fD_plus_O(const ora_layout *L, int64_t x, coord_t *c) {
  c->n = 0;
  int64_t p = 1;
  for (int i = L->nD - 1; i >= 0; i--) {
    int64_t d = (x / p) % L->D[i].extent;
    if (coord_add(c, L->D[i].axis, d * L->D[i].stride)) return ORA_EINVAL;
    p *= L->D[i].extent;
  }
  for (int i = 0; i < L->nO; i++)
    if (coord_add(c, L->O[i].axis, L->O[i].value)) return ORA_EINVAL;
  return ORA_OK;
}

/* f_R(r) for the r-th replica in lexicographic order (last replica iter fastest) */
static int fR_add(const ora_layout *L, int64_t r, coord_t *c) {
  int64_t p = 1;
  for (int t = L->nR - 1; t >= 0; t--) {
    int64_t d = (r / p) % L->R[t].extent;
    if (coord_add(c, L->R[t].axis, d * L->R[t].stride)) return ORA_EINVAL;
    p *= L->R[t].extent;
  }
  return ORA_OK;
}

/* The r-th element of f_L(x). */
static int fL(const ora_layout *L, int64_t x, int64_t r, coord_t *c) {
  int st = fD_plus_O(L, x, c);
  if (st) return st;
  return fR_add(L, r, c);
}

/* Axes of L in first-appearance order over D, R, O. */
static int layout_axes(const ora_layout *L, const char **axes, int *n) {
  *n = 0;
  for (int k = 0; k < L->nD + L->nR + L->nO; k++) {
    const char *a = k < L->nD ? L->D[k].axis
                  : k < L->nD + L->nR ? L->R[k - L->nD].axis
                  : L->O[k - L->nD - L->nR].axis;
    int found = 0;
    for (int i = 0; i < *n; i++)
      if (strcmp(axes[i], a) == 0) found = 1;
    if (!found) {
      if (*n == ORA_MAX_AXES) return ORA_EINVAL;
      axes[(*n)++] = a;
    }
  }
  return ORA_OK;
}

/*
 * ora_eval: rows_out[r * n_axes + i] = axis i of the r-th coordinate of f_L(x).
 * axes_out receives the axis names (pointers into L).  capacity = rows_out length.
 */
int ora_eval(const ora_layout *L, int64_t x, const char **axes_out, int *n_axes, int64_t *rows_out,
             int64_t capacity) {
  int64_t ED, ER;
  int st = check_layout(L, &ED, &ER);
  if (st) return st;
  if (x < 0 || x >= ED) return ORA_EDOMAIN;
  st = layout_axes(L, axes_out, n_axes);
  if (st) return st;
  if (ER * (int64_t)(*n_axes) > capacity) return ORA_ECAPACITY;
  for (int64_t r = 0; r < ER; r++) {
    coord_t c;
    st = fL(L, x, r, &c);
    if (st) return st;
    for (int i = 0; i < *n_axes; i++) rows_out[r * (*n_axes) + i] = coord_get(&c, axes_out[i]);
  }
  return ORA_OK;
}

/* Brute-force per-axis min / max over every element of every f_L(x) (the plain
 * definition of Vals_{L,a}).  Returns ORA_EBOUNDS if the axis never
 * appears (callers treat it as span 1). */
int ora_bounds(const ora_layout *L, const char *axis, int64_t *mn, int64_t *mx) {
  int64_t ED, ER;
  int st = check_layout(L, &ED, &ER);
  if (st) return st;
  const char *axes[ORA_MAX_AXES];
  int n;
  layout_axes(L, axes, &n);
  int present = 0;
  for (int i = 0; i < n; i++)
    if (strcmp(axes[i], axis) == 0) present = 1;
  if (!present) return ORA_EBOUNDS;
  int first = 1;
  for (int64_t x = 0; x < ED; x++)
    for (int64_t r = 0; r < ER; r++) {
      coord_t c;
      fL(L, x, r, &c);
      int64_t v = coord_get(&c, axis);
      if (first || v < *mn) *mn = v;
      if (first || v > *mx) *mx = v;
      first = 0;
    }
  return ORA_OK;
}

/* ---- storage: coordinate -> element index -> byte offset (readings R16, R17) ---- */

int ora_storage_check(const ora_storage *st) {
  if (st->n < 1) return ORA_EINVAL;
  for (int k = 0; k < st->n; k++) {
    if (!valid_axis_name(st->digits[k].axis) || st->digits[k].extent < 1 || st->digits[k].divisor < 1)
      return ORA_EINVAL;
    /* digits of one axis form a chain: div_k = ext_k' * div_k' for the next (inner) digit k' of the
       same axis; the innermost digit of each axis has div = 1 */
    int next = -1;
    for (int j = k + 1; j < st->n; j++)
      if (strcmp(st->digits[j].axis, st->digits[k].axis) == 0) { next = j; break; }
    if (next < 0) {
      if (st->digits[k].divisor != 1) return ORA_EINVAL;
    } else if (st->digits[k].divisor != st->digits[next].extent * st->digits[next].divisor) {
      return ORA_EINVAL;
    }
  }
  if (st->swz_b < 0 || st->swz_m < 0 || st->swz_s < 0 || st->swz_b + st->swz_m + st->swz_s > 40)
    return ORA_EINVAL;
  if (st->swz_b > 0 && st->swz_s < st->swz_b) return ORA_EINVAL;
  return ORA_OK;
}

int64_t ora_storage_cells(const ora_storage *st) {
  int64_t n = 1;
  for (int k = 0; k < st->n; k++) n *= st->digits[k].extent;
  return n;
}

/* Element index of coordinate c, or -1 when c is outside the bound box or has
 * a nonzero component on an axis the storage does not bind.  `skip` names an
 * axis that is ignored (the device axis in redistribute) or NULL. */
static int64_t storage_index(const ora_storage *st, const coord_t *c, const char *skip) {
  for (int i = 0; i < c->n; i++) {
    if (skip && strcmp(c->axis[i], skip) == 0) continue;
    int bound = 0;
    for (int k = 0; k < st->n; k++)
      if (strcmp(st->digits[k].axis, c->axis[i]) == 0) bound = 1;
    if (!bound && c->value[i] != 0) return -1;
  }
  int64_t idx = 0;
  for (int k = 0; k < st->n; k++) {
    const ora_sdigit *g = &st->digits[k];
    int64_t v = coord_get(c, g->axis);
    /* the outermost digit of an axis bounds the coordinate: 0 <= v < ext * div */
    int outermost = 1;
    for (int j = 0; j < k; j++)
      if (strcmp(st->digits[j].axis, g->axis) == 0) outermost = 0;
    if (outermost && (v < 0 || v >= g->extent * g->divisor)) return -1;
    idx = idx * g->extent + (v / g->divisor) % g->extent;
  }
  return idx;
}

static int64_t swizzle_byte(const ora_storage *st, int64_t b) {
  if (st->swz_b == 0) return b;
  int64_t mask = ((int64_t)1 << st->swz_b) - 1;
  return b ^ (((b >> (st->swz_m + st->swz_s)) & mask) << st->swz_m);
}

/* Public single-coordinate helper for tests: byte offset of the coordinate given
 * as parallel arrays, or -1 if out of bounds. */
int64_t ora_storage_byte(const ora_storage *st, int n, const char **axes, const int64_t *vals, int es) {
  coord_t c;
  c.n = 0;
  for (int i = 0; i < n; i++)
    if (coord_add(&c, axes[i], vals[i])) return -1;
  int64_t idx = storage_index(st, &c, NULL);
  if (idx < 0) return -1;
  return swizzle_byte(st, idx * es);
}

/* ---- copy and redistribute (readings R4, R6, R7) ---- */

typedef struct {
  const ora_layout *src, *dst;
  const ora_storage *sst, *dstst;
  const uint8_t *const *sbufs;
  uint8_t *const *dbufs;
  int64_t sbytes, dbytes, es;
  int nranks;      /* 0: plain copy (no device axis); >0: redistribute */
  int only_rank;   /* redistribute: write only this rank's dst (-1: all) */
  uint64_t *seen;  /* one bit per dst cell, per rank */
  int64_t cells;   /* dst cells per rank */
  int64_t x0, x1;
  int status;
} job_t;

static int test_and_set(uint64_t *bits, int64_t k) {
  uint64_t m = (uint64_t)1 << (k & 63);
  uint64_t old = __atomic_fetch_or(&bits[k >> 6], m, __ATOMIC_RELAXED);
  return (old & m) != 0;
}

static void *run_job(void *arg) {
  job_t *J = (job_t *)arg;
  const char *dev = J->nranks > 0 ? "gpuid" : NULL;
  int64_t ED, ER;
  check_layout(J->dst, &ED, &ER);
  int64_t *done = (int64_t *)malloc(sizeof(int64_t) * (size_t)ER * 2);
  if (!done) { J->status = ORA_ENOMEM; return NULL; }
  uint8_t v[16];
  for (int64_t x = J->x0; x < J->x1; x++) {
    coord_t c;
    /* source: the representative f_D(x) + O of the source layout (r = 0) */
    fD_plus_O(J->src, x, &c);
    int g = 0;
    if (dev) {
      int64_t gv = coord_get(&c, dev);
      if (gv < 0 || gv >= J->nranks) { J->status = ORA_EBOUNDS; break; }
      g = (int)gv;
    }
    int64_t si = storage_index(J->sst, &c, dev);
    if (si < 0) { J->status = ORA_EBOUNDS; break; }
    int64_t sb = swizzle_byte(J->sst, si * J->es);
    if (sb + J->es > J->sbytes) { J->status = ORA_EBOUNDS; break; }
    memcpy(v, J->sbufs[g] + sb, (size_t)J->es);
    /* destination: every element of f_L(x); identical cells of the same x collapse (set semantics) */
    int64_t ndone = 0;
    for (int64_t r = 0; r < ER && J->status == ORA_OK; r++) {
      fL(J->dst, x, r, &c);
      int gd = 0;
      if (dev) {
        int64_t gv = coord_get(&c, dev);
        if (gv < 0 || gv >= J->nranks) { J->status = ORA_EBOUNDS; break; }
        gd = (int)gv;
      }
      int64_t di = storage_index(J->dstst, &c, dev);
      if (di < 0) { J->status = ORA_EBOUNDS; break; }
      int64_t db = swizzle_byte(J->dstst, di * J->es);
      if (db + J->es > J->dbytes) { J->status = ORA_EBOUNDS; break; }
      int dup = 0;
      for (int64_t k = 0; k < ndone; k++)
        if (done[2 * k] == gd && done[2 * k + 1] == di) dup = 1;
      if (dup) continue;
      done[2 * ndone] = gd;
      done[2 * ndone + 1] = di;
      ndone++;
      if (test_and_set(J->seen, (int64_t)gd * J->cells + di)) { J->status = ORA_ECOLLIDE; break; }
      if (J->only_rank < 0 || J->only_rank == gd) memcpy(J->dbufs[gd] + db, v, (size_t)J->es);
    }
    if (J->status) break;
  }
  free(done);
  return NULL;
}

static int run_all(job_t *base, int64_t ED, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if ((int64_t)nthreads > ED) nthreads = (int)(ED > 0 ? ED : 1);
  job_t *jobs = (job_t *)calloc((size_t)nthreads, sizeof(job_t));
  pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  if (!jobs || !th) { free(jobs); free(th); return ORA_ENOMEM; }
  for (int t = 0; t < nthreads; t++) {
    jobs[t] = *base;
    jobs[t].x0 = ED * t / nthreads;
    jobs[t].x1 = ED * (t + 1) / nthreads;
    jobs[t].status = ORA_OK;
  }
  for (int t = 1; t < nthreads; t++) pthread_create(&th[t], NULL, run_job, &jobs[t]);
  run_job(&jobs[0]);
  for (int t = 1; t < nthreads; t++) pthread_join(th[t], NULL);
  int st = ORA_OK;
  for (int t = 0; t < nthreads; t++)
    if (jobs[t].status && !st) st = jobs[t].status;
  free(jobs);
  free(th);
  return st;
}

static int common_checks(const ora_layout *src, const ora_storage *sst, const ora_layout *dst,
                         const ora_storage *dstst, int es, int64_t *ED) {
  int64_t eds, ers, edd, erd;
  int st;
  if ((st = check_layout(src, &eds, &ers))) return st;
  if ((st = check_layout(dst, &edd, &erd))) return st;
  if ((st = ora_storage_check(sst))) return st;
  if ((st = ora_storage_check(dstst))) return st;
  if (es != 1 && es != 2 && es != 4 && es != 8 && es != 16) return ORA_EINVAL;
  if (eds != edd) return ORA_ESIZE;
  *ED = eds;
  return ORA_OK;
}

/*
 * ora_copy: for every x in [0, E_D): read src at f_D^src(x) + O^src, write the
 * raw es bytes to every cell of f_L^dst(x).  Cells not hit are left untouched
 * (P:124).  The caller pre-fills dst.  On error dst may be partially written.
 */
int ora_copy(const ora_layout *src, const ora_storage *sst, const uint8_t *sbuf, int64_t sbytes,
             const ora_layout *dst, const ora_storage *dstst, uint8_t *dbuf, int64_t dbytes, int es,
             int nthreads) {
  int64_t ED;
  int st = common_checks(src, sst, dst, dstst, es, &ED);
  if (st) return st;
  int64_t cells = ora_storage_cells(dstst);
  uint64_t *seen = (uint64_t *)calloc((size_t)(cells / 64 + 1), sizeof(uint64_t));
  if (!seen) return ORA_ENOMEM;
  const uint8_t *sb[1] = {sbuf};
  uint8_t *db[1] = {dbuf};
  job_t J;
  memset(&J, 0, sizeof(J));
  J.src = src; J.dst = dst; J.sst = sst; J.dstst = dstst;
  J.sbufs = sb; J.dbufs = db;
  J.sbytes = sbytes; J.dbytes = dbytes; J.es = es;
  J.nranks = 0; J.only_rank = -1; J.seen = seen; J.cells = cells;
  st = run_all(&J, ED, nthreads);
  free(seen);
  return st;
}

/*
 * ora_redistribute: as ora_copy, with the `gpuid` coordinate of each side
 * selecting sbufs[g] / dbufs[g'] (removed before the storage index).  With
 * only_rank >= 0 only that rank's destination buffer is written (dbufs[g] for
 * other g may be NULL), but collisions are still checked over all ranks.
 */
int ora_redistribute(const ora_layout *src, const ora_storage *sst, const uint8_t *const *sbufs,
                     int64_t sbytes, const ora_layout *dst, const ora_storage *dstst, uint8_t *const *dbufs,
                     int64_t dbytes, int es, int nranks, int only_rank, int nthreads) {
  int64_t ED;
  int st = common_checks(src, sst, dst, dstst, es, &ED);
  if (st) return st;
  if (nranks < 1) return ORA_EINVAL;
  int64_t cells = ora_storage_cells(dstst);
  uint64_t *seen = (uint64_t *)calloc((size_t)((cells * nranks) / 64 + 1), sizeof(uint64_t));
  if (!seen) return ORA_ENOMEM;
  job_t J;
  memset(&J, 0, sizeof(J));
  J.src = src; J.dst = dst; J.sst = sst; J.dstst = dstst;
  J.sbufs = sbufs; J.dbufs = dbufs;
  J.sbytes = sbytes; J.dbytes = dbytes; J.es = es;
  J.nranks = nranks; J.only_rank = only_rank; J.seen = seen; J.cells = cells;
  st = run_all(&J, ED, nthreads);
  free(seen);
  return st;
}

/* ---- reduction: SURVEY §8(f) f3 ----------------------------------------------
 * P:399-403 (the DTensor reduce-scatter signature: an input of shape (4,64,64)
 * "sums over 0", producing a (64,64) output) and P:628 ("invokes the sum
 * operator").  Reading R24 of DESIGN.md: the leading logical dimension of the
 * source is summed away,
 *
 *   K = E_D(src) / E_D(dst),   dst(y) = sum_{k=0}^{K-1} src(k * E_D(dst) + y),
 *
 * the source element read for x being the representative f_D(x) + O (R4) and
 * the sum written to every cell of f_L^dst(y).  Floating point summands are
 * added in fp64 in k order and the sum is rounded ONCE to the element type
 * (round to nearest, ties to even); integers add modulo 2^bits.
 * --------------------------------------------------------------------------- */
#include <math.h>

#define ORA_DT_F32 1
#define ORA_DT_F64 2
#define ORA_DT_F16 3
#define ORA_DT_BF16 4
#define ORA_DT_I32 5
#define ORA_DT_I64 6

static int dt_size(int dt) {
  switch (dt) {
    case ORA_DT_F32: case ORA_DT_I32: return 4;
    case ORA_DT_F64: case ORA_DT_I64: return 8;
    case ORA_DT_F16: case ORA_DT_BF16: return 2;
  }
  return 0;
}

/* IEEE-754 binary16: 1 sign, 5 exponent (bias 15), 10 fraction bits */
static double f16_value(uint16_t h) {
  int s = h >> 15, e = (h >> 10) & 31, f = h & 1023;
  double v;
  if (e == 0) v = ldexp((double)f, -24);
  else if (e == 31) v = f ? NAN : INFINITY;
  else v = ldexp((double)(1024 + f), e - 25);
  return s ? -v : v;
}

/* bfloat16: the upper half of an IEEE-754 binary32 */
static double bf16_value(uint16_t h) {
  uint32_t w = (uint32_t)h << 16;
  float f;
  memcpy(&f, &w, 4);
  return (double)f;
}

/* v rounded to p significant bits (ties to even), exponents below emin kept at
 * emin (gradual underflow); magnitudes above max_finite become infinite. */
static double round_sig(double v, int p, int emin, double max_finite) {
  if (v == 0 || isnan(v) || isinf(v)) return v;
  int e;
  frexp(v, &e); /* |v| = m 2^e, 1/2 <= m < 1: leading bit weight 2^(e-1) */
  int lead = e - 1 < emin ? emin : e - 1;
  int q = lead - (p - 1); /* weight of the last kept bit */
  double r = ldexp(nearbyint(ldexp(v, -q)), q);
  if (fabs(r) > max_finite) r = r > 0 ? INFINITY : -INFINITY;
  return r;
}

static void put_f16(uint8_t *p, double v) {
  uint16_t h;
  double r = round_sig(v, 11, -14, 65504.0);
  if (isnan(r)) h = 0x7e00;
  else {
    uint16_t s = signbit(r) ? 0x8000 : 0;
    double a = fabs(r);
    if (isinf(a)) h = s | 0x7c00;
    else if (a < ldexp(1.0, -14)) h = s | (uint16_t)ldexp(a, 24); /* subnormal: a = f 2^-24 */
    else {
      int e;
      double m = frexp(a, &e); /* a = (2m) 2^(e-1), 1 <= 2m < 2 */
      h = s | (uint16_t)((e - 1 + 15) << 10) | (uint16_t)ldexp(2 * m - 1, 10);
    }
  }
  memcpy(p, &h, 2);
}

static void put_bf16(uint8_t *p, double v) {
  uint16_t h;
  double r = round_sig(v, 8, -126, ldexp(255.0, 120)); /* max (2 - 2^-7) 2^127 */
  if (isnan(r)) h = 0x7fc0;
  else {
    float f = (float)r; /* exact: r has <= 8 significant bits */
    uint32_t w;
    memcpy(&w, &f, 4);
    h = (uint16_t)(w >> 16);
  }
  memcpy(p, &h, 2);
}

typedef struct {
  const ora_layout *src, *dst;
  const ora_storage *sst, *dstst;
  const uint8_t *const *sbufs;
  uint8_t *const *dbufs;
  int64_t sbytes, dbytes, K, Y;
  int dt, nranks, only_rank;
  uint64_t *seen;
  int64_t cells;
  int64_t y0, y1;
  int status;
} rjob_t;

static void *run_reduce_job(void *arg) {
  rjob_t *J = (rjob_t *)arg;
  const char *dev = J->nranks > 0 ? "gpuid" : NULL;
  const int es = dt_size(J->dt);
  int64_t ED, ER;
  check_layout(J->dst, &ED, &ER);
  int64_t *done = (int64_t *)malloc(sizeof(int64_t) * (size_t)ER * 2);
  if (!done) { J->status = ORA_ENOMEM; return NULL; }
  for (int64_t y = J->y0; y < J->y1 && J->status == ORA_OK; y++) {
    double fsum = 0;
    uint64_t isum = 0;
    for (int64_t k = 0; k < J->K; k++) {
      coord_t c;
      fD_plus_O(J->src, k * J->Y + y, &c); /* source representative (R4) */
      int g = 0;
      if (dev) {
        int64_t gv = coord_get(&c, dev);
        if (gv < 0 || gv >= J->nranks) { J->status = ORA_EBOUNDS; break; }
        g = (int)gv;
      }
      int64_t si = storage_index(J->sst, &c, dev);
      if (si < 0) { J->status = ORA_EBOUNDS; break; }
      int64_t sb = swizzle_byte(J->sst, si * es);
      if (sb + es > J->sbytes) { J->status = ORA_EBOUNDS; break; }
      const uint8_t *p = J->sbufs[g] + sb;
      switch (J->dt) {
        case ORA_DT_F32: { float f; memcpy(&f, p, 4); fsum += (double)f; break; }
        case ORA_DT_F64: { double f; memcpy(&f, p, 8); fsum += f; break; }
        case ORA_DT_F16: { uint16_t h; memcpy(&h, p, 2); fsum += f16_value(h); break; }
        case ORA_DT_BF16: { uint16_t h; memcpy(&h, p, 2); fsum += bf16_value(h); break; }
        case ORA_DT_I32: { uint32_t w; memcpy(&w, p, 4); isum += w; break; }
        case ORA_DT_I64: { uint64_t w; memcpy(&w, p, 8); isum += w; break; }
      }
    }
    if (J->status) break;
    uint8_t v[8];
    switch (J->dt) {
      case ORA_DT_F32: { float f = (float)fsum; memcpy(v, &f, 4); break; } /* C cast: nearest even */
      case ORA_DT_F64: memcpy(v, &fsum, 8); break;
      case ORA_DT_F16: put_f16(v, fsum); break;
      case ORA_DT_BF16: put_bf16(v, fsum); break;
      case ORA_DT_I32: { uint32_t w = (uint32_t)isum; memcpy(v, &w, 4); break; }
      case ORA_DT_I64: memcpy(v, &isum, 8); break;
    }
    int64_t ndone = 0;
    for (int64_t r = 0; r < ER; r++) {
      coord_t c;
      fL(J->dst, y, r, &c);
      int gd = 0;
      if (dev) {
        int64_t gv = coord_get(&c, dev);
        if (gv < 0 || gv >= J->nranks) { J->status = ORA_EBOUNDS; break; }
        gd = (int)gv;
      }
      int64_t di = storage_index(J->dstst, &c, dev);
      if (di < 0) { J->status = ORA_EBOUNDS; break; }
      int64_t db = swizzle_byte(J->dstst, di * es);
      if (db + es > J->dbytes) { J->status = ORA_EBOUNDS; break; }
      int dup = 0;
      for (int64_t q = 0; q < ndone; q++)
        if (done[2 * q] == gd && done[2 * q + 1] == di) dup = 1;
      if (dup) continue;
      done[2 * ndone] = gd;
      done[2 * ndone + 1] = di;
      ndone++;
      if (test_and_set(J->seen, (int64_t)gd * J->cells + di)) { J->status = ORA_ECOLLIDE; break; }
      if (J->only_rank < 0 || J->only_rank == gd) memcpy(J->dbufs[gd] + db, v, (size_t)es);
    }
  }
  free(done);
  return NULL;
}

/*
 * ora_reduce: dst(y) = sum_k src(k * E_D(dst) + y) (reading R24).  nranks = 0: one
 * buffer per side (no device axis); nranks > 0: the `gpuid` coordinate selects
 * sbufs[g] / dbufs[g'] as in ora_redistribute (only_rank as there).
 */
int ora_reduce(const ora_layout *src, const ora_storage *sst, const uint8_t *const *sbufs, int64_t sbytes,
               const ora_layout *dst, const ora_storage *dstst, uint8_t *const *dbufs, int64_t dbytes, int dt,
               int nranks, int only_rank, int nthreads) {
  int64_t eds, ers, edd, erd;
  int st;
  if ((st = check_layout(src, &eds, &ers))) return st;
  if ((st = check_layout(dst, &edd, &erd))) return st;
  if ((st = ora_storage_check(sst))) return st;
  if ((st = ora_storage_check(dstst))) return st;
  if (!dt_size(dt) || nranks < 0) return ORA_EINVAL;
  if (eds % edd) return ORA_ESIZE;
  int64_t cells = ora_storage_cells(dstst);
  int nr = nranks > 0 ? nranks : 1;
  uint64_t *seen = (uint64_t *)calloc((size_t)((cells * nr) / 64 + 1), sizeof(uint64_t));
  if (!seen) return ORA_ENOMEM;
  if (nthreads < 1) nthreads = 1;
  if ((int64_t)nthreads > edd) nthreads = (int)edd;
  rjob_t *jobs = (rjob_t *)calloc((size_t)nthreads, sizeof(rjob_t));
  pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  if (!jobs || !th) { free(jobs); free(th); free(seen); return ORA_ENOMEM; }
  for (int t = 0; t < nthreads; t++) {
    rjob_t *J = &jobs[t];
    J->src = src; J->dst = dst; J->sst = sst; J->dstst = dstst;
    J->sbufs = sbufs; J->dbufs = dbufs; J->sbytes = sbytes; J->dbytes = dbytes;
    J->K = eds / edd; J->Y = edd; J->dt = dt; J->nranks = nranks; J->only_rank = only_rank;
    J->seen = seen; J->cells = cells;
    J->y0 = edd * t / nthreads;
    J->y1 = edd * (t + 1) / nthreads;
  }
  for (int t = 1; t < nthreads; t++) pthread_create(&th[t], NULL, run_reduce_job, &jobs[t]);
  run_reduce_job(&jobs[0]);
  for (int t = 1; t < nthreads; t++) pthread_join(th[t], NULL);
  st = ORA_OK;
  for (int t = 0; t < nthreads; t++)
    if (jobs[t].status && !st) st = jobs[t].status;
  free(jobs);
  free(th);
  free(seen);
  return st;
}
