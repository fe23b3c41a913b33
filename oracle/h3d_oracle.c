/* TEST INFRASTRUCTURE ONLY — CPU oracle for the HODLR3D hot path.
 *
 * Plain-C restatement of the reference algorithm. Every function cites the
 * reference file:line it follows (paths relative to /root/reference/proj).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker; the product never does.
 *
 * Floating-point order mirrors the reference compiled against oracle/shim
 * (ascending sums, no FMA contraction: both are built with -ffp-contract=off),
 * so pivots, LU factors and matvec output are bit-identical to oracle/_ref.
 * Pinned by tests/test_oracle_pin.py against tests/golden/ (generated from
 * oracle/_ref by tests/golden/make_golden.py).
 */
#include "h3d_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_MAX_LEVELS 21

static __thread char g_err[256];

static void set_err(const char* msg) {
  strncpy(g_err, msg, sizeof(g_err) - 1);
  g_err[sizeof(g_err) - 1] = 0;
}

const char* orc_last_error(void) { return g_err; }

void orc_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* ------------------------------------------------------------------------ */
/* mt19937_64 (the C++ <random> engine the reference seeds; kernel.hpp:24-26) */
typedef struct {
  uint64_t mt[312];
  int mti;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->mti = 312;
}

static uint64_t mt64_next(mt64* s) {
  static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (s->mti >= 312) {
    int i;
    uint64_t x;
    for (i = 0; i < 312 - 156; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    for (; i < 311; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + (156 - 312)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    x = (s->mt[311] & UM) | (s->mt[0] & LM);
    s->mt[311] = s->mt[155] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    s->mti = 0;
  }
  uint64_t x = s->mt[s->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* kernel.hpp:24-26 */
static double uniform01(mt64* s) { return (double)(mt64_next(s) >> 11) * 0x1.0p-53; }

/* kernel.cpp:88-95 */
int orc_generate_points(int64_t n, uint64_t seed, double* xyz) {
  if (n < 1) {
    set_err("generate_points: N must be >= 1");
    return ORC_EINVAL;
  }
  mt64 g;
  mt64_seed(&g, seed);
  for (int64_t i = 0; i < n; ++i) {
    const double x = 2.0 * uniform01(&g) - 1.0;
    const double y = 2.0 * uniform01(&g) - 1.0;
    const double z = 2.0 * uniform01(&g) - 1.0;
    xyz[3 * i] = x;
    xyz[3 * i + 1] = y;
    xyz[3 * i + 2] = z;
  }
  return ORC_OK;
}

void orc_random_vector(int64_t n, uint64_t seed, double* out) {
  mt64 g;
  mt64_seed(&g, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = 2.0 * uniform01(&g) - 1.0;
}

/* ------------------------------------------------------------------------ */
/* Radial maps on r^2 (lowrank.cpp:51-62: LaplaceF, QuarticF, HelmholtzF). */
static inline double kernel_r2(int kid, double r2) {
  switch (kid) {
    case ORC_LAPLACE: return 1.0 / sqrt(r2);
    case ORC_R4: return 1.0 / (r2 * r2);
    default: {
      const double r = sqrt(r2);
      return cos(r) / r;
    }
  }
}

/* Kernel entries on r (kernel.cpp:7-21) via eval_pair (kernel.cpp:59-71). */
static inline int eval_pair(int kid, const double* a, const double* b, double* v) {
  const double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
  const double r = sqrt(dx * dx + dy * dy + dz * dz);
  if (r < 1e-14) return ORC_EDEGEN_GEOM;
  double out;
  switch (kid) {
    case ORC_LAPLACE: out = 1.0 / r; break;
    case ORC_R4: {
      const double r2 = r * r;
      out = 1.0 / (r2 * r2);
      break;
    }
    default: out = cos(r) / r;
  }
  if (!isfinite(out)) return ORC_EDEGEN_GEOM;
  *v = out;
  return ORC_OK;
}

/* A kernel block in local coordinates: rows X, cols Y, SoA coordinates
 * (lowrank.cpp:87-121 KernelBlock). diag_offset = x.begin - y.begin. */
typedef struct {
  int kid;
  double diag;
  const double *rx, *ry, *rz;
  const double *cx, *cy, *cz;
  int64_t m, n;
  int64_t diag_offset; /* INT64_MIN: none */
} kblock;

#define NO_DIAG INT64_MIN

/* fill_values (lowrank.cpp:17-41): r^2, coincidence scan, radial map,
 * diagonal patch at local index `diag`. Returns nonzero on coincidence. */
static int fill_values(const kblock* b, double px, double py, double pz, const double* qx,
                       const double* qy, const double* qz, int64_t n, double* out,
                       int64_t diag) {
  const double tol2 = 1e-14 * 1e-14;
  for (int64_t j = 0; j < n; ++j) {
    const double dx = px - qx[j];
    const double dy = py - qy[j];
    const double dz = pz - qz[j];
    double r2 = dx * dx + dy * dy + dz * dz;
    if (j == diag) r2 = 1.0; /* patched below */
    if (r2 < tol2) return ORC_EDEGEN_GEOM;
    out[j] = kernel_r2(b->kid, r2);
  }
  if (diag >= 0 && diag < n) out[diag] = b->diag;
  return ORC_OK;
}

/* KernelBlock::row / ::col (lowrank.cpp:128-139) */
static int kb_row(const kblock* b, int64_t i, double* out) {
  const int64_t diag = b->diag_offset == NO_DIAG ? -1 : i + b->diag_offset;
  return fill_values(b, b->rx[i], b->ry[i], b->rz[i], b->cx, b->cy, b->cz, b->n, out, diag);
}
static int kb_col(const kblock* b, int64_t j, double* out) {
  const int64_t diag = b->diag_offset == NO_DIAG ? -1 : j - b->diag_offset;
  return fill_values(b, b->cx[j], b->cy[j], b->cz[j], b->rx, b->ry, b->rz, b->m, out, diag);
}

/* ------------------------------------------------------------------------ */
/* Partially pivoted ACA (lowrank.cpp:157-289). Returns status; on success
 * *rank_out, *rpiv/*cpiv (malloc'd, rank entries) and *lu (rank x rank,
 * row-major, strict lower = L, upper incl. diagonal = R). */
static int aca_compress(const kblock* blk, double eps, int64_t max_rank, int* rank_out,
                        int32_t** rpiv_out, int32_t** cpiv_out, double** lu_out) {
  const int64_t m = blk->m, n = blk->n;
  if (m <= 0 || n <= 0) {
    set_err("aca_compress: empty block");
    return ORC_EINVAL;
  }
  if (!(eps > 0)) {
    set_err("aca_compress: eps <= 0");
    return ORC_EINVAL;
  }
  const int64_t mn = m < n ? m : n;
  const int64_t cap = max_rank > 0 ? (max_rank < mn ? max_rank : mn) : mn;
  int64_t alloc = cap < 16 ? cap : 16;
  double* us = (double*)malloc(sizeof(double) * (size_t)(m * alloc)); /* col-major m x alloc */
  double* vs = (double*)malloc(sizeof(double) * (size_t)(n * alloc));
  double* deltas = (double*)malloc(sizeof(double) * (size_t)(cap > 0 ? cap : 1));
  int32_t* rp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cap > 0 ? cap : 1));
  int32_t* cp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cap > 0 ? cap : 1));
  char* row_used = (char*)calloc((size_t)m, 1);
  char* col_used = (char*)calloc((size_t)n, 1);
  double* rowbuf = (double*)malloc(sizeof(double) * (size_t)n);
  double* colbuf = (double*)malloc(sizeof(double) * (size_t)m);
  double* vbuf = (double*)malloc(sizeof(double) * (size_t)n);
  double* cu = (double*)malloc(sizeof(double) * (size_t)(cap > 0 ? cap : 1));
  double fro2 = 0.0;
  int status = ORC_OK;

  int64_t suggested = 0, rank = 0;
  int hits = 0;
  while (rank < cap) {
    int64_t pi = -1, pj = -1;
    for (;;) {
      int64_t i = -1;
      if (suggested >= 0 && suggested < m && !row_used[suggested]) {
        i = suggested;
      } else {
        for (int64_t t = 0; t < m; ++t)
          if (!row_used[t]) {
            i = t;
            break;
          }
      }
      if (i < 0) break;
      if ((status = kb_row(blk, i, rowbuf)) != ORC_OK) goto done;
      if (rank > 0) {
        /* rowbuf -= vs(:, :rank) * us(i, :rank)^T  (lowrank.cpp:192-194) */
        for (int64_t j = 0; j < n; ++j) {
          double acc = 0.0;
          for (int64_t a = 0; a < rank; ++a) acc += vs[a * n + j] * us[a * m + i];
          rowbuf[j] -= acc;
        }
      }
      double best = -1.0;
      int64_t bestj = -1;
      for (int64_t j = 0; j < n; ++j) {
        if (col_used[j]) continue;
        const double a = fabs(rowbuf[j]);
        if (a > best) {
          best = a;
          bestj = j;
        }
      }
      if (bestj < 0) break;
      if (best < 1e-30) { /* AcaOptions::pivot_floor (lowrank.hpp:99) */
        row_used[i] = 1;
        suggested = -1;
        continue;
      }
      pi = i;
      pj = bestj;
      break;
    }
    if (pi < 0) break;

    const double delta = rowbuf[pj];
    if ((status = kb_col(blk, pj, colbuf)) != ORC_OK) goto done;
    if (rank > 0) {
      /* colbuf -= us(:, :rank) * vs(pj, :rank)^T  (lowrank.cpp:220-222) */
      for (int64_t i = 0; i < m; ++i) {
        double acc = 0.0;
        for (int64_t a = 0; a < rank; ++a) acc += us[a * m + i] * vs[a * n + pj];
        colbuf[i] -= acc;
      }
    }
    for (int64_t j = 0; j < n; ++j) vbuf[j] = rowbuf[j] / delta;

    double u2 = 0.0, v2 = 0.0;
    for (int64_t i = 0; i < m; ++i) u2 += colbuf[i] * colbuf[i];
    for (int64_t j = 0; j < n; ++j) v2 += vbuf[j] * vbuf[j];
    const double uv = sqrt(u2 * v2);
    /* two-hit stop rule (lowrank.cpp:225-239) */
    if (rank > 0) {
      const double ns = sqrt(fro2 > 0.0 ? fro2 : 0.0);
      if (uv <= 1e-12 * ns) break;
      if (uv <= eps * ns) {
        if (++hits >= 2) break;
      } else {
        hits = 0;
      }
    }
    if (rank == alloc) { /* conservativeResize (lowrank.cpp:241-244) */
      const int64_t na = cap < 2 * rank ? cap : 2 * rank;
      us = (double*)realloc(us, sizeof(double) * (size_t)(m * na));
      vs = (double*)realloc(vs, sizeof(double) * (size_t)(n * na));
      alloc = na;
    }
    double cross = 0.0;
    if (rank > 0) { /* lowrank.cpp:245-249 */
      for (int64_t a = 0; a < rank; ++a) {
        double acc = 0.0;
        for (int64_t i = 0; i < m; ++i) acc += us[a * m + i] * colbuf[i];
        cu[a] = acc;
      }
      for (int64_t a = 0; a < rank; ++a) {
        double acc = 0.0;
        for (int64_t j = 0; j < n; ++j) acc += vs[a * n + j] * vbuf[j];
        cross += cu[a] * acc;
      }
    }
    fro2 += u2 * v2 + 2.0 * cross;
    memcpy(us + rank * m, colbuf, sizeof(double) * (size_t)m);
    memcpy(vs + rank * n, vbuf, sizeof(double) * (size_t)n);
    deltas[rank] = delta;
    rp[rank] = (int32_t)pi;
    cp[rank] = (int32_t)pj;
    row_used[pi] = 1;
    col_used[pj] = 1;
    ++rank;

    /* next row pivot: largest entry of the new residual column (:260-270) */
    double best = -1.0;
    suggested = -1;
    for (int64_t i = 0; i < m; ++i) {
      if (row_used[i]) continue;
      const double a = fabs(colbuf[i]);
      if (a > best) {
        best = a;
        suggested = i;
      }
    }
  }

  {
    /* packed LU from the elimination history (lowrank.cpp:277-287) */
    const int r = (int)rank;
    double* lu = (double*)malloc(sizeof(double) * (size_t)(r > 0 ? r * r : 1));
    for (int a = 0; a < r; ++a) {
      for (int b = a + 1; b < r; ++b) lu[b * r + a] = us[a * m + rp[b]] / deltas[a];
      for (int b = a; b < r; ++b) lu[a * r + b] = deltas[a] * vs[a * n + cp[b]];
    }
    *rank_out = r;
    *rpiv_out = rp;
    *cpiv_out = cp;
    *lu_out = lu;
    rp = cp = NULL;
  }

done:
  free(us);
  free(vs);
  free(deltas);
  free(rp);
  free(cp);
  free(row_used);
  free(col_used);
  free(rowbuf);
  free(colbuf);
  free(vbuf);
  free(cu);
  if (status == ORC_EDEGEN_GEOM) set_err("coincident distinct points in block");
  return status;
}

/* lr_apply (lowrank.cpp:291-327): b += K(X,tau) R^-1 L^-1 K(sigma,Y) x */
static int lr_apply(const kblock* blk, int r, const int32_t* rp, const int32_t* cp,
                    const double* lu, const double* x, double* b, double* rowbuf,
                    double* colbuf, double* t) {
  if (r == 0) return ORC_OK;
  const int64_t m = blk->m, n = blk->n;
  int st;
  for (int k = 0; k < r; ++k) {
    if ((st = kb_row(blk, rp[k], rowbuf)) != ORC_OK) return st;
    double acc = 0.0;
    for (int64_t j = 0; j < n; ++j) acc += rowbuf[j] * x[j];
    t[k] = acc;
  }
  for (int k = 0; k < r; ++k) {
    double acc = t[k];
    for (int a = 0; a < k; ++a) acc -= lu[k * r + a] * t[a];
    t[k] = acc;
  }
  for (int k = r - 1; k >= 0; --k) {
    double acc = t[k];
    for (int a = k + 1; a < r; ++a) acc -= lu[k * r + a] * t[a];
    t[k] = acc / lu[k * r + k];
  }
  for (int k = 0; k < r; ++k) {
    if ((st = kb_col(blk, cp[k], colbuf)) != ORC_OK) return st;
    const double tk = t[k];
    for (int64_t i = 0; i < m; ++i) b[i] += tk * colbuf[i];
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Octree (octree.cpp:30-171) and HODLR3D lists (octree.cpp:197-260). */

static int64_t morton_encode(int ix, int iy, int iz, int level) { /* octree.cpp:30-38 */
  int64_t code = 0;
  for (int b = 0; b < level; ++b) {
    code |= ((int64_t)((ix >> b) & 1) << (3 * b));
    code |= ((int64_t)((iy >> b) & 1) << (3 * b + 1));
    code |= ((int64_t)((iz >> b) & 1) << (3 * b + 2));
  }
  return code;
}

static void morton_decode(int64_t code, int level, int* ix, int* iy, int* iz) {
  *ix = *iy = *iz = 0;
  for (int b = 0; b < level; ++b) {
    *ix |= (int)((code >> (3 * b)) & 1) << b;
    *iy |= (int)((code >> (3 * b + 1)) & 1) << b;
    *iz |= (int)((code >> (3 * b + 2)) & 1) << b;
  }
}

/* grid_coord (octree.cpp:67-72) */
static int grid_coord(double x, double lo, double inv_w, int64_t cells) {
  int64_t k = (int64_t)((x - lo) * inv_w * (double)cells);
  if (k < 0) k = 0;
  if (k >= cells) k = cells - 1;
  return (int)k;
}

typedef struct {
  int64_t code;
  int32_t idx;
} coded_t;

static int cmp_coded(const void* a, const void* b) {
  const coded_t* x = (const coded_t*)a;
  const coded_t* y = (const coded_t*)b;
  if (x->code != y->code) return x->code < y->code ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

/* classify_offset (octree.hpp:27-37): 0 self, 1 face, 2 edge, 3 vertex, 4 ws */
static int classify_offset(int dx, int dy, int dz) {
  const int ax = dx < 0 ? -dx : dx, ay = dy < 0 ? -dy : dy, az = dz < 0 ? -dz : dz;
  if ((ax | ay | az) == 0) return 0;
  if (ax >= 2 || ay >= 2 || az >= 2) return 4;
  const int nz = (ax != 0) + (ay != 0) + (az != 0);
  return nz == 1 ? 1 : nz == 2 ? 2 : 3;
}

static int cmp_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return x < y ? -1 : (x > y);
}

typedef struct {
  int64_t count;
  int32_t* target;
  int32_t* source;
  int32_t* rank;
  int64_t* piv_off; /* into rep->piv_* */
  int64_t* lu_off;  /* into rep->lu */
} lr_level;

struct orc_rep {
  int64_t n;
  int depth;
  int kid;
  double diag;
  double eps;
  int64_t max_rank;
  int32_t* perm;
  double *px, *py, *pz;              /* permuted SoA coordinates */
  int64_t* off[ORC_MAX_LEVELS];      /* 8^l + 1 node offsets */
  int variant;                       /* 0 hodlr3d, 1 hodlr, 2 hstrong (octree.hpp:80) */
  int32_t* lst_off[ORC_MAX_LEVELS][4];  /* kinds: inter, near_edge, near_face, near_vertex */
  int32_t* lst_ids[ORC_MAX_LEVELS][4];
  lr_level lr[ORC_MAX_LEVELS];
  int32_t *piv_row, *piv_col;
  double* lu;
  int64_t ndense;
  int32_t *d_target, *d_source;
};

static int64_t nodes_at(int l) { return (int64_t)1 << (3 * l); }

/* build_tree (octree.cpp:76-171) into rep. */
static int build_tree(orc_rep* rep, const double* xyz, int64_t n, int n_max, int depth_cap) {
  if (n_max < 1) {
    set_err("build_tree: n_max must be >= 1");
    return ORC_EINVAL;
  }
  if (n == 0) {
    set_err("build_tree: empty point set");
    return ORC_EINVAL;
  }
  if (depth_cap < 0 || depth_cap > 20) {
    set_err("build_tree: unreasonable depth cap");
    return ORC_EINVAL;
  }
  const double lo = -1.0, inv_w = 1.0 / 2.0;
  const int64_t cells = (int64_t)1 << depth_cap;
  for (int64_t i = 0; i < n; ++i) {
    const double* p = xyz + 3 * i;
    if (p[0] < lo || p[0] > lo + 2.0 || p[1] < lo || p[1] > lo + 2.0 || p[2] < lo ||
        p[2] > lo + 2.0) {
      set_err("build_tree: point outside the domain cube");
      return ORC_EINVAL;
    }
  }
  coded_t* coded = (coded_t*)malloc(sizeof(coded_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    const double* p = xyz + 3 * i;
    coded[i].code = morton_encode(grid_coord(p[0], lo, inv_w, cells),
                                  grid_coord(p[1], lo, inv_w, cells),
                                  grid_coord(p[2], lo, inv_w, cells), depth_cap);
    coded[i].idx = (int32_t)i;
  }
  qsort(coded, (size_t)n, sizeof(coded_t), cmp_coded);

  int depth = -1;
  for (int l = 0; l <= depth_cap && depth < 0; ++l) { /* octree.cpp:110-130 */
    const int shift = 3 * (depth_cap - l);
    int64_t best = 0, run = 0, prev = -1;
    for (int64_t i = 0; i < n; ++i) {
      const int64_t c = coded[i].code >> shift;
      run = (c == prev) ? run + 1 : 1;
      prev = c;
      if (run > best) best = run;
    }
    if (best < n_max) depth = l;
  }
  if (depth < 0) {
    free(coded);
    snprintf(g_err, sizeof(g_err),
             "build_tree: depth cap %d exceeded; distribution too concentrated for n_max = %d",
             depth_cap, n_max);
    return ORC_EDEGEN_DIST;
  }
  rep->depth = depth;
  rep->n = n;
  rep->perm = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  rep->px = (double*)malloc(sizeof(double) * (size_t)n);
  rep->py = (double*)malloc(sizeof(double) * (size_t)n);
  rep->pz = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    const int32_t o = coded[i].idx;
    rep->perm[i] = o;
    rep->px[i] = xyz[3 * o];
    rep->py[i] = xyz[3 * o + 1];
    rep->pz[i] = xyz[3 * o + 2];
  }
  /* leaf ranges by one scan; parents by grouping (octree.cpp:148-169) */
  {
    const int64_t nl = nodes_at(depth);
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nl + 1));
    const int shift = 3 * (depth_cap - depth);
    int64_t p = 0;
    for (int64_t m = 0; m < nl; ++m) {
      off[m] = p;
      while (p < n && (coded[p].code >> shift) == m) ++p;
    }
    off[nl] = p;
    rep->off[depth] = off;
  }
  for (int l = depth - 1; l >= 0; --l) {
    const int64_t nl = nodes_at(l);
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nl + 1));
    for (int64_t m = 0; m <= nl; ++m) off[m] = rep->off[l + 1][8 * m];
    rep->off[l] = off;
  }
  free(coded);
  return ORC_OK;
}

/* build_interaction_lists (octree.cpp:197-260). Candidates: the 7 siblings,
 * plus (hodlr3d / hstrong) the children of the parent's near_edge and
 * near_face (and near_vertex for hstrong), sorted ascending. hodlr: every
 * candidate is inter. hodlr3d: ws + vertex -> inter. hstrong: ws -> inter,
 * vertex -> near_vertex. Edge / face -> near_edge / near_face. */
static void build_lists(orc_rep* rep) {
  const int L = rep->depth;
  const int V = rep->variant;
  for (int k = 0; k < 4; ++k) {
    rep->lst_off[0][k] = (int32_t*)calloc(2, sizeof(int32_t));
    rep->lst_ids[0][k] = (int32_t*)malloc(sizeof(int32_t));
  }
  int32_t cand[8 + 8 * 32];
  for (int l = 1; l <= L; ++l) {
    const int64_t count = nodes_at(l);
    int64_t cap[4] = {count * 16 + 16, count * 12 + 16, count * 6 + 16, count * 8 + 16};
    int64_t tot[4] = {0, 0, 0, 0};
    for (int k = 0; k < 4; ++k) {
      rep->lst_off[l][k] = (int32_t*)malloc(sizeof(int32_t) * (size_t)(count + 1));
      rep->lst_ids[l][k] = (int32_t*)malloc(sizeof(int32_t) * (size_t)cap[k]);
    }
    for (int64_t m = 0; m < count; ++m) {
      int nc = 0;
      const int64_t base = (m >> 3) << 3;
      for (int64_t s = base; s < base + 8; ++s)
        if (s != m) cand[nc++] = (int32_t)s;
      const int64_t par = m >> 3;
      const int kmax = V == 1 ? 0 : V == 2 ? 3 : 2;
      for (int k = 1; k <= kmax; ++k) { /* parent near_edge, near_face[, near_vertex] */
        const int32_t* po = rep->lst_off[l - 1][k];
        const int32_t* pi = rep->lst_ids[l - 1][k];
        for (int32_t e = po[par]; e < po[par + 1]; ++e)
          for (int c = 0; c < 8; ++c) cand[nc++] = (int32_t)(8 * (int64_t)pi[e] + c);
      }
      qsort(cand, (size_t)nc, sizeof(int32_t), cmp_i32);
      int mx, my, mz;
      morton_decode(m, l, &mx, &my, &mz);
      for (int k = 0; k < 4; ++k) rep->lst_off[l][k][m] = (int32_t)tot[k];
      for (int q = 0; q < nc; ++q) {
        int k = 0;
        if (V != 1) {
          int cx, cy, cz;
          morton_decode(cand[q], l, &cx, &cy, &cz);
          const int cls = classify_offset(cx - mx, cy - my, cz - mz); /* self impossible */
          k = cls == 4 ? 0 : cls == 3 ? (V == 2 ? 3 : 0) : cls == 2 ? 1 : 2;
        }
        if (tot[k] == cap[k]) {
          cap[k] *= 2;
          rep->lst_ids[l][k] =
              (int32_t*)realloc(rep->lst_ids[l][k], sizeof(int32_t) * (size_t)cap[k]);
        }
        rep->lst_ids[l][k][tot[k]++] = cand[q];
      }
    }
    for (int k = 0; k < 4; ++k) rep->lst_off[l][k][count] = (int32_t)tot[k];
  }
}

static kblock make_block(const orc_rep* rep, int level, int32_t target, int32_t source) {
  /* HMatrixRep::make_block (hmatrix.cpp:43-50) */
  const int64_t xb = rep->off[level][target], xe = rep->off[level][target + 1];
  const int64_t yb = rep->off[level][source], ye = rep->off[level][source + 1];
  kblock b;
  b.kid = rep->kid;
  b.diag = rep->diag;
  b.rx = rep->px + xb;
  b.ry = rep->py + xb;
  b.rz = rep->pz + xb;
  b.cx = rep->px + yb;
  b.cy = rep->py + yb;
  b.cz = rep->pz + yb;
  b.m = xe - xb;
  b.n = ye - yb;
  b.diag_offset = xb - yb;
  return b;
}

void orc_free(orc_rep* rep) {
  if (!rep) return;
  free(rep->perm);
  free(rep->px);
  free(rep->py);
  free(rep->pz);
  for (int l = 0; l < ORC_MAX_LEVELS; ++l) {
    free(rep->off[l]);
    for (int k = 0; k < 4; ++k) {
      free(rep->lst_off[l][k]);
      free(rep->lst_ids[l][k]);
    }
    free(rep->lr[l].target);
    free(rep->lr[l].source);
    free(rep->lr[l].rank);
    free(rep->lr[l].piv_off);
    free(rep->lr[l].lu_off);
  }
  free(rep->piv_row);
  free(rep->piv_col);
  free(rep->lu);
  free(rep->d_target);
  free(rep->d_source);
  free(rep);
}

/* initialize (hmatrix.cpp:52-151) */
int orc_initialize(const double* xyz, int64_t n, int kernel_id, double diag, int n_max,
                   double eps, int depth_cap, int64_t max_rank, int variant, orc_rep** out) {
  *out = NULL;
  if (n == 0) {
    set_err("initialize: empty point set");
    return ORC_EINVAL;
  }
  if (!(eps > 0)) {
    set_err("initialize: eps <= 0");
    return ORC_EINVAL;
  }
  orc_rep* rep = (orc_rep*)calloc(1, sizeof(orc_rep));
  rep->kid = kernel_id;
  rep->diag = diag;
  rep->eps = eps;
  rep->max_rank = max_rank;
  if (variant < 0 || variant > 2) {
    orc_free(rep);
    set_err("unknown variant");
    return ORC_EINVAL;
  }
  rep->variant = variant;
  int st = build_tree(rep, xyz, n, n_max, depth_cap);
  if (st != ORC_OK) {
    orc_free(rep);
    return st;
  }
  build_lists(rep);
  const int L = rep->depth;

  /* per-level ACA jobs: (m, j in inter) with both non-empty (hmatrix.cpp:74-98) */
  int64_t piv_total = 0, lu_total = 0;
  typedef struct {
    int32_t* rp;
    int32_t* cp;
    double* lu;
  } res_t;
  for (int l = 1; l <= L; ++l) {
    const int64_t cnt = nodes_at(l);
    const int64_t* off = rep->off[l];
    const int32_t* lo = rep->lst_off[l][0];
    const int32_t* li = rep->lst_ids[l][0];
    int64_t nj = 0;
    for (int64_t m = 0; m < cnt; ++m) {
      if (off[m] == off[m + 1]) continue;
      for (int32_t e = lo[m]; e < lo[m + 1]; ++e)
        if (off[li[e]] != off[li[e] + 1]) ++nj;
    }
    lr_level* lv = &rep->lr[l];
    lv->count = nj;
    lv->target = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nj + 1));
    lv->source = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nj + 1));
    lv->rank = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nj + 1));
    lv->piv_off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nj + 1));
    lv->lu_off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nj + 1));
    nj = 0;
    for (int64_t m = 0; m < cnt; ++m) {
      if (off[m] == off[m + 1]) continue;
      for (int32_t e = lo[m]; e < lo[m + 1]; ++e)
        if (off[li[e]] != off[li[e] + 1]) {
          lv->target[nj] = (int32_t)m;
          lv->source[nj] = li[e];
          ++nj;
        }
    }
    res_t* res = (res_t*)calloc((size_t)(nj + 1), sizeof(res_t));
    int bad = ORC_OK;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t k = 0; k < nj; ++k) {
      const kblock b = make_block(rep, l, lv->target[k], lv->source[k]);
      int r = 0;
      const int s = aca_compress(&b, eps, max_rank, &r, &res[k].rp, &res[k].cp, &res[k].lu);
      if (s != ORC_OK) {
#pragma omp critical
        bad = s;
      } else {
        lv->rank[k] = r;
      }
    }
    if (bad != ORC_OK) {
      for (int64_t k = 0; k < nj; ++k) {
        free(res[k].rp);
        free(res[k].cp);
        free(res[k].lu);
      }
      free(res);
      orc_free(rep);
      return bad;
    }
    /* pack into pools */
    for (int64_t k = 0; k < nj; ++k) {
      lv->piv_off[k] = piv_total;
      lv->lu_off[k] = lu_total;
      piv_total += lv->rank[k];
      lu_total += (int64_t)lv->rank[k] * lv->rank[k];
    }
    rep->piv_row = (int32_t*)realloc(rep->piv_row, sizeof(int32_t) * (size_t)(piv_total + 1));
    rep->piv_col = (int32_t*)realloc(rep->piv_col, sizeof(int32_t) * (size_t)(piv_total + 1));
    rep->lu = (double*)realloc(rep->lu, sizeof(double) * (size_t)(lu_total + 1));
    for (int64_t k = 0; k < nj; ++k) {
      const int r = lv->rank[k];
      memcpy(rep->piv_row + lv->piv_off[k], res[k].rp, sizeof(int32_t) * (size_t)r);
      memcpy(rep->piv_col + lv->piv_off[k], res[k].cp, sizeof(int32_t) * (size_t)r);
      memcpy(rep->lu + lv->lu_off[k], res[k].lu, sizeof(double) * (size_t)r * (size_t)r);
      free(res[k].rp);
      free(res[k].cp);
      free(res[k].lu);
    }
    free(res);
  }

  /* leaf dense blocks in visit order: self, edge, face, vertex (hmatrix.cpp:105-120) */
  {
    const int64_t cnt = nodes_at(L);
    const int64_t* off = rep->off[L];
    int64_t nd = 0;
    for (int pass = 0; pass < 2; ++pass) {
      nd = 0;
      for (int64_t m = 0; m < cnt; ++m) {
        if (off[m] == off[m + 1]) continue;
        if (pass) {
          rep->d_target[nd] = (int32_t)m;
          rep->d_source[nd] = (int32_t)m;
        }
        ++nd;
        for (int k = 1; k <= 3; ++k) {
          const int32_t* lo = rep->lst_off[L][k];
          const int32_t* li = rep->lst_ids[L][k];
          for (int32_t e = lo[m]; e < lo[m + 1]; ++e) {
            if (off[li[e]] == off[li[e] + 1]) continue;
            if (pass) {
              rep->d_target[nd] = (int32_t)m;
              rep->d_source[nd] = li[e];
            }
            ++nd;
          }
        }
      }
      if (!pass) {
        rep->d_target = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nd + 1));
        rep->d_source = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nd + 1));
      }
    }
    rep->ndense = nd;
  }
  *out = rep;
  return ORC_OK;
}

/* matvec (hmatrix.cpp:153-226) */
int orc_matvec(const orc_rep* rep, const double* x, double* b) {
  const int64_t n = rep->n;
  const int L = rep->depth;
  double* xp = (double*)malloc(sizeof(double) * (size_t)n);
  double* bp = (double*)calloc((size_t)n, sizeof(double));
  for (int64_t p = 0; p < n; ++p) xp[p] = x[rep->perm[p]];
  int bad = ORC_OK;

  /* dense leaf pass: runs of equal target, one writer per run */
  {
    int64_t* runs = (int64_t*)malloc(sizeof(int64_t) * (size_t)(rep->ndense + 2));
    int64_t nr = 0;
    for (int64_t k = 0; k < rep->ndense; ++k)
      if (k == 0 || rep->d_target[k] != rep->d_target[k - 1]) runs[nr++] = k;
    runs[nr] = rep->ndense;
#pragma omp parallel
    {
      double* mat = NULL;
      int64_t matcap = 0;
#pragma omp for schedule(dynamic, 4)
      for (int64_t t = 0; t < nr; ++t) {
        for (int64_t kk = runs[t]; kk < runs[t + 1]; ++kk) {
          const kblock blk = make_block(rep, L, rep->d_target[kk], rep->d_source[kk]);
          if (blk.m * blk.n > matcap) {
            matcap = blk.m * blk.n;
            mat = (double*)realloc(mat, sizeof(double) * (size_t)matcap);
          }
          int s = ORC_OK;
          for (int64_t i = 0; i < blk.m && s == ORC_OK; ++i) s = kb_row(&blk, i, mat + i * blk.n);
          if (s != ORC_OK) {
#pragma omp critical
            bad = s;
            continue;
          }
          const int64_t xb = rep->off[L][rep->d_target[kk]];
          const int64_t yb = rep->off[L][rep->d_source[kk]];
          for (int64_t i = 0; i < blk.m; ++i) { /* bx += mat * xy (hmatrix.cpp:193) */
            double acc = 0.0;
            for (int64_t j = 0; j < blk.n; ++j) acc += mat[i * blk.n + j] * xp[yb + j];
            bp[xb + i] += acc;
          }
        }
      }
      free(mat);
    }
    free(runs);
  }

  /* low-rank passes, levels ascending (hmatrix.cpp:200-214) */
  for (int l = 1; l <= L && bad == ORC_OK; ++l) {
    const lr_level* lv = &rep->lr[l];
    int64_t* runs = (int64_t*)malloc(sizeof(int64_t) * (size_t)(lv->count + 2));
    int64_t nr = 0;
    for (int64_t k = 0; k < lv->count; ++k)
      if (k == 0 || lv->target[k] != lv->target[k - 1]) runs[nr++] = k;
    runs[nr] = lv->count;
    const int64_t blkmax = rep->off[l][1] - rep->off[l][0] + rep->n; /* generous */
    (void)blkmax;
#pragma omp parallel
    {
      double* rowbuf = (double*)malloc(sizeof(double) * (size_t)n);
      double* colbuf = (double*)malloc(sizeof(double) * (size_t)n);
      double* t = (double*)malloc(sizeof(double) * (size_t)n);
#pragma omp for schedule(dynamic, 2)
      for (int64_t r = 0; r < nr; ++r) {
        for (int64_t kk = runs[r]; kk < runs[r + 1]; ++kk) {
          const kblock blk = make_block(rep, l, lv->target[kk], lv->source[kk]);
          const int64_t xb = rep->off[l][lv->target[kk]];
          const int64_t yb = rep->off[l][lv->source[kk]];
          const int s = lr_apply(&blk, lv->rank[kk], rep->piv_row + lv->piv_off[kk],
                                 rep->piv_col + lv->piv_off[kk], rep->lu + lv->lu_off[kk],
                                 xp + yb, bp + xb, rowbuf, colbuf, t);
          if (s != ORC_OK) {
#pragma omp critical
            bad = s;
          }
        }
      }
      free(rowbuf);
      free(colbuf);
      free(t);
    }
    free(runs);
  }
  for (int64_t p = 0; p < n; ++p) b[rep->perm[p]] = bp[p];
  free(xp);
  free(bp);
  if (bad == ORC_EDEGEN_GEOM) set_err("coincident distinct points in block");
  return bad;
}

int orc_depth(const orc_rep* rep) { return rep->depth; }

void orc_export_perm(const orc_rep* rep, int32_t* perm) {
  memcpy(perm, rep->perm, sizeof(int32_t) * (size_t)rep->n);
}

void orc_export_offsets(const orc_rep* rep, int level, int64_t* off) {
  memcpy(off, rep->off[level], sizeof(int64_t) * (size_t)(nodes_at(level) + 1));
}

int64_t orc_export_list(const orc_rep* rep, int level, int kind, int32_t* offsets,
                        int32_t* ids) {
  const int64_t cnt = nodes_at(level);
  const int32_t* o = rep->lst_off[level][kind];
  if (offsets) memcpy(offsets, o, sizeof(int32_t) * (size_t)(cnt + 1));
  if (ids) memcpy(ids, rep->lst_ids[level][kind], sizeof(int32_t) * (size_t)o[cnt]);
  return o[cnt];
}

int64_t orc_lr_blocks(const orc_rep* rep, int level, int32_t* target, int32_t* source,
                      int32_t* rank) {
  const lr_level* lv = &rep->lr[level];
  if (level < 1 || level > rep->depth) return 0;
  if (target) {
    memcpy(target, lv->target, sizeof(int32_t) * (size_t)lv->count);
    memcpy(source, lv->source, sizeof(int32_t) * (size_t)lv->count);
    memcpy(rank, lv->rank, sizeof(int32_t) * (size_t)lv->count);
  }
  return lv->count;
}

void orc_lr_block_detail(const orc_rep* rep, int level, int64_t k, int32_t* row_piv,
                         int32_t* col_piv, double* lu) {
  const lr_level* lv = &rep->lr[level];
  const int r = lv->rank[k];
  memcpy(row_piv, rep->piv_row + lv->piv_off[k], sizeof(int32_t) * (size_t)r);
  memcpy(col_piv, rep->piv_col + lv->piv_off[k], sizeof(int32_t) * (size_t)r);
  memcpy(lu, rep->lu + lv->lu_off[k], sizeof(double) * (size_t)r * (size_t)r);
}

/* stats (hmatrix.cpp:228-251) */
void orc_stats(const orc_rep* rep, uint64_t* out5) {
  uint64_t fl = 0, in = 0, mr = 0;
  for (int l = 1; l <= rep->depth; ++l) {
    const lr_level* lv = &rep->lr[l];
    for (int64_t k = 0; k < lv->count; ++k) {
      const uint64_t r = (uint64_t)lv->rank[k];
      fl += r * r;
      in += 2 * r;
      if (r > mr) mr = r;
    }
  }
  const int L = rep->depth;
  for (int64_t k = 0; k < rep->ndense; ++k) {
    const int64_t* off = rep->off[L];
    fl += (uint64_t)(off[rep->d_target[k] + 1] - off[rep->d_target[k]]) *
          (uint64_t)(off[rep->d_source[k] + 1] - off[rep->d_source[k]]);
  }
  out5[0] = fl;
  out5[1] = in;
  out5[2] = 8 * fl + 4 * in;
  out5[3] = mr;
  out5[4] = (uint64_t)rep->depth;
}

/* reference_error (hmatrix.cpp:253-291): all rows for N <= 4096, else 2000
 * rows drawn by mt19937_64(7). */
double orc_reference_error(const orc_rep* rep, const double* x, const double* b) {
  const int64_t n = rep->n;
  double* xp = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t p = 0; p < n; ++p) xp[p] = x[rep->perm[p]];
  int64_t nrows = n <= 4096 ? n : 2000;
  int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)nrows);
  if (n <= 4096) {
    for (int64_t i = 0; i < n; ++i) rows[i] = i;
  } else {
    mt64 g;
    mt64_seed(&g, 7);
    for (int64_t k = 0; k < nrows; ++k) rows[k] = (int64_t)(uniform01(&g) * (double)n);
  }
  kblock whole;
  whole.kid = rep->kid;
  whole.diag = rep->diag;
  whole.rx = whole.cx = rep->px;
  whole.ry = whole.cy = rep->py;
  whole.rz = whole.cz = rep->pz;
  whole.m = whole.n = n;
  whole.diag_offset = 0;
  double err2 = 0.0, ref2 = 0.0;
#pragma omp parallel reduction(+ : err2, ref2)
  {
    double* buf = (double*)malloc(sizeof(double) * (size_t)n);
#pragma omp for schedule(dynamic, 16)
    for (int64_t k = 0; k < nrows; ++k) {
      const int64_t p = rows[k];
      kb_row(&whole, p, buf);
      double exact = 0.0;
      for (int64_t j = 0; j < n; ++j) exact += buf[j] * xp[j];
      const double approx = b[rep->perm[p]];
      err2 += (approx - exact) * (approx - exact);
      ref2 += exact * exact;
    }
    free(buf);
  }
  free(rows);
  free(xp);
  return sqrt(err2 / ref2);
}

int orc_aca_block(const double* xs, int64_t m, const double* ys, int64_t n, int kernel_id,
                  double eps, int64_t max_rank, int32_t* row_piv, int32_t* col_piv,
                  double* lu, int64_t cap, int* rank_out) {
  double* s = (double*)malloc(sizeof(double) * (size_t)(3 * (m + n)));
  for (int64_t i = 0; i < m; ++i)
    for (int d = 0; d < 3; ++d) s[d * m + i] = xs[3 * i + d];
  double* t = s + 3 * m;
  for (int64_t j = 0; j < n; ++j)
    for (int d = 0; d < 3; ++d) t[d * n + j] = ys[3 * j + d];
  kblock b;
  b.kid = kernel_id;
  b.diag = 0.0;
  b.rx = s;
  b.ry = s + m;
  b.rz = s + 2 * m;
  b.cx = t;
  b.cy = t + n;
  b.cz = t + 2 * n;
  b.m = m;
  b.n = n;
  b.diag_offset = NO_DIAG;
  int r = 0;
  int32_t *rp = NULL, *cp = NULL;
  double* l = NULL;
  const int st = aca_compress(&b, eps, max_rank, &r, &rp, &cp, &l);
  if (st == ORC_OK) {
    *rank_out = r;
    if (r <= cap) {
      memcpy(row_piv, rp, sizeof(int32_t) * (size_t)r);
      memcpy(col_piv, cp, sizeof(int32_t) * (size_t)r);
      memcpy(lu, l, sizeof(double) * (size_t)r * (size_t)r);
    }
  }
  free(rp);
  free(cp);
  free(l);
  free(s);
  return st;
}

/* tests/oracles.cpp:18-33 */
int orc_dense_matvec(const double* xyz, int64_t n, int kernel_id, double diag,
                     const double* x, double* b) {
  int bad = ORC_OK;
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      if (i == j) continue;
      double v;
      if (eval_pair(kernel_id, xyz + 3 * i, xyz + 3 * j, &v) != ORC_OK) {
#pragma omp critical
        bad = ORC_EDEGEN_GEOM;
        v = 0.0;
      }
      acc += v * x[j];
    }
    b[i] = acc + diag * x[i];
  }
  if (bad) set_err("coincident distinct points");
  return bad;
}

int orc_exact_rows(const double* xyz, int64_t n, int kernel_id, double diag,
                   const double* x, const int64_t* rows, int64_t nrows, double* out) {
  int bad = ORC_OK;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t k = 0; k < nrows; ++k) {
    const int64_t i = rows[k];
    double acc = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      if (i == j) continue;
      double v;
      if (eval_pair(kernel_id, xyz + 3 * i, xyz + 3 * j, &v) != ORC_OK) {
#pragma omp critical
        bad = ORC_EDEGEN_GEOM;
        v = 0.0;
      }
      acc += v * x[j];
    }
    out[k] = acc + diag * x[i];
  }
  return bad;
}

/* Raw uniform01 stream (kernel.hpp:24-26), for reproducing the reference
 * tests' geometries (test_lowrank.cpp:13-21 unit_cube_points). */
void orc_uniform_stream(int64_t n, uint64_t seed, double* out) {
  mt64 g;
  mt64_seed(&g, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = uniform01(&g);
}

/* Tree and lists only (no ACA): for bit-exact parity at full BASELINE sizes. */
int orc_tree_lists(const double* xyz, int64_t n, int n_max, int depth_cap, int variant,
                   orc_rep** out) {
  *out = NULL;
  if (variant < 0 || variant > 2) {
    set_err("unknown variant");
    return ORC_EINVAL;
  }
  orc_rep* rep = (orc_rep*)calloc(1, sizeof(orc_rep));
  rep->variant = variant;
  int st = build_tree(rep, xyz, n, n_max, depth_cap);
  if (st != ORC_OK) {
    orc_free(rep);
    return st;
  }
  build_lists(rep);
  *out = rep;
  return ORC_OK;
}
