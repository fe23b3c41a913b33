/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the HODLR3D hot path.
 *
 * A plain-C restatement of the reference algorithm
 * (/root/reference/proj/src/{kernel,octree,lowrank,hmatrix}.cpp). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it, and
 * only as the checker. The product library (paper_2307_16303_b200/) never
 * links or calls it.
 *
 * Pinned against the in-place build of the reference (oracle/_ref, see
 * oracle/Makefile) through tests/golden/ and tests/test_oracle_pin.py:
 * tree, lists, pivots and matvec are bit-identical to the shim-built
 * reference when both are compiled with -ffp-contract=off.
 */
#ifndef H3D_ORACLE_H
#define H3D_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* kernel ids follow h3d::KernelId (kernel.hpp:42) */
enum { ORC_LAPLACE = 0, ORC_R4 = 1, ORC_HELMHOLTZ = 2 };

enum {
  ORC_OK = 0,
  ORC_EINVAL = 1,     /* std::invalid_argument */
  ORC_EDEGEN_GEOM = 2,/* DegenerateGeometryError */
  ORC_EDEGEN_DIST = 3 /* DegenerateDistributionError */
};

typedef struct orc_rep orc_rep;

const char* orc_last_error(void);

/* kernel.cpp:88-95 (uniform) */
int orc_generate_points(int64_t n, uint64_t seed, double* xyz);
/* tools/h3d.cpp:135-137: mt19937_64(seed), 2u-1 */
void orc_random_vector(int64_t n, uint64_t seed, double* out);

/* hmatrix.cpp:52-151 (on-the-fly dense); variant 0 hodlr3d, 1 hodlr, 2 hstrong */
int orc_initialize(const double* xyz, int64_t n, int kernel_id, double diag, int n_max,
                   double eps, int depth_cap, int64_t max_rank, int variant, orc_rep** out);
void orc_free(orc_rep* rep);
/* hmatrix.cpp:153-226 */
int orc_matvec(const orc_rep* rep, const double* x, double* b);

int orc_depth(const orc_rep* rep);
void orc_export_perm(const orc_rep* rep, int32_t* perm);
/* 8^l + 1 offsets: node m covers [off[m], off[m+1]) */
void orc_export_offsets(const orc_rep* rep, int level, int64_t* off);
/* kind 0 inter, 1 near_edge, 2 near_face, 3 near_vertex; offsets has 8^l + 1 entries */
int64_t orc_export_list(const orc_rep* rep, int level, int kind, int32_t* offsets,
                        int32_t* ids);
int64_t orc_lr_blocks(const orc_rep* rep, int level, int32_t* target, int32_t* source,
                      int32_t* rank);
void orc_lr_block_detail(const orc_rep* rep, int level, int64_t k, int32_t* row_piv,
                         int32_t* col_piv, double* lu);
/* {float_count, int_count, memory_bytes, max_rank, depth} (hmatrix.cpp:228-251) */
void orc_stats(const orc_rep* rep, uint64_t* out5);
/* hmatrix.cpp:253-291 */
double orc_reference_error(const orc_rep* rep, const double* x, const double* b);

/* Standalone ACA of the block K(xs, ys) (lowrank.cpp:157-289), AoS inputs. */
int orc_aca_block(const double* xs, int64_t m, const double* ys, int64_t n, int kernel_id,
                  double eps, int64_t max_rank, int32_t* row_piv, int32_t* col_piv,
                  double* lu, int64_t cap, int* rank_out);

/* tests/oracles.cpp:18-33 — direct O(N^2) sum in original order. */
int orc_dense_matvec(const double* xyz, int64_t n, int kernel_id, double diag,
                     const double* x, double* b);

/* Exact rows of K x (permuted-order rows given, original-order x); used for
 * sampled error checks at large N (hmatrix.cpp:253-291 row rule). */
int orc_exact_rows(const double* xyz, int64_t n, int kernel_id, double diag,
                   const double* x, const int64_t* rows, int64_t nrows, double* out);

void orc_set_threads(int n);

/* raw uniform01 stream of mt19937_64(seed) (kernel.hpp:24-26) */
void orc_uniform_stream(int64_t n, uint64_t seed, double* out);
/* build_tree + build_interaction_lists only (octree.cpp:76-260), no ACA */
int orc_tree_lists(const double* xyz, int64_t n, int n_max, int depth_cap, int variant,
                   orc_rep** out);

#ifdef __cplusplus
}
#endif
#endif
