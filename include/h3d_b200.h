/*
 * h3d_b200 — C-ABI of the B200-native HODLR3D engine (drop-in boundary).
 *
 * The reference has no C ABI; its operator surface for this path is the C++
 * free-function API of /root/reference/proj/include/h3d/hmatrix.hpp and
 * parallel.hpp. Each entry point below names the reference interface it
 * replaces. Plain pointers and sizes only; no torch types. The C++ host layer
 * (include/h3d_b200.hpp, implemented in paper_2307_16303_b200/csrc/hmatrix_b200.cpp,
 * built as lib/libh3d_b200pp.so) restores the reference's C++ signatures and
 * exception types on top of this header.
 *
 * Error convention: every int-returning call returns H3D_OK (0) or a status
 * below; h3d_last_error() returns the thread-local message. Status codes map
 * to the reference exceptions:
 *   H3D_EINVAL       -> std::invalid_argument
 *   H3D_EDEGEN_GEOM  -> h3d::DegenerateGeometryError   (kernel.hpp:64-66)
 *   H3D_EDEGEN_DIST  -> h3d::DegenerateDistributionError (octree.hpp:41-43)
 *   H3D_ECUDA / H3D_ENCCL / H3D_ENOMEM -> std::runtime_error
 *   H3D_EUNSUPPORTED -> std::invalid_argument (e.g. custom std::function kernels,
 *                       kernel.hpp:56-57, cannot cross to the device)
 */
#ifndef H3D_B200_H
#define H3D_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define H3D_B200_ABI_VERSION 5

enum h3d_status {
  H3D_OK = 0,
  H3D_EINVAL = 1,
  H3D_EDEGEN_GEOM = 2,
  H3D_EDEGEN_DIST = 3,
  H3D_ECUDA = 4,
  H3D_ENCCL = 5,
  H3D_ENOMEM = 6,
  H3D_EUNSUPPORTED = 7
};

/* Kernel ids follow h3d::KernelId (reference kernel.hpp:42). */
enum h3d_kernel { H3D_LAPLACE3D = 0, H3D_R4 = 1, H3D_HELMHOLTZ_RE = 2 };

/* Block-structure variants, h3d::Variant order (reference octree.hpp:80):
 * HODLR3D (vertex partners compressed), HODLR (every sibling compressed, weak
 * admissibility) and H-strong (only well-separated partners compressed; vertex
 * partners join the dense near field). Lists: octree.cpp:197-260. */
enum h3d_variant { H3D_HODLR3D = 0, H3D_HODLR = 1, H3D_HSTRONG = 2 };

/* Near-field (dense leaf block) storage; mirrors h3d::DenseMode
 * (reference hmatrix.hpp:12-14): Cached stores the blocks at initialize,
 * OnTheFly regenerates them in every matvec. */
enum h3d_near_mode { H3D_NEAR_STORED = 0, H3D_NEAR_MATRIX_FREE = 1 };

/* Options; the first six fields are h3d::HmatOptions (hmatrix.hpp:16-22) and
 * KernelSpec (kernel.hpp:46-53). */
typedef struct {
  int kernel_id;        /* h3d_kernel */
  double diagonal;      /* KernelSpec::diagonal, entry (i,i) */
  int n_max;            /* leaf threshold: depth = min l with max occupancy < n_max */
  double epsilon;       /* ACA tolerance */
  int depth_cap;        /* Morton resolution / DegenerateDistributionError cap */
  int64_t max_rank;     /* 0: min(|X|,|Y|) per block */
  int near_mode;        /* h3d_near_mode */
  int device;           /* CUDA device ordinal */
  int shard_rank;       /* Morton-subtree row ownership (parallel.hpp:9-30 analogue) */
  int shard_world;      /* 1 = single GPU owns every row */
  /* How each level's admissible blocks are applied:
   * 0 = stream explicit ACA factors at every level;
   * 1 = auto (default): leaf level evaluated exactly, upper levels split
   *     between streamed factors and matrix-free proxies (pivots + LU, the
   *     reference's own storage, lowrank.cpp:291-327) by a HBM/FP64 cost model;
   *     stream levels of >= 8 GB per phase become half levels (laplace3d, r4);
   * 2 = explicit per level from level_modes[l] (0 stream, 1 proxy, 2 direct,
   *     3 pair = explicit factors, one pair-major pass (U read once, V twice,
   *     the second time from L2), 4 fused = proxy storage, pair-major, each
   *     regenerated entry evaluated once for both orientations, 5 half =
   *     U' = K(X, tau) (LR)^-1 streamed and K(sigma, Y) regenerated, no solves
   *     (laplace3d and r4 only), 6 split = proxy storage in three passes: the
   *     X-role entries twice, the Y-role entries once for both uses between two
   *     solve rounds; direct only at the leaf level, pair and fused ranks <= 128,
   *     fused nodes <= 352 points). */
  int mode_policy;
  int level_modes[16];
  int variant;          /* h3d_variant (Variant argument of initialize, hmatrix.hpp:57-58) */
  /* Multi-GPU: 1 = every rank returns the FULL b, as parallel_matvec does
   * (its final gather in fixed worker order, parallel.cpp:284-290): the owned
   * Morton slices are all-gathered over NCCL after the matvec. 0 (default):
   * each rank writes only its owned rows of b. */
  int64_t gather_b;
  int64_t reserved[3];
} h3d_options;

/* Per-call matvec timing, milliseconds (CUDA events on the engine stream);
 * analogue of h3d::MatvecTiming (hmatrix.hpp:60-66). */
typedef struct {
  double total_ms;      /* whole call incl. copies */
  double h2d_ms;        /* host x -> device (host mode only) */
  double gather_ms;     /* x permutation to Morton order */
  double exchange_ms;   /* multi-GPU all-gather of x (0 on one GPU) */
  double phase1_ms;     /* V^T x over the factor pool (+ partial reduce) */
  double phase2_ms;     /* near field + U t, fused un-permute */
  double d2h_ms;        /* device b -> host (host mode only) */
  int64_t launches;     /* kernels launched by this call */
  double device_ms;     /* device part (gather .. un-permute). A call replayed as one
                           CUDA graph reports only this, h2d_ms, d2h_ms and total_ms
                           (the per-phase fields stay 0; H3D_TUNE=graphs=0 splits them) */
} h3d_timing;

/* Representation statistics; superset of h3d::RepStats (hmatrix.hpp:73-85). */
typedef struct {
  int depth;
  int max_rank;
  int64_t n;
  int64_t lowrank_blocks;     /* ordered admissible blocks (reference lr_levels total) */
  int64_t aca_pairs;          /* unordered pairs compressed (symmetric storage) */
  int64_t sum_rank;           /* sum over pairs */
  int64_t factor_doubles;     /* sum over pairs of r (m + n): the factor pool */
  int64_t factor_bytes_alloc; /* W incl. padding */
  int64_t tvec_doubles;       /* S pool */
  int64_t near_blocks;        /* dense leaf blocks (reference dense_blocks) */
  int64_t near_entries;       /* sum |X||Y| over dense blocks */
  int64_t near_bytes_stored;  /* 0 in matrix-free mode */
  uint64_t ref_float_count;   /* reference RepStats::float_count convention: sum r^2 (ordered
                                 blocks, each pair counted twice) + dense areas */
  uint64_t ref_int_count;     /* 2 * sum r over ordered blocks */
  double compression_ratio;   /* ref_float_count / N^2 */
  double build_ms_tree;
  double build_ms_lists;
  double build_ms_aca_rank;
  double build_ms_aca_write;
  double build_ms_total;
  int64_t phase1_items;
  int64_t owned_row_begin;    /* shard rows [begin, end) in Morton order */
  int64_t owned_row_end;
  int level_modes[16];        /* applied mode per level (0 stream, 1 proxy, 2 direct, 3 pair, 4 fused,
                                 5 half, 6 split) */
  int64_t proxy_units;        /* sum over proxy-level pairs of r (m + n) */
  int64_t direct_evals;       /* leaf-level admissible entries evaluated exactly */
  int64_t lu_doubles;         /* packed LU storage of proxy-level pairs */
  int64_t level_units[16];    /* per level: sum over pairs of r (m + n) */
  double level_aca_ms[16];    /* per level: ACA wall time (rank + write pass) */
  double build_ms_plan;       /* mode choice, layout, descriptor upload (host planner) */
  double build_ms_post;       /* proxy pivot gather + LU triangular inverses */
  double build_ms_near;       /* near-field symmetry scan */
  int64_t half_units;         /* half levels: sum over pairs of r n (the regenerated side) */
} h3d_stats;

typedef struct h3d_dev h3d_dev;

const char* h3d_last_error(void);
int h3d_abi_version(void);
void h3d_default_options(h3d_options* opt);

/* Input generation, bit-identical to the reference:
 * generate_points(UniformRandom, n, seed) (kernel.cpp:88-95), AoS xyz[3n];
 * the CLI right-hand side mt19937_64(seed), 2u-1 (reference proj/tools/h3d.cpp:135-137). */
int h3d_generate_points(int64_t n, uint64_t seed, double* xyz);
void h3d_random_vector(int64_t n, uint64_t seed, double* out);

/* Replaces h3d::initialize(PointSet, KernelSpec, Variant, HmatOptions)
 * (hmatrix.hpp:57-58 / hmatrix.cpp:52-151): octree + lists (opt->variant) +
 * batched ACA on the device. xyz is host AoS (Point3[n]). */
int h3d_dev_create(const double* xyz, int64_t n, const h3d_options* opt, h3d_dev** out);
void h3d_dev_destroy(h3d_dev* dev);

/* Replaces h3d::matvec(rep, x, MatvecTiming*) (hmatrix.hpp:70-71): b = A~ x in
 * ORIGINAL point order. where = 0: x/b are host pointers (copies included,
 * returns after b is written); where = 1: device pointers on dev's GPU
 * (returns after the result is complete). timing may be NULL. */
int h3d_dev_matvec(h3d_dev* dev, const double* x, double* b, int where, h3d_timing* timing);

/* Stream-ordered variant for device-resident vectors: enqueue one matvec on
 * the caller's cudaStream_t (may be the caller's framework stream) and return
 * without synchronising. Same numerics as h3d_dev_matvec. */
int h3d_dev_matvec_async(h3d_dev* dev, const double* x_dev, double* b_dev, void* stream);
/* Per-phase CUDA-event timing of async matvecs: enable (resets) with room for
 * `capacity` calls; read = synchronise and sum the phases over the recorded
 * calls (*steps). Used by bench.py for live per-kernel durations. */
int h3d_dev_profile(h3d_dev* dev, int enable, int64_t capacity);
int h3d_dev_profile_read(h3d_dev* dev, h3d_timing* sum, int64_t* steps);
/* Per-kernel CUDA-event durations of the profiled calls, summed (ms), launch
 * counts and (optional, may be NULL) summed start offsets from the call's
 * first event, in the order of h3d_kernel_slot; filled by the last
 * h3d_dev_profile_read. Kernels of different lanes overlap in time. */
typedef enum {
  H3D_K_GATHER = 0,    /* x -> Morton order (+ packed weights) */
  H3D_K_P1_STREAM,     /* phase 1, stream levels (bulk-copy tile pipeline, HBM) */
  H3D_K_RED_STREAM,    /* phase-1 partial reductions, stream levels */
  H3D_K_P2_STREAM,     /* phase 2, stream levels */
  H3D_K_P1_PROXY,      /* phase 1, proxy levels (FP64) */
  H3D_K_RED_PROXY,     /* phase-1 partial reductions, proxy levels */
  H3D_K_SOLVE,         /* proxy triangular solves */
  H3D_K_P2_PROXY,      /* phase 2, proxy levels (FP64) */
  H3D_K_NEAR,          /* near field + direct leaf blocks (FP64) */
  H3D_K_COMBINE,       /* sum of the per-level partials, un-permute */
  H3D_K_PAIR,          /* pair levels: fused one-read pass + per-node gather (HBM) */
  H3D_K_FUSED,         /* fused levels: one evaluation per entry, both orientations (FP64) */
  H3D_K_HALF,          /* half levels, regenerated side: both uses per entry (FP64) */
  H3D_K_COUNT
} h3d_kernel_slot;
int h3d_dev_profile_kernels(const h3d_dev* dev, double* ms_sum, int64_t* launches, double* start_sum,
                            int count);

/* GMRES on the device (replaces h3d::gmres + IEOperator::apply,
 * solver.hpp:10-28,39-53; solver.cpp:22-125,199-206): solves
 * (alpha I + beta A) x = rhs with A this handle's HODLR3D operator
 * (alpha = 0, beta = 1: the plain matvec; the IE operator uses
 * alpha = 1 + cell self-integral, beta = cell volume). Arnoldi with modified
 * Gram-Schmidt and Givens rotations, restart 0 = unrestarted, iterate
 * returned with converged = 0 when max_iter is exhausted. hist (may be NULL)
 * receives up to hist_cap relative residuals, one per iteration. rhs / x are
 * host (where = 0) or device (where = 1) arrays in original point order. */
typedef struct {
  int iterations;
  int converged;
  int history_len;
  int reserved;
  double solve_ms;
  double final_relres;  /* |rhs - op(x)| / |rhs| of the returned iterate */
} h3d_gmres_info;
int h3d_dev_gmres(h3d_dev* dev, const double* rhs, double* x, int where, double alpha, double beta,
                  double tol, int restart, int max_iter, double* hist, int hist_cap, h3d_gmres_info* info);
/* Exact dense product b = K x (diagonal rule), O(N^2) on the device: the
 * reference's dense row sums for manufactured right-hand sides
 * (solver.cpp:247-258). Single-shard handles only. */
int h3d_dev_direct_matvec(h3d_dev* dev, const double* x, double* b, int where);
/* Replaces h3d::reference_error(rep, x, b_approx, exact_limit, sample_rows,
 * seed) (hmatrix.hpp:87-93, hmatrix.cpp:253-291): relative 2-norm error of
 * b (original order) against exact row sums of K x, every row when
 * N <= exact_limit, else sample_rows Morton positions p drawn as
 * floor(uniform01(mt19937_64(seed)) * N) (duplicates possible), exactly the
 * reference's rows. The exact sums run on the device (full-accuracy radial
 * map, diagonal rule); x and b are host (where = 0) or device (where = 1)
 * arrays of length N. Defaults of the reference: 4096, 2000, 7. */
int h3d_dev_reference_error(h3d_dev* dev, const double* x, const double* b, int where, int64_t exact_limit,
                            int64_t sample_rows, uint64_t seed, double* out);
/* Collocation helpers of the IE driver: the tensor grid (kernel.cpp:96-109)
 * and the cell self-integral of 1/r (solver.cpp:127-193). */
int h3d_generate_grid_points(int64_t n, double* xyz);
double h3d_cell_self_integral(double h);

/* Replaces h3d::stats(rep) (hmatrix.hpp:85). */
int h3d_dev_stats(const h3d_dev* dev, h3d_stats* out);

/* Parity exports (tree and lists are bit-exact with reference octree.cpp):
 * perm[n] (permuted position -> original index, Octree::perm, octree.hpp:61);
 * offsets[8^level + 1] (node m = [off[m], off[m+1]), Octree::levels). */
int h3d_dev_export_tree(const h3d_dev* dev, int32_t* perm, int level, int64_t* offsets);
/* Interaction list CSR at a level, kind 0 inter / 1 near_edge / 2 near_face /
 * 3 near_vertex (H-strong only) (NodeLists, octree.hpp:88-93). ids may be NULL to query *count. */
int h3d_dev_export_list(const h3d_dev* dev, int level, int kind, int32_t* offsets,
                        int32_t* ids, int64_t* count);
/* Compressed pairs at a level: (X, Y, rank) with X < Y (Morton ids). */
int h3d_dev_export_pairs(const h3d_dev* dev, int level, int32_t* x, int32_t* y, int32_t* rank,
                         int64_t* count);

/* Multi-GPU (Morton-subtree ownership; replaces parallel_matvec,
 * parallel.hpp:65-66). One process per GPU: rank 0 calls h3d_nccl_get_id and
 * broadcasts the 128 bytes; every rank attaches before its first matvec. */
int h3d_nccl_get_id(void* id128);
int h3d_dev_attach_nccl(h3d_dev* dev, const void* id128, int rank, int world);
/* Exchange volume of this rank (analogue of h3d::CommLedger,
 * parallel.hpp:38-51): doubles received per matvec by the x all-gather and
 * (gather_b) the b all-gather, NCCL collectives per matvec, and matvecs run
 * with the communicator attached. Zero with no communicator. */
typedef struct {
  int64_t x_gather_doubles;
  int64_t b_gather_doubles;
  int64_t collectives;
  int64_t matvecs;
  int64_t reserved[4];
} h3d_comm_ledger;
int h3d_dev_comm_ledger(const h3d_dev* dev, h3d_comm_ledger* out);

/* Host planner (no GPU): the shard ownership, column layout, work items and
 * leaf lists the engine derives from the tree, for CPU verification of the
 * multi-GPU logic. offsets = concat over levels of 8^l + 1 int64; list_off =
 * concat over (level 1..L, kind 0..3) of 8^l + 1 int32; list_ids = concat of
 * the ids; list_counts[4*l + k] = ids per (level, kind); modes = L + 1 ints
 * (0 stream, 1 proxy, 2 direct) or NULL. */
typedef struct h3d_plan h3d_plan;
int h3d_plan_create(int depth, int64_t n, const int64_t* offsets, const int32_t* list_off,
                    const int32_t* list_ids, const int64_t* list_counts, int shard_rank,
                    int shard_world, const int* modes, h3d_plan** out);
void h3d_plan_destroy(h3d_plan* plan);
int h3d_plan_pairs(const h3d_plan* plan, int level, int32_t* x, int32_t* y, int64_t* count);
int h3d_plan_set_ranks(h3d_plan* plan, int level, const int32_t* ranks);
int h3d_plan_set_mode(h3d_plan* plan, int level, int mode);
int h3d_plan_layout(h3d_plan* plan);
/* Named result arrays (raw bytes; *count = elements); see planner.h. */
int h3d_plan_array(const h3d_plan* plan, const char* name, int level, void* out, int64_t* count);

#ifdef __cplusplus
}
#endif
#endif /* H3D_B200_H */
