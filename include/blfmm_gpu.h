/*
 * blfmm_gpu.h — C ABI of the B200-native band-limited FMM RBF matvec.
 *
 * Drop-in boundary for the reference library blfmm (/root/reference/proj/core).
 * Plain pointers and sizes only; no CUDA or torch types in the signatures
 * (streams are passed as void*). Every entry point returns a status code and
 * leaves a thread-local message for blfmm_last_error().
 *
 * Reference interfaces replaced (file:line under /root/reference/proj/core):
 *   blfmm_plan_create   build_tree(const PointSet&, int)        include/blfmm/geometry.hpp:72
 *                       + make_level_grids(kernel, sigma_leaf, m_leaf, d,
 *                         leaf_level, GridMode, stencil_k)      include/blfmm/mlfmm.hpp:61-63
 *                       (the immutable BoxTree / LevelGrids pair a caller
 *                        builds once and reuses, solver.cpp:280-293)
 *   blfmm_execute       SumResult mlfmm_matvec(const SumRequest&, const BoxTree&,
 *                         const LevelGrids&)                    include/blfmm/mlfmm.hpp:98-99
 *   blfmm_execute_single SumResult fmm_matvec_single(const SumRequest&,
 *                         const BoxTree&)                       include/blfmm/fmm.hpp:55
 *   blfmm_direct        SumResult direct_matvec(kernel, ps, weights,
 *                         use_bandlimited=false, ...)           include/blfmm/fmm.hpp:33-36
 *   blfmm_direct_bandlimited  direct_matvec(kernel, ps, weights,
 *                         use_bandlimited=true, sigma, refinement)  include/blfmm/fmm.hpp:33-36
 *                       and direct_matvec_hybrid(kernel, ps, tree, weights,
 *                         sigma, refinement)                    include/blfmm/fmm.hpp:40-43
 *   blfmm_eval_bandlimited  eval_bandlimited(k, sigma, x, d, refinement)
 *                                                               include/blfmm/bandlimit.hpp:56-62
 *   blfmm_bandlimited_radial_table  bandlimited_radial_table(k, sigma, rmax,
 *                         refinement)                           include/blfmm/bandlimit.hpp:77-79
 *   blfmm_parse_kernel_spec  RadialKernel parse_kernel_spec(const std::string&)
 *                                                               include/blfmm/kernels.hpp:23
 *   blfmm_translation_coefficients  translation_coefficients(k, grid, spectral)
 *                                                               include/blfmm/bandlimit.hpp:106-108
 *   blfmm_get_expansions upsweep / couple / downsweep stage outputs
 *                                                               include/blfmm/mlfmm.hpp:79-94
 *   status codes        std::invalid_argument / std::domain_error /
 *                       blfmm::accuracy_error                   include/blfmm/common.hpp:33-41
 */
#ifndef BLFMM_GPU_H
#define BLFMM_GPU_H

#ifdef __cplusplus
extern "C" {
#endif

#define BLFMM_GPU_ABI_VERSION 4

/* Status codes (reference exception class in parentheses). */
enum blfmm_status {
  BLFMM_OK = 0,
  BLFMM_EINVAL = 1,    /* std::invalid_argument                       */
  BLFMM_EDOMAIN = 2,   /* std::domain_error (unsupported d / kernel)  */
  BLFMM_EACCURACY = 3, /* blfmm::accuracy_error; see blfmm_last_error_value */
  BLFMM_ECUDA = 4,     /* CUDA runtime error, or no usable device     */
  BLFMM_ENCCL = 5,     /* multi-GPU exchange error                    */
  BLFMM_ENOMEM = 6,    /* device allocation failed                    */
  BLFMM_ELENGTH = 7    /* std::length_error (dense backend, N > 8192) */
};

/* RadialKernel::type (kernels.hpp:12-17). The band-limited FMM plan takes the
 * north star's three kernels; the O(N^2) sum (blfmm_direct) and the dense
 * Krylov backend (blfmm_solve_dense) evaluate every type (eval_kernel,
 * kernels.cpp:131-161). */
enum blfmm_kernel_type {
  BLFMM_KERNEL_GAUSSIAN = 0, /* phi = exp(-c r^2)      */
  BLFMM_KERNEL_MQ = 1,       /* phi = sqrt(r^2 + c^2)  */
  BLFMM_KERNEL_IMQ = 2,      /* phi = 1/sqrt(r^2+c^2)  */
  BLFMM_KERNEL_TPS = 3,         /* phi = (-1)^{1+beta/2} r^beta log r; EDOMAIN for a plan */
  BLFMM_KERNEL_WENDLAND_C2 = 4, /* phi = (1 - eps r)_+^4 (4 eps r + 1); EDOMAIN for a plan */
  BLFMM_KERNEL_WENDLAND31 = 5   /* phi = (1 - eps r)_+^3 (3 eps r + 1); EDOMAIN for a plan */
};

/* GridMode (mlfmm.hpp:21-28). `scaled` (per-level halved band, Lagrange
 * M2M/L2L transfers, direct interaction-list couple) needs world == 1 and
 * M^d <= 6400 (EDOMAIN else). */
enum blfmm_grid_mode { BLFMM_GRID_SHARED = 0, BLFMM_GRID_SCALED = 1 };

typedef struct blfmm_plan blfmm_plan;

typedef struct blfmm_plan_desc {
  int d;                  /* 1, 2 or 3 */
  long long n;            /* number of points (>= 0) */
  const double* coords;   /* HOST, n*d doubles, AoS (x0,y0,[z0],x1,...) caller order */
  double domain_lo[3];    /* BoundingBox::lo (geometry.hpp:10-14); unused axes ignored */
  double domain_hi[3];    /* BoundingBox::hi */
  int kernel_type;        /* enum blfmm_kernel_type */
  double kernel_shape;    /* c (Gaussian c = eps^2) */
  double sigma;           /* leaf band limit (> 0) */
  int m_per_dim;          /* quadrature nodes per axis M (>= 2); K = M^d */
  int leaf_level;         /* uniform tree depth L (>= 2, d*L <= 24) */
  int grid_mode;          /* enum blfmm_grid_mode */
  int stencil_k;          /* scaled-mode Lagrange stencil, clamped to M (ignored for shared) */
  int nrhs;               /* right-hand sides per execute (>= 1) */
  int device;             /* CUDA device ordinal, -1 = current */
  const double* c_table;  /* optional HOST override of C(xi_m), K doubles
                             (LowRankFactors::c_vals); scaled mode: (L-1)*K
                             doubles, levels 2..L in order; NULL = compute */
  int rank;               /* multi-GPU: this plan's Morton-range index ... */
  int world;              /* ... of `world` ranges (1 = whole problem) */
} blfmm_plan_desc;

/* SumStats (fmm.hpp:10-14). */
typedef struct blfmm_stats {
  long long near_pairs;
  long long far_work;
  double max_imag_residual;
} blfmm_stats;

/* Plan facts (sizes of the device-resident tree and expansion sets). */
typedef struct blfmm_plan_info {
  int d, m_per_dim, leaf_level, nrhs;
  long long n, K;
  long long boxes[25];      /* nonempty boxes per level 0..L (levels >= 2 used) */
  long long near_pairs;     /* of the owned targets */
  long long far_work;       /* reference formula, mlfmm.cpp:398-404 */
  long long far_work_single;/* fmm.cpp:152,179,209 */
  long long il_pairs;       /* nonempty (target, source) IL pairs, all levels */
  long long owned_begin, owned_end; /* owned sorted-point range (multi-GPU) */
  double plan_seconds;
  long long device_bytes;
  long long stored_nodes;   /* complex coefficients stored per expansion: K, or
                               the Hermitian half spectrum (3-D, M = 16: 2528) */
  int telescoped;           /* 1: execute evaluates G_L from the root multipole
                               (leaf-level couple only) */
  long long near_sym_items; /* symmetric near-field items (leaf pairs evaluated
                               once for both sides; nrhs = 1) */
  long long near_items;     /* one-sided near-field items (up to 96 targets) */
  char kernels[256];        /* the kernel each stage of blfmm_execute launches,
                               "p2m=... m2m=... couple=... l2p=... near=..." */
} blfmm_plan_info;

/* Optional plan tuning (blfmm_plan_create_tuned). blfmm_tuning_defaults
 * fills the values blfmm_plan_create uses; every field selects between
 * kernels or schedules of the same matvec (results agree to rounding). */
typedef struct blfmm_tuning {
  int telescope;        /* 1: 3-D shared grids evaluate the leaf locals from the
                           root multipole (one leaf-level couple launch);
                           0: level-by-level couple + L2L sweep (mlfmm.cpp:268-340) */
  int graphs;           /* 1: replay the launch sequence as a CUDA graph */
  int near_sym_min;     /* symmetric near-field items for neighbouring leaves
                           that both hold >= this many points (0: off) */
  int near_ctas_per_sm; /* persistent near-field CTAs per SM (0: plan heuristic) */
  int near_reg_cap;     /* near-field register cap: 80, or 255 uncapped
                           (0: plan heuristic) */
  int couple_tile;      /* telescoped 3-D leaf couple: 0 per-parent 4^3 regions
                           (k_couple3<ROOT>), 1 z-streamed 2x2 column tiles
                           (k_couple_col); -1: plan default (1) */
  int rhs_gemm;         /* 3-D M = 16 with >= 8 right-hand sides: P2M / L2P as
                           real-weight DMMA GEMMs over all right-hand sides
                           (k_p2m_mr / k_l2p_mr); 0: one right-hand side per
                           CTA (k_p2m_m2m_h16 / k_l2p_h16S); -1: default (1) */
  int half_spectrum;    /* 3-D shared grids, even M in [16, 64]: store the
                           Hermitian half spectrum (0: the full grid);
                           -1: default (1) */
} blfmm_tuning;

/* Per-stage device times of the last execute (CUDA events on the launch
 * stream), enabled by blfmm_set_profiling. Order: tree/gather, p2m, m2m,
 * m2l(+l2l), l2p, near, combine. */
#define BLFMM_NSTAGES 7
typedef struct blfmm_stage_times {
  double ms[BLFMM_NSTAGES];
  int launches[BLFMM_NSTAGES];
} blfmm_stage_times;

const char* blfmm_last_error(void);
double blfmm_last_error_value(void); /* accuracy_error::achieved() */
int blfmm_abi_version(void);

/* parse_kernel_spec grammar: "name[:key=value]", case-insensitive. */
int blfmm_parse_kernel_spec(const char* spec, int* kernel_type, double* shape);

/* Host plan-time translation spectrum, K = M^d doubles in make_quadrature's
 * row-major node order. */
int blfmm_translation_coefficients(int d, int kernel_type, double shape,
                                   double sigma, int m_per_dim, double* c_out);

int blfmm_plan_create(const blfmm_plan_desc* desc, blfmm_plan** out);
void blfmm_tuning_defaults(blfmm_tuning* t);
int blfmm_plan_create_tuned(const blfmm_plan_desc* desc, const blfmm_tuning* tuning,
                            blfmm_plan** out);
int blfmm_plan_destroy(blfmm_plan* plan);
int blfmm_plan_get_info(const blfmm_plan* plan, blfmm_plan_info* info);

/* One matvec with HOST buffers: lambda [nrhs][n] (rhs-major, caller point
 * order), out [nrhs][n]. H2D / D2H copies are part of the call. stream may be
 * NULL (the plan's own stream). Synchronises before returning.
 * stats may be NULL: SumResult's stats (fmm.hpp:10-14) are then not produced,
 * and the max|Im| diagnostic of the far field (mlfmm.cpp:342-357) is not
 * evaluated (the half-spectrum L2P skips its imaginary-residual GEMM); out is
 * identical either way. The reference always fills them. */
int blfmm_execute(blfmm_plan* plan, const double* lambda, double* out,
                  blfmm_stats* stats, void* stream);

/* Same with DEVICE buffers (no copies, no host synchronisation; stats may be
 * NULL to skip max_imag_residual and its D2H read, as above). The work is ordered after
 * and before `stream` (NULL = the legacy default stream). */
int blfmm_execute_device(blfmm_plan* plan, const double* d_lambda,
                         double* d_out, blfmm_stats* stats, void* stream);

/* fmm_matvec_single semantics (single-level sum, which the shared-grid
 * multilevel sweep equals to rounding, mlfmm.hpp:17-20); stats.far_work uses
 * the single-level count. HOST buffers. */
int blfmm_execute_single(blfmm_plan* plan, const double* lambda, double* out,
                         blfmm_stats* stats, void* stream);

/* Stage expansions of one level, dense reference box-id order (row-major),
 * out[(box*K + node)*2 + {re,im}] for right-hand side `rhs`, zeros for empty
 * boxes. kind 0 = multipoles (upsweep), 1 = couple() locals before L2L (needs
 * blfmm_set_keep_couple(plan,1) before the execute), 2 = locals after L2L.
 * Reflects the last execute. */
int blfmm_get_expansions(blfmm_plan* plan, int level, int kind, int rhs,
                         double* out);
int blfmm_set_keep_couple(blfmm_plan* plan, int enable);

int blfmm_set_profiling(blfmm_plan* plan, int enable);
int blfmm_get_stage_times(const blfmm_plan* plan, blfmm_stage_times* t);

/* Morton-range sharding (multi-GPU). A plan created with world > 1 builds
 * the same tree on every rank, runs the full upsweep, and evaluates the
 * downsweep and near field only for its own contiguous range of leaves
 * (equal estimated cost). blfmm_execute writes the owned targets and zeros
 * elsewhere, so an all-reduce(sum) of the outputs of all ranks is u.
 * blfmm_partition is the host-side splitter (bounds[0..world]);
 * blfmm_plan_owned_points lists the owned targets' caller indices
 * (info.owned_end - info.owned_begin entries). */
int blfmm_partition(const double* cost, long long n, int world, long long* bounds);
int blfmm_plan_owned_points(const blfmm_plan* plan, long long* idx);

/* Exchange mode (world > 1, leaf level >= 3): the upsweep is partitioned too.
 * Each rank runs P2M on its leaves plus a two-leaf halo (complete multipoles
 * at levels L and L-1 where its downsweep reads them) and writes PARTIAL
 * coarse multipoles (own leaves only, disjoint across ranks) into a
 * caller-bound device buffer of blfmm_plan_exchange_size doubles: level 1
 * only when blfmm_plan_info.telescoped (3-D: the leaf locals need just the
 * root multipole; 0.3 MB for P3), levels 1..L-2 otherwise. The caller
 * all-reduces (sum) that buffer across ranks — the upper-level expansion
 * exchange over NCCL / NVLink — between the two halves:
 *   blfmm_execute_upsweep -> all-reduce(buffer) -> blfmm_execute_downsweep
 * and then all-reduces the outputs as above. */
int blfmm_plan_exchange_size(const blfmm_plan* plan, long long* n_doubles);
int blfmm_plan_bind_exchange(blfmm_plan* plan, double* d_buffer);
int blfmm_execute_upsweep(blfmm_plan* plan, const double* d_lambda, void* stream);
int blfmm_execute_downsweep(blfmm_plan* plan, double* d_out, blfmm_stats* stats,
                            void* stream);

/* Multi-GPU inside the library (SURVEY §8e, §8b "Multi-GPU is internal to
 * the plan"): attach a communicator to a world > 1 plan and blfmm_execute /
 * blfmm_execute_device run the whole sharded matvec - upsweep (exchange
 * mode) -> sum all-reduce of the upper-level expansion buffer -> downsweep
 * and near field of the owned leaves -> gather of the owned slices of u
 * (one broadcast per rank and right-hand side) -> u in the caller's order
 * on every rank. lambda is the full vector on every rank (the reference's
 * SumRequest::weights). Stats: max_imag_residual is max-reduced over ranks.
 *
 * NCCL: rank 0 calls blfmm_nccl_get_unique_id, the caller broadcasts the 128
 * bytes (any channel), every rank calls blfmm_plan_attach_nccl on its plan
 * (created with its rank / world / device). libnccl.so.2 is loaded on first
 * use (dlopen); failures return BLFMM_ENCCL. Collectives are enqueued on the
 * plan stream. A world = 1 plan accepts a one-rank communicator (same path,
 * trivial collectives).
 *
 * blfmm_comm_ops: the same orchestration over caller-supplied collectives
 * (MPI, a host transport, a test harness). Each callback receives a DEVICE
 * pointer and the stream the data is ordered on, and returns 0 on success;
 * it must leave the result in place before its stream work completes. */
#define BLFMM_NCCL_ID_BYTES 128
typedef struct blfmm_comm_ops {
  void* ctx;
  int (*all_reduce_sum)(void* ctx, double* d_buf, long long count, void* stream);
  int (*all_reduce_max)(void* ctx, double* d_buf, long long count, void* stream);
  int (*broadcast)(void* ctx, double* d_buf, long long count, int root, void* stream);
} blfmm_comm_ops;
int blfmm_nccl_get_unique_id(unsigned char id[BLFMM_NCCL_ID_BYTES]);
int blfmm_plan_attach_nccl(blfmm_plan* plan, const unsigned char id[BLFMM_NCCL_ID_BYTES]);
int blfmm_plan_attach_comm(blfmm_plan* plan, const blfmm_comm_ops* ops);

/* Krylov caller (solve_interpolation's iteration, solver.cpp:43-203, 269-300):
 * solves A x = b with A the plan's matvec (one right-hand side), CG
 * (BLFMM_SOLVE_CG, symmetric positive definite kernels) or GMRES restarted
 * every 300 iterations (BLFMM_SOLVE_GMRES), the reference's recurrences and
 * stopping rules; the vectors stay on the device, reductions are
 * deterministic. b / x are HOST arrays in the caller's point order. Not
 * reaching tol returns BLFMM_EACCURACY with the best relative residual in
 * blfmm_last_error_value (the reference's accuracy_error), stats filled. */
#define BLFMM_SOLVE_CG 1
#define BLFMM_SOLVE_GMRES 2
typedef struct blfmm_solve_stats {
  int method;       /* BLFMM_SOLVE_CG / BLFMM_SOLVE_GMRES */
  int iterations;
  int matvecs;
  int converged;
  double residual;  /* relative residual (best seen if not converged) */
} blfmm_solve_stats;
int blfmm_solve(blfmm_plan* plan, int method, const double* b, double* x, double tol,
                int max_iter, blfmm_solve_stats* stats);

/* solve_interpolation's Backend::dense (solver.cpp:207-262, 269-275): the same
 * Krylov loops on the dense kernel matrix A_ij = phi(|x_i - x_j|), applied
 * matrix-free on the device (the O(N^2) kernel of blfmm_direct) instead of
 * assembled with Eigen. coords: HOST [n][d]; every RadialKernel type. N > 8192
 * returns BLFMM_ELENGTH (assemble_dense's std::length_error). */
int blfmm_solve_dense(int d, long long n, const double* coords, int kernel_type, double shape,
                      int method, const double* b, double* x, double tol, int max_iter,
                      blfmm_solve_stats* stats, int device);

/* Independent O(N^2) check (direct_matvec, fmm.cpp:30-75): values for
 * n_targets target indices (NULL = all n) into HOST out. */
int blfmm_direct(int d, long long n, const double* coords, int kernel_type,
                 double shape, const double* lambda, long long n_targets,
                 const long long* targets, double* out, int device);

/* Band-limited oracles, d = 1 (fmm.cpp:57-70, 77-113): values of
 * sum_j lambda_j Phi_sigma(x_i - x_j) with Phi_sigma from the cubic-interpolated
 * radial table over [0, hi[0] - lo[0]] (the domain diameter), or, when
 * hybrid_leaf_level >= 2, the original kernel for sources in the target's
 * 3-leaf neighbourhood of build_tree(ps, hybrid_leaf_level) and Phi_sigma
 * elsewhere (hybrid_leaf_level = -1: the pure band-limited sum). All n
 * targets into HOST out. d != 1 -> BLFMM_EDOMAIN, as the reference. */
int blfmm_direct_bandlimited(int d, long long n, const double* coords, const double* lo,
                             const double* hi, int kernel_type, double shape,
                             const double* lambda, double sigma, int refinement,
                             int hybrid_leaf_level, double* out, int device);
/* Phi_sigma(x) in d = 1 (host, plan-time math; d = 2 -> BLFMM_EDOMAIN). */
int blfmm_eval_bandlimited(int d, int kernel_type, double shape, double sigma, double x,
                           int refinement, double* out);
/* BLFMM_RADIAL_TABLE_SIZE samples of Phi_sigma at step = rmax / 1024 (host,
 * cached per (kernel, clipped sigma, rmax, refinement) like the reference). */
#define BLFMM_RADIAL_TABLE_SIZE 1027
int blfmm_bandlimited_radial_table(int kernel_type, double shape, double sigma, double rmax,
                                   int refinement, double* vals, double* step);

#ifdef __cplusplus
}
#endif
#endif /* BLFMM_GPU_H */
