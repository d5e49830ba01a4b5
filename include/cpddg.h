/* cpddg -- B200-native (sm_100a, FP64) solve path for the closest-point
 * surface Helmholtz discretisation with RAS / ORAS Schwarz methods.
 *
 * The C ABI that a reference ("cpdd", proj/include/cpdd/) caller binds to in
 * place of its own hot path.  Plain pointers and sizes only; no exceptions
 * cross it.  Every entry point cites the reference interface it replaces.
 *
 * Status codes map 1:1 to the reference exception hierarchy
 * (proj/include/cpdd/core.hpp:73-95) and thus to the CLI exit codes of
 * proj/tools/cpm.cpp:181-193:
 *   0 ok, 1 InternalError, 2 ConfigError, 3 DivergenceError (singular local
 *   factorisation, non-finite residual, divergence), 4 IoError, 5 CUDA error.
 * cpddg_last_error() returns the message of the calling thread's last failure.
 *
 * Memory: arguments named *_dev are device pointers (FP64, length n);
 * `stream` is a cudaStream_t (NULL = legacy default stream).  Handles own
 * their device buffers and are released by the matching *_destroy.  Calls on
 * one handle must be serialised by the caller (the reference's const apply()
 * is likewise not re-entrant across pools, proj/include/cpdd/solve.hpp:62-86).
 */
#ifndef CPDDG_H
#define CPDDG_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define CPDDG_API __attribute__((visibility("default")))
#else
#define CPDDG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum {
    CPDDG_OK = 0,
    CPDDG_ERR_INTERNAL = 1,
    CPDDG_ERR_CONFIG = 2,
    CPDDG_ERR_DIVERGENCE = 3,
    CPDDG_ERR_IO = 4,
    CPDDG_ERR_CUDA = 5
};

/** Copy the calling thread's last error message into buf; returns its code. */
CPDDG_API int cpddg_last_error(char* buf, size_t len);
CPDDG_API const char* cpddg_version(void);

/* ======================================================================
 * Host setup.  Mirrors build_problem (proj/include/cpdd/pipeline.hpp:155-168)
 * and the setup half of run_solve (pipeline.hpp:186-216): band, E, A,
 * partition alignment, subdomains, local systems.  Bit-exact with the
 * reference (index sets, orderings, and the bits of every matrix entry).
 * ==================================================================== */
typedef struct cpddg_setup cpddg_setup;

enum { CPDDG_CIRCLE = 0, CPDDG_SPHERE = 1, CPDDG_TORUS = 2, CPDDG_TRIMESH = 3 };

typedef struct {
    int dim;              /* 2 (circle) or 3 */
    int surface;          /* CPDDG_CIRCLE ... CPDDG_TRIMESH (RunConfig::surface, config.hpp:21) */
    double radius;        /* circle / sphere (config.hpp:22) */
    double major_radius;  /* torus (config.hpp:25-26) */
    double minor_radius;
    const char* obj_path; /* trimesh: Wavefront OBJ (geometry.hpp:137-170) */
    double h;             /* lattice spacing (config.hpp:32) */
    int p;                /* interpolation degree (config.hpp:33) */
    double tube_radius;   /* <= 0: reference (p+1)/2 sqrt(d) h (interp.hpp:95-98) */
    double c;             /* Helmholtz shift (SolverConfig::c, solve.hpp:31) */
    int workers;          /* host threads for setup; 0 = all */
    int device_setup;     /* 1: band + closest points (cpddg_setup_create) and alignment + subdomain
                             sets (cpddg_setup_decompose) built on the current CUDA device,
                             bit-identical to the host setup; 0: host */
} cpddg_problem_desc;

/** build_band_tube + build_extension + assemble_helmholtz
 *  (band.hpp:150-182, operators.hpp:30-51, 96-112). */
CPDDG_API int cpddg_setup_create(const cpddg_problem_desc* desc, cpddg_setup** out);
CPDDG_API int cpddg_setup_destroy(cpddg_setup* s);
/** n_active, n_ghost, nnz(E), nnz(A). */
CPDDG_API int cpddg_setup_sizes(const cpddg_setup* s, int* n_active, int* n_ghost, int64_t* nnz_E,
                      int64_t* nnz_A);
/** Band nodes in band-code order (BandGrid::active then ::ghost,
 *  band.hpp:36-60): lattice index (N_B x dim), cp, normal (N_B x dim), dist. */
CPDDG_API int cpddg_setup_band(const cpddg_setup* s, int32_t* ix, double* cp, double* normal, double* dist);
/** CSR of E (which = 0) or A (which = 1) (SparseOperator, sparse.hpp:19-103). */
CPDDG_API int cpddg_setup_csr(const cpddg_setup* s, int which, int64_t* row_ptr, int32_t* col, double* val);

enum { CPDDG_RAS = 0, CPDDG_ORAS = 1 };

/** Partition (validated as load_partition, partition.hpp:519-552), then
 *  align_interfaces (partition.hpp:474-508), build_subdomains
 *  (subdomain.hpp:153-313) and assemble_local for every subdomain
 *  (transmission.hpp:73-138, factor = false).  n_part must equal n_active
 *  (ConfigError otherwise, as load_partition).  alpha_cross < 0 means alpha
 *  (SolverConfig::effective_alpha_cross, solve.hpp:38).  part_out (may be
 *  NULL) receives the aligned labels, moves the alignment move count. */
CPDDG_API int cpddg_setup_decompose(cpddg_setup* s, const int32_t* part, int n_part, int n_overlap, int method,
                          double alpha, double alpha_cross, int32_t* part_out, int* moves);
CPDDG_API int cpddg_setup_n_subdomains(const cpddg_setup* s);
/** Phase seconds t[6] = band, E, A (cpddg_setup_create), alignment,
 *  subdomain sets, local systems (cpddg_setup_decompose). */
CPDDG_API int cpddg_setup_timings(const cpddg_setup* s, double* t);
/** counts[8] = |disjoint|, |overlap|, |final_layer|, |ghosts|, |bc|,
 *  fallback_count, n_lambda, #cross_flagged (Subdomain, subdomain.hpp:47-56). */
CPDDG_API int cpddg_setup_subdomain_counts(const cpddg_setup* s, int j, int32_t* counts);
/** bc_int: |bc| x (dim+4) = ix..., global_active, is_ghost_type,
 *  cross_flagged, fallback; bc_real: |bc| x (4 dim + 1) = x, cp, cp_local,
 *  conormal, dq (BoundaryNode, subdomain.hpp:30-44). */
CPDDG_API int cpddg_setup_subdomain_sets(const cpddg_setup* s, int j, int32_t* disjoint, int32_t* overlap,
                               int32_t* final_layer, int32_t* ghosts, int32_t* bc_int,
                               double* bc_real);
/** sizes[4] = n_overlap, n_bc, nnz, |scatter| (LocalOperator,
 *  transmission.hpp:47-70). */
CPDDG_API int cpddg_setup_local_sizes(const cpddg_setup* s, int j, int64_t* sizes);
CPDDG_API int cpddg_setup_local(const cpddg_setup* s, int j, int64_t* row_ptr, int32_t* col, double* val,
                      int32_t* scatter_local, int32_t* scatter_global);

/* ======================================================================
 * Device operator.  Replaces Eigen::VectorXd SparseOperator::apply(x) on the
 * assembled Helmholtz matrix A (sparse.hpp:65-75, A from operators.hpp:96-112)
 * with the matrix-free form y = (c + 2d/h^2) x - h^-2 sum_{2d nbrs} (E x).
 * ==================================================================== */
typedef struct cpddg_op cpddg_op;

typedef struct {
    int dim, p;
    int n_active, n_ghost;
    double h, c;
    const int32_t* ix; /* (n_active + n_ghost) x dim lattice indices, band-code order */
    const double* cp;  /* (n_active + n_ghost) x dim closest points */
} cpddg_band_desc;

CPDDG_API int cpddg_op_create(const cpddg_band_desc* band, cpddg_op** out);
CPDDG_API int cpddg_op_create_from_setup(const cpddg_setup* s, cpddg_op** out);
/** y_dev = A x_dev (sizes n_active). */
CPDDG_API int cpddg_op_apply(cpddg_op* op, const double* x_dev, double* y_dev, void* stream);
/** r_dev = b_dev - A x_dev, and ||r||_2 into *rnorm (host, synchronises). */
CPDDG_API int cpddg_op_residual(cpddg_op* op, const double* b_dev, const double* x_dev, double* r_dev,
                      double* rnorm, void* stream);
CPDDG_API int cpddg_op_size(const cpddg_op* op);
/** Bytes one apply must move at minimum (SURVEY.md 8(d) B_op) and the bytes
 *  the kernels stream (index tables included). */
CPDDG_API int cpddg_op_bytes(const cpddg_op* op, int64_t* algorithmic, int64_t* streamed);
CPDDG_API int cpddg_op_destroy(cpddg_op* op);

/* ======================================================================
 * Device Schwarz preconditioner.  Replaces the factored LocalOperator
 * vector (assemble_local(..., factor = true), transmission.hpp:73-138;
 * DirectSolver::factor, direct.hpp:41-52) and
 * SchwarzPreconditioner::apply (solve.hpp:64-86): z = sum_j Rt_j^T A_j^-1 R_j r.
 * ==================================================================== */
typedef struct cpddg_pc cpddg_pc;

typedef struct {
    int n_overlap, n_bc;
    const int32_t* overlap;        /* n_overlap global ordinals (LocalOperator::overlap) */
    int n_scatter;
    const int32_t* scatter_local;  /* LocalOperator::scatter .first  */
    const int32_t* scatter_global; /* LocalOperator::scatter .second */
    const int64_t* row_ptr;        /* n_local + 1 (SparseOperator::row_ptr) */
    const int32_t* col;
    const double* val;
} cpddg_local_desc;

typedef struct {
    int workers;        /* host threads for ordering / symbolic analysis; 0 = all */
    int check_residual; /* 1: verify every local factor on a probe vector */
} cpddg_pc_options;

typedef struct {
    int n_sub;
    int n_reduced;              /* subdomains whose Dirichlet closure block was eliminated */
    int64_t n_rows_total;       /* sum of factored system sizes */
    int64_t factor_entries;     /* stored L + U + diag entries */
    int64_t profile_entries;    /* envelope entries: sum_i (i - fL_i) + sum_c (c - fU_c) + n (nonsymmetric envelopes) */
    int64_t factor_bytes;       /* bytes the apply streams (factors, or the dense inverses in apply_mode 1) */
    int64_t algorithmic_bytes;  /* B_pc of SURVEY.md 8(d) */
    int max_rows;
    double factor_seconds;      /* device factorisation time */
    double analyse_seconds;     /* host ordering + symbolic time */
    double max_probe_residual;  /* when check_residual */
    int apply_mode;             /* 0: register-staged record / envelope solves (k_solve); 1: dense local inverses
                                   (small systems); 2: persistent TMA-streamed record solve (k_solve_tma);
                                   3: windowed TMA-streamed record solve (k_solve_win, the default);
                                   4: k_solve_win with the local vector in HBM (windows beyond shared memory) */
    int n_pivoted;              /* local systems factored with partial pivoting (host band LU fallback) */
    int win_cuts;               /* k_solve_win: subdomains cut across two SMs by the balanced schedule (0: LPT lists) */
    double win_lpt_efficiency;  /* modelled work / (SMs x longest list), whole subdomains per SM (LPT) */
    double win_bal_efficiency;  /* the same for the balanced (cut) schedule */
    int64_t n_dropped;          /* local unknowns no other row refers to and no scatter returns (ORAS ring /
                                   ghost-type closure rows, transmission.hpp:84-92), removed before the factorisation */
} cpddg_pc_stats;

CPDDG_API int cpddg_pc_create(int n_global, int n_sub, const cpddg_local_desc* locals,
                    const cpddg_pc_options* opt, cpddg_pc** out);
CPDDG_API int cpddg_pc_create_from_setup(const cpddg_setup* s, const cpddg_pc_options* opt, cpddg_pc** out);
/** Host only (no device call): dropped[q] = 1 for the local unknowns cpddg_pc_create removes before
 *  the factorisation -- closure unknowns that no row but their own refers to and that no scatter
 *  returns (transmission.hpp:84-92, :66-69), to the fixed point; dropped has n_overlap + n_bc
 *  entries.  The remaining unknowns' solution is unchanged. */
CPDDG_API int cpddg_local_unreferenced(const cpddg_local_desc* d, unsigned char* dropped, int* n_dropped);
/** z_dev = M r_dev (sizes n_global). */
CPDDG_API int cpddg_pc_apply(cpddg_pc* pc, const double* r_dev, double* z_dev, void* stream);
CPDDG_API int cpddg_pc_stats_get(const cpddg_pc* pc, cpddg_pc_stats* st);
CPDDG_API int cpddg_pc_destroy(cpddg_pc* pc);

/* ======================================================================
 * Solvers.  Replace stationary_solve and gmres_solve (solve.hpp:95-214);
 * the log mirrors IterationLog (solve.hpp:49-55): residuals start with the
 * initial residual, iterations = preconditioner applications counted as
 * the reference counts them, final_true_residual = ||b - A u|| at exit.
 * ==================================================================== */
typedef struct {
    double rel_tol;
    int max_iter;
    int restart;         /* gmres: 0 = no restart (cycle = max_iter) */
    int profile_kernels; /* 1: time every preconditioner / operator launch with CUDA events */
} cpddg_solve_params;

typedef struct {
    double* residuals;   /* caller buffer of `capacity` entries (may be NULL) */
    int capacity;
    int n_residuals;     /* entries produced (may exceed capacity) */
    int iterations;
    int converged;
    double final_true_residual;
    double seconds;      /* device-timed solve loop (CUDA events) */
    int64_t kernel_launches;
    /* filled when profile_kernels: summed device time and count of the
     * preconditioner applies (k_solve) and operator applies (k_extend + k_helm) */
    double pc_seconds;
    int64_t pc_launches;
    double op_seconds;
    int64_t op_launches;
} cpddg_log;

CPDDG_API int cpddg_gmres(cpddg_op* op, cpddg_pc* pc, const double* b_dev, double* u_dev,
                const cpddg_solve_params* prm, cpddg_log* log, void* stream);
CPDDG_API int cpddg_stationary(cpddg_op* op, cpddg_pc* pc, const double* b_dev, double* u_dev,
                     const cpddg_solve_params* prm, cpddg_log* log, void* stream);

/* ----------------------------------------------------------------------
 * Development / profiling entry points (not part of the reference boundary).
 * -------------------------------------------------------------------- */
/** One preconditioner pass: mode 0 full apply, 1 forward substitution only,
 *  2 backward only, 3 factor probe (r, z per-row arrays in factor order). */
CPDDG_API int cpddg_pc_apply_mode(cpddg_pc* pc, const double* r_dev, double* z_dev, int mode, void* stream);
/** Per-block timing trace of CTA 0 from the last solve run with
 *  CPDDG_SOLVE_DEBUG & 16 (1024 x 20 clock64 values). */
CPDDG_API int cpddg_dev_trace(long long* out);
/** Exact zeros among the stored factor entries: out[6] = L entries, L zeros,
 *  all-zero 16-entry L segments, U entries, U zeros, U zero segments. */
CPDDG_API int cpddg_pc_debug_zero_stats(const cpddg_pc* pc, int64_t* out);

#ifdef __cplusplus
}
#endif

#endif /* CPDDG_H */
