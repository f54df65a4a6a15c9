/*
 * mprec_gpu.h -- C ABI of the B200-native GMRES / CPR / CPTR3 solve path.
 *
 * Drop-in boundary for the reference `mprec` hot path.  Each
 * entry point names the reference interface it replaces.  Plain pointers and
 * sizes only; no C++ or torch types cross this boundary.  All `const double*`
 * / `double*` vector arguments are HOST pointers unless the name ends in
 * `_dev`.  Every function returns an mprec_status; on failure
 * mprec_gpu_last_error() / mprec_gpu_error_payload() give the message and the
 * cell/row payload (thread-local), mirroring the exception classes of
 * proj/include/mprec/errors.hpp:9-59.
 *
 * Threading: a handle's setup is not thread-safe; apply/solve calls on one
 * handle are serialised on the handle's CUDA stream; distinct handles are
 * independent (one handle per system, any number per process/GPU).
 */
#ifndef MPREC_GPU_H
#define MPREC_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: proj/include/mprec/errors.hpp:9-59 */
typedef enum mprec_status {
    MPREC_OK = 0,
    MPREC_DIMENSION = 1,      /* DimensionError                                   */
    MPREC_INDEX = 2,          /* IndexError                                       */
    MPREC_SINGULAR_BLOCK = 3, /* SingularBlockError{cell_id} (payload = cell / i) */
    MPREC_ZERO_PIVOT = 4,     /* ZeroPivotError{row_id}      (payload = row)      */
    MPREC_SETUP = 5,          /* SetupError                                       */
    MPREC_CONFIG = 6,         /* ConfigError                                      */
    MPREC_INTERNAL = 7,
    MPREC_CUDA = 8,           /* CUDA runtime failure (no GPU, OOM, ...)           */
    MPREC_IO = 9,             /* IoError (matrix_io.cpp, harness.cpp:153-188)      */
} mprec_status;

/* MethodSpec (proj/include/mprec/scaling.hpp:10-20); parse_method strings
 * "ilu0", "cpr-amg", "cpr-direct", "cptr3-amg", "cptr-direct", "cptr3-direct"
 * (scaling.cpp:5-15).  The -direct sub-solvers factor the sub-system densely
 * (DenseFactor, dense_factor.cpp) and are meant for small grids (<= 20000
 * sub-system rows). */
typedef enum mprec_method {
    MPREC_METHOD_ILU0 = 0,
    MPREC_METHOD_CPR_AMG = 1,
    MPREC_METHOD_CPR_DIRECT = 2,   /* dense LU of B_PP (small systems)           */
    MPREC_METHOD_CPTR3_AMG = 3,
    MPREC_METHOD_CPTR_DIRECT = 4,  /* dense LU of the 2n_c B_ee (scaling.cpp:90) */
    MPREC_METHOD_CPTR3_DIRECT = 5, /* dense LU of C_TT and B_PP                  */
} mprec_method;

/* AMGParams (proj/include/mprec/amg.hpp:12-16). */
typedef struct mprec_amg_params {
    double strength_threshold; /* 0.25 */
    int max_coarse_size;       /* 1000 */
    int max_levels;            /* 25   */
} mprec_amg_params;

/* ScalingOptions (proj/include/mprec/scaling.hpp:22-30): the square D factors
 * of the left scaling are the full per-cell block (BLOCK) or its scalar
 * diagonal (SCALAR, BlockMatrix::block_diagonal_of block_matrix.cpp:186-193);
 * CPTR3's second scaling divides by the diagonal of the post-step-1 B_PP
 * (default) or of the original A_PP (second_scaling_from_original = 1,
 * scaling.cpp:126). */
typedef enum mprec_diag_mode {
    MPREC_DIAG_BLOCK = 0,
    MPREC_DIAG_SCALAR = 1,
} mprec_diag_mode;

typedef struct mprec_scaling_options {
    int diag_mode;                    /* mprec_diag_mode, default BLOCK */
    int second_scaling_from_original; /* default 0 */
} mprec_scaling_options;

/* Uniform-layout BlockMatrix (proj/include/mprec/block_matrix.hpp:50-101):
 * n_cells block rows, nb unknowns per cell in (s..., P, T) order
 * (field_layout.hpp:62-66), block columns sorted ascending per row with the
 * diagonal block present (BlockMatrix::assemble, block_matrix.cpp:32-69),
 * values = nnzb column-major nb x nb blocks (Eigen's default storage).  The
 * caller keeps ownership; create copies to the device. */
typedef struct mprec_bsr {
    int n_cells;
    int nb;
    const int* row_ptr; /* n_cells + 1 */
    const int* col_idx; /* row_ptr[n_cells] */
    const double* values;
} mprec_bsr;

/* Scalar CSR (ScalarMatrix, scalar_matrix.hpp:20-62), canonical form. */
typedef struct mprec_csr {
    int n_rows;
    const int* row_ptr;
    const int* col_idx;
    const double* values;
} mprec_csr;

/* SolveResult (gmres.hpp:28-36) + SolveOutcome (harness.hpp:79-83). */
typedef struct mprec_solve_result {
    int iterations;             /* of the last attempt */
    int converged;
    int breakdown;
    int attempts;               /* tolerance-tightening attempts (harness.cpp:209) */
    int history_len;            /* entries written to `history` */
    double final_true_residual; /* ||b - A x|| / ||b|| on the ORIGINAL system */
    double setup_s;             /* left_scale + build_preconditioner */
    double solve_s;             /* all GMRES attempts */
    int total_iterations;       /* summed over all attempts */
    /* per tolerance-tightening attempt (harness.cpp:209-217), index < attempts */
    int attempt_iterations[3];
    int attempt_converged[3];        /* GMRES' own convergence flag */
    double attempt_tol[3];           /* the GMRES tolerance of the attempt */
    double attempt_true_residual[3]; /* residual_check on the original system */
} mprec_solve_result;

/* GlobalJacobian (condense.hpp:64-81) in plain arrays.  Primary blocks are
 * uniform np x np in the canonical (s..., P, T) order (FieldLayout::uniform);
 * cell c has sec_off[c+1]-sec_off[c] secondary unknowns.  All dense blocks
 * are column-major and packed in cell / entry order:
 *   j22: sum ns_c^2, j21: ns_c x np per cell, j12 entry e: np x ns_{col[e]},
 *   r1: n_cells*np, r2: sec_off[n_cells]. */
typedef struct mprec_global_jacobian {
    int n_cells, np;
    const int* row_ptr;  /* J11 block CSR (n_cells+1), sorted columns, diagonal present */
    const int* col_idx;
    const double* j11;
    const int* sec_off;  /* n_cells+1 */
    const double* j22;
    const double* j21;
    int n_j12;
    const int* j12_row;
    const int* j12_col;
    const double* j12;
    const double* r1;
    const double* r2;
} mprec_global_jacobian;

typedef struct mprec_gpu_system mprec_gpu_system; /* opaque */
typedef struct mprec_gpu_amg mprec_gpu_amg;       /* opaque */
typedef struct mprec_gpu_ilu mprec_gpu_ilu;       /* opaque */
typedef struct mprec_gpu_condensed mprec_gpu_condensed; /* opaque */

const char* mprec_gpu_last_error(void);
int mprec_gpu_error_payload(void);
/* sm / device sanity: returns MPREC_OK if a CUDA device is usable. */
int mprec_gpu_device_info(int* sm_count, int* cc_major, int* cc_minor, int64_t* mem_bytes);

/* ---- whole-system path --------------------------------------------------- */

/* Copies A to the device.  Replaces constructing the BlockMatrix the solve
 * path starts from (block_matrix.cpp:32-69); non-uniform layouts are not
 * representable here (MPREC_DIMENSION). */
int mprec_gpu_create(const mprec_bsr* a, mprec_gpu_system** out);

/* left_scale (scaling.cpp:149-158) + build_preconditioner (stages.cpp:129-138)
 * with ScalingOptions{Block, second_scaling_from_original=false}.  amg may be
 * NULL (defaults).  b: host rhs (n_cells*nb). */
int mprec_gpu_setup(mprec_gpu_system* h, int method, const mprec_amg_params* amg,
                    const double* b);

/* Same with explicit ScalingOptions (scaling.hpp:22-30, left_scale's 4th
 * argument, scaling.cpp:149-158); opts may be NULL (defaults). */
int mprec_gpu_setup_opts(mprec_gpu_system* h, int method, const mprec_amg_params* amg,
                         const mprec_scaling_options* opts, const double* b);

/* ScaledSystem::scaling_record joined with ", " as SolveOutcome::scaling_record
 * (harness.cpp:197-201), e.g. "[D_Ps;D_Ts]*D_ss^-1, D_Tp*D_PP^-1"; truncated
 * to cap-1 characters, always NUL-terminated. */
int mprec_gpu_scaling_record(mprec_gpu_system* h, char* buf, int cap);

/* StagePreconditioner::apply (stages.cpp:36-59) / apply_stage (stages.hpp:54). */
int mprec_gpu_apply(mprec_gpu_system* h, const double* r, double* z);
int mprec_gpu_apply_stage(mprec_gpu_system* h, int stage, const double* r, double* z);

/* y = A x (which=0: original A, BlockMatrix::apply block_matrix.cpp:103-114;
 * which=1: scaled Ā, the GMRES operator ScalarMatrix::apply on a_flat_). */
int mprec_gpu_spmv(mprec_gpu_system* h, int which, const double* x, double* y);

/* solve_system after setup (harness.cpp:198-218): GMRES on (Ā, b̄) with the
 * stage preconditioner, true residual on the original A, <=3 attempts with
 * tol <- tol*0.5*tol/true_resid.  x: host out (n).  history (optional, may be
 * NULL): relative preconditioned residuals of the last attempt. */
int mprec_gpu_solve(mprec_gpu_system* h, double tol, int max_iter, double* x,
                    mprec_solve_result* out, double* history, int history_cap);

/* Same as mprec_gpu_solve but leaves x on the device (x_dev may be NULL: the
 * handle keeps it); used to time the device-resident hot path. */
int mprec_gpu_solve_dev(mprec_gpu_system* h, double tol, int max_iter, double* x_dev,
                        mprec_solve_result* out);

/* Residual history (SolveResult::residual_history, gmres.hpp:31) of the last
 * solve on the handle's last attempt: up to history_cap entries into history
 * (may be NULL), the full length into *len. */
int mprec_gpu_last_history(mprec_gpu_system* h, double* history, int history_cap, int* len);

/* Whole solve_system (harness.cpp:190-219) from host buffers: create + setup
 * + solve + destroy. */
int mprec_gpu_solve_system(const mprec_bsr* a, const double* b, int method, double tol,
                           int max_iter, double* x, mprec_solve_result* out);

/* ingest_external (harness.cpp:153-188): Matrix Market "coordinate real
 * general" + layout sidecar + rhs (matrix_io.cpp:40-121) read and assembled
 * into a device BSR; every cell must carry P and T and (this path) the layout
 * must be uniform.  The rhs is kept by the handle: mprec_gpu_setup(h, m, amg,
 * NULL) uses it. */
int mprec_gpu_ingest(const char* matrix_path, const char* layout_path, const char* rhs_path,
                     mprec_gpu_system** out);
int mprec_gpu_get_shape(mprec_gpu_system* h, int* n_cells, int* nb, int* nnzb);
/* original A (BSR, column-major blocks) and the rhs the handle holds (either may be NULL) */
int mprec_gpu_get_matrix(mprec_gpu_system* h, int* row_ptr, int* col_idx, double* values, double* b);
/* write_block_matrix + write_vector (matrix_io.cpp:93-114), %.17g round-trip exact */
int mprec_gpu_write_system(mprec_gpu_system* h, const char* matrix_path, const char* layout_path,
                           const char* rhs_path);

/* ---- static condensation (condense.hpp:92-107, condense.cpp:206-258) ----
 * condense: per-cell partial-pivot LU of J22 (SingularBlockError(cell,
 * "secondary") when |u_ii| <= 1e-14 * max|J22_c|, first failing cell),
 * A = J11 - J12 J22^-1 J21 assembled like BlockMatrix::assemble (duplicate
 * blocks summed in entry order: J11 first, then the J12 list),
 * b = -r1 + J12 J22^-1 r2.  Everything stays on the device; the J22 factors
 * are kept for back_substitute. */
int mprec_gpu_condense(const mprec_global_jacobian* j, mprec_gpu_condensed** out);
int mprec_gpu_condensed_shape(mprec_gpu_condensed* h, int* n_cells, int* np, int* nnzb, int* n_secondary);
/* reduced system A (BSR, column-major blocks) and b (any may be NULL) */
int mprec_gpu_condensed_get(mprec_gpu_condensed* h, int* row_ptr, int* col_idx, double* values, double* b);
/* a solver handle on the reduced system (device to device); its rhs is b */
int mprec_gpu_condensed_system(mprec_gpu_condensed* h, mprec_gpu_system** out);
/* d2 = J22^-1 (-r2 - J21 d1) per cell (condense.cpp:243-258); host buffers */
int mprec_gpu_back_substitute(mprec_gpu_condensed* h, const double* d1, double* d2);
void mprec_gpu_condensed_destroy(mprec_gpu_condensed* h);

/* Parity diagnostics. */
int mprec_gpu_get_scaled(mprec_gpu_system* h, double* abar_values, double* b_bar);
int mprec_gpu_get_ilu(mprec_gpu_system* h, double* lu_values);
int mprec_gpu_n_stages(mprec_gpu_system* h, int* n_stages);
/* stage: index of an AMG stage (CPR: 0; CPTR3: 0 = C_TT, 1 = B_PP). */
int mprec_gpu_stage_amg(mprec_gpu_system* h, int stage, mprec_gpu_amg** amg);

/* Level sets of the block-row DAG the ILU(0) factorisation and solves are
 * scheduled on (ilu0.cpp:16-38, 48-57 on the block pattern):
 * dir = +1 forward (cell c waits for stored block columns < c), -1 backward;
 * same convention as mprec_gpu_amg_get_levelsets, one entry per cell. */
int mprec_gpu_get_levelsets(mprec_gpu_system* h, int dir, int* levels, int* n_levels);

/* Release (also releases the AMG handles returned by mprec_gpu_stage_amg;
 * a re-setup leaves earlier views stale: they then return MPREC_SETUP). */
void mprec_gpu_destroy(mprec_gpu_system* h);

/* ---- sub-solver entry points (amg.hpp:21-56, ilu0.hpp:9-24) -------------- */

/* AMGHierarchy::setup (amg.cpp:188-214) on a scalar CSR. */
int mprec_gpu_amg_create(const mprec_csr* a, const mprec_amg_params* p, mprec_gpu_amg** out);
/* AMGHierarchy::apply (amg.cpp:233-238): one V(1,1) cycle, zero initial guess. */
int mprec_gpu_amg_apply(mprec_gpu_amg* h, const double* r, double* x);
int mprec_gpu_amg_n_levels(mprec_gpu_amg* h, int* n_levels);
/* level sizes; nnz_p = 0 on level 0 (levels_[0].p unused, amg.hpp:47) */
int mprec_gpu_amg_level_info(mprec_gpu_amg* h, int level, int* n, int* nnz_a, int* nnz_p);
/* which: 0 = A_l, 1 = P_l (n_{l-1} x n_l), 2 = R_l = P_l^T */
int mprec_gpu_amg_get_csr(mprec_gpu_amg* h, int level, int which, int* row_ptr, int* col_idx,
                          double* values);
/* C/F splitting of level l (1 = C) that produced level l+1 (rs_coarsen). */
int mprec_gpu_amg_get_cf(mprec_gpu_amg* h, int level, signed char* cf);
/* Level sets of the symmetric Gauss-Seidel sweep DAG of level l (< n_levels-1):
 * dir = +1 forward sweep (row i waits for every stored k < i, amg.cpp:31-36),
 * dir = -1 backward sweep (k > i, amg.cpp:37-42).  levels[i] = 0 for a row
 * with no dependency, else 1 + max over its dependencies (the Kahn round the
 * device schedule processes it in); *n_levels = DAG depth.  levels may be NULL. */
int mprec_gpu_amg_get_levelsets(mprec_gpu_amg* h, int level, int dir, int* levels, int* n_levels);
void mprec_gpu_amg_destroy(mprec_gpu_amg* h);

/* ILU0Factor::factor / apply (ilu0.cpp:7-59) on a BSR (nb = 1: scalar ILU(0)). */
int mprec_gpu_ilu_create(const mprec_bsr* a, mprec_gpu_ilu** out);
int mprec_gpu_ilu_apply(mprec_gpu_ilu* h, const double* r, double* y);
int mprec_gpu_ilu_get(mprec_gpu_ilu* h, double* lu_values);
void mprec_gpu_ilu_destroy(mprec_gpu_ilu* h);

/* gmres (gmres.cpp:8-106) with A = BSR operator (flat order) and
 * preconditioner: prec_kind 0 = identity, 1 = AMG handle, 2 = ILU handle. */
int mprec_gpu_gmres(const mprec_bsr* a, const double* b, int prec_kind, void* prec,
                    double tol, int max_iter, double* x, mprec_solve_result* out,
                    double* history, int history_cap);

/* ---- measurement ---------------------------------------------------------- */

/* Kernel classes timed with CUDA events on the handle's stream when profiling
 * is on (mprec_gpu_profile). */
typedef enum mprec_kernel_class {
    MPREC_K_SPMV = 0,      /* BSR SpMV (GMRES operator, true residual)        */
    MPREC_K_SPMV_COL = 1,  /* scoped residual update z = r - Ā[:,f] x_f       */
    MPREC_K_ILU_FWD = 2,
    MPREC_K_ILU_BWD = 3,
    MPREC_K_GS = 4,        /* symmetric Gauss-Seidel sweeps (all levels)      */
    MPREC_K_CSR = 5,       /* level residual / restriction / prolongation     */
    MPREC_K_COARSE = 6,    /* coarsest dense solve                            */
    MPREC_K_MGS = 7,       /* Arnoldi MGS dot/axpy                            */
    MPREC_K_BLAS1 = 8,     /* scale/copy/norm/gather/scatter                  */
    MPREC_K_COUNT = 9
} mprec_kernel_class;

int mprec_gpu_profile(mprec_gpu_system* h, int enable);
/* The handle's CUDA stream (cudaStream_t) -- every kernel of the handle runs
 * on it, so callers can bracket work with their own CUDA events. */
int mprec_gpu_stream(mprec_gpu_system* h, void** stream);
/* accumulated since the last reset: total device ms, launches, algorithmic bytes */
int mprec_gpu_kernel_stats(mprec_gpu_system* h, int kclass, double* ms, int64_t* launches,
                           double* bytes);
int mprec_gpu_reset_stats(mprec_gpu_system* h);
/* number of kernel launches issued on the handle since the last reset */
int mprec_gpu_launch_count(mprec_gpu_system* h, int64_t* launches);

#ifdef __cplusplus
}
#endif

#endif /* MPREC_GPU_H */
