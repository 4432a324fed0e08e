/*
 * epicorr_b200.h — C ABI of the B200-native epicorr hot path.
 *
 * This is the drop-in boundary: every entry point replaces one reference
 * C++ solver entry point of `epicorr` (paths below are relative to the
 * reference tree, proj/...). Plain C types only: pointers, sizes, POD
 * structs. No exceptions cross the ABI: every call returns an EPC_* status
 * and, on failure, the message the reference would have thrown (its
 * `e.what()` text) is available from epc_last_error().
 *
 * Memory: functions taking `int mem` accept EPC_MEM_HOST (pageable or pinned
 * host buffers; the call copies in and out on the context stream and
 * synchronises) or EPC_MEM_DEVICE (pointers into the context device's HBM;
 * the call still synchronises before returning so row/scalar outputs are
 * valid). Layouts are the reference's (proj/include/epicorr/grid.hpp:1-6,
 * 39-44): axis 1 fastest; faces `i + n1*(j + m2*k)` with n1 = m1 + 1;
 * cells `i + m1*(j + m2*k)`; a column (j,k) is contiguous.
 */
#ifndef EPICORR_B200_H
#define EPICORR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (map onto the reference's exception types) ---------- */
enum {
    EPC_OK = 0,
    EPC_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    EPC_ERR_RUNTIME = 2,          /* std::runtime_error    */
    EPC_ERR_DOMAIN = 3,           /* std::domain_error     */
    EPC_ERR_CUDA = 4,             /* CUDA runtime failure (no reference analogue) */
    EPC_ERR_UNSUPPORTED = 5       /* path out of scope of this build (e.g. SGS) */
};

enum { EPC_MEM_HOST = 0, EPC_MEM_DEVICE = 1 };

/* proj/include/epicorr/report.hpp:12 */
enum { EPC_STOP_CONVERGED = 0, EPC_STOP_MAX_ITERATIONS = 1, EPC_STOP_LINE_SEARCH_FAILURE = 2,
       EPC_STOP_ERROR = 3 };
/* proj/include/epicorr/admm.hpp:31 */
enum { EPC_RHO_FIXED = 0, EPC_RHO_ADAPTIVE = 1, EPC_RHO_ADAPTIVE_BOUNDED = 2 };
/* proj/include/epicorr/gn_pcg.hpp:21 */
enum { EPC_PRECOND_NONE = 0, EPC_PRECOND_JACOBI = 1, EPC_PRECOND_BLOCK_JACOBI = 2,
       EPC_PRECOND_SGS = 3 };

/* GridSpec, proj/include/epicorr/grid.hpp:16-52 */
typedef struct epc_grid {
    int dim;          /* 2 or 3 */
    int m[3];         /* cells per axis; m[2] == 1 in 2D */
    double h[3];      /* spacings */
    double origin[3];
} epc_grid;

/* ObjectiveParams, proj/include/epicorr/objective.hpp:25-34 */
typedef struct epc_objective_params {
    double alpha; /* 50   */
    double beta;  /* 10   */
    double gamma; /* 1e-3 */
    int enforce_linf_box;
} epc_objective_params;

/* ADMMConfig, proj/include/epicorr/admm.hpp:36-50 */
typedef struct epc_admm_config {
    double rho0, rho_min;
    int schedule;
    double eps_abs, eps_rel;
    int max_iter;
    double tau_incr, tau_decr, mu;
    int sqp_max_iter;
    double sqp_tol_rel;
    int check_kkt;
    int threads; /* accepted for API parity; the device path ignores it */
} epc_admm_config;

/* GNConfig, proj/include/epicorr/gn_pcg.hpp:26-40 */
typedef struct epc_gn_config {
    double eta;
    int max_outer;
    double eps_obj, eps_iter, eps_grad;
    double wolfe_c1, wolfe_c2;
    int max_pcg, max_ls;
    int precond;
    int threads;
} epc_gn_config;

/* AdmmIterRow, proj/include/epicorr/report.hpp:28-40 */
typedef struct epc_admm_row {
    int level, iter;
    double primal_res, dual_res, eps_pri, eps_dual, rho, lagrangian, kkt_violation;
    double b_update_s, wall_s;
} epc_admm_row;

/* GnIterRow, proj/include/epicorr/report.hpp:16-26 */
typedef struct epc_gn_row {
    int level, iter;
    double j_value, grad_norm, step;
    int pcg_iters;
    double pcg_relres, pcg_relres_prec, wall_s;
} epc_gn_row;

/* BUpdateStats, proj/include/epicorr/admm.hpp:91-95 */
typedef struct epc_bupdate_stats {
    long sqp_iters, qp_iters;
    double kkt_violation;
    int max_active; /* largest active set met in any column QP (diagnostic) */
} epc_bupdate_stats;

/* Result of one solve: stop reason + message, SolveReport
 * (proj/include/epicorr/report.hpp:42-51). Rows go to caller arrays. */
typedef struct epc_solve_status {
    int stop;
    int nrows;
    char message[256];
} epc_solve_status;

/* Objective values, ObjectiveEval (proj/include/epicorr/objective.hpp:84-90) */
typedef struct epc_objective_eval {
    double value, dist, smooth, pen;
    int feasible;
} epc_objective_eval;

/* PcgResult scalars (proj/include/epicorr/gn_pcg.hpp:49-55) */
typedef struct epc_pcg_result {
    int iters;
    double relres, relres_prec;
    int reached_tol;
} epc_pcg_result;

/* DualUpdate scalars (proj/include/epicorr/admm.hpp:107-111) */
typedef struct epc_dual_result {
    double primal_res, dual_res, eps_pri, eps_dual;
} epc_dual_result;

typedef struct epc_context epc_context;

/* ---- defaults matching the reference's default member initialisers ----- */
void epc_default_params(epc_objective_params* p);     /* objective.hpp:26-31 */
void epc_default_admm_config(epc_admm_config* c);     /* admm.hpp:37-47 */
void epc_default_gn_config(epc_gn_config* c);         /* gn_pcg.hpp:27-37 */

/* ---- context ------------------------------------------------------------
 * One context per device; all work goes to `stream` (a cudaStream_t; NULL
 * means a stream owned by the context). Not thread-safe per context. */
int epc_context_create(int device, void* stream, epc_context** out);
void epc_context_destroy(epc_context* ctx);
int epc_set_stream(epc_context* ctx, void* stream);
const char* epc_last_error(const epc_context* ctx);
/* Bitmask of optional modes, EPC_MODE_*; default 0 (reference-exact). */
enum {
    EPC_MODE_BSTEP_TIMING = 1, /* accumulate b-step phase cycles and counters (diagnostic) */
    /* decide every b-step SQP / line-search test on the reference's sequential
     * sums instead of certified enclosures (diagnostic; identical results) */
    EPC_MODE_BSTEP_CHAINED = 1 << 13,
    /* take every ADMM stop / rho decision on the reference's sequential sums
     * (k_seq_sums) instead of certifying it from the tree sums (diagnostic;
     * identical decisions, and the rows' residuals become bitwise the
     * reference's) */
    EPC_MODE_EXACT_SUMS = 1 << 14,
    /* take the ADMM stop / rho decisions on the device (k_admm_decide) and
     * keep one iteration in flight instead of reading every iteration's sums
     * back before enqueueing the next (identical results; measured no faster
     * at C1-C3, where the round trip is < 0.3% of an iteration) */
    EPC_MODE_DEVICE_LOOP = 1 << 15
};
int epc_set_mode(epc_context* ctx, int mode_bits);
/* Cumulative ADMM counters of the context (epc_admm_solve / _batch):
 * out4[0] stop/rho decisions taken on certified enclosures of the
 * reference's sequential sums, out4[1] decisions taken on the exact
 * sequential sums (undecidable enclosure, or EPC_MODE_EXACT_SUMS),
 * out4[2] b-step SQP iterations, out4[3] QP iterations (BUpdateStats sums). */
int epc_admm_counters(epc_context* ctx, long long* out4);
/* Guard mode (dev aid; EPC_GUARD=1 in the environment when the context is
 * created): every device scratch slot carries 4 KB guard zones; this checks
 * them all and returns the first overwritten slot in *bad_slot (-1: none). */
int epc_guard_check(epc_context* ctx, int* bad_slot);
/* Phase cycle totals of the b-step kernel since timing was enabled (lane 0
 * clock64 deltas): model, fval sums, factor, solves, QP rest, KKT, step
 * sums, line search, clamp+store, column fetch. */
int epc_bstep_timing(epc_context* ctx, long long* out10);
/* b-step event counters since timing was enabled: line-search trials,
 * trials an enclosure could not decide, undecided stopping tests, failed
 * line searches, SQP iterations reaching the line search, exact fval
 * fallbacks, then a histogram of the accepted trial index (0, 1, 2-3, 4-7,
 * 8-15, 16-31, 32-39), the failed-search count, and the Schur solves
 * (count, sum na, sum na^2, sum na^3). */
int epc_bstep_counters(epc_context* ctx, long long* out18);
/* Per-kernel CUDA-event timing on the context stream (for the roofline). */
int epc_profile_enable(epc_context* ctx, int on);
/* Fills up to `cap` entries: name (static string), total ms, launch count. */
int epc_profile_read(epc_context* ctx, const char** names, double* total_ms, long* launches,
                     int cap, int* count);
void epc_profile_reset(epc_context* ctx);
/* Kernel launches issued on this context since creation / last reset. */
long epc_launch_count(const epc_context* ctx);
void epc_reset_launch_count(epc_context* ctx);

/* ---- ADMM (proj/src/admm.cpp) ------------------------------------------- */

/* admm_solve, proj/include/epicorr/admm.hpp:127-129, proj/src/admm.cpp:488-560.
 * b, z, u: in = initial state (NULL = zero start, like an empty StaggeredField),
 * out = final state (must be non-NULL to receive it). *rho: in = init.rho
 * (<= 0 selects cfg->rho0), out = final rho. rows: capacity max_rows.
 * Errors thrown by the reference before the loop (validate, infeasible start)
 * return EPC_ERR_INVALID_ARGUMENT; in-loop errors give stop = EPC_STOP_ERROR
 * with the reference's message and return EPC_OK, as the reference does. */
int epc_admm_solve(epc_context* ctx, const epc_grid* g, int mem, const double* iplus,
                   const double* iminus, const double* b_in, const double* z_in,
                   const double* u_in, double* b_out, double* z_out, double* u_out,
                   double* rho, const epc_objective_params* p, const epc_admm_config* cfg,
                   int level_tag, epc_admm_row* rows, int max_rows, epc_solve_status* status);

/* Batched admm_solve over `npairs` independent volume pairs sharing one grid
 * (C4 config). Arrays are pair-major (pair p at offset p*cells / p*faces);
 * rho[npairs], rows[npairs*max_rows], status[npairs]. Each pair keeps its
 * own rho schedule and stop test; results equal npairs separate calls. */
int epc_admm_solve_batch(epc_context* ctx, const epc_grid* g, int npairs, int mem,
                         const double* iplus, const double* iminus, const double* b_in,
                         const double* z_in, const double* u_in, double* b_out,
                         double* z_out, double* u_out, double* rho,
                         const epc_objective_params* p, const epc_admm_config* cfg,
                         int level_tag, epc_admm_row* rows, int max_rows,
                         epc_solve_status* status);

/* b_update, admm.hpp:100-102, admm.cpp:301-443 (with residual_column,
 * qp_active_set, verify_qp_kkt, clamp_column_diffs). stats may be NULL. */
int epc_b_update(epc_context* ctx, const epc_grid* g, int mem, const double* iplus,
                 const double* iminus, const double* b, const double* z, const double* u,
                 double rho, const epc_objective_params* p, const epc_admm_config* cfg,
                 double* b_out, epc_bupdate_stats* stats);

/* z_update, admm.hpp:105, admm.cpp:445-451 (DctCoupledSolver::solve,
 * operators.cpp:388-418). */
int epc_z_update(epc_context* ctx, const epc_grid* g, int mem, const double* b, const double* u,
                 double rho, double alpha, double* z_out);

/* DctCoupledSolver::solve on an arbitrary right-hand side, operators.hpp:99. */
int epc_dct_solve(epc_context* ctx, const epc_grid* g, int mem, const double* rhs, double alpha,
                  double rho, double* out);

/* dual_update_and_residuals, admm.hpp:113-115, admm.cpp:453-476. */
int epc_dual_update(epc_context* ctx, const epc_grid* g, int mem, const double* b_new,
                    const double* z_new, const double* z_old, const double* u_old, double rho,
                    double eps_abs, double eps_rel, double* u_out, epc_dual_result* out);

/* augmented_lagrangian, admm.hpp:87-89, admm.cpp:287-299. */
int epc_augmented_lagrangian(epc_context* ctx, const epc_grid* g, int mem, const double* iplus,
                             const double* iminus, const double* b, const double* z,
                             const double* u, double rho, double alpha, double* out);

/* rho_schedule, admm.hpp:119-120, admm.cpp:478-486 (host scalar logic). */
double epc_rho_schedule(int schedule, double rho, double rho_min, double primal_res,
                        double dual_res, double tau_incr, double tau_decr, double mu);

/* qp_active_set + verify_qp_kkt over `nqp` independent column QPs of size n
 * (admm.hpp:74-81, admm.cpp:114-265), host memory, QP-major arrays of n
 * (gd, go, c, x0, x) and n-1 (lambda, active_sign) per QP. status[q] is an
 * EPC_* code; its message for the lowest failing QP is in epc_last_error.
 * kkt[q] = verify_qp_kkt of the result (may be NULL). */
int epc_qp_active_set_batch(epc_context* ctx, int nqp, int n, double h, const double* gd,
                            const double* go, const double* c, const double* x0, int max_iter,
                            double* x, double* lambda, int* active_sign, int* iters,
                            double* kkt, int* status);

/* ---- GN-PCG (proj/src/gn_pcg.cpp, proj/src/objective.cpp) ---------------- */

/* gauss_newton_solve, gn_pcg.hpp:81-83, gn_pcg.cpp:197-292. */
int epc_gn_solve(epc_context* ctx, const epc_grid* g, int mem, const double* iplus,
                 const double* iminus, const double* b0, double* b_out,
                 const epc_objective_params* p, const epc_gn_config* cfg, int level_tag,
                 epc_gn_row* rows, int max_rows, epc_solve_status* status);

/* objective_gn, objective.hpp:93-94, objective.cpp:231-264. grad (faces) is
 * written only when need_grad and the point is feasible; residual (cells)
 * may be NULL. */
int epc_objective_gn(epc_context* ctx, const epc_grid* g, int mem, const double* iplus,
                     const double* iminus, const double* b, const epc_objective_params* p,
                     int need_grad, epc_objective_eval* out, double* grad, double* residual);

/* GnHessian ctor + column_part + preconditioner_blocks (objective.cpp:266-348).
 * diag/off: column part; pdiag: preconditioner_blocks().diag (any may be NULL). */
int epc_gn_hessian_build(epc_context* ctx, const epc_grid* g, int mem, const double* iplus,
                         const double* iminus, const double* b, const epc_objective_params* p,
                         double* diag, double* off, double* pdiag);

/* GnHessian::apply at linearisation point b, objective.cpp:302-331. */
int epc_gn_hessian_apply(epc_context* ctx, const epc_grid* g, int mem, const double* iplus,
                         const double* iminus, const double* b, const epc_objective_params* p,
                         const double* x, double* y);

/* make_preconditioner(kind) applied to r at linearisation point b,
 * gn_pcg.cpp:37-90 (none / jacobi / block_jacobi; sgs -> EPC_ERR_UNSUPPORTED). */
int epc_precond_apply(epc_context* ctx, const epc_grid* g, int mem, const double* iplus,
                      const double* iminus, const double* b, const epc_objective_params* p,
                      int kind, const double* r, double* z);

/* pcg(H(b), M_kind, grad, eta, max_iters), gn_pcg.cpp:92-131. */
int epc_pcg(epc_context* ctx, const epc_grid* g, int mem, const double* iplus,
            const double* iminus, const double* b, const epc_objective_params* p, int kind,
            const double* grad, double eta, int max_iters, double* d, epc_pcg_result* out);

/* The GN operators from a GnHessian's parts (the shim's GnHessian and
 * make_preconditioner, objective.hpp:99-131, gn_pcg.hpp:47):
 * GnHessian::apply (objective.cpp:302-331), y = T x + w2 (2x - x_{j+-1})
 *   + w3 (2x - x_{k+-1}) with Neumann ends, from the column part diag/off;
 * preconditioner_blocks().diag == full_diagonal() (objective.cpp:333-348),
 *   out = diag + cross_diag(j, k);
 * the Jacobi apply z = r / diag (gn_pcg.cpp:41-47) over n entries. The
 * block-Jacobi apply is epc_tridiag_solve_batched on the preconditioner
 * blocks. */
int epc_gn_stencil_apply(epc_context* ctx, const epc_grid* g, int mem, const double* diag,
                         const double* off, double w2, double w3, const double* x, double* y);
int epc_gn_cross_diag_add(epc_context* ctx, const epc_grid* g, int mem, const double* diag,
                          double w2, double w3, double* out);
int epc_jacobi_apply(epc_context* ctx, long long n, int mem, const double* diag, const double* r,
                     double* z);

/* residual, objective.hpp:48, objective.cpp:77-91 (cells). */
int epc_residual(epc_context* ctx, const epc_grid* g, int mem, const double* iplus,
                 const double* iminus, const double* b, double* r);

/* Library build identity (arch, mode) for logs. */
/* The reference's test-side helpers of the path, bitwise:
 * avg_x1 / diff_x1 (faces -> cells) and diff_x1_adjoint (cells -> faces),
 * operators.hpp:25-32; smoother_hessian_apply, operators.hpp:43;
 * TridiagBlocks::apply (y += s T x), operators.hpp:61; tridiag_solve_batched
 * (nonpositive pivot: EPC_ERR_RUNTIME naming the column), operators.hpp:80;
 * DctCoupledSolver::apply (Gt z), operators.hpp:102;
 * DistanceEval::hessian_apply at b (V Jr^T Jr p), objective.hpp:57;
 * is_strictly_feasible (max |D1 b| <= 1 - 1e-10), objective.hpp:46. */
int epc_avg_x1(epc_context* ctx, const epc_grid* g, int mem, const double* b, double* out);
int epc_diff_x1(epc_context* ctx, const epc_grid* g, int mem, const double* b, double* out);
int epc_diff_x1_adjoint(epc_context* ctx, const epc_grid* g, int mem, const double* r,
                        double* out);
int epc_smoother_hessian_apply(epc_context* ctx, const epc_grid* g, int mem, const double* b,
                               double* out);
int epc_tridiag_apply(epc_context* ctx, const epc_grid* g, int mem, const double* diag,
                      const double* off, const double* x, double s, double* y);
int epc_tridiag_solve_batched(epc_context* ctx, const epc_grid* g, int mem, const double* diag,
                              const double* off, const double* rhs, double* x);
int epc_dct_apply(epc_context* ctx, const epc_grid* g, int mem, const double* z, double alpha,
                  double rho, double* out);
int epc_distance_hessian_apply(epc_context* ctx, const epc_grid* g, int mem, const double* iplus,
                               const double* iminus, const double* b, const double* p,
                               double* out);
int epc_is_strictly_feasible(epc_context* ctx, const epc_grid* g, int mem, const double* b,
                             int* feasible);

/* fp32 variant of admm_solve (BASELINE configs[2] "fp64 and an fp32 variant";
 * SURVEY 8(d)): the same algorithm with fp32 storage and element arithmetic,
 * sums accumulated in fp64, QP/SQP thresholds rescaled for fp32 (admm_f32.cu).
 * Not bitwise: its deviation from the fp64 reference is stated in DESIGN.md.
 * Arrays are float32 (cells for the images, faces for b, z, u); NULL starts
 * are zero; rows/status as epc_admm_solve. */
int epc_admm_solve_f32(epc_context* ctx, const epc_grid* g, int mem, const float* iplus,
                       const float* iminus, const float* b0, const float* z0, const float* u0,
                       float* b_out, float* z_out, float* u_out, double* rho,
                       const epc_objective_params* p, const epc_admm_config* cfg, int level_tag,
                       epc_admm_row* rows, int max_rows, epc_solve_status* status);

const char* epc_build_info(void);

/* ---- either side of the solve (image.hpp:62-86) -------- */
/* correct_pair (image.cpp:226-253): the two corrected volumes. */
int epc_correct_pair(epc_context* ctx, const epc_grid* grid, int mem, const double* iplus,
                     const double* iminus, const double* b, double* out_plus, double* out_minus);
/* ssd (image.cpp:255-263) and ncc (:265-283) of two cell fields. */
int epc_ssd(epc_context* ctx, const epc_grid* grid, int mem, const double* a, const double* b,
            double* out);
int epc_ncc(epc_context* ctx, const epc_grid* grid, int mem, const double* a, const double* b,
            double* out);
/* simulate_pair (image.cpp:187-224) with SimulateOptions {noise_sigma, seed,
 * feas_margin} (image.hpp:62-66). */
int epc_simulate_pair(epc_context* ctx, const epc_grid* grid, int mem, const double* truth,
                      const double* b_true, double noise_sigma, unsigned long long seed,
                      double feas_margin, double* out_plus, double* out_minus);

/* ---- volume files and the phase-encoding permutation (volume_io.hpp) ------- */
/* GridKind (volume_io.hpp:29) */
enum { EPC_VOL_CELL = 0, EPC_VOL_FACE1 = 1, EPC_VOL_FACE2 = 2, EPC_VOL_FACE3 = 3 };
/* write_volume / read_volume (volume_io.cpp:68-171): 512-byte EPIVOL 1 header,
 * float32 little-endian payload. Host-only (no context). read: v = NULL
 * returns the grid, kind and payload length n only. */
int epc_write_volume(const char* path, const epc_grid* grid, int kind, const double* v);
int epc_read_volume(const char* path, epc_grid* grid, int* kind, double* v, long long cap,
                    long long* n);
/* permute_to_axis1 (volume_io.cpp:203-209) of a cell volume, and
 * unpermute_field (:211-223) of a face1 field, on the device. */
int epc_permute_to_axis1(epc_context* ctx, const epc_grid* grid, int pe_axis, int mem,
                         const double* in, double* out, epc_grid* out_grid);
int epc_unpermute_field(epc_context* ctx, const epc_grid* grid, int pe_axis, int mem,
                        const double* in, double* out, epc_grid* out_grid, int* kind);

/* ---- multilevel (multilevel.hpp:13-63) -------------------- */
enum { EPC_SOLVER_GN = 0, EPC_SOLVER_ADMM = 1 };
/* AdmmRestart (multilevel.hpp:46-50) */
enum { EPC_RESTART_PROLONG_ALL = 1, EPC_RESTART_B_FOR_BOTH = 2, EPC_RESTART_AVERAGE = 3 };
/* SolveReport of a multilevel solve: both row lists appended level by level
 * (report.cpp:23-28); stop / message are the last level's. */
typedef struct {
    int stop;
    int n_admm_rows, n_gn_rows;
    int b_level; /* the level whose grid b_out holds: nlev - 1, or the level an
                    error / line-search failure stopped at (multilevel.cpp:246-249, 263) */
    char message[256];
} epc_multilevel_status;
/* default_schedule (multilevel.cpp:22-41): coarse-to-fine grids into out[cap];
 * host-only, no context. */
int epc_default_schedule(const epc_grid* fine, int max_levels, int min_cells, epc_grid* out,
                         int cap, int* nlev);
/* restrict_image (multilevel.cpp:98-131): area-weighted block averaging of a
 * cell field from `fine` to `coarse`. */
int epc_restrict_image(epc_context* ctx, const epc_grid* fine, const epc_grid* coarse, int mem,
                       const double* in, double* out);
/* prolong_field (multilevel.cpp:157-203): linear interpolation of a face
 * field from `coarse` to `fine`, rescaled to max|D1 b| = 0.95 if infeasible. */
int epc_prolong_field(epc_context* ctx, const epc_grid* coarse, const epc_grid* fine, int mem,
                      const double* in, double* out);
/* multilevel_solve (multilevel.cpp:205-289) over `levels` (coarse -> fine,
 * the last equal to `fine`); per-level overrides gn_max_outer /
 * admm_max_iter (NULL or -1 entries: none). The images stay on the device
 * between levels. b_out: the finest field. */
int epc_multilevel_solve(epc_context* ctx, const epc_grid* fine, int mem, const double* iplus,
                         const double* iminus, const epc_grid* levels, int nlev,
                         const int* gn_max_outer, const int* admm_max_iter, int solver,
                         const epc_objective_params* params, const epc_gn_config* gn_cfg,
                         const epc_admm_config* admm_cfg, int restart, double* b_out,
                         epc_admm_row* admm_rows, int max_admm_rows, epc_gn_row* gn_rows,
                         int max_gn_rows, epc_multilevel_status* status);

/* ---- slab-distributed ADMM building blocks -------------
 * One volume split into k-slabs over ranks: rank r owns layers
 * [k0, k0 + mk) of `full` in the reference face layout. These are the local
 * steps of one admm_solve iteration (admm.cpp:488-560); the caller performs
 * the collectives between them (paper_1607_00531_b200/dist_admm.py: two
 * all-to-all transposes for the axis-3 DCT, a one-layer halo of z, an
 * all-gather of the scalars). All pointers are device pointers.
 * Rank blocks: on the sender, the block for rank s holds s's i range
 * (shard_range over n1) of the local layers in the order [kl][j][il];
 * concatenated over senders they form the receiver's i-slab layout
 * il + ni (j + m2 k). */
/* b_update (admm.cpp:301-443) on the slab's columns. sums3 = {max kkt,
 * sum r^2, sum (D1 b)^2}; ints4 = {lowest failing column in the global
 * numbering j + m2 k (-1: none), failure code, sqp iters, qp iters}. */
int epc_slab_bstep(epc_context* ctx, const epc_grid* full, int k0, int mk, const double* iplus,
                   const double* iminus, const double* b, const double* z, const double* u,
                   double rho, const epc_objective_params* params, const epc_admm_config* cfg,
                   double* b_out, double* sums3, long long* ints4);
/* z_update first half (operators.cpp:388-400): rho V (b + u), the axis-2
 * DCT (transform_axis2, operators.cpp:347-366), packed into rank blocks. */
int epc_slab_zforward(epc_context* ctx, const epc_grid* full, int k0, int mk, int world,
                      const double* b, const double* u, double rho, double* blocks);
/* on an i-slab of ni faces per row: the axis-3 DCT, the spectral divide and
 * the inverse axis-3 DCT (operators.cpp:367-386, 400-412). */
int epc_slab_zsolve3(epc_context* ctx, const epc_grid* full, int ni, const double* in,
                     double alpha, double rho, double* out);
/* z_update second half: unpack, inverse axis-2 DCT -> z_new, and
 * dual_update_and_residuals (admm.cpp:453-476): u_new = u_old + b - z_new;
 * sums6 = {|b-z|^2, |z_old-z|^2, |b|^2, |z|^2, |u_new|^2, u_new.(b-z)}. */
int epc_slab_zbackward(epc_context* ctx, const epc_grid* full, int k0, int mk, int world,
                       const double* blocks, const double* b, const double* u_old,
                       const double* z_old, double rho, double* z_new, double* u_new,
                       double* sums6);
/* g_value parts (admm.cpp:275-285): sums2 = {sum (D2 z)^2, sum (D3 z)^2}
 * over the slab, the D3 terms across the upper boundary from `halo` (the
 * next rank's first face layer; NULL on the last rank). */
int epc_slab_zdiff(epc_context* ctx, const epc_grid* full, int k0, int mk, const double* z,
                   const double* halo, double* sums2);
/* x *= factor (the u rescale after a rho change, admm.cpp:546-552). */
int epc_slab_scale(epc_context* ctx, long long n, double* x, double factor);
/* ---- multi-GPU variants of admm_solve ---------------------- */

/* C4: npairs independent pairs (pair-major host arrays, as
 * epc_admm_solve_batch) over a device list: contexts ctxs[0..nctx) (one per
 * device), pairs split into contiguous balanced blocks, each block solved by
 * epc_admm_solve_batch on its device from its own host thread. Results,
 * rows and statuses land at the pairs' own offsets. No collective: pairs
 * never couple. */
int epc_admm_solve_batch_devices(epc_context* const* ctxs, int nctx, const epc_grid* g, int npairs,
                                 const double* iplus, const double* iminus, const double* b_in,
                                 const double* z_in, const double* u_in, double* b_out,
                                 double* z_out, double* u_out, double* rho,
                                 const epc_objective_params* p, const epc_admm_config* cfg,
                                 int level_tag, epc_admm_row* rows, int max_rows,
                                 epc_solve_status* status);

/* NCCL communicator plumbing (NCCL is opened at run time): a 128-byte
 * ncclUniqueId from rank 0, broadcast by the caller; one communicator per
 * rank on `device`. comm is an ncclComm_t. */
int epc_nccl_unique_id(char* out128);
int epc_nccl_comm_create(int device, int world, int rank, const char* id128, void** comm);
int epc_nccl_comm_destroy(void* comm);

/* C5: admm_solve (admm.hpp:127-129) of ONE volume in k-slabs over the ranks
 * of an NCCL communicator (comm may be NULL at world = 1). Rank r owns face
 * layers [k0, k0 + mk) by shard_range over m3; ip/im are its cell slab,
 * b_in/z_in/u_in (optional) and b_out/z_out/u_out its face slab, all DEVICE
 * pointers on ctx's device. Per iteration: b-step, axis-2 DCT, a grouped
 * ncclSend/ncclRecv all-to-all to i-slabs, axis-3 DCT + divide + inverse,
 * the all-to-all back, inverse axis-2 DCT + dual update, a one-layer z halo
 * from rank + 1, an ncclAllGather of 16 scalars; rows (replicated on every
 * rank), stop test and rho schedule as epc_admm_solve. b, z, u are bitwise
 * the single-GPU solve's (and the reference's) at every world size. */
int epc_slab_admm_solve(epc_context* ctx, void* comm, int rank, int world, const epc_grid* full,
                        const double* ip, const double* im, const double* b_in, const double* z_in,
                        const double* u_in, double* b_out, double* z_out, double* u_out,
                        double* rho, const epc_objective_params* p, const epc_admm_config* cfg,
                        int level_tag, epc_admm_row* rows, int max_rows, epc_solve_status* status);

/* The reference's five sequential dual-update sums (sum (b-z)^2, (zo-z)^2,
 * b^2, z^2, u^2 in index order, admm.cpp:461-469, grid.cpp:60-64) over n
 * faces, continuing the chains in io5[5] (host, in/out). The slab loop calls
 * it rank after rank when a certified decision is undecidable. */
int epc_slab_seq_sums(epc_context* ctx, long long n, const double* b_new, const double* z_new,
                      const double* z_old, const double* u_new, double* io5);
/* max |D1 b| over the slab (admm_solve's feasibility check, admm.cpp:501-502). */
int epc_slab_d1_norm_inf(epc_context* ctx, const epc_grid* full, int k0, int mk, const double* b,
                         double* out);

/* ---- GN-PCG in k-slabs (GN row) -------------------------------
 * Vectors are *extended*: the owned layers [k0, k0 + mk) plus one halo layer
 * below (lo = 1 unless k0 = 0) and above (hi = 1 unless k0 + mk = m3), in the
 * face (cell) layout of layers k0 - lo .. k0 + mk + hi - 1. Sums cover the
 * owned layers; halos are the caller's (paper_1607_00531_b200/dist_gn.py). */
/* objective_gn (objective.cpp:231-264) partials: out8 = {sum r^2,
 * sum (D1 b)^2, sum phi, max |D1 b|, sum (D2 b)^2, sum (D3 b)^2, sum grad.dir,
 * max |b|}; grad_ext (owned faces) when need_grad; keep_jac for _hessian. */
int epc_gnslab_objective(epc_context* ctx, const epc_grid* full, int k0, int mk, int lo, int hi,
                         const double* iplus_ext, const double* iminus_ext, const double* b_ext,
                         const epc_objective_params* params, int need_grad, double* grad_ext,
                         const double* dir_ext, int keep_jac, double* out8);
/* GnHessian blocks at b (objective.cpp:266-300) and the block-Jacobi
 * factor of the owned columns (gn_pcg.cpp:48-54); fail_col = lowest global
 * column with a nonpositive pivot or -1. */
int epc_gnslab_hessian(epc_context* ctx, const epc_grid* full, int k0, int mk, int lo, int hi,
                       const double* iplus_ext, const double* iminus_ext, const double* b_ext,
                       const epc_objective_params* params, int precond, long long* fail_col);
/* q = H p (GnHessian::apply, objective.cpp:302-331); pq = owned sum p.q. */
int epc_gnslab_hv(epc_context* ctx, const epc_grid* full, int k0, int mk, int lo, int hi,
                  const epc_objective_params* params, const double* p_ext, double* q_ext,
                  double* pq);
/* pcg update on owned columns (gn_pcg.cpp:114-120): if do_axpy d += a p,
 * r -= a q; z = M^{-1} r; rr_rz = {sum r.r, sum r.z}. */
int epc_gnslab_update(epc_context* ctx, const epc_grid* full, int k0, int mk, int lo, int hi,
                      const epc_objective_params* params, int precond, double a, int do_axpy,
                      double* d_ext, double* r_ext, double* z_ext, const double* p_ext,
                      const double* q_ext, double* rr_rz);
/* y = x + t d; r = -g with gg = sum g.g; ab_bb = {sum a.b, sum b.b}. */
int epc_gnslab_axpy(epc_context* ctx, long long n, const double* x, double t, const double* d,
                    double* y);
int epc_gnslab_negate(epc_context* ctx, long long n, const double* g, double* r, double* gg);
int epc_gnslab_dot(epc_context* ctx, long long n, const double* a, const double* b,
                   double* ab_bb);

#ifdef __cplusplus
}
#endif

#endif /* EPICORR_B200_H */
