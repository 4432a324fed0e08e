/*
 * oracle_api.h — TEST INFRASTRUCTURE ONLY. Never linked into the product.
 *
 * One C API, two implementations:
 *   oracle/_ref/libepicorr_ref.so     the unmodified reference library
 *                                     (/root/reference/proj/src) behind a thin
 *                                     extern "C" harness (ref_harness.cpp);
 *   oracle/_build/libepicorr_oracle.so the plain-C restatement
 *                                     (epicorr_oracle.c) used as the checker
 *                                     where the reference tree is absent.
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may load them.
 *
 * Types are the product's POD structs (include/epicorr_b200.h). Return codes
 * are EPC_* status codes; `msg` receives the reference's e.what() text.
 */
#ifndef EPICORR_ORACLE_API_H
#define EPICORR_ORACLE_API_H

#include "../include/epicorr_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

int oracle_admm_solve(const epc_grid* g, const double* iplus, const double* iminus,
                      const double* b_in, const double* z_in, const double* u_in,
                      double* b_out, double* z_out, double* u_out, double* rho,
                      const epc_objective_params* p, const epc_admm_config* cfg, int level_tag,
                      epc_admm_row* rows, int max_rows, epc_solve_status* status);

int oracle_gn_solve(const epc_grid* g, const double* iplus, const double* iminus,
                    const double* b0, double* b_out, const epc_objective_params* p,
                    const epc_gn_config* cfg, int level_tag, epc_gn_row* rows, int max_rows,
                    epc_solve_status* status);

int oracle_b_update(const epc_grid* g, const double* iplus, const double* iminus,
                    const double* b, const double* z, const double* u, double rho,
                    const epc_objective_params* p, const epc_admm_config* cfg, double* b_out,
                    epc_bupdate_stats* stats, char* msg, size_t msglen);

int oracle_z_update(const epc_grid* g, const double* b, const double* u, double rho,
                    double alpha, double* z_out, char* msg, size_t msglen);

int oracle_dct_solve(const epc_grid* g, const double* rhs, double alpha, double rho,
                     double* out, char* msg, size_t msglen);

int oracle_dual_update(const epc_grid* g, const double* b_new, const double* z_new,
                       const double* z_old, const double* u_old, double rho, double eps_abs,
                       double eps_rel, double* u_out, epc_dual_result* out);

double oracle_augmented_lagrangian(const epc_grid* g, const double* iplus, const double* iminus,
                                   const double* b, const double* z, const double* u,
                                   double rho, double alpha);

int oracle_qp_active_set(int n, double h, const double* gd, const double* go, const double* c,
                         const double* x0, int max_iter, double* x, double* lambda,
                         int* active_sign, int* iters, char* msg, size_t msglen);

double oracle_verify_qp_kkt(int n, double h, const double* gd, const double* go,
                            const double* c, const double* x, const double* lambda,
                            const int* active_sign);

int oracle_objective_gn(const epc_grid* g, const double* iplus, const double* iminus,
                        const double* b, const epc_objective_params* p, int need_grad,
                        epc_objective_eval* out, double* grad, double* residual);

int oracle_gn_hessian_build(const epc_grid* g, const double* iplus, const double* iminus,
                            const double* b, const epc_objective_params* p, double* diag,
                            double* off, double* pdiag, char* msg, size_t msglen);

int oracle_gn_hessian_apply(const epc_grid* g, const double* iplus, const double* iminus,
                            const double* b, const epc_objective_params* p, const double* x,
                            double* y, char* msg, size_t msglen);

int oracle_precond_apply(const epc_grid* g, const double* iplus, const double* iminus,
                         const double* b, const epc_objective_params* p, int kind,
                         const double* r, double* z, char* msg, size_t msglen);

int oracle_pcg(const epc_grid* g, const double* iplus, const double* iminus, const double* b,
               const epc_objective_params* p, int kind, const double* grad, double eta,
               int max_iters, double* d, epc_pcg_result* out, char* msg, size_t msglen);

int oracle_residual(const epc_grid* g, const double* iplus, const double* iminus,
                    const double* b, double* r);

double oracle_rho_schedule(int schedule, double rho, double rho_min, double primal_res,
                           double dual_res, double tau_incr, double tau_decr, double mu);

/* Thread count used by the reference harness (ignored by the C restatement). */
void oracle_set_threads(int threads);

/* multilevel (multilevel.cpp): see the epc_* counterparts in epicorr_b200.h */
int oracle_default_schedule(const epc_grid* fine, int max_levels, int min_cells, epc_grid* out,
                            int cap, int* nlev, char* msg, size_t msglen);
int oracle_restrict_image(const epc_grid* fine, const epc_grid* coarse, const double* in,
                          double* out, char* msg, size_t msglen);
int oracle_prolong_field(const epc_grid* coarse, const epc_grid* fine, const double* in,
                         double* out, char* msg, size_t msglen);
int oracle_multilevel_solve(const epc_grid* fine, const double* iplus, const double* iminus,
                            const epc_grid* levels, int nlev, const int* gn_max_outer,
                            const int* admm_max_iter, int solver,
                            const epc_objective_params* p, const epc_gn_config* gcfg,
                            const epc_admm_config* acfg, int restart, double* b_out,
                            epc_admm_row* arows, int max_arows, epc_gn_row* grows,
                            int max_grows, epc_multilevel_status* st);

/* image.cpp: correct_pair, ssd, ncc, simulate_pair */
int oracle_correct_pair(const epc_grid* g, const double* iplus, const double* iminus,
                        const double* b, double* out_plus, double* out_minus, char* msg,
                        size_t msglen);
int oracle_ssd(const epc_grid* g, const double* a, const double* b, double* out, char* msg,
               size_t msglen);
int oracle_ncc(const epc_grid* g, const double* a, const double* b, double* out, char* msg,
               size_t msglen);
int oracle_simulate_pair(const epc_grid* g, const double* truth, const double* b_true,
                         double noise_sigma, unsigned long long seed, double feas_margin,
                         double* out_plus, double* out_minus, char* msg, size_t msglen);

/* the reference's test-side helpers of the path */
int oracle_avg_x1(const epc_grid* g, const double* b, double* out);
int oracle_diff_x1(const epc_grid* g, const double* b, double* out);
int oracle_diff_x1_adjoint(const epc_grid* g, const double* r, double* out);
int oracle_smoother_hessian_apply(const epc_grid* g, const double* b, double* out);
int oracle_tridiag_apply(const epc_grid* g, const double* diag, const double* off,
                         const double* x, double s, double* y);
int oracle_tridiag_solve_batched(const epc_grid* g, const double* diag, const double* off,
                                 const double* rhs, double* x, char* msg, size_t msglen);
int oracle_dct_apply(const epc_grid* g, const double* z, double alpha, double rho, double* out);
int oracle_distance_hessian_apply(const epc_grid* g, const double* iplus, const double* iminus,
                                  const double* b, const double* p, double* out);
int oracle_is_strictly_feasible(const epc_grid* g, const double* b);

#ifdef __cplusplus
}
#endif

#endif
