// ref_harness.cpp — TEST INFRASTRUCTURE ONLY (oracle/, never shipped).
//
// extern "C" adapter from oracle_api.h onto the UNMODIFIED reference library
// compiled from /root/reference/proj/src (see oracle/Makefile). It only
// marshals plain arrays into the reference's own types and calls its public
// entry points; no reference arithmetic is restated here.

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <span>
#include <vector>

#include "epicorr/admm.hpp"
#include "epicorr/gn_pcg.hpp"
#include "epicorr/grid.hpp"
#include "epicorr/image.hpp"
#include "epicorr/multilevel.hpp"
#include "epicorr/volume_io.hpp"
#include "epicorr/objective.hpp"
#include "epicorr/operators.hpp"

#include "oracle_api.h"

using namespace epicorr;

namespace {

int g_threads = 1;

GridSpec to_grid(const epc_grid* g) {
    GridSpec s;
    s.dim = g->dim;
    for (int a = 0; a < 3; ++a) {
        s.m[a] = g->m[a];
        s.h[a] = g->h[a];
        s.origin[a] = g->origin[a];
    }
    s.validate();
    return s;
}

StaggeredField faces(const GridSpec& g, const double* v) {
    StaggeredField f(g);
    if (v) std::memcpy(f.v.data(), v, sizeof(double) * f.v.size());
    return f;
}

ImageVolume cells(const GridSpec& g, const double* v) {
    ImageVolume f(g);
    std::memcpy(f.v.data(), v, sizeof(double) * f.v.size());
    return f;
}

ObjectiveParams to_params(const epc_objective_params* p) {
    ObjectiveParams o;
    o.alpha = p->alpha;
    o.beta = p->beta;
    o.gamma = p->gamma;
    o.enforce_linf_box = p->enforce_linf_box != 0;
    return o;
}

ADMMConfig to_admm(const epc_admm_config* c) {
    ADMMConfig o;
    o.rho0 = c->rho0;
    o.rho_min = c->rho_min;
    o.schedule = RhoSchedule(c->schedule);
    o.eps_abs = c->eps_abs;
    o.eps_rel = c->eps_rel;
    o.max_iter = c->max_iter;
    o.tau_incr = c->tau_incr;
    o.tau_decr = c->tau_decr;
    o.mu = c->mu;
    o.sqp_max_iter = c->sqp_max_iter;
    o.sqp_tol_rel = c->sqp_tol_rel;
    o.check_kkt = c->check_kkt != 0;
    o.threads = c->threads > 0 ? c->threads : g_threads;
    return o;
}

GNConfig to_gn(const epc_gn_config* c) {
    GNConfig o;
    o.eta = c->eta;
    o.max_outer = c->max_outer;
    o.eps_obj = c->eps_obj;
    o.eps_iter = c->eps_iter;
    o.eps_grad = c->eps_grad;
    o.wolfe_c1 = c->wolfe_c1;
    o.wolfe_c2 = c->wolfe_c2;
    o.max_pcg = c->max_pcg;
    o.max_ls = c->max_ls;
    o.precond = PrecondKind(c->precond);
    o.threads = c->threads > 0 ? c->threads : g_threads;
    return o;
}

void put_msg(char* msg, size_t len, const char* text) {
    if (!msg || len == 0) return;
    std::snprintf(msg, len, "%s", text);
}

template <class F>
int guarded(char* msg, size_t len, F&& f) {
    put_msg(msg, len, "");
    try {
        f();
        return EPC_OK;
    } catch (const std::invalid_argument& e) {
        put_msg(msg, len, e.what());
        return EPC_ERR_INVALID_ARGUMENT;
    } catch (const std::domain_error& e) {
        put_msg(msg, len, e.what());
        return EPC_ERR_DOMAIN;
    } catch (const std::exception& e) {
        put_msg(msg, len, e.what());
        return EPC_ERR_RUNTIME;
    }
}

void copy_out(const StaggeredField& f, double* out) {
    if (out) std::memcpy(out, f.v.data(), sizeof(double) * f.v.size());
}

} // namespace

extern "C" {

void oracle_set_threads(int threads) { g_threads = threads > 0 ? threads : 1; }

int oracle_admm_solve(const epc_grid* gg, const double* iplus, const double* iminus,
                      const double* b_in, const double* z_in, const double* u_in,
                      double* b_out, double* z_out, double* u_out, double* rho,
                      const epc_objective_params* p, const epc_admm_config* cfg, int level_tag,
                      epc_admm_row* rows, int max_rows, epc_solve_status* status) {
    char* msg = status ? status->message : nullptr;
    return guarded(msg, status ? sizeof status->message : 0, [&] {
        const GridSpec g = to_grid(gg);
        const VolumePair pair(cells(g, iplus), cells(g, iminus));
        ADMMState init;
        if (b_in) init.b = faces(g, b_in);
        if (z_in) init.z = faces(g, z_in);
        if (u_in) init.u = faces(g, u_in);
        init.rho = rho ? *rho : 0.0;
        AdmmSolveResult res = admm_solve(pair, std::move(init), to_params(p), to_admm(cfg), level_tag);
        copy_out(res.state.b, b_out);
        copy_out(res.state.z, z_out);
        copy_out(res.state.u, u_out);
        if (rho) *rho = res.state.rho;
        const int n = int(std::min<std::size_t>(res.report.admm.size(), std::size_t(max_rows)));
        for (int i = 0; i < n; ++i) {
            const AdmmIterRow& r = res.report.admm[i];
            rows[i] = epc_admm_row{r.level,    r.iter,       r.primal_res, r.dual_res,
                                   r.eps_pri,  r.eps_dual,   r.rho,        r.lagrangian,
                                   r.kkt_violation, r.b_update_s, r.wall_s};
        }
        if (status) {
            status->stop = int(res.report.stop);
            status->nrows = int(res.report.admm.size());
            std::snprintf(status->message, sizeof status->message, "%s", res.report.message.c_str());
        }
    });
}

int oracle_gn_solve(const epc_grid* gg, const double* iplus, const double* iminus,
                    const double* b0, double* b_out, const epc_objective_params* p,
                    const epc_gn_config* cfg, int level_tag, epc_gn_row* rows, int max_rows,
                    epc_solve_status* status) {
    char* msg = status ? status->message : nullptr;
    return guarded(msg, status ? sizeof status->message : 0, [&] {
        const GridSpec g = to_grid(gg);
        const VolumePair pair(cells(g, iplus), cells(g, iminus));
        GnSolveResult res =
            gauss_newton_solve(pair, faces(g, b0), to_params(p), to_gn(cfg), level_tag);
        copy_out(res.b, b_out);
        const int n = int(std::min<std::size_t>(res.report.gn.size(), std::size_t(max_rows)));
        for (int i = 0; i < n; ++i) {
            const GnIterRow& r = res.report.gn[i];
            rows[i] = epc_gn_row{r.level,     r.iter,       r.j_value,        r.grad_norm, r.step,
                                 r.pcg_iters, r.pcg_relres, r.pcg_relres_prec, r.wall_s};
        }
        if (status) {
            status->stop = int(res.report.stop);
            status->nrows = int(res.report.gn.size());
            std::snprintf(status->message, sizeof status->message, "%s", res.report.message.c_str());
        }
    });
}

int oracle_b_update(const epc_grid* gg, const double* iplus, const double* iminus,
                    const double* b, const double* z, const double* u, double rho,
                    const epc_objective_params* p, const epc_admm_config* cfg, double* b_out,
                    epc_bupdate_stats* stats, char* msg, size_t msglen) {
    return guarded(msg, msglen, [&] {
        const GridSpec g = to_grid(gg);
        const VolumePair pair(cells(g, iplus), cells(g, iminus));
        ADMMState st;
        st.b = faces(g, b);
        st.z = faces(g, z);
        st.u = faces(g, u);
        st.rho = rho;
        BUpdateStats s;
        StaggeredField out = b_update(pair, st, to_params(p), to_admm(cfg), &s);
        copy_out(out, b_out);
        if (stats) {
            stats->sqp_iters = s.sqp_iters;
            stats->qp_iters = s.qp_iters;
            stats->kkt_violation = s.kkt_violation;
            stats->max_active = -1;
        }
    });
}

int oracle_z_update(const epc_grid* gg, const double* b, const double* u, double rho,
                    double alpha, double* z_out, char* msg, size_t msglen) {
    return guarded(msg, msglen, [&] {
        const GridSpec g = to_grid(gg);
        ADMMState st;
        st.b = faces(g, b);
        st.u = faces(g, u);
        st.rho = rho;
        const DctCoupledSolver dct(g, g_threads);
        copy_out(z_update(st, alpha, dct), z_out);
    });
}

int oracle_dct_solve(const epc_grid* gg, const double* rhs, double alpha, double rho,
                     double* out, char* msg, size_t msglen) {
    return guarded(msg, msglen, [&] {
        const GridSpec g = to_grid(gg);
        const DctCoupledSolver dct(g, g_threads);
        copy_out(dct.solve(faces(g, rhs), alpha, rho), out);
    });
}

int oracle_dual_update(const epc_grid* gg, const double* b_new, const double* z_new,
                       const double* z_old, const double* u_old, double rho, double eps_abs,
                       double eps_rel, double* u_out, epc_dual_result* out) {
    return guarded(nullptr, 0, [&] {
        const GridSpec g = to_grid(gg);
        DualUpdate du = dual_update_and_residuals(faces(g, b_new), faces(g, z_new),
                                                  faces(g, z_old), faces(g, u_old), rho,
                                                  eps_abs, eps_rel);
        copy_out(du.u, u_out);
        if (out) *out = epc_dual_result{du.primal_res, du.dual_res, du.eps_pri, du.eps_dual};
    });
}

double oracle_augmented_lagrangian(const epc_grid* gg, const double* iplus, const double* iminus,
                                   const double* b, const double* z, const double* u,
                                   double rho, double alpha) {
    const GridSpec g = to_grid(gg);
    const VolumePair pair(cells(g, iplus), cells(g, iminus));
    return augmented_lagrangian(pair, faces(g, b), faces(g, z), faces(g, u), rho, alpha,
                                g_threads);
}

int oracle_qp_active_set(int n, double h, const double* gd, const double* go, const double* c,
                         const double* x0, int max_iter, double* x, double* lambda,
                         int* active_sign, int* iters, char* msg, size_t msglen) {
    return guarded(msg, msglen, [&] {
        QpResult r = qp_active_set(n, h, std::span<const double>(gd, n),
                                   std::span<const double>(go, n), std::span<const double>(c, n),
                                   std::span<const double>(x0, n), max_iter);
        std::memcpy(x, r.x.data(), sizeof(double) * n);
        std::memcpy(lambda, r.lambda.data(), sizeof(double) * (n - 1));
        std::memcpy(active_sign, r.active_sign.data(), sizeof(int) * (n - 1));
        if (iters) *iters = r.iters;
    });
}

double oracle_verify_qp_kkt(int n, double h, const double* gd, const double* go,
                            const double* c, const double* x, const double* lambda,
                            const int* active_sign) {
    QpResult r;
    r.x.assign(x, x + n);
    r.lambda.assign(lambda, lambda + (n - 1));
    r.active_sign.assign(active_sign, active_sign + (n - 1));
    return verify_qp_kkt(n, h, std::span<const double>(gd, n), std::span<const double>(go, n),
                         std::span<const double>(c, n), r);
}

int oracle_objective_gn(const epc_grid* gg, const double* iplus, const double* iminus,
                        const double* b, const epc_objective_params* p, int need_grad,
                        epc_objective_eval* out, double* grad, double* residual) {
    return guarded(nullptr, 0, [&] {
        const GridSpec g = to_grid(gg);
        const VolumePair pair(cells(g, iplus), cells(g, iminus));
        ObjectiveEval ev = objective_gn(pair, faces(g, b), to_params(p), g_threads, need_grad != 0);
        if (out) *out = epc_objective_eval{ev.value, ev.dist, ev.smooth, ev.pen, ev.feasible ? 1 : 0};
        if (grad && !ev.grad.v.empty()) copy_out(ev.grad, grad);
        if (residual && !ev.residual.v.empty())
            std::memcpy(residual, ev.residual.v.data(), sizeof(double) * ev.residual.v.size());
    });
}

int oracle_gn_hessian_build(const epc_grid* gg, const double* iplus, const double* iminus,
                            const double* b, const epc_objective_params* p, double* diag,
                            double* off, double* pdiag, char* msg, size_t msglen) {
    return guarded(msg, msglen, [&] {
        const GridSpec g = to_grid(gg);
        const VolumePair pair(cells(g, iplus), cells(g, iminus));
        GnHessian h(pair, faces(g, b), to_params(p), g_threads);
        const std::size_t n = std::size_t(g.faces());
        if (diag) std::memcpy(diag, h.column_part().diag.data(), sizeof(double) * n);
        if (off) std::memcpy(off, h.column_part().off.data(), sizeof(double) * n);
        if (pdiag) {
            TridiagBlocks t = h.preconditioner_blocks();
            std::memcpy(pdiag, t.diag.data(), sizeof(double) * n);
        }
    });
}

int oracle_gn_hessian_apply(const epc_grid* gg, const double* iplus, const double* iminus,
                            const double* b, const epc_objective_params* p, const double* x,
                            double* y, char* msg, size_t msglen) {
    return guarded(msg, msglen, [&] {
        const GridSpec g = to_grid(gg);
        const VolumePair pair(cells(g, iplus), cells(g, iminus));
        GnHessian h(pair, faces(g, b), to_params(p), g_threads);
        copy_out(h.apply(faces(g, x)), y);
    });
}

int oracle_precond_apply(const epc_grid* gg, const double* iplus, const double* iminus,
                         const double* b, const epc_objective_params* p, int kind,
                         const double* r, double* z, char* msg, size_t msglen) {
    return guarded(msg, msglen, [&] {
        const GridSpec g = to_grid(gg);
        const VolumePair pair(cells(g, iplus), cells(g, iminus));
        GnHessian h(pair, faces(g, b), to_params(p), g_threads);
        LinOp m = make_preconditioner(PrecondKind(kind), h, g_threads);
        std::vector<double> rv(r, r + g.faces()), zv;
        m(rv, zv);
        std::memcpy(z, zv.data(), sizeof(double) * zv.size());
    });
}

int oracle_pcg(const epc_grid* gg, const double* iplus, const double* iminus, const double* b,
               const epc_objective_params* p, int kind, const double* grad, double eta,
               int max_iters, double* d, epc_pcg_result* out, char* msg, size_t msglen) {
    return guarded(msg, msglen, [&] {
        const GridSpec g = to_grid(gg);
        const VolumePair pair(cells(g, iplus), cells(g, iminus));
        GnHessian h(pair, faces(g, b), to_params(p), g_threads);
        LinOp m = make_preconditioner(PrecondKind(kind), h, g_threads);
        LinOp apply_h = [&h](const std::vector<double>& x, std::vector<double>& y) {
            y.resize(x.size());
            h.apply(x, y);
        };
        std::vector<double> gv(grad, grad + g.faces());
        PcgResult res = pcg(apply_h, m, gv, eta, max_iters);
        std::memcpy(d, res.d.data(), sizeof(double) * res.d.size());
        if (out) *out = epc_pcg_result{res.iters, res.relres, res.relres_prec, res.reached_tol ? 1 : 0};
    });
}

int oracle_residual(const epc_grid* gg, const double* iplus, const double* iminus,
                    const double* b, double* r) {
    return guarded(nullptr, 0, [&] {
        const GridSpec g = to_grid(gg);
        const VolumePair pair(cells(g, iplus), cells(g, iminus));
        CellField rr = residual(pair, faces(g, b), g_threads);
        std::memcpy(r, rr.v.data(), sizeof(double) * rr.v.size());
    });
}

double oracle_rho_schedule(int schedule, double rho, double rho_min, double primal_res,
                           double dual_res, double tau_incr, double tau_decr, double mu) {
    return rho_schedule(RhoSchedule(schedule), rho, rho_min, primal_res, dual_res, tau_incr,
                        tau_decr, mu);
}


int oracle_default_schedule(const epc_grid* fine, int max_levels, int min_cells, epc_grid* out,
                            int cap, int* nlev, char* msg, size_t msglen) {
    return guarded(msg, msglen, [&] {
        const LevelSchedule s = default_schedule(to_grid(fine), max_levels, min_cells);
        if (s.levels() > cap) throw std::invalid_argument("default_schedule: output capacity too small");
        for (int l = 0; l < s.levels(); ++l) {
            out[l].dim = s.grids[l].dim;
            for (int a = 0; a < 3; ++a) {
                out[l].m[a] = s.grids[l].m[a];
                out[l].h[a] = s.grids[l].h[a];
                out[l].origin[a] = s.grids[l].origin[a];
            }
        }
        *nlev = s.levels();
    });
}

int oracle_restrict_image(const epc_grid* fine, const epc_grid* coarse, const double* in,
                          double* out, char* msg, size_t msglen) {
    return guarded(msg, msglen, [&] {
        const GridSpec gf = to_grid(fine);
        const ImageVolume r = restrict_image(cells(gf, in), to_grid(coarse));
        std::memcpy(out, r.v.data(), sizeof(double) * r.v.size());
    });
}

int oracle_prolong_field(const epc_grid* coarse, const epc_grid* fine, const double* in,
                         double* out, char* msg, size_t msglen) {
    return guarded(msg, msglen, [&] {
        const GridSpec gc = to_grid(coarse);
        copy_out(prolong_field(faces(gc, in), to_grid(fine)), out);
    });
}

int oracle_multilevel_solve(const epc_grid* fine, const double* iplus, const double* iminus,
                            const epc_grid* levels, int nlev, const int* gn_max_outer,
                            const int* admm_max_iter, int solver,
                            const epc_objective_params* p, const epc_gn_config* gcfg,
                            const epc_admm_config* acfg, int restart, double* b_out,
                            epc_admm_row* arows, int max_arows, epc_gn_row* grows,
                            int max_grows, epc_multilevel_status* st) {
    st->stop = EPC_STOP_CONVERGED;
    st->n_admm_rows = st->n_gn_rows = 0;
    st->b_level = nlev - 1;
    return guarded(st->message, sizeof st->message, [&] {
        const GridSpec g = to_grid(fine);
        const VolumePair pair(cells(g, iplus), cells(g, iminus));
        LevelSchedule sched;
        for (int l = 0; l < nlev; ++l) {
            GridSpec s;
            s.dim = levels[l].dim;
            for (int a = 0; a < 3; ++a) {
                s.m[a] = levels[l].m[a];
                s.h[a] = levels[l].h[a];
                s.origin[a] = levels[l].origin[a];
            }
            sched.grids.push_back(s);
        }
        if (gn_max_outer || admm_max_iter) {
            sched.overrides.resize(nlev);
            for (int l = 0; l < nlev; ++l) {
                if (gn_max_outer && gn_max_outer[l] >= 0) sched.overrides[l].gn_max_outer = gn_max_outer[l];
                if (admm_max_iter && admm_max_iter[l] >= 0) sched.overrides[l].admm_max_iter = admm_max_iter[l];
            }
        }
        const MultilevelResult res = multilevel_solve(
            pair, sched, solver == EPC_SOLVER_GN ? SolverKind::gn : SolverKind::admm, to_params(p),
            to_gn(gcfg), to_admm(acfg), AdmmRestart(restart));
        for (int l = 0; l < nlev; ++l)
            if (res.b.grid == sched.grids[l]) st->b_level = l;
        copy_out(res.b, b_out);
        for (std::size_t i = 0; i < res.report.admm.size(); ++i) {
            const AdmmIterRow& r = res.report.admm[i];
            if (int(i) < max_arows)
                arows[i] = epc_admm_row{r.level,   r.iter,       r.primal_res, r.dual_res,
                                        r.eps_pri, r.eps_dual,   r.rho,        r.lagrangian,
                                        r.kkt_violation, r.b_update_s, r.wall_s};
        }
        for (std::size_t i = 0; i < res.report.gn.size(); ++i) {
            const GnIterRow& r = res.report.gn[i];
            if (int(i) < max_grows)
                grows[i] = epc_gn_row{r.level,     r.iter,       r.j_value,        r.grad_norm, r.step,
                                      r.pcg_iters, r.pcg_relres, r.pcg_relres_prec, r.wall_s};
        }
        st->n_admm_rows = int(res.report.admm.size());
        st->n_gn_rows = int(res.report.gn.size());
        st->stop = int(res.report.stop);
        std::snprintf(st->message, sizeof st->message, "%s", res.report.message.c_str());
    });
}


int oracle_correct_pair(const epc_grid* gg, const double* iplus, const double* iminus,
                        const double* b, double* out_plus, double* out_minus, char* msg,
                        size_t msglen) {
    return guarded(msg, msglen, [&] {
        const GridSpec g = to_grid(gg);
        const VolumePair pair(cells(g, iplus), cells(g, iminus));
        auto [cp, cm] = correct_pair(pair, faces(g, b), g_threads);
        std::memcpy(out_plus, cp.v.data(), sizeof(double) * cp.v.size());
        std::memcpy(out_minus, cm.v.data(), sizeof(double) * cm.v.size());
    });
}

int oracle_ssd(const epc_grid* gg, const double* a, const double* b, double* out, char* msg,
               size_t msglen) {
    return guarded(msg, msglen, [&] {
        const GridSpec g = to_grid(gg);
        *out = ssd(cells(g, a), cells(g, b));
    });
}

int oracle_ncc(const epc_grid* gg, const double* a, const double* b, double* out, char* msg,
               size_t msglen) {
    return guarded(msg, msglen, [&] {
        const GridSpec g = to_grid(gg);
        *out = ncc(cells(g, a), cells(g, b));
    });
}

int oracle_simulate_pair(const epc_grid* gg, const double* truth, const double* b_true,
                         double noise_sigma, unsigned long long seed, double feas_margin,
                         double* out_plus, double* out_minus, char* msg, size_t msglen) {
    return guarded(msg, msglen, [&] {
        const GridSpec g = to_grid(gg);
        SimulateOptions o;
        o.noise_sigma = noise_sigma;
        o.seed = seed;
        o.feas_margin = feas_margin;
        const VolumePair p = simulate_pair(cells(g, truth), faces(g, b_true), o);
        std::memcpy(out_plus, p.plus.v.data(), sizeof(double) * p.plus.v.size());
        std::memcpy(out_minus, p.minus.v.data(), sizeof(double) * p.minus.v.size());
    });
}


// ---- volume_io (reference only; the product's counterparts are checked
// against these in tests/test_volume_io.py) --------------------------------
static epc_grid from_grid(const GridSpec& g) {
    epc_grid o;
    o.dim = g.dim;
    for (int a = 0; a < 3; ++a) {
        o.m[a] = g.m[a];
        o.h[a] = g.h[a];
        o.origin[a] = g.origin[a];
    }
    return o;
}

int oracle_write_volume(const char* path, const epc_grid* gg, int kind, const double* v,
                        char* msg, size_t msglen) {
    return guarded(msg, msglen, [&] {
        VolumeData vd;
        vd.grid = to_grid(gg);
        vd.kind = GridKind(kind);
        vd.v.assign(v, v + vd.payload_size());
        write_volume(path, vd);
    });
}

int oracle_read_volume(const char* path, epc_grid* g, int* kind, double* v, long long cap,
                       long long* n, char* msg, size_t msglen) {
    return guarded(msg, msglen, [&] {
        const VolumeData vd = read_volume(path);
        *g = from_grid(vd.grid);
        *kind = int(vd.kind);
        *n = (long long)vd.v.size();
        if (v && cap >= *n) std::memcpy(v, vd.v.data(), sizeof(double) * vd.v.size());
    });
}

int oracle_permute_to_axis1(const epc_grid* gg, int pe_axis, const double* in, double* out,
                            epc_grid* out_grid, char* msg, size_t msglen) {
    return guarded(msg, msglen, [&] {
        const GridSpec g = to_grid(gg);
        const ImageVolume r = permute_to_axis1(cells(g, in), pe_axis);
        *out_grid = from_grid(r.grid);
        std::memcpy(out, r.v.data(), sizeof(double) * r.v.size());
    });
}

int oracle_unpermute_field(const epc_grid* gg, int pe_axis, const double* in, double* out,
                           epc_grid* out_grid, int* kind, char* msg, size_t msglen) {
    return guarded(msg, msglen, [&] {
        const GridSpec g = to_grid(gg);
        const VolumeData vd = unpermute_field(faces(g, in), pe_axis);
        *out_grid = from_grid(vd.grid);
        *kind = int(vd.kind);
        std::memcpy(out, vd.v.data(), sizeof(double) * vd.v.size());
    });
}


// ---- the reference's test-side helpers of the path ----
namespace {
CellField cellfield(const GridSpec& g, const double* v) {
    CellField c(g);
    c.v.assign(v, v + g.cells());
    return c;
}
TridiagBlocks blocks(const GridSpec& g, const double* diag, const double* off) {
    TridiagBlocks t(g);
    t.diag.assign(diag, diag + g.faces());
    t.off.assign(off, off + g.faces());
    return t;
}
}  // namespace

int oracle_avg_x1(const epc_grid* gg, const double* b, double* out) {
    return guarded(nullptr, 0, [&] {
        const GridSpec g = to_grid(gg);
        const CellField c = avg_x1(faces(g, b));
        std::memcpy(out, c.v.data(), sizeof(double) * c.v.size());
    });
}

int oracle_diff_x1(const epc_grid* gg, const double* b, double* out) {
    return guarded(nullptr, 0, [&] {
        const GridSpec g = to_grid(gg);
        const CellField c = diff_x1(faces(g, b));
        std::memcpy(out, c.v.data(), sizeof(double) * c.v.size());
    });
}

int oracle_diff_x1_adjoint(const epc_grid* gg, const double* r, double* out) {
    return guarded(nullptr, 0, [&] {
        const GridSpec g = to_grid(gg);
        copy_out(diff_x1_adjoint(cellfield(g, r)), out);
    });
}

int oracle_smoother_hessian_apply(const epc_grid* gg, const double* b, double* out) {
    return guarded(nullptr, 0, [&] {
        const GridSpec g = to_grid(gg);
        copy_out(smoother_hessian_apply(faces(g, b), g_threads), out);
    });
}

int oracle_tridiag_apply(const epc_grid* gg, const double* diag, const double* off,
                         const double* x, double s, double* y) {
    return guarded(nullptr, 0, [&] {
        const GridSpec g = to_grid(gg);
        const TridiagBlocks t = blocks(g, diag, off);
        const std::size_t n = std::size_t(g.faces());
        t.apply(std::span<const double>(x, n), std::span<double>(y, n), s);
    });
}

int oracle_tridiag_solve_batched(const epc_grid* gg, const double* diag, const double* off,
                                 const double* rhs, double* x, char* msg, size_t msglen) {
    return guarded(msg, msglen, [&] {
        const GridSpec g = to_grid(gg);
        copy_out(tridiag_solve_batched(blocks(g, diag, off), faces(g, rhs), g_threads), x);
    });
}

int oracle_dct_apply(const epc_grid* gg, const double* z, double alpha, double rho, double* out) {
    return guarded(nullptr, 0, [&] {
        const GridSpec g = to_grid(gg);
        const DctCoupledSolver solver(g, g_threads);
        copy_out(solver.apply(faces(g, z), alpha, rho), out);
    });
}

int oracle_distance_hessian_apply(const epc_grid* gg, const double* iplus, const double* iminus,
                                  const double* b, const double* p, double* out) {
    return guarded(nullptr, 0, [&] {
        const GridSpec g = to_grid(gg);
        const VolumePair pair(cells(g, iplus), cells(g, iminus));
        const DistanceEval de = distance(pair, faces(g, b), g_threads);
        copy_out(de.hessian_apply(faces(g, p), g_threads), out);
    });
}

int oracle_is_strictly_feasible(const epc_grid* gg, const double* b) {
    int res = 0;
    const int rc = guarded(nullptr, 0, [&] {
        const GridSpec g = to_grid(gg);
        res = is_strictly_feasible(faces(g, b)) ? 1 : 0;
    });
    return rc ? -rc : res;
}

} // extern "C"
