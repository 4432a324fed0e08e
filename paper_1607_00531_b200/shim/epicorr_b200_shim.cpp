// epicorr_b200_shim.cpp — C++ drop-in for the reference solver API.
//
// Compiled against the reference's own headers (proj/include/epicorr), this
// translation unit defines the reference's solver entry points on top of
// the C ABI of libepicorr_b200.so:
//
//   admm_solve                (proj/include/epicorr/admm.hpp:127-129)
//   b_update                  (admm.hpp:100-102)
//   z_update                  (admm.hpp:105)
//   dual_update_and_residuals (admm.hpp:113-115)
//   augmented_lagrangian      (admm.hpp:87-89)
//   qp_active_set             (admm.hpp:74-76)
//   gauss_newton_solve        (proj/include/epicorr/gn_pcg.hpp:81-83)
//   objective_gn              (proj/include/epicorr/objective.hpp:93-94)
//   GnHessian                 (objective.hpp:99-131: ctor, apply, cross_diag,
//                              preconditioner_blocks, full_diagonal, dense)
//   make_preconditioner       (gn_pcg.hpp:47; none / jacobi / block_jacobi on
//                              the device; sgs, sequential by design and out
//                              of this build's scope, stays the reference's)
//   multilevel_solve, restrict_image, prolong_field (multilevel.hpp)
//
// with the same signatures, ownership and exception behaviour (the C ABI's
// status codes are rethrown as std::invalid_argument / std::runtime_error /
// std::domain_error with the reference's message text). A maintainer links
// it in place of the reference's definitions of those functions; every other
// reference translation unit (multilevel.cpp, the CLI, the tests) links
// unchanged. INTEGRATION.md gives the recipe (the reference's admm.cpp /
// gn_pcg.cpp / objective.cpp stay in the build for their generic helpers,
// with the replaced symbols renamed by -D at compile time; objective.cpp's
// GnHessian becomes ref_cpu_GnHessian there, and the shim defines the class's
// members on the device).
//
// Device: EPICORR_B200_DEVICE (default 0); one context per process, created
// on first use, owning its stream. Threading: the reference's free functions
// may be called from several host threads at once; every entry point here
// holds one process-wide lock for its whole call (the context's scratch
// slots, pinned staging and stream are shared), so concurrent callers are
// serialised on the one device instead of corrupting each other.
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "epicorr/admm.hpp"
#include "epicorr/gn_pcg.hpp"
#include "epicorr/objective.hpp"
#include "epicorr/multilevel.hpp"
#include "epicorr_b200.h"

namespace {

std::recursive_mutex& shim_mutex() {
    static std::recursive_mutex m;
    return m;
}
#define SHIM_LOCK std::lock_guard<std::recursive_mutex> shim_lock_(shim_mutex())

epc_context* ctx() {
    static std::once_flag once;
    static epc_context* c = nullptr;
    static int rc = 0;
    std::call_once(once, [] {
        const char* dv = std::getenv("EPICORR_B200_DEVICE");
        rc = epc_context_create(dv ? std::atoi(dv) : 0, nullptr, &c);
    });
    if (!c) throw std::runtime_error("epicorr_b200: no usable B200 device (status " + std::to_string(rc) + ")");
    return c;
}

[[noreturn]] void rethrow(int code, const std::string& msg) {
    switch (code) {
        case EPC_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case EPC_ERR_DOMAIN: throw std::domain_error(msg);
        default: throw std::runtime_error(msg);
    }
}

void check(int code) {
    if (code != EPC_OK) rethrow(code, epc_last_error(ctx()));
}

epc_grid to_c(const epicorr::GridSpec& g) {
    epc_grid o;
    o.dim = g.dim;
    for (int a = 0; a < 3; ++a) {
        o.m[a] = g.m[a];
        o.h[a] = g.h[a];
        o.origin[a] = g.origin[a];
    }
    return o;
}

epc_objective_params to_c(const epicorr::ObjectiveParams& p) {
    return epc_objective_params{p.alpha, p.beta, p.gamma, p.enforce_linf_box ? 1 : 0};
}

epc_admm_config to_c(const epicorr::ADMMConfig& c) {
    epc_admm_config o;
    o.rho0 = c.rho0;
    o.rho_min = c.rho_min;
    o.schedule = int(c.schedule);
    o.eps_abs = c.eps_abs;
    o.eps_rel = c.eps_rel;
    o.max_iter = c.max_iter;
    o.tau_incr = c.tau_incr;
    o.tau_decr = c.tau_decr;
    o.mu = c.mu;
    o.sqp_max_iter = c.sqp_max_iter;
    o.sqp_tol_rel = c.sqp_tol_rel;
    o.check_kkt = c.check_kkt ? 1 : 0;
    o.threads = c.threads;
    return o;
}

epc_gn_config to_c(const epicorr::GNConfig& c) {
    epc_gn_config o;
    o.eta = c.eta;
    o.max_outer = c.max_outer;
    o.eps_obj = c.eps_obj;
    o.eps_iter = c.eps_iter;
    o.eps_grad = c.eps_grad;
    o.wolfe_c1 = c.wolfe_c1;
    o.wolfe_c2 = c.wolfe_c2;
    o.max_pcg = c.max_pcg;
    o.max_ls = c.max_ls;
    o.precond = int(c.precond);
    o.threads = c.threads;
    return o;
}

const double* data_or_null(const epicorr::StaggeredField& f) { return f.v.empty() ? nullptr : f.v.data(); }

}  // namespace

namespace epicorr {

AdmmSolveResult admm_solve(const VolumePair& pair, ADMMState init, const ObjectiveParams& params,
                           const ADMMConfig& config, int level_tag) {
    SHIM_LOCK;
    const GridSpec& g = pair.grid();
    const epc_grid cg = to_c(g);
    const epc_objective_params cp = to_c(params);
    const epc_admm_config cc = to_c(config);
    // admm.cpp:490-498, in the reference's order (a field on another grid
    // would otherwise be over-read by the ABI)
    params.validate();
    config.validate();
    if ((!init.b.v.empty() && !(init.b.grid == g)) || (!init.z.v.empty() && !(init.z.grid == g)) ||
        (!init.u.v.empty() && !(init.u.grid == g)))
        throw std::invalid_argument("admm_solve: state grids do not match the pair");
    AdmmSolveResult out;
    out.state.b = StaggeredField(g);
    out.state.z = StaggeredField(g);
    out.state.u = StaggeredField(g);
    double rho = init.rho;
    std::vector<epc_admm_row> rows(std::max(config.max_iter, 1));
    epc_solve_status st{};
    const int rc = epc_admm_solve(ctx(), &cg, EPC_MEM_HOST, pair.plus.v.data(), pair.minus.v.data(),
                                  data_or_null(init.b), data_or_null(init.z), data_or_null(init.u),
                                  out.state.b.v.data(), out.state.z.v.data(), out.state.u.v.data(),
                                  &rho, &cp, &cc, level_tag, rows.data(), int(rows.size()), &st);
    if (rc != EPC_OK) rethrow(rc, st.message[0] ? st.message : epc_last_error(ctx()));
    out.state.rho = rho;
    out.state.iter = st.nrows;
    const int n = std::min<int>(st.nrows, int(rows.size()));
    for (int i = 0; i < n; ++i) {
        const epc_admm_row& r = rows[i];
        AdmmIterRow row;
        row.level = r.level;
        row.iter = r.iter;
        row.primal_res = r.primal_res;
        row.dual_res = r.dual_res;
        row.eps_pri = r.eps_pri;
        row.eps_dual = r.eps_dual;
        row.rho = r.rho;
        row.lagrangian = r.lagrangian;
        row.kkt_violation = r.kkt_violation;
        row.b_update_s = r.b_update_s;
        row.wall_s = r.wall_s;
        out.report.admm.push_back(row);
    }
    if (n > 0) out.state.lagrangian = rows[n - 1].lagrangian;
    out.report.stop = StopReason(st.stop);
    out.report.message = st.message;
    return out;
}

StaggeredField b_update(const VolumePair& pair, const ADMMState& state, const ObjectiveParams& params,
                        const ADMMConfig& config, BUpdateStats* stats) {
    SHIM_LOCK;
    const GridSpec& g = pair.grid();
    if (!(state.b.grid == g) || !(state.z.grid == g) || !(state.u.grid == g))
        throw std::invalid_argument("b_update: state grids do not match the pair");
    const epc_grid cg = to_c(g);
    const epc_objective_params cp = to_c(params);
    const epc_admm_config cc = to_c(config);
    StaggeredField out(g);
    epc_bupdate_stats s{};
    check(epc_b_update(ctx(), &cg, EPC_MEM_HOST, pair.plus.v.data(), pair.minus.v.data(),
                       state.b.v.data(), state.z.v.data(), state.u.v.data(), state.rho, &cp, &cc,
                       out.v.data(), &s));
    if (stats) {
        stats->sqp_iters += s.sqp_iters;
        stats->qp_iters += s.qp_iters;
        stats->kkt_violation = std::max(stats->kkt_violation, s.kkt_violation);
    }
    return out;
}

StaggeredField z_update(const ADMMState& state, double alpha, const DctCoupledSolver&) {
    SHIM_LOCK;
    const GridSpec& g = state.b.grid;
    const epc_grid cg = to_c(g);
    StaggeredField out(g);
    check(epc_z_update(ctx(), &cg, EPC_MEM_HOST, state.b.v.data(), state.u.v.data(), state.rho,
                       alpha, out.v.data()));
    return out;
}

DualUpdate dual_update_and_residuals(const StaggeredField& b_new, const StaggeredField& z_new,
                                     const StaggeredField& z_old, const StaggeredField& u_old,
                                     double rho, double eps_abs, double eps_rel) {
    SHIM_LOCK;
    const GridSpec& g = b_new.grid;
    if (!(z_new.grid == g) || !(z_old.grid == g) || !(u_old.grid == g))
        throw std::invalid_argument("dual_update_and_residuals: grid mismatch");
    const epc_grid cg = to_c(g);
    DualUpdate out;
    out.u = StaggeredField(g);
    epc_dual_result r{};
    check(epc_dual_update(ctx(), &cg, EPC_MEM_HOST, b_new.v.data(), z_new.v.data(), z_old.v.data(),
                          u_old.v.data(), rho, eps_abs, eps_rel, out.u.v.data(), &r));
    out.primal_res = r.primal_res;
    out.dual_res = r.dual_res;
    out.eps_pri = r.eps_pri;
    out.eps_dual = r.eps_dual;
    return out;
}

double augmented_lagrangian(const VolumePair& pair, const StaggeredField& b, const StaggeredField& z,
                            const StaggeredField& u, double rho, double alpha, int) {
    SHIM_LOCK;
    const epc_grid cg = to_c(pair.grid());
    double v = 0.0;
    check(epc_augmented_lagrangian(ctx(), &cg, EPC_MEM_HOST, pair.plus.v.data(),
                                   pair.minus.v.data(), b.v.data(), z.v.data(), u.v.data(), rho,
                                   alpha, &v));
    return v;
}

QpResult qp_active_set(int n, double h, std::span<const double> gdiag, std::span<const double> goff,
                       std::span<const double> c, std::span<const double> x0, int max_iter) {
    SHIM_LOCK;
    QpResult r;
    r.x.assign(n, 0.0);
    r.lambda.assign(n - 1, 0.0);
    r.active_sign.assign(n - 1, 0);
    int iters = 0, status = 0;
    double kkt = 0.0;
    check(epc_qp_active_set_batch(ctx(), 1, n, h, gdiag.data(), goff.data(), c.data(), x0.data(),
                                  max_iter, r.x.data(), r.lambda.data(), r.active_sign.data(), &iters,
                                  &kkt, &status));
    if (status != EPC_OK) rethrow(status, epc_last_error(ctx()));
    r.iters = iters;
    return r;
}

GnSolveResult gauss_newton_solve(const VolumePair& pair, const StaggeredField& b0,
                                 const ObjectiveParams& params, const GNConfig& config,
                                 int level_tag) {
    SHIM_LOCK;
    const GridSpec& g = pair.grid();
    if (!(b0.grid == g)) throw std::invalid_argument("gauss_newton_solve: grid mismatch");
    const epc_grid cg = to_c(g);
    const epc_objective_params cp = to_c(params);
    const epc_gn_config cc = to_c(config);
    GnSolveResult out;
    out.b = StaggeredField(g);
    std::vector<epc_gn_row> rows(config.max_outer + 1);
    epc_solve_status st{};
    const int rc = epc_gn_solve(ctx(), &cg, EPC_MEM_HOST, pair.plus.v.data(), pair.minus.v.data(),
                                b0.v.data(), out.b.v.data(), &cp, &cc, level_tag, rows.data(),
                                int(rows.size()), &st);
    if (rc != EPC_OK) rethrow(rc, epc_last_error(ctx()));
    const int n = std::min<int>(st.nrows, int(rows.size()));
    for (int i = 0; i < n; ++i) {
        const epc_gn_row& r = rows[i];
        out.report.gn.push_back(GnIterRow{r.level, r.iter, r.j_value, r.grad_norm, r.step,
                                          r.pcg_iters, r.pcg_relres, r.pcg_relres_prec, r.wall_s});
    }
    out.report.stop = StopReason(st.stop);
    out.report.message = st.message;
    return out;
}


// ---- GN building blocks (objective.hpp:93-131, gn_pcg.hpp:47) ----------------

ObjectiveEval objective_gn(const VolumePair& pair, const StaggeredField& b, const ObjectiveParams& p,
                           int, bool need_grad) {
    SHIM_LOCK;
    p.validate();
    const GridSpec& g = pair.grid();
    if (!(b.grid == g)) throw std::invalid_argument("objective_gn: field grid mismatch");
    const epc_grid cg = to_c(g);
    const epc_objective_params cp = to_c(p);
    std::vector<double> grad(g.faces()), res(g.cells());
    epc_objective_eval ev{};
    check(epc_objective_gn(ctx(), &cg, EPC_MEM_HOST, pair.plus.v.data(), pair.minus.v.data(),
                           b.v.data(), &cp, need_grad ? 1 : 0, &ev, grad.data(), res.data()));
    ObjectiveEval out;
    out.value = ev.value;
    out.dist = ev.dist;
    out.smooth = ev.smooth;
    out.pen = ev.pen;
    out.feasible = ev.feasible != 0;
    if (out.feasible) {  // objective.cpp:241-263: residual always, grad on request
        out.residual = CellField(g);
        out.residual.v = std::move(res);
        if (need_grad) {
            out.grad = StaggeredField(g);
            out.grad.v = std::move(grad);
        }
    }
    return out;
}

GnHessian::GnHessian(const VolumePair& pair, const StaggeredField& b, const ObjectiveParams& p,
                     int threads)
    : grid_(pair.grid()), col_(pair.grid()), threads_(threads) {
    SHIM_LOCK;
    p.validate();
    const double V = grid_.cell_volume();
    w2_ = p.alpha * V / (grid_.h[1] * grid_.h[1]);  // objective.cpp:271-272
    w3_ = grid_.dim == 3 ? p.alpha * V / (grid_.h[2] * grid_.h[2]) : 0.0;
    const epc_grid cg = to_c(grid_);
    const epc_objective_params cp = to_c(p);
    check(epc_gn_hessian_build(ctx(), &cg, EPC_MEM_HOST, pair.plus.v.data(), pair.minus.v.data(),
                               b.v.data(), &cp, col_.diag.data(), col_.off.data(), nullptr));
}

double GnHessian::cross_diag(int j, int k) const {  // objective.cpp:296-300 (a scalar)
    double d = w2_ * ((j == 0 || j == grid_.m[1] - 1) ? 1.0 : 2.0);
    if (grid_.dim == 3) d += w3_ * ((k == 0 || k == grid_.m[2] - 1) ? 1.0 : 2.0);
    return d;
}

void GnHessian::apply(std::span<const double> x, std::span<double> y) const {
    SHIM_LOCK;
    const epc_grid cg = to_c(grid_);
    check(epc_gn_stencil_apply(ctx(), &cg, EPC_MEM_HOST, col_.diag.data(), col_.off.data(), w2_, w3_,
                               x.data(), y.data()));
}

StaggeredField GnHessian::apply(const StaggeredField& x) const {
    StaggeredField out(grid_);
    apply(x.v, out.v);
    return out;
}

TridiagBlocks GnHessian::preconditioner_blocks() const {
    SHIM_LOCK;
    TridiagBlocks t = col_;
    const epc_grid cg = to_c(grid_);
    check(epc_gn_cross_diag_add(ctx(), &cg, EPC_MEM_HOST, col_.diag.data(), w2_, w3_, t.diag.data()));
    return t;
}

std::vector<double> GnHessian::full_diagonal() const {
    SHIM_LOCK;
    std::vector<double> d(col_.diag.size());
    const epc_grid cg = to_c(grid_);
    check(epc_gn_cross_diag_add(ctx(), &cg, EPC_MEM_HOST, col_.diag.data(), w2_, w3_, d.data()));
    return d;
}

// Dense row-major assembly for small-problem diagnostics (objective.cpp:
// 350-384): the values are the device's (full_diagonal, the column part's
// off-diagonals, the cross weights); the host only places them.
std::vector<double> GnHessian::dense() const {
    const std::int64_t n = grid_.faces();
    const int n1 = grid_.n1(), m2 = grid_.m[1], m3 = grid_.m[2];
    const std::vector<double> dg = full_diagonal();
    std::vector<double> a(std::size_t(n) * n, 0.0);
    const std::int64_t layer = std::int64_t(n1) * m2;
    for (std::int64_t f = 0; f < n; ++f) {
        const std::int64_t c = f / n1;
        const int i = int(f % n1), j = int(c % m2), k = int(c / m2);
        a[std::size_t(f) * n + f] = dg[f];
        if (i + 1 < n1) {
            a[std::size_t(f) * n + f + 1] = col_.off[f];
            a[std::size_t(f + 1) * n + f] = col_.off[f];
        }
        if (j > 0) a[std::size_t(f) * n + (f - n1)] = -w2_;
        if (j + 1 < m2) a[std::size_t(f) * n + (f + n1)] = -w2_;
        if (m3 > 1) {
            if (k > 0) a[std::size_t(f) * n + (f - layer)] = -w3_;
            if (k + 1 < m3) a[std::size_t(f) * n + (f + layer)] = -w3_;
        }
    }
    return a;
}

// the reference's own make_preconditioner (gn_pcg.cpp, compiled renamed):
// the symmetric Gauss-Seidel sweeps are sequential by design
LinOp ref_cpu_make_preconditioner(PrecondKind kind, const GnHessian& h, int threads);

LinOp make_preconditioner(PrecondKind kind, const GnHessian& h, int threads) {
    switch (kind) {
        case PrecondKind::none:
            return [](const std::vector<double>& r, std::vector<double>& z) { z = r; };
        case PrecondKind::jacobi: {  // gn_pcg.cpp:41-47
            auto diag = h.full_diagonal();
            return [diag](const std::vector<double>& r, std::vector<double>& z) {
                SHIM_LOCK;
                z.resize(r.size());
                check(epc_jacobi_apply(ctx(), (long long)r.size(), EPC_MEM_HOST, diag.data(), r.data(),
                                       z.data()));
            };
        }
        case PrecondKind::block_jacobi: {  // gn_pcg.cpp:48-54
            const TridiagBlocks t = h.preconditioner_blocks();
            const epc_grid cg = to_c(h.grid());
            {
                // TridiagFactor::factorize throws here (operators.cpp:230-240), not at apply
                SHIM_LOCK;
                std::vector<double> zero(t.diag.size(), 0.0), x(t.diag.size());
                check(epc_tridiag_solve_batched(ctx(), &cg, EPC_MEM_HOST, t.diag.data(), t.off.data(),
                                                zero.data(), x.data()));
            }
            return [t, cg](const std::vector<double>& r, std::vector<double>& z) {
                SHIM_LOCK;
                z.resize(r.size());
                check(epc_tridiag_solve_batched(ctx(), &cg, EPC_MEM_HOST, t.diag.data(), t.off.data(),
                                                r.data(), z.data()));
            };
        }
        case PrecondKind::sgs:
            return ref_cpu_make_preconditioner(kind, h, threads);
    }
    throw std::logic_error("make_preconditioner: bad kind");
}

// ---- multilevel (multilevel.hpp:37-63) on the device --------------------------
ImageVolume restrict_image(const ImageVolume& img, const GridSpec& coarse) {
    SHIM_LOCK;
    const epc_grid cf = to_c(img.grid), cc = to_c(coarse);
    coarse.validate();
    ImageVolume out(coarse);
    check(epc_restrict_image(ctx(), &cf, &cc, EPC_MEM_HOST, img.v.data(), out.v.data()));
    return out;
}

StaggeredField prolong_field(const StaggeredField& b_coarse, const GridSpec& fine) {
    SHIM_LOCK;
    const epc_grid cc = to_c(b_coarse.grid), cf = to_c(fine);
    fine.validate();
    StaggeredField out(fine);
    check(epc_prolong_field(ctx(), &cc, &cf, EPC_MEM_HOST, b_coarse.v.data(), out.v.data()));
    return out;
}

MultilevelResult multilevel_solve(const VolumePair& pair, const LevelSchedule& schedule,
                                  SolverKind solver, const ObjectiveParams& params,
                                  const GNConfig& gn_config, const ADMMConfig& admm_config,
                                  AdmmRestart restart) {
    SHIM_LOCK;
    schedule.validate();
    const int nlev = schedule.levels();
    std::vector<epc_grid> lv;
    for (const GridSpec& g : schedule.grids) lv.push_back(to_c(g));
    std::vector<int> gmo, ami;
    int cap_g = 0, cap_a = 0;
    for (int l = 0; l < nlev; ++l) {
        const bool has = !schedule.overrides.empty();
        gmo.push_back(has && schedule.overrides[l].gn_max_outer ? *schedule.overrides[l].gn_max_outer : -1);
        ami.push_back(has && schedule.overrides[l].admm_max_iter ? *schedule.overrides[l].admm_max_iter : -1);
        cap_g += (gmo.back() >= 0 ? gmo.back() : gn_config.max_outer) + 1;
        cap_a += (ami.back() >= 0 ? ami.back() : admm_config.max_iter) + 1;
    }
    const epc_grid cg = to_c(pair.grid());
    const epc_objective_params cp = to_c(params);
    const epc_gn_config gc = to_c(gn_config);
    const epc_admm_config ac = to_c(admm_config);
    std::vector<epc_admm_row> arows(cap_a);
    std::vector<epc_gn_row> grows(cap_g);
    std::vector<double> b(pair.grid().faces());
    epc_multilevel_status st{};
    const int rc = epc_multilevel_solve(
        ctx(), &cg, EPC_MEM_HOST, pair.plus.v.data(), pair.minus.v.data(), lv.data(), nlev,
        gmo.data(), ami.data(), solver == SolverKind::gn ? EPC_SOLVER_GN : EPC_SOLVER_ADMM, &cp,
        &gc, &ac, int(restart), b.data(), arows.data(), cap_a, grows.data(), cap_g, &st);
    if (rc != EPC_OK) rethrow(rc, st.message[0] ? st.message : epc_last_error(ctx()));
    MultilevelResult out;
    out.b = StaggeredField(schedule.grids[st.b_level]);
    std::memcpy(out.b.v.data(), b.data(), sizeof(double) * out.b.v.size());
    for (int i = 0; i < std::min(st.n_gn_rows, cap_g); ++i) {
        const epc_gn_row& r = grows[i];
        out.report.gn.push_back(GnIterRow{r.level, r.iter, r.j_value, r.grad_norm, r.step,
                                          r.pcg_iters, r.pcg_relres, r.pcg_relres_prec, r.wall_s});
    }
    for (int i = 0; i < std::min(st.n_admm_rows, cap_a); ++i) {
        const epc_admm_row& r = arows[i];
        out.report.admm.push_back(AdmmIterRow{r.level, r.iter, r.primal_res, r.dual_res, r.eps_pri,
                                              r.eps_dual, r.rho, r.lagrangian, r.kkt_violation,
                                              r.b_update_s, r.wall_s});
    }
    out.report.stop = StopReason(st.stop);
    out.report.message = st.message;
    return out;
}

}  // namespace epicorr
