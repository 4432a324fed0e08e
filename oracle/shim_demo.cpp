// shim_demo.cpp — TEST INFRASTRUCTURE: drives the reference's own public
// API (simulate_pair, admm_solve, gauss_newton_solve, multilevel_solve) on
// a small synthetic problem and writes the fields to a binary file.
//
// Built twice by oracle/Makefile (target `shim`):
//   _ref/ref_demo   all reference translation units (CPU reference);
//   _ref/shim_demo  the same, with the solver entry points taken from
//                   paper_1607_00531_b200/shim/epicorr_b200_shim.cpp (GPU),
//                   i.e. the drop-in: multilevel.cpp links unchanged.
// tests/test_gpu_shim.py runs both and compares their outputs.
#include <cstdio>
#include <vector>

#include "epicorr/admm.hpp"
#include "epicorr/gn_pcg.hpp"
#include "epicorr/image.hpp"
#include "epicorr/multilevel.hpp"
#include "epicorr/objective.hpp"

using namespace epicorr;

static void put(std::FILE* f, const std::vector<double>& v) {
    const long long n = (long long)v.size();
    std::fwrite(&n, sizeof n, 1, f);
    std::fwrite(v.data(), sizeof(double), v.size(), f);
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const GridSpec g = GridSpec::make3d(24, 20, 12);
    const ImageVolume truth = phantom_gaussian(g);
    const StaggeredField bt = bump_field(g, 0.4);
    SimulateOptions so;
    so.noise_sigma = 2.0;
    so.seed = 7;
    const VolumePair pair = simulate_pair(truth, bt, so);
    const ObjectiveParams p;
    ADMMConfig ac;
    ac.max_iter = 15;
    ac.eps_abs = ac.eps_rel = 1e-300;
    GNConfig gc;
    gc.eta = 1e-2;
    gc.max_pcg = 40;
    gc.max_outer = 5;

    std::FILE* f = std::fopen(argv[1], "wb");
    if (!f) return 3;
    // single-level ADMM and GN
    const AdmmSolveResult a = admm_solve(pair, ADMMState{}, p, ac, 0);
    put(f, a.state.b.v);
    put(f, a.state.z.v);
    put(f, a.state.u.v);
    std::vector<double> lag;
    for (const auto& r : a.report.admm) lag.push_back(r.lagrangian);
    put(f, lag);
    const GnSolveResult gsol = gauss_newton_solve(pair, StaggeredField(g), p, gc, 0);
    put(f, gsol.b.v);
    // the reference's coarse-to-fine driver, unchanged, over both solvers
    const LevelSchedule s = default_schedule(g, 2, 8);
    const MultilevelResult ma = multilevel_solve(pair, s, SolverKind::admm, p, gc, ac);
    put(f, ma.b.v);
    const MultilevelResult mg = multilevel_solve(pair, s, SolverKind::gn, p, gc, ac);
    put(f, mg.b.v);
    std::vector<double> meta{double(a.report.stop), double(gsol.report.stop), double(ma.report.stop),
                             double(mg.report.stop), double(ma.report.admm.size()),
                             double(mg.report.gn.size())};
    put(f, meta);
    // the GN building blocks (objective_gn, GnHessian, make_preconditioner)
    // driven through the reference's own generic pcg (gn_pcg.cpp:92-131)
    // a feasible, nonzero field that both builds hold bitwise (the ADMM
    // result is bitwise; halving it is exact and keeps |D1 b| < 1)
    StaggeredField bq = a.state.b;
    for (double& v : bq.v) v *= 0.5;
    const ObjectiveEval ev = objective_gn(pair, bq, p);
    put(f, ev.grad.v);
    put(f, ev.residual.v);
    put(f, {ev.value, ev.dist, ev.smooth, ev.pen, double(ev.feasible)});
    const GnHessian H(pair, bq, p);
    put(f, H.apply(ev.grad).v);
    put(f, H.preconditioner_blocks().diag);
    put(f, H.full_diagonal());
    const LinOp ah = [&](const std::vector<double>& x, std::vector<double>& y) {
        y.resize(x.size());
        H.apply(x, y);
    };
    for (PrecondKind kind : {PrecondKind::none, PrecondKind::jacobi, PrecondKind::block_jacobi,
                             PrecondKind::sgs}) {
        const LinOp m = make_preconditioner(kind, H);
        std::vector<double> z;
        m(ev.grad.v, z);
        put(f, z);
        const PcgResult pr = pcg(ah, m, ev.grad.v, 1e-3, 30);
        put(f, pr.d);
        put(f, {double(pr.iters), pr.relres, pr.relres_prec});
    }
    {  // dense() on a small grid (diagnostics)
        const GridSpec gs = GridSpec::make3d(6, 5, 4);
        SimulateOptions o2;
        o2.seed = 3;
        const VolumePair ps = simulate_pair(phantom_gaussian(gs), bump_field(gs, 0.3), o2);
        const GnHessian Hs(ps, StaggeredField(gs), p);
        put(f, Hs.dense());
    }
    // an infeasible point: +inf, no gradient
    {
        StaggeredField bad(g);
        bad.v[1] = 5.0;
        const ObjectiveEval e2 = objective_gn(pair, bad, p);
        put(f, {e2.value, double(e2.feasible), double(e2.grad.v.size()), double(e2.residual.v.size())});
    }
    std::fclose(f);
    std::printf("ok %zu admm rows, %zu ml-admm rows, %zu ml-gn rows\n", a.report.admm.size(),
                ma.report.admm.size(), mg.report.gn.size());
    return 0;
}
