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
    std::fclose(f);
    std::printf("ok %zu admm rows, %zu ml-admm rows, %zu ml-gn rows\n", a.report.admm.size(),
                ma.report.admm.size(), mg.report.gn.size());
    return 0;
}
