// admm_decide.h — the ADMM loop's two scalar decisions (stop test and rho
// schedule, proj/src/admm.cpp:542-548 with :461-474 and :478-486), taken on
// the device's fixed-order tree sums but certified to be the ones the
// reference takes on its sequential sums.
//
// The reference forms five sums of non-negative terms sequentially in index
// order: pr = sum (b-z)^2, du = sum (z_old-z)^2 (dual_update_and_residuals,
// admm.cpp:461-469) and norm2(b), norm2(z), norm2(u) (grid.cpp:60-64). The
// device sums the very same rounded terms in a different order. For n
// non-negative terms any summation order has |s - S| <= gamma_{n-1} S
// (S the exact sum of the terms; additions never underflow inexactly), so
// the reference's value lies within a factor [1-k, 1+k] of the device's,
// k = 2.02 gamma_n + 8u. Every quantity the decisions read (sqrt, rho V *,
// eps_abs sqrt(n) + eps_rel max(..), mu *) is a composition of correctly
// rounded monotone operations, so evaluating it at both ends encloses the
// reference's rounded value. A comparison whose enclosures do not overlap
// is decided; otherwise the caller computes the five sequential sums
// exactly (k_seq_sums) and decides on those. Shared by the single-GPU loop
// (api.cu: on the host, or on the device in k_admm_decide) and the C++ slab
// loop (multi_gpu_host.inc). The same IEEE operations on host and device.
#pragma once

#include <cmath>
#include <limits>

#ifdef __CUDACC__
#define EPC_HD __host__ __device__
#else
#define EPC_HD
#endif

namespace epc_decide {

struct Iv {
    double lo, hi;
};

// Enclosure of the reference's sequential sum of n >= 1 non-negative terms
// from any-order sum t of the same terms. Returns false when t is not finite.
EPC_HD inline bool enclose_seq(double t, long long n, Iv* out) {
    if (!std::isfinite(t)) return false;
    if (t == 0.0) {  // non-negative terms: zero only if every term is zero
        *out = {0.0, 0.0};
        return true;
    }
    const double u = 0x1p-53;
    const double nu = (double)n * u;
    if (nu >= 0.01) return false;
    const double g = nu / (1.0 - nu);
    const double k = 2.02 * g + 8.0 * u;
    out->lo = std::nextafter(t * (1.0 - k), 0.0);
    out->hi = std::nextafter(t * (1.0 + k), HUGE_VAL);
    return true;
}

// The reference's residual/tolerance expressions (admm.cpp:470-474) on one
// set of the five sums.
struct Res {
    double pr, du, eps_pri, eps_dual;
};
EPC_HD inline Res residuals(const double s[5], double rho, double V, double sqrt_n, double eps_abs,
                     double eps_rel) {
    Res r;
    r.pr = std::sqrt(s[0]);
    r.du = rho * V * std::sqrt(s[1]);
    const double nb = std::sqrt(s[2]), nz = std::sqrt(s[3]);
    r.eps_pri = sqrt_n * eps_abs + eps_rel * ((nb < nz) ? nz : nb);  // std::max(nb, nz)
    r.eps_dual = sqrt_n * eps_abs + eps_rel * rho * V * std::sqrt(s[4]);
    return r;
}

enum { NO = 0, YES = 1, UNKNOWN = 2 };

// Three-valued a <= b and a > b from enclosures.
EPC_HD inline int le(double a_lo, double a_hi, double b_lo, double b_hi) {
    if (a_hi <= b_lo) return YES;
    if (a_lo > b_hi) return NO;
    return UNKNOWN;
}
EPC_HD inline int gt(double a_lo, double a_hi, double b_lo, double b_hi) {
    const int r = le(a_lo, a_hi, b_lo, b_hi);
    return r == UNKNOWN ? UNKNOWN : 1 - r;
}

struct Decision {
    bool decided;    // false: recompute the sums sequentially and call exact()
    bool converged;  // admm.cpp:542
    int rho_move;    // +1: rho * tau_incr, -1: rho / tau_decr, 0: unchanged (before the clamp)
};

// Certified decisions from the device's five tree sums.
EPC_HD inline Decision certified(const double tree[5], long long n, double rho, double V, double sqrt_n,
                          double eps_abs, double eps_rel, double mu, bool adaptive) {
    Decision d{false, false, 0};
    double lo[5], hi[5];
    for (int i = 0; i < 5; ++i) {
        Iv v;
        if (!enclose_seq(tree[i], n, &v)) return d;
        lo[i] = v.lo;
        hi[i] = v.hi;
    }
    const Res a = residuals(lo, rho, V, sqrt_n, eps_abs, eps_rel);
    const Res b = residuals(hi, rho, V, sqrt_n, eps_abs, eps_rel);
    const int c1 = le(a.pr, b.pr, a.eps_pri, b.eps_pri);
    const int c2 = le(a.du, b.du, a.eps_dual, b.eps_dual);
    if (c1 == YES && c2 == YES) {
        d.decided = d.converged = true;
        return d;
    }
    if (!(c1 == NO || c2 == NO)) return d;  // undecided stop test
    if (!adaptive) {
        d.decided = true;
        return d;
    }
    // rho_schedule (admm.cpp:482-483): pr > mu*du, else du > mu*pr
    const int r1 = gt(a.pr, b.pr, mu * a.du, mu * b.du);
    if (r1 == UNKNOWN) return d;
    if (r1 == YES) {
        d.decided = true;
        d.rho_move = 1;
        return d;
    }
    const int r2 = gt(a.du, b.du, mu * a.pr, mu * b.pr);
    if (r2 == UNKNOWN) return d;
    d.decided = true;
    d.rho_move = r2 == YES ? -1 : 0;
    return d;
}

// The reference's decisions on exact sequential sums (the fallback).
EPC_HD inline Decision exact(const double seq[5], double rho, double V, double sqrt_n, double eps_abs,
                      double eps_rel, double mu, bool adaptive) {
    const Res r = residuals(seq, rho, V, sqrt_n, eps_abs, eps_rel);
    Decision d{true, false, 0};
    if (r.pr <= r.eps_pri && r.du <= r.eps_dual) {
        d.converged = true;
        return d;
    }
    if (!adaptive) return d;
    if (r.pr > mu * r.du) d.rho_move = 1;
    else if (r.du > mu * r.pr) d.rho_move = -1;
    return d;
}

}  // namespace epc_decide
