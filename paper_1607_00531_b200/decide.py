"""The ADMM loop's stop test and rho decision, certified against the
reference's sequential sums — the Python twin of csrc/admm_decide.h, used by
the slab-distributed host loop (dist_admm.py).

The reference sums the five non-negative dual-update terms sequentially in
index order (proj/src/admm.cpp:461-469, grid.cpp:60-64); the device (and the
rank-ordered gather of per-slab tree sums) sums the same rounded terms in
another order. For n non-negative terms every order is within gamma_{n-1}
of the exact sum, so the reference's value lies within [1-k, 1+k] times the
tree sum (k = 2.02 gamma_n + 8u). Every expression the decisions read is a
composition of correctly rounded monotone operations, so evaluating it at
both ends of the enclosure brackets the reference's rounded value; a
comparison whose brackets do not overlap is decided, otherwise the caller
recomputes the sums sequentially (rank by rank, in index order) and calls
`exact`.
"""
from __future__ import annotations

import math

NO, YES, UNKNOWN = 0, 1, 2


def enclose_seq(t, n):
    """(lo, hi) around the reference's sequential sum, or None."""
    if not math.isfinite(t):
        return None
    if t == 0.0:
        return 0.0, 0.0
    u = 2.0 ** -53
    nu = n * u
    if nu >= 0.01:
        return None
    g = nu / (1.0 - nu)
    k = 2.02 * g + 8.0 * u
    return math.nextafter(t * (1.0 - k), 0.0), math.nextafter(t * (1.0 + k), math.inf)


def residuals(s, rho, V, sqrt_n, eps_abs, eps_rel):
    """admm.cpp:470-474 on one set of the five sums -> (pr, du, eps_pri, eps_dual)."""
    pr = math.sqrt(s[0])
    du = rho * V * math.sqrt(s[1])
    nb, nz = math.sqrt(s[2]), math.sqrt(s[3])
    eps_pri = sqrt_n * eps_abs + eps_rel * (nz if nb < nz else nb)
    eps_dual = sqrt_n * eps_abs + eps_rel * rho * V * math.sqrt(s[4])
    return pr, du, eps_pri, eps_dual


def _le(alo, ahi, blo, bhi):
    if ahi <= blo:
        return YES
    if alo > bhi:
        return NO
    return UNKNOWN


def _gt(alo, ahi, blo, bhi):
    r = _le(alo, ahi, blo, bhi)
    return UNKNOWN if r == UNKNOWN else 1 - r


def certified(tree, n, rho, V, sqrt_n, eps_abs, eps_rel, mu, adaptive):
    """(converged, rho_move) from the tree sums, or None when undecidable."""
    lo, hi = [], []
    for t in tree[:5]:
        e = enclose_seq(t, n)
        if e is None:
            return None
        lo.append(e[0])
        hi.append(e[1])
    a = residuals(lo, rho, V, sqrt_n, eps_abs, eps_rel)
    b = residuals(hi, rho, V, sqrt_n, eps_abs, eps_rel)
    c1 = _le(a[0], b[0], a[2], b[2])
    c2 = _le(a[1], b[1], a[3], b[3])
    if c1 == YES and c2 == YES:
        return True, 0
    if not (c1 == NO or c2 == NO):
        return None
    if not adaptive:
        return False, 0
    r1 = _gt(a[0], b[0], mu * a[1], mu * b[1])
    if r1 == UNKNOWN:
        return None
    if r1 == YES:
        return False, 1
    r2 = _gt(a[1], b[1], mu * a[0], mu * b[0])
    if r2 == UNKNOWN:
        return None
    return False, (-1 if r2 == YES else 0)


def exact(seq, rho, V, sqrt_n, eps_abs, eps_rel, mu, adaptive):
    """The reference's decisions on its own sequential sums."""
    pr, du, ep, ed = residuals(seq, rho, V, sqrt_n, eps_abs, eps_rel)
    if pr <= ep and du <= ed:
        return True, 0
    if not adaptive:
        return False, 0
    if pr > mu * du:
        return False, 1
    if du > mu * pr:
        return False, -1
    return False, 0


def rho_apply(schedule, rho, rho_min, move, ti, td, fixed, bounded):
    """rho_schedule's arithmetic (admm.cpp:478-486) for a taken decision."""
    if schedule == fixed:
        return rho
    nxt = rho
    if move > 0:
        nxt = rho * ti
    elif move < 0:
        nxt = rho / td
    if schedule == bounded:
        nxt = rho_min if nxt < rho_min else nxt  # std::max(next, rho_min)
    return nxt
