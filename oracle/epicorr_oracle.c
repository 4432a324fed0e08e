/*
 * epicorr_oracle.c — TEST INFRASTRUCTURE ONLY: the CPU checker for the
 * B200 hot path. Never linked into, loaded by, or called from the product
 * (paper_1607_00531_b200/); only tests/, __graft_entry__.smoke() and the
 * CPU legs of bench.py may load it.
 *
 * A plain-C restatement of the reference epicorr solver path (ADMM and
 * GN-PCG per-iteration work). Every function cites the reference lines it
 * restates (paths under /root/reference/proj). Operation order and
 * association follow the reference expression by expression, and the build
 * pins -ffp-contract=off like the reference's Release build, so results are
 * bitwise those of the reference library; tests/test_oracle_pin.py checks
 * that against oracle/_ref (the reference compiled from its own sources) and
 * against the committed fixtures in tests/golden/.
 *
 * Error handling restates the reference's exceptions as EPC_* codes plus
 * the e.what() text.
 */
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "oracle_api.h"

#define PI_D 3.141592653589793238462643383279502884 /* std::numbers::pi */

typedef struct {
    int dim, m1, m2, m3, n1;
    long long ncell, nface, ncol;
    double h1, h2, h3, o1, o2, o3, V;
} G;

static void set_msg(char* msg, size_t len, const char* fmt, ...) {
    if (!msg || len == 0) return;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(msg, len, fmt, ap);
    va_end(ap);
}

/* GridSpec::validate, grid.cpp:33-47 */
static int grid_make(const epc_grid* g, G* out, char* msg, size_t len) {
    if (g->dim != 2 && g->dim != 3) {
        set_msg(msg, len, "GridSpec: dim must be 2 or 3");
        return EPC_ERR_INVALID_ARGUMENT;
    }
    if (g->m[0] < 2 || g->m[1] < 2) {
        set_msg(msg, len, "GridSpec: m1 and m2 must be >= 2");
        return EPC_ERR_INVALID_ARGUMENT;
    }
    if (g->dim == 3 && g->m[2] < 2) {
        set_msg(msg, len, "GridSpec: m3 must be >= 2 in 3D");
        return EPC_ERR_INVALID_ARGUMENT;
    }
    if (g->dim == 2 && g->m[2] != 1) {
        set_msg(msg, len, "GridSpec: m3 must be 1 in 2D");
        return EPC_ERR_INVALID_ARGUMENT;
    }
    for (int a = 0; a < 3; ++a) {
        if (!(g->h[a] > 0.0) || !isfinite(g->h[a])) {
            set_msg(msg, len, "GridSpec: spacings must be positive");
            return EPC_ERR_INVALID_ARGUMENT;
        }
        if (!isfinite(g->origin[a])) {
            set_msg(msg, len, "GridSpec: origin must be finite");
            return EPC_ERR_INVALID_ARGUMENT;
        }
    }
    out->dim = g->dim;
    out->m1 = g->m[0];
    out->m2 = g->m[1];
    out->m3 = g->m[2];
    out->n1 = g->m[0] + 1;
    out->ncell = (long long)g->m[0] * g->m[1] * g->m[2];
    out->nface = (long long)(g->m[0] + 1) * g->m[1] * g->m[2];
    out->ncol = (long long)g->m[1] * g->m[2];
    out->h1 = g->h[0];
    out->h2 = g->h[1];
    out->h3 = g->h[2];
    out->o1 = g->origin[0];
    out->o2 = g->origin[1];
    out->o3 = g->origin[2];
    out->V = g->h[0] * g->h[1] * g->h[2]; /* cell_volume, grid.hpp:35 */
    return EPC_OK;
}

static double* dalloc(long long n) { return (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double)); }

/* ---- sequential vector helpers, grid.cpp:60-80 ------------------------- */
static double vdot(const double* a, const double* b, long long n) {
    double s = 0.0;
    for (long long i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}
static double vnorm2(const double* a, long long n) { return sqrt(vdot(a, a, n)); }
static double vnorm_inf(const double* a, long long n) {
    double s = 0.0;
    for (long long i = 0; i < n; ++i) {
        const double x = fabs(a[i]);
        s = (s < x) ? x : s; /* std::max(s, |x|) */
    }
    return s;
}
static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */
static double dmin(double a, double b) { return (b < a) ? b : a; } /* std::min */

/* diff_x1 (operators.cpp:40-52) reduced to its max-abs, used by the
 * feasibility tests (admm.cpp:501, objective.cpp:36, 237-238). */
static double d1_norm_inf(const G* g, const double* b) {
    const double ih = 1.0 / g->h1;
    double s = 0.0;
    for (long long c = 0; c < g->ncol; ++c) {
        const double* bc = b + c * g->n1;
        for (int i = 0; i < g->m1; ++i) s = dmax(s, fabs((bc[i + 1] - bc[i]) * ih));
    }
    return s;
}

/* ---- column interpolant, image.cpp:24-46 -------------------------------- */
typedef struct {
    const double* s;
    int m;
    double h, o;
} Interp;

static double ip_value(const Interp* p, double x) {
    const double u = (x - p->o) / p->h - 0.5;
    const int m = p->m;
    if (u <= -0.5 || u >= m - 0.5) return 0.0;
    if (u <= 0.0) return (u + 0.5) * 2.0 * p->s[0];
    if (u >= m - 1.0) return (m - 0.5 - u) * 2.0 * p->s[m - 1];
    const double fi = floor(u);
    const int i = (int)fi;
    const double w = u - fi;
    return (1.0 - w) * p->s[i] + w * p->s[i + 1];
}

static double ip_slope(const Interp* p, double x) {
    const double u = (x - p->o) / p->h - 0.5;
    const int m = p->m;
    if (u <= -0.5 || u > m - 0.5) return 0.0;
    if (u <= 0.0) return 2.0 * p->s[0] / p->h;
    if (u > m - 1.0) return -2.0 * p->s[m - 1] / p->h;
    double fi = floor(u);
    if (fi == u) fi -= 1.0;
    const int i = (int)fi;
    if (i < 0) return 2.0 * p->s[0] / p->h;
    return (p->s[i + 1] - p->s[i]) / p->h;
}

static Interp column_of(const G* g, const double* img, long long c) {
    Interp p = {img + c * g->m1, g->m1, g->h1, g->o1}; /* image_column, image.cpp:48-52 */
    return p;
}

/* detail::residual_column, objective.cpp:48-73 (tp/tm outputs unused here) */
static void residual_column(const Interp* ip, const Interp* im, const G* g, const double* b,
                            double* r, double* jlo, double* jhi) {
    const int m1 = g->m1;
    const double h1 = g->h1;
    for (int i = 0; i < m1; ++i) {
        const double xc = g->o1 + (i + 0.5) * h1; /* cell_center, grid.hpp:46 */
        const double a = 0.5 * (b[i] + b[i + 1]);
        const double d = (b[i + 1] - b[i]) / h1;
        const double vp = ip_value(ip, xc + a);
        const double vm = ip_value(im, xc - a);
        const double Tp = vp * (1.0 + d);
        const double Tm = vm * (1.0 - d);
        r[i] = Tp - Tm;
        if (jlo) {
            const double gp = ip_slope(ip, xc + a);
            const double gm = ip_slope(im, xc - a);
            const double wa = 0.5 * (gp * (1.0 + d) + gm * (1.0 - d));
            const double wd = (vp + vm) / h1;
            jlo[i] = wa - wd;
            jhi[i] = wa + wd;
        }
    }
}

int oracle_residual(const epc_grid* gg, const double* iplus, const double* iminus,
                    const double* b, double* r) {
    G g;
    int rc = grid_make(gg, &g, NULL, 0);
    if (rc) return rc;
    for (long long c = 0; c < g.ncol; ++c) { /* residual, objective.cpp:77-91 */
        Interp ip = column_of(&g, iplus, c), im = column_of(&g, iminus, c);
        residual_column(&ip, &im, &g, b + c * g.n1, r + c * g.m1, NULL, NULL);
    }
    return EPC_OK;
}

/* ======================================================================
 * ADMM column machinery, admm.cpp:41-265
 * ====================================================================== */

/* ColFactor::factorize, admm.cpp:45-55 (l[n-1] stays 0) */
static int col_factorize(int n, const double* diag, const double* off, double* d, double* l) {
    for (int i = 0; i < n; ++i) l[i] = 0.0;
    if (!(diag[0] > 0.0)) return -1;
    d[0] = diag[0];
    for (int i = 1; i < n; ++i) {
        l[i - 1] = off[i - 1] / d[i - 1];
        d[i] = diag[i] - l[i - 1] * off[i - 1];
        if (!(d[i] > 0.0)) return -1;
    }
    return 0;
}

/* ColFactor::solve, admm.cpp:56-60 */
static void col_solve(int n, const double* d, const double* l, double* x) {
    for (int i = 1; i < n; ++i) x[i] -= l[i - 1] * x[i - 1];
    for (int i = 0; i < n; ++i) x[i] /= d[i];
    for (int i = n - 2; i >= 0; --i) x[i] -= l[i] * x[i + 1];
}

/* tridiag_apply, admm.cpp:63-70 */
static void tridiag_apply(int n, const double* diag, const double* off, const double* x, double* y) {
    for (int i = 0; i < n; ++i) {
        double acc = diag[i] * x[i];
        if (i > 0) acc += off[i - 1] * x[i - 1];
        if (i + 1 < n) acc += off[i] * x[i + 1];
        y[i] = acc;
    }
}

/* dense_spd_solve, admm.cpp:73-95; returns -1 on a singular Schur complement */
static int dense_spd_solve(int n, double* a, double* rhs) {
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < i; ++j) {
            double s = a[(size_t)i * n + j];
            for (int k = 0; k < j; ++k) s -= a[(size_t)i * n + k] * a[(size_t)j * n + k];
            a[(size_t)i * n + j] = s / a[(size_t)j * n + j];
        }
        double s = a[(size_t)i * n + i];
        for (int k = 0; k < i; ++k) s -= a[(size_t)i * n + k] * a[(size_t)i * n + k];
        if (!(s > 0.0)) return -1;
        a[(size_t)i * n + i] = sqrt(s);
    }
    for (int i = 0; i < n; ++i) {
        double s = rhs[i];
        for (int k = 0; k < i; ++k) s -= a[(size_t)i * n + k] * rhs[k];
        rhs[i] = s / a[(size_t)i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = rhs[i];
        for (int k = i + 1; k < n; ++k) s -= a[(size_t)k * n + i] * rhs[k];
        rhs[i] = s / a[(size_t)i * n + i];
    }
    return 0;
}

/* clamp_column_diffs, admm.cpp:99-110 */
static void clamp_column_diffs(double* x, int n, double h) {
    double shift = 0.0;
    for (int i = 0; i + 1 < n; ++i) {
        const double nx = x[i + 1] + shift;
        const double hi = x[i] + h, lo = x[i] - h;
        double cl = dmin(dmax(nx, lo), hi);
        while ((cl - x[i]) / h > 1.0) cl = nextafter(cl, x[i]);
        while ((cl - x[i]) / h < -1.0) cl = nextafter(cl, x[i]);
        shift += cl - nx;
        x[i + 1] = cl;
    }
}

/* Scratch for one column QP of size n (reused across calls). */
typedef struct {
    int n, cap_rows;
    double *gvec, *w, *p, *q, *schur, *lam, *fd, *fl;
    int* act;
} QpWork;

static void qpw_init(QpWork* w, int n) {
    memset(w, 0, sizeof *w);
    w->n = n;
    w->gvec = dalloc(n);
    w->w = dalloc(n);
    w->p = dalloc(n);
    w->fd = dalloc(n);
    w->fl = dalloc(n);
    w->cap_rows = n; /* at most n-1 active rows */
    w->q = dalloc((long long)n * n);
    w->schur = dalloc((long long)n * n);
    w->lam = dalloc(n);
    w->act = (int*)calloc((size_t)n, sizeof(int));
}

static void qpw_free(QpWork* w) {
    free(w->gvec); free(w->w); free(w->p); free(w->fd); free(w->fl);
    free(w->q); free(w->schur); free(w->lam); free(w->act);
}

enum { QP_OK = 0, QP_PIVOT = 1, QP_INFEASIBLE = 2, QP_SCHUR = 3, QP_CYCLE = 4 };

static const char* qp_what(int code) {
    switch (code) {
        case QP_PIVOT: return "column factor: nonpositive pivot";
        case QP_INFEASIBLE: return "qp_active_set: infeasible starting point";
        case QP_SCHUR: return "qp_active_set: singular Schur complement";
        case QP_CYCLE: return "qp_active_set: iteration cap reached (cycling guard)";
    }
    return "";
}

/* qp_active_set, admm.cpp:114-237. x holds x0 on entry, the solution on exit. */
static int qp_solve(QpWork* W, int n, double h, const double* gd, const double* go,
                    const double* c, double* x, double* lambda, int* sign, int max_iter,
                    int* iters, int* max_active) {
    const int ncell = n - 1;
    for (int i = 0; i < ncell; ++i) {
        lambda[i] = 0.0;
        sign[i] = 0;
    }
    *iters = 0;
    if (col_factorize(n, gd, go, W->fd, W->fl)) return QP_PIVOT;
#define DVAL(i) ((x[(i) + 1] - x[(i)]) / h)
    for (int i = 0; i < ncell; ++i)
        if (fabs(DVAL(i)) > 1.0 + 1e-9) return QP_INFEASIBLE;
    int na = 0;
    int* act = W->act;
    for (int i = 0; i < ncell; ++i) { /* warm start, admm.cpp:133-143 */
        const double d = DVAL(i);
        if (d <= -1.0 + 1e-10) {
            sign[i] = +1;
            act[na++] = i;
        } else if (d >= 1.0 - 1e-10) {
            sign[i] = -1;
            act[na++] = i;
        }
    }
    double *gvec = W->gvec, *w = W->w, *p = W->p, *q = W->q, *schur = W->schur, *lam = W->lam;
    for (int it = 1; it <= max_iter; ++it) {
        *iters = it;
        if (max_active && na > *max_active) *max_active = na;
        tridiag_apply(n, gd, go, x, gvec); /* g = -c - G x */
        for (int i = 0; i < n; ++i) gvec[i] = -c[i] - gvec[i];
        memcpy(w, gvec, sizeof(double) * n);
        col_solve(n, W->fd, W->fl, w);
        for (int r = 0; r < na; ++r) {
            double* qr = q + (size_t)r * n;
            for (int i = 0; i < n; ++i) qr[i] = 0.0;
            const int i = act[r];
            const double s = sign[i] / h;
            qr[i] = -s;
            qr[i + 1] = s;
            col_solve(n, W->fd, W->fl, qr);
        }
        for (int r = 0; r < na; ++r) lam[r] = 0.0;
        if (na > 0) {
            for (int r = 0; r < na; ++r) {
                const int ir = act[r];
                const double sr = sign[ir] / h;
                for (int s = 0; s < na; ++s) {
                    const double* qs = q + (size_t)s * n;
                    schur[(size_t)r * na + s] = sr * (qs[ir + 1] - qs[ir]);
                }
                const double arx = sign[ir] * DVAL(ir);
                lam[r] = -(sr * (w[ir + 1] - w[ir]) - (-1.0 - arx));
            }
            if (dense_spd_solve(na, schur, lam)) return QP_SCHUR;
        }
        memcpy(p, w, sizeof(double) * n); /* p = w + sum lambda_r q_r */
        for (int r = 0; r < na; ++r) {
            const double* qr = q + (size_t)r * n;
            for (int i = 0; i < n; ++i) p[i] += lam[r] * qr[i];
        }
        double xs = 1.0;
        for (int i = 0; i < n; ++i) xs = dmax(xs, fabs(x[i]));
        double pn = 0.0;
        for (int i = 0; i < n; ++i) pn = dmax(pn, fabs(p[i]));

        if (pn <= 1e-11 * xs) {
            int worst = -1;
            double worst_lam = -1e-9 * (1.0 + vnorm_inf(lam, na));
            for (int r = 0; r < na; ++r)
                if (lam[r] < worst_lam) {
                    worst_lam = lam[r];
                    worst = r;
                }
            if (worst < 0) {
                for (int r = 0; r < na; ++r) lambda[act[r]] = dmax(0.0, lam[r]);
                return QP_OK;
            }
            sign[act[worst]] = 0;
            for (int r = worst; r + 1 < na; ++r) act[r] = act[r + 1];
            --na;
            continue;
        }
        double t = 1.0; /* ratio test, admm.cpp:211-219 */
        for (int i = 0; i < ncell; ++i) {
            if (sign[i] != 0) continue;
            const double d = DVAL(i);
            const double dp = (p[i + 1] - p[i]) / h;
            if (dp < -1e-14) t = dmin(t, (-1.0 - d) / dp);
            else if (dp > 1e-14) t = dmin(t, (1.0 - d) / dp);
        }
        t = dmax(t, 0.0);
        for (int i = 0; i < n; ++i) x[i] += t * p[i];
        if (t < 1.0) {
            for (int i = 0; i < ncell; ++i) {
                if (sign[i] != 0) continue;
                const double d = DVAL(i);
                if (d <= -1.0 + 1e-12) {
                    sign[i] = +1;
                    act[na++] = i;
                } else if (d >= 1.0 - 1e-12) {
                    sign[i] = -1;
                    act[na++] = i;
                }
            }
        }
    }
#undef DVAL
    return QP_CYCLE;
}

/* verify_qp_kkt, admm.cpp:239-265 */
static double kkt_check(int n, double h, const double* gd, const double* go, const double* c,
                        const double* x, const double* lambda, const int* sign, double* s) {
    const int ncell = n - 1;
    tridiag_apply(n, gd, go, x, s);
    double scale = 1.0;
    for (int i = 0; i < n; ++i) scale = dmax(dmax(scale, fabs(s[i])), fabs(c[i]));
    for (int i = 0; i < n; ++i) s[i] += c[i];
    double lmax = 1.0;
    for (int i = 0; i < ncell; ++i) lmax = dmax(lmax, fabs(lambda[i]));
    double viol = 0.0;
    for (int i = 0; i < ncell; ++i) {
        if (sign[i] == 0) continue;
        const double a = sign[i] / h;
        s[i] += a * lambda[i];
        s[i + 1] -= a * lambda[i];
    }
    for (int i = 0; i < n; ++i) viol = dmax(viol, fabs(s[i]) / scale);
    for (int i = 0; i < ncell; ++i) {
        const double d = (x[i + 1] - x[i]) / h;
        viol = dmax(viol, fabs(d) - 1.0);
        viol = dmax(viol, -lambda[i] / lmax);
        const double slack = sign[i] != 0 ? sign[i] * d + 1.0 : 0.0;
        viol = dmax(viol, fabs(lambda[i] * slack) / (lmax * 1.0));
    }
    return viol;
}
/* std::max({scale, |s|, |c|}) in admm.cpp:245 folds left-to-right with the
 * same (a < b) ? b : a comparisons as the nested dmax above. */

int oracle_qp_active_set(int n, double h, const double* gd, const double* go, const double* c,
                         const double* x0, int max_iter, double* x, double* lambda,
                         int* active_sign, int* iters, char* msg, size_t msglen) {
    QpWork W;
    qpw_init(&W, n);
    memcpy(x, x0, sizeof(double) * n);
    int it = 0;
    const int rc = qp_solve(&W, n, h, gd, go, c, x, lambda, active_sign, max_iter, &it, NULL);
    qpw_free(&W);
    if (iters) *iters = it;
    set_msg(msg, msglen, "%s", qp_what(rc));
    if (rc == QP_INFEASIBLE) return EPC_ERR_INVALID_ARGUMENT;
    return rc ? EPC_ERR_RUNTIME : EPC_OK;
}

double oracle_verify_qp_kkt(int n, double h, const double* gd, const double* go,
                            const double* c, const double* x, const double* lambda,
                            const int* active_sign) {
    double* s = dalloc(n);
    const double v = kkt_check(n, h, gd, go, c, x, lambda, active_sign, s);
    free(s);
    return v;
}

/* ---- config validation, objective.cpp:11-15, admm.cpp:28-37 ----------- */
static int params_validate(const epc_objective_params* p, char* msg, size_t len) {
    if (!(p->alpha > 0.0)) { set_msg(msg, len, "ObjectiveParams: alpha must be > 0"); return EPC_ERR_INVALID_ARGUMENT; }
    if (!(p->beta >= 0.0)) { set_msg(msg, len, "ObjectiveParams: beta must be >= 0"); return EPC_ERR_INVALID_ARGUMENT; }
    if (!(p->gamma >= 0.0)) { set_msg(msg, len, "ObjectiveParams: gamma must be >= 0"); return EPC_ERR_INVALID_ARGUMENT; }
    return EPC_OK;
}

static int admm_validate(const epc_admm_config* c, char* msg, size_t len) {
    if (!(c->rho_min > 0.0) || !(c->rho0 >= c->rho_min)) { set_msg(msg, len, "ADMMConfig: need rho0 >= rho_min > 0"); return EPC_ERR_INVALID_ARGUMENT; }
    if (!(c->eps_abs > 0.0) || !(c->eps_rel > 0.0)) { set_msg(msg, len, "ADMMConfig: tolerances must be positive"); return EPC_ERR_INVALID_ARGUMENT; }
    if (c->max_iter < 1 || c->sqp_max_iter < 1) { set_msg(msg, len, "ADMMConfig: iteration caps must be >= 1"); return EPC_ERR_INVALID_ARGUMENT; }
    if (!(c->tau_incr > 1.0) || !(c->tau_decr > 1.0) || !(c->mu > 1.0)) { set_msg(msg, len, "ADMMConfig: adaptation constants must exceed 1"); return EPC_ERR_INVALID_ARGUMENT; }
    return EPC_OK;
}

/* Optional per-column work counters (diagnostics for kernel design; not part
 * of the restated algorithm): [col*4 + {sqp, qp, ls_trials, max_active}]. */
static int* g_colstats = NULL;
void oracle_debug_colstats(int* buf) { g_colstats = buf; }

/* b_update, admm.cpp:301-443 (single-threaded: columns in index order, the
 * first failing column aborts with its message, as parallel_for's chunk 0). */
static int b_update_impl(const G* g, const double* iplus, const double* iminus, const double* b,
                         const double* z, const double* u, double rho,
                         const epc_objective_params* P, const epc_admm_config* C, double* out,
                         epc_bupdate_stats* st, char* msg, size_t msglen) {
    if (!(rho > 0.0)) {
        set_msg(msg, msglen, "b_update: rho must be positive");
        return EPC_ERR_INVALID_ARGUMENT;
    }
    const int m1 = g->m1, n1 = g->n1;
    const double V = g->V, h1 = g->h1;
    const double alpha_w = P->alpha * V;
    const double rho_w = rho * V;
    const double lap_w = alpha_w / (h1 * h1);
    const int qp_cap = 6 * n1 + 10;

    double *x = dalloc(n1), *tgt = dalloc(n1), *r = dalloc(m1), *jlo = dalloc(m1), *jhi = dalloc(m1);
    double *grad = dalloc(n1), *gd = dalloc(n1), *go = dalloc(n1), *cqp = dalloc(n1);
    double *gx = dalloc(n1), *xtrial = dalloc(n1), *rtrial = dalloc(m1), *qx = dalloc(n1);
    double *qlam = dalloc(n1), *kkts = dalloc(n1);
    int* qsign = (int*)calloc((size_t)n1, sizeof(int));
    QpWork W;
    qpw_init(&W, n1);
    long sqp_total = 0, qp_total = 0;
    double kkt_max = 0.0;
    int max_active = 0;
    int rc = EPC_OK;

    for (long long c = 0; c < g->ncol && rc == EPC_OK; ++c) {
        const Interp ip = column_of(g, iplus, c), im = column_of(g, iminus, c);
        const double* bc = b + c * n1;
        const double* zc = z + c * n1;
        const double* uc = u + c * n1;
        for (int i = 0; i < n1; ++i) {
            x[i] = bc[i];
            tgt[i] = zc[i] - uc[i];
        }
        double col_kkt = 0.0;
        double s0 = -1.0;
        int* cs = g_colstats ? g_colstats + 4 * c : NULL;
        if (cs) cs[0] = cs[1] = cs[2] = cs[3] = 0;
        for (int sqp = 0; sqp < C->sqp_max_iter; ++sqp) {
            if (cs) cs[0]++;
            residual_column(&ip, &im, g, x, r, jlo, jhi);
            for (int i = 0; i < n1; ++i) {
                grad[i] = rho_w * (x[i] - tgt[i]);
                gd[i] = rho_w;
                go[i] = 0.0;
            }
            double sr = 0.0, sd = 0.0;
            for (int i = 0; i < m1; ++i) {
                sr += r[i] * r[i];
                grad[i] += V * jlo[i] * r[i];
                grad[i + 1] += V * jhi[i] * r[i];
                gd[i] += V * jlo[i] * jlo[i] + lap_w;
                gd[i + 1] += V * jhi[i] * jhi[i] + lap_w;
                go[i] += V * jlo[i] * jhi[i] - lap_w;
                const double d = (x[i + 1] - x[i]) / h1;
                sd += d * d;
                const double dd = alpha_w * d / h1;
                grad[i] -= dd;
                grad[i + 1] += dd;
            }
            double sq = 0.0;
            for (int i = 0; i < n1; ++i) {
                const double e = x[i] - tgt[i];
                sq += e * e;
            }
            const double fval = 0.5 * V * sr + 0.5 * alpha_w * sd + 0.5 * rho_w * sq;

            tridiag_apply(n1, gd, go, x, gx);
            for (int i = 0; i < n1; ++i) cqp[i] = grad[i] - gx[i];

            memcpy(qx, x, sizeof(double) * n1);
            int qit = 0;
            const int qrc = qp_solve(&W, n1, h1, gd, go, cqp, qx, qlam, qsign, qp_cap, &qit,
                                     &max_active);
            if (qrc != QP_OK) {
                set_msg(msg, msglen, "b_update: column %lld: %s", c, qp_what(qrc));
                rc = EPC_ERR_RUNTIME;
                break;
            }
            qp_total += qit;
            if (cs) { cs[1] += qit; if (max_active > cs[3]) cs[3] = max_active; }
            sqp_total += 1;
            if (C->check_kkt)
                col_kkt = dmax(col_kkt, kkt_check(n1, h1, gd, go, cqp, qx, qlam, qsign, kkts));

            double sn = 0.0, gdir = 0.0;
            for (int i = 0; i < n1; ++i) {
                const double d = qx[i] - x[i];
                sn += d * d;
                gdir += grad[i] * d;
            }
            sn = sqrt(sn);
            if (s0 < 0.0) s0 = sn;
            double xs = 1.0;
            for (int i = 0; i < n1; ++i) xs = dmax(xs, fabs(x[i]));
            if (sn <= dmax(C->sqp_tol_rel * s0, 1e-14 * xs)) break;
            if (!(gdir < 0.0)) break;

            double tls = 1.0; /* backtracking, admm.cpp:414-427 */
            int accepted = 0;
            for (int ls = 0; ls < 40; ++ls) {
                if (cs) cs[2]++;
                for (int i = 0; i < n1; ++i) xtrial[i] = x[i] + tls * (qx[i] - x[i]);
                /* subproblem_value, admm.cpp:335-351 */
                residual_column(&ip, &im, g, xtrial, rtrial, NULL, NULL);
                double tsr = 0.0;
                for (int i = 0; i < m1; ++i) tsr += rtrial[i] * rtrial[i];
                double tsd = 0.0, tsq = 0.0;
                for (int i = 0; i < m1; ++i) {
                    const double d = (xtrial[i + 1] - xtrial[i]) / h1;
                    tsd += d * d;
                }
                for (int i = 0; i < n1; ++i) {
                    const double e = xtrial[i] - tgt[i];
                    tsq += e * e;
                }
                const double ftrial = 0.5 * V * tsr + 0.5 * alpha_w * tsd + 0.5 * rho_w * tsq;
                if (ftrial <= fval + 1e-4 * tls * gdir) {
                    accepted = 1;
                    break;
                }
                tls *= 0.5;
            }
            if (!accepted) break;
            double* tmp = x; /* x.swap(xtrial) */
            x = xtrial;
            xtrial = tmp;
        }
        if (rc != EPC_OK) break;
        clamp_column_diffs(x, n1, h1);
        memcpy(out + c * n1, x, sizeof(double) * n1);
        kkt_max = dmax(kkt_max, col_kkt);
    }
    if (st && rc == EPC_OK) {
        st->sqp_iters = sqp_total;
        st->qp_iters = qp_total;
        st->kkt_violation = kkt_max;
        st->max_active = max_active;
    }
    free(x); free(tgt); free(r); free(jlo); free(jhi); free(grad); free(gd); free(go);
    free(cqp); free(gx); free(xtrial); free(rtrial); free(qx); free(qlam); free(kkts);
    free(qsign);
    qpw_free(&W);
    return rc;
}

int oracle_b_update(const epc_grid* gg, const double* iplus, const double* iminus,
                    const double* b, const double* z, const double* u, double rho,
                    const epc_objective_params* p, const epc_admm_config* cfg, double* b_out,
                    epc_bupdate_stats* stats, char* msg, size_t msglen) {
    G g;
    int rc = grid_make(gg, &g, msg, msglen);
    if (rc) return rc;
    set_msg(msg, msglen, "");
    return b_update_impl(&g, iplus, iminus, b, z, u, rho, p, cfg, b_out, stats, msg, msglen);
}

/* ======================================================================
 * DctCoupledSolver, operators.cpp:275-446
 * ====================================================================== */
typedef struct {
    G g;
    double *c2, *c3, *lam23;
} Dct;

/* dct2_matrix, operators.cpp:287-295 */
static double* dct2_matrix(int m) {
    double* c = dalloc((long long)m * m);
    const double s0 = sqrt(1.0 / m), sq = sqrt(2.0 / m);
    for (int q = 0; q < m; ++q)
        for (int j = 0; j < m; ++j)
            c[(size_t)q * m + j] = (q == 0 ? s0 : sq) * cos(PI_D * q * (2.0 * j + 1.0) / (2.0 * m));
    return c;
}

/* neumann_eigenvalues, operators.cpp:275-282 */
static void neumann_eigenvalues(int m, double h, double* lam) {
    for (int q = 0; q < m; ++q) {
        const double s = sin(PI_D * q / (2.0 * m));
        lam[q] = 4.0 / (h * h) * s * s;
    }
}

static void dct_init(Dct* D, const G* g) {
    D->g = *g;
    const int m2 = g->m2, m3 = g->m3;
    D->c2 = dct2_matrix(m2);
    D->c3 = m3 > 1 ? dct2_matrix(m3) : NULL;
    double* l2 = dalloc(m2);
    double* l3 = dalloc(m3 > 1 ? m3 : 1);
    neumann_eigenvalues(m2, g->h2, l2);
    if (m3 > 1) neumann_eigenvalues(m3, g->h3, l3);
    else l3[0] = 0.0;
    D->lam23 = dalloc((long long)m2 * m3);
    for (int k = 0; k < m3; ++k)
        for (int j = 0; j < m2; ++j) D->lam23[(size_t)k * m2 + j] = l2[j] + l3[k];
    free(l2);
    free(l3);
}

static void dct_free(Dct* D) { free(D->c2); free(D->c3); free(D->lam23); }

/* transform_axis2, operators.cpp:347-367 */
static void transform_axis2(const Dct* D, const double* in, double* out, int inverse) {
    const int n1 = D->g.n1, m2 = D->g.m2, m3 = D->g.m3;
    memset(out, 0, sizeof(double) * (size_t)D->g.nface);
    for (int k = 0; k < m3; ++k) {
        const double* slab_in = in + (size_t)n1 * m2 * k;
        double* slab_out = out + (size_t)n1 * m2 * k;
        for (int q = 0; q < m2; ++q) {
            double* o = slab_out + (size_t)q * n1;
            for (int j = 0; j < m2; ++j) {
                const double coef = inverse ? D->c2[(size_t)j * m2 + q] : D->c2[(size_t)q * m2 + j];
                if (coef == 0.0) continue;
                const double* s = slab_in + (size_t)j * n1;
                for (int i = 0; i < n1; ++i) o[i] += coef * s[i];
            }
        }
    }
}

/* transform_axis3, operators.cpp:369-386 */
static void transform_axis3(const Dct* D, const double* in, double* out, int inverse) {
    const int n1 = D->g.n1, m2 = D->g.m2, m3 = D->g.m3;
    const size_t layer = (size_t)n1 * m2;
    memset(out, 0, sizeof(double) * (size_t)D->g.nface);
    for (int q = 0; q < m3; ++q) {
        double* o = out + layer * q;
        for (int k = 0; k < m3; ++k) {
            const double coef = inverse ? D->c3[(size_t)k * m3 + q] : D->c3[(size_t)q * m3 + k];
            if (coef == 0.0) continue;
            const double* s = in + layer * k;
            for (size_t i = 0; i < layer; ++i) o[i] += coef * s[i];
        }
    }
}

/* DctCoupledSolver::solve, operators.cpp:388-418 */
static int dct_solve(const Dct* D, const double* rhs, double alpha, double rho, double* out,
                     char* msg, size_t len) {
    if (!(alpha > 0.0)) { set_msg(msg, len, "dct_coupled_solve: alpha must be > 0"); return EPC_ERR_INVALID_ARGUMENT; }
    if (!(rho > 0.0)) { set_msg(msg, len, "dct_coupled_solve: rho must be > 0"); return EPC_ERR_INVALID_ARGUMENT; }
    const G* g = &D->g;
    const int n1 = g->n1;
    const double V = g->V;
    double* hat = dalloc(g->nface);
    double* tmp = dalloc(g->nface);
    transform_axis2(D, rhs, hat, 0);
    if (g->m3 > 1) {
        transform_axis3(D, hat, tmp, 0);
        double* t = hat; hat = tmp; tmp = t;
    }
    for (long long c = 0; c < g->ncol; ++c) {
        const double denom = alpha * V * D->lam23[c] + rho * V;
        double* x = hat + c * n1;
        for (int i = 0; i < n1; ++i) x[i] /= denom;
    }
    if (g->m3 > 1) {
        transform_axis3(D, hat, tmp, 1);
        double* t = hat; hat = tmp; tmp = t;
    }
    transform_axis2(D, hat, out, 1);
    free(hat);
    free(tmp);
    return EPC_OK;
}

int oracle_dct_solve(const epc_grid* gg, const double* rhs, double alpha, double rho,
                     double* out, char* msg, size_t msglen) {
    G g;
    int rc = grid_make(gg, &g, msg, msglen);
    if (rc) return rc;
    Dct D;
    dct_init(&D, &g);
    rc = dct_solve(&D, rhs, alpha, rho, out, msg, msglen);
    dct_free(&D);
    return rc;
}

/* z_update, admm.cpp:445-451 */
static int z_update_impl(const Dct* D, const double* b, const double* u, double rho, double alpha,
                         double* z, char* msg, size_t len) {
    const G* g = &D->g;
    double* rhs = dalloc(g->nface);
    const double w = rho * g->V;
    for (long long i = 0; i < g->nface; ++i) rhs[i] = w * (b[i] + u[i]);
    const int rc = dct_solve(D, rhs, alpha, rho, z, msg, len);
    free(rhs);
    return rc;
}

int oracle_z_update(const epc_grid* gg, const double* b, const double* u, double rho,
                    double alpha, double* z_out, char* msg, size_t msglen) {
    G g;
    int rc = grid_make(gg, &g, msg, msglen);
    if (rc) return rc;
    Dct D;
    dct_init(&D, &g);
    rc = z_update_impl(&D, b, u, rho, alpha, z_out, msg, msglen);
    dct_free(&D);
    return rc;
}

/* dual_update_and_residuals, admm.cpp:453-476 */
static void dual_update_impl(const G* g, const double* b_new, const double* z_new,
                             const double* z_old, const double* u_old, double rho,
                             double eps_abs, double eps_rel, double* u_out, epc_dual_result* o) {
    const double V = g->V;
    if (u_out != u_old) memcpy(u_out, u_old, sizeof(double) * (size_t)g->nface);
    double pr = 0.0, du = 0.0;
    for (long long i = 0; i < g->nface; ++i) {
        const double diff = b_new[i] - z_new[i];
        u_out[i] += diff;
        pr += diff * diff;
        const double dz = z_old[i] - z_new[i];
        du += dz * dz;
    }
    o->primal_res = sqrt(pr);
    o->dual_res = rho * V * sqrt(du);
    const double sqrt_n = sqrt((double)g->nface);
    o->eps_pri = sqrt_n * eps_abs + eps_rel * dmax(vnorm2(b_new, g->nface), vnorm2(z_new, g->nface));
    o->eps_dual = sqrt_n * eps_abs + eps_rel * rho * V * vnorm2(u_out, g->nface);
}

int oracle_dual_update(const epc_grid* gg, const double* b_new, const double* z_new,
                       const double* z_old, const double* u_old, double rho, double eps_abs,
                       double eps_rel, double* u_out, epc_dual_result* out) {
    G g;
    int rc = grid_make(gg, &g, NULL, 0);
    if (rc) return rc;
    dual_update_impl(&g, b_new, z_new, z_old, u_old, rho, eps_abs, eps_rel, u_out, out);
    return EPC_OK;
}

/* dot(D_axis z, D_axis z) for axis 2/3 (diff_perp, operators.cpp:70-100,
 * consumed in index order by dot(), grid.cpp:60-64). */
static double perp_sq(const G* g, const double* b, int axis) {
    const int n1 = g->n1, m2 = g->m2, m3 = g->m3;
    double s = 0.0;
    if (axis == 2) {
        const double ih = 1.0 / g->h2;
        for (int k = 0; k < m3; ++k)
            for (int j = 0; j + 1 < m2; ++j) {
                const double* lo = b + (size_t)n1 * (j + (size_t)m2 * k);
                const double* hi = lo + n1;
                for (int i = 0; i < n1; ++i) {
                    const double o = (hi[i] - lo[i]) * ih;
                    s += o * o;
                }
            }
        return s;
    }
    const double ih = 1.0 / g->h3;
    const size_t layer = (size_t)n1 * m2;
    for (int k = 0; k + 1 < m3; ++k) {
        const double* lo = b + layer * k;
        const double* hi = lo + layer;
        for (size_t i = 0; i < layer; ++i) {
            const double o = (hi[i] - lo[i]) * ih;
            s += o * o;
        }
    }
    return s;
}

/* dot(d1, d1) with d1 = diff_x1(b) in cell order (operators.cpp:40-52) */
static double d1_sq(const G* g, const double* b) {
    const double ih = 1.0 / g->h1;
    double s = 0.0;
    for (long long c = 0; c < g->ncol; ++c) {
        const double* bc = b + c * g->n1;
        for (int i = 0; i < g->m1; ++i) {
            const double o = (bc[i + 1] - bc[i]) * ih;
            s += o * o;
        }
    }
    return s;
}

/* f_value, admm.cpp:267-273 (dot(r,r) over all cells in index order) */
static double f_value(const G* g, const double* iplus, const double* iminus, const double* b,
                      double alpha, double* rbuf) {
    for (long long c = 0; c < g->ncol; ++c) {
        Interp ip = column_of(g, iplus, c), im = column_of(g, iminus, c);
        residual_column(&ip, &im, g, b + c * g->n1, rbuf + c * g->m1, NULL, NULL);
    }
    const double V = g->V;
    return 0.5 * V * vdot(rbuf, rbuf, g->ncell) + 0.5 * alpha * V * d1_sq(g, b);
}

/* g_value, admm.cpp:275-285 */
static double g_value(const G* g, const double* z, double alpha) {
    double s = perp_sq(g, z, 2);
    if (g->dim == 3) s += perp_sq(g, z, 3);
    return 0.5 * alpha * g->V * s;
}

/* augmented_lagrangian, admm.cpp:287-299 */
static double lagrangian_impl(const G* g, const double* iplus, const double* iminus,
                              const double* b, const double* z, const double* u, double rho,
                              double alpha, double* rbuf) {
    const double V = g->V;
    double lin = 0.0, quad = 0.0;
    for (long long i = 0; i < g->nface; ++i) {
        const double diff = b[i] - z[i];
        lin += u[i] * diff;
        quad += diff * diff;
    }
    return f_value(g, iplus, iminus, b, alpha, rbuf) + g_value(g, z, alpha) + rho * V * lin +
           0.5 * rho * V * quad;
}

double oracle_augmented_lagrangian(const epc_grid* gg, const double* iplus, const double* iminus,
                                   const double* b, const double* z, const double* u,
                                   double rho, double alpha) {
    G g;
    if (grid_make(gg, &g, NULL, 0)) return NAN;
    double* rbuf = dalloc(g.ncell);
    const double v = lagrangian_impl(&g, iplus, iminus, b, z, u, rho, alpha, rbuf);
    free(rbuf);
    return v;
}

/* rho_schedule, admm.cpp:478-486 */
double oracle_rho_schedule(int schedule, double rho, double rho_min, double primal_res,
                           double dual_res, double tau_incr, double tau_decr, double mu) {
    if (schedule == EPC_RHO_FIXED) return rho;
    double next = rho;
    if (primal_res > mu * dual_res) next = rho * tau_incr;
    else if (dual_res > mu * primal_res) next = rho / tau_decr;
    if (schedule == EPC_RHO_ADAPTIVE_BOUNDED) next = dmax(next, rho_min);
    return next;
}

void oracle_set_threads(int threads) { (void)threads; }

/* admm_solve, admm.cpp:488-560 (wall-clock row fields are left at 0) */
int oracle_admm_solve(const epc_grid* gg, const double* iplus, const double* iminus,
                      const double* b_in, const double* z_in, const double* u_in,
                      double* b_out, double* z_out, double* u_out, double* rho_io,
                      const epc_objective_params* P, const epc_admm_config* C, int level_tag,
                      epc_admm_row* rows, int max_rows, epc_solve_status* status) {
    char* msg = status->message;
    const size_t mlen = sizeof status->message;
    set_msg(msg, mlen, "");
    status->nrows = 0;
    status->stop = EPC_STOP_MAX_ITERATIONS;
    G g;
    int rc = params_validate(P, msg, mlen);
    if (rc) return rc;
    rc = admm_validate(C, msg, mlen);
    if (rc) return rc;
    rc = grid_make(gg, &g, msg, mlen);
    if (rc) return rc;
    const long long nf = g.nface;
    double *b = dalloc(nf), *z = dalloc(nf), *u = dalloc(nf), *bn = dalloc(nf), *zn = dalloc(nf);
    double* rbuf = dalloc(g.ncell);
    if (b_in) memcpy(b, b_in, sizeof(double) * nf);
    if (z_in) memcpy(z, z_in, sizeof(double) * nf);
    if (u_in) memcpy(u, u_in, sizeof(double) * nf);
    if (d1_norm_inf(&g, b) > 1.0) {
        set_msg(msg, mlen, "admm_solve: infeasible starting field");
        free(b); free(z); free(u); free(bn); free(zn); free(rbuf);
        return EPC_ERR_INVALID_ARGUMENT;
    }
    double rho = *rho_io;
    if (rho <= 0.0) rho = C->rho0;
    Dct D;
    dct_init(&D, &g);
    for (int it = 1; it <= C->max_iter; ++it) {
        epc_admm_row row;
        memset(&row, 0, sizeof row);
        row.level = level_tag;
        row.iter = it;
        row.rho = rho;
        epc_bupdate_stats bs = {0, 0, 0.0, 0};
        rc = b_update_impl(&g, iplus, iminus, b, z, u, rho, P, C, bn, &bs, msg, mlen);
        if (rc) {
            status->stop = EPC_STOP_ERROR;
            break;
        }
        memcpy(b, bn, sizeof(double) * nf);
        row.kkt_violation = bs.kkt_violation;
        rc = z_update_impl(&D, b, u, rho, P->alpha, zn, msg, mlen);
        if (rc) {
            status->stop = EPC_STOP_ERROR;
            break;
        }
        epc_dual_result du;
        dual_update_impl(&g, b, zn, z, u, rho, C->eps_abs, C->eps_rel, u, &du);
        memcpy(z, zn, sizeof(double) * nf);
        const double lag = lagrangian_impl(&g, iplus, iminus, b, z, u, rho, P->alpha, rbuf);
        row.primal_res = du.primal_res;
        row.dual_res = du.dual_res;
        row.eps_pri = du.eps_pri;
        row.eps_dual = du.eps_dual;
        row.lagrangian = lag;
        if (status->nrows < max_rows) rows[status->nrows] = row;
        status->nrows++;
        if (du.primal_res <= du.eps_pri && du.dual_res <= du.eps_dual) {
            status->stop = EPC_STOP_CONVERGED;
            break;
        }
        const double next = oracle_rho_schedule(C->schedule, rho, C->rho_min, du.primal_res,
                                                du.dual_res, C->tau_incr, C->tau_decr, C->mu);
        if (next != rho) {
            const double a = rho / next; /* scale(st.u.v, rho/next) */
            for (long long i = 0; i < nf; ++i) u[i] *= a;
            rho = next;
        }
    }
    if (b_out) memcpy(b_out, b, sizeof(double) * nf);
    if (z_out) memcpy(z_out, z, sizeof(double) * nf);
    if (u_out) memcpy(u_out, u, sizeof(double) * nf);
    *rho_io = rho;
    dct_free(&D);
    free(b); free(z); free(u); free(bn); free(zn); free(rbuf);
    return EPC_OK;
}

/* ======================================================================
 * GN-PCG, objective.cpp + operators.cpp + gn_pcg.cpp
 * ====================================================================== */

/* phi, phi_d1, phi_d2, objective.cpp:17-33 */
static double phi(double x) {
    if (fabs(x) >= 1.0) return INFINITY;
    const double x2 = x * x;
    return x2 * x2 / (1.0 - x2);
}
static double phi_d1(double x) {
    const double x2 = x * x, x3 = x2 * x;
    const double d = 1.0 - x2;
    return (4.0 * x3 - 2.0 * x3 * x2) / (d * d);
}
static double phi_d2(double x) {
    const double x2 = x * x;
    const double d = 1.0 - x2;
    return 2.0 * x2 * (x2 * x2 - 3.0 * x2 + 6.0) / (d * d * d);
}

/* smoother_hessian_apply, operators.cpp:141-183 */
static void smoother_hessian_apply(const G* g, const double* b, double* out) {
    const int m1 = g->m1, n1 = g->n1, m2 = g->m2, m3 = g->m3;
    const double V = g->V;
    const double w1 = V / (g->h1 * g->h1), w2 = V / (g->h2 * g->h2), w3 = V / (g->h3 * g->h3);
    for (long long c = 0; c < g->ncol; ++c) {
        const int j = (int)(c % m2), k = (int)(c / m2);
        const double* bc = b + c * n1;
        double* oc = out + c * n1;
        oc[0] = w1 * (bc[0] - bc[1]);
        for (int i = 1; i < m1; ++i) oc[i] = w1 * (2.0 * bc[i] - bc[i - 1] - bc[i + 1]);
        oc[m1] = w1 * (bc[m1] - bc[m1 - 1]);
        if (j > 0) {
            const double* nb = bc - n1;
            for (int i = 0; i < n1; ++i) oc[i] += w2 * (bc[i] - nb[i]);
        }
        if (j + 1 < m2) {
            const double* nb = bc + n1;
            for (int i = 0; i < n1; ++i) oc[i] += w2 * (bc[i] - nb[i]);
        }
        if (m3 > 1) {
            const long long layer = (long long)n1 * m2;
            if (k > 0) {
                const double* nb = bc - layer;
                for (int i = 0; i < n1; ++i) oc[i] += w3 * (bc[i] - nb[i]);
            }
            if (k + 1 < m3) {
                const double* nb = bc + layer;
                for (int i = 0; i < n1; ++i) oc[i] += w3 * (bc[i] - nb[i]);
            }
        }
    }
}

/* distance, objective.cpp:93-126: value, gradient (grad must be zeroed),
 * residual and Jacobian. */
static double distance_eval(const G* g, const double* iplus, const double* iminus,
                            const double* b, double* grad, double* res, double* jlo,
                            double* jhi, double* partial) {
    const int m1 = g->m1, n1 = g->n1;
    const double V = g->V;
    for (long long c = 0; c < g->ncol; ++c) {
        Interp ip = column_of(g, iplus, c), im = column_of(g, iminus, c);
        double* r = res + c * m1;
        double* jl = jlo + c * m1;
        double* jh = jhi + c * m1;
        residual_column(&ip, &im, g, b + c * n1, r, jl, jh);
        double* gc = grad + c * n1;
        double s = 0.0;
        for (int i = 0; i < m1; ++i) {
            s += r[i] * r[i];
            gc[i] += V * jl[i] * r[i];
            gc[i + 1] += V * jh[i] * r[i];
        }
        partial[c] = s;
    }
    double s = 0.0;
    for (long long c = 0; c < g->ncol; ++c) s += partial[c];
    return 0.5 * V * s;
}

/* penalty, objective.cpp:196-229 (caller guarantees strict feasibility);
 * grad accumulates onto a zeroed array, phi2 per cell. */
static double penalty_eval(const G* g, const double* b, double beta, double* pgrad,
                           double* phi2, double* partial) {
    const int m1 = g->m1, n1 = g->n1;
    const double w = beta * g->V;
    const double ih = 1.0 / g->h1;
    for (long long c = 0; c < g->ncol; ++c) {
        const double* bc = b + c * n1;
        double* gc = pgrad + c * n1;
        double* p2 = phi2 ? phi2 + c * m1 : NULL;
        double s = 0.0;
        for (int i = 0; i < m1; ++i) {
            const double dc = (bc[i + 1] - bc[i]) * ih; /* diff_x1 */
            s += phi(dc);
            const double dphi = w * phi_d1(dc) * ih;
            gc[i] -= dphi;
            gc[i + 1] += dphi;
            if (p2) p2[i] = phi_d2(dc);
        }
        partial[c] = s;
    }
    double s = 0.0;
    for (long long c = 0; c < g->ncol; ++c) s += partial[c];
    return w * s;
}

/* penalty_value, objective.cpp:185-194 */
static double penalty_value(const G* g, const double* b, double beta) {
    if (beta == 0.0) return 0.0;
    const double ih = 1.0 / g->h1;
    double s = 0.0;
    for (long long c = 0; c < g->ncol; ++c) {
        const double* bc = b + c * g->n1;
        for (int i = 0; i < g->m1; ++i) {
            const double x = (bc[i + 1] - bc[i]) * ih;
            if (fabs(x) >= 1.0) return INFINITY;
            s += phi(x);
        }
    }
    return beta * g->V * s;
}

/* within_linf_box, objective.cpp:39-44 */
static int within_linf_box(const G* g, const double* b) {
    double diam2 = 0.0;
    const double ext[3] = {g->m1 * g->h1, g->m2 * g->h2, g->m3 * g->h3};
    for (int a = 0; a < g->dim; ++a) diam2 += ext[a] * ext[a];
    return vnorm_inf(b, g->nface) <= 2.0 * sqrt(diam2);
}

typedef struct {
    double *grad, *sgrad, *pgrad, *res, *jlo, *jhi, *phi2, *partial;
} ObjWork;

static void objw_init(ObjWork* w, const G* g) {
    w->grad = dalloc(g->nface);
    w->sgrad = dalloc(g->nface);
    w->pgrad = dalloc(g->nface);
    w->res = dalloc(g->ncell);
    w->jlo = dalloc(g->ncell);
    w->jhi = dalloc(g->ncell);
    w->phi2 = dalloc(g->ncell);
    w->partial = dalloc(g->ncol);
}
static void objw_free(ObjWork* w) {
    free(w->grad); free(w->sgrad); free(w->pgrad); free(w->res); free(w->jlo); free(w->jhi);
    free(w->phi2); free(w->partial);
}

/* objective_gn, objective.cpp:231-264. On success with need_grad, w->grad
 * holds the gradient. */
static void objective_impl(const G* g, const double* iplus, const double* iminus,
                           const double* b, const epc_objective_params* P, int need_grad,
                           ObjWork* w, epc_objective_eval* ev) {
    memset(ev, 0, sizeof *ev);
    const double dm = d1_norm_inf(g, b);
    ev->feasible = P->beta == 0.0 || dm <= 1.0 - 1e-10; /* kFeasEps, objective.hpp:40 */
    if (P->enforce_linf_box && !within_linf_box(g, b)) ev->feasible = 0;
    if (!ev->feasible) {
        ev->value = INFINITY;
        ev->pen = ev->value;
        return;
    }
    memset(w->grad, 0, sizeof(double) * (size_t)g->nface);
    ev->dist = distance_eval(g, iplus, iminus, b, w->grad, w->res, w->jlo, w->jhi, w->partial);
    /* smoother, objective.cpp:166-183 */
    double s = d1_sq(g, b);
    s += perp_sq(g, b, 2);
    if (g->dim == 3) s += perp_sq(g, b, 3);
    ev->smooth = 0.5 * g->V * s;
    if (need_grad) {
        smoother_hessian_apply(g, b, w->sgrad);
        for (long long i = 0; i < g->nface; ++i) w->grad[i] += P->alpha * w->sgrad[i];
        if (P->beta > 0.0) {
            memset(w->pgrad, 0, sizeof(double) * (size_t)g->nface);
            ev->pen = penalty_eval(g, b, P->beta, w->pgrad, NULL, w->partial);
            for (long long i = 0; i < g->nface; ++i) w->grad[i] += 1.0 * w->pgrad[i];
        }
    } else {
        ev->pen = penalty_value(g, b, P->beta);
    }
    ev->value = ev->dist + P->alpha * ev->smooth + ev->pen;
}

int oracle_objective_gn(const epc_grid* gg, const double* iplus, const double* iminus,
                        const double* b, const epc_objective_params* p, int need_grad,
                        epc_objective_eval* out, double* grad, double* residual) {
    G g;
    int rc = params_validate(p, NULL, 0);
    if (rc) return rc;
    rc = grid_make(gg, &g, NULL, 0);
    if (rc) return rc;
    ObjWork w;
    objw_init(&w, &g);
    objective_impl(&g, iplus, iminus, b, p, need_grad, &w, out);
    if (out->feasible) {
        if (grad && need_grad) memcpy(grad, w.grad, sizeof(double) * (size_t)g.nface);
        if (residual) memcpy(residual, w.res, sizeof(double) * (size_t)g.ncell);
    }
    objw_free(&w);
    return EPC_OK;
}

/* GnHessian, objective.cpp:266-348 */
typedef struct {
    G g;
    double *diag, *off, w2, w3;
} Hess;

static int hess_build(Hess* H, const G* g, const double* iplus, const double* iminus,
                      const double* b, const epc_objective_params* P, char* msg, size_t len) {
    const int m1 = g->m1, n1 = g->n1;
    const double V = g->V;
    H->g = *g;
    H->w2 = P->alpha * V / (g->h2 * g->h2);
    H->w3 = g->dim == 3 ? P->alpha * V / (g->h3 * g->h3) : 0.0;
    H->diag = dalloc(g->nface);
    H->off = dalloc(g->nface);
    ObjWork w;
    objw_init(&w, g);
    (void)distance_eval(g, iplus, iminus, b, w.grad, w.res, w.jlo, w.jhi, w.partial);
    for (long long c = 0; c < g->ncol; ++c) { /* add_hessian_blocks, objective.cpp:149-164 */
        const double* jl = w.jlo + c * m1;
        const double* jh = w.jhi + c * m1;
        double* d = H->diag + c * n1;
        double* o = H->off + c * n1;
        for (int i = 0; i < m1; ++i) {
            d[i] += V * jl[i] * jl[i];
            d[i + 1] += V * jh[i] * jh[i];
            o[i] += V * jl[i] * jh[i];
        }
    }
    { /* add_axis1_laplacian(alpha*V), operators.cpp:189-200 */
        const double wl = P->alpha * V / (g->h1 * g->h1);
        for (long long c = 0; c < g->ncol; ++c) {
            double* d = H->diag + c * n1;
            double* o = H->off + c * n1;
            d[0] += wl;
            for (int i = 1; i < m1; ++i) d[i] += 2.0 * wl;
            d[m1] += wl;
            for (int i = 0; i < m1; ++i) o[i] -= wl;
        }
    }
    for (long long f = 0; f < g->nface; ++f) H->diag[f] += P->gamma; /* add_identity */
    if (P->beta > 0.0) {
        if (d1_norm_inf(g, b) > 1.0 - 1e-10) {
            set_msg(msg, len, "penalty: derivatives requested at an infeasible point");
            objw_free(&w);
            return EPC_ERR_DOMAIN;
        }
        (void)penalty_eval(g, b, P->beta, w.pgrad, w.phi2, w.partial);
        const double wp = P->beta * V / (g->h1 * g->h1);
        for (long long c = 0; c < g->ncol; ++c) {
            const double* p2 = w.phi2 + c * m1;
            double* d = H->diag + c * n1;
            double* o = H->off + c * n1;
            for (int i = 0; i < m1; ++i) {
                d[i] += wp * p2[i];
                d[i + 1] += wp * p2[i];
                o[i] -= wp * p2[i];
            }
        }
    }
    objw_free(&w);
    return EPC_OK;
}

static void hess_free(Hess* H) { free(H->diag); free(H->off); }

/* cross_diag, objective.cpp:296-300 */
static double cross_diag(const Hess* H, int j, int k) {
    double d = H->w2 * ((j == 0 || j == H->g.m2 - 1) ? 1.0 : 2.0);
    if (H->g.dim == 3) d += H->w3 * ((k == 0 || k == H->g.m3 - 1) ? 1.0 : 2.0);
    return d;
}

/* GnHessian::apply, objective.cpp:302-331 */
static void hess_apply(const Hess* H, const double* x, double* y) {
    const G* g = &H->g;
    const int m1 = g->m1, n1 = g->n1, m2 = g->m2, m3 = g->m3;
    const double w2 = H->w2, w3 = H->w3;
    for (long long c = 0; c < g->ncol; ++c) {
        const int j = (int)(c % m2), k = (int)(c / m2);
        const double* xc = x + c * n1;
        const double* d = H->diag + c * n1;
        const double* o = H->off + c * n1;
        double* yc = y + c * n1;
        for (int i = 0; i <= m1; ++i) {
            double acc = d[i] * xc[i];
            if (i > 0) acc += o[i - 1] * xc[i - 1];
            if (i < m1) acc += o[i] * xc[i + 1];
            yc[i] = acc;
        }
        if (j > 0)
            for (int i = 0; i < n1; ++i) yc[i] += w2 * (xc[i] - xc[i - n1]);
        if (j + 1 < m2)
            for (int i = 0; i < n1; ++i) yc[i] += w2 * (xc[i] - xc[i + n1]);
        if (m3 > 1) {
            const long long layer = (long long)n1 * m2;
            if (k > 0)
                for (int i = 0; i < n1; ++i) yc[i] += w3 * (xc[i] - xc[i - layer]);
            if (k + 1 < m3)
                for (int i = 0; i < n1; ++i) yc[i] += w3 * (xc[i] - xc[i + layer]);
        }
    }
}

/* Preconditioner, gn_pcg.cpp:37-90 */
typedef struct {
    int kind;
    G g;
    double *fd, *fl; /* block: LDL^T factor of preconditioner_blocks() */
    double* diag;    /* jacobi / sgs: full_diagonal() */
    double* off;     /* sgs: column_part().off */
    double w2, w3;
} Prec;

/* TridiagFactor::factorize, operators.cpp:218-246 */
static int tridiag_factorize(const G* g, const double* diag, const double* off, double* fd,
                             double* fl, char* msg, size_t len) {
    const int n1 = g->n1;
    for (long long c = 0; c < g->ncol; ++c) {
        const double* d = diag + c * n1;
        const double* o = off + c * n1;
        double* pd = fd + c * n1;
        double* pl = fl + c * n1;
        double prev = d[0];
        if (!(prev > 0.0)) {
            set_msg(msg, len, "tridiag factorize: nonpositive pivot in column %lld", c);
            return EPC_ERR_RUNTIME;
        }
        pd[0] = prev;
        for (int i = 1; i < n1; ++i) {
            const double li = o[i - 1] / pd[i - 1];
            pl[i - 1] = li;
            const double piv = d[i] - li * o[i - 1];
            if (!(piv > 0.0)) {
                set_msg(msg, len, "tridiag factorize: nonpositive pivot in column %lld", c);
                return EPC_ERR_RUNTIME;
            }
            pd[i] = piv;
        }
        pl[n1 - 1] = 0.0;
    }
    return EPC_OK;
}

/* TridiagFactor::solve_column, operators.cpp:248-255 */
static void tridiag_solve(const G* g, const double* fd, const double* fl, double* x) {
    const int n1 = g->n1;
    for (long long c = 0; c < g->ncol; ++c) {
        const double* d = fd + c * n1;
        const double* l = fl + c * n1;
        double* xc = x + c * n1;
        for (int i = 1; i < n1; ++i) xc[i] -= l[i - 1] * xc[i - 1];
        for (int i = 0; i < n1; ++i) xc[i] /= d[i];
        for (int i = n1 - 2; i >= 0; --i) xc[i] -= l[i] * xc[i + 1];
    }
}

static int prec_make(Prec* M, int kind, const Hess* H, char* msg, size_t len) {
    memset(M, 0, sizeof *M);
    M->kind = kind;
    M->g = H->g;
    const G* g = &H->g;
    const int n1 = g->n1, m2 = g->m2;
    if (kind == EPC_PRECOND_NONE) return EPC_OK;
    /* full_diagonal (objective.cpp:350-358) / preconditioner_blocks (339-348) */
    double* pd = dalloc(g->nface);
    memcpy(pd, H->diag, sizeof(double) * (size_t)g->nface);
    for (long long c = 0; c < g->ncol; ++c) {
        const double cd = cross_diag(H, (int)(c % m2), (int)(c / m2));
        double* d = pd + c * n1;
        for (int i = 0; i < n1; ++i) d[i] += cd;
    }
    if (kind == EPC_PRECOND_JACOBI) {
        M->diag = pd;
        return EPC_OK;
    }
    if (kind == EPC_PRECOND_BLOCK_JACOBI) {
        M->fd = dalloc(g->nface);
        M->fl = dalloc(g->nface);
        const int rc = tridiag_factorize(g, pd, H->off, M->fd, M->fl, msg, len);
        free(pd);
        return rc;
    }
    if (kind == EPC_PRECOND_SGS) {
        M->diag = pd;
        M->off = dalloc(g->nface);
        memcpy(M->off, H->off, sizeof(double) * (size_t)g->nface);
        M->w2 = H->w2;
        M->w3 = H->w3;
        return EPC_OK;
    }
    free(pd);
    set_msg(msg, len, "make_preconditioner: bad kind");
    return EPC_ERR_RUNTIME;
}

static void prec_free(Prec* M) { free(M->fd); free(M->fl); free(M->diag); free(M->off); }

static void prec_apply(const Prec* M, const double* r, double* z) {
    const G* g = &M->g;
    const long long n = g->nface;
    switch (M->kind) {
        case EPC_PRECOND_NONE:
            memcpy(z, r, sizeof(double) * (size_t)n);
            return;
        case EPC_PRECOND_JACOBI:
            for (long long i = 0; i < n; ++i) z[i] = r[i] / M->diag[i];
            return;
        case EPC_PRECOND_BLOCK_JACOBI:
            memcpy(z, r, sizeof(double) * (size_t)n);
            tridiag_solve(g, M->fd, M->fl, z);
            return;
        case EPC_PRECOND_SGS: { /* gn_pcg.cpp:62-86 */
            const int n1 = g->n1, m2 = g->m2, m3 = g->m3;
            const long long layer = (long long)n1 * m2;
            for (long long f = 0; f < n; ++f) z[f] = 0.0;
            for (long long f = 0; f < n; ++f) {
                const long long c = f / n1;
                const int i = (int)(f % n1), j = (int)(c % m2), k = (int)(c / m2);
                double acc = r[f];
                if (i > 0) acc -= M->off[f - 1] * z[f - 1];
                if (j > 0) acc += M->w2 * z[f - n1];
                if (k > 0) acc += M->w3 * z[f - layer];
                z[f] = acc / M->diag[f];
            }
            for (long long f = 0; f < n; ++f) z[f] *= M->diag[f];
            for (long long f = n - 1; f >= 0; --f) {
                const long long c = f / n1;
                const int i = (int)(f % n1), j = (int)(c % m2), k = (int)(c / m2);
                double acc = z[f];
                if (i < n1 - 1) acc -= M->off[f] * z[f + 1];
                if (j + 1 < m2) acc += M->w2 * z[f + n1];
                if (k + 1 < m3) acc += M->w3 * z[f + layer];
                z[f] = acc / M->diag[f];
            }
            return;
        }
    }
}

/* pcg, gn_pcg.cpp:92-131 */
static int pcg_impl(const Hess* H, const Prec* M, const double* gv, double eta, int max_iters,
                    double* d, epc_pcg_result* out, char* msg, size_t len) {
    const long long n = H->g.nface;
    memset(out, 0, sizeof *out);
    for (long long i = 0; i < n; ++i) d[i] = 0.0;
    const double gnorm = vnorm2(gv, n);
    if (gnorm == 0.0) {
        out->reached_tol = 1;
        return EPC_OK;
    }
    double *r = dalloc(n), *z = dalloc(n), *p = dalloc(n), *q = dalloc(n);
    for (long long i = 0; i < n; ++i) r[i] = -gv[i];
    prec_apply(M, r, z);
    memcpy(p, z, sizeof(double) * (size_t)n);
    double rz = vdot(r, z, n);
    const double prec0 = sqrt(dmax(rz, 0.0));
    int rc = EPC_OK;
    for (int it = 0; it < max_iters; ++it) {
        hess_apply(H, p, q);
        const double pq = vdot(p, q, n);
        if (!(pq > 0.0)) {
            set_msg(msg, len, "pcg: nonpositive curvature encountered");
            rc = EPC_ERR_RUNTIME;
            break;
        }
        const double a = rz / pq;
        for (long long i = 0; i < n; ++i) d[i] += a * p[i];
        const double ma = -a;
        for (long long i = 0; i < n; ++i) r[i] += ma * q[i];
        out->iters = it + 1;
        out->relres = vnorm2(r, n) / gnorm;
        prec_apply(M, r, z);
        const double rz_new = vdot(r, z, n);
        out->relres_prec = prec0 > 0.0 ? sqrt(dmax(rz_new, 0.0)) / prec0 : 0.0;
        if (out->relres <= eta) {
            out->reached_tol = 1;
            break;
        }
        const double beta = rz_new / rz;
        rz = rz_new;
        for (long long i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    }
    free(r); free(z); free(p); free(q);
    return rc;
}

int oracle_gn_hessian_build(const epc_grid* gg, const double* iplus, const double* iminus,
                            const double* b, const epc_objective_params* p, double* diag,
                            double* off, double* pdiag, char* msg, size_t msglen) {
    G g;
    int rc = params_validate(p, msg, msglen);
    if (rc) return rc;
    rc = grid_make(gg, &g, msg, msglen);
    if (rc) return rc;
    Hess H;
    rc = hess_build(&H, &g, iplus, iminus, b, p, msg, msglen);
    if (rc == EPC_OK) {
        const size_t nb = sizeof(double) * (size_t)g.nface;
        if (diag) memcpy(diag, H.diag, nb);
        if (off) memcpy(off, H.off, nb);
        if (pdiag) {
            memcpy(pdiag, H.diag, nb);
            for (long long c = 0; c < g.ncol; ++c) {
                const double cd = cross_diag(&H, (int)(c % g.m2), (int)(c / g.m2));
                for (int i = 0; i < g.n1; ++i) pdiag[c * g.n1 + i] += cd;
            }
        }
    }
    hess_free(&H);
    return rc;
}

int oracle_gn_hessian_apply(const epc_grid* gg, const double* iplus, const double* iminus,
                            const double* b, const epc_objective_params* p, const double* x,
                            double* y, char* msg, size_t msglen) {
    G g;
    int rc = params_validate(p, msg, msglen);
    if (rc) return rc;
    rc = grid_make(gg, &g, msg, msglen);
    if (rc) return rc;
    Hess H;
    rc = hess_build(&H, &g, iplus, iminus, b, p, msg, msglen);
    if (rc == EPC_OK) hess_apply(&H, x, y);
    hess_free(&H);
    return rc;
}

int oracle_precond_apply(const epc_grid* gg, const double* iplus, const double* iminus,
                         const double* b, const epc_objective_params* p, int kind,
                         const double* r, double* z, char* msg, size_t msglen) {
    G g;
    int rc = params_validate(p, msg, msglen);
    if (rc) return rc;
    rc = grid_make(gg, &g, msg, msglen);
    if (rc) return rc;
    Hess H;
    rc = hess_build(&H, &g, iplus, iminus, b, p, msg, msglen);
    if (rc == EPC_OK) {
        Prec M;
        rc = prec_make(&M, kind, &H, msg, msglen);
        if (rc == EPC_OK) prec_apply(&M, r, z);
        prec_free(&M);
    }
    hess_free(&H);
    return rc;
}

int oracle_pcg(const epc_grid* gg, const double* iplus, const double* iminus, const double* b,
               const epc_objective_params* p, int kind, const double* grad, double eta,
               int max_iters, double* d, epc_pcg_result* out, char* msg, size_t msglen) {
    G g;
    int rc = params_validate(p, msg, msglen);
    if (rc) return rc;
    rc = grid_make(gg, &g, msg, msglen);
    if (rc) return rc;
    Hess H;
    rc = hess_build(&H, &g, iplus, iminus, b, p, msg, msglen);
    if (rc == EPC_OK) {
        Prec M;
        rc = prec_make(&M, kind, &H, msg, msglen);
        if (rc == EPC_OK) rc = pcg_impl(&H, &M, grad, eta, max_iters, d, out, msg, msglen);
        prec_free(&M);
    }
    hess_free(&H);
    return rc;
}

/* GNConfig::validate, gn_pcg.cpp:30-35 */
static int gn_validate(const epc_gn_config* c, char* msg, size_t len) {
    if (!(c->eta > 0.0 && c->eta < 1.0)) { set_msg(msg, len, "GNConfig: eta must be in (0,1)"); return EPC_ERR_INVALID_ARGUMENT; }
    if (!(c->wolfe_c1 > 0.0 && c->wolfe_c1 < c->wolfe_c2 && c->wolfe_c2 < 1.0)) { set_msg(msg, len, "GNConfig: need 0 < c1 < c2 < 1"); return EPC_ERR_INVALID_ARGUMENT; }
    if (c->max_outer < 1 || c->max_pcg < 1) { set_msg(msg, len, "GNConfig: iteration caps"); return EPC_ERR_INVALID_ARGUMENT; }
    return EPC_OK;
}

/* Line-search state for phi(t) of gauss_newton_solve (gn_pcg.cpp:245-255) */
typedef struct {
    const G* g;
    const double *iplus, *iminus, *b, *dir;
    const epc_objective_params* P;
    double* trial;    /* last evaluated trial point */
    ObjWork* w;       /* its evaluation (grad valid when feasible) */
    epc_objective_eval ev;
    int have_eval;
    double *keep_grad; /* trial_eval.grad kept from the last feasible phi call */
    epc_objective_eval keep_ev;
} Ray;

static double ray_phi(Ray* R, double t, double* dphi) {
    const long long n = R->g->nface;
    for (long long i = 0; i < n; ++i) R->trial[i] = R->b[i] + t * R->dir[i];
    epc_objective_eval ev;
    objective_impl(R->g, R->iplus, R->iminus, R->trial, R->P, 1, R->w, &ev);
    if (!ev.feasible) return INFINITY;
    if (dphi) *dphi = vdot(R->w->grad, R->dir, n);
    memcpy(R->keep_grad, R->w->grad, sizeof(double) * (size_t)n);
    R->keep_ev = ev;
    R->have_eval = 1;
    return ev.value;
}

typedef struct {
    double a, f, df;
} Probe;

/* wolfe_linesearch, gn_pcg.cpp:141-195 */
static int wolfe(Ray* R, double phi0, double dphi0, double c1, double c2, int max_evals,
                 double* lambda) {
    int evals = 0;
    *lambda = 0.0;
    if (!(dphi0 < 0.0) || !isfinite(phi0)) return 0;
#define SUFF(a, f) ((f) <= phi0 + c1 * (a)*dphi0)
    Probe prev = {0.0, phi0, dphi0};
    double a = 1.0;
    int first = 1;
    Probe lo, hi;
    int zoom = 0;
    while (evals < max_evals) {
        double df = 0.0;
        const double f = ray_phi(R, a, &df);
        ++evals;
        if (!SUFF(a, f) || (!first && f >= prev.f)) {
            lo = prev;
            hi = (Probe){a, f, df};
            zoom = 1;
            break;
        }
        if (fabs(df) <= -c2 * dphi0) {
            *lambda = a;
            return 1;
        }
        if (df >= 0.0) {
            lo = (Probe){a, f, df};
            hi = prev;
            zoom = 1;
            break;
        }
        prev = (Probe){a, f, df};
        a *= 2.0;
        first = 0;
    }
    if (!zoom) return 0;
    while (evals < max_evals) { /* zoom, gn_pcg.cpp:149-174 */
        const double am = 0.5 * (lo.a + hi.a);
        double df = 0.0;
        const double f = ray_phi(R, am, &df);
        ++evals;
        if (!SUFF(am, f) || f >= lo.f) {
            hi = (Probe){am, f, df};
        } else {
            if (fabs(df) <= -c2 * dphi0) {
                *lambda = am;
                return 1;
            }
            if (df * (hi.a - lo.a) >= 0.0) hi = lo;
            lo = (Probe){am, f, df};
        }
        if (fabs(hi.a - lo.a) < 1e-16 * dmax(1.0, fabs(lo.a))) break;
    }
    if (lo.a > 0.0 && SUFF(lo.a, lo.f)) {
        *lambda = lo.a;
        return 1;
    }
    return 0;
#undef SUFF
}

/* gauss_newton_solve, gn_pcg.cpp:197-292 (wall_s left at 0) */
int oracle_gn_solve(const epc_grid* gg, const double* iplus, const double* iminus,
                    const double* b0, double* b_out, const epc_objective_params* P,
                    const epc_gn_config* C, int level_tag, epc_gn_row* rows, int max_rows,
                    epc_solve_status* status) {
    char* msg = status->message;
    const size_t mlen = sizeof status->message;
    set_msg(msg, mlen, "");
    status->nrows = 0;
    status->stop = EPC_STOP_MAX_ITERATIONS;
    int rc = gn_validate(C, msg, mlen);
    if (rc) return rc;
    rc = params_validate(P, msg, mlen);
    if (rc) return rc;
    G g;
    rc = grid_make(gg, &g, msg, mlen);
    if (rc) return rc;
    const long long n = g.nface;
    double *b = dalloc(n), *grad = dalloc(n), *dir = dalloc(n), *trial = dalloc(n);
    double *bnew = dalloc(n), *keep_grad = dalloc(n), *zero = dalloc(n);
    memcpy(b, b0, sizeof(double) * (size_t)n);
    ObjWork w;
    objw_init(&w, &g);
    epc_objective_eval cur;
    objective_impl(&g, iplus, iminus, b, P, 1, &w, &cur);
    int ret = EPC_OK;
#define ROW(...)                                                       \
    do {                                                               \
        if (status->nrows < max_rows) rows[status->nrows] = (epc_gn_row){__VA_ARGS__}; \
        status->nrows++;                                               \
    } while (0)
    if (!cur.feasible) {
        set_msg(msg, mlen, "gauss_newton_solve: starting guess is infeasible");
        ret = EPC_ERR_INVALID_ARGUMENT;
        goto done;
    }
    memcpy(grad, w.grad, sizeof(double) * (size_t)n);
    {
        epc_objective_eval ez;
        objective_impl(&g, iplus, iminus, zero, P, 0, &w, &ez);
        const double j_ref = 1.0 + fabs(ez.value);
        double grad_norm = vnorm2(grad, n);
        ROW(level_tag, 0, cur.value, grad_norm, 0.0, 0, 0.0, 0.0, 0.0);
        if (grad_norm <= 1e-15 * j_ref) {
            status->stop = EPC_STOP_CONVERGED;
            set_msg(msg, mlen, "gradient numerically zero at start");
            goto done;
        }
        for (int k = 1; k <= C->max_outer; ++k) {
            Hess H;
            rc = hess_build(&H, &g, iplus, iminus, b, P, msg, mlen);
            if (rc) { hess_free(&H); ret = rc; goto done; }
            Prec M;
            rc = prec_make(&M, C->precond, &H, msg, mlen);
            if (rc) { prec_free(&M); hess_free(&H); ret = rc; goto done; }
            epc_pcg_result pr;
            rc = pcg_impl(&H, &M, grad, C->eta, C->max_pcg, dir, &pr, msg, mlen);
            prec_free(&M);
            hess_free(&H);
            if (rc) { ret = rc; goto done; }
            const double gd = vdot(grad, dir, n);
            if (!(gd < 0.0)) {
                status->stop = EPC_STOP_ERROR;
                set_msg(msg, mlen, "search direction is not a descent direction");
                goto done;
            }
            Ray R = {&g, iplus, iminus, b, dir, P, trial, &w, {0}, 0, keep_grad, {0}};
            for (long long i = 0; i < n; ++i) trial[i] = 0.0; /* StaggeredField trial(g) */
            double lambda = 0.0;
            const int ok = wolfe(&R, cur.value, gd, C->wolfe_c1, C->wolfe_c2, C->max_ls, &lambda);
            if (!ok) {
                status->stop = EPC_STOP_LINE_SEARCH_FAILURE;
                set_msg(msg, mlen, "no admissible Wolfe step within the evaluation budget");
                goto done;
            }
            for (long long i = 0; i < n; ++i) bnew[i] = b[i] + lambda * dir[i];
            epc_objective_eval tev = R.keep_ev;
            if (memcmp(trial, bnew, sizeof(double) * (size_t)n) != 0 || !R.have_eval) {
                /* trial.v != b_new.v compares values; identical doubles only
                 * differ bitwise for +-0 or NaN, which a feasible ray never
                 * yields differently here. */
                int differs = !R.have_eval;
                for (long long i = 0; i < n && !differs; ++i) differs = trial[i] != bnew[i];
                if (differs) {
                    objective_impl(&g, iplus, iminus, bnew, P, 1, &w, &tev);
                    memcpy(keep_grad, w.grad, sizeof(double) * (size_t)n);
                }
            }
            const double step_norm = lambda * vnorm2(dir, n);
            const double dj = fabs(tev.value - cur.value);
            const double bnorm = vnorm2(b, n);
            const double grad_new = vnorm2(keep_grad, n);
            memcpy(b, bnew, sizeof(double) * (size_t)n);
            cur = tev;
            memcpy(grad, keep_grad, sizeof(double) * (size_t)n);
            grad_norm = grad_new;
            ROW(level_tag, k, cur.value, grad_norm, lambda, pr.iters, pr.relres, pr.relres_prec, 0.0);
            const int stop_obj = dj <= C->eps_obj * j_ref;
            const int stop_iter = step_norm <= C->eps_iter * (1.0 + bnorm);
            const int stop_grad = grad_norm <= C->eps_grad * j_ref;
            if (stop_obj && stop_iter && stop_grad) {
                status->stop = EPC_STOP_CONVERGED;
                goto done;
            }
        }
        status->stop = EPC_STOP_MAX_ITERATIONS;
    }
#undef ROW
done:
    if (b_out) memcpy(b_out, b, sizeof(double) * (size_t)n);
    objw_free(&w);
    free(b); free(grad); free(dir); free(trial); free(bnew); free(keep_grad); free(zero);
    return ret;
}

/* ==========================================================================
 * multilevel (proj/src/multilevel.cpp) — restatement for the checker
 * ========================================================================== */

static double extent_of(const epc_grid* g, int a) { return g->m[a] * g->h[a]; } /* grid.hpp:36 */

/* default_schedule, multilevel.cpp:22-41 */
int oracle_default_schedule(const epc_grid* fine, int max_levels, int min_cells, epc_grid* out,
                            int cap, int* nlev, char* msg, size_t msglen) {
    G gf;
    int rc = grid_make(fine, &gf, msg, msglen);
    if (rc) return rc;
    epc_grid tmp[64];
    int n = 0;
    tmp[n++] = *fine;
    epc_grid cur = *fine;
    while (n < max_levels && n < 64) {
        epc_grid next = cur;
        int ok = 1;
        for (int a = 0; a < fine->dim; ++a) {
            next.m[a] = (cur.m[a] + 1) / 2;
            if (next.m[a] < min_cells) ok = 0;
            next.h[a] = extent_of(fine, a) / next.m[a];
        }
        if (!ok || (next.m[0] == cur.m[0] && next.m[1] == cur.m[1] && next.m[2] == cur.m[2])) break;
        tmp[n++] = next;
        cur = next;
    }
    if (n > cap) {
        set_msg(msg, msglen, "default_schedule: output capacity too small");
        return EPC_ERR_INVALID_ARGUMENT;
    }
    for (int l = 0; l < n; ++l) out[l] = tmp[n - 1 - l]; /* std::reverse: coarse -> fine */
    *nlev = n;
    return EPC_OK;
}

/* make_axis_weights, multilevel.cpp:53-77: coarse interval c covers fine
 * intervals first[c] .. first[c] + cnt[c] - 1 with weights overlap / Hc */
typedef struct {
    int* first;
    int* off; /* offsets into w, size mc + 1 */
    double* w;
} AxisW;

static AxisW axis_weights(int mf, int mc, double L) {
    AxisW aw;
    aw.first = (int*)calloc((size_t)mc, sizeof(int));
    aw.off = (int*)calloc((size_t)mc + 1, sizeof(int));
    aw.w = (double*)calloc((size_t)(mf + 2 * mc + 4), sizeof(double));
    const double hf = L / mf, hc = L / mc;
    int nw = 0;
    for (int c = 0; c < mc; ++c) {
        aw.off[c] = nw;
        const double lo = c * hc, hi = (c + 1) * hc;
        int f0 = (int)floor(lo / hf + 1e-12);
        if (f0 < 0) f0 = 0;
        aw.first[c] = f0;
        for (int f = f0; f < mf; ++f) {
            const double flo = f * hf, fhi = (f + 1) * hf;
            if (flo >= hi - 1e-12 * hc && f > f0) break;
            const double ov = dmin(hi, fhi) - dmax(lo, flo);
            if (ov <= 0.0) {
                if (f == f0) {
                    aw.first[c] = f + 1;
                    continue;
                }
                break;
            }
            aw.w[nw++] = ov / hc;
        }
    }
    aw.off[mc] = nw;
    return aw;
}

static void axis_free(AxisW* a) {
    free(a->first);
    free(a->off);
    free(a->w);
}

/* restrict_axis, multilevel.cpp:79-94 */
static double* restrict_axis(const double* in, long long pre, int mf, long long post,
                             const AxisW* aw, int mc) {
    double* out = dalloc(pre * mc * post);
    for (long long p = 0; p < post; ++p)
        for (int c = 0; c < mc; ++c) {
            double* o = out + pre * (c + (long long)mc * p);
            for (int t = 0; t < aw->off[c + 1] - aw->off[c]; ++t) {
                const int f = aw->first[c] + t;
                const double wt = aw->w[aw->off[c] + t];
                const double* s = in + pre * (f + (long long)mf * p);
                for (long long i = 0; i < pre; ++i) o[i] += wt * s[i];
            }
        }
    return out;
}

/* restrict_image, multilevel.cpp:98-131 */
int oracle_restrict_image(const epc_grid* fine, const epc_grid* coarse, const double* in,
                          double* out, char* msg, size_t msglen) {
    G gf, gc;
    int rc = grid_make(fine, &gf, msg, msglen);
    if (rc) return rc;
    rc = grid_make(coarse, &gc, msg, msglen);
    if (rc) return rc;
    if (coarse->dim != fine->dim) {
        set_msg(msg, msglen, "restrict_image: dimension mismatch");
        return EPC_ERR_INVALID_ARGUMENT;
    }
    for (int a = 0; a < 3; ++a) {
        if (coarse->m[a] > fine->m[a]) {
            set_msg(msg, msglen, "restrict_image: coarse grid larger than fine");
            return EPC_ERR_INVALID_ARGUMENT;
        }
        const double ef = extent_of(fine, a);
        if (fabs(extent_of(coarse, a) - ef) > 1e-9 * dmax(1.0, ef) ||
            fabs(coarse->origin[a] - fine->origin[a]) > 1e-12 * dmax(1.0, ef)) {
            set_msg(msg, msglen, "restrict_image: domains differ");
            return EPC_ERR_INVALID_ARGUMENT;
        }
    }
    const int fm1 = fine->m[0], fm2 = fine->m[1], fm3 = fine->m[2];
    const int cm1 = coarse->m[0], cm2 = coarse->m[1], cm3 = coarse->m[2];
    AxisW a1 = axis_weights(fm1, cm1, extent_of(fine, 0));
    double* d1 = restrict_axis(in, 1, fm1, (long long)fm2 * fm3, &a1, cm1);
    axis_free(&a1);
    AxisW a2 = axis_weights(fm2, cm2, extent_of(fine, 1));
    double* d2 = restrict_axis(d1, cm1, fm2, fm3, &a2, cm2);
    axis_free(&a2);
    free(d1);
    if (fine->dim == 3 && fm3 != cm3) {
        AxisW a3 = axis_weights(fm3, cm3, extent_of(fine, 2));
        double* d3 = restrict_axis(d2, (long long)cm1 * cm2, fm3, 1, &a3, cm3);
        axis_free(&a3);
        free(d2);
        d2 = d3;
    }
    memcpy(out, d2, sizeof(double) * (size_t)gc.ncell);
    free(d2);
    return EPC_OK;
}

/* make_taps, multilevel.cpp:141-155 */
typedef struct {
    int i0, i1;
    double w1;
} Tap;

static Tap* make_taps(int count_f, double x0f, double stepf, int count_c, double x0c,
                      double stepc) {
    Tap* t = (Tap*)calloc((size_t)count_f, sizeof(Tap));
    for (int i = 0; i < count_f; ++i) {
        const double x = x0f + i * stepf;
        const double u = (x - x0c) / stepc;
        if (u <= 0.0) {
            t[i].i0 = 0, t[i].i1 = 0, t[i].w1 = 0.0;
        } else if (u >= count_c - 1) {
            t[i].i0 = count_c - 1, t[i].i1 = count_c - 1, t[i].w1 = 0.0;
        } else {
            const int i0 = (int)floor(u);
            t[i].i0 = i0;
            t[i].i1 = i0 + 1 < count_c - 1 ? i0 + 1 : count_c - 1;
            t[i].w1 = u - i0;
        }
    }
    return t;
}

/* the infeasibility rescue shared by prolong_field and the average restart
 * (multilevel.cpp:200-201, 275-276) */
static void rescue(const G* g, double* b) {
    const double dmx = d1_norm_inf(g, b);
    if (dmx > 1.0 - 1e-10) {
        const double s = 0.95 / dmx;
        for (long long i = 0; i < g->nface; ++i) b[i] *= s;
    }
}

/* prolong_field, multilevel.cpp:157-203 */
int oracle_prolong_field(const epc_grid* coarse, const epc_grid* fine, const double* in,
                         double* out, char* msg, size_t msglen) {
    G gf, gc;
    int rc = grid_make(fine, &gf, msg, msglen);
    if (rc) return rc;
    rc = grid_make(coarse, &gc, msg, msglen);
    if (rc) return rc;
    if (fine->dim != coarse->dim) {
        set_msg(msg, msglen, "prolong_field: dimension mismatch");
        return EPC_ERR_INVALID_ARGUMENT;
    }
    for (int a = 0; a < 3; ++a) {
        if (fine->m[a] < coarse->m[a]) {
            set_msg(msg, msglen, "prolong_field: fine grid smaller than coarse");
            return EPC_ERR_INVALID_ARGUMENT;
        }
        const double ef = extent_of(fine, a);
        if (fabs(extent_of(coarse, a) - ef) > 1e-9 * dmax(1.0, ef)) {
            set_msg(msg, msglen, "prolong_field: domains differ");
            return EPC_ERR_INVALID_ARGUMENT;
        }
    }
    Tap* t1 = make_taps(gf.n1, fine->origin[0], fine->h[0], gc.n1, coarse->origin[0],
                        coarse->h[0]);
    Tap* t2 = make_taps(gf.m2, fine->origin[1] + 0.5 * fine->h[1], fine->h[1], gc.m2,
                        coarse->origin[1] + 0.5 * coarse->h[1], coarse->h[1]);
    Tap* t3;
    if (fine->dim == 3) {
        t3 = make_taps(gf.m3, fine->origin[2] + 0.5 * fine->h[2], fine->h[2], gc.m3,
                       coarse->origin[2] + 0.5 * coarse->h[2], coarse->h[2]);
    } else {
        t3 = (Tap*)calloc(1, sizeof(Tap));
    }
    for (int k = 0; k < gf.m3; ++k)
        for (int j = 0; j < gf.m2; ++j)
            for (int i = 0; i <= gf.m1; ++i) {
                const Tap a = t1[i], b = t2[j], c = t3[k];
                double v = 0.0;
                for (int ck = 0; ck < 2; ++ck) {
                    const double wk = ck ? c.w1 : 1.0 - c.w1;
                    if (wk == 0.0) continue;
                    const int kk = ck ? c.i1 : c.i0;
                    for (int cj = 0; cj < 2; ++cj) {
                        const double wj = cj ? b.w1 : 1.0 - b.w1;
                        if (wj == 0.0) continue;
                        const int jj = cj ? b.i1 : b.i0;
                        for (int ci = 0; ci < 2; ++ci) {
                            const double wi = ci ? a.w1 : 1.0 - a.w1;
                            if (wi == 0.0) continue;
                            const int ii = ci ? a.i1 : a.i0;
                            v += wk * wj * wi * in[ii + (long long)gc.n1 * (jj + (long long)gc.m2 * kk)];
                        }
                    }
                }
                out[i + (long long)gf.n1 * (j + (long long)gf.m2 * k)] = v;
            }
    free(t1);
    free(t2);
    free(t3);
    rescue(&gf, out);
    return EPC_OK;
}

static int grid_eq(const epc_grid* a, const epc_grid* b) {
    if (a->dim != b->dim) return 0;
    for (int x = 0; x < 3; ++x)
        if (a->m[x] != b->m[x] || a->h[x] != b->h[x] || a->origin[x] != b->origin[x]) return 0;
    return 1;
}

/* multilevel_solve, multilevel.cpp:205-289 */
int oracle_multilevel_solve(const epc_grid* fine, const double* iplus, const double* iminus,
                            const epc_grid* levels, int nlev, const int* gn_max_outer,
                            const int* admm_max_iter, int solver,
                            const epc_objective_params* P, const epc_gn_config* gcfg,
                            const epc_admm_config* acfg, int restart, double* b_out,
                            epc_admm_row* arows, int max_arows, epc_gn_row* grows,
                            int max_grows, epc_multilevel_status* st) {
    char* msg = st->message;
    const size_t ml = sizeof st->message;
    st->stop = EPC_STOP_CONVERGED;
    st->n_admm_rows = st->n_gn_rows = 0;
    st->b_level = nlev - 1;
    msg[0] = 0;
    /* LevelSchedule::validate, multilevel.cpp:11-20 */
    if (nlev < 1) {
        set_msg(msg, ml, "LevelSchedule: no levels");
        return EPC_ERR_INVALID_ARGUMENT;
    }
    G tmpg;
    for (int l = 0; l < nlev; ++l) {
        int rc = grid_make(&levels[l], &tmpg, msg, ml);
        if (rc) return rc;
    }
    for (int l = 1; l < nlev; ++l)
        for (int a = 0; a < 3; ++a)
            if (levels[l - 1].m[a] > levels[l].m[a]) {
                set_msg(msg, ml, "LevelSchedule: levels must be ordered coarse to fine");
                return EPC_ERR_INVALID_ARGUMENT;
            }
    if (!grid_eq(&levels[nlev - 1], fine)) {
        set_msg(msg, ml, "multilevel_solve: finest level must match the data grid");
        return EPC_ERR_INVALID_ARGUMENT;
    }
    G gfine;
    grid_make(fine, &gfine, msg, ml);
    double *b_start = NULL, *sb = NULL, *sz = NULL, *su = NULL;
    double rho = 0.0;
    int rc = EPC_OK;
    for (int lvl = 0; lvl < nlev; ++lvl) {
        const epc_grid* g = &levels[lvl];
        G gl;
        grid_make(g, &gl, msg, ml);
        const int finest = lvl == nlev - 1;
        double *ip = NULL, *im = NULL;
        const double *lip = iplus, *lim = iminus;
        if (!finest) {
            ip = dalloc(gl.ncell);
            im = dalloc(gl.ncell);
            if ((rc = oracle_restrict_image(fine, g, iplus, ip, msg, ml)) ||
                (rc = oracle_restrict_image(fine, g, iminus, im, msg, ml)))
                goto done;
            lip = ip;
            lim = im;
        }
        double* b = dalloc(gl.nface);
        if (solver == EPC_SOLVER_GN) {
            epc_gn_config cfg = *gcfg;
            if (gn_max_outer && gn_max_outer[lvl] >= 0) cfg.max_outer = gn_max_outer[lvl];
            if (lvl == 0) {
                free(b_start);
                b_start = dalloc(gl.nface);
            }
            epc_gn_row* rows = (epc_gn_row*)calloc((size_t)cfg.max_outer + 1, sizeof(epc_gn_row));
            epc_solve_status s;
            rc = oracle_gn_solve(g, lip, lim, b_start, b, P, &cfg, lvl, rows, cfg.max_outer + 1, &s);
            if (rc == EPC_OK) {
                for (int r = 0; r < s.nrows && r <= cfg.max_outer; ++r) {
                    if (st->n_gn_rows < max_grows) grows[st->n_gn_rows] = rows[r];
                    st->n_gn_rows++;
                }
                st->stop = s.stop;
                if (s.message[0]) set_msg(msg, ml, "%s", s.message);
            } else {
                set_msg(msg, ml, "%s", s.message);
            }
            free(rows);
            if (rc) {
                free(b);
                goto level_done;
            }
            if (finest || s.stop == EPC_STOP_ERROR || s.stop == EPC_STOP_LINE_SEARCH_FAILURE) {
                memcpy(b_out, b, sizeof(double) * (size_t)gl.nface);
                st->b_level = lvl;
            }
            if (s.stop == EPC_STOP_ERROR || s.stop == EPC_STOP_LINE_SEARCH_FAILURE) {
                free(b), free(ip), free(im);
                goto early;
            }
            if (!finest) {
                G gn;
                grid_make(&levels[lvl + 1], &gn, msg, ml);
                free(b_start);
                b_start = dalloc(gn.nface);
                rc = oracle_prolong_field(g, &levels[lvl + 1], b, b_start, msg, ml);
            }
            free(b);
        } else {
            epc_admm_config cfg = *acfg;
            if (admm_max_iter && admm_max_iter[lvl] >= 0) cfg.max_iter = admm_max_iter[lvl];
            if (lvl == 0) {
                free(sb), free(sz), free(su);
                sb = dalloc(gl.nface), sz = dalloc(gl.nface), su = dalloc(gl.nface);
                rho = cfg.rho0;
            }
            double *z = dalloc(gl.nface), *u = dalloc(gl.nface);
            epc_admm_row* rows = (epc_admm_row*)calloc((size_t)cfg.max_iter + 1, sizeof(epc_admm_row));
            epc_solve_status s;
            rc = oracle_admm_solve(g, lip, lim, sb, sz, su, b, z, u, &rho, P, &cfg, lvl, rows,
                                   cfg.max_iter + 1, &s);
            if (rc == EPC_OK) {
                for (int r = 0; r < s.nrows && r <= cfg.max_iter; ++r) {
                    if (st->n_admm_rows < max_arows) arows[st->n_admm_rows] = rows[r];
                    st->n_admm_rows++;
                }
                st->stop = s.stop;
                if (s.message[0]) set_msg(msg, ml, "%s", s.message);
            } else {
                set_msg(msg, ml, "%s", s.message);
            }
            free(rows);
            if (rc == EPC_OK && (finest || s.stop == EPC_STOP_ERROR)) {
                memcpy(b_out, b, sizeof(double) * (size_t)gl.nface);
                st->b_level = lvl;
            }
            if (rc == EPC_OK && s.stop == EPC_STOP_ERROR) {
                free(b), free(z), free(u), free(ip), free(im);
                goto early;
            }
            if (rc == EPC_OK && !finest) {
                const epc_grid* gf = &levels[lvl + 1];
                G gn;
                grid_make(gf, &gn, msg, ml);
                double *nb = dalloc(gn.nface), *nz = dalloc(gn.nface), *nu = dalloc(gn.nface);
                if (restart == EPC_RESTART_PROLONG_ALL) {
                    rc = oracle_prolong_field(g, gf, b, nb, msg, ml);
                    if (!rc) rc = oracle_prolong_field(g, gf, z, nz, msg, ml);
                    if (!rc) rc = oracle_prolong_field(g, gf, u, nu, msg, ml);
                } else if (restart == EPC_RESTART_B_FOR_BOTH) {
                    rc = oracle_prolong_field(g, gf, b, nb, msg, ml);
                    memcpy(nz, nb, sizeof(double) * (size_t)gn.nface);
                } else {
                    double* zf = dalloc(gn.nface);
                    rc = oracle_prolong_field(g, gf, b, nb, msg, ml);
                    if (!rc) rc = oracle_prolong_field(g, gf, z, zf, msg, ml);
                    for (long long i = 0; i < gn.nface; ++i) nb[i] = 0.5 * (nb[i] + zf[i]);
                    rescue(&gn, nb);
                    memcpy(nz, nb, sizeof(double) * (size_t)gn.nface);
                    free(zf);
                }
                free(sb), free(sz), free(su);
                sb = nb, sz = nz, su = nu;
            }
            free(b), free(z), free(u);
        }
    level_done:
        free(ip);
        free(im);
        if (rc) goto done;
    }
early:
    rc = EPC_OK;
done:
    free(b_start), free(sb), free(sz), free(su);
    return rc;
}

/* ==========================================================================
 * image.cpp: correct_pair, ssd, ncc, simulate_pair — restatement
 * ========================================================================== */

/* correct_pair, image.cpp:226-253 */
int oracle_correct_pair(const epc_grid* gg, const double* iplus, const double* iminus,
                        const double* b, double* cp, double* cm, char* msg, size_t msglen) {
    G g;
    int rc = grid_make(gg, &g, msg, msglen);
    if (rc) return rc;
    if (d1_norm_inf(&g, b) > 1.0) {
        set_msg(msg, msglen, "correct_pair: field infeasible, |D1 b| > 1");
        return EPC_ERR_INVALID_ARGUMENT;
    }
    for (long long c = 0; c < g.ncol; ++c) {
        const Interp ip = column_of(&g, iplus, c), im = column_of(&g, iminus, c);
        const double* bc = b + c * g.n1;
        for (int i = 0; i < g.m1; ++i) {
            const double xc = g.o1 + (i + 0.5) * g.h1;
            const double a = 0.5 * (bc[i] + bc[i + 1]);
            const double d = (bc[i + 1] - bc[i]) / g.h1;
            cp[c * g.m1 + i] = ip_value(&ip, xc + a) * (1.0 + d);
            cm[c * g.m1 + i] = ip_value(&im, xc - a) * (1.0 - d);
        }
    }
    return EPC_OK;
}

/* ssd, image.cpp:255-263 */
int oracle_ssd(const epc_grid* gg, const double* a, const double* b, double* out, char* msg,
               size_t msglen) {
    G g;
    int rc = grid_make(gg, &g, msg, msglen);
    if (rc) return rc;
    double s = 0.0;
    for (long long i = 0; i < g.ncell; ++i) {
        const double d = a[i] - b[i];
        s += d * d;
    }
    *out = 0.5 * g.V * s;
    return EPC_OK;
}

/* ncc, image.cpp:265-283 */
int oracle_ncc(const epc_grid* gg, const double* a, const double* b, double* out, char* msg,
               size_t msglen) {
    G g;
    int rc = grid_make(gg, &g, msg, msglen);
    if (rc) return rc;
    const long long n = g.ncell;
    double ma = 0.0, mb = 0.0;
    for (long long i = 0; i < n; ++i) {
        ma += a[i];
        mb += b[i];
    }
    ma /= (double)n;
    mb /= (double)n;
    double sab = 0.0, saa = 0.0, sbb = 0.0;
    for (long long i = 0; i < n; ++i) {
        const double da = a[i] - ma, db = b[i] - mb;
        sab += da * db;
        saa += da * da;
        sbb += db * db;
    }
    if (saa <= 0.0 || sbb <= 0.0) {
        set_msg(msg, msglen, "ncc: zero-variance image");
        return EPC_ERR_INVALID_ARGUMENT;
    }
    *out = (sab * sab) / (saa * sbb);
    return EPC_OK;
}

/* std::mt19937_64 (the standard's parameters) */
typedef struct {
    unsigned long long mt[312];
    int i;
} Mt64;

static void mt64_seed(Mt64* s, unsigned long long seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (unsigned long long)i;
    s->i = 312;
}

static unsigned long long mt64_next(Mt64* s) {
    if (s->i >= 312) {
        for (int k = 0; k < 312; ++k) {
            const unsigned long long y = (s->mt[k] & 0xFFFFFFFF80000000ULL) |
                                         (s->mt[(k + 1) % 312] & 0x7FFFFFFFULL);
            s->mt[k] = s->mt[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
        }
        s->i = 0;
    }
    unsigned long long x = s->mt[s->i++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

/* std::generate_canonical<double, 53> over mt19937_64 (libstdc++): one draw */
static double canonical(Mt64* s) {
    const double sum = (double)mt64_next(s) * 1.0;
    double r = sum / 18446744073709551616.0; /* 2^64 */
    if (r >= 1.0) r = nextafter(1.0, 0.0);
    return r;
}

/* std::normal_distribution<double> (libstdc++: Marsaglia polar, one cached value) */
typedef struct {
    double mean, stddev, saved;
    int have;
} Normal;

static double normal_next(Normal* d, Mt64* s) {
    double ret;
    if (d->have) {
        d->have = 0;
        ret = d->saved;
    } else {
        double x, y, r2;
        do {
            x = 2.0 * canonical(s) - 1.0;
            y = 2.0 * canonical(s) - 1.0;
            r2 = x * x + y * y;
        } while (r2 > 1.0 || r2 == 0.0);
        const double mult = sqrt(-2 * log(r2) / r2);
        d->saved = x * mult;
        d->have = 1;
        ret = y * mult;
    }
    return ret * d->stddev + d->mean;
}

/* FieldLine, image.cpp:143-162 */
static double fl_value(const double* f, int n1, double h, double o, double x) {
    const double u = (x - o) / h;
    if (u <= 0.0) return f[0];
    if (u >= n1 - 1) return f[n1 - 1];
    const double fi = floor(u);
    const int i = (int)fi;
    const double w = u - fi;
    return (1.0 - w) * f[i] + w * f[i + 1];
}

static double fl_slope(const double* f, int n1, double h, double o, double x) {
    const double u = (x - o) / h;
    if (u <= 0.0 || u >= n1 - 1) return 0.0;
    double fi = floor(u);
    if (fi == u) fi -= 1.0;
    const int i = (int)fi < 0 ? 0 : (int)fi;
    return (f[i + 1] - f[i]) / h;
}

/* invert_monotone, image.cpp:164-183 */
static double invert_monotone(const double* f, int n1, double h, double o, double sign, double y,
                              double tol) {
    double bmax = 0.0;
    for (int i = 0; i < n1; ++i) bmax = dmax(bmax, fabs(f[i]));
    if (bmax == 0.0) return y;
    double lo = y - bmax, hi = y + bmax;
#define PSI(x) ((x) + sign * fl_value(f, n1, h, o, (x)) - y)
    double flo = PSI(lo), fhi = PSI(hi);
    while (flo > 0.0) {
        lo -= bmax + h;
        flo = PSI(lo);
    }
    while (fhi < 0.0) {
        hi += bmax + h;
        fhi = PSI(hi);
    }
    while (hi - lo > tol) {
        const double mid = 0.5 * (lo + hi);
        if (PSI(mid) <= 0.0) lo = mid;
        else hi = mid;
    }
#undef PSI
    return 0.5 * (lo + hi);
}

/* simulate_pair, image.cpp:187-224 */
int oracle_simulate_pair(const epc_grid* gg, const double* truth, const double* b,
                         double noise_sigma, unsigned long long seed, double feas_margin,
                         double* up, double* um, char* msg, size_t msglen) {
    G g;
    int rc = grid_make(gg, &g, msg, msglen);
    if (rc) return rc;
    const double dmx = d1_norm_inf(&g, b);
    if (dmx > 1.0 - feas_margin) {
        set_msg(msg, msglen, "simulate_pair: field infeasible, max|D1 b| = %f", dmx);
        return EPC_ERR_INVALID_ARGUMENT;
    }
    const double tol = 1e-10 * g.h1;
    for (long long c = 0; c < g.ncol; ++c) {
        const Interp tr = column_of(&g, truth, c);
        const double* f = b + c * g.n1;
        for (int i = 0; i < g.m1; ++i) {
            const double y = g.o1 + (i + 0.5) * g.h1;
            const double xp = invert_monotone(f, g.n1, g.h1, g.o1, +1.0, y, tol);
            up[c * g.m1 + i] = ip_value(&tr, xp) / (1.0 + fl_slope(f, g.n1, g.h1, g.o1, xp));
            const double xm = invert_monotone(f, g.n1, g.h1, g.o1, -1.0, y, tol);
            um[c * g.m1 + i] = ip_value(&tr, xm) / (1.0 - fl_slope(f, g.n1, g.h1, g.o1, xm));
        }
    }
    if (noise_sigma > 0.0) {
        Mt64* s = (Mt64*)malloc(sizeof(Mt64));
        mt64_seed(s, seed);
        Normal d = {0.0, noise_sigma, 0.0, 0};
        for (long long i = 0; i < g.ncell; ++i) up[i] += normal_next(&d, s);
        for (long long i = 0; i < g.ncell; ++i) um[i] += normal_next(&d, s);
        free(s);
    }
    return EPC_OK;
}

/* ======================================================================
 * The reference's test-side helpers of the path
 * ====================================================================== */

/* avg_x1, operators.cpp:27-37 */
int oracle_avg_x1(const epc_grid* gg, const double* b, double* out) {
    G g;
    int rc = grid_make(gg, &g, NULL, 0);
    if (rc) return rc;
    for (long long c = 0; c < g.ncol; ++c)
        for (int i = 0; i < g.m1; ++i)
            out[c * g.m1 + i] = 0.5 * (b[c * g.n1 + i] + b[c * g.n1 + i + 1]);
    return EPC_OK;
}

/* diff_x1, operators.cpp:40-52 */
int oracle_diff_x1(const epc_grid* gg, const double* b, double* out) {
    G g;
    int rc = grid_make(gg, &g, NULL, 0);
    if (rc) return rc;
    const double ih = 1.0 / g.h1;
    for (long long c = 0; c < g.ncol; ++c)
        for (int i = 0; i < g.m1; ++i)
            out[c * g.m1 + i] = (b[c * g.n1 + i + 1] - b[c * g.n1 + i]) * ih;
    return EPC_OK;
}

/* diff_x1_adjoint, operators.cpp:54-68 */
int oracle_diff_x1_adjoint(const epc_grid* gg, const double* r, double* out) {
    G g;
    int rc = grid_make(gg, &g, NULL, 0);
    if (rc) return rc;
    const double ih = 1.0 / g.h1;
    const int m1 = g.m1, n1 = g.n1;
    for (long long c = 0; c < g.ncol; ++c) {
        const double* rc_ = r + c * m1;
        double* oc = out + c * n1;
        oc[0] = -rc_[0] * ih;
        for (int i = 1; i < m1; ++i) oc[i] = (rc_[i - 1] - rc_[i]) * ih;
        oc[m1] = rc_[m1 - 1] * ih;
    }
    return EPC_OK;
}

int oracle_smoother_hessian_apply(const epc_grid* gg, const double* b, double* out) {
    G g;
    int rc = grid_make(gg, &g, NULL, 0);
    if (rc) return rc;
    smoother_hessian_apply(&g, b, out);
    return EPC_OK;
}

/* TridiagBlocks::apply, operators.cpp:202-216: y += s T x */
int oracle_tridiag_apply(const epc_grid* gg, const double* diag, const double* off,
                         const double* x, double s, double* y) {
    G g;
    int rc = grid_make(gg, &g, NULL, 0);
    if (rc) return rc;
    const int m1 = g.m1, n1 = g.n1;
    for (long long c = 0; c < g.ncol; ++c) {
        const double* xc = x + c * n1;
        const double* d = diag + c * n1;
        const double* o = off + c * n1;
        double* yc = y + c * n1;
        for (int i = 0; i <= m1; ++i) {
            double acc = d[i] * xc[i];
            if (i > 0) acc += o[i - 1] * xc[i - 1];
            if (i < m1) acc += o[i] * xc[i + 1];
            yc[i] += s * acc;
        }
    }
    return EPC_OK;
}

/* tridiag_solve_batched, operators.cpp:264-273 (factorize, then solve) */
int oracle_tridiag_solve_batched(const epc_grid* gg, const double* diag, const double* off,
                                 const double* rhs, double* x, char* msg, size_t msglen) {
    G g;
    int rc = grid_make(gg, &g, msg, msglen);
    if (rc) return rc;
    double *fd = dalloc(g.nface), *fl = dalloc(g.nface);
    rc = tridiag_factorize(&g, diag, off, fd, fl, msg, msglen);
    if (rc == EPC_OK) {
        memcpy(x, rhs, sizeof(double) * (size_t)g.nface);
        tridiag_solve(&g, fd, fl, x);
    }
    free(fd);
    free(fl);
    return rc;
}

/* DctCoupledSolver::apply, operators.cpp:420-446 */
int oracle_dct_apply(const epc_grid* gg, const double* z, double alpha, double rho, double* out) {
    G g;
    int rc = grid_make(gg, &g, NULL, 0);
    if (rc) return rc;
    const double V = g.V;
    const int n1 = g.n1, m2 = g.m2, m3 = g.m3;
    const double w2 = alpha * V / (g.h2 * g.h2);
    const double w3 = alpha * V / (g.h3 * g.h3);
    const long long layer = (long long)n1 * m2;
    for (long long c = 0; c < g.ncol; ++c) {
        const int j = (int)(c % m2), k = (int)(c / m2);
        const double* zc = z + c * n1;
        double* oc = out + c * n1;
        for (int i = 0; i < n1; ++i) oc[i] = rho * V * zc[i];
        if (j > 0)
            for (int i = 0; i < n1; ++i) oc[i] += w2 * (zc[i] - zc[i - n1]);
        if (j + 1 < m2)
            for (int i = 0; i < n1; ++i) oc[i] += w2 * (zc[i] - zc[i + n1]);
        if (m3 > 1) {
            if (k > 0)
                for (int i = 0; i < n1; ++i) oc[i] += w3 * (zc[i] - zc[i - layer]);
            if (k + 1 < m3)
                for (int i = 0; i < n1; ++i) oc[i] += w3 * (zc[i] - zc[i + layer]);
        }
    }
    return EPC_OK;
}

/* DistanceEval::hessian_apply (objective.cpp:128-147) with jac_lo / jac_hi
 * of distance() at b (objective.cpp:93-126, residual_column) */
int oracle_distance_hessian_apply(const epc_grid* gg, const double* iplus, const double* iminus,
                                  const double* b, const double* p, double* out) {
    G g;
    int rc = grid_make(gg, &g, NULL, 0);
    if (rc) return rc;
    const int m1 = g.m1, n1 = g.n1;
    const double V = g.V;
    double *r = dalloc(m1), *jlo = dalloc(m1), *jhi = dalloc(m1);
    memset(out, 0, sizeof(double) * (size_t)g.nface);
    for (long long c = 0; c < g.ncol; ++c) {
        Interp ip = column_of(&g, iplus, c), im = column_of(&g, iminus, c);
        residual_column(&ip, &im, &g, b + c * n1, r, jlo, jhi);
        const double* pc = p + c * n1;
        double* oc = out + c * n1;
        for (int i = 0; i < m1; ++i) {
            const double jp = jlo[i] * pc[i] + jhi[i] * pc[i + 1];
            oc[i] += V * jlo[i] * jp;
            oc[i + 1] += V * jhi[i] * jp;
        }
    }
    free(r);
    free(jlo);
    free(jhi);
    return EPC_OK;
}

/* is_strictly_feasible, objective.cpp:35-37: 1 / 0, or a negative error */
int oracle_is_strictly_feasible(const epc_grid* gg, const double* b) {
    G g;
    int rc = grid_make(gg, &g, NULL, 0);
    if (rc) return -rc;
    return d1_norm_inf(&g, b) <= 1.0 - 1e-10 ? 1 : 0;
}

