// model.cuh — per-cell image model shared by the ADMM and GN kernels.
//
// Restates, per cell, the reference's 1D column interpolant
// (AxisInterpolant::value/slope, proj/src/image.cpp:24-46) and the residual /
// Jacobian of one cell (detail::residual_column, proj/src/objective.cpp:48-73)
// with the same operation order, so values are bitwise the reference's.
#pragma once

#include <cmath>

#include "common.cuh"

// Division by the spacing h. IEEE division costs ~112 dependent cycles on
// sm_100a and stalls in-order issue; when h is a power of two (h = 1 in every
// BASELINE config) x / h and x * (1/h) are the same real number, hence round
// identically, so the multiply is bitwise exact. HDiv selects at run time;
// HPow2 / HGen are the compile-time policies the column kernels are
// instantiated with.
struct HDiv {
    double h, inv;
    bool pow2;
    __device__ __forceinline__ double operator()(double x) const { return pow2 ? x * inv : x / h; }
};
struct HPow2 {
    double h, inv;
    __device__ __forceinline__ double operator()(double x) const { return x * inv; }
};
struct HGen {
    double h, inv;
    __device__ __forceinline__ double operator()(double x) const { return x / h; }
};

inline HDiv make_hdiv(double h) {
    int e = 0;
    const double m = std::frexp(h, &e);
    HDiv d;
    d.h = h;
    d.inv = 1.0 / h;
    d.pow2 = (m == 0.5) && std::isnormal(h) && std::isnormal(d.inv);
    return d;
}

template <class DH>
struct ColGeomT {
    int m1;
    double o1;
    DH dh;
};
using ColGeom = ColGeomT<HDiv>;

// Interior sample index of a position u for an m-sample column, clamped so
// that s[i] and s[i + 1] are in range (m >= 2); for u outside the interior the
// loaded values are discarded by the caller's select.
__device__ __forceinline__ int interp_index(double fi, int m) {
    int i = (int)fi;  // saturating conversion; NaN -> 0
    i = i < 0 ? 0 : i;
    return i > m - 2 ? (m - 2 < 0 ? 0 : m - 2) : i;
}

// AxisInterpolant::value (image.cpp:24-33); `s` = one image column (m1
// samples, shared or global memory). Branch-free: every case's value is
// formed with the reference's expression and the case tests pick one, so the
// two interpolations of a cell (and neighbouring cells) overlap in the
// pipeline instead of serialising on dependent branches.
template <class DH>
__device__ __forceinline__ double interp_value(const double* __restrict__ s,
                                               const ColGeomT<DH>& g, double x) {
#ifdef EPC_INTERP_BRANCHY
    const double u = g.dh(x - g.o1) - 0.5;
    const int m = g.m1;
    if (u <= -0.5 || u >= m - 0.5) return 0.0;
    if (u <= 0.0) return (u + 0.5) * 2.0 * s[0];
    if (u >= m - 1.0) return (m - 0.5 - u) * 2.0 * s[m - 1];
    const double fi = floor(u);
    const int i = (int)fi;
    const double w = u - fi;
    return (1.0 - w) * s[i] + w * s[i + 1];
#else
    const double u = g.dh(x - g.o1) - 0.5;
    const int m = g.m1;
    const double fi = floor(u);
    const int i = interp_index(fi, m);
    const int i1 = i + 1 < m ? i + 1 : i;
    const double w = u - fi;
    const double s0 = s[0], sm = s[m - 1], si = s[i], si1 = s[i1];
    const double v_in = (1.0 - w) * si + w * si1;
    const double v_lo = (u + 0.5) * 2.0 * s0;
    const double v_hi = (m - 0.5 - u) * 2.0 * sm;
    double v = (u >= m - 1.0) ? v_hi : v_in;
    v = (u <= 0.0) ? v_lo : v;
    return (u <= -0.5 || u >= m - 0.5) ? 0.0 : v;
#endif
}

// AxisInterpolant::slope (image.cpp:35-46): left-interval slope at kinks.
template <class DH>
__device__ __forceinline__ double interp_slope(const double* __restrict__ s,
                                               const ColGeomT<DH>& g, double x) {
#ifdef EPC_INTERP_BRANCHY
    const double u = g.dh(x - g.o1) - 0.5;
    const int m = g.m1;
    if (u <= -0.5 || u > m - 0.5) return 0.0;
    if (u <= 0.0) return g.dh(2.0 * s[0]);
    if (u > m - 1.0) return g.dh(-2.0 * s[m - 1]);
    double fi = floor(u);
    if (fi == u) fi -= 1.0;
    const int i = (int)fi;
    if (i < 0) return g.dh(2.0 * s[0]);
    return g.dh(s[i + 1] - s[i]);
#else
    const double u = g.dh(x - g.o1) - 0.5;
    const int m = g.m1;
    double fi = floor(u);
    if (fi == u) fi -= 1.0;
    const int iraw = (int)fi;
    const int i = interp_index(fi, m);
    const int i1 = i + 1 < m ? i + 1 : i;
    const double s0 = s[0], sm = s[m - 1], si = s[i], si1 = s[i1];
    // select the numerator, then one division by h (same rounded quotient)
    const double n_lo = 2.0 * s0, n_hi = -2.0 * sm, n_in = si1 - si;
    double num = iraw < 0 ? n_lo : n_in;
    num = (u > m - 1.0) ? n_hi : num;
    num = (u <= 0.0) ? n_lo : num;
    const double v = g.dh(num);
    return (u <= -0.5 || u > m - 0.5) ? 0.0 : v;
#endif
}

// One cell of detail::residual_column (objective.cpp:54-71). b0, b1 are the
// two faces of cell i. Jacobian only when jlo != nullptr.
template <class DH>
__device__ __forceinline__ double residual_cell(const double* __restrict__ ip,
                                                const double* __restrict__ im,
                                                const ColGeomT<DH>& g, int i, double b0, double b1,
                                                double* jlo, double* jhi) {
    const double xc = g.o1 + (i + 0.5) * g.dh.h;  // GridSpec::cell_center, grid.hpp:46
    const double a = 0.5 * (b0 + b1);
    const double d = g.dh(b1 - b0);
    const double vp = interp_value(ip, g, xc + a);
    const double vm = interp_value(im, g, xc - a);
    const double Tp = vp * (1.0 + d);
    const double Tm = vm * (1.0 - d);
    if (jlo) {
        const double gp = interp_slope(ip, g, xc + a);
        const double gm = interp_slope(im, g, xc - a);
        const double wa = 0.5 * (gp * (1.0 + d) + gm * (1.0 - d));
        const double wd = g.dh(vp + vm);
        *jlo = wa - wd;
        *jhi = wa + wd;
    }
    return Tp - Tm;
}
