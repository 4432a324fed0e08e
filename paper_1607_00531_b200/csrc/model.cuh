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

// AxisInterpolant::value (image.cpp:24-33); `s` = one image column (m1
// samples, shared or global memory).
template <class DH>
__device__ __forceinline__ double interp_value(const double* __restrict__ s,
                                               const ColGeomT<DH>& g, double x) {
    const double u = g.dh(x - g.o1) - 0.5;
    const int m = g.m1;
    if (u <= -0.5 || u >= m - 0.5) return 0.0;
    if (u <= 0.0) return (u + 0.5) * 2.0 * s[0];
    if (u >= m - 1.0) return (m - 0.5 - u) * 2.0 * s[m - 1];
    const double fi = floor(u);
    const int i = (int)fi;
    const double w = u - fi;
    return (1.0 - w) * s[i] + w * s[i + 1];
}

// AxisInterpolant::slope (image.cpp:35-46): left-interval slope at kinks.
template <class DH>
__device__ __forceinline__ double interp_slope(const double* __restrict__ s,
                                               const ColGeomT<DH>& g, double x) {
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
