// image.cu — the steps either side of the solve (
// proj/src/image.cpp): correct_pair (:226-253) and the metrics ssd (:255-263)
// and ncc (:265-283) after it, simulate_pair (:187-224) before it.
//
// correct_pair is per cell and uses the same interpolant arithmetic as the
// residual (model.cuh), so it is bitwise the reference's. simulate_pair
// inverts the monotone map x -> x +- b(x) per cell by the reference's
// bisection (invert_monotone, :141-183), one thread per cell, with the
// column's max|b| precomputed by a warp per column.
#include "common.cuh"
#include "kernels.h"
#include "model.cuh"

#include <algorithm>

// correct_pair (image.cpp:241-250): cp = I+(xc + a) (1 + d), cm = I-(xc - a) (1 - d)
template <class DH>
__global__ void k_correct_pair(const double* __restrict__ ip, const double* __restrict__ im,
                               const double* __restrict__ b, int m1, long long ncell, DH dh,
                               double o1, double* __restrict__ cp, double* __restrict__ cm) {
    const int n1 = m1 + 1;
    const ColGeomT<DH> geo{m1, o1, dh};
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < ncell;
         e += (long long)gridDim.x * blockDim.x) {
        const long long c = e / m1;
        const int i = (int)(e - c * m1);
        const double* bc = b + c * n1;
        const double xc = o1 + (i + 0.5) * dh.h;  // GridSpec::cell_center
        const double a = 0.5 * (bc[i] + bc[i + 1]);
        const double d = dh(bc[i + 1] - bc[i]);
        cp[e] = interp_value(ip + c * m1, geo, xc + a) * (1.0 + d);
        cm[e] = interp_value(im + c * m1, geo, xc - a) * (1.0 - d);
    }
}

// launched from this translation unit (a template kernel launched from
// another TU under -rdc=false may bind a host stub without device code)
void launch_correct_pair(epc_context* ctx, const double* ip, const double* im, const double* b,
                         int m1, long long ncell, HDiv hd, double o1, double* cp, double* cm) {
    const int blocks = (int)std::max<long long>(1, std::min<long long>((ncell + 255) / 256,
                                                                       (long long)ctx->num_sms * 16));
    if (hd.pow2)
        EPC_LAUNCH(ctx, "correct_pair", k_correct_pair<HPow2>, blocks, 256, 0, ip, im, b, m1, ncell,
                   HPow2{hd.h, hd.inv}, o1, cp, cm);
    else
        EPC_LAUNCH(ctx, "correct_pair", k_correct_pair<HGen>, blocks, 256, 0, ip, im, b, m1, ncell,
                   HGen{hd.h, hd.inv}, o1, cp, cm);
}

// max |b| over each column of n1 faces (invert_monotone's bmax, image.cpp:165-166)
__global__ void k_col_absmax(const double* __restrict__ b, int n1, long long ncol,
                             double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long c = w0; c < ncol; c += nw) {
        double m = 0.0;
        for (int i = lane; i < n1; i += 32) {
            const double v = fabs(b[c * n1 + i]);
            m = (m < v) ? v : m;
        }
        m = warp_max(m);
        if (lane == 0) out[c] = m;
    }
}

namespace {
// FieldLine (image.cpp:143-162): piecewise-linear b along one column
template <class DH>
struct FieldLine {
    const double* f;
    int n1;
    DH dh;
    double origin;
    __device__ double value(double x) const {
        const double u = dh(x - origin);
        if (u <= 0.0) return f[0];
        if (u >= n1 - 1) return f[n1 - 1];
        const double fi = floor(u);
        const int i = (int)fi;
        const double w = u - fi;
        return (1.0 - w) * f[i] + w * f[i + 1];
    }
    __device__ double slope(double x) const {
        const double u = dh(x - origin);
        if (u <= 0.0 || u >= n1 - 1) return 0.0;
        double fi = floor(u);
        if (fi == u) fi -= 1.0;
        const int i = (int)fi < 0 ? 0 : (int)fi;
        return dh(f[i + 1] - f[i]);
    }
};

// invert_monotone (image.cpp:164-183)
template <class DH>
__device__ double invert_monotone(const FieldLine<DH>& b, double bmax, double sign, double y,
                                  double tol) {
    if (bmax == 0.0) return y;
    double lo = y - bmax, hi = y + bmax;
    auto psi = [&](double x) { return x + sign * b.value(x) - y; };
    double flo = psi(lo), fhi = psi(hi);
    while (flo > 0.0) {
        lo -= bmax + b.dh.h;
        flo = psi(lo);
    }
    while (fhi < 0.0) {
        hi += bmax + b.dh.h;
        fhi = psi(hi);
    }
    while (hi - lo > tol) {
        const double mid = 0.5 * (lo + hi);
        if (psi(mid) <= 0.0) lo = mid;
        else hi = mid;
    }
    return 0.5 * (lo + hi);
}
}  // namespace

// simulate_pair's noiseless observations (image.cpp:200-214), thread per cell
template <class DH>
__global__ void k_simulate(const double* __restrict__ truth, const double* __restrict__ b,
                           const double* __restrict__ colmax, int m1, long long ncell, DH dh,
                           double o1, double tol, double* __restrict__ up,
                           double* __restrict__ um) {
    const int n1 = m1 + 1;
    const ColGeomT<DH> geo{m1, o1, dh};
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < ncell;
         e += (long long)gridDim.x * blockDim.x) {
        const long long c = e / m1;
        const int i = (int)(e - c * m1);
        const FieldLine<DH> fl{b + c * n1, n1, dh, o1};
        const double* tr = truth + c * m1;
        const double y = o1 + (i + 0.5) * dh.h;  // cell_center(0, i)
        const double bmax = colmax[c];
        const double xp = invert_monotone(fl, bmax, +1.0, y, tol);
        up[e] = interp_value(tr, geo, xp) / (1.0 + fl.slope(xp));
        const double xm = invert_monotone(fl, bmax, -1.0, y, tol);
        um[e] = interp_value(tr, geo, xm) / (1.0 - fl.slope(xm));
    }
}

void launch_simulate(epc_context* ctx, const double* truth, const double* b, const double* colmax,
                     int m1, long long ncell, HDiv hd, double o1, double tol, double* up,
                     double* um) {
    const int blocks = (int)std::max<long long>(1, std::min<long long>((ncell + 127) / 128,
                                                                       (long long)ctx->num_sms * 32));
    if (hd.pow2)
        EPC_LAUNCH(ctx, "simulate", k_simulate<HPow2>, blocks, 128, 0, truth, b, colmax, m1, ncell,
                   HPow2{hd.h, hd.inv}, o1, tol, up, um);
    else
        EPC_LAUNCH(ctx, "simulate", k_simulate<HGen>, blocks, 128, 0, truth, b, colmax, m1, ncell,
                   HGen{hd.h, hd.inv}, o1, tol, up, um);
}

// x += n (the additive noise, image.cpp:216-221)
__global__ void k_add(double* __restrict__ x, const double* __restrict__ n, long long len) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < len;
         i += (long long)gridDim.x * blockDim.x)
        x[i] += n[i];
}

// per-block partials of {sum a, sum b} (pass 1 of ncc) or, given the means,
// {sum da db, sum da^2, sum db^2} (pass 2); ssd uses pass 2 with zero means
// and takes sum (a - b)^2 from slot 3.
__global__ void __launch_bounds__(256) k_image_sums(const double* __restrict__ a,
                                                   const double* __restrict__ b, long long n,
                                                   int pass, double ma, double mb,
                                                   double* partials) {
    __shared__ double sh[8];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        if (pass == 1) {
            s0 += a[i];
            s1 += b[i];
        } else {
            const double da = a[i] - ma, db = b[i] - mb;
            s0 += da * db;
            s1 += da * da;
            s2 += db * db;
            const double d = a[i] - b[i];
            s3 += d * d;
        }
    }
    const double t0 = block_sum(s0, sh);
    __syncthreads();
    const double t1 = block_sum(s1, sh);
    __syncthreads();
    const double t2 = block_sum(s2, sh);
    __syncthreads();
    const double t3 = block_sum(s3, sh);
    if (threadIdx.x == 0) {
        double* o = partials + (size_t)blockIdx.x * 4;
        o[0] = t0;
        o[1] = t1;
        o[2] = t2;
        o[3] = t3;
    }
}

// swap axes a and b of a 3D array (axis 0 fastest), dims d of the input
// (swap_axes_raw, volume_io.cpp:184-201), thread per input element
__global__ void k_swap_axes(const double* __restrict__ in, double* __restrict__ out, int d0, int d1,
                            int d2, int a, int b) {
    const long long n = (long long)d0 * d1 * d2;
    int od[3] = {d0, d1, d2};
    const int t = od[a];
    od[a] = od[b];
    od[b] = t;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x) {
        int idx[3];
        idx[0] = (int)(e % d0);
        const long long q = e / d0;
        idx[1] = (int)(q % d1);
        idx[2] = (int)(q / d1);
        const int s = idx[a];
        idx[a] = idx[b];
        idx[b] = s;
        out[idx[0] + (long long)od[0] * (idx[1] + (long long)od[1] * idx[2])] = in[e];
    }
}
