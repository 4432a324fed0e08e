// multilevel.cu — restriction / prolongation between levels of the
// coarse-to-fine solve (proj/src/multilevel.cpp).
//
// restrict_image: area-weighted block averaging, one axis per pass
// (restrict_axis, multilevel.cpp:79-94). One thread per output element sums
// its fine intervals in the reference's order (o += w * s from 0), so the
// result is bitwise the reference's. The overlap weights are built on the
// host with the reference's formulas (make_axis_weights, :53-77).
//
// prolong_field: trilinear interpolation of the coarse staggered samples
// (:157-198), one thread per fine face, the reference's tap loop order with
// its zero-weight skips. Taps from the host (make_taps, :141-155). The
// feasibility rescue (:200-201) reuses the D1 max and the scale kernels.
#include "common.cuh"
#include "kernels.h"

__global__ void k_restrict_axis(const double* __restrict__ in, double* __restrict__ out,
                                long long pre, int mf, int mc, long long post,
                                const int* __restrict__ first, const int* __restrict__ off,
                                const double* __restrict__ w) {
    const long long n = pre * mc * post;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x) {
        const long long i = e % pre;
        const long long t2 = e / pre;
        const int c = (int)(t2 % mc);
        const long long p = t2 / mc;
        double o = 0.0;
        const int t0 = off[c], t1 = off[c + 1], f0 = first[c];
        for (int t = t0; t < t1; ++t) {
            const int f = f0 + (t - t0);
            o += w[t] * in[pre * (f + (long long)mf * p) + i];
        }
        out[e] = o;
    }
}

__global__ void k_prolong(const double* __restrict__ in, double* __restrict__ out, int fn1,
                          int fm2, int fm3, int cn1, int cm2, const MlTap* __restrict__ t1,
                          const MlTap* __restrict__ t2, const MlTap* __restrict__ t3) {
    const long long n = (long long)fn1 * fm2 * fm3;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e % fn1);
        const long long q = e / fn1;
        const int j = (int)(q % fm2);
        const int k = (int)(q / fm2);
        const MlTap a = t1[i], b = t2[j], c = t3[k];
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
                    v += wk * wj * wi * in[ii + (long long)cn1 * (jj + (long long)cm2 * kk)];
                }
            }
        }
        out[e] = v;
    }
}

// b = 0.5 (b + z) (the average restart, multilevel.cpp:271-274)
__global__ void k_average(double* __restrict__ b, const double* __restrict__ z, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        b[i] = 0.5 * (b[i] + z[i]);
}
