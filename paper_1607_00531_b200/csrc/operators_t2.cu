// operators_t2.cu — the reference's test-side helpers of the hot path as
// device entry points: the operators the reference's
// own tests use to check the path, each restating its loop's operations in
// the same order (bitwise):
//   avg_x1, diff_x1, diff_x1_adjoint        operators.cpp:27-68
//   smoother_hessian_apply                  operators.cpp:141-183
//   TridiagBlocks::apply                    operators.cpp:202-216
//   tridiag_solve_batched                   operators.cpp:218-273
//   DctCoupledSolver::apply                 operators.cpp:420-446
//   DistanceEval::hessian_apply             objective.cpp:128-147
//   is_strictly_feasible                    objective.cpp:35-37
// Thread per face or cell; the batched tridiagonal solve is a thread per
// column running the reference's factorize / solve_column loops.
#include "common.cuh"
#include "kernels.h"

namespace {

__global__ void k_avg_x1(const double* __restrict__ b, int m1, long long ncell,
                         double* __restrict__ out) {
    const int n1 = m1 + 1;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < ncell;
         e += (long long)gridDim.x * blockDim.x) {
        const long long c = e / m1;
        const int i = (int)(e - c * m1);
        const double* bc = b + c * n1;
        out[e] = 0.5 * (bc[i] + bc[i + 1]);
    }
}

__global__ void k_diff_x1(const double* __restrict__ b, int m1, long long ncell, double ih,
                          double* __restrict__ out) {
    const int n1 = m1 + 1;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < ncell;
         e += (long long)gridDim.x * blockDim.x) {
        const long long c = e / m1;
        const int i = (int)(e - c * m1);
        const double* bc = b + c * n1;
        out[e] = (bc[i + 1] - bc[i]) * ih;
    }
}

// oc[0] = -r[0] ih, oc[i] = (r[i-1] - r[i]) ih, oc[m1] = r[m1-1] ih
__global__ void k_diff_x1_adjoint(const double* __restrict__ r, int m1, long long nface, double ih,
                                  double* __restrict__ out) {
    const int n1 = m1 + 1;
    for (long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x; f < nface;
         f += (long long)gridDim.x * blockDim.x) {
        const long long c = f / n1;
        const int i = (int)(f - c * n1);
        const double* rc = r + c * m1;
        double v;
        if (i == 0) v = -rc[0] * ih;
        else if (i == m1) v = rc[m1 - 1] * ih;
        else v = (rc[i - 1] - rc[i]) * ih;
        out[f] = v;
    }
}

// V (D1^T D1 + D2^T D2 [+ D3^T D3]) b: the axis-1 stencil, then the j-1,
// j+1, k-1, k+1 neighbour terms, accumulated in that order
__global__ void k_smoother_apply(const double* __restrict__ b, int m1, int m2, int m3,
                                 long long nface, double w1, double w2, double w3,
                                 double* __restrict__ out) {
    const int n1 = m1 + 1;
    const long long layer = (long long)n1 * m2;
    for (long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x; f < nface;
         f += (long long)gridDim.x * blockDim.x) {
        const long long c = f / n1;
        const int i = (int)(f - c * n1);
        const int j = (int)(c % m2), k = (int)(c / m2);
        const double x = b[f];
        double v;
        if (i == 0) v = w1 * (x - b[f + 1]);
        else if (i == m1) v = w1 * (x - b[f - 1]);
        else v = w1 * (2.0 * x - b[f - 1] - b[f + 1]);
        if (j > 0) v += w2 * (x - b[f - n1]);
        if (j + 1 < m2) v += w2 * (x - b[f + n1]);
        if (m3 > 1) {
            if (k > 0) v += w3 * (x - b[f - layer]);
            if (k + 1 < m3) v += w3 * (x - b[f + layer]);
        }
        out[f] = v;
    }
}

// y += s T x per column (acc = d x_i + o_{i-1} x_{i-1} + o_i x_{i+1})
__global__ void k_tridiag_apply(const double* __restrict__ d, const double* __restrict__ o,
                                const double* __restrict__ x, int m1, long long nface, double s,
                                double* __restrict__ y) {
    const int n1 = m1 + 1;
    for (long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x; f < nface;
         f += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(f % n1);
        double acc = d[f] * x[f];
        if (i > 0) acc += o[f - 1] * x[f - 1];
        if (i < m1) acc += o[f] * x[f + 1];
        y[f] += s * acc;
    }
}

// TridiagFactor::factorize + solve_column, one thread per column; the lowest
// column with a nonpositive pivot is reported through bad (atomicMin)
__global__ void k_tridiag_solve_cols(const double* __restrict__ d, const double* __restrict__ o,
                                     double* __restrict__ fd, double* __restrict__ fl,
                                     double* __restrict__ x, int n1, long long ncol,
                                     long long* bad) {
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < ncol;
         c += (long long)gridDim.x * blockDim.x) {
        const double* dc = d + c * n1;
        const double* oc = o + c * n1;
        double* pd = fd + c * n1;
        double* pl = fl + c * n1;
        double* xc = x + c * n1;
        double prev = dc[0];
        bool ok = prev > 0.0;
        pd[0] = prev;
        for (int i = 1; i < n1 && ok; ++i) {
            const double li = oc[i - 1] / pd[i - 1];
            pl[i - 1] = li;
            const double piv = dc[i] - li * oc[i - 1];
            ok = piv > 0.0;
            pd[i] = piv;
        }
        if (!ok) {
            atomicMin((unsigned long long*)bad, (unsigned long long)c);
            continue;
        }
        pl[n1 - 1] = 0.0;
        for (int i = 1; i < n1; ++i) xc[i] -= pl[i - 1] * xc[i - 1];
        for (int i = 0; i < n1; ++i) xc[i] /= pd[i];
        for (int i = n1 - 2; i >= 0; --i) xc[i] -= pl[i] * xc[i + 1];
    }
}

// Gt z = rho V z + w2 (z - z_{j-1}) + w2 (z - z_{j+1}) [+ w3 k terms]
__global__ void k_dct_apply(const double* __restrict__ z, int n1, int m2, int m3, long long nface,
                            double rv, double w2, double w3, double* __restrict__ out) {
    const long long layer = (long long)n1 * m2;
    for (long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x; f < nface;
         f += (long long)gridDim.x * blockDim.x) {
        const long long c = f / n1;
        const int j = (int)(c % m2), k = (int)(c / m2);
        const double x = z[f];
        double v = rv * x;
        if (j > 0) v += w2 * (x - z[f - n1]);
        if (j + 1 < m2) v += w2 * (x - z[f + n1]);
        if (m3 > 1) {
            if (k > 0) v += w3 * (x - z[f - layer]);
            if (k + 1 < m3) v += w3 * (x - z[f + layer]);
        }
        out[f] = v;
    }
}

// H_D p = V Jr^T (Jr p): face f gathers cell f-1 (V jhi jp) then cell f
// (V jlo jp), the order of the reference's cell loop, from 0
__global__ void k_distance_hv(const double* __restrict__ jlo, const double* __restrict__ jhi,
                              const double* __restrict__ p, int m1, long long nface, double V,
                              double* __restrict__ out) {
    const int n1 = m1 + 1;
    for (long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x; f < nface;
         f += (long long)gridDim.x * blockDim.x) {
        const long long c = f / n1;
        const int i = (int)(f - c * n1);
        const double* pc = p + c * n1;
        const long long cc = c * m1;
        double v = 0.0;
        if (i > 0) {
            const double jp = jlo[cc + i - 1] * pc[i - 1] + jhi[cc + i - 1] * pc[i];
            v += V * jhi[cc + i - 1] * jp;
        }
        if (i < m1) {
            const double jp = jlo[cc + i] * pc[i] + jhi[cc + i] * pc[i + 1];
            v += V * jlo[cc + i] * jp;
        }
        out[f] = v;
    }
}

// max_i |(D1 b)_i| per block (norm_inf(diff_x1(b)), objective.cpp:36)
__global__ void k_d1_absmax(const double* __restrict__ b, int m1, long long ncell, double ih,
                            double* part) {
    __shared__ double sh[32];
    const int n1 = m1 + 1;
    double m = 0.0;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < ncell;
         e += (long long)gridDim.x * blockDim.x) {
        const long long c = e / m1;
        const int i = (int)(e - c * m1);
        const double v = fabs((b[c * n1 + i + 1] - b[c * n1 + i]) * ih);
        m = m < v ? v : m;
    }
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = t < sh[w] ? sh[w] : t;
        part[blockIdx.x] = t;
    }
}

}  // namespace

namespace {
int blocks_for(epc_context* ctx, long long n) {
    return (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, (long long)ctx->num_sms * 16));
}
}  // namespace

void launch_avg_x1(epc_context* ctx, const double* b, int m1, long long ncell, double* out) {
    EPC_LAUNCH(ctx, "avg_x1", k_avg_x1, blocks_for(ctx, ncell), 256, 0, b, m1, ncell, out);
}
void launch_diff_x1(epc_context* ctx, const double* b, int m1, long long ncell, double ih,
                    double* out) {
    EPC_LAUNCH(ctx, "diff_x1", k_diff_x1, blocks_for(ctx, ncell), 256, 0, b, m1, ncell, ih, out);
}
void launch_diff_x1_adjoint(epc_context* ctx, const double* r, int m1, long long nface, double ih,
                            double* out) {
    EPC_LAUNCH(ctx, "diff_x1_adjoint", k_diff_x1_adjoint, blocks_for(ctx, nface), 256, 0, r, m1,
               nface, ih, out);
}
void launch_smoother_apply(epc_context* ctx, const double* b, int m1, int m2, int m3,
                           long long nface, double w1, double w2, double w3, double* out) {
    EPC_LAUNCH(ctx, "smoother_apply", k_smoother_apply, blocks_for(ctx, nface), 256, 0, b, m1, m2,
               m3, nface, w1, w2, w3, out);
}
void launch_tridiag_apply(epc_context* ctx, const double* d, const double* o, const double* x,
                          int m1, long long nface, double s, double* y) {
    EPC_LAUNCH(ctx, "tridiag_apply", k_tridiag_apply, blocks_for(ctx, nface), 256, 0, d, o, x, m1,
               nface, s, y);
}
void launch_tridiag_solve_cols(epc_context* ctx, const double* d, const double* o, double* fd,
                               double* fl, double* x, int n1, long long ncol, long long* bad) {
    EPC_LAUNCH(ctx, "tridiag_solve", k_tridiag_solve_cols, blocks_for(ctx, ncol), 256, 0, d, o, fd,
               fl, x, n1, ncol, bad);
}
void launch_dct_apply(epc_context* ctx, const double* z, int n1, int m2, int m3, long long nface,
                      double rv, double w2, double w3, double* out) {
    EPC_LAUNCH(ctx, "dct_apply", k_dct_apply, blocks_for(ctx, nface), 256, 0, z, n1, m2, m3, nface,
               rv, w2, w3, out);
}
void launch_distance_hv(epc_context* ctx, const double* jlo, const double* jhi, const double* p,
                        int m1, long long nface, double V, double* out) {
    EPC_LAUNCH(ctx, "distance_hv", k_distance_hv, blocks_for(ctx, nface), 256, 0, jlo, jhi, p, m1,
               nface, V, out);
}
int launch_d1_absmax(epc_context* ctx, const double* b, int m1, long long ncell, double ih,
                     double* part) {
    const int nb = std::min(blocks_for(ctx, ncell), 1024);
    EPC_LAUNCH(ctx, "d1_absmax", k_d1_absmax, nb, 256, 0, b, m1, ncell, ih, part);
    return nb;
}

// GnHessian::preconditioner_blocks().diag == full_diagonal()
// (objective.cpp:333-348): the column part's diagonal plus cross_diag(j, k)
// (objective.cpp:296-300), w2 * (1 or 2) [+ w3 * (1 or 2) in 3D].
__global__ void k_cross_diag_add(const double* diag, int n1, int m2, int m3, int dim,
                                 long long nface, double w2, double w3, double* out) {
    for (long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x; f < nface;
         f += (long long)gridDim.x * blockDim.x) {
        const long long c = f / n1;
        const int j = (int)(c % m2), k = (int)(c / m2);
        double cd = w2 * ((j == 0 || j == m2 - 1) ? 1.0 : 2.0);
        if (dim == 3) cd += w3 * ((k == 0 || k == m3 - 1) ? 1.0 : 2.0);
        out[f] = diag[f] + cd;
    }
}

// the Jacobi preconditioner's apply (gn_pcg.cpp:41-47): z = r / diag
__global__ void k_div_elem(const double* r, const double* d, long long n, double* z) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        z[i] = r[i] / d[i];
}

void launch_cross_diag_add(epc_context* ctx, const double* diag, int n1, int m2, int m3, int dim,
                           long long nface, double w2, double w3, double* out) {
    EPC_LAUNCH(ctx, "cross_diag_add", k_cross_diag_add, blocks_for(ctx, nface), 256, 0, diag, n1, m2,
               m3, dim, nface, w2, w3, out);
}
void launch_div_elem(epc_context* ctx, const double* r, const double* d, long long n, double* z) {
    EPC_LAUNCH(ctx, "div_elem", k_div_elem, blocks_for(ctx, n), 256, 0, r, d, n, z);
}
