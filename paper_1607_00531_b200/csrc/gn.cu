// gn.cu — GN-PCG per-iteration kernels on sm_100a.
//
// Restates objective_gn (proj/src/objective.cpp:231-264) with distance
// (:93-126), smoother (:166-183, smoother_hessian_apply operators.cpp:141-183)
// and penalty (:185-229); the GnHessian column blocks (:266-300) and its
// matrix-free apply (:302-331); TridiagFactor::factorize / solve_column
// (operators.cpp:218-255) for the block-Jacobi preconditioner
// (gn_pcg.cpp:48-54); and the vector work of pcg (gn_pcg.cpp:92-131).
//
// Every per-element quantity (residual, Jacobian, gradient, Hessian blocks,
// stencil products, axpys, the per-column LDL^T and its solves) is computed
// with the reference's operation order and is bitwise identical. The global
// scalar reductions (dot/norm2, grid.cpp:60-64, sequential in the
// reference) are fixed-order tree sums here: deterministic run to run,
// within a few ulps of the sequential sums.
#include "common.cuh"
#include "kernels.h"

#include <algorithm>
#include "model.cuh"

// phi, phi_d1, phi_d2 (objective.cpp:17-33)
__device__ __forceinline__ double phi_v(double x) {
    if (fabs(x) >= 1.0) return __longlong_as_double(0x7ff0000000000000LL);  // +inf
    const double x2 = x * x;
    return x2 * x2 / (1.0 - x2);
}
__device__ __forceinline__ double phi_d1(double x) {
    const double x2 = x * x, x3 = x2 * x;
    const double d = 1.0 - x2;
    return (4.0 * x3 - 2.0 * x3 * x2) / (d * d);
}
__device__ __forceinline__ double phi_d2(double x) {
    const double x2 = x * x;
    const double d = 1.0 - x2;
    return 2.0 * x2 * (x2 * x2 - 3.0 * x2 + 6.0) / (d * d * d);
}

// ---------------------------------------------------------------------------
// cells: residual, Jacobian, penalty terms; partial sums per block:
// {sum r^2, sum (D1 b)^2, sum phi(D1 b), max |D1 b|}
// ---------------------------------------------------------------------------
#ifndef EPC_GN_CELLS_MINB
#define EPC_GN_CELLS_MINB 4  // 64 registers, 4 blocks per SM: 41 -> 30 us at C2 (measured)
#endif
__global__ void __launch_bounds__(256, EPC_GN_CELLS_MINB) k_gn_cells(GnCellArgs A) {
    __shared__ double sh[16];
    const ColGeom geo{A.m1, A.o1, A.dh};
    const double ih = 1.0 / A.dh.h;
    const double wpen = A.beta * A.V;
    double s_r = 0.0, s_d = 0.0, s_p = 0.0, mx = 0.0;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < A.ncell;
         e += (long long)gridDim.x * blockDim.x) {
        const long long c = e / A.m1;
        const int i = (int)(e - c * A.m1);
        const double* bc = A.b + c * A.n1;
        const double b0 = bc[i], b1 = bc[i + 1];
        double jl = 0.0, jh = 0.0;
        const double r = residual_cell(A.ip + c * A.m1, A.im + c * A.m1, geo, i, b0, b1,
                                       A.jlo ? &jl : nullptr, &jh);
        if (A.r) A.r[e] = r;
        if (A.jlo) {
            A.jlo[e] = jl;
            A.jhi[e] = jh;
        }
        const bool own = e >= A.sum_lo && e < A.sum_hi;
        if (own) s_r += r * r;
        const double d1 = (b1 - b0) * ih;  // diff_x1 (operators.cpp:40-52)
        if (own) s_d += d1 * d1;
        const double ad = fabs(d1);
        if (own) mx = (mx < ad) ? ad : mx;
        if (A.beta > 0.0) {
            if (own) s_p += phi_v(d1);
            if (A.dphi) A.dphi[e] = wpen * phi_d1(d1) * ih;  // penalty(), objective.cpp:217
            if (A.phi2) A.phi2[e] = phi_d2(d1);
        }
    }
    const double t0 = block_sum(s_r, sh);
    __syncthreads();
    const double t1 = block_sum(s_d, sh);
    __syncthreads();
    const double t2 = block_sum(s_p, sh);
    __syncthreads();
    double m = warp_max(mx);
    if ((threadIdx.x & 31) == 0) sh[8 + (threadIdx.x >> 5)] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double mm = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mm = (mm < sh[8 + w]) ? sh[8 + w] : mm;
        double* o = A.partials + (size_t)blockIdx.x * 4;
        o[0] = t0;
        o[1] = t1;
        o[2] = t2;
        o[3] = mm;
    }
}

// ---------------------------------------------------------------------------
// faces: gradient of J_GN = D + alpha S + P (objective.cpp:93-126, 166-183,
// 196-229, axpys at 252-257); partial sums per block: {sum (D2 b)^2,
// sum (D3 b)^2, sum grad . dir}
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_gn_faces(GnFaceArgs A) {
    __shared__ double sh[8];
    const int n1 = A.n1, m1 = A.m1, m2 = A.m2, m3 = A.m3;
    const long long layer = (long long)n1 * m2;
    double s2 = 0.0, s3 = 0.0, sgd = 0.0;
    for (long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x; f < A.nface;
         f += (long long)gridDim.x * blockDim.x) {
        const long long c = f / n1;
        const int i = (int)(f - c * n1);
        const int j = (int)(c % m2), k = (int)(c / m2);
        const double* b = A.b;
        const double bf = b[f];
        const bool own = f >= A.sum_lo && f < A.sum_hi;
        // diff_perp sums (g_value / smoother value)
        if (own && j + 1 < m2) {
            const double o = (b[f + n1] - bf) * A.ih2;
            s2 += o * o;
        }
        if (own && m3 > 1 && k + 1 < m3) {
            const double o = (b[f + layer] - bf) * A.ih3;
            s3 += o * o;
        }
        if (A.grad) {
            const long long ce = c * m1 + i;  // cell i of this column
            // distance gradient: cell f-1 then cell f (objective.cpp:114-118)
            double dg = 0.0;
            if (i >= 1) dg += A.V * A.jhi[ce - 1] * A.r[ce - 1];
            if (i < m1) dg += A.V * A.jlo[ce] * A.r[ce];
            // smoother_hessian_apply (operators.cpp:141-183)
            double sg;
            if (i == 0) sg = A.w1 * (bf - b[f + 1]);
            else if (i == m1) sg = A.w1 * (bf - b[f - 1]);
            else sg = A.w1 * (2.0 * bf - b[f - 1] - b[f + 1]);
            if (j > 0) sg += A.w2 * (bf - b[f - n1]);
            if (j + 1 < m2) sg += A.w2 * (bf - b[f + n1]);
            if (m3 > 1) {
                if (k > 0) sg += A.w3 * (bf - b[f - layer]);
                if (k + 1 < m3) sg += A.w3 * (bf - b[f + layer]);
            }
            double g = dg + A.alpha * sg;
            if (A.beta > 0.0) {  // penalty gradient: += dphi(f-1), -= dphi(f)
                double pg = 0.0;
                if (i >= 1) pg += A.dphi[ce - 1];
                if (i < m1) pg -= A.dphi[ce];
                g += 1.0 * pg;
            }
            A.grad[f] = g;
            if (A.dir && own) sgd += g * A.dir[f];
        }
    }
    const double t0 = block_sum(s2, sh);
    __syncthreads();
    const double t1 = block_sum(s3, sh);
    __syncthreads();
    const double t2 = block_sum(sgd, sh);
    if (threadIdx.x == 0) {
        double* o = A.partials + (size_t)blockIdx.x * 3;
        o[0] = t0;
        o[1] = t1;
        o[2] = t2;
    }
}

// ---------------------------------------------------------------------------
// GnHessian column blocks (objective.cpp:266-294) + preconditioner_blocks
// diagonal (objective.cpp:296-300, 339-348), per face.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_gn_hess(GnHessArgs A) {
    const int n1 = A.n1, m1 = A.m1, m2 = A.m2, m3 = A.m3;
    for (long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x; f < A.nface;
         f += (long long)gridDim.x * blockDim.x) {
        const long long c = f / n1;
        const int i = (int)(f - c * n1);
        const int j = (int)(c % m2), k = (int)(c / m2);
        const long long ce = c * m1 + i;
        // add_hessian_blocks: cell f-1 (d[i+1] += V jhi^2) then cell f (d[i] += V jlo^2)
        double d = 0.0, o = 0.0;
        if (i >= 1) d += A.V * A.jhi[ce - 1] * A.jhi[ce - 1];
        if (i < m1) {
            d += A.V * A.jlo[ce] * A.jlo[ce];
            o += A.V * A.jlo[ce] * A.jhi[ce];
        }
        // add_axis1_laplacian(alpha V) (operators.cpp:189-200)
        d += (i == 0 || i == m1) ? A.wl : 2.0 * A.wl;
        if (i < m1) o -= A.wl;
        d += A.gamma;  // add_identity
        if (A.beta > 0.0) {  // penalty blocks, objective.cpp:283-292
            if (i >= 1) d += A.wp * A.phi2[ce - 1];
            if (i < m1) {
                d += A.wp * A.phi2[ce];
                o -= A.wp * A.phi2[ce];
            }
        }
        A.diag[f] = d;
        A.off[f] = o;
        // cross_diag(j, k) (objective.cpp:296-300)
        double cd = A.w2 * ((j == 0 || j == m2 - 1) ? 1.0 : 2.0);
        if (A.dim == 3) cd += A.w3 * ((k == 0 || k == m3 - 1) ? 1.0 : 2.0);
        A.pdiag[f] = d + cd;
    }
}

// TridiagFactor::factorize (operators.cpp:218-246), one warp per column:
// coalesced staging, lane-0 pivot chain, coalesced write-back.
__global__ void __launch_bounds__(128) k_gn_factor(const double* pdiag, const double* off,
                                                  double* fd, double* fl, int n1, long long ncol,
                                                  int* col_err) {
    extern __shared__ __align__(16) double fsm[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double* sd = fsm + (size_t)wib * 4 * n1;
    double* so = sd + n1;
    double* rd = so + n1;
    double* rl = rd + n1;
    const int wpb = blockDim.x >> 5;
    for (long long c = (long long)blockIdx.x * wpb + wib; c < ncol; c += (long long)gridDim.x * wpb) {
        const size_t o = (size_t)c * n1;
        for (int i = lane; i < n1; i += 32) {
            sd[i] = pdiag[o + i];
            so[i] = off[o + i];
        }
        __syncwarp();
        int bad = 0;
        if (lane == 0) {
            double prev = sd[0];
            if (!(prev > 0.0)) bad = 1;
            else {
                rd[0] = prev;
                for (int i = 1; i < n1; ++i) {
                    const double oo = so[i - 1];
                    const double li = oo / rd[i - 1];
                    rl[i - 1] = li;
                    const double piv = sd[i] - li * oo;
                    if (!(piv > 0.0)) {
                        bad = 1;
                        break;
                    }
                    rd[i] = piv;
                }
                rl[n1 - 1] = 0.0;
            }
            col_err[c] = bad;
        }
        __syncwarp();
        for (int i = lane; i < n1; i += 32) {
            fd[o + i] = rd[i];
            fl[o + i] = rl[i];
        }
        __syncwarp();
    }
}

// The same factorization with one thread per column: a 256-thread block
// stages FCPW consecutive columns (one contiguous span) with coalesced loads,
// then thread c runs column c's pivot chain in shared memory (d over the
// staged diagonal, l over the staged off-diagonal, each read before it is
// overwritten) and the span is stored coalesced. Same operations in the same
// order as TridiagFactor::factorize (operators.cpp:218-246): bitwise.
constexpr int FCPW = 16;
__global__ void __launch_bounds__(256) k_gn_factor_cols(const double* pdiag, const double* off,
                                                       double* fd, double* fl, int n1,
                                                       long long ncol, int rs, int* col_err) {
    extern __shared__ __align__(16) double fsm[];
    double* X = fsm;            // diagonal -> pivots d
    double* Y = fsm + FCPW * rs;  // off-diagonal -> multipliers l
    const int tid = threadIdx.x;
    const unsigned un1 = (unsigned)n1;
    const long long ngroups = (ncol + FCPW - 1) / FCPW;
    for (long long gi = blockIdx.x; gi < ngroups; gi += gridDim.x) {
        const long long c0 = gi * FCPW;
        const int nc = (int)(ncol - c0 < FCPW ? ncol - c0 : FCPW);
        const size_t base = (size_t)c0 * n1;
        const int ne = nc * n1;
#pragma unroll 4
        for (int e = tid; e < ne; e += blockDim.x) {
            const int cc = (int)((unsigned)e / un1), i = e - cc * n1;
            X[cc * rs + i] = pdiag[base + e];
            Y[cc * rs + i] = off[base + e];
        }
        __syncthreads();
        if (tid < nc) {
            double* x = X + tid * rs;
            double* y = Y + tid * rs;
            int bad = 0;
            double prev = x[0];
            if (!(prev > 0.0)) {
                bad = 1;
            } else {
                for (int i = 1; i < n1; ++i) {
                    const double oo = y[i - 1];
                    const double li = oo / prev;
                    y[i - 1] = li;
                    const double piv = x[i] - li * oo;
                    if (!(piv > 0.0)) {
                        bad = 1;
                        break;
                    }
                    x[i] = piv;
                    prev = piv;
                }
                y[n1 - 1] = 0.0;
            }
            col_err[c0 + tid] = bad;
        }
        __syncthreads();
#pragma unroll 4
        for (int e = tid; e < ne; e += blockDim.x) {
            const int cc = (int)((unsigned)e / un1), i = e - cc * n1;
            fd[base + e] = X[cc * rs + i];
            fl[base + e] = Y[cc * rs + i];
        }
        __syncthreads();
    }
}

void launch_gn_factor_cols(epc_context* ctx, const double* pdiag, const double* off, double* fd,
                           double* fl, int n1, long long ncol, int* col_err) {
    const int rs = n1 | 1;
    const size_t smem = (size_t)2 * FCPW * rs * sizeof(double);
    cudaFuncSetAttribute(k_gn_factor_cols, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const long long groups = (ncol + FCPW - 1) / FCPW;
    const int blocks = (int)std::max<long long>(1, std::min<long long>(groups, (long long)ctx->num_sms * 8));
    EPC_LAUNCH(ctx, "gn_factor", k_gn_factor_cols, blocks, 256, smem, pdiag, off, fd, fl, n1, ncol, rs,
               col_err);
}

size_t gn_factor_cols_smem(int n1) { return (size_t)2 * FCPW * (n1 | 1) * sizeof(double); }

// GnHessian::apply (objective.cpp:302-331) fused with the PCG direction
// update p = z + beta p (gn_pcg.cpp:128); beta_mode: 0 -> p = z (first
// iteration: p = z copy), 1 -> p_new = z + beta * p_old, 2 -> use p_old as is.
// Writes p_new (when mode != 2) and y = H p; partial sum p . y per block.
__global__ void __launch_bounds__(256) k_gn_hv(GnHvArgs A) {
    __shared__ double sh[8];
    const int n1 = A.n1, m1 = A.m1, m2 = A.m2, m3 = A.m3;
    const long long layer = (long long)n1 * m2;
    auto P = [&](long long f) -> double {
        if (A.mode == 2) return A.p_old[f];
        if (A.mode == 0) return A.z[f];
        return A.z[f] + A.beta * A.p_old[f];
    };
    double s = 0.0;
    for (long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x; f < A.nface;
         f += (long long)gridDim.x * blockDim.x) {
        const long long c = f / n1;
        const int i = (int)(f - c * n1);
        const int j = (int)(c % m2), k = (int)(c / m2);
        const double x = P(f);
        double acc = A.diag[f] * x;
        if (i > 0) acc += A.off[f - 1] * P(f - 1);
        if (i < m1) acc += A.off[f] * P(f + 1);
        double y = acc;
        if (j > 0) y += A.w2 * (x - P(f - n1));
        if (j + 1 < m2) y += A.w2 * (x - P(f + n1));
        if (m3 > 1) {
            if (k > 0) y += A.w3 * (x - P(f - layer));
            if (k + 1 < m3) y += A.w3 * (x - P(f + layer));
        }
        A.y[f] = y;
        if (A.mode != 2) A.p_new[f] = x;
        if (f >= A.sum_lo && f < A.sum_hi) s += x * y;
    }
    const double t = block_sum(s, sh);
    if (threadIdx.x == 0 && A.partials) A.partials[blockIdx.x] = t;
}

// PCG update + preconditioner (gn_pcg.cpp:114-120) per column (warp):
// d += a p; r += (-a) q; partial sum r.r; z = M^{-1} r (none / jacobi /
// block-Jacobi LDL^T solve, operators.cpp:248-262); partial sum r.z.
// a_mode 0 skips the axpys (PCG start: z = M r0).
__global__ void __launch_bounds__(128) k_gn_update_prec(GnUpdArgs A) {
    extern __shared__ __align__(16) double usm[];
    __shared__ double red[2][4];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int n1 = A.n1;
    double* sv = usm + (size_t)wib * n1;
    const int wpb = blockDim.x >> 5;
    double rr = 0.0, rz = 0.0;
    for (long long c = (long long)blockIdx.x * wpb + wib; c < A.ncol; c += (long long)gridDim.x * wpb) {
        const size_t o = (size_t)c * n1;
        for (int i = lane; i < n1; i += 32) {
            double r = A.r[o + i];
            if (A.do_axpy) {
                A.d[o + i] += A.a * A.p[o + i];
                r += A.ma * A.q[o + i];
                A.r[o + i] = r;
            }
            rr += r * r;
            sv[i] = r;
        }
        __syncwarp();
        if (A.kind == EPC_PRECOND_BLOCK_JACOBI) {
            const double* fl = A.fl + o;
            const double* fd = A.fd + o;
            if (lane == 0) {
                double prev = sv[0];
                for (int i = 1; i < n1; ++i) {
                    const double cur = sv[i] - fl[i - 1] * prev;
                    sv[i] = cur;
                    prev = cur;
                }
            }
            __syncwarp();
            for (int i = lane; i < n1; i += 32) sv[i] = sv[i] / fd[i];
            __syncwarp();
            if (lane == 0) {
                double nxt = sv[n1 - 1];
                for (int i = n1 - 2; i >= 0; --i) {
                    const double cur = sv[i] - fl[i] * nxt;
                    sv[i] = cur;
                    nxt = cur;
                }
            }
            __syncwarp();
        } else if (A.kind == EPC_PRECOND_JACOBI) {
            for (int i = lane; i < n1; i += 32) sv[i] = sv[i] / A.pdiag[o + i];
            __syncwarp();
        }
        for (int i = lane; i < n1; i += 32) {
            const double zz = sv[i];
            A.z[o + i] = zz;
            rz += A.r[o + i] * zz;
        }
        __syncwarp();
    }
    rr = warp_sum(rr);
    rz = warp_sum(rz);
    if (lane == 0) {
        red[0][wib] = rr;
        red[1][wib] = rz;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < wpb; ++w) {
            a += red[0][w];
            b += red[1][w];
        }
        A.partials[(size_t)blockIdx.x * 2 + 0] = a;
        A.partials[(size_t)blockIdx.x * 2 + 1] = b;
    }
}

// y = x + t * d (the Wolfe trial point, gn_pcg.cpp:248-249; b_new at 265-266)
__global__ void k_axpy_point(const double* x, const double* d, double t, double* y, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        y[i] = x[i] + t * d[i];
}

// r = -g, plus partial sums {g.g} (pcg start, gn_pcg.cpp:97-103)
__global__ void __launch_bounds__(256) k_neg_norm(const double* g, double* r, long long n,
                                                 double* partials) {
    __shared__ double sh[8];
    double s = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double v = g[i];
        r[i] = -v;
        s += v * v;
    }
    const double t = block_sum(s, sh);
    if (threadIdx.x == 0) partials[blockIdx.x] = t;
}

// partial sums of {a.b, b.b} (dot(grad, d) and norm2(d))
__global__ void __launch_bounds__(256) k_dot2(const double* a, const double* b, long long n,
                                             double* partials) {
    __shared__ double sh[8];
    double s0 = 0.0, s1 = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        s0 += a[i] * b[i];
        s1 += b[i] * b[i];
    }
    const double t0 = block_sum(s0, sh);
    __syncthreads();
    const double t1 = block_sum(s1, sh);
    if (threadIdx.x == 0) {
        partials[blockIdx.x * 2] = t0;
        partials[blockIdx.x * 2 + 1] = t1;
    }
}

// GnHessian::apply alone (x given)
__global__ void k_gn_copy(const double* src, double* dst, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        dst[i] = src[i];
}
