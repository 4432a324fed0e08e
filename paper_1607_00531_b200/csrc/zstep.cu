// zstep.cu — ADMM z-step and dual update on sm_100a.
//
// The reference z-step (z_update, proj/src/admm.cpp:445-451, through
// DctCoupledSolver::solve, proj/src/operators.cpp:388-418) applies dense
// orthonormal DCT-II matrices along axes 2 and 3 (transform_axis2/3,
// operators.cpp:347-386): out[q][.] = sum_j C[q][j] in[j][.], j ascending,
// starting from 0. Each transform is therefore a small-M GEMM whose
// K-loop order we keep: every output accumulates k = 0..K-1 in order with
// separate multiply and add (-fmad=false), so z is bitwise the reference's.
// rhs formation (rho*V*(b+u)) is fused into the first GEMM's operand load,
// the spectral divide into the axis-3 forward GEMM's epilogue and the dual
// update (dual_update_and_residuals, admm.cpp:453-476) plus the residual /
// Lagrangian partial sums into the last GEMM's epilogue.
//
// Tiling: 64x64 output tile per 256-thread CTA, 16-deep K slabs staged in
// shared memory with register prefetch of the next slab; each thread owns a
// 4x4 strided sub-tile (conflict-free/broadcast shared loads). fp64 has no
// tensor-core path on this part that preserves the reference's rounding, so
// this is an FP64-pipe kernel by design.
#include "common.cuh"
#include "kernels.h"

#include <cstdlib>
#include <string>

namespace {
#ifndef EPC_GEMM_BK
#define EPC_GEMM_BK 16  // k-slab depth; 32 measured slower for three of the four transforms
#endif
#ifndef EPC_GEMM_MINB
#define EPC_GEMM_MINB 1  // resident CTAs per SM asked of the RM = 4 non-dual GEMMs (3: forward axis 2 0.287 -> 0.296 ms, scripts/r02mb_gpu.sh)
#endif
#ifndef EPC_GEMM_DB
#define EPC_GEMM_DB 1
#endif
#ifndef EPC_GEMM_MFIRST
#define EPC_GEMM_MFIRST 1
#endif
constexpr int BN = 64, BK = EPC_GEMM_BK, NT = 256;
constexpr int AR = NT / BK;  // A-tile rows loaded per pass (a thread per k column)
}

// RM rows per thread: BM = 16 RM output rows per CTA (RM = 4: 64; RM = 6: 96,
// which tiles the axis-3 transforms of m3 = 96 without a half-empty tile)
template <int PRO, int EPI, int RM>
// The dual epilogue needs more registers than the plain ones; capping it to
// three resident CTAs per SM (<= 85 registers) is faster than two with more
// registers (measured), the other variants fit three CTAs unforced.
__global__ void __launch_bounds__(NT, EPI == EPI_DUAL ? 3 : (RM == 4 ? EPC_GEMM_MINB : 1)) k_dct_gemm(GemmParams p) {
    constexpr int BM = 16 * RM;
    // DB: two K-slab buffers, one barrier per slab (the next slab is stored
    // into the other buffer while this one is read). Measured per transform
    // (scripts/r02db_gpu.sh): the dual GEMM (three CTAs per SM) 0.309 ->
    // 0.287 ms; the others (two CTAs per SM) 1-2% slower, so single-buffered
    constexpr bool DB = EPC_GEMM_DB && EPI == EPI_DUAL;
    __shared__ double As[DB ? 2 : 1][BK][BM + 1];  // +1: the transposing store is conflict-free
    __shared__ double Bs[DB ? 2 : 1][BK][BN];
    __shared__ double red[(NT / 32) * 6];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    // M tiles innermost in launch order: the CTAs sharing one B (column)
    // tile run together and its re-reads hit L2 (EPC_GEMM_MFIRST=0: N first)
    const bool mf = p.mfirst != 0;
    const int tm = mf ? blockIdx.x : blockIdx.y, tn = mf ? blockIdx.y : blockIdx.x;
    const int ntm = mf ? gridDim.x : gridDim.y, ntn = mf ? gridDim.y : gridDim.x;
    const int row0 = tm * BM;
    const long long col0 = (long long)tn * BN;
    const int pair = blockIdx.z;
    const long long zoff = (long long)pair * p.zstride;

    // this thread's B-load column (fixed across the K loop)
    const int ln = tid & 63, lk = tid >> 6;  // BK/4 rows lk, lk+4, ...
    const long long lcol = col0 + ln;
    const bool lcol_ok = lcol < p.N;
    const long long lmap = lcol_ok ? (lcol / p.cdiv) * p.cstride + (lcol % p.cdiv) : 0;
    double wrhs = 0.0;
    if (PRO == PRO_RHS) wrhs = p.rho[pair] * p.V;
    // this thread's A-load element
    const int am = tid / BK, ak = tid % BK;
    constexpr int NA = BM / AR, NB = BK / 4;  // A and B elements per thread per slab

    double acc[RM][4];
#pragma unroll
    for (int r = 0; r < RM; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;

    double ra[NA], rb[NB];
    auto load_tile = [&](int k0) {
#pragma unroll
        for (int t = 0; t < NA; ++t) {
            const int m = am + AR * t, k = k0 + ak;
            ra[t] = (row0 + m < p.M && k < p.K) ? __ldg(p.A + (size_t)(row0 + m) * p.K + k) : 0.0;
        }
#pragma unroll
        for (int t = 0; t < NB; ++t) {
            const int k = k0 + lk + 4 * t;
            double v = 0.0;
            if (lcol_ok && k < p.K) {
                const long long a = zoff + (long long)k * p.kstride + lmap;
                if (PRO == PRO_RHS) v = wrhs * (__ldg(p.in0 + a) + __ldg(p.in1 + a));
                else v = __ldg(p.in0 + a);
            }
            rb[t] = v;
        }
    };

    auto store_tile = [&](int buf) {
#pragma unroll
        for (int t = 0; t < NA; ++t) As[buf][ak][am + AR * t] = ra[t];
#pragma unroll
        for (int t = 0; t < NB; ++t) Bs[buf][lk + 4 * t][ln] = rb[t];
    };
    auto mac_slab = [&](int buf, int kend) {
        if (kend == BK) {
#pragma unroll
            for (int kk = 0; kk < BK; ++kk) {
                double a[RM], b[4];
#pragma unroll
                for (int r = 0; r < RM; ++r) a[r] = As[buf][kk][ty + 16 * r];
#pragma unroll
                for (int c = 0; c < 4; ++c) b[c] = Bs[buf][kk][tx + 16 * c];
#pragma unroll
                for (int r = 0; r < RM; ++r)
#pragma unroll
                    for (int c = 0; c < 4; ++c) acc[r][c] = acc[r][c] + a[r] * b[c];
            }
        } else {
            for (int kk = 0; kk < kend; ++kk) {
                double a[RM], b[4];
#pragma unroll
                for (int r = 0; r < RM; ++r) a[r] = As[buf][kk][ty + 16 * r];
#pragma unroll
                for (int c = 0; c < 4; ++c) b[c] = Bs[buf][kk][tx + 16 * c];
#pragma unroll
                for (int r = 0; r < RM; ++r)
#pragma unroll
                    for (int c = 0; c < 4; ++c) acc[r][c] = acc[r][c] + a[r] * b[c];
            }
        }
    };

    load_tile(0);
    if constexpr (DB) {
        store_tile(0);
        __syncthreads();
        int buf = 0;
        for (int k0 = 0; k0 < p.K; k0 += BK) {
            const bool more = k0 + BK < p.K;
            if (more) load_tile(k0 + BK);
            mac_slab(buf, min(BK, p.K - k0));
            if (more) store_tile(buf ^ 1);  // last read at the previous slab, behind its barrier
            __syncthreads();
            buf ^= 1;
        }
    } else {
        for (int k0 = 0; k0 < p.K; k0 += BK) {
            __syncthreads();
            store_tile(0);
            __syncthreads();
            if (k0 + BK < p.K) load_tile(k0 + BK);
            mac_slab(0, min(BK, p.K - k0));
        }
    }

    double ps[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    const bool act = (EPI == EPI_DUAL) ? (p.active == nullptr || p.active[pair] != 0) : true;
    // column index arithmetic once per column, in 32 bits when N allows
    // (every configuration here; 64-bit division costs ~100 instructions)
    const bool narrow = p.N <= 0x7fffffffLL;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const long long col = col0 + tx + 16 * c;
        if (col >= p.N) continue;
        long long cmap;
        int cq = 0;
        if (narrow) {
            const unsigned cu = (unsigned)col, cd = (unsigned)p.cdiv;
            const unsigned qd = cu / cd;
            cmap = (long long)qd * p.cstride + (long long)(cu - qd * cd);
            if (EPI == EPI_DIVIDE) cq = (int)(cu / (unsigned)p.n1);
        } else {
            cmap = (col / p.cdiv) * p.cstride + (col % p.cdiv);
            if (EPI == EPI_DIVIDE) cq = (int)(col / p.n1);
        }
        const int cbase = (EPI == EPI_DIVIDE) ? (p.div_axis == 3 ? cq : p.m2 * (cq % p.m3)) : 0;
#pragma unroll
        for (int r = 0; r < RM; ++r) {
            const int row = row0 + ty + 16 * r;
            if (row >= p.M) continue;
            const long long f = zoff + (long long)row * p.kstride + cmap;
            double v = acc[r][c];
            if (EPI == EPI_DIVIDE) {
                // axis 3: j = col / n1, cidx = j + m2 q3; axis 2: k = (col / n1) % m3, cidx = q2 + m2 k
                const int cidx = p.div_axis == 3 ? cbase + p.m2 * row : row + cbase;
                const double denom = p.alpha * p.V * p.lam23[cidx] + p.rho[pair] * p.V;
                p.out[f] = v / denom;
            } else if (EPI == EPI_DUAL) {
                if (act) {
                    p.out[f] = v;
                    const double bb = p.bvec[f];
                    const double diff = bb - v;
                    const double un = p.u_old[f] + diff;
                    p.u_new[f] = un;
                    const double dz = p.z_old[f] - v;
                    ps[0] += diff * diff;
                    ps[1] += dz * dz;
                    ps[2] += bb * bb;
                    ps[3] += v * v;
                    ps[4] += un * un;
                    ps[5] += un * diff;
                } else {
                    p.out[f] = p.z_old[f];
                    p.u_new[f] = p.u_old[f];
                }
            } else {
                p.out[f] = v;
            }
        }
    }
    if (EPI == EPI_DUAL) {
        const int w = tid >> 5, l = tid & 31;
#pragma unroll
        for (int s = 0; s < 6; ++s) {
            const double v = warp_sum(ps[s]);
            if (l == 0) red[w * 6 + s] = v;
        }
        __syncthreads();
        if (tid < 6) {
            double t = 0.0;
            for (int i = 0; i < NT / 32; ++i) t += red[i * 6 + tid];
            const long long blk = (long long)tm * ntn + tn;  // the same order either way
            const long long nblk = (long long)ntm * ntn;
            p.partials[((long long)pair * nblk + blk) * 6 + tid] = t;
        }
    }
}

// M tiles in grid x (launched first) unless the column tiles exceed grid y
static dim3 gemm_grid(GemmParams& p, int BM, int nz) {
    const unsigned tn = (unsigned)((p.N + BN - 1) / BN), tm = (unsigned)((p.M + BM - 1) / BM);
    p.mfirst = EPC_GEMM_MFIRST && tn <= 65535u;
    return p.mfirst ? dim3(tm, tn, (unsigned)nz) : dim3(tn, tm, (unsigned)nz);
}

void launch_dct_gemm_64(epc_context* ctx, const char* name, const GemmParams& p, int pro, int epi,
                        int nz, int* nblocks_out) {
    constexpr int BM = 64;
    GemmParams q = p;
    const dim3 grid = gemm_grid(q, BM, nz);
    if (nblocks_out) *nblocks_out = (int)(grid.x * grid.y);
    if (pro == PRO_RHS && epi == EPI_STORE)
        EPC_LAUNCH(ctx, name, (k_dct_gemm<PRO_RHS, EPI_STORE, 4>), grid, NT, 0, q);
    else if (pro == PRO_RHS && epi == EPI_DIVIDE)
        EPC_LAUNCH(ctx, name, (k_dct_gemm<PRO_RHS, EPI_DIVIDE, 4>), grid, NT, 0, q);
    else if (pro == PRO_PLAIN && epi == EPI_DIVIDE)
        EPC_LAUNCH(ctx, name, (k_dct_gemm<PRO_PLAIN, EPI_DIVIDE, 4>), grid, NT, 0, q);
    else if (pro == PRO_PLAIN && epi == EPI_DUAL)
        EPC_LAUNCH(ctx, name, (k_dct_gemm<PRO_PLAIN, EPI_DUAL, 4>), grid, NT, 0, q);
    else
        EPC_LAUNCH(ctx, name, (k_dct_gemm<PRO_PLAIN, EPI_STORE, 4>), grid, NT, 0, q);
}

// 96-row tiles for the plain-store transforms when M is a multiple of 96
// (the inverse axis-3 transform at m3 = 96: 0.130 -> 0.111 ms at C3), else
// 64: the divide and dual epilogues are slower with 96 and 128-row tiles are
// slower for the axis-2 transforms (measured). EPC_GEMM_RM=4 forces 64-row
// tiles (dev aid).
void launch_dct_gemm(epc_context* ctx, const char* name, const GemmParams& p, int pro, int epi,
                     int nz, int* nblocks_out) {
    static const bool force64 = getenv("EPC_GEMM_RM") && atoi(getenv("EPC_GEMM_RM")) == 4;
    if (!force64 && epi == EPI_DIVIDE && p.M % 64 != 0 && p.M % 48 == 0) {
        // 48-row tiles: no half-empty second tile at m3 = 96, and the divide
        // epilogue's registers stay at the 64-row kernel's occupancy
        constexpr int BM = 48;
        GemmParams q = p;
        const dim3 grid = gemm_grid(q, BM, nz);
        if (nblocks_out) *nblocks_out = (int)(grid.x * grid.y);
        if (pro == PRO_RHS)
            EPC_LAUNCH(ctx, name, (k_dct_gemm<PRO_RHS, EPI_DIVIDE, 3>), grid, NT, 0, q);
        else
            EPC_LAUNCH(ctx, name, (k_dct_gemm<PRO_PLAIN, EPI_DIVIDE, 3>), grid, NT, 0, q);
    } else if (!force64 && pro == PRO_PLAIN && epi == EPI_STORE && p.M % 96 == 0) {
        constexpr int BM = 96;
        GemmParams q = p;
        const dim3 grid = gemm_grid(q, BM, nz);
        if (nblocks_out) *nblocks_out = (int)(grid.x * grid.y);
        EPC_LAUNCH(ctx, name, (k_dct_gemm<PRO_PLAIN, EPI_STORE, 6>), grid, NT, 0, q);
    } else {
        launch_dct_gemm_64(ctx, name, p, pro, epi, nz, nblocks_out);
    }
}

// g_value parts (admm.cpp:275-285): sum over faces of (D2 z)^2 and (D3 z)^2,
// differences scaled by 1/h exactly as diff_perp (operators.cpp:70-100).
// grid: (blocks, npairs); partials[(pair*gridDim.x + blk)*2 + {0,1}].
__global__ void __launch_bounds__(256) k_zdiff_sums(const double* z, long long nface, int n1,
                                                   int m2, int m3, double ih2, double ih3,
                                                   double* partials) {
    __shared__ double sh[16];
    const int pair = blockIdx.y;
    const double* zp = z + (long long)pair * nface;
    const long long layer = (long long)n1 * m2;
    double s2 = 0.0, s3 = 0.0;
    // block b owns one contiguous range of faces; each thread walks it with a
    // stride of the block size, ZU faces' loads in flight, tracking its
    // position in the layer incrementally (no index division per face):
    // (D2 z) exists unless the face is in the layer's last column, (D3 z)
    // unless it is in the last layer
    constexpr int ZU = 4;
    const long long per = (nface + gridDim.x - 1) / gridDim.x;
    const long long f0 = (long long)blockIdx.x * per;
    const long long f1 = f0 + per < nface ? f0 + per : nface;
    long long f = f0 + threadIdx.x;
    long long k = f / layer, off = f - k * layer;  // once per thread
    const long long step = blockDim.x;
    const long long jlim = layer - n1, klim = m3 - 1;
    for (; f < f1; f += ZU * step) {
        double zf[ZU], zj[ZU], zk[ZU];
        bool hj[ZU], hk[ZU], in[ZU];
        long long o = off, kk = k;
#pragma unroll
        for (int u = 0; u < ZU; ++u) {
            const long long g = f + u * step;
            in[u] = g < f1;
            hj[u] = in[u] && o < jlim;
            hk[u] = in[u] && kk < klim;
            zf[u] = in[u] ? zp[g] : 0.0;
            zj[u] = hj[u] ? zp[g + n1] : 0.0;
            zk[u] = hk[u] ? zp[g + layer] : 0.0;
            o += step;
            while (o >= layer) {  // once at most unless a layer is smaller than a block
                o -= layer;
                ++kk;
            }
        }
        off = o;
        k = kk;
#pragma unroll
        for (int u = 0; u < ZU; ++u) {
            if (hj[u]) {
                const double d = (zj[u] - zf[u]) * ih2;
                s2 += d * d;
            }
            if (hk[u]) {
                const double d = (zk[u] - zf[u]) * ih3;
                s3 += d * d;
            }
        }
    }
    const double t2 = block_sum(s2, sh);
    const double t3 = block_sum(s3, sh + 8);
    if (threadIdx.x == 0) {
        partials[((long long)pair * gridDim.x + blockIdx.x) * 2 + 0] = t2;
        partials[((long long)pair * gridDim.x + blockIdx.x) * 2 + 1] = t3;
    }
}

// out[pair*nsum + s] = sum over blk of in[(pair*nblk + blk)*stride + s]; one
// CTA per pair, fixed order (strided per-thread scan + fixed tree).
__global__ void __launch_bounds__(256) k_reduce_partials(const double* in, int nblk, int stride,
                                                        int nsum, double* out) {
    __shared__ double sh[8];
    const int pair = blockIdx.x;
    for (int s = 0; s < nsum; ++s) {
        double v = 0.0;
        for (int b = threadIdx.x; b < nblk; b += blockDim.x)
            v += in[((long long)pair * nblk + b) * stride + s];
        const double t = block_sum(v, sh);
        if (threadIdx.x == 0) out[pair * nsum + s] = t;
        __syncthreads();
    }
}

// Per-pair reduction of the b-step's per-column outputs. out_d[pair*4]:
// {kkt max, sum r^2, sum (D1 b)^2, 0}; out_i[pair*6]: {first failing column or
// -1, its error code, sqp total, qp total, max active, 0}.
__global__ void __launch_bounds__(1024) k_reduce_columns(const int* col_err, const int* col_sqp,
                                                       const int* col_qp, const int* col_maxact,
                                                       const double* col_kkt, const double* col_fr,
                                                       const double* col_fd, long long ncol,
                                                       const int* active, double* out_d,
                                                       long long* out_i) {
    __shared__ double sh[32];
    __shared__ long long shi[32][4];
    const int pair = blockIdx.x;
    if (active && !active[pair]) return;
    const long long base = (long long)pair * ncol;
    double kk = 0.0, fr = 0.0, fd = 0.0;
    long long first = 0x7fffffffffffffffLL, sqp = 0, qp = 0, mact = 0;
    for (long long c = threadIdx.x; c < ncol; c += blockDim.x) {
        const long long g = base + c;
        if (col_err[g] != 0 && c < first) first = c;
        sqp += col_sqp[g];
        qp += col_qp[g];
        mact = max(mact, (long long)col_maxact[g]);
        kk = dmax_ref(kk, col_kkt[g]);
        fr += col_fr[g];
        fd += col_fd[g];
    }
    const double tfr = block_sum(fr, sh);
    __syncthreads();
    const double tfd = block_sum(fd, sh);
    __syncthreads();
    // max / min / integer sums (exact in any order)
    double km = warp_max(kk);
    for (int o = 16; o > 0; o >>= 1) {
        first = min(first, __shfl_xor_sync(FULL_MASK, first, o));
        sqp += __shfl_xor_sync(FULL_MASK, sqp, o);
        qp += __shfl_xor_sync(FULL_MASK, qp, o);
        mact = max(mact, __shfl_xor_sync(FULL_MASK, mact, o));
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sh[w] = km;
        shi[w][0] = first;
        shi[w][1] = sqp;
        shi[w][2] = qp;
        shi[w][3] = mact;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int nw = blockDim.x >> 5;
        double K = 0.0;
        long long F = 0x7fffffffffffffffLL, S = 0, Q = 0, M = 0;
        for (int i = 0; i < nw; ++i) {
            K = dmax_ref(K, sh[i]);
            F = min(F, shi[i][0]);
            S += shi[i][1];
            Q += shi[i][2];
            M = max(M, shi[i][3]);
        }
        out_d[pair * 4 + 0] = K;
        out_d[pair * 4 + 1] = tfr;
        out_d[pair * 4 + 2] = tfd;
        out_d[pair * 4 + 3] = 0.0;
        const bool bad = F != 0x7fffffffffffffffLL;
        out_i[pair * 6 + 0] = bad ? F : -1;
        out_i[pair * 6 + 1] = bad ? col_err[base + F] : 0;
        out_i[pair * 6 + 2] = S;
        out_i[pair * 6 + 3] = Q;
        out_i[pair * 6 + 4] = M;
        out_i[pair * 6 + 5] = 0;
    }
}

// u *= factor[pair] (scale(st.u.v, rho/next), admm.cpp:549-552)
__global__ void k_scale_pairs(double* u, long long nface, int npairs, const double* factor) {
    const long long n = nface * npairs;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double a = factor[i / nface];
        if (a != 1.0) u[i] *= a;
    }
}

__global__ void k_copy_masked(const double* src, double* dst, long long nface, int npairs,
                              const int* mask) {
    const long long n = nface * npairs;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        if (mask[i / nface]) dst[i] = src[i];
}
