// pcg.cu — device-resident PCG loop for GN (pcg, proj/src/gn_pcg.cpp:92-131).
//
// The loop scalars (rz, p.q, alpha, beta, relres) never leave the device:
// each kernel reduces its per-block partials in a fixed order in the last
// block to finish (threadfence + atomic ticket; deterministic), then applies
// the reference's scalar update. The host enqueues iterations in chunks and
// reads the state once per chunk; kernels of iterations after convergence
// (or after a curvature failure) return immediately.
//
// Per iteration: k_pcg_hvp (p = z + beta p; q = H p; p.q; alpha = rz / pq)
// and k_pcg_update_bj / k_pcg_update (d += alpha p; r += (-alpha) q;
// z = M^{-1} r; r.r, r.z; relres, relres_prec, stop test, beta = rz_new /
// rz). Element-wise work is bitwise the reference's. The block-Jacobi sweeps
// run over shared-memory tiles: k_pcg_update_ws (8-column groups: memory
// warps and sweep warps pipelined over two stages) or k_pcg_update_bj
// (one role per block; 16-column groups); k_pcg_update (one warp per
// column, lane-0 sweeps) serves the other preconditioners.
#include "common.cuh"
#include "kernels.h"

namespace {

// Fixed-order sum of n partials by one block; result valid in thread 0.
// Four independent accumulators per thread keep several L2 loads in flight
// (the last block runs alone, so its latency is on the critical path).
__device__ double last_block_sum(const double* part, int n, int stride, int off, double* sh) {
    double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
    const int bd = blockDim.x;
    int b = threadIdx.x;
    for (; b + 3 * bd < n; b += 4 * bd) {
        v0 += __ldcg(part + (size_t)b * stride + off);
        v1 += __ldcg(part + (size_t)(b + bd) * stride + off);
        v2 += __ldcg(part + (size_t)(b + 2 * bd) * stride + off);
        v3 += __ldcg(part + (size_t)(b + 3 * bd) * stride + off);
    }
    for (; b < n; b += bd) v0 += __ldcg(part + (size_t)b * stride + off);
    return block_sum((v0 + v1) + (v2 + v3), sh);
}

// Returns true in every thread of the last block to arrive.
__device__ bool arrive_last(unsigned int* counter) {
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int t = atomicAdd(counter, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    return last;
}

// TridiagFactor::solve_column (operators.cpp:248-255) on lane 0 / all lanes:
// forward sweep, lane-parallel divisions, backward sweep. Restrict-qualified
// so the compiler hoists the independent loads ahead of the chain.
// Forward / backward sweeps with the operands of the next 4 steps loaded
// while the current 4 run (two register banks, no rotation moves): fewer
// issued instructions per step than the generic helpers, which matters
// because these single-lane chains are issue-bound with many warps per SMSP.
__device__ __forceinline__ void fwd4(double* __restrict__ v, const double* __restrict__ l, int n) {
    double prev = v[0];
    int i = 1;
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0, b0 = 0, b1 = 0, b2 = 0, b3 = 0;
    if (i + 4 <= n) {
        a0 = l[0]; a1 = l[1]; a2 = l[2]; a3 = l[3];
        b0 = v[1]; b1 = v[2]; b2 = v[3]; b3 = v[4];
    }
    for (; i + 4 <= n; i += 4) {
        double c0 = 0, c1 = 0, c2 = 0, c3 = 0, e0 = 0, e1 = 0, e2 = 0, e3 = 0;
        if (i + 8 <= n) {
            c0 = l[i + 3]; c1 = l[i + 4]; c2 = l[i + 5]; c3 = l[i + 6];
            e0 = v[i + 4]; e1 = v[i + 5]; e2 = v[i + 6]; e3 = v[i + 7];
        }
        prev = b0 - a0 * prev; v[i] = prev;
        prev = b1 - a1 * prev; v[i + 1] = prev;
        prev = b2 - a2 * prev; v[i + 2] = prev;
        prev = b3 - a3 * prev; v[i + 3] = prev;
        a0 = c0; a1 = c1; a2 = c2; a3 = c3;
        b0 = e0; b1 = e1; b2 = e2; b3 = e3;
    }
    for (; i < n; ++i) {
        prev = v[i] - l[i - 1] * prev;
        v[i] = prev;
    }
}

__device__ __forceinline__ void bwd4(double* __restrict__ v, const double* __restrict__ l, int n) {
    double nxt = v[n - 1];
    int i = n - 2;
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0, b0 = 0, b1 = 0, b2 = 0, b3 = 0;
    if (i - 3 >= 0) {
        a0 = l[i]; a1 = l[i - 1]; a2 = l[i - 2]; a3 = l[i - 3];
        b0 = v[i]; b1 = v[i - 1]; b2 = v[i - 2]; b3 = v[i - 3];
    }
    for (; i - 3 >= 0; i -= 4) {
        double c0 = 0, c1 = 0, c2 = 0, c3 = 0, e0 = 0, e1 = 0, e2 = 0, e3 = 0;
        if (i - 7 >= 0) {
            c0 = l[i - 4]; c1 = l[i - 5]; c2 = l[i - 6]; c3 = l[i - 7];
            e0 = v[i - 4]; e1 = v[i - 5]; e2 = v[i - 6]; e3 = v[i - 7];
        }
        nxt = b0 - a0 * nxt; v[i] = nxt;
        nxt = b1 - a1 * nxt; v[i - 1] = nxt;
        nxt = b2 - a2 * nxt; v[i - 2] = nxt;
        nxt = b3 - a3 * nxt; v[i - 3] = nxt;
        a0 = c0; a1 = c1; a2 = c2; a3 = c3;
        b0 = e0; b1 = e1; b2 = e2; b3 = e3;
    }
    for (; i >= 0; --i) {
        nxt = v[i] - l[i] * nxt;
        v[i] = nxt;
    }
}

__device__ __forceinline__ void ldlt_solve_warp(double* __restrict__ v, const double* __restrict__ l,
                                                const double* __restrict__ d, int n) {
    const int lane = threadIdx.x & 31;
    if (lane == 0) fwd4(v, l, n);
    __syncwarp();
    for (int i = lane; i < n; i += 32) v[i] = v[i] / d[i];
    __syncwarp();
    if (lane == 0) bwd4(v, l, n);
    __syncwarp();
}

// The scalar end of an iteration (gn_pcg.cpp:105-108 for phase 0, :115-129):
// rz / prec0 at the start; relres, relres_prec, the stop test and beta.
__device__ void pcg_finish(PcgState* S, int phase, double srr, double srz) {
    if (phase == 0) {
        S->rz = srz;
        S->prec0 = sqrt((srz < 0.0) ? 0.0 : srz);  // sqrt(std::max(rz, 0.0))
    } else {
        S->iters += 1;
        S->relres = sqrt(srr) / S->gnorm;
        S->relres_prec = S->prec0 > 0.0 ? sqrt((srz < 0.0) ? 0.0 : srz) / S->prec0 : 0.0;
        if (S->relres <= S->eta) {
            S->reached = 1;
            S->done = 1;
        } else {
            S->beta = srz / S->rz;
            S->rz = srz;
            if (S->iters >= S->max_iters) S->done = 1;
        }
    }
    S->cnt = 0;
}

}  // namespace

// flag = (a != b) anywhere (values compared with ==, like std::vector's !=);
// the Wolfe driver's re-evaluation test (gn_pcg.cpp:267-269).
__global__ void k_vec_differs(const double* a, const double* b, long long n, int* flag) {
    int d = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        d |= !(a[i] == b[i]);
    if (__any_sync(FULL_MASK, d) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// lowest column with a failed pivot (col_err[c] != 0), or INT_MAX
__global__ void k_first_error(const int* col_err, long long ncol, int* out) {
    int m = 0x7fffffff;
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < ncol;
         c += (long long)gridDim.x * blockDim.x)
        if (col_err[c]) m = min(m, (int)c);
    m = warp_min_int(m);
    if ((threadIdx.x & 31) == 0 && m != 0x7fffffff) atomicMin(out, m);
}

// r = -g; gnorm = ||g||; zero-gradient short circuit (gn_pcg.cpp:96-103).
__global__ void __launch_bounds__(256) k_pcg_start(const double* g, double* r, double* d,
                                                  long long n, double* partials, PcgState* S) {
    __shared__ double sh[8];
    double s = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double v = g[i];
        r[i] = -v;
        d[i] = 0.0;
        s += v * v;
    }
    const double t = block_sum(s, sh);
    if (threadIdx.x == 0) partials[blockIdx.x] = t;
    if (arrive_last(&S->cnt)) {
        __syncthreads();
        const double gg = last_block_sum(partials, gridDim.x, 1, 0, sh);
        if (threadIdx.x == 0) {
            const double gnorm = sqrt(gg);
            S->gnorm = gnorm;
            S->iters = 0;
            S->err = 0;
            S->reached = 0;
            S->done = gnorm == 0.0 ? 1 : 0;
            if (gnorm == 0.0) S->reached = 1;
            S->cnt = 0;
        }
    }
}

// d += alpha p; r += (-alpha) q (phase 1) then z = M^{-1} r and the partial
// sums r.r, r.z; the last block finishes the iteration (gn_pcg.cpp:115-129).
// phase 0 (start): no axpys; sets rz and prec0 (gn_pcg.cpp:105-108).
// One warp per column; r, fd, fl staged in shared memory for the sweeps.
__global__ void __launch_bounds__(128) k_pcg_update(PcgUpdArgs A, PcgState* S) {
    extern __shared__ __align__(16) double usm[];
    __shared__ double red[2][4];
    __shared__ double sh[8];
    if (S->done) return;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int n1 = A.n1;
    const int wpb = blockDim.x >> 5;
    double* sv = usm + (size_t)wib * 3 * n1;
    double* sd = sv + n1;
    double* sl = sd + n1;
    const double a = S->alpha, ma = -a;
    // distinct buffers: restrict lets the unrolled staging batch its loads
    double* __restrict__ Dv = A.d;
    double* __restrict__ Rv = A.r;
    const double* __restrict__ Pv = A.p;
    const double* __restrict__ Qv = A.q;
    const double* __restrict__ FD = A.fd;
    const double* __restrict__ FL = A.fl;
    const bool upd = A.phase == 1, block = A.kind == EPC_PRECOND_BLOCK_JACOBI;
    double rr = 0.0, rz = 0.0;
    for (long long c = (long long)blockIdx.x * wpb + wib; c < A.ncol; c += (long long)gridDim.x * wpb) {
        const size_t o = (size_t)c * n1;
#pragma unroll 4
        for (int i = lane; i < n1; i += 32) {
            double r = Rv[o + i];
            if (upd) {
                Dv[o + i] += a * Pv[o + i];
                r += ma * Qv[o + i];
                Rv[o + i] = r;
            }
            rr += r * r;
            sv[i] = r;
            if (block) {
                sd[i] = FD[o + i];
                sl[i] = FL[o + i];
            }
        }
        __syncwarp();
        if (A.kind == EPC_PRECOND_BLOCK_JACOBI) {
            ldlt_solve_warp(sv, sl, sd, n1);
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
        double x = 0.0, y = 0.0;
        for (int w = 0; w < wpb; ++w) {
            x += red[0][w];
            y += red[1][w];
        }
        A.partials[(size_t)blockIdx.x * 2 + 0] = x;
        A.partials[(size_t)blockIdx.x * 2 + 1] = y;
    }
    if (arrive_last(&S->cnt)) {
        __syncthreads();
        const double srr = last_block_sum(A.partials, gridDim.x, 2, 0, sh);
        __syncthreads();
        const double srz = last_block_sum(A.partials, gridDim.x, 2, 1, sh);
        if (threadIdx.x == 0) pcg_finish(S, A.phase, srr, srz);
    }
}

// ---- fused p / Hessian apply, face-parallel ---------------------------------
// p = z (first iteration) or z + beta p_old, then q = H p (GnHessian::apply,
// objective.cpp:302-331) and the partial p.q; the last block forms alpha
// (gn_pcg.cpp:110-114). The neighbours' p are recomputed from z and p_old
// with the same operations, so they equal the stored p bit for bit; one
// coalesced pass replaces k_pcg_p + k_pcg_hv (48 B/face instead of 56).
// One face: neighbour indices are clamped so that every load is
// unconditional (a load under a boundary branch cannot be hoisted, which
// serialises the round trips); the boundary terms are then selected.
// COH: z and p_old were written earlier in the same (persistent) kernel by
// other blocks, so they are read with ld.global.cg (L2, no stale L1 line).
template <bool COH>
__device__ __forceinline__ double ld_vec(const double* p) {
    return COH ? __ldcg(p) : __ldg(p);
}

template <bool FIRST, bool COH>
__device__ __forceinline__ void hvp_face(const PcgHvArgs& A, double beta, unsigned f, double& xo,
                                         double& yo) {
    const double* __restrict__ Z = A.z;
    const double* __restrict__ PO = A.p_old;
    const unsigned n1 = A.n1, m1 = A.m1, m2 = A.m2, m3 = A.m3, layer = n1 * m2;
    const unsigned c = f / n1, i = f - c * n1, k = c / m2, j = c - k * m2;
    const bool bim = i > 0, bip = i < m1, bjm = j > 0, bjp = j + 1 < m2;
    const bool bkm = m3 > 1 && k > 0, bkp = m3 > 1 && k + 1 < m3;
    const unsigned fim = bim ? f - 1 : f, fip = bip ? f + 1 : f;
    const unsigned fjm = bjm ? f - n1 : f, fjp = bjp ? f + n1 : f;
    const unsigned fkm = bkm ? f - layer : f, fkp = bkp ? f + layer : f;
    // all loads first (the seven z and p_old values, then diag / off), then
    // p = z + beta p_old at the seven points
    const unsigned idx[7] = {f, fim, fip, fjm, fjp, fkm, fkp};
    double zv[7], pv[7];
#pragma unroll
    for (int t = 0; t < 7; ++t) zv[t] = ld_vec<COH>(Z + idx[t]);
    if (!FIRST) {
#pragma unroll
        for (int t = 0; t < 7; ++t) pv[t] = ld_vec<COH>(PO + idx[t]);
    }
    const double dg = __ldg(A.diag + f), oim = __ldg(A.off + fim), oi = __ldg(A.off + f);
    double xv[7];
#pragma unroll
    for (int t = 0; t < 7; ++t) xv[t] = FIRST ? zv[t] : zv[t] + beta * pv[t];
    const double x = xv[0], xim = xv[1], xip = xv[2], xjm = xv[3], xjp = xv[4], xkm = xv[5],
                 xkp = xv[6];
    double acc = dg * x;
    if (bim) acc += oim * xim;
    if (bip) acc += oi * xip;
    double y = acc;
    if (bjm) y += A.w2 * (x - xjm);
    if (bjp) y += A.w2 * (x - xjp);
    if (bkm) y += A.w3 * (x - xkm);
    if (bkp) y += A.w3 * (x - xkp);
    xo = x;
    yo = y;
}

// The loop kernel's form of one face (its 64-register cap): p at the seven
// points formed as loaded, the stores right after (the PR-1 sequence).
template <bool FIRST, bool COH>
__device__ __forceinline__ void hvp_face_lean(const PcgHvArgs& A, double beta, unsigned f, double& s) {
    const double* __restrict__ Z = A.z;
    const double* __restrict__ PO = A.p_old;
    const unsigned n1 = A.n1, m1 = A.m1, m2 = A.m2, m3 = A.m3, layer = n1 * m2;
    const unsigned c = f / n1, i = f - c * n1, k = c / m2, j = c - k * m2;
    const bool bim = i > 0, bip = i < m1, bjm = j > 0, bjp = j + 1 < m2;
    const bool bkm = m3 > 1 && k > 0, bkp = m3 > 1 && k + 1 < m3;
    const unsigned fim = bim ? f - 1 : f, fip = bip ? f + 1 : f;
    const unsigned fjm = bjm ? f - n1 : f, fjp = bjp ? f + n1 : f;
    const unsigned fkm = bkm ? f - layer : f, fkp = bkp ? f + layer : f;
    auto P = [&](unsigned g) {
        return FIRST ? ld_vec<COH>(Z + g) : ld_vec<COH>(Z + g) + beta * ld_vec<COH>(PO + g);
    };
    const double x = P(f), xim = P(fim), xip = P(fip), xjm = P(fjm), xjp = P(fjp);
    const double xkm = P(fkm), xkp = P(fkp);
    const double dg = __ldg(A.diag + f), oim = __ldg(A.off + fim), oi = __ldg(A.off + f);
    A.p_new[f] = x;
    double acc = dg * x;
    if (bim) acc += oim * xim;
    if (bip) acc += oi * xip;
    double y = acc;
    if (bjm) y += A.w2 * (x - xjm);
    if (bjp) y += A.w2 * (x - xjp);
    if (bkm) y += A.w3 * (x - xkm);
    if (bkp) y += A.w3 * (x - xkp);
    A.q[f] = y;
    s += x * y;
}

// EPC_HVP_UNROLL faces per thread in flight: every face's loads are issued
// before any of their stores (the stores come last, so the compiler need
// not assume they alias the next face's loads); s sums the faces in the
// same order whatever the unroll.
#ifndef EPC_HVP_UNROLL
#define EPC_HVP_UNROLL 2
#endif
#ifndef EPC_HVP_LEAN_LOOP
#define EPC_HVP_LEAN_LOOP 1
#endif
template <bool FIRST, bool COH>
__device__ __forceinline__ double hvp_sweep(const PcgHvArgs& A, double beta) {
    if constexpr (COH && EPC_HVP_LEAN_LOOP) {  // inside the persistent loop kernel
        const unsigned n = A.n1 * A.m2 * A.m3;
        const unsigned stride = gridDim.x * blockDim.x;
        double s = 0.0;
        unsigned f = blockIdx.x * blockDim.x + threadIdx.x;
        for (; f + stride < n; f += 2 * stride) {
            hvp_face_lean<FIRST, COH>(A, beta, f, s);
            hvp_face_lean<FIRST, COH>(A, beta, f + stride, s);
        }
        if (f < n) hvp_face_lean<FIRST, COH>(A, beta, f, s);
        return s;
    }
    constexpr int U = EPC_HVP_UNROLL;
    const unsigned n = A.n1 * A.m2 * A.m3;
    const unsigned stride = gridDim.x * blockDim.x;
    double* __restrict__ PN = A.p_new;
    double* __restrict__ Q = A.q;
    double s = 0.0;
    unsigned f = blockIdx.x * blockDim.x + threadIdx.x;
    for (; f + (U - 1) * stride < n; f += U * stride) {
        double x[U], y[U];
#pragma unroll
        for (int u = 0; u < U; ++u) hvp_face<FIRST, COH>(A, beta, f + u * stride, x[u], y[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            PN[f + u * stride] = x[u];
            Q[f + u * stride] = y[u];
            s += x[u] * y[u];
        }
    }
    for (; f < n; f += stride) {
        double x, y;
        hvp_face<FIRST, COH>(A, beta, f, x, y);
        PN[f] = x;
        Q[f] = y;
        s += x * y;
    }
    return s;
}

#ifndef EPC_HVP_MINB
#define EPC_HVP_MINB 4  // 64 registers, 4 blocks per SM: C3 72 -> 68 us (1, 5, 6, 8 measured)
#endif
__global__ void __launch_bounds__(256, EPC_HVP_MINB) k_pcg_hvp(PcgHvArgs A, PcgState* S) {
    __shared__ double sh[8];
    if (S->done) return;
    const double s = S->iters == 0 ? hvp_sweep<true, false>(A, 0.0) : hvp_sweep<false, false>(A, S->beta);
    const double t = block_sum(s, sh);
    if (threadIdx.x == 0) A.partials[blockIdx.x] = t;
    if (arrive_last(&S->cnt)) {
        __syncthreads();
        const double pq = last_block_sum(A.partials, gridDim.x, 1, 0, sh);
        if (threadIdx.x == 0) {
            if (!(pq > 0.0)) {
                S->err = 1;  // "pcg: nonpositive curvature encountered"
                S->done = 1;
            } else {
                S->alpha = S->rz / pq;
            }
            S->cnt = 0;
        }
    }
}

// ---- block-Jacobi update, one thread per column in the sweeps ---------------
// d += alpha p; r += (-alpha) q; z = (L D L^T)^{-1} r (TridiagFactor::
// solve_column, operators.cpp:248-255); partial r.r and r.z. A block of
// PCG_NT threads owns CPW consecutive columns, i.e. one contiguous span of
// CPW * n1 faces, held whole in shared memory (r, then v, in X; l in Y; rows
// of odd stride RS so the per-thread sweeps are bank-conflict free):
//   1. all threads: coalesced flat pass over the span, element-wise updates
//      of d and r (written back), r and l staged;
//   2. forward sweep v_i = r_i - l_{i-1} v_{i-1}: a warp per column as a
//      segmented chain (sweeps_seg, into a third staged array T), or thread
//      cc < CPW as the plain chain (sweeps_thread; seg = 0);
//   3. all threads: v_i / d_i (d read coalesced from the factor);
//   4. backward sweep w_i = v_i - l_i w_{i+1}, the same way;
//   5. all threads: z written coalesced, partial r.z.
// The sweeps do the operations of ldlt_solve_warp in the same order, so z
// is bitwise the same; every global access is a flat coalesced pass.
constexpr int PCG_NT = 256;

// TridiagFactor::solve_in_place (operators.cpp:248-262) on the staged group:
// forward sweep x[i] -= l[i-1] x[i-1], the divisions by d, backward sweep
// x[i] -= l[i] x[i+1]. Thread-per-column form (the reference's chains as
// written): CPW of the block's threads run the sweeps.
template <class SIDX>
__device__ __forceinline__ void sweeps_thread(const PcgUpdArgs& A, int nc, double* X,
                                              const double* Y, size_t base, const SIDX& sidx,
                                              int ne, int ne2) {
    const int tid = threadIdx.x, n1 = A.n1, RS = A.tile_rs;
    const double* __restrict__ FD = A.fd;
    if (tid < nc) {
        double* x = X + tid * RS;
        const double* y = Y + tid * RS;
        double prev = x[0];
#pragma unroll 4
        for (int i = 1; i < n1; ++i) {
            prev = x[i] - y[i - 1] * prev;
            x[i] = prev;
        }
    }
    __syncthreads();
#pragma unroll 2
    for (int h = tid; h < ne2; h += (int)blockDim.x) {
        const double2 dd = __ldg(reinterpret_cast<const double2*>(FD + base + 2 * (size_t)h));
        const int k0 = sidx(2 * h), k1 = sidx(2 * h + 1);
        X[k0] = X[k0] / dd.x;
        X[k1] = X[k1] / dd.y;
    }
    if ((ne & 1) && tid == 0) {
        const int k = sidx(ne - 1);
        X[k] = X[k] / __ldg(FD + base + ne - 1);
    }
    __syncthreads();
    if (tid < nc) {
        double* x = X + tid * RS;
        const double* y = Y + tid * RS;
        double nxt = x[n1 - 1];
#pragma unroll 4
        for (int i = n1 - 2; i >= 0; --i) {
            nxt = x[i] - y[i] * nxt;
            x[i] = nxt;
        }
    }
    __syncthreads();
}

// Segmented form of the same sweeps, bitwise: one warp per column, each lane
// a segment of S steps started from a guess, repeated until every lane's
// start equals its predecessor's end bit for bit (then, by induction from
// lane 0's exact start, every stored value is the one-thread chain's: same
// operations on the same operands). The block-Jacobi factor has |l| well
// below 1 (the alpha V Laplacian plus the cross-column diagonal dominate),
// so a wrong start is forgotten within a few segments: 3-4 rounds of S
// steps instead of n1 - 1. Out of place (X -> T forward, T -> X backward) so
// a lane's guess is never overwritten under it; after SEG_ROUNDS rounds lane
// 0 runs the one-thread chain instead.
constexpr int PCG_SEG_ROUNDS = 8;
#ifndef EPC_PCG_UMULHI
#define EPC_PCG_UMULHI 1
#endif
template <int S, bool BWD, bool PIPE, int W = 0>
__device__ __forceinline__ bool pcg_seg_sweep(const double* __restrict__ src,
                                              double* __restrict__ dst,
                                              const double* __restrict__ l, int n) {
    const int lane = threadIdx.x & 31;
    const int r0 = 1 + lane * S;
    const int cnt = max(0, min(S, n - r0));
    if (lane == 0) dst[BWD ? n - 1 : 0] = src[BWD ? n - 1 : 0];
    double st = src[BWD ? n - min(r0, n) : min(r0, n) - 1];
    if constexpr (W > 0) {
        // warm-up: the start guess is the chain run over the W elements
        // before the segment (nothing stored), from that element's own
        // value; a wrong start decays like prod |l|, so the first round's
        // guesses are already the chain's bits when W covers that decay
        // (C3: one round instead of four). Only the speed depends on W --
        // the rounds below still verify every start.
        if (cnt > 0) {
            if (BWD) {
                int e = min(n - r0 + W, n - 1);
                double p = src[e];
#pragma unroll 1
                for (--e; e >= n - r0; --e) p = src[e] - l[e] * p;
                st = p;
            } else {
                int e = max(r0 - 1 - W, 0);
                double p = src[e];
#pragma unroll 1
                for (++e; e <= r0 - 1; ++e) p = src[e] - l[e - 1] * p;
                st = p;
            }
        }
    }
    // rolled (the loop kernel runs at a 64-register cap); lanes past the end
    // (cnt < S) only repeat their last valid element
    const int e0 = BWD ? n - 1 - min(r0, n - 1) : min(r0, n - 1);
    for (int round = 0; round < PCG_SEG_ROUNDS; ++round) {
        double p = st;
        int e = e0;
        if constexpr (PIPE) {
            // the next step's operands loaded while this step runs (index
            // clamped into the column), so no shared-memory round trip sits
            // on the chain
            double sv = src[e], lv = l[BWD ? e : e - 1];
#pragma unroll 1
            for (int j = 0; j < cnt; ++j) {
                const int en = BWD ? max(e - 1, 0) : min(e + 1, n - 1);
                const double sn = src[en], ln = l[BWD ? en : en - 1];
                p = sv - lv * p;
                dst[e] = p;
                sv = sn;
                lv = ln;
                e = en;
            }
        } else {
#pragma unroll 1
            for (int j = 0; j < cnt; ++j, e += BWD ? -1 : 1) {
                p = src[e] - l[BWD ? e : e - 1] * p;
                dst[e] = p;
            }
        }
        const double end = cnt > 0 ? p : st;
        const double pe = __shfl_up_sync(FULL_MASK, end, 1);
        const bool ok = lane == 0 || cnt == 0 ||
                        __double_as_longlong(pe) == __double_as_longlong(st);
        if (__all_sync(FULL_MASK, ok)) return true;
        if (lane > 0) st = pe;
    }
    return false;
}

#ifndef EPC_PCG_SEG_WARM
#define EPC_PCG_SEG_WARM 1
#endif
template <int S, int CPW, class SIDX>
__device__ __forceinline__ void sweeps_seg(const PcgUpdArgs& A, int nc, double* X, const double* Y,
                                           size_t base, const SIDX& sidx, int ne, int ne2) {
    const int tid = threadIdx.x, lane = tid & 31, n1 = A.n1, RS = A.tile_rs;
    constexpr int SEG_WARM = EPC_PCG_SEG_WARM ? (S <= 9 ? 3 * S : 2 * S) : 0;  // see pcg_seg_sweep
    double* const T = const_cast<double*>(Y) + CPW * RS;  // third staged array
    const double* __restrict__ FD = A.fd;
    for (int cc = tid >> 5; cc < nc; cc += (int)(blockDim.x >> 5)) {
        const double* x = X + cc * RS;
        double* t = T + cc * RS;
        const double* y = Y + cc * RS;
        if (!pcg_seg_sweep<S, false, false, SEG_WARM>(x, t, y, n1) && lane == 0) {
            double prev = x[0];
            t[0] = prev;
            for (int i = 1; i < n1; ++i) {
                prev = x[i] - y[i - 1] * prev;
                t[i] = prev;
            }
        }
    }
    __syncthreads();
#pragma unroll 2
    for (int h = tid; h < ne2; h += (int)blockDim.x) {
        const double2 dd = __ldg(reinterpret_cast<const double2*>(FD + base + 2 * (size_t)h));
        const int k0 = sidx(2 * h), k1 = sidx(2 * h + 1);
        T[k0] = T[k0] / dd.x;
        T[k1] = T[k1] / dd.y;
    }
    if ((ne & 1) && tid == 0) {
        const int k = sidx(ne - 1);
        T[k] = T[k] / __ldg(FD + base + ne - 1);
    }
    __syncthreads();
    for (int cc = tid >> 5; cc < nc; cc += (int)(blockDim.x >> 5)) {
        double* x = X + cc * RS;
        const double* t = T + cc * RS;
        const double* y = Y + cc * RS;
        if (!pcg_seg_sweep<S, true, false, SEG_WARM>(t, x, y, n1) && lane == 0) {
            double nxt = t[n1 - 1];
            x[n1 - 1] = nxt;
            for (int i = n1 - 2; i >= 0; --i) {
                nxt = t[i] - y[i] * nxt;
                x[i] = nxt;
            }
        }
    }
    __syncthreads();
}

// This block's columns: an even-aligned, balanced share of the ncol columns
// (pairs split evenly over the grid, so the 16-byte passes stay aligned and
// no block does more than 2 ceil(ncol / 2 / grid) columns; equal-sized
// rounds of CPW columns would leave blocks with a whole extra round).
__device__ __forceinline__ void block_columns(long long ncol, long long& c0, long long& c1) {
    const long long pairs = (ncol + 1) / 2, B = gridDim.x, b = blockIdx.x;
    c0 = 2 * (pairs * b / B);
    c1 = 2 * (pairs * (b + 1) / B);
    if (c1 > ncol) c1 = ncol;
}

// 16-byte load; COH: written by other blocks of the same persistent kernel
// (read through L2, not the incoherent L1 path).
template <bool COH>
__device__ __forceinline__ double2 ld_vec2(const double* p) {
    return COH ? __ldcg(reinterpret_cast<const double2*>(p)) : __ldg(reinterpret_cast<const double2*>(p));
}

// One column group (steps 1-5 above) for the block; accumulates r.r, r.z.
// COH: p and q come from other blocks of the same persistent kernel. The
// flat passes move two faces per thread (16-byte accesses): a group starts
// at face c0 n1 with c0 a multiple of CPW (even), and the span nc n1 is even
// unless nc is odd (the last group), whose final face goes scalar.
template <int CPW, bool UPD, bool COH, int SEG>
__device__ __forceinline__ void bj_group(const PcgUpdArgs& A, double a, long long c0, int nc, double* X,
                                         double* Y, double& rr, double& rz) {
    const int tid = threadIdx.x;
    const int n1 = A.n1, RS = A.tile_rs;
    const unsigned un1 = (unsigned)n1;
    const double ma = -a;
    double* __restrict__ Dv = A.d;
    double* __restrict__ Rv = A.r;
    double* __restrict__ Zv = A.z;
    const double* __restrict__ Pv = A.p;
    const double* __restrict__ Qv = A.q;
    const double* __restrict__ FL = A.fl;
    const size_t base = (size_t)c0 * n1;
    const int ne = nc * n1;
    const int ne2 = ne >> 1;
#if EPC_PCG_UMULHI
    // e / n1 as a multiply-high by ceil(2^32 / n1): exact for e < 2^32 / n1
    // (a group spans CPW n1 faces)
    const unsigned mg = 0xffffffffu / un1 + 1u;
    auto sidx = [&](int e) {
        const int cc = (int)__umulhi((unsigned)e, mg);
        return cc * RS + (e - cc * n1);
    };
#else
    auto sidx = [&](int e) {
        const int cc = (int)((unsigned)e / un1);
        return cc * RS + (e - cc * n1);
    };
#endif
    auto stage1 = [&](int e, double r0, double l0) {
        rr += r0 * r0;
        const int k = sidx(e);
        X[k] = r0;
        Y[k] = l0;
    };
    // Per-iteration kernel: two face pairs per thread, all ten 16-byte loads
    // issued before any store (the compiler does not move loads across the d
    // / r stores itself). The loop kernel (64-register cap) keeps the lean form.
    if constexpr (COH) {
#pragma unroll 2
        for (int h = tid; h < ne2; h += (int)blockDim.x) {
            const size_t o = base + 2 * (size_t)h;
            double2 r = *reinterpret_cast<const double2*>(Rv + o);
            const double2 pp = ld_vec2<COH>(Pv + o), qq = ld_vec2<COH>(Qv + o);
            double2 dd = *reinterpret_cast<const double2*>(Dv + o);
            dd.x = dd.x + a * pp.x;
            dd.y = dd.y + a * pp.y;
            r.x += ma * qq.x;
            r.y += ma * qq.y;
            *reinterpret_cast<double2*>(Dv + o) = dd;
            *reinterpret_cast<double2*>(Rv + o) = r;
            const double2 l = __ldg(reinterpret_cast<const double2*>(FL + o));
            stage1(2 * h, r.x, l.x);
            stage1(2 * h + 1, r.y, l.y);
        }
    } else for (int h0 = tid; h0 < ne2; h0 += 2 * (int)blockDim.x) {
        double2 r[2], pp[2], qq[2], dd[2], l[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int h = min(h0 + u * (int)blockDim.x, ne2 - 1);
            const size_t o = base + 2 * (size_t)h;
            r[u] = *reinterpret_cast<const double2*>(Rv + o);
            if (UPD) {
                pp[u] = ld_vec2<COH>(Pv + o);
                qq[u] = ld_vec2<COH>(Qv + o);
                dd[u] = *reinterpret_cast<const double2*>(Dv + o);
            }
            l[u] = __ldg(reinterpret_cast<const double2*>(FL + o));
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int h = h0 + u * (int)blockDim.x;
            if (h >= ne2) break;
            const size_t o = base + 2 * (size_t)h;
            if (UPD) {
                dd[u].x = dd[u].x + a * pp[u].x;
                dd[u].y = dd[u].y + a * pp[u].y;
                r[u].x += ma * qq[u].x;
                r[u].y += ma * qq[u].y;
                *reinterpret_cast<double2*>(Dv + o) = dd[u];
                *reinterpret_cast<double2*>(Rv + o) = r[u];
            }
            stage1(2 * h, r[u].x, l[u].x);
            stage1(2 * h + 1, r[u].y, l[u].y);
        }
    }
    if ((ne & 1) && tid == 0) {
        const size_t o = base + ne - 1;
        double r = Rv[o];
        if (UPD) {
            const double dn = Dv[o] + a * ld_vec<COH>(Pv + o);
            r += ma * ld_vec<COH>(Qv + o);
            Dv[o] = dn;
            Rv[o] = r;
        }
        stage1(ne - 1, r, __ldg(FL + o));
    }
    __syncthreads();
    if constexpr (SEG != 0) sweeps_seg<SEG, CPW>(A, nc, X, Y, base, sidx, ne, ne2);
    else sweeps_thread(A, nc, X, Y, base, sidx, ne, ne2);
    if constexpr (COH) {
#pragma unroll 2
        for (int h = tid; h < ne2; h += (int)blockDim.x) {
            const size_t o = base + 2 * (size_t)h;
            const double2 r = *reinterpret_cast<const double2*>(Rv + o);
            const double2 z = make_double2(X[sidx(2 * h)], X[sidx(2 * h + 1)]);
            *reinterpret_cast<double2*>(Zv + o) = z;
            rz += r.x * z.x;
            rz += r.y * z.y;
        }
    } else for (int h0 = tid; h0 < ne2; h0 += 2 * (int)blockDim.x) {  // loads of both pairs first
        double2 r[2];
#pragma unroll
        for (int u = 0; u < 2; ++u)
            r[u] = *reinterpret_cast<const double2*>(Rv + base + 2 * (size_t)min(h0 + u * (int)blockDim.x, ne2 - 1));
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int h = h0 + u * (int)blockDim.x;
            if (h >= ne2) break;
            const double2 z = make_double2(X[sidx(2 * h)], X[sidx(2 * h + 1)]);
            *reinterpret_cast<double2*>(Zv + base + 2 * (size_t)h) = z;
            rz += r[u].x * z.x;
            rz += r[u].y * z.y;
        }
    }
    if ((ne & 1) && tid == 0) {
        const size_t o = base + ne - 1;
        const double zz = X[sidx(ne - 1)];
        Zv[o] = zz;
        rz += Rv[o] * zz;
    }
    __syncthreads();
}

// threads per block of the per-iteration update (4 columns per 128-thread
// block measured within 2% of 8 per 256 at C3: not kept)
template <int CPW> constexpr int bj_threads() { return PCG_NT; }

template <int CPW, bool UPD, int SEG>
#ifndef EPC_PCG_BJ_MINB
#define EPC_PCG_BJ_MINB 4  // shared memory holds 4 blocks per SM at C3 (n1 = 257): keep 64 registers
#endif
__global__ void __launch_bounds__(bj_threads<CPW>(), EPC_PCG_BJ_MINB) k_pcg_update_bj(PcgUpdArgs A, PcgState* S) {
    extern __shared__ __align__(16) double usm[];
    __shared__ double sh[8];
    if (S->done) return;
    double* const X = usm;
    double* const Y = X + CPW * A.tile_rs;
    const double a = S->alpha;
    double rr = 0.0, rz = 0.0;
    long long cb0, cb1;
    block_columns(A.ncol, cb0, cb1);
    for (long long c0 = cb0; c0 < cb1; c0 += CPW)
        bj_group<CPW, UPD, false, SEG>(A, a, c0, (int)min((long long)CPW, cb1 - c0), X, Y, rr, rz);
    const double srr_b = block_sum(rr, sh);
    __syncthreads();
    const double srz_b = block_sum(rz, sh);
    if (threadIdx.x == 0) {
        A.partials[(size_t)blockIdx.x * 2 + 0] = srr_b;
        A.partials[(size_t)blockIdx.x * 2 + 1] = srz_b;
    }
    if (arrive_last(&S->cnt)) {
        __syncthreads();
        const double srr = last_block_sum(A.partials, gridDim.x, 2, 0, sh);
        __syncthreads();
        const double srz = last_block_sum(A.partials, gridDim.x, 2, 1, sh);
        if (threadIdx.x == 0) pcg_finish(S, A.phase, srr, srz);
    }
}

// ---- block-Jacobi update, warp-specialised and pipelined ---------------------
// The same five steps, with the memory passes and the sweeps of different
// column groups in flight at once. A block of 2 x PCG_NT threads: the first
// PCG_NT (the "memory" warps) run steps 1 and 5, the second PCG_NT (one
// "sweep" warp per column) steps 2-4, over two shared-memory stages. While
// the sweep warps solve group g in one stage, the memory warps finish group
// g-1 (z written, r.z) and stage group g+1 in the other, so HBM is busy
// during the serial chains instead of idling behind a block barrier (the
// single-role kernel's blocks on an SM start together and stay in step).
// Named barriers hand a stage over: FULL (memory -> sweep), SWEPT (sweep ->
// memory). Each column's sweeps are the same operations on the same operands
// as k_pcg_update_bj's, so z is bitwise the same; the r.r / r.z partials
// follow this kernel's own fixed thread mapping.
__device__ __forceinline__ void named_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
enum { WS_FULL = 1, WS_SWEPT = 3, WS_MEM = 5 };  // FULL / SWEPT: + stage (0, 1)

// step 1 for one group by the memory warps (thread t of PCG_NT): d += a p,
// r += (-a) q written back, r and l staged; accumulates r.r
template <bool UPD, class SIDX>
__device__ __forceinline__ void ws_stage(const PcgUpdArgs& A, double a, size_t base, int ne,
                                         double* X, double* Y, const SIDX& sidx, int t, double& rr) {
    const double ma = -a;
    double* __restrict__ Dv = A.d;
    double* __restrict__ Rv = A.r;
    const double* __restrict__ Pv = A.p;
    const double* __restrict__ Qv = A.q;
    const double* __restrict__ FL = A.fl;
    const int ne2 = ne >> 1;
    auto put = [&](int e, double r0, double l0) {
        rr += r0 * r0;
        const int k = sidx(e);
        X[k] = r0;
        Y[k] = l0;
    };
    for (int h0 = t; h0 < ne2; h0 += 2 * PCG_NT) {
        double2 r[2], pp[2], qq[2], dd[2], l[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int h = min(h0 + u * PCG_NT, ne2 - 1);
            const size_t o = base + 2 * (size_t)h;
            r[u] = *reinterpret_cast<const double2*>(Rv + o);
            if (UPD) {
                pp[u] = __ldg(reinterpret_cast<const double2*>(Pv + o));
                qq[u] = __ldg(reinterpret_cast<const double2*>(Qv + o));
                dd[u] = *reinterpret_cast<const double2*>(Dv + o);
            }
            l[u] = __ldg(reinterpret_cast<const double2*>(FL + o));
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int h = h0 + u * PCG_NT;
            if (h >= ne2) break;
            const size_t o = base + 2 * (size_t)h;
            if (UPD) {
                dd[u].x = dd[u].x + a * pp[u].x;
                dd[u].y = dd[u].y + a * pp[u].y;
                r[u].x += ma * qq[u].x;
                r[u].y += ma * qq[u].y;
                *reinterpret_cast<double2*>(Dv + o) = dd[u];
                *reinterpret_cast<double2*>(Rv + o) = r[u];
            }
            put(2 * h, r[u].x, l[u].x);
            put(2 * h + 1, r[u].y, l[u].y);
        }
    }
    if ((ne & 1) && t == 0) {
        const size_t o = base + ne - 1;
        double r = Rv[o];
        if (UPD) {
            const double dn = Dv[o] + a * __ldg(Pv + o);
            r += ma * __ldg(Qv + o);
            Dv[o] = dn;
            Rv[o] = r;
        }
        put(ne - 1, r, __ldg(FL + o));
    }
}

// step 5 for one group by the memory warps: z written, r.z accumulated
template <class SIDX>
__device__ __forceinline__ void ws_final(const PcgUpdArgs& A, size_t base, int ne, const double* X,
                                         const SIDX& sidx, int t, double& rz) {
    double* __restrict__ Zv = A.z;
    const double* __restrict__ Rv = A.r;
    const int ne2 = ne >> 1;
    for (int h0 = t; h0 < ne2; h0 += 2 * PCG_NT) {
        double2 r[2];
#pragma unroll
        for (int u = 0; u < 2; ++u)
            r[u] = *reinterpret_cast<const double2*>(Rv + base + 2 * (size_t)min(h0 + u * PCG_NT, ne2 - 1));
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int h = h0 + u * PCG_NT;
            if (h >= ne2) break;
            const double2 z = make_double2(X[sidx(2 * h)], X[sidx(2 * h + 1)]);
            *reinterpret_cast<double2*>(Zv + base + 2 * (size_t)h) = z;
            rz += r[u].x * z.x;
            rz += r[u].y * z.y;
        }
    }
    if ((ne & 1) && t == 0) {
        const size_t o = base + ne - 1;
        const double zz = X[sidx(ne - 1)];
        Zv[o] = zz;
        rz += Rv[o] * zz;
    }
}

// steps 2-4 for one column by its sweep warp: forward sweep, divisions by
// d, backward sweep (segmented chains, or lane 0's chain when SEG = 0)
#ifndef EPC_PCG_WS_PIPE
#define EPC_PCG_WS_PIPE 1
#endif
#ifndef EPC_PCG_WS_WARM
#define EPC_PCG_WS_WARM 1
#endif
template <int SEG>
__device__ __forceinline__ void ws_sweep_column(double* x, double* t, const double* y,
                                                const double* __restrict__ fd, int n1) {
    const int lane = threadIdx.x & 31;
    constexpr bool WS_PIPE = EPC_PCG_WS_PIPE;
    // warm-up length: about 27 steps cover the start's decay at C3 (|l| ~ 0.17)
    constexpr int WS_WARM = EPC_PCG_WS_WARM ? (SEG <= 9 ? 3 * SEG : 2 * SEG) : 0;
    if constexpr (SEG == 0) {
        ldlt_solve_warp(x, y, fd, n1);
        (void)t;
    } else {
        // the divisors of the lane's forward segment, loaded ahead of the
        // forward chain (their HBM latency hidden behind it)
        const int r0 = 1 + lane * SEG;
        const int cnt = max(0, min(SEG, n1 - r0));
        double dv[SEG];
#pragma unroll
        for (int j = 0; j < SEG; ++j) dv[j] = __ldg(fd + min(r0 + j, n1 - 1));
        const double d0 = __ldg(fd);
        if (!pcg_seg_sweep<SEG, false, WS_PIPE, WS_WARM>(x, t, y, n1) && lane == 0) {
            double prev = x[0];
            t[0] = prev;
            for (int i = 1; i < n1; ++i) {
                prev = x[i] - y[i - 1] * prev;
                t[i] = prev;
            }
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < SEG; ++j)
            if (j < cnt) t[r0 + j] = t[r0 + j] / dv[j];
        if (lane == 0) t[0] = t[0] / d0;
        __syncwarp();
        if (!pcg_seg_sweep<SEG, true, WS_PIPE, WS_WARM>(t, x, y, n1) && lane == 0) {
            double nxt = t[n1 - 1];
            x[n1 - 1] = nxt;
            for (int i = n1 - 2; i >= 0; --i) {
                nxt = t[i] - y[i] * nxt;
                x[i] = nxt;
            }
        }
        __syncwarp();
    }
}

template <int CPW, bool UPD, int SEG>
__global__ void __launch_bounds__(2 * PCG_NT, 2) k_pcg_update_ws(PcgUpdArgs A, PcgState* S) {
    static_assert(CPW * 32 <= PCG_NT, "one sweep warp per column");
    extern __shared__ __align__(16) double usm[];
    __shared__ double sh[2 * PCG_NT / 32];
    if (S->done) return;
    const int n1 = A.n1, RS = A.tile_rs;
    const unsigned un1 = (unsigned)n1;
    const size_t stage_elems = (size_t)3 * CPW * RS;
    const double a = S->alpha;
    long long cb0, cb1;
    block_columns(A.ncol, cb0, cb1);
    const int G = (int)((cb1 - cb0 + CPW - 1) / CPW);
    const unsigned mg = 0xffffffffu / un1 + 1u;  // e / n1 = umulhi(e, mg) for e < 2^32 / n1
    auto sidx = [&](int e) {
        const int cc = (int)__umulhi((unsigned)e, mg);
        return cc * RS + (e - cc * n1);
    };
    constexpr int NB = 2 * PCG_NT;
    double rr = 0.0, rz = 0.0;
    if (threadIdx.x < PCG_NT) {  // memory warps
        const int t = threadIdx.x;
        auto stage = [&](int g) {
            double* X = usm + (g & 1) * stage_elems;
            const long long c0 = cb0 + (long long)g * CPW;
            const int nc = (int)min((long long)CPW, cb1 - c0);
            ws_stage<UPD>(A, a, (size_t)c0 * n1, nc * n1, X, X + CPW * RS, sidx, t, rr);
            named_arrive(WS_FULL + (g & 1), NB);
        };
        for (int g = 0; g < min(G, 2); ++g) stage(g);
        for (int g = 0; g < G; ++g) {
            named_sync(WS_SWEPT + (g & 1), NB);
            const long long c0 = cb0 + (long long)g * CPW;
            const int nc = (int)min((long long)CPW, cb1 - c0);
            ws_final(A, (size_t)c0 * n1, nc * n1, usm + (g & 1) * stage_elems, sidx, t, rz);
            if (g + 2 < G) {
                named_sync(WS_MEM, PCG_NT);  // every z read from the stage before it is refilled
                stage(g + 2);
            }
        }
    } else {  // sweep warps: warp w solves column w of each group
        const int w = (threadIdx.x - PCG_NT) >> 5;
        for (int g = 0; g < G; ++g) {
            named_sync(WS_FULL + (g & 1), NB);
            const long long c0 = cb0 + (long long)g * CPW;
            const int nc = (int)min((long long)CPW, cb1 - c0);
            if (w < nc) {
                double* X = usm + (g & 1) * stage_elems;
                ws_sweep_column<SEG>(X + w * RS, X + 2 * CPW * RS + w * RS, X + CPW * RS + w * RS,
                                     A.fd + (size_t)(c0 + w) * n1, n1);
            }
            named_arrive(WS_SWEPT + (g & 1), NB);
        }
    }
    __syncthreads();
    const double srr_b = block_sum(rr, sh);
    __syncthreads();
    const double srz_b = block_sum(rz, sh);
    if (threadIdx.x == 0) {
        A.partials[(size_t)blockIdx.x * 2 + 0] = srr_b;
        A.partials[(size_t)blockIdx.x * 2 + 1] = srz_b;
    }
    if (arrive_last(&S->cnt)) {
        __syncthreads();
        const double srr = last_block_sum(A.partials, gridDim.x, 2, 0, sh);
        __syncthreads();
        const double srz = last_block_sum(A.partials, gridDim.x, 2, 1, sh);
        if (threadIdx.x == 0) pcg_finish(S, A.phase, srr, srz);
    }
}

// ---- the whole PCG loop in one cooperative launch ---------------------------
// Phase A (k_pcg_hvp's work) and phase B (k_pcg_update_bj's) alternate with
// a grid barrier after each; every block then forms the same fixed-order sum
// of the per-block partials and takes the same scalar decision (alpha; then
// relres, the stop test and beta, gn_pcg.cpp:110-129), so no block waits on
// a "last block". Block 0 publishes the final state. The barrier spin is
// bounded: a block that waits > ~2 s marks S->err = 2 and leaves (no hang).
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ bool grid_barrier(unsigned* bar, unsigned& target) {
    __shared__ int ok;
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        ok = 1;
        const long long t0 = clock64();
        while (ld_acquire_u32(bar) < target) {
            __nanosleep(64);
            if (clock64() - t0 > 4000000000LL) {
                ok = 0;
                break;
            }
        }
        __threadfence();
    }
    __syncthreads();
    return ok != 0;
}

// Fixed-order sum of n partials (stride, offset) by the whole block; the
// same in every block (same order, same tree).
__device__ double block_fixed_sum(const double* part, int n, int stride, int off, double* sh) {
    double v = 0.0;
    for (int b = threadIdx.x; b < n; b += blockDim.x) v += __ldcg(part + (size_t)b * stride + off);
    const double t = block_sum(v, sh);
    __shared__ double out;
    if (threadIdx.x == 0) out = t;
    __syncthreads();
    return out;
}

template <int CPW, int SEG>
#ifndef EPC_PCG_LOOP_MINB
#define EPC_PCG_LOOP_MINB 4  // 64 registers: 4 resident blocks per SM (C2 GN solve 29.4 -> 23.0 ms; 5 spills)
#endif
__global__ void __launch_bounds__(PCG_NT, EPC_PCG_LOOP_MINB) k_pcg_loop(PcgLoopArgs L, PcgState* S) {
    extern __shared__ __align__(16) double usm[];
    __shared__ double sh[8];
    double* const X = usm;
    double* const Y = X + CPW * L.U.tile_rs;
    // state after the start phase (identical in every block)
    int iters = S->iters, done = S->done;
    double rz = S->rz, beta = S->beta, alpha = S->alpha, relres = S->relres,
           relres_prec = S->relres_prec;
    const double gnorm = S->gnorm, prec0 = S->prec0, eta = S->eta;
    const int max_iters = S->max_iters;
    int reached = S->reached, err = 0;
    unsigned target = 0;
    for (int k = 0; !done; ++k) {
        PcgHvArgs H = L.H;
        H.p_new = (k & 1) ? L.pbuf1 : L.pbuf0;
        H.p_old = (k & 1) ? L.pbuf0 : L.pbuf1;
        const double s = iters == 0 ? hvp_sweep<true, true>(H, 0.0) : hvp_sweep<false, true>(H, beta);
        const double sb = block_sum(s, sh);
        if (threadIdx.x == 0) L.part_a[blockIdx.x] = sb;
        if (!grid_barrier(L.bar, target)) {
            err = 2;
            break;
        }
        const double pq = block_fixed_sum(L.part_a, gridDim.x, 1, 0, sh);
        if (!(pq > 0.0)) {
            err = 1;  // "pcg: nonpositive curvature encountered"
            break;
        }
        alpha = rz / pq;
        PcgUpdArgs U = L.U;
        U.p = H.p_new;
        double rr = 0.0, rzp = 0.0;
        // whole groups of CPW columns round-robin (balanced ranges measured no
        // faster here, and cost the 64-register loop a spill)
        for (long long c0 = (long long)blockIdx.x * CPW; c0 < U.ncol; c0 += (long long)gridDim.x * CPW)
            bj_group<CPW, true, true, SEG>(U, alpha, c0, (int)min((long long)CPW, U.ncol - c0), X, Y,
                                           rr, rzp);
        const double srr_b = block_sum(rr, sh);
        __syncthreads();
        const double srz_b = block_sum(rzp, sh);
        if (threadIdx.x == 0) {
            L.part_b[(size_t)blockIdx.x * 2 + 0] = srr_b;
            L.part_b[(size_t)blockIdx.x * 2 + 1] = srz_b;
        }
        if (!grid_barrier(L.bar, target)) {
            err = 2;
            break;
        }
        const double srr = block_fixed_sum(L.part_b, gridDim.x, 2, 0, sh);
        const double srz = block_fixed_sum(L.part_b, gridDim.x, 2, 1, sh);
        iters += 1;
        relres = sqrt(srr) / gnorm;
        relres_prec = prec0 > 0.0 ? sqrt((srz < 0.0) ? 0.0 : srz) / prec0 : 0.0;
        if (relres <= eta) {
            reached = 1;
            done = 1;
        } else {
            beta = srz / rz;
            rz = srz;
            if (iters >= max_iters) done = 1;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        S->iters = iters;
        S->rz = rz;
        S->beta = beta;
        S->alpha = alpha;
        S->relres = relres;
        S->relres_prec = relres_prec;
        S->reached = reached;
        S->err = err;
        S->done = 1;
    }
}

// Cooperative launch of the loop; false when the device cannot hold the grid.
// (CPW, SEG) instantiations: 16 columns per block (n1 <= ~160) keep the
// thread chains; 8 for longer columns, segments 9 or 17
#define PCG_VARIANTS(X) X(16, 0) X(8, 0) X(8, 9) X(8, 17)

static const void* pcg_loop_fn(int cpw, int seg) {
#define PCG_PICK(C, S) if (cpw == C && seg == S) return (const void*)k_pcg_loop<C, S>;
    PCG_VARIANTS(PCG_PICK)
#undef PCG_PICK
    return nullptr;
}

bool pcg_variant_ok(int cpw, int seg) { return pcg_loop_fn(cpw, seg) != nullptr; }

bool launch_pcg_loop(epc_context* ctx, int cpw, int seg, size_t smem, const PcgLoopArgs& L,
                     PcgState* S) {
    const void* fn = pcg_loop_fn(cpw, seg);
    if (!fn) return false;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return false;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, PCG_NT, smem) != cudaSuccess || per_sm < 1)
        return false;
    int coop = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx->device);
    if (!coop) return false;
    const int blocks = ctx->num_sms * per_sm;
    if ((size_t)blocks * 2 + 8 > L.part_cap) return false;
    PcgLoopArgs La = L;
    PcgState* Sa = S;
    void* args[] = {&La, &Sa};
    cudaEvent_t ev0 = nullptr;
    if (ctx->profiling) epc_prof_begin(ctx, "pcg_loop", &ev0);
    const cudaError_t e = cudaLaunchCooperativeKernel(fn, blocks, PCG_NT, args, smem, ctx->stream);
    ctx->launches++;
    if (ctx->profiling) epc_prof_end(ctx, "pcg_loop", ev0);
    return e == cudaSuccess;
}

// the warp-specialised kernel's instantiations (8 columns per group)
#define PCG_WS_VARIANTS(X) X(8, 0) X(8, 9) X(8, 17)

bool pcg_ws_ok(int cpw, int seg) {
#define PCG_WS_HAS(C, SG) if (cpw == C && seg == SG) return true;
    PCG_WS_VARIANTS(PCG_WS_HAS)
#undef PCG_WS_HAS
    return false;
}

void launch_pcg_update_bj(epc_context* ctx, int cpw, int seg, bool ws, int blocks, size_t smem,
                          const PcgUpdArgs& U, PcgState* S) {
    const bool upd = U.phase == 1;
    if (ws) {
#define PCG_LAUNCH_WS(C, SG)                                                                        \
    if (cpw == C && seg == SG) {                                                                   \
        if (upd) EPC_LAUNCH(ctx, "pcg_update", (k_pcg_update_ws<C, true, SG>), blocks, 2 * PCG_NT, smem, U, S); \
        else EPC_LAUNCH(ctx, "pcg_update", (k_pcg_update_ws<C, false, SG>), blocks, 2 * PCG_NT, smem, U, S); \
        return;                                                                                    \
    }
        PCG_WS_VARIANTS(PCG_LAUNCH_WS)
#undef PCG_LAUNCH_WS
    }
#define PCG_LAUNCH_UPD(C, SG)                                                                       \
    if (cpw == C && seg == SG) {                                                                   \
        if (upd) EPC_LAUNCH(ctx, "pcg_update", (k_pcg_update_bj<C, true, SG>), blocks, bj_threads<C>(), smem, U, S); \
        else EPC_LAUNCH(ctx, "pcg_update", (k_pcg_update_bj<C, false, SG>), blocks, bj_threads<C>(), smem, U, S); \
        return;                                                                                    \
    }
    PCG_VARIANTS(PCG_LAUNCH_UPD)
#undef PCG_LAUNCH_UPD
}

// resident blocks per SM of the per-iteration kernels (grids sized to one wave)
int pcg_update_bj_per_sm(int cpw, int seg, bool ws, size_t smem) {
    int per = 0;
    if (ws) {
#define PCG_WS_OCC(C, SG)                                                                   \
    if (cpw == C && seg == SG)                                                              \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pcg_update_ws<C, true, SG>, 2 * PCG_NT, smem);
        PCG_WS_VARIANTS(PCG_WS_OCC)
#undef PCG_WS_OCC
        return per > 0 ? per : 1;
    }
#define PCG_OCC(C, SG)                                                                      \
    if (cpw == C && seg == SG)                                                              \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pcg_update_bj<C, true, SG>, bj_threads<C>(), smem);
    PCG_VARIANTS(PCG_OCC)
#undef PCG_OCC
    return per > 0 ? per : 1;
}
int pcg_hvp_per_sm() {
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pcg_hvp, 256, 0);
    return per > 0 ? per : 1;
}

void set_pcg_update_bj_smem(int cpw, int seg, bool ws, int bytes) {
    const auto attr = cudaFuncAttributeMaxDynamicSharedMemorySize;
    if (ws) {
#define PCG_WS_SET(C, SG)                                                       \
    if (cpw == C && seg == SG) {                                               \
        cudaFuncSetAttribute(k_pcg_update_ws<C, true, SG>, attr, bytes);        \
        cudaFuncSetAttribute(k_pcg_update_ws<C, false, SG>, attr, bytes);       \
    }
        PCG_WS_VARIANTS(PCG_WS_SET)
#undef PCG_WS_SET
        return;
    }
#define PCG_SET_SMEM(C, SG)                                                     \
    if (cpw == C && seg == SG) {                                               \
        cudaFuncSetAttribute(k_pcg_update_bj<C, true, SG>, attr, bytes);        \
        cudaFuncSetAttribute(k_pcg_update_bj<C, false, SG>, attr, bytes);       \
    }
    PCG_VARIANTS(PCG_SET_SMEM)
#undef PCG_SET_SMEM
}
