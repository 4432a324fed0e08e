// admm_f32.cu — the fp32 variant of the ADMM solve (BASELINE configs[2],
// SURVEY §8(d) "fp32: reported separately against the fp64 oracle with a
// stated tolerance"). Same algorithm as the fp64 path (admm.cpp:301-560),
// fp32 storage and element arithmetic, sums accumulated in fp64. There is no
// bitwise claim here: the QP / SQP thresholds that the reference tunes for
// fp64 (admm.cpp:129-141,192-196,216-229,410-421) are rescaled for fp32
// (F32_* below) and the tolerance against the fp64 oracle is measured and
// stated in tests/test_gpu_admm_f32.py and DESIGN.md.
//
//  * k_bstep_f32: b_update (admm.cpp:301-443), one warp per column, the
//    column's vectors in shared memory (fp32: ~11 columns per SM at
//    n1 = 257 instead of 8), persistent CTAs with an atomic column queue,
//    lane-parallel model / line-search passes, lane-0 factor and sweeps, the
//    Schur rows of the active set in per-warp global scratch.
//  * z-step: the dense DCT products (operators.cpp:347-386) are plain GEMMs
//    (cuBLAS SGEMM, strided-batched along axis 2); rhs, spectral divide and
//    the dual update + residual / Lagrangian sums are fp32 kernels here.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

#include <algorithm>

namespace {

// fp32 counterparts of the reference's fp64 thresholds
constexpr float F32_INFEAS = 1e-5f;    // admm.cpp:129  (1e-9)
constexpr float F32_WARM = 1e-6f;      // admm.cpp:135  (1e-10)
constexpr float F32_PZERO = 1e-6f;     // admm.cpp:192  (1e-11 * xs)
constexpr float F32_LAMTOL = 1e-5f;    // admm.cpp:196  (1e-9)
constexpr float F32_DPTOL = 1e-7f;     // admm.cpp:215  (1e-14)
constexpr float F32_ACT = 1e-6f;       // admm.cpp:224  (1e-12)
constexpr float F32_STEP = 1e-7f;      // admm.cpp:410  (1e-14 * xs)

enum { F_X, F_TG, F_GRAD, F_GD, F_GO, F_CQ, F_QX, F_W, F_P, F_FD, F_FL, F_LAM, F_R, F_JL, F_JH,
       F_IP, F_IM, F_COUNT };

struct ColF {
    float* base;
    int ns;
    signed char* sign;
    short* act;
    __device__ float* a(int k) const { return base + k * ns; }
};

__device__ __forceinline__ float wmaxf(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(FULL_MASK, v, o));
    return v;
}
__device__ __forceinline__ float wminf(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(FULL_MASK, v, o));
    return v;
}

// AxisInterpolant::value / slope (image.cpp:24-46) in fp32, evaluated at
// u = (x - o)/h - 0.5 with x = cell_center(c) +- a. In fp32 the absolute
// position x_c + a (x_c up to m h) would keep only ~m h 2^-24 of the small
// displacement a, so the position is carried as u = c + t, t = +-a/h, split
// into the integer cell i and the fraction w; the reference's edge cases are
// the same tests written on (i, w).
#ifndef EPC_F32_BRANCHY
#define EPC_F32_BRANCHY 0
#endif
#if EPC_F32_BRANCHY
__device__ __forceinline__ float ipv_l(const float* s, int m, int c, float t) {
    const float ft = floorf(t);
    const int i = c + (int)ft;
    const float w = t - ft;  // u = i + w, 0 <= w < 1
    if (i < -1 || (i == -1 && w <= 0.5f) || i > m - 1 || (i == m - 1 && w >= 0.5f)) return 0.0f;
    if (i < 0 || (i == 0 && w == 0.0f)) return ((float)(i + 1) + (w - 0.5f)) * 2.0f * s[0];
    if (i >= m - 1) return ((float)(m - 1 - i) + (0.5f - w)) * 2.0f * s[m - 1];
    return (1.0f - w) * s[i] + w * s[i + 1];
}
__device__ __forceinline__ float ips_l(const float* s, int m, float ih, int c, float t) {
    const float ft = floorf(t);
    int i = c + (int)ft;
    const float w = t - ft;
    if (i < -1 || (i == -1 && w <= 0.5f) || i > m - 1 || (i == m - 1 && w > 0.5f)) return 0.0f;
    if (i < 0 || (i == 0 && w == 0.0f)) return 2.0f * s[0] * ih;
    if (i > m - 1 || (i == m - 1 && w > 0.0f)) return -2.0f * s[m - 1] * ih;
    if (w == 0.0f) i -= 1;  // fi == u: the left interval
    if (i < 0) return 2.0f * s[0] * ih;
    return (s[i + 1] - s[i]) * ih;
}
#else
// Branch-free forms of the two above (the same cases in the same order, every
// case's value formed and the tests selecting one; loads clamped in range)
__device__ __forceinline__ float ipv_l(const float* s, int m, int c, float t) {
    const float ft = floorf(t);
    const int i = c + (int)ft;
    const float w = t - ft;  // u = i + w, 0 <= w < 1
    const int ic = min(max(i, 0), max(m - 2, 0));
    const float v_in = (1.0f - w) * s[ic] + w * s[ic + 1];
    const float v_lo = ((float)(i + 1) + (w - 0.5f)) * 2.0f * s[0];
    const float v_hi = ((float)(m - 1 - i) + (0.5f - w)) * 2.0f * s[m - 1];
    const bool zero = i < -1 || (i == -1 && w <= 0.5f) || i > m - 1 || (i == m - 1 && w >= 0.5f);
    const bool lo = i < 0 || (i == 0 && w == 0.0f);
    float v = (i >= m - 1) ? v_hi : v_in;
    v = lo ? v_lo : v;
    return zero ? 0.0f : v;
}
__device__ __forceinline__ float ips_l(const float* s, int m, float ih, int c, float t) {
    const float ft = floorf(t);
    const int i0 = c + (int)ft;
    const float w = t - ft;
    const float n_lo = 2.0f * s[0] * ih, n_hi = -2.0f * s[m - 1] * ih;
    const int i = (w == 0.0f) ? i0 - 1 : i0;  // fi == u: the left interval
    const int ic = min(max(i, 0), max(m - 2, 0));
    const float v_in = (s[ic + 1] - s[ic]) * ih;
    const bool zero = i0 < -1 || (i0 == -1 && w <= 0.5f) || i0 > m - 1 || (i0 == m - 1 && w > 0.5f);
    const bool lo = i0 < 0 || (i0 == 0 && w == 0.0f);
    const bool hi = i0 > m - 1 || (i0 == m - 1 && w > 0.0f);
    float v = (i < 0) ? n_lo : v_in;
    v = hi ? n_hi : v;
    v = lo ? n_lo : v;
    return zero ? 0.0f : v;
}
#endif

// residual of cell c at faces (xa, xb) (residual_column, objective.cpp:48-73)
__device__ __forceinline__ float cell_r(const BStepF32Params& P, const float* ip, const float* im,
                                        int c, float xa, float xb) {
    const float a = 0.5f * (xa + xb), d = (xb - xa) * P.inv_h, t = a * P.inv_h;
    return ipv_l(ip, P.m1, c, t) * (1.0f + d) - ipv_l(im, P.m1, c, -t) * (1.0f - d);
}

// LDL^T of the tridiagonal G (lane 0); false on a nonpositive pivot. fp32
// keeps the pivot reciprocals (rd = 1/d): the sweeps are then FMA chains
// and the factor's chain is one reciprocal, not an IEEE division, per step.
__device__ bool factor_f(const float* __restrict__ gd, const float* __restrict__ go,
                         float* __restrict__ rd, float* __restrict__ fl, int n) {
    float prev = gd[0];
    bool ok = prev > 0.0f;
    float r = __frcp_rn(prev);
    rd[0] = r;
#pragma unroll 8
    for (int i = 1; i < n; ++i) {
        const float o = go[i - 1];
        const float l = o * r;
        const float d = __fmaf_rn(-l, o, gd[i]);
        r = __frcp_rn(d);
        fl[i - 1] = l;
        rd[i] = r;
        ok = ok && d > 0.0f;
    }
    fl[n - 1] = 0.0f;
    return ok;
}
// ColFactor::solve (admm.cpp:56-60), one thread, any (generic) memory; the
// unrolled loops let the operand loads run ahead of the FMA chain
__device__ void solve_f(float* __restrict__ x, const float* __restrict__ rd,
                        const float* __restrict__ fl, int n) {
    float prev = x[0];
#pragma unroll 8
    for (int i = 1; i < n; ++i) {
        prev = __fmaf_rn(-fl[i - 1], prev, x[i]);
        x[i] = prev;
    }
    float nxt = x[n - 1] * rd[n - 1];
    x[n - 1] = nxt;
#pragma unroll 8
    for (int i = n - 2; i >= 0; --i) {
        nxt = __fmaf_rn(-fl[i], nxt, x[i] * rd[i]);
        x[i] = nxt;
    }
}

// The same factor and w solve as 32-lane segmented chains with agreement
// rounds (bstep.cu, seg_sweep): each lane runs S steps from a start value
// (exact on lane 0, a guess elsewhere) until every lane's start equals its
// predecessor's end bitwise; the stored values are then the one-thread
// loops' above. Falls back to them after FSEG_ROUNDS rounds.
constexpr int FSEG_ROUNDS = 8;
__device__ __forceinline__ int fseg_len(int steps) { return ((steps + 31) >> 5) | 1; }
__device__ __forceinline__ bool fseg_agree(float end, int cnt, float& st) {
    const int lane = threadIdx.x & 31;
    const float pe = __shfl_up_sync(FULL_MASK, end, 1);
    const bool ok = lane == 0 || cnt == 0 || __float_as_int(pe) == __float_as_int(st);
    if (__all_sync(FULL_MASK, ok)) return true;
    if (lane > 0) st = pe;
    return false;
}

// factor_f in segments: 1 ok, 0 nonpositive pivot, -1 no agreement
template <int S>
__device__ __forceinline__ int factor_f_seg(const float* __restrict__ gd,
                                            const float* __restrict__ go, float* __restrict__ rd,
                                            float* __restrict__ fl, int n) {
    const int lane = threadIdx.x & 31;
    const int i0 = 1 + lane * S;
    const int cnt = max(0, min(S, n - i0));
    if (lane == 0) {
        rd[0] = __frcp_rn(gd[0]);
        fl[n - 1] = 0.0f;
    }
    float st = gd[min(i0, n) - 1];
    for (int round = 0; round < FSEG_ROUNDS; ++round) {
        float prev = st, end = st;
        bool ok = lane != 0 || gd[0] > 0.0f;
        float r = __frcp_rn(prev);
#pragma unroll
        for (int j = 0; j < S; ++j) {
            const int i = min(i0 + j, n - 1);
            const float o = go[i - 1];
            const float l = o * r;
            const float d = __fmaf_rn(-l, o, gd[i]);
            r = __frcp_rn(d);
            if (j < cnt) {
                fl[i - 1] = l;
                rd[i] = r;
                ok = ok && d > 0.0f;
            }
            if (j == cnt - 1) end = d;
            prev = d;
        }
        if (fseg_agree(end, cnt, st)) return __all_sync(FULL_MASK, ok) ? 1 : 0;
    }
    return -1;
}

// solve_f's sweeps, out of place: forward src -> dst, or backward with the
// pivot reciprocals (dst[e] = src[e] rd[e] - fl[e] dst[e+1])
template <int S, bool BWD>
__device__ __forceinline__ bool fseg_sweep(const float* __restrict__ src, float* __restrict__ dst,
                                           const float* __restrict__ rd,
                                           const float* __restrict__ fl, int n) {
    const int lane = threadIdx.x & 31;
    const int r0 = 1 + lane * S;
    const int cnt = max(0, min(S, n - r0));
    if (lane == 0) dst[BWD ? n - 1 : 0] = BWD ? src[n - 1] * rd[n - 1] : src[0];
    const int e0 = BWD ? n - min(r0, n) : min(r0, n) - 1;
    float st = BWD ? src[e0] * rd[e0] : src[e0];
    for (int round = 0; round < FSEG_ROUNDS; ++round) {
        float p = st, end = st;
#pragma unroll
        for (int j = 0; j < S; ++j) {
            const int r = min(r0 + j, n - 1);
            const int e = BWD ? n - 1 - r : r;
            p = BWD ? __fmaf_rn(-fl[e], p, src[e] * rd[e]) : __fmaf_rn(-fl[e - 1], p, src[e]);
            if (j < cnt) dst[e] = p;
            if (j == cnt - 1) end = p;
        }
        if (fseg_agree(end, cnt, st)) return true;
    }
    return false;
}

// w = G^{-1} w through the scratch t (all lanes)
template <int S>
__device__ __forceinline__ void solve_w_f_seg(float* __restrict__ w, float* __restrict__ t,
                                              const float* __restrict__ rd,
                                              const float* __restrict__ fl, int n) {
    const int lane = threadIdx.x & 31;
    if (!fseg_sweep<S, false>(w, t, rd, fl, n)) {  // w untouched: the one-thread solve
        __syncwarp();
        if (lane == 0) solve_f(w, rd, fl, n);
        __syncwarp();
        return;
    }
    __syncwarp();
    if (fseg_sweep<S, true>(t, w, rd, fl, n)) {
        __syncwarp();
        return;
    }
    __syncwarp();
    if (lane == 0) {  // solve_f's backward loop from the forward result in t
        float nxt = t[n - 1] * rd[n - 1];
        w[n - 1] = nxt;
        for (int i = n - 2; i >= 0; --i) {
            nxt = __fmaf_rn(-fl[i], nxt, t[i] * rd[i]);
            w[i] = nxt;
        }
    }
    __syncwarp();
}

enum { FQ_OK = 0, FQ_PIVOT = 1, FQ_INFEASIBLE = 2, FQ_SCHUR = 3, FQ_CYCLE = 4 };

// qp_active_set (admm.cpp:114-237) in fp32: x (= QX) on entry and exit
__device__ int qp_f32(const BStepF32Params& P, const ColF& s, int n, float* qscr, float* sscr,
                      int* iters, int* max_active) {
    const int lane = threadIdx.x & 31, ncell = n - 1;
    const float ih = P.inv_h;
    float *gd = s.a(F_GD), *go = s.a(F_GO), *cq = s.a(F_CQ), *x = s.a(F_QX), *w = s.a(F_W);
    float *p = s.a(F_P), *fd = s.a(F_FD), *fl = s.a(F_FL), *lam = s.a(F_LAM);
    int bad = 0;
    {
        const int S = fseg_len(n - 1);
        const int seg = S <= 9 ? factor_f_seg<9>(gd, go, fd, fl, n)
                                : (S <= 17 ? factor_f_seg<17>(gd, go, fd, fl, n) : -1);
        __syncwarp();
        if (seg >= 0) bad = !seg;
        else if (lane == 0) bad = !factor_f(gd, go, fd, fl, n);
    }
    if (__shfl_sync(FULL_MASK, bad, 0)) return FQ_PIVOT;
    int infeas = 0;
    for (int i = lane; i < ncell; i += 32) {
        s.sign[i] = 0;
        if (fabsf((x[i + 1] - x[i]) * ih) > 1.0f + F32_INFEAS) infeas = 1;
    }
    if (__any_sync(FULL_MASK, infeas)) return FQ_INFEASIBLE;
    __syncwarp();
    // warm start (admm.cpp:133-143): rows in index order via ballots
    int na = 0;
    for (int i0 = 0; i0 < ncell; i0 += 32) {
        const int i = i0 + lane;
        int sg = 0;
        if (i < ncell) {
            const float d = (x[i + 1] - x[i]) * ih;
            sg = d <= -1.0f + F32_WARM ? 1 : (d >= 1.0f - F32_WARM ? -1 : 0);
        }
        const unsigned m = __ballot_sync(FULL_MASK, sg != 0);
        if (sg) {
            s.sign[i] = (signed char)sg;
            s.act[na + __popc(m & ((1u << lane) - 1))] = (short)i;
        }
        na += __popc(m);
    }
    __syncwarp();
    for (int it = 1; it <= P.qp_cap; ++it) {
        *iters = it;
        if (na > *max_active) *max_active = na;
        for (int i = lane; i < n; i += 32) {
            float acc = gd[i] * x[i];
            if (i > 0) acc += go[i - 1] * x[i - 1];
            if (i + 1 < n) acc += go[i] * x[i + 1];
            w[i] = -cq[i] - acc;
        }
        __syncwarp();
        // lane 0: w = G^-1 g; lanes: q rows G^-1 a_r (global scratch)
        // w alone (no active rows): segmented over all lanes, p as scratch
        const int S = fseg_len(n - 1);
        if (na == 0 && S <= 17) {
            if (S <= 9) solve_w_f_seg<9>(w, p, fd, fl, n);
            else solve_w_f_seg<17>(w, p, fd, fl, n);
        } else if (lane == 0) {
            solve_f(w, fd, fl, n);
        }
        for (int r = lane; r < na; r += 32) {
            float* q = qscr + (size_t)r * n;
            const int ir = s.act[r];
            for (int i = 0; i < n; ++i) q[i] = 0.0f;
            const float sr = s.sign[ir] * ih;
            q[ir] = -sr;
            q[ir + 1] = sr;
            solve_f(q, fd, fl, n);
        }
        __syncwarp();
        if (na > 0) {
            for (int e = lane; e < na * na; e += 32) {
                const int r = e / na, c = e - r * na;
                const int ir = s.act[r];
                const float* qs = qscr + (size_t)c * n;
                sscr[e] = s.sign[ir] * ih * (qs[ir + 1] - qs[ir]);
            }
            for (int r = lane; r < na; r += 32) {
                const int ir = s.act[r];
                const float sr = s.sign[ir] * ih;
                const float arx = s.sign[ir] * (x[ir + 1] - x[ir]) * ih;
                lam[r] = -(sr * (w[ir + 1] - w[ir]) - (-1.0f - arx));
            }
            __syncwarp();
            // dense_spd_solve (admm.cpp:73-95), lane 0
            int sbad = 0;
            if (lane == 0) {
                for (int i = 0; i < na && !sbad; ++i) {
                    for (int j = 0; j < i; ++j) {
                        float t = sscr[i * na + j];
                        for (int k = 0; k < j; ++k) t -= sscr[i * na + k] * sscr[j * na + k];
                        sscr[i * na + j] = t / sscr[j * na + j];
                    }
                    float t = sscr[i * na + i];
                    for (int k = 0; k < i; ++k) t -= sscr[i * na + k] * sscr[i * na + k];
                    if (!(t > 0.0f)) sbad = 1;
                    else sscr[i * na + i] = sqrtf(t);
                }
                if (!sbad) {
                    for (int i = 0; i < na; ++i) {
                        float t = lam[i];
                        for (int k = 0; k < i; ++k) t -= sscr[i * na + k] * lam[k];
                        lam[i] = t / sscr[i * na + i];
                    }
                    for (int i = na - 1; i >= 0; --i) {
                        float t = lam[i];
                        for (int k = i + 1; k < na; ++k) t -= sscr[k * na + i] * lam[k];
                        lam[i] = t / sscr[i * na + i];
                    }
                }
            }
            if (__shfl_sync(FULL_MASK, sbad, 0)) return FQ_SCHUR;
            __syncwarp();
        }
        float xs = 0.0f, pn = 0.0f;
        for (int i = lane; i < n; i += 32) {
            float v = w[i];
            for (int r = 0; r < na; ++r) v += lam[r] * qscr[(size_t)r * n + i];
            p[i] = v;
            xs = fmaxf(xs, fabsf(x[i]));
            pn = fmaxf(pn, fabsf(v));
        }
        xs = wmaxf(xs);
        pn = wmaxf(pn);
        __syncwarp();
        // fp32: "p = 0" is relative to |x| only (the reference's floor of 1 in
        // max(1, |x|) would swallow the small steps of the high-rho iterations)
        bool converged = pn <= F32_PZERO * xs;
        if (!converged) {
            // ratio test (admm.cpp:211-219)
            float t = 1.0f;
            for (int i = lane; i < ncell; i += 32) {
                if (s.sign[i] != 0) continue;
                const float d = (x[i + 1] - x[i]) * ih, dp = (p[i + 1] - p[i]) * ih;
                if (dp < -F32_DPTOL) t = fminf(t, (-1.0f - d) / dp);
                else if (dp > F32_DPTOL) t = fminf(t, (1.0f - d) / dp);
            }
            t = fmaxf(wminf(t), 0.0f);
            for (int i = lane; i < n; i += 32) x[i] += t * p[i];
            __syncwarp();
            if (t < 1.0f) {
                for (int i0 = 0; i0 < ncell; i0 += 32) {
                    const int i = i0 + lane;
                    int sg = 0;
                    if (i < ncell && s.sign[i] == 0) {
                        const float d = (x[i + 1] - x[i]) * ih;
                        sg = d <= -1.0f + F32_ACT ? 1 : (d >= 1.0f - F32_ACT ? -1 : 0);
                    }
                    const unsigned m = __ballot_sync(FULL_MASK, sg != 0);
                    if (sg) {
                        s.sign[i] = (signed char)sg;
                        s.act[na + __popc(m & ((1u << lane) - 1))] = (short)i;
                    }
                    na += __popc(m);
                }
                __syncwarp();
                continue;
            }
            // a full step solved the equality-constrained KKT system: the
            // multipliers of this iteration are those of the new point, which
            // is what the reference's confirming iteration (p ~ 0) examines
            converged = true;
        }
        if (converged) {
            float lmax = 0.0f;
            for (int r = lane; r < na; r += 32) lmax = fmaxf(lmax, fabsf(lam[r]));
            lmax = wmaxf(lmax);
            float best = -F32_LAMTOL * (1.0f + lmax);
            int worst = -1;
            for (int r = lane; r < na; r += 32)
                if (lam[r] < best) {
                    best = lam[r];
                    worst = r;
                }
            // warp argmin, ties to the lower row
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float ob = __shfl_xor_sync(FULL_MASK, best, o);
                const int ow = __shfl_xor_sync(FULL_MASK, worst, o);
                if (ow >= 0 && (worst < 0 || ob < best || (ob == best && ow < worst))) {
                    best = ob;
                    worst = ow;
                }
            }
            if (worst < 0) {
                // multipliers by cell for the KKT check (lam indexed by cell in W)
                for (int i = lane; i < ncell; i += 32) w[i] = 0.0f;
                __syncwarp();
                for (int r = lane; r < na; r += 32) w[s.act[r]] = fmaxf(0.0f, lam[r]);
                __syncwarp();
                return FQ_OK;
            }
            if (lane == 0) {
                s.sign[s.act[worst]] = 0;
                for (int r = worst; r + 1 < na; ++r) s.act[r] = s.act[r + 1];
            }
            --na;
            __syncwarp();
            continue;
        }
    }
    return FQ_CYCLE;
}

// verify_qp_kkt (admm.cpp:239-265); multipliers by cell in W
__device__ float kkt_f32(const BStepF32Params& P, const ColF& s, int n) {
    const int lane = threadIdx.x & 31, ncell = n - 1;
    const float ih = P.inv_h;
    const float *gd = s.a(F_GD), *go = s.a(F_GO), *cq = s.a(F_CQ), *x = s.a(F_QX), *lm = s.a(F_W);
    float scale = 1.0f, lmax = 1.0f, ms = 0.0f, viol = 0.0f;
    for (int i = lane; i < n; i += 32) {
        float acc = gd[i] * x[i];
        if (i > 0) acc += go[i - 1] * x[i - 1];
        if (i + 1 < n) acc += go[i] * x[i + 1];
        scale = fmaxf(scale, fmaxf(fabsf(acc), fabsf(cq[i])));
        float sv = acc + cq[i];
        if (i > 0 && s.sign[i - 1] != 0) sv -= s.sign[i - 1] * ih * lm[i - 1];
        if (i < ncell && s.sign[i] != 0) sv += s.sign[i] * ih * lm[i];
        ms = fmaxf(ms, fabsf(sv));
        if (i < ncell) lmax = fmaxf(lmax, fabsf(lm[i]));
    }
    scale = wmaxf(scale);
    lmax = wmaxf(lmax);
    ms = wmaxf(ms);
    for (int i = lane; i < ncell; i += 32) {
        const float d = (x[i + 1] - x[i]) * ih, l = lm[i];
        viol = fmaxf(viol, fabsf(d) - 1.0f);
        viol = fmaxf(viol, -l / lmax);
        const float slack = s.sign[i] != 0 ? s.sign[i] * d + 1.0f : 0.0f;
        viol = fmaxf(viol, fabsf(l * slack) / lmax);
    }
    viol = fmaxf(wmaxf(viol), ms / scale);
    return fmaxf(viol, 0.0f);
}

__device__ __forceinline__ double wsumd(double v) { return warp_sum(v); }

}  // namespace

// b_update (admm.cpp:301-443) in fp32: one warp per column
__global__ void __launch_bounds__(32, 16) k_bstep_f32(BStepF32Params P) {
    extern __shared__ __align__(16) float fsm[];
    const int lane = threadIdx.x & 31;
    const int m1 = P.m1, n1 = P.n1;
    ColF s;
    s.ns = n1 + 1;
    s.base = fsm;
    s.act = reinterpret_cast<short*>(fsm + F_COUNT * s.ns);
    s.sign = reinterpret_cast<signed char*>(s.act + n1);
    float* qscr = P.qscr + (size_t)blockIdx.x * P.qstride;
    float* sscr = P.sscr + (size_t)blockIdx.x * P.sstride;
    const float V = P.V, rw = P.rho * P.V, aw = P.alpha * P.V, h = P.h, ih = P.inv_h;
    const float lapw = aw * ih * ih;
    float *x = s.a(F_X), *tg = s.a(F_TG), *grad = s.a(F_GRAD), *gd = s.a(F_GD), *go = s.a(F_GO);
    float *cq = s.a(F_CQ), *qx = s.a(F_QX), *R = s.a(F_R), *JL = s.a(F_JL), *JH = s.a(F_JH);
    float *ip = s.a(F_IP), *im = s.a(F_IM);
    for (;;) {
        long long col = 0;
        if (lane == 0) col = (long long)atomicAdd(P.counter, 1ull);
        col = __shfl_sync(FULL_MASK, col, 0);
        if (col >= P.ncol) break;
        const float* bc = P.b + col * n1;
        for (int i = lane; i < n1; i += 32) {
            x[i] = bc[i];
            tg[i] = P.z[col * n1 + i] - P.u[col * n1 + i];
        }
        for (int i = lane; i < m1; i += 32) {
            ip[i] = P.ip[col * m1 + i];
            im[i] = P.im[col * m1 + i];
        }
        __syncwarp();
        float col_kkt = 0.0f, s0 = -1.0f;
        int err = 0, nsqp = 0, nqp = 0, maxact = 0, nls = 0;
        for (int sqp = 0; sqp < P.sqp_max; ++sqp) {
            // model at x: r, jlo, jhi per cell; fval pieces
            double sr = 0.0, sd = 0.0, sq = 0.0;
            for (int c = lane; c < m1; c += 32) {
                const float a = 0.5f * (x[c] + x[c + 1]), d = (x[c + 1] - x[c]) * ih, t = a * ih;
                const float vp = ipv_l(ip, m1, c, t), vm = ipv_l(im, m1, c, -t);
                const float gp = ips_l(ip, m1, ih, c, t), gm = ips_l(im, m1, ih, c, -t);
                const float r = vp * (1.0f + d) - vm * (1.0f - d);
                const float wa = 0.5f * (gp * (1.0f + d) + gm * (1.0f - d)), wd = (vp + vm) * ih;
                R[c] = r;
                JL[c] = wa - wd;
                JH[c] = wa + wd;
                sr += (double)r * r;
                sd += (double)d * d;
            }
            __syncwarp();
            for (int i = lane; i < n1; i += 32) {
                const float e = x[i] - tg[i];
                sq += (double)e * e;
                float g = rw * e, dg = rw, og = 0.0f;
                if (i < m1) {
                    g += V * JL[i] * R[i] - aw * ((x[i + 1] - x[i]) * ih) * ih;
                    dg += V * JL[i] * JL[i] + lapw;
                    og = V * JL[i] * JH[i] - lapw;
                }
                if (i > 0) {
                    g += V * JH[i - 1] * R[i - 1] + aw * ((x[i] - x[i - 1]) * ih) * ih;
                    dg += V * JH[i - 1] * JH[i - 1] + lapw;
                }
                grad[i] = g;
                gd[i] = dg;
                go[i] = og;
            }
            sr = wsumd(sr);
            sd = wsumd(sd);
            sq = wsumd(sq);
            const double fval = 0.5 * V * sr + 0.5 * (double)aw * sd + 0.5 * (double)rw * sq;
            __syncwarp();
            for (int i = lane; i < n1; i += 32) {
                float acc = gd[i] * x[i];
                if (i > 0) acc += go[i - 1] * x[i - 1];
                if (i + 1 < n1) acc += go[i] * x[i + 1];
                cq[i] = grad[i] - acc;
                qx[i] = x[i];
            }
            __syncwarp();
            int qit = 0;
            const int q = qp_f32(P, s, n1, qscr, sscr, &qit, &maxact);
            if (q != FQ_OK) {
                err = q;
                break;
            }
            nqp += qit;
            nsqp += 1;
            if (P.check_kkt) col_kkt = fmaxf(col_kkt, kkt_f32(P, s, n1));
            double sn = 0.0, gdir = 0.0;
            float xs = 0.0f;  // fp32: relative to |x| only (see qp_f32)
            for (int i = lane; i < n1; i += 32) {
                const float d = qx[i] - x[i];
                cq[i] = d;  // the search direction for the trials (cq is free after the QP)
                sn += (double)d * d;
                gdir += (double)grad[i] * d;
                xs = fmaxf(xs, fabsf(x[i]));
            }
            __syncwarp();
            sn = sqrt(wsumd(sn));
            gdir = wsumd(gdir);
            xs = wmaxf(xs);
            if (s0 < 0.0f) s0 = (float)sn;
            if (sn <= fmaxf(P.sqp_tol_rel * s0, F32_STEP * xs)) break;
            if (!(gdir < 0.0)) break;
            // backtracking (admm.cpp:414-427)
            float tls = 1.0f;
            int acc = 0;
            for (int ls = 0; ls < 40; ++ls) {
                ++nls;
                double tr = 0.0, td = 0.0, tq = 0.0;
                for (int f = lane; f < n1; f += 32) {
                    const float xf = x[f] + tls * cq[f];
                    const float e = xf - tg[f];
                    tq += (double)e * e;
                    if (f < m1) {
                        const float xb = x[f + 1] + tls * cq[f + 1];
                        const float r = cell_r(P, ip, im, f, xf, xb);
                        const float d = (xb - xf) * ih;
                        tr += (double)r * r;
                        td += (double)d * d;
                    }
                }
                tr = wsumd(tr);
                td = wsumd(td);
                tq = wsumd(tq);
                const double ft = 0.5 * V * tr + 0.5 * (double)aw * td + 0.5 * (double)rw * tq;
                if (ft <= fval + 1e-4 * tls * gdir) {
                    acc = 1;
                    break;
                }
                tls *= 0.5f;
            }
            if (!acc) break;
            for (int i = lane; i < n1; i += 32) x[i] = x[i] + tls * cq[i];
            __syncwarp();
        }
        if (err) {
            if (lane == 0) P.col_err[col] = err;
            continue;
        }
        // clamp_column_diffs (admm.cpp:99-110), lane 0, fp32 nextafter; skipped
        // when it is the identity (every step's own comparisons hold with a
        // zero shift; -0.0 + 0.0 would turn into +0.0)
        int ident = 1;
        for (int i = lane; i + 1 < n1; i += 32) {
            const float xi = x[i], nx = x[i + 1], t = (nx - xi) / h;
            if ((nx == 0.0f && signbit(nx)) || nx < xi - h || xi + h < nx || t > 1.0f || t < -1.0f)
                ident = 0;
        }
        const bool identity = __all_sync(FULL_MASK, ident) != 0;
        if (lane == 0 && !identity) {
            float shift = 0.0f;
            for (int i = 0; i + 1 < n1; ++i) {
                const float nx = x[i + 1] + shift;
                float cl = fminf(fmaxf(nx, x[i] - h), x[i] + h);
                while ((cl - x[i]) / h > 1.0f) cl = nextafterf(cl, x[i]);
                while ((cl - x[i]) / h < -1.0f) cl = nextafterf(cl, x[i]);
                shift += cl - nx;
                x[i + 1] = cl;
            }
        }
        __syncwarp();
        // b out; f(b) pieces for the Lagrangian (admm.cpp:267-273)
        double sr = 0.0, sd = 0.0;
        for (int i = lane; i < n1; i += 32) {
            P.b_out[col * n1 + i] = x[i];
            if (i < m1) {
                const float r = cell_r(P, ip, im, i, x[i], x[i + 1]);
                const float d = (x[i + 1] - x[i]) / h;
                sr += (double)r * r;
                sd += (double)d * d;
            }
        }
        sr = wsumd(sr);
        sd = wsumd(sd);
        if (lane == 0) {
            P.col_err[col] = 0;
            P.col_kkt[col] = col_kkt;
            P.col_sr[col] = sr;
            P.col_sd[col] = sd;
            P.col_work[col] = ((long long)min(nls, 32767) << 48) | ((long long)min(nsqp, 255) << 40) |
                              ((long long)min(nqp, 16777215) << 16) | min(maxact, 65535);
        }
    }
}

size_t bstep_f32_smem_bytes(int n1) {
    return (size_t)F_COUNT * (n1 + 1) * sizeof(float) + (size_t)n1 * (sizeof(short) + 1) + 16;
}

// column reductions -> [kkt max, sum sr, sum sd], [first error column, its code, sqp, qp,
// max_active, line-search trials]
__global__ void k_reduce_f32cols(const float* kkt, const double* sr, const double* sd,
                                 const int* err, const long long* work, long long ncol,
                                 double* out_d, long long* out_i) {
    __shared__ double sh[32];
    __shared__ double smax[32];
    __shared__ long long sfirst[32], ssqp[32], sqp[32], smact[32], sls[32];
    double a = 0.0, b = 0.0, m = 0.0;
    long long first = ncol, nsqp = 0, nqp = 0, mact = 0, nls = 0;
    for (long long c = threadIdx.x; c < ncol; c += blockDim.x) {
        if (err[c] != 0) {
            first = c < first ? c : first;
            continue;
        }
        a += sr[c];
        b += sd[c];
        m = fmax(m, (double)kkt[c]);
        nsqp += (work[c] >> 40) & 0xff;
        nqp += (work[c] >> 16) & 0xffffff;
        nls += work[c] >> 48;
        mact = max(mact, work[c] & 0xffff);
    }
    const double ta = block_sum(a, sh);
    __syncthreads();
    const double tb = block_sum(b, sh);
    m = warp_max(m);
    for (int o = 16; o > 0; o >>= 1) {
        first = min(first, __shfl_xor_sync(FULL_MASK, first, o));
        nsqp += __shfl_xor_sync(FULL_MASK, nsqp, o);
        nqp += __shfl_xor_sync(FULL_MASK, nqp, o);
        nls += __shfl_xor_sync(FULL_MASK, nls, o);
        mact = max(mact, __shfl_xor_sync(FULL_MASK, mact, o));
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        smax[w] = m;
        sfirst[w] = first;
        ssqp[w] = nsqp;
        sqp[w] = nqp;
        sls[w] = nls;
        smact[w] = mact;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int nw = blockDim.x >> 5;
        for (int i = 0; i < nw; ++i) {
            m = fmax(m, smax[i]);
            first = min(first, sfirst[i]);
            mact = max(mact, smact[i]);
        }
        nsqp = nqp = nls = 0;
        for (int i = 0; i < nw; ++i) {
            nsqp += ssqp[i];
            nqp += sqp[i];
            nls += sls[i];
        }
        out_d[0] = m;
        out_d[1] = ta;
        out_d[2] = tb;
        out_i[0] = first < ncol ? first : -1;
        out_i[1] = first < ncol ? err[first] : 0;
        out_i[2] = nsqp;
        out_i[3] = nqp;
        out_i[4] = mact;
        out_i[5] = nls;
    }
}



// dual update + residual / Lagrangian partial sums (admm.cpp:453-476,
// 287-299): u_new = u + b - z; per block {sum (b-z)^2, sum (zo-z)^2,
// sum b^2, sum z^2, sum u_new^2, sum u_new (b - z)} and the g(z) sums
// {sum (D2 z)^2, sum (D3 z)^2}
__global__ void __launch_bounds__(256) k_dual_f32(const float* b, const float* z, const float* zo,
                                                  const float* u, float* un, int n1, int m2, int m3,
                                                  float ih2, float ih3, long long n,
                                                  double* part) {
    __shared__ double sh[8];
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const long long layer = (long long)n1 * m2;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const float zi = z[i], bi = b[i];
        const float df = bi - zi, dz = zo[i] - zi;
        const float uu = u[i] + df;
        un[i] = uu;
        acc[0] += (double)df * df;
        acc[1] += (double)dz * dz;
        acc[2] += (double)bi * bi;
        acc[3] += (double)zi * zi;
        acc[4] += (double)uu * uu;
        acc[5] += (double)uu * df;
        // 32-bit index arithmetic when the volume allows (64-bit division
        // costs ~100 instructions)
        int j;
        long long k;
        if (n <= 0xffffffffLL) {
            const unsigned c = (unsigned)i / (unsigned)n1;
            const unsigned kq = c / (unsigned)m2;
            j = (int)(c - kq * (unsigned)m2);
            k = kq;
        } else {
            const long long c = i / n1;
            j = (int)(c % m2);
            k = c / m2;
        }
        if (j + 1 < m2) {
            const float o = (z[i + n1] - zi) * ih2;
            acc[6] += (double)o * o;
        }
        if (k + 1 < m3) {
            const float o = (z[i + layer] - zi) * ih3;
            acc[7] += (double)o * o;
        }
    }
    for (int q = 0; q < 8; ++q) {
        const double t = block_sum(acc[q], sh);
        if (threadIdx.x == 0) part[(size_t)blockIdx.x * 8 + q] = t;
        __syncthreads();
    }
}

__global__ void k_scale_f32(float* x, float a, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        x[i] *= a;
}

__global__ void k_d2f(const double* a, float* b, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        b[i] = (float)a[i];
}

// launch wrappers (kernels launched from their defining translation unit)
void launch_bstep_f32(epc_context* ctx, int slots, size_t smem, const BStepF32Params& P) {
    cudaFuncSetAttribute(k_bstep_f32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    EPC_LAUNCH(ctx, "admm_bstep_f32", k_bstep_f32, slots, 32, smem, P);
}
int bstep_f32_slots_per_sm(size_t smem) {
    int per = 0;
    cudaFuncSetAttribute(k_bstep_f32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_bstep_f32, 32, smem);
    return per;
}
void launch_reduce_f32cols(epc_context* ctx, const BStepF32Params& P, long long ncol, double* od,
                           long long* oi) {
    EPC_LAUNCH(ctx, "reduce_f32cols", k_reduce_f32cols, 1, 512, 0, P.col_kkt, P.col_sr, P.col_sd,
               P.col_err, P.col_work, ncol, od, oi);
}
void launch_dual_f32(epc_context* ctx, int blocks, const float* b, const float* z, const float* zo,
                     const float* u, float* un, int n1, int m2, int m3, float ih2, float ih3,
                     long long n, double* part) {
    EPC_LAUNCH(ctx, "dual_f32", k_dual_f32, blocks, 256, 0, b, z, zo, u, un, n1, m2, m3, ih2, ih3, n,
               part);
}
void launch_scale_f32(epc_context* ctx, int blocks, float* x, float a, long long n) {
    EPC_LAUNCH(ctx, "scale_f32", k_scale_f32, blocks, 256, 0, x, a, n);
}
void launch_d2f(epc_context* ctx, int blocks, const double* a, float* b, long long n) {
    EPC_LAUNCH(ctx, "d2f", k_d2f, blocks, 256, 0, a, b, n);
}

// ---------------------------------------------------------------------------
// fp32 z-step transforms: the dense DCT-II products of DctCoupledSolver
// (operators.cpp:347-418) as one hand-written FFMA GEMM, out = C * in along
// axis 2 or 3, with the rhs formation rho V (b + u) fused into the operand
// load and the spectral divide into the epilogue (the fp32 variant has no
// bitwise contract: contraction to FMA is on, k ascending).
//
// C is M x K row-major (the DCT matrix or its transpose); the data operand
// element (k, n) sits at k * kstride + (n / cdiv) * cstride + n % cdiv, so
// one kernel serves both axes (axis 2: k = j, n = i + n1 k3; axis 3: k = k3,
// n = i + n1 j). Tile BM = 16 RM rows x 128 columns per 256-thread CTA,
// 16-deep K slabs double-buffered through registers, each thread an RM x 8
// strided microtile (conflict-free shared reads).
// ---------------------------------------------------------------------------
namespace {
constexpr int F32_BN = 128, F32_BK = 16, F32_NT = 256;
}

template <int PRO, int EPI, int RM>
__global__ void __launch_bounds__(F32_NT) k_dct_gemm_f32(DctGemmF32 p) {
    constexpr int BM = 16 * RM;
    __shared__ float As[F32_BK][BM + 4];
    __shared__ float Bs[F32_BK][F32_BN];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int row0 = blockIdx.y * BM;
    const long long col0 = (long long)blockIdx.x * F32_BN;
    // B loads: column ln fixed, rows lk + 2 t
    const int ln = tid & (F32_BN - 1), lk = tid >> 7;
    const long long lcol = col0 + ln;
    const bool lok = lcol < p.N;
    const long long lmap = lok ? (lcol / p.cdiv) * p.cstride + (lcol % p.cdiv) : 0;
    // A loads: (am + 16 t, ak)
    const int am = tid >> 4, ak = tid & 15;
    constexpr int NA = RM, NB = F32_BK / 2;
    // fp32 accumulators: an fp64-accumulated variant measured 3.9e-3 instead
    // of 4.0e-3 at C3 (the fp32 b-step sets the deviation) and 50% slower
    float acc[RM][8];
#pragma unroll
    for (int r = 0; r < RM; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[r][c] = 0.0f;
    float ra[NA], rb[NB];
    auto load = [&](int k0) {
#pragma unroll
        for (int t = 0; t < NA; ++t) {
            const int m = row0 + am + 16 * t, k = k0 + ak;
            ra[t] = (m < p.M && k < p.K) ? __ldg(p.A + (size_t)m * p.K + k) : 0.0f;
        }
#pragma unroll
        for (int t = 0; t < NB; ++t) {
            const int k = k0 + lk + 2 * t;
            float v = 0.0f;
            if (lok && k < p.K) {
                const long long a = (long long)k * p.kstride + lmap;
                v = PRO == PRO_RHS ? p.w * (__ldg(p.in0 + a) + __ldg(p.in1 + a)) : __ldg(p.in0 + a);
            }
            rb[t] = v;
        }
    };
    load(0);
    for (int k0 = 0; k0 < p.K; k0 += F32_BK) {
        __syncthreads();
#pragma unroll
        for (int t = 0; t < NA; ++t) As[ak][am + 16 * t] = ra[t];
#pragma unroll
        for (int t = 0; t < NB; ++t) Bs[lk + 2 * t][ln] = rb[t];
        __syncthreads();
        if (k0 + F32_BK < p.K) load(k0 + F32_BK);
#pragma unroll
        for (int kk = 0; kk < F32_BK; ++kk) {
            float a[RM], b[8];
#pragma unroll
            for (int r = 0; r < RM; ++r) a[r] = As[kk][ty + 16 * r];
#pragma unroll
            for (int c = 0; c < 8; ++c) b[c] = Bs[kk][tx + 16 * c];
#pragma unroll
            for (int r = 0; r < RM; ++r)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[r][c] = fmaf(a[r], b[c], acc[r][c]);
        }
    }
    // index arithmetic per column in 32 bits (64-bit division is ~100
    // instructions); lam23's index f / n1 = row (kstride / n1) + cmap / n1
    // when the transformed axis' stride is a multiple of n1 (always here)
    const bool narrow = p.N <= 0x7fffffffLL && (long long)p.M * p.kstride <= 0x7fffffffLL;
    const bool ksplit = narrow && p.kstride % p.n1 == 0;
    const unsigned kq = ksplit ? (unsigned)(p.kstride / p.n1) : 0u;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const long long col = col0 + tx + 16 * c;
        if (col >= p.N) continue;
        long long cmap;
        unsigned cq = 0;
        if (narrow) {
            const unsigned cu = (unsigned)col, cd = (unsigned)p.cdiv;
            const unsigned qd = cu / cd;
            cmap = (long long)qd * p.cstride + (long long)(cu - qd * cd);
            if (EPI == EPI_DIVIDE && ksplit) cq = (unsigned)cmap / (unsigned)p.n1;
        } else {
            cmap = (col / p.cdiv) * p.cstride + (col % p.cdiv);
        }
#pragma unroll
        for (int r = 0; r < RM; ++r) {
            const int row = row0 + ty + 16 * r;
            if (row >= p.M) continue;
            const long long f = (long long)row * p.kstride + cmap;
            float v = acc[r][c];
            if (EPI == EPI_DIVIDE) {
                const long long li = ksplit ? (long long)((unsigned)row * kq + cq)
                                            : (narrow ? (long long)((unsigned)f / (unsigned)p.n1) : f / p.n1);
                v = v / (p.aV * p.lam23[li] + p.rV);
            }
            p.out[f] = v;
        }
    }
}

void launch_dct_gemm_f32(epc_context* ctx, const char* name, const DctGemmF32& p, int pro, int epi) {
    const bool t96 = p.M % 96 == 0;
    const int bm = t96 ? 96 : 64;
    dim3 grid((unsigned)((p.N + F32_BN - 1) / F32_BN), (unsigned)((p.M + bm - 1) / bm));
#define F32_GEMM(PRO, EPI)                                                                  \
    if (t96) EPC_LAUNCH(ctx, name, (k_dct_gemm_f32<PRO, EPI, 6>), grid, F32_NT, 0, p);      \
    else EPC_LAUNCH(ctx, name, (k_dct_gemm_f32<PRO, EPI, 4>), grid, F32_NT, 0, p);
    if (pro == PRO_RHS && epi == EPI_DIVIDE) {
        F32_GEMM(PRO_RHS, EPI_DIVIDE)
    } else if (pro == PRO_RHS) {
        F32_GEMM(PRO_RHS, EPI_STORE)
    } else if (epi == EPI_DIVIDE) {
        F32_GEMM(PRO_PLAIN, EPI_DIVIDE)
    } else {
        F32_GEMM(PRO_PLAIN, EPI_STORE)
    }
#undef F32_GEMM
}
