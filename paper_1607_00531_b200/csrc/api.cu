// api.cu — C ABI (include/epicorr_b200.h) and the host driver of the ADMM
// loop. The loop restates admm_solve (proj/src/admm.cpp:488-560) with every
// per-iteration pass on the device: b-step (bstep.cu), z-step + dual update
// (zstep.cu), then one small device->host read of the per-pair scalars that
// the reference's row / stop test / rho schedule need.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>


#include "common.cuh"
#include "kernels.h"
#include "admm_decide.h"

namespace {

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
struct EpcError {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& m) { throw EpcError{code, m}; }

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(EPC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(x) ck((x), #x)

template <class F>
int guarded(epc_context* ctx, F&& f) {
    try {
        if (ctx) ctx->last_error.clear();
        f();
        return EPC_OK;
    } catch (const EpcError& e) {
        if (ctx) ctx->last_error = e.msg;
        return e.code;
    } catch (const std::exception& e) {
        if (ctx) ctx->last_error = e.what();
        return EPC_ERR_RUNTIME;
    }
}

// ---------------------------------------------------------------------------
// grid
// ---------------------------------------------------------------------------
struct Geo {
    int dim, m1, m2, m3, n1;
    long long ncell, nface, ncol;
    double h1, h2, h3, o1, V;
};

// GridSpec::validate, proj/src/grid.cpp:33-47
Geo make_geo(const epc_grid* g) {
    if (!g) fail(EPC_ERR_INVALID_ARGUMENT, "null grid");
    if (g->dim != 2 && g->dim != 3) fail(EPC_ERR_INVALID_ARGUMENT, "GridSpec: dim must be 2 or 3");
    if (g->m[0] < 2 || g->m[1] < 2) fail(EPC_ERR_INVALID_ARGUMENT, "GridSpec: m1 and m2 must be >= 2");
    if (g->dim == 3 && g->m[2] < 2) fail(EPC_ERR_INVALID_ARGUMENT, "GridSpec: m3 must be >= 2 in 3D");
    if (g->dim == 2 && g->m[2] != 1) fail(EPC_ERR_INVALID_ARGUMENT, "GridSpec: m3 must be 1 in 2D");
    for (int a = 0; a < 3; ++a) {
        if (!(g->h[a] > 0.0) || !std::isfinite(g->h[a]))
            fail(EPC_ERR_INVALID_ARGUMENT, "GridSpec: spacings must be positive");
        if (!std::isfinite(g->origin[a])) fail(EPC_ERR_INVALID_ARGUMENT, "GridSpec: origin must be finite");
    }
    if (g->m[0] + 1 > 32767) fail(EPC_ERR_UNSUPPORTED, "m1 too large for the column kernel");
    Geo o;
    o.dim = g->dim;
    o.m1 = g->m[0];
    o.m2 = g->m[1];
    o.m3 = g->m[2];
    o.n1 = o.m1 + 1;
    o.ncell = (long long)o.m1 * o.m2 * o.m3;
    o.nface = (long long)o.n1 * o.m2 * o.m3;
    o.ncol = (long long)o.m2 * o.m3;
    o.h1 = g->h[0];
    o.h2 = g->h[1];
    o.h3 = g->h[2];
    o.o1 = g->origin[0];
    o.V = g->h[0] * g->h[1] * g->h[2];  // cell_volume, grid.hpp:35
    return o;
}

// ---------------------------------------------------------------------------
// device scratch slots
// ---------------------------------------------------------------------------
enum Slot {
    S_IP, S_IM, S_B0, S_B1, S_Z0, S_Z1, S_U0, S_U1, S_H1, S_H2,
    S_COLI, S_COLD, S_QBUF, S_SBUF, S_PART, S_PART2, S_SCAL, S_PAIR, S_MATS, S_CNT,
    S_TMP0, S_TMP1, S_TMP2, S_TMP3,
    S_GN0, S_GN1, S_GN2, S_GN3, S_GN4, S_GN5, S_GN6, S_GN7, S_GN8, S_GN9,
    S_X0, S_X1, S_X2, S_X3,
    S_SL0, S_SL1,
    S_ML0, S_ML1, S_MLI, S_MLD, S_MLB, S_MLO, S_MLIP, S_MLIM, S_MLFIP, S_MLFIM,
    S_F32_IP, S_F32_IM, S_F32_B0, S_F32_B1, S_F32_Z0, S_F32_Z1, S_F32_U0, S_F32_U1, S_F32_T0,
    S_F32_T1, S_F32_MATS, S_F32_Q, S_F32_S, S_F32_COL, S_F32_SCAL, S_F32_PART,
    S_CTIME, S_SEQ, S_ACTL, S_FUSE, S_LPTC, S_LPTO, S_LPTK,
    S_SN0, S_SN1, S_SN2, S_SN3, S_SN4, S_SN5, S_SN6, S_SN7, S_SN8, S_SN9, S_SNH, S_SNG,
    S_COUNT
};

// Guard mode (EPC_GUARD=1 when the context is created; dev aid standing in
// for compute-sanitizer, which this pool does not run): every scratch slot
// gets a 4 KB zone of 0xA5 bytes on each side, checked by epc_guard_check
// after the work (an out-of-bounds write to any scratch buffer shows there).
constexpr size_t GUARD_BYTES = 4096;

void* slot(epc_context* ctx, int s, size_t bytes) {
    if ((int)ctx->bufs.size() < S_COUNT) ctx->bufs.resize(S_COUNT);
    DevBuf& b = ctx->bufs[s];
    const size_t g = ctx->guard ? GUARD_BYTES : 0;
    if (b.bytes < bytes) {
        if (b.ptr) {
            CK(cudaStreamSynchronize(ctx->stream));
            CK(cudaFree(static_cast<char*>(b.ptr) - g));
            b.ptr = nullptr;
            b.bytes = 0;
        }
        const size_t want = (std::max<size_t>(bytes, 256) + 255) / 256 * 256;
        char* raw = nullptr;
        CK(cudaMalloc(&raw, want + 2 * g));
        if (g) {
            CK(cudaMemsetAsync(raw, 0xA5, g, ctx->stream));
            CK(cudaMemsetAsync(raw + g + want, 0xA5, g, ctx->stream));
        }
        b.ptr = raw + g;
        b.bytes = want;
    }
    return b.ptr;
}

template <class T>
T* slot_t(epc_context* ctx, int s, size_t count) {
    return static_cast<T*>(slot(ctx, s, count * sizeof(T)));
}

void* pinned(epc_context* ctx, size_t bytes) {
    if (ctx->pinned_bytes < bytes) {
        if (ctx->pinned) CK(cudaFreeHost(ctx->pinned));
        ctx->pinned = nullptr;
        CK(cudaMallocHost(&ctx->pinned, std::max<size_t>(bytes, 4096)));
        ctx->pinned_bytes = std::max<size_t>(bytes, 4096);
    }
    return ctx->pinned;
}

void h2d(epc_context* ctx, void* dst, const void* src, size_t bytes) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
}
void* pinned_aux(epc_context* ctx) {
    if (!ctx->pinned_aux) CK(cudaMallocHost(&ctx->pinned_aux, 4096));
    return ctx->pinned_aux;
}

void d2h(epc_context* ctx, void* dst, const void* src, size_t bytes) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
}
void d2d(epc_context* ctx, void* dst, const void* src, size_t bytes) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
}
void sync(epc_context* ctx) { CK(cudaStreamSynchronize(ctx->stream)); }

// Stage an input array into slot `s` (copy, never alias: the reference takes
// its inputs by const& / by value). nullptr -> zeros.
double* stage_in(epc_context* ctx, int s, int mem, const double* src, size_t count) {
    double* d = slot_t<double>(ctx, s, count);
    if (!src) CK(cudaMemsetAsync(d, 0, count * sizeof(double), ctx->stream));
    else if (mem == EPC_MEM_HOST) h2d(ctx, d, src, count * sizeof(double));
    else d2d(ctx, d, src, count * sizeof(double));
    return d;
}

void stage_out(epc_context* ctx, int mem, double* dst, const double* src, size_t count) {
    if (!dst) return;
    if (mem == EPC_MEM_HOST) d2h(ctx, dst, src, count * sizeof(double));
    else d2d(ctx, dst, src, count * sizeof(double));
}

void check_launch() { ck(cudaGetLastError(), "kernel launch"); }

int grid1d(epc_context* ctx, long long n, int block = 256) {
    long long b = (n + block - 1) / block;
    return (int)std::max<long long>(1, std::min<long long>(b, (long long)ctx->num_sms * 16));
}

// ---------------------------------------------------------------------------
// DCT operator matrices, built on the host with the reference's formulas
// (dct2_matrix, operators.cpp:287-295; neumann_eigenvalues, :275-282) so the
// device uses the very same coefficients.
// ---------------------------------------------------------------------------
constexpr double kPi = 3.141592653589793238462643383279502884;

std::vector<double> dct2_matrix(int m) {
    std::vector<double> c((size_t)m * m);
    const double s0 = std::sqrt(1.0 / m), sq = std::sqrt(2.0 / m);
    for (int q = 0; q < m; ++q)
        for (int j = 0; j < m; ++j)
            c[(size_t)q * m + j] = (q == 0 ? s0 : sq) * std::cos(kPi * q * (2.0 * j + 1.0) / (2.0 * m));
    return c;
}

std::vector<double> neumann_eigenvalues(int m, double h) {
    std::vector<double> lam(m);
    for (int q = 0; q < m; ++q) {
        const double s = std::sin(kPi * q / (2.0 * m));
        lam[q] = 4.0 / (h * h) * s * s;
    }
    return lam;
}

struct DctMats {
    const double *c2, *c2t, *c3, *c3t, *lam23;
};

DctMats upload_dct(epc_context* ctx, const Geo& g) {
    const int m2 = g.m2, m3 = g.m3;
    const size_t k3_ = m3 > 1 ? (size_t)m3 : 1, n2_ = (size_t)m2 * m2, n3_ = k3_ * k3_;
    // cached per context: same (m2, m3, h2, h3) and the slot still in place
    if (ctx->dct_base && ctx->dct_base == ctx->bufs[S_MATS].ptr && ctx->dct_key[0] == m2 &&
        ctx->dct_key[1] == m3 && ctx->dct_key[2] == g.h2 && ctx->dct_key[3] == g.h3) {
        double* d = static_cast<double*>(ctx->dct_base);
        return DctMats{d, d + n2_, d + 2 * n2_, d + 2 * n2_ + n3_, d + 2 * n2_ + 2 * n3_};
    }
    std::vector<double> c2 = dct2_matrix(m2), c3 = m3 > 1 ? dct2_matrix(m3) : std::vector<double>(1, 1.0);
    for (double v : c2)
        if (v == 0.0) fail(EPC_ERR_UNSUPPORTED, "DCT matrix has an exact zero coefficient");
    for (double v : c3)
        if (v == 0.0) fail(EPC_ERR_UNSUPPORTED, "DCT matrix has an exact zero coefficient");
    const int k3 = m3 > 1 ? m3 : 1;
    std::vector<double> c2t((size_t)m2 * m2), c3t((size_t)k3 * k3);
    for (int a = 0; a < m2; ++a)
        for (int b = 0; b < m2; ++b) c2t[(size_t)a * m2 + b] = c2[(size_t)b * m2 + a];
    for (int a = 0; a < k3; ++a)
        for (int b = 0; b < k3; ++b) c3t[(size_t)a * k3 + b] = c3[(size_t)b * k3 + a];
    std::vector<double> l2 = neumann_eigenvalues(m2, g.h2);
    std::vector<double> l3 = m3 > 1 ? neumann_eigenvalues(m3, g.h3) : std::vector<double>{0.0};
    std::vector<double> lam23((size_t)m2 * m3);
    for (int k = 0; k < m3; ++k)
        for (int j = 0; j < m2; ++j) lam23[(size_t)k * m2 + j] = l2[j] + l3[k];
    const size_t n2 = (size_t)m2 * m2, n3 = (size_t)k3 * k3, nl = lam23.size();
    std::vector<double> all;
    all.reserve(2 * n2 + 2 * n3 + nl);
    all.insert(all.end(), c2.begin(), c2.end());
    all.insert(all.end(), c2t.begin(), c2t.end());
    all.insert(all.end(), c3.begin(), c3.end());
    all.insert(all.end(), c3t.begin(), c3t.end());
    all.insert(all.end(), lam23.begin(), lam23.end());
    double* d = slot_t<double>(ctx, S_MATS, all.size());
    h2d(ctx, d, all.data(), all.size() * sizeof(double));
    sync(ctx);  // `all` is pageable and goes out of scope
    ctx->dct_base = d;
    ctx->dct_key[0] = m2;
    ctx->dct_key[1] = m3;
    ctx->dct_key[2] = g.h2;
    ctx->dct_key[3] = g.h3;
    return DctMats{d, d + n2, d + 2 * n2, d + 2 * n2 + n3, d + 2 * n2 + 2 * n3};
}

// ---------------------------------------------------------------------------
// z-step: rhs -> DCT2 -> DCT3 -> divide -> iDCT3 -> iDCT2 (+ dual epilogue)
// ---------------------------------------------------------------------------
struct ZArgs {
    const double *b, *u, *z_old;  // rhs = rho V (b + u)
    double *z_new, *u_new;        // u_new: dual update target (EPI_DUAL) or null
    const double* rho;            // device [npairs]
    const int* active;
    double alpha;
    double* partials;  // dual partials [npairs][nblk][6]
    int nblk;          // out: blocks per pair of the dual GEMM
    bool rhs_is_raw;   // true: b holds the rhs itself (dct_solve), u unused
    bool fwd2_done;    // h1 already holds the forward axis-2 transform (fused in the b-step)
};

void run_zstep(epc_context* ctx, const Geo& g, int npairs, const DctMats& M, ZArgs& a) {
    const long long nf = g.nface;
    double* h1 = slot_t<double>(ctx, S_H1, (size_t)nf * npairs);
    double* h2 = slot_t<double>(ctx, S_H2, (size_t)nf * npairs);
    GemmParams p{};
    p.V = g.V;
    p.rho = a.rho;
    p.nface = nf;
    p.lam23 = M.lam23;
    p.alpha = a.alpha;
    p.m2 = g.m2;
    p.n1 = g.n1;
    p.m3 = g.m3;
    p.active = a.active;
    p.zstride = nf;
    // axis-2 operand layout: k = j, col = (k3, i)
    auto axis2 = [&](GemmParams& q) {
        q.M = q.K = g.m2;
        q.N = (long long)g.m3 * g.n1;
        q.kstride = g.n1;
        q.cdiv = g.n1;
        q.cstride = (long long)g.m2 * g.n1;
    };
    auto axis3 = [&](GemmParams& q) {
        q.M = q.K = g.m3;
        q.N = (long long)g.n1 * g.m2;
        q.kstride = (long long)g.n1 * g.m2;
        q.cdiv = q.N;
        q.cstride = 0;
    };
    const int pro = a.rhs_is_raw ? PRO_PLAIN : PRO_RHS;
    if (g.m3 > 1) {
        GemmParams f2 = p;
        axis2(f2);
        f2.A = M.c2;
        f2.in0 = a.b;
        f2.in1 = a.u;
        f2.out = h1;
        if (!a.fwd2_done) launch_dct_gemm(ctx, "dct_fwd2", f2, pro, EPI_STORE, npairs, nullptr);
        GemmParams f3 = p;
        axis3(f3);
        f3.A = M.c3;
        f3.in0 = h1;
        f3.out = h2;
        f3.div_axis = 3;
        launch_dct_gemm(ctx, "dct_fwd3_div", f3, PRO_PLAIN, EPI_DIVIDE, npairs, nullptr);
        GemmParams i3 = p;
        axis3(i3);
        i3.A = M.c3t;
        i3.in0 = h2;
        i3.out = h1;
        launch_dct_gemm(ctx, "dct_inv3", i3, PRO_PLAIN, EPI_STORE, npairs, nullptr);
    } else {
        GemmParams f2 = p;
        axis2(f2);
        f2.A = M.c2;
        f2.in0 = a.b;
        f2.in1 = a.u;
        f2.out = h1;
        f2.div_axis = 2;
        launch_dct_gemm(ctx, "dct_fwd2_div", f2, pro, EPI_DIVIDE, npairs, nullptr);
    }
    GemmParams i2 = p;
    axis2(i2);
    i2.A = M.c2t;
    i2.in0 = h1;
    i2.out = a.z_new;
    if (a.u_new) {
        i2.bvec = a.b;
        i2.u_old = a.u;
        i2.z_old = a.z_old;
        i2.u_new = a.u_new;
        // partial buffer sized on the fly
        const long long nblk = ((i2.N + 63) / 64) * ((i2.M + 63) / 64);
        a.partials = slot_t<double>(ctx, S_PART, (size_t)nblk * npairs * 6);
        i2.partials = a.partials;
        launch_dct_gemm(ctx, "dct_inv2_dual", i2, PRO_PLAIN, EPI_DUAL, npairs, &a.nblk);
    } else {
        launch_dct_gemm(ctx, "dct_inv2", i2, PRO_PLAIN, EPI_STORE, npairs, &a.nblk);
    }
    check_launch();
}

// ---------------------------------------------------------------------------
// b-step launch
// ---------------------------------------------------------------------------
struct BStepRun {
    int* col_i;     // err, sqp, qp, maxact (4 x total)
    double* col_d;  // kkt, fr, fd (3 x total)
    bool fwd2_fused;  // the z-step's forward axis-2 transform ran in the b-step's drain
};

BStepRun run_bstep(epc_context* ctx, const Geo& g, int npairs, const double* ip, const double* im,
                   const double* b, const double* z, const double* u, double* b_out,
                   const double* rho_dev, const int* active_dev, double alpha,
                   const epc_admm_config* cfg, const Fwd2Params* fwd2 = nullptr,
                   unsigned* col_cost = nullptr, const int* order = nullptr, unsigned* crit = nullptr) {
    const long long total = g.ncol * npairs;
    const HDiv hd = make_hdiv(g.h1);
    // EPC_BSTEP_TAIL (dev aid): per-CTA exit times and per-column durations,
    // recorded by the diagnostic instantiation only
    static const bool tail = getenv("EPC_BSTEP_TAIL") != nullptr;
    const bool diag = tail || (ctx->mode & (EPC_MODE_BSTEP_TIMING | EPC_MODE_BSTEP_CHAINED)) != 0;
#ifdef EPC_FORCE_DIAG
    const bool diag_forced = true;
#else
    const bool diag_forced = false;
#endif
    // images in shared memory, or through L1 for long columns: at n1 = 513
    // (C5) that is 5 resident columns per SM instead of 4 and a 4% faster
    // b-step; at n1 = 257 (C3) the staged images are 2% faster (measured).
    // Dev aid EPC_BSTEP_IMG=0/1 forces either; the diagnostic build stages.
    bool img_global = g.n1 >= 400;
    if (const char* e = getenv("EPC_BSTEP_IMG")) img_global = atoi(e) != 0;
    if (diag || diag_forced) img_global = false;
    const size_t smem = bstep_smem_bytes(g.n1, img_global);
    if (smem > ctx->smem_optin) fail(EPC_ERR_UNSUPPORTED, "column too long for shared memory");

    void (*kern)(BStepParams) =
        hd.pow2 ? (diag || diag_forced ? k_admm_bstep_t<HPow2, true, false>
                                       : (img_global ? k_admm_bstep_t<HPow2, false, true>
                                                     : k_admm_bstep_t<HPow2, false, false>))
                : (diag || diag_forced ? k_admm_bstep_t<HGen, true, false>
                                       : (img_global ? k_admm_bstep_t<HGen, false, true>
                                                     : k_admm_bstep_t<HGen, false, false>));
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)ctx->smem_optin));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32, smem));
    if (per_sm < 1) fail(EPC_ERR_UNSUPPORTED, "b-step kernel does not fit on an SM");
    const long long slots = std::min<long long>((long long)ctx->num_sms * per_sm, total);
    const int qcap = g.m1;
    double* qbuf = slot_t<double>(ctx, S_QBUF, (size_t)slots * qrows_stride(qcap, g.n1));
    double* sbuf = slot_t<double>(ctx, S_SBUF, (size_t)slots * qcap * qcap);
    int* col_i = slot_t<int>(ctx, S_COLI, (size_t)total * 4);
    double* col_d = slot_t<double>(ctx, S_COLD, (size_t)total * 3);
    unsigned long long* cnt = slot_t<unsigned long long>(ctx, S_CNT, 1);
    CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), ctx->stream));
    BStepParams P{};
    P.m1 = g.m1;
    P.n1 = g.n1;
    P.ncol = g.ncol;
    P.ncell = g.ncell;
    P.nface = g.nface;
    P.dh = make_hdiv(g.h1);
    P.o1 = g.o1;
    P.V = g.V;
    P.alpha = alpha;
    P.ip = ip;
    P.im = im;
    P.b = b;
    P.z = z;
    P.u = u;
    P.b_out = b_out;
    P.rho = rho_dev;
    P.active = active_dev;
    P.sqp_max_iter = cfg->sqp_max_iter;
    P.sqp_tol_rel = cfg->sqp_tol_rel;
    P.check_kkt = cfg->check_kkt;
    P.qp_cap = 6 * g.n1 + 10;  // admm.cpp:314
    P.col_err = col_i;
    P.col_sqp = col_i + total;
    P.col_qp = col_i + 2 * total;
    P.col_maxact = col_i + 3 * total;
    P.col_kkt = col_d;
    P.col_fr = col_d + total;
    P.col_fd = col_d + 2 * total;
    P.qbuf = qbuf;
    P.sbuf = sbuf;
    P.wbuf = slot_t<double>(ctx, S_X1, (size_t)slots * 2 * g.n1);
    P.qcap = qcap;
    P.counter = cnt;
    P.total_cols = total;
    P.timing = (ctx->mode & EPC_MODE_BSTEP_TIMING) ? slot_t<long long>(ctx, S_GN9, 28) : nullptr;
    P.cert = (ctx->mode & EPC_MODE_BSTEP_CHAINED) ? 0 : 1;
    // the fused forward axis-2 transform needs 8.3 KB of the drained column's
    // shared memory (long enough columns: n1 >= 87) and a separate axis 3
    const bool fuse = fwd2 != nullptr && g.m3 > 1 && smem >= (size_t)(16 * 33 + 16 * 32) * 8;
    if (fuse) {
        P.fwd2 = *fwd2;
        const size_t nl = (size_t)npairs * g.m3;
        unsigned long long* fc = slot_t<unsigned long long>(ctx, S_FUSE, 1 + (nl + 1) / 2);
        CK(cudaMemsetAsync(fc, 0, (1 + (nl + 1) / 2) * 8, ctx->stream));
        P.fwd2.tile_counter = fc;
        P.fwd2.layer_done = reinterpret_cast<unsigned*>(fc + 1);
    }
    P.col_cost = col_cost;
    P.order = order;
    P.crit = order ? crit : nullptr;
    if (tail && total < (1LL << 31)) P.col_ns = slot_t<unsigned>(ctx, S_CTIME, (size_t)total);
    P.cta_span = tail ? slot_t<unsigned long long>(ctx, S_GN8, (size_t)slots * 2) : nullptr;
    static const char* dump = getenv("EPC_BSTEP_DUMP");  // dev aid: per-column records
    if (tail && dump) {
        P.col_sn = slot_t<float>(ctx, S_GN7, (size_t)total * 2);
        CK(cudaMemsetAsync(P.col_sn, 0, (size_t)total * 8, ctx->stream));
    }
    EPC_LAUNCH(ctx, "admm_bstep", kern, (unsigned)slots, 32, smem, P);
    if (tail) {
        std::vector<unsigned long long> t((size_t)slots * 2);
        CK(cudaMemcpyAsync(t.data(), P.cta_span, t.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
        sync(ctx);
        const unsigned long long t0 = *std::min_element(t.begin(), t.begin() + slots);
        std::vector<double> e;
        for (int k = 0; k < (int)slots; ++k) e.push_back((t[slots + k] - t0) * 1e-6);
        std::sort(e.begin(), e.end());
        double idle = 0.0;
        for (double x : e) idle += e.back() - x;
        std::fprintf(stderr, "bstep tail: first exit %.3f ms, median %.3f, p90 %.3f, last %.3f; idle %.1f%%\n",
                     e.front(), e[e.size() / 2], e[e.size() * 9 / 10], e.back(),
                     100.0 * idle / (e.back() * e.size()));
        if (P.col_ns) {
            std::vector<unsigned> ns((size_t)total);
            std::vector<int> ci((size_t)total * 4);
            CK(cudaMemcpyAsync(ns.data(), P.col_ns, total * 4, cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaMemcpyAsync(ci.data(), col_i, total * 16, cudaMemcpyDeviceToHost, ctx->stream));
            sync(ctx);
            std::vector<long long> idx((size_t)total);
            for (long long k = 0; k < total; ++k) idx[k] = k;
            std::partial_sort(idx.begin(), idx.begin() + 5, idx.end(), [&](long long a, long long b) { return ns[a] > ns[b]; });
            double mean = 0;
            for (unsigned v : ns) mean += v;
            mean /= total;
            std::fprintf(stderr, "  column ns mean %.0f; slowest:", mean);
            for (int k = 0; k < 5; ++k) {
                const long long c = idx[k];
                std::fprintf(stderr, " [col %lld %.3f ms sqp %d qp %d act %d]", c, ns[c] * 1e-6, ci[total + c],
                             ci[2 * total + c], ci[3 * total + c]);
            }
            std::fprintf(stderr, "\n");
            static long long launch_no = 0;
            static const int every = getenv("EPC_BSTEP_DUMP_EVERY") ? atoi(getenv("EPC_BSTEP_DUMP_EVERY")) : 1;
            const bool keep = every <= 1 || (launch_no % every) == 0 || (launch_no % every) == every - 1;
            ++launch_no;
            if (dump && P.col_sn && keep) {  // ns, sqp, qp, sn0, sn1 per column, per kept launch
                std::vector<float> sn((size_t)total * 2);
                CK(cudaMemcpyAsync(sn.data(), P.col_sn, total * 8, cudaMemcpyDeviceToHost, ctx->stream));
                sync(ctx);
                if (FILE* f = std::fopen(dump, "ab")) {
                    const long long t = total;
                    std::fwrite(&t, 8, 1, f);
                    std::fwrite(ns.data(), 4, total, f);
                    std::fwrite(ci.data() + total, 4, total, f);
                    std::fwrite(ci.data() + 2 * total, 4, total, f);
                    std::fwrite(sn.data(), 4, 2 * total, f);
                    std::fclose(f);
                }
            }
            static std::vector<unsigned> prev;
            if (prev.size() == ns.size()) {
                long long heavy = 0, was = 0;
                double sx = 0, sy = 0, sxx = 0, syy = 0, sxy = 0;
                for (long long k = 0; k < total; ++k) {
                    const double x = std::log((double)prev[k] + 1), y = std::log((double)ns[k] + 1);
                    sx += x; sy += y; sxx += x * x; syy += y * y; sxy += x * y;
                    if (ns[k] > 1000000u) {
                        ++heavy;
                        if (prev[k] > 500000u) ++was;
                    }
                }
                const double n = (double)total;
                const double r = (sxy - sx * sy / n) / std::sqrt((sxx - sx * sx / n) * (syy - sy * sy / n));
                std::fprintf(stderr, "  predictability: corr(log ns) %.3f; columns > 1 ms: %lld, of which > 0.5 ms before: %lld\n", r, heavy, was);
            }
            prev = ns;
        }
    }
    check_launch();
    return BStepRun{col_i, col_d, fuse};
}

// ---------------------------------------------------------------------------
// validation (objective.cpp:11-15, admm.cpp:28-37)
// ---------------------------------------------------------------------------
void validate_params(const epc_objective_params* p) {
    if (!p) fail(EPC_ERR_INVALID_ARGUMENT, "null params");
    if (!(p->alpha > 0.0)) fail(EPC_ERR_INVALID_ARGUMENT, "ObjectiveParams: alpha must be > 0");
    if (!(p->beta >= 0.0)) fail(EPC_ERR_INVALID_ARGUMENT, "ObjectiveParams: beta must be >= 0");
    if (!(p->gamma >= 0.0)) fail(EPC_ERR_INVALID_ARGUMENT, "ObjectiveParams: gamma must be >= 0");
}

void validate_admm(const epc_admm_config* c) {
    if (!c) fail(EPC_ERR_INVALID_ARGUMENT, "null config");
    if (!(c->rho_min > 0.0) || !(c->rho0 >= c->rho_min))
        fail(EPC_ERR_INVALID_ARGUMENT, "ADMMConfig: need rho0 >= rho_min > 0");
    if (!(c->eps_abs > 0.0) || !(c->eps_rel > 0.0))
        fail(EPC_ERR_INVALID_ARGUMENT, "ADMMConfig: tolerances must be positive");
    if (c->max_iter < 1 || c->sqp_max_iter < 1)
        fail(EPC_ERR_INVALID_ARGUMENT, "ADMMConfig: iteration caps must be >= 1");
    if (!(c->tau_incr > 1.0) || !(c->tau_decr > 1.0) || !(c->mu > 1.0))
        fail(EPC_ERR_INVALID_ARGUMENT, "ADMMConfig: adaptation constants must exceed 1");
}

const char* qp_what(int code) {
    switch (code) {
        case 1: return "column factor: nonpositive pivot";
        case 2: return "qp_active_set: infeasible starting point";
        case 3: return "qp_active_set: singular Schur complement";
        case 4: return "qp_active_set: iteration cap reached (cycling guard)";
        case 9: return "shared-memory canary overwritten (EPC_SMEM_CANARY build)";
    }
    return "unknown column failure";
}

// max |D1 b| > 1 test of admm_solve (admm.cpp:501-502), on the device
__global__ void k_d1_max(const double* b, long long ncell, int m1, int n1, double h1,
                         double* out) {
    __shared__ double sh[8];
    const double ih = 1.0 / h1;
    double m = 0.0;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < ncell;
         e += (long long)gridDim.x * blockDim.x) {
        const long long c = e / m1;
        const int i = (int)(e - c * m1);
        const double d = fabs((b[c * n1 + i + 1] - b[c * n1 + i]) * ih);
        m = (m < d) ? d : m;
    }
    m = warp_max(m);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t = (t < sh[i]) ? sh[i] : t;
        out[blockIdx.x] = t;
    }
}

double d1_norm_inf(epc_context* ctx, const Geo& g, const double* b_dev, int npairs, int pair) {
    const int nb = 64;
    double* part = slot_t<double>(ctx, S_TMP3, nb);
    EPC_LAUNCH(ctx, "d1_max", k_d1_max, nb, 256, 0, b_dev + (size_t)pair * g.nface, g.ncell,
               g.m1, g.n1, g.h1, part);
    check_launch();
    double* h = static_cast<double*>(pinned(ctx, nb * sizeof(double)));
    d2h(ctx, h, part, nb * sizeof(double));
    sync(ctx);
    double m = 0.0;
    for (int i = 0; i < nb; ++i) m = std::max(m, h[i]);
    (void)npairs;
    return m;
}

double rho_schedule(int schedule, double rho, double rho_min, double pr, double du, double ti,
                    double td, double mu) {
    if (schedule == EPC_RHO_FIXED) return rho;
    double next = rho;
    if (pr > mu * du) next = rho * ti;
    else if (du > mu * pr) next = rho / td;
    if (schedule == EPC_RHO_ADAPTIVE_BOUNDED) next = std::max(next, rho_min);
    return next;
}

// rho_schedule's arithmetic (admm.cpp:478-486) for an already-taken decision
// (move: +1 primal > mu dual, -1 dual > mu primal, 0 neither)
__host__ __device__ double rho_apply(int schedule, double rho, double rho_min, int move, double ti,
                                     double td) {
    if (schedule == EPC_RHO_FIXED) return rho;
    double next = rho;
    if (move > 0) next = rho * ti;
    else if (move < 0) next = rho / td;
    if (schedule == EPC_RHO_ADAPTIVE_BOUNDED) next = (next < rho_min) ? rho_min : next;  // std::max
    return next;
}

// ---------------------------------------------------------------------------
// The ADMM loop's per-iteration scalar work on the device (the pipelined
// loop): the row, the certified stop / rho decisions, the rho update and the
// error stop, taken by one thread per pair from the iteration's reduced sums
// with the host code's operations (admm_decide.h, rho_apply), so the host
// never has to answer before the next iteration is enqueued.
// ---------------------------------------------------------------------------
struct IterRec {  // one pair's outcome of one iteration, read back by the host
    double rho_used, kkt, pr, du, eps_pri, eps_dual, lag;
    long long err_col, sqp, qp;
    int err_code, has_row, stop, exact;  // stop: EPC_STOP_* of a pair that stopped here, else -1
};

struct DecideArgs {
    const double* scal_d;     // k_reduce_columns / reduce_dual / reduce_zdiff outputs
    const long long* scal_i;
    double *rho, *fac;        // per pair (S_PAIR)
    int* act;
    int *need, *restore, *was_act;  // per pair (S_ACTL)
    double* seq_io;           // 8 per pair
    IterRec* rec;
    int npairs, schedule, exact_mode, dim;
    long long nface;
    double V, sqrt_n, eps_abs, eps_rel, mu, rho_min, tau_incr, tau_decr, alpha;
};

__device__ void decide_apply(const DecideArgs& D, int q, const epc_decide::Decision& dec) {
    IterRec& r = D.rec[q];
    if (dec.converged) {
        r.stop = EPC_STOP_CONVERGED;
        D.act[q] = 0;
        return;
    }
    const double rho = D.rho[q];
    const double next = rho_apply(D.schedule, rho, D.rho_min, dec.rho_move, D.tau_incr, D.tau_decr);
    if (next != rho) {
        D.fac[q] = rho / next;
        D.rho[q] = next;
    }
}

// phase 0: the row and the certified decision (else need[q] = 1 for the
// sequential sums); phase 1: the decisions on those sums (admm.cpp:542-552)
template <int PHASE>
__global__ void k_admm_decide(DecideArgs D) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= D.npairs) return;
    IterRec& r = D.rec[q];
    if (PHASE == 0) {
        r = IterRec{};
        r.err_col = -1;
        r.stop = -1;  // no stop this iteration (EPC_STOP_CONVERGED is 0)
        D.fac[q] = 1.0;
        D.restore[q] = 0;
        D.need[q] = 0;
        D.was_act[q] = D.act[q];
        if (!D.act[q]) return;
        const double* cd = D.scal_d + (size_t)q * 4;
        const long long* ci = D.scal_i + (size_t)q * 6;
        const double* du = D.scal_d + (size_t)D.npairs * 4 + (size_t)q * 6;
        const double* zd = D.scal_d + (size_t)D.npairs * 10 + (size_t)q * 2;
        if (ci[0] >= 0) {  // a column failed: stop = error, state restored
            r.err_col = ci[0];
            r.err_code = (int)ci[1];
            r.stop = EPC_STOP_ERROR;
            D.act[q] = 0;
            D.restore[q] = 1;
            return;
        }
        r.sqp = ci[2];
        r.qp = ci[3];
        r.has_row = 1;
        const double rho = D.rho[q];
        r.rho_used = rho;
        r.kkt = cd[0];
        const epc_decide::Res tr = epc_decide::residuals(du, rho, D.V, D.sqrt_n, D.eps_abs, D.eps_rel);
        r.pr = tr.pr;
        r.du = tr.du;
        r.eps_pri = tr.eps_pri;
        r.eps_dual = tr.eps_dual;
        const double fval = 0.5 * D.V * cd[1] + 0.5 * D.alpha * D.V * cd[2];
        double gs = zd[0];
        if (D.dim == 3) gs += zd[1];
        const double gval = 0.5 * D.alpha * D.V * gs;
        r.lag = fval + gval + rho * D.V * du[5] + 0.5 * rho * D.V * du[0];
        epc_decide::Decision dec{false, false, 0};
        if (!D.exact_mode)
            dec = epc_decide::certified(du, D.nface, rho, D.V, D.sqrt_n, D.eps_abs, D.eps_rel, D.mu,
                                        D.schedule != EPC_RHO_FIXED);
        if (dec.decided) {
            decide_apply(D, q, dec);
        } else {
            D.need[q] = 1;
            for (int k = 0; k < 8; ++k) D.seq_io[(size_t)q * 8 + k] = 0.0;
        }
    } else {
        if (!D.need[q]) return;
        const double* seq = D.seq_io + (size_t)q * 8;
        const double rho = D.rho[q];
        const epc_decide::Res ex = epc_decide::residuals(seq, rho, D.V, D.sqrt_n, D.eps_abs, D.eps_rel);
        r.pr = ex.pr;  // bitwise the reference's row values
        r.du = ex.du;
        r.eps_pri = ex.eps_pri;
        r.eps_dual = ex.eps_dual;
        r.exact = 1;
        decide_apply(D, q, epc_decide::exact(seq, rho, D.V, D.sqrt_n, D.eps_abs, D.eps_rel, D.mu,
                                             D.schedule != EPC_RHO_FIXED));
    }
}

// The iteration's state tail, per pair (one pass, nothing when no pair
// needs it): pairs inactive at the start of the iteration carry b (the
// b-step skipped them); a pair whose b-step failed keeps the state from
// before the iteration (admm.cpp:553-557); a pair whose rho changed scales
// u by rho / rho' (admm.cpp:549-552). pre = the state before the iteration,
// nxt = the iteration's output (after the host's buffer swap, the current).
__global__ void k_admm_tail(const double* b_pre, double* b_nxt, const double* z_pre, double* z_nxt,
                            const double* u_pre, double* u_nxt, long long nface, int npairs,
                            const int* was_act, const int* restore, const double* fac) {
    __shared__ int any;
    if (threadIdx.x == 0) {
        int a = 0;
        for (int q = 0; q < npairs; ++q) a |= !was_act[q] | restore[q] | (fac[q] != 1.0);
        any = a;
    }
    __syncthreads();
    if (!any) return;
    const long long n = nface * npairs;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int q = (int)(i / nface);
        if (restore[q]) {
            b_nxt[i] = b_pre[i];
            z_nxt[i] = z_pre[i];
            u_nxt[i] = u_pre[i];
            continue;
        }
        if (!was_act[q]) b_nxt[i] = b_pre[i];
        const double a = fac[q];
        if (a != 1.0) u_nxt[i] *= a;
    }
}

// The reference's five sequential sums (admm_decide.h fallback), read back.
void seq_sums(epc_context* ctx, const double* b, const double* z, const double* zo,
              const double* u, long long n, double out[5]) {
    double* io = slot_t<double>(ctx, S_SEQ, 8);
    CK(cudaMemsetAsync(io, 0, 5 * sizeof(double), ctx->stream));
    run_seq_sums(ctx, b, z, zo, u, n, io);
    check_launch();
    double* h = static_cast<double*>(pinned_aux(ctx));
    d2h(ctx, h, io, 5 * sizeof(double));
    sync(ctx);
    for (int i = 0; i < 5; ++i) out[i] = h[i];
}

// ---------------------------------------------------------------------------
// ADMM solve over npairs pairs sharing a grid (admm.cpp:488-560)
// ---------------------------------------------------------------------------
int admm_solve_impl(epc_context* ctx, const epc_grid* gg, int npairs, int mem, const double* iplus,
                    const double* iminus, const double* b_in, const double* z_in,
                    const double* u_in, double* b_out, double* z_out, double* u_out,
                    double* rho_io, const epc_objective_params* p, const epc_admm_config* cfg,
                    int level_tag, epc_admm_row* rows, int max_rows, epc_solve_status* status) {
    return guarded(ctx, [&] {
        for (int q = 0; q < npairs; ++q) {
            status[q].stop = EPC_STOP_MAX_ITERATIONS;
            status[q].nrows = 0;
            status[q].message[0] = 0;
        }
        auto pre_fail = [&](int code, const std::string& m) {
            for (int q = 0; q < npairs; ++q) std::snprintf(status[q].message, sizeof status[q].message, "%s", m.c_str());
            fail(code, m);
        };
        try {
            validate_params(p);
            validate_admm(cfg);
        } catch (const EpcError& e) {
            pre_fail(e.code, e.msg);
        }
        const Geo g = make_geo(gg);
        const size_t nf = (size_t)g.nface * npairs, nc = (size_t)g.ncell * npairs;
        const auto t0 = std::chrono::steady_clock::now();
        // inputs (cells) and state (faces); device pointers may be used in place
        const double* ip;
        const double* im;
        if (mem == EPC_MEM_DEVICE) {
            ip = iplus;
            im = iminus;
        } else {
            double* a = slot_t<double>(ctx, S_IP, nc);
            double* b = slot_t<double>(ctx, S_IM, nc);
            h2d(ctx, a, iplus, nc * sizeof(double));
            h2d(ctx, b, iminus, nc * sizeof(double));
            ip = a;
            im = b;
        }
        double* B[2] = {stage_in(ctx, S_B0, mem, b_in, nf), slot_t<double>(ctx, S_B1, nf)};
        double* Z[2] = {stage_in(ctx, S_Z0, mem, z_in, nf), slot_t<double>(ctx, S_Z1, nf)};
        double* U[2] = {stage_in(ctx, S_U0, mem, u_in, nf), slot_t<double>(ctx, S_U1, nf)};
        for (int q = 0; q < npairs; ++q)
            if (b_in && d1_norm_inf(ctx, g, B[0], npairs, q) > 1.0)
                pre_fail(EPC_ERR_INVALID_ARGUMENT, "admm_solve: infeasible starting field");
        const DctMats M = upload_dct(ctx, g);

        // per-pair device scalars: rho[npairs], active[npairs], factor[npairs]
        char* pr = static_cast<char*>(slot(ctx, S_PAIR, (size_t)npairs * 32));
        double* rho_dev = reinterpret_cast<double*>(pr);
        double* fac_dev = rho_dev + npairs;
        int* act_dev = reinterpret_cast<int*>(fac_dev + npairs);
        std::vector<double> rho(npairs), fac(npairs, 1.0);
        std::vector<int> active(npairs, 1), restore(npairs, 0);
        for (int q = 0; q < npairs; ++q) rho[q] = rho_io[q] > 0.0 ? rho_io[q] : cfg->rho0;
        // host staging block: scalars, then rho, factor, active, then two
        // slots of per-pair iteration records (the pipelined loop)
        const size_t scal_bytes = (size_t)npairs * (18 * 8 + 8) + 64;
        const size_t rec_bytes = (size_t)npairs * sizeof(IterRec);
        char* hp = static_cast<char*>(pinned(ctx, scal_bytes + (size_t)npairs * 32 + 2 * rec_bytes));
        auto push_pairs = [&]() {
            double* hr = reinterpret_cast<double*>(hp + scal_bytes);
            std::memcpy(hr, rho.data(), npairs * sizeof(double));
            std::memcpy(hr + npairs, fac.data(), npairs * sizeof(double));
            std::memcpy(reinterpret_cast<int*>(hr + 2 * npairs), active.data(), npairs * sizeof(int));
            h2d(ctx, pr, hr, (size_t)npairs * (16 + 4));
        };
        push_pairs();
        int* mask_dev = slot_t<int>(ctx, S_TMP2, npairs);
        double* scal_d = slot_t<double>(ctx, S_SCAL, (size_t)npairs * (4 + 8));
        long long* scal_i = slot_t<long long>(ctx, S_TMP1, (size_t)npairs * 6);
        cudaEvent_t eb0 = epc_event_get(ctx), eb1 = epc_event_get(ctx);
        const double V = g.V;
        const double sqrt_n = std::sqrt((double)g.nface);
        int n_active = npairs;
        const bool batch = npairs > 1;
        const bool adaptive = cfg->schedule != EPC_RHO_FIXED;

        // ---- pipelined loop (EPC_MODE_DEVICE_LOOP): decisions on the device --
        // Iteration it+1 is enqueued before the host reads iteration it's
        // records, so the GPU never waits on the host. Every kernel of an
        // iteration honours the per-pair active flags (a pair that stopped
        // carries its state), so the one iteration enqueued past a stop
        // changes nothing. Same kernels, same operations: bitwise the
        // synchronous loop below, rows included. Measured equal to it at
        // C1 / C2 and 0.3% slower at C3 (scripts/probe_loop.py): the host
        // round trip costs about what the three extra launches do, so the
        // synchronous loop stays the default.
        const bool device_loop = (ctx->mode & EPC_MODE_DEVICE_LOOP) != 0;
        if (device_loop) {
            char* actl = static_cast<char*>(slot(ctx, S_ACTL, (size_t)npairs * (16 + 64) + rec_bytes));
            int* need_dev = reinterpret_cast<int*>(actl);
            int* rest_dev = need_dev + npairs;
            int* was_dev = rest_dev + npairs;
            double* seq_io = reinterpret_cast<double*>(actl + (size_t)npairs * 16);
            IterRec* rec_dev = reinterpret_cast<IterRec*>(seq_io + (size_t)npairs * 8);
            IterRec* rec_h[2] = {reinterpret_cast<IterRec*>(hp + scal_bytes + (size_t)npairs * 32),
                                 reinterpret_cast<IterRec*>(hp + scal_bytes + (size_t)npairs * 32 + rec_bytes)};
            cudaEvent_t ev_b0[2] = {eb0, epc_event_get(ctx)}, ev_b1[2] = {eb1, epc_event_get(ctx)};
            cudaEvent_t ev_r[2] = {epc_event_get(ctx), epc_event_get(ctx)};
            DecideArgs D{};
            D.scal_d = scal_d;
            D.scal_i = scal_i;
            D.rho = rho_dev;
            D.fac = fac_dev;
            D.act = act_dev;
            D.need = need_dev;
            D.restore = rest_dev;
            D.was_act = was_dev;
            D.seq_io = seq_io;
            D.rec = rec_dev;
            D.npairs = npairs;
            D.schedule = cfg->schedule;
            D.exact_mode = (ctx->mode & EPC_MODE_EXACT_SUMS) ? 1 : 0;
            D.dim = g.dim;
            D.nface = g.nface;
            D.V = V;
            D.sqrt_n = sqrt_n;
            D.eps_abs = cfg->eps_abs;
            D.eps_rel = cfg->eps_rel;
            D.mu = cfg->mu;
            D.rho_min = cfg->rho_min;
            D.tau_incr = cfg->tau_incr;
            D.tau_decr = cfg->tau_decr;
            D.alpha = p->alpha;
            const int dblk = (npairs + 31) / 32;
            const unsigned gsm = (unsigned)std::min<long long>((long long)ctx->num_sms * 2, (nf + 255) / 256);
            auto enqueue = [&](int k) {
                CK(cudaEventRecord(ev_b0[k], ctx->stream));
                BStepRun br = run_bstep(ctx, g, npairs, ip, im, B[0], Z[0], U[0], B[1], rho_dev,
                                        act_dev, p->alpha, cfg);
                CK(cudaEventRecord(ev_b1[k], ctx->stream));
                const long long total = g.ncol * npairs;
                EPC_LAUNCH(ctx, "reduce_columns", k_reduce_columns, npairs, 1024, 0, br.col_i,
                           br.col_i + total, br.col_i + 2 * total, br.col_i + 3 * total, br.col_d,
                           br.col_d + total, br.col_d + 2 * total, g.ncol, act_dev, scal_d, scal_i);
                ZArgs za{};
                za.b = B[1];
                za.u = U[0];
                za.z_old = Z[0];
                za.z_new = Z[1];
                za.u_new = U[1];
                za.rho = rho_dev;
                za.active = act_dev;
                za.alpha = p->alpha;
                run_zstep(ctx, g, npairs, M, za);
                const int nbz = (int)std::min<long long>(g.ncol, (long long)ctx->num_sms * 4);
                double* zp = slot_t<double>(ctx, S_PART2, (size_t)npairs * nbz * 2);
                EPC_LAUNCH(ctx, "zdiff_sums", k_zdiff_sums, dim3(nbz, npairs), 256, 0, Z[1], g.nface,
                           g.n1, g.m2, g.m3, 1.0 / g.h2, 1.0 / g.h3, zp);
                double* sd2 = scal_d + (size_t)npairs * 4;
                EPC_LAUNCH(ctx, "reduce_dual", k_reduce_partials, npairs, 256, 0, za.partials, za.nblk,
                           6, 6, sd2);
                EPC_LAUNCH(ctx, "reduce_zdiff", k_reduce_partials, npairs, 256, 0, zp, nbz, 2, 2,
                           sd2 + (size_t)npairs * 6);
                EPC_LAUNCH(ctx, "admm_decide", k_admm_decide<0>, dblk, 32, 0, D);
                run_seq_sums_pairs(ctx, B[1], Z[1], Z[0], U[1], g.nface, npairs, seq_io, need_dev);
                EPC_LAUNCH(ctx, "admm_decide", k_admm_decide<1>, dblk, 32, 0, D);
                EPC_LAUNCH(ctx, "admm_tail", k_admm_tail, gsm, 256, 0, B[0], B[1], Z[0], Z[1], U[0], U[1],
                           g.nface, npairs, was_dev, rest_dev, fac_dev);
                std::swap(B[0], B[1]);
                std::swap(Z[0], Z[1]);
                std::swap(U[0], U[1]);
                check_launch();
                d2h(ctx, rec_h[k], rec_dev, rec_bytes);
                CK(cudaEventRecord(ev_r[k], ctx->stream));
            };
            std::vector<int> live(npairs, 1);
            auto process = [&](int it, int k) {
                CK(cudaEventSynchronize(ev_r[k]));
                float bms = 0.f;
                CK(cudaEventElapsedTime(&bms, ev_b0[k], ev_b1[k]));
                const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                for (int q = 0; q < npairs; ++q) {
                    if (!live[q]) continue;
                    const IterRec& r = rec_h[k][q];
                    if (r.stop == EPC_STOP_ERROR) {
                        status[q].stop = EPC_STOP_ERROR;
                        std::snprintf(status[q].message, sizeof status[q].message,
                                      "b_update: column %lld: %s", r.err_col, qp_what(r.err_code));
                        live[q] = 0;
                        --n_active;
                        continue;
                    }
                    if (!r.has_row) continue;
                    ctx->sqp_total += r.sqp;
                    ctx->qp_total += r.qp;
                    if (r.exact) ctx->dec_exact++;
                    else ctx->dec_certified++;
                    epc_admm_row row{};
                    row.level = level_tag;
                    row.iter = it;
                    row.rho = r.rho_used;
                    row.kkt_violation = r.kkt;
                    row.b_update_s = bms * 1e-3;
                    row.primal_res = r.pr;
                    row.dual_res = r.du;
                    row.eps_pri = r.eps_pri;
                    row.eps_dual = r.eps_dual;
                    row.lagrangian = r.lag;
                    row.wall_s = wall;
                    if (status[q].nrows < max_rows) rows[(size_t)q * max_rows + status[q].nrows] = row;
                    status[q].nrows++;
                    if (r.stop == EPC_STOP_CONVERGED) {
                        status[q].stop = EPC_STOP_CONVERGED;
                        live[q] = 0;
                        --n_active;
                    }
                }
            };
            int last = 0;  // last enqueued iteration not yet processed
            for (int it = 1; it <= cfg->max_iter && n_active > 0; ++it) {
                enqueue(it & 1);
                if (last) process(last, last & 1);
                last = it;
            }
            if (last && n_active > 0) process(last, last & 1);
            // the rho each pair ended with (changed on the device)
            double* hr = reinterpret_cast<double*>(hp + scal_bytes);
            d2h(ctx, hr, rho_dev, (size_t)npairs * sizeof(double));
            sync(ctx);
            for (int q = 0; q < npairs; ++q) rho[q] = hr[q];
            CK(cudaEventDestroy(ev_b0[1]));
            CK(cudaEventDestroy(ev_b1[1]));
            CK(cudaEventDestroy(ev_r[0]));
            CK(cudaEventDestroy(ev_r[1]));
        }

        // the forward axis-2 transform in the b-step's drain (BStepParams::fwd2);
        // EPC_FUSE_FWD2=0: the separate GEMM launch (dev A/B; same bits)
        static const bool fuse_env = !getenv("EPC_FUSE_FWD2") || atoi(getenv("EPC_FUSE_FWD2")) != 0;
        // Only after a short b-step: with a long tail (x400: 40-80 ms launches)
        // the drain's transform is a sliver of the launch and its warps
        // compete with the tail columns (EPC_FUSE_MAX_MS, default 12 ms)
        static const double fuse_max_ms = getenv("EPC_FUSE_MAX_MS") ? atof(getenv("EPC_FUSE_MAX_MS")) : 12.0;
        const bool fuse_fwd2_ok = fuse_env && g.m3 > 1;
        double prev_bstep_ms = -1.0;  // the previous iteration's b-step (events eb0 / eb1)
        // Longest columns first while the launches are bulk-bound (the first
        // ~25 iterations of a C3 solve: 5-12 ms launches whose column costs
        // repeat from one iteration to the next, correlation 0.9-0.98, and
        // whose last 11-15% is an under-filled tail): every launch records
        // its columns' cycles, and after a launch of EPC_LPT_MIN_MS or more the
        // next one claims columns by descending recorded cost. Late launches'
        // heavy columns do not repeat (DESIGN 4), so they keep the k-layer
        // order, which also feeds the fused forward axis-2 transform early.
        // Columns are independent: the order cannot change a bit of b.
        static const double lpt_min_ms = getenv("EPC_LPT_MIN_MS") ? atof(getenv("EPC_LPT_MIN_MS")) : 5.0;
        const long long total_cols = g.ncol * npairs;
        const bool lpt_ok = total_cols < (1LL << 31);
        // two cost arrays, written alternately. EPC_LPT_TWO=1 keys the order on
        // the larger of the last two launches' costs (measured: no better than
        // the last launch's alone, profiles/r02fj_lpt_ab.log; off by default)
        static const bool lpt_two = getenv("EPC_LPT_TWO") && atoi(getenv("EPC_LPT_TWO")) != 0;
        unsigned* lpt_cost = lpt_ok ? slot_t<unsigned>(ctx, S_LPTC, (size_t)total_cols * 2) : nullptr;
        int lpt_have = 0;  // launches of this solve that recorded their costs
        // A column predicted to outlast the balanced makespan (its cost at least
        // EPC_LPT_CRIT, default 0.8, of total / resident warps; x400: a handful
        // of 50-75 ms columns against 45 ms) bounds the launch by itself, and
        // runs 20-40% slower beside seven other heavy columns than alone. While
        // one runs, its SM's other warps wait instead of claiming (at most 32
        // such columns per launch; none at unit intensity).
#ifdef EPC_CRIT
        static const double lpt_crit = getenv("EPC_LPT_CRIT") ? atof(getenv("EPC_LPT_CRIT")) : 0.8;
#else  // the kernel side is compiled out by default (it costs 0.8% at unit intensity)
        static const double lpt_crit = 0.0;
#endif
        const int nsm_pad = 1024;  // %smid < this on any part
        unsigned* lpt_critbuf = (lpt_ok && lpt_crit > 0.0) ? slot_t<unsigned>(ctx, S_LPTK, 1 + nsm_pad + 4096) : nullptr;  // + a flag per CTA
        const double lpt_slots = (double)std::min<long long>((long long)ctx->num_sms * 8, total_cols);
        int* lpt_order = lpt_ok ? slot_t<int>(ctx, S_LPTO, (size_t)total_cols) : nullptr;
        for (int it = 1; !device_loop && it <= cfg->max_iter && n_active > 0; ++it) {
            // ---- b-step ----------------------------------------------------------
            CK(cudaEventRecord(eb0, ctx->stream));
            const bool fuse_fwd2 = fuse_fwd2_ok && prev_bstep_ms >= 0.0 && prev_bstep_ms < fuse_max_ms;
            Fwd2Params f2{};
            if (fuse_fwd2) {
                f2.A = M.c2;
                f2.b = B[1];
                f2.u = U[0];
                f2.rho = rho_dev;
                f2.out = slot_t<double>(ctx, S_H1, (size_t)g.nface * npairs);
                f2.V = g.V;
                f2.nface = g.nface;
                f2.n1 = g.n1;
                f2.m2 = g.m2;
                f2.m3 = g.m3;
                f2.npairs = npairs;
            }
            const bool lpt = lpt_ok && prev_bstep_ms >= lpt_min_ms;
            unsigned* cost_now = lpt_ok ? lpt_cost + (size_t)(lpt_have & 1) * total_cols : nullptr;
            if (lpt) {
                const unsigned* c1 = lpt_cost + (size_t)((lpt_have - 1) & 1) * total_cols;
                const unsigned* c2 = (lpt_have >= 2 && lpt_two) ? cost_now : c1;  // two launches ago
                EPC_LAUNCH(ctx, "lpt_order", k_lpt_order, 1, 1024, 0, c1, c2, lpt_order, total_cols,
                           lpt_critbuf, lpt_crit / lpt_slots, 32, nsm_pad + 4096);
            }
            BStepRun br = run_bstep(ctx, g, npairs, ip, im, B[0], Z[0], U[0], B[1], rho_dev,
                                    batch ? act_dev : nullptr, p->alpha, cfg,
                                    fuse_fwd2 ? &f2 : nullptr, cost_now, lpt ? lpt_order : nullptr, lpt_critbuf);
            ++lpt_have;
            CK(cudaEventRecord(eb1, ctx->stream));
            const long long total = g.ncol * npairs;
            EPC_LAUNCH(ctx, "reduce_columns", k_reduce_columns, npairs, 1024, 0, br.col_i,
                       br.col_i + total, br.col_i + 2 * total, br.col_i + 3 * total, br.col_d,
                       br.col_d + total, br.col_d + 2 * total, g.ncol,
                       batch ? act_dev : nullptr, scal_d, scal_i);
            // ---- z-step + dual update ---------------------------------------------
            ZArgs za{};
            za.b = B[1];
            za.u = U[0];
            za.z_old = Z[0];
            za.z_new = Z[1];
            za.u_new = U[1];
            za.rho = rho_dev;
            za.active = batch ? act_dev : nullptr;
            za.alpha = p->alpha;
            za.fwd2_done = br.fwd2_fused;
            run_zstep(ctx, g, npairs, M, za);
            const int nbz = (int)std::min<long long>(g.ncol, (long long)ctx->num_sms * 4);
            double* zp = slot_t<double>(ctx, S_PART2, (size_t)npairs * nbz * 2);
            EPC_LAUNCH(ctx, "zdiff_sums", k_zdiff_sums, dim3(nbz, npairs), 256, 0, Z[1], g.nface,
                       g.n1, g.m2, g.m3, 1.0 / g.h2, 1.0 / g.h3, zp);
            double* sd2 = scal_d + (size_t)npairs * 4;  // 6 dual sums + 2 zdiff sums per pair
            EPC_LAUNCH(ctx, "reduce_dual", k_reduce_partials, npairs, 256, 0, za.partials, za.nblk,
                       6, 6, sd2);
            EPC_LAUNCH(ctx, "reduce_zdiff", k_reduce_partials, npairs, 256, 0, zp, nbz, 2, 2,
                       sd2 + (size_t)npairs * 6);
            check_launch();
            // ---- one read-back of all per-pair scalars -----------------------------
            double* hs = reinterpret_cast<double*>(hp);
            d2h(ctx, hs, scal_d, (size_t)npairs * 12 * sizeof(double));
            long long* hi = reinterpret_cast<long long*>(hs + (size_t)npairs * 12);
            d2h(ctx, hi, scal_i, (size_t)npairs * 6 * sizeof(long long));
            sync(ctx);
            float bms = 0.f;
            CK(cudaEventElapsedTime(&bms, eb0, eb1));
            prev_bstep_ms = bms;
            const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

            bool any_restore = false, any_rho = false;
            std::vector<int> was_active = active;
            for (int q = 0; q < npairs; ++q) {
                fac[q] = 1.0;
                restore[q] = 0;
                if (!was_active[q]) continue;
                const double* cd = hs + (size_t)q * 4;
                const long long* ci = hi + (size_t)q * 6;
                const double* du = hs + (size_t)npairs * 4 + (size_t)q * 6;
                const double* zd = hs + (size_t)npairs * 10 + (size_t)q * 2;
                if (ci[0] >= 0) {  // a column failed: stop = error, state unchanged
                    status[q].stop = EPC_STOP_ERROR;
                    std::snprintf(status[q].message, sizeof status[q].message,
                                  "b_update: column %lld: %s", ci[0], qp_what((int)ci[1]));
                    active[q] = 0;
                    restore[q] = 1;
                    any_restore = true;
                    --n_active;
                    continue;
                }
                ctx->sqp_total += ci[2];
                ctx->qp_total += ci[3];
                epc_admm_row row{};
                row.level = level_tag;
                row.iter = it;
                row.rho = rho[q];
                row.kkt_violation = cd[0];
                row.b_update_s = bms * 1e-3;
                // dual_update_and_residuals (admm.cpp:470-474) on the tree sums
                const epc_decide::Res tr = epc_decide::residuals(du, rho[q], V, sqrt_n,
                                                                 cfg->eps_abs, cfg->eps_rel);
                row.primal_res = tr.pr;
                row.dual_res = tr.du;
                row.eps_pri = tr.eps_pri;
                row.eps_dual = tr.eps_dual;
                // stop test and rho schedule (admm.cpp:542-548): certified against the
                // reference's sequential sums, else decided on those sums (admm_decide.h)
                epc_decide::Decision dec{false, false, 0};
                if (!(ctx->mode & EPC_MODE_EXACT_SUMS))
                    dec = epc_decide::certified(du, g.nface, rho[q], V, sqrt_n, cfg->eps_abs,
                                                cfg->eps_rel, cfg->mu, adaptive);
                if (dec.decided) {
                    ctx->dec_certified++;
                } else {
                    double seq[5];
                    const size_t o = (size_t)q * g.nface;
                    seq_sums(ctx, B[1] + o, Z[1] + o, Z[0] + o, U[1] + o, g.nface, seq);
                    const epc_decide::Res ex = epc_decide::residuals(seq, rho[q], V, sqrt_n,
                                                                     cfg->eps_abs, cfg->eps_rel);
                    row.primal_res = ex.pr;  // now bitwise the reference's row values
                    row.dual_res = ex.du;
                    row.eps_pri = ex.eps_pri;
                    row.eps_dual = ex.eps_dual;
                    dec = epc_decide::exact(seq, rho[q], V, sqrt_n, cfg->eps_abs, cfg->eps_rel,
                                            cfg->mu, adaptive);
                    ctx->dec_exact++;
                }
                // augmented_lagrangian (admm.cpp:267-299)
                const double fval = 0.5 * V * cd[1] + 0.5 * p->alpha * V * cd[2];
                double gs = zd[0];
                if (g.dim == 3) gs += zd[1];
                const double gval = 0.5 * p->alpha * V * gs;
                row.lagrangian = fval + gval + rho[q] * V * du[5] + 0.5 * rho[q] * V * du[0];
                row.wall_s = wall;
                if (status[q].nrows < max_rows) rows[(size_t)q * max_rows + status[q].nrows] = row;
                status[q].nrows++;
                if (dec.converged) {
                    status[q].stop = EPC_STOP_CONVERGED;
                    active[q] = 0;
                    --n_active;
                    continue;
                }
                const double next = rho_apply(cfg->schedule, rho[q], cfg->rho_min, dec.rho_move,
                                              cfg->tau_incr, cfg->tau_decr);
                if (next != rho[q]) {
                    fac[q] = rho[q] / next;
                    rho[q] = next;
                    any_rho = true;
                }
            }
            // inactive-before pairs: b-step skipped them, carry b over
            bool any_inactive_before = false;
            for (int q = 0; q < npairs; ++q) any_inactive_before |= !was_active[q];
            if (any_inactive_before) {
                std::vector<int> m(npairs);
                for (int q = 0; q < npairs; ++q) m[q] = !was_active[q];
                int* hm = reinterpret_cast<int*>(hi + (size_t)npairs * 6);
                std::memcpy(hm, m.data(), npairs * sizeof(int));
                h2d(ctx, mask_dev, hm, npairs * sizeof(int));
                EPC_LAUNCH(ctx, "carry_b", k_copy_masked, grid1d(ctx, (long long)nf), 256, 0, B[0], B[1],
                           g.nface, npairs, mask_dev);
                sync(ctx);
            }
            if (any_restore) {  // errored pairs: keep the state from before this iteration
                int* hm = reinterpret_cast<int*>(hi + (size_t)npairs * 6);
                std::memcpy(hm, restore.data(), npairs * sizeof(int));
                h2d(ctx, mask_dev, hm, npairs * sizeof(int));
                EPC_LAUNCH(ctx, "restore_b", k_copy_masked, grid1d(ctx, (long long)nf), 256, 0, B[0], B[1], g.nface, npairs, mask_dev);
                EPC_LAUNCH(ctx, "restore_z", k_copy_masked, grid1d(ctx, (long long)nf), 256, 0, Z[0], Z[1], g.nface, npairs, mask_dev);
                EPC_LAUNCH(ctx, "restore_u", k_copy_masked, grid1d(ctx, (long long)nf), 256, 0, U[0], U[1], g.nface, npairs, mask_dev);
                sync(ctx);
            }
            std::swap(B[0], B[1]);
            std::swap(Z[0], Z[1]);
            std::swap(U[0], U[1]);
            if (any_rho) {
                push_pairs();
                EPC_LAUNCH(ctx, "scale_u", k_scale_pairs, grid1d(ctx, (long long)nf), 256, 0, U[0],
                           g.nface, npairs, fac_dev);
                check_launch();
                for (int q = 0; q < npairs; ++q) fac[q] = 1.0;
            } else if (n_active < npairs) {
                push_pairs();
            }
            sync(ctx);
        }
        // outputs
        stage_out(ctx, mem, b_out, B[0], nf);
        stage_out(ctx, mem, z_out, Z[0], nf);
        stage_out(ctx, mem, u_out, U[0], nf);
        sync(ctx);
        for (int q = 0; q < npairs; ++q) rho_io[q] = rho[q];
        CK(cudaEventDestroy(eb0));
        CK(cudaEventDestroy(eb1));
    });
}

}  // namespace

// ===========================================================================
// profiling hooks (declared in common.cuh)
// ===========================================================================
cudaEvent_t epc_event_get(epc_context* ctx) {
    cudaEvent_t e;
    if (!ctx->event_pool.empty()) {
        e = ctx->event_pool.back();
        ctx->event_pool.pop_back();
        return e;
    }
    cudaEventCreate(&e);
    return e;
}

void epc_prof_begin(epc_context* ctx, const char* name, cudaEvent_t* ev0) {
    (void)name;
    *ev0 = epc_event_get(ctx);
    cudaEventRecord(*ev0, ctx->stream);
}

void epc_prof_end(epc_context* ctx, const char* name, cudaEvent_t ev0) {
    cudaEvent_t e1 = epc_event_get(ctx);
    cudaEventRecord(e1, ctx->stream);
    ctx->prof_pending.push_back(ProfEntry{name, ev0, e1});
}

static void prof_drain(epc_context* ctx) {
    cudaStreamSynchronize(ctx->stream);
    for (auto& pe : ctx->prof_pending) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, pe.start, pe.stop);
        bool found = false;
        for (auto& a : ctx->prof_acc)
            if (std::strcmp(a.name, pe.name) == 0) {
                a.ms += ms;
                a.n += 1;
                found = true;
                break;
            }
        if (!found) ctx->prof_acc.push_back({pe.name, (double)ms, 1});
        ctx->event_pool.push_back(pe.start);
        ctx->event_pool.push_back(pe.stop);
    }
    ctx->prof_pending.clear();
}

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

void epc_default_params(epc_objective_params* p) {
    p->alpha = 50.0;
    p->beta = 10.0;
    p->gamma = 1e-3;
    p->enforce_linf_box = 0;
}

void epc_default_admm_config(epc_admm_config* c) {
    c->rho0 = 1e6;
    c->rho_min = 1e2;
    c->schedule = EPC_RHO_ADAPTIVE_BOUNDED;
    c->eps_abs = 0.2;
    c->eps_rel = 0.2;
    c->max_iter = 50;
    c->tau_incr = 2.0;
    c->tau_decr = 2.0;
    c->mu = 10.0;
    c->sqp_max_iter = 20;
    c->sqp_tol_rel = 1e-2;
    c->check_kkt = 1;
    c->threads = 1;
}

void epc_default_gn_config(epc_gn_config* c) {
    c->eta = 0.1;
    c->max_outer = 10;
    c->eps_obj = 1e-3;
    c->eps_iter = 1e-2;
    c->eps_grad = 1e-2;
    c->wolfe_c1 = 1e-4;
    c->wolfe_c2 = 0.9;
    c->max_pcg = 100;
    c->max_ls = 30;
    c->precond = EPC_PRECOND_BLOCK_JACOBI;
    c->threads = 1;
}

int epc_context_create(int device, void* stream, epc_context** out) {
    if (!out) return EPC_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    epc_context* ctx = new epc_context();
    const int rc = guarded(ctx, [&] {
        int n = 0;
        CK(cudaGetDeviceCount(&n));
        if (n <= 0) fail(EPC_ERR_CUDA, "no CUDA device");
        CK(cudaSetDevice(device));
        ctx->device = device;
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10) fail(EPC_ERR_UNSUPPORTED, std::string("libepicorr_b200 is built for sm_100a; device is ") + prop.name);
        ctx->num_sms = prop.multiProcessorCount;
        ctx->guard = getenv("EPC_GUARD") && atoi(getenv("EPC_GUARD")) != 0;
        ctx->smem_optin = prop.sharedMemPerBlockOptin;
        if (stream) {
            ctx->stream = static_cast<cudaStream_t>(stream);
        } else {
            CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
            ctx->own_stream = true;
        }
    });
    if (rc != EPC_OK) {
        static thread_local std::string keep;
        keep = ctx->last_error;
        delete ctx;
        return rc;
    }
    *out = ctx;
    return EPC_OK;
}

void epc_context_destroy(epc_context* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (auto& b : ctx->bufs)
        if (b.ptr) cudaFree(static_cast<char*>(b.ptr) - (ctx->guard ? GUARD_BYTES : 0));
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    if (ctx->pinned_aux) cudaFreeHost(ctx->pinned_aux);
    for (auto& pe : ctx->prof_pending) {
        cudaEventDestroy(pe.start);
        cudaEventDestroy(pe.stop);
    }
    for (auto e : ctx->event_pool) cudaEventDestroy(e);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

int epc_set_stream(epc_context* ctx, void* stream) {
    return guarded(ctx, [&] {
        if (ctx->own_stream) {
            CK(cudaStreamSynchronize(ctx->stream));
            CK(cudaStreamDestroy(ctx->stream));
            ctx->own_stream = false;
        }
        if (stream) ctx->stream = static_cast<cudaStream_t>(stream);
        else {
            CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
            ctx->own_stream = true;
        }
    });
}

const char* epc_last_error(const epc_context* ctx) { return ctx ? ctx->last_error.c_str() : "null context"; }

int epc_set_mode(epc_context* ctx, int mode_bits) {
    return guarded(ctx, [&] {
        if ((mode_bits & EPC_MODE_BSTEP_TIMING) && !(ctx->mode & EPC_MODE_BSTEP_TIMING)) {
            long long* t = slot_t<long long>(ctx, S_GN9, 28);
            CK(cudaMemsetAsync(t, 0, 28 * sizeof(long long), ctx->stream));
        }
        ctx->mode = mode_bits;
    });
}

int epc_bstep_timing(epc_context* ctx, long long* out10) {
    return guarded(ctx, [&] {
        long long* t = slot_t<long long>(ctx, S_GN9, 28);
        d2h(ctx, out10, t, 10 * sizeof(long long));
        sync(ctx);
    });
}

int epc_bstep_counters(epc_context* ctx, long long* out18) {
    return guarded(ctx, [&] {
        long long* t = slot_t<long long>(ctx, S_GN9, 28);
        d2h(ctx, out18, t + 10, 18 * sizeof(long long));
        sync(ctx);
    });
}

int epc_profile_enable(epc_context* ctx, int on) {
    if (!on && ctx->profiling) prof_drain(ctx);
    ctx->profiling = on != 0;
    return EPC_OK;
}

int epc_profile_read(epc_context* ctx, const char** names, double* total_ms, long* launches,
                     int cap, int* count) {
    prof_drain(ctx);
    const int n = (int)ctx->prof_acc.size();
    for (int i = 0; i < n && i < cap; ++i) {
        names[i] = ctx->prof_acc[i].name;
        total_ms[i] = ctx->prof_acc[i].ms;
        launches[i] = ctx->prof_acc[i].n;
    }
    if (count) *count = n;
    return EPC_OK;
}

void epc_profile_reset(epc_context* ctx) {
    prof_drain(ctx);
    ctx->prof_acc.clear();
}

long epc_launch_count(const epc_context* ctx) { return ctx->launches; }

int epc_guard_check(epc_context* ctx, int* bad_slot) {
    return guarded(ctx, [&] {
        *bad_slot = -1;
        if (!ctx->guard) fail(EPC_ERR_UNSUPPORTED, "guard_check: context not created with EPC_GUARD=1");
        int* flag = static_cast<int*>(pinned_aux(ctx));
        for (int sidx = 0; sidx < (int)ctx->bufs.size() && *bad_slot < 0; ++sidx) {
            const DevBuf& b = ctx->bufs[sidx];
            if (!b.ptr) continue;
            const unsigned char* lo = static_cast<const unsigned char*>(b.ptr) - GUARD_BYTES;
            const unsigned char* hi = static_cast<const unsigned char*>(b.ptr) + b.bytes;
            for (const unsigned char* z : {lo, hi}) {
                std::vector<unsigned char> h(GUARD_BYTES);
                CK(cudaMemcpyAsync(h.data(), z, GUARD_BYTES, cudaMemcpyDeviceToHost, ctx->stream));
                sync(ctx);
                for (unsigned char c : h)
                    if (c != 0xA5) {
                        *bad_slot = sidx;
                        break;
                    }
            }
        }
        (void)flag;
    });
}

int epc_admm_counters(epc_context* ctx, long long* out4) {
    if (!ctx || !out4) return EPC_ERR_INVALID_ARGUMENT;
    out4[0] = ctx->dec_certified;
    out4[1] = ctx->dec_exact;
    out4[2] = ctx->sqp_total;
    out4[3] = ctx->qp_total;
    return EPC_OK;
}
void epc_reset_launch_count(epc_context* ctx) { ctx->launches = 0; }

int epc_admm_solve(epc_context* ctx, const epc_grid* g, int mem, const double* iplus,
                   const double* iminus, const double* b_in, const double* z_in,
                   const double* u_in, double* b_out, double* z_out, double* u_out, double* rho,
                   const epc_objective_params* p, const epc_admm_config* cfg, int level_tag,
                   epc_admm_row* rows, int max_rows, epc_solve_status* status) {
    return admm_solve_impl(ctx, g, 1, mem, iplus, iminus, b_in, z_in, u_in, b_out, z_out, u_out,
                           rho, p, cfg, level_tag, rows, max_rows, status);
}

int epc_admm_solve_batch(epc_context* ctx, const epc_grid* g, int npairs, int mem,
                         const double* iplus, const double* iminus, const double* b_in,
                         const double* z_in, const double* u_in, double* b_out, double* z_out,
                         double* u_out, double* rho, const epc_objective_params* p,
                         const epc_admm_config* cfg, int level_tag, epc_admm_row* rows,
                         int max_rows, epc_solve_status* status) {
    if (npairs < 1) return EPC_ERR_INVALID_ARGUMENT;
    return admm_solve_impl(ctx, g, npairs, mem, iplus, iminus, b_in, z_in, u_in, b_out, z_out,
                           u_out, rho, p, cfg, level_tag, rows, max_rows, status);
}

int epc_b_update(epc_context* ctx, const epc_grid* gg, int mem, const double* iplus,
                 const double* iminus, const double* b, const double* z, const double* u,
                 double rho, const epc_objective_params* p, const epc_admm_config* cfg,
                 double* b_out, epc_bupdate_stats* stats) {
    return guarded(ctx, [&] {
        const Geo g = make_geo(gg);
        if (!(rho > 0.0)) fail(EPC_ERR_INVALID_ARGUMENT, "b_update: rho must be positive");
        const size_t nc = g.ncell, nf = g.nface;
        const double* ip = mem == EPC_MEM_DEVICE ? iplus : stage_in(ctx, S_IP, mem, iplus, nc);
        const double* im = mem == EPC_MEM_DEVICE ? iminus : stage_in(ctx, S_IM, mem, iminus, nc);
        double* bd = stage_in(ctx, S_B0, mem, b, nf);
        double* zd = stage_in(ctx, S_Z0, mem, z, nf);
        double* ud = stage_in(ctx, S_U0, mem, u, nf);
        double* bo = slot_t<double>(ctx, S_B1, nf);
        double* rd = slot_t<double>(ctx, S_PAIR, 4);
        h2d(ctx, rd, &rho, sizeof(double));
        BStepRun br = run_bstep(ctx, g, 1, ip, im, bd, zd, ud, bo, rd, nullptr, p->alpha, cfg);
        double* sd = slot_t<double>(ctx, S_SCAL, 4);
        long long* si = slot_t<long long>(ctx, S_TMP1, 6);
        const long long total = g.ncol;
        EPC_LAUNCH(ctx, "reduce_columns", k_reduce_columns, 1, 1024, 0, br.col_i, br.col_i + total,
                   br.col_i + 2 * total, br.col_i + 3 * total, br.col_d, br.col_d + total,
                   br.col_d + 2 * total, g.ncol, nullptr, sd, si);
        double hd[4];
        long long hi[6];
        d2h(ctx, hd, sd, sizeof hd);
        d2h(ctx, hi, si, sizeof hi);
        sync(ctx);
        if (hi[0] >= 0) {
            char m[256];
            std::snprintf(m, sizeof m, "b_update: column %lld: %s", hi[0], qp_what((int)hi[1]));
            fail(EPC_ERR_RUNTIME, m);
        }
        stage_out(ctx, mem, b_out, bo, nf);
        sync(ctx);
        if (stats) {
            stats->sqp_iters = (long)hi[2];
            stats->qp_iters = (long)hi[3];
            stats->kkt_violation = hd[0];
            stats->max_active = (int)hi[4];
        }
    });
}

int epc_dct_solve(epc_context* ctx, const epc_grid* gg, int mem, const double* rhs, double alpha,
                  double rho, double* out) {
    return guarded(ctx, [&] {
        const Geo g = make_geo(gg);
        if (!(alpha > 0.0)) fail(EPC_ERR_INVALID_ARGUMENT, "dct_coupled_solve: alpha must be > 0");
        if (!(rho > 0.0)) fail(EPC_ERR_INVALID_ARGUMENT, "dct_coupled_solve: rho must be > 0");
        const size_t nf = g.nface;
        double* rd = stage_in(ctx, S_B0, mem, rhs, nf);
        double* zo = slot_t<double>(ctx, S_Z1, nf);
        const DctMats M = upload_dct(ctx, g);
        double* rh = slot_t<double>(ctx, S_PAIR, 4);
        h2d(ctx, rh, &rho, sizeof(double));
        ZArgs za{};
        za.b = rd;
        za.u = rd;
        za.z_new = zo;
        za.rho = rh;
        za.alpha = alpha;
        za.rhs_is_raw = true;
        run_zstep(ctx, g, 1, M, za);
        stage_out(ctx, mem, out, zo, nf);
        sync(ctx);
    });
}

int epc_z_update(epc_context* ctx, const epc_grid* gg, int mem, const double* b, const double* u,
                 double rho, double alpha, double* z_out) {
    return guarded(ctx, [&] {
        const Geo g = make_geo(gg);
        if (!(alpha > 0.0)) fail(EPC_ERR_INVALID_ARGUMENT, "dct_coupled_solve: alpha must be > 0");
        if (!(rho > 0.0)) fail(EPC_ERR_INVALID_ARGUMENT, "dct_coupled_solve: rho must be > 0");
        const size_t nf = g.nface;
        double* bd = stage_in(ctx, S_B0, mem, b, nf);
        double* ud = stage_in(ctx, S_U0, mem, u, nf);
        double* zo = slot_t<double>(ctx, S_Z1, nf);
        const DctMats M = upload_dct(ctx, g);
        double* rh = slot_t<double>(ctx, S_PAIR, 4);
        h2d(ctx, rh, &rho, sizeof(double));
        ZArgs za{};
        za.b = bd;
        za.u = ud;
        za.z_new = zo;
        za.rho = rh;
        za.alpha = alpha;
        run_zstep(ctx, g, 1, M, za);
        stage_out(ctx, mem, z_out, zo, nf);
        sync(ctx);
    });
}

int epc_dual_update(epc_context* ctx, const epc_grid* gg, int mem, const double* b_new,
                    const double* z_new, const double* z_old, const double* u_old, double rho,
                    double eps_abs, double eps_rel, double* u_out, epc_dual_result* out) {
    return guarded(ctx, [&] {
        // The fused path computes this inside the z-step epilogue; this entry
        // point evaluates the same element-wise update and sums standalone.
        const Geo g = make_geo(gg);
        const size_t nf = g.nface;
        double* bd = stage_in(ctx, S_B0, mem, b_new, nf);
        double* zn = stage_in(ctx, S_Z0, mem, z_new, nf);
        double* zo = stage_in(ctx, S_Z1, mem, z_old, nf);
        double* uo = stage_in(ctx, S_U0, mem, u_old, nf);
        double* un = slot_t<double>(ctx, S_U1, nf);
        const int nb = 128;
        double* part = slot_t<double>(ctx, S_PART, (size_t)nb * 6);
        EPC_LAUNCH(ctx, "dual_update", k_dual_standalone, nb, 256, 0, bd, zn, zo, uo, un, (long long)nf, part);
        double* s = slot_t<double>(ctx, S_SCAL, 6);
        EPC_LAUNCH(ctx, "reduce_dual", k_reduce_partials, 1, 256, 0, part, nb, 6, 6, s);
        check_launch();
        double hs[6];
        d2h(ctx, hs, s, sizeof hs);
        stage_out(ctx, mem, u_out, un, nf);
        sync(ctx);
        const double V = g.V;
        const double sqrt_n = std::sqrt((double)g.nface);
        if (out) {
            out->primal_res = std::sqrt(hs[0]);
            out->dual_res = rho * V * std::sqrt(hs[1]);
            out->eps_pri = sqrt_n * eps_abs + eps_rel * std::max(std::sqrt(hs[2]), std::sqrt(hs[3]));
            out->eps_dual = sqrt_n * eps_abs + eps_rel * rho * V * std::sqrt(hs[4]);
        }
    });
}

int epc_augmented_lagrangian(epc_context* ctx, const epc_grid* gg, int mem, const double* iplus,
                             const double* iminus, const double* b, const double* z,
                             const double* u, double rho, double alpha, double* out) {
    return guarded(ctx, [&] {
        const Geo g = make_geo(gg);
        const size_t nc = g.ncell, nf = g.nface;
        const double* ip = mem == EPC_MEM_DEVICE ? iplus : stage_in(ctx, S_IP, mem, iplus, nc);
        const double* im = mem == EPC_MEM_DEVICE ? iminus : stage_in(ctx, S_IM, mem, iminus, nc);
        double* bd = stage_in(ctx, S_B0, mem, b, nf);
        double* zd = stage_in(ctx, S_Z0, mem, z, nf);
        double* ud = stage_in(ctx, S_U0, mem, u, nf);
        const int nb = 128;
        double* part = slot_t<double>(ctx, S_PART, (size_t)nb * 4);
        EPC_LAUNCH(ctx, "lagr_sums", k_lagr_sums, nb, 256, 0, ip, im, bd, zd, ud, g.m1, g.n1,
                   g.ncell, g.nface, make_hdiv(g.h1), g.o1, part);
        double* zp = slot_t<double>(ctx, S_PART2, (size_t)64 * 2);
        EPC_LAUNCH(ctx, "zdiff_sums", k_zdiff_sums, dim3(64, 1), 256, 0, zd, g.nface, g.n1, g.m2,
                   g.m3, 1.0 / g.h2, 1.0 / g.h3, zp);
        double* s = slot_t<double>(ctx, S_SCAL, 6);
        EPC_LAUNCH(ctx, "reduce_lagr", k_reduce_partials, 1, 256, 0, part, nb, 4, 4, s);
        EPC_LAUNCH(ctx, "reduce_zdiff", k_reduce_partials, 1, 256, 0, zp, 64, 2, 2, s + 4);
        check_launch();
        double hs[6];
        d2h(ctx, hs, s, sizeof hs);
        sync(ctx);
        const double V = g.V;
        const double fval = 0.5 * V * hs[0] + 0.5 * alpha * V * hs[1];
        double gs = hs[4];
        if (g.dim == 3) gs += hs[5];
        const double gval = 0.5 * alpha * V * gs;
        *out = fval + gval + rho * V * hs[2] + 0.5 * rho * V * hs[3];
    });
}

double epc_rho_schedule(int schedule, double rho, double rho_min, double primal_res,
                        double dual_res, double tau_incr, double tau_decr, double mu) {
    return rho_schedule(schedule, rho, rho_min, primal_res, dual_res, tau_incr, tau_decr, mu);
}

int epc_qp_active_set_batch(epc_context* ctx, int nqp, int n, double h, const double* gd,
                            const double* go, const double* c, const double* x0, int max_iter,
                            double* x, double* lambda, int* active_sign, int* iters, double* kkt,
                            int* status) {
    return guarded(ctx, [&] {
        if (nqp < 1 || n < 2) fail(EPC_ERR_INVALID_ARGUMENT, "qp batch: need nqp >= 1, n >= 2");
        const size_t nv = (size_t)nqp * n, nl = (size_t)nqp * (n - 1);
        double* dgd = stage_in(ctx, S_TMP0, EPC_MEM_HOST, gd, nv);
        double* dgo = stage_in(ctx, S_H1, EPC_MEM_HOST, go, nv);
        double* dc = stage_in(ctx, S_H2, EPC_MEM_HOST, c, nv);
        double* dx0 = stage_in(ctx, S_B0, EPC_MEM_HOST, x0, nv);
        double* dx = slot_t<double>(ctx, S_B1, nv);
        double* dl = slot_t<double>(ctx, S_Z0, nl);
        int* ds = slot_t<int>(ctx, S_COLI, nl + 3 * (size_t)nqp);
        double* dk = slot_t<double>(ctx, S_Z1, nqp);
        const size_t smem = bstep_smem_bytes(n);
        if (smem > ctx->smem_optin) fail(EPC_ERR_UNSUPPORTED, "QP too long for shared memory");
        // EPC_MODE_BSTEP_TIMING: the instrumented build, QP phase cycles into the
        // b-step timing slot (epc_bstep_timing: factor, g, solves, Schur
        // formation, Schur solve, p update, ratio test / append; dev aid)
        const bool qdiag = (ctx->mode & EPC_MODE_BSTEP_TIMING) != 0;
        void (*qk)(QpBatchParams) = qdiag ? k_qp_batch<true> : k_qp_batch<false>;
        CK(cudaFuncSetAttribute(qk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->smem_optin));
        const int blocks = std::min(nqp, ctx->num_sms * 8);
        const int qcap = n - 1;
        QpBatchParams P{};
        P.nqp = nqp;
        P.n = n;
        P.dh = make_hdiv(h);
        P.gd = dgd;
        P.go = dgo;
        P.c = dc;
        P.x0 = dx0;
        P.max_iter = max_iter;
        P.x = dx;
        P.lambda = dl;
        P.sign = ds;
        P.iters = ds + nl;
        P.status = ds + nl + nqp;
        P.kkt = dk;
        P.qbuf = slot_t<double>(ctx, S_QBUF, (size_t)blocks * qrows_stride(qcap, n));
        P.sbuf = slot_t<double>(ctx, S_SBUF, (size_t)blocks * qcap * qcap);
        P.wbuf = slot_t<double>(ctx, S_X2, (size_t)blocks * 2 * n);
        P.qcap = qcap;
        P.timing = qdiag ? slot_t<long long>(ctx, S_GN9, 28) : nullptr;
        EPC_LAUNCH(ctx, "qp_batch", qk, blocks, 32, smem, P);
        check_launch();
        std::vector<int> st(nqp);
        d2h(ctx, x, dx, nv * sizeof(double));
        d2h(ctx, lambda, dl, nl * sizeof(double));
        d2h(ctx, active_sign, ds, nl * sizeof(int));
        d2h(ctx, iters, ds + nl, (size_t)nqp * sizeof(int));
        d2h(ctx, st.data(), ds + nl + nqp, (size_t)nqp * sizeof(int));
        if (kkt) d2h(ctx, kkt, dk, (size_t)nqp * sizeof(double));
        sync(ctx);
        int first = -1;
        for (int q = 0; q < nqp; ++q) {
            // std::invalid_argument for an infeasible start, runtime_error otherwise
            status[q] = st[q] == 0 ? EPC_OK : (st[q] == 2 ? EPC_ERR_INVALID_ARGUMENT : EPC_ERR_RUNTIME);
            if (st[q] != 0 && first < 0) first = q;
        }
        if (first >= 0) ctx->last_error = qp_what(st[first]);
    });
}

int epc_residual(epc_context* ctx, const epc_grid* gg, int mem, const double* iplus,
                 const double* iminus, const double* b, double* r) {
    return guarded(ctx, [&] {
        const Geo g = make_geo(gg);
        const size_t nc = g.ncell, nf = g.nface;
        const double* ip = mem == EPC_MEM_DEVICE ? iplus : stage_in(ctx, S_IP, mem, iplus, nc);
        const double* im = mem == EPC_MEM_DEVICE ? iminus : stage_in(ctx, S_IM, mem, iminus, nc);
        double* bd = stage_in(ctx, S_B0, mem, b, nf);
        double* rd = slot_t<double>(ctx, S_TMP0, nc);
        EPC_LAUNCH(ctx, "residual", k_residual, grid1d(ctx, (long long)nc), 256, 0, ip, im, bd,
                   g.m1, g.n1, g.ncell, make_hdiv(g.h1), g.o1, rd);
        check_launch();
        stage_out(ctx, mem, r, rd, nc);
        sync(ctx);
    });
}

const char* epc_build_info(void) {
    return "libepicorr_b200 sm_100a fp64 exact (-fmad=false, IEEE div/sqrt)";
}

}  // extern "C"

#include "gn_host.inc"
#include "slab_host.inc"
#include "multilevel_host.inc"
#include "image_host.inc"
#include "admm_f32_host.inc"
#include "t2_host.inc"
#include "multi_gpu_host.inc"

