// kernels.h — kernel parameter blocks and launch helpers shared by api.cu.
#pragma once

#include "common.cuh"
#include <climits>

#include "model.cuh"

// ---- ADMM b-step (bstep.cu) ---------------------------------------------
// The z-step's forward axis-2 transform fused into the b-step's drain
// (bstep.cu: bstep_drain_fwd2): out = C2 x (rho V (b + u)) per k-layer, each
// layer started once its m2 columns are counted done in layer_done.
struct Fwd2Params {
    const double* A;  // C2, m2 x m2 row-major
    const double *b, *u;
    const double* rho;
    double* out;
    double V;
    long long nface;
    int n1, m2, m3, npairs;
    unsigned* layer_done;                // [npairs * m3], zeroed before the launch
    unsigned long long* tile_counter;    // zeroed before the launch
};

struct BStepParams {
    Fwd2Params fwd2;  // fwd2.layer_done == nullptr: not fused
    int m1, n1;
    long long ncol;  // columns per pair
    long long ncell, nface;
    HDiv dh;         // spacing h1 and its exact-division mode
    double o1, V, alpha;
    const double *ip, *im, *b, *z, *u;
    double* b_out;
    const double* rho;  // [npairs]
    const int* active;  // [npairs] or nullptr
    int sqp_max_iter;
    double sqp_tol_rel;
    int check_kkt, qp_cap;
    int *col_err, *col_sqp, *col_qp, *col_maxact;
    double *col_kkt, *col_fr, *col_fd;
    double *qbuf, *sbuf, *wbuf;  // per-warp scratch: q rows, Schur, {gradient, multipliers}
    int qcap;
    unsigned long long* counter;
    long long total_cols;
    long long* timing;  // optional [16]: phase cycles [0..9] (lane 0), counters [10..15]
    int cert;           // 1: decide SQP / line-search tests on certified enclosures
    unsigned long long* cta_span;  // optional [2 x grid]: %globaltimer at CTA start / exit (dev aid)
    unsigned* col_ns;   // optional: each column's duration in ns (dev aid, EPC_BSTEP_TAIL)
    float* col_sn;      // optional [2 x total]: step norms of SQP iterations 0, 1 (dev aid)
    // longest-columns-first scheduling (api.cu: the early, bulk-bound launches):
    unsigned* col_cost;  // optional [total]: each column's cycles / 16, for the next launch's order
    const int* order;    // optional [total]: the queue's n-th claim runs column order[n]
    // with order: crit[0] = n, the first n claims are columns predicted to outlast
    // the balanced makespan; crit[1 + smid] counts those running on an SM, whose
    // other warps wait instead of claiming (0 / nullptr: no reservation)
    unsigned* crit;
};
// columns by descending cost, the larger of the last two launches' (256 linear
// buckets, unordered within a bucket: columns are independent, any order
// gives the same bits)
__global__ void k_lpt_order(const unsigned* cost, const unsigned* cost2, int* order, long long total,
                            unsigned* crit, double crit_share, int max_crit, int nsm);
// DH = HPow2 | HGen (model.cuh); DIAG: phase timing / counters and the
// chained mode compiled in (diagnostic instantiation, selected by ctx->mode)
// IMG: I+/I- read from global memory through L1 instead of staged in shared
// memory (long columns: two fewer vectors per column, more resident columns)
template <class DH, bool DIAG, bool IMG = false>
__global__ void k_admm_bstep_t(BStepParams P);

struct QpBatchParams {
    int nqp, n;
    HDiv dh;
    const double *gd, *go, *c, *x0;
    int max_iter;
    double *x, *lambda;
    int *sign, *iters;
    double* kkt;
    int* status;
    double *qbuf, *sbuf, *wbuf;
    int qcap;
    long long* timing;  // optional (the instrumented instantiation): QP phase cycles
};
template <bool DIAG>
__global__ void k_qp_batch(QpBatchParams P);
size_t bstep_smem_bytes(int n1, bool img_global = false);
// Per-warp q-row scratch: qcap rows of n doubles plus CHAIN_PAD before and
// after (the chain sweeps read the pads).
__host__ __device__ inline size_t qrows_stride(int qcap, int n) {
    return (size_t)qcap * n + 2 * CHAIN_PAD;
}

// ---- dense DCT z-step (zstep.cu) ------------------------------------------
// Out[row][col] = sum_k A[row][k] * In[k][col], k ascending, unfused mul/add.
// Element (k, col) of an operand lives at k*kstride + (col/cdiv)*cstride + col%cdiv
// (+ blockIdx.z * zstride for a batch of independent volumes).
struct GemmParams {
    const double* A;  // M x K row-major
    int M, K;
    long long N;
    const double *in0, *in1;  // in1 only for the rhs prologue
    long long kstride, cdiv, cstride, zstride;
    double* out;
    // prologue: B = rho[pair] * V * (in0 + in1)
    const double* rho;
    double V;
    long long nface;  // for pair = face / nface
    // divide epilogue
    const double* lam23;
    double alpha;
    int m2, n1, m3;
    int div_axis;  // 3: row = q3, j = col / n1; 2: row = q2, k = col / n1
    // dual epilogue
    const double *bvec, *u_old, *z_old;
    double* u_new;
    double* partials;  // per CTA: 6 sums
    const int* active;
    int mfirst;  // set by the launcher: M tiles in grid x
};
enum { PRO_PLAIN = 0, PRO_RHS = 1 };
enum { EPI_STORE = 0, EPI_DIVIDE = 1, EPI_DUAL = 2 };
void launch_dct_gemm(epc_context* ctx, const char* name, const GemmParams& p, int pro, int epi,
                     int nz, int* nblocks_out);

// Sum of squared D2 / D3 differences of z (g_value, admm.cpp:275-285): per CTA
// partials [2] over faces of all pairs.
__global__ void k_zdiff_sums(const double* z, long long nface_total, int n1, int m2, int m3,
                             double ih2, double ih3, double* partials);

// Fixed-order reduction of per-block partials: out[s] = sum_b in[b*stride + s]
// for s < nsum, segment per pair (pairs x nblk_per_pair blocks).
__global__ void k_reduce_partials(const double* in, int nblk, int stride, int nsum,
                                  double* out);

// ---- per-column b-step statistics -> per pair scalars ---------------------
__global__ void k_reduce_columns(const int* col_err, const int* col_sqp, const int* col_qp,
                                 const int* col_maxact, const double* col_kkt,
                                 const double* col_fr, const double* col_fd, long long ncol,
                                 const int* active, double* out_d, long long* out_i);

// ---- element-wise helpers ---------------------------------------------------
// the reference's five sequential dual-update sums (fallback of admm_decide.h)
constexpr int SEQ_THREADS = 512;
__global__ void k_seq_sums(const double* b, const double* z, const double* zo, const double* u,
                           long long n, double* io, const int* need);
size_t seq_sums_smem();
// launches k_seq_sums (one CTA) on the context stream; io_dev: 5 doubles in/out
void run_seq_sums(epc_context* ctx, const double* b, const double* z, const double* zo,
                  const double* u, long long n, double* io_dev);
// per pair q with need[q] != 0: io[8 q .. 8 q + 4] += the five sums of pair q
void run_seq_sums_pairs(epc_context* ctx, const double* b, const double* z, const double* zo,
                        const double* u, long long n, int npairs, double* io_dev, const int* need);
__global__ void k_scale_pairs(double* u, long long nface, int npairs, const double* factor);
__global__ void k_copy_masked(const double* src, double* dst, long long nface, int npairs,
                              const int* mask);

// aux_kernels.cu
__global__ void k_residual(const double* ip, const double* im, const double* b, int m1, int n1,
                           long long ncell, HDiv dh, double o1, double* r);
__global__ void k_lagr_sums(const double* ip, const double* im, const double* b, const double* z,
                            const double* u, int m1, int n1, long long ncell, long long nface,
                            HDiv dh, double o1, double* partials);

__global__ void k_dual_standalone(const double* b, const double* zn, const double* zo,
                                  const double* uo, double* un, long long n, double* partials);

// ---- GN (gn.cu) -------------------------------------------------------------
struct GnCellArgs {
    const double *ip, *im, *b;
    int m1, n1;
    long long ncell;
    HDiv dh;
    double o1, V, beta;
    double *r, *jlo, *jhi, *dphi, *phi2;  // outputs (cells), any may be null except as needed
    double* partials;                      // per block: {r^2, (D1b)^2, phi, max|D1b|}
    long long sum_lo = 0, sum_hi = LLONG_MAX;  // cells entering the sums (k-slab halos excluded)
};
struct GnFaceArgs {
    const double *b, *r, *jlo, *jhi, *dphi, *dir;
    int m1, n1, m2, m3;
    long long nface;
    double V, alpha, beta, w1, w2, w3, ih2, ih3;
    double* grad;      // null: sums only
    double* partials;  // per block: {(D2b)^2, (D3b)^2, grad.dir}
    long long sum_lo = 0, sum_hi = LLONG_MAX;  // faces entering the sums
};
struct GnHessArgs {
    const double *jlo, *jhi, *phi2;
    int m1, n1, m2, m3, dim;
    long long nface;
    double V, wl, wp, gamma, beta, w2, w3;
    double *diag, *off, *pdiag;
};
struct GnHvArgs {
    const double *diag, *off, *z, *p_old;
    double *p_new, *y;
    int mode;  // 0: p = z, 1: p = z + beta p_old, 2: p = p_old
    double beta, w2, w3;
    int m1, n1, m2, m3;
    long long nface;
    double* partials;
    long long sum_lo = 0, sum_hi = LLONG_MAX;  // faces entering p.q
};
struct GnUpdArgs {
    double *d, *r, *z;
    const double *p, *q, *fd, *fl, *pdiag;
    double a, ma;
    int do_axpy, kind, n1;
    long long ncol;
    double* partials;  // per block {r.r, r.z}
};
// ---- device-resident PCG (pcg.cu) ---------------------------------------------
struct PcgState {
    int done, err, iters, reached, max_iters;
    unsigned int cnt;  // last-block ticket, reset by the last block
    double rz, alpha, beta, gnorm, prec0, relres, relres_prec, eta;
};
struct PcgHvArgs {
    const double *diag, *off, *z, *p_old;
    double *p_new, *q;
    double w2, w3;
    int m1, n1, m2, m3, ncol;
    double* partials;
};
struct PcgUpdArgs {
    double *d, *r, *z;
    const double *p, *q, *fd, *fl, *pdiag;
    int phase, kind, n1;
    long long ncol;
    double* partials;
    int tile_rs;  // k_pcg_update_bj: shared-memory row stride (odd, >= n1)
    int seg;      // block-Jacobi sweeps: segment length of the warp-per-column chains
                  // (5, 9 or 17; three staged arrays), 0 = thread-per-column chains
};
__global__ void k_pcg_start(const double* g, double* r, double* d, long long n, double* partials,
                            PcgState* S);
__global__ void k_pcg_hvp(PcgHvArgs A, PcgState* S);
// ws: the warp-specialised pipelined kernel (k_pcg_update_ws; pcg_ws_ok)
void launch_pcg_update_bj(epc_context* ctx, int cpw, int seg, bool ws, int blocks, size_t smem,
                          const PcgUpdArgs& U, PcgState* S);
void set_pcg_update_bj_smem(int cpw, int seg, bool ws, int bytes);
bool pcg_variant_ok(int cpw, int seg);
bool pcg_ws_ok(int cpw, int seg);
int pcg_update_bj_per_sm(int cpw, int seg, bool ws, size_t smem);  // after set_pcg_update_bj_smem
int pcg_hvp_per_sm();  // an instantiated (columns per block, segment) pair
struct PcgLoopArgs {
    PcgHvArgs H;
    PcgUpdArgs U;
    double *pbuf0, *pbuf1;     // p alternates: iteration k writes pbuf[k & 1]
    double *part_a, *part_b;   // per-block partials (p.q; r.r and r.z)
    size_t part_cap;           // doubles available in each partials buffer
    unsigned* bar;             // grid barrier counter, zeroed before the launch
};
bool launch_pcg_loop(epc_context* ctx, int cpw, int seg, size_t smem, const PcgLoopArgs& L,
                     PcgState* S);
__global__ void k_vec_differs(const double* a, const double* b, long long n, int* flag);
__global__ void k_first_error(const int* col_err, long long ncol, int* out);
__global__ void k_pcg_update(PcgUpdArgs A, PcgState* S);

__global__ void k_gn_cells(GnCellArgs A);
__global__ void k_gn_faces(GnFaceArgs A);
__global__ void k_gn_hess(GnHessArgs A);
__global__ void k_gn_factor(const double* pdiag, const double* off, double* fd, double* fl, int n1,
                            long long ncol, int* col_err);
__global__ void k_gn_hv(GnHvArgs A);
__global__ void k_gn_update_prec(GnUpdArgs A);
__global__ void k_axpy_point(const double* x, const double* d, double t, double* y, long long n);
__global__ void k_neg_norm(const double* g, double* r, long long n, double* partials);
__global__ void k_dot2(const double* a, const double* b, long long n, double* partials);
__global__ void k_gn_copy(const double* src, double* dst, long long n);

// ---- slab-distributed ADMM data movement (slab.cu) -----------------------------
__global__ void k_slab_transpose(const double* in, double* out, int n1, int m2, int mk, int world,
                                 int to_blocks);
__global__ void k_zdiff_halo(const double* last, const double* halo, long long n, double ih3,
                             double* partials);

// ---- multilevel (multilevel.cu) ------------------------------------------------
struct MlTap {
    int i0, i1;
    double w1;  // value = (1 - w1) v[i0] + w1 v[i1]  (make_taps, multilevel.cpp:135-139)
};
__global__ void k_restrict_axis(const double* in, double* out, long long pre, int mf, int mc,
                                long long post, const int* first, const int* off, const double* w);
__global__ void k_prolong(const double* in, double* out, int fn1, int fm2, int fm3, int cn1,
                          int cm2, const MlTap* t1, const MlTap* t2, const MlTap* t3);
__global__ void k_average(double* b, const double* z, long long n);

// ---- correct_pair / metrics / simulate_pair (image.cu) --------------------------
void launch_correct_pair(epc_context* ctx, const double* ip, const double* im, const double* b,
                         int m1, long long ncell, HDiv hd, double o1, double* cp, double* cm);
__global__ void k_col_absmax(const double* b, int n1, long long ncol, double* out);
void launch_simulate(epc_context* ctx, const double* truth, const double* b, const double* colmax,
                     int m1, long long ncell, HDiv hd, double o1, double tol, double* up,
                     double* um);
__global__ void k_add(double* x, const double* n, long long len);
__global__ void k_image_sums(const double* a, const double* b, long long n, int pass, double ma,
                             double mb, double* partials);
__global__ void k_swap_axes(const double* in, double* out, int d0, int d1, int d2, int a, int b);

// ---- fp32 ADMM variant (admm_f32.cu) ----------------------------------------
struct BStepF32Params {
    const float *ip, *im, *b, *z, *u;
    float* b_out;
    int m1, n1;
    long long ncol;
    float h, inv_h, o1, V, rho, alpha, sqp_tol_rel;
    int sqp_max, qp_cap, check_kkt;
    unsigned long long* counter;
    float *qscr, *sscr;  // per-CTA scratch: Schur rows (m1 x n1) and matrix (m1 x m1)
    long long qstride, sstride;
    float* col_kkt;
    double *col_sr, *col_sd;
    int* col_err;
    long long* col_work;  // sqp << 40 | qp << 16 | max_active
};
size_t bstep_f32_smem_bytes(int n1);
int bstep_f32_slots_per_sm(size_t smem);
void launch_bstep_f32(epc_context* ctx, int slots, size_t smem, const BStepF32Params& P);
void launch_reduce_f32cols(epc_context* ctx, const BStepF32Params& P, long long ncol, double* od,
                           long long* oi);
void launch_dual_f32(epc_context* ctx, int blocks, const float* b, const float* z, const float* zo,
                     const float* u, float* un, int n1, int m2, int m3, float ih2, float ih3,
                     long long n, double* part);
void launch_scale_f32(epc_context* ctx, int blocks, float* x, float a, long long n);
// fp32 DCT GEMM (admm_f32.cu): out = A (M x K) * data along one axis; the data
// element (k, n) sits at k*kstride + (n/cdiv)*cstride + n%cdiv. PRO_RHS forms
// w (in0 + in1) on load; EPI_DIVIDE divides by aV lam23[f / n1] + rV.
struct DctGemmF32 {
    const float* A;
    int M, K;
    long long N;
    const float *in0, *in1;
    float w;
    long long kstride, cdiv, cstride;
    float* out;
    const float* lam23;
    float aV, rV;
    int n1;
};
void launch_dct_gemm_f32(epc_context* ctx, const char* name, const DctGemmF32& p, int pro, int epi);
void launch_d2f(epc_context* ctx, int blocks, const double* a, float* b, long long n);

// ---- the reference's test-side helpers (operators_t2.cu) ----
void launch_avg_x1(epc_context* ctx, const double* b, int m1, long long ncell, double* out);
void launch_diff_x1(epc_context* ctx, const double* b, int m1, long long ncell, double ih,
                    double* out);
void launch_diff_x1_adjoint(epc_context* ctx, const double* r, int m1, long long nface, double ih,
                            double* out);
void launch_smoother_apply(epc_context* ctx, const double* b, int m1, int m2, int m3,
                           long long nface, double w1, double w2, double w3, double* out);
void launch_cross_diag_add(epc_context* ctx, const double* diag, int n1, int m2, int m3, int dim,
                           long long nface, double w2, double w3, double* out);
void launch_div_elem(epc_context* ctx, const double* r, const double* d, long long n, double* z);
void launch_tridiag_apply(epc_context* ctx, const double* d, const double* o, const double* x,
                          int m1, long long nface, double s, double* y);
void launch_tridiag_solve_cols(epc_context* ctx, const double* d, const double* o, double* fd,
                               double* fl, double* x, int n1, long long ncol, long long* bad);
void launch_dct_apply(epc_context* ctx, const double* z, int n1, int m2, int m3, long long nface,
                      double rv, double w2, double w3, double* out);
void launch_distance_hv(epc_context* ctx, const double* jlo, const double* jhi, const double* p,
                        int m1, long long nface, double V, double* out);
int launch_d1_absmax(epc_context* ctx, const double* b, int m1, long long ncell, double ih,
                     double* part);

// TridiagFactor::factorize with one thread per column over staged column groups (gn.cu)
void launch_gn_factor_cols(epc_context* ctx, const double* pdiag, const double* off, double* fd,
                           double* fl, int n1, long long ncol, int* col_err);
size_t gn_factor_cols_smem(int n1);
