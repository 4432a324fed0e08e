// aux_kernels.cu — small kernels behind the per-step ABI entry points
// (residual, Lagrangian parts, batched column QPs).
#include "common.cuh"
#include "kernels.h"
#include "model.cuh"

// residual, objective.cpp:77-91: one thread per cell.
__global__ void k_residual(const double* ip, const double* im, const double* b, int m1, int n1,
                           long long ncell, HDiv dh, double o1, double* r) {
    const ColGeom g{m1, o1, dh};
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < ncell;
         e += (long long)gridDim.x * blockDim.x) {
        const long long c = e / m1;
        const int i = (int)(e - c * m1);
        const double* bc = b + c * n1;
        r[e] = residual_cell(ip + c * m1, im + c * m1, g, i, bc[i], bc[i + 1], nullptr, nullptr);
    }
}

// Lagrangian face/cell sums for one volume: partials per block of
// {sum r^2, sum (D1 b)^2 (x 1/h), sum u.(b-z), sum (b-z)^2}.
__global__ void __launch_bounds__(256) k_lagr_sums(const double* ip, const double* im,
                                                  const double* b, const double* z,
                                                  const double* u, int m1, int n1,
                                                  long long ncell, long long nface, HDiv dh,
                                                  double o1, double* partials) {
    __shared__ double sh[8];
    const ColGeom g{m1, o1, dh};
    const double ih = 1.0 / dh.h;
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < ncell;
         e += (long long)gridDim.x * blockDim.x) {
        const long long c = e / m1;
        const int i = (int)(e - c * m1);
        const double* bc = b + c * n1;
        const double r = residual_cell(ip + c * m1, im + c * m1, g, i, bc[i], bc[i + 1], nullptr, nullptr);
        s[0] += r * r;
        const double d = (bc[i + 1] - bc[i]) * ih;
        s[1] += d * d;
    }
    for (long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x; f < nface;
         f += (long long)gridDim.x * blockDim.x) {
        const double diff = b[f] - z[f];
        s[2] += u[f] * diff;
        s[3] += diff * diff;
    }
    for (int k = 0; k < 4; ++k) {
        const double t = block_sum(s[k], sh);
        if (threadIdx.x == 0) partials[blockIdx.x * 4 + k] = t;
        __syncthreads();
    }
}

// standalone dual update (dual_update_and_residuals, admm.cpp:453-476)
__global__ void __launch_bounds__(256) k_dual_standalone(const double* b, const double* zn,
                                                        const double* zo, const double* uo,
                                                        double* un, long long n,
                                                        double* partials) {
    __shared__ double sh[8];
    double s[6] = {0, 0, 0, 0, 0, 0};
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double diff = b[i] - zn[i];
        const double u = uo[i] + diff;
        un[i] = u;
        const double dz = zo[i] - zn[i];
        s[0] += diff * diff;
        s[1] += dz * dz;
        s[2] += b[i] * b[i];
        s[3] += zn[i] * zn[i];
        s[4] += u * u;
        s[5] += u * diff;
    }
    for (int k = 0; k < 6; ++k) {
        const double t = block_sum(s[k], sh);
        if (threadIdx.x == 0) partials[blockIdx.x * 6 + k] = t;
        __syncthreads();
    }
}

// The reference's five sequential sums of the dual update, in index order
// (admm.cpp:461-469 and norm2 = sqrt(dot), grid.cpp:60-64): io[0..4] +=
// sum (b-z)^2, sum (zo-z)^2, sum b^2, sum z^2, sum u^2 over i = 0..n-1, each
// a one-thread chain (io carries a start value, so a chain can continue
// across slabs in rank order). The fallback of the certified decisions
// (admm_decide.h): warps 1.. form the terms of the next chunk in shared
// memory (the same rounded products the reference adds) while thread 0 adds
// the current chunk. One CTA of SEQ_THREADS threads per pair; with `need`,
// CTA q sums pair q (vectors pair-major, n per pair; io + 8 q) only when
// need[q] is set (the device-side ADMM decisions, api.cu).
constexpr int SEQ_CHUNK = 1024;
__global__ void __launch_bounds__(SEQ_THREADS) k_seq_sums(const double* b, const double* z,
                                                          const double* zo, const double* u,
                                                          long long n, double* io, const int* need) {
    extern __shared__ double seq_sh[];  // [2][5][SEQ_CHUNK]
    if (need) {
        if (!need[blockIdx.x]) return;
        const long long o = (long long)blockIdx.x * n;
        b += o;
        z += o;
        zo += o;
        u += o;
        io += 8 * blockIdx.x;
    }
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0, s4 = 0.0;
    if (threadIdx.x == 0) {
        s0 = io[0];
        s1 = io[1];
        s2 = io[2];
        s3 = io[3];
        s4 = io[4];
    }
    const long long nchunk = (n + SEQ_CHUNK - 1) / SEQ_CHUNK;
    auto fill = [&](long long c, double* buf) {
        const long long base = c * SEQ_CHUNK;
        for (int t = threadIdx.x - 32; t < SEQ_CHUNK; t += blockDim.x - 32) {
            const long long i = base + t;
            if (i >= n) break;
            const double bi = b[i], zi = z[i];
            const double diff = bi - zi;
            const double dz = zo[i] - zi;
            const double ui = u[i];
            buf[t] = diff * diff;
            buf[SEQ_CHUNK + t] = dz * dz;
            buf[2 * SEQ_CHUNK + t] = bi * bi;
            buf[3 * SEQ_CHUNK + t] = zi * zi;
            buf[4 * SEQ_CHUNK + t] = ui * ui;
        }
    };
    if (threadIdx.x >= 32 && nchunk > 0) fill(0, seq_sh);
    __syncthreads();
    for (long long c = 0; c < nchunk; ++c) {
        double* cur = seq_sh + (c & 1) * 5 * SEQ_CHUNK;
        double* nxt = seq_sh + ((c + 1) & 1) * 5 * SEQ_CHUNK;
        if (threadIdx.x >= 32) {
            if (c + 1 < nchunk) fill(c + 1, nxt);
        } else if (threadIdx.x == 0) {
            const long long cnt = min((long long)SEQ_CHUNK, n - c * SEQ_CHUNK);
#pragma unroll 4
            for (int t = 0; t < (int)cnt; ++t) {
                s0 += cur[t];
                s1 += cur[SEQ_CHUNK + t];
                s2 += cur[2 * SEQ_CHUNK + t];
                s3 += cur[3 * SEQ_CHUNK + t];
                s4 += cur[4 * SEQ_CHUNK + t];
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        io[0] = s0;
        io[1] = s1;
        io[2] = s2;
        io[3] = s3;
        io[4] = s4;
    }
}
size_t seq_sums_smem() { return 2 * 5 * SEQ_CHUNK * sizeof(double); }

void run_seq_sums(epc_context* ctx, const double* b, const double* z, const double* zo,
                  const double* u, long long n, double* io_dev) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_seq_sums, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)seq_sums_smem());
        attr = true;
    }
    EPC_LAUNCH(ctx, "seq_sums", k_seq_sums, 1, SEQ_THREADS, seq_sums_smem(), b, z, zo, u, n, io_dev,
               (const int*)nullptr);
}

void run_seq_sums_pairs(epc_context* ctx, const double* b, const double* z, const double* zo,
                        const double* u, long long n, int npairs, double* io_dev, const int* need) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_seq_sums, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)seq_sums_smem());
        attr = true;
    }
    EPC_LAUNCH(ctx, "seq_sums", k_seq_sums, npairs, SEQ_THREADS, seq_sums_smem(), b, z, zo, u, n, io_dev,
               need);
}
