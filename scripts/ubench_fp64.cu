// ubench_fp64.cu — dependent-chain latency of fp64 ops on one lane (dev aid).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false ubench_fp64.cu -o ubench
#include <cstdio>
#include <cuda_runtime.h>

#define N 4096

__global__ void k(const double* in, double* out, long long* cyc) {
    __shared__ double sm[N];
    for (int i = threadIdx.x; i < N; i += blockDim.x) sm[i] = in[i];
    __syncthreads();
    if (threadIdx.x != 0) return;
    double a = in[0], b = in[1], c = in[2];
    long long t0, t1;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) a = a + b;
    t1 = clock64();
    cyc[0] = t1 - t0;
    // DMUL chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) a = a * c;
    t1 = clock64();
    cyc[1] = t1 - t0;
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) a = __fma_rn(a, c, b);
    t1 = clock64();
    cyc[2] = t1 - t0;
    // DDIV dependent chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) a = b / a;
    t1 = clock64();
    cyc[3] = t1 - t0;
    // DDIV independent (results summed)
    double s = 0.0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) s = s + sm[i] / c;
    t1 = clock64();
    cyc[4] = t1 - t0;
    // mul+sub chain with smem operand (Thomas forward sweep)
    double p = a;
    t0 = clock64();
    for (int i = 1; i < N; ++i) p = sm[i] - sm[i - 1] * p;
    t1 = clock64();
    cyc[5] = t1 - t0;
    // dependent LDS pointer-chase-ish: add of smem values (sum chain)
    double q = 0.0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) q = q + sm[i];
    t1 = clock64();
    cyc[6] = t1 - t0;
    // sqrt chain
    double r = in[3];
    t0 = clock64();
    for (int i = 0; i < N; ++i) r = sqrt(r + 1.0);
    t1 = clock64();
    cyc[7] = t1 - t0;
    // reciprocal approx + 2 newton + correction (branchless division)
    double d = in[4], num = in[5];
    t0 = clock64();
    for (int i = 0; i < N; ++i) {
        double y;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
        double e = __fma_rn(-d, y, 1.0);
        y = __fma_rn(y, e, y);
        e = __fma_rn(-d, y, 1.0);
        y = __fma_rn(y, e, y);
        double qq = num * y;
        double rr = __fma_rn(-d, qq, num);
        d = __fma_rn(rr, y, qq) + 1.0;
    }
    t1 = clock64();
    cyc[8] = t1 - t0;
    // generic-pointer chain through smem (same as LD via generic address)
    const double* gp = sm;
    double g = 0.0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) g = g + gp[i];
    t1 = clock64();
    cyc[9] = t1 - t0;
    out[0] = a + s + p + q + r + d + g;
}

int main() {
    double h[N];
    for (int i = 0; i < N; ++i) h[i] = 1.0 + 1e-3 * (i % 7);
    double *din, *dout;
    long long* dc;
    cudaMalloc(&din, sizeof h);
    cudaMalloc(&dout, 64);
    cudaMalloc(&dc, 16 * sizeof(long long));
    cudaMemcpy(din, h, sizeof h, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(din, dout, dc);
    k<<<1, 32>>>(din, dout, dc);
    long long c[16];
    cudaMemcpy(c, dc, sizeof c, cudaMemcpyDeviceToHost);
    const char* names[] = {"dadd chain", "dmul chain", "dfma chain", "ddiv chain", "ddiv indep+add",
                           "thomas mul-sub (smem)", "sum chain (smem)", "sqrt chain",
                           "rcp+newton div chain", "sum chain (generic ptr)"};
    for (int i = 0; i < 10; ++i) printf("%-26s %8.1f cycles/op\n", names[i], (double)c[i] / N);
    return 0;
}
