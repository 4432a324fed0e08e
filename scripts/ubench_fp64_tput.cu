// fp64 pipe throughput on sm_100a (dev aid): independent DADD / DMUL / DFMA
// streams, 8 chains per thread, enough warps to saturate; reports ops/clk/SM
// and the device-wide rate at the measured clock.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(double* out, int iters, double s) {
    double a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-9 + j;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (OP == 0) a[j] = a[j] + s;
            else if (OP == 1) a[j] = a[j] * s;
            else a[j] = fma(a[j], s, 1e-9);
        }
    }
    double t = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) t += a[j];
    if (t == 12345.0) out[0] = t;
}

template <int OP>
void run(const char* name, int sms) {
    double* out;
    cudaMalloc(&out, 8);
    const int iters = 1 << 14, threads = 256, blocks = sms * 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<OP><<<blocks, threads>>>(out, 16, 1.0000001);
    cudaEventRecord(e0);
    k<OP><<<blocks, threads>>>(out, iters, 1.0000001);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double ops = (double)blocks * threads * iters * 8;
    const double rate = ops / (ms * 1e-3);
    printf("%-5s %.2f Tops/s  (%.1f ops/clk/SM at %d MHz nominal)\n", name, rate / 1e12,
           rate / (sms * clk * 1e3), clk / 1000);
    cudaFree(out);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0>("dadd", sms);
    run<1>("dmul", sms);
    run<2>("dfma", sms);
    return 0;
}
