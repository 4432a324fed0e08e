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
