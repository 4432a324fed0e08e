// slab.cu — data movement for the slab-distributed ADMM.
//
// One volume is split into k-slabs (internal axis 3): rank r owns layers
// [k0_r, k0_r + mk_r) in the reference face layout i + n1 (j + m2 kl). The
// b-step and the axis-2 DCT are local. The axis-3 DCT needs every k of a
// face row, so the z-step transposes to i-slabs (rank s owns faces
// i in [i0_s, i0_s + ni_s), all j and k, layout il + ni (j + m2 k)) and
// back (admm.cpp:445-451; operators.cpp:347-386). The i ranges follow
// shard_range (paper_1607_00531_b200/shard.py).
//
// Rank blocks. On rank r, the block bound for rank s holds that rank's i
// range of the local layers in the order [kl][j][il]. Concatenated in rank
// order, the blocks a rank receives from every sender are exactly its
// i-slab layout (the k ranges of the senders tile k in order). So the
// forward transpose is: gather into blocks, all-to-all, done; the return
// trip is: all-to-all the i-slab as is, scatter the received blocks.
#include "common.cuh"
#include "kernels.h"

namespace {
// shard_range(n, s, world) closed form and its inverse (owner of i)
__device__ __forceinline__ void split_of(int i, int n, int world, int& s, int& i0, int& ni) {
    const int base = n / world, extra = n % world;
    const int cut = extra * (base + 1);
    if (i < cut) {
        s = i / (base + 1);
        i0 = s * (base + 1);
        ni = base + 1;
    } else {
        s = extra + (i - cut) / base;
        i0 = cut + (s - extra) * base;
        ni = base;
    }
}
}  // namespace

// to_blocks = 1: slab layout -> rank blocks (gather); 0: blocks -> slab (scatter)
__global__ void k_slab_transpose(const double* __restrict__ in, double* __restrict__ out, int n1,
                                 int m2, int mk, int world, int to_blocks) {
    const long long n = (long long)n1 * m2 * mk;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e % n1);
        const long long t = e / n1;
        const int j = (int)(t % m2);
        const int kl = (int)(t / m2);
        int s, i0, ni;
        split_of(i, n1, world, s, i0, ni);
        const long long blk =
            (long long)i0 * m2 * mk + (i - i0) + (long long)ni * (j + (long long)m2 * kl);
        if (to_blocks) out[blk] = in[e];
        else out[e] = in[blk];
    }
}

// sum over one face layer of ((halo - last) / h3)^2: the D3 differences
// across a slab boundary (diff_perp, operators.cpp:70-100), block partials
__global__ void __launch_bounds__(256) k_zdiff_halo(const double* __restrict__ last,
                                                   const double* __restrict__ halo, long long n,
                                                   double ih3, double* partials) {
    __shared__ double sh[8];
    double s = 0.0;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x) {
        const double o = (halo[e] - last[e]) * ih3;
        s += o * o;
    }
    const double t = block_sum(s, sh);
    if (threadIdx.x == 0) partials[blockIdx.x] = t;
}
