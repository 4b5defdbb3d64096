// ghost.cu — K4: periodic refill of a grid's ghost shell (config 3).
//
// The oracle fills the shell axis by axis (x, then y, then z, each over the
// full extent of the other axes; oracle/stencils.py: periodic_fill), which
// makes every ghost point equal to the interior point at its periodic image
// (wrap each coordinate into [0, n)).  This kernel writes that closed form
// directly, one thread per ghost point, in a single launch: z slabs (full
// planes, coalesced), y slabs (full rows of interior planes), x slabs (the
// g leading and g trailing elements of every interior row).  Pure copies,
// so the result is bit-exact by construction.
#include "common.cuh"
#include "internal.h"

namespace sb {

namespace {

__device__ __forceinline__ int wrap(int c, int n) { return c < 0 ? c + n : (c >= n ? c - n : c); }

__global__ void ghost_periodic_kernel(Grid a, int nx, int ny, int nz, int g, long long n_zs, long long n_ys,
                                      long long n_xs) {
    const long long total = n_zs + n_ys + n_xs;
    const int NX = nx + 2 * g, NY = ny + 2 * g;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        int x, y, z;
        if (t < n_zs) {                       // z slabs: 2g planes of NX*NY
            long long r = t;
            x = (int)(r % NX) - g;
            r /= NX;
            y = (int)(r % NY) - g;
            r /= NY;
            const int k = (int)r;             // 0..2g-1
            z = k < g ? k - g : nz + (k - g);
        } else if (t < n_zs + n_ys) {         // y slabs inside interior planes
            long long r = t - n_zs;
            x = (int)(r % NX) - g;
            r /= NX;
            const int k = (int)(r % (2 * g));
            z = (int)(r / (2 * g));
            y = k < g ? k - g : ny + (k - g);
        } else {                              // x slabs of interior rows
            long long r = t - n_zs - n_ys;
            const int k = (int)(r % (2 * g));
            r /= 2 * g;
            y = (int)(r % ny);
            z = (int)(r / ny);
            x = k < g ? k - g : nx + (k - g);
        }
        *a.at(x, y, z) = *a.at(wrap(x, nx), wrap(y, ny), wrap(z, nz));
    }
}

}  // namespace

int launch_ghost_periodic(const sb_array &a, cudaStream_t st) {
    const int g = a.ghost;
    if (g == 0) return SB_OK;
    if (g > a.nx || g > a.ny || g > a.nz) return fail(SB_USAGE, "ghost width exceeds an interior extent");
    const long long NX = a.nx + 2 * g, NY = a.ny + 2 * g;
    const long long n_zs = 2LL * g * NX * NY;
    const long long n_ys = (long long)a.nz * 2 * g * NX;
    const long long n_xs = (long long)a.nz * a.ny * 2 * g;
    const long long total = n_zs + n_ys + n_xs;
    const int threads = 256;
    long long blocks = (total + threads - 1) / threads;
    if (blocks > 148LL * 64) blocks = 148LL * 64;
    ghost_periodic_kernel<<<(unsigned)blocks, threads, 0, st>>>(grid_of(a), a.nx, a.ny, a.nz, g, n_zs, n_ys,
                                                                 n_xs);
    return check_cuda(cudaGetLastError(), "ghost_periodic_kernel launch");
}

}  // namespace sb
