// regions.cu — F1: inter-box ghost fill of a refinement level.
//
// The schedule (which part of which box's interior feeds which box's ghost
// zone) is host-side region algebra — expand, intersect (the reference's
// bboxset operations, bboxset.py:339-385, lattice.py:156-191) — computed in
// level.ghost_schedule.  The device side is one launch over all copies of a
// schedule chunk: blockIdx -> (job, block of points) through a prefix table,
// one thread per point, x fastest so rows are coalesced.
#include <cstring>

#include "common.cuh"
#include "internal.h"

namespace sb {

namespace {

struct CopyDesc {
    Grid dst, src;
    int dlo[3], slo[3], ext[3];
    long long begin;     // first linear point index of this job
};

struct CopyParams {
    CopyDesc job[SB_MAX_COPY_JOBS];
    int njobs;
    long long total;
};

__global__ void copy_regions_kernel(const __grid_constant__ CopyParams P) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < P.total;
         t += (long long)gridDim.x * blockDim.x) {
        int j = 0;
        while (j + 1 < P.njobs && t >= P.job[j + 1].begin) ++j;
        const CopyDesc &J = P.job[j];
        long long r = t - J.begin;
        const int x = (int)(r % J.ext[0]);
        r /= J.ext[0];
        const int y = (int)(r % J.ext[1]);
        const int z = (int)(r / J.ext[1]);
        *J.dst.at(J.dlo[0] + x, J.dlo[1] + y, J.dlo[2] + z) = *J.src.at(J.slo[0] + x, J.slo[1] + y, J.slo[2] + z);
    }
}

bool inside(const sb_array &a, const int lo[3], const int ext[3], int halo) {
    const int n[3] = {a.nx, a.ny, a.nz};
    for (int d = 0; d < 3; ++d)
        if (lo[d] < -halo || lo[d] + ext[d] > n[d] + halo) return false;
    return true;
}

// Dense rows (w doubles each, rows_y rows per plane) -> padded rows of a grid.
__global__ void unpack_rows_kernel(double *dst, long long sy, long long sz, int w, int rows_y, const double *src,
                                   long long n) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
        const long long row = t / w;
        const int col = (int)(t - row * w);
        const int y = (int)(row % rows_y);
        const long long z = row / rows_y;
        dst[col + y * sy + z * sz] = src[t];
    }
}

}  // namespace

int launch_unpack_rows(double *dst, long long sy, long long sz, int w, int rows_y, const double *src, long long n,
                       cudaStream_t st) {
    if (n <= 0) return SB_OK;
    const int threads = 256;
    long long blocks = (n + threads - 1) / threads;
    if (blocks > 148LL * 32) blocks = 148LL * 32;
    unpack_rows_kernel<<<(unsigned)blocks, threads, 0, st>>>(dst, sy, sz, w, rows_y, src, n);
    return check_cuda(cudaGetLastError(), "unpack_rows_kernel launch");
}

int launch_copy_regions(const sb_copy_job *jobs, int njobs, cudaStream_t st) {
    if (njobs == 0) return SB_OK;
    if (njobs < 0 || njobs > SB_MAX_COPY_JOBS) return fail(SB_RESOURCE, "copy_regions: 0..SB_MAX_COPY_JOBS jobs per call");
    CopyParams P;
    memset(&P, 0, sizeof(P));
    long long total = 0;
    int n = 0;
    for (int j = 0; j < njobs; ++j) {
        const sb_copy_job &J = jobs[j];
        if (J.ext[0] <= 0 || J.ext[1] <= 0 || J.ext[2] <= 0) continue;
        if (!inside(J.dst, J.dst_lo, J.ext, J.dst.ghost) || !inside(J.src, J.src_lo, J.ext, J.src.ghost))
            return fail(SB_USAGE, "copy_regions: region outside a grid's interior + ghost zone");
        CopyDesc &D = P.job[n++];
        D.dst = grid_of(J.dst);
        D.src = grid_of(J.src);
        for (int d = 0; d < 3; ++d) {
            D.dlo[d] = J.dst_lo[d];
            D.slo[d] = J.src_lo[d];
            D.ext[d] = J.ext[d];
        }
        D.begin = total;
        total += (long long)J.ext[0] * J.ext[1] * J.ext[2];
    }
    if (total == 0) return SB_OK;
    P.njobs = n;
    P.total = total;
    const int threads = 256;
    long long blocks = (total + threads - 1) / threads;
    if (blocks > 148LL * 32) blocks = 148LL * 32;
    copy_regions_kernel<<<(unsigned)blocks, threads, 0, st>>>(P);
    return check_cuda(cudaGetLastError(), "copy_regions_kernel launch");
}

}  // namespace sb
