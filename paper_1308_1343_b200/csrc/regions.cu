// regions.cu — F1: inter-box ghost fill of a refinement level.
//
// The schedule (which part of which box's interior feeds which box's ghost
// zone) is host-side region algebra — expand, intersect (the reference's
// bboxset operations, bboxset.py:339-385, lattice.py:156-191) — computed in
// level.ghost_schedule.  The device side is one launch over all copies of a
// schedule chunk: a CTA takes whole rows (blockIdx -> (job, row) through a
// prefix table over rows, one 32-bit divide per row), its threads walk the
// row in x, so accesses are coalesced and no per-point index arithmetic is
// paid.
#include <cstring>

#include "common.cuh"
#include "internal.h"

namespace sb {

namespace {

struct CopyDesc {
    Grid dst, src;
    int dlo[3], slo[3], ext[3];
    int row_begin;       // first row (y, z pair) of this job in the launch
};

struct CopyParams {
    CopyDesc job[SB_MAX_COPY_JOBS];
    int njobs;
    int rows;
};

__global__ void __launch_bounds__(128) copy_regions_kernel(const __grid_constant__ CopyParams P) {
    int j = 0;
    for (int row = blockIdx.x; row < P.rows; row += gridDim.x) {
        while (j + 1 < P.njobs && row >= P.job[j + 1].row_begin) ++j;   // rows ascend per CTA
        const CopyDesc &J = P.job[j];
        const int r = row - J.row_begin;
        const int y = r % J.ext[1], z = r / J.ext[1];
        double *d = J.dst.at(J.dlo[0], J.dlo[1] + y, J.dlo[2] + z);
        const double *s = J.src.at(J.slo[0], J.slo[1] + y, J.slo[2] + z);
        for (int x = threadIdx.x; x < J.ext[0]; x += blockDim.x) d[x] = s[x];
    }
}

bool inside(const sb_array &a, const int lo[3], const int ext[3], int halo) {
    const int n[3] = {a.nx, a.ny, a.nz};
    for (int d = 0; d < 3; ++d)
        if (lo[d] < -halo || lo[d] + ext[d] > n[d] + halo) return false;
    return true;
}

// Dense rows (w doubles each, rows_y rows per plane) -> padded rows of a
// grid: a CTA per row (grid-stride over rows), threads along the row.
__global__ void __launch_bounds__(256) unpack_rows_kernel(double *dst, long long sy, long long sz, int w, int rows_y,
                                                          const double *src, long long rows) {
    for (long long row = blockIdx.x; row < rows; row += gridDim.x) {
        const int y = (int)(row % rows_y);
        const long long z = row / rows_y;
        double *d = dst + y * sy + z * sz;
        const double *s = src + row * w;
        for (int c = threadIdx.x; c < w; c += blockDim.x) d[c] = s[c];
    }
}

}  // namespace

int launch_unpack_rows(double *dst, long long sy, long long sz, int w, int rows_y, const double *src, long long n,
                       cudaStream_t st) {
    if (n <= 0 || w <= 0) return SB_OK;
    const long long rows = n / w;
    const long long blocks = rows < 148LL * 16 ? rows : 148LL * 16;
    unpack_rows_kernel<<<(unsigned)blocks, 256, 0, st>>>(dst, sy, sz, w, rows_y, src, rows);
    return check_cuda(cudaGetLastError(), "unpack_rows_kernel launch");
}

int launch_copy_regions(const sb_copy_job *jobs, int njobs, cudaStream_t st) {
    if (njobs == 0) return SB_OK;
    if (njobs < 0 || njobs > SB_MAX_COPY_JOBS) return fail(SB_RESOURCE, "copy_regions: 0..SB_MAX_COPY_JOBS jobs per call");
    CopyParams P;
    memset(&P, 0, sizeof(P));
    long long rows = 0;
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
        D.row_begin = (int)rows;
        rows += (long long)J.ext[1] * J.ext[2];
        if (rows > 0x7fffffffLL) return fail(SB_RESOURCE, "copy_regions: too many rows for one launch");
    }
    if (rows == 0) return SB_OK;
    P.njobs = n;
    P.rows = (int)rows;
    const long long blocks = rows < 148LL * 16 ? rows : 148LL * 16;
    copy_regions_kernel<<<(unsigned)blocks, 128, 0, st>>>(P);
    return check_cuda(cudaGetLastError(), "copy_regions_kernel launch");
}

}  // namespace sb
