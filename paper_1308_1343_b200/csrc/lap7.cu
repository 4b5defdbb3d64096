// lap7.cu — K1: the reference's 7-point update (stencil.py:31-39) and K0:
// the vlanes 1-D difference kernels (vlanes.py:342-360).
//
// K1 is the config-1 kernel: a 64^3 box is 4.4 MB, L2-resident, so the
// launch is latency-bound; the kernel keeps the z neighbours of its two x
// points in registers while streaming its z chunk and reads the in-plane
// neighbours through L1.  Expression tree (stencil.py:35-39):
//   dst = C0*b + C1*(((xm + xp) + (ym + yp)) + (zm + zp))
#include "common.cuh"
#include "internal.h"

namespace sb {

namespace {

__global__ void __launch_bounds__(256) lap7_kernel(Grid dst, Grid src, int lo0, int lo1, int lo2, int hi0,
                                                   int hi1, int hi2, int ax0, int zc, double c0, double c1) {
    const int x = ax0 + (blockIdx.x * 32 + threadIdx.x) * 2;
    const int y = lo1 + blockIdx.y * blockDim.y + threadIdx.y;
    const int z0 = lo2 + blockIdx.z * zc;
    const int z1 = min(z0 + zc, hi2);
    const bool yin = y < hi1;
    const bool m0 = yin && x >= lo0 && x < hi0;
    const bool m1 = yin && x + 1 >= lo0 && x + 1 < hi0;
    if (!(m0 || m1)) return;
    const int xa = m0 ? x : x + 1;   // first active point (single-point edge case)

    double zm[2], cc[2], zp[2];
    const double *pc = src.at(x, y, z0);
    if (m0 && m1) {
        const double2 a = load_pair(pc - src.sz), b = load_pair(pc);
        zm[0] = a.x; zm[1] = a.y; cc[0] = b.x; cc[1] = b.y;
    } else {
        zm[0] = zm[1] = src.at(xa, y, z0 - 1)[0];
        cc[0] = cc[1] = src.at(xa, y, z0)[0];
    }
    for (int z = z0; z < z1; ++z) {
        const double *p = src.at(x, y, z);
        double xm[2], xp[2], ym[2], yp[2];
        if (m0 && m1) {
            const double2 n = load_pair(p + src.sz);
            zp[0] = n.x; zp[1] = n.y;
            const double2 s = load_pair(p - src.sy), t = load_pair(p + src.sy);
            ym[0] = s.x; ym[1] = s.y; yp[0] = t.x; yp[1] = t.y;
            xm[0] = p[-1]; xp[0] = cc[1]; xm[1] = cc[0]; xp[1] = p[2];
        } else {
            const double *q = src.at(xa, y, z);
            zp[0] = zp[1] = q[src.sz];
            ym[0] = ym[1] = q[-src.sy];
            yp[0] = yp[1] = q[src.sy];
            xm[0] = xm[1] = q[-1];
            xp[0] = xp[1] = q[1];
        }
        double o[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const double nb = add(add(add(xm[j], xp[j]), add(ym[j], yp[j])), add(zm[j], zp[j]));
            o[j] = add(mul(c0, cc[j]), mul(c1, nb));
        }
        if (m0 && m1) store_pair(dst.at(x, y, z), o[0], o[1], true, true);
        else dst.at(xa, y, z)[0] = o[0];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            zm[j] = cc[j];
            cc[j] = zp[j];
        }
    }
}

// vlanes semantics: lane i of the grid covers index i; only lanes inside the
// iteration range store (iterate_masked + vstore_partial, vlanes.py:158-169).
__global__ void diff1d_kernel(int kind, double *dst, const double *src, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (kind == 0) {
        if (i < n - 1) dst[i] = sub(src[i + 1], src[i]);
    } else {
        if (i >= 1 && i < n - 1) dst[i] = mul(0.5, sub(src[i + 1], src[i - 1]));
    }
}

}  // namespace

int launch_lap7(const sb_array &dst, const sb_array &src, const sb_space &sp, double c0, double c1,
                const sb_launch &p, cudaStream_t st) {
    const int ty = p.tile_y > 0 ? p.tile_y : 8;
    const int zc = p.z_chunk > 0 ? p.z_chunk : 16;
    if (ty > 8 || 32 * ty > 256) return fail(SB_USAGE, "lap7: tile_y must be 1..8");
    for (int d = 0; d < 3; ++d)
        if (sp.hi[d] <= sp.lo[d]) return SB_OK;
    const int ax0 = (sp.lo[0] >= 0 ? sp.lo[0] / 2 : -((-sp.lo[0] + 1) / 2)) * 2;
    const int pairs = (sp.hi[0] - ax0 + 1) / 2;
    dim3 block(32, ty);
    dim3 grid((pairs + 31) / 32, (sp.hi[1] - sp.lo[1] + ty - 1) / ty, (sp.hi[2] - sp.lo[2] + zc - 1) / zc);
    lap7_kernel<<<grid, block, 0, st>>>(grid_of(dst), grid_of(src), sp.lo[0], sp.lo[1], sp.lo[2], sp.hi[0],
                                        sp.hi[1], sp.hi[2], ax0, zc, c0, c1);
    return check_cuda(cudaGetLastError(), "lap7_kernel launch");
}

int launch_diff1d(int kind, double *dst, const double *src, int n, cudaStream_t st) {
    if (n < 1) return SB_OK;
    const int threads = 128;
    diff1d_kernel<<<(n + threads - 1) / threads, threads, 0, st>>>(kind, dst, src, n);
    return check_cuda(cudaGetLastError(), "diff1d_kernel launch");
}

}  // namespace sb
