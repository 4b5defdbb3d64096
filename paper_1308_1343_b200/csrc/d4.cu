// d4.cu — the 4th-order z-streaming stencil family (K2 d4_all, K3 lap4 over
// a box table, K5 RK4 stages) for sm_100a.
//
// Reference path: the tiled loop iterator (traverse.py:130-209) calling a
// slab kernel (_update_rows, stencil.py:31-39) per fine slice.  Here one
// launch covers every tile of every box of a level:
//   * blockIdx.x -> (box, tile) through the device box table (tile prefix);
//   * a CTA owns a TX x TY tile of (x, y) columns and streams z planes
//     Z0-2 .. Z1+1 (z_chunk = Z1-Z0 output planes);
//   * one producer warp moves each plane of the tile plus its 2-point halo
//     (TX+4) x (TY+4) from HBM into a 4-stage shared-memory ring with TMA
//     (cp.async.bulk.tensor.3d), completion on mbarriers; consumer warps
//     release a stage with one arrive per warp;
//   * each consumer thread owns two adjacent x points (double2 loads and
//     stores, x tiles anchored on absolute multiples of TX so pairs are
//     16-byte aligned — the iterate_masked frame rule, vlanes.py:322-337:
//     lanes outside [lo, hi) compute but never store);
//   * in-plane terms (Dx, Dy, Dxx, Dyy, Dxy) come from shared memory; the z
//     terms (Dz, Dzz, Dxz, Dyz) from per-thread register windows of u, of
//     the unscaled x/y first differences and of Dxx+Dyy over five planes.
//
// Every expression tree and association matches oracle/stencils.py
// (SURVEY.md App. A):  d1u = (u[-2]-u[+2]) + 8*(u[+1]-u[-1]),
//   D1 = d1u*k1, D2 = ((16*(u[-1]+u[+1]) - (u[-2]+u[+2])) - 30*u)*k2,
//   D_ab = d1u_a(d1u_b)*k11 with b the inner (x for xy/xz, y for yz) axis,
//   Lap4 = (Dxx + Dyy) + Dzz.
#include <cstring>

#include "common.cuh"
#include "internal.h"

namespace sb {

namespace {

constexpr int kStages = 4;
// (tile_x/2)*tile_y limit per mode: ALL10 keeps ~36 doubles of z windows per
// thread (~140 registers), the single-output modes ~75 registers.
__host__ __device__ constexpr int max_consumers(int mode) { return mode == 0 ? 256 : 512; }

struct BoxDesc {
    CUtensorMap tmap;          // plane boxes of (TX+4) x (TY+4) x 1 over the source grid
    Grid g[10];                // mode-dependent outputs / pointwise inputs
    int tma0[3];               // TMA coordinates of interior (0,0,0)
    int lo[3], hi[3];
    int ax0;                   // x tile anchor: floor(lo.x / TX) * TX
    int ntx, nty, ntz;
    int tile_begin;
};

struct D4Params {
    BoxDesc box[SB_MAX_BOXES];
    int nbox;
    int ty, zc;
    double k1, k2, k11;
    double ca, cb;
};

template <int MODE, int TX>
__global__ void __launch_bounds__(max_consumers(MODE) + 32, 1) d4_kernel(const __grid_constant__ D4Params P) {
    constexpr int CPR = TX / 2;     // column pairs per row
    constexpr int W = TX + 4;       // smem row width (elements)
    const int TY = P.ty;
    const int H = TY + 4;
    const int ncons = CPR * TY;
    const int stage_elems = round_up(W * H, 16);

    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint64_t *empty = full + kStages;
    double *stages = reinterpret_cast<double *>(smem + 128);
    double *rxb = stages + kStages * stage_elems;   // ALL10: [2][H][TX]

    // ---- box table lookup: blockIdx.x -> (box, tile) ----
    int t = blockIdx.x;
    int b = 0;
    while (b + 1 < P.nbox && t >= P.box[b + 1].tile_begin) ++b;
    const BoxDesc &B = P.box[b];
    t -= B.tile_begin;
    const int bx = t % B.ntx;
    t /= B.ntx;
    const int by = t % B.nty;
    const int bz = t / B.nty;
    const int X0 = B.ax0 + bx * TX;
    const int Y0 = B.lo[1] + by * TY;
    const int Z0 = B.lo[2] + bz * P.zc;
    const int Z1 = min(Z0 + P.zc, B.hi[2]);
    const int nplanes = Z1 - Z0 + 4;

    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], ncons / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (tid >= ncons) {
        // ---------------- producer warp: TMA plane loads ----------------
        if (tid == ncons) {
            tma_prefetch_desc(&B.tmap);
            const uint32_t bytes = (uint32_t)(W * H * 8);
            const int cx0 = B.tma0[0] + X0 - 2, cy0 = B.tma0[1] + Y0 - 2, cz0 = B.tma0[2] + Z0 - 2;
            for (int i = 0; i < nplanes; ++i) {
                const int s = i % kStages;
                if (i >= kStages) mbar_wait(&empty[s], ((i / kStages) - 1) & 1);
                mbar_arrive_expect_tx(&full[s], bytes);
                tma_load_3d(stages + s * stage_elems, &B.tmap, cx0, cy0, cz0 + i, &full[s]);
            }
        }
        return;
    }

    // ---------------- consumer threads ----------------
    const int lane = tid & 31;
    const int cx = tid % CPR;
    const int ry = tid / CPR;
    const int x = X0 + 2 * cx;
    const int y = Y0 + ry;
    const bool yin = y < B.hi[1];
    const bool m0 = yin && x >= B.lo[0] && x < B.hi[0];
    const bool m1 = yin && x + 1 >= B.lo[0] && x + 1 < B.hi[0];
    const double k1 = P.k1, k2 = P.k2, k11 = P.k11;

    double uw[5][2], sw[3][2];
    double rxw[5][2], ryw[5][2];   // ALL10 only (dead otherwise)
#pragma unroll
    for (int k = 0; k < 5; ++k)
#pragma unroll
        for (int j = 0; j < 2; ++j) uw[k][j] = rxw[k][j] = ryw[k][j] = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) sw[k][0] = sw[k][1] = 0.0;

    for (int i = 0; i < nplanes; ++i) {
        const int s = i % kStages;
        const int z = Z0 - 2 + i;      // plane held by this stage
        const int zc = z - 2;          // plane whose z terms complete now (i >= 4)

        // pointwise operands of the RK stages for plane zc, issued before the wait
        double2 pw[5];
        if (MODE >= D4_RK1 && i >= 4) {
            const int np = (MODE == D4_RK1) ? 1 : 5;
#pragma unroll
            for (int a = 0; a < 5; ++a) {
                if (a < np) {
                    const double *q = B.g[4 + a].at(x, y, zc);
                    if (m0 && m1) pw[a] = load_pair(q);
                    else {
                        pw[a].x = m0 ? q[0] : 0.0;
                        pw[a].y = m1 ? q[1] : 0.0;
                    }
                }
            }
        }

        mbar_wait(&full[s], (i / kStages) & 1);
        const double *pl = stages + s * stage_elems;
        const double *row = pl + (ry + 2) * W + 2 * cx;   // element x-2 of row y
        const double2 a0 = load_pair(row), a1 = load_pair(row + 2), a2 = load_pair(row + 4);
        const double2 ym2 = load_pair(pl + (ry + 0) * W + 2 * cx + 2);
        const double2 ym1 = load_pair(pl + (ry + 1) * W + 2 * cx + 2);
        const double2 yp1 = load_pair(pl + (ry + 3) * W + 2 * cx + 2);
        const double2 yp2 = load_pair(pl + (ry + 4) * W + 2 * cx + 2);

        double rx[2] = {0.0, 0.0}, ryv[2] = {0.0, 0.0};
        if (MODE == D4_ALL10) {
            // x-direction unscaled first differences of this thread's halo rows
            double *rxs = rxb + (i & 1) * H * TX;
            for (int h = ry; h < 4; h += TY) {
                const int hr = h < 2 ? h : TY + h;
                const double *hrow = pl + hr * W + 2 * cx;
                const double2 b0 = load_pair(hrow), b1 = load_pair(hrow + 2), b2 = load_pair(hrow + 4);
                double2 r;
                r.x = d1u(b0.x, b0.y, b1.y, b2.x);
                r.y = d1u(b0.y, b1.x, b2.x, b2.y);
                *reinterpret_cast<double2 *>(rxs + hr * TX + 2 * cx) = r;
            }
            rx[0] = d1u(a0.x, a0.y, a1.y, a2.x);
            rx[1] = d1u(a0.y, a1.x, a2.x, a2.y);
            ryv[0] = d1u(ym2.x, ym1.x, yp1.x, yp2.x);
            ryv[1] = d1u(ym2.y, ym1.y, yp1.y, yp2.y);
            *reinterpret_cast<double2 *>(rxs + (ry + 2) * TX + 2 * cx) = make_double2(rx[0], rx[1]);
        }
        // this warp is done reading the stage
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);

        const double u0[2] = {a1.x, a1.y};
        double dxx[2], dyy[2];
        dxx[0] = d2(a0.x, a0.y, a1.x, a1.y, a2.x, k2);
        dxx[1] = d2(a0.y, a1.x, a1.y, a2.x, a2.y, k2);
        dyy[0] = d2(ym2.x, ym1.x, a1.x, yp1.x, yp2.x, k2);
        dyy[1] = d2(ym2.y, ym1.y, a1.y, yp1.y, yp2.y, k2);

        const bool in_plane = (z >= Z0) && (z < Z1);
        if (MODE == D4_ALL10) {
            named_bar(1, ncons);   // rx of all rows (incl. halo) of this plane visible
            const double *rxs = rxb + (i & 1) * H * TX + 2 * cx;
            const double2 r_m2 = load_pair(rxs + (ry + 0) * TX);
            const double2 r_m1 = load_pair(rxs + (ry + 1) * TX);
            const double2 r_p1 = load_pair(rxs + (ry + 3) * TX);
            const double2 r_p2 = load_pair(rxs + (ry + 4) * TX);
            if (in_plane) {
                const double dxy0 = mul(d1u(r_m2.x, r_m1.x, r_p1.x, r_p2.x), k11);
                const double dxy1 = mul(d1u(r_m2.y, r_m1.y, r_p1.y, r_p2.y), k11);
                store_pair(B.g[0].at(x, y, z), mul(rx[0], k1), mul(rx[1], k1), m0, m1);
                store_pair(B.g[1].at(x, y, z), mul(ryv[0], k1), mul(ryv[1], k1), m0, m1);
                store_pair(B.g[3].at(x, y, z), dxx[0], dxx[1], m0, m1);
                store_pair(B.g[4].at(x, y, z), dyy[0], dyy[1], m0, m1);
                store_pair(B.g[6].at(x, y, z), dxy0, dxy1, m0, m1);
            }
        }

        // ---- slide the z windows ----
#pragma unroll
        for (int j = 0; j < 2; ++j) {
#pragma unroll
            for (int k = 0; k < 4; ++k) uw[k][j] = uw[k + 1][j];
            uw[4][j] = u0[j];
            sw[0][j] = sw[1][j];
            sw[1][j] = sw[2][j];
            sw[2][j] = add(dxx[j], dyy[j]);
            if (MODE == D4_ALL10) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    rxw[k][j] = rxw[k + 1][j];
                    ryw[k][j] = ryw[k + 1][j];
                }
                rxw[4][j] = rx[j];
                ryw[4][j] = ryv[j];
            }
        }

        if (i < 4) continue;

        // ---- plane zc: z terms complete ----
        double dzz[2], lap[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            dzz[j] = d2(uw[0][j], uw[1][j], uw[2][j], uw[3][j], uw[4][j], k2);
            lap[j] = add(sw[0][j], dzz[j]);
        }
        if (MODE == D4_ALL10) {
            double dz[2], dxz[2], dyz[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                dz[j] = mul(d1u(uw[0][j], uw[1][j], uw[3][j], uw[4][j]), k1);
                dxz[j] = mul(d1u(rxw[0][j], rxw[1][j], rxw[3][j], rxw[4][j]), k11);
                dyz[j] = mul(d1u(ryw[0][j], ryw[1][j], ryw[3][j], ryw[4][j]), k11);
            }
            store_pair(B.g[2].at(x, y, zc), dz[0], dz[1], m0, m1);
            store_pair(B.g[5].at(x, y, zc), dzz[0], dzz[1], m0, m1);
            store_pair(B.g[7].at(x, y, zc), dxz[0], dxz[1], m0, m1);
            store_pair(B.g[8].at(x, y, zc), dyz[0], dyz[1], m0, m1);
            store_pair(B.g[9].at(x, y, zc), lap[0], lap[1], m0, m1);
        } else if (MODE == D4_LAP4) {
            store_pair(B.g[0].at(x, y, zc), lap[0], lap[1], m0, m1);
        } else if (MODE == D4_RK1) {
            // k1 = (pi0, L(phi0)); phi2 = phi0 + (dt/2) pi0; pi2 = pi0 + (dt/2) L; acc = k1
            const double c = P.ca;
            const double p0[2] = {pw[0].x, pw[0].y};
            double fo[2], po[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                fo[j] = add(uw[2][j], mul(c, p0[j]));
                po[j] = add(p0[j], mul(c, lap[j]));
            }
            store_pair(B.g[0].at(x, y, zc), fo[0], fo[1], m0, m1);
            store_pair(B.g[1].at(x, y, zc), po[0], po[1], m0, m1);
            store_pair(B.g[2].at(x, y, zc), p0[0], p0[1], m0, m1);
            store_pair(B.g[3].at(x, y, zc), lap[0], lap[1], m0, m1);
        } else {
            // pw: 0 pi_s, 1 phi0, 2 pi0, 3 acc_phi, 4 acc_pi
            const double c = P.ca;
            const double ps[2] = {pw[0].x, pw[0].y}, f0[2] = {pw[1].x, pw[1].y};
            const double p0[2] = {pw[2].x, pw[2].y}, af[2] = {pw[3].x, pw[3].y};
            const double ap[2] = {pw[4].x, pw[4].y};
            double o0[2], o1[2], o2[2], o3[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                if (MODE == D4_RK23) {
                    o0[j] = add(f0[j], mul(c, ps[j]));
                    o1[j] = add(p0[j], mul(c, lap[j]));
                    o2[j] = add(af[j], mul(2.0, ps[j]));
                    o3[j] = add(ap[j], mul(2.0, lap[j]));
                } else {
                    o0[j] = add(f0[j], mul(c, add(af[j], ps[j])));
                    o1[j] = add(p0[j], mul(c, add(ap[j], lap[j])));
                }
            }
            store_pair(B.g[0].at(x, y, zc), o0[0], o0[1], m0, m1);
            store_pair(B.g[1].at(x, y, zc), o1[0], o1[1], m0, m1);
            if (MODE == D4_RK23) {
                store_pair(B.g[2].at(x, y, zc), o2[0], o2[1], m0, m1);
                store_pair(B.g[3].at(x, y, zc), o3[0], o3[1], m0, m1);
            }
        }
    }
}

template <int MODE, int TX>
int launch_mode_tx(const D4Params &P, int nblocks, cudaStream_t st) {
    const int ncons = (TX / 2) * P.ty;
    const int threads = ncons + 32;
    const int H = P.ty + 4;
    size_t smem = 128 + (size_t)kStages * round_up((TX + 4) * H, 16) * 8;
    if (MODE == D4_ALL10) smem += (size_t)2 * H * TX * 8;
    auto fn = d4_kernel<MODE, TX>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return check_cuda(e, "cudaFuncSetAttribute(d4)");
    fn<<<nblocks, threads, smem, st>>>(P);
    return check_cuda(cudaGetLastError(), "d4_kernel launch");
}

template <int MODE>
int launch_mode(const D4Params &P, int tx, int nblocks, cudaStream_t st) {
    switch (tx) {
        case 32: return launch_mode_tx<MODE, 32>(P, nblocks, st);
        case 64: return launch_mode_tx<MODE, 64>(P, nblocks, st);
        case 128: return launch_mode_tx<MODE, 128>(P, nblocks, st);
        default: return fail(SB_USAGE, "tile_x must be 32, 64 or 128");
    }
}

}  // namespace

int launch_d4(int mode, const D4Job *jobs, int njobs, const sb_d4_constants &k, double ca, double cb,
              const sb_launch &p, cudaStream_t st) {
    if (njobs < 1 || njobs > SB_MAX_BOXES) return fail(SB_RESOURCE, "box count outside 1..SB_MAX_BOXES");
    const int TX = p.tile_x, TY = p.tile_y, ZC = p.z_chunk;
    if (TX != 32 && TX != 64 && TX != 128) return fail(SB_USAGE, "tile_x must be 32, 64 or 128");
    if (TY < 1 || ZC < 1) return fail(SB_USAGE, "tile_y and z_chunk must be positive");
    const int ncons = (TX / 2) * TY;
    if (ncons % 32 != 0 || ncons > max_consumers(mode))
        return fail(SB_USAGE, "(tile_x/2)*tile_y must be a multiple of 32 and <= 256 (d4_all) / 512 (others)");
    if (TY + 4 > 256) return fail(SB_USAGE, "tile_y + 4 exceeds the TMA box limit of 256");
    const int H = TY + 4;
    size_t smem = 128 + (size_t)kStages * round_up((TX + 4) * H, 16) * 8;
    if (mode == D4_ALL10) smem += (size_t)2 * H * TX * 8;
    if (smem > 227 * 1024) return fail(SB_RESOURCE, "tile needs more than 227 KB of shared memory");

    D4Params P;
    memset(&P, 0, sizeof(P));
    P.ty = TY;
    P.zc = ZC;
    P.k1 = k.k1;
    P.k2 = k.k2;
    P.k11 = k.k11;
    P.ca = ca;
    P.cb = cb;
    int total = 0;
    int nbox = 0;
    for (int j = 0; j < njobs; ++j) {
        const D4Job &J = jobs[j];
        const sb_space &sp = J.space;
        bool empty = false;
        for (int d = 0; d < 3; ++d) empty |= sp.hi[d] <= sp.lo[d];
        if (empty) continue;
        BoxDesc &D = P.box[nbox];
        int rc = make_tmap(&D.tmap, J.src, TX + 4, TY + 4, 1);
        if (rc) return rc;
        for (int a = 0; a < 10; ++a) D.g[a] = grid_of(J.g[a]);
        D.tma0[0] = J.src.xpad;
        D.tma0[1] = J.src.ghost;
        D.tma0[2] = J.src.ghost;
        for (int d = 0; d < 3; ++d) {
            D.lo[d] = sp.lo[d];
            D.hi[d] = sp.hi[d];
        }
        D.ax0 = (sp.lo[0] >= 0 ? sp.lo[0] / TX : -((-sp.lo[0] + TX - 1) / TX)) * TX;
        D.ntx = (sp.hi[0] - D.ax0 + TX - 1) / TX;
        D.nty = (sp.hi[1] - sp.lo[1] + TY - 1) / TY;
        D.ntz = (sp.hi[2] - sp.lo[2] + ZC - 1) / ZC;
        D.tile_begin = total;
        const long long nt = (long long)D.ntx * D.nty * D.ntz;
        if (total + nt > 0x7fffffffLL) return fail(SB_RESOURCE, "too many tiles for one launch");
        total += (int)nt;
        ++nbox;
    }
    if (nbox == 0) return SB_OK;
    P.nbox = nbox;
    switch (mode) {
        case D4_ALL10: return launch_mode<D4_ALL10>(P, TX, total, st);
        case D4_LAP4: return launch_mode<D4_LAP4>(P, TX, total, st);
        case D4_RK1: return launch_mode<D4_RK1>(P, TX, total, st);
        case D4_RK23: return launch_mode<D4_RK23>(P, TX, total, st);
        case D4_RK4: return launch_mode<D4_RK4>(P, TX, total, st);
        default: return fail(SB_USAGE, "unknown d4 mode");
    }
}

}  // namespace sb
