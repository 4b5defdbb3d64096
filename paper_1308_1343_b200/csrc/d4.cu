// d4.cu — the 4th-order z-streaming stencil family (K2 d4_all, K3 lap4 over
// a box table, K5 RK4 stages) for sm_100a.
//
// Reference path: the tiled loop iterator (traverse.py:130-209) calling a
// slab kernel (_update_rows, stencil.py:31-39) per fine slice.  Here one
// launch covers every tile of every box of a level:
//   * blockIdx.x -> (box, tile) through the device box table (tile prefix);
//   * a CTA owns a TX x TY tile of (x, y) columns and streams z planes
//     Z0-2 .. Z1+1 (z_chunk = Z1-Z0 output planes);
//   * each plane of the tile plus its 2-point halo, (TX+4) x (TY+4), moves
//     from HBM into a 4-stage shared-memory ring by TMA
//     (cp.async.bulk.tensor.3d) with mbarrier completion; after the one
//     CTA barrier per plane (all reads of that stage done) thread 0 re-arms
//     the stage for plane i+4 — no producer warp, no spinning; the ten-output
//     sweep loads its input with an L2 evict_last policy (the 11x larger .cs
//     output stream would otherwise push out planes other CTAs re-read);
//   * each thread owns NP (1 or 2) adjacent x points; x tiles are anchored on
//     absolute multiples of TX, so pairs are 16-byte aligned and lanes outside
//     [lo, hi) compute but never store (the iterate_masked frame rule,
//     vlanes.py:322-337);
//   * in-plane terms (Dx, Dy, Dxx, Dyy, Dxy) come from shared memory; the z
//     terms (Dz, Dzz, Dxz, Dyz, Lap) from five-slot register rings of u, of the
//     unscaled x/y first differences and of Dxx+Dyy; the plane loop is
//     unrolled five ways so ring slots are compile-time registers (no moves).
//
// Every expression tree and association matches oracle/stencils.py
// (SURVEY.md App. A):  d1u = (u[-2]-u[+2]) + 8*(u[+1]-u[-1]),
//   D1 = d1u*k1, D2 = ((16*(u[-1]+u[+1]) - (u[-2]+u[+2])) - 30*u)*k2,
//   D_ab = d1u_a(d1u_b)*k11 with b the inner (x for xy/xz, y for yz) axis,
//   Lap4 = (Dxx + Dyy) + Dzz.
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"
#include "internal.h"
#include "stencil_ops.cuh"

namespace sb {

namespace {

using namespace ops;

constexpr int kStages = 4;

// consumer threads per CTA allowed for (mode, points per thread)
__host__ __device__ constexpr bool all10(int mode) { return mode == D4_ALL10 || mode == D2_ALL10; }

// Unscaled first difference and scaled second difference of the mode's order:
// 4th: (u[-2]-u[+2]) + 8(u[+1]-u[-1]),  ((16(u[-1]+u[+1]) - (u[-2]+u[+2])) - 30u) k2
// 2nd: u[+1]-u[-1],                     ((u[-1]+u[+1]) - 2u) k2
template <int MODE>
__device__ __forceinline__ double dfirst(double m2, double m1, double p1, double p2) {
    if constexpr (MODE == D2_ALL10) return sub(p1, m1);
    else return d1u(m2, m1, p1, p2);
}
template <int MODE>
__device__ __forceinline__ double dsecond(double m2, double m1, double c, double p1, double p2, double k2) {
    if constexpr (MODE == D2_ALL10) return mul(sub(add(m1, p1), mul(2.0, c)), k2);
    else return d2(m2, m1, c, p1, p2, k2);
}

__host__ __device__ constexpr int max_threads(int mode, int np) {
    return (np == 2 && mode != D4_LAP4) ? 256 : 512;
}

// Minimum resident CTAs (of max_threads) the register allocation must allow.
#ifndef SB_D4_ALL10_MINB
#define SB_D4_ALL10_MINB 1
#endif
__host__ __device__ constexpr int min_blocks(int mode) { return all10(mode) ? SB_D4_ALL10_MINB : 1; }
// Compile-time default shapes (CTA size known exactly): resident CTAs the
// Laplacian's register allocation must allow (profiles/README.md)
#ifndef SB_D4_LAP4_MINB_T
#define SB_D4_LAP4_MINB_T 1
#endif
__host__ __device__ constexpr int lb_threads(int mode, int tx, int np, int tyc) {
    return tyc > 0 ? tx / np * tyc : max_threads(mode, np);
}
__host__ __device__ constexpr int lb_minb(int mode, int tyc) {
    return tyc > 0 && mode == D4_LAP4 ? SB_D4_LAP4_MINB_T : min_blocks(mode);
}

// One box of the launch's box table.
struct alignas(64) BoxDesc {
    CUtensorMap tmap;          // plane boxes of (TX+4) x (TY+4) x 1 over the source grid
    double *g[10];             // mode-dependent outputs / pointwise inputs (origins)
    long long sy, sz;          // strides shared by every g[] of the box
    int tma0[3];               // TMA coordinates of interior (0,0,0)
    int lo[3], hi[3];
    int ax0;                   // x tile anchor: floor(lo.x / TX) * TX
    int ntx, nty;
    int tile_begin;
};

// RK stages: TMA maps of a box's pointwise operands (TX x TY x 1 boxes at
// interior coordinates), staged next to the stencil plane.
struct alignas(64) PwDesc {
    CUtensorMap map[5];
    int tma0[5][3];
};

constexpr int kInlineBoxes = 8;

struct D4Params {
    // Box table: up to kInlineBoxes boxes travel in the parameters; larger
    // levels (and RK stages over several boxes) use a device-resident table
    // (gbox / gpw / gbegin, built once per level shape and cached by the
    // library, box_table() below) searched by binary search on tile_begin.
    BoxDesc box[kInlineBoxes];
    PwDesc pw0;                // pointwise maps of box 0 (inline table)
    const BoxDesc *gbox;       // device table, or null
    const PwDesc *gpw;         // device pointwise maps (RK modes), or null
    const int *gbegin;         // device tile_begin[nbox]
    int per[3];                // periodic extents for fused ghost stores (0 = none)
    int pghost;                // ghost width refreshed by the fused stores
    double *zlo, *zhi;         // z targets of points near the low / high face
    int zlo_dz, zhi_dz;        //   and their z shifts (periodic box: same grid, +nz / -nz)
    int nbox;
    int ty, zc;
    double k1, k2, k11;
    double ca;
};

__host__ __device__ constexpr int n_pointwise(int mode) {
    return mode == D4_RK1 ? 1 : mode == D4_RK2 ? 4 : (mode == D4_RK23 || mode == D4_RK4) ? 5 : 0;
}

template <int NP>
struct Rings {
    double u[5][NP], s[5][NP], rx[5][NP], ry[5][NP];
};

struct Ctx {
    const double *stages;
    double *rxb;
    uint64_t *full;
    int stage_elems, plane_elems, pw_elems, H, TY, nthr, tid, cx, ry;
    int X0, Y0, Z0, Z1, nplanes;
    long long off_xy;   // x + y*sy of the thread's first point
};

// Thread 0: arm stage s with plane j of the CTA's stream — the stencil plane
// (with halo) and, for the RK stages once outputs start (j >= 4), the
// pointwise operand planes of output plane Z0-4+j.
template <int MODE, int TX>
__device__ __forceinline__ void issue_plane(const Ctx &c, const PwDesc &PW, const BoxDesc &B, int j, int s) {
    constexpr int NPW = n_pointwise(MODE);
    double *st = const_cast<double *>(c.stages) + s * c.stage_elems;
    const bool with_pw = NPW > 0 && j >= 4;
    const uint32_t bytes = (uint32_t)((TX + 4) * c.H * 8 + (with_pw ? NPW * TX * c.TY * 8 : 0));
    mbar_arrive_expect_tx(&c.full[s], bytes);
    if constexpr (all10(MODE))   // ten output streams: keep the (11x smaller) input resident for its re-reads
        tma_load_3d_hint(st, &B.tmap, B.tma0[0] + c.X0 - 2, B.tma0[1] + c.Y0 - 2, B.tma0[2] + c.Z0 - 2 + j, &c.full[s],
                         l2_policy_evict_last());
    else
        tma_load_3d(st, &B.tmap, B.tma0[0] + c.X0 - 2, B.tma0[1] + c.Y0 - 2, B.tma0[2] + c.Z0 - 2 + j, &c.full[s]);
    if constexpr (NPW > 0) {
        if (with_pw) {
            const int zc = c.Z0 - 4 + j;
#pragma unroll
            for (int a = 0; a < NPW; ++a)
                tma_load_3d(st + c.plane_elems + a * c.pw_elems, &PW.map[a], PW.tma0[a][0] + c.X0,
                            PW.tma0[a][1] + c.Y0, PW.tma0[a][2] + zc, &c.full[s]);
        }
    }
}

template <int NP>
__device__ __forceinline__ void store_periodic(double *base, long long sy, long long sz, const D4Params &P, int x,
                                               int y, int z, const double (&v)[NP], const Lanes<NP> &L) {
    const int g = P.pghost;
    if (x >= g && x + NP <= P.per[0] - g && y >= g && y < P.per[1] - g && z >= g && z < P.per[2] - g) return;
#pragma unroll
    for (int j = 0; j < NP; ++j)
        if (L.m[j])
            store_images(base, sy, sz, P.per[0], P.per[1], P.per[2], g, P.zlo, P.zlo_dz, P.zhi, P.zhi_dz, x + j, y, z,
                         v[j]);
}

template <int MODE, int TX, int NP, int R>
__device__ __forceinline__ bool plane_step(int i, const Ctx &c, const D4Params &P, const BoxDesc &B,
                                           const PwDesc &PW, const Lanes<NP> &L, Rings<NP> &rg) {
    constexpr int W = TX + 4;
    if (i >= c.nplanes) return true;
    const int s = i & (kStages - 1);
    const int z = c.Z0 - 2 + i;    // plane held by this stage
    const int zc = z - 2;          // plane whose z terms complete now (i >= 4)
    const long long offc = c.off_xy + (long long)zc * B.sz;

    mbar_wait(&c.full[s], (i / kStages) & 1);
    const double *pl = c.stages + s * c.stage_elems;

    // pointwise operands of the RK stages for plane zc (TMA-staged with the plane)
    constexpr int NPW = n_pointwise(MODE);
    double pw[5][NP];
    if constexpr (NPW > 0) {
        if (i >= 4) {
#pragma unroll
            for (int a = 0; a < NPW; ++a)
                col_vals<NP>(pl + c.plane_elems + a * c.pw_elems + c.ry * TX + NP * c.cx, pw[a]);
        }
    }
    double xr[NP + 4], ym2[NP], ym1[NP], yp1[NP], yp2[NP];
    row_vals<NP>(pl + (c.ry + 2) * W + NP * c.cx, xr);
    col_vals<NP>(pl + (c.ry + 0) * W + NP * c.cx + 2, ym2);
    col_vals<NP>(pl + (c.ry + 1) * W + NP * c.cx + 2, ym1);
    col_vals<NP>(pl + (c.ry + 3) * W + NP * c.cx + 2, yp1);
    col_vals<NP>(pl + (c.ry + 4) * W + NP * c.cx + 2, yp2);

    double rx[NP], ryv[NP];
    double *rxs = c.rxb + (i & 1) * c.H * TX;
    if constexpr (all10(MODE)) {
        // unscaled x differences of this thread's share of the 4 halo rows
        for (int h = c.ry; h < 4; h += c.TY) {
            const int hr = h < 2 ? h : c.TY + h;
            double hv[NP + 4];
            row_vals<NP>(pl + hr * W + NP * c.cx, hv);
            double r[NP];
#pragma unroll
            for (int j = 0; j < NP; ++j) r[j] = dfirst<MODE>(hv[j], hv[j + 1], hv[j + 3], hv[j + 4]);
            if constexpr (NP == 2)
                *reinterpret_cast<double2 *>(rxs + hr * TX + 2 * c.cx) = make_double2(r[0], r[1]);
            else
                rxs[hr * TX + c.cx] = r[0];
        }
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            rx[j] = dfirst<MODE>(xr[j], xr[j + 1], xr[j + 3], xr[j + 4]);
            ryv[j] = dfirst<MODE>(ym2[j], ym1[j], yp1[j], yp2[j]);
        }
        if constexpr (NP == 2)
            *reinterpret_cast<double2 *>(rxs + (c.ry + 2) * TX + 2 * c.cx) = make_double2(rx[0], rx[1]);
        else
            rxs[(c.ry + 2) * TX + c.cx] = rx[0];
    }
    double dxx[NP], dyy[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) {
        dxx[j] = dsecond<MODE>(xr[j], xr[j + 1], xr[j + 2], xr[j + 3], xr[j + 4], P.k2);
        dyy[j] = dsecond<MODE>(ym2[j], ym1[j], xr[j + 2], yp1[j], yp2[j], P.k2);
        rg.u[R][j] = xr[j + 2];
        rg.s[R][j] = add(dxx[j], dyy[j]);
        if constexpr (all10(MODE)) {
            rg.rx[R][j] = rx[j];
            rg.ry[R][j] = ryv[j];
        }
    }

    // every thread is done with stage s (and rx of this plane is visible)
    named_bar(1, c.nthr);
    if (c.tid == 0 && i + kStages < c.nplanes) issue_plane<MODE, TX>(c, PW, B, i + kStages, s);

    if constexpr (all10(MODE)) {
        if (z >= c.Z0 && z < c.Z1) {
            double r_m2[NP], r_m1[NP], r_p1[NP], r_p2[NP];
            const double *rc = rxs + NP * c.cx;
            col_vals<NP>(rc + (c.ry + 0) * TX, r_m2);
            col_vals<NP>(rc + (c.ry + 1) * TX, r_m1);
            col_vals<NP>(rc + (c.ry + 3) * TX, r_p1);
            col_vals<NP>(rc + (c.ry + 4) * TX, r_p2);
            const long long off = c.off_xy + (long long)z * B.sz;
            double o[NP];
#pragma unroll
            for (int j = 0; j < NP; ++j) o[j] = mul(rx[j], P.k1);
            store<NP>(B.g[0] + off, o, L);
#pragma unroll
            for (int j = 0; j < NP; ++j) o[j] = mul(ryv[j], P.k1);
            store<NP>(B.g[1] + off, o, L);
            store<NP>(B.g[3] + off, dxx, L);
            store<NP>(B.g[4] + off, dyy, L);
#pragma unroll
            for (int j = 0; j < NP; ++j) o[j] = mul(dfirst<MODE>(r_m2[j], r_m1[j], r_p1[j], r_p2[j]), P.k11);
            store<NP>(B.g[6] + off, o, L);
        }
    }

    if (i < 4) return false;

    // ---- plane zc: ring slot of logical window position k is (R + 1 + k) % 5 ----
    constexpr int K0 = (R + 1) % 5, K1 = (R + 2) % 5, K2 = (R + 3) % 5, K3 = (R + 4) % 5, K4 = R;
    double dzz[NP], lap[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) {
        dzz[j] = dsecond<MODE>(rg.u[K0][j], rg.u[K1][j], rg.u[K2][j], rg.u[K3][j], rg.u[K4][j], P.k2);
        lap[j] = add(rg.s[K2][j], dzz[j]);
    }
    if constexpr (all10(MODE)) {
        double o[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) o[j] = mul(dfirst<MODE>(rg.u[K0][j], rg.u[K1][j], rg.u[K3][j], rg.u[K4][j]), P.k1);
        store<NP>(B.g[2] + offc, o, L);
        store<NP>(B.g[5] + offc, dzz, L);
#pragma unroll
        for (int j = 0; j < NP; ++j) o[j] = mul(dfirst<MODE>(rg.rx[K0][j], rg.rx[K1][j], rg.rx[K3][j], rg.rx[K4][j]), P.k11);
        store<NP>(B.g[7] + offc, o, L);
#pragma unroll
        for (int j = 0; j < NP; ++j) o[j] = mul(dfirst<MODE>(rg.ry[K0][j], rg.ry[K1][j], rg.ry[K3][j], rg.ry[K4][j]), P.k11);
        store<NP>(B.g[8] + offc, o, L);
        store<NP>(B.g[9] + offc, lap, L);
    } else if constexpr (MODE == D4_LAP4) {
        store<NP>(B.g[0] + offc, lap, L);
    } else if constexpr (MODE == D4_RK1) {
        // k1 = (pi0, L(phi0)); phi2 = phi0 + (dt/2) pi0; pi2 = pi0 + (dt/2) L;
        // acc_pi = L (acc_phi = k1_phi = pi0 is formed by stage 2 from pi0 itself)
        const double cc = P.ca;
        double fo[NP], po[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            fo[j] = add(rg.u[K2][j], mul(cc, pw[0][j]));
            po[j] = add(pw[0][j], mul(cc, lap[j]));
        }
        store<NP>(B.g[0] + offc, fo, L);
        if (P.per[0]) store_periodic<NP>(B.g[0], B.sy, B.sz, P, c.X0 + NP * c.cx, c.Y0 + c.ry, zc, fo, L);
        store<NP>(B.g[1] + offc, po, L);
        store<NP>(B.g[3] + offc, lap, L);
    } else if constexpr (MODE == D4_RK2) {
        // pw: 0 pi_s, 1 phi0, 2 pi0, 3 acc_pi;  acc_phi = pi0 + 2 pi_s  (= k1 + 2 k2)
        const double cc = P.ca;
        double o0[NP], o1[NP], o2[NP], o3[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            o0[j] = add(pw[1][j], mul(cc, pw[0][j]));
            o1[j] = add(pw[2][j], mul(cc, lap[j]));
            o2[j] = add(pw[2][j], mul(2.0, pw[0][j]));
            o3[j] = add(pw[3][j], mul(2.0, lap[j]));
        }
        store<NP>(B.g[0] + offc, o0, L);
        if (P.per[0]) store_periodic<NP>(B.g[0], B.sy, B.sz, P, c.X0 + NP * c.cx, c.Y0 + c.ry, zc, o0, L);
        store<NP>(B.g[1] + offc, o1, L);
        store<NP>(B.g[2] + offc, o2, L);
        store<NP>(B.g[3] + offc, o3, L);
    } else {
        // pw: 0 pi_s, 1 phi0, 2 pi0, 3 acc_phi, 4 acc_pi
        const double cc = P.ca;
        double o0[NP], o1[NP];
        if constexpr (MODE == D4_RK23) {
            double o2[NP], o3[NP];
#pragma unroll
            for (int j = 0; j < NP; ++j) {
                o0[j] = add(pw[1][j], mul(cc, pw[0][j]));
                o1[j] = add(pw[2][j], mul(cc, lap[j]));
                o2[j] = add(pw[3][j], mul(2.0, pw[0][j]));
                o3[j] = add(pw[4][j], mul(2.0, lap[j]));
            }
            store<NP>(B.g[2] + offc, o2, L);
            store<NP>(B.g[3] + offc, o3, L);
        } else {
#pragma unroll
            for (int j = 0; j < NP; ++j) {
                o0[j] = add(pw[1][j], mul(cc, add(pw[3][j], pw[0][j])));
                o1[j] = add(pw[2][j], mul(cc, add(pw[4][j], lap[j])));
            }
        }
        store<NP>(B.g[0] + offc, o0, L);
        if (P.per[0]) store_periodic<NP>(B.g[0], B.sy, B.sz, P, c.X0 + NP * c.cx, c.Y0 + c.ry, zc, o0, L);
        store<NP>(B.g[1] + offc, o1, L);
    }
    return false;
}

// TYC > 0: compile-time tile height (the default shapes), so staged-plane
// offsets fold into immediates; TYC = 0: P.ty
// GT: the box table is device-resident (P.gbox / P.gpw / P.gbegin) instead
// of inline in the parameters (whose fields the compiler reads as
// constant-bank operands, keeping them out of registers).
template <int MODE, int TX, int NP, int TYC, bool GT>
__global__ void __launch_bounds__(lb_threads(MODE, TX, NP, TYC), lb_minb(MODE, TYC))
    d4_kernel(const __grid_constant__ D4Params P) {
    pdl_launch_dependents();    // PDL: see lap7.cu
    pdl_wait_prerequisites();
    constexpr int TPR = TX / NP;    // threads per row
    constexpr int W = TX + 4;       // smem row width (elements)
    extern __shared__ __align__(1024) unsigned char smem[];

    Ctx c;
    c.TY = TYC > 0 ? TYC : P.ty;
    c.H = c.TY + 4;
    c.nthr = TPR * c.TY;
    c.plane_elems = round_up(W * c.H, 16);
    c.pw_elems = round_up(TX * c.TY, 16);
    c.stage_elems = c.plane_elems + n_pointwise(MODE) * c.pw_elems;
    c.full = reinterpret_cast<uint64_t *>(smem);
    c.stages = reinterpret_cast<const double *>(smem + 128);
    c.rxb = reinterpret_cast<double *>(smem + 128) + kStages * c.stage_elems;

    // ---- box table lookup: blockIdx.x -> (box, tile) ----
    int t = blockIdx.x;
    int b = 0;
    if constexpr (GT) {        // device table: binary search on tile_begin
        int lo = 0, hi = P.nbox - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (t >= __ldg(P.gbegin + mid)) lo = mid;
            else hi = mid - 1;
        }
        b = lo;
    } else {
        while (b + 1 < P.nbox && t >= P.box[b + 1].tile_begin) ++b;
    }
    const BoxDesc &B = GT ? P.gbox[b] : P.box[b];
    const PwDesc &PW = GT && n_pointwise(MODE) > 0 ? P.gpw[b] : P.pw0;
    t -= B.tile_begin;
    const int bx = t % B.ntx;
    t /= B.ntx;
    const int by = t % B.nty;
    const int bz = t / B.nty;
    c.X0 = B.ax0 + bx * TX;
    c.Y0 = B.lo[1] + by * c.TY;
    c.Z0 = B.lo[2] + bz * P.zc;
    c.Z1 = min(c.Z0 + P.zc, B.hi[2]);
    c.nplanes = c.Z1 - c.Z0 + 4;

    c.tid = threadIdx.x;
    c.cx = c.tid % TPR;
    c.ry = c.tid / TPR;
    const int x = c.X0 + NP * c.cx;
    const int y = c.Y0 + c.ry;
    c.off_xy = (long long)x + (long long)y * B.sy;
    Lanes<NP> L;
    const bool yin = y < B.hi[1];
#pragma unroll
    for (int j = 0; j < NP; ++j) L.m[j] = (yin && x + j >= B.lo[0] && x + j < B.hi[0]) ? 1 : 0;
    if constexpr (NP == 2) {
        L.full = L.m[0] & L.m[1];
        L.only0 = L.m[0] & (L.m[1] ^ 1);
        L.only1 = L.m[1] & (L.m[0] ^ 1);
    }

    if (c.tid == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&c.full[s], 1);
        fence_mbar_init();
        if constexpr (GT) {    // descriptors written through the generic proxy (host copy)
            tensormap_acquire(&B.tmap);
            if constexpr (n_pointwise(MODE) > 0)
                for (int a = 0; a < n_pointwise(MODE); ++a) tensormap_acquire(&PW.map[a]);
        }
        tma_prefetch_desc(&B.tmap);
        for (int i = 0; i < kStages && i < c.nplanes; ++i) issue_plane<MODE, TX>(c, PW, B, i, i);
    }
    __syncthreads();

    Rings<NP> rg;
#pragma unroll
    for (int k = 0; k < 5; ++k)
#pragma unroll
        for (int j = 0; j < NP; ++j) rg.u[k][j] = rg.s[k][j] = rg.rx[k][j] = rg.ry[k][j] = 0.0;

    for (int i = 0;; i += 5) {
        if (plane_step<MODE, TX, NP, 0>(i + 0, c, P, B, PW, L, rg)) break;
        if (plane_step<MODE, TX, NP, 1>(i + 1, c, P, B, PW, L, rg)) break;
        if (plane_step<MODE, TX, NP, 2>(i + 2, c, P, B, PW, L, rg)) break;
        if (plane_step<MODE, TX, NP, 3>(i + 3, c, P, B, PW, L, rg)) break;
        if (plane_step<MODE, TX, NP, 4>(i + 4, c, P, B, PW, L, rg)) break;
    }
}

size_t smem_bytes(int mode, int tx, int ty) {
    const int H = ty + 4;
    const int stage = round_up((tx + 4) * H, 16) + n_pointwise(mode) * round_up(tx * ty, 16);
    size_t smem = 128 + (size_t)kStages * stage * 8;
    if (all10(mode)) smem += (size_t)2 * H * tx * 8;
    return smem;
}

template <int MODE, int TX, int NP, int TYC, bool GT>
int launch_mode_gt(const D4Params &P, int nblocks, cudaStream_t st) {
    const int threads = (TX / NP) * P.ty;
    const size_t smem = smem_bytes(MODE, TX, P.ty);
    auto fn = d4_kernel<MODE, TX, NP, TYC, GT>;
    if (int rc = ensure_smem_limit((const void *)fn, 227 * 1024, "cudaFuncSetAttribute(d4)")) return rc;
    return launch_pdl(fn, dim3(nblocks), dim3(threads), smem, st, "d4_kernel launch", P);
}

template <int MODE, int TX, int NP, int TYC>
int launch_mode_ty(const D4Params &P, int nblocks, cudaStream_t st) {
    if (P.gbox) return launch_mode_gt<MODE, TX, NP, TYC, true>(P, nblocks, st);
    return launch_mode_gt<MODE, TX, NP, TYC, false>(P, nblocks, st);
}

template <int MODE, int TX, int NP>
int launch_mode_tx(const D4Params &P, int nblocks, cudaStream_t st) {
    // the swept default shapes of configs 2 and 4 (32 x 4, point pairs)
    constexpr bool kDefault = TX == 32 && NP == 2 && (MODE == D4_ALL10 || MODE == D4_LAP4);
    if constexpr (kDefault)
        if (P.ty == 4) return launch_mode_ty<MODE, TX, NP, 4>(P, nblocks, st);
    return launch_mode_ty<MODE, TX, NP, 0>(P, nblocks, st);
}

template <int MODE, int NP>
int launch_mode(const D4Params &P, int tx, int nblocks, cudaStream_t st) {
    switch (tx) {
        case 32: return launch_mode_tx<MODE, 32, NP>(P, nblocks, st);
        case 64: return launch_mode_tx<MODE, 64, NP>(P, nblocks, st);
        case 128: return launch_mode_tx<MODE, 128, NP>(P, nblocks, st);
        default: return fail(SB_USAGE, "tile_x must be 32, 64 or 128");
    }
}

template <int MODE>
int launch_np(const D4Params &P, int tx, int np, int nblocks, cudaStream_t st) {
    return np == 1 ? launch_mode<MODE, 1>(P, tx, nblocks, st) : launch_mode<MODE, 2>(P, tx, nblocks, st);
}

bool same_strides(const sb_array &a, const sb_array &b) { return a.sy == b.sy && a.sz == b.sz; }

bool empty_space(const sb_space &sp) {
    bool e = false;
    for (int d = 0; d < 3; ++d) e |= sp.hi[d] <= sp.lo[d];
    return e;
}

int n_used(int mode) { return all10(mode) ? 10 : mode == D4_LAP4 ? 1 : mode == D4_RK1 ? 5 : mode == D4_RK2 ? 8 : 9; }

// Fill one box-table entry; advances `total` (tiles before the next box).
int fill_box(BoxDesc &D, const D4Job &J, int TX, int TY, int ZC, long long &total) {
    const sb_space &sp = J.space;
    if (int rc = make_tmap(&D.tmap, J.src, TX + 4, TY + 4, 1)) return rc;
    for (int a = 0; a < 10; ++a) D.g[a] = J.g[a].origin;
    D.sy = J.g[0].sy;
    D.sz = J.g[0].sz;
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
    const int ntz = (sp.hi[2] - sp.lo[2] + ZC - 1) / ZC;
    D.tile_begin = (int)total;
    total += (long long)D.ntx * D.nty * ntz;
    if (total > 0x7fffffffLL) return fail(SB_RESOURCE, "too many tiles for one launch");
    return SB_OK;
}

int fill_pw(PwDesc &W, const D4Job &J, int npw, int TX, int TY) {
    for (int a = 0; a < npw; ++a) {
        const sb_array &A = J.g[4 + a];
        if (int rc = make_tmap(&W.map[a], A, TX, TY, 1)) return rc;
        W.tma0[a][0] = A.xpad;
        W.tma0[a][1] = A.ghost;
        W.tma0[a][2] = A.ghost;
    }
    return SB_OK;
}

// ---- device-resident box tables ------------------------------------------
// Built on the first launch of a (mode, launch shape, box list) and cached
// per device: [BoxDesc x n][PwDesc x n (RK modes)][int tile_begin x n].  The
// key is the launch's geometry (array origins, strides, extents, spaces), so
// a level swept again with the same shape reuses its table; tables are
// released by sb_release_tables.  The first launch of a shape uploads the
// table and waits for the copy (refused inside a CUDA-graph capture).
struct DevTable {
    void *buf = nullptr;
    long long total = 0;
};
std::mutex g_tab_mu;
std::map<std::pair<int, std::string>, DevTable> g_tables;
constexpr size_t kMaxTables = 4096;   // (level shape, launch shape) pairs kept per process

void put(std::string &k, const void *p, size_t n) { k.append(static_cast<const char *>(p), n); }
void put_array(std::string &k, const sb_array &a) {
    put(k, &a.origin, sizeof a.origin);
    put(k, &a.sy, sizeof a.sy);
    put(k, &a.sz, sizeof a.sz);
    const int32_t v[5] = {a.nx, a.ny, a.nz, a.ghost, a.xpad};
    put(k, v, sizeof v);
}

int box_table(int mode, const D4Job *jobs, const std::vector<int> &live, int TX, int TY, int ZC, int NP,
              cudaStream_t st, D4Params &P, long long &total_out) {
    const int npw = n_pointwise(mode), nb = (int)live.size(), nused = n_used(mode);
    int dev = 0;
    if (int rc = check_cuda(cudaGetDevice(&dev), "cudaGetDevice")) return rc;
    std::string key;
    const int32_t hdr[5] = {mode, TX, TY, ZC, NP};
    put(key, hdr, sizeof hdr);
    for (int j : live) {
        put_array(key, jobs[j].src);
        put(key, jobs[j].space.lo, sizeof jobs[j].space.lo);
        put(key, jobs[j].space.hi, sizeof jobs[j].space.hi);
        for (int a = 0; a < nused; ++a) put_array(key, jobs[j].g[a]);
    }
    const size_t box_bytes = sizeof(BoxDesc) * nb, pw_bytes = npw ? sizeof(PwDesc) * nb : 0;
    std::lock_guard<std::mutex> lock(g_tab_mu);
    auto it = g_tables.find({dev, key});
    if (it == g_tables.end()) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone)
            return fail(SB_USAGE, "box table: first launch of this level shape inside a CUDA-graph capture "
                                  "(launch it once before capturing)");
        if (g_tables.size() >= kMaxTables) {   // bound the cache: start over (waits for the device)
            if (int rc = check_cuda(cudaDeviceSynchronize(), "box table cache reset (wait)")) return rc;
            int cur = dev;
            for (auto &kv : g_tables) {
                cudaSetDevice(kv.first.first);
                cudaFree(kv.second.buf);
            }
            cudaSetDevice(cur);
            g_tables.clear();
        }
        std::vector<BoxDesc> boxes(nb);
        std::vector<PwDesc> pws(npw ? nb : 0);
        std::vector<int> begin(nb);
        long long total = 0;
        for (int i = 0; i < nb; ++i) {
            if (int rc = fill_box(boxes[i], jobs[live[i]], TX, TY, ZC, total)) return rc;
            begin[i] = boxes[i].tile_begin;
            if (npw)
                if (int rc = fill_pw(pws[i], jobs[live[i]], npw, TX, TY)) return rc;
        }
        std::vector<unsigned char> host(box_bytes + pw_bytes + sizeof(int) * nb);
        memcpy(host.data(), boxes.data(), box_bytes);
        if (npw) memcpy(host.data() + box_bytes, pws.data(), pw_bytes);
        memcpy(host.data() + box_bytes + pw_bytes, begin.data(), sizeof(int) * nb);
        DevTable t;
        if (int rc = check_cuda(cudaMalloc(&t.buf, host.size()), "box table allocation")) return rc;
        int rc = check_cuda(cudaMemcpyAsync(t.buf, host.data(), host.size(), cudaMemcpyHostToDevice, st),
                            "box table upload");
        if (!rc) rc = check_cuda(cudaStreamSynchronize(st), "box table upload (wait)");
        if (rc) {
            cudaFree(t.buf);
            return rc;
        }
        t.total = total;
        it = g_tables.emplace(std::make_pair(dev, std::move(key)), t).first;
    }
    unsigned char *b = static_cast<unsigned char *>(it->second.buf);
    P.gbox = reinterpret_cast<const BoxDesc *>(b);
    P.gpw = npw ? reinterpret_cast<const PwDesc *>(b + box_bytes) : nullptr;
    P.gbegin = reinterpret_cast<const int *>(b + box_bytes + pw_bytes);
    P.nbox = nb;
    total_out = it->second.total;
    return SB_OK;
}

}  // namespace

int release_box_tables() {
    std::lock_guard<std::mutex> lock(g_tab_mu);
    if (g_tables.empty()) return SB_OK;
    int rc = check_cuda(cudaDeviceSynchronize(), "release box tables (wait)");
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto &kv : g_tables) {
        cudaSetDevice(kv.first.first);
        cudaFree(kv.second.buf);
    }
    cudaSetDevice(cur);
    g_tables.clear();
    return rc;
}

int launch_d4(int mode, const D4Job *jobs, int njobs, const sb_d4_constants &k, double ca, const sb_launch &p,
              cudaStream_t st, const sb_zslab *zslab) {
    if (njobs < 0 || (njobs > 0 && !jobs)) return fail(SB_USAGE, "bad box job table");
    const int TX = p.tile_x, TY = p.tile_y, ZC = p.z_chunk;
    const int NP = (p.flags & SB_LAUNCH_SCALAR) ? 1 : 2;
    if (TX != 32 && TX != 64 && TX != 128) return fail(SB_USAGE, "tile_x must be 32, 64 or 128");
    if (TY < 1 || ZC < 1) return fail(SB_USAGE, "tile_y and z_chunk must be positive");
    const int threads = (TX / NP) * TY;
    if (threads % 32 != 0 || threads > max_threads(mode, NP))
        return fail(SB_USAGE, "threads per CTA ((tile_x/points per thread)*tile_y) must be a multiple of 32 and "
                              "within the mode's limit (256 for paired d4_all / RK stages, else 512)");
    if (TY + 4 > 256) return fail(SB_USAGE, "tile_y + 4 exceeds the TMA box limit of 256");
    if (smem_bytes(mode, TX, TY) > 227 * 1024) return fail(SB_RESOURCE, "tile needs more than 227 KB of shared memory");
    const int nused = n_used(mode), npw = n_pointwise(mode);

    std::vector<int> live;
    for (int j = 0; j < njobs; ++j) {
        if (empty_space(jobs[j].space)) continue;
        for (int a = 1; a < nused; ++a)
            if (!same_strides(jobs[j].g[a], jobs[j].g[0]))
                return fail(SB_USAGE, "all output / pointwise grids of one box must share row and plane strides");
        live.push_back(j);
    }
    if (live.empty()) return SB_OK;
    const bool periodic = npw > 0 && (p.flags & SB_LAUNCH_PERIODIC_GHOSTS);
    if ((periodic || zslab) && live.size() != 1)
        return fail(SB_USAGE, "periodic ghost refresh / z-slab halo stores sweep exactly one box");

    D4Params P;
    memset(&P, 0, sizeof(P));
    P.ty = TY;
    P.zc = ZC;
    P.k1 = k.k1;
    P.k2 = k.k2;
    P.k11 = k.k11;
    P.ca = ca;
    long long total = 0;
    if (live.size() <= (size_t)kInlineBoxes && (npw == 0 || live.size() == 1)) {
        for (size_t i = 0; i < live.size(); ++i)
            if (int rc = fill_box(P.box[i], jobs[live[i]], TX, TY, ZC, total)) return rc;
        if (npw)
            if (int rc = fill_pw(P.pw0, jobs[live[0]], npw, TX, TY)) return rc;
        P.nbox = (int)live.size();
    } else {
        if (int rc = box_table(mode, jobs, live, TX, TY, ZC, NP, st, P, total)) return rc;
    }
    const D4Job &J0 = jobs[live[0]];
    if (periodic) {
        const sb_array &O = J0.g[0];
        if (O.ghost < 1 || O.ghost > O.nx || O.ghost > O.ny || O.ghost > O.nz)
            return fail(SB_USAGE, "periodic ghost refresh needs 1 <= ghost <= every extent of phi_out");
        const sb_space &sp = J0.space;
        for (int d = 0; d < 3; ++d)
            if (sp.lo[d] != 0 || sp.hi[d] != (d == 0 ? O.nx : d == 1 ? O.ny : O.nz))
                return fail(SB_USAGE, "periodic ghost refresh needs the stage to sweep the whole interior");
        P.per[0] = O.nx;
        P.per[1] = O.ny;
        P.per[2] = O.nz;
        P.pghost = O.ghost;
        if (zslab) {
            P.zlo = zslab->lo_phi_out;
            P.zlo_dz = zslab->lo_dz;
            P.zhi = zslab->hi_phi_out;
            P.zhi_dz = zslab->hi_dz;
        } else {   // periodic in z within this grid
            P.zlo = P.zhi = O.origin;
            P.zlo_dz = O.nz;
            P.zhi_dz = -O.nz;
        }
    } else if (zslab) {
        return fail(SB_USAGE, "z-slab halo stores need SB_LAUNCH_PERIODIC_GHOSTS");
    }
    if (total == 0) return SB_OK;
    const int nb = (int)total;
    switch (mode) {
        case D4_ALL10: return launch_np<D4_ALL10>(P, TX, NP, nb, st);
        case D2_ALL10: return launch_np<D2_ALL10>(P, TX, NP, nb, st);
        case D4_LAP4: return launch_np<D4_LAP4>(P, TX, NP, nb, st);
        case D4_RK1: return launch_np<D4_RK1>(P, TX, NP, nb, st);
        case D4_RK23: return launch_np<D4_RK23>(P, TX, NP, nb, st);
        case D4_RK4: return launch_np<D4_RK4>(P, TX, NP, nb, st);
        case D4_RK2: return launch_np<D4_RK2>(P, TX, NP, nb, st);
        default: return fail(SB_USAGE, "unknown d4 mode");
    }
}

}  // namespace sb
