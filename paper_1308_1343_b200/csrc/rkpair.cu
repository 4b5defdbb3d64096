// rkpair.cu — K5b: classical RK4 for d/dt(phi, pi) = (pi, Lap4 phi) with the
// stages fused in pairs (temporal blocking), two launches per step.
//
// The RK right-hand side only differentiates phi, and each stage's phi is a
// pointwise combination of phi0 and the previous pi:
//     phi2 = phi0 + (dt/2) pi0,   phi4 = phi0 + dt pi3.
// So stage 2's Laplacian of phi2 needs only phi0 and pi0 within the stencil
// radius, and stage 4's Laplacian of phi4 only phi0 and pi3 — the ghost width
// of 2 suffices and no intermediate phi ever has to reach HBM:
//   pair A (stages 1+2): reads phi0, pi0 (with halo);
//                        writes phi3, pi3, acc_phi = pi0 + 2 pi2, acc_pi = L1 + 2 L2;
//   pair B (stages 3+4): reads phi3, phi0, pi3 (with halo), pi0, acc_phi, acc_pi;
//                        writes phi', pi'.
// 14 array passes per step instead of 32 for four separate stage sweeps.
//
// The Laplacian pairs (PAIR_LA / PAIR_LB) go further: every stage quantity is
// a pointwise function of phi0, pi0 and the stage Laplacians, and
//     phi3 = phi0 + (dt/2)(pi0 + (dt/2) L1),   phi4 = phi0 + dt (pi0 + (dt/2) L2),
// so it is enough to store L1 and L2 (with their periodic ghosts):
//   pair LA (stages 1+2): reads phi0, pi0 (with halo); writes L1, L2;
//   pair LB (stages 3+4): reads phi0, pi0, L1, L2 (with halo); forms phi3 and
//                         phi4 on the stencil neighbourhood, their Laplacians
//                         L3, L4, and writes phi', pi'.
// 10 array passes per step; the derived values repeat the stage formulas
// operation for operation, so the bits are again those of the stage path.
// Every value is produced by exactly the expression tree the per-stage
// kernels (d4.cu, mode RK1/RK2/RK23/RK4) and the oracle (oracle/stencils.py:
// rk4_step) use — the derived phi2 / phi4 are formed in registers from the
// staged planes with the same single rounding per operation — so the results
// are bit-identical to the four-stage path.
//
// Structure as in d4.cu: a CTA owns a TX x TY column tile and streams z; every
// plane of the halo inputs ((TX+4) x (TY+4)) and, once outputs start, the
// tile planes of the pointwise inputs arrive by TMA in a 4-stage ring; z
// terms come from five-slot register rings (loop unrolled five ways); the
// producing stores also refresh the periodic ghost images of phi and pi.
#include <cstring>

#include "common.cuh"
#include "internal.h"
#include "stencil_ops.cuh"

namespace sb {

namespace {

using namespace ops;

constexpr int kStages = 4;
// CTA barrier (stage release) after every plane (1) or every second plane
// (2: both stages consumed since the last barrier are re-armed together)
#ifndef SB_RKPAIR_BARRIER_EVERY
#define SB_RKPAIR_BARRIER_EVERY 2
#endif
enum { PAIR_A = 0, PAIR_B = 1, PAIR_LA = 2, PAIR_LB = 3 };
// Laplacian pairs, experiment (off): form the derived stage fields (LA: phi2;
// LB: phi3, phi4) ONCE per staged point, one plane ahead, into a two-plane
// shared ring, instead of re-forming them on every thread's 9-value stencil
// neighbourhood (each staged value is combined by up to 9 threads).  The
// pre-pass of plane i+1 runs in iteration i before its CTA barrier, so
// iteration i+1 reads it after that barrier — no extra barrier, but one per
// plane.  Same bits; 11-13 % SLOWER (1.49-1.50 vs 1.32-1.37 ms per 384^3
// step, three interleaved rounds, profiles/r02/c3_prepass_ab.log): the
// per-plane barrier and the wait for the next plane's TMA stage serialise the
// pipeline, and pair LB hits the register cap of four resident CTAs (spills).
#ifndef SB_RKPAIR_PREPASS
#define SB_RKPAIR_PREPASS 0
#endif
__host__ __device__ constexpr bool prepass(int pair) { return SB_RKPAIR_PREPASS && (pair == PAIR_LA || pair == PAIR_LB); }
__host__ __device__ constexpr int n_derived(int pair) { return !prepass(pair) ? 0 : pair == PAIR_LA ? 1 : 2; }

__host__ __device__ constexpr int n_halo(int pair) { return pair == PAIR_A || pair == PAIR_LA ? 2 : pair == PAIR_B ? 3 : 4; }
__host__ __device__ constexpr int n_out(int pair) { return pair == PAIR_A ? 4 : 2; }
__host__ __device__ constexpr int n_tile(int pair) { return pair == PAIR_B ? 3 : 0; }
__host__ __device__ constexpr int max_threads_pair(int np) { return np == 2 ? 256 : 512; }
#ifndef SB_RKPAIR_MINB
#define SB_RKPAIR_MINB 1
#endif
// Resident CTAs the register allocation must allow for the compile-time
// default shape (exact CTA size known): first pairs (A, LA) / second pairs
// (B, LB).  Register-cap experiments: profiles/README.md.
#ifndef SB_RKPAIR_MINB_FIRST
#define SB_RKPAIR_MINB_FIRST 5
#endif
#ifndef SB_RKPAIR_MINB_SECOND
#define SB_RKPAIR_MINB_SECOND 4
#endif
__host__ __device__ constexpr int lb_threads(int tx, int np, int tyc) {
    return tyc > 0 ? tx / np * tyc : max_threads_pair(np);
}
__host__ __device__ constexpr int lb_minb(int pair, int tyc) {
    return tyc == 0 ? SB_RKPAIR_MINB : (pair == 0 || pair == 2) ? SB_RKPAIR_MINB_FIRST : SB_RKPAIR_MINB_SECOND;
}

struct PairParams {
    CUtensorMap hmap[4];       // (TX+4) x (TY+4) x 1 boxes: A: phi0, pi0   B: phi3, phi0, pi3
                               //                            LA: phi0, pi0  LB: phi0, pi0, L1, L2
    CUtensorMap tmap[3];       // TX x TY x 1 boxes:         B: pi0, acc_phi, acc_pi
    int htma0[4][3], ttma0[3][3];
    double *out[4];            // A: phi3, pi3, acc_phi, acc_pi   B, LB: phi', pi'   LA: L1, L2
    long long sy, sz;          // strides shared by the outputs
    int lo[3], hi[3];
    int ax0, ntx, nty, ty, zc;
    double k2, hdt, dt, dt6;
    int per[3], pghost;        // periodic extents (0: no ghost refresh) and ghost width
    double *zlo[2], *zhi[2];   // z-image targets of out[0] / out[1] (periodic box: the outputs themselves)
    int zlo_dz[2], zhi_dz[2];
};

struct PCtx {
    const double *stages;
    double *derived;   // [2][n_derived][plane_elems] (pre-pass pairs)
    uint64_t *full;
    int plane_elems, tile_elems, stage_elems, H, TY, nthr, tid, cx, ry;
    int X0, Y0, Z0, Z1, nplanes;
    long long off_xy;
    bool xy_edge;   // periodic refresh: the thread's points lie within pghost of an x or y face
};

template <int NP>
struct PRings {
    double ua[5][NP], sa[5][NP];   // A: phi0       B: phi3   (value, Dxx + Dyy)
    double ub[5][NP], sb[5][NP];   // A: phi2       B: phi4
    double c1[5][NP];              // A: pi0        B: phi0   (centre values)
    double c2[5][NP];              //               B: pi3    LB: pi0
    double c3[5][NP], c4[5][NP];   //                         LB: L1, L2
    double *o[4];                  // the thread's output addresses in the current plane
};

template <int PAIR, int TX>
__device__ __forceinline__ void issue(const PCtx &c, const PairParams &P, int j, int s) {
    constexpr int NH = n_halo(PAIR), NT = n_tile(PAIR);
    double *st = const_cast<double *>(c.stages) + s * c.stage_elems;
    const bool with_tile = NT > 0 && j >= 4;
    const uint32_t bytes = (uint32_t)(NH * (TX + 4) * c.H * 8 + (with_tile ? NT * TX * c.TY * 8 : 0));
    mbar_arrive_expect_tx(&c.full[s], bytes);
#pragma unroll
    for (int h = 0; h < NH; ++h)
        tma_load_3d(st + h * c.plane_elems, &P.hmap[h], P.htma0[h][0] + c.X0 - 2, P.htma0[h][1] + c.Y0 - 2,
                    P.htma0[h][2] + c.Z0 - 2 + j, &c.full[s]);
    if constexpr (NT > 0) {
        if (with_tile) {
            const int zc = c.Z0 - 4 + j;
#pragma unroll
            for (int t = 0; t < NT; ++t)
                tma_load_3d(st + NH * c.plane_elems + t * c.tile_elems, &P.tmap[t], P.ttma0[t][0] + c.X0,
                            P.ttma0[t][1] + c.Y0, P.ttma0[t][2] + zc, &c.full[s]);
        }
    }
}

// The thread's stencil neighbourhood in one staged plane: row x-2..x+NP+1
// and the y neighbours y-2, y-1, y+1, y+2 of its NP points.
template <int TX, int NP>
struct Nbhd {
    double xr[NP + 4], ym2[NP], ym1[NP], yp1[NP], yp2[NP];
    __device__ __forceinline__ void load(const double *pl, int ry, int cx) {
        constexpr int W = TX + 4;
        row_vals<NP>(pl + (ry + 2) * W + NP * cx, xr);
        col_vals<NP>(pl + (ry + 0) * W + NP * cx + 2, ym2);
        col_vals<NP>(pl + (ry + 1) * W + NP * cx + 2, ym1);
        col_vals<NP>(pl + (ry + 3) * W + NP * cx + 2, yp1);
        col_vals<NP>(pl + (ry + 4) * W + NP * cx + 2, yp2);
    }
    // this = a + c * b, elementwise (the derived stage field phi0 + c pi)
    __device__ __forceinline__ void combine(const Nbhd &a, double cc, const Nbhd &b) {
#pragma unroll
        for (int k = 0; k < NP + 4; ++k) xr[k] = add(a.xr[k], mul(cc, b.xr[k]));
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            ym2[j] = add(a.ym2[j], mul(cc, b.ym2[j]));
            ym1[j] = add(a.ym1[j], mul(cc, b.ym1[j]));
            yp1[j] = add(a.yp1[j], mul(cc, b.yp1[j]));
            yp2[j] = add(a.yp2[j], mul(cc, b.yp2[j]));
        }
    }
    // Dxx + Dyy at the thread's points
    __device__ __forceinline__ void lap_xy(double k2, double (&s)[NP]) const {
#pragma unroll
        for (int j = 0; j < NP; ++j)
            s[j] = add(d2(xr[j], xr[j + 1], xr[j + 2], xr[j + 3], xr[j + 4], k2),
                       d2(ym2[j], ym1[j], xr[j + 2], yp1[j], yp2[j], k2));
    }
};

// store v at off; points within pghost of a periodic face (edge: hoisted
// per thread in x/y, per plane in z) also write their ghost images
// (output k = 0 / 1: the x/y images stay in out[k], the z images go to
// zlo[k] / zhi[k] — out[k] itself for a periodic box, the neighbouring
// slabs' grids for a z-slab decomposition)
template <int NP>
__device__ __forceinline__ void out_periodic(const PairParams &P, int k, double *at, bool edge, int x, int y, int z,
                                             const double (&v)[NP], const Lanes<NP> &L) {
    store<NP>(at, v, L);
    if (!edge) return;
#pragma unroll
    for (int j = 0; j < NP; ++j)
        if (L.m[j])
            store_images(P.out[k], P.sy, P.sz, P.per[0], P.per[1], P.per[2], P.pghost, P.zlo[k], P.zlo_dz[k],
                         P.zhi[k], P.zhi_dz[k], x + j, y, z, v[j]);
}

// The derived stage fields of staged plane j, every point of the halo plane
// once (same single-rounding trees as Nbhd::combine):
//   LA: phi2 = phi0 + (dt/2) pi0
//   LB: phi3 = phi0 + (dt/2)(pi0 + (dt/2) L1),  phi4 = phi0 + dt (pi0 + (dt/2) L2)
template <int PAIR, int TX>
__device__ __forceinline__ void derive_plane(const PCtx &c, const PairParams &P, int j) {
    const double *pl = c.stages + (j & (kStages - 1)) * c.stage_elems;
    double *db = c.derived + (j & 1) * n_derived(PAIR) * c.plane_elems;
    const int n = (TX + 4) * c.H;
#pragma unroll 1
    for (int e = c.tid; e < n; e += c.nthr) {
        const double f0 = pl[e], q0 = pl[c.plane_elems + e];
        if constexpr (PAIR == PAIR_LA) {
            db[e] = add(f0, mul(P.hdt, q0));
        } else {
            const double l1 = pl[2 * c.plane_elems + e], l2 = pl[3 * c.plane_elems + e];
            db[e] = add(f0, mul(P.hdt, add(q0, mul(P.hdt, l1))));
            db[c.plane_elems + e] = add(f0, mul(P.dt, add(q0, mul(P.hdt, l2))));
        }
    }
}

template <int PAIR, int TX, int NP, int R>
__device__ __forceinline__ bool pair_plane(int i, const PCtx &c, const PairParams &P, const Lanes<NP> &L,
                                           PRings<NP> &rg) {
    constexpr int NH = n_halo(PAIR);
    if (i >= c.nplanes) return true;
    const int s = i & (kStages - 1);
    const int z = c.Z0 - 2 + i;
    const int zc = z - 2;
    mbar_wait(&c.full[s], (i / kStages) & 1);
    const double *pl = c.stages + s * c.stage_elems;

    double tv[3][NP];   // B: pi0, acc_phi, acc_pi at the thread's points of plane zc
    if constexpr (prepass(PAIR)) {
        // derived fields of the next plane (read after this iteration's barrier)
        if (i + 1 < c.nplanes) {
            mbar_wait(&c.full[(i + 1) & (kStages - 1)], ((i + 1) / kStages) & 1);
            derive_plane<PAIR, TX>(c, P, i + 1);
        }
        const double *db = c.derived + (i & 1) * n_derived(PAIR) * c.plane_elems;
        constexpr int W = TX + 4;
        const int ctr = (c.ry + 2) * W + NP * c.cx + 2;   // the thread's points in a staged plane
        if constexpr (PAIR == PAIR_LB) {
            Nbhd<TX, NP> d;
            double s3[NP], s4[NP], f0[NP], q0[NP], l1[NP], l2[NP];
            d.load(db, c.ry, c.cx);
            d.lap_xy(P.k2, s3);
#pragma unroll
            for (int j = 0; j < NP; ++j) {
                rg.ua[R][j] = d.xr[j + 2];
                rg.sa[R][j] = s3[j];
            }
            d.load(db + c.plane_elems, c.ry, c.cx);
            d.lap_xy(P.k2, s4);
            col_vals<NP>(pl + ctr, f0);
            col_vals<NP>(pl + c.plane_elems + ctr, q0);
            col_vals<NP>(pl + 2 * c.plane_elems + ctr, l1);
            col_vals<NP>(pl + 3 * c.plane_elems + ctr, l2);
#pragma unroll
            for (int j = 0; j < NP; ++j) {
                rg.ub[R][j] = d.xr[j + 2];
                rg.sb[R][j] = s4[j];
                rg.c1[R][j] = f0[j];
                rg.c2[R][j] = q0[j];
                rg.c3[R][j] = l1[j];
                rg.c4[R][j] = l2[j];
            }
        } else {   // PAIR_LA
            Nbhd<TX, NP> a;
            double sa[NP], sb2[NP];
            a.load(pl, c.ry, c.cx);
            a.lap_xy(P.k2, sa);
#pragma unroll
            for (int j = 0; j < NP; ++j) {
                rg.ua[R][j] = a.xr[j + 2];
                rg.sa[R][j] = sa[j];
            }
            a.load(db, c.ry, c.cx);
            a.lap_xy(P.k2, sb2);
#pragma unroll
            for (int j = 0; j < NP; ++j) {
                rg.ub[R][j] = a.xr[j + 2];
                rg.sb[R][j] = sb2[j];
            }
        }
    } else if constexpr (PAIR == PAIR_LB) {
        // phi3 = phi0 + (dt/2) pi2, pi2 = pi0 + (dt/2) L1;  phi4 = phi0 + dt pi3, pi3 = pi0 + (dt/2) L2
        Nbhd<TX, NP> f0, q0, l, p, d;
        f0.load(pl, c.ry, c.cx);
        q0.load(pl + c.plane_elems, c.ry, c.cx);
        l.load(pl + 2 * c.plane_elems, c.ry, c.cx);
        double s3[NP], s4[NP];
        p.combine(q0, P.hdt, l);
        d.combine(f0, P.hdt, p);
        d.lap_xy(P.k2, s3);
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            rg.ua[R][j] = d.xr[j + 2];
            rg.sa[R][j] = s3[j];
            rg.c3[R][j] = l.xr[j + 2];
        }
        l.load(pl + 3 * c.plane_elems, c.ry, c.cx);
        p.combine(q0, P.hdt, l);
        d.combine(f0, P.dt, p);
        d.lap_xy(P.k2, s4);
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            rg.ub[R][j] = d.xr[j + 2];
            rg.sb[R][j] = s4[j];
            rg.c4[R][j] = l.xr[j + 2];
            rg.c1[R][j] = f0.xr[j + 2];
            rg.c2[R][j] = q0.xr[j + 2];
        }
    } else {
        Nbhd<TX, NP> a, b, d;
        a.load(pl, c.ry, c.cx);                       // A: phi0   B: phi3
        b.load(pl + c.plane_elems, c.ry, c.cx);       // A: pi0    B: phi0
        double sa[NP], sb2[NP];
        a.lap_xy(P.k2, sa);
        if constexpr (PAIR == PAIR_A) {
            d.combine(a, P.hdt, b);                   // phi2 = phi0 + (dt/2) pi0
            d.lap_xy(P.k2, sb2);
#pragma unroll
            for (int j = 0; j < NP; ++j) {
                rg.ua[R][j] = a.xr[j + 2];
                rg.sa[R][j] = sa[j];
                rg.ub[R][j] = d.xr[j + 2];
                rg.sb[R][j] = sb2[j];
                rg.c1[R][j] = b.xr[j + 2];
            }
        } else if constexpr (PAIR == PAIR_LA) {
            d.combine(a, P.hdt, b);                   // phi2 = phi0 + (dt/2) pi0
            d.lap_xy(P.k2, sb2);
#pragma unroll
            for (int j = 0; j < NP; ++j) {
                rg.ua[R][j] = a.xr[j + 2];
                rg.sa[R][j] = sa[j];
                rg.ub[R][j] = d.xr[j + 2];
                rg.sb[R][j] = sb2[j];
            }
        } else if constexpr (PAIR == PAIR_B) {
            Nbhd<TX, NP> p3;
            p3.load(pl + 2 * c.plane_elems, c.ry, c.cx);   // pi3
            d.combine(b, P.dt, p3);                   // phi4 = phi0 + dt pi3
            d.lap_xy(P.k2, sb2);
#pragma unroll
            for (int j = 0; j < NP; ++j) {
                rg.ua[R][j] = a.xr[j + 2];
                rg.sa[R][j] = sa[j];
                rg.ub[R][j] = d.xr[j + 2];
                rg.sb[R][j] = sb2[j];
                rg.c1[R][j] = b.xr[j + 2];
                rg.c2[R][j] = p3.xr[j + 2];
            }
            if (i >= 4) {
#pragma unroll
                for (int t = 0; t < 3; ++t)
                    col_vals<NP>(pl + NH * c.plane_elems + t * c.tile_elems + c.ry * TX + NP * c.cx, tv[t]);
            }
        }
    }

#if SB_RKPAIR_BARRIER_EVERY == 2
    if constexpr (prepass(PAIR)) {
        named_bar(1, c.nthr);   // stage s and derived plane i consumed; derived plane i+1 visible
        if (c.tid == 0 && i + kStages < c.nplanes) issue<PAIR, TX>(c, P, i + kStages, s);
    } else if ((i & 1) || i + 1 == c.nplanes) {   // uniform: every second plane, and the last
        named_bar(1, c.nthr);              // every thread is done with the stages of planes <= i
        if (c.tid == 0) {
            if ((i & 1) && i - 1 + kStages < c.nplanes) issue<PAIR, TX>(c, P, i - 1 + kStages, (i - 1) & (kStages - 1));
            if (i + kStages < c.nplanes) issue<PAIR, TX>(c, P, i + kStages, s);
        }
    }
#else
    named_bar(1, c.nthr);   // every thread is done with stage s
    if (c.tid == 0 && i + kStages < c.nplanes) issue<PAIR, TX>(c, P, i + kStages, s);
#endif
    if (i < 4) return false;

    constexpr int K0 = (R + 1) % 5, K1 = (R + 2) % 5, K2 = (R + 3) % 5, K3 = (R + 4) % 5, K4 = R;
    const int x = c.X0 + NP * c.cx, y = c.Y0 + c.ry;
    const bool edge = c.xy_edge || (P.per[0] && (zc < P.pghost || zc >= P.per[2] - P.pghost));
    double la[NP], lb[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) {
        la[j] = add(rg.sa[K2][j], d2(rg.ua[K0][j], rg.ua[K1][j], rg.ua[K2][j], rg.ua[K3][j], rg.ua[K4][j], P.k2));
        lb[j] = add(rg.sb[K2][j], d2(rg.ub[K0][j], rg.ub[K1][j], rg.ub[K2][j], rg.ub[K3][j], rg.ub[K4][j], P.k2));
    }
    if constexpr (PAIR == PAIR_A) {
        // stage 1: pi2 = pi0 + (dt/2) L1          stage 2: phi3 = phi0 + (dt/2) pi2
        //          (acc_pi = L1)                           pi3  = pi0 + (dt/2) L2
        //                                                  acc_phi = pi0 + 2 pi2, acc_pi = L1 + 2 L2
        double f3[NP], p3[NP], af[NP], ap[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const double phi0 = rg.ua[K2][j], pi0 = rg.c1[K2][j];
            const double pi2 = add(pi0, mul(P.hdt, la[j]));
            f3[j] = add(phi0, mul(P.hdt, pi2));
            p3[j] = add(pi0, mul(P.hdt, lb[j]));
            af[j] = add(pi0, mul(2.0, pi2));
            ap[j] = add(la[j], mul(2.0, lb[j]));
        }
        out_periodic<NP>(P, 0, rg.o[0], edge, x, y, zc, f3, L);
        out_periodic<NP>(P, 1, rg.o[1], edge, x, y, zc, p3, L);
        store<NP>(rg.o[2], af, L);
        store<NP>(rg.o[3], ap, L);
    } else if constexpr (PAIR == PAIR_LA) {
        out_periodic<NP>(P, 0, rg.o[0], edge, x, y, zc, la, L);   // L1 = Lap(phi0)
        out_periodic<NP>(P, 1, rg.o[1], edge, x, y, zc, lb, L);   // L2 = Lap(phi2)
    } else if constexpr (PAIR == PAIR_LB) {
        // la = L3, lb = L4; the stage 1-3 quantities are re-formed from phi0, pi0, L1, L2
        double fn[NP], pn[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const double phi0 = rg.c1[K2][j], pi0 = rg.c2[K2][j], l1 = rg.c3[K2][j], l2 = rg.c4[K2][j];
            const double pi2 = add(pi0, mul(P.hdt, l1));
            const double pi3 = add(pi0, mul(P.hdt, l2));
            const double pi4 = add(pi0, mul(P.dt, la[j]));
            const double acf = add(add(pi0, mul(2.0, pi2)), mul(2.0, pi3));
            const double acp = add(add(l1, mul(2.0, l2)), mul(2.0, la[j]));
            fn[j] = add(phi0, mul(P.dt6, add(acf, pi4)));
            pn[j] = add(pi0, mul(P.dt6, add(acp, lb[j])));
        }
        out_periodic<NP>(P, 0, rg.o[0], edge, x, y, zc, fn, L);
        out_periodic<NP>(P, 1, rg.o[1], edge, x, y, zc, pn, L);
    } else {
        // stage 3: pi4 = pi0 + dt L3, acc_phi += 2 pi3, acc_pi += 2 L3   (phi4 = phi0 + dt pi3)
        // stage 4: phi' = phi0 + (dt/6)(acc_phi + pi4), pi' = pi0 + (dt/6)(acc_pi + L4)
        double fn[NP], pn[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const double phi0 = rg.c1[K2][j], pi3 = rg.c2[K2][j];
            const double pi0 = tv[0][j], acf = tv[1][j], acp = tv[2][j];
            const double pi4 = add(pi0, mul(P.dt, la[j]));
            const double acf3 = add(acf, mul(2.0, pi3));
            const double acp3 = add(acp, mul(2.0, la[j]));
            fn[j] = add(phi0, mul(P.dt6, add(acf3, pi4)));
            pn[j] = add(pi0, mul(P.dt6, add(acp3, lb[j])));
        }
        out_periodic<NP>(P, 0, rg.o[0], edge, x, y, zc, fn, L);
        out_periodic<NP>(P, 1, rg.o[1], edge, x, y, zc, pn, L);
    }
#pragma unroll
    for (int k = 0; k < n_out(PAIR); ++k) rg.o[k] += P.sz;
    return false;
}

// TYC > 0: the tile height is a compile-time constant (the default shape),
// so every staged-plane offset folds into an immediate; TYC = 0: P.ty
template <int PAIR, int TX, int NP, int TYC>
__global__ void __launch_bounds__(lb_threads(TX, NP, TYC), lb_minb(PAIR, TYC))
    rkpair_kernel(const __grid_constant__ PairParams P) {
    pdl_launch_dependents();    // PDL: see lap7.cu
    pdl_wait_prerequisites();
    constexpr int TPR = TX / NP;
    constexpr int W = TX + 4;
    extern __shared__ __align__(1024) unsigned char smem[];
    PCtx c;
    c.TY = TYC > 0 ? TYC : P.ty;
    c.H = c.TY + 4;
    c.nthr = TPR * c.TY;
    c.plane_elems = round_up(W * c.H, 16);
    c.tile_elems = round_up(TX * c.TY, 16);
    c.stage_elems = n_halo(PAIR) * c.plane_elems + n_tile(PAIR) * c.tile_elems;
    c.full = reinterpret_cast<uint64_t *>(smem);
    c.stages = reinterpret_cast<const double *>(smem + 128);
    c.derived = const_cast<double *>(c.stages) + kStages * c.stage_elems;

    int t = blockIdx.x;
    const int bx = t % P.ntx;
    t /= P.ntx;
    const int by = t % P.nty;
    const int bz = t / P.nty;
    c.X0 = P.ax0 + bx * TX;
    c.Y0 = P.lo[1] + by * c.TY;
    c.Z0 = P.lo[2] + bz * P.zc;
    c.Z1 = min(c.Z0 + P.zc, P.hi[2]);
    c.nplanes = c.Z1 - c.Z0 + 4;
    c.tid = threadIdx.x;
    c.cx = c.tid % TPR;
    c.ry = c.tid / TPR;
    const int x = c.X0 + NP * c.cx, y = c.Y0 + c.ry;
    c.off_xy = (long long)x + (long long)y * P.sy;
    Lanes<NP> L;
    const bool yin = y < P.hi[1];
#pragma unroll
    for (int j = 0; j < NP; ++j) L.m[j] = (yin && x + j >= P.lo[0] && x + j < P.hi[0]) ? 1 : 0;
    c.xy_edge = P.per[0] && !(x >= P.pghost && x + NP <= P.per[0] - P.pghost && y >= P.pghost &&
                              y < P.per[1] - P.pghost);
    if constexpr (NP == 2) {
        L.full = L.m[0] & L.m[1];
        L.only0 = L.m[0] & (L.m[1] ^ 1);
        L.only1 = L.m[1] & (L.m[0] ^ 1);
    }

    if (c.tid == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&c.full[s], 1);
        fence_mbar_init();
        for (int i = 0; i < kStages && i < c.nplanes; ++i) issue<PAIR, TX>(c, P, i, i);
    }
    __syncthreads();
    if constexpr (prepass(PAIR)) {   // derived fields of plane 0
        mbar_wait(&c.full[0], 0);
        derive_plane<PAIR, TX>(c, P, 0);
        named_bar(1, c.nthr);
    }

    PRings<NP> rg;
#pragma unroll
    for (int k = 0; k < 5; ++k)
#pragma unroll
        for (int j = 0; j < NP; ++j)
            rg.ua[k][j] = rg.sa[k][j] = rg.ub[k][j] = rg.sb[k][j] = rg.c1[k][j] = rg.c2[k][j] = rg.c3[k][j] =
                rg.c4[k][j] = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) rg.o[k] = P.out[k] + c.off_xy + (long long)c.Z0 * P.sz;
    for (int i = 0;; i += 5) {
        if (pair_plane<PAIR, TX, NP, 0>(i + 0, c, P, L, rg)) break;
        if (pair_plane<PAIR, TX, NP, 1>(i + 1, c, P, L, rg)) break;
        if (pair_plane<PAIR, TX, NP, 2>(i + 2, c, P, L, rg)) break;
        if (pair_plane<PAIR, TX, NP, 3>(i + 3, c, P, L, rg)) break;
        if (pair_plane<PAIR, TX, NP, 4>(i + 4, c, P, L, rg)) break;
    }
}

size_t pair_smem(int pair, int tx, int ty) {
    const size_t plane = round_up((tx + 4) * (ty + 4), 16);
    return 128 + (size_t)kStages * 8 * (n_halo(pair) * plane + n_tile(pair) * round_up(tx * ty, 16)) +
           (size_t)2 * n_derived(pair) * plane * 8;
}

template <int PAIR, int TX, int NP, int TYC>
int launch_pair_ty(const PairParams &P, int nblocks, cudaStream_t st) {
    auto fn = rkpair_kernel<PAIR, TX, NP, TYC>;
    if (int rc = ensure_smem_limit((const void *)fn, 227 * 1024, "cudaFuncSetAttribute(rkpair)")) return rc;
    return launch_pdl(fn, dim3(nblocks), dim3((TX / NP) * P.ty), pair_smem(PAIR, TX, P.ty), st,
                      "rkpair_kernel launch", P);
}

template <int PAIR, int TX, int NP>
int launch_pair_tx(const PairParams &P, int nblocks, cudaStream_t st) {
    if constexpr (TX == 32 && NP == 1)
        if (P.ty == 4) return launch_pair_ty<PAIR, TX, NP, 4>(P, nblocks, st);
    return launch_pair_ty<PAIR, TX, NP, 0>(P, nblocks, st);
}

template <int PAIR, int NP>
int launch_pair_np(const PairParams &P, int tx, int nblocks, cudaStream_t st) {
    switch (tx) {
        case 32: return launch_pair_tx<PAIR, 32, NP>(P, nblocks, st);
        case 64: return launch_pair_tx<PAIR, 64, NP>(P, nblocks, st);
        case 128: return launch_pair_tx<PAIR, 128, NP>(P, nblocks, st);
        default: return fail(SB_USAGE, "tile_x must be 32, 64 or 128");
    }
}

}  // namespace

int launch_rk4_pair(int pair, const sb_array *halo, int nh, const sb_array *tile, int nt, const sb_array *out, int no,
                    const sb_space &sp, const sb_rk4_constants &k, const sb_launch &p, cudaStream_t st,
                    const sb_zslab *zs) {
    const int TX = p.tile_x, TY = p.tile_y, ZC = p.z_chunk;
    const int NP = (p.flags & SB_LAUNCH_SCALAR) ? 1 : 2;
    if (TX != 32 && TX != 64 && TX != 128) return fail(SB_USAGE, "tile_x must be 32, 64 or 128");
    if (TY < 1 || ZC < 1) return fail(SB_USAGE, "tile_y and z_chunk must be positive");
    const int threads = (TX / NP) * TY;
    if (threads % 32 || threads > max_threads_pair(NP))
        return fail(SB_USAGE, "threads per CTA must be a multiple of 32 and <= 256 (pairs) / 512 (scalar)");
    if (TY + 4 > 256) return fail(SB_USAGE, "tile_y + 4 exceeds the TMA box limit of 256");
    if (pair_smem(pair, TX, TY) > 227 * 1024) return fail(SB_RESOURCE, "tile needs more than 227 KB of shared memory");
    for (int d = 0; d < 3; ++d)
        if (sp.hi[d] <= sp.lo[d]) return SB_OK;
    for (int a = 1; a < no; ++a)
        if (out[a].sy != out[0].sy || out[a].sz != out[0].sz)
            return fail(SB_USAGE, "rk4_pair: outputs must share row and plane strides");

    PairParams P;
    memset(&P, 0, sizeof(P));
    for (int h = 0; h < nh; ++h) {
        int rc = make_tmap(&P.hmap[h], halo[h], TX + 4, TY + 4, 1);
        if (rc) return rc;
        P.htma0[h][0] = halo[h].xpad;
        P.htma0[h][1] = halo[h].ghost;
        P.htma0[h][2] = halo[h].ghost;
    }
    for (int t = 0; t < nt; ++t) {
        int rc = make_tmap(&P.tmap[t], tile[t], TX, TY, 1);
        if (rc) return rc;
        P.ttma0[t][0] = tile[t].xpad;
        P.ttma0[t][1] = tile[t].ghost;
        P.ttma0[t][2] = tile[t].ghost;
    }
    for (int a = 0; a < no; ++a) P.out[a] = out[a].origin;
    P.sy = out[0].sy;
    P.sz = out[0].sz;
    for (int d = 0; d < 3; ++d) {
        P.lo[d] = sp.lo[d];
        P.hi[d] = sp.hi[d];
    }
    P.ax0 = (sp.lo[0] >= 0 ? sp.lo[0] / TX : -((-sp.lo[0] + TX - 1) / TX)) * TX;
    P.ntx = (sp.hi[0] - P.ax0 + TX - 1) / TX;
    P.nty = (sp.hi[1] - sp.lo[1] + TY - 1) / TY;
    const int ntz = (sp.hi[2] - sp.lo[2] + ZC - 1) / ZC;
    P.ty = TY;
    P.zc = ZC;
    P.k2 = k.lap.k2;
    P.hdt = k.half_dt;
    P.dt = k.dt;
    P.dt6 = k.dt6;
    if (p.flags & SB_LAUNCH_PERIODIC_GHOSTS) {
        const sb_array &O = out[0];
        if (O.ghost < 1 || O.ghost > O.nx || O.ghost > O.ny || O.ghost > O.nz)
            return fail(SB_USAGE, "periodic ghost refresh needs 1 <= ghost <= every extent");
        for (int d = 0; d < 3; ++d)
            if (sp.lo[d] != 0 || sp.hi[d] != (d == 0 ? O.nx : d == 1 ? O.ny : O.nz))
                return fail(SB_USAGE, "periodic ghost refresh needs the sweep to cover the whole interior");
        if (out[1].ghost != O.ghost || out[1].nx != O.nx || out[1].ny != O.ny || out[1].nz != O.nz)
            return fail(SB_USAGE, "periodic ghost refresh: phi and pi outputs must share geometry");
        P.per[0] = O.nx;
        P.per[1] = O.ny;
        P.per[2] = O.nz;
        P.pghost = O.ghost;
        for (int a = 0; a < 2; ++a) {
            if (zs) {   // z-slab decomposition: z images go to the neighbouring slabs
                P.zlo[a] = zs[a].lo_phi_out;
                P.zlo_dz[a] = zs[a].lo_dz;
                P.zhi[a] = zs[a].hi_phi_out;
                P.zhi_dz[a] = zs[a].hi_dz;
            } else {
                P.zlo[a] = P.zhi[a] = out[a].origin;
                P.zlo_dz[a] = O.nz;
                P.zhi_dz[a] = -O.nz;
            }
        }
    } else if (zs) {
        return fail(SB_USAGE, "z-slab halo stores need SB_LAUNCH_PERIODIC_GHOSTS");
    }
    const long long nb = (long long)P.ntx * P.nty * ntz;
    if (nb > 0x7fffffffLL) return fail(SB_RESOURCE, "too many tiles for one launch");
    switch (pair) {
        case PAIR_A:
            return NP == 1 ? launch_pair_np<PAIR_A, 1>(P, TX, (int)nb, st) : launch_pair_np<PAIR_A, 2>(P, TX, (int)nb, st);
        case PAIR_B:
            return NP == 1 ? launch_pair_np<PAIR_B, 1>(P, TX, (int)nb, st) : launch_pair_np<PAIR_B, 2>(P, TX, (int)nb, st);
        case PAIR_LA:
            return NP == 1 ? launch_pair_np<PAIR_LA, 1>(P, TX, (int)nb, st)
                           : launch_pair_np<PAIR_LA, 2>(P, TX, (int)nb, st);
        default:
            return NP == 1 ? launch_pair_np<PAIR_LB, 1>(P, TX, (int)nb, st)
                           : launch_pair_np<PAIR_LB, 2>(P, TX, (int)nb, st);
    }
}

}  // namespace sb
