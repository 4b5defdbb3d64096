// rhs24.cu — K6: config-5 fused many-variable right-hand side (sm_100a).
//
// For every interior point: 24 fields, each with its value and 9 fourth-order
// derivatives (Dx Dy Dz Dxx Dyy Dzz Dxy Dxz Dyz — the expression trees of
// d4.cu), give 240 inputs v[10*var + slot]; output o is the seed-generated
// polynomial  ((t_0 + t_1) + ...) + t_63,  t_k = (c_ok * v_p) * v_q
// (oracle/stencils.py: rhs24).
//
// One CTA = 12 warps owns an 8 x 4 tile of (x, y) columns and streams z:
//   * every plane of all 24 fields (tile + 2-point halo, 12 x 8) arrives by
//     TMA (24 cp.async.bulk.tensor.3d per plane, one mbarrier) into a
//     2-stage shared-memory ring (a plane is read only in its own iteration);
//   * phase A — warp w reduces fields w and w + 12 (SB_RHS24_FPW = 2; 160
//     registers per thread, twice the independent work per warp, no idle
//     warps in phase B; 24 warps of one field each: 80-register cap,
//     4.5 % slower), lane = column: u and the unscaled x/y
//     first differences of the newest plane go into five-slot register rings
//     (plane loop unrolled five ways), its in-plane second differences Dxx,
//     Dyy into two-plane register queues (computed while its row and column
//     values are in registers), the x differences of the plane (with halo
//     rows) into a 3-plane shared ring for Dxy; two planes later the ten
//     slots of the completed plane go to a [240][32] shared array;
//   * phase B — half-warp h of warp w evaluates output 2w + h for
//     the 32 columns, two per lane: the half-warp runs the same term, so the
//     packed (c, p, q) words are broadcast 16-byte shared-memory reads that
//     serve two outputs per LDS.128 (the table is copied to shared memory per
//     CTA: 24 warps walking 24 different 1 KB slices of __constant__ memory
//     thrash the constant cache), and the two operand loads per term are
//     conflict-free 16-byte reads of rows of [240][32].
// Two CTA barriers per plane.  Bound: shared-memory bandwidth (two 8-byte
// operand loads per term per point), then the FP64 pipe.
#include <cstring>

#include "common.cuh"
#include "internal.h"

namespace sb {

namespace {

constexpr int TXc = 8, TYc = 4, NCOL = TXc * TYc;      // 32 columns per CTA
constexpr int HXc = TXc + 4, HYc = TYc + 4;             // 12 x 8 halo plane
constexpr int PLANE = HXc * HYc;                        // 96 doubles
constexpr int NV = SB_N_VARS, NT = SB_N_TERMS;
#ifndef SB_RHS24_NSTAGE
#define SB_RHS24_NSTAGE 2
#endif
constexpr int NSTAGE = SB_RHS24_NSTAGE;                 // staged planes: the newest + NSTAGE-1 in flight
#ifndef SB_RHS24_FPW
#define SB_RHS24_FPW 2   // fields per warp in phase A (1: 24 warps, 2: 12 warps)
#endif
constexpr int FPW = SB_RHS24_FPW;
constexpr int NWARPS = NV / FPW;
constexpr int NTHREADS = NWARPS * 32;                   // 768 / 384
#ifndef SB_RHS24_PHASEB_UNROLL
#define SB_RHS24_PHASEB_UNROLL 8
#endif
constexpr int kPhaseBUnroll = SB_RHS24_PHASEB_UNROLL;  // eight-term groups per phase-B loop iteration

// One polynomial term is 10 bytes: the coefficient and a 16-bit operand
// pair, p in the low byte and q in the high byte (both < 240; a row of the
// [240][32] operand array is 256 bytes, so the byte offsets are p << 8 and
// q << 8).  Eight terms pack into five 16-byte words — four of coefficient
// pairs, one of the eight operand pairs — so a warp fetches eight terms with
// five broadcast LDS.128 (five shared-memory wavefronts instead of eight).
constexpr int TW = NT / 8 * 5;                          // 16-byte words per output's table
static_assert(NT % 8 == 0, "terms are fetched eight at a time");
static_assert(NCOL * 8 == 256, "operand offsets are row index << 8");
static_assert(sizeof(uint4) * NV * TW < 20 * 1024, "term table must fit the kernel parameter space with the maps");
constexpr size_t SMEM_BYTES = 128 + sizeof(uint4) * NV * TW +
                              sizeof(double) * ((size_t)NSTAGE * NV * PLANE + (size_t)3 * NV * HYc * TXc +
                                                (size_t)10 * NV * NCOL);

struct Rhs24Params {
    // the packed term table travels with the launch (kernel parameter space,
    // copied to shared memory by every CTA): a launch never depends on state
    // another launch or stream may change, and a captured graph replays the
    // table it was captured with
    uint4 terms[NV][TW];
    CUtensorMap tmap[NV];
    double *out[NV];
    long long osy, osz;      // output strides (shared by all outputs)
    int tma0[NV][3];
    int lo[3], hi[3];
    int ax0, ntx, nty, zc;   // x tiles anchored on multiples of 8: TMA boxes start 16-byte aligned
    double k1, k2, k11;
};

struct Ctx {
    uint64_t *full;          // NSTAGE mbarriers
    const uint4 *terms;      // [NV][TW] copy of the packed table in shared memory (broadcast reads)
    double *ring;            // [NSTAGE][NV][PLANE]
    double *rxb;             // [3][NV][HYc][TXc]
    double *vals;            // [240][NCOL]
    int tid, warp, lane, cx, cy;
    int X0, Y0, Z0, Z1, nplanes;
};

struct Rings {
    double u[5], rx[5], ry[5];
    double dxx[2], dyy[2];   // Dxx, Dyy of the two planes before the newest ([0]: z-1, [1]: z-2)
};

// Physical row of logical row r (0..7) of an 8-wide rx plane: parity pattern
// 0,0,1,1,0,0,1,1 keeps rows r and r+2 in different 64-byte bank halves.
__device__ __forceinline__ int rxrow(int r) {
    constexpr unsigned kPerm = 0u | (2u << 3) | (1u << 6) | (3u << 9) | (4u << 12) | (6u << 15) | (5u << 18) | (7u << 21);
    return (kPerm >> (3 * r)) & 7;
}

// Row values x = cx .. cx+4 of a staged 12-wide row: three 16-byte loads of
// the aligned pairs from cx & ~1 (lanes cx and cx^1 read the same words), the
// five values selected by the parity of cx — 6 shared wavefronts per warp
// instead of 10 for five 8-byte loads.
__device__ __forceinline__ void row5(const double *r, int cx, double (&v)[5]) {
    const double2 *q = reinterpret_cast<const double2 *>(r + (cx & ~1));
    const double2 a = q[0], b = q[1], d = q[2];
    const bool odd = cx & 1;
    v[0] = odd ? a.y : a.x;
    v[1] = odd ? b.x : a.y;
    v[2] = odd ? b.y : b.x;
    v[3] = odd ? d.x : b.y;
    v[4] = odd ? d.y : d.x;
}

// thread 0: all 24 field planes of stream plane j into stage j % NSTAGE
__device__ __forceinline__ void issue(const Rhs24Params &P, const Ctx &c, int j) {
    const int s = j % NSTAGE;
    mbar_arrive_expect_tx(&c.full[s], NV * PLANE * 8);
    double *dst = c.ring + s * NV * PLANE;
#pragma unroll 4
    for (int v = 0; v < NV; ++v)
        tma_load_3d(dst + v * PLANE, &P.tmap[v], P.tma0[v][0] + c.X0 - 2, P.tma0[v][1] + c.Y0 - 2,
                    P.tma0[v][2] + c.Z0 - 2 + j, &c.full[s]);
}

template <int R>
__device__ __forceinline__ bool plane(int i, const Rhs24Params &P, const Ctx &c, Rings (&rgs)[FPW]) {
    if (i >= c.nplanes) return true;
    const int s = i % NSTAGE;
    mbar_wait(&c.full[s], (i / NSTAGE) & 1);

    double dxx_new[FPW], dyy_new[FPW];
    // ---- phase A, newest plane z = Z0-2+i: u, rx, ry into the rings; rx plane (+ halo rows) ----
#pragma unroll
    for (int f = 0; f < FPW; ++f) {
        const int v = c.warp + f * NWARPS;   // this warp's field f
        Rings &rg = rgs[f];
        const double *pl = c.ring + (s * NV + v) * PLANE;
        const double *col = pl + c.cy * HXc + c.cx + 2;
        double row[5];
        row5(pl + (c.cy + 2) * HXc, c.cx, row);
        rg.u[R] = row[2];
        rg.rx[R] = d1u(row[0], row[1], row[3], row[4]);
        rg.ry[R] = d1u(col[0], col[HXc], col[3 * HXc], col[4 * HXc]);
        // the in-plane second differences of this plane now, while its row and
        // column values are in registers (used two planes later)
        dxx_new[f] = d2(row[0], row[1], row[2], row[3], row[4], P.k2);
        dyy_new[f] = d2(col[0], col[HXc], row[2], col[3 * HXc], col[4 * HXc], P.k2);
        double *rxs = c.rxb + ((i % 3) * NV + v) * (HYc * TXc);
        rxs[rxrow(c.cy + 2) * TXc + c.cx] = rg.rx[R];
        // lanes double as the 4 halo rows x 8 columns; half-warps take rows {0, 6} and {1, 7}
        const int h = c.lane >> 3, hc = c.lane & 7;
        const int hr = (h & 1) ? 6 + (h >> 1) : (h >> 1);
        double hrow[5];
        row5(pl + hr * HXc, hc, hrow);
        rxs[rxrow(hr) * TXc + hc] = d1u(hrow[0], hrow[1], hrow[3], hrow[4]);
    }

    // ---- phase A, completed plane zc = z-2: the ten slots ----
    const bool out_plane = i >= 4;
    if (out_plane) __syncwarp();    // rx plane of zc was written by this warp two planes ago; keep lanes in step
#pragma unroll
    for (int f = 0; f < FPW; ++f) {
        if (!out_plane) break;
        const int v = c.warp + f * NWARPS;
        Rings &rg = rgs[f];
        constexpr int K0 = (R + 1) % 5, K1 = (R + 2) % 5, K2 = (R + 3) % 5, K3 = (R + 4) % 5, K4 = R;
        const double uc = rg.u[K2];
        const double *rxs = c.rxb + (((i - 2) % 3) * NV + v) * (HYc * TXc) + c.cx;
        double *o = c.vals + (10 * v) * NCOL + c.lane;
        o[0 * NCOL] = uc;
        o[1 * NCOL] = mul(rg.rx[K2], P.k1);
        o[2 * NCOL] = mul(rg.ry[K2], P.k1);
        o[3 * NCOL] = mul(d1u(rg.u[K0], rg.u[K1], rg.u[K3], rg.u[K4]), P.k1);
        o[4 * NCOL] = rg.dxx[1];
        o[5 * NCOL] = rg.dyy[1];
        o[6 * NCOL] = d2(rg.u[K0], rg.u[K1], uc, rg.u[K3], rg.u[K4], P.k2);
        o[7 * NCOL] = mul(d1u(rxs[rxrow(c.cy + 0) * TXc], rxs[rxrow(c.cy + 1) * TXc], rxs[rxrow(c.cy + 3) * TXc],
                              rxs[rxrow(c.cy + 4) * TXc]),
                          P.k11);
        o[8 * NCOL] = mul(d1u(rg.rx[K0], rg.rx[K1], rg.rx[K3], rg.rx[K4]), P.k11);
        o[9 * NCOL] = mul(d1u(rg.ry[K0], rg.ry[K1], rg.ry[K3], rg.ry[K4]), P.k11);
    }

#pragma unroll
    for (int f = 0; f < FPW; ++f) {
        rgs[f].dxx[1] = rgs[f].dxx[0];
        rgs[f].dxx[0] = dxx_new[f];
        rgs[f].dyy[1] = rgs[f].dyy[0];
        rgs[f].dyy[0] = dyy_new[f];
    }
    // every slot of plane zc is written, and every staged plane is read only
    // in its own iteration (phase A of the newest plane): stage s is free for
    // plane i + NSTAGE
    __syncthreads();
    if (c.tid == 0 && i + NSTAGE < c.nplanes) issue(P, c, i + NSTAGE);
    if (!out_plane) return false;

    // ---- phase B: warps 0..11, half-warp h of warp w evaluates output 2w + h
    // for the 32 columns of plane zc, two adjacent columns per lane ----
    // Every lane of a half-warp runs the same term, so a table word is a
    // broadcast within the half-warp and one LDS.128 (two half-warp phases)
    // serves two outputs: half the table wavefronts of one output per warp,
    // while the 16-byte operand loads move the same bytes per point.
    if (c.warp < NV / 2) {
        const int o = 2 * c.warp + (c.lane >> 4), l16 = c.lane & 15;
        const uint4 *tt = c.terms + o * TW;
        const char *vb = reinterpret_cast<const char *>(c.vals) + 16 * l16;
        auto V = [vb](uint32_t off) { return *reinterpret_cast<const double2 *>(vb + off); };
        double a0 = 0.0, a1 = 0.0;
        // pq: p in bits 0-7, q in bits 8-15 -> byte offsets p << 8, q << 8 of the operand rows
        auto term = [&](double cf, uint32_t pq, bool first) {
            const double2 vp = V((pq << 8) & 0xff00u), vq = V(pq & 0xff00u);
            const double t0 = mul(mul(cf, vp.x), vq.x), t1 = mul(mul(cf, vp.y), vq.y);
            a0 = first ? t0 : add(a0, t0);
            a1 = first ? t1 : add(a1, t1);
        };
#pragma unroll kPhaseBUnroll
        for (int g = 0; g < NT / 8; ++g) {
            // five 16-byte loads carry terms 8g .. 8g+7 (eight coefficients, eight operand pairs)
            const double2 c01 = *reinterpret_cast<const double2 *>(tt + 5 * g);
            const double2 c23 = *reinterpret_cast<const double2 *>(tt + 5 * g + 1);
            const double2 c45 = *reinterpret_cast<const double2 *>(tt + 5 * g + 2);
            const double2 c67 = *reinterpret_cast<const double2 *>(tt + 5 * g + 3);
            const uint4 w = tt[5 * g + 4];
            term(c01.x, w.x & 0xffffu, g == 0);
            term(c01.y, w.x >> 16, false);
            term(c23.x, w.y & 0xffffu, false);
            term(c23.y, w.y >> 16, false);
            term(c45.x, w.z & 0xffffu, false);
            term(c45.y, w.z >> 16, false);
            term(c67.x, w.w & 0xffffu, false);
            term(c67.y, w.w >> 16, false);
        }
        // vals column k was written by phase-A lane k: (x, y) = (k & 7, ((k >> 3) & 1) * 2 + (k >> 4));
        // columns 2 l16 and 2 l16 + 1 are adjacent points of one row
        const int k = 2 * l16;
        const int x = c.X0 + (k & 7), y = c.Y0 + ((k >> 3) & 1) * 2 + (k >> 4), zc = c.Z0 - 4 + i;
        const bool yin = y < P.hi[1];
        store_pair(P.out[o] + x + (long long)y * P.osy + (long long)zc * P.osz, a0, a1,
                   yin && x >= P.lo[0] && x < P.hi[0], yin && x + 1 >= P.lo[0] && x + 1 < P.hi[0]);
    }
    __syncthreads();   // the [240][32] array is rewritten by the next plane
    return false;
}

__global__ void __launch_bounds__(NTHREADS, 1) rhs24_kernel(const __grid_constant__ Rhs24Params P) {
    pdl_launch_dependents();    // PDL: see lap7.cu
    pdl_wait_prerequisites();
    extern __shared__ __align__(1024) unsigned char smem[];
    Ctx c;
    c.full = reinterpret_cast<uint64_t *>(smem);
    uint4 *terms = reinterpret_cast<uint4 *>(smem + 128);
    c.terms = terms;
    c.ring = reinterpret_cast<double *>(terms + NV * TW);
    c.rxb = c.ring + NSTAGE * NV * PLANE;
    c.vals = c.rxb + 3 * NV * HYc * TXc;
    c.tid = threadIdx.x;
    c.warp = c.tid >> 5;
    c.lane = c.tid & 31;
    // lanes 0-7 -> row 0, 8-15 -> row 2, 16-23 -> row 1, 24-31 -> row 3: each
    // half-warp reads two rows 24 doubles apart in the 12-wide staged planes,
    // i.e. disjoint bank halves (rows 12 apart would share 4 bank pairs)
    c.cx = c.lane & 7;
    c.cy = ((c.lane >> 3) & 1) * 2 + (c.lane >> 4);
    int t = blockIdx.x;
    const int bx = t % P.ntx;
    t /= P.ntx;
    const int by = t % P.nty;
    const int bz = t / P.nty;
    c.X0 = P.ax0 + bx * TXc;
    c.Y0 = P.lo[1] + by * TYc;
    c.Z0 = P.lo[2] + bz * P.zc;
    c.Z1 = min(c.Z0 + P.zc, P.hi[2]);
    c.nplanes = c.Z1 - c.Z0 + 4;

    if (c.tid == 0) {
        for (int s = 0; s < NSTAGE; ++s) mbar_init(&c.full[s], 1);
        fence_mbar_init();
        for (int j = 0; j < NSTAGE && j < c.nplanes; ++j) issue(P, c, j);
    }
    for (int e = c.tid; e < NV * TW; e += NTHREADS) terms[e] = (&P.terms[0][0])[e];
    __syncthreads();

    Rings rg[FPW];
#pragma unroll
    for (int f = 0; f < FPW; ++f) {
#pragma unroll
        for (int k = 0; k < 5; ++k) rg[f].u[k] = rg[f].rx[k] = rg[f].ry[k] = 0.0;
        rg[f].dxx[0] = rg[f].dxx[1] = rg[f].dyy[0] = rg[f].dyy[1] = 0.0;
    }
    for (int i = 0;; i += 5) {
        if (plane<0>(i + 0, P, c, rg)) break;
        if (plane<1>(i + 1, P, c, rg)) break;
        if (plane<2>(i + 2, P, c, rg)) break;
        if (plane<3>(i + 3, P, c, rg)) break;
        if (plane<4>(i + 4, P, c, rg)) break;
    }
}

}  // namespace

int launch_rhs24(const sb_array *in, const sb_array *out, const sb_space &sp, const sb_d4_constants &k,
                 const sb_poly &poly, const sb_launch &p, cudaStream_t st) {
    for (int d = 0; d < 3; ++d)
        if (sp.hi[d] <= sp.lo[d]) return SB_OK;
    if (!poly.coef || !poly.p || !poly.q) return fail(SB_USAGE, "rhs24: null polynomial table");
    for (int v = 1; v < NV; ++v)
        if (out[v].sy != out[0].sy || out[v].sz != out[0].sz)
            return fail(SB_USAGE, "rhs24: all outputs must share row and plane strides");

    Rhs24Params P;
    memset(&P, 0, sizeof(P));
    for (int o = 0; o < NV; ++o)
        for (int g = 0; g < NT / 8; ++g) {
            double *cf = reinterpret_cast<double *>(&P.terms[o][5 * g]);          // 8 coefficients
            uint16_t *pq = reinterpret_cast<uint16_t *>(&P.terms[o][5 * g + 4]);  // 8 operand pairs
            for (int k = 0; k < 8; ++k) {
                const int t = 8 * g + k;
                const int pi = poly.p[o * NT + t], qi = poly.q[o * NT + t];
                if (pi < 0 || pi >= 10 * NV || qi < 0 || qi >= 10 * NV)
                    return fail(SB_USAGE, "rhs24: polynomial input index outside 0..239");
                cf[k] = poly.coef[o * NT + t];
                pq[k] = (uint16_t)(pi | (qi << 8));
            }
        }
    for (int v = 0; v < NV; ++v) {
        int rc = make_tmap(&P.tmap[v], in[v], HXc, HYc, 1);
        if (rc) return rc;
        P.tma0[v][0] = in[v].xpad;
        P.tma0[v][1] = in[v].ghost;
        P.tma0[v][2] = in[v].ghost;
        P.out[v] = out[v].origin;
    }
    P.osy = out[0].sy;
    P.osz = out[0].sz;
    for (int d = 0; d < 3; ++d) {
        P.lo[d] = sp.lo[d];
        P.hi[d] = sp.hi[d];
    }
    P.zc = p.z_chunk > 0 ? p.z_chunk : 32;
    P.ax0 = (sp.lo[0] >= 0 ? sp.lo[0] / TXc : -((-sp.lo[0] + TXc - 1) / TXc)) * TXc;
    P.ntx = (sp.hi[0] - P.ax0 + TXc - 1) / TXc;
    P.nty = (sp.hi[1] - sp.lo[1] + TYc - 1) / TYc;
    const int ntz = (sp.hi[2] - sp.lo[2] + P.zc - 1) / P.zc;
    P.k1 = k.k1;
    P.k2 = k.k2;
    P.k11 = k.k11;
    const long long nblocks = (long long)P.ntx * P.nty * ntz;
    if (nblocks > 0x7fffffffLL) return fail(SB_RESOURCE, "rhs24: too many tiles");
    if (int rc = ensure_smem_limit((const void *)rhs24_kernel, (int)SMEM_BYTES, "cudaFuncSetAttribute(rhs24)"))
        return rc;
    return launch_pdl(rhs24_kernel, dim3((unsigned)nblocks), dim3(NTHREADS), SMEM_BYTES, st, "rhs24_kernel launch", P);
}

}  // namespace sb
