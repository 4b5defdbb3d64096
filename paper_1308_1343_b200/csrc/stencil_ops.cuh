// stencil_ops.cuh — lane-level helpers shared by the z-streaming stencil
// kernels (d4.cu, rkpair.cu): predicated pair/single stores (the
// iterate_masked frame rule, vlanes.py:322-337), shared-memory row/column
// reads, and the out-of-line periodic ghost-image store.
#pragma once

#include "common.cuh"

namespace sb {
namespace ops {

// Predicated stores (no branches): pair / single lanes.  SB_STORE_HINT is
// the cache operator of the output stream (default .cs: streaming,
// evict-first — outputs are never re-read by the sweep).
#ifndef SB_STORE_HINT
#define SB_STORE_HINT ".cs"
#endif
__device__ __forceinline__ void st_v2(double *p, double a, double b, int pred) {
    asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %3, 0;\n@q st.global" SB_STORE_HINT
                 ".v2.f64 [%0], {%1, %2};\n}\n" ::"l"(p),
                 "d"(a), "d"(b), "r"(pred)
                 : "memory");
}
__device__ __forceinline__ void st_1(double *p, double a, int pred) {
    asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q st.global" SB_STORE_HINT ".f64 [%0], %1;\n}\n" ::"l"(p),
                 "d"(a), "r"(pred)
                 : "memory");
}

template <int NP>
struct Lanes {
    int m[NP];           // per-point store masks
    int full, only0, only1;  // NP == 2 store classes
};

template <int NP>
__device__ __forceinline__ void store(double *p, const double (&v)[NP], const Lanes<NP> &L) {
#ifdef SB_PROBE_NOSTORE
    // probe builds only (tools/ab_c3.sh): values stay live, the stores never issue
    if (v[0] != -1234.5678) return;
#endif
    if constexpr (NP == 2) {
        st_v2(p, v[0], v[1], L.full);
        st_1(p, v[0], L.only0);
        st_1(p + 1, v[1], L.only1);
    } else {
        st_1(p, v[0], L.m[0]);
    }
}

// Row values x-2 .. x+NP+1 of shared-memory row `r` starting at column c (= x-2).
template <int NP>
__device__ __forceinline__ void row_vals(const double *r, double (&v)[NP + 4]) {
    if constexpr (NP == 2) {
        const double2 a = load_pair(r), b = load_pair(r + 2), c = load_pair(r + 4);
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y; v[4] = c.x; v[5] = c.y;
    } else {
#pragma unroll
        for (int k = 0; k < 5; ++k) v[k] = r[k];
    }
}

template <int NP>
__device__ __forceinline__ void col_vals(const double *r, double (&v)[NP]) {
    if constexpr (NP == 2) {
        const double2 a = load_pair(r);
        v[0] = a.x; v[1] = a.y;
    } else {
        v[0] = r[0];
    }
}

// Store-side periodic ghost refresh: also write v at every ghost point that is
// a periodic image of interior point (x+j, y, z).  Per axis the images are
// +n (when the point is within g of the low face) and -n (within g of the
// high face) — both when 2g > n.  Exact copies.
__device__ __forceinline__ int images(int c, int n, int g, int (&o)[3]) {
    const bool lo = c < g, hi = c >= n - g;
    o[0] = 0;
    o[1] = lo ? n : -n;
    o[2] = -n;
    return 1 + (int)lo + (int)hi;
}

// Rare path, kept out of line so the unrolled plane loop stays small.  x/y
// images stay in each target; z images go to the z targets (this grid when
// the box is periodic in z, the neighbouring slabs' grids for a z-slab
// decomposition).
static __device__ __noinline__ void store_images(double *base, long long sy, long long sz, int nx, int ny, int nz, int g,
                                          double *zlo, int zlo_dz, double *zhi, int zhi_dz, int x, int y, int z,
                                          double v) {
    int ox[3], oy[3];
    const int kx = images(x, nx, g, ox), ky = images(y, ny, g, oy);
    double *tb[3];
    int tz[3], kt = 0;
    tb[kt] = base;
    tz[kt++] = 0;
    if (z < g && zlo) {
        tb[kt] = zlo;
        tz[kt++] = zlo_dz;
    }
    if (z >= nz - g && zhi) {
        tb[kt] = zhi;
        tz[kt++] = zhi_dz;
    }
    for (int t = 0; t < kt; ++t)
        for (int b = 0; b < ky; ++b)
            for (int d = 0; d < kx; ++d)
                if (t | b | d) tb[t][(x + ox[d]) + (long long)(y + oy[b]) * sy + (long long)(z + tz[t]) * sz] = v;
}


}  // namespace ops
}  // namespace sb
