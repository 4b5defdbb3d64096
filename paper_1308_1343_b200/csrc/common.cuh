// common.cuh — device helpers shared by the stencil kernels (sm_100a).
//
// Arithmetic helpers spell out one IEEE rounding per operation so that the
// device evaluates exactly the expression trees of the reference's numpy
// kernels (stencil.py:35-39) and of the oracle (oracle/stencils.py); the
// library is additionally compiled with -fmad=false.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/stencil_b200.h"

namespace sb {

// ---- exact-order fp64 arithmetic -------------------------------------------
#if SB_FMA
// tolerance mode (experiment): plain operators, contractible into FMAs with -fmad=true
__device__ __forceinline__ double add(double a, double b) { return a + b; }
__device__ __forceinline__ double sub(double a, double b) { return a - b; }
__device__ __forceinline__ double mul(double a, double b) { return a * b; }
#else
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
#endif

// Unscaled 4th-order first difference: (u[-2] - u[+2]) + 8*(u[+1] - u[-1]).
__device__ __forceinline__ double d1u(double m2, double m1, double p1, double p2) {
    return add(sub(m2, p2), mul(8.0, sub(p1, m1)));
}
// Scaled 4th-order second difference: ((16*(u[-1]+u[+1]) - (u[-2]+u[+2])) - 30*u) * k2.
__device__ __forceinline__ double d2(double m2, double m1, double c, double p1, double p2, double k2) {
    return mul(sub(sub(mul(16.0, add(m1, p1)), add(m2, p2)), mul(30.0, c)), k2);
}

// ---- device-side grid view ---------------------------------------------------
struct Grid {
    double *o;
    long long sy, sz;
    __device__ __forceinline__ double *at(int x, int y, int z) const {
        return o + (long long)x + (long long)y * sy + (long long)z * sz;
    }
};

__host__ __forceinline__ Grid grid_of(const sb_array &a) { return Grid{a.origin, a.sy, a.sz}; }

// Store one or two adjacent points (x even => 16-byte aligned pair).
__device__ __forceinline__ void store_pair(double *p, double v0, double v1, bool m0, bool m1) {
    if (m0 && m1) {
        asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v0), "d"(v1) : "memory");
    } else {
        if (m0) __stcs(p, v0);
        if (m1) __stcs(p + 1, v1);
    }
}

__device__ __forceinline__ double2 load_pair(const double *p) {
    return *reinterpret_cast<const double2 *>(p);
}

// ---- mbarrier + TMA (PTX) ----------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// One bounded hardware wait for phase `parity` of an mbarrier.
__device__ __forceinline__ bool mbar_try(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return done != 0;
}

// Out of line: keep retrying; a wait that has not completed after ~2^24
// polls traps (turns a pipeline bug into a launch error instead of a hung
// GPU).
static __device__ __noinline__ void mbar_wait_slow(uint64_t *bar, uint32_t parity) {
    for (uint32_t n = 0; !mbar_try(bar, parity); ++n)
        if (n > (1u << 24)) __trap();
}

// Wait for phase `parity` of an mbarrier: the common case (data already
// there, or arriving within the hardware's wait window) is one try_wait.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    if (__builtin_expect(!mbar_try(bar, parity), 0)) mbar_wait_slow(bar, parity);
}

// A tensor map that lives in global memory and was written through the
// generic proxy (a host copy into a library-owned table): order that write
// before the TMA unit reads the descriptor (and drop any stale copy the
// tensor-map cache holds for a reused address).
__device__ __forceinline__ void tensormap_acquire(const CUtensorMap *m) {
    asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(reinterpret_cast<uint64_t>(m))
                 : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap *m) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}

// 3-D tiled TMA load of one box into shared memory, completing on `bar`.
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *m, int c0, int c1, int c2,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// L2 cache policy: keep the lines (evict_last) — for a stencil input whose
// planes other CTAs re-read (x/y halos, the z halo of the next chunk) while
// a much larger output stream (.cs stores, evict_first) passes through L2.
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// tma_load_3d with an L2 cache-policy hint.
__device__ __forceinline__ void tma_load_3d_hint(void *dst, const CUtensorMap *m, int c0, int c1, int c2,
                                                 uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// Programmatic dependent launch (PDL): let the next kernel on the stream be
// scheduled before this one finishes / wait until the previous kernel on the
// stream has completed and its memory is visible.  Both are no-ops for a
// kernel launched without the programmatic-serialization attribute.
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait_prerequisites() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Named barrier among `nthreads` threads (id 0 is __syncthreads).
__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__host__ __device__ constexpr int round_up(int a, int b) { return (a + b - 1) / b * b; }

}  // namespace sb
