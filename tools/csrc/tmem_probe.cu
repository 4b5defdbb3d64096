// TMEM probes for the config-5 (rhs24) phase-B redesign (tools/tmem_probe.py).
//
// Question: can Tensor Memory feed the per-term operand loads of the
// 24 x 64-term polynomial evaluation faster than shared memory (whose
// 128 B/clk per SM binds today's rhs24, K6)?
//
//  * ldtm_bw<N, K>: every warp issues K tcgen05.ld.32x32b.xN per wait::ld —
//    raw TMEM read bandwidth (bytes / clk / SM) by shape and batch size;
//  * phaseb<SRC>: the real phase-B inner loop on 128 points per CTA (lane =
//    point, TMEM lane = point, one output per warp at a time, table entries
//    broadcast from shared memory), with both operands from TMEM (SRC 0),
//    v_p from TMEM and v_q from shared memory (SRC 1), or both from shared
//    memory (SRC 2); outputs are written so the host can check the bits.
// Built with -fmad=false like the product.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tmem_alloc(uint32_t *slot, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void st_x2(uint32_t taddr, uint32_t a, uint32_t b) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void ld_x2(uint32_t taddr, uint32_t &a, uint32_t &b) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "r"(taddr) : "memory");
}
__device__ __forceinline__ void ld_x4(uint32_t taddr, uint32_t (&v)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(taddr)
                 : "memory");
}
__device__ __forceinline__ void ld_x8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr)
                 : "memory");
}
__device__ __forceinline__ double2 lds128(uint32_t a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ double lds64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
// keeps uses of r after the preceding wait::ld (volatile asms are not reordered)
__device__ __forceinline__ void pin(uint32_t &r) { asm volatile("" : "+r"(r)); }

// ---- raw bandwidth ---------------------------------------------------------
template <int N, int K>
__global__ void ldtm_bw_kernel(unsigned long long *out, int iters) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t base = slot + ((uint32_t)(32 * (warp & 3)) << 16);
    uint32_t acc = 0;
    uint32_t col = (warp * 8) & 255;
    for (int it = 0; it < iters; ++it) {
        uint32_t v[K][N];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint32_t a = base + ((col + k * 24) & 255);
            if constexpr (N == 2) ld_x2(a, v[k][0], v[k][1]);
            if constexpr (N == 4) ld_x4(a, *reinterpret_cast<uint32_t(*)[4]>(&v[k][0]));
            if constexpr (N == 8) ld_x8(a, *reinterpret_cast<uint32_t(*)[8]>(&v[k][0]));
        }
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
            for (int n = 0; n < N; ++n) {
                pin(v[k][n]);
                acc ^= v[k][n];
            }
        col += 2;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(slot, 512);
    if (acc == 0x12345678u) out[blockIdx.x] = acc;
}

// ---- does LDTM share the shared-memory data path? -------------------------
// 8 LDS.64 (optional) + K tcgen05.ld.32x32b.x2 per step, integer accumulation
template <int K>
__global__ void ldtm_lds_mix_kernel(unsigned long long *out, int iters, int with_lds) {
    __shared__ uint32_t slot;
    __shared__ double buf[4096];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = i;
    if (warp == 0) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t base = slot + ((uint32_t)(32 * (warp & 3)) << 16);
    unsigned long long s = 0;
    uint32_t acc = 0;
    int b = (warp * 32) % 2048;
    for (int it = 0; it < iters; ++it) {
        if (with_lds) {
#pragma unroll
            for (int k = 0; k < 8; ++k) s ^= __double_as_longlong(buf[((b + k * 256) & 2047) + lane]);
            b += 32;
        }
        if constexpr (K > 0) {
            uint32_t v[K][2];
#pragma unroll
            for (int k = 0; k < K; ++k) ld_x2(base + ((it * 2 + k * 24) & 255), v[k][0], v[k][1]);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < K; ++k) {
                pin(v[k][0]);
                pin(v[k][1]);
                acc ^= v[k][0] ^ v[k][1];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(slot, 512);
    if ((s ^ acc) == 0x12345678u) out[blockIdx.x] = s ^ acc;
}

// ---- phase-B loop ------------------------------------------------------------
constexpr int NOPS = 240, NOUT = 24, NTERM = 64, NPTS = 128, NSM_OPS = 112;

struct Term {
    double c;
    uint32_t p, q;   // operand indices
};

// SRC 0: p, q from TMEM; 1: p from TMEM, q from smem; 2: both from smem (p, q < NSM_OPS)
template <int SRC, int NW>
__global__ void __launch_bounds__(NW * 32, 1)
    phaseb_kernel(const double *ops /*[NOPS][NPTS]*/, const Term *table /*[NOUT][NTERM]*/, double *out /*[NOUT][NPTS]*/,
                  int reps) {
    extern __shared__ __align__(1024) unsigned char smem[];
    uint32_t *slot = reinterpret_cast<uint32_t *>(smem);
    Term *tt = reinterpret_cast<Term *>(smem + 128);
    double *sv = reinterpret_cast<double *>(smem + 128 + sizeof(Term) * NOUT * NTERM);   // [NSM_OPS][NPTS]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, sp = warp & 3;
    const int pt = 32 * sp + lane;
    if (warp == 0) tmem_alloc(slot, 512);
    for (int e = threadIdx.x; e < NOUT * NTERM; e += NW * 32) tt[e] = table[e];
    if constexpr (SRC > 0)
        for (int e = threadIdx.x; e < NSM_OPS * NPTS; e += NW * 32) sv[e] = ops[e];
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = *slot;
    const uint32_t lanebits = tb + ((uint32_t)(32 * sp) << 16);
    // warps of subpartition sp fill its 32 lanes: operand j -> columns 2j, 2j+1
    if constexpr (SRC < 2) {
        for (int j = warp >> 2; j < NOPS; j += NW / 4) {
            const double v = ops[j * NPTS + pt];
            st_x2(lanebits + 2 * j, (uint32_t)__double_as_longlong(v), (uint32_t)(__double_as_longlong(v) >> 32));
        }
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    const char *svb = reinterpret_cast<const char *>(sv) + 8 * pt;
    for (int r = 0; r < reps; ++r) {
        for (int o = warp >> 2; o < NOUT; o += NW / 4) {
            const Term *T = tt + o * NTERM;
            double acc = 0.0;
#pragma unroll 1
            for (int g = 0; g < NTERM; g += 8) {
                double cf[8], vp[8], vq[8];
                uint32_t lo[16], hi[16];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const Term t = T[g + k];
                    cf[k] = t.c;
                    if constexpr (SRC < 2) ld_x2(lanebits + 2 * t.p, lo[2 * k], hi[2 * k]);
                    else vp[k] = lds64(smem_u32(svb + t.p * (NPTS * 8)));
                    if constexpr (SRC == 0) ld_x2(lanebits + 2 * t.q, lo[2 * k + 1], hi[2 * k + 1]);
                    else vq[k] = lds64(smem_u32(svb + t.q * (NPTS * 8)));
                }
                if constexpr (SRC < 2) {
                    tmem_wait_ld();
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        pin(lo[2 * k]);
                        pin(hi[2 * k]);
                        vp[k] = __hiloint2double((int)hi[2 * k], (int)lo[2 * k]);
                        if constexpr (SRC == 0) {
                            pin(lo[2 * k + 1]);
                            pin(hi[2 * k + 1]);
                            vq[k] = __hiloint2double((int)hi[2 * k + 1], (int)lo[2 * k + 1]);
                        }
                    }
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const double t = __dmul_rn(__dmul_rn(cf[k], vp[k]), vq[k]);
                    acc = (g == 0 && k == 0) ? t : __dadd_rn(acc, t);
                }
            }
            if (r == reps - 1) out[o * NPTS + pt] = acc;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 512);
}

// Two points per lane (SRC 3: v_p by tcgen05.ld.32x32b.x4 from TMEM, whose
// lanes hold points 2l, 2l+1 of a 64-point group in columns 4j..4j+3; v_q by
// LDS.128 from [NSM_OPS][NPTS]; SRC 4: both by LDS.128).  Subpartition sp
// serves point group sp & 1 (lanes 64-127 replicate lanes 0-63).
constexpr int NTM_OPS = 128;
template <int SRC, int NW>
__global__ void __launch_bounds__(NW * 32, 1)
    phaseb2_kernel(const double *ops, const Term *table, double *out, int reps) {
    extern __shared__ __align__(1024) unsigned char smem[];
    uint32_t *slot = reinterpret_cast<uint32_t *>(smem);
    Term *tt = reinterpret_cast<Term *>(smem + 128);
    double *sv = reinterpret_cast<double *>(smem + 128 + sizeof(Term) * NOUT * NTERM);   // [NSM_OPS][NPTS]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, sp = warp & 3;
    const int pt = 64 * (sp & 1) + 2 * lane;
    if (warp == 0) tmem_alloc(slot, 512);
    for (int e = threadIdx.x; e < NOUT * NTERM; e += NW * 32) tt[e] = table[e];
    for (int e = threadIdx.x; e < NSM_OPS * NPTS; e += NW * 32) sv[e] = ops[e];
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = *slot;
    const uint32_t lanebits = tb + ((uint32_t)(32 * sp) << 16);
    if constexpr (SRC == 3) {
        for (int j = warp >> 2; j < NTM_OPS; j += NW / 4) {
            const unsigned long long a = __double_as_longlong(ops[j * NPTS + pt]);
            const unsigned long long b = __double_as_longlong(ops[j * NPTS + pt + 1]);
            asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(lanebits + 4 * j),
                         "r"((uint32_t)a), "r"((uint32_t)(a >> 32)), "r"((uint32_t)b), "r"((uint32_t)(b >> 32))
                         : "memory");
        }
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t svb = smem_u32(sv) + 8 * pt;
    const int grp = NW / 2;   // warps per point group
    for (int r = 0; r < reps; ++r) {
        for (int o = warp >> 1; o < NOUT; o += grp) {
            const Term *T = tt + o * NTERM;
            double a0 = 0.0, a1 = 0.0;
#pragma unroll 1
            for (int g = 0; g < NTERM; g += 8) {
                double cf[8];
                double2 vp[8], vq[8];
                uint32_t w[8][4];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const Term t = T[g + k];
                    cf[k] = t.c;
                    if constexpr (SRC == 3) ld_x4(lanebits + 4 * t.p, w[k]);
                    else vp[k] = lds128(svb + t.p * (NPTS * 8));
                    vq[k] = lds128(svb + t.q * (NPTS * 8));
                }
                if constexpr (SRC == 3) {
                    tmem_wait_ld();
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
#pragma unroll
                        for (int n = 0; n < 4; ++n) pin(w[k][n]);
                        vp[k].x = __hiloint2double((int)w[k][1], (int)w[k][0]);
                        vp[k].y = __hiloint2double((int)w[k][3], (int)w[k][2]);
                    }
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const double t0 = __dmul_rn(__dmul_rn(cf[k], vp[k].x), vq[k].x);
                    const double t1 = __dmul_rn(__dmul_rn(cf[k], vp[k].y), vq[k].y);
                    a0 = (g == 0 && k == 0) ? t0 : __dadd_rn(a0, t0);
                    a1 = (g == 0 && k == 0) ? t1 : __dadd_rn(a1, t1);
                }
            }
            if (r == reps - 1 && (sp >> 1) == 0) {
                out[o * NPTS + pt] = a0;
                out[o * NPTS + pt + 1] = a1;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 512);
}

template <int SRC, int NW>
int phaseb2_launch_t(const double *ops, const Term *table, double *out, int blocks, int reps, cudaStream_t st) {
    const size_t smem = 128 + sizeof(Term) * NOUT * NTERM + sizeof(double) * NSM_OPS * NPTS;
    cudaFuncSetAttribute(phaseb2_kernel<SRC, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    phaseb2_kernel<SRC, NW><<<blocks, NW * 32, smem, st>>>(ops, table, out, reps);
    return (int)cudaGetLastError();
}

// SRC 5 — the configuration a 64-point config-5 phase B would use: 64 points
// per CTA, two per lane (a warp covers the tile), ONE output per warp at a
// time; operands 0..127 in TMEM (columns 4j..4j+3 hold points 2l, 2l+1 of
// lane l, replicated in all four subpartitions), operands 128..239 in shared
// memory ([112][64], LDS.128); the term table packed as in rhs24.cu (eight
// terms per five 16-byte words, broadcast reads) with p, q in 0..239 — every
// operand comes from TMEM or shared memory by a warp-uniform branch.
constexpr int NPT5 = 64, NSM5 = NOPS - NTM_OPS;
template <int NW>
__global__ void __launch_bounds__(NW * 32, 1)
    phaseb5_kernel(const double *ops /*[NOPS][NPT5]*/, const uint4 *table /*[NOUT][40]*/, double *out, int reps) {
    extern __shared__ __align__(1024) unsigned char smem[];
    uint32_t *slot = reinterpret_cast<uint32_t *>(smem);
    uint4 *tt = reinterpret_cast<uint4 *>(smem + 128);
    double *sv = reinterpret_cast<double *>(smem + 128 + sizeof(uint4) * NOUT * 40);   // [NSM5][NPT5]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, sp = warp & 3;
    const int pt = 2 * lane;
    if (warp == 0) tmem_alloc(slot, 512);
    for (int e = threadIdx.x; e < NOUT * 40; e += NW * 32) tt[e] = table[e];
    for (int e = threadIdx.x; e < NSM5 * NPT5; e += NW * 32) sv[e] = ops[NTM_OPS * NPT5 + e];
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = *slot;
    const uint32_t lanebits = tb + ((uint32_t)(32 * sp) << 16);
    for (int j = warp >> 2; j < NTM_OPS; j += NW / 4) {
        const unsigned long long a = __double_as_longlong(ops[j * NPT5 + pt]);
        const unsigned long long b = __double_as_longlong(ops[j * NPT5 + pt + 1]);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(lanebits + 4 * j),
                     "r"((uint32_t)a), "r"((uint32_t)(a >> 32)), "r"((uint32_t)b), "r"((uint32_t)(b >> 32))
                     : "memory");
    }
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t svb = smem_u32(sv) + 8 * pt - NTM_OPS * (NPT5 * 8);
    for (int r = 0; r < reps; ++r) {
        for (int o = warp; o < NOUT; o += NW) {
            const uint4 *T = tt + o * 40;
            double a0 = 0.0, a1 = 0.0;
#pragma unroll 1
            for (int g = 0; g < 8; ++g) {
                const double2 c01 = *reinterpret_cast<const double2 *>(T + 5 * g);
                const double2 c23 = *reinterpret_cast<const double2 *>(T + 5 * g + 1);
                const double2 c45 = *reinterpret_cast<const double2 *>(T + 5 * g + 2);
                const double2 c67 = *reinterpret_cast<const double2 *>(T + 5 * g + 3);
                const uint4 w = T[5 * g + 4];
                const double cf[8] = {c01.x, c01.y, c23.x, c23.y, c45.x, c45.y, c67.x, c67.y};
                const uint32_t pq[8] = {w.x & 0xffffu, w.x >> 16, w.y & 0xffffu, w.y >> 16,
                                        w.z & 0xffffu, w.z >> 16, w.w & 0xffffu, w.w >> 16};
                uint32_t tw[16][4];
                double2 v[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const uint32_t op = (k & 1) ? (pq[k >> 1] >> 8) : (pq[k >> 1] & 0xffu);
                    if (op < NTM_OPS) ld_x4(lanebits + 4 * op, tw[k]);
                    else v[k] = lds128(svb + op * (NPT5 * 8));
                }
                tmem_wait_ld();
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const uint32_t op = (k & 1) ? (pq[k >> 1] >> 8) : (pq[k >> 1] & 0xffu);
#pragma unroll
                    for (int n = 0; n < 4; ++n) pin(tw[k][n]);
                    if (op < NTM_OPS) {
                        v[k].x = __hiloint2double((int)tw[k][1], (int)tw[k][0]);
                        v[k].y = __hiloint2double((int)tw[k][3], (int)tw[k][2]);
                    }
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const double t0 = __dmul_rn(__dmul_rn(cf[k], v[2 * k].x), v[2 * k + 1].x);
                    const double t1 = __dmul_rn(__dmul_rn(cf[k], v[2 * k].y), v[2 * k + 1].y);
                    a0 = (g == 0 && k == 0) ? t0 : __dadd_rn(a0, t0);
                    a1 = (g == 0 && k == 0) ? t1 : __dadd_rn(a1, t1);
                }
            }
            if (r == reps - 1 && sp == 0) {
                out[o * NPT5 + pt] = a0;
                out[o * NPT5 + pt + 1] = a1;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 512);
}

template <int NW>
int phaseb5_launch_t(const double *ops, const uint4 *table, double *out, int blocks, int reps, cudaStream_t st) {
    const size_t smem = 128 + sizeof(uint4) * NOUT * 40 + sizeof(double) * NSM5 * NPT5;
    cudaFuncSetAttribute(phaseb5_kernel<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    phaseb5_kernel<NW><<<blocks, NW * 32, smem, st>>>(ops, table, out, reps);
    return (int)cudaGetLastError();
}

template <int SRC, int NW>
int phaseb_launch_t(const double *ops, const Term *table, double *out, int blocks, int reps, cudaStream_t st) {
    const size_t smem = 128 + sizeof(Term) * NOUT * NTERM + (SRC > 0 ? sizeof(double) * NSM_OPS * NPTS : 0);
    cudaFuncSetAttribute(phaseb_kernel<SRC, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    phaseb_kernel<SRC, NW><<<blocks, NW * 32, smem, st>>>(ops, table, out, reps);
    return (int)cudaGetLastError();
}

}  // namespace

extern "C" {

int ldtm_launch(int n, int k, unsigned long long *out, int blocks, int threads, int iters, void *st) {
    cudaStream_t s = (cudaStream_t)st;
#define L(N, K)                                                                    \
    if (n == N && k == K) {                                                        \
        ldtm_bw_kernel<N, K><<<blocks, threads, 0, s>>>(out, iters);               \
        return (int)cudaGetLastError();                                            \
    }
    L(2, 4) L(2, 8) L(2, 16) L(4, 4) L(4, 8) L(8, 4) L(8, 8)
#undef L
    return -1;
}

int phaseb_launch(int src, int nw, const double *ops, const void *table, double *out, int blocks, int reps, void *st) {
    cudaStream_t s = (cudaStream_t)st;
    const Term *t = (const Term *)table;
#define P(S, W) \
    if (src == S && nw == W) return phaseb_launch_t<S, W>(ops, t, out, blocks, reps, s);
    P(0, 4) P(0, 8) P(0, 12) P(0, 16) P(1, 8) P(1, 12) P(1, 16) P(2, 8) P(2, 12) P(2, 16)
#undef P
#define P(S, W) \
    if (src == S && nw == W) return phaseb2_launch_t<S, W>(ops, t, out, blocks, reps, s);
    P(3, 8) P(3, 16) P(3, 24) P(4, 8) P(4, 16) P(4, 24)
#undef P
    if (src == 5) {
        const uint4 *t5 = (const uint4 *)table;
        if (nw == 8) return phaseb5_launch_t<8>(ops, t5, out, blocks, reps, s);
        if (nw == 12) return phaseb5_launch_t<12>(ops, t5, out, blocks, reps, s);
        if (nw == 16) return phaseb5_launch_t<16>(ops, t5, out, blocks, reps, s);
        if (nw == 24) return phaseb5_launch_t<24>(ops, t5, out, blocks, reps, s);
    }
    return -1;
}

int mix_launch(int k, int with_lds, unsigned long long *out, int blocks, int threads, int iters, void *st) {
    cudaStream_t s = (cudaStream_t)st;
    if (k == 0) ldtm_lds_mix_kernel<0><<<blocks, threads, 0, s>>>(out, iters, with_lds);
    else if (k == 4) ldtm_lds_mix_kernel<4><<<blocks, threads, 0, s>>>(out, iters, with_lds);
    else if (k == 8) ldtm_lds_mix_kernel<8><<<blocks, threads, 0, s>>>(out, iters, with_lds);
    else return -1;
    return (int)cudaGetLastError();
}

int last_error() { return (int)cudaDeviceSynchronize(); }
}
