// Microbenchmark (not product code): can TMA bulk-tensor STORES beat the
// st.global ceiling of config 2's output mix (ten 256^3 fp64 output streams,
// optionally one read stream) that tools/csrc/store_probe.cu measured?
//
// d4_all's pattern: a CTA owns a TX x 4 column tile and a z4 chunk of a
// 256^3 box; per plane each thread (two consecutive x points, like d4_all's
// NP = 2) writes its ten output pairs into a shared staging tile
// [NBUF][10][4][TX], the CTA fences the generic-proxy writes for the async
// proxy, and one thread issues ten cp.async.bulk.tensor.3d stores (box
// TX x 4 x 1, one per output) as one bulk group.  A staging buffer is
// rewritten only after wait_group.read says its previous group has been read.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

struct Maps {
    CUtensorMap m[10];
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tma_store_3d(const CUtensorMap *m, const void *src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void tma_store_3d_hint(const CUtensorMap *m, const void *src, int c0, int c1, int c2,
                                                  uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3, %4}], [%1], %5;" ::"l"(
            reinterpret_cast<uint64_t>(m)),
        "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async_shared() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int TX, int READ, int NBUF, int HINT>
__global__ void __launch_bounds__(TX / 2 * 4) tma_tile_kernel(const double *__restrict__ in,
                                                              const __grid_constant__ Maps M, int nout) {
    constexpr int N = 256, TPR = TX / 2, PLANE = 4 * TX;
    extern __shared__ __align__(128) double sbuf[];   // [NBUF][10][4][TX]
    int t = blockIdx.x;
    const int bx = t % (N / TX);
    t /= N / TX;
    const int by = t % (N / 4);
    const int bz = t / (N / 4);
    const int tid = threadIdx.x, cx = tid % TPR, ry = tid / TPR;
    const int x = bx * TX + 2 * cx, y = by * 4 + ry;
    uint64_t pol = 0;
    if (HINT) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#pragma unroll 1
    for (int zz = 0; zz < 4; ++zz) {
        const int b = zz % NBUF;
        if (zz >= NBUF) {   // buffer b's previous group (plane zz - NBUF) must have been read
            if (tid == 0) bulk_wait_read<NBUF - 1>();
            __syncthreads();
        }
        const int z = bz * 4 + zz;
        const long long off = x + (long long)y * N + (long long)z * N * N;
        double2 v = READ ? __ldcs(reinterpret_cast<const double2 *>(in + off)) : make_double2((double)off, 1.0);
        double *sb = sbuf + b * 10 * PLANE;
#pragma unroll
        for (int k = 0; k < 10; ++k)
            if (k < nout)
                *reinterpret_cast<double2 *>(sb + k * PLANE + ry * TX + 2 * cx) =
                    make_double2(v.x * (k + 1), v.y * (k + 1));
        fence_async_shared();
        __syncthreads();
        if (tid == 0) {
            for (int k = 0; k < nout; ++k) {
                if (HINT) tma_store_3d_hint(&M.m[k], sb + k * PLANE, bx * TX, by * 4, z, pol);
                else tma_store_3d(&M.m[k], sb + k * PLANE, bx * TX, by * 4, z);
            }
            bulk_commit();
        }
    }
    if (tid == 0) bulk_wait_read<0>();   // smem stays valid until the stores have read it
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int TX, int READ, int NBUF, int HINT>
int go(const double *in, const Maps &M, int nout, cudaStream_t s) {
    const int smem = NBUF * 10 * 4 * TX * 8;
    auto fn = tma_tile_kernel<TX, READ, NBUF, HINT>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    fn<<<(256 / TX) * 64 * 64, TX / 2 * 4, smem, s>>>(in, M, nout);
    return (int)cudaGetLastError();
}

template <int TX, int READ>
int go_b(int nbuf, int hint, const double *in, const Maps &M, int nout, cudaStream_t s) {
    if (nbuf == 1) return hint ? go<TX, READ, 1, 1>(in, M, nout, s) : go<TX, READ, 1, 0>(in, M, nout, s);
    if (nbuf == 2) return hint ? go<TX, READ, 2, 1>(in, M, nout, s) : go<TX, READ, 2, 0>(in, M, nout, s);
    return hint ? go<TX, READ, 4, 1>(in, M, nout, s) : go<TX, READ, 4, 0>(in, M, nout, s);
}

}  // namespace

extern "C" int tma_store_probe(int tx, int read, int nbuf, int hint, const double *in, double **outs, int nout,
                               void *stream) {
    static EncodeTiledFn enc = nullptr;
    if (!enc) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess) return -1;
        enc = reinterpret_cast<EncodeTiledFn>(fn);
    }
    Maps M;
    for (int k = 0; k < nout; ++k) {
        cuuint64_t dims[3] = {256, 256, 256};
        cuuint64_t strides[2] = {256 * 8, 256 * 256 * 8};
        cuuint32_t box[3] = {(cuuint32_t)tx, 4, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        if (enc(&M.m[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, outs[k], dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return -2;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (tx == 32) return read ? go_b<32, 1>(nbuf, hint, in, M, nout, s) : go_b<32, 0>(nbuf, hint, in, M, nout, s);
    if (tx == 64) return read ? go_b<64, 1>(nbuf, hint, in, M, nout, s) : go_b<64, 0>(nbuf, hint, in, M, nout, s);
    return read ? go_b<128, 1>(nbuf, hint, in, M, nout, s) : go_b<128, 0>(nbuf, hint, in, M, nout, s);
}
