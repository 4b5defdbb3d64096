// lap7.cu — K1: the reference's 7-point update (stencil.py:31-39) and K0:
// the vlanes 1-D difference kernels (vlanes.py:342-360).
//
// K1 is the config-1 kernel: a 64^3 box is 4.4 MB, L2-resident, so the
// launch is latency-bound; the kernel keeps the z neighbours of its two x
// points in registers while streaming its z chunk and reads the in-plane
// neighbours through L1.  Expression tree (stencil.py:35-39):
//   dst = C0*b + C1*(((xm + xp) + (ym + yp)) + (zm + zp))
#include <algorithm>
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"
#include "internal.h"

namespace sb {

namespace {

// Loads of the source field: through L1 for one sweep per launch; at L2
// (ld.global.cg) for the persistent multi-sweep kernel, whose source was
// written by other SMs since their lines could last sit in this SM's L1.
template <bool CG>
__device__ __forceinline__ double ld1(const double *p) {
    if constexpr (CG) return __ldcg(p);
    else return *p;
}
template <bool CG>
__device__ __forceinline__ double2 ld2(const double *p) {
    if constexpr (CG) return __ldcg(reinterpret_cast<const double2 *>(p));
    else return load_pair(p);
}

// One thread's column segment: two x points (a 16-byte pair) at (x, y),
// planes [z0, z1); z neighbours carried in registers.
template <bool CG>
__device__ __forceinline__ void lap7_column(const Grid &dst, const Grid &src, int x, int y, int z0, int z1, int lo0,
                                            int hi0, int hi1, double c0, double c1) {
    const bool yin = y < hi1;
    const bool m0 = yin && x >= lo0 && x < hi0;
    const bool m1 = yin && x + 1 >= lo0 && x + 1 < hi0;
    if (!(m0 || m1)) return;
    const int xa = m0 ? x : x + 1;   // first active point (single-point edge case)

    double zm[2], cc[2], zp[2];
    const double *pc = src.at(x, y, z0);
    if (m0 && m1) {
        const double2 a = ld2<CG>(pc - src.sz), b = ld2<CG>(pc);
        zm[0] = a.x; zm[1] = a.y; cc[0] = b.x; cc[1] = b.y;
    } else {
        zm[0] = zm[1] = ld1<CG>(src.at(xa, y, z0 - 1));
        cc[0] = cc[1] = ld1<CG>(src.at(xa, y, z0));
    }
    if (m0 && m1) {
        // blocks of ZB planes: every load of a block is issued before its
        // stores (dst may alias src as far as the compiler knows, so loads
        // cannot move past stores on their own) — ZB L2 round trips overlap
        constexpr int ZB = 4;
        for (int zb = z0; zb < z1; zb += ZB) {
            const int nb = min(ZB, z1 - zb);
            double2 vn[ZB], vs[ZB], vt[ZB];
            double vxm[ZB], vxp[ZB];
#pragma unroll
            for (int k = 0; k < ZB; ++k) {
                if (k < nb) {
                    const double *p = src.at(x, y, zb + k);
                    vn[k] = ld2<CG>(p + src.sz);
                    vs[k] = ld2<CG>(p - src.sy);
                    vt[k] = ld2<CG>(p + src.sy);
                    vxm[k] = ld1<CG>(p - 1);
                    vxp[k] = ld1<CG>(p + 2);
                }
            }
#pragma unroll
            for (int k = 0; k < ZB; ++k) {
                if (k < nb) {
                    zp[0] = vn[k].x;
                    zp[1] = vn[k].y;
                    const double xm[2] = {vxm[k], cc[0]}, xp[2] = {cc[1], vxp[k]};
                    const double ym[2] = {vs[k].x, vs[k].y}, yp[2] = {vt[k].x, vt[k].y};
                    double o[2];
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const double nbr = add(add(add(xm[j], xp[j]), add(ym[j], yp[j])), add(zm[j], zp[j]));
                        o[j] = add(mul(c0, cc[j]), mul(c1, nbr));
                    }
                    store_pair(dst.at(x, y, zb + k), o[0], o[1], true, true);
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        zm[j] = cc[j];
                        cc[j] = zp[j];
                    }
                }
            }
        }
        return;
    }
    // single-point edge lane
    for (int z = z0; z < z1; ++z) {
        const double *q = src.at(xa, y, z);
        zp[0] = ld1<CG>(q + src.sz);
        const double nbr = add(add(add(ld1<CG>(q - 1), ld1<CG>(q + 1)), add(ld1<CG>(q - src.sy), ld1<CG>(q + src.sy))),
                               add(zm[0], zp[0]));
        dst.at(xa, y, z)[0] = add(mul(c0, cc[0]), mul(c1, nbr));
        zm[0] = cc[0];
        cc[0] = zp[0];
    }
}

__global__ void __launch_bounds__(256) lap7_kernel(Grid dst, Grid src, int lo0, int lo1, int lo2, int hi0,
                                                   int hi1, int hi2, int ax0, int zc, double c0, double c1) {
    // Programmatic dependent launch: the next sweep of a back-to-back loop may
    // be scheduled now; this one touches memory only once the previous
    // kernel on the stream has completed (a no-op without such a predecessor).
    pdl_launch_dependents();
    pdl_wait_prerequisites();
    const int x = ax0 + (blockIdx.x * 32 + threadIdx.x) * 2;
    const int y = lo1 + blockIdx.y * blockDim.y + threadIdx.y;
    const int z0 = lo2 + blockIdx.z * zc;
    lap7_column<false>(dst, src, x, y, z0, min(z0 + zc, hi2), lo0, hi0, hi1, c0, c1);
}

// Grid-wide barrier of a cooperative (co-resident) launch: a monotone 64-bit
// arrival counter, zeroed before the launch; generation k completes when it
// reaches k * gridDim.x (64 bits: no wrap for any int32 sweep count).
__device__ __forceinline__ void grid_barrier(unsigned long long *ctr, unsigned long long target) {
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        __threadfence();
        atomicAdd(ctr, 1ull);
        unsigned long long v;
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

// Persistent multi-sweep Jacobi (the reference's run_serial loop,
// stencil.py:55-65, on the device): sweep k reads a (k even) or b and writes
// the other; the CTAs walk the same tile grid as lap7_kernel, grid-stride,
// and meet at a grid barrier between sweeps — one launch for all sweeps.
__global__ void __launch_bounds__(256) lap7_iterate_kernel(Grid a, Grid b, int lo0, int lo1, int lo2, int hi0, int hi1,
                                                           int hi2, int ax0, int zc, int gx, int gy, int gz,
                                                           double c0, double c1, int iters, unsigned long long *ctr) {
    const int ntiles = gx * gy * gz;
    for (int it = 0; it < iters; ++it) {
        const Grid &src = (it & 1) ? b : a;
        const Grid &dst = (it & 1) ? a : b;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const int tx = t % gx, ty = (t / gx) % gy, tz = t / (gx * gy);
            const int x = ax0 + (tx * 32 + threadIdx.x) * 2;
            const int y = lo1 + ty * blockDim.y + threadIdx.y;
            const int z0 = lo2 + tz * zc;
            lap7_column<true>(dst, src, x, y, z0, min(z0 + zc, hi2), lo0, hi0, hi1, c0, c1);
        }
        if (it + 1 < iters) grid_barrier(ctr, (unsigned long long)(it + 1) * gridDim.x);
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

// Barrier counters of sb_lap7_iterate: a pool of kCounterPool 64-bit
// counters per device, allocated by sb_init (reserve_barrier_counters) so a
// first call inside a CUDA-graph capture needs no cudaMalloc; a (device,
// stream) pair keeps its slot.  Without sb_init the pool is allocated on
// first use, which is refused while the stream is capturing.
namespace {
constexpr int kCounterPool = 256;
std::mutex g_ctr_mu;
std::map<int, unsigned long long *> g_ctr_pool;                       // device -> pool
std::map<std::pair<int, cudaStream_t>, unsigned long long *> g_ctr;  // (device, stream) -> slot
std::map<int, int> g_ctr_used;

int reserve_locked(int dev) {
    if (g_ctr_pool.count(dev)) return SB_OK;
    unsigned long long *pool = nullptr;
    if (cudaError_t e = cudaMalloc(&pool, kCounterPool * sizeof(unsigned long long)); e != cudaSuccess)
        return check_cuda(e, "barrier counter pool");
    g_ctr_pool[dev] = pool;
    g_ctr_used[dev] = 0;
    return SB_OK;
}
}  // namespace

int release_barrier_counters() {
    std::lock_guard<std::mutex> lock(g_ctr_mu);
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto &kv : g_ctr_pool) {
        cudaSetDevice(kv.first);
        cudaFree(kv.second);   // implicitly waits for the device's work
    }
    cudaSetDevice(cur);
    g_ctr_pool.clear();
    g_ctr.clear();
    g_ctr_used.clear();
    return SB_OK;
}

int reserve_barrier_counters(int dev) {
    std::lock_guard<std::mutex> lock(g_ctr_mu);
    return reserve_locked(dev);
}

int barrier_counter(int dev, cudaStream_t st, unsigned long long **out) {
    std::lock_guard<std::mutex> lock(g_ctr_mu);
    auto it = g_ctr.find({dev, st});
    if (it != g_ctr.end()) {
        *out = it->second;
        return SB_OK;
    }
    if (!g_ctr_pool.count(dev)) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone)
            return fail(SB_USAGE, "lap7_iterate: first use on this device inside a CUDA-graph capture; call sb_init first");
        if (int rc = reserve_locked(dev)) return rc;
    }
    int &used = g_ctr_used[dev];
    if (used >= kCounterPool) return fail(SB_RESOURCE, "lap7_iterate: more than 256 streams per device");
    *out = g_ctr[{dev, st}] = g_ctr_pool[dev] + used++;
    return SB_OK;
}

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
    return launch_pdl(lap7_kernel, grid, block, 0, st, "lap7_kernel launch", grid_of(dst), grid_of(src), sp.lo[0],
                      sp.lo[1], sp.lo[2], sp.hi[0], sp.hi[1], sp.hi[2], ax0, zc, c0, c1);
}

int launch_lap7_iterate(const sb_array &a, const sb_array &b, const sb_space &sp, double c0, double c1, int iters,
                        const sb_launch &p, cudaStream_t st) {
    const int ty = p.tile_y > 0 ? p.tile_y : 8;
    const int zc = p.z_chunk > 0 ? p.z_chunk : 16;
    if (ty > 8 || 32 * ty > 256) return fail(SB_USAGE, "lap7: tile_y must be 1..8");
    if (iters < 0) return fail(SB_USAGE, "lap7_iterate: negative iteration count");
    if (iters == 0) return SB_OK;
    for (int d = 0; d < 3; ++d)
        if (sp.hi[d] <= sp.lo[d]) return SB_OK;
    const int ax0 = (sp.lo[0] >= 0 ? sp.lo[0] / 2 : -((-sp.lo[0] + 1) / 2)) * 2;
    const int pairs = (sp.hi[0] - ax0 + 1) / 2;
    const int gx = (pairs + 31) / 32, gy = (sp.hi[1] - sp.lo[1] + ty - 1) / ty, gz = (sp.hi[2] - sp.lo[2] + zc - 1) / zc;
    const long long ntiles = (long long)gx * gy * gz;
    if (ntiles > 0x7fffffffLL) return fail(SB_RESOURCE, "lap7_iterate: too many tiles");

    // co-resident grid: resident CTAs per SM x SMs (cooperative launch checks it)
    int dev = 0, sms = 0, per_sm = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lap7_iterate_kernel, 32 * ty, 0);
    if (e != cudaSuccess) return check_cuda(e, "lap7_iterate occupancy");
    const int blocks = (int)std::min<long long>(ntiles, (long long)per_sm * sms);

    // one arrival counter per (device, stream), owned by the library and
    // zeroed on the stream: launches on one stream are ordered, so they can
    // share it; launches on different streams may run concurrently and must not
    unsigned long long *ctr_dev = nullptr;
    if (int rc = barrier_counter(dev, st, &ctr_dev)) return rc;
    if ((e = cudaMemsetAsync(ctr_dev, 0, sizeof(unsigned long long), st)) != cudaSuccess)
        return check_cuda(e, "lap7_iterate counter reset");

    Grid ga = grid_of(a), gb = grid_of(b);
    int lo0 = sp.lo[0], lo1 = sp.lo[1], lo2 = sp.lo[2], hi0 = sp.hi[0], hi1 = sp.hi[1], hi2 = sp.hi[2];
    unsigned long long *ctr = ctr_dev;
    void *args[] = {&ga, &gb, &lo0, &lo1, &lo2, &hi0, &hi1, &hi2, (void *)&ax0, (void *)&zc, (void *)&gx,
                    (void *)&gy, (void *)&gz, &c0, &c1, &iters, &ctr};
    e = cudaLaunchCooperativeKernel((const void *)lap7_iterate_kernel, dim3(blocks), dim3(32, ty), args, 0, st);
    return check_cuda(e, "lap7_iterate_kernel launch");
}

int launch_diff1d(int kind, double *dst, const double *src, int n, cudaStream_t st) {
    if (n < 1) return SB_OK;
    const int threads = 128;
    diff1d_kernel<<<(n + threads - 1) / threads, threads, 0, st>>>(kind, dst, src, n);
    return check_cuda(cudaGetLastError(), "diff1d_kernel launch");
}

}  // namespace sb
