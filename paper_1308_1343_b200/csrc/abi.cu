// abi.cu — extern "C" entry points of libstencil_b200.so (include/stencil_b200.h).
//
// Validation mirrors the reference's contract checks: inverted index spaces
// and bad shapes are usage errors (traverse.py:36-42 raises UsageError), as
// are geometry violations of the device layout (alignment, ghost width).
// Resource limits (shared memory, boxes per launch) are ResourceError-class.
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace sb {

namespace {
thread_local std::string t_last_error;

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn g_encode = nullptr;
std::once_flag g_encode_once;

void resolve_encode() {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
        g_encode = reinterpret_cast<EncodeTiledFn>(fn);
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Geometry contract of an sb_array; `need_ghost` is the stencil radius read.
int check_array(const sb_array &a, int need_ghost, const char *name) {
    char buf[256];
    if (!a.origin) {
        snprintf(buf, sizeof buf, "%s: null origin", name);
        return fail(SB_USAGE, buf);
    }
    if (!aligned16(a.origin) || (a.sy & 1) || (a.sz & 1) || (a.xpad & 1)) {
        snprintf(buf, sizeof buf, "%s: origin must be 16-byte aligned and sy, sz, xpad even", name);
        return fail(SB_USAGE, buf);
    }
    if (a.nx < 0 || a.ny < 0 || a.nz < 0 || a.ghost < 0 || a.xpad < a.ghost) {
        snprintf(buf, sizeof buf, "%s: negative extent or xpad < ghost", name);
        return fail(SB_USAGE, buf);
    }
    if (a.sy < (int64_t)a.xpad + a.nx + a.ghost || a.sz < a.sy * (int64_t)(a.ny + 2 * a.ghost)) {
        snprintf(buf, sizeof buf, "%s: strides too small for extents", name);
        return fail(SB_USAGE, buf);
    }
    if (a.ghost < need_ghost) {
        snprintf(buf, sizeof buf, "%s: ghost width %d < stencil radius %d", name, a.ghost, need_ghost);
        return fail(SB_USAGE, buf);
    }
    return SB_OK;
}

int check_space(const sb_space &s, const sb_array &a, const char *name) {
    char buf[256];
    const int n[3] = {a.nx, a.ny, a.nz};
    for (int d = 0; d < 3; ++d) {
        if (s.hi[d] < s.lo[d]) {
            snprintf(buf, sizeof buf, "%s: index space with inverted bounds in dim %d", name, d);
            return fail(SB_USAGE, buf);
        }
        if (s.hi[d] > s.lo[d] && (s.lo[d] < 0 || s.hi[d] > n[d])) {
            snprintf(buf, sizeof buf, "%s: index space [%d,%d) outside interior 0..%d in dim %d", name, s.lo[d],
                     s.hi[d], n[d], d);
            return fail(SB_USAGE, buf);
        }
    }
    return SB_OK;
}

cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace

int fail(int code, const std::string &msg) {
    t_last_error = msg;
    return code;
}

int check_cuda(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return SB_OK;
    t_last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return SB_CUDA;
}

int make_tmap(CUtensorMap *m, const sb_array &a, int bx, int by, int bz) {
    std::call_once(g_encode_once, resolve_encode);
    if (!g_encode) return fail(SB_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
    // The driver-API encoder needs a current context.  A host thread whose
    // first CUDA call this is (e.g. a worker thread of the reference's
    // execute_plan / run_static, traverse.py:162-260) has none until the
    // runtime binds the current device's primary context: do that once per
    // thread (cudaSetDevice binds it on later device switches).
    thread_local bool t_bound = false;
    if (!t_bound) {
        if (int rc = check_cuda(cudaFree(nullptr), "bind the primary context to this thread")) return rc;
        t_bound = true;
    }
    double *base = a.origin - a.xpad - (int64_t)a.ghost * a.sy - (int64_t)a.ghost * a.sz;
    if (!aligned16(base)) return fail(SB_USAGE, "TMA base (row start of the first ghost row) not 16-byte aligned");
    cuuint64_t dims[3] = {(cuuint64_t)a.sy, (cuuint64_t)(a.ny + 2 * a.ghost), (cuuint64_t)(a.nz + 2 * a.ghost)};
    cuuint64_t strides[2] = {(cuuint64_t)a.sy * 8, (cuuint64_t)a.sz * 8};
    cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)bz};
    cuuint32_t estr[3] = {1, 1, 1};
#ifndef SB_TMA_L2_PROMOTION
// 128-byte L2 promotion: a staged row (TX + 4 doubles) is 288 bytes for the
// default 32-wide tiles, so 256-byte granules over-fetch at row ends
// (level Laplacian -0.5 %, the other kernels unchanged:
// profiles/r01/v16_ab_l2_policy.log)
#define SB_TMA_L2_PROMOTION CU_TENSOR_MAP_L2_PROMOTION_L2_128B
#endif
    CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, SB_TMA_L2_PROMOTION,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        char buf[160];
        snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (%d) for box %dx%dx%d", (int)r, bx, by, bz);
        return fail(SB_CUDA, buf);
    }
    return SB_OK;
}

namespace {
struct SmemLimit {
    const void *fn;
    int device, bytes;
};
std::mutex g_smem_mutex;
std::vector<SmemLimit> g_smem_limits;
}  // namespace

int ensure_smem_limit(const void *fn, int bytes, const char *what) {
    int dev = 0;
    int rc = check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    if (rc) return rc;
    std::lock_guard<std::mutex> lock(g_smem_mutex);
    for (const SmemLimit &l : g_smem_limits)
        if (l.fn == fn && l.device == dev && l.bytes >= bytes) return SB_OK;
    rc = check_cuda(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), what);
    if (rc) return rc;
    g_smem_limits.push_back({fn, dev, bytes});
    return SB_OK;
}

}  // namespace sb

using namespace sb;

extern "C" {

int sb_abi_version(void) { return SB_ABI_VERSION; }

const char *sb_last_error(void) { return t_last_error.c_str(); }

int sb_init(int device) {
    int rc = check_cuda(cudaSetDevice(device), "cudaSetDevice");
    if (rc) return rc;
    if ((rc = check_cuda(cudaFree(nullptr), "context init"))) return rc;
    return reserve_barrier_counters(device);
}

int sb_enable_peer_access(int peer) {
    int dev = 0;
    if (int rc = check_cuda(cudaGetDevice(&dev), "cudaGetDevice")) return rc;
    if (peer == dev) return SB_OK;
    int can = 0;
    if (int rc = check_cuda(cudaDeviceCanAccessPeer(&can, dev, peer), "cudaDeviceCanAccessPeer")) return rc;
    if (!can) return fail(SB_RESOURCE, "enable_peer_access: the current device cannot access the peer device");
    cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();   // clear the sticky-free "already enabled" status
        return SB_OK;
    }
    return check_cuda(e, "cudaDeviceEnablePeerAccess");
}

int sb_get_device_info(sb_device_info *info) {
    if (!info) return fail(SB_USAGE, "null info");
    int dev = 0;
    int rc = check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    if (rc) return rc;
    cudaDeviceProp p;
    rc = check_cuda(cudaGetDeviceProperties(&p, dev), "cudaGetDeviceProperties");
    if (rc) return rc;
    info->device = dev;
    info->sm_count = p.multiProcessorCount;
    info->cc_major = p.major;
    info->cc_minor = p.minor;
    info->l2_bytes = p.l2CacheSize;
    info->smem_optin_bytes = (int64_t)p.sharedMemPerBlockOptin;
    info->global_mem_bytes = (int64_t)p.totalGlobalMem;
    return SB_OK;
}

int sb_diff1d(int32_t kind, double *dst, const double *src, int32_t n, void *stream) {
    if (kind != 0 && kind != 1) return fail(SB_USAGE, "diff1d: kind must be 0 (forward) or 1 (centered)");
    if (n < 0) return fail(SB_USAGE, "diff1d: negative length");
    if (n > 0 && (!dst || !src)) return fail(SB_USAGE, "diff1d: null pointer");
    return launch_diff1d(kind, dst, src, n, as_stream(stream));
}

int sb_lap7(sb_array dst, sb_array src, sb_space space, double c0, double c1, sb_launch p, void *stream) {
    int rc;
    if ((rc = check_array(src, 1, "lap7 src")) || (rc = check_array(dst, 0, "lap7 dst"))) return rc;
    if ((rc = check_space(space, src, "lap7")) || (rc = check_space(space, dst, "lap7 dst"))) return rc;
    return launch_lap7(dst, src, space, c0, c1, p, as_stream(stream));
}

int sb_lap7_iterate(sb_array a, sb_array b, sb_space space, double c0, double c1, int32_t iters, sb_launch p,
                    void *stream) {
    int rc;
    if ((rc = check_array(a, 1, "lap7_iterate a")) || (rc = check_array(b, 1, "lap7_iterate b"))) return rc;
    if ((rc = check_space(space, a, "lap7_iterate")) || (rc = check_space(space, b, "lap7_iterate b"))) return rc;
    if (a.origin == b.origin) return fail(SB_USAGE, "lap7_iterate: a and b must be different grids");
    return launch_lap7_iterate(a, b, space, c0, c1, iters, p, as_stream(stream));
}

namespace {
int all10_job(const char *nm, const sb_array *out, const sb_array &src, const sb_space &space, D4Job &job) {
    int rc;
    if (!out) return fail(SB_USAGE, "all outputs: null output table");
    if ((rc = check_array(src, 2, nm)) || (rc = check_space(space, src, nm))) return rc;
    memset(&job, 0, sizeof(job));
    job.src = src;
    job.space = space;
    for (int i = 0; i < SB_N_D4_OUT; ++i) {
        if ((rc = check_array(out[i], 0, nm)) || (rc = check_space(space, out[i], nm)))
            return rc;
        job.g[i] = out[i];
    }
    return SB_OK;
}

int all10(int mode, const char *nm, const sb_array *out, sb_array src, sb_space space, sb_d4_constants k,
          sb_launch p, void *stream) {
    D4Job job;
    if (int rc = all10_job(nm, out, src, space, job)) return rc;
    return launch_d4(mode, &job, 1, k, 0.0, p, as_stream(stream));
}

int all10_boxes(int mode, const char *nm, const sb_d4_all_job *jobs, int32_t njobs, sb_d4_constants k, sb_launch p,
                void *stream) {
    if (njobs == 0) return SB_OK;
    if (!jobs || njobs < 0) return fail(SB_USAGE, "all outputs over boxes: bad job table");
    std::vector<D4Job> dj(njobs);
    for (int j = 0; j < njobs; ++j)
        if (int rc = all10_job(nm, jobs[j].out, jobs[j].src, jobs[j].space, dj[j])) return rc;
    return launch_d4(mode, dj.data(), njobs, k, 0.0, p, as_stream(stream));
}

// The D4Job of one RK4 stage (mode, the stage's pointwise coefficient).
int rk_job(int32_t stage, const sb_rk4_fields *f, const sb_space &space, const sb_rk4_constants &c, D4Job &job,
           int &mode, double &ca) {
    if (!f) return fail(SB_USAGE, "rk4_stage: null fields");
    if (stage < 1 || stage > 4) return fail(SB_USAGE, "rk4_stage: stage must be 1..4");
    int rc;
    if ((rc = check_array(f->phi_s, 2, "rk4 phi_s")) || (rc = check_space(space, f->phi_s, "rk4"))) return rc;
    const sb_array *pw[] = {&f->pi_s, &f->phi0, &f->pi0, &f->acc_phi, &f->acc_pi, &f->phi_out, &f->pi_out};
    for (const sb_array *a : pw) {
        if (stage == 1 && (a == &f->pi_s || a == &f->phi0)) continue;
        if ((rc = check_array(*a, 0, "rk4 field")) || (rc = check_space(space, *a, "rk4 field"))) return rc;
    }
    memset(&job, 0, sizeof(job));
    job.src = f->phi_s;
    job.space = space;
    job.g[0] = f->phi_out;
    job.g[1] = f->pi_out;
    job.g[2] = f->acc_phi;
    job.g[3] = f->acc_pi;
    if (stage == 1) {
        job.g[4] = f->pi0;
        mode = D4_RK1;
        ca = c.half_dt;
    } else if (stage == 2) {
        job.g[4] = f->pi_s;
        job.g[5] = f->phi0;
        job.g[6] = f->pi0;
        job.g[7] = f->acc_pi;
        mode = D4_RK2;
        ca = c.half_dt;
    } else {
        job.g[4] = f->pi_s;
        job.g[5] = f->phi0;
        job.g[6] = f->pi0;
        job.g[7] = f->acc_phi;
        job.g[8] = f->acc_pi;
        mode = stage == 4 ? D4_RK4 : D4_RK23;
        ca = stage == 3 ? c.dt : c.dt6;
    }
    return SB_OK;
}

}  // namespace

int sb_d4_all(const sb_array *out, sb_array src, sb_space space, sb_d4_constants k, sb_launch p, void *stream) {
    return all10(D4_ALL10, "d4_all", out, src, space, k, p, stream);
}

int sb_d2_all(const sb_array *out, sb_array src, sb_space space, sb_d4_constants k, sb_launch p, void *stream) {
    return all10(D2_ALL10, "d2_all", out, src, space, k, p, stream);
}

int sb_d4_all_boxes(const sb_d4_all_job *jobs, int32_t njobs, sb_d4_constants k, sb_launch p, void *stream) {
    return all10_boxes(D4_ALL10, "d4_all_boxes", jobs, njobs, k, p, stream);
}

int sb_d2_all_boxes(const sb_d4_all_job *jobs, int32_t njobs, sb_d4_constants k, sb_launch p, void *stream) {
    return all10_boxes(D2_ALL10, "d2_all_boxes", jobs, njobs, k, p, stream);
}

int sb_lap4_boxes(const sb_box_job *jobs, int32_t njobs, sb_d4_constants k, sb_launch p, void *stream) {
    if (njobs == 0) return SB_OK;
    if (!jobs || njobs < 0) return fail(SB_USAGE, "lap4_boxes: bad job table");
    std::vector<D4Job> dj(njobs);
    int rc;
    for (int j = 0; j < njobs; ++j) {
        if ((rc = check_array(jobs[j].src, 2, "lap4 src")) || (rc = check_array(jobs[j].dst, 0, "lap4 dst")))
            return rc;
        if ((rc = check_space(jobs[j].space, jobs[j].src, "lap4")) ||
            (rc = check_space(jobs[j].space, jobs[j].dst, "lap4 dst")))
            return rc;
        memset(&dj[j], 0, sizeof(D4Job));
        dj[j].src = jobs[j].src;
        dj[j].space = jobs[j].space;
        dj[j].g[0] = jobs[j].dst;
    }
    return launch_d4(D4_LAP4, dj.data(), njobs, k, 0.0, p, as_stream(stream));
}

int sb_rk4_stage_boxes(int32_t stage, const sb_rk4_box_job *jobs, int32_t njobs, sb_rk4_constants c, sb_launch p,
                       void *stream) {
    if (njobs == 0) return SB_OK;
    if (!jobs || njobs < 0) return fail(SB_USAGE, "rk4_stage_boxes: bad job table");
    if (p.flags & SB_LAUNCH_PERIODIC_GHOSTS)
        return fail(SB_USAGE, "rk4_stage_boxes: the periodic ghost refresh is for one periodic box (sb_rk4_stage)");
    std::vector<D4Job> dj(njobs);
    int mode = 0;
    double ca = 0;
    for (int j = 0; j < njobs; ++j)
        if (int rc = rk_job(stage, &jobs[j].f, jobs[j].space, c, dj[j], mode, ca)) return rc;
    return launch_d4(mode, dj.data(), njobs, c.lap, ca, p, as_stream(stream));
}

int sb_release_tables(void) { return release_box_tables(); }

int sb_shutdown(void) {
    int rc = release_box_tables();
    int rc2 = release_barrier_counters();
    return rc ? rc : rc2;
}

int sb_ghost_periodic(sb_array a, void *stream) {
    int rc = check_array(a, 0, "ghost_periodic");
    if (rc) return rc;
    return launch_ghost_periodic(a, as_stream(stream));
}

int sb_rk4_stage(int32_t stage, const sb_rk4_fields *f, sb_space space, sb_rk4_constants c, sb_launch p,
                 void *stream) {
    return sb_rk4_stage_zslab(stage, f, space, c, p, nullptr, stream);
}

int sb_rk4_stage_zslab(int32_t stage, const sb_rk4_fields *f, sb_space space, sb_rk4_constants c, sb_launch p,
                       const sb_zslab *zs, void *stream) {
    D4Job job;
    int mode = 0;
    double ca = 0;
    if (int rc = rk_job(stage, f, space, c, job, mode, ca)) return rc;
    if (zs && ((zs->lo_phi_out && !aligned16(zs->lo_phi_out)) || (zs->hi_phi_out && !aligned16(zs->hi_phi_out))))
        return fail(SB_USAGE, "rk4_stage_zslab: peer origins must be 16-byte aligned");
    return launch_d4(mode, &job, 1, c.lap, ca, p, as_stream(stream), zs);
}

int sb_rk4_pair(int32_t pair, const sb_rk4_fields *f, sb_space space, sb_rk4_constants c, sb_launch p,
                void *stream) {
    return sb_rk4_pair_zslab(pair, f, space, c, p, nullptr, stream);
}

int sb_rk4_pair_zslab(int32_t pair, const sb_rk4_fields *f, sb_space space, sb_rk4_constants c, sb_launch p,
                      const sb_zslab *zs, void *stream) {
    if (!f) return fail(SB_USAGE, "rk4_pair: null fields");
    if (pair < 1 || pair > 4)
        return fail(SB_USAGE, "rk4_pair: pair must be 1/2 (stages 1+2 / 3+4) or 3/4 (Laplacian pairs)");
    sb_array halo[4], tile[3], out[4];
    int nh, nt, no;
    if (pair == 3) {
        halo[0] = f->phi0;
        halo[1] = f->pi0;
        nh = 2;
        nt = 0;
        out[0] = f->phi_out;   // L1
        out[1] = f->pi_out;    // L2
        no = 2;
    } else if (pair == 4) {
        halo[0] = f->phi0;
        halo[1] = f->pi0;
        halo[2] = f->phi_s;    // L1
        halo[3] = f->pi_s;     // L2
        nh = 4;
        nt = 0;
        out[0] = f->phi_out;
        out[1] = f->pi_out;
        no = 2;
    } else if (pair == 1) {
        halo[0] = f->phi0;
        halo[1] = f->pi0;
        nh = 2;
        nt = 0;
        out[0] = f->phi_out;
        out[1] = f->pi_out;
        out[2] = f->acc_phi;
        out[3] = f->acc_pi;
        no = 4;
    } else {
        halo[0] = f->phi_s;
        halo[1] = f->phi0;
        halo[2] = f->pi_s;
        nh = 3;
        tile[0] = f->pi0;
        tile[1] = f->acc_phi;
        tile[2] = f->acc_pi;
        nt = 3;
        out[0] = f->phi_out;
        out[1] = f->pi_out;
        no = 2;
    }
    int rc;
    for (int h = 0; h < nh; ++h)
        if ((rc = check_array(halo[h], 2, "rk4_pair halo input")) || (rc = check_space(space, halo[h], "rk4_pair")))
            return rc;
    for (int t = 0; t < nt; ++t)
        if ((rc = check_array(tile[t], 0, "rk4_pair input")) || (rc = check_space(space, tile[t], "rk4_pair")))
            return rc;
    for (int o = 0; o < no; ++o)
        if ((rc = check_array(out[o], 0, "rk4_pair output")) || (rc = check_space(space, out[o], "rk4_pair")))
            return rc;
    if (zs)
        for (int a = 0; a < 2; ++a)
            if (!zs[a].lo_phi_out || !zs[a].hi_phi_out)
                return fail(SB_USAGE, "rk4_pair_zslab: null neighbour grid");
    return launch_rk4_pair(pair - 1, halo, nh, tile, nt, out, no, space, c, p, as_stream(stream), zs);
}

int sb_rhs24(const sb_array *in, const sb_array *out, sb_space space, sb_d4_constants k, sb_poly poly, sb_launch p,
             void *stream) {
    if (!in || !out) return fail(SB_USAGE, "rhs24: null array table");
    int rc;
    for (int v = 0; v < SB_N_VARS; ++v) {
        if ((rc = check_array(in[v], 2, "rhs24 in")) || (rc = check_space(space, in[v], "rhs24 in"))) return rc;
        if ((rc = check_array(out[v], 0, "rhs24 out")) || (rc = check_space(space, out[v], "rhs24 out"))) return rc;
    }
    return launch_rhs24(in, out, space, k, poly, p, as_stream(stream));
}

int sb_copy_regions(const sb_copy_job *jobs, int32_t njobs, void *stream) {
    if (njobs > 0 && !jobs) return fail(SB_USAGE, "copy_regions: null job table");
    int rc;
    for (int j = 0; j < njobs; ++j)
        if ((rc = check_array(jobs[j].dst, 0, "copy_regions dst")) || (rc = check_array(jobs[j].src, 0, "copy_regions src")))
            return rc;
    return launch_copy_regions(jobs, njobs, as_stream(stream));
}

namespace {
// Copy host planes [p0, p1) of a dense (z,y,x) host array to/from a grid.
int copy_planes(bool h2d, double *host, const sb_array &a, int with_ghosts, int p0, int p1, cudaStream_t st) {
    const int g = with_ghosts ? a.ghost : 0;
    const size_t w = (size_t)(a.nx + 2 * g), rows_y = (size_t)(a.ny + 2 * g);
    const int planes = a.nz + 2 * g;
    if (p0 < 0 || p1 > planes || p0 > p1) return fail(SB_USAGE, "copy: plane range outside the array");
    if (p0 == p1) return SB_OK;
    double *d0 = a.origin - g - (int64_t)g * a.sy - (int64_t)g * a.sz + (int64_t)p0 * a.sz;
    double *h0 = host + (size_t)p0 * rows_y * w;
    const cudaMemcpyKind kind = h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
    if (a.sz == a.sy * (int64_t)(a.ny + 2 * a.ghost) && g == a.ghost) {
        // planes are back to back: one copy of all rows of the range
        const size_t rows = rows_y * (size_t)(p1 - p0);
        if ((size_t)a.sy == w)   // dense rows too: a plain 1-D copy (faster than 2-D over PCIe)
            return h2d ? check_cuda(cudaMemcpyAsync(d0, h0, rows * w * 8, kind, st), "cudaMemcpyAsync h2d")
                       : check_cuda(cudaMemcpyAsync(h0, d0, rows * w * 8, kind, st), "cudaMemcpyAsync d2h");
        return h2d ? check_cuda(cudaMemcpy2DAsync(d0, a.sy * 8, h0, w * 8, w * 8, rows, kind, st), "cudaMemcpy2DAsync h2d")
                   : check_cuda(cudaMemcpy2DAsync(h0, w * 8, d0, a.sy * 8, w * 8, rows, kind, st), "cudaMemcpy2DAsync d2h");
    }
    for (int z = 0; z < p1 - p0; ++z) {
        double *dz = d0 + (int64_t)z * a.sz;
        double *hz = h0 + (size_t)z * rows_y * w;
        int rc = h2d ? check_cuda(cudaMemcpy2DAsync(dz, a.sy * 8, hz, w * 8, w * 8, rows_y, kind, st), "cudaMemcpy2DAsync h2d")
                     : check_cuda(cudaMemcpy2DAsync(hz, w * 8, dz, a.sy * 8, w * 8, rows_y, kind, st), "cudaMemcpy2DAsync d2h");
        if (rc) return rc;
    }
    return SB_OK;
}
}  // namespace

int sb_copy_h2d(sb_array dst, const double *host, int32_t with_ghosts, void *stream) {
    int rc = check_array(dst, 0, "copy_h2d");
    if (rc) return rc;
    if (!host) return fail(SB_USAGE, "copy_h2d: null host pointer");
    const int g = with_ghosts ? dst.ghost : 0;
    return copy_planes(true, const_cast<double *>(host), dst, with_ghosts, 0, dst.nz + 2 * g, as_stream(stream));
}

int sb_copy_d2h(double *host, sb_array src, int32_t with_ghosts, void *stream) {
    int rc = check_array(src, 0, "copy_d2h");
    if (rc) return rc;
    if (!host) return fail(SB_USAGE, "copy_d2h: null host pointer");
    const int g = with_ghosts ? src.ghost : 0;
    return copy_planes(false, host, src, with_ghosts, 0, src.nz + 2 * g, as_stream(stream));
}

int sb_copy_h2d_planes(sb_array dst, const double *host, int32_t with_ghosts, int32_t p0, int32_t p1, void *stream) {
    int rc = check_array(dst, 0, "copy_h2d_planes");
    if (rc) return rc;
    if (!host) return fail(SB_USAGE, "copy_h2d_planes: null host pointer");
    return copy_planes(true, const_cast<double *>(host), dst, with_ghosts, p0, p1, as_stream(stream));
}

int sb_copy_d2h_planes(double *host, sb_array src, int32_t with_ghosts, int32_t p0, int32_t p1, void *stream) {
    int rc = check_array(src, 0, "copy_d2h_planes");
    if (rc) return rc;
    if (!host) return fail(SB_USAGE, "copy_d2h_planes: null host pointer");
    return copy_planes(false, host, src, with_ghosts, p0, p1, as_stream(stream));
}

int sb_copy_h2d_planes_staged(sb_array dst, const double *host, double *staging, int32_t with_ghosts, int32_t p0,
                              int32_t p1, void *stream) {
    int rc = check_array(dst, 0, "copy_h2d_planes_staged");
    if (rc) return rc;
    if (!host || !staging) return fail(SB_USAGE, "copy_h2d_planes_staged: null pointer");
    const int g = with_ghosts ? dst.ghost : 0;
    const size_t w = (size_t)(dst.nx + 2 * g), rows_y = (size_t)(dst.ny + 2 * g);
    const int planes = dst.nz + 2 * g;
    if (p0 < 0 || p1 > planes || p0 > p1) return fail(SB_USAGE, "copy_h2d_planes_staged: plane range outside the array");
    if (p0 == p1) return SB_OK;
    const size_t off = (size_t)p0 * rows_y * w, n = (size_t)(p1 - p0) * rows_y * w;
    rc = check_cuda(cudaMemcpyAsync(staging + off, host + off, n * 8, cudaMemcpyHostToDevice, as_stream(stream)),
                    "cudaMemcpyAsync h2d (staged)");
    if (rc) return rc;
    double *d0 = dst.origin - g - (int64_t)g * dst.sy - (int64_t)g * dst.sz + (int64_t)p0 * dst.sz;
    return launch_unpack_rows(d0, dst.sy, dst.sz, (int)w, (int)rows_y, staging + off, (long long)n, as_stream(stream));
}

}  // extern "C"
