/*
 * stencil_b200.h — C ABI of libstencil_b200.so, the B200 (sm_100a) hot path
 * behind the reference's loop-iterator / stencil-kernel plugin interface.
 *
 * The reference (package `stencilrt`, pure Python) has no native code; its
 * plugin boundary is `Kernel = Callable[[IndexSpace], None]`
 * (pkg/src/stencilrt/traverse.py:159) called by `execute_plan`
 * (traverse.py:162-209) / `run_loop` (traverse.py:220-232) /
 * `run_static` (traverse.py:235-260), with the arithmetic in
 * `_update_rows` (stencil.py:31-39).  Each entry point below replaces one
 * such kernel body for a whole index space (or a whole bboxset level) in a
 * single launch.  The Python host layer binds these through ctypes
 * (paper_1308_1343_b200/_lib.py); INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - Grids are fp64, x contiguous (the reference's numpy (z,y,x) C-order,
 *    stencil.py:9-10).  `sb_array.origin` points at interior point (0,0,0);
 *    element (x,y,z) is origin[x + y*sy + z*sz] for -ghost <= x,y,z <
 *    n+ghost.  Every row additionally owns `xpad` readable elements before
 *    x = 0 so rows start 128-byte aligned (TMA base).
 *  - Index spaces are half-open [lo, hi), innermost dimension first, in
 *    interior coordinates (traverse.py:31-56 uses the same ordering).
 *  - Arithmetic is IEEE fp64, one rounding per + - *, association exactly as
 *    the reference's numpy expression trees (no FMA contraction; the library
 *    is built with -fmad=false and uses __d*_rn intrinsics).  This is the
 *    reference's unfused-FMA contract, vlanes.py:33 / vlanes.py:243-249.
 *  - All launches are asynchronous on the caller's stream (a cudaStream_t
 *    passed as void*; NULL = legacy default stream).  No entry point
 *    allocates or frees caller memory.  Kernels are launched with
 *    programmatic stream serialization (programmatic dependent launch): a
 *    sweep may be scheduled while the previous kernel on the stream drains,
 *    but it reads or writes memory only after that kernel has completed, so
 *    stream order is preserved exactly as for a plain launch.
 *  - Return codes: SB_OK, SB_USAGE (contract violation, maps to the
 *    reference's UsageError, lattice.py:22), SB_RESOURCE (ResourceError,
 *    lattice.py:26), SB_CUDA (CUDA failure).  sb_last_error() returns a
 *    thread-local message for the last failing call.  No C++ exception
 *    crosses this boundary.
 */
#ifndef STENCIL_B200_H
#define STENCIL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SB_ABI_VERSION 2   /* 2: level box tables, multi-box d4_all/d2_all/RK stages, peer access, shutdown */

#if defined(__GNUC__)
#define SB_API __attribute__((visibility("default")))
#else
#define SB_API
#endif

#define SB_OK 0
#define SB_USAGE 1
#define SB_RESOURCE 2
#define SB_CUDA 3

#define SB_MAX_BOXES 8     /* boxes whose table travels in the launch parameters; a
                              launch over more boxes (any number) uses a device-resident
                              box table the library builds once per level shape */
#define SB_N_D4_OUT 10     /* Dx Dy Dz Dxx Dyy Dzz Dxy Dxz Dyz Lap4 */
#define SB_N_VARS 24       /* config-5 grid functions */
#define SB_N_TERMS 64      /* config-5 terms per output polynomial */

/* One fp64 grid in device memory (the device-resident form of the numpy
 * arrays the reference's kernels close over, stencil.py:42-46). */
typedef struct sb_array {
    double *origin;   /* interior (0,0,0); 16-byte aligned */
    int64_t sy;       /* row pitch in elements (even) */
    int64_t sz;       /* plane pitch in elements (even) */
    int32_t nx, ny, nz; /* interior extents */
    int32_t ghost;    /* ghost width on every face */
    int32_t xpad;     /* readable elements before x = 0 in a row (>= ghost, even) */
} sb_array;

/* Half-open index space, innermost first (traverse.py:31-56). */
typedef struct sb_space {
    int32_t lo[3];
    int32_t hi[3];
} sb_space;

/* One point of the GPU tuning space (the device counterpart of the
 * reference's ExecParams, tuner.py:99-111): CTA tile in x and y, the number
 * of z planes one CTA streams, and whether a thread owns one x point or a
 * 16-byte pair (the SIMD width W of vlanes.py).  tile_x is 32, 64 or 128. */
typedef struct sb_launch {
    int32_t tile_x;
    int32_t tile_y;
    int32_t z_chunk;
    int32_t flags;    /* SB_LAUNCH_* bits */
} sb_launch;

/* sb_launch.flags: one x point per thread instead of a 16-byte pair. */
#define SB_LAUNCH_SCALAR 1
/* sb_launch.flags (sb_rk4_stage): also write every ghost point of phi_out
 * that is the periodic image of an updated interior point, so the next
 * stage needs no separate sb_ghost_periodic (the space must be the whole
 * interior). */
#define SB_LAUNCH_PERIODIC_GHOSTS 2

/* 4th-order constants: k1 = 1/(12h), k2 = 1/(12h^2), k11 = 1/(144h^2). */
typedef struct sb_d4_constants {
    double k1, k2, k11;
} sb_d4_constants;

/* One box of a refinement level: its source grid (ghost >= 2), the output
 * grid and the index space to update (interior coordinates of the box). */
typedef struct sb_box_job {
    sb_array dst;
    sb_array src;
    sb_space space;
} sb_box_job;

/* Classical RK4 state for the scalar wave equation (phi, pi). */
typedef struct sb_rk4_fields {
    sb_array phi_s;   /* stencil input of this stage (ghost >= 2, filled) */
    sb_array pi_s;    /* pi of this stage (unused by stage 1) */
    sb_array phi0, pi0;   /* state at the start of the step */
    sb_array acc_phi, acc_pi; /* running k1 + 2k2 + 2k3 (in place) */
    sb_array phi_out, pi_out; /* next stage (or new state at stage 4) */
} sb_rk4_fields;

typedef struct sb_rk4_constants {
    sb_d4_constants lap;
    double half_dt, dt, dt6;
} sb_rk4_constants;

/* Config-5 polynomial table, row-major [output][term]. */
typedef struct sb_poly {
    const double *coef;   /* SB_N_VARS * SB_N_TERMS */
    const int32_t *p;     /* input index 10*var + slot, 0..239 */
    const int32_t *q;
} sb_poly;

/* One region copy between two grids of a level (inter-box ghost fill):
 * dst[dst_lo + i] = src[src_lo + i] for 0 <= i < ext, coordinates relative to
 * each grid's interior origin (dst_lo may lie in the ghost zone). */
typedef struct sb_copy_job {
    sb_array dst;
    sb_array src;
    int32_t dst_lo[3];
    int32_t src_lo[3];
    int32_t ext[3];
} sb_copy_job;

#define SB_MAX_COPY_JOBS 64   /* region copies per launch (sb_copy_regions) */

typedef struct sb_device_info {
    int32_t device, sm_count, cc_major, cc_minor;
    int64_t l2_bytes, smem_optin_bytes, global_mem_bytes;
} sb_device_info;

SB_API int sb_abi_version(void);
SB_API const char *sb_last_error(void);
SB_API int sb_init(int device);
SB_API int sb_get_device_info(sb_device_info *info);
/* Let kernels on the current device load/store the memory of device `peer`
 * (NVLink peer access; the z-slab halo stores into a neighbour GPU's ghost
 * planes).  SB_OK if enabled, already enabled or peer is the current device;
 * SB_RESOURCE if the devices cannot be peers. */
SB_API int sb_enable_peer_access(int peer);

/* K0 — vlanes.forward_difference (vlanes.py:342-349) when kind == 0:
 * dst[i] = src[i+1] - src[i], 0 <= i < n-1;  vlanes.centered_difference
 * (vlanes.py:352-360) when kind == 1: dst[i] = 0.5*(src[i+1]-src[i-1]),
 * 1 <= i < n-1.  Lanes outside the range never store (iterate_masked,
 * vlanes.py:322-337). */
SB_API int sb_diff1d(int32_t kind, double *dst, const double *src, int32_t n, void *stream);

/* K1 — 7-point update (stencil.py:31-39, _update_rows):
 * dst = c0*b + c1*(((xm+xp) + (ym+yp)) + (zm+zp)) over `space`. */
SB_API int sb_lap7(sb_array dst, sb_array src, sb_space space, double c0, double c1,
            sb_launch p, void *stream);

/* K1 iterated — `iters` Jacobi sweeps of the same update in ONE persistent
 * cooperative launch (the reference's run_serial loop, stencil.py:55-65):
 * sweep k reads a and writes b for even k, the reverse for odd k, with a
 * grid-wide barrier between sweeps; the result is in b for odd `iters`, in
 * a for even.  Both grids need ghost >= 1 with the same (fixed) boundary
 * values.  Bit-identical to `iters` sb_lap7 calls.  The grid barrier uses a
 * library-owned 64-bit counter per (device, stream) from a pool that
 * sb_init reserves; without a prior sb_init the first call on a device
 * allocates the pool and is therefore refused inside a CUDA-graph capture. */
SB_API int sb_lap7_iterate(sb_array a, sb_array b, sb_space space, double c0, double c1, int32_t iters,
                           sb_launch p, void *stream);

/* K2 — all ten 4th-order outputs of one box (config 2).  out[i] follows
 * SB_N_D4_OUT order.  src ghost >= 2. */
SB_API int sb_d4_all(const sb_array *out, sb_array src, sb_space space,
              sb_d4_constants k, sb_launch p, void *stream);

/* K2' — the same ten outputs with the 2nd-order centred operators:
 * D1 = (u[+1]-u[-1]) k1, D2 = ((u[-1]+u[+1]) - 2u) k2, D_ab = d_a(d_b) k11,
 * Lap2 = (Dxx + Dyy) + Dzz with k1 = 1/(2h), k2 = 1/h^2, k11 = 1/(4h^2).
 * src ghost >= 2 (the kernel stages radius-2 halos). */
SB_API int sb_d2_all(const sb_array *out, sb_array src, sb_space space,
                     sb_d4_constants k, sb_launch p, void *stream);

/* K3 — 4th-order Laplacian over every box of a level in ONE launch
 * (config 4; the boxes of BBoxSet.to_bboxes(), bboxset.py:313-317 ->
 * traverse.py:59-65).  The box table (blockIdx -> box by binary search on
 * each box's first tile) replaces execute_plan's block queue
 * (traverse.py:162-209).  Up to SB_MAX_BOXES boxes travel in the launch
 * parameters; larger levels use a device-resident table that the first
 * launch of a (box list, launch shape) builds and uploads — that first
 * launch waits for the upload and is refused inside a CUDA-graph capture;
 * later launches of the same shape are pure launches.  Tables are released
 * by sb_release_tables. */
SB_API int sb_lap4_boxes(const sb_box_job *jobs, int32_t njobs, sb_d4_constants k,
                  sb_launch p, void *stream);

/* K2 over a level: all ten 4th-order (sb_d4_all_boxes) or 2nd-order
 * (sb_d2_all_boxes) outputs of every box in one launch (same box table). */
typedef struct sb_d4_all_job {
    sb_array out[SB_N_D4_OUT];
    sb_array src;
    sb_space space;
} sb_d4_all_job;

SB_API int sb_d4_all_boxes(const sb_d4_all_job *jobs, int32_t njobs, sb_d4_constants k, sb_launch p, void *stream);
SB_API int sb_d2_all_boxes(const sb_d4_all_job *jobs, int32_t njobs, sb_d4_constants k, sb_launch p, void *stream);

/* Free the library's cached device box tables (waits for the device). */
SB_API int sb_release_tables(void);

/* Release every device allocation the library owns (box tables, the
 * barrier-counter pools of sb_init); waits for the devices.  The library
 * stays usable: later calls allocate again on first use. */
SB_API int sb_shutdown(void);

/* K4 — periodic refill of the ghost shell of `a` (every ghost point becomes
 * the interior point at its periodic image). */
SB_API int sb_ghost_periodic(sb_array a, void *stream);

/* K5 — one classical RK4 stage (1..4) of d/dt(phi, pi) = (pi, Lap4 phi). */
SB_API int sb_rk4_stage(int32_t stage, const sb_rk4_fields *f, sb_space space,
                 sb_rk4_constants c, sb_launch p, void *stream);

/* K5 over a level: one RK4 stage of every box in one launch (the boxes'
 * phi_s ghosts filled beforehand, e.g. by sb_copy_regions; no periodic
 * refresh: SB_LAUNCH_PERIODIC_GHOSTS is refused). */
typedef struct sb_rk4_box_job {
    sb_rk4_fields f;
    sb_space space;
} sb_rk4_box_job;

SB_API int sb_rk4_stage_boxes(int32_t stage, const sb_rk4_box_job *jobs, int32_t njobs, sb_rk4_constants c,
                              sb_launch p, void *stream);

/* K5b — the same RK4 step as two fused launches (temporal blocking):
 * pair 1 = stages 1+2: reads phi0, pi0 (ghosts valid), writes phi_out = phi3,
 *   pi_out = pi3, acc_phi = pi0 + 2 pi2, acc_pi = L1 + 2 L2;
 * pair 2 = stages 3+4: reads phi_s = phi3, phi0, pi_s = pi3 (ghosts valid),
 *   pi0, acc_phi, acc_pi, writes phi_out = phi', pi_out = pi'.
 * Bit-identical to the four sb_rk4_stage launches; 14 array passes instead
 * of 32.  With SB_LAUNCH_PERIODIC_GHOSTS both phi_out and pi_out get their
 * periodic ghost shells refreshed (pi's ghosts feed the next pair).
 * Laplacian pairs (10 array passes, same bits):
 * pair 3 = stages 1+2: reads phi0, pi0 (ghosts valid), writes phi_out = L1 =
 *   Lap4(phi0), pi_out = L2 = Lap4(phi0 + (dt/2) pi0);
 * pair 4 = stages 3+4: reads phi0, pi0, phi_s = L1, pi_s = L2 (ghosts valid),
 *   writes phi_out = phi', pi_out = pi' (acc_phi / acc_pi unused). */
SB_API int sb_rk4_pair(int32_t pair, const sb_rk4_fields *f, sb_space space, sb_rk4_constants c, sb_launch p,
                       void *stream);

/* F4 — z-slab decomposition of one periodic box over several GPUs (or
 * several slabs of one GPU): the stage that produces phi also writes the
 * halo planes straight into the neighbouring slabs' ghost planes (peer
 * stores over NVLink when the neighbour lives on another GPU).  Points
 * within `ghost` of the slab's low z face are also written to lo_phi_out at
 * z + lo_dz, points within `ghost` of the high face to hi_phi_out at
 * z + hi_dz (normally lo_dz = +nz of the lower slab, hi_dz = -nz of this
 * slab); x/y ghosts are refreshed periodically in every target.  Peer grids
 * must share phi_out's row and plane strides.  Requires
 * SB_LAUNCH_PERIODIC_GHOSTS. */
typedef struct sb_zslab {
    double *lo_phi_out;   /* origin of the lower neighbour's phi_out */
    int32_t lo_dz;
    double *hi_phi_out;   /* origin of the upper neighbour's phi_out */
    int32_t hi_dz;
} sb_zslab;

SB_API int sb_rk4_stage_zslab(int32_t stage, const sb_rk4_fields *f, sb_space space, sb_rk4_constants c,
                              sb_launch p, const sb_zslab *zs, void *stream);

/* F4 for the pair schedules (sb_rk4_pair): both outputs of a pair launch
 * write their boundary planes into the neighbouring slabs' ghost planes —
 * zs[0] names phi_out's neighbours, zs[1] pi_out's (each of the pair's
 * outputs feeds a stencil of the next launch).  Same conventions as
 * sb_rk4_stage_zslab; requires SB_LAUNCH_PERIODIC_GHOSTS. */
SB_API int sb_rk4_pair_zslab(int32_t pair, const sb_rk4_fields *f, sb_space space, sb_rk4_constants c,
                             sb_launch p, const sb_zslab *zs /* [2] */, void *stream);

/* K6 — config-5 fused right-hand side: 24 inputs (ghost >= 2) -> 24 outputs. */
SB_API int sb_rhs24(const sb_array *in, const sb_array *out, sb_space space,
             sb_d4_constants k, sb_poly poly, sb_launch p, void *stream);

/* F1 — inter-box ghost fill of a refinement level: every region copy of the
 * schedule (built on the host from the level's boxes, level.ghost_schedule)
 * in one launch; pure copies, bit-exact. */
SB_API int sb_copy_regions(const sb_copy_job *jobs, int32_t njobs, void *stream);

/* Host <-> device transfer of a whole ghosted grid (with_ghosts = 1) or of
 * its interior (0).  `host` is dense (z,y,x), x contiguous. */
SB_API int sb_copy_h2d(sb_array dst, const double *host, int32_t with_ghosts, void *stream);
SB_API int sb_copy_d2h(double *host, sb_array src, int32_t with_ghosts, void *stream);

/* The same for the z-plane range [p0, p1) of the host array's plane
 * numbering (with ghosts: plane 0 is the first ghost plane); `host` is the
 * base of the whole host array.  Lets a caller pipeline transfers with
 * compute over z chunks. */
SB_API int sb_copy_h2d_planes(sb_array dst, const double *host, int32_t with_ghosts, int32_t p0, int32_t p1,
                              void *stream);
SB_API int sb_copy_d2h_planes(double *host, sb_array src, int32_t with_ghosts, int32_t p0, int32_t p1,
                              void *stream);

/* Upload host planes [p0, p1) through a dense device staging buffer (at
 * least as large as the whole dense host array): one linear H2D copy at
 * full PCIe speed, then an on-device unpack into the padded rows of `dst`.
 * (A pitched 2-D H2D copy runs at a third of the link rate and does not
 * overlap D2H traffic.) */
SB_API int sb_copy_h2d_planes_staged(sb_array dst, const double *host, double *staging, int32_t with_ghosts,
                                     int32_t p0, int32_t p1, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* STENCIL_B200_H */
