// internal.h — host-side declarations shared by the C-ABI translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <string>
#include <utility>

#include "../../include/stencil_b200.h"

namespace sb {

// Thread-local last-error message + status helpers (abi.cu).
int fail(int code, const std::string &msg);
int check_cuda(cudaError_t e, const char *what);

// Raise kernel fn's dynamic shared-memory limit to `bytes` once per (kernel,
// device): the attribute is per device, so a process that drives several
// GPUs sets it on each; later calls are a lookup (no CUDA call, so the launch
// path stays free of non-stream calls during CUDA-graph capture).
int ensure_smem_limit(const void *fn, int bytes, const char *what);

// Launch `kernel` with programmatic stream serialization allowed (PDL): it
// may start while the previous kernel on `st` drains and must itself wait
// (griddepcontrol.wait, pdl_wait_prerequisites) before touching memory.
template <typename... KArgs, typename... Args>
int launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, const char *what,
               Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
#ifndef SB_PDL
#define SB_PDL 1
#endif
    cfg.numAttrs = SB_PDL ? 1 : 0;
    return check_cuda(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), what);
}

// Build a 3-D tiled TMA descriptor over the ghosted grid `a` whose boxes are
// (bx, by, bz) elements.  Coordinates of interior (0,0,0) in the map are
// (a.xpad, a.ghost, a.ghost).
int make_tmap(CUtensorMap *m, const sb_array &a, int bx, int by, int bz);

// Launchers (one per kernel family, defined next to their kernels).
int launch_lap7(const sb_array &dst, const sb_array &src, const sb_space &sp, double c0, double c1,
                const sb_launch &p, cudaStream_t st);
int launch_lap7_iterate(const sb_array &a, const sb_array &b, const sb_space &sp, double c0, double c1, int iters,
                        const sb_launch &p, cudaStream_t st);
// sb_lap7_iterate's grid-barrier counters (lap7.cu): reserve the device's
// pool (sb_init), and the slot of a (device, stream) pair.
int reserve_barrier_counters(int dev);
int release_barrier_counters();
int barrier_counter(int dev, cudaStream_t st, unsigned long long **out);
int launch_diff1d(int kind, double *dst, const double *src, int n, cudaStream_t st);

// RK stages: RK1 = stage 1, RK2 = stage 2 (acc_phi = pi0 + 2 pi_s: stage 1 never
// materialises acc_phi = pi0), RK23 = stage 3, RK4 = stage 4.
// D2_ALL10: the same ten outputs with the 2nd-order centred operators.
enum D4Mode { D4_ALL10 = 0, D4_LAP4 = 1, D4_RK1 = 2, D4_RK23 = 3, D4_RK4 = 4, D4_RK2 = 5, D2_ALL10 = 6 };

struct D4Job {
    sb_array src;         // stencil input (ghost >= 2)
    sb_space space;       // region to update
    sb_array g[10];       // mode-dependent outputs / pointwise inputs
};

int launch_d4(int mode, const D4Job *jobs, int njobs, const sb_d4_constants &k, double ca, const sb_launch &p,
              cudaStream_t st, const sb_zslab *zslab = nullptr);

// Free the device-resident box tables launch_d4 caches (sb_release_tables).
int release_box_tables();

int launch_ghost_periodic(const sb_array &a, cudaStream_t st);

int launch_rk4_pair(int pair, const sb_array *halo, int nh, const sb_array *tile, int nt, const sb_array *out, int no,
                    const sb_space &sp, const sb_rk4_constants &k, const sb_launch &p, cudaStream_t st,
                    const sb_zslab *zs = nullptr);

int launch_copy_regions(const sb_copy_job *jobs, int njobs, cudaStream_t st);
int launch_unpack_rows(double *dst, long long sy, long long sz, int w, int rows_y, const double *src, long long n,
                       cudaStream_t st);

int launch_rhs24(const sb_array *in, const sb_array *out, const sb_space &sp, const sb_d4_constants &k,
                 const sb_poly &poly, const sb_launch &p, cudaStream_t st);

}  // namespace sb
