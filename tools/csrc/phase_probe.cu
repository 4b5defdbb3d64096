// Microbenchmark (not product code): does separating HBM reads from HBM
// writes in time raise throughput for config 2's 1-read/10-write mix (and for
// a plain 1:1 copy)?  One CTA per SM; each phase every CTA reads a chunk of
// the input into shared memory, then writes it to `nout` outputs.  SYNC = 1
// puts a grid barrier between the read and the write half of every phase
// (the whole chip reads, then the whole chip writes); SYNC = 0 is the same
// code without the barriers (CTAs drift apart and the DRAM sees a mix).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

namespace {

struct Outs { double *o[10]; };

template <int SYNC>
__global__ void __launch_bounds__(1024, 1)
    phase_kernel(const double2 *__restrict__ in, Outs outs, long long n2, int nout, int chunk2) {
    extern __shared__ double2 buf[];
    cg::grid_group grid = cg::this_grid();
    const long long per_phase = (long long)gridDim.x * chunk2;
    for (long long base = 0; base < n2; base += per_phase) {
        const long long c0 = base + (long long)blockIdx.x * chunk2;
        // read: 8 independent 16-byte loads per thread in flight
        for (int i = threadIdx.x; i < chunk2; i += blockDim.x * 8) {
            double2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int k = i + u * blockDim.x;
                v[u] = (k < chunk2 && c0 + k < n2) ? __ldcs(in + c0 + k) : make_double2(0, 0);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int k = i + u * blockDim.x;
                if (k < chunk2) buf[k] = v[u];
            }
        }
        __syncthreads();
        if (SYNC) grid.sync();
        for (int o = 0; o < nout; ++o) {
            double2 *dst = reinterpret_cast<double2 *>(outs.o[o]);
            for (int k = threadIdx.x; k < chunk2; k += blockDim.x)
                if (c0 + k < n2) {
                    const double2 v = buf[k];
                    __stcs(dst + c0 + k, make_double2(v.x * (o + 1), v.y));
                }
        }
        __syncthreads();
        if (SYNC) grid.sync();
    }
}

}  // namespace

extern "C" int phase_probe(int sync, const double *in, double **outs, long long n, int nout, int chunk_bytes,
                           int blocks, void *stream) {
    Outs o;
    for (int k = 0; k < 10; ++k) o.o[k] = k < nout ? outs[k] : nullptr;
    long long n2 = n / 2;
    int chunk2 = chunk_bytes / 16;
    const double2 *src = reinterpret_cast<const double2 *>(in);
    void *args[] = {(void *)&src, (void *)&o, (void *)&n2, (void *)&nout, (void *)&chunk2};
    size_t smem = (size_t)chunk_bytes;
    cudaStream_t st = (cudaStream_t)stream;
    if (sync) {
        cudaFuncSetAttribute(phase_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        return (int)cudaLaunchCooperativeKernel((void *)phase_kernel<1>, blocks, 1024, args, smem, st);
    }
    cudaFuncSetAttribute(phase_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return (int)cudaLaunchCooperativeKernel((void *)phase_kernel<0>, blocks, 1024, args, smem, st);
}
