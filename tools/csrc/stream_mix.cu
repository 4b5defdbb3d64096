// Microbenchmark (not product code): how many bytes/s HBM sustains for
// config 2's stream mix under different access shapes.
//   mode 0: write-only, `nout` output streams (no read)
//   mode 1: 1 read + `nout` writes, UNROLL independent loads in flight per thread
// Each CTA owns a contiguous chunk of every stream and walks it in
// 16-byte-per-thread rows (blockDim * 16 B contiguous per stream per step).
#include <cuda_runtime.h>

struct Outs { double *o[10]; };

template <int MODE, int UNROLL>
__global__ void stream_kernel(const double2 *__restrict__ in, Outs outs, long long n2, int nout, long long chunk) {
    const long long b0 = blockIdx.x * chunk, b1 = min(n2, b0 + chunk);
    for (long long i0 = b0 + threadIdx.x; i0 < b1; i0 += (long long)blockDim.x * UNROLL) {
        double2 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const long long i = i0 + (long long)u * blockDim.x;
            if (MODE == 1) v[u] = i < b1 ? __ldcs(in + i) : make_double2(0, 0);
            else v[u] = make_double2((double)i, 1.0);
        }
#pragma unroll
        for (int k = 0; k < 10; ++k) {
            if (k < nout) {
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    const long long i = i0 + (long long)u * blockDim.x;
                    if (i < b1) __stcs(reinterpret_cast<double2 *>(outs.o[k]) + i, make_double2(v[u].x * (k + 1), v[u].y));
                }
            }
        }
    }
}

// front layout: the whole grid sweeps each stream as one coalesced front
// (consecutive threads of consecutive CTAs on consecutive 16-byte words)
template <int READ, int UNROLL>
__global__ void front_kernel(const double2 *__restrict__ in, Outs outs, long long n2, int nout) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < n2; i0 += stride * UNROLL) {
        double2 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const long long i = i0 + u * stride;
            if (READ) v[u] = i < n2 ? __ldcs(in + i) : make_double2(0, 0);
            else v[u] = make_double2((double)i, 1.0);
        }
#pragma unroll
        for (int k = 0; k < 10; ++k) {
            if (k < nout) {
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    const long long i = i0 + u * stride;
                    if (i < n2) __stcs(reinterpret_cast<double2 *>(outs.o[k]) + i, make_double2(v[u].x * (k + 1), v[u].y));
                }
            }
        }
    }
}

extern "C" int stream_launch(int mode, int unroll, const double *in, double **outs, long long n, int nout, int blocks,
                             int threads, void *stream) {
    Outs o;
    for (int k = 0; k < 10; ++k) o.o[k] = k < nout ? outs[k] : nullptr;
    const long long n2 = n / 2, chunk = (n2 + blocks - 1) / blocks;
    cudaStream_t st = (cudaStream_t)stream;
    const double2 *src = (const double2 *)in;
    if (mode == 2) {
        if (unroll == 1) front_kernel<0, 1><<<blocks, threads, 0, st>>>(src, o, n2, nout);
        else front_kernel<0, 4><<<blocks, threads, 0, st>>>(src, o, n2, nout);
        return (int)cudaGetLastError();
    }
    if (mode == 3) {
        if (unroll == 1) front_kernel<1, 1><<<blocks, threads, 0, st>>>(src, o, n2, nout);
        else if (unroll == 4) front_kernel<1, 4><<<blocks, threads, 0, st>>>(src, o, n2, nout);
        else front_kernel<1, 8><<<blocks, threads, 0, st>>>(src, o, n2, nout);
        return (int)cudaGetLastError();
    }
    if (mode == 0 && unroll == 1) stream_kernel<0, 1><<<blocks, threads, 0, st>>>(src, o, n2, nout, chunk);
    else if (mode == 0) stream_kernel<0, 4><<<blocks, threads, 0, st>>>(src, o, n2, nout, chunk);
    else if (unroll == 1) stream_kernel<1, 1><<<blocks, threads, 0, st>>>(src, o, n2, nout, chunk);
    else if (unroll == 4) stream_kernel<1, 4><<<blocks, threads, 0, st>>>(src, o, n2, nout, chunk);
    else stream_kernel<1, 8><<<blocks, threads, 0, st>>>(src, o, n2, nout, chunk);
    return (int)cudaGetLastError();
}
