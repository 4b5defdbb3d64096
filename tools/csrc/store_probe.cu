// Microbenchmark (not product code): HBM write throughput of config 2's
// output mix (10 streams of 256^3 doubles, optionally 1 read stream) as a
// function of the store instruction — width (8 / 16 / 32 bytes per thread)
// and cache hint (none, .cs, L1::no_allocate) — and of the access pattern:
//   front: the whole grid sweeps every stream as one coalesced front;
//   tile : d4_all's pattern — a CTA owns a TX x 4 column tile and a z4 chunk
//          of a 256^3 box and writes, plane by plane, ten outputs' rows.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

struct Outs { double *o[10]; };

template <int W, int H>
__device__ __forceinline__ void st(double *p, double a) {
    if constexpr (W == 8) {
        if constexpr (H == 0) asm volatile("st.global.f64 [%0], %1;" ::"l"(p), "d"(a) : "memory");
        else if constexpr (H == 1) asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(p), "d"(a) : "memory");
        else asm volatile("st.global.L1::no_allocate.f64 [%0], %1;" ::"l"(p), "d"(a) : "memory");
    } else if constexpr (W == 16) {
        if constexpr (H == 0) asm volatile("st.global.v2.f64 [%0], {%1, %1};" ::"l"(p), "d"(a) : "memory");
        else if constexpr (H == 1) asm volatile("st.global.cs.v2.f64 [%0], {%1, %1};" ::"l"(p), "d"(a) : "memory");
        else asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %1};" ::"l"(p), "d"(a) : "memory");
    } else {
        if constexpr (H == 0) asm volatile("st.global.v4.f64 [%0], {%1, %1, %1, %1};" ::"l"(p), "d"(a) : "memory");
        else if constexpr (H == 1) asm volatile("st.global.cs.v4.f64 [%0], {%1, %1, %1, %1};" ::"l"(p), "d"(a) : "memory");
        else asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1, %1, %1, %1};" ::"l"(p), "d"(a) : "memory");
    }
}

// n doubles per stream; each thread stores W bytes per stream per step
template <int W, int H, int READ>
__global__ void front_kernel(const double *__restrict__ in, Outs outs, long long n, int nout) {
    constexpr int E = W / 8;
    const long long stride = (long long)gridDim.x * blockDim.x * E;
    for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * E; i < n; i += stride) {
        double v = READ ? __ldcs(in + i) : (double)i;
#pragma unroll
        for (int k = 0; k < 10; ++k)
            if (k < nout) st<W, H>(outs.o[k] + i, v * (k + 1));
    }
}

// d4_all's store pattern on a dense 256^3 box: CTA = TX x 4 tile, z4 chunk,
// thread = W/8 consecutive x points of one row; x tiles fastest.
template <int W, int H, int TX, int READ>
__global__ void tile_kernel(const double *__restrict__ in, Outs outs, int nout) {
    constexpr int E = W / 8, TPR = TX / E, N = 256;
    int t = blockIdx.x;
    const int bx = t % (N / TX);
    t /= N / TX;
    const int by = t % (N / 4);
    const int bz = t / (N / 4);
    const int x = bx * TX + (threadIdx.x % TPR) * E, y = by * 4 + threadIdx.x / TPR;
    for (int zz = 0; zz < 4; ++zz) {
        const long long off = x + (long long)y * N + (long long)(bz * 4 + zz) * N * N;
        double v = READ ? __ldcs(in + off) : (double)off;
#pragma unroll
        for (int k = 0; k < 10; ++k)
            if (k < nout) st<W, H>(outs.o[k] + off, v * (k + 1));
    }
}

template <int W, int H>
int launch_w(int pattern, int read, int tx, const double *in, Outs o, long long n, int nout, int blocks, int threads,
             cudaStream_t s) {
    if (pattern == 0) {
        if (read) front_kernel<W, H, 1><<<blocks, threads, 0, s>>>(in, o, n, nout);
        else front_kernel<W, H, 0><<<blocks, threads, 0, s>>>(in, o, n, nout);
    } else {
        const int E = W / 8;
        const int nb = (256 / tx) * 64 * 64;
        const int thr = tx / E * 4;
        if (tx == 32) {
            if (read) tile_kernel<W, H, 32, 1><<<nb, thr, 0, s>>>(in, o, nout);
            else tile_kernel<W, H, 32, 0><<<nb, thr, 0, s>>>(in, o, nout);
        } else if (tx == 64) {
            if (read) tile_kernel<W, H, 64, 1><<<nb, thr, 0, s>>>(in, o, nout);
            else tile_kernel<W, H, 64, 0><<<nb, thr, 0, s>>>(in, o, nout);
        } else {
            if (read) tile_kernel<W, H, 128, 1><<<nb, thr, 0, s>>>(in, o, nout);
            else tile_kernel<W, H, 128, 0><<<nb, thr, 0, s>>>(in, o, nout);
        }
    }
    return (int)cudaGetLastError();
}

template <int W>
int launch_h(int hint, int pattern, int read, int tx, const double *in, Outs o, long long n, int nout, int blocks,
             int threads, cudaStream_t s) {
    if (hint == 0) return launch_w<W, 0>(pattern, read, tx, in, o, n, nout, blocks, threads, s);
    if (hint == 1) return launch_w<W, 1>(pattern, read, tx, in, o, n, nout, blocks, threads, s);
    return launch_w<W, 2>(pattern, read, tx, in, o, n, nout, blocks, threads, s);
}

}  // namespace

// pattern 0: front (blocks x threads), 1: tile (tx = 32 / 64 / 128, n must be 256^3)
extern "C" int store_probe(int width, int hint, int pattern, int read, int tx, const double *in, double **outs,
                           long long n, int nout, int blocks, int threads, void *stream) {
    Outs o;
    for (int k = 0; k < 10; ++k) o.o[k] = k < nout ? outs[k] : nullptr;
    cudaStream_t s = (cudaStream_t)stream;
    if (width == 8) return launch_h<8>(hint, pattern, read, tx, in, o, n, nout, blocks, threads, s);
    if (width == 16) return launch_h<16>(hint, pattern, read, tx, in, o, n, nout, blocks, threads, s);
    return launch_h<32>(hint, pattern, read, tx, in, o, n, nout, blocks, threads, s);
}
