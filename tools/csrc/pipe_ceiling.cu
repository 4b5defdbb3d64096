// Pipe ceilings for the K6 (config 5) roofline: FP64 add/mul issue rate and
// shared-memory LDS.64 wavefront rate on this B200, measured with trivial
// kernels (tools/pipe_ceiling.py).  Built with -fmad=false like the product
// so DADD/DMUL stay unfused.
#include <cuda_runtime.h>

extern "C" {

// 8 independent chains of (x = x*a + b) written as DMUL + DADD: 2 FP64 ops
// per chain step, ITERS steps.
__global__ void fp64_kernel(double *out, double a, double b, int iters) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = __dadd_rn(__dmul_rn(x[k], a), b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.678) out[blockIdx.x] = s;   // keep the work alive
}

// every thread reads consecutive doubles of a 32-wide row (2 wavefronts per
// warp instruction) from a 48 KB shared buffer, 8 independent loads per step
__global__ void lds_kernel(double *out, int iters) {
    __shared__ double buf[6144];
    for (int i = threadIdx.x; i < 6144; i += blockDim.x) buf[i] = i;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long s = 0;   // integer xor keeps the FP64 pipe out of the way
    int base = (warp * 32) % 4096;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) s ^= __double_as_longlong(buf[((base + k * 256) & 4095) + lane]);
        base += 32;
    }
    if (s == 0x123456789ull) out[blockIdx.x] = (double)s;
}

int fp64_launch(double *out, int blocks, int threads, int iters, void *st) {
    fp64_kernel<<<blocks, threads, 0, (cudaStream_t)st>>>(out, 0.999999, 1e-7, iters);
    return (int)cudaGetLastError();
}

int lds_launch(double *out, int blocks, int threads, int iters, void *st) {
    lds_kernel<<<blocks, threads, 0, (cudaStream_t)st>>>(out, iters);
    return (int)cudaGetLastError();
}

}
