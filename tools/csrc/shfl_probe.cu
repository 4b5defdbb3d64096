// Does SHFL share the shared-memory data path?  (tools/shfl_probe.py)
// lds: 8 independent LDS.64 per step; shfl: 8 independent SHFL.32 per step;
// mix: 8 LDS.64 + K SHFL per step.  Integer accumulation keeps the FP64
// pipe out of it.
#include <cuda_runtime.h>

__global__ void lds_k(unsigned long long *out, int iters) {
    __shared__ double buf[6144];
    for (int i = threadIdx.x; i < 6144; i += blockDim.x) buf[i] = i;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long s = 0;
    int base = (warp * 32) % 4096;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) s ^= __double_as_longlong(buf[((base + k * 256) & 4095) + lane]);
        base += 32;
    }
    if (s == 0x123456789ull) out[blockIdx.x] = s;
}

template <int K>
__global__ void mix_k(unsigned long long *out, int iters, int with_lds) {
    __shared__ double buf[6144];
    for (int i = threadIdx.x; i < 6144; i += blockDim.x) buf[i] = i;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long s = 0;
    unsigned v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = threadIdx.x * 7 + k;
    int base = (warp * 32) % 4096;
    for (int i = 0; i < iters; ++i) {
        if (with_lds) {
#pragma unroll
            for (int k = 0; k < 8; ++k) s ^= __double_as_longlong(buf[((base + k * 256) & 4095) + lane]);
        }
#pragma unroll
        for (int k = 0; k < K; ++k) v[k] = __shfl_sync(0xffffffffu, v[k], (lane + i + k) & 31) + 1u;
        base += 32;
    }
    unsigned t = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) t ^= v[k];
    if ((s ^ t) == 0x123456789ull) out[blockIdx.x] = s ^ t;
}

extern "C" {
int probe(int which, unsigned long long *out, int blocks, int threads, int iters, void *st) {
    cudaStream_t s = (cudaStream_t)st;
    switch (which) {
        case 0: lds_k<<<blocks, threads, 0, s>>>(out, iters); break;
        case 1: mix_k<8><<<blocks, threads, 0, s>>>(out, iters, 0); break;
        case 2: mix_k<8><<<blocks, threads, 0, s>>>(out, iters, 1); break;
        case 3: mix_k<4><<<blocks, threads, 0, s>>>(out, iters, 1); break;
        case 4: mix_k<16><<<blocks, threads, 0, s>>>(out, iters, 1); break;
        default: return -1;
    }
    return (int)cudaGetLastError();
}
}
