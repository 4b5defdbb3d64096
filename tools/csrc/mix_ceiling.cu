// Microbenchmark (not product code): HBM ceiling of config 2's traffic mix —
// read one fp64 array, write ten (out_k = in * c_k), grid-stride, double2.
#include <cuda_runtime.h>
#include <stdint.h>

struct Outs { double *o[10]; };

__global__ void mix_kernel(const double2 *__restrict__ in, Outs outs, long long n2, int nout) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x) {
        double2 v = in[i];
#pragma unroll
        for (int k = 0; k < 10; ++k) {
            if (k < nout) {
                double2 w = make_double2(v.x * (k + 1), v.y * (k + 1));
                __stcs(reinterpret_cast<double2 *>(outs.o[k]) + i, w);
            }
        }
    }
}

extern "C" int mix_launch(const double *in, double **outs, long long n, int nout, int blocks, int threads, void *stream) {
    Outs o;
    for (int k = 0; k < 10; ++k) o.o[k] = k < nout ? outs[k] : nullptr;
    mix_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>((const double2 *)in, o, n / 2, nout);
    return (int)cudaGetLastError();
}
