#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1505_08023_b200/csrc/exact.cuh"
using namespace minife;
__global__ void k(const unsigned long long *g, double *out, long long *cyc, int reps) {
    __shared__ unsigned long long s[ACC_WORDS];
    for (int i = threadIdx.x; i < ACC_WORDS; i += blockDim.x) s[i] = g[i];
    __syncwarp();
    double acc = 0.0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        double v = acc_finalize_warp(s);
        acc += v;
        if (threadIdx.x == 0) s[5] ^= (unsigned long long)(v == 12345.0);   // keep the loop live
        __syncwarp();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = acc; cyc[0] = (t1 - t0) / reps; }
}
int main() {
    // a typical positive accumulator: a few adjacent nonzero words around 2^0
    unsigned long long h[ACC_WORDS] = {0};
    h[33] = 0x123456789abcull; h[34] = 0x3fffffffull; h[35] = 0x2ull; h[32] = 0xfedcba987ull;
    unsigned long long *d; double *o; long long *c;
    cudaMalloc(&d, sizeof h); cudaMalloc(&o, 8); cudaMalloc(&c, 8);
    cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(d, o, c, 1000); cudaDeviceSynchronize();
    long long cy; double v; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&v, o, 8, cudaMemcpyDeviceToHost);
    printf("{\"cycles_per_finalize\": %lld, \"check\": %.17g}\n", cy, v);
    return 0;
}
