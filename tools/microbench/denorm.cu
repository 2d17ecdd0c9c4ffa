// FP64 throughput with normal vs subnormal operands (fma/mul/add chains and
// the IEEE division), to see whether subnormals take a slow path on B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_fma(const double* in, double* out, int iters) {
    double a = in[threadIdx.x & 31], b = in[32 + (threadIdx.x & 31)], c = a;
    for (int i = 0; i < iters; ++i) { c = __fma_rn(a, 0.5, c); c = __dmul_rn(c, 1.0); c = __dadd_rn(c, -a * 0.5); }
    out[blockIdx.x * blockDim.x + threadIdx.x] = c + b;
}
__global__ void k_div(const double* in, double* out, int iters, double d) {
    double a = in[threadIdx.x & 31], c = 0.0;
    for (int i = 0; i < iters; ++i) { c += a / d; a = a * 1.0000001; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = c;
}
int main() {
    double h[64], *din, *dout;
    cudaMalloc(&din, 64 * 8); cudaMalloc(&dout, 148 * 8 * 256 * 8);
    const char* names[3] = {"normal 1.0", "tiny 1e-300", "subnormal 1e-310"};
    const double vals[3] = {1.0, 1e-300, 1e-310};
    for (int m = 0; m < 3; ++m) {
        for (int i = 0; i < 64; ++i) h[i] = vals[m] * (1.0 + i * 1e-3);
        cudaMemcpy(din, h, 64 * 8, cudaMemcpyHostToDevice);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int kind = 0; kind < 2; ++kind) {
            k_fma<<<148 * 8, 256>>>(din, dout, 10);
            cudaEventRecord(e0);
            if (kind == 0) k_fma<<<148 * 8, 256>>>(din, dout, 20000);
            else k_div<<<148 * 8, 256>>>(din, dout, 2000, 3.7e-6);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("%-18s %s: %.3f ms\n", names[m], kind == 0 ? "fma/mul/add chain" : "x / d", ms);
        }
    }
    return 0;
}
