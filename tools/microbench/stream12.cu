// Streaming ceiling for the sweep's access pattern: read 6 fp64 fields and
// write 6 (ping-pong), the same 96 B/cell the Yee step moves.  Trivial math;
// measures what HBM delivers for 6R+6W streams on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)
struct P { const double2* a[6]; double2* b[6]; };
__global__ void __launch_bounds__(256) k12(P p, long n2) {
    for (long i = blockIdx.x * 256L + threadIdx.x; i < n2; i += (long)gridDim.x * 256) {
        double2 v[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) v[c] = __ldcs(p.a[c] + i);
#pragma unroll
        for (int c = 0; c < 6; ++c) {
            double2 w = v[c]; w.x += v[(c + 1) % 6].x; w.y += v[(c + 1) % 6].y;
            __stcs(p.b[c] + i, w);
        }
    }
}
__global__ void copy1(const double2* a, double2* b, long n2) {
    for (long i = blockIdx.x * 256L + threadIdx.x; i < n2; i += (long)gridDim.x * 256) b[i] = a[i];
}
int main() {
    const long n = 1024L * 1024 * 128, n2 = n / 2;
    P p; double* buf;
    CK(cudaMalloc(&buf, 12 * n * 8)); CK(cudaMemset(buf, 0, 12 * n * 8));
    for (int c = 0; c < 6; ++c) { p.a[c] = (double2*)(buf + c * n); p.b[c] = (double2*)(buf + (6 + c) * n); }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int g : {148 * 4, 148 * 8, 148 * 16, 148 * 32}) {
        for (int w = 0; w < 3; ++w) k12<<<g, 256>>>(p, n2);
        cudaEventRecord(e0);
        for (int r = 0; r < 20; ++r) k12<<<g, 256>>>(p, n2);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 20;
        printf("6R+6W grid %d: %.3f ms  %.1f GB/s\n", g, ms, 12.0 * n * 8 / ms / 1e6);
    }
    for (int g : {148 * 8, 148 * 32}) {
        for (int w = 0; w < 3; ++w) copy1<<<g, 256>>>(p.a[0], p.b[0], 6 * n2);
        cudaEventRecord(e0);
        for (int r = 0; r < 20; ++r) copy1<<<g, 256>>>(p.a[0], p.b[0], 6 * n2);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 20;
        printf("copy grid %d: %.3f ms  %.1f GB/s\n", g, ms, 12.0 * n * 8 / ms / 1e6);
    }
    return 0;
}
