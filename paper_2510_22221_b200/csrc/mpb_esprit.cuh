// mpb_esprit.cuh -- products with the Hankel data matrix of a probe series,
// the O(M L r) work of the subspace (ESPRIT) mode extraction
// (reference analysis.py:64-115) on the GPU.
//
// X[t][a] = x[t + a], t < M = n - L + 1, a < L (numpy's
// sliding_window_view(x, L)).  With r probe vectors (r <= kHankelMaxR):
//   forward:   out[t][c] = sum_a x[t+a] in[a][c]     (Y = X W,  M x r)
//   transpose: out[a][c] = sum_t x[t+a] in[t][c]     (Z = X^T Y, L x r)
// Row-major operands.  The transpose product splits t over kHankelSplit
// slices whose partial sums are added in a fixed order, so results are
// deterministic run to run.  The small dense algebra of the randomized SVD
// (QR of M x r / L x r panels, the r x r eigenproblem, the K x K shift
// solve) stays on the host (paper_2510_22221_b200/analysis.py).
#pragma once

#include <cuda_runtime.h>

namespace mpb {

constexpr int kHankelMaxR = 32;
constexpr int kHankelTile = 128;
constexpr int kHankelSplit = 32;

// Y = X W: one output row t per thread; x and W staged per a-tile.
__global__ void __launch_bounds__(kHankelTile) k_hankel_fwd(const double* __restrict__ x,
                                                            int64_t M, int L, int r,
                                                            const double* __restrict__ W,
                                                            double* __restrict__ Y) {
    __shared__ double xs[2 * kHankelTile];
    __shared__ double ws[kHankelTile * kHankelMaxR];
    const int64_t t0 = (int64_t)blockIdx.x * kHankelTile;
    const int64_t t = t0 + threadIdx.x;
    double acc[kHankelMaxR];
#pragma unroll
    for (int c = 0; c < kHankelMaxR; ++c) acc[c] = 0.0;
    for (int a0 = 0; a0 < L; a0 += kHankelTile) {
        const int na = min(kHankelTile, L - a0);
        __syncthreads();
        for (int q = threadIdx.x; q < 2 * kHankelTile; q += kHankelTile) {
            const int64_t src = t0 + a0 + q;
            xs[q] = src < M + L - 1 ? x[src] : 0.0;
        }
        for (int q = threadIdx.x; q < na * r; q += kHankelTile) ws[q] = W[(int64_t)a0 * r + q];
        __syncthreads();
        if (t < M)
            for (int a = 0; a < na; ++a) {
                const double xv = xs[threadIdx.x + a];
#pragma unroll
                for (int c = 0; c < kHankelMaxR; ++c)
                    if (c < r) acc[c] = fma(xv, ws[a * r + c], acc[c]);
            }
    }
    if (t < M)
#pragma unroll
        for (int c = 0; c < kHankelMaxR; ++c)
            if (c < r) Y[t * r + c] = acc[c];
}

// Z partial sums: slice s of t, one output row a per thread.
__global__ void __launch_bounds__(kHankelTile) k_hankel_tr(const double* __restrict__ x,
                                                           int64_t M, int L, int r,
                                                           const double* __restrict__ Y,
                                                           double* __restrict__ part) {
    __shared__ double xs[2 * kHankelTile];
    __shared__ double ys[kHankelTile * kHankelMaxR];
    const int a0 = blockIdx.x * kHankelTile;
    const int a = a0 + threadIdx.x;
    const int s = blockIdx.y;
    const int64_t per = (M + gridDim.y - 1) / gridDim.y;
    const int64_t tb = (int64_t)s * per, te = (tb + per < M) ? tb + per : M;
    double acc[kHankelMaxR];
#pragma unroll
    for (int c = 0; c < kHankelMaxR; ++c) acc[c] = 0.0;
    for (int64_t t0 = tb; t0 < te; t0 += kHankelTile) {
        const int nt = (int)(te - t0 < kHankelTile ? te - t0 : kHankelTile);
        __syncthreads();
        for (int q = threadIdx.x; q < 2 * kHankelTile; q += kHankelTile) {
            const int64_t src = t0 + a0 + q;
            xs[q] = src < M + L - 1 ? x[src] : 0.0;
        }
        for (int q = threadIdx.x; q < nt * r; q += kHankelTile) ys[q] = Y[t0 * r + q];
        __syncthreads();
        if (a < L)
            for (int tt = 0; tt < nt; ++tt) {
                const double xv = xs[threadIdx.x + tt];
#pragma unroll
                for (int c = 0; c < kHankelMaxR; ++c)
                    if (c < r) acc[c] = fma(xv, ys[tt * r + c], acc[c]);
            }
    }
    if (a < L)
#pragma unroll
        for (int c = 0; c < kHankelMaxR; ++c)
            if (c < r) part[((int64_t)s * L + a) * r + c] = acc[c];
}

// Z = sum over the slices, in slice order.
__global__ void k_hankel_sum(const double* __restrict__ part, int nslices, int64_t n,
                             double* __restrict__ Z) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
         q += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int k = 0; k < nslices; ++k) s += part[(int64_t)k * n + q];
        Z[q] = s;
    }
}

}  // namespace mpb
