// Memory-pattern ceiling of the sweep: the same tiling, 3-slot TMA ring,
// per-plane barrier, bulk H stores and per-entry E stores as k_sweep on the
// C4 lattice, with the stencil arithmetic replaced by one add per value.
// Tells whether the sweep is bound by its access pattern or by its compute.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void tma_ld(void* d, const void* s, uint32_t n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(d)), "l"(s), "r"(n), "r"(su32(b)) : "memory"); }
__device__ __forceinline__ void tma_st(void* g, const void* s, uint32_t n) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(su32(s)), "r"(n) : "memory"); }
__device__ __forceinline__ void wait_par(uint64_t* b, uint32_t ph) {
    asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}" ::"r"(su32(b)), "r"(ph) : "memory"); }

struct Cfg { int T, tiles, chunk, nchunks, hl, ecap, hcap, FyFz, Fx; long PP; int stage; int ebulk; };
struct Ptr { const double* Ea[3]; const double* Ha[3]; double* Eb[3]; double* Hb[3]; };

__global__ void __launch_bounds__(256, 2) k_pattern(Ptr P, Cfg c) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t bars[3];
    const int tid = threadIdx.x, NT = 256;
    const int tile = blockIdx.x % c.tiles, chunk = blockIdx.x / c.tiles;
    const int f0 = tile * c.T, f1 = min(f0 + c.T, c.FyFz);
    const int i0 = chunk * c.chunk, i1 = min(i0 + c.chunk, c.Fx);
    if (i0 >= i1) return;
    const int pstart = i0 > 0 ? i0 - 1 : 0, plast = i1 < c.Fx ? i1 : i1 - 1;
    const int hlo = max(0, f0 - c.hl), ehi = min(c.FyFz, f1 + c.hl);
    const int a0 = hlo & ~1, ae = (ehi + 1) & ~1, ah = (f1 + 1) & ~1;
    const uint32_t eb = (ae - a0) * 8u, hb = (ah - a0) * 8u, hst = (((f1 + 1) & ~1) - f0) * 8u;
    auto E = [&](int s, int k) { return (double*)(smem + (size_t)s * c.stage) + k * c.ecap; };
    auto H = [&](int s, int k) { return (double*)(smem + (size_t)s * c.stage) + 3 * c.ecap + k * c.hcap; };
    if (tid == 0) { for (int q = 0; q < 3; ++q) mbar_init(&bars[q], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    auto issue = [&](int p) {
        const int s = (p - pstart) % 3; const bool full = p < i1;
        expect_tx(&bars[s], 3 * eb + (full ? 3 * hb : 0));
        for (int k = 0; k < 3; ++k) tma_ld(E(s, k), P.Ea[k] + p * c.PP + a0, eb, &bars[s]);
        if (full) for (int k = 0; k < 3; ++k) tma_ld(H(s, k), P.Ha[k] + p * c.PP + a0, hb, &bars[s]);
    };
    const int issuer = NT - 32;
    if (tid == issuer) for (int p = pstart; p <= plast && p < pstart + 3; ++p) issue(p);
    double acc = 0.0;
    for (int p = pstart; p < i1; ++p) {
        const int s = (p - pstart) % 3, s1 = (p + 1 - pstart) % 3;
        wait_par(&bars[s], ((p - pstart) / 3) & 1);
        if (p + 1 <= plast) wait_par(&bars[s1], ((p + 1 - pstart) / 3) & 1);
        for (int g = hlo + tid; g < f1; g += NT) {   // "H": one add per component from E(p), E(p+1)
            const int e = g - a0;
            for (int k = 0; k < 3; ++k) H(s, k)[e] = H(s, k)[e] + E(s, k)[e] + E(s1, k)[e + 1];
        }
        __syncthreads();
        if (tid == issuer) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (c.ebulk == 2 && p - 1 >= i0) {   // E of the previous plane, written in place
                const int sp = (p - 1 - pstart) % 3;
                for (int k = 0; k < 3; ++k) tma_st(P.Eb[k] + (p - 1) * c.PP + f0, E(sp, k) + (f0 - a0), hst);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            if (p >= i0) for (int k = 0; k < 3; ++k) tma_st(P.Hb[k] + p * c.PP + f0, H(s, k) + (f0 - a0), hst);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            if (p > pstart && p + 2 <= plast) { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); issue(p + 2); }
        }
        if (p >= i0 && !c.ebulk)
            for (int f = f0 + tid; f < f1; f += NT) {   // "E": per-entry stores
                const int e = f - a0;
                for (int k = 0; k < 3; ++k) P.Eb[k][p * c.PP + f] = E(s, k)[e] + H(s, k)[e] + H(s, (k + 1) % 3)[e - 1];
            }
        if (p >= i0 && c.ebulk == 2)   // "E": in place, stored at the next barrier
            for (int f = f0 + tid; f < f1; f += NT) {
                const int e = f - a0;
                for (int k = 0; k < 3; ++k) E(s, k)[e] = E(s, k)[e] + H(s, k)[e];
            }
        if (p >= i0 && c.ebulk == 1) {   // "E": in place + bulk store after a barrier
            for (int f = f0 + tid; f < f1; f += NT) {
                const int e = f - a0;
                for (int k = 0; k < 3; ++k) E(s, k)[e] = E(s, k)[e] + H(s, k)[e];
            }
            __syncthreads();
            if (tid == issuer) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                for (int k = 0; k < 3; ++k) tma_st(P.Eb[k] + p * c.PP + f0, E(s, k) + (f0 - a0), hst);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        }
    }
    if (c.ebulk == 2) {
        __syncthreads();
        if (tid == issuer) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            const int sp = (i1 - 1 - pstart) % 3;
            for (int k = 0; k < 3; ++k) tma_st(P.Eb[k] + (i1 - 1) * c.PP + f0, E(sp, k) + (f0 - a0), hst);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (tid == issuer) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (acc == 1.2345) P.Eb[0][0] = acc;
}

int main(int argc, char** argv) {
    const int nx = 1024, ny = 1024, nz = 128, Fx = nx + 1, Fy = ny + 1, Fz = nz + 1;
    Cfg c{}; c.FyFz = Fy * Fz; c.PP = (c.FyFz + 31) / 32 * 32; c.Fx = Fx; c.T = argc > 1 ? atoi(argv[1]) : 512; c.hl = argc > 2 ? atoi(argv[2]) : Fz; c.ebulk = argc > 3 ? atoi(argv[3]) : 0;
    c.tiles = (c.FyFz + c.T - 1) / c.T; c.nchunks = 19; c.chunk = (Fx + c.nchunks - 1) / c.nchunks;
    c.ecap = (c.T + 2 * c.hl + 5) & ~1; c.hcap = (c.T + c.hl + 5) & ~1;
    c.stage = ((3 * c.ecap + 3 * c.hcap) * 8 + 127) / 128 * 128;
    const size_t n = (size_t)Fx * c.PP; double* buf;
    CK(cudaMalloc(&buf, 12 * n * 8)); CK(cudaMemset(buf, 0, 12 * n * 8));
    Ptr P; for (int k = 0; k < 3; ++k) { P.Ea[k] = buf + k * n; P.Ha[k] = buf + (3 + k) * n; P.Eb[k] = buf + (6 + k) * n; P.Hb[k] = buf + (9 + k) * n; }
    const int smem = 3 * c.stage;
    CK(cudaFuncSetAttribute(k_pattern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int grid = c.tiles * c.nchunks;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) k_pattern<<<grid, 256, smem>>>(P, c);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 20; ++r) k_pattern<<<grid, 256, smem>>>(P, c);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 20;
    const double cells = (double)nx * ny * nz;
    printf("pattern T=%d hl=%d ebulk=%d: %.3f ms  %.1f GB/s algorithmic (96 B/cell)\n", c.T, c.hl, c.ebulk, ms, cells * 96 / ms / 1e6);
    return 0;
}
