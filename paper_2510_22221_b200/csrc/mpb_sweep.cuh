// mpb_sweep.cuh -- the fused coupled-step sweep for sm_100a.
//
// One kernel computes, per entry, the plain H^{n+1} (magnetic cells too; the
// LLG of the few magnetic cells runs afterwards in k_llg_local / k_edefer) and
// E^{n+1} in a single pass over the lattice, so each of the 6 field arrays is
// read once and written once per step (96 B/cell in fp64, the roofline
// numerator of SURVEY 8d).
//
// Decomposition: each CTA owns a contiguous range [f0,f1) of T entries of an
// x-plane (a few z-rows; z is contiguous) and a chunk [i0,i1) of planes, and
// marches along x.  Per plane it stages, with 1-D TMA bulk copies into a
// 3-slot shared-memory ring (one mbarrier per slot):
//    E^n  on [f0 - Fz, f1 + Fz)  (row halo either side: H needs E at j+1,
//                                 k+1, the E update needs H at j-1, k-1)
//    H^n, material id on [f0 - Fz, f1)
// H^{n+1} of the plane is computed in place in shared memory (including the
// j-1 halo row, recomputed rather than exchanged), then E^{n+1} of the owned
// range is formed from it plus the previous plane's Hy, Hz kept in registers
// (the x-backward difference), so no x-halo is ever re-read from HBM except
// one plane per chunk.  One CTA barrier per plane (between the H and E
// phases); every thread waits on the slot's mbarrier itself.  Reads come from
// one ping-pong buffer set and writes go to the other, so CTAs never race on
// halos.
//
// Exactness: same operation order as the split kernels / the reference
// (em.py:117-139, 171-182, 206-272; llg.py:108-148); divisions by dx,dy,dz use
// ddiv() (bitwise IEEE, see mpb_device.cuh).
#pragma once

#include <type_traits>

#include "mpb_device.cuh"
#include "mpb_kernels_split.cuh"

namespace mpb {

// ---------------------------------------------------------------------------
// TMA 1-D bulk copy + mbarrier helpers (PTX)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
        "[%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// shared -> global bulk copy (async proxy), tracked by bulk groups
__device__ __forceinline__ void tma_store_1d(void* gdst, const void* ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
                 "r"(smem_u32(ssrc)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// all but the newest bulk group have finished reading shared memory
__device__ __forceinline__ void bulk_wait_read_all_but_1() {
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// ---------------------------------------------------------------------------
// launch-time layout of one CTA's staging ring
// ---------------------------------------------------------------------------
struct SweepCfg {
    int T;              // owned entries per CTA per plane
    int tiles;          // tiles per plane
    int chunk;          // planes per chunk
    int nchunks;
    int hl;             // low halo (entries) = Fz if y active, 1 if only z, else 0
    int eh;             // high E halo, same rule
    int ecap;           // doubles per E component slot
    int hcap;           // doubles per H component slot
    int icap;           // bytes of ids per slot
    uint32_t fz_magic;  // j = umulhi(f, magic) for f < FyFz
    int stage_bytes;    // bytes per ring slot
    int ch_base;        // chunk of blockIdx.x / tiles == 0 (launch subsets)
    int ch_step;        // chunk stride between consecutive block rows
    int nmat;           // entries of the material table
    int fastdiv;        // spacings within [2^-40, 2^10]: range-guarded divisions
    double rd[3];       // recip_of(d[a]) evaluated on the device at setup
    float rdf[3];       // fp32 storage mode: 1/d[a] rounded to float
    float coef_hf;      // fp32 storage mode: dt/mu0 rounded to float
    int mpre;           // LLG-first order: magnetic entries keep their staged H
    int mf0, mf1;       // entry range [mf0, mf1] of the magnetic cells in a plane
    int eguard;         // E-range flags maintained: the H phase may skip its guard
};

__global__ void k_recips(double dx, double dy, double dz, double* out) {
    out[0] = recip_of(dx);
    out[1] = recip_of(dy);
    out[2] = recip_of(dz);
}

constexpr int kSweepThreads = 512;
constexpr int kSlots = 3;

__device__ __forceinline__ int fz_div(uint32_t f, uint32_t magic) {
    return magic ? (int)__umulhi(f, magic) : (int)f;   // magic 0 <=> Fz == 1
}

// Self-test kernel: ddiv() against the compiler's IEEE division, bitwise.
__global__ void k_div_selftest(const double* __restrict__ x, int64_t n, double d,
                               unsigned long long* mismatches, double* first_bad) {
    const double y = recip_of(d);
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
         q += (int64_t)gridDim.x * blockDim.x) {
        const double a = ddiv(x[q], d, y);
        const double r = x[q] / d;
        if (__double_as_longlong(a) != __double_as_longlong(r) && !(a != a && r != r)) {
            if (atomicAdd(mismatches, 1ull) == 0ull) *first_bad = x[q];
        }
    }
}

// The exact slow path of a batch of six divisions (guard failed: zeros,
// subnormals, extreme exponents), out of line so the hot loop stays compact
// in the instruction cache.  Divisors (dy, dy, dz, dz, dx, dx) as in both
// curl batches.
struct Q6 { double q0, q1, q2, q3, q4, q5; };

// A failed batch guard is mostly exact zeros (fresh runs are zero almost
// everywhere for thousands of steps).  For x = +-0 the fast-path value is a
// zero of possibly the wrong sign, which cannot change any result: every
// quotient enters the curl sums (em.py:130-138, 217-231) that start from
// +0.0, and under round-to-nearest +0 + (+-0) and +0 - (+-0) are +0, so a
// sum never holds -0 and the sign of a zero term never shows.  So a batch
// whose failing numerators are all zeros keeps its fast-path quotients.
__device__ __forceinline__ bool in_range_or_zero(double x) {
    const unsigned u = ((unsigned)__double2hiint(x) << 1) - kGuardBias;
    return u <= kGuardSpan || x == 0.0;
}
__device__ __noinline__ Q6 slow_div6(double a0, double a1, double a2, double a3, double a4,
                                     double a5, double dx, double dy, double dz, double rx,
                                     double ry, double rz) {
    Q6 o;
    o.q0 = xdiv(a0, dy, ry); o.q1 = xdiv(a1, dy, ry);
    o.q2 = xdiv(a2, dz, rz); o.q3 = xdiv(a3, dz, rz);
    o.q4 = xdiv(a4, dx, rx); o.q5 = xdiv(a5, dx, rx);
    return o;
}

// H^{n+1} at one entry of the staged plane (in place in shared memory).
// Straight-line: all six differences and divisions are issued back to back
// and the division guard is checked once for the batch.
template <typename T>
struct HCtx {
    const T* Ex; const T* Ey; const T* Ez;
    const T* Ey1; const T* Ez1;
    T* Hx; T* Hy; T* Hz;
};

// fp32 storage mode: the same stencil in float arithmetic, divisions by the
// spacings as products with 1/d rounded to float (no bitwise contract: the
// mode is checked against the fp64 oracle within a stated tolerance)
__device__ __forceinline__ void h_entry_f32(const Geom& g, const HCtx<float>& c, int e, int j,
                                            int k, bool cellplane, int Fz, float ry, float rz,
                                            float rx, float& cx, float& cy, float& cz,
                                            bool& vx, bool& vy, bool& vz, bool ax, bool ay,
                                            bool az) {
    vx = j < g.n[1] && k < g.n[2];
    vy = cellplane && k < g.n[2];
    vz = cellplane && j < g.n[1];
    const float ex = c.Ex[e], ey = c.Ey[e], ez = c.Ez[e];
    const float q0 = (c.Ez[e + Fz] - ez) * ry;   // dEz/dy
    const float q1 = (c.Ex[e + Fz] - ex) * ry;   // dEx/dy
    const float q2 = (c.Ey[e + 1] - ey) * rz;    // dEy/dz
    const float q3 = (c.Ex[e + 1] - ex) * rz;    // dEx/dz
    const float q4 = (c.Ez1[e] - ez) * rx;       // dEz/dx
    const float q5 = (c.Ey1[e] - ey) * rx;       // dEy/dx
    cx = 0.f; cy = 0.f; cz = 0.f;
    if (ay) { cx = cx + q0; cz = cz - q1; }
    if (az) { cx = cx - q2; cy = cy + q3; }
    if (ax) { cy = cy - q4; cz = cz + q5; }
}

template <bool GUARD = true>
__device__ __forceinline__ void h_entry(const Geom& g, const HCtx<double>& c, int e, int j, int k,
                                        bool cellplane, int Fz, double ry, double rz,
                                        double rx, double& cx, double& cy, double& cz,
                                        bool& vx, bool& vy, bool& vz, bool g_fastdiv,
                                        bool ax, bool ay, bool az) {
    vx = j < g.n[1] && k < g.n[2];
    vy = cellplane && k < g.n[2];
    vz = cellplane && j < g.n[1];
    const double ex = c.Ex[e], ey = c.Ey[e], ez = c.Ez[e];
    const double a0 = c.Ez[e + Fz] - ez;   // dEz/dy
    const double a1 = c.Ex[e + Fz] - ex;   // dEx/dy
    const double a2 = c.Ey[e + 1] - ey;    // dEy/dz
    const double a3 = c.Ex[e + 1] - ex;    // dEx/dz
    const double a4 = c.Ez1[e] - ez;       // dEz/dx
    const double a5 = c.Ey1[e] - ey;       // dEy/dx
    // range guard per component group, masked by validity (padding entries
    // and collapsed axes never send an entry to the slow path)
    unsigned gX = 0, gY = 0, gZ = 0;
    double q0 = qdiv(a0, g.d[1], ry, gX);   // -> cEx
    double q1 = qdiv(a1, g.d[1], ry, gZ);   // -> cEz
    double q2 = qdiv(a2, g.d[2], rz, gX);   // -> cEx
    double q3 = qdiv(a3, g.d[2], rz, gY);   // -> cEy
    double q4 = qdiv(a4, g.d[0], rx, gY);   // -> cEy
    double q5 = qdiv(a5, g.d[0], rx, gZ);   // -> cEz
    // (GUARD = false: every E entry is known to be in range, kSafeBias)
    const bool bad = GUARD && (!g_fastdiv || (vx && gX > kGuardSpan) ||
                               (vy && gY > kGuardSpan) || (vz && gZ > kGuardSpan));
    if (__builtin_expect(bad, 0)) {
        bool fine = g_fastdiv;
        if (vx) fine = fine && in_range_or_zero(a0) && in_range_or_zero(a2);
        if (vy) fine = fine && in_range_or_zero(a3) && in_range_or_zero(a4);
        if (vz) fine = fine && in_range_or_zero(a1) && in_range_or_zero(a5);
        if (!fine) {
            const Q6 o = slow_div6(a0, a1, a2, a3, a4, a5, g.d[0], g.d[1], g.d[2], rx, ry, rz);
            q0 = o.q0; q1 = o.q1; q2 = o.q2; q3 = o.q3; q4 = o.q4; q5 = o.q5;
        }
    }
    // em.py:130-138 accumulation order, collapsed axes omitted
    cx = 0.0; cy = 0.0; cz = 0.0;
    if (ay) { cx = cx + q0; cz = cz - q1; }
    if (az) { cx = cx - q2; cy = cy + q3; }
    if (ax) { cy = cy - q4; cz = cz + q5; }
}

// PMC: some face is PMC (its ghost values enter the curl-H differences);
// false removes the ghost selects from the E phase at compile time (grids
// walled by PEC / MUR1 only, e.g. every benchmark configuration).
template <int V, bool F3, int NT = kSweepThreads, typename T = double, bool PMC = true>
// (fp32 two-CTA form: bound for 3 CTAs/SM -- 60 registers, +5% even at 2
// CTAs/SM; fp64: register caps of 88/80/72 all cost 6-8%)
#ifndef MPB_F32_CTAS
#define MPB_F32_CTAS 3
#endif
__global__ void __launch_bounds__(NT, NT == 256 ? (sizeof(T) == 4 ? MPB_F32_CTAS : 2) : 1)
k_sweep(Geom g, BufsT<T> b, const mpb_material* __restrict__ mats,
        const uint8_t* __restrict__ gids, StepState* st, SweepCfg sc) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t bars[kSlots];
    constexpr bool kF32 = sizeof(T) == 4;
    constexpr int A = 16 / (int)sizeof(T);   // entries per 16 bytes (TMA alignment)

    __shared__ T s_cacb[MPB_MAX_MATERIALS * 2];

    __shared__ T s_murz[MPB_MAX_MATERIALS];
    unsigned char* ring = smem;

    // launched behind the previous step's k_finish (see pdl_wait) -- or, with
    // Geom.llg_sync, behind the cooperative LLG kernel, which itself started
    // after that k_finish completed: no grid-wide wait then; the CTAs whose
    // staged H holds magnetic entries wait for the LLG's stamp instead
    if (!g.llg_sync) pdl_wait();
    if (st->fail) return;
    const int tid = threadIdx.x;
    const int tile = blockIdx.x % sc.tiles;
    const int chunk = sc.ch_base + (blockIdx.x / sc.tiles) * sc.ch_step;
    const int f0 = tile * sc.T;
    const int f1 = min(f0 + sc.T, g.FyFz);
    const int Fx = g.F[0];
    const int i0 = g.c0 + chunk * sc.chunk;          // owned planes [c0, c1)
    const int i1 = min(i0 + sc.chunk, g.c1);
    if (i0 >= i1) return;
    const int pstart = i0 > 0 ? i0 - 1 : 0;
    // last plane whose stage is needed: i1 (E only, for dEz/dx, dEy/dx of
    // plane i1-1) when it exists and x is active
    // F3: every axis active (3D grids) -- axis tests fold away at compile time
    const bool ax = F3 || g.act[0], ay = F3 || g.act[1], az = F3 || g.act[2];
    const int plast = (ax && i1 < Fx) ? i1 : i1 - 1;
    const int hlo = max(0, f0 - sc.hl);
    const int ehi = min(g.FyFz, f1 + sc.eh);
    const int a0 = hlo & ~(A - 1);                   // 16-byte aligned starts
    const int ae = (ehi + A - 1) & ~(A - 1);
    const int ah = (f1 + A - 1) & ~(A - 1);
    const int ia0 = hlo & ~15;
    const int iae = min((f1 + 16) & ~15, (int)g.PP);   // +1: z1-wall neighbour id
    const uint32_t ebytes = (uint32_t)(ae - a0) * (uint32_t)sizeof(T);
    const uint32_t hbytes = (uint32_t)(ah - a0) * (uint32_t)sizeof(T);
    const uint32_t ibytes = (uint32_t)(iae - ia0);
    const uint32_t hst_bytes = (uint32_t)(ah - f0) * (uint32_t)sizeof(T);   // 16-byte multiple

    for (int q = tid; q < sc.nmat; q += blockDim.x) {
        s_cacb[2 * q] = (T)mats[q].ca;
        s_cacb[2 * q + 1] = (T)mats[q].cb;
        s_murz[q] = (T)mats[q].mur_k[2];
    }
    if (tid == 0) {
        for (int q = 0; q < kSlots; ++q) mbar_init(&bars[q], 1);
        mbar_fence_init();
    }
    // Geom.llg_sync: a CTA whose staged planes / entries hold magnetic cells
    // waits here for the LLG of this step (the barrier below passes the
    // acquire on to the whole CTA)
    if (g.llg_sync && tid == NT - 32 && a0 <= sc.mf1 && ah > sc.mf0 && pstart < g.mx1 &&
        plast >= g.mx0)
        llg_await_tma(st);
    __syncthreads();

    // slot layout: E[3][ecap] | H[3][hcap] | ids[icap]
    auto slot = [&](int p) { return (p - pstart) % kSlots; };
    auto sE = [&](int s, int c) {
        return reinterpret_cast<T*>(ring + (size_t)s * sc.stage_bytes) + c * sc.ecap;
    };
    auto sH = [&](int s, int c) {
        return reinterpret_cast<T*>(ring + (size_t)s * sc.stage_bytes) +
               3 * sc.ecap + c * sc.hcap;
    };
    auto sI = [&](int s) {
        return ring + (size_t)s * sc.stage_bytes + (3 * sc.ecap + 3 * sc.hcap) * sizeof(T);
    };
    auto issue = [&](int p) {   // issuing thread only
        const int s = slot(p);
        const bool full = p < i1;
        const uint32_t bytes = 3 * ebytes + (full ? 3 * hbytes + ibytes : 0u);
        mbar_expect_tx(&bars[s], bytes);
        const int64_t base = (int64_t)p * g.PP;
        for (int c = 0; c < 3; ++c) tma_load_1d(sE(s, c), b.Ea[c] + base + a0, ebytes, &bars[s]);
        if (full) {
            for (int c = 0; c < 3; ++c)
                tma_load_1d(sH(s, c), b.Ha[c] + base + a0, hbytes, &bars[s]);
            tma_load_1d(sI(s), gids + base + ia0, ibytes, &bars[s]);
        }
    };
    // the refills are issued by lane 0 of the LAST warp: the strided H loop
    // gives low thread ids the extra (halo) entries, so the last warp has
    // slack to absorb the issue time before the plane barrier
    constexpr int kIssuer = NT - 32;
    // H^{n+1} written by bulk stores from the slot (two-CTA 256-thread form:
    // +3-4% on C4); the one-CTA forms keep per-entry stores -- there the
    // issuing warp's wait for the previous plane's stores stalls the whole SM
    constexpr bool kBulkH = NT == 256;
    if (tid == kIssuer)
        for (int p = pstart; p <= plast && p < pstart + kSlots; ++p) issue(p);

    // reciprocals of the spacings: recip_of() evaluated once at setup on the
    // device (identical bits); passing them keeps MUFU + 5 DFMA out of the loop
    const double rx = sc.rd[0], ry = sc.rd[1], rz = sc.rd[2];
    const float rfx = sc.rdf[0], rfy = sc.rdf[1], rfz = sc.rdf[2];
    const int Fz = g.F[2];
    const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
    // collapsed axes: their (unused) quotients must not trip the guard
    const bool fastdiv = sc.fastdiv != 0 && ax && ay && az;
    // the E set this sweep reads is in range: no guard in the H phase
    const bool hsafe = !kF32 && fastdiv && sc.eguard && st->eunsafe_a == 0;
    unsigned eg = 0;   // e_range of the valid E values written (next step's flag)
    const bool zw0 = g.zin && az && g.faces[4] != MPB_FACE_PMC;
    const bool zw1 = g.zin && az && g.faces[5] != MPB_FACE_PMC;
    const bool z0pec = g.faces[4] == MPB_FACE_PEC, z1pec = g.faces[5] == MPB_FACE_PEC;
    const bool pmc_x0 = PMC && g.faces[0] == MPB_FACE_PMC;
    const bool pmc_x1 = PMC && g.faces[1] == MPB_FACE_PMC;
    const bool pmc_y0 = PMC && g.faces[2] == MPB_FACE_PMC;
    const bool pmc_y1 = PMC && g.faces[3] == MPB_FACE_PMC;
    const bool pmc_z0 = PMC && g.faces[4] == MPB_FACE_PMC;
    const bool pmc_z1 = PMC && g.faces[5] == MPB_FACE_PMC;

    T hy_prev[V], hz_prev[V];
#pragma unroll
    for (int v = 0; v < V; ++v) { hy_prev[v] = T(0); hz_prev[v] = T(0); }
    // The E-phase entries of a thread are the same on every plane: in fp32
    // their row / column tests are evaluated once, as bits, before the plane
    // loop (+4% on C4: that kernel is issue-bound); fp64 keeps the direct
    // per-plane comparisons (the extra registers cost it 4%)
    constexpr unsigned kLive = 1u, kJ0 = 2u, kJn = 4u, kK0 = 8u, kKn = 16u, kK1 = 32u,
                       kKn1 = 64u, kZx = 128u, kJlt = 256u, kKlt = 512u;
    auto entry_flags = [&](int f) -> unsigned {
        if (f >= f1) return 0u;
        const int j = fz_div((uint32_t)f, sc.fz_magic);
        const int k = f - j * Fz;
        return kLive | (j == 0 ? kJ0 : 0u) | (j == ny ? kJn : 0u) | (k == 0 ? kK0 : 0u) |
               (k == nz ? kKn : 0u) | (k == 1 ? kK1 : 0u) | (k == nz - 1 ? kKn1 : 0u) |
               (!(ay && (j <= 1 || j >= ny - 1)) ? kZx : 0u) | (j < ny ? kJlt : 0u) |
               (k < nz ? kKlt : 0u);
    };
    unsigned efl[V];
#pragma unroll
    for (int v = 0; v < V; ++v) efl[v] = kF32 ? entry_flags(f0 + tid + v * NT) : 0u;

    for (int p = pstart; p <= i1 - 1; ++p) {
        const int s = slot(p);
        const bool xnext = ax && p < nx;                 // plane p+1 used by dx terms
        const int s1 = slot(p + 1);
        // every thread waits for the staged planes itself (no CTA barrier
        // here): the only barrier per plane is the one between the phases
        mbar_wait(&bars[s], ((p - pstart) / kSlots) & 1);
        if (xnext) mbar_wait(&bars[s1], ((p + 1 - pstart) / kSlots) & 1);
        HCtx<T> hc{sE(s, 0), sE(s, 1), sE(s, 2), sE(s1, 1), sE(s1, 2),
                   sH(s, 0), sH(s, 1), sH(s, 2)};
        const unsigned char* ids = sI(s);
        const bool emit = p >= i0;
        const bool cellplane = p < nx || !ax;

        // ---- H^{n+1}(p, g) for g in [hlo, f1), in place --------------------
        // LLG-first order: the staged H of a magnetic cell is already its
        // H^{n+1} (k_llg_pre); a plane / tile outside the cells' box skips the test
        const bool pm = sc.mpre && p >= g.mx0 && p < g.mx1 && hlo <= sc.mf1 && f1 > sc.mf0;
        // two copies of the loop: the test sits only in the one run by the
        // planes / tiles that hold magnetic cells (in the common loop even a
        // predicated test cost the C4 sweep 2.5%)
        auto h_phase = [&](auto PM, auto SAFE) {
            for (int gg = hlo + tid; gg < f1; gg += NT) {
                const int j = fz_div((uint32_t)gg, sc.fz_magic);
                const int k = gg - j * Fz;
                const int e = gg - a0;
                bool vx, vy, vz;
                // otherwise magnetic cells get the plain update here too;
                // k_llg_local replaces their H (and the E entries around them, k_edefer)
                bool keep = false;
                if constexpr (decltype(PM)::value)
                    keep = (ids[gg - ia0] & 0x80u) && j < ny && k < nz && cellplane;
                if constexpr (kF32) {
                    float cx, cy, cz;
                    h_entry_f32(g, hc, e, j, k, cellplane, Fz, rfy, rfz, rfx, cx, cy, cz, vx,
                                vy, vz, ax, ay, az);
                    vx = vx && !keep; vy = vy && !keep; vz = vz && !keep;
                    if (vx) hc.Hx[e] = hc.Hx[e] - sc.coef_hf * cx;
                    if (vy) hc.Hy[e] = hc.Hy[e] - sc.coef_hf * cy;
                    if (vz) hc.Hz[e] = hc.Hz[e] - sc.coef_hf * cz;
                } else {
                    double cx, cy, cz;
                    h_entry<!decltype(SAFE)::value>(g, hc, e, j, k, cellplane, Fz, ry, rz, rx,
                                                      cx, cy, cz, vx, vy, vz, fastdiv, ax, ay,
                                                      az);
                    vx = vx && !keep; vy = vy && !keep; vz = vz && !keep;
                    if (vx) hc.Hx[e] = hc.Hx[e] - g.coef_h * cx;
                    if (vy) hc.Hy[e] = hc.Hy[e] - g.coef_h * cy;
                    if (vz) hc.Hz[e] = hc.Hz[e] - g.coef_h * cz;
                }
            }
        };
        if (hsafe) {
            if (pm) h_phase(std::true_type{}, std::true_type{});
            else h_phase(std::false_type{}, std::true_type{});
        } else {
            if (pm) h_phase(std::true_type{}, std::false_type{});
            else h_phase(std::false_type{}, std::false_type{});
        }
        // H^{n+1}(p) complete everywhere, and every thread is past E(p-1) and
        // H(p), the last readers of plane p-1's slot: refill it with p+2
        __syncthreads();
        if (tid == kIssuer) {
            fence_proxy_async();   // the H updates above -> async proxy
            if constexpr (kBulkH) {
                // H^{n+1} of the owned range leaves straight from the slot:
                // three bulk stores instead of a store per entry and component
                // (padding entries carry their staged zeros); the ghost plane
                // of a slab is written too (k_edefer reads it pre-exchange)
                if (p >= i0 || p == g.c0 - 1) {
                    const int64_t pb = (int64_t)p * g.PP;
                    for (int c = 0; c < 3; ++c)
                        tma_store_1d(b.Hb[c] + pb + f0, sH(s, c) + (f0 - a0), hst_bytes);
                }
                bulk_commit();
            }
            if (p > pstart && p + 2 <= plast) {
                if constexpr (kBulkH) bulk_wait_read_all_but_1();   // p-1's stores left its slot
                issue(p + 2);
            }
        }

        // ---- E^{n+1}(p, f) for the owned range ------------------------------
        const T* Hx = hc.Hx;
        const T* Hy = hc.Hy;
        const T* Hz = hc.Hz;
        const int64_t base = (int64_t)p * g.PP;
        const bool zy = !(ax && (p <= 1 || p >= nx - 1));   // (per plane)
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const int f = f0 + tid + v * NT;
            // the entry's row / column tests: fp32 from the precomputed bits,
            // fp64 as direct comparisons
            bool live, j0, jn, k0, kn, k1, kn1, zx, jlt, klt;
            if constexpr (kF32) {
                const unsigned fl = efl[v];
                live = fl & kLive; j0 = fl & kJ0; jn = fl & kJn; k0 = fl & kK0; kn = fl & kKn;
                k1 = fl & kK1; kn1 = fl & kKn1; zx = fl & kZx; jlt = fl & kJlt; klt = fl & kKlt;
            } else {
                live = f < f1;
                const int j = fz_div((uint32_t)f, sc.fz_magic);
                const int k = f - j * Fz;
                j0 = j == 0; jn = j == ny; k0 = k == 0; kn = k == nz; k1 = k == 1;
                kn1 = k == nz - 1; zx = !(ay && (j <= 1 || j >= ny - 1)); jlt = j < ny;
                klt = k < nz;
            }
            if (live) {
                const int e = f - a0;
                const T hx = Hx[e], hy = Hy[e], hz = Hz[e];
                if (emit) {
                    const int ejm = j0 ? e : e - Fz;      // clamp: never read off-range
                    const int ekm = k0 ? e : e - 1;
                    const T hz_jm = Hz[ejm], hx_jm = Hx[ejm];
                    const T hy_km = Hy[ekm], hx_km = Hx[ekm];
                    const T zero = T(0);
                    // backward differences with PMC ghosts (em.py:185-203)
                    const T zhi = jn ? (pmc_y1 ? -hz_jm : zero) : hz;
                    const T zlo = j0 ? (pmc_y0 ? -hz : zero) : hz_jm;
                    const T xhi = jn ? (pmc_y1 ? -hx_jm : zero) : hx;
                    const T xlo = j0 ? (pmc_y0 ? -hx : zero) : hx_jm;
                    const T yhi_k = kn ? (pmc_z1 ? -hy_km : zero) : hy;
                    const T ylo_k = k0 ? (pmc_z0 ? -hy : zero) : hy_km;
                    const T xhi_k = kn ? (pmc_z1 ? -hx_km : zero) : hx;
                    const T xlo_k = k0 ? (pmc_z0 ? -hx : zero) : hx_km;
                    const T zhi_i = (p == nx) ? (pmc_x1 ? -hz_prev[v] : zero) : hz;
                    const T zlo_i = (p == 0) ? (pmc_x0 ? -hz : zero) : hz_prev[v];
                    const T yhi_i = (p == nx) ? (pmc_x1 ? -hy_prev[v] : zero) : hy;
                    const T ylo_i = (p == 0) ? (pmc_x0 ? -hy : zero) : hy_prev[v];
                    const T b0 = zhi - zlo, b1 = xhi - xlo, b2 = yhi_k - ylo_k;
                    const T b3 = xhi_k - xlo_k, b4 = zhi_i - zlo_i, b5 = yhi_i - ylo_i;
                    T q0, q1, q2, q3, q4, q5;
                    if constexpr (kF32) {
                        q0 = b0 * rfy; q1 = b1 * rfy; q2 = b2 * rfz;
                        q3 = b3 * rfz; q4 = b4 * rfx; q5 = b5 * rfx;
                    } else {
                        unsigned gg2 = 0;
                        q0 = qdiv(b0, g.d[1], ry, gg2); q1 = qdiv(b1, g.d[1], ry, gg2);
                        q2 = qdiv(b2, g.d[2], rz, gg2); q3 = qdiv(b3, g.d[2], rz, gg2);
                        q4 = qdiv(b4, g.d[0], rx, gg2); q5 = qdiv(b5, g.d[0], rx, gg2);
                        if (__builtin_expect(!fastdiv || gg2 > kGuardSpan, 0)) {
                            const bool fine = fastdiv && in_range_or_zero(b0) &&
                                              in_range_or_zero(b1) && in_range_or_zero(b2) &&
                                              in_range_or_zero(b3) && in_range_or_zero(b4) &&
                                              in_range_or_zero(b5);
                            if (!fine) {
                                const Q6 o = slow_div6(b0, b1, b2, b3, b4, b5, g.d[0], g.d[1],
                                                       g.d[2], rx, ry, rz);
                                q0 = o.q0; q1 = o.q1; q2 = o.q2; q3 = o.q3; q4 = o.q4;
                                q5 = o.q5;
                            }
                        }
                    }
                    T cx = zero, cy = zero, cz = zero;   // em.py:217-231 order
                    if (ay) { cx = cx + q0; cz = cz - q1; }
                    if (az) { cx = cx - q2; cy = cy + q3; }
                    if (ax) { cy = cy - q4; cz = cz + q5; }
                    const int id = ids[f - ia0];
                    const T ca = s_cacb[2 * id], cb = s_cacb[2 * id + 1];
                    const T* Ex = hc.Ex;
                    const T* Ey = hc.Ey;
                    const T* Ez = hc.Ez;
                    const T exa = Ex[e], eya = Ey[e];
                    const T w0 = ca * (cx - cb * exa);
                    const T w1 = ca * (cy - cb * eya);
                    const T w2 = ca * (cz - cb * Ez[e]);
                    const uint32_t o = (uint32_t)base + (uint32_t)f;
                    // z walls (em.py:336-359) in the sweep: the owner of the inner
                    // entry (k=1 / k=nz-1) writes the tangential wall value; lines
                    // an x/y wall reads or writes are left to k_zfix (run after the
                    // x/y wall kernels, preserving the face order x0..z1)
                    bool wx = true, wy = true;
                    if ((zw0 && k0) || (zw1 && kn)) { wx = !zx; wy = !zy; }
                    if (wx) b.Eb[0][o] = w0;
                    if (wy) b.Eb[1][o] = w1;
                    b.Eb[2][o] = w2;
                    // valid entries: Ex on cell planes, Ey below row ny, Ez below nz
                    if constexpr (!kF32) {
                        if (wx && cellplane) eg = max(eg, e_range(w0));
                        if (wy && jlt) eg = max(eg, e_range(w1));
                        if (klt) eg = max(eg, e_range(w2));
                    }
                    if (zw0 && k1) {
                        const T kk = s_murz[ids[f - 1 - ia0]];
                        const T v0 = z0pec ? zero : exa + kk * (w0 - Ex[e - 1]);
                        const T v1 = z0pec ? zero : eya + kk * (w1 - Ey[e - 1]);
                        if (zx) b.Eb[0][o - 1] = v0;
                        if (zy) b.Eb[1][o - 1] = v1;
                        if constexpr (!kF32) {
                            if (zx && cellplane) eg = max(eg, e_range(v0));
                            if (zy && jlt) eg = max(eg, e_range(v1));
                        }
                    }
                    if (zw1 && kn1) {
                        const T kk = s_murz[ids[f + 1 - ia0]];
                        const T v0 = z1pec ? zero : exa + kk * (w0 - Ex[e + 1]);
                        const T v1 = z1pec ? zero : eya + kk * (w1 - Ey[e + 1]);
                        if (zx) b.Eb[0][o + 1] = v0;
                        if (zy) b.Eb[1][o + 1] = v1;
                        if constexpr (!kF32) {
                            if (zx && cellplane) eg = max(eg, e_range(v0));
                            if (zy && jlt) eg = max(eg, e_range(v1));
                        }
                    }
                    if constexpr (!kBulkH) {
                        const bool cp = p < nx || !ax;
                        if (jlt && klt) b.Hb[0][o] = hx;
                        if (cp && klt) b.Hb[1][o] = hy;
                        if (cp && jlt) b.Hb[2][o] = hz;
                    }
                } else if (!kBulkH && p == g.c0 - 1) {
                    // low ghost plane of a slab: its H^{n+1} is read by k_edefer
                    // (x-backward difference at plane c0) before the exchange
                    // delivers the owner's copy (identical values)
                    const uint32_t o = (uint32_t)base + (uint32_t)f;
                    if (jlt && klt) b.Hb[0][o] = hx;
                    if (klt) b.Hb[1][o] = hy;
                    if (jlt) b.Hb[2][o] = hz;
                }
                hy_prev[v] = hy;
                hz_prev[v] = hz;
            }
        }
    }
    if constexpr (!kF32)
        if (sc.eguard) flag_e_range(eg, &st->eunsafe_b);
    if (kBulkH && tid == kIssuer) bulk_wait_all();   // slots live until the stores read them
}

// LLG of the magnetic cells after the (pure Maxwell) sweep: each cell runs
// its fixed point to its local stop from the untouched step-n state (E^n for
// curl E, H^n, M^n) and writes H^{n+1}, M^{n+1}; per-block residual history and
// local-stop range feed the global stop rule (k_llg_fixup / all-reduce).
// Ghost-plane copies (slabs) are computed for their H only.
#ifndef MPB_LLG_MINB
#define MPB_LLG_MINB 2
#endif
// One magnetic cell's fixed point to its local stop (CTA statistics in cs).
template <typename T>
__device__ __forceinline__ void llg_local_cell(const Geom& g, const BufsT<T>& b,
                                               const mpb_material* __restrict__ mats,
                                               const uint8_t* __restrict__ ids,
                                               const int2* __restrict__ cells,
                                               const unsigned char* __restrict__ owned, int q,
                                               CtaLlgStats& cs) {
    {
        const int i = cells[q].x, f = cells[q].y;
        const int64_t o = i * g.PP + f;
        const int64_t om = (int64_t)(i - g.mx0) * g.PP + f;
        LlgCell s;
        // H^n, M^n and the material id are loaded before the curl's divisions
        // (see curl_e_at) so every load of the cell is in flight at once
        for (int k = 0; k < 3; ++k) { s.Hn[k] = b.Ha[k][o]; s.Mn[k] = b.Ma[k][om]; }
        const uint8_t id = ids[o];
        const Curl3 c = curl_e_at(g, b.Ea, o, g.PP, g.F[2], true, true, true);
        s.cE[0] = c.x; s.cE[1] = c.y; s.cE[2] = c.z;
        llg_setup(s, mats[id]);
        const bool own = owned[q] != 0;
        double Hr[3] = {s.Hn[0], s.Hn[1], s.Hn[2]};
        double Mr[3] = {s.Mn[0], s.Mn[1], s.Mn[2]};
        int rc = g.max_iters + 1;
        for (int r = 1; r <= g.max_iters; ++r) {
            const double res = llg_iterate(s, g.coef_h, Hr, Mr);
            if (own) atomicMax(&cs.hist[r], dbits(res));
            if (res <= g.tol) { rc = r; break; }
        }
        for (int k = 0; k < 3; ++k) b.Hb[k][o] = Hr[k];
        if (own) {
            for (int k = 0; k < 3; ++k) b.Mb[k][om] = Mr[k];
            atomicMin(&cs.rc[0], rc);
            atomicMax(&cs.rc[1], rc);
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(256, MPB_LLG_MINB) k_llg_local(Geom g, BufsT<T> b,
                                                   const mpb_material* __restrict__ mats,
                                                   const uint8_t* __restrict__ ids,
                                                   const int2* __restrict__ cells,
                                                   const unsigned char* __restrict__ owned,
                                                   int ncells, StepState* st) {
    extern __shared__ unsigned long long lhist[];
    __shared__ int lrc[2];
    pdl_wait();
    pdl_trigger();
    if (st->fail) return;
    CtaLlgStats cs{lhist, lrc};
    cta_stats_init(cs, g.max_iters);
    __syncthreads();
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < ncells) llg_local_cell(g, b, mats, ids, cells, owned, q, cs);
    __syncthreads();
    if (lrc[1] > 0) cta_stats_flush(cs, g.max_iters, st);
}

// LLG-first order (MagPre): one magnetic cell to its local stop from the
// compact step-n copy; H^{n+1} goes to the compact copy and, in place, to the
// lattice H^n the sweep stages next; M^{n+1} to the compact copy only (the
// lattice M of magnetic cells is refreshed from it when a snapshot or the
// energy reads it; M probes read the compact copy).  Single rank: every cell
// is owned.
template <typename T>
__global__ void __launch_bounds__(256, MPB_LLG_MINB) k_llg_pre(Geom g, BufsT<T> b,
                                                 const mpb_material* __restrict__ mats,
                                                 MagPre<T> mp, const int2* __restrict__ cells,
                                                 int ncells, StepState* st) {
    extern __shared__ unsigned long long lhist[];
    __shared__ int lrc[2];
    pdl_wait();
    pdl_trigger();
    if (st->fail) return;
    CtaLlgStats cs{lhist, lrc};
    cta_stats_init(cs, g.max_iters);
    __syncthreads();
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < ncells) {
        const int i = cells[q].x, f = cells[q].y;
        const int64_t o = i * g.PP + f;
        LlgCell s;
        for (int k = 0; k < 3; ++k) { s.Hn[k] = (double)mp.Hn[k][q]; s.Mn[k] = mp.Mn[k][q]; }
        const uint8_t id = mp.cid[q];
        const Curl3 c = curl_e_at(g, b.Ea, o, g.PP, g.F[2], true, true, true);
        s.cE[0] = c.x; s.cE[1] = c.y; s.cE[2] = c.z;
        llg_setup(s, mats[id]);
        double Hr[3] = {s.Hn[0], s.Hn[1], s.Hn[2]};
        double Mr[3] = {s.Mn[0], s.Mn[1], s.Mn[2]};
        int rc = g.max_iters + 1;
        for (int r = 1; r <= g.max_iters; ++r) {
            const double res = llg_iterate(s, g.coef_h, Hr, Mr);
            atomicMax(&cs.hist[r], dbits(res));
            if (res <= g.tol) { rc = r; break; }
        }
        for (int k = 0; k < 3; ++k) {
            const T hv = (T)Hr[k];
            mp.Hl[k][o] = hv;
            mp.Hn1[k][q] = hv;
            mp.Mn1[k][q] = Mr[k];
        }
        atomicMin(&cs.rc[0], rc);
        atomicMax(&cs.rc[1], rc);
    }
    __syncthreads();
    if (lrc[1] > 0) cta_stats_flush(cs, g.max_iters, st);
}

// The same, fused with the r* settlement: a cooperative grid of co-resident
// blocks strides over the cells, then one grid barrier and the fixup
// (uniform replay or lockstep recompute) -- one launch instead of two.
template <typename T>
__global__ void __launch_bounds__(256, MPB_LLG_MINB) k_llg_pre_coop(
    Geom g, BufsT<T> b, const mpb_material* __restrict__ mats, MagPre<T> mp,
    const uint8_t* __restrict__ ids, const int2* __restrict__ cells, int ncells,
    MagScratch scr, StepState* st) {
    extern __shared__ unsigned long long lhist[];
    __shared__ int lrc[2];
    if (g.llg_sync) pdl_trigger();   // the sweep's blocks may start now
    const long long step = st->step;
    if (st->fail) {
        if (g.llg_sync && threadIdx.x == 0) llg_publish(st, step);
        return;
    }
    CtaLlgStats cs{lhist, lrc};
    cta_stats_init(cs, g.max_iters);
    __syncthreads();
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < ncells; q += gridDim.x * blockDim.x) {
        const int i = cells[q].x, f = cells[q].y;
        const int64_t o = i * g.PP + f;
        LlgCell s;
        for (int k = 0; k < 3; ++k) { s.Hn[k] = (double)mp.Hn[k][q]; s.Mn[k] = mp.Mn[k][q]; }
        const uint8_t id = mp.cid[q];
        const Curl3 c = curl_e_at(g, b.Ea, o, g.PP, g.F[2], true, true, true);
        s.cE[0] = c.x; s.cE[1] = c.y; s.cE[2] = c.z;
        llg_setup(s, mats[id]);
        double Hr[3] = {s.Hn[0], s.Hn[1], s.Hn[2]};
        double Mr[3] = {s.Mn[0], s.Mn[1], s.Mn[2]};
        int rc = g.max_iters + 1;
        for (int r = 1; r <= g.max_iters; ++r) {
            const double res = llg_iterate(s, g.coef_h, Hr, Mr);
            atomicMax(&cs.hist[r], dbits(res));
            if (res <= g.tol) { rc = r; break; }
        }
        for (int k = 0; k < 3; ++k) {
            const T hv = (T)Hr[k];
            mp.Hl[k][o] = hv;
            mp.Hn1[k][q] = hv;
            mp.Mn1[k][q] = Mr[k];
        }
        atomicMin(&cs.rc[0], rc);
        atomicMax(&cs.rc[1], rc);
    }
    __syncthreads();
    if (lrc[1] > 0) cta_stats_flush(cs, g.max_iters, st);
    cg::this_grid().sync();
    llg_fixup_grid(g, b, mats, ids, cells, ncells, scr, st, mp);
    if (g.llg_sync) {
        __syncthreads();
        if (threadIdx.x == 0) llg_publish(st, step);
    }
}

// compact step-n copy of the magnetic cells' H and M from the lattice
// (after a state load)
template <typename T>
__global__ void k_mag_pack(Geom g, BufsT<T> b, MagPre<T> mp, const int2* __restrict__ cells,
                           int ncells) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= ncells) return;
    const int i = cells[q].x, f = cells[q].y;
    const int64_t o = i * g.PP + f;
    const int64_t om = (int64_t)(i - g.mx0) * g.PP + f;
    for (int k = 0; k < 3; ++k) {
        const_cast<T*>(mp.Hn[k])[q] = b.Ha[k][o];
        const_cast<double*>(mp.Mn[k])[q] = b.Ma[k][om];
    }
}

// lattice M of the magnetic cells from the compact copy (LLG-first order:
// before a snapshot / energy evaluation reads the lattice)
template <typename T>
__global__ void k_mag_unpack(Geom g, double* M0, double* M1, double* M2, MagPre<T> mp,
                             const int2* __restrict__ cells, int ncells) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= ncells) return;
    const int64_t om = (int64_t)(cells[q].x - g.mx0) * g.PP + cells[q].y;
    M0[om] = mp.Mn[0][q];
    M1[om] = mp.Mn[1][q];
    M2[om] = mp.Mn[2][q];
}

// E entries whose curl-H stencil touches a magnetic H entry, recomputed after
// the LLG fixup settled r* (only when the fixup had to recompute).  Uses the
// sweep's z-wall write rules so the in-sweep z walls stay consistent.
// One deferred E entry (the sweep's z-wall write rules).
template <typename T>
__device__ __forceinline__ void edefer_entry(const Geom& g, const BufsT<T>& b,
                                             const mpb_material* __restrict__ mats,
                                             const uint8_t* __restrict__ ids,
                                             const int2* __restrict__ list, int q) {
    const int i = list[q].x, f = list[q].y;
    const int j = f / g.F[2];
    const int k = f - j * g.F[2];
    const int64_t o = i * g.PP + f;
    const E3 w = e_plain_at(g, b, mats, ids, i, j, k, o);
    const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
    const bool az = g.act[2];
    const bool zw0 = g.zin && az && g.faces[4] != MPB_FACE_PMC;
    const bool zw1 = g.zin && az && g.faces[5] != MPB_FACE_PMC;
    const bool z0pec = g.faces[4] == MPB_FACE_PEC, z1pec = g.faces[5] == MPB_FACE_PEC;
    const bool zx = !(g.act[1] && (j <= 1 || j >= ny - 1));
    const bool zy = !(g.act[0] && (i <= 1 || i >= nx - 1));
    bool wx = true, wy = true;
    if ((zw0 && k == 0) || (zw1 && k == nz)) { wx = !zx; wy = !zy; }
    if (wx) b.Eb[0][o] = w.x;
    if (wy) b.Eb[1][o] = w.y;
    b.Eb[2][o] = w.z;
    if (zw0 && k == 1) {
        const double kk = mats[ids[o - 1]].mur_k[2];
        if (zx) b.Eb[0][o - 1] = z0pec ? 0.0 : b.Ea[0][o] + kk * (w.x - b.Ea[0][o - 1]);
        if (zy) b.Eb[1][o - 1] = z0pec ? 0.0 : b.Ea[1][o] + kk * (w.y - b.Ea[1][o - 1]);
    }
    if (zw1 && k == nz - 1) {
        const double kk = mats[ids[o + 1]].mur_k[2];
        if (zx) b.Eb[0][o + 1] = z1pec ? 0.0 : b.Ea[0][o] + kk * (w.x - b.Ea[0][o + 1]);
        if (zy) b.Eb[1][o + 1] = z1pec ? 0.0 : b.Ea[1][o] + kk * (w.y - b.Ea[1][o + 1]);
    }
}

template <typename T>
__global__ void __launch_bounds__(256) k_edefer(Geom g, BufsT<T> b,
                                                const mpb_material* __restrict__ mats,
                                                const uint8_t* __restrict__ ids,
                                                const int2* __restrict__ list, int n,
                                                const StepState* st, int always) {
    pdl_wait();
    pdl_trigger();
    if (st->fail || (!always && !st->fixup_ran)) return;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < n) edefer_entry(g, b, mats, ids, list, q);
}

// z walls on the lines the sweep leaves alone: Ex on rows j in {0,1,ny-1,ny}
// and Ey on planes i in {0,1,nx-1,nx} -- the lines x/y walls read (pre-z
// values) or write (post-x/y inner values).  Runs after the x/y wall
// kernels, so the reference face order x0,x1,y0,y1,z0,z1 holds.
// list entries: (comp, i, j) packed as int3.
// One z-wall fix-up line entry (see k_zfix).
template <typename T>
__device__ __forceinline__ unsigned zfix_line(const Geom& g, const BufsT<T>& b,
                                              const mpb_material* __restrict__ mats,
                                              const uint8_t* __restrict__ ids,
                                              const int3* __restrict__ lines, int q,
                                              int fail) {
    const int c = lines[q].x, i = lines[q].y, j = lines[q].z;
    const int64_t row = i * g.PP + (int64_t)j * g.F[2];
    const int nz = g.n[2];
    const bool valid = c == 0 ? i < g.n[0] : j < g.n[1];   // Ex / Ey entry exists
    // both faces' loads before either store (one round trip, not two); with
    // nz == 1 the z1 inner entry is the z0 wall just written: re-read it
    const bool m0 = g.faces[4] == MPB_FACE_MUR1, m1 = g.faces[5] == MPB_FACE_MUR1;
    const int64_t ow0 = row, oi0 = row + 1, ow1 = row + nz, oi1 = row + nz - 1;
    double a0i = 0, b0i = 0, a0w = 0, a1i = 0, b1i = 0, a1w = 0;
    uint8_t id0 = 0, id1 = 0;
    if (m0) { a0i = b.Ea[c][oi0]; b0i = b.Eb[c][oi0]; a0w = b.Ea[c][ow0]; id0 = ids[ow0]; }
    if (m1) { a1i = b.Ea[c][oi1]; b1i = b.Eb[c][oi1]; a1w = b.Ea[c][ow1]; id1 = ids[ow1]; }
    if (fail) return 0u;
    unsigned eg = 0;
    if (g.faces[4] != MPB_FACE_PMC) {     // z0: wall 0, inner 1
        const T v = !m0 ? T(0) : T(a0i + mats[id0].mur_k[2] * (b0i - a0w));
        b.Eb[c][ow0] = v;
        if (valid) eg = max(eg, e_range((double)v));
    }
    if (g.faces[5] != MPB_FACE_PMC) {     // z1: wall nz, inner nz-1
        if (m1 && oi1 == ow0) b1i = b.Eb[c][oi1];
        const T v = !m1 ? T(0) : T(a1i + mats[id1].mur_k[2] * (b1i - a1w));
        b.Eb[c][ow1] = v;
        if (valid) eg = max(eg, e_range((double)v));
    }
    return eg;
}

template <typename T>
__global__ void __launch_bounds__(256) k_zfix(Geom g, BufsT<T> b,
                                              const mpb_material* __restrict__ mats,
                                              const uint8_t* __restrict__ ids,
                                              const int3* __restrict__ lines, int n,
                                              StepState* st) {
    pdl_wait();
    pdl_trigger();
    const int fail = st->fail;   // in flight with the line's loads
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned eg = q < n ? zfix_line(g, b, mats, ids, lines, q, fail) : 0u;
    if (fail) return;
    if (g.eguard) flag_e_range(eg, &st->eunsafe_b);
}

}  // namespace mpb
