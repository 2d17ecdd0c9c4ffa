// mpb_sweep.cuh -- the fused coupled-step sweep for sm_100a.
//
// One kernel computes, per entry, H^{n+1} (plain update or the cell's LLG
// fixed point to its local stop) and E^{n+1} in a single pass over the
// lattice, so each of the 6 field arrays is read once and written once per
// step (96 B/cell in fp64, the roofline numerator of SURVEY 8d).
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
// one plane per chunk.  Reads come from one ping-pong buffer set and writes
// go to the other, so CTAs never race on halos.
//
// Exactness: same operation order as the split kernels / the reference
// (em.py:117-139, 171-182, 206-272; llg.py:108-148); divisions by dx,dy,dz use
// ddiv() (bitwise IEEE, see mpb_device.cuh).
#pragma once

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
    int ring_offset;    // bytes of dynamic smem before the ring (LLG history)
    int nmat;           // entries of the material table
    int fastdiv;        // spacings within [2^-40, 2^10]: range-guarded divisions
    int slots;          // ring depth (3 or 4)
};

constexpr int kMagneticIdBit = 0x80;   // material ids >= 128 are magnetic
constexpr int kMaxSlots = 4;

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

// LLG for one cell, kept out of line so the rare path does not inflate the
// register allocation of the streaming path.
__device__ __noinline__ int llg_cell_local(const mpb_material* __restrict__ mats, int id,
                                          const Geom* gp, const double* hn,
                                          const double* mn, const double* ce, double* hout,
                                          double* mout, unsigned long long* shist,
                                          int record) {
    const Geom& g = *gp;
    LlgCell s;
    for (int c = 0; c < 3; ++c) { s.Hn[c] = hn[c]; s.Mn[c] = mn[c]; s.cE[c] = ce[c]; }
    llg_setup(s, mats[id]);
    double Hr[3] = {s.Hn[0], s.Hn[1], s.Hn[2]};
    double Mr[3] = {s.Mn[0], s.Mn[1], s.Mn[2]};
    int rc = g.max_iters + 1;
    for (int r = 1; r <= g.max_iters; ++r) {
        const double res = llg_iterate(s, g.coef_h, Hr, Mr);
        if (record) atomicMax(&shist[r], dbits(res));
        if (res <= g.tol) { rc = r; break; }
    }
    for (int c = 0; c < 3; ++c) { hout[c] = Hr[c]; mout[c] = Mr[c]; }
    return rc;
}

// Per-thread entry descriptors.  A thread owns the same (j,k) entries on
// every plane of its x-march, so indices, ghost predicates and store masks
// are computed once before the march.
enum : unsigned {
    kJ0 = 1u, kJN = 2u, kK0 = 4u, kKN = 8u,      // j==0, j==ny, k==0, k==nz
    kVX = 16u, kVKZ = 32u, kVJY = 64u,           // Hx valid (j<ny&&k<nz), k<nz, j<ny
    kLIVE = 128u, kOWN = 256u,
    kK1 = 512u, kKNm1 = 1024u,                   // k==1, k==nz-1 (z-wall inner rows)
    kXLINE = 2048u                               // Ex z-wall deferred (j<=1 || j>=ny-1)
};

struct EntryIdx {
    int e;        // shared-memory index of the entry (relative to a0)
    int ejm;      // index of (j-1) neighbour (clamped to e when j == 0)
    int ekm;      // index of (k-1) neighbour (clamped to e when k == 0)
    int f;        // flat index in the plane
    unsigned fl;  // flags above
};

__device__ __forceinline__ EntryIdx make_entry(int f, int f_end, int own_from, int a0,
                                               int Fz, uint32_t magic, int ny, int nz,
                                               bool ay) {
    EntryIdx x;
    x.f = f;
    x.e = f - a0;
    x.fl = 0;
    if (f < f_end) {
        const int j = fz_div((uint32_t)f, magic);
        const int k = f - j * Fz;
        x.fl |= kLIVE;
        if (f >= own_from) x.fl |= kOWN;
        if (j == 0) x.fl |= kJ0;
        if (j == ny) x.fl |= kJN;
        if (k == 0) x.fl |= kK0;
        if (k == nz) x.fl |= kKN;
        if (j < ny && k < nz) x.fl |= kVX;
        if (k < nz) x.fl |= kVKZ;
        if (j < ny) x.fl |= kVJY;
        if (k == 1) x.fl |= kK1;
        if (k == nz - 1) x.fl |= kKNm1;
        if (ay && (j <= 1 || j >= ny - 1)) x.fl |= kXLINE;
        x.ejm = j > 0 ? x.e - Fz : x.e;
        x.ekm = k > 0 ? x.e - 1 : x.e;
    } else {
        x.ejm = x.ekm = x.e = 0;
    }
    return x;
}

// Ghost-aware backward-difference numerators of curl H at one E entry
// (em.py:185-203): "hi - lo" per term, PMC ghosts = -edge, other walls 0.
struct ENum { double b0, b1, b2, b3, b4, b5; };

template <int NT, int V, int MH>
__global__ void __launch_bounds__(NT, 1)
k_sweep(Geom g, Bufs b, const mpb_material* __restrict__ mats,
        const uint8_t* __restrict__ gids, StepState* st, SweepCfg sc) {
    extern __shared__ __align__(128) double smem_d[];
    __shared__ uint64_t bars[kMaxSlots];
    __shared__ int s_rc[2];
    __shared__ int s_anymag;
    __shared__ double2 s_cacb[MPB_MAX_MATERIALS];
    __shared__ double s_murz[MPB_MAX_MATERIALS];
    unsigned long long* s_hist = reinterpret_cast<unsigned long long*>(smem_d);
    unsigned char* smem_b = reinterpret_cast<unsigned char*>(smem_d);
    const int ring0 = sc.ring_offset / 8;            // in doubles
    const int sd = sc.stage_bytes / 8;               // doubles per slot
    const int nslots = sc.slots;
    // producer: the last thread -- it owns the fewest E entries (T < V*NT)
    const int prod = NT - 1;

    if (st->fail) return;
    const int tid = threadIdx.x;
    const int tile = blockIdx.x % sc.tiles;
    const int chunk = blockIdx.x / sc.tiles;
    const int f0 = tile * sc.T;
    const int f1 = min(f0 + sc.T, g.FyFz);
    const int Fx = g.F[0];
    const int i0 = chunk * sc.chunk;
    const int i1 = min(i0 + sc.chunk, Fx);
    if (i0 >= i1) return;
    const int pstart = i0 > 0 ? i0 - 1 : 0;
    // last plane whose stage is needed: i1 (E only, for dEz/dx, dEy/dx of
    // plane i1-1) when it exists and x is active
    const int plast = (g.act[0] && i1 < Fx) ? i1 : i1 - 1;
    const int hlo = max(0, f0 - sc.hl);
    const int ehi = min(g.FyFz, f1 + sc.eh);
    const int a0 = hlo & ~1;                         // 16-byte aligned starts
    const int ae = (ehi + 1) & ~1;
    const int ah = (f1 + 1) & ~1;
    const int ia0 = hlo & ~15;
    const int iae = min((f1 + 16) & ~15, (int)g.PP);   // +1: z1-wall neighbour id
    const uint32_t ebytes = (uint32_t)(ae - a0) * 8u;
    const uint32_t hbytes = (uint32_t)(ah - a0) * 8u;
    const uint32_t ibytes = (uint32_t)(iae - ia0);

    for (int q = tid; q < sc.nmat; q += NT) {
        s_cacb[q] = make_double2(mats[q].ca, mats[q].cb);
        s_murz[q] = mats[q].mur_k[2];
    }
    for (int r = tid; r <= g.max_iters + 1; r += NT) s_hist[r] = 0ull;
    if (tid == prod) {
        s_rc[0] = 0x7fffffff; s_rc[1] = 0; s_anymag = 0;
        for (int q = 0; q < nslots; ++q) mbar_init(&bars[q], 1);
        mbar_fence_init();
    }
    __syncthreads();

    // slot layout (doubles): E[3][ecap] | H[3][hcap] | ids (bytes)
    auto slot = [&](int p) { return (p - pstart) % nslots; };
    auto sbase = [&](int s) { return ring0 + s * sd; };
    auto issue = [&](int p) {   // producer only
        const int s = slot(p);
        const bool full = p < i1;
        const uint32_t bytes = 3 * ebytes + (full ? 3 * hbytes + ibytes : 0u);
        mbar_expect_tx(&bars[s], bytes);
        const int64_t base = (int64_t)p * g.PP;
        double* sb = smem_d + sbase(s);
        for (int c = 0; c < 3; ++c)
            tma_load_1d(sb + c * sc.ecap, b.Ea[c] + base + a0, ebytes, &bars[s]);
        if (full) {
            for (int c = 0; c < 3; ++c)
                tma_load_1d(sb + 3 * sc.ecap + c * sc.hcap, b.Ha[c] + base + a0, hbytes,
                            &bars[s]);
            tma_load_1d(sb + 3 * sc.ecap + 3 * sc.hcap, gids + base + ia0, ibytes, &bars[s]);
        }
    };
    if (tid == prod)
        for (int p = pstart; p <= plast && p < pstart + nslots; ++p) issue(p);

    const double ry = g.act[1] ? recip_of(g.d[1]) : 1.0;
    const double rz = g.act[2] ? recip_of(g.d[2]) : 1.0;
    const double rx = g.act[0] ? recip_of(g.d[0]) : 1.0;
    const double dx = g.d[0], dy = g.d[1], dz = g.d[2];
    const double coef = g.coef_h;
    const int Fz = g.F[2];
    const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
    const bool ax = g.act[0], ay = g.act[1], az = g.act[2];
    const bool pmc_x0 = g.faces[0] == MPB_FACE_PMC, pmc_x1 = g.faces[1] == MPB_FACE_PMC;
    const bool pmc_y0 = g.faces[2] == MPB_FACE_PMC, pmc_y1 = g.faces[3] == MPB_FACE_PMC;
    const bool pmc_z0 = g.faces[4] == MPB_FACE_PMC, pmc_z1 = g.faces[5] == MPB_FACE_PMC;
    const bool guarded = sc.fastdiv != 0;
    const bool zw0 = az && g.faces[4] != MPB_FACE_PMC, zw1 = az && g.faces[5] != MPB_FACE_PMC;
    const bool z0pec = g.faces[4] == MPB_FACE_PEC, z1pec = g.faces[5] == MPB_FACE_PEC;
    const uint32_t PP = (uint32_t)g.PP;              // element offsets fit 32 bits

    EntryIdx he[MH], ee[V];
    bool warp_interior[V];
#pragma unroll
    for (int m = 0; m < MH; ++m)
        he[m] = make_entry(hlo + tid + m * NT, f1, f0, a0, Fz, sc.fz_magic, ny, nz, ay);
#pragma unroll
    for (int v = 0; v < V; ++v) {
        ee[v] = make_entry(f0 + tid + v * NT, f1, f0, a0, Fz, sc.fz_magic, ny, nz, ay);
        const bool inner = !(ee[v].fl & (kJ0 | kJN | kK0 | kKN)) || !(ee[v].fl & kLIVE);
        warp_interior[v] = __all_sync(0xffffffffu, inner);
    }
    const int iofs = a0 - ia0;   // ids index = e + iofs

    double hy_prev[V], hz_prev[V];
#pragma unroll
    for (int v = 0; v < V; ++v) { hy_prev[v] = 0.0; hz_prev[v] = 0.0; }

    for (int p = pstart; p <= i1 - 1; ++p) {
        const int s = slot(p);
        const bool xnext = ax && p < nx;                 // plane p+1 used by dx terms
        const int s1 = slot(p + 1);
        if (tid == prod) {
            mbar_wait(&bars[s], ((p - pstart) / nslots) & 1);
            if (xnext) mbar_wait(&bars[s1], ((p + 1 - pstart) / nslots) & 1);
        }
        __syncthreads();   // staged data visible; E phase of p-1 done everywhere
        if (tid == prod && p > pstart && p + nslots - 1 <= plast) {
            fence_proxy_async();
            issue(p + nslots - 1);  // into the slot plane p-1 just released
        }
        const int bE = sbase(s);
        const int bEx = bE, bEy = bE + sc.ecap, bEz = bE + 2 * sc.ecap;
        const int bEy1 = sbase(s1) + sc.ecap, bEz1 = sbase(s1) + 2 * sc.ecap;
        const int bHx = bE + 3 * sc.ecap, bHy = bHx + sc.hcap, bHz = bHy + sc.hcap;
        const unsigned char* ids = smem_b + (size_t)(bE + 3 * sc.ecap + 3 * sc.hcap) * 8;
        const bool emit = p >= i0;
        const bool cellplane = p < nx || !ax;

        // ---- H^{n+1}(p, g) on [hlo, f1), in place (em.py:117-182) -----------
#pragma unroll
        for (int m = 0; m < MH; ++m) {
            const EntryIdx& x = he[m];
            if (!(x.fl & kLIVE)) continue;
            const int e = x.e;
            const double ex = smem_d[bEx + e], ey = smem_d[bEy + e], ez = smem_d[bEz + e];
            const double a0v = smem_d[bEz + e + Fz] - ez;   // dEz/dy
            const double a1v = smem_d[bEx + e + Fz] - ex;   // dEx/dy
            const double a2v = smem_d[bEy + e + 1] - ey;    // dEy/dz
            const double a3v = smem_d[bEx + e + 1] - ex;    // dEx/dz
            const double a4v = smem_d[bEz1 + e] - ez;       // dEz/dx
            const double a5v = smem_d[bEy1 + e] - ey;       // dEy/dx
            unsigned gy = 0, gz = 0, gx = 0;
            double q0 = qdiv(a0v, dy, ry, gy), q1 = qdiv(a1v, dy, ry, gy);
            double q2 = qdiv(a2v, dz, rz, gz), q3 = qdiv(a3v, dz, rz, gz);
            double q4 = qdiv(a4v, dx, rx, gx), q5 = qdiv(a5v, dx, rx, gx);
            const bool vx = x.fl & kVX;
            const bool vy = cellplane && (x.fl & kVKZ);
            const bool vz = cellplane && (x.fl & kVJY);
            const bool bad = !guarded || (ay && gy > kGuardSpan) || (az && gz > kGuardSpan) ||
                             (ax && gx > kGuardSpan);
            if (__builtin_expect(bad, 0)) {
                q0 = xdiv(a0v, dy, ry); q1 = xdiv(a1v, dy, ry);
                q2 = xdiv(a2v, dz, rz); q3 = xdiv(a3v, dz, rz);
                q4 = xdiv(a4v, dx, rx); q5 = xdiv(a5v, dx, rx);
            }
            double cx = 0.0, cy = 0.0, cz = 0.0;            // em.py:130-138 order
            if (ay) { cx = cx + q0; cz = cz - q1; }
            if (az) { cx = cx - q2; cy = cy + q3; }
            if (ax) { cy = cy - q4; cz = cz + q5; }
            const int id = ids[e + iofs];
            const bool magnetic = cellplane && vx && (id & kMagneticIdBit);
            if (__builtin_expect(!magnetic, 1)) {
                if (vx) smem_d[bHx + e] = smem_d[bHx + e] - coef * cx;
                if (vy) smem_d[bHy + e] = smem_d[bHy + e] - coef * cy;
                if (vz) smem_d[bHz + e] = smem_d[bHz + e] - coef * cz;
            } else {
                const int64_t om = (int64_t)(p - g.mx0) * g.PP + x.f;
                const double hn[3] = {smem_d[bHx + e], smem_d[bHy + e], smem_d[bHz + e]};
                const double mn[3] = {b.Ma[0][om], b.Ma[1][om], b.Ma[2][om]};
                const double ce[3] = {cx, cy, cz};
                double ho[3], mo[3];
                const bool own = emit && (x.fl & kOWN);
                const int rc = llg_cell_local(mats, id, &g, hn, mn, ce, ho, mo, s_hist, own);
                smem_d[bHx + e] = ho[0]; smem_d[bHy + e] = ho[1]; smem_d[bHz + e] = ho[2];
                if (own) {
                    b.Mb[0][om] = mo[0]; b.Mb[1][om] = mo[1]; b.Mb[2][om] = mo[2];
                    atomicMin(&s_rc[0], rc);
                    atomicMax(&s_rc[1], rc);
                    s_anymag = 1;
                }
            }
        }
        __syncthreads();

        // ---- E^{n+1}(p, f) for the owned range (em.py:206-272) -------------
        const uint32_t base = (uint32_t)p * PP;
        const bool xedge = p == 0 || p == nx;            // plane-uniform
        const bool exEy = ax && (p <= 1 || p >= nx - 1); // Ey z-wall deferred to k_zfix
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const EntryIdx& x = ee[v];
            if (!(x.fl & kLIVE)) continue;
            const int e = x.e;
            const double hx = smem_d[bHx + e], hy = smem_d[bHy + e], hz = smem_d[bHz + e];
            if (emit) {
                const double hz_jm = smem_d[bHz + x.ejm], hx_jm = smem_d[bHx + x.ejm];
                const double hy_km = smem_d[bHy + x.ekm], hx_km = smem_d[bHx + x.ekm];
                double b0, b1, b2, b3, b4, b5;
                if (warp_interior[v] && !xedge) {
                    b0 = hz - hz_jm; b1 = hx - hx_jm; b2 = hy - hy_km;
                    b3 = hx - hx_km; b4 = hz - hz_prev[v]; b5 = hy - hy_prev[v];
                } else {
                    // backward differences with PMC ghosts (em.py:185-203)
                    const bool j0 = x.fl & kJ0, jn = x.fl & kJN, k0 = x.fl & kK0,
                               kn = x.fl & kKN;
                    const double zhi = jn ? (pmc_y1 ? -hz_jm : 0.0) : hz;
                    const double zlo = j0 ? (pmc_y0 ? -hz : 0.0) : hz_jm;
                    const double xhi_j = jn ? (pmc_y1 ? -hx_jm : 0.0) : hx;
                    const double xlo_j = j0 ? (pmc_y0 ? -hx : 0.0) : hx_jm;
                    const double yhi_k = kn ? (pmc_z1 ? -hy_km : 0.0) : hy;
                    const double ylo_k = k0 ? (pmc_z0 ? -hy : 0.0) : hy_km;
                    const double xhi_k = kn ? (pmc_z1 ? -hx_km : 0.0) : hx;
                    const double xlo_k = k0 ? (pmc_z0 ? -hx : 0.0) : hx_km;
                    const bool xl = p == 0, xh = p == nx;
                    const double zhi_i = xh ? (pmc_x1 ? -hz_prev[v] : 0.0) : hz;
                    const double zlo_i = xl ? (pmc_x0 ? -hz : 0.0) : hz_prev[v];
                    const double yhi_i = xh ? (pmc_x1 ? -hy_prev[v] : 0.0) : hy;
                    const double ylo_i = xl ? (pmc_x0 ? -hy : 0.0) : hy_prev[v];
                    b0 = zhi - zlo; b1 = xhi_j - xlo_j; b2 = yhi_k - ylo_k;
                    b3 = xhi_k - xlo_k; b4 = zhi_i - zlo_i; b5 = yhi_i - ylo_i;
                }
                unsigned gy = 0, gz = 0, gx = 0;
                double q0 = qdiv(b0, dy, ry, gy), q1 = qdiv(b1, dy, ry, gy);
                double q2 = qdiv(b2, dz, rz, gz), q3 = qdiv(b3, dz, rz, gz);
                double q4 = qdiv(b4, dx, rx, gx), q5 = qdiv(b5, dx, rx, gx);
                const bool bad = !guarded || (ay && gy > kGuardSpan) ||
                                 (az && gz > kGuardSpan) || (ax && gx > kGuardSpan);
                if (__builtin_expect(bad, 0)) {
                    q0 = xdiv(b0, dy, ry); q1 = xdiv(b1, dy, ry);
                    q2 = xdiv(b2, dz, rz); q3 = xdiv(b3, dz, rz);
                    q4 = xdiv(b4, dx, rx); q5 = xdiv(b5, dx, rx);
                }
                double cx = 0.0, cy = 0.0, cz = 0.0;   // em.py:217-231 order
                if (ay) { cx = cx + q0; cz = cz - q1; }
                if (az) { cx = cx - q2; cy = cy + q3; }
                if (ax) { cy = cy - q4; cz = cz + q5; }
                const double2 cc = s_cacb[ids[e + iofs]];
                const uint32_t o = base + (uint32_t)x.f;
                const double exa = smem_d[bEx + e], eya = smem_d[bEy + e];
                const double w0 = cc.x * (cx - cc.y * exa);
                const double w1 = cc.x * (cy - cc.y * eya);
                const double w2 = cc.x * (cz - cc.y * smem_d[bEz + e]);
                // z walls (em.py:336-359) applied in the sweep: the owner of the
                // inner entry (k=1 / k=nz-1) writes the tangential wall value;
                // lines an x/y wall touches are left to k_zfix (after x/y walls)
                const bool zx = !(x.fl & kXLINE), zy = !exEy;
                bool wx = true, wy = true;
                if ((zw0 && (x.fl & kK0)) || (zw1 && (x.fl & kKN))) { wx = !zx; wy = !zy; }
                if (wx) b.Eb[0][o] = w0;
                if (wy) b.Eb[1][o] = w1;
                b.Eb[2][o] = w2;
                if (zw0 && (x.fl & kK1)) {
                    const double kk = s_murz[ids[e - 1 + iofs]];
                    if (zx) b.Eb[0][o - 1] = z0pec ? 0.0 : exa + kk * (w0 - smem_d[bEx + e - 1]);
                    if (zy) b.Eb[1][o - 1] = z0pec ? 0.0 : eya + kk * (w1 - smem_d[bEy + e - 1]);
                }
                if (zw1 && (x.fl & kKNm1)) {
                    const double kk = s_murz[ids[e + 1 + iofs]];
                    if (zx) b.Eb[0][o + 1] = z1pec ? 0.0 : exa + kk * (w0 - smem_d[bEx + e + 1]);
                    if (zy) b.Eb[1][o + 1] = z1pec ? 0.0 : eya + kk * (w1 - smem_d[bEy + e + 1]);
                }
                if (x.fl & kVX) b.Hb[0][o] = hx;
                if (cellplane && (x.fl & kVKZ)) b.Hb[1][o] = hy;
                if (cellplane && (x.fl & kVJY)) b.Hb[2][o] = hz;
            }
            hy_prev[v] = hy;
            hz_prev[v] = hz;
        }
    }
    __syncthreads();
    if (s_anymag) {
        for (int r = 1 + tid; r <= g.max_iters; r += NT) {
            const unsigned long long v = s_hist[r];
            if (v) atomicMax(&st->hist[r], v);
        }
        if (tid == 0) {
            atomicMin(&st->rc_min, s_rc[0]);
            atomicMax(&st->rc_max, s_rc[1]);
        }
    }
}

// E entries whose curl-H stencil touches a magnetic H entry, recomputed after
// the LLG fixup settled r* (only when the fixup had to recompute).  Uses the
// sweep's z-wall write rules so the in-sweep z walls stay consistent.
__global__ void __launch_bounds__(256) k_edefer(Geom g, Bufs b,
                                                const mpb_material* __restrict__ mats,
                                                const uint8_t* __restrict__ ids,
                                                const int2* __restrict__ list, int n,
                                                const StepState* st) {
    if (st->fail || !st->fixup_ran) return;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int i = list[q].x, f = list[q].y;
    const int j = f / g.F[2];
    const int k = f - j * g.F[2];
    const int64_t o = i * g.PP + f;
    const E3 w = e_plain_at(g, b, mats, ids, i, j, k, o);
    const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
    const bool az = g.act[2];
    const bool zw0 = az && g.faces[4] != MPB_FACE_PMC, zw1 = az && g.faces[5] != MPB_FACE_PMC;
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

// z walls on the lines the sweep leaves alone: Ex on rows j in {0,1,ny-1,ny}
// and Ey on planes i in {0,1,nx-1,nx} -- the lines x/y walls read (pre-z
// values) or write (post-x/y inner values).  Runs after the x/y wall
// kernels, so the reference face order x0,x1,y0,y1,z0,z1 holds.
// list entries: (comp, i, j) packed as int3.
__global__ void __launch_bounds__(256) k_zfix(Geom g, Bufs b,
                                              const mpb_material* __restrict__ mats,
                                              const uint8_t* __restrict__ ids,
                                              const int3* __restrict__ lines, int n,
                                              const StepState* st) {
    if (st->fail) return;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int c = lines[q].x, i = lines[q].y, j = lines[q].z;
    const int64_t row = i * g.PP + (int64_t)j * g.F[2];
    const int nz = g.n[2];
    if (g.faces[4] != MPB_FACE_PMC) {     // z0: wall 0, inner 1
        const int64_t ow = row, oi = row + 1;
        if (g.faces[4] == MPB_FACE_PEC) b.Eb[c][ow] = 0.0;
        else b.Eb[c][ow] = b.Ea[c][oi] + mats[ids[ow]].mur_k[2] * (b.Eb[c][oi] - b.Ea[c][ow]);
    }
    if (g.faces[5] != MPB_FACE_PMC) {     // z1: wall nz, inner nz-1
        const int64_t ow = row + nz, oi = row + nz - 1;
        if (g.faces[5] == MPB_FACE_PEC) b.Eb[c][ow] = 0.0;
        else b.Eb[c][ow] = b.Ea[c][oi] + mats[ids[ow]].mur_k[2] * (b.Eb[c][oi] - b.Ea[c][ow]);
    }
}

}  // namespace mpb
