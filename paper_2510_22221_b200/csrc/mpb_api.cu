// mpb_api.cu -- C ABI of the B200 Maxwell-LLG stepper (include/magphon_b200.h).
//
// Owns device memory, streams, CUDA graphs and (multi-rank) the NCCL
// communicator of one run; sequences the per-step kernels.
// Build: paper_2510_22221_b200/csrc/Makefile.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/magphon_b200.h"
#include "mpb_device.cuh"
#include "mpb_kernels_split.cuh"
#include "mpb_sweep.cuh"
#include "mpb_line.cuh"
#include "mpb_esprit.cuh"

using namespace mpb;

namespace {

thread_local std::string g_err;

inline uint64_t dbits_host(double x) {
    uint64_t u;
    memcpy(&u, &x, sizeof u);
    return u;
}

int fail_msg(int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CU(call)                                                                  \
    do {                                                                          \
        cudaError_t e_ = (call);                                                  \
        if (e_ != cudaSuccess)                                                    \
            return fail_msg(MPB_ECUDA, "%s failed: %s (%s:%d)", #call,            \
                            cudaGetErrorString(e_), __FILE__, __LINE__);          \
    } while (0)

#define NC(call)                                                                  \
    do {                                                                          \
        ncclResult_t r_ = (call);                                                 \
        if (r_ != ncclSuccess)                                                    \
            return fail_msg(MPB_ECUDA, "%s failed: %s (%s:%d)", #call,            \
                            ncclGetErrorString(r_), __FILE__, __LINE__);          \
    } while (0)

constexpr int kDefaultGraphSteps = 16;
constexpr int64_t kRunChunk = 1 << 16;   // steps per host<->device staging chunk

}  // namespace

struct mpb_handle {
    int device = 0;
    Geom g{};
    int variant = 0;
    int graph_steps = kDefaultGraphSteps;
    // slab: local field planes [lo, hi); owned [g.c0, g.c1); cell planes
    // [clo, chi) of the host material / M arrays
    int nranks = 1, rank = 0;
    int lo = 0, hi = 1, clo = 0, chi = 1;
    int any_magnetic = 0;
    ncclComm_t comm = nullptr;     // LLG all-reduces (library stream)
    ncclComm_t comm_x = nullptr;   // boundary exchange (comm stream): its own
                                   // communicator, so the two streams never
                                   // share one concurrently
    int64_t nloc = 0;              // (hi - lo) * PP
    int64_t mplanes = 0;           // mx1 - mx0
    void* E[2][3] = {};            // allocations (local planes); element type
    void* H[2][3] = {};            // double, or float in the fp32 storage mode
    int f32 = 0;                   // fp32 storage of E/H (M stays fp64)
    size_t esz = sizeof(double);   // bytes per E/H element
    double* M[2][3] = {};
    uint8_t* ids = nullptr;        // allocation (local planes)
    mpb_material* mats = nullptr;
    int nmat_table = 0;
    int2* magcells = nullptr;      // local magnetic cells (owned + ghost plane)
    unsigned char* magowned = nullptr;
    int nmag = 0;                  // local cells (incl. ghost copies)
    int nmag_owned = 0;
    double* scratch = nullptr;
    // LLG-first step order (MagPre, single rank): compact per-cell H, M
    // (double-buffered like the lattice) and material ids
    bool pre = false;
    bool pre_coop = false;         // k_llg_pre + fixup as one cooperative launch
    int coop_blocks = 0;
    void* Hc[2][3] = {};
    double* Mc[2][3] = {};
    uint8_t* cid = nullptr;
    std::vector<int2> hcells;      // host copy of magcells (sorted by plane, entry)
    StepState* st = nullptr;
    ProbeDesc* probes = nullptr;
    int nprobes = 0;
    std::vector<int32_t> probe_comp;
    std::vector<int32_t> probe_loc;
    SourceDesc src{};
    int parity = 0;                // buffer set holding the current state
    int fixup_blocks = 0;
    int faces_active[6] = {};
    // staging for mpb_run
    double* d_src = nullptr;
    double* d_probe = nullptr;
    int* d_iters = nullptr;
    int64_t stage_cap = 0;
    // mpb_run, single rank: two staging sets (device + pinned host) so chunk
    // c+1 runs while chunk c's probes / r* are copied out (double buffering)
    struct RunStage {
        double* d_src = nullptr; double* d_probe = nullptr; int* d_iters = nullptr;
        double* h_src = nullptr; double* h_probe = nullptr; int* h_iters = nullptr;
        StepState* h_st = nullptr;
        cudaEvent_t done = nullptr;
        int64_t s0 = 0, cnt = 0;
        bool busy = false;
    } rs[2];
    int64_t rs_cap = 0;
    cudaStream_t stream = nullptr;
    cudaGraphExec_t graph[2] = {nullptr, nullptr};
    int64_t graph_launches[2] = {0, 0};   // kernels captured in each graph
    // slab exchange overlapped with the next step's interior sweep: the
    // exchange runs on comm_stream after ev_post, the edge chunks wait ev_exch
    bool overlap = false;
    bool exch_pending = false;
    // lines along z: the whole run in one shared-memory-resident CTA (mpb_line.cuh)
    bool line = false;
    // MPB_WALLS=face: x/y walls as one k_wall launch per face (the unfused
    // form, kept for the parity tests of k_walls_xy)
    bool wall_per_face = false;
    bool pdl = true;          // programmatic dependent launch of the step's tail (MPB_PDL=0: off)
    size_t line_smem = 0;
    LineProbe* lprobes = nullptr;
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_post = nullptr, ev_exch = nullptr;
    // M of the cell planes outside the device's magnetic planes [mx0, mx1)
    // (constant: only magnetic cells evolve); empty when it is all zero,
    // the normal case -- saves 3 doubles/cell of host memory on large grids
    std::vector<double> hostM;
    // MPB_GUARD=1: allocation base and size of every guarded dev_alloc buffer
    std::vector<std::pair<void*, size_t>> guarded;
    // timing
    int timing = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events;
    cudaEvent_t sweep_end = nullptr;   // timing: recorded right after the sweep launch
    double timed_ms = 0.0;
    int64_t timed_launches = 0;
    int64_t launches_last = 0;
    int64_t continued_steps = 0;   // suspended multi-rank steps continued on the host
    int64_t bytes = 0;
    void* fused = nullptr;         // FusedState (mpb_fused.cuh)
};

namespace {
// Fused single-sweep variant hooks (mpb_fused.cuh).
int prepare_fused(mpb_handle* h, const Geom& g);
void destroy_fused(mpb_handle* h);
template <typename T>
int launch_fused(mpb_handle* h, const Geom& g, const BufsT<T>& b, cudaStream_t s, int part,
                 int64_t& launches);
template <typename T>
int launch_deferred(mpb_handle* h, const Geom& g, const BufsT<T>& b, cudaStream_t s);
template <typename T>
int launch_zfix(mpb_handle* h, const Geom& g, const BufsT<T>& b, cudaStream_t s);
int zfix_launches(mpb_handle* h);
template <typename T>
int launch_llg_local(mpb_handle* h, const Geom& g, const BufsT<T>& b, cudaStream_t s);
template <typename T>
int launch_llg_pre(mpb_handle* h, int pa, cudaStream_t s);
template <typename T>
int launch_llg_pre_coop(mpb_handle* h, int pa, cudaStream_t s);
template <typename T>
int pack_magnetic(mpb_handle* h, int pa);
int unpack_magnetic(mpb_handle* h);

const char* fused_kernel_name();
void fused_form(mpb_handle* h, int32_t out[4]);
}  // namespace

namespace {

// View pointers: buffers are addressed with GLOBAL plane indices in every
// kernel; the allocation holds planes [lo, hi), so the view is offset.
template <typename T>
T* view(T* alloc, const mpb_handle* h) {
    return alloc ? alloc - (int64_t)h->lo * h->g.PP : nullptr;
}

// typed view of an E/H allocation (storage type T)
template <typename T>
T* fview(void* alloc, const mpb_handle* h) {
    return view(static_cast<T*>(alloc), h);
}

template <typename T>
BufsT<T> make_bufs(const mpb_handle* h, int pa) {
    BufsT<T> b{};
    const int pb = 1 - pa;
    for (int c = 0; c < 3; ++c) {
        b.Ea[c] = fview<T>(h->E[pa][c], h);
        b.Ha[c] = fview<T>(h->H[pa][c], h);
        b.Ma[c] = h->M[pa][c];      // M arrays are indexed (i - mx0) already
        b.Eb[c] = fview<T>(h->E[pb][c], h);
        b.Hb[c] = fview<T>(h->H[pb][c], h);
        b.Mb[c] = h->M[pb][c];
    }
    return b;
}

const uint8_t* ids_view(const mpb_handle* h) { return view(h->ids, h); }

template <typename T>
MagPre<T> make_magpre(const mpb_handle* h, int pa) {
    MagPre<T> m{};
    if (!h->pre) return m;
    const int pb = 1 - pa;
    for (int c = 0; c < 3; ++c) {
        m.Hn[c] = static_cast<const T*>(h->Hc[pa][c]);
        m.Mn[c] = h->Mc[pa][c];
        m.Hn1[c] = static_cast<T*>(h->Hc[pb][c]);
        m.Mn1[c] = h->Mc[pb][c];
        m.Hl[c] = fview<T>(h->H[pa][c], h);
    }
    m.cid = h->cid;
    m.on = 1;
    return m;
}

// Stream-ordered allocations on the handle's stream: neither allocating nor
// freeing a handle synchronises the device, so concurrent runs on one GPU
// (bias sweeps) do not stall each other's kernels.
//
// Debug mode MPB_GUARD=1 (the device-side bounds check; see tools/guard_tests.sh):
// each buffer gets a kGuardBytes band of 0xA5 bytes on both sides.  dev_free
// checks the bands and aborts the process if a kernel wrote outside its
// buffer; a stray read of a band yields a garbage value that breaks the
// bit-exact parity tests.
constexpr size_t kGuardBytes = 4096;
constexpr unsigned char kGuardByte = 0xA5;

bool guard_mode() {
    static const bool on = [] {
        const char* e = getenv("MPB_GUARD");
        const bool g = e && e[0] == '1';
        if (g) fprintf(stderr, "MPB_GUARD: on (%zu-byte bands)\n", kGuardBytes);
        return g;
    }();
    return on;
}

template <typename T>
int dev_alloc(mpb_handle* h, T** p, size_t count) {
    if (count == 0) { *p = nullptr; return MPB_OK; }
    const size_t bytes = count * sizeof(T);
    if (guard_mode()) {
        unsigned char* raw = nullptr;
        CU(cudaMallocAsync(reinterpret_cast<void**>(&raw), bytes + 2 * kGuardBytes, h->stream));
        CU(cudaMemsetAsync(raw, kGuardByte, bytes + 2 * kGuardBytes, h->stream));
        CU(cudaMemsetAsync(raw + kGuardBytes, 0, bytes, h->stream));
        *p = reinterpret_cast<T*>(raw + kGuardBytes);
        h->guarded.emplace_back(raw, bytes);
    } else {
        CU(cudaMallocAsync(reinterpret_cast<void**>(p), bytes, h->stream));
        CU(cudaMemsetAsync(*p, 0, bytes, h->stream));
    }
    CU(cudaStreamSynchronize(h->stream));   // ready for synchronous copies
    h->bytes += (int64_t)bytes;
    return MPB_OK;
}

// E/H field allocation of `count` elements of the handle's storage type
int field_alloc(mpb_handle* h, void** p, size_t count) {
    if (h->f32) {
        float* q = nullptr;
        const int rc = dev_alloc(h, &q, count);
        *p = q;
        return rc;
    }
    double* q = nullptr;
    const int rc = dev_alloc(h, &q, count);
    *p = q;
    return rc;
}

void dev_free(mpb_handle* h, void* p) {
    if (!p) return;
    if (guard_mode()) {
        for (auto it = h->guarded.begin(); it != h->guarded.end(); ++it) {
            unsigned char* raw = static_cast<unsigned char*>(it->first);
            if (raw + kGuardBytes != p) continue;
            std::vector<unsigned char> band(2 * kGuardBytes);
            cudaStreamSynchronize(h->stream);
            cudaMemcpy(band.data(), raw, kGuardBytes, cudaMemcpyDeviceToHost);
            cudaMemcpy(band.data() + kGuardBytes, raw + kGuardBytes + it->second, kGuardBytes,
                       cudaMemcpyDeviceToHost);
            for (size_t b = 0; b < band.size(); ++b)
                if (band[b] != kGuardByte) {
                    fprintf(stderr, "MPB_GUARD: %s guard band of a %zu-byte buffer overwritten "
                            "at byte %zd\n", b < kGuardBytes ? "low" : "high", it->second,
                            b < kGuardBytes ? (ssize_t)b - (ssize_t)kGuardBytes
                                            : (ssize_t)(it->second + b - kGuardBytes));
                    abort();
                }
            cudaFreeAsync(raw, h->stream);
            h->guarded.erase(it);
            return;
        }
    }
    cudaFreeAsync(p, h->stream);
}

int reset_state(mpb_handle* h) {
    StepState s{};
    memset(&s, 0, sizeof s);
    s.rc_negmin = -0x7fffffff;
    s.fail_step = -1;
    s.eunsafe_a = 1;      // loaded values unchecked: the first sweep keeps the guard
    s.llg_stamp = -1;
    CU(cudaMemcpyAsync(h->st, &s, sizeof s, cudaMemcpyHostToDevice, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    return MPB_OK;
}

// End-of-step boundary exchange over NCCL (multi-rank): the last owned plane
// (E, H and M when magnetic) goes up to rank+1's low ghost plane, the first
// owned plane (E) goes down to rank-1's high ghost plane.  Operates on the
// buffer set `pb` that holds the state after the step.
int exchange(mpb_handle* h, int pb, cudaStream_t s) {
    const Geom& g = h->g;
    const size_t n = (size_t)g.PP;
    const ncclDataType_t ft = h->f32 ? ncclFloat : ncclDouble;   // E/H element type
    auto plane = [&](void* alloc, int i) {
        return static_cast<char*>(alloc) + (int64_t)(i - h->lo) * g.PP * (int64_t)h->esz;
    };
    auto mplane = [&](double* alloc, int i) { return alloc + (int64_t)(i - g.mx0) * g.PP; };
    auto has_m = [&](int i) { return h->mplanes > 0 && i >= g.mx0 && i < g.mx1; };
    ncclComm_t xc = h->comm_x ? h->comm_x : h->comm;
    NC(ncclGroupStart());
    if (h->rank + 1 < h->nranks) {
        const int up = h->rank + 1;
        for (int c = 0; c < 3; ++c) {
            NC(ncclSend(plane(h->E[pb][c], g.c1 - 1), n, ft, up, xc, s));
            NC(ncclSend(plane(h->H[pb][c], g.c1 - 1), n, ft, up, xc, s));
            if (has_m(g.c1 - 1))
                NC(ncclSend(mplane(h->M[pb][c], g.c1 - 1), n, ncclDouble, up, xc, s));
            // the high ghost plane feeds only dEz/dx, dEy/dx of plane c1-1:
            // its Ex is never read, so it does not travel
            if (c > 0) NC(ncclRecv(plane(h->E[pb][c], g.c1), n, ft, up, xc, s));
        }
    }
    if (h->rank > 0) {
        const int dn = h->rank - 1;
        for (int c = 0; c < 3; ++c) {
            NC(ncclRecv(plane(h->E[pb][c], g.c0 - 1), n, ft, dn, xc, s));
            NC(ncclRecv(plane(h->H[pb][c], g.c0 - 1), n, ft, dn, xc, s));
            if (has_m(g.c0 - 1))
                NC(ncclRecv(mplane(h->M[pb][c], g.c0 - 1), n, ncclDouble, dn, xc, s));
            if (c > 0) NC(ncclSend(plane(h->E[pb][c], g.c0), n, ft, dn, xc, s));
        }
    }
    NC(ncclGroupEnd());
    return MPB_OK;
}

// ---- step phases (shared by the NCCL path and the in-process group) ----

// part 0: whole sweep + LLG; 1: interior chunks only (overlaps the slab
// exchange of the previous step); 2: edge chunks + LLG (after the exchange).
template <typename T>
int phase_sweep_t(mpb_handle* h, int pa, cudaStream_t s, int64_t& launches, int part) {
    const Geom& g = h->g;
    const BufsT<T> b = make_bufs<T>(h, pa);
    if constexpr (sizeof(T) == 8) {
        if (h->variant == 1) {
            const size_t hist_smem = (size_t)(g.max_iters + 2) * sizeof(unsigned long long);
            const dim3 plane_grid((g.FyFz + 255) / 256, g.c1 - g.c0);
            k_hsweep<<<plane_grid, 256, hist_smem, s>>>(g, b, h->mats, ids_view(h), h->st);
            ++launches;
            return MPB_OK;
        }
    }
    int rc = launch_fused(h, g, b, s, part, launches);
    if (rc) return rc;
    if (h->sweep_end && part != 1) {   // kernel timing: the sweep alone, not the LLG
        CU(cudaEventRecord(h->sweep_end, s));
        h->sweep_end = nullptr;
    }
    if (part != 1 && h->nmag > 0 && !h->pre) {
        if ((rc = launch_llg_local(h, g, b, s))) return rc;
        ++launches;
    }
    return MPB_OK;
}

int phase_sweep(mpb_handle* h, int pa, cudaStream_t s, int64_t& launches, int part = 0) {
    return h->f32 ? phase_sweep_t<float>(h, pa, s, launches, part)
                  : phase_sweep_t<double>(h, pa, s, launches, part);
}

// Sweep of a slab step: when the previous step's boundary exchange is still
// in flight on the comm stream, the interior chunks run first and only the
// edge chunks wait for it (exchange overlapped with the interior).
int phase_sweep_overlapped(mpb_handle* const* hs, int n, int pa, cudaStream_t s,
                           int64_t& launches) {
    int rc;
    mpb_handle* h0 = hs[0];
    if (!h0->exch_pending) {
        for (int r = 0; r < n; ++r)
            if ((rc = phase_sweep(hs[r], pa, s, launches, 0))) return rc;
        return MPB_OK;
    }
    for (int r = 0; r < n; ++r)
        if ((rc = phase_sweep(hs[r], pa, s, launches, 1))) return rc;
    CU(cudaStreamWaitEvent(s, h0->ev_exch, 0));
    h0->exch_pending = false;
    for (int r = 0; r < n; ++r)
        if ((rc = phase_sweep(hs[r], pa, s, launches, 2))) return rc;
    return MPB_OK;
}

template <typename T>
int phase_fixup_single_t(mpb_handle* h, int pa, cudaStream_t s, int64_t& launches) {
    if (h->nmag == 0) return MPB_OK;
    const Geom& g = h->g;
    const BufsT<T> b = make_bufs<T>(h, pa);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(h->fixup_blocks);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    // cooperative only: programmatic serialization could place the grid's
    // blocks while k_llg_local still holds SMs, and co-residency of every
    // block is what grid.sync() needs
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    MagScratch scr{h->scratch};
    CU(cudaLaunchKernelEx(&cfg, k_llg_fixup<T>, g, b, (const mpb_material*)h->mats,
                          ids_view(h), (const int2*)h->magcells, h->nmag, scr, h->st,
                          make_magpre<T>(h, pa)));
    ++launches;
    return MPB_OK;
}

int phase_fixup_single(mpb_handle* h, int pa, cudaStream_t s, int64_t& launches) {
    return h->f32 ? phase_fixup_single_t<float>(h, pa, s, launches)
                  : phase_fixup_single_t<double>(h, pa, s, launches);
}

template <typename T>
int phase_topup_t(mpb_handle* h, int pa, cudaStream_t s, int64_t& launches) {
    if (h->nmag == 0) return MPB_OK;
    const BufsT<T> b = make_bufs<T>(h, pa);
    k_llg_topup<T><<<(h->nmag + 255) / 256, 256, 0, s>>>(h->g, b, h->mats, ids_view(h),
                                                         h->magcells, h->magowned, h->nmag,
                                                         h->st);
    ++launches;
    return MPB_OK;
}

int phase_topup(mpb_handle* h, int pa, cudaStream_t s, int64_t& launches) {
    return h->f32 ? phase_topup_t<float>(h, pa, s, launches)
                  : phase_topup_t<double>(h, pa, s, launches);
}

int phase_decide(mpb_handle* h, cudaStream_t s, int64_t& launches) {
    k_llg_decide<<<1, 32, 0, s>>>(h->g, h->st);
    ++launches;
    return MPB_OK;
}

// after r* is settled: deferred E, x/y walls, z-wall fix-up, source + probes
template <typename T>
int phase_post_t(mpb_handle* h, int pa, cudaStream_t s, int64_t& launches, bool esweep) {
    const Geom& g = h->g;
    const BufsT<T> b = make_bufs<T>(h, pa);
    const uint8_t* ids = ids_view(h);
    if (h->variant != 1 && h->nmag > 0 && !h->pre) {
        int rc = launch_deferred(h, g, b, s);
        if (rc) return rc;
        ++launches;
    }
    if constexpr (sizeof(T) == 8) {
        if (h->variant == 1 && esweep) {
            const dim3 plane_grid((g.FyFz + 255) / 256, g.c1 - g.c0);
            k_esweep<<<plane_grid, 256, 0, s>>>(g, b, h->mats, ids, h->st);
            ++launches;
        }
    }
    // x and y walls: one launch for the four faces (k_walls_xy); z walls
    // are in the sweep (+ k_zfix) or, unfused, one k_wall launch per face
    {
        int act = 0;
        int64_t cnt = 0;
        for (int face = 0; face < 4; ++face)
            if (h->faces_active[face]) {
                act |= 1 << face;
                cnt = std::max<int64_t>(cnt, face < 2 ? (int64_t)g.F[1] * g.F[2]
                                                      : (int64_t)(g.c1 - g.c0) * g.F[2]);
            }
        if (act && !h->wall_per_face) {
            CU(launch_pdl(h->pdl, k_walls_xy<T>, dim3((unsigned)((cnt + 255) / 256), 4), dim3(256),
                          s, g, b, (const mpb_material*)h->mats, ids, h->st,
                          act));
            ++launches;
        }
    }
    const int nface = g.zin ? 4 : 6;   // fused: z walls are in the sweep
    for (int face = h->wall_per_face ? 0 : 4; face < nface; ++face) {
        if (!h->faces_active[face]) continue;
        const int axis = face >> 1;
        const int u = axis == 0 ? 1 : 0, w = axis == 2 ? 1 : 2;
        const int64_t nu = u == 0 ? g.c1 - g.c0 : g.F[u];
        const int64_t cnt = nu * g.F[w];
        k_wall<T><<<(unsigned)((cnt + 255) / 256), 256, 0, s>>>(g, b, h->mats, ids, h->st,
                                                                face);
        ++launches;
    }
    if (g.zin) {
        int rc = launch_zfix(h, g, b, s);
        if (rc) return rc;
        launches += zfix_launches(h);
    }
    CU(launch_pdl(h->pdl, k_finish<T>, dim3(1), dim3(256), s, g, b, h->src,
                  (const ProbeDesc*)h->probes, h->nprobes, 1 - pa,
                  h->any_magnetic ? 1 : 0, h->st));
    ++launches;
    return MPB_OK;
}

int phase_post(mpb_handle* h, int pa, cudaStream_t s, int64_t& launches,
               bool esweep = true) {
    return h->f32 ? phase_post_t<float>(h, pa, s, launches, esweep)
                  : phase_post_t<double>(h, pa, s, launches, esweep);
}

// End of a slab step: the boundary planes of the new state (set 1 - pa)
// to the neighbours, on the comm stream overlapping the next interior sweep.
int end_step_exchange(mpb_handle* h, int pa) {
    int rc;
    cudaStream_t s = h->stream;
    if (h->overlap) {
        CU(cudaEventRecord(h->ev_post, s));
        CU(cudaStreamWaitEvent(h->comm_stream, h->ev_post, 0));
        if ((rc = exchange(h, 1 - pa, h->comm_stream))) return rc;
        CU(cudaEventRecord(h->ev_exch, h->comm_stream));
        h->exch_pending = true;
    } else if ((rc = exchange(h, 1 - pa, s))) {
        return rc;
    }
    return MPB_OK;
}

// Enqueue one coupled step reading buffer set `pa` (single rank or NCCL).
int enqueue_step(mpb_handle* h, int pa, bool timed) {
    const Geom& g = h->g;
    cudaStream_t s = h->stream;
    int64_t launches = 0;
    int rc;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timed) {
        CU(cudaEventCreate(&e0));
        CU(cudaEventCreate(&e1));
        CU(cudaEventRecord(e0, s));
        h->sweep_end = e1;
    }
    if (h->pre) {   // LLG-first: local LLG + r* settlement, then the sweep
        if (h->pre_coop) {
            if ((rc = h->f32 ? launch_llg_pre_coop<float>(h, pa, s)
                             : launch_llg_pre_coop<double>(h, pa, s)))
                return rc;
            ++launches;
        } else {
            if ((rc = h->f32 ? launch_llg_pre<float>(h, pa, s) : launch_llg_pre<double>(h, pa, s)))
                return rc;
            ++launches;
            if ((rc = phase_fixup_single(h, pa, s, launches))) return rc;
        }
        if (timed) CU(cudaEventRecord(e0, s));
    }
    if ((rc = phase_sweep_overlapped(&h, 1, pa, s, launches))) return rc;
    if (timed) {
        if (h->sweep_end) CU(cudaEventRecord(e1, s));   // split variant: after k_hsweep
        h->sweep_end = nullptr;
        h->events.emplace_back(e0, e1);
    }
    if (h->nranks == 1) {
        if (!h->pre && (rc = phase_fixup_single(h, pa, s, launches))) return rc;
    } else if (h->any_magnetic) {
        // global r*: all-reduce the residual history and local-stop range
        NC(ncclGroupStart());
        NC(ncclAllReduce(&h->st->hist[1], &h->st->hist[1], (size_t)g.max_iters, ncclUint64,
                         ncclMax, h->comm, s));
        NC(ncclAllReduce(&h->st->rc_max, &h->st->rc_max, 2, ncclInt32, ncclMax, h->comm, s));
        NC(ncclGroupEnd());
        if ((rc = phase_topup(h, pa, s, launches))) return rc;
        NC(ncclAllReduce(&h->st->hist2[1], &h->st->hist2[1], (size_t)g.max_iters, ncclUint64,
                         ncclMax, h->comm, s));
        if ((rc = phase_decide(h, s, launches))) return rc;
    }
    if (timed && h->variant == 1) {   // split variant: time the E sweep too
        cudaEvent_t ea = nullptr, eb = nullptr;
        CU(cudaEventCreate(&ea));
        CU(cudaEventCreate(&eb));
        CU(cudaEventRecord(ea, s));
        const Bufs b = make_bufs<double>(h, pa);
        const dim3 plane_grid((g.FyFz + 255) / 256, g.c1 - g.c0);
        k_esweep<<<plane_grid, 256, 0, s>>>(g, b, h->mats, ids_view(h), h->st);
        CU(cudaEventRecord(eb, s));
        h->events.emplace_back(ea, eb);
        ++launches;
        if ((rc = phase_post(h, pa, s, launches, false))) return rc;
    } else {
        if ((rc = phase_post(h, pa, s, launches))) return rc;
    }
    if (h->nranks > 1 && (rc = end_step_exchange(h, pa))) return rc;
    h->launches_last += launches;
    CU(cudaGetLastError());
    return MPB_OK;
}

// In-process group: the boundary exchange of exchange() as device copies.
int exchange_group(mpb_handle* const* hs, int n, int pb, cudaStream_t s) {
    for (int r = 0; r + 1 < n; ++r) {
        mpb_handle* a = hs[r];
        mpb_handle* b = hs[r + 1];
        const Geom& ga = a->g;
        const Geom& gb = b->g;
        const size_t bytes = (size_t)ga.PP * a->esz;           // an E/H plane
        const size_t mbytes = (size_t)ga.PP * sizeof(double);  // an M plane
        auto plane = [](mpb_handle* h, void* alloc, int i) {
            return static_cast<char*>(alloc) + (int64_t)(i - h->lo) * h->g.PP * (int64_t)h->esz;
        };
        const int up_src = ga.c1 - 1;   // a's last owned plane -> b's low ghost
        const int dn_src = gb.c0;       // b's first owned plane -> a's high ghost
        const bool m_up = a->mplanes > 0 && up_src >= ga.mx0 && up_src < ga.mx1;
        for (int c = 0; c < 3; ++c) {
            CU(cudaMemcpyAsync(plane(b, b->E[pb][c], up_src), plane(a, a->E[pb][c], up_src),
                               bytes, cudaMemcpyDeviceToDevice, s));
            CU(cudaMemcpyAsync(plane(b, b->H[pb][c], up_src), plane(a, a->H[pb][c], up_src),
                               bytes, cudaMemcpyDeviceToDevice, s));
            if (m_up)
                CU(cudaMemcpyAsync(b->M[pb][c] + (int64_t)(up_src - gb.mx0) * gb.PP,
                                   a->M[pb][c] + (int64_t)(up_src - ga.mx0) * ga.PP, mbytes,
                                   cudaMemcpyDeviceToDevice, s));
            if (c > 0)   // Ex of the high ghost plane is never read (see exchange)
                CU(cudaMemcpyAsync(plane(a, a->E[pb][c], dn_src), plane(b, b->E[pb][c], dn_src),
                                   bytes, cudaMemcpyDeviceToDevice, s));
        }
    }
    return MPB_OK;
}

int group_step(mpb_handle* const* hs, int n, int pa, cudaStream_t s) {
    int rc;
    int64_t launches = 0;
    if ((rc = phase_sweep_overlapped(hs, n, pa, s, launches))) return rc;
    if (hs[0]->any_magnetic) {
        StatePtrs sp{};
        sp.n = n;
        for (int r = 0; r < n; ++r) sp.s[r] = hs[r]->st;
        k_group_reduce<<<1, 256, 0, s>>>(sp, hs[0]->g.max_iters, 0);
        for (int r = 0; r < n; ++r)
            if ((rc = phase_topup(hs[r], pa, s, launches))) return rc;
        k_group_reduce<<<1, 256, 0, s>>>(sp, hs[0]->g.max_iters, 1);
        for (int r = 0; r < n; ++r)
            if ((rc = phase_decide(hs[r], s, launches))) return rc;
    }
    for (int r = 0; r < n; ++r)
        if ((rc = phase_post(hs[r], pa, s, launches))) return rc;
    if (hs[0]->overlap) {   // device copies on the comm stream, like exchange()
        mpb_handle* h0 = hs[0];
        CU(cudaEventRecord(h0->ev_post, s));
        CU(cudaStreamWaitEvent(h0->comm_stream, h0->ev_post, 0));
        if ((rc = exchange_group(hs, n, 1 - pa, h0->comm_stream))) return rc;
        CU(cudaEventRecord(h0->ev_exch, h0->comm_stream));
        h0->exch_pending = true;
    } else if ((rc = exchange_group(hs, n, 1 - pa, s))) {
        return rc;
    }
    CU(cudaGetLastError());
    return MPB_OK;
}

// Make `s` wait for a boundary exchange still in flight (end of a run).
int drain_exchange(mpb_handle* h, cudaStream_t s) {
    if (h->exch_pending) {
        CU(cudaStreamWaitEvent(s, h->ev_exch, 0));
        h->exch_pending = false;
    }
    return MPB_OK;
}

// Host replay of llg_decide (mpb_device.cuh) on an all-reduced history.
int host_decide(const unsigned long long* hist, int upto, int max_iters, double tol,
                double* fres, int* fit, int* fkind) {
    double prev = INFINITY;
    int growth = 0;
    for (int it = 1; it <= upto; ++it) {
        double res;
        memcpy(&res, &hist[it], sizeof res);
        if (res <= tol) return it;
        growth = (res > prev) ? growth + 1 : 0;
        if (growth >= 3) { *fres = res; *fit = it; *fkind = 1; return 0; }
        prev = res;
        if (it == max_iters) { *fres = prev; *fit = max_iters; *fkind = 2; return 0; }
    }
    return -1;
}

// Continue a suspended multi-rank step (k_llg_decide, kMpbSuspend) exactly
// as the reference's lockstep loop does (llg.py:131-148): every rank
// recomputes its cells from the step-n state one iterate at a time, the
// owned residual maxima are all-reduced after each iterate and the stop /
// failure rule is replayed on the host until it decides.  Then the step is
// finished as usual (deferred E, walls, source, probes, exchange).  hs are
// the n local handles (one for NCCL, all ranks for the in-process group),
// positioned at the suspended step's parity; the sweep's E^{n+1} of that
// step is intact (only k_llg_decide's successors were skipped).
int recover_suspended(mpb_handle* const* hs, int n, bool group, cudaStream_t s) {
    mpb_handle* h0 = hs[0];
    const Geom& g = h0->g;
    const int pa = h0->parity;
    int rc;
    int64_t launches = 0;
    if ((rc = drain_exchange(h0, s))) return rc;
    for (int q = 0; q < n; ++q) {
        k_suspend_clear<<<1, 256, 0, s>>>(hs[q]->st, g.max_iters);
        if (!hs[q]->nmag) continue;
        const dim3 grid((hs[q]->nmag + 255) / 256);
        const MagScratch scr{hs[q]->scratch};
        if (hs[q]->f32)
            k_llg_cont_init<float><<<grid, 256, 0, s>>>(hs[q]->g, make_bufs<float>(hs[q], pa),
                                                        hs[q]->magcells, hs[q]->nmag, scr);
        else
            k_llg_cont_init<double><<<grid, 256, 0, s>>>(hs[q]->g, make_bufs<double>(hs[q], pa),
                                                         hs[q]->magcells, hs[q]->nmag, scr);
    }
    CU(cudaGetLastError());
    std::vector<unsigned long long> hist((size_t)g.max_iters + 2, 0ull);
    int rstar = -1, fit = 0, fkind = 0;
    double fres = 0.0;
    StatePtrs sp{};
    sp.n = n;
    for (int q = 0; q < n; ++q) sp.s[q] = hs[q]->st;
    for (int r = 1; r <= g.max_iters && rstar < 0; ++r) {
        for (int q = 0; q < n; ++q)
            if (hs[q]->nmag)
                k_llg_cont_iter<<<(hs[q]->nmag + 255) / 256, 256, 0, s>>>(
                    hs[q]->g, hs[q]->mats, ids_view(hs[q]), hs[q]->magcells,
                    hs[q]->magowned, hs[q]->nmag, MagScratch{hs[q]->scratch}, hs[q]->st, r);
        CU(cudaGetLastError());
        if (group) {
            k_group_reduce<<<1, 256, 0, s>>>(sp, g.max_iters, 1);
        } else {
            NC(ncclAllReduce(&h0->st->hist2[r], &h0->st->hist2[r], 1, ncclUint64, ncclMax,
                             h0->comm, s));
        }
        CU(cudaMemcpyAsync(hist.data(), h0->st->hist2, sizeof(unsigned long long) * (r + 1),
                           cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        const int d = host_decide(hist.data(), r, g.max_iters, g.tol, &fres, &fit, &fkind);
        if (d > 0) rstar = d;
        else if (d == 0) rstar = 0;
    }
    if (rstar <= 0) {   // the reference raises StepFailure at this step
        for (int q = 0; q < n; ++q)
            k_set_failure<<<1, 1, 0, s>>>(hs[q]->st, fres, fit, fkind);
        CU(cudaGetLastError());
        return MPB_OK;   // the caller reads the failure record
    }
    for (int q = 0; q < n; ++q) {
        const dim3 grid((std::max(hs[q]->nmag, 1) + 255) / 256);
        const MagScratch scr{hs[q]->scratch};
        if (hs[q]->f32)
            k_llg_cont_write<float><<<grid, 256, 0, s>>>(
                hs[q]->g, make_bufs<float>(hs[q], pa), hs[q]->magcells, hs[q]->magowned,
                hs[q]->nmag, scr, hs[q]->st, rstar);
        else
            k_llg_cont_write<double><<<grid, 256, 0, s>>>(
                hs[q]->g, make_bufs<double>(hs[q], pa), hs[q]->magcells, hs[q]->magowned,
                hs[q]->nmag, scr, hs[q]->st, rstar);
    }
    CU(cudaGetLastError());
    for (int q = 0; q < n; ++q)
        if ((rc = phase_post(hs[q], pa, s, launches))) return rc;
    if (group) {
        if ((rc = exchange_group(hs, n, 1 - pa, s))) return rc;
    } else if ((rc = end_step_exchange(h0, pa))) {
        return rc;
    }
    for (int q = 0; q < n; ++q) ++hs[q]->continued_steps;
    CU(cudaGetLastError());
    return MPB_OK;
}

int build_graph(mpb_handle* h, int start_parity) {
    cudaGraph_t graph;
    CU(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    int rc = MPB_OK;
    const int64_t saved = h->launches_last;
    for (int s = 0; s < h->graph_steps && rc == MPB_OK; ++s)
        rc = enqueue_step(h, (start_parity + s) & 1, false);
    h->graph_launches[start_parity] = h->launches_last - saved;
    h->launches_last = saved;
    cudaError_t e = cudaStreamEndCapture(h->stream, &graph);
    if (rc) return rc;
    if (e != cudaSuccess)
        return fail_msg(MPB_ECUDA, "graph capture failed: %s", cudaGetErrorString(e));
    CU(cudaGraphInstantiate(&h->graph[start_parity], graph, 0));
    CU(cudaGraphDestroy(graph));
    return MPB_OK;
}

// Enqueue nsteps steps; buffers already pointed to by the device state.
int launch_line(mpb_handle* h, int64_t nsteps);

int enqueue_steps(mpb_handle* h, int64_t nsteps) {
    if (h->line) return launch_line(h, nsteps);
    int64_t s = 0;
    const bool use_graph = !h->timing && h->graph_steps > 1;
    while (s < nsteps) {
        if (use_graph && nsteps - s >= h->graph_steps) {
            if (!h->graph[h->parity]) {
                int rc = build_graph(h, h->parity);
                if (rc) return rc;
            }
            CU(cudaGraphLaunch(h->graph[h->parity], h->stream));
            h->launches_last += h->graph_launches[h->parity];
            if (h->graph_steps & 1) h->parity ^= 1;
            s += h->graph_steps;
        } else {
            int rc = enqueue_step(h, h->parity, h->timing != 0);
            if (rc) return rc;
            h->parity ^= 1;
            ++s;
        }
    }
    return drain_exchange(h, h->stream);
}

// Point the device bookkeeping at a run's staging buffers, stream-ordered
// (a one-thread kernel: no host-side lifetime to wait for).
int set_run_buffers(mpb_handle* h, int64_t n0, const double* src, double* probe,
                    int* iters) {
    k_set_run<<<1, 1, 0, h->stream>>>(h->st, (long long)n0, src, probe, iters);
    CU(cudaGetLastError());
    return MPB_OK;
}

void free_run_stages(mpb_handle* h) {
    for (auto& r : h->rs) {
        dev_free(h, r.d_src); dev_free(h, r.d_probe); dev_free(h, r.d_iters);
        if (r.h_src) cudaFreeHost(r.h_src);
        if (r.h_probe) cudaFreeHost(r.h_probe);
        if (r.h_iters) cudaFreeHost(r.h_iters);
        if (r.h_st) cudaFreeHost(r.h_st);
        if (r.done) cudaEventDestroy(r.done);
        r = mpb_handle::RunStage{};
    }
    h->rs_cap = 0;
}

int alloc_run_stages(mpb_handle* h, int64_t cap) {
    if (cap <= h->rs_cap) return MPB_OK;
    CU(cudaStreamSynchronize(h->stream));
    free_run_stages(h);
    const int np = std::max(1, h->nprobes);
    for (auto& r : h->rs) {
        int rc = dev_alloc(h, &r.d_src, (size_t)cap);
        if (!rc) rc = dev_alloc(h, &r.d_probe, (size_t)(cap * np));
        if (!rc) rc = dev_alloc(h, &r.d_iters, (size_t)cap);
        if (rc) return rc;
        CU(cudaMallocHost(&r.h_src, sizeof(double) * cap));
        CU(cudaMallocHost(&r.h_probe, sizeof(double) * cap * np));
        CU(cudaMallocHost(&r.h_iters, sizeof(int) * cap));
        CU(cudaMallocHost(&r.h_st, sizeof(StepState)));
        CU(cudaEventCreateWithFlags(&r.done, cudaEventDisableTiming));
    }
    h->rs_cap = cap;
    return MPB_OK;
}

int read_failure(mpb_handle* h, mpb_failure* fail) {
    StepState s;
    CU(cudaStreamSynchronize(h->stream));
    CU(cudaMemcpy(&s, h->st, sizeof s, cudaMemcpyDeviceToHost));
    if (fail) {
        fail->step = s.fail ? s.fail_step : -1;
        fail->residual = s.fail_res;
        fail->iterations = s.fail_it;
        fail->kind = s.fail_kind;
    }
    return s.fail ? MPB_ESTEP : MPB_OK;
}

int upload_probes(mpb_handle* h) {
    const Geom& g = h->g;
    std::vector<ProbeDesc> pd((size_t)std::max(1, h->nprobes));
    const int ny = g.n[1], nz = g.n[2];
    const int ncl = h->chi - h->clo;
    for (int p = 0; p < h->nprobes; ++p) {
        const int comp = h->probe_comp[p];
        const int* L = &h->probe_loc[3 * p];
        const int64_t f = (int64_t)L[1] * g.F[2] + L[2];
        ProbeDesc d{};
        const bool owned = L[0] >= g.c0 && L[0] < g.c1;   // other ranks report 0
        auto fptr = [&](void* a) -> const void* {         // typed view of an E/H buffer
            return h->f32 ? (const void*)fview<float>(a, h) : (const void*)fview<double>(a, h);
        };
        if (!owned) {
            d.ptr0 = d.ptr1 = nullptr;
            d.constant = 0.0;
        } else if (comp < MPB_COMP_HX) {
            d.ptr0 = fptr(h->E[0][comp]); d.ptr1 = fptr(h->E[1][comp]);
            d.off = L[0] * g.PP + f;
            d.f32 = h->f32;
        } else if (comp < MPB_COMP_MX) {
            d.ptr0 = fptr(h->H[0][comp - 3]); d.ptr1 = fptr(h->H[1][comp - 3]);
            d.off = L[0] * g.PP + f;
            d.f32 = h->f32;
        } else if (L[0] >= g.mx0 && L[0] < g.mx1) {
            d.ptr0 = h->M[0][comp - 6]; d.ptr1 = h->M[1][comp - 6];
            d.off = (int64_t)(L[0] - g.mx0) * g.PP + f;
            if (h->pre) {   // a magnetic cell's M lives in the compact copy
                const int2 key = make_int2(L[0], (int)f);
                auto it = std::lower_bound(h->hcells.begin(), h->hcells.end(), key,
                                           [](const int2& a, const int2& b) {
                                               return a.x != b.x ? a.x < b.x : a.y < b.y;
                                           });
                if (it != h->hcells.end() && it->x == key.x && it->y == key.y) {
                    d.ptr0 = h->Mc[0][comp - 6]; d.ptr1 = h->Mc[1][comp - 6];
                    d.off = it - h->hcells.begin();
                }
            }
        } else {
            d.ptr0 = d.ptr1 = nullptr;
            d.constant = h->hostM.empty() ? 0.0 :
                h->hostM[(((size_t)(comp - 6) * ncl + (L[0] - h->clo)) * ny + L[1]) * nz + L[2]];
        }
        pd[(size_t)p] = d;
    }
    CU(cudaMemcpy(h->probes, pd.data(), sizeof(ProbeDesc) * pd.size(),
                  cudaMemcpyHostToDevice));
    if (h->line) {   // the same probes, addressed in the line kernel's shared state
        std::vector<LineProbe> lp((size_t)std::max(1, h->nprobes));
        for (int p = 0; p < h->nprobes; ++p) {
            const int comp = h->probe_comp[p];
            const int k = h->probe_loc[3 * p + 2];
            LineProbe q{};
            if (comp < MPB_COMP_MX || h->mplanes) { q.src = comp; q.idx = k; }
            else { q.src = -1; q.constant = pd[(size_t)p].constant; }
            lp[(size_t)p] = q;
        }
        CU(cudaMemcpy(h->lprobes, lp.data(), sizeof(LineProbe) * lp.size(),
                      cudaMemcpyHostToDevice));
    }
    return MPB_OK;
}

// The whole of nsteps in one launch of the line kernel (mpb_line.cuh).
int launch_line(mpb_handle* h, int64_t nsteps) {
    if (nsteps <= 0) return MPB_OK;
    const int pa = h->parity, pb = (int)((h->parity + nsteps) & 1);
    LineArgs a{};
    for (int c = 0; c < 3; ++c) {
        // (the line kernel runs only in fp64 storage)
        a.E[c] = static_cast<double*>(h->E[pa][c]); a.H[c] = static_cast<double*>(h->H[pa][c]);
        a.M[c] = h->mplanes ? h->M[pa][c] : nullptr;
        a.Eo[c] = static_cast<double*>(h->E[pb][c]); a.Ho[c] = static_cast<double*>(h->H[pb][c]);
        a.Mo[c] = h->mplanes ? h->M[pb][c] : nullptr;
        a.src_pol[c] = h->src.pol[c];
    }
    a.ids = h->ids;
    a.mats = h->mats;
    a.magcells = h->magcells;
    a.nmag = h->nmag;
    a.nmat = h->nmat_table;
    a.probes = h->lprobes;
    a.nprobes = h->nprobes;
    a.src_off = (int)h->src.off;
    a.any_magnetic = h->any_magnetic;
    a.nsteps = (int)nsteps;
    k_line<<<1, kLineThreads, h->line_smem, h->stream>>>(h->g, a, h->st);
    CU(cudaGetLastError());
    h->parity = pb;
    h->launches_last += 1;
    return MPB_OK;
}

}  // namespace

namespace {
// The body of mpb_create after the handle exists (errors return; the caller
// destroys the partially built handle).
int create_body(const mpb_setup* su, mpb_handle* h, int nranks, int x_lo, int x_hi) {
    const int nx = su->n[0], ny = su->n[1], nz = su->n[2];
    h->device = su->device;
    h->variant = su->kernel_variant;
    h->f32 = su->storage == MPB_STORAGE_F32;
    h->esz = h->f32 ? sizeof(float) : sizeof(double);
    h->graph_steps = su->graph_steps > 0 ? su->graph_steps : kDefaultGraphSteps;
    if (nranks > 1) h->graph_steps = 1;   // NCCL steps are enqueued eagerly
    h->nranks = nranks;
    h->rank = nranks == 1 ? 0 : su->rank;
    CU(cudaSetDevice(h->device));
    CU(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    if (nranks > 1) {
        CU(cudaStreamCreateWithFlags(&h->comm_stream, cudaStreamNonBlocking));
        CU(cudaEventCreateWithFlags(&h->ev_post, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&h->ev_exch, cudaEventDisableTiming));
        const char* e = getenv("MPB_OVERLAP");
        h->overlap = su->kernel_variant != 1 && !(e && atoi(e) == 0);
    }

    Geom& g = h->g;
    int64_t F[3];
    for (int a = 0; a < 3; ++a) {
        g.n[a] = su->n[a];
        g.F[a] = su->n[a] > 1 ? su->n[a] + 1 : 1;
        g.act[a] = su->n[a] > 1;
        g.d[a] = su->d[a];
        F[a] = g.F[a];
    }
    g.FyFz = (int)(F[1] * F[2]);
    g.PP = (F[1] * F[2] + 31) / 32 * 32;
    if ((uint64_t)F[0] * (uint64_t)g.PP >= (1ull << 32)) { return fail_msg(MPB_EINVAL, "grid too large for 32-bit element offsets");
    }
    g.coef_h = su->coef_h;
    g.max_iters = su->llg_max_iters;
    g.tol = su->llg_tol;
    g.zin = su->kernel_variant == 1 ? 0 : 1;
    if (const char* e = getenv("MPB_WALLS"))        // "face": one x/y wall launch per face
        h->wall_per_face = !strcmp(e, "face");
    if (const char* e = getenv("MPB_PDL")) h->pdl = strcmp(e, "0") != 0;
    if (const char* e = getenv("MPB_ZWALL"))        // "kernel": separate z-wall launches
        if (!strcmp(e, "kernel")) g.zin = 0;
    g.c0 = x_lo;
    g.c1 = x_hi == nx ? (int)F[0] : x_hi;
    h->lo = std::max(0, g.c0 - 1);
    h->hi = std::min((int)F[0], g.c1 + 1);
    h->clo = std::max(0, x_lo - 1);
    h->chi = std::min(nx, x_hi + 1);
    for (int f = 0; f < 6; ++f) {
        g.faces[f] = su->faces[f];
        bool act = g.act[f >> 1] && su->faces[f] != MPB_FACE_PMC;
        if (f == 0 && g.c0 != 0) act = false;            // x walls on the end ranks
        if (f == 1 && g.c1 != (int)F[0]) act = false;
        h->faces_active[f] = act;
    }
    h->nloc = (int64_t)(h->hi - h->lo) * g.PP;
    h->nmat_table = MPB_MAX_MATERIALS;

    // material table renumbered so that magnetic materials carry bit 7 of
    // the id (the sweep tests magnetism without a table lookup)
    std::vector<int> remap((size_t)su->n_materials);
    std::vector<mpb_material> table(MPB_MAX_MATERIALS);
    memset(table.data(), 0, sizeof(mpb_material) * table.size());
    {
        int nm = 0, mm = 0;
        for (int q = 0; q < su->n_materials; ++q) {
            const int id = su->materials[q].magnetic ? 128 + mm++ : nm++;
            if (nm > 128 || mm > 128) { return fail_msg(MPB_EINVAL, "at most 128 magnetic and 128 non-magnetic materials");
            }
            remap[(size_t)q] = id;
            table[(size_t)id] = su->materials[q];
        }
    }
    // material ids on the local field planes, edge-padded (em.py:248-252);
    // magnetic cells of planes [lo, c1) (owned + the low ghost plane)
    std::vector<uint8_t> ids((size_t)h->nloc, 0);
    std::vector<int2> cells;
    std::vector<unsigned char> owned;
    int mx0 = nx, mx1 = 0;
    for (int i = h->lo; i < h->hi; ++i)
        for (int j = 0; j < F[1]; ++j)
            for (int k = 0; k < F[2]; ++k) {
                const int ci = std::min(i, nx - 1), cj = std::min(j, ny - 1),
                          ck = std::min(k, nz - 1);
                const uint8_t id0 =
                    su->cell_material[((size_t)(ci - h->clo) * ny + cj) * nz + ck];
                if (id0 >= su->n_materials) { return fail_msg(MPB_EINVAL, "material id %d out of range", id0);
                }
                const uint8_t id = (uint8_t)remap[id0];
                const int64_t f = (int64_t)j * F[2] + k;
                ids[(size_t)((i - h->lo) * g.PP + f)] = id;
                if (i < nx && i < g.c1 && j < ny && k < nz && table[id].magnetic) {
                    cells.push_back(make_int2(i, (int)f));
                    owned.push_back(i >= g.c0 ? 1 : 0);
                    mx0 = std::min(mx0, i);
                    mx1 = std::max(mx1, i + 1);
                }
            }
    h->nmag = (int)cells.size();
    for (unsigned char o : owned) h->nmag_owned += o;
    h->any_magnetic = nranks == 1 ? (h->nmag > 0) : (su->any_magnetic != 0);
    if (h->nmag == 0) { mx0 = 0; mx1 = 0; }
    g.mx0 = mx0;
    g.mx1 = mx1;
    h->mplanes = mx1 - mx0;

    int rc = MPB_OK;
    auto chk = [&](int r) { if (r && !rc) rc = r; };
    for (int p = 0; p < 2; ++p)
        for (int c = 0; c < 3; ++c) {
            chk(field_alloc(h, &h->E[p][c], (size_t)h->nloc));
            chk(field_alloc(h, &h->H[p][c], (size_t)h->nloc));
            chk(dev_alloc(h, &h->M[p][c], (size_t)(h->mplanes * g.PP)));
        }
    chk(dev_alloc(h, &h->ids, (size_t)h->nloc));
    chk(dev_alloc(h, &h->mats, (size_t)MPB_MAX_MATERIALS));
    chk(dev_alloc(h, &h->magcells, (size_t)h->nmag));
    chk(dev_alloc(h, &h->magowned, (size_t)h->nmag));
    chk(dev_alloc(h, &h->scratch, (size_t)h->nmag * 12));
    chk(dev_alloc(h, &h->st, 1));
    if (rc) return rc;
    CU(cudaMemcpy(h->ids, ids.data(), ids.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->mats, table.data(), sizeof(mpb_material) * table.size(),
                  cudaMemcpyHostToDevice));
    if (h->nmag) {
        CU(cudaMemcpy(h->magcells, cells.data(), sizeof(int2) * cells.size(),
                      cudaMemcpyHostToDevice));
        CU(cudaMemcpy(h->magowned, owned.data(), owned.size(), cudaMemcpyHostToDevice));
    }

    // cooperative fixup grid (single rank): co-resident blocks only
    if (h->nmag && nranks == 1) {
        int per_sm = 0, sms = 0;
        if (h->f32) {
            CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_llg_fixup<float>, 256, 0));
        } else {
            CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_llg_fixup<double>, 256,
                                                             0));
        }
        CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
        const int need = (h->nmag + 255) / 256;
        h->fixup_blocks = std::max(1, std::min(need, per_sm * sms));
    }
    {   // reciprocals of the spacings for the exact-division fast path
        double* dr = nullptr;
        CU(cudaMallocAsync(&dr, 3 * sizeof(double), h->stream));
        k_recips<<<1, 1, 0, h->stream>>>(g.d[0], g.d[1], g.d[2], dr);
        CU(cudaGetLastError());
        CU(cudaMemcpyAsync(g.rd, dr, 3 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        CU(cudaFreeAsync(dr, h->stream));
        CU(cudaStreamSynchronize(h->stream));
    }
    {   // lines along z that fit in one CTA's shared memory run in k_line
        const char* e = getenv("MPB_LINE");
        const bool want = !(e && atoi(e) == 0);
        const size_t need = ((size_t)9 * g.F[2] + 3 * (size_t)h->nmat_table) * sizeof(double) +
                            (size_t)g.F[2] + 16;
        int optin = 0;
        CU(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
        if (want && !h->f32 && h->nranks == 1 && h->variant == 0 && g.n[0] == 1 && g.n[1] == 1 &&
            g.act[2] && g.n[2] >= 2 && h->nmag <= kLineThreads &&
            need + 1024 <= (size_t)optin) {
            h->line = true;
            h->line_smem = need;
            CU(cudaFuncSetAttribute(k_line, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)need));
        }
    }

    // LLG-first step order for single-rank runs of the fused sweep
    // (MPB_LLG_PRE=0: the LLG after the sweep + deferred E, as multi-rank runs do)
    {
        const char* e = getenv("MPB_LLG_PRE");
        h->pre = !(e && atoi(e) == 0) && nranks == 1 && h->variant == 0 && !h->line &&
                 h->nmag > 0;
    }
    if (h->pre) {
        for (int p = 0; p < 2; ++p)
            for (int c = 0; c < 3; ++c) {
                chk(field_alloc(h, &h->Hc[p][c], (size_t)h->nmag));
                chk(dev_alloc(h, &h->Mc[p][c], (size_t)h->nmag));
            }
        chk(dev_alloc(h, &h->cid, (size_t)h->nmag));
        if (rc) return rc;
        std::vector<uint8_t> cid((size_t)h->nmag);
        for (size_t q = 0; q < cid.size(); ++q)
            cid[q] = ids[(size_t)((cells[q].x - h->lo) * g.PP + cells[q].y)];
        CU(cudaMemcpy(h->cid, cid.data(), cid.size(), cudaMemcpyHostToDevice));
        h->hcells = cells;
        // one cooperative launch for the local LLG + r* (MPB_LLG_COOP=0: two
        // launches, k_llg_pre with programmatic launch + k_llg_fixup)
        h->pre_coop = true;
        if (const char* e = getenv("MPB_LLG_COOP")) h->pre_coop = atoi(e) != 0;
        if (h->pre_coop) {
            const size_t smem = (size_t)(g.max_iters + 2) * sizeof(unsigned long long);
            int per_sm = 0, sms = 0;
            if (h->f32) {
                CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_llg_pre_coop<float>,
                                                                 256, smem));
            } else {
                CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_llg_pre_coop<double>,
                                                                 256, smem));
            }
            CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
            h->coop_blocks = std::max(1, std::min((h->nmag + 255) / 256, per_sm * sms));
            // the sweep overlaps the cooperative LLG when the LLG is small:
            // fp64, at most half of the co-resident blocks (C1 +8-13%, C2
            // +4%); fp32, at most one block per 16 SMs (C1 +13%) -- the fp32
            // sweep's three CTAs per SM lose the slots the LLG blocks hold
            // (C2's 33 blocks: -5%).  A GPU-filling LLG (C3's film, 590K
            // cells) loses to the early sweep CTAs' competing traffic (fp32
            // C3 -14%).  MPB_LLG_OVERLAP=0 / 1: never / always
            const char* ov = getenv("MPB_LLG_OVERLAP");
            const int lb = (h->nmag + 255) / 256;
            g.llg_sync = (h->f32 ? 16 * lb <= sms : 2 * lb <= per_sm * sms) ? 1 : 0;
            if (ov) g.llg_sync = atoi(ov) != 0 ? 1 : 0;
        }
    }
    // E-range flags (kSafeBias) let the sweep's H phase skip its division
    // guard; every E writer of this configuration maintains them
    // (MPB_EGUARD=0: always guarded)
    {
        const char* e = getenv("MPB_EGUARD");
        g.eguard = (!(e && atoi(e) == 0) && nranks == 1 && h->variant == 0 && !h->line &&
                    !h->f32 && g.zin && !h->wall_per_face && (h->pre || h->nmag == 0)) ? 1 : 0;
    }
    if (h->variant != 1) {
        rc = prepare_fused(h, g);
        if (rc) return rc;
    }
    // source (em.py:276-282): only the owning rank injects
    for (int a = 0; a < 3; ++a) {
        if (su->src_loc[a] < 0 || su->src_loc[a] >= g.F[a]) { return fail_msg(MPB_EINVAL, "source location out of range");
        }
        h->src.pol[a] = su->src_pol[a];
    }
    if (su->src_loc[0] < g.c0 || su->src_loc[0] >= g.c1)
        h->src.pol[0] = h->src.pol[1] = h->src.pol[2] = 0.0;
    h->src.off = su->src_loc[0] * g.PP + (int64_t)su->src_loc[1] * F[2] + su->src_loc[2];

    // probes
    h->nprobes = su->n_probes;
    h->probe_comp.assign(su->probe_comp, su->probe_comp + su->n_probes);
    h->probe_loc.assign(su->probe_loc, su->probe_loc + 3 * su->n_probes);
    for (int p = 0; p < h->nprobes; ++p) {
        const int comp = h->probe_comp[p];
        const int* L = &h->probe_loc[3 * p];
        const int* lim = comp >= MPB_COMP_MX ? g.n : g.F;
        if (comp < 0 || comp > 8) { return fail_msg(MPB_EINVAL, "bad probe component"); }
        for (int a = 0; a < 3; ++a)
            if (L[a] < 0 || L[a] >= lim[a]) { return fail_msg(MPB_EINVAL, "probe %d outside grid", p);
            }
    }
    chk(dev_alloc(h, &h->probes, (size_t)std::max(1, h->nprobes)));
    if (h->line) chk(dev_alloc(h, &h->lprobes, (size_t)std::max(1, h->nprobes)));
    h->hostM.clear();
    if (rc) return rc;
    bool zero_id = true;
    for (int q = 0; q < 128; ++q) zero_id = zero_id && su->nccl_id[q] == 0;
    if (nranks > 1 && !zero_id) {   // all-zero id: in-process group (mpb_group_run)
        ncclUniqueId id;
        memcpy(&id, su->nccl_id, sizeof id);
        ncclResult_t r = ncclCommInitRank(&h->comm, nranks, id, h->rank);
        if (r != ncclSuccess) { return fail_msg(MPB_ECUDA, "ncclCommInitRank failed: %s", ncclGetErrorString(r));
        }
        if (h->overlap) {   // collective over the ranks, same order everywhere
            r = ncclCommSplit(h->comm, 0, h->rank, &h->comm_x, nullptr);
            if (r != ncclSuccess) { return fail_msg(MPB_ECUDA, "ncclCommSplit failed: %s", ncclGetErrorString(r));
            }
        }
    }
    rc = reset_state(h);
    if (rc) return rc;
    return MPB_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* mpb_version(void) {
    return "magphon_b200 0.3 sm_100a fp64 (+fp32 storage) fmad=false nccl";
}

const char* mpb_last_error(void) { return g_err.c_str(); }

int mpb_nccl_unique_id(uint8_t out[128]) {
    g_err.clear();
    if (!out) return fail_msg(MPB_EINVAL, "null argument");
    ncclUniqueId id;
    NC(ncclGetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    memcpy(out, &id, 128);
    return MPB_OK;
}

int mpb_create(const mpb_setup* su, mpb_handle** out) {
    g_err.clear();
    if (!su || !out) return fail_msg(MPB_EINVAL, "null argument");
    *out = nullptr;
    for (int a = 0; a < 3; ++a) {
        if (su->n[a] < 1) return fail_msg(MPB_EINVAL, "cell counts must be >= 1");
        if (!(su->d[a] > 0) || !std::isfinite(su->d[a]))
            return fail_msg(MPB_EINVAL, "cell sizes must be finite and > 0");
    }
    if (su->n_materials < 1 || su->n_materials > MPB_MAX_MATERIALS)
        return fail_msg(MPB_EINVAL, "need 1..%d materials, got %d", MPB_MAX_MATERIALS,
                        su->n_materials);
    if (su->llg_max_iters < 1 || su->llg_max_iters > MPB_MAX_ITERS_CAP)
        return fail_msg(MPB_EINVAL, "llg_max_iters must be in 1..%d", MPB_MAX_ITERS_CAP);
    if (!(su->llg_tol > 0)) return fail_msg(MPB_EINVAL, "llg_tol must be > 0");
    for (int f = 0; f < 6; ++f) {
        if (su->faces[f] < 0 || su->faces[f] > 2)
            return fail_msg(MPB_EINVAL, "bad face code on face %d", f);
        if (su->faces[f] == MPB_FACE_MUR1 && su->n[f >> 1] <= 1)
            return fail_msg(MPB_EINVAL, "MUR1 on collapsed axis face %d", f);
    }
    if (su->storage != MPB_STORAGE_F64 && su->storage != MPB_STORAGE_F32)
        return fail_msg(MPB_EINVAL, "bad storage mode %d", su->storage);
    if (su->storage == MPB_STORAGE_F32 && su->kernel_variant != 0)
        return fail_msg(MPB_EINVAL, "fp32 storage runs the fused sweep (variant 0) only");
    const int nranks = std::max(1, su->nranks);
    const int nx = su->n[0];
    const int x_lo = nranks == 1 ? 0 : su->x_lo;
    const int x_hi = nranks == 1 ? nx : su->x_hi;
    if (nranks > 1) {
        if (su->rank < 0 || su->rank >= nranks)
            return fail_msg(MPB_EINVAL, "rank %d out of range", su->rank);
        if (nx < 2 || x_lo < 0 || x_hi > nx || x_hi - x_lo < 2)
            return fail_msg(MPB_EINVAL, "slab [%d,%d) of %d cells: need >= 2 planes per rank",
                            x_lo, x_hi, nx);
        if ((su->rank == 0) != (x_lo == 0) || (su->rank == nranks - 1) != (x_hi == nx))
            return fail_msg(MPB_EINVAL, "slab ranges must be ordered by rank");
        if (su->kernel_variant == 1)
            return fail_msg(MPB_EINVAL, "multi-rank runs use the fused sweep (variant 0)");
    }
    auto* h = new mpb_handle();
    // every failure past this point releases what was set up so far
    const int rc = create_body(su, h, nranks, x_lo, x_hi);
    if (rc) { mpb_destroy(h); return rc; }
    *out = h;
    return MPB_OK;
}

void mpb_destroy(mpb_handle* h) {
    if (!h) return;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    for (auto& e : h->events) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
    dev_free(h, h->lprobes);
    for (int p = 0; p < 2; ++p) {
        if (h->graph[p]) cudaGraphExecDestroy(h->graph[p]);
        for (int c = 0; c < 3; ++c) {
            dev_free(h, h->E[p][c]);
            dev_free(h, h->H[p][c]);
            dev_free(h, h->M[p][c]);
        }
    }
    dev_free(h, h->ids);
    dev_free(h, h->mats);
    dev_free(h, h->magcells);
    dev_free(h, h->magowned);
    dev_free(h, h->scratch);
    for (int p = 0; p < 2; ++p)
        for (int c = 0; c < 3; ++c) { dev_free(h, h->Hc[p][c]); dev_free(h, h->Mc[p][c]); }
    dev_free(h, h->cid);
    dev_free(h, h->st);
    dev_free(h, h->probes);
    dev_free(h, h->d_src);
    dev_free(h, h->d_probe);
    dev_free(h, h->d_iters);
    free_run_stages(h);
    destroy_fused(h);
    if (h->stream) cudaStreamSynchronize(h->stream);
    if (h->comm_x) ncclCommDestroy(h->comm_x);
    if (h->comm) ncclCommDestroy(h->comm);
    if (h->ev_post) cudaEventDestroy(h->ev_post);
    if (h->ev_exch) cudaEventDestroy(h->ev_exch);
    if (h->comm_stream) cudaStreamDestroy(h->comm_stream);
    if (h->stream) cudaStreamDestroy(h->stream);
    delete h;
}

int mpb_load_state(mpb_handle* h, const double* const fields[6], const double* m) {
    g_err.clear();
    if (!h || !fields || !m) return fail_msg(MPB_EINVAL, "null argument");
    const Geom& g = h->g;
    CU(cudaSetDevice(h->device));
    CU(cudaStreamSynchronize(h->stream));
    const size_t row = (size_t)g.FyFz * sizeof(double);
    const int nplanes = h->hi - h->lo;
    const size_t whole = (size_t)nplanes * g.PP * h->esz;
    // fp32 storage: host doubles pass through a device staging buffer of
    // whole planes (bounded, so C5-size slabs never need a second full copy)
    const int batch = h->f32 ? (int)std::max<int64_t>(1, std::min<int64_t>(
                                   nplanes, (64ll << 20) / (g.PP * (int64_t)sizeof(double))))
                             : 0;
    double* stage = nullptr;
    if (h->f32) {   // the 2-D copies fill [0, FyFz) of each plane: pitch padding stays 0
        CU(cudaMalloc(&stage, (size_t)batch * g.PP * sizeof(double)));
        CU(cudaMemset(stage, 0, (size_t)batch * g.PP * sizeof(double)));
    }
    int rc = MPB_OK;
    for (int c = 0; c < 6 && !rc; ++c) {
        void* d0 = c < 3 ? h->E[0][c] : h->H[0][c - 3];
        void* d1 = c < 3 ? h->E[1][c] : h->H[1][c - 3];
        if (!fields[c]) {  // NULL: the component starts at zero
            if (cudaMemset(d0, 0, whole) != cudaSuccess || cudaMemset(d1, 0, whole) != cudaSuccess)
                rc = fail_msg(MPB_ECUDA, "cudaMemset failed");
            continue;
        }
        if (!h->f32) {     // upload once, replicate into the second buffer set
            CU(cudaMemcpy2D(d0, g.PP * sizeof(double), fields[c], row, row, nplanes,
                            cudaMemcpyHostToDevice));
        } else {
            for (int p0 = 0; p0 < nplanes && !rc; p0 += batch) {
                const int np = std::min(batch, nplanes - p0);
                // on the handle's stream: a pageable H2D cudaMemcpy2D may return
                // before its DMA lands, and the conversion must see the data
                if (cudaMemcpy2DAsync(stage, g.PP * sizeof(double),
                                      fields[c] + (size_t)p0 * g.FyFz, row, row, np,
                                      cudaMemcpyHostToDevice, h->stream) != cudaSuccess) {
                    rc = fail_msg(MPB_ECUDA, "staging upload failed");
                    break;
                }
                k_convert<double, float><<<1184, 256, 0, h->stream>>>(
                    stage, static_cast<float*>(d0) + (size_t)p0 * g.PP, (int64_t)np * g.PP);
                if (cudaStreamSynchronize(h->stream) != cudaSuccess)
                    rc = fail_msg(MPB_ECUDA, "fp32 conversion failed");
            }
        }
        if (!rc && cudaMemcpy(d1, d0, whole, cudaMemcpyDeviceToDevice) != cudaSuccess)
            rc = fail_msg(MPB_ECUDA, "device copy failed");
    }
    if (stage) cudaFree(stage);
    if (rc) return rc;
    // the device-to-device replicas above are asynchronous on the legacy
    // stream; the handle's (non-blocking) stream must not start before them
    CU(cudaStreamSynchronize(cudaStreamLegacy));
    const int ny = g.n[1], nz = g.n[2];
    const int ncl = h->chi - h->clo;
    {
        const size_t plane = (size_t)ny * nz, total = (size_t)3 * ncl * plane;
        bool zero = true;
        for (int c = 0; c < 3 && zero; ++c)
            for (int i = h->clo; i < h->chi && zero; ++i) {
                if (h->mplanes && i >= g.mx0 && i < g.mx1) continue;   // on the device
                const double* q = m + ((size_t)c * ncl + (i - h->clo)) * plane;
                for (size_t e = 0; e < plane; ++e)
                    if (dbits_host(q[e]) != 0) { zero = false; break; }
            }
        if (zero) {
            h->hostM.clear();
            h->hostM.shrink_to_fit();
        } else {
            h->hostM.assign(m, m + total);
        }
    }
    if (h->mplanes) {   // M planes, packed a bounded batch of planes at a time
        const int mb = (int)std::max<int64_t>(1, std::min<int64_t>(
            h->mplanes, (64ll << 20) / (g.PP * (int64_t)sizeof(double))));
        std::vector<double> pk((size_t)mb * g.PP, 0.0);
        for (int c = 0; c < 3; ++c)
            for (int i0 = g.mx0; i0 < g.mx1; i0 += mb) {
                const int np = std::min(mb, g.mx1 - i0);
                for (int i = i0; i < i0 + np; ++i)
                    for (int j = 0; j < ny; ++j)
                        for (int k = 0; k < nz; ++k)
                            pk[(size_t)((i - i0) * g.PP + (int64_t)j * g.F[2] + k)] =
                                m[(((size_t)c * ncl + (i - h->clo)) * ny + j) * nz + k];
                for (int p = 0; p < 2; ++p)
                    CU(cudaMemcpy(h->M[p][c] + (size_t)(i0 - g.mx0) * g.PP, pk.data(),
                                  (size_t)np * g.PP * sizeof(double), cudaMemcpyHostToDevice));
            }
    }
    h->parity = 0;
    rc = h->f32 ? pack_magnetic<float>(h, 0) : pack_magnetic<double>(h, 0);
    if (rc) return rc;
    rc = upload_probes(h);
    if (rc) return rc;
    return reset_state(h);
}

int mpb_save_state(mpb_handle* h, double* const fields[6], double* m) {
    g_err.clear();
    if (!h || !fields || !m) return fail_msg(MPB_EINVAL, "null argument");
    const Geom& g = h->g;
    CU(cudaSetDevice(h->device));
    CU(cudaStreamSynchronize(h->stream));
    if (int rc0 = unpack_magnetic(h)) return rc0;
    const size_t row = (size_t)g.FyFz * sizeof(double);
    const int p = h->parity;
    const int nplanes = h->hi - h->lo;
    const int batch = h->f32 ? (int)std::max<int64_t>(1, std::min<int64_t>(
                                   nplanes, (64ll << 20) / (g.PP * (int64_t)sizeof(double))))
                             : 0;
    double* stage = nullptr;
    if (h->f32) CU(cudaMalloc(&stage, (size_t)batch * g.PP * sizeof(double)));
    int rc = MPB_OK;
    for (int c = 0; c < 6 && !rc; ++c) {
        const void* src = c < 3 ? h->E[p][c] : h->H[p][c - 3];
        if (!h->f32) {
            CU(cudaMemcpy2D(fields[c], row, src, g.PP * sizeof(double), row, nplanes,
                            cudaMemcpyDeviceToHost));
            continue;
        }
        for (int p0 = 0; p0 < nplanes && !rc; p0 += batch) {   // widen, then download
            const int np = std::min(batch, nplanes - p0);
            k_convert<float, double><<<1184, 256, 0, h->stream>>>(
                static_cast<const float*>(src) + (size_t)p0 * g.PP, stage, (int64_t)np * g.PP);
            if (cudaStreamSynchronize(h->stream) != cudaSuccess ||
                cudaMemcpy2D(fields[c] + (size_t)p0 * g.FyFz, row, stage, g.PP * sizeof(double),
                             row, np, cudaMemcpyDeviceToHost) != cudaSuccess)
                rc = fail_msg(MPB_ECUDA, "staging download failed");
        }
    }
    if (stage) cudaFree(stage);
    if (rc) return rc;
    const int ny = g.n[1], nz = g.n[2];
    const int ncl = h->chi - h->clo;
    if (h->hostM.empty())
        memset(m, 0, sizeof(double) * (size_t)3 * ncl * ny * nz);
    else
        memcpy(m, h->hostM.data(), h->hostM.size() * sizeof(double));
    if (h->mplanes) {   // M planes, a bounded batch of planes at a time
        const int mb = (int)std::max<int64_t>(1, std::min<int64_t>(
            h->mplanes, (64ll << 20) / (g.PP * (int64_t)sizeof(double))));
        std::vector<double> pk((size_t)mb * g.PP);
        for (int c = 0; c < 3; ++c)
            for (int i0 = g.mx0; i0 < g.mx1; i0 += mb) {
                const int np = std::min(mb, g.mx1 - i0);
                CU(cudaMemcpy(pk.data(), h->M[p][c] + (size_t)(i0 - g.mx0) * g.PP,
                              (size_t)np * g.PP * sizeof(double), cudaMemcpyDeviceToHost));
                for (int i = i0; i < i0 + np; ++i)
                    for (int j = 0; j < ny; ++j)
                        for (int k = 0; k < nz; ++k)
                            m[(((size_t)c * ncl + (i - h->clo)) * ny + j) * nz + k] =
                                pk[(size_t)((i - i0) * g.PP + (int64_t)j * g.F[2] + k)];
            }
    }
    return MPB_OK;
}

int mpb_run_device(mpb_handle* h, int64_t n0, int64_t nsteps, const double* d_src_vals,
                   double* d_probe_out, int32_t* d_iters_out, void* stream) {
    g_err.clear();
    if (!h || nsteps < 0) return fail_msg(MPB_EINVAL, "bad arguments");
    CU(cudaSetDevice(h->device));
    // order our stream after the caller's work (0 = legacy default stream)
    cudaStream_t cs = stream ? (cudaStream_t)stream : cudaStreamLegacy;
    cudaEvent_t ev = nullptr;
    CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CU(cudaEventRecord(ev, cs));
    CU(cudaStreamWaitEvent(h->stream, ev, 0));
    h->launches_last = 0;
    int rc = set_run_buffers(h, n0, d_src_vals, d_probe_out, d_iters_out);
    if (!rc) rc = enqueue_steps(h, nsteps);
    // and the caller's stream after ours
    CU(cudaEventRecord(ev, h->stream));
    CU(cudaStreamWaitEvent(cs, ev, 0));
    CU(cudaEventDestroy(ev));
    return rc;
}

namespace {
// Multi-rank mpb_run: one chunk at a time with a host check after each, so a
// suspended step (kMpbSuspend) can be continued before the chunk goes on.
int run_sync(mpb_handle* h, int64_t n0, int64_t nsteps, const double* src_vals,
             double* probe_out, int32_t* iters_out, mpb_failure* fail) {
    const int64_t cap = std::min<int64_t>(std::max<int64_t>(nsteps, 1), kRunChunk);
    if (cap > h->stage_cap) {
        dev_free(h, h->d_src); dev_free(h, h->d_probe); dev_free(h, h->d_iters);
        h->d_src = nullptr; h->d_probe = nullptr; h->d_iters = nullptr;
        int rc = dev_alloc(h, &h->d_src, (size_t)cap);
        if (!rc) rc = dev_alloc(h, &h->d_probe, (size_t)(cap * std::max(1, h->nprobes)));
        if (!rc) rc = dev_alloc(h, &h->d_iters, (size_t)cap);
        if (rc) return rc;
        h->stage_cap = cap;
    }
    int64_t launches = 0;
    for (int64_t s0 = 0; s0 < nsteps; s0 += cap) {
        const int64_t cnt = std::min(cap, nsteps - s0);
        CU(cudaMemcpyAsync(h->d_src, src_vals + s0, cnt * sizeof(double),
                           cudaMemcpyHostToDevice, h->stream));
        h->launches_last = 0;
        const int p0 = h->parity;
        int rc = set_run_buffers(h, n0 + s0, h->d_src, h->d_probe, h->d_iters);
        if (!rc) rc = enqueue_steps(h, cnt);
        if (rc) return rc;
        mpb_failure fl;
        rc = read_failure(h, &fl);
        // a multi-rank step whose global residual went back above tol was
        // suspended (every later step of the chunk did nothing): continue it
        // on the host, then run the rest of the chunk
        while (rc == MPB_ESTEP && fl.kind == kMpbSuspend) {
            const int64_t k = fl.step - (n0 + s0);     // index within the chunk
            h->parity = p0 ^ (int)(k & 1);
            if ((rc = recover_suspended(&h, 1, false, h->stream))) return rc;
            h->parity ^= 1;
            rc = read_failure(h, &fl);
            if (rc != MPB_OK) break;                   // the continuation failed
            if ((rc = enqueue_steps(h, cnt - k - 1))) return rc;
            rc = read_failure(h, &fl);
        }
        launches += h->launches_last;
        if (h->nprobes && probe_out)
            CU(cudaMemcpyAsync(probe_out + s0 * h->nprobes, h->d_probe,
                               cnt * h->nprobes * sizeof(double), cudaMemcpyDeviceToHost,
                               h->stream));
        if (iters_out)
            CU(cudaMemcpyAsync(iters_out + s0, h->d_iters, cnt * sizeof(int),
                               cudaMemcpyDeviceToHost, h->stream));
        CU(cudaStreamSynchronize(h->stream));
        if (rc == MPB_ESTEP) {
            if (fail) *fail = fl;
            h->launches_last = launches;
            return fail_msg(MPB_ESTEP, "LLG fixed point failed at step %lld",
                            (long long)fl.step);
        }
        if (rc) return rc;
    }
    h->launches_last = launches;
    return MPB_OK;
}

// Single rank: chunks are double-buffered.  Chunk c is enqueued (source
// values staged through pinned memory, the steps, then its probes, r* and
// the step state copied to pinned memory behind an event) before the host
// waits for chunk c-1 and hands its rows to the caller, so the GPU never
// idles on the host between chunks.  A failure found in chunk c-1 returns
// after the stream drains (the later chunk's kernels were no-ops).
int run_pipelined(mpb_handle* h, int64_t n0, int64_t nsteps, const double* src_vals,
                  double* probe_out, int32_t* iters_out, mpb_failure* fail) {
    const int64_t cap = std::min<int64_t>(std::max<int64_t>(nsteps, 1), kRunChunk);
    int rc = alloc_run_stages(h, cap);
    if (rc) return rc;
    const int np = h->nprobes;
    int64_t launches = 0;
    auto harvest = [&](mpb_handle::RunStage& r) -> int {
        CU(cudaEventSynchronize(r.done));
        r.busy = false;
        if (np && probe_out)
            memcpy(probe_out + r.s0 * np, r.h_probe, sizeof(double) * r.cnt * np);
        if (iters_out) memcpy(iters_out + r.s0, r.h_iters, sizeof(int) * r.cnt);
        const StepState& st = *r.h_st;
        if (st.fail) {
            CU(cudaStreamSynchronize(h->stream));
            for (auto& o : h->rs) o.busy = false;
            if (fail) {
                fail->step = st.fail_step; fail->residual = st.fail_res;
                fail->iterations = st.fail_it; fail->kind = st.fail_kind;
            }
            return fail_msg(MPB_ESTEP, "LLG fixed point failed at step %lld",
                            (long long)st.fail_step);
        }
        return MPB_OK;
    };
    int c = 0;
    for (int64_t s0 = 0; s0 < nsteps; s0 += cap, ++c) {
        mpb_handle::RunStage& r = h->rs[c & 1];
        if (r.busy && (rc = harvest(r))) { h->launches_last = launches; return rc; }
        const int64_t cnt = std::min(cap, nsteps - s0);
        memcpy(r.h_src, src_vals + s0, sizeof(double) * cnt);
        CU(cudaMemcpyAsync(r.d_src, r.h_src, sizeof(double) * cnt, cudaMemcpyHostToDevice,
                           h->stream));
        h->launches_last = 0;
        if ((rc = set_run_buffers(h, n0 + s0, r.d_src, r.d_probe, r.d_iters))) return rc;
        if ((rc = enqueue_steps(h, cnt))) return rc;
        launches += h->launches_last;
        if (np)
            CU(cudaMemcpyAsync(r.h_probe, r.d_probe, sizeof(double) * cnt * np,
                               cudaMemcpyDeviceToHost, h->stream));
        CU(cudaMemcpyAsync(r.h_iters, r.d_iters, sizeof(int) * cnt, cudaMemcpyDeviceToHost,
                           h->stream));
        CU(cudaMemcpyAsync(r.h_st, h->st, sizeof(StepState), cudaMemcpyDeviceToHost,
                           h->stream));
        CU(cudaEventRecord(r.done, h->stream));
        r.s0 = s0; r.cnt = cnt; r.busy = true;
    }
    // the older of the two outstanding chunks first
    for (int k = 0; k < 2; ++k) {
        mpb_handle::RunStage& r = h->rs[(c + k) & 1];
        if (r.busy && (rc = harvest(r))) { h->launches_last = launches; return rc; }
    }
    h->launches_last = launches;
    return MPB_OK;
}

}  // namespace

int mpb_run(mpb_handle* h, int64_t n0, int64_t nsteps, const double* src_vals,
            double* probe_out, int32_t* iters_out, mpb_failure* fail) {
    g_err.clear();
    if (fail) { fail->step = -1; fail->residual = 0; fail->iterations = 0; fail->kind = 0; }
    if (!h || nsteps < 0 || (nsteps && !src_vals))
        return fail_msg(MPB_EINVAL, "bad arguments");
    CU(cudaSetDevice(h->device));
    if (h->nranks > 1) return run_sync(h, n0, nsteps, src_vals, probe_out, iters_out, fail);
    return run_pipelined(h, n0, nsteps, src_vals, probe_out, iters_out, fail);
}

int mpb_check_failure(mpb_handle* h, mpb_failure* fail) {
    g_err.clear();
    if (!h) return fail_msg(MPB_EINVAL, "null handle");
    CU(cudaSetDevice(h->device));
    return read_failure(h, fail);
}

int mpb_set_kernel_timing(mpb_handle* h, int enable) {
    if (!h) return fail_msg(MPB_EINVAL, "null handle");
    CU(cudaSetDevice(h->device));
    CU(cudaStreamSynchronize(h->stream));
    for (auto& e : h->events) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
    h->events.clear();
    h->timed_ms = 0.0;
    h->timed_launches = 0;
    h->timing = enable;
    return MPB_OK;
}

int mpb_kernel_time(mpb_handle* h, double* ms_total, int64_t* launches,
                    const char** kernel_name) {
    if (!h) return fail_msg(MPB_EINVAL, "null handle");
    CU(cudaSetDevice(h->device));
    CU(cudaStreamSynchronize(h->stream));
    for (auto& e : h->events) {
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, e.first, e.second));
        h->timed_ms += ms;
        ++h->timed_launches;
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    h->events.clear();
    if (ms_total) *ms_total = h->timed_ms;
    // the split variant brackets two kernels per step; report per step
    if (launches) *launches = h->variant == 1 ? h->timed_launches / 2 : h->timed_launches;
    if (kernel_name) *kernel_name = h->variant == 1 ? "k_hsweep+k_esweep" : fused_kernel_name();
    return MPB_OK;
}

int mpb_selftest_division(int32_t device, double d, const double* x, int64_t n,
                          int64_t* mismatches, double* first_bad) {
    g_err.clear();
    if (!x || n < 0 || !mismatches) return fail_msg(MPB_EINVAL, "bad arguments");
    CU(cudaSetDevice(device));
    double* dx = nullptr;
    unsigned long long* dm = nullptr;
    double* db = nullptr;
    CU(cudaMalloc(&dx, sizeof(double) * std::max<int64_t>(n, 1)));
    CU(cudaMalloc(&dm, sizeof(unsigned long long)));
    CU(cudaMalloc(&db, sizeof(double)));
    CU(cudaMemset(dm, 0, sizeof(unsigned long long)));
    CU(cudaMemset(db, 0, sizeof(double)));
    CU(cudaMemcpy(dx, x, sizeof(double) * n, cudaMemcpyHostToDevice));
    k_div_selftest<<<1184, 256>>>(dx, n, d, dm, db);
    CU(cudaGetLastError());
    unsigned long long mm = 0;
    double bad = 0;
    CU(cudaMemcpy(&mm, dm, sizeof mm, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(&bad, db, sizeof bad, cudaMemcpyDeviceToHost));
    cudaFree(dx); cudaFree(dm); cudaFree(db);
    *mismatches = (int64_t)mm;
    if (first_bad) *first_bad = bad;
    return MPB_OK;
}

int mpb_group_run(mpb_handle* const* hs, int32_t n, int64_t n0, int64_t nsteps,
                  const double* src_vals, double* const* probe_out, int32_t* iters_out,
                  mpb_failure* fail) {
    g_err.clear();
    if (fail) { fail->step = -1; fail->residual = 0; fail->iterations = 0; fail->kind = 0; }
    if (!hs || n < 2 || n > kMaxGroup || nsteps < 0 || (nsteps && !src_vals))
        return fail_msg(MPB_EINVAL, "bad arguments");
    for (int r = 0; r < n; ++r) {
        if (!hs[r] || hs[r]->nranks != n || hs[r]->rank != r || hs[r]->comm ||
            hs[r]->device != hs[0]->device || hs[r]->parity != hs[0]->parity)
            return fail_msg(MPB_EINVAL, "group: handles must be ranks 0..n-1 of one "
                                        "decomposition on one device, created without NCCL");
    }
    CU(cudaSetDevice(hs[0]->device));
    cudaStream_t s = hs[0]->stream;
    std::vector<double*> dprobe((size_t)n, nullptr);
    double* dsrc = nullptr;
    int* diters = nullptr;
    const int64_t cnt = std::max<int64_t>(nsteps, 1);
    CU(cudaMalloc(&dsrc, cnt * sizeof(double)));
    CU(cudaMalloc(&diters, cnt * sizeof(int) * n));
    CU(cudaMemcpy(dsrc, src_vals, nsteps * sizeof(double), cudaMemcpyHostToDevice));
    int rc = MPB_OK;
    for (int r = 0; r < n && !rc; ++r) {
        CU(cudaMalloc(&dprobe[(size_t)r], cnt * std::max(1, hs[r]->nprobes) * sizeof(double)));
        rc = set_run_buffers(hs[r], n0, dsrc, dprobe[(size_t)r], diters + r * cnt);
        // (on rank r's own stream; the group steps on rank 0's)
        if (!rc) CU(cudaStreamSynchronize(hs[r]->stream));
    }
    int64_t t = 0;
    while (t < nsteps && !rc) {
        const int64_t t0 = t;
        const int p0 = hs[0]->parity;
        for (; t < nsteps && !rc; ++t) {
            rc = group_step(hs, n, hs[0]->parity, s);
            for (int r = 0; r < n; ++r) hs[r]->parity ^= 1;
        }
        if (!rc) rc = drain_exchange(hs[0], s);
        if (rc) break;
        mpb_failure fl;
        if (read_failure(hs[0], &fl) != MPB_ESTEP || fl.kind != kMpbSuspend) break;
        // suspended step (see recover_suspended): continue it, then go on
        const int64_t k = fl.step - n0;
        for (int r = 0; r < n; ++r) hs[r]->parity = p0 ^ (int)((k - t0) & 1);
        rc = recover_suspended(hs, n, true, s);
        for (int r = 0; r < n; ++r) hs[r]->parity ^= 1;
        t = k + 1;
        if (!rc && read_failure(hs[0], &fl) == MPB_ESTEP) break;
    }
    if (!rc) {
        CU(cudaStreamSynchronize(s));
        for (int r = 0; r < n; ++r)
            if (probe_out && probe_out[r] && hs[r]->nprobes)
                CU(cudaMemcpy(probe_out[r], dprobe[(size_t)r],
                              nsteps * hs[r]->nprobes * sizeof(double), cudaMemcpyDeviceToHost));
        if (iters_out) CU(cudaMemcpy(iters_out, diters, nsteps * sizeof(int), cudaMemcpyDeviceToHost));
        mpb_failure fl;
        rc = read_failure(hs[0], &fl);
        if (rc == MPB_ESTEP) {
            if (fail) *fail = fl;
            fail_msg(MPB_ESTEP, "LLG fixed point failed at step %lld", (long long)fl.step);
        }
    }
    cudaFree(dsrc);
    cudaFree(diters);
    for (double* p : dprobe) cudaFree(p);
    return rc;
}

int mpb_total_energy(mpb_handle* h, double* out) {
    g_err.clear();
    if (!h || !out) return fail_msg(MPB_EINVAL, "null argument");
    CU(cudaSetDevice(h->device));
    CU(cudaStreamSynchronize(h->stream));
    if (int rc0 = unpack_magnetic(h)) return rc0;
    const Geom& g = h->g;
    const int p = h->parity;
    const void* hp[9];
    for (int c = 0; c < 3; ++c) {
        hp[c] = h->f32 ? (const void*)fview<float>(h->E[p][c], h)
                       : (const void*)fview<double>(h->E[p][c], h);
        hp[3 + c] = h->f32 ? (const void*)fview<float>(h->H[p][c], h)
                           : (const void*)fview<double>(h->H[p][c], h);
        hp[6 + c] = h->M[p][c];
    }
    const void** dptr = nullptr;
    CU(cudaMallocAsync(&dptr, 9 * sizeof(void*), h->stream));
    CU(cudaMemcpyAsync(dptr, hp, sizeof hp, cudaMemcpyHostToDevice, h->stream));
    const int blocks = 1184;
    double* partial = nullptr;
    CU(cudaMallocAsync(&partial, 3 * blocks * sizeof(double), h->stream));
    const double* const* dm = reinterpret_cast<const double* const*>(dptr + 6);
    if (h->f32)
        k_energy_partial<float><<<blocks, 256, 0, h->stream>>>(
            g, reinterpret_cast<const float* const*>(dptr),
            reinterpret_cast<const float* const*>(dptr + 3), dm, h->mats, ids_view(h), partial);
    else
        k_energy_partial<double><<<blocks, 256, 0, h->stream>>>(
            g, reinterpret_cast<const double* const*>(dptr),
            reinterpret_cast<const double* const*>(dptr + 3), dm, h->mats, ids_view(h), partial);
    CU(cudaGetLastError());
    std::vector<double> hpart((size_t)3 * blocks);
    CU(cudaMemcpyAsync(hpart.data(), partial, hpart.size() * sizeof(double),
                       cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    dev_free(h, partial);
    dev_free(h, dptr);
    double se = 0.0, sh = 0.0, sm = 0.0;
    for (int b = 0; b < blocks; ++b) {
        se += hpart[3 * b];
        sh += hpart[3 * b + 1];
        sm += hpart[3 * b + 2];
    }
    const double mu0 = 4e-7 * 3.141592653589793;
    const double vol = g.d[0] * g.d[1] * g.d[2];
    *out = (0.5 * se + 0.5 * mu0 * sh + (-mu0) * sm) * vol;
    return MPB_OK;
}

int mpb_comm_info(mpb_handle* h, int32_t* nranks, int32_t* rank, int32_t* nccl_version) {
    g_err.clear();
    if (!h || !nranks || !rank || !nccl_version) return fail_msg(MPB_EINVAL, "null argument");
    int v = 0;
    NC(ncclGetVersion(&v));
    *nccl_version = v;
    *nranks = h->nranks;
    *rank = h->rank;
    if (h->comm) {   // what the communicator itself reports
        int cnt = 0, me = 0;
        NC(ncclCommCount(h->comm, &cnt));
        NC(ncclCommUserRank(h->comm, &me));
        *nranks = cnt;
        *rank = me;
    }
    return MPB_OK;
}

int64_t mpb_launch_count(mpb_handle* h) { return h ? h->launches_last : 0; }

int mpb_hankel_mul(int32_t device, const double* x, int64_t n, int32_t columns, int32_t r,
                   int32_t transpose, const double* in, double* out) {
    g_err.clear();
    if (!x || !in || !out || columns < 1 || n < columns || r < 1 || r > kHankelMaxR)
        return fail_msg(MPB_EINVAL, "hankel: need 1 <= columns <= n and 1 <= r <= %d",
                        kHankelMaxR);
    CU(cudaSetDevice(device));
    const int64_t M = n - columns + 1, L = columns;
    const int64_t nin = (transpose ? M : L) * r, nout = (transpose ? L : M) * r;
    double *dx = nullptr, *din = nullptr, *dout = nullptr, *part = nullptr;
    cudaStream_t s = nullptr;
    int rc = MPB_OK;
    auto ok = [&](cudaError_t e, const char* what) {
        if (e != cudaSuccess && !rc) rc = fail_msg(MPB_ECUDA, "hankel %s: %s", what,
                                                   cudaGetErrorString(e));
        return rc == MPB_OK;
    };
    if (ok(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream") &&
        ok(cudaMallocAsync(&dx, sizeof(double) * n, s), "alloc") &&
        ok(cudaMallocAsync(&din, sizeof(double) * nin, s), "alloc") &&
        ok(cudaMallocAsync(&dout, sizeof(double) * nout, s), "alloc") &&
        ok(cudaMemcpyAsync(dx, x, sizeof(double) * n, cudaMemcpyHostToDevice, s), "upload") &&
        ok(cudaMemcpyAsync(din, in, sizeof(double) * nin, cudaMemcpyHostToDevice, s), "upload")) {
        if (!transpose) {
            k_hankel_fwd<<<(unsigned)((M + kHankelTile - 1) / kHankelTile), kHankelTile, 0, s>>>(
                dx, M, (int)L, r, din, dout);
        } else {
            const int split = (int)std::min<int64_t>(kHankelSplit, (M + kHankelTile - 1) / kHankelTile);
            if (ok(cudaMallocAsync(&part, sizeof(double) * split * nout, s), "alloc")) {
                k_hankel_tr<<<dim3((unsigned)((L + kHankelTile - 1) / kHankelTile), split),
                              kHankelTile, 0, s>>>(dx, M, (int)L, r, din, part);
                k_hankel_sum<<<(unsigned)std::min<int64_t>(1184, (nout + 255) / 256), 256, 0, s>>>(
                    part, split, nout, dout);
            }
        }
        if (ok(cudaGetLastError(), "launch"))
            ok(cudaMemcpyAsync(out, dout, sizeof(double) * nout, cudaMemcpyDeviceToHost, s),
               "download");
        ok(cudaStreamSynchronize(s), "sync");
    }
    if (s) {
        for (double* p : {dx, din, dout, part}) if (p) cudaFreeAsync(p, s);
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
    }
    return rc;
}

int64_t mpb_continued_steps(mpb_handle* h) { return h ? h->continued_steps : 0; }

int mpb_sweep_form(mpb_handle* h, int32_t out[4]) {
    g_err.clear();
    if (!h || !out) return fail_msg(MPB_EINVAL, "null argument");
    fused_form(h, out);
    return MPB_OK;
}

int64_t mpb_device_bytes(mpb_handle* h) { return h ? h->bytes : 0; }

}  // extern "C"

#include "mpb_fused.cuh"
