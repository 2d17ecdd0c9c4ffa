// mpb_api.cu -- C ABI of the B200 Maxwell-LLG stepper (include/magphon_b200.h).
//
// Owns device memory, streams and CUDA graphs for one run; sequences the
// per-step kernels.  Build: see paper_2510_22221_b200/csrc/Makefile.
#include <cuda_runtime.h>

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

using namespace mpb;

namespace {

thread_local std::string g_err;

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

constexpr int kDefaultGraphSteps = 16;
constexpr int64_t kRunChunk = 1 << 16;   // steps per host<->device staging chunk

}  // namespace

struct mpb_handle {
    int device = 0;
    Geom g{};
    int variant = 0;
    int graph_steps = kDefaultGraphSteps;
    int Fx = 1;
    int64_t nentries = 0;          // Fx * PP
    int64_t mplanes = 0;           // mx1 - mx0
    double* E[2][3] = {};
    double* H[2][3] = {};
    double* M[2][3] = {};
    uint8_t* ids = nullptr;
    mpb_material* mats = nullptr;
    int2* magcells = nullptr;
    int nmag = 0;
    double* scratch = nullptr;
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
    cudaStream_t stream = nullptr;
    cudaGraphExec_t graph[2] = {nullptr, nullptr};
    // host copy of M (cells outside the device M range never change)
    std::vector<double> hostM;
    // timing
    int timing = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events;
    double timed_ms = 0.0;
    int64_t timed_launches = 0;
    int64_t launches_last = 0;
    int64_t bytes = 0;
    int nmat_table = 0;
    void* fused = nullptr;         // FusedState (mpb_fused.cuh)
};


namespace {
// Fused single-sweep variant hooks (filled in by mpb_fused.cuh).
int prepare_fused(mpb_handle* h, const Geom& g);
void destroy_fused(mpb_handle* h);
int launch_fused(mpb_handle* h, const Geom& g, const Bufs& b, cudaStream_t s);
int launch_deferred(mpb_handle* h, const Geom& g, const Bufs& b, cudaStream_t s);
int launch_zfix(mpb_handle* h, const Geom& g, const Bufs& b, cudaStream_t s);
int zfix_launches(mpb_handle* h);
const char* fused_kernel_name();
}  // namespace

namespace {

Bufs make_bufs(const mpb_handle* h, int pa) {
    Bufs b{};
    const int pb = 1 - pa;
    for (int c = 0; c < 3; ++c) {
        b.Ea[c] = h->E[pa][c];
        b.Ha[c] = h->H[pa][c];
        b.Ma[c] = h->M[pa][c];
        b.Eb[c] = h->E[pb][c];
        b.Hb[c] = h->H[pb][c];
        b.Mb[c] = h->M[pb][c];
    }
    return b;
}

template <typename T>
int dev_alloc(mpb_handle* h, T** p, size_t count) {
    if (count == 0) { *p = nullptr; return MPB_OK; }
    CU(cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T)));
    CU(cudaMemset(*p, 0, count * sizeof(T)));
    h->bytes += (int64_t)(count * sizeof(T));
    return MPB_OK;
}

int reset_state(mpb_handle* h) {
    StepState s{};
    memset(&s, 0, sizeof s);
    s.rc_min = 0x7fffffff;
    s.fail_step = -1;
    CU(cudaMemcpyAsync(h->st, &s, sizeof s, cudaMemcpyHostToDevice, h->stream));
    return MPB_OK;
}

// Enqueue one coupled step reading buffer set `pa`.
int enqueue_step(mpb_handle* h, int pa, bool timed) {
    const Geom& g = h->g;
    const Bufs b = make_bufs(h, pa);
    cudaStream_t s = h->stream;
    int64_t launches = 0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timed) {
        CU(cudaEventCreate(&e0));
        CU(cudaEventCreate(&e1));
        CU(cudaEventRecord(e0, s));
    }
    const size_t hist_smem = (size_t)(g.max_iters + 2) * sizeof(unsigned long long);
    if (h->variant == 1) {
        dim3 grid((g.FyFz + 255) / 256, h->Fx);
        k_hsweep<<<grid, 256, hist_smem, s>>>(g, b, h->mats, h->ids, h->st);
        ++launches;
    } else {
        int rc = launch_fused(h, g, b, s);
        if (rc) return rc;
        ++launches;
    }
    if (timed && h->variant == 1) CU(cudaEventRecord(e1, s));
    if (h->nmag > 0) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(h->fixup_blocks);
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        MagScratch scr{h->scratch};
        CU(cudaLaunchKernelEx(&cfg, k_llg_fixup, g, b, (const mpb_material*)h->mats,
                              (const uint8_t*)h->ids, (const int2*)h->magcells, h->nmag,
                              scr, h->st));
        ++launches;
        if (h->variant != 1) {
            // fused sweep: E entries next to magnetic cells are recomputed
            // once r* is settled
            int rc = launch_deferred(h, g, b, s);
            if (rc) return rc;
            ++launches;
        }
    }
    if (h->variant == 1) {
        cudaEvent_t ea = nullptr, eb = nullptr;
        if (timed) {
            CU(cudaEventCreate(&ea));
            CU(cudaEventCreate(&eb));
            CU(cudaEventRecord(ea, s));
        }
        dim3 grid((g.FyFz + 255) / 256, h->Fx);
        k_esweep<<<grid, 256, 0, s>>>(g, b, h->mats, h->ids, h->st);
        ++launches;
        if (timed) {
            CU(cudaEventRecord(eb, s));
            h->events.emplace_back(ea, eb);
        }
    }
    if (timed && h->variant != 1) CU(cudaEventRecord(e1, s));
    if (timed) h->events.emplace_back(e0, e1);
    // fused variant: z walls are applied inside the sweep (+ k_zfix below)
    const int nface = h->variant == 1 ? 6 : 4;
    for (int face = 0; face < nface; ++face) {
        if (!h->faces_active[face]) continue;
        const int axis = face >> 1;
        const int u = axis == 0 ? 1 : 0, w = axis == 2 ? 1 : 2;
        const int64_t cnt = (int64_t)g.F[u] * g.F[w];
        k_wall<<<(unsigned)((cnt + 255) / 256), 256, 0, s>>>(g, b, h->mats, h->ids, h->st,
                                                            face);
        ++launches;
    }
    if (h->variant != 1) {
        int rc = launch_zfix(h, g, b, s);
        if (rc) return rc;
        launches += zfix_launches(h);
    }
    k_finish<<<1, 256, 0, s>>>(g, b, h->src, h->probes, h->nprobes, 1 - pa,
                               h->nmag > 0 ? 1 : 0, h->st);
    ++launches;
    h->launches_last += launches;
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
    h->launches_last = saved;
    cudaError_t e = cudaStreamEndCapture(h->stream, &graph);
    if (rc) return rc;
    if (e != cudaSuccess)
        return fail_msg(MPB_ECUDA, "graph capture failed: %s", cudaGetErrorString(e));
    CU(cudaGraphInstantiate(&h->graph[start_parity], graph, 0));
    CU(cudaGraphDestroy(graph));
    return MPB_OK;
}

int64_t launches_per_step(const mpb_handle* h) {
    int64_t n = (h->variant == 1 ? 2 : 1) + 1;
    if (h->nmag > 0) n += (h->variant == 1 ? 1 : 2);
    for (int f = 0; f < (h->variant == 1 ? 6 : 4); ++f) n += h->faces_active[f];
    if (h->variant != 1) n += zfix_launches(const_cast<mpb_handle*>(h));
    return n;
}

// Enqueue nsteps steps; buffers already pointed to by the device state.
int enqueue_steps(mpb_handle* h, int64_t nsteps) {
    int64_t s = 0;
    const bool use_graph = !h->timing && h->graph_steps > 1;
    while (s < nsteps) {
        if (use_graph && nsteps - s >= h->graph_steps) {
            if (!h->graph[h->parity]) {
                int rc = build_graph(h, h->parity);
                if (rc) return rc;
            }
            CU(cudaGraphLaunch(h->graph[h->parity], h->stream));
            h->launches_last += launches_per_step(h) * h->graph_steps;
            if (h->graph_steps & 1) h->parity ^= 1;
            s += h->graph_steps;
        } else {
            int rc = enqueue_step(h, h->parity, h->timing != 0);
            if (rc) return rc;
            h->parity ^= 1;
            ++s;
        }
    }
    return MPB_OK;
}

int set_run_buffers(mpb_handle* h, int64_t n0, const double* src, double* probe,
                    int* iters) {
    struct {
        long long step, local;
        const double* s;
        double* p;
        int* it;
    } v{n0, 0, src, probe, iters};
    // step, local, src_vals, probe_out, iters_out are laid out contiguously
    static_assert(offsetof(StepState, local) == offsetof(StepState, step) + 8, "layout");
    CU(cudaMemcpyAsync(&h->st->step, &v.step, sizeof(long long), cudaMemcpyHostToDevice,
                       h->stream));
    CU(cudaMemcpyAsync(&h->st->local, &v.local, sizeof(long long),
                       cudaMemcpyHostToDevice, h->stream));
    CU(cudaMemcpyAsync(&h->st->src_vals, &v.s, sizeof(void*), cudaMemcpyHostToDevice,
                       h->stream));
    CU(cudaMemcpyAsync(&h->st->probe_out, &v.p, sizeof(void*), cudaMemcpyHostToDevice,
                       h->stream));
    CU(cudaMemcpyAsync(&h->st->iters_out, &v.it, sizeof(void*), cudaMemcpyHostToDevice,
                       h->stream));
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

}  // namespace

// ---------------------------------------------------------------------------
// ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* mpb_version(void) {
    return "magphon_b200 0.1 sm_100a fp64 fmad=false";
}

const char* mpb_last_error(void) { return g_err.c_str(); }

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
    auto* h = new mpb_handle();
    h->device = su->device;
    h->variant = su->kernel_variant;
    h->graph_steps = su->graph_steps > 0 ? su->graph_steps : kDefaultGraphSteps;
    CU(cudaSetDevice(h->device));
    CU(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));

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
    g.coef_h = su->coef_h;
    for (int f = 0; f < 6; ++f) {
        g.faces[f] = su->faces[f];
        h->faces_active[f] = g.act[f >> 1] && su->faces[f] != MPB_FACE_PMC;
    }
    g.max_iters = su->llg_max_iters;
    g.tol = su->llg_tol;
    h->Fx = (int)F[0];
    h->nmat_table = MPB_MAX_MATERIALS;
    h->nentries = F[0] * g.PP;

    // material table renumbered so that magnetic materials carry bit 7 of
    // the id (the sweep tests magnetism without a table lookup)
    std::vector<int> remap((size_t)su->n_materials);
    std::vector<mpb_material> table(MPB_MAX_MATERIALS);
    memset(table.data(), 0, sizeof(mpb_material) * table.size());
    {
        int nm = 0, mm = 0;
        for (int q = 0; q < su->n_materials; ++q) {
            const int id = su->materials[q].magnetic ? 128 + mm++ : nm++;
            if (nm > 128 || mm > 128) {
                delete h;
                return fail_msg(MPB_EINVAL, "at most 128 magnetic and 128 non-magnetic materials");
            }
            remap[(size_t)q] = id;
            table[(size_t)id] = su->materials[q];
        }
    }
    // material ids on the allocation layout, edge-padded (em.py:248-252)
    const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
    std::vector<uint8_t> ids((size_t)h->nentries, 0);
    std::vector<int2> cells;
    int mx0 = nx, mx1 = 0;
    for (int i = 0; i < F[0]; ++i)
        for (int j = 0; j < F[1]; ++j)
            for (int k = 0; k < F[2]; ++k) {
                const int ci = std::min(i, nx - 1), cj = std::min(j, ny - 1),
                          ck = std::min(k, nz - 1);
                const uint8_t id0 = su->cell_material[((size_t)ci * ny + cj) * nz + ck];
                if (id0 >= su->n_materials) {
                    delete h;
                    return fail_msg(MPB_EINVAL, "material id %d out of range", id0);
                }
                const uint8_t id = (uint8_t)remap[id0];
                const int64_t f = (int64_t)j * F[2] + k;
                ids[(size_t)(i * g.PP + f)] = id;
                if (i < nx && j < ny && k < nz && table[id].magnetic) {
                    cells.push_back(make_int2(i, (int)f));
                    mx0 = std::min(mx0, i);
                    mx1 = std::max(mx1, i + 1);
                }
            }
    h->nmag = (int)cells.size();
    if (h->nmag == 0) { mx0 = 0; mx1 = 0; }
    g.mx0 = mx0;
    g.mx1 = mx1;
    h->mplanes = mx1 - mx0;

    int rc = MPB_OK;
    auto chk = [&](int r) { if (r && !rc) rc = r; };
    for (int p = 0; p < 2; ++p)
        for (int c = 0; c < 3; ++c) {
            chk(dev_alloc(h, &h->E[p][c], (size_t)h->nentries));
            chk(dev_alloc(h, &h->H[p][c], (size_t)h->nentries));
            chk(dev_alloc(h, &h->M[p][c], (size_t)(h->mplanes * g.PP)));
        }
    chk(dev_alloc(h, &h->ids, (size_t)h->nentries));
    chk(dev_alloc(h, &h->mats, (size_t)MPB_MAX_MATERIALS));
    chk(dev_alloc(h, &h->magcells, (size_t)h->nmag));
    chk(dev_alloc(h, &h->scratch, (size_t)h->nmag * 12));
    chk(dev_alloc(h, &h->st, 1));
    if (rc) { mpb_destroy(h); return rc; }
    CU(cudaMemcpy(h->ids, ids.data(), ids.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->mats, table.data(), sizeof(mpb_material) * table.size(),
                  cudaMemcpyHostToDevice));
    if (h->nmag)
        CU(cudaMemcpy(h->magcells, cells.data(), sizeof(int2) * cells.size(),
                      cudaMemcpyHostToDevice));

    // cooperative fixup grid: co-resident blocks only
    if (h->nmag) {
        int per_sm = 0, sms = 0;
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_llg_fixup, 256, 0));
        CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
        const int need = (h->nmag + 255) / 256;
        h->fixup_blocks = std::max(1, std::min(need, per_sm * sms));
    }
    if (h->variant != 1) {
        rc = prepare_fused(h, g);
        if (rc) { mpb_destroy(h); return rc; }
    }

    // source (em.py:276-282)
    for (int a = 0; a < 3; ++a) {
        if (su->src_loc[a] < 0 || su->src_loc[a] >= g.F[a]) {
            mpb_destroy(h);
            return fail_msg(MPB_EINVAL, "source location out of range");
        }
        h->src.pol[a] = su->src_pol[a];
    }
    h->src.off = su->src_loc[0] * g.PP + (int64_t)su->src_loc[1] * F[2] + su->src_loc[2];

    // probes
    h->nprobes = su->n_probes;
    h->probe_comp.assign(su->probe_comp, su->probe_comp + su->n_probes);
    h->probe_loc.assign(su->probe_loc, su->probe_loc + 3 * su->n_probes);
    for (int p = 0; p < h->nprobes; ++p) {
        const int comp = h->probe_comp[p];
        const int* L = &h->probe_loc[3 * p];
        const int* lim = comp >= MPB_COMP_MX ? g.n : g.F;
        if (comp < 0 || comp > 8) { mpb_destroy(h); return fail_msg(MPB_EINVAL, "bad probe component"); }
        for (int a = 0; a < 3; ++a)
            if (L[a] < 0 || L[a] >= lim[a]) {
                mpb_destroy(h);
                return fail_msg(MPB_EINVAL, "probe %d outside grid", p);
            }
    }
    chk(dev_alloc(h, &h->probes, (size_t)std::max(1, h->nprobes)));
    h->hostM.assign((size_t)3 * nx * ny * nz, 0.0);
    if (rc) { mpb_destroy(h); return rc; }
    rc = reset_state(h);
    if (rc) { mpb_destroy(h); return rc; }
    // probe table is (re)built by load_state; build it once for the zero state
    const double* zf[6];
    std::vector<double> zeros;
    (void)zf; (void)zeros;
    CU(cudaStreamSynchronize(h->stream));
    *out = h;
    return MPB_OK;
}

void mpb_destroy(mpb_handle* h) {
    if (!h) return;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    for (auto& e : h->events) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
    for (int p = 0; p < 2; ++p) {
        if (h->graph[p]) cudaGraphExecDestroy(h->graph[p]);
        for (int c = 0; c < 3; ++c) {
            cudaFree(h->E[p][c]);
            cudaFree(h->H[p][c]);
            cudaFree(h->M[p][c]);
        }
    }
    cudaFree(h->ids);
    cudaFree(h->mats);
    cudaFree(h->magcells);
    cudaFree(h->scratch);
    cudaFree(h->st);
    cudaFree(h->probes);
    cudaFree(h->d_src);
    cudaFree(h->d_probe);
    cudaFree(h->d_iters);
    destroy_fused(h);
    if (h->stream) cudaStreamDestroy(h->stream);
    delete h;
}

static int upload_probes(mpb_handle* h) {
    const Geom& g = h->g;
    std::vector<ProbeDesc> pd((size_t)std::max(1, h->nprobes));
    const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
    for (int p = 0; p < h->nprobes; ++p) {
        const int comp = h->probe_comp[p];
        const int* L = &h->probe_loc[3 * p];
        const int64_t f = (int64_t)L[1] * g.F[2] + L[2];
        ProbeDesc d{};
        if (comp < MPB_COMP_HX) {
            d.ptr0 = h->E[0][comp]; d.ptr1 = h->E[1][comp];
            d.off = L[0] * g.PP + f;
        } else if (comp < MPB_COMP_MX) {
            d.ptr0 = h->H[0][comp - 3]; d.ptr1 = h->H[1][comp - 3];
            d.off = L[0] * g.PP + f;
        } else if (L[0] >= g.mx0 && L[0] < g.mx1) {
            d.ptr0 = h->M[0][comp - 6]; d.ptr1 = h->M[1][comp - 6];
            d.off = (int64_t)(L[0] - g.mx0) * g.PP + f;
        } else {
            d.ptr0 = d.ptr1 = nullptr;
            d.constant = h->hostM[(((size_t)(comp - 6) * nx + L[0]) * ny + L[1]) * nz + L[2]];
        }
        pd[(size_t)p] = d;
    }
    CU(cudaMemcpy(h->probes, pd.data(), sizeof(ProbeDesc) * pd.size(),
                  cudaMemcpyHostToDevice));
    return MPB_OK;
}

int mpb_load_state(mpb_handle* h, const double* const fields[6], const double* m) {
    g_err.clear();
    if (!h || !fields || !m) return fail_msg(MPB_EINVAL, "null argument");
    const Geom& g = h->g;
    CU(cudaSetDevice(h->device));
    CU(cudaStreamSynchronize(h->stream));
    const size_t row = (size_t)g.FyFz * sizeof(double);
    for (int p = 0; p < 2; ++p)
        for (int c = 0; c < 6; ++c) {
            double* dst = c < 3 ? h->E[p][c] : h->H[p][c - 3];
            CU(cudaMemcpy2D(dst, g.PP * sizeof(double), fields[c], row, row, h->Fx,
                            cudaMemcpyHostToDevice));
        }
    const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
    memcpy(h->hostM.data(), m, h->hostM.size() * sizeof(double));
    if (h->mplanes) {
        std::vector<double> pk((size_t)(h->mplanes * g.PP), 0.0);
        for (int c = 0; c < 3; ++c) {
            for (int i = g.mx0; i < g.mx1; ++i)
                for (int j = 0; j < ny; ++j)
                    for (int k = 0; k < nz; ++k)
                        pk[(size_t)((i - g.mx0) * g.PP + (int64_t)j * g.F[2] + k)] =
                            m[(((size_t)c * nx + i) * ny + j) * nz + k];
            for (int p = 0; p < 2; ++p)
                CU(cudaMemcpy(h->M[p][c], pk.data(), pk.size() * sizeof(double),
                              cudaMemcpyHostToDevice));
        }
    }
    h->parity = 0;
    int rc = upload_probes(h);
    if (rc) return rc;
    rc = reset_state(h);
    if (rc) return rc;
    CU(cudaStreamSynchronize(h->stream));
    return MPB_OK;
}

int mpb_save_state(mpb_handle* h, double* const fields[6], double* m) {
    g_err.clear();
    if (!h || !fields || !m) return fail_msg(MPB_EINVAL, "null argument");
    const Geom& g = h->g;
    CU(cudaSetDevice(h->device));
    CU(cudaStreamSynchronize(h->stream));
    const size_t row = (size_t)g.FyFz * sizeof(double);
    const int p = h->parity;
    for (int c = 0; c < 6; ++c) {
        const double* src = c < 3 ? h->E[p][c] : h->H[p][c - 3];
        CU(cudaMemcpy2D(fields[c], row, src, g.PP * sizeof(double), row, h->Fx,
                        cudaMemcpyDeviceToHost));
    }
    const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
    memcpy(m, h->hostM.data(), h->hostM.size() * sizeof(double));
    if (h->mplanes) {
        std::vector<double> pk((size_t)(h->mplanes * g.PP));
        for (int c = 0; c < 3; ++c) {
            CU(cudaMemcpy(pk.data(), h->M[p][c], pk.size() * sizeof(double),
                          cudaMemcpyDeviceToHost));
            for (int i = g.mx0; i < g.mx1; ++i)
                for (int j = 0; j < ny; ++j)
                    for (int k = 0; k < nz; ++k)
                        m[(((size_t)c * nx + i) * ny + j) * nz + k] =
                            pk[(size_t)((i - g.mx0) * g.PP + (int64_t)j * g.F[2] + k)];
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

int mpb_run(mpb_handle* h, int64_t n0, int64_t nsteps, const double* src_vals,
            double* probe_out, int32_t* iters_out, mpb_failure* fail) {
    g_err.clear();
    if (fail) { fail->step = -1; fail->residual = 0; fail->iterations = 0; fail->kind = 0; }
    if (!h || nsteps < 0 || (nsteps && !src_vals))
        return fail_msg(MPB_EINVAL, "bad arguments");
    CU(cudaSetDevice(h->device));
    const int64_t cap = std::min<int64_t>(std::max<int64_t>(nsteps, 1), kRunChunk);
    if (cap > h->stage_cap) {
        cudaFree(h->d_src); cudaFree(h->d_probe); cudaFree(h->d_iters);
        h->d_src = nullptr; h->d_probe = nullptr; h->d_iters = nullptr;
        CU(cudaMalloc(&h->d_src, cap * sizeof(double)));
        CU(cudaMalloc(&h->d_probe, cap * std::max(1, h->nprobes) * sizeof(double)));
        CU(cudaMalloc(&h->d_iters, cap * sizeof(int)));
        h->stage_cap = cap;
    }
    int64_t launches = 0;
    for (int64_t s0 = 0; s0 < nsteps; s0 += cap) {
        const int64_t cnt = std::min(cap, nsteps - s0);
        CU(cudaMemcpyAsync(h->d_src, src_vals + s0, cnt * sizeof(double),
                           cudaMemcpyHostToDevice, h->stream));
        h->launches_last = 0;
        int rc = set_run_buffers(h, n0 + s0, h->d_src, h->d_probe, h->d_iters);
        if (!rc) rc = enqueue_steps(h, cnt);
        if (rc) return rc;
        launches += h->launches_last;
        if (h->nprobes && probe_out)
            CU(cudaMemcpyAsync(probe_out + s0 * h->nprobes, h->d_probe,
                               cnt * h->nprobes * sizeof(double), cudaMemcpyDeviceToHost,
                               h->stream));
        if (iters_out)
            CU(cudaMemcpyAsync(iters_out + s0, h->d_iters, cnt * sizeof(int),
                               cudaMemcpyDeviceToHost, h->stream));
        mpb_failure fl;
        rc = read_failure(h, &fl);
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
    unsigned long long m = 0;
    double bad = 0;
    CU(cudaMemcpy(&m, dm, sizeof m, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(&bad, db, sizeof bad, cudaMemcpyDeviceToHost));
    cudaFree(dx); cudaFree(dm); cudaFree(db);
    *mismatches = (int64_t)m;
    if (first_bad) *first_bad = bad;
    return MPB_OK;
}

int64_t mpb_launch_count(mpb_handle* h) { return h ? h->launches_last : 0; }

int64_t mpb_device_bytes(mpb_handle* h) { return h ? h->bytes : 0; }

}  // extern "C"

#include "mpb_fused.cuh"
