// mpb_fused.cuh -- host side of the fused sweep (included by mpb_api.cu after
// the handle definition).
#pragma once
#include <set>

namespace {

struct FusedState {
    SweepCfg sc{};
    int V = 2;
    int NT = kSweepThreads;
    bool F3 = true;
    bool pmc = true;          // some face is PMC (two-CTA form: else the PMC-free build)
    int grid = 0;
    size_t smem = 0;
    int2* defer = nullptr;
    int ndefer = 0;
    int3* zlines = nullptr;
    int nzlines = 0;
};

FusedState* fused_of(mpb_handle* h) { return reinterpret_cast<FusedState*>(h->fused); }

template <int V, bool F3, int NT = kSweepThreads, typename T = double, bool PMC = true>
int set_smem_attr(size_t smem) {
    CU(cudaFuncSetAttribute(k_sweep<V, F3, NT, T, PMC>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    return MPB_OK;
}

int prepare_fused(mpb_handle* h, const Geom& g) {
    auto* fs = new FusedState();
    h->fused = fs;
    SweepCfg& sc = fs->sc;
    const int Fz = g.F[2];
    int sms = 0, smem_optin = 0;
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
    CU(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin,
                              h->device));
    sc.hl = g.act[1] ? Fz : (g.act[2] ? 1 : 0);
    sc.eh = sc.hl;
    sc.nmat = h->nmat_table;
    if ((uint64_t)g.FyFz * (uint64_t)Fz >= (1ull << 32))
        return fail_msg(MPB_EINVAL, "x-plane too large for the fused sweep (%d entries)",
                        g.FyFz);
    sc.fz_magic = (uint32_t)(((1ull << 32) + Fz - 1) / Fz);
    if (Fz == 1) sc.fz_magic = 0;   // j = f for Fz == 1 handled below
    // staging ring bytes for a tile of T entries: 3 slots of E (T + both halo
    // rows), H^n (T + low halo) and material ids.  Field elements are esz
    // bytes (8, or 4 in the fp32 storage mode); every staged run starts on a
    // 16-byte boundary, i.e. a multiple of A entries.
    const int esz = (int)h->esz;
    const int A = 16 / esz;
    // a staged run [a0, a1) spans at most its entries + 2(A-1): 2A of slack
    auto cap_of = [&](int n) { return (n + 2 * A + A - 1) & ~(A - 1); };
    auto ring_bytes = [&](int T) {
        const int ecap = cap_of(T + sc.hl + sc.eh);
        const int hcap = cap_of(T + sc.hl);
        const int icap = T + sc.hl + 48;
        return (size_t)kSlots * (((3 * ecap + 3 * hcap) * esz + icap + 127) / 128 * 128);
    };
    // Tile form, first that fits (V entries per thread, NT threads per CTA):
    //  * 3D planes of >= 8K entries: V=2, NT=256, two CTAs per SM (each one's
    //    barrier waits overlap the other's work) when two rings fit in the
    //    SM's shared memory -- z-rows up to ~140 entries (C2, C3, C4);
    //  * large planes with longer rows: V=2, NT=512, one CTA per SM with a
    //    1024-entry tile (C5: 2049x257 planes);
    //  * otherwise (small / 1D / 2D planes): V=1, NT=512.
    // MPB_SWEEP_V / MPB_SWEEP_NT=512 override (experiments and tests).
    int smem_sm = 0, reserved = 0;
    CU(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, h->device));
    CU(cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, h->device));
    cudaFuncAttributes fa{};
    if (h->f32) { CU(cudaFuncGetAttributes(&fa, k_sweep<2, true, 256, float>)); }
    else        { CU(cudaFuncGetAttributes(&fa, k_sweep<2, true, 256>)); }
    const size_t fixed = fa.sharedSizeBytes + (size_t)reserved;
    const bool f3 = g.act[0] && g.act[1] && g.act[2];
    if (f3 && g.FyFz >= 8 * 512 && 2 * (ring_bytes(512) + fixed) <= (size_t)smem_sm) {
        fs->V = 2; fs->NT = 256;
    } else if (g.FyFz >= 2 * kSweepThreads * 64 &&
               ring_bytes(1024) + fixed <= (size_t)smem_optin) {
        fs->V = 2; fs->NT = kSweepThreads;
    } else {
        fs->V = 1; fs->NT = kSweepThreads;
    }
    bool any_pmc = false;
    for (int f = 0; f < 6; ++f) any_pmc = any_pmc || g.faces[f] == MPB_FACE_PMC;
    // fp32 with long z-rows (the halo row > a third of a 512-entry tile,
    // C5's 257): 1024-entry tiles in the two-CTA form (C5 +2.4%; on C4's
    // 129-entry rows the 512-entry tiles at three CTAs/SM win by 17%)
    if (h->f32 && fs->NT == 256 && !any_pmc && 3 * sc.hl > 512 &&
        2 * (ring_bytes(1024) + fixed) <= (size_t)smem_sm)
        fs->V = 4;
    if (const char* e = getenv("MPB_SWEEP_V")) {
        const int v = atoi(e);
        if (v == 4 && h->f32 && fs->NT == 256 && !any_pmc &&
            2 * (ring_bytes(1024) + fixed) <= (size_t)smem_sm) {
            fs->V = 4;   // fp32: 1024-entry tiles in the two-CTA form
        } else if (v == 1 || v == 2) {
            fs->V = v;
            if (fs->V != 2) fs->NT = kSweepThreads;
        }
    }
    if (const char* e = getenv("MPB_SWEEP_NT"))
        if (atoi(e) == 512) fs->NT = kSweepThreads;
    // x-chunks: for a tile count, the chunk count that maximises (CTA slots
    // kept busy over the whole grid of waves) x (useful planes / (planes + ~3
    // of halo plane and pipeline fill)) -- whole waves and long chunks (C4: 8
    // chunks = 7.0 waves, +2% over a fixed 32-wave split; C2 +7%, C3 +3%, C5 +3%)
    const int Fx = g.c1 - g.c0;                      // owned planes of this rank
    // fp32 two-CTA form: three CTAs per SM when three rings fit (71
    // registers; MPB_SWEEP_CTAS=2 keeps two)
    int per_sm = fs->NT == 256 ? 2 : 1;
    if (fs->NT == 256 && h->f32) {
        int want = MPB_F32_CTAS;
        if (const char* e = getenv("MPB_SWEEP_CTAS")) want = std::max(2, std::min(4, atoi(e)));
        while (want > 2 && (size_t)want * (ring_bytes(fs->V * 256) + fixed) > (size_t)smem_sm)
            --want;
        per_sm = want;
    }
    const double slots = (double)per_sm * sms;
    // x-chunks of at least 2 planes (C1: 64 planes of 9 tiles need 32 chunks
    // to fill the 296 CTA slots; the larger grids' choice is unchanged)
    int minch = 2;
    if (const char* e = getenv("MPB_SWEEP_MINCHUNK")) minch = std::max(2, atoi(e));
    const int maxch = std::max(1, Fx / minch);
    auto chunks_for = [&](int tiles, double* waves_out) {
        double best = -1.0;
        int pick = 1;
        for (int n = 1; n <= maxch; ++n) {
            const int len = (Fx + n - 1) / n;
            const int used = (Fx + len - 1) / len;              // chunks actually made
            const double ctas = (double)tiles * used;
            // slabs with an overlapped exchange launch the interior chunks and
            // the two edge chunks separately: count both launches' waves
            const bool split = h->nranks > 1 && h->overlap && used > 2;
            const double waves =
                split ? std::ceil(tiles * (used - 2.0) / slots) + std::ceil(tiles * 2.0 / slots)
                      : std::ceil(ctas / slots);
            const double eff = ctas / (waves * slots) * ((double)len / (len + 3.0));
            if (eff > best + 1e-9) { best = eff; pick = used; *waves_out = waves; }
        }
        return pick;
    };
    // tile size: the full V x NT tile, unless a smaller even tile lets the
    // tiles x chunks grid fill its last wave with >2% less modelled time.
    // Model: waves x (chunk planes + 3) x (per-plane latency + T), the latency
    // worth ~1400 entries of streaming (fitted to A/B runs: a CTA's time per
    // plane is mostly the wait for its staged plane, little of it scales with
    // T).  Planes of ~17K entries (C2, C3) leave a tenth of the wave idle with
    // 512-entry tiles; 452/458-entry tiles fill it (+3% measured).  C4 and C5
    // keep the full tile.
    const int Tmax = fs->V * fs->NT;
    auto model = [&](int T, int* nch) {
        double waves = 1.0;
        *nch = chunks_for((g.FyFz + T - 1) / T, &waves);
        return waves * (1400.0 + T) * (((Fx + *nch - 1) / *nch) + 3.0);
    };
    sc.T = Tmax;
    if (const char* e = getenv("MPB_SWEEP_T")) {   // multiple of A: 16-byte aligned tile starts
        const int t = atoi(e) & ~(A - 1);
        if (t > 0 && t <= sc.T) sc.T = t;
    } else {
        int nch = 1;
        const double full = model(Tmax, &nch);
        double best = full;
        int bestT = Tmax;
        for (int T = Tmax - A; T >= Tmax / 2; T -= A) {
            const double t = model(T, &nch);
            if (t < best - 1e-9) { best = t; bestT = T; }
        }
        if (best < full / 1.02) sc.T = bestT;
    }
    sc.tiles = (g.FyFz + sc.T - 1) / sc.T;
    {
        bool fastdiv = true;
        for (int a = 0; a < 3; ++a)
            if (g.act[a] && !(g.d[a] >= 0x1p-40 && g.d[a] <= 0x1p10)) fastdiv = false;
        sc.fastdiv = fastdiv ? 1 : 0;
    }
    sc.ecap = cap_of(sc.T + sc.hl + sc.eh);
    sc.hcap = cap_of(sc.T + sc.hl);
    sc.icap = sc.T + sc.hl + 48;
    sc.stage_bytes = ((3 * sc.ecap + 3 * sc.hcap) * esz + sc.icap + 127) / 128 * 128;
    fs->smem = (size_t)kSlots * sc.stage_bytes;

    const size_t static_smem = 8 * 1024;
    if (fs->smem + static_smem > (size_t)smem_optin)
        return fail_msg(MPB_EINVAL, "fused sweep staging (%zu B) exceeds shared memory",
                        fs->smem);
    {
        double waves = 1.0;
        sc.nchunks = chunks_for(sc.tiles, &waves);
    }
    if (const char* e = getenv("MPB_SWEEP_WAVES")) {        // the earlier fixed-wave rule
        const int want = std::max(1, (std::max(1, atoi(e)) * sms + sc.tiles - 1) / sc.tiles);
        sc.nchunks = std::max(1, std::min(want, maxch));
    }
    if (const char* e = getenv("MPB_SWEEP_CHUNKS")) sc.nchunks = std::max(1, atoi(e));
    sc.chunk = (Fx + sc.nchunks - 1) / sc.nchunks;
    sc.nchunks = (Fx + sc.chunk - 1) / sc.chunk;
    sc.ch_base = 0;
    sc.ch_step = 1;
    fs->grid = sc.tiles * sc.nchunks;
    fs->F3 = g.act[0] && g.act[1] && g.act[2];
    for (int f = 0; f < 6; ++f) fs->pmc = f == 0 ? g.faces[f] == MPB_FACE_PMC
                                                  : (fs->pmc || g.faces[f] == MPB_FACE_PMC);
    if (const char* e = getenv("MPB_SWEEP_PMC"))   // 1: the generic build (A/B, tests)
        if (atoi(e) == 1) fs->pmc = true;
    int rc;
    if (h->f32) {
        if (fs->NT == 256 && fs->V == 4)
            rc = set_smem_attr<4, true, 256, float, false>(fs->smem);
        else if (fs->NT == 256)
            rc = fs->pmc ? set_smem_attr<2, true, 256, float>(fs->smem)
                         : set_smem_attr<2, true, 256, float, false>(fs->smem);
        else if (fs->F3 && fs->V == 2 && !fs->pmc)
            rc = set_smem_attr<2, true, kSweepThreads, float, false>(fs->smem);
        else if (fs->F3)
            rc = fs->V == 2 ? set_smem_attr<2, true, kSweepThreads, float>(fs->smem)
                            : set_smem_attr<1, true, kSweepThreads, float>(fs->smem);
        else
            rc = fs->V == 2 ? set_smem_attr<2, false, kSweepThreads, float>(fs->smem)
                            : set_smem_attr<1, false, kSweepThreads, float>(fs->smem);
    } else if (fs->NT == 256) {
        rc = fs->pmc ? set_smem_attr<2, true, 256>(fs->smem)
                     : set_smem_attr<2, true, 256, double, false>(fs->smem);
    } else if (fs->F3 && fs->V == 2 && !fs->pmc) {   // PMC-free one-CTA form (C5)
        rc = set_smem_attr<2, true, kSweepThreads, double, false>(fs->smem);
    } else if (fs->F3) {
        rc = fs->V == 2 ? set_smem_attr<2, true>(fs->smem) : set_smem_attr<1, true>(fs->smem);
    } else {
        rc = fs->V == 2 ? set_smem_attr<2, false>(fs->smem) : set_smem_attr<1, false>(fs->smem);
    }
    if (rc) return rc;
    {   // reciprocals of the spacings, computed once on the device
        for (int a = 0; a < 3; ++a) {
            sc.rd[a] = g.rd[a];                        // set in mpb_create
            sc.rdf[a] = (float)(1.0 / g.d[a]);         // fp32 storage mode
        }
        sc.coef_hf = (float)g.coef_h;
    }
    if (rc) return rc;
    sc.eguard = g.eguard;
    // LLG-first order: entry range of the magnetic cells within a plane
    sc.mpre = h->pre ? 1 : 0;
    sc.mf0 = 0;
    sc.mf1 = -1;
    if (h->pre) {
        std::vector<int2> cells((size_t)h->nmag);
        CU(cudaMemcpy(cells.data(), h->magcells, sizeof(int2) * cells.size(),
                      cudaMemcpyDeviceToHost));
        sc.mf0 = g.FyFz;
        for (const int2& c : cells) { sc.mf0 = std::min(sc.mf0, c.y); sc.mf1 = std::max(sc.mf1, c.y); }
    }
    // deferred E entries: {c, c+x, c+y, c+z} over magnetic cells
    std::vector<int64_t> keys;
    if (h->nmag && !h->pre) {
        std::vector<int2> cells((size_t)h->nmag);
        CU(cudaMemcpy(cells.data(), h->magcells, sizeof(int2) * cells.size(),
                      cudaMemcpyDeviceToHost));
        keys.reserve(cells.size() * 4);
        auto add = [&](int i, int64_t f) {
            if (i >= g.c0 && i < g.c1) keys.push_back((int64_t)i * g.FyFz + f);
        };
        for (const int2& c : cells) {
            const int i = c.x, f = c.y;
            const int j = f / Fz, k = f - j * Fz;
            add(i, f);
            if (g.act[0] && i + 1 < g.F[0]) add(i + 1, f);
            if (g.act[1] && j + 1 < g.F[1]) add(i, f + Fz);
            if (g.act[2] && k + 1 < g.F[2]) add(i, f + 1);
        }
        std::sort(keys.begin(), keys.end());
        keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
        std::vector<int2> list(keys.size());
        for (size_t q = 0; q < keys.size(); ++q)
            list[q] = make_int2((int)(keys[q] / g.FyFz), (int)(keys[q] % g.FyFz));
        fs->ndefer = (int)list.size();
        CU(cudaMallocAsync(&fs->defer, sizeof(int2) * list.size(), h->stream));
        CU(cudaStreamSynchronize(h->stream));
        h->bytes += (int64_t)(sizeof(int2) * list.size());
        CU(cudaMemcpy(fs->defer, list.data(), sizeof(int2) * list.size(),
                      cudaMemcpyHostToDevice));
    }
    // z-wall lines deferred to k_zfix (see mpb_sweep.cuh)
    if (g.zin && g.act[2] && (g.faces[4] != MPB_FACE_PMC || g.faces[5] != MPB_FACE_PMC)) {
        std::set<int> jset, iset;
        if (g.act[1]) for (int j : {0, 1, g.n[1] - 1, g.n[1]}) jset.insert(j);
        if (g.act[0])
            for (int i : {0, 1, g.n[0] - 1, g.n[0]})
                if (i >= g.c0 && i < g.c1) iset.insert(i);
        std::vector<int3> lines;
        for (int j : jset)
            for (int i = g.c0; i < g.c1; ++i) lines.push_back(make_int3(0, i, j));
        for (int i : iset)
            for (int j = 0; j < g.F[1]; ++j) lines.push_back(make_int3(1, i, j));
        fs->nzlines = (int)lines.size();
        if (fs->nzlines) {
            CU(cudaMallocAsync(&fs->zlines, sizeof(int3) * lines.size(), h->stream));
            CU(cudaStreamSynchronize(h->stream));
            h->bytes += (int64_t)(sizeof(int3) * lines.size());
            CU(cudaMemcpy(fs->zlines, lines.data(), sizeof(int3) * lines.size(),
                          cudaMemcpyHostToDevice));
        }
    }
    return MPB_OK;
}

template <typename T>
int launch_zfix(mpb_handle* h, const Geom& g, const BufsT<T>& b, cudaStream_t s) {
    FusedState* fs = fused_of(h);
    if (!fs->nzlines) return MPB_OK;
    CU(launch_pdl(h->pdl, k_zfix<T>, dim3((fs->nzlines + 255) / 256), dim3(256), s, g, b,
                  (const mpb_material*)h->mats, ids_view(h), (const int3*)fs->zlines,
                  fs->nzlines, h->st));
    return MPB_OK;
}

int zfix_launches(mpb_handle* h) { return fused_of(h)->nzlines ? 1 : 0; }

// LLG of the magnetic cells after the pure-Maxwell sweep (fused variant).
template <typename T>
int launch_llg_local(mpb_handle* h, const Geom& g, const BufsT<T>& b, cudaStream_t s) {
    if (!h->nmag) return MPB_OK;
    const size_t smem = (size_t)(g.max_iters + 2) * sizeof(unsigned long long);
    CU(launch_pdl_smem(h->pdl, k_llg_local<T>, dim3((h->nmag + 255) / 256), dim3(256), smem, s,
                       g, b, (const mpb_material*)h->mats, ids_view(h),
                       (const int2*)h->magcells, (const unsigned char*)h->magowned, h->nmag,
                       h->st));
    return MPB_OK;
}

// LLG-first order: the magnetic cells' local LLG before the sweep.
template <typename T>
int launch_llg_pre(mpb_handle* h, int pa, cudaStream_t s) {
    const Geom& g = h->g;
    const size_t smem = (size_t)(g.max_iters + 2) * sizeof(unsigned long long);
    CU(launch_pdl_smem(h->pdl, k_llg_pre<T>, dim3((h->nmag + 255) / 256), dim3(256), smem, s,
                       g, make_bufs<T>(h, pa), (const mpb_material*)h->mats,
                       make_magpre<T>(h, pa), (const int2*)h->magcells, h->nmag, h->st));
    return MPB_OK;
}

template <typename T>
int launch_llg_pre_coop(mpb_handle* h, int pa, cudaStream_t s) {
    const Geom& g = h->g;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(h->coop_blocks);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = (size_t)(g.max_iters + 2) * sizeof(unsigned long long);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CU(cudaLaunchKernelEx(&cfg, k_llg_pre_coop<T>, g, make_bufs<T>(h, pa),
                          (const mpb_material*)h->mats, make_magpre<T>(h, pa), ids_view(h),
                          (const int2*)h->magcells, h->nmag, MagScratch{h->scratch}, h->st));
    return MPB_OK;
}

// compact step-n copy of the magnetic cells from the lattice of parity pa
template <typename T>
int pack_magnetic(mpb_handle* h, int pa) {
    if (!h->pre || !h->nmag) return MPB_OK;
    k_mag_pack<T><<<(h->nmag + 255) / 256, 256, 0, h->stream>>>(
        h->g, make_bufs<T>(h, pa), make_magpre<T>(h, pa), (const int2*)h->magcells, h->nmag);
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(h->stream));
    return MPB_OK;
}

// lattice M of the magnetic cells (current parity) from the compact copy
int unpack_magnetic(mpb_handle* h) {
    if (!h->pre || !h->nmag) return MPB_OK;
    const int p = h->parity;
    const dim3 grid((h->nmag + 255) / 256);
    if (h->f32)
        k_mag_unpack<float><<<grid, 256, 0, h->stream>>>(
            h->g, h->M[p][0], h->M[p][1], h->M[p][2], make_magpre<float>(h, p),
            (const int2*)h->magcells, h->nmag);
    else
        k_mag_unpack<double><<<grid, 256, 0, h->stream>>>(
            h->g, h->M[p][0], h->M[p][1], h->M[p][2], make_magpre<double>(h, p),
            (const int2*)h->magcells, h->nmag);
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(h->stream));
    return MPB_OK;
}

void destroy_fused(mpb_handle* h) {
    FusedState* fs = fused_of(h);
    if (!fs) return;
    if (fs->defer) cudaFreeAsync(fs->defer, h->stream);
    if (fs->zlines) cudaFreeAsync(fs->zlines, h->stream);
    delete fs;
    h->fused = nullptr;
}

// part 0: every x-chunk; 1: the interior chunks (no ghost plane read or
// written); 2: the first and last chunk (the only ones touching the ghost
// planes a slab exchange fills).  Adds the launches made to `launches`.
template <typename T>
int launch_fused(mpb_handle* h, const Geom& g, const BufsT<T>& b, cudaStream_t s, int part,
                 int64_t& launches) {
    FusedState* fs = fused_of(h);
    SweepCfg sc = fs->sc;
    int grid = fs->grid;
    if (part == 1) {
        if (sc.nchunks <= 2) return MPB_OK;
        sc.ch_base = 1;
        grid = sc.tiles * (sc.nchunks - 2);
    } else if (part == 2) {
        sc.ch_step = std::max(1, sc.nchunks - 1);
        grid = sc.tiles * std::min(2, sc.nchunks);
    }
    ++launches;
#define MPB_LAUNCH(VV, FF)                                                              \
    CU(launch_pdl_smem(h->pdl, k_sweep<VV, FF, kSweepThreads, T>, dim3(grid),              \
                       dim3(kSweepThreads), fs->smem, s, g, b, (const mpb_material*)h->mats,  \
                       ids_view(h), h->st, sc))
    if (fs->NT == 256 && fs->V == 4) {
        if constexpr (sizeof(T) == 4)   // fp32, PMC-free only (prepare_fused)
            CU(launch_pdl_smem(h->pdl, k_sweep<4, true, 256, T, false>, dim3(grid), dim3(256),
                               fs->smem, s, g, b, (const mpb_material*)h->mats, ids_view(h),
                               h->st, sc));
    } else if (fs->NT == 256 && !fs->pmc) {
        CU(launch_pdl_smem(h->pdl, k_sweep<2, true, 256, T, false>, dim3(grid), dim3(256),
                           fs->smem, s, g, b, (const mpb_material*)h->mats, ids_view(h), h->st,
                           sc));
    } else if (fs->NT == 256) {
        CU(launch_pdl_smem(h->pdl, k_sweep<2, true, 256, T>, dim3(grid), dim3(256), fs->smem,
                           s, g, b, (const mpb_material*)h->mats, ids_view(h), h->st, sc));
    } else if (fs->F3 && fs->V == 2 && !fs->pmc) {
        CU(launch_pdl_smem(h->pdl, k_sweep<2, true, kSweepThreads, T, false>, dim3(grid),
                           dim3(kSweepThreads), fs->smem, s, g, b, (const mpb_material*)h->mats,
                           ids_view(h), h->st, sc));
    } else if (fs->F3) {
        if (fs->V == 2) MPB_LAUNCH(2, true);
        else MPB_LAUNCH(1, true);
    } else {
        if (fs->V == 2) MPB_LAUNCH(2, false);
        else MPB_LAUNCH(1, false);
    }
#undef MPB_LAUNCH
    return MPB_OK;
}

template <typename T>
int launch_deferred(mpb_handle* h, const Geom& g, const BufsT<T>& b, cudaStream_t s) {
    FusedState* fs = fused_of(h);
    if (!fs->ndefer) return MPB_OK;
    CU(launch_pdl(h->pdl, k_edefer<T>, dim3((fs->ndefer + 255) / 256), dim3(256), s, g, b,
                  (const mpb_material*)h->mats, ids_view(h), (const int2*)fs->defer,
                  fs->ndefer, (const StepState*)h->st, 1));
    return MPB_OK;
}

const char* fused_kernel_name() { return "k_sweep"; }

// tile form of the fused sweep: {entries per thread V, CTA threads NT,
// entries per tile T, x-chunks}; zeros for the split variant / line kernel
void fused_form(mpb_handle* h, int32_t out[4]) {
    FusedState* fs = fused_of(h);
    out[0] = out[1] = out[2] = out[3] = 0;
    if (!fs || h->line) return;
    out[0] = fs->V; out[1] = fs->NT; out[2] = fs->sc.T; out[3] = fs->sc.nchunks;
}

}  // namespace
