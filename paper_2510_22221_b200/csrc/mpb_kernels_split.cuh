// mpb_kernels_split.cuh -- per-step kernels shared by both sweep variants
// (LLG fixup, walls, source+probes) and the split H / E sweeps.
#pragma once

#include <cooperative_groups.h>

#include "mpb_device.cuh"

namespace mpb {

namespace cg = cooperative_groups;

// ---------------------------------------------------------------------------
// Per-CTA LLG statistics: residual history and local stop range, reduced in
// shared memory and flushed with one global atomic per iterate per CTA.
// ---------------------------------------------------------------------------
struct CtaLlgStats {
    unsigned long long* hist;   // dynamic smem, max_iters + 2 entries
    int* rc;                    // [0] = min, [1] = max
};

__device__ __forceinline__ void cta_stats_init(CtaLlgStats& s, int max_iters) {
    for (int r = threadIdx.x; r <= max_iters + 1; r += blockDim.x) s.hist[r] = 0ull;
    if (threadIdx.x == 0) { s.rc[0] = 0x7fffffff; s.rc[1] = 0; }
}

__device__ __forceinline__ void cta_stats_flush(const CtaLlgStats& s, int max_iters,
                                                StepState* st) {
    for (int r = 1 + threadIdx.x; r <= max_iters; r += blockDim.x) {
        const unsigned long long v = s.hist[r];
        if (v) atomicMax(&st->hist[r], v);
    }
    if (threadIdx.x == 0) {
        atomicMax(&st->rc_negmin, -s.rc[0]);
        atomicMax(&st->rc_max, s.rc[1]);
    }
}

// Run one magnetic cell to its local stop: the first iterate whose own
// residual is <= tol, or max_iters.  Because cells couple only through the
// global stop test, the iterate sequence of a cell is the same as in the
// reference's lockstep loop; the global r* is settled afterwards
// (k_llg_fixup).  Returns the local stop index (max_iters+1 if none).
__device__ __forceinline__ int llg_local(LlgCell& s, const Geom& g, double Hr[3],
                                         double Mr[3], CtaLlgStats& cs) {
    Hr[0] = s.Hn[0]; Hr[1] = s.Hn[1]; Hr[2] = s.Hn[2];
    Mr[0] = s.Mn[0]; Mr[1] = s.Mn[1]; Mr[2] = s.Mn[2];
    for (int r = 1; r <= g.max_iters; ++r) {
        const double res = llg_iterate(s, g.coef_h, Hr, Mr);
        atomicMax(&cs.hist[r], dbits(res));
        if (res <= g.tol) return r;
    }
    return g.max_iters + 1;
}

// ---------------------------------------------------------------------------
// Split variant, kernel 1: H^{n+1} everywhere (em.py:171-182 plus the local
// part of llg.coupled_cell_step).  One thread per allocation entry (i, f).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_hsweep(Geom g, Bufs b,
                                                const mpb_material* __restrict__ mats,
                                                const uint8_t* __restrict__ ids,
                                                StepState* st) {
    extern __shared__ unsigned long long smem_hist[];
    __shared__ int smem_rc[2];
    if (st->fail) return;
    const int i = blockIdx.y;
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = f < g.FyFz;
    int j = 0, k = 0;
    if (live) { j = f / g.F[2]; k = f - j * g.F[2]; }
    const int64_t o = i * g.PP + f;
    const bool cellin = live && i < g.n[0] && j < g.n[1] && k < g.n[2];
    const bool magnetic = cellin && mats[ids[o]].magnetic;
    const int anymag = __syncthreads_or(magnetic);
    CtaLlgStats cs{smem_hist, smem_rc};
    if (anymag) { cta_stats_init(cs, g.max_iters); __syncthreads(); }
    if (live) {
        const bool vx = j < g.n[1] && k < g.n[2];
        const bool vy = i < g.n[0] && k < g.n[2];
        const bool vz = i < g.n[0] && j < g.n[1];
        const Curl3 c = curl_e_at(g, b.Ea, o, g.PP, g.F[2], vx, vy, vz);
        if (!magnetic) {
            if (vx) b.Hb[0][o] = b.Ha[0][o] - g.coef_h * c.x;
            if (vy) b.Hb[1][o] = b.Ha[1][o] - g.coef_h * c.y;
            if (vz) b.Hb[2][o] = b.Ha[2][o] - g.coef_h * c.z;
        } else {
            const mpb_material m = mats[ids[o]];
            const int64_t om = (int64_t)(i - g.mx0) * g.PP + f;
            LlgCell s;
            s.Hn[0] = b.Ha[0][o]; s.Hn[1] = b.Ha[1][o]; s.Hn[2] = b.Ha[2][o];
            s.Mn[0] = b.Ma[0][om]; s.Mn[1] = b.Ma[1][om]; s.Mn[2] = b.Ma[2][om];
            s.cE[0] = c.x; s.cE[1] = c.y; s.cE[2] = c.z;
            llg_setup(s, m);
            double Hr[3], Mr[3];
            const int rc = llg_local(s, g, Hr, Mr, cs);
            atomicMin(&cs.rc[0], rc);
            atomicMax(&cs.rc[1], rc);
            b.Hb[0][o] = Hr[0]; b.Hb[1][o] = Hr[1]; b.Hb[2][o] = Hr[2];
            b.Mb[0][om] = Mr[0]; b.Mb[1][om] = Mr[1]; b.Mb[2][om] = Mr[2];
        }
    }
    if (anymag) { __syncthreads(); cta_stats_flush(cs, g.max_iters, st); }
}

// ---------------------------------------------------------------------------
// Split variant, kernel 2: E^{n+1} = ca (curl H - cb E) on every allocation
// entry (em.py:206-232, 257-272).  Walls are applied afterwards.
// ---------------------------------------------------------------------------
struct E3 { double x, y, z; };

// Plain E^{n+1} at one entry (no walls), reading the new H from b.Hb.
template <typename T>
__device__ __forceinline__ E3 e_plain_at(const Geom& g, const BufsT<T>& b,
                                         const mpb_material* __restrict__ mats,
                                         const uint8_t* __restrict__ ids, int i, int j, int k,
                                         int64_t o) {
    T* const* H = b.Hb;
    double cx = 0.0, cy = 0.0, cz = 0.0;
    const int64_t sx = g.PP, sy = g.F[2];
    const bool p[6] = {g.faces[0] == MPB_FACE_PMC, g.faces[1] == MPB_FACE_PMC,
                       g.faces[2] == MPB_FACE_PMC, g.faces[3] == MPB_FACE_PMC,
                       g.faces[4] == MPB_FACE_PMC, g.faces[5] == MPB_FACE_PMC};
    // every load first (see curl_e_at); same differences in the same order
    const bool ay = g.act[1], az = g.act[2], ax = g.act[0];
    const double h0 = H[0][o], h1 = H[1][o], h2 = H[2][o];
    const double h2_y = ay ? bwd_lo_load(H[2], o, sy, j) : 0.0;
    const double h0_y = ay ? bwd_lo_load(H[0], o, sy, j) : 0.0;
    const double h1_z = az ? bwd_lo_load(H[1], o, 1, k) : 0.0;
    const double h0_z = az ? bwd_lo_load(H[0], o, 1, k) : 0.0;
    const double h2_x = ax ? bwd_lo_load(H[2], o, sx, i) : 0.0;
    const double h1_x = ax ? bwd_lo_load(H[1], o, sx, i) : 0.0;
    const double e0 = b.Ea[0][o], e1 = b.Ea[1][o], e2 = b.Ea[2][o];
    const uint8_t id = ids[o];
    const double ca = mats[id].ca, cb = mats[id].cb;
    if (ay) {   // cHx += dHz/dy ; cHz -= dHx/dy
        cx = cx + bwd_diff_v(h2, h2_y, j, g.n[1], g.d[1], g.rd[1], p[2], p[3]);
        cz = cz - bwd_diff_v(h0, h0_y, j, g.n[1], g.d[1], g.rd[1], p[2], p[3]);
    }
    if (az) {   // cHx -= dHy/dz ; cHy += dHx/dz
        cx = cx - bwd_diff_v(h1, h1_z, k, g.n[2], g.d[2], g.rd[2], p[4], p[5]);
        cy = cy + bwd_diff_v(h0, h0_z, k, g.n[2], g.d[2], g.rd[2], p[4], p[5]);
    }
    if (ax) {   // cHy -= dHz/dx ; cHz += dHy/dx
        cy = cy - bwd_diff_v(h2, h2_x, i, g.n[0], g.d[0], g.rd[0], p[0], p[1]);
        cz = cz + bwd_diff_v(h1, h1_x, i, g.n[0], g.d[0], g.rd[0], p[0], p[1]);
    }
    E3 r;
    r.x = ca * (cx - cb * e0);
    r.y = ca * (cy - cb * e1);
    r.z = ca * (cz - cb * e2);
    return r;
}

// E^{n+1} = ca (curl H - cb E) on one allocation entry (em.py:206-232,
// 257-272); walls are applied afterwards by k_wall.
__device__ __forceinline__ void e_update_at(const Geom& g, const Bufs& b,
                                            const mpb_material* __restrict__ mats,
                                            const uint8_t* __restrict__ ids, int i,
                                            int j, int k, int64_t o) {
    const E3 r = e_plain_at(g, b, mats, ids, i, j, k, o);
    b.Eb[0][o] = r.x;
    b.Eb[1][o] = r.y;
    b.Eb[2][o] = r.z;
}

__global__ void __launch_bounds__(256) k_esweep(Geom g, Bufs b,
                                                const mpb_material* __restrict__ mats,
                                                const uint8_t* __restrict__ ids,
                                                const StepState* st) {
    if (st->fail) return;
    const int i = blockIdx.y;
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= g.FyFz) return;
    const int j = f / g.F[2];
    const int k = f - j * g.F[2];
    e_update_at(g, b, mats, ids, i, j, k, i * g.PP + f);
}

// ---------------------------------------------------------------------------
// LLG fixup: settles r* for the step (llg.py:131-148).
//  * uniform case -- every magnetic cell stopped locally at the same iterate
//    R <= max_iters: the sweep's results are final; replay the stop/failure
//    rule on the complete residual history.
//  * otherwise: recompute all magnetic cells in lockstep exactly as the
//    reference does (one grid barrier per iterate) and overwrite H, M.
// Cooperative launch; every block takes the same branch.
// ---------------------------------------------------------------------------
struct MagScratch {    // per magnetic cell, structure of arrays
    double* v;         // 12 * nmag: Hn[3] Mn[3] cE[3] Mr[3]
};

// The fixup proper, run by every block of a cooperative grid (k_llg_fixup,
// and the merged tail k_post); returns in every block.
template <typename T>
__device__ void llg_fixup_grid(const Geom& g, const BufsT<T>& b,
                               const mpb_material* __restrict__ mats,
                               const uint8_t* __restrict__ ids, const int2* __restrict__ cells,
                               int nmag, MagScratch scr, StepState* st,
                               const MagPre<T>& mp) {
    __shared__ unsigned long long red[32];
    if (st->fail) return;
    const int rmin = -st->rc_negmin, rmax = st->rc_max;
    if (rmin == rmax && rmax <= g.max_iters) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            double fr; int fi, fk;
            const int r = llg_decide(st->hist, rmax, g.max_iters, g.tol, &fr, &fi, &fk);
            if (r > 0) {
                st->rstar = r;
            } else {   // r == -1 is impossible here: hist[rmax] <= tol
                st->fail = 1; st->fail_step = st->step; st->fail_res = fr;
                st->fail_it = fi; st->fail_kind = fk;
            }
        }
        return;
    }
    cg::grid_group grid = cg::this_grid();
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int nth = gridDim.x * blockDim.x;
    double* v = scr.v;
    // gather Hn, Mn, curl E (from the untouched read buffers)
    for (int q = tid; q < nmag; q += nth) {
        const int i = cells[q].x, f = cells[q].y;
        const int j = f / g.F[2], k = f - j * g.F[2];
        (void)k;
        const int64_t o = i * g.PP + f;
        const int64_t om = (int64_t)(i - g.mx0) * g.PP + f;
        const Curl3 c = curl_e_at(g, b.Ea, o, g.PP, g.F[2], true, true, true);
        double* w = v + (size_t)q * 12;
        if (mp.on) {   // LLG-first: the lattice H^n of the cell is overwritten
            for (int cc = 0; cc < 3; ++cc) { w[cc] = mp.Hn[cc][q]; w[3 + cc] = mp.Mn[cc][q]; }
        } else {
            w[0] = b.Ha[0][o]; w[1] = b.Ha[1][o]; w[2] = b.Ha[2][o];
            w[3] = b.Ma[0][om]; w[4] = b.Ma[1][om]; w[5] = b.Ma[2][om];
        }
        w[6] = c.x; w[7] = c.y; w[8] = c.z;
        w[9] = w[3]; w[10] = w[4]; w[11] = w[5];
    }
    double prev = __longlong_as_double(0x7ff0000000000000LL);
    int growth = 0, rstar = 0, failed = 0;
    double fres = 0.0; int fit = 0, fkind = 0;
    for (int r = 1; r <= g.max_iters; ++r) {
        unsigned long long lmax = 0ull;
        for (int q = tid; q < nmag; q += nth) {
            const int i = cells[q].x, f = cells[q].y;
            const int64_t o = i * g.PP + f;
            double* w = v + (size_t)q * 12;
            LlgCell s;
            for (int c = 0; c < 3; ++c) { s.Hn[c] = w[c]; s.Mn[c] = w[3 + c]; s.cE[c] = w[6 + c]; }
            llg_setup(s, mats[ids[o]]);
            double Mr[3] = {w[9], w[10], w[11]};
            double Hr[3];
            if (r == 1) { Hr[0] = s.Hn[0]; Hr[1] = s.Hn[1]; Hr[2] = s.Hn[2]; }
            else {
                for (int c = 0; c < 3; ++c)
                    Hr[c] = (s.Hn[c] + (s.Mn[c] - Mr[c])) - g.coef_h * s.cE[c];
            }
            const unsigned long long rb = dbits(llg_iterate(s, g.coef_h, Hr, Mr));
            lmax = rb > lmax ? rb : lmax;
            w[9] = Mr[0]; w[10] = Mr[1]; w[11] = Mr[2];
        }
        // block max -> one atomic per block
        for (int sh = 16; sh > 0; sh >>= 1) {
            const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, lmax, sh);
            lmax = o2 > lmax ? o2 : lmax;
        }
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = lmax;
        __syncthreads();
        if (threadIdx.x < 32) {
            unsigned long long x = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0ull;
            for (int sh = 16; sh > 0; sh >>= 1) {
                const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, x, sh);
                x = o2 > x ? o2 : x;
            }
            if (threadIdx.x == 0 && x) atomicMax(&st->hist2[r], x);
        }
        grid.sync();
        const double res = bitsd(*((volatile unsigned long long*)&st->hist2[r]));
        if (res <= g.tol) { rstar = r; break; }
        growth = (res > prev) ? growth + 1 : 0;
        if (growth >= 3) { failed = 1; fres = res; fit = r; fkind = 1; break; }
        prev = res;
        if (r == g.max_iters) { failed = 1; fres = prev; fit = r; fkind = 2; }
        __syncthreads();   // red[] reuse
    }
    if (failed) {
        if (tid == 0) {
            st->fail = 1; st->fail_step = st->step; st->fail_res = fres;
            st->fail_it = fit; st->fail_kind = fkind;
        }
        return;
    }
    for (int q = tid; q < nmag; q += nth) {
        const int i = cells[q].x, f = cells[q].y;
        const int64_t o = i * g.PP + f;
        const int64_t om = (int64_t)(i - g.mx0) * g.PP + f;
        const double* w = v + (size_t)q * 12;
        for (int c = 0; c < 3; ++c) {
            const double hv = (w[c] + (w[3 + c] - w[9 + c])) - g.coef_h * w[6 + c];
            if (mp.on) {
                mp.Hl[c][o] = (T)hv;
                mp.Hn1[c][q] = (T)hv;
                mp.Mn1[c][q] = w[9 + c];
            } else {
                b.Hb[c][o] = hv;
                b.Mb[c][om] = w[9 + c];
            }
        }
    }
    if (tid == 0) { st->rstar = rstar; st->fixup_ran = 1; }
}

template <typename T>
__global__ void __launch_bounds__(256) k_llg_fixup(Geom g, BufsT<T> b,
                                                   const mpb_material* __restrict__ mats,
                                                   const uint8_t* __restrict__ ids,
                                                   const int2* __restrict__ cells, int nmag,
                                                   MagScratch scr, StepState* st,
                                                   MagPre<T> mp) {
    pdl_wait();
    pdl_trigger();
    llg_fixup_grid(g, b, mats, ids, cells, nmag, scr, st, mp);
}

// ---------------------------------------------------------------------------
// Multi-rank LLG settlement (no grid-wide barrier across GPUs).  After the
// sweep, hist and (rc_max, -rc_min) are all-reduced (max) over the ranks.
//  * uniform: every cell stopped at the same R -> replay the stop rule.
//  * otherwise: every cell (owned + ghost-plane copies) is recomputed from
//    scratch to R' = min(R, max_iters) (k_llg_topup), the owned residuals of
//    iterates 1..R' are all-reduced into hist2, and k_llg_decide replays the
//    rule on hist2.  A cell that had stopped earlier cannot make hist2[r]
//    <= tol for r < R' (the cell with r_c = R' is still > tol there), so the
//    rule stops at R' -- unless the global residual is non-monotone at R'
//    (a cell that stopped early is back above tol).  The reference then
//    keeps iterating (llg.py:131-148); the step is suspended (kMpbSuspend:
//    every later kernel of the chunk is a no-op) and the host continues it
//    in lockstep, one iterate and one all-reduce at a time
//    (k_llg_cont_*, mpb_api.cu recover_suspended), then resumes the run.
// ---------------------------------------------------------------------------
constexpr int kMpbSuspend = 4;   // StepState.fail_kind of a suspended step

template <typename T>
__global__ void __launch_bounds__(256) k_llg_topup(Geom g, BufsT<T> b,
                                                   const mpb_material* __restrict__ mats,
                                                   const uint8_t* __restrict__ ids,
                                                   const int2* __restrict__ cells,
                                                   const unsigned char* __restrict__ owned,
                                                   int ncells, StepState* st) {
    __shared__ unsigned long long sh[MPB_MAX_ITERS_CAP + 2];
    if (st->fail) return;
    const int rmin = -st->rc_negmin, rmax = st->rc_max;
    if (rmin == rmax && rmax <= g.max_iters) return;       // uniform case
    const int R = min(rmax, g.max_iters);
    for (int r = threadIdx.x; r <= R + 1; r += blockDim.x) sh[r] = 0ull;
    __syncthreads();
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < ncells) {
        const int i = cells[q].x, f = cells[q].y;
        const int64_t o = i * g.PP + f;
        const int64_t om = (int64_t)(i - g.mx0) * g.PP + f;
        LlgCell s;
        const Curl3 c = curl_e_at(g, b.Ea, o, g.PP, g.F[2], true, true, true);
        for (int k = 0; k < 3; ++k) { s.Hn[k] = b.Ha[k][o]; s.Mn[k] = b.Ma[k][om]; }
        s.cE[0] = c.x; s.cE[1] = c.y; s.cE[2] = c.z;
        llg_setup(s, mats[ids[o]]);
        double Hr[3] = {s.Hn[0], s.Hn[1], s.Hn[2]};
        double Mr[3] = {s.Mn[0], s.Mn[1], s.Mn[2]};
        const bool own = owned[q] != 0;
        for (int r = 1; r <= R; ++r) {
            const double res = llg_iterate(s, g.coef_h, Hr, Mr);
            if (own) atomicMax(&sh[r], dbits(res));
        }
        for (int k = 0; k < 3; ++k) b.Hb[k][o] = Hr[k];
        if (own)
            for (int k = 0; k < 3; ++k) b.Mb[k][om] = Mr[k];
    }
    __syncthreads();
    for (int r = 1 + threadIdx.x; r <= R; r += blockDim.x)
        if (sh[r]) atomicMax(&st->hist2[r], sh[r]);
}

// In-process multi-rank emulation (mpb_group_run): the all-reduce(max) of
// the NCCL path over the ranks' states, one block.
constexpr int kMaxGroup = 16;
struct StatePtrs {
    StepState* s[kMaxGroup];
    int n;
};

__global__ void k_group_reduce(StatePtrs sp, int max_iters, int mode) {
    for (int r = 1 + threadIdx.x; r <= max_iters + 1; r += blockDim.x) {
        if (r <= max_iters) {
            unsigned long long m = 0ull;
            for (int q = 0; q < sp.n; ++q) {
                const unsigned long long v = mode == 0 ? sp.s[q]->hist[r] : sp.s[q]->hist2[r];
                m = v > m ? v : m;
            }
            for (int q = 0; q < sp.n; ++q) {
                if (mode == 0) sp.s[q]->hist[r] = m;
                else sp.s[q]->hist2[r] = m;
            }
        } else if (mode == 0) {
            int a = sp.s[0]->rc_max, b = sp.s[0]->rc_negmin;
            for (int q = 1; q < sp.n; ++q) {
                a = max(a, sp.s[q]->rc_max);
                b = max(b, sp.s[q]->rc_negmin);
            }
            for (int q = 0; q < sp.n; ++q) { sp.s[q]->rc_max = a; sp.s[q]->rc_negmin = b; }
        }
    }
}

__global__ void k_llg_decide(Geom g, StepState* st) {
    if (threadIdx.x != 0 || st->fail) return;
    const int rmin = -st->rc_negmin, rmax = st->rc_max;
    double fr = 0.0; int fi = 0, fk = 0, r;
    if (rmax == 0) return;                                 // no magnetic cell anywhere
    if (rmin == rmax && rmax <= g.max_iters) {
        r = llg_decide(st->hist, rmax, g.max_iters, g.tol, &fr, &fi, &fk);
    } else {
        const int R = min(rmax, g.max_iters);
        r = llg_decide(st->hist2, R, g.max_iters, g.tol, &fr, &fi, &fk);
        st->fixup_ran = 1;
        if (r < 0) {   // still above tol at R: continue on the host (see above)
            st->fail = 1; st->fail_step = st->step; st->fail_res = bitsd(st->hist2[R]);
            st->fail_it = R; st->fail_kind = kMpbSuspend;
            return;
        }
    }
    if (r > 0) {
        st->rstar = r;
    } else {
        st->fail = 1; st->fail_step = st->step; st->fail_res = fr;
        st->fail_it = fi; st->fail_kind = fk;
    }
}

// Lockstep continuation of a suspended multi-rank step (host-driven, one
// iterate per launch).  Scratch per local cell: Hn[3] Mn[3] cE[3] Mr[3].
template <typename T>
__global__ void __launch_bounds__(256) k_llg_cont_init(Geom g, BufsT<T> b,
                                                       const int2* __restrict__ cells, int n,
                                                       MagScratch scr) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int i = cells[q].x, f = cells[q].y;
    const int64_t o = i * g.PP + f;
    const int64_t om = (int64_t)(i - g.mx0) * g.PP + f;
    const Curl3 c = curl_e_at(g, b.Ea, o, g.PP, g.F[2], true, true, true);
    double* w = scr.v + (size_t)q * 12;
    for (int k = 0; k < 3; ++k) {
        w[k] = b.Ha[k][o];
        w[3 + k] = b.Ma[k][om];
        w[9 + k] = w[3 + k];
    }
    w[6] = c.x; w[7] = c.y; w[8] = c.z;
}

// iterate r of every local cell (llg.py:131-137); owned cells' residuals
// max-reduced into st->hist2[r]
__global__ void __launch_bounds__(256) k_llg_cont_iter(Geom g,
                                                       const mpb_material* __restrict__ mats,
                                                       const uint8_t* __restrict__ ids,
                                                       const int2* __restrict__ cells,
                                                       const unsigned char* __restrict__ owned,
                                                       int n, MagScratch scr, StepState* st,
                                                       int r) {
    __shared__ unsigned long long red[8];
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long lmax = 0ull;
    if (q < n) {
        const int i = cells[q].x, f = cells[q].y;
        double* w = scr.v + (size_t)q * 12;
        LlgCell s;
        for (int c = 0; c < 3; ++c) { s.Hn[c] = w[c]; s.Mn[c] = w[3 + c]; s.cE[c] = w[6 + c]; }
        llg_setup(s, mats[ids[i * g.PP + f]]);
        double Mr[3] = {w[9], w[10], w[11]};
        double Hr[3];
        for (int c = 0; c < 3; ++c)   // H^{n+1,r-1} (llg.py:105); H^n before iterate 1
            Hr[c] = r == 1 ? s.Hn[c] : (s.Hn[c] + (s.Mn[c] - Mr[c])) - g.coef_h * s.cE[c];
        const unsigned long long rb = dbits(llg_iterate(s, g.coef_h, Hr, Mr));
        if (owned[q]) lmax = rb;
        w[9] = Mr[0]; w[10] = Mr[1]; w[11] = Mr[2];
    }
    for (int sh = 16; sh > 0; sh >>= 1) {
        const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, lmax, sh);
        lmax = o2 > lmax ? o2 : lmax;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = lmax;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long x = 0ull;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) x = red[w] > x ? red[w] : x;
        if (x) atomicMax(&st->hist2[r], x);
    }
}

// the settled iterate r*: H^{n+1} (every local cell) and M^{n+1} (owned)
template <typename T>
__global__ void __launch_bounds__(256) k_llg_cont_write(Geom g, BufsT<T> b,
                                                        const int2* __restrict__ cells,
                                                        const unsigned char* __restrict__ owned,
                                                        int n, MagScratch scr, StepState* st,
                                                        int rstar) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q == 0) { st->rstar = rstar; st->fixup_ran = 1; }
    if (q >= n) return;
    const int i = cells[q].x, f = cells[q].y;
    const int64_t o = i * g.PP + f;
    const int64_t om = (int64_t)(i - g.mx0) * g.PP + f;
    const double* w = scr.v + (size_t)q * 12;
    for (int c = 0; c < 3; ++c) {
        b.Hb[c][o] = (w[c] + (w[3 + c] - w[9 + c])) - g.coef_h * w[6 + c];
        if (owned[q]) b.Mb[c][om] = w[9 + c];
    }
}

// Start of a run chunk: absolute step, output row 0, staging pointers.
__global__ void k_set_run(StepState* st, long long step, const double* src, double* probe,
                          int* iters) {
    st->step = step;
    st->local = 0;
    st->src_vals = src;
    st->probe_out = probe;
    st->iters_out = iters;
    st->llg_count = 0;
    st->llg_stamp = -1;   // no stale stamp can match a step of this run
}

// Clear a suspension (and the lockstep history) before the host continues
// the step; record a failure the host-driven continuation found.
__global__ void k_suspend_clear(StepState* st, int max_iters) {
    for (int r = threadIdx.x; r <= max_iters + 1; r += blockDim.x) st->hist2[r] = 0ull;
    if (threadIdx.x == 0) { st->fail = 0; st->fail_kind = 0; st->fail_step = -1; }
}

__global__ void k_set_failure(StepState* st, double res, int it, int kind) {
    st->fail = 1; st->fail_step = st->step; st->fail_res = res;
    st->fail_it = it; st->fail_kind = kind;
}

// ---------------------------------------------------------------------------
// Walls, one launch per face in the order x0,x1,y0,y1,z0,z1 (em.py:324-359).
// MUR1 reads the pre-update planes straight from the read buffer Ea (the
// reference copies them before the update, em.py:306-321).
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) k_wall(Geom g, BufsT<T> b,
                                              const mpb_material* __restrict__ mats,
                                              const uint8_t* __restrict__ ids,
                                              const StepState* st, int face) {
    if (st->fail) return;
    const int axis = face >> 1, side = face & 1;
    const int u = axis == 0 ? 1 : 0;          // the two in-plane axes
    const int w = axis == 2 ? 1 : 2;
    // x is the slab axis: y/z faces cover the owned planes only
    const int u0 = u == 0 ? g.c0 : 0;
    const int nu = u == 0 ? g.c1 - g.c0 : g.F[u], nw = g.F[w];
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)nu * nw) return;
    const int iu = u0 + (int)(t / nw), iw = (int)(t - (int64_t)(iu - u0) * nw);
    const int64_t stride[3] = {g.PP, g.F[2], 1};
    const int wall = side == 0 ? 0 : g.n[axis];
    const int inner = side == 0 ? 1 : g.n[axis] - 1;
    const int64_t base = iu * stride[u] + iw * stride[w];
    const int64_t ow = base + wall * stride[axis];
    const int64_t oi = base + inner * stride[axis];
    const int c0 = axis == 0 ? 1 : 0;         // tangential E components
    const int c1 = axis == 2 ? 1 : 2;
    if (g.faces[face] == MPB_FACE_PEC) {
        b.Eb[c0][ow] = 0.0;
        b.Eb[c1][ow] = 0.0;
    } else {   // MUR1: wall = prev_inner + k (inner_new - prev_wall)
        const double kk = mats[ids[ow]].mur_k[axis];
        b.Eb[c0][ow] = b.Ea[c0][oi] + kk * (b.Eb[c0][oi] - b.Ea[c0][ow]);
        b.Eb[c1][ow] = b.Ea[c1][oi] + kk * (b.Eb[c1][oi] - b.Ea[c1][ow]);
    }
}

// The x0, x1, y0, y1 walls in ONE launch (blockIdx.y = face), with the
// result of the sequential face order (em.py:324-359).  The faces interact
// only on the edge lines: y walls overwrite Ez on the x walls' j = 0 / ny
// rows (so the x-face thread skips those entries), and a y wall's MUR reads
// Ez at its inner row, which an x wall has already written on i = 0 / nx (so
// the y-face thread recomputes the x wall's value there instead of reading
// it).  Every other read is of entries no wall writes.  act: bit f = face f
// active on this rank.
// ---------------------------------------------------------------------------
// One entry t of x/y wall `face` (active faces: bits of act).
// Returns max e_range over the valid E entries written (StepState.eunsafe_b).
// Every load of the entry is issued before the first store and alongside the
// kernel's fail flag (the stores go to other arrays than the loads read, which
// the compiler cannot prove): two round trips (E + ids, then the material's
// MUR coefficient) instead of a chain of five.
template <typename T>
__device__ __forceinline__ unsigned wall_xy_entry(const Geom& g, const BufsT<T>& b,
                                                  const mpb_material* __restrict__ mats,
                                                  const uint8_t* __restrict__ ids, int act,
                                                  int face, int64_t t, int fail) {
    const int side = face & 1;
    const int Fz = g.F[2];
    const bool mur = g.faces[face] != MPB_FACE_PEC;
    unsigned eg = 0;
    if (face < 2) {                            // x wall: entries (j, k), Ey and Ez
        if (t >= (int64_t)g.F[1] * Fz) return 0u;
        const int j = (int)(t / Fz);
        const int k = (int)(t - (int64_t)j * Fz);
        const int64_t ow = (int64_t)(side ? g.n[0] : 0) * g.PP + t;
        const int64_t oi = (int64_t)(side ? g.n[0] - 1 : 1) * g.PP + t;
        const bool y_over = (j == 0 && (act & 4)) || (j == g.n[1] && (act & 8));
        double a1i = 0, b1i = 0, a1w = 0, a2i = 0, b2i = 0, a2w = 0;
        uint8_t id = 0;
        if (mur) {
            id = ids[ow];
            a1i = b.Ea[1][oi]; b1i = b.Eb[1][oi]; a1w = b.Ea[1][ow];
            if (!y_over) { a2i = b.Ea[2][oi]; b2i = b.Eb[2][oi]; a2w = b.Ea[2][ow]; }
        }
        if (fail) return 0u;
        const double kk = mur ? mats[id].mur_k[0] : 0.0;
        // MUR1: wall = prev_inner + k (inner_new - prev_wall)
        const T vy = mur ? T(a1i + kk * (b1i - a1w)) : T(0);
        b.Eb[1][ow] = vy;
        if (j < g.n[1]) eg = max(eg, e_range((double)vy));
        if (!y_over) {
            const T vz = mur ? T(a2i + kk * (b2i - a2w)) : T(0);
            b.Eb[2][ow] = vz;
            if (k < g.n[2]) eg = max(eg, e_range((double)vz));
        }
        return eg;
    } else {                                   // y wall: entries (i, k) of owned planes, Ex and Ez
        const int nown = g.c1 - g.c0;
        if (t >= (int64_t)nown * Fz) return 0u;
        const int i = g.c0 + (int)(t / Fz);
        const int k = (int)(t - (int64_t)(i - g.c0) * Fz);
        const int jw = side ? g.n[1] : 0, jn = side ? g.n[1] - 1 : 1;
        const int64_t ow = (int64_t)i * g.PP + (int64_t)jw * Fz + k;
        const int64_t oi = (int64_t)i * g.PP + (int64_t)jn * Fz + k;
        // Ez at the inner row, after the x walls (recomputed: the x faces run
        // in the same launch)
        const int xf = (i == 0 && (act & 1)) ? 0 : ((i == g.n[0] && (act & 2)) ? 1 : -1);
        const bool xmur = xf >= 0 && g.faces[xf] != MPB_FACE_PEC;
        double a0i = 0, b0i = 0, a0w = 0, a2i = 0, a2w = 0, b2i = 0, b2x = 0, a2x = 0;
        uint8_t id = 0, idx = 0;
        if (mur) {
            id = ids[ow];
            a0i = b.Ea[0][oi]; b0i = b.Eb[0][oi]; a0w = b.Ea[0][ow];
            a2i = b.Ea[2][oi]; a2w = b.Ea[2][ow];
            if (xf < 0) b2i = b.Eb[2][oi];
        }
        if (mur && xmur) {
            const int64_t xin = (int64_t)(xf ? g.n[0] - 1 : 1) * g.PP + (int64_t)jn * Fz + k;
            idx = ids[oi]; b2x = b.Eb[2][xin]; a2x = b.Ea[2][xin];
        }
        if (fail) return 0u;
        const double kk = mur ? mats[id].mur_k[1] : 0.0;
        const T vx = mur ? T(a0i + kk * (b0i - a0w)) : T(0);
        b.Eb[0][ow] = vx;
        if (i < g.n[0]) eg = max(eg, e_range((double)vx));
        T vz;
        if (!mur) {
            vz = T(0);
        } else {
            double ez_in;
            if (xf >= 0) ez_in = xmur ? a2x + mats[idx].mur_k[0] * (b2x - a2i) : 0.0;
            else ez_in = b2i;
            vz = T(a2i + kk * (ez_in - a2w));
        }
        b.Eb[2][ow] = vz;
        if (k < g.n[2]) eg = max(eg, e_range((double)vz));
        return eg;
    }
}

template <typename T>
__global__ void __launch_bounds__(256) k_walls_xy(Geom g, BufsT<T> b,
                                                  const mpb_material* __restrict__ mats,
                                                  const uint8_t* __restrict__ ids,
                                                  StepState* st, int act) {
    pdl_wait();
    pdl_trigger();
    const int face = blockIdx.y;
    if (!((act >> face) & 1)) return;
    const int fail = st->fail;   // in flight with the entry's loads
    const unsigned eg = wall_xy_entry(g, b, mats, ids, act, face,
                                      (int64_t)blockIdx.x * blockDim.x + threadIdx.x, fail);
    if (fail) return;
    if (g.eguard) flag_e_range(eg, &st->eunsafe_b);
}

// Element-type conversion for fp32-storage uploads/downloads (round to
// nearest; double -> float -> double is the identity on the stored values).
template <typename Tin, typename Tout>
__global__ void k_convert(const Tin* __restrict__ in, Tout* __restrict__ out, int64_t n) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
         q += (int64_t)gridDim.x * blockDim.x)
        out[q] = (Tout)in[q];
}

// ---------------------------------------------------------------------------
// Energy diagnostic (em.py:366-383): per-block partial sums in a fixed
// order, then one block combines them -- deterministic run to run.
// out[0..2] per block: sum eps E^2, sum H^2, sum M.Hbias.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) k_energy_partial(Geom g, const T* const* E,
                                                        const T* const* H,
                                                        const double* const* M,
                                                        const mpb_material* __restrict__ mats,
                                                        const uint8_t* __restrict__ ids,
                                                        double* partial) {
    __shared__ double red[3][256];
    const int64_t nent = (int64_t)(g.c1 - g.c0) * g.FyFz;
    double se = 0.0, sh = 0.0, sm = 0.0;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nent;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int i = g.c0 + (int)(q / g.FyFz);
        const int f = (int)(q - (int64_t)(i - g.c0) * g.FyFz);
        const int64_t o = i * g.PP + f;
        const mpb_material& m = mats[ids[o]];
        const double e0 = E[0][o], e1 = E[1][o], e2 = E[2][o];
        const double h0 = H[0][o], h1 = H[1][o], h2 = H[2][o];
        se += m.eps * (e0 * e0) + m.eps * (e1 * e1) + m.eps * (e2 * e2);
        sh += h0 * h0 + h1 * h1 + h2 * h2;
        const int j = f / g.F[2], k = f - j * g.F[2];
        if (M[0] && i >= g.mx0 && i < g.mx1 && i < g.n[0] && j < g.n[1] && k < g.n[2]) {
            const int64_t om = (int64_t)(i - g.mx0) * g.PP + f;
            sm += M[0][om] * m.hbias[0] + M[1][om] * m.hbias[1] + M[2][om] * m.hbias[2];
        }
    }
    red[0][threadIdx.x] = se; red[1][threadIdx.x] = sh; red[2][threadIdx.x] = sm;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            for (int c = 0; c < 3; ++c) red[c][threadIdx.x] += red[c][threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int c = 0; c < 3; ++c) partial[3 * blockIdx.x + c] = red[c][0];
}

// ---------------------------------------------------------------------------
// End of step: soft source (em.py:276-282), probes (sim.py:170-171), r*
// record (sim.py:167), reset of the LLG bookkeeping for the next step.
// One block.
// ---------------------------------------------------------------------------
struct SourceDesc {
    int64_t off;
    double pol[3];
};

// Source, probes, r* record and the bookkeeping reset, by one block.
template <typename T>
__device__ void finish_block(const Geom& g, const BufsT<T>& b, const SourceDesc& src,
                             const ProbeDesc* __restrict__ probes, int nprobes, int parity_b,
                             int record_iters, StepState* st) {
    // A chain of dependent round trips is this kernel's whole cost, so every
    // load that does not depend on another is issued up front: the fail flag,
    // the row, the source entries and each thread's first probe value (a
    // probe on the source entry is re-read after the injection).
    const int fail = st->fail;
    const long long row = st->local;
    double e0[3] = {0.0, 0.0, 0.0};
    unsigned eub = 0;
    if (threadIdx.x == 0) {
        for (int c = 0; c < 3; ++c)
            if (src.pol[c] != 0.0) e0[c] = (double)b.Eb[c][src.off];
        if (g.eguard) eub = st->eunsafe_b;
    }
    auto probe_value = [&](const ProbeDesc& pd) -> double {
        const void* base = parity_b ? pd.ptr1 : pd.ptr0;
        return !base ? pd.constant
                     : (pd.f32 ? (double)static_cast<const float*>(base)[pd.off]
                               : static_cast<const double*>(base)[pd.off]);
    };
    double pv0 = 0.0;
    ProbeDesc pd0{};
    if ((int)threadIdx.x < nprobes) {
        pd0 = probes[threadIdx.x];
        pv0 = probe_value(pd0);
    }
    if (fail) return;
    if (threadIdx.x == 0) {
        const double v = st->src_vals[row];
        unsigned eg = 0;
        for (int c = 0; c < 3; ++c)
            if (src.pol[c] != 0.0) {
                const double pv = src.pol[c] * v;
                const T nv = e0[c] + pv;
                b.Eb[c][src.off] = nv;
                eg = max(eg, e_range((double)nv));
            }
        // the E set just completed becomes the next sweep's input
        if (g.eguard) {
            st->eunsafe_a = eub | (eg > kSafeSpan ? 1 : 0);
            st->eunsafe_b = 0;
        }
    }
    __syncthreads();
    if ((int)threadIdx.x < nprobes) {
        if (pd0.off == src.off) pv0 = probe_value(pd0);   // may sample the injected entry
        st->probe_out[row * nprobes + threadIdx.x] = pv0;
    }
    for (int p = threadIdx.x + blockDim.x; p < nprobes; p += blockDim.x)
        st->probe_out[row * nprobes + p] = probe_value(probes[p]);
    for (int r = threadIdx.x; r <= g.max_iters + 1; r += blockDim.x) {
        st->hist[r] = 0ull;
        st->hist2[r] = 0ull;
    }
    if (threadIdx.x == 0) {
        if (record_iters) st->iters_out[row] = st->rstar;
        st->rstar = 0;
        st->fixup_ran = 0;
        st->rc_negmin = -0x7fffffff;
        st->rc_max = 0;
        st->local = row + 1;
        st->step = st->step + 1;
    }
}

template <typename T>
__global__ void __launch_bounds__(256) k_finish(Geom g, BufsT<T> b, SourceDesc src,
                                                const ProbeDesc* __restrict__ probes,
                                                int nprobes, int parity_b, int record_iters,
                                                StepState* st) {
    pdl_wait();
    pdl_trigger();
    finish_block(g, b, src, probes, nprobes, parity_b, record_iters, st);
}

}  // namespace mpb
