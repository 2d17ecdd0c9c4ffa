// mpb_line.cuh -- whole-run kernel for lines along z (nx = ny = 1): the
// reference's 1D cavities (pkg/configs/cavity1d.cfg, the acceptance sweeps).
//
// A line of a few thousand entries cannot fill a GPU; stepped with the
// general kernels it costs ~5 launches (~19 us) per step.  Here ONE CTA keeps
// the whole state -- E, H and the M line -- in shared memory and runs every
// step of a chunk in a loop, phases separated by __syncthreads: curl E / H
// update, the LLG fixed point with the global stop rule as a block
// reduction, MUR capture, curl H / E update, z walls, source, probes.  The
// arithmetic is the general kernels' entry for entry (same expressions, same
// order, the same LLG helpers), so results are bit-identical; every other
// SM stays free for concurrent runs (bias sweeps).
//
// Collapsed x and y: only z derivatives exist, x/y walls are skipped
// (em.py:336-338), Ez gets ca*(0 - cb*Ez) and Hz is never changed
// (Hz - coef*0.0 == Hz bitwise).
#pragma once

namespace mpb {

struct LineProbe {
    int src;       // 0..5 E/H component, 6..8 M component, -1 constant
    int idx;       // entry along z
    double constant;
};

struct LineArgs {
    double* E[3];          // state buffers to read (set pa) ...
    double* H[3];
    double* M[3];          // M plane (nullptr if no magnetic cell)
    double* Eo[3];         // ... and to write the final state to (set pb)
    double* Ho[3];
    double* Mo[3];
    const uint8_t* ids;    // entry -> material (edge-padded)
    const mpb_material* mats;
    const int2* magcells;  // (plane, entry)
    int nmag;
    int nmat;
    const LineProbe* probes;
    int nprobes;
    int src_off;           // source entry
    double src_pol[3];
    int any_magnetic;
    int nsteps;
};

constexpr int kLineThreads = 512;

__global__ void __launch_bounds__(kLineThreads, 1) k_line(Geom g, LineArgs a, StepState* st) {
    extern __shared__ __align__(16) double sm[];
    const int Fz = g.F[2];
    const int nz = g.n[2];
    double* E0 = sm;            double* E1 = E0 + Fz;   double* E2 = E1 + Fz;
    double* H0 = E2 + Fz;       double* H1 = H0 + Fz;   double* H2 = H1 + Fz;
    double* M0 = H2 + Fz;       double* M1 = M0 + Fz;   double* M2 = M1 + Fz;
    double* s_ca = M2 + Fz;     // per material: ca, cb, mur_k[2]
    double* s_cb = s_ca + a.nmat;
    double* s_mk = s_cb + a.nmat;
    uint8_t* s_id = reinterpret_cast<uint8_t*>(s_mk + a.nmat);
    __shared__ unsigned long long s_res;    // block max of the iterate's residual bits
    __shared__ int s_stop;                  // r* (> 0), 0 continue, -1 failed
    __shared__ double s_mur[8];             // (Ex, Ey) x (wall, inner) x (z0, z1) at step n
    double* Ef[3] = {E0, E1, E2};
    double* Hf[3] = {H0, H1, H2};
    double* Mf[3] = {M0, M1, M2};

    const int tid = threadIdx.x;
    if (st->fail) return;
    for (int e = tid; e < Fz; e += blockDim.x) {
        for (int c = 0; c < 3; ++c) {
            Ef[c][e] = a.E[c][e];
            Hf[c][e] = a.H[c][e];
            Mf[c][e] = a.M[c] ? a.M[c][e] : 0.0;
        }
        s_id[e] = a.ids[e];
    }
    for (int q = tid; q < a.nmat; q += blockDim.x) {
        s_ca[q] = a.mats[q].ca; s_cb[q] = a.mats[q].cb; s_mk[q] = a.mats[q].mur_k[2];
    }
    const double dz = g.d[2], rz = g.rd[2];
    const bool pmc_z0 = g.faces[4] == MPB_FACE_PMC, pmc_z1 = g.faces[5] == MPB_FACE_PMC;
    // this thread's magnetic cell (one per thread), kept in registers
    const bool owner = tid < a.nmag;
    const int mk = owner ? a.magcells[tid].y : 0;
    mpb_material mm{};
    if (owner) mm = a.mats[a.ids[mk]];
    __syncthreads();

    long long step = st->step, row = st->local;
    for (int t = 0; t < a.nsteps; ++t, ++step, ++row) {
        // ---- curl E (em.py:117-139) and the non-magnetic H update
        //      (em.py:171-182); magnetic entries keep H^n for the LLG ------------
        double cEx = 0.0, cEy = 0.0;      // curl E at this thread's magnetic cell
        if (owner) {
            cEx = 0.0 - ddiv(E1[mk + 1] - E1[mk], dz, rz);
            cEy = 0.0 + ddiv(E0[mk + 1] - E0[mk], dz, rz);
        }
        for (int k = tid; k < nz; k += blockDim.x) {
            if (s_id[k] & 0x80) continue;      // magnetic (id bit 7): LLG below
            const double cx = 0.0 - ddiv(E1[k + 1] - E1[k], dz, rz);
            const double cy = 0.0 + ddiv(E0[k + 1] - E0[k], dz, rz);
            H0[k] = H0[k] - g.coef_h * cx;
            H1[k] = H1[k] - g.coef_h * cy;
        }
        if (tid == 0) {                    // MUR capture (em.py:306-323), pre-update E
            s_mur[0] = E0[0];  s_mur[1] = E0[1];  s_mur[2] = E1[0];  s_mur[3] = E1[1];
            s_mur[4] = E0[nz]; s_mur[5] = E0[nz - 1]; s_mur[6] = E1[nz]; s_mur[7] = E1[nz - 1];
            s_res = 0ull;
            s_stop = 0;
        }
        __syncthreads();

        // ---- LLG fixed point with the global stop rule (llg.py:108-148) ----
        int rstar = 0;
        if (a.nmag > 0) {
            LlgCell s;
            double Hr[3], Mr[3];
            if (owner) {
                s.Hn[0] = H0[mk]; s.Hn[1] = H1[mk]; s.Hn[2] = H2[mk];
                s.Mn[0] = M0[mk]; s.Mn[1] = M1[mk]; s.Mn[2] = M2[mk];
                s.cE[0] = cEx; s.cE[1] = cEy; s.cE[2] = 0.0;
                llg_setup(s, mm);
                for (int c = 0; c < 3; ++c) { Hr[c] = s.Hn[c]; Mr[c] = s.Mn[c]; }
            }
            double prev = __longlong_as_double(0x7ff0000000000000LL);   // +inf
            int growth = 0;
            for (int it = 1;; ++it) {
                if (owner) {
                    const unsigned long long rb = dbits(llg_iterate(s, g.coef_h, Hr, Mr));
                    atomicMax(&s_res, rb);
                }
                __syncthreads();
                if (tid == 0) {            // llg_decide, one iterate at a time
                    const double res = bitsd(s_res);
                    int stop = 0;
                    if (res <= g.tol) {
                        stop = it;
                    } else {
                        growth = (res > prev) ? growth + 1 : 0;
                        if (growth >= 3) {                      // diverging
                            st->fail_res = res; st->fail_it = it; st->fail_kind = 1;
                            stop = -1;
                        } else {
                            prev = res;
                            if (it == g.max_iters) {            // budget exhausted
                                st->fail_res = prev; st->fail_it = g.max_iters;
                                st->fail_kind = 2;
                                stop = -1;
                            }
                        }
                        if (stop < 0) { st->fail = 1; st->fail_step = step; }
                    }
                    s_stop = stop;
                    s_res = 0ull;
                }
                __syncthreads();
                if (s_stop != 0) break;
            }
            if (s_stop < 0) return;        // StepFailure: the host raises
            rstar = s_stop;
            if (owner) {
                H0[mk] = Hr[0]; H1[mk] = Hr[1]; H2[mk] = Hr[2];
                M0[mk] = Mr[0]; M1[mk] = Mr[1]; M2[mk] = Mr[2];
            }
            __syncthreads();
        }

        // ---- curl H with PMC ghosts (em.py:185-232) and the E update
        //      (em.py:257-272), every entry, in place ----------------------------
        for (int k = tid; k <= nz; k += blockDim.x) {
            const int km = k > 0 ? k - 1 : k;
            const double hx = H0[k], hy = H1[k], hx_km = H0[km], hy_km = H1[km];
            const double yhi = (k == nz) ? (pmc_z1 ? -hy_km : 0.0) : hy;
            const double ylo = (k == 0) ? (pmc_z0 ? -hy : 0.0) : hy_km;
            const double xhi = (k == nz) ? (pmc_z1 ? -hx_km : 0.0) : hx;
            const double xlo = (k == 0) ? (pmc_z0 ? -hx : 0.0) : hx_km;
            const double cx = 0.0 - ddiv(yhi - ylo, dz, rz);
            const double cy = 0.0 + ddiv(xhi - xlo, dz, rz);
            const double cz = 0.0;
            const int id = s_id[k];            // table index (magnetic ids carry bit 7)
            const double ca = s_ca[id], cb = s_cb[id];
            E0[k] = ca * (cx - cb * E0[k]);
            E1[k] = ca * (cy - cb * E1[k]);
            E2[k] = ca * (cz - cb * E2[k]);
        }
        __syncthreads();

        if (tid == 0) {
            // ---- z walls in face order z0, z1 (em.py:326-359) ---------------
            for (int side = 0; side < 2; ++side) {
                const int face = g.faces[4 + side];
                const int w = side == 0 ? 0 : nz, in = side == 0 ? 1 : nz - 1;
                if (face == MPB_FACE_PEC) {
                    E0[w] = 0.0; E1[w] = 0.0;
                } else if (face == MPB_FACE_MUR1) {
                    const double kk = s_mk[s_id[w]];
                    E0[w] = s_mur[4 * side + 1] + kk * (E0[in] - s_mur[4 * side + 0]);
                    E1[w] = s_mur[4 * side + 3] + kk * (E1[in] - s_mur[4 * side + 2]);
                }
            }
            // ---- soft source (em.py:276-282) --------------------------------
            const double v = st->src_vals[row];
            for (int c = 0; c < 3; ++c)
                if (a.src_pol[c] != 0.0) {
                    const double pv = a.src_pol[c] * v;
                    Ef[c][a.src_off] = Ef[c][a.src_off] + pv;
                }
            if (a.any_magnetic) st->iters_out[row] = rstar;
        }
        __syncthreads();
        // ---- probes (sim.py:170-171) ----------------------------------------
        for (int p = tid; p < a.nprobes; p += blockDim.x) {
            const LineProbe lp = a.probes[p];
            double v = lp.constant;
            if (lp.src >= 0 && lp.src < 3) v = Ef[lp.src][lp.idx];
            else if (lp.src >= 3 && lp.src < 6) v = Hf[lp.src - 3][lp.idx];
            else if (lp.src >= 6) v = Mf[lp.src - 6][lp.idx];
            st->probe_out[row * a.nprobes + p] = v;
        }
        // the next step's first phase reads E and writes H / s_mur / s_res:
        // fence it off from the probe reads and the source above
        __syncthreads();
    }
    // ---- final state -> buffer set pb ---------------------------------------
    for (int e = tid; e < Fz; e += blockDim.x)
        for (int c = 0; c < 3; ++c) {
            a.Eo[c][e] = Ef[c][e];
            a.Ho[c][e] = Hf[c][e];
            if (a.Mo[c]) a.Mo[c][e] = Mf[c][e];
        }
    if (tid == 0) { st->step = step; st->local = row; }
}

}  // namespace mpb
