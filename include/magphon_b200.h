/*
 * magphon_b200.h -- C ABI of the B200 coupled Maxwell-LLG stepper.
 *
 * This is the drop-in boundary for the hot loop of the reference solver,
 * ``magphon.sim.run`` (reference pkg/src/magphon/sim.py:151-171): one call
 * advances the lattice through whole coupled steps (curl E -> H / LLG fixed
 * point -> curl H -> semi-implicit E -> walls -> soft source -> probes).
 * The reference has no FFI of its own (it is pure numpy); each entry point
 * below names the reference function(s) whose work it takes over.  The
 * Python host mirror (paper_2510_22221_b200/_native.py) binds it with
 * ctypes; INTEGRATION.md shows the binding a magphon maintainer would add.
 *
 * Conventions
 *  - Plain C types only; no torch / CUDA types in signatures.  Host arrays
 *    are C-order float64 in the reference allocation layout (grid.py:82-99):
 *    each E/H component has field_shape = (n+1 on active axes, 1 on
 *    collapsed ones); M is (3, nx, ny, nz).
 *  - Every function returns MPB_OK (0) or an error code; the message of the
 *    last error on the calling thread is available from mpb_last_error().
 *  - A handle owns all of its device memory and streams; it is not
 *    thread-safe.  Do not fork after mpb_create.
 *  - Arithmetic is IEEE fp64 without FMA contraction, in the reference's
 *    operation order, so results are bit-identical to the reference CPU path
 *    (the opt-in fp32 field storage, mpb_setup.storage, trades that for half
 *    the HBM traffic and is held to a tolerance instead).
 */
#ifndef MAGPHON_B200_H
#define MAGPHON_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define MPB_API __attribute__((visibility("default")))
#else
#define MPB_API
#endif

#define MPB_OK 0
#define MPB_EINVAL 1        /* invalid argument      -> ValueError          */
#define MPB_ESTEP 2         /* LLG fixed point failed -> llg.StepFailure    */
#define MPB_ECUDA 3         /* CUDA / NCCL error      -> RuntimeError       */

#define MPB_FACE_PEC 0
#define MPB_FACE_PMC 1
#define MPB_FACE_MUR1 2

#define MPB_MAX_MATERIALS 256
#define MPB_MAX_ITERS_CAP 1000

/* Probe / field component codes: Ex Ey Ez Hx Hy Hz Mx My Mz. */
#define MPB_COMP_EX 0
#define MPB_COMP_HX 3
#define MPB_COMP_MX 6

/* One entry of the material table.  Every coefficient is precomputed on the
 * host with the reference's own numpy expressions so the device only ever
 * multiplies/adds/divides them in the reference order:
 *   ca, cb      em.py:239-254   (1/(sigma/2+eps/dt), sigma/2-eps/dt)
 *   mur_k[a]    em.py:352-357   ((c dt - d_a)/(c dt + d_a), c = 1/sqrt(mu0 eps))
 *   c_llg       llg.py:125      (mu0*|gamma|*dt/2)
 *   alpha_ms    llg.py:132      (alpha/Ms)                                  */
typedef struct mpb_material {
    double ca, cb;
    double mur_k[3];
    double Ms;
    double alpha_ms;
    double c_llg;
    double hbias[3];
    int32_t magnetic;       /* Ms > 0 */
    int32_t pad_;
    double eps;             /* eps0*eps_r      em.py:377 (energy diagnostic)  */
} mpb_material;

typedef struct mpb_setup {
    int32_t n[3];           /* cell counts nx, ny, nz (grid.py:41-74)        */
    double d[3];            /* spacings dx, dy, dz                            */
    double dt;              /* SimConfig.dt  (sim.py:52-54)                   */
    double coef_h;          /* dt/mu0        (em.py:178, llg.py:105)          */
    int32_t faces[6];       /* x0 x1 y0 y1 z0 z1, MPB_FACE_*                  */
    int32_t n_materials;
    const mpb_material* materials;
    const uint8_t* cell_material;   /* (nx,ny,nz) C-order material ids        */
    int32_t src_loc[3];     /* already wrapped into range by the caller       */
    double src_pol[3];      /* SourceSpec.polarization                        */
    int32_t n_probes;
    const int32_t* probe_comp;      /* n_probes codes                         */
    const int32_t* probe_loc;       /* 3*n_probes indices                     */
    double llg_tol;         /* LlgIterationParams (llg.py:49-58)             */
    int32_t llg_max_iters;
    int32_t device;         /* CUDA ordinal                                   */
    int32_t kernel_variant; /* 0 = default (fused sweep), 1 = split H/E sweeps */
    int32_t graph_steps;    /* steps per captured CUDA graph (0 = default)    */
    /* x-slab decomposition.  Single GPU: nranks = 1, x_lo = 0,
     * x_hi = n[0].  This rank owns cell planes [x_lo, x_hi) (the last rank
     * also the field plane n[0]); cell_material then covers cell planes
     * [max(0, x_lo-1), min(n[0], x_hi+1)) and the state arrays of
     * mpb_load_state / mpb_save_state cover field planes
     * [max(0, x_lo-1), min(F[0], x_hi'+1)) with x_hi' = F[0] on the last
     * rank (one ghost plane per side).  Boundary planes travel over NCCL at
     * the end of every step; the LLG residual history is all-reduced. */
    int32_t nranks;
    int32_t rank;
    int32_t x_lo, x_hi;
    int32_t any_magnetic;   /* 1 if any rank owns magnetic cells             */
    uint8_t nccl_id[128];   /* ncclUniqueId from mpb_nccl_unique_id (rank 0) */
    /* Field storage: MPB_STORAGE_F64 (default; the reference's fp64, results
     * bit-identical) or MPB_STORAGE_F32 (opt-in: E and H stored and updated
     * in fp32 -- 48 B/cell instead of 96 -- while M and the whole LLG fixed
     * point stay fp64; agrees with the fp64 reference within a stated
     * tolerance, not bitwise.  Fused sweep only, no line kernel). */
    int32_t storage;
} mpb_setup;

#define MPB_STORAGE_F64 0
#define MPB_STORAGE_F32 1

/* Failure record of an LLG step (llg.py:139-148 + sim.py:161-164). */
typedef struct mpb_failure {
    int64_t step;           /* -1 if no failure                                */
    double residual;
    int32_t iterations;
    int32_t kind;           /* 1 = diverging, 2 = budget exhausted (llg.py:139-148);
                               4 = multi-rank step suspended: its global residual
                                   went back above tol after the last local stop.
                                   mpb_run / mpb_group_run continue such a step in
                                   lockstep (one all-reduce per iterate) and never
                                   return 4; only mpb_run_device + mpb_check_failure
                                   can report it. */
} mpb_failure;

typedef struct mpb_handle mpb_handle;

/* Library / build identification, e.g. "magphon_b200 0.1 sm_100a fmad=false". */
MPB_API const char* mpb_version(void);

/* NCCL unique id for a multi-rank run (call on rank 0, broadcast the 128
 * bytes to every rank, pass in mpb_setup.nccl_id). */
MPB_API int mpb_nccl_unique_id(uint8_t out[128]);

/* Message of the last error on this thread ("" if none). */
MPB_API const char* mpb_last_error(void);

/* Allocate device state for one run and upload the material table.
 * Replaces: grid.allocate + _MagneticCells + em._e_coefficients /
 * _nonmagnetic_H_masks setup (grid.py:140-156, sim.py:100-111,
 * em.py:152-168, em.py:239-254).  Fields start at zero; call
 * mpb_load_state to set E, H, M (the host computes the initial M). */
MPB_API int mpb_create(const mpb_setup* setup, mpb_handle** out);

MPB_API void mpb_destroy(mpb_handle* h);

/* Upload / download the full state in reference layout
 * (FieldLattice.load_state / state_arrays, grid.py:125-137).
 * fields[0..5] = Ex Ey Ez Hx Hy Hz, each prod(field_shape) doubles
 * (mpb_load_state: a NULL entry loads that component as all zeros, the
 * reference's fresh-run state, without a host array); m = 3*nx*ny*nz doubles. */
MPB_API int mpb_load_state(mpb_handle* h, const double* const fields[6], const double* m);
MPB_API int mpb_save_state(mpb_handle* h, double* const fields[6], double* m);

/* Advance nsteps coupled steps.  Replaces the body of sim.run's time loop
 * (sim.py:151-171).  Host buffers:
 *   src_vals[s]            source value v((n0+s+1) dt) (em.py:96-101, host)
 *   probe_out[s*n_probes+p] probe p after step n0+s (sim.py:170-171)
 *   iters_out[s]           LLG iterations r* of step n0+s (sim.py:167)
 * On an LLG failure returns MPB_ESTEP and fills *fail (step = n0+s);
 * probe/iteration rows after the failing step are unspecified, and so is the
 * device state (the reference raises mid-step too, after its non-magnetic H
 * update): reload it with mpb_load_state before running again. */
MPB_API int mpb_run(mpb_handle* h, int64_t n0, int64_t nsteps, const double* src_vals,
            double* probe_out, int32_t* iters_out, mpb_failure* fail);

/* Device-resident variant for benchmarking / chained pipelines: all three
 * buffers are DEVICE pointers on the handle's device.  The work runs on the
 * handle's stream, ordered after all work already enqueued on `stream` and
 * with `stream` ordered after it (a cudaStream_t; 0 = the legacy default
 * stream).  The call returns without synchronising; check failures with
 * mpb_check_failure. */
MPB_API int mpb_run_device(mpb_handle* h, int64_t n0, int64_t nsteps,
                   const double* d_src_vals, double* d_probe_out,
                   int32_t* d_iters_out, void* stream);

/* In-process emulation of an n-rank slab decomposition on ONE device (test
 * and validation entry point; production runs use one process per GPU and
 * NCCL).  hs[r] is rank r, created with nranks = n and an all-zero nccl_id.
 * The ranks are stepped in lockstep on one stream with exactly the kernels of
 * the NCCL path; the boundary planes move by device copies and the LLG
 * all-reduce is a kernel.  probe_out[r] receives rank r's probe rows (zeros
 * for probes it does not own); iters_out receives r* per step. */
MPB_API int mpb_group_run(mpb_handle* const* hs, int32_t n, int64_t n0, int64_t nsteps,
                          const double* src_vals, double* const* probe_out,
                          int32_t* iters_out, mpb_failure* fail);

/* Synchronise and report the first LLG failure since the last call. */
MPB_API int mpb_check_failure(mpb_handle* h, mpb_failure* fail);

/* Per-kernel device timing of the main sweep kernel(s): when enabled, each
 * launch of the dominant kernel is bracketed by CUDA events on the stream it
 * runs on (graphs are bypassed).  mpb_kernel_time returns the summed
 * milliseconds and launch count since enabling, and the name of the kernel. */
MPB_API int mpb_set_kernel_timing(mpb_handle* h, int enable);
MPB_API int mpb_kernel_time(mpb_handle* h, double* ms_total, int64_t* launches,
                    const char** kernel_name);

/* Number of kernel launches the last mpb_run / mpb_run_device enqueued. */
MPB_API int64_t mpb_launch_count(mpb_handle* h);

/* Self-test of the exact-division fast path used by the sweep kernels:
 * divides each x[q] by d on the GPU both ways (hoisted-reciprocal fast path
 * and the compiler's IEEE x/d) and counts bitwise mismatches. */
MPB_API int mpb_selftest_division(int32_t device, double d, const double* x, int64_t n,
                                  int64_t* mismatches, double* first_bad);

/* Discrete field energy of the current device state (reference
 * em.total_energy, em.py:366-383): (1/2 sum eps E^2 + 1/2 mu0 sum H^2
 * - mu0 sum M.Hbias) dV over this rank's owned planes (multi-rank: sum the
 * ranks).  Deterministic fixed-order reduction; equal to the reference to
 * rounding (summation order differs), not bitwise. */
MPB_API int mpb_total_energy(mpb_handle* h, double* out);

/* Product with the Hankel data matrix X[t][a] = x[t+a] (t < n-columns+1,
 * a < columns) of a probe series on the GPU: transpose = 0 computes
 * out (M x r) = X in (columns x r), transpose = 1 computes out (columns x r)
 * = X^T in (M x r); row-major host arrays, r <= 32.  The O(M columns r)
 * work of the subspace mode extraction (reference analysis.esprit,
 * analysis.py:64-115: SVD of the Hankel matrix), used by the randomized
 * range finder in paper_2510_22221_b200/analysis.py; deterministic. */
MPB_API int mpb_hankel_mul(int32_t device, const double* x, int64_t n, int32_t columns,
                           int32_t r, int32_t transpose, const double* in, double* out);

/* Multi-rank steps whose global residual went back above tol after the
 * last local stop and were continued in host-driven lockstep since the
 * handle was created (see mpb_failure.kind 4). */
MPB_API int64_t mpb_continued_steps(mpb_handle* h);

/* Tile form the fused sweep was set up with: out = {entries per thread,
 * threads per CTA, entries per tile, x-chunks} (zeros when the split
 * variant or the line kernel runs).  Lets a test pin the exact kernel
 * instantiation a benchmark times. */
MPB_API int mpb_sweep_form(mpb_handle* h, int32_t out[4]);

/* Device bytes held by the handle. */
MPB_API int64_t mpb_device_bytes(mpb_handle* h);

/* Rank layout of the handle as its NCCL communicator reports it
 * (ncclCommCount / ncclCommUserRank; single rank or in-process group: the
 * setup values) and the NCCL version the library runs against.  Lets a
 * multi-GPU driver prove how many ranks actually joined the exchange. */
MPB_API int mpb_comm_info(mpb_handle* h, int32_t* nranks, int32_t* rank,
                          int32_t* nccl_version);

#ifdef __cplusplus
}
#endif

#endif /* MAGPHON_B200_H */
