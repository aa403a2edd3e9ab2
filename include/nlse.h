/*
 * nlse.h -- C ABI of libnlse_b200.so: the B200-native RK4 + CD/2SHOC time step
 * of the cubic NLSE / Gross-Pitaevskii equation (NLSEmagic, arXiv:1203.1263).
 *
 *   i Psi_t + a Lap(Psi) - V(r) Psi + s |Psi|^2 Psi = 0        (NLSE) P:76-80
 *
 * The paper's integrators take (Psi, V, a, s, h, k, scheme, BC), "simulate a
 * 'chunk' of time-steps ... and return the resulting solution Psi" (P:415,
 * P:480).  This ABI splits that call into create / set_psi / step / get_psi so
 * that Psi stays resident in HBM across chunks.
 *
 * Conventions for every function:
 *   - Plain C types; no torch or CUDA types in signatures (streams are void*).
 *   - Grid layout: x fastest, offset(i,j,k) = (k*ny + j)*nx + i;
 *     unused dims are 1.  Complex values are interleaved (re, im) pairs.
 *   - Host Psi buffers are always double (numpy complex128 layout).  fp32
 *     contexts round once with round-to-nearest on input (as the paper's single
 *     precision MEX codes cast their input) and widen exactly on output.
 *   - All buffers passed in are caller-owned; the library copies at the call and
 *     keeps no pointer.  The context owns all device memory it allocates.
 *   - Return value: NLSE_OK (0) or an error status; nlse_last_error() gives a
 *     message.  A CUDA error is sticky: the context then returns NLSE_ERR_CUDA
 *     from every call except nlse_destroy / nlse_last_error.
 *   - Calls are synchronous at return (the device work they enqueue has
 *     completed), except where noted.  One context per host thread.
 *   - There is no CPU fallback: without a CUDA device nlse_create returns
 *     NLSE_ERR_CUDA.
 */
#ifndef NLSE_B200_H
#define NLSE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NLSE_ABI_VERSION 1

typedef struct nlse_ctx nlse_ctx;   /* opaque */

typedef enum {
    NLSE_OK = 0,
    NLSE_ERR_ARG = 1,       /* invalid argument (message names it) */
    NLSE_ERR_UNSTABLE = 2,  /* k above the linear stability bound, see nlse_stability_bound */
    NLSE_ERR_OOM = 3,       /* device allocation failed */
    NLSE_ERR_CUDA = 4,      /* CUDA error or no device (sticky) */
    NLSE_ERR_COMM = 5,      /* multi-GPU communication error */
    NLSE_ERR_DIVERGED = 6   /* a non-finite Psi appeared; the first step index is in nlse_last_error */
} nlse_status;

/* Boundary conditions, section "Boundary conditions" P:303-357.
 *   DIRICHLET: Psi_b = B fixed (BCDdef) P:310-313, dPsi_b/dt = 0 (BCDdt) P:315-318,
 *              Laplacian form (BCDlap) P:320-323 for 2SHOC.
 *   MSD:       |Psi_b|^2 = B fixed (BCMSDdef) P:326-329, time-derivative form (msd)
 *              P:331-335, Laplacian form (BCMSDlap) P:336-344.
 *   L0:        Laplacian zero: dPsi_b/dt = i(s|Psi_b|^2 - V_b)Psi_b (BCL0dt) P:347-350,
 *              Lap Psi_b = 0 (BCL0lap) P:352-355 (reading R-L0).            */
typedef enum { NLSE_BC_DIRICHLET = 0, NLSE_BC_MSD = 1, NLSE_BC_L0 = 2 } nlse_bc;

/* Laplacian: CD = 2nd-order central differences; 2SHOC = the 4th-order
 * two-step compact scheme (2shoc1d)-(3d2shocs2) P:195-299.                          */
typedef enum { NLSE_CD2 = 2, NLSE_2SHOC4 = 4 } nlse_order;

/* Working precision of the whole run: complex float or double. */
typedef enum { NLSE_FP32 = 4, NLSE_FP64 = 8 } nlse_precision;

enum {
    NLSE_FLAG_FORCE_DT = 1u,          /* allow k above the linear bound */
    NLSE_FLAG_GENERIC_KERNELS = 2u    /* use the one-thread-per-point kernels everywhere
                                         (second GPU implementation, for tests) */
};

/* Create a context for an ndim-dimensional grid of dims[0] x dims[1] x dims[2]
 * points (nx, ny, nz; dims beyond ndim must be 1), spacing h (same in every
 * direction), coefficients a > 0 and s.
 *   V:  host array of prod(dims) doubles, x fastest, or NULL for V = 0 (no V
 *       array is stored and no V bytes are moved).  Copied (rounded to the
 *       working precision) at the call.
 * Errors: NLSE_ERR_ARG if ndim not in {1,2,3}, an active dim < 3, an inactive
 * dim != 1, h <= 0, a <= 0, s or V not finite, or an unknown enum;
 * NLSE_ERR_CUDA if no CUDA device; NLSE_ERR_OOM.  *out is NULL on error. */
nlse_status nlse_create(int ndim, const int64_t dims[3], double h, double a, double s,
                        const double *V, nlse_bc bc, nlse_order order, nlse_precision prec,
                        uint32_t flags, nlse_ctx **out);

/* Upload Psi: host array of 2*prod(dims) doubles (re, im interleaved). */
nlse_status nlse_set_psi(nlse_ctx *ctx, const double *psi);
/* Download Psi into a caller-owned host array of 2*prod(dims) doubles. */
nlse_status nlse_get_psi(nlse_ctx *ctx, double *psi_out);

/* Device-side I/O (for torch-owned tensors): d_psi points to prod(dims)
 * interleaved complex values of the WORKING precision (float2 / double2) in
 * device memory, x fastest.  Copies device-to-device on the context stream. */
nlse_status nlse_set_psi_device(nlse_ctx *ctx, const void *d_psi);
nlse_status nlse_get_psi_device(nlse_ctx *ctx, void *d_psi);

/* Advance Psi by nsteps classic RK4 steps of size k ((RK4) P:164-180, computed
 * in the paper's GPU form (RK4_GPU) P:495-519: four fused stage kernels per
 * step with the Psi_tmp / Psi_out ping-pong).  Psi stays on the device.
 * nsteps = 0 is a no-op.  Errors: NLSE_ERR_ARG (k not finite or <= 0,
 * nsteps < 0); NLSE_ERR_UNSTABLE if k exceeds the linear bound of
 * nlse_stability_bound and NLSE_FLAG_FORCE_DT was not given; NLSE_ERR_DIVERGED
 * if Psi became non-finite (checked once per step inside the last stage
 * kernel; the state is left as computed; the report is sticky -- later steps
 * return it again -- until Psi is replaced by nlse_set_psi / nlse_set_psi_device).
 * Results are bitwise independent of how a run is split into nlse_step calls
 * (chunk invariance). */
nlse_status nlse_step(nlse_ctx *ctx, double k, int64_t nsteps);

/* ---------------------------------------------------------------- slab mode (§8(e))
 * A 3D grid partitioned into contiguous z slabs (a 2D grid into y-row slabs, a 1D grid into
 * x segments),
 * one per rank (one GPU per process, or several "virtual ranks" in one process).  Rank r
 * owns global planes (rows) [z0, z0 + nloc) of nlse_slab_range over nz (ny).  Buffers read
 * with a halo carry w ghost planes (rows) on each side (w = 1 CD, 2 2SHOC); every stage
 * kernel stores the outputs of its first / last w planes (rows) also into the neighbours'
 * ghosts over peer memory (NVLink P2P through CUDA IPC), and a device-side neighbour
 * barrier separates the stages.  Results are bitwise identical to the single-GPU run.
 *
 * In slab mode nlse_set_psi*, nlse_step and nlse_diagnostics are COLLECTIVE: every
 * rank calls them in the same order (like NCCL collectives).  Psi / V host buffers
 * hold the local slab (nloc planes / rows / points).  The 3D temporally blocked CD path (two
 * stages per pass), the 1D persistent CTA and the 2D cooperative stepper are single-GPU only;
 * slab contexts use one pass per stage. */
#define NLSE_MAX_RANKS 16
#define NLSE_DIST_HANDLE_BYTES 512

/* Balanced split of nz planes (ny rows in 2D, nx points in 1D) over nranks: rank r gets
 * nz/nranks, +1 for the first nz % nranks ranks, starting at *z0.  Host only. */
nlse_status nlse_slab_range(int64_t nz, int nranks, int rank, int64_t *z0, int64_t *nloc);

/* Create the slab context of `rank`: dims are the GLOBAL grid; the slab axis is the slowest
 * one (z in 3D, y in 2D, x in 1D); V_local is the rank's slab of V or NULL.  Errors as
 * nlse_create, plus NLSE_ERR_ARG if a slab has fewer than 2w planes / rows / points or
 * rank/nranks are out of range. */
nlse_status nlse_create_dist(int ndim, const int64_t dims[3], double h, double a, double s,
                             const double *V_local, nlse_bc bc, nlse_order order,
                             nlse_precision prec, uint32_t flags, int rank, int nranks,
                             nlse_ctx **out);
/* Write this rank's NLSE_DIST_HANDLE_BYTES-byte handle (CUDA IPC handles of its halo'd
 * buffers and comm block) into `handle`; the caller exchanges them (e.g. an
 * all-gather over torch.distributed). */
nlse_status nlse_dist_export(nlse_ctx *ctx, void *handle);
/* Map the peers: `handles` = nranks handles in rank order (this rank's included).
 * NLSE_ERR_COMM if a handle is malformed or cannot be opened. */
nlse_status nlse_dist_connect(nlse_ctx *ctx, const void *handles);
/* Virtual ranks: connect the n slab contexts of ONE process (ranks 0..n-1 in order, all
 * created on the same device; NLSE_ERR_ARG otherwise).  They share one stream; drive them
 * with the _group calls below. */
nlse_status nlse_dist_connect_local(nlse_ctx *const *ctxs, int n);
/* Give up on a slab-mode job: set the abort flag in every rank's comm block (this rank's and
 * the mapped peers'), so that ranks waiting at a neighbour barrier stop waiting; their next
 * nlse_step / nlse_diagnostics returns NLSE_ERR_COMM, and so does every later call on this
 * context.  A rank that waits longer than NLSE_BARRIER_TIMEOUT_S seconds (environment at
 * nlse_create_dist, default 60) for a neighbour also stops and reports NLSE_ERR_COMM instead of
 * hanging.  Safe to call while another thread is blocked in nlse_step on the same context. */
nlse_status nlse_dist_abort(nlse_ctx *ctx);
/* nlse_step / nlse_diagnostics over a group of contexts driven by one host thread
 * (work is enqueued interleaved per stage; mass[j], hamiltonian[j] per context, all
 * equal in slab mode). */
nlse_status nlse_step_group(nlse_ctx *const *ctxs, int n, double k, int64_t nsteps);
nlse_status nlse_diagnostics_group(nlse_ctx *const *ctxs, int n, double *mass, double *hamiltonian);

/* The paper's frames model: nframes chunks of `chunk` RK4 steps; after
 * each chunk Psi (widened to double) is written to frames + f * 2*prod(dims) (caller-owned
 * host buffer of nframes * 2*prod(dims) doubles; pinned memory gives full PCIe speed).  The
 * download of frame f runs on a copy stream from a device snapshot (two, double-buffered)
 * and overlaps the compute of chunk f+1.  Frames are bitwise what nlse_step(k, chunk) +
 * nlse_get_psi would return.  Errors as nlse_step; NLSE_ERR_OOM if the two snapshots
 * (2 x 16 bytes per point) do not fit.  Slab mode: collective, frames of the local slab. */
nlse_status nlse_run_frames(nlse_ctx *ctx, double k, int64_t chunk, int nframes, double *frames);

/* Mass M = h^d sum |Psi|^2 and Hamiltonian
 *   H = h^d sum_p [ a sum_axes |Psi_{p+e} - Psi_p|^2 / h^2 + V_p |Psi_p|^2 - (s/2) |Psi_p|^4 ]
 * (forward differences over pairs inside the grid; reading R-DIAG;
 * north_star (c)).  Accumulated in fp64 with warp-shuffle + block reductions and
 * a fixed-order final pass (deterministic).  Slab mode: global sums (per-rank partials
 * exchanged over peer memory and added in rank order; collective). */
nlse_status nlse_diagnostics(nlse_ctx *ctx, double *mass, double *hamiltonian);

/* Linear stability bounds (stblincd) P:363-367 / (stblin2shoc) P:368-372:
 *   CD:    k_max = h^2 / (d sqrt(2) a);   2SHOC: k_max = (3/4) h^2 / (d sqrt(2) a)
 * and the drivers' recommended k_rec = 0.8 k_max.  No context or device needed. */
nlse_status nlse_stability_bound(int ndim, double a, double h, nlse_order order,
                                 double *k_max, double *k_rec);

/* Message describing the last error on ctx (or the last nlse_create failure
 * when ctx is NULL).  Valid until the next call on the same context. */
const char *nlse_last_error(const nlse_ctx *ctx);
const char *nlse_status_string(nlse_status st);

/* Free all device memory of the context.  NULL is allowed. */
void nlse_destroy(nlse_ctx *ctx);

/* ---------------------------------------------------------------- measurement */

/* The CUDA stream (cudaStream_t) the context launches on, as void*. */
nlse_status nlse_get_stream(nlse_ctx *ctx, void **stream);

/* Per-kernel timing: when enabled, nlse_step brackets every kernel launch with
 * CUDA events on the context stream and accumulates device time per kernel
 * kind.  Adds one event pair per launch; off by default. */
nlse_status nlse_set_timing(nlse_ctx *ctx, int enable);

#define NLSE_MAX_KINDS 12
typedef struct {
    int n_kinds;
    char name[NLSE_MAX_KINDS][48];       /* kernel kind, e.g. "stage3d_stream" */
    double ms[NLSE_MAX_KINDS];           /* accumulated device milliseconds */
    int64_t launches[NLSE_MAX_KINDS];    /* accumulated launch count */
    int64_t points[NLSE_MAX_KINDS];      /* accumulated grid points processed */
} nlse_timing;
nlse_status nlse_get_timing(nlse_ctx *ctx, nlse_timing *out);
nlse_status nlse_reset_timing(nlse_ctx *ctx);

typedef struct {
    int64_t points;            /* prod(dims) */
    int64_t launches_per_step; /* kernel launches per RK4 step (0: 1D grids run all steps of an
                                  nlse_step call in one persistent launch) */
    int64_t min_bytes_per_step;/* algorithmic HBM bytes per RK4 step, (16c + 4 r_V) * points */
    int64_t device_bytes;      /* device memory held by the context */
    int elem_bytes;            /* sizeof(real): 4 or 8 */
    char variant[64];          /* kernel family used for the interior */
    int rank, nranks;          /* slab mode (0, 1 otherwise) */
    int64_t z0, nz_local;      /* owned global planes (2D: rows, 1D: points) [z0, z0 + nz_local) */
} nlse_info;
nlse_status nlse_get_info(nlse_ctx *ctx, nlse_info *out);

#ifdef __cplusplus
}
#endif
#endif /* NLSE_B200_H */
