/*
 * kfvm_b200.h — C-ABI of the B200-native KFVM-WENO FP64 stage update.
 *
 * This is the drop-in boundary for the hot path named by BASELINE.json
 * `north_star`: the per-RK-stage KFVM-WENO finite-volume update (kernel
 * reconstruction + WENO-AO in linearized-primitive variables, positivity
 * limiter, per-quadrature-point Riemann solve, face quadrature, SSP-RK3 stage
 * combine, CFL max-wavespeed reduction, z-slab decomposition).
 *
 * The reference has no C interface; the path sits behind two C++ APIs
 * (SURVEY.md §8(b)).  Each entry point below names the reference interface it
 * replaces (paths relative to the reference tree; S: = SPEC.md).
 *
 *   table  <- kfvm::precompute / ReconstructionSet / StencilVectors
 *             (proj/core/include/kfvm/kernel_recon.hpp:67-110)
 *   solver <- compute_rhs, ssp43_step (replaced by SSP-RK3 per
 *             BASELINE.json), select_dt, advance_to,
 *             fill_ghost, reconstruct_states
 *
 * Conventions
 *   - No exceptions cross this boundary.  Return codes mirror the reference
 *     CLI exit codes: 0 ok, 1 config error, 2 runtime abort (NaN,
 *     inadmissible average, limiter abort), 3 device / I/O / NCCL error.
 *   - The caller owns host buffers; a handle owns all device memory.
 *   - A handle is not thread-safe.  Calls are synchronous at return unless
 *     the name ends in _async.
 *   - Host state buffers use the reference AoS order: cell-major with x
 *     fastest, then y, then z; the nvar = dim+2 conservative components
 *     (rho, m_x, m_y, [m_z], E) of one cell are contiguous.
 */
#ifndef KFVM_B200_H_
#define KFVM_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KFVM_OK 0
#define KFVM_ERR_CONFIG 1
#define KFVM_ERR_RUNTIME 2
#define KFVM_ERR_DEVICE 3

/* Boundary kinds (BoundaryKind; fill_ghost).  Every
 * kind defines the value of every ghost cell (an infinite extension, so the
 * ghost cells' own reconstructions give the exterior face states):
 *   PERIODIC   wrap (sides come in pairs)
 *   OUTFLOW    zeroth-order extrapolation: the nearest interior cell
 *   REFLECTING mirror image across the wall, wall-normal momentum negated
 *   DIRICHLET  the fixed conservative state bc_state[side]
 *   SLIT       "user" inflow of S:561 / P:§6.4: bc_state[side] where the
 *              ghost cell centre lies strictly inside the slit (r^2 < radius^2
 *              in the side's tangential axes), outflow elsewhere
 * At edges and corners the per-axis maps compose in axis order x, y, z:
 * value = T_z(T_y(T_x(U[src]))), src the composed index map. */
#define KFVM_BC_PERIODIC 0
#define KFVM_BC_OUTFLOW 1
#define KFVM_BC_REFLECTING 2
#define KFVM_BC_DIRICHLET 3
#define KFVM_BC_SLIT 4

#define KFVM_RIEMANN_HLLC 0
#define KFVM_RIEMANN_HLL 1

#define KFVM_MAX_STENCILS 8

/* Immutable reconstruction table: the a1 row of SURVEY.md §8(a).
 * Replaces kfvm::ReconstructionSet / StencilVectors
 * (proj/core/include/kfvm/kernel_recon.hpp:67-101), generalised to 3-D.
 * Stencil q=0 is the full stencil S0, q=1 the central substencil, q>=2 the
 * axis-biased substencils in the order +x,-x,+y,-y(,+z,-z)
 * (§3.1; proj/core/src/geometry.cpp:22-34).
 * Face quadrature point s = face*R^(d-1) + m, faces W,E,S,N(,B,T)
 * (proj/core/include/kfvm/geometry.hpp:35-45); within a face m = a + R*b
 * with a the GL node index along the first tangential axis.            */
typedef struct kfvm_table {
  int dim;          /* 2 or 3 */
  int radius;       /* R = 2 or 3 */
  int n_stencils;   /* N_S + 1 = 2*dim + 2 */
  int n_points;     /* face quadrature points per cell = 2*dim*R^(dim-1) */
  int n_alpha;      /* derivative multi-indices 0 < |alpha| <= R */
  int n_full;       /* N_0 */
  int total_cells;  /* sum_q N_q */
  int size[KFVM_MAX_STENCILS];        /* N_q */
  int degree[KFVM_MAX_STENCILS];      /* assigned monomial degree p_q */
  int cell_offset[KFVM_MAX_STENCILS]; /* prefix sum of N_q */
  const int* offsets;  /* [n_full][3] (i,j,k) of S0, lexicographic by (k,j,i) */
  const int* gather;   /* [total_cells] position in S0 of each cell of S_q */
  const int* alpha;    /* [n_alpha][3] graded multi-indices */
  const double* face;  /* per q at cell_offset[q]*n_points: [n_points][N_q] */
  const double* deriv; /* per q at cell_offset[q]*n_alpha:  [n_alpha][N_q] */
  const double* gamma_lin;    /* [n_stencils] WENO-AO linear weights */
  const double* face_weights; /* [n_points] tensor GL weight of each point */
  const double* points;       /* [n_points][3] unit-cell coordinates */
  const double* gl_nodes;     /* [R] on [-1/2,1/2] ascending */
  const double* gl_weights;   /* [R] sum to 1 */
  double ell_over_delta;      /* KernelConfig::ell_over_delta */
  uint64_t hash;              /* FNV-1a 64 over every array above */
} kfvm_table;

/* Build the table once in extended precision (binary128 LU + refinement,
 * rounded to FP64).  Replaces kfvm::precompute (kernel_recon.hpp:107) and
 * build_stencil_geometry (geometry.hpp:75-76).  Errors: 1 for an
 * unsupported radius/dimension (geometry.cpp:11-12), 2 when a block solve's
 * residual exceeds 1e-9 (kernel_recon.hpp:56-59). */
int kfvm_table_build(int dim, int radius, double ell_over_delta, kfvm_table** out);
void kfvm_table_free(kfvm_table* t);

/* Run configuration (the solver/driver subset of RunConfig). */
typedef struct kfvm_config {
  int dim;            /* 2 or 3 */
  int radius;         /* 2 or 3 */
  int nx, ny, nz;     /* global interior cells; nz = 1 in 2-D */
  int bc;             /* KFVM_BC_PERIODIC or KFVM_BC_OUTFLOW: every side, unless
                         bc_per_side is set */
  int riemann;        /* KFVM_RIEMANN_HLLC (default) or KFVM_RIEMANN_HLL */
  double dx;          /* uniform spacing Delta (dx = dy = dz) */
  double gamma;       /* ratio of specific heats */
  double cfl;         /* CFL number of select_dt */
  double eps;         /* WENO epsilon, 1e-40 */
  double kappa;       /* positivity bound relaxation, 0.4 */
  double flattener_kf;/* flattener kappa_f, 0.33 */
  int kxrcf;          /* KXRCF troubled-cell indicator (
                         config key kxrcf.enabled): 0 = WENO in every
                         cell (default), 1 = unlimited full-stencil states with
                         WENO only in flagged cells */
  double kxrcf_m;     /* the indicator's power m on Delta (kxrcf.m), 1.5 */
  int integrator;     /* KFVM_SSPRK3 (BASELINE, default) or KFVM_SSP43: the
                         reference's SSP(4,3) with embedded SSP(3,2) and a PI
                         step-size controller, used by
                         kfvm_gpu_advance_to */
  double atol, rtol;  /* error-norm tolerances, 1e-4 */
  double safety;      /* controller safety factor, 0.9 */
  double dt_min;      /* abort below (0 = none) */
  double dt_max;      /* clamp above (0 = none) */
  /* Navier-Stokes terms (PAPER.md eqs nsVisc/shearTensor/
   * thermalFlux): face-centre second-order differences of the
   * cell-average primitives, midpoint rule per face, subtracted from the
   * face-averaged inviscid flux. */
  int viscous;        /* 0 = Euler (default), 1 = add the viscous fluxes */
  double reynolds;    /* Re */
  double prandtl;     /* Pr, 0.71 */
  double mach;        /* Ma: temperature T = gamma Ma^2 p / rho */
  /* Gravity source (PAPER.md eq rtSource): per cell
   * S = (1/Fr^2) (0, 0, rho, [0,] rho u_2) from the cell averages, added to
   * the flux divergence.  0 = no source. */
  double inv_froude2;
  /* Per-side boundary kinds (Field's "registered boundary kinds per side",
   * S:531).  Side 2*a + s: axis a = 0 (x), 1 (y), 2 (z); s = 0 low, 1 high.
   * bc_per_side = 0 (kfvm_config_defaults, or a zeroed struct): every side
   * takes `bc`, the arrays below are ignored. */
  int bc_per_side;
  int bc_side[6];           /* KFVM_BC_* per side */
  double bc_state[6][5];    /* DIRICHLET / SLIT inflow state, conservative
                               (rho, m_1..m_d, E); unused entries ignored */
  double slit_center[6][2]; /* SLIT: centre in the side's tangential axes
                               (increasing axis order), measured from the
                               domain's low corner */
  double slit_radius[6];    /* SLIT: inflow where r^2 < radius^2 */
} kfvm_config;

#define KFVM_SSPRK3 0
#define KFVM_SSP43 1

/* Fill cfg with the reference defaults for the given geometry. */
void kfvm_config_defaults(kfvm_config* cfg, int dim, int radius, int nx, int ny,
                          int nz, int bc);

/* Seeded synthetic initial conditions of BASELINE.json configs 1-5
 * (host, multithreaded).  Cell averages by the tensor R^d Gauss-Legendre
 * rule from pointwise primitives (§5.2). */
#define KFVM_IC_FOURIER 0      /* configs 1 and 3 */
#define KFVM_IC_VORONOI 1      /* configs 2 and 4 */
#define KFVM_IC_FOURIER_SPHERE 2 /* config 5 */
#define KFVM_IC_UNIFORM 3      /* free stream (rho,u,v,w,p) = params */
#define KFVM_IC_VORTEX 4       /* 2-D isentropic vortex on [-10,10]^2 */
#define KFVM_IC_DENSITY_WAVE 5 /* rho = 1 + amp*sin(2pi k.x), u = const, p = 1 */
typedef struct kfvm_ic_params {
  int kind;
  int n_modes;       /* Fourier modes per field */
  int n_regions;     /* Voronoi regions */
  uint64_t seed;
  double origin[3];  /* lower corner of the global domain */
  double value[5];   /* uniform / density-wave parameters */
} kfvm_ic_params;

/* Generate cell averages for the sub-box [z0, z0+nz_local) of the global
 * grid described by cfg into U_host (AoS, nvar per cell). */
int kfvm_ic_generate(const kfvm_config* cfg, const kfvm_ic_params* ic, int z0,
                     int nz_local, int nthreads, double* U_host);

/* ----------------------------------------------------------------------- */
/* GPU solver handle (one per GPU / rank).                                 */
typedef struct kfvm_handle kfvm_handle;

/* Multi-GPU slab decomposition (one process per GPU): the slab axis is the
 * last axis (z in 3-D, y in 2-D), split into nranks contiguous slabs.
 * nccl_id is the 128-byte ncclUniqueId produced by kfvm_nccl_unique_id on
 * rank 0 and broadcast by the caller.  Pass NULL for a single GPU. */
typedef struct kfvm_dist {
  int rank;
  int nranks;
  int device;              /* CUDA device ordinal for this rank */
  unsigned char nccl_id[128];
} kfvm_dist;

int kfvm_nccl_unique_id(unsigned char id[128]);
/* In-process loopback group id (no reference counterpart; test transport):
 * pass it as kfvm_dist.nccl_id to nranks handles created in ONE process on
 * the same device, each then driven by its own host thread like a rank.
 * Halo planes, KXRCF edge flags, the dt maximum and the SSP(4,3) error
 * planes are exchanged by device-to-device copies with NCCL's send/recv and
 * collective semantics; loopback handles run their steps eagerly (the
 * host-side rendezvous cannot be graph-captured). */
int kfvm_loopback_id(unsigned char id[128]);

/* Slab owned by `rank`: planes [*p0, *p0 + *np) of the slab axis. */
void kfvm_slab_range(int n_global, int nranks, int rank, int* p0, int* np);

/* Create the handle: uploads the table to device constant/global memory,
 * allocates the state buffers and creates streams (+ NCCL comm if dist). */
int kfvm_gpu_create(const kfvm_config* cfg, const kfvm_table* table,
                    const kfvm_dist* dist, kfvm_handle** out);
void kfvm_gpu_destroy(kfvm_handle* h);

/* State upload / readback of the rank's interior planes (AoS host).
 * Replaces Field construction / read-out. */
int kfvm_gpu_set_state(kfvm_handle* h, const double* U_host);
int kfvm_gpu_get_state(kfvm_handle* h, double* U_host);
/* Asynchronous upload / readback on the handle's stream (no host sync; the
 * host buffer must not be touched until kfvm_gpu_sync).  Pinned buffers and
 * one handle per field let the copies of one field overlap the steps of
 * another (ensemble pipelining). */
int kfvm_gpu_set_state_async(kfvm_handle* h, const double* U_host);
int kfvm_gpu_get_state_async(kfvm_handle* h, double* U_host);
/* Same on device memory (AoS, caller-owned device pointer). */
int kfvm_gpu_set_state_device(kfvm_handle* h, const double* U_dev);
int kfvm_gpu_get_state_device(kfvm_handle* h, double* U_dev);

/* KXRCF troubled-cell flags (1 = WENO) of the rank's cells for the current
 * state, AoS cell order; replaces kxrcf_flag on the path.  Requires a
 * handle created with cfg->kxrcf = 1. */
int kfvm_gpu_kxrcf_flags(kfvm_handle* h, unsigned char* flags_host);

/* One compute_rhs: dU/dt of the current state (AoS host). */
int kfvm_gpu_rhs(kfvm_handle* h, double* dUdt_host);
/* Face states after WENO-AO + positivity limiting of the current state,
 * reconstruct_states; [cell][point][var] over interior cells. */
int kfvm_gpu_states(kfvm_handle* h, double* states_host);
/* select_dt with the fixed-CFL rule of BASELINE.json:
 * dt = cfl*dx / max_cells sum_d (|u_d| + c). */
int kfvm_gpu_select_dt(kfvm_handle* h, double* dt);
/* One SSP-RK3 stage (1,2,3) with the given dt (replaces ssp43_step S:598). */
int kfvm_gpu_stage(kfvm_handle* h, int stage, double dt);
/* One SSP-RK3 step with dt selected on the device; dt_out may be NULL. */
int kfvm_gpu_step(kfvm_handle* h, double* dt_out);
/* nsteps SSP-RK3 steps (CUDA-graph captured); dt_seq[nsteps] may be NULL.
 * Replaces advance_to for a fixed step count. */
int kfvm_gpu_run(kfvm_handle* h, int nsteps, double* dt_seq);
/* advance_to: step until t = t_final (the last step is clipped to
 * land on it) or max_steps.  cfg->integrator = KFVM_SSPRK3: fixed-CFL SSP-RK3
 * steps; KFVM_SSP43: SSP(4,3) + embedded SSP(3,2) with the PI controller
 * (accept when the error norm <= 1; max_steps bounds the attempts; *steps =
 * accepted steps). */
int kfvm_gpu_advance_to(kfvm_handle* h, double t_final, int max_steps, int* steps,
                        double* t_reached);
/* Accepted and rejected steps of the last kfvm_gpu_advance_to with the
 * SSP(4,3) integrator (advance_to run statistics). */
int kfvm_gpu_step_stats(kfvm_handle* h, int* accepted, int* rejected);
/* Asynchronous variant on the handle's stream; kfvm_gpu_sync waits and
 * reports device-side errors. */
int kfvm_gpu_run_async(kfvm_handle* h, int nsteps);
int kfvm_gpu_sync(kfvm_handle* h);
/* Device dt sequence of the last run (nsteps doubles). */
int kfvm_gpu_dt_sequence(kfvm_handle* h, double* dt_seq, int nsteps);
/* The stream the handle launches on (cudaStream_t as void*). */
void* kfvm_gpu_stream(kfvm_handle* h);
/* Number of kernel launches issued by the handle so far. */
long long kfvm_gpu_launch_count(kfvm_handle* h);
/* Tuning/diagnostics: set a named integer option (e.g. "chunk_planes"). */
int kfvm_gpu_set_option(kfvm_handle* h, const char* name, long long value);
/* Per-kernel CUDA-event timing of the next run (ms summed per kernel). */
int kfvm_gpu_kernel_times(kfvm_handle* h, double* ms_states, double* ms_flux,
                          double* ms_update, double* ms_other);
int kfvm_gpu_last_error(kfvm_handle* h, char* buf, size_t n);
/* Generate the seeded IC (kinds FOURIER, VORONOI, FOURIER_SPHERE, UNIFORM)
 * directly into the handle's state on the device; bit-identical to
 * kfvm_ic_generate (the per-point arithmetic is IEEE add/mul/div only). */
int kfvm_gpu_ic_generate(kfvm_handle* h, const kfvm_ic_params* ic);

/* Diagnostics: per-phase cycle counters of the reconstruction kernels
 * (non-zero only in a -DKFVM_PHASE_TIMING build). */
int kfvm_phase_cycles(unsigned long long* out8, int reset);

/* FP64 roofline denominators measured on the current device: DFMA pipe
 * (8 independent chains per thread) and DMMA (mma.sync m8n8k4.f64). */
int kfvm_fp64_peak(double* dfma_tflops, double* dmma_tflops, double* sm_clock_ghz);

#ifdef __cplusplus
}
#endif

#endif
