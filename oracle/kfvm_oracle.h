/*
 * kfvm_oracle.h — CPU oracle of the KFVM-WENO FP64 stage update.
 *
 * TEST INFRASTRUCTURE ONLY.  This is a plain C++ restatement of the
 * reference algorithm (SPEC.md modules weno S:241-300, euler_state
 * S:302-384, limiters/positivity S:410-446, riemann S:466-519, solver
 * S:521-645; §3-§5 for 3-D) used as the parity checker by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg.
 * The product (paper_2401_16543_b200/) never links or calls it.
 *
 * Parity: the reference tree ships no tests, fixtures or golden vectors for
 * this path and does not build; the oracle is pinned by
 * the SPEC's inline known-answer examples and invariants (tests/golden/
 * spec_examples.json, tests/test_oracle_*.py) and by PAPER.md Table 1 EOCs.
 */
#ifndef KFVM_ORACLE_H_
#define KFVM_ORACLE_H_

#include "../include/kfvm_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Whole-grid operations on AoS interior state (reference layout). */
int kfo_rhs(const kfvm_config* cfg, const kfvm_table* t, const double* U,
            double* dUdt, int nthreads);
int kfo_states(const kfvm_config* cfg, const kfvm_table* t, const double* U,
               double* states, int nthreads);
int kfo_select_dt(const kfvm_config* cfg, const double* U, double* dt);
int kfo_stage(const kfvm_config* cfg, const kfvm_table* t, const double* U0,
              const double* Uk, double* Uout, int stage, double dt, int nthreads);
/* nsteps SSP-RK3 steps in place; dt_seq may be NULL.  nslabs > 1 runs the
 * virtual slab decomposition (halo copies between slabs) of SURVEY §4(iii). */
int kfo_run(const kfvm_config* cfg, const kfvm_table* t, double* U, int nsteps,
            double* dt_seq, int nslabs, int nthreads);
/* advance_to with SSP(4,3)+embedded SSP(3,2) and the PI controller
 * (S:598-616); stats = {accepted, rejected}; dt_seq = accepted dts. */
int kfo_advance43(const kfvm_config* cfg, const kfvm_table* t, double* U, double t_final,
                  int max_attempts, double* dt_seq, int cap, int* stats, double* t_reached,
                  int nthreads);
/* Same, restricted to the planes [p0, p0+np) of the slab axis of a bigger
 * global grid: one RHS (stage-1 update) of the sub-box, for timing samples. */
int kfo_sample_stage(const kfvm_config* cfg, const kfvm_table* t, const double* U,
                     int p0, int np, int nthreads, double* seconds);

/* KXRCF troubled-cell flags (1 = WENO) of every cell, and the
 * pinned power function the indicator uses (q = p / rho^gamma). */
int kfo_kxrcf_flags(const kfvm_config* cfg, const kfvm_table* t, const double* U,
                    unsigned char* flags, int nthreads);
double kfo_pow(double x, double y);
void kfo_viscous_face(const kfvm_config* cfg, const double* U, int i, int j, int k, int d,
                      double* Fv);
/* SSP(4,3)+SSP(3,2) stage combine, stage codes 11..14 (uhat written at 13). */
void kfo_combine43(int stage, long long n, const double* U0, const double* Uk, const double* L,
                   double dt, double* out, double* uhat);

/* Slab pieces for the multi-process decomposition test. */
int kfo_slab_rhs(const kfvm_config* cfg, const kfvm_table* t, int p0, int np,
                 const double* U_local, double* out, int nthreads);
/* the whole domain padded with R+1 ghost cells per side by fill_ghost */
int kfo_fill_ghost(const kfvm_config* cfg, const double* U, double* out);
double kfo_max_speed(const kfvm_config* cfg, const double* U, long long ncells);
void kfo_combine(int stage, long long n, const double* U0, const double* Uk, const double* L,
                 double dt, double* out);

/* Seeded BASELINE initial conditions (fourier / voronoi / fourier_sphere /
 * uniform), restated independently of the product generator
 * (kfvm_oracle_ic.cpp): cell averages of the slab-axis planes [z0, z0+nz),
 * AoS, x fastest. */
int kfo_ic_generate(const kfvm_config* cfg, const kfvm_ic_params* ic, int z0, int nz_local,
                    int nthreads, double* U);

/* Point functions (unit tests against the SPEC examples). */
double kfo_pressure(int dim, const double* U, double gamma);
double kfo_sound_speed(int dim, const double* U, double gamma);
void kfo_transform(int dim, const double* Uref, double gamma, double* phi,
                   double* phi_inv);
void kfo_to_recon(int dim, const double* Uref, double gamma, const double* U,
                  double* W);
void kfo_from_recon(int dim, const double* Uref, double gamma, const double* W,
                    double* U);
void kfo_riemann(int dim, int solver, int axis, const double* UL,
                 const double* UR, double gamma, double* F);
void kfo_wavespeeds(int dim, int axis, const double* UL, const double* UR,
                    double gamma, double* sl_sr_sstar);
void kfo_exact_flux(int dim, int axis, const double* U, double gamma, double* F);
/* beta/omega/WENO-AO for one scalar field on S0 (g has n_full entries). */
void kfo_weno(const kfvm_table* t, double dx, double eps, const double* g,
              double* beta, double* omega, double* values);
/* Positivity limiter on n states of one cell; nbr holds the 3^dim
 * neighbourhood averages (i fastest), nbr[(3^dim)/2] is the cell itself. */
int kfo_limit(int dim, int n, double* states, const double* nbr, double gamma,
              double kappa, double kf, double* info);

#ifdef __cplusplus
}
#endif
#endif
