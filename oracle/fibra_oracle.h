/*
 * fibra_oracle.h -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE).
 *
 * This is the parity CHECKER for the B200 solver, never the product: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load it.  Every function restates one reference function in plain C99 with the
 * reference's floating-point operation order (compile with -ffp-contract=off),
 * citing the file:line it follows under /root/reference/proj.
 *
 * Pinning: oracle/_ref builds the reference's own Eigen-free translation units
 * (network.cpp relax.cpp kernels*.cpp netgen.cpp pool.cpp) and
 * tests/test_oracle_vs_ref.py checks this restatement against them bitwise
 * (topology, packed layout, DR trajectories, iteration counts, stress).
 * The Eigen-dependent pieces (polar_decompose tensor.cpp:203-224 and the 6x6
 * FullPivLU of stiffness.cpp:26-39) cannot be built here (Eigen is absent); they are
 * restated (Jacobi 3x3 eigensolver, full-pivot LU) and pinned only to the
 * reference tests' tolerances -- see DESIGN.md "Oracle".
 */
#ifndef FIBRA_ORACLE_H
#define FIBRA_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; identical numbering to include/fibra_cuda.h */
enum {
  OR_OK = 0,
  OR_CONFIG = 1,          /* ConfigError */
  OR_KINEMATICS = 2,      /* KinematicsError: det(F) <= 0 */
  OR_COLLAPSE = 3,        /* SolverError: fiber collapsed (network.cpp:291-293) */
  OR_BAD_DT = 4,          /* SolverError: bad time step (relax.cpp:151-153) */
  OR_DIVERGED = 5,        /* SolverError: non-finite residual (relax.cpp:159-161) */
  OR_NOT_CONVERGED = 6,   /* SolverError: base not converged (stiffness.cpp:75-77) */
  OR_PROBE_FAILED = 7,    /* SolverError: probe failed / not converged (stiffness.cpp:106-118) */
  OR_SINGULAR = 8,        /* SolverError: probing system singular (stiffness.cpp:33-34) */
  OR_NOT_CONVERGED_STATE = 9, /* SolverError: homogenized stress on unconverged state */
  OR_ASM_STRESS = 10,     /* SolverError: non-finite stress response (macrofem.cpp:122-125) */
  OR_ASM_RESIDUAL = 11    /* SolverError: non-finite assembled residual (macrofem.cpp:186-187) */
};

/* FiberNetwork (network.hpp:55-101) after construction (network.cpp:67-157). */
typedef struct {
  int n_nodes, n_fibers, n_free, n_boundary;
  double box_half, tol_bnd, max_ea;
  double* coords;          /* 3N node order */
  int32_t* fib_a;          /* M */
  int32_t* fib_b;          /* M */
  double* area;            /* M */
  double* modulus;         /* M */
  double* rest_length;     /* M */
  uint8_t* boundary_mask;  /* N */
  int32_t* boundary_nodes; /* B ascending */
  int32_t* packed_of_dof;  /* 3N */
  int32_t* dof_of_packed;  /* 3N */
  double* packed_ref;      /* 3N */
  int32_t* fiber_dofs;     /* 6M */
  double* node_lump;       /* N */
} or_network;

typedef struct {
  int kind;            /* 0 linear, 1 exponential (network.hpp:27-38) */
  double ea_scale;     /* 1.0 */
  double nonlinearity; /* 1.2 */
  int buckling_off;    /* 0 */
} or_law;

typedef struct {       /* RelaxConfig relax.hpp:15-26 */
  double damping, tolerance;
  int64_t max_iterations;
  double dt_safety, density_scale;
} or_relax_cfg;

typedef struct {       /* RelaxReport relax.hpp:28-36 */
  int64_t iterations;
  double residual, eps_eff, kinetic_fraction, dt;
  int32_t converged;
  double energy_drift;
} or_relax_report;

typedef struct {       /* RveStateView network.hpp:105-115 */
  double *u, *v, *a, *f_int, *f_damp, *mass, *inv_mass;
  double* t;
  int64_t* iters;
  uint8_t* converged;
  int n_free, n_dof;
} or_state;

typedef struct {       /* Response stiffness.hpp:25-33 + ResponseStats :19-23 */
  double sigma[6];     /* SymTensor3 order xx yy zz yz xz xy */
  double spatial_c[36];
  double pk2[6];
  double material_a[36];
  double stress_asymmetry;
  or_relax_report base_report;
  int32_t solves;
  int64_t relax_iterations;
  int32_t failed_probe;
} or_response;

/* ---- network ---- */
int or_network_build(const double* coords, int n_nodes, const int32_t* fib_a,
                     const int32_t* fib_b, const double* area, const double* modulus,
                     int n_fibers, double box_half, double tol_bnd, or_network* out);
void or_network_free(or_network* net);

/* ---- forces / BC / stress ---- */
int or_apply_affine_bc(const or_network* net, const double F[9], or_state st);
int or_internal_forces_cfl(const or_network* net, const or_law* law, const double* u,
                           double* f_int, const double* mred_l0, double* min_dtsq);
int or_homogenized_stress(const or_network* net, const or_state* st, const double F[9],
                          double sigma[6], double* asym);
double or_strain_energy(const or_network* net, const or_law* law, const double* u);
/* orientation_p2 (network.cpp:398-415): length-weighted P2 order parameter of the fibres
 * about ref_dir in the state u (packed DOFs) */
double or_orientation_p2(const or_network* net, const double* u, const double ref_dir[3]);

/* ---- BLAS-1 contract (kernels.hpp:8-15) ---- */
double or_norm2_sq(int64_t n, const double* x);
double or_weighted_sq(int64_t n, const double* w, const double* x);

/* ---- DR solver ---- */
int or_relax_solve(const or_network* net, const or_law* law, const double F[9],
                   const or_relax_cfg* cfg, or_state st, int warm_reuse,
                   or_relax_report* rep);

/* ---- tensor (tensor.cpp) ---- */
double or_det(const double F[9]);
int or_inverse(const double F[9], double out[9]);
void or_matmul(const double a[9], const double b[9], double out[9]);
void or_sym_full(const double s[6], double out[9]);
void or_sym_from_full(const double a[9], double s[6]);
int or_polar_decompose(const double F[9], double R[9], double U[6]);
/* Eigen 3.4.0 SelfAdjointEigenSolver<Matrix3d> restatement: 0 Success, 1 NoConvergence */
int or_eigen_sym3(const double a[9], double lam[3], double Q[9]);
/* host libm exp (which 0) / expm1 (which 1) over an array */
void or_libm(int which, const double* x, int64_t n, double* out);
int or_pull_back_stress(const double sigma[6], const double F[9], double pk2[6]);
void or_mandel(const double s[6], double v[6]);
void or_mandel_M_of_U(const double U[6], double M[36]);
void or_probing_matrix(double T[36]);
void or_probing_direction(int q, double dir[6]);
int or_push_forward_stiffness(const double A[36], const double F[9], double C[36]);
int or_material_stiffness_from_probes(const double U[6], const double base_pk2[6],
                                      const double probe_pk2[36], double h, double A[36]);

/* ---- stiffness / batch ---- */
int or_constitutive_response(const or_network* net, const or_law* law, const double F[9],
                             const or_relax_cfg* rcfg, double fd_rel_step, int reuse_warm,
                             int want_tangent, or_state st, or_response* out);
/* batch_response (batch.cpp:155-187): points solved in order; n_threads>1 uses a
   pthread pool that, like WorkerPool, only writes per-point slots (bitwise equal to
   sequential).  states are packed CRS (offsets n+1). status[p] != 0 marks a failed point. */
int or_batch_response(const or_network* const* entries, const int32_t* entry_of_point,
                      int n_points, const int64_t* offsets, double* u, double* v, double* a,
                      double* f_int, double* f_damp, double* mass, double* inv_mass, double* t,
                      int64_t* iters, uint8_t* converged, const int32_t* n_free,
                      const or_law* law, const double* F, const or_relax_cfg* rcfg,
                      double fd_rel_step, int reuse_warm, int want_tangent, int n_threads,
                      or_response* out, int32_t* status);

/* ---- macro assembly (macrofem.cpp:41-187) ---- */
int or_tet_geom(const double* coords, const int32_t n[4], double grad[12], double* volume);
void or_mandel_b(const double grad[12], double b[72]);
int or_element_matrices(const double* coords, const int32_t n[4], const double sigma[6],
                        const double c66[36], double fe[12], double ke[144]);
int or_assemble(const int32_t* tets, int32_t n_tets, const double* coords,
                const double* sigma, const double* c66, const int32_t* free_of_dof,
                int32_t n_free, const double* f_ext, double* residual, int64_t* col_ptr,
                int32_t* row_idx, double* values, int64_t cap, int64_t* nnz,
                int32_t* bad_element);

#ifdef __cplusplus
}
#endif
#endif
