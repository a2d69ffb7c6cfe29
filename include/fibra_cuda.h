/*
 * fibra_cuda.h -- C-ABI of the B200-native batched fiber-network RVE solver.
 *
 * This is the drop-in boundary under the reference's batched-RVE interface
 *   fibra::batch_response(const RveLibrary&, const BatchAssignment&, PackedStates&,
 *                         const FiberLaw&, std::span<const Def3>, const RelaxConfig&,
 *                         const StiffnessConfig&, WorkerPool&)
 *   (/root/reference/proj/include/fibra/batch.hpp:71-77, body src/batch.cpp:155-187).
 * Plain C: POD structs, int status codes, no exceptions and no torch types cross it.
 * One context per host thread; calls on a context are serialized.
 * The C++ shim that re-creates fibra::batch_response on top of this header is
 * include/fibra_b200/batch_response.hpp; the ctypes binding is paper_2306_09427_b200/_capi.py.
 */
#ifndef FIBRA_CUDA_H
#define FIBRA_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (per point and per call) ----------------------------------------
 * Reference exception taxonomy (error.hpp:8-28) mapped to codes:                      */
#define FIBRA_OK 0
#define FIBRA_E_CONFIG 1          /* ConfigError (propagates out of batch_response)    */
#define FIBRA_E_KINEMATICS 2      /* KinematicsError: det(F) <= 0 (network.cpp:255)    */
#define FIBRA_E_COLLAPSE 3        /* SolverError: fiber collapse (network.cpp:291-293) */
#define FIBRA_E_BAD_DT 4          /* SolverError: bad time step (relax.cpp:151-153)    */
#define FIBRA_E_DIVERGED 5        /* SolverError: non-finite residual (relax.cpp:159)  */
#define FIBRA_E_NOT_CONVERGED 6   /* SolverError: base not converged (stiffness.cpp:75)*/
#define FIBRA_E_PROBE_FAILED 7    /* SolverError: probe q failed (stiffness.cpp:106-118)*/
#define FIBRA_E_SINGULAR 8        /* SolverError: [M][T] singular (stiffness.cpp:33)   */
#define FIBRA_E_ASM_STRESS 10     /* SolverError: non-finite stress response (macrofem.cpp:122-125) */
#define FIBRA_E_ASM_RESIDUAL 11   /* SolverError: non-finite assembled residual (macrofem.cpp:186-187) */
#define FIBRA_E_CUDA 20           /* CUDA runtime error (call-level)                   */
#define FIBRA_E_ARG 21            /* bad argument / call order (call-level)            */
#define FIBRA_E_IO 22             /* IoError (network files)                           */

/* ---- host-side network construction (product mirror of network.cpp / netgen.cpp) --- */
typedef struct fibra_network fibra_network; /* immutable FiberNetwork (network.hpp:55-101) */

typedef struct {          /* NetGenSpec netgen.hpp:16-33 (defaults in comments)      */
  int32_t style;          /* 0 segments, 1 knn                                       */
  int32_t fibers;         /* 200 */
  int32_t nodes;          /* 60, knn only */
  double half_length;     /* 0.3, segments only */
  double merge_radius;    /* 0.05 */
  int32_t neighbors;      /* 8 */
  double align_bias;      /* 0 */
  double align_axis[3];   /* {1,0,0} */
  double fiber_area;      /* 1 */
  double fiber_modulus;   /* 1 */
  double box_half;        /* 0.5 */
  double tol_bnd;         /* 1e-6 */
} fibra_netgen_spec;

/* Views into a network's storage: exactly the derived arrays the reference
 * fibra::FiberNetwork exposes, so the reference-side shim fills it from its own object. */
typedef struct {
  int32_t n_nodes, n_fibers, n_free, n_boundary; /* n_free = free DOFs (DofMap::n_free) */
  const double* coords;            /* 3N node order       FiberNetwork::coords()        */
  const int32_t* fiber_nodes;      /* 2M (a,b)            fibers()[f].a/.b              */
  const double* fiber_area;        /* M                   fibers()[f].area              */
  const double* fiber_modulus;     /* M                   fibers()[f].modulus           */
  const int32_t* packed_of_dof;    /* 3N                  dof_map().packed_of_dof       */
  const double* packed_ref;        /* 3N packed order     packed_ref_coords()           */
  const int32_t* fiber_packed_dofs;/* 6M                  fiber_packed_dofs()           */
  const double* rest_length;       /* M                   rest_lengths()                */
  const double* node_lump;         /* N node order        node_lumping()                */
  const int32_t* boundary_nodes;   /* B ascending         boundary_nodes()              */
  double box_half;                 /*                     box().half                    */
  double max_ea;                   /*                     max_ea()                      */
} fibra_net_desc;

int fibra_network_create(const double* coords, int32_t n_nodes, const int32_t* fiber_nodes,
                         const double* area, const double* modulus, int32_t n_fibers,
                         double box_half, double tol_bnd, fibra_network** out);
int fibra_network_generate(const fibra_netgen_spec* spec, uint64_t seed, fibra_network** out);
int fibra_network_read(const char* path, double box_half, double tol_bnd, fibra_network** out);
/* Builder-side jittered lattice (no reference generator exists for config-4 sizes, SURVEY
 * 8d): n_side^3 nodes, face nodes exactly on the box faces, every axis bond plus seeded face
 * diagonals up to `fibers`; constructed like a file read (write it with
 * fibra_network_write to obtain the reference file format). */
int fibra_network_generate_lattice(int32_t n_side, int32_t fibers, double jitter, double area,
                                   double modulus, double box_half, double tol_bnd,
                                   uint64_t seed, fibra_network** out);
int fibra_network_write(const fibra_network* net, const char* path);
int fibra_network_describe(const fibra_network* net, fibra_net_desc* out);
void fibra_network_free(fibra_network* net);
const char* fibra_host_last_error(void);
/* init_batch random policy (batch.cpp:101-104): entry_of_point[p] = mt19937_64(seed)() % n */
int fibra_assign_random(uint64_t seed, int32_t n_points, int32_t n_entries, int32_t* out);
/* Diagnostics: quality of the bank-aware slot schedule (csrc/host/schedule.cpp) of one
 * network for a kernel shape (T threads, FPT fibers and NPT nodes per thread).
 * out[7] = {fits, conflicting fiber groups, gather excess wavefronts, gather steps,
 *           g*d records, node slots, store excess wavefronts}. */
int fibra_schedule_report(const fibra_net_desc* net, int T, int FPT, int NPT, int64_t* out);
/* Diagnostics: that schedule's node slot placement, pn_of_slot[cap] (-1 = empty slot). */
int fibra_schedule_slots(const fibra_net_desc* net, int T, int FPT, int NPT, int32_t* pn_of_slot,
                         int32_t cap);
/* Diagnostics: the cluster partition (csrc/host/cluster_schedule.cpp) of one network over C
 * CTAs of shape (T, FPT, NPT).  out[8] = {fits, max fibers per CTA, min fibers per CTA, max
 * node slots, max halo nodes, max records, max halo copies of a node, cross-CTA fibers}. */
int fibra_cluster_report(const fibra_net_desc* net, int C, int T, int FPT, int NPT, int64_t* out);
/* Diagnostics (no CUDA): one cluster-kernel force pass emulated on the host from the
 * uploaded per-CTA arrays (f_emul) vs direct assembly (f_direct); u, f over 3 n_nodes packed
 * dofs.  shape indexes the cluster shapes. */
int fibra_debug_cluster_forces(const fibra_net_desc* net, int C, int shape, int mirror,
                               const double* u, double* f_emul, double* f_direct);
int fibra_debug_resident_forces(const fibra_net_desc* net, int shape, const double* u,
                                double* f_emul, double* f_direct);
/* Diagnostics (no CUDA): one node-centric force pass (csrc/dr_node.cuh) emulated on the host
 * from the uploaded incidence tables, linear law with ea_scale 1, f_emul in packed order;
 * report[4] = {half-warp gather steps, excess bank wavefronts before / after the placement
 * search, incidence rows}.  shape indexes the node shapes. */
int fibra_debug_node_forces(const fibra_net_desc* net, int shape, const double* u,
                            double* f_emul, int64_t* report);
/* Diagnostics (no CUDA): out[4] = {plan found, mirror mode, dynamic shared bytes, static
 * control-block bytes} of the cluster plan of `net` on C CTAs of cluster shape `shape`. */
int fibra_debug_cluster_smem(const fibra_net_desc* net, int C, int shape, int64_t* out);

/* ---- solver configuration records ------------------------------------------------- */
typedef struct {          /* FiberLaw network.hpp:27-38                              */
  int32_t kind;           /* 0 linear, 1 exponential                                 */
  double ea_scale;        /* 1.0 */
  double nonlinearity;    /* 1.2 */
  int32_t buckling_off;   /* 0 */
} fibra_law;

typedef struct {          /* RelaxConfig relax.hpp:15-26                             */
  double damping;         /* 2.0 */
  double tolerance;       /* 1e-6 */
  int64_t max_iterations; /* 500000 */
  double dt_safety;       /* 0.8 */
  double density_scale;   /* 1.0 */
  int32_t energy_check;   /* must be 0 on the device path (verification-only feature) */
} fibra_relax_cfg;

typedef struct {          /* StiffnessConfig stiffness.hpp:12-17                     */
  double fd_rel_step;     /* 1e-5 */
  int32_t reuse_warm;     /* 1 */
} fibra_stiff_cfg;

typedef struct {          /* RelaxReport relax.hpp:28-36                             */
  int64_t iterations;
  double residual, eps_eff, kinetic_fraction, dt;
  int32_t converged;
  int32_t reserved0;      /* explicit padding, always 0 (records compare bytewise)   */
  double energy_drift;
} fibra_relax_report;

typedef struct {          /* PointResponse macrofem.hpp:48-51 + Response/ResponseStats
                             stiffness.hpp:19-33; SymTensor3 order xx,yy,zz,yz,xz,xy;
                             Mandel66 row-major                                        */
  double sigma[6];
  double spatial_c[36];
  double pk2[6];
  double material_a[36];
  double stress_asymmetry;
  fibra_relax_report base_report;
  int32_t solves;
  int32_t reserved1;      /* explicit padding, always 0                              */
  int64_t relax_iterations;
  int32_t failed_probe;
  int32_t status;         /* FIBRA_OK or the point's failure code                    */
} fibra_point_result;

typedef struct {          /* per-call counters for reporting                         */
  int64_t solves;         /* DR solves run (base + probes)                           */
  int64_t iterations;     /* sum of DR iterations over all solves                    */
  int64_t fiber_iterations;  /* sum over solves of iterations * n_fibers             */
  int64_t pipe_ops;       /* sum over solves of iterations * W_pipe(net)             */
  float dr_kernel_ms;     /* device time of the persistent DR kernel                 */
  float total_ms;         /* device time of the whole solve (prep + DR + post)       */
  int32_t kernel_launches;
  int64_t alg_flops;      /* sum over solves of iterations * F_alg(net), F_alg = 28 M +
                             12 n_free + 2 n_fix (div/sqrt count 1)         */
} fibra_solve_stats;

/* ---- device context ----------------------------------------------------------------- */
typedef struct fibra_ctx fibra_ctx;

int fibra_cuda_open(int device, fibra_ctx** out);
/* One context over several GPUs of this process (the reference's single-process
 * batch_response, batch.cpp:155-187, on 1/2/4/8 B200).  The library is replicated on every
 * device; bind_points splits the points into per-device shards by longest-processing-time
 * on the per-point cost (fibra_plan_shards: the entry's topology cost at bind time, the
 * caller's FIBRA_SCHED_HINT costs afterwards -- a new hint re-plans and moves the warm
 * states of the points that change device); every call solves the shards concurrently and
 * returns the 760-byte records with ONE ncclAllGather over NVLink (NCCL loaded at run time)
 * plus a permutation into point order on the first device.  All other calls behave as on
 * a single-device context; F_dev / out_dev of solve_device live on devices[0]. */
int fibra_cuda_open_devices(const int32_t* devices, int32_t n_dev, fibra_ctx** out);
/* Host only: devices of n points by longest-processing-time on cost[] (descending cost,
 * each point to the least-loaded device, ties to the lower index; deterministic). */
int fibra_plan_shards(const double* cost, int32_t n, int32_t n_dev, int32_t* dev_of_point);
/* Host only: the schedule cost model's work estimate of one network, exp(log iterations)
 * x fibres, with the topology term of the input-only model. */
int fibra_network_cost(const fibra_net_desc* net, double* cost);
int fibra_cuda_close(fibra_ctx* ctx);
const char* fibra_cuda_last_error(const fibra_ctx* ctx);
/* use an external cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream); NULL = own */
int fibra_cuda_set_stream(fibra_ctx* ctx, void* cuda_stream);

/* RveLibrary entries (batch.hpp:33-49): topology to HBM, batched SoA + per-node CSR. */
int fibra_cuda_upload_library(fibra_ctx* ctx, const fibra_net_desc* entries, int32_t n);

/* BatchAssignment (batch.hpp:53-55): allocates the device PackedStates, zero-filled like
 * init_batch (batch.cpp:125-143); offsets are the prefix sums of 3*n_nodes. */
int fibra_cuda_bind_points(fibra_ctx* ctx, const int32_t* entry_of_point, int32_t n_points);
int fibra_cuda_reset_states(fibra_ctx* ctx);

/* Order in which the persistent kernel starts base solves (probes always follow base
 * completion).  Results are independent of it (every solve is computed bit-identically
 * wherever it runs); only the batch makespan changes.  The reference's WorkerPool takes
 * points in index order (batch.cpp:160-186), which is FIBRA_SCHED_BATCH.
 *   FIBRA_SCHED_STRAIN (default): descending input-only cost estimate, log iterations ~
 *     7.2 (share of nodes with <= 2 fibres) - 3.3 (fibres per node) + 1.75 log(fibres)
 *     - 0.37 log |F^T F - I| -- floppy and small-strain networks relax longest (for one
 *     network topology: ascending strain);
 *   FIBRA_SCHED_HINT: descending caller cost (e.g. the previous call's relax_iterations
 *     per point, n_points values, copied); cleared by fibra_cuda_bind_points. */
enum { FIBRA_SCHED_BATCH = 0, FIBRA_SCHED_STRAIN = 1, FIBRA_SCHED_HINT = 2 };

/* Diagnostics: the kernel shape library entry `entry` was assigned by upload_library.
 * out[4] = {cluster size C (1: resident one-CTA kernel), threads per CTA, fibers per
 * thread, nodes per thread}.  RVEs beyond one CTA's shared memory (about 1.3k fibers) run
 * on a thread-block cluster of C = 2..16 CTAs (csrc/dr_cluster.cuh). */
int fibra_cuda_entry_kernel(const fibra_ctx* ctx, int32_t entry, int32_t* out);

/* orientation_p2 (network.cpp:398-415; NetworkBatchProvider::orientation, batch.cpp:
 * 296-302) of the device-resident state u of `points`, about ref_dir[3]: the length-
 * weighted P2 order parameter of the fibres, in the reference's summation order. */
int fibra_cuda_orientation(fibra_ctx* ctx, const int32_t* points, int32_t n,
                           const double* ref_dir, double* out);
int fibra_cuda_set_schedule(fibra_ctx* ctx, int32_t mode, const double* cost_hint);
/* Warm data host->device: u (total dofs), t, iters, converged (n_points); any may be NULL */
int fibra_cuda_upload_states(fibra_ctx* ctx, const double* u, const double* t,
                             const int64_t* iters, const uint8_t* converged);
/* Device->host writeback of PackedStates; any pointer may be NULL to skip that array. */
int fibra_cuda_download_states(fibra_ctx* ctx, double* u, double* v, double* a, double* f_int,
                               double* f_damp, double* mass, double* inv_mass, double* t,
                               int64_t* iters, uint8_t* converged);

/* batch_response: F (n x 9 row-major Def3) in, one result record per point out.
 * want_tangent = 1: 1 base + 6 probe solves per point (constitutive_response,
 * stiffness.cpp:153-175); 0: base solve only (stress).  Host pointers; blocks. */
int fibra_cuda_solve(fibra_ctx* ctx, const double* F, const fibra_law* law,
                     const fibra_relax_cfg* relax, const fibra_stiff_cfg* stiff,
                     int32_t want_tangent, fibra_point_result* out);
/* Same with F and out already in device memory; asynchronous on the context stream. */
int fibra_cuda_solve_device(fibra_ctx* ctx, const double* F_dev, const fibra_law* law,
                            const fibra_relax_cfg* relax, const fibra_stiff_cfg* stiff,
                            int32_t want_tangent, fibra_point_result* out_dev);
int fibra_cuda_synchronize(fibra_ctx* ctx);
/* counters of the last solve (synchronizes) */
int fibra_cuda_last_stats(fibra_ctx* ctx, fibra_solve_stats* out);
int fibra_cuda_device_count(int* n);
/* Diagnostics: the exponential law's expm1 (which = 1) / exp (which = 0) on the device
 * (csrc/libm_glibc.cuh, the host libm's operation sequences) for n host operands. */
int fibra_cuda_eval_libm(fibra_ctx* ctx, int32_t which, const double* x, int64_t n, double* out);
/* FP64-pipe roofline denominator measured on this device: independent DADD chains on every
 * SM; returns lane-operations per second (one DADD/DMUL/DFMA lane = 1 op). */
int fibra_cuda_fp64_peak(fibra_ctx* ctx, double* lane_ops_per_s);
/* Self-test: the DR kernel's branch-free division / square root (csrc/fastmath.cuh) against
 * the built-in IEEE operators on n pseudo-random operand pairs; counts bit mismatches. */
int fibra_cuda_selftest_fastmath(fibra_ctx* ctx, uint64_t n, uint64_t seed, uint64_t* mismatches);
/* Diagnostics: with FIBRA_PHASE_PROF set in the environment, the last solve accumulated
 * per-warp cycles [fiber work, barrier 1, node work, barrier 2] for every CTA. */
int fibra_cuda_phase_profile(fibra_ctx* ctx, unsigned long long* out, size_t cap, size_t* n);
/* Diagnostics: with FIBRA_TRACE set at solve time, per solve {start ns, end ns,
 * sm << 32 | block, iterations} of the last solve call (solve index layout of the results). */
int fibra_cuda_trace(fibra_ctx* ctx, unsigned long long* out, size_t cap, size_t* n);

/* ---- macro assembly (csrc/assembly.cu) ---------------------------------
 * Replaces fibra::assemble(const MacroMesh&, const DofNumbering&, std::span<const
 * PointResponse>, const Eigen::VectorXd& f_ext_free)  (macrofem.hpp:77-79, body
 * macrofem.cpp:104-187).  The mesh topology and DofNumbering (macrofem.hpp:29-33) fix the
 * sparsity pattern, so it is planned once: assembly_create takes tets[4 n_tets] (node ids),
 * free_of_dof[3 n_nodes] (-1 = constrained) and n_free.  Each assemble call then takes the
 * current coords[3 n_nodes], one response record per tet (sigma as SymTensor3 xx,yy,zz,yz,
 * xz,xy followed by the Mandel66 spatial_c row-major: 42 doubles at the start of every
 * record; response_stride in doubles = 42 for a PointResponse array, sizeof(
 * fibra_point_result)/8 for solve results) and f_ext_free[n_free] (NULL = zero), and
 * returns residual[n_free] = f_int - f_ext and the nnz values of Assembly::stiffness in
 * Eigen's compressed column-major order (assembly_pattern: col_ptr[n_free+1], row_idx[nnz],
 * rows ascending per column) -- bit-identical to the reference's setFromTriplets result.
 * Errors: FIBRA_E_ASM_STRESS / FIBRA_E_KINEMATICS with *bad_element = the first failing
 * element in element order (the reference's exception), then FIBRA_E_ASM_RESIDUAL. */
typedef struct fibra_assembly fibra_assembly;
int fibra_cuda_assembly_create(int device, const int32_t* tets, int32_t n_tets, int32_t n_nodes,
                               const int32_t* free_of_dof, int32_t n_free, fibra_assembly** out);
int fibra_cuda_assembly_set_stream(fibra_assembly* as, void* cuda_stream);
int fibra_cuda_assembly_pattern(const fibra_assembly* as, int64_t* nnz, int64_t* col_ptr,
                                int32_t* row_idx);
/* host buffers in and out; blocks */
int fibra_cuda_assemble(fibra_assembly* as, const double* coords, const double* responses,
                        int64_t response_stride, const double* f_ext_free, double* residual,
                        double* values, int32_t* bad_element);
/* device buffers (e.g. the out_dev of fibra_cuda_solve_device); asynchronous on the
 * assembly's stream -- fibra_cuda_assembly_status synchronizes and reports errors */
int fibra_cuda_assemble_device(fibra_assembly* as, const double* coords_dev,
                               const double* responses_dev, int64_t response_stride,
                               const double* f_ext_dev, double* residual_dev, double* values_dev);
int fibra_cuda_assembly_status(fibra_assembly* as, int32_t* bad_element);
/* device time of the last assemble: ms[3] = {element kernel, pair gather, residual} */
int fibra_cuda_assembly_times(fibra_assembly* as, float* ms);
/* out[5] = {n_tets, n_nodes, n_free, nnz, node pairs} */
int fibra_cuda_assembly_info(const fibra_assembly* as, int64_t* out);
const char* fibra_cuda_assembly_last_error(const fibra_assembly* as);
int fibra_cuda_assembly_free(fibra_assembly* as);

#ifdef __cplusplus
}
#endif
#endif
