/*
 * klref_b200 — C-ABI of the B200-native hot path of the kl-refinement method
 * (arXiv 2508.06049): matrix-free FMG on the hierarchical hybrid grid (HHG)
 * plus the FMG-byproduct error estimator, as sm_100a CUDA kernels.
 *
 * The reference ships no C-ABI (proj/src/CMakeLists.txt:18 names a capi.cpp
 * that is absent); its interface for this path is the C++ API of
 * proj/include/klref/{hhg,fem,multigrid,estimator}.hpp.  Every entry point
 * below names the reference function it replaces.  Conventions:
 *   - plain pointers and sizes, opaque handles, no torch / CUDA types;
 *   - every function returns a status (KLREF_OK = 0) and never throws; the
 *     message of the last failure on the calling thread is klref_last_error()
 *     and the codes mirror proj/include/klref/errors.hpp:10-53;
 *   - host arrays of grid functions use the reference layout: macro-major
 *     (slot order = ascending active element id), each macro a triangular
 *     lattice row-major in j, index j(n+1) - j(j-1)/2 + i
 *     (proj/include/klref/hhg.hpp:13), interface copies included;
 *   - there is no CPU fallback: without a CUDA device every compute entry
 *     point fails with KLREF_ERR_CUDA.
 */
#ifndef KLREF_B200_H
#define KLREF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (proj/include/klref/errors.hpp) */
#define KLREF_OK 0
#define KLREF_ERR_STRUCTURAL 1 /* StructuralError */
#define KLREF_ERR_DOMAIN 2     /* DomainError */
#define KLREF_ERR_SOLVER 3     /* SolverError: see klref_last_error_residual() */
#define KLREF_ERR_IO 4         /* IoError */
#define KLREF_ERR_INTERNAL 5   /* InternalError */
#define KLREF_ERR_RESOURCE 6   /* ResourceError: see klref_last_error_level() */
#define KLREF_ERR_CUDA 7       /* CUDA runtime failure / no device */

/* problem kinds (BASELINE.json configs; proj/src/problems.cpp:36-53) */
#define KLREF_PROBLEM_ZERO 0
#define KLREF_PROBLEM_SIN2D 1  /* u = sin(pi x) sin(pi y), f = 2 pi^2 u     (config 1) */
#define KLREF_PROBLEM_LSHAPE 2 /* make_lshape_spec: f = 0, g = r^2/3 sin(2t/3) (config 2) */
/* 3-d problems (no reference solver; BASELINE.json configs 3-5) */
#define KLREF_PROBLEM_SIN3D 3  /* u = prod sin(pi x_i), f = 3 pi^2 u                 (config 3) */
#define KLREF_PROBLEM_GAUSS3D 4 /* u = exp(-1000 |x - c|^2), c = (1/2, 1/2, 1/2)       (config 4) */
#define KLREF_PROBLEM_SERIES3D 5 /* f = sum C_abc sin(a pi x) sin(b pi y) sin(c pi z), g = 0 (config 5) */

/* operator kinds (OperatorKind, proj/include/klref/fem.hpp:13) */
#define KLREF_STIFFNESS 0
#define KLREF_MASS 1

/* estimator kinds (EstimatorKind, proj/include/klref/estimator.hpp:10) */
#define KLREF_UNSCALED 0
#define KLREF_SCALED 1

/* sync modes (SyncMode, proj/include/klref/hhg.hpp:16) */
#define KLREF_SYNC_REPLACE 0
#define KLREF_SYNC_ADDITIVE 1

/* FmgState components */
#define KLREF_STATE_U 0 /* u[l], l = 0..L */
#define KLREF_STATE_B 1 /* b[l], l = 0..L */
#define KLREF_STATE_W 2 /* w[l-1] = P u[l-1], lives on level l = 1..L */

/* marking rules for klref_mark (proj/src/amr.cpp:41-68, BASELINE.json configs 2/4) */
#define KLREF_MARK_TOP_FRACTION 0
#define KLREF_MARK_HALF_MAX 1

/* kernel kinds of the per-kernel device-time probes (klref_solver_kernel_stats) */
#define KLREF_KERNEL_ALL (-1)
#define KLREF_KERNEL_GS 0       /* gauss_seidel sweeps            multigrid.cpp:127 */
#define KLREF_KERNEL_RESIDUAL 1 /* residual                       multigrid.cpp:183 */
#define KLREF_KERNEL_RESTRICT 2 /* restrict_transpose             multigrid.cpp:55 */
#define KLREF_KERNEL_PROLONG 3  /* prolongate (+correction, w)    multigrid.cpp:22, 243, 265 */
#define KLREF_KERNEL_RHS 4      /* assemble_rhs + Dirichlet rows  fem.cpp:175-228 */
#define KLREF_KERNEL_CG0 5      /* cg_level0                      multigrid.cpp:198 */
#define KLREF_KERNEL_ESTIMATE 6 /* error_estimate norms           estimator.cpp:8-45 */
#define KLREF_KERNEL_OTHER 7    /* boundary initialisation, memsets */

typedef struct klref_mesh_s* klref_mesh;
typedef struct klref_hierarchy_s* klref_hierarchy;
typedef struct klref_problem_s* klref_problem;
typedef struct klref_solver_s* klref_solver;
typedef struct klref_gf_s* klref_gf;

/* SolverConfig, proj/include/klref/multigrid.hpp:19-29 (finest_policy: 0 = None,
 * 1 = ValidationTwoDigits, 2 = ResidualVsEstimate, both on 2-d hierarchies;
 * the reference default is 1) */
typedef struct {
  int nu;
  int pre_smooth;
  int post_smooth;
  double coarse_rel_tol;
  double coarse_abs_floor;
  int coarse_max_iter;
  int finest_policy;
  int faithful_source; /* 1: host-tabulated f (bitwise-faithful RHS); 0: device-evaluated f */
  int use_graph;       /* 1: replay the FMG as one CUDA graph */
  int max_extra_cycles; /* SolverConfig::max_extra_cycles (ValidationTwoDigits) */
} klref_solver_config;

/* EstimateReport, proj/include/klref/estimator.hpp:15-24 (eta_local returned separately) */
typedef struct {
  int offset;
  int base_level;
  int kind;
  double norm_coarser;
  double norm_base;
  double conv_factor;
  double eta;
} klref_estimate_report;

/* ---- errors ---------------------------------------------------------- */
const char* klref_last_error(void);
double klref_last_error_residual(void); /* SolverError::last_residual */
int klref_last_error_level(void);       /* ResourceError::level */
int klref_abi_version(void);
/* Creates the CUDA context of the current device (no reference counterpart:
 * a cold process pays it on the first hierarchy build otherwise); KLREF_ERR_CUDA
 * without a device. */
int klref_device_init(void);

/* ---- coarse mesh ------------------------------------------------------ */
/* Conforming macro mesh in slot order (MacroMesh::create,
 * proj/src/macro_mesh.cpp:115-204, restricted to what the hot path reads):
 * coords[dim * num_vertices], corners[(dim + 1) * num_elements] (vertex ids);
 * elements are oriented positively as the reference does.  dim = 2
 * (triangles) or 3 (tetrahedra; the reference has no 3-d solver, the 3-d
 * path is the builder's design -- DESIGN.md). */
int klref_mesh_create(int dim, int num_vertices, const double* coords, int num_elements,
                      const int* corners, klref_mesh* out);
void klref_mesh_destroy(klref_mesh mesh);

/* ---- hierarchy -------------------------------------------------------- */
/* GridHierarchy::build, proj/src/hhg.cpp:48-144 (+ device upload) */
int klref_hierarchy_build(klref_mesh mesh, int max_level, klref_hierarchy* out);
/* host-only build (no device memory touched): tables for CPU tests */
int klref_hierarchy_build_host(klref_mesh mesh, int max_level, klref_hierarchy* out);
void klref_hierarchy_destroy(klref_hierarchy h);
int klref_hierarchy_num_macros(klref_hierarchy h, int* out);            /* num_macros() */
int klref_hierarchy_max_level(klref_hierarchy h, int* out);             /* max_level() */
int klref_hierarchy_dof_count(klref_hierarchy h, int level, int64_t* out); /* dof_count(l) */
int klref_hierarchy_fine_element_count(klref_hierarchy h, int level, int64_t* out);
int klref_hierarchy_lattice_size(klref_hierarchy h, int level, int* out); /* lattice_size(2^l) */
int klref_hierarchy_dag_depth(klref_hierarchy h, int* out);
/* Level(l).groups (proj/include/klref/hhg.hpp:19-27): ptr[num_groups + 1],
 * members[4 * num_members] = (slot, idx, i, j) (3-d: (slot, idx, 0, 0)).
 * Pass NULL to query sizes. */
int klref_hierarchy_groups(klref_hierarchy h, int level, int* num_groups, int* num_members, int* ptr,
                           int* members);
/* OperatorP1::matrices/stencil (proj/include/klref/fem.hpp:30-37): mats[18 * M]
 * (up, down per macro), stencil[7 * M] (stiffness only; may be NULL).
 * 3-d: mats[96 * M] (six micro-tet types, 4x4 each), stencil[15 * M]. */
int klref_hierarchy_element_matrices(klref_hierarchy h, int level, int kind, double* mats, double* stencil);

/* ---- problems --------------------------------------------------------- */
int klref_problem_create(int kind, klref_problem* out);
/* ProblemSpec with host callbacks (proj/include/klref/fem.hpp:55-64); f is
 * tabulated on the host at the quadrature points (bitwise-faithful RHS). */
int klref_problem_create_host(double (*source)(double, double, void*), double (*boundary)(double, double, void*),
                              void* ctx, klref_problem* out);
/* 3-d host callbacks (f, g of x, y, z), tabulated on the host in faithful mode */
int klref_problem_create_host3(double (*source)(double, double, double, void*),
                               double (*boundary)(double, double, double, void*), void* ctx, klref_problem* out);
/* ProblemSpec::exact for a host problem (proj/include/klref/fem.hpp:57-60): has_exact = true */
int klref_problem_set_exact(klref_problem p, double (*exact)(double, double, void*), void* ctx);
/* parameters of KLREF_PROBLEM_SERIES3D: count = 64 coefficients C_abc, a fastest */
int klref_problem_set_params(klref_problem p, const double* params, int count);
void klref_problem_destroy(klref_problem p);

/* ---- solver ----------------------------------------------------------- */
void klref_solver_config_default(klref_solver_config* cfg);
/* MultigridSolver(h, p, cfg), proj/src/multigrid.cpp:113-119 */
int klref_solver_create(klref_hierarchy h, klref_problem p, const klref_solver_config* cfg, klref_solver* out);
void klref_solver_destroy(klref_solver s);
/* MultigridSolver::fmg, proj/src/multigrid.cpp:248-321 (state kept device-resident in the solver) */
int klref_solver_fmg(klref_solver s);
/* asynchronous variant + completion (error status is checked by synchronize) */
int klref_solver_fmg_enqueue(klref_solver s);
int klref_solver_synchronize(klref_solver s);
/* the cudaStream_t the solver launches on (for event timing), as void* */
int klref_solver_stream(klref_solver s, void** stream);
/* number of kernel launches one FMG enqueues (graph nodes that are kernels/memsets) */
int klref_solver_launch_count(klref_solver s, int* out);
int klref_solver_last_cg_iterations(klref_solver s, int* out);
/* number of kernel launches one error_estimate enqueues */
int klref_solver_estimate_launch_count(klref_solver s, int* out);
/* launch on a caller-owned cudaStream_t (passed as void*; NULL = the solver's own stream) */
int klref_solver_set_stream(klref_solver s, void* stream);
/* re-tabulate the problem's data (Dirichlet g at the boundary nodes, f at the
 * quadrature points in faithful mode) on the host and copy it host->device
 * from pinned staging; *h2d_bytes (may be NULL) receives the bytes copied.
 * ProblemSpec hand-over of MultigridSolver(h, p, cfg), multigrid.cpp:113-119 */
int klref_solver_set_problem(klref_solver s, klref_problem p, int64_t* h2d_bytes);
/* per-kernel CUDA-event probes: with profiling on, every kernel of the FMG /
 * estimator is bracketed by event records; kernel_stats sums, for one kernel
 * kind (or KLREF_KERNEL_ALL), the device milliseconds, launch count and
 * algorithmic bytes of the most recent FMG + estimate. */
int klref_solver_set_profiling(klref_solver s, int on);
int klref_solver_kernel_stats(klref_solver s, int kind, double* ms, int* launches, double* bytes);
/* FmgState::u/b/w (proj/include/klref/multigrid.hpp:43-53), copied to the host */
int klref_solver_state_read(klref_solver s, int which, int level, double* host_out);

/* ExactErrorEvaluator(h, p, L).evaluate(u_L), proj/src/fem.cpp:358-420 (three-term
 * moment form, pointwise fallback :422-455); per_macro[M] may be NULL (2-d) */
int klref_solver_exact_error(klref_solver s, double* global, double* per_macro);
/* ExactErrorEvaluator(h, p, L).evaluate(u) of a level-L function u (the solver's
 * finest level), proj/src/fem.cpp:395-420; 2-d */
int klref_solver_exact_error_of(klref_solver s, klref_gf u, double* global, double* per_macro);
/* FmgState::extra_cycles of the last fmg() (FinestPolicy::ValidationTwoDigits / ResidualVsEstimate) */
int klref_solver_extra_cycles(klref_solver s, int* out);
/* MultigridSolver::solve_direct(l), proj/src/multigrid.cpp:323-357: level_rhs(l), u = g
 * on the boundary, then cg_level0 (l = 0) or the reference's level-l CG; result into u
 * (a level-l function of the solver's hierarchy); 2-d */
int klref_solver_solve_direct(klref_solver s, int level, klref_gf u);

/* error_estimate(state, j, kind), proj/src/estimator.cpp:8-45; eta_local[M] may be NULL */
int klref_error_estimate(klref_solver s, int offset, int kind, klref_estimate_report* out, double* eta_local);
int klref_error_estimate_enqueue(klref_solver s, int offset);
int klref_error_estimate_finish(klref_solver s, int offset, int kind, klref_estimate_report* out,
                                double* eta_local);

/* ---- device grid functions and single operations ---------------------- */
int klref_gf_create(klref_hierarchy h, int level, klref_gf* out); /* create_function(l) (zeros) */
void klref_gf_destroy(klref_gf f);
int klref_gf_upload(klref_gf f, const double* host);
int klref_gf_download(klref_gf f, double* host);
int klref_apply(klref_solver s, int kind, klref_gf x, klref_gf y);            /* OperatorP1::apply   fem.cpp:95 */
int klref_residual(klref_solver s, klref_gf u, klref_gf b, klref_gf r);       /* residual      multigrid.cpp:183 */
int klref_gauss_seidel(klref_solver s, klref_gf u, klref_gf b, int sweeps);   /* gauss_seidel  multigrid.cpp:127 */
int klref_restrict_transpose(klref_solver s, klref_gf fine, klref_gf coarse); /* multigrid.cpp:55 */
int klref_prolongate(klref_solver s, klref_gf coarse, klref_gf fine);         /* multigrid.cpp:22 */
int klref_cg_level0(klref_solver s, klref_gf u, klref_gf b);                  /* cg_level0     multigrid.cpp:198 */
int klref_dot_unique(klref_solver s, klref_gf a, klref_gf b, double* out);    /* hhg.cpp:227 */
int klref_interface_sync(klref_solver s, klref_gf f, int mode);               /* hhg.cpp:206 */

/* ---- host marking (mark_and_refine's reversion aggregate + rule) ------ */
/* proj/src/amr.cpp:41-66 and mark_top_fraction proj/src/macro_mesh.cpp:678-695.
 * active_ids[num_active] with green_parent[num_active] (-1 if not a green child),
 * indicator[num_active]; reverted_ids[num_reverted] = active ids after revert_green.
 * marks_out[num_reverted] receives the sorted marked ids, *num_marks their count. */
int klref_mark(int rule, double fraction, int num_active, const int* active_ids, const int* green_parent,
               const double* indicator, int num_reverted, const int* reverted_ids, int* marks_out, int* num_marks);

/* ---- effectivity constants and indices (host) -------------------------- */
/* effectivity_constants, local_spread_bound_scaled / _unscaled and
 * effectivity_index, proj/include/klref/estimator.hpp:27-68,
 * proj/src/estimator.cpp:47-123.  Domain violations return KLREF_ERR_DOMAIN
 * (the reference throws DomainError).  effectivity_index: gamma = eta /
 * exact_global (gamma_valid = exact_global > 0), gamma_local[num_local] = NaN
 * where the macro's exact error is <= 1e-14 of the global one, spread =
 * max / min of the valid local indices. */
int klref_effectivity_constants(double theta, double eps, int offset, double* lower, double* upper);
int klref_local_spread_bound_scaled(double theta_max, double eps, int offset, double* out);
int klref_local_spread_bound_unscaled(double theta_min, double theta_max, int offset, double* out);
int klref_effectivity_index(double eta, int num_local, const double* eta_local, double exact_global,
                            int num_exact, const double* exact_local, double* gamma, int* gamma_valid,
                            double* gamma_local, double* spread, int* spread_valid);

/* ---- sharded 3-d solve (no reference counterpart) ------
 * The reference is single-process.  Its paper partitions macro
 * elements with ghost layers on the interface primitives;
 * these entry points run MultigridSolver::fmg / error_estimate
 * (proj/src/multigrid.cpp:248-321, proj/src/estimator.cpp:8-45) over
 * contiguous macro slot ranges, one shard per GPU over NCCL (comm != NULL)
 * or `local_shards` shards in this process on one device (comm == NULL, the
 * parity harness).  Levels <= rep_level are replicated on every shard.
 * Results are bit-identical to klref_solver_* on the same hierarchy. */
typedef struct klref_comm_s* klref_comm;
typedef struct klref_sharded_s* klref_sharded;
int klref_comm_unique_id(unsigned char id[128]);
int klref_comm_create(int nranks, int rank, const unsigned char id[128], klref_comm* out);
void klref_comm_destroy(klref_comm c);
int klref_sharded_create(klref_hierarchy h, klref_problem p, const klref_solver_config* cfg, klref_comm comm,
                         int local_shards, int rep_level, klref_sharded* out);
void klref_sharded_destroy(klref_sharded s);
int klref_sharded_fmg(klref_sharded s);
int klref_sharded_fmg_enqueue(klref_sharded s);
int klref_sharded_synchronize(klref_sharded s);
int klref_sharded_stream(klref_sharded s, void** stream);
/* kernel launches per FMG / per estimate (all local shards), bytes one FMG exchanges */
int klref_sharded_counts(klref_sharded s, int* fmg_launches, int* estimate_launches, double* exchange_bytes);
int klref_sharded_error_estimate_enqueue(klref_sharded s, int offset);
int klref_sharded_error_estimate_finish(klref_sharded s, int offset, int kind, klref_estimate_report* out,
                                        double* eta_local);
/* full level array (M * S); over NCCL only this rank's slot range and the replicated levels are written */
int klref_sharded_state_read(klref_sharded s, int which, int level, double* host_out);
/* exchange plan of one shard on one level (host only; plan checks):
 * send_counts / recv_counts[nshards * colors] (peer-major), *colors, and per
 * buffer position the (global group, slot, lattice index) of the member whose
 * contribution travels there: send_keys[3 * send_total], recv_keys[3 * recv_total].
 * NULL key arrays query the counts only. */
int klref_shard_plan(klref_hierarchy h, int nshards, int rank, int rep_level, int level, int* colors,
                     int64_t* send_counts, int64_t* recv_counts, int* send_keys, int* recv_keys);
/* shard slot ranges starts[nshards + 1] of the hierarchy (host only) */
int klref_shard_starts(int num_macros, int nshards, int* starts);

#ifdef __cplusplus
}
#endif

#endif /* KLREF_B200_H */
