/*
 * lsg.h — C ABI of the B200-native Hamilton–Jacobi time-integration hot path.
 *
 * This is the drop-in boundary for the reference C++ library `levelset`
 * (/root/reference/proj/core).  Every entry point below names the reference
 * interface it replaces (file:line, paths relative to /root/reference/proj/core).
 * Plain C types only: pointers, sizes, doubles, ints.  No exceptions cross this
 * boundary; every function returns an lsg status code and leaves a message in
 * lsg_last_error() (thread-local).  The C++ drop-in layer
 * (include/levelset_b200/levelset.hpp) maps the codes back onto the exact
 * exception types the reference throws:
 *     LSG_EINVAL   -> std::invalid_argument   (preconditions, e.g. grid.cpp:13-26)
 *     LSG_ERANGE   -> std::out_of_range       (grid.cpp:75, :87)
 *     LSG_ENUMERIC -> std::runtime_error      (hamiltonian.cpp:38-40, :49-53,
 *                                              integrator.cpp:55-56)
 *     LSG_ECUDA / LSG_ENCCL / LSG_ENOMEM -> std::runtime_error (device faults)
 *
 * All arithmetic is IEEE fp64, round-to-nearest, no FMA contraction, in the
 * reference's operation order, so ENO/First paths, dt and step bounds are
 * bit-identical to the reference.
 *
 * There is no CPU fallback.  When no CUDA device is usable every compute
 * entry point fails with LSG_ECUDA.
 */
#ifndef LSG_H_
#define LSG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LSG_ABI_VERSION 1
#define LSG_MAX_DIM 6
#define LSG_MAX_PARAMS 16

/* ---- status codes ------------------------------------------------------ */
#define LSG_OK 0
#define LSG_EINVAL 1
#define LSG_ERANGE 2
#define LSG_ENUMERIC 3
#define LSG_ECUDA 4
#define LSG_ENCCL 5
#define LSG_ENOMEM 6

/* ---- enums (values follow the reference enum order) --------------------- */
/* grid.hpp:16  enum class BoundaryCondition { Periodic, ExtrapolateLinear } */
#define LSG_BC_PERIODIC 0
#define LSG_BC_EXTRAPOLATE 1
/* spatial_derivatives.hpp:8  enum class DerivativeScheme { First, Eno2, Eno3, Weno5 } */
#define LSG_SCHEME_FIRST 0
#define LSG_SCHEME_ENO2 1
#define LSG_SCHEME_ENO3 2
#define LSG_SCHEME_WENO5 3
/* hamiltonian.hpp:14  enum class UpdateDirection { Grow, Shrink } */
#define LSG_GROW 0
#define LSG_SHRINK 1
/* integrator.hpp:68  enum class TimeIntegrator { Cfl1, Cfl2, Cfl3 } */
#define LSG_CFL1 0
#define LSG_CFL2 1
#define LSG_CFL3 2

/*
 * Device Hamiltonian kinds.  The reference passes H and the dissipation bound
 * as host std::function plugins (hamiltonian.hpp:18-25), which a GPU cannot
 * call; the device path takes a kind tag plus POD parameters instead.
 * params[] layout per kind (all doubles):
 *   LINEAR    H = (0 + c0 p0 + c1 p1 + ...) + offset; bound_d = b_d (constant)
 *             params[0..5] = c_d, params[6..11] = b_d, params[12] = offset.
 *             (test_hamiltonian.cpp:18-36 advection_problem and the test lambdas)
 *   ROTATION  H = -y p0 + x p1; bounds |y|, |x|            (reachability.cpp:105-133)
 *   ROCKETS   reference rocket game (reachability.cpp:12-66);
 *             params = {a, g, capture_radius, u_min, u_max}
 *   AIR3D     ToolboxLS air3D form (builder-defined);
 *             params = {v_a, v_b, w_a, w_b}
 *   DBLINT4   4-D double-integrator pair (cfg3): H = p0 x1 + p2 x3 - |p1| - |p3|
 *   DUBINS6   6-D two-vehicle Dubins (cfg4):
 *             H = p0 cos(th_a) + p1 sin(th_a) + p3 cos(th_b) + p4 sin(th_b) - |p2| + |p5|
 *   NORMAL    motion in the normal direction (cfg5): H = speed * |p|_2; params = {speed}
 */
#define LSG_HAM_LINEAR 1
#define LSG_HAM_ROTATION 2
#define LSG_HAM_ROCKETS 3
#define LSG_HAM_AIR3D 4
#define LSG_HAM_DBLINT4 5
#define LSG_HAM_DUBINS6 6
#define LSG_HAM_NORMAL 7

/* ---- descriptors --------------------------------------------------------- */

/* Grid::create arguments (grid.hpp:29-32).  periodic_mask bit d marks dim d
 * periodic.  Layout is the reference's column-major order (grid.hpp:21-23). */
typedef struct lsg_grid {
    int dim;
    int counts[LSG_MAX_DIM];
    double mins[LSG_MAX_DIM];
    double maxs[LSG_MAX_DIM];
    unsigned periodic_mask;
} lsg_grid;

/* HamiltonianProblem (hamiltonian.hpp:29-36) with a device Hamiltonian. */
typedef struct lsg_problem {
    int kind;            /* LSG_HAM_* */
    int scheme;          /* costate_scheme, LSG_SCHEME_* */
    int direction;       /* update_direction, LSG_GROW / LSG_SHRINK */
    int restrict_update; /* bool */
    int options;         /* LSG_OPT_* bits */
    double params[LSG_MAX_PARAMS];
} lsg_problem;

/* lsg_problem.options: WENO5 with one division per side (common-denominator
 * weights, constant reciprocals) instead of the reference's 13; results agree
 * with the reference within a few ulps per derivative (north_star: 1e-10
 * relative), not bit for bit.  Off by default. */
#define LSG_OPT_WENO5_FAST 1u

/* IntegratorOptions (integrator.hpp:14-24). */
typedef struct lsg_opts {
    double cfl_factor;          /* default 0.32 */
    double max_step;            /* default +inf */
    double termination_epsilon; /* default 1e-6 */
    const double* checkpoint_times;
    size_t n_checkpoint_times;
} lsg_opts;

/* StepLogEntry (integrator.hpp:29-35). */
typedef struct lsg_steplog {
    double t, dt, step_bound, v_min, v_max;
} lsg_steplog;

typedef struct lsg_ctx lsg_ctx;
typedef struct lsg_solver lsg_solver;

/* ---- library / context --------------------------------------------------- */
int lsg_abi_version(void);
const char* lsg_last_error(void);
void lsg_opts_default(lsg_opts* opts);
int lsg_device_count(int* count);

/* One context = one CUDA device + one stream, used by one host thread. */
int lsg_ctx_create(int device, lsg_ctx** out);
/* Distributed context: one process per GPU, slabs along the last grid axis.
 * nccl_id is the 128-byte ncclUniqueId rank 0 produced with lsg_nccl_unique_id
 * and shared out of band (bench.py uses the torch.distributed store).  On such
 * a context the solver-backed calls (lsg_solver_*, lsg_integrate,
 * lsg_solve_brt, lsg_term_lf) take and return this rank's slab
 * (lsg_slab_partition; solve_brt's checkpoints are slabs too), grids stay
 * global, and all ranks must make the same calls in the same order (halo
 * exchanges and all-reduces inside).  The other stateless calls (lsg_upwind,
 * lsg_pad_ghost, shapes, set operations, evaluations) work per process on
 * the whole grid they are given. */
int lsg_nccl_unique_id(void* out128);
int lsg_ctx_create_dist(int device, int rank, int nranks, const void* nccl_id128, lsg_ctx** out);
/* Solvers created on a context must be destroyed before it (their buffers are
 * released on its stream). */
int lsg_ctx_destroy(lsg_ctx* ctx);
int lsg_ctx_synchronize(lsg_ctx* ctx);
/* Number of device kernels this context has launched so far. */
int lsg_ctx_launch_count(const lsg_ctx* ctx, uint64_t* count);

/* Page-locked host buffers for the host<->device copies of the reference-facing
 * calls (allocated by this library's CUDA runtime). */
int lsg_host_alloc(size_t bytes, void** out);
int lsg_host_free(void* p);

/* ---- grid (grid.cpp:9-66, :69-91) ---------------------------------------- */
/* Validates like Grid::create (grid.cpp:13-26). */
int lsg_grid_check(const lsg_grid* g);
/* spacing(d) = (max-min)/(n-1) (grid.cpp:41); node_count; axis(d)[i] = min + i*dx (grid.cpp:50). */
int lsg_grid_spacing(const lsg_grid* g, int d, double* dx);
int lsg_grid_node_count(const lsg_grid* g, size_t* n);
int lsg_grid_axis(const lsg_grid* g, int d, double* out);

/* Slab of rank r among P along an axis of n planes: the first n % P ranks
 * hold ceil(n/P) planes, the rest floor(n/P) (host-only, no device needed). */
int lsg_slab_partition(int n, int nranks, int rank, int* z0, int* nz);
/* The halo messages a rank issues per exchange, in order (host-only; the
 * distributed exchange issues exactly these as one NCCL group): kinds[i] 0 =
 * send, 1 = recv; peers[i] the other rank; planes[i] the first plane relative
 * to the slab's plane 0 (ghost planes are < 0 or >= its plane count);
 * counts[i] planes.  At most 4 messages (arrays of 4). */
int lsg_halo_plan(int n, int nranks, int rank, int width, int periodic, int* kinds, int* peers, int* planes,
                  int* counts, int* n_messages);

/* ---- stateless reference-facing calls (host buffers in and out) ------------
 * Each call copies its host inputs to the device, runs the kernels, and copies
 * the results back; these are what a reference call site binds to. */

/* pad_ghost (grid.hpp:110, grid.cpp:132-165).  out has
 * node_count / n_dim * (n_dim + 2*width) doubles. */
int lsg_pad_ghost(lsg_ctx* ctx, const lsg_grid* g, const double* field, int dim, int width,
                  double* out);
/* shift_along_dim (grid.hpp:114, grid.cpp:167-193). */
int lsg_shift_along_dim(lsg_ctx* ctx, const lsg_grid* g, const double* padded, int dim,
                        int width, int offset, double* out);
/* upwind_derivative / upwind_first_* (spatial_derivatives.hpp:28-45,
 * spatial_derivatives.cpp:37-224). */
int lsg_upwind(lsg_ctx* ctx, const lsg_grid* g, const double* v, int dim, int scheme,
               double* left, double* right);
/* term_lax_friedrichs (hamiltonian.hpp:57, hamiltonian.cpp:11-76). */
int lsg_term_lf(lsg_ctx* ctx, const lsg_grid* g, const lsg_problem* p, double t,
                const double* v, double* dvdt, double* step_bound);
/* restrict_update (hamiltonian.hpp:62, hamiltonian.cpp:78-88). */
int lsg_restrict_update(lsg_ctx* ctx, size_t n, const double* dvdt, int direction, double* out);
/* The reference's Hamiltonian / dissipation plugins (HamiltonianFn / DissipationFn,
 * hamiltonian.hpp:16-25) for a device kind, on host fields: H at every node from
 * dim costate fields (costate[d] = central derivative along d), or the per-node
 * bound on |dH/dp_dim|.  Raw values (term_lax_friedrichs validates them);
 * e.g. rocket_hamiltonian / rocket_dissipation, reachability.cpp:12-66. */
int lsg_eval_hamiltonian(lsg_ctx* ctx, const lsg_grid* g, const lsg_problem* p, double t,
                         const double* const* costate, double* out);
int lsg_eval_dissipation(lsg_ctx* ctx, const lsg_grid* g, const lsg_problem* p, double t, int dim, double* out);
/* set_union / set_intersection / set_complement on host fields (implicit_surfaces.cpp:128-151):
 * op 1 = std::min(a, b), 2 = std::max(a, b), 3 = -a (b unused). */
int lsg_set_op(lsg_ctx* ctx, int op, size_t n, const double* a, const double* b, double* out);
/* integrate / ode_cfl_1/2/3 with the Lax-Friedrichs term
 * (integrator.hpp:49-72, integrator.cpp:22-125).  v is the initial value on
 * entry and the final value on return; steps receives up to log_cap entries
 * and *n_steps the total accepted step count. */
int lsg_integrate(lsg_ctx* ctx, const lsg_grid* g, const lsg_problem* p, int method,
                  double t0, double tf, double* v, const lsg_opts* opts,
                  lsg_steplog* steps, size_t log_cap, size_t* n_steps, double* t_final);
/* solve_brt (reachability.hpp:80-82, reachability.cpp:135-174).  checkpoints
 * receives n_checkpoints * node_count doubles when n_checkpoints > 1 (only
 * the initial field when the span is empty; *n_out says how many). */
int lsg_solve_brt(lsg_ctx* ctx, const lsg_grid* g, const lsg_problem* p, const double* v0,
                  double t_first, double t_second, int n_checkpoints, int method,
                  const lsg_opts* opts, double* checkpoints, double* checkpoint_times,
                  int* n_out, lsg_steplog* steps, size_t log_cap, size_t* n_steps,
                  double* integration_seconds);

/* Resume a checkpointed solve_brt (the reference has none): the
 * field v_k of checkpoint k (e.g. read back with lsg_read_snapshot) at the
 * integration time t_k where that leg stopped (the snapshot's time when the
 * leg landed on its checkpoint time, as legs do unless the termination
 * epsilon stops them short, integrator.cpp:37-40).  Runs legs k+1 ..
 * n_checkpoints-1 exactly as lsg_solve_brt does; checkpoints receives
 * (n_checkpoints - k) fields starting with v_k, and the step log and
 * checkpoints equal those of the uninterrupted solve. */
int lsg_solve_brt_resume(lsg_ctx* ctx, const lsg_grid* g, const lsg_problem* p, const double* v_k, int k, double t_k,
                         double t_first, double t_second, int n_checkpoints, int method, const lsg_opts* opts,
                         double* checkpoints, double* checkpoint_times, int* n_out, lsg_steplog* steps,
                         size_t log_cap, size_t* n_steps, double* integration_seconds);

/* ---- checkpoint output in the reference's snapshot format ----------------
 * snapshot.cpp:69-129: text header "dims/counts/mins/maxs/time" (reals with 17
 * significant digits) + little-endian fp64 payload in column-major order. */
int lsg_write_snapshot(const lsg_grid* g, const double* field, double time, const char* path);
/* Reads the header (periodic_mask is 0: the format does not store boundary tags,
 * snapshot.hpp:9-11) and, when field != NULL, the payload (cap doubles). */
int lsg_read_snapshot(const char* path, lsg_grid* g, double* time, double* field, size_t cap);

/* ---- zero-level-set extraction (contour.cpp:27-135) --------------------------
 * Marching squares on a 2-D field: segments as {ax, ay, bx, by} quadruples in
 * the reference's order and arithmetic.  *n_segments receives the total; when
 * it exceeds cap, nothing is written and LSG_ERANGE is returned.
 * lsg_slice_2d restricts a 3-D field to fixed_dim = index (out: the 2-D slice,
 * column-major over the remaining dimensions). */
int lsg_extract_zero_set_2d(lsg_ctx* ctx, const lsg_grid* g, const double* field, double* segments, size_t cap,
                            size_t* n_segments);
int lsg_slice_2d(lsg_ctx* ctx, const lsg_grid* g, const double* field, int fixed_dim, int index, double* out);

/* ---- device-resident solver (the fast path bench.py measures) --------------
 * Holds the value function in HBM across steps; in a distributed context it
 * holds this rank's slab of the global grid. */
int lsg_solver_create(lsg_ctx* ctx, const lsg_grid* global_grid, const lsg_problem* p,
                      int method, lsg_solver** out);
/* In-process slab emulation: nslabs slabs of the same grid on one device,
 * halos exchanged by device copies.  Used to prove P-slab == 1-slab bitwise. */
int lsg_solver_create_slabs(lsg_ctx* ctx, const lsg_grid* global_grid, const lsg_problem* p,
                            int method, int nslabs, lsg_solver** out);
int lsg_solver_destroy(lsg_solver* s);
/* This rank's slab: first global plane along the last axis and plane count. */
int lsg_solver_slab(const lsg_solver* s, int* z0, int* nz, size_t* local_nodes);
/* Host <-> device value transfer of the local slab (column-major, local_nodes doubles). */
int lsg_solver_set_field(lsg_solver* s, const double* host_v);
int lsg_solver_get_field(lsg_solver* s, double* host_v);
/* Device pointer transfer (stream-ordered on the context stream). */
int lsg_solver_set_field_device(lsg_solver* s, const double* dev_v);
int lsg_solver_field_device(lsg_solver* s, double** dev_v);
/* Device initial-condition generator (implicit_surfaces.cpp:20-71):
 * shape 0 = sphere(center, radius), 1 = cylinder(ignored_mask, center, radius),
 * 2 = planar pair distance (6-D).  Writes a fresh field. */
int lsg_solver_init_shape(lsg_solver* s, int shape, unsigned ignored_mask, const double* center,
                          double radius);
/* The same generator with every implicit_surfaces.cpp shape, composed with the
 * resident field on the device: op 0 = replace, 1 = set_union (std::min(field,
 * shape)), 2 = set_intersection (std::max(field, shape)) (implicit_surfaces.cpp:128-145).
 * shape 3 = rectangle(lower = center[], upper[]) (:73-94), 4 = ellipsoid(radius),
 * 2-D/3-D (:96-116); shapes 0-2 as in lsg_solver_init_shape. */
int lsg_solver_apply_shape(lsg_solver* s, int op, int shape, unsigned ignored_mask, const double* center,
                           const double* upper, double radius);
/* field = -field (set_complement, implicit_surfaces.cpp:147-151). */
int lsg_solver_complement(lsg_solver* s);
/* CFL step bound 1/sum(alpha_d/dx_d) at time t (hamiltonian.cpp:44-71). */
int lsg_solver_step_bound(lsg_solver* s, double t, double* bound);
/* Enqueue one TVD-RK step of size dt from time t (integrator.cpp:58-85) on the
 * context stream, no host synchronisation. */
int lsg_solver_step(lsg_solver* s, double t, double dt);
/* One step with the field coming from host memory and the result going back
 * to it (set_field + step + get_field in one call, the reference's
 * integrate(term, {t, t+dt}, v0) with host vectors).  On a single-slab solver
 * the copies are chunked along the last axis and overlapped with the stage
 * kernels (bit-identical result; overlap needs page-locked buffers, e.g.
 * lsg_host_alloc).  host_in and host_out may alias.  Returns when host_out is
 * complete.  LSG_PIPE=0 disables the overlap. */
int lsg_solver_step_host(lsg_solver* s, double t, double dt, const double* host_in, double* host_out);
/* Same as lsg_solver_step, bracketed by CUDA events recorded on the context
 * stream before the step and after every stage; synchronises and returns the
 * device time of each stage (stage_ms[0..stages-1]) and of the whole step. */
int lsg_solver_step_timed(lsg_solver* s, double t, double dt, double* stage_ms, double* step_ms);
/* run_cfl over [t0, tf] with the reference's step control (integrator.cpp:22-97). */
int lsg_solver_integrate(lsg_solver* s, double t0, double tf, const lsg_opts* opts,
                         lsg_steplog* steps, size_t log_cap, size_t* n_steps, double* t_final);
/* Snapshot of the resident value function in the reference's format
 * (snapshot.cpp:68-93).  In a distributed context the call is collective: the
 * slabs are gathered on rank 0 (NCCL point-to-point, 1 GiB chunks), which
 * writes the whole grid to `path`; the other ranks write nothing (their path
 * may be NULL). */
int lsg_solver_write_snapshot(lsg_solver* s, double time, const char* path);
/* Gather a distributed field held as host slabs (e.g. solve_brt's per-rank
 * checkpoints) into global_out on rank 0 (node_count(g) doubles; unused and
 * may be NULL elsewhere).  Collective on a multi-rank context; a plain copy
 * otherwise. */
int lsg_gather_field(lsg_ctx* ctx, const lsg_grid* g, const double* local, double* global_out);
/* Raw CUDA stream (cudaStream_t) of the context, for external event timing. */
int lsg_solver_stream(lsg_solver* s, void** stream);
/* ---- diagnostics ------------------------------------------------------------
 * Measured FP64 DADD/DMUL issue rate of the context's device (instructions/s):
 * the second roofline of this FMA-free fp64 stencil, probed in the same run
 * that reports against it (about 10 ms of device time). */
int lsg_probe_fp64_rate(lsg_ctx* ctx, double* instr_per_s);
/* Size of the context's NCCL communicator and this process's rank in it, read
 * back from NCCL (ncclCommCount / ncclCommUserRank); 0 and -1 without one. */
int lsg_ctx_comm_info(const lsg_ctx* ctx, int* nranks, int* rank);
/* Kernels one lsg_solver_step launches. */
int lsg_solver_launches_per_step(const lsg_solver* s, int* n);

#ifdef __cplusplus
}
#endif
#endif /* LSG_H_ */
