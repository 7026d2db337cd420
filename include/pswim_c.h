/*
 * pswim_c.h — C-ABI drop-in boundary of the B200-native MRS / rod / Parareal hot path.
 *
 * Every entry point replaces one reference interface of arxiv/paper_2604_12083's CPU
 * library `pintswim` (paths relative to /root/reference/proj).  Plain pointers and sizes
 * only: no torch, no C++ types.  Layout conventions follow the reference exactly:
 *
 *   Vec3            3 doubles, AoS                         (include/pintswim/geom.hpp:10-18)
 *   Mat3 / Rot3     9 doubles, row-major                   (include/pintswim/geom.hpp:37-40)
 *   packed state    per node 12 doubles [x, d1, d2, d3],   (src/io.cpp:10-25, io.hpp:14-17)
 *                   rods concatenated in order
 *
 * Errors: every call returns 0 (PSWIM_OK) or a PSWIM_E* code; pswim_last_error() gives text.
 * Device-side failures (non-finite loads, stiffness guard, degenerate segment) are raised
 * through a device flag and reported by the first call that synchronises the context
 * (pswim_sync, every *_host entry point, pswim_propagate).
 *
 * Device pointers ("d_" prefix) must be cudaMalloc'd memory of the context's device.
 * Host pointers ("h_" prefix) are ordinary (or pinned) host memory.
 */
#ifndef PSWIM_C_H
#define PSWIM_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes ------------------------------------------------------------------ */
enum {
    PSWIM_OK = 0,
    PSWIM_EINVAL = 1,            /* std::invalid_argument in the reference               */
    PSWIM_EUNSUPPORTED_WALL = 2, /* stokes.cpp:15-17 image_wall throws runtime_error     */
    PSWIM_ENONFINITE = 3,        /* stokes.cpp:21-25 non-finite load entry                */
    PSWIM_ESTIFF = 4,            /* propagators.hpp:24-26 StiffnessError                 */
    PSWIM_EDEGENERATE = 5,       /* rod.cpp:53-55 degenerate segment                      */
    PSWIM_ECUDA = 6,             /* CUDA runtime failure                                  */
    PSWIM_ECOMM = 7,             /* transport (NCCL / peer copy / callback) failure       */
    PSWIM_ESTATE = 8             /* std::logic_error in the reference                    */
};

/* ---- parameter blocks ---------------------------------------------------------------- */
/* KernelParams, include/pintswim/stokes.hpp:13-17.  wall_mode: 0 free_space, 1 image_wall. */
typedef struct pswim_kernel_params {
    double epsilon;
    double mu;
    int32_t wall_mode;
    int32_t _pad;
} pswim_kernel_params;

/* ScenarioConfig, include/pintswim/scenario.hpp:16-35.  epsilon = 0 / lj_sigma = 0 mean
 * "derive the default" exactly as make_scenario (scenario.cpp:10-29).
 * placement: 0 grid, 1 random. */
typedef struct pswim_scenario {
    int64_t rod_count;
    int64_t nodes_per_rod;
    double rod_length;
    double a1, a2, a3;          /* MaterialParams bending, bending, torsion  (rod.hpp:28-31) */
    double b1, b2, b3;          /* shear, shear, stretch                                      */
    double amplitude;           /* WaveformParams A, f, lambda               (rod.hpp:34-39) */
    double frequency;
    double wavelength;
    double epsilon;
    double mu;
    int32_t wall_mode;
    int32_t placement;
    double lj_well_depth;
    double lj_sigma;
    double wall_clearance;
    uint64_t seed;
    double fine_dt;
    double horizon;
} pswim_scenario;

/* Fills the reference defaults of ScenarioConfig (scenario.hpp:16-35). */
void pswim_scenario_defaults(pswim_scenario* sc);

/* Scenario (scenario.hpp:38-44) after make_scenario: derived ds, epsilon, sigma, window. */
typedef struct pswim_resolved {
    double ds;
    double epsilon;
    double mu;
    double lj_sigma;
    double lj_cutoff;
    int64_t lj_self_exclusion;
    int64_t total_nodes;
} pswim_resolved;

/* make_scenario, src/scenario.cpp:10-29 (validation + derivation). */
int pswim_scenario_resolve(const pswim_scenario* sc, pswim_resolved* out);

/* build_initial_state + pack_state, src/scenario.cpp:71-120 and src/io.cpp:10-25.
 * h_state must hold 12 * rod_count * nodes_per_rod doubles. */
int pswim_build_initial_state(const pswim_scenario* sc, double* h_state);

/* ---- context ------------------------------------------------------------------------- */
typedef struct pswim_ctx pswim_ctx;

/* Creates a context on `device` with its own non-blocking stream (priority 0 = default,
 * <0 = higher priority as cudaStreamCreateWithPriority).  `sc` may be NULL for an
 * MRS-only context (pswim_mrs_velocities / pswim_sqrt_rotation_batched).
 * Replaces the implicit global state of the reference (OpenMP team + timing atomics,
 * src/propagators.cpp:11-36); one context per device stream, not shared across threads
 * without external synchronisation. */
pswim_ctx* pswim_create(int device, const pswim_scenario* sc, int stream_priority);
void pswim_destroy(pswim_ctx* ctx);
const char* pswim_last_error(const pswim_ctx* ctx);
void* pswim_stream(pswim_ctx* ctx);            /* cudaStream_t of the context             */
int pswim_sync(pswim_ctx* ctx);                /* stream sync + device error-flag check   */
int pswim_device(const pswim_ctx* ctx);

/* ---- MRS operator -------------------------------------------------------------------- */
/* evaluate_velocities, include/pintswim/stokes.hpp:43-44 / src/stokes.cpp:76-95.
 * u_i = (1/mu) sum_j [f_j H1 + (f_j.r) r H2 + (n_j x r) H3], omega likewise, r = t_i - s_j,
 * all targets x all sources, self term included.  Deterministic: fixed launch geometry and
 * fixed-order split-source reduction, bitwise reproducible run to run.
 * Stream-ordered on the context stream, no host sync inside.  ENONFINITE (non-finite f/n)
 * is reported at the next sync. */
int pswim_mrs_velocities(pswim_ctx* ctx, const double* d_targets, int64_t n_targets,
                         const double* d_sources, const double* d_f, const double* d_n,
                         int64_t n_sources, const pswim_kernel_params* kp, double* d_u,
                         double* d_omega);

/* Same operator through host buffers (H2D copies, kernel, D2H copies, sync, error check).
 * Page-locked (cudaHostAlloc / cudaHostRegister) output buffers are written by the kernel
 * directly (mapped host memory, no D2H copies) and page-locked inputs are read by an upload
 * kernel; pageable buffers take DMA copies.  Synchronous: the outputs are complete when the
 * call returns. */
int pswim_mrs_velocities_host(pswim_ctx* ctx, const double* h_targets, int64_t n_targets,
                              const double* h_sources, const double* h_f, const double* h_n,
                              int64_t n_sources, const pswim_kernel_params* kp, double* h_u,
                              double* h_omega);

/* h_functions, src/stokes.cpp:59-74 (device evaluation, batched). */
int pswim_h_functions(pswim_ctx* ctx, const double* d_r, int64_t count, double epsilon,
                      double* d_h5 /* count x 5 */);

/* ---- rotation square root ------------------------------------------------------------ */
/* sqrt_rotation, include/pintswim/rotation.hpp:34 / src/rotation.cpp:91-107, batched:
 * `count` row-major 3x3 rotations in, their half-angle square roots out. */
int pswim_sqrt_rotation_batched(pswim_ctx* ctx, const double* d_r9, int64_t count, double* d_s9);
int pswim_sqrt_rotation_host(pswim_ctx* ctx, const double* h_r9, int64_t count, double* h_s9);

/* ---- rod mechanics ------------------------------------------------------------------- */
/* internal_loads + nodal_loads, src/rod.cpp:36-109, over every rod of the context's
 * scenario.  d_state: packed state.  Outputs per node (N = total nodes) f, n as N x 3;
 * optional d_seg_force / d_seg_moment (rods x (M-1) x 3) receive the segment loads. */
int pswim_rod_loads(pswim_ctx* ctx, const double* d_state, double t, double* d_f, double* d_n,
                    double* d_seg_force, double* d_seg_moment);

/* lj_repulsion, src/rod.cpp:124-174 (raw pair forces, N x 3, before the 1/ds factor). */
int pswim_lj_forces(pswim_ctx* ctx, const double* d_state, double* d_forces);
/* Host-buffer form (packed 12 N state in, N x 3 forces out). */
int pswim_lj_forces_host(pswim_ctx* ctx, const double* h_state, double* h_forces);

/* LJ pair search used by pswim_lj_forces and rhs: 0 = auto (all-pairs tiles below 2048
 * nodes, hashed cell list of side 2^(1/6) sigma above), 1 = all-pairs, 2 = cell list.
 * Replaces the reference's O(N^2) pair loop (src/rod.cpp:146-172) without changing the pair
 * law; the modes differ only in summation order.  Returns the previous mode. */
int pswim_set_lj_mode(pswim_ctx* ctx, int mode);

/* ---- propagators --------------------------------------------------------------------- */
enum { PSWIM_EULER = 0, PSWIM_RK2 = 1 };

/* rhs, src/propagators.cpp:38-91.  d_extra_f / d_extra_n (N x 3) may be NULL. */
int pswim_rhs(pswim_ctx* ctx, const double* d_state, double t, const double* d_extra_f,
              const double* d_extra_n, double* d_u, double* d_omega);

/* advance_state, src/propagators.cpp:93-124 (Euler position update, exact Rodrigues triad
 * rotation, stiffness guard, reorthonormalize).  d_out may not alias d_state. */
int pswim_advance_state(pswim_ctx* ctx, const double* d_state, const double* d_u,
                        const double* d_omega, double dt, double* d_out);

/* step_euler / step_rk2, src/propagators.cpp:126-133. */
int pswim_step(pswim_ctx* ctx, int scheme, const double* d_state, double t, double dt,
               double* d_out);

/* propagate, src/propagators.cpp:135-162.  steps_per_interval > 0 overrides dt exactly as
 * StepperConfig (propagators.hpp:15-20); otherwise (t1-t0)/dt must be integral to 1e-9.
 * t accumulates as t += dt (propagators.cpp:157-160).  d_in and d_out may alias.
 * Synchronises the context (returns ESTIFF / EDEGENERATE / ENONFINITE). */
int pswim_propagate(pswim_ctx* ctx, const double* d_in, double t0, double t1, int scheme,
                    int64_t steps_per_interval, double dt, double* d_out);

/* Small systems (N <= 256 nodes) propagate a whole interval in one fused cluster kernel
 * (state resident in shared memory, MRS partials exchanged through distributed shared
 * memory), bitwise identical to the per-step launched path.  enable: 0 off, 1 on (default:
 * clusters of <= 8 CTAs), 2 / 4 / 8 / 16 on with that cluster-size cap (16: a lone small
 * system on an otherwise idle GPU).  Returns the cluster size used for the context's
 * scenario (0 = not eligible). */
int pswim_set_fused(pswim_ctx* ctx, int enable);

/* The fused small-system propagate (pswim_set_fused) with its in-kernel phase timer on:
 * clock64 cycles of cluster rank 0 spent in 7 phases summed over all steps -- segment loads
 * (+LJ), nodal loads, MRS source staging, MRS pairs, chunk reduction + velocity push,
 * cluster barrier, advance (the reference's stage timers, propagators.hpp:55-65, for a path
 * that is a single kernel).  PSWIM_EINVAL when the scenario is not fused-eligible. */
int pswim_fused_profile(pswim_ctx* ctx, const double* d_in, double t0, double t1, int scheme,
                        int64_t steps_per_interval, double* d_out, uint64_t* h_cycles7);

/* CUDA-graph replay of the per-step kernels for propagations of >= 32 steps of systems of
 * <= 8192 nodes outside the fused path (one graph launch per 32 steps, times read from
 * device memory; larger systems are not launch bound and run the plain loop): bitwise
 * identical to the launch-per-kernel loop.  Enabled by default; returns the previous state. */
int pswim_set_graphs(pswim_ctx* ctx, int enable);

/* Host-buffer propagate (e2e boundary: H2D, propagate, D2H). */
int pswim_propagate_host(pswim_ctx* ctx, const double* h_in, double t0, double t1, int scheme,
                         int64_t steps_per_interval, double dt, double* h_out);

/* Stage timers, propagators.hpp:55-65 (CUDA events: initialization = load assembly,
 * velocity = MRS, triad_update = advance).  Seconds, accumulated since the last reset. */
typedef struct pswim_timing {
    double initialization;
    double velocity;
    double triad_update;
} pswim_timing;
void pswim_timing_enable(pswim_ctx* ctx, int on);
void pswim_timing_reset(pswim_ctx* ctx);
pswim_timing pswim_timing_snapshot(pswim_ctx* ctx);

/* ---- metric / corrector -------------------------------------------------------------- */
/* rod_position_metric, src/io.cpp:49-68 (denominator from the FIRST argument). */
int pswim_position_metric(pswim_ctx* ctx, const double* d_x, const double* d_y, int64_t len,
                          double* h_result);

/* corrected, src/parareal.cpp:47-54: out = (x_prime + g_new) - g_old, elementwise. */
int pswim_parareal_correct(pswim_ctx* ctx, const double* d_x_prime, const double* d_g_new,
                           const double* d_g_old, int64_t len, double* d_out);

/* ---- Parareal ------------------------------------------------------------------------ */
/* ParallelPlan, include/pintswim/parareal.hpp:30-45.  mode: 0 regular, 1 pipelined. */
typedef struct pswim_plan {
    double t0;
    double horizon;
    int32_t intervals;
    int32_t workers;
    double cost_ratio;
    int32_t max_iterations;
    int32_t mode;
    double tolerance;
} pswim_plan;

/* ConvergenceReport, parareal.hpp:47-52.  Arrays sized by the caller (>= intervals). */
typedef struct pswim_report {
    double* eta_tilde;
    double* eta;          /* may be NULL */
    int32_t iterations_used;
    int32_t converged;
    int32_t eta_count;
    int32_t _pad;
    double wall_seconds;
    double schedule_idle; /* W, schedule_trace.cpp:43-49 */
} pswim_report;

/* Propagator hook, the C form of parareal::PropagatorFn (parareal.hpp:19):
 * out = F(t0, t1, in).  `stream` is the CUDA stream (or NULL for host propagators) the
 * call must be ordered on; buffers live where the driver's memory kind says. */
typedef int (*pswim_propagator_fn)(void* user, double t0, double t1, const double* in,
                                   double* out, int64_t len, void* stream);

/* Trace event (schedule_trace.hpp:14-19).  kind: 0 coarse, 1 fine, 2 correct, 3 idle.
 * iteration / interval: the task's (k, n) in the Parareal grid (-1 for idle gaps), so a
 * trace shows which iteration's wavefront ran when. */
typedef struct pswim_trace_event {
    int32_t worker;
    int32_t kind;
    double t_start;
    double t_end;
    int32_t iteration;
    int32_t interval;
} pswim_trace_event;

/* parareal::run (parareal.hpp:85-86, src/parareal.cpp:118-438) over HOST states with
 * caller-supplied host propagators: the physics-agnostic engine (regular / pipelined task
 * graph, worker lanes, stop rule, trace).  metric: point_dim-wise pointwise metric
 * (parareal.cpp:15-34) with point stride `metric_stride` (12 and dim 3 = rod positions,
 * io.cpp:49-68; stride = dim = d for pointwise_metric(d)).
 * states_out: (intervals+1) x len.  trace_out may be NULL; trace_cap bounds it and
 * *trace_len receives the number of events. */
int pswim_parareal_run_host(const pswim_plan* plan, pswim_propagator_fn coarse, void* coarse_user,
                            pswim_propagator_fn fine, void* fine_user, const double* h_x0,
                            int64_t len, int32_t metric_dim, int32_t metric_stride,
                            const double* h_reference /* (n+1) x len or NULL */,
                            double* h_states_out, pswim_report* report,
                            pswim_trace_event* trace_out, int64_t trace_cap, int64_t* trace_len);

/* parareal::run with GPU propagators: coarse = Euler(coarse_steps), fine = RK2(fine_steps)
 * as harness::prepare (src/harness.cpp:5-33).  Each engine worker owns one device context
 * (stream) on `device`; states stay in HBM.  h_x0 / h_states_out / h_reference are host. */
int pswim_parareal_run_gpu(const pswim_plan* plan, const pswim_scenario* sc, int device,
                           int64_t fine_steps, int64_t coarse_steps, const double* h_x0,
                           const double* h_reference, double* h_states_out, pswim_report* report,
                           pswim_trace_event* trace_out, int64_t trace_cap, int64_t* trace_len);

/* ---- time-sliced Parareal across ranks (one slice per GPU) ---------------------------- */
/* Transport between slice ranks.  Buffers are device pointers for GPU transports, host
 * pointers for host transports.  All calls are ordered on `stream` (NULL for host). */
typedef struct pswim_transport {
    void* user;
    int32_t rank;
    int32_t world;
    int (*send)(void* user, const double* buf, int64_t len, int32_t peer, void* stream);
    int (*recv)(void* user, double* buf, int64_t len, int32_t peer, void* stream);
    /* in-place elementwise max over ranks of `len` doubles */
    int (*allreduce_max)(void* user, double* buf, int64_t len, void* stream);
    /* recv[r * count + i] = send_of_rank_r[i] for every rank r (rank-major) */
    int (*allgather)(void* user, const double* send, double* recv, int64_t count, void* stream);
    /* optional (NULL = always healthy): 0 while the transport works, else a PSWIM_E* code
     * (NCCL: ncclCommGetAsyncError).  The rank drivers poll it while they wait on the device. */
    int (*health)(void* user);
    /* optional: abandon every pending operation so waits return (NCCL: ncclCommAbort).  Called
     * on a failure or on the PSWIM_COMM_TIMEOUT_S timeout (default 900 s). */
    void (*abort)(void* user);
} pswim_transport;

/* Device-buffer transport over a host-buffer wire (e.g. a torch.distributed gloo group or a
 * socket): each call drains the stream, stages through pinned host memory and calls the
 * wire's callbacks with host pointers.  For ranks that cannot use NCCL (several ranks on one
 * GPU); NCCL (pswim_nccl_transport_create) is the NVLink path.  The wire struct is copied. */
pswim_transport* pswim_staged_transport_create(const pswim_transport* host_wire, int device);
void pswim_staged_transport_destroy(pswim_transport* t);

/* Slice hand-off over peer memory (NVLink P2P / CUDA IPC; csrc/handoff.cu): the producing
 * kernel of rank p -- the corrector, or a push after the coarse sweep / the exact fine solve --
 * stores X[k][n] straight into rank p+1's receive slot k and releases a system-scope flag;
 * rank p+1 waits on the flag on its coarse stream and reads the slot in place.  Each rank
 * creates one on its device with `slots` >= max_iterations + 1 slots of `len` doubles, shares
 * the IPC handle (64 bytes; or the local base for ranks that are threads of one process) and
 * connects to rank p+1's (the last rank connects to nothing).  Replaces the ncclSend/ncclRecv
 * pair of the state hand-off; the transport then carries only the metric allreduce. */
typedef struct pswim_handoff pswim_handoff;
pswim_handoff* pswim_handoff_create(int device, int64_t len, int32_t slots);
int pswim_handoff_handle(pswim_handoff* h, uint8_t* handle64);
void* pswim_handoff_local_base(pswim_handoff* h);
int pswim_handoff_connect(pswim_handoff* h, const uint8_t* next_handle64 /* or NULL */,
                          void* next_local_base /* or NULL */);
/* Ranks that are threads of one process: the producing kernel still stores into the next
 * rank's slot, but the arrival is a CUDA event posted under a host lock instead of a
 * device-side flag spin (streams of one process share its hardware work queues, so a spin
 * could sit in front of the very store it waits for). */
int pswim_handoff_connect_local(pswim_handoff* h, pswim_handoff* next);
void pswim_handoff_destroy(pswim_handoff* h);

/* Rank driver: rank p owns interval p+1 of a plan with intervals == world.  Runs the
 * pipelined (or regular) Parareal recurrence of src/parareal.cpp:58-89 with one state
 * hand-off per iteration to rank p+1 (transport send/recv, or `handoff` when non-NULL) and
 * one allreduce(max) of the iteration metric.  Whole iterations are enqueued ahead of the
 * stop decisions (PSWIM_PARAREAL_LOOKAHEAD for tolerance plans; fixed-iteration plans, tol
 * < 1e-200, decide at the end), so the host never blocks per task.
 * Final boundary state X[k_final][p+1] goes to h_state_out; the report is identical on
 * every rank, and so is the schedule trace (every rank's coarse / corrector tasks on worker 0,
 * rank p's fine solves on worker p+1, device timestamps against a common start barrier,
 * idle gaps as ScheduleTrace::finalize_idle, schedule_trace.cpp:17-49; report.schedule_idle =
 * W).  trace_out may be NULL.  GPU form: fine = RK2, coarse = Euler on `device`. */
int pswim_parareal_rank_gpu(const pswim_plan* plan, const pswim_scenario* sc, int device,
                            const pswim_transport* tr, pswim_handoff* handoff /* or NULL */,
                            int64_t fine_steps, int64_t coarse_steps, const double* h_x0,
                            const double* h_reference_slice /* or NULL */, double* h_state_out,
                            pswim_report* report, pswim_trace_event* trace_out, int64_t trace_cap,
                            int64_t* trace_len);

/* Hybrid space x time: the rank is member q of the space group of slice
 * p.  time_tr connects the q-th members of all slices (rank = slice, world = intervals) and
 * carries the slice hand-offs and the metric allreduce exactly as pswim_parareal_rank_gpu;
 * space_coarse / space_fine (same group, rank = q, one per stream) all-gather (u, omega) of
 * the MRS sharded over the group inside every coarse / fine rhs.  Every member of a slice
 * computes the same values, bitwise equal to the unsharded rank driver. */
int pswim_parareal_rank_gpu_hybrid(const pswim_plan* plan, const pswim_scenario* sc, int device,
                                   const pswim_transport* time_tr, const pswim_transport* space_coarse,
                                   const pswim_transport* space_fine, int64_t fine_steps,
                                   int64_t coarse_steps, const double* h_x0,
                                   const double* h_reference_slice /* or NULL */, double* h_state_out,
                                   pswim_report* report, pswim_trace_event* trace_out,
                                   int64_t trace_cap, int64_t* trace_len);

/* Host form of the same rank driver (host propagators + host transport): used by the
 * world_size>1 CPU tests of the rank logic. */
int pswim_parareal_rank_host(const pswim_plan* plan, pswim_propagator_fn coarse, void* coarse_user,
                             pswim_propagator_fn fine, void* fine_user, const pswim_transport* tr,
                             const double* h_x0, int64_t len, int32_t metric_dim,
                             int32_t metric_stride, const double* h_reference_slice,
                             double* h_state_out, pswim_report* report, pswim_trace_event* trace_out,
                             int64_t trace_cap, int64_t* trace_len);

/* NCCL transport for one process per GPU.  The unique id (128 bytes) is produced by rank 0
 * with pswim_nccl_unique_id and distributed by the caller (e.g. torch.distributed store). */
int pswim_nccl_unique_id(uint8_t* id128);
pswim_transport* pswim_nccl_transport_create(const uint8_t* id128, int32_t rank, int32_t world,
                                             int device);
void pswim_nccl_transport_destroy(pswim_transport* tr);

/* In-process transports: `world` ranks as threads of one process (any device mix).  Returns
 * an array of `world` transports (index = rank); hand-offs are stream-ordered peer copies +
 * events, collectives host barriers.  `len` / `slots` size the send/recv staging (doubles per
 * message, messages per link). */
pswim_transport* pswim_threads_transports_create(int32_t world, const int* devices, int64_t len, int32_t slots);
void pswim_threads_transports_destroy(pswim_transport* trs);

/* ---- space-parallel MRS ------------------------------------------ */
/* propagate with the O(N^2) MRS sharded over the transport's ranks: every rank holds the full
 * state and does the O(N) rod loads / advance redundantly, computes the velocities of its own
 * 256-target blocks of the single-GPU launch plan, and all-gathers (u, omega) once per rhs
 * (48 B/node).  Bitwise identical to pswim_propagate on one GPU.  All ranks call it together. */
int pswim_propagate_sharded(pswim_ctx* ctx, const pswim_transport* tr, const double* d_in, double t0,
                            double t1, int scheme, int64_t steps_per_interval, double dt,
                            double* d_out);

/* Fused compute + collective: the same sharded propagate with the all-gather folded into
 * the MRS kernel's epilogue over peer memory.  Each rank creates a group on its context
 * (exchange block [arrival counter | u,w x 2] in its HBM), shares it either as a CUDA IPC
 * handle (64 bytes; one process per GPU, NVLink P2P) or as a raw device pointer (ranks as
 * threads of one process), and connects to every other rank's block.  The MRS kernel then
 * stores each target's (u, omega) into every rank's block and bumps every rank's counter with
 * a system-scope atomic; consumers wait with an acquire spin.  Bitwise identical to
 * pswim_propagate on one GPU. */
typedef struct pswim_peer_group pswim_peer_group;
pswim_peer_group* pswim_peer_group_create(pswim_ctx* ctx, int32_t rank, int32_t world);
int pswim_peer_group_handle(pswim_peer_group* g, uint8_t* handle64);
void* pswim_peer_group_local_base(pswim_peer_group* g);
/* handles: world x 64 bytes (IPC, other processes) or NULL; local_bases: world device
 * pointers (ranks of this process) or NULL.  Entry `rank` is ignored. */
int pswim_peer_group_connect(pswim_peer_group* g, const uint8_t* handles, void* const* local_bases);
void pswim_peer_group_destroy(pswim_peer_group* g);
int pswim_propagate_sharded_peer(pswim_ctx* ctx, pswim_peer_group* g, const double* d_in, double t0,
                                 double t1, int scheme, int64_t steps_per_interval, double dt,
                                 double* d_out);

/* In-process transport: `world` slice ranks as threads of one process, each on its own
 * context (any device mix), hand-offs by stream-ordered peer copies + events, or (handoff = 1)
 * by the peer-memory hand-off.  The trace is rank 0's (= every rank's) gathered trace. */
int pswim_parareal_run_threads(const pswim_plan* plan, const pswim_scenario* sc,
                               const int* devices /* world entries */, int64_t fine_steps,
                               int64_t coarse_steps, const double* h_x0,
                               const double* h_reference, double* h_states_out,
                               pswim_report* report, int32_t handoff, pswim_trace_event* trace_out,
                               int64_t trace_cap, int64_t* trace_len);

/* ---- microbenchmarks used by bench.py for the roofline denominators ------------------- */
/* Measured FP64 FMA throughput (FLOP/s, 2 per DFMA) of a register-resident DFMA loop over
 * the whole chip on the context's device; ms = kernel time. */
int pswim_dfma_peak(pswim_ctx* ctx, double* flops_per_s, double* ms);

/* Developer diagnostics: FP64 pipe microbenchmarks (kind 0 constant operands, 1 shared
 * register operands, 2 three distinct register pairs per DFMA, 3 DMUL, 4 kind 2 + MUFU.RSQ64H);
 * returns FP64 instructions per second (one lane-op each). */
int pswim_dev_fp64_probe(pswim_ctx* ctx, int kind, double* ops_per_s, double* ms);
/* Latency floors of the fused small-system kernel's per-rhs phases on this GPU, cycles each:
 * out4[0] front-pass chain (one warp per SMSP), out4[1] MRS items (ns sources per item, `warps`
 * warps), out4[2] the in-order reduction of `chunks` partials, out4[3] the velocity exchange of a
 * 16-CTA cluster (per_cta values per CTA, total over the cluster).  Dev diagnostics. */
int pswim_dev_latency_probe(pswim_ctx* ctx, int ns, int warps, int chunks, int per_cta, int total, double* out4);

/* Library version string. */
const char* pswim_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PSWIM_C_H */
