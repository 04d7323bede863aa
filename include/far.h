/* far.h — C-ABI of the B200-native batched FAR solver (arXiv 2507.13601).
 *
 * FAR = "Family of Allocations and Repartitioning", the three-phase moldable
 * scheduler of PAPER.md §3 (citations "P:<line>" refer to PAPER.md):
 *   phase 1  Turek family of allocations
 *   phase 2  Alg. 1, LPT + list scheduling over the MIG
 *            repartitioning tree with sequential reconfiguration P:374-463
 *   phase 3  Alg. 2, critical-task moves and swaps, then the
 *            line-26 replay of start/reconfiguration times
 * plus the multi-batch concatenation of §4.
 *
 * Every entry point runs on the GPU (sm_100a kernels in libfar.so).  There is
 * no CPU fallback: without a CUDA device every compute call returns FAR_E_CUDA.
 *
 * Units and layout
 *   - All times are int32 "ticks" chosen by the caller (1 tick = 1 ms in the
 *     bundled Table 2 costs).  Runtimes t_i(s) must be >= 1 (t_i maps to
 *     R+); they need NOT be monotone in s.
 *   - A runtime table is int32 [n][nsizes] per instance (C-contiguous), sizes in
 *     the profile's order: A30 {1,2,4}; A100/H100 {1,2,3,4,7}.  Many
 *     instances: [I][n][nsizes].
 *   - Integer range: per instance, sum_i max_s t_i(s) + sum over tree nodes of
 *     (t_create + t_destroy) must be < 2^29, so every makespan, start and the
 *     |2x - m| comparisons of Alg. 2 fit in int32 and a frontier key (end << 3 |
 *     first slice) fits in 32 bits.  Violations: FAR_E_BAD_TIME.
 *   - Tree node ids (far_task_slot.node) index the fixed repartitioning trees of
 *     Fig. 3: A30 0=[0,4) 1=[0,2) 2=[2,4) 3..6 = leaves S0..S3;
 *     A100/H100 0=[0,7) 1=[0,4) (hosts sizes 4 then 3) 2=[4,7) 3=[0,2) 4=[2,4)
 *     5=[4,6) 6=[6,7) 7..12 = leaves S0..S5.
 *
 * Ownership: the caller owns every buffer passed in; the library never frees
 * caller memory.  The library owns the far_ctx (constant tables, a lazily grown
 * device workspace and private streams), released by far_destroy.
 * Threading: one far_ctx per host thread; concurrent calls on one ctx are not
 * allowed.  Successive asynchronous calls on one ctx may use DIFFERENT streams:
 * the context orders the reuse of its internal workspaces across streams (an
 * event per launch), so a later call never overwrites a workspace an earlier
 * call on another stream is still reading.
 * Errors: every call returns far_status; far_last_error(ctx) gives a message.
 * Argument errors are reported synchronously.  Asynchronous calls
 * (far_solve_many, far_concat_streams) report per-instance input errors in
 * far_result.status (makespan = -1) and raise a sticky device flag that the next
 * far_sync() returns (bit 1: FAR_E_BAD_TIME, bit 2: FAR_E_INVALID_ARG, bit 4:
 * stream window overflow, FAR_E_TOO_LARGE); CUDA faults surface as FAR_E_CUDA.
 * The synchronous host-memory calls (far_schedule_batch, far_local_search,
 * far_solve_many_host) report only their OWN errors, through a private flag:
 * they never consume or misreport the asynchronous calls' pending flag.
 */
#ifndef FAR_H
#define FAR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct far_ctx far_ctx; /* opaque; owned by the library */

typedef enum { FAR_A30 = 0, FAR_A100 = 1, FAR_H100 = 2 } far_profile;

typedef enum {
  FAR_OK = 0,
  FAR_E_INVALID_ARG = 1,
  FAR_E_UNSUPPORTED_PROFILE = 2,
  FAR_E_BAD_TIME = 3,
  FAR_E_TOO_LARGE = 4,
  FAR_E_CUDA = 5,
  FAR_E_OOM = 6
} far_status;

/* far_opts.flags */
enum {
  FAR_NO_REFINE = 1u,     /* skip phase 3 (Alg. 2) and its replay */
  FAR_NO_GUARD = 2u,      /* return the replayed refined schedule even if worse than phase 2 */
  FAR_ZERO_RECONFIG = 4u, /* ignore the ctx's create/destroy costs (all zero) */
  FAR_NO_SCHEDULE = 8u,   /* solve_many: do not write per-task slots (makespans/results only) */
  FAR_EXHAUSTIVE = 16u,   /* run Alg. 1 on every family member (disable the exact lower-bound skip) */
  FAR_NONEMPTY_ALT = 32u, /* reading variant (R16): Alg. 2's alternative I^a must
                             already hold a task (default: any same-size node, P:524 literally) */
  FAR_NO_SEAM_MOVES = 64u,/* far_concat_streams: reversal + seam offset only, no seam move/swap
                             (Table 7's p_rev) */
  FAR_GROW_TIES = 128u    /* reading variant (R2): phase 1 grows every task tied for the
                             longest time in one step, as the formula of P:349 (default: one task,
                             the lowest index) */,
  FAR_BEST_IMPROVEMENT = 256u /* reading variant (R30; the north star's "evaluates every task
                             move and swap, recomputes the makespan and takes an argmin"): phase 3
                             scores every move to a same-size node and every swap pair on two
                             same-size nodes by (max slice end, #slices at it) and applies the
                             argmin while it improves; evals = candidates scored (default: Alg. 2,
                             P:495-560, FAR_NONEMPTY_ALT ignored) */,
  FAR_SWITCH_COST = 512u  /* reading variant (R7): the A100/H100 {S0..S3}
                             node runs an instance of its current task's size -- created with
                             t_create and destroyed with t_destroy of that size -- and is destroyed
                             and re-created (sequentially) when it switches from its size-4 to its
                             size-3 tasks (default: Alg. 1 literally, one size-4 instance).  Runs the
                             fused kernel; far_concat_streams, far_schedule_events and
                             far_validate_schedules reject it (FAR_E_INVALID_ARG) */
};

typedef struct {
  int32_t max_iterations;      /* Alg. 2 iteration cap; default 100 */
  int32_t min_improvement_ppm; /* 0 = off; else stop when 1e6*(w_prev - w) < ppm*w_prev */
  uint32_t flags;
} far_opts;

/* Per-instance report: 56 bytes. */
typedef struct {
  int32_t makespan;        /* final makespan (ticks); -1 on error */
  int32_t makespan_phase2; /* min over the family of Alg. 1 makespans (phase 2 result) */
  int32_t alloc_index;     /* k* : the winning family member (0-based) */
  int32_t family_size;     /* K : number of allocations in the family */
  int32_t moves, swaps;    /* phase 3 operations performed (Table 6 columns) */
  int32_t iterations;      /* phase 3 outer iterations executed */
  int32_t reverted;        /* 1 if the keep-best guard returned the phase-2 schedule */
  int32_t status;          /* far_status for this instance */
  int32_t reserved;
  int64_t evals;           /* phase 3 move/swap candidate evaluations */
  int64_t events;          /* Alg. 1 heap pops simulated: summed over every family member with
                              FAR_EXHAUSTIVE; otherwise over the members not skipped because
                              their lower bound max(h_max, ceil(area/#slices)) already reaches
                              the best makespan of earlier members (the result is identical) */
} far_result;

/* Per-task placement: 8 bytes.  start in ticks from the batch start. */
typedef struct {
  uint8_t node;      /* tree node id (see above) */
  uint8_t size_used; /* slices the task runs with: the node size, or 3 on the A100 4-slice node */
  uint8_t pad[2];
  int32_t start;
} far_task_slot;

/* Create a context for a MIG profile.
 * reconfig_cost: NULL -> Table 2 in 1 ms ticks; else int32[2][nsizes] =
 * {create[], destroy[]} in the profile's size order, each >= 0 (all zero = no
 * reconfiguration cost).  Unknown profile -> FAR_E_UNSUPPORTED_PROFILE. */
far_status far_create(far_profile profile, const int32_t *reconfig_cost, far_ctx **out);
/* Multi-target FAR (R31): one context schedules each instance on num_gpus
 * MIG GPUs of the profile at once -- "as many trees as GPUs, and initially, there is one node for
 * the root of each tree to start repartitioning on"; one Alg. 1 heap and one reconfig_end over the
 * forest, Alg. 2 alternatives among the same-size nodes of every tree.  Node ids: tree t's node v
 * is t*NN + v (NN = 7 A30, 13 A100/H100), its slices t*S + [lo, hi).  num_gpus in [1, 8]
 * (else FAR_E_INVALID_ARG); far_create(p, c, out) == far_create_multi(p, 1, c, out).  With
 * num_gpus > 1: far_solve_many / far_solve_many_host / far_schedule_batch / far_local_search /
 * far_lower_bounds take n <= 256 (else FAR_E_TOO_LARGE) and every flag (with
 * FAR_BEST_IMPROVEMENT the classes are the same-size nodes of all trees); far_concat_streams, far_schedule_events and
 * far_validate_schedules return FAR_E_UNSUPPORTED_PROFILE. */
far_status far_create_multi(far_profile profile, int32_t num_gpus, const int32_t *reconfig_cost, far_ctx **out);
int32_t far_num_gpus(const far_ctx *ctx);
void far_destroy(far_ctx *ctx);
int32_t far_num_sizes(const far_ctx *ctx);
const int32_t *far_sizes(const far_ctx *ctx);          /* nsizes values, host memory owned by ctx */
int32_t far_num_nodes(const far_ctx *ctx);   /* all trees of the context */
int32_t far_num_slices(const far_ctx *ctx);  /* all trees of the context */
/* Tree node table (host): lo[v], hi[v] slice interval [lo,hi), parent[v] (-1 for a root);
 * far_num_nodes(ctx) entries. */
far_status far_node_table(const far_ctx *ctx, int32_t *lo, int32_t *hi, int32_t *parent);
const char *far_last_error(const far_ctx *ctx);
/* Wait for all work queued by this ctx; returns FAR_E_BAD_TIME if any instance failed
 * its input checks since the last far_sync, FAR_E_CUDA on a device fault. */
far_status far_sync(far_ctx *ctx);

/* Phases 1-2 on ONE batch (host memory, synchronous): the family, Alg. 1 on
 * every member, k* = argmin (makespan, k).  sched[n] receives the
 * phase-2 schedule, res its report (moves = swaps = 0).  n in [0, 1024]. */
far_status far_schedule_batch(far_ctx *ctx, const int32_t *times, int32_t n, const far_opts *opts,
                              far_task_slot *sched, far_result *res);

/* Phase 3 (Alg. 2) + line-26 replay + keep-best guard on a given schedule
 * (host memory, synchronous).  sched[n] in/out: node lists are rebuilt from it ordered
 * by (start, task).  res in/out: on input res->makespan_phase2 is the guard reference
 * (if <= 0 the input schedule's own makespan is used). */
far_status far_local_search(far_ctx *ctx, const int32_t *times, int32_t n, const far_opts *opts,
                            far_task_slot *sched, far_result *res);

/* Phases 1-3 on I independent instances, DEVICE pointers, asynchronous on cuda_stream
 * (a cudaStream_t; NULL = legacy default stream).
 *   d_times    int32 [I][n][nsizes]
 *   d_makespan int32 [I]            (required)
 *   d_sched    far_task_slot [I][n] (or NULL, or ignored with FAR_NO_SCHEDULE)
 *   d_res      far_result [I]       (or NULL)
 * The buffers must stay valid until the stream reaches the call. */
far_status far_solve_many(far_ctx *ctx, const int32_t *d_times, int64_t I, int32_t n, const far_opts *opts,
                          int32_t *d_makespan, far_task_slot *d_sched, far_result *d_res, void *cuda_stream);

/* Same as far_solve_many on HOST buffers (synchronous).  The library pipelines chunks of
 * instances through its device workspace on two streams (H2D copy, solve, D2H copy
 * overlapped); host buffers may be pageable or pinned (pinned is faster).
 * This is the end-to-end public API the benchmark's "e2e" number measures. */
far_status far_solve_many_host(far_ctx *ctx, const int32_t *h_times, int64_t I, int32_t n, const far_opts *opts,
                               int32_t *h_makespan, far_task_slot *h_sched, far_result *h_res);

/* Multi-batch concatenation (§4) of S independent streams of B batches each,
 * DEVICE pointers, asynchronous on cuda_stream.  Every batch is FAR-scheduled (phases 1-3),
 * odd batches are reversed, and each stream is folded left to right with the seam
 * offset rule and the seam move/swap of DESIGN.md §9.
 *   d_times           int32 [S][B][n][nsizes]
 *   d_stream_makespan int64 [S][2]  {stream makespan (last task end), trivial-concatenation
 *                                     makespan}
 *   d_offsets         int64 [S][B]  absolute start offset of each batch
 *   d_sched           far_task_slot [S][B][n] (or NULL): node, size used and start RELATIVE to
 *                     the batch offset in the batch's final (possibly reversed) timeline
 *   d_batch_res       far_result [S][B] (or NULL): each batch's FAR report
 *   d_seam            int32 [S][B][4] (or NULL): {reversed, seam moves, seam swaps, reused instances}
 * The ctx workspace holds the intermediate per-batch schedules: calls on one ctx must be ordered
 * on one stream.  A stream whose placed-event window (256 events) overflows raises FAR_E_TOO_LARGE
 * at the next far_sync. */
far_status far_concat_streams(far_ctx *ctx, const int32_t *d_times, int64_t S, int32_t B, int32_t n,
                              const far_opts *opts, int64_t *d_stream_makespan, int64_t *d_offsets,
                              far_task_slot *d_sched, far_result *d_batch_res, int32_t *d_seam, void *cuda_stream);

/* ---- Checking and export of schedules.
 *
 * A reconfiguration event: kind 0 = create, 1 = destroy; node id; start and duration in
 * ticks (the create/destroy cost of the node's size, Table 2 / the ctx costs). */
typedef struct {
  int32_t kind;
  int32_t node;
  int32_t start;
  int32_t dur;
} far_event;

/* Reconfiguration events of I schedules (device memory, async on cuda_stream).  For each
 * instance the node lists are rebuilt from d_sched[I][n] (a task belongs to its node's list,
 * ordered by (start, task)) and the line-26 replay (Alg. 1's event loop taking each node's
 * tasks from its list) is run; its create events and the destroy events
 * issued while tasks remain unscheduled (Alg. 1 l.17-20) are written to
 * d_events[I][2 * far_num_nodes(ctx)] in start order (events are disjoint in time: sequential
 * reconfiguration), d_nev[I] = their number, d_makespan[I] (optional) = the
 * replay's makespan.  For a schedule returned by far_solve_many the replay reproduces its
 * starts (fixpoint), so these are exactly the schedule's reconfigurations.  An instance whose
 * slot names a node that does not host its size gets d_nev = -1.  Costs: the ctx's, or zero
 * with FAR_ZERO_RECONFIG in opts->flags.  Multi-target contexts (far_create_multi): the
 * replay runs over the forest (one heap, one reconfiguration sequence), node ids as in
 * far_node_table, n <= 256 (FAR_E_TOO_LARGE).  FAR_SWITCH_COST: FAR_E_INVALID_ARG. */
far_status far_schedule_events(far_ctx *ctx, const int32_t *d_times, int64_t I, int32_t n,
                               const far_task_slot *d_sched, const far_opts *opts, far_event *d_events,
                               int32_t *d_nev, int32_t *d_makespan, void *cuda_stream);

/* Feasibility check of I schedules with their events (device memory, async): d_violations[I]
 * = the number of violated conditions, 0 for a feasible schedule: (0) every slot names a node
 * hosting its size with start >= 0 (if not, only these are counted); (1) tasks on instances
 * sharing a slice never overlap in time; (2) at every task start the running
 * instances are pairwise disjoint tree nodes, i.e. a valid partition; (3) events
 * have the node's create/destroy duration, are pairwise disjoint in time, every
 * node with tasks is created exactly once before its first task and destroyed at most once
 * after its last, nodes without tasks have no events, and of two nodes sharing a slice the
 * earlier-created one is destroyed before the other is created.  d_events/d_nev as written
 * by far_schedule_events (nev <= 2 * far_num_nodes).  Multi-target contexts: the same
 * conditions over the forest's nodes and slices (n <= 256). */
far_status far_validate_schedules(far_ctx *ctx, const int32_t *d_times, int64_t I, int32_t n,
                                  const far_task_slot *d_sched, const far_opts *opts, const far_event *d_events,
                                  const int32_t *d_nev, int32_t *d_violations, void *cuda_stream);

/* Lower bound of the optimal makespan of I instances (device memory, async):
 * d_sum_min_work[I] = sum_i min_s s * t_i(s) (the paper's baseline is this / #slices, and
 * rho = makespan / baseline, Tables 4 and 9) and d_max_min_time[I] (or NULL) = max_i min_s t_i(s).
 * Both bound every schedule's makespan with or without reconfiguration. */
far_status far_lower_bounds(far_ctx *ctx, const int32_t *d_times, int64_t I, int32_t n, int64_t *d_sum_min_work,
                            int32_t *d_max_min_time, void *cuda_stream);

/* ---- Diagnostics (no compute; for bench.py and profiling).
 * Kernel stages of far_solve_many / far_concat_streams:
 *   PREP     H0-H3 (input checks, phase-1 family, per-size LPT lists), warp per instance
 *   MEMBER0  Alg. 1 for family member 0 (recorded), lane per instance
 *   MEMBERS  Alg. 1 for the members whose lower bound can still win, lane per (instance, member)
 *   WINNER   Alg. 1 re-run of k* != 0 (recorded), lane per instance
 *   FINISH   H6-H7 (phase 3, line-26 replay, guard, output), warp per instance
 *   OVERFLOW fused H0-H7 for the instances PREP deferred (family > 64 members), warp per instance
 *   FUSED    fused H0-H7 (far_schedule_batch, far_local_search, n = 1024), warp per instance
 *   STREAM   multi-batch fold of far_concat_streams, warp per stream
 *   CHECK    far_schedule_events / far_validate_schedules, warp per instance */
enum { FAR_STAGE_PREP = 0, FAR_STAGE_MEMBER0, FAR_STAGE_MEMBERS, FAR_STAGE_WINNER, FAR_STAGE_FINISH,
       FAR_STAGE_OVERFLOW, FAR_STAGE_FUSED, FAR_STAGE_STREAM, FAR_STAGE_CHECK, FAR_NUM_STAGES };
/* enable != 0: from now on every launch of the context is bracketed by CUDA events recorded
 * on the caller's stream (one event per stage boundary; the events add no synchronisation). */
far_status far_stage_timing(far_ctx *ctx, int32_t enable);
/* Waits for the timed launches, writes ms[FAR_NUM_STAGES] = device milliseconds per stage
 * summed over them, resets the sums, returns the number of timed solver launches (< 0 on a
 * CUDA error). ms may be NULL (reset only). */
int32_t far_stage_times(far_ctx *ctx, float *ms);
/* Number of kernels the context has launched since far_create (host-side count). */
int64_t far_launch_count(const far_ctx *ctx);
/* Roofline denominators measured on this GPU: a microbenchmark kernel of
 * independent 32-bit chains, timed with CUDA events on the default stream (synchronous).
 * mode 0: alu-pipe integer ops (IADD3/LOP3) -> *per_s = lane-ops/s; mode 1: alu + fma-pipe
 * integer ops (IADD3 + IMAD, the issue limit) -> lane-ops/s; mode 2: shared-memory loads ->
 * bytes/s.  Errors: FAR_E_INVALID_ARG, FAR_E_CUDA. */
far_status far_measure_peak(far_ctx *ctx, int32_t mode, double *per_s);

#ifdef __cplusplus
}
#endif
#endif /* FAR_H */
