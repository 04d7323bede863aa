/* far_oracle.h — C interface of the CPU ORACLE for FAR (arXiv 2507.13601).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load liboracle.so.  It
 * shares no code, header, table or helper with the CUDA path
 * (paper_2507_13601_b200/csrc, include/far.h).
 *
 * Conventions: profile 0 = A30, 1 = A100, 2 = H100.  times are int32
 * [n][|C_G|] in the profile's size order (A30: 1,2,4; A100/H100: 1,2,3,4,7),
 * in caller ticks.  costs are int32[2][|C_G|] = {create[], destroy[]}.
 * All internal arithmetic is int64.  Return value 0 = ok, <0 = error:
 *   -1 invalid argument, -2 unsupported profile, -3 bad time (t < 1 or
 *   negative cost), -4 too large (n > 1024).
 * Domain: every int32 time >= 1 and cost >= 0 (all arithmetic is int64; the
 * CUDA path's narrower range, include/far.h "Integer range", is its own).
 */
#ifndef FAR_ORACLE_H
#define FAR_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct { int32_t node, size_used; int64_t start; } orc_slot;
typedef struct { int32_t kind; /* 0 create, 1 destroy */ int32_t node; int64_t start, dur; } orc_event;
typedef struct {
  int64_t makespan;        /* final (after refinement+replay, or phase 2 if reverted/no refine) */
  int64_t makespan_phase2; /* H5: min over the family of Alg. 1 makespans */
  int64_t evals;           /* move/swap candidate evaluations */
  int64_t events;          /* Alg. 1 heap pops summed over all family members */
  int32_t alloc_index, family_size, moves, swaps, reverted, iterations;
} orc_result;

/* ORC_NONEMPTY_ALT: reading variant -- Alg. 2's alternative I^a
 * must hold at least one task (default: any same-size node, P:524 literally). */
/* ORC_NO_SEAM_MOVES: concatenation with reversal and seam offset only (Table 7's p_rev). */
/* ORC_GROW_TIES: reading variant: phase 1 grows every task tied for the
 * longest time in one step, as the formula of P:349 does (default: the lowest index only). */
/* ORC_BEST_IMPROVEMENT: reading variant (SURVEY.md §0 discrepancy 2 / NEXT-3, R30): phase 3
 * scores every same-size move and every swap pair by the resulting (makespan, #critical slices) and
 * applies the argmin while it improves (default: Alg. 2). */
/* ORC_SWITCH_COST: reading variant (R7): the A100/H100 {S0..S3} node
 * runs an instance of its current task's size (create/destroy cost of that size) and is destroyed and
 * re-created when it switches from its size-4 to its size-3 tasks (default: Alg. 1 literally). */
enum { ORC_NO_REFINE = 1u, ORC_NO_GUARD = 2u, ORC_ZERO_RECONFIG = 4u, ORC_NONEMPTY_ALT = 32u, ORC_NO_SEAM_MOVES = 64u,
       ORC_GROW_TIES = 128u, ORC_BEST_IMPROVEMENT = 256u, ORC_SWITCH_COST = 512u };

int orc_num_sizes(int profile);
int orc_num_nodes(int profile);
int orc_num_slices(int profile);
/* node table: lo[], hi[] (slice interval [lo,hi)), parent[] (-1 root) */
int orc_nodes(int profile, int32_t *lo, int32_t *hi, int32_t *parent);
/* All valid partitions: out[k*2*maxinst ...] = (start,size) pairs; counts[k] = #instances.
 * returns the number of partitions (or needed count if > maxparts). */
int orc_partitions(int profile, int32_t *out, int32_t *counts, int maxparts, int maxinst);
/* Phase 1 family: out[k][n] = size VALUES; returns K. */
int orc_family(int profile, const int32_t *times, int n, int32_t *out, int maxK);
int orc_family_flags(int profile, const int32_t *times, int n, uint32_t flags, int32_t *out, int maxK);
/* Alg. 1 on one allocation (size VALUES).  ev may be NULL. */
int orc_schedule_allocation(int profile, const int32_t *costs, const int32_t *times, int n,
                            const int32_t *alloc, orc_slot *slots, orc_event *ev, int32_t *nev,
                            int64_t *makespan, int64_t *pops);
/* FAR phases 1-3 + replay/guard.  ev may be NULL (events of the returned schedule). */
int orc_far(int profile, const int32_t *costs, const int32_t *times, int n, int32_t max_iterations,
            int32_t min_improvement_ppm, uint32_t flags, orc_slot *slots, orc_result *res,
            orc_event *ev, int32_t *nev);
/* Phase 3 + replay/guard on a given schedule (slots in/out).  res->makespan_phase2 in = the
 * input schedule's makespan (the guard's reference). */
int orc_refine(int profile, const int32_t *costs, const int32_t *times, int n, int32_t max_iterations,
               int32_t min_improvement_ppm, uint32_t flags, orc_slot *slots, orc_result *res,
               orc_event *ev, int32_t *nev);
int orc_schedule_allocation_flags(int profile, const int32_t *costs, const int32_t *times, int n,
                                  const int32_t *alloc, uint32_t flags, orc_slot *slots, orc_event *ev,
                                  int32_t *nev, int64_t *makespan, int64_t *pops);
/* orc_validate, or with ORC_SWITCH_COST the validator of that variant (instances change size). */
int orc_validate_flags(int profile, const int32_t *costs, const int32_t *times, int n, const orc_slot *slots,
                       const orc_event *ev, int32_t nev, uint32_t flags);
/* Zero-reconfiguration optimum by exhaustive branch and bound (tiny n). */
int64_t orc_bruteforce(int profile, const int32_t *times, int n);
/* Constraints 1-3 + lifecycle checks; returns #violations (0 = feasible). */
int orc_validate(int profile, const int32_t *costs, const int32_t *times, int n, const orc_slot *slots,
                 const orc_event *ev, int32_t nev);
/* Lower bound pieces: sum_i min_s s*t_i(s) and max_i min_s t_i(s). */
int orc_lower_bound(int profile, const int32_t *times, int n, int64_t *sum_min_work, int64_t *max_min_time);
/* Solve many instances [I][n][|C|] sequentially (for timing the baseline). */
/* Test entry (oracle pins of the seam offset): violations of the concatenation of batches 0..k
 * of orc_stream's fold when batch k starts delta ticks before its seam offset. */
int orc_stream_probe(int profile, const int32_t *costs, const int32_t *times, int B, int n, int k,
                     int64_t delta, int64_t *offset_k, int32_t *violations);
int orc_far_many(int profile, const int32_t *costs, const int32_t *times, int64_t I, int n,
                 int32_t max_iterations, int32_t min_improvement_ppm, uint32_t flags,
                 int64_t *makespans, orc_result *res);
/* orc_far_many plus every instance's schedule: slots[I][n] (NULL: none). */
int orc_far_many_slots(int profile, const int32_t *costs, const int32_t *times, int64_t I, int n,
                       int32_t max_iterations, int32_t ppm, uint32_t flags, int64_t *makespans, orc_result *res,
                       orc_slot *slots);

#ifdef __cplusplus
}
#endif
#endif
