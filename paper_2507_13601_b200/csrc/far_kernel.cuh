// far_kernel.cuh — fused sm_100a kernel: one WARP solves one FAR instance end to end.
//
//   H0 stage   : the instance's runtime table t[n][|C|] -> shared memory (int4 loads)
//   H1/H2      : phase 1, Turek family — warp argmax per growth step
//   H3         : per-size LPT lists (Alg. 1 lines 1-2) of every (task, size)
//                that some family member uses, each entry tagged with the member
//                interval [lo, hi) in which the task has that size
//   H4         : phase 2, Alg. 1 for every family member IN PARALLEL, one
//                member per lane; the heap of frontier nodes is a register array
//                indexed by first slice (the frontier is an antichain, so the first
//                slice is a unique key and the (end, lo) tie-break is the scan order)
//   H5         : k* = argmin (makespan_k, k) by two REDUX.MIN
//   H6         : phase 3, Alg. 2: warp-parallel move / swap candidate
//                search with deterministic packed-key argmins
//   H7         : line-26 replay + keep-best guard, coalesced output stores
//
// Readings of the paper: DESIGN.md "Readings" (identical to the oracle's; the two
// share no code).  All times int32.
#pragma once
#include <climits>
#include <cstdint>
#include <type_traits>

#include "../../include/far.h"
#include "far_tree.cuh"

namespace farb {

constexpr unsigned FULL = 0xffffffffu;
constexpr int MAXN = 1024;
constexpr int BOUND = 1 << 29;
enum { MODE_SOLVE = 0, MODE_LOCAL = 1 };
// internal flag bits (never part of the public far_opts.flags; set by the C-ABI for experiments)
constexpr unsigned FAR_I_NO_ROUND_BALANCE = 1u << 30;  // FAR_DEBUG_NO_ROUND_BALANCE: members keep the full grid

struct KParams {
  const int32_t* times;
  int64_t I;
  int n;
  int32_t* makespan;
  far_task_slot* sched;
  far_result* res;
  const far_task_slot* sched_in;  // MODE_LOCAL
  const far_result* res_in;       // MODE_LOCAL
  int cr[8], de[8];               // create / destroy cost per size index (ticks)
  int max_it, ppm;
  unsigned flags;
  int mode;
  unsigned long long* counter;  // dynamic instance scheduler (reset to 0 before launch)
  int* errflag;                 // sticky input-error flag
  int kcap;                     // family-size capacity of the shared-memory layout
  unsigned* ovf;                // bit per instance: family larger than kcap -> overflow pass
  unsigned long long* ovf_count;
  int ovf_pass;                 // 1: solve only the instances flagged in ovf (full layout)
  // pipelined phase 2 workspace (far_pipeline.cuh), strides in elements
  int2* ws_ent;                 // [I][ws_ecap1] list entries {t | task << 22, lo | hi << 16}
  int* ws_lb;                   // [I][ws_kcap]  lower bound of each member's makespan
  unsigned long long* ws_cnt;   // [I][ws_kcap]  packed size counts of each member
  int* ws_meta;                 // [I][16]       loff[0..NC], flag (WS_FLAG), K (WS_K)
  unsigned long long* ws_best;  // [I]           min over simulated members of (makespan << 16 | k)
  unsigned long long* ws_evt;   // [I]           Alg. 1 pops simulated
  uint32_t* ws_rec;             // [I][n]        k*'s placement: node | size idx << 4 | position << 7
  int* ws_sl;                   // [I][8]        k*'s slice ends
  int ws_ecap1, ws_kcap;
  int rsum;                     // sum over tree nodes of create + destroy cost (integer-range check)
  uint16_t* ws_ncnt;            // [I][16]       k*'s node list lengths (lane-per-instance finish)
  uint32_t* ws_m0;              // [I][ws_n4]    member 0's compact per-size LPT lists (t | task << 22)
  int ws_n4;
  uint32_t* ws_d0;              // [I][ws_n4]    member 0's duration per task t_j(a1_j) (finish, k* = 0)
  int64_t* gen_list;            // [I]           instances for the general prep (far_prep.cuh)
  unsigned long long* gen_count;
};
enum { PIPE_NONE = 0, PIPE_PREP = 1 };  // far_solve_kernel template modes: fused / H0-H3 -> ws
enum { WS_FLAG = 8, WS_K = 9 };  // ws_meta slots: flag 0 = phase 2 pending, 1 = finished or deferred

// misc int slots (PIPE_PREP keeps only the first M_PREP_END: list offsets, node table, costs)
enum { M_LOFF = 0, M_NINFO = 8, M_CR = 24, M_DE = 32, M_PREP_END = 40, M_NCNT = 40, M_NSUM = 56, M_SEND = 72,
       M_BSEND = 80, M_LIFE = 88, M_MEMB = 184, M_END = 216 };

// Per-warp shared-memory layout (bytes), identical on host and device.  kcap bounds the
// family size K this layout holds (the per-size lists hold at most n + K - 1 entries).
struct Layout {
  int times, lent, ltask, cnts, lbs, lbh, cur, su, bestnode, scratch, lstate, start, misc, bytes, ecap, scr;
};

__host__ __device__ inline int al16(int x) { return (x + 15) & ~15; }

__host__ __device__ inline Layout make_layout(int n, int NC, int S, int NN, int kcap, int pipe = 0) {
  Layout L;
  (void)S;
  int Ecap = n + kcap - 1;
  if (Ecap > n * NC) Ecap = n * NC;
  if (Ecap < 0) Ecap = 0;
  L.ecap = Ecap;
  int o = 0;
  L.times = o;    o = al16(o + 4 * n * NC);
  L.lent = o;     o = al16(o + 8 * (Ecap + 1));
  L.ltask = o;    o = al16(o + 2 * (Ecap + 1));
  L.cnts = o;     o = al16(o + 8 * kcap);
  L.lbs = o;      o = al16(o + 4 * kcap);
  L.lbh = o;      o = al16(o + 4 * kcap);
  L.cur = o;      o = al16(o + n);
  L.su = o;       o = al16(o + n);
  L.bestnode = o; o = al16(o + n);
  int sc;
  if (pipe == 1) {  // PIPE_PREP: u16 member intervals, the rank-sort keys, the long-list sort
    sc = 2 * n * NC;
    if (4 * n > sc) sc = 4 * n;
    if (n > 128 && 10 * Ecap > sc) sc = 10 * Ecap;
  } else {
    sc = 32 * n;                                  // phase-2 node record [n][32]
    if (10 * Ecap > sc) sc = 10 * Ecap;           // list sort scratch
    if (4 * n * NC > sc) sc = 4 * n * NC;         // phase-1 member intervals
    if (2 * NN * n + 4 * n + 4 > sc) sc = 2 * NN * n + 4 * n + 4;  // node lists + durations
  }
  L.scratch = o;  o = al16(o + sc);
  L.scr = sc;
  L.lstate = o;   o = al16(o + (pipe == 1 ? 4 * kcap : 4 * NC * 32));  // PIPE_PREP: growth-step ranks only
  L.start = o;    o = al16(o + (pipe == 1 ? 0 : 4 * n));
  L.misc = o;     o = al16(o + 4 * (pipe == 1 ? (int)M_PREP_END : (int)M_END));
  L.bytes = o;
  return L;
}

// c += (v >= k) for unsigned v, k: the carry of v - k (no borrow) added in one pair
__device__ __forceinline__ void count_ge(int& c, unsigned v, unsigned k) {
  asm("{\n\t.reg .u32 t;\n\tsub.cc.u32 t, %1, %2;\n\taddc.u32 %0, %0, 0;\n\t}" : "+r"(c) : "r"(v), "r"(k));
}

// c += ((vhi, vlo) >= (khi, klo)) as unsigned 64-bit
__device__ __forceinline__ void count_ge64(int& c, unsigned vlo, unsigned vhi, unsigned klo, unsigned khi) {
  asm("{\n\t.reg .u32 t;\n\tsub.cc.u32 t, %1, %3;\n\tsubc.cc.u32 t, %2, %4;\n\taddc.u32 %0, %0, 0;\n\t}"
      : "+r"(c) : "r"(vlo), "r"(vhi), "r"(klo), "r"(khi));
}

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// slices of size index c: A30 {1,2,4}; A100/H100 {1,2,3,4,7}
template <int NC> __host__ __device__ __forceinline__ int size_of(int c) {
  return NC == 3 ? (c == 2 ? 4 : c + 1) : (c == 4 ? 7 : c + 1);
}
// leaf node of slice s (node ids of include/far.h)
template <int NC> __device__ __forceinline__ int leaf_of(int s) {
  return NC == 3 ? 3 + s : (s < 6 ? 7 + s : 6);
}

// ---------------------------------------------------------------------------
// Frontier of Alg. 1: slot s (= first slice) holds the node starting at s, its end
// time, and whether it already has tasks.  Pop = min (end, slot) by an unrolled scan.
// ---------------------------------------------------------------------------
template <int S> struct Frontier {
  // e[s] = end << 3 | s (ends < 2^29, include/far.h "Integer range"); 0xFFFFFFFF = empty.
  // The unsigned min over the slots is exactly the (end, first slice) tie-break.
  unsigned e[S];
  uint32_t slotnode = 0, live = 1, has = 0;
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int s = 0; s < S; ++s) e[s] = 0xFFFFFFFFu;
    e[0] = 0;
    slotnode = 0;  // root (node 0) in slot 0
    live = 1;
    has = 0;
  }
  __device__ __forceinline__ void pop(int& bs, int& be) const {
    unsigned m;
    if (S == 7) {
      m = min(min(min(e[0], e[1]), min(e[2], e[3])), min(min(e[4], e[5]), e[S - 1]));
    } else {
      m = e[0];
#pragma unroll
      for (int s = 1; s < S; ++s) m = min(m, e[s]);
    }
    bs = (int)(m & 7u);
    be = (int)(m >> 3);
  }
  __device__ __forceinline__ void set(int bs, int v) {
    const unsigned key = ((unsigned)v << 3) | (unsigned)bs;
#pragma unroll
    for (int s = 0; s < S; ++s) e[s] = (s == bs) ? key : e[s];
  }
  __device__ __forceinline__ void clear(int bs) {
#pragma unroll
    for (int s = 0; s < S; ++s) e[s] = (s == bs) ? 0xFFFFFFFFu : e[s];
  }
  __device__ __forceinline__ int endv(int s) const { return (int)(e[s] >> 3); }
  __device__ __forceinline__ int node(int s) const { return (slotnode >> (4 * s)) & 15; }
  // Alg. 1 lines 17-24 (repartitioning) after the optional destroy; returns false if v was a leaf.
  __device__ __forceinline__ bool split(int bs, int be, uint32_t w) {
    has &= ~(1u << bs);
    const int ch1 = nd_ch1(w);
    if (ch1 != LEAF) {
      const int s2 = nd_ch2lo(w);
      slotnode = (slotnode & ~(15u << (4 * bs))) | ((uint32_t)ch1 << (4 * bs));
      slotnode = (slotnode & ~(15u << (4 * s2))) | ((uint32_t)nd_ch2(w) << (4 * s2));
      live |= 1u << s2;
      set(s2, be);  // C.end := I.end for both children (slot bs keeps be)
      return true;
    }
    live &= ~(1u << bs);
    clear(bs);
    return false;
  }
};

// The same frontier kept SORTED by key (end << 3 | slot), for the hot Alg. 1 simulations of the
// member kernels: the pop is k[0] (no min tree); a placement replaces the popped key by a larger one
// (remove the front, sorted insert: one min and one max per position), a split inserts the second
// child's key (the first child keeps slot bs and the popped key), a dropped leaf shifts the keys
// down.  The keys are unique (slot bits), so the order -- and every pop -- is Frontier's.
template <int S> struct SFrontier {
  unsigned k[S];  // ascending; 0xFFFFFFFF = empty
  uint32_t slotnode = 0, live = 1, has = 0;
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int s = 0; s < S; ++s) k[s] = 0xFFFFFFFFu;
    k[0] = 0;  // root (node 0) in slot 0 at time 0
    slotnode = 0;
    live = 1;
    has = 0;
  }
  __device__ __forceinline__ void pop(int& bs, int& be) const {
    bs = (int)(k[0] & 7u);
    be = (int)(k[0] >> 3);
  }
  __device__ __forceinline__ int node(int s) const { return (slotnode >> (4 * s)) & 15; }
  // the popped slot bs gets end v (>= its old end): remove the front, insert the new key
  __device__ __forceinline__ void set_front(int bs, int v) {
    const unsigned key = ((unsigned)v << 3) | (unsigned)bs;
    unsigned f[S];
    f[0] = min(k[1], key);
#pragma unroll
    for (int s = 1; s < S - 1; ++s) f[s] = min(k[s + 1], max(k[s], key));
    f[S - 1] = max(k[S - 1], key);
#pragma unroll
    for (int s = 0; s < S; ++s) k[s] = f[s];
  }
  __device__ __forceinline__ void insert(unsigned key) {  // k[S - 1] is empty
    unsigned f[S];
    f[0] = min(k[0], key);
#pragma unroll
    for (int s = 1; s < S; ++s) f[s] = min(k[s], max(k[s - 1], key));
#pragma unroll
    for (int s = 0; s < S; ++s) k[s] = f[s];
  }
  __device__ __forceinline__ int endv(int s) const {
    int e = 0;
#pragma unroll
    for (int q = 0; q < S; ++q)
      if (k[q] != 0xFFFFFFFFu && (int)(k[q] & 7u) == s) e = (int)(k[q] >> 3);
    return e;
  }
  // Alg. 1 lines 17-24 (repartitioning) after the optional destroy; returns false if v was a leaf.
  __device__ __forceinline__ bool split(int bs, int be, uint32_t w) {
    has &= ~(1u << bs);
    const int ch1 = nd_ch1(w);
    if (ch1 != LEAF) {
      const int s2 = nd_ch2lo(w);
      slotnode = (slotnode & ~(15u << (4 * bs))) | ((uint32_t)ch1 << (4 * bs));
      slotnode = (slotnode & ~(15u << (4 * s2))) | ((uint32_t)nd_ch2(w) << (4 * s2));
      live |= 1u << s2;
      insert(((unsigned)be << 3) | (unsigned)s2);  // C.end := I.end for both children
      return true;
    }
    live &= ~(1u << bs);
#pragma unroll
    for (int s = 0; s < S - 1; ++s) k[s] = k[s + 1];
    k[S - 1] = 0xFFFFFFFFu;
    return false;
  }
};

// ---------------------------------------------------------------------------
// Node-level replay (Alg. 2 line 26, O7).  Between two reconfiguration events of the
// Alg. 1 event loop only task placements happen, and a node's tasks run back to back, so
// the loop is replayed at node granularity: each node contributes a CREATE event at its
// push key (a_v, lo_v) and a SPLIT event at (f_v, lo_v), f_v = creation end + sum of its
// durations.  The event loop pops keys in non-decreasing (time, first slice) order, so
// both loops apply the same reconfiguration events in the same order and give identical
// starts (a destroy charged after the last task started cannot delay any creation).  This
// takes <= 2*#nodes heap steps instead of n + #nodes; task starts are then prefix sums
// over each node list (one lane per node).  life[v*6] = {cs, ce, ds, de, creation pop time, end}.
// The frontier is spread over the warp: lane s < S holds slot s's key
// (end << 3 | s); the control state (rec, has, slot -> node map, live) is uniform, so every
// lane follows the same path and a pop is one REDUX.MIN instead of an unrolled scan.
template <int NC>
__device__ int node_sim_warp(const int* ncnt, const int* nsum, int* life, const uint32_t* ninfo, const int* cr,
                             const int* de, int lane, int& Eout) {
  constexpr int NN = Tree<NC>::NN;
  if (lane < NN) {
    life[lane * 6 + 0] = -1;  // not created
    life[lane * 6 + 2] = -1;  // not destroyed
  }
  __syncwarp();  // lane 0 writes these slots below
  unsigned e = lane == 0 ? 0u : 0xFFFFFFFFu;  // root in slot 0 at time 0
  uint32_t slotnode = 0, live = 1, has = 0;
  int rec = 0, ms = 0, E = 0;
  while (live) {
    const unsigned m = __reduce_min_sync(FULL, e);
    const int bs = (int)(m & 7u), be = (int)(m >> 3);
    const int v = (int)((slotnode >> (4 * bs)) & 15u);
    const uint32_t w = ninfo[v];
    if (!((has >> bs) & 1) && ncnt[v] > 0) {  // creation (lines 8-11), then all of v's tasks
      const int cs = max(rec, be);
      rec = cs + cr[nd_szi(w)];
      const int f = rec + nsum[v];
      if (lane == 0) {
        life[v * 6 + 0] = cs;
        life[v * 6 + 1] = rec;
        life[v * 6 + 4] = be;  // pop time of the creation (= first task's placement pop)
        life[v * 6 + 5] = f;   // end of the node's tasks (its split / destroy pop)
      }
      ms = max(ms, f);
      E = max(E, f);
      has |= 1u << bs;
      if (lane == bs) e = ((unsigned)f << 3) | (unsigned)bs;
    } else {  // repartitioning (lines 17-24): destroy if it had tasks, then split or drop
      if ((has >> bs) & 1) {
        const int ds = max(rec, be);
        rec = ds + de[nd_szi(w)];
        if (lane == 0) {
          life[v * 6 + 2] = ds;
          life[v * 6 + 3] = rec;
        }
        E = max(E, rec);
      }
      has &= ~(1u << bs);
      const int ch1 = nd_ch1(w);
      if (ch1 != LEAF) {  // children: slot bs (keeps its key) and slot ch2lo, both at be
        const int s2 = nd_ch2lo(w);
        slotnode = (slotnode & ~(15u << (4 * bs))) | ((uint32_t)ch1 << (4 * bs));
        slotnode = (slotnode & ~(15u << (4 * s2))) | ((uint32_t)nd_ch2(w) << (4 * s2));
        live |= 1u << s2;
        if (lane == s2) e = ((unsigned)be << 3) | (unsigned)s2;
      } else {
        live &= ~(1u << bs);
        if (lane == bs) e = 0xFFFFFFFFu;
      }
    }
  }
  Eout = E;
  return ms;
}

template <int NC>
__device__ __forceinline__ int dur_of(const int32_t* T, const uint8_t* su, int j) {
  return T[j * NC + su[j]];
}

// Replay of node lists nlist[v][0..ncnt[v]) with task durations D[j] -> start[j], onode[j];
// returns the makespan.  Prefix sums over each node list are warp scans.
template <int NC>
__device__ int replay_warp(int n, const int* D, const uint16_t* nlist, const int* ncnt, int* nsum, int* life,
                           int* start, uint8_t* onode, const uint32_t* ninfo, const int* cr, const int* de, int lane,
                           int* Eout = nullptr) {
  constexpr int NN = Tree<NC>::NN;
  if (lane < NN) {  // one lane per node: exclusive prefix of durations along its list
    int acc = 0;
    for (int q = 0; q < ncnt[lane]; ++q) {
      const int j = nlist[lane * n + q];
      start[j] = acc;  // relative to the node's creation end
      onode[j] = (uint8_t)lane;
      acc += D[j];
    }
    nsum[lane] = acc;
  }
  __syncwarp();
  int E = 0;
  const int ms = node_sim_warp<NC>(ncnt, nsum, life, ninfo, cr, de, lane, E);
  __syncwarp();
  for (int j2 = lane; j2 < n; j2 += 32) start[j2] += life[onode[j2] * 6 + 1];
  __syncwarp();
  if (Eout) *Eout = E;
  return ms;
}

// Task-level replay (Alg. 2 line 26) for the reading variant FAR_SWITCH_COST (R7): the
// Alg. 1 event loop taking each node's tasks from its list, where the two-size {S0..S3} node
// runs an instance of its task's size (su[j]) -- created with that size's cost, destroyed and
// re-created when consecutive tasks differ in size -- so a node's tasks no longer run back to
// back and the node-level replay does not apply.  Frontier spread over the lanes as in
// node_sim_warp; cursor[NN] is scratch.  Writes start[j], onode[j]; returns the makespan.
template <int NC>
__device__ __noinline__ int replay_tasks_warp(int n, const int* D, const uint16_t* nlist, const int* ncnt,
                                              const uint8_t* su, int* cursor, int* start, uint8_t* onode,
                                              const uint32_t* ninfo, const int* cr, const int* de, int lane) {
  constexpr int NN = Tree<NC>::NN;
  if (lane < NN) cursor[lane] = 0;
  __syncwarp();
  unsigned e = lane == 0 ? 0u : 0xFFFFFFFFu;  // root in slot 0 at time 0
  uint32_t slotnode = 0, live = 1, has = 0;
  int rec = 0, ms = 0, unsched = n, isz = 0;
  while (live) {
    const unsigned m = __reduce_min_sync(FULL, e);
    const int bs = (int)(m & 7u);
    int be = (int)(m >> 3);
    const int v = (int)((slotnode >> (4 * bs)) & 15u);
    const uint32_t w = ninfo[v];
    const int q = cursor[v];
    __syncwarp();
    if (q < ncnt[v]) {  // lines 7-16: the node's next task
      const int j = nlist[v * n + q];
      const int c = su[j];
      if (!((has >> bs) & 1)) {
        rec = max(rec, be) + cr[c];
        be = rec;
        has |= 1u << bs;
        if (nd_c1(w) != NONE) isz = c;  // the (one) two-size node's instance
      } else if (nd_c1(w) != NONE && c != isz) {  // the instance changes size
        rec = max(rec, be) + de[isz];
        rec += cr[c];
        be = rec;
        isz = c;
      }
      if (lane == 0) {
        start[j] = be;
        onode[j] = (uint8_t)v;
        cursor[v] = q + 1;
      }
      be += D[j];
      ms = max(ms, be);
      --unsched;
      if (lane == bs) e = ((unsigned)be << 3) | (unsigned)bs;
    } else if (unsched > 0) {  // lines 17-24
      if ((has >> bs) & 1) rec = max(rec, be) + de[nd_c1(w) != NONE ? isz : nd_szi(w)];
      has &= ~(1u << bs);
      const int ch1 = nd_ch1(w);
      if (ch1 != LEAF) {
        const int s2 = nd_ch2lo(w);
        slotnode = (slotnode & ~(15u << (4 * bs))) | ((uint32_t)ch1 << (4 * bs));
        slotnode = (slotnode & ~(15u << (4 * s2))) | ((uint32_t)nd_ch2(w) << (4 * s2));
        live |= 1u << s2;
        if (lane == s2) e = ((unsigned)be << 3) | (unsigned)s2;
      } else {
        live &= ~(1u << bs);
        if (lane == bs) e = 0xFFFFFFFFu;
      }
    } else {  // drop
      live &= ~(1u << bs);
      if (lane == bs) e = 0xFFFFFFFFu;
    }
    __syncwarp();
  }
  return ms;
}

// ---------------------------------------------------------------------------
// Phase 3: Alg. 2 on node lists (warp-cooperative).  sliceEnd in smem.
// ---------------------------------------------------------------------------
// Remove task j from an ordered node list (warp: ballot to find it, chunked shift left).
template <int NC>
__device__ void list_remove(uint16_t* lst, int* cnt, int j, int lane) {
  const int c = *cnt;
  if (c <= 32) {  // one chunk: find by ballot, shift left by a shuffle
    const int x = lane < c ? lst[lane] : -1;
    const unsigned m = __ballot_sync(FULL, x == j);
    const int q = __ffs(m) - 1;
    const int y = __shfl_down_sync(FULL, x, 1);
    __syncwarp();
    if (lane >= q && lane < c - 1) lst[lane] = (uint16_t)y;
    if (lane == 0) *cnt = c - 1;
    __syncwarp();
    return;
  }
  int q = c;
  for (int b = 0; b < c; b += 32) {
    const unsigned m = __ballot_sync(FULL, b + lane < c && lst[b + lane] == j);
    if (m) { q = b + __ffs(m) - 1; break; }
  }
  for (int b = q; b < c - 1; b += 32) {
    const int i = b + lane;
    const uint16_t v = i < c - 1 ? lst[i + 1] : 0;
    __syncwarp();
    if (i < c - 1) lst[i] = v;
    __syncwarp();
  }
  if (lane == 0) *cnt = c - 1;
  __syncwarp();
}

// "Insert T in I^a.tasks ordered by T.time": decreasing time, ties -> lower index.
// Warp: the insertion point is the first entry not ordered before j (the oracle's linear scan;
// on a sorted list it is the number of entries before j, and input schedules of
// far_local_search need not be sorted); chunked shift right.
template <int NC>
__device__ void list_insert(uint16_t* lst, int* cnt, int j, const int* D, int lane) {
  const int c = *cnt;
  const int dj = D[j];
  if (c < 32) {  // one chunk: position by ballot, shift right by a shuffle
    const int x = lane < c ? lst[lane] : 0;
    bool nb = false;
    if (lane < c) {
      const int dx = D[x];
      nb = !(dx > dj || (dx == dj && x < j));
    }
    const unsigned m = __ballot_sync(FULL, nb);
    const int pos = m ? __ffs(m) - 1 : c;
    const int y = __shfl_up_sync(FULL, x, 1);
    __syncwarp();
    if (lane <= c) lst[lane] = (uint16_t)(lane < pos ? x : (lane == pos ? j : y));
    if (lane == 0) *cnt = c + 1;
    __syncwarp();
    return;
  }
  int pos = c;
  for (int b = 0; b < c; b += 32) {
    const int i = b + lane;
    bool nb = false;
    if (i < c) {
      const int x = lst[i];
      const int dx = D[x];
      nb = !(dx > dj || (dx == dj && x < j));
    }
    const unsigned m = __ballot_sync(FULL, nb);
    if (m) { pos = b + __ffs(m) - 1; break; }
  }
  for (int top = c - 1; top >= pos; top -= 32) {
    const int i = top - lane;
    const uint16_t v = i >= pos ? lst[i] : 0;
    __syncwarp();
    if (i >= pos) lst[i + 1] = v;
    __syncwarp();
  }
  if (lane == 0) {
    lst[pos] = (uint16_t)j;
    *cnt = c + 1;
  }
  __syncwarp();
}

template <int NC>
__device__ void refine_warp(int n, const int* D, uint16_t* nlist, int* ncnt, int* send,
                            const uint32_t* ninfo, int max_it, int ppm, bool nonempty_alt, int lane, int& moves,
                            int& swaps, int& iters, long long& evals) {
  constexpr int S = Tree<NC>::S, NN = Tree<NC>::NN;
  auto end_of = [&](uint32_t w) {
    int e = 0;
    const int lo = nd_lo(w), hi = lo + nd_sz(w);
    for (int s = lo; s < hi; ++s) e = max(e, send[s]);
    return e;
  };
  auto add_on = [&](uint32_t w, int d) {
    const int lo = nd_lo(w);
    if (lane >= lo && lane < lo + nd_sz(w)) send[lane] += d;
    __syncwarp();
  };
  int omega = __reduce_max_sync(FULL, lane < S ? send[lane] : 0);
  moves = swaps = iters = 0;
  evals = 0;
  bool stop = false;
  while (!stop && iters < max_it) {
    ++iters;
    const int omega_prev = omega;
    unsigned long long Q = 0;  // FIFO of node ids, 4 bits each
    int qh = 0, qt = 0;
    uint32_t opened = 0;
    // line 5: leaves of the slices reaching omega, ascending slice order
    for (unsigned crit = __ballot_sync(FULL, lane < S && send[lane] == omega); crit; crit &= crit - 1) {
      const int leaf = leaf_of<NC>(__ffs(crit) - 1);
      Q |= (unsigned long long)leaf << (4 * qt++);
      opened |= 1u << leaf;
    }
    while (qh < qt) {
      const int I = (int)((Q >> (4 * qh++)) & 15);
      if (I == 0) { stop = true; break; }
      const uint32_t wI = ninfo[I];
      // alternative I^a: same size, != I, minimum (end, first slice) -- lanes over nodes
      bool valid = false;
      int eu = INT_MAX, lou = 15;
      if (lane < NN && lane != I && nd_sz(ninfo[lane]) == nd_sz(wI) && (!nonempty_alt || ncnt[lane] > 0)) {
        valid = true;
        eu = end_of(ninfo[lane]);
        lou = nd_lo(ninfo[lane]);
      }
      const int eA = __reduce_min_sync(FULL, eu);
      const bool c1 = valid && eu == eA;
      const int lmin = __reduce_min_sync(FULL, c1 ? lou : 15);
      const unsigned sel = __ballot_sync(FULL, c1 && lou == lmin);
      const int A = sel ? __ffs(sel) - 1 : -1;
      bool done = false;
      if (A >= 0) {
        const int m = omega - eA;
        const int nI = ncnt[I];
        uint16_t* LI = nlist + I * n;
        uint16_t* LA = nlist + A * n;
        evals += nI;
        // move: argmin (|2t - m|, index) over t < m
        unsigned bd = UINT_MAX;
        int bj = INT_MAX;
        for (int q = lane; q < nI; q += 32) {
          const int j = LI[q];
          const int t = D[j];
          if (t < m) {
            const unsigned d = (unsigned)abs(2 * t - m);
            if (d < bd || (d == bd && j < bj)) { bd = d; bj = j; }
          }
        }
        const unsigned dmin = __reduce_min_sync(FULL, bd);
        // an operation is one or two transfers (task, from, to); one call site keeps code small
        int nt = 0, tk0 = 0, tk1 = 0, delta = 0;
        if (dmin != UINT_MAX) {
          tk0 = __reduce_min_sync(FULL, (unsigned)(bd == dmin ? bj : INT_MAX));
          delta = D[tk0];
          nt = 1;
          ++moves;
        } else {
          const int nA = ncnt[A];
          evals += (long long)nI * nA;
          unsigned bd2 = UINT_MAX, bkey = UINT_MAX;
          const int tot = nI * nA;
          const int di = 32 / max(nA, 1), da = 32 - di * nA;
          int qi = lane / max(nA, 1), qa = lane - qi * nA;
          for (int p = lane; p < tot; p += 32) {
            const int k = LI[qi], j = LA[qa];
            qi += di;
            qa += da;
            if (qa >= nA) { qa -= nA; ++qi; }
            const int dl = D[k] - D[j];
            if (0 < dl && dl < m) {
              const unsigned d = (unsigned)abs(2 * dl - m);
              const unsigned key = ((unsigned)k << 10) | (unsigned)j;
              if (d < bd2 || (d == bd2 && key < bkey)) { bd2 = d; bkey = key; }
            }
          }
          const unsigned d2 = __reduce_min_sync(FULL, bd2);
          if (d2 != UINT_MAX) {
            const unsigned key = __reduce_min_sync(FULL, bd2 == d2 ? bkey : UINT_MAX);
            tk0 = (int)(key >> 10);
            tk1 = (int)(key & 1023);
            delta = D[tk0] - D[tk1];
            nt = 2;
            ++swaps;
          }
        }
        // move: K from I to A; swap: remove K from I and J from A, then insert K into A and J
        // into I (the oracle's order: insertion points do not see the other swapped task)
        for (int x = 0; x < nt; ++x)
          list_remove<NC>(nlist + (x == 0 ? I : A) * n, &ncnt[x == 0 ? I : A], x == 0 ? tk0 : tk1, lane);
        for (int x = 0; x < nt; ++x)
          list_insert<NC>(nlist + (x == 0 ? A : I) * n, &ncnt[x == 0 ? A : I], x == 0 ? tk0 : tk1, D, lane);
        if (nt) {
          add_on(wI, -delta);
          add_on(ninfo[A], delta);
          done = true;
        }
      }
      if (!done) {
        const int par = nd_par(wI);
        if (par != ROOTP && !((opened >> par) & 1)) {
          opened |= 1u << par;
          Q |= (unsigned long long)par << (4 * qt++);
        }
      }
    }
    omega = __reduce_max_sync(FULL, lane < S ? send[lane] : 0);
    if (ppm > 0 && (long long)(omega_prev - omega) * 1000000LL < (long long)ppm * omega_prev) break;
  }
}

// ---------------------------------------------------------------------------
// Phase-3 variant FAR_BEST_IMPROVEMENT (R30; the north star's literal "evaluates
// every task move and swap, recomputes the makespan and takes an argmin"): each iteration
// scores EVERY move of a task to another node of the same size and EVERY swap of two tasks
// on different same-size nodes by (w', c') = (max slice end after the operation, #slices at
// w') under Alg. 2's time model (slice ends +-t), and applies the argmin of
// (w', c', kind, first, second) if it lowers (w, c).  Same-size nodes form contiguous id
// ranges in both trees (A30: {1,2}, {3..6}; A100: {3,4,5}, {6..12}).  Candidates are spread
// over the lanes: moves as a flat (list entry, alternative) index, swaps as (entry, lanes
// over the entries of later nodes of the class); one 64-bit packed key per lane, REDUX
// min.  evals = candidates scored (closed form per class: m(|V|-1) + (m^2 - sum cnt^2)/2).
// ---------------------------------------------------------------------------
template <int NC>
__device__ __noinline__ void refine_best_warp(int n, const int* D, uint16_t* nlist, int* ncnt, int* send,
                                              const uint32_t* ninfo, int max_it, int ppm, int lane, int& moves,
                                              int& swaps, int& iters, long long& evals, uint16_t* flat) {
  constexpr int S = Tree<NC>::S, NN = Tree<NC>::NN;
  // per-warp tables of one class, rebuilt every iteration: (max, count) of the slice ends of each
  // node and of the slices outside each node pair (the score of a transfer between two disjoint
  // nodes a -> b of d ticks is max(out(a,b), M_a - d, M_b + d) with the counts of those reaching it)
  __shared__ int2 s_pair[4][64];
  __shared__ int2 s_node[4][8];
  int2* pairt = s_pair[(threadIdx.x >> 5) & 3];
  int2* nodet = s_node[(threadIdx.x >> 5) & 3];
  // classes of >= 2 same-size nodes: contiguous id runs [cf, cl)
  int cf[2] = {0, 0}, cl[2] = {0, 0}, ncls = 0;
  for (int v = 1; v <= NN; ++v) {
    const bool brk = v == NN || nd_sz(ninfo[v]) != nd_sz(ninfo[v - 1]);
    if (brk) {
      int f = v - 1;
      while (f > 0 && nd_sz(ninfo[f - 1]) == nd_sz(ninfo[v - 1])) --f;
      if (v - f >= 2 && ncls < 2) { cf[ncls] = f; cl[ncls] = v; ++ncls; }
    }
  }
  auto mask_of = [&](int v) {
    const uint32_t w = ninfo[v];
    return ((1u << nd_sz(w)) - 1u) << nd_lo(w);
  };
  auto score = [&](int ia, int ib, int d) {  // class-local node indices a (loses d), b (gains d)
    const int2 o = pairt[ia * 8 + ib], na = nodet[ia], nb = nodet[ib];
    const int x = na.x - d, y = nb.x + d;
    const int w = max(o.x, max(x, y));
    const int c = (o.x == w ? o.y : 0) + (x == w ? na.y : 0) + (y == w ? nb.y : 0);
    return ((unsigned long long)(unsigned)w << 24) | ((unsigned long long)c << 21);
  };
  moves = swaps = iters = 0;
  evals = 0;
  while (iters < max_it) {
    ++iters;
    int e[S];
#pragma unroll
    for (int s = 0; s < S; ++s) e[s] = send[s];
    unsigned long long cur;
    {
      int w = -1, c = 0;
#pragma unroll
      for (int s = 0; s < S; ++s) {
        if (e[s] > w) { w = e[s]; c = 1; } else if (e[s] == w) { ++c; }
      }
      cur = ((unsigned long long)(unsigned)w << 24) | ((unsigned long long)c << 21);
    }
    const int omega_prev = (int)(cur >> 24);
    unsigned long long best = ~0ull;
    for (int g = 0; g < ncls; ++g) {
      const int f = cf[g], V = cl[g] - f, A = V - 1;
      // tables of this class
      __syncwarp();
      for (int p = lane; p < V * 8; p += 32) {
        const int ia = p >> 3, ib = p & 7;
        if (ib < V) {
          const unsigned mx = mask_of(f + ia) | (ia != ib ? mask_of(f + ib) : 0u);
          int w = -1, c = 0;
#pragma unroll
          for (int s = 0; s < S; ++s) {
            if ((mx >> s) & 1u) continue;
            if (e[s] > w) { w = e[s]; c = 1; } else if (e[s] == w) { ++c; }
          }
          pairt[p] = make_int2(w, c);
        }
      }
      if (lane < V) {
        const unsigned mv = mask_of(f + lane);
        int w = -1, c = 0;
#pragma unroll
        for (int s = 0; s < S; ++s) {
          if (!((mv >> s) & 1u)) continue;
          if (e[s] > w) { w = e[s]; c = 1; } else if (e[s] == w) { ++c; }
        }
        nodet[lane] = make_int2(w, c);
      }
      // flat entries of the class: task | local node index << 10, in node order
      int m = 0, sq = 0;
      for (int v = f; v < f + V; ++v) {
        const int cv = ncnt[v];
        for (int q = lane; q < cv; q += 32) flat[m + q] = (uint16_t)(nlist[v * n + q] | ((v - f) << 10));
        m += cv;
        sq += cv * cv;
      }
      __syncwarp();
      evals += (long long)m * A + (long long)(m * m - sq) / 2;
      // moves: flat p = idx * A + r, r-th other node of the class
      {
        int idx = lane / A, r = lane - (lane / A) * A;
        const int di = 32 / A, dr = 32 - di * A;
        for (int p = lane; p < m * A; p += 32) {
          const int x = flat[idx], T = x & 1023, ia = x >> 10;
          const int ib = r + (r >= ia ? 1 : 0);
          const unsigned long long k = score(ia, ib, D[T]) | ((unsigned long long)T << 10) | (unsigned)(f + ib);
          best = k < best ? k : best;
          idx += di;
          r += dr;
          if (r >= A) { r -= A; ++idx; }
        }
      }
      // swaps: every pair of class nodes (a < b), lanes over the |a| x |b| task pairs (flat index
      // stepped incrementally: no division in the loop)
      int abase = 0;
      for (int ia = 0; ia < V; ++ia) {
        const int na = ncnt[f + ia];
        int bbase = abase + na;
        for (int ib = ia + 1; ib < V; ++ib) {
          const int nb = ncnt[f + ib], tot = na * nb;
          if (tot > 0) {
            const int di = 32 / nb, da = 32 - di * nb;
            int qi = lane / nb, qa = lane - (lane / nb) * nb;
            for (int p = lane; p < tot; p += 32) {
              const int tx = flat[abase + qi] & 1023, ty = flat[bbase + qa] & 1023;
              const bool lo = tx < ty;
              const int k = lo ? tx : ty, j = lo ? ty : tx;
              const int dd = D[k] - D[j];
              const unsigned long long key = score(lo ? ia : ib, lo ? ib : ia, dd) | (1ull << 20) |
                                             ((unsigned long long)k << 10) | (unsigned)j;
              best = key < best ? key : best;
              qi += di;
              qa += da;
              if (qa >= nb) { qa -= nb; ++qi; }
            }
          }
          bbase += nb;
        }
        abase += na;
      }
    }
    // warp argmin of the packed keys
    const unsigned hi = __reduce_min_sync(FULL, (unsigned)(best >> 32));
    const unsigned lo = __reduce_min_sync(FULL, (unsigned)(best >> 32) == hi ? (unsigned)best : ~0u);
    best = ((unsigned long long)hi << 32) | lo;
    if ((best >> 21) >= (cur >> 21)) break;  // no candidate lowers (w, c)
    const int x = (int)((best >> 10) & 1023), y = (int)(best & 1023);
    int from, to, tk0, tk1 = -1, d;
    if (!((best >> 20) & 1)) {  // move x to node y
      tk0 = x;
      to = y;
      from = -1;
      for (int v = 0; v < NN; ++v)
        for (int q = lane; q < ncnt[v]; q += 32)
          if (nlist[v * n + q] == x) from = v;
      from = __reduce_max_sync(FULL, from);
      d = D[x];
      ++moves;
    } else {  // swap x (its node) with y (its node)
      int vx = -1, vy = -1;
      for (int v = 0; v < NN; ++v)
        for (int q = lane; q < ncnt[v]; q += 32) {
          const int t = nlist[v * n + q];
          if (t == x) vx = v;
          if (t == y) vy = v;
        }
      from = __reduce_max_sync(FULL, vx);
      to = __reduce_max_sync(FULL, vy);
      tk0 = x;
      tk1 = y;
      d = D[x] - D[y];
      ++swaps;
    }
    // the oracle's order: remove both, then insert each into the other node's list
    list_remove<NC>(nlist + from * n, &ncnt[from], tk0, lane);
    if (tk1 >= 0) list_remove<NC>(nlist + to * n, &ncnt[to], tk1, lane);
    list_insert<NC>(nlist + to * n, &ncnt[to], tk0, D, lane);
    if (tk1 >= 0) list_insert<NC>(nlist + from * n, &ncnt[from], tk1, D, lane);
    const unsigned mf = mask_of(from), mt = mask_of(to);
    if (lane < S) send[lane] += (((mt >> lane) & 1u) ? d : 0) - (((mf >> lane) & 1u) ? d : 0);
    __syncwarp();
    int om = __reduce_max_sync(FULL, lane < S ? send[lane] : 0);
    if (ppm > 0 && (long long)(omega_prev - om) * 1000000LL < (long long)ppm * omega_prev) break;
  }
}

// Build per-node ordered lists of member k from the per-size LPT lists: sizes in
// decreasing order so the A100 {S0..S3} node lists its size-4 tasks before its size-3
// tasks.  Lanes over list entries; __match_any_sync ranks entries per node.
template <int NC>
__device__ void build_node_lists(int n, int k, const int2* lent, const uint16_t* ltask, const int* loff,
                                 const uint8_t* node_of, uint16_t* nlist, int* ncnt, uint8_t* su, int lane) {
  constexpr int NN = Tree<NC>::NN;
  if (lane < NN) ncnt[lane] = 0;
  __syncwarp();
  for (int c = NC - 1; c >= 0; --c) {
    const int pe = loff[c + 1];
    for (int p0 = loff[c]; p0 < pe; p0 += 32) {
      const int p = p0 + lane;
      int v = -1, j = 0;
      if (p < pe) {
        const int y = lent[p].y;
        const int lo = y & 0xFFFF, hi = (int)((unsigned)y >> 16);
        if (lo <= k && k < hi) {
          j = ltask[p];
          v = node_of[j];
          su[j] = (uint8_t)c;
        }
      }
      const unsigned grp = __match_any_sync(FULL, v);
      const int rank = __popc(grp & ((1u << lane) - 1));
      const int base = v >= 0 ? ncnt[v] : 0;
      __syncwarp();
      if (v >= 0) {
        nlist[v * n + base + rank] = (uint16_t)j;
        if (rank == __popc(grp) - 1) ncnt[v] = base + __popc(grp);
      }
      __syncwarp();
    }
  }
}

// Phase 3 + replay + guard on an input schedule (far_local_search, MODE_LOCAL).
template <int NC>
__device__ __noinline__ void solve_local(const KParams& P, int64_t inst, unsigned char* wsm, const Layout& L,
                                         const uint32_t* ninfo, const int* cr, const int* de, int lane,
                                         far_result R, bool want_sched, bool refine) {
  constexpr int S = Tree<NC>::S, NN = Tree<NC>::NN;
  const int n = P.n;
  int32_t* T = (int32_t*)(wsm + L.times);
  uint8_t* cur = wsm + L.cur;
  uint8_t* su = wsm + L.su;
  uint8_t* bestnode = wsm + L.bestnode;
  unsigned char* scratch = wsm + L.scratch;
  int* start = (int*)(wsm + L.start);
  int* misc = (int*)(wsm + L.misc);
  int* ncnt = misc + M_NCNT;
  int* nsum = misc + M_NSUM;
  int* send = misc + M_SEND;
  int* life = misc + M_LIFE;
  int ms2 = 0;

    // ---- rebuild the tree from an input schedule: node lists ordered by (start, task)
    const far_task_slot* in = P.sched_in + inst * (int64_t)n;
    int bad = 0, msIn = 0;
    for (int j = lane; j < n; j += 32) {
      const far_task_slot s = in[j];
      int c = -1;
      if (s.node < NN) {
        const uint32_t w = ninfo[s.node];
        if (size_of<NC>(nd_c0(w)) == s.size_used) c = nd_c0(w);
        else if (nd_c1(w) != NONE && size_of<NC>(nd_c1(w)) == s.size_used) c = nd_c1(w);
      }
      if (c < 0 || s.start < 0 || s.start > BOUND) { bad = 1; c = 0; }
      cur[j] = s.node < NN ? s.node : 0;
      su[j] = (uint8_t)c;
      start[j] = s.start;
      msIn = max(msIn, s.start + T[j * NC + c]);
    }
    bad = __any_sync(FULL, bad);
    msIn = __reduce_max_sync(FULL, msIn);
    if (bad) {
      if (lane == 0) {
        R.makespan = -1;
        R.status = FAR_E_INVALID_ARG;
        P.makespan[inst] = -1;
        if (P.res) P.res[inst] = R;
        atomicOr(P.errflag, 2);
      }
      return;
    }
    __syncwarp();
    uint16_t* nlist = (uint16_t*)scratch;
    for (int j = lane; j < n; j += 32) {
      const int v = cur[j], sj = start[j];
      int pos = 0;
      for (int q = 0; q < n; ++q)
        pos += (cur[q] == v) && (start[q] < sj || (start[q] == sj && q < j));
      nlist[v * n + pos] = (uint16_t)j;
    }
    for (int v = 0; v < NN; ++v) {
      int c = 0;
      for (int j = lane; j < n; j += 32) c += (cur[j] == v);
      c = __reduce_add_sync(FULL, c);
      if (lane == 0) ncnt[v] = c;
    }
    for (int s = 0; s < S; ++s) {
      int e = 0;
      for (int j = lane; j < n; j += 32) {
        const uint32_t w = ninfo[cur[j]];
        if (s >= nd_lo(w) && s < nd_lo(w) + nd_sz(w)) e = max(e, start[j] + T[j * NC + su[j]]);
      }
      e = __reduce_max_sync(FULL, e);
      if (lane == 0) send[s] = e;
    }
    __syncwarp();
    const far_result rin = P.res_in ? P.res_in[inst] : R;
    R.alloc_index = rin.alloc_index;
    R.family_size = rin.family_size;
    R.events = rin.events;
    ms2 = (P.res_in && rin.makespan_phase2 > 0) ? rin.makespan_phase2 : msIn;
    R.makespan_phase2 = ms2;
    int msF = msIn;
    bool use_input = true;
    if (refine && n > 0) {
      int mv, sw, it;
      long long ev;
      int* D = (int*)(scratch + ((2 * NN * n + 3) & ~3));  // durations at the tasks' sizes
      for (int j = lane; j < n; j += 32) D[j] = T[j * NC + su[j]];
      __syncwarp();
      if (P.flags & FAR_BEST_IMPROVEMENT)
        refine_best_warp<NC>(n, D, nlist, ncnt, send, ninfo, P.max_it, P.ppm, lane, mv, sw, it, ev,
                             (uint16_t*)start);
      else
        refine_warp<NC>(n, D, nlist, ncnt, send, ninfo, P.max_it, P.ppm, (P.flags & FAR_NONEMPTY_ALT) != 0, lane, mv,
                        sw, it, ev);
      R.moves = mv; R.swaps = sw; R.iterations = it; R.evals = ev;
      __syncwarp();  // refine_best_warp's scratch is start[], which the replay writes
      const int msR = (P.flags & FAR_SWITCH_COST)
                          ? replay_tasks_warp<NC>(n, D, nlist, ncnt, su, nsum, start, bestnode, ninfo, cr, de, lane)
                          : replay_warp<NC>(n, D, nlist, ncnt, nsum, life, start, bestnode, ninfo, cr, de, lane);
      if (!(P.flags & FAR_NO_GUARD) && msR > ms2) {
        R.reverted = 1;
      } else {
        use_input = false;
        msF = msR;
      }
    }
    R.makespan = msF;
    if (want_sched) {
      far_task_slot* out = P.sched + inst * (int64_t)n;
      for (int j = lane; j < n; j += 32) {
        if (use_input) {
          out[j] = in[j];
        } else {
          far_task_slot s;
          s.node = bestnode[j];
          s.size_used = (uint8_t)size_of<NC>(su[j]);
          s.pad[0] = s.pad[1] = 0;
          s.start = start[j];
          out[j] = s;
        }
      }
    }
    if (lane == 0) {
      P.makespan[inst] = R.makespan;
      if (P.res) P.res[inst] = R;
    }
    return;
  }

// Node lists of k* from the pipelined phase-2 record (node, size index, position per task).
template <int NC>
__device__ void lists_from_record(int n, const uint32_t* rec, const int32_t* t, uint16_t* nlist, int* ncnt,
                                  uint8_t* su, int* D, int lane, const uint32_t* d0) {
  constexpr int NN = Tree<NC>::NN;
  if (lane < NN) ncnt[lane] = 0;
  __syncwarp();
  for (int j = lane; j < n; j += 32) {
    const uint32_t r = __ldcs(rec + j);
    const int v = (int)(r & 15u);
    nlist[v * n + (int)(r >> 7)] = (uint16_t)j;
    su[j] = (uint8_t)((r >> 4) & 7u);
    // k* = 0: member 0's durations written by prep (coalesced); else gather the runtime table
    D[j] = d0 ? (int)__ldcs(d0 + j) : __ldg(t + j * NC + su[j]);
    atomicAdd(&ncnt[v], 1);
  }
  __syncwarp();
}

// H6/H7 of one instance (warp): node lists of k*, phase 3, replay, keep-best guard, stores.
// FROM_REC: k*'s lists come from the pipelined phase-2 record (far_pipeline.cuh) and the
// durations from the global runtime table; else from the fused kernel's H3 lists in smem.
template <int NC, bool FROM_REC>
__device__ void finish_core(const KParams& P, int64_t inst, uint16_t* nlist, int* D, int* start, uint8_t* onode,
                            uint8_t* su, int* misc, const int32_t* T, const int2* lent, const uint16_t* ltask,
                            const uint8_t* bestnode, const uint32_t* ninfo, const int* cr, const int* de, int lane,
                            far_result R, int ms2, int bestk, bool want_sched, bool refine) {
  constexpr int S = Tree<NC>::S;
  const int n = P.n;
  int* loff = misc + M_LOFF;
  int* ncnt = misc + M_NCNT;
  int* nsum = misc + M_NSUM;
  int* send = misc + M_SEND;
  int* bsend = misc + M_BSEND;
  int* life = misc + M_LIFE;
  // One call site per helper (pass 1 only runs when the guard reverts to the phase-2 tree)
  // keeps the code small enough for the instruction cache.
  int msF = ms2;
  const bool need_replay = refine || want_sched;
  for (int pass = 0; pass < 2; ++pass) {
    if (FROM_REC) {
      lists_from_record<NC>(n, P.ws_rec + inst * (int64_t)n, P.times + inst * (int64_t)n * NC, nlist, ncnt, su, D,
                            lane, bestk == 0 ? P.ws_d0 + inst * (int64_t)P.ws_n4 : nullptr);
    } else {
      build_node_lists<NC>(n, bestk, lent, ltask, loff, bestnode, nlist, ncnt, su, lane);
      for (int j = lane; j < n; j += 32) D[j] = T[j * NC + su[j]];
    }
    __syncwarp();
    const bool ref = refine && pass == 0;
    if (ref) {
      if (lane < S) send[lane] = bsend[lane];
      __syncwarp();
      int mv, sw, it;
      long long ev;
      if (P.flags & FAR_BEST_IMPROVEMENT)
        refine_best_warp<NC>(n, D, nlist, ncnt, send, ninfo, P.max_it, P.ppm, lane, mv, sw, it, ev,
                             (uint16_t*)start);
      else
        refine_warp<NC>(n, D, nlist, ncnt, send, ninfo, P.max_it, P.ppm, (P.flags & FAR_NONEMPTY_ALT) != 0, lane, mv,
                        sw, it, ev);
      R.moves = mv; R.swaps = sw; R.iterations = it; R.evals = ev;
      __syncwarp();  // refine_best_warp's scratch is start[], which the replay writes
    }
    if (!need_replay) break;
    const int msR = (P.flags & FAR_SWITCH_COST)
                        ? replay_tasks_warp<NC>(n, D, nlist, ncnt, su, nsum, start, onode, ninfo, cr, de, lane)
                        : replay_warp<NC>(n, D, nlist, ncnt, nsum, life, start, onode, ninfo, cr, de, lane);
    if (ref && !(P.flags & FAR_NO_GUARD) && msR > ms2) {
      R.reverted = 1;  // keep-best guard: return the phase-2 schedule (replayed in pass 1)
      if (!want_sched) break;
      continue;
    }
    if (ref) msF = msR;
    break;
  }
  R.makespan = msF;
  if (want_sched) {
    far_task_slot* out = P.sched + inst * (int64_t)n;
    for (int j = lane; j < n; j += 32) {
      far_task_slot s;
      s.node = onode[j];
      s.size_used = (uint8_t)size_of<NC>(su[j]);
      s.pad[0] = s.pad[1] = 0;
      s.start = start[j];
      out[j] = s;
    }
  }
  if (lane == 0) {
    P.makespan[inst] = R.makespan;
    if (P.res) P.res[inst] = R;
  }
  __syncwarp();
}

template <int NC>
__device__ __forceinline__ void finish_instance(const KParams& P, int64_t inst, unsigned char* wsm, const Layout& L,
                                                const uint32_t* ninfo, const int* cr, const int* de, int lane,
                                                far_result R, int ms2, int bestk, bool want_sched, bool refine) {
  constexpr int NN = Tree<NC>::NN;
  unsigned char* scratch = wsm + L.scratch;
  finish_core<NC, false>(P, inst, (uint16_t*)scratch, (int*)(scratch + ((2 * NN * P.n + 3) & ~3)),
                         (int*)(wsm + L.start), wsm + L.cur, wsm + L.su, (int*)(wsm + L.misc),
                         (const int32_t*)(wsm + L.times), (const int2*)(wsm + L.lent),
                         (const uint16_t*)(wsm + L.ltask), wsm + L.bestnode, ninfo, cr, de, lane, R, ms2, bestk,
                         want_sched, refine);
}

// ---------------------------------------------------------------------------
// One instance, one warp.
// ---------------------------------------------------------------------------
template <int NC, int PIPE>
__device__ void solve_instance(const KParams& P, int64_t inst, unsigned char* wsm, const Layout& L,
                               const uint32_t* ninfo, const int* cr, const int* de, int lane) {
  constexpr int S = Tree<NC>::S, NN = Tree<NC>::NN;
  const int n = P.n;
  int32_t* T = (int32_t*)(wsm + L.times);
  int2* lent = (int2*)(wsm + L.lent);
  uint16_t* ltask = (uint16_t*)(wsm + L.ltask);
  unsigned long long* cnts = (unsigned long long*)(wsm + L.cnts);
  // lower bound of each member's Alg. 1 makespan: its longest task h_k (lbh) and its area
  // spread over all slices, ceil(W_k / #slices) (lbs) -- reconfiguration only adds idle time
  int* lbs = (int*)(wsm + L.lbs);
  int* lbh = (int*)(wsm + L.lbh);
  uint8_t* cur = wsm + L.cur;
  uint8_t* su = wsm + L.su;
  uint8_t* bestnode = wsm + L.bestnode;
  unsigned char* scratch = wsm + L.scratch;
  uint32_t* lstate = (uint32_t*)(wsm + L.lstate);
  int* start = (int*)(wsm + L.start);
  int* misc = (int*)(wsm + L.misc);
  int* loff = misc + M_LOFF;
  int* bsend = misc + M_BSEND;

  // ---- H0: stage the runtime table (contiguous n*NC int32) into shared memory
  const int cntT = n * NC;
  const int32_t* src = P.times + inst * (int64_t)cntT;
  if ((((uintptr_t)src) & 15) == 0) {
    const int n4 = cntT >> 2;
    const int4* s4 = (const int4*)src;
    int4* d4 = (int4*)T;
    for (int q = lane; q < n4; q += 32) d4[q] = __ldcs(s4 + q);
    for (int q = (n4 << 2) + lane; q < cntT; q += 32) T[q] = __ldcs(src + q);
  } else {
    for (int q = lane; q < cntT; q += 32) T[q] = __ldcs(src + q);
  }
  __syncwarp();

  far_result R;
  R.makespan = 0; R.makespan_phase2 = 0; R.alloc_index = 0; R.family_size = 0;
  R.moves = 0; R.swaps = 0; R.iterations = 0; R.reverted = 0; R.status = FAR_OK; R.reserved = 0;
  R.evals = 0; R.events = 0;
  const bool want_sched = P.sched != nullptr && !(P.flags & FAR_NO_SCHEDULE);
  const bool refine = !(P.flags & FAR_NO_REFINE);

  // ---- input checks (include/far.h "Integer range")
  int tmax = 0;
  {
    int bad = 0;
    long long bsum = 0;
    for (int j = lane; j < n; j += 32) {
      int mx = 0;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int t = T[j * NC + c];
        bad |= (t < 1);
        mx = max(mx, t);
      }
      bsum += mx;
      tmax = max(tmax, mx);
    }
    bad = __any_sync(FULL, bad);
    bsum = warp_sum_ll(bsum);
    tmax = __reduce_max_sync(FULL, tmax);
    if (bad || bsum + P.rsum >= BOUND) {
      if (lane == 0) {
        R.makespan = -1;
        R.status = FAR_E_BAD_TIME;
        P.makespan[inst] = -1;
        if (P.res) P.res[inst] = R;
        atomicOr(P.errflag, 1);
        if (PIPE == PIPE_PREP) P.ws_meta[inst * 16 + WS_FLAG] = 1;
      }
      return;
    }
  }

  if (PIPE == PIPE_NONE && P.mode == MODE_LOCAL) {
    solve_local<NC>(P, inst, wsm, L, ninfo, cr, de, lane, R, want_sched, refine);
    return;
  }
  int ms2 = 0, bestk = 0;
  if (n == 0) {
    if (lane == 0) {
      P.makespan[inst] = 0;
      if (P.res) P.res[inst] = R;
      if (PIPE == PIPE_PREP) P.ws_meta[inst * 16 + WS_FLAG] = 1;
    }
    return;
  }
  // ---- H1: first allocation a^1_i = argmin_s s*t_i(s), ties -> smallest s
  // [n][NC] member interval lo | hi << IB (lo = IM: absent; hi = IM: open).  PIPE_PREP holds
  // families of <= 64 members, so 8-bit bounds (half the shared memory) suffice there.
  using IV = typename std::conditional<PIPE == PIPE_PREP, uint16_t, uint32_t>::type;
  constexpr int IB = PIPE == PIPE_PREP ? 8 : 16;
  constexpr uint32_t IM = (1u << IB) - 1u;
  IV* ivl = (IV*)scratch;
  unsigned long long c0pack = 0;
  // total area sum_i a_i t_i(a_i) of the current member (uniform); < 7 * 2^29 by the range check
  unsigned W = 0;
  bool mono = true;
  unsigned tstar = 0;
  {
    int cnt_c[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) cnt_c[c] = 0;
    // (the checks above bound every t below 2^29, so size * t < 7 * 2^29 fits 32 bits unsigned)
    for (int j = lane; j < n; j += 32) {
      unsigned tv[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) tv[c] = (unsigned)T[j * NC + c];
      int best = 0;
      unsigned bw = (unsigned)size_of<NC>(0) * tv[0];
#pragma unroll
      for (int c = 1; c < NC; ++c) {
        const unsigned w = (unsigned)size_of<NC>(c) * tv[c];
        if (w < bw) { bw = w; best = c; }
      }
      cur[j] = (uint8_t)best;
      W += bw;
      // next size for phase-1 growth: nx(c) = argmin_{c' > c} (size(c') t(c'), c')
      {
        unsigned packed = 0;
        int above = NC - 1;
        unsigned wa = (unsigned)size_of<NC>(NC - 1) * tv[NC - 1];
#pragma unroll
        for (int c = NC - 2; c >= 0; --c) {
          packed |= (unsigned)above << (3 * c);
          const unsigned wc = (unsigned)size_of<NC>(c) * tv[c];
          if (wc <= wa) { wa = wc; above = c; }
        }
        su[j] = (uint8_t)(packed & 0xFF);
        bestnode[j] = (uint8_t)(packed >> 8);
        // growth chain a^1 -> nx -> ... -> max size (strictly increasing sizes, so one ascending
        // scan): monotone (non-increasing t) chains allow the parallel phase-1 below
        int nextc = best;
        unsigned tprev = 0xFFFFFFFFu;
#pragma unroll
        for (int c = 0; c < NC; ++c)
          if (c == nextc) {
            mono = mono && tv[c] <= tprev;
            tprev = tv[c];
            nextc = c == NC - 1 ? NC : (int)((packed >> (3 * c)) & 7u);
          }
        tstar = max(tstar, (tv[NC - 1] << 10) | (unsigned)(1023 - j));
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        cnt_c[c] += (c == best);
        ivl[j * NC + c] = (IV)((c == best) ? (IM << IB) : ((IM << IB) | IM));
      }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) c0pack |= (unsigned long long)__reduce_add_sync(FULL, cnt_c[c]) << (11 * c);
    W = __reduce_add_sync(FULL, W);
  }
  if (lane == 0) cnts[0] = c0pack;
  __syncwarp();

  // ---- H2: a^{k+1}: grow the longest task (ties -> lowest index) to
  //          argmin_{s > a_j} s*t_j(s) (ties -> smallest s); stop when it is at max size
  const bool small = tmax < (1 << 22);
  if (PIPE == PIPE_PREP && (!small || n > 1023)) {  // entries pack t < 2^22 and task < 1023
    if (lane == 0) {
      atomicOr(P.ovf + (inst >> 5), 1u << (inst & 31));
      atomicAdd(P.ovf_count, 1ull);
      P.ws_meta[inst * 16 + WS_FLAG] = 1;
    }
    return;
  }
  int K = 1;
  // list entries per size (11-bit fields): member 0's sizes + one entry per growth step at the
  // size it enters (a task enters each size at most once, so a field stays <= n)
  unsigned long long entp = c0pack;
  // Parallel form for monotone chains (every task's t non-increasing along its growth chain;
  // property 1 of P:260-263 implies it).  With key(t, j) = t << 10 | (1023 - j) the growth
  // process is the merge of the per-task chains by (key desc, chain position asc): each step
  // takes the largest current key, and a chain's later keys are never larger.  It stops at
  // the first terminal element (max size) on top, i.e. at T* = the largest terminal key, so
  // the growth steps are exactly the non-terminal chain elements with key >= T*, in that order.
  // (growth-step ranks live in lstate: PIPE_PREP sizes it by kcap, the fused layout holds 160)
  mono = __all_sync(FULL, mono && small && (PIPE == PIPE_PREP || P.kcap <= 160) && !(P.flags & FAR_GROW_TIES));
  tstar = __reduce_max_sync(FULL, tstar);
  if (mono) {
    int2* G = lent;  // temporary (filled in H3): {key, task | from << 10 | to << 13 | pos << 16}
    int* rnk = (int*)lstate;  // step rank per element (lstate is free until H4)
    int cntl = 0;
    for (int j = lane; j < n; j += 32) {
      const unsigned nxp = (unsigned)su[j] | ((unsigned)bestnode[j] << 8);
      for (int c = cur[j]; c != NC - 1; c = (int)((nxp >> (3 * c)) & 7u)) {
        if ((((unsigned)T[j * NC + c] << 10) | (unsigned)(1023 - j)) < tstar) break;
        ++cntl;
      }
    }
    int excl = cntl;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, excl, o);
      if (lane >= o) excl += y;
    }
    const int Gn = __shfl_sync(FULL, excl, 31);
    excl -= cntl;
    if (Gn + 1 > P.kcap) {  // family larger than this layout holds: defer to the overflow pass
      if (lane == 0) {
        atomicOr(P.ovf + (inst >> 5), 1u << (inst & 31));
        atomicAdd(P.ovf_count, 1ull);
        if (PIPE == PIPE_PREP) P.ws_meta[inst * 16 + WS_FLAG] = 1;
      }
      return;
    }
    unsigned long long myent = 0;
    for (int j = lane; j < n; j += 32) {
      const unsigned nxp = (unsigned)su[j] | ((unsigned)bestnode[j] << 8);
      int pos = 0;
      for (int c = cur[j]; c != NC - 1; ++pos) {
        const unsigned key = ((unsigned)T[j * NC + c] << 10) | (unsigned)(1023 - j);
        if (key < tstar) break;
        const int c2 = (int)((nxp >> (3 * c)) & 7u);
        G[excl++] = make_int2((int)key, j | (c << 10) | (c2 << 13) | (pos << 16));
        myent += 1ull << (11 * c2);
        c = c2;
      }
    }
    entp += (unsigned long long)warp_sum_ll((long long)myent);
    __syncwarp();
    // rank of each step: larger keys first; equal keys (same task) in chain order
    // (64-bit compare of (key, 63 - pos): count the elements <= own, rank = Gn - that)
    for (int e = lane; e < Gn; e += 32) {
      const unsigned ke = (unsigned)G[e].x;
      const int pe = G[e].y >> 16;
      int ge = 0;
      for (int f = 0; f < Gn; ++f) {
        const int2 g = G[f];
        count_ge64(ge, 63u - (unsigned)pe, ke, 63u - ((unsigned)g.y >> 16), (unsigned)g.x);
      }
      const int rk = Gn - ge;
      // step rk produces member rk + 1: longest task of member rk, deltas of member rk + 1
      const int j = G[e].y & 1023, cf = (G[e].y >> 10) & 7, ct = (G[e].y >> 13) & 7;
      lbh[rk] = (int)(ke >> 10);
      cnts[rk + 1] = (1ull << (11 * ct)) - (1ull << (11 * cf));
      // area delta (>= 0: work is non-decreasing along a growth chain, nx(c) minimises over c' > c)
      lbs[rk + 1] = (int)((unsigned)size_of<NC>(ct) * (unsigned)T[j * NC + ct] -
                          (unsigned)size_of<NC>(cf) * (unsigned)T[j * NC + cf]);
      rnk[e] = rk;
    }
    __syncwarp();
    // member intervals: entering size ct at member rk + 1, leaving it at the task's next step
    for (int e = lane; e < Gn; e += 32) {
      const int y = G[e].y, j = y & 1023, cf = (y >> 10) & 7, ct = (y >> 13) & 7, pos = y >> 16;
      const int rk = rnk[e];
      const bool next = e + 1 < Gn && (G[e + 1].y & 1023) == j;
      ivl[j * NC + ct] = (IV)((uint32_t)(rk + 1) | ((next ? (uint32_t)(rnk[e + 1] + 1) : IM) << IB));
      if (pos == 0) ivl[j * NC + cf] = (IV)((uint32_t)(rk + 1) << IB);  // a^1 interval [0, rk + 1)
    }
    if (lane == 0) {
      lbh[Gn] = (int)(tstar >> 10);
      cnts[0] = c0pack;
      lbs[0] = (int)W;
    }
    __syncwarp();
    // prefix sums over members of the packed size counts and of the area (W_k < 2^32 unsigned)
    unsigned long long cc = 0;
    unsigned ww = 0;
    for (int k0 = 0; k0 <= Gn; k0 += 32) {
      const int k = k0 + lane;
      unsigned long long dc = k <= Gn ? cnts[k] : 0;
      unsigned dw = k <= Gn ? (unsigned)lbs[k] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long yc = __shfl_up_sync(FULL, dc, o);
        const unsigned yw = __shfl_up_sync(FULL, dw, o);
        if (lane >= o) { dc += yc; dw += yw; }
      }
      if (k <= Gn) {
        cnts[k] = cc + dc;
        lbs[k] = (int)((ww + dw + (unsigned)(S - 1)) / (unsigned)S);  // ceil(W_k / #slices)
      }
      cc += __shfl_sync(FULL, dc, 31);
      ww += __shfl_sync(FULL, dw, 31);
    }
    __syncwarp();
    K = Gn + 1;
  } else {
    unsigned long long cp = c0pack;
    // packed current key per task (start[] is free until H7; PIPE_PREP has no start[] and
    // recomputes the keys)
    uint32_t* ck = (uint32_t*)start;
    unsigned lk = 0;
    if (small) {
      for (int j = lane; j < n; j += 32) {
        const unsigned key = ((unsigned)T[j * NC + cur[j]] << 10) | (unsigned)(1023 - j);
        if (PIPE != PIPE_PREP) ck[j] = key;
        lk = max(lk, key);
      }
    }
    for (;;) {
      int jj, hmax;
      if (small) {
        const unsigned gk = __reduce_max_sync(FULL, lk);
        jj = 1023 - (int)(gk & 1023u);
        hmax = (int)(gk >> 10);
      } else {
        int lm = -1, lj = INT_MAX;
        for (int j = lane; j < n; j += 32) {
          const int t = T[j * NC + cur[j]];
          if (t > lm) { lm = t; lj = j; }
        }
        hmax = __reduce_max_sync(FULL, lm);
        jj = (int)__reduce_min_sync(FULL, (unsigned)(lm == hmax ? lj : INT_MAX));
      }
      // lower bound of member K-1's Alg. 1 makespan: its longest task and its area spread
      // over all slices (reconfiguration only adds idle time) -- used to prune phase 2
      if (lane == 0) {
        lbh[K - 1] = hmax;
        lbs[K - 1] = (int)((W + (unsigned)(S - 1)) / (unsigned)S);
      }
      const int cj = cur[jj];
      if (P.flags & FAR_GROW_TIES) {
        // variant (the formula of P:349): every task tied for the longest time grows in this
        // step; the family ends when one of them is already at the largest size
        bool stuck = false;
        for (int j = lane; j < n; j += 32) stuck |= cur[j] == NC - 1 && T[j * NC + cur[j]] == hmax;
        if (__any_sync(FULL, stuck)) break;
        if (K >= P.kcap) {
          if (lane == 0) {
            atomicOr(P.ovf + (inst >> 5), 1u << (inst & 31));
            atomicAdd(P.ovf_count, 1ull);
            if (PIPE == PIPE_PREP) P.ws_meta[inst * 16 + WS_FLAG] = 1;
          }
          return;
        }
        unsigned long long dcp = 0, dent = 0;
        unsigned dW = 0;
        __syncwarp();
        for (int j = lane; j < n; j += 32) {
          const int c = cur[j];
          if (T[j * NC + c] != hmax) continue;
          const unsigned nx = (unsigned)su[j] | ((unsigned)bestnode[j] << 8);
          const int b = (int)((nx >> (3 * c)) & 7u);
          dcp += (1ull << (11 * b)) - (1ull << (11 * c));
          dent += 1ull << (11 * b);
          dW += (unsigned)size_of<NC>(b) * (unsigned)T[j * NC + b] - (unsigned)size_of<NC>(c) * (unsigned)T[j * NC + c];
          cur[j] = (uint8_t)b;
          ivl[j * NC + c] = (IV)((ivl[j * NC + c] & IM) | ((uint32_t)K << IB));
          ivl[j * NC + b] = (IV)((uint32_t)K | (IM << IB));
          if (small && PIPE != PIPE_PREP) ck[j] = ((unsigned)T[j * NC + b] << 10) | (unsigned)(1023 - j);
        }
        cp += (unsigned long long)warp_sum_ll((long long)dcp);
        entp += (unsigned long long)warp_sum_ll((long long)dent);
        W += __reduce_add_sync(FULL, dW);
        if (lane == 0) cnts[K] = cp;
        __syncwarp();
        if (small) {
          lk = 0;
          for (int j = lane; j < n; j += 32)
            lk = max(lk, PIPE == PIPE_PREP ? (((unsigned)T[j * NC + cur[j]] << 10) | (unsigned)(1023 - j)) : ck[j]);
        }
        ++K;
        continue;
      }
      if (cj == NC - 1) break;
      if (K >= P.kcap) {  // family larger than this layout holds: defer to the overflow pass
        if (lane == 0) {
          atomicOr(P.ovf + (inst >> 5), 1u << (inst & 31));
          atomicAdd(P.ovf_count, 1ull);
          if (PIPE == PIPE_PREP) P.ws_meta[inst * 16 + WS_FLAG] = 1;
        }
        return;
      }
      const unsigned nxp = (unsigned)su[jj] | ((unsigned)bestnode[jj] << 8);
      const int best = (int)((nxp >> (3 * cj)) & 7u);
      cp = cp - (1ull << (11 * cj)) + (1ull << (11 * best));
      entp += 1ull << (11 * best);
      W += (unsigned)size_of<NC>(best) * (unsigned)T[jj * NC + best] -
           (unsigned)size_of<NC>(cj) * (unsigned)T[jj * NC + cj];
      __syncwarp();
      if (lane == 0) {
        cur[jj] = (uint8_t)best;
        ivl[jj * NC + cj] = (IV)((ivl[jj * NC + cj] & IM) | ((uint32_t)K << IB));  // leaves size cj at member K
        ivl[jj * NC + best] = (IV)((uint32_t)K | (IM << IB));                     // enters size best at member K
        cnts[K] = cp;
        if (small && PIPE != PIPE_PREP) ck[jj] = ((unsigned)T[jj * NC + best] << 10) | (unsigned)(1023 - jj);
      }
      __syncwarp();
      if (small && lane == (jj & 31)) {
        lk = 0;
        for (int j = lane; j < n; j += 32)
          lk = max(lk, PIPE == PIPE_PREP ? (((unsigned)T[j * NC + cur[j]] << 10) | (unsigned)(1023 - j)) : ck[j]);
      }
      ++K;
    }
  }
  R.family_size = K;

  // ---- H3: per-size LPT lists of the (task, size) pairs used by some member, with the
  //          member interval; order (-t(s), task) (Alg. 1 lines 1-2)
  {
    int acc = 0;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      if (lane == 0) loff[c] = acc;
      acc += (int)((entp >> (11 * c)) & 2047u);
    }
    // FAR_GROW_TIES adds an entry per tied task per step, so its lists can outgrow the layout
    // (n + kcap - 1 entries) before the family does: defer to the full-layout overflow pass
    if (acc > L.ecap) {
      if (lane == 0) {
        atomicOr(P.ovf + (inst >> 5), 1u << (inst & 31));
        atomicAdd(P.ovf_count, 1ull);
        if (PIPE == PIPE_PREP) P.ws_meta[inst * 16 + WS_FLAG] = 1;
      }
      return;
    }
    if (lane == 0) loff[NC] = acc;
    __syncwarp();
    // compaction (unsorted) into the final segments
    for (int c = 0; c < NC; ++c) {
      int base = loff[c];
      for (int j0 = 0; j0 < n; j0 += 32) {
        const int j = j0 + lane;
        uint32_t iv = (IM << IB) | IM;
        if (j < n) iv = ivl[j * NC + c];
        const bool pres = (iv & IM) != IM;
        const unsigned bal = __ballot_sync(FULL, pres);
        if (pres) {
          const int pos = base + __popc(bal & ((1u << lane) - 1));
          uint32_t hi = iv >> IB;
          if (hi == IM) hi = (uint32_t)K;
          lent[pos] = make_int2(T[j * NC + c], (int)((iv & IM) | (hi << 16)));
          ltask[pos] = (uint16_t)j;
        }
        base += __popc(bal);
      }
    }
    __syncwarp();
    // sort each segment by (-t, task).  With t < 2^22 the order is the ascending order of the
    // packed key ((2^22-1-t) << 10 | task); each lane ranks its <= 4 entries against every key
    // read once by broadcast.  Otherwise (or > 128 entries) a rank sort through scratch.
    int2* sent = (int2*)scratch;
    uint16_t* stask = (uint16_t*)(scratch + 8 * L.ecap);
    for (int c = 0; c < NC; ++c) {
      const int b = loff[c], m = loff[c + 1] - loff[c];
      if (m <= 1) continue;
      if (small && m <= 128) {
        unsigned* kk = (unsigned*)scratch;  // ivl is dead
        for (int i = lane; i < m; i += 32) kk[i] = ((unsigned)(0x3FFFFF - lent[b + i].x) << 10) | ltask[b + i];
        __syncwarp();
        unsigned key[4];
        int yv[4], rk[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int i = r * 32 + lane;
          key[r] = i < m ? kk[i] : 0xFFFFFFFFu;
          yv[r] = i < m ? lent[b + i].y : 0;
          rk[r] = 0;
        }
        // rk counts the keys >= own key (itself included) with one subtract-with-carry pair
        // per comparison; the rank is then m - rk (keys are distinct)
        if (m <= 32) {
          for (int f = 0; f < m; ++f) count_ge(rk[0], kk[f], key[0]);
        } else if (m <= 64) {
          for (int f = 0; f < m; ++f) {
            const unsigned v = kk[f];
            count_ge(rk[0], v, key[0]);
            count_ge(rk[1], v, key[1]);
          }
        } else {
          for (int f = 0; f < m; ++f) {
            const unsigned v = kk[f];
#pragma unroll
            for (int r = 0; r < 4; ++r) count_ge(rk[r], v, key[r]);
          }
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) rk[r] = m - rk[r];
        __syncwarp();
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (r * 32 + lane < m) {
            lent[b + rk[r]] = make_int2(0x3FFFFF - (int)(key[r] >> 10), yv[r]);
            ltask[b + rk[r]] = (uint16_t)(key[r] & 1023u);
          }
        }
      } else {
        for (int e = lane; e < m; e += 32) {
          const int2 x = lent[b + e];
          const int tj = ltask[b + e];
          int rank = 0;
          for (int f = 0; f < m; ++f) {
            const int tf = lent[b + f].x;
            rank += (tf > x.x) || (tf == x.x && (int)ltask[b + f] < tj);
          }
          sent[b + rank] = x;
          stask[b + rank] = (uint16_t)tj;
        }
        __syncwarp();
        for (int p = b + lane; p < b + m; p += 32) {
          lent[p] = sent[p];
          ltask[p] = stask[p];
        }
      }
      __syncwarp();
    }
  }

  if (PIPE == PIPE_PREP) {  // hand the lists and the family to the lane-level phase 2
    const int E = loff[NC];
    int2* ge = P.ws_ent + inst * (int64_t)P.ws_ecap1;
    for (int e = lane; e < E; e += 32) {
      const int2 x = lent[e];
      ge[e] = make_int2((int)((unsigned)x.x | ((unsigned)ltask[e] << 22)), x.y);
    }
    if (lane == 0) ge[E] = make_int2(0, 0xFFFF);  // padding entry (never a member)
    int* gl = P.ws_lb + inst * (int64_t)P.ws_kcap;
    unsigned long long* gc = P.ws_cnt + inst * (int64_t)P.ws_kcap;
    for (int k = lane; k < K; k += 32) {
      gl[k] = max(lbh[k], lbs[k]);  // max(h_k, ceil(W_k / #slices))
      gc[k] = cnts[k];
    }
    if (K + lane < ((K + 3) & ~3)) gl[K + lane] = INT_MAX;  // row padding (16-B loads in member0)
    // member 0's entries (interval lo == 0: the a^1 sizes), compacted per size for K2
    {
      uint32_t* gm = P.ws_m0 + inst * (int64_t)P.ws_n4;
      int base = 0;
      for (int i0 = 0; i0 < E; i0 += 32) {
        const int i = i0 + lane;
        bool z = false;
        uint32_t x = 0;
        if (i < E) {
          const int2 en = lent[i];
          z = (en.y & 0xFFFF) == 0;
          x = (uint32_t)en.x | ((uint32_t)ltask[i] << 22);
        }
        const unsigned bal = __ballot_sync(FULL, z);
        if (z) {
          gm[base + __popc(bal & ((1u << lane) - 1))] = x;
          P.ws_d0[inst * (int64_t)P.ws_n4 + ltask[i]] = (uint32_t)lent[i].x;  // t_j(a1_j)
        }
        base += __popc(bal);
      }
    }
    int* meta = P.ws_meta + inst * 16;
    if (lane <= NC) meta[lane] = loff[lane];
    if (lane == 0) {
      meta[WS_K] = K;
      meta[WS_FLAG] = 0;
    }
    return;
  }

  // ---- H4: Alg. 1 for every family member, one member per lane
  uint8_t* recnode = scratch;  // [n][32]: node of task j in this lane's member
  int bestms = INT_MAX;
  long long events = 0;
  // Members are taken in increasing k, 32 per pass; a member whose lower bound LB_k
  // (H2) is >= the best makespan of the earlier passes cannot become k* = argmin
  // (makespan, k) and is skipped (exact; FAR_EXHAUSTIVE disables it).
  const bool prune = !(P.flags & FAR_EXHAUSTIVE);
  // reading variant FAR_SWITCH_COST (R7): the two-size {S0..S3} node runs an instance of
  // its task's size (isz) and is destroyed + re-created when the size changes
  const bool r7 = (P.flags & FAR_SWITCH_COST) != 0;
  int* memb = misc + M_MEMB;
  int nextk = 0;
  while (nextk < K) {
    int got = 0;
    while (got < 32 && nextk < K) {
      const int cand = nextk + lane;
      // prune iff max(h_k, ceil(W_k / S)) >= bestms
      const bool ok = cand < K && (!prune || (lbh[cand] < bestms && lbs[cand] < bestms));
      const unsigned bal = __ballot_sync(FULL, ok);
      const int pos = __popc(bal & ((1u << lane) - 1));
      const int need = 32 - got;
      if (ok && pos < need) memb[got + pos] = cand;
      const unsigned over = __ballot_sync(FULL, ok && pos == need);
      if (over) {
        nextk += __ffs(over) - 1;
        got = 32;
      } else {
        got += __popc(bal);
        nextk += 32;
      }
    }
    __syncwarp();
    if (got == 0) break;
    const int k = lane < got ? memb[lane] : -1;
    int ms = INT_MAX, pops = 0;
    int sl[S];  // slice ends of this lane's member at termination
    if (k >= 0) {
      const unsigned long long cp = cnts[k];
      int total = 0;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int r = (int)((cp >> (11 * c)) & 2047);
        lstate[c * 32 + lane] = ((uint32_t)r << 16) | (uint32_t)loff[c];  // remaining | absolute cursor
        total += r;
      }
      Frontier<S> F;
      F.init();
      int rec = 0, isz = 0;
      ms = 0;
#pragma unroll
      for (int s = 0; s < S; ++s) sl[s] = 0;
      while (total > 0) {
        int bs, be;
        F.pop(bs, be);
        const int v = F.node(bs);
        const uint32_t w = ninfo[v];
        // line 7: unscheduled tasks of a hosted size (A100 {S0..S3}: size 4 first, then 3)
        int c = nd_c0(w);
        uint32_t sv = lstate[c * 32 + lane];
        if (!(sv >> 16)) {
          c = nd_c1(w);
          sv = 0;
          if (c != NONE) sv = lstate[c * 32 + lane];
        }
        ++pops;
        if (sv >> 16) {
          if (!((F.has >> bs) & 1)) {  // lines 8-11: creation, sequenced on reconfig_end
            rec = max(rec, be) + cr[r7 ? c : nd_szi(w)];
            be = rec;
            F.has |= 1u << bs;
            if (nd_c1(w) != NONE) isz = c;  // the (one) two-size node's instance
          } else if (r7 && nd_c1(w) != NONE && c != isz) {  // variant: destroy, then re-create
            rec = max(rec, be) + de[isz];
            rec += cr[c];
            be = rec;
            isz = c;
          }
          // line 12: longest unscheduled task of size c for member k (skip other members'
          // entries; two entries per step -- the list has one padding entry)
          int p = (int)(sv & 0xFFFFu);
          int2 ent;
          for (;;) {
            const int2 e0 = lent[p], e1 = lent[p + 1];
            if ((e0.y & 0xFFFF) <= k && k < (int)((unsigned)e0.y >> 16)) { ent = e0; p += 1; break; }
            if ((e1.y & 0xFFFF) <= k && k < (int)((unsigned)e1.y >> 16)) { ent = e1; p += 2; break; }
            p += 2;
          }
          recnode[(int)ltask[p - 1] * 32 + lane] = (uint8_t)v;
          lstate[c * 32 + lane] = ((sv & 0xFFFF0000u) - 0x10000u) | (uint32_t)p;
          be += ent.x;  // lines 13-15
          ms = max(ms, be);
          --total;
          F.set(bs, be);
        } else {  // lines 17-24 (total > 0 here)
          if ((F.has >> bs) & 1) rec = max(rec, be) + de[(r7 && nd_c1(w) != NONE) ? isz : nd_szi(w)];
          if (!F.split(bs, be, w)) {  // a removed leaf keeps its slice end
#pragma unroll
            for (int s = 0; s < S; ++s) sl[s] = (s == bs) ? be : sl[s];
          }
        }
      }
      pops += __popc(F.live);  // the remaining frontier nodes are popped and dropped (heap empties)
#pragma unroll
      for (int s = 0; s < S; ++s)
        if ((F.live >> s) & 1) {
          const int sz = nd_sz(ninfo[F.node(s)]);
#pragma unroll
          for (int q = 0; q < S; ++q) sl[q] = (q >= s && q < s + sz) ? F.endv(s) : sl[q];
        }
    }
    events += warp_sum_ll(pops);
    // ---- H5: k* = argmin (makespan_k, k)
    const int m = __reduce_min_sync(FULL, ms);
    const int kw = (int)__reduce_min_sync(FULL, (unsigned)(k >= 0 && ms == m ? k : INT_MAX));
    __syncwarp();
    if (m < bestms) {
      bestms = m;
      bestk = kw;
      const int wl = __ffs(__ballot_sync(FULL, k == kw)) - 1;
      for (int j = lane; j < n; j += 32) bestnode[j] = recnode[j * 32 + wl];
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int x = __shfl_sync(FULL, sl[s], wl);
        if (lane == 0) bsend[s] = x;
      }
    }
    __syncwarp();
  }
  R.events = events;
  R.alloc_index = bestk;
  R.makespan_phase2 = bestms;
  ms2 = bestms;

  finish_instance<NC>(P, inst, wsm, L, ninfo, cr, de, lane, R, ms2, bestk, want_sched, refine);
}

__constant__ uint32_t c_nodes3[7] = {
    Tree<3>::node[0], Tree<3>::node[1], Tree<3>::node[2], Tree<3>::node[3],
    Tree<3>::node[4], Tree<3>::node[5], Tree<3>::node[6]};
__constant__ uint32_t c_nodes5[13] = {
    Tree<5>::node[0], Tree<5>::node[1], Tree<5>::node[2],  Tree<5>::node[3],  Tree<5>::node[4],
    Tree<5>::node[5], Tree<5>::node[6], Tree<5>::node[7],  Tree<5>::node[8],  Tree<5>::node[9],
    Tree<5>::node[10], Tree<5>::node[11], Tree<5>::node[12]};

template <int NC, int PIPE>
__global__ void __launch_bounds__(128, PIPE == PIPE_PREP ? 5 : 1) far_solve_kernel(KParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t ninfo[16];
  __shared__ int cr[8], de[8];
  constexpr int NN = Tree<NC>::NN;
  if (threadIdx.x < NN) ninfo[threadIdx.x] = (NC == 3) ? c_nodes3[threadIdx.x] : c_nodes5[threadIdx.x];
  if (threadIdx.x < 8) {
    cr[threadIdx.x] = P.cr[threadIdx.x];
    de[threadIdx.x] = P.de[threadIdx.x];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Layout L = make_layout(P.n, NC, Tree<NC>::S, NN, P.kcap, PIPE);
  unsigned char* wsm = smem + (size_t)warp * L.bytes;
  // per-warp copies of the node table and costs (addressed off the warp's base register)
  {
    int* misc = (int*)(wsm + L.misc);
    if (lane < 16) misc[M_NINFO + lane] = (int)ninfo[lane];
    if (lane < 8) {
      misc[M_CR + lane] = cr[lane];
      misc[M_DE + lane] = de[lane];
    }
    __syncwarp();
  }
  const uint32_t* wninfo = (const uint32_t*)(wsm + L.misc) + M_NINFO;
  const int* wcr = (const int*)(wsm + L.misc) + M_CR;
  const int* wde = (const int*)(wsm + L.misc) + M_DE;
  if (!P.ovf_pass) {
    // dynamic instance scheduler; the next index is claimed one instance ahead so the atomic's
    // latency overlaps the current instance's work
    unsigned long long nxt = 0;
    if (lane == 0) nxt = atomicAdd(P.counter, 1ull);
    for (;;) {
      const unsigned long long inst = __shfl_sync(FULL, nxt, 0);
      if ((int64_t)inst >= P.I) break;
      if (lane == 0) nxt = atomicAdd(P.counter, 1ull);
      solve_instance<NC, PIPE>(P, (int64_t)inst, wsm, L, wninfo, wcr, wde, lane);
      __syncwarp();
    }
  } else {
    if (*(volatile unsigned long long*)P.ovf_count == 0) return;
    const int64_t nwords = (P.I + 31) >> 5;
    for (;;) {
      unsigned long long wd = 0;
      if (lane == 0) wd = atomicAdd(P.counter, 1ull);
      wd = __shfl_sync(FULL, wd, 0);
      if ((int64_t)wd >= nwords) break;
      unsigned bits = P.ovf[wd];
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        solve_instance<NC, PIPE>(P, (int64_t)wd * 32 + b, wsm, L, wninfo, wcr, wde, lane);
        __syncwarp();
      }
    }
  }
}

}  // namespace farb
