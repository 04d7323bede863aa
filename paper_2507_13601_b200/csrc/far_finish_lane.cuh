// far_finish_lane.cuh — H6/H7 (Alg. 2, line-26 replay P:557, keep-best guard P:812)
// with ONE THREAD PER INSTANCE, for the pipelined solver (far_pipeline.cuh K5).
//
// Phase 3 on a realistic instance touches node lists of ~10-20 tasks: a warp spends most of
// its issue slots on reductions, ballots and list shifts whose lanes are mostly idle.  Here
// each thread runs Alg. 2 and the replay of its own instance sequentially, so a warp issues
// one instruction for 32 instances.  The readings, tie-breaks and counters are those of
// refine_warp / replay_warp (far_kernel.cuh); the two paths are bit-identical by construction
// and both are checked against the oracle (tests/test_gpu_parity.py).
//
// Per-thread state in shared memory (one row per thread):
//   ent[n]   u32  the node lists, concatenated in node-id order; entry = D << 10 | (1023 - task)
//                 (D = duration at the task's size, < 2^22 on this path), so "ordered by
//                 T.time, ties -> lower index" is the descending order of entries
//   off[NN+1] u16 segment offsets of the node lists inside ent
//   bit 9 of an entry is CLEARED for a task that runs at the second size its node hosts (A100
//                 {S0..S3} running a 3-slice task; for n <= 256 the bit is 1 in every 1023 - task, and
//                 such tasks never change node or get compared: that node has no same-size alternative)
// Slice ends live in registers (7 slots, compile-time indexed).
#pragma once
#include "far_pipeline.cuh"

namespace farb {

struct LRow {
  int ent, off, bytes;  // byte offsets inside one thread's row
};
__host__ __device__ inline LRow make_lrow(int n, int NN) {
  LRow r;
  int o = 0;
  r.ent = o; o += 4 * ((n + 3) & ~3);
  r.off = o; o += 2 * (NN + 1);
  o = (o + 15) & ~15;
  r.bytes = o + 4;  // odd word stride: the 32 rows of a warp start in 32 different banks
  return r;
}

// entry word of task j with duration d; `second`: the task runs at its node's second size
__device__ __forceinline__ uint32_t lane_entry(int d, int j, bool second) {
  return ((uint32_t)d << 10) | ((uint32_t)(1023 - j) & (second ? ~512u : ~0u));
}
__device__ __forceinline__ int entry_task(uint32_t x) { return 1023 - (int)((x & 1023u) | 512u); }

template <int NC>
__device__ __forceinline__ uint32_t cnode(int u) {
  return NC == 3 ? c_nodes3[u] : c_nodes5[u];
}

// Move the entry x from node `from` to node `to` at its ordered position.
template <int NN>
__device__ __forceinline__ void lane_transfer(uint32_t* ent, uint16_t* off, int from, int to, uint32_t x) {
  // index of x in from's segment
  int g = off[from];
  while (ent[g] != x) ++g;
  // position in to's segment: entries ordered before x
  int p = 0;
  const int b = off[to], e = off[to + 1];
  for (int q = b; q < e; ++q) p += ent[q] > x;
  if (to > from) {  // segments (from, to] move left by one
    const int tgt = e - 1 - (e - b - p);  // = off[to] - 1 + p
    for (int q = g; q < tgt; ++q) ent[q] = ent[q + 1];
    ent[tgt] = x;
    for (int v = from + 1; v <= to; ++v) off[v] = (uint16_t)(off[v] - 1);
  } else {  // segments (to, from] move right by one
    const int tgt = b + p;
    for (int q = g; q > tgt; --q) ent[q] = ent[q - 1];
    ent[tgt] = x;
    for (int v = to + 1; v <= from; ++v) off[v] = (uint16_t)(off[v] + 1);
  }
}

// Replace entry x_old at index g of the ordered segment [b, e) by x_new, keeping the segment in
// descending entry order.  A swap removes T_k from I and inserts T_j, and removes T_j
// from I^a and inserts T_k: on ordered lists this is the same as the two transfers of the warp
// path (K: I -> I^a, then J: I^a -> I), without moving the segments in between.
__device__ __forceinline__ void lane_replace(uint32_t* ent, int b, int e, int g, uint32_t x_new) {
  if (x_new < ent[g]) {  // later in the order
    for (; g + 1 < e && ent[g + 1] > x_new; ++g) ent[g] = ent[g + 1];
  } else {  // earlier in the order
    for (; g > b && ent[g - 1] < x_new; --g) ent[g] = ent[g - 1];
  }
  ent[g] = x_new;
}

// Alg. 2 line 11: I^a = the node of I's size, != I, with the minimum end of its last
// slice (ties -> lower first slice).  Only the leaves and the 2-slice nodes have same-size
// alternatives in the Fig. 3 trees (every other size has one node: A30 4; A100 7, 4, 3), so the
// search is over those two compile-time classes; key = end << 3 | first slice.  Returns -1 if
// there is no alternative (then lines 23-24 open the parent).
template <int NC>
__device__ __forceinline__ int lane_alt(int I, const int (&send)[Tree<NC>::S], uint32_t cand, int& eA) {
  constexpr int S = Tree<NC>::S;
  const uint32_t wI = cnode<NC>(I);
  const int szI = nd_sz(wI), loI = nd_lo(wI);
  unsigned key = 0xFFFFFFFFu;
  if (szI == 1) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int u = tree_leaf<NC>(s);
      const unsigned k = ((unsigned)send[s] << 3) | (unsigned)s;
      if (s != loI && ((cand >> u) & 1)) key = min(key, k);
    }
  } else if (szI == 2) {
#pragma unroll
    for (int u = 0; u < Tree<NC>::NN; ++u) {
      const uint32_t wu = tree_node<NC>(u);
      if (nd_sz(wu) != 2) continue;
      const int lo = nd_lo(wu);
      const unsigned k = ((unsigned)max(send[lo], send[lo + 1]) << 3) | (unsigned)lo;
      if (u != I && ((cand >> u) & 1)) key = min(key, k);
    }
  }
  if (key == 0xFFFFFFFFu) return -1;
  eA = (int)(key >> 3);
  const int lo = (int)(key & 7u);
  if (szI == 1) return tree_leaf<NC>(lo);
#pragma unroll
  for (int u = 0; u < Tree<NC>::NN; ++u)
    if (nd_sz(tree_node<NC>(u)) == 2 && nd_lo(tree_node<NC>(u)) == lo) return u;
  return -1;
}

// Alg. 2 on one thread; same readings as refine_warp.
template <int NC>
__device__ void refine_lane(uint32_t* ent, uint16_t* off, int (&send)[Tree<NC>::S], int max_it, int ppm,
                            bool nonempty_alt, int& moves, int& swaps, int& iters, long long& evals) {
  constexpr int S = Tree<NC>::S, NN = Tree<NC>::NN;
  int omega = 0;
#pragma unroll
  for (int s = 0; s < S; ++s) omega = max(omega, send[s]);
  moves = swaps = iters = 0;
  evals = 0;
  // candidate nodes for I^a: all, or (FAR_NONEMPTY_ALT) those holding a task -- a bit mask kept
  // up to date by the transfers
  uint32_t cand = 0xFFFFu;
  if (nonempty_alt) {
    cand = 0;
    for (int v = 0; v < NN; ++v) cand |= (uint32_t)(off[v + 1] > off[v]) << v;
  }
  auto upd = [&](int v) {
    if (nonempty_alt) cand = (cand & ~(1u << v)) | ((uint32_t)(off[v + 1] > off[v]) << v);
  };
  bool stop = false;
  while (!stop && iters < max_it) {
    ++iters;
    const int omega_prev = omega;
    unsigned long long Q = 0;  // FIFO of node ids, 4 bits each
    int qh = 0, qt = 0;
    uint32_t opened = 0;
    // line 5: leaves of the slices reaching omega, ascending slice order
#pragma unroll
    for (int s = 0; s < S; ++s)
      if (send[s] == omega) {
        const int leaf = leaf_of<NC>(s);
        Q |= (unsigned long long)leaf << (4 * qt++);
        opened |= 1u << leaf;
      }
    while (qh < qt) {
      const int I = (int)((Q >> (4 * qh++)) & 15);
      if (I == 0) { stop = true; break; }
      const uint32_t wI = cnode<NC>(I);
      // alternative I^a: same size, != I, minimum (end, first slice)
      int eA = INT_MAX;
      const int A = lane_alt<NC>(I, send, cand, eA);
      bool done = false;
      if (A >= 0) {
        const int m = omega - eA;
        const int bI = off[I], nI = off[I + 1] - bI;
        evals += nI;
        // move: argmin (|2t - m|, index) over t < m; I is ordered by t descending, so there is no
        // candidate unless its last (shortest) task is shorter than m -- the common case
        unsigned bd = UINT_MAX;
        int bj = INT_MAX;
        uint32_t bx = 0;
        const bool movable = nI > 0 && (int)(ent[bI + nI - 1] >> 10) < m;
        for (int q = bI; movable && q < bI + nI; ++q) {
          const uint32_t x = ent[q];
          const int t = (int)(x >> 10), j = 1023 - (int)(x & 1023u);
          if (t < m) {
            const unsigned d = (unsigned)abs(2 * t - m);
            if (d < bd || (d == bd && j < bj)) { bd = d; bj = j; bx = x; }
          }
        }
        if (bd != UINT_MAX) {
          lane_transfer<NN>(ent, off, I, A, bx);
          upd(I);
          upd(A);
          const int delta = (int)(bx >> 10);
#pragma unroll
          for (int s = 0; s < S; ++s) {
            if (s >= nd_lo(wI) && s < nd_lo(wI) + nd_sz(wI)) send[s] -= delta;
          }
          const uint32_t wA = cnode<NC>(A);
#pragma unroll
          for (int s = 0; s < S; ++s) {
            if (s >= nd_lo(wA) && s < nd_lo(wA) + nd_sz(wA)) send[s] += delta;
          }
          ++moves;
          done = true;
        } else {
          const int bA = off[A], nA = off[A + 1] - bA;
          evals += (long long)nI * nA;
          // argmin over pairs of (|2(t_k - t_j) - m|, k, j), 0 < t_k - t_j < m.  Both lists are
          // ordered by (t desc, task asc) (single-size nodes: LPT order of Alg. 1, kept by the
          // ordered inserts; the two-size {S0..S3} node has no same-size alternative), so for
          // t_k descending the best partners -- the first entry with 2 t_j <= 2 t_k - m and the
          // first entry of the block of equal t just above it -- move monotonically: a
          // two-pointer sweep instead of the |I| * |A| scan (same argmin, same tie-breaks).
          unsigned bd2 = UINT_MAX, bkey = UINT_MAX;
          uint32_t xk = 0, xj = 0;
          int gk = 0, gj = 0;  // indices of the chosen T_k (in I) and T_j (in I^a)
          const int eAo = bA + nA;
          // a pair needs t_k > t_j: none if I's longest task is not longer than I^a's shortest
          const bool any = m > 1 && nI > 0 && nA > 0 && (ent[bI] >> 10) > (ent[eAo - 1] >> 10);
          if (any) {
            // r: first entry of I^a with 2t <= T (cur = ent[r], 0 past the end); bst: start of the
            // equal-t block before r (bv = ent[bst]); registers hold the entries so that a
            // pointer step is one shared-memory load
            int r = bA, bst = bA;
            uint32_t cur = ent[bA], bv = cur, prevt = 0xFFFFFFFFu;
            uint32_t a = ent[bI];
            for (int q = bI; q < bI + nI; ++q) {
              const uint32_t an = q + 1 < bI + nI ? ent[q + 1] : 0u;  // next T_k, loaded ahead
              const int tk = (int)(a >> 10), k = 1023 - (int)(a & 1023u);
              const int T = 2 * tk - m;
              while (r < eAo && 2 * (int)(cur >> 10) > T) {
                if ((cur >> 10) != prevt) { bst = r; bv = cur; }
                prevt = cur >> 10;
                ++r;
                cur = r < eAo ? ent[r] : 0u;
              }
              // below (or equal): entry r (first of its equal-t block); needs t_j > t_k - m
              if (r < eAo) {
                const int dl = tk - (int)(cur >> 10);
                if (dl < m) {  // dl > 0 since 2 t_j <= 2 t_k - m < 2 t_k
                  const unsigned d = (unsigned)abs(2 * dl - m);
                  const unsigned key = ((unsigned)k << 10) | (unsigned)(1023 - (int)(cur & 1023u));
                  if (d < bd2 || (d == bd2 && key < bkey)) { bd2 = d; bkey = key; xk = a; xj = cur; gk = q; gj = r; }
                }
              }
              // above: first entry of the block before r; needs t_j < t_k
              if (r > bA) {
                const int dl = tk - (int)(bv >> 10);
                if (dl > 0) {  // dl < m since 2 t_j > 2 t_k - m
                  const unsigned d = (unsigned)abs(2 * dl - m);
                  const unsigned key = ((unsigned)k << 10) | (unsigned)(1023 - (int)(bv & 1023u));
                  if (d < bd2 || (d == bd2 && key < bkey)) { bd2 = d; bkey = key; xk = a; xj = bv; gk = q; gj = bst; }
                }
              }
              a = an;
            }
          }
          if (bd2 != UINT_MAX) {  // T_k: I -> I^a and T_j: I^a -> I, both lists kept ordered
            lane_replace(ent, bI, bI + nI, gk, xj);
            lane_replace(ent, bA, eAo, gj, xk);
            const int delta = (int)(xk >> 10) - (int)(xj >> 10);
            const uint32_t wA = cnode<NC>(A);
#pragma unroll
            for (int s = 0; s < S; ++s) {
              if (s >= nd_lo(wI) && s < nd_lo(wI) + nd_sz(wI)) send[s] -= delta;
              if (s >= nd_lo(wA) && s < nd_lo(wA) + nd_sz(wA)) send[s] += delta;
            }
            ++swaps;
            done = true;
          }
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
    omega = 0;
#pragma unroll
    for (int s = 0; s < S; ++s) omega = max(omega, send[s]);
    if (ppm > 0 && (long long)(omega_prev - omega) * 1000000LL < (long long)ppm * omega_prev) break;
  }
}

// Node lists of k* from the phase-2 record (node | size index << 4 | position << 7 per task,
// node list lengths in ncnt); fills ent/off.
template <int NC>
__device__ void lane_lists(int n, const uint32_t* __restrict__ rec, const uint16_t* __restrict__ ncnt,
                           const int32_t* __restrict__ t, uint32_t* ent, uint16_t* off) {
  constexpr int NN = Tree<NC>::NN;
  int acc = 0;
#pragma unroll
  for (int v = 0; v < NN; ++v) {
    off[v] = (uint16_t)acc;
    acc += __ldg(ncnt + v);
  }
  off[NN] = (uint16_t)acc;
#pragma unroll 4
  for (int j = 0; j < n; ++j) {
    const uint32_t r = __ldg(rec + j);
    const int v = (int)(r & 15u), c = (int)((r >> 4) & 7u), pos = (int)(r >> 7);
    ent[off[v] + pos] = lane_entry(__ldg(t + j * NC + c), j, c != nd_c0(cnode<NC>(v)));
  }
}

// Warp-cooperative form of lane_lists for the active lanes' instances (mask am): the record of
// instance i is read by the whole warp with coalesced 16-B loads (instead of one thread walking
// 512 B with dependent loads) and its entries are written into lane i's row; the loads of four
// instances are in flight together.  k0: bit i set if instance i's winner is member 0 (then the
// durations prep wrote are read coalesced instead of gathered from the runtime table).  The rows'
// off[] must already hold the node offsets.
template <int NC>
__device__ void lane_lists_coop(int n, int64_t base, unsigned am, unsigned k0, const KParams& P, unsigned char* wrows,
                                int rbytes, const LRow& L, int lane) {
  auto put = [&](uint32_t* ent, const uint16_t* off, const int32_t* t, int j, uint32_t r, int d) {
    const int v = (int)(r & 15u), c = (int)((r >> 4) & 7u), pos = (int)(r >> 7);
    if (d < 0) d = __ldg(t + j * NC + c);
    ent[off[v] + pos] = lane_entry(d, j, c != nd_c0(cnode<NC>(v)));
  };
  if ((n & 3) == 0) {
    const int n4 = n >> 2;
    const uint4 NOD = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
    auto load = [&](int i, int q, uint4& x, uint4& dd) {
      const int64_t inst = base + i;
      x = __ldcs((const uint4*)(P.ws_rec + inst * (int64_t)n) + q);
      dd = ((k0 >> i) & 1) ? __ldcs((const uint4*)(P.ws_d0 + inst * (int64_t)P.ws_n4) + q) : NOD;
    };
    // groups of 4 instances: their 16-B record / duration loads are issued together, then scattered
    // (one exposed load latency per group instead of per instance)
    for (; am;) {
      int ids[4];
      uint4 x[4], dd[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        ids[u] = am ? __ffs(am) - 1 : -1;
        am &= am - 1;
      }
      for (int q = lane; q < n4; q += 32) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          x[u] = NOD;
          dd[u] = NOD;
          if (ids[u] >= 0) load(ids[u], q, x[u], dd[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (ids[u] < 0) continue;
          const int64_t inst = base + ids[u];
          unsigned char* row = wrows + (size_t)ids[u] * rbytes;
          uint32_t* ent = (uint32_t*)(row + L.ent);
          const uint16_t* off = (const uint16_t*)(row + L.off);
          const int32_t* t = P.times + inst * (int64_t)n * NC;
          put(ent, off, t, 4 * q, x[u].x, (int)dd[u].x);
          put(ent, off, t, 4 * q + 1, x[u].y, (int)dd[u].y);
          put(ent, off, t, 4 * q + 2, x[u].z, (int)dd[u].z);
          put(ent, off, t, 4 * q + 3, x[u].w, (int)dd[u].w);
        }
      }
    }
  } else {
    for (; am; am &= am - 1) {
      const int i = __ffs(am) - 1;
      const int64_t inst = base + i;
      unsigned char* row = wrows + (size_t)i * rbytes;
      const uint32_t* rec = P.ws_rec + inst * (int64_t)n;
      const int32_t* t = P.times + inst * (int64_t)n * NC;
      for (int j = lane; j < n; j += 32)
        put((uint32_t*)(row + L.ent), (const uint16_t*)(row + L.off), t, j, __ldcs(rec + j), -1);
    }
  }
  __syncwarp();
}

// Node-level replay (the frontier in registers of this thread); writes the schedule when
// `out` is not null; returns the makespan.
template <int NC>
__device__ int lane_replay(const uint32_t* ent, const uint16_t* off, const int* cr,
                           const int* de, far_task_slot* out) {
  constexpr int S = Tree<NC>::S;
  Frontier<S> F;
  F.init();
  int rec = 0, ms = 0;
  while (F.live) {
    int bs, be;
    F.pop(bs, be);
    const int v = F.node(bs);
    const uint32_t w = cnode<NC>(v);
    const int b = off[v], e = off[v + 1];
    if (!((F.has >> bs) & 1) && e > b) {  // creation (lines 8-11), then all of v's tasks
      rec = max(rec, be) + cr[nd_szi(w)];
      int acc = rec;
      if (out) {
        // slot word node | size << 8 | start << 32; only the two-size node has second-size entries
        const unsigned lo0 = (unsigned)v | ((unsigned)size_of<NC>(nd_c0(w)) << 8);
        const bool two = nd_c1(w) != NONE;
        const unsigned lo1 = two ? (unsigned)v | ((unsigned)size_of<NC>(nd_c1(w)) << 8) : lo0;
        for (int q = b; q < e; ++q) {
          const uint32_t x = ent[q];
          const int j = entry_task(x);
          const unsigned lo = (two && !(x & 512u)) ? lo1 : lo0;
          *(unsigned long long*)(out + j) = (unsigned long long)lo | ((unsigned long long)(unsigned)acc << 32);
          acc += (int)(x >> 10);
        }
      } else {
        for (int q = b; q < e; ++q) acc += (int)(ent[q] >> 10);
      }
      ms = max(ms, acc);
      F.has |= 1u << bs;
      F.set(bs, acc);
    } else {  // repartitioning (lines 17-24): destroy if it had tasks, then split or drop
      if ((F.has >> bs) & 1) rec = max(rec, be) + de[nd_szi(w)];
      F.split(bs, be, w);
    }
  }
  return ms;
}

template <int NC>
__global__ void __launch_bounds__(128, 3) far_finish_lane_kernel(KParams P) {
  constexpr int S = Tree<NC>::S, NN = Tree<NC>::NN;
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ int s_cr[8], s_de[8];
  if (threadIdx.x < 8) {
    s_cr[threadIdx.x] = P.cr[threadIdx.x];
    s_de[threadIdx.x] = P.de[threadIdx.x];
  }
  __syncthreads();
  const int n = P.n;
  const LRow L = make_lrow(n, NN);
  unsigned char* row = dsm + (size_t)threadIdx.x * L.bytes;
  uint32_t* ent = (uint32_t*)(row + L.ent);
  uint16_t* off = (uint16_t*)(row + L.off);
  const bool want_sched = P.sched != nullptr && !(P.flags & FAR_NO_SCHEDULE);
  const bool refine = !(P.flags & FAR_NO_REFINE);
  const bool need_replay = refine || want_sched;
  const int lane = threadIdx.x & 31;
  unsigned char* wrows = dsm + (size_t)(threadIdx.x & ~31) * L.bytes;
  // the lanes of a warp hold 32 consecutive instances and step together (the list staging is
  // warp-cooperative); batches of 32 are claimed from a counter, one ahead, so that the warps
  // finish together although their batches' refine work differs
  // (a grid that covers every instance in one pass takes its batch by position: no atomics)
  const bool one_pass = (int64_t)gridDim.x * blockDim.x >= P.I;
  unsigned long long nb = (unsigned long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
  if (!one_pass && lane == 0) nb = atomicAdd(P.counter, 32ull);
  for (;;) {
    const int64_t base = (int64_t)__shfl_sync(FULL, nb, 0);
    if (base >= P.I) break;
    if (one_pass) nb = (unsigned long long)P.I;
    else if (lane == 0) nb = atomicAdd(P.counter, 32ull);
    const int64_t inst = base + lane;
    // error / empty (K1 wrote the outputs) / deferred to the overflow pass: nothing to finish
    const bool active = inst < P.I && !P.ws_meta[inst * 16 + WS_FLAG];
    if (active) {
      int acc = 0;
      const uint16_t* nc = P.ws_ncnt + inst * 16;
#pragma unroll
      for (int v = 0; v < NN; ++v) {
        off[v] = (uint16_t)acc;
        acc += __ldg(nc + v);
      }
      off[NN] = (uint16_t)acc;
    }
    const unsigned long long best = active ? P.ws_best[inst] : 0ull;
    __syncwarp();
    lane_lists_coop<NC>(n, inst - lane, __ballot_sync(FULL, active), __ballot_sync(FULL, active && !(best & 0xFFFFull)),
                        P, wrows, L.bytes, L, lane);
    if (!active) continue;
    const int* meta = P.ws_meta + inst * 16;
    const int ms2 = (int)(best >> 16), bestk = (int)(best & 0xFFFFu);
    far_result R;
    R.makespan = 0; R.makespan_phase2 = ms2; R.alloc_index = bestk; R.family_size = meta[WS_K];
    R.moves = 0; R.swaps = 0; R.iterations = 0; R.reverted = 0; R.status = FAR_OK; R.reserved = 0;
    R.evals = 0; R.events = (long long)P.ws_evt[inst];
    const uint32_t* rec = P.ws_rec + inst * (int64_t)n;
    const int32_t* t = P.times + inst * (int64_t)n * NC;
    far_task_slot* out = want_sched ? P.sched + inst * (int64_t)n : nullptr;
    int msF = ms2;
    for (int pass = 0; pass < 2; ++pass) {
      if (pass) lane_lists<NC>(n, rec, P.ws_ncnt + inst * 16, t, ent, off);
      const bool ref = refine && pass == 0;
      if (ref) {
        int send[S];
#pragma unroll
        for (int s = 0; s < S; ++s) send[s] = P.ws_sl[inst * 8 + s];
        int mv, sw, it;
        long long ev;
        refine_lane<NC>(ent, off, send, P.max_it, P.ppm, (P.flags & FAR_NONEMPTY_ALT) != 0, mv, sw, it, ev);
        R.moves = mv; R.swaps = sw; R.iterations = it; R.evals = ev;
      }
      if (!need_replay) break;
      const int msR = lane_replay<NC>(ent, off, s_cr, s_de, out);
      if (ref && !(P.flags & FAR_NO_GUARD) && msR > ms2) {
        R.reverted = 1;  // keep-best guard: return the phase-2 schedule (replayed in pass 1)
        if (!want_sched) break;
        continue;
      }
      if (ref) msF = msR;
      break;
    }
    R.makespan = msF;
    P.makespan[inst] = R.makespan;
    if (P.res) P.res[inst] = R;
  }
}

}  // namespace farb
