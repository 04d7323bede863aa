// far_forest.cuh — multi-target FAR: FAR for g MIG GPUs scheduled together.
//
// "the method can be used seamlessly for multiple A30s and multiple
// A100/H100s; for that, there would be as many trees as GPUs, and initially, there is one
// node for the root of each tree to start repartitioning on."  Everything else is FAR as
// for one GPU (R31): the Turek family, Alg. 1 with one heap over the
// forest and one reconfig_end, Alg. 2 with alternatives among the same-size
// nodes of every tree, stopping when a root is opened, line-26 replay + guard.
// Node ids: tree t's node v is t*NN + v, its slices t*S + [lo, hi) (include/far.h).
//
// One WARP per instance, everything in shared memory, generic node tables (g <= 8 trees,
// <= 104 nodes, <= 56 slices, n <= 256):
//   phases 1+2 fused in one loop: member k's longest task by a warp argmax, its lower bound
//     max(h_k, ceil(W_k / #slices)) (exact pruning as in the single-GPU chain: a member
//     whose bound reaches the best makespan so far cannot win), Alg. 1 on the member
//     if it can, then the growth step as an ordered remove/insert on the per-size
//     LPT lists of the current allocation (Alg. 1 lines 1-2);
//   Alg. 1: the frontier is an antichain, so slot s = the frontier node whose first slice is
//     s; lane l holds slots l and l + 32; a pop is two REDUX.MIN (end, then first slice);
//   each simulated member records (node, start, size, position) into a double buffer; the
//     best member's buffer becomes the phase-2 schedule (no re-simulation);
//   Alg. 2 on node lists concatenated in node-id order (one u16 array + segment offsets);
//   replay = the same Alg. 1 loop taking each node's tasks from its list.
// The single-GPU trees keep their specialised pipeline (far_kernel.cuh / far_pipeline.cuh).
#pragma once
#include "far_kernel.cuh"

namespace farb {

constexpr int FMAXN = 256, FMAXG = 8, FMAXNN = 104, FMAXS = 56;
constexpr int FNONE = 255;

// node word: x = lo | sz << 8 | szi << 12 | c0 << 16 | c1 << 20 ; y = ch1 | ch2 << 8 | par << 16
struct FParams {
  KParams P;
  const uint2* nodes;  // [NNF]
  int NNF, SF;
};

__device__ __forceinline__ int fn_lo(uint2 w) { return (int)(w.x & 255u); }
__device__ __forceinline__ int fn_sz(uint2 w) { return (int)((w.x >> 8) & 15u); }
__device__ __forceinline__ int fn_szi(uint2 w) { return (int)((w.x >> 12) & 15u); }
__device__ __forceinline__ int fn_c0(uint2 w) { return (int)((w.x >> 16) & 15u); }
__device__ __forceinline__ int fn_c1(uint2 w) { return (int)((w.x >> 20) & 15u); }
__device__ __forceinline__ int fn_ch1(uint2 w) { return (int)(w.y & 255u); }
__device__ __forceinline__ int fn_ch2(uint2 w) { return (int)((w.y >> 8) & 255u); }
__device__ __forceinline__ int fn_par(uint2 w) { return (int)((w.y >> 16) & 255u); }

// per-warp shared-memory layout (bytes)
struct FLay {
  int T, glist, cur, rs[2], rn[2], rp[2], ru[2], ncnt, L, off, cursor, send, D, Q, opened, leaf, misc, tnode, srt,
      nstat, isz, bytes;
};
__host__ __device__ inline FLay make_flay(int n, int NC, int NNF, int SF) {
  FLay L;
  int o = 0;
  auto take = [&](int b) { const int r = o; o = al16(o + b); return r; };
  L.T = take(4 * n * NC);
  L.glist = take(2 * n * NC);
  L.cur = take(n);
  for (int b = 0; b < 2; ++b) {
    L.rs[b] = take(4 * n);
    L.rn[b] = take(n);
    L.rp[b] = take(n);
    L.ru[b] = take(n);
  }
  L.ncnt = take(4 * NNF);
  L.L = take(2 * n + 2);
  L.off = take(4 * (NNF + 1));
  L.cursor = take(4 * NNF);
  L.send = take(4 * SF);
  L.D = take(4 * n);
  L.Q = take(NNF + 1);
  L.opened = take(NNF + 1);
  L.leaf = take(SF);
  L.misc = take(4 * 32);
  L.tnode = take(n);        // best-improvement: node of each task
  L.srt = take(8 * SF);     // best-improvement: slice ends sorted descending (value, slice)
  L.nstat = take(8 * NNF);  // best-improvement: (max, count) of each node's slice ends
  L.isz = take(NNF);        // FAR_SWITCH_COST: size index of each node's current instance
  L.bytes = o;
  return L;
}
enum { FM_GCNT = 0, FM_GPTR = 8, FM_END = 16 };

// Alg. 1 over the forest.  LISTS = false: tasks from the per-size LPT lists of the
// current allocation (glist / gcnt); true: the line-26 replay taking node v's tasks from its
// segment of the concatenated lists (L, off), with size index su[j].  Records each placement.
template <int NC, bool LISTS>
__device__ int forest_sim(const FParams& F, int n, const int32_t* T, const uint16_t* glist, const int* gcnt, int* gptr,
                          const uint16_t* L, const int* off, int* cursor, const uint8_t* su, int* rstart,
                          uint8_t* rnode, uint8_t* rpos, uint8_t* rsu, int* ncnt, long long& pops, int lane,
                          uint8_t* isz, far_event* ev = nullptr, int* nevp = nullptr) {
  // ev (optional): the reconfiguration events in the order rec issues them (creates, and the
  // destroys of lines 18-20 while tasks remain), nevp their count
  const KParams& P = F.P;
  int nev = 0;
  const int NNF = F.NNF;
  const bool r7 = (P.flags & FAR_SWITCH_COST) != 0;  // DESIGN.md R7 variant
  for (int v = lane; v < NNF; v += 32) {
    ncnt[v] = 0;
    if (LISTS) cursor[v] = off[v];
  }
  if (!LISTS && lane < NC) gptr[lane] = 0;
  int nd0 = -1, nd1 = -1, e0 = 0, e1 = 0, h0 = 0, h1 = 0;
  for (int v = 0; v < NNF; ++v) {  // the root of every tree starts at time 0
    const uint2 w = __ldg(F.nodes + v);
    if (fn_par(w) != FNONE) continue;
    const int s = fn_lo(w);
    if ((s & 31) == lane) {
      if (s < 32) nd0 = v; else nd1 = v;
    }
  }
  __syncwarp();
  int rec = 0, ms = 0, unsched = n;
  for (;;) {
    const unsigned em = min(nd0 >= 0 ? (unsigned)e0 : UINT_MAX, nd1 >= 0 ? (unsigned)e1 : UINT_MAX);
    const unsigned emin = __reduce_min_sync(FULL, em);
    if (emin == UINT_MAX) break;
    const int sc = (nd0 >= 0 && (unsigned)e0 == emin) ? lane : ((nd1 >= 0 && (unsigned)e1 == emin) ? lane + 32 : 64);
    const int smin = __reduce_min_sync(FULL, (unsigned)sc);
    const int owner = smin & 31;
    const bool hi = smin >= 32;
    const int pk = __shfl_sync(FULL, hi ? (nd1 | (h1 << 8)) : (nd0 | (h0 << 8)), owner);
    const int v = pk & 255;
    int has = pk >> 8;
    int end = (int)emin;
    ++pops;
    const uint2 w = __ldg(F.nodes + v);
    const int cur_isz = r7 ? isz[v] : 0;
    int take = -1, tc = 0;
    if (LISTS) {
      if (cursor[v] < off[v + 1]) {
        take = L[cursor[v]];
        tc = su[take];
      }
    } else {
      const int c0 = fn_c0(w), c1 = fn_c1(w);
      if (gptr[c0] < gcnt[c0]) {
        take = glist[c0 * n + gptr[c0]];
        tc = c0;
      } else if (c1 != NONE && gptr[c1] < gcnt[c1]) {
        take = glist[c1 * n + gptr[c1]];
        tc = c1;
      }
    }
    __syncwarp();
    int nslot_node = -1, nslot2 = -1, ch2 = -1, s2 = 0, ne = end;
    bool clear = false;
    if (take >= 0) {
      if (!has) {  // lines 8-11: give time for I's creation
        const int cs = max(rec, end);
        rec = cs + P.cr[r7 ? tc : fn_szi(w)];
        if (ev) {
          if (lane == 0) ev[nev] = far_event{0, v, cs, rec - cs};
          ++nev;
        }
        end = rec;
        has = 1;
        if (lane == 0) isz[v] = (uint8_t)tc;
      } else if (r7 && fn_c1(w) != NONE && tc != cur_isz) {  // variant: destroy, then re-create
        rec = max(rec, end) + P.de[cur_isz];
        rec += P.cr[tc];
        end = rec;
        if (lane == 0) isz[v] = (uint8_t)tc;
      }
      const int st = end;
      end += T[take * NC + tc];
      ms = max(ms, end);
      --unsched;
      if (lane == 0) {
        if (LISTS) ++cursor[v]; else ++gptr[tc];
        rstart[take] = st;
        rnode[take] = (uint8_t)v;
        rsu[take] = (uint8_t)tc;
        rpos[take] = (uint8_t)ncnt[v];
        ++ncnt[v];
      }
      nslot_node = v;
      ne = end;
    } else if (unsched > 0) {  // line 17: repartition
      if (has) {  // lines 18-20
        const int ds = max(rec, end);
        rec = ds + P.de[(r7 && fn_c1(w) != NONE) ? cur_isz : fn_szi(w)];
        if (ev) {
          if (lane == 0) ev[nev] = far_event{1, v, ds, rec - ds};
          ++nev;
        }
      }
      if (fn_ch1(w) == FNONE) {
        clear = true;
      } else {  // lines 21-24: children start at I.end
        nslot_node = fn_ch1(w);
        ch2 = fn_ch2(w);
        s2 = fn_lo(__ldg(F.nodes + ch2));
        nslot2 = ch2;
        has = 0;
      }
    } else {
      clear = true;  // drop
    }
    if (lane == owner) {
      if (hi) {
        if (clear) nd1 = -1; else { nd1 = nslot_node; e1 = ne; h1 = has; }
      } else {
        if (clear) nd0 = -1; else { nd0 = nslot_node; e0 = ne; h0 = has; }
      }
    }
    if (nslot2 >= 0 && lane == (s2 & 31)) {
      if (s2 >= 32) { nd1 = nslot2; e1 = ne; h1 = 0; } else { nd0 = nslot2; e0 = ne; h0 = 0; }
    }
    __syncwarp();
  }
  if (nevp && lane == 0) *nevp = nev;
  return ms;
}

// concatenated node lists: remove task x (segment of node a)
__device__ void fl_remove(uint16_t* L, int* off, int NNF, int n, int x, int a, int lane) {
  int p = -1;
  for (int b = off[a]; b < off[a + 1]; b += 32) {
    const unsigned m = __ballot_sync(FULL, b + lane < off[a + 1] && L[b + lane] == x);
    if (m) { p = b + __ffs(m) - 1; break; }
  }
  const int len = off[NNF];
  for (int b = p; b < len - 1; b += 32) {  // shift left, chunk by chunk in increasing order
    const int i = b + lane;
    const uint16_t val = i < len - 1 ? L[i + 1] : 0;
    __syncwarp();
    if (i < len - 1) L[i] = val;
    __syncwarp();
  }
  for (int v = a + 1 + lane; v <= NNF; v += 32) off[v] -= 1;
  __syncwarp();
}

// insert task x into node b's segment at the first entry not ordered before it by (-t, index)
// (the oracle's linear "Insert T ordered by T.time"; lists need not be sorted: the
// A100 4-slice nodes hold their size-4 tasks before their size-3 tasks)
__device__ void fl_insert(uint16_t* L, int* off, int NNF, int x, int b, const int* D, int lane) {
  const int lo = off[b], hi = off[b + 1], dx = D[x];
  int q = hi;
  for (int c = lo; c < hi; c += 32) {
    const int i = c + lane;
    bool nb = false;
    if (i < hi) {
      const int y = L[i], dy = D[y];
      nb = !(dy > dx || (dy == dx && y < x));
    }
    const unsigned m = __ballot_sync(FULL, nb);
    if (m) { q = c + __ffs(m) - 1; break; }
  }
  const int len = off[NNF];
  for (int top = len - 1; top >= q; top -= 32) {  // shift right, chunk by chunk from the top
    const int i = top - lane;
    const uint16_t val = i >= q ? L[i] : 0;
    __syncwarp();
    if (i >= q) L[i + 1] = val;
    __syncwarp();
  }
  if (lane == 0) L[q] = (uint16_t)x;
  for (int v = b + 1 + lane; v <= NNF; v += 32) off[v] += 1;
  __syncwarp();
}

// Alg. 2 over the forest on the concatenated lists; same readings as refine_warp.
template <int NC>
__device__ void forest_refine(const FParams& F, int n, const int* D, uint16_t* L, int* off, int* send, uint8_t* Q,
                              uint8_t* opened, const uint8_t* leaf, int lane, int& moves, int& swaps, int& iters,
                              long long& evals) {
  const KParams& P = F.P;
  const int NNF = F.NNF, SF = F.SF;
  const bool nonempty_alt = (P.flags & FAR_NONEMPTY_ALT) != 0;
  auto smax = [&]() {
    int m = 0;
    for (int s = lane; s < SF; s += 32) m = max(m, send[s]);
    return (int)__reduce_max_sync(FULL, (unsigned)m);
  };
  int omega = smax();
  moves = swaps = iters = 0;
  evals = 0;
  bool stop = false;
  while (!stop && iters < P.max_it) {
    ++iters;
    const int omega_prev = omega;
    for (int v = lane; v < NNF; v += 32) opened[v] = 0;
    __syncwarp();
    int qt = 0, qh = 0;
    for (int b = 0; b < SF; b += 32) {  // line 5: leaves of the critical slices, ascending
      const int s = b + lane;
      unsigned crit = __ballot_sync(FULL, s < SF && send[s] == omega);
      const int before = qt;
      if (s < SF && send[s] == omega) {
        const int r = __popc(crit & ((1u << lane) - 1));
        Q[before + r] = leaf[s];
        opened[leaf[s]] = 1;
      }
      qt += __popc(crit);
    }
    __syncwarp();
    while (qh < qt) {
      const int I = Q[qh++];
      const uint2 wI = __ldg(F.nodes + I);
      if (fn_par(wI) == FNONE) { stop = true; break; }  // lines 8-10: a root is opened
      // line 11: I^a = argmin (end, first slice) over same-size nodes != I
      unsigned be = UINT_MAX, bl = 255;
      int bu = -1;
      for (int u = lane; u < NNF; u += 32) {
        if (u == I) continue;
        const uint2 wu = __ldg(F.nodes + u);
        if (fn_sz(wu) != fn_sz(wI)) continue;
        if (nonempty_alt && off[u + 1] == off[u]) continue;
        int e = 0;
        for (int s = fn_lo(wu); s < fn_lo(wu) + fn_sz(wu); ++s) e = max(e, send[s]);
        if ((unsigned)e < be || ((unsigned)e == be && (unsigned)fn_lo(wu) < bl)) { be = e; bl = fn_lo(wu); bu = u; }
      }
      const unsigned eA = __reduce_min_sync(FULL, be);
      const unsigned lA = __reduce_min_sync(FULL, be == eA ? bl : 255u);
      const int A = (int)__reduce_max_sync(FULL, (be == eA && bl == lA && bu >= 0) ? (unsigned)bu : 0u);
      bool done = false;
      if (eA != UINT_MAX) {
        const int m = omega - (int)eA;
        const int i0 = off[I], nI = off[I + 1] - i0;
        evals += nI;
        unsigned bd = UINT_MAX, bj = UINT_MAX;
        for (int q = lane; q < nI; q += 32) {
          const int j = L[i0 + q], t = D[j];
          if (t < m) {
            const unsigned d = (unsigned)abs(2 * t - m);
            if (d < bd || (d == bd && (unsigned)j < bj)) { bd = d; bj = j; }
          }
        }
        const unsigned dmin = __reduce_min_sync(FULL, bd);
        int nt = 0, tk0 = 0, tk1 = 0, delta = 0;
        if (dmin != UINT_MAX) {  // lines 13-16: move
          tk0 = (int)__reduce_min_sync(FULL, bd == dmin ? bj : UINT_MAX);
          delta = D[tk0];
          nt = 1;
          ++moves;
        } else {  // lines 17-22: swap
          const int a0 = off[A], nA = off[A + 1] - a0;
          evals += (long long)nI * nA;
          unsigned bd2 = UINT_MAX, bkey = UINT_MAX;
          for (int p = lane; p < nI * nA; p += 32) {
            const int k = L[i0 + p / nA], j = L[a0 + p % nA];
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
            tk1 = (int)(key & 1023u);
            delta = D[tk0] - D[tk1];
            nt = 2;
            ++swaps;
          }
        }
        if (nt) {  // the oracle's order: remove both, then insert each into the other list
          fl_remove(L, off, NNF, n, tk0, I, lane);
          if (nt == 2) fl_remove(L, off, NNF, n, tk1, A, lane);
          fl_insert(L, off, NNF, tk0, A, D, lane);
          if (nt == 2) fl_insert(L, off, NNF, tk1, I, D, lane);
          const uint2 wA = __ldg(F.nodes + A);
          for (int s = lane; s < SF; s += 32) {
            if (s >= fn_lo(wI) && s < fn_lo(wI) + fn_sz(wI)) send[s] -= delta;
            if (s >= fn_lo(wA) && s < fn_lo(wA) + fn_sz(wA)) send[s] += delta;
          }
          __syncwarp();
          done = true;
        }
      }
      if (!done) {  // lines 23-24: open the parent once
        const int par = fn_par(wI);
        if (!opened[par]) {
          __syncwarp();
          if (lane == 0) { opened[par] = 1; Q[qt] = (uint8_t)par; }
          ++qt;
          __syncwarp();
        }
      }
    }
    omega = smax();
    if (P.ppm > 0 && (long long)(omega_prev - omega) * 1000000LL < (long long)P.ppm * omega_prev) break;
  }
}

// Phase-3 variant FAR_BEST_IMPROVEMENT (R30) over the forest: every move of a task to
// another node of the same size (any tree) and every swap of two tasks on different same-size
// nodes is scored by (w', c') = (max slice end after it, #slices at w'); the argmin of (w', c',
// move before swap, first id, second id) is applied while it lowers (w, c).  Same-size nodes are
// disjoint, so a transfer of d ticks a -> b scores max(out(a, b), M_a - d, M_b + d), out(a, b)
// read off the slice ends sorted in descending order (first entries outside a and b).
template <int NC>
__device__ void forest_refine_best(const FParams& F, int n, const int* D, uint16_t* L, int* off, int* send,
                                   uint8_t* tnode, int2* srt, int2* nstat, int lane, int& moves, int& swaps,
                                   int& iters, long long& evals) {
  const KParams& P = F.P;
  const int NNF = F.NNF, SF = F.SF;
  for (int v = 0; v < NNF; ++v)
    for (int q = off[v] + lane; q < off[v + 1]; q += 32) tnode[L[q]] = (uint8_t)v;
  __syncwarp();
  auto lo_of = [&](int v) { return fn_lo(__ldg(F.nodes + v)); };
  auto sz_of = [&](int v) { return fn_sz(__ldg(F.nodes + v)); };
  // (w', c') of moving d ticks from node a to node b (disjoint, same size)
  auto score = [&](int a, int b, int d) {
    const int la = lo_of(a), lb = lo_of(b), z = sz_of(a);
    const int2 na = nstat[a], nb = nstat[b];
    int ow = -1, oc = 0;
    for (int r = 0; r < SF; ++r) {
      const int2 e = srt[r];
      const bool in = (e.y >= la && e.y < la + z) || (e.y >= lb && e.y < lb + z);
      if (in) continue;
      if (ow < 0) ow = e.x;
      if (e.x != ow) break;
      ++oc;
    }
    const int x = na.x - d, y = nb.x + d;
    const int w = max(ow, max(x, y));
    const int c = (ow == w ? oc : 0) + (x == w ? na.y : 0) + (y == w ? nb.y : 0);
    return ((unsigned long long)(unsigned)w << 27) | ((unsigned long long)c << 21);
  };
  moves = swaps = iters = 0;
  evals = 0;
  while (iters < P.max_it) {
    ++iters;
    // slice ends sorted descending (rank by (value desc, slice asc)), node stats, current (w, c)
    for (int s = lane; s < SF; s += 32) {
      const int x = send[s];
      int r = 0;
      for (int u = 0; u < SF; ++u) r += send[u] > x || (send[u] == x && u < s);
      srt[r] = make_int2(x, s);
    }
    for (int v = lane; v < NNF; v += 32) {
      const int l0 = lo_of(v), z = sz_of(v);
      int w = -1, c = 0;
      for (int s = l0; s < l0 + z; ++s) {
        if (send[s] > w) { w = send[s]; c = 1; } else if (send[s] == w) { ++c; }
      }
      nstat[v] = make_int2(w, c);
    }
    __syncwarp();
    int cw = srt[0].x, cc = 0;
    for (int r = 0; r < SF && srt[r].x == cw; ++r) ++cc;
    const unsigned long long cur = ((unsigned long long)(unsigned)cw << 27) | ((unsigned long long)cc << 21);
    unsigned long long best = ~0ull;
    long long ev = 0;
    for (int x = lane; x < n; x += 32) {  // moves
      const int a = tnode[x], z = sz_of(a);
      for (int u = 0; u < NNF; ++u) {
        if (u == a || sz_of(u) != z) continue;
        ++ev;
        const unsigned long long k = score(a, u, D[x]) | ((unsigned long long)x << 10) | (unsigned)u;
        best = k < best ? k : best;
      }
    }
    for (int k = 0; k < n; ++k) {  // swaps k < j
      const int a = tnode[k], z = sz_of(a), dk = D[k];
      for (int j = k + 1 + lane; j < n; j += 32) {
        const int b = tnode[j];
        if (b == a || sz_of(b) != z) continue;
        ++ev;
        const unsigned long long key = score(a, b, dk - D[j]) | (1ull << 20) | ((unsigned long long)k << 10) |
                                       (unsigned)j;
        best = key < best ? key : best;
      }
    }
    evals += warp_sum_ll(ev);
    const unsigned hi = __reduce_min_sync(FULL, (unsigned)(best >> 32));
    const unsigned lo = __reduce_min_sync(FULL, (unsigned)(best >> 32) == hi ? (unsigned)best : ~0u);
    best = ((unsigned long long)hi << 32) | lo;
    if ((best >> 21) >= (cur >> 21)) break;
    const int x = (int)((best >> 10) & 1023), y = (int)(best & 1023);
    int from, to, d, tk1 = -1;
    if (!((best >> 20) & 1)) {
      from = tnode[x]; to = y; d = D[x];
      ++moves;
    } else {
      from = tnode[x]; to = tnode[y]; d = D[x] - D[y]; tk1 = y;
      ++swaps;
    }
    fl_remove(L, off, NNF, n, x, from, lane);
    if (tk1 >= 0) fl_remove(L, off, NNF, n, tk1, to, lane);
    fl_insert(L, off, NNF, x, to, D, lane);
    if (tk1 >= 0) fl_insert(L, off, NNF, tk1, from, D, lane);
    if (lane == 0) {
      tnode[x] = (uint8_t)to;
      if (tk1 >= 0) tnode[tk1] = (uint8_t)from;
    }
    const int lf = lo_of(from), lt = lo_of(to), z = sz_of(from);
    for (int s = lane; s < SF; s += 32) {
      if (s >= lf && s < lf + z) send[s] -= d;
      if (s >= lt && s < lt + z) send[s] += d;
    }
    __syncwarp();
    int om = 0;
    for (int s = lane; s < SF; s += 32) om = max(om, send[s]);
    om = (int)__reduce_max_sync(FULL, (unsigned)om);
    if (P.ppm > 0 && (long long)(cw - om) * 1000000LL < (long long)P.ppm * cw) break;
  }
}

template <int NC>
__global__ void __launch_bounds__(128) far_forest_kernel(FParams F) {
  extern __shared__ __align__(16) unsigned char fsm[];
  const KParams& P = F.P;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int n = P.n, NNF = F.NNF, SF = F.SF;
  const FLay Ly = make_flay(n, NC, NNF, SF);
  unsigned char* wsm = fsm + (size_t)wib * Ly.bytes;
  int32_t* T = (int32_t*)(wsm + Ly.T);
  uint16_t* glist = (uint16_t*)(wsm + Ly.glist);
  uint8_t* cur = wsm + Ly.cur;
  int* ncnt = (int*)(wsm + Ly.ncnt);
  uint16_t* L = (uint16_t*)(wsm + Ly.L);
  int* off = (int*)(wsm + Ly.off);
  int* cursor = (int*)(wsm + Ly.cursor);
  int* send = (int*)(wsm + Ly.send);
  int* D = (int*)(wsm + Ly.D);
  uint8_t* Q = wsm + Ly.Q;
  uint8_t* opened = wsm + Ly.opened;
  uint8_t* leaf = wsm + Ly.leaf;
  int* misc = (int*)(wsm + Ly.misc);
  int* gcnt = misc + FM_GCNT;
  int* gptr = misc + FM_GPTR;
  const bool want_sched = P.sched != nullptr && !(P.flags & FAR_NO_SCHEDULE);
  const bool refine = !(P.flags & FAR_NO_REFINE);
  for (int v = lane; v < NNF; v += 32) {
    const uint2 w = __ldg(F.nodes + v);
    if (fn_ch1(w) == FNONE) leaf[fn_lo(w)] = (uint8_t)v;
  }
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t inst = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; inst < P.I; inst += nw) {
    far_result R;
    memset(&R, 0, sizeof(R));
    __syncwarp();
    // ---- H0: runtime table -> smem, input checks
    const int32_t* gt = P.times + inst * (int64_t)n * NC;
    int bad = 0;
    long long mxs = 0;
    for (int j = lane; j < n; j += 32) {
      int mx = 0;
      for (int c = 0; c < NC; ++c) {
        const int t = __ldg(gt + j * NC + c);
        T[j * NC + c] = t;
        bad |= t < 1;
        mx = max(mx, t);
      }
      mxs += mx;
    }
    mxs = warp_sum_ll(mxs);
    if (__any_sync(FULL, bad) || mxs + P.rsum >= BOUND) {
      if (lane == 0) {
        R.makespan = -1;
        R.status = FAR_E_BAD_TIME;
        P.makespan[inst] = -1;
        if (P.res) P.res[inst] = R;
        atomicOr(P.errflag, 1);
      }
      continue;
    }
    if (n == 0) {
      if (lane == 0) {
        P.makespan[inst] = 0;
        if (P.res) P.res[inst] = R;
      }
      continue;
    }
    __syncwarp();
    int b2 = 0;  // buffer holding the phase-2 (best member's) record
    int ms2 = 0;
    long long pops = 0;
    if (P.mode == MODE_SOLVE) {
      // ---- phase 1a: a1_i = argmin_s (s * t_i(s), s)
      long long Wl = 0;
      for (int j = lane; j < n; j += 32) {
        int bc = 0;
        long long bw = (long long)size_of<NC>(0) * T[j * NC];
        for (int c = 1; c < NC; ++c) {
          const long long wv = (long long)size_of<NC>(c) * T[j * NC + c];
          if (wv < bw) { bw = wv; bc = c; }
        }
        cur[j] = (uint8_t)bc;
        Wl += bw;
      }
      long long W = warp_sum_ll(Wl);
      __syncwarp();
      // per-size LPT lists of a1 (Alg. 1 lines 1-2): rank by (-t, index)
      for (int c = 0; c < NC; ++c) {
        int cnt = 0;
        for (int j = lane; j < n; j += 32) cnt += cur[j] == c;
        cnt = __reduce_add_sync(FULL, cnt);
        if (lane == 0) gcnt[c] = cnt;
      }
      for (int j = lane; j < n; j += 32) {
        const int c = cur[j], tj = T[j * NC + c];
        int r = 0;
        for (int i = 0; i < n; ++i) {
          const int ti = T[i * NC + c];
          r += cur[i] == c && (ti > tj || (ti == tj && i < j));
        }
        glist[c * n + r] = (uint16_t)j;
      }
      __syncwarp();
      const bool exhaustive = (P.flags & FAR_EXHAUSTIVE) != 0, ties = (P.flags & FAR_GROW_TIES) != 0;
      int best = INT_MAX, bestk = 0, K = 0;
      for (;;) {
        // member K: longest task (ties -> lowest index) = h_K
        unsigned bt = 0, bj = UINT_MAX;
        for (int j = lane; j < n; j += 32) {
          const unsigned t = (unsigned)T[j * NC + cur[j]];
          if (t > bt) { bt = t; bj = j; }
        }
        const unsigned h = __reduce_max_sync(FULL, bt);
        const int jl = (int)__reduce_min_sync(FULL, bt == h ? bj : UINT_MAX);
        const long long lb = max((long long)h, (W + SF - 1) / SF);
        if (K == 0 || exhaustive || lb < best) {
          const int bb = b2 ^ 1;
          const int ms = forest_sim<NC, false>(F, n, T, glist, gcnt, gptr, L, off, cursor, cur,
                                               (int*)(wsm + Ly.rs[bb]), wsm + Ly.rn[bb], wsm + Ly.rp[bb],
                                               wsm + Ly.ru[bb], ncnt, pops, lane, wsm + Ly.isz);
          if (ms < best) { best = ms; bestk = K; b2 = bb; }
        }
        ++K;
        // growth: the longest task, or (FAR_GROW_TIES) every tied one
        unsigned grow;
        if (ties) {
          bool stuck = false;
          for (int j = lane; j < n; j += 32) stuck |= cur[j] == NC - 1 && (unsigned)T[j * NC + cur[j]] == h;
          if (__any_sync(FULL, stuck)) break;
          grow = 0;
        } else {
          if (cur[jl] == NC - 1) break;
        }
        for (int j0 = 0; j0 < n; j0 += 32) {
          const int jj = j0 + lane;
          grow = __ballot_sync(FULL, jj < n && (ties ? (unsigned)T[jj * NC + cur[jj]] == h : jj == jl));
          while (grow) {
            const int j = j0 + __ffs(grow) - 1;
            grow &= grow - 1;
            const int c = cur[j];
            int nc = -1;
            long long bw = 0;
            for (int c2 = c + 1; c2 < NC; ++c2) {
              const long long wv = (long long)size_of<NC>(c2) * T[j * NC + c2];
              if (nc < 0 || wv < bw) { bw = wv; nc = c2; }
            }
            W += bw - (long long)size_of<NC>(c) * T[j * NC + c];
            // ordered remove from list c, ordered insert into list nc (lists sorted by (-t, j))
            {
              const int cnt = gcnt[c];
              int p = 0;
              for (int b = 0; b < cnt; b += 32) {
                const unsigned m = __ballot_sync(FULL, b + lane < cnt && glist[c * n + b + lane] == j);
                if (m) { p = b + __ffs(m) - 1; break; }
              }
              for (int b = p; b < cnt - 1; b += 32) {
                const int i = b + lane;
                const uint16_t val = i < cnt - 1 ? glist[c * n + i + 1] : 0;
                __syncwarp();
                if (i < cnt - 1) glist[c * n + i] = val;
                __syncwarp();
              }
              const int cn = gcnt[nc], tj = T[j * NC + nc];
              int q = 0;
              for (int b = 0; b < cn; b += 32) {
                const int i = b + lane;
                bool bef = false;
                if (i < cn) {
                  const int y = glist[nc * n + i], ty = T[y * NC + nc];
                  bef = ty > tj || (ty == tj && y < j);
                }
                q += __popc(__ballot_sync(FULL, bef));
              }
              for (int top = cn - 1; top >= q; top -= 32) {
                const int i = top - lane;
                const uint16_t val = i >= q ? glist[nc * n + i] : 0;
                __syncwarp();
                if (i >= q) glist[nc * n + i + 1] = val;
                __syncwarp();
              }
              __syncwarp();  // every lane has read gcnt[] (the shift loop may not have run)
              if (lane == 0) {
                glist[nc * n + q] = (uint16_t)j;
                gcnt[c] = cnt - 1;
                gcnt[nc] = cn + 1;
                cur[j] = (uint8_t)nc;
              }
              __syncwarp();
            }
          }
        }
      }
      ms2 = best;
      R.alloc_index = bestk;
      R.family_size = K;
      R.events = pops;
    } else {
      // ---- MODE_LOCAL: the input schedule becomes the record (lists ordered by (start, task))
      const far_task_slot* in = P.sched_in + inst * (int64_t)n;
      int* rs = (int*)(wsm + Ly.rs[0]);
      uint8_t *rn = wsm + Ly.rn[0], *rp = wsm + Ly.rp[0], *ru = wsm + Ly.ru[0];
      int badin = 0, msIn = 0;
      for (int j = lane; j < n; j += 32) {
        const far_task_slot s = in[j];
        int c = -1;
        if (s.node < NNF) {
          const uint2 w = __ldg(F.nodes + s.node);
          if (size_of<NC>(fn_c0(w)) == s.size_used) c = fn_c0(w);
          else if (fn_c1(w) != NONE && size_of<NC>(fn_c1(w)) == s.size_used) c = fn_c1(w);
        }
        if (c < 0 || s.start < 0 || s.start > BOUND) { badin = 1; c = 0; }
        rn[j] = s.node < NNF ? s.node : 0;
        ru[j] = (uint8_t)c;
        rs[j] = s.start;
        msIn = max(msIn, s.start + T[j * NC + c]);
      }
      badin = __any_sync(FULL, badin);
      msIn = (int)__reduce_max_sync(FULL, (unsigned)msIn);
      if (badin) {
        if (lane == 0) {
          R.makespan = -1;
          R.status = FAR_E_INVALID_ARG;
          P.makespan[inst] = -1;
          if (P.res) P.res[inst] = R;
          atomicOr(P.errflag, 2);
        }
        continue;
      }
      __syncwarp();
      for (int j = lane; j < n; j += 32) {
        int pos = 0;
        for (int q = 0; q < n; ++q)
          pos += rn[q] == rn[j] && (rs[q] < rs[j] || (rs[q] == rs[j] && q < j));
        rp[j] = (uint8_t)pos;
      }
      const far_result rin = P.res_in ? P.res_in[inst] : R;
      R.alloc_index = rin.alloc_index;
      R.family_size = rin.family_size;
      R.events = rin.events;
      ms2 = (P.res_in && rin.makespan_phase2 > 0) ? rin.makespan_phase2 : msIn;
      b2 = 0;
    }
    R.makespan_phase2 = ms2;
    int* rs2 = (int*)(wsm + Ly.rs[b2]);
    uint8_t *rn2 = wsm + Ly.rn[b2], *rp2 = wsm + Ly.rp[b2], *ru2 = wsm + Ly.ru[b2];
    int outb = b2, msF = ms2;
    if (refine) {
      // ---- H6: Alg. 2 on the phase-2 tree (node lists concatenated in node-id order)
      for (int v = lane; v < NNF; v += 32) ncnt[v] = 0;
      for (int s = lane; s < SF; s += 32) send[s] = 0;
      __syncwarp();
      for (int j = lane; j < n; j += 32) {
        atomicAdd(&ncnt[rn2[j]], 1);
        D[j] = T[j * NC + ru2[j]];
        const uint2 w = __ldg(F.nodes + rn2[j]);
        for (int s = fn_lo(w); s < fn_lo(w) + fn_sz(w); ++s) atomicMax(&send[s], rs2[j] + D[j]);
      }
      __syncwarp();
      if (lane == 0) {
        int a = 0;
        for (int v = 0; v < NNF; ++v) { off[v] = a; a += ncnt[v]; }
        off[NNF] = a;
      }
      __syncwarp();
      for (int j = lane; j < n; j += 32) L[off[rn2[j]] + rp2[j]] = (uint16_t)j;
      __syncwarp();
      int mv, sw, it;
      long long ev;
      if (P.flags & FAR_BEST_IMPROVEMENT)
        forest_refine_best<NC>(F, n, D, L, off, send, wsm + Ly.tnode, (int2*)(wsm + Ly.srt), (int2*)(wsm + Ly.nstat),
                               lane, mv, sw, it, ev);
      else
        forest_refine<NC>(F, n, D, L, off, send, Q, opened, leaf, lane, mv, sw, it, ev);
      R.moves = mv; R.swaps = sw; R.iterations = it; R.evals = ev;
      // ---- H7: line-26 replay + keep-best guard
      const int ob = b2 ^ 1;
      long long rp_pops = 0;
      const int msR = forest_sim<NC, true>(F, n, T, glist, gcnt, gptr, L, off, cursor, ru2, (int*)(wsm + Ly.rs[ob]),
                                           wsm + Ly.rn[ob], wsm + Ly.rp[ob], wsm + Ly.ru[ob], ncnt, rp_pops, lane,
                                           wsm + Ly.isz);
      if (!(P.flags & FAR_NO_GUARD) && msR > ms2) {
        R.reverted = 1;
      } else {
        outb = ob;
        msF = msR;
      }
    }
    R.makespan = msF;
    if (want_sched) {
      const int* rs = (const int*)(wsm + Ly.rs[outb]);
      const uint8_t *rn = wsm + Ly.rn[outb], *ru = wsm + Ly.ru[outb];
      far_task_slot* out = P.sched + inst * (int64_t)n;
      for (int j = lane; j < n; j += 32) {
        far_task_slot s;
        s.node = rn[j];
        s.size_used = (uint8_t)size_of<NC>(ru[j]);
        s.pad[0] = s.pad[1] = 0;
        s.start = rs[j];
        out[j] = s;
      }
    }
    if (lane == 0) {
      P.makespan[inst] = R.makespan;
      if (P.res) P.res[inst] = R;
    }
    __syncwarp();
  }
}

}  // namespace farb
