// far_stream.cuh — §4 multi-batch concatenation, one WARP per stream.
//
// Every batch of every stream is first FAR-scheduled by far_solve_kernel (phases 1-3,
// data-parallel over S*B instances).  This kernel then folds each stream left to right:
//   - full-lifecycle timeline of the batch tree (creates, tasks, a destroy for every
//     instance), reversed for odd batches: the loop runs with t_create<->t_destroy
//     swapped and is mirrored about its last event end;
//   - seam offset: least O >= previous offset with per-slice disjoint lifecycles,
//     reuse of an identical boundary instance (its destroy/create pair elided), and
//     no overlap of reconfiguration events (sequential reconfiguration);
//   - seam move/swap on reversed batches: Alg. 2's candidates with the
//     inter-batch idle time as the margin, each evaluated by recomputing timeline + offset
//     and kept only if the batch ends earlier.
// Readings R21-R25; identical to oracle/far_oracle.cpp (no shared code).
#pragma once
#include "far_kernel.cuh"

namespace farb {

constexpr int WCAP = 256;  // placed-event window per stream (events ending after the last offset)
constexpr long long LL_MAX = 0x7fffffffffffffffLL;

struct SParams {
  const int32_t* times;          // [S][B][n][NC]
  const far_task_slot* sched;    // [S][B][n]  FAR schedules (forward, relative)
  int64_t S;
  int B, n;
  int cr[8], de[8];
  int max_it;
  int seam_moves;                // 0: FAR_NO_SEAM_MOVES
  int64_t* stream_ms;            // [S][2]
  int64_t* offsets;              // [S][B]
  far_task_slot* out_sched;      // [S][B][n] or null
  int32_t* seam;                 // [S][B][4] or null
  int* errflag;
};

struct SLayout {
  int times, su, onode, nl, nl2, ncnt, ncnt2, nsum, start, fstart, dur, life, win, misc, bytes;
};

__host__ __device__ inline SLayout make_slayout(int n, int NC, int NN) {
  SLayout L;
  int o = 0;
  L.times = o;  o = al16(o + 4 * n * NC);
  L.su = o;     o = al16(o + n);
  L.onode = o;  o = al16(o + n);
  L.nl = o;     o = al16(o + 2 * NN * n);
  L.nl2 = o;    o = al16(o + 2 * NN * n);
  L.ncnt = o;   o = al16(o + 4 * 16);
  L.ncnt2 = o;  o = al16(o + 4 * 16);
  L.nsum = o;   o = al16(o + 4 * 16);
  L.start = o;  o = al16(o + 4 * n);
  L.fstart = o; o = al16(o + 4 * n);
  L.dur = o;    o = al16(o + 4 * n);
  L.life = o;   o = al16(o + 4 * 16 * 6 + 32 + 64);  // + eval_seam's per-slice scratch
  L.win = o;    o = al16(o + WCAP * 24);
  L.misc = o;   o = al16(o + 8 * 64);
  L.bytes = o;
  return L;
}

struct WinEv {
  long long s, e;
  int id, alive;
};

__device__ __forceinline__ long long warp_max_ll(long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, (long long)__shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ long long warp_min_ll(long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = min(v, (long long)__shfl_xor_sync(FULL, v, o));
  return v;
}

// The full-lifecycle timeline of a batch (R22) is the node-level replay of far_kernel.cuh:
// node_sim charges a destroy for every node with tasks at its SPLIT key, which is exactly
// the O7 loop extended with a destroy at drop time.

// Per-stream fold state (shared memory, misc region)
struct StreamSt {
  long long tail[8];        // end of the last lifecycle on each slice (0 = none)
  long long tail_lt[8];     // last task end of that lifecycle
  int tail_node[8];         // its node (-1 = none)
  int tail_dev[8];          // id of its destroy event
  long long last_off;
  int nwin, next_id, overflow;
};

// Result of one timeline + seam evaluation (uniform across lanes)
struct SeamRes {
  long long O, end;
  long long gap[8];
  unsigned reuse;     // bit v: node v reuses the boundary instance
  unsigned touched;   // bit s: slice used by the batch
  int E, task_end;
};

// Timeline of the batch described by (nl, ncnt) + its seam against the stream state.
template <int NC>
__device__ __noinline__ SeamRes eval_seam(int n, const int32_t* T, const uint8_t* su, const int* D, const uint16_t* nl,
                             const int* ncnt, int* nsum, uint8_t* onode, int* start, int* life, const uint32_t* ninfo,
                             const int* cr, const int* de, bool rev, const StreamSt* st, const WinEv* win, int lane) {
  constexpr int S = Tree<NC>::S, NN = Tree<NC>::NN;
  int E = 0;
  replay_warp<NC>(n, D, nl, ncnt, nsum, life, start, onode, ninfo, rev ? de : cr, rev ? cr : de, lane, &E);
  if (rev) {  // mirror about E: tasks and lifecycles (a mirrored forward destroy is the create)
    for (int j = lane; j < n; j += 32) start[j] = E - (start[j] + T[j * NC + su[j]]);
    if (lane < NN && life[lane * 6] >= 0) {
      const int cs = life[lane * 6 + 0], ce = life[lane * 6 + 1], ds = life[lane * 6 + 2], dd = life[lane * 6 + 3];
      life[lane * 6 + 0] = E - dd;
      life[lane * 6 + 1] = E - ds;
      life[lane * 6 + 2] = E - ce;
      life[lane * 6 + 3] = E - cs;
    }
    __syncwarp();
  }
  // first task start / last task end per node; batch task end
  int tend = 0;
  for (int v = 0; v < NN; ++v) {
    if (ncnt[v] == 0) continue;
    int ft = INT_MAX, lt = INT_MIN;
    for (int q = lane; q < ncnt[v]; q += 32) {
      const int j = nl[v * n + q];
      ft = min(ft, start[j]);
      lt = max(lt, start[j] + T[j * NC + su[j]]);
    }
    ft = __reduce_min_sync(FULL, ft);
    lt = __reduce_max_sync(FULL, lt);
    if (lane == 0) {
      life[v * 6 + 4] = ft;
      life[v * 6 + 5] = lt;
    }
    tend = max(tend, lt);
  }
  __syncwarp();
  SeamRes R;
  R.E = E;
  R.task_end = tend;
  if (NC == 3) {  // the A30 tree (4 slices, 7 nodes): per-slice registers are cheaper
    // first lifecycle on each slice; reuse (R23 ii)
    int first[S];
    unsigned touched = 0;
#pragma unroll
    for (int s = 0; s < S; ++s) first[s] = -1;
    for (int v = 0; v < NN; ++v) {
      if (ncnt[v] == 0) continue;
      const uint32_t w = ninfo[v];
#pragma unroll
      for (int s = 0; s < S; ++s)
        if (s >= nd_lo(w) && s < nd_lo(w) + nd_sz(w)) {
          touched |= 1u << s;
          if (first[s] < 0 || life[v * 6] < life[first[s] * 6]) first[s] = v;
        }
    }
    unsigned reuse = 0;
    for (int v = 0; v < NN; ++v) {
      if (ncnt[v] == 0) continue;
      const uint32_t w = ninfo[v];
      bool ok = true;
#pragma unroll
      for (int s = 0; s < S; ++s)
        if (s >= nd_lo(w) && s < nd_lo(w) + nd_sz(w)) ok = ok && first[s] == v && st->tail_node[s] == v;
      if (ok) reuse |= 1u << v;
    }
    long long bound[S];
    long long O = max(st->last_off, 0LL);
#pragma unroll
    for (int s = 0; s < S; ++s) {
      bound[s] = 0;
      if (first[s] >= 0) {
        const int v = first[s];
        bound[s] = ((reuse >> v) & 1) ? st->tail_lt[s] - life[v * 6 + 4] : st->tail[s] - life[v * 6 + 0];
        O = max(O, bound[s]);
      }
    }
    // (iii) sequential reconfiguration against the placed window
    unsigned skipmask_dev[8];
#pragma unroll
    for (int s = 0; s < S; ++s) skipmask_dev[s] = (first[s] >= 0 && ((reuse >> first[s]) & 1)) ? 1u : 0u;
    for (;;) {
      long long push = O;
      for (int p = lane; p < st->nwin; p += 32) {
        const WinEv ev = win[p];
        if (!ev.alive) continue;
        bool skip = false;
#pragma unroll
        for (int s = 0; s < S; ++s) skip = skip || (skipmask_dev[s] && st->tail_dev[s] == ev.id);
        if (skip) continue;
        for (int v = 0; v < NN; ++v) {
          if (ncnt[v] == 0) continue;
          if (!((reuse >> v) & 1)) {
            const long long a = life[v * 6 + 0], b = life[v * 6 + 1];
            if (a + O < ev.e && ev.s < b + O) push = max(push, ev.e - a);
          }
          const long long a = life[v * 6 + 2], b = life[v * 6 + 3];
          if (a + O < ev.e && ev.s < b + O) push = max(push, ev.e - a);
        }
      }
      push = warp_max_ll(push);
      if (push == O) break;
      O = push;
    }
    R.O = O;
    R.end = O + E;
    R.reuse = reuse;
    R.touched = touched;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const long long g = first[s] >= 0 ? O - bound[s] : O + E - st->tail[s];
      R.gap[s] = max(g, 0LL);
    }
    return R;
  } else {
    // first lifecycle on each slice (lane s < S), reuse (R23 ii; lane v < NN), offset bound per slice
    //   -- lane-parallel instead of per-slice register arrays: a much smaller kernel body
    int* firsts = life + 16 * 6;  // scratch after the lifecycle table (make_slayout reserves it)
    long long* skipid = (long long*)(firsts + 8);
    int fs = -1;
    if (lane < S) {
      for (int v = 0; v < NN; ++v) {
        const uint32_t w = ninfo[v];
        if (ncnt[v] > 0 && lane >= nd_lo(w) && lane < nd_lo(w) + nd_sz(w) && (fs < 0 || life[v * 6] < life[fs * 6]))
          fs = v;
      }
      firsts[lane] = fs;
    }
    const unsigned touched = __ballot_sync(FULL, lane < S && fs >= 0);
    __syncwarp();
    bool ok = lane < NN && ncnt[lane] > 0;
    if (ok) {
      const uint32_t w = ninfo[lane];
      for (int q = nd_lo(w); q < nd_lo(w) + nd_sz(w); ++q) ok = ok && firsts[q] == lane && st->tail_node[q] == lane;
    }
    const unsigned reuse = __ballot_sync(FULL, ok);
    long long bnd = 0;
    long long O = max(st->last_off, 0LL);
    if (lane < S) {
      if (fs >= 0) {
        bnd = ((reuse >> fs) & 1) ? st->tail_lt[lane] - life[fs * 6 + 4] : st->tail[lane] - life[fs * 6 + 0];
        O = max(O, bnd);
      }
      // (iii) the destroy event of a reused boundary instance is elided: skip it below
      skipid[lane] = (fs >= 0 && ((reuse >> fs) & 1)) ? (long long)st->tail_dev[lane] : -2;
    }
    O = warp_max_ll(O);
    __syncwarp();
    // (iii) sequential reconfiguration against the placed window
    for (;;) {
      long long push = O;
      for (int p = lane; p < st->nwin; p += 32) {
        const WinEv ev = win[p];
        if (!ev.alive) continue;
        bool skip = false;
#pragma unroll
        for (int q = 0; q < S; ++q) skip = skip || skipid[q] == (long long)ev.id;
        if (skip) continue;
        for (int v = 0; v < NN; ++v) {
          if (ncnt[v] == 0) continue;
          if (!((reuse >> v) & 1)) {
            const long long a = life[v * 6 + 0], b = life[v * 6 + 1];
            if (a + O < ev.e && ev.s < b + O) push = max(push, ev.e - a);
          }
          const long long a = life[v * 6 + 2], b = life[v * 6 + 3];
          if (a + O < ev.e && ev.s < b + O) push = max(push, ev.e - a);
        }
      }
      push = warp_max_ll(push);
      if (push == O) break;
      O = push;
    }
    const long long gl = lane < S ? max(fs >= 0 ? O - bnd : O + E - st->tail[lane], 0LL) : 0LL;
#pragma unroll
    for (int q = 0; q < S; ++q) R.gap[q] = __shfl_sync(FULL, gl, q);
    R.O = O;
    R.end = O + E;
    R.reuse = reuse;
    R.touched = touched;
    return R;
  }
}

// Move task k from node I to node A and (swap) task j from A to I, keeping lists ordered.
template <int NC>
__device__ __noinline__ void transfer(int n, uint16_t* nl, int* ncnt, int I, int A, int k, int j, const int* D,
                                      int lane) {
  for (int x = 0; x < (j >= 0 ? 2 : 1); ++x) {
    const int from = x == 0 ? I : A, to = x == 0 ? A : I, task = x == 0 ? k : j;
    list_remove<NC>(nl + from * n, &ncnt[from], task, lane);
    list_insert<NC>(nl + to * n, &ncnt[to], task, D, lane);
  }
}

template <int NC>
__device__ void copy_lists(int n, const uint16_t* a, const int* ca, uint16_t* b, int* cb, int lane) {
  constexpr int NN = Tree<NC>::NN;
  for (int q = lane; q < NN * n; q += 32) b[q] = a[q];
  if (lane < NN) cb[lane] = ca[lane];
  __syncwarp();
}

template <int NC>
__global__ void __launch_bounds__(128) far_stream_kernel(SParams P) {
  constexpr int S = Tree<NC>::S, NN = Tree<NC>::NN;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t ninfo[16];
  __shared__ int cr[8], de[8];
  if (threadIdx.x < NN) ninfo[threadIdx.x] = (NC == 3) ? c_nodes3[threadIdx.x] : c_nodes5[threadIdx.x];
  if (threadIdx.x < 8) {
    cr[threadIdx.x] = P.cr[threadIdx.x];
    de[threadIdx.x] = P.de[threadIdx.x];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t sid = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (sid >= P.S) return;
  const int n = P.n, B = P.B;
  const SLayout L = make_slayout(n, NC, NN);
  unsigned char* wsm = smem + (size_t)(threadIdx.x >> 5) * L.bytes;
  int32_t* T = (int32_t*)(wsm + L.times);
  uint8_t* su = wsm + L.su;
  uint16_t* nl = (uint16_t*)(wsm + L.nl);
  uint16_t* nl2 = (uint16_t*)(wsm + L.nl2);
  int* ncnt = (int*)(wsm + L.ncnt);
  int* ncnt2 = (int*)(wsm + L.ncnt2);
  int* nsum = (int*)(wsm + L.nsum);
  uint8_t* onode = wsm + L.onode;
  int* start = (int*)(wsm + L.start);
  int* fstart = (int*)(wsm + L.fstart);
  int* D = (int*)(wsm + L.dur);
  int* life = (int*)(wsm + L.life);
  WinEv* win = (WinEv*)(wsm + L.win);
  StreamSt* st = (StreamSt*)(wsm + L.misc);
  if (lane == 0) {
    for (int s = 0; s < 8; ++s) {
      st->tail[s] = 0;
      st->tail_lt[s] = 0;
      st->tail_node[s] = -1;
      st->tail_dev[s] = -1;
    }
    st->last_off = 0;
    st->nwin = 0;
    st->next_id = 0;
    st->overflow = 0;
  }
  __syncwarp();
  long long ms = 0, triv_ms = 0, prev_end = 0;
  for (int k = 0; k < B; ++k) {
    const int64_t bi = sid * B + k;
    // ---- load the batch table and its FAR schedule; node lists ordered by (start, task)
    const int32_t* src = P.times + bi * (int64_t)n * NC;
    for (int q = lane; q < n * NC; q += 32) T[q] = __ldg(src + q);
    __syncwarp();  // T is read below at other lanes' indices
    const far_task_slot* fs = P.sched + bi * (int64_t)n;
    for (int j = lane; j < n; j += 32) {
      const far_task_slot s = fs[j];
      const uint32_t w = ninfo[s.node];
      su[j] = (uint8_t)(size_of<NC>(nd_c0(w)) == s.size_used ? nd_c0(w) : nd_c1(w));
      fstart[j] = s.start;
      start[j] = s.node;  // temporarily: node per task
      D[j] = T[j * NC + su[j]];
    }
    __syncwarp();
    // node lists ordered by (start, task): the tasks grouped by node with ballots (into nl2, free
    // until the seam refinement; group offsets in nsum, rewritten by the replay), then each task
    // ranked among its node's few tasks
    {
      const unsigned lt = (1u << lane) - 1u;
      int goff = 0;
      for (int v = 0; v < NN; ++v) {
        int c = 0;
        for (int j0 = 0; j0 < n; j0 += 32) {
          const int j = j0 + lane;
          const bool in = j < n && start[j] == v;
          const unsigned b = __ballot_sync(FULL, in);
          if (in) nl2[goff + c + __popc(b & lt)] = (uint16_t)j;
          c += __popc(b);
        }
        if (lane == 0) {
          ncnt[v] = c;
          nsum[v] = goff;
        }
        goff += c;
      }
      __syncwarp();
      for (int j = lane; j < n; j += 32) {
        const int v = start[j], sj = fstart[j];
        const int b = nsum[v], c = ncnt[v];
        int pos = 0;
        for (int q = 0; q < c; ++q) {
          const int x = nl2[b + q];
          pos += fstart[x] < sj || (fstart[x] == sj && x < j);
        }
        nl[v * n + pos] = (uint16_t)j;
      }
    }
    __syncwarp();
    // ---- trivial concatenation: forward timeline, right after all previous activity
    {
      SeamRes fr;
      StreamSt dummy;
      (void)dummy;
      int E = 0;
      replay_warp<NC>(n, D, nl, ncnt, nsum, life, start, onode, ninfo, cr, de, lane, &E);
      int te = 0;
      for (int j = lane; j < n; j += 32) te = max(te, start[j] + T[j * NC + su[j]]);
      te = __reduce_max_sync(FULL, te);
      const long long O = k == 0 ? 0 : prev_end;
      triv_ms = max(triv_ms, O + te);
      prev_end = O + E;
      (void)fr;
    }
    const bool rev = (k & 1) == 1;
    int moves = 0, swaps = 0;
    // ---- seam move/swap on reversed batches (R24)
    if (rev && k > 0 && P.seam_moves) {
      SeamRes cur = eval_seam<NC>(n, T, su, D, nl, ncnt, nsum, onode, start, life, ninfo, cr, de, true, st, win, lane);
      for (int it = 0; it < P.max_it; ++it) {
        unsigned long long Q = 0;
        int qh = 0, qt = 0;
        uint32_t opened = 0;
        for (int s = 0; s < S; ++s)
          if (((cur.touched >> s) & 1) && cur.gap[s] == 0) {
            const int leaf = leaf_of<NC>(s);
            Q |= (unsigned long long)leaf << (4 * qt++);
            opened |= 1u << leaf;
          }
        if (qt == 0) break;
        bool accepted = false, stop = false;
        while (qh < qt && !accepted) {
          const int I = (int)((Q >> (4 * qh++)) & 15);
          if (I == 0) { stop = true; break; }
          const uint32_t wI = ninfo[I];
          int A = -1;
          long long sA = 0;
          for (int u = 0; u < NN; ++u) {
            const uint32_t wu = ninfo[u];
            if (u == I || nd_sz(wu) != nd_sz(wI)) continue;
            long long g = LL_MAX;
            for (int s = nd_lo(wu); s < nd_lo(wu) + nd_sz(wu); ++s) g = min(g, cur.gap[s]);
            if (A < 0 || g > sA) { A = u; sA = g; }
          }
          if (A >= 0 && sA > 0) {
            const long long m = sA;
            const int nI = ncnt[I];
            // move candidate: argmin (|2t - m|, task) over t < m
            long long bd = LL_MAX;
            int bj = INT_MAX;
            for (int q = lane; q < nI; q += 32) {
              const int j = nl[I * n + q];
              const long long t = T[j * NC + su[j]];
              if (t < m) {
                const long long d = llabs(2 * t - m);
                if (d < bd || (d == bd && j < bj)) { bd = d; bj = j; }
              }
            }
            const long long dmin = warp_min_ll(bd);
            if (dmin != LL_MAX) {
              const int Tm = (int)__reduce_min_sync(FULL, (unsigned)(bd == dmin ? bj : INT_MAX));
              copy_lists<NC>(n, nl, ncnt, nl2, ncnt2, lane);
              transfer<NC>(n, nl2, ncnt2, I, A, Tm, -1, D, lane);
              SeamRes e2 = eval_seam<NC>(n, T, su, D, nl2, ncnt2, nsum, onode, start, life, ninfo, cr, de, true, st, win, lane);
              if (e2.end < cur.end) {
                copy_lists<NC>(n, nl2, ncnt2, nl, ncnt, lane);
                cur = e2;
                ++moves;
                accepted = true;
              }
            }
            if (!accepted) {
              const int nA = ncnt[A];
              long long bd2 = LL_MAX;
              unsigned bkey = UINT_MAX;
              for (int p = lane; p < nI * nA; p += 32) {
                const int qi = p / nA, qa = p - qi * nA;
                const int kk = nl[I * n + qi], jj = nl[A * n + qa];
                const long long dl = (long long)T[kk * NC + su[kk]] - T[jj * NC + su[jj]];
                if (0 < dl && dl < m) {
                  const long long d = llabs(2 * dl - m);
                  const unsigned key = ((unsigned)kk << 10) | (unsigned)jj;
                  if (d < bd2 || (d == bd2 && key < bkey)) { bd2 = d; bkey = key; }
                }
              }
              const long long d2 = warp_min_ll(bd2);
              if (d2 != LL_MAX) {
                const unsigned key = __reduce_min_sync(FULL, bd2 == d2 ? bkey : UINT_MAX);
                const int kk = (int)(key >> 10), jj = (int)(key & 1023);
                copy_lists<NC>(n, nl, ncnt, nl2, ncnt2, lane);
                transfer<NC>(n, nl2, ncnt2, I, A, kk, jj, D, lane);
                SeamRes e2 = eval_seam<NC>(n, T, su, D, nl2, ncnt2, nsum, onode, start, life, ninfo, cr, de, true, st, win, lane);
                if (e2.end < cur.end) {
                  copy_lists<NC>(n, nl2, ncnt2, nl, ncnt, lane);
                  cur = e2;
                  ++swaps;
                  accepted = true;
                }
              }
            }
          }
          if (!accepted) {
            const int par = nd_par(wI);
            if (par != ROOTP && !((opened >> par) & 1)) {
              opened |= 1u << par;
              Q |= (unsigned long long)par << (4 * qt++);
            }
          }
        }
        if (stop || !accepted) break;
      }
    }
    // ---- final timeline + seam of the (refined) batch; place it
    const SeamRes R = eval_seam<NC>(n, T, su, D, nl, ncnt, nsum, onode, start, life, ninfo, cr, de, rev, st, win, lane);
    const long long O = R.O;
    ms = max(ms, O + R.task_end);
    __syncwarp();  // every lane's reads of the stream state (eval_seam) precede lane 0's update
    if (lane == 0) {
      // elide the destroys of reused boundary instances
      for (int s = 0; s < S; ++s) {
        const int v = st->tail_node[s];
        if (v >= 0 && ((R.reuse >> v) & 1))
          for (int p = 0; p < st->nwin; ++p)
            if (win[p].id == st->tail_dev[s]) win[p].alive = 0;
      }
      int dev_id[16];
      for (int v = 0; v < NN; ++v) {
        dev_id[v] = -1;
        if (ncnt[v] == 0) continue;
        if (!((R.reuse >> v) & 1)) {
          if (st->nwin < WCAP) win[st->nwin++] = WinEv{O + life[v * 6 + 0], O + life[v * 6 + 1], st->next_id, 1};
          else st->overflow = 1;
          st->next_id++;
        }
        dev_id[v] = st->next_id;
        if (st->nwin < WCAP) win[st->nwin++] = WinEv{O + life[v * 6 + 2], O + life[v * 6 + 3], st->next_id, 1};
        else st->overflow = 1;
        st->next_id++;
      }
      for (int s = 0; s < S; ++s) {
        int best = -1;
        for (int v = 0; v < NN; ++v) {
          if (ncnt[v] == 0) continue;
          const uint32_t w = ninfo[v];
          if (s >= nd_lo(w) && s < nd_lo(w) + nd_sz(w) && (best < 0 || life[v * 6 + 3] > life[best * 6 + 3])) best = v;
        }
        if (best >= 0) {
          st->tail[s] = O + life[best * 6 + 3];
          st->tail_lt[s] = O + life[best * 6 + 5];
          st->tail_node[s] = best;
          st->tail_dev[s] = dev_id[best];
        }
      }
      st->last_off = O;
      // prune events that cannot overlap later batches (they start at >= O)
      int w2 = 0;
      for (int p = 0; p < st->nwin; ++p)
        if (win[p].alive && win[p].e > O) win[w2++] = win[p];
      st->nwin = w2;
    }
    __syncwarp();
    if (P.offsets && lane == 0) P.offsets[bi] = O;
    if (P.seam && lane == 0) {
      int reused = __popc(R.reuse);
      P.seam[bi * 4 + 0] = rev;
      P.seam[bi * 4 + 1] = moves;
      P.seam[bi * 4 + 2] = swaps;
      P.seam[bi * 4 + 3] = reused;
    }
    if (P.out_sched) {
      // node per task from the lists
      for (int v = 0; v < NN; ++v)
        for (int q = lane; q < ncnt[v]; q += 32) {
          const int j = nl[v * n + q];
          far_task_slot s;
          s.node = (uint8_t)v;
          s.size_used = (uint8_t)size_of<NC>(su[j]);
          s.pad[0] = s.pad[1] = 0;
          s.start = start[j];
          P.out_sched[bi * (int64_t)n + j] = s;
        }
    }
    __syncwarp();
  }
  if (lane == 0) {
    P.stream_ms[sid * 2 + 0] = ms;
    P.stream_ms[sid * 2 + 1] = triv_ms;
    if (st->overflow) atomicOr(P.errflag, 4);
  }
}

}  // namespace farb
