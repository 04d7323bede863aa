// far_check.cuh — schedule export and checking on the GPU, one warp per
// instance:
//   far_events_kernel    node lists from a schedule -> line-26 replay -> the create
//                        events and the destroys issued while tasks remain (Alg. 1 l.8-11,
//                        l.17-20), sorted by start
//   far_validate_kernel  constraints 1-3 of the problem statement plus the
//                        reconfiguration lifecycle, as a violation count
// Same definitions as the oracle's orc_validate / event loop (oracle/far_oracle.cpp); the two
// share no code (tests/test_gpu_check.py compares them element by element).
#pragma once
#include "far_kernel.cuh"

namespace farb {

struct CParams {
  const int32_t* times;
  const far_task_slot* sched;
  int64_t I;
  int n;
  int cr[8], de[8];
  far_event* events;  // [I][2 * NN]
  int32_t* nev;       // [I]
  int32_t* makespan;  // [I] or null
  const far_event* events_in;
  const int32_t* nev_in;
  int32_t* violations;  // [I]
  unsigned long long* counter;
};

// per-warp shared memory of the events kernel
struct ELayout {
  int nlist, D, start, onode, su, sin, misc, bytes;
};
__host__ __device__ inline ELayout make_elayout(int n, int NN) {
  ELayout L;
  int o = 0;
  L.misc = o;  o = al16(o + 4 * M_END);
  L.nlist = o; o = al16(o + 2 * NN * n);
  L.D = o;     o = al16(o + 4 * n);
  L.start = o; o = al16(o + 4 * n);
  L.sin = o;   o = al16(o + 4 * n);
  L.onode = o; o = al16(o + n);
  L.su = o;    o = al16(o + n);
  L.bytes = o;
  return L;
}

template <int NC>
__device__ __forceinline__ int hosted_index(uint32_t w, int size) {
  if (size_of<NC>(nd_c0(w)) == size) return nd_c0(w);
  if (nd_c1(w) != NONE && size_of<NC>(nd_c1(w)) == size) return nd_c1(w);
  return -1;
}

template <int NC>
__global__ void __launch_bounds__(128) far_events_kernel(CParams P) {
  constexpr int NN = Tree<NC>::NN;
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = P.n;
  const ELayout L = make_elayout(n, NN);
  unsigned char* wsm = smem + (size_t)warp * L.bytes;
  int* misc = (int*)(wsm + L.misc);
  if (lane < 16) misc[M_NINFO + lane] = lane < NN ? (int)((NC == 3) ? c_nodes3[lane] : c_nodes5[lane]) : 0;
  if (lane < 8) {
    misc[M_CR + lane] = P.cr[lane];
    misc[M_DE + lane] = P.de[lane];
  }
  __syncwarp();
  const uint32_t* ninfo = (const uint32_t*)misc + M_NINFO;
  const int* cr = misc + M_CR;
  const int* de = misc + M_DE;
  int* ncnt = misc + M_NCNT;
  int* nsum = misc + M_NSUM;
  int* life = misc + M_LIFE;
  uint16_t* nlist = (uint16_t*)(wsm + L.nlist);
  int* D = (int*)(wsm + L.D);
  int* start = (int*)(wsm + L.start);
  int* sin = (int*)(wsm + L.sin);
  uint8_t* onode = wsm + L.onode;
  uint8_t* su = wsm + L.su;
  for (;;) {
    unsigned long long u = 0;
    if (lane == 0) u = atomicAdd(P.counter, 1ull);
    u = __shfl_sync(FULL, u, 0);
    const int64_t inst = (int64_t)u;
    if (inst >= P.I) break;
    const far_task_slot* in = P.sched + inst * (int64_t)n;
    const int32_t* t = P.times + inst * (int64_t)n * NC;
    int bad = 0;
    for (int j = lane; j < n; j += 32) {
      const far_task_slot sl = in[j];
      int c = -1;
      if (sl.node < NN) c = hosted_index<NC>(ninfo[sl.node], sl.size_used);
      if (c < 0) { bad = 1; c = 0; }
      onode[j] = sl.node < NN ? sl.node : 0;
      su[j] = (uint8_t)c;
      sin[j] = sl.start;
      D[j] = t[j * NC + c];
    }
    if (__any_sync(FULL, bad)) {
      if (lane == 0) {
        P.nev[inst] = -1;
        if (P.makespan) P.makespan[inst] = -1;
      }
      __syncwarp();
      continue;
    }
    __syncwarp();
    // node lists ordered by (start, task)
    for (int j = lane; j < n; j += 32) {
      const int v = onode[j], sj = sin[j];
      int pos = 0;
      for (int q = 0; q < n; ++q) pos += (onode[q] == v) && (sin[q] < sj || (sin[q] == sj && q < j));
      nlist[v * n + pos] = (uint16_t)j;
    }
    for (int v = 0; v < NN; ++v) {
      int c = 0;
      for (int j = lane; j < n; j += 32) c += (onode[j] == v);
      c = __reduce_add_sync(FULL, c);
      if (lane == 0) ncnt[v] = c;
    }
    __syncwarp();
    const int ms = replay_warp<NC>(n, D, nlist, ncnt, nsum, life, start, onode, ninfo, cr, de, lane);
    // the last placement pop of the replay (Alg. 1 l.7-16): a node's first task is taken at its
    // creation pop, the others at the end of the previous task; keys (time, first slice)
    unsigned lpk = 0;
    if (lane < NN && ncnt[lane] > 0) {
      const int c = ncnt[lane];
      const int tl = c >= 2 ? start[nlist[lane * n + c - 1]] : life[lane * 6 + 4];
      lpk = ((unsigned)tl << 3) | (unsigned)nd_lo(ninfo[lane]);
    }
    lpk = __reduce_max_sync(FULL, lpk);
    // events: lane v < NN holds node v's create (if any) and its destroy if it happened while
    // tasks remained unscheduled, i.e. at a pop key (end_v, lo_v) not after the last placement.
    // (Equal keys: v's first child is pushed by v's split with v's key and popped after it --
    // its creation pop takes its first task -- so a last placement with v's key comes later.)
    int kind0 = -1, kind1 = -1, s0 = 0, s1 = 0, d0 = 0, d1 = 0;
    if (lane < NN && life[lane * 6] >= 0) {
      const uint32_t w = ninfo[lane];
      kind0 = 0;
      s0 = life[lane * 6 + 0];
      d0 = cr[nd_szi(w)];
      const unsigned dk = ((unsigned)life[lane * 6 + 5] << 3) | (unsigned)nd_lo(w);
      if (life[lane * 6 + 2] >= 0 && dk <= lpk) {
        kind1 = 1;
        s1 = life[lane * 6 + 2];
        d1 = de[nd_szi(w)];
      }
    }
    // rank by start (events are disjoint in time; a zero-duration event at the same start as
    // another is ordered by (start, node, kind))
    const unsigned m0 = __ballot_sync(FULL, kind0 >= 0), m1 = __ballot_sync(FULL, kind1 >= 0);
    const int ne = __popc(m0) + __popc(m1);
    auto key_of = [](int s, int v, int k) { return ((unsigned long long)(unsigned)s << 8) | (unsigned)(v << 1) | k; };
    const unsigned long long k0 = kind0 >= 0 ? key_of(s0, lane, 0) : ~0ull;
    const unsigned long long k1 = kind1 >= 0 ? key_of(s1, lane, 1) : ~0ull;
    int r0 = 0, r1 = 0;
    for (int x = 0; x < NN; ++x) {
      const unsigned long long a = __shfl_sync(FULL, k0, x), b = __shfl_sync(FULL, k1, x);
      r0 += (a < k0) + (b < k0);
      r1 += (a < k1) + (b < k1);
    }
    far_event* out = P.events + inst * (int64_t)(2 * NN);
    if (kind0 >= 0) out[r0] = far_event{0, lane, s0, d0};
    if (kind1 >= 0) out[r1] = far_event{1, lane, s1, d1};
    if (lane == 0) {
      P.nev[inst] = ne;
      if (P.makespan) P.makespan[inst] = ms;
    }
    __syncwarp();
  }
}

// per-warp shared memory of the validator
struct VLayout {
  int b, f, node, cnt, bytes;
};
__host__ __device__ inline VLayout make_vlayout(int n, int NN) {
  VLayout L;
  int o = 0;
  L.b = o;    o = al16(o + 8 * n);
  L.f = o;    o = al16(o + 8 * n);
  L.node = o; o = al16(o + n);
  L.cnt = o;  o = al16(o + 2 * NN * 32);
  L.bytes = o;
  return L;
}

template <int NC>
__global__ void __launch_bounds__(128) far_validate_kernel(CParams P) {
  constexpr int NN = Tree<NC>::NN;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t ninfo[16];
  __shared__ int s_cr[8], s_de[8];
  if (threadIdx.x < 16) ninfo[threadIdx.x] = threadIdx.x < NN ? ((NC == 3) ? c_nodes3[threadIdx.x] : c_nodes5[threadIdx.x]) : 0;
  if (threadIdx.x < 8) {
    s_cr[threadIdx.x] = P.cr[threadIdx.x];
    s_de[threadIdx.x] = P.de[threadIdx.x];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = P.n;
  const VLayout L = make_vlayout(n, NN);
  unsigned char* wsm = smem + (size_t)warp * L.bytes;
  long long* b = (long long*)(wsm + L.b);
  long long* f = (long long*)(wsm + L.f);
  uint8_t* nd = wsm + L.node;
  uint16_t* cnt = (uint16_t*)(wsm + L.cnt);  // [NN][32] running tasks per node, per lane
  auto overlap = [&](int u, int v) {
    const uint32_t a = ninfo[u], c = ninfo[v];
    return nd_lo(a) < nd_lo(c) + nd_sz(c) && nd_lo(c) < nd_lo(a) + nd_sz(a);
  };
  for (;;) {
    unsigned long long uu = 0;
    if (lane == 0) uu = atomicAdd(P.counter, 1ull);
    uu = __shfl_sync(FULL, uu, 0);
    const int64_t inst = (int64_t)uu;
    if (inst >= P.I) break;
    const far_task_slot* in = P.sched + inst * (int64_t)n;
    const int32_t* t = P.times + inst * (int64_t)n * NC;
    // (0) slots
    int bad = 0;
    for (int j = lane; j < n; j += 32) {
      const far_task_slot sl = in[j];
      int c = -1;
      if (sl.node < NN) c = hosted_index<NC>(ninfo[sl.node], sl.size_used);
      if (c < 0) {
        bad++;
        nd[j] = 0;
        continue;
      }
      nd[j] = sl.node;
      b[j] = sl.start;
      f[j] = (long long)sl.start + t[j * NC + c];
      if (sl.start < 0) bad++;
    }
    bad = __reduce_add_sync(FULL, bad);
    if (bad) {
      if (lane == 0) P.violations[inst] = bad;
      __syncwarp();
      continue;
    }
    __syncwarp();
    long long v1 = 0;
    // (1) tasks on overlapping instances never run at the same time
    for (int i = lane; i < n; i += 32)
      for (int j = i + 1; j < n; ++j)
        v1 += overlap(nd[i], nd[j]) && b[i] < f[j] && b[j] < f[i];
    // (2) at every task start the running instances are pairwise disjoint nodes: pairs of
    //     running tasks on different overlapping nodes
    for (int k0 = 0; k0 < n; k0 += 32) {
      const int k = k0 + lane;
      for (int v = 0; v < NN; ++v) cnt[v * 32 + lane] = 0;
      if (k < n) {
        for (int j = 0; j < n; ++j)
          if (b[j] <= b[k] && b[k] < f[j]) cnt[nd[j] * 32 + lane]++;
        for (int u = 0; u < NN; ++u)
          for (int v = u + 1; v < NN; ++v)
            if (overlap(u, v)) v1 += (long long)cnt[u * 32 + lane] * cnt[v * 32 + lane];
      }
    }
    long long viol = (long long)warp_sum_ll(v1);
    // (3) events: one lane walks them in order (the last create / destroy of a node wins, as
    //     in the oracle), the per-node checks run on lanes over nodes
    const int ne = min(max(P.nev_in[inst], 0), 2 * NN);
    const far_event* ev = P.events_in + inst * (int64_t)(2 * NN);
    int ncr = 0, nds = 0;
    long long cst = 0, cen = 0, dst = LLONG_MAX, den = LLONG_MAX;
    long long first = LLONG_MAX, last = LLONG_MIN;
    bool used = false;
    if (lane < NN) {
      for (int j = 0; j < n; ++j)
        if (nd[j] == lane) {
          used = true;
          first = min(first, b[j]);
          last = max(last, f[j]);
        }
    }
    long long v3 = 0;
    for (int e = 0; e < ne; ++e) {
      const far_event E = ev[e];
      const bool ok = E.node >= 0 && E.node < NN;
      if (!ok) {
        v3 += lane == 0;
        continue;
      }
      const uint32_t w = ninfo[E.node];
      const int want = E.kind == 0 ? s_cr[nd_szi(w)] : s_de[nd_szi(w)];
      if (lane == 0 && (E.dur != want || E.start < 0)) v3++;
      if (lane == E.node) {
        if (E.kind == 0) { ncr++; cst = E.start; cen = (long long)E.start + E.dur; }
        else { nds++; dst = E.start; den = (long long)E.start + E.dur; }
      }
      // pairwise disjoint in time: lanes over the later events
      for (int g = e + 1 + lane; g < ne; g += 32) {
        const far_event G = ev[g];
        v3 += (long long)E.start < (long long)G.start + G.dur && (long long)G.start < (long long)E.start + E.dur;
      }
    }
    if (lane < NN) {
      if (!used) {
        if (ncr || nds) v3++;
      } else if (ncr != 1 || nds > 1) {
        v3++;
      } else {
        if (cen > first) v3++;
        if (nds && dst < last) v3++;
      }
    }
    // lifecycles of overlapping used nodes: the earlier-created one is destroyed before the
    // other is created
    {
      const unsigned umask = __ballot_sync(FULL, lane < NN && used);
      for (int u = 0; u < NN; ++u) {
        const long long cu = __shfl_sync(FULL, cst, u), du = __shfl_sync(FULL, den, u);
        const int nu = __shfl_sync(FULL, nds, u);
        if (lane < NN && lane > u && ((umask >> u) & 1) && used && overlap(u, lane)) {
          const bool u_first = cu < cst;
          const long long dend_a = u_first ? du : den;
          const int nd_a = u_first ? nu : nds;
          const long long cstart_c = u_first ? cst : cu;
          if (nd_a == 0 || dend_a > cstart_c) v3++;
        }
      }
    }
    viol += warp_sum_ll(v3);
    if (lane == 0) P.violations[inst] = (int32_t)min(viol, (long long)INT_MAX);
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Lower bound of the optimal makespan: baseline = sum_i min_s s * t_i(s) / #slices
// and max_i min_s t_i(s); one thread per instance (the evaluation metric rho = omega / baseline of
// Tables 4 and 9).
// ---------------------------------------------------------------------------
template <int NC>
__global__ void __launch_bounds__(256) far_lower_bound_kernel(const int32_t* __restrict__ times, int64_t I, int n,
                                                              long long* sum_min_work, int32_t* max_min_time) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < I; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t* t = times + i * (int64_t)n * NC;
    long long W = 0;
    int H = 0;
    for (int j = 0; j < n; ++j) {
      long long w = LLONG_MAX;
      int h = INT_MAX;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int x = __ldg(t + j * NC + c);
        w = min(w, (long long)size_of<NC>(c) * x);
        h = min(h, x);
      }
      W += w;
      H = max(H, h);
    }
    sum_min_work[i] = W;
    if (max_min_time) max_min_time[i] = H;
  }
}

}  // namespace farb
