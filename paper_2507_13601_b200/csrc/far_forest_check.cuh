// far_forest_check.cuh — reconfiguration events and the feasibility validator (SURVEY.md §8(f)
// NEXT-4) for multi-target contexts (NEXT-2: g trees, one heap, one reconfiguration
// sequence), one warp per instance over the generic forest node table of far_forest.cuh.
//   far_forest_events_kernel    node lists from a schedule, ordered by (start, task) -> the
//                               line-26 replay over the forest (forest_sim)
//                               recording its creates and the destroys issued while tasks remain
//   far_forest_validate_kernel  the conditions of far_validate_kernel (P:214-230 + lifecycles)
//                               over the forest's nodes and slices, as a violation count
// Same definitions as the oracle's orc_far events / orc_validate on profile | g << 8; the two
// share no code (tests/test_gpu_forest.py compares them element by element).
#pragma once
#include "far_check.cuh"
#include "far_forest.cuh"

namespace farb {

struct FCParams {
  FParams F;   // F.P: costs and flags; F.nodes, F.NNF, F.SF: the forest
  CParams Q;   // schedules, events, outputs, counter
};

struct FELayout {
  int T, su, onode, sin, L, off, cursor, ncnt, rs, rn, rp, ru, isz, bytes;
};
__host__ __device__ inline FELayout make_felayout(int n, int NC, int NNF) {
  FELayout L;
  int o = 0;
  auto take = [&](int b) { const int r = o; o = al16(o + b); return r; };
  L.T = take(4 * n * NC);
  L.su = take(n);
  L.onode = take(n);
  L.sin = take(4 * n);
  L.L = take(2 * n + 2);
  L.off = take(4 * (NNF + 1));
  L.cursor = take(4 * NNF);
  L.ncnt = take(4 * NNF);
  L.rs = take(4 * n);
  L.rn = take(n);
  L.rp = take(n);
  L.ru = take(n);
  L.isz = take(NNF);
  L.bytes = o;
  return L;
}

// size index of `size` on forest node w, -1 if w does not host it
template <int NC>
__device__ __forceinline__ int fhosted(uint2 w, int size) {
  if (size_of<NC>(fn_c0(w)) == size) return fn_c0(w);
  if (fn_c1(w) != NONE && size_of<NC>(fn_c1(w)) == size) return fn_c1(w);
  return -1;
}

template <int NC>
__global__ void __launch_bounds__(128) far_forest_events_kernel(FCParams C) {
  extern __shared__ __align__(16) unsigned char smem[];
  const FParams& F = C.F;
  const CParams& P = C.Q;
  const int NNF = F.NNF, n = P.n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const FELayout L = make_felayout(n, NC, NNF);
  unsigned char* wsm = smem + (size_t)warp * L.bytes;
  int32_t* T = (int32_t*)(wsm + L.T);
  uint8_t* su = wsm + L.su;
  uint8_t* onode = wsm + L.onode;
  int* sin = (int*)(wsm + L.sin);
  uint16_t* lst = (uint16_t*)(wsm + L.L);
  int* off = (int*)(wsm + L.off);
  int* cursor = (int*)(wsm + L.cursor);
  int* ncnt = (int*)(wsm + L.ncnt);
  for (;;) {
    unsigned long long u = 0;
    if (lane == 0) u = atomicAdd(P.counter, 1ull);
    const int64_t inst = (int64_t)__shfl_sync(FULL, u, 0);
    if (inst >= P.I) break;
    const far_task_slot* in = P.sched + inst * (int64_t)n;
    const int32_t* t = P.times + inst * (int64_t)n * NC;
    for (int q = lane; q < n * NC; q += 32) T[q] = __ldg(t + q);
    int bad = 0;
    for (int j = lane; j < n; j += 32) {
      const far_task_slot sl = in[j];
      int c = -1;
      if (sl.node < NNF) c = fhosted<NC>(__ldg(F.nodes + sl.node), sl.size_used);
      if (c < 0) { bad = 1; c = 0; }
      onode[j] = sl.node < NNF ? sl.node : 0;
      su[j] = (uint8_t)c;
      sin[j] = sl.start;
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
    // node lists ordered by (start, task), concatenated in node-id order
    for (int v = lane; v < NNF; v += 32) {
      int c = 0;
      for (int j = 0; j < n; ++j) c += onode[j] == v;
      ncnt[v] = c;
    }
    __syncwarp();
    if (lane == 0) {
      int acc = 0;
      for (int v = 0; v < NNF; ++v) {
        off[v] = acc;
        acc += ncnt[v];
      }
      off[NNF] = acc;
    }
    __syncwarp();
    for (int j = lane; j < n; j += 32) {
      const int v = onode[j], sj = sin[j];
      int pos = 0;
      for (int q = 0; q < n; ++q) pos += (onode[q] == v) && (sin[q] < sj || (sin[q] == sj && q < j));
      lst[off[v] + pos] = (uint16_t)j;
    }
    __syncwarp();
    long long pops = 0;
    far_event* out = P.events + inst * (int64_t)(2 * NNF);
    const int ms = forest_sim<NC, true>(F, n, T, nullptr, nullptr, nullptr, lst, off, cursor, su, (int*)(wsm + L.rs),
                                        wsm + L.rn, wsm + L.rp, wsm + L.ru, ncnt, pops, lane, wsm + L.isz, out,
                                        P.nev + inst);
    if (lane == 0 && P.makespan) P.makespan[inst] = ms;
    __syncwarp();
  }
}

struct FVLayout {
  int b, f, node, cnt, ust, bytes;
};
__host__ __device__ inline FVLayout make_fvlayout(int n, int NNF) {
  FVLayout L;
  int o = 0;
  L.b = o;    o = al16(o + 8 * n);
  L.f = o;    o = al16(o + 8 * n);
  L.node = o; o = al16(o + n);
  L.cnt = o;  o = al16(o + 2 * NNF * 32);
  L.ust = o;  o = al16(o + 8 * 5 * NNF);  // per node: used, #creates, #destroys, create start, destroy end
  L.bytes = o;
  return L;
}

template <int NC>
__global__ void __launch_bounds__(128) far_forest_validate_kernel(FCParams C) {
  extern __shared__ __align__(16) unsigned char smem[];
  const FParams& F = C.F;
  const CParams& P = C.Q;
  const int NNF = F.NNF, n = P.n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const FVLayout L = make_fvlayout(n, NNF);
  unsigned char* wsm = smem + (size_t)warp * L.bytes;
  long long* b = (long long*)(wsm + L.b);
  long long* f = (long long*)(wsm + L.f);
  uint8_t* nd = wsm + L.node;
  uint16_t* cnt = (uint16_t*)(wsm + L.cnt);  // [NNF][32] running tasks per node, per lane
  long long* ust = (long long*)(wsm + L.ust);  // [NNF][5]
  auto overlap = [&](int u, int v) {
    const uint2 a = __ldg(F.nodes + u), c = __ldg(F.nodes + v);
    return fn_lo(a) < fn_lo(c) + fn_sz(c) && fn_lo(c) < fn_lo(a) + fn_sz(a);
  };
  for (;;) {
    unsigned long long uu = 0;
    if (lane == 0) uu = atomicAdd(P.counter, 1ull);
    const int64_t inst = (int64_t)__shfl_sync(FULL, uu, 0);
    if (inst >= P.I) break;
    const far_task_slot* in = P.sched + inst * (int64_t)n;
    const int32_t* t = P.times + inst * (int64_t)n * NC;
    // (0) slots
    int bad = 0;
    for (int j = lane; j < n; j += 32) {
      const far_task_slot sl = in[j];
      int c = -1;
      if (sl.node < NNF) c = fhosted<NC>(__ldg(F.nodes + sl.node), sl.size_used);
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
      for (int j = i + 1; j < n; ++j) v1 += overlap(nd[i], nd[j]) && b[i] < f[j] && b[j] < f[i];
    // (2) at every task start the running instances are pairwise disjoint nodes
    for (int k0 = 0; k0 < n; k0 += 32) {
      const int k = k0 + lane;
      for (int v = 0; v < NNF; ++v) cnt[v * 32 + lane] = 0;
      if (k < n) {
        for (int j = 0; j < n; ++j)
          if (b[j] <= b[k] && b[k] < f[j]) cnt[nd[j] * 32 + lane]++;
        for (int u = 0; u < NNF; ++u) {
          if (!cnt[u * 32 + lane]) continue;
          for (int v = u + 1; v < NNF; ++v)
            if (cnt[v * 32 + lane] && overlap(u, v)) v1 += (long long)cnt[u * 32 + lane] * cnt[v * 32 + lane];
        }
      }
    }
    __syncwarp();
    // (3) events (one pass in order: the last create / destroy of a node wins, as in the oracle)
    const int ne = min(max(P.nev_in[inst], 0), 2 * NNF);
    const far_event* ev = P.events_in + inst * (int64_t)(2 * NNF);
    for (int v = lane; v < NNF; v += 32) {
      long long first = LLONG_MAX, last = LLONG_MIN;
      bool used = false;
      for (int j = 0; j < n; ++j)
        if (nd[j] == v) {
          used = true;
          first = min(first, b[j]);
          last = max(last, f[j]);
        }
      int ncr = 0, nds = 0;
      long long cst = 0, cen = 0, dst = LLONG_MAX, den = LLONG_MAX;
      for (int e = 0; e < ne; ++e) {
        const far_event E = ev[e];
        if (E.node != v) continue;
        if (E.kind == 0) { ncr++; cst = E.start; cen = (long long)E.start + E.dur; }
        else { nds++; dst = E.start; den = (long long)E.start + E.dur; }
      }
      long long v3 = 0;
      if (!used) {
        if (ncr || nds) v3++;
      } else if (ncr != 1 || nds > 1) {
        v3++;
      } else {
        if (cen > first) v3++;
        if (nds && dst < last) v3++;
      }
      v1 += v3;
      ust[v * 5 + 0] = used;
      ust[v * 5 + 1] = ncr;
      ust[v * 5 + 2] = nds;
      ust[v * 5 + 3] = cst;
      ust[v * 5 + 4] = den;
    }
    // events: valid node, correct duration, start >= 0; pairwise disjoint in time
    long long v4 = 0;
    for (int e = lane; e < ne; e += 32) {
      const far_event E = ev[e];
      if (E.node < 0 || E.node >= NNF) { v4++; continue; }
      const uint2 w = __ldg(F.nodes + E.node);
      const int want = E.kind == 0 ? F.P.cr[fn_szi(w)] : F.P.de[fn_szi(w)];
      if (E.dur != want || E.start < 0) v4++;
    }
    for (int e = 0; e < ne; ++e) {
      const far_event E = ev[e];
      if (E.node < 0 || E.node >= NNF) continue;
      for (int g = e + 1 + lane; g < ne; g += 32) {
        const far_event G = ev[g];
        v4 += (long long)E.start < (long long)G.start + G.dur && (long long)G.start < (long long)E.start + E.dur;
      }
    }
    __syncwarp();
    // lifecycles of overlapping used nodes: the earlier-created one is destroyed before the other
    // is created
    for (int v = lane; v < NNF; v += 32) {
      if (!ust[v * 5 + 0]) continue;
      for (int u = 0; u < v; ++u) {
        if (!ust[u * 5 + 0] || !overlap(u, v)) continue;
        const bool u_first = ust[u * 5 + 3] < ust[v * 5 + 3];
        const int a = u_first ? u : v, c = u_first ? v : u;
        if (ust[a * 5 + 2] == 0 || ust[a * 5 + 4] > ust[c * 5 + 3]) v4++;
      }
    }
    const long long viol = warp_sum_ll(v1 + v4);
    if (lane == 0) P.violations[inst] = (int32_t)min(viol, (long long)INT_MAX);
    __syncwarp();
  }
}

}  // namespace farb
