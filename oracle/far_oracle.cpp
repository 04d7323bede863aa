// far_oracle.cpp — plain, slow, single-threaded CPU ORACLE of FAR (arXiv 2507.13601).
//
// TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library.  It shares no code
// with the CUDA path.  Every function follows PAPER.md step by step (citations
// "P:<line>" = /root/reference/PAPER.md line) under the readings of SURVEY.md §8(c)
// / DESIGN.md "Readings".  Library primitives used as steps: std::sort,
// std::priority_queue.  All arithmetic in int64.
//
// Parity pins: see tests/test_oracle_*.py (partition counts, SPEC traces, bounds,
// brute force, validator, golden phase-3 examples).  The multi-batch stream fold
// (O8) is stream_fold / orc_stream at the end of this file.

#include "far_oracle.h"

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <deque>
#include <functional>
#include <limits>
#include <queue>
#include <tuple>
#include <vector>

namespace {

using i64 = int64_t;

// ---------------------------------------------------------------------------
// L0: MIG model.  P:71-87 (slices, instances, partitions), Fig. 3 repartition
// trees (image stripped; reconstructed from P:386, P:726, P:783 — the odd-size
// split gives the first child one extra slice — and P:84-85, the 3-in-4 node).
// SURVEY.md §8c O1 fixes node ids.
// ---------------------------------------------------------------------------
struct TreeNode {
  int lo, hi;                 // slice interval [lo, hi)
  std::vector<int> hosted;    // hosted task sizes, in priority order
  std::vector<int> children;  // child node ids
  int parent;
  int size() const { return hi - lo; }
};

struct Model {
  int slices = 0;
  std::vector<int> sizes;     // C_G
  std::vector<TreeNode> node; // node 0 = root
  bool ok = false;
};

// Multi-target FAR: "as many trees as GPUs, and initially, there is one
// node for the root of each tree to start repartitioning on".  profile = base | (g << 8) with
// g in [2, 8] GPUs: tree t's node v gets id t*NN + v and slices t*S + [lo, hi); every other
// step of FAR is unchanged (one heap, one reconfig_end, R31).
Model make_model_one(int profile);
Model make_model(int profile) {
  const int g = profile >> 8;
  Model one = make_model_one(profile & 255);
  if (g == 0 || g == 1 || !one.ok) return one;
  Model m;
  if (g < 0 || g > 8) return m;
  m.sizes = one.sizes;
  m.slices = g * one.slices;
  const int NN = (int)one.node.size();
  for (int t = 0; t < g; ++t)
    for (const TreeNode& v : one.node) {
      TreeNode w = v;
      w.lo += t * one.slices;
      w.hi += t * one.slices;
      for (int& c : w.children) c += t * NN;
      w.parent = v.parent < 0 ? -1 : v.parent + t * NN;
      m.node.push_back(w);
    }
  m.ok = true;
  return m;
}

Model make_model_one(int profile) {
  Model m;
  if (profile == 0) {  // A30: 4 -> {2,2} -> 4 leaves
    m.slices = 4;
    m.sizes = {1, 2, 4};
    m.node = {
        {0, 4, {4}, {1, 2}, -1}, {0, 2, {2}, {3, 4}, 0}, {2, 4, {2}, {5, 6}, 0},
        {0, 1, {1}, {}, 1},      {1, 2, {1}, {}, 1},     {2, 3, {1}, {}, 2}, {3, 4, {1}, {}, 2},
    };
    m.ok = true;
  } else if (profile == 1 || profile == 2) {  // A100/H100: same tree (Q29)
    m.slices = 7;
    m.sizes = {1, 2, 3, 4, 7};
    m.node = {
        {0, 7, {7}, {1, 2}, -1},
        {0, 4, {4, 3}, {3, 4}, 0},  // {S0..S3}: size-4 tasks first, then size-3 tasks
        {4, 7, {3}, {5, 6}, 0},     // {S4..S6}
        {0, 2, {2}, {7, 8}, 1},  {2, 4, {2}, {9, 10}, 1}, {4, 6, {2}, {11, 12}, 2},
        {6, 7, {1}, {}, 2},
        {0, 1, {1}, {}, 3},  {1, 2, {1}, {}, 3}, {2, 3, {1}, {}, 4}, {3, 4, {1}, {}, 4},
        {4, 5, {1}, {}, 5},  {5, 6, {1}, {}, 5},
    };
    m.ok = true;
  }
  return m;
}

int size_index(const Model& m, int s) {
  for (size_t c = 0; c < m.sizes.size(); ++c)
    if (m.sizes[c] == s) return (int)c;
  return -1;
}

struct Costs {
  std::vector<i64> create, destroy;  // per size index (Table 2)
  i64 cr(const Model& m, int node) const { return create[size_index(m, m.node[node].size())]; }
  i64 de(const Model& m, int node) const { return destroy[size_index(m, m.node[node].size())]; }
};

struct Problem {
  Model m;
  Costs c;
  int n = 0;
  // Variant ORC_SWITCH_COST (R7 variant): a node hosting two sizes (the A100/H100
  // {S0..S3} node) runs an instance of its current task's size: created with t_create of
  // that size, destroyed with t_destroy of that size, and destroyed + re-created (sequentially on
  // reconfig_end) whenever consecutive tasks on it differ in size.  Default: the literal Alg. 1
  // (P:418-424): one instance of the node's size, no reconfiguration between its 4- and 3-tasks.
  bool switch_cost = false;
  std::vector<std::vector<i64>> t;  // t[i][c] = t_i(sizes[c])
  i64 time(int i, int size) const { return t[i][size_index(m, size)]; }
};

// Input checks shared by every entry point.
int load_problem(int profile, const int32_t* costs, const int32_t* times, int n, bool zero, Problem& P) {
  P.m = make_model(profile);
  if (!P.m.ok) return -2;
  if (n < 0 || (n > 0 && !times)) return -1;
  if (n > 1024) return -4;
  const int nc = (int)P.m.sizes.size();
  P.n = n;
  P.c.create.assign(nc, 0);
  P.c.destroy.assign(nc, 0);
  if (costs && !zero) {
    for (int c = 0; c < nc; ++c) {
      P.c.create[c] = costs[c];
      P.c.destroy[c] = costs[nc + c];
      if (costs[c] < 0 || costs[nc + c] < 0) return -3;
    }
  }
  // The oracle's domain is every int32 time >= 1 and cost >= 0: with n <= 1024 every makespan
  // is < 2^10 * 2^31 + 2 * 13 * 8 * 2^31 < 2^42, and the largest product it forms (the ppm stop
  // rule, omega * 10^6) stays below 2^62.  The CUDA path's narrower int32 range (include/far.h
  // "Integer range") is the kernel's contract, not the oracle's.
  P.t.assign(n, std::vector<i64>(nc, 0));
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < nc; ++c) {
      P.t[i][c] = times[(size_t)i * nc + c];
      if (P.t[i][c] < 1) return -3;
    }
  return 0;
}

// ---------------------------------------------------------------------------
// Phase 1: Turek family of allocations.  Allocations hold size VALUES.
// ---------------------------------------------------------------------------
std::vector<std::vector<int>> allocation_family(const Problem& P, bool grow_ties) {
  const Model& m = P.m;
  std::vector<std::vector<int>> fam;
  if (P.n == 0) return fam;
  // First allocation: a_i = argmin_{s in C_G} s * t_i(s); ties -> smallest s (Q3).
  std::vector<int> a(P.n);
  for (int i = 0; i < P.n; ++i) {
    int best = -1;
    i64 bw = 0;
    for (int s : m.sizes) {
      i64 w = (i64)s * P.time(i, s);
      if (best < 0 || w < bw) { best = s; bw = w; }
    }
    a[i] = best;
  }
  fam.push_back(a);
  // a^{k+1} from a^k: grow the longest task (ties -> lowest index, Q2)
  // to argmin_{s > a_j} s * t_j(s) (ties -> smallest s, Q3); stop when it cannot grow (Q4).
  // Variant ORC_GROW_TIES (the formula of P:349 literally): every task whose time equals the
  // maximum grows in the same step; the family ends when one of them cannot grow.
  auto next_size = [&](int j) {
    int best = -1;
    i64 bw = 0;
    for (int s : m.sizes) {
      if (s <= a[j]) continue;
      i64 w = (i64)s * P.time(j, s);
      if (best < 0 || w < bw) { best = s; bw = w; }
    }
    return best;
  };
  for (;;) {
    int j = 0;
    for (int i = 1; i < P.n; ++i)
      if (P.time(i, a[i]) > P.time(j, a[j])) j = i;
    if (!grow_ties) {
      if (a[j] == m.sizes.back()) break;
      a[j] = next_size(j);
    } else {
      const i64 h = P.time(j, a[j]);
      bool stuck = false;
      for (int i = 0; i < P.n; ++i) stuck |= (P.time(i, a[i]) == h && a[i] == m.sizes.back());
      if (stuck) break;
      std::vector<int> grow;
      for (int i = 0; i < P.n; ++i)
        if (P.time(i, a[i]) == h) grow.push_back(i);
      for (int i : grow) a[i] = next_size(i);
    }
    fam.push_back(a);
  }
  return fam;
}

// ---------------------------------------------------------------------------
// Schedule representation: the output tree of Alg. 1 — per node an
// ordered task list — plus per-task start times and the reconfiguration events.
// ---------------------------------------------------------------------------
struct Sched {
  std::vector<std::vector<int>> list;  // per node: task ids in execution order
  std::vector<int> node, size_used;    // per task
  std::vector<i64> start;              // per task
  std::vector<orc_event> events;
  i64 makespan = 0;
  i64 pops = 0;
};

i64 dur(const Problem& P, const Sched& S, int j) { return P.time(j, S.size_used[j]); }

// ---------------------------------------------------------------------------
// Phase 2: Alg. 1 "Schedule an allocation by repartitioning", and the
// line-26 replay of Alg. 2 (O7), which is the same event loop taking each node's
// tasks from its (refined) list instead of from the per-size LPT groups.
//   mode ALLOC : alloc given; groups by size, LPT (lines 1-2)
//   mode LISTS : lists given (per node, in order) with size_used per task
// ---------------------------------------------------------------------------
//   full_lifecycle : also destroy every node with tasks when it is dropped (multi-batch
//                    lifecycle timeline); the single-batch result never
//                    includes these final destroys (R12).
Sched run_event_loop(const Problem& P, const std::vector<int>* alloc,
                     const std::vector<std::vector<int>>* lists, const std::vector<int>* size_used_in,
                     bool full_lifecycle = false) {
  const Model& m = P.m;
  const int N = (int)m.node.size();
  Sched S;
  S.list.assign(N, {});
  S.node.assign(P.n, -1);
  S.size_used.assign(P.n, 0);
  S.start.assign(P.n, 0);

  // Lines 1-2: group the tasks by allotted size, order each group by decreasing
  // time (LPT); ties -> lower task index (Q9).
  std::vector<std::vector<int>> group(m.sizes.size());
  std::vector<size_t> gptr(m.sizes.size(), 0);
  std::vector<size_t> lptr(N, 0);
  if (alloc) {
    for (int i = 0; i < P.n; ++i) group[size_index(m, (*alloc)[i])].push_back(i);
    for (size_t c = 0; c < group.size(); ++c) {
      const int s = m.sizes[c];
      std::sort(group[c].begin(), group[c].end(), [&](int x, int y) {
        if (P.time(x, s) != P.time(y, s)) return P.time(x, s) > P.time(y, s);
        return x < y;
      });
    }
  }
  int unscheduled = P.n;

  std::vector<i64> end(N, 0);
  std::vector<bool> has_tasks(N, false);
  std::vector<int> inst_size(N, 0);  // size of the node's current instance (switch_cost variant)
  i64 reconfig_end = 0;  // line 3
  auto cr_of = [&](int v, int size) {
    return P.switch_cost ? P.c.create[size_index(m, size)] : P.c.cr(m, v);
  };
  auto de_of = [&](int v) { return P.switch_cost ? P.c.destroy[size_index(m, inst_size[v])] : P.c.de(m, v); };
  // Min-heap of instances ordered by end time (line 4); ties -> lower first slice (Q8).
  using Key = std::pair<i64, int>;  // (end, lo) ; node recovered from lo via map below
  auto cmp = [](const std::pair<Key, int>& a, const std::pair<Key, int>& b) { return a.first > b.first; };
  std::priority_queue<std::pair<Key, int>, std::vector<std::pair<Key, int>>, decltype(cmp)> heap(cmp);
  for (int v = 0; v < N; ++v)  // the root (of every tree), R.end = 0, R.tasks = []
    if (m.node[v].parent < 0) heap.push({{0, m.node[v].lo}, v});

  while (!heap.empty()) {  // line 5
    const int v = heap.top().second;  // line 6: pop the first instance to end
    heap.pop();
    S.pops++;
    const int vs = m.node[v].size();
    // Line 7: are there unscheduled tasks assigned to |I| (a hosted size of I)?
    int take = -1, take_size = 0;
    if (alloc) {
      for (int h : m.node[v].hosted) {
        int c = size_index(m, h);
        if (gptr[c] < group[c].size()) { take = group[c][gptr[c]]; take_size = h; gptr[c]++; break; }
      }
    } else if (lptr[v] < (*lists)[v].size()) {
      take = (*lists)[v][lptr[v]++];
      take_size = (*size_used_in)[take];
    }
    if (take >= 0) {
      if (has_tasks[v] && P.switch_cost && inst_size[v] != take_size) {
        // variant: the instance changes size -- destroy it, then create the new one
        i64 ds = std::max(reconfig_end, end[v]);
        reconfig_end = ds + de_of(v);
        S.events.push_back({1, v, ds, de_of(v)});
        const i64 cs = reconfig_end;
        reconfig_end = cs + cr_of(v, take_size);
        S.events.push_back({0, v, cs, cr_of(v, take_size)});
        end[v] = reconfig_end;
        inst_size[v] = take_size;
      }
      if (!has_tasks[v]) {  // lines 8-11: give time for I's creation
        i64 cs = std::max(reconfig_end, end[v]);
        reconfig_end = cs + cr_of(v, take_size);
        S.events.push_back({0, v, cs, cr_of(v, take_size)});
        end[v] = reconfig_end;
        has_tasks[v] = true;
        inst_size[v] = take_size;
      }
      // lines 12-15: longest unscheduled task T_j, executed right after in I
      S.node[take] = v;
      S.size_used[take] = take_size;
      S.start[take] = end[v];
      S.list[v].push_back(take);
      end[v] += P.time(take, take_size);
      S.makespan = std::max(S.makespan, end[v]);
      unscheduled--;
      heap.push({{end[v], m.node[v].lo}, v});  // line 16
    } else if (unscheduled > 0) {             // line 17: repartitioning
      if (has_tasks[v]) {                     // lines 18-20: give time to destroy I
        i64 ds = std::max(reconfig_end, end[v]);
        reconfig_end = ds + de_of(v);
        S.events.push_back({1, v, ds, de_of(v)});
      }
      for (int ch : m.node[v].children) {  // lines 21-24
        end[ch] = end[v];
        has_tasks[ch] = false;
        heap.push({{end[ch], m.node[ch].lo}, ch});
      }
      (void)vs;
    } else if (full_lifecycle && has_tasks[v]) {  // drop: final destroy of the lifecycle timeline
      i64 ds = std::max(reconfig_end, end[v]);
      reconfig_end = ds + de_of(v);
      S.events.push_back({1, v, ds, de_of(v)});
    }
    // else: drop the instance (no tasks remain anywhere)
  }
  return S;
}

Sched schedule_allocation(const Problem& P, const std::vector<int>& alloc) {
  return run_event_loop(P, &alloc, nullptr, nullptr);
}

Sched replay(const Problem& P, const Sched& S) {  // Alg. 2 line 26 (O7)
  return run_event_loop(P, nullptr, &S.list, &S.size_used);
}

// ---------------------------------------------------------------------------
// Phase 3: Alg. 2 "Schedule refinement", moves and
// swaps with the readings Q14-Q19 of SURVEY.md §8c.
// ---------------------------------------------------------------------------
struct RefineStats { int moves = 0, swaps = 0, iterations = 0; i64 evals = 0; };

void insert_ordered(const Problem& P, const Sched& S, std::vector<int>& lst, int j) {
  // "Insert T in I^a.tasks ordered by T.time": decreasing time, ties -> index (Q18)
  auto before = [&](int x, int y) {
    if (dur(P, S, x) != dur(P, S, y)) return dur(P, S, x) > dur(P, S, y);
    return x < y;
  };
  auto it = lst.begin();
  while (it != lst.end() && before(*it, j)) ++it;
  lst.insert(it, j);
}

RefineStats refine(const Problem& P, Sched& S, int max_iterations, int ppm, bool nonempty_alt) {
  const Model& m = P.m;
  const int N = (int)m.node.size();
  RefineStats st;
  // slice ends from the phase-2 times (Q14)
  std::vector<i64> send(m.slices, 0);
  for (int j = 0; j < P.n; ++j) {
    const TreeNode& nd = m.node[S.node[j]];
    for (int s = nd.lo; s < nd.hi; ++s) send[s] = std::max(send[s], S.start[j] + dur(P, S, j));
  }
  auto end_of = [&](int u) {  // end(I) = max_{s in I} s.end
    i64 e = 0;
    for (int s = m.node[u].lo; s < m.node[u].hi; ++s) e = std::max(e, send[s]);
    return e;
  };
  auto add_on = [&](int u, i64 d) {
    for (int s = m.node[u].lo; s < m.node[u].hi; ++s) send[s] += d;
  };
  i64 omega = *std::max_element(send.begin(), send.end());  // line 3
  std::vector<int> leaf_of(m.slices, -1);
  for (int v = 0; v < N; ++v)
    if (m.node[v].children.empty()) leaf_of[m.node[v].lo] = v;

  bool stop = false;
  while (!stop && st.iterations < max_iterations) {  // line 4 (+ iteration cap, Q19)
    st.iterations++;
    const i64 omega_prev = omega;
    // line 5: push the leaves whose slices reach omega (ascending slice order, Q15)
    std::deque<int> Q;
    std::vector<bool> opened(N, false);
    for (int s = 0; s < m.slices; ++s)
      if (send[s] == omega) { Q.push_back(leaf_of[s]); opened[leaf_of[s]] = true; }
    while (!Q.empty()) {  // line 6
      const int I = Q.front();  // line 7
      Q.pop_front();
      if (m.node[I].parent < 0) { stop = true; break; }  // lines 8-10: root opened
      // line 11: alternative I^a, same size, != I, minimum end (ties -> lower slice, Q16)
      int A = -1;
      i64 eA = 0;
      for (int u = 0; u < N; ++u) {
        if (u == I || m.node[u].size() != m.node[I].size()) continue;
        if (nonempty_alt && S.list[u].empty()) continue;  // variant ORC_NONEMPTY_ALT
        i64 e = end_of(u);
        if (A < 0 || e < eA || (e == eA && m.node[u].lo < m.node[A].lo)) { A = u; eA = e; }
      }
      bool done = false;
      if (A >= 0) {
        const i64 marg = omega - eA;  // omega - end(I^a)
        // line 12: task T with T.time < marg closest to marg/2 -> argmin(|2t - marg|, index) (Q17)
        st.evals += (i64)S.list[I].size();
        int T = -1;
        i64 bestd = 0;
        for (int j : S.list[I]) {
          i64 t = dur(P, S, j);
          if (!(t < marg)) continue;
          i64 d = std::llabs(2 * t - marg);
          if (T < 0 || d < bestd || (d == bestd && j < T)) { T = j; bestd = d; }
        }
        if (T >= 0) {  // lines 13-16: move
          const i64 t = dur(P, S, T);
          S.list[I].erase(std::find(S.list[I].begin(), S.list[I].end(), T));
          S.node[T] = A;
          insert_ordered(P, S, S.list[A], T);
          add_on(I, -t);
          add_on(A, +t);
          st.moves++;
          done = true;
        } else {  // lines 17-22: swap
          st.evals += (i64)S.list[I].size() * (i64)S.list[A].size();
          int K = -1, J = -1;
          i64 bd = 0;
          for (int k : S.list[I])
            for (int j : S.list[A]) {
              i64 delta = dur(P, S, k) - dur(P, S, j);
              if (!(0 < delta && delta < marg)) continue;
              i64 d = std::llabs(2 * delta - marg);
              if (K < 0 || d < bd || (d == bd && (k < K || (k == K && j < J)))) { K = k; J = j; bd = d; }
            }
          if (K >= 0) {
            const i64 delta = dur(P, S, K) - dur(P, S, J);
            S.list[I].erase(std::find(S.list[I].begin(), S.list[I].end(), K));
            S.list[A].erase(std::find(S.list[A].begin(), S.list[A].end(), J));
            S.node[K] = A;
            S.node[J] = I;
            insert_ordered(P, S, S.list[A], K);
            insert_ordered(P, S, S.list[I], J);
            add_on(I, -delta);
            add_on(A, +delta);
            st.swaps++;
            done = true;
          }
        }
      }
      if (!done) {  // lines 23-24: open the parent once
        const int par = m.node[I].parent;
        if (par >= 0 && !opened[par]) { opened[par] = true; Q.push_back(par); }
      }
    }
    omega = *std::max_element(send.begin(), send.end());  // line 25
    // optional minimum-improvement stop: integer ppm
    if (ppm > 0 && (omega_prev - omega) * 1000000 < (i64)ppm * omega_prev) break;
  }
  return st;
}

// ---------------------------------------------------------------------------
// Variant ORC_BEST_IMPROVEMENT (R30; SURVEY.md §0 discrepancy 2 / NEXT-3): the
// north star's literal phase 3, "evaluates every task move and swap, recomputes the
// makespan and takes an argmin".  Same node lists, same time model as Alg. 2 (slice ends
// from the phase-2 finishes, moved by +-t; reconfiguration recomputed by the
// line-26 replay), same neighbourhood shape as Alg. 2 (a task only changes to a node of
// the same size, |I^a| = |I|), but every candidate is scored:
//   moves : task T on node I to every node u != I with |u| = |I|
//   swaps : every task pair k < j on two different nodes of the same size
//   score : (w', c') = (max slice end after the operation, #slices reaching w')
//   pick  : argmin (w', c', kind [move 0 < swap 1], first id, second id) where (first,
//           second) = (T, u) for a move and (k, j) for a swap
// The best candidate is applied if (w', c') < (w, c) lexicographically, else the search
// stops (a strict decrease of a well-founded key: it terminates).  evals = number of
// candidates scored.  max_iterations and min-improvement (ppm on w) as in Alg. 2.
// ---------------------------------------------------------------------------
RefineStats refine_best(const Problem& P, Sched& S, int max_iterations, int ppm) {
  const Model& m = P.m;
  const int N = (int)m.node.size();
  RefineStats st;
  std::vector<i64> send(m.slices, 0);
  for (int j = 0; j < P.n; ++j) {
    const TreeNode& nd = m.node[S.node[j]];
    for (int s = nd.lo; s < nd.hi; ++s) send[s] = std::max(send[s], S.start[j] + dur(P, S, j));
  }
  // score of the slice ends after moving d ticks of work from node a to node b
  auto score = [&](int a, int b, i64 d) {
    std::vector<i64> e = send;
    for (int s = m.node[a].lo; s < m.node[a].hi; ++s) e[s] -= d;
    for (int s = m.node[b].lo; s < m.node[b].hi; ++s) e[s] += d;
    const i64 w = *std::max_element(e.begin(), e.end());
    const i64 c = std::count(e.begin(), e.end(), w);
    return std::make_pair(w, c);
  };
  auto cur = score(0, 0, 0);
  while (st.iterations < max_iterations) {
    st.iterations++;
    const i64 omega_prev = cur.first;
    // (w', c', kind, first, second)
    std::tuple<i64, i64, int, int, int> best{std::numeric_limits<i64>::max(), 0, 0, 0, 0};
    bool found = false;
    for (int T = 0; T < P.n; ++T) {  // every move
      const int I = S.node[T];
      for (int u = 0; u < N; ++u) {
        if (u == I || m.node[u].size() != m.node[I].size()) continue;
        st.evals++;
        auto sc = score(I, u, dur(P, S, T));
        std::tuple<i64, i64, int, int, int> key{sc.first, sc.second, 0, T, u};
        if (!found || key < best) { best = key; found = true; }
      }
    }
    for (int k = 0; k < P.n; ++k)  // every swap
      for (int j = k + 1; j < P.n; ++j) {
        const int a = S.node[k], b = S.node[j];
        if (a == b || m.node[a].size() != m.node[b].size()) continue;
        st.evals++;
        auto sc = score(a, b, dur(P, S, k) - dur(P, S, j));
        std::tuple<i64, i64, int, int, int> key{sc.first, sc.second, 1, k, j};
        if (!found || key < best) { best = key; found = true; }
      }
    if (!found || std::make_pair(std::get<0>(best), std::get<1>(best)) >= cur) break;
    const int kind = std::get<2>(best), x = std::get<3>(best), y = std::get<4>(best);
    if (kind == 0) {  // move x to node y
      const int I = S.node[x];
      S.list[I].erase(std::find(S.list[I].begin(), S.list[I].end(), x));
      S.node[x] = y;
      insert_ordered(P, S, S.list[y], x);
      for (int s = m.node[I].lo; s < m.node[I].hi; ++s) send[s] -= dur(P, S, x);
      for (int s = m.node[y].lo; s < m.node[y].hi; ++s) send[s] += dur(P, S, x);
      st.moves++;
    } else {  // swap x (node a) with y (node b)
      const int a = S.node[x], b = S.node[y];
      const i64 d = dur(P, S, x) - dur(P, S, y);
      S.list[a].erase(std::find(S.list[a].begin(), S.list[a].end(), x));
      S.list[b].erase(std::find(S.list[b].begin(), S.list[b].end(), y));
      S.node[x] = b;
      S.node[y] = a;
      insert_ordered(P, S, S.list[b], x);
      insert_ordered(P, S, S.list[a], y);
      for (int s = m.node[a].lo; s < m.node[a].hi; ++s) send[s] -= d;
      for (int s = m.node[b].lo; s < m.node[b].hi; ++s) send[s] += d;
      st.swaps++;
    }
    cur = score(0, 0, 0);
    if (ppm > 0 && (omega_prev - cur.first) * 1000000 < (i64)ppm * omega_prev) break;
  }
  return st;
}

void write_slots(const Sched& S, int n, orc_slot* slots) {
  if (!slots) return;
  for (int j = 0; j < n; ++j) slots[j] = {S.node[j], S.size_used[j], S.start[j]};
}
void write_events(const Sched& S, orc_event* ev, int32_t* nev) {
  if (nev) *nev = (int32_t)S.events.size();
  if (ev)
    for (size_t k = 0; k < S.events.size(); ++k) ev[k] = S.events[k];
}

// Phase 3 + line-26 replay + keep-best guard (Q14), on schedule S whose phase-2
// makespan is ms2.  Returns the final schedule.
Sched refine_and_replay(const Problem& P, const Sched& S2, i64 ms2, int max_it, int ppm, uint32_t flags,
                        orc_result* res) {
  Sched S = S2;
  RefineStats st = (flags & ORC_BEST_IMPROVEMENT) ? refine_best(P, S, max_it, ppm)
                                                  : refine(P, S, max_it, ppm, (flags & ORC_NONEMPTY_ALT) != 0);
  Sched R = replay(P, S);
  res->moves = st.moves;
  res->swaps = st.swaps;
  res->evals = st.evals;
  res->iterations = st.iterations;
  res->reverted = 0;
  if (!(flags & ORC_NO_GUARD) && R.makespan > ms2) {
    res->reverted = 1;
    return S2;
  }
  return R;
}


// ===========================================================================
// §4 Multi-batch concatenation under the readings R21-R25 of
// DESIGN.md §9.  Times of a batch timeline are relative to the batch start;
// the stream state holds absolute times.
// ===========================================================================
struct Life {  // one instance lifecycle inside a batch timeline
  int node = -1;
  i64 cs = 0, ce = 0;  // create  [cs, ce)
  i64 ds = 0, de = 0;  // destroy [ds, de)
  i64 first_task = 0, last_task = 0;
};

struct Timeline {
  std::vector<i64> start;       // per task (relative)
  std::vector<Life> life;       // lifecycles, ordered by node id
  i64 E = 0;                    // end of the last event (relative)
  i64 task_end = 0;             // last task finish (relative)
};

// Full-lifecycle timeline of a batch tree (R22).  forward: the O7 replay where every
// node with tasks is also destroyed when dropped.  reversed: the same loop with
// t_create <-> t_destroy swapped, mirrored about its last event end E, so each mirrored
// destroy has the create duration and vice versa (tasks of a node run in reverse order).
Timeline batch_timeline(const Problem& P, const Sched& S, bool reversed) {
  const Model& m = P.m;
  Problem Q = P;
  if (reversed) std::swap(Q.c.create, Q.c.destroy);
  Sched R = run_event_loop(Q, nullptr, &S.list, &S.size_used, /*full_lifecycle=*/true);
  Timeline T;
  i64 E = 0;
  for (const orc_event& e : R.events) E = std::max(E, e.start + e.dur);
  for (int j = 0; j < P.n; ++j) E = std::max(E, R.start[j] + dur(P, S, j));
  T.E = E;
  T.start.assign(P.n, 0);
  for (int j = 0; j < P.n; ++j) T.start[j] = reversed ? E - (R.start[j] + dur(P, S, j)) : R.start[j];
  for (int j = 0; j < P.n; ++j) T.task_end = std::max(T.task_end, T.start[j] + dur(P, S, j));
  for (int v = 0; v < (int)m.node.size(); ++v) {
    if (S.list[v].empty()) continue;
    Life L;
    L.node = v;
    for (const orc_event& e : R.events) {
      if (e.node != v) continue;
      i64 a = e.start, b = e.start + e.dur;
      if (reversed) { i64 a2 = E - b, b2 = E - a; a = a2; b = b2; }
      const bool is_create = reversed ? (e.kind == 1) : (e.kind == 0);
      if (is_create) { L.cs = a; L.ce = b; } else { L.ds = a; L.de = b; }
    }
    L.first_task = std::numeric_limits<i64>::max();
    L.last_task = std::numeric_limits<i64>::min();
    for (int j : S.list[v]) {
      L.first_task = std::min(L.first_task, T.start[j]);
      L.last_task = std::max(L.last_task, T.start[j] + dur(P, S, j));
    }
    T.life.push_back(L);
  }
  return T;
}

struct LifeAbs {
  int node;
  bool has_create;
  i64 cs, ce, ds, de;        // absolute
  i64 last_task;
  int destroy_ev;            // index into StreamState::events
};
struct EvAbs { i64 s, e; int kind, node; bool alive; };
struct TaskAbs { i64 s, e; int node, life; };

struct StreamState {
  std::vector<i64> tail;       // per slice: end of the last lifecycle on the slice (0 if none)
  std::vector<int> tail_life;  // per slice: that lifecycle (-1 if none)
  std::vector<LifeAbs> lives;
  std::vector<EvAbs> events;
  std::vector<TaskAbs> tasks;
  i64 last_offset = 0;
};

struct SeamEval {
  i64 O = 0, end = 0;
  std::vector<bool> reuse;   // per node
  std::vector<i64> gap;      // per slice
};

// Seam offset (R23): the least O >= max(previous offset, 0) such that (i) on every slice
// B_k's first lifecycle starts after the last placed lifecycle ends, (ii) with the
// destroy/create pair elided where the last placed instance on a node's slices is that
// node and B_k's first instance there is the same node (then task times bound), and
// (iii) B_k's non-elided reconfiguration events overlap no placed event.
SeamEval seam_offset(const Model& m, const StreamState& st, const Timeline& T) {
  const int N = (int)m.node.size();
  SeamEval R;
  R.reuse.assign(N, false);
  std::vector<int> first(m.slices, -1);  // index into T.life of the first lifecycle on s
  for (int q = 0; q < (int)T.life.size(); ++q) {
    const TreeNode& nd = m.node[T.life[q].node];
    for (int s = nd.lo; s < nd.hi; ++s)
      if (first[s] < 0 || T.life[q].cs < T.life[first[s]].cs) first[s] = q;
  }
  for (const Life& L : T.life) {
    const TreeNode& nd = m.node[L.node];
    bool ok = true;
    for (int s = nd.lo; s < nd.hi && ok; ++s) {
      ok = first[s] >= 0 && T.life[first[s]].node == L.node && st.tail_life[s] >= 0 &&
           st.lives[st.tail_life[s]].node == L.node;
    }
    R.reuse[L.node] = ok;
  }
  std::vector<i64> bound(m.slices, 0);
  i64 O = std::max<i64>(st.last_offset, 0);
  for (int s = 0; s < m.slices; ++s) {
    if (first[s] < 0) continue;
    const Life& L = T.life[first[s]];
    bound[s] = R.reuse[L.node] ? st.lives[st.tail_life[s]].last_task - L.first_task : st.tail[s] - L.cs;
    O = std::max(O, bound[s]);
  }
  // (iii): push O past conflicting placed events until none conflicts
  std::vector<std::pair<i64, i64>> mine;
  for (const Life& L : T.life) {
    if (!R.reuse[L.node]) mine.push_back({L.cs, L.ce});
    mine.push_back({L.ds, L.de});
  }
  std::vector<bool> skip(st.events.size(), false);
  for (int s = 0; s < m.slices; ++s)
    if (first[s] >= 0 && R.reuse[T.life[first[s]].node]) skip[st.lives[st.tail_life[s]].destroy_ev] = true;
  for (;;) {
    i64 push = O;
    for (auto& e : mine)
      for (size_t p = 0; p < st.events.size(); ++p) {
        const EvAbs& P = st.events[p];
        if (!P.alive || skip[p]) continue;
        if (e.first + O < P.e && P.s < e.second + O) push = std::max(push, P.e - e.first);
      }
    if (push == O) break;
    O = push;
  }
  R.O = O;
  R.end = O + T.E;
  R.gap.assign(m.slices, 0);
  for (int s = 0; s < m.slices; ++s) {
    i64 g = first[s] >= 0 ? O - bound[s] : O + T.E - st.tail[s];
    R.gap[s] = std::max<i64>(g, 0);
  }
  return R;
}

void place_batch(const Problem& P, const Sched& S, StreamState& st, const Timeline& T, const SeamEval& ev) {
  const Model& m = P.m;
  const i64 O = ev.O;
  std::vector<int> life_id(m.node.size(), -1);
  for (const Life& L : T.life) {
    const TreeNode& nd = m.node[L.node];
    int lid;
    if (ev.reuse[L.node]) {
      lid = st.tail_life[nd.lo];
      st.events[st.lives[lid].destroy_ev].alive = false;  // elided destroy of the previous batch
    } else {
      lid = (int)st.lives.size();
      st.lives.push_back({L.node, true, O + L.cs, O + L.ce, 0, 0, 0, -1});
      st.events.push_back({O + L.cs, O + L.ce, 0, L.node, true});
    }
    st.lives[lid].ds = O + L.ds;
    st.lives[lid].de = O + L.de;
    st.lives[lid].last_task = O + L.last_task;
    st.lives[lid].destroy_ev = (int)st.events.size();
    st.events.push_back({O + L.ds, O + L.de, 1, L.node, true});
    life_id[L.node] = lid;
  }
  for (int j = 0; j < P.n; ++j)
    st.tasks.push_back({O + T.start[j], O + T.start[j] + dur(P, S, j), S.node[j], life_id[S.node[j]]});
  for (int s = 0; s < m.slices; ++s) {  // the last lifecycle on each slice is the one ending last
    int best = -1;
    for (const Life& L : T.life) {
      const TreeNode& nd = m.node[L.node];
      if (s >= nd.lo && s < nd.hi && (best < 0 || L.de > T.life[best].de)) best = (int)(&L - &T.life[0]);
    }
    if (best >= 0) {
      st.tail[s] = O + T.life[best].de;
      st.tail_life[s] = life_id[T.life[best].node];
    }
  }
  st.last_offset = O;
}

// Seam move/swap (R24): Alg. 2's operations on a reversed B_k with the
// inter-batch idle time of a node's slices as the margin; each candidate is evaluated by
// recomputing the mirrored timeline and the seam, and kept only if B_k ends earlier.
struct SeamStats { int moves = 0, swaps = 0; i64 evals = 0; };

SeamStats seam_refine(const Problem& P, Sched& S, const StreamState& st, int max_it) {
  const Model& m = P.m;
  const int N = (int)m.node.size();
  SeamStats stt;
  auto eval = [&](const Sched& X) { return seam_offset(m, st, batch_timeline(P, X, true)); };
  SeamEval cur = eval(S);
  std::vector<int> leaf_of(m.slices, -1);
  for (int v = 0; v < N; ++v)
    if (m.node[v].children.empty()) leaf_of[m.node[v].lo] = v;
  for (int it = 0; it < max_it; ++it) {
    std::vector<bool> touched(m.slices, false);  // slices used by the current B_k
    for (int v = 0; v < N; ++v)
      if (!S.list[v].empty())
        for (int s = m.node[v].lo; s < m.node[v].hi; ++s) touched[s] = true;
    std::deque<int> Q;
    std::vector<bool> opened(N, false);
    for (int s = 0; s < m.slices; ++s)
      if (touched[s] && cur.gap[s] == 0) { Q.push_back(leaf_of[s]); opened[leaf_of[s]] = true; }
    if (Q.empty()) break;
    bool accepted = false, stop = false;
    while (!Q.empty() && !accepted) {
      const int I = Q.front();
      Q.pop_front();
      if (m.node[I].parent < 0) { stop = true; break; }
      auto slack = [&](int u) {
        i64 g = std::numeric_limits<i64>::max();
        for (int s = m.node[u].lo; s < m.node[u].hi; ++s) g = std::min(g, cur.gap[s]);
        return g;
      };
      int A = -1;
      i64 sA = 0;
      for (int u = 0; u < N; ++u) {  // the same-size node with the most idle time (ties -> lower slice)
        if (u == I || m.node[u].size() != m.node[I].size()) continue;
        i64 g = slack(u);
        if (A < 0 || g > sA) { A = u; sA = g; }
      }
      if (A >= 0 && sA > 0) {
        const i64 marg = sA;
        stt.evals += (i64)S.list[I].size();
        int T = -1;
        i64 bd = 0;
        for (int j : S.list[I]) {
          i64 t = dur(P, S, j);
          if (!(t < marg)) continue;
          i64 d = std::llabs(2 * t - marg);
          if (T < 0 || d < bd || (d == bd && j < T)) { T = j; bd = d; }
        }
        if (T >= 0) {
          Sched X = S;
          X.list[I].erase(std::find(X.list[I].begin(), X.list[I].end(), T));
          X.node[T] = A;
          insert_ordered(P, X, X.list[A], T);
          SeamEval e2 = eval(X);
          if (e2.end < cur.end) { S = X; cur = e2; stt.moves++; accepted = true; }
        }
        if (!accepted) {
          stt.evals += (i64)S.list[I].size() * (i64)S.list[A].size();
          int K = -1, J = -1;
          i64 bd2 = 0;
          for (int k : S.list[I])
            for (int j : S.list[A]) {
              i64 delta = dur(P, S, k) - dur(P, S, j);
              if (!(0 < delta && delta < marg)) continue;
              i64 d = std::llabs(2 * delta - marg);
              if (K < 0 || d < bd2 || (d == bd2 && (k < K || (k == K && j < J)))) { K = k; J = j; bd2 = d; }
            }
          if (K >= 0) {
            Sched X = S;
            X.list[I].erase(std::find(X.list[I].begin(), X.list[I].end(), K));
            X.list[A].erase(std::find(X.list[A].begin(), X.list[A].end(), J));
            X.node[K] = A;
            X.node[J] = I;
            insert_ordered(P, X, X.list[A], K);
            insert_ordered(P, X, X.list[I], J);
            SeamEval e2 = eval(X);
            if (e2.end < cur.end) { S = X; cur = e2; stt.swaps++; accepted = true; }
          }
        }
      }
      if (!accepted) {
        const int par = m.node[I].parent;
        if (par >= 0 && !opened[par]) { opened[par] = true; Q.push_back(par); }
      }
    }
    if (stop || !accepted) break;
  }
  return stt;
}

// Stream validator: constraints 1-3 across the concatenated timeline.
int validate_stream(const Model& m, const StreamState& st) {
  int bad = 0;
  auto overlap = [&](int u, int v) { return m.node[u].lo < m.node[v].hi && m.node[v].lo < m.node[u].hi; };
  const size_t nt = st.tasks.size();
  for (size_t a = 0; a < nt; ++a)
    for (size_t b = a + 1; b < nt; ++b)
      if (overlap(st.tasks[a].node, st.tasks[b].node) && st.tasks[a].s < st.tasks[b].e &&
          st.tasks[b].s < st.tasks[a].e)
        bad++;
  for (size_t a = 0; a < st.events.size(); ++a) {
    if (!st.events[a].alive) continue;
    for (size_t b = a + 1; b < st.events.size(); ++b)
      if (st.events[b].alive && st.events[a].s < st.events[b].e && st.events[b].s < st.events[a].e) bad++;
  }
  for (const TaskAbs& t : st.tasks) {
    const LifeAbs& L = st.lives[t.life];
    if (t.s < L.ce || t.e > L.ds) bad++;
  }
  for (size_t a = 0; a < st.lives.size(); ++a)
    for (size_t b = a + 1; b < st.lives.size(); ++b) {
      const LifeAbs &A = st.lives[a], &B = st.lives[b];
      if (overlap(A.node, B.node) && A.cs < B.de && B.cs < A.de) bad++;
    }
  return bad;
}


}  // namespace

// ===========================================================================
// C interface
// ===========================================================================
extern "C" {

int orc_num_sizes(int profile) { Model m = make_model(profile); return m.ok ? (int)m.sizes.size() : -2; }
int orc_num_nodes(int profile) { Model m = make_model(profile); return m.ok ? (int)m.node.size() : -2; }
int orc_num_slices(int profile) { Model m = make_model(profile); return m.ok ? m.slices : -2; }

int orc_nodes(int profile, int32_t* lo, int32_t* hi, int32_t* parent) {
  Model m = make_model(profile);
  if (!m.ok) return -2;
  for (size_t v = 0; v < m.node.size(); ++v) {
    lo[v] = m.node[v].lo;
    hi[v] = m.node[v].hi;
    parent[v] = m.node[v].parent;
  }
  return (int)m.node.size();
}

// Valid partitions: every way of cutting the tree — a node is used
// whole, or (A100/H100 {S0..S3}) as the 3-slice instance {S0,S1,S2} with S3
// unusable, or split into its children.  Each partition is listed as the
// instances (start, size) it creates.
int orc_partitions(int profile, int32_t* out, int32_t* counts, int maxparts, int maxinst) {
  Model m = make_model(profile);
  if (!m.ok) return -2;
  std::function<std::vector<std::vector<std::pair<int, int>>>(int)> cuts = [&](int v) {
    std::vector<std::vector<std::pair<int, int>>> r;
    const TreeNode& nd = m.node[v];
    for (int h : nd.hosted) r.push_back({{nd.lo, h}});  // whole node (or 3-in-4)
    if (!nd.children.empty()) {
      std::vector<std::vector<std::pair<int, int>>> acc = {{}};
      for (int ch : nd.children) {
        std::vector<std::vector<std::pair<int, int>>> nxt;
        for (auto& a : acc)
          for (auto& b : cuts(ch)) {
            auto x = a;
            x.insert(x.end(), b.begin(), b.end());
            nxt.push_back(x);
          }
        acc = nxt;
      }
      r.insert(r.end(), acc.begin(), acc.end());
    }
    return r;
  };
  auto all = cuts(0);
  int k = 0;
  for (auto& p : all) {
    if (k < maxparts && (int)p.size() <= maxinst) {
      counts[k] = (int32_t)p.size();
      for (size_t q = 0; q < p.size(); ++q) {
        out[(size_t)k * 2 * maxinst + 2 * q] = p[q].first;
        out[(size_t)k * 2 * maxinst + 2 * q + 1] = p[q].second;
      }
    }
    ++k;
  }
  return k;
}

int orc_family(int profile, const int32_t* times, int n, int32_t* out, int maxK) {
  return orc_family_flags(profile, times, n, 0u, out, maxK);
}

int orc_family_flags(int profile, const int32_t* times, int n, uint32_t flags, int32_t* out, int maxK) {
  Problem P;
  int rc = load_problem(profile, nullptr, times, n, true, P);
  if (rc) return rc;
  auto fam = allocation_family(P, (flags & ORC_GROW_TIES) != 0);
  for (size_t k = 0; k < fam.size() && (int)k < maxK; ++k)
    for (int i = 0; i < n; ++i) out[k * n + i] = fam[k][i];
  return (int)fam.size();
}

int orc_schedule_allocation(int profile, const int32_t* costs, const int32_t* times, int n, const int32_t* alloc,
                            orc_slot* slots, orc_event* ev, int32_t* nev, int64_t* makespan, int64_t* pops) {
  return orc_schedule_allocation_flags(profile, costs, times, n, alloc, 0, slots, ev, nev, makespan, pops);
}

int orc_schedule_allocation_flags(int profile, const int32_t* costs, const int32_t* times, int n,
                                  const int32_t* alloc, uint32_t flags, orc_slot* slots, orc_event* ev, int32_t* nev,
                                  int64_t* makespan, int64_t* pops) {
  Problem P;
  int rc = load_problem(profile, costs, times, n, (flags & ORC_ZERO_RECONFIG) != 0, P);
  if (rc) return rc;
  P.switch_cost = (flags & ORC_SWITCH_COST) != 0;
  std::vector<int> a(alloc, alloc + n);
  for (int s : a)
    if (size_index(P.m, s) < 0) return -1;
  Sched S = schedule_allocation(P, a);
  write_slots(S, n, slots);
  write_events(S, ev, nev);
  if (makespan) *makespan = S.makespan;
  if (pops) *pops = S.pops;
  return 0;
}

int orc_far(int profile, const int32_t* costs, const int32_t* times, int n, int32_t max_iterations,
            int32_t ppm, uint32_t flags, orc_slot* slots, orc_result* res, orc_event* ev, int32_t* nev) {
  Problem P;
  int rc = load_problem(profile, costs, times, n, (flags & ORC_ZERO_RECONFIG) != 0, P);
  if (rc) return rc;
  P.switch_cost = (flags & ORC_SWITCH_COST) != 0;
  orc_result r{};
  // Phase 1 + phase 2 on every member; k* = argmin (makespan_k, k)  (Q13)
  auto fam = allocation_family(P, (flags & ORC_GROW_TIES) != 0);
  r.family_size = (int)fam.size();
  Sched best;
  int kbest = -1;
  for (size_t k = 0; k < fam.size(); ++k) {
    Sched S = schedule_allocation(P, fam[k]);
    r.events += S.pops;
    if (kbest < 0 || S.makespan < best.makespan) { best = S; kbest = (int)k; }
  }
  if (n == 0) best = Sched{}, best.list.assign(P.m.node.size(), {});
  r.alloc_index = kbest < 0 ? 0 : kbest;
  r.makespan_phase2 = best.makespan;
  Sched fin = best;
  if (!(flags & ORC_NO_REFINE) && n > 0) fin = refine_and_replay(P, best, best.makespan, max_iterations, ppm, flags, &r);
  r.makespan = fin.makespan;
  write_slots(fin, n, slots);
  write_events(fin, ev, nev);
  if (res) *res = r;
  return 0;
}

int orc_refine(int profile, const int32_t* costs, const int32_t* times, int n, int32_t max_iterations, int32_t ppm,
               uint32_t flags, orc_slot* slots, orc_result* res, orc_event* ev, int32_t* nev) {
  Problem P;
  int rc = load_problem(profile, costs, times, n, (flags & ORC_ZERO_RECONFIG) != 0, P);
  if (rc) return rc;
  P.switch_cost = (flags & ORC_SWITCH_COST) != 0;
  if (!slots || !res) return -1;
  const int N = (int)P.m.node.size();
  // Rebuild the tree from the slots: node lists ordered by start time (then index).
  Sched S;
  S.list.assign(N, {});
  S.node.resize(n);
  S.size_used.resize(n);
  S.start.resize(n);
  std::vector<int> order(n);
  for (int j = 0; j < n; ++j) {
    if (slots[j].node < 0 || slots[j].node >= N) return -1;
    bool hosted = false;
    for (int h : P.m.node[slots[j].node].hosted) hosted |= (h == slots[j].size_used);
    if (!hosted) return -1;
    S.node[j] = slots[j].node;
    S.size_used[j] = slots[j].size_used;
    S.start[j] = slots[j].start;
    order[j] = j;
  }
  std::sort(order.begin(), order.end(), [&](int x, int y) {
    return S.start[x] != S.start[y] ? S.start[x] < S.start[y] : x < y;
  });
  for (int j : order) S.list[S.node[j]].push_back(j);
  for (int j = 0; j < n; ++j) S.makespan = std::max(S.makespan, S.start[j] + dur(P, S, j));
  const i64 ms2 = res->makespan_phase2;
  orc_result r = *res;
  Sched fin = S;
  if (n > 0) fin = refine_and_replay(P, S, ms2, max_iterations, ppm, flags, &r);
  r.makespan = fin.makespan;
  write_slots(fin, n, slots);
  write_events(fin, ev, nev);
  *res = r;
  return 0;
}

// Zero-reconfiguration optimum: each task picks a node hosting
// some size; for a fixed choice, running ancestors before descendants is optimal
// and the makespan is the max over slices of the summed loads of the nodes that
// cover the slice (nodes covering one slice form a root-leaf chain).
int64_t orc_bruteforce(int profile, const int32_t* times, int n) {
  Problem P;
  int rc = load_problem(profile, nullptr, times, n, true, P);
  if (rc) return rc;
  const Model& m = P.m;
  std::vector<std::pair<int, int>> choice;  // (node, size)
  for (size_t v = 0; v < m.node.size(); ++v)
    for (int h : m.node[v].hosted) choice.push_back({(int)v, h});
  std::vector<i64> slice_load(m.slices, 0);
  i64 best = std::numeric_limits<i64>::max();
  // order tasks by decreasing minimum time for better pruning
  std::vector<int> ord(n);
  for (int i = 0; i < n; ++i) ord[i] = i;
  std::function<void(int)> rec = [&](int d) {
    i64 cur = *std::max_element(slice_load.begin(), slice_load.end());
    if (cur >= best) return;
    if (d == n) { best = cur; return; }
    const int i = ord[d];
    for (auto& ch : choice) {
      const TreeNode& nd = m.node[ch.first];
      i64 t = P.time(i, ch.second);
      for (int s = nd.lo; s < nd.hi; ++s) slice_load[s] += t;
      rec(d + 1);
      for (int s = nd.lo; s < nd.hi; ++s) slice_load[s] -= t;
    }
  };
  if (n == 0) return 0;
  rec(0);
  return best;
}

// Constraints 1-3 of P:214-230 plus lifecycle consistency of the explicit
// reconfiguration events.  Returns the number of violations.
// Validator of the ORC_SWITCH_COST variant: constraints 1-2 as orc_validate; constraint 3 with
// instances that change size -- per node the events must alternate create, destroy, create, ...
// (a final destroy optional); each create/destroy pair is one instance whose tasks all have one
// size s and lie inside [create end, destroy start), with durations t_create(s) / t_destroy(s);
// every task lies in exactly one instance of its node; events pairwise disjoint; instances of
// overlapping nodes disjoint in time.
static int validate_switch(const Problem& P, const orc_slot* slots, const orc_event* ev, int32_t nev) {
  const Model& m = P.m;
  const int N = (int)m.node.size(), n = P.n;
  int bad = 0;
  auto overlap = [&](int u, int v) { return m.node[u].lo < m.node[v].hi && m.node[v].lo < m.node[u].hi; };
  std::vector<i64> b(n), f(n);
  for (int j = 0; j < n; ++j) {
    const int v = slots[j].node;
    if (v < 0 || v >= N) { bad++; continue; }
    bool hosted = false;
    for (int h : m.node[v].hosted) hosted |= (h == slots[j].size_used);
    if (!hosted) { bad++; continue; }
    b[j] = slots[j].start;
    f[j] = b[j] + P.time(j, slots[j].size_used);
    if (b[j] < 0) bad++;
  }
  if (bad) return bad;
  for (int i = 0; i < n; ++i)  // (1)
    for (int j = i + 1; j < n; ++j)
      if (overlap(slots[i].node, slots[j].node) && b[i] < f[j] && b[j] < f[i]) bad++;
  for (int k = 0; k < n; ++k) {  // (2)
    std::vector<int> run;
    for (int j = 0; j < n; ++j)
      if (b[j] <= b[k] && b[k] < f[j]) run.push_back(slots[j].node);
    for (size_t x = 0; x < run.size(); ++x)
      for (size_t y = x + 1; y < run.size(); ++y)
        if (run[x] != run[y] && overlap(run[x], run[y])) bad++;
  }
  for (int e = 0; e < nev; ++e) {  // (3) sequential reconfiguration
    if (ev[e].node < 0 || ev[e].node >= N || ev[e].start < 0) { bad++; continue; }
    for (int g = e + 1; g < nev; ++g)
      if (ev[e].start < ev[g].start + ev[g].dur && ev[g].start < ev[e].start + ev[e].dur) bad++;
  }
  struct Inst { int node; i64 cs, de; };
  std::vector<Inst> inst;
  std::vector<int> covered(n, 0);
  for (int v = 0; v < N; ++v) {
    std::vector<orc_event> E;
    for (int e = 0; e < nev; ++e)
      if (ev[e].node == v) E.push_back(ev[e]);
    std::sort(E.begin(), E.end(), [](const orc_event& x, const orc_event& y) { return x.start < y.start; });
    for (size_t q = 0; q < E.size(); q += 2) {
      if (E[q].kind != 0 || (q + 1 < E.size() && E[q + 1].kind != 1)) { bad++; break; }
      const i64 cs = E[q].start, ce = cs + E[q].dur;
      const bool closed = q + 1 < E.size();
      const i64 ds = closed ? E[q + 1].start : std::numeric_limits<i64>::max();
      const i64 de = closed ? ds + E[q + 1].dur : ds;
      int size = -1, ntask = 0;
      for (int j = 0; j < n; ++j) {
        if (slots[j].node != v || b[j] < ce || f[j] > ds) continue;
        ntask++;
        covered[j]++;
        if (size < 0) size = slots[j].size_used;
        else if (size != slots[j].size_used) bad++;
      }
      if (ntask == 0) { bad++; continue; }
      if (E[q].dur != P.c.create[size_index(m, size)]) bad++;
      if (closed && E[q + 1].dur != P.c.destroy[size_index(m, size)]) bad++;
      inst.push_back({v, cs, de});
    }
  }
  for (int j = 0; j < n; ++j)
    if (covered[j] != 1) bad++;
  for (size_t x = 0; x < inst.size(); ++x)
    for (size_t y = x + 1; y < inst.size(); ++y) {
      if (inst[x].node == inst[y].node || !overlap(inst[x].node, inst[y].node)) continue;
      const Inst& a = inst[x].cs < inst[y].cs ? inst[x] : inst[y];
      const Inst& c = inst[x].cs < inst[y].cs ? inst[y] : inst[x];
      if (a.de > c.cs) bad++;
    }
  return bad;
}

int orc_validate_flags(int profile, const int32_t* costs, const int32_t* times, int n, const orc_slot* slots,
                       const orc_event* ev, int32_t nev, uint32_t flags) {
  if (!(flags & ORC_SWITCH_COST)) return orc_validate(profile, costs, times, n, slots, ev, nev);
  Problem P;
  int rc = load_problem(profile, costs, times, n, costs == nullptr, P);
  if (rc) return 1000000 - rc;
  return validate_switch(P, slots, ev, nev);
}

int orc_validate(int profile, const int32_t* costs, const int32_t* times, int n, const orc_slot* slots,
                 const orc_event* ev, int32_t nev) {
  Problem P;
  int rc = load_problem(profile, costs, times, n, costs == nullptr, P);
  if (rc) return 1000000 - rc;
  const Model& m = P.m;
  const int N = (int)m.node.size();
  int bad = 0;
  auto overlap = [&](int u, int v) { return m.node[u].lo < m.node[v].hi && m.node[v].lo < m.node[u].hi; };
  std::vector<i64> b(n), f(n);
  for (int j = 0; j < n; ++j) {
    int v = slots[j].node;
    if (v < 0 || v >= N) { bad++; continue; }
    bool hosted = false;
    for (int h : m.node[v].hosted) hosted |= (h == slots[j].size_used);
    if (!hosted) { bad++; continue; }
    b[j] = slots[j].start;
    f[j] = b[j] + P.time(j, slots[j].size_used);
    if (b[j] < 0) bad++;
  }
  if (bad) return bad;
  // (1) tasks whose instances share a slice do not run at the same time
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j)
      if (overlap(slots[i].node, slots[j].node) && b[i] < f[j] && b[j] < f[i]) bad++;
  // (2) at every task start the running instances are pairwise disjoint tree nodes
  //     (the tree's disjoint node sets are exactly the valid partitions' subsets)
  for (int k = 0; k < n; ++k) {
    std::vector<int> run;
    for (int j = 0; j < n; ++j)
      if (b[j] <= b[k] && b[k] < f[j]) run.push_back(slots[j].node);
    for (size_t x = 0; x < run.size(); ++x)
      for (size_t y = x + 1; y < run.size(); ++y)
        if (run[x] != run[y] && overlap(run[x], run[y])) bad++;
  }
  // (3) sequential reconfiguration: events pairwise disjoint, correctly sized; every
  //     node with tasks is created before its first task; lifecycles of nodes with
  //     overlapping slices are disjoint (destroy before the next create).
  std::vector<i64> first(N, std::numeric_limits<i64>::max()), last(N, std::numeric_limits<i64>::min());
  std::vector<bool> used(N, false);
  for (int j = 0; j < n; ++j) {
    int v = slots[j].node;
    used[v] = true;
    first[v] = std::min(first[v], b[j]);
    last[v] = std::max(last[v], f[j]);
  }
  std::vector<i64> cstart(N, 0), cend(N, 0), dstart(N, std::numeric_limits<i64>::max()),
      dend(N, std::numeric_limits<i64>::max());
  std::vector<int> ncreate(N, 0), ndestroy(N, 0);
  for (int e = 0; e < nev; ++e) {
    const orc_event& E = ev[e];
    if (E.node < 0 || E.node >= N) { bad++; continue; }
    i64 want = E.kind == 0 ? P.c.cr(m, E.node) : P.c.de(m, E.node);
    if (E.dur != want || E.start < 0) bad++;
    if (E.kind == 0) { ncreate[E.node]++; cstart[E.node] = E.start; cend[E.node] = E.start + E.dur; }
    else { ndestroy[E.node]++; dstart[E.node] = E.start; dend[E.node] = E.start + E.dur; }
    for (int g = e + 1; g < nev; ++g)
      if (E.start < ev[g].start + ev[g].dur && ev[g].start < E.start + E.dur) bad++;
  }
  for (int v = 0; v < N; ++v) {
    if (!used[v]) { if (ncreate[v] || ndestroy[v]) bad++; continue; }
    if (ncreate[v] != 1 || ndestroy[v] > 1) { bad++; continue; }
    if (cend[v] > first[v]) bad++;
    if (ndestroy[v] && dstart[v] < last[v]) bad++;
  }
  for (int u = 0; u < N; ++u)
    for (int v = u + 1; v < N; ++v) {
      if (!used[u] || !used[v] || !overlap(u, v)) continue;
      // lifecycle [cstart, dend) ; the earlier one must be destroyed before the later is created
      bool u_first = cstart[u] < cstart[v];
      int a = u_first ? u : v, c = u_first ? v : u;
      if (ndestroy[a] == 0 || dend[a] > cstart[c]) bad++;
    }
  return bad;
}

int orc_lower_bound(int profile, const int32_t* times, int n, int64_t* sum_min_work, int64_t* max_min_time) {
  Problem P;
  int rc = load_problem(profile, nullptr, times, n, true, P);
  if (rc) return rc;
  i64 W = 0, H = 0;
  for (int i = 0; i < n; ++i) {
    i64 w = std::numeric_limits<i64>::max(), h = std::numeric_limits<i64>::max();
    for (int s : P.m.sizes) {
      w = std::min(w, (i64)s * P.time(i, s));
      h = std::min(h, P.time(i, s));
    }
    W += w;
    H = std::max(H, h);
  }
  *sum_min_work = W;
  *max_min_time = H;
  return 0;
}

int orc_far_many(int profile, const int32_t* costs, const int32_t* times, int64_t I, int n, int32_t max_iterations,
                 int32_t ppm, uint32_t flags, int64_t* makespans, orc_result* res) {
  return orc_far_many_slots(profile, costs, times, I, n, max_iterations, ppm, flags, makespans, res, nullptr);
}

int orc_far_many_slots(int profile, const int32_t* costs, const int32_t* times, int64_t I, int n,
                       int32_t max_iterations, int32_t ppm, uint32_t flags, int64_t* makespans, orc_result* res,
                       orc_slot* slots) {
  const int nc = orc_num_sizes(profile);
  if (nc < 0) return nc;
  int worst = 0;
  for (int64_t i = 0; i < I; ++i) {
    orc_result r{};
    int rc = orc_far(profile, costs, times + (size_t)i * n * nc, n, max_iterations, ppm, flags,
                     slots ? slots + (size_t)i * n : nullptr, &r, nullptr, nullptr);
    if (rc) { worst = rc; r.makespan = -1; }
    if (makespans) makespans[i] = r.makespan;
    if (res) res[i] = r;
  }
  return worst;
}

}  // extern "C"

// The fold of orc_stream; with probe_k >= 0 it stops after batch probe_k, which is placed
// delta ticks before its seam offset (test entry orc_stream_probe: minimality of R23's offset).
static int stream_fold(int profile, const int32_t* costs, const int32_t* times, int B, int n,
                       int32_t max_iterations, int32_t ppm, uint32_t flags, int64_t* out2, int64_t* offsets,
                       int32_t* seam, orc_slot* slots, orc_result* batch_res, int32_t* violations, int probe_k,
                       int64_t delta, int64_t* ends = nullptr);

extern "C" int orc_stream(int profile, const int32_t* costs, const int32_t* times, int B, int n,
                          int32_t max_iterations, int32_t ppm, uint32_t flags, int64_t* out2, int64_t* offsets,
                          int32_t* seam, orc_slot* slots, orc_result* batch_res, int32_t* violations) {
  return stream_fold(profile, costs, times, B, n, max_iterations, ppm, flags, out2, offsets, seam, slots, batch_res,
                     violations, -1, 0);
}

// Test entry: orc_stream plus ends[k] = O_k + E_k, the end of batch k's placed timeline (the
// quantity R24's keep-best rule compares).
extern "C" int orc_stream_ends(int profile, const int32_t* costs, const int32_t* times, int B, int n,
                               int32_t max_iterations, int32_t ppm, uint32_t flags, int64_t* out2, int64_t* offsets,
                               int32_t* seam, orc_slot* slots, orc_result* batch_res, int32_t* violations,
                               int64_t* ends) {
  return stream_fold(profile, costs, times, B, n, max_iterations, ppm, flags, out2, offsets, seam, slots, batch_res,
                     violations, -1, 0, ends);
}

// Test entry: violations of the concatenation of batches 0..k when batch k starts delta ticks
// before its seam offset (everything else as orc_stream).  *offset_k = the unshifted offset.
extern "C" int orc_stream_probe(int profile, const int32_t* costs, const int32_t* times, int B, int n, int k,
                                int64_t delta, int64_t* offset_k, int32_t* violations) {
  std::vector<int64_t> offs(B > 0 ? B : 1, 0);
  int rc = stream_fold(profile, costs, times, B, n, 100, 0, 0, nullptr, offs.data(), nullptr, nullptr, nullptr,
                       violations, k, delta);
  if (offset_k && k >= 0 && k < B) *offset_k = offs[k];
  return rc;
}

static int stream_fold(int profile, const int32_t* costs, const int32_t* times, int B, int n,
                       int32_t max_iterations, int32_t ppm, uint32_t flags, int64_t* out2, int64_t* offsets,
                       int32_t* seam, orc_slot* slots, orc_result* batch_res, int32_t* violations, int probe_k,
                       int64_t delta, int64_t* ends) {
  const int nc = orc_num_sizes(profile);
  if (nc < 0) return nc;
  if (B < 0 || n < 0) return -1;
  std::vector<Problem> Pb(B);
  std::vector<Sched> fin(B);
  // each batch: FAR phases 1-3
  for (int k = 0; k < B; ++k) {
    int rc = load_problem(profile, costs, times + (size_t)k * n * nc, n, (flags & ORC_ZERO_RECONFIG) != 0, Pb[k]);
    if (rc) return rc;
    Pb[k].switch_cost = (flags & ORC_SWITCH_COST) != 0;
    const Problem& P = Pb[k];
    orc_result r{};
    auto fam = allocation_family(P, (flags & ORC_GROW_TIES) != 0);
    r.family_size = (int)fam.size();
    Sched best;
    int kbest = -1;
    for (size_t q = 0; q < fam.size(); ++q) {
      Sched S = schedule_allocation(P, fam[q]);
      r.events += S.pops;
      if (kbest < 0 || S.makespan < best.makespan) { best = S; kbest = (int)q; }
    }
    if (n == 0) best = Sched{}, best.list.assign(P.m.node.size(), {});
    r.alloc_index = kbest < 0 ? 0 : kbest;
    r.makespan_phase2 = best.makespan;
    Sched f = best;
    if (!(flags & ORC_NO_REFINE) && n > 0) f = refine_and_replay(P, best, best.makespan, max_iterations, ppm, flags, &r);
    r.makespan = f.makespan;
    fin[k] = f;
    if (batch_res) batch_res[k] = r;
  }
  // trivial concatenation (R25): forward batches one after another
  i64 triv_ms = 0, prev_end = 0;
  for (int k = 0; k < B; ++k) {
    Timeline T = batch_timeline(Pb[k], fin[k], false);
    const i64 O = k == 0 ? 0 : prev_end;
    triv_ms = std::max(triv_ms, O + T.task_end);
    prev_end = O + T.E;
  }
  // reversal + seam offset + seam move/swap fold (R21-R24)
  StreamState st;
  const Model& m = Pb.empty() ? make_model(profile) : Pb[0].m;
  Model mm = make_model(profile);
  st.tail.assign(mm.slices, 0);
  st.tail_life.assign(mm.slices, -1);
  i64 ms = 0;
  for (int k = 0; k < B; ++k) {
    const bool rev = (k % 2) == 1;
    Sched S = fin[k];
    SeamStats ss;
    if (rev && k > 0 && !(flags & ORC_NO_SEAM_MOVES)) ss = seam_refine(Pb[k], S, st, max_iterations);
    Timeline T = batch_timeline(Pb[k], S, rev);
    SeamEval ev = seam_offset(mm, st, T);
    int reused = 0;
    for (bool b : ev.reuse) reused += b;
    if (offsets) offsets[k] = ev.O;
    if (ends) ends[k] = ev.end;
    if (k == probe_k) {  // probe: place this batch delta ticks early, validate, stop
      ev.O -= delta;
      place_batch(Pb[k], S, st, T, ev);
      if (violations) *violations = validate_stream(mm, st);
      return 0;
    }
    place_batch(Pb[k], S, st, T, ev);
    ms = std::max(ms, ev.O + T.task_end);
    if (seam) {
      seam[4 * k + 0] = rev;
      seam[4 * k + 1] = ss.moves;
      seam[4 * k + 2] = ss.swaps;
      seam[4 * k + 3] = reused;
    }
    if (slots)
      for (int j = 0; j < n; ++j) slots[(size_t)k * n + j] = {S.node[j], S.size_used[j], T.start[j]};
  }
  (void)m;
  if (out2) { out2[0] = ms; out2[1] = triv_ms; }
  if (violations) *violations = validate_stream(mm, st);
  return 0;
}

// Test entry (tests/test_oracle_stream.py): the seam offset of a batch whose first use of
// slice s starts at first[s] (first[s] < 0: slice unused), after placed lifecycles ending at
// tail[s], with zero-length reconfiguration events and no reuse (SPEC.md:345-350 examples).
extern "C" int64_t orc_seam_offset_simple(int profile, const int64_t* tail, const int64_t* first) {
  Model m = make_model(profile);
  if (!m.ok) return -2;
  StreamState st;
  st.tail.assign(tail, tail + m.slices);
  st.tail_life.assign(m.slices, -1);
  Timeline T;
  for (int s = 0; s < m.slices; ++s) {
    if (first[s] < 0) continue;
    Life L;
    for (int v = 0; v < (int)m.node.size(); ++v)
      if (m.node[v].children.empty() && m.node[v].lo == s) L.node = v;
    L.cs = L.ce = L.first_task = first[s];
    L.ds = L.de = L.last_task = first[s] + 1;
    T.life.push_back(L);
    T.E = std::max(T.E, first[s] + 1);
  }
  return seam_offset(m, st, T).O;
}
