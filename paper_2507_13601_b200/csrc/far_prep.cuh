// far_prep.cuh — K1 of the pipelined solver (far_pipeline.cuh) for batches of n <= 128 tasks:
// H0-H3 of one instance per warp, every per-task quantity in registers (lane l owns tasks
// l, l + 32, ..., l + 32(R-1)), the per-size LPT lists rank-scattered straight into the workspace.
//
//   H0  runtime table t[n][|C|] -> shared memory (16-B streaming loads)
//   H1  a^1_j = argmin_s s*t_j(s), ties -> smallest s; the growth chain of every task,
//       a^1 -> nx(a^1) -> ... -> max size with nx(c) = argmin_{c' > c} (size(c') t(c'), c')
//   H2  the family: with t non-increasing along every chain (property 1)
//       the growth process is the merge of the chains by key (t, -task, -position): each step
//       grows the longest current task, so the steps are the non-terminal chain elements whose key
//       exceeds the largest terminal key T*, in decreasing key order.  Keys are unique 32-bit words
//       t << 10 | (127 - task) << 3 | (7 - position), so a step's rank is one count over the steps
//   H3  per-size lists of the (task, size) pairs some member uses, each tagged with its member
//       interval [lo, hi), in LPT order (-t, task) (Alg. 1 lines 1-2): the a^1 entries of
//       a size and its growth entries are compacted into two padded shared-memory segments by packed
//       per-lane counters, then every entry is ranked against the keys of its size (LDS.128
//       broadcasts + carry counting) and stored at its rank -- and, for an a^1 entry, at its rank
//       among the a^1 entries in member 0's compact list
//
// Same workspace contract and results as far_solve_kernel<NC, PIPE_PREP> (far_kernel.cuh); an
// instance outside this kernel's domain (t >= 2^22, a chain along which t increases, a family of
// more than kcap members) is deferred to the fused overflow pass exactly as there.  Input errors
// are reported the same way (include/far.h "Integer range").
#pragma once
#include "far_kernel.cuh"

namespace farb {

#ifndef FAR_PREP_TMA
#define FAR_PREP_TMA 1  // H0 stages the runtime table with one TMA bulk copy per instance
#endif

struct PLayout {
  int T, info, gk, ginfo, rnk, cnts, lbs, lbh, kk, bytes;
};

// Per-warp shared memory: the table, per-task words, the growth steps (keys, descriptors, ranks),
// per-member counts / area / longest time, and the sorted list keys (kk aliases the growth keys,
// which are dead once the steps are ranked).
__host__ __device__ inline PLayout make_playout(int n, int NC, int kcap) {
  PLayout L;
  int o = 0;
  L.T = o;     o = al16(o + 4 * n * NC);
  L.info = o;  o = al16(o + 4 * n);
  L.gk = o;    o = al16(o + 4 * (kcap + 4 > 256 ? kcap + 4 : 256));
  L.kk = L.gk;
  L.ginfo = o; o = al16(o + 4 * kcap);
  L.rnk = o;   o = al16(o + 4 * kcap);
  L.cnts = o;  o = al16(o + 8 * kcap);
  L.lbs = o;   o = al16(o + 4 * kcap);
  L.lbh = o;   o = al16(o + 4 * kcap);
  L.bytes = o;
  return L;
}

// Ascending bitonic sort of 256 keys, 8 per lane, element i = lane * 8 + q in v[q] (blocked: the
// 21 stages whose partners differ only in q are register pairs, the other 15 shuffles).  Every
// comparator keeps the minimum at the lower index (block step: i <-> i ^ (k - 1), then
// half-cleaners i <-> i ^ j), so no stage needs a direction.
__device__ __forceinline__ void warp_sort256(unsigned (&v)[8], int lane) {
#pragma unroll
  for (int k = 2; k <= 256; k <<= 1) {
    if (k <= 8) {
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < (q ^ (k - 1))) {
          const unsigned x = v[q], y = v[q ^ (k - 1)];
          v[q] = min(x, y);
          v[q ^ (k - 1)] = max(x, y);
        }
    } else {
      const bool lower = (lane & (k >> 4)) == 0;
      unsigned o[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) o[q] = __shfl_xor_sync(FULL, v[q ^ 7], (k - 1) >> 3);
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = lower ? min(v[q], o[q]) : max(v[q], o[q]);
    }
#pragma unroll
    for (int j = k >> 2; j > 0; j >>= 1) {
      if (j < 8) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if ((q & j) == 0) {
            const unsigned x = v[q], y = v[q | j];
            v[q] = min(x, y);
            v[q | j] = max(x, y);
          }
      } else {
        const bool lower = (lane & (j >> 3)) == 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const unsigned o = __shfl_xor_sync(FULL, v[q], j >> 3);
          v[q] = lower ? min(v[q], o) : max(v[q], o);
        }
      }
    }
  }
}

__device__ __forceinline__ int fld11(unsigned long long p, int c) { return (int)((p >> (11 * c)) & 2047u); }

// #{f in [f0, f1): seg[f] <= key} for a 16-B aligned, 4-padded key segment (LDS.128 broadcasts,
// one carry-chain compare per key)
__device__ __forceinline__ int count_le(const unsigned* seg, int f0, int f1, unsigned key) {
  int c = 0;
#pragma unroll 2
  for (int f = f0; f < f1; f += 4) {
    const uint4 v = *(const uint4*)(seg + f);
    count_ge(c, key, v.x);
    count_ge(c, key, v.y);
    count_ge(c, key, v.z);
    count_ge(c, key, v.w);
  }
  return c;
}

template <int NC>
__device__ __forceinline__ unsigned growth_key(int t, int j, int p) {
  return ((unsigned)t << 10) | ((unsigned)(127 - j) << 3) | (unsigned)(7 - p);
}

// H2 when some task's t increases along its growth chain: the growth process step by step
// (P:343-352): grow the longest current task (ties -> lowest index) to its next chain size; stop
// when it is already at the largest size.  Writes steps[k] = task | its step number << 8 (into gk),
// counts each task's steps in info (bits 8-10), returns the number of steps (-1 if the family
// exceeds kcap) and the longest time of the last member in tlast.
template <int NC>
__device__ __forceinline__ int seq_growth(const int32_t* T, uint32_t* info, uint32_t* gk, int n, int kcap, int lane,
                                       unsigned& tlast) {
  uint32_t* steps = gk;                     // dead until the list keys are built
  uint8_t* curc = (uint8_t*)(gk + kcap);    // current size index per task
  for (int j = lane; j < n; j += 32) curc[j] = (uint8_t)(info[j] & 7u);
  __syncwarp();
  unsigned lk = 0;
  for (int j = lane; j < n; j += 32) lk = max(lk, ((unsigned)T[j * NC + curc[j]] << 10) | (unsigned)(1023 - j));
  int K = 1;
  for (;;) {
    const unsigned gkey = __reduce_max_sync(FULL, lk);
    const int jj = 1023 - (int)(gkey & 1023u);
    const int c = curc[jj];
    if (c == NC - 1) {
      tlast = gkey >> 10;
      return K - 1;
    }
    if (K >= kcap) return -1;
    const uint32_t w = info[jj];
    __syncwarp();
    if (lane == 0) {
      steps[K - 1] = (uint32_t)jj | (((w >> 8) & 7u) << 8);
      info[jj] = w + (1u << 8);
      curc[jj] = (uint8_t)(__ffs(((w >> 3) & 31u) & ~((2u << c) - 1u)) - 1);
    }
    __syncwarp();
    if (lane == (jj & 31)) {
      lk = 0;
      for (int j = lane; j < n; j += 32) lk = max(lk, ((unsigned)T[j * NC + curc[j]] << 10) | (unsigned)(1023 - j));
    }
    ++K;
  }
}

// The sequential steps as elements: step k is task j's p-th, its element index is first_j + p;
// its rank is k.
template <int NC>
__device__ __forceinline__ void seq_elements(const uint32_t* info, const uint32_t* steps, uint32_t* ginfo, int* rnk,
                                          int Gn, int lane) {
  for (int k = lane; k < Gn; k += 32) {
    const uint32_t x = steps[k];
    const int j = (int)(x & 255u), p = (int)(x >> 8);
    const uint32_t w = info[j];
    const int g = (int)((w >> 8) & 7u);
    unsigned m = (w >> 3) & 31u;
    for (int q = 0; q < p; ++q) m &= m - 1;
    const int c = __ffs(m) - 1;
    m &= m - 1;
    const int e = (int)(w >> 11) + p;
    rnk[e] = k;
    ginfo[e] = (uint32_t)j | ((uint32_t)c << 8) | ((uint32_t)(__ffs(m) - 1) << 11) | ((uint32_t)(p == g - 1) << 14);
  }
}

// Defer an instance to the fused overflow pass (outside the prep kernel's domain).
__device__ __forceinline__ void defer_instance(const KParams& P, int64_t inst, int lane) {
  if (lane == 0) {
    atomicOr(P.ovf + (inst >> 5), 1u << (inst & 31));
    atomicAdd(P.ovf_count, 1ull);
    P.ws_meta[inst * 16 + WS_FLAG] = 1;
  }
}

// H2-H3 and the workspace outputs.  MONO: every task's t is non-increasing along its growth chain
// (the hot path: the merge form of H2); otherwise the step-by-step growth (out of line).
template <int NC, bool MONO>
__device__ __forceinline__ void prep_rest(const KParams& P, int64_t inst, unsigned char* wsm, const PLayout& L,
                                          int lane, unsigned tstar, unsigned W, unsigned long long c0) {
  constexpr int S = Tree<NC>::S;
  const int n = P.n;
  int32_t* T = (int32_t*)(wsm + L.T);
  uint32_t* info = (uint32_t*)(wsm + L.info);
  unsigned* gk = (unsigned*)(wsm + L.gk);
  uint32_t* ginfo = (uint32_t*)(wsm + L.ginfo);
  int* rnk = (int*)(wsm + L.rnk);
  unsigned long long* cnts = (unsigned long long*)(wsm + L.cnts);
  unsigned* lbs = (unsigned*)(wsm + L.lbs);
  int* lbh = (int*)(wsm + L.lbh);
  unsigned* kk = (unsigned*)(wsm + L.kk);
  int* meta = P.ws_meta + inst * 16;
  const unsigned lt = (1u << lane) - 1u;
  auto defer = [&]() { defer_instance(P, inst, lane); };
  int Gn = 0;
  unsigned tlast = tstar >> 10;  // longest task of the last member
  int gsum = 0;  // this lane's steps
  if (MONO) {
    // ---- H2: growth steps = non-terminal chain elements with key > T*, a prefix of each chain
    //      (keys strictly decrease along a chain, so the count needs no early exit)
#pragma unroll 1
    for (int j = lane; j < n; j += 32) {
      const uint32_t w = info[j];
      const unsigned m = (w >> 3) & ((1u << (NC - 1)) - 1u);  // non-terminal chain elements
      int g = 0, p = 0;
#pragma unroll
      for (int c = 0; c < NC - 1; ++c) {  // size index c (compile-time offset), chain position p
        const bool on = (m >> c) & 1u;
        g += on & (growth_key<NC>(T[j * NC + c], j, p) > tstar);
        p += on;
      }
      info[j] = w | ((uint32_t)g << 8);
      gsum += g;
    }
    Gn = __reduce_add_sync(FULL, gsum);
  } else {
    // ---- H2, general form (a chain along which t increases), out of line: keeps the hot
    //      monotone path inside the instruction cache
    Gn = seq_growth<NC>(T, info, gk, n, P.kcap, lane, tlast);
    if (Gn < 0) {
      defer();
      return;
    }
    for (int j = lane; j < n; j += 32) gsum += (int)((info[j] >> 8) & 7u);
  }
  if (Gn + 1 > P.kcap) {
    defer();
    return;
  }
  const int K = Gn + 1;
  // first step index per task (lane-major order of tasks; a task's steps are consecutive and in
  // chain order); the growing tasks (g > 0, at most Gn of them) listed in gt
  {
    int excl = gsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, excl, o);
      if (lane >= o) excl += y;
    }
    excl -= gsum;
    uint32_t* gt = (uint32_t*)lbh;  // lbh is written after the steps are ranked
    int ng = 0;
#pragma unroll 1
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      const uint32_t w = j < n ? info[j] : 0u;
      const int g = (int)((w >> 8) & 7u);
      if (j < n) info[j] = w | ((uint32_t)excl << 11);
      const unsigned b = __ballot_sync(FULL, g > 0);
      if (g > 0) gt[ng + __popc(b & lt)] = (uint32_t)j | ((uint32_t)excl << 8);
      ng += __popc(b);
      excl += g;
    }
    __syncwarp();
    if (MONO) {
      // steps of each growing task in chain order (lane per growing task), keyed for the ranking
#pragma unroll 1
      for (int i = lane; i < ng; i += 32) {
        const uint32_t x = gt[i];
        const int j = (int)(x & 255u);
        int e = (int)(x >> 8);
        const uint32_t w = info[j];
        const int g = (int)((w >> 8) & 7u);
        unsigned m = (w >> 3) & 31u;
        for (int p = 0; p < g; ++p, ++e) {
          const int c = __ffs(m) - 1;
          m &= m - 1;
          gk[e] = growth_key<NC>(T[j * NC + c], j, p);
          ginfo[e] = (uint32_t)j | ((uint32_t)c << 8) | ((uint32_t)(__ffs(m) - 1) << 11) | ((uint32_t)(p == g - 1) << 14);
        }
      }
      if (lane < ((Gn + 3) & ~3) - Gn) gk[Gn + lane] = 0u;  // pads: never above a key
      __syncwarp();
      // rank of each step = #steps with a larger key (step rk turns member rk into member rk + 1)
      const int Gp = (Gn + 3) & ~3;
#pragma unroll 1
      for (int e = lane; e - lane < Gn; e += 32) {
        const unsigned key = e < Gn ? gk[e] : 0xFFFFFFFFu;
        const int c = count_le(gk, 0, Gp, key);
        if (e < Gn) rnk[e] = Gp - c;
      }
    } else {
      seq_elements<NC>(info, gk, ginfo, rnk, Gn, lane);
    }
  }
  __syncwarp();
  // per step: member rk's longest time, member rk + 1's count and area deltas
  unsigned long long gent = 0;  // growth entries per size (packed)
#pragma unroll 1
  for (int e = lane; e < Gn; e += 32) {
    const uint32_t gi = ginfo[e];
    const int j = (int)(gi & 255u), c = (int)((gi >> 8) & 7u), ct = (int)((gi >> 11) & 7u);
    const int rk = rnk[e];
    const int tf = T[j * NC + c], tt = T[j * NC + ct];
    lbh[rk] = tf;
    cnts[rk + 1] = (1ull << (11 * ct)) - (1ull << (11 * c));
    lbs[rk + 1] = (unsigned)size_of<NC>(ct) * (unsigned)tt - (unsigned)size_of<NC>(c) * (unsigned)tf;
    gent += 1ull << (11 * ct);
  }
  if (lane == 0) {
    lbh[Gn] = (int)tlast;
    cnts[0] = c0;
    lbs[0] = W;
  }
  gent = (unsigned long long)warp_sum_ll((long long)gent);
  __syncwarp();
  // prefix sums over members: packed size counts and area; lower bound max(h_k, ceil(W_k / #slices))
  {
    unsigned long long cc = 0;
    unsigned ww = 0;
    int* gl = P.ws_lb + inst * (int64_t)P.ws_kcap;
    unsigned long long* gcn = P.ws_cnt + inst * (int64_t)P.ws_kcap;
#pragma unroll 1
    for (int k0 = 0; k0 < K; k0 += 32) {
      const int k = k0 + lane;
      unsigned long long dc = k < K ? cnts[k] : 0;
      unsigned dw = k < K ? lbs[k] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long yc = __shfl_up_sync(FULL, dc, o);
        const unsigned yw = __shfl_up_sync(FULL, dw, o);
        if (lane >= o) { dc += yc; dw += yw; }
      }
      if (k < K) {
        gcn[k] = cc + dc;
        gl[k] = max(lbh[k], (int)((ww + dw + (unsigned)(S - 1)) / (unsigned)S));
      }
      cc += __shfl_sync(FULL, dc, 31);
      ww += __shfl_sync(FULL, dw, 31);
    }
    if (K + lane < ((K + 3) & ~3)) gl[K + lane] = INT_MAX;  // row padding (16-B loads in member0)
  }

  // ---- H3: every list entry -- the a^1 entry of each task and one growth entry per step (at the
  //      size it enters) -- keyed size << 29 | (2^22 - 1 - t) << 7 | task: one sort gives the per-size
  //      LPT lists (-t, task) concatenated in size order, i.e. the workspace layout
  {
    unsigned v[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = lane + 32 * q;
      v[q] = 0xFFFFFFFFu;
      if (j < n) {
        const int c = (int)(info[j] & 7u);
        v[q] = ((unsigned)c << 29) | ((unsigned)(0x3FFFFF - T[j * NC + c]) << 7) | (unsigned)j;
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = lane + 32 * q;
      v[4 + q] = 0xFFFFFFFFu;
      if (e < Gn) {
        const uint32_t gi = ginfo[e];
        const int j = (int)(gi & 255u), ct = (int)((gi >> 11) & 7u);
        v[4 + q] = ((unsigned)ct << 29) | ((unsigned)(0x3FFFFF - T[j * NC + ct]) << 7) | (unsigned)j;
      }
    }
    warp_sort256(v, lane);
    *(uint4*)(kk + lane * 8) = make_uint4(v[0], v[1], v[2], v[3]);  // sorted order, blocked
    *(uint4*)(kk + lane * 8 + 4) = make_uint4(v[4], v[5], v[6], v[7]);
  }
  __syncwarp();
  // ---- outputs: ws_ent[i] = {t | task << 22, lo | hi << 16} (member interval of the entry), the a^1
  //      entries again, in the same order, as member 0's compact lists
  const int E = n + Gn;
  int2* ge = P.ws_ent + inst * (int64_t)P.ws_ecap1;
  uint32_t* gm = P.ws_m0 + inst * (int64_t)P.ws_n4;
  // entry i (lane-strided): chain position p of its size in its task's chain (0 for the a^1
  // entry), member interval [lo, hi) = [p ? rank of step p-1 + 1 : 0, p < g ? rank of step p + 1 : K),
  // computed branch-free (both rank loads issued), stores through running pointers
  int2* gep = ge + lane;
  uint32_t* gmp = gm;
#pragma unroll 1
  for (int i = lane; i - lane < E; i += 32, gep += 32) {
    const bool valid = i < E;
    const unsigned key = valid ? kk[i] : 0u;
    const int c = (int)(key >> 29), j = (int)(key & 127u);
    const unsigned tj = ((0x3FFFFFu - ((key >> 7) & 0x3FFFFFu)) | ((unsigned)j << 22));
    const uint32_t w = info[j];
    const int g = (int)((w >> 8) & 7u), first = (int)(w >> 11);
    const bool a1 = valid && c == (int)(w & 7u);
    const int p = a1 ? 0 : __popc(((w >> 3) & 31u) & ((1u << c) - 1u));
    const int rlo = rnk[max(first + p - 1, 0)], rhi = rnk[first + p];
    const int lo = p ? rlo + 1 : 0, hi = p < g ? rhi + 1 : K;
    if (valid) *gep = make_int2((int)tj, lo | (hi << 16));
    const unsigned b = __ballot_sync(FULL, a1);
    if (a1) gmp[__popc(b & lt)] = tj;
    gmp += __popc(b);
  }
  // list offsets per size (meta[0..NC]) from the member-0 and growth counts
  {
    int lv = 0, eo = 0;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      if (lane == c) lv = eo;
      eo += fld11(c0, c) + fld11(gent, c);
    }
    if (lane == NC) lv = eo;
    if (lane <= NC) meta[lane] = lv;
  }
  if (lane == 0) {
    ge[E] = make_int2(0, 0xFFFF);  // padding entry (never a member)
    meta[WS_K] = K;
    meta[WS_FLAG] = 0;
  }
}

template <int NC, bool MONO>
__device__ __forceinline__ void prep_instance(const KParams& P, int64_t inst, unsigned char* wsm, const PLayout& L,
                                           int lane, unsigned bar, unsigned& phase) {
  constexpr int S = Tree<NC>::S;
  const int n = P.n;
  int32_t* T = (int32_t*)(wsm + L.T);
  uint32_t* info = (uint32_t*)(wsm + L.info);  // a^1 | chain mask << 3 | #steps << 8 | first step << 11
  unsigned* gk = (unsigned*)(wsm + L.gk);
  uint32_t* ginfo = (uint32_t*)(wsm + L.ginfo);  // task | from << 8 | to << 11 | last-of-task << 14
  int* rnk = (int*)(wsm + L.rnk);
  unsigned long long* cnts = (unsigned long long*)(wsm + L.cnts);
  unsigned* lbs = (unsigned*)(wsm + L.lbs);
  int* lbh = (int*)(wsm + L.lbh);
  unsigned* kk = (unsigned*)(wsm + L.kk);
  int* meta = P.ws_meta + inst * 16;
  const unsigned lt = (1u << lane) - 1u;

  // ---- H0
  {
    const int cntT = n * NC;
    const int32_t* src = P.times + inst * (int64_t)cntT;
    if (FAR_PREP_TMA && (((uintptr_t)src) & 15) == 0 && (cntT & 3) == 0) {
      // one TMA bulk copy of the whole table (global -> this warp's T), issued by lane 0 on the
      // warp's mbarrier; the table's generic reads of the previous instance are ordered first
      if (lane == 0) {
        const unsigned bytes = 4u * (unsigned)cntT;
        const unsigned dst = (unsigned)__cvta_generic_to_shared(T);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                     "l"(src), "r"(bytes), "r"(bar)
                     : "memory");
      }
      unsigned done = 0;
      while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(phase)
            : "memory");
      }
      phase ^= 1u;
    } else if ((((uintptr_t)src) & 15) == 0) {
      const int n4 = cntT >> 2;
      const int4* s4 = (const int4*)src;
      int4* d4 = (int4*)T;
      for (int q = lane; q < n4; q += 32) d4[q] = __ldcs(s4 + q);
      for (int q = (n4 << 2) + lane; q < cntT; q += 32) T[q] = __ldcs(src + q);
    } else {
      for (int q = lane; q < cntT; q += 32) T[q] = __ldcs(src + q);
    }
  }
  __syncwarp();

  // ---- H1: a^1, chains, member-0 counts and area, input checks
  int bad = 0, mono = 1;
  long long bsum = 0;
  int tmax = 0;
  unsigned W = 0, tstar = 0;
  unsigned long long c0 = 0;
  uint32_t* d0 = P.ws_d0 + inst * (int64_t)P.ws_n4;
#pragma unroll 1
  for (int j = lane; j < n; j += 32) {
    int tv[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) tv[c] = T[j * NC + c];
    int mx = tv[0], mn = tv[0];
#pragma unroll
    for (int c = 1; c < NC; ++c) {
      mx = max(mx, tv[c]);
      mn = min(mn, tv[c]);
    }
    bad |= mn < 1;
    bsum += mx;
    tmax = max(tmax, mx);
    // 32-bit products: meaningful once t < 2^22 is established (checked below).
    // The growth chain a^1 -> nx(a^1) -> ... (nx(c) = argmin_{c' > c} (size(c') t(c'), c')) is the
    // set of suffix-minimum positions of w_c = size(c) t(c): c is on it iff w_c <= w_c'' for every
    // c'' > c (ties -> smallest index, as in nx), and a^1 (the first minimum) is its lowest element.
    // One downward pass gives the chain mask, a^1, its work and duration, and the monotonicity of t
    // along the chain.
    unsigned cb = 1u << (NC - 1);
    unsigned bw = (unsigned)size_of<NC>(NC - 1) * (unsigned)tv[NC - 1];
    int tb = tv[NC - 1];
#pragma unroll
    for (int c = NC - 2; c >= 0; --c) {
      const unsigned wc = (unsigned)size_of<NC>(c) * (unsigned)tv[c];
      if (wc <= bw) {
        bw = wc;
        cb |= 1u << c;
        mono &= tv[c] >= tb;
        tb = tv[c];
      }
    }
    const int best = __ffs(cb) - 1;
    tstar = max(tstar, growth_key<NC>(tv[NC - 1], j, __popc(cb) - 1));
    W += bw;
    c0 += 1ull << (11 * best);
    d0[j] = (uint32_t)tb;  // t_j(a^1_j): member 0's duration (finish, k* = 0)
    info[j] = (uint32_t)best | (cb << 3);
  }
  bad = __any_sync(FULL, bad);
  bsum = warp_sum_ll(bsum);
  if (bad || bsum + P.rsum >= BOUND) {
    if (lane == 0) {
      far_result R0;
      R0.makespan = -1; R0.makespan_phase2 = 0; R0.alloc_index = 0; R0.family_size = 0;
      R0.moves = 0; R0.swaps = 0; R0.iterations = 0; R0.reverted = 0; R0.status = FAR_E_BAD_TIME; R0.reserved = 0;
      R0.evals = 0; R0.events = 0;
      P.makespan[inst] = -1;
      if (P.res) P.res[inst] = R0;
      atomicOr(P.errflag, 1);
      meta[WS_FLAG] = 1;
    }
    return;
  }
  tmax = __reduce_max_sync(FULL, tmax);
  auto defer = [&]() {  // outside this kernel's domain: the fused kernel solves it (overflow pass)
    if (lane == 0) {
      atomicOr(P.ovf + (inst >> 5), 1u << (inst & 31));
      atomicAdd(P.ovf_count, 1ull);
      meta[WS_FLAG] = 1;
    }
  };
  if (tmax >= (1 << 22)) {
    defer();
    return;
  }
  const bool allmono = __all_sync(FULL, mono);
  tstar = __reduce_max_sync(FULL, tstar);
  W = __reduce_add_sync(FULL, W);
  c0 = (unsigned long long)warp_sum_ll((long long)c0);
  if (MONO) {
    if (!allmono) {  // the general prep kernel (next launch) takes it
      if (lane == 0) {
        P.gen_list[atomicAdd(P.gen_count, 1ull)] = inst;
        meta[WS_FLAG] = 1;
      }
      return;
    }
    prep_rest<NC, true>(P, inst, wsm, L, lane, tstar, W, c0);
  } else {
    prep_rest<NC, false>(P, inst, wsm, L, lane, tstar, W, c0);
  }
}

// MONO = true: every instance (the monotone merge form of H2); instances with a chain along which
// t increases are appended to P.gen_list.  MONO = false: the instances of P.gen_list, with the
// step-by-step H2 (a separate, normally empty launch keeps that code out of the hot kernel's
// instruction-cache footprint).
template <int NC, bool MONO>
__global__ void __launch_bounds__(128, 8) far_prep_kernel(KParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const PLayout L = make_playout(P.n, NC, P.kcap);
  unsigned char* wsm = smem + (size_t)warp * L.bytes;
  __shared__ __align__(8) unsigned long long tbar[4];  // one mbarrier per warp (blocks of 128)
  const unsigned bar = (unsigned)__cvta_generic_to_shared(&tbar[warp]);
  unsigned phase = 0;
  if (FAR_PREP_TMA && lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncwarp();
  const int64_t total = MONO ? P.I : (int64_t)*(volatile unsigned long long*)P.gen_count;
  // dynamic instance scheduler, next index claimed one instance ahead
  unsigned long long nxt = 0;
  if (lane == 0) nxt = atomicAdd(P.counter, 1ull);
  for (;;) {
    const unsigned long long it = __shfl_sync(FULL, nxt, 0);
    if ((int64_t)it >= total) break;
    if (lane == 0) nxt = atomicAdd(P.counter, 1ull);
    prep_instance<NC, MONO>(P, MONO ? (int64_t)it : P.gen_list[it], wsm, L, lane, bar, phase);
    __syncwarp();
  }
}

}  // namespace farb
