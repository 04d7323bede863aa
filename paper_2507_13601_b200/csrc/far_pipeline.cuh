// far_pipeline.cuh — phase 2 (Alg. 1 over the family) at lane granularity.
//
// The fused kernel gives each instance one warp and each family member one lane, so a warp
// always pays a full 32-lane pass although, on realistic inputs, the exact lower bound
// max(h_k, ceil(W_k / #slices)) (far_kernel.cuh H2) rules out almost every member once one
// member's makespan is known (k* = 0 on ~90 % of M5 instances).  The pipelined solver
// therefore splits the solve into
//   K1 far_solve_kernel PIPE_PREP    warp / instance: H0-H3, lists + family -> workspace
//   K2 far_member0_kernel            lane / instance: Alg. 1 for member 0 (recorded), then the
//                                    members whose (LB_k, k) is below (ms_0, 0) become items
//   K3 far_members_kernel            lane / item (instance, member): Alg. 1, atomicMin of
//                                    (makespan << 16 | k) per instance -- argmin (makespan, k)
//   K4 far_winner_kernel             lane / instance: re-runs k* when k* != 0, recording it
//   K5 far_finish_kernel             warp / instance: H6-H7 from the record (compact layout:
//                                    node lists + durations, no runtime table in smem)
// Every lane does useful work, and an instance costs ~1 + (candidates) member simulations
// instead of a 32-lane pass.  The result is identical to the fused kernel's (same readings,
// same tie-breaks: the packed key orders (makespan, k) lexicographically).
#pragma once
#include "far_kernel.cuh"

namespace farb {

__device__ __forceinline__ unsigned long long best_key(int ms, int k) {
  return ((unsigned long long)(unsigned)ms << 16) | (unsigned)k;
}

// Alg. 1 for member k of one instance on ONE thread.  ent: the instance's per-size LPT lists
// (global, read-only), absolute cursors; st: this thread's [NC] cursor words in shared memory
// (stride bdim); with REC the placement of every task is recorded (node | size << 4 |
// position-in-node << 7) and the slice ends are returned.
template <int NC, bool REC>
__device__ int sim_member(const int2* __restrict__ ent, const int* loff, unsigned long long cp, int k,
                          const uint32_t* ninfo, const int* cr, const int* de, uint32_t* st, uint16_t* npos,
                          int bdim, uint32_t* rec, int* sl_out, int& pops) {
  constexpr int S = Tree<NC>::S, NN = Tree<NC>::NN;
  // the list base stays in a register (otherwise it is rematerialised from the 64-bit instance
  // offset at every placement: 6 instructions instead of 1)
  asm volatile("" : "+l"(ent));
  int total = 0;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int r = (int)((cp >> (11 * c)) & 2047);
    st[c * bdim] = ((uint32_t)r << 16) | (uint32_t)loff[c];
    total += r;
  }
  if (REC)
    for (int v = 0; v < NN; ++v) npos[v * bdim] = 0;
  SFrontier<S> F;
  F.init();
  int rec_end = 0, ms = 0;
  int sl[S];
#pragma unroll
  for (int s = 0; s < S; ++s) sl[s] = 0;
  while (total > 0) {
    int bs, be;
    F.pop(bs, be);
    const int v = F.node(bs);
    int c = node_c0<NC>(v);
    uint32_t sv = st[c * bdim];
    if (!(sv >> 16)) {
      c = node_c1<NC>(v);
      sv = 0;
      if (c != NONE) sv = st[c * bdim];
    }
    ++pops;
    if (sv >> 16) {
      if (!((F.has >> bs) & 1)) {
        rec_end = max(rec_end, be) + cr[node_szi<NC>(v)];
        be = rec_end;
        F.has |= 1u << bs;
      }
      int p = (int)(sv & 0xFFFFu);
      int2 e;
      for (;;) {
        const int2 e0 = __ldg(ent + p), e1 = __ldg(ent + p + 1);
        if ((e0.y & 0xFFFF) <= k && k < (int)((unsigned)e0.y >> 16)) { e = e0; p += 1; break; }
        if ((e1.y & 0xFFFF) <= k && k < (int)((unsigned)e1.y >> 16)) { e = e1; p += 2; break; }
        p += 2;
      }
      if (REC) {
        const int task = (int)((unsigned)e.x >> 22);
        const int pos = npos[v * bdim];
        npos[v * bdim] = (uint16_t)(pos + 1);
        rec[task] = (uint32_t)v | ((uint32_t)c << 4) | ((uint32_t)pos << 7);
      }
      st[c * bdim] = ((sv & 0xFFFF0000u) - 0x10000u) | (uint32_t)p;
      be += e.x & 0x3FFFFF;
      ms = max(ms, be);
      --total;
      F.set_front(bs, be);
    } else {
      const uint32_t w = ninfo[v];
      if ((F.has >> bs) & 1) rec_end = max(rec_end, be) + de[nd_szi(w)];
      if (!F.split(bs, be, w)) {
#pragma unroll
        for (int s = 0; s < S; ++s) sl[s] = (s == bs) ? be : sl[s];
      }
    }
  }
  pops += __popc(F.live);
  if (REC) {
#pragma unroll
    for (int s = 0; s < S; ++s)
      if ((F.live >> s) & 1) {
        const int sz = nd_sz(ninfo[F.node(s)]);
#pragma unroll
        for (int q = 0; q < S; ++q) sl[q] = (q >= s && q < s + sz) ? F.endv(s) : sl[q];
      }
#pragma unroll
    for (int s = 0; s < S; ++s) sl_out[s] = sl[s];
  }
  return ms;
}

// Alg. 1 for member 0 from its compact per-size LPT lists: row = this thread's shared-memory
// copy of the a^1 entries (t | task << 22), size c's list at offset sum_{c' < c} count_c'.
// No other member's entries interleave, so every placement is one shared-memory load.
template <int NC>
__device__ int sim_member0(const uint32_t* row, unsigned long long cp, const uint32_t* ninfo, const int* cr,
                           const int* de, uint32_t* st, uint16_t* npos, int bdim, uint32_t* rec, int* sl_out,
                           int& pops) {
  constexpr int S = Tree<NC>::S, NN = Tree<NC>::NN;
  int total = 0;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int r = (int)((cp >> (11 * c)) & 2047);
    st[c * bdim] = ((uint32_t)r << 16) | (uint32_t)total;
    total += r;
  }
  for (int v = 0; v < NN; ++v) npos[v * bdim] = 0;
  SFrontier<S> F;
  F.init();
  int rec_end = 0, ms = 0;
  int sl[S];
#pragma unroll
  for (int s = 0; s < S; ++s) sl[s] = 0;
  while (total > 0) {
    int bs, be;
    F.pop(bs, be);
    const int v = F.node(bs);
    int c = node_c0<NC>(v);
    uint32_t sv = st[c * bdim];
    if (!(sv >> 16)) {
      c = node_c1<NC>(v);
      sv = 0;
      if (c != NONE) sv = st[c * bdim];
    }
    ++pops;
    if (sv >> 16) {
      if (!((F.has >> bs) & 1)) {
        rec_end = max(rec_end, be) + cr[node_szi<NC>(v)];
        be = rec_end;
        F.has |= 1u << bs;
      }
      const int p = (int)(sv & 0xFFFFu);
      const uint32_t x = row[p];
      const int task = (int)(x >> 22);
      const int pos = npos[v * bdim];
      npos[v * bdim] = (uint16_t)(pos + 1);
      rec[task] = (uint32_t)v | ((uint32_t)c << 4) | ((uint32_t)pos << 7);
      st[c * bdim] = sv - 0x10000u + 1u;
      be += (int)(x & 0x3FFFFFu);
      ms = max(ms, be);
      --total;
      F.set_front(bs, be);
    } else {
      const uint32_t w = ninfo[v];
      if ((F.has >> bs) & 1) rec_end = max(rec_end, be) + de[nd_szi(w)];
      if (!F.split(bs, be, w)) {
#pragma unroll
        for (int s = 0; s < S; ++s) sl[s] = (s == bs) ? be : sl[s];
      }
    }
  }
  pops += __popc(F.live);
#pragma unroll
  for (int s = 0; s < S; ++s)
    if ((F.live >> s) & 1) {
      const int sz = nd_sz(ninfo[F.node(s)]);
#pragma unroll
      for (int q = 0; q < S; ++q) sl[q] = (q >= s && q < s + sz) ? F.endv(s) : sl[q];
    }
#pragma unroll
  for (int s = 0; s < S; ++s) sl_out[s] = sl[s];
  return ms;
}

struct PParams {
  int64_t I;
  int n;
  int cr[8], de[8];
  unsigned flags;
  int2* ws_ent;
  int* ws_lb;
  unsigned long long* ws_cnt;
  int* ws_meta;
  unsigned long long* ws_best;
  unsigned long long* ws_evt;
  uint32_t* ws_rec;
  int* ws_sl;
  int ws_ecap1, ws_kcap;
  const uint32_t* ws_m0;        // [I][n4] member 0's compact per-size LPT lists (t | task << 22)
  int ws_n4;
  uint16_t* ws_ncnt;            // [I][16] node list lengths of the recorded member
  int2* items;                  // (instance, member) work items of K3
  unsigned long long* nitems;   // item counter
  unsigned long long* counter;  // K2 batch counter
  unsigned long long* counter2; // K3 item batch counter
};

template <int NC> struct PipeSmem {
  uint32_t ninfo[16];
  int cr[8], de[8];
};

template <int NC>
__device__ __forceinline__ void pipe_prologue(const PParams& P, PipeSmem<NC>& sm) {
  constexpr int NN = Tree<NC>::NN;
  if (threadIdx.x < NN) sm.ninfo[threadIdx.x] = (NC == 3) ? c_nodes3[threadIdx.x] : c_nodes5[threadIdx.x];
  if (threadIdx.x < 8) {
    sm.cr[threadIdx.x] = P.cr[threadIdx.x];
    sm.de[threadIdx.x] = P.de[threadIdx.x];
  }
  __syncthreads();
}

#ifndef FAR_M0_TMA
#define FAR_M0_TMA 1  // member0 stages its lists with TMA bulk copies
#endif

// K2: member 0 of every pending instance (recorded), then the candidate members as items.
template <int NC>
__global__ void __launch_bounds__(128) far_member0_kernel(PParams P) {
  constexpr int NN = Tree<NC>::NN;
  __shared__ PipeSmem<NC> sm;
  extern __shared__ __align__(16) unsigned char dsm[];
  pipe_prologue<NC>(P, sm);
  const int bdim = blockDim.x, tid = threadIdx.x;
  uint32_t* st = (uint32_t*)dsm + tid;
  uint16_t* npos = (uint16_t*)(dsm + 4 * NC * bdim) + tid;
  // this thread's copy of member 0's lists.  FAR_M0_TMA: row stride n4 + 4 words (16-B aligned rows,
  // filled by TMA bulk copies); otherwise n4 + 1 (odd: the rows of a warp start in 32 different banks)
#if FAR_M0_TMA
  const int nw = P.ws_n4, rs = nw + 4, lane = tid & 31;
  __shared__ __align__(8) unsigned long long m0bar[4];  // one mbarrier per warp (blocks of <= 128)
  const unsigned bar = (unsigned)__cvta_generic_to_shared(&m0bar[tid >> 5]);
  unsigned phase = 0;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncwarp();
#else
  const int nw = P.ws_n4, rs = nw + 1, lane = tid & 31;
#endif
  uint32_t* wrows = (uint32_t*)(dsm + (4 * NC + 2 * NN) * bdim) + (size_t)(tid & ~31) * rs;
  uint32_t* row = wrows + (size_t)lane * rs;
  const bool exhaustive = (P.flags & FAR_EXHAUSTIVE) != 0;
  // the lanes of a warp hold 32 consecutive instances and step together (the list staging is
  // warp-cooperative); batches of 32 are claimed from a counter, one ahead
  // (a grid that covers every instance in one pass takes its batch by position: no atomics)
  const bool one_pass = (int64_t)gridDim.x * blockDim.x >= P.I;
  unsigned long long nb = (unsigned long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
  if (!one_pass && lane == 0) nb = atomicAdd(P.counter, 32ull);
  for (;;) {
    const int64_t base = (int64_t)__shfl_sync(FULL, nb, 0);
    if (base >= P.I) break;
    if (one_pass) nb = (unsigned long long)P.I;
    else if (lane == 0) nb = atomicAdd(P.counter, 32ull);
    const int64_t i = base + lane;
    const bool active = i < P.I && !P.ws_meta[i * 16 + WS_FLAG];
    __syncwarp();  // every lane is done with its row (previous instance)
#if FAR_M0_TMA
    {  // lane 0 issues one TMA bulk copy per active instance (its whole member-0 list row, global ->
       // this warp's rows) on the warp's mbarrier; every lane waits for the transaction bytes
      const unsigned am = __ballot_sync(FULL, active);
      if (am) {
        if (lane == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the rows' generic reads first
          const unsigned bytes = 4u * (unsigned)nw;
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes * __popc(am))
                       : "memory");
          const uint32_t* src0 = P.ws_m0 + (i - lane) * (int64_t)nw;
          for (unsigned m = am; m; m &= m - 1) {
            const int u = __ffs(m) - 1;
            const unsigned dst = (unsigned)__cvta_generic_to_shared(wrows + (size_t)u * rs);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                "l"(src0 + (int64_t)u * nw), "r"(bytes), "r"(bar)
                : "memory");
          }
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
      }
    }
#else
    {  // the warp copies its instances' lists: coalesced 128-B loads, eight instances' loads in
       // flight per lane (one exposed latency per eight instances), conflict-free stores into the rows
      const uint32_t* src = P.ws_m0 + (i - lane) * (int64_t)nw;
      for (unsigned am = __ballot_sync(FULL, active); am;) {
        int ids[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          ids[u] = am ? __ffs(am) - 1 : -1;
          am &= am - 1;
        }
        for (int w0 = 0; w0 < nw; w0 += 128) {
          uint32_t x[8][4];
#pragma unroll
          for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const int w = w0 + 32 * v + lane;
              x[u][v] = (ids[u] >= 0 && w < nw) ? __ldcs(src + (int64_t)ids[u] * nw + w) : 0u;
            }
#pragma unroll
          for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const int w = w0 + 32 * v + lane;
              if (ids[u] >= 0 && w < nw) wrows[(size_t)ids[u] * rs + w] = x[u][v];
            }
        }
      }
      __syncwarp();
    }
#endif
    int K = 0, ms0 = 0;
    const int* lb = P.ws_lb + i * (int64_t)P.ws_kcap;
    if (active) {
      K = P.ws_meta[i * 16 + WS_K];
      int pops = 0;
      ms0 = sim_member0<NC>(row, P.ws_cnt[i * (int64_t)P.ws_kcap], sm.ninfo, sm.cr, sm.de, st, npos, bdim,
                            P.ws_rec + i * (int64_t)P.n, P.ws_sl + i * 8, pops);
      for (int v = 0; v < NN; ++v) P.ws_ncnt[i * 16 + v] = npos[v * bdim];
      P.ws_best[i] = best_key(ms0, 0);
      P.ws_evt[i] = (unsigned long long)pops;
    }
    // members that can still beat (ms_0, 0): (LB_k, k) < (ms_0, 0) lexicographically, i.e.
    // LB_k < ms_0 (k >= 1).  32 members per chunk: 16-B loads (ws_kcap is a multiple of 4), a bit
    // per candidate; the warp's candidates of a chunk take one atomic (lane offsets by a warp scan),
    // each lane's items stay consecutive
    const int Kw = __reduce_max_sync(FULL, (unsigned)K);
    for (int k0 = 0; k0 < Kw; k0 += 32) {
      unsigned mask = 0;
      if (k0 < K) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (k0 + 4 * u < K) {
            const int4 x = __ldg((const int4*)(lb + k0) + u);
            mask |= (unsigned)(exhaustive || x.x < ms0) << (4 * u);
            mask |= (unsigned)(exhaustive || x.y < ms0) << (4 * u + 1);
            mask |= (unsigned)(exhaustive || x.z < ms0) << (4 * u + 2);
            mask |= (unsigned)(exhaustive || x.w < ms0) << (4 * u + 3);
          }
        }
        if (k0 == 0) mask &= ~1u;                                // member 0 itself
        if (K - k0 < 32) mask &= (1u << (K - k0)) - 1u;         // past the family
      }
      const int cnt = __popc(mask);
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
      const int tot = __shfl_sync(FULL, incl, 31);
      if (tot == 0) continue;
      unsigned long long slot = 0;
      if (lane == 31) slot = atomicAdd(P.nitems, (unsigned long long)tot);
      slot = __shfl_sync(FULL, slot, 31) + (unsigned long long)(incl - cnt);
      for (; mask; mask &= mask - 1) P.items[slot++] = make_int2((int)i, k0 + __ffs(mask) - 1);
    }
  }
  (void)NN;
}

// K3: the candidate members (lane per item), pruned again against the instance's current best.
template <int NC>
__global__ void __launch_bounds__(128) far_members_kernel(PParams P) {
  __shared__ PipeSmem<NC> sm;
  extern __shared__ __align__(16) unsigned char dsm[];
  pipe_prologue<NC>(P, sm);
  const int bdim = blockDim.x, tid = threadIdx.x;
  uint32_t* st = (uint32_t*)dsm + tid;
  const bool exhaustive = (P.flags & FAR_EXHAUSTIVE) != 0;
  const unsigned long long nit = *(volatile unsigned long long*)P.nitems;
  // batches of 32 consecutive items claimed per warp from a counter, one ahead (the items' costs
  // differ: a pruned item is a few loads, a simulated one ~n + #nodes events)
  const int lane = tid & 31;
  // The batches are whole rounds of the warps (a lane per item).  When the items need between one
  // and two rounds of the grid (few instances, e.g. a rank's 125k-instance shard of config 5 at
  // N = 8), they are split evenly over the fewest warps that take two batches each and the other
  // warps exit: measured on M5 125k, members 0.315 -> 0.258 ms; at three or more rounds the full
  // grid with dynamic claiming is faster (250k: 0.383 against 0.456 ms), so it is kept there.
  if (!(P.flags & FAR_I_NO_ROUND_BALANCE)) {
    const unsigned long long nbt = (nit + 31) / 32, W = (unsigned long long)gridDim.x * (bdim >> 5);
    const unsigned long long wid = (unsigned long long)blockIdx.x * (bdim >> 5) + (tid >> 5);
    if (nbt > W && nbt <= 2 * W && wid >= (nbt + 1) / 2) return;
  }
  unsigned long long nb = 0;
  if (lane == 0) nb = atomicAdd(P.counter2, 32ull);
  for (;;) {
    const unsigned long long b0 = __shfl_sync(FULL, nb, 0);
    if (b0 >= nit) break;
    if (lane == 0) nb = atomicAdd(P.counter2, 32ull);
    const unsigned long long it = b0 + lane;
    if (it >= nit) continue;
    const int2 item = P.items[it];
    const int64_t i = item.x;
    const int k = item.y;
    const int lbk = P.ws_lb[i * (int64_t)P.ws_kcap + k];
    if (!exhaustive && best_key(lbk, k) >= *(volatile unsigned long long*)(P.ws_best + i)) continue;
    const int* meta = P.ws_meta + i * 16;
    int loff[NC + 1];
#pragma unroll
    for (int c = 0; c <= NC; ++c) loff[c] = meta[c];
    int pops = 0;
    const int ms = sim_member<NC, false>(P.ws_ent + i * (int64_t)P.ws_ecap1, loff,
                                         P.ws_cnt[i * (int64_t)P.ws_kcap + k], k, sm.ninfo, sm.cr, sm.de, st,
                                         nullptr, bdim, nullptr, nullptr, pops);
    atomicMin(P.ws_best + i, best_key(ms, k));
    atomicAdd(P.ws_evt + i, (unsigned long long)pops);
  }
}

// K4: re-run the winner when it is not member 0, recording its placements.
template <int NC>
__global__ void __launch_bounds__(128) far_winner_kernel(PParams P) {
  constexpr int NN = Tree<NC>::NN;
  __shared__ PipeSmem<NC> sm;
  __shared__ int64_t queue[4][64];  // per warp: instances whose winner is not member 0
  extern __shared__ __align__(16) unsigned char dsm[];
  pipe_prologue<NC>(P, sm);
  const int bdim = blockDim.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t* st = (uint32_t*)dsm + tid;
  uint16_t* npos = (uint16_t*)(dsm + 4 * NC * bdim) + tid;
  int64_t* q = queue[warp];
  // ~10 % of the instances have k* != 0: each warp scans 32 instances at a time and compacts
  // them into its queue, so that the re-simulations run with every lane busy
  auto resim = [&](int64_t i) {
    const int* meta = P.ws_meta + i * 16;
    const int k = (int)(P.ws_best[i] & 0xFFFFu);
    int loff[NC + 1];
#pragma unroll
    for (int c = 0; c <= NC; ++c) loff[c] = meta[c];
    int pops = 0;
    sim_member<NC, true>(P.ws_ent + i * (int64_t)P.ws_ecap1, loff, P.ws_cnt[i * (int64_t)P.ws_kcap + k], k,
                         sm.ninfo, sm.cr, sm.de, st, npos, bdim, P.ws_rec + i * (int64_t)P.n, P.ws_sl + i * 8, pops);
    for (int v = 0; v < NN; ++v) P.ws_ncnt[i * 16 + v] = npos[v * bdim];
  };
  int count = 0;
  const int64_t nwarps = (int64_t)gridDim.x * (bdim >> 5);
  for (int64_t base = ((int64_t)blockIdx.x * (bdim >> 5) + warp) * 32; base < P.I; base += nwarps * 32) {
    const int64_t i = base + lane;
    bool need = false;
    if (i < P.I && !P.ws_meta[i * 16 + WS_FLAG]) need = (P.ws_best[i] & 0xFFFFu) != 0;
    const unsigned bal = __ballot_sync(FULL, need);
    if (need) q[count + __popc(bal & ((1u << lane) - 1))] = i;
    count += __popc(bal);
    __syncwarp();
    if (count >= 32) {
      resim(q[lane]);
      const int64_t rest = lane + 32 < count ? q[lane + 32] : 0;
      __syncwarp();
      if (lane + 32 < count) q[lane] = rest;
      count -= 32;
      __syncwarp();
    }
  }
  if (lane < count) resim(q[lane]);
}

// ---------------------------------------------------------------------------
// K5: H6/H7 per instance (warp) from the record of k*.  Per-warp shared memory holds only
// what phase 3 and the replay touch: node lists [NN][n] u16, durations D[n] (gathered from
// the global runtime table at the recorded sizes; durations never change in phase 3),
// starts, nodes, size indices and the small misc block.
// ---------------------------------------------------------------------------
struct FLayout {
  int misc, nlist, D, start, onode, su, bytes;
};
__host__ __device__ inline FLayout make_flayout(int n, int NN) {
  FLayout L;
  int o = 0;
  L.misc = o;  o = al16(o + 4 * 224);
  L.nlist = o; o = al16(o + 2 * NN * n);
  L.D = o;     o = al16(o + 4 * n);
  L.start = o; o = al16(o + 4 * n);
  L.onode = o; o = al16(o + n);
  L.su = o;    o = al16(o + n);
  L.bytes = o;
  return L;
}

template <int NC>
__global__ void __launch_bounds__(128, 8) far_finish_kernel(KParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int S = Tree<NC>::S, NN = Tree<NC>::NN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const FLayout L = make_flayout(P.n, NN);
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
  const bool want_sched = P.sched != nullptr && !(P.flags & FAR_NO_SCHEDULE);
  const bool refine = !(P.flags & FAR_NO_REFINE);
  unsigned long long nxt = 0;  // next instance claimed one ahead (atomic latency hidden)
  if (lane == 0) nxt = atomicAdd(P.counter, 1ull);
  for (;;) {
    const int64_t inst = (int64_t)__shfl_sync(FULL, nxt, 0);
    if (inst >= P.I) break;
    if (lane == 0) nxt = atomicAdd(P.counter, 1ull);
    const int* meta = P.ws_meta + inst * 16;
    if (meta[WS_FLAG]) continue;  // error / empty (K1 wrote the outputs) / deferred to the overflow pass
    const unsigned long long best = P.ws_best[inst];
    const int ms2 = (int)(best >> 16), bestk = (int)(best & 0xFFFFu);
    far_result R;
    R.makespan = 0; R.makespan_phase2 = ms2; R.alloc_index = bestk; R.family_size = meta[WS_K];
    R.moves = 0; R.swaps = 0; R.iterations = 0; R.reverted = 0; R.status = FAR_OK; R.reserved = 0;
    R.evals = 0; R.events = (long long)P.ws_evt[inst];
    if (lane < S) misc[M_BSEND + lane] = P.ws_sl[inst * 8 + lane];
    __syncwarp();
    finish_core<NC, true>(P, inst, (uint16_t*)(wsm + L.nlist), (int*)(wsm + L.D), (int*)(wsm + L.start),
                          wsm + L.onode, wsm + L.su, misc, nullptr, nullptr, nullptr, nullptr, ninfo, cr, de, lane,
                          R, ms2, bestk, want_sched, refine);
  }
}

}  // namespace farb
