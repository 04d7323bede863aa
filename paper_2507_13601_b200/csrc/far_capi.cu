// far_capi.cu — C-ABI of libfar.so (include/far.h): context, argument checks, launches,
// host-memory paths (staging + a 2-stream chunk pipeline).  No compute happens here;
// every step of FAR runs in far_kernel.cuh / far_stream.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>

#include "far_kernel.cuh"
#include "far_stream.cuh"
#include "far_pipeline.cuh"
#include "far_prep.cuh"
#include "far_finish_lane.cuh"
#include "far_check.cuh"
#include "far_forest.cuh"
#include "far_forest_check.cuh"
#include "far_peak.cuh"

using namespace farb;

namespace {
constexpr int NREC = 32, CPL = 16, RING = NREC * CPL;  // launch records; counters per launch
}  // namespace

struct far_ctx {
  int profile = 0, nc = 0, ns = 0, nn = 0;  // ns, nn: one tree
  int gpus = 1;                             // multi-target FAR: g trees
  uint2 fnodes[FMAXNN];                     // forest node table (far_forest.cuh encoding)
  uint2* d_fnodes = nullptr;
  int32_t sizes[8] = {0};
  int cr[8] = {0}, de[8] = {0};
  std::string err;
  int device = -1, sms = 0;
  unsigned long long* d_counter = nullptr;  // RING launch counters
  int64_t launch_id = 0;
  // d_errflag[0]: sticky flag of the asynchronous calls (reported and cleared by far_sync);
  // d_errflag[1]: private flag of the synchronous host-memory calls (cleared before and read
  // after each such call, so they neither consume nor misreport the asynchronous flag)
  int* d_errflag = nullptr;
  // cross-stream ordering of the context's device workspaces: every launch records an event on
  // its stream; a launch that reuses a workspace last used on ANOTHER stream waits on that event
  struct LaunchRec { cudaEvent_t ev; cudaStream_t stream; bool valid; };
  LaunchRec recs[NREC] = {};
  int64_t pws_last[2] = {-1, -1}, ovf_last[4] = {-1, -1, -1, -1}, cbuf_last = -1;
  // staging for host-memory calls
  char* d_buf = nullptr;   // staging of the synchronous host-memory calls (ctx streams)
  size_t d_buf_bytes = 0;
  char* d_cbuf = nullptr;  // per-batch schedules of far_concat_streams (caller's stream)
  size_t d_cbuf_bytes = 0;
  char* d_pws[2] = {nullptr, nullptr};  // pipelined phase-2 workspaces (ring of 2 launches)
  size_t d_pws_bytes[2] = {0, 0};
  int smem_max = 0;        // opt-in shared memory per block minus the kernels' static smem
  cudaStream_t s[2] = {nullptr, nullptr};
  bool inited = false;
  // overflow bitmasks (instances whose family exceeds the fast layout), ring of 4
  unsigned* d_ovf[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t ovf_words[4] = {0, 0, 0, 0};
  // launch-shape cache: (kernel, layout bytes) -> (warps per CTA, CTAs per SM)
  struct Shape { const void* fn; int bytes, warps, per_sm; };
  Shape shapes[16];
  int nshapes = 0;
  // diagnostics: kernel launch count, optional per-stage CUDA-event timing (ring of event sets)
  int64_t launches = 0;
  bool timing = false;
  struct EvSet { cudaEvent_t ev[10]; int stage[10]; int nev; bool created, pending; };
  static constexpr int NSETS = 32;
  EvSet tsets[NSETS] = {};
  int tnext = 0, timed = 0;
  double stage_ms[FAR_NUM_STAGES] = {0};
};

static far_status fail(far_ctx* c, far_status st, const std::string& m) {
  if (c) c->err = m;
  return st;
}

static far_status cuda_fail(far_ctx* c, cudaError_t e, const char* where) {
  return fail(c, FAR_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(call)                                              \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call);  \
  } while (0)

static far_status ensure_device(far_ctx* ctx) {
  if (ctx->inited) return FAR_OK;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(ctx, FAR_E_CUDA, "no CUDA device: libfar has no CPU fallback");
  CK(cudaGetDevice(&ctx->device));
  CK(cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, ctx->device));
  CK(cudaMalloc(&ctx->d_counter, RING * sizeof(unsigned long long)));
  CK(cudaMemset(ctx->d_counter, 0, RING * sizeof(unsigned long long)));
  CK(cudaMalloc(&ctx->d_errflag, 2 * sizeof(int)));
  CK(cudaMemset(ctx->d_errflag, 0, 2 * sizeof(int)));
  for (auto& r : ctx->recs) {
    CK(cudaEventCreateWithFlags(&r.ev, cudaEventDisableTiming));
    r.valid = false;
  }
  CK(cudaStreamCreateWithFlags(&ctx->s[0], cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&ctx->s[1], cudaStreamNonBlocking));
  // allow every kernel the full opt-in shared memory; each launch passes its own size
  int optin = 0;
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  ctx->smem_max = optin - 3072;  // minus the largest static shared memory of a kernel (2.4 KB)
  const void* fns[6] = {(const void*)far_solve_kernel<3, PIPE_NONE>, (const void*)far_solve_kernel<5, PIPE_NONE>,
                        (const void*)far_solve_kernel<3, PIPE_PREP>, (const void*)far_solve_kernel<5, PIPE_PREP>,
                        (const void*)far_stream_kernel<3>, (const void*)far_stream_kernel<5>};
  const void* pfns[6] = {(const void*)far_member0_kernel<3>, (const void*)far_member0_kernel<5>,
                         (const void*)far_members_kernel<3>, (const void*)far_members_kernel<5>,
                         (const void*)far_winner_kernel<3>, (const void*)far_winner_kernel<5>};
  for (const void* f : pfns) CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
  CK(cudaFuncSetAttribute((const void*)far_member0_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, ctx->smem_max));
  CK(cudaFuncSetAttribute((const void*)far_member0_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, ctx->smem_max));
  CK(cudaFuncSetAttribute((const void*)far_finish_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, ctx->smem_max));
  CK(cudaFuncSetAttribute((const void*)far_finish_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, ctx->smem_max));
  CK(cudaFuncSetAttribute((const void*)far_finish_lane_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, ctx->smem_max));
  CK(cudaFuncSetAttribute((const void*)far_finish_lane_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, ctx->smem_max));
  {
    const void* cf[4] = {(const void*)far_events_kernel<3>, (const void*)far_events_kernel<5>,
                         (const void*)far_validate_kernel<3>, (const void*)far_validate_kernel<5>};
    for (const void* f : cf) CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, ctx->smem_max));
  }
  for (const void* f : fns) CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, ctx->smem_max));
  {
    const void* ff[4] = {(const void*)far_forest_events_kernel<3>, (const void*)far_forest_events_kernel<5>,
                         (const void*)far_forest_validate_kernel<3>, (const void*)far_forest_validate_kernel<5>};
    for (const void* f : ff) CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, ctx->smem_max));
  }
  CK(cudaFuncSetAttribute((const void*)far_forest_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, ctx->smem_max));
  CK(cudaFuncSetAttribute((const void*)far_forest_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, ctx->smem_max));
  {
    const void* pf[4] = {(const void*)far_prep_kernel<3, true>, (const void*)far_prep_kernel<3, false>,
                         (const void*)far_prep_kernel<5, true>, (const void*)far_prep_kernel<5, false>};
    for (const void* f : pf) CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, ctx->smem_max));
  }
  if (ctx->gpus > 1) {
    CK(cudaMalloc(&ctx->d_fnodes, sizeof(uint2) * FMAXNN));
    CK(cudaMemcpy(ctx->d_fnodes, ctx->fnodes, sizeof(uint2) * ctx->nn * ctx->gpus, cudaMemcpyHostToDevice));
  }
  ctx->inited = true;
  return FAR_OK;
}

static far_status grow(far_ctx* ctx, char** buf, size_t* have, size_t bytes) {
  if (*have >= bytes) return FAR_OK;
  if (*buf) {
    CK(cudaDeviceSynchronize());  // the old buffer may still be in use by queued work
    CK(cudaFree(*buf));
    *buf = nullptr;
    *have = 0;
  }
  size_t b = std::max(bytes, (size_t)1 << 20);
  cudaError_t e = cudaMalloc(buf, b);
  if (e != cudaSuccess) return fail(ctx, FAR_E_OOM, "device workspace allocation failed");
  *have = b;
  return FAR_OK;
}
static far_status ensure_buf(far_ctx* ctx, size_t bytes) { return grow(ctx, &ctx->d_buf, &ctx->d_buf_bytes, bytes); }

// Make `stream` wait for launch q (a previous user of a workspace) when q ran on another stream.
// A ring entry overwritten by launch q + 32 is a later launch that itself waited for q (it reused
// q's counter slot), so waiting on the newer event is still sufficient.
static far_status order_after(far_ctx* ctx, int64_t q, cudaStream_t stream) {
  if (q < 0) return FAR_OK;
  far_ctx::LaunchRec& r = ctx->recs[q % NREC];
  if (r.valid && r.stream != stream) CK(cudaStreamWaitEvent(stream, r.ev, 0));
  return FAR_OK;
}
static far_status record_launch(far_ctx* ctx, int64_t id, cudaStream_t stream) {
  far_ctx::LaunchRec& r = ctx->recs[id % NREC];
  CK(cudaEventRecord(r.ev, stream));
  r.stream = stream;
  r.valid = true;
  return FAR_OK;
}

// ---- per-stage timing (far_stage_timing): one event set per solver launch, stage boundaries
static far_status t_collect(far_ctx* ctx, far_ctx::EvSet& e) {
  if (!e.pending) return FAR_OK;
  CK(cudaEventSynchronize(e.ev[e.nev - 1]));
  for (int i = 1; i < e.nev; ++i) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e.ev[i - 1], e.ev[i]));
    ctx->stage_ms[e.stage[i]] += ms;
  }
  e.pending = false;
  ++ctx->timed;
  return FAR_OK;
}
static far_status t_begin(far_ctx* ctx, cudaStream_t s, far_ctx::EvSet*& set) {
  set = nullptr;
  if (!ctx->timing) return FAR_OK;
  far_ctx::EvSet& e = ctx->tsets[ctx->tnext];
  ctx->tnext = (ctx->tnext + 1) % far_ctx::NSETS;
  far_status st = t_collect(ctx, e);
  if (st) return st;
  if (!e.created) {
    for (int i = 0; i < 10; ++i) CK(cudaEventCreate(&e.ev[i]));
    e.created = true;
  }
  e.nev = 0;
  CK(cudaEventRecord(e.ev[e.nev], s));
  e.stage[e.nev++] = -1;
  set = &e;
  return FAR_OK;
}
static far_status t_mark(far_ctx* ctx, far_ctx::EvSet* set, cudaStream_t s, int stage) {
  if (!set || set->nev >= 10) return FAR_OK;
  CK(cudaEventRecord(set->ev[set->nev], s));
  set->stage[set->nev++] = stage;
  set->pending = true;
  return FAR_OK;
}

template <int NC> static Layout layout_for(int n, int kcap) {
  return make_layout(n, NC, Tree<NC>::S, Tree<NC>::NN, kcap);
}

// Warps per CTA maximising resident warps per SM for a per-warp shared-memory footprint.
static far_status pick_shape(far_ctx* ctx, const void* fn, int bytes, int& warps, int& per_sm) {
  for (int i = 0; i < ctx->nshapes; ++i)
    if (ctx->shapes[i].fn == fn && ctx->shapes[i].bytes == bytes) {
      warps = ctx->shapes[i].warps;
      per_sm = ctx->shapes[i].per_sm;
      return FAR_OK;
    }
  int best_w = 0, best_b = 0, best_tot = 0;
  for (int w = 1; w <= 4; ++w) {
    const size_t smem = (size_t)w * bytes;
    if (smem > (size_t)ctx->smem_max) break;
    int b = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, w * 32, smem));
    if (b * w > best_tot || (b * w == best_tot && w > best_w)) { best_tot = b * w; best_w = w; best_b = b; }
  }
  if (best_w == 0) return fail(ctx, FAR_E_TOO_LARGE, "instance does not fit in shared memory");
  warps = best_w;
  per_sm = std::max(1, best_b);
  if (ctx->nshapes < 16) ctx->shapes[ctx->nshapes++] = {fn, bytes, warps, per_sm};
  return FAR_OK;
}

// One launch of the warp-per-instance kernel over I instances (or over the flagged ones).
static far_status launch_warp_kernel(far_ctx* ctx, KParams& P, cudaStream_t stream, int64_t units, int pipe) {
  const bool a30 = ctx->nc == 3;
  const void* fn = pipe == PIPE_PREP
                       ? (a30 ? (const void*)far_solve_kernel<3, PIPE_PREP> : (const void*)far_solve_kernel<5, PIPE_PREP>)
                       : (a30 ? (const void*)far_solve_kernel<3, PIPE_NONE> : (const void*)far_solve_kernel<5, PIPE_NONE>);
  Layout L = make_layout(P.n, ctx->nc, ctx->ns, ctx->nn, P.kcap, pipe);
  if (const char* pad = getenv("FAR_DEBUG_SMEM_PAD")) L.bytes += (atoi(pad) + 15) & ~15;  // occupancy experiments
  int warps = 0, per_sm = 0;
  far_status st = pick_shape(ctx, fn, L.bytes, warps, per_sm);
  if (st) return st;
  const size_t smem = (size_t)warps * L.bytes;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((units + warps - 1) / warps, (int64_t)ctx->sms * per_sm));
  if (pipe == PIPE_PREP) {
    if (a30) far_solve_kernel<3, PIPE_PREP><<<grid, warps * 32, smem, stream>>>(P);
    else far_solve_kernel<5, PIPE_PREP><<<grid, warps * 32, smem, stream>>>(P);
  } else {
    if (a30) far_solve_kernel<3, PIPE_NONE><<<grid, warps * 32, smem, stream>>>(P);
    else far_solve_kernel<5, PIPE_NONE><<<grid, warps * 32, smem, stream>>>(P);
  }
  CK(cudaGetLastError());
  ++ctx->launches;
  return FAR_OK;
}

// K1 for n <= 128 (far_prep.cuh): far_prep_kernel<NC, true> over every instance, then
// far_prep_kernel<NC, false> over the instances it listed (non-monotone chains; exits at once when
// the list is empty).  P.counter / P.gen_count: two counter slots of this launch.
static far_status launch_prep(far_ctx* ctx, KParams& P, cudaStream_t stream, unsigned long long* counter2) {
  const bool a30 = ctx->nc == 3;
  const PLayout L = make_playout(P.n, ctx->nc, P.kcap);
  for (int pass = 0; pass < 2; ++pass) {
    const void* fn = pass == 0 ? (a30 ? (const void*)far_prep_kernel<3, true> : (const void*)far_prep_kernel<5, true>)
                               : (a30 ? (const void*)far_prep_kernel<3, false> : (const void*)far_prep_kernel<5, false>);
    int warps = 0, per_sm = 0;
    far_status st = pick_shape(ctx, fn, L.bytes, warps, per_sm);
    if (st) return st;
    const size_t smem = (size_t)warps * L.bytes;
    if (const char* e = getenv("FAR_DEBUG_PREP_BPS")) per_sm = std::max(1, std::min(per_sm, atoi(e)));  // experiments
    int64_t units = pass == 0 ? P.I : std::min<int64_t>(P.I, (int64_t)ctx->sms * per_sm * warps);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((units + warps - 1) / warps, (int64_t)ctx->sms * per_sm));
    KParams Q = P;
    if (pass == 1) Q.counter = counter2;
    void* args[] = {&Q};
    CK(cudaLaunchKernel(fn, grid, warps * 32, args, smem, stream));
    ++ctx->launches;
  }
  return FAR_OK;
}

// Launch the solver for I instances on `stream`.
//   MODE_SOLVE: the pipelined solver (far_pipeline.cuh: K1 prep -> K2 member 0 -> K3 candidate
//   members -> K4 winner record -> K5 finish) for families of <= 96 members with t < 2^22,
//   then the fused kernel with the full layout over the instances K1 deferred (overflow mask).
//   FAR_FUSED_PHASE2 (debug env) forces the fused warp-per-instance kernel for everything.
//   MODE_LOCAL: the fused kernel (phase 3 only).
static far_status launch_forest(far_ctx* ctx, KParams& P, cudaStream_t stream) {
  if (!P.errflag) P.errflag = ctx->d_errflag;
  FParams F;
  F.P = P;
  F.nodes = ctx->d_fnodes;
  F.NNF = ctx->nn * ctx->gpus;
  F.SF = ctx->ns * ctx->gpus;
  const FLay L = make_flay(P.n, ctx->nc, F.NNF, F.SF);
  const int warps = (int)std::max<int64_t>(1, std::min<int64_t>(4, ctx->smem_max / L.bytes));
  const void* fn = ctx->nc == 3 ? (const void*)far_forest_kernel<3> : (const void*)far_forest_kernel<5>;
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, warps * 32, (size_t)warps * L.bytes));
  if (per_sm < 1) return fail(ctx, FAR_E_TOO_LARGE, "forest layout does not fit in shared memory");
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((P.I + warps - 1) / warps, (int64_t)ctx->sms * per_sm));
  if (ctx->nc == 3) far_forest_kernel<3><<<grid, warps * 32, (size_t)warps * L.bytes, stream>>>(F);
  else far_forest_kernel<5><<<grid, warps * 32, (size_t)warps * L.bytes, stream>>>(F);
  CK(cudaGetLastError());
  ++ctx->launches;
  return FAR_OK;
}

static far_status launch_solve(far_ctx* ctx, KParams& P, cudaStream_t stream) {
  if (P.I <= 0) return FAR_OK;
  if (ctx->gpus > 1) return launch_forest(ctx, P, stream);
  const bool a30 = ctx->nc == 3;
  const int NC = ctx->nc, NN = ctx->nn;
  const int kmax = 1 + P.n * (NC - 1);
  int kcap_fast = 96;  // M5: P(K > 64) ~ 0.4%, P(K > 96) ~ 0: larger families go to the overflow pass
  if (const char* e = getenv("FAR_DEBUG_KFAST")) kcap_fast = std::max(2, std::min(254, atoi(e)));  // experiments (8-bit intervals)
  int kfast = std::min(kmax, kcap_fast);
  if (P.mode != MODE_SOLVE) kfast = 1;
  // small batches (latency): the fused warp-per-instance kernel is one launch instead of five
  // (the reading variant FAR_SWITCH_COST runs the fused kernel only)
  const bool pipe = P.mode == MODE_SOLVE && P.n > 0 && P.n <= 1023 && !getenv("FAR_FUSED_PHASE2") &&
                    !(P.flags & FAR_SWITCH_COST) && (P.I >= 256 || getenv("FAR_PIPELINE_ALWAYS"));
  const bool need_ovf = P.mode == MODE_SOLVE && (kfast < kmax || pipe);
  if (getenv("FAR_DEBUG_NO_ROUND_BALANCE")) P.flags |= FAR_I_NO_ROUND_BALANCE;  // experiments (A/B)
  const int64_t lid = ctx->launch_id++;
  const int slot = (int)(lid % NREC) * CPL;
  far_status st;
  if ((st = order_after(ctx, lid - NREC, stream))) return st;  // previous user of the counter slot
  CK(cudaMemsetAsync(ctx->d_counter + slot, 0, CPL * sizeof(unsigned long long), stream));
  if (!P.errflag) P.errflag = ctx->d_errflag;
  P.ovf_count = ctx->d_counter + slot + 2;
  P.ovf = nullptr;
  if (need_ovf) {
    const int r = (slot / CPL) & 3;
    if ((st = order_after(ctx, ctx->ovf_last[r], stream))) return st;
    ctx->ovf_last[r] = lid;
    const size_t words = (size_t)((P.I + 31) / 32);
    if (ctx->ovf_words[r] < words) {
      if (ctx->d_ovf[r]) {
        CK(cudaDeviceSynchronize());
        CK(cudaFree(ctx->d_ovf[r]));
      }
      if (cudaMalloc(&ctx->d_ovf[r], words * 4) != cudaSuccess) return fail(ctx, FAR_E_OOM, "overflow mask");
      ctx->ovf_words[r] = words;
    }
    P.ovf = ctx->d_ovf[r];
    CK(cudaMemsetAsync(P.ovf, 0, words * 4, stream));
  }
  far_ctx::EvSet* tset = nullptr;
  if ((st = t_begin(ctx, stream, tset))) return st;
  if (pipe) {
    // ---- workspace for this launch
    const Layout LF = a30 ? layout_for<3>(P.n, kfast) : layout_for<5>(P.n, kfast);
    const int ecap1 = LF.ecap + 1;
    auto a256 = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t I = (size_t)P.I;
    const int kstride = (kfast + 3) & ~3;  // per-instance stride of ws_lb / ws_cnt (16-B rows)
    const size_t o_ent = 0, o_lb = o_ent + a256(I * ecap1 * 8), o_cnt = o_lb + a256(I * kstride * 4),
                 o_meta = o_cnt + a256(I * kstride * 8), o_best = o_meta + a256(I * 64), o_evt = o_best + a256(I * 8),
                 o_rec = o_evt + a256(I * 8), o_sl = o_rec + a256(I * P.n * 4), o_items = o_sl + a256(I * 32),
                 o_m0 = o_items + a256(I * (size_t)(kfast - 1 > 0 ? kfast - 1 : 1) * 8);
    const int n4 = (P.n + 3) & ~3;
    const size_t o_ncnt = o_m0 + a256(I * (size_t)n4 * 4);
    const size_t o_d0 = o_ncnt + a256(I * 32);
    const size_t o_gen = o_d0 + a256(I * (size_t)n4 * 4);
    const size_t o_end = o_gen + a256(I * 8);
    const int r = (int)(lid & 1);
    if ((st = order_after(ctx, ctx->pws_last[r], stream))) return st;
    ctx->pws_last[r] = lid;
    if ((st = grow(ctx, &ctx->d_pws[r], &ctx->d_pws_bytes[r], o_end))) return st;
    char* w = ctx->d_pws[r];
    P.ws_ent = (int2*)(w + o_ent);
    P.ws_lb = (int*)(w + o_lb);
    P.ws_cnt = (unsigned long long*)(w + o_cnt);
    P.ws_meta = (int*)(w + o_meta);
    P.ws_best = (unsigned long long*)(w + o_best);
    P.ws_evt = (unsigned long long*)(w + o_evt);
    P.ws_rec = (uint32_t*)(w + o_rec);
    P.ws_sl = (int*)(w + o_sl);
    P.ws_ecap1 = ecap1;
    P.ws_kcap = kstride;
    P.ws_m0 = (uint32_t*)(w + o_m0);
    P.ws_n4 = n4;
    P.ws_ncnt = (uint16_t*)(w + o_ncnt);
    P.ws_d0 = (uint32_t*)(w + o_d0);
    // ---- K1: H0-H3 per instance (warp): the register-resident prep for n <= 128 (far_prep.cuh),
    //      the general PIPE_PREP instantiation of the fused kernel otherwise (and for FAR_GROW_TIES)
    P.kcap = kfast;
    P.ovf_pass = 0;
    P.counter = ctx->d_counter + slot + 0;
    if (P.n <= 128 && kfast <= 129 && !(P.flags & FAR_GROW_TIES) && !getenv("FAR_OLD_PREP")) {
      P.gen_list = (int64_t*)(w + o_gen);
      P.gen_count = ctx->d_counter + slot + 6;
      if ((st = launch_prep(ctx, P, stream, ctx->d_counter + slot + 7))) return st;
    } else if ((st = launch_warp_kernel(ctx, P, stream, P.I, PIPE_PREP))) {
      return st;
    }
    if ((st = t_mark(ctx, tset, stream, FAR_STAGE_PREP))) return st;
    // ---- K2-K4: phase 2 at lane granularity
    PParams Q;
    memset(&Q, 0, sizeof(Q));
    Q.I = P.I;
    Q.n = P.n;
    for (int c = 0; c < 8; ++c) {
      Q.cr[c] = P.cr[c];
      Q.de[c] = P.de[c];
    }
    Q.flags = P.flags;
    Q.ws_ent = P.ws_ent; Q.ws_lb = P.ws_lb; Q.ws_cnt = P.ws_cnt; Q.ws_meta = P.ws_meta;
    Q.ws_best = P.ws_best; Q.ws_evt = P.ws_evt; Q.ws_rec = P.ws_rec; Q.ws_sl = P.ws_sl;
    Q.ws_ecap1 = ecap1; Q.ws_kcap = kstride;
    Q.ws_m0 = P.ws_m0; Q.ws_n4 = n4; Q.ws_ncnt = P.ws_ncnt;
    Q.items = (int2*)(w + o_items);
    Q.nitems = ctx->d_counter + slot + 3;
    Q.counter = ctx->d_counter + slot + 4;
    Q.counter2 = ctx->d_counter + slot + 8;
    const int tb = 128;
    const size_t psm = (size_t)4 * NC * tb + (size_t)2 * NN * tb;
    int winner_per_sm = 16;
    if (const char* e = getenv("FAR_DEBUG_WINNER_BPS")) winner_per_sm = std::max(1, atoi(e));  // experiments
    const int g_inst = (int)std::min<int64_t>((P.I + tb - 1) / tb, (int64_t)ctx->sms * winner_per_sm);
    int items_per_sm = 12;  // blocks of 128 per SM for K3: 12 measured 1.68 ms per 1M M5, 16: 1.71, 14: 1.85
    if (const char* e = getenv("FAR_DEBUG_MEMBERS_BPS")) items_per_sm = std::max(1, std::min(16, atoi(e)));  // experiments
    const int g_items = ctx->sms * items_per_sm;
    {  // K2: per-thread shared-memory copy of member 0's lists -> block size by footprint
      const size_t per_thread = (size_t)4 * NC + 2 * NN + 4 * (size_t)(n4 + 4);  // row stride n4 + 4 (TMA) or n4 + 1
      int tbmax = 128;
      if (const char* e = getenv("FAR_DEBUG_M0_TB")) tbmax = std::max(32, std::min(128, atoi(e)));  // experiments
      const int tb0 = (int)std::min<size_t>(tbmax, (size_t)ctx->smem_max / per_thread / 32 * 32);
      if (tb0 < 32) return fail(ctx, FAR_E_TOO_LARGE, "member-0 lists do not fit in shared memory");
      const size_t sm0 = per_thread * tb0;
      const void* f0 = a30 ? (const void*)far_member0_kernel<3> : (const void*)far_member0_kernel<5>;
      int per_sm = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f0, tb0, sm0));
      // n > 64: at most 12 warps per SM -- measured on M5 (1M x n = 128): with one atomic per lane for
      // the candidate items 8 warps were best (1.33 ms, 1.48 at 12); since the warp-aggregated item
      // emission 12 (the shared-memory limit at n = 128) is: 1.067 ms against 1.18 at 8 and 10 (block
      // size 64 or 128); M3 (100k x n = 32, short rows, one pass over the instances) keeps full occupancy
      int m0_warps = 12;
      if (const char* e = getenv("FAR_DEBUG_M0_WARPS")) m0_warps = std::max(1, atoi(e));  // experiments
      if (P.n > 64) per_sm = std::min(per_sm, std::max(1, m0_warps * 32 / tb0));
      if (const char* e = getenv("FAR_DEBUG_M0_BPS")) per_sm = std::min(per_sm, atoi(e));  // experiments
      const int g0 = (int)std::max<int64_t>(1, std::min<int64_t>((P.I + tb0 - 1) / tb0, (int64_t)ctx->sms * std::max(1, per_sm)));
      if (a30) far_member0_kernel<3><<<g0, tb0, sm0, stream>>>(Q);
      else far_member0_kernel<5><<<g0, tb0, sm0, stream>>>(Q);
    }
    CK(cudaGetLastError());
    if ((st = t_mark(ctx, tset, stream, FAR_STAGE_MEMBER0))) return st;
    if (a30) far_members_kernel<3><<<g_items, tb, psm, stream>>>(Q);
    else far_members_kernel<5><<<g_items, tb, psm, stream>>>(Q);
    CK(cudaGetLastError());
    if ((st = t_mark(ctx, tset, stream, FAR_STAGE_MEMBERS))) return st;
    if (a30) far_winner_kernel<3><<<g_inst, tb, psm, stream>>>(Q);
    else far_winner_kernel<5><<<g_inst, tb, psm, stream>>>(Q);
    CK(cudaGetLastError());
    ctx->launches += 3;
    if ((st = t_mark(ctx, tset, stream, FAR_STAGE_WINNER))) return st;
    // ---- K5: H6-H7, one thread per instance (n <= 256), else (and for FAR_BEST_IMPROVEMENT) one warp
    //      per instance
    P.counter = ctx->d_counter + slot + 5;
    const LRow LR = make_lrow(P.n, NN);
    int tblmax = 128;
    if (const char* e = getenv("FAR_DEBUG_FIN_TB")) tblmax = std::max(32, std::min(128, atoi(e)));  // experiments
    const int tbl = (int)std::min<int64_t>(tblmax, (int64_t)ctx->smem_max / LR.bytes / 32 * 32);
    if (P.n <= 256 && tbl >= 32 && !(P.flags & FAR_BEST_IMPROVEMENT) && !getenv("FAR_DEBUG_WARP_FINISH")) {
      const void* lfn = a30 ? (const void*)far_finish_lane_kernel<3> : (const void*)far_finish_lane_kernel<5>;
      const size_t lsm = (size_t)tbl * LR.bytes;
      int per_sm = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lfn, tbl, lsm));
      if (const char* e = getenv("FAR_DEBUG_FIN_BPS")) per_sm = std::min(per_sm, atoi(e));  // experiments
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((P.I + tbl - 1) / tbl, (int64_t)ctx->sms * std::max(1, per_sm)));
      if (a30) far_finish_lane_kernel<3><<<grid, tbl, lsm, stream>>>(P);
      else far_finish_lane_kernel<5><<<grid, tbl, lsm, stream>>>(P);
      CK(cudaGetLastError());
      ++ctx->launches;
    } else {
      const FLayout FL = make_flayout(P.n, NN);
      const int fw = 4;
      int per_sm = 0;
      const void* ffn = a30 ? (const void*)far_finish_kernel<3> : (const void*)far_finish_kernel<5>;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ffn, fw * 32, (size_t)fw * FL.bytes));
      if (per_sm < 1) return fail(ctx, FAR_E_TOO_LARGE, "finish layout does not fit in shared memory");
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((P.I + fw - 1) / fw, (int64_t)ctx->sms * per_sm));
      if (a30) far_finish_kernel<3><<<grid, fw * 32, (size_t)fw * FL.bytes, stream>>>(P);
      else far_finish_kernel<5><<<grid, fw * 32, (size_t)fw * FL.bytes, stream>>>(P);
      CK(cudaGetLastError());
      ++ctx->launches;
    }
    if ((st = t_mark(ctx, tset, stream, FAR_STAGE_FINISH))) return st;
  } else {
    P.kcap = kfast;
    P.ovf_pass = 0;
    P.counter = ctx->d_counter + slot + 0;
    if ((st = launch_warp_kernel(ctx, P, stream, P.I, PIPE_NONE))) return st;
    if ((st = t_mark(ctx, tset, stream, FAR_STAGE_FUSED))) return st;
  }
  if (need_ovf) {  // instances deferred by the fast layout / the pipeline: fused kernel, full layout
    P.kcap = kmax;
    P.ovf_pass = 1;
    P.counter = ctx->d_counter + slot + 1;
    if ((st = launch_warp_kernel(ctx, P, stream, (P.I + 31) / 32, PIPE_NONE))) return st;
    if ((st = t_mark(ctx, tset, stream, FAR_STAGE_OVERFLOW))) return st;
  }
  return record_launch(ctx, lid, stream);
}

static far_status check_opts(far_ctx* ctx, const far_opts* o) {
  if (o && (o->max_iterations < 0 || o->min_improvement_ppm < 0 || o->min_improvement_ppm > 1000000))
    return fail(ctx, FAR_E_INVALID_ARG, "far_opts out of range");
  return FAR_OK;
}

static void fill_params(far_ctx* ctx, const far_opts* o, KParams& P) {
  memset(&P, 0, sizeof(P));
  P.max_it = o ? o->max_iterations : 100;
  P.ppm = o ? o->min_improvement_ppm : 0;
  P.flags = o ? o->flags : 0u;
  const bool zero = (P.flags & FAR_ZERO_RECONFIG) != 0;
  for (int c = 0; c < 8; ++c) {
    P.cr[c] = zero ? 0 : ctx->cr[c];
    P.de[c] = zero ? 0 : ctx->de[c];
  }
  P.rsum = 0;
  for (int v = 0; v < ctx->nn; ++v) {
    const int szi = nd_szi(ctx->nc == 3 ? Tree<3>::node[v] : Tree<5>::node[v]);
    P.rsum += P.cr[szi] + P.de[szi];
  }
  P.rsum *= ctx->gpus;  // every tree of a multi-target forest
}

extern "C" {

far_status far_create(far_profile profile, const int32_t* reconfig_cost, far_ctx** out) {
  return far_create_multi(profile, 1, reconfig_cost, out);
}

far_status far_create_multi(far_profile profile, int32_t num_gpus, const int32_t* reconfig_cost, far_ctx** out) {
  if (!out) return FAR_E_INVALID_ARG;
  *out = nullptr;
  if (profile != FAR_A30 && profile != FAR_A100 && profile != FAR_H100) return FAR_E_UNSUPPORTED_PROFILE;
  if (num_gpus < 1 || num_gpus > FMAXG) return FAR_E_INVALID_ARG;
  far_ctx* c = new far_ctx();
  c->profile = profile;
  c->gpus = num_gpus;
  if (profile == FAR_A30) {
    c->nc = 3; c->ns = Tree<3>::S; c->nn = Tree<3>::NN;
  } else {
    c->nc = 5; c->ns = Tree<5>::S; c->nn = Tree<5>::NN;
  }
  // forest node table: tree t's node v -> id t*NN + v, slices t*S + [lo, hi)
  for (int t = 0; t < num_gpus; ++t)
    for (int v = 0; v < c->nn; ++v) {
      const uint32_t w = c->nc == 3 ? Tree<3>::node[v] : Tree<5>::node[v];
      auto id = [&](int u) { return u == LEAF ? FNONE : t * c->nn + u; };
      const int par = nd_par(w) == ROOTP ? FNONE : t * c->nn + nd_par(w);
      uint2 f;
      f.x = (uint32_t)(nd_lo(w) + t * c->ns) | ((uint32_t)nd_sz(w) << 8) | ((uint32_t)nd_szi(w) << 12) |
            ((uint32_t)nd_c0(w) << 16) | ((uint32_t)nd_c1(w) << 20);
      f.y = (uint32_t)id(nd_ch1(w)) | ((uint32_t)id(nd_ch2(w)) << 8) | ((uint32_t)par << 16);
      c->fnodes[t * c->nn + v] = f;
    }
  for (int i = 0; i < c->nc; ++i) c->sizes[i] = c->nc == 3 ? size_of<3>(i) : size_of<5>(i);
  // Table 2 in 1 ms ticks
  static const int a30c[3] = {110, 120, 130}, a30d[3] = {100, 100, 100};
  static const int a100c[5] = {160, 170, 200, 210, 240}, a100d[5] = {200, 200, 210, 210, 220};
  static const int h100c[5] = {160, 210, 330, 380, 420}, h100d[5] = {210, 230, 250, 260, 260};
  for (int i = 0; i < c->nc; ++i) {
    if (reconfig_cost) {
      c->cr[i] = reconfig_cost[i];
      c->de[i] = reconfig_cost[c->nc + i];
      if (c->cr[i] < 0 || c->de[i] < 0 || c->cr[i] >= BOUND || c->de[i] >= BOUND) {
        delete c;
        return FAR_E_BAD_TIME;
      }
    } else if (profile == FAR_A30) {
      c->cr[i] = a30c[i]; c->de[i] = a30d[i];
    } else if (profile == FAR_A100) {
      c->cr[i] = a100c[i]; c->de[i] = a100d[i];
    } else {
      c->cr[i] = h100c[i]; c->de[i] = h100d[i];
    }
  }
  *out = c;
  return FAR_OK;
}

void far_destroy(far_ctx* ctx) {
  if (!ctx) return;
  if (ctx->inited) {
    cudaDeviceSynchronize();
    cudaFree(ctx->d_counter);
    cudaFree(ctx->d_errflag);
    for (auto& r : ctx->recs) cudaEventDestroy(r.ev);
    if (ctx->d_fnodes) cudaFree(ctx->d_fnodes);
    for (int r = 0; r < 4; ++r)
      if (ctx->d_ovf[r]) cudaFree(ctx->d_ovf[r]);
    if (ctx->d_buf) cudaFree(ctx->d_buf);
    if (ctx->d_cbuf) cudaFree(ctx->d_cbuf);
    for (int r = 0; r < 2; ++r)
      if (ctx->d_pws[r]) cudaFree(ctx->d_pws[r]);
    cudaStreamDestroy(ctx->s[0]);
    cudaStreamDestroy(ctx->s[1]);
    for (auto& e : ctx->tsets)
      if (e.created)
        for (auto& v : e.ev) cudaEventDestroy(v);
  }
  delete ctx;
}

int32_t far_num_sizes(const far_ctx* ctx) { return ctx ? ctx->nc : -1; }
const int32_t* far_sizes(const far_ctx* ctx) { return ctx ? ctx->sizes : nullptr; }
int32_t far_num_nodes(const far_ctx* ctx) { return ctx ? ctx->nn * ctx->gpus : -1; }
int32_t far_num_slices(const far_ctx* ctx) { return ctx ? ctx->ns * ctx->gpus : -1; }
int32_t far_num_gpus(const far_ctx* ctx) { return ctx ? ctx->gpus : -1; }
const char* far_last_error(const far_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

far_status far_stage_timing(far_ctx* ctx, int32_t enable) {
  if (!ctx) return FAR_E_INVALID_ARG;
  ctx->timing = enable != 0;
  return FAR_OK;
}

int32_t far_stage_times(far_ctx* ctx, float* ms) {
  if (!ctx) return -1;
  for (int i = 0; i < far_ctx::NSETS; ++i)  // oldest first
    if (t_collect(ctx, ctx->tsets[(ctx->tnext + i) % far_ctx::NSETS]) != FAR_OK) return -1;
  if (ms)
    for (int s = 0; s < FAR_NUM_STAGES; ++s) ms[s] = (float)ctx->stage_ms[s];
  const int n = ctx->timed;
  for (double& v : ctx->stage_ms) v = 0.0;
  ctx->timed = 0;
  return n;
}

int64_t far_launch_count(const far_ctx* ctx) { return ctx ? ctx->launches : -1; }

far_status far_measure_peak(far_ctx* ctx, int32_t mode, double* per_s) {
  if (!ctx || !per_s || mode < 0 || mode > 2) return FAR_E_INVALID_ARG;
  far_status st = ensure_device(ctx);
  if (st) return st;
  unsigned* d_out = nullptr;
  CK(cudaMalloc(&d_out, 4));
  const int blocks = ctx->sms * 2, threads = 1024, iters = mode == 2 ? 2048 : 4096;
  auto launch = [&](int it) {
    if (mode == 0) far_peak_kernel<0><<<blocks, threads>>>(d_out, it);
    else if (mode == 1) far_peak_kernel<1><<<blocks, threads>>>(d_out, it);
    else far_peak_kernel<2><<<blocks, threads>>>(d_out, it);
  };
  launch(64);  // warm-up (clocks, module load)
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a));
  launch(iters);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(d_out);
  const double ops = (double)blocks * threads * iters * 16.0 * 8.0;
  *per_s = (mode == 2 ? 4.0 : 1.0) * ops / (ms * 1e-3);
  return FAR_OK;
}

far_status far_node_table(const far_ctx* ctx, int32_t* lo, int32_t* hi, int32_t* parent) {
  if (!ctx || !lo || !hi || !parent) return FAR_E_INVALID_ARG;
  for (int v = 0; v < ctx->nn * ctx->gpus; ++v) {
    const uint2 f = ctx->fnodes[v];
    lo[v] = (int)(f.x & 255u);
    hi[v] = lo[v] + (int)((f.x >> 8) & 15u);
    const int par = (int)((f.y >> 16) & 255u);
    parent[v] = par == FNONE ? -1 : par;
  }
  return FAR_OK;
}

far_status far_sync(far_ctx* ctx) {
  if (!ctx) return FAR_E_INVALID_ARG;
  far_status st = ensure_device(ctx);
  if (st) return st;
  CK(cudaDeviceSynchronize());
  int flag = 0;
  CK(cudaMemcpy(&flag, ctx->d_errflag, sizeof(int), cudaMemcpyDeviceToHost));
  if (flag) {
    CK(cudaMemset(ctx->d_errflag, 0, sizeof(int)));
    if (flag & 4) return fail(ctx, FAR_E_TOO_LARGE, "a stream overflowed its placed-event window");
    return fail(ctx, (flag & 1) ? FAR_E_BAD_TIME : FAR_E_INVALID_ARG,
                (flag & 1) ? "an instance failed the input checks (t < 1 or makespan bound)"
                           : "an instance had an invalid input schedule");
  }
  return FAR_OK;
}

far_status far_solve_many(far_ctx* ctx, const int32_t* d_times, int64_t I, int32_t n, const far_opts* opts,
                          int32_t* d_makespan, far_task_slot* d_sched, far_result* d_res, void* cuda_stream) {
  if (!ctx) return FAR_E_INVALID_ARG;
  if (I < 0 || n < 0) return fail(ctx, FAR_E_INVALID_ARG, "negative I or n");
  if (n > MAXN) return fail(ctx, FAR_E_TOO_LARGE, "n > 1024");
  if (ctx->gpus > 1 && n > FMAXN) return fail(ctx, FAR_E_TOO_LARGE, "multi-GPU forest: n > 256");
  if (I > 0 && (!d_makespan || (n > 0 && !d_times))) return fail(ctx, FAR_E_INVALID_ARG, "null device pointer");
  far_status st = check_opts(ctx, opts);
  if (st) return st;
  if ((st = ensure_device(ctx))) return st;
  KParams P;
  fill_params(ctx, opts, P);
  P.times = d_times;
  P.I = I;
  P.n = n;
  P.makespan = d_makespan;
  P.sched = d_sched;
  P.res = d_res;
  P.mode = MODE_SOLVE;
  return launch_solve(ctx, P, (cudaStream_t)cuda_stream);
}

// one instance through device staging; mode SOLVE (phases 1-2 only) or LOCAL
static far_status one_instance(far_ctx* ctx, const int32_t* times, int32_t n, const far_opts* opts,
                               far_task_slot* sched, far_result* res, int mode) {
  if (!ctx) return FAR_E_INVALID_ARG;
  if (n < 0) return fail(ctx, FAR_E_INVALID_ARG, "negative n");
  if (n > MAXN) return fail(ctx, FAR_E_TOO_LARGE, "n > 1024");
  if (ctx->gpus > 1 && n > FMAXN) return fail(ctx, FAR_E_TOO_LARGE, "multi-GPU forest: n > 256");
  if ((n > 0 && (!times || !sched)) || !res) return fail(ctx, FAR_E_INVALID_ARG, "null host pointer");
  far_status st = check_opts(ctx, opts);
  if (st) return st;
  if ((st = ensure_device(ctx))) return st;
  const size_t tb = (size_t)n * ctx->nc * 4, sb = (size_t)n * sizeof(far_task_slot);
  const size_t o_t = 0, o_s = (tb + 255) & ~(size_t)255, o_si = o_s + ((sb + 255) & ~(size_t)255);
  const size_t o_r = o_si + ((sb + 255) & ~(size_t)255), o_ri = o_r + 256, o_m = o_ri + 256;
  if ((st = ensure_buf(ctx, o_m + 256))) return st;
  cudaStream_t s = ctx->s[0];
  KParams P;
  fill_params(ctx, opts, P);
  if (mode == MODE_SOLVE) P.flags |= FAR_NO_REFINE;
  P.flags &= ~(unsigned)FAR_NO_SCHEDULE;
  P.errflag = ctx->d_errflag + 1;  // private flag of the synchronous calls
  CK(cudaMemsetAsync(P.errflag, 0, sizeof(int), s));
  P.times = (const int32_t*)(ctx->d_buf + o_t);
  P.I = 1;
  P.n = n;
  P.makespan = (int32_t*)(ctx->d_buf + o_m);
  P.sched = n > 0 ? (far_task_slot*)(ctx->d_buf + o_s) : nullptr;
  P.res = (far_result*)(ctx->d_buf + o_r);
  P.mode = mode;
  if (tb) CK(cudaMemcpyAsync(ctx->d_buf + o_t, times, tb, cudaMemcpyHostToDevice, s));
  if (mode == MODE_LOCAL) {
    if (sb) CK(cudaMemcpyAsync(ctx->d_buf + o_si, sched, sb, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(ctx->d_buf + o_ri, res, sizeof(far_result), cudaMemcpyHostToDevice, s));
    P.sched_in = (const far_task_slot*)(ctx->d_buf + o_si);
    P.res_in = (const far_result*)(ctx->d_buf + o_ri);
  }
  if ((st = launch_solve(ctx, P, s))) return st;
  far_result r;
  CK(cudaMemcpyAsync(&r, P.res, sizeof(far_result), cudaMemcpyDeviceToHost, s));
  if (sb) CK(cudaMemcpyAsync(sched, P.sched, sb, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  *res = r;  // the call's own error is the status in its record (the private flag is not needed)
  if (r.status != FAR_OK)
    return fail(ctx, (far_status)r.status,
                r.status == FAR_E_BAD_TIME ? "input check failed (t < 1 or makespan bound)" : "invalid input schedule");
  return FAR_OK;
}

far_status far_schedule_batch(far_ctx* ctx, const int32_t* times, int32_t n, const far_opts* opts,
                              far_task_slot* sched, far_result* res) {
  return one_instance(ctx, times, n, opts, sched, res, MODE_SOLVE);
}

far_status far_local_search(far_ctx* ctx, const int32_t* times, int32_t n, const far_opts* opts,
                            far_task_slot* sched, far_result* res) {
  return one_instance(ctx, times, n, opts, sched, res, MODE_LOCAL);
}

far_status far_solve_many_host(far_ctx* ctx, const int32_t* h_times, int64_t I, int32_t n, const far_opts* opts,
                               int32_t* h_makespan, far_task_slot* h_sched, far_result* h_res) {
  if (!ctx) return FAR_E_INVALID_ARG;
  if (I < 0 || n < 0) return fail(ctx, FAR_E_INVALID_ARG, "negative I or n");
  if (n > MAXN) return fail(ctx, FAR_E_TOO_LARGE, "n > 1024");
  if (ctx->gpus > 1 && n > FMAXN) return fail(ctx, FAR_E_TOO_LARGE, "multi-GPU forest: n > 256");
  if (I > 0 && (!h_makespan || (n > 0 && !h_times))) return fail(ctx, FAR_E_INVALID_ARG, "null host pointer");
  far_status st = check_opts(ctx, opts);
  if (st) return st;
  if ((st = ensure_device(ctx))) return st;
  if (I == 0) return FAR_OK;
  const bool want_sched = h_sched && !(opts && (opts->flags & FAR_NO_SCHEDULE));
  const size_t per_t = (size_t)n * ctx->nc * 4, per_s = want_sched ? (size_t)n * sizeof(far_task_slot) : 0;
  const size_t per_r = h_res ? sizeof(far_result) : 0, per_m = 4;
  const size_t per = per_t + per_s + per_r + per_m;
  // chunk: ~192 MB of staging per stream (PCIe copies of large chunks run near the link rate)
  size_t chunk_mb = 192;  // measured: 48 MB 61 ms, 96 MB 52 ms, 192 MB 50 ms, 384 MB 52 ms per 1M M5 instances
  if (const char* e = getenv("FAR_HOST_CHUNK_MB")) chunk_mb = (size_t)std::max(1, std::min(4096, atoi(e)));  // experiments
  int64_t chunk = std::max<int64_t>(1, (chunk_mb << 20) / std::max<size_t>(per, 1));
  chunk = std::min<int64_t>(chunk, I);
  auto a256 = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t bt = a256(chunk * per_t), bs = a256(chunk * per_s), br = a256(chunk * per_r), bm = a256(chunk * per_m);
  const size_t per_stream = bt + bs + br + bm;
  if ((st = ensure_buf(ctx, 2 * per_stream))) return st;
  KParams P;
  fill_params(ctx, opts, P);
  P.n = n;
  P.mode = MODE_SOLVE;
  P.errflag = ctx->d_errflag + 1;  // private flag of the synchronous calls
  CK(cudaMemsetAsync(P.errflag, 0, sizeof(int), ctx->s[0]));
  CK(cudaStreamSynchronize(ctx->s[0]));
  int64_t nchunks = (I + chunk - 1) / chunk;
  for (int64_t q = 0; q < nchunks; ++q) {
    const int si = (int)(q & 1);
    cudaStream_t s = ctx->s[si];
    char* base = ctx->d_buf + si * per_stream;
    const int64_t i0 = q * chunk, cnt = std::min(chunk, I - i0);
    if (per_t) CK(cudaMemcpyAsync(base, (const char*)h_times + i0 * per_t, cnt * per_t, cudaMemcpyHostToDevice, s));
    P.times = (const int32_t*)base;
    P.I = cnt;
    P.sched = want_sched ? (far_task_slot*)(base + bt) : nullptr;
    P.res = h_res ? (far_result*)(base + bt + bs) : nullptr;
    P.makespan = (int32_t*)(base + bt + bs + br);
    if ((st = launch_solve(ctx, P, s))) return st;
    CK(cudaMemcpyAsync(h_makespan + i0, P.makespan, cnt * per_m, cudaMemcpyDeviceToHost, s));
    if (want_sched)
      CK(cudaMemcpyAsync((char*)h_sched + i0 * per_s, P.sched, cnt * per_s, cudaMemcpyDeviceToHost, s));
    if (h_res) CK(cudaMemcpyAsync(h_res + i0, P.res, cnt * per_r, cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(ctx->s[0]));
  CK(cudaStreamSynchronize(ctx->s[1]));
  int flag = 0;
  CK(cudaMemcpy(&flag, ctx->d_errflag + 1, sizeof(int), cudaMemcpyDeviceToHost));
  if (flag) {  // this call's own bits, decoded as far_sync does
    CK(cudaMemset(ctx->d_errflag + 1, 0, sizeof(int)));
    return fail(ctx, (flag & 1) ? FAR_E_BAD_TIME : FAR_E_INVALID_ARG,
                (flag & 1) ? "an instance failed the input checks (t < 1 or makespan bound)"
                           : "an instance had an invalid input schedule");
  }
  return FAR_OK;
}

}  // extern "C"

extern "C" far_status far_concat_streams(far_ctx* ctx, const int32_t* d_times, int64_t S, int32_t B, int32_t n,
                                         const far_opts* opts, int64_t* d_stream_makespan, int64_t* d_offsets,
                                         far_task_slot* d_sched, far_result* d_batch_res, int32_t* d_seam,
                                         void* cuda_stream) {
  if (!ctx) return FAR_E_INVALID_ARG;
  if (ctx->gpus > 1) return fail(ctx, FAR_E_UNSUPPORTED_PROFILE, "streams: single-GPU trees only");
  if (opts && (opts->flags & FAR_SWITCH_COST)) return fail(ctx, FAR_E_INVALID_ARG, "streams: no FAR_SWITCH_COST");
  if (S < 0 || B < 0 || n < 0) return fail(ctx, FAR_E_INVALID_ARG, "negative S, B or n");
  if (n > MAXN) return fail(ctx, FAR_E_TOO_LARGE, "n > 1024");
  if (S > 0 && B > 0 && (!d_stream_makespan || !d_offsets || (n > 0 && !d_times)))
    return fail(ctx, FAR_E_INVALID_ARG, "null device pointer");
  far_status st = check_opts(ctx, opts);
  if (st) return st;
  if ((st = ensure_device(ctx))) return st;
  if (S == 0) return FAR_OK;
  cudaStream_t stream = (cudaStream_t)cuda_stream;
  if (B == 0) {
    CK(cudaMemsetAsync(d_stream_makespan, 0, S * 2 * sizeof(int64_t), stream));
    return FAR_OK;
  }
  const int64_t IB = S * (int64_t)B;
  auto a256 = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t bs = a256((size_t)IB * n * sizeof(far_task_slot)), br = a256((size_t)IB * sizeof(far_result)),
               bm = a256((size_t)IB * 4);
  cudaStream_t stream0 = (cudaStream_t)cuda_stream;
  if ((st = order_after(ctx, ctx->cbuf_last, stream0))) return st;  // d_cbuf's previous user
  if ((st = grow(ctx, &ctx->d_cbuf, &ctx->d_cbuf_bytes, bs + br + bm))) return st;
  // 1) FAR phases 1-3 on every batch of every stream (data-parallel)
  KParams P;
  fill_params(ctx, opts, P);
  P.flags &= ~(unsigned)FAR_NO_SCHEDULE;
  P.times = d_times;
  P.I = IB;
  P.n = n;
  P.sched = (far_task_slot*)ctx->d_cbuf;
  P.res = d_batch_res ? d_batch_res : (far_result*)(ctx->d_cbuf + bs);
  P.makespan = (int32_t*)(ctx->d_cbuf + bs + br);
  P.mode = MODE_SOLVE;
  if ((st = launch_solve(ctx, P, stream))) return st;
  // 2) the per-stream fold (one warp per stream)
  SParams Q;
  memset(&Q, 0, sizeof(Q));
  Q.times = d_times;
  Q.sched = P.sched;
  Q.S = S;
  Q.B = B;
  Q.n = n;
  for (int c = 0; c < 8; ++c) {
    Q.cr[c] = P.cr[c];
    Q.de[c] = P.de[c];
  }
  Q.max_it = P.max_it;
  Q.seam_moves = (P.flags & FAR_NO_SEAM_MOVES) ? 0 : 1;
  Q.stream_ms = d_stream_makespan;
  Q.offsets = d_offsets;
  Q.out_sched = d_sched;
  Q.seam = d_seam;
  Q.errflag = ctx->d_errflag;
  const bool a30 = ctx->nc == 3;
  const SLayout L = make_slayout(n, ctx->nc, ctx->nn);
  int warps = std::min(4, ctx->smem_max / std::max(1, L.bytes));
  if (warps < 1) return fail(ctx, FAR_E_TOO_LARGE, "stream state does not fit in shared memory");
  const size_t smem = (size_t)warps * L.bytes;
  const int grid = (int)((S + warps - 1) / warps);
  far_ctx::EvSet* tset = nullptr;
  if ((st = t_begin(ctx, stream, tset))) return st;
  if (a30)
    far_stream_kernel<3><<<grid, warps * 32, smem, stream>>>(Q);
  else
    far_stream_kernel<5><<<grid, warps * 32, smem, stream>>>(Q);
  CK(cudaGetLastError());
  ++ctx->launches;
  if ((st = t_mark(ctx, tset, stream, FAR_STAGE_STREAM))) return st;
  // the fold is the last user of d_cbuf: order the next concat after it (same event ring)
  ctx->cbuf_last = ctx->launch_id++;
  if ((st = order_after(ctx, ctx->cbuf_last - NREC, stream))) return st;
  return record_launch(ctx, ctx->cbuf_last, stream);
}

// ---- schedule events and validation (far_check.cuh), one warp per instance
static far_status launch_check(far_ctx* ctx, CParams& Q, int64_t I, int n, bool validate, cudaStream_t stream) {
  const bool a30 = ctx->nc == 3;
  const bool forest = ctx->gpus > 1;
  const int NNF = ctx->nn * ctx->gpus;
  const int bytes = forest ? (validate ? make_fvlayout(n, NNF).bytes : make_felayout(n, ctx->nc, NNF).bytes)
                           : (validate ? make_vlayout(n, ctx->nn).bytes : make_elayout(n, ctx->nn).bytes);
  const void* fn =
      forest ? (validate ? (a30 ? (const void*)far_forest_validate_kernel<3> : (const void*)far_forest_validate_kernel<5>)
                         : (a30 ? (const void*)far_forest_events_kernel<3> : (const void*)far_forest_events_kernel<5>))
             : (validate ? (a30 ? (const void*)far_validate_kernel<3> : (const void*)far_validate_kernel<5>)
                         : (a30 ? (const void*)far_events_kernel<3> : (const void*)far_events_kernel<5>));
  int warps = 0, per_sm = 0;
  far_status st = pick_shape(ctx, fn, bytes, warps, per_sm);
  if (st) return st;
  const int64_t lid = ctx->launch_id++;
  const int slot = (int)(lid % NREC) * CPL;
  if ((st = order_after(ctx, lid - NREC, stream))) return st;
  CK(cudaMemsetAsync(ctx->d_counter + slot, 0, sizeof(unsigned long long), stream));
  Q.counter = ctx->d_counter + slot;
  far_ctx::EvSet* tset = nullptr;
  if ((st = t_begin(ctx, stream, tset))) return st;
  const size_t smem = (size_t)warps * bytes;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((I + warps - 1) / warps, (int64_t)ctx->sms * per_sm));
  if (forest) {  // multi-target contexts: the generic forest kernels (far_forest_check.cuh)
    FCParams C;
    memset(&C, 0, sizeof(C));
    fill_params(ctx, nullptr, C.F.P);
    for (int c = 0; c < 8; ++c) {
      C.F.P.cr[c] = Q.cr[c];
      C.F.P.de[c] = Q.de[c];
    }
    C.F.nodes = ctx->d_fnodes;
    C.F.NNF = NNF;
    C.F.SF = ctx->ns * ctx->gpus;
    C.Q = Q;
    void* args[] = {&C};
    CK(cudaLaunchKernel(fn, grid, warps * 32, args, smem, stream));
  } else if (validate) {
    if (a30) far_validate_kernel<3><<<grid, warps * 32, smem, stream>>>(Q);
    else far_validate_kernel<5><<<grid, warps * 32, smem, stream>>>(Q);
  } else {
    if (a30) far_events_kernel<3><<<grid, warps * 32, smem, stream>>>(Q);
    else far_events_kernel<5><<<grid, warps * 32, smem, stream>>>(Q);
  }
  CK(cudaGetLastError());
  ++ctx->launches;
  if ((st = t_mark(ctx, tset, stream, FAR_STAGE_CHECK))) return st;
  return record_launch(ctx, lid, stream);
}

static far_status check_args(far_ctx* ctx, const int32_t* d_times, int64_t I, int32_t n, const far_task_slot* d_sched,
                             const far_opts* opts, CParams& Q) {
  if (ctx->gpus > 1 && n > FMAXN) return fail(ctx, FAR_E_TOO_LARGE, "multi-GPU forest: n > 256");
  if (opts && (opts->flags & FAR_SWITCH_COST))
    return fail(ctx, FAR_E_INVALID_ARG, "events / validator: no FAR_SWITCH_COST");
  if (I < 0 || n < 0) return fail(ctx, FAR_E_INVALID_ARG, "negative I or n");
  if (n > MAXN) return fail(ctx, FAR_E_TOO_LARGE, "n > 1024");
  if (I > 0 && n > 0 && (!d_times || !d_sched)) return fail(ctx, FAR_E_INVALID_ARG, "null device pointer");
  far_status st = check_opts(ctx, opts);
  if (st) return st;
  if ((st = ensure_device(ctx))) return st;
  KParams P;
  fill_params(ctx, opts, P);
  memset(&Q, 0, sizeof(Q));
  Q.times = d_times;
  Q.sched = d_sched;
  Q.I = I;
  Q.n = n;
  for (int c = 0; c < 8; ++c) {
    Q.cr[c] = P.cr[c];
    Q.de[c] = P.de[c];
  }
  return FAR_OK;
}

extern "C" {

far_status far_schedule_events(far_ctx* ctx, const int32_t* d_times, int64_t I, int32_t n,
                               const far_task_slot* d_sched, const far_opts* opts, far_event* d_events,
                               int32_t* d_nev, int32_t* d_makespan, void* cuda_stream) {
  if (!ctx) return FAR_E_INVALID_ARG;
  CParams Q;
  far_status st = check_args(ctx, d_times, I, n, d_sched, opts, Q);
  if (st) return st;
  if (I > 0 && (!d_events || !d_nev)) return fail(ctx, FAR_E_INVALID_ARG, "null device pointer");
  if (I == 0) return FAR_OK;
  Q.events = d_events;
  Q.nev = d_nev;
  Q.makespan = d_makespan;
  return launch_check(ctx, Q, I, n, false, (cudaStream_t)cuda_stream);
}

far_status far_validate_schedules(far_ctx* ctx, const int32_t* d_times, int64_t I, int32_t n,
                                  const far_task_slot* d_sched, const far_opts* opts, const far_event* d_events,
                                  const int32_t* d_nev, int32_t* d_violations, void* cuda_stream) {
  if (!ctx) return FAR_E_INVALID_ARG;
  CParams Q;
  far_status st = check_args(ctx, d_times, I, n, d_sched, opts, Q);
  if (st) return st;
  if (I > 0 && (!d_events || !d_nev || !d_violations)) return fail(ctx, FAR_E_INVALID_ARG, "null device pointer");
  if (I == 0) return FAR_OK;
  Q.events_in = d_events;
  Q.nev_in = d_nev;
  Q.violations = d_violations;
  return launch_check(ctx, Q, I, n, true, (cudaStream_t)cuda_stream);
}

far_status far_lower_bounds(far_ctx* ctx, const int32_t* d_times, int64_t I, int32_t n, int64_t* d_sum_min_work,
                            int32_t* d_max_min_time, void* cuda_stream) {
  if (!ctx) return FAR_E_INVALID_ARG;
  if (I < 0 || n < 0) return fail(ctx, FAR_E_INVALID_ARG, "negative I or n");
  if (I > 0 && (!d_sum_min_work || (n > 0 && !d_times))) return fail(ctx, FAR_E_INVALID_ARG, "null device pointer");
  far_status st = ensure_device(ctx);
  if (st) return st;
  if (I == 0) return FAR_OK;
  cudaStream_t stream = (cudaStream_t)cuda_stream;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((I + 255) / 256, (int64_t)ctx->sms * 8));
  if (ctx->nc == 3)
    far_lower_bound_kernel<3><<<grid, 256, 0, stream>>>(d_times, I, n, (long long*)d_sum_min_work, d_max_min_time);
  else
    far_lower_bound_kernel<5><<<grid, 256, 0, stream>>>(d_times, I, n, (long long*)d_sum_min_work, d_max_min_time);
  CK(cudaGetLastError());
  ++ctx->launches;
  return FAR_OK;
}

}  // extern "C"
