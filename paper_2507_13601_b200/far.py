"""Thin Python binding of libfar.so (include/far.h) — argument marshalling only.

Every step of FAR runs in the sm_100a kernels behind the C-ABI.  There is no CPU
fallback: if libfar.so is missing this module raises at import-time use, and on a
machine without a CUDA device every compute call raises FarError(FAR_E_CUDA).
PyTorch is used only for device memory and streams (tensor.data_ptr(),
torch.cuda.current_stream().cuda_stream).
"""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FAR_LIB_OVERRIDE") or os.path.join(HERE, "libfar.so")  # override: A/B experiments only
HEADER = os.path.join(os.path.dirname(HERE), "include", "far.h")

PROFILES = {"A30": 0, "A100": 1, "H100": 2}
NO_REFINE, NO_GUARD, ZERO_RECONFIG, NO_SCHEDULE, EXHAUSTIVE, NONEMPTY_ALT, NO_SEAM_MOVES, GROW_TIES, \
    BEST_IMPROVEMENT, SWITCH_COST = 1, 2, 4, 8, 16, 32, 64, 128, 256, 512
STATUS = {0: "FAR_OK", 1: "FAR_E_INVALID_ARG", 2: "FAR_E_UNSUPPORTED_PROFILE", 3: "FAR_E_BAD_TIME",
          4: "FAR_E_TOO_LARGE", 5: "FAR_E_CUDA", 6: "FAR_E_OOM"}

STAGES = ("prep", "member0", "members", "winner", "finish", "overflow", "fused", "stream", "check")  # FAR_STAGE_*

SLOT_DT = np.dtype([("node", "u1"), ("size_used", "u1"), ("pad", "u1", 2), ("start", "<i4")])
RESULT_DT = np.dtype([("makespan", "<i4"), ("makespan_phase2", "<i4"), ("alloc_index", "<i4"),
                      ("family_size", "<i4"), ("moves", "<i4"), ("swaps", "<i4"), ("iterations", "<i4"),
                      ("reverted", "<i4"), ("status", "<i4"), ("reserved", "<i4"), ("evals", "<i8"),
                      ("events", "<i8")])
EVENT_DT = np.dtype([("kind", "<i4"), ("node", "<i4"), ("start", "<i4"), ("dur", "<i4")])  # far_event
assert SLOT_DT.itemsize == 8 and RESULT_DT.itemsize == 56 and EVENT_DT.itemsize == 16


class FarError(RuntimeError):
    def __init__(self, status, msg=""):
        self.status = status
        super().__init__(f"{STATUS.get(status, status)}: {msg}")


class Opts(C.Structure):
    _fields_ = [("max_iterations", C.c_int32), ("min_improvement_ppm", C.c_int32), ("flags", C.c_uint32)]


_lib = None


def declared_functions() -> list[str]:
    """Function names declared in include/far.h."""
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(far_[a-z_]+)\s*\(", txt)))


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FarError(5, f"{LIB_PATH} not built (run __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        p, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        sig = {
            "far_create": ([C.c_int, p, C.POINTER(p)], C.c_int),
            "far_create_multi": ([C.c_int, i32, p, C.POINTER(p)], C.c_int),
            "far_measure_peak": ([p, i32, C.POINTER(C.c_double)], C.c_int),
            "far_num_gpus": ([p], i32),
            "far_destroy": ([p], None),
            "far_num_sizes": ([p], i32),
            "far_sizes": ([p], C.POINTER(i32)),
            "far_num_nodes": ([p], i32),
            "far_num_slices": ([p], i32),
            "far_node_table": ([p, p, p, p], C.c_int),
            "far_last_error": ([p], C.c_char_p),
            "far_sync": ([p], C.c_int),
            "far_schedule_batch": ([p, p, i32, p, p, p], C.c_int),
            "far_local_search": ([p, p, i32, p, p, p], C.c_int),
            "far_solve_many": ([p, p, i64, i32, p, p, p, p, p], C.c_int),
            "far_solve_many_host": ([p, p, i64, i32, p, p, p, p], C.c_int),
            "far_concat_streams": ([p, p, i64, i32, i32, p, p, p, p, p, p, p], C.c_int),
            "far_schedule_events": ([p, p, i64, i32, p, p, p, p, p, p], C.c_int),
            "far_validate_schedules": ([p, p, i64, i32, p, p, p, p, p, p], C.c_int),
            "far_lower_bounds": ([p, p, i64, i32, p, p, p], C.c_int),
            "far_stage_timing": ([p, i32], C.c_int),
            "far_stage_times": ([p, p], i32),
            "far_launch_count": ([p], i64),
        }
        for name, (a, r) in sig.items():
            f = getattr(L, name)
            f.argtypes, f.restype = a, r
        _lib = L
    return _lib


def _np_ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _t_ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _opts(max_iterations=100, min_improvement_ppm=0, flags=0):
    return Opts(max_iterations, min_improvement_ppm, flags)


class Far:
    """One far_ctx (a MIG profile + reconfiguration costs)."""

    def __init__(self, profile="A100", reconfig_cost=None, gpus=1):
        """profile 'A30' / 'A100' / 'H100'; gpus > 1 (or a profile 'A100x4') = multi-target FAR over
        that many MIG GPUs (far_create_multi)."""
        if isinstance(profile, str) and "x" in profile:
            profile, g = profile.split("x")
            gpus = int(g)
        self.profile = profile
        self.gpus = gpus
        self._h = C.c_void_p()
        cost = None if reconfig_cost is None else np.ascontiguousarray(reconfig_cost, dtype=np.int32)
        self._cost = cost
        rc = lib().far_create_multi(PROFILES.get(profile, -1) if isinstance(profile, str) else int(profile), gpus,
                                    _np_ptr(cost), C.byref(self._h))
        if rc:
            raise FarError(rc, "far_create_multi")
        self.nsizes = lib().far_num_sizes(self._h)
        self.sizes = [lib().far_sizes(self._h)[i] for i in range(self.nsizes)]
        self.nnodes = lib().far_num_nodes(self._h)
        self.nslices = lib().far_num_slices(self._h)

    def close(self):
        if self._h:
            lib().far_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc:
            raise FarError(rc, lib().far_last_error(self._h).decode())

    def node_table(self):
        lo, hi, par = (np.zeros(self.nnodes, np.int32) for _ in range(3))
        self._check(lib().far_node_table(self._h, _np_ptr(lo), _np_ptr(hi), _np_ptr(par)))
        return lo, hi, par

    def measure_peak(self, mode):
        """Microbenchmark (far_measure_peak): 0 alu-pipe int lane-ops/s, 1 alu+fma int lane-ops/s,
        2 shared-memory load bytes/s."""
        v = C.c_double()
        self._check(lib().far_measure_peak(self._h, mode, C.byref(v)))
        return v.value

    def sync(self):
        self._check(lib().far_sync(self._h))

    # -- diagnostics ------------------------------------------------------------------
    def stage_timing(self, enable=True):
        self._check(lib().far_stage_timing(self._h, 1 if enable else 0))

    def stage_times(self):
        """-> (number of timed launches, {stage: device ms summed over them}); resets the sums."""
        ms = np.zeros(len(STAGES), np.float32)
        k = lib().far_stage_times(self._h, _np_ptr(ms))
        if k < 0:
            raise FarError(5, lib().far_last_error(self._h).decode())
        return k, {name: float(v) for name, v in zip(STAGES, ms)}

    def launch_count(self):
        return int(lib().far_launch_count(self._h))

    # -- single batch, host memory -------------------------------------------------
    def schedule_batch(self, times, **kw):
        t = np.ascontiguousarray(times, dtype=np.int32).reshape(-1, self.nsizes)
        n = t.shape[0]
        slots = np.zeros(n, SLOT_DT)
        res = np.zeros(1, RESULT_DT)
        o = _opts(**kw)
        self._check(lib().far_schedule_batch(self._h, _np_ptr(t), n, C.byref(o), _np_ptr(slots), _np_ptr(res)))
        return slots, res[0]

    def local_search(self, times, slots, makespan_phase2=0, **kw):
        t = np.ascontiguousarray(times, dtype=np.int32).reshape(-1, self.nsizes)
        n = t.shape[0]
        s = np.ascontiguousarray(slots, dtype=SLOT_DT).copy()
        res = np.zeros(1, RESULT_DT)
        res["makespan_phase2"] = makespan_phase2
        o = _opts(**kw)
        self._check(lib().far_local_search(self._h, _np_ptr(t), n, C.byref(o), _np_ptr(s), _np_ptr(res)))
        return s, res[0]

    # -- many instances, device memory (torch tensors) ------------------------------
    def solve_many(self, d_times, *, sched=True, res=True, stream=None, out=None, **kw):
        """d_times: int32 CUDA tensor [I][n][nsizes].  Returns (makespan, sched|None, res|None)
        as CUDA tensors (sched: uint8 [I][n][8] viewable as SLOT_DT; res: uint8 [I][56])."""
        import torch
        assert d_times.is_cuda and d_times.dtype == torch.int32 and d_times.is_contiguous()
        I, n = d_times.shape[0], d_times.shape[1]
        dev = d_times.device
        if out is None:
            ms = torch.empty(I, dtype=torch.int32, device=dev)
            sd = torch.empty((I, n, 8), dtype=torch.uint8, device=dev) if sched else None
            rs = torch.empty((I, 56), dtype=torch.uint8, device=dev) if res else None
        else:
            ms, sd, rs = out
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        flags = kw.pop("flags", 0) | (0 if sched else NO_SCHEDULE)
        o = _opts(flags=flags, **kw)
        self._check(lib().far_solve_many(self._h, _t_ptr(d_times), I, n, C.byref(o), _t_ptr(ms), _t_ptr(sd),
                                         _t_ptr(rs), C.c_void_p(st.cuda_stream)))
        return ms, sd, rs

    def solve_many_host(self, times, *, sched=True, res=True, out=None, **kw):
        """times: int32 numpy [I][n][nsizes] (pinned memory recommended).  Synchronous."""
        t = times
        assert t.dtype == np.int32 and t.flags.c_contiguous
        I, n = t.shape[0], t.shape[1]
        if out is None:
            ms = np.zeros(I, np.int32)
            sd = np.zeros((I, n), SLOT_DT) if sched else None
            rs = np.zeros(I, RESULT_DT) if res else None
        else:
            ms, sd, rs = out
        flags = kw.pop("flags", 0) | (0 if sched else NO_SCHEDULE)
        o = _opts(flags=flags, **kw)
        self._check(lib().far_solve_many_host(self._h, _np_ptr(t), I, n, C.byref(o), _np_ptr(ms), _np_ptr(sd),
                                              _np_ptr(rs)))
        return ms, sd, rs

    def concat_streams(self, d_times, *, sched=True, batch_res=True, seam=True, stream=None, **kw):
        """d_times: int32 CUDA tensor [S][B][n][nsizes] -> (stream_makespan int64 [S][2],
        offsets int64 [S][B], sched uint8 [S][B][n][8] | None, batch_res uint8 [S][B][56] | None,
        seam int32 [S][B][4] | None)."""
        import torch
        assert d_times.is_cuda and d_times.dtype == torch.int32 and d_times.is_contiguous()
        S, B, n = d_times.shape[0], d_times.shape[1], d_times.shape[2]
        dev = d_times.device
        sm = torch.empty((S, 2), dtype=torch.int64, device=dev)
        off = torch.empty((S, B), dtype=torch.int64, device=dev)
        sd = torch.empty((S, B, n, 8), dtype=torch.uint8, device=dev) if sched else None
        br = torch.empty((S, B, 56), dtype=torch.uint8, device=dev) if batch_res else None
        se = torch.empty((S, B, 4), dtype=torch.int32, device=dev) if seam else None
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        o = _opts(**kw)
        self._check(lib().far_concat_streams(self._h, _t_ptr(d_times), S, B, n, C.byref(o), _t_ptr(sm),
                                             _t_ptr(off), _t_ptr(sd), _t_ptr(br), _t_ptr(se),
                                             C.c_void_p(st.cuda_stream)))
        return sm, off, sd, br, se


    # -- schedule export and checking (device memory) ----------------------------------
    def schedule_events(self, d_times, d_sched, *, stream=None, flags=0):
        """Reconfiguration events of schedules (include/far.h far_schedule_events).
        d_times int32 [I][n][nsizes], d_sched uint8 [I][n][8] (far_task_slot) CUDA tensors ->
        (events uint8 [I][2*nnodes][16] viewable as EVENT_DT, nev int32 [I], makespan int32 [I])."""
        import torch
        I, n = d_times.shape[0], d_times.shape[1]
        dev = d_times.device
        ev = torch.empty((I, 2 * self.nnodes, 16), dtype=torch.uint8, device=dev)
        nev = torch.empty(I, dtype=torch.int32, device=dev)
        ms = torch.empty(I, dtype=torch.int32, device=dev)
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        o = _opts(flags=flags)
        self._check(lib().far_schedule_events(self._h, _t_ptr(d_times), I, n, _t_ptr(d_sched), C.byref(o), _t_ptr(ev),
                                              _t_ptr(nev), _t_ptr(ms), C.c_void_p(st.cuda_stream)))
        return ev, nev, ms

    def validate_schedules(self, d_times, d_sched, d_events, d_nev, *, stream=None, flags=0):
        """Violation count per schedule (include/far.h far_validate_schedules) -> int32 [I]."""
        import torch
        I, n = d_times.shape[0], d_times.shape[1]
        dev = d_times.device
        viol = torch.empty(I, dtype=torch.int32, device=dev)
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        o = _opts(flags=flags)
        self._check(lib().far_validate_schedules(self._h, _t_ptr(d_times), I, n, _t_ptr(d_sched), C.byref(o),
                                                 _t_ptr(d_events), _t_ptr(d_nev), _t_ptr(viol),
                                                 C.c_void_p(st.cuda_stream)))
        return viol

    def lower_bounds(self, d_times, *, stream=None):
        """-> (sum_min_work int64 [I], max_min_time int32 [I]) CUDA tensors (far_lower_bounds)."""
        import torch
        I, n = d_times.shape[0], d_times.shape[1]
        dev = d_times.device
        w = torch.empty(I, dtype=torch.int64, device=dev)
        h = torch.empty(I, dtype=torch.int32, device=dev)
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        self._check(lib().far_lower_bounds(self._h, _t_ptr(d_times), I, n, _t_ptr(w), _t_ptr(h),
                                           C.c_void_p(st.cuda_stream)))
        return w, h


def events_np(ev_tensor, nev_tensor):
    """-> list of EVENT_DT arrays, one per instance."""
    ev = ev_tensor.cpu().numpy().view(EVENT_DT)[..., 0]
    nev = nev_tensor.cpu().numpy()
    return [ev[i, :max(int(nev[i]), 0)].copy() for i in range(ev.shape[0])]


def slots_np(sd_tensor):
    """uint8 [..., 8] CUDA/CPU tensor -> numpy SLOT_DT array."""
    return sd_tensor.cpu().numpy().view(SLOT_DT)[..., 0]


def results_np(rs_tensor):
    return rs_tensor.cpu().numpy().view(RESULT_DT)[..., 0]
