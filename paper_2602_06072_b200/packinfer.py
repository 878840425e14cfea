"""Thin Python binding of libpackinfer.so (include/packinfer.h) — argument marshalling only.

Every step of the hot path runs inside the library: the planner in C++, relayout / attention /
merge in sm_100a CUDA kernels.  torch is used for device memory, streams and pinned host
memory.  There is NO CPU fallback: if the shared library is missing or was built for another
architecture, every call raises.

Function names mirror the C ABI (packinfer_plan, packinfer_relayout_kv,
packinfer_attention_prefill, packinfer_attention_decode, packinfer_merge); PackedBatch strings
them together for one batch step.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

_LIB_PATH = os.environ.get("PACKINFER_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                             "libpackinfer.so")

PI_OK, PI_EINVAL, PI_ENOSPC, PI_ECUDA, PI_EUNSUP, PI_EREGROUP = 0, -1, -2, -3, -4, -5
PI_BF16, PI_FP32, PI_BF16_OUT_F32 = 0, 1, 2

EXPORTS = [
    "packinfer_strerror", "packinfer_last_error", "packinfer_version", "packinfer_default_config",
    "packinfer_plan", "packinfer_plan_rows", "packinfer_plan_upload", "packinfer_relayout_kv",
    "packinfer_attention_prefill", "packinfer_attention_decode", "packinfer_attention", "packinfer_attention_merge",
    "packinfer_attention_decode_paged",
    "packinfer_merge",
    "packinfer_plan_step", "packinfer_should_regroup", "packinfer_append_kv",
]


class PackInferError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: status {status}: {detail}")
        self.status = status


# ----------------------------------------------------------------------------- C structs
class pi_config(C.Structure):
    _fields_ = [("capacity", C.c_int32), ("num_groups", C.c_int32), ("mem_cap", C.c_int64),
                ("headroom", C.c_int32), ("tile_q", C.c_int32), ("tile_k", C.c_int32),
                ("decode_chunk", C.c_int32), ("gqa_ratio", C.c_int32), ("flags", C.c_int32)]


PI_PLAN_NO_QPACK = 1   # ablation: one Q tile set per request (include/packinfer.h)
PI_PLAN_DPACK = 2      # option: pack short decode suffixes of a group into one decode item
PI_PLAN_PAGED = 4      # ablation (NEXT-4): decode items over logical tokens, read from the paged cache
PI_PLAN_LPT_EXACT = 8  # scheduling hint: exact LPT order of prefill items (few units per SM)


PIECE_DT = np.dtype([("request", "<i4"), ("piece", "<i4"), ("kv_begin", "<i4"), ("kv_len", "<i4"), ("group", "<i4")])
OFFSET_DT = np.dtype([("d_prefix", "<i4"), ("l_prefix", "<i4"), ("d_suffix", "<i4"), ("l_suffix", "<i4")])
GROUP_DT = np.dtype([("base", "<i8"), ("load", "<i4"), ("members", "<i4"), ("cap", "<i4"), ("reserved", "<i4")])
COPY_DT = np.dtype([("src_kind", "<i4"), ("src_id", "<i4"), ("src_begin", "<i4"), ("len", "<i4"), ("dst", "<i8")])
WORK_DT = np.dtype([("kind", "<i4"), ("group", "<i4"), ("row_begin", "<i4"), ("row_count", "<i4"),
                    ("span_begin", "<i4"), ("span_count", "<i4"), ("n_ktiles", "<i4"), ("reserved", "<i4")])
ROW_DT = np.dtype([("q_token", "<i4"), ("lo", "<i4"), ("hi", "<i4"), ("out", "<i4")])
SPAN_DT = np.dtype([("begin", "<i4"), ("len", "<i4")])
SEG_DT = np.dtype([("row_begin", "<i4"), ("count", "<i4"), ("q_token", "<i4"), ("lo", "<i4"), ("hi", "<i4"),
                   ("out", "<i4"), ("kind", "<i4"), ("reserved", "<i4")])
MERGE_DT = np.dtype([("q_token", "<i4"), ("slot_begin", "<i4"), ("slot_count", "<i4"), ("reserved", "<i4")])


class pi_plan(C.Structure):
    _fields_ = [("pieces", C.c_void_p), ("n_pieces", C.c_int32),
                ("offsets", C.c_void_p),
                ("groups", C.c_void_p), ("n_groups", C.c_int32), ("g0", C.c_int32),
                ("copies", C.c_void_p), ("n_copies", C.c_int32),
                ("copy_prefix", C.c_void_p),
                ("prefill_work", C.c_void_p), ("n_prefill_work", C.c_int32),
                ("decode_work", C.c_void_p), ("n_decode_work", C.c_int32),
                ("segs", C.c_void_p), ("n_segs", C.c_int32), ("n_rows", C.c_int32),
                ("spans", C.c_void_p), ("n_spans", C.c_int32),
                ("merges", C.c_void_p), ("n_merges", C.c_int32), ("n_partial_slots", C.c_int32),
                ("slot_merge", C.c_void_p),
                ("buffer_tokens", C.c_int64), ("copy_tokens", C.c_int64),
                ("n_requests", C.c_int32), ("n_prefix", C.c_int32), ("total_q", C.c_int32),
                ("gqa_ratio", C.c_int32),
                ("eta_num", C.c_int64), ("eta_den", C.c_int64),
                ("valid_cells", C.c_int64), ("tile_cells", C.c_int64),
                ("discrepancy", C.c_int32), ("reserved", C.c_int32),
                ("append_pos", C.c_void_p), ("drift", C.c_int64), ("appended_total", C.c_int64),
                ("arena", C.c_void_p), ("arena_bytes", C.c_size_t),
                ("rows_offset", C.c_size_t), ("sched_offset", C.c_size_t), ("device_arena_bytes", C.c_size_t)]


class pi_device_plan(C.Structure):
    _fields_ = [("copies", C.c_void_p), ("copy_prefix", C.c_void_p), ("n_copies", C.c_int32),
                ("copy_tokens", C.c_int64),
                ("prefill_work", C.c_void_p), ("n_prefill_work", C.c_int32),
                ("decode_work", C.c_void_p), ("n_decode_work", C.c_int32),
                ("rows", C.c_void_p), ("spans", C.c_void_p),
                ("merges", C.c_void_p), ("n_merges", C.c_int32), ("n_partial_slots", C.c_int32),
                ("buffer_tokens", C.c_int64),
                ("n_requests", C.c_int32), ("total_q", C.c_int32), ("gqa_ratio", C.c_int32),
                ("tile_k", C.c_int32), ("append_pos", C.c_void_p), ("slot_merge", C.c_void_p),
                ("sched", C.c_void_p)]


_lib = None


def lib():
    """Loads libpackinfer.so (raises if it is missing — there is no fallback)."""
    global _lib
    if _lib is None:
        path = os.environ.get("PACKINFER_LIB") or _LIB_PATH   # read at first load (A/B variants)
        if not os.path.exists(path):
            raise PackInferError(PI_EUNSUP, "load", f"{path} not built (run __graft_entry__.build())")
        L = C.CDLL(path)
        vp, i32, i64, f32 = C.c_void_p, C.c_int32, C.c_int64, C.c_float
        L.packinfer_strerror.restype = C.c_char_p
        L.packinfer_strerror.argtypes = [C.c_int]
        L.packinfer_last_error.restype = C.c_char_p
        L.packinfer_version.restype = C.c_char_p
        L.packinfer_default_config.argtypes = [C.POINTER(pi_config)]
        L.packinfer_plan.restype = C.c_int
        L.packinfer_plan.argtypes = [i32, vp, vp, vp, i32, vp, C.POINTER(pi_config), vp, C.c_size_t,
                                     C.POINTER(pi_plan)]
        L.packinfer_plan_rows.restype = C.c_int
        L.packinfer_plan_rows.argtypes = [C.POINTER(pi_plan), vp, i32]
        L.packinfer_plan_step.restype = C.c_int
        L.packinfer_plan_step.argtypes = [i32, vp, vp, vp, i32, vp, vp, C.POINTER(pi_config), vp, C.c_size_t,
                                          C.POINTER(pi_plan)]
        L.packinfer_should_regroup.restype = C.c_int32
        L.packinfer_should_regroup.argtypes = [i32, i64, i32]
        L.packinfer_append_kv.restype = C.c_int
        L.packinfer_append_kv.argtypes = [C.POINTER(pi_device_plan), vp, vp, i32, i32, i32, i32, C.c_int, vp, vp, vp]
        L.packinfer_plan_upload.restype = C.c_int
        L.packinfer_plan_upload.argtypes = [C.POINTER(pi_plan), vp, C.c_size_t, vp, C.POINTER(pi_device_plan)]
        L.packinfer_relayout_kv.restype = C.c_int
        L.packinfer_relayout_kv.argtypes = [C.POINTER(pi_device_plan), vp, vp, vp, i32, i32, i32, i32, i32, i32,
                                            C.c_int, vp, vp, vp]
        for name in ("packinfer_attention_prefill", "packinfer_attention_decode", "packinfer_attention"):
            f = getattr(L, name)
            f.restype = C.c_int
            f.argtypes = [C.POINTER(pi_device_plan), vp, i64, vp, vp, i32, i32, i32, f32, C.c_int, vp, i64, vp,
                          vp, vp, vp]
        L.packinfer_attention_merge.restype = C.c_int
        L.packinfer_attention_merge.argtypes = [C.POINTER(pi_device_plan), vp, i64, vp, vp, i32, i32, i32, f32, C.c_int,
                                                vp, i64, vp, vp, vp, vp, vp]
        L.packinfer_attention_decode_paged.restype = C.c_int
        L.packinfer_attention_decode_paged.argtypes = [C.POINTER(pi_device_plan), vp, i64, vp, vp, vp, i32, i32, i32, i32,
                                                       i32, i32, i32, i32, f32, C.c_int, vp, i64, vp, vp, vp, vp]
        L.packinfer_merge.restype = C.c_int
        L.packinfer_merge.argtypes = [C.POINTER(pi_device_plan), vp, vp, i32, i32, C.c_int, vp, i64, vp, vp]
        _lib = L
    return _lib


def _check(st: int, where: str):
    if st != PI_OK:
        raise PackInferError(st, where, lib().packinfer_last_error().decode())


def version() -> str:
    return lib().packinfer_version().decode()


def default_config(**kw) -> pi_config:
    cfg = pi_config()
    lib().packinfer_default_config(C.byref(cfg))
    for k, v in kw.items():
        setattr(cfg, k, int(v))
    return cfg


# ----------------------------------------------------------------------------- planning
@dataclass
class HostPlan:
    """Result of packinfer_plan: the C struct plus numpy views of its tables (host arena)."""
    c: pi_plan
    arena: object            # keeps the host arena alive (torch pinned tensor or numpy array)

    def _view(self, name, n, dt):
        ptr = getattr(self.c, name)
        if n == 0 or not ptr:
            return np.zeros(0, dt)
        buf = (C.c_char * (n * dt.itemsize)).from_address(ptr)
        return np.frombuffer(buf, dtype=dt, count=n)

    @property
    def pieces(self): return self._view("pieces", self.c.n_pieces, PIECE_DT)
    @property
    def offsets(self): return self._view("offsets", self.c.n_pieces, OFFSET_DT)
    @property
    def groups(self): return self._view("groups", self.c.n_groups, GROUP_DT)
    @property
    def copies(self): return self._view("copies", self.c.n_copies, COPY_DT)
    @property
    def copy_prefix(self): return self._view("copy_prefix", self.c.n_copies + 1, np.dtype("<i8"))
    @property
    def prefill_work(self): return self._view("prefill_work", self.c.n_prefill_work, WORK_DT)
    @property
    def decode_work(self): return self._view("decode_work", self.c.n_decode_work, WORK_DT)
    @property
    def segs(self): return self._view("segs", self.c.n_segs, SEG_DT)
    @property
    def rows(self):
        """The row table, expanded on the host from the row segments (packinfer_plan_rows; the
        device builds the same table in packinfer_plan_upload)."""
        rows = np.zeros(int(self.c.n_rows), ROW_DT)
        _check(lib().packinfer_plan_rows(C.byref(self.c), rows.ctypes.data if rows.size else None, rows.size),
               "packinfer_plan_rows")
        return rows
    @property
    def spans(self): return self._view("spans", self.c.n_spans, SPAN_DT)
    @property
    def merges(self): return self._view("merges", self.c.n_merges, MERGE_DT)
    @property
    def append_pos(self): return self._view("append_pos", self.c.n_requests, np.dtype("<i4"))


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def packinfer_plan(kv_len, q_len, prefix_id=None, prefix_len=(), cfg: Optional[pi_config] = None,
                   pinned: bool = False, arena=None, appended=None) -> HostPlan:
    """Alg. 1 Parts 1-2 + packed execution domain (two-call sizing handled here).  With `appended`
    (decode tokens appended per request since the consolidation) this is packinfer_plan_step."""
    L = lib()
    kv, q = _i32(kv_len), _i32(q_len)
    app = None if appended is None else _i32(appended)
    n = int(kv.shape[0])
    pid = None if prefix_id is None else _i32(prefix_id)
    pl = _i32(prefix_len) if len(prefix_len) else np.zeros(1, np.int32)
    n_prefix = len(prefix_len)
    cfg = cfg or default_config()
    out = pi_plan()
    ptr = lambda a: None if a is None else a.ctypes.data
    def call(a_ptr, a_bytes):
        if app is None:
            return L.packinfer_plan(n, ptr(kv), ptr(q), ptr(pid), n_prefix, ptr(pl), C.byref(cfg), a_ptr, a_bytes,
                                    C.byref(out))
        return L.packinfer_plan_step(n, ptr(kv), ptr(q), ptr(pid), n_prefix, ptr(pl), ptr(app), C.byref(cfg),
                                     a_ptr, a_bytes, C.byref(out))
    for _ in range(2):
        if arena is None:
            st = call(None, 0)
        else:
            st = call(_arena_ptr(arena), _arena_bytes(arena))
        if st == PI_ENOSPC:
            arena = _alloc_arena(int(out.arena_bytes), pinned)
            continue
        _check(st, "packinfer_plan")
        return HostPlan(out, arena)
    raise PackInferError(PI_ENOSPC, "packinfer_plan", "arena sizing did not converge")


def _alloc_arena(nbytes: int, pinned: bool):
    if pinned:
        import torch
        return torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    return np.empty(nbytes, dtype=np.uint8)


def _arena_ptr(a) -> int:
    return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data


def _arena_bytes(a) -> int:
    return a.numel() if hasattr(a, "numel") else a.nbytes


# ----------------------------------------------------------------------------- device calls
def _stream_ptr(stream) -> Optional[int]:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def packinfer_plan_upload(plan: HostPlan, dev_arena, stream=None) -> pi_device_plan:
    dp = pi_device_plan()
    _check(lib().packinfer_plan_upload(C.byref(plan.c), dev_arena.data_ptr(), dev_arena.numel(),
                                       _stream_ptr(stream), C.byref(dp)), "packinfer_plan_upload")
    return dp


def _dt(t) -> int:
    import torch
    if t.dtype == torch.bfloat16:
        return PI_BF16
    if t.dtype == torch.float32:
        return PI_FP32
    raise PackInferError(PI_EUNSUP, "dtype", f"unsupported dtype {t.dtype}")


def packinfer_relayout_kv(dp: pi_device_plan, k_paged, v_paged, block_table, k_buf, v_buf,
                          hkv_begin: int = 0, hkv_count: Optional[int] = None, stream=None):
    nb, page, hkv_total, d = k_paged.shape
    hkv_count = hkv_total - hkv_begin if hkv_count is None else hkv_count
    _check(lib().packinfer_relayout_kv(C.byref(dp), k_paged.data_ptr(), v_paged.data_ptr(), block_table.data_ptr(),
                                       block_table.shape[1], page, hkv_total, hkv_begin, hkv_count, d, _dt(k_paged),
                                       k_buf.data_ptr(), v_buf.data_ptr(), _stream_ptr(stream)),
           "packinfer_relayout_kv")


def _attention(fn, name, dp, q, k_buf, v_buf, out, lse, partial_o, partial_lse, gqa_ratio, scale, stream):
    import torch
    hkv_count, _, d = k_buf.shape
    dt = _dt(q)
    if dt == PI_BF16 and out.dtype == torch.float32:
        dt = PI_BF16_OUT_F32
    _check(getattr(lib(), fn)(C.byref(dp), q.data_ptr(), q.stride(0), k_buf.data_ptr(), v_buf.data_ptr(),
                              hkv_count, gqa_ratio, d, float(scale), dt, out.data_ptr(), out.stride(0),
                              None if lse is None else lse.data_ptr(),
                              None if partial_o is None else partial_o.data_ptr(),
                              None if partial_lse is None else partial_lse.data_ptr(), _stream_ptr(stream)), name)


def packinfer_attention_prefill(dp, q, k_buf, v_buf, out, lse=None, partial_o=None, partial_lse=None,
                                gqa_ratio: int = 1, scale: float = 0.0, stream=None):
    _attention("packinfer_attention_prefill", "packinfer_attention_prefill", dp, q, k_buf, v_buf, out, lse,
               partial_o, partial_lse, gqa_ratio, scale, stream)


def packinfer_attention_decode(dp, q, k_buf, v_buf, out, lse=None, partial_o=None, partial_lse=None,
                               gqa_ratio: int = 1, scale: float = 0.0, stream=None):
    _attention("packinfer_attention_decode", "packinfer_attention_decode", dp, q, k_buf, v_buf, out, lse,
               partial_o, partial_lse, gqa_ratio, scale, stream)


def packinfer_attention(dp, q, k_buf, v_buf, out, lse=None, partial_o=None, partial_lse=None,
                        gqa_ratio: int = 1, scale: float = 0.0, stream=None):
    """Fused: one launch over the plan's prefill and decode work items (include/packinfer.h)."""
    _attention("packinfer_attention", "packinfer_attention", dp, q, k_buf, v_buf, out, lse,
               partial_o, partial_lse, gqa_ratio, scale, stream)


def packinfer_attention_merge(dp, q, k_buf, v_buf, out, lse, partial_o, partial_lse, merge_counters,
                              gqa_ratio: int = 1, scale: float = 0.0, stream=None):
    """Fully fused (include/packinfer.h): one launch over prefill + decode work items with the LSE
    merge of split rows inside it (last arriver); merge_counters: int32 zeros [n_merges * Hq_local]."""
    import torch
    hkv_count, _, d = k_buf.shape
    dt = _dt(q)
    if dt == PI_BF16 and out.dtype == torch.float32:
        dt = PI_BF16_OUT_F32
    _check(lib().packinfer_attention_merge(C.byref(dp), q.data_ptr(), q.stride(0), k_buf.data_ptr(), v_buf.data_ptr(),
                                           hkv_count, gqa_ratio, d, float(scale), dt, out.data_ptr(), out.stride(0),
                                           None if lse is None else lse.data_ptr(),
                                           None if partial_o is None else partial_o.data_ptr(),
                                           None if partial_lse is None else partial_lse.data_ptr(),
                                           None if merge_counters is None else merge_counters.data_ptr(),
                                           _stream_ptr(stream)), "packinfer_attention_merge")


def packinfer_attention_decode_paged(dp, q, k_paged, v_paged, block_table, out, lse=None, partial_o=None,
                                     partial_lse=None, gqa_ratio: int = 1, hkv_begin: int = 0,
                                     hkv_count: Optional[int] = None, scale: float = 0.0, stream=None):
    """NEXT-4 ablation: decode straight from the paged cache (plan made with PI_PLAN_PAGED)."""
    import torch
    nb, page, hkv_total, d = k_paged.shape
    hkv_count = hkv_total - hkv_begin if hkv_count is None else hkv_count
    dt = _dt(q)
    if dt == PI_BF16 and out.dtype == torch.float32:
        dt = PI_BF16_OUT_F32
    _check(lib().packinfer_attention_decode_paged(
        C.byref(dp), q.data_ptr(), q.stride(0), k_paged.data_ptr(), v_paged.data_ptr(), block_table.data_ptr(),
        block_table.shape[1], page, nb, hkv_total, hkv_begin, hkv_count, gqa_ratio, d, float(scale), dt,
        out.data_ptr(), out.stride(0), None if lse is None else lse.data_ptr(),
        None if partial_o is None else partial_o.data_ptr(), None if partial_lse is None else partial_lse.data_ptr(),
        _stream_ptr(stream)), "packinfer_attention_decode_paged")


def packinfer_should_regroup(steps: int, drift: int, capacity: int) -> bool:
    """Eq. 4: t * dL >= C / 2."""
    return bool(lib().packinfer_should_regroup(int(steps), int(drift), int(capacity)))


def packinfer_append_kv(dp: pi_device_plan, k_new, v_new, k_buf, v_buf, hkv_begin: int = 0,
                        hkv_count: Optional[int] = None, stream=None):
    """k_new / v_new: [n_requests, Hkv_total, d] — one new decode token per request."""
    n, hkv_total, d = k_new.shape
    hkv_count = hkv_total - hkv_begin if hkv_count is None else hkv_count
    _check(lib().packinfer_append_kv(C.byref(dp), k_new.data_ptr(), v_new.data_ptr(), hkv_total, hkv_begin,
                                     hkv_count, d, _dt(k_new), k_buf.data_ptr(), v_buf.data_ptr(),
                                     _stream_ptr(stream)), "packinfer_append_kv")


def packinfer_merge(dp, partial_o, partial_lse, out, lse=None, stream=None):
    n_slots, hq, d = partial_o.shape
    _check(lib().packinfer_merge(C.byref(dp), partial_o.data_ptr(), partial_lse.data_ptr(), hq, d, _dt(out),
                                 out.data_ptr(), out.stride(0), None if lse is None else lse.data_ptr(),
                                 _stream_ptr(stream)), "packinfer_merge")


# ----------------------------------------------------------------------------- one batch step
class PackedBatch:
    """Plans a batch once and runs the hot path: upload -> relayout -> prefill -> decode -> merge.

    q: [total_q, Hq_local, d] (varlen, request order); k/v_paged: [blocks, page, Hkv, d]; the
    local KV heads are [hkv_begin, hkv_begin + hkv_count) (KV-head sharding)."""

    def __init__(self, kv_len, q_len, prefix_id, prefix_len, hkv_count: int, gqa_ratio: int, head_dim: int,
                 dtype, device, capacity: int = 8192, headroom: int = 0, num_groups: int = 0,
                 decode_chunk: int = 1024, mem_cap: int = 0, flags: Optional[int] = None):
        import torch
        kw = {} if flags is None else {"flags": flags}   # None: packinfer_default_config's flags
        self.cfg = default_config(capacity=capacity, headroom=headroom, num_groups=num_groups,
                                  decode_chunk=decode_chunk, gqa_ratio=gqa_ratio, mem_cap=mem_cap, **kw)
        self.args = (kv_len, q_len, prefix_id, prefix_len)
        self.plan = packinfer_plan(kv_len, q_len, prefix_id, prefix_len, self.cfg, pinned=True)
        # Two pinned host arenas alternate: a plan is never rewritten while its asynchronous upload
        # may still be reading it (each upload records an event; replanning into an arena waits on it).
        self._arenas = [self.plan.arena, None]
        self._events = [None, None]
        self._slot = 0
        self.device = torch.device(device)
        self.hkv, self.r, self.d, self.dtype = hkv_count, gqa_ratio, head_dim, dtype
        c = self.plan.c
        self.dev_arena = torch.empty(max(int(c.device_arena_bytes), 256), dtype=torch.uint8, device=self.device)
        self.dp = packinfer_plan_upload(self.plan, self.dev_arena)
        self._events[0] = torch.cuda.Event()
        self._events[0].record()
        bt = max(int(c.buffer_tokens), 1)
        self.k_buf = torch.empty((hkv_count, bt, head_dim), dtype=dtype, device=self.device)
        self.v_buf = torch.empty((hkv_count, bt, head_dim), dtype=dtype, device=self.device)
        self.partial_o = self.partial_lse = None
        self._ensure_partials()

    def _ensure_partials(self):
        """partial_o / partial_lse hold at least the current plan's n_partial_slots rows."""
        import torch
        ns = max(int(self.plan.c.n_partial_slots), 1)
        hq = self.hkv * self.r
        if self.partial_o is None or self.partial_o.shape[0] < ns:
            self.partial_o = torch.empty((ns, hq, self.d), dtype=torch.float32, device=self.device)
            self.partial_lse = torch.empty((ns, hq), dtype=torch.float32, device=self.device)
        nm = max(int(self.plan.c.n_merges), 1) * hq
        if getattr(self, "merge_counters", None) is None or self.merge_counters.numel() < nm:
            # zero once; the in-kernel merge leaves them zero after every launch
            self.merge_counters = torch.zeros(nm, dtype=torch.int32, device=self.device)

    def replan(self, stream=None, appended=None, upload: bool = True):
        """Host planning + plan upload (the per-step host part of the hot path).  `appended`:
        decode tokens appended per request since the last consolidation (packinfer_plan_step).
        upload=False: host planning only - the upload is then part of the step's CUDA graph
        (graph_run)."""
        import torch
        kv_len, q_len, prefix_id, prefix_len = self.args
        s = self._slot = 1 - self._slot
        if self._events[s] is not None:
            self._events[s].synchronize()          # the upload that last read this arena is done
        if self._arenas[s] is None:
            self._arenas[s] = _alloc_arena(int(self.plan.c.arena_bytes), pinned=True)
        self.plan = packinfer_plan(kv_len, q_len, prefix_id, prefix_len, self.cfg, arena=self._arenas[s],
                                   appended=appended)
        self._arenas[s] = self.plan.arena          # may have grown
        if int(self.plan.c.device_arena_bytes) > self.dev_arena.numel():
            self.dev_arena = torch.empty(int(self.plan.c.device_arena_bytes), dtype=torch.uint8, device=self.device)
        if upload:
            self.dp = packinfer_plan_upload(self.plan, self.dev_arena, stream)
        # appended tokens can push a decode suffix across a decode_chunk boundary: more decode items,
        # more partial slots (the kernels index partial_o / partial_lse by the plan's slot ids)
        self._ensure_partials()
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream() if stream is None else stream)
        self._events[s] = ev

    # ------------------------------------------------------------------ CUDA graph of a step
    def _graph_key(self, tensors, relayout):
        """What a captured step depends on besides the plan tables' CONTENTS: the plan's shape
        (table counts and arena offsets fix every kernel parameter and device pointer) and the
        buffers the graph reads and writes."""
        c = self.plan.c
        shape = (int(c.arena_bytes), int(c.device_arena_bytes), int(c.n_segs), int(c.n_rows),
                 int(c.n_prefill_work), int(c.n_decode_work), int(c.n_spans), int(c.n_merges),
                 int(c.n_partial_slots), int(c.n_copies), int(c.buffer_tokens), int(c.rows_offset),
                 int(c.sched_offset), int(c.total_q))
        ptrs = tuple(0 if t is None else int(t.data_ptr()) for t in tensors)
        return shape + ptrs + (bool(relayout), _arena_ptr(self._arenas[self._slot]), int(self.dev_arena.data_ptr()),
                               int(self.partial_o.data_ptr()))

    def graph_run(self, q, out, lse=None, k_paged=None, v_paged=None, block_table=None, hkv_begin: int = 0,
                  relayout: bool = False):
        """The device part of one step as ONE CUDA graph launch on the current stream: plan upload
        (H2D of the host tables + row expansion) [+ KV relayout] + ONE attention launch + LSE merge.
        Call after replan(upload=False).  A graph is captured per host-arena slot and replayed while
        the plan's shape and the buffers stay the same (e.g. every decode step between regroups,
        whose tables change only in content); a new shape captures another graph (up to 16 are kept,
        so a loop that cycles through a few shapes replays all of them).  The memcpy node reads the
        pinned host arena at replay time, so the tables of THIS step are what the kernels see."""
        import torch
        if not hasattr(self, "_graphs"):
            self._graphs = {}                     # (slot, key) -> graph, most recent last
        tens = (q, out, lse, k_paged, v_paged, block_table, self.k_buf, self.v_buf)
        gk = (self._slot,) + self._graph_key(tens, relayout)
        g = self._graphs.pop(gk, None)
        self.graph_captures = getattr(self, "graph_captures", 0)
        if g is None:
            g = torch.cuda.CUDAGraph()
            cur = torch.cuda.current_stream()
            cs = torch.cuda.Stream(device=self.device)
            cs.wait_stream(cur)
            with torch.cuda.stream(cs):
                g.capture_begin()
                try:
                    dp = packinfer_plan_upload(self.plan, self.dev_arena, cs)
                    if relayout:
                        packinfer_relayout_kv(dp, k_paged, v_paged, block_table, self.k_buf, self.v_buf, hkv_begin,
                                              self.hkv, cs)
                    packinfer_attention(dp, q, self.k_buf, self.v_buf, out, lse, self.partial_o, self.partial_lse,
                                        self.r, 0.0, cs)
                    packinfer_merge(dp, self.partial_o, self.partial_lse, out, lse, cs)
                finally:
                    g.capture_end()
            cur.wait_stream(cs)
            self.graph_captures += 1
            self._dp_of = getattr(self, "_dp_of", {})
            self._dp_of[gk] = dp
            while len(self._graphs) >= 16:        # a decode loop cycles through a few plan shapes
                self._graphs.pop(next(iter(self._graphs)))
        self._graphs[gk] = g
        self.dp = self._dp_of[gk]
        g.replay()
        ev = torch.cuda.Event()
        ev.record()
        self._events[self._slot] = ev            # the replay's memcpy reads this host arena

    def append(self, k_new, v_new, hkv_begin: int = 0, stream=None):
        """Write one new decode token per request into its headroom slot (current plan)."""
        packinfer_append_kv(self.dp, k_new, v_new, self.k_buf, self.v_buf, hkv_begin, self.hkv, stream)

    def run(self, q, k_paged, v_paged, block_table, out, lse=None, hkv_begin: int = 0, stream=None,
            relayout: bool = True, fused: bool = True, kernel_merge: Optional[bool] = None):
        """relayout -> attention -> merge.  fused: ONE attention launch over prefill and decode work
        items (packinfer_attention); else one launch per kind (prefill, then decode).  kernel_merge
        (default False): the LSE merge of split rows inside that launch (packinfer_attention_merge)
        instead of a packinfer_merge launch (bitwise equal; the separate launch is faster on long
        split rows, profiles/r02b)."""
        if relayout:
            packinfer_relayout_kv(self.dp, k_paged, v_paged, block_table, self.k_buf, self.v_buf,
                                  hkv_begin, self.hkv, stream)
        if kernel_merge is None:
            kernel_merge = False
        if fused and kernel_merge:
            packinfer_attention_merge(self.dp, q, self.k_buf, self.v_buf, out, lse, self.partial_o,
                                      self.partial_lse, self.merge_counters, self.r, 0.0, stream)
            return
        if fused:
            packinfer_attention(self.dp, q, self.k_buf, self.v_buf, out, lse, self.partial_o,
                                self.partial_lse, self.r, 0.0, stream)
        else:
            packinfer_attention_prefill(self.dp, q, self.k_buf, self.v_buf, out, lse, self.partial_o,
                                        self.partial_lse, self.r, 0.0, stream)
            packinfer_attention_decode(self.dp, q, self.k_buf, self.v_buf, out, lse, self.partial_o,
                                       self.partial_lse, self.r, 0.0, stream)
        packinfer_merge(self.dp, self.partial_o, self.partial_lse, out, lse, stream)
