"""ctypes mirror of the kvrail C-ABI (include/kvrail_c.h, include/kvr_cuda.h).

This is the Python face of the drop-in boundary: the same verbs, argument
meaning and error behaviour as the reference C++ API (kvrail::Pager,
stage/reduce, the scenario Driver; /root/reference/proj/include/kvrail/*.hpp),
bound to the in-tree shared library ``lib/libkvrail.so``. The binding factory
is parameterised by symbol prefix so the parity tests can drive the reference
oracle (``oracle/_ref/libkvrail_ref.so``, prefix ``kvr_ref_``) through the very
same classes.

There is no fallback: if the native library is missing, importing this module
raises.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import Iterable, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "lib")
LIB_PATH = os.path.join(LIB_DIR, "libkvrail.so")

# ---- error taxonomy (types.hpp:45-68 order; status = 1 + code) -------------
ERRC_NAMES = [
    "OutOfPages", "PrefixOutOfRange", "AliasOverlap", "UnmappedRange", "FutureDelta",
    "UnknownSession", "SessionClosed", "EmptyChunk", "DimensionMismatch", "ShapeViolation",
    "MultiCommit", "UnmappedBlock", "ParseError", "NonMonotoneTime", "EmptyStream",
    "UnknownRegime", "InfeasibleSpec", "WorkloadAuditFailed", "EmptyRun", "WorkloadMismatch",
    "BadConfig", "IoError",
]
KVR_E_CUDA = 100


class KvrailError(RuntimeError):
    """kvrail::Error: ``code`` is the Errc name (e.g. "OutOfPages")."""

    def __init__(self, status: int, message: str):
        if 1 <= status <= len(ERRC_NAMES):
            code = ERRC_NAMES[status - 1]
        elif status == KVR_E_CUDA:
            code = "CudaError"
        else:
            code = "InternalError"
        super().__init__(message)
        self.status = status
        self.code = code


# ---- POD structs ------------------------------------------------------------
class PagerConfig(C.Structure):
    _fields_ = [("page_bytes", C.c_uint64), ("arena_pages", C.c_uint32), ("layers", C.c_uint32),
                ("kv_head_dim", C.c_uint32), ("elem_bytes", C.c_uint32)]

    def token_bytes(self) -> int:
        return 2 * self.layers * self.kv_head_dim * self.elem_bytes

    def tokens_per_page(self) -> int:
        return max(1, self.page_bytes // self.token_bytes())


class TokenRange(C.Structure):
    _fields_ = [("begin", C.c_uint64), ("end", C.c_uint64)]


class ViewEntry(C.Structure):
    _fields_ = [("tok_begin", C.c_uint64), ("tok_end", C.c_uint64), ("block", C.c_uint32),
                ("slot_begin", C.c_uint32)]

    def astuple(self):
        return (self.tok_begin, self.tok_end, self.block, self.slot_begin)


class ViewInfo(C.Structure):
    _fields_ = [("session", C.c_uint32), ("eos", C.c_uint32), ("epoch", C.c_uint64),
                ("live_tokens", C.c_uint64), ("extent", C.c_uint64), ("n_entries", C.c_uint64)]


class ReservedBlock(C.Structure):
    _fields_ = [("block", C.c_uint32), ("token_capacity", C.c_uint32)]


class ArenaStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in
                ("free_pages", "live_pages", "shared_pages", "reserved_bytes", "active_bytes")]

    def astuple(self):
        return tuple(getattr(self, f) for f, _ in self._fields_)


class WorkCounters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in
                ("commits", "commit_entries_touched", "reserve_calls", "reserve_blocks",
                 "reserve_alloc_steps", "trim_calls", "trim_blocks", "free_list_steps")]

    def astuple(self):
        return tuple(getattr(self, f) for f, _ in self._fields_)


class FreeRun(C.Structure):
    _fields_ = [("head", C.c_uint32), ("length", C.c_uint32)]


class FrameDelta(C.Structure):
    _fields_ = [("session", C.c_uint32), ("trim_eos", C.c_uint32), ("step", C.c_uint64),
                ("reserves", C.POINTER(C.c_uint64)), ("n_reserves", C.c_uint64),
                ("alias_src", C.POINTER(C.c_uint32)), ("alias_prefix", C.POINTER(C.c_uint64)),
                ("n_aliases", C.c_uint64), ("trims", C.POINTER(TokenRange)), ("n_trims", C.c_uint64)]


class StagedSpan(C.Structure):
    _fields_ = [("block", C.c_uint32), ("slot_begin", C.c_uint32), ("slot_count", C.c_uint32)]


class StageNeed(C.Structure):
    _fields_ = [("session", C.c_uint32), ("kind", C.c_uint32), ("span_begin", C.c_uint64),
                ("span_count", C.c_uint64)]


class Descriptor(C.Structure):
    _fields_ = [("phys_offset", C.c_uint64), ("length", C.c_uint64), ("stage_time", C.c_double),
                ("kind", C.c_uint32), ("block", C.c_uint32), ("session", C.c_uint32),
                ("pad_", C.c_uint32)]

    def astuple(self):
        return (self.phys_offset, self.length, self.stage_time, self.kind, self.block, self.session)


class TransportConfig(C.Structure):
    _fields_ = [("merge_threshold", C.c_uint64), ("max_hold", C.c_double),
                ("max_trains_per_step", C.c_uint32), ("merge", C.c_uint32),
                ("run_page_bytes", C.c_uint64), ("run_span_bytes", C.c_uint64)]


class Train(C.Structure):
    _fields_ = [("total_bytes", C.c_uint64), ("oldest_stage_time", C.c_double),
                ("issue_time", C.c_double), ("kind", C.c_uint32), ("reason", C.c_uint32),
                ("desc_begin", C.c_uint64), ("desc_count", C.c_uint64)]


class StepRecord(C.Structure):
    _fields_ = [("step", C.c_uint64), ("live_sessions", C.c_uint32), ("trains", C.c_uint32),
                ("near_trains", C.c_uint32), ("far_trains", C.c_uint32), ("dma_bytes", C.c_uint64),
                ("mean_train_bytes", C.c_double), ("max_hold", C.c_double),
                ("submit_time", C.c_double), ("commit_time", C.c_double),
                ("step_latency", C.c_double), ("reserved_bytes", C.c_uint64),
                ("active_bytes", C.c_uint64), ("commits", C.c_uint32), ("pad_", C.c_uint32),
                ("emitted_tokens", C.c_uint64), ("device_ms", C.c_double),
                ("gather_ms", C.c_double), ("attn_ms", C.c_double), ("phase_ms", C.c_double * 8),
                ("writeback_tokens", C.c_uint64), ("gather_bytes", C.c_uint64),
                ("attn_bytes", C.c_uint64), ("h2d_bytes", C.c_uint64), ("end_ns", C.c_uint64),
                ("global_live", C.c_uint64), ("global_emitted", C.c_uint64),
                ("global_commits", C.c_uint64), ("global_eos", C.c_uint64)]


class Geometry(C.Structure):
    """kvr_geometry (include/kvr_cuda.h)."""
    _fields_ = [("device", C.c_int32), ("elem_kind", C.c_int32), ("elem_bytes", C.c_uint32),
                ("payload_mode", C.c_uint32), ("page_bytes", C.c_uint64),
                ("token_bytes", C.c_uint64), ("arena_pages", C.c_uint32),
                ("tokens_per_page", C.c_uint32), ("layers", C.c_uint32), ("kv_heads", C.c_uint32),
                ("head_dim", C.c_uint32), ("q_heads", C.c_uint32), ("n_slots", C.c_uint32),
                ("near_window", C.c_uint32), ("ring_rows", C.c_uint32), ("far_cap", C.c_uint32),
                ("chunk_tokens", C.c_uint32), ("max_chunks", C.c_uint32),
                ("max_tokens", C.c_uint64), ("seed", C.c_uint64), ("attention", C.c_uint32),
                ("use_graph", C.c_uint32), ("max_desc_bytes", C.c_uint64),
                ("max_scan_descs", C.c_uint32), ("max_trains", C.c_uint32),
                ("utility", C.c_uint32), ("utility_layer", C.c_uint32),
                ("lane_shift", C.c_uint32), ("query_mode", C.c_uint32)]


class MassRun(C.Structure):
    """kvr_mass_run (include/kvr_cuda.h): one block's attention-utility mass."""
    _fields_ = [("block", C.c_uint32), ("mass", C.c_float)]


ELEM_F32, ELEM_F16, ELEM_BF16 = 0, 1, 2
U64P = C.POINTER(C.c_uint64)
U32P = C.POINTER(C.c_uint32)


# ---- library binding --------------------------------------------------------
class Api:
    """Binds the pager / transport / far-view entry points under ``prefix``."""

    def __init__(self, lib: C.CDLL, prefix: str):
        self.lib = lib
        self.prefix = prefix
        g = lambda n: getattr(lib, prefix + n)  # noqa: E731
        self.last_error = g("last_error")
        self.last_error.restype = C.c_char_p
        vp = C.c_void_p
        sig = {
            "pager_create": [C.POINTER(PagerConfig), C.POINTER(vp)],
            "pager_destroy": [vp],
            "pager_config_validate": [C.POINTER(PagerConfig)],
            "pager_create_session": [vp, C.c_uint32],
            "pager_has_session": [vp, C.c_uint32, C.POINTER(C.c_int)],
            "pager_reserve": [vp, C.c_uint32, C.c_uint64, C.POINTER(ReservedBlock), C.c_uint64, U64P],
            "pager_reserve_range": [vp, C.c_uint32, TokenRange, C.POINTER(ReservedBlock), C.c_uint64,
                                    U64P],
            "pager_alias": [vp, C.c_uint32, C.c_uint32, C.c_uint64, U64P],
            "pager_write_tokens": [vp, C.c_uint32, TokenRange, C.c_void_p, C.c_uint64],
            "pager_trim": [vp, C.c_uint32, C.POINTER(TokenRange), C.c_uint64, U64P],
            "pager_trim_eos": [vp, C.c_uint32, U64P],
            "pager_frame_commit": [vp, C.c_uint32, C.c_uint64, U64P],
            "pager_apply_frame": [vp, C.POINTER(FrameDelta), U64P],
            "pager_active_view": [vp, C.c_uint32, C.POINTER(ViewInfo), C.POINTER(ViewEntry),
                                  C.c_uint64],
            "pager_session_eos": [vp, C.c_uint32, C.POINTER(C.c_int)],
            "pager_session_cursor": [vp, C.c_uint32, U64P],
            "pager_next_step": [vp, C.c_uint32, U64P],
            "pager_touched_in_last_commit": [vp, C.c_uint32, U64P],
            "pager_stats": [vp, C.POINTER(ArenaStats)],
            "pager_counters": [vp, C.POINTER(WorkCounters)],
            "pager_read_slots": [vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p],
            "pager_free_runs": [vp, C.POINTER(FreeRun), C.c_uint64, U64P],
            "pager_block_refcount": [vp, C.c_uint32, U32P],
            "stage": [C.POINTER(StageNeed), C.c_uint64, C.POINTER(StagedSpan), C.c_uint64,
                      C.c_uint64, C.c_double, C.POINTER(Descriptor), C.c_uint64, U64P],
            "reduce": [C.POINTER(Descriptor), C.c_uint64, C.POINTER(TransportConfig), C.c_double,
                       C.POINTER(Train), C.c_uint64, U64P, C.POINTER(Descriptor)],
            "summarize_chunk": [C.POINTER(C.c_float), C.c_uint32, C.c_uint64, C.POINTER(C.c_float)],
            "select_chunks": [C.POINTER(C.c_double), C.c_uint64, C.c_uint32, U64P, U64P],
            "attend_history": [C.POINTER(C.c_float), C.c_uint64, C.POINTER(C.c_double), C.c_uint64,
                               C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                               C.POINTER(C.c_float), C.c_uint32, C.c_uint32, C.POINTER(C.c_float)],
        }
        for name, args in sig.items():
            fn = g(name)
            fn.argtypes = args
            fn.restype = C.c_int
            setattr(self, name, self._checked(fn))

    def _checked(self, fn):
        def call(*a):
            rc = fn(*a)
            if rc != 0:
                raise KvrailError(rc, self.last_error().decode(errors="replace"))
            return rc
        return call


_API: Api | None = None
_LIB: C.CDLL | None = None


def native_lib() -> C.CDLL:
    """The product library (loads libkvr_cuda.so through its rpath). Fails loudly."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() first")
        _LIB = C.CDLL(LIB_PATH)
    return _LIB


def api() -> Api:
    global _API
    if _API is None:
        _API = Api(native_lib(), "kvr_")
        _bind_extras(native_lib())
    return _API


def _bind_extras(lib: C.CDLL) -> None:
    vp = C.c_void_p
    sig = {
        "kvr_pager_create_on_device": [C.POINTER(PagerConfig), vp, C.POINTER(vp)],
        "kvr_driver_create": [C.c_char_p, C.c_int, C.POINTER(vp)],
        "kvr_driver_destroy": [vp],
        "kvr_driver_step": [vp, C.POINTER(StepRecord)],
        "kvr_driver_record": [vp, C.c_uint64, C.POINTER(StepRecord)],
        "kvr_driver_sync": [vp],
        "kvr_driver_progress": [vp, U64P, U64P],
        "kvr_driver_steps_csv": [vp, C.c_char_p, C.c_uint64, U64P],
        "kvr_driver_measured_csv": [vp, C.c_char_p, C.c_uint64, U64P],
        "kvr_driver_measured_json": [vp, C.c_char_p, C.c_uint64, U64P],
        "kvr_driver_prefill_backlog": [vp, U64P, U64P],
        "kvr_driver_report_json": [vp, C.c_char_p, C.c_uint64, U64P],
        "kvr_driver_trace": [vp, C.c_char_p, C.c_uint64, U64P],
        "kvr_driver_pager": [vp, C.POINTER(vp)],
        "kvr_driver_live": [vp, U32P, U32P, U64P, C.c_uint64, U64P],
        "kvr_driver_workload_hash": [vp, U64P],
        "kvr_driver_device": [vp, C.POINTER(vp)],
        "kvr_driver_device_check": [vp, U64P, U64P, C.c_char_p, C.c_uint64],
        "kvr_driver_staged_rows": [vp, U64P, U64P, U64P],
        "kvr_driver_fault": [vp, C.c_int, C.c_uint64],
        "kvr_driver_comm_init": [vp, C.c_char_p, C.c_int, C.c_int],
        "kvr_comm_unique_id": [C.c_char_p],
        "kvr_comm_destroy": [vp],
        "kvr_device_open": [C.POINTER(Geometry), C.POINTER(vp)],
        "kvr_device_close": [vp],
        "kvr_device_flush": [vp],
        "kvr_device_geometry": [vp, C.POINTER(Geometry)],
        "kvr_device_bind": [vp, C.c_uint32, C.c_uint32],
        "kvr_device_raw": [vp, C.POINTER(vp)],
        "kvr_device_read_ring_token": [vp, C.c_uint32, C.c_uint64, C.c_void_p],
        "kvr_device_read_page_table": [vp, C.c_uint32, C.c_uint64, C.c_uint64, U32P],
        "kvr_device_read_attention": [vp, C.c_uint32, C.POINTER(C.c_float)],
        "kvr_device_read_query": [vp, C.c_uint32, C.POINTER(C.c_float)],
        "kvr_device_read_far_row": [vp, C.c_uint32, C.c_uint64, C.c_void_p],
        "kvr_device_far_selection": [vp, C.c_uint32, U64P, C.c_uint64, U64P],
        "kvr_device_read_scan": [vp, C.POINTER(Train), C.c_uint64, U64P, C.POINTER(Descriptor),
                                 C.c_uint64, U64P],
        "kvr_device_utility": [vp, C.c_uint64, C.POINTER(MassRun), U32P],
        "kvr_dev_count": [C.POINTER(C.c_int)],
        "kvr_dev_time_attention": [vp, C.c_uint32, C.POINTER(C.c_double)],
        "kvr_dev_time_gather": [vp, C.c_uint32, C.POINTER(C.c_double)],
        "kvr_dev_timeline": [vp, U64P],
        "kvr_dev_read": [vp, C.c_int, C.c_uint64, C.c_uint64, C.c_void_p],
        "kvr_dev_read_staged": [vp, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p],
        "kvr_dev_ring_plane_rows": [vp, U32P],
        "kvr_dev_fault": [vp, C.c_int, C.c_uint64],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    lib.kvr_dev_attention_variant.argtypes = [vp]
    lib.kvr_dev_attention_variant.restype = C.c_char_p
    lib.kvr_dev_step_kernels.argtypes = [vp, C.POINTER(C.c_uint32)]
    lib.kvr_dev_graph_captures.argtypes = [vp, C.POINTER(C.c_uint32)]
    lib.kvr_dev_last_error.restype = C.c_char_p


def check(rc: int) -> None:
    if rc != 0:
        msg = native_lib().kvr_last_error
        msg.restype = C.c_char_p
        raise KvrailError(rc, msg().decode(errors="replace"))


# ---- Pager ------------------------------------------------------------------
class Pager:
    """Mirror of kvrail::Pager (pager.hpp:121-183)."""

    def __init__(self, cfg: PagerConfig, api_: Api | None = None, device: "Device | None" = None,
                 _handle=None):
        self.api = api_ or api()
        self.cfg = cfg
        self._owned = _handle is None
        self.h = C.c_void_p(_handle) if _handle is not None else C.c_void_p()
        if _handle is None:
            if device is not None:
                check(native_lib().kvr_pager_create_on_device(C.byref(cfg), device.h, C.byref(self.h)))
            else:
                self.api.pager_create(C.byref(cfg), C.byref(self.h))

    def close(self):
        if self._owned and self.h:
            self.api.pager_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def create_session(self, s: int):
        self.api.pager_create_session(self.h, s)

    def has_session(self, s: int) -> bool:
        o = C.c_int()
        self.api.pager_has_session(self.h, s, C.byref(o))
        return bool(o.value)

    def reserve(self, s: int, count: int):
        cap = count // max(1, self.cfg.tokens_per_page()) + 2
        buf = (ReservedBlock * cap)()
        n = C.c_uint64()
        self.api.pager_reserve(self.h, s, count, buf, cap, C.byref(n))
        return [(buf[i].block, buf[i].token_capacity) for i in range(n.value)]

    def reserve_range(self, s: int, begin: int, end: int):
        cap = max(0, end - begin) // max(1, self.cfg.tokens_per_page()) + 2
        buf = (ReservedBlock * cap)()
        n = C.c_uint64()
        self.api.pager_reserve_range(self.h, s, TokenRange(begin, end), buf, cap, C.byref(n))
        return [(buf[i].block, buf[i].token_capacity) for i in range(n.value)]

    def alias(self, dst: int, src: int, prefix: int) -> int:
        o = C.c_uint64()
        self.api.pager_alias(self.h, dst, src, prefix, C.byref(o))
        return o.value

    def write_tokens(self, s: int, begin: int, end: int, payload: bytes):
        self.api.pager_write_tokens(self.h, s, TokenRange(begin, end), payload, len(payload))

    def trim(self, s: int, ranges: Sequence[tuple[int, int]]) -> int:
        arr = (TokenRange * max(1, len(ranges)))(*[TokenRange(a, b) for a, b in ranges])
        o = C.c_uint64()
        self.api.pager_trim(self.h, s, arr, len(ranges), C.byref(o))
        return o.value

    def trim_eos(self, s: int) -> int:
        o = C.c_uint64()
        self.api.pager_trim_eos(self.h, s, C.byref(o))
        return o.value

    def frame_commit(self, s: int, step: int) -> int:
        o = C.c_uint64()
        self.api.pager_frame_commit(self.h, s, step, C.byref(o))
        return o.value

    def apply_frame(self, session: int, step: int, reserves=(), aliases=(), trims=(),
                    trim_eos=False) -> int:
        res = (C.c_uint64 * max(1, len(reserves)))(*reserves)
        asrc = (C.c_uint32 * max(1, len(aliases)))(*[a for a, _ in aliases])
        apre = (C.c_uint64 * max(1, len(aliases)))(*[p for _, p in aliases])
        tr = (TokenRange * max(1, len(trims)))(*[TokenRange(a, b) for a, b in trims])
        d = FrameDelta(session, int(trim_eos), step, res, len(reserves), asrc, apre, len(aliases),
                       tr, len(trims))
        o = C.c_uint64()
        self.api.pager_apply_frame(self.h, C.byref(d), C.byref(o))
        return o.value

    def active_view(self, s: int):
        info = ViewInfo()
        self.api.pager_active_view(self.h, s, C.byref(info), None, 0)
        buf = (ViewEntry * max(1, info.n_entries))()
        self.api.pager_active_view(self.h, s, C.byref(info), buf, info.n_entries)
        return {"session": info.session, "epoch": info.epoch, "live_tokens": info.live_tokens,
                "extent": info.extent, "eos": bool(info.eos),
                "entries": [buf[i].astuple() for i in range(info.n_entries)]}

    def session_eos(self, s: int) -> bool:
        o = C.c_int()
        self.api.pager_session_eos(self.h, s, C.byref(o))
        return bool(o.value)

    def session_cursor(self, s: int) -> int:
        o = C.c_uint64()
        self.api.pager_session_cursor(self.h, s, C.byref(o))
        return o.value

    def next_step(self, s: int) -> int:
        o = C.c_uint64()
        self.api.pager_next_step(self.h, s, C.byref(o))
        return o.value

    def touched_in_last_commit(self, s: int) -> int:
        o = C.c_uint64()
        self.api.pager_touched_in_last_commit(self.h, s, C.byref(o))
        return o.value

    def stats(self) -> ArenaStats:
        o = ArenaStats()
        self.api.pager_stats(self.h, C.byref(o))
        return o

    def counters(self) -> WorkCounters:
        o = WorkCounters()
        self.api.pager_counters(self.h, C.byref(o))
        return o

    def read_slots(self, block: int, slot: int, count: int) -> bytes:
        buf = C.create_string_buffer(count * self.cfg.token_bytes())
        self.api.pager_read_slots(self.h, block, slot, count, buf)
        return buf.raw

    def free_runs(self):
        n = C.c_uint64()
        self.api.pager_free_runs(self.h, None, 0, C.byref(n))
        buf = (FreeRun * max(1, n.value))()
        self.api.pager_free_runs(self.h, buf, n.value, C.byref(n))
        return [(buf[i].head, buf[i].length) for i in range(n.value)]

    def block_refcount(self, b: int) -> int:
        o = C.c_uint32()
        self.api.pager_block_refcount(self.h, b, C.byref(o))
        return o.value

    def reconstruct_view(self, s: int) -> bytes:
        """reconstruct_view (sim_engine.cpp:74-86)."""
        v = self.active_view(s)
        return b"".join(self.read_slots(b, sb, e - t) for t, e, b, sb in v["entries"])


# ---- transport ----------------------------------------------------------------
def stage(needs: Sequence[tuple[int, int, Sequence[tuple[int, int, int]]]], page_bytes: int,
          token_bytes: int, now: float, api_: Api | None = None):
    """stage(): needs = [(session, kind, [(block, slot_begin, slot_count), ...]), ...]."""
    a = api_ or api()
    spans, recs = [], []
    for sess, kind, sp in needs:
        recs.append(StageNeed(sess, kind, len(spans), len(sp)))
        spans.extend(StagedSpan(*x) for x in sp)
    nn = (StageNeed * max(1, len(recs)))(*recs)
    ss = (StagedSpan * max(1, len(spans)))(*spans)
    cap = len(spans) + 1
    out = (Descriptor * cap)()
    n = C.c_uint64()
    a.stage(nn, len(recs), ss, page_bytes, token_bytes, now, out, cap, C.byref(n))
    return [out[i].astuple() for i in range(n.value)]


def reduce(descs: Sequence[tuple], tau: int, max_hold: float, merge: bool, now: float,
           api_: Api | None = None, run_page: int = 0, run_span: int = 0):
    """reduce(): returns [(kind, reason, total_bytes, oldest, issue, [descs...]), ...].
    run_page / run_span: the B200 page-run merge (TransportConfig::run_page_bytes)."""
    a = api_ or api()
    arr = (Descriptor * max(1, len(descs)))(*[
        Descriptor(off, ln, st, k, b, s, 0) for off, ln, st, k, b, s in descs])
    cfg = TransportConfig(tau, max_hold, 2, int(merge), run_page, run_span)
    cap = len(descs) + 1
    trains = (Train * cap)()
    ordered = (Descriptor * max(1, len(descs)))()
    n = C.c_uint64()
    a.reduce(arr, len(descs), C.byref(cfg), now, trains, cap, C.byref(n), ordered)
    out = []
    for i in range(n.value):
        t = trains[i]
        ds = [ordered[k].astuple() for k in range(t.desc_begin, t.desc_begin + t.desc_count)]
        out.append((t.kind, t.reason, t.total_bytes, t.oldest_stage_time, t.issue_time, ds))
    return out


# ---- device -------------------------------------------------------------------
def comm_unique_id() -> bytes:
    """A fresh NCCL unique id (128 bytes) for kvr_driver_comm_init; create it on one
    rank and hand it to the others (e.g. with a torch.distributed broadcast)."""
    api()
    buf = C.create_string_buffer(128)
    check(native_lib().kvr_comm_unique_id(buf))
    return buf.raw


def device_count() -> int:
    n = C.c_int(0)
    api()
    native_lib().kvr_dev_count(C.byref(n))
    return n.value


class Device:
    """A B200 device context (kvrail::DeviceStep)."""

    def __init__(self, geometry: Geometry | None = None, _handle=None, _owner=None):
        api()
        self._owner = _owner
        self.h = C.c_void_p()
        if _handle is not None:
            self.h = C.c_void_p(_handle)
            self._owned = False
        else:
            check(native_lib().kvr_device_open(C.byref(geometry), C.byref(self.h)))
            self._owned = True
        self.geometry = Geometry()
        check(native_lib().kvr_device_geometry(self.h, C.byref(self.geometry)))

    def close(self):
        if self._owned and self.h:
            check(native_lib().kvr_device_close(self.h))
            self.h = C.c_void_p()

    def flush(self):
        check(native_lib().kvr_device_flush(self.h))

    def bind(self, session: int, slot: int):
        check(native_lib().kvr_device_bind(self.h, session, slot))

    def raw(self):
        r = C.c_void_p()
        check(native_lib().kvr_device_raw(self.h, C.byref(r)))
        return r

    def row_bytes(self) -> int:
        g = self.geometry
        return 2 * g.kv_heads * g.head_dim * g.elem_bytes

    def ring_plane(self, slot: int, layer: int) -> tuple[bytes, int]:
        """Raw rows of one (slot, layer) ring plane (ring_rows + guard rows) and the
        plane's row count."""
        g = self.geometry
        rows = C.c_uint32()
        check(native_lib().kvr_dev_ring_plane_rows(self.raw(), C.byref(rows)))
        n = rows.value * self.row_bytes()
        buf = C.create_string_buffer(n)
        check(native_lib().kvr_dev_read(self.raw(), 1, (slot * g.layers + layer) * n, n, buf))
        return buf.raw, rows.value

    def ring_token(self, slot: int, token: int) -> bytes:
        buf = C.create_string_buffer(self.geometry.token_bytes)
        check(native_lib().kvr_device_read_ring_token(self.h, slot, token, buf))
        return buf.raw

    def far_row(self, slot: int, chunk: int) -> bytes:
        buf = C.create_string_buffer(self.geometry.token_bytes)
        check(native_lib().kvr_device_read_far_row(self.h, slot, chunk, buf))
        return buf.raw

    def far_selection(self, slot: int) -> list[int]:
        buf = (C.c_uint64 * 4096)()
        n = C.c_uint64()
        check(native_lib().kvr_device_far_selection(self.h, slot, buf, 4096, C.byref(n)))
        return list(buf)[:n.value]

    def utility(self, step: int) -> list[list[tuple[int, float]]]:
        """K-mass observations of `step` per device slot: [(block, mass), ...]."""
        g = self.geometry
        runs = (MassRun * (g.n_slots * g.near_window))()
        counts = (C.c_uint32 * g.n_slots)()
        check(native_lib().kvr_device_utility(self.h, step, runs, counts))
        return [[(runs[s * g.near_window + i].block, runs[s * g.near_window + i].mass)
                 for i in range(counts[s])] for s in range(g.n_slots)]

    def page_table(self, slot: int, begin: int, count: int):
        buf = (C.c_uint32 * max(1, count))()
        check(native_lib().kvr_device_read_page_table(self.h, slot, begin, count, buf))
        return list(buf)[:count]

    def _floats(self, fn, slot):
        g = self.geometry
        n = g.layers * g.q_heads * g.head_dim
        buf = (C.c_float * n)()
        check(fn(self.h, slot, buf))
        return list(buf)

    def attention(self, slot: int):
        """[layer][q_head][head_dim] flattened (f32)."""
        return self._floats(native_lib().kvr_device_read_attention, slot)

    def query(self, slot: int):
        return self._floats(native_lib().kvr_device_read_query, slot)

    def scan(self):
        cap = 4096
        trains = (Train * cap)()
        descs = (Descriptor * cap)()
        nt, nd = C.c_uint64(), C.c_uint64()
        check(native_lib().kvr_device_read_scan(self.h, trains, cap, C.byref(nt), descs, cap,
                                                C.byref(nd)))
        d = [descs[i].astuple() for i in range(nd.value)]
        return [(t.kind, t.reason, t.total_bytes, t.oldest_stage_time, t.issue_time,
                 d[t.desc_begin:t.desc_begin + t.desc_count]) for t in trains[:nt.value]]

    def time_attention(self, iters: int = 10) -> float:
        ms = C.c_double()
        check(native_lib().kvr_dev_time_attention(self.raw(), iters, C.byref(ms)))
        return ms.value

    def time_gather(self, iters: int = 10) -> float:
        ms = C.c_double()
        check(native_lib().kvr_dev_time_gather(self.raw(), iters, C.byref(ms)))
        return ms.value

    TIMELINE_NAMES = ("apply", "queries", "scan", "write_hot", "far_map_prime", "gather", "attention",
                      "write_cold", "presum", "attention_entry")

    def timeline(self) -> dict:
        """Diagnostic (KVR_TIMELINE=1 at open): {kernel: (start_ns, end_ns)} since the last
        call, %globaltimer of the first CTA start / last warp exit; resets."""
        buf = (C.c_uint64 * 32)()
        check(native_lib().kvr_dev_timeline(self.raw(), buf))
        return {n: (buf[2 * i], buf[2 * i + 1]) for i, n in enumerate(self.TIMELINE_NAMES)
                if buf[2 * i + 1] != 0}

    def attention_variant(self) -> str:
        return native_lib().kvr_dev_attention_variant(self.raw()).decode()

    def step_kernels(self) -> int:
        """Kernel nodes in the captured step graph (launches per step)."""
        n = C.c_uint32()
        check(native_lib().kvr_dev_step_kernels(self.raw(), C.byref(n)))
        return n.value

    def graph_captures(self) -> int:
        """Step graphs captured so far (2 after warm-up, never more)."""
        n = C.c_uint32()
        check(native_lib().kvr_dev_graph_captures(self.raw(), C.byref(n)))
        return n.value


# ---- scenario driver ------------------------------------------------------------
class Driver:
    """Steppable twin of the reference Driver (scenario.cpp:124-683) behind the C-ABI."""

    def __init__(self, config: dict | str, device: int = -1):
        api()
        text = config if isinstance(config, str) else json.dumps(config)
        self.config = json.loads(text)
        self.h = C.c_void_p()
        check(native_lib().kvr_driver_create(text.encode(), device, C.byref(self.h)))

    def close(self):
        if self.h:
            check(native_lib().kvr_driver_destroy(self.h))
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self) -> StepRecord:
        r = StepRecord()
        check(native_lib().kvr_driver_step(self.h, C.byref(r)))
        return r

    def record(self, step: int) -> StepRecord:
        """Record of an executed step with its device measurements."""
        r = StepRecord()
        check(native_lib().kvr_driver_record(self.h, step, C.byref(r)))
        return r

    def sync(self):
        check(native_lib().kvr_driver_sync(self.h))

    def progress(self) -> tuple[int, int]:
        a, b = C.c_uint64(), C.c_uint64()
        check(native_lib().kvr_driver_progress(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def run(self) -> list[StepRecord]:
        out = []
        done, total = self.progress()
        for _ in range(total - done):
            out.append(self.step())
        return out

    def _text(self, fn) -> str:
        n = C.c_uint64()
        check(fn(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        check(fn(self.h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def steps_csv(self) -> str:
        return self._text(native_lib().kvr_driver_steps_csv)

    def report_json(self) -> str:
        return self._text(native_lib().kvr_driver_report_json)

    def measured_csv(self) -> str:
        """steps.csv columns + the B200 measurements of every executed step."""
        return self._text(native_lib().kvr_driver_measured_csv)

    def prefill_backlog(self) -> tuple[int, int]:
        """(cold prompt tokens queued, tokens dropped unwritten) under b200.prefill_budget."""
        q, dr = C.c_uint64(), C.c_uint64()
        check(native_lib().kvr_driver_prefill_backlog(self.h, C.byref(q), C.byref(dr)))
        return q.value, dr.value

    def measured_json(self) -> str:
        """Measured report over the post-warm-up steps (device runs only)."""
        return self._text(native_lib().kvr_driver_measured_json)

    def trace(self) -> str:
        return self._text(native_lib().kvr_driver_trace)

    def pager(self) -> Pager:
        h = C.c_void_p()
        check(native_lib().kvr_driver_pager(self.h, C.byref(h)))
        p = Pager.__new__(Pager)
        p.api = api()
        p._owned = False
        p.h = h
        p._driver = self
        p.cfg = self.pager_config()
        return p

    def pager_config(self) -> PagerConfig:
        pc = self.config.get("pager", {})
        return PagerConfig(pc.get("page_bytes", 16384), pc.get("arena_pages", 4096),
                           pc.get("layers", 4), pc.get("kv_head_dim", 64), pc.get("elem_bytes", 2))

    def device(self) -> Device:
        h = C.c_void_p()
        check(native_lib().kvr_driver_device(self.h, C.byref(h)))
        return Device(_handle=h.value, _owner=self)

    def live(self):
        cap = 4096
        sl, se = (C.c_uint32 * cap)(), (C.c_uint32 * cap)()
        wr = (C.c_uint64 * cap)()
        n = C.c_uint64()
        check(native_lib().kvr_driver_live(self.h, sl, se, wr, cap, C.byref(n)))
        return [(sl[i], se[i], wr[i]) for i in range(n.value)]

    def workload_hash(self) -> int:
        o = C.c_uint64()
        check(native_lib().kvr_driver_workload_hash(self.h, C.byref(o)))
        return o.value

    def device_check(self) -> tuple[int, int, str]:
        """(steps checked, mismatching steps, first mismatch) of b200.check."""
        a, b = C.c_uint64(), C.c_uint64()
        buf = C.create_string_buffer(512)
        check(native_lib().kvr_driver_device_check(self.h, C.byref(a), C.byref(b), buf, 512))
        return a.value, b.value, buf.value.decode()

    def staged_rows(self) -> tuple[int, int, int]:
        """Staged tokens of the device trace: (delivered by K-gather into the window,
        behind the live window, missing from the window otherwise)."""
        a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(native_lib().kvr_driver_staged_rows(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def comm_init(self, unique_id: bytes, rank: int, world: int) -> None:
        """Join the in-graph per-step counts all-reduce over NCCL (before the first step)."""
        assert len(unique_id) == 128
        check(native_lib().kvr_driver_comm_init(self.h, unique_id, rank, world))

    def comm_destroy(self) -> None:
        """Drop the counts communicator again (only before the first step)."""
        check(native_lib().kvr_comm_destroy(self.device().raw()))

    FAULT_DROP_SPAN, FAULT_SHIFT_ROWS, FAULT_ALL = 1, 2, 0xFFFFFFFFFFFFFFFE

    def fault(self, what: int, arg: int) -> None:
        """Test hook (kvr_dev_fault): KVR_FAULT_DROP_SPAN (span index, FAULT_ALL, -1 off)
        or KVR_FAULT_SHIFT_ROWS (ring rows, 0 off) in K-gather on every later step."""
        check(native_lib().kvr_driver_fault(self.h, what, arg & 0xFFFFFFFFFFFFFFFF))
