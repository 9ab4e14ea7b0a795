"""Thin ctypes binding of libkvring (include/kvring.h): argument marshalling only.

Every function keeps the C name.  Arrays are numpy int64/int32 (host);
device buffers and streams are passed as integer addresses.  A non-zero
status raises ``KvError`` carrying the C code and ``kv_last_error()``.
There is no fallback: if libkvring.so is missing this module fails loudly.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkvring.so")

KV_OK, KV_EINVAL, KV_ENOMEM, KV_ECUDA, KV_ESTATE, KV_ENOREPLICA, KV_EPEER = 0, -1, -2, -3, -4, -5, -6
KV_SRC_HOST = 1
KV_MODE_TOKENS, KV_MODE_BLOCKS = 0, 1
CODE_NAMES = {0: "KV_OK", -1: "KV_EINVAL", -2: "KV_ENOMEM", -3: "KV_ECUDA", -4: "KV_ESTATE",
              -5: "KV_ENOREPLICA", -6: "KV_EPEER"}

EXPORTED = ["kv_abi_version", "kv_append", "kv_append_multi", "kv_begin_step", "kv_block_bytes",
            "kv_dump_slots", "kv_fail_stage", "kv_inject_abort", "kv_kernel_launch_count",
            "kv_last_error", "kv_meta_bytes", "kv_pack_bytes", "kv_pack_step", "kv_pool_create",
            "kv_pool_destroy", "kv_query", "kv_release", "kv_replicate_step",
            "kv_replicate_step_multi", "kv_restore", "kv_set_successor", "kv_stats", "kv_sync",
            "kv_unpack", "kv_time_next_launch", "kv_run_steps", "kv_host_profile",
            "kv_plan_targets", "kv_set_mode", "kv_replicate_step_ce",
            "kv_set_successor_shared", "kv_drop_replicas", "kv_pool_set_mirror",
            "kv_mirror_blocks", "kv_last_alloc", "kv_loop_create", "kv_loop_destroy",
            "kv_loop_step", "kv_loop_run", "kv_loop_flush", "kv_launch_log"]


class KvError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{CODE_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.name = CODE_NAMES.get(code, str(code))


class kv_geom_t(ctypes.Structure):
    _fields_ = [("layers", ctypes.c_int32), ("kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("block_size", ctypes.c_int32),
                ("elem_bytes", ctypes.c_int32)]


class kv_pool_desc_t(ctypes.Structure):
    _fields_ = [("g", kv_geom_t), ("num_blocks", ctypes.c_int32), ("max_reqs", ctypes.c_int32),
                ("max_blocks_per_req", ctypes.c_int32), ("device", ctypes.c_int32),
                ("node_id", ctypes.c_int32), ("replica_blocks", ctypes.c_int32),
                ("pool", ctypes.c_void_p), ("replica", ctypes.c_void_p),
                ("replica_meta", ctypes.c_void_p)]


class kv_append_args_t(ctypes.Structure):
    _fields_ = [("pool", ctypes.c_void_p), ("begin_step", ctypes.c_int32),
                ("n_release", ctypes.c_int32), ("release_ids", ctypes.c_void_p),
                ("n", ctypes.c_int32), ("req_ids", ctypes.c_void_p), ("n_new", ctypes.c_void_p),
                ("src_kv", ctypes.c_void_p), ("flags", ctypes.c_int32)]


class kv_step_t(ctypes.Structure):
    _fields_ = [("n_append", ctypes.c_int32), ("append", ctypes.c_void_p),
                ("n_repl", ctypes.c_int32), ("repl_pools", ctypes.c_void_p),
                ("step", ctypes.c_uint64), ("ev_call", ctypes.c_void_p),
                ("ev_kernel_start", ctypes.c_void_p), ("ev_kernel_end", ctypes.c_void_p),
                ("ev_done", ctypes.c_void_p), ("ev_append_start", ctypes.c_void_p),
                ("ev_append_end", ctypes.c_void_p)]


class kv_stats_t(ctypes.Structure):
    _fields_ = [("free_blocks", ctypes.c_int32), ("quarantined_blocks", ctypes.c_int32),
                ("used_blocks", ctypes.c_int32), ("free_slots", ctypes.c_int32),
                ("quarantined_slots", ctypes.c_int32), ("live_reqs", ctypes.c_int32),
                ("dead", ctypes.c_int32), ("has_successor", ctypes.c_int32),
                ("last_step", ctypes.c_uint64), ("bytes_replicated", ctypes.c_uint64),
                ("tasks_launched", ctypes.c_uint64), ("kernels_launched", ctypes.c_uint64),
                ("last_step_bytes", ctypes.c_uint64),
                ("replica_blocks_held", ctypes.c_int64), ("replica_evictions", ctypes.c_uint64),
                ("replica_drops", ctypes.c_uint64), ("shared_holder", ctypes.c_int32),
                ("pad0", ctypes.c_int32)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None
_P = ctypes.c_void_p
_I32, _I64, _U64, _SZ = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_size_t


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        sig = {
            "kv_abi_version": (_I32, []),
            "kv_last_error": (ctypes.c_char_p, []),
            "kv_kernel_launch_count": (_U64, []),
            "kv_block_bytes": (_SZ, [ctypes.POINTER(kv_geom_t)]),
            "kv_meta_bytes": (_SZ, [_I32, _I32]),
            "kv_pool_create": (ctypes.c_int, [ctypes.POINTER(kv_pool_desc_t), ctypes.POINTER(_P)]),
            "kv_pool_destroy": (ctypes.c_int, [_P]),
            "kv_set_successor": (ctypes.c_int, [_P, _I32, _P, _I32, _P]),
            "kv_begin_step": (ctypes.c_int, [_P]),
            "kv_release": (ctypes.c_int, [_P, _I32, _P]),
            "kv_append": (ctypes.c_int, [_P, _I32, _P, _P, _P, _I32, _P]),
            "kv_append_multi": (ctypes.c_int, [_I32, _P, _P]),
            "kv_replicate_step": (ctypes.c_int, [_P, _U64, _P]),
            "kv_replicate_step_multi": (ctypes.c_int, [_I32, _P, _U64, _P]),
            "kv_inject_abort": (ctypes.c_int, [_P, _I32]),
            "kv_fail_stage": (ctypes.c_int, [_P, _P]),
            "kv_restore": (ctypes.c_int, [_P, _P, _I32, _P, _P, ctypes.POINTER(_U64), _P, _P, _I32,
                                          ctypes.POINTER(_I32)]),
            "kv_pack_bytes": (ctypes.c_int, [_P, ctypes.POINTER(_SZ)]),
            "kv_pack_step": (ctypes.c_int, [_P, _U64, _P, _SZ, ctypes.POINTER(_SZ), _P]),
            "kv_unpack": (ctypes.c_int, [_P, _SZ, _P, _I32, _P, ctypes.POINTER(kv_geom_t), _I32,
                                         _I32, _P]),
            "kv_query": (ctypes.c_int, [_P, _I64, ctypes.POINTER(_I32), _P, _I32,
                                        ctypes.POINTER(_I32)]),
            "kv_stats": (ctypes.c_int, [_P, ctypes.POINTER(kv_stats_t)]),
            "kv_dump_slots": (ctypes.c_int, [_P, _P, _P, _P, _P]),
            "kv_sync": (ctypes.c_int, [_P]),
            "kv_time_next_launch": (ctypes.c_int, [_P, _P]),
            "kv_run_steps": (ctypes.c_int, [_I32, _P, _P, _P]),
            "kv_loop_create": (ctypes.c_int, [ctypes.POINTER(_P)]),
            "kv_loop_destroy": (ctypes.c_int, [_P]),
            "kv_loop_step": (ctypes.c_int, [_P, _P, _P]),
            "kv_loop_run": (ctypes.c_int, [_P, _I32, _P, _P]),
            "kv_loop_flush": (ctypes.c_int, [_P, _P]),
            "kv_launch_log": (ctypes.c_int, [_P, _I32, _I32]),
            "kv_replicate_step_ce": (ctypes.c_int, [_I32, _P, _U64, _P]),
            "kv_set_successor_shared": (ctypes.c_int, [_P, _P]),
            "kv_drop_replicas": (ctypes.c_int, [_P]),
            "kv_pool_set_mirror": (ctypes.c_int, [_P, _I32]),
            "kv_mirror_blocks": (ctypes.c_int, [_P, _I32, _P]),
            "kv_last_alloc": (ctypes.c_int, [_P, _P, _I32]),
            "kv_host_profile": (ctypes.c_int, [_P, _I32, _I32]),
            "kv_plan_targets": (ctypes.c_int, [_I32, _P, _P, _P]),
            "kv_set_mode": (ctypes.c_int, [_P, _I32]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != KV_OK:
        raise KvError(rc, lib().kv_last_error().decode(errors="replace"))


def _ptr(a) -> int | None:
    if a is None:
        return None
    if isinstance(a, int):
        return a
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()      # torch tensor


def _i64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int64).reshape(-1))


def _i32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32).reshape(-1))


def geom(layers, kv_heads=8, head_dim=128, block_size=16, elem_bytes=2) -> kv_geom_t:
    return kv_geom_t(layers, kv_heads, head_dim, block_size, elem_bytes)


def kv_abi_version() -> int:
    return lib().kv_abi_version()


def kv_kernel_launch_count() -> int:
    return lib().kv_kernel_launch_count()


def kv_block_bytes(g: kv_geom_t) -> int:
    return lib().kv_block_bytes(ctypes.byref(g))


def kv_meta_bytes(max_reqs: int, max_blocks_per_req: int) -> int:
    return lib().kv_meta_bytes(max_reqs, max_blocks_per_req)


def kv_pool_create(desc: kv_pool_desc_t) -> int:
    h = _P()
    _check(lib().kv_pool_create(ctypes.byref(desc), ctypes.byref(h)))
    return h.value


def kv_pool_destroy(p: int) -> None:
    _check(lib().kv_pool_destroy(p))


def kv_set_successor(p: int, succ_node: int, succ_replica, succ_replica_blocks: int, succ_meta) -> None:
    _check(lib().kv_set_successor(p, succ_node, _ptr(succ_replica), succ_replica_blocks,
                                  _ptr(succ_meta)))


def kv_begin_step(p: int) -> None:
    _check(lib().kv_begin_step(p))


def kv_release(p: int, req_ids) -> None:
    a = _i64(req_ids)
    _check(lib().kv_release(p, a.size, _ptr(a)))


def kv_append(p: int, req_ids, n_new, src_kv, flags: int = 0, stream: int = 0) -> None:
    a, n = _i64(req_ids), _i32(n_new)
    _check(lib().kv_append(p, a.size, _ptr(a), _ptr(n), _ptr(src_kv), flags, stream))


def kv_append_multi(entries, stream: int = 0) -> None:
    """entries: list of dicts {pool, begin_step, release, req_ids, n_new, src, flags}."""
    arr, keep = _append_array(entries)
    _check(lib().kv_append_multi(len(entries), ctypes.addressof(arr), stream))


def _append_array(entries):
    keep = []
    arr = (kv_append_args_t * max(1, len(entries)))()
    for k, e in enumerate(entries):
        rel = _i64(e.get("release", []))
        ids = _i64(e.get("req_ids", []))
        nn = _i32(e.get("n_new", []))
        keep.extend([rel, ids, nn, e.get("src")])
        arr[k] = kv_append_args_t(e["pool"], int(e.get("begin_step", 0)), rel.size, _ptr(rel),
                                  ids.size, _ptr(ids), _ptr(nn), _ptr(e.get("src")),
                                  int(e.get("flags", 0)))
    return arr, keep


class PreparedSteps:
    """Marshalled arguments of a run of decode steps for kv_run_steps (built ahead
    of time: per step the append entries, the pools to publish and optional
    timing events)."""

    def __init__(self, steps):
        self.keep = []
        self.arr = (kv_step_t * len(steps))()
        for k, st in enumerate(steps):
            app, keep = _append_array(st.get("append", []))
            pools = st.get("repl_pools", [])
            parr = (_P * max(1, len(pools)))(*pools)
            self.keep.extend([app, keep, parr])
            ev = [st.get(x) for x in ("ev_call", "ev_kernel_start", "ev_kernel_end", "ev_done",
                                      "ev_append_start", "ev_append_end")]
            self.keep.append(ev)
            self.arr[k] = kv_step_t(len(st.get("append", [])), ctypes.addressof(app), len(pools),
                                    ctypes.addressof(parr), int(st.get("step", 0)),
                                    *[_event_handle(e) for e in ev])
        self.n = len(steps)


def _event_handle(e):
    if e is None:
        return None
    if isinstance(e, int):
        return e
    if e.cuda_event == 0:   # torch creates events lazily
        e.record()
    return e.cuda_event


def kv_run_steps(prepared: "PreparedSteps", append_stream: int = 0, repl_stream: int = 0) -> None:
    _check(lib().kv_run_steps(prepared.n, ctypes.addressof(prepared.arr), append_stream,
                              repl_stream))


class KvLoop:
    """One-launch-per-step decode loop (kv_loop_*): each step's launch carries its
    appends and the previous step's publication."""

    def __init__(self):
        h = _P()
        _check(lib().kv_loop_create(ctypes.byref(h)))
        self.h = h.value

    def step(self, prepared: "PreparedSteps", k: int = 0, stream: int = 0) -> None:
        _check(lib().kv_loop_step(self.h, ctypes.addressof(prepared.arr) +
                                  k * ctypes.sizeof(kv_step_t), stream))

    def run(self, prepared: "PreparedSteps", stream: int = 0) -> None:
        _check(lib().kv_loop_run(self.h, prepared.n, ctypes.addressof(prepared.arr), stream))

    def flush(self, stream: int = 0) -> None:
        _check(lib().kv_loop_flush(self.h, stream))

    def destroy(self) -> None:
        if self.h:
            _check(lib().kv_loop_destroy(self.h))
            self.h = None


def kv_launch_log(start: bool, cap: int = 1 << 16):
    """start=True clears and starts the calling thread's launch log; start=False stops
    it and returns a list of dicts (kind, app_bytes, rep_bytes, grid, blob_bytes)."""
    if start:
        lib().kv_launch_log(None, 0, 1)
        return []
    out = np.zeros(5 * cap, dtype=np.uint64)
    n = lib().kv_launch_log(_ptr(out), cap, 0)
    keys = ("kind", "app_bytes", "rep_bytes", "grid", "blob_bytes")
    return [dict(zip(keys, (int(x) for x in out[5 * i:5 * i + 5]))) for i in range(min(n, cap))]


def kv_replicate_step(p: int, step: int, stream: int = 0) -> None:
    _check(lib().kv_replicate_step(p, step, stream))


def kv_replicate_step_multi(pools, step: int, stream: int = 0) -> None:
    arr = (_P * len(pools))(*pools)
    _check(lib().kv_replicate_step_multi(len(pools), ctypes.addressof(arr), step, stream))


def kv_set_mode(p: int, mode: int) -> None:
    _check(lib().kv_set_mode(p, mode))


def kv_set_successor_shared(p: int, holder: int) -> None:
    _check(lib().kv_set_successor_shared(p, holder))


def kv_drop_replicas(holder: int) -> None:
    _check(lib().kv_drop_replicas(holder))


def kv_pool_set_mirror(p: int, on: bool = True) -> None:
    _check(lib().kv_pool_set_mirror(p, 1 if on else 0))


def kv_mirror_blocks(mirror: int, block_ids) -> None:
    a = _i32(list(block_ids))
    _check(lib().kv_mirror_blocks(mirror, a.size, _ptr(a)))


def kv_last_alloc(p: int) -> list[int]:
    n = lib().kv_last_alloc(p, None, 0)
    _check(min(n, 0))
    out = np.zeros(max(1, n), dtype=np.int32)
    lib().kv_last_alloc(p, _ptr(out), n)
    return [int(x) for x in out[:n]]


def kv_replicate_step_ce(pools, step: int, stream: int = 0) -> None:
    arr = (_P * len(pools))(*pools)
    _check(lib().kv_replicate_step_ce(len(pools), ctypes.addressof(arr), step, stream))


def kv_inject_abort(p: int, slices: int) -> None:
    _check(lib().kv_inject_abort(p, slices))


def kv_fail_stage(p: int, stream: int = 0) -> None:
    _check(lib().kv_fail_stage(p, stream))


def kv_restore(dst: int, holder_replica, holder_replica_blocks: int, holder_meta, stream: int = 0,
               cap: int = 4096):
    """Returns (t_star, [(req_id, resume_len), ...])."""
    t = _U64()
    n = _I32()
    ids = np.zeros(cap, dtype=np.int64)
    lens = np.zeros(cap, dtype=np.int32)
    _check(lib().kv_restore(dst, _ptr(holder_replica), holder_replica_blocks, _ptr(holder_meta),
                            stream, ctypes.byref(t), _ptr(ids), _ptr(lens), cap, ctypes.byref(n)))
    return int(t.value), [(int(ids[i]), int(lens[i])) for i in range(n.value)]


def kv_pack_bytes(p: int) -> int:
    b = _SZ()
    _check(lib().kv_pack_bytes(p, ctypes.byref(b)))
    return int(b.value)


def kv_pack_step(p: int, step: int, packed, cap: int, stream: int = 0) -> int:
    b = _SZ()
    _check(lib().kv_pack_step(p, step, _ptr(packed), cap, ctypes.byref(b), stream))
    return int(b.value)


def kv_unpack(packed, packed_bytes: int, replica, replica_blocks: int, replica_meta,
              g: kv_geom_t, max_reqs: int, max_blocks_per_req: int, stream: int = 0) -> None:
    _check(lib().kv_unpack(_ptr(packed), packed_bytes, _ptr(replica), replica_blocks,
                           _ptr(replica_meta), ctypes.byref(g), max_reqs, max_blocks_per_req,
                           stream))


def kv_query(p: int, req_id: int, cap: int = 4096):
    ln, nb = _I32(), _I32()
    blocks = np.zeros(cap, dtype=np.int32)
    _check(lib().kv_query(p, req_id, ctypes.byref(ln), _ptr(blocks), cap, ctypes.byref(nb)))
    return int(ln.value), [int(x) for x in blocks[:min(nb.value, cap)]]


def kv_stats(p: int) -> dict:
    s = kv_stats_t()
    _check(lib().kv_stats(p, ctypes.byref(s)))
    return s.as_dict()


def kv_dump_slots(p: int, max_reqs: int):
    req = np.zeros(max_reqs, dtype=np.int64)
    ln = np.zeros(max_reqs, dtype=np.int32)
    pub = np.zeros(max_reqs, dtype=np.int32)
    nb = np.zeros(max_reqs, dtype=np.int32)
    _check(lib().kv_dump_slots(p, _ptr(req), _ptr(ln), _ptr(pub), _ptr(nb)))
    return req, ln, pub, nb


def kv_time_next_launch(ev_before, ev_after) -> None:
    """ev_*: torch.cuda.Event (recorded by libkvring around its next kernel) or None."""
    _check(lib().kv_time_next_launch(_event_handle(ev_before), _event_handle(ev_after)))


def kv_plan_targets(succ, excluded=None):
    """succ: successor node id per node (list); excluded: iterable of node ids.
    Returns the re-protection targets (-1 = none / excluded)."""
    n = len(succ)
    sa = _i32(succ)
    ex = np.zeros(n, dtype=np.uint8)
    for e in (excluded or []):
        ex[e] = 1
    out = np.zeros(n, dtype=np.int32)
    _check(lib().kv_plan_targets(n, _ptr(sa), _ptr(ex), _ptr(out)))
    return [int(x) for x in out]


HOST_PHASES = ["prepare.append", "prepare.replicate", "stage", "launch", "stage.pack",
               "stage.acquire", "stage.h2d_call", "stage.events"]


def kv_host_profile(reset: bool = True) -> dict:
    out = np.zeros(len(HOST_PHASES), dtype=np.float64)
    n = lib().kv_host_profile(_ptr(out), len(HOST_PHASES), 1 if reset else 0)
    return {HOST_PHASES[i] if i < len(HOST_PHASES) else str(i): float(out[i]) for i in range(n)}


def kv_sync(p: int) -> None:
    _check(lib().kv_sync(p))
