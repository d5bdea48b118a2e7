"""Thin Python binding of libepg.so (include/epg.h): argument marshalling only.

Every step of the path runs in the library (host C++ partitioner, CUDA kernels); torch
tensors only supply device memory and the CUDA stream. There is no fallback: if
libepg.so is missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# EPG_LIB_PATH overrides the library file (development builds, e.g. the -DEPG_TRACE one)
LIB_PATH = os.environ.get("EPG_LIB_PATH", os.path.join(_HERE, "libepg.so"))

OK, ERR_INPUT, ERR_INFEASIBLE, ERR_CUDA, ERR_NCCL, ERR_NOMEM, ERR_STATE = 0, 2, 3, 4, 5, 6, 7
KERNEL_CFD_FLUX, KERNEL_GATHER_SCATTER, KERNEL_SPMV = 1, 2, 3
PARTITION_EPG1, PARTITION_EPG2, PARTITION_RB = 1, 2, 3
KERNELS = {"cfd": KERNEL_CFD_FLUX, "gather_scatter": KERNEL_GATHER_SCATTER, "spmv": KERNEL_SPMV}
ROW = {KERNEL_CFD_FLUX: 5, KERNEL_GATHER_SCATTER: 1, KERNEL_SPMV: 1}
MAX_PART_SIZE = 4096
PERM_GATHER, PERM_SCATTER = 0, 1

# every symbol include/epg.h declares (checked by tests/test_abi.py)
SYMBOLS = ["epg_create", "epg_destroy", "epg_last_error", "epg_num_parts", "epg_partition_host", "epg_partition",
           "epg_default_partition", "epg_load_count", "epg_remap", "epg_plan_destroy", "epg_plan_info",
           "epg_permute_rows", "epg_run", "epg_run_naive", "epg_set_variant", "epg_set_profiling",
           "epg_profile_read", "epg_shard_ranges", "epg_shard_halos_host", "epg_run_edges", "epg_run_finalise",
           "epg_shard_reduce", "epg_accumulate_rows", "epg_remapped_edges", "epg_set_hub_split", "epg_plan_hubs",
           "epg_set_exec_limits", "epg_partition_random_host", "epg_partition_greedy_host",
           "epg_adaptive_create", "epg_adaptive_step", "epg_adaptive_wait", "epg_adaptive_read_state",
           "epg_adaptive_info", "epg_adaptive_destroy", "epg_partition_host_method", "epg_set_partition_method",
           "epg_run_host", "epg_run_host_join", "epg_partition_rb", "epg_comm_unique_id", "epg_comm_init",
           "epg_comm_init_local", "epg_run_sharded", "epg_run_sharded_group", "epg_set_hub_l2", "epg_remap_keyed",
           "epg_partition_ranked", "epg_partition_host_ranked"]


class _Report(C.Structure):
    _fields_ = [(f, C.c_int64) for f in ("k", "load_count", "touched", "cut_cost", "max_size", "min_size")]


class _Layout(C.Structure):
    _fields_ = [("edge_perm", C.c_void_p), ("part_edge_begin", C.c_void_p), ("vertex_perm", C.c_void_p),
                ("part_vertex_begin", C.c_void_p), ("halo_begin", C.c_void_p), ("halo_ids", C.c_void_p),
                ("halo_cap", C.c_int64), ("slots", C.c_void_p)]


class _AdaptiveReport(C.Structure):
    _fields_ = [("phase", C.c_int32), ("partition_done", C.c_int32), ("steps_original", C.c_int64),
                ("steps_ep", C.c_int64), ("partition_seconds", C.c_double), ("original_ms", C.c_double),
                ("ep_first_ms", C.c_double)]


class _State(C.Structure):
    _fields_ = [("state_in", C.c_void_p), ("state_out", C.c_void_p), ("edge_payload", C.c_void_p),
                ("vertex_const", C.c_void_p)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libepg.so not built at {LIB_PATH}; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(LIB_PATH)
    P, i32, i64, st = C.c_void_p, C.c_int32, C.c_int64, C.c_int
    sig = {
        "epg_create": (st, [C.c_int, P, C.POINTER(P)]),
        "epg_destroy": (None, [P]),
        "epg_last_error": (C.c_char_p, [P]),
        "epg_num_parts": (i64, [i64, i32]),
        "epg_partition_host": (st, [P, i64, i32, i32, i32, P, C.c_char_p, i64]),
        "epg_partition_host_method": (st, [P, i64, i32, i32, i32, i32, P, C.c_char_p, i64]),
        "epg_set_partition_method": (st, [P, i32]),
        "epg_partition": (st, [P, P, i64, i32, i32, i32, P, C.POINTER(_Report)]),
        "epg_partition_rb": (st, [P, P, i64, i32, i32, i32, i32, P, P, C.POINTER(_Report)]),
        "epg_partition_ranked": (st, [P, P, i64, i32, i32, i32, P, P, C.POINTER(_Report)]),
        "epg_partition_host_ranked": (st, [P, i64, i32, i32, i32, i32, P, P, C.c_char_p, i64]),
        "epg_remap_keyed": (st, [P, P, i64, i32, P, P, i64, C.POINTER(_Layout), C.POINTER(P)]),
        "epg_default_partition": (st, [P, i64, i32, P]),
        "epg_load_count": (st, [P, P, i64, i32, P, i64, P, C.POINTER(_Report)]),
        "epg_remap": (st, [P, P, i64, i32, P, i64, C.POINTER(_Layout), C.POINTER(P)]),
        "epg_plan_destroy": (None, [P]),
        "epg_plan_info": (st, [P, P]),
        "epg_permute_rows": (st, [P, P, P, i64, i32, P, i32]),
        "epg_run": (st, [P, P, C.c_int, C.POINTER(_State), i32]),
        "epg_run_host": (st, [P, P, C.c_int, P, P, P, P, P, i32]),
        "epg_run_host_join": (st, [P]),
        "epg_run_naive": (st, [P, C.c_int, P, i64, i32, C.POINTER(_State), i32]),
        "epg_set_variant": (st, [P, i32]),
        "epg_set_hub_split": (st, [P, i32]),
        "epg_set_hub_l2": (st, [P, i32]),
        "epg_set_exec_limits": (st, [P, i32, i32]),
        "epg_partition_random_host": (st, [i64, i32, C.c_uint64, P, C.c_char_p, i64]),
        "epg_partition_greedy_host": (st, [P, i64, i32, i32, P, C.c_char_p, i64]),
        "epg_adaptive_create": (st, [P, C.c_int, P, i64, i32, i32, P, P, P, C.c_double, C.POINTER(P)]),
        "epg_adaptive_step": (st, [P, i32]),
        "epg_adaptive_wait": (st, [P]),
        "epg_adaptive_read_state": (st, [P, P]),
        "epg_adaptive_info": (st, [P, C.POINTER(_AdaptiveReport)]),
        "epg_adaptive_destroy": (None, [P]),
        "epg_plan_hubs": (i64, [P, P]),
        "epg_shard_ranges": (st, [P, i32, i32, P]),
        "epg_shard_halos_host": (st, [P, P, P, i64, i32, P, P, i64, P]),
        "epg_run_edges": (st, [P, P, C.c_int, C.POINTER(_State), i64, i64]),
        "epg_run_finalise": (st, [P, P, C.c_int, C.POINTER(_State), i64, i64, i64, i64, P, i32]),
        "epg_shard_reduce": (st, [P, P, C.c_int, P, i64, i64, i64, P]),
        "epg_accumulate_rows": (st, [P, P, P, i64, i32, P]),
        "epg_remapped_edges": (st, [P, P, i64, P, P, P]),
        "epg_comm_unique_id": (st, [P]),
        "epg_comm_init": (st, [P, P, i32, i32]),
        "epg_comm_init_local": (st, [P, i32]),
        "epg_run_sharded": (st, [P, P, C.c_int, C.POINTER(_State), i32]),
        "epg_run_sharded_group": (st, [P, P, C.c_int, P, i32]),
        "epg_set_profiling": (st, [P, i32]),
        "epg_profile_read": (st, [P, P, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


class EpgError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"epg status {status}: {message}")
        self.status = status
        self.message = message


@dataclass
class Report:
    k: int
    load_count: int
    touched: int
    cut_cost: int
    max_size: int
    min_size: int

    @property
    def replication(self) -> float:
        return self.load_count / self.touched

    @property
    def redundant_fraction(self) -> float:
        return self.cut_cost / self.load_count


def _rep(r: _Report) -> Report:
    return Report(r.k, r.load_count, r.touched, r.cut_cost, r.max_size, r.min_size)


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        assert t.flags.c_contiguous
        return t.ctypes.data
    assert t.is_contiguous(), "tensors passed to libepg must be contiguous"
    return t.data_ptr()


def num_parts(m: int, part_size: int) -> int:
    return int(lib.epg_num_parts(m, part_size))


def shard_halos_host(part_vertex_begin, halo_begin, halo_ids, k: int, G: int):
    """O7 halo sets from the EP layout (host arrays) -> (begin [G*G+1], ids)."""
    pvb = np.ascontiguousarray(part_vertex_begin, np.int32)
    hb = np.ascontiguousarray(halo_begin, np.int32)
    hid = np.ascontiguousarray(halo_ids, np.int32)
    begin = np.zeros(G * G + 1, np.int32)
    cnt = np.zeros(1, np.int64)
    s = lib.epg_shard_halos_host(pvb.ctypes.data, hb.ctypes.data, hid.ctypes.data if hid.size else None, k, G,
                                 begin.ctypes.data, None, 0, cnt.ctypes.data)
    if s != OK:
        raise EpgError(s, "epg_shard_halos_host")
    ids = np.zeros(max(int(cnt[0]), 1), np.int32)
    s = lib.epg_shard_halos_host(pvb.ctypes.data, hb.ctypes.data, hid.ctypes.data if hid.size else None, k, G,
                                 begin.ctypes.data, ids.ctypes.data, ids.size, cnt.ctypes.data)
    if s != OK:
        raise EpgError(s, "epg_shard_halos_host")
    return begin, ids[: int(cnt[0])]


def partition_host(edges, n: int, part_size: int, shards: int = 1, method: int = PARTITION_EPG1) -> np.ndarray:
    """Host EPG-1 / EPG-2 (epg_partition_host_method); edges int32 [m][2] numpy or CPU tensor."""
    e = np.ascontiguousarray(edges.cpu().numpy() if isinstance(edges, torch.Tensor) else edges, dtype=np.int32)
    m = e.shape[0]
    part = np.zeros(max(m, 1), np.int32)
    buf = C.create_string_buffer(512)
    s = lib.epg_partition_host_method(e.ctypes.data if m else None, m, n, part_size, shards, method,
                                      part.ctypes.data, buf, 512)
    if s != OK:
        raise EpgError(s, buf.value.decode())
    return part[:m]


def partition_host_ranked(edges, n: int, part_size: int, shards: int = 1, method: int = PARTITION_EPG1):
    """epg_partition_host_ranked -> (part, rank) (HOST numpy)."""
    e = np.ascontiguousarray(edges.cpu().numpy() if isinstance(edges, torch.Tensor) else edges, dtype=np.int32)
    m = e.shape[0]
    part = np.zeros(max(m, 1), np.int32)
    rank = np.zeros(max(m, 1), np.int32)
    buf = C.create_string_buffer(512)
    s = lib.epg_partition_host_ranked(e.ctypes.data if m else None, m, n, part_size, shards, method,
                                      part.ctypes.data, rank.ctypes.data, buf, 512)
    if s != OK:
        raise EpgError(s, buf.value.decode())
    return part[:m], rank[:m]


def partition_random_host(m: int, part_size: int, seed: int = 1605) -> np.ndarray:
    """PowerGraph random baseline (epg_partition_random_host)."""
    part = np.zeros(max(m, 1), np.int32)
    buf = C.create_string_buffer(512)
    s = lib.epg_partition_random_host(m, part_size, seed & 0xFFFFFFFFFFFFFFFF, part.ctypes.data, buf, 512)
    if s != OK:
        raise EpgError(s, buf.value.decode())
    return part[:m]


def partition_greedy_host(edges, n: int, part_size: int) -> np.ndarray:
    """PowerGraph greedy baseline (epg_partition_greedy_host)."""
    e = np.ascontiguousarray(edges.cpu().numpy() if isinstance(edges, torch.Tensor) else edges, dtype=np.int32)
    m = e.shape[0]
    part = np.zeros(max(m, 1), np.int32)
    buf = C.create_string_buffer(512)
    s = lib.epg_partition_greedy_host(e.ctypes.data if m else None, m, n, part_size, part.ctypes.data, buf, 512)
    if s != OK:
        raise EpgError(s, buf.value.decode())
    return part[:m]


def comm_unique_id() -> bytes:
    """epg_comm_unique_id: a fresh NCCL unique id (128 bytes) to broadcast to every rank."""
    buf = C.create_string_buffer(128)
    s = lib.epg_comm_unique_id(buf)
    if s != OK:
        raise EpgError(s, "epg_comm_unique_id (NCCL unavailable?)")
    return buf.raw


def comm_init_local(ctxs: list):
    """epg_comm_init_local: the contexts become an in-process group (ranks 0..G-1)."""
    arr = (C.c_void_p * len(ctxs))(*[c.handle.value for c in ctxs])
    s = lib.epg_comm_init_local(arr, len(ctxs))
    if s != OK:
        raise EpgError(s, "epg_comm_init_local")


def run_sharded_group(ctxs: list, plans: list, kernel: int, states: list):
    """epg_run_sharded_group: one sharded step of every member; states[g] = (in, out, payload, vconst)."""
    G = len(ctxs)
    carr = (C.c_void_p * G)(*[c.handle.value for c in ctxs])
    parr = (C.c_void_p * G)(*[p.handle.value for p in plans])
    sarr = (_State * G)(*[_State(_ptr(a), _ptr(b), _ptr(pw), _ptr(vc)) for a, b, pw, vc in states])
    s = lib.epg_run_sharded_group(carr, parr, kernel, sarr, G)
    if s != OK:
        msgs = "; ".join(lib.epg_last_error(c.handle).decode() for c in ctxs)
        raise EpgError(s, f"epg_run_sharded_group: {msgs}")


ADAPTIVE_ORIGINAL, ADAPTIVE_EP, ADAPTIVE_FELL_BACK, ADAPTIVE_NO_PARTITION = 0, 1, 2, 3


class Adaptive:
    """epg_adaptive: the paper's adaptive overhead control -- original kernel
    while host EPG-1 runs on a thread, EP plan applied when ready, kept iff its first
    step is not slower (include/epg.h)."""

    def __init__(self, ctx: "Context", kernel: int, edges, n: int, part_size: int, state: torch.Tensor,
                 payload: torch.Tensor | None = None, vconst: torch.Tensor | None = None,
                 fallback_ratio: float = 1.0):
        self.ctx = ctx
        self._edges = np.ascontiguousarray(edges.cpu().numpy() if isinstance(edges, torch.Tensor) else edges,
                                           dtype=np.int32)
        self.n = n
        self.shape, self.dtype, self.device = state.shape, state.dtype, state.device
        h = C.c_void_p()
        ctx._check(lib.epg_adaptive_create(ctx.handle, kernel, self._edges.ctypes.data, self._edges.shape[0], n,
                                           part_size, _ptr(payload), _ptr(vconst), _ptr(state), fallback_ratio,
                                           C.byref(h)))
        self.handle = h

    def step(self, steps: int = 1):
        self.ctx._check(lib.epg_adaptive_step(self.handle, steps))

    def wait(self):
        self.ctx._check(lib.epg_adaptive_wait(self.handle))

    def read_state(self, out: torch.Tensor | None = None) -> torch.Tensor:
        if out is None:
            out = torch.empty(self.shape, dtype=self.dtype, device=self.device)
        self.ctx._check(lib.epg_adaptive_read_state(self.handle, _ptr(out)))
        return out

    def info(self) -> dict:
        r = _AdaptiveReport()
        lib.epg_adaptive_info(self.handle, C.byref(r))
        return {f: getattr(r, f) for f, _ in _AdaptiveReport._fields_}

    def close(self):
        if self.handle:
            lib.epg_adaptive_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class Layout:
    edge_perm: torch.Tensor
    part_edge_begin: torch.Tensor
    vertex_perm: torch.Tensor
    part_vertex_begin: torch.Tensor
    halo_begin: torch.Tensor
    halo_ids: torch.Tensor
    slots: torch.Tensor


class Plan:
    def __init__(self, handle, ctx):
        self.handle = handle
        self.ctx = ctx
        info = np.zeros(8, np.int64)
        lib.epg_plan_info(handle, info.ctypes.data)
        (self.m, self.n, self.k, self.touched, self.cut_cost, self.shared,
         self.k_exec, self.cut_cost_exec) = (int(x) for x in info)
        hm = C.c_int32(0)
        self.hubs = int(lib.epg_plan_hubs(handle, C.byref(hm)))
        self.hub_min = int(hm.value)

    def close(self):
        if self.handle:
            lib.epg_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context:
    """An epg_ctx bound to a CUDA device and stream (default: torch's current stream)."""

    def __init__(self, device: int = 0, stream: torch.cuda.Stream | None = None):
        self.device = torch.device("cuda", device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        h = C.c_void_p()
        s = lib.epg_create(device, C.c_void_p(self.stream.cuda_stream), C.byref(h))
        if s != OK:
            raise EpgError(s, f"epg_create(device={device}) failed")
        self.handle = h

    def close(self):
        if self.handle:
            lib.epg_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, s: int):
        if s != OK:
            raise EpgError(s, lib.epg_last_error(self.handle).decode())

    # -- partition -----------------------------------------------------------------
    def partition(self, edges: torch.Tensor, n: int, part_size: int, shards: int = 1, out: torch.Tensor | None = None):
        m = edges.shape[0]
        if out is None:
            out = torch.empty(m, dtype=torch.int32, device=edges.device)
        r = _Report()
        self._check(lib.epg_partition(self.handle, _ptr(edges), m, n, part_size, shards, _ptr(out), C.byref(r)))
        return out, _rep(r)

    def partition_rb(self, edges: torch.Tensor, n: int, part_size: int, shards: int = 1, leaf_parts: int = 512,
                     out: torch.Tensor | None = None, ranked: bool = False):
        """EPG-RB (epg_partition_rb): GPU bisection levels + EPG-2 leaves on the host cores.
        -> (part, report), or (part, rank, report) with ranked=True (growth steps, reading Z22)."""
        m = edges.shape[0]
        if out is None:
            out = torch.empty(m, dtype=torch.int32, device=edges.device)
        rank = torch.empty(m, dtype=torch.int32, device=edges.device) if ranked else None
        r = _Report()
        self._check(lib.epg_partition_rb(self.handle, _ptr(edges), m, n, part_size, shards, leaf_parts, _ptr(out),
                                         _ptr(rank), C.byref(r)))
        return (out, rank, _rep(r)) if ranked else (out, _rep(r))

    def partition_ranked(self, edges: torch.Tensor, n: int, part_size: int, shards: int = 1):
        """epg_partition_ranked (ctx's method) -> (part, rank, report)."""
        m = edges.shape[0]
        out = torch.empty(m, dtype=torch.int32, device=edges.device)
        rank = torch.empty(m, dtype=torch.int32, device=edges.device)
        r = _Report()
        self._check(lib.epg_partition_ranked(self.handle, _ptr(edges), m, n, part_size, shards, _ptr(out), _ptr(rank),
                                             C.byref(r)))
        return out, rank, _rep(r)

    def default_partition(self, m: int, part_size: int) -> torch.Tensor:
        out = torch.empty(m, dtype=torch.int32, device=self.device)
        self._check(lib.epg_default_partition(self.handle, m, part_size, _ptr(out)))
        return out

    def load_count(self, edges: torch.Tensor, n: int, part: torch.Tensor, k: int, per_part: bool = False):
        pp = torch.empty(k, dtype=torch.int32, device=self.device) if per_part else None
        r = _Report()
        self._check(lib.epg_load_count(self.handle, _ptr(edges), edges.shape[0], n, _ptr(part), k, _ptr(pp), C.byref(r)))
        return (_rep(r), pp) if per_part else _rep(r)

    # -- remap ---------------------------------------------------------------------
    def remap(self, edges: torch.Tensor, n: int, part: torch.Tensor, k: int, halo_cap: int | None = None,
              order_key: torch.Tensor | None = None):
        m = edges.shape[0]
        if halo_cap is None:
            halo_cap = self.load_count(edges, n, part, k).cut_cost
        d = self.device
        i32 = torch.int32
        L = Layout(torch.empty(m, dtype=i32, device=d), torch.empty(k + 1, dtype=i32, device=d),
                   torch.empty(n, dtype=i32, device=d), torch.empty(k + 1, dtype=i32, device=d),
                   torch.empty(k + 1, dtype=i32, device=d), torch.empty(max(halo_cap, 1), dtype=i32, device=d),
                   torch.empty((m, 2), dtype=torch.uint16, device=d))
        cl = _Layout(_ptr(L.edge_perm), _ptr(L.part_edge_begin), _ptr(L.vertex_perm), _ptr(L.part_vertex_begin),
                     _ptr(L.halo_begin), _ptr(L.halo_ids), halo_cap, _ptr(L.slots))
        h = C.c_void_p()
        self._check(lib.epg_remap_keyed(self.handle, _ptr(edges), m, n, _ptr(part), _ptr(order_key), k, C.byref(cl),
                                        C.byref(h)))
        plan = Plan(h, self)
        L.halo_ids = L.halo_ids[: plan.cut_cost]
        return L, plan

    def remapped_edges(self, edges: torch.Tensor, layout: Layout) -> torch.Tensor:
        out = torch.empty_like(edges)
        self._check(lib.epg_remapped_edges(self.handle, _ptr(edges), edges.shape[0], _ptr(layout.edge_perm),
                                           _ptr(layout.vertex_perm), _ptr(out)))
        return out

    def permute_rows(self, src: torch.Tensor, perm: torch.Tensor, mode: int, out: torch.Tensor | None = None):
        rows = perm.shape[0]
        if out is None:
            out = torch.empty_like(src)
        row_bytes = src[0].numel() * src.element_size() if src.dim() > 1 else src.element_size()
        self._check(lib.epg_permute_rows(self.handle, _ptr(src), _ptr(out), rows, row_bytes, _ptr(perm), mode))
        return out

    # -- run -------------------------------------------------------------------------
    def run(self, plan: Plan, kernel: int, state_in: torch.Tensor, state_out: torch.Tensor,
            payload: torch.Tensor | None = None, vconst: torch.Tensor | None = None, steps: int = 1):
        st = _State(_ptr(state_in), _ptr(state_out), _ptr(payload), _ptr(vconst))
        self._check(lib.epg_run(self.handle, plan.handle, kernel, C.byref(st), steps))
        return state_out if steps % 2 else state_in

    def run_host(self, plan: Plan, kernel: int, vertex_perm: torch.Tensor, state_in_host: torch.Tensor,
                 state_out_host: torch.Tensor, payload: torch.Tensor | None = None,
                 vconst: torch.Tensor | None = None, steps: int = 1):
        """epg_run_host: host (ideally pinned) state in original vertex order -> device ->
        `steps` steps -> host; asynchronous, complete after join() has run on the stream."""
        for t in (state_in_host, state_out_host):
            if t.is_cuda or not t.is_contiguous() or t.dtype != torch.float32:
                raise ValueError("run_host: host state must be contiguous float32 CPU tensors")
        self._check(lib.epg_run_host(self.handle, plan.handle, kernel, _ptr(vertex_perm), state_in_host.data_ptr(),
                                     state_out_host.data_ptr(), _ptr(payload), _ptr(vconst), steps))
        return state_out_host

    def join(self):
        """epg_run_host_join: the ctx stream waits for every pending epg_run_host copy-out."""
        self._check(lib.epg_run_host_join(self.handle))

    # -- multi-GPU shards ---------------------------------------------------------------
    def shard_ranges(self, plan: Plan, G: int, g: int) -> dict:
        out = np.zeros(8, np.int64)
        self._check(lib.epg_shard_ranges(plan.handle, G, g, out.ctypes.data))
        keys = ("exec_first", "exec_count", "halo_first", "halo_count", "vertex_first", "vertex_count",
                "shared_first", "shared_count")
        return {k: int(v) for k, v in zip(keys, out)}

    def run_edges(self, plan: Plan, kernel: int, state_in, state_out, payload=None, vconst=None, first=0, count=None):
        count = plan.k_exec - first if count is None else count
        st = _State(_ptr(state_in), _ptr(state_out), _ptr(payload), _ptr(vconst))
        self._check(lib.epg_run_edges(self.handle, plan.handle, kernel, C.byref(st), first, count))

    def run_finalise(self, plan: Plan, kernel: int, state_in, state_out, payload=None, vconst=None,
                     shared_first=0, shared_count=None, halo_first=0, halo_count=None, acc=None, untouched=True):
        shared_count = plan.shared - shared_first if shared_count is None else shared_count
        halo_count = plan.cut_cost_exec - halo_first if halo_count is None else halo_count
        st = _State(_ptr(state_in), _ptr(state_out), _ptr(payload), _ptr(vconst))
        self._check(lib.epg_run_finalise(self.handle, plan.handle, kernel, C.byref(st), shared_first, shared_count,
                                         halo_first, halo_count, _ptr(acc), 1 if untouched else 0))

    def shard_reduce(self, plan: Plan, kernel: int, ids: torch.Tensor, halo_first: int, halo_count: int,
                     out: torch.Tensor):
        self._check(lib.epg_shard_reduce(self.handle, plan.handle, kernel, _ptr(ids), ids.numel(), halo_first,
                                         halo_count, _ptr(out)))
        return out

    def accumulate_rows(self, src: torch.Tensor, ids: torch.Tensor, acc: torch.Tensor):
        w = src[0].numel() if src.dim() > 1 else 1
        self._check(lib.epg_accumulate_rows(self.handle, _ptr(src), _ptr(ids), ids.numel(), w, _ptr(acc)))

    # -- multi-GPU inside the library (epg_comm_* / epg_run_sharded) ----------------------
    def comm_init(self, unique_id: bytes, nranks: int, rank: int):
        """epg_comm_init: NCCL communicator of this context (id from comm_unique_id())."""
        buf = C.create_string_buffer(bytes(unique_id), 128)
        self._check(lib.epg_comm_init(self.handle, buf, nranks, rank))

    def run_sharded(self, plan: Plan, kernel: int, state_in, state_out, payload=None, vconst=None, steps: int = 1):
        """epg_run_sharded: `steps` sharded time steps of this rank (owned rows authoritative)."""
        st = _State(_ptr(state_in), _ptr(state_out), _ptr(payload), _ptr(vconst))
        self._check(lib.epg_run_sharded(self.handle, plan.handle, kernel, C.byref(st), steps))
        return state_out if steps % 2 else state_in

    def set_variant(self, variant: int):
        """0 auto, 1 one CTA per partition, 2 pipelined TMA kernel, 3 occupancy TMA kernel."""
        self._check(lib.epg_set_variant(self.handle, variant))

    def set_partition_method(self, method: int):
        """Partitioner of epg_partition / the adaptive executor (PARTITION_EPG1 or _EPG2)."""
        self._check(lib.epg_set_partition_method(self.handle, method))

    def set_exec_limits(self, max_rows: int = -1, max_edges: int = -1):
        """Execution-split caps for plans remapped after this call (-1 = default)."""
        self._check(lib.epg_set_exec_limits(self.handle, max_rows, max_edges))

    def set_hub_split(self, min_halo_entries: int):
        """Hub split for plans remapped after this call (0 off; default 7, see include/epg.h)."""
        self._check(lib.epg_set_hub_split(self.handle, min_halo_entries))

    def set_hub_l2(self, enable: bool):
        """Persisting L2 window over the hubs' rows for the edge kernel (default on)."""
        self._check(lib.epg_set_hub_l2(self.handle, 1 if enable else 0))

    def set_profiling(self, enable: bool):
        self._check(lib.epg_set_profiling(self.handle, 1 if enable else 0))

    def profile_read(self):
        """-> ((edge_ms, finalise_ms), (edge_launches, finalise_launches)) since the last read."""
        ms = np.zeros(2, np.float32)
        n = np.zeros(2, np.int64)
        self._check(lib.epg_profile_read(self.handle, ms.ctypes.data, n.ctypes.data))
        return (float(ms[0]), float(ms[1])), (int(n[0]), int(n[1]))

    def run_naive(self, kernel: int, edges: torch.Tensor, n: int, state_in: torch.Tensor, state_out: torch.Tensor,
                  payload: torch.Tensor | None = None, vconst: torch.Tensor | None = None, steps: int = 1):
        st = _State(_ptr(state_in), _ptr(state_out), _ptr(payload), _ptr(vconst))
        self._check(lib.epg_run_naive(self.handle, kernel, _ptr(edges), edges.shape[0], n, C.byref(st), steps))
        return state_out if steps % 2 else state_in
