"""CPU oracle for the EP hot path of arXiv 1605.02043 -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package. It shares no code with the CUDA path
(paper_1605_02043_b200/) and neither imports the other. The arithmetic lives in
epg_oracle.c (plain C, fp64, one function per definition of the paper, cited there);
this module only marshals numpy arrays through ctypes.

Parity pins: tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "epg_oracle.c")
_LIB = os.path.join(_HERE, "libepg_oracle.so")

OK, ERR_INPUT, ERR_INFEASIBLE = 0, 2, 3


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        i64, i32, P = C.c_int64, C.c_int32, C.c_void_p
        sig = {
            "orc_num_parts": (i64, [i64, i32]),
            "orc_part_sizes": (None, [i64, i64, P]),
            "orc_first_bad_edge": (i64, [P, i64, i32]),
            "orc_cost": (C.c_int, [P, i64, i32, P, i64, P, P]),
            "orc_default_partition": (C.c_int, [i64, i32, P]),
            "orc_build_T": (C.c_int, [P, i64, i32, P, P, P, i64, P]),
            "orc_epg1": (C.c_int, [i64, P, P, P, P, i64, P]),
            "orc_partition": (C.c_int, [P, i64, i32, i32, i32, P]),
            "orc_partition_method": (C.c_int, [P, i64, i32, i32, i32, i32, P]),
            "orc_epg2": (C.c_int, [i64, P, i32, P, i64, i64, P]),
            "orc_partition_rb": (C.c_int, [P, i64, i32, i32, i32, i32, P]),
            "orc_partition_rb_ranked": (C.c_int, [P, i64, i32, i32, i32, i32, P, P]),
            "orc_partition_method_ranked": (C.c_int, [P, i64, i32, i32, i32, i32, P, P]),
            "orc_remap_keyed": (C.c_int, [P, i64, i32, P, P, i64, P, P, P, P, P, P, i64, P]),
            "orc_rb_depth": (C.c_int, [i64, i32, i32]),
            "orc_remap": (C.c_int, [P, i64, i32, P, i64, P, P, P, P, P, P, i64, P]),
            "orc_shard_halos": (C.c_int, [P, i64, i32, P, i64, i32, P, P, P, P, i64]),
            "orc_cfd_flux": (None, [P, i64, i32, P, P, P]),
            "orc_cfd_flux_abs": (None, [P, i64, i32, P, P, P]),
            "orc_cfd_step": (None, [P, i64, i32, P, P, P, P, P]),
            "orc_cfd_step_omp": (C.c_int, [P, i64, i32, P, P, P, P, P, P, P]),
            "orc_incidence": (None, [P, i64, i32, P, P]),
            "orc_gather_scatter": (None, [P, i64, i32, P, P, P]),
            "orc_spmv": (None, [P, i64, i32, P, P, P]),
            "orc_partition_random": (C.c_int, [i64, i32, C.c_uint64, P]),
            "orc_partition_greedy": (C.c_int, [P, i64, i32, i32, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: status {status}")
        self.status = status


def _p(a):
    return None if a is None else a.ctypes.data


def _edges(edges):
    e = np.ascontiguousarray(edges, dtype=np.int32).reshape(-1, 2)
    return e, int(e.shape[0])


def num_parts(m: int, P: int) -> int:
    return int(lib().orc_num_parts(m, P))


def part_sizes(m: int, k: int) -> np.ndarray:
    s = np.zeros(k, dtype=np.int64)
    lib().orc_part_sizes(m, k, _p(s))
    return s


@dataclass
class CostReport:
    k: int
    load_count: int     # L = sum_p |V_p|
    touched: int
    cut_cost: int       # C = L - touched (Eq. 1)
    max_size: int
    min_size: int
    per_part: np.ndarray

    @property
    def replication(self) -> float:
        return self.load_count / self.touched

    @property
    def redundant_fraction(self) -> float:
        return self.cut_cost / self.load_count

    m: int = 0

    @property
    def balance_factor(self) -> float:
        """max partition size / average partition size."""
        return float(self.max_size) / (self.m / self.k)


def cost(edges, n: int, part, k: int) -> CostReport:
    e, m = _edges(edges)
    part = np.ascontiguousarray(part, dtype=np.int32)
    per = np.zeros(k, dtype=np.int64)
    rep = np.zeros(6, dtype=np.int64)
    st = lib().orc_cost(_p(e), m, n, _p(part), k, _p(per), _p(rep))
    if st:
        raise OracleError(st, "orc_cost")
    return CostReport(*[int(x) for x in rep], per_part=per, m=m)


def default_partition(m: int, P: int) -> np.ndarray:
    part = np.zeros(m, dtype=np.int32)
    st = lib().orc_default_partition(m, P, _p(part))
    if st:
        raise OracleError(st, "orc_default_partition")
    return part


def build_T(edges, n: int):
    """Contracted clone-and-connect graph T as CSR (t_ptr[m+1], t_adj, t_w)."""
    e, m = _edges(edges)
    cap = 4 * m
    t_ptr = np.zeros(m + 1, dtype=np.int64)
    t_adj = np.zeros(max(cap, 1), dtype=np.int32)
    t_w = np.zeros(max(cap, 1), dtype=np.int32)
    nnz = np.zeros(1, dtype=np.int64)
    st = lib().orc_build_T(_p(e), m, n, _p(t_ptr), _p(t_adj), _p(t_w), cap, _p(nnz))
    if st:
        raise OracleError(st, "orc_build_T")
    z = int(nnz[0])
    return t_ptr, t_adj[:z].copy(), t_w[:z].copy()


def epg1(t_ptr, t_adj, t_w, sizes) -> np.ndarray:
    sizes = np.ascontiguousarray(sizes, dtype=np.int64)
    ntask = int(t_ptr.size - 1)
    part = np.zeros(ntask, dtype=np.int32)
    t_ptr = np.ascontiguousarray(t_ptr, dtype=np.int64)
    t_adj = np.ascontiguousarray(t_adj, dtype=np.int32)
    t_w = np.ascontiguousarray(t_w, dtype=np.int32)
    st = lib().orc_epg1(ntask, _p(t_ptr), _p(t_adj) if t_adj.size else None, _p(t_w) if t_w.size else None,
                        _p(sizes), sizes.size, _p(part))
    if st:
        raise OracleError(st, "orc_epg1")
    return part


def epg2(edges, n: int, sizes, hub: int) -> np.ndarray:
    """EPG-2 (O5') with explicit cluster sizes; vertices with more than `hub` tasks
    attract none (the partitioner passes hub = 4P)."""
    e, m = _edges(edges)
    sizes = np.ascontiguousarray(sizes, dtype=np.int64)
    part = np.zeros(max(m, 1), dtype=np.int32)
    st = lib().orc_epg2(m, _p(e), n, _p(sizes), sizes.size, hub, _p(part))
    if st:
        raise OracleError(st, "orc_epg2")
    return part[:m]


def partition(edges, n: int, P: int, shards: int = 1, method: int = 1, ranked: bool = False):
    """method 1: EPG-1 on the contracted clone-and-connect graph T (O5); method 2: EPG-2,
    growing on the EP objective of Eq. (1) directly (O5', reading Z20). ranked: also return
    each task's growth step within its partition (reading Z22)."""
    e, m = _edges(edges)
    part = np.zeros(max(m, 1), dtype=np.int32)
    rank = np.zeros(max(m, 1), dtype=np.int32)
    st = lib().orc_partition_method_ranked(_p(e), m, n, P, shards, method, _p(part), _p(rank))
    if st:
        raise OracleError(st, "orc_partition")
    return (part[:m], rank[:m]) if ranked else part[:m]


@dataclass
class Layout:
    edge_perm: np.ndarray          # [m] new -> old
    part_edge_begin: np.ndarray    # [k+1]
    vertex_perm: np.ndarray        # [n] old -> new
    part_vertex_begin: np.ndarray  # [k+1] (beginA)
    halo_begin: np.ndarray         # [k+1]
    halo_ids: np.ndarray           # [C]
    slots: np.ndarray              # [m][2] uint16


def rb_depth(k: int, shards: int = 1, leaf_parts: int = 256) -> int:
    """Bisection depth of EPG-RB (O5'', reading Z21)."""
    return int(lib().orc_rb_depth(k, shards, leaf_parts))


def partition_rb(edges, n: int, P: int, shards: int = 1, leaf_parts: int = 256, ranked: bool = False):
    """EPG-RB (O5''): recursive graph-growing bisection, EPG-2 in every leaf (ranked: also
    the growth step of every task within its partition, reading Z22)."""
    e, m = _edges(edges)
    part = np.zeros(max(m, 1), np.int32)
    rank = np.zeros(max(m, 1), np.int32)
    st = lib().orc_partition_rb_ranked(_p(e), m, n, P, shards, leaf_parts, _p(part), _p(rank))
    if st:
        raise OracleError(st, "orc_partition_rb")
    return (part[:m], rank[:m]) if ranked else part[:m]


def remap(edges, n: int, part, k: int, key=None) -> Layout:
    """O6; key (optional, reading Z22): tasks of a partition ordered by (key, id)."""
    e, m = _edges(edges)
    part = np.ascontiguousarray(part, dtype=np.int32)
    kk = None if key is None else np.ascontiguousarray(key, dtype=np.int32)
    out = Layout(np.zeros(m, np.int32), np.zeros(k + 1, np.int32), np.zeros(n, np.int32),
                 np.zeros(k + 1, np.int32), np.zeros(k + 1, np.int32), np.zeros(2 * m, np.int32),
                 np.zeros((m, 2), np.uint16))
    st = lib().orc_remap_keyed(_p(e), m, n, _p(part), _p(kk) if kk is not None else None, k, _p(out.edge_perm),
                               _p(out.part_edge_begin), _p(out.vertex_perm), _p(out.part_vertex_begin),
                               _p(out.halo_begin), _p(out.halo_ids), 2 * m, _p(out.slots))
    if st:
        raise OracleError(st, "orc_remap")
    out.halo_ids = out.halo_ids[: int(out.halo_begin[k])].copy()
    return out


def shard_halos(edges, n: int, part, k: int, G: int, vertex_perm, part_vertex_begin):
    e, m = _edges(edges)
    begin = np.zeros(G * G + 1, np.int32)
    ids = np.zeros(2 * m, np.int32)
    # converted inputs are bound to names: a temporary would be freed before the C call
    part = np.ascontiguousarray(part, np.int32)
    vertex_perm = np.ascontiguousarray(vertex_perm, np.int32)
    part_vertex_begin = np.ascontiguousarray(part_vertex_begin, np.int32)
    st = lib().orc_shard_halos(_p(e), m, n, _p(part), k, G, _p(vertex_perm), _p(part_vertex_begin), _p(begin),
                               _p(ids), 2 * m)
    if st:
        raise OracleError(st, "orc_shard_halos")
    return begin, ids[: int(begin[-1])].copy()


def cfd_flux(edges, n: int, normals, U) -> np.ndarray:
    e, m = _edges(edges)
    F = np.zeros((n, 5), np.float64)
    normals = np.ascontiguousarray(normals, np.float32)
    U = np.ascontiguousarray(U, np.float32)
    lib().orc_cfd_flux(_p(e), m, n, _p(normals), _p(U), _p(F))
    return F


def cfd_flux_abs(edges, n: int, normals, U) -> np.ndarray:
    """S[v] = sum of |Phi_e| over v's edges (scale of the componentwise metric, Z14)."""
    e, m = _edges(edges)
    Sv = np.zeros((n, 5), np.float64)
    normals = np.ascontiguousarray(normals, np.float32)
    U = np.ascontiguousarray(U, np.float32)
    lib().orc_cfd_flux_abs(_p(e), m, n, _p(normals), _p(U), _p(Sv))
    return Sv


def cfd_step(edges, n: int, normals, U, dt):
    e, m = _edges(edges)
    Uout = np.zeros((n, 5), np.float64)
    F = np.zeros((n, 5), np.float64)
    normals = np.ascontiguousarray(normals, np.float32)
    U = np.ascontiguousarray(U, np.float32)
    dt = np.ascontiguousarray(dt, np.float32)
    lib().orc_cfd_step(_p(e), m, n, _p(normals), _p(U), _p(dt), _p(Uout), _p(F))
    return Uout, F


def incidence(edges, n: int):
    """orc_incidence: per-vertex (edge, side) lists, ascending edge -> (off [n+1], inc [2m])."""
    e, m = _edges(edges)
    off = np.zeros(n + 1, np.int64)
    inc = np.zeros(max(2 * m, 1), np.int64)
    lib().orc_incidence(_p(e), m, n, _p(off), _p(inc))
    return off, inc


def cfd_step_omp(edges, n: int, normals, U, dt, inc=None):
    """orc_cfd_step over all host cores (CPU-baseline timing only; bit-identical to cfd_step)
    -> (U', F, threads). inc: incidence(edges, n), built once per mesh, or None."""
    e, m = _edges(edges)
    Uout = np.zeros((n, 5), np.float64)
    F = np.zeros((n, 5), np.float64)
    normals = np.ascontiguousarray(normals, np.float32)
    U = np.ascontiguousarray(U, np.float32)
    dt = np.ascontiguousarray(dt, np.float32)
    off, ic = (None, None) if inc is None else inc
    th = lib().orc_cfd_step_omp(_p(e), m, n, _p(normals), _p(U), _p(dt), _p(Uout), _p(F),
                                _p(off) if off is not None else None, _p(ic) if ic is not None else None)
    return Uout, F, int(th)


def gather_scatter(edges, n: int, x, w=None) -> np.ndarray:
    e, m = _edges(edges)
    y = np.zeros(n, np.float64)
    wa = None if w is None else np.ascontiguousarray(w, np.float32)
    x = np.ascontiguousarray(x, np.float32)
    lib().orc_gather_scatter(_p(e), m, n, _p(wa), _p(x), _p(y))
    return y


def spmv(edges, n: int, w, x) -> np.ndarray:
    e, m = _edges(edges)
    y = np.zeros(n, np.float64)
    w = np.ascontiguousarray(w, np.float32)
    x = np.ascontiguousarray(x, np.float32)
    lib().orc_spmv(_p(e), m, n, _p(w), _p(x), _p(y))
    return y


def partition_random(m: int, P: int, seed: int = 1605) -> np.ndarray:
    """PowerGraph random edge placement, exactly balanced (reading Z18)."""
    part = np.empty(m, np.int32)
    st = lib().orc_partition_random(m, P, seed & 0xFFFFFFFFFFFFFFFF, _p(part))
    if st:
        raise OracleError(st, "partition_random")
    return part


def partition_greedy(edges, n: int, P: int) -> np.ndarray:
    """PowerGraph greedy edge placement (reading Z19)."""
    e, m = _edges(edges)
    part = np.empty(m, np.int32)
    st = lib().orc_partition_greedy(_p(e), m, n, P, _p(part))
    if st:
        raise OracleError(st, "partition_greedy")
    return part
