"""CPU emulation of the library calls a Shard makes (test infrastructure: uses oracle/).

It follows the kernel contract of include/epg.h with the oracle's fp64 arithmetic on the EP
layout (no execution split): epg_run_edges writes U + dt F_local for owned rows and the
halo partials per halo position; epg_shard_reduce / epg_accumulate_rows /
epg_run_finalise as documented. Lets the multi-process exchange logic of
paper_1605_02043_b200/shard.py run under gloo on CPU."""
from __future__ import annotations

from types import SimpleNamespace

import numpy as np
import torch

import oracle as O


class EmuCtx:
    device = torch.device("cpu")

    def __init__(self, edges, n, normals, part, k):
        L = O.remap(edges, n, part, k)
        self.L = L
        self.k, self.n = k, n
        self.edges_new = L.vertex_perm[edges[L.edge_perm]].astype(np.int32)
        self.normals_new = normals[L.edge_perm].astype(np.float32)
        C = L.halo_ids.size
        self.shared_ids = np.unique(L.halo_ids).astype(np.int32)
        self.sidx = -np.ones(n, np.int64)
        self.sidx[self.shared_ids] = np.arange(self.shared_ids.size)
        order = np.argsort(L.halo_ids, kind="stable")
        self.hv = {}
        for h in order:
            self.hv.setdefault(int(self.sidx[L.halo_ids[h]]), []).append(int(h))
        self.halo_buf = np.zeros((C, 5))
        self.plan = SimpleNamespace(m=edges.shape[0], n=n, k=k, k_exec=k, touched=int(L.part_vertex_begin[k]),
                                    cut_cost=C, cut_cost_exec=C, shared=self.shared_ids.size)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a))
        self.layout = SimpleNamespace(part_vertex_begin=t(L.part_vertex_begin), halo_begin=t(L.halo_begin),
                                      halo_ids=t(L.halo_ids), vertex_perm=t(L.vertex_perm), edge_perm=t(L.edge_perm))

    def shard_ranges(self, plan, G, g):
        pb, pe = g * self.k // G, (g + 1) * self.k // G
        pvb, hb = self.L.part_vertex_begin, self.L.halo_begin
        s0 = int(np.searchsorted(self.shared_ids, pvb[pb]))
        s1 = int(np.searchsorted(self.shared_ids, pvb[pe]))
        return dict(exec_first=pb, exec_count=pe - pb, halo_first=int(hb[pb]), halo_count=int(hb[pe] - hb[pb]),
                    vertex_first=int(pvb[pb]), vertex_count=int(pvb[pe] - pvb[pb]), shared_first=s0,
                    shared_count=s1 - s0)

    def permute_rows(self, src, ids, mode, out):
        if mode == 0:
            out[:] = src[ids.long()]
        else:
            out[ids.long()] = src
        return out

    def run_edges(self, plan, kernel, state_in, state_out, payload, vconst, first, count):
        U = state_in.numpy()
        dt = vconst.numpy()
        peb, pvb, hb = self.L.part_edge_begin, self.L.part_vertex_begin, self.L.halo_begin
        out = state_out.numpy()
        for p in range(first, first + count):
            e = self.edges_new[peb[p]:peb[p + 1]]
            F = O.cfd_flux(e, self.n, self.normals_new[peb[p]:peb[p + 1]], U.astype(np.float32))
            own = np.arange(pvb[p], pvb[p + 1])
            out[own] = U[own] + dt[own, None] * F[own]
            for h in range(hb[p], hb[p + 1]):
                self.halo_buf[h] = F[self.L.halo_ids[h]]

    def _partial(self, s, h0, h1):
        tot = np.zeros(5)
        for h in self.hv.get(s, []):
            if h0 <= h < h1:
                tot += self.halo_buf[h]
        return tot

    def shard_reduce(self, plan, kernel, ids, halo_first, halo_count, out):
        for i, u in enumerate(ids.tolist()):
            out[i] = torch.from_numpy(self._partial(int(self.sidx[u]), halo_first, halo_first + halo_count))
        return out

    def accumulate_rows(self, src, ids, acc):
        acc[ids.long()] += src

    def run_finalise(self, plan, kernel, state_in, state_out, payload, vconst, shared_first, shared_count,
                     halo_first, halo_count, acc, untouched=True):
        out, dt, a = state_out.numpy(), vconst.numpy(), acc.numpy()
        for s in range(shared_first, shared_first + shared_count):
            v = int(self.shared_ids[s])
            tot = self._partial(s, halo_first, halo_first + halo_count) + a[v]
            a[v] = 0.0
            out[v] += dt[v] * tot
        if untouched:
            t0 = self.plan.touched
            out[t0:] = state_in.numpy()[t0:]
