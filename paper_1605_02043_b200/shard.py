"""Multi-GPU execution of a plan across G shards (the paper is single-GPU).

One process per GPU. Every rank holds the same plan (built from the same hierarchical EPG-1
map with shards = G) and full-size state arrays; rank g is authoritative for the vertices
its shard owns. A time step on rank g:

  1. pull   : owners send the rows of Halo^{g<-g'} (O7) -- state flows from lower shards up
  2. edges  : the staged kernel over g's execution partitions (epg_run_edges)
  3. push   : g sends to each lower owner one partial sum per vertex of Halo^{g<-g'}
              (epg_shard_reduce); g accumulates what higher shards push, in ascending peer
              order (epg_accumulate_rows)
  4. finalise: g completes its shared vertices (epg_run_finalise)

The exchanges are grouped point-to-point transfers over a torch.distributed process group
(NCCL over NVLink on GPUs; gloo in the CPU tests). Pack / unpack run in the library
(epg_permute_rows gather / scatter). The phases are separate methods so tests can run G
virtual shards in one process.
"""
from __future__ import annotations

import numpy as np
import torch

from . import epg


class Comm:
    """Grouped point-to-point exchange over a torch.distributed process group."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def exchange(self, sends: dict, recvs: dict):
        """sends / recvs: {peer: tensor}. Blocks until every transfer completed."""
        d = self.dist
        ops = [d.P2POp(d.isend, t, peer, self.group) for peer, t in sorted(sends.items()) if t.numel()]
        ops += [d.P2POp(d.irecv, t, peer, self.group) for peer, t in sorted(recvs.items()) if t.numel()]
        if ops:
            for r in d.batch_isend_irecv(ops):
                r.wait()


class Shard:
    """Rank g's part of a plan split into G shards (compute backend: an epg.Context)."""

    def __init__(self, ctx, plan, layout, kernel: int, G: int, g: int, dtype=torch.float32):
        self.ctx, self.plan, self.kernel, self.G, self.g = ctx, plan, kernel, G, g
        self.dtype = dtype
        self.row = epg.ROW[kernel]
        self.r = ctx.shard_ranges(plan, G, g)
        pvb = layout.part_vertex_begin.cpu().numpy()
        hb = layout.halo_begin.cpu().numpy()
        hid = layout.halo_ids.cpu().numpy()
        begin, ids = epg.shard_halos_host(pvb, hb, hid, plan.k, G)
        dev = ctx.device
        # recv_ids[p]: Halo^{g<-p} (p < g); send_ids[p]: Halo^{p<-g} (p > g)
        self.recv_ids = {p: torch.from_numpy(ids[begin[g * G + p]:begin[g * G + p + 1]].copy()).to(dev)
                         for p in range(g)}
        self.send_ids = {p: torch.from_numpy(ids[begin[p * G + g]:begin[p * G + g + 1]].copy()).to(dev)
                         for p in range(g + 1, G)}
        self.acc = torch.zeros((plan.n, self.row) if self.row > 1 else plan.n, dtype=dtype, device=dev)

    def _rows(self, count):
        shape = (count, self.row) if self.row > 1 else (count,)
        return torch.empty(shape, dtype=self.dtype, device=self.ctx.device)

    # -- phases ----------------------------------------------------------------------
    def pull_out(self, state_in) -> dict:
        return {p: self.ctx.permute_rows(state_in, ids, epg.PERM_GATHER, out=self._rows(ids.numel()))
                for p, ids in self.send_ids.items()}

    def pull_buffers(self) -> dict:
        return {p: self._rows(ids.numel()) for p, ids in self.recv_ids.items()}

    def pull_in(self, state_in, rows: dict):
        for p in sorted(rows):
            if rows[p].numel():
                self.ctx.permute_rows(rows[p], self.recv_ids[p], epg.PERM_SCATTER, out=state_in)

    def edges(self, state_in, state_out, payload=None, vconst=None):
        self.ctx.run_edges(self.plan, self.kernel, state_in, state_out, payload, vconst,
                           self.r["exec_first"], self.r["exec_count"])

    def push_out(self) -> dict:
        return {p: self.ctx.shard_reduce(self.plan, self.kernel, ids, self.r["halo_first"], self.r["halo_count"],
                                         self._rows(ids.numel()))
                for p, ids in self.recv_ids.items()}

    def push_buffers(self) -> dict:
        return {p: self._rows(ids.numel()) for p, ids in self.send_ids.items()}

    def push_in(self, rows: dict):
        for p in sorted(rows):                        # ascending peer order: deterministic sums
            if rows[p].numel():
                self.ctx.accumulate_rows(rows[p], self.send_ids[p], self.acc)

    def finalise(self, state_in, state_out, payload=None, vconst=None):
        self.ctx.run_finalise(self.plan, self.kernel, state_in, state_out, payload, vconst,
                              self.r["shared_first"], self.r["shared_count"], self.r["halo_first"],
                              self.r["halo_count"], self.acc, untouched=True)

    # -- one time step over a process group --------------------------------------------
    def step(self, comm: Comm, state_in, state_out, payload=None, vconst=None):
        recv = self.pull_buffers()
        comm.exchange(self.pull_out(state_in), recv)
        self.pull_in(state_in, recv)
        self.edges(state_in, state_out, payload, vconst)
        recv = self.push_buffers()
        comm.exchange(self.push_out(), recv)
        self.push_in(recv)
        self.finalise(state_in, state_out, payload, vconst)

    def owned(self):
        lo = self.r["vertex_first"]
        return lo, lo + self.r["vertex_count"]


def run_virtual(shards: list, states_in: list, states_out: list, payload=None, vconst=None):
    """One step of G shards held in this process (tests on one GPU): the phases of all
    shards interleaved, transfers by tensor copies."""
    G = len(shards)
    sends = [sh.pull_out(states_in[g]) for g, sh in enumerate(shards)]
    for g, sh in enumerate(shards):
        sh.pull_in(states_in[g], {p: sends[p][g] for p in range(g)})
    for g, sh in enumerate(shards):
        sh.edges(states_in[g], states_out[g], payload, vconst)
    pushes = [sh.push_out() for sh in shards]
    for g, sh in enumerate(shards):
        sh.push_in({p: pushes[p][g] for p in range(g + 1, G)})
    for g, sh in enumerate(shards):
        sh.finalise(states_in[g], states_out[g], payload, vconst)


def assemble_owned(shards: list, states_out: list) -> np.ndarray:
    """The authoritative rows of every shard, concatenated in vertex order (host)."""
    parts = []
    for sh, s in zip(shards, states_out):
        lo, hi = sh.owned()
        parts.append(s[lo:hi].cpu().numpy())
    return np.concatenate(parts)
