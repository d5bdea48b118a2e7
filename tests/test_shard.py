"""The multi-GPU path on CPU: halo sets against the oracle (bit-exact) and
the sharded time step over gloo with world size 2 and 4 (compute emulated, exchange real)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth as S


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("sched", ["ep", "ep2", "default"])
def test_shard_halos_host_matches_oracle(small_mesh, G, sched):
    from paper_1605_02043_b200 import epg
    M = small_mesh
    P = 256
    k = O.num_parts(M.m, P)
    if sched == "default":
        part = O.default_partition(M.m, P)
    else:
        part = O.partition(M.edges, M.n, P, G, method=2 if sched == "ep2" else 1)
    L = O.remap(M.edges, M.n, part, k)
    begin, ids = epg.shard_halos_host(L.part_vertex_begin, L.halo_begin, L.halo_ids, k, G)
    rb, rids = O.shard_halos(M.edges, M.n, part, k, G, L.vertex_perm, L.part_vertex_begin)
    assert np.array_equal(begin, rb) and np.array_equal(ids, rids)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, result_q, method=1):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    sys.path.insert(0, here)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth as S2
        import oracle as O2
        from shard_emulator import EmuCtx
        from paper_1605_02043_b200 import epg
        from paper_1605_02043_b200.shard import Shard, Comm
        M = S2.kuhn_mesh(nbox=7, n_keep=1900)
        P = 128
        k = O2.num_parts(M.m, P)
        part = O2.partition(M.edges, M.n, P, world, method=method)
        emu = EmuCtx(M.edges, M.n, M.normals, part, k)
        U = S2.cfd_state(M.n).astype(np.float64)
        dt = S2.cfd_dt(M.volume).astype(np.float64)
        vp = emu.L.vertex_perm
        Un = np.empty_like(U); Un[vp] = U
        dtn = np.empty_like(dt); dtn[vp] = dt
        # every rank: full-size arrays; only owned rows are authoritative. Make the foreign
        # rows stale so the pull must deliver them.
        sh = Shard(emu, emu.plan, emu.layout, epg.KERNEL_CFD_FLUX, world, rank, dtype=torch.float64)
        lo, hi = sh.owned()
        state_in = torch.from_numpy(Un.copy())
        stale = np.ones(M.n, bool); stale[lo:hi] = False; stale[emu.plan.touched:] = False
        state_in[torch.from_numpy(stale)] = 1e9
        state_out = torch.zeros_like(state_in)
        sh.step(Comm(), state_in, state_out, None, torch.from_numpy(dtn))
        ref, _ = O2.cfd_step(M.edges, M.n, M.normals, U.astype(np.float32), dt.astype(np.float32))
        refn = np.empty_like(ref); refn[vp] = ref
        got = state_out.numpy()
        err = np.abs(got[lo:hi] - refn[lo:hi]).max() / np.abs(refn).max()
        unt = np.abs(got[emu.plan.touched:] - refn[emu.plan.touched:]).max() if emu.plan.touched < M.n else 0.0
        result_q.put((rank, float(err), float(unt), hi - lo, sum(v.numel() for v in sh.recv_ids.values())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,method", [(2, 1), (4, 1), (2, 2), (4, 2)])
def test_sharded_step_gloo(world, method):
    """method 1: hierarchical EPG-1 shards; method 2: hierarchical EPG-2 (the bench's)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, method)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(world))
    assert sum(r[3] for r in res) > 0
    assert sum(r[4] for r in res) > 0            # halos actually crossed ranks
    for rank, err, unt, owned, halos in res:
        assert err <= 1e-12 and unt == 0.0, (rank, err, unt)
