"""Peer mode across processes: two ranks on one device share their output buffers
through CUDA IPC (torch.multiprocessing reductions, gathered over a gloo process group)
and add their halo rows straight into each other's buffers.  Host barriers order the
phases; no kernel waits on another.  The concatenated rows equal the global oracle."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, name, n, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2510_00884_b200 as pc
        from synth import gen
        c = gen.slab_partition(name, world, rank, n=n)
        lib = pc.Commet(c, c["ncm"])
        res, val = lib.alloc_outputs()
        pc.setup_peer_exchange(lib, res, val, rank, world)
        lib.zero_outputs(res, val)
        torch.cuda.synchronize()
        dist.barrier()
        lib.assemble(torch.from_numpy(c["u"]).cuda(), res, val)
        torch.cuda.synchronize()
        dist.barrier()
        q.put((rank, res.cpu().numpy(), val.cpu().numpy(), lib.pattern()[1]))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_peer_mode_two_processes_ipc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    import oracle
    from synth import gen
    name, n, world = "c2", 6, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, name, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict()
    for _ in range(world):
        rank, r, v, ci = q.get(timeout=300)
        got[rank] = (r, v, ci)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = gen.make_config(name, n=n)
    grp, gci = oracle.pattern(g["n_nodes"], g["conn"])
    gr, gv, _ = oracle.assemble(g["ncm"], g["n_nodes"], g["conn"], g["gradN"], g["qp_w"], g["u"], grp, gci)
    r_all = np.concatenate([got[k][0] for k in range(world)])
    v_all = np.concatenate([got[k][1] for k in range(world)])
    assert np.array_equal(np.concatenate([got[k][2] for k in range(world)]), gci)
    assert np.abs(r_all - gr).max() <= 1e-10 * np.abs(gr).max()
    assert np.abs(v_all - gv).max() <= 1e-10 * np.abs(gv).max()
