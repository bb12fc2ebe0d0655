"""The multi-rank (z-slab) path on CPU: world_size 2/3 over torch.distributed
gloo.  Each rank builds the library's host plan (commet_plan_*: owned CSR with
ghost elements, halo rows, per-peer maps, the interface-first colour split),
assembles its own elements with the ORACLE into the plan's owned and halo
layouts in the assemble's two phases (interface elements, then the exchange
started, then the interior), exchanges the halo segments with gloo send/recv
exactly as the NCCL path does, unpacks with the plan's maps and must reproduce
the global oracle's rows bit-for-bit in the pattern and to 1e-13 in the
values.  (The kernels and NCCL calls themselves need a GPU: -m gpu tests.)"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, n, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import oracle
    import paper_2510_00884_b200 as pc
    from synth import gen
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = gen.slab_partition(name, world, rank, n=n)
        plan = pc.Plan(c)
        rp, ci = plan.csr()
        nb, ne = c["owned_node_begin"], c["owned_node_end"]
        # global reference (every rank computes it; small meshes)
        g = gen.make_config(name, n=n)
        grp, gci = oracle.pattern(g["n_nodes"], g["conn"])
        gr, gv, _ = oracle.assemble(g["ncm"], g["n_nodes"], g["conn"], g["gradN"], g["qp_w"], g["u"], grp, gci)
        pattern_ok = (np.array_equal(ci, gci[grp[3 * nb]:grp[3 * ne]]) and
                      np.array_equal(rp, grp[3 * nb:3 * ne + 1] - grp[3 * nb]))
        # the assemble's two phases (NCCL mode): every colour's interface elements first, then the
        # exchange, started before the interior elements are assembled
        n_el = c["conn"].shape[0]
        cs, perm = plan.colours(n_el)
        nif = plan.colour_iface()
        iface = np.concatenate([perm[cs[k]:cs[k] + nif[k]] for k in range(plan.n_colours)] + [np.zeros(0, np.int64)])
        inter = np.concatenate([perm[cs[k] + nif[k]:cs[k + 1]] for k in range(plan.n_colours)] + [np.zeros(0, np.int64)])
        touches_halo = ((c["conn"] < nb) | (c["conn"] >= ne)).any(axis=1)
        iface_ok = (np.array_equal(np.sort(iface), np.nonzero(touches_halo)[0]) and
                    np.array_equal(np.sort(np.concatenate([iface, inter])), np.arange(n_el)))

        def part(els, rp_, ci_, b0, b1):
            sub = np.ascontiguousarray(c["conn"][els])
            return oracle.assemble(c["ncm"], c["n_nodes"], sub, c["gradN"][els], c["qp_w"][els], c["u"],
                                   rp_, ci_, node_begin=b0, node_end=b1)[:2]
        # phase 0: interface elements into the owned rows and the halo rows (contiguous plane
        # above the slab) -- the halo rows are complete after this phase
        hn, hrp, hci = plan.halo()
        r_own, v_own = part(iface, rp, ci, nb, ne)
        if hn.size:
            assert np.array_equal(hn, np.arange(hn[0], hn[-1] + 1))
            r_h, v_h = part(iface, hrp, hci, int(hn[0]), int(hn[-1]) + 1)
        # exchange: sends first (gloo isend) ...
        reqs = []
        for k in range(plan.n_send):
            peer, (v0, v1), (r0, r1) = plan.send(k)
            reqs.append(dist.isend(torch.from_numpy(v_h[v0:v1].copy()), peer))
            reqs.append(dist.isend(torch.from_numpy(r_h[r0:r1].copy()), peer))
        # ... phase 1: the interior elements while the halo is in flight; receives, unpack in rank order
        r_in, v_in = part(inter, rp, ci, nb, ne)
        r_own += r_in
        v_own += v_in
        for k in range(plan.n_recv):
            peer, vmap, rmap = plan.recv(k)
            bv, br = torch.empty(vmap.size, dtype=torch.float64), torch.empty(rmap.size, dtype=torch.float64)
            dist.recv(bv, peer)
            dist.recv(br, peer)
            v_own[vmap] += bv.numpy()
            r_own[rmap] += br.numpy()
        for q in reqs:
            q.wait()
        ref_r = gr[3 * nb:3 * ne]
        ref_v = gv[grp[3 * nb]:grp[3 * ne]]
        er = np.abs(r_own - ref_r).max() / np.abs(gr).max()
        ev = np.abs(v_own - ref_v).max() / np.abs(gv).max()
        out_q.put((rank, bool(pattern_ok and iface_ok), float(er), float(ev), plan.n_send, plan.n_recv))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,n,world", [("c1", 4, 2), ("c2", 6, 3), ("c4", 3, 2)])
def test_slab_exchange_gloo(name, n, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, pattern_ok, er, ev, ns, nr in sorted(res):
        assert pattern_ok, f"rank {rank}: plan CSR or interface split differs from the global pattern"
        assert er < 1e-13 and ev < 1e-13, (rank, er, ev)
        assert ns == (1 if rank < world - 1 else 0) and nr == (1 if rank > 0 else 0)


def test_plan_rejects_inconsistent_partition():
    import paper_2510_00884_b200 as pc
    from synth import gen
    c = gen.slab_partition("c1", 2, 1)
    c["rank_node_begin"] = c["rank_node_begin"].copy()
    c["rank_node_begin"][1] += 1
    with pytest.raises(pc.CommetError, match="owned range"):
        pc.Plan(c)
    c = gen.slab_partition("c1", 2, 0)
    c["n_ranks"] = 1  # halo nodes without a partition
    with pytest.raises(pc.CommetError, match="outside the owned range"):
        pc.Plan(c)
