"""Multi-process (world_size 2 and 4, gloo on CPU) checks of the N>1 host logic.

Each rank computes its partition plan with the library's host code (the same RCB
partition and halo ordering ``bbwadg_setup`` uses for the NCCL face-trace halo),
the ranks exchange their plans over gloo, and every rank verifies that
  * the partitions cover every element exactly once;
  * interior elements have no off-rank neighbour, boundary elements have one;
  * rank r's message to r' lists exactly the faces r' expects, in the same order,
    and every ghost face really is shared with the claimed neighbour (checked with
    an independent numpy face matching).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _faces_numpy(e):
    faces = {}
    for k in range(len(e)):
        for f in range(4):
            key = tuple(sorted(int(x) for i, x in enumerate(e[k]) if i != f))
            faces.setdefault(key, []).append((k, f))
    nbr = -np.ones((len(e), 4), dtype=np.int64)
    for lst in faces.values():
        if len(lst) == 2:
            (a, fa), (b, fb) = lst
            nbr[a, fa], nbr[b, fb] = b, a
    return nbr


def _worker(rank, world, port, shape, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1808_08645_b200 import lib as L
        from workloads import kuhn

        v, e = kuhn.kuhn_mesh(shape, h=0.25)
        plan = L.bbwadg_partition_plan(v, e, world, rank)
        plans = [None] * world
        dist.all_gather_object(plans, plan)
        nbr = _faces_numpy(e)
        owner = -np.ones(len(e), dtype=np.int64)
        for r, p in enumerate(plans):
            assert np.all(owner[p["gid"]] == -1)
            owner[p["gid"]] = r
        assert np.all(owner >= 0)
        me = plans[rank]
        gid = me["gid"]
        for i, k in enumerate(gid):
            off = [owner[n] != rank for n in nbr[k] if n >= 0]
            assert (i >= me["n_interior"]) == any(off)
        for peer in range(world):
            if peer == rank:
                continue
            sent = me["send"][me["send"][:, 2] == peer][:, [0, 1]]
            expected = plans[peer]["recv"][plans[peer]["recv"][:, 2] == rank][:, [3]]
            # what peer expects (source global element per ghost slot, in order) == what I send
            assert np.array_equal(sent[:, 0], expected[:, 0])
            for (k, f), (kk, ff, src, nb) in zip(sent, plans[peer]["recv"][plans[peer]["recv"][:, 2] == rank]):
                assert nbr[kk, ff] == k and nb == k
        # balanced equal-count blocks
        sizes = [p["K_local"] for p in plans]
        assert max(sizes) - min(sizes) <= 1
        q.put((rank, "ok"))
    except Exception as ex:  # pragma: no cover - reported to the parent
        q.put((rank, repr(ex)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shape", [(2, (4, 2, 2)), (4, (4, 4, 2))])
def test_partition_plans_consistent_across_ranks(world, shape):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(60)
    assert all(r[1] == "ok" for r in res), res
