#!/usr/bin/env python
"""2+-rank NCCL parity check (torchrun, one process per GPU): the element-partitioned run with the NCCL
p / u.n face-trace halo must match the single-GPU run to 1e-13 (per element, relative to the state max).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 scripts/nccl_parity.py [N M n]
Prints one JSON line on rank 0 and exits non-zero on mismatch.
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1808_08645_b200 import Solver  # noqa: E402
from paper_1808_08645_b200 import lib as L  # noqa: E402
from workloads import kuhn, media, states  # noqa: E402


def main():
    N, M, n = (int(x) for x in (sys.argv[1:4] if len(sys.argv) >= 4 else (4, 2, 6)))
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    v, e = kuhn.kuhn_mesh(n)
    c2 = media.random_c2(len(e), M)
    Q0 = states.random_state(len(e), N)
    dt, nsteps = 1e-3, 4
    idbuf = [L.bbwadg_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(idbuf, src=0)
    plan = L.bbwadg_partition_plan(v, e, world, rank)
    gid = np.ascontiguousarray(plan["gid"], dtype=np.int64)
    s = Solver(v, e, N, M, c2[gid], device=local, rank=rank, world_size=world, nccl_id=idbuf[0], c2_gids=gid)
    s.set_state(Q0)
    for i in range(nsteps):
        s.step(i * dt, dt)
    s.run(nsteps * dt, dt, 1)  # + one more step through bbwadg_run (finiteness + NCCL async-error poll)
    loc = s.get_state()
    g = s.info()["global_ids"]
    parts = [None] * world
    dist.all_gather_object(parts, (g, loc))
    ok = True
    if rank == 0:
        ref_s = Solver(v, e, N, M, c2, device=local)
        ref_s.set_state(Q0)
        for i in range(nsteps):
            ref_s.step(i * dt, dt)
        ref_s.run(nsteps * dt, dt, 1)
        ref = ref_s.get_state()
        out = np.zeros_like(ref)
        for gg, ll in parts:
            out[gg] = ll
        err = float(np.max(np.abs(out - ref)) / np.max(np.abs(ref)))
        ok = err <= 1e-13
        print(json.dumps({"world": world, "N": N, "M": M, "K": len(e), "max_rel_err": err, "ok": ok,
                          "halo_faces": [int(p[0].shape[0]) for p in parts]}), flush=True)
    okt = torch.tensor([1 if ok else 0], device=dev)
    dist.broadcast(okt, 0)
    s.close()
    dist.destroy_process_group()
    sys.exit(0 if okt.item() else 1)


if __name__ == "__main__":
    main()
