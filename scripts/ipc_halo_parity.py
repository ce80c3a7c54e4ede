"""Two (or more) processes, one partition each, peer-read halo over CUDA IPC (halo_transport 1).

    python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 --master-port 29533 \
        scripts/ipc_halo_parity.py OUT.npz [n N M steps [host|device]]

Each rank sets up its partition of the Kuhn mesh with world_size P, exports the CUDA IPC handles of its
two state buffers and its stage-epoch flag, opens every other rank's (exchanged over a gloo process group),
and advances `steps` LSRK45 steps either by bbwadg_stage with a host barrier + stream synchronisation
between stages ("host"), or by one bbwadg_run whose stages are ordered by the library's device-side epoch
barrier alone ("device"; the stage kernel reads the peers' stage inputs in place).  Rank 0 gathers the final state in global order and
writes OUT.npz (state, per-rank K_local / halo faces).  Works with several processes sharing one GPU
(the test on the 1-GPU box) or one process per GPU (NVLink peer reads).
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1808_08645_b200 import lib as L  # noqa: E402
from workloads import kuhn, media, states  # noqa: E402


def main():
    out = sys.argv[1]
    n, N, M, steps = (int(x) for x in (sys.argv[2:6] if len(sys.argv) >= 6 else (4, 5, 3, 3)))
    mode = sys.argv[6] if len(sys.argv) >= 7 else "host"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    dev = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    v, e = kuhn.kuhn_mesh(n)
    c2 = media.random_c2(len(e), M)
    Q0 = states.random_state(len(e), N)
    o = L.bbwadg_default_options()
    o.device = dev
    o.rank, o.world_size = rank, world
    o.halo_transport = 1
    ctx = L.bbwadg_setup(v, e, N, M, c2, o)
    info = L.bbwadg_query(ctx)
    gid = np.ctypeslib.as_array(info.global_ids, shape=(info.num_elements_local,)).copy()
    L.bbwadg_set_state(ctx, np.ascontiguousarray(Q0[gid]), 0)
    handles = [None] * world
    dist.all_gather_object(handles, L.bbwadg_ipc_get_handles(ctx))
    for r in range(world):
        if r != rank:
            L.bbwadg_ipc_open_peer(ctx, r, handles[r])
    dt = 1e-3
    dist.barrier()
    if mode == "device":
        L.bbwadg_run(ctx, 0.0, dt, steps)  # stages ordered by the device-side epoch barrier
    else:
        for i in range(steps):
            for s in range(5):
                L.bbwadg_stage(ctx, s, i * dt, dt)
                L.bbwadg_synchronize(ctx)
                dist.barrier()
    L.bbwadg_synchronize(ctx)
    dist.barrier()
    loc = np.empty((len(gid), 4, states.num_coeffs(N)))
    L.bbwadg_get_state(ctx, loc, 0)
    parts = [None] * world
    dist.all_gather_object(parts, (gid, loc, int(info.num_halo_faces)))
    if rank == 0:
        Q = np.zeros_like(Q0)
        for g, q, _ in parts:
            Q[g] = q
        np.savez(out, Q=Q, K_local=np.array([len(p[0]) for p in parts]), halo=np.array([p[2] for p in parts]))
    dist.barrier()
    L.bbwadg_destroy(ctx)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
