#!/usr/bin/env python
"""CPU dry run of the host-side multi-GPU setup at the 8-GPU weak-scaling size (BASELINE config 5:
176^3 Kuhn cubes = 32.7M tets, cuts (2,2,2)): for each rank, in its own process as on a real node,
build the global mesh, run bbwadg_partition_plan (validation, face connectivity, RCB partition, halo
lists) and size that rank's local c^2 rows (the c2_gids setup path; projected on the device by bench.py).  Records wall seconds and
peak RSS per rank.

    python scripts/dryrun_8rank_setup.py [n=176] [ranks=8] > profiles/r2_dryrun_8rank_setup.json
"""
import json
import os
import resource
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, resource, sys, time
sys.path.insert(0, ROOT)
import numpy as np
t0 = time.perf_counter()
from workloads import kuhn, media
from paper_1808_08645_b200 import lib as L
n, world, rank = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
v, e = kuhn.kuhn_mesh((n, n, n), h=2.0 / (n // 2))
t1 = time.perf_counter()
plan = L.bbwadg_partition_plan(v, e, world, rank, (2, 2, 2) if world == 8 else None)
t2 = time.perf_counter()
gid = plan["gid"]
t3 = time.perf_counter()  # local c^2 rows: [K_local][35] fp64 (projected on the device in bench.py)
c2_local_bytes = int(gid.shape[0]) * 35 * 8
print(json.dumps({"rank": rank, "K_global": int(e.shape[0]), "K_local": plan["K_local"], "n_interior": plan["n_interior"],
                  "send_faces": int(plan["send"].shape[0]), "ghost_slots": int(plan["recv"].shape[0]),
                  "mesh_s": t1 - t0, "partition_plan_s": t2 - t1,
                  "c2_local_bytes": c2_local_bytes, "c2_global_bytes_if_full": int(e.shape[0]) * 35 * 8,
                  "peak_rss_gb": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6}))
'''


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 176
    world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    rows = []
    for r in range(world):
        t = time.perf_counter()
        out = subprocess.run([sys.executable, "-c", "ROOT=%r\n" % ROOT + CHILD, str(n), str(world), str(r)],
                             capture_output=True, text=True)
        if out.returncode != 0:
            rows.append({"rank": r, "error": out.stderr[-2000:]})
            continue
        d = json.loads(out.stdout.strip().splitlines()[-1])
        d["process_wall_s"] = time.perf_counter() - t
        rows.append(d)
        print(json.dumps(d), file=sys.stderr, flush=True)
    print(json.dumps({"what": f"8-rank host setup dry run, {n}^3 Kuhn cubes ({6 * n ** 3:,} tets), cuts (2,2,2)",
                      "host": os.uname().nodename, "cpu_count": os.cpu_count(), "ranks": rows}, indent=1))


if __name__ == "__main__":
    main()
