"""Launch overhead: steps/s of bbwadg_run with the CUDA-graph replay vs individual launches (BBWADG_NO_GRAPH)
on small meshes, where host launch cost is a large share of the step.   python scripts/graph_timing.py"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1808_08645_b200 import Solver  # noqa: E402
from workloads import kuhn, media, states  # noqa: E402

rows = []
for n, N, M in [(2, 3, 1), (4, 3, 1), (8, 5, 3), (16, 7, 4)]:
    v, e = kuhn.kuhn_mesh(n)
    s = Solver(v, e, N, M, media.random_c2(len(e), M))
    s.set_state(states.random_state(len(e), N))
    res = {}
    for mode in ("graph", "launches"):
        if mode == "launches":
            os.environ["BBWADG_NO_GRAPH"] = "1"
        s.run(0.0, 1e-4, 20)
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(3):
            t = time.perf_counter()
            s.run(0.0, 1e-4, 200)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t)
        res[mode] = 200 / best
        os.environ.pop("BBWADG_NO_GRAPH", None)
    rows.append({"K": len(e), "N": N, "M": M, "steps_per_s_graph": res["graph"], "steps_per_s_launches": res["launches"],
                 "speedup": res["graph"] / res["launches"]})
    s.close()
print(json.dumps(rows, indent=1))
