#!/usr/bin/env python
"""BBWADG hot-path benchmark: DOF-stage updates/s per B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                    [--config 5|3|4] [--N n --M m] [--dtype f64|f32] [--sweep]

A "step" is one LSRK45 step = 5 fused RK stages (volume + surface + WADG
multiply/project + LSRK update) over every element of the workload.

Default workload (``config.workload``): BASELINE config 5 per GPU -- a Kuhn-cube
mesh of 88^3 cubes = 4,088,832 tets per GPU (weak scaling: boxes 176x88x88,
176x176x88, 176^3 at 2/4/8 GPUs, element-partitioned with the NCCL face-trace
halo), N=7, M=4, smooth c^2 = 1 + 1/2 sin(pi x) sin(pi y) sin(pi z) projected to
P^4, fp64.  Inputs are synthetic (seeded) and far larger than L2 (state 15.7 GB
per GPU), so no L2 flush is needed between timed steps.

value      = 4 * K_total * Np * 5 * K_steps / (max over ranks of the device time of
             the K timed steps), CUDA events on the library's stream;
e2e        = the same metric through the public API with host buffers:
             bbwadg_set_state(pinned host) + K x bbwadg_run(1 step; includes the
             device->host read of the finiteness flag) + bbwadg_get_state(pinned host);
roofline   = the stage kernel: algorithmic bytes per launch / average launch time
             vs the measured HBM copy peak (MEASURED_PEAKS.json);
cpu_baseline = the CPU oracle (oracle/, test infrastructure) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from math import comb

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("DOF-stage updates/sec, whole job over n_gpus B200s (value_per_gpu = per B200; BBWADG acoustic RK "
          "stage, fused RHS + LSRK45)")
UNIT = "DOF-stage/s"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def factor_cuts(p: int):
    best = None
    for px in range(1, p + 1):
        for py in range(1, px + 1):
            if p % (px * py):
                continue
            pz = p // (px * py)
            if pz > py:
                continue
            sc = px - pz
            if best is None or sc < best[0]:
                best = (sc, (px, py, pz))
    return best[1]


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return os.uname().machine


def pulse_state(v, e, N, device, width=50.0):
    """SURVEY 8(d) bench state: p = exp(-width |x|^2), u = 0 (L2-projected on the device)."""
    import torch

    from workloads._l2fit import l2_fit

    Np = comb(N + 3, 3)
    Q = torch.zeros((e.shape[0], 4, Np), dtype=torch.float64, device=device)
    p = l2_fit(v, e, lambda x, y, z, xp=np: xp.exp(-width * (x * x + y * y + z * z)), N, device=device)
    Q[:, 0] = torch.from_numpy(p).to(device)
    return Q


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return pk, "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def build_workload(args, rank, world, device=None):
    from workloads import kuhn, media

    n = args.n_cubes
    if args.config == 5:
        cuts = factor_cuts(world)
        shape = (n * cuts[0], n * cuts[1], n * cuts[2])
        h = 2.0 / n
        v, e = kuhn.kuhn_mesh(shape, h=h)
        cfunc = media.c2_smooth(1.0)
        name = f"config5: Kuhn {shape[0]}x{shape[1]}x{shape[2]} cubes ({n}^3 = {6 * n ** 3:,} tets per GPU), smooth c^2 k=1"
    elif args.config == 3:
        cuts = factor_cuts(world)
        v, e = kuhn.kuhn_mesh((n * cuts[0], n * cuts[1], n * cuts[2]), h=2.0 / n)
        cfunc = media.c2_smooth(8.0)
        name = f"config3: Kuhn {n}^3 cubes per GPU ({6 * n ** 3:,} tets), sub-cell c^2 k=8"
    elif args.config == 4:
        cuts = factor_cuts(world)
        v, e = kuhn.kuhn_mesh((n * cuts[0], n * cuts[1], n * cuts[2]), h=2.0 / n)
        cfunc = media.c2_layered()
        name = f"config4: Kuhn {n}^3 cubes per GPU ({6 * n ** 3:,} tets), layered c^2"
    else:
        raise SystemExit("unknown config")
    return v, e, cfunc, cuts, name


def local_c2(v, e, cfunc, M, rank, world, cuts, device):
    """c^2_M for the elements this rank owns (rows of other ranks are ignored by the library:
    filled with 1.0)."""
    from paper_1808_08645_b200 import lib as L
    from workloads import media

    Mp = comb(M + 3, 3)
    if world == 1:
        return media.project_c2(v, e, cfunc, M, device=device), None
    plan = L.bbwadg_partition_plan(v, e, world, rank, cuts)
    gid = np.ascontiguousarray(plan["gid"], dtype=np.int64)
    return media.project_c2(v, e[gid], cfunc, M, device=device), gid  # local rows only (Solver c2_gids)


def run_ours(args):
    import torch

    rank, world, local = dist_env()
    local = local % max(1, torch.cuda.device_count())  # (oversubscription only for debugging)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        # control plane over gloo (handle / NCCL-id exchange, max-over-ranks timing): the library's own
        # transports (peer reads over CUDA IPC, or its NCCL communicator) carry the face traces
        dist.init_process_group("gloo")
    from paper_1808_08645_b200 import Solver
    from paper_1808_08645_b200 import lib as L

    N, M = args.N, args.M
    Np = comb(N + 3, 3)
    v, e, cfunc, cuts, wname = build_workload(args, rank, world, device=dev)
    c2, c2_gids = local_c2(v, e, cfunc, M, rank, world, cuts, dev)
    stream = torch.cuda.current_stream(dev)

    def make_solver(transport):
        nccl_id = None
        if world > 1 and transport == "nccl":
            import torch.distributed as dist

            idbuf = [L.bbwadg_nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(idbuf, src=0)
            nccl_id = idbuf[0]
        return Solver(v, e, N, M, c2, dtype=args.dtype, device=local, stream=stream, rank=rank, world_size=world,
                      nccl_id=nccl_id, partition=cuts if world > 1 else None, c2_gids=c2_gids,
                      halo_transport=1 if (transport == "peer" and world > 1) else 0)

    halo = args.halo if world > 1 else "none"
    if halo in ("peer", "auto"):
        # peer-read halo: map every rank's state buffers and epoch flag (CUDA IPC); "auto" falls back to the
        # NCCL transport if any rank cannot map its peers
        import torch.distributed as dist

        s = make_solver("peer")
        ok = 1
        try:
            handles = [None] * world
            dist.all_gather_object(handles, s.ipc_handles())
            s.ipc_open_peers(handles)
        except Exception as ex:  # noqa: BLE001
            if halo == "peer":
                raise
            print(f"rank {rank}: peer-read halo unavailable ({ex}); falling back to NCCL", file=sys.stderr)
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int32)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 1:
            halo = "peer"
        else:
            s.close()
            halo = "nccl"
            s = make_solver("nccl")
        dist.barrier()
    else:
        s = make_solver(halo)
    info = s.info()
    K_local = info["num_elements_local"]
    tdt = torch.float64 if args.dtype == "f64" else torch.float32
    gen = torch.Generator(device=dev)
    gen.manual_seed(1808 + rank)
    Q0 = torch.randn((K_local, 4, Np), dtype=tdt, device=dev, generator=gen)
    s.set_state(Q0)
    del Q0
    torch.cuda.synchronize()
    if world > 1:  # every rank's state is in place before any stage reads a peer's (peer-read halo)
        import torch.distributed as dist

        dist.barrier()
    h_min = 2.0 / args.n_cubes / (1 + np.sqrt(2) + np.sqrt(3))  # Kuhn tet inradius-scale height bound
    dt = 0.5 * h_min / (np.sqrt(1.5) * (N + 1) ** 2)

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    for i in range(args.warmup):
        s.step(i * dt, dt)
    torch.cuda.synchronize()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier()
        ev0.record(stream)
        for i in range(args.steps):
            s.step((args.warmup + i) * dt, dt)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = ev0.elapsed_time(ev1)
    ms_max = ms
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    K_total = info["num_elements_global"]
    dof_stage = 4.0 * K_total * Np * 5 * args.steps
    value = dof_stage / (ms_max / 1e3)
    launches = info["kernels_per_stage"] * 5 * args.steps

    # roofline of the stage kernel (only kernel at N=1: ms / launches is its average duration)
    peaks, peak_kind = load_peaks()
    stage_launches = 5 * args.steps * (2 if world > 1 else 1)
    avg_launch_s = ms / 1e3 / (5 * args.steps) if world == 1 else ms / 1e3 / (5 * args.steps)
    bytes_per_stage = info["algorithmic_bytes_per_stage"]
    achieved = bytes_per_stage / avg_launch_s / 1e9
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tfile):
        try:
            with open(tfile) as fh:
                tr = json.load(fh).get(f"N{N}M{M}{args.dtype}")
            if tr:
                traffic = tr["dram_bytes_per_launch"] * (K_local / tr["K_local"])
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": traffic,
                "peak_source": f"{peak_kind} MEASURED_PEAKS.json hbm_gbs (copy)" if peak_kind == "measured" else "fallback",
                "kernel": f"bbw::stage_kernel<N={N},M={M},{args.dtype}>",
                "algorithmic_bytes_per_launch": bytes_per_stage,
                "flops_per_launch": info["flops_per_stage"],
                "achieved_tflops": round(info["flops_per_stage"] / avg_launch_s / 1e12, 3)}

    # end-to-end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        hostQ = torch.empty((K_local, 4, Np), dtype=tdt, pin_memory=True)
        hostQ.normal_(generator=torch.Generator().manual_seed(1808 + rank)) if args.e2e_random else hostQ.fill_(0.5)
        hQ = hostQ.numpy()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        L.bbwadg_set_state(s.ctx, hQ, 0)
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
        for i in range(args.steps):
            L.bbwadg_run(s.ctx, i * dt, dt, 1)
        L.bbwadg_get_state(s.ctx, hQ, 0)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        el = t1 - t0
        if world > 1:
            import torch.distributed as dist

            t = torch.tensor([el], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        sb = K_local * 4 * Np * (8 if args.dtype == "f64" else 4)
        e2e = {"value": dof_stage / el, "unit": UNIT, "h2d_bytes_per_step": sb / args.steps,
               "d2h_bytes_per_step": (sb + 4 * args.steps) / args.steps,
               "how": "bbwadg_set_state(pinned host) + K x bbwadg_run(1 step, D2H finiteness flag) + "
                      "bbwadg_get_state(pinned host), host wall clock, max over ranks"}
        del hostQ

    out = {"metric": METRIC, "value": value, "value_per_gpu": value / world, "unit": UNIT, "n_gpus": world,
           "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
           "config": {"workload": wname, "N": N, "M": M, "K_total": K_total, "K_per_gpu": K_local,
                      "Np": Np, "dofs_per_stage": 4 * K_total * Np,
                      "parallelism": f"element-partitioned x{world} (RCB cuts {list(cuts)}) + "
                                     + ("peer-read halo (CUDA IPC, device stage barrier)" if halo == "peer"
                                        else "NCCL face-trace halo")
                      if world > 1 else "single GPU",
                      "l2": "inputs (state %.1f GB/GPU) far larger than the 126 MB L2; no flush needed"
                            % (K_local * 4 * Np * (8 if args.dtype == 'f64' else 4) / 1e9)},
           "roofline": roofline, "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary()}
    s.close()
    if rank == 0 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(N, M, args.cpu_seconds, extras=True)
    if rank == 0 and not args.no_config4:
        out["config4"] = config4_runs(args, dev)
    if rank == 0 and args.elastic:
        out["elastic"] = elastic_runs(args, dev)
    if rank == 0 and args.two_d:
        out["two_d"] = runs_2d(args, dev)
    if rank == 0 and not args.no_sweep:
        out["sweep"] = sweep(args, dev)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


def config4_runs(args, dev):
    """BASELINE config 4: layered (discontinuous) c^2, n=56 Kuhn mesh (1,053,696 tets), N=5, M=3, fp64 and
    fp32, Gaussian pulse state, 3 warm-up + 10 timed steps each, clocks sampled during the timed steps."""
    import torch

    from paper_1808_08645_b200 import Solver
    from workloads import kuhn, media

    n, N, M = 56, 5, 3
    v, e = kuhn.kuhn_mesh(n)
    c2 = media.project_c2(v, e, media.c2_layered(), M, device=dev)
    Np = comb(N + 3, 3)
    peaks, _ = load_peaks()
    Q0 = pulse_state(v, e, N, dev)
    out = {}
    for dt_name in ("f64", "f32"):
        s = Solver(v, e, N, M, c2, dtype=dt_name, device=dev.index, stream=torch.cuda.current_stream(dev))
        s.set_state(Q0 if dt_name == "f64" else Q0.float())
        h_min = 2.0 / n / (1 + np.sqrt(2) + np.sqrt(3))
        dt = 0.5 * h_min / (np.sqrt(2.25) * (N + 1) ** 2)
        for i in range(3):
            s.step(i * dt, dt)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(dev.index) as clk:
            torch.cuda.synchronize()
            a.record()
            for i in range(10):
                s.step((3 + i) * dt, dt)
            b.record()
            torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        info = s.info()
        gbs = info["algorithmic_bytes_per_stage"] / (ms / 5 / 1e3) / 1e9
        out[dt_name] = {"value": 4.0 * len(e) * Np * 5 / (ms / 1e3), "unit": UNIT, "ms_per_step": ms,
                        "hbm_frac": gbs / peaks["hbm_gbs"], "achieved_gbs": gbs, "warmup": 3, "steps": 10,
                        "clocks": clk.summary()}
        s.close()
    out["workload"] = (f"config4: Kuhn n={n} ({len(e):,} tets), N={N}, M={M}, layered c^2 1/1.5/2.25 (sub-cell "
                       f"jumps), Gaussian pulse")
    return out


def runs_2d(args, dev):
    """2D triangles: [-1,1]^2 cut into n x n x 2 triangles (n = 512: 524,288
    triangles; state 0.45 GB at N = 7, far above the L2), c^2 = 1 + 1/2 sin(pi x) sin(pi y) projected to P^M, Gaussian pulse; 3 warm-up + 10
    timed steps per line, clocks sampled; value = 3 K Np2 5 steps / device time."""
    import torch

    from paper_1808_08645_b200 import Solver2D
    from workloads import tri2d

    n = args.n2d
    v, e = tri2d.tri_mesh(n)
    peaks, _ = load_peaks()
    out = {"workload": f"2D: {n}x{n}x2 triangles ({len(e):,}), smooth c^2 (P:672), Gaussian pulse exp(-50|x|^2)"}
    c2c, qc = {}, {}
    for spec in args.two_d.split(","):
        N, M, dt_name = spec.split(":")
        N, M = int(N), int(M)
        Np = (N + 1) * (N + 2) // 2
        if M not in c2c:
            c2c[M] = tri2d.project_c2(v, e, tri2d.c2_smooth_2d(1.0), M)
        if N not in qc:
            qc[N] = tri2d.gaussian_pulse(v, e, N)
        c2, Q0 = c2c[M], qc[N]
        s = Solver2D(v, e, N, M, c2, dtype=dt_name, device=dev.index, stream=torch.cuda.current_stream(dev))
        s.set_state(Q0 if dt_name == "f64" else Q0.astype(np.float32))
        dt = 0.5 * tri2d.min_height(v, e) / (np.sqrt(c2.max()) * (N + 1) ** 2)
        for i in range(3):
            s.step(i * dt, dt)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(dev.index) as clk:
            torch.cuda.synchronize()
            a.record()
            for i in range(10):
                s.step((3 + i) * dt, dt)
            b.record()
            torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        info = s.info()
        gbs = info["algorithmic_bytes_per_stage"] / (ms / 5 / 1e3) / 1e9
        out[f"N{N}M{M}{dt_name}"] = {
            "value": 3.0 * len(e) * Np * 5 / (ms / 1e3), "unit": UNIT, "ms_per_step": ms,
            "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": round(gbs / peaks["hbm_gbs"], 4), "kernel": f"bbw::stage2d_kernel<N={N},M={M},{dt_name}>",
                         "algorithmic_bytes_per_launch": info["algorithmic_bytes_per_stage"],
                         "achieved_tflops": round(info["flops_per_stage"] / (ms / 5 / 1e3) / 1e12, 3)},
            "warmup": 3, "steps": 10, "gpu_launches": 50, "clocks": clk.summary()}
        s.close()
        del s
        torch.cuda.empty_cache()
    return out


def elastic_runs(args, dev):
    """Elastic BBWADG: n=56 Kuhn mesh (1,053,696 tets), smooth Lame fields
    (workloads.elastic.smooth_material) projected to P^M, Gaussian pressure pulse in the normal stresses;
    the paper's elastic runtime study uses M = 1, 2.  3 warm-up + 10 timed steps per line,
    clocks sampled during the timed steps; value = 9 K Np 5 steps / device time."""
    import torch

    from paper_1808_08645_b200 import ElasticSolver
    from workloads import elastic as ew
    from workloads import kuhn

    n = args.elastic_n
    v, e = kuhn.kuhn_mesh(n)
    peaks, _ = load_peaks()
    out = {"workload": f"elastic: Kuhn n={n} ({len(e):,} tets), smooth rho^-1/lambda/mu, pressure pulse in s11/s22/s33"}
    for spec in args.elastic.split(","):
        N, M, dt_name = spec.split(":")
        N, M = int(N), int(M)
        Np = comb(N + 3, 3)
        mats = ew.smooth_material(v, e, M, device=dev)
        from workloads._l2fit import l2_fit

        g = torch.from_numpy(l2_fit(v, e, lambda x, y, z, xp=np: xp.exp(-50.0 * (x * x + y * y + z * z)), N,
                                    device=dev)).to(dev)
        Q0 = torch.zeros((len(e), 9, Np), dtype=torch.float64, device=dev)
        Q0[:, 3:6] = -g[:, None, :]  # the pulse of workloads.elastic.gaussian_pulse, built on the device
        del g
        s = ElasticSolver(v, e, N, M, *mats, dtype=dt_name, device=dev.index, stream=torch.cuda.current_stream(dev))
        s.set_state(Q0 if dt_name == "f64" else Q0.float())
        del Q0
        h_min = 2.0 / n / (1 + np.sqrt(2) + np.sqrt(3))
        cp = np.sqrt((mats[1].max() + 2 * mats[2].max()) * mats[0].max())
        dt = 0.5 * h_min / (cp * (N + 1) ** 2)
        for i in range(3):
            s.step(i * dt, dt)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(dev.index) as clk:
            torch.cuda.synchronize()
            a.record()
            for i in range(10):
                s.step((3 + i) * dt, dt)
            b.record()
            torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        info = s.info()
        gbs = info["algorithmic_bytes_per_stage"] / (ms / 5 / 1e3) / 1e9
        out[f"N{N}M{M}{dt_name}"] = {
            "value": 9.0 * len(e) * Np * 5 / (ms / 1e3), "unit": UNIT, "ms_per_step": ms,
            "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": round(gbs / peaks["hbm_gbs"], 4), "kernel": f"bbw::elastic_stage_kernel<N={N},M={M},{dt_name}>",
                         "algorithmic_bytes_per_launch": info["algorithmic_bytes_per_stage"],
                         "achieved_tflops": round(info["flops_per_stage"] / (ms / 5 / 1e3) / 1e12, 3)},
            "warmup": 3, "steps": 10, "gpu_launches": 50, "clocks": clk.summary()}
        s.close()
        del s
        torch.cuda.empty_cache()
    return out


def _time_row(v, e, n, N, M, c2, dev, warmup, steps):
    """One acoustic (N, M) configuration on mesh (v, e): Gaussian pulse state, `warmup` + `steps` LSRK45
    steps, clocks sampled during the timed steps."""
    import torch

    from paper_1808_08645_b200 import Solver

    peaks, _ = load_peaks()
    Np = comb(N + 3, 3)
    s = Solver(v, e, N, M, c2, device=dev.index, stream=torch.cuda.current_stream(dev))
    s.set_state(pulse_state(v, e, N, dev))
    h_min = 2.0 / n / (1 + np.sqrt(2) + np.sqrt(3))
    dt = 0.5 * h_min / (np.sqrt(1.5) * (N + 1) ** 2)
    for i in range(warmup):
        s.step(i * dt, dt)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        torch.cuda.synchronize()
        a.record()
        for i in range(steps):
            s.step((warmup + i) * dt, dt)
        b.record()
        torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    info = s.info()
    gbs = info["algorithmic_bytes_per_stage"] / (ms / 5 / 1e3) / 1e9
    row = {"N": N, "M": M, "value": 4.0 * len(e) * Np * 5 / (ms / 1e3), "ms_per_step": ms,
           "ns_per_element_stage": ms * 1e6 / (5 * len(e)), "hbm_frac": gbs / peaks["hbm_gbs"],
           "tflops": info["flops_per_stage"] / (ms / 5 / 1e3) / 1e12,
           "flops_per_element_stage": info["flops_per_stage"] / len(e),
           "bytes_per_element_stage": info["algorithmic_bytes_per_stage"] / len(e),
           "warmup": warmup, "steps": steps, "clocks": clk.summary()}
    s.close()
    return row


def sweep(args, dev):
    """BASELINE config 3: N = 1..9, M = N on the n=44 Kuhn mesh (511,104 tets), fp64; plus the paper's
    fixed-M runtime study (BBWADG-1: M = 1, N = 1..9) and an M sweep at N = 7 (M = 0..7)
    on the same mesh and media (c^2 k = 8)."""
    from workloads import kuhn, media

    v, e = kuhn.kuhn_mesh(args.sweep_n)
    f = media.c2_smooth(8.0)
    c2cache = {}

    def c2_of(M):
        if M not in c2cache:
            c2cache[M] = media.project_c2(v, e, f, M, device=dev)
        return c2cache[M]

    def run(pairs):
        return [_time_row(v, e, args.sweep_n, N, M, c2_of(M), dev, args.sweep_warmup, args.sweep_steps) for N, M in pairs]

    def slope(rows, key):
        sel = [r for r in rows if r["N"] >= 4]
        Ns = np.log(np.array([r["N"] for r in sel], dtype=float))
        return float(np.polyfit(Ns, np.log(np.array([r[key] for r in sel], dtype=float)), 1)[0])

    rows = run([(N, N) for N in range(1, 10)])
    out = {"workload": f"config3: Kuhn n={args.sweep_n} ({len(e):,} tets), M=N, c^2 k=8, Gaussian pulse "
                       f"p = exp(-50|x|^2), u = 0, fp64; {args.sweep_warmup} warm-up + {args.sweep_steps} timed steps per N",
           "rows": rows, "loglog_slope_time_per_element_N4to9": slope(rows, "ns_per_element_stage"),
           "loglog_slope_algorithmic_flops_N4to9": slope(rows, "flops_per_element_stage"),
           "loglog_slope_algorithmic_bytes_N4to9": slope(rows, "bytes_per_element_stage"),
           "paper_prediction": "O(N^4) per element for the WADG update at fixed M (P:1693); bytes O(N^3)"}
    if not args.no_msweep:
        m1 = run([(N, 1) for N in range(1, 10)])
        out["fixed_M1"] = {"rows": m1, "loglog_slope_time_per_element_N4to9": slope(m1, "ns_per_element_stage"),
                           "loglog_slope_algorithmic_flops_N4to9": slope(m1, "flops_per_element_stage"),
                           "note": "M = 1 (the paper's BBWADG-1): the generic row-convolution product is the "
                                   "4-nonzero stencil of P:311-324 (3 row loads per output row)"}
        out["M_sweep_N7"] = {"rows": run([(7, M) for M in (0, 1, 2, 3, 4, 5, 7)]),
                             "note": "M = 0 takes the BBDG fast path (P:134: WADG = constant c^2)"}
    return out


def cpu_baseline(N, M, seconds, extras=False):
    """The CPU oracle as it stands, timed on this host on a bounded sample."""
    import threadpoolctl

    from oracle.acoustic import AcousticOracle
    from workloads import kuhn, media, states

    n = 4 if N >= 7 else 6
    v, e = kuhn.kuhn_mesh(n)
    c2 = media.project_c2(v, e, media.c2_smooth(1.0), M)
    Q = states.random_state(len(e), N)
    t0 = time.perf_counter()
    o = AcousticOracle(v, e, N, M, c2)
    setup = time.perf_counter() - t0
    res = np.zeros_like(Q)
    steps = 0
    t0 = time.perf_counter()
    while True:
        o.step(Q, res, 0.0, 1e-4)
        steps += 1
        el = time.perf_counter() - t0
        if el > seconds or steps >= 50:
            break
    Np = comb(N + 3, 3)
    info = threadpoolctl.threadpool_info()
    cores = max([i.get("num_threads", 1) for i in info] + [1])
    out = {"value": 4.0 * len(e) * Np * 5 * steps / el, "unit": UNIT, "cores": cores, "kind": "oracle",
           "sample": f"{steps} LSRK45 step(s) of the oracle on a {len(e)}-tet Kuhn mesh (n={n}), N={N}, M={M}, "
                     f"fp64 numpy/BLAS; table setup {setup:.1f}s excluded",
           "cpu": cpu_model(), "os_cpu_count": os.cpu_count()}
    if extras:
        out.update(cpu_extras())
    return out


def cpu_extras():
    """SURVEY 8(d) oracle timings: total seconds of config 1 (48 tets, N=3, M=1, 10 LSRK45 steps with the
    dt rule), and oracle DOF-stage/s on the 3072-tet mesh (n=8) at the (N, M) of configs 4 and 5 (one step
    each, measured, not extrapolated)."""
    from oracle.acoustic import AcousticOracle
    from workloads import kuhn, media, states

    v, e = kuhn.kuhn_mesh(2)
    c2 = media.project_c2(v, e, media.c2_smooth(1.0), 1)
    Q = states.random_state(len(e), 3)
    t0 = time.perf_counter()
    o = AcousticOracle(v, e, 3, 1, c2)
    h = kuhn.min_height(v, e)
    dt = 0.5 * h / (np.sqrt(1.5) * 16)
    res = np.zeros_like(Q)
    for i in range(10):
        o.step(Q, res, i * dt, dt)
    cfg1 = time.perf_counter() - t0
    rates = {}
    v, e = kuhn.kuhn_mesh(8)
    for N, M in ((5, 3), (7, 4)):
        c2 = media.project_c2(v, e, media.c2_smooth(1.0), M)
        Q = states.random_state(len(e), N)
        o = AcousticOracle(v, e, N, M, c2)
        res = np.zeros_like(Q)
        t0 = time.perf_counter()
        o.step(Q, res, 0.0, 1e-4)
        el = time.perf_counter() - t0
        rates[f"N{N}M{M}"] = 4.0 * len(e) * comb(N + 3, 3) * 5 / el
    return {"config1_total_seconds": cfg1, "oracle_dofstage_per_s_3072tets": rates}


def run_reference(args):
    """The reference arm of this tier: the CPU oracle (oracle/, as it stands) on the host cores, on a bounded
    sample of the same workload (same N, M, media and state recipe; a small Kuhn mesh), W untimed + K timed
    LSRK45 steps.  ms_per_step is the MEASURED time of one step of that sample (not extrapolated)."""
    import threadpoolctl

    from oracle.acoustic import AcousticOracle
    from workloads import kuhn, media, states

    rank, world, _ = dist_env()
    if rank != 0:
        return
    N, M = args.N, args.M
    n = 3 if N >= 7 else 4
    v, e = kuhn.kuhn_mesh(n)
    cf = {5: media.c2_smooth(1.0), 3: media.c2_smooth(8.0), 4: media.c2_layered()}.get(args.config, media.c2_smooth(1.0))
    c2 = media.project_c2(v, e, cf, M)
    Q = states.gaussian_pulse(v, e, N)
    t0 = time.perf_counter()
    o = AcousticOracle(v, e, N, M, c2)
    setup = time.perf_counter() - t0
    res = np.zeros_like(Q)
    dt = 0.5 * kuhn.min_height(v, e) / (np.sqrt(float(c2.max())) * (N + 1) ** 2)
    for i in range(args.warmup):
        o.step(Q, res, i * dt, dt)
    t0 = time.perf_counter()
    for i in range(args.steps):
        o.step(Q, res, (args.warmup + i) * dt, dt)
    el = time.perf_counter() - t0
    Np = comb(N + 3, 3)
    value = 4.0 * len(e) * Np * 5 * args.steps / el
    info = threadpoolctl.threadpool_info()
    cores = max([i.get("num_threads", 1) for i in info] + [1])
    sample = (f"{args.warmup} warm-up + {args.steps} timed LSRK45 steps of the CPU oracle on a {len(e)}-tet Kuhn "
              f"mesh (n={n}; the GPU arm runs {6 * args.n_cubes ** 3:,} tets per GPU), N={N}, M={M}, config-"
              f"{args.config} media, Gaussian pulse, fp64 numpy/BLAS; table setup {setup:.1f}s excluded")
    cb = {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample, "cpu": cpu_model(),
          "os_cpu_count": os.cpu_count()}
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": el * 1e3 / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"config{args.config} sample: {len(e)} tets (n={n}), N={N}, M={M}",
                      "N": N, "M": M, "K_total": len(e), "same_size_as_gpu_arm": False},
           "cpu_baseline": cb, "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                                       "d2h_bytes_per_step": 0}, "gpu_launches": 0}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--halo", choices=["auto", "nccl", "peer"], default="auto",
                    help="multi-GPU face-trace transport: peer reads of the owners' Q_in over CUDA IPC (halo_transport "
                         "1; exercised on hardware across processes), pack + NCCL send/recv, or auto = peer with a "
                         "fallback to NCCL when the peers cannot be mapped")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--N", type=int, default=None)
    ap.add_argument("--M", type=int, default=None)
    ap.add_argument("--n-cubes", type=int, default=None)
    ap.add_argument("--dtype", choices=["f64", "f32"], default="f64")
    ap.add_argument("--no-sweep", action="store_true", help="skip the config-3 N=1..9 sweep (rank 0, after the timed run)")
    ap.add_argument("--sweep-n", type=int, default=44)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-random", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--sweep-warmup", type=int, default=3)
    ap.add_argument("--sweep-steps", type=int, default=10)
    ap.add_argument("--no-config4", action="store_true", help="skip the config-4 fp64/fp32 extra lines")
    ap.add_argument("--elastic", default="7:2:f64,7:2:f32,5:1:f64,3:1:f64,9:2:f64",
                    help="elastic BBWADG lines N:M:dtype (comma separated; '' skips them)")
    ap.add_argument("--elastic-n", type=int, default=56)
    ap.add_argument("--two-d", default="7:4:f64,7:4:f32,3:1:f64,9:2:f64",
                    help="2D triangle lines N:M:dtype (comma separated; '' skips them)")
    ap.add_argument("--n2d", type=int, default=512)
    ap.add_argument("--no-msweep", action="store_true", help="skip the M=1 N-sweep and the N=7 M-sweep")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus != world and not (args.gpus == 1 and world == 1):
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch N>1 runs with "
                         f"python -m torch.distributed.run --nproc-per-node {args.gpus} bench.py --gpus {args.gpus}")
    defaults = {5: (7, 4, 88), 3: (7, 7, 44), 4: (5, 3, 56)}
    dN, dM, dn = defaults.get(args.config, (7, 4, 88))
    args.N = args.N if args.N is not None else dN
    args.M = args.M if args.M is not None else dM
    args.n_cubes = args.n_cubes if args.n_cubes is not None else dn
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
