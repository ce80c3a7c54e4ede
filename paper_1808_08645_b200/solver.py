"""User-facing wrapper over the C ABI (PyTorch provides device memory and streams).

    from paper_1808_08645_b200 import Solver
    s = Solver(vertices, elements, N=7, M=4, c2=c2M)        # c2M: [K, Np(M)] float64
    s.set_state(Q0)                                        # numpy [K,4,Np] or CUDA tensor
    s.run(t0=0.0, dt=dt, nsteps=100)
    Q = s.get_state()                                      # numpy, global element order

    e = ElasticSolver(vertices, elements, N=5, M=1, rho_inv=ri, lam=la, mu=mu)  # [K, Np(M)] each
    e.set_state(Q9)                                        # [K,9,Np]: v1..3, s11 s22 s33 s23 s13 s12

No arithmetic of the method happens here: every call forwards to libbbwadg.so.
"""
from __future__ import annotations

from math import comb

import numpy as np

from . import lib as L


class Solver:
    NF = 4  # fields per element: p, u_x, u_y, u_z

    def __init__(self, vertices, elements, N: int, M: int, c2, *, dtype: str = "f64", tau_p: float = 1.0,
                 tau_u: float = 1.0, device: int = 0, stream=None, rank: int = 0, world_size: int = 1,
                 nccl_id: bytes | None = None, partition=None, check_c2: bool = True, c2_gids=None,
                 halo_transport: int = 0):
        import torch

        self.torch = torch
        self.N, self.M = int(N), int(M)
        self.Np, self.Mp = comb(N + 3, 3), comb(M + 3, 3)
        self.dtype = dtype
        self.tdtype = torch.float64 if dtype == "f64" else torch.float32
        self.device = torch.device("cuda", device)
        self._v = np.ascontiguousarray(vertices, dtype=np.float64)
        self._e = np.ascontiguousarray(elements, dtype=np.int64)
        c2 = np.ascontiguousarray(c2, dtype=np.float64)
        self._c2_gids = None
        if c2_gids is not None:  # rows for these global ids only (e.g. this rank's partition)
            self._c2_gids = np.ascontiguousarray(c2_gids, dtype=np.int64)
            if c2.shape != (self._c2_gids.shape[0], self.Mp):
                raise ValueError(f"c2 must have shape [len(c2_gids), {self.Mp}]")
        elif c2.shape != (self._e.shape[0], self.Mp):
            raise ValueError(f"c2 must have shape [K, {self.Mp}]")
        o = L.bbwadg_default_options()
        o.dtype = L.BBWADG_F64 if dtype == "f64" else L.BBWADG_F32
        o.tau_p, o.tau_u, o.device = float(tau_p), float(tau_u), int(device)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        o.cuda_stream = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        self.stream = stream
        o.rank, o.world_size = int(rank), int(world_size)
        self._nccl_id = None
        o.halo_transport = int(halo_transport)
        if world_size > 1 and halo_transport == 0:
            if nccl_id is None:
                raise ValueError("world_size > 1 needs the NCCL unique id (bbwadg_nccl_unique_id on rank 0)")
            import ctypes
            self._nccl_id = ctypes.create_string_buffer(bytes(nccl_id), 128)
            o.nccl_unique_id = ctypes.cast(self._nccl_id, ctypes.c_void_p)
        if partition is not None:
            for i in range(3):
                o.partition[i] = int(partition[i])
        o.check_c2 = 1 if check_c2 else 0
        if self._c2_gids is not None:
            o.c2_gids = self._c2_gids.ctypes.data
            o.c2_rows = int(self._c2_gids.shape[0])
        self.ctx = L.bbwadg_setup(self._v, self._e, self.N, self.M, c2, o)
        info = self.info()
        self.K_local = info["num_elements_local"]
        self.global_ids = info["global_ids"]

    # -------------------------------------------------------------------------------- state
    def _host_dtype(self):
        return np.float64 if self.dtype == "f64" else np.float32

    def set_state(self, Q):
        """Q: numpy [K_global,NF,Np] (global order) or a CUDA tensor [K_local,NF,Np] (local order)."""
        if isinstance(Q, np.ndarray):
            if Q.shape[0] != self.K_local:
                Q = Q[self.global_ids]
            Q = np.ascontiguousarray(Q, dtype=self._host_dtype())
            L.bbwadg_set_state(self.ctx, Q, 0)
        else:
            L.bbwadg_set_state(self.ctx, self._check_dev(Q, (self.K_local, self.NF, self.Np), "Q"), 1)

    def get_state(self, device: bool = False):
        if device:
            out = self.torch.empty((self.K_local, self.NF, self.Np), dtype=self.tdtype, device=self.device)
            L.bbwadg_get_state(self.ctx, out, 1)
            return out
        out = np.empty((self.K_local, self.NF, self.Np), dtype=self._host_dtype())
        L.bbwadg_get_state(self.ctx, out, 0)
        return out

    def set_source(self, g):
        L.bbwadg_set_source(self.ctx, None if g is None else np.ascontiguousarray(g, dtype=np.float64))

    def _check_dev(self, x, shape, what: str):
        """Device tensors go to the C side as raw pointers: validate before they do."""
        if not isinstance(x, self.torch.Tensor):
            raise TypeError(f"{what} must be a torch tensor on {self.device}")
        if x.device != self.device:
            raise ValueError(f"{what} is on {x.device}, the solver on {self.device}")
        if x.dtype != self.tdtype:
            raise TypeError(f"{what} has dtype {x.dtype}, the solver computes in {self.tdtype}")
        if tuple(x.shape) != shape:
            raise ValueError(f"{what} has shape {tuple(x.shape)}, expected {shape}")
        return x.contiguous()

    # -------------------------------------------------------------------------------- compute
    def rhs(self, Q_dev, t: float = 0.0):
        Q_dev = self._check_dev(Q_dev, (self.K_local, self.NF, self.Np), "Q")
        out = self.torch.empty(Q_dev.shape, dtype=self.tdtype, device=self.device)
        L.bbwadg_rhs(self.ctx, Q_dev, t, out)
        return out

    def wadg_apply(self, r_dev):
        shape = (self.K_local, self.NF, self.Np) if self.NF == 9 else (self.K_local, self.Np)
        r_dev = self._check_dev(r_dev, shape, "r")
        out = self.torch.empty(r_dev.shape, dtype=self.tdtype, device=self.device)
        L.bbwadg_wadg_apply(self.ctx, r_dev, out)
        return out

    def step(self, t: float, dt: float):
        L.bbwadg_step(self.ctx, t, dt)

    def ipc_handles(self) -> bytes:
        """CUDA IPC handles of this partition's state buffers and stage-epoch flag (halo_transport 1)."""
        return L.bbwadg_ipc_get_handles(self.ctx)

    def ipc_open_peers(self, handles):
        """Map every other rank's handles (list indexed by rank, e.g. from all_gather_object)."""
        info = self.info()
        for r, h in enumerate(handles):
            if r != info["rank"]:
                L.bbwadg_ipc_open_peer(self.ctx, r, h)

    def run(self, t0: float, dt: float, nsteps: int):
        L.bbwadg_run(self.ctx, t0, dt, nsteps)

    def synchronize(self):
        L.bbwadg_synchronize(self.ctx)

    def info(self) -> dict:
        i = L.bbwadg_query(self.ctx)
        d = {f: getattr(i, f) for f, _ in L.bbwadg_info._fields_ if f != "global_ids"}
        d["global_ids"] = np.ctypeslib.as_array(i.global_ids, shape=(i.num_elements_local,)).copy()
        return d

    def close(self):
        if getattr(self, "ctx", None):
            L.bbwadg_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ElasticSolver(Solver):
    """Elastic BBWADG (Eq. ewave / ewadg) through bbwadg_elastic_setup: state
    [K, 9, Np] = (v_1, v_2, v_3, s11, s22, s33, s23, s13, s12); material rho_inv, lam, mu [K, Np(M)];
    tau_s / tau_v the stress / velocity penalties.  Single GPU."""

    NF = 9

    def __init__(self, vertices, elements, N: int, M: int, rho_inv, lam, mu, *, dtype: str = "f64",
                 tau_v: float = 1.0, tau_s: float = 1.0, device: int = 0, stream=None, check: bool = True):
        import torch

        self.torch = torch
        self.N, self.M = int(N), int(M)
        self.Np, self.Mp = comb(N + 3, 3), comb(M + 3, 3)
        self.dtype = dtype
        self.tdtype = torch.float64 if dtype == "f64" else torch.float32
        self.device = torch.device("cuda", device)
        self._v = np.ascontiguousarray(vertices, dtype=np.float64)
        self._e = np.ascontiguousarray(elements, dtype=np.int64)
        mats = []
        for name, a in (("rho_inv", rho_inv), ("lam", lam), ("mu", mu)):
            a = np.ascontiguousarray(a, dtype=np.float64)
            if a.shape != (self._e.shape[0], self.Mp):
                raise ValueError(f"{name} must have shape [K, {self.Mp}]")
            mats.append(a)
        o = L.bbwadg_default_options()
        o.dtype = L.BBWADG_F64 if dtype == "f64" else L.BBWADG_F32
        o.tau_p, o.tau_u, o.device = float(tau_s), float(tau_v), int(device)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        o.cuda_stream = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        self.stream = stream
        o.check_c2 = 1 if check else 0
        self.ctx = L.bbwadg_elastic_setup(self._v, self._e, self.N, self.M, *mats, o)
        info = self.info()
        self.K_local = info["num_elements_local"]
        self.global_ids = info["global_ids"]


class Solver2D(Solver):
    """2D (triangle) acoustic BBWADG through bbwadg2d_setup: vertices [nv, 2],
    triangles [K, 3] counter-clockwise, c2 [K, Np2(M)], state [K, 3, Np2] = (p, u_x, u_y).  Single GPU."""

    NF = 3

    def __init__(self, vertices, elements, N: int, M: int, c2, *, dtype: str = "f64", tau_p: float = 1.0,
                 tau_u: float = 1.0, device: int = 0, stream=None, check_c2: bool = True):
        import torch

        self.torch = torch
        self.N, self.M = int(N), int(M)
        self.Np, self.Mp = (N + 1) * (N + 2) // 2, (M + 1) * (M + 2) // 2
        self.dtype = dtype
        self.tdtype = torch.float64 if dtype == "f64" else torch.float32
        self.device = torch.device("cuda", device)
        self._v = np.ascontiguousarray(vertices, dtype=np.float64)
        self._e = np.ascontiguousarray(elements, dtype=np.int64)
        c2 = np.ascontiguousarray(c2, dtype=np.float64)
        if self._v.ndim != 2 or self._v.shape[1] != 2 or self._e.ndim != 2 or self._e.shape[1] != 3:
            raise ValueError("2D mesh: vertices [nv, 2], triangles [K, 3]")
        if c2.shape != (self._e.shape[0], self.Mp):
            raise ValueError(f"c2 must have shape [K, {self.Mp}]")
        o = L.bbwadg_default_options()
        o.dtype = L.BBWADG_F64 if dtype == "f64" else L.BBWADG_F32
        o.tau_p, o.tau_u, o.device = float(tau_p), float(tau_u), int(device)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        o.cuda_stream = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        self.stream = stream
        o.check_c2 = 1 if check_c2 else 0
        self.ctx = L.bbwadg2d_setup(self._v, self._e, self.N, self.M, c2, o)
        info = self.info()
        self.K_local = info["num_elements_local"]
        self.global_ids = info["global_ids"]
