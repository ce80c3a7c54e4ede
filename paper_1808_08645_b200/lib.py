"""ctypes binding of libbbwadg.so -- argument marshalling only.

Every function here has the name and semantics of the C entry point declared in
include/bbwadg.h; all compute runs in the library's CUDA kernels.  There is no
CPU fallback: if the shared library is missing or fails to load, importing this
module raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BBWADG_LIB", os.path.join(HERE, "native", "libbbwadg.so"))

BBWADG_F64, BBWADG_F32 = 0, 1
STATUS = {0: "OK", 1: "INVALID_ARG", 2: "MESH", 3: "NONPOSITIVE_C2", 4: "UNSUPPORTED", 5: "CUDA", 6: "NCCL",
          7: "NONFINITE", 8: "OOM", 9: "NO_DEVICE"}


class bbwadg_mesh(ctypes.Structure):
    _fields_ = [("num_vertices", ctypes.c_int64), ("vertices", ctypes.c_void_p),
                ("num_elements", ctypes.c_int64), ("elements", ctypes.c_void_p)]


class bbwadg_mesh2d(ctypes.Structure):
    _fields_ = [("num_vertices", ctypes.c_int64), ("vertices", ctypes.c_void_p),
                ("num_elements", ctypes.c_int64), ("elements", ctypes.c_void_p)]


class bbwadg_options(ctypes.Structure):
    _fields_ = [("dtype", ctypes.c_int), ("tau_p", ctypes.c_double), ("tau_u", ctypes.c_double),
                ("device", ctypes.c_int), ("cuda_stream", ctypes.c_void_p), ("rank", ctypes.c_int),
                ("world_size", ctypes.c_int), ("nccl_unique_id", ctypes.c_void_p),
                ("partition", ctypes.c_int * 3), ("check_c2", ctypes.c_int), ("halo_transport", ctypes.c_int),
                ("c2_gids", ctypes.c_void_p), ("c2_rows", ctypes.c_int64), ("reserved", ctypes.c_int * 4)]


class bbwadg_info(ctypes.Structure):
    _fields_ = [("num_elements_global", ctypes.c_int64), ("num_elements_local", ctypes.c_int64),
                ("num_interior_local", ctypes.c_int64), ("num_halo_faces", ctypes.c_int64),
                ("N", ctypes.c_int), ("M", ctypes.c_int), ("Np", ctypes.c_int), ("Mp", ctypes.c_int),
                ("dtype", ctypes.c_int), ("rank", ctypes.c_int), ("world_size", ctypes.c_int),
                ("global_ids", ctypes.POINTER(ctypes.c_int64)),
                ("algorithmic_bytes_per_stage", ctypes.c_double), ("flops_per_stage", ctypes.c_double),
                ("kernels_per_stage", ctypes.c_int), ("steps_taken", ctypes.c_int64), ("time", ctypes.c_double)]


class BBWADGError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"bbwadg error {status} ({STATUS.get(status, '?')}): {msg}")
        self.status = status


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not found: build it with `python -m paper_1808_08645_b200.build` "
                          "(there is no CPU fallback)")
    try:  # make sure the CUDA runtime torch uses is mapped first (same libcudart.so.12)
        import torch  # noqa: F401
    except Exception:
        pass
    L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    P, I, D, V, S = ctypes.POINTER, ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_int
    ctx_p = V
    sig = {
        "bbwadg_default_options": (None, [P(bbwadg_options)]),
        "bbwadg_setup": (S, [P(bbwadg_mesh), I, I, V, P(bbwadg_options), P(ctx_p)]),
        "bbwadg_setup_group": (S, [P(bbwadg_mesh), I, I, V, P(bbwadg_options), I, V]),
        "bbwadg_elastic_setup": (S, [P(bbwadg_mesh), I, I, V, V, V, P(bbwadg_options), P(ctx_p)]),
        "bbwadg2d_setup": (S, [P(bbwadg_mesh2d), I, I, V, P(bbwadg_options), P(ctx_p)]),
        "bbwadg_set_state": (S, [ctx_p, V, I]),
        "bbwadg_get_state": (S, [ctx_p, V, I]),
        "bbwadg_set_source": (S, [ctx_p, V]),
        "bbwadg_rhs": (S, [ctx_p, V, D, V]),
        "bbwadg_wadg_apply": (S, [ctx_p, V, V]),
        "bbwadg_step": (S, [ctx_p, D, D]),
        "bbwadg_stage": (S, [ctx_p, I, D, D]),
        "bbwadg_ipc_get_handles": (S, [ctx_p, V]),
        "bbwadg_ipc_open_peer": (S, [ctx_p, I, V]),
        "bbwadg_group_step": (S, [V, I, D, D]),
        "bbwadg_run": (S, [ctx_p, D, D, ctypes.c_int64]),
        "bbwadg_synchronize": (S, [ctx_p]),
        "bbwadg_query": (S, [ctx_p, P(bbwadg_info)]),
        "bbwadg_error_string": (ctypes.c_char_p, [ctx_p]),
        "bbwadg_last_error": (ctypes.c_char_p, []),
        "bbwadg_destroy": (None, [ctx_p]),
        "bbwadg_projection_constants": (S, [I, I, V]),
        "bbwadg_mass_inverse_constants": (S, [I, V]),
        "bbwadg_nccl_unique_id": (S, [V]),
        "bbwadg_version": (ctypes.c_char_p, []),
        "bbwadg_partition_plan": (S, [P(bbwadg_mesh), I, V, I, V, V, V, V]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


_L = _load()
EXPORTED = [n for n in dir(_L) if n.startswith("bbwadg_")]


def _check(status: int, ctx=None):
    if status != 0:
        msg = (_L.bbwadg_error_string(ctx) if ctx else _L.bbwadg_last_error()) or b""
        raise BBWADGError(status, msg.decode(errors="replace"))


def _ptr(x):
    """Raw pointer of a numpy array or torch tensor (contiguity checked), or an int."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return x.data_ptr()
    if not x.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return x.ctypes.data


# ---- same-named thin wrappers --------------------------------------------------------------
def bbwadg_default_options() -> bbwadg_options:
    o = bbwadg_options()
    _L.bbwadg_default_options(ctypes.byref(o))
    return o


def bbwadg_setup(vertices, elements, N: int, M: int, c2, opts: bbwadg_options):
    m = bbwadg_mesh(vertices.shape[0], _ptr(vertices), elements.shape[0], _ptr(elements))
    ctx = ctypes.c_void_p()
    _check(_L.bbwadg_setup(ctypes.byref(m), N, M, _ptr(c2), ctypes.byref(opts), ctypes.byref(ctx)))
    return ctx


def bbwadg_elastic_setup(vertices, elements, N: int, M: int, rho_inv, lam, mu, opts: bbwadg_options):
    m = bbwadg_mesh(vertices.shape[0], _ptr(vertices), elements.shape[0], _ptr(elements))
    ctx = ctypes.c_void_p()
    _check(_L.bbwadg_elastic_setup(ctypes.byref(m), N, M, _ptr(rho_inv), _ptr(lam), _ptr(mu), ctypes.byref(opts),
                                   ctypes.byref(ctx)))
    return ctx


def bbwadg2d_setup(vertices, elements, N: int, M: int, c2, opts: bbwadg_options):
    m = bbwadg_mesh2d(vertices.shape[0], _ptr(vertices), elements.shape[0], _ptr(elements))
    ctx = ctypes.c_void_p()
    _check(_L.bbwadg2d_setup(ctypes.byref(m), N, M, _ptr(c2), ctypes.byref(opts), ctypes.byref(ctx)))
    return ctx


def bbwadg_setup_group(vertices, elements, N: int, M: int, c2, opts: bbwadg_options, nparts: int):
    m = bbwadg_mesh(vertices.shape[0], _ptr(vertices), elements.shape[0], _ptr(elements))
    arr = (ctypes.c_void_p * nparts)()
    _check(_L.bbwadg_setup_group(ctypes.byref(m), N, M, _ptr(c2), ctypes.byref(opts), nparts, arr))
    return [ctypes.c_void_p(a) for a in arr]


def bbwadg_set_state(ctx, Q, on_device: int):
    _check(_L.bbwadg_set_state(ctx, _ptr(Q), on_device), ctx)


def bbwadg_get_state(ctx, Q, on_device: int):
    _check(_L.bbwadg_get_state(ctx, _ptr(Q), on_device), ctx)


def bbwadg_set_source(ctx, g):
    _check(_L.bbwadg_set_source(ctx, _ptr(g)), ctx)


def bbwadg_rhs(ctx, Q_dev, t: float, dQdt_dev):
    _check(_L.bbwadg_rhs(ctx, _ptr(Q_dev), float(t), _ptr(dQdt_dev)), ctx)


def bbwadg_wadg_apply(ctx, r_dev, out_dev):
    _check(_L.bbwadg_wadg_apply(ctx, _ptr(r_dev), _ptr(out_dev)), ctx)


def bbwadg_step(ctx, t: float, dt: float):
    _check(_L.bbwadg_step(ctx, float(t), float(dt)), ctx)


def bbwadg_stage(ctx, s: int, t: float, dt: float):
    _check(_L.bbwadg_stage(ctx, s, t, dt), ctx)


def bbwadg_ipc_get_handles(ctx) -> bytes:
    buf = ctypes.create_string_buffer(192)
    _check(_L.bbwadg_ipc_get_handles(ctx, buf), ctx)
    return buf.raw


def bbwadg_ipc_open_peer(ctx, peer: int, handles: bytes):
    buf = ctypes.create_string_buffer(bytes(handles), 192)
    _check(_L.bbwadg_ipc_open_peer(ctx, peer, buf), ctx)


def bbwadg_group_step(ctxs, t: float, dt: float):
    arr = (ctypes.c_void_p * len(ctxs))(*[c.value for c in ctxs])
    _check(_L.bbwadg_group_step(arr, len(ctxs), float(t), float(dt)), ctxs[0])


def bbwadg_run(ctx, t0: float, dt: float, nsteps: int):
    _check(_L.bbwadg_run(ctx, float(t0), float(dt), int(nsteps)), ctx)


def bbwadg_synchronize(ctx):
    _check(_L.bbwadg_synchronize(ctx), ctx)


def bbwadg_query(ctx) -> bbwadg_info:
    info = bbwadg_info()
    _check(_L.bbwadg_query(ctx, ctypes.byref(info)), ctx)
    return info


def bbwadg_destroy(ctx):
    if ctx:
        _L.bbwadg_destroy(ctx)


def bbwadg_projection_constants(N: int, M: int):
    import numpy as np
    out = np.zeros(N + 1)
    _check(_L.bbwadg_projection_constants(N, M, _ptr(out)))
    return out


def bbwadg_mass_inverse_constants(N: int):
    import numpy as np
    out = np.zeros(N + 1)
    _check(_L.bbwadg_mass_inverse_constants(N, _ptr(out)))
    return out


def bbwadg_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_L.bbwadg_nccl_unique_id(buf))
    return buf.raw


def bbwadg_partition_plan(vertices, elements, nparts: int, rank: int, cuts=None):
    """Host-only partition plan (see include/bbwadg.h): returns dict with gid, send, recv arrays."""
    import numpy as np
    vertices = np.ascontiguousarray(vertices, dtype=np.float64)
    elements = np.ascontiguousarray(elements, dtype=np.int64)
    m = bbwadg_mesh(vertices.shape[0], _ptr(vertices), elements.shape[0], _ptr(elements))
    c = None if cuts is None else (ctypes.c_int * 3)(*cuts)
    sizes = np.zeros(4, dtype=np.int64)
    _check(_L.bbwadg_partition_plan(ctypes.byref(m), nparts, c, rank, _ptr(sizes), None, None, None))
    gid = np.zeros(sizes[0], dtype=np.int64)
    send = np.zeros((sizes[2], 4), dtype=np.int64)
    recv = np.zeros((sizes[3], 4), dtype=np.int64)
    _check(_L.bbwadg_partition_plan(ctypes.byref(m), nparts, c, rank, _ptr(sizes), _ptr(gid) if gid.size else None,
                                     _ptr(send) if send.size else None, _ptr(recv) if recv.size else None))
    return {"K_local": int(sizes[0]), "n_interior": int(sizes[1]), "gid": gid, "send": send, "recv": recv}


def bbwadg_version() -> str:
    return _L.bbwadg_version().decode()
