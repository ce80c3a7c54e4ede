"""B200-native BBWADG hot path (Guo & Chan, arXiv 1808.08645).

The product is ``native/libbbwadg.so`` (C ABI in ``include/bbwadg.h``): fused sm_100a
CUDA kernels for the per-element, per-RK-stage BBWADG right-hand side and the
LSRK45 update, host C++ for mesh connectivity / partitioning / operator tables,
and an NCCL face-trace halo for element-partitioned multi-GPU runs.

``lib`` holds same-named ctypes wrappers of every C entry point; ``Solver`` is a
convenience class.  Both are loaded on first access (so that ``build`` can run
before the library exists); accessing them raises ImportError if the shared
library is missing: there is no CPU fallback (the CPU oracle in ``oracle/`` is
test infrastructure and is never imported from here).
"""
import importlib

__all__ = ["lib", "Solver", "ElasticSolver", "Solver2D", "build"]


def __getattr__(name):
    if name == "lib":
        return importlib.import_module(".lib", __name__)
    if name == "Solver":
        return importlib.import_module(".solver", __name__).Solver
    if name == "Solver2D":
        return importlib.import_module(".solver", __name__).Solver2D
    if name == "ElasticSolver":
        return importlib.import_module(".solver", __name__).ElasticSolver
    if name == "build":
        return importlib.import_module(".build", __name__)
    raise AttributeError(name)
