"""paper_2010_12548_b200 -- B200-native engine for epsilon-bounded
point-polygon aggregation (arXiv 2010.12548, "The Case for Distance-Bounded
Spatial Approximations"), behind the reference `rasterbound` Python API.

Modules mirror the reference package: errors, geometry, grid,
raster, act, query.  All bulk work runs in librasterbound_b200.so
(hand-written sm_100a CUDA behind the C-ABI in include/rasterbound_b200.h);
there is no CPU fallback.
"""
from . import errors  # noqa: F401
from .errors import *  # noqa: F401,F403

__version__ = "0.1.0"


def __getattr__(name):
    import importlib

    if name in ("geometry", "grid", "raster", "act", "query", "engine", "workloads", "_native", "pointindex", "canvas",
                "formats", "cli"):
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
