"""Drop-in import path: `rasterbound.raster` -> paper_2010_12548_b200.raster."""
from paper_2010_12548_b200.raster import *  # noqa: F401,F403
from paper_2010_12548_b200 import raster as _impl

__all__ = getattr(_impl, "__all__", [])
