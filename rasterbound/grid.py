"""Drop-in import path: `rasterbound.grid` -> paper_2010_12548_b200.grid."""
from paper_2010_12548_b200.grid import *  # noqa: F401,F403
from paper_2010_12548_b200 import grid as _impl

__all__ = getattr(_impl, "__all__", [])
