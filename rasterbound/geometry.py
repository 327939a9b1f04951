"""Drop-in import path: `rasterbound.geometry` -> paper_2010_12548_b200.geometry."""
from paper_2010_12548_b200.geometry import *  # noqa: F401,F403
from paper_2010_12548_b200 import geometry as _impl

__all__ = getattr(_impl, "__all__", [])
