"""Drop-in import path: `rasterbound.pointindex` -> paper_2010_12548_b200.pointindex."""
from paper_2010_12548_b200.pointindex import *  # noqa: F401,F403
from paper_2010_12548_b200 import pointindex as _impl

__all__ = getattr(_impl, "__all__", [])
