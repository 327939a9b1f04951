"""Drop-in import path: `rasterbound.canvas` -> paper_2010_12548_b200.canvas."""
from paper_2010_12548_b200.canvas import *  # noqa: F401,F403
from paper_2010_12548_b200 import canvas as _impl

__all__ = getattr(_impl, "__all__", [])
