"""Drop-in import path: `rasterbound.act` -> paper_2010_12548_b200.act."""
from paper_2010_12548_b200.act import *  # noqa: F401,F403
from paper_2010_12548_b200 import act as _impl

__all__ = getattr(_impl, "__all__", [])
