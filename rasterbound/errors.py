"""Drop-in import path: `rasterbound.errors` -> paper_2010_12548_b200.errors."""
from paper_2010_12548_b200.errors import *  # noqa: F401,F403
from paper_2010_12548_b200 import errors as _impl

__all__ = getattr(_impl, "__all__", [])
