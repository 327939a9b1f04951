"""Drop-in import path: `rasterbound.query` -> paper_2010_12548_b200.query."""
from paper_2010_12548_b200.query import *  # noqa: F401,F403
from paper_2010_12548_b200 import query as _impl

__all__ = getattr(_impl, "__all__", [])
