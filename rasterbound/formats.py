"""`rasterbound.formats` -> paper_2010_12548_b200.formats (ingest / file formats)."""
from paper_2010_12548_b200.formats import *  # noqa: F401,F403
from paper_2010_12548_b200 import formats as _impl

__all__ = getattr(_impl, "__all__", [])
