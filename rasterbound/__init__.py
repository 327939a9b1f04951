"""Drop-in `rasterbound` package name (reference pyproject.toml:6) backed by
the B200-native implementation in paper_2010_12548_b200."""
__version__ = "0.1.0"
