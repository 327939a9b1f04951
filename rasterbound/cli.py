"""Drop-in entry point `rasterbound.cli:main` (reference pyproject.toml:23-24)."""
from paper_2010_12548_b200.cli import main  # noqa: F401

if __name__ == "__main__":
    main()
