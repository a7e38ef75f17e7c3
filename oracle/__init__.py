"""CPU oracle (test infrastructure only — see linop_oracle.py)."""

from . import linop_oracle  # noqa: F401
