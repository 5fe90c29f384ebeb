"""Tree-level types of the reference (tree.py) that cross the engine boundary.

The node store itself lives in HBM as a structure-of-arrays pool (csrc/engine.cu);
these are the Python-side names and exception classes the reference exposes
(tree.py:42-100), so callers can switch without code changes.
"""

from __future__ import annotations

from dataclasses import dataclass

DEFAULT_DEPTH_CAP = 16  # tree.py:39


class TreeStructureError(Exception):
    """Raised when an operation would violate the tree shape (tree.py:42)."""


class NoExpandableLeafError(Exception):
    """Raised when selection finds no non-terminal leaf (tree.py:46)."""


class AccountingError(Exception):
    """Raised when visit or in-flight bookkeeping would go inconsistent (tree.py:50)."""


@dataclass(frozen=True)
class SelectionParams:
    """Exploration constant for WU-PUCT (tree.py:92-100)."""

    c_puct: float = 1.0

    def __post_init__(self) -> None:
        if self.c_puct <= 0.0:
            raise ValueError(f"c_puct must be positive, got {self.c_puct}")
