"""ctypes loader for the in-tree native libraries.

There is no fallback: if a library is missing or fails to load, every entry
point that needs it raises ``NativeLibraryError``.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

LIB_DIR = Path(__file__).resolve().parent / "_lib"


class NativeLibraryError(RuntimeError):
    """The native planner or executor library is missing or broken."""


_cache: dict[str, ctypes.CDLL] = {}


def load(name: str) -> ctypes.CDLL:
    lib = _cache.get(name)
    if lib is not None:
        return lib
    path = LIB_DIR / f"lib{name}.so"
    if not path.exists():
        raise NativeLibraryError(
            f"{path} is missing; run `python -m paper_1801_04380_b200._build` "
            "(or __graft_entry__.build())")
    try:
        lib = ctypes.CDLL(str(path), mode=ctypes.RTLD_GLOBAL)
    except OSError as exc:
        raise NativeLibraryError(f"cannot load {path}: {exc}") from exc
    _cache[name] = lib
    return lib


def planner() -> ctypes.CDLL:
    return load("snplan")


def executor() -> ctypes.CDLL:
    planner()
    return load("snexec")


def testing() -> ctypes.CDLL:
    """Test-only hooks and probes (libsntest.so); never used by the product path."""
    executor()
    return load("sntest")
