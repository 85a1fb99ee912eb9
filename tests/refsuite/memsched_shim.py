"""Test infrastructure: a ``memsched`` import alias for the drop-in package.

Installed as ``memsched/__init__.py`` in a scratch directory by
tests/test_reference_suite.py, so the reference's own test files
(/root/reference/pkg/tests, imported unchanged) exercise
``paper_1801_04380_b200`` through the reference's module paths.
"""

import importlib
import sys

_PKG = "paper_1801_04380_b200"
_SUBMODULES = ("cli", "convselect", "costmodel", "errors", "liveness", "netgen", "netgraph", "offload",
               "poolalloc", "recompute", "report", "simulator")

_root = importlib.import_module(_PKG)
sys.modules["memsched"] = _root
for _name in _SUBMODULES:
    sys.modules[f"memsched.{_name}"] = importlib.import_module(f"{_PKG}.{_name}")
