"""pytest plugin: run the reference's own test suite against the drop-in.

Loaded with ``-p refalias`` by tests/test_gpu_reference_suite.py. It makes the
package name ``trackforge`` resolve to this repository's modules for every
hot-path module (errors, core, postproc, motion, assoc, tracker, moteval),
so ``from trackforge.tracker import Tracker`` in the reference's tests gets
the GPU tracker. The reference's own modules outside the hot path (the
synthetic source ``detgen``, the thread pipeline ``pipeline`` and the CLI) are
loaded unmodified from the pip-installed reference (baseline/_ref); their
relative imports (``from .tracker import Tracker``) resolve to the drop-in
too, so the pipeline and CLI tests drive the GPU path through the
reference's own call sites (tf/pipeline.py:291-302).
"""

from __future__ import annotations

import importlib
import os
import sys
import types
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF = Path(os.environ.get("TF_REFERENCE_PKG", ROOT / "baseline" / "_ref" / "trackforge"))
OURS = ("errors", "core", "postproc", "motion", "assoc", "tracker", "moteval")
THEIRS = ("detgen", "pipeline", "cli")


def _install() -> None:
    if str(ROOT) not in sys.path:
        sys.path.insert(0, str(ROOT))
    pkg = types.ModuleType("trackforge")
    pkg.__path__ = [str(REF)]
    pkg.__file__ = str(REF / "__init__.py")
    pkg.__package__ = "trackforge"
    sys.modules["trackforge"] = pkg
    for name in OURS:
        mod = importlib.import_module(f"paper_2011_03910_b200.{name}")
        sys.modules[f"trackforge.{name}"] = mod
        setattr(pkg, name, mod)
    for name in THEIRS:
        setattr(pkg, name, importlib.import_module(f"trackforge.{name}"))
    # package-level names, as tf/__init__.py:1-42 exports them
    for mod in [getattr(pkg, n) for n in OURS + THEIRS]:
        for attr in getattr(mod, "__all__", None) or [a for a in dir(mod) if not a.startswith("_")]:
            if not hasattr(pkg, attr):
                setattr(pkg, attr, getattr(mod, attr))
    pkg.__version__ = "0.1.0"


_install()
