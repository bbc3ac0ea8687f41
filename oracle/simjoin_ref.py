"""Import the UNMODIFIED reference package (test / baseline infrastructure).

The reference ``simjoin`` is installed, unmodified, into ``baseline/_ref`` by

    python -m pip install --no-index --no-build-isolation --no-deps \\
        --find-links /opt/wheelhouse --target baseline/_ref <copy of /root/reference/pkg>

(``--no-deps``: the wheelhouse has no numpy wheel, numpy is already in the
image; the copy because the Cython build writes into its source tree).  Its
compiled backend (``simjoin._ckern``: _kernelcore.c, -O3 -march=native,
FMA) is the reference's fastest path.  ``baseline/_ref`` is git-ignored but
travels to the GPU box with the snapshot.

Stock ``import simjoin`` fails on Python >= 3.11: ``MatchSet`` declares
``field(default=<ndarray>)`` (core.py:112-114) and dataclasses rejects
unhashable defaults.  ``load()`` wraps ``dataclasses.field`` for the
duration of the import so an ndarray default becomes an equivalent
``default_factory`` -- no reference file is edited, and every function runs
as shipped.

Only tests/, bench.py's reference arm and its cpu_baseline leg use this
module; the product never imports it.
"""

from __future__ import annotations

import dataclasses
import os
import sys
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
REF_DIR = os.path.join(REPO, "baseline", "_ref")

_mod = None
_err: Optional[str] = None


def load(path: str = REF_DIR):
    """The reference's ``simjoin`` module, or None (see ``error()``)."""
    global _mod, _err
    if _mod is not None:
        return _mod
    if "simjoin" in sys.modules:
        _mod = sys.modules["simjoin"]
        return _mod
    if not os.path.isdir(os.path.join(path, "simjoin")):
        _err = f"reference not installed at {path}"
        return None
    orig = dataclasses.field

    def field(*a, **kw):
        d = kw.get("default", dataclasses.MISSING)
        if isinstance(d, np.ndarray):
            kw.pop("default")
            kw["default_factory"] = (lambda v=d: v)
        return orig(*a, **kw)

    dataclasses.field = field
    sys.path.insert(0, path)
    try:
        import simjoin  # noqa: F401
        _mod = sys.modules["simjoin"]
    except Exception as exc:  # noqa: BLE001  (an unusable install is reported, not fatal)
        _err = f"import simjoin failed: {type(exc).__name__}: {exc}"
        for k in [k for k in sys.modules if k == "simjoin" or k.startswith("simjoin.")]:
            del sys.modules[k]
        return None
    finally:
        dataclasses.field = orig
        if sys.path and sys.path[0] == path:
            sys.path.pop(0)
    return _mod


def error() -> Optional[str]:
    return _err


def compiled(mod=None) -> bool:
    """True when the reference runs its compiled backend (the fast path)."""
    mod = mod or load()
    return mod is not None and mod.kernels.active_backend() == "compiled"
