"""Import the live reference package (container only) -- TEST INFRASTRUCTURE ONLY.

``/root/reference`` exists only in the build container, never on the GPU box.
``load()`` imports ``pagetopk`` straight from the read-only tree and, when
``oracle/_ref`` holds the reference's own compiled backend (built by
``make -C oracle ref`` from ``pkg/src/pagetopk/_kernels_cy.pyx``), registers it
as ``pagetopk._kernels_cy`` so ``set_backend("cython")`` selects the shipped
compiled kernels exactly as an installed reference would.
"""

from __future__ import annotations

import glob
import importlib.util
import os
import sys

REF_SRC = "/root/reference/pkg/src"
_HERE = os.path.dirname(os.path.abspath(__file__))


def available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "pagetopk"))


def load(backend: str = "cython"):
    """Return the reference ``pagetopk`` module with ``backend`` active."""
    if not available():
        raise ImportError("reference tree not present (/root/reference)")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import pagetopk  # noqa: E402

    if "pagetopk._kernels_cy" not in sys.modules:
        so = glob.glob(os.path.join(_HERE, "_ref", "_kernels_cy*.so"))
        if so:
            spec = importlib.util.spec_from_file_location("pagetopk._kernels_cy", so[0])
            mod = importlib.util.module_from_spec(spec)
            spec.loader.exec_module(mod)
            sys.modules["pagetopk._kernels_cy"] = mod
            pagetopk._kernels_cy = mod
    from pagetopk import backend as _b

    _b.set_backend(backend)
    return pagetopk
