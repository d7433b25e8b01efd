"""The reference package `hekan`, which this engine plugs into.

The engine is a drop-in backend for the reference's `HeBackend` contract
(/root/reference/pkg/src/hekan/backend.py:132-270), so everything on the
reference side of that boundary — the model types, the planner types, the
plaintext forwards, the fitters, the exception taxonomy — is imported from the
reference itself rather than restated. Only the engine's program deltas
(hoisted/grouped BSGS, Chebyshev evaluators, fused combines) live in this
package.

`hekan` is found, in order: already importable; $HEKAN_PATH; the offline
install under <repo>/baseline/_ref (made by __graft_entry__.build(), which
installs /root/reference/pkg there with pip --no-index --no-deps). The install
is git-ignored but ships with the tree to the GPU box.
"""

from __future__ import annotations

import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INSTALL_DIR = os.path.join(ROOT, "baseline", "_ref")


def _candidates():
    env = os.environ.get("HEKAN_PATH")
    if env:
        yield env
    yield INSTALL_DIR


def load():
    try:
        return importlib.import_module("hekan")
    except ImportError:
        pass
    for path in _candidates():
        if os.path.isfile(os.path.join(path, "hekan", "__init__.py")):
            if path not in sys.path:
                sys.path.append(path)
            return importlib.import_module("hekan")
    raise ImportError(
        "the reference package `hekan` is not importable: run "
        "`python -c 'import __graft_entry__ as g; g.build()'` (installs it into "
        f"{INSTALL_DIR}) or set HEKAN_PATH")


hekan = load()
