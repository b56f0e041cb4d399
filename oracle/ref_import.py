"""Import the REAL reference package from /root/reference (this container
only — /root/reference does not exist on the GPU box) — TEST INFRASTRUCTURE.

The reference package is also named ``btas`` and uses relative imports, so it
is loaded under the alias ``btas_ref`` with an explicit spec.  Used to pin
the oracle and to generate tests/golden fixtures; never at GPU run time.
"""

from __future__ import annotations

import importlib.util
import os
import sys
from pathlib import Path

REF_ROOT = Path(os.environ.get("BTAS_REFERENCE_ROOT", "/root/reference"))
REF_PKG = REF_ROOT / "pkg" / "src" / "btas"


def available() -> bool:
    return (REF_PKG / "__init__.py").exists()


def load_reference():
    """Return the reference ``btas`` package imported as ``btas_ref``."""
    if "btas_ref" in sys.modules:
        return sys.modules["btas_ref"]
    if not available():
        raise ImportError(f"reference package not found under {REF_PKG}")
    spec = importlib.util.spec_from_file_location(
        "btas_ref", REF_PKG / "__init__.py", submodule_search_locations=[str(REF_PKG)]
    )
    mod = importlib.util.module_from_spec(spec)
    sys.modules["btas_ref"] = mod
    spec.loader.exec_module(mod)
    return mod
