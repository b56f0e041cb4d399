"""Build recipe for ``oracle/_ref`` — TEST INFRASTRUCTURE ONLY.

The reference (/root/reference/pkg/src/btas) is pure Python, so its "build"
is byte-compilation: every module is compiled with ``py_compile`` from the
sources where they lie into ``oracle/_ref/btas/<module>.pyc`` (sourceless
bytecode, CPython 3.12 — the interpreter of this image and of the GPU box).
``oracle/_ref`` is git-ignored (no reference source enters the history) but
not gpurun-ignored, so the compiled reference travels to the GPU box, where
/root/reference does not exist.  There it is the stock reference for
``bench.py --impl reference`` and for bench's cpu_baseline / parity legs:
the unmodified ``btas.matmul`` / ``btas.apsp_by_squaring`` code path.

    python -m oracle.ref_build          # or __graft_entry__.build()
"""

from __future__ import annotations

import importlib.util
import py_compile
import sys
from pathlib import Path

from .ref_import import REF_PKG

HERE = Path(__file__).resolve().parent
OUT = HERE / "_ref" / "btas"
MODULES = ("__init__", "semiring", "matrix", "apsp", "graph_io", "bench", "cli", "__main__")


def build(force: bool = False) -> "Path | None":
    """Byte-compile the reference package into oracle/_ref/btas; a no-op
    (returns the existing build, or None) when /root/reference is absent."""
    if not (REF_PKG / "__init__.py").exists():
        return OUT if (OUT / "__init__.pyc").exists() else None
    OUT.mkdir(parents=True, exist_ok=True)
    for name in MODULES:
        src = REF_PKG / f"{name}.py"
        dst = OUT / f"{name}.pyc"
        if not src.exists():
            continue
        if force or not dst.exists() or dst.stat().st_mtime < src.stat().st_mtime:
            py_compile.compile(str(src), cfile=str(dst), doraise=True,
                               invalidation_mode=py_compile.PycInvalidationMode.UNCHECKED_HASH)
    (OUT / "SOURCE").write_text(f"byte-compiled from {REF_PKG} by oracle/ref_build.py\n")
    return OUT


def available() -> bool:
    return (OUT / "__init__.pyc").exists()


def load():
    """Import the compiled stock reference as ``btas_ref`` (same alias as
    oracle.ref_import, which prefers the sources when they are present)."""
    if "btas_ref" in sys.modules:
        return sys.modules["btas_ref"]
    if not available():
        raise ImportError(f"the compiled reference is missing under {OUT}; run python -m oracle.ref_build")
    spec = importlib.util.spec_from_file_location("btas_ref", OUT / "__init__.pyc",
                                                  submodule_search_locations=[str(OUT)])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["btas_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
