"""Build recipe for ``oracle/_ref`` — TEST INFRASTRUCTURE ONLY.

The reference (/root/reference/pkg/src/btas) is pure Python, so its "build"
is byte-compilation: every module is compiled with ``py_compile`` from the
sources where they lie, and the sourceless bytecode (CPython 3.12 — the
interpreter of this image and of the GPU box) is packed as the package
``btas_ref`` into ``oracle/_ref/btas_ref.zip`` (zipimport loads sourceless
``.pyc`` entries; loose ``.pyc`` files do not survive the GPU-box snapshot).
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
OUT = HERE / "_ref" / "btas_ref.zip"
MODULES = ("__init__", "semiring", "matrix", "apsp", "graph_io", "bench", "cli", "__main__")


def build(force: bool = False) -> "Path | None":
    """Byte-compile the reference package into oracle/_ref/btas_ref.zip; a
    no-op (returns the existing build, or None) when /root/reference is
    absent."""
    import tempfile
    import zipfile

    if not (REF_PKG / "__init__.py").exists():
        return OUT if OUT.exists() else None
    srcs = [REF_PKG / f"{m}.py" for m in MODULES if (REF_PKG / f"{m}.py").exists()]
    if not force and OUT.exists() and all(OUT.stat().st_mtime >= p.stat().st_mtime for p in srcs):
        return OUT
    OUT.parent.mkdir(parents=True, exist_ok=True)
    tmp = OUT.with_suffix(".tmp")
    with tempfile.TemporaryDirectory() as td, zipfile.ZipFile(tmp, "w", zipfile.ZIP_STORED) as zf:
        for src in srcs:
            pyc = Path(td) / f"{src.stem}.pyc"
            py_compile.compile(str(src), cfile=str(pyc), doraise=True,
                               invalidation_mode=py_compile.PycInvalidationMode.UNCHECKED_HASH)
            zf.write(pyc, f"btas_ref/{src.stem}.pyc")
        zf.writestr("btas_ref/SOURCE", f"byte-compiled from {REF_PKG} by oracle/ref_build.py\n")
    tmp.replace(OUT)
    return OUT


def available() -> bool:
    return OUT.exists()


def load():
    """Import the compiled stock reference as ``btas_ref`` (the same alias
    oracle.ref_import gives the sources)."""
    if "btas_ref" in sys.modules:
        return sys.modules["btas_ref"]
    if not available():
        raise ImportError(f"the compiled reference is missing ({OUT}); run python -m oracle.ref_build")
    if str(OUT) not in sys.path:
        sys.path.insert(0, str(OUT))
    return importlib.import_module("btas_ref")


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
