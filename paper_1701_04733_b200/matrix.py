"""Dense tropical matrices and vectors resident in B200 HBM.

Drop-in for the reference ``btas.matrix`` (/root/reference/pkg/src/btas/
matrix.py).  Same names, argument meaning and exceptions; the storage is a
CUDA tensor instead of a NumPy array and every operation is one or a few
launches of the sm_100a kernels in libbtas_cuda.so (include/btas_cuda.h).

Storage ("oriented" form, as in the reference matrix.py:3-7):
  * float64 (default, the reference's own dtype — bit-identical results),
    float32 (every result is the reference's float64 result rounded once to
    float32), or int32 (exact while |x| < 2^28);
  * Infinity is stored as +inf under min-plus and -inf under max-plus;
    int32 encodes it as +/-(2^30 - 1).
``.data`` is the device tensor; ``.to_numpy()`` / ``.tobytes()`` give the
reference's float64 oriented array / bytes.

Determinism contract (reference matrix.py:9-13): the k dimension is never
split across CTAs, entries carry no NaN and no -0.0, and min/max is exact, so
results are bit-identical for every TileSpec, tile configuration and GPU
count.  TileSpec is accepted and validated for API compatibility; the CUDA
tile shape is a compile-time property of the kernels.
"""

from __future__ import annotations

import ctypes
import math
import os
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .semiring import SemiringKind, TropicalWeight, _register_device_flags

I32_LIMIT = _lib.I32_LIMIT  # int32 storage: finite |x| < 2^28


class DimensionMismatch(ValueError):
    """Operand shapes do not line up."""


class SemiringMismatch(ValueError):
    """Operands carry different SemiringKinds."""


class DtypeMismatch(ValueError):
    """Operands are stored with different element types."""


def available_parallelism() -> int:
    """CPUs this process may use (reference matrix.py:42-47)."""
    try:
        return len(os.sched_getaffinity(0)) or 1
    except (AttributeError, OSError):
        return os.cpu_count() or 1


@dataclass(frozen=True, slots=True)
class TileSpec:
    """Output-tile partition hint (reference matrix.py:50-71).

    Validated exactly like the reference; the GPU kernels use their own
    compile-time CTA tiles, and results are byte-identical for any TileSpec.
    """

    tile_rows: int
    tile_cols: int
    worker_count: int

    def __post_init__(self) -> None:
        for field in ("tile_rows", "tile_cols", "worker_count"):
            v = getattr(self, field)
            if not isinstance(v, int) or v < 1:
                raise ValueError(f"{field} must be a positive integer, got {v!r}")

    @classmethod
    def default(cls) -> "TileSpec":
        return cls(tile_rows=8, tile_cols=8, worker_count=available_parallelism())


# ---------------------------------------------------------------------------
# dtype / device plumbing
# ---------------------------------------------------------------------------
_DTYPE_CODES = {torch.float32: _lib.F32, torch.int32: _lib.I32, torch.float64: _lib.F64}
_default_dtype = torch.float64


def set_default_dtype(dtype: torch.dtype) -> None:
    """Storage dtype for matrices built without an explicit ``dtype``."""
    global _default_dtype
    if dtype not in _DTYPE_CODES:
        raise ValueError(f"unsupported storage dtype {dtype}; use float64, float32 or int32")
    _default_dtype = dtype


def get_default_dtype() -> torch.dtype:
    return _default_dtype


def _dtype_code(dtype: torch.dtype) -> int:
    try:
        return _DTYPE_CODES[dtype]
    except KeyError:
        raise ValueError(f"unsupported storage dtype {dtype}; use float64, float32 or int32") from None


def _kind_code(kind: SemiringKind) -> int:
    return _lib.MIN_PLUS if kind is SemiringKind.MIN_PLUS else _lib.MAX_PLUS


def _resolve_device(device) -> torch.device:
    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1701_04733_b200 needs a CUDA device (B200); there is no CPU fallback")
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise ValueError(f"tropical matrices live on a CUDA device, got {dev}")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def _on_operand_device(fn):
    """Run ``fn`` with the CUDA device of its first matrix/vector/tensor
    argument current, so its kernels launch on the operands' device even when
    one process drives several GPUs (one process per GPU needs nothing)."""
    import functools

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        for a in args:
            t = a.data if hasattr(a, "data") and isinstance(getattr(a, "data"), torch.Tensor) else a
            if isinstance(t, torch.Tensor) and t.is_cuda:
                if t.device.index == torch.cuda.current_device():
                    return fn(*args, **kwargs)
                with torch.cuda.device(t.device):
                    return fn(*args, **kwargs)
        return fn(*args, **kwargs)

    return wrapper


def _device_ctx(device: torch.device):
    """Context making ``device`` current for the kernels a call launches."""
    import contextlib

    if device.type != "cuda" or device.index == torch.cuda.current_device():
        return contextlib.nullcontext()
    return torch.cuda.device(device)


def _stream(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


class _Workspace:
    """Growable scratch buffer for the C-ABI calls, one per (device, stream):
    calls on different streams may run concurrently, calls on one stream are
    ordered, so a per-stream buffer is never shared by two running kernels.
    A replaced buffer goes back to the caching allocator, which only reuses it
    on the same stream (stream-ordered)."""

    def __init__(self):
        self._bufs: "dict[tuple[int, int], torch.Tensor]" = {}
        self._lock = threading.Lock()

    def get(self, device: torch.device, nbytes: int) -> torch.Tensor:
        key = (device.index, torch.cuda.current_stream(device).cuda_stream)
        with self._lock:
            buf = self._bufs.get(key)
            if buf is None or buf.numel() < nbytes:
                buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
                self._bufs[key] = buf
            return buf


_workspace = _Workspace()


class _FlagLedger:
    """Set-only device flag words (dev_flags of the C ABI), read lazily.

    Every kernel call gets a fresh int32[NUM_FLAGS] buffer; the ones whose
    saturation bit has not been read yet are kept here, each with the CUDA
    stream that was current when the kernel writing it was launched, so that
    ``saturation_seen()`` can fold them in with a single synchronising read.
    Reads and folds run on the reader's current stream after making it wait
    for every producing stream (a flag written by a kernel on another stream
    or thread is never read before that kernel ran), and the folded buffers
    are marked used on the reader's stream for the caching allocator.
    """

    def __init__(self):
        self._pending: "list[tuple[torch.Tensor, torch.cuda.Stream]]" = []
        self._lock = threading.Lock()

    def new(self, device: torch.device) -> torch.Tensor:
        return torch.zeros(_lib.NUM_FLAGS, dtype=torch.int32, device=device)

    def track(self, flags: torch.Tensor) -> None:
        """Call right after launching the kernel(s) that write ``flags``, on
        the stream they were launched on (the current one)."""
        entry = (flags, torch.cuda.current_stream(flags.device))
        with self._lock:
            self._pending.append(entry)
            if len(self._pending) > 256:
                self._fold_locked()

    @staticmethod
    def _by_device(pending):
        by_dev: "dict[torch.device, list]" = {}
        for f, s in pending:
            by_dev.setdefault(f.device, []).append((f, s))
        return by_dev

    @staticmethod
    def _gather_sat(dev, entries) -> torch.Tensor:
        """max of the saturation words of ``entries`` on ``dev``'s current
        stream, ordered after every producing stream."""
        cur = torch.cuda.current_stream(dev)
        waited = set()
        for f, s in entries:
            if s.cuda_stream != cur.cuda_stream:
                if s.cuda_stream not in waited:
                    cur.wait_stream(s)
                    waited.add(s.cuda_stream)
                f.record_stream(cur)
        return torch.stack([f[_lib.FLAG_SATURATED] for f, _ in entries]).amax()

    def _fold_locked(self) -> None:
        folded = []
        for dev, entries in self._by_device(self._pending).items():
            with torch.cuda.device(dev):
                sat = self._gather_sat(dev, entries)
                out = torch.zeros(_lib.NUM_FLAGS, dtype=torch.int32, device=dev)
                out[_lib.FLAG_SATURATED] = sat
                folded.append((out, torch.cuda.current_stream(dev)))
        self._pending = folded

    def read_saturation(self) -> bool:
        with self._lock:
            pending, self._pending = self._pending, []
        seen = False
        for dev, entries in self._by_device(pending).items():
            with torch.cuda.device(dev):
                sat = self._gather_sat(dev, entries).reshape(1)
                seen |= int(_host_read(sat)[0]) != 0
        return seen

    def reset(self) -> None:
        with self._lock:
            self._pending = []


_flags = _FlagLedger()
_register_device_flags(_flags.read_saturation, _flags.reset)


class _HostReader:
    """Small device results (stats, flag words, counts) read through a
    page-locked host buffer written by SM stores (btas_export_words), not by a
    device-to-host copy: a copy would queue on the copy engine behind any bulk
    download another stream has in flight (a pipelined caller's result
    transfer), stalling every validation read for its duration."""

    _CAP = 16384

    def __init__(self):
        self._tls = threading.local()

    def read(self, t: torch.Tensor) -> np.ndarray:
        t = t.detach().contiguous()
        nbytes = t.numel() * t.element_size()
        np_dtype = torch.empty(0, dtype=t.dtype).numpy().dtype
        if nbytes == 0:
            return np.zeros(t.shape, dtype=np_dtype)
        if nbytes % 4 or nbytes > self._CAP or t.device.type != "cuda":
            return t.cpu().numpy()
        buf = getattr(self._tls, "buf", None)
        if buf is None:
            buf = torch.empty(self._CAP, dtype=torch.uint8, pin_memory=True)
            self._tls.buf = buf
        stream = torch.cuda.current_stream(t.device)
        _lib.call("btas_export_words", t.data_ptr(), buf.data_ptr(), nbytes // 4, stream.cuda_stream)
        done = torch.cuda.Event()
        done.record(stream)
        done.synchronize()
        return buf[:nbytes].numpy().view(np_dtype).reshape(t.shape).copy()


_host = _HostReader()


def _host_read(t: torch.Tensor) -> np.ndarray:
    """Synchronously read a small device tensor (see _HostReader)."""
    return _host.read(t)


def _read_stats(stats: torch.Tensor) -> _lib.Stats:
    host = _host_read(stats).view(np.uint64)
    s = _lib.Stats()
    for i, (name, _) in enumerate(_lib.Stats._fields_):
        setattr(s, name, int(host[i]))
    return s


def _new_stats(device: torch.device) -> torch.Tensor:
    st = torch.empty(_lib.STATS_WORDS, dtype=torch.int64, device=device)
    _lib.call("btas_stats_init", _ptr(st), _stream(device))
    return st


def _ingest(kind: SemiringKind, values, dtype: torch.dtype, device: torch.device, ndim: int):
    with _device_ctx(device):
        return _ingest_on_device(kind, values, dtype, device, ndim)


def _ingest_on_device(kind: SemiringKind, values, dtype: torch.dtype, device: torch.device, ndim: int):
    """Validate symbolic-form input and produce oriented device storage.

    Mirrors _orient/_detect_integer (reference matrix.py:82-115) on the GPU:
    NaN and -inf are rejected, -0.0 normalised, Infinity oriented per kind.
    Returns (tensor, stats).
    """
    if isinstance(values, torch.Tensor):
        src = values.detach()
        if src.dtype not in (torch.float32, torch.float64):
            src = src.to(torch.float64)
        src = src.to(device).contiguous()
    else:
        try:
            arr = np.asarray(values, dtype=np.float64)
        except (TypeError, ValueError) as exc:
            raise DimensionMismatch(f"entries do not form a rectangular array: {exc}") from None
        src = torch.from_numpy(np.ascontiguousarray(arr)).to(device)
    if src.dim() != ndim:
        what = "matrix needs 2 dimensions" if ndim == 2 else "vector needs 1 dimension"
        raise DimensionMismatch(f"{what}, got {src.dim()}")
    if ndim == 2 and (src.shape[0] < 1 or src.shape[1] < 1):
        raise DimensionMismatch(f"matrix dimensions must be positive, got {tuple(src.shape)}")
    if ndim == 1 and src.shape[0] < 1:
        raise DimensionMismatch("vector length must be positive")
    out = torch.empty(tuple(src.shape), dtype=dtype, device=device)
    stats = _new_stats(device)
    src_code = _lib.F64 if src.dtype == torch.float64 else _lib.F32
    _lib.call(
        "btas_ingest", _kind_code(kind), src_code, _ptr(src), src.numel(), _dtype_code(dtype), _ptr(out),
        _ptr(stats), _stream(device),
    )
    st = _read_stats(stats)
    noun = "matrix" if ndim == 2 else "vector"
    if st.nan_count:
        raise ValueError(f"{noun} entries cannot be NaN")
    if st.neg_inf_count:
        raise ValueError("use math.inf for the symbolic no-path weight; -inf is not a valid input")
    if st.out_of_range:
        if dtype == torch.int32:
            raise ValueError(f"int32 storage needs integral entries with magnitude below {I32_LIMIT}")
        raise ValueError(f"entries do not fit {dtype} storage")
    return out, st


def _integer_flag(st: _lib.Stats, requested, dtype: torch.dtype) -> bool:
    """_detect_integer (reference matrix.py:98-115) from device statistics."""
    if dtype == torch.int32:
        if requested is False:
            raise ValueError("int32 storage is always integer mode")
        return True
    if requested is False:
        return False
    ok = st.non_integral == 0 and st.over_limit == 0
    if requested is None:
        return ok
    if not ok:
        raise ValueError(f"integer mode needs integral entries with magnitude below {2**53}")
    return True


def _stats_bound(st: _lib.Stats) -> float:
    """max |finite stored value| from ingest statistics (0 when none)."""
    return _lib.key_to_float(st.max_abs_key) if st.finite_count else 0.0


def _sum_bound(*bounds: "float | None") -> "float | None":
    """|a ⊗ b| <= |a| + |b| for finite entries: the bound of a product's
    finite results (None when an operand's bound is unknown).  Widened by
    2^-20 relative: a float32 / float64 sum is rounded once and may land just
    above the exact |a| + |b|, and the bound must stay an upper bound."""
    if any(b is None for b in bounds):
        return None
    return float(sum(bounds)) * (1.0 + 2.0**-20)


def _max_bound(*bounds: "float | None") -> "float | None":
    if any(b is None for b in bounds):
        return None
    return float(max(bounds))


def _symbolic(v: float) -> float:
    return math.inf if math.isinf(v) else v


# ---------------------------------------------------------------------------
# matrices and vectors
# ---------------------------------------------------------------------------
class TropicalMatrix:
    """Immutable dense matrix over one tropical semiring, stored on a GPU.

    ``rows`` may be nested lists, an ndarray, a torch tensor (symbolic form:
    ``math.inf`` is Infinity for both kinds) or contain TropicalWeight
    objects.  integer=None auto-detects exact-integer mode, True demands it,
    False disables it (reference matrix.py:122-156).  ``dtype`` selects the
    storage (float64 default, float32, int32), ``device`` the GPU.

    ``abs_bound`` is an upper bound on max |finite entry| (exact for ingested
    matrices, propagated through products and ⊕; None when unknown): the
    matvec kernels use it to skip their overflow screen (immutable data, so
    the bound never goes stale).
    """

    __slots__ = ("kind", "data", "integer", "abs_bound")

    def __init__(self, kind: SemiringKind, rows: object, integer: "bool | None" = None, *,
                 dtype: "torch.dtype | None" = None, device=None):
        if not isinstance(kind, SemiringKind):
            raise SemiringMismatch(f"not a SemiringKind: {kind!r}")
        dt = dtype if dtype is not None else _default_dtype
        _dtype_code(dt)
        dev = _resolve_device(device)
        data, st = _ingest(kind, rows, dt, dev, 2)
        self._fix(kind, data, _integer_flag(st, integer, dt), _stats_bound(st))

    def _fix(self, kind: SemiringKind, data: torch.Tensor, integer: bool, abs_bound: "float | None" = None) -> None:
        object.__setattr__(self, "kind", kind)
        object.__setattr__(self, "data", data)
        object.__setattr__(self, "integer", bool(integer))
        object.__setattr__(self, "abs_bound", abs_bound)

    def __setattr__(self, name: str, value: object) -> None:
        raise AttributeError("TropicalMatrix is immutable")

    @classmethod
    def _wrap(cls, kind: SemiringKind, data: torch.Tensor, integer: bool,
              abs_bound: "float | None" = None) -> "TropicalMatrix":
        """Adopt already-oriented device storage (internal)."""
        self = object.__new__(cls)
        self._fix(kind, data, integer, abs_bound)
        return self

    @classmethod
    def filled(cls, kind: SemiringKind, n_rows: int, n_cols: int,
               weight: "TropicalWeight | float | int" = math.inf, *,
               dtype: "torch.dtype | None" = None, device=None) -> "TropicalMatrix":
        """Constant matrix; the default fill is Infinity."""
        value = TropicalWeight(float(weight)).value
        n_rows, n_cols = int(n_rows), int(n_cols)
        if n_rows < 1 or n_cols < 1:
            raise DimensionMismatch(f"matrix dimensions must be positive, got {(n_rows, n_cols)}")
        dt = dtype if dtype is not None else _default_dtype
        dev = _resolve_device(device)
        if dt == torch.int32 and not math.isinf(value) and (value != math.floor(value) or abs(value) >= I32_LIMIT):
            raise ValueError(f"int32 storage needs integral entries with magnitude below {I32_LIMIT}")
        if dt == torch.float32 and not math.isinf(value) and math.isinf(float(np.float32(value))):
            raise ValueError(f"entries do not fit {dt} storage")
        data = torch.empty((n_rows, n_cols), dtype=dt, device=dev)
        _lib.call("btas_fill", _dtype_code(dt), _kind_code(kind), _ptr(data), data.numel(), value, _stream(dev))
        stored = float(np.float32(value)) if dt == torch.float32 else value
        integer = dt == torch.int32 or math.isinf(value) or (stored == math.floor(stored) and abs(stored) < 2**53)
        return cls._wrap(kind, data, integer, 0.0 if math.isinf(stored) else abs(stored))

    # -- shape / access ------------------------------------------------------
    @property
    def n_rows(self) -> int:
        return self.data.shape[0]

    @property
    def n_cols(self) -> int:
        return self.data.shape[1]

    @property
    def shape(self) -> "tuple[int, int]":
        return (self.data.shape[0], self.data.shape[1])

    @property
    def dtype(self) -> torch.dtype:
        return self.data.dtype

    @property
    def device(self) -> torch.device:
        return self.data.device

    def to_numpy(self) -> np.ndarray:
        """The reference's oriented float64 array (reference ``.data``)."""
        return _to_f64(self.data).cpu().numpy()

    def weight_at(self, i: int, j: int) -> TropicalWeight:
        v = float(_to_f64(self.data[i, j].reshape(1))[0])
        return TropicalWeight(_symbolic(v))

    def to_lists(self) -> "list[list[float]]":
        """Symbolic-form rows: plain floats with math.inf for Infinity."""
        arr = self.to_numpy()
        sym = np.where(np.isinf(arr), math.inf, arr)
        return [[float(v) for v in row] for row in sym]

    def tobytes(self) -> bytes:
        """Bytes of the oriented float64 array: equal to the reference's tobytes()."""
        return self.to_numpy().tobytes()

    def __eq__(self, other: object) -> bool:
        if not isinstance(other, TropicalMatrix):
            return NotImplemented
        return self.kind is other.kind and self.shape == other.shape and _bytes_equal(self.data, other.data)

    __hash__ = None  # mutable-by-identity objects with value equality

    def __matmul__(self, other: "TropicalMatrix") -> "TropicalMatrix":
        if not isinstance(other, TropicalMatrix):
            return NotImplemented
        return matmul(self, other)

    def __repr__(self) -> str:
        dt = str(self.dtype).replace("torch.", "")
        return (f"TropicalMatrix({self.kind.value}, {self.n_rows}x{self.n_cols}, {dt}"
                f"{', integer' if self.integer else ''})")


class TropicalVector:
    """Immutable dense vector on a GPU; same conventions as TropicalMatrix."""

    __slots__ = ("kind", "data", "integer", "abs_bound")

    def __init__(self, kind: SemiringKind, values: object, integer: "bool | None" = None, *,
                 dtype: "torch.dtype | None" = None, device=None):
        if not isinstance(kind, SemiringKind):
            raise SemiringMismatch(f"not a SemiringKind: {kind!r}")
        dt = dtype if dtype is not None else _default_dtype
        _dtype_code(dt)
        dev = _resolve_device(device)
        data, st = _ingest(kind, values, dt, dev, 1)
        self._fix(kind, data, _integer_flag(st, integer, dt), _stats_bound(st))

    def _fix(self, kind, data, integer, abs_bound=None) -> None:
        object.__setattr__(self, "kind", kind)
        object.__setattr__(self, "data", data)
        object.__setattr__(self, "integer", bool(integer))
        object.__setattr__(self, "abs_bound", abs_bound)

    @classmethod
    def _wrap(cls, kind: SemiringKind, data: torch.Tensor, integer: bool,
              abs_bound: "float | None" = None) -> "TropicalVector":
        self = object.__new__(cls)
        self._fix(kind, data, integer, abs_bound)
        return self

    def __setattr__(self, name: str, value: object) -> None:
        raise AttributeError("TropicalVector is immutable")

    def __len__(self) -> int:
        return self.data.shape[0]

    @property
    def dtype(self) -> torch.dtype:
        return self.data.dtype

    @property
    def device(self) -> torch.device:
        return self.data.device

    def to_numpy(self) -> np.ndarray:
        return _to_f64(self.data).cpu().numpy()

    def weight_at(self, i: int) -> TropicalWeight:
        return TropicalWeight(_symbolic(float(_to_f64(self.data[i].reshape(1))[0])))

    def to_list(self) -> "list[float]":
        return [float(_symbolic(v)) for v in self.to_numpy()]

    def tobytes(self) -> bytes:
        return self.to_numpy().tobytes()

    def __eq__(self, other: object) -> bool:
        if not isinstance(other, TropicalVector):
            return NotImplemented
        return self.kind is other.kind and len(self) == len(other) and _bytes_equal(self.data, other.data)

    __hash__ = None

    def __repr__(self) -> str:
        return f"TropicalVector({self.kind.value}, len={len(self)}, {str(self.dtype).replace('torch.', '')})"


def _to_f64(t: torch.Tensor) -> torch.Tensor:
    t = t.contiguous()
    out = torch.empty(t.shape, dtype=torch.float64, device=t.device)
    if t.numel():
        _lib.call("btas_to_f64", _dtype_code(t.dtype), _ptr(t), t.numel(), _ptr(out), _stream(t.device))
    return out


_INT_VIEW = {4: torch.int32, 8: torch.int64}


def _bytes_equal(a: torch.Tensor, b: torch.Tensor) -> bool:
    if a.shape != b.shape:
        return False
    if a.dtype == b.dtype:
        ia = a.contiguous().view(_INT_VIEW[a.element_size()])
        ib = b.contiguous().view(_INT_VIEW[b.element_size()])
        return bool(torch.equal(ia, ib))
    return bool(torch.equal(_to_f64(a).view(torch.int64), _to_f64(b).view(torch.int64)))


# ---------------------------------------------------------------------------
# operations
# ---------------------------------------------------------------------------
def identity_matrix(kind: SemiringKind, n: int, *, dtype: "torch.dtype | None" = None, device=None) -> TropicalMatrix:
    """0 on the diagonal, Infinity elsewhere (reference matrix.py:257-263)."""
    if not isinstance(n, int) or n < 1:
        raise DimensionMismatch(f"identity size must be a positive integer, got {n!r}")
    dt = dtype if dtype is not None else _default_dtype
    dev = _resolve_device(device)
    data = torch.empty((n, n), dtype=dt, device=dev)
    with _device_ctx(dev):
        _lib.call("btas_identity", _dtype_code(dt), _kind_code(kind), _ptr(data), n, n, _stream(dev))
    return TropicalMatrix._wrap(kind, data, True, 0.0)


def _check_same_kind(a, b) -> None:
    if a.kind is not b.kind:
        raise SemiringMismatch(f"mixed semiring kinds: {a.kind.value} vs {b.kind.value}")


def _check_same_storage(a, b) -> None:
    if a.dtype != b.dtype:
        raise DtypeMismatch(f"mixed storage dtypes: {a.dtype} vs {b.dtype}")
    if a.device != b.device:
        raise ValueError(f"operands live on different devices: {a.device} vs {b.device}")


@_on_operand_device
def ew_add(a, b):
    """Elementwise ⊕ (reference matrix.py:271-277), for matrices and vectors.

    The reference accepts only matrices (a vector has no ``shape``,
    SURVEY §9 quirk 3); vectors are supported here as the natural extension.
    """
    _check_same_kind(a, b)
    if isinstance(a, TropicalMatrix) != isinstance(b, TropicalMatrix):
        raise DimensionMismatch("elementwise ⊕ needs two matrices or two vectors")
    a_shape = a.shape if isinstance(a, TropicalMatrix) else (len(a),)
    b_shape = b.shape if isinstance(b, TropicalMatrix) else (len(b),)
    if a_shape != b_shape:
        raise DimensionMismatch(f"elementwise ⊕ needs equal shapes, got {a_shape} and {b_shape}")
    _check_same_storage(a, b)
    x, y = a.data.contiguous(), b.data.contiguous()
    out = torch.empty_like(x)
    _lib.call("btas_ewadd", _dtype_code(x.dtype), _kind_code(a.kind), _ptr(x), _ptr(y), _ptr(out), x.numel(),
              _stream(x.device))
    return type(a)._wrap(a.kind, out, a.integer and b.integer, _max_bound(a.abs_bound, b.abs_bound))


def _gemm(x: torch.Tensor, y: torch.Tensor, kind: SemiringKind, integer: bool, *, z: "torch.Tensor | None" = None,
          out: "torch.Tensor | None" = None, cprev: "torch.Tensor | None" = None,
          peers: "list[int] | None" = None) -> "tuple[torch.Tensor, torch.Tensor]":
    """One btas_gemm call on the current stream; returns (C, flags).  ``peers``
    (device addresses, same layout as ``out``) selects btas_gemm_peers."""
    m, k = x.shape
    n = y.shape[1]
    dev = x.device
    if out is None:
        out = torch.empty((m, n), dtype=x.dtype, device=dev)
    flags = _flags.new(dev)
    code = _dtype_code(x.dtype)
    nbytes = _lib.load().btas_gemm_workspace_bytes(code, m, n, k)
    ws = _workspace.get(dev, nbytes)
    if peers:
        # fused all-gather: the epilogue also stores C into each peer buffer
        if z is not None:
            raise ValueError("peer stores are not combined with accumulate_into")
        arr = (ctypes.c_void_p * len(peers))(*peers)
        _lib.call(
            "btas_gemm_peers", code, _kind_code(kind), 1 if integer else 0,
            _ptr(x), x.stride(0), _ptr(y), y.stride(0), _ptr(out), out.stride(0), m, n, k,
            _ptr(cprev) if cprev is not None else None, cprev.stride(0) if cprev is not None else 0,
            arr, len(peers), _ptr(flags), _ptr(ws), ws.numel(), _stream(dev),
        )
    else:
        _lib.call(
            "btas_gemm", code, _kind_code(kind), 1 if integer else 0,
            _ptr(x), x.stride(0), _ptr(y), y.stride(0),
            _ptr(z) if z is not None else None, z.stride(0) if z is not None else 0,
            _ptr(out), out.stride(0), m, n, k,
            _ptr(cprev) if cprev is not None else None, cprev.stride(0) if cprev is not None else 0,
            _ptr(flags), _ptr(ws), ws.numel(), _stream(dev),
        )
    _flags.track(flags)
    return out, flags


def _rowmajor(t: torch.Tensor) -> torch.Tensor:
    return t if t.stride(1) == 1 else t.contiguous()


@_on_operand_device
def matmul(x: TropicalMatrix, y: TropicalMatrix, accumulate_into: "TropicalMatrix | None" = None,
           tiles: "TileSpec | None" = None) -> TropicalMatrix:
    """Tropical product, optionally fused with an elementwise ⊕.

    out(i,j) = ⊕_k x(i,k) ⊗ y(k,j), then ⊕ accumulate_into(i,j) when given
    (reference matrix.py:349-400).  accumulate_into is read, never written.
    Finite ⊗ finite sums that overflow (or reach the integer limit in integer
    mode) saturate to Infinity and set the saturation flag, exactly as the
    reference's masked tiles do.
    """
    _check_same_kind(x, y)
    if x.n_cols != y.n_rows:
        raise DimensionMismatch(f"matmul inner dimensions differ: {x.shape} x {y.shape}")
    integer = x.integer and y.integer
    z = None
    if accumulate_into is not None:
        _check_same_kind(x, accumulate_into)
        if accumulate_into.shape != (x.n_rows, y.n_cols):
            raise DimensionMismatch(
                f"accumulate_into shape {accumulate_into.shape} does not match output {(x.n_rows, y.n_cols)}"
            )
        _check_same_storage(x, accumulate_into)
        integer = integer and accumulate_into.integer
        z = _rowmajor(accumulate_into.data)
    if tiles is not None and not isinstance(tiles, TileSpec):
        raise TypeError(f"tiles must be a TileSpec, got {type(tiles).__name__}")
    _check_same_storage(x, y)
    out, _ = _gemm(_rowmajor(x.data), _rowmajor(y.data), x.kind, integer, z=z)
    bound = _sum_bound(x.abs_bound, y.abs_bound)
    if accumulate_into is not None:
        bound = _max_bound(bound, accumulate_into.abs_bound)
    return TropicalMatrix._wrap(x.kind, out, integer, bound)


@_on_operand_device
def matvec(a: TropicalMatrix, v: TropicalVector) -> TropicalVector:
    """out(i) = ⊕_k a(i,k) ⊗ v(k) (reference matrix.py:403-425)."""
    _check_same_kind(a, v)
    if a.n_cols != len(v):
        raise DimensionMismatch(f"matvec dimensions differ: {a.shape} x {len(v)}")
    _check_same_storage(a, v)
    out = matvec_batched(a, v.data.reshape(1, -1), a.integer and v.integer, v_bound=v.abs_bound)
    return TropicalVector._wrap(a.kind, out.reshape(-1), a.integer and v.integer, _sum_bound(a.abs_bound, v.abs_bound))


@_on_operand_device
def matvec_batched(a: TropicalMatrix, vs: "torch.Tensor | TropicalMatrix", integer: "bool | None" = None,
                   v_bound: "float | None" = None) -> torch.Tensor:
    """Batched matvec: rows of ``vs`` (B x K, oriented storage of a's dtype)
    are B vectors; returns the B x M oriented results (one HBM pass over A
    per 8 vectors).  When a's and the vectors' magnitude bounds are known
    (TropicalMatrix operands, or ``v_bound`` for a raw tensor) and prove that
    no candidate can overflow, the kernels run without their screen."""
    if isinstance(vs, TropicalMatrix):
        _check_same_kind(a, vs)
        integer = a.integer and vs.integer if integer is None else integer
        v_bound = vs.abs_bound
        vs = vs.data
    if integer is None:
        integer = a.integer
    if vs.dim() != 2 or vs.shape[1] != a.n_cols:
        raise DimensionMismatch(f"batched matvec needs B x {a.n_cols} vectors, got {tuple(vs.shape)}")
    if vs.dtype != a.dtype:
        raise DtypeMismatch(f"mixed storage dtypes: {a.dtype} vs {vs.dtype}")
    out, _ = _matvec(_rowmajor(a.data), _rowmajor(vs), a.kind, integer, _sum_bound(a.abs_bound, v_bound))
    return out


def _matvec(A: torch.Tensor, V: torch.Tensor, kind: SemiringKind, integer: bool,
            bound: "float | None") -> "tuple[torch.Tensor, torch.Tensor]":
    """One btas_matvec_bounded call on the current stream: (B x M result,
    flag words)."""
    dev = A.device
    out = torch.empty((V.shape[0], A.shape[0]), dtype=A.dtype, device=dev)
    flags = _flags.new(dev)
    _lib.call(
        "btas_matvec_bounded", _dtype_code(A.dtype), _kind_code(kind), 1 if integer else 0,
        _ptr(A), A.stride(0), A.shape[0], A.shape[1], _ptr(V), V.stride(0), V.shape[0], _ptr(out), out.stride(0),
        -1.0 if bound is None else bound, _ptr(flags), _stream(dev),
    )
    _flags.track(flags)
    return out, flags


@_on_operand_device
def matrix_power(a: TropicalMatrix, p: int, tiles: "TileSpec | None" = None) -> TropicalMatrix:
    """Semiring p-th power by LSB-first binary exponentiation
    (reference matrix.py:428-448); ``matrix_power(a, 1) is a``."""
    if a.n_rows != a.n_cols:
        raise DimensionMismatch(f"matrix_power needs a square matrix, got {a.shape}")
    if not isinstance(p, int) or p < 1:
        raise ValueError(f"power must be a positive integer, got {p!r}")
    result = None
    base = a
    e = p
    while True:
        if e & 1:
            result = base if result is None else matmul(result, base, tiles=tiles)
        e >>= 1
        if not e:
            return result
        base = matmul(base, base, tiles=tiles)
