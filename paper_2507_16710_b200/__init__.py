"""paper_2507_16710_b200 -- B200-native sorting-centred primitives (arXiv 2507.16710).

Python mirror of the reference C++ API (/root/reference/proj/include/ak/*.hpp)
over the C ABI of ``lib/libak_cuda.so`` (declared in ``include/ak_cuda.h``).
Names, argument meaning and error behaviour follow the reference:

    merge_sort, merge_sort_copy, merge_sort_by_key, sortperm, sortperm_lowmem
        (sort.hpp:180-290)
    reduce, mapreduce (reduce.hpp:62-75)
    accumulate (scan.hpp:29-88)
    searchsorted (search.hpp:36-50)
    sihsort, sihsort_loopback (sihsort.hpp:508-569 over NCCL / sim::world)

Device data are torch CUDA tensors; PyTorch is only the allocator/stream
plumbing. There is NO CPU fallback: if the CUDA library is missing the import
fails, and every call runs the sm_100a kernels.

Errors map to the reference's exception types: std::invalid_argument ->
``ValueError`` (``InvalidArgument``), sim::protocol_error -> ``ProtocolError``,
sim::transport_error -> ``TransportError``.
"""
from __future__ import annotations

import ctypes as C
import operator
import os
from dataclasses import dataclass

import numpy as np
import torch

__all__ = [
    "ExecBackend", "InvalidArgument", "ProtocolError", "TransportError", "CapacityError",
    "SortBuffers", "SortByKeyBuffers", "SortpermBuffers", "SortpermLowmemBuffers",
    "merge_sort", "merge_sort_copy", "merge_sort_by_key", "sortperm", "sortperm_lowmem",
    "reduce", "mapreduce", "accumulate", "searchsorted", "SihConfig", "SihStats",
    "NcclComm", "sihsort", "sihsort_host", "sihsort_loopback", "bench_keys", "lib", "LIB_PATH",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AKB_LIB") or os.path.join(HERE, "lib", "libak_cuda.so")


class InvalidArgument(ValueError):
    """std::invalid_argument of the reference (sort.hpp:182-184 etc.)."""


class ProtocolError(RuntimeError):
    """ak::sim::protocol_error (sim_comm.hpp:24-26)."""


class TransportError(RuntimeError):
    """ak::sim::transport_error (sim_comm.hpp:19-21)."""


class CapacityError(RuntimeError):
    def __init__(self, msg: str, required: int):
        super().__init__(msg)
        self.required = required


class CudaError(RuntimeError):
    pass


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    return C.CDLL(LIB_PATH)


_lib = _load()


def lib() -> C.CDLL:
    return _lib


_lib.ak_last_error.restype = C.c_char_p
_lib.ak_version.restype = C.c_char_p
_lib.ak_ctx_kernel_launches.restype = C.c_uint64
_lib.ak_ctx_kernel_launches.argtypes = [C.c_void_p]
_lib.ak_ctx_stream.restype = C.c_void_p
_lib.ak_ctx_stream.argtypes = [C.c_void_p]
for _f in ("ak_sort_scratch_bytes", "ak_sort_by_key_scratch_bytes", "ak_sortperm_scratch_bytes",
           "ak_sortperm_lowmem_scratch_bytes", "ak_sort_ctx_bytes"):
    getattr(_lib, _f).restype = C.c_uint64
_lib.ak_sort_scratch_bytes.argtypes = [C.c_uint64, C.c_int]
_lib.ak_sort_by_key_scratch_bytes.argtypes = [C.c_uint64, C.c_int, C.c_int]
_lib.ak_sortperm_scratch_bytes.argtypes = [C.c_uint64, C.c_int, C.c_int]
_lib.ak_sortperm_lowmem_scratch_bytes.argtypes = [C.c_uint64, C.c_int]
_lib.ak_sort_ctx_bytes.argtypes = [C.c_uint64, C.c_int]

_SUFFIX = {torch.int32: "i32", torch.uint32: "u32", torch.int64: "i64", torch.uint64: "u64",
           torch.float32: "f32", torch.float64: "f64"}
# sort family only (dtype.hpp:14-21): int16, and int128 as an (n, 2) int64 tensor (low, high
# words, little endian -- the memory layout of __int128)
_SORT_SUFFIX = {**_SUFFIX, torch.int16: "i16"}
_NP_SUFFIX = {np.dtype(np.int32): "i32", np.dtype(np.uint32): "u32", np.dtype(np.int64): "i64",
              np.dtype(np.uint64): "u64", np.dtype(np.float32): "f32", np.dtype(np.float64): "f64"}
_CT = {"i32": C.c_int32, "u32": C.c_uint32, "i64": C.c_int64, "u64": C.c_uint64, "f32": C.c_float,
       "f64": C.c_double}
_U64 = C.c_uint64
_P = C.c_void_p


def _check(rc: int, extra_required: int | None = None) -> None:
    if rc == 0:
        return
    msg = (_lib.ak_last_error() or b"").decode()
    if rc == 1:
        raise InvalidArgument(msg)
    if rc == 2:
        raise ProtocolError(msg)
    if rc == 3:
        raise TransportError(msg)
    if rc == 6:
        raise CapacityError(msg, extra_required or 0)
    if rc == 4:
        raise CudaError(msg)
    raise RuntimeError(f"ak error {rc}: {msg}")


_FN_CACHE: dict = {}


def _fn(name: str, argtypes, restype=C.c_int):
    """The C-ABI symbol with its prototype set (once per symbol: one signature per name)."""
    f = _FN_CACHE.get(name)
    if f is None:
        f = getattr(_lib, name)
        f.argtypes = argtypes
        f.restype = restype
        _FN_CACHE[name] = f
    return f


# ----------------------------------------------------------------------------- exec backend

class ExecBackend:
    """exec_backend with exec_kind::cuda (exec.hpp:31-60): device + stream + ctx scratch.

    Handles are shareable; calls on one handle are serialised. Blocking by
    default (reference SPEC.md:64); ``set_blocking(False)`` leaves work queued on
    ``stream`` for CUDA-event timing and graph capture.
    """

    _default: dict[int, "ExecBackend"] = {}

    def __init__(self, device: int = 0, stream: torch.cuda.Stream | None = None):
        self.device = device
        h = C.c_void_p()
        raw = None if stream is None else C.c_void_p(stream.cuda_stream)
        _check(_fn("ak_ctx_create", [C.c_int, _P, C.POINTER(C.c_void_p)])(device, raw, C.byref(h)))
        self._h = h
        sp = _lib.ak_ctx_stream(h)
        self.stream = stream if stream is not None else torch.cuda.ExternalStream(sp, device=device)
        self.blocking = True

    @staticmethod
    def cuda(device: int = 0) -> "ExecBackend":
        if device not in ExecBackend._default:
            ExecBackend._default[device] = ExecBackend(device)
        return ExecBackend._default[device]

    kind = "cuda"

    @property
    def handle(self) -> C.c_void_p:
        """The C handle; ordering point: work queued on torch's current stream (e.g. the
        producer of an input tensor) completes before the ctx stream runs the next op."""
        cur = torch.cuda.current_stream(self.device)
        if cur.cuda_stream != self.stream.cuda_stream:
            self.stream.wait_stream(cur)
        return self._h

    def fence(self) -> None:
        """Make torch's current stream wait for everything queued on the ctx stream
        (only needed after non-blocking calls)."""
        torch.cuda.current_stream(self.device).wait_stream(self.stream)

    def set_blocking(self, blocking: bool) -> None:
        _check(_fn("ak_ctx_set_blocking", [_P, C.c_int])(self._h, int(blocking)))
        self.blocking = blocking

    def synchronize(self) -> None:
        _check(_fn("ak_ctx_synchronize", [_P])(self._h))

    def reserve(self, aux_bytes: int) -> None:
        _check(_fn("ak_ctx_reserve", [_P, _U64])(self._h, aux_bytes))

    def kernel_launches(self) -> int:
        return int(_lib.ak_ctx_kernel_launches(self._h))

    KF = {"onesweep": 0, "hist": 1, "merge": 2, "reduce": 3, "scan": 4, "search": 5, "exchange": 6,
          "other": 7, "local": 8, "msd": 9}

    def set_profiling(self, on: bool) -> None:
        """Bracket every hot kernel with CUDA events on the ctx stream."""
        _check(_fn("ak_ctx_set_profiling", [_P, C.c_int])(self._h, int(on)))

    def kernel_time(self, family: str) -> tuple[float, int]:
        ms, cnt = C.c_double(), _U64()
        _check(_fn("ak_ctx_kernel_time", [_P, C.c_int, C.POINTER(C.c_double), C.POINTER(_U64)])(
            self._h, self.KF[family], C.byref(ms), C.byref(cnt)))
        return ms.value, int(cnt.value)

    def reset_kernel_time(self) -> None:
        _check(_fn("ak_ctx_reset_kernel_time", [_P])(self._h))

    def close(self) -> None:
        if getattr(self, "_h", None):
            _fn("ak_ctx_destroy", [_P])(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass


def _ex(ex: ExecBackend | None, t: torch.Tensor | None = None) -> ExecBackend:
    if ex is not None:
        return ex
    dev = t.device.index if (t is not None and t.is_cuda and t.device.index is not None) else 0
    return ExecBackend.cuda(dev)


def _dev(t: torch.Tensor, what: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise InvalidArgument(f"{what}: expected a CUDA tensor (device data); use the *_host entry points "
                              "for host arrays")
    if not t.is_contiguous():
        raise InvalidArgument(f"{what}: tensor must be contiguous")
    return t


def _suffix(t: torch.Tensor) -> str:
    try:
        return _SUFFIX[t.dtype]
    except KeyError:
        raise InvalidArgument(f"unsupported dtype {t.dtype}") from None


def _sort_keys(t: torch.Tensor) -> tuple[str, int]:
    """(suffix, element count) of a sort-family key tensor; (n, 2) int64 = n int128 keys."""
    if t.dtype == torch.int64 and t.dim() == 2 and t.shape[1] == 2:
        return "i128", t.shape[0]
    try:
        return _SORT_SUFFIX[t.dtype], t.numel()
    except KeyError:
        raise InvalidArgument(f"unsupported dtype {t.dtype}") from None


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _desc(cmp) -> int:
    """Comparator: std::less (default / operator.lt / 'less') or std::greater."""
    if cmp is None or cmp in ("less", operator.lt):
        return 0
    if cmp in ("greater", operator.gt):
        return 1
    raise InvalidArgument("comparator must be less or greater (no custom comparators on the cuda kind)")


# ----------------------------------------------------------------------------- buffers (sort.hpp:22-65)

@dataclass
class SortBuffers:
    scratch_keys: torch.Tensor

    @staticmethod
    def required_bytes(n: int, key_bytes: int = 8) -> int:
        return int(_lib.ak_sort_scratch_bytes(n, key_bytes))

    @staticmethod
    def with_capacity(n: int, dtype=torch.int64, device: int = 0) -> "SortBuffers":
        return SortBuffers(torch.empty(n, dtype=dtype, device=f"cuda:{device}"))


@dataclass
class SortByKeyBuffers:
    scratch_keys: torch.Tensor
    scratch_payload: torch.Tensor

    @staticmethod
    def required_bytes(n: int, key_bytes: int, payload_bytes: int) -> int:
        return int(_lib.ak_sort_by_key_scratch_bytes(n, key_bytes, payload_bytes))

    @staticmethod
    def with_capacity(n: int, key_dtype, payload_dtype, device: int = 0) -> "SortByKeyBuffers":
        d = f"cuda:{device}"
        return SortByKeyBuffers(torch.empty(n, dtype=key_dtype, device=d),
                                torch.empty(n, dtype=payload_dtype, device=d))


@dataclass
class SortpermBuffers:
    working_keys: torch.Tensor
    scratch_keys: torch.Tensor
    scratch_index: torch.Tensor

    @staticmethod
    def required_bytes(n: int, key_bytes: int, index_bytes: int) -> int:
        return int(_lib.ak_sortperm_scratch_bytes(n, key_bytes, index_bytes))

    @staticmethod
    def with_capacity(n: int, key_dtype, index_dtype=torch.int64, device: int = 0) -> "SortpermBuffers":
        d = f"cuda:{device}"
        return SortpermBuffers(torch.empty(n, dtype=key_dtype, device=d),
                               torch.empty(n, dtype=key_dtype, device=d),
                               torch.empty(n, dtype=index_dtype, device=d))


@dataclass
class SortpermLowmemBuffers:
    scratch_index: torch.Tensor

    @staticmethod
    def required_bytes(n: int, index_bytes: int) -> int:
        return int(_lib.ak_sortperm_lowmem_scratch_bytes(n, index_bytes))

    @staticmethod
    def with_capacity(n: int, index_dtype=torch.int64, device: int = 0) -> "SortpermLowmemBuffers":
        return SortpermLowmemBuffers(torch.empty(n, dtype=index_dtype, device=f"cuda:{device}"))


# ----------------------------------------------------------------------------- sort family

def merge_sort(data: torch.Tensor, scratch=None, ex: ExecBackend | None = None, cmp=None) -> None:
    """Stable in-place sort (sort.hpp:180-194). scratch: tensor, SortBuffers or None (allocated)."""
    _dev(data, "merge_sort")
    e = _ex(ex, data)
    if isinstance(scratch, SortBuffers):
        scratch = scratch.scratch_keys
    if scratch is None:
        scratch = torch.empty_like(data)
    s, n = _sort_keys(data)
    f = _fn(f"ak_merge_sort_{s}", [_P, _P, _U64, _P, _U64, C.c_int])
    _check(f(e.handle, _ptr(data), n, _ptr(scratch), _sort_keys(scratch)[1], _desc(cmp)))


def merge_sort_copy(data: torch.Tensor, ex: ExecBackend | None = None, cmp=None) -> torch.Tensor:
    """Allocating variant (sort.hpp:197-203): returns a sorted copy."""
    out = data.clone()
    merge_sort(out, None, ex, cmp)
    return out


def merge_sort_host(data: np.ndarray, ex: ExecBackend | None = None, cmp=None) -> None:
    """merge_sort on a host array (H2D, device sort, D2H inside the call)."""
    data = np.ascontiguousarray(data)
    s = _NP_SUFFIX[data.dtype]
    f = _fn(f"ak_merge_sort_host_{s}", [_P, _P, _U64, C.c_int])
    _check(f(_ex(ex).handle, data.ctypes.data, data.size, _desc(cmp)))


def merge_sort_by_key(keys: torch.Tensor, payload: torch.Tensor, buffers=None,
                      ex: ExecBackend | None = None, cmp=None) -> None:
    """Stable key sort with co-moving payload (sort.hpp:211-229); payload is any 4/8-byte dtype."""
    _dev(keys, "merge_sort_by_key")
    _dev(payload, "merge_sort_by_key")
    e = _ex(ex, keys)
    if buffers is None:
        buffers = SortByKeyBuffers(torch.empty_like(keys), torch.empty_like(payload))
    sk, sp = buffers.scratch_keys, buffers.scratch_payload
    w = payload.element_size()
    if w not in (4, 8) or sp.element_size() != w:
        raise InvalidArgument("merge_sort_by_key: payload must be 4- or 8-byte elements")
    ks, kn = _sort_keys(keys)
    f = _fn(f"ak_merge_sort_by_key_{ks}_b{8 * w}",
            [_P, _P, _U64, _P, _U64, _P, _U64, _P, _U64, C.c_int])
    _check(f(e.handle, _ptr(keys), kn, _ptr(payload), payload.numel(), _ptr(sk), _sort_keys(sk)[1],
             _ptr(sp), sp.numel(), _desc(cmp)))


def _index_suffix(dt) -> str:
    if dt in (torch.int32, torch.uint32):
        return "i32"
    if dt in (torch.int64, torch.uint64):
        return "i64"
    raise InvalidArgument("sortperm: index dtype must be a 32- or 64-bit integer")


def sortperm(data: torch.Tensor, out: torch.Tensor | None = None, buffers: SortpermBuffers | None = None,
             ex: ExecBackend | None = None, cmp=None, index_dtype=torch.int64) -> torch.Tensor:
    """Stable index permutation (sort.hpp:238-262); equal keys keep ascending indices."""
    _dev(data, "sortperm")
    e = _ex(ex, data)
    ks, n = _sort_keys(data)
    if out is None:
        out = torch.empty(n, dtype=index_dtype, device=data.device)
    if buffers is None:
        buffers = SortpermBuffers(torch.empty_like(data), torch.empty_like(data),
                                  torch.empty(n, dtype=out.dtype, device=data.device))
    isuf = _index_suffix(out.dtype)
    f = _fn(f"ak_sortperm_{ks}_{isuf}", [_P, _P, _U64, _P, _U64, _P, _U64, _P, _U64, _P, _U64, C.c_int])
    _check(f(e.handle, _ptr(data), n, _ptr(out), out.numel(), _ptr(buffers.working_keys),
             _sort_keys(buffers.working_keys)[1], _ptr(buffers.scratch_keys), _sort_keys(buffers.scratch_keys)[1],
             _ptr(buffers.scratch_index), buffers.scratch_index.numel(), _desc(cmp)))
    return out


def sortperm_lowmem(data: torch.Tensor, out: torch.Tensor | None = None,
                    buffers: SortpermLowmemBuffers | None = None, ex: ExecBackend | None = None, cmp=None,
                    index_dtype=torch.int64) -> torch.Tensor:
    """Low-memory sortperm (sort.hpp:267-290): index scratch only, keys gathered per pass."""
    _dev(data, "sortperm_lowmem")
    e = _ex(ex, data)
    ks, n = _sort_keys(data)
    if out is None:
        out = torch.empty(n, dtype=index_dtype, device=data.device)
    if buffers is None:
        buffers = SortpermLowmemBuffers(torch.empty(n, dtype=out.dtype, device=data.device))
    isuf = _index_suffix(out.dtype)
    f = _fn(f"ak_sortperm_lowmem_{ks}_{isuf}", [_P, _P, _U64, _P, _U64, _P, _U64, C.c_int])
    _check(f(e.handle, _ptr(data), n, _ptr(out), out.numel(), _ptr(buffers.scratch_index),
             buffers.scratch_index.numel(), _desc(cmp)))
    return out


# ----------------------------------------------------------------------------- reduce / scan

_OPS = {"sum": 0, "+": 0, operator.add: 0, "min": 1, min: 1, "max": 2, max: 2}
_MAPS = {"identity": 0, None: 0, "abs": 1, abs: 1, operator.abs: 1, "square": 2}


def _op(op) -> int:
    try:
        return _OPS[op]
    except (KeyError, TypeError):
        raise InvalidArgument("op must be sum/min/max (no arbitrary callables on the cuda kind)") from None


def _neutral(dtype: torch.dtype, op: int):
    if op == 0:
        return 0
    if dtype.is_floating_point:
        return float("inf") if op == 1 else float("-inf")
    info = torch.iinfo(dtype)
    return info.max if op == 1 else info.min


def reduce(op, data: torch.Tensor, init=None, ex: ExecBackend | None = None, switch_below: int = 256):
    """reduce(op, data, reduce_config{init}) (reduce.hpp:62-66). init must be neutral
    (the reference folds a non-neutral init once per chunk, reduce.hpp:34; here exactly once)."""
    return mapreduce("identity", op, data, init, ex, switch_below)


def mapreduce(f, op, data: torch.Tensor, init=None, ex: ExecBackend | None = None, switch_below: int = 256):
    """mapreduce(f, op, data, cfg) (reduce.hpp:70-75) with f in {identity, abs, square}."""
    _dev(data, "reduce")
    e = _ex(ex, data)
    o = _op(op)
    try:
        m = _MAPS[f]
    except (KeyError, TypeError):
        raise InvalidArgument("map must be identity/abs/square (no arbitrary callables on the cuda kind)") from None
    s = _suffix(data)
    ct = _CT[s]
    res = ct()
    if init is None:
        init = _neutral(data.dtype, o)
    fn = _fn(f"ak_reduce_{s}", [_P, _P, _U64, C.c_int, C.c_int, ct, C.POINTER(ct)])
    _check(fn(e.handle, _ptr(data), data.numel(), o, m, init, C.byref(res)))
    return res.value


def reduce_device(op, data: torch.Tensor, result: torch.Tensor, init=None, ex: ExecBackend | None = None,
                  f="identity") -> None:
    """Device-result reduce (no host sync in non-blocking mode)."""
    _dev(data, "reduce")
    e = _ex(ex, data)
    o = _op(op)
    s = _suffix(data)
    ct = _CT[s]
    if init is None:
        init = _neutral(data.dtype, o)
    fn = _fn(f"ak_reduce_device_{s}", [_P, _P, _U64, C.c_int, C.c_int, ct, _P])
    _check(fn(e.handle, _ptr(data), data.numel(), o, _MAPS[f], init, _ptr(result)))


def accumulate(op, data: torch.Tensor, out: torch.Tensor | None = None, inclusive: bool = True, init=0,
               chunk_size: int = 4096, ex: ExecBackend | None = None) -> torch.Tensor:
    """Prefix scan (scan.hpp:29-88). out may be data (in place)."""
    _dev(data, "accumulate")
    e = _ex(ex, data)
    if out is None:
        out = torch.empty_like(data)
    s = _suffix(data)
    ct = _CT[s]
    fn = _fn(f"ak_accumulate_{s}", [_P, _P, _U64, _P, _U64, C.c_int, C.c_int, ct, _U64])
    _check(fn(e.handle, _ptr(data), data.numel(), _ptr(out), out.numel(), _op(op), int(inclusive), init,
              chunk_size))
    return out


def searchsorted(haystack: torch.Tensor, needles: torch.Tensor, side: str = "first",
                 ex: ExecBackend | None = None, cmp=None, validate: bool = False) -> torch.Tensor:
    """Batched insertion indices (search.hpp:36-50) -> int64 tensor (values are size_t)."""
    _dev(haystack, "searchsorted")
    _dev(needles, "searchsorted")
    if needles.dtype != haystack.dtype:
        raise InvalidArgument("searchsorted: needles and haystack dtypes differ")
    if side not in ("first", "last"):
        raise InvalidArgument("side must be 'first' or 'last'")
    e = _ex(ex, haystack)
    out = torch.empty(needles.numel(), dtype=torch.int64, device=haystack.device)
    fn = _fn(f"ak_searchsorted_{_suffix(haystack)}", [_P, _P, _U64, _P, _U64, C.c_int, C.c_int, C.c_int, _P])
    _check(fn(e.handle, _ptr(haystack), haystack.numel(), _ptr(needles), needles.numel(), int(side == "last"),
              _desc(cmp), int(validate), _ptr(out)))
    return out


def merge_runs(runs: list, out: torch.Tensor | None = None, ex: ExecBackend | None = None, cmp=None,
               scratch: torch.Tensor | None = None) -> torch.Tensor:
    """Stable P-way merge of sorted device runs (1 <= P <= 4096); equal keys keep run order,
    i.e. the result is the stable sort of the runs' concatenation (sihsort.hpp:555)."""
    if not runs:
        raise InvalidArgument("merge_runs: no runs")
    for r in runs:
        _dev(r, "merge_runs")
        if r.dtype != runs[0].dtype:
            raise InvalidArgument("merge_runs: runs must share a dtype")
    e = _ex(ex, runs[0])
    total = sum(r.numel() for r in runs)
    if out is None:
        out = torch.empty(total, dtype=runs[0].dtype, device=runs[0].device)
    if scratch is None:
        scratch = torch.empty(max(total, 1), dtype=runs[0].dtype, device=runs[0].device)
    P = len(runs)
    ptrs = (C.c_void_p * P)(*[_ptr(r) for r in runs])
    lens = (C.c_uint64 * P)(*[r.numel() for r in runs])
    fn = _fn(f"ak_merge_runs_{_suffix(runs[0])}", [_P, C.c_int, _P, _P, _P, _P, C.c_int])
    _check(fn(e.handle, P, C.cast(ptrs, C.c_void_p), C.cast(lens, C.c_void_p), _ptr(out), _ptr(scratch),
              _desc(cmp)))
    return out


# ----------------------------------------------------------------------------- sihsort

class SihConfig(C.Structure):
    """sih_config (sihsort.hpp:21-26)."""
    _fields_ = [("sample_per_rank", _U64), ("bins", _U64), ("max_refine_rounds", _U64),
                ("imbalance_tol", C.c_double)]

    def __init__(self, sample_per_rank=0, bins=0, max_refine_rounds=4, imbalance_tol=0.25):
        super().__init__(sample_per_rank, bins, max_refine_rounds, imbalance_tol)


class SihStats(C.Structure):
    """sih_stats (sihsort.hpp:45-53)."""
    _fields_ = [("rounds_used", _U64), ("converged", _U64), ("max_deviation", C.c_double),
                ("redistribution_sends", _U64), ("redistribution_bytes", _U64),
                ("collective_ops", _U64), ("output_count", _U64)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


class NcclComm:
    """rank_comm over NCCL (replaces sim::rank_comm, sim_comm.hpp:84-181).

    Bootstrap: rank 0 calls ``NcclComm.unique_id()``, the id is broadcast by any
    side channel (torch.distributed in bench.py), then every rank constructs.
    """

    def __init__(self, unique_id: bytes, nranks: int, rank: int, device: int):
        h = C.c_void_p()
        buf = C.create_string_buffer(unique_id, len(unique_id))
        _check(_fn("ak_comm_nccl_create", [_P, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)])(
            buf, nranks, rank, device, C.byref(h)))
        self._h = h
        self.rank, self.size = rank, nranks

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(_fn("ak_nccl_unique_id", [_P, _U64])(buf, 128))
        return buf.raw

    @property
    def handle(self):
        return self._h

    def bytes_sent(self) -> int:
        v = _U64()
        _check(_fn("ak_comm_bytes_sent", [_P, C.POINTER(_U64)])(self._h, C.byref(v)))
        return int(v.value)

    def allreduce_max(self, values: list[float], ex: ExecBackend) -> list[float]:
        arr = (C.c_double * len(values))(*values)
        _check(_fn("ak_comm_allreduce_max_f64", [_P, _P, _P, _U64])(self._h, ex.handle, arr, len(values)))
        return list(arr)

    def barrier(self, ex: ExecBackend) -> None:
        _check(_fn("ak_comm_barrier", [_P, _P])(self._h, ex.handle))

    def close(self) -> None:
        if getattr(self, "_h", None):
            _fn("ak_comm_destroy", [_P])(self._h)
            self._h = None


_AG_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p)
_AR_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64)


class IpcComm:
    """rank_comm of one process per GPU whose bulk exchange is a peer-store kernel writing
    straight into the peers' receive buffers (CUDA IPC mappings: P2P over NVLink/NVSwitch,
    or the same GPU). Control messages (tiny allgather / allreduce) go over a torch.distributed
    gloo group. Requires torch.distributed to be initialised (any backend)."""

    def __init__(self, device: int, group=None):
        import torch.distributed as dist
        self._dist = dist
        self.rank, self.size = dist.get_rank(), dist.get_world_size()
        self._group = group if group is not None else dist.new_group(backend="gloo")
        world = self.size

        def ag(user, inp, nbytes, out):
            try:
                buf = torch.frombuffer(bytearray(C.string_at(inp, nbytes)), dtype=torch.uint8) if nbytes else \
                    torch.empty(0, dtype=torch.uint8)
                outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
                dist.all_gather(outs, buf, group=self._group)
                if nbytes:
                    cat = torch.cat(outs).numpy()
                    C.memmove(out, cat.ctypes.data, nbytes * world)
                return 0
            except Exception:  # pragma: no cover - surfaced as AK_ETRANSPORT
                return 1

        def ar(user, ptr, n):
            try:
                arr = np.frombuffer(C.string_at(ptr, 8 * n), dtype=np.int64).copy()
                t = torch.from_numpy(arr)
                dist.all_reduce(t, group=self._group)  # wrapping int64 sum == uint64 sum
                C.memmove(ptr, t.numpy().ctypes.data, 8 * n)
                return 0
            except Exception:  # pragma: no cover
                return 1

        self._cb = (_AG_FN(ag), _AR_FN(ar))
        h = C.c_void_p()
        _check(_fn("ak_comm_ipc_create", [C.c_int, C.c_int, C.c_int, _P, _AG_FN, _AR_FN, C.POINTER(C.c_void_p)])(
            self.size, self.rank, device, None, self._cb[0], self._cb[1], C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def bytes_sent(self) -> int:
        v = _U64()
        _check(_fn("ak_comm_bytes_sent", [_P, C.POINTER(_U64)])(self._h, C.byref(v)))
        return int(v.value)

    def allreduce_max(self, values: list[float], ex: ExecBackend) -> list[float]:
        arr = (C.c_double * len(values))(*values)
        _check(_fn("ak_comm_allreduce_max_f64", [_P, _P, _P, _U64])(self._h, ex.handle, arr, len(values)))
        return list(arr)

    def barrier(self, ex: ExecBackend) -> None:
        _check(_fn("ak_comm_barrier", [_P, _P])(self._h, ex.handle))

    def close(self) -> None:
        if getattr(self, "_h", None):
            _fn("ak_comm_destroy", [_P])(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


class LoopbackWorld:
    """sim::world on one device (sim_comm.hpp:41-80): P logical ranks, each driven by its own
    host thread with its own ExecBackend; ``comm(r)`` is rank r's rank_comm."""

    def __init__(self, ranks: int):
        h = C.c_void_p()
        _check(_fn("ak_world_create", [C.c_int, C.POINTER(C.c_void_p)])(ranks, C.byref(h)))
        self._h = h
        self.size = ranks

    def comm(self, rank: int) -> "LoopbackComm":
        return LoopbackComm(self, rank)

    def abort(self) -> None:
        _fn("ak_world_abort", [_P])(self._h)

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            if getattr(self, "_h", None):
                _fn("ak_world_destroy", [_P])(self._h)
        except Exception:
            pass


class LoopbackComm:
    def __init__(self, world: LoopbackWorld, rank: int):
        h = C.c_void_p()
        _check(_fn("ak_comm_loopback_create", [_P, C.c_int, C.POINTER(C.c_void_p)])(world._h, rank, C.byref(h)))
        self._h, self.rank, self.size, self._world = h, rank, world.size, world

    @property
    def handle(self):
        return self._h

    def __del__(self):  # pragma: no cover
        try:
            if getattr(self, "_h", None):
                _fn("ak_comm_destroy", [_P])(self._h)
        except Exception:
            pass


def reduce_all(op, data: torch.Tensor, comm, init=None, ex: ExecBackend | None = None, f="identity"):
    """Reduce over every rank of ``comm``: device pass per rank + one
    allgather of the rank partials folded in rank order. Collective."""
    _dev(data, "reduce_all")
    e = _ex(ex, data)
    o = _op(op)
    try:
        m = _MAPS[f]
    except (KeyError, TypeError):
        raise InvalidArgument("map must be identity/abs/square") from None
    s = _suffix(data)
    ct = _CT[s]
    res = ct()
    if init is None:
        init = _neutral(data.dtype, o)
    fn = _fn(f"ak_reduce_all_{s}", [_P, _P, _P, _U64, C.c_int, C.c_int, ct, C.POINTER(ct)])
    _check(fn(e.handle, comm.handle if comm is not None else None, _ptr(data), data.numel(), o, m, init,
              C.byref(res)))
    return res.value


def accumulate_all(op, data: torch.Tensor, comm, out: torch.Tensor | None = None, inclusive: bool = True, init=0,
                   ex: ExecBackend | None = None) -> torch.Tensor:
    """Prefix scan over the concatenation of every rank's data in rank order: each rank gets its
    slice of the global scan (local scan seeded with init and the lower ranks' totals). Collective."""
    _dev(data, "accumulate_all")
    e = _ex(ex, data)
    if out is None:
        out = torch.empty_like(data)
    s = _suffix(data)
    ct = _CT[s]
    fn = _fn(f"ak_accumulate_all_{s}", [_P, _P, _P, _U64, _P, _U64, C.c_int, C.c_int, ct])
    _check(fn(e.handle, comm.handle if comm is not None else None, _ptr(data), data.numel(), _ptr(out), out.numel(),
              _op(op), int(inclusive), init))
    return out


_PRED_OPS = {"<": 0, "lt": 0, "<=": 1, "le": 1, ">": 2, "gt": 2, ">=": 3, "ge": 3, "==": 4, "eq": 4, "!=": 5,
             "ne": 5}
_PRED_SUFFIX = {**_SUFFIX, torch.uint8: "u8", torch.int8: "i8", torch.int16: "i16"}
_PRED_CT = dict(_CT, u8=C.c_uint8, i8=C.c_int8, i16=C.c_int16)


def _pred(which: str, data: torch.Tensor, op: str, value, ex, algo: str) -> bool:
    _dev(data, which)
    e = _ex(ex, data)
    try:
        s = _PRED_SUFFIX[data.dtype]
        o = _PRED_OPS[op]
    except KeyError:
        raise InvalidArgument(f"{which}: predicate must be x OP value with OP in < <= > >= == !=") from None
    if algo not in ("early_exit", "via_mapreduce"):
        raise InvalidArgument("algo must be early_exit or via_mapreduce")
    ct = _PRED_CT[s]
    r = C.c_int()
    fn = _fn(f"ak_{which}_{s}", [_P, _P, _U64, C.c_int, ct, C.c_int, C.POINTER(C.c_int)])
    _check(fn(e.handle, _ptr(data), data.numel(), o, value, int(algo == "via_mapreduce"), C.byref(r)))
    return bool(r.value)


def any_pred(data: torch.Tensor, op: str, value, ex: ExecBackend | None = None, algo: str = "early_exit") -> bool:
    """True iff (x OP value) for some element (predicates.hpp:57-66); empty -> False."""
    return _pred("any_pred", data, op, value, ex, algo)


def all_pred(data: torch.Tensor, op: str, value, ex: ExecBackend | None = None, algo: str = "early_exit") -> bool:
    """True iff (x OP value) for every element (predicates.hpp:69-78); empty -> True."""
    return _pred("all_pred", data, op, value, ex, algo)


def sihsort(local_data: torch.Tensor, comm: NcclComm | None = None, cfg: SihConfig | None = None,
            ex: ExecBackend | None = None, out: torch.Tensor | None = None, capacity: int | None = None):
    """Distributed sample sort (sihsort.hpp:508-569) of this rank's device keys.

    Returns (sorted local output tensor, SihStats). local_data is not modified.
    ``out``/``capacity`` preallocate the output; by default capacity is 2n (+1024)
    and is retried once with the exact requirement on CapacityError.
    """
    _dev(local_data, "sihsort")
    e = _ex(ex, local_data)
    n = local_data.numel()
    s = _suffix(local_data)
    fn = _fn(f"ak_sihsort_{s}", [_P, _P, _P, _U64, _P, _U64, C.POINTER(_U64), C.POINTER(SihConfig),
                                  C.POINTER(SihStats)])
    cfg = cfg or SihConfig()
    for _ in range(2):
        if out is None:
            cap = capacity if capacity is not None else 2 * n + 1024
            out = torch.empty(cap, dtype=local_data.dtype, device=local_data.device)
        oc = _U64(0)
        st = SihStats()
        rc = fn(e.handle, comm.handle if comm else None, _ptr(local_data), n, _ptr(out), out.numel(),
                C.byref(oc), C.byref(cfg), C.byref(st))
        if rc == 6 and capacity is None:
            out = torch.empty(int(oc.value), dtype=local_data.dtype, device=local_data.device)
            continue
        _check(rc, int(oc.value))
        return out[: oc.value], st
    raise CapacityError("sihsort: capacity retry failed", 0)


def sihsort_host(local_data: np.ndarray, comm: NcclComm | None = None, cfg: SihConfig | None = None,
                 ex: ExecBackend | None = None, out: np.ndarray | None = None):
    """sihsort on host arrays: H2D, device sort + exchange, D2H inside one C-ABI call."""
    local_data = np.ascontiguousarray(local_data)
    s = _NP_SUFFIX[local_data.dtype]
    e = _ex(ex)
    if out is None:
        out = np.empty(2 * local_data.size + 1024, dtype=local_data.dtype)
    fn = _fn(f"ak_sihsort_host_{s}", [_P, _P, _P, _U64, _P, _U64, C.POINTER(_U64), C.POINTER(SihConfig),
                                       C.POINTER(SihStats)])
    oc = _U64(0)
    st = SihStats()
    cfg = cfg or SihConfig()
    _check(fn(e.handle, comm.handle if comm else None, local_data.ctypes.data, local_data.size,
              out.ctypes.data, out.size, C.byref(oc), C.byref(cfg), C.byref(st)), int(oc.value))
    return out[: oc.value], st


def sihsort_loopback(inputs: list[torch.Tensor], cfg: SihConfig | None = None, capacity: int | None = None):
    """P logical ranks on ONE GPU (the reference's sim::world + run_ranks,
    sim_comm.hpp:190-218): host-level collectives, device slice copies.
    Returns (list of per-rank outputs, list of SihStats)."""
    P = len(inputs)
    if P < 1:
        raise InvalidArgument("world: rank count must be >= 1")
    dt = inputs[0].dtype
    for t in inputs:
        _dev(t, "sihsort_loopback")
        if t.dtype != dt:
            raise InvalidArgument("sihsort_loopback: all ranks need one dtype")
    s = _suffix(inputs[0])
    dev = inputs[0].device.index or 0
    total = sum(t.numel() for t in inputs)
    cap = capacity if capacity is not None else total + 1024
    outs = [torch.empty(cap, dtype=dt, device=inputs[0].device) for _ in range(P)]
    in_p = (_P * P)(*[t.data_ptr() for t in inputs])
    out_p = (_P * P)(*[t.data_ptr() for t in outs])
    ns = (_U64 * P)(*[t.numel() for t in inputs])
    caps = (_U64 * P)(*[cap] * P)
    oc = (_U64 * P)()
    stats = (SihStats * P)()
    cfg = cfg or SihConfig()
    fn = _fn(f"ak_sihsort_loopback_{s}", [C.c_int, _U64, _P, _P, _P, _P, _P, C.POINTER(SihConfig), _P])
    _check(fn(dev, P, C.cast(in_p, _P), C.cast(ns, _P), C.cast(out_p, _P), C.cast(caps, _P), C.cast(oc, _P),
              C.byref(cfg), C.cast(stats, _P)), max(oc) if P else 0)
    return [outs[r][: oc[r]] for r in range(P)], [stats[r] for r in range(P)]


def sihsort_perm(local_data: torch.Tensor, comm: NcclComm | None = None, cfg: SihConfig | None = None,
                 ex: ExecBackend | None = None, capacity: int | None = None):
    """Distributed sortperm (new: the reference sihsort is keys-only, sihsort.hpp:472-501):
    SIHSort of (key, global index) pairs. Rank r's key i has global index sum of the lower
    ranks' counts + i. Returns (this rank's keys, their global indices as int64, SihStats);
    the ranks' outputs concatenated are the globally stable sort order and its permutation."""
    _dev(local_data, "sihsort_perm")
    e = _ex(ex, local_data)
    n = local_data.numel()
    s = _suffix(local_data)
    fn = _fn(f"ak_sihsort_perm_{s}", [_P, _P, _P, _U64, _P, _P, _U64, C.POINTER(_U64), C.POINTER(SihConfig),
                                       C.POINTER(SihStats)])
    cfg = cfg or SihConfig()
    cap = capacity if capacity is not None else 2 * n + 1024
    for _ in range(2):
        out = torch.empty(cap, dtype=local_data.dtype, device=local_data.device)
        idx = torch.empty(cap, dtype=torch.int64, device=local_data.device)
        oc = _U64(0)
        st = SihStats()
        rc = fn(e.handle, comm.handle if comm else None, _ptr(local_data), n, _ptr(out), _ptr(idx), cap,
                C.byref(oc), C.byref(cfg), C.byref(st))
        if rc == 6 and capacity is None:
            cap = int(oc.value)
            continue
        _check(rc, int(oc.value))
        return out[: oc.value], idx[: oc.value], st
    raise CapacityError("sihsort_perm: capacity retry failed", 0)


def sihsort_perm_loopback(inputs: list[torch.Tensor], cfg: SihConfig | None = None, capacity: int | None = None):
    """sihsort_perm over P logical ranks on ONE GPU (loopback world). Returns (list of per-rank
    keys, list of per-rank global indices (int64), list of SihStats)."""
    P = len(inputs)
    if P < 1:
        raise InvalidArgument("world: rank count must be >= 1")
    dt = inputs[0].dtype
    for t in inputs:
        _dev(t, "sihsort_perm_loopback")
        if t.dtype != dt:
            raise InvalidArgument("sihsort_perm_loopback: all ranks need one dtype")
    s = _suffix(inputs[0])
    dev = inputs[0].device.index or 0
    total = sum(t.numel() for t in inputs)
    cap = capacity if capacity is not None else total + 1024
    outs = [torch.empty(cap, dtype=dt, device=inputs[0].device) for _ in range(P)]
    idxs = [torch.empty(cap, dtype=torch.int64, device=inputs[0].device) for _ in range(P)]
    in_p = (_P * P)(*[t.data_ptr() for t in inputs])
    out_p = (_P * P)(*[t.data_ptr() for t in outs])
    idx_p = (_P * P)(*[t.data_ptr() for t in idxs])
    ns = (_U64 * P)(*[t.numel() for t in inputs])
    caps = (_U64 * P)(*[cap] * P)
    oc = (_U64 * P)()
    stats = (SihStats * P)()
    cfg = cfg or SihConfig()
    fn = _fn(f"ak_sihsort_perm_loopback_{s}", [C.c_int, _U64, _P, _P, _P, _P, _P, _P, C.POINTER(SihConfig), _P])
    _check(fn(dev, P, C.cast(in_p, _P), C.cast(ns, _P), C.cast(out_p, _P), C.cast(idx_p, _P), C.cast(caps, _P),
              C.cast(oc, _P), C.byref(cfg), C.cast(stats, _P)), max(oc) if P else 0)
    return ([outs[r][: oc[r]] for r in range(P)], [idxs[r][: oc[r]] for r in range(P)],
            [stats[r] for r in range(P)])


_DTYPE_CODE = {np.dtype(np.int32): 2, np.dtype(np.int64): 3, np.dtype(np.float32): 5,
               np.dtype(np.float64): 6, np.dtype(np.uint64): 7, np.dtype(np.uint32): 8}


def bench_keys(seed: int, rank: int, n: int, dtype=np.int64, out: np.ndarray | None = None) -> np.ndarray:
    """Per-rank keys of the reference bench (bench.cpp:44-58, :164-173), generated by
    std::mt19937_64 in the C++ library: identical to the reference's inputs."""
    dt = np.dtype(dtype)
    if out is None:
        out = np.empty(n, dtype=dt)
    _check(_fn("ak_bench_keys", [_U64, _U64, _U64, C.c_int, _P])(seed, rank, n, _DTYPE_CODE[dt], out.ctypes.data))
    return out


def version() -> str:
    return _lib.ak_version().decode()
