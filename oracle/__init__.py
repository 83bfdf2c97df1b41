"""ctypes access to the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Two libraries live here:

* ``liboracle.so`` -- ``oracle/ak_oracle.c``, a plain-C restatement of the
  reference hot path (sort.hpp, reduce.hpp, scan.hpp, search.hpp, sihsort.hpp
  of /root/reference/proj), each function citing the file:line it follows.
* ``_ref/libakref.so`` -- the reference library itself, compiled in place from
  /root/reference/proj by ``oracle/Makefile`` through ``oracle/ref_shim.cpp``.
  It pins the restatement (tests/test_oracle.py) and is the reference CPU arm
  of bench.py.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package. The product package
``paper_2507_16710_b200`` never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libakref.so")

_u64 = C.c_uint64
_p = C.c_void_p

SUFFIX = {np.dtype(np.int32): "i32", np.dtype(np.uint32): "u32", np.dtype(np.int64): "i64",
          np.dtype(np.uint64): "u64", np.dtype(np.float32): "f32", np.dtype(np.float64): "f64"}


def build() -> None:
    """Compile liboracle.so (always) and _ref/libakref.so (when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


_orc = None
_ref = None


def lib() -> C.CDLL:
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            build()
        _orc = C.CDLL(ORACLE_SO)
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError("oracle/_ref/libakref.so not built (needs /root/reference at build time)")
        _ref = C.CDLL(REF_SO)
    return _ref


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class SihConfig(C.Structure):
    _fields_ = [("sample_per_rank", _u64), ("bins", _u64), ("max_refine_rounds", _u64),
                ("imbalance_tol", C.c_double)]


class SihStats(C.Structure):
    _fields_ = [("rounds_used", _u64), ("converged", _u64), ("max_deviation", C.c_double),
                ("redistribution_sends", _u64), ("redistribution_bytes", _u64),
                ("collective_ops", _u64), ("output_count", _u64)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


def default_config() -> SihConfig:
    return SihConfig(0, 0, 4, 0.25)


# ----------------------------------------------------------------------------- oracle (C)

def sortperm(data: np.ndarray, descending: bool = False) -> np.ndarray:
    data = np.ascontiguousarray(data)
    out = np.empty(data.size, dtype=np.uint64)
    fn = getattr(lib(), "orc_sortperm_" + SUFFIX[data.dtype])
    fn.argtypes = [_p, _u64, _p, C.c_int]
    if fn(_ptr(data), data.size, _ptr(out), int(descending)) != 0:
        raise MemoryError("oracle sortperm")
    return out


def merge_sort(data: np.ndarray, descending: bool = False) -> np.ndarray:
    out = np.array(data, copy=True)
    fn = getattr(lib(), "orc_merge_sort_" + SUFFIX[out.dtype])
    fn.argtypes = [_p, _u64, C.c_int]
    if fn(_ptr(out), out.size, int(descending)) != 0:
        raise MemoryError("oracle merge_sort")
    return out


def merge_sort_by_key(keys: np.ndarray, payload: np.ndarray, descending: bool = False):
    perm = sortperm(keys, descending)
    return keys[perm], payload[perm]


_REDUCE_RET = {"i32": C.c_int32, "i64": C.c_int64, "u64": C.c_uint64, "f32_f64acc": C.c_double,
               "f64": C.c_double}


def reduce(data: np.ndarray, op: str = "sum", mapf: str = "identity", init=None):
    """Sequential fold (tests/test_utils.hpp:64-71); f32 accumulates in double."""
    data = np.ascontiguousarray(data)
    suf = SUFFIX[data.dtype]
    if suf == "f32":
        suf = "f32_f64acc"
    opi = {"sum": 0, "min": 1, "max": 2}[op]
    mi = {"identity": 0, "abs": 1, "square": 2}[mapf]
    if init is None:
        init = _neutral(data.dtype, op)
    fn = getattr(lib(), "orc_reduce_" + suf)
    ret = _REDUCE_RET[suf]
    fn.restype = ret
    fn.argtypes = [_p, _u64, C.c_int, C.c_int, ret]
    return fn(_ptr(data), data.size, opi, mi, init)


def _neutral(dt: np.dtype, op: str):
    if op == "sum":
        return 0
    if dt.kind == "f":
        return float("inf") if op == "min" else float("-inf")
    info = np.iinfo(dt)
    return int(info.max) if op == "min" else int(info.min)


def scan(data: np.ndarray, inclusive: bool = True, init=0) -> np.ndarray:
    """Sequential scan (tests/test_utils.hpp:74-88). f32 input -> float64 prefix."""
    data = np.ascontiguousarray(data)
    suf = SUFFIX[data.dtype]
    if suf == "f32":
        out = np.empty(data.size, dtype=np.float64)
        fn = lib().orc_scan_f32_f64acc
        fn.argtypes = [_p, _u64, _p, C.c_int, C.c_double]
    elif suf == "f64":
        out = np.empty(data.size, dtype=np.float64)
        fn = lib().orc_scan_f64
        fn.argtypes = [_p, _u64, _p, C.c_int, C.c_double]
    else:
        out = np.empty_like(data)
        fn = getattr(lib(), "orc_scan_" + suf)
        fn.argtypes = [_p, _u64, _p, C.c_int, C.c_int64 if suf == "i64" else C.c_int32]
    fn(_ptr(data), data.size, _ptr(out), int(inclusive), init)
    return out


def searchsorted(hay: np.ndarray, needles: np.ndarray, side: str = "first",
                 descending: bool = False) -> np.ndarray:
    hay = np.ascontiguousarray(hay)
    needles = np.ascontiguousarray(needles, dtype=hay.dtype)
    out = np.empty(needles.size, dtype=np.uint64)
    fn = getattr(lib(), "orc_searchsorted_" + SUFFIX[hay.dtype])
    fn.argtypes = [_p, _u64, _p, _u64, C.c_int, C.c_int, _p]
    fn(_ptr(hay), hay.size, _ptr(needles), needles.size, int(side == "last"), int(descending),
       _ptr(out))
    return out


def sample_positions(n: int, k: int) -> np.ndarray:
    pos = np.empty(max(k, 1), dtype=np.uint64)
    fn = lib().orc_sample_positions
    fn.restype = _u64
    fn.argtypes = [_u64, _u64, _p]
    m = fn(n, k, _ptr(pos))
    return pos[:m]


def _sihsort_call(lib_: C.CDLL, prefix: str, inputs, cfg, extra_threads=None):
    dt = inputs[0].dtype
    P = len(inputs)
    arrs = [np.ascontiguousarray(a, dtype=dt) for a in inputs]
    counts = np.array([a.size for a in arrs], dtype=np.uint64)
    ptrs = (C.c_void_p * P)(*[a.ctypes.data for a in arrs])
    total = int(counts.sum())
    out = np.empty(max(total, 1), dtype=dt)
    out_counts = np.empty(P, dtype=np.uint64)
    stats = (SihStats * P)()
    spl = np.empty(max(P - 1, 1), dtype=dt)
    fn = getattr(lib_, prefix + SUFFIX[dt])
    fn.restype = C.c_int
    cfg = cfg or default_config()
    if extra_threads is None:
        fn.argtypes = [_u64, _p, _p, C.POINTER(SihConfig), _p, _p, _p, _p]
        rc = fn(P, C.cast(ptrs, _p), _ptr(counts), C.byref(cfg), _ptr(out), _ptr(out_counts),
                C.cast(stats, _p), _ptr(spl))
    else:
        fn.argtypes = [_u64, _p, _p, C.POINTER(SihConfig), _u64, _p, _p, _p]
        rc = fn(P, C.cast(ptrs, _p), _ptr(counts), C.byref(cfg), extra_threads, _ptr(out),
                _ptr(out_counts), C.cast(stats, _p))
    if rc != 0:
        raise RuntimeError(f"{prefix} failed rc={rc}")
    outs, base = [], 0
    for c in out_counts.tolist():
        outs.append(out[base:base + c].copy())
        base += c
    return outs, [s.as_dict() for s in stats], spl[:P - 1].copy()


def sihsort(inputs, cfg: SihConfig | None = None):
    """Oracle SIHSort over len(inputs) ranks -> (per-rank outputs, per-rank stats, splitters)."""
    return _sihsort_call(lib(), "orc_sihsort_", inputs, cfg)


# ----------------------------------------------------------------------------- reference (_ref)

def ref_merge_sort(data: np.ndarray, threads: int = 0, descending: bool = False) -> np.ndarray:
    out = np.array(data, copy=True)
    fn = getattr(ref(), "ref_merge_sort_" + SUFFIX[out.dtype])
    fn.argtypes = [_p, _u64, C.c_int, _u64]
    if fn(_ptr(out), out.size, int(descending), threads) != 0:
        raise RuntimeError("ref merge_sort")
    return out


def ref_sortperm(data: np.ndarray, index_dtype=np.uint64, threads: int = 0, lowmem: bool = False,
                 descending: bool = False) -> np.ndarray:
    data = np.ascontiguousarray(data)
    out = np.empty(data.size, dtype=index_dtype)
    isuf = "u64" if np.dtype(index_dtype) == np.uint64 else "i32"
    fn = getattr(ref(), f"ref_sortperm_{SUFFIX[data.dtype]}_{isuf}")
    fn.argtypes = [_p, _u64, _p, C.c_int, C.c_int, _u64]
    if fn(_ptr(data), data.size, _ptr(out), int(descending), int(lowmem), threads) != 0:
        raise RuntimeError("ref sortperm")
    return out


def ref_merge_sort_by_key(keys: np.ndarray, payload: np.ndarray, threads: int = 0,
                          descending: bool = False):
    k = np.array(keys, copy=True)
    v = np.array(payload, copy=True)
    isuf = "u64" if v.dtype == np.uint64 else "i32"
    fn = getattr(ref(), f"ref_merge_sort_by_key_{SUFFIX[k.dtype]}_{isuf}")
    fn.argtypes = [_p, _p, _u64, C.c_int, _u64]
    if fn(_ptr(k), _ptr(v), k.size, int(descending), threads) != 0:
        raise RuntimeError("ref merge_sort_by_key")
    return k, v


_REF_T = {"i32": C.c_int32, "i64": C.c_int64, "u64": C.c_uint64, "f32": C.c_float, "f64": C.c_double}


def ref_reduce(data: np.ndarray, op: str = "sum", init=None, threads: int = 0):
    data = np.ascontiguousarray(data)
    suf = SUFFIX[data.dtype]
    fn = getattr(ref(), "ref_reduce_" + suf)
    fn.restype = _REF_T[suf]
    fn.argtypes = [_p, _u64, C.c_int, _REF_T[suf], _u64]
    if init is None:
        init = _neutral(data.dtype, op)
    return fn(_ptr(data), data.size, {"sum": 0, "min": 1, "max": 2}[op], init, threads)


def ref_accumulate(data: np.ndarray, inclusive: bool = True, init=0, chunk: int = 4096,
                   threads: int = 0, out: np.ndarray | None = None) -> np.ndarray:
    data = np.ascontiguousarray(data)
    suf = SUFFIX[data.dtype]
    if out is None:
        out = np.empty_like(data)
    fn = getattr(ref(), "ref_accumulate_" + suf)
    fn.argtypes = [_p, _u64, _p, C.c_int, _REF_T[suf], _u64, _u64]
    if fn(_ptr(data), data.size, _ptr(out), int(inclusive), init, chunk, threads) != 0:
        raise RuntimeError("ref accumulate")
    return out


def ref_searchsorted(hay: np.ndarray, needles: np.ndarray, side: str = "first",
                     threads: int = 0) -> np.ndarray:
    hay = np.ascontiguousarray(hay)
    needles = np.ascontiguousarray(needles, dtype=hay.dtype)
    out = np.empty(needles.size, dtype=np.uint64)
    fn = getattr(ref(), "ref_searchsorted_" + SUFFIX[hay.dtype])
    fn.argtypes = [_p, _u64, _p, _u64, C.c_int, _p, _u64]
    if fn(_ptr(hay), hay.size, _ptr(needles), needles.size, int(side == "last"), _ptr(out),
          threads) != 0:
        raise RuntimeError("ref searchsorted")
    return out


def ref_sihsort(inputs, cfg: SihConfig | None = None, threads_per_rank: int = 0):
    """The reference sihsort over sim::world(P) + run_ranks (reference bench.cpp:146-162)."""
    outs, stats, _ = _sihsort_call(ref(), "ref_sihsort_", inputs, cfg, extra_threads=threads_per_rank)
    return outs, stats


def ref_bench_keys(seed: int, rank: int, n: int, dtype=np.int64, out: np.ndarray | None = None) -> np.ndarray:
    """Per-rank inputs of the reference bench (bench.cpp:44-62, :164-173) made inside oracle/_ref,
    so a process timing the reference never loads the product library."""
    dt = np.dtype(dtype)
    if out is None:
        out = np.empty(n, dtype=dt)
    fn = getattr(ref(), "ref_bench_keys_" + SUFFIX[dt])
    fn.argtypes = [_u64, _u64, _u64, _p]
    if fn(seed, rank, n, _ptr(out)) != 0:
        raise RuntimeError("ref bench_keys")
    return out


def ref_sortperm_bytes(n: int, key_bytes: int, index_bytes: int, lowmem: bool) -> int:
    fn = ref().ref_sortperm_bytes
    fn.restype = _u64
    fn.argtypes = [_u64, C.c_int, C.c_int, C.c_int]
    return int(fn(n, key_bytes, index_bytes, int(lowmem)))
