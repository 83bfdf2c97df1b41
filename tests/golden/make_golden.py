"""Record golden vectors from the REFERENCE itself (oracle/_ref/libakref.so, compiled in
place from /root/reference/proj by oracle/Makefile). Run here (the reference exists in
this container); the .npz fixtures are committed and travel to the GPU box.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def keys(rng, dt, n):
    dt = np.dtype(dt)
    if dt.kind == "f":
        x = rng.uniform(-1e6, 1e6, n).astype(dt)
        x[rng.integers(0, n, n // 8)] = 0.0
        x[rng.integers(0, n, n // 8)] = -0.0
        x[rng.integers(0, n, n // 8)] = x[0]
        return x
    info = np.iinfo(dt)
    x = rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)
    x[rng.integers(0, n, n // 8)] = x[1]
    return x


def main():
    if not oracle.ref_available():
        raise SystemExit("oracle/_ref/libakref.so missing: run `make -C oracle` where /root/reference exists")
    rng = np.random.default_rng(20250716)
    out = {}
    for dt in (np.int32, np.uint32, np.int64, np.uint64, np.float32, np.float64):
        s = np.dtype(dt).name
        x = keys(rng, dt, 3001)
        out[f"sort_{s}_in"] = x
        out[f"sort_{s}_asc"] = oracle.ref_merge_sort(x, threads=3)
        out[f"sort_{s}_desc"] = oracle.ref_merge_sort(x, threads=2, descending=True)
        out[f"sortperm_{s}_u64"] = oracle.ref_sortperm(x, np.uint64, threads=4)
        out[f"sortperm_{s}_i32_desc"] = oracle.ref_sortperm(x, np.int32, threads=2, descending=True)
        out[f"sortperm_lowmem_{s}_u64"] = oracle.ref_sortperm(x, np.uint64, threads=4, lowmem=True)
        pay = np.arange(x.size, dtype=np.int32)[::-1].copy()
        k, v = oracle.ref_merge_sort_by_key(x, pay, threads=3)
        out[f"bykey_{s}_keys"], out[f"bykey_{s}_payload_in"], out[f"bykey_{s}_payload"] = k, pay, v
    # signed zero case
    z = np.array([0.0, -0.0, 1, -0.0, 0.0, -1], dtype=np.float32)
    out["signed_zero_in"] = z
    out["signed_zero_sortperm"] = oracle.ref_sortperm(z)
    # reduce / accumulate: ints U[-10000, 10000] (tests/test_utils.hpp:30-33)
    xi = rng.integers(-10000, 10001, 20_000).astype(np.int64)
    out["reduce_i64_in"] = xi
    out["reduce_i64_sum"] = np.array([oracle.ref_reduce(xi, "sum", threads=8)], dtype=np.int64)
    out["reduce_i64_min"] = np.array([oracle.ref_reduce(xi, "min", threads=8)], dtype=np.int64)
    out["reduce_i64_max"] = np.array([oracle.ref_reduce(xi, "max", threads=8)], dtype=np.int64)
    out["scan_i64_incl"] = oracle.ref_accumulate(xi, True, 0, 7, threads=8)
    out["scan_i64_excl"] = oracle.ref_accumulate(xi, False, 0, 1024, threads=2)
    xs = rng.integers(-10000, 10001, 5000).astype(np.int32)
    out["scan_i32_init100_in"] = xs
    out["scan_i32_init100"] = oracle.ref_accumulate(xs, True, 100, 64, threads=8)
    xf = rng.uniform(0, 1, 20_000).astype(np.float32)
    out["reduce_f32_in"] = xf
    out["reduce_f32_sum_ref"] = np.array([oracle.ref_reduce(xf, "sum", threads=8)], dtype=np.float32)
    # searchsorted (tests/test_primitives.cpp:177-195 shape)
    hay = np.sort(rng.integers(-10000, 10001, 2000).astype(np.int32))
    nd = rng.integers(-10000, 10001, 500).astype(np.int32)
    out["search_hay"], out["search_needles"] = hay, nd
    out["search_first"] = oracle.ref_searchsorted(hay, nd, "first", threads=4)
    out["search_last"] = oracle.ref_searchsorted(hay, nd, "last", threads=4)
    # sihsort over sim::world: uniform P=4 and P=8, zipf P=4, all-equal P=4
    cases = {
        "sih_uniform_p4": [keys(rng, np.int64, 2500 + 37 * r) for r in range(4)],
        "sih_uniform_p8": [keys(rng, np.int64, 1200) for r in range(8)],
        "sih_zipf_p4": [np.minimum(rng.zipf(1.1, 2000), 10**6).astype(np.int64) for _ in range(4)],
        "sih_equal_p4": [np.full(1000, 5, dtype=np.int64) for _ in range(4)],
        "sih_u64_p3": [keys(rng, np.uint64, 1500) for _ in range(3)],
        "sih_f64_p4": [keys(rng, np.float64, 1500) for _ in range(4)],
    }
    for name, ins in cases.items():
        outs, stats = oracle.ref_sihsort(ins, threads_per_rank=2)
        for r, (a, b) in enumerate(zip(ins, outs)):
            out[f"{name}_in{r}"] = a
            out[f"{name}_out{r}"] = b
        out[f"{name}_stats"] = np.array([[s["rounds_used"], s["converged"], s["max_deviation"],
                                          s["redistribution_sends"], s["redistribution_bytes"],
                                          s["collective_ops"], s["output_count"]] for s in stats], dtype=np.float64)
        out[f"{name}_P"] = np.array([len(ins)])
    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
