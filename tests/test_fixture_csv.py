"""On-disk formats either side of the sort path: SIHS per-rank input
fixtures and the benchmark CSV, written by the B200 build's headers (include/ak/fixture.hpp,
csv.hpp) and by the reference itself (src/fixture.cpp, src/csv.cpp compiled in place into
oracle/_ref) -- each must read the other's files, and CSV output must be byte-identical.
No GPU needed.
"""
import ctypes as C
import os
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GXX = shutil.which("g++")


@pytest.fixture(scope="module")
def tool(tmp_path_factory):
    if GXX is None:
        pytest.skip("g++ not available")
    exe = str(tmp_path_factory.mktemp("fcsv") / "fixture_csv")
    r = subprocess.run([GXX, "-std=c++20", "-O1", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "fixture_csv.cpp"), "-o", exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


@pytest.fixture(scope="module")
def ref(orc):
    if not orc.ref_available():
        pytest.skip("oracle/_ref (the reference compiled in place) not built")
    lib = orc.ref()
    if not hasattr(lib, "ref_read_fixture_i64"):
        pytest.skip("oracle/_ref predates the fixture shim")
    return lib


NP = {"i32": np.int32, "i64": np.int64, "f32": np.float32, "f64": np.float64}


def run(tool, *args):
    r = subprocess.run([tool, *map(str, args)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return r.stdout


def digest(a):
    s = 0
    for b in a.view(np.uint32 if a.itemsize == 4 else np.uint64).astype(np.uint64):
        s = (s * 1099511628211 + int(b)) % (1 << 64)
    return s


@pytest.mark.parametrize("dt", ["i32", "i64", "f32", "f64"])
def test_ours_written_reference_read(tool, ref, tmp_path, dt):
    path = str(tmp_path / "rank_3.sihs")
    run(tool, "write", path, 3, dt, 1001, 42)
    rank, n = C.c_uint32(), C.c_uint64()
    out = np.empty(1001, NP[dt])
    fn = getattr(ref, f"ref_read_fixture_{dt}")
    fn.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]
    assert fn(path.encode(), C.byref(rank), out.ctypes.data, out.size, C.byref(n)) == 0
    assert rank.value == 3 and n.value == 1001
    r, cnt, s = run(tool, "read", path, dt).split()
    assert int(cnt) == 1001 and digest(out) == int(s)


@pytest.mark.parametrize("dt", ["i32", "i64", "f32", "f64"])
def test_reference_written_ours_read(tool, ref, tmp_path, dt):
    path = str(tmp_path / "rank_5.sihs")
    x = (np.arange(777) * 2654435761 % 100003 - 50000).astype(NP[dt])
    fn = getattr(ref, f"ref_write_fixture_{dt}")
    fn.argtypes = [C.c_char_p, C.c_uint32, C.c_void_p, C.c_uint64]
    assert fn(path.encode(), 5, x.ctypes.data, x.size) == 0
    r, cnt, s = run(tool, "read", path, dt).split()
    assert int(r) == 5 and int(cnt) == 777 and int(s) == digest(x)


def test_u64_fixture_roundtrip_and_reference_rejects_new_code(tool, ref, tmp_path):
    # u64 (code 7) is new in this build: our reader round-trips it; the reference reader
    # rejects the unknown code instead of misreading it
    path = str(tmp_path / "rank_0.sihs")
    run(tool, "write", path, 0, "u64", 50, 9)
    assert run(tool, "read", path, "u64").split()[1] == "50"
    rank, n = C.c_uint32(), C.c_uint64()
    out = np.empty(50, np.int64)
    ref.ref_read_fixture_i64.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]
    assert ref.ref_read_fixture_i64(path.encode(), C.byref(rank), out.ctypes.data, 50, C.byref(n)) != 0


def test_dtype_mismatch_and_bad_magic(tool, tmp_path):
    path = str(tmp_path / "x.sihs")
    run(tool, "write", path, 0, "i32", 10, 1)
    r = subprocess.run([tool, "read", path, "i64"], capture_output=True, text=True)
    assert r.returncode == 1 and "dtype mismatch" in r.stderr
    with open(path, "r+b") as f:
        f.write(b"XXXX")
    r = subprocess.run([tool, "read", path, "i32"], capture_output=True, text=True)
    assert r.returncode == 1 and "bad magic" in r.stderr


def test_csv_byte_identical_to_reference(tool, ref, tmp_path):
    ours = str(tmp_path / "ours.csv")
    theirs = str(tmp_path / "ref.csv")
    run(tool, "csv", ours)
    recs = [("sort-weak", "i64", 100000, 1, 5, 1.25, 0.015625, 0.64, 1.25),
            ("sihsort-sim", "f32", 268435456, 8, 3, 12.345678901234, 0.1, 1234.5678901, 271.6),
            ('odd,"name"', "u64", 7, 2, 3, 1e-9, 0.0, 3.14159265358979, 2.0)]
    # the reference's emit_csv is called from a numpy-free interpreter: inside this process
    # (numpy's OpenBLAS loaded) its stream formatting crashes, which says nothing about
    # either implementation
    prog = (
        "import ctypes as C, sys\n"
        f"ref = C.CDLL({os.path.join(ROOT, 'oracle', '_ref', 'libakref.so')!r})\n"
        f"recs = {recs!r}\n"
        "k = len(recs)\n"
        "cs = (C.c_char_p * k)(*[r[0].encode() for r in recs]); ds = (C.c_char_p * k)(*[r[1].encode() for r in recs])\n"
        "u = [(C.c_uint64 * k)(*[r[i] for r in recs]) for i in (2, 3, 4)]\n"
        "d = [(C.c_double * k)(*[r[i] for r in recs]) for i in (5, 6, 7, 8)]\n"
        "ref.ref_emit_csv.argtypes = [C.c_char_p, C.c_int] + [C.c_void_p] * 9\n"
        "sys.exit(ref.ref_emit_csv(sys.argv[1].encode(), k, C.cast(cs, C.c_void_p), C.cast(ds, C.c_void_p),"
        " *[C.cast(a, C.c_void_p) for a in u], *[C.cast(a, C.c_void_p) for a in d]))\n")
    r = subprocess.run(["python3", "-c", prog, theirs], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    assert run(tool, "parse", theirs) == open(theirs).read()
