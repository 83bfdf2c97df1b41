"""The C++ drop-in headers (include/ak/*.hpp) against the reference's own test cases.

CPU: the headers compile with g++ -std=c++20 (as the reference's tests do) and reject,
at compile time, callables that cannot cross the C ABI (no CPU fallback).
GPU: tests/cpp/test_dropin.cpp runs the reference's test_primitives.cpp cases and the SPEC
known answers through the headers -> libak_cuda.so on the B200.
"""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2507_16710_b200", "lib")
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
GXX = shutil.which("g++")

pytestmark = pytest.mark.skipif(GXX is None, reason="g++ not available")


def _compile(src_text_or_path, out, link=True):
    args = [GXX, "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include")]
    if isinstance(src_text_or_path, str) and os.path.exists(src_text_or_path):
        args.append(src_text_or_path)
    else:
        args += ["-x", "c++", "-"]
    if link:
        args += ["-L", LIBDIR, "-lak_cuda", f"-Wl,-rpath,{LIBDIR}", "-lpthread", "-o", out]
    else:
        args += ["-fsyntax-only"]
    inp = None if os.path.exists(str(src_text_or_path)) else src_text_or_path
    return subprocess.run(args, input=inp, capture_output=True, text=True)


def test_headers_compile(tmp_path):
    r = _compile(SRC, str(tmp_path / "t"), link=False)
    assert r.returncode == 0, r.stderr


@pytest.mark.parametrize("snippet", [
    # a generic lambda comparator cannot cross the C ABI
    "std::vector<int> v{3,1}; auto b = ak::sort_buffers<int>::with_capacity(2);"
    "ak::merge_sort(std::span<int>(v), b, ak::exec_backend::cuda(), [](int a, int c){ return a < c; });",
    # a lambda reduction operator likewise
    "std::vector<int> v{3,1}; (void)ak::reduce<int>([](int a, int c){ return a + c; }, v, {0, 256},"
    " ak::exec_backend::cuda());",
    # unsupported key type (the reference's dtype.hpp list is i16/i32/i64/i128/f32/f64)
    "std::vector<unsigned char> v{3,1}; auto b = ak::sort_buffers<unsigned char>::with_capacity(2);"
    "ak::merge_sort(std::span<unsigned char>(v), b, ak::exec_backend::cuda());",
])
def test_unsupported_callables_are_compile_errors(snippet):
    src = ('#include "ak/sort.hpp"\n#include "ak/reduce.hpp"\n#include <vector>\n'
           f"int main() {{ {snippet} return 0; }}\n")
    r = _compile(src, None, link=False)
    assert r.returncode != 0
    assert "B200 build" in r.stderr


@pytest.mark.gpu
def test_dropin_reference_cases(tmp_path):
    assert os.path.exists(os.path.join(LIBDIR, "libak_cuda.so")), "libak_cuda.so not built"
    exe = str(tmp_path / "test_dropin")
    r = _compile(SRC, exe)
    assert r.returncode == 0, r.stderr
    run = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert run.returncode == 0, run.stdout + run.stderr
    assert "0 failures" in run.stdout
