"""ak_bench: the reference benchmark CLI's sorting subcommands (proj/tools/bench_main.cpp) on
the B200 build -- same subcommands, options, exit codes, record table, CSV and sihsort-sim
stats block; rank inputs from the reference generator or SIHS fixtures.
"""
import csv
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_2507_16710_b200", "bin", "ak_bench")

pytestmark = pytest.mark.skipif(not os.path.exists(EXE), reason="ak_bench not built (make -C paper_2507_16710_b200/csrc)")


def run(*args, timeout=600):
    return subprocess.run([EXE, *map(str, args)], capture_output=True, text=True, timeout=timeout)


@pytest.mark.parametrize("args,msg", [
    ([], "subcommand is required"),
    (["rbf"], "outside the B200 build"),
    (["sort-weak", "--reps", "2"], "--reps must be >= 3"),
    (["sort-weak", "--warmup", "0"], "--warmup must be >= 1"),
    (["sort-weak", "--n", "5"], "unknown option --n"),
    (["sort-strong", "--transport", "mpi"], "--transport"),
    (["sihsort-sim", "--dtype", "i128"], "no device sort"),
])
def test_usage_errors_exit_2(args, msg):
    r = run(*args)
    assert r.returncode == 2
    assert msg in r.stderr


def stats_of(stdout):
    kv = {}
    for line in stdout.splitlines():
        if "=" in line and " " not in line:
            k, v = line.split("=", 1)
            kv[k] = v
    return kv


@pytest.mark.gpu
def test_sihsort_sim_matches_oracle_per_rank(orc, tmp_path):
    P, n = 4, 100_000
    fx = tmp_path / "fx"
    r = run("sihsort-sim", "--dtype", "i64", "--ranks", P, "--per-rank", n, "--reps", 3, "--save-fixtures", fx)
    assert r.returncode == 0, r.stderr
    st = stats_of(r.stdout)
    assert st["case"] == "sihsort-sim" and st["ranks"] == str(P) and st["total_elements"] == str(P * n)
    # the same inputs through the C oracle: identical per-rank output sizes and message counts
    import paper_2507_16710_b200 as ak
    ins = [ak.bench_keys(42, q, n, np.int64) for q in range(P)]
    want, wstats, _ = orc.sihsort(ins)
    for q in range(P):
        assert int(st[f"out_count_rank_{q}"]) == want[q].size
        assert int(st[f"msg_count_rank_{q}"]) == wstats[q]["redistribution_sends"]
        assert int(st[f"collectives_rank_{q}"]) == wstats[q]["collective_ops"]
    # reloading the saved fixtures reproduces the run
    r2 = run("sihsort-sim", "--dtype", "i64", "--ranks", P, "--reps", 3, "--load-fixtures", fx)
    assert r2.returncode == 0, r2.stderr
    st2 = stats_of(r2.stdout)
    assert all(st2[f"out_count_rank_{q}"] == st[f"out_count_rank_{q}"] for q in range(P))
    # a fixture for the wrong dtype is a runtime failure (exit 1)
    r3 = run("sihsort-sim", "--dtype", "f64", "--ranks", P, "--reps", 3, "--load-fixtures", fx)
    assert r3.returncode == 1 and "dtype mismatch" in r3.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("extra", [[], ["--device-resident"], ["--transport", "nccl"]])
def test_sort_weak_strong_csv(tmp_path, extra):
    out = tmp_path / "r.csv"
    r = run("sort-weak", "--dtype", "u64", "--ranks", "1" if "nccl" in extra else "1,2", "--per-rank", 200_000,
            "--reps", 3, "--csv", out, *extra)
    assert r.returncode == 0, r.stderr
    rows = list(csv.DictReader(open(out)))
    assert rows and rows[0]["case"] == "sort-weak" and rows[0]["dtype"] == "u64" and rows[0]["n"] == "200000"
    assert float(rows[0]["throughput_gbps"]) > 0
    r = run("sort-strong", "--dtype", "f32", "--n", 1_000_003, "--ranks", 1, "--reps", 3, *extra)
    assert r.returncode == 0, r.stderr
    assert "sort-strong" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("ranks", [2, 4, 8])
def test_sort_weak_nccl_multi_gpu(orc, ranks):
    """ak_bench with one rank per GPU over NCCL (thread per GPU, one process): per-rank output
    counts and message counts equal the oracle's (skipped below `ranks` GPUs)."""
    import torch
    if torch.cuda.device_count() < ranks:
        pytest.skip(f"needs {ranks} GPUs")
    n = 1 << 20
    r = run("sihsort-sim", "--dtype", "i64", "--ranks", ranks, "--per-rank", n, "--reps", 3, "--transport", "nccl")
    assert r.returncode == 0, r.stderr
    st = stats_of(r.stdout)
    import paper_2507_16710_b200 as ak
    want, wstats, _ = orc.sihsort([ak.bench_keys(42, q, n, np.int64) for q in range(ranks)])
    for q in range(ranks):
        assert int(st[f"out_count_rank_{q}"]) == want[q].size
        assert int(st[f"msg_count_rank_{q}"]) == wstats[q]["redistribution_sends"]
