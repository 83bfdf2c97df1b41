"""Device time of one merge_sort of uniform 64-bit keys per size (CUDA events around the public
API call, median of 5 after one warm-up), with an on-device sortedness check.

    python tools/sort_sizes.py 24 26 28 30 30:u64      # log2(n)[:i64|u64]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_16710_b200 as ak  # noqa: E402

ex = ak.ExecBackend(0)
for arg in sys.argv[1:] or ["28"]:
    lg, dt = arg.split(":") if ":" in arg else (arg, "i64")
    n = 1 << int(lg)
    g = torch.Generator(device="cuda")
    g.manual_seed(int(lg))
    x = torch.randint(-(1 << 63), (1 << 63) - 1, (n,), dtype=torch.int64, device="cuda", generator=g)
    w, s = torch.empty_like(x), torch.empty_like(x)
    wv, sv = (w.view(torch.uint64), s.view(torch.uint64)) if dt == "u64" else (w, s)
    ts = []
    for r in range(6):
        w.copy_(x)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ak.merge_sort(wv, sv, ex)
        b.record()
        torch.cuda.synchronize()
        if r:
            ts.append(a.elapsed_time(b))
    y = w ^ (-(1 << 63)) if dt == "u64" else w
    ok = bool((y[1:] >= y[:-1]).all())
    ts.sort()
    med = ts[len(ts) // 2]
    print(f"{dt} 2^{lg}: median {med:.3f} ms (min {ts[0]:.3f}) = {n * 8 / med / 1e6:.0f} GB/s of keys, sorted={ok}",
          flush=True)
    del x, w, s, wv, sv
    torch.cuda.empty_cache()
