"""P-way merge (K8) timing: P sorted int64 runs totalling 2^log2n keys, one-pass merge_runs
vs the log2(P)-level pairwise merge tree it replaced (modelled with merge_runs on 2 runs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2507_16710_b200 as ak
log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
ex = ak.ExecBackend(0)
n = 1 << log2n
for P in (2, 4, 8):
    runs = [torch.sort(torch.randint(-2**62, 2**62, (n // P,), device="cuda"))[0] for _ in range(P)]
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    scr = torch.empty_like(out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ak.merge_runs(runs, out=out, scratch=scr, ex=ex)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0.record(ex.stream); ak.merge_runs(runs, out=out, scratch=scr, ex=ex); e1.record(ex.stream)
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    print(f"merge_runs P={P} 2^{log2n} int64: {ms:.3f} ms = {16 * n / ms / 1e6:.0f} GB/s (16 B/key)", flush=True)
    del runs
# family breakdown of one P=8 merge
P = 8
runs = [torch.sort(torch.randint(-2**62, 2**62, (n // P,), device="cuda"))[0] for _ in range(P)]
out = torch.empty(n, dtype=torch.int64, device="cuda"); scr = torch.empty_like(out)
ak.merge_runs(runs, out=out, scratch=scr, ex=ex)
ex.reset_kernel_time(); ex.set_profiling(True)
ak.merge_runs(runs, out=out, scratch=scr, ex=ex)
ex.set_profiling(False)
print("families:", {k: ex.kernel_time(k) for k in ("merge", "onesweep", "local", "hist", "other")})
