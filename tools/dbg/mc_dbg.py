import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2507_16710_b200 as ak
ex = ak.ExecBackend(0)
P = int(sys.argv[1]); n = 1 << int(sys.argv[2])
g = torch.Generator(device="cuda").manual_seed(1)
runs = [torch.sort(torch.randint(-2**62, 2**62, (n // P,), device="cuda", generator=g))[0] for _ in range(P)]
out = torch.empty(n, dtype=torch.int64, device="cuda"); scr = torch.empty_like(out)
ex.reset_kernel_time(); ex.set_profiling(True)
ak.merge_runs(runs, out=out, scratch=scr, ex=ex)
ex.set_profiling(False)
want = torch.sort(torch.cat(runs))[0]
print("P", P, "n", n, "equal", bool(torch.equal(out, want)), "merge fam", ex.kernel_time("merge"), "local", ex.kernel_time("local"))
