import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2507_16710_b200 as ak, oracle
ex = ak.ExecBackend.cuda(0)
fails = 0
for it in range(40):
  for dt in (np.int32, np.int64):
    for n in (100000, 1000000, 3000000):
        for inc in (True, False):
            rng = np.random.default_rng(n)
            x = rng.integers(-10000, 10001, n).astype(dt)
            got = ak.accumulate("sum", torch.from_numpy(x).cuda(), inclusive=inc, init=100, ex=ex).cpu().numpy()
            want = oracle.scan(x, inc, 100)
            bad = np.nonzero(got != want)[0]
            if len(bad):
                fails += 1
                d = (got[bad[:3]].astype(np.int64) - want[bad[:3]].astype(np.int64))
                print(it, dt.__name__, n, inc, "bad", len(bad), bad[:5], "diff", d, "tile", bad[0] // 4096, flush=True)
print("fails", fails)
