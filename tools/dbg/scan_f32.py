import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, paper_2507_16710_b200 as ak
ex = ak.ExecBackend(0)
x = torch.rand(1 << 28, device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    ak.accumulate("sum", x, out=y, ex=ex)
torch.cuda.synchronize()
print("ok")
