"""One subword embedding (cfg3: 200k strings, 2M x 100 table) and one
normalise-and-cast (cfg2 S: 1M x 100) for ncu captures of the prep kernels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_01476_b200 import datagen, device as D
dev = torch.device("cuda:0")
left, _ = datagen.strings(200_000, 10, 0.3, seed=0)
g = torch.Generator(device=dev).manual_seed(0)
table = torch.randn((2_000_000, 100), generator=g, device=dev) * 0.1
(L, S), c = datagen.config_vectors("cfg2")
Sd = torch.from_numpy(S).to(dev)
for _ in range(2):
    D.subword_rows(left, table, 3, 6, prepared=True)
    D.prepare(Sd)
torch.cuda.synchronize()
print("ok")
