import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2312_01476_b200 import device as D
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
X = torch.randn((400_000, 768), generator=g, device=dev)
for _ in range(3): D.prepare(X)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(5): D.prepare(X)
ev[1].record(); torch.cuda.synchronize()
print(f"prepare 400k x 768: {ev[0].elapsed_time(ev[1]) / 5:.3f} ms", flush=True)
