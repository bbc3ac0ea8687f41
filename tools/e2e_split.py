"""cfg2 host-input join (tensor_join_vectors) e2e by first-part share of the left split."""
import os, sys, time, statistics
sys.path.insert(0, os.getcwd())
import torch
from paper_2312_01476_b200 import datagen
from paper_2312_01476_b200.join import tensor_join_vectors
(L, S), c = datagen.config_vectors("cfg2")
Lp, Sp = torch.from_numpy(L).pin_memory(), torch.from_numpy(S).pin_memory()
dev = torch.device("cuda:0")
for frac in (sys.argv[1:] or ["0.5", "0.55", "0.6", "0.65", "0.5", "0.58"]):
    os.environ["SJB_SPLIT_FIRST"] = frac
    for _ in range(2): tensor_join_vectors(Lp, Sp, c["theta"], device=dev)
    ts = []
    for _ in range(7):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        ms, _ = tensor_join_vectors(Lp, Sp, c["theta"], device=dev)
        ts.append(time.perf_counter() - t0)
    print(f"first={frac}: e2e median {1e3*statistics.median(ts):.2f} ms min {1e3*min(ts):.2f}", flush=True)
