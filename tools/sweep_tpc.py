import sys, statistics
sys.path.insert(0, '/root/repo')
import torch
from paper_2312_01476_b200 import device as D, datagen
(L, S), c = datagen.config_vectors("cfg2")
PL, PS = D.prepare(torch.from_numpy(L).cuda()), D.prepare(torch.from_numpy(S).cuda())
ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
for tpc in (16, 32, 64, 128, 256):
    fl = []
    for i in range(9):
        D.join_prepared(PL, PS, c["theta"], tiles_per_chunk=tpc, filter_events=ev)
        torch.cuda.synchronize()
        if i: fl.append(ev[0].elapsed_time(ev[1]))
    print(f"tpc={tpc}: median {statistics.median(fl):.3f} min {min(fl):.3f}", flush=True)
