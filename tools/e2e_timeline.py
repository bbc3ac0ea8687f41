"""Timeline of the cfg2 host-input join (tensor_join_vectors) under
torch.profiler: kernels, copies and host gaps, written to
gpurun_out/e2e_timeline.json as (name, stream, start_us, dur_us) rows."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2312_01476_b200 import datagen
from paper_2312_01476_b200.join import tensor_join_vectors

(L, S), c = datagen.config_vectors("cfg2")
Lp, Sp = torch.from_numpy(L).pin_memory(), torch.from_numpy(S).pin_memory()
dev = torch.device("cuda:0")
for _ in range(3):
    tensor_join_vectors(Lp, Sp, c["theta"], device=dev)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        t0 = time.perf_counter()
        ms, _ = tensor_join_vectors(Lp, Sp, c["theta"], device=dev)
        torch.cuda.synchronize()
        print(f"e2e {1e3 * (time.perf_counter() - t0):.2f} ms, {len(ms)} matches", flush=True)
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace("gpurun_out/e2e_trace.json")
rows = []
with open("gpurun_out/e2e_trace.json") as fh:
    tr = json.load(fh)
for e in tr.get("traceEvents", []):
    if e.get("ph") != "X":
        continue
    cat = e.get("cat", "")
    if cat in ("kernel", "gpu_memcpy", "gpu_memset", "cuda_runtime", "cuda_driver"):
        rows.append((cat, e.get("name", "")[:80], e.get("args", {}).get("stream", e.get("tid")),
                     e["ts"], e.get("dur", 0)))
rows.sort(key=lambda r: r[3])
with open("gpurun_out/e2e_timeline.json", "w") as fh:
    json.dump(rows, fh)
print(len(rows), "events")
