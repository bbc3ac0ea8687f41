"""cosine_vm / dots_vm kernel bandwidth: CUDA-event medians of the C-ABI
calls on n x d fp32 device matrices (the GEMV reads 4*d bytes per row)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_01476_b200 import _lib, device as D
L = _lib.lib()
dev = torch.device("cuda:0")
st = D._stream(dev)
for n, d in ((1_000_000, 100), (262_144, 256), (100_000, 768), (4_000_000, 100), (1000, 100)):
    m = torch.randn((n, d), device=dev)
    a = torch.randn(d, device=dev)
    out = torch.empty(n, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    for name, call in (("cosine_vm", lambda: L.sjb_cosine_vm(D._vp(a), D._vp(m), n, d, D._vp(out), D._vp(flags), st)),
                       ("dots_vm", lambda: L.sjb_dots_vm(D._vp(a), D._vp(m), n, d, D._vp(out), st))):
        for _ in range(3): call()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); call(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
        t = statistics.median(ts)
        print(f"{name} n={n} d={d}: {t*1e3:.1f} us  {4*n*d/t/1e6:.0f} GB/s")
