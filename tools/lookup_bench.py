"""Host token -> row lookup for LookupModel: dict probes in Python, one C
loop of dict probes, the C vocabulary index on 1..16 threads (1.1M tokens)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_01476_b200 import build
build.build_pack()
from paper_2312_01476_b200 import _sjbpack  # noqa: E402
n = 1_100_000
toks = [f"tok{i}" for i in range(n)]
d = {t: i for i, t in enumerate(toks)}
get = d.get
t = time.perf_counter(); [get(x, -1) for x in toks]; print("python", time.perf_counter() - t)
t = time.perf_counter(); _sjbpack.lookup(d, toks); print("C dict", time.perf_counter() - t)
c = _sjbpack.build_index(d)
for th in (1, 2, 4, 8, 16):
    ts = []
    for _ in range(3):
        t = time.perf_counter(); _sjbpack.lookup_mt(c, toks, th); ts.append(time.perf_counter() - t)
    print("C index", th, min(ts))
print("cpus", os.cpu_count())
