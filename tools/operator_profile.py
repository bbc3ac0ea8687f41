"""cfg2 through the drop-in operator tensor_join(RawRelation, RawRelation,
LookupModel): wall per call and a cProfile of one warm call (host hot spots)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_01476_b200 import build, datagen
build.build()
from paper_2312_01476_b200 import LookupModel, RawRelation, tensor_join  # noqa: E402
if "--cfg3" in sys.argv:   # strings through the subword model
    from paper_2312_01476_b200 import SubwordModel  # noqa: E402
    tl, tr = datagen.strings(200_000, 200_000, 0.3, seed=0)
    g = torch.Generator(device="cuda").manual_seed(0)
    model = SubwordModel(torch.randn((2_000_000, 100), generator=g, device="cuda") * 0.1)
    c = {"theta": 0.85}
else:
    (L, S), c = datagen.config_vectors("cfg2")
    tl = [f"l{i}" for i in range(len(L))]
    tr = [f"r{i}" for i in range(len(S))]
    model = LookupModel.from_matrix(tl + tr, np.concatenate([L, S]))
lrel, rrel = RawRelation("left", tl), RawRelation("right", tr)
for _ in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    ms, st = tensor_join(lrel, rrel, model, c["theta"], 64 << 20)
    torch.cuda.synchronize(); print("wall", time.perf_counter() - t, len(ms))
pr = cProfile.Profile()
pr.enable()
ms, st = tensor_join(lrel, rrel, model, c["theta"], 64 << 20)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
