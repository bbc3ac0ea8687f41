"""Golden cost estimates from the reference's own cost model.

Runs /root/reference's simjoin.cost (built and imported exactly as
make_golden.py does) over a grid of shapes, budgets and parameter sets, and
writes tests/golden/cost_golden.json: every estimate and the chosen plan.
tests/test_host.py checks paper_2312_01476_b200.cost against it to the bit.
Run here (the build container); the JSON is committed.
"""
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import build_reference, import_reference  # noqa: E402

PARAMS = [
    dict(access_ns=2.0, model_ns=500.0, compare_base_ns=1.0, compare_per_dim_ns=0.25,
         tensor_efficiency=0.1),
    dict(access_ns=0.0, model_ns=0.0, compare_base_ns=0.0, compare_per_dim_ns=1e-6,
         tensor_efficiency=1.0),          # all-equal: ties resolve to tensor
    dict(access_ns=1e-3, model_ns=3.3, compare_base_ns=7e-4, compare_per_dim_ns=1.1e-5,
         tensor_efficiency=0.0123),
    dict(access_ns=50.0, model_ns=0.0, compare_base_ns=0.5, compare_per_dim_ns=0.01,
         tensor_efficiency=1.0),          # tile re-touch makes tensor lose
]
SHAPES = [(1, 1, 1), (10, 10, 4), (1000, 1000, 100), (10_000, 10_000, 100),
          (100_000, 1_000_000, 100), (1_000_000, 4_000_000, 768), (7, 3_000, 13)]
BUDGETS = [4, 4096, 1 << 20, 64 << 20]


def main():
    sj = import_reference(build_reference())
    cost = sys.modules["simjoin.cost"]
    cases = []
    for p, (l, r, d), b in itertools.product(PARAMS, SHAPES, BUDGETS):
        cp = cost.CostParams(**p)
        side = max(1, int((b // 4) ** 0.5))
        if -(-l // side) * -(-r // side) > 2_000_000:
            continue                       # plan_batches would enumerate too many tiles
        plan, est = cost.choose_plan(l, r, d, b, cp)
        cases.append(dict(params=p, left=l, right=r, dim=d, budget=b, plan=plan,
                          estimates={k: float(v).hex() for k, v in est.items()},
                          selection=float(cost.estimate_selection(l, d, cp)).hex()))
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cost_golden.json")
    with open(out, "w") as fh:
        json.dump({"generator": "reference simjoin.cost (cost.py:70-125)", "cases": cases}, fh,
                  indent=0)
    print(len(cases), "cases ->", out)


if __name__ == "__main__":
    main()
