# last check of the final tree on one GPU: smoke, -m gpu tests, the default bench line, the cfg4 tensor-sims line
set -u
O=gpurun_out; T=${TAG:-fin}
python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${T}_gputest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_gputest.log
timeout 900 python bench.py > $O/${T}_bench_cfg2.log 2>&1; tail -n 1 $O/${T}_bench_cfg2.log > $O/${T}_bench_cfg2.json
timeout 1500 python bench.py --config cfg4 --sims tensor --no-cpu-baseline > $O/${T}_bench_cfg4_tensor.log 2>&1; tail -n 1 $O/${T}_bench_cfg4_tensor.log > $O/${T}_bench_cfg4_tensor.json
tail -n 2 $O/${T}_smoke.log; tail -n 3 $O/${T}_gputest.log
python - <<PY
import json
for f in ("bench_cfg2", "bench_cfg4_tensor"):
    try:
        d = json.loads(open("gpurun_out/${T}_" + f + ".json").read())
    except Exception as e:
        print(f, "ERR", e)
        continue
    print(f, "%.3e" % d["value"], "%.2f ms" % d["ms_per_step"], "e2e %.3e" % d["e2e"]["value"],
          d.get("parity", {}).get("digest"))
PY
