# round-2 final evidence on one GPU (TAG names the outputs): smoke, every bench line incl. cfg4 in
# both similarity modes, then the ncu launch lists and full captures of tools/profile_round.sh
set -u
O=gpurun_out; T=${TAG:-r2j}
python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.log
timeout 900 python bench.py > $O/${T}_bench_cfg2.log 2>&1; tail -n 1 $O/${T}_bench_cfg2.log > $O/${T}_bench_cfg2.json
timeout 900 python bench.py --config cfg3 > $O/${T}_bench_cfg3.log 2>&1; tail -n 1 $O/${T}_bench_cfg3.log > $O/${T}_bench_cfg3.json
for th in 0.95 0.8 0.6 0.4; do timeout 600 python bench.py --config cfg5 --theta $th > $O/${T}_bench_cfg5_$th.log 2>&1; tail -n 1 $O/${T}_bench_cfg5_$th.log > $O/${T}_bench_cfg5_$th.json; done
timeout 1500 python bench.py --config cfg4 --sims tensor > $O/${T}_bench_cfg4_tensor.log 2>&1; tail -n 1 $O/${T}_bench_cfg4_tensor.log > $O/${T}_bench_cfg4_tensor.json
timeout 1500 python bench.py --config cfg4 > $O/${T}_bench_cfg4_exact.log 2>&1; tail -n 1 $O/${T}_bench_cfg4_exact.log > $O/${T}_bench_cfg4_exact.json
TAG=$T bash tools/profile_round.sh > $O/${T}_profile_round.log 2>&1
tail -n 2 $O/${T}_smoke.log; ls $O | grep $T | head -40
