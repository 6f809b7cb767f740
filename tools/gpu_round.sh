#!/bin/bash
# Round checkpoint on the GPU box: GPU tests, smoke, bench lines of configs 1-5, the
# reference arm, and (each only after its own command ran without ncu) the ncu launch
# list of one config-2 decomposition and one --set full capture of K1 at config 2.
# usage: tools/gpu_round.sh <tag>   (outputs under gpurun_out/<tag>/)
T=${1:-r02}
O=gpurun_out/$T
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --config 2 --steps 20 --warmup 5 > $O/bench_config2.json 2> $O/bench_config2.err; echo "bench 2 rc=$?" >> $O/status.log
for c in 1 3 4 5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_config$c.json 2> $O/bench_config$c.err
  echo "bench $c rc=$?" >> $O/status.log
done
timeout 900 python bench.py --impl reference --config 2 --steps 1 --warmup 0 > $O/bench_reference_config2.json 2> $O/bench_reference_config2.err; echo "reference rc=$?" >> $O/status.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ncu_launches_config2.csv python tools/one_decomp.py 2 1 > $O/ncu_launches.log 2>&1; echo "ncu launches rc=$?" >> $O/status.log
python tools/launch_table.py $O/ncu_launches_config2.csv > $O/launch_table_config2.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1s_kernel -c 1 -o $O/k1s_cfg2 -f python tools/k1_sweep.py 2 - > $O/ncu_k1.log 2>&1; echo "ncu k1 rc=$?" >> $O/status.log
tail -n 3 $O/pytest.log; cat $O/status.log; tail -n 2 $O/smoke.log
for c in 1 2 3 4 5; do python - <<EOF
import json
try:
    d=json.loads(open("$O/bench_config$c.json").read().strip().splitlines()[-1])
    print($c, d["ms_per_step"], d.get("stages_ms"), d["roofline"]["frac"], {k:v.get("frac") for k,v in d.get("kernels",{}).items()}, d["e2e"]["value"], d["gpu_launches"])
except Exception as e:
    print($c, "ERR", e)
EOF
done
tail -c 600 $O/bench_reference_config2.json
