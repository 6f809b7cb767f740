#!/bin/bash
# Round checkpoint on the GPU box: GPU tests, bench lines of configs 1-5, reference arm, launch list.
# usage: tools/gpu_round.sh <tag>   (outputs under gpurun_out/<tag>/)
T=${1:-r02}
O=gpurun_out/$T
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for c in 2 1 3 4 5; do
  extra=""; [ $c = 5 ] && extra="--no-cpu-baseline"
  [ $c != 2 ] && extra="--no-cpu-baseline"
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 $extra > $O/bench_config$c.json 2> $O/bench_config$c.err
  echo "bench $c rc=$?" >> $O/status.log
done
tail -n 3 $O/pytest.log; cat $O/status.log; cat $O/smoke.log | tail -n 2
for c in 1 2 3 4 5; do python - <<EOF
import json
try:
    d=json.loads(open("$O/bench_config$c.json").read().strip().splitlines()[-1])
    print($c, d["ms_per_step"], d.get("stages_ms"), d["roofline"]["frac"], {k:v.get("frac") for k,v in d.get("kernels",{}).items()}, d["e2e"]["value"])
except Exception as e:
    print($c, "ERR", e)
EOF
done
