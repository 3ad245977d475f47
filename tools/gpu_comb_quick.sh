#!/usr/bin/env bash
# combined-TSDF quick pass: GPU tests of the combined path, combined benches, launch list
TAG=${1:-cq}
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_combined.py -x -q > $OUT/pytest_comb_$TAG.log 2>&1; echo "pytest_rc=$?"; tail -2 $OUT/pytest_comb_$TAG.log
timeout 600 python bench.py --mode combined --steps 200 --warmup 10 --e2e-steps 20 > $OUT/bench_comb_c1_$TAG.log 2>&1; echo "bcomb_rc=$?"
timeout 600 python bench.py --config C3 --views 256 --mode combined --steps 5 --warmup 3 --e2e-steps 2 > $OUT/bench_comb_c3_$TAG.log 2>&1; echo "bc3c_rc=$?"
for f in $OUT/bench_comb_c1_$TAG.log $OUT/bench_comb_c3_$TAG.log; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], d['value'], d['roofline']['kernel_ms'], d['roofline'].get('combine_ms_per_step'), d['roofline'].get('recombinations_per_step'), d['e2e']['value'])"; done
CMD="python bench.py --mode combined --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $OUT/launches_comb_$TAG.csv $CMD > /dev/null 2>&1; echo "ncu_rc=$?"
