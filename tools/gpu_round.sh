#!/usr/bin/env bash
# One GPU-box pass: build, smoke, GPU tests, default bench (+ cpu_baseline), reference arm,
# ncu launch list and one `ncu --set full` capture of k_raycast.  Logs land in gpurun_out/.
#   gpurun --timeout 1500 -- 'bash tools/gpu_round.sh [tag]'
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
nproc > $OUT/host_$TAG.txt; grep -m1 "model name" /proc/cpuinfo >> $OUT/host_$TAG.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> $OUT/host_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke_rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest_rc=$?"
tail -3 $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.log 2>&1; echo "bench_rc=$?"
cat $OUT/bench_$TAG.log | tail -2
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref_$TAG.log 2>&1; echo "ref_rc=$?"
tail -1 $OUT/bench_ref_$TAG.log
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 5 --batch-views 0"
$CMD > $OUT/plain_$TAG.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_launch_$TAG.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_raycast -s 5 -c 1 \
      -o $OUT/prof_$TAG -f $CMD > $OUT/ncu_full_$TAG.log 2>&1
echo "ncu_rc=$?"
