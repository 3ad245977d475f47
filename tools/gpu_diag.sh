#!/usr/bin/env bash
# Diagnostics of k_raycast on one GPU box: the DTSDF_STATS build's per-ray counters and per-ray
# timeline (tools/dump_stats.py, tools/timeline.py), then one ncu --set full capture of k_raycast.
#   gpurun --timeout 1200 -- 'bash tools/gpu_diag.sh r2g'
TAG=${1:-diag}
OUT=gpurun_out
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I include -DDTSDF_STATS"
python -c "import __graft_entry__ as g; g.build()"
nvcc $FL paper_2301_12796_b200/csrc/*.cu -o paper_2301_12796_b200/libdtsdf_stats.so
python tools/dump_stats.py C1 C2 > $OUT/stats_$TAG.log 2>&1; echo stats_rc=$?
python tools/timeline.py C1 C2 > $OUT/timeline_$TAG.log 2>&1; echo timeline_rc=$?
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 5 --batch-views 0"
$CMD > $OUT/plain_$TAG.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_launch_$TAG.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_raycast -s 5 -c 1 -o $OUT/prof_$TAG -f $CMD > $OUT/ncu_full_$TAG.log 2>&1
echo ncu_rc=$?
