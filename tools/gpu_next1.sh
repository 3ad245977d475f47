#!/usr/bin/env bash
# NEXT-1 GPU pass: full GPU suite, default bench, combined-mode benches (C1 static, C3 trajectory)
# and the direct C3 trajectory for comparison.   gpurun --timeout 1800 -- 'bash tools/gpu_next1.sh TAG'
TAG=${1:-n1}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke_rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest_rc=$?"
tail -2 $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 20 > $OUT/bench_direct_$TAG.log 2>&1; echo "bench_rc=$?"
tail -1 $OUT/bench_direct_$TAG.log | cut -c1-400
timeout 600 python bench.py --mode combined --steps 200 --warmup 10 --e2e-steps 20 > $OUT/bench_comb_c1_$TAG.log 2>&1; echo "bcomb_rc=$?"
tail -1 $OUT/bench_comb_c1_$TAG.log | cut -c1-600
timeout 600 python bench.py --config C3 --views 256 --mode combined --steps 5 --warmup 3 --e2e-steps 2 > $OUT/bench_comb_c3_$TAG.log 2>&1; echo "bc3c_rc=$?"
tail -1 $OUT/bench_comb_c3_$TAG.log | cut -c1-600
timeout 600 python bench.py --config C3 --views 256 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $OUT/bench_direct_c3_$TAG.log 2>&1; echo "bc3d_rc=$?"
tail -1 $OUT/bench_direct_c3_$TAG.log | cut -c1-600
