#!/usr/bin/env bash
# Bench lines for every config and mode on the current build (evidence for profiles/<tag>_*):
#   gpurun --timeout 2400 -- 'bash tools/gpu_configs.sh r1f'
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="python bench.py --no-cpu-baseline"
run() { local name=$1; shift; timeout 900 "$@" > $OUT/cfg_${TAG}_$name.log 2>&1; echo "$name rc=$?"; tail -1 $OUT/cfg_${TAG}_$name.log | cut -c1-200; }
run c2_views20 $B --config C2 --views 20 --steps 20 --warmup 3 --e2e-steps 5
run c3_views256 $B --config C3 --views 256 --steps 10 --warmup 3 --e2e-steps 3
run c1_combined $B --mode combined --steps 200 --warmup 10 --e2e-steps 20
run c3_combined $B --config C3 --views 256 --mode combined --steps 5 --warmup 3 --e2e-steps 2
timeout 1200 python -m pytest tests/test_gpu_large.py -x -q -s > $OUT/cfg_${TAG}_c4_pytest.log 2>&1; echo "c4 parity rc=$?"; tail -4 $OUT/cfg_${TAG}_c4_pytest.log
run c4_views64 $B --config C4 --views 64 --steps 10 --warmup 3 --e2e-steps 3
run c1_boxes64 $B --boxes 64 --steps 100 --warmup 5 --e2e-steps 10 --batch-views 0
run c3_shard_views $B --config C3 --views 256 --shard views --steps 10 --warmup 3 --e2e-steps 3
# one ncu --set full capture of k_raycast on C4 (ncu counters on C1 and C4)
C4CMD="python bench.py --config C4 --views 1 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --batch-views 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_raycast -s 3 -c 1 -o $OUT/prof_${TAG}_c4 -f $C4CMD > $OUT/ncu_${TAG}_c4.log 2>&1; echo "c4 ncu rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 1 --steps 50 --warmup 3 --dist --no-cpu-baseline --e2e-steps 5 > $OUT/cfg_${TAG}_torchrun_dist.log 2>&1; echo "torchrun dist rc=$?"; tail -1 $OUT/cfg_${TAG}_torchrun_dist.log | cut -c1-200
