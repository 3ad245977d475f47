mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 
timeout 900 python -m pytest tests/test_gpu_large.py -x -q -s > gpurun_out/pytest_c4.log 2>&1; echo "c4_rc=$?"
tail -12 gpurun_out/pytest_c4.log
timeout 900 python bench.py --config C4 --views 64 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench_c4.log 2>&1; echo "bc4=$?"
tail -2 gpurun_out/bench_c4.log
timeout 600 python bench.py --config C3 --views 256 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench_c3.log 2>&1; echo "bc3=$?"
tail -2 gpurun_out/bench_c3.log
free -g; nproc
