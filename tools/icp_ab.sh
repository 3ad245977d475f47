for v in 4 5 8; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I include -DDTSDF_ICP_PIX=$v paper_2301_12796_b200/csrc/*.cu -o gpurun_out/icp$v.so
  echo "== ICP_PIX $v"; DTSDF_LIB=$PWD/gpurun_out/icp$v.so python tools/bench_icp.py 2>&1 | tail -1
done
