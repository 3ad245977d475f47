# ICP reduce variants (-D flags), each timed by tools/bench_icp.py:  bash tools/icp_ab.sh "name:-DFOO=1" ...
for v in "$@"; do
  n=${v%%:*}; d=${v#*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I include $d paper_2301_12796_b200/csrc/*.cu -o /tmp/icp_$n.so 2>/dev/null
  for r in 1 2; do echo "== $n"; DTSDF_LIB=/tmp/icp_$n.so python tools/bench_icp.py 2>&1 | tail -1 | cut -c90-230; done
done
