set -e
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I include -DDTSDF_STATS"
for v in ${VARIANTS:-"cur:"}; do
  n=${v%%:*}; d=${v#*:}
  nvcc $FL $d paper_2301_12796_b200/csrc/*.cu -o gpurun_out/stats_$n.so
  echo "== $n"; DTSDF_LIB=$PWD/gpurun_out/stats_$n.so python tools/dump_stats.py C1 C2
done
