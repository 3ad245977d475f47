#!/usr/bin/env bash
# A/B of compile-time variants of the fusion kernels: tools/ab_fusion.sh "name:-DFOO=1" ...
set -e
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I include"
for v in "$@"; do
  n=${v%%:*}; d=${v#*:}
  nvcc $FL $d paper_2301_12796_b200/csrc/*.cu -o gpurun_out/abf_$n.so
done
for r in 1 2; do
  for v in "$@"; do
    n=${v%%:*}
    echo -n "$n "; DTSDF_LIB=$PWD/gpurun_out/abf_$n.so python tools/bench_fusion.py
  done
done
