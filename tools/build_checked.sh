#!/usr/bin/env bash
# Debug build with device-side bounds checks (-DDTSDF_CHECKS): paper_2301_12796_b200/libdtsdf_checked.so.
# Use with DTSDF_LIB=paper_2301_12796_b200/libdtsdf_checked.so (tests, tools/sanitize_workload.py).
cd "$(dirname "$0")/../paper_2301_12796_b200" && \
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -DDTSDF_CHECKS -I ../include csrc/*.cu -o libdtsdf_checked.so
