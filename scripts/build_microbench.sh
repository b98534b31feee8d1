#!/bin/bash
# Build the microbenchmarks (sm_100a) in-tree; the binaries are git-ignored but travel to the
# GPU box with gpurun.  usage: bash scripts/build_microbench.sh [name ...]
cd "$(dirname "$0")"
names=${@:-dsmem_bench issue_bench tma_bench tma_bench2 tma_mc_bench umma_bench umma_tma_bench}
for n in $names; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o $n $n.cu -lcuda || exit 1
done
