#!/bin/bash
# Build librt.so variants for occupancy / pool sweeps (experiments, not product):
#   bash tools/build_variants.sh name "-DRT_CTAS_D3=10 -DRT_POOL_D3=112" [name2 "flags2" ...]
# -> variants/librt_<name>.so ; run them on the GPU box by copying over librt.so.
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
pids=()
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  ( /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared \
      -Xcompiler -fPIC -Xptxas -v -Iinclude $flags paper_2402_06491_b200/csrc/rt_api.cu \
      -o variants/librt_$name.so > variants/build_$name.log 2>&1 && echo "built $name" ) &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
