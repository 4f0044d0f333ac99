#!/bin/bash
# One GPU round trip: parity tests, cfg4/cfg2 bench lines, ncu --set full of the
# tree-walk kernel on a reduced cfg4 launch.  Usage (under gpurun):
#   bash tools/gpu_cycle.sh <tag> [tests|notests]
tag=${1:-run}
mkdir -p gpurun_out
if [ "${2:-tests}" = "tests" ]; then
  timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 -rf -x > gpurun_out/gpu_tests_$tag.log 2>&1
  echo "tests rc=$?" >> gpurun_out/gpu_tests_$tag.log
fi
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4_$tag.log 2>&1
python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2_$tag.log 2>&1
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --trees 200000 > gpurun_out/plain_small_$tag.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:tree_walk -s 1 -c 1 \
      -o gpurun_out/prof_tw_$tag python bench.py --steps 1 --warmup 1 --no-cpu-baseline --trees 200000 \
      > gpurun_out/ncu_full_$tag.log 2>&1
echo done
