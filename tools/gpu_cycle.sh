#!/bin/bash
# One GPU round trip (run under gpurun):
#   bash tools/gpu_cycle.sh <tag> [tests|notests] [full|nofull]
# 1. parity tests (-m gpu); 2. the default bench line (cfg4) and cfg2;
# 3. the ncu launch list of the default bench command (per-launch device time);
# 4. ncu --set full of the tree-walk kernel on a reduced cfg4 launch.
tag=${1:-run}
mkdir -p gpurun_out
nproc > gpurun_out/host_$tag.txt; lscpu | grep -E 'Model name|^CPU\(s\)' >> gpurun_out/host_$tag.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv >> gpurun_out/host_$tag.txt
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_$tag.log 2>&1
rc=$?; echo "smoke rc=$rc" >> gpurun_out/smoke_$tag.log
if [ $rc -ne 0 ]; then echo "smoke failed"; tail -20 gpurun_out/smoke_$tag.log; exit 1; fi
if [ "${2:-tests}" = "tests" ]; then
  timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 -rf -x > gpurun_out/gpu_tests_$tag.log 2>&1
  echo "tests rc=$?" >> gpurun_out/gpu_tests_$tag.log
fi
timeout 600 python bench.py > gpurun_out/bench_cfg4_$tag.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_cfg4_$tag.log
timeout 300 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2_$tag.log 2>&1
if [ "${3:-full}" = "full" ]; then
  timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_launch_$tag.log 2>&1 && \
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
        > gpurun_out/ncu_launch_$tag.log 2>&1
  timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --trees 200000 > gpurun_out/plain_small_$tag.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_walk -s 1 -c 1 \
        -o gpurun_out/prof_tw_$tag python bench.py --steps 1 --warmup 1 --no-cpu-baseline --trees 200000 \
        > gpurun_out/ncu_full_$tag.log 2>&1
fi
echo done
RT_WARP_TIMES=gpurun_out/wt4_$tag.txt timeout 300 python tools/warp_times.py cfg4 1000000 > gpurun_out/wt_cfg4_$tag.log 2>&1
RT_WARP_TIMES=gpurun_out/wt2_$tag.txt timeout 300 python tools/warp_times.py cfg2 1000000 > gpurun_out/wt_cfg2_$tag.log 2>&1
rm -f gpurun_out/wt4_$tag.txt gpurun_out/wt4_$tag.txt.npy gpurun_out/wt2_$tag.txt gpurun_out/wt2_$tag.txt.npy
