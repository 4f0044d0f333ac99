#!/bin/bash
# Perf round trip (run under gpurun): bash tools/gpu_perf.sh <tag> [configs...]
# 1. bench lines (cfg4 default + the listed configs); 2. ncu hardware
# counters of ONE full-size tree-walk launch of the default bench command
# (DRAM / L2 traffic, FP64-pipe and issue utilisation, instructions) —
# profiles/r2/traffic_<workload>.json is written from it by
# tools/traffic_json.py; 3. the ncu launch list (per-launch device times).
tag=${1:-perf}; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/host_$tag.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4_$tag.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_cfg4_$tag.log
for c in "$@"; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_$tag.log 2>&1
done
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_issued.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__cycles_elapsed.avg,smsp__thread_inst_executed_per_inst_executed.ratio
timeout 900 ncu --metrics $M --clock-control none --csv -k regex:tree_walk -s 3 -c 1 \
    --log-file gpurun_out/traffic_cfg4_$tag.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --graph off \
    > gpurun_out/ncu_traffic_$tag.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_launch_$tag.log 2>&1
timeout 300 python bench.py --config cfg1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg1_$tag.log 2>&1
echo done
