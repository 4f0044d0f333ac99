#!/bin/bash
# Round-2 GPU cycle (run under gpurun): bash tools/gpu_cycle_r2.sh <tag>
# smoke, pytest -m gpu, the default bench line (driver form, with the oracle
# baseline), cfg1-3 lines, the ncu launch list of the default command, the
# ncu hardware counters of one full-size cfg4 launch, ncu --set full of the
# tree walk on reduced cfg4 and cfg2 launches.
tag=${1:-r2}
mkdir -p gpurun_out
nproc > gpurun_out/host_$tag.txt; lscpu | grep -E 'Model name|^CPU\(s\)' >> gpurun_out/host_$tag.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv >> gpurun_out/host_$tag.txt
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$tag.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 -rf > gpurun_out/gpu_tests_$tag.log 2>&1
echo "tests rc=$?" >> gpurun_out/gpu_tests_$tag.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_cfg4_$tag.log 2>&1
for c in cfg1 cfg2 cfg3; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_$tag.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_launch_$tag.log 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_issued.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__cycles_elapsed.avg,smsp__thread_inst_executed_per_inst_executed.ratio
timeout 900 ncu --metrics $M --clock-control none --csv -k regex:tree_walk -s 3 -c 1 \
    --log-file gpurun_out/traffic_cfg4_$tag.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --graph off \
    > gpurun_out/ncu_traffic_$tag.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_walk -s 1 -c 1 \
    -o gpurun_out/prof_tw_cfg4_$tag python bench.py --steps 1 --warmup 1 --no-cpu-baseline --trees 200000 --graph off \
    > gpurun_out/ncu_full_cfg4_$tag.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_walk -s 1 -c 1 \
    -o gpurun_out/prof_tw_cfg2_$tag python bench.py --config cfg2 --steps 1 --warmup 1 --no-cpu-baseline --graph off \
    > gpurun_out/ncu_full_cfg2_$tag.log 2>&1

# keep the merge-back under gpurun's 64 MiB: compress the reports
for f in gpurun_out/prof_tw_cfg4_$tag.ncu-rep gpurun_out/prof_tw_cfg2_$tag.ncu-rep; do
  [ -f "$f" ] && xz -T0 -6 "$f"
done
du -sh gpurun_out
