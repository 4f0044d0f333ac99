mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_pdd.py -q -p no:cacheprovider -k "pade or interface or degenerate" -s > gpurun_out/pade_r2g.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg1_r2g.csv python bench.py --config cfg1 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:pade --log-file gpurun_out/launches_cfg4pade_r2g.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --trees 20000 > /dev/null 2>&1
timeout 300 python bench.py --config cfg1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg1_r2g.log 2>&1
echo done
