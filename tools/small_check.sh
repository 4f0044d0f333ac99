# small-workload task floor check: GPU parity tests + cfg1 bench + small sweep points
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 -rf -x > gpurun_out/gpu_tests_small.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_small.log
timeout 600 python bench.py --config cfg1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg1_small.log 2>&1
timeout 900 python tools/sweep_cfg5.py --quick --out gpurun_out/cfg5_sweep_small > gpurun_out/sweep_small.log 2>&1
