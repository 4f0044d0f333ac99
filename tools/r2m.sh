mkdir -p gpurun_out
python -m pytest tests/test_gpu_pdd.py -q -p no:cacheprovider > gpurun_out/pdd_tests_r2m.log 2>&1; tail -2 gpurun_out/pdd_tests_r2m.log
timeout 600 python tools/bench_pdd.py --out gpurun_out/pdd_bench_r2m > gpurun_out/pdd_bench_r2m.log 2>&1
echo done
