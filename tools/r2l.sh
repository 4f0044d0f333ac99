mkdir -p gpurun_out
python -m pytest tests/test_gpu_pdd.py tests/test_pdd_oracle.py -q -p no:cacheprovider > gpurun_out/pdd_tests_r2l.log 2>&1; tail -2 gpurun_out/pdd_tests_r2l.log
timeout 600 python tools/bench_pdd.py --out gpurun_out/pdd_bench_r2l > gpurun_out/pdd_bench_r2l.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pdd_adi -s 1 -c 1 -o gpurun_out/prof_adi_r2l python tools/bench_pdd.py --trees 10000 --out gpurun_out/pdd_tmp > gpurun_out/ncu_adi_r2l.log 2>&1
echo done
