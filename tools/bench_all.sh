mkdir -p gpurun_out
for c in cfg1 cfg2 cfg3; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_all2_$c.log 2>&1; done
timeout 900 python bench.py > gpurun_out/bench_all2_cfg4.log 2>&1
timeout 900 python tools/bench_next.py > gpurun_out/next2.log 2>&1
timeout 900 python tools/bench_pdd.py > gpurun_out/pdd2.log 2>&1
timeout 1500 python tools/sweep_cfg5.py > gpurun_out/sweep2.log 2>&1
echo done
