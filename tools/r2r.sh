mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pdd_adi -s 1 -c 1 -o gpurun_out/prof_adic_r2r python tools/bench_pdd.py --trees 10000 --out gpurun_out/pdd_tmp > gpurun_out/ncu_adic_r2r.log 2>&1
echo done
