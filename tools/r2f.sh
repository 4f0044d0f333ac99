mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "pade or interface" -s > gpurun_out/pade_r2f.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg1_r2f.csv python bench.py --config cfg1 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_walk -s 1 -c 1 -o gpurun_out/prof_tw_cfg2_r2f python bench.py --config cfg2 --steps 1 --warmup 1 --no-cpu-baseline --graph off > gpurun_out/ncu_cfg2_r2f.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_walk -s 1 -c 1 -o gpurun_out/prof_tw_cfg3_r2f python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline --graph off > gpurun_out/ncu_cfg3_r2f.log 2>&1
echo done
