#!/bin/bash
# Run the bench on librt.so variants (tools/build_variants.sh) on the GPU box:
#   bash tools/sweep_variants.sh <tag> <cfgs> <variant> [<variant> ...]
tag=$1; cfgs=$2; shift 2
mkdir -p gpurun_out
out=gpurun_out/sweep_$tag.jsonl; : > $out
cp paper_2402_06491_b200/librt.so /tmp/librt_orig.so
for rep in 1 2; do
for v in "$@"; do
  cp variants/librt_$v.so paper_2402_06491_b200/librt.so
  for c in $cfgs; do
    st=10; [ $c = cfg4 ] && st=3
    line=$(timeout 300 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline 2>gpurun_out/sweep_${tag}_err.log | tail -1)
    echo "{\"variant\": \"$v\", \"cfg\": \"$c\", \"rep\": $rep, \"line\": $line}" >> $out
  done
done
done
cp /tmp/librt_orig.so paper_2402_06491_b200/librt.so
python3 - $out <<'PY'
import json,sys
for ln in open(sys.argv[1]):
    d=json.loads(ln); l=d["line"]
    print(f'{d["variant"]:8s} {d["cfg"]} rep{d["rep"]} {l["value"]:.4e} trees/s frac {l["roofline"]["frac"]:.4f} clocks {l["clocks"]["sm_mhz"]}')
PY
