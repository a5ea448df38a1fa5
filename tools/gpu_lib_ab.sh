#!/bin/bash
# A/B of whole library builds (paper_2402_03307_b200/_ab/<name>.so via RGS_LIB): render-only bench,
# K5 serialised ms per C2 frame.  Usage: gpu_lib_ab.sh OUT name1 name2 ...
out=gpurun_out/$1; shift
mkdir -p $out
for rep in 1 2; do for v in "$@"; do
  RGS_LIB=$PWD/paper_2402_03307_b200/_ab/$v.so timeout 300 python bench.py --no-train --no-c4 --no-c5 --no-cpu-baseline --no-dropin --no-e2e > $out/bench_$v.json 2>> $out/bench.err
  python -c "
import json;d=json.loads(open('$out/bench_$v.json').read().strip().splitlines()[-1])
st=d['stages']
print('$v', round(d['value'],1), {k: round(v['ms_per_frame'],4) for k,v in st.items()}, d['config']['slow_pixels_mid'])" >> $out/ab.txt
done; done
cat $out/ab.txt
