#!/bin/bash
# A/B of whole library builds on the C3 training leg (train-only bench).  Usage: gpu_train_ab.sh OUT name1 name2 ...
out=gpurun_out/$1; shift
mkdir -p $out
for rep in 1 2; do for v in "$@"; do
  RGS_LIB=$PWD/paper_2402_03307_b200/_ab/$v.so timeout 400 python bench.py --train-only --no-cpu-baseline --no-dropin > $out/train_$v.json 2>> $out/train.err
  python -c "
import json;d=json.loads(open('$out/train_$v.json').read().strip().splitlines()[-1])
t=d.get('train', d)
print('$v', round(t['value'],1), {k: round(v,4) for k,v in t['stage_ms_one_step'].items()})" >> $out/ab.txt
done; done
cat $out/ab.txt
