#!/bin/bash
mkdir -p gpurun_out/r2
trn() {
  timeout 900 python bench.py --train-only --no-cpu-baseline --no-dropin > gpurun_out/r2/bench_tr.json 2>/dev/null
  python - "$1" <<'PY'
import json, sys
d = json.load(open("gpurun_out/r2/bench_tr.json"))["train"]
print(sys.argv[1], "train", round(d["value"],1), "e2e", round(d["e2e"]["value"],1), {k: round(v,3) for k,v in d["stage_ms_one_step"].items() if k in ("depth_rank","pair_offsets_scan","duplicate_k3","tile_radix_sort_k4","tile_counts","tile_scatter_k4","preprocess_k1")})
PY
}
RGS_BINNING=radix trn radix
trn sc16
RGS_SCATTER_ROUNDS=8 trn sc8
RGS_SCATTER_ROUNDS=32 trn sc32
