"""One-line summary of a render bench line and a train-only bench line (A/B runs)."""
import json
import sys

b = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
t = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
t = t.get("train", t)
print(sys.argv[3], "C2", round(b["value"], 1), "K5", round(b["stages"]["blend_fp32_k5"]["ms_per_frame"], 4),
      "frac", round(b["roofline"]["frac"], 4), "ser", round(b["roofline"]["frac_serialised"], 4),
      "| train", round(t["value"], 1), "K6", round(t["stage_ms_one_step"]["backward_tiles_k6"], 4),
      "K5", round(t["stage_ms_one_step"]["blend_fp32_k5"], 4))
