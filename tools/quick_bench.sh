#!/bin/bash
# quick per-kernel timing of the C5 bed (no oracle, no e2e, no NEXT legs): tools/quick_bench.sh [tag]
tag=${1:-q}
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-next > gpurun_out/qb_$tag.json 2> gpurun_out/qb_$tag.err
python - "$tag" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/qb_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print("ms/step %.3f  value %.3e  clocks %s" % (d["ms_per_step"], d["value"], d["clocks"]))
for k, v in sorted(d["kernels"].items(), key=lambda kv: -kv[1]["ms_per_step"]):
    print("  %-16s %8.3f ms  %s" % (k, v["ms_per_step"], ("alu_frac %.3f" % v["alu_frac"]) if "alu_frac" in v else ""))
PY
