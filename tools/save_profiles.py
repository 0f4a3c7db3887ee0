"""Copy a gpurun evidence set into profiles/ under a round tag:
python tools/save_profiles.py TAG NOTE
  gpurun_out/bench_full.log  -> profiles/TAG_bench_bed32M.json   (the bench JSON line)
  gpurun_out/launches.csv    -> profiles/TAG_launches_bed32M.csv (ncu launch list) + shares
  gpurun_out/full_bed32M.ncu-rep -> profiles/TAG_ncu_full_bed32M.txt (summary + stalls),
                                    profiles/ncu_traffic.json (DRAM bytes per launch)"""
import collections
import csv
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, note = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
out = os.path.join(ROOT, "profiles")
g = os.path.join(ROOT, "gpurun_out")
line = open(os.path.join(g, "bench_full.log")).read().strip().splitlines()[-1]
json.loads(line)
open(os.path.join(out, f"{tag}_bench_bed32M.json"), "w").write(line + "\n")
shutil.copy(os.path.join(g, "launches.csv"), os.path.join(out, f"{tag}_launches_bed32M.csv"))
rows = [r for r in csv.reader(open(os.path.join(g, "launches.csv"))) if len(r) > 10 and r[0].isdigit()]
t = collections.Counter()
for r in rows:
    t[r[4].split("(")[0].replace("void ", "").split("<")[0]] += float(r[-1])
tot = sum(t.values())
shares = "\n".join(f"  {k:24s} {v / 1e6:9.2f} ms {v / tot:6.1%}" for k, v in t.most_common(12))
rep = os.path.join(g, "full_bed32M.ncu-rep")
summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep], capture_output=True, text=True).stdout
stalls = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_stalls.py"), rep], capture_output=True, text=True).stdout
with open(os.path.join(out, f"{tag}_ncu_full_bed32M.txt"), "w") as f:
    f.write(f"# ncu --set full --clock-control none --import-source on -k regex:\"k_filter_t|k_rates_t|k_bce_t\" -s 5 -c 5, tools/prof_step.py bed32M 3. {note}\n")
    f.write(summ + "\n" + stalls + "\n# serialized launch list shares (ncu --metrics gpu__time_duration.sum, bench.py --steps 2 --warmup 3)\n" + shares + "\n")
traffic, cur = {}, None
for ln in summ.splitlines():
    m = re.match(r"----- (?:void )?(k_\w+)(?:<(\d), \d>)?", ln)
    if m:
        name = m.group(1)
        if name in ("k_rates_t", "k_bce_t"):
            name = ("k_rates_" if name == "k_rates_t" else "k_bce_") + ("A" if m.group(2) == "0" else "B")
        elif name == "k_filter_t":
            name = "k_filter"
        cur = name
        traffic[cur] = 0.0
    m = re.match(r"\s+dram__bytes_(read|write)\.sum: ([\d.]+) (\w+)", ln)
    if m and cur:
        traffic[cur] += float(m.group(2)) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[m.group(3)]
json.dump({"bed32M": traffic, "_source": f"profiles/{tag}_ncu_full_bed32M.txt: dram__bytes_read.sum + dram__bytes_write.sum",
           "_unit": "bytes per launch"}, open(os.path.join(out, "ncu_traffic.json"), "w"), indent=1)
print(shares)
print(json.dumps(traffic))
