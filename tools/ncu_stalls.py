"""Warp-stall breakdown per kernel from an ncu --set full report:
python tools/ncu_stalls.py REPORT.ncu-rep [kernel-regex]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    if pat and not pat.search(name):
        continue
    st = []
    for k, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(r[k].replace(",", "")), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    tot = sum(v for v, _ in st)
    print(f"===== {name[:60]}  warp-cycles per issued instruction, by stall reason")
    for v, h in sorted(st, reverse=True)[:10]:
        print(f"  {v:6.2f}  ({100 * v / tot:4.1f} %)  {h}")
