"""Per-CUDA-source-line totals of one kernel from an ncu report (needs -lineinfo/--import-source):
python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [top]
prints warp instructions, thread instructions (lane efficiency) and stall samples per source line."""
import csv
import io
import subprocess
import sys

rep, want = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
fsub = sys.argv[4] if len(sys.argv) > 4 else None   # keep only functions whose name contains this
raw = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass,cuda', '-k',
                      f'regex:{want}'], capture_output=True, text=True).stdout
fname, hdr, rows = None, None, {}
cur = None
keep = True
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == 'File Path':
        fname = r[1].split('/')[-1]
        continue
    if r[0] == 'Line No':
        hdr = {h: i for i, h in enumerate(r)}
        hdr['n'] = len(r)
        continue
    if r[0] == 'Function Name':
        keep = fsub is None or fsub in r[1]
        continue
    if hdr is None or not keep:
        continue
    n = hdr['n']
    r = r[:2] + r[len(r) - (n - 2):] if len(r) > n else r   # unescaped quotes in the source text
    if r[0]:   # a source line row (totals of its SASS)
        key = (fname, int(r[0]), r[1].strip()[:70])
        ie = int(r[hdr['Instructions Executed']] or 0)
        te = int(r[hdr['Thread Instructions Executed']] or 0)
        s = int(r[hdr['Warp Stall Sampling (All Samples)']] or 0)
        a = rows.setdefault(key, [0, 0, 0])
        a[0] += ie; a[1] += te; a[2] += s
W = sum(v[0] for v in rows.values()); S = sum(v[2] for v in rows.values())
print(f'total warp-instr {W:.4e}, lanes/instr {sum(v[1] for v in rows.values()) / max(W, 1):.1f}')
for k, v in sorted(rows.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f'{v[0] / W:6.1%} instr {v[2] / max(S, 1):6.1%} stall  lanes {v[1] / max(v[0], 1):4.1f}  {k[0]}:{k[1]}  {k[2]}')
