"""Per-kernel SASS hot spots from an ncu report (needs -lineinfo/--import-source):
python tools/ncu_source.py REPORT.ncu-rep KERNEL_SUBSTR [top]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, want = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for row in csv.reader(io.StringIO(raw)):
    if row and row[0] == 'Kernel Name':
        cur = [row[1], None, []]
        blocks.append(cur)
    elif row and row[0] == 'Address':
        cur[1] = row
    elif cur is not None and row:
        cur[2].append(row)
for name, hdr, rows in blocks:
    if want not in name:
        continue
    H = {h: i for i, h in enumerate(hdr)}
    samp = H['Warp Stall Sampling (All Samples)']
    tie = H['Thread Instructions Executed']
    ie = H['Instructions Executed']
    tot_s = sum(int(r[samp]) for r in rows)
    tot_t = sum(int(r[tie]) for r in rows)
    tot_i = sum(int(r[ie]) for r in rows)
    print(f'== {name[:90]}\n   samples {tot_s}, warp-instr {tot_i:.3e}, thread-instr {tot_t:.3e}')
    cls = collections.Counter()
    for r in rows:
        op = re.sub(r'^@!?U?P\w+\s+', '', r[1].strip()).split(' ')[0].split('.')[0]
        cls[op] += int(r[tie])
    print('   thread-instr by opcode:', ', '.join(f'{k} {v / tot_t:.1%}' for k, v in cls.most_common(14)))
    for r in sorted(rows, key=lambda r: -int(r[samp]))[:top]:
        print(f'   {int(r[samp]) / max(tot_s, 1):6.1%}  {int(r[ie]):>11}  {r[1].strip()[:70]}')
    break
