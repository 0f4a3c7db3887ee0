"""Do two independent contexts stepping concurrently on separate streams gain from co-scheduling?
python tools/corun.py  (two 16M-fluid beds; sequential vs two host threads)"""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
from paper_2507_05643_b200 import crm  # noqa: E402

sc = workloads.bed(n=(512, 512, 64))
a = crm.load_scenario(sc)
b = crm.load_scenario(sc)
for g in (a, b):
    g.step(sc.dt, 3)
K = 10
t0 = time.perf_counter(); a.step(sc.dt, K); b.step(sc.dt, K); t1 = time.perf_counter()
seq = (t1 - t0) / K
th = [threading.Thread(target=g.step, args=(sc.dt, K)) for g in (a, b)]
t0 = time.perf_counter()
for t in th: t.start()
for t in th: t.join()
t1 = time.perf_counter()
con = (t1 - t0) / K
print(f"two contexts, per step pair: sequential {seq*1e3:.2f} ms, concurrent {con*1e3:.2f} ms, ratio {con/seq:.3f}")
