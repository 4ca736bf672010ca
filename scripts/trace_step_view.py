"""Timeline of one traced ETD2RK step (bench.py with SWX_TRACE_OUT, trace build):
the step's last synthesis (slots 0..), table analysis (1024..), grid stage
(2048..) and last lg pole sum (REXI buffer); us from the synthesis' first mark."""
import sys
import numpy as np

b = np.load(sys.argv[1]).astype(np.int64)
sht, rx = (b[0], b[1]) if b.ndim == 3 else (b, None)
def rows(buf, lo, hi):
    r = buf[lo:hi]
    return r[(r[:, 1:] > 0).any(axis=1)]
s, a, g = rows(sht, 0, 1024), rows(sht, 1024, 2048), rows(sht, 2048, 4096)
t0 = s[:, 1].min()
def show(name, r):
    print(name, "CTAs", len(r))
    for k in range(7):
        v = r[:, 1 + k]
        v = v[v > 0]
        if len(v):
            print(f"   mark {k}", np.percentile((v - t0) / 1e3, [0, 50, 90, 100]).round(2))
show("synth", s)
show("grid", g)
show("analysis", a)
if rx is not None:
    show("lg (last pole sum)", rows(rx, 0, 4096))
