"""Summarise a raw trace (scripts/trace_dump.py): synthesis CTAs at slots
[0, 2048), grid-stage CTAs at [2048, 4096); times in us from the first mark."""
import sys
import numpy as np

b = np.load(sys.argv[1]).astype(np.int64)
s = b[:2048]
s = s[s[:, 2] > 0]
g = b[2048:]
g = g[g[:, 2] > 0]
t0 = s[:, 1].min()
pct = lambda x: np.percentile(x, [0, 50, 90, 100]).round(2)
print("synth CTAs", len(s), "grid CTAs", len(g))
for k in range(5):
    v = s[:, 1 + k]
    v = v[v > 0]
    if len(v):
        print(" synth mark", k, pct((v - t0) / 1e3))
for k in range(7):
    v = g[:, 1 + k]
    v = v[v > 0]
    if len(v):
        print(" grid mark", k, pct((v - t0) / 1e3))
