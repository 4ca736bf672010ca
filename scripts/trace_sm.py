"""Per-SM load vs finish time of the state synthesis (trace marks, default kernel)."""
import json, numpy as np, torch
from paper_1805_06557_b200 import _lib
from paper_1805_06557_b200.sphere import SphereConfig, plan_for
from paper_1805_06557_b200.device import to_device, pack
from paper_1805_06557_b200.workloads import seeded_balanced_state
cfg = SphereConfig.for_truncation(256); T = 256
plan = plan_for(cfg)
st = to_device(pack(seeded_balanced_state(cfg)))
lib = _lib.load()
for _ in range(3): plan.tendency_dev(3, st)
torch.cuda.synchronize()
lib.swx_trace(1, None, 0)
plan.tendency_dev(3, st)
buf = np.zeros((4096, 8), dtype=np.uint64)
lib.swx_trace(0, buf.ctypes.data, 4096)
r = buf[:257].astype(np.int64)
t0 = r[:, 1].min()
sm = r[:, 0]; start = (r[:, 1] - t0) / 1e3; end = (r[:, 3] - t0) / 1e3
load = {}
fin = {}
for m in range(257):
    s = int(sm[m]); load[s] = load.get(s, 0) + (T + 2 - m); fin[s] = max(fin.get(s, 0), end[m])
xs = np.array([load[s] for s in load]); ys = np.array([fin[s] for s in load])
order = np.argsort(-ys)[:10]
keys = list(load)
print("slowest SMs (sm, degree-steps, finish us, columns):")
for k in order:
    s = keys[k]
    print(s, load[s], round(ys[k], 2), [m for m in range(257) if sm[m] == s])
print("corr(load, finish)", float(np.corrcoef(xs, ys)[0, 1]))
print("per-column duration (us) m=0..8:", [round(float(end[m] - start[m]), 2) for m in range(9)])
print("m=128..136:", [round(float(end[m] - start[m]), 2) for m in range(128, 137)])
