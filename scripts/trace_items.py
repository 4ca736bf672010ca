"""Per-CTA durations of the state synthesis (build with --trace)."""
import os, numpy as np, torch
from paper_1805_06557_b200 import _lib
from paper_1805_06557_b200.sphere import SphereConfig, plan_for
from paper_1805_06557_b200.device import to_device, pack
from paper_1805_06557_b200.workloads import seeded_balanced_state
cfg = SphereConfig.for_truncation(256)
plan = plan_for(cfg)
st = to_device(pack(seeded_balanced_state(cfg)))
lib = _lib.load()
for _ in range(3): plan.tendency_dev(3, st)
torch.cuda.synchronize()
lib.swx_trace(1, None, 0)
plan.tendency_dev(3, st)
buf = np.zeros((4096, 8), dtype=np.uint64)
lib.swx_trace(0, buf.ctypes.data, 4096)
n = 385 if int(os.environ.get("SWX_SYNTH_PSPLIT", "64")) else 257
r = buf[:n].astype(np.int64)
r = r[r[:, 1] > 0]
t0 = r[:, 1].min()
st_ = (r[:, 1] - t0) / 1e3; en = (r[:, 3] - t0) / 1e3
print(os.environ.get("SWX_SYNTH_PSPLIT"), "n", len(r), "end max", en.max().round(2))
print("first 6 CTAs (start, dur):", [(round(a, 2), round(b - a, 2)) for a, b in zip(st_[:6], en[:6])])
print("CTAs 126..131:", [(round(a, 2), round(b - a, 2)) for a, b in zip(st_[126:132], en[126:132])])
print("last starters:", sorted([(round(a, 2), round(b - a, 2)) for a, b in zip(st_, en)])[-5:])
