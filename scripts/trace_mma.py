"""Per-CTA phase times of the DMMA state synthesis (trace build: SWX_LIB=.../libswx_trace.so)."""
import numpy as np, torch
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
torch.cuda.synchronize()
buf = np.zeros((4096, 8), dtype=np.uint64)
lib.swx_trace(0, buf.ctypes.data, 4096)
n = 514
r = buf[:n].astype(np.int64)
t0 = r[:, 1].min()
t = (r[:, 1:6] - t0) / 1e3
print("kernel span us", t[:, 4].max())
print("cta  m blk sm  start  wait->  stage  loop  epi  end")
for b in list(range(0, 12)) + list(range(250, 262)) + list(range(500, 514)):
    ph = t[b]
    print(b, b // 2, b % 2, int(r[b, 0]), *[round(float(x), 2) for x in (ph[0], ph[1] - ph[0], ph[2] - ph[1], ph[3] - ph[2], ph[4] - ph[3], ph[4])])
d = t[:, 4] - t[:, 0]
print("mean CTA duration", d.mean(), "phases mean", [(t[:, k + 1] - t[:, k]).mean().round(2) for k in range(4)])
sm = r[:, 0]
print("CTAs per SM max", np.bincount(sm).max(), "SMs used", len(set(sm.tolist())))
