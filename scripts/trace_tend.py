"""Per-CTA phase trace of one cfg2 tendency (synthesis + fused grid stage)."""
import json
import numpy as np
import torch
from paper_1805_06557_b200 import _lib
from paper_1805_06557_b200.sphere import SphereConfig, plan_for
from paper_1805_06557_b200.device import to_device, pack
from paper_1805_06557_b200.workloads import seeded_balanced_state

cfg = SphereConfig.for_truncation(256)
plan = plan_for(cfg)
st = to_device(pack(seeded_balanced_state(cfg)))
lib = _lib.load()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    plan.tendency_dev(3, st)
torch.cuda.synchronize()
flush.zero_()
torch.cuda.synchronize()
lib.swx_trace(1, None, 0)
plan.tendency_dev(3, st)
buf = np.zeros((4096, 8), dtype=np.uint64)
lib.swx_trace(0, buf.ctypes.data, 4096)
out = {}
for name, lo, hi, nm in (("synth", 0, 257, 3), ("grid", 2048, 2048 + 208, 6)):
    r = buf[lo:hi].astype(np.int64)
    r = r[r[:, 1] > 0]
    t0 = r[:, 1].min()
    rel = (r[:, 1:1 + nm] - t0) / 1e3  # us
    out[name] = {"n": int(len(r)), "start_us": [float(x) for x in np.percentile(rel[:, 0], [0, 50, 100])],
                 "end_us": [float(x) for x in np.percentile(rel[:, -1], [0, 50, 100])],
                 "phase_med_us": [float(np.median(rel[:, k + 1] - rel[:, k])) for k in range(nm - 1)],
                 "phase_max_us": [float(np.max(rel[:, k + 1] - rel[:, k])) for k in range(nm - 1)]}
    dur = rel[:, -1] - rel[:, 0]
    out[name]["dur_us"] = [float(x) for x in np.percentile(dur, [0, 50, 90, 100])]
    if name == "grid":
        out[name]["ph0_load_dft_med_us"] = float(np.median((r[:, 7] - r[:, 1]) / 1e3))
    sm = r[:, 0]
    per_sm = np.bincount(sm.astype(int))
    out[name]["ctas_per_sm_hist"] = np.bincount(per_sm).tolist()
    out[name]["late_starts"] = sorted([(int(lo + k), round(float(rel[k, 0]), 2), int(sm[k]))
                                       for k in range(len(r)) if rel[k, 0] > 2.0], key=lambda x: x[1])[:12]
    if name == "synth":
        order = np.argsort(-dur)[:8]
        out[name]["slowest"] = [(int(lo + k), float(dur[k]), int(sm[k])) for k in order]
print(json.dumps(out, indent=1))
