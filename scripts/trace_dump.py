"""Dump the raw per-CTA phase marks of one cfg2 tendency (trace build):
gpurun_out/trace_raw.npy rows = (smid, t_mark0..t_mark6) in ns; synthesis CTAs
at slots [0, 2048), grid-stage CTAs at [2048, 4096)."""
import os
import numpy as np
import torch
from paper_1805_06557_b200 import _lib
from paper_1805_06557_b200.sphere import SphereConfig, plan_for
from paper_1805_06557_b200.device import to_device, pack
from paper_1805_06557_b200.workloads import seeded_balanced_state

T = int(os.environ.get("TRUNC", "256"))
cfg = SphereConfig.for_truncation(T)
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
torch.cuda.synchronize()
buf = np.zeros((4096, 8), dtype=np.uint64)
lib.swx_trace(0, buf.ctypes.data, 4096)
os.makedirs("gpurun_out", exist_ok=True)
np.save(os.environ.get("TRACE_OUT", "gpurun_out/trace_raw.npy"), buf)
print("ok")
