"""Table analysis time with cold vs warm L2 (T256 tendency stages)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1805_06557_b200 import _lib
from paper_1805_06557_b200.device import pack, to_device
from paper_1805_06557_b200.sphere import SphereConfig, plan_for
from paper_1805_06557_b200.workloads import seeded_balanced_state

cfg = SphereConfig.for_truncation(256)
plan = plan_for(cfg)
st = to_device(pack(seeded_balanced_state(cfg)))
out = torch.empty_like(st)
lib = _lib.load()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
buf = np.zeros(7)
for mode in ("cold", "warm", "cold", "warm"):
    acc = np.zeros(7)
    for _ in range(10):
        if mode == "cold":
            flush.zero_()
        else:
            plan.tendency_dev(3, st, out)
        torch.cuda.synchronize()
        _lib.check(lib.swx_sht_tendency_profile(plan._h, 3, st.data_ptr(), out.data_ptr(),
                                                plan.workspace.data_ptr(), plan.workspace.numel(),
                                                buf.ctypes.data, torch.cuda.current_stream().cuda_stream))
        acc += buf
    acc /= 10
    print(mode, "synth %.1f grid %.1f analysis %.1f total %.1f us" % (acc[0] * 1e3, acc[3] * 1e3, acc[5] * 1e3, acc[6] * 1e3))
