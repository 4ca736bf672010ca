"""T1279 SH round trip (synthesis + analysis of one field) for profiling."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1805_06557_b200.device import pack, to_device
from paper_1805_06557_b200.sphere import SphereConfig, plan_for
from paper_1805_06557_b200.workloads import seeded_linear_state

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1279
cfg = SphereConfig.for_truncation(T)
plan = plan_for(cfg)
phi = to_device(pack(seeded_linear_state(T, 0)))[0:1].contiguous()
g = plan.synthesis_dev(phi)
b = plan.analysis_dev(g)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3):
    e0.record(); plan.synthesis_dev(phi, g); e1.record(); e1.synchronize(); ts = e0.elapsed_time(e1)
    e0.record(); plan.analysis_dev(g, b); e1.record(); e1.synchronize(); ta = e0.elapsed_time(e1)
print(f"T{T} synthesis {ts:.3f} ms analysis {ta:.3f} ms err {float((b - phi).abs().max() / phi.abs().max()):.2e}")
