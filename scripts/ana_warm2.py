"""Two back-to-back cfg2 tendencies (for ncu --cache-control none: the second
table analysis runs with the Legendre table warm in L2)."""
import torch
from paper_1805_06557_b200.sphere import SphereConfig, plan_for
from paper_1805_06557_b200.device import to_device, pack
from paper_1805_06557_b200.workloads import seeded_balanced_state

cfg = SphereConfig.for_truncation(256)
plan = plan_for(cfg)
st = to_device(pack(seeded_balanced_state(cfg)))
for _ in range(3):
    plan.tendency_dev(3, st)
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush.zero_()
torch.cuda.synchronize()
plan.tendency_dev(3, st)
plan.tendency_dev(3, st)
torch.cuda.synchronize()
print("ok")
