"""Device ETD2RK step time at a large truncation (no table, non-fused tendency path)."""
import sys
import time
import torch
sys.path.insert(0, ".")
from paper_1805_06557_b200.rexi import RexiSetup
from paper_1805_06557_b200.sphere import SphereConfig
from paper_1805_06557_b200.steppers import EtdrkStepper
from paper_1805_06557_b200.swe import LC_N, LG, ModelParams
from paper_1805_06557_b200.workloads import seeded_balanced_state

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1279
dt = float(sys.argv[2]) if len(sys.argv) > 2 else 300.0
cfg = SphereConfig.for_truncation(T)
par = ModelParams(1e4 * 9.80616, cfg)
eng = EtdrkStepper(LG, LC_N, par, RexiSetup(num_poles=256)).engine(dt)
eng.load(seeded_balanced_state(cfg))
eng.step_dev()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    eng.step_dev()
e1.record()
e1.synchronize()
print(f"T{T} ETD2RK step {e0.elapsed_time(e1) / 5:.3f} ms, finite={bool(torch.isfinite(eng.u).all())}")
