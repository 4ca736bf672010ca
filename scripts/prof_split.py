import time, torch, numpy as np
from paper_1805_06557_b200.steppers import build_stepper
from paper_1805_06557_b200.rexi import RexiSetup
from paper_1805_06557_b200.swe import ModelParams, PrognosticState
from paper_1805_06557_b200.sphere import SphereConfig
from paper_1805_06557_b200.workloads import seeded_balanced_state
from paper_1805_06557_b200.device import to_device, pack
cfg = SphereConfig.for_truncation(85); par = ModelParams(1e4*9.80616, cfg)
st = build_stepper("lg_rexi_lc_n_erk_ver1", par, RexiSetup(num_poles=128))
u = to_device(pack(seeded_balanced_state(cfg)))
erk, rex = st.remainder, st.linear
def tm(f, k=10):
    f(); torch.cuda.synchronize(); t=time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize(); return (time.perf_counter()-t)/k*1e3
print("erk step_dev dt/2 ms", tm(lambda: erk.step_dev(u, 300.0)))
print("rhs_dev ms", tm(lambda: erk.rhs_dev(u)))
print("rexi step_dev ms", tm(lambda: rex.step_dev(u, 600.0)))
s0 = PrognosticState.from_stack(seeded_balanced_state(cfg), cfg)
print("split step ms", tm(lambda: st.step(s0, 600.0)))
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(5): st.step(s0, 600.0)
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(15)
