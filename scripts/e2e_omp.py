import os, time, numpy as np, torch
from paper_1805_06557_b200.sphere import SphereConfig
from paper_1805_06557_b200.swe import LC_N, LG, ModelParams, PrognosticState
from paper_1805_06557_b200.steppers import EtdrkStepper
from paper_1805_06557_b200.rexi import RexiSetup
from paper_1805_06557_b200.workloads import seeded_balanced_state
from paper_1805_06557_b200.device import pack_fields, unpack_fields, HostStage
cfg = SphereConfig.for_truncation(256)
par = ModelParams(1e4 * 9.80616, cfg)
st = EtdrkStepper(LG, LC_N, par, RexiSetup(num_poles=256))
s0 = PrognosticState.from_stack(seeded_balanced_state(cfg), cfg)
eng = st.engine(1800.0)
stage = HostStage(256)
def tm(f, k=50):
    for _ in range(5): f()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize()
    return round((time.perf_counter() - t) / k * 1e6, 1)
fields = (s0.phi_pert.coeffs, s0.vort.coeffs, s0.div.coeffs)
def pack_after_gpu():
    eng.step_dev(); torch.cuda.synchronize(); pack_fields(fields, stage.np_in)
print(os.environ.get("OMP_WAIT_POLICY"), os.environ.get("OMP_NUM_THREADS"),
      "e2e", tm(lambda: st.step(s0, 1800.0)), "pack(hot)", tm(lambda: pack_fields(fields, stage.np_in)),
      "step+pack", tm(pack_after_gpu), "step", tm(lambda: (eng.step_dev(), torch.cuda.synchronize())))
