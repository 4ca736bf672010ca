"""Time the pieces of EtdrkStepper.step on the GPU box (host pack/unpack, copies, step)."""
import time
import numpy as np
import torch
from paper_1805_06557_b200.device import pack_fields, unpack_fields, HostStage, ncoef, flat_index
from paper_1805_06557_b200.sphere import SphereConfig
from paper_1805_06557_b200.swe import LC_N, LG, ModelParams, PrognosticState
from paper_1805_06557_b200.steppers import EtdrkStepper
from paper_1805_06557_b200.rexi import RexiSetup
from paper_1805_06557_b200.workloads import seeded_balanced_state

T = 256
cfg = SphereConfig.for_truncation(T)
par = ModelParams(1e4 * 9.80616, cfg)
st = EtdrkStepper(LG, LC_N, par, RexiSetup(num_poles=256))
ic = seeded_balanced_state(cfg)
s0 = PrognosticState.from_stack(ic, cfg)
eng = st.engine(1800.0)
stage = HostStage(T)
def tm(f, k=30):
    for _ in range(3): f()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize()
    return round((time.perf_counter() - t) / k * 1e6, 1)
fields = (s0.phi_pert.coeffs, s0.vort.coeffs, s0.div.coeffs)
print("pack_fields us", tm(lambda: pack_fields(fields, stage.np_in)))
print("unpack_fields us", tm(lambda: unpack_fields(stage.np_out, T)))
print("h2d packed us", tm(lambda: eng.u.copy_(stage.h_in, non_blocking=True)))
print("d2h packed us", tm(lambda: stage.h_out.copy_(eng.u, non_blocking=True)))
print("step_dev us", tm(lambda: eng.step_dev()))
print("step (e2e) us", tm(lambda: st.step(s0, 1800.0)))
print("np.take one field us", tm(lambda: np.take(np.ascontiguousarray(fields[0]).reshape(-1), flat_index(T), out=stage.np_in[0])))
print("host cpus", torch.get_num_threads())
