"""A/B of host-edge variants of EtdrkStepper.step at cfg2 (GPU box)."""
import time
import numpy as np
import torch
from paper_1805_06557_b200.device import pack_fields, unpack_fields, HostStage
from paper_1805_06557_b200.sphere import SphereConfig, SpectralField
from paper_1805_06557_b200.swe import LC_N, LG, ModelParams, PrognosticState
from paper_1805_06557_b200.steppers import EtdrkStepper
from paper_1805_06557_b200.rexi import RexiSetup
from paper_1805_06557_b200.workloads import seeded_balanced_state

T = 256
cfg = SphereConfig.for_truncation(T)
par = ModelParams(1e4 * 9.80616, cfg)
st = EtdrkStepper(LG, LC_N, par, RexiSetup(num_poles=256))
s0 = PrognosticState.from_stack(seeded_balanced_state(cfg), cfg)
eng = st.engine(1800.0)
stage = HostStage(T)
evs = [torch.cuda.Event() for _ in range(3)]


def v0(s):
    return st.step(s, 1800.0)


def v1(s):  # per-field pack + async H2D (no extra syncs)
    fields = (s.phi_pert.coeffs, s.vort.coeffs, s.div.coeffs)
    for k in range(3):
        pack_fields((fields[k],), stage.np_in[k:k + 1])
        eng.u[k].copy_(stage.h_in[k], non_blocking=True)
    eng._step_plain()
    f = stage.download(eng.u)
    return PrognosticState(SpectralField(f[0]), SpectralField(f[1]), SpectralField(f[2]), cfg)


def v2(s):  # v1 + per-field D2H with events, unpack overlapping the next copy
    fields = (s.phi_pert.coeffs, s.vort.coeffs, s.div.coeffs)
    for k in range(3):
        pack_fields((fields[k],), stage.np_in[k:k + 1])
        eng.u[k].copy_(stage.h_in[k], non_blocking=True)
    eng._step_plain()
    for k in range(3):
        stage.h_out[k].copy_(eng.u[k], non_blocking=True)
        evs[k].record()
    f = []
    for k in range(3):
        evs[k].synchronize()
        f += unpack_fields(stage.np_out[k:k + 1], T)
    return PrognosticState(SpectralField(f[0]), SpectralField(f[1]), SpectralField(f[2]), cfg)


def v3(s):  # v1 upload, one D2H, unpack (as v0 download)
    return v1(s)


def tm(fn, k=60):
    x = s0
    for _ in range(5):
        x = fn(s0)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(k):
        x = fn(s0)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / k * 1e6, x


ref = v0(s0).stack()
for name, fn in (("v0 plain", v0), ("v1 field-upload", v1), ("v2 field-up+down", v2),
                 ("v0 plain", v0), ("v1 field-upload", v1), ("v2 field-up+down", v2)):
    us, x = tm(fn)
    print(f"{name:20s} {us:7.1f} us  same={np.array_equal(x.stack(), ref)}")
t = time.perf_counter()
for _ in range(60):
    eng._step_plain()
torch.cuda.synchronize()
print("graph only", (time.perf_counter() - t) / 60 * 1e6)
