"""Race and bounds evidence for the hot kernels (compute-sanitizer is closed on
this GPU pool: profiles/r02/sanitizer_unavailable.txt).

* Repeat determinism: every kernel of the ETD2RK step graph (warp-specialised
  DMMA synthesis with its mbarrier hand-off, fused grid stage, TMA/mbarrier
  table analysis, lg pole sums with PDL) and the l-group chain kernel (pivot
  cache streamed through a bulk-copy ring) is run many times on the same
  input; a shared-memory or cross-CTA race shows up as a bitwise difference
  between runs.
* Hand-off: the pole sum that starts on columns as the table analysis
  completes them (generation-counted, no stream-order wait) is checked across
  back-to-back steps against steps with a full synchronisation in between.
* Canaries: outputs are written into the middle of larger buffers whose
  guard regions hold a NaN bit pattern; a write outside the output slice
  (a bad index or a tail CTA) changes a guard word.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1805_06557_b200.device import ncoef, pack, to_device  # noqa: E402
from paper_1805_06557_b200.rexi import RexiSetup  # noqa: E402
from paper_1805_06557_b200.solvers import ShiftedLinearSolver  # noqa: E402
from paper_1805_06557_b200.sphere import SphereConfig, plan_for  # noqa: E402
from paper_1805_06557_b200.steppers import EtdrkStepper  # noqa: E402
from paper_1805_06557_b200.swe import L, LC_N, LG, ModelParams  # noqa: E402
from paper_1805_06557_b200.workloads import seeded_balanced_state, seeded_linear_state  # noqa: E402

GUARD = 4096  # complex128 guard words on each side
NAN_BITS = np.frombuffer(np.uint64(0x7FF8DEADBEEF0001).tobytes(), dtype=np.float64)[0]


def guarded(n: int):
    """(buffer, view): a complex128 buffer with NaN-pattern guards around a
    length-n output view."""
    buf = torch.full((2 * (n + 2 * GUARD),), NAN_BITS, dtype=torch.float64, device="cuda")
    buf = torch.view_as_complex(buf.view(-1, 2))
    return buf, buf[GUARD:GUARD + n]


def guards_intact(buf, n: int) -> bool:
    raw = torch.view_as_real(buf).reshape(-1).view(torch.int64).cpu().numpy()
    pat = np.frombuffer(np.float64(NAN_BITS).tobytes(), dtype=np.int64)[0]
    lo, hi = raw[:2 * GUARD], raw[2 * (GUARD + n):]
    return bool(np.all(lo == pat) and np.all(hi == pat))


@pytest.mark.parametrize("trunc", [63, 85, 256])
def test_etdrk_step_graph_repeat_bitwise(trunc):
    """30 replays of the captured ETD2RK step from the same state: identical bits
    (the step includes the analysis -> pole-sum column hand-off, whose early
    starts are most likely at small T where the kernels co-reside)."""
    g = 9.80616
    cfg = SphereConfig.for_truncation(trunc)
    par = ModelParams(1e4 * g, cfg)
    st = EtdrkStepper(LG, LC_N, par, RexiSetup(num_poles=256 if trunc == 256 else 128))
    eng = st.engine(1800.0)
    u0 = to_device(pack(seeded_balanced_state(cfg)))
    outs = []
    for _ in range(30):
        eng.u.copy_(u0)
        eng.step_dev()
        outs.append(eng.u.clone())
    torch.cuda.synchronize()
    ref = outs[0]
    assert torch.isfinite(torch.view_as_real(ref)).all()
    for k, o in enumerate(outs[1:], 1):
        assert torch.equal(o, ref), f"replay {k} differs"


def test_tendency_repeat_bitwise_and_guards():
    """The T256 tendency (synthesis -> grid stage -> table analysis) 50 times
    into a guarded output: identical bits, guards untouched."""
    cfg = SphereConfig.for_truncation(256)
    plan = plan_for(cfg)
    st = to_device(pack(seeded_balanced_state(cfg)))
    n = 3 * ncoef(256)
    buf, out = guarded(n)
    out = out.view(3, -1)
    ref = None
    for _ in range(50):
        plan.tendency_dev(3, st, out)
        cur = out.clone()
        if ref is None:
            ref = cur
        assert torch.equal(cur, ref)
    torch.cuda.synchronize()
    assert guards_intact(buf, n)


@pytest.mark.parametrize("group,trunc,n_poles", [(LG, 256, 256), (L, 128, 256), (L, 42, 100)])
def test_pole_sum_repeat_bitwise_and_guards(group, trunc, n_poles):
    """The fused pole sums (lg two-mode kernel; l chains over the pivot cache
    and the tree combine, including a pole count that is not a multiple of
    32): identical bits over 40 runs, guards untouched."""
    cfg = SphereConfig.for_truncation(trunc)
    par = ModelParams(1e4 * 9.80616, cfg)
    c = RexiSetup(num_poles=n_poles).coefficients("psi0", 1800.0)
    solver = ShiftedLinearSolver(group, 1800.0, par)
    rhs = to_device(pack(seeded_linear_state(trunc, 3)))[None]
    betas = to_device(np.asarray(c.betas, dtype=np.complex128).reshape(1, -1))
    n = 3 * ncoef(trunc)
    buf, out = guarded(n)
    out = out.view(1, 3, -1)
    ref = None
    for _ in range(40):
        solver.rexi_sum_dev(c.alphas, betas, rhs, out)
        cur = out.clone()
        if ref is None:
            ref = cur
        assert torch.equal(cur, ref)
    torch.cuda.synchronize()
    assert guards_intact(buf, n)


@pytest.mark.parametrize("trunc", [42, 85])
def test_handoff_steps_equal_synchronised_steps(trunc):
    """Ten back-to-back captured ETD2RK steps (each pole sum may start while
    the preceding analysis still runs, and the next step's kernels launch
    early) equal ten steps with a device synchronisation after each: bitwise."""
    g = 9.80616
    cfg = SphereConfig.for_truncation(trunc)
    par = ModelParams(1e4 * g, cfg)
    st = EtdrkStepper(LG, LC_N, par, RexiSetup(num_poles=256))
    eng = st.engine(900.0)
    u0 = to_device(pack(seeded_balanced_state(cfg)))
    eng.u.copy_(u0)
    for _ in range(10):
        eng.step_dev()
    back_to_back = eng.u.clone()
    eng.u.copy_(u0)
    for _ in range(10):
        eng.step_dev()
        torch.cuda.synchronize()
    assert torch.equal(back_to_back, eng.u)
