"""Oracle verdict (blow-up step or stable) of selected cfg3 cases at T256, for
tests/golden/cfg3_verdicts.json.  Test infrastructure: runs the oracle ETD2RK
(oracle/stepping.py) with the reference's blow-up check (steppers.py:516-520:
synthesis of phi', max |phi'| > 1e6, or non-finite)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import rexi as orx  # noqa: E402
from oracle import sht as osh  # noqa: E402
from oracle import stepping as ost  # noqa: E402
from paper_1805_06557_b200.workloads import stiffness_cases  # noqa: E402

want = [tuple(map(float, a.split(","))) for a in sys.argv[1:]] or None
grid = osh.grid_for(256)
ic = ost.seeded_balanced_state(grid)
out = {}
for case in stiffness_cases():
    if want and (case.phibar_g, case.dt) not in want:
        continue
    model = orx.Model(256, case.phibar)
    sets = {k: ost.contour_coeffs(k, 10.0, case.p1, case.n_poles) for k in (0, 1, 2)}
    u, blow, t0 = ic, None, time.time()
    for k in range(1, case.steps + 1):
        u = ost.etdrk2_step(model, grid, case.dt, sets, u)
        phi = grid.synthesis(u[0])
        if not np.all(np.isfinite(u)) or not np.all(np.isfinite(phi)) or np.max(np.abs(phi)) > 1e6:
            blow = k
            break
    key = f"{case.phibar_g:.0f},{case.dt:.0f}"
    out[key] = {"blow_up_step": blow, "steps": case.steps, "p1": case.p1, "n_poles": case.n_poles}
    print(key, out[key], f"{time.time() - t0:.0f}s", flush=True)
json.dump(out, open("tests/golden/cfg3_verdicts.json", "w"), indent=1)
