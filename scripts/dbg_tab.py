import os, sys, numpy as np, torch
from paper_1805_06557_b200.sphere import SphereConfig, plan_for
from paper_1805_06557_b200.device import to_device, pack
from paper_1805_06557_b200.workloads import seeded_balanced_state
T = int(sys.argv[1])
cfg = SphereConfig.for_truncation(T)
plan = plan_for(cfg)
st = to_device(pack(seeded_balanced_state(cfg)))
outs = [plan.tendency_dev(3, st).cpu().numpy() for _ in range(4)]
torch.cuda.synchronize()
outs2 = []
for _ in range(3):
    o = plan.tendency_dev(3, st); torch.cuda.synchronize(); outs2.append(o.cpu().numpy())
np.save(f"gpurun_out/tend_T{T}_{os.environ.get('SWX_SYNTH_TAB','1')}.npy", outs2[-1])
ref = outs2[-1]
sc = np.abs(ref).max()
print(T, os.environ.get('SWX_SYNTH_TAB'), os.environ.get('SWX_PDL'), "max", sc,
      "diffs", [float(np.abs(o - ref).max() / sc) for o in outs + outs2], "nan", [int(np.isnan(o).sum()) for o in outs+outs2])
