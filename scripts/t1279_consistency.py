"""T1279 tendency: table analysis (default plan) vs the column walk (SWX_SHT_TABLE=0 plan)."""
import os
import sys
import time
import torch
sys.path.insert(0, ".")
from paper_1805_06557_b200.device import pack, to_device
from paper_1805_06557_b200.sphere import ShtPlan, SphereConfig
from paper_1805_06557_b200.workloads import seeded_balanced_state

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1279
cfg = SphereConfig.for_truncation(T)
t0 = time.time()
pa = ShtPlan(cfg)
print(f"plan (table={pa.fused_stages() or 'n/a'}) {time.time() - t0:.2f}s")
st = to_device(pack(seeded_balanced_state(cfg)))
a = pa.tendency_dev(3, st)
os.environ["SWX_SHT_TABLE"] = "0"
pb = ShtPlan(cfg)
b = pb.tendency_dev(3, st)
err = float((a - b).abs().max() / b.abs().max())
print(f"T{T} tendency table vs column walk: rel Linf {err:.2e}")
