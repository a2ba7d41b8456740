"""DEV: NEXT-1 (fine_operator=1) V-cycle time and per-class kernel times on config 4 (variant libraries)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2509_06347_b200 import gmg  # noqa: E402
from synth import configs, state  # noqa: E402

m = configs.config(4)
fs = configs.FREESTREAM[4]
W, Winf = state.bow_shock(m, *fs), state.winf(*fs)
s = gmg.Solver(m, n_levels=3, fine_operator=1, setup_device=1)
s.set_state(W, Winf)
for _ in range(2):
    s.vcycle(1)
s.set_state(W, Winf)
s.set_ho_state()
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(st)
gmg.gmg_vcycle(s.ctx, 10, None)
e1.record(st)
torch.cuda.synchronize()
out = {"vcycle_ms": e0.elapsed_time(e1) / 10}
s.set_state(W, Winf)
s.set_ho_state()
pms, pcnt, pby = s.profile_vcycle(3)
for name, k in (("flux", gmg.K_HO_FLUX), ("recon", gmg.K_HO_RECON)):
    out[f"{name}_ms_per_launch"] = float(pms[k]) / max(int(pcnt[k]), 1)
print(json.dumps(out))
