"""Quick sweep-kernel experiment (dev tool): time_smooth per level for a given GMG_LPC."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_06347_b200 import gmg
from synth import configs, state
m = configs.config(4)
fs = configs.FREESTREAM[4]
W = state.bow_shock(m, *fs)
s = gmg.Solver(m, n_levels=3)
s.set_state(W, state.winf(*fs))
s.vcycle(2)
out = {"lpc": os.environ.get("GMG_LPC", "4")}
for l in range(3):
    t, cu, by = s.time_smooth(l, 6, 5)
    out[f"L{l}"] = {"Gcu/s": cu / t / 1e6, "GB/s": by / t / 1e6, "us_per_halfsweep": t * 1e3 / 60}
h = s.vcycle(5)
import torch
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); gmg.gmg_vcycle(s.ctx, 20, None); e1.record(); torch.cuda.synchronize()
out["vcycle_ms"] = e0.elapsed_time(e1) / 20
print(json.dumps(out))
