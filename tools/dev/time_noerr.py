"""DEV (timing only, state errors ignored -- for variants that skip work): time one smoothing step's sweeps per coarse level (graph replays, in-step view) and the whole
V-cycle for the sweep kernel variants selected by GMG_DEV_VAR / GMG_DEV_GRID (config 4)."""
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
s = gmg.Solver(m, n_levels=3, setup_device=1, sweep_lanes=int(os.environ.get("LANES", "0")),
               l2_persist_mb=int(os.environ.get("L2MB", "0")))
s.set_state(W, Winf)
def quiet(f, *a):
    try:
        return f(*a)
    except gmg.GmgError:
        return None


for _ in range(3):
    quiet(s.vcycle, 1)
out = {"lanes": os.environ.get("LANES", "0"), "l2mb": os.environ.get("L2MB", "0")}
for l in (1, 2):
    ms, cu, by = s.time_smooth(l, 6, 10)
    out[f"L{l}_ms"] = ms / 10
s.set_state(W, Winf)
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(2):
    torch.cuda.synchronize()
    e0.record(st)
    quiet(gmg.gmg_vcycle, s.ctx, 100, None)
    e1.record(st)
    torch.cuda.synchronize()
out["vcycle_ms"] = e0.elapsed_time(e1) / 100
print(json.dumps(out))
