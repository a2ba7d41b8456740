"""Dev tool: per-launch device times of one V-cycle (event-bracketed, eager
launches, GMG_PROF_DUMP), with the color block sizes of every level, so that
the cost of the small color phases can be read off directly."""
import json, os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2509_06347_b200 import gmg
from synth import configs, state

k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
m = configs.config(k)
fs = configs.FREESTREAM[k]
s = gmg.Solver(m, n_levels=3)
s.set_state(state.bow_shock(m, *fs), state.winf(*fs))
s.vcycle(2)
dump = os.path.join(tempfile.mkdtemp(), "prof.txt")
os.environ["GMG_PROF_DUMP"] = dump
s.profile_vcycle(1)
rows = [l.split() for l in open(dump)]
names = ["face", "gather", "sweep", "restrict", "prolong", "norm"]
out = {"colors": {}, "launches": []}
for l in range(3):
    col = s.maps(l)[0]
    out["colors"][f"L{l}"] = np.bincount(col)[1:].tolist()
tot = {}
for c, t, b in rows:
    n = names[int(c)]
    tot[n] = tot.get(n, 0.0) + float(t)
    out["launches"].append([n, round(float(t) * 1e3, 2), int(float(b))])
out["total_ms"] = {n: round(v, 4) for n, v in tot.items()}
sw = [(t, b) for n, t, b in out["launches"] if n == "sweep"]
out["sweep_small_us"] = round(sum(t for t, b in sw if b < 5e6), 1)   # launches with < 5 MB algorithmic
out["sweep_small_count"] = sum(1 for t, b in sw if b < 5e6)
print(json.dumps(out))
