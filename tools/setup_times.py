"""Dev tool: host vs device setup (gmg_build_hierarchy) wall time on a config mesh,
with the per-phase breakdown (GMG_SETUP_TIMES) on stderr."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["GMG_SETUP_TIMES"] = "1"
from paper_2509_06347_b200 import gmg
from synth import configs

k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
P = int(sys.argv[2]) if len(sys.argv) > 2 else 1
t = time.time()
m = configs.config(k, P) if k == 5 else configs.config(k)
out = {"config": k, "P": P, "cells": int(m.vol.size), "mesh_gen_s": time.time() - t}
import torch
torch.cuda.init()
for dev in (0, 1, 0, 1):
    t = time.time()
    s = gmg.Solver(m, n_levels=3, build_only=True, setup_device=dev)
    out[f"build_s_setup_device{dev}"] = time.time() - t
    s.close()
print(json.dumps(out))
