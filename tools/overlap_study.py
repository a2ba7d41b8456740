"""Dev tool: V-cycle time of the partitioned path on one GPU (local domains),
exchange overlap on/off (gmg_options.overlap), and the agreement of the two."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2509_06347_b200 import gmg
from synth import configs, state

k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
m = configs.config(k)
fs = configs.FREESTREAM[k]
W = state.bow_shock(m, *fs)
out = {"config": k, "n_cells": int(m.vol.size)}
for P in (1, 2, 4):
    part = gmg.gmg_partition_rcb(m.ctr, P) if P > 1 else None
    ref = None
    for ov in (0, 1):  # gmg_options.overlap (default -1: off for local domains, on for NCCL ranks)
        s = gmg.Solver(m, n_levels=3, part=part, local_domains=P, overlap=ov) if P > 1 else gmg.Solver(m, n_levels=3)
        s.set_state(W, state.winf(*fs))
        h = s.vcycle(3)
        Wn = s.get_state()
        if ref is None:
            ref = Wn
        dev = float(np.abs(Wn - ref).max() / np.abs(ref).max())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        gmg.gmg_vcycle(s.ctx, 20, None)
        e1.record()
        torch.cuda.synchronize()
        out[f"P{P}_overlap{ov}"] = {"vcycle_ms": e0.elapsed_time(e1) / 20, "launches": s.vcycle_launches(),
                                    "rel_dev_vs_overlap0": dev}
        s.close()
        if P == 1:
            break
print(json.dumps(out))
