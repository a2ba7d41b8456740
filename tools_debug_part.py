import numpy as np, sys, os
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import oracle as orc
from paper_2509_06347_b200 import gmg
from synth import configs, state
m = configs.config(1); fs = configs.FREESTREAM[1]
W = state.gaussian_bump(m, *fs, jump=True); Winf = state.winf(*fs)
P = 2
part = gmg.gmg_partition_rcb(m.ctr, P)
for nl in (1, 2, 3):
    s = gmg.Solver(m, n_levels=nl, part=part, local_domains=P)
    s.set_state(W, Winf)
    R, a, S = s.residual(0)
    H = orc.build_hierarchy(m, nl, 0.5, part=part)
    Ro, ao, So, rf = orc.residual(H[0]["level"], W, Winf)
    print("nl", nl, "res err", np.abs(R - Ro).max(), np.abs(S - So).max(), "W back", np.abs(s.get_state(0) - W).max())
    try:
        h = s.vcycle(1)
        Wo, ho = orc.vcycle(H, W, Winf, orc.Options(n_levels=nl), 1)
        print("  hist", h[:, 0], ho[:, 0], "W err", np.abs(s.get_state(0) - Wo).max())
    except Exception as e:
        print("  vcycle failed:", e)
        for l in range(nl):
            Wl = s.get_state(l); print("   level", l, "nan count", np.isnan(Wl).sum(), Wl.shape)
