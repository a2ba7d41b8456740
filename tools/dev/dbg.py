import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2509_06347_b200 import gmg
from synth import configs, state
m = configs.config(1); fs = configs.FREESTREAM[1]
W = state.gaussian_bump(m, *fs, jump=True); Winf = state.winf(*fs)
for lanes in (2, 0):
    s = gmg.Solver(m, n_levels=3, sweep_lanes=lanes)
    s.set_state(W, Winf)
    try:
        h = s.vcycle(1); print(lanes, 'hist', h[:, 0])
    except Exception as e:
        print(lanes, 'ERR', e)
    for l in (1, 2):
        for f, nm in ((gmg.FIELD_W0, 'W0'), (gmg.FIELD_DW, 'dW'), (gmg.FIELD_RS, 'Rs')):
            v = s.level_field(l, f)
            print(lanes, l, nm, np.isfinite(v).all(), np.abs(v).max())
    s.close()
