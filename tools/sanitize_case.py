"""Small driver for compute-sanitizer runs (memcheck / racecheck / synccheck):
config 1 (2D) and a small 3D box, 2 V-cycles each, single domain and 2 local
domains (halo path).  Exits non-zero on any API error."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2509_06347_b200 import gmg  # noqa: E402
from synth import configs, state  # noqa: E402


def run(m, fs, W, **kw):
    s = gmg.Solver(m, n_levels=3, **kw)
    s.set_state(W, state.winf(*fs))
    h = s.vcycle(2)
    s.smooth(1, 2)
    assert np.all(np.isfinite(h))
    s.close()


m1 = configs.config(1)
fs1 = configs.FREESTREAM[1]
W1 = state.gaussian_bump(m1, *fs1, jump=True)
run(m1, fs1, W1)
run(m1, fs1, W1, part=gmg.gmg_partition_rcb(m1.ctr, 2), local_domains=2)
mb = configs.box3d(6, 5, 4, 2, seed=3)
fsb = (1.0, (0.6, 0.2, -0.1), 0.7)
run(mb, fsb, state.perturbed(mb, *fsb, eps=0.1, seed=4), fine_smoother=1)
print("sanitize case ok")
