import time, json, sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2509_06347_b200 import gmg
from synth import configs, state
m = configs.config(4); fs = configs.FREESTREAM[4]
W, Winf = state.bow_shock(m, *fs), state.winf(*fs)
s = gmg.Solver(m, n_levels=3, setup_device=1)
s.set_state(W, Winf); s.vcycle(2)
winf = np.asarray(Winf, dtype=np.float64)
bufs = [torch.from_numpy(np.ascontiguousarray(W)).pin_memory()]; bufs.append(torch.empty_like(bufs[0]).pin_memory())
def sync_step(k):
    gmg.gmg_set_state(s.ctx, bufs[k % 2], winf); gmg.gmg_vcycle(s.ctx, 1, None); gmg.gmg_get_state(s.ctx, 0, bufs[(k + 1) % 2])
def async_step(k):
    gmg.gmg_set_state_async(s.ctx, bufs[k % 2], winf); gmg.gmg_vcycle_async(s.ctx, 1); gmg.gmg_get_state_async(s.ctx, bufs[(k + 1) % 2]); gmg.gmg_sync(s.ctx)
out = {}
for name, f in (("sync", sync_step), ("async", async_step), ("sync2", sync_step), ("async2", async_step)):
    for k in range(3): f(k)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for k in range(20): f(k)
    torch.cuda.synchronize(); out[name] = (time.perf_counter() - t0) / 20 * 1e3
print(json.dumps(out))
