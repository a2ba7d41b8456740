"""The multi-rank (NCCL) path's communication protocol, checked without a
multi-GPU box.  P rank processes (one GPU shared) run the
partitioned V-cycle through libgmg with a logging NCCL stand-in
(tests/native/nccl_shim.c, loaded through libgmg's GMG_NCCL_LIB hook: no
data moves, so no rank waits on another).  The recorded sequences must match
pairwise -- group k of rank r and group k of rank p hold r's sends to p and
p's receives from r with the same element counts in the same order, and the
all-reduces agree -- which is what makes the real exchange deadlock-free and
element-wise consistent (the halo groups are (color, peer) blocks, natural id
ascending).  Also counts the exchanges per V-cycle."""
import json
import os
import subprocess
import sys
import tempfile

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_RANK = r'''
import json, os, sys
sys.path.insert(0, sys.argv[1])
import torch
import torch.distributed as dist
rank, world, n = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:" + sys.argv[5], rank=rank, world_size=world)
from paper_2509_06347_b200 import gmg
from synth import configs, state
m = configs.sphere_shell(n, 6, 4)
fs = configs.FREESTREAM[5]
part = gmg.gmg_partition_rcb(m.ctr, world)
s = gmg.Solver(m, n_levels=3, part=part, nranks=world, rank=rank, nccl_id=bytes(128))
W, Winf = state.bow_shock(m, *fs), state.winf(*fs)
s.set_state(W, Winf)
try:
    s.vcycle(1)     # the shim moves no data: ghosts stay unset and the state goes non-finite; only the
except gmg.GmgError as e:   # recorded protocol matters here
    assert e.status == gmg.GMG_ENONFINITE, e
print(json.dumps({"rank": rank, "launches": s.vcycle_launches(), "cells": int(m.n_cells)}))
s.close()
dist.barrier()
'''


def _parse(path):
    groups, cur, ar = [], None, []
    for ln in open(path):
        f = ln.split()
        if f[0] == "group":
            cur = []
        elif f[0] == "end":
            groups.append(cur)
            cur = None
        elif f[0] in ("send", "recv"):
            (cur if cur is not None else groups.append([]) or groups[-1]).append((f[0], int(f[1]), int(f[2])))
        elif f[0] == "allreduce":
            ar.append(int(f[1]))
            groups.append([("allreduce", -1, int(f[1]))])
    return groups, ar


@pytest.mark.parametrize("P", [2, 4])
def test_rank_protocol_matches_pairwise(P):
    shim = os.path.join(tempfile.mkdtemp(), "libnccl_shim.so")
    subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", shim, os.path.join(ROOT, "tests", "native", "nccl_shim.c")])
    log = os.path.join(tempfile.mkdtemp(), "log")
    env = dict(os.environ, GMG_NCCL_LIB=shim, GMG_SHIM_LOG=log, CUDA_VISIBLE_DEVICES=os.environ.get("CUDA_VISIBLE_DEVICES", "0"))
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    procs = [subprocess.Popen([sys.executable, "-c", _RANK, ROOT, str(r), str(P), "16", str(port)], env=env,
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True) for r in range(P)]
    outs = [p.communicate(timeout=600) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-3000:]
    info = [json.loads(o.strip().splitlines()[-1]) for o, _ in outs]
    seqs = [_parse(f"{log}_{r}") for r in range(P)]
    ng = {len(g) for g, _ in seqs}
    assert len(ng) == 1, f"ranks recorded different numbers of groups: {ng}"
    n_groups = ng.pop()
    for k in range(n_groups):
        kinds = {r: [x[0] for x in seqs[r][0][k]] for r in range(P)}
        if any("allreduce" in v for v in kinds.values()):
            counts = {seqs[r][0][k][0][2] for r in range(P)}
            assert all(kinds[r] == ["allreduce"] for r in range(P)) and len(counts) == 1, (k, kinds)
            continue
        for r in range(P):
            for p in range(P):
                if p == r:
                    continue
                sends = [c for op, peer, c in seqs[r][0][k] if op == "send" and peer == p]
                recvs = [c for op, peer, c in seqs[p][0][k] if op == "recv" and peer == r]
                assert sends == recvs, f"group {k}: rank {r} -> {p} sends {sends}, rank {p} receives {recvs}"
    # every rank has the same all-reduces, and exchanges happened
    assert len({tuple(ar) for _, ar in seqs}) == 1
    n_sr = sum(1 for g in seqs[0][0] if g and g[0][0] != "allreduce")
    assert n_sr > 0
    out = {"P": P, "cells": info[0]["cells"], "groups_recorded": n_groups, "send_recv_groups": n_sr,
           "allreduces": len(seqs[0][1])}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"nccl_shim_P{P}.json"), "w") as f:
        json.dump(out, f)
