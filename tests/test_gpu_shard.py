"""The one-unit sharded walk with the CUDA kernels.

The CPU test (`test_cpu_host.py::test_one_unit_walk_sharded_over_gloo_equals_one_rank`)
checks the exchange protocol with the kernels' logic compiled as host code.  Here the
same protocol runs with the sm_100a library: two processes on the one GPU of this
machine, each walking its share of every level with the real kernels, exchanging
new instances, edge slots, launch seeds and diagnostics through host copies over
gloo (`shard.make_allgather(stage_host=True)`).  This is a functional check of the
device code path (the ranks never wait on each other on the device), not a
multi-GPU measurement: diagnostics, walk counts and walk keys must equal the
one-process run.
"""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu

WORKER = r"""
import os, sys, json
sys.path.insert(0, @ROOT@); sys.path.insert(0, @TESTS@)
import torch.distributed as dist
from paper_2309_03912_b200 import exspace as X
from paper_2309_03912_b200.shard import analyze_unit_sharded
from shard_units import UNITS
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:@PORT@", rank=rank, world_size=world)
eng = X.Engine(0)
out = []
for name, text, mode in UNITS:
    a = analyze_unit_sharded(text, name, rank, world, mode=X.Mode(mode), engine=eng, device="cuda:0",
                             want_walks=True, stage_host=True)
    out.append(ROW(a))
if rank == 0:
    print(json.dumps(out))
dist.destroy_process_group()
"""

ROW_SRC = r"""
def ROW(a):
    rows = [[d.code, d.loc.line, d.loc.col, d.message, d.suppressed] for d in a.all_diagnostics]
    walks = {k.value: [w.n_instances, w.n_edges, w.n_demands, sorted(w.instances),
                       sorted([k2, v] for k2, v in w.edges.items()),
                       sorted([k2, d, l[0], l[1]] for k2, (d, l) in w.demands.items())]
             for k, w in a.walks.items()}
    return [rows, walks]
"""


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_one_unit_walk_sharded_two_ranks_on_the_gpu_equals_one_rank():
    port = _free_port()
    code = (ROW_SRC + WORKER).replace("@ROOT@", repr(str(ROOT))).replace("@TESTS@", repr(str(ROOT / "tests")))
    code = code.replace("@PORT@", str(port))
    procs = []
    for rank in range(2):
        env = dict(os.environ, RANK=str(rank), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1")
        procs.append(subprocess.Popen([sys.executable, "-c", code], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=900) for p in procs]
    assert all(p.returncode == 0 for p in procs), [o[1][-2000:] for o in outs]
    got = json.loads(outs[0][0].strip().splitlines()[-1])

    sys.path.insert(0, str(ROOT / "tests"))
    from shard_units import UNITS
    from paper_2309_03912_b200 import exspace as X
    ns = {}
    exec(ROW_SRC, ns)
    eng = X.get_engine(0)
    want = []
    for name, text, mode in UNITS:
        a = eng.run_batch([(text, name, X.CompileProfile(), X.Mode(mode), X.TraitConfig())], want_walks=True)[0]
        want.append(json.loads(json.dumps(ns["ROW"](a))))
    bad = [UNITS[i][0] for i, (g, w) in enumerate(zip(got, want)) if g != w]
    assert not bad, bad
