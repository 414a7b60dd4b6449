"""Dev tool: where the e2e time goes (pinned H2D, device pipeline, D2H, diags())."""
import os, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch
from paper_2309_03912_b200 import _native
import bench
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
blobs, offs = bench.make_corpus(n, 100_000, 0, os.cpu_count())
data = np.frombuffer(b"".join(blobs), np.uint8)
host = torch.from_numpy(data.copy()).pin_memory()
cfg = np.zeros(n, np.uint8)
h = _native.Handle(0)
for it in range(4):
    t0 = time.perf_counter()
    h.lib.exs_run(h.h, _native.C.c_void_p(host.data_ptr()), data.nbytes, _native._ptr(offs), n, _native._ptr(cfg))
    t1 = time.perf_counter()
    recs = h.diags(copy=False)
    t15 = time.perf_counter()
    recs2 = h.diags()
    t2 = time.perf_counter()
    st = h.stats()
    print(f"exs_run {1e3*(t1-t0):.1f} ms (h2d {st['ms_h2d']:.1f}, device total {st['ms_total']:.1f}, d2h {st['ms_d2h']:.1f}) view {1e3*(t15-t1):.1f} ms, copy {1e3*(t2-t15):.1f} ms, {recs.nbytes/1e6:.0f} MB", flush=True)
