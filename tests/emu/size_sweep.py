"""Dev tool: per-stage device ms per MB across batch sizes (working-set / L2
effects).  Usage: size_sweep.py [n_files ...]"""
import os, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np
from paper_2309_03912_b200 import _native
import bench

ns = [int(a) for a in sys.argv[1:]] or [125, 250, 500, 1000, 2000, 4000, 10000]
N = max(ns)
blobs, offs_all = bench.make_corpus(N, 100_000, 0, os.cpu_count())
h = _native.Handle(0, os.environ.get("EXS_LIB"))
if os.environ.get("EXS_SPLIT"):  # statement-parallel body parsing threshold (tokens)
    h.set_option(3, int(os.environ["EXS_SPLIT"]))
for n in ns:
    data = np.frombuffer(b"".join(blobs[:n]), np.uint8)
    offs = np.zeros(n + 1, np.uint64); offs[1:] = np.cumsum([len(b) for b in blobs[:n]])
    cfg = np.zeros(n, np.uint8)
    for it in range(3):
        h.run(data, offs, cfg)
    st = h.stats()
    mb = st["bytes"] / 1e6
    print(f"n={n:6d} {mb:8.1f} MB  total {st['ms_total']:8.2f} ms  = {mb / st['ms_total']:.2f} GB/s |"
          + " ".join(f"{k[3:]} {1e3 * st[k] / mb:6.1f}" for k in ("ms_lex", "ms_parse", "ms_sema", "ms_walk"))
          + f" us/MB, retries {st['retries']}", flush=True)
