"""Dev tool: one C2 batch through the library (for ncu captures)."""
import os, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np
from paper_2309_03912_b200 import _native
import bench
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
blobs, offs = bench.make_corpus(n, 100_000, 0, os.cpu_count())  # noqa
data = np.frombuffer(b"".join(blobs), np.uint8)
h = _native.Handle(0)
for _ in range(reps):
    h.run(data, offs, np.zeros(n, np.uint8))
print(h.stats())
