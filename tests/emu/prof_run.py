"""Dev tool: per-launch-site device times (EXS_PROFILE=1) for a C2 batch."""
import os, sys, time
os.environ["EXS_PROFILE"] = "1"
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np
from paper_2309_03912_b200 import synth, _native
import bench
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
blobs, offs = bench.make_corpus(n, 100_000, 0, os.cpu_count())
data = np.frombuffer(b"".join(blobs), np.uint8)
cfg = np.zeros(n, np.uint8)
h = _native.Handle(0, os.environ.get("EXS_LIB"))
for it in range(3):
    t0 = time.time(); h.run(data, offs, cfg); t1 = time.time()
st = h.stats()
print({k: (round(v, 2) if isinstance(v, float) else v) for k, v in st.items()})
print(h.lib.exs_profile_text().decode())
