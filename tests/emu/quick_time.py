"""Quick GPU timing probe (dev): C2-shaped batch through the engine."""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np
from paper_2309_03912_b200 import synth, _native
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
texts = [synth.gen_c2_file(i, 100_000) for i in range(min(n, 64))]
blobs = [t.encode() for t in texts]
blobs = [blobs[i % len(blobs)] for i in range(n)]
offs = np.zeros(n + 1, np.uint64); offs[1:] = np.cumsum([len(b) for b in blobs])
data = np.frombuffer(b"".join(blobs), np.uint8)
cfg = np.zeros(n, np.uint8)
h = _native.Handle(0)
for it in range(3):
    t0 = time.time(); h.run(data, offs, cfg); t1 = time.time()
    st = h.stats()
    print(f"run {it}: wall {1e3*(t1-t0):.1f} ms, bytes {st['bytes']/1e6:.1f} MB", {k: round(v, 2) if isinstance(v, float) else v for k, v in st.items()})
