"""Dev tool: C4 probe at small sizes with per-kernel times."""
import os, sys, time
os.environ["EXS_PROFILE"] = "1"
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np
from paper_2309_03912_b200 import synth, _native
h = _native.Handle(0)
for n in [int(x) for x in sys.argv[1:]]:
    text = synth.gen_callgraph(n, 10, 1)
    data = np.frombuffer(text.encode(), np.uint8)
    t0 = time.time(); h.run(data, np.array([0, len(data)], np.uint64), np.array([2], np.uint8)); t1 = time.time()
    st = h.stats()
    print(n, f"wall {1e3*(t1-t0):.1f} ms", {k: st[k] for k in ("instances", "callsites", "levels", "retries", "diagnostics")}, {k: round(st[k], 1) for k in ("ms_lex", "ms_parse", "ms_sema", "ms_walk")}, flush=True)
    print(h.lib.exs_profile_text().decode(), flush=True)
