"""Dev tool: C3 (deep chains) and C4 (one large call graph) single-unit runs."""
import os, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np
from paper_2309_03912_b200 import synth, _native
h = _native.Handle(0)
def run(name, text, mode):
    data = np.frombuffer(text.encode(), np.uint8)
    offs = np.array([0, len(data)], np.uint64)
    cfg = np.array([mode], np.uint8)
    for it in range(2):
        t0 = time.time(); h.run(data, offs, cfg); t1 = time.time()
    st = h.stats()
    print(name, f"{len(data)/1e6:.1f} MB wall {1e3*(t1-t0):.1f} ms", {k: st[k] for k in ("instances", "callsites", "edges", "levels", "retries", "diagnostics")},
          {k: round(st[k], 1) for k in ("ms_lex", "ms_parse", "ms_sema", "ms_walk", "ms_total")}, flush=True)
run("C3 d64 x 1024", synth.gen_chain(64, 1024), 0)
run("C3 d64 x 10300", synth.gen_chain(64, 10300), 0)
run("C4 100k x10", synth.gen_callgraph(100_000, 10, 1), 2)
if "big" in sys.argv:
    run("C4 1M x10", synth.gen_callgraph(1_000_000, 10, 1), 2)
