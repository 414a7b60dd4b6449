"""Dev tool: Python-side profile of Engine.run_batch on the C2 corpus (where the
e2e time outside exs_run_units goes)."""
import cProfile
import os
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2309_03912_b200 import exspace as X  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
texts = bench.make_texts("c2", range(n), 100_000, os.cpu_count())
units = [(t, f"f{i}.cu", X.CompileProfile(), X.Mode.CLASSIC, X.TraitConfig()) for i, t in enumerate(texts)]
eng = X.Engine(0, batch_mib=256)
keep = []
for it in range(4):
    t0 = time.perf_counter()
    r = eng.run_batch(units)
    t1 = time.perf_counter()
    keep.append(r)
    keep = keep[-1:]
    print(f"run_batch {1e3 * (t1 - t0):.1f} ms (library wall {eng.last_stats['ms_wall']:.1f})", flush=True)
pr = cProfile.Profile()
pr.enable()
r = eng.run_batch(units)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
