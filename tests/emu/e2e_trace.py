"""Dev tool: per-batch timeline of analyze_corpus on C2 (EXS_TRACE_UNITS=1)."""
import os
import sys
import time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2309_03912_b200 import exspace as X  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
texts = bench.make_texts("c2", range(n), 100_000, os.cpu_count())
units = [(f"f{i}.cu", t) for i, t in enumerate(texts)]
eng = X.Engine(0, batch_mib=int(sys.argv[2]) if len(sys.argv) > 2 else 256)
keep = None
for it in range(4):
    t0 = time.perf_counter()
    keep = X.analyze_corpus(units, engine=eng)
    t1 = time.perf_counter()
    print(f"analyze_corpus {1e3 * (t1 - t0):.1f} ms (library wall {eng.last_stats['ms_wall']:.1f})", file=sys.stderr, flush=True)
