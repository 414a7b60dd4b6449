"""Dev tool: where the e2e time of analyze_corpus goes (text pointers, packing +
H2D + device pipeline inside exs_run_units, results copy, Analysis objects),
for a few batch sizes and packing thread counts.
    python tests/emu/e2e_probe.py [n_files] [batch_mib,...] [threads,...]"""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import bench  # noqa: E402
from paper_2309_03912_b200 import _native  # noqa: E402
from paper_2309_03912_b200 import exspace as X  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
mibs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "256,1100").split(",")]
thr = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "0,4,8").split(",")]
texts = bench.make_texts("c2", range(n), 100_000, os.cpu_count())
units = [(f"f{i}.cu", t) for i, t in enumerate(texts)]
nbytes = sum(len(t) for t in texts)
cfg = np.zeros(n, np.uint8)
for mib in mibs:
    for th in thr:
        eng = X.Engine(0, batch_mib=mib)
        eng.handle.set_option(8, th)
        for it in range(4):
            t0 = time.perf_counter()
            ptrs, lens, keep = _native.text_pointers(texts)
            t1 = time.perf_counter()
            eng.handle._check(eng.handle.lib.exs_run_units(eng.handle.h, _native._ptr(ptrs), _native._ptr(lens),
                                                           n, _native._ptr(cfg)))
            t2 = time.perf_counter()
            recs, text, first = eng.handle.results(copy=True)
            t3 = time.perf_counter()
            res = X.CorpusResults(recs, text, first, [u[0] for u in units])
            out = [X.Analysis(u[0], X.CompileProfile(), X.Mode.CLASSIC, res, f) for f, u in enumerate(units)]
            t4 = time.perf_counter()
            st = eng.handle.stats()
            t5 = time.perf_counter()
            eng.run_batch([(t, p, X.CompileProfile(), X.Mode.CLASSIC, X.TraitConfig()) for p, t in units])
            t6 = time.perf_counter()
            print(f"batch {mib} MiB threads {th}: ptrs {1e3*(t1-t0):.1f} run_units {1e3*(t2-t1):.1f} "
                  f"(wall {st['ms_wall']:.1f}, device {st['ms_total']:.1f}, batches {st['batches']}) "
                  f"copy {1e3*(t3-t2):.1f} objs {1e3*(t4-t3):.1f} | run_batch {1e3*(t6-t5):.1f} ms "
                  f"= {nbytes/(t6-t5)/1e9:.2f} GB/s", flush=True)
