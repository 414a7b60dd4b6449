"""Dev tool: one-GPU measurements of the SURVEY.md 8(d) configurations other than
the bench's C2 (C3 chains, C4 call graphs, C5 lexer stressors).  Device times
from the library's CUDA events; synthetic inputs from paper_2309_03912_b200.synth.

Usage: configs_run.py [c5] [c4big]
"""
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

from paper_2309_03912_b200 import _native, synth  # noqa: E402


def _c5(seed):
    return synth.gen_c5_file(seed, 100_000, 0.01).encode()


def run(h, name, blobs, mode):
    data = np.frombuffer(b"".join(blobs), np.uint8)
    offs = np.zeros(len(blobs) + 1, np.uint64)
    offs[1:] = np.cumsum([len(b) for b in blobs])
    cfg = np.full(len(blobs), mode, np.uint8)
    best = None
    for _ in range(3):
        h.run(data, offs, cfg)
        st = h.stats()
        if best is None or st["ms_total"] < best["ms_total"]:
            best = st
    mb = data.nbytes / 1e6
    st = best
    print(f"{name}: {mb:.1f} MB, {len(blobs)} files -> {st['ms_total']:.1f} ms = {mb / st['ms_total']:.2f} GB/s;"
          f" lex {st['ms_lex']:.1f} ({mb / st['ms_lex']:.1f} GB/s) parse {st['ms_parse']:.1f} sema {st['ms_sema']:.1f}"
          f" walk {st['ms_walk']:.1f} ms; tokens {st['tokens']}, directives {st['directives']}, instances {st['instances']},"
          f" edges {st['edges']} ({st['edges'] / st['ms_walk'] / 1e3:.1f} M edges/s in the walk), diagnostics {st['diagnostics']},"
          f" retries {st['retries']}", flush=True)


def main():
    h = _native.Handle(0)
    args = sys.argv[1:]
    if not args or "c5" in args:
        with mp.Pool(os.cpu_count()) as pool:
            blobs = pool.map(_c5, range(10_000), chunksize=16)
        run(h, "C5 stressors 1k x 100 KB", blobs[:1000], 2)   # sound mode
        run(h, "C5 stressors 10k x 100 KB", blobs, 2)
        del blobs
    if "c4big" in args:
        t0 = time.time()
        text = synth.gen_callgraph(10_000_000, 10, 1).encode()
        print(f"generated C4 10M in {time.time() - t0:.0f} s, {len(text) / 1e6:.0f} MB", flush=True)
        run(h, "C4 10M functions x 10 calls", [text], 2)


if __name__ == "__main__":
    main()
