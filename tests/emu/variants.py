"""Dev tool: time library variants (build/variants/*.so, tests/emu/build_variants.sh)
on one C2 batch: stage ms and the named kernels (CUDA events, library stream),
best of 3 after 2 warm-ups; the diagnostic count must agree across variants.

Usage: variants.py N_FILES lib1.so [lib2.so ...]
"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2309_03912_b200 import _native  # noqa: E402


def main():
    n = int(sys.argv[1])
    libs = sys.argv[2:]
    blobs, offs = bench.make_corpus(n, 100_000, 0, os.cpu_count())
    data = np.frombuffer(b"".join(blobs), np.uint8)
    cfg = np.zeros(n, np.uint8)
    mb = data.nbytes / 1e6
    for lib in libs:
        h = _native.Handle(0, lib)
        for _ in range(2):
            h.run(data, offs, cfg)
        best, kbest = None, None
        for _ in range(3):
            h.set_option(2, 1)
            h.run(data, offs, cfg)
            st = h.stats()
            kern = {}
            for ln in h.lib.exs_profile_text().decode().splitlines():
                p = ln.split()
                if len(p) >= 4 and not p[0].startswith("["):
                    kern[p[0]] = kern.get(p[0], 0.0) + float(p[1])
            h.set_option(2, 0)
            if best is None or st["ms_total"] < best["ms_total"]:
                best, kbest = st, kern
        st = best
        ks = " ".join(f"{k}={v:.1f}" for k, v in sorted(kbest.items(), key=lambda kv: -kv[1])[:int(os.environ.get("TOPK", "8"))])
        print(f"{Path(lib).name}: {st['ms_total']:.1f} ms = {mb / st['ms_total']:.2f} GB/s | lex {st['ms_lex']:.1f}"
              f" parse {st['ms_parse']:.1f} sema {st['ms_sema']:.1f} walk {st['ms_walk']:.1f} | diags"
              f" {st['diagnostics']} inst {st['instances']} retries {st['retries']} | {ks}", flush=True)
        del h


if __name__ == "__main__":
    main()
