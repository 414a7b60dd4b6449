"""Dev tool: a large seeded differential run (GPU library vs the oracle) over the
synthetic generators, every mode, both profiles.  python tests/emu/diff_big.py SEED N"""
import random, sys, time
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from paper_2309_03912_b200 import exspace as X, synth
from oracle import exs_oracle as O
from concurrent.futures import ProcessPoolExecutor
rng = random.Random(int(sys.argv[1]) if len(sys.argv) > 1 else 7)
modes = [m.value for m in X.Mode]
cases = []
for k in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2000):
    kind = k % 5
    if kind == 0: t = synth.gen_c2_file(rng.randrange(10**6), rng.randrange(800, 8000))
    elif kind == 1: t = synth.gen_c5_file(rng.randrange(10**6), rng.randrange(800, 8000), rng.random())
    elif kind == 2: t = synth.gen_chain(rng.randrange(2, 16), rng.randrange(2, 24))
    elif kind == 3: t = synth.gen_callgraph(rng.randrange(5, 120), rng.randrange(1, 12), rng.randrange(10**6))
    else: t = synth.gen_c5_file(rng.randrange(10**6), rng.randrange(200, 3000), 1.0)
    cases.append((t, modes[k % 5], k % 7 == 0))
def orc(c):
    t, m, p = c
    r = O.analyze_unit(t, m, "plain" if p else "nvcc")
    return [(d[0], d[1], d[2], d[3], d[4]) for d in r.all_diagnostics]
t0 = time.time()
with ProcessPoolExecutor() as ex:
    want = list(ex.map(orc, cases, chunksize=8))
t1 = time.time()
res = X.get_engine(0).run_batch([(t, f"u{i}.cu", X.CompileProfile("plain") if p else X.CompileProfile(), X.Mode(m), X.TraitConfig()) for i, (t, m, p) in enumerate(cases)])
bad = [i for i, (a, w) in enumerate(zip(res, want)) if [(d.code, d.loc.line, d.loc.col, d.message, d.suppressed) for d in a.all_diagnostics] != w]
print(len(cases), "units,", sum(len(w) for w in want), "diagnostics; mismatches", len(bad), bad[:10], "oracle s", round(t1 - t0, 1))
