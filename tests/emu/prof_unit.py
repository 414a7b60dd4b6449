"""Dev tool: per-launch-site device times (EXS_PROFILE=1) of one synthetic unit.
    python tests/emu/prof_unit.py c3|c4 [size]"""
import os
import sys
os.environ["EXS_PROFILE"] = "1"
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2309_03912_b200 import exspace as X, synth  # noqa: E402
kind = sys.argv[1] if len(sys.argv) > 1 else "c3"
if kind == "c3":
    t, mode = synth.gen_chain(64, int(sys.argv[2]) if len(sys.argv) > 2 else 10_300), X.Mode.CLASSIC
else:
    t, mode = synth.gen_callgraph(int(sys.argv[2]) if len(sys.argv) > 2 else 10_000_000, 10, 7), X.Mode.SOUND
e = X.Engine(0)
for it in range(3):
    e.run_batch([(t, "u.cu", X.CompileProfile(), mode, X.TraitConfig())])
print({k: (round(v, 2) if isinstance(v, float) else v) for k, v in e.last_stats.items()})
rows = []
for ln in e.handle.lib.exs_profile_text().decode().splitlines():
    parts = ln.split()
    if len(parts) >= 4:
        rows.append((float(parts[-3]), ln))
for ms, ln in sorted(rows, reverse=True)[:50]:
    print(ln)
