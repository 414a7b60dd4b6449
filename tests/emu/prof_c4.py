"""Dev tool: per-launch-site device times (EXS_PROFILE=1) of one C4 unit."""
import os
import sys
os.environ["EXS_PROFILE"] = "1"
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2309_03912_b200 import exspace as X, synth  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
t = synth.gen_callgraph(n, 10, 7)
e = X.Engine(0)
for it in range(3):
    e.run_batch([(t, "c4.cu", X.CompileProfile(), X.Mode.SOUND, X.TraitConfig())])
print({k: (round(v, 2) if isinstance(v, float) else v) for k, v in e.last_stats.items()})
rows = []
for ln in e.handle.lib.exs_profile_text().decode().splitlines():
    parts = ln.split()
    if len(parts) >= 4:
        rows.append((float(parts[-3]), ln))
for ms, ln in sorted(rows, reverse=True)[:45]:
    print(ln)
