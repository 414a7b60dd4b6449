"""Units of the sharded-walk tests (tests/test_cpu_host.py): shapes that
exercise the per-level exchange -- deep template chains (many levels, new
instances created by several ranks), a call graph, lexer stressors, the
sema-diagnostic goldens (E0103/E1301/E1302/E1401), and an all-stray unit
whose diagnostics overflow the first buffer (a collective retry)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
from paper_2309_03912_b200 import synth  # noqa: E402
from exs_testlib import load_golden  # noqa: E402


def _all_stray(n):
    lines = [f"void h{i}() {{}}" for i in range(10)]
    lines += [f"__device__ void f{i}() {{ " + " ".join(f"h{(i + k) % 10}();" for k in range(10)) + " }"
              for i in range(n)]
    return "\n".join(lines + ["int main() { return 0; }"]) + "\n"


UNITS = [("c3.cu", synth.gen_chain(64, 12), "classic"), ("c3s.cu", synth.gen_chain(8, 16), "sound"),
         ("c4.cu", synth.gen_callgraph(400, 10, 3), "sound"), ("c5.cu", synth.gen_c5_file(7, 20000, 0.3), "proposal2"),
         ("c2.cu", synth.gen_c2_file(11, 20000), "fidelity"), ("stray.cu", _all_stray(16000), "sound")]
UNITS += [(c["name"], c["text"], c["mode"]) for c in load_golden("semadiag")[:40:4]]
UNITS += [(c["name"], c["text"], c["mode"]) for c in load_golden("corpus")[::9]]
