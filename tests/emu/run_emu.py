"""DEVELOPER HARNESS (not a test of the product): runs the kernels' logic
compiled as sequential host code (EXS_EMU build, build/libexspace_emu.so)
against the golden vectors, to debug the CUDA sources without a GPU.
The package never loads this library."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from exs_testlib import GOLDEN_GROUPS, load_golden  # noqa: E402
from paper_2309_03912_b200 import exspace as X  # noqa: E402

LIB = ROOT / "build" / "libexspace_emu.so"


def unit_of(c):
    prof = X.CompileProfile(c["compiler"], 12, c["relaxed"], c["erase"])
    return (c["text"], "u.mcu", prof, X.Mode(c["mode"]), X.TraitConfig(c["fund"]))


def main(groups, limit=None, batch=64, verbose=3):
    eng = X.Engine(0, LIB)
    if os.environ.get("EXS_SPLIT"):  # force statement-parallel body parsing on small items
        eng.handle.set_option(3, int(os.environ["EXS_SPLIT"]))
    bad = total = 0
    for g in [g for g in groups if g != "lexfuzz"]:
        cases = load_golden(g)[:limit]
        for i in range(0, len(cases), batch):
            chunk = cases[i:i + batch]
            res = eng.run_batch([unit_of(c) for c in chunk], want_walks=True)
            for c, a in zip(chunk, res):
                total += 1
                got = [[d.code, d.severity.value, d.loc.line, d.loc.col, d.message, d.suppressed]
                       for d in a.all_diagnostics]
                ok = got == c["diags"]
                wok = True
                for side, ent in c["walks"].items():
                    w = a.walks.get(X.ExecSpace(side))
                    if w is None or (w.n_instances, w.n_edges, w.n_demands) != (
                            ent["n_instances"], ent["n_edges"], ent["n_demands"]):
                        wok = False
                if set(c["walks"]) != {s.value for s in a.walks}:
                    wok = False
                if not ok or not wok:
                    bad += 1
                    if bad <= verbose:
                        print("MISMATCH", c["name"], c["mode"], c["compiler"])
                        if not ok:
                            print("  got ", got)
                            print("  want", c["diags"])
                        if not wok:
                            print("  walks got", {k.value: (w.n_instances, w.n_edges, w.n_demands) for k, w in a.walks.items()})
                            print("  walks want", {k: (e["n_instances"], e["n_edges"], e["n_demands"]) for k, e in c["walks"].items()})
    print(f"{total - bad}/{total} match")
    if "lexfuzz" in groups or not groups:
        from exs_testlib import lex_stream_mismatches
        lb = lex_stream_mismatches(X, eng, load_golden("lexfuzz"))
        print(f"lexfuzz stream mismatches: {len(lb)}", lb[:10])
        bad += len(lb)
    return bad


if __name__ == "__main__":
    gs = sys.argv[1:] or GOLDEN_GROUPS
    sys.exit(1 if main(gs) else 0)
