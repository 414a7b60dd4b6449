"""Generate golden vectors from the REAL reference (build container only).

Run:  python tests/golden/make_golden.py
Needs /root/reference (read-only) importable; writes tests/golden/*.json.gz.
The GPU box never runs this -- it only reads the committed fixtures.

Each case records the reference's ``analyze`` output for one unit and config:
all diagnostics (with the suppressed flag) in the reference's order, and for
small units the per-pass token streams and the walk internals (instances,
demands, legal edges) in a canonical string form (``canon_key``).
"""
from __future__ import annotations

import ast as pyast
import gzip
import json
import random
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from exspace.corpus import parse_header  # noqa: E402
from exspace.sema import TraitConfig, Type  # noqa: E402
from exspace.spacecheck import Mode, analyze  # noqa: E402
from exspace.syntax.lexer import tokenize  # noqa: E402
from exspace.syntax.preprocess import CompileProfile, PreprocessorError, preprocess  # noqa: E402
from exspace.syntax.lexer import LexError  # noqa: E402
import genprog  # noqa: E402

from paper_2309_03912_b200 import synth  # noqa: E402

OUT = Path(__file__).resolve().parent
MODES = [m.value for m in Mode]
SMALL = 4096


def canon_val(v):
    if isinstance(v, Type):
        return v.name + ("<" + ",".join(a.value for a in v.targs) + ">" if v.targs else "")
    return "HDC::" + v.value


def canon_key(key):
    """Canonical text of a walk key ("decl"/"inst" tuples of spacecheck.py:256,336-337)."""
    if key[0] == "decl":
        owner, name, params, req, spaces = key[1]
        return f"decl|{owner}|{name}|{';'.join(params)}|{req}|{spaces}"
    sig = key[1]
    owner, name, params, req, spaces = sig
    binds = ",".join(f"{k}={canon_val(v)}" for k, v in key[2])
    ot = canon_val(key[3]) if key[3] is not None else ""
    s = f"inst|{owner}|{name}|{';'.join(params)}|{req}|{spaces}|{binds}|{ot}"
    if len(key) > 4:
        s += "|" + key[4].value
    return s


def run_case(name, text, mode="classic", compiler="nvcc", relaxed=False, erase=False,
             fund=False, detail=None):
    profile = CompileProfile(compiler, 12, relaxed, erase)
    try:
        a = analyze(text, "u.mcu", profile, Mode(mode), TraitConfig(fund))
    except (RecursionError, ValueError, IndexError, KeyError, TypeError):
        return None  # out-of-contract input: the reference itself crashes
    case = {
        "name": name, "text": text, "mode": mode, "compiler": compiler,
        "relaxed": relaxed, "erase": erase, "fund": fund,
        "diags": [[d.code, d.severity.value, d.loc.line, d.loc.col, d.message, d.suppressed]
                  for d in a.all_diagnostics],
    }
    if detail is None:
        detail = len(text.encode()) <= SMALL
    walks = {}
    for side, w in a.walks.items():
        ent = {"n_instances": len(w.instances), "n_demands": len(w.demands),
               "n_edges": sum(len(v) for v in w.edges.values())}
        if detail:
            ent["instances"] = sorted(canon_key(k) for k in w.instances)
            ent["demands"] = sorted(
                [canon_key(k), disp, loc.line, loc.col] for k, (disp, loc) in w.demands.items())
            ent["edges"] = sorted(
                [canon_key(k), [canon_key(c) for c in v]] for k, v in w.edges.items())
        walks[side.value] = ent
    case["walks"] = walks
    if detail:
        lex = {}
        for pp in profile.passes():
            try:
                pt = preprocess(text, pp, "u.mcu")
            except PreprocessorError as e:
                lex[pp.kind] = {"pp_error": [e.loc.line, e.loc.col, e.message]}
                continue
            try:
                toks = tokenize(pt, "u.mcu")
                lex[pp.kind] = {"tokens": [[t.kind, t.text, t.loc.line, t.loc.col] for t in toks]}
            except LexError as e:
                lex[pp.kind] = {"lex_error": [e.loc.line, e.loc.col, e.message]}
        case["lex"] = lex
    return case


def harvest_snippets():
    """String constants of the reference tests that look like MiniCU units."""
    out = []
    for f in sorted((REF / "tests").glob("test_*.py")):
        tree = pyast.parse(f.read_text())
        for node in pyast.walk(tree):
            if isinstance(node, pyast.Constant) and isinstance(node.value, str):
                s = node.value
                if ("(" in s or "{" in s or "#" in s) and len(s) >= 8:
                    out.append((f.stem, s))
    seen = set()
    uniq = []
    for stem, s in out:
        if s not in seen:
            seen.add(s)
            uniq.append((stem, s))
    return uniq


_MUT_CHARS = list('/*"\\\n#{}()<>;:=!&|+,. \tabT_0') + ["\\\n", "/*", "*/", "//", "<<<", ">>>",
                                                         "#ifdef __CUDA_ARCH__\n", "#endif\n",
                                                         "#else\n", "\r\n", "\x0c", "é"]


def mutate(rng, text):
    t = text
    for _ in range(rng.randint(1, 4)):
        if not t:
            break
        p = rng.randrange(len(t))
        op = rng.randrange(3)
        if op == 0:
            t = t[:p] + t[p + rng.randint(1, 6):]
        elif op == 1:
            t = t[:p] + rng.choice(_MUT_CHARS) + t[p:]
        else:
            t = t[:p] + rng.choice(_MUT_CHARS) + t[p + 1:]
    return t


def main():
    corpus = sorted((REF / "corpus").glob("*.mcu"))
    groups = {}

    # 1. the shipped corpus under its headers, then under every mode
    g = []
    for f in corpus:
        text = f.read_text()
        cfg = parse_header(text, Mode.CLASSIC, CompileProfile())
        p = cfg.profile
        g.append(run_case(f"corpus/{f.name}", text, cfg.mode.value, p.compiler,
                          p.relaxed_constexpr, p.erase_specifiers, detail=True))
        for m in MODES:
            if m != cfg.mode.value:
                g.append(run_case(f"corpus/{f.name}@{m}", text, m, p.compiler,
                                  p.relaxed_constexpr, p.erase_specifiers, detail=True))
    groups["corpus"] = g

    # 2. the reference's own seeded generator
    g = []
    for seed in range(120):
        u = genprog.gen_unit(random.Random(seed))
        g.append(run_case(f"genunit/{seed}", u.with_pragmas, MODES[seed % 5]))
        if seed % 3 == 0:
            g.append(run_case(f"genunit/{seed}/nop", u.without_pragmas, MODES[(seed + 2) % 5]))
    groups["genunit"] = g

    # 3. snippets from the reference tests, under several configs
    g = []
    configs = [("classic", "nvcc", False, False), ("sound", "nvcc", False, False),
               ("proposal1", "nvcc", False, False), ("proposal2", "nvcc", False, False),
               ("fidelity", "nvcc", False, False), ("classic", "nvcc", True, False),
               ("classic", "plain", False, True), ("classic", "plain", False, False)]
    for k, (stem, s) in enumerate(harvest_snippets()):
        for j, (m, c, r, e) in enumerate(configs):
            if (k + j) % 3 and j >= 2:
                continue
            g.append(run_case(f"snippet/{stem}/{k}/{m}/{c}{'R' if r else ''}{'E' if e else ''}",
                              s, m, c, r, e, fund=(k % 7 == 0 and j == 0)))
    groups["snippets"] = g

    # 4. synthetic shapes of the bench configs (small instances)
    g = []
    for seed in range(6):
        g.append(run_case(f"c2/{seed}", synth.gen_c2_file(seed, 6000), "classic"))
    g.append(run_case("c2/big", synth.gen_c2_file(99, 30000), "classic", detail=False))
    for m in MODES:
        g.append(run_case(f"c3/{m}", synth.gen_chain(6, 12), m, detail=True))
    g.append(run_case("c3/classic/deep", synth.gen_chain(16, 24), "classic", detail=False))
    g.append(run_case("c4/small", synth.gen_callgraph(60, 4, 1), "sound", detail=True))
    g.append(run_case("c4/classic", synth.gen_callgraph(300, 10, 2), "classic", detail=False))
    for seed in range(16):
        g.append(run_case(f"c5/{seed}", synth.gen_c5_file(seed, 5000, 0.4), MODES[seed % 5],
                          detail=True))
    groups["synthetic"] = g

    # 5. byte-level mutations of the corpus (lexer/parser error paths)
    g = []
    rng = random.Random(2309)
    texts = [f.read_text() for f in corpus]
    for k in range(700):
        base = texts[k % len(texts)]
        g.append(run_case(f"mut/{k}", mutate(rng, base), MODES[k % 5],
                          "plain" if k % 11 == 0 else "nvcc", False, k % 22 == 0, detail=True))
    groups["mutations"] = g

    for name, cases in groups.items():
        cases = [c for c in cases if c is not None]
        path = OUT / f"{name}.json.gz"
        with gzip.open(path, "wt", encoding="utf-8") as fh:
            json.dump(cases, fh, separators=(",", ":"))
        print(f"{path.name}: {len(cases)} cases, {path.stat().st_size} bytes")


if __name__ == "__main__":
    main()
