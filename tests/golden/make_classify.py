"""Golden vectors for the classification exports, from the REAL reference
(build container only; the GPU box reads the committed fixture).

Run:  python tests/golden/make_classify.py
Reads the units of the committed fixtures (corpus, snippets, synthetic,
genunit), runs the reference's ``analyze`` + ``propagate_spaces``
(spacecheck.py:770-782) and, on the first compile pass's AST,
``struct_member_spaces`` (spacecheck.py:785-793) -- the AST parsed with the
specifier mode ``analyze`` uses for the profile (spacecheck.py:697-699) -- and writes
tests/golden/classify.json.gz:

  {"name", "text", "mode", "compiler", "relaxed", "erase", "fund",
   "spaces": {display: sorted space values},
   "structs": [[struct name, {member: sorted space values}], ...] | null}
"""
from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
OUT = Path(__file__).resolve().parent

from exspace.sema import TraitConfig  # noqa: E402
from exspace.spacecheck import Mode, analyze, propagate_spaces, struct_member_spaces  # noqa: E402
from exspace.syntax.parser import parse  # noqa: E402
from exspace.syntax.preprocess import CompileProfile, preprocess  # noqa: E402

GROUPS = ("corpus", "snippets", "synthetic", "genunit")
MAX_BYTES = 16384


def classify(c):
    profile = CompileProfile(c["compiler"], 12, c["relaxed"], c["erase"])
    try:
        a = analyze(c["text"], "u.mcu", profile, Mode(c["mode"]), TraitConfig(c["fund"]))
        spaces = {k: sorted(s.value for s in v) for k, v in propagate_spaces(a).items()}
    except (RecursionError, ValueError, IndexError, KeyError, TypeError):
        return None
    try:
        smode = ("erase" if c["erase"] else "reject") if c["compiler"] == "plain" else "keep"
        ast = parse(preprocess(c["text"], profile.passes()[0], "u.mcu"), "u.mcu", smode)
        structs = [[s.name, {m: sorted(x.value for x in v) for m, v in struct_member_spaces(s).items()}]
                   for s in ast.items if hasattr(s, "members")]
    except Exception:  # the first pass does not preprocess / lex / parse
        structs = None
    keep = ("name", "text", "mode", "compiler", "relaxed", "erase", "fund")
    return {**{k: c[k] for k in keep}, "spaces": spaces, "structs": structs}


def main():
    cases = []
    for g in GROUPS:
        with gzip.open(OUT / f"{g}.json.gz", "rt", encoding="utf-8") as fh:
            for c in json.load(fh):
                if len(c["text"].encode()) <= MAX_BYTES:
                    r = classify(c)
                    if r is not None:
                        cases.append(r)
    path = OUT / "classify.json.gz"
    with gzip.open(path, "wt", encoding="utf-8") as fh:
        json.dump(cases, fh, separators=(",", ":"))
    n_s = sum(len(c["structs"] or []) for c in cases)
    print(f"{path.name}: {len(cases)} cases, {n_s} structs, {path.stat().st_size} bytes")


if __name__ == "__main__":
    main()
