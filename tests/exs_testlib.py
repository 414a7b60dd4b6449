"""Shared helpers for the test suite (golden fixtures, canonical keys)."""
import gzip
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"
GOLDEN_GROUPS = ["corpus", "genunit", "snippets", "synthetic", "mutations", "semadiag"]

from oracle import exs_oracle as O  # noqa: E402


def load_golden(name):
    with gzip.open(GOLDEN / f"{name}.json.gz", "rt", encoding="utf-8") as fh:
        return json.load(fh)


def oracle_results(units, mode):
    """The oracle's diagnostics of (path, text) units as columnar results in
    the library's layout (exs_result records, message bytes, unit_first):
    stands in for a GPU engine in the CPU tests of the result plumbing."""
    import numpy as np
    from paper_2309_03912_b200._native import RESULT_DTYPE
    from paper_2309_03912_b200.messages import CODES
    rows, text, first = [], bytearray(), [0]
    for u, unit in enumerate(units):
        r = O.analyze_unit(unit[1], mode)
        for code, line, col, msg, sup in r.all_diagnostics:
            m = msg.encode("utf-8", "surrogateescape")
            rows.append((u, line, col, len(m), len(text), CODES.index(code), int(sup), (0,) * 5))
            text += m
        first.append(len(rows))
    return (np.array(rows, dtype=RESULT_DTYPE), np.frombuffer(bytes(text), dtype=np.uint8),
            np.array(first, dtype=np.uint64))


def canon_val(v):
    if isinstance(v, O.Ty):
        return v.name + ("<" + ",".join(v.targs) + ">" if v.targs else "")
    return "HDC::" + v.v


def canon_key(key):
    """Canonical text of an oracle walk key (same form as make_golden.canon_key)."""
    if key[0] == "decl":
        owner, name, params, req, spaces = key[1]
        return f"decl|{owner}|{name}|{';'.join(params)}|{req}|{spaces}"
    owner, name, params, req, spaces = key[1]
    binds = ",".join(f"{k}={canon_val(v)}" for k, v in key[2])
    ot = canon_val(key[3]) if key[3] is not None else ""
    s = f"inst|{owner}|{name}|{';'.join(params)}|{req}|{spaces}|{binds}|{ot}"
    if len(key) > 4:
        s += "|" + key[4]
    return s


PUNCT_TEXT = [None, "<<<", ">>>", "::", "==", "!=", "&&", "||", "++", "{", "}", "(", ")", "<",
              ">", ",", ";", ".", "!", "="]
TOKEN_KIND = {1: "ident", 2: "int", 3: "string", 4: "punct", 5: "pragma"}


def lex_stream_mismatches(X, eng, cases):
    """Run ``cases`` (dicts with text/compiler/relaxed/erase and the reference's
    per-pass ``lex`` record) through ``eng`` in ONE batch and compare, per pass,
    the token stream + EOF position, or the first E0002 line, or the first
    lexical error line/column.  Returns the mismatching (name, pass) pairs."""
    from paper_2309_03912_b200.messages import Renderer
    units = [(c["text"], "u.mcu", X.CompileProfile(c["compiler"], 12, c["relaxed"], c["erase"]),
              X.Mode(c.get("mode", "classic")), X.TraitConfig(c.get("fund", False))) for c in cases]
    eng.run_batch(units, want_walks=True)
    h = eng.handle
    st = h.pass_status(len(cases))
    data = b"".join(c["text"].encode() for c in cases)
    offs = [0]
    for c in cases:
        offs.append(offs[-1] + len(c["text"].encode()))
    ren = Renderer(data, offs, h.arena())
    bad = []
    for f, c in enumerate(cases):
        toks = h.tokens(f)
        for p, kind in enumerate(["host", "device"][: len(c["lex"])]):
            want = c["lex"][kind]
            s = st[2 * f + p]
            if "pp_error" in want:
                ok = s["pp_line"] == want["pp_error"][0]
            elif "lex_error" in want:
                ok = (s["pp_line"] == 0 and s["lex_line"] == want["lex_error"][0]
                      and s["lex_col"] == want["lex_error"][1])
            else:
                got = []
                for t in toks:
                    if not (int(t["mask"]) >> p) & 1:
                        continue
                    k = TOKEN_KIND[int(t["kind"])]
                    if k == "punct":
                        text = PUNCT_TEXT[int(t["id"])]
                    elif k == "int":
                        text = None
                    else:
                        text = ren.span_text((int(t["pos"]) << 32) | (int(t["end"]) - int(t["pos"])))
                    got.append([k, text, int(t["line"]), int(t["col"])])
                got.append(["eof", "", int(s["eof_line"]), int(s["eof_col"])])
                exp = [[k, (None if k == "int" else tx), ln, co] for k, tx, ln, co in want["tokens"]]
                ok = s["pp_line"] == 0 and s["lex_line"] == 0 and got == exp
            if not ok:
                bad.append((c["name"], kind))
    return bad
