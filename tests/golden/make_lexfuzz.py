"""Generate lexer fuzz vectors from the REAL reference (build container only).

Run:  python tests/golden/make_lexfuzz.py
Writes tests/golden/lexfuzz.json.gz: seeded lexer-stress units (long
identifiers and numbers, punctuator runs, strings and comments with
delimiters inside, backslash-newline splices anywhere, pragmas, directives,
UTF-8, CR/tab/form-feed) and, per preprocessing pass, the reference's token
stream (syntax/preprocess.py + syntax/lexer.py) or its first error.
Units are concatenated in one batch by the tests, so every token boundary
lands at many offsets of the 32-byte words the GPU lexer works on.
"""
from __future__ import annotations

import gzip
import json
import random
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
from exspace.syntax.lexer import LexError, tokenize  # noqa: E402
from exspace.syntax.preprocess import CompileProfile, PreprocessorError, preprocess  # noqa: E402

OUT = Path(__file__).resolve().parent / "lexfuzz.json.gz"
PUNCT_CH = "<>:=!&|+"
SINGLE = "{}(),;."
WORDS = ["int", "bool", "void", "template", "typename", "struct", "__host__", "__device__",
         "__global__", "HDC", "Hst", "Dev", "HstDev", "printf", "main", "std", "return",
         "constexpr", "static_assert", "cuda_arch", "hdc", "release_assert", "x", "_y1"]


def ident(rng):
    r = rng.random()
    if r < 0.3:
        return rng.choice(WORDS)
    n = rng.choice([1, 2, 3, 5, 8, 13, 31, 33, 40, 70])
    s = rng.choice("abcXYZ_")
    s += "".join(rng.choice("abcdefxyz_0123456789") for _ in range(n - 1))
    return s


def number(rng):
    n = rng.choice([1, 1, 2, 3, 9, 19, 20, 21, 25, 40])
    return "".join(rng.choice("0123456789") for _ in range(n))


def fragment(rng, errors):
    r = rng.random()
    if r < 0.25:
        return ident(rng)
    if r < 0.35:
        return number(rng)
    if r < 0.40:
        return number(rng) + ident(rng)           # 12abc: int then ident
    if r < 0.55:
        if errors and rng.random() < 0.1:
            return "".join(rng.choice(PUNCT_CH) for _ in range(rng.choice([1, 2, 3, 5, 7])))
        valid = ["<<<", ">>>", "::", "==", "!=", "&&", "||", "++", "<", ">", "!", "="]
        return "".join(rng.choice(valid) for _ in range(rng.choice([1, 1, 2, 3])))
    if r < 0.65:
        return rng.choice(SINGLE)
    if r < 0.72:
        body = "".join(rng.choice(['a', ' ', '/', '*', '//', '/*', '*/', 'x1', '!', '(']) for _ in range(rng.randint(0, 6)))
        return '"' + body + '"'
    if r < 0.78:
        pick = ['a', ' ', '/', '*', '"', '\n', '**', 'z9', '/*'] if errors else ['a', ' ', '"', '\n', '*a', '**a', 'z9', ' /', '//']
        body = "".join(rng.choice(pick) for _ in range(rng.randint(0, 8)))
        return "/*" + body + "*/"
    if r < 0.82:
        return "//" + "".join(rng.choice(['a', ' ', '*/', '"', '/*']) for _ in range(rng.randint(0, 5))) + "\n"
    if r < 0.84:
        return "\\\n"
    if r < 0.86:
        return rng.choice(["é", "日本", "xé", "€" if errors else "ü"])
    if r < 0.87:
        return rng.choice(["\t", "\r", "  ", "\x0c" if errors else "\t"])
    if r < 0.885 and errors:
        return rng.choice(["@", "$", "&", "|", "/", ":", "+", '"unterminated'])
    return rng.choice([" ", " ", " ", "\n", "\n  ", "\n\t"])


def unit(rng):
    parts = []
    errors = rng.random() < 0.3
    size = rng.choice([60, 200, 500, 1200, 3000])
    n = 0
    stack = []  # else seen, per open conditional
    while n < size:
        r = rng.random()
        if r < 0.03:
            d = rng.choice(["#pragma hd_warning_disable", "#pragma nv_exec_check_disable",
                            "  #  pragma  hd_warning_disable", "#pragma x y", "#ifdef __CUDA_ARCH__",
                            "#ifndef __CUDACC__", "#else", "#endif", "#error oops", "#bogus"])
            if not errors and d in ("#error oops", "#bogus", "#pragma x y"):
                d = "#pragma hd_warning_disable"
            if d == "#else" and stack and stack[-1] and not errors:
                d = "#endif"
            if d.startswith("#if"):
                stack.append(False)
            elif d in ("#else", "#endif") and not stack:
                d = "#ifdef __CUDA_ARCH__"
                stack.append(False)
            elif d == "#else":
                stack[-1] = True
            elif d == "#endif":
                stack.pop()
            parts.append("\n" + d + "\n")
        else:
            f = fragment(rng, errors)
            parts.append(f)
            if rng.random() < 0.6:
                parts.append(rng.choice([" ", " ", "\n", "\t"]))
        n += len(parts[-1])
    parts.extend(["\n#endif\n"] * len(stack))
    text = "".join(parts)
    if rng.random() < 0.5:
        text += "\n"
    return text


def lex_ref(text, profile):
    out = {}
    for pp in profile.passes():
        try:
            pt = preprocess(text, pp, "u.mcu")
        except PreprocessorError as e:
            out[pp.kind] = {"pp_error": [e.loc.line, e.loc.col, e.message]}
            continue
        try:
            toks = tokenize(pt, "u.mcu")
            out[pp.kind] = {"tokens": [[t.kind, t.text, t.loc.line, t.loc.col] for t in toks]}
        except LexError as e:
            out[pp.kind] = {"lex_error": [e.loc.line, e.loc.col, e.message]}
    return out


def main():
    rng = random.Random(903912)
    cases = []
    for k in range(360):
        text = unit(rng)
        compiler = "plain" if k % 9 == 0 else "nvcc"
        relaxed = k % 5 == 0 and compiler == "nvcc"
        prof = CompileProfile(compiler, 12, relaxed, False)
        cases.append({"name": f"lexfuzz/{k}", "text": text, "mode": "classic", "compiler": compiler,
                      "relaxed": relaxed, "erase": False, "fund": False, "lex": lex_ref(text, prof)})
    with gzip.open(OUT, "wt", encoding="utf-8") as fh:
        json.dump(cases, fh, separators=(",", ":"))
    nt = sum(1 for c in cases for v in c["lex"].values() if "tokens" in v)
    print(f"{OUT.name}: {len(cases)} cases, {nt} token streams, {OUT.stat().st_size} bytes")


if __name__ == "__main__":
    main()
