"""Pin the CPU oracle against the real reference's golden vectors (CPU only)."""
import pytest

from oracle import exs_oracle as O
from exs_testlib import GOLDEN_GROUPS, canon_key, load_golden


def _lex(text, kind, compiler, relaxed):
    defined = dict(O.profile_passes(compiler, relaxed))[kind]
    try:
        pt = O.directives(text, defined)
    except O.PpError as e:
        return {"pp_error": [e.loc[0], e.loc[1], e.msg]}
    try:
        return {"tokens": [list(t) for t in O.tokens(pt)]}
    except O.SyntaxErr as e:
        return {"lex_error": [e.loc[0], e.loc[1], e.msg]}


@pytest.mark.parametrize("group", GOLDEN_GROUPS)
def test_oracle_matches_reference(group):
    bad = []
    for c in load_golden(group):
        r = O.analyze_unit(c["text"], c["mode"], c["compiler"], c["relaxed"], c["erase"], c["fund"])
        got = [[d[0], O.SEVERITY[d[0]], d[1], d[2], d[3], d[4]] for d in r.all_diagnostics]
        if got != c["diags"]:
            bad.append((c["name"], "diags", got, c["diags"]))
            continue
        for side, ent in c["walks"].items():
            w = r.walks.get(side)
            if w is None:
                bad.append((c["name"], "walk missing", side))
                continue
            n_edges = sum(len(v) for v in w.edges.values())
            if (len(w.instances), len(w.demands), n_edges) != (
                    ent["n_instances"], ent["n_demands"], ent["n_edges"]):
                bad.append((c["name"], "walk counts", side))
                continue
            if "instances" in ent:
                if sorted(canon_key(k) for k in w.instances) != ent["instances"]:
                    bad.append((c["name"], "instances", side))
                dem = sorted([canon_key(k), d, l[0], l[1]] for k, (d, l) in w.demands.items())
                if dem != ent["demands"]:
                    bad.append((c["name"], "demands", side))
                edges = sorted([canon_key(k), [canon_key(x) for x in v]] for k, v in w.edges.items())
                if edges != ent["edges"]:
                    bad.append((c["name"], "edges", side))
        if set(c["walks"]) != set(r.walks):
            bad.append((c["name"], "walk sides"))
        for kind, want in c.get("lex", {}).items():
            got = _lex(c["text"], kind, c["compiler"], c["relaxed"])
            if got != want:
                bad.append((c["name"], "lex", kind))
    assert not bad, bad[:5]


def test_oracle_lexer_fuzz():
    """The oracle's preprocess + tokenize against the reference on the lexer
    fuzz vectors (tests/golden/make_lexfuzz.py)."""
    bad = []
    for c in load_golden("lexfuzz"):
        for kind, want in c["lex"].items():
            got = _lex(c["text"], kind, c["compiler"], c["relaxed"])
            if got != want:
                bad.append((c["name"], kind))
    assert not bad, bad[:5]
