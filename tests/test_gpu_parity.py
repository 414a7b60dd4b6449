"""GPU parity: the sm_100a pipeline (through the C ABI) against the reference's
golden vectors and against the CPU oracle on seeded synthetic corpora.

Bar: bit-exact ordered diagnostics (code, severity, line, col, message,
suppressed) and identical per-walk instance / legal-edge / demand counts.
Out of contract (excluded): units the reference itself crashes on.
"""
import random

import pytest

from exs_testlib import GOLDEN_GROUPS, lex_stream_mismatches, load_golden
from oracle import exs_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def X():
    from paper_2309_03912_b200 import exspace
    return exspace


@pytest.fixture(scope="module")
def eng(X):
    return X.Engine(0)


def unit_of(X, c, path="u.mcu"):
    prof = X.CompileProfile(c["compiler"], 12, c["relaxed"], c["erase"])
    return (c["text"], path, prof, X.Mode(c["mode"]), X.TraitConfig(c["fund"]))


def as_rows(a):
    return [[d.code, d.severity.value, d.loc.line, d.loc.col, d.message, d.suppressed]
            for d in a.all_diagnostics]


@pytest.fixture(scope="module")
def eng_split(X):
    """An engine that parses every function body of >= 4 tokens statement-
    parallel (run_parse step 4b), so the golden vectors exercise that path."""
    e = X.Engine(0)
    e.handle.set_option(3, 4)
    return e


@pytest.fixture(scope="module")
def eng_flag(X):
    """An engine whose ordered selections all take the flag pass + flagged
    compaction (csrc/exs_par.cuh select_idx), which by default only inputs of
    >= 4M indices reach."""
    e = X.Engine(0)
    e.handle.set_option(4, 0)
    return e


@pytest.mark.parametrize("split", [False, True], ids=["items", "stmt_split"])
@pytest.mark.parametrize("group", GOLDEN_GROUPS)
def test_golden_vectors(X, eng, eng_split, group, split):
    cases = load_golden(group)
    res = (eng_split if split else eng).run_batch([unit_of(X, c) for c in cases], want_walks=True)
    bad = []
    for c, a in zip(cases, res):
        if as_rows(a) != c["diags"]:
            bad.append((c["name"], as_rows(a)[:3], c["diags"][:3]))
            continue
        sides = {s.value for s in a.walks}
        if sides != set(c["walks"]):
            bad.append((c["name"], "walk sides", sides))
            continue
        for side, ent in c["walks"].items():
            w = a.walks[X.ExecSpace(side)]
            if (w.n_instances, w.n_edges, w.n_demands) != (
                    ent["n_instances"], ent["n_edges"], ent["n_demands"]):
                bad.append((c["name"], side, (w.n_instances, w.n_edges, w.n_demands),
                            (ent["n_instances"], ent["n_edges"], ent["n_demands"])))
    assert not bad, bad[:5]


@pytest.mark.parametrize("source", ["golden", "lexfuzz"])
def test_golden_token_streams(X, eng, source):
    """K1-K3 lexer parity: per-pass token streams / first E0002 / LexError,
    against the reference's own preprocess + tokenize."""
    if source == "golden":
        cases = [c for g in ("corpus", "mutations", "synthetic") for c in load_golden(g) if "lex" in c]
    else:
        cases = load_golden("lexfuzz")
    bad = lex_stream_mismatches(X, eng, cases)
    assert not bad, bad[:8]


def _oracle_rows(text, mode):
    r = O.analyze_unit(text, mode)
    rows = [[d[0], O.SEVERITY[d[0]], d[1], d[2], d[3], d[4]] for d in r.all_diagnostics]
    walks = {w.native: (len(w.instances), sum(len(v) for v in w.edges.values()))
             for w in r.walks.values()}
    return rows, walks, O.edge_count(r)


def _check_against_oracle(X, eng, texts, modes):
    units = [(t, f"f{i:05d}.cu", X.CompileProfile(), X.Mode(m), X.TraitConfig())
             for i, (t, m) in enumerate(zip(texts, modes))]
    res = eng.run_batch(units, want_walks=True)
    callsites = 0
    want_calls = 0
    for t, m, a in zip(texts, modes, res):
        rows, walks, ec = _oracle_rows(t, m)
        assert as_rows(a) == rows
        for side, (ni, ne) in walks.items():
            w = a.walks[X.ExecSpace(side)]
            assert (w.n_instances, w.n_edges) == (ni, ne)
        want_calls += ec
    callsites = eng.last_stats["callsites"]
    assert callsites == want_calls


@pytest.mark.parametrize("flagged", [False, True], ids=["select_if", "select_flagged"])
def test_c2_files_vs_oracle(X, eng, eng_flag, flagged):
    eng = eng_flag if flagged else eng
    from paper_2309_03912_b200 import synth
    texts = [synth.gen_c2_file(1000 + s, 15000) for s in range(8)]
    _check_against_oracle(X, eng, texts, ["classic", "sound", "fidelity", "proposal1"] * 2)


def test_c2_100kb_files_vs_oracle(X, eng):
    """Full-size C2 files (the bench's ~100 KB shape, seeds the bench times)."""
    from paper_2309_03912_b200 import synth
    texts = [synth.gen_c2_file(s, 100_000) for s in (0, 1, 4242)]
    _check_against_oracle(X, eng, texts, ["classic", "sound", "proposal2"])


def _ckey_unit(n, nested):
    """g<A>() demanded on the host pass only (E1201 at its first demand), then
    n calls, then g<A>() again: the second creator sits past the old 12-bit
    ordinal (nested) or 16-bit statement field (top level) of the creation key
    (exs_walk.cuh creation-key widths)."""
    ind = "    " if nested else "  "
    lines = ["struct A { __host__ __device__ void call() {} };", "template< typename T >",
             "__host__ __device__ void g() { T{}.call(); }", "__host__ __device__ void h() {}",
             "__host__ __device__ void run() {"]
    if nested:
        lines.append("  if ( true ) {")
    lines += ["#ifndef __CUDA_ARCH__", ind + "g< A >();"] + [ind + "h();"] * n + [ind + "g< A >();", "#endif"]
    if nested:
        lines.append("  }")
    lines += ["}", "int main() { run(); }"]
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("shape", ["ordinal_4096", "statement_65536"])
def test_creation_key_fields_do_not_wrap(X, eng, shape):
    text = _ckey_unit(4095, True) if shape == "ordinal_4096" else _ckey_unit(65535, False)
    for m in ("sound", "proposal2"):
        a = eng.run_batch([(text, "u.mcu", X.CompileProfile(), X.Mode(m), X.TraitConfig())])[0]
        rows, _, _ = _oracle_rows(text, m)
        assert as_rows(a) == rows
        assert [r[0] for r in rows] == ["E1201"]


@pytest.mark.parametrize("flagged", [False, True], ids=["select_if", "select_flagged"])
def test_c5_stressors_vs_oracle(X, eng, eng_flag, flagged):
    eng = eng_flag if flagged else eng
    from paper_2309_03912_b200 import synth
    texts = [synth.gen_c5_file(500 + s, 12000, 0.5) for s in range(10)]
    _check_against_oracle(X, eng, texts, ["classic", "sound", "proposal2", "fidelity", "proposal1"] * 2)


@pytest.mark.parametrize("flagged", [False, True], ids=["select_if", "select_flagged"])
def test_c3_chain_vs_oracle(X, eng, eng_flag, flagged):
    eng = eng_flag if flagged else eng
    from paper_2309_03912_b200 import synth
    text = synth.gen_chain(24, 48)
    _check_against_oracle(X, eng, [text, text], ["classic", "sound"])


@pytest.mark.parametrize("flagged", [False, True], ids=["select_if", "select_flagged"])
def test_c4_callgraph_vs_oracle(X, eng, eng_flag, flagged):
    eng = eng_flag if flagged else eng
    from paper_2309_03912_b200 import synth
    text = synth.gen_callgraph(2000, 10, 7)
    _check_against_oracle(X, eng, [text], ["sound"])


@pytest.mark.parametrize("split", [False, True], ids=["items", "stmt_split"])
def test_batch_invariance_and_determinism(X, eng, eng_split, split):
    """A unit's result does not depend on its batch neighbours or on the run."""
    from paper_2309_03912_b200 import synth
    eng = eng_split if split else eng
    rng = random.Random(5)
    texts = [synth.gen_c5_file(rng.randrange(10**6), 4000, 0.3) for _ in range(12)]
    units = [(t, f"b{i}.cu", X.CompileProfile(), X.Mode.SOUND, X.TraitConfig()) for i, t in enumerate(texts)]
    together = eng.run_batch(units)
    again = eng.run_batch(units)
    alone = [eng.run_batch([u])[0] for u in units]
    for a, b, c in zip(together, again, alone):
        assert as_rows(a) == as_rows(b) == as_rows(c)


def test_public_api_check_unit(X):
    src = """struct D { __device__ void call() {} };
void a() { D{}.call(); }
void b() { D{}.call(); }
"""
    got = [(d.code, d.loc.line) for d in X.check_unit(src, "u.mcu")]
    assert got == [("E1001", 2), ("E1001", 3)]


def test_diagnostic_overflow_regrows_inside_the_walk(X, eng):
    """A unit whose walk emits more diagnostics than the buffer sized from its
    call sites holds (every call a stray: 120k E1002 against the 1-in-2
    estimate) is re-walked with a grown buffer, keeping the earlier stages'
    diagnostics -- same ordered set as the oracle."""
    lines = [f"void h{i}() {{}}" for i in range(10)]
    lines += [f"__device__ void f{i}() {{ " + " ".join(f"h{(i + k) % 10}();" for k in range(10)) + " }"
              for i in range(16000)]
    lines += ["int main() { return 0; }"]
    text = "\n".join(lines) + "\n"
    a = eng.run_batch([(text, "c4.cu", X.CompileProfile(), X.Mode.SOUND, X.TraitConfig())])[0]
    assert eng.last_stats["retries"] >= 1
    rows, _, _ = _oracle_rows(text, "sound")
    assert as_rows(a) == rows


@pytest.mark.parametrize("group", GOLDEN_GROUPS)
def test_walk_keys_match_the_reference(X, eng, group):
    """Analysis.walks[side].instances / .demands / .edges (spacecheck.py:239-346,585),
    rendered from the GPU arrays, equal the reference's keys (canonical text form,
    with demand display names and first-demand locations, edges in post-order)."""
    cases = [c for c in load_golden(group) if any("instances" in e for e in c["walks"].values())]
    res = eng.run_batch([unit_of(X, c) for c in cases], want_walks=True)
    bad = []
    for c, a in zip(cases, res):
        for side, ent in c["walks"].items():
            if "instances" not in ent:
                continue
            w = a.walks[X.ExecSpace(side)]
            if sorted(w.instances) != ent["instances"]:
                bad.append((c["name"], side, "instances"))
            if sorted([k, d, l[0], l[1]] for k, (d, l) in w.demands.items()) != ent["demands"]:
                bad.append((c["name"], side, "demands"))
            if sorted([k, v] for k, v in w.edges.items()) != ent["edges"]:
                bad.append((c["name"], side, "edges"))
    assert not bad, bad[:5]


def test_classification_exports_match_the_reference(X, eng):
    """propagate_spaces (spacecheck.py:770-782) over every walk, and
    struct_member_spaces (spacecheck.py:785-793) of each struct of the first
    pass's AST, equal the reference's on the golden units (classify.json.gz,
    made by tests/golden/make_classify.py)."""
    cases = load_golden("classify")
    res = eng.run_batch([unit_of(X, c) for c in cases], want_walks=True)
    bad, n_structs = [], 0
    for c, a in zip(cases, res):
        got = {k: sorted(s.value for s in v) for k, v in X.propagate_spaces(a).items()}
        if got != c["spaces"]:
            bad.append((c["name"], "spaces", got, c["spaces"]))
        first = a.profile.pass_kinds()[0]
        if c["structs"] is None or a.passes[first]["parse_failed"]:
            continue
        mine = [[s.name, {m: sorted(x.value for x in v) for m, v in X.struct_member_spaces(s).items()}]
                for s in a.structs(0)]
        n_structs += len(mine)
        if mine != c["structs"]:
            bad.append((c["name"], "structs", mine, c["structs"]))
    assert not bad, bad[:3]
    assert len(cases) > 800 and n_structs > 1000


def test_select_paths_agree_at_scale(X, eng):
    """At ~24 MB (about 6M view tokens) the default engine's parser selections
    take the flag pass; an engine that never takes it must report the same
    diagnostics for every unit, in the same order."""
    from paper_2309_03912_b200 import synth
    texts = [synth.gen_c2_file(7000 + s, 100_000) for s in range(240)]
    units = [(t, f"s{i}.cu", X.CompileProfile(), X.Mode.CLASSIC, X.TraitConfig()) for i, t in enumerate(texts)]
    flagged = eng.run_batch(units)
    assert eng.last_stats["view_tokens"] >= 1 << 22
    e_if = X.Engine(0)
    e_if.handle.set_option(4, 2**31 - 1)
    plain = e_if.run_batch(units)
    assert sum(len(a.all_diagnostics) for a in flagged) > 0
    for a, b in zip(flagged, plain):
        assert as_rows(a) == as_rows(b)


def test_diag_sort_paths_agree(X, eng):
    """Diagnostic order (reference: sorted by file, line, column, code) from the
    single packed-key radix sort must equal the two-sort fallback used when the
    fields exceed 64 bits, over a batch with thousands of diagnostics."""
    from paper_2309_03912_b200 import synth
    texts = [synth.gen_c2_file(9100 + s, 60_000) for s in range(64)]
    units = [(t, f"d{i}.cu", X.CompileProfile(), X.Mode.CLASSIC, X.TraitConfig()) for i, t in enumerate(texts)]
    packed = eng.run_batch(units)
    e2 = X.Engine(0)
    e2.handle.set_option(5, 1)
    two = e2.run_batch(units)
    assert sum(len(a.all_diagnostics) for a in packed) > 1000
    for a, b in zip(packed, two):
        assert as_rows(a) == as_rows(b)


def test_streamed_batches_equal_one_batch(X):
    """exs_run_units cut into 1 MiB batches (copies of batch k+1 overlapping the
    analysis of batch k) reports exactly what one batch reports, and both
    equal the oracle on a sample."""
    from paper_2309_03912_b200 import synth
    texts = ([synth.gen_c2_file(300 + s, 60_000) for s in range(40)] +
             [synth.gen_c5_file(700 + s, 30_000, 0.5) for s in range(16)])
    modes = ["classic", "sound", "proposal2", "fidelity", "proposal1"]
    units = [(t, f"s{i:03d}.cu", X.CompileProfile(), X.Mode(modes[i % 5]), X.TraitConfig())
             for i, t in enumerate(texts)]
    one = X.Engine(0).run_batch(units)
    e = X.Engine(0, batch_mib=1)
    many = e.run_batch(units)
    assert e.last_stats["batches"] >= 3
    for a, b in zip(one, many):
        assert as_rows(a) == as_rows(b)
    for i in range(0, len(texts), 7):
        want = O.check(texts[i], modes[i % 5])
        assert [(d.code, d.loc.line, d.loc.col, d.message) for d in many[i].diagnostics] == want


def test_results_view_is_ordered_and_complete(X, eng):
    """exs_results_view: per-unit ranges cover every record once, records are
    in (unit, line, col, code string, message) order -- Diagnostic.sort_key,
    diagnostics.py:73-74 -- and messages decode as UTF-8."""
    from paper_2309_03912_b200.messages import CODES
    from paper_2309_03912_b200 import synth
    texts = [synth.gen_c5_file(900 + s, 20_000, 0.5) for s in range(20)]
    units = [(t, f"v{i}.cu", X.CompileProfile(), X.Mode.SOUND, X.TraitConfig()) for i, t in enumerate(texts)]
    eng.run_batch(units)
    recs, text, first = eng.handle.results(copy=False)
    assert int(first[0]) == 0 and int(first[-1]) == len(recs) and len(first) == len(units) + 1
    keys = []
    for u in range(len(units)):
        r = recs[int(first[u]):int(first[u + 1])]
        assert (r["unit"] == u).all()
        for x in r:
            msg = text[int(x["msg_off"]):int(x["msg_off"]) + int(x["msg_len"])].tobytes().decode()
            keys.append((u, int(x["line"]), int(x["col"]), CODES[int(x["code"])], msg))
    assert keys == sorted(keys) and len(set(keys)) == len(keys)


@pytest.mark.parametrize("n_shards", [2, 3])
def test_logical_shards_merge_to_the_one_shard_run(X, n_shards):
    """The corpus cut into byte-balanced shards (shard.shard_ranges, the
    multi-GPU partition), each analysed alone on this device and merged in
    rank order (shard.merge_results, what gather_results does on rank 0),
    equals the one-shard run record for record."""
    from paper_2309_03912_b200 import synth
    from paper_2309_03912_b200.shard import merge_results, shard_ranges
    texts = [synth.gen_c5_file(1200 + s, 8_000 + 3_000 * (s % 4), 0.4) for s in range(23)]
    units = [(f"m{i:03d}.cu", t) for i, t in enumerate(texts)]
    e = X.Engine(0)
    X.analyze_corpus(units, mode=X.Mode.SOUND, engine=e)
    whole = e.handle.results(copy=True)
    parts = []
    for lo, hi in shard_ranges([len(t) for t in texts], n_shards):
        X.analyze_corpus(units[lo:hi], mode=X.Mode.SOUND, engine=e)
        parts.append(e.handle.results(copy=True))
    merged = merge_results(parts)
    res_w = X.CorpusResults(*whole, [u[0] for u in units])
    res_m = X.CorpusResults(*merged, [u[0] for u in units])
    assert list(merged[2]) == list(whole[2])
    for u in range(len(units)):
        rows = lambda r: [(d.code, d.loc.line, d.loc.col, d.message, d.suppressed) for d in r.diagnostics(u)]  # noqa
        assert rows(res_m) == rows(res_w)



def test_leased_results_survive_later_runs(X):
    """analyze_corpus hands out zero-copy views of the library's result buffers
    (exs_results_lease): a run's diagnostics read after two later runs on the
    same engine equal a fresh run's."""
    from paper_2309_03912_b200 import synth
    eng = X.Engine(0)
    t1 = [synth.gen_c2_file(s, 5000) for s in range(6)]
    t2 = [synth.gen_c5_file(s, 5000, 0.5) for s in range(6)]
    mk = lambda ts, m: [(t, "a.cu", X.CompileProfile(), m, X.TraitConfig()) for t in ts]  # noqa: E731
    first = eng.run_batch(mk(t1, X.Mode.SOUND))
    eng.run_batch(mk(t2, X.Mode.SOUND))
    eng.run_batch(mk(t2, X.Mode.CLASSIC))
    again = eng.run_batch(mk(t1, X.Mode.SOUND))
    assert [as_rows(a) for a in first] == [as_rows(a) for a in again]
    assert sum(len(a.all_diagnostics) for a in first) > 0


EDGE_UNITS = [
    "",                                   # empty file
    "\n\n\n",                             # only newlines
    "   \t  ",                            # whitespace, no newline at the end
    "// only a comment",
    "/* unterminated block comment\nint main() { return 0; }\n",
    "int main() { return 0; }\\",         # a backslash at the very end
    "int main() { return 0; }\\\n",       # a splice at the end of the file
    'void f() { printf("unterminated); }\n',
    "int main() { return 0; }" * 2000,    # one 48 KB line
    "\n".join("void f%d() {}" % i for i in range(3000)) + "\nint main() { f1(); return 0; }\n",
    "#pragma hd_warning_disable\n",       # a directive as the last line, no unit body
    "struct A { __device__ void call() {} };\nint main() { A{}.call(); return 0; }",  # no final newline
    "int m\\\nain() { return 0; }\n",     # an identifier spliced across lines
    "__device__ void d() {}\nvoid h() { d(); }\n" * 300,
]


def test_edge_units_vs_oracle(X, eng):
    """Inputs at the edges of the lexer and the streaming driver: empty and
    whitespace-only units, a comment or an unterminated comment/string at EOF, a
    trailing backslash or splice, one very long line, a spliced identifier, a
    directive as the last line, no final newline -- each against the oracle, in
    one batch and one unit at a time."""
    modes = ["classic", "sound", "fidelity", "proposal1", "proposal2"]
    units = [(t, f"e{i}.cu", X.CompileProfile(), X.Mode(modes[i % 5]), X.TraitConfig()) for i, t in enumerate(EDGE_UNITS)]
    together = eng.run_batch(units)
    for i, (t, a) in enumerate(zip(EDGE_UNITS, together)):
        rows, _, _ = _oracle_rows(t, modes[i % 5])
        assert as_rows(a) == rows, i
        alone = eng.run_batch([units[i]])[0]
        assert as_rows(alone) == rows, i


def test_empty_corpus_and_tiny_units(X):
    assert len(X.analyze_corpus([])) == 0
    many = [(f"t{i}.cu", "int main() { return 0; }\n" if i % 2 else "") for i in range(20000)]
    res = X.analyze_corpus(many)
    assert len(res) == 20000 and all(len(a.diagnostics) == 0 for a in res)
