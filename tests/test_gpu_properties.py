"""Property tests of the reference (pkg/tests/test_properties.py:20-129) on the
GPU path, over seeded generated units, plus a differential check of many
seeded units against the oracle.

The reference's generator (pkg/tests/genprog.py) is not available on the GPU
box; `synth.gen_c2_file` builds the same module shape (structs with optional
hdc tags, host-device templates calling T{}.call(), optional kernels, pragma
slots with p = 0.7, one main), and the "without pragmas" spelling blanks the
pragma lines as genprog does (same line numbers).
"""
import random

import pytest

from oracle import exs_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def X():
    from paper_2309_03912_b200 import exspace
    return exspace


@pytest.fixture(scope="module")
def units():
    from paper_2309_03912_b200 import synth
    out = []
    for seed in range(100):
        text = synth.gen_c2_file(20_000 + seed, 1_500 + 40 * seed)
        bare = "\n".join("" if ln.startswith("#pragma") else ln for ln in text.split("\n"))
        out.append((text, bare))
    return out


def _keys(diags):
    return {(d.loc.line, d.loc.col, d.code, d.message) for d in diags}


def _run(X, texts, profile=None, mode=None, want_walks=False):
    p = profile or X.CompileProfile()
    m = mode or X.Mode.CLASSIC
    return X.get_engine(0).run_batch([(t, "g.mcu", p, m, X.TraitConfig()) for t in texts], want_walks=want_walks)


def test_pragma_suppression_is_monotone_over_100_units(X, units):
    """test_properties.py:20-28: pragmas only ever drop warnings."""
    with_p = _run(X, [u[0] for u in units])
    without_p = _run(X, [u[1] for u in units])
    for seed, (a, b) in enumerate(zip(with_p, without_p)):
        ka, kb = _keys(a.diagnostics), _keys(b.diagnostics)
        assert ka <= kb, seed
        assert all(code.startswith("W") for _, _, code, _ in kb - ka), seed


def test_relaxed_constexpr_is_monotone_over_100_units(X, units):
    """test_properties.py:31-36: relaxed constexpr only ever drops diagnostics."""
    strict = _run(X, [u[1] for u in units], X.CompileProfile())
    relaxed = _run(X, [u[1] for u in units], X.CompileProfile(relaxed_constexpr=True))
    for seed, (a, b) in enumerate(zip(strict, relaxed)):
        assert _keys(b.diagnostics) <= _keys(a.diagnostics), seed


def test_check_is_deterministic_byte_for_byte(X, units):
    """test_properties.py:39-47."""
    for mode in (X.Mode.CLASSIC, X.Mode.SOUND, X.Mode.FIDELITY):
        a = _run(X, [u[0] for u in units[:20]], mode=mode)
        b = _run(X, [u[0] for u in units[:20]], mode=mode)
        for x, y in zip(a, b):
            assert [X.format_diagnostic(d) for d in x.diagnostics] == [X.format_diagnostic(d) for d in y.diagnostics]


def test_instantiation_sets_agree_without_directives(X, units):
    """test_properties.py:120-129: with no #ifdef, both passes demand the same
    instantiations."""
    for mode in (X.Mode.CLASSIC, X.Mode.SOUND):
        res = _run(X, [u[1] for u in units[:30]], mode=mode, want_walks=True)
        for seed, a in enumerate(res):
            assert set(a.walks[X.ExecSpace.Host].demands) == set(a.walks[X.ExecSpace.Device].demands), seed


def test_many_seeded_units_equal_the_oracle(X):
    """Differential check: 600 seeded units (module shapes, lexer stressors,
    template chains, call graphs; every mode, both profiles) in one batch,
    each equal to the oracle's ordered diagnostics."""
    from paper_2309_03912_b200 import synth
    rng = random.Random(2309_03912)
    modes = [m.value for m in X.Mode]
    cases = []
    for k in range(600):
        kind = k % 4
        if kind == 0:
            t = synth.gen_c2_file(rng.randrange(10**6), rng.randrange(800, 6000))
        elif kind == 1:
            t = synth.gen_c5_file(rng.randrange(10**6), rng.randrange(800, 6000), 0.5)
        elif kind == 2:
            t = synth.gen_chain(rng.randrange(2, 12), rng.randrange(2, 20))
        else:
            t = synth.gen_callgraph(rng.randrange(5, 80), rng.randrange(1, 6), rng.randrange(10**6))
        plain = k % 9 == 0
        cases.append((t, modes[k % 5], plain))
    res = X.get_engine(0).run_batch([(t, f"u{i}.cu", X.CompileProfile("plain") if p else X.CompileProfile(),
                                      X.Mode(m), X.TraitConfig()) for i, (t, m, p) in enumerate(cases)])
    bad = []
    for i, ((t, m, p), a) in enumerate(zip(cases, res)):
        r = O.analyze_unit(t, m, "plain" if p else "nvcc")
        want = [(d[0], d[1], d[2], d[3], d[4]) for d in r.all_diagnostics]
        got = [(d.code, d.loc.line, d.loc.col, d.message, d.suppressed) for d in a.all_diagnostics]
        if got != want:
            bad.append(i)
    assert not bad, bad[:10]
