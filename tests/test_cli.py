"""The CLI mirror (paper_2309_03912_b200/cli.py) of the reference's exspace CLI.

CPU: argument handling, ``//!`` headers and ``//~`` expectations (corpus.py:18-120)
on the shipped corpus texts held in the golden fixture.  GPU: ``corpus`` over those
32 files passes every diagnostic expectation (the reference prints
"passed 32 / failed 0", cli.py:114-132), and ``check`` prints the golden
diagnostics in the reference's machine format.
"""
import pytest

from exs_testlib import load_golden


def _corpus_files():
    """(file name, text) of the 32 shipped corpus files (their header configs)."""
    out = {}
    for c in load_golden("corpus"):
        name = c["name"].split("/", 1)[1]
        if "@" not in name:
            out[name] = c
    return out


def test_corpus_headers_and_expectations_parse():
    from paper_2309_03912_b200 import cli, exspace as X
    files = _corpus_files()
    assert len(files) == 32
    n_exp = n_run = 0
    for name, c in files.items():
        mode, prof, wants_run = cli.parse_header(c["text"], X.Mode.CLASSIC, X.CompileProfile())
        assert mode.value == c["mode"] and prof.compiler == c["compiler"]
        assert prof.relaxed_constexpr == c["relaxed"] and prof.erase_specifiers == c["erase"]
        n_exp += len(cli.parse_expectations(c["text"]))
        n_run += wants_run
    assert n_exp == 16 and n_run == 8  # corpus.py counts on the shipped files


def test_run_and_usage_exit_codes(capsys):
    from paper_2309_03912_b200 import cli
    assert cli.main(["run", "x.mcu"]) == 2
    with pytest.raises(SystemExit) as e:
        cli.main(["check", "--profile", "plain", "--relaxed-constexpr", "x.mcu"])
    assert e.value.code == 2  # invalid profile -> parser.error (cli.py:55-63)


@pytest.mark.gpu
def test_corpus_command_passes_the_shipped_corpus(tmp_path, capsys):
    from paper_2309_03912_b200 import cli
    for name, c in _corpus_files().items():
        (tmp_path / name).write_text(c["text"], encoding="utf-8")
    rc = cli.main(["corpus", str(tmp_path)])
    out = capsys.readouterr().out
    assert "passed 32 / failed 0" in out and rc == 0, out[-2000:]


@pytest.mark.gpu
def test_check_command_prints_the_golden_diagnostics(tmp_path, capsys):
    from paper_2309_03912_b200 import cli
    files = _corpus_files()
    names = sorted(n for n, c in files.items() if c["mode"] == "classic" and c["compiler"] == "nvcc"
                   and not c["relaxed"] and not c["erase"])[:6]
    paths = []
    want = []
    for n in names:
        p = tmp_path / n
        p.write_text(files[n]["text"], encoding="utf-8")
        paths.append(str(p))
        want += [f"{p}:{ln}:{col}: {sev}[{code}]: {msg}"
                 for code, sev, ln, col, msg, sup in files[n]["diags"] if not sup]
    rc = cli.main(["check", *paths])
    got = capsys.readouterr().out.splitlines()
    assert got == want
    assert rc == (1 if any(w.split(": ")[1].startswith("error") for w in want) else 0)
