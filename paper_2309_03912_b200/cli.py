"""Command-line driver mirroring the reference's ``exspace`` CLI (cli.py:18-142)
on the GPU batch API: every unit of one invocation goes to the GPU as one batch.

  python -m paper_2309_03912_b200 check [flags] PATH...   (cli.py:82-91)
  python -m paper_2309_03912_b200 corpus [flags] DIR      (cli.py:114-132, corpus.py:18-175)

Flags, output lines, and exit codes (0 ok / 1 diagnostics or failures / 2 usage
or I/O) follow the reference.  ``run`` executes a unit with the reference's
interpreter, which is not on the analysis path: it exits 2
with a message.  In ``corpus``, files whose ``//!`` header expects a run outcome
have their diagnostics checked as usual.  The run expectation itself is reported
as not checked and does not count as a failure.
"""
from __future__ import annotations

import argparse
import os
import re
import sys
from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional

from . import exspace as X

_MODES = [m.value for m in X.Mode]

# corpus.py:18-22
_EXPECT_RE = re.compile(
    r"//~(?:@(?P<line>\d+))?\s+(?P<sev>error|warning|note)\s+"
    r"(?P<code>[EWN]\d{4})(?:\s+\"(?P<substr>[^\"]*)\")?"
)
_HEADER_RE = re.compile(r"^\s*//!\s*(?P<key>[a-z-]+)(?:\s*:\s*(?P<value>.*?))?\s*$")


def _add_common_flags(p: argparse.ArgumentParser):
    p.add_argument("--mode", choices=_MODES, default="classic")
    p.add_argument("--profile", choices=["nvcc", "plain"], default="nvcc")
    p.add_argument("--cuda-version", type=int, choices=[9, 10, 11, 12], default=12)
    p.add_argument("--relaxed-constexpr", action="store_true")
    p.add_argument("--erase-specifiers", action="store_true")
    p.add_argument("--emit", choices=["human", "machine"], default="machine")


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="exspace", description="Static checker for MiniCU execution spaces (B200 batch engine).")
    sub = parser.add_subparsers(dest="command", required=True)
    p_check = sub.add_parser("check", help="diagnose one or more units")
    _add_common_flags(p_check)
    p_check.add_argument("paths", nargs="+")
    p_run = sub.add_parser("run", help="check, then execute a unit (not on the analysis path)")
    _add_common_flags(p_run)
    p_run.add_argument("--force", action="store_true")
    p_run.add_argument("path")
    p_corpus = sub.add_parser("corpus", help="run an expected-diagnostics corpus")
    _add_common_flags(p_corpus)
    p_corpus.add_argument("dir")
    return parser


def _profile_from(args, parser) -> X.CompileProfile:
    try:
        return X.CompileProfile(args.profile, args.cuda_version, args.relaxed_constexpr,
                                args.erase_specifiers)
    except ValueError as e:
        parser.error(str(e))  # exits 2


def _read(path: str) -> str:
    try:
        return Path(path).read_text(encoding="utf-8")
    except OSError as e:
        print(f"exspace: cannot read {path}: {e.strerror}", file=sys.stderr)
        raise SystemExit(2)


def _print_diags(diags, style, source):
    color = os.environ.get("EXSPACE_COLOR", "0") == "1"
    for d in diags:
        line = X.format_diagnostic(d, style, source if style == "human" else None, color)
        if line is not None:
            print(line)


def cmd_check(args, parser) -> int:
    profile = _profile_from(args, parser)
    mode = X.Mode(args.mode)
    texts = [_read(p) for p in args.paths]
    analyses = X.analyze_corpus(list(zip(args.paths, texts)), profile, mode)
    any_error = False
    for text, a in zip(texts, analyses):
        _print_diags(a.diagnostics, args.emit, text)
        any_error = any_error or a.has_errors
    return 1 if any_error else 0


# ---------------------------------------------------------------- corpus

@dataclass
class Expectation:
    line: int
    severity: str
    code: str
    substring: Optional[str]

    def describe(self) -> str:
        extra = f' "{self.substring}"' if self.substring else ""
        return f"line {self.line}: {self.severity}[{self.code}]{extra}"

    def matches(self, d) -> bool:
        return (d.loc.line == self.line and d.code == self.code and d.severity.value == self.severity
                and (self.substring is None or self.substring in d.message))


@dataclass
class CorpusResult:
    file: str
    matched: int = 0
    unmatched_expectations: list = field(default_factory=list)
    unexpected_diagnostics: list = field(default_factory=list)
    run_check: Optional[str] = None
    run_unchecked: bool = False

    @property
    def passed(self) -> bool:
        return not self.unmatched_expectations and not self.unexpected_diagnostics and self.run_check is None


def parse_expectations(text: str) -> list:
    """corpus.py:76-84"""
    out = []
    for lineno, line in enumerate(text.split("\n"), start=1):
        for m in _EXPECT_RE.finditer(line):
            target = int(m.group("line")) if m.group("line") else lineno
            out.append(Expectation(target, m.group("sev"), m.group("code"), m.group("substr")))
    return out


def parse_header(text: str, mode: X.Mode, profile: X.CompileProfile):
    """corpus.py:87-120: (mode, profile, wants_run)."""
    compiler, version = profile.compiler, profile.cuda_version
    relaxed, erase = profile.relaxed_constexpr, profile.erase_specifiers
    wants_run = False
    for line in text.split("\n"):
        m = _HEADER_RE.match(line)
        if not m:
            continue
        key, value = m.group("key"), m.group("value")
        if key == "mode":
            mode = X.Mode(value)
        elif key == "profile":
            compiler = value
        elif key == "cuda-version":
            version = int(value)
        elif key == "relaxed-constexpr":
            relaxed = True
        elif key == "erase-specifiers":
            erase = True
        elif key in ("expect-exit", "expect-stdout"):
            wants_run = True
        elif key != "force":
            raise ValueError(f"unknown corpus directive //! {key}")
    return mode, X.CompileProfile(compiler, version, relaxed, erase), wants_run


def run_corpus(directory: Path, mode: X.Mode, profile: X.CompileProfile):
    """corpus.py:123-175, all files in one GPU batch."""
    files = sorted(Path(directory).glob("*.mcu"))
    if not files:
        raise FileNotFoundError(f"no .mcu files under {directory}")
    texts = [f.read_text(encoding="utf-8") for f in files]
    heads = [parse_header(t, mode, profile) for t in texts]
    units = [(str(f), t, h[1], h[0], X.TraitConfig()) for f, t, h in zip(files, texts, heads)]
    analyses = X.analyze_corpus(units)
    results = []
    for f, t, h, a in zip(files, texts, heads, analyses):
        r = CorpusResult(str(f))
        unclaimed = list(a.diagnostics)
        for exp in parse_expectations(t):
            hit = next((d for d in unclaimed if exp.matches(d)), None)
            if hit is None:
                r.unmatched_expectations.append(exp.describe())
            else:
                unclaimed.remove(hit)
                r.matched += 1
        r.unexpected_diagnostics = [f"{d.loc.line}:{d.loc.col}: {d.severity.value}[{d.code}]: {d.message}"
                                    for d in unclaimed]
        r.run_unchecked = h[2]
        results.append(r)
    failed = sum(1 for r in results if not r.passed)
    return results, f"passed {len(results) - failed} / failed {failed}"


def cmd_corpus(args, parser) -> int:
    profile = _profile_from(args, parser)
    try:
        results, summary = run_corpus(Path(args.dir), X.Mode(args.mode), profile)
    except FileNotFoundError as e:
        print(f"exspace: {e}", file=sys.stderr)
        return 2
    for r in results:
        print(f"{'ok' if r.passed else 'FAIL':4} {r.file} ({r.matched} expectation(s) matched)")
        for miss in r.unmatched_expectations:
            print(f"     missing: {miss}")
        for extra in r.unexpected_diagnostics:
            print(f"     unexpected: {extra}")
        if r.run_unchecked:
            print("     run: not checked (the interpreter is not on the analysis path)")
    print(summary)
    return 0 if summary.endswith("failed 0") else 1


def main(argv=None) -> int:
    parser = build_parser()
    args = parser.parse_args(argv)
    if args.command == "check":
        return cmd_check(args, parser)
    if args.command == "run":
        print("exspace: 'run' executes the unit with the reference interpreter, which is not part "
              "of this engine (analysis path only); use 'check'", file=sys.stderr)
        return 2
    return cmd_corpus(args, parser)


if __name__ == "__main__":
    sys.exit(main())
