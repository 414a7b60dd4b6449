"""Drop-in mirror of the reference ``exspace`` analysis API, GPU-backed.

Same names, argument meaning, result schema and ordering as
``exspace.spacecheck.analyze``/``check_unit`` (spacecheck.py:687-750) and the
types they return (diagnostics.py:8-121, preprocess.py:31-78, sema.py:12-62).
Every unit is analysed by the sm_100a pipeline behind the C ABI
(include/exspace_b200.h); the host only packs inputs and renders messages.
``analyze_corpus`` is the batch entry point (many units per GPU launch).
"""
from __future__ import annotations

import threading
from dataclasses import dataclass, field
from enum import Enum
from collections.abc import Sequence
from typing import Iterable, Optional

import numpy as np

from . import _native
from .walks import GLOBAL, BatchWalks, StructInfo
from .messages import CODES, Renderer, stray_text  # noqa: F401  (stray_text re-exported)


# ---------------------------------------------------------------------------
# result schema (diagnostics.py)

class Severity(Enum):
    ERROR = "error"
    WARNING = "warning"
    NOTE = "note"


CODE_REGISTRY: dict = {
    "E0001": (Severity.ERROR, "parse error"),
    "E0002": (Severity.ERROR, "preprocessor error"),
    "E0101": (Severity.ERROR, "undefined name"),
    "E0102": (Severity.ERROR, "duplicate definition"),
    "E0103": (Severity.ERROR, "hdc member is not an HDC constant"),
    "E0104": (Severity.ERROR, "static assertion failed"),
    "E1001": (Severity.ERROR, "host code calls a device function"),
    "E1002": (Severity.ERROR, "device code calls a host function"),
    "E1003": (Severity.ERROR, "kernel launch from device code"),
    "E1004": (Severity.ERROR, "misused __global__ function"),
    "W1101": (Severity.WARNING, "host device function calls a host-only function"),
    "W1102": (Severity.WARNING, "host device function calls a device-only function"),
    "E1101": (Severity.ERROR, "reachable stray call to a host-only function"),
    "E1102": (Severity.ERROR, "reachable stray call to a device-only function"),
    "E1201": (Severity.ERROR, "instantiation depends on the compile pass"),
    "E1301": (Severity.ERROR, "no viable overload candidate"),
    "E1302": (Severity.ERROR, "ambiguous call"),
    "E1401": (Severity.ERROR, "empty execution-space set"),
    "E1501": (Severity.ERROR, "stray call"),
    "W1502": (Severity.WARNING, "host device function calls a one-sided function"),
    "N0001": (Severity.NOTE, "kernel launch skipped after device error"),
    # the analyser's own marker for inputs beyond its recursion/nesting bounds,
    # where the reference raises RecursionError
    "X9999": (Severity.ERROR, "input outside the analyser contract"),
}

STRAY_CODES = frozenset({"E1001", "E1002", "W1101", "W1102", "E1101", "E1102", "E1501", "W1502"})


@dataclass(frozen=True, order=True)
class SrcLoc:
    file: str
    line: int
    col: int

    def __post_init__(self):
        if self.line < 1 or self.col < 1:
            raise ValueError(f"source positions are 1-based: {self.line}:{self.col}")

    def __str__(self):
        return f"{self.file}:{self.line}:{self.col}"


@dataclass
class Diagnostic:
    code: str
    severity: Severity
    loc: SrcLoc
    message: str
    suppressed: bool = field(default=False)

    @classmethod
    def make(cls, code: str, loc: SrcLoc, message: str) -> "Diagnostic":
        return cls(code, CODE_REGISTRY[code][0], loc, message)

    @property
    def is_error(self) -> bool:
        return self.severity is Severity.ERROR

    def sort_key(self):
        return (self.loc.file, self.loc.line, self.loc.col, self.code, self.message)

    def dedup_key(self):
        return (self.loc, self.code, self.message)


_COLORS = {Severity.ERROR: "\x1b[31;1m", Severity.WARNING: "\x1b[35;1m", Severity.NOTE: "\x1b[36m"}


def format_diagnostic(d: Diagnostic, style: str = "machine", source: Optional[str] = None,
                      color: bool = False) -> Optional[str]:
    """diagnostics.py:88-113."""
    if d.suppressed:
        return None
    word = d.severity.value
    if color:
        word = f"{_COLORS[d.severity]}{word}\x1b[0m"
    line = f"{d.loc.file}:{d.loc.line}:{d.loc.col}: {word}[{d.code}]: {d.message}"
    if style == "machine" or source is None:
        return line
    lines = source.splitlines()
    if 1 <= d.loc.line <= len(lines):
        return f"{line}\n{lines[d.loc.line - 1]}\n{' ' * (d.loc.col - 1)}^"
    return line


def finish_diagnostics(diags: list) -> list:
    """diagnostics.py:116-121."""
    seen = {}
    for d in diags:
        seen.setdefault(d.dedup_key(), d)
    return sorted(seen.values(), key=Diagnostic.sort_key)


# ---------------------------------------------------------------------------
# configuration (preprocess.py:46-78, spacecheck.py:53-58, sema.py:54-62)

@dataclass(frozen=True)
class CompileProfile:
    compiler: str = "nvcc"
    cuda_version: int = 12
    relaxed_constexpr: bool = False
    erase_specifiers: bool = False

    def __post_init__(self):
        if self.compiler not in ("nvcc", "plain"):
            raise ValueError(f"unknown compiler {self.compiler!r}")
        if self.cuda_version not in (9, 10, 11, 12):
            raise ValueError(f"unsupported cuda version {self.cuda_version}")
        if self.relaxed_constexpr and self.compiler != "nvcc":
            raise ValueError("relaxed constexpr is an nvcc-only flag")
        if self.erase_specifiers and self.compiler != "plain":
            raise ValueError("specifier erasure applies to the plain profile only")

    def pass_kinds(self) -> list:
        return ["host"] if self.compiler == "plain" else ["host", "device"]

    def trap_error_code(self) -> int:
        return 4 if self.cuda_version == 9 else 207


class Mode(Enum):
    CLASSIC = "classic"
    FIDELITY = "fidelity"
    SOUND = "sound"
    PROPOSAL1 = "proposal1"
    PROPOSAL2 = "proposal2"


_MODE_ID = {Mode.CLASSIC: 0, Mode.FIDELITY: 1, Mode.SOUND: 2, Mode.PROPOSAL1: 3, Mode.PROPOSAL2: 4}


@dataclass(frozen=True)
class TraitConfig:
    fundamentals_hstdev: bool = False


class ExecSpace(Enum):
    Host = "host"
    Device = "device"
    Global = "global"
    HostDevice = "host device"


HOST, DEVICE = ExecSpace.Host, ExecSpace.Device


def cfg_byte(profile: CompileProfile, mode: Mode, cfg: TraitConfig) -> int:
    b = _MODE_ID[mode]
    if profile.compiler == "plain":
        b |= 8
    if profile.relaxed_constexpr:
        b |= 16
    if profile.erase_specifiers:
        b |= 32
    if cfg.fundamentals_hstdev:
        b |= 64
    return b


# ---------------------------------------------------------------------------
# legality matrix (host-side mirror of spacecheck.py:86-132; the GPU kernels
# carry the same table in exs_walk.cuh:verdict)

@dataclass(frozen=True)
class Verdict:
    kind: str
    code: Optional[str] = None

    @property
    def ok(self) -> bool:
        return self.kind == "ok"


def legality(caller_side, callee_space, kind: str = "direct", *, caller_from_hd: bool = False,
             relaxed_constexpr: bool = False, callee_is_constexpr: bool = False,
             mode: Mode = Mode.CLASSIC, mismatched_side_reachable: bool = True) -> Verdict:
    if caller_side not in (HOST, DEVICE):
        raise ValueError("the caller side must be host or device")
    if kind == "launch":
        if caller_side is DEVICE:
            return Verdict("error", "E1003")
        return Verdict("ok") if callee_space is ExecSpace.Global else Verdict("error", "E1004")
    if callee_space is ExecSpace.Global:
        return Verdict("error", "E1004")
    if relaxed_constexpr and callee_is_constexpr:
        return Verdict("ok")
    if callee_space is ExecSpace.HostDevice or callee_space is caller_side:
        return Verdict("ok")
    host_only = callee_space is HOST
    if not caller_from_hd:
        if mode is Mode.PROPOSAL2:
            return Verdict("error", "E1501")
        return Verdict("error", "E1001" if caller_side is HOST else "E1002")
    if mode is Mode.FIDELITY and not host_only:
        return Verdict("ok")
    if mode is Mode.SOUND and mismatched_side_reachable:
        return Verdict("error", "E1101" if host_only else "E1102")
    if mode is Mode.PROPOSAL2:
        return Verdict("error", "E1501") if mismatched_side_reachable else Verdict("warn", "W1502")
    return Verdict("warn", "W1101" if host_only else "W1102")


# ---------------------------------------------------------------------------
# results

@dataclass
class WalkSummary:
    """One walk of an analysis (spacecheck.py _Walk): counts, and -- rendered from
    the GPU arrays on first access -- the instance, demand and edge maps keyed by
    the reference's keys in canonical text form (walks.py)."""
    native: ExecSpace
    n_instances: int
    n_edges: int
    n_demands: int
    _batch: object = field(default=None, repr=False, compare=False)
    _where: tuple = field(default=(0, 0), repr=False, compare=False)
    _maps: Optional[tuple] = field(default=None, repr=False, compare=False)

    def _get(self, i: int):
        if self._maps is None:
            if self._batch is None:
                raise RuntimeError("walk keys need an analysis run with want_walks=True")
            self._maps = self._batch.walk(*self._where)
        return self._maps[i]

    @property
    def instances(self) -> dict:
        """{instance key: walks.InstanceInfo} in creation (FIFO) order."""
        return self._get(0)

    @property
    def demands(self) -> dict:
        """{demand key: (display name, (line, col) of the first demand)}."""
        return self._get(1)

    @property
    def edges(self) -> dict:
        """{caller instance key: [callee instance keys in post-order]} (legal edges)."""
        return self._get(2)


class CorpusResults:
    """Columnar results of one run: the finished diagnostic records of every
    unit (include/exspace_b200.h exs_result, rendered and ordered natively)
    and their message bytes.  Diagnostic objects are built per unit on first
    access (a corpus of 1 GB has ~4M diagnostics)."""

    def __init__(self, recs: np.ndarray, text: np.ndarray, unit_first: np.ndarray, paths: list, lease=None):
        self.recs = recs
        self.text = text
        self.unit_first = unit_first
        self.paths = paths
        self._lease = lease  # zero-copy views of the library's buffers stay valid while this lives

    def n_diagnostics(self, unit: int) -> int:
        return int(self.unit_first[unit + 1] - self.unit_first[unit])

    def diagnostics(self, unit: int) -> list:
        lo, hi = int(self.unit_first[unit]), int(self.unit_first[unit + 1])
        if lo == hi:
            return []
        r = self.recs[lo:hi]
        path = self.paths[unit]
        tx = self.text
        out = []
        for line, col, code, sup, off, ln in zip(r["line"].tolist(), r["col"].tolist(), r["code"].tolist(),
                                                 r["suppressed"].tolist(), r["msg_off"].tolist(),
                                                 r["msg_len"].tolist()):
            c = CODES[code]
            d = Diagnostic(c, CODE_REGISTRY[c][0], SrcLoc(path, line, col),
                           tx[off:off + ln].tobytes().decode("utf-8", "surrogateescape"))
            if sup:
                d.suppressed = True
            out.append(d)
        return out

    def codes(self, unit: int) -> list:
        """The codes of a unit's unsuppressed diagnostics, without building objects."""
        r = self.recs[int(self.unit_first[unit]):int(self.unit_first[unit + 1])]
        return [CODES[c] for c, s in zip(r["code"].tolist(), r["suppressed"].tolist()) if not s]


class Analysis:
    """Result of analysing one unit (spacecheck.py:669-681 Analysis).

    ``diagnostics`` (ordered, unsuppressed) and ``all_diagnostics`` (with the
    suppressed ones) are built from the run's columnar results on first access."""

    __slots__ = ("path", "profile", "mode", "walks", "passes", "_results", "_unit", "_batch", "_all")

    def __init__(self, path: str, profile: CompileProfile, mode: Mode, results: CorpusResults = None,
                 unit: int = 0, batch=None, diagnostics: list = None):
        self.path = path
        self.profile = profile
        self.mode = mode
        self.walks = {}
        self.passes = {}  # pass kind -> status dict
        self._results = results
        self._unit = unit
        self._batch = batch
        self._all = diagnostics

    @property
    def all_diagnostics(self) -> list:
        if self._all is None:
            self._all = self._results.diagnostics(self._unit) if self._results is not None else []
        return self._all

    @property
    def diagnostics(self) -> list:
        return [d for d in self.all_diagnostics if not d.suppressed]

    @property
    def has_errors(self) -> bool:
        return any(d.is_error for d in self.diagnostics)

    def structs(self, pass_index: int = 0) -> list:
        """The struct declarations of one compile pass's AST, in source order
        (walks.StructInfo: name, struct-level specifiers, member functions) --
        the StructDecl items of ``parse(preprocess(text, profile.passes()[i]))``
        (test_acceptance.py:132-135) as far as the classification needs them.
        This is the AST the analysis walks: under the plain profile with
        erase_specifiers its specifiers are erased (spacecheck.py:697-699)."""
        if self._batch is None:
            raise RuntimeError("struct declarations need an analysis run with want_walks=True")
        return self._batch.structs_of(self._unit, pass_index)

    def __repr__(self):
        return f"Analysis(path={self.path!r}, mode={self.mode}, diagnostics={len(self.diagnostics)})"


class AnalysisList(Sequence):
    """The Analysis of every unit of one run, in input order, each built on
    first access (a corpus run returns ~10k of them per GB).  ``settings`` is
    one (profile, mode) for every unit or a list of them."""

    def __init__(self, paths: list, settings, results: CorpusResults):
        self._paths = paths
        self._settings = settings
        self._uniform = isinstance(settings, tuple)
        self._results = results
        self._made: dict = {}

    def __len__(self):
        return len(self._paths)

    def _get(self, i: int) -> "Analysis":
        a = self._made.get(i)
        if a is None:
            prof, mode = self._settings if self._uniform else self._settings[i]
            a = self._made[i] = Analysis(self._paths[i], prof, mode, self._results, i)
        return a

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self._get(k) for k in range(*i.indices(len(self._paths)))]
        if i < 0:
            i += len(self._paths)
        if not 0 <= i < len(self._paths):
            raise IndexError(i)
        return self._get(i)

    def __iter__(self):
        return (self._get(i) for i in range(len(self._paths)))


# ---------------------------------------------------------------------------
# the engine

class Engine:
    """A GPU-resident analyser; one instance per device."""

    def __init__(self, device: int = 0, lib_path=None, batch_mib: int = 1024):
        self.handle = _native.Handle(device, lib_path)
        self.lock = threading.Lock()
        self.last_stats: dict = {}
        self.last_result_bytes = 0
        self.batch_mib = batch_mib
        self.handle.set_option(7, batch_mib)

    def _run(self, texts: list, paths: list, cfg: np.ndarray, settings) -> "AnalysisList":
        """Streamed run without walk records; ``settings`` as in AnalysisList."""
        with self.lock:
            self.handle.set_option(1, 0)
            self.handle.run_units(texts, cfg)
            recs, text, first, lease = self.handle.lease_results()
            self.last_stats = self.handle.stats()
            self.last_result_bytes = recs.nbytes + text.nbytes + first.nbytes
        return AnalysisList(paths, settings, CorpusResults(recs, text, first, paths, lease))

    def run_batch(self, units: list, want_walks: bool = False):
        """units: list of (text, path, CompileProfile, Mode, TraitConfig).

        Returns a list of Analysis in input order.  The texts go to the
        library without copies (exs_run_units streams them in batches); the
        diagnostics come back rendered, ordered and de-duplicated."""
        texts = [u[0] for u in units]
        memo: dict = {}

        def cb(u):
            k = (id(u[2]), id(u[3]), id(u[4]))  # the units hold these objects: ids are stable
            b = memo.get(k)
            if b is None:
                b = memo[k] = cfg_byte(u[2], u[3], u[4])
            return b
        cfg = np.fromiter(map(cb, units), dtype=np.uint8, count=len(units))
        paths = [u[1] for u in units]
        if not want_walks:
            return self._run(texts, paths, cfg, [(u[2], u[3]) for u in units])
        with self.lock:
            # walk arrays describe one batch: keep the whole run in one
            self.handle.set_option(7, 2047)
            self.handle.set_option(1, 1)
            try:
                self.handle.run_units(texts, cfg)
            finally:
                self.handle.set_option(7, self.batch_mib)
            recs, text, first, lease = self.handle.lease_results()
            self.last_stats = self.handle.stats()
            self.last_result_bytes = recs.nbytes + text.nbytes + first.nbytes
            results = CorpusResults(recs, text, first, paths, lease)
            if self.last_stats["batches"] != 1:
                raise ValueError("want_walks needs the units to fit one batch (< 2 GiB)")
            walks = self.handle.walk_stats(len(units))
            status = self.handle.pass_status(len(units))
            blobs = [t.encode("utf-8", "surrogateescape") if isinstance(t, str) else bytes(t) for t in texts]
            offsets = [0]
            for b in blobs:
                offsets.append(offsets[-1] + len(b))
            ren = Renderer(b"".join(blobs), offsets, self.handle.arena(), self.handle.describe)
            # the walk arrays stay valid until the next run on this engine:
            # snapshot them now (lazily rendered afterwards)
            batch = BatchWalks(self.handle, ren, status, [u[3] for u in units])
            batch._load()
        out = []
        for f, u in enumerate(units):
            a = Analysis(u[1], u[2], u[3], results, f, batch)
            for p, side in ((0, HOST), (1, DEVICE)):
                w = walks[2 * f + p]
                if w["exists"]:
                    a.walks[side] = WalkSummary(side, int(w["instances"]), int(w["edges"]),
                                                int(w["demands"]), batch, (f, p))
            for p, kind in enumerate(u[2].pass_kinds()):
                s = status[2 * f + p]
                a.passes[kind] = {"pp_line": int(s["pp_line"]), "lex_line": int(s["lex_line"]),
                                  "parse_failed": bool(s["parse_failed"])}
            out.append(a)
        return out


_ENGINES: dict = {}
_ENGINE_LOCK = threading.Lock()


def get_engine(device: int = 0) -> Engine:
    with _ENGINE_LOCK:
        e = _ENGINES.get(device)
        if e is None:
            e = Engine(device)
            _ENGINES[device] = e
        return e


def analyze(text: str, path: str = "<unit>", profile: CompileProfile = CompileProfile(),
            mode: Mode = Mode.CLASSIC, cfg: TraitConfig = TraitConfig()) -> Analysis:
    """Preprocess, parse, resolve and space-check one unit (spacecheck.py:687-739)."""
    return get_engine().run_batch([(text, path, profile, mode, cfg)], want_walks=True)[0]


def check_unit(text: str, path: str = "<unit>", profile: CompileProfile = CompileProfile(),
               mode: Mode = Mode.CLASSIC, cfg: TraitConfig = TraitConfig()) -> list:
    """The ordered diagnostic list for one unit (spacecheck.py:742-750)."""
    return analyze(text, path, profile, mode, cfg).diagnostics


def analyze_corpus(units: Iterable, profile: CompileProfile = CompileProfile(),
                   mode: Mode = Mode.CLASSIC, cfg: TraitConfig = TraitConfig(),
                   device: int = 0, want_walks: bool = False, engine: Optional[Engine] = None) -> list:
    """Batch analysis: ``analyze`` over every unit (corpus.py:163-175).

    ``units`` yields (path, text) or (path, text, profile, mode, cfg); any
    total size (the library streams them in batches).  Returns one Analysis
    per unit, in input order."""
    units = units if isinstance(units, list) else list(units)
    eng = engine or get_engine(device)
    if not want_walks and all(len(u) == 2 for u in units):
        # one setting for every unit: no per-unit tuples or cfg lookups
        cfg_all = np.full(len(units), cfg_byte(profile, mode, cfg), dtype=np.uint8)
        return eng._run([u[1] for u in units], [u[0] for u in units], cfg_all, (profile, mode))
    packed = [(u[1], u[0], profile, mode, cfg) if len(u) == 2 else (u[1], u[0], u[2], u[3], u[4]) for u in units]
    return eng.run_batch(packed, want_walks=want_walks)


def declared_spaces(spec: int) -> frozenset:
    """sema.py:627-635 on specifier bits (1 host, 2 device; global counts as host)."""
    out = {sp for b, sp in ((1, HOST), (2, DEVICE)) if spec & b}
    return frozenset(out or {HOST})


def propagate_spaces(analysis: Analysis) -> dict:
    """Instance display name -> effective spaces over all walks (spacecheck.py:770-782)."""
    out: dict = {}
    for walk in analysis.walks.values():
        for inst in walk.instances.values():
            acc = out.setdefault(inst.display, set())
            if inst.spaces == GLOBAL:
                acc.add(ExecSpace.Global)
            else:
                acc.update(inst.spaces)
    return {k: frozenset(v) for k, v in out.items()}


def struct_member_spaces(struct: StructInfo) -> dict:
    """Declared member spaces with the struct-level decoration distributed to
    undecorated members (spacecheck.py:785-793)."""
    out = {}
    for name, spec in struct.members:
        if not spec & 7 and struct.spec & 7:
            spec = struct.spec
        out[name] = declared_spaces(spec)
    return out


def stray_set(analysis: Analysis) -> list:
    """The stray-coded subset of the ordered diagnostics."""
    return [d for d in analysis.diagnostics if d.code in STRAY_CODES]


__all__ = [
    "Analysis", "AnalysisList", "CODE_REGISTRY", "CompileProfile", "CorpusResults", "Diagnostic", "Engine", "ExecSpace", "GLOBAL",
    "Mode", "Severity", "SrcLoc", "StructInfo", "TraitConfig", "Verdict", "analyze",
    "analyze_corpus", "check_unit", "declared_spaces", "finish_diagnostics", "format_diagnostic",
    "get_engine", "legality", "propagate_spaces", "stray_set", "stray_text",
    "struct_member_spaces",
]
