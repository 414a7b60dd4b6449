"""ctypes binding of the C ABI in include/exspace_b200.h.

The product library is ``libexspace_b200.so`` (sm_100a, built in-tree by
``__graft_entry__.build()``).  There is no CPU fallback: if the library or a
CUDA device is missing, ``Engine()`` raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libexspace_b200.so"

DIAG_DTYPE = np.dtype([
    ("file", "<u4"), ("line", "<u4"), ("col", "<u4"), ("code", "<u2"), ("msg", "<u2"),
    ("a0", "<u8"), ("a1", "<u8"), ("a2", "<u8"), ("a3", "<u4"),
    ("suppressed", "u1"), ("pad", "u1", (3,)),
])
assert DIAG_DTYPE.itemsize == 48

TOKEN_DTYPE = np.dtype([
    ("pos", "<u4"), ("end", "<u4"), ("line", "<u4"), ("col", "<u4"), ("hv", "<u8"),
    ("kind", "u1"), ("id", "u1"), ("mask", "u1"), ("flags", "u1"), ("file", "<u4"),
])
assert TOKEN_DTYPE.itemsize == 32

PASS_DTYPE = np.dtype([
    ("pp_line", "<u4"), ("pp_msg", "<u2"), ("exists", "<u2"), ("lex_line", "<u4"),
    ("lex_col", "<u4"), ("lex_msg", "<u2"), ("pad", "<u2"), ("eof_line", "<u4"),
    ("eof_col", "<u4"), ("view", "<u4"), ("parse_failed", "<u4"),
])

WALK_DTYPE = np.dtype([("instances", "<u4"), ("edges", "<u4"), ("demands", "<u4"), ("exists", "<u4")])

DESC_DTYPE = np.dtype([
    ("name", "<u8"), ("owner", "<u8"), ("otype", "<u8"), ("otarg", "u1"), ("nb", "u1"),
    ("pad", "u1", (6,)), ("bname", "<u8", (2,)), ("bval", "<u8", (2,)), ("bkind", "u1", (2,)),
    ("bvx", "u1", (2,)), ("pad2", "u1", (4,)),
])


class Stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "bytes", "files", "lines", "directives", "tokens", "views", "view_tokens", "items",
        "functions", "structs", "instances", "edges", "callsites", "levels", "diagnostics",
        "retries", "gpu_launches")] + [(n, C.c_float) for n in (
        "ms_lex", "ms_parse", "ms_sema", "ms_walk", "ms_total", "ms_h2d", "ms_d2h", "ms_wall")] + [
        ("batches", C.c_uint32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


EXPORTS = [
    "exs_create", "exs_destroy", "exs_last_error", "exs_run", "exs_run_device", "exs_get_stats",
    "exs_get_diags", "exs_diags_view", "exs_get_arena", "exs_get_pass_status", "exs_get_tokens",
    "exs_get_walk_stats", "exs_describe", "exs_set_option", "exs_stage_times", "exs_profile_text",
    "exs_get_decls", "exs_get_structs", "exs_get_instances", "exs_get_edges", "exs_get_nodes",
    "exs_get_token_range", "exs_run_units", "exs_results_view", "exs_results_copy", "exs_set_collective",
    "exs_results_lease", "exs_results_release",
]

# exs_allgather_fn (include/exspace_b200.h)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.POINTER(C.c_uint64))

# one finished diagnostic (include/exspace_b200.h exs_result)
RESULT_DTYPE = np.dtype([("unit", "<u4"), ("line", "<u4"), ("col", "<u4"), ("msg_len", "<u4"),
                         ("msg_off", "<u8"), ("code", "<u2"), ("suppressed", "u1"), ("pad", "u1", (5,))])
assert RESULT_DTYPE.itemsize == 32

_AS_UTF8 = C.pythonapi.PyUnicode_AsUTF8AndSize
_AS_UTF8.argtypes = [C.py_object, C.POINTER(C.c_ssize_t)]
_AS_UTF8.restype = C.c_void_p


def _ascii_data_offset():
    """Offset of a compact ASCII str's characters from the object address
    (CPython: sizeof(PyASCIIObject), PyUnicode_DATA of a compact ASCII string),
    verified on probe strings; None if this interpreter lays strings out
    differently (text_pointers then asks CPython per string)."""
    probes = ["exs-probe", "x" * 257, "".join(chr(97 + k % 26) for k in range(64))]
    for off in (40, 48, 32, 56, 24):
        if all(C.string_at(id(p) + off, len(p)) == p.encode("ascii") for p in probes):
            return off
    return None


_ASCII_OFF = _ascii_data_offset()


def text_pointers(texts):
    """(pointer array, length array, keep-alive list) for a list of str/bytes
    without copying them: an ASCII str's characters are its UTF-8 bytes, read
    in place; other strs give CPython's cached UTF-8 form; text with lone
    surrogates is encoded with surrogateescape (the reference's byte view of
    such input)."""
    n = len(texts)
    if _ASCII_OFF is not None and n and all(type(t) is str for t in texts) and all(map(str.isascii, texts)):
        ptrs = np.fromiter(map(id, texts), dtype=np.uint64, count=n) + np.uint64(_ASCII_OFF)
        lens = np.fromiter(map(len, texts), dtype=np.uint64, count=n)
        return ptrs, lens, []
    ptrs = np.zeros(n, dtype=np.uint64)
    lens = np.zeros(n, dtype=np.uint64)
    keep = []
    size = C.c_ssize_t()
    for i, t in enumerate(texts):
        if isinstance(t, str):
            try:
                p = _AS_UTF8(t, C.byref(size))
                ptrs[i] = p or 0
                lens[i] = size.value
                continue
            except UnicodeEncodeError:
                t = t.encode("utf-8", "surrogateescape")
        b = bytes(t)
        keep.append(b)
        cp = C.c_char_p(b)
        keep.append(cp)
        ptrs[i] = C.cast(cp, C.c_void_p).value or 0
        lens[i] = len(b)
    return ptrs, lens, keep


DECL_DTYPE = np.dtype([("node", "<u4"), ("view", "<u4"), ("rec", "<u4"), ("order", "<u4"),
                       ("ncalls", "<u4"), ("flags", "<u4")])
STRUCT_DTYPE = np.dtype([("node", "<u4"), ("view", "<u4")])
_VAL = [("k", "u1"), ("targ", "u1"), ("bt", "u1"), ("pad", "u1"), ("rec", "<u4"), ("x", "<u8")]
INST_DTYPE = np.dtype([("decl", "<u4"), ("walk", "<u4"), ("side", "<u4"), ("at", "<u4"),
                       ("ebase", "<u4"), ("ecnt", "<u4"), ("flags", "<u4"), ("spaces", "<u4"),
                       ("ckey", "<u8")] + [(f"{v}_{n}", t) for v in ("tb", "hb", "ot") for n, t in _VAL])
NODE_DTYPE = np.dtype([("kind", "u1"), ("sub", "u1"), ("n", "<u2"), ("tok", "<u4"), ("c0", "<u4"),
                       ("c1", "<u4"), ("c2", "<u4"), ("next", "<u4"), ("hv", "<u8")])
assert DECL_DTYPE.itemsize == 24 and INST_DTYPE.itemsize == 88 and NODE_DTYPE.itemsize == 32


class NativeError(RuntimeError):
    pass


def load_library(path: str | os.PathLike | None = None) -> C.CDLL:
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise NativeError(
            f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (the analyser has no CPU fallback)")
    lib = C.CDLL(str(p))
    vp, u8p, u32p, u64p = C.c_void_p, C.POINTER(C.c_uint8), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)
    lib.exs_create.argtypes = [C.c_int, C.POINTER(vp)]
    lib.exs_destroy.argtypes = [vp]
    lib.exs_last_error.restype = C.c_char_p
    lib.exs_profile_text.restype = C.c_char_p
    lib.exs_run.argtypes = [vp, vp, C.c_uint64, vp, C.c_uint32, vp]
    lib.exs_run_device.argtypes = [vp, vp, C.c_uint64, vp, C.c_uint32, vp]
    lib.exs_get_stats.argtypes = [vp, C.POINTER(Stats)]
    lib.exs_get_diags.argtypes = [vp, vp, C.c_uint64, u64p]
    lib.exs_diags_view.argtypes = [vp, C.POINTER(C.c_void_p), u64p]
    for fn in ("exs_get_decls", "exs_get_structs", "exs_get_instances", "exs_get_edges", "exs_get_nodes"):
        getattr(lib, fn).argtypes = [vp, vp, C.c_uint64, u64p]
    lib.exs_get_token_range.argtypes = [vp, C.c_uint64, C.c_uint64, vp]
    lib.exs_get_arena.argtypes = [vp, vp, C.c_uint64, u64p]
    lib.exs_get_pass_status.argtypes = [vp, vp, C.c_uint64]
    lib.exs_get_tokens.argtypes = [vp, C.c_uint32, vp, C.c_uint64, u64p]
    lib.exs_get_walk_stats.argtypes = [vp, vp, C.c_uint64]
    lib.exs_describe.argtypes = [vp, vp, vp, C.c_uint32, vp]
    lib.exs_set_option.argtypes = [vp, C.c_int, C.c_int]
    lib.exs_stage_times.argtypes = [vp, C.POINTER(C.c_float)]
    lib.exs_run_units.argtypes = [vp, vp, vp, C.c_uint64, vp]
    lib.exs_results_copy.argtypes = [vp, vp, vp, vp]
    lib.exs_results_lease.argtypes = [vp, u64p]
    lib.exs_results_release.argtypes = [vp, C.c_uint64]
    lib.exs_set_collective.argtypes = [vp, C.c_int, C.c_int, ALLGATHER_FN, vp]
    lib.exs_results_view.argtypes = [vp, C.POINTER(C.c_void_p), u64p, C.POINTER(C.c_void_p), u64p,
                                     C.POINTER(C.c_void_p), u64p]
    for name in EXPORTS:
        if name not in ("exs_last_error", "exs_profile_text"):
            getattr(lib, name).restype = C.c_int
    _ = (u8p, u32p)
    return lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class ResultsLease:
    """Keeps a run's result buffers (and their handle) alive; released when
    the last view of them is garbage-collected."""

    def __init__(self, handle: "Handle", lease: int):
        self.handle = handle
        self.lease = lease

    def __del__(self):
        try:
            if self.handle.h:
                self.handle.lib.exs_results_release(self.handle.h, self.lease)
        except Exception:
            pass


class Handle:
    """One analyser instance bound to one GPU."""

    def __init__(self, device: int = 0, lib_path=None):
        self.lib = load_library(lib_path)
        h = C.c_void_p()
        self._check(self.lib.exs_create(device, C.byref(h)))
        self.h = h

    def _check(self, rc):
        if rc != 0:
            raise NativeError(self.lib.exs_last_error().decode(errors="replace"))

    def close(self):
        if getattr(self, "h", None):
            self.lib.exs_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, key: int, value: int):
        self._check(self.lib.exs_set_option(self.h, key, value))

    def run(self, data: np.ndarray, offsets: np.ndarray, cfg: np.ndarray):
        data = np.ascontiguousarray(data, dtype=np.uint8)
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        cfg = np.ascontiguousarray(cfg, dtype=np.uint8)
        self._check(self.lib.exs_run(self.h, _ptr(data), data.size, _ptr(offsets),
                                     len(offsets) - 1, _ptr(cfg)))

    def run_device(self, dev_ptr: int, n_bytes: int, offsets: np.ndarray, cfg: np.ndarray):
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        cfg = np.ascontiguousarray(cfg, dtype=np.uint8)
        self._check(self.lib.exs_run_device(self.h, C.c_void_p(dev_ptr), n_bytes, _ptr(offsets),
                                            len(offsets) - 1, _ptr(cfg)))

    def run_units(self, texts, cfg: np.ndarray):
        """Analyse units given as str/bytes (exs_run_units: streamed batches)."""
        ptrs, lens, keep = text_pointers(texts)
        cfg = np.ascontiguousarray(cfg, dtype=np.uint8)
        self._check(self.lib.exs_run_units(self.h, _ptr(ptrs), _ptr(lens), len(ptrs), _ptr(cfg)))
        del keep

    def lease_results(self):
        """Zero-copy results of the last run: (records, message bytes,
        unit_first, lease).  The views stay valid while `lease` lives (the
        handle's later runs fill other buffers)."""
        n = C.c_uint64()
        self._check(self.lib.exs_results_lease(self.h, C.byref(n)))
        lease = ResultsLease(self, n.value)
        recs, text, first = self.results(copy=False)
        return recs, text, first, lease

    def results(self, copy: bool = True):
        """(records, message bytes, unit_first) of the last run.  copy=False
        returns views of the handle's page-locked buffers, valid until its
        next run."""
        rp, tp, up = C.c_void_p(), C.c_void_p(), C.c_void_p()
        n, tb, nu = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self._check(self.lib.exs_results_view(self.h, C.byref(rp), C.byref(n), C.byref(tp), C.byref(tb),
                                              C.byref(up), C.byref(nu)))

        def view(ptr, nbytes):
            if not nbytes:
                return np.zeros(0, dtype=np.uint8)
            return np.frombuffer((C.c_uint8 * nbytes).from_address(ptr.value), dtype=np.uint8)

        if copy:  # into fresh arrays, by the library's copy threads
            recs = np.empty(n.value, dtype=RESULT_DTYPE)
            text = np.empty(tb.value, dtype=np.uint8)
            first = np.zeros(nu.value + 1, dtype=np.uint64)
            self._check(self.lib.exs_results_copy(self.h, _ptr(recs), _ptr(text), _ptr(first)))
            return recs, text, first
        recs = view(rp, n.value * RESULT_DTYPE.itemsize)
        text = view(tp, tb.value)
        first = view(up, (nu.value + 1) * 8) if up.value else np.zeros(8, dtype=np.uint8)
        return recs.view(RESULT_DTYPE), text, first.view(np.uint64)

    def set_collective(self, rank: int, world: int, allgather=None):
        """Walk every batch across `world` ranks (exs_set_collective);
        `allgather` is an ALLGATHER_FN (kept alive here)."""
        self._allgather = allgather
        self._check(self.lib.exs_set_collective(self.h, rank, world,
                                                allgather if allgather is not None else ALLGATHER_FN(0), None))

    def stats(self) -> dict:
        s = Stats()
        self._check(self.lib.exs_get_stats(self.h, C.byref(s)))
        return s.as_dict()

    def diags(self, copy: bool = True) -> np.ndarray:
        """Ordered diagnostic records of the last run.  copy=False returns a
        read-only view of the handle's page-locked buffer (valid until the
        next run on this handle) instead of copying it."""
        n = C.c_uint64()
        p = C.c_void_p()
        self._check(self.lib.exs_diags_view(self.h, C.byref(p), C.byref(n)))
        if not n.value:
            return np.zeros(0, dtype=DIAG_DTYPE)
        buf = (C.c_uint8 * (n.value * DIAG_DTYPE.itemsize)).from_address(p.value)
        raw = np.frombuffer(buf, dtype=np.uint8)
        if copy:  # a byte copy: numpy copies structured records field by field
            return raw.copy().view(DIAG_DTYPE)
        view = raw.view(DIAG_DTYPE)
        view.flags.writeable = False
        return view

    def _records(self, fn: str, dtype) -> np.ndarray:
        n = C.c_uint64()
        f = getattr(self.lib, fn)
        self._check(f(self.h, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=dtype)
        if n.value:
            self._check(f(self.h, _ptr(out), n.value, C.byref(n)))
        return out

    # walk materialisation (include/exspace_b200.h): arrays of the last run
    def decls(self) -> np.ndarray:
        return self._records("exs_get_decls", DECL_DTYPE)

    def structs(self) -> np.ndarray:
        return self._records("exs_get_structs", STRUCT_DTYPE)

    def instances(self) -> np.ndarray:
        return self._records("exs_get_instances", INST_DTYPE)

    def edges(self) -> np.ndarray:
        return self._records("exs_get_edges", np.dtype("<u4"))

    def nodes(self) -> np.ndarray:
        return self._records("exs_get_nodes", NODE_DTYPE)

    def token_range(self, first: int, count: int) -> np.ndarray:
        out = np.zeros(count, dtype=TOKEN_DTYPE)
        if count:
            self._check(self.lib.exs_get_token_range(self.h, first, count, _ptr(out)))
        return out

    def arena(self) -> bytes:
        n = C.c_uint64()
        self._check(self.lib.exs_get_arena(self.h, None, 0, C.byref(n)))
        out = np.zeros(max(n.value, 1), dtype=np.uint8)
        if n.value:
            self._check(self.lib.exs_get_arena(self.h, _ptr(out), n.value, C.byref(n)))
        return out[: n.value].tobytes()

    def pass_status(self, n_files: int) -> np.ndarray:
        out = np.zeros(2 * n_files, dtype=PASS_DTYPE)
        self._check(self.lib.exs_get_pass_status(self.h, _ptr(out), 2 * n_files))
        return out

    def tokens(self, file: int) -> np.ndarray:
        n = C.c_uint64()
        self._check(self.lib.exs_get_tokens(self.h, file, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=TOKEN_DTYPE)
        if n.value:
            self._check(self.lib.exs_get_tokens(self.h, file, _ptr(out), n.value, C.byref(n)))
        return out

    def walk_stats(self, n_files: int) -> np.ndarray:
        out = np.zeros(2 * n_files, dtype=WALK_DTYPE)
        self._check(self.lib.exs_get_walk_stats(self.h, _ptr(out), 2 * n_files))
        return out

    def describe(self, ids, kinds) -> np.ndarray:
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        kinds = np.ascontiguousarray(kinds, dtype=np.uint8)
        out = np.zeros(len(ids), dtype=DESC_DTYPE)
        if len(ids):
            self._check(self.lib.exs_describe(self.h, _ptr(ids), _ptr(kinds), len(ids), _ptr(out)))
        return out

    def stage_times(self):
        out = (C.c_float * 4)()
        self._check(self.lib.exs_stage_times(self.h, out))
        return list(out)
