"""Seeded synthetic MiniCU corpora for the BASELINE.json configs (C2-C5).

The unit shape follows the reference's property-suite generator
(``pkg/tests/genprog.py:29-89``): structs ``S{i}`` with an optional ``hdc`` tag
and a ``call()`` member of random execution space, host-device templates
``w{j}<T>`` calling ``T{}.call()``, an optional kernel, and ``main``.  For the
large corpora every module gets a unique name prefix so that one file holds
many modules and exactly one ``main`` (a second ``main`` would be E0102).

All output is ASCII with LF line ends.  Deterministic for a given seed.
"""
from __future__ import annotations

import random

SPECS = ["", "__host__", "__device__", "__host__ __device__"]
HDCS = [None, "Hst", "Dev", "HstDev"]


def _module(rng: random.Random, pfx: str, lines: list, main_calls: list,
            pragma_p: float = 0.7, kernel_p: float = 0.7):
    nstructs = rng.randint(2, 4)
    has_value = []
    for i in range(nstructs):
        lines.append(f"struct {pfx}S{i} {{")
        tag = rng.choice(HDCS)
        if tag:
            lines.append(f"  static constexpr HDC hdc = HDC::{tag};")
        spec = rng.choice(SPECS)
        lines.append(f"  {spec} void call() {{}}" if spec else "  void call() {}")
        value = rng.random() < 0.5
        has_value.append(value)
        if value:
            lines.append("  constexpr static int value() { return 1; }")
        lines.append("};")
    ntmpl = rng.randint(1, 2)
    for j in range(ntmpl):
        if rng.random() < pragma_p:
            lines.append("#pragma " + rng.choice(["hd_warning_disable", "nv_exec_check_disable"]))
        lines.append("template< typename T >")
        lines.append("__host__ __device__")
        body = "T{}.call();"
        if rng.random() < 0.3:
            body += " T{}.call();"
        lines.append(f"void {pfx}w{j}() {{ {body} }}")
    if rng.random() < kernel_p:
        lines.append(f"__global__ void {pfx}kern() {{")
        lines.append(f"  {pfx}w{rng.randrange(ntmpl)}< {pfx}S{rng.randrange(nstructs)} >();")
        cands = [i for i in range(nstructs) if has_value[i]]
        if cands and rng.random() < 0.6:
            lines.append(f"  {pfx}S{rng.choice(cands)}{{}}.value();")
        lines.append("}")
        if rng.random() < 0.8:
            main_calls.append(f"  {pfx}kern<<< {rng.randint(1, 3)}, {rng.randint(1, 3)} >>>();")
    for _ in range(rng.randint(1, 3)):
        main_calls.append(f"  {pfx}w{rng.randrange(ntmpl)}< {pfx}S{rng.randrange(nstructs)} >();")


def gen_c2_file(seed: int, target_bytes: int = 100_000) -> str:
    """One C2 unit of about ``target_bytes``: many modules, one main."""
    rng = random.Random(seed * 7919 + 17)
    lines: list = []
    calls: list = []
    size = 0
    k = 0
    while size < target_bytes - 2_000 or k == 0:
        before = len(lines)
        _module(rng, f"M{k}_", lines, calls)
        size += sum(len(x) + 1 for x in lines[before:])
        size += 40  # main-call lines, roughly
        k += 1
    lines.append("int main() {")
    lines.extend(calls)
    lines.append("  return cudaDeviceSynchronize();")
    lines.append("}")
    return "\n".join(lines) + "\n"


def gen_c2(n_files: int, target_bytes: int = 100_000, seed0: int = 0):
    """(paths, texts) of a C2 corpus; flat, path-sorted names."""
    paths = [f"c2/f{seed0 + i:07d}.cu" for i in range(n_files)]
    texts = [gen_c2_file(seed0 + i, target_bytes) for i in range(n_files)]
    return paths, texts


def gen_chain(depth: int = 64, nstructs: int = 1024) -> str:
    """C3: template chains w{d}<T> -> w{d-1}<T>."""
    specs = ["", "__host__ ", "__device__ ", "__host__ __device__ "]
    tags = [None, "Dev", "HstDev"]
    out = []
    for i in range(nstructs):
        out.append(f"struct S{i} {{")
        if tags[i % 3]:
            out.append(f"  static constexpr HDC hdc = HDC::{tags[i % 3]};")
        out.append(f"  {specs[i % 4]}void call() {{}}")
        out.append("};")
    out.append("template< typename T >\n__host__ __device__\nvoid w0() { T{}.call(); }")
    for d in range(1, depth):
        out.append(f"template< typename T >\n__host__ __device__\nvoid w{d}() {{ w{d - 1}< T >(); }}")
    out.append("__global__ void kern() {")
    for i in range(0, nstructs, 2):
        out.append(f"  w{depth - 1}< S{i} >();")
    out.append("}")
    out.append("int main() {")
    for i in range(1, nstructs, 2):
        out.append(f"  w{depth - 1}< S{i} >();")
    out.append("  kern<<< 1, 1 >>>();")
    out.append("  return cudaDeviceSynchronize();")
    out.append("}")
    return "\n".join(out) + "\n"


def gen_callgraph(nfuncs: int, fanout: int = 10, seed: int = 0) -> str:
    """C4: one unit, ``nfuncs`` free functions each calling ``fanout`` others."""
    rng = random.Random(seed)
    specs = ["", "__host__ ", "__device__ ", "__host__ __device__ "]
    out = []
    for i in range(nfuncs):
        calls = " ".join(f"f{rng.randrange(nfuncs)}();" for _ in range(fanout))
        out.append(f"{rng.choice(specs)}void f{i}() {{ {calls} }}")
    out.append("__global__ void kern() { f0(); }")
    out.append("int main() { f1(); kern<<< 1, 1 >>>(); return 0; }")
    return "\n".join(out) + "\n"


_GUARDS = ["__CUDA_ARCH__", "__CUDACC__", "__CUDACC_RELAXED_CONSTEXPR__"]


def _stress_module(rng: random.Random, pfx: str, lines: list, calls: list):
    """A C2 module decorated with valid lexer/preprocessor stressors."""
    inner: list = []
    _module(rng, pfx, inner, calls)
    for ln in inner:
        r = rng.random()
        if r < 0.05:
            lines.append("/* block /* not nested " + pfx + " ** / still in comment")
            lines.append("   // slashes inside a block */ " + ln)
        elif r < 0.10:
            lines.append("// line comment continued \\")
            lines.append("   still a comment " + pfx)
            lines.append(ln)
        elif r < 0.15 and ln.startswith("void ") and "(" in ln:
            # split an identifier with a backslash continuation
            cut = 2
            lines.append(ln[:cut] + "\\")
            lines.append(ln[cut:])
        elif r < 0.20:
            g = rng.choice(_GUARDS)
            lines.append(f"#ifdef {g}")
            lines.append(ln)
            lines.append("#else")
            lines.append(ln)
            lines.append("#endif")
        elif r < 0.23:
            lines.append("#ifndef __CUDACC__")
            lines.append("#error this branch is never active under nvcc")
            lines.append("#endif")
            lines.append(ln)
        else:
            lines.append(ln)
    if rng.random() < 0.3:
        lines.append(f"__host__ __device__ void {pfx}say() {{ printf( \"// not /* a comment %d\", 1 ); }}")


def gen_c5_file(seed: int, target_bytes: int = 100_000, malformed_p: float = 0.01) -> str:
    rng = random.Random(seed * 104729 + 3)
    lines: list = []
    calls: list = []
    size = 0
    k = 0
    while size < target_bytes - 2_000 or k == 0:
        before = len(lines)
        _stress_module(rng, f"M{k}_", lines, calls)
        size += sum(len(x) + 1 for x in lines[before:]) + 40
        k += 1
    lines.append("int main() {")
    lines.extend(calls)
    lines.append("  return cudaDeviceSynchronize();")
    lines.append("}")
    text = "\n".join(lines) + "\n"
    if rng.random() < malformed_p:
        kind = rng.randrange(3)
        pos = rng.randrange(len(text) // 2, len(text))
        if kind == 0:
            text = text[:pos] + " void broken( {\n" + text[pos:]
        elif kind == 1:
            text = "#ifdef __CUDA_ARCH__\n" + text
        else:
            text = text[:pos] + " @ " + text[pos:]
    return text
