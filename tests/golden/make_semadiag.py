"""Golden group ``semadiag``: seeded units that drive the sema diagnostics the
other groups never reach -- E0103 (hdc member not an HDC constant,
sema.py:395-402,437-438), E1301/E1302 (no viable / ambiguous overload,
sema.py:535-541), E1401 (all execution-space predicates false,
sema.py:651-657) -- mixed with the stray codes, under every mode.

Run (build container only; needs /root/reference):
    python tests/golden/make_semadiag.py
Writes tests/golden/semadiag.json.gz with make_golden.run_case, i.e. the
REAL reference's ``analyze`` output.  The GPU box only reads the fixture.
"""
from __future__ import annotations

import collections
import gzip
import json
import random
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
import make_golden as MG  # noqa: E402  (puts the reference on sys.path)

MODES = MG.MODES
HDCV = ["Hst", "Dev", "HstDev"]
SPECS = ["", "__host__", "__device__", "__host__ __device__"]

# struct shapes: (name, text); B*/I*/V* have an hdc member that is not an HDC
# constant (E0103 once a trait or default reads it)
STRUCTS = [
    ("H", "struct H {{\n  __host__ void call() {{}}\n}};"),
    ("D", "struct D {{\n  static constexpr HDC hdc = HDC::Dev;\n  __device__ void call() {{}}\n}};"),
    ("HD", "struct HD {{\n  static constexpr HDC hdc = HDC::HstDev;\n  __host__ __device__ void call() {{}}\n}};"),
    ("B", "struct B {{\n  static constexpr bool hdc = true;\n  {spec} void call() {{}}\n}};"),
    ("I", "struct I {{\n  static constexpr int hdc = 1;\n  {spec} void call() {{}}\n}};"),
    ("V", "struct V {{\n  static constexpr HDC hdc = false;\n  {spec} void call() {{}}\n}};"),
    ("W", "struct W {{\n  static constexpr bool on = true;\n  static constexpr HDC hdc = on;\n  {spec} void call() {{}}\n}};"),
    ("Q", "struct Q {{\n  static constexpr bool on = {b};\n  static constexpr HDC hdc = HDC::{h};\n  {spec} void call() {{}}\n}};"),
    ("P", "template< HDC x >\nstruct P {{\n  static constexpr HDC hdc = x;\n  {spec} void call() {{}}\n}};"),
]


def gate(rng, var):
    """A requires-clause body over one HDC parameter."""
    atoms = [f"{var} == HDC::{rng.choice(HDCV)}", f"{var} != HDC::{rng.choice(HDCV)}",
             "true", "false", f"{var} == {var}"]
    e = rng.choice(atoms)
    r = rng.random()
    if r < 0.25:
        e = f"{e} && {rng.choice(atoms)}"
    elif r < 0.45:
        e = f"{e} || {rng.choice(atoms)}"
    elif r < 0.55:
        e = f"!( {e} )"
    return e


def targ(rng, names):
    r = rng.random()
    if r < 0.55:
        n = rng.choice(names)
        return f"P< HDC::{rng.choice(HDCV)} >" if n == "P" else n
    if r < 0.7:
        return "int"
    if r < 0.8:
        return "bool"
    return f"P< HDC::{rng.choice(HDCV)} >" if "P" in names else rng.choice(names)


def gen_unit(rng: random.Random, mode: str) -> str:
    out = []
    chosen = rng.sample(STRUCTS, rng.randint(3, 6))
    names = [n for n, _ in chosen]
    for n, t in chosen:
        out.append(t.format(spec=rng.choice(SPECS), b=rng.choice(["true", "false"]),
                            h=rng.choice(HDCV)))
        out.append("")
    fns = []  # (name, kind) kind: g = HDC-targ gated, f = deduced T + trait default, w = wrapper
    # 1. HDC-gated overload sets g<x>()
    for k in range(rng.randint(1, 2)):
        name = f"g{k}"
        for _ in range(rng.randint(1, 3)):
            out.append("template< HDC x >")
            out.append(f"requires( {gate(rng, 'x')} )")
            sp = rng.choice(SPECS)
            out.append(f"{sp + ' ' if sp else ''}void {name}() {{}}")
        fns.append((name, "g"))
        out.append("")
    # 2. deduced overloads f(T) with an hdc<T> default (E0103 through the trait)
    if rng.random() < 0.8:
        for _ in range(rng.randint(1, 3)):
            out.append("template< typename T, HDC h = hdc<T> >")
            out.append(f"requires( {gate(rng, 'h')} )")
            sp = rng.choice(SPECS)
            out.append(f"{sp + ' ' if sp else ''}void f( T t ) {{ t.call(); }}")
        fns.append(("f", "f"))
        out.append("")
    # 3. conditional-space wrappers (E1401 under proposal1; E0001 elsewhere)
    for k in range(rng.randint(1, 2) if mode == "proposal1" or rng.random() < 0.1 else 0):
        name = f"w{k}"
        hp = f"hdc<T> == HDC::{rng.choice(HDCV)}"
        dp = f"hdc<T> == HDC::{rng.choice(HDCV)}"
        if rng.random() < 0.3:
            dp = f"hdc<T> != HDC::{rng.choice(HDCV)}"
        form = rng.randrange(4)
        if form == 0:
            spec = f"__host__( {hp} )\n__device__( {dp} )"
        elif form == 1:
            spec = f"__host__( {hp} )"
        elif form == 2:
            spec = f"__device__( {dp} )"
        else:
            spec = f"__host__ __device__( {dp} )"
        out.append("template< typename T >")
        out.append(spec)
        out.append(f"void {name}() {{\n  T{{}}.call();\n}}")
        fns.append((name, "w"))
        out.append("")
    # 4. a trait-reading default without gates (E0103 at the member)
    if rng.random() < 0.6:
        sp = rng.choice(["__host__ __device__", "", "__device__"])
        out.append("template< typename T, HDC y = hdc<T> >")
        out.append(f"{sp + ' ' if sp else ''}void k() {{}}")
        fns.append(("k", "k"))
        out.append("")

    def call(rng):
        name, kind = rng.choice(fns)
        if kind == "g":
            return f"{name}< HDC::{rng.choice(HDCV)} >();"
        if kind == "f":
            n = rng.choice(names)
            return f"f( {'P< HDC::' + rng.choice(HDCV) + ' >' if n == 'P' else n}{{}} );"
        return f"{name}< {targ(rng, names)} >();"

    have_kernel = rng.random() < 0.7
    if have_kernel:
        out.append("__global__ void kern() {")
        for _ in range(rng.randint(1, 3)):
            out.append("  " + call(rng))
        out.append("}")
        out.append("")
    out.append("int main() {")
    for _ in range(rng.randint(2, 5)):
        out.append("  " + call(rng))
    if have_kernel:
        out.append("  kern<<< 1, 1 >>>();")
    out.append("  return cudaDeviceSynchronize();")
    out.append("}")
    return "\n".join(out) + "\n"


# hand-written units from the verdict/tests (sema.py:395-402,535-541,651-657)
FIXED = [
    ("e1301_e1302_e0103", """struct B { static constexpr bool hdc = true; };
template< HDC x >
requires( x == HDC::Hst )
void g() {}
template< HDC x >
requires( x == HDC::Dev )
void g() {}
template< HDC x >
requires( true )
void h() {}
template< HDC x >
requires( x == x )
void h() {}
template< typename T, HDC y = hdc<T> >
void k() {}
int main() {
  g< HDC::HstDev >();
  h< HDC::Hst >();
  k< B >();
}
"""),
    ("e1401_wrap_hd", """struct D { static constexpr HDC hdc = HDC::Dev; __device__ void call() {} };
struct HD { static constexpr HDC hdc = HDC::HstDev; __host__ __device__ void call() {} };
template< typename T >
__host__( hdc<T> == HDC::Hst )
__device__( hdc<T> == HDC::Dev )
void wrap() { T{}.call(); }
int main() {
  wrap< HD >();
  wrap< D >();
  wrap< int >();
}
"""),
]


def main():
    cases = []
    for name, text in FIXED:
        for m in MODES:
            cases.append(MG.run_case(f"semadiag/{name}/{m}", text, m, detail=True))
    for seed in range(400):
        rng = random.Random(90_000 + seed)
        m = MODES[seed % 5]
        text = gen_unit(rng, m)
        comp = "plain" if seed % 13 == 0 else "nvcc"
        cases.append(MG.run_case(f"semadiag/{seed}/{m}/{comp}", text, m, comp,
                                 relaxed=(seed % 17 == 0 and comp == "nvcc"),
                                 fund=(seed % 7 == 0), detail=True))
    cases = [c for c in cases if c is not None]
    cnt = collections.Counter(d[0] for c in cases for d in c["diags"])
    units = collections.Counter(code for c in cases for code in {d[0] for d in c["diags"]})
    path = HERE / "semadiag.json.gz"
    with gzip.open(path, "wt", encoding="utf-8") as fh:
        json.dump(cases, fh, separators=(",", ":"))
    print(f"{path.name}: {len(cases)} cases, {path.stat().st_size} bytes")
    print("diagnostics per code:", dict(sorted(cnt.items())))
    print("units per code:", dict(sorted(units.items())))


if __name__ == "__main__":
    main()
