"""Render GPU diagnostic records into the reference's exact message strings.

Template ids mirror ``Msg`` in csrc/exs_common.cuh; texts are the reference's
(preprocess.py:177-202, lexer.py:75,86,116, parser.py, sema.py,
spacecheck.py:146-176,306-572,760-763).
"""
from __future__ import annotations

CODES = [None, "E0001", "E0002", "E0101", "E0102", "E0103", "E0104", "E1001", "E1002",
         "E1003", "E1004", "W1101", "W1102", "E1101", "E1102", "E1201", "E1301", "E1302",
         "E1401", "E1501", "W1502", "X9999"]

(M_NONE, M_PP_EXPECTS_ONE, M_PP_UNKNOWN_MACRO, M_PP_ELSE_NOMATCH, M_PP_SECOND_ELSE,
 M_PP_ENDIF_NOMATCH, M_PP_ERROR, M_PP_UNKNOWN_DIRECTIVE, M_PP_UNTERMINATED,
 M_LEX_PRAGMA, M_LEX_STRING, M_LEX_CHAR,
 M_P_EXPECTED, M_P_EXPECTED_NAME, M_P_UNKNOWN_PRAGMA, M_P_PRAGMA_FN,
 M_P_REQ_STRUCT, M_P_TPARAM_KIND, M_P_TPARAM_LIMIT, M_P_SPEC_REJECT,
 M_P_SPEC_DUP, M_P_GLOBAL_EXCL, M_P_STRUCT_SPEC, M_P_STRUCT_TPARAM,
 M_P_MEMBER_GLOBAL, M_P_MCONST_DECL, M_P_MCONST_TYPE, M_P_MCONST_STATIC,
 M_P_MCONST_SPEC, M_P_REQ_TEMPLATE, M_P_GLOBAL_VOID, M_P_GLOBAL_MEMBER,
 M_P_MAIN_SPEC, M_P_MAIN_SIG, M_P_FOR_VAR, M_P_PRINTF_FMT, M_P_PRINTF_TEXT,
 M_P_PRINTF_ONE, M_P_PRINTF_COUNT, M_P_ARITY, M_P_HDC_VALUE, M_P_EXPR,
 M_P_TARGS, M_P_DEPTH,
 M_S_DUP, M_S_STRUCT_SPEC_MODE, M_S_COND_SPEC_MODE, M_S_UNDEF_NAME,
 M_S_ASSERT_EVAL, M_S_ASSERT_FAIL, M_S_NO_TARGS_BUILTIN, M_S_UNDEF_TYPE,
 M_S_MISSING_TARGS, M_S_TOO_MANY_TARGS, M_S_HDC_MEMBER, M_S_NO_VIABLE,
 M_S_AMBIGUOUS, M_S_EMPTY_SPACES,
 M_W_PRED_CONST, M_W_NOT_TYPE, M_W_LAUNCH_DEVICE, M_W_LAUNCH_NONGLOBAL,
 M_W_RECEIVER, M_W_NO_MEMBER, M_W_GLOBAL_CALL, M_W_STRAY, M_W_E1201,
 M_W_SUBST, M_X_CONTRACT) = range(69)

FIXED = {
    M_PP_ELSE_NOMATCH: "#else without matching #ifdef/#ifndef",
    M_PP_SECOND_ELSE: "second #else in one conditional",
    M_PP_ENDIF_NOMATCH: "#endif without matching #ifdef/#ifndef",
    M_PP_UNTERMINATED: "unterminated #ifdef/#ifndef",
    M_LEX_PRAGMA: "malformed #pragma directive",
    M_LEX_STRING: "unterminated string literal",
    M_P_PRAGMA_FN: "a pragma must precede a function",
    M_P_REQ_STRUCT: "a requires clause cannot constrain a struct",
    M_P_TPARAM_KIND: "expected 'typename' or 'HDC' template parameter",
    M_P_TPARAM_LIMIT: "at most one type parameter and one HDC parameter are supported",
    M_P_GLOBAL_EXCL: "__global__ excludes __host__ and __device__",
    M_P_STRUCT_SPEC: "invalid specifier on a struct",
    M_P_STRUCT_TPARAM: "struct templates support only HDC parameters",
    M_P_MEMBER_GLOBAL: "__global__ is not allowed on member functions",
    M_P_GLOBAL_MEMBER: "__global__ is not allowed on member functions",
    M_P_MCONST_DECL: "invalid declaration of a member constant",
    M_P_MCONST_TYPE: "member constants must have type HDC, bool, or int",
    M_P_MCONST_STATIC: "member constants must be static constexpr",
    M_P_MCONST_SPEC: "invalid specifier on a member constant",
    M_P_REQ_TEMPLATE: "a requires clause needs a template header",
    M_P_GLOBAL_VOID: "a __global__ function must return void",
    M_P_MAIN_SPEC: "main takes no specifiers and no template",
    M_P_MAIN_SIG: "main must be declared as int main()",
    M_P_FOR_VAR: "the loop condition and increment must use the loop variable",
    M_P_PRINTF_FMT: "printf needs a literal format string",
    M_P_PRINTF_TEXT: "printf supports only literal text and %d",
    M_P_PRINTF_ONE: "printf supports at most one %d",
    M_P_PRINTF_COUNT: "printf argument count does not match the format",
    M_S_STRUCT_SPEC_MODE: "struct-level execution-space specifiers require --mode=proposal2",
    M_S_COND_SPEC_MODE: "conditional execution-space specifiers require --mode=proposal1",
    M_S_ASSERT_EVAL: "static assertion cannot be evaluated",
    M_S_ASSERT_FAIL: "static assertion failed",
    M_W_PRED_CONST: "specifier predicate is not a constant",
    M_W_LAUNCH_DEVICE: "a kernel launch is not allowed from device code",
    M_W_LAUNCH_NONGLOBAL: "only __global__ functions can be launched with <<< >>>",
    M_W_RECEIVER: "a member-call receiver must be a variable or a temporary",
    M_W_GLOBAL_CALL: "a __global__ function must be launched with <<< >>>, not called directly",
    M_X_CONTRACT: "input outside the analyser's contract (nesting/recursion bound)",
    M_P_DEPTH: "input outside the analyser's contract (nesting/recursion bound)",
}

EXPECT = [None, "enum", "class", "the HDC enum name", "{", ",", "enumerator 'Hst'",
          "enumerator 'Dev'", "enumerator 'HstDev'", "}", ";", "static_assert", "(", ")",
          "template", "<", ">", "requires", "a function body or ';'", "for", "int", "=", "++",
          ">>>"]
NAME_WHAT = [None, "template parameter name", "struct name", "member name", "function name",
             "parameter name", "type name", "template argument", "variable name", "loop variable"]
HDC_NAMES = [None, "Hst", "Dev", "HstDev"]
BUILTIN_TYPES = {1: "void", 2: "int", 3: "bool"}
ARITY = {31: ("release_assert", 1), 32: ("__trap", 0), 33: ("abort", 0), 34: ("cudaDeviceSynchronize", 0),
         0xFF: ("std::abort", 0)}
NODE_CLASS = {2: "StringLit", 7: "TempObj", 10: "CallExpr", 11: "MemberCallExpr", 12: "StaticCallExpr"}
SPAN_EOF = 0xFFFFFFFFFFFFFFFF
ARENA_BIT = 1 << 63

SF = ["", "{0} is not a template", "{0} does not name a type",
      "struct template arguments must be HDC constants", "expected an HDC constant",
      '"{0}" is not an HDC constant', '"{T}" has no members', '"{T}" has no member "{1}"',
      "cuda_arch is not usable in constant expressions", 'unbound name "{0}"',
      '"{0}" is a type, not a constant', "operand of ! is not a boolean",
      "comparison between unrelated kinds", "logical operands are not booleans",
      "not a constant expression: {C}", '"{T}" has no compatibility value', "substitution failure"]


class Renderer:
    """Turns records of one batch into message strings."""

    def __init__(self, data: bytes, offsets, arena: bytes, describe=None):
        self.data = data
        self.offsets = offsets
        self.arena = arena
        self.describe = describe  # callable(ids, kinds) -> desc records
        self._desc_cache = {}

    # -- text of spans -----------------------------------------------------
    def _spliced(self, p: int, lo: int, hi: int) -> bool:
        d = self.data
        c = d[p]
        if c == 0x5C:  # backslash
            e = p
            while e < hi and d[e] == 0x5C:
                e += 1
            need = e - p
            m = 0
            q = e
            while q < hi and m < need and d[q] == 0x0A:
                m += 1
                q += 1
            return m >= need
        if c == 0x0A:
            idx = 0
            q = p
            while q > lo and d[q - 1] == 0x0A:
                idx += 1
                q -= 1
            lb = 0
            while q > lo and d[q - 1] == 0x5C and lb <= idx:
                lb += 1
                q -= 1
            return idx < lb
        return False

    def file_bounds(self, pos: int):
        import bisect
        f = bisect.bisect_right(self.offsets, pos) - 1
        return int(self.offsets[f]), int(self.offsets[f + 1])

    def span_text(self, span: int) -> str:
        if span == SPAN_EOF:
            return None
        if span & ARENA_BIT:
            off = (span >> 32) & 0x7FFFFFFF
            ln = span & 0xFFFFFFFF
            if off == 0x7FFFFFFF:
                return "?"
            return self.arena[off: off + ln].decode("utf-8", "surrogateescape")
        pos = span >> 32
        ln = span & 0xFFFFFFFF
        raw = self.data[pos: pos + ln]
        if b"\\" in raw or b"\n" in raw:
            lo, hi = self.file_bounds(pos)
            raw = bytes(self.data[p] for p in range(pos, pos + ln)
                        if not (self.data[p] in (0x5C, 0x0A) and self._spliced(p, lo, hi)))
        return raw.decode("utf-8", "surrogateescape")

    def found(self, span: int) -> str:
        t = self.span_text(span)
        return "end of input" if t is None else t

    def type_name(self, arg: int) -> str:
        if (arg >> 32) == 0xFFFFFFFF:
            return BUILTIN_TYPES.get(arg & 0xFF, "?")
        return self.span_text(arg)

    def type_display(self, arg: int, targ: int) -> str:
        n = self.type_name(arg)
        return f"{n}<{HDC_NAMES[targ]}>" if targ else n

    def char_at(self, pos: int) -> str:
        b = self.data[pos: pos + 4]
        for k in range(1, 5):
            try:
                return b[:k].decode("utf-8")
            except UnicodeDecodeError:
                continue
        return chr(self.data[pos])

    # -- E1201 display (spacecheck.py:196-206) --------------------------------
    def display(self, ident: int, kind: int) -> str:
        key = (ident, kind)
        if key not in self._desc_cache:
            d = self.describe([ident], [kind])[0]
            self._desc_cache[key] = d
        d = self._desc_cache[key]
        name = self.span_text(int(d["name"]))
        base = f"{self.span_text(int(d['owner']))}::{name}" if d["owner"] else name
        if kind == 1:
            return base
        if d["otype"]:
            base = f"{self.type_display(int(d['otype']), int(d['otarg']))}::{name}"
        if d["nb"]:
            items = []
            for k in range(int(d["nb"])):
                bn = self.span_text(int(d["bname"][k]))
                if d["bkind"][k] == 1:
                    val = self.type_display(int(d["bval"][k]), int(d["bvx"][k]))
                else:
                    val = HDC_NAMES[int(d["bvx"][k])]
                items.append((bn, val))
            items.sort(key=lambda kv: kv[0])
            base = f"{base}<{', '.join(v for _, v in items)}>"
        return base

    # -- the message ------------------------------------------------------------
    def message(self, r) -> str:
        m = int(r["msg"])
        code = CODES[int(r["code"])]
        a0, a1, a2, a3 = int(r["a0"]), int(r["a1"]), int(r["a2"]), int(r["a3"])
        if m in FIXED:
            return FIXED[m]
        if m == M_PP_EXPECTS_ONE:
            return f"#{'ifndef' if a3 else 'ifdef'} expects exactly one macro name"
        if m == M_PP_UNKNOWN_MACRO:
            return f'unknown macro "{self.span_text(a0)}" in #{"ifndef" if a3 else "ifdef"}'
        if m == M_PP_ERROR:
            return f"#error: {self.span_text(a0) if a0 else ''}"
        if m == M_PP_UNKNOWN_DIRECTIVE:
            return f"unknown preprocessor directive #{self.span_text(a0) if a0 else ''}"
        if m == M_LEX_CHAR:
            return f"unexpected character {self.char_at(a0 >> 32)!r}"
        if m == M_P_EXPECTED:
            return f"expected {EXPECT[a0]!r}, found {self.found(a1)!r}"
        if m == M_P_EXPECTED_NAME:
            return f"expected {NAME_WHAT[a0]}, found {self.found(a1)!r}"
        if m == M_P_UNKNOWN_PRAGMA:
            return f"unknown pragma {self.span_text(a0)!r}"
        if m == M_P_SPEC_REJECT:
            return f"{self.span_text(a0)} is not recognized by this compiler profile"
        if m == M_P_SPEC_DUP:
            return f"duplicate specifier {self.span_text(a0)}"
        if m == M_P_ARITY:
            name, n = ARITY[a0]
            return f"{name} takes exactly {n} argument(s)"
        if m == M_P_HDC_VALUE:
            t = self.span_text(a0)
            return f"unknown HDC value {t if t is not None else ''!r}"
        if m == M_P_EXPR:
            return f"expected an expression, found {self.found(a0)!r}"
        if m == M_P_TARGS:
            return f"unexpected template arguments on {self.span_text(a0)!r}"
        if m == M_S_DUP:
            name = self.span_text(a0)
            if a1:
                name = f"{self.span_text(a1)}::{name}"
            return f'duplicate definition of "{name}"'
        if m == M_S_UNDEF_NAME:
            name = f"std::{self.span_text(a1)}" if a3 == 1 else self.span_text(a0)
            return f'undefined name "{name}"'
        if m == M_S_NO_TARGS_BUILTIN:
            return f"{BUILTIN_TYPES[a0]} takes no template arguments"
        if m == M_S_UNDEF_TYPE:
            return f'undefined type "{self.span_text(a0)}"'
        if m == M_S_MISSING_TARGS:
            return f'missing template arguments for "{self.span_text(a0)}"'
        if m == M_S_TOO_MANY_TARGS:
            return f'too many template arguments for "{self.span_text(a0)}"'
        if m == M_S_HDC_MEMBER:
            return f'member "hdc" of "{self.type_name(a0)}" is not an HDC constant'
        if m in (M_S_NO_VIABLE, M_S_AMBIGUOUS):
            name = self.span_text(a0)
            if a1:
                name = f"{self.type_display(a1, a3)}::{name}"
            if m == M_S_NO_VIABLE:
                return f'no viable candidate for call to "{name}"'
            return f'call to "{name}" is ambiguous ({a2} candidates survive)'
        if m == M_S_EMPTY_SPACES:
            name = self.span_text(a0)
            if a1:
                name = f"{self.span_text(a1)}::{name}"
            return (f'all execution-space predicates of "{name}" are false; '
                    "the instance has no execution space")
        if m == M_W_NOT_TYPE:
            return f'"{self.span_text(a0)}" does not name a type here'
        if m == M_W_NO_MEMBER:
            return f'type "{self.type_display(a0, a2)}" has no member "{self.span_text(a1)}"'
        if m == M_W_STRAY:
            return stray_text(code, a0, a1, a2)
        if m == M_W_E1201:
            return (f'the instantiation of "{self.display(a0, a3)}" must not depend on '
                    "whether __CUDA_ARCH__ is defined")
        if m == M_W_SUBST:
            sf = SF[a3]
            return sf.format(self.span_text(a0) if "{0}" in sf else "",
                             self.span_text(a1) if "{1}" in sf else "",
                             T=self.type_name(a0) if "{T}" in sf else "",
                             C=NODE_CLASS.get(a0, "?") if "{C}" in sf else "")
        return f"<message {m}>"


SIDE = {0: "host", 1: "device"}
CALLEE = {1: "host", 2: "device", 3: "host device"}


def stray_text(code: str, callee: int, side: int, from_hd: int) -> str:
    """spacecheck.py:146-176."""
    cw = CALLEE[callee]
    if code == "E1001":
        return "calling a device function from a host function is not allowed"
    if code == "E1002":
        return "calling a host function from a device function is not allowed"
    if code in ("W1101", "W1102"):
        return f"calling a {cw} function from a host device function is not allowed"
    if code == "E1101":
        return ("calling a host function from a host device function is not allowed; "
                "the device path is reachable from a kernel launch")
    if code == "E1102":
        return ("calling a device function from a host device function is not allowed; "
                "the host path is reachable from main")
    if code == "W1502":
        return f"calling a {cw} function from a host device function"
    if code == "E1501":
        if from_hd:
            return (f"stray call: calling a {cw} function from a host device function "
                    f"on a reachable {SIDE[side]} path")
        return f"stray call: calling a {cw} function from {SIDE[side]} code"
    raise ValueError(code)
