// exs_render.cuh -- K9: diagnostic message text on the GPU.
//
// Every ordered diagnostic record (template id + typed arguments, exs_common.cuh
// Msg) is rendered into the reference's exact message string, one thread per
// record, in two passes over the same code: a length pass (Out.p == nullptr),
// an exclusive scan of the lengths, and a write pass into one byte arena.
// Texts follow the reference's f-strings (preprocess.py:177-202, lexer.py:75,86,
// 116, parser.py, sema.py, spacecheck.py:146-176,306-572,760-763); `{x!r}` is
// Python's repr() of the argument, reproduced byte for byte (quote choice,
// backslash escapes, str.isprintable() from exs_unicode.cuh).  Arguments that
// are source spans are the logical text: bytes removed by backslash-newline
// splicing (the lexer's splice bitmap) are skipped.
//
// Then finish_diagnostics (diagnostics.py:116-121): records are already sorted
// by (file, line, col, code); inside a run of equal keys they are ordered by
// message text and exact (loc, code, message) duplicates are dropped.
#pragma once
#include "exs_stage_walk.cuh"

namespace exs {

#ifndef EXS_EMU
__device__ const u32 kNonPrintDev[EXS_NONPRINT_N] = {EXS_NONPRINT_TABLE};
#endif
static const u32 kNonPrintHost[EXS_NONPRINT_N] = {EXS_NONPRINT_TABLE};

// str.isprintable() of one code point
EXS_HD inline bool py_printable(u32 cp) {
  if (cp < 0x80) return cp >= 0x20 && cp != 0x7F;
#if defined(__CUDA_ARCH__) && !defined(EXS_EMU)
  const u32* t = kNonPrintDev;
#else
  const u32* t = kNonPrintHost;
#endif
  u32 lo = 0, hi = EXS_NONPRINT_N;  // number of transitions <= cp
  while (lo < hi) {
    u32 mid = (lo + hi) / 2;
    if (t[mid] <= cp) lo = mid + 1; else hi = mid;
  }
  return (lo & 1u) == 0;
}

#define RSPAN_EOF 0xFFFFFFFFFFFFFFFFull
#define RSPAN_ARENA (1ull << 63)

struct RenderCtx {
  const u8* src;       // batch bytes
  const u32* splice;   // bit p: byte p removed by splicing
  const u8* arena;     // lexer text arena (directive texts)
  const FnRec* fns;
  const RecRec* recs;
  const Node* nodes;
  const Tok* toks;
  const Inst* inst;
  u32 n_src;           // batch bytes (char_at reads at most 4, bounded here)
};

// message writer: counts when p is null
struct Out {
  char* p;
  u32 n;
  EXS_HD void c(char ch) { if (p) p[n] = ch; n++; }
  EXS_HD void s(const char* z) { while (*z) c(*z++); }
  EXS_HD void u(u64 v) {
    char b[24];
    int k = 0;
    do { b[k++] = (char)('0' + v % 10); v /= 10; } while (v);
    while (k) c(b[--k]);
  }
  EXS_HD void hex(u32 v, int digits) {
    for (int i = digits - 1; i >= 0; i--) c("0123456789abcdef"[(v >> (4 * i)) & 15]);
  }
};

// the logical bytes of a span (or of a C string)
struct Bytes {
  const u8* b;
  u32 p, end;
  const u32* splice;  // null: no splice skipping
  EXS_HD void skip() {
    if (splice) while (p < end && ((splice[p >> 5] >> (p & 31)) & 1u)) p++;
  }
  EXS_HD bool more() { skip(); return p < end; }
  EXS_HD u8 next() { skip(); return b[p++]; }
};

// Python's UTF-8 decoder with surrogateescape (Renderer.span_text's
// decode("utf-8", "surrogateescape")): a byte that does not start a complete,
// valid sequence becomes U+DC00 + byte
EXS_HD inline u32 next_cp(Bytes& it) {
  const u8 c = it.next();
  if (c < 0x80) return c;
  u32 need, cp;
  u8 lo = 0x80, hi = 0xBF;
  if (c >= 0xC2 && c <= 0xDF) { need = 1; cp = c & 0x1F; }
  else if (c >= 0xE0 && c <= 0xEF) {
    need = 2; cp = c & 0x0F;
    if (c == 0xE0) lo = 0xA0;
    if (c == 0xED) hi = 0x9F;
  } else if (c >= 0xF0 && c <= 0xF4) {
    need = 3; cp = c & 0x07;
    if (c == 0xF0) lo = 0x90;
    if (c == 0xF4) hi = 0x8F;
  } else {
    return 0xDC00u + c;
  }
  Bytes la = it;
  for (u32 k = 0; k < need; k++) {
    if (!la.more()) return 0xDC00u + c;
    const u8 d = la.next();
    if (d < (k == 0 ? lo : 0x80) || d > (k == 0 ? hi : 0xBF)) return 0xDC00u + c;
    cp = (cp << 6) | (d & 0x3F);
  }
  it = la;
  return cp;
}

EXS_HD inline void put_utf8(Out& o, u32 cp) {
  if (cp < 0x80) o.c((char)cp);
  else if (cp >= 0xDC80 && cp <= 0xDCFF) o.c((char)(cp - 0xDC00));  // surrogateescape round trip
  else if (cp < 0x800) { o.c((char)(0xC0 | (cp >> 6))); o.c((char)(0x80 | (cp & 0x3F))); }
  else if (cp < 0x10000) {
    o.c((char)(0xE0 | (cp >> 12))); o.c((char)(0x80 | ((cp >> 6) & 0x3F))); o.c((char)(0x80 | (cp & 0x3F)));
  } else {
    o.c((char)(0xF0 | (cp >> 18))); o.c((char)(0x80 | ((cp >> 12) & 0x3F)));
    o.c((char)(0x80 | ((cp >> 6) & 0x3F))); o.c((char)(0x80 | (cp & 0x3F)));
  }
}

// repr() of the text (CPython unicode_repr)
EXS_HD inline void put_repr(Out& o, Bytes it) {
  bool sq = false, dq = false;
  {
    Bytes s = it;
    while (s.more()) {
      const u8 c = s.next();
      sq |= c == '\'';
      dq |= c == '"';
    }
  }
  const char q = (sq && !dq) ? '"' : '\'';
  o.c(q);
  while (it.more()) {
    const u32 cp = next_cp(it);
    if (cp == (u32)q || cp == '\\') { o.c('\\'); o.c((char)cp); }
    else if (cp == '\t') o.s("\\t");
    else if (cp == '\n') o.s("\\n");
    else if (cp == '\r') o.s("\\r");
    else if (cp < 0x20 || cp == 0x7F) { o.s("\\x"); o.hex(cp, 2); }
    else if (cp < 0x7F) o.c((char)cp);
    else if (py_printable(cp)) put_utf8(o, cp);
    else if (cp <= 0xFF) { o.s("\\x"); o.hex(cp, 2); }
    else if (cp <= 0xFFFF) { o.s("\\u"); o.hex(cp, 4); }
    else { o.s("\\U"); o.hex(cp, 8); }
  }
  o.c(q);
}

EXS_HD inline Bytes cstr(const char* z) {
  u32 n = 0;
  while (z[n]) n++;
  return Bytes{(const u8*)z, 0, n, nullptr};
}

// Renderer.span_text: raw batch span (pos << 32 | len) or arena span (bit 63)
EXS_HD inline Bytes span_bytes(const RenderCtx& C, u64 span) {
  if (span & RSPAN_ARENA) {
    const u32 off = (u32)((span >> 32) & 0x7FFFFFFFu), ln = (u32)span;
    if (off == 0x7FFFFFFFu) return cstr("?");
    return Bytes{C.arena, off, off + ln, nullptr};
  }
  const u32 pos = (u32)(span >> 32), ln = (u32)span;
  return Bytes{C.src, pos, pos + ln, C.splice};
}
EXS_HD inline void put_bytes(Out& o, Bytes it) {
  while (it.more()) o.c((char)it.next());
}
EXS_HD inline void put_span(Out& o, const RenderCtx& C, u64 span) { put_bytes(o, span_bytes(C, span)); }

EXS_HD inline const char* builtin_type(u64 a) {
  const u32 k = (u32)(a & 0xFF);
  return k == 1 ? "void" : k == 2 ? "int" : k == 3 ? "bool" : "?";
}
EXS_HD inline const char* hdc_name(u32 t) { return t == 1 ? "Hst" : t == 2 ? "Dev" : t == 3 ? "HstDev" : "?"; }
// Renderer.type_name / type_display
EXS_HD inline void put_type(Out& o, const RenderCtx& C, u64 a, u32 targ) {
  if ((a >> 32) == 0xFFFFFFFFull) o.s(builtin_type(a));
  else put_span(o, C, a);
  if (targ) { o.c('<'); o.s(hdc_name(targ)); o.c('>'); }
}

EXS_HD inline u64 tok_span(const RenderCtx& C, u32 t) {
  return ((u64)C.toks[t].pos << 32) | (C.toks[t].end - C.toks[t].pos);
}
// logical-text order of two spans (binding names of one instance: identifiers)
EXS_HD inline int span_cmp(const RenderCtx& C, u64 x, u64 y) {
  Bytes a = span_bytes(C, x), b = span_bytes(C, y);
  while (true) {
    const bool ma = a.more(), mb = b.more();
    if (!ma || !mb) return ma ? 1 : (mb ? -1 : 0);
    const u8 ca = a.next(), cb = b.next();
    if (ca != cb) return ca < cb ? -1 : 1;
  }
}

// E1201 display name (spacecheck.py:196-206; Renderer.display over exs_describe)
EXS_HD inline void put_display(Out& o, const RenderCtx& C, u32 id, u32 kind) {
  const u32 fi = kind == 1 ? id : C.inst[id].fn;
  const FnRec& r = C.fns[fi];
  const u64 name = tok_span(C, C.nodes[r.node].tok);
  u64 owner = 0;
  if (r.flags & FR_OWNER) owner = tok_span(C, C.nodes[C.recs[r.rec].node].tok);
  if (kind == 1) {
    if (owner) { put_span(o, C, owner); o.s("::"); }
    put_span(o, C, name);
    return;
  }
  const Inst& I = C.inst[id];
  if (I.ot.k == V_TYPE && I.ot.targ && I.ot.rec != NONE) {
    put_type(o, C, tok_span(C, C.nodes[C.recs[I.ot.rec].node].tok), I.ot.targ);
    o.s("::");
  } else if (owner) {
    put_span(o, C, owner);
    o.s("::");
  }
  put_span(o, C, name);
  // bindings, sorted by parameter name
  u64 bn[2], bv[2];
  u8 bk[2], bx[2];
  u32 nb = 0;
  for (u32 tp = C.nodes[r.node].c0; tp != NONE && nb < 2; tp = C.nodes[tp].next) {
    const Val& v = C.nodes[tp].sub == 0 ? I.tb : I.hb;
    if (v.k == V_NONE) continue;
    bn[nb] = tok_span(C, C.nodes[tp].tok);
    if (v.k == V_TYPE) {
      bk[nb] = 1;
      bv[nb] = v.rec != NONE ? tok_span(C, C.nodes[C.recs[v.rec].node].tok) : (0xFFFFFFFF00000000ull | v.bt);
      bx[nb] = v.targ;
    } else {
      bk[nb] = 2; bv[nb] = 0; bx[nb] = (u8)v.x;
    }
    nb++;
  }
  if (!nb) return;
  u32 ord[2] = {0, 1};
  if (nb == 2 && span_cmp(C, bn[1], bn[0]) < 0) { ord[0] = 1; ord[1] = 0; }
  o.c('<');
  for (u32 k = 0; k < nb; k++) {
    const u32 j = ord[k];
    if (k) o.s(", ");
    if (bk[j] == 1) put_type(o, C, bv[j], bx[j]);
    else o.s(hdc_name(bx[j]));
  }
  o.c('>');
}

// spacecheck.py:146-176
EXS_HD inline void put_stray(Out& o, u16 code, u64 callee, u64 side, u64 from_hd) {
  const char* cw = callee == 1 ? "host" : callee == 2 ? "device" : "host device";
  switch (code) {
    case C_E1001: o.s("calling a device function from a host function is not allowed"); return;
    case C_E1002: o.s("calling a host function from a device function is not allowed"); return;
    case C_W1101:
    case C_W1102: o.s("calling a "); o.s(cw); o.s(" function from a host device function is not allowed"); return;
    case C_E1101:
      o.s("calling a host function from a host device function is not allowed; "
          "the device path is reachable from a kernel launch");
      return;
    case C_E1102:
      o.s("calling a device function from a host device function is not allowed; "
          "the host path is reachable from main");
      return;
    case C_W1502: o.s("calling a "); o.s(cw); o.s(" function from a host device function"); return;
    case C_E1501:
      o.s("stray call: calling a "); o.s(cw);
      if (from_hd) { o.s(" function from a host device function on a reachable "); o.s(side ? "device" : "host"); o.s(" path"); }
      else { o.s(" function from "); o.s(side ? "device" : "host"); o.s(" code"); }
      return;
    default: o.s("?"); return;
  }
}

EXS_HD inline const char* fixed_text(u16 m) {
  switch (m) {
    case M_PP_ELSE_NOMATCH: return "#else without matching #ifdef/#ifndef";
    case M_PP_SECOND_ELSE: return "second #else in one conditional";
    case M_PP_ENDIF_NOMATCH: return "#endif without matching #ifdef/#ifndef";
    case M_PP_UNTERMINATED: return "unterminated #ifdef/#ifndef";
    case M_LEX_PRAGMA: return "malformed #pragma directive";
    case M_LEX_STRING: return "unterminated string literal";
    case M_P_PRAGMA_FN: return "a pragma must precede a function";
    case M_P_REQ_STRUCT: return "a requires clause cannot constrain a struct";
    case M_P_TPARAM_KIND: return "expected 'typename' or 'HDC' template parameter";
    case M_P_TPARAM_LIMIT: return "at most one type parameter and one HDC parameter are supported";
    case M_P_GLOBAL_EXCL: return "__global__ excludes __host__ and __device__";
    case M_P_STRUCT_SPEC: return "invalid specifier on a struct";
    case M_P_STRUCT_TPARAM: return "struct templates support only HDC parameters";
    case M_P_MEMBER_GLOBAL:
    case M_P_GLOBAL_MEMBER: return "__global__ is not allowed on member functions";
    case M_P_MCONST_DECL: return "invalid declaration of a member constant";
    case M_P_MCONST_TYPE: return "member constants must have type HDC, bool, or int";
    case M_P_MCONST_STATIC: return "member constants must be static constexpr";
    case M_P_MCONST_SPEC: return "invalid specifier on a member constant";
    case M_P_REQ_TEMPLATE: return "a requires clause needs a template header";
    case M_P_GLOBAL_VOID: return "a __global__ function must return void";
    case M_P_MAIN_SPEC: return "main takes no specifiers and no template";
    case M_P_MAIN_SIG: return "main must be declared as int main()";
    case M_P_FOR_VAR: return "the loop condition and increment must use the loop variable";
    case M_P_PRINTF_FMT: return "printf needs a literal format string";
    case M_P_PRINTF_TEXT: return "printf supports only literal text and %d";
    case M_P_PRINTF_ONE: return "printf supports at most one %d";
    case M_P_PRINTF_COUNT: return "printf argument count does not match the format";
    case M_S_STRUCT_SPEC_MODE: return "struct-level execution-space specifiers require --mode=proposal2";
    case M_S_COND_SPEC_MODE: return "conditional execution-space specifiers require --mode=proposal1";
    case M_S_ASSERT_EVAL: return "static assertion cannot be evaluated";
    case M_S_ASSERT_FAIL: return "static assertion failed";
    case M_W_PRED_CONST: return "specifier predicate is not a constant";
    case M_W_LAUNCH_DEVICE: return "a kernel launch is not allowed from device code";
    case M_W_LAUNCH_NONGLOBAL: return "only __global__ functions can be launched with <<< >>>";
    case M_W_RECEIVER: return "a member-call receiver must be a variable or a temporary";
    case M_W_GLOBAL_CALL: return "a __global__ function must be launched with <<< >>>, not called directly";
    case M_X_CONTRACT:
    case M_P_DEPTH: return "input outside the analyser's contract (nesting/recursion bound)";
    default: return nullptr;
  }
}

// parser.py expect() descriptions and expect_ident() "what" texts
EXS_HD inline const char* expect_text(u64 k) {
  switch (k) {
    case 1: return "enum"; case 2: return "class"; case 3: return "the HDC enum name";
    case 4: return "{"; case 5: return ","; case 6: return "enumerator 'Hst'";
    case 7: return "enumerator 'Dev'"; case 8: return "enumerator 'HstDev'"; case 9: return "}";
    case 10: return ";"; case 11: return "static_assert"; case 12: return "("; case 13: return ")";
    case 14: return "template"; case 15: return "<"; case 16: return ">"; case 17: return "requires";
    case 18: return "a function body or ';'"; case 19: return "for"; case 20: return "int";
    case 21: return "="; case 22: return "++"; case 23: return ">>>";
    default: return "?";
  }
}
EXS_HD inline const char* name_what(u64 k) {
  switch (k) {
    case 1: return "template parameter name"; case 2: return "struct name"; case 3: return "member name";
    case 4: return "function name"; case 5: return "parameter name"; case 6: return "type name";
    case 7: return "template argument"; case 8: return "variable name"; case 9: return "loop variable";
    default: return "?";
  }
}

// Renderer.found: the span's text, "end of input" at EOF -- repr'd
EXS_HD inline void put_found_repr(Out& o, const RenderCtx& C, u64 span) {
  put_repr(o, span == RSPAN_EOF ? cstr("end of input") : span_bytes(C, span));
}

// Renderer.char_at: the first 1..4 bytes at pos that decode strictly, else
// the byte as a Latin-1 character -- repr'd
EXS_HD inline void put_char_repr(Out& o, const RenderCtx& C, u32 pos) {
  Bytes it{C.src, pos, pos + 4 < C.n_src ? pos + 4 : C.n_src, nullptr};
  const u8 c = C.src[pos];
  u32 cp;
  Bytes la = it;
  cp = next_cp(la);
  const bool strict_ok = !(cp >= 0xDC80 && cp <= 0xDCFF && c >= 0x80);
  if (!strict_ok) cp = c;  // chr(byte)
  // repr of one code point
  const char q = cp == '\'' ? '"' : '\'';
  o.c(q);
  if (cp == (u32)q || cp == '\\') { o.c('\\'); o.c((char)cp); }
  else if (cp == '\t') o.s("\\t");
  else if (cp == '\n') o.s("\\n");
  else if (cp == '\r') o.s("\\r");
  else if (cp < 0x20 || cp == 0x7F) { o.s("\\x"); o.hex(cp, 2); }
  else if (cp < 0x7F) o.c((char)cp);
  else if (py_printable(cp)) put_utf8(o, cp);
  else if (cp <= 0xFF) { o.s("\\x"); o.hex(cp, 2); }
  else if (cp <= 0xFFFF) { o.s("\\u"); o.hex(cp, 4); }
  else { o.s("\\U"); o.hex(cp, 8); }
  o.c(q);
}

// Renderer.message (messages.py) for one record
EXS_HD inline void render_message(const RenderCtx& C, const Diag& d, Out& o) {
  const u16 m = d.msg;
  const u64 a0 = d.a0, a1 = d.a1, a2 = d.a2;
  const u32 a3 = d.a3;
  const char* fx = fixed_text(m);
  if (fx) { o.s(fx); return; }
  switch (m) {
    case M_PP_EXPECTS_ONE: o.c('#'); o.s(a3 ? "ifndef" : "ifdef"); o.s(" expects exactly one macro name"); return;
    case M_PP_UNKNOWN_MACRO:
      o.s("unknown macro \""); put_span(o, C, a0); o.s("\" in #"); o.s(a3 ? "ifndef" : "ifdef"); return;
    case M_PP_ERROR: o.s("#error: "); if (a0) put_span(o, C, a0); return;
    case M_PP_UNKNOWN_DIRECTIVE: o.s("unknown preprocessor directive #"); if (a0) put_span(o, C, a0); return;
    case M_LEX_CHAR: o.s("unexpected character "); put_char_repr(o, C, (u32)(a0 >> 32)); return;
    case M_P_EXPECTED:
      o.s("expected "); put_repr(o, cstr(expect_text(a0))); o.s(", found "); put_found_repr(o, C, a1); return;
    case M_P_EXPECTED_NAME:
      o.s("expected "); o.s(name_what(a0)); o.s(", found "); put_found_repr(o, C, a1); return;
    case M_P_UNKNOWN_PRAGMA: o.s("unknown pragma "); put_repr(o, span_bytes(C, a0)); return;
    case M_P_SPEC_REJECT: put_span(o, C, a0); o.s(" is not recognized by this compiler profile"); return;
    case M_P_SPEC_DUP: o.s("duplicate specifier "); put_span(o, C, a0); return;
    case M_P_ARITY: {
      const char* nm = a0 == 31 ? "release_assert" : a0 == 32 ? "__trap" : a0 == 33 ? "abort"
                       : a0 == 34 ? "cudaDeviceSynchronize" : a0 == 0xFF ? "std::abort" : "?";
      o.s(nm); o.s(" takes exactly "); o.u(a0 == 31 ? 1 : 0); o.s(" argument(s)");
      return;
    }
    case M_P_HDC_VALUE:
      o.s("unknown HDC value "); put_repr(o, a0 == RSPAN_EOF ? cstr("") : span_bytes(C, a0)); return;
    case M_P_EXPR: o.s("expected an expression, found "); put_found_repr(o, C, a0); return;
    case M_P_TARGS: o.s("unexpected template arguments on "); put_repr(o, span_bytes(C, a0)); return;
    case M_S_DUP:
      o.s("duplicate definition of \"");
      if (a1) { put_span(o, C, a1); o.s("::"); }
      put_span(o, C, a0); o.c('"');
      return;
    case M_S_UNDEF_NAME:
      o.s("undefined name \"");
      if (a3 == 1) { o.s("std::"); put_span(o, C, a1); }
      else put_span(o, C, a0);
      o.c('"');
      return;
    case M_S_NO_TARGS_BUILTIN: o.s(builtin_type(a0)); o.s(" takes no template arguments"); return;
    case M_S_UNDEF_TYPE: o.s("undefined type \""); put_span(o, C, a0); o.c('"'); return;
    case M_S_MISSING_TARGS: o.s("missing template arguments for \""); put_span(o, C, a0); o.c('"'); return;
    case M_S_TOO_MANY_TARGS: o.s("too many template arguments for \""); put_span(o, C, a0); o.c('"'); return;
    case M_S_HDC_MEMBER: o.s("member \"hdc\" of \""); put_type(o, C, a0, 0); o.s("\" is not an HDC constant"); return;
    case M_S_NO_VIABLE:
    case M_S_AMBIGUOUS:
      o.s(m == M_S_NO_VIABLE ? "no viable candidate for call to \"" : "call to \"");
      if (a1) { put_type(o, C, a1, a3); o.s("::"); }
      put_span(o, C, a0);
      if (m == M_S_NO_VIABLE) o.c('"');
      else { o.s("\" is ambiguous ("); o.u(a2); o.s(" candidates survive)"); }
      return;
    case M_S_EMPTY_SPACES:
      o.s("all execution-space predicates of \"");
      if (a1) { put_span(o, C, a1); o.s("::"); }
      put_span(o, C, a0);
      o.s("\" are false; the instance has no execution space");
      return;
    case M_W_NOT_TYPE: o.c('"'); put_span(o, C, a0); o.s("\" does not name a type here"); return;
    case M_W_NO_MEMBER:
      o.s("type \""); put_type(o, C, a0, (u32)a2); o.s("\" has no member \""); put_span(o, C, a1); o.c('"'); return;
    case M_W_STRAY: put_stray(o, d.code, a0, a1, a2); return;
    case M_W_E1201:
      o.s("the instantiation of \""); put_display(o, C, (u32)a0, a3);
      o.s("\" must not depend on whether __CUDA_ARCH__ is defined");
      return;
    case M_W_SUBST:
      switch (a3) {
        case SF_NOT_TEMPLATE: put_span(o, C, a0); o.s(" is not a template"); return;
        case SF_NOT_TYPE_NAME: put_span(o, C, a0); o.s(" does not name a type"); return;
        case SF_STRUCT_TARGS_HDC: o.s("struct template arguments must be HDC constants"); return;
        case SF_EXPECTED_HDC: o.s("expected an HDC constant"); return;
        case SF_NOT_HDC_CONST: o.c('"'); put_span(o, C, a0); o.s("\" is not an HDC constant"); return;
        case SF_NO_MEMBERS: o.c('"'); put_type(o, C, a0, 0); o.s("\" has no members"); return;
        case SF_NO_MEMBER:
          o.c('"'); put_type(o, C, a0, 0); o.s("\" has no member \""); put_span(o, C, a1); o.c('"'); return;
        case SF_ARCH: o.s("cuda_arch is not usable in constant expressions"); return;
        case SF_UNBOUND: o.s("unbound name \""); put_span(o, C, a0); o.c('"'); return;
        case SF_IS_TYPE: o.c('"'); put_span(o, C, a0); o.s("\" is a type, not a constant"); return;
        case SF_NOT_BOOL_OPERAND: o.s("operand of ! is not a boolean"); return;
        case SF_UNRELATED: o.s("comparison between unrelated kinds"); return;
        case SF_LOGICAL: o.s("logical operands are not booleans"); return;
        case SF_NOT_CONST: {
          o.s("not a constant expression: ");
          o.s(a0 == 2 ? "StringLit" : a0 == 7 ? "TempObj" : a0 == 10 ? "CallExpr" : a0 == 11 ? "MemberCallExpr"
              : a0 == 12 ? "StaticCallExpr" : "?");
          return;
        }
        case SF_NO_COMPAT: o.c('"'); put_type(o, C, a0, 0); o.s("\" has no compatibility value"); return;
        case SF_OTHER: o.s("substitution failure"); return;
        default: return;
      }
    default:
      o.s("<message "); o.u(m); o.c('>');
      return;
  }
}

// -- byte comparison of two rendered messages (str order = code-point order =
// UTF-8 byte order; a surrogate-escaped byte 0x80..0xFF decodes to U+DC80..
// U+DCFF, which sorts below U+E000.. but above U+0800..U+D7FF, unlike the raw
// byte -- such messages only come from invalid UTF-8 input)
EXS_HD inline int msg_cmp(const char* a, u32 na, const char* b, u32 nb) {
  const u32 n = na < nb ? na : nb;
  for (u32 i = 0; i < n; i++)
    if (a[i] != b[i]) return (u8)a[i] < (u8)b[i] ? -1 : 1;
  return na < nb ? -1 : (na > nb ? 1 : 0);
}

}  // namespace exs

namespace exs {

// Messages without a text argument are the bulk of a corpus's diagnostics
// (the stray-call texts).  They are rendered once per handle into a static
// section at the start of the text arena and referenced from there.
#define EXS_STATIC_KEYS 320
EXS_HD inline int static_key(const Diag& d) {
  if (fixed_text(d.msg)) return d.msg;  // < 70
  if (d.msg == M_PP_EXPECTS_ONE) return 70 + (d.a3 ? 1 : 0);
  if (d.msg == M_W_STRAY && d.code >= C_E1001 && d.code <= C_W1502 && d.a0 >= 1 && d.a0 <= 3 && d.a1 <= 1 &&
      d.a2 <= 1)
    return 128 + (int)(((d.code - C_E1001) * 3 + (d.a0 - 1)) * 4 + d.a1 * 2 + d.a2);
  return -1;
}
// a record that renders the static message `key` (inverse of static_key)
inline bool static_diag(int key, Diag& d) {
  memset(&d, 0, sizeof d);
  if (key < 70) { d.msg = (u16)key; return fixed_text(d.msg) != nullptr; }
  if (key < 72) { d.msg = M_PP_EXPECTS_ONE; d.a3 = (u32)(key - 70); return true; }
  if (key < 128) return false;
  int x = key - 128;
  d.msg = M_W_STRAY;
  d.a2 = x & 1; d.a1 = (x >> 1) & 1; x >>= 2;
  d.a0 = (u64)(x % 3 + 1); x /= 3;
  d.code = (u16)(C_E1001 + x);
  return d.code <= C_W1502;
}

}  // namespace exs
