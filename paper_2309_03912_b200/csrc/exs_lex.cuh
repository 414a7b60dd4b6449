// exs_lex.cuh -- K1..K3: byte-parallel splice map, logical-line scanner,
// directive parser and tokenizer (reference: syntax/preprocess.py:81-203,
// syntax/lexer.py:46-118).
//
// Layout in HBM (one batch = concatenated files):
//   src[N]          corpus bytes
//   fstart[N/32+1]  bit p set iff p is a file start
//   splice[N/32+1]  bit p set iff byte p is removed by backslash-newline
//                   splicing (preprocess.py:81-95: the last min(k,m) bytes of
//                   a k-backslash run and the first min(k,m) of the m-newline
//                   run that follows it)
//   line_start[L]   logical line starts (file start, or after a non-spliced \n)
// A logical line is processed by one thread (the reference's line loop,
// preprocess.py:163); the comment DFA state at a line start is CODE or BLOCK,
// so lines compose as {CODE,BLOCK}->{CODE,BLOCK} maps under a scan.
#pragma once
#include "exs_common.cuh"
#include "exs_unicode.cuh"

namespace exs {

EXS_HD inline bool bit_get(const u32* b, u32 p) { return (b[p >> 5] >> (p & 31)) & 1u; }

// comment DFA (same formulation as oracle/exs_oracle.py:_step)
enum { S_CODE = 0, S_SLASH, S_STR, S_LINE, S_BLOCK, S_STAR };

EXS_HD inline u8 dfa_step(u8 s, u8 c) {
  if (s == S_SLASH) {
    if (c == '/') return S_LINE;
    if (c == '*') return S_BLOCK;
    s = S_CODE;
  }
  switch (s) {
    case S_CODE: return c == '"' ? S_STR : (c == '/' ? S_SLASH : S_CODE);
    case S_STR: return (c == '"' || c == '\n') ? S_CODE : S_STR;
    case S_LINE: return c == '\n' ? S_CODE : S_LINE;
    case S_BLOCK: return c == '*' ? S_STAR : S_BLOCK;
    default: return c == '/' ? S_CODE : (c == '*' ? S_STAR : S_BLOCK);
  }
}

struct SrcView {
  const u8* src;
  const u32* splice;
  const u32* fstart;
  u32 n;
};

// Is the byte at p removed by splicing?  (p must hold '\\' or '\n')
EXS_HD inline bool compute_spliced(const SrcView& v, u32 p) {
  const u8* s = v.src;
  if (s[p] == '\\') {
    u32 e = p;
    while (e < v.n && s[e] == '\\' && (e == p || !bit_get(v.fstart, e))) e++;
    u32 need = e - p, m = 0;
    u32 q = e;
    while (q < v.n && m < need && s[q] == '\n' && !bit_get(v.fstart, q)) { m++; q++; }
    return m >= need;
  }
  if (s[p] == '\n') {
    u32 idx = 0, q = p;
    while (!bit_get(v.fstart, q) && q > 0 && s[q - 1] == '\n') { idx++; q--; }
    // q = newline run start; count backslashes before it (need idx+1)
    u32 lb = 0;
    while (!bit_get(v.fstart, q) && q > 0 && s[q - 1] == '\\' && lb <= idx) { lb++; q--; }
    return idx < lb;
  }
  return false;
}

// Iterator over the comment-blanked logical characters of one logical line
// (preprocess.py:98-145 applied after splicing).  Yields (char, raw pos, width);
// width is 0 for UTF-8 continuation bytes so columns count code points.
struct Blanker {
  const u8* src;
  const u32* splice;
  u32 p, hi;   // next raw position, logical line end (terminator or file end)
  u8 st;       // S_CODE / S_STR / S_LINE / S_BLOCK  (S_SLASH/S_STAR never stored)
  u8 pend;     // a second blank of a 2-char comment token is pending
  u32 pend_pos;

  bool nospl;  // no spliced byte in [lo, hi): skip the bitmap on every character

  EXS_HD void init(const u8* s, const u32* sp, u32 lo, u32 hi_, u8 start_state) {
    src = s; splice = sp; p = lo; hi = hi_; st = start_state; pend = 0; pend_pos = 0;
    u32 any = 0;
    if (hi > lo) {
      u32 w0 = lo >> 5, w1 = (hi - 1) >> 5;
      for (u32 w = w0; w <= w1 && !any; w++) {
        u32 m = sp[w];
        if (w == w0) m &= ~0u << (lo & 31);
        if (w == w1) m &= (~0u) >> (31 - ((hi - 1) & 31));
        any |= m;
      }
    }
    nospl = any == 0;
  }
  EXS_HD u32 next_logical(u32 q) const {
    if (nospl) return q < hi ? q : hi;
    while (q < hi && bit_get(splice, q)) q++;
    return q;
  }
  // returns false at line end
  EXS_HD bool next(u8& c, u32& pos, u8& width) {
    if (pend) {
      pend = 0; c = ' '; pos = pend_pos; width = 1;
      return true;
    }
    u32 q = next_logical(p);
    if (q >= hi) { p = q; return false; }
    u8 ch = src[q];
    u32 q2 = next_logical(q + 1);
    u8 nx = q2 < hi ? src[q2] : 0;   // '\n' never appears inside a logical line
    width = is_cont_byte(ch) ? 0 : 1;
    pos = q;
    p = q + 1;
    switch (st) {
      case S_BLOCK:
        if (ch == '*' && nx == '/') {
          c = ' '; pend = 1; pend_pos = q2; p = q2 + 1; st = S_CODE;
        } else {
          c = ' ';
        }
        return true;
      case S_LINE:
        c = ' ';
        return true;
      case S_STR:
        c = ch;
        if (ch == '"') st = S_CODE;
        return true;
      default:
        if (ch == '"') { st = S_STR; c = ch; return true; }
        if (ch == '/' && nx == '/') { c = ' '; pend = 1; pend_pos = q2; p = q2 + 1; st = S_LINE; return true; }
        if (ch == '/' && nx == '*') { c = ' '; pend = 1; pend_pos = q2; p = q2 + 1; st = S_BLOCK; return true; }
        c = ch;
        return true;
    }
  }
  // comment state after the line terminator ('\n' resets STR and LINE)
  EXS_HD u8 end_state() const { return st == S_BLOCK ? S_BLOCK : S_CODE; }
};

// Run the blanker from CODE and from BLOCK; return 2-bit map (bit0: end from
// CODE is BLOCK, bit1: end from BLOCK is BLOCK).
EXS_HD inline u8 line_fsm_map(const u8* s, const u32* sp, u32 lo, u32 hi) {
  u8 r = 0;
  for (int k = 0; k < 2; k++) {
    Blanker b;
    b.init(s, sp, lo, hi, k ? S_BLOCK : S_CODE);
    u8 c, w; u32 pos;
    while (b.next(c, pos, w)) {}
    if (b.end_state() == S_BLOCK) r |= (1u << k);
  }
  return r;
}

// ---------------------------------------------------------------------------
// vocabulary (exs_common.cuh Word) -- matched on logical token text

#define EXS_VOCAB_TEXT                                                                   \
  "struct\0class\0enum\0template\0typename\0requires\0return\0if\0else\0for\0void\0int\0" \
  "bool\0true\0false\0constexpr\0static\0static_assert\0HDC\0__host__\0__device__\0"      \
  "__global__\0main\0cuda_arch\0hdc\0std\0Hst\0Dev\0HstDev\0printf\0release_assert\0"    \
  "__trap\0abort\0cudaDeviceSynchronize\0hd_warning_disable\0nv_exec_check_disable\0!\0(\0"
#ifndef EXS_EMU
__constant__ char kVocabDev[] = EXS_VOCAB_TEXT;
#endif
static const char kVocabHost[] = EXS_VOCAB_TEXT;

constexpr u32 len_c(const char* s) { return *s ? 1 + len_c(s + 1) : 0; }
// Vocabulary id from the token's text hash and length: a perfect hash over
// the 38 words (multiplier found offline: slot = (hv * K) >> 57, collision-
// free) -- one table load, no divergent compare tree.
struct VEnt { u64 hv; u32 len; u32 id; };
struct VTable { VEnt e[128]; };
constexpr u64 kVocabK = 0x83595d744d2f1383ull;  // tests/emu/vocab_k.py
EXS_HD constexpr u32 vocab_slot(u64 hv) { return (u32)((hv * kVocabK) >> 57); }
constexpr VTable make_vtable() {
  VTable t{};
  const char* ws[] = {"struct", "class", "enum", "template", "typename", "requires", "return", "if",
                      "else", "for", "void", "int", "bool", "true", "false", "constexpr", "static",
                      "static_assert", "HDC", "__host__", "__device__", "__global__", "main",
                      "cuda_arch", "hdc", "std", "Hst", "Dev", "HstDev", "printf", "release_assert",
                      "__trap", "abort", "cudaDeviceSynchronize", "hd_warning_disable",
                      "nv_exec_check_disable", "!", "("};
  const u8 ids[] = {W_STRUCT, W_CLASS, W_ENUM, W_TEMPLATE, W_TYPENAME, W_REQUIRES, W_RETURN, W_IF,
                    W_ELSE, W_FOR, W_VOID, W_INT, W_BOOL, W_TRUE, W_FALSE, W_CONSTEXPR, W_STATIC,
                    W_STATIC_ASSERT, W_HDC, W_HOST, W_DEVICE, W_GLOBAL, W_MAIN, W_CUDA_ARCH,
                    W_HDC_TRAIT, W_STD, W_HST, W_DEV, W_HSTDEV, W_PRINTF, W_RELEASE_ASSERT, W_TRAP,
                    W_ABORT, W_CUDASYNC, W_HD_WARNING_DISABLE, W_NV_EXEC_CHECK_DISABLE, W_BANG_STR,
                    W_LPAREN_STR};
  for (u32 i = 0; i < sizeof(ids); i++) {
    const u64 h = name_hash_c(ws[i]);
    t.e[vocab_slot(h)] = VEnt{h, len_c(ws[i]), ids[i]};
  }
  return t;
}
constexpr u32 vtable_fill() {
  VTable t = make_vtable();
  u32 n = 0;
  for (u32 i = 0; i < 128; i++) n += t.e[i].len != 0;
  return n;
}
static_assert(vtable_fill() == W_COUNT - 1, "vocabulary perfect hash: collision or missing word");
#ifndef EXS_EMU
__device__ const VTable kVTabDev = make_vtable();
#endif
static constexpr VTable kVTabHost = make_vtable();

EXS_HD inline u8 vocab_hash(u64 hv, u32 len) {
  // body-only __CUDA_ARCH__ switch, never in a signature
#if defined(__CUDA_ARCH__) && !defined(EXS_EMU)
  const VEnt& e = kVTabDev.e[vocab_slot(hv)];
#else
  const VEnt& e = kVTabHost.e[vocab_slot(hv)];
#endif
  return (e.hv == hv && e.len == len) ? (u8)e.id : (u8)W_NONE;
}

EXS_HD inline u8 vocab_lookup(const u8* t, u32 len) {
  if (len == 0 || len > 24) return W_NONE;
  // body-only __CUDA_ARCH__ switch, never in a signature
#if defined(__CUDA_ARCH__) && !defined(EXS_EMU)
  const char* v = kVocabDev;
#else
  const char* v = kVocabHost;
#endif
  for (u8 id = 1; id < W_COUNT; id++) {
    u32 l = 0;
    while (v[l]) l++;
    if (l == len) {
      bool eq = true;
      for (u32 i = 0; i < len; i++)
        if ((u8)v[i] != t[i]) { eq = false; break; }
      if (eq) return id;
    }
    v += l + 1;
  }
  return W_NONE;
}

// ---------------------------------------------------------------------------
// Unicode classes of Python's str predicates (exs_unicode.cuh, generated)

enum { UC_ALPHA = 1, UC_DIGIT = 2, UC_ALNUM = 4, UC_DECIMAL = 8, UC_SPACE = 16 };
#ifndef EXS_EMU
__device__ const u32 kUclsDev[EXS_UCLS_N] = {EXS_UCLS_TABLE};
#endif
static const u32 kUclsHost[EXS_UCLS_N] = {EXS_UCLS_TABLE};

struct UClass { u8 cls; u32 start; };  // class bits, start of its run

EXS_HD inline UClass uclass(u32 cp) {
  if (cp < 0x80) {
    u8 c = (u8)cp, k = 0;
    if (is_alpha(c)) k = UC_ALPHA | UC_ALNUM;
    else if (is_digit(c)) k = UC_DIGIT | UC_ALNUM | UC_DECIMAL;
    else if (is_pyspace(c)) k = UC_SPACE;
    return UClass{k, is_digit(c) ? (u32)'0' : cp};
  }
#if defined(__CUDA_ARCH__) && !defined(EXS_EMU)
  const u32* t = kUclsDev;
#else
  const u32* t = kUclsHost;
#endif
  u32 lo = 0, hi = EXS_UCLS_N;  // last entry with start <= cp
  while (hi - lo > 1) {
    u32 mid = (lo + hi) / 2;
    if ((t[mid] >> 8) <= cp) lo = mid; else hi = mid;
  }
  return UClass{(u8)(t[lo] & 0xFF), t[lo] >> 8};
}

// code point of the UTF-8 sequence whose lead byte is at p (no splice can fall
// inside a code point of valid UTF-8)
EXS_HD inline u32 utf8_at(const u8* s, u32 p, u32 lim) {
  u8 c = s[p];
  if (c < 0xC0) return c;
  u32 n = c >= 0xF0 ? 3 : (c >= 0xE0 ? 2 : 1);
  u32 cp = c & (0x3Fu >> n);
  for (u32 k = 1; k <= n && p + k < lim; k++) cp = (cp << 6) | (s[p + k] & 0x3Fu);
  return cp;
}

// class of the (blanked) character c yielded at raw position pos
EXS_HD inline u8 char_class(const u8* s, u8 c, u32 pos, u32 lim) {
  if (c < 0x80) return uclass(c).cls;
  return uclass(utf8_at(s, pos, lim)).cls;
}

// directive kinds (per logical line)
enum {
  LK_NORMAL = 0, LK_PRAGMA_DIR, LK_IFDEF, LK_IFNDEF, LK_ELSE, LK_ENDIF, LK_ERROR,
  LK_UNKNOWN, LK_BAD_ARITY, LK_BAD_MACRO,
};
enum { MAC_CUDACC = 1, MAC_CUDA_ARCH = 2, MAC_RELAXED = 4 };

struct LineInfo {
  u8 kind;      // LK_*
  u8 macro;     // MAC_* for ifdef/ifndef
  u8 has_splice;
  u8 is_ifndef; // for LK_BAD_ARITY / LK_BAD_MACRO: which directive
  u32 cps;      // code points of the logical line (for the EOF column)
  u64 span;     // text-arena span (offset<<32 | len) for messages
};

EXS_HD inline bool text_eq(const u8* a, u32 la, const char* b) {
  u32 lb = 0;
  while (b[lb]) lb++;
  if (la != lb) return false;
  for (u32 i = 0; i < la; i++)
    if (a[i] != (u8)b[i]) return false;
  return true;
}

// Directive detection and parsing for one logical line (preprocess.py:163-200).
// Writes message text (if any) into the arena.
EXS_HD inline LineInfo scan_line_directive(const u8* s, const u32* sp, u32 lo, u32 hi, u8 st,
                                           u8* arena, u32* arena_top, u32 arena_cap) {
  LineInfo li;
  li.kind = LK_NORMAL; li.macro = 0; li.has_splice = 0; li.is_ifndef = 0; li.cps = 0; li.span = 0;
  Blanker b;
  b.init(s, sp, lo, hi, st);
  u8 c, w; u32 pos;
  // pass 1: first non-space char, code points
  bool seen = false, directive = false;
  u32 hash_pos = 0;
  bool ws = false;  // str.isspace of the current code point (continuation bytes inherit it)
  while (b.next(c, pos, w)) {
    li.cps += w;
    if (w) ws = (char_class(s, c, pos, hi) & UC_SPACE) != 0;
    if (!seen && !ws) {
      seen = true;
      if (c == '#') { directive = true; hash_pos = pos; }
    }
  }
  for (u32 q = lo; q < hi; q++)
    if (bit_get(sp, q)) { li.has_splice = 1; break; }
  if (!directive) return li;
  // pass 2: words after '#': name = first run of non-space chars; rest = stripped remainder
  b.init(s, sp, lo, hi, st);
  while (b.next(c, pos, w) && pos != hash_pos) {}
  u8 name[16]; u32 nlen = 0;
  u8 rest[32]; u32 rlen = 0;       // first 32 chars of rest (for macro compare)
  u32 rest_first = NONE, rest_last_end = 0;  // positions in blanked-char order
  bool rest_has_inner_space = false;
  int phase = 0;  // 0 before name, 1 in name, 2 after name, 3 in rest
  u32 idx = 0, rest_start_idx = 0, rest_end_idx = 0, name_start_idx = 0, name_end_idx = 0;
  bool pending_space = false;
  ws = false;
  while (b.next(c, pos, w)) {
    if (w) ws = (char_class(s, c, pos, hi) & UC_SPACE) != 0;
    bool sp_ = (w != 0) && ws;
    if (w == 0) {   // continuation byte: part of the current char
      if (c != ' ' && !ws) {
        if (phase == 1) name_end_idx = idx + 1;
        else if (phase == 3 && !pending_space) rest_end_idx = idx + 1;
      }
      idx++;
      continue;
    }
    if (phase == 0) {
      if (!sp_) { phase = 1; name_start_idx = idx; if (nlen < 16) name[nlen] = c; nlen++; name_end_idx = idx + 1; }
    } else if (phase == 1) {
      if (sp_) phase = 2;
      else { if (nlen < 16) name[nlen] = c; nlen++; name_end_idx = idx + 1; }
    } else {
      if (!sp_) {
        if (phase == 2) { phase = 3; rest_start_idx = idx; rest_first = idx; }
        else if (pending_space) rest_has_inner_space = true;
        pending_space = false;
        if (rlen < 32) rest[rlen] = c;
        rlen++;
        rest_end_idx = idx + 1; rest_last_end = idx + 1;
      } else if (phase == 3) {
        pending_space = true;
      }
    }
    idx++;
  }
  (void)rest_first; (void)rest_last_end;
  bool n_pragma = nlen <= 16 && text_eq(name, nlen, "pragma");
  if (n_pragma) { li.kind = LK_PRAGMA_DIR; return li; }
  bool n_ifdef = nlen <= 16 && text_eq(name, nlen, "ifdef");
  bool n_ifndef = nlen <= 16 && text_eq(name, nlen, "ifndef");
  u32 span_from = 0, span_to = 0;  // blanked-char index range to copy to the arena
  bool want_text = false;
  if (n_ifdef || n_ifndef) {
    li.is_ifndef = n_ifndef;
    if (phase < 3 || rest_has_inner_space) {
      li.kind = LK_BAD_ARITY;
    } else {
      u8 m = 0;
      if (rlen <= 32) {
        if (text_eq(rest, rlen, "__CUDACC__")) m = MAC_CUDACC;
        else if (text_eq(rest, rlen, "__CUDA_ARCH__")) m = MAC_CUDA_ARCH;
        else if (text_eq(rest, rlen, "__CUDACC_RELAXED_CONSTEXPR__")) m = MAC_RELAXED;
      }
      if (m) { li.kind = n_ifdef ? LK_IFDEF : LK_IFNDEF; li.macro = m; }
      else { li.kind = LK_BAD_MACRO; want_text = true; span_from = rest_start_idx; span_to = rest_end_idx; }
    }
  } else if (nlen <= 16 && text_eq(name, nlen, "else")) {
    li.kind = LK_ELSE;
  } else if (nlen <= 16 && text_eq(name, nlen, "endif")) {
    li.kind = LK_ENDIF;
  } else if (nlen <= 16 && text_eq(name, nlen, "error")) {
    li.kind = LK_ERROR;
    want_text = true;
    if (phase == 3) { span_from = rest_start_idx; span_to = rest_end_idx; }
  } else {
    li.kind = LK_UNKNOWN;
    want_text = true;
    if (nlen) { span_from = name_start_idx; span_to = name_end_idx; }
  }
  if (want_text && span_to > span_from) {
    // copy blanked chars [span_from, span_to) (indices count every yielded byte)
    b.init(s, sp, lo, hi, st);
    while (b.next(c, pos, w) && pos != hash_pos) {}
    u32 len = 0, i = 0;
    // measure bytes first
    Blanker b2 = b;
    while (b2.next(c, pos, w)) {
      if (i >= span_from && i < span_to && !(w == 0 && c == ' ')) len++;
      i++;
      if (i >= span_to) break;
    }
    u32 off = at_add(arena_top, len);
    if (off + len <= arena_cap) {
      i = 0;
      u32 k = 0;
      while (b.next(c, pos, w)) {
        if (i >= span_from && i < span_to && !(w == 0 && c == ' ')) {
          arena[off + k++] = c;  // blanked continuation bytes vanish; real ones are copied
        }
        i++;
        if (i >= span_to) break;
      }
      li.span = (1ull << 63) | ((u64)off << 32) | len;  // arena-tagged span
    } else {
      li.span = ((u64)0xFFFFFFFFu << 32);
    }
  }
  return li;
}

// Tokenizer over one active logical line (lexer.py:46-118).  mode 0 counts,
// mode 1 emits into out[].  Returns the token count; on a lexical error sets
// *err (M_LEX_*), *err_col, *err_pos and stops.
struct LexErr { u16 msg; u32 col, pos; };

// Writes a token built in registers with two 16-byte stores at scope exit.
struct TokStore {
  Tok* dst;
  const Tok* src;
  EXS_HD ~TokStore() {
#if defined(__CUDA_ARCH__) && !defined(EXS_EMU)
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(dst);
    d[0] = s[0];
    d[1] = s[1];
#else
    *dst = *src;
#endif
  }
};

EXS_HD inline u32 lex_line(const u8* s, const u32* sp, u32 lo, u32 hi, u8 st, u32 line_no,
                           u32 file, u8 mask, Tok* out, LexErr* err) {
  Blanker b;
  b.init(s, sp, lo, hi, st);
  u32 col = 1, n = 0;
  err->msg = 0;
  u8 c, w; u32 pos;
  bool have = b.next(c, pos, w);
  while (have) {
    if (c == ' ' || c == '\t' || c == '\r') {
      col += w;
      have = b.next(c, pos, w);
      continue;
    }
    if (w == 0) {  // stray continuation byte of a blanked char or string: width 0
      have = b.next(c, pos, w);
      continue;
    }
    u32 tcol = col, tpos = pos;
    if (c == '#') {
      // scan [alnum _ space tab]*, then words must be exactly "pragma NAME"
      u32 consumed = 1;
      int nw = 0; bool inword = false, first_ok = true;
      u8 wbuf[8]; u32 wl = 0;
      u32 name_pos = 0, name_end = 0; NameHash nh; u32 nl = 0;
      have = b.next(c, pos, w);
      bool acc = true;
      // lexer.py:67-70: isalnum, '_', ' ' and '\t' continue the directive
      while (have) {
        bool ok;
        if (w == 0) ok = c == ' ' || (acc && c >= 0x80);
        else ok = c == ' ' || c == '\t' || c == '_' || (char_class(s, c, pos, hi) & UC_ALNUM) != 0;
        if (w) acc = ok;
        if (!ok) break;
        bool spc = (c == ' ' || c == '\t');
        if (!spc) {
          if (!inword) { nw++; inword = true; if (nw == 2) name_pos = pos; }
          if (nw == 1) { if (wl < 8) wbuf[wl] = c; wl++; }
          if (nw == 2) { nh.step(c); nl++; name_end = pos + 1; }
        } else {
          inword = false;
        }
        consumed += w;
        have = b.next(c, pos, w);
      }
      first_ok = (wl == 6 && text_eq(wbuf, 6, "pragma"));
      if (nw != 2 || !first_ok) {
        err->msg = M_LEX_PRAGMA; err->col = tcol; err->pos = tpos;
        return n;
      }
      if (out) {
        Tok t;
        TokStore ts_{out + n, &t};
        const u64 h = nh.done();
        t.pos = name_pos; t.end = name_end; t.line = line_no; t.col = tcol; t.hv = h;
        t.kind = TK_PRAGMA; t.id = vocab_hash(h, nl); t.mask = mask; t.flags = 0; t.file = file;
      }
      n++;
      col += consumed;
      continue;
    }
    if (c == '"') {
      u32 cw = 1;
      NameHash nh; u32 nl = 0;
      u32 cstart = NONE, cend = 0;
      bool closed = false;
      have = b.next(c, pos, w);
      while (have) {
        if (c == '"' && w) { closed = true; cw += 1; break; }
        if (cstart == NONE) cstart = pos;
        cend = pos + 1;
        nh.step(c);
        nl++;
        cw += w;
        have = b.next(c, pos, w);
      }
      if (!closed) {
        err->msg = M_LEX_STRING; err->col = tcol; err->pos = tpos;
        return n;
      }
      if (out) {
        Tok t;
        TokStore ts_{out + n, &t};
        t.pos = cstart == NONE ? pos : cstart; t.end = cstart == NONE ? pos : cend;
        const u64 h = nh.done();
        t.line = line_no; t.col = tcol; t.hv = h;
        t.kind = TK_STRING; t.id = vocab_hash(h, nl); t.mask = mask; t.flags = 0; t.file = file;
      }
      n++;
      col += cw;
      have = b.next(c, pos, w);
      continue;
    }
    // integers and identifiers (lexer.py:86-104): str.isdigit starts a
    // number continued by isdigit; isalpha or '_' starts an identifier
    // continued by isalnum or '_' (Unicode classes, exs_unicode.cuh)
    const u8 k0 = char_class(s, c, pos, hi);
    if ((k0 & (UC_DIGIT | UC_ALPHA)) || c == '_') {
      bool digits = (k0 & UC_DIGIT) != 0;
      NameHash nh; u64 val = 0; bool ovf = false;
      u32 nl = 0, ncp = 0; u32 last = pos; bool spl = false;
      u32 prevpos = pos;
      bool acc = true;  // the current code point is part of the token
      while (have) {
        bool ok;
        if (w == 0) {
          ok = acc && c >= 0x80;  // continuation byte of the current code point
        } else {
          const u32 cp = c < 0x80 ? (u32)c : utf8_at(s, pos, hi);
          const UClass u = uclass(cp);
          ok = digits ? (u.cls & UC_DIGIT) != 0 : ((u.cls & UC_ALNUM) != 0 || c == '_');
          acc = ok;
          if (ok && digits) {
            // int(text): decimal digits only (a non-decimal digit makes the
            // reference raise -- outside its contract; flagged like overflow)
            u32 dv = (u.cls & UC_DECIMAL) ? (cp - u.start) % 10 : 0;
            if (!(u.cls & UC_DECIMAL)) ovf = true;
            u64 nv = val * 10 + dv;
            if (val > 1844674407370955161ull || nv < val) ovf = true;
            val = nv;
          }
        }
        if (!ok) break;
        if (pos != prevpos + 1 && nl) spl = true;
        prevpos = pos;
        nh.step(c);
        nl++;
        ncp += w;
        last = pos;
        have = b.next(c, pos, w);
      }
      if (out) {
        const u64 h = nh.done();
        Tok t;
        TokStore ts_{out + n, &t};
        t.pos = tpos; t.end = last + 1; t.line = line_no; t.col = tcol;
        t.hv = digits ? val : h;
        t.kind = digits ? TK_INT : TK_IDENT;
        t.id = digits ? 0 : vocab_hash(h, nl);
        t.mask = mask; t.flags = (ovf ? TF_INT_OVERFLOW : 0) | (spl ? TF_HAS_SPLICE : 0); t.file = file;
      }
      n++;
      col += ncp;
      continue;
    }
    // punctuators, greedy in reference order
    {
      Blanker la = b;
      u8 c1 = 0, c2 = 0, w1 = 0, w2 = 0; u32 p1 = 0, p2 = 0;
      bool h1 = la.next(c1, p1, w1);
      Blanker la2 = la;
      bool h2 = h1 && la2.next(c2, p2, w2);
      if (!h1 || !w1) c1 = 0;
      if (!h2 || !w2) c2 = 0;
      u8 pid = 0, plen = 0;
      if (c == '<' && c1 == '<' && c2 == '<') { pid = P_LLL; plen = 3; }
      else if (c == '>' && c1 == '>' && c2 == '>') { pid = P_GGG; plen = 3; }
      else if (c == ':' && c1 == ':') { pid = P_SCOPE; plen = 2; }
      else if (c == '=' && c1 == '=') { pid = P_EQ; plen = 2; }
      else if (c == '!' && c1 == '=') { pid = P_NE; plen = 2; }
      else if (c == '&' && c1 == '&') { pid = P_AND; plen = 2; }
      else if (c == '|' && c1 == '|') { pid = P_OR; plen = 2; }
      else if (c == '+' && c1 == '+') { pid = P_INC; plen = 2; }
      else {
        plen = 1;
        switch (c) {
          case '{': pid = P_LBRACE; break;
          case '}': pid = P_RBRACE; break;
          case '(': pid = P_LPAREN; break;
          case ')': pid = P_RPAREN; break;
          case '<': pid = P_LT; break;
          case '>': pid = P_GT; break;
          case ',': pid = P_COMMA; break;
          case ';': pid = P_SEMI; break;
          case '.': pid = P_DOT; break;
          case '!': pid = P_BANG; break;
          case '=': pid = P_ASSIGN; break;
          default: pid = 0;
        }
      }
      if (!pid) {
        err->msg = M_LEX_CHAR; err->col = tcol; err->pos = tpos;
        return n;
      }
      u32 endp = plen == 1 ? tpos + 1 : (plen == 2 ? p1 + 1 : p2 + 1);
      if (out) {
        Tok t;
        TokStore ts_{out + n, &t};
        t.pos = tpos; t.end = endp; t.line = line_no; t.col = tcol; t.hv = 0;
        t.kind = TK_PUNCT; t.id = pid; t.mask = mask; t.flags = 0; t.file = file;
      }
      n++;
      col += plen;
      if (plen == 1) have = b.next(c, pos, w);
      else if (plen == 2) { b = la; have = b.next(c, pos, w); }
      else { b = la2; have = b.next(c, pos, w); }
    }
  }
  return n;
}

}  // namespace exs
