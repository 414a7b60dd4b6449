// exs_lexw.cuh -- K2/K3 word-parallel lexing: one thread per 32-byte word.
//
// The reference preprocesses and lexes line by line (syntax/preprocess.py:
// 81-203, syntax/lexer.py:46-118).  Here the unit of work is a fixed 32-byte
// word of the concatenated corpus, so every thread does the same amount of
// work regardless of line lengths:
//   * lex_words (word_info): the comment-DFA transfer map of the word over its
//     logical (non-spliced) bytes, its line starts and newlines, and whether it
//     holds a "special" byte (spliced byte, non-ASCII byte or '#');
//   * one inclusive scan of WScan composes the maps (DFA state at every word
//     start), counts line starts / newlines and carries the last line start;
//   * plain logical lines (no special byte) are tokenized byte-parallel: a
//     word emits the tokens that START in it; the token in progress at its
//     first byte is recovered by a short look-back (identifier/number run, or
//     the greedy alignment of a punctuator run);
//   * special lines (continuations, UTF-8, directives, pragmas) are lexed
//     whole by the word holding their first byte, with the sequential line
//     lexer of exs_lex.cuh (same code as the reference's line loop).
// Token counts per word -> exclusive scan -> emit pass writes tokens in source
// order.  Lexical errors are reduced per (file, pass) with atomicMin on the
// byte position; line/column/message are recovered from the position.
#pragma once
#include "exs_lex.cuh"

namespace exs {

// per (file, pass) status -- fp = 2*file + pass (pass 0 host, 1 device)
struct FP {
  u32 pp_line;    // line number of the first E0002 directive (NONE = ok, NONE-1 = no such pass)
  u16 pp_msg;
  u16 lex_msg;    // first lexical error: message (resolved from lex_pos)
  u64 pp_a0;      // text span / flags for the message
  u32 pp_a1;
  u32 lex_line;   // first lexical error in an active line: line number (NONE = ok)
  u32 lex_col;
  u32 lex_pos;    // its byte position (atomicMin over the emit pass)
  u32 eof_line, eof_col;
  u32 view;       // view serving this pass (NONE if none)
  u32 perr;       // parse failed (1) / ok (0)
};

// packed 6-state map of the comment DFA: 4 bits per start state
constexpr u32 MAP_ID = 0x543210u;
EXS_HD inline u32 map_at(u32 m, u32 s) { return (m >> (4 * s)) & 15u; }
EXS_HD inline u32 map_compose(u32 a, u32 b) {  // a, then b
  u32 r = 0;
#pragma unroll
  for (u32 s = 0; s < 6; s++) r |= map_at(b, map_at(a, s)) << (4 * s);
  return r;
}

struct WScan {
  u32 map;  // comment-DFA transfer map over the word's logical bytes
  u32 lsp;  // last logical-line start in the word (0 if none; max-scanned)
  u64 lc;   // line starts << 32 | newline bytes (summed)
};
struct WScanOp {
  EXS_HD WScan operator()(const WScan& a, const WScan& b) const {
    WScan r;
    r.map = map_compose(a.map, b.map);
    r.lsp = a.lsp > b.lsp ? a.lsp : b.lsp;
    r.lc = a.lc + b.lc;
    return r;
  }
};

// one directive line (preprocess.py:168-200), in source order after sorting
struct DirRec {
  u32 pos, file, line_no;
  u8 kind, macro, is_ifndef, pad;
  u64 span;
};

// one special logical line (continuation, UTF-8, '#'): lexed by its own
// thread with the reference's sequential line loop (run_lex K3s)
struct SRec {
  u32 pos, file, line_no;
  u32 count;   // tokens (0 for a directive line)
  u32 slot;    // first token index (emit pass)
  u8 lst;      // comment state at the line start (S_CODE / S_BLOCK)
  u8 kind;     // LK_* of the line
  u8 mask;     // pass activity of the line (emit pass)
  u8 pad;
};

// per-word masks of phases 1-2, written by the count pass for the emit pass
struct alignas(16) WordMasks {
  u32 f, lsb, nl, own, starts, err, idst, DGc, IDc, qs, qt, sm, pst, pad[3];
};

struct LexW {
  const u8* src; u32 n; bool vec;  // vec: 16-byte aligned source, vector loads allowed
  const u32* sp; const u32* fs;    // splice / file-start bitmaps
  const WScan* wsc;                // inclusive scan (word w reads wsc[w-1])
  u32* special;                    // per logical line: 0 plain, else special (count pass: SRec index + 1)
  const u32* foff; u32 F; const u8* cfg;
  const u32* fnl;                  // global newline count before each file start
  u32* nspecial;                   // special lines (upper bound, mark pass)
  // count pass: special-line records
  SRec* srec; u32* nsrec; u32 srcap;
  u32 ns;                          // special lines recorded
  // emit pass
  const u32* fdir; const DirRec* dirs; const u8* dlive; FP* fp;
  WordMasks* wm;                   // count pass writes, emit pass reads (nullptr: recompute)
  // emit passes: the parser's per-token arrays (file, kind << 8 | id) and flags
  // (tsplit[f]: a token of file f is live in one pass only; tsplit[F]: some
  // token is not live in all its file's passes) -- no second pass over the records
  u32* tfile; u16* tkid; u32* tsplit;
};
// the parser's arrays for token t (emit passes)
EXS_HD inline void tok_meta(const LexW& X, u32 t, const Tok& k) {
  X.tfile[t] = k.file;
  X.tkid[t] = (u16)(((u32)k.kind << 8) | k.id);
  const u8 m = k.mask;
  if (m == 1 || m == 2) at_or(&X.tsplit[k.file], 1u);
  if (m != ((X.cfg[k.file] & CFG_PLAIN) ? 1 : 3) && !ld_volatile(X.tsplit + X.F)) at_or(X.tsplit + X.F, 1u);
}

EXS_HD inline u32 upper_file(const u32* foff, u32 F, u32 p) {
  // last f with foff[f] <= p
  u32 lo = 0, hi = F;
  while (hi - lo > 1) {
    u32 mid = (lo + hi) / 2;
    if (foff[mid] <= p) lo = mid; else hi = mid;
  }
  return lo;
}
EXS_HD inline u8 file_passes(u8 cfg) { return (cfg & CFG_PLAIN) ? 1 : 3; }

// punctuators that can start a multi-character token (lexer.py:30-39)
EXS_HD inline bool is_pset(u8 c) {
  return c == '<' || c == '>' || c == ':' || c == '=' || c == '!' || c == '&' || c == '|' || c == '+';
}
// greedy punctuator at c followed by c1, c2 (0 = none); pid 0: not a punctuator
EXS_HD inline u32 punct_len(u8 c, u8 c1, u8 c2, u8& pid) {
  if (c == '<' && c1 == '<' && c2 == '<') { pid = P_LLL; return 3; }
  if (c == '>' && c1 == '>' && c2 == '>') { pid = P_GGG; return 3; }
  if (c == ':' && c1 == ':') { pid = P_SCOPE; return 2; }
  if (c == '=' && c1 == '=') { pid = P_EQ; return 2; }
  if (c == '!' && c1 == '=') { pid = P_NE; return 2; }
  if (c == '&' && c1 == '&') { pid = P_AND; return 2; }
  if (c == '|' && c1 == '|') { pid = P_OR; return 2; }
  if (c == '+' && c1 == '+') { pid = P_INC; return 2; }
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
  return 1;
}

EXS_HD inline u32 word_of(const u32 r[8], u32 k) {  // r[k] without local memory
  return k < 4 ? (k < 2 ? (k == 0 ? r[0] : r[1]) : (k == 2 ? r[2] : r[3]))
               : (k < 6 ? (k == 4 ? r[4] : r[5]) : (k == 6 ? r[6] : r[7]));
}
EXS_HD inline u8 byte_of(const u32 r[8], u32 j) { return (u8)(word_of(r, j >> 2) >> (8 * (j & 3))); }
// dynamic-index reads of a word mirrored in shared memory (lex_word): one load
// where the register select chain of word_of takes seven selects
EXS_HD inline u8 byte_at(const u32* R, u32 j) { return (u8)(R[j >> 2] >> (8 * (j & 3))); }
EXS_HD inline u32 ffs32(u32 x) {  // index of the lowest set bit (x != 0)
#if defined(__CUDA_ARCH__) && !defined(EXS_EMU)
  return (u32)__ffs((int)x) - 1;
#else
  return (u32)__builtin_ctz(x);
#endif
}
EXS_HD inline u32 hib32(u32 x) {  // index of the highest set bit (x != 0)
#if defined(__CUDA_ARCH__) && !defined(EXS_EMU)
  return 31u - (u32)__clz((int)x);
#else
  return 31u - (u32)__builtin_clz(x);
#endif
}
EXS_HD inline u32 popc32(u32 x) {
#if defined(__CUDA_ARCH__) && !defined(EXS_EMU)
  return (u32)__popc(x);
#else
  return (u32)__builtin_popcount(x);
#endif
}

// sequential reader of a token's bytes: registers inside the word (one select
// chain per 4 bytes), global memory past it
struct ByteCursor {
  const u32* r; const u8* src; u32 base, cur;
  u32 wv;
  EXS_HD u8 at(u32 q) {
    if (q < base + 32) {
      const u32 j = q - base;
      if ((j >> 2) != cur) { cur = j >> 2; wv = r[cur]; }
      return (u8)(wv >> (8 * (j & 3)));
    }
    return src[q];
  }
};

// SWAR byte classes of a little-endian word: 0x80 in every byte that is an
// ASCII digit / identifier character (bytes >= 0x80 never match)
EXS_HD inline u32 swar_range(u32 x, u32 lo, u32 hi) {  // lo <= b <= hi, for b < 0x80
  const u32 ge = ((x | 0x80808080u) - lo * 0x01010101u) & 0x80808080u;
  const u32 le = ((0x80u + hi) * 0x01010101u - (x & 0x7F7F7F7Fu)) & 0x80808080u;
  return ge & le;
}
EXS_HD inline u32 swar_digit(u32 x) { return swar_range(x, 0x30, 0x39) & ~x; }
EXS_HD inline u32 swar_ident(u32 x) {
  const u32 t = x ^ 0x5F5F5F5Fu;  // '_'
  const u32 us = ~(((t & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | t) & 0x80808080u;
  return (swar_range(x, 0x30, 0x39) | swar_range(x | 0x20202020u, 0x61, 0x7A) | us) & ~x;
}
// end of the digit / identifier run continuing at q (a word boundary, so
// 4-aligned) before the file end: four bytes per step
EXS_HD inline u32 run_end(const LexW& X, u32 q, u32 fend, bool num) {
  if (X.vec) {
    const u32* s32 = reinterpret_cast<const u32*>(X.src);
    while (q < fend) {
      const u32 x = s32[q >> 2];
      const u32 miss = ~(num ? swar_digit(x) : swar_ident(x)) & 0x80808080u;
      if (miss) { q += ffs32(miss) >> 3; break; }
      q += 4;
    }
    return q < fend ? q : fend;
  }
  while (q < fend && (num ? is_digit(X.src[q]) : is_ident_char(X.src[q]))) q++;
  return q;
}

// NameHash of the bytes [lo, hi), four at a step
// aligned source word a (absolute word index): registers inside the word at
// `base`, else global memory (the batch ends in 64 zero bytes)
EXS_HD inline u32 word_at(const LexW& X, const u32* r, u32 base, u32 a) {
  const u32 k = a - (base >> 2);
  if (k < 8) return r[k];
  if (X.vec) return reinterpret_cast<const u32*>(X.src)[a];
  u32 x = 0;
  for (u32 i = 0; i < 4; i++) x |= (u32)X.src[4 * a + i] << (8 * i);
  return x;
}
EXS_HD inline u64 name_hash_range(const LexW& X, const u32* r, u32 base, u32 lo, u32 hi) {
  u64 h = 1469598103934665603ull;
  const u32 sh = 8 * (lo & 3);
  u32 a = lo >> 2;
  u32 w0 = word_at(X, r, base, a);
  for (u32 q = lo; q < hi; q += 4) {
    const u32 w1 = word_at(X, r, base, ++a);  // one word per chunk: the next chunk's low word
#if defined(__CUDA_ARCH__) && !defined(EXS_EMU)
    u32 x = __funnelshift_r(w0, w1, sh);
#else
    u32 x = sh ? (w0 >> sh) | (w1 << (32 - sh)) : w0;
#endif
    if (hi - q < 4) x &= (1u << (8 * (hi - q))) - 1;
    h = nh_mix(h, x);
    w0 = w1;
  }
  return nh_fin(h, hi - lo);
}

// bit k (k < 4) set where byte k of x equals c
EXS_HD inline u32 byte_eq_mask(u32 x, u8 c) {
#if defined(__CUDA_ARCH__) && !defined(EXS_EMU)
  const u32 e = __vcmpeq4(x, 0x01010101u * c);  // 0xFF per equal byte
  return (e & 1u) | ((e >> 7) & 2u) | ((e >> 14) & 4u) | ((e >> 21) & 8u);
#else
  u32 o = 0;
  for (u32 k = 0; k < 4; k++) o |= (((x >> (8 * k)) & 0xFFu) == c ? 1u : 0u) << k;
  return o;
#endif
}

EXS_HD inline void load_word(const LexW& X, u32 base, u32 r[8]) {
#if defined(__CUDA_ARCH__) && !defined(EXS_EMU)
  if (X.vec && base + 32 <= X.n) {
    const uint4* q = reinterpret_cast<const uint4*>(X.src + base);
    uint4 a = __ldg(q), b = __ldg(q + 1);
    r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w;
    r[4] = b.x; r[5] = b.y; r[6] = b.z; r[7] = b.w;
    return;
  }
#endif
  for (u32 k = 0; k < 8; k++) r[k] = 0;
  for (u32 j = 0; j < 32 && base + j < X.n; j++) r[j >> 2] |= (u32)X.src[base + j] << (8 * (j & 3));
}

// comment-DFA step as a table: the transition map of the character's class
// (other, '"', '/', '*', '\n'), 4 bits per state -- branch-free
EXS_HD inline u32 dfa_class_map(u8 c) {
  return c == '"' ? 0x443022u : (c == '/' ? 0x043231u : (c == '*' ? 0x553240u : (c == '\n' ? 0x440000u : 0x443200u)));
}
EXS_HD inline bool is_single(u8 c) {
  return c == '{' || c == '}' || c == '(' || c == ')' || c == ',' || c == ';' || c == '.';
}

// Byte classes of a whole word, eight at a time: a 256-entry table gives each
// byte its class bits, eight class bytes are packed into 64 bits and one 8x8
// bit transpose turns them into eight 8-bit position masks (one per class).
// About 10 ALU operations per byte for eight classes, where a compare chain per
// byte and class took ~45 (the masks phase was ALU-bound).
enum : u32 {  // kTokClass bits (lex_count / lex_emit)
  TC_ID = 1, TC_DG = 2, TC_WS = 4, TC_PS = 8, TC_SG = 16, TC_QT = 32, TC_SL = 64, TC_ST = 128
};
enum : u32 {  // kLineClass bits (lex_words / mark_special)
  LC_QT = 1, LC_SL = 2, LC_ST = 4, LC_NL = 8, LC_HS = 16, LC_HI = 32
};
struct ClassTable { u8 c[256]; };
constexpr ClassTable make_tok_class() {
  ClassTable t{};
  for (u32 c = 0; c < 256; c++) {
    u32 v = 0;
    const bool dg = c >= '0' && c <= '9';
    const bool al = (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z');
    if (al || dg || c == '_') v |= TC_ID;
    if (dg) v |= TC_DG;
    if (c == ' ' || c == '\t' || c == '\r') v |= TC_WS;
    if (c == '<' || c == '>' || c == ':' || c == '=' || c == '!' || c == '&' || c == '|' || c == '+') v |= TC_PS;
    if (c == '{' || c == '}' || c == '(' || c == ')' || c == ',' || c == ';' || c == '.') v |= TC_SG;
    if (c == '"') v |= TC_QT;
    if (c == '/') v |= TC_SL;
    if (c == '*') v |= TC_ST;
    t.c[c] = (u8)v;
  }
  return t;
}
constexpr ClassTable make_line_class() {
  ClassTable t{};
  for (u32 c = 0; c < 256; c++) {
    u32 v = 0;
    if (c == '"') v |= LC_QT;
    if (c == '/') v |= LC_SL;
    if (c == '*') v |= LC_ST;
    if (c == '\n') v |= LC_NL;
    if (c == '#') v |= LC_HS;
    if (c >= 0x80) v |= LC_HI;
    t.c[c] = (u8)v;
  }
  return t;
}
#ifndef EXS_EMU
__device__ const ClassTable kTokClassDev = make_tok_class();
__device__ const ClassTable kLineClassDev = make_line_class();
#endif
static constexpr ClassTable kTokClassHost = make_tok_class();
static constexpr ClassTable kLineClassHost = make_line_class();

// 8x8 bit transpose: bit i of byte k of the result = bit k of byte i of x
EXS_HD inline u64 transpose8(u64 x) {
  u64 t = (x ^ (x >> 7)) & 0x00AA00AA00AA00AAull; x ^= t ^ (t << 7);
  t = (x ^ (x >> 14)) & 0x0000CCCC0000CCCCull; x ^= t ^ (t << 14);
  t = (x ^ (x >> 28)) & 0x00000000F0F0F0F0ull; x ^= t ^ (t << 28);
  return x;
}
// per-class 32-bit position masks of the word r: m[k] bit j = class bit k of byte j
template <bool TOK>
EXS_HD inline void word_classes(const u32 r[8], u32 m[8]) {
#if defined(__CUDA_ARCH__) && !defined(EXS_EMU)
  const u8* tab = TOK ? kTokClassDev.c : kLineClassDev.c;
#else
  const u8* tab = TOK ? kTokClassHost.c : kLineClassHost.c;
#endif
#pragma unroll
  for (u32 k = 0; k < 8; k++) m[k] = 0;
#pragma unroll
  for (u32 g = 0; g < 4; g++) {
    const u32 a = r[2 * g], b = r[2 * g + 1];
    const u32 lo = (u32)tab[a & 0xFFu] | ((u32)tab[(a >> 8) & 0xFFu] << 8) | ((u32)tab[(a >> 16) & 0xFFu] << 16) |
                   ((u32)tab[a >> 24] << 24);
    const u32 hi = (u32)tab[b & 0xFFu] | ((u32)tab[(b >> 8) & 0xFFu] << 8) | ((u32)tab[(b >> 16) & 0xFFu] << 16) |
                   ((u32)tab[b >> 24] << 24);
    const u64 x = transpose8(((u64)hi << 32) | lo);
#pragma unroll
    for (u32 k = 0; k < 8; k++) m[k] |= (u32)((x >> (8 * k)) & 0xFFu) << (8 * g);
  }
}

// The comment DFA over one word from state st, event-driven: between the
// bytes where the current state can change -- '"' or '/' in code, '"' or '\n'
// in a string, '\n' in a line comment, '*' in a block comment, any byte after
// a '/' in code or a '*' in a block comment, and file starts (reset to code);
// never a spliced byte -- the state is constant, so a word costs one step per
// such byte instead of one per byte.  Q, SL, ST, NL: byte masks of '"', '/',
// '*', '\n'; only bytes of `lim` are events.  With MASKS, the state before
// every byte is reported as bl (comment text and openers), sm (string),
// sbb (block comment) -- the per-byte loop it replaces: lex_word phase 1.
// Returns the state after the word.
template <bool MASKS>
EXS_HD inline u32 dfa_word(u32 st, const u32 r[8], u32 Q, u32 SL, u32 ST, u32 NL, u32 spw, u32 fsw, u32 lim,
                           u32& bl, u32& sm, u32& sbb) {
  const u32 ns = ~spw;
  u32 p = 0;
  while (true) {
    u32 evs;
    if (st == S_CODE) evs = (Q | SL) & ns;
    else if (st == S_STR) evs = (Q | NL) & ns;
    else if (st == S_LINE) evs = NL & ns;
    else if (st == S_BLOCK) evs = ST & ns;
    else evs = ns;  // S_SLASH, S_STAR: the next byte decides
    const u32 cand = (evs | fsw) & lim & (p >= 32 ? 0u : (~0u << p));
    const u32 e = cand ? ffs32(cand) : 32u;
    if (MASKS && e > p) {
      const u32 run = (e >= 32 ? ~0u : ((1u << e) - 1)) & ~((1u << p) - 1);
      if (st >= S_LINE) bl |= run;
      if (st == S_STR) sm |= run;
      if (st == S_BLOCK) sbb |= run;
    }
    if (e >= 32) break;
    const u32 b = 1u << e;
    if (fsw & b) st = S_CODE;
    if (MASKS) {
      if (st >= S_LINE) bl |= b;
      if (st == S_STR) sm |= b;
      if (st == S_BLOCK) sbb |= b;
      if (st == S_SLASH && (ns & b) && ((SL | ST) & b)) bl |= b | (b >> 1);  // opener
    }
    if (ns & b) st = (dfa_class_map(byte_of(r, e)) >> (4 * st)) & 15u;
    p = e + 1;
  }
  return st;
}

// K2: per-word scan record and special flag
EXS_HD inline WScan word_info(const LexW& X, u32 w, u8& special, u32& nhash) {
  WScan o{MAP_ID, 0, 0};
  special = 0; nhash = 0;
  const u32 base = w * 32;
  if (base >= X.n) return o;
  u32 r[8];
  load_word(X, base, r);
  const u32 spw = X.sp[w], fsw = X.fs[w];
  const bool prev_nl = base > 0 && X.src[base - 1] == '\n' && !bit_get(X.sp, base - 1);
  const u32 m = X.n - base < 32 ? X.n - base : 32;
  const u32 valid = m == 32 ? ~0u : ((1u << m) - 1);
  // byte masks (table + bit transpose)
  u32 cm[8];
  word_classes<false>(r, cm);
  const u32 Q = cm[0] & valid, SL = cm[1] & valid, ST = cm[2] & valid, NL = cm[3] & valid,
            HS = cm[4] & valid, HI = cm[5] & valid;
  // logical line starts: file starts and bytes after a non-spliced newline
  const u32 ls = (fsw | ((NL & ~spw) << 1) | (prev_nl ? 1u : 0u)) & valid;
  if (ls) o.lsp = base + hib32(ls);
  const u32 nls = popc32(ls), nnl = popc32(NL);
  const u32 spec = ((spw & valid) | HS | HI) != 0, nh = popc32(HS);
  // the comment-DFA transfer map: one event-driven pass per start state
  u32 d0 = 0, d1 = 0, d2 = 0;
  const u32 s0 = dfa_word<false>(0, r, Q, SL, ST, NL, spw, fsw & valid, valid, d0, d1, d2);
  const u32 s1 = dfa_word<false>(1, r, Q, SL, ST, NL, spw, fsw & valid, valid, d0, d1, d2);
  const u32 s2 = dfa_word<false>(2, r, Q, SL, ST, NL, spw, fsw & valid, valid, d0, d1, d2);
  const u32 s3 = dfa_word<false>(3, r, Q, SL, ST, NL, spw, fsw & valid, valid, d0, d1, d2);
  const u32 s4 = dfa_word<false>(4, r, Q, SL, ST, NL, spw, fsw & valid, valid, d0, d1, d2);
  const u32 s5 = dfa_word<false>(5, r, Q, SL, ST, NL, spw, fsw & valid, valid, d0, d1, d2);
  special = (u8)spec; nhash = nh;
  o.map = s0 | (s1 << 4) | (s2 << 8) | (s3 << 12) | (s4 << 16) | (s5 << 20);
  o.lc = ((u64)nls << 32) | nnl;
  return o;
}

// K2b: flag the logical lines holding a special byte (word w has one)
EXS_HD inline void mark_special(const LexW& X, u32 w) {
  const u32 base = w * 32;
  const u32 li0 = w ? (u32)(X.wsc[w - 1].lc >> 32) - 1 : NONE;  // NONE + 1 wraps to line 0
  const bool prev_nl = base > 0 && X.src[base - 1] == '\n' && !bit_get(X.sp, base - 1);
  const u32 spw = X.sp[w], fsw = X.fs[w];
  const u32 m = X.n - base < 32 ? X.n - base : 32;
  const u32 valid = m == 32 ? ~0u : ((1u << m) - 1);
  u32 r[8];
  load_word(X, base, r);
  u32 cm[8];
  word_classes<false>(r, cm);
  const u32 NL = cm[3], SPC = cm[4] | cm[5];
  const u32 ls = (fsw | ((NL & ~spw) << 1) | (prev_nl ? 1u : 0u)) & valid;
  u32 spc = (SPC | spw) & valid;
  while (spc) {  // the first special byte of each logical line
    const u32 j = ffs32(spc);
    const u32 upto = j == 31 ? ~0u : ((2u << j) - 1);
    const u32 li = li0 + popc32(ls & upto);
    if (!X.special[li]) {
      X.special[li] = 1;
      at_add(X.nspecial, 1u);
    }
    const u32 later = ls & ~upto;  // skip to the next line start
    spc &= later ? ~((1u << ffs32(later)) - 1) : 0u;
  }
}

// end of the logical line starting at lo: first non-spliced '\n' or the file end
EXS_HD inline u32 logical_line_end(const LexW& X, u32 lo, u32 fend) {
  u32 q = lo;
  while (q < fend && !(X.src[q] == '\n' && !bit_get(X.sp, q))) q++;
  return q;
}

// K3: count (EMIT=false) or emit (EMIT=true) the tokens attributed to word w.
//
// Phase 1 (branch-uniform, unrolled): comment-DFA state before every byte and
// byte-class bitmasks.  Phase 2 (bit arithmetic): token starts of the plain
// lines -- identifier/number runs (a number is the all-digit prefix of a run
// that starts with a digit: X & ~(X + S) over the digit mask), single
// punctuators, string openers and the greedy alignment of punctuator runs.
// The count pass is a popcount; the emit pass walks the starts in order,
// interleaved with the special lines this word owns and with file starts.
template <bool EMIT>
EXS_HD inline u32 lex_word(const LexW& X, u32 w, Tok* out, u32 tbase) {
  const u32 base = w * 32;
  if (base >= X.n) return 0;
  u32 r[8];
  load_word(X, base, r);
#if defined(__CUDA_ARCH__) && !defined(EXS_EMU)
  // the word mirrored in this thread's shared-memory row (stride 9 words: no
  // bank conflicts), for the reads at run-time offsets
  __shared__ u32 sw_rows[256 * 9];
  u32* R = sw_rows + threadIdx.x * 9;
#pragma unroll
  for (u32 k = 0; k < 8; k++) R[k] = r[k];
#else
  const u32* R = r;
#endif
  const u32 m = X.n - base < 32 ? X.n - base : 32;
  const u32 valid = m == 32 ? ~0u : ((1u << m) - 1);
  const u32 spw = X.sp[w], fsw = X.fs[w] & valid;
  u32 st = S_CODE, lsp0 = 0, li0 = NONE, gnl0 = 0;
  if (w) {
    const WScan e = X.wsc[w - 1];
    st = map_at(e.map, S_CODE);
    lsp0 = e.lsp;
    li0 = (u32)(e.lc >> 32) - 1;
    gnl0 = (u32)e.lc;
  }
  const u32 st0 = st;
  u32 f, fend, sm, sbb, nl, lsb, own, IDc, DGc, idst, qs, qt, pst, starts, err;
  if (EMIT && X.wm) {
    // the count pass left the word's masks (phases 1-2 are not redone)
    const WordMasks M = X.wm[w];
    f = M.f; lsb = M.lsb; nl = M.nl; own = M.own; starts = M.starts; err = M.err; idst = M.idst;
    DGc = M.DGc; IDc = M.IDc; qs = M.qs; qt = M.qt; sm = M.sm; pst = M.pst; sbb = 0;
    fend = X.foff[f + 1];
  } else {
  const bool prev_nl = base > 0 && X.src[base - 1] == '\n' && !bit_get(X.sp, base - 1);
  // ---- phase 1: byte-class masks (branch-uniform, unrolled), then the
  // comment-DFA states before every byte, event-driven (dfa_word)
  u32 bl = 0;
  sm = 0; sbb = 0; nl = 0; qt = 0;
  u32 cm[8];
  word_classes<true>(r, cm);
  const u32 id = cm[0], dg = cm[1], ws = cm[2], ps = cm[3], sg = cm[4], sl = cm[6], star = cm[7];
  qt = cm[5];
#pragma unroll
  for (u32 k = 0; k < 8; k++) nl |= byte_eq_mask(r[k], '\n') << (4 * k);
  lsb = fsw | ((nl & ~spw) << 1) | (prev_nl ? 1u : 0u);
  dfa_word<true>(st, r, qt, sl, star, nl, spw, fsw, ~0u, bl, sm, sbb);
  lsb &= valid; nl &= valid;
  // ---- special lines: bytes excluded from the plain tokenizer; owned ones
  u32 spm = 0;
  own = 0;
  {
    u32 li = li0, seg = 0, rest = lsb;
    bool cur = li != NONE && X.special[li] != 0;
    while (true) {
      const u32 nx = rest ? ffs32(rest) : 32;
      if (cur && nx > seg) spm |= (nx >= 32 ? ~0u : ((1u << nx) - 1)) & ~((1u << seg) - 1);
      if (nx >= 32) break;
      li++;
      cur = X.special[li] != 0;
      if (cur) own |= 1u << nx;
      seg = nx;
      rest &= rest - 1;
    }
    spm &= valid;
  }
  // file of the word's first byte
  f = upper_file(X.foff, X.F, base);
  fend = X.foff[f + 1];
  // end of the file holding the word's last byte (look-ahead past the word)
  const u32 fe_last = (fsw & ~1u) ? X.foff[upper_file(X.foff, X.F, base + m - 1) + 1] : fend;
  // ---- phase 2: code characters and token starts
  u32 code = valid & ~(bl | sm | spw | nl | spm);
  if ((sl & code) >> 31) {  // a '/' opening a comment in the next word
    const u32 q = base + 32;
    const u8 nx = q < fe_last ? X.src[q] : 0;
    if (nx == '/' || nx == '*') code &= ~0x80000000u;
  }
  IDc = id & code; DGc = dg & code;
  const u32 ALc = IDc & ~DGc;
  u32 cin_id = 0, cin_num = 0, cin_ps = 0, pskip = 0;
  if ((code & 1u) && !(lsb & 1u) && base > 0 && st0 == S_CODE) {
    const u8 pc = X.src[base - 1];
    if (is_ident_char(pc)) {
      cin_id = 1;
      u32 q = base - 1;  // all-digit run back to its start -> inside a number
      while (q > lsp0 && is_digit(X.src[q])) q--;
      cin_num = (is_digit(X.src[q]) || !is_ident_char(X.src[q])) ? 1u : 0u;
    } else if (is_pset(pc)) {
      cin_ps = 1;
      u32 q = base - 1;
      while (q > lsp0 && is_pset(X.src[q - 1])) q--;
      while (q < base) {
        const u8 c1 = q + 1 < fend ? X.src[q + 1] : 0, c2 = q + 2 < fend ? X.src[q + 2] : 0;
        u8 pid;
        q += punct_len(X.src[q], c1, c2, pid);
      }
      pskip = q - base;
    }
  }
  // runs never continue across a file start (files are concatenated)
  const u32 rs = IDc & ~(((IDc << 1) | cin_id) & ~fsw);
  const u32 S = (rs & DGc) | (cin_num & DGc & 1u);
  u32 P = 0;  // digits of number prefixes, per file segment of the word
  {
    u32 lo = 0, rest = fsw & ~1u;
    while (true) {
      const u32 hi = rest ? ffs32(rest) : 32;
      const u32 seg = (hi >= 32 ? ~0u : ((1u << hi) - 1)) & ~((1u << lo) - 1);
      const u32 Xs = DGc & seg;
      P |= Xs & ~(Xs + (S & seg)) & seg;
      if (hi >= 32) break;
      lo = hi;
      rest &= rest - 1;
    }
  }
  idst = rs | (ALc & ((P << 1) | cin_num));
  qs = qt & code;
  const u32 sgs = sg & code;
  const u32 PSc = ps & code;
  pst = 0;
  u32 perr = 0;
  {
    u32 runs = PSc & ~(((PSc << 1) | cin_ps) & ~fsw);
    if (cin_ps && pskip < 32 && ((PSc >> pskip) & 1u)) runs |= 1u << pskip;
    while (runs) {
      u32 p = ffs32(runs);
      runs &= runs - 1;
      while (p < 32 && ((PSc >> p) & 1u)) {
        const u8 c = byte_at(R, p);
        u8 c1 = 0, c2 = 0;
        if (p + 1 < 32) { if (!((fsw >> (p + 1)) & 1u)) c1 = byte_at(R, p + 1); }
        else if (base + p + 1 < fe_last) c1 = X.src[base + p + 1];
        if (c1) {
          if (p + 2 < 32) { if (!((fsw >> (p + 2)) & 1u)) c2 = byte_at(R, p + 2); }
          else if (base + p + 2 < fe_last) c2 = X.src[base + p + 2];
        }
        u8 pid;
        const u32 len = punct_len(c, c1, c2, pid);
        if (pid) pst |= 1u << p; else perr |= 1u << p;
        p += len;
      }
    }
  }
  starts = idst | qs | sgs | pst;
  err = (code & ~(id | ws | ps | sg | qt | sl)) | (sl & code) | perr;
  if (!EMIT && X.wm) {
    WordMasks M;
    M.f = f; M.lsb = lsb; M.nl = nl; M.own = own; M.starts = starts; M.err = err; M.idst = idst;
    M.DGc = DGc; M.IDc = IDc; M.qs = qs; M.qt = qt; M.sm = sm; M.pst = pst; M.pad[0] = M.pad[1] = M.pad[2] = 0;
    X.wm[w] = M;
  }
  }
  u32 ntok = EMIT ? 0 : popc32(starts);
  // ---- phase 3: events in source order
  u32 fnl0 = X.fnl[f];
  u8 fmask = 0, live = 3;
  u32 dcur = 0, dend = 0;
  auto file_state = [&](u32 pos) {
    fnl0 = X.fnl[f];
    if (EMIT) {
      fmask = 0;
      for (u32 p = 0; p < 2; p++)
        if (X.fp[2 * f + p].pp_line == NONE) fmask |= (u8)(1u << p);
      dcur = X.fdir[f]; dend = X.fdir[f + 1]; live = 3;
      if (dcur < dend) {
        u32 lo = dcur, hi = dend;  // first directive at or after pos
        while (lo < hi) { u32 mid = (lo + hi) / 2; if (X.dirs[mid].pos < pos) lo = mid + 1; else hi = mid; }
        if (lo > dcur) live = X.dlive[lo - 1];
        dcur = lo;
      }
    }
  };
  file_state(base);
  u32 ev = own | fsw | (EMIT ? (starts | err) : 0u);
  while (ev) {
    const u32 j = ffs32(ev);
    ev &= ev - 1;
    const u32 i = base + j, bj = 1u << j, below = bj - 1;
    if (fsw & bj) {
      while (X.foff[f + 1] <= i) f++;
      fend = X.foff[f + 1];
      file_state(i);
    }
    const u32 lsj = lsb & (below | bj);
    const u32 lsp = lsj ? base + hib32(lsj) : lsp0;
    const u32 gnl = gnl0 + popc32(nl & below);
    const u8 mask = fmask & live;
    if (own & bj) {
      // a special line this word owns: recorded here, lexed by run_lex K3s
      const u32 lij = li0 + popc32(lsb & (below | bj));  // this line's index
      if (!EMIT) {
        const u32 k = at_add(X.nsrec, 1u);
        if (k < X.srcap) {
          SRec q;
          q.pos = i; q.file = f; q.line_no = 1 + gnl - fnl0; q.count = 0; q.slot = 0;
          q.lst = (sbb & bj) ? S_BLOCK : S_CODE; q.kind = 0; q.mask = 0; q.pad = 0;
          X.srec[k] = q;
          X.special[lij] = k + 1;  // the emit pass finds its record here
        }
      } else {
        SRec& q = X.srec[X.special[lij] - 1];
        if (q.kind >= LK_IFDEF) {
          if (dcur < dend && X.dirs[dcur].pos == i) { live = X.dlive[dcur]; dcur++; }
        } else {
          q.slot = tbase + ntok;
          q.mask = mask;
          ntok += q.count;
        }
      }
      continue;
    }
    if (!EMIT) continue;
    if (err & bj)
      for (u32 p = 0; p < 2; p++)
        if ((mask >> p) & 1u) at_min(&X.fp[2 * f + p].lex_pos, i);
    if (!(starts & bj)) continue;
    const u32 tl = 1 + gnl - fnl0, col = i - lsp + 1;
    const u8 c = byte_at(R, j);
    Tok t;
    t.pos = i; t.line = tl; t.col = col; t.mask = mask; t.flags = 0; t.file = f; t.hv = 0; t.id = 0;
    if (idst & bj) {
      const bool num = (DGc & bj) != 0;
      const u32 run = num ? DGc : IDc;
      const u32 stop = (~run | fsw) & ~(below | bj);
      u32 end;
      if (stop) {
        end = base + ffs32(stop);
      } else {
        end = run_end(X, base + 32, fend, num);
      }
      t.end = end;
      if (num) {
        u64 v = 0;
        bool ovf = false;
        ByteCursor bc{R, X.src, base, 8u, 0u};
        for (u32 q = i; q < end; q++) {
          const u64 nv = v * 10 + (bc.at(q) - '0');
          if (v > 1844674407370955161ull || nv < v) ovf = true;
          v = nv;
        }
        t.kind = TK_INT; t.hv = v; t.flags = ovf ? TF_INT_OVERFLOW : 0;
      } else {
        const u64 h = name_hash_range(X, R, base, i, end);
        t.kind = TK_IDENT; t.hv = h; t.id = vocab_hash(h, end - i);
      }
    } else if (qs & bj) {
      // the closing quote: first quote in string state after i, unless a newline
      // or the file end comes first (unterminated: an error and a dead slot)
      const u32 above = ~(below | bj);
      const u32 cq = qt & sm & above, nlm = (nl | fsw) & above;
      u32 close = NONE;
      bool term;
      if (cq && (!nlm || ffs32(cq) < ffs32(nlm))) { close = base + ffs32(cq); term = true; }
      else if (nlm) { term = false; }
      else {
        u32 q = base + 32;
        while (q < fend && X.src[q] != '"' && X.src[q] != '\n') q++;
        term = q < fend && X.src[q] == '"';
        close = q;
      }
      t.kind = TK_STRING;
      if (term) {
        const u64 h = name_hash_range(X, R, base, i + 1, close);
        const u32 len = close - i - 1;
        t.pos = len ? i + 1 : close; t.end = close; t.hv = h; t.id = vocab_hash(h, len);
      } else {
        for (u32 p = 0; p < 2; p++)
          if ((mask >> p) & 1u) at_min(&X.fp[2 * f + p].lex_pos, i);
        t.end = i + 1; t.mask = 0;
      }
    } else {
      u8 c1 = 0, c2 = 0;
      if (pst & bj) {
        if (j + 1 < 32) { if (!((fsw >> (j + 1)) & 1u)) c1 = byte_at(R, j + 1); }
        else if (i + 1 < fend) c1 = X.src[i + 1];
        if (c1) {
          if (j + 2 < 32) { if (!((fsw >> (j + 2)) & 1u)) c2 = byte_at(R, j + 2); }
          else if (i + 2 < fend) c2 = X.src[i + 2];
        }
      }
      u8 pid;
      const u32 len = punct_len(c, c1, c2, pid);
      t.kind = TK_PUNCT; t.id = pid; t.end = i + len;
    }
    {
      TokStore ts_{out + ntok, &t};
    }
    tok_meta(X, tbase + ntok, t);
    ntok++;
  }
  return ntok;
}

}  // namespace exs
