// exs_stage_lex.cuh -- driver for K1..K3: splice map, word scan, directives,
// per-pass activity, tokens, EOF positions and lexical/preprocessor errors.
//
// Launch sequence (one batch; N bytes, W = N/32 + 1 words, F files):
//   lex_splice          W threads   splice bitmap (preprocess.py:81-95)
//   lex_words           W threads   WScan record per word (exs_lexw.cuh)
//   scan                            WScan inclusive scan (CUB)
//   lex_mark_special    W threads   flag special logical lines
//   lex_count           W threads   plain tokens per word; special-line records
//   lex_special_count   NS threads  special lines: directive records / token counts
//   scan / sort                     token offsets; directives in source order
//   per-file conditional stacks     (preprocess.py:159-203)
//   lex_emit            W threads   32-byte token records in source order
//   lex_special_emit    NS threads  tokens of the special lines
//   per-file EOF / first error      (preprocess.py:203, lexer.py:118-123)
#pragma once
#include "exs_par.cuh"
#include "exs_lexw.cuh"
#include "exs_walk.cuh"

namespace exs {

// segmented sum of depth deltas: the depth mod 2^31 in bits 0-30, the segment
// (view) reset flag in bit 31; depths are only compared with 0 and 1
struct DepthOp {
  EXS_HD u32 operator()(u32 a, u32 b) const {
    if (b & 0x80000000u) return b;
    return (a & 0x80000000u) | ((a + b) & 0x7FFFFFFFu);
  }
};
EXS_HD inline u32 depth_of(u32 x) { return x & 0x7FFFFFFFu; }

struct LexState {
  u32 N = 0, F = 0, W = 0, L = 0, D = 0, T = 0, NS = 0;
  u8* src = nullptr;
  u32* foff = nullptr;      // F+1
  u8* cfg = nullptr;        // F
  u32* fstart = nullptr;    // W bitmap
  u32* splice = nullptr;    // W bitmap
  WScan* wsc = nullptr;     // W inclusive word scan
  u8* wflag = nullptr;      // W: word holds a special byte
  u32* special = nullptr;   // L: logical line holds a special byte (0 / SRec index + 1)
  u32* fnl = nullptr;       // F+1 global newline count before each file
  u32* wtok = nullptr;      // W+1 first token of each word
  u32* ftok = nullptr;      // F+1 first token of each file
  DirRec* dirs = nullptr;   // D, source order
  SRec* srec = nullptr;     // NS special lines, source order
  u32* fdir = nullptr;      // F+1
  u8* dlive = nullptr;      // D: passes live after the directive
  u32* stk = nullptr;       // D
  FP* fp = nullptr;         // 2F
  Tok* toks = nullptr;      // T
  u32* tfile = nullptr;     // T+1 file of every token (handed to the parser)
  u16* tkid = nullptr;      // T+1 kind << 8 | id (handed to the parser)
  u32* tsplit = nullptr;    // F+2 pass-split flags per file, [F]: irregular (handed to the parser)
  u8* arena = nullptr;
  u32* arena_top = nullptr;
  u32 arena_cap = 0;
  u32* cnt = nullptr;       // scratch counters
  void free_all() {
    void* ps[] = {fstart, splice, wsc, wflag, special, fnl, wtok, ftok, dirs, srec, fdir, dlive, stk,
                  fp, toks, arena, arena_top, cnt, foff, cfg, tfile, tkid, tsplit};
    for (void* p : ps) dfree(p);
  }
};

// newlines before byte p (whole corpus)
EXS_HD inline u32 gnl_at(const u8* s, const WScan* wsc, u32 p) {
  u32 w = p >> 5;
  u32 g = w ? (u32)wsc[w - 1].lc : 0;
  for (u32 q = w * 32; q < p; q++) g += s[q] == '\n';
  return g;
}

inline void run_lex(LexState& S, const WalkBufs& WB, Scratch& sc, cudaStream_t st) {
  const u32 N = S.N, F = S.F;
  const u32 W = N / 32 + 1;
  S.W = W;
  S.fstart = dalloc<u32>(W);
  S.splice = dalloc<u32>(W);
  S.cnt = dalloc<u32>(8);
  dzero(S.fstart, W * 4, st);
  dzero(S.splice, W * 4, st);
  dzero(S.cnt, 32, st);
  {
    u32* fs = S.fstart; const u32* fo = S.foff;
    par_for(F, [=] EXS_HD (i64 f) {
      u32 p = fo[f];
      if (p < N && fo[f + 1] > p) at_or(&fs[p >> 5], 1u << (p & 31));
    }, st);
  }
  {
    SrcView v{S.src, S.splice, S.fstart, N};
    u32* sp = S.splice;
    const u8* s = S.src;
    EXS_TAG("lex_splice");
    LexW Xs{};
    Xs.src = S.src; Xs.n = N; Xs.vec = (((uintptr_t)S.src) & 15) == 0;
    par_for(W, [=] EXS_HD (i64 w) {
      const u32 base = (u32)w * 32;
      if (base >= N) { sp[w] = 0; return; }
      u32 r[8];
      load_word(Xs, base, r);
      // candidates: backslashes and newlines of the word (byte-parallel compares)
      u32 bsm = 0, nlm = 0;
      const u32 m = N - base < 32 ? N - base : 32;
#pragma unroll
      for (u32 k = 0; k < 8; k++) {
        bsm |= byte_eq_mask(r[k], '\\') << (4 * k);
        nlm |= byte_eq_mask(r[k], '\n') << (4 * k);
      }
      const u32 valid = m == 32 ? ~0u : ((1u << m) - 1);
      bsm &= valid; nlm &= valid;
      // a newline is spliced only after a backslash (possibly through a run of
      // newlines): none in the word and none carried in from the byte before
      const u8 prev = base ? s[base - 1] : 0;
      if (!bsm && prev != '\\' && prev != '\n') { sp[w] = 0; return; }
      u32 bits = 0, cand = bsm | nlm;
      while (cand) {
        const u32 j = ffs32(cand);
        cand &= cand - 1;
        if (compute_spliced(v, base + j)) bits |= 1u << j;
      }
      sp[w] = bits;
    }, st);
  }
  LexW X{};
  X.src = S.src; X.n = N; X.vec = (((uintptr_t)S.src) & 15) == 0;
  X.sp = S.splice; X.fs = S.fstart;
  X.foff = S.foff; X.F = F; X.cfg = S.cfg;
  // word records and their scan
  S.wsc = dalloc<WScan>(W);
  S.wflag = dalloc<u8>(W);
  {
    WScan* rec = dalloc<WScan>(W);
    u8* wf = S.wflag; u32* nh = S.cnt + 1;
    const LexW Xc = X;
    EXS_TAG("lex_words");
    par_for(W, [=] EXS_HD (i64 w) {
      u8 spc; u32 h;
      rec[w] = word_info(Xc, (u32)w, spc, h);
      wf[w] = spc;
      if (h) at_add(nh, h);
    }, st);
    incl_scan(rec, S.wsc, W, WScanOp(), sc, st);
    dfree(rec);
  }
  X.wsc = S.wsc;
  {
    WScan last = get1(S.wsc + (W - 1), st);
    S.L = (u32)(last.lc >> 32);
  }
  S.special = dalloc<u32>(S.L + 1);
  dzero(S.special, 4ull * (S.L + 1), st);
  X.special = S.special;
  X.nspecial = S.cnt + 3;
  {
    const LexW Xc = X; const u8* wf = S.wflag;
    EXS_TAG("lex_mark_special");
    par_for(W, [=] EXS_HD (i64 w) { if (wf[w]) mark_special(Xc, (u32)w); }, st);
  }
  S.fnl = dalloc<u32>(F + 1);
  {
    const u8* s = S.src; const WScan* wsc = S.wsc; const u32* fo = S.foff; u32* fnl = S.fnl;
    par_for(F + 1, [=] EXS_HD (i64 f) { fnl[f] = gnl_at(s, wsc, fo[f]); }, st);
  }
  X.fnl = S.fnl;
  // count pass: plain tokens per word; special lines recorded by their owner
  S.arena_cap = N + 65536;
  S.arena = dalloc<u8>(S.arena_cap);
  S.arena_top = dalloc<u32>(1);
  dzero(S.arena_top, 4, st);
  const u32 drcap = get1(S.cnt + 1, st) + 1;
  const u32 srcap = get1(S.cnt + 3, st) + 1;
  DirRec* drec = dalloc<DirRec>(drcap);
  SRec* srec = dalloc<SRec>(srcap);
  X.srec = srec; X.nsrec = S.cnt + 4; X.srcap = srcap;
  u32* wcnt = dalloc<u32>(W + 1);
  WordMasks* wmask = dalloc<WordMasks>(W + 1);  // 64 B per word, read back by lex_emit
  X.wm = wmask;
  {
    const LexW Xc = X;
    EXS_TAG("lex_count");
    par_for(W + 1, [=] EXS_HD (i64 w) { wcnt[w] = w == W ? 0 : lex_word<false>(Xc, (u32)w, nullptr, 0); }, st);
  }
  const u32 NS = std::min(get1(S.cnt + 4, st), srcap);
  S.NS = NS;
  if (NS) {
    // K3s: special lines, one thread each (preprocess.py:163-200 + lexer.py:46-118)
    const u8* s = S.src; const u32* sp = S.splice; const u32* fo = S.foff;
    u8* ar = S.arena; u32* at = S.arena_top; const u32 acap = S.arena_cap; u32* nd = S.cnt + 2;
    const LexW Xc = X;
    EXS_TAG("lex_special_count");
    par_for(NS, [=] EXS_HD (i64 k) {
      SRec& r = srec[k];
      const u32 hi = logical_line_end(Xc, r.pos, fo[r.file + 1]);
      LineInfo x = scan_line_directive(s, sp, r.pos, hi, r.lst, ar, at, acap);
      r.kind = x.kind;
      if (x.kind >= LK_IFDEF) {
        r.count = 0;
        u32 d = at_add(nd, 1u);
        if (d < drcap) {
          DirRec q;
          q.pos = r.pos; q.file = r.file; q.line_no = r.line_no;
          q.kind = x.kind; q.macro = x.macro; q.is_ifndef = x.is_ifndef; q.pad = 0; q.span = x.span;
          drec[d] = q;
        }
        return;
      }
      LexErr e;
      r.count = lex_line(s, sp, r.pos, hi, r.lst, r.line_no, r.file, 0, nullptr, &e);
      if (r.count) at_add(&wcnt[r.pos >> 5], r.count);
    }, st);
  }
  S.srec = srec;  // the emit pass finds a line's record through special[line]
  X.srec = S.srec; X.ns = NS;
  S.wtok = dalloc<u32>(W + 1);
  excl_scan_u32(wcnt, S.wtok, W + 1, sc, st);
  S.T = get1(S.wtok + W, st);
  dfree(wcnt);
  // directives in source order
  S.D = std::min(get1(S.cnt + 2, st), drcap);
  const u32 D = S.D;
  S.dirs = dalloc<DirRec>(D + 1);
  if (D) {
    u32* dk = dalloc<u32>(D);
    u32* dv = dalloc<u32>(D);
    par_for(D, [=] EXS_HD (i64 i) { dk[i] = drec[i].pos; dv[i] = (u32)i; }, st);
    sort_pairs(dk, dv, D, sc, st, 32);
    DirRec* ds = S.dirs;
    par_for(D, [=] EXS_HD (i64 i) { ds[i] = drec[dv[i]]; }, st);
    dfree(dk); dfree(dv);
  }
  dfree(drec);
  S.fdir = dalloc<u32>(F + 1);
  S.dlive = dalloc<u8>(D + 1);
  S.stk = dalloc<u32>(D + 1);
  dzero(S.dlive, D + 1, st);
  S.fp = dalloc<FP>(2 * (size_t)F + 2);
  {
    const DirRec* dr = S.dirs; u32* fd = S.fdir;
    par_for(F + 1, [=] EXS_HD (i64 f) {
      u32 lo = 0, hi = D;
      while (lo < hi) { u32 mid = (lo + hi) / 2; if (dr[mid].file < f) lo = mid + 1; else hi = mid; }
      fd[f] = lo;
    }, st);
  }
  {
    // per-file conditional stack for both passes (preprocess.py:159-203)
    const u32* fd = S.fdir; const DirRec* dr = S.dirs;
    const u8* cf = S.cfg; u8* live_out = S.dlive; u32* stk = S.stk; FP* fp = S.fp;
    par_for(F, [=] EXS_HD (i64 f) {
      u32 d0 = fd[f], d1 = fd[f + 1];
      u8 c = cf[f];
      u8 np = file_passes(c);
      for (u32 p = 0; p < 2; p++) {
        FP& r = fp[2 * f + p];
        r.pp_line = NONE; r.pp_msg = 0; r.pp_a0 = 0; r.pp_a1 = 0;
        r.lex_line = NONE; r.lex_col = 0; r.lex_msg = 0; r.lex_pos = NONE;
        r.view = NONE; r.perr = 0; r.eof_line = 1; r.eof_col = 1;
        if (!((np >> p) & 1)) { r.pp_line = NONE - 1; continue; }  // pass does not exist
        u8 defined = 0;
        if (!(c & CFG_PLAIN)) {
          defined = MAC_CUDACC | ((c & CFG_RELAXED) ? MAC_RELAXED : 0) | (p ? MAC_CUDA_ARCH : 0);
        }
        bool live = true;
        u32 depth = 0;
        for (u32 d = d0; d < d1; d++) {
          const DirRec& x = dr[d];
          u16 msg = 0; u64 a0 = 0; u32 a1 = 0;
          switch (x.kind) {
            case LK_BAD_ARITY: msg = M_PP_EXPECTS_ONE; a1 = x.is_ifndef; break;
            case LK_BAD_MACRO: msg = M_PP_UNKNOWN_MACRO; a0 = x.span; a1 = x.is_ifndef; break;
            case LK_UNKNOWN: msg = M_PP_UNKNOWN_DIRECTIVE; a0 = x.span; break;
            case LK_IFDEF:
            case LK_IFNDEF: {
              bool cond = ((x.macro & defined) != 0) == (x.kind == LK_IFDEF);
              stk[d0 + depth] = (live ? 1u : 0u) | (cond ? 2u : 0u) | (d << 3);
              depth++;
              live = live && cond;
              break;
            }
            case LK_ELSE: {
              if (!depth) { msg = M_PP_ELSE_NOMATCH; break; }
              u32& t = stk[d0 + depth - 1];
              if (t & 4) { msg = M_PP_SECOND_ELSE; break; }
              t |= 4;
              t ^= 2;
              live = (t & 1) && (t & 2);
              break;
            }
            case LK_ENDIF:
              if (!depth) { msg = M_PP_ENDIF_NOMATCH; break; }
              depth--;
              live = stk[d0 + depth] & 1;
              break;
            case LK_ERROR:
              if (live) { msg = M_PP_ERROR; a0 = x.span; }
              break;
            default: break;
          }
          if (msg) { r.pp_line = x.line_no; r.pp_msg = msg; r.pp_a0 = a0; r.pp_a1 = a1; break; }
          if (live) live_out[d] |= (u8)(1u << p); else live_out[d] &= (u8)~(1u << p);
        }
        if (r.pp_line == NONE && depth) {
          r.pp_line = dr[stk[d0 + depth - 1] >> 3].line_no;
          r.pp_msg = M_PP_UNTERMINATED;
        }
      }
    }, st);
  }
  // emit pass
  S.toks = dalloc<Tok>((size_t)S.T + 1);
  S.tfile = dalloc<u32>((size_t)S.T + 1);
  S.tkid = dalloc<u16>((size_t)S.T + 1);
  S.tsplit = dalloc<u32>((size_t)F + 2);
  dzero(S.tsplit, 4ull * (F + 2), st);
  X.tfile = S.tfile; X.tkid = S.tkid; X.tsplit = S.tsplit;
  X.fdir = S.fdir; X.dirs = S.dirs; X.dlive = S.dlive; X.fp = S.fp;
  {
    const LexW Xc = X; const u32* wt = S.wtok; Tok* tk = S.toks;
    EXS_TAG("lex_emit");
    par_for(W, [=] EXS_HD (i64 w) { lex_word<true>(Xc, (u32)w, tk + wt[w], wt[w]); }, st);
  }
  dfree(wmask);
  X.wm = nullptr;
  if (S.NS) {
    const u8* s = S.src; const u32* sp = S.splice; const u32* fo = S.foff; const SRec* sr = S.srec;
    Tok* tk = S.toks; FP* fp = S.fp;
    const LexW Xc = X;
    EXS_TAG("lex_special_emit");
    par_for(S.NS, [=] EXS_HD (i64 k) {
      const SRec& r = sr[k];
      if (r.kind >= LK_IFDEF) return;
      const u32 hi = logical_line_end(Xc, r.pos, fo[r.file + 1]);
      LexErr e;
      lex_line(s, sp, r.pos, hi, r.lst, r.line_no, r.file, r.mask, tk + r.slot, &e);
      for (u32 q = 0; q < r.count; q++) tok_meta(Xc, r.slot + q, tk[r.slot + q]);
      if (e.msg)
        for (u32 p = 0; p < 2; p++)
          if ((r.mask >> p) & 1u) at_min(&fp[2 * r.file + p].lex_pos, e.pos);
    }, st);
  }
  S.ftok = dalloc<u32>(F + 1);
  {
    const Tok* tk = S.toks; u32* ft = S.ftok; const u32 T = S.T;
    par_for(F + 1, [=] EXS_HD (i64 f) {
      u32 lo = 0, hi = T;  // first token of a file >= f
      while (lo < hi) { u32 mid = (lo + hi) / 2; if (tk[mid].file < f) lo = mid + 1; else hi = mid; }
      ft[f] = lo;
    }, st);
  }
  // EOF positions and first errors per (file, pass)
  {
    const u8* s = S.src; const u32* sp = S.splice; const u32* fo = S.foff; const u32* fnl = S.fnl;
    const WScan* wsc = S.wsc; const u32* fd = S.fdir; const DirRec* dr = S.dirs; const u8* dl = S.dlive;
    FP* fp = S.fp;
    WalkBufs B = WB;
    par_for(F, [=] EXS_HD (i64 f) {
      const u32 f0 = fo[f], fend = fo[f + 1];
      for (u32 p = 0; p < 2; p++) {
        FP& r = fp[2 * f + p];
        if (r.pp_line == NONE - 1) continue;  // no such pass
        if (r.pp_line != NONE) {
          emit_diag(B, mkdiag((u32)f, r.pp_line, 1, C_E0002, r.pp_msg, r.pp_a0, 0, 0, r.pp_a1));
          continue;
        }
        if (r.lex_pos != NONE) {
          const u32 pos = r.lex_pos;
          u32 lo = pos;
          while (lo > f0 && !(s[lo - 1] == '\n' && !bit_get(sp, lo - 1))) lo--;
          u32 col = 1;
          for (u32 q = lo; q < pos; q++)
            if (!bit_get(sp, q) && !is_cont_byte(s[q])) col++;
          const u8 c = s[pos];
          r.lex_line = 1 + gnl_at(s, wsc, lo) - fnl[f];
          r.lex_col = col;
          r.lex_msg = c == '"' ? M_LEX_STRING : (c == '#' ? M_LEX_PRAGMA : M_LEX_CHAR);
          emit_diag(B, mkdiag((u32)f, r.lex_line, col, C_E0001, r.lex_msg, ((u64)pos << 32) | 1));
          continue;
        }
        if (f0 == fend) { r.eof_line = 1; r.eof_col = 1; continue; }
        r.eof_line = 1 + gnl_at(s, wsc, fend) - fnl[f];
        if (s[fend - 1] == '\n' && !bit_get(sp, fend - 1)) { r.eof_col = 1; continue; }
        u32 lo = fend;  // last logical line [lo, fend)
        while (lo > f0 && !(s[lo - 1] == '\n' && !bit_get(sp, lo - 1))) lo--;
        bool one = false;
        for (u32 q = lo; q < fend && !one; q++) one = bit_get(sp, q);
        const u32 d0 = fd[f], d1 = fd[f + 1];
        if (!one && d1 > d0) {
          u32 d = d1 - 1;
          if (dr[d].pos == lo) one = true;                      // a directive line
          else if (!((dl[d] >> p) & 1)) one = true;             // inactive in this pass
        }
        if (one) { r.eof_col = 1; continue; }
        u32 cps = 0;
        for (u32 q = lo; q < fend; q++) cps += !is_cont_byte(s[q]);
        r.eof_col = 1 + cps;
      }
    }, st);
  }
  sync(st);
}

}  // namespace exs
