// exs_stage_lex.cuh -- driver for K1..K3 (splice map, logical lines, comment
// state scan, directives, per-pass activity, tokens, EOF positions).
#pragma once
#include "exs_par.cuh"
#include "exs_lex.cuh"
#include "exs_walk.cuh"

namespace exs {

// per (file, pass) status -- fp = 2*file + pass (pass 0 host, 1 device)
struct FP {
  u32 pp_line;    // directive line index of the first E0002 (NONE = ok)
  u16 pp_msg;
  u16 pad;
  u64 pp_a0;      // text span / flags for the message
  u32 pp_a1;
  u32 lex_line;   // first line (index) with a lexical error active in this pass
  u32 eof_line, eof_col;
  u32 view;       // view serving this pass (NONE if none)
  u32 perr;       // parse failed (1) / ok (0)
};

struct LineScanOp {
  // element: bit0-1 fsm map, bit2 reset (first line of a file), bits 8.. newline count
  EXS_HD u64 operator()(u64 a, u64 b) const {
    if (b & 4) return b;
    u64 am = a & 3, bm = b & 3;
    // compose: state after (a then b) from CODE: bm bit [am&1]; from BLOCK: bm bit [(am>>1)&1]
    u64 m0 = (bm >> (am & 1)) & 1;
    u64 m1 = (bm >> ((am >> 1) & 1)) & 1;
    u64 nl = (a >> 8) + (b >> 8);
    return (nl << 8) | (a & 4) | (m1 << 1) | m0;
  }
};

struct DepthOp {  // segmented sum of (depth delta) with reset flag in bit 32
  EXS_HD i64 operator()(i64 a, i64 b) const {
    if (b & (1ll << 40)) return b;
    i64 v = (a & 0xFFFFFFFFll) + (b & 0xFFFFFFFFll);
    return (a & (1ll << 40)) | (v & 0xFFFFFFFFll);
  }
};

struct LexState {
  u32 N = 0, F = 0, L = 0, D = 0, T = 0;
  u8* src = nullptr;
  u32* foff = nullptr;      // F+1
  u8* cfg = nullptr;        // F
  u32* fstart = nullptr;
  u32* splice = nullptr;
  u32* line_start = nullptr, *line_file = nullptr, *line_hi = nullptr, *line_no = nullptr;
  u8* line_st = nullptr;    // comment state at line start (S_CODE/S_BLOCK)
  u64* line_scan = nullptr;
  LineInfo* line_info = nullptr;
  u8* line_mask = nullptr;
  u32* line_ntok = nullptr, *line_tok = nullptr;
  u16* line_err = nullptr;
  u32* line_err_col = nullptr, *line_err_pos = nullptr;
  u32* fline = nullptr;     // F+1 first line of each file
  u32* dir_line = nullptr;  // D
  u32* fdir = nullptr;      // F+1
  u8* dir_live = nullptr;   // D
  u32* stk = nullptr;       // D
  FP* fp = nullptr;         // 2F
  Tok* toks = nullptr;      // T
  u8* arena = nullptr;
  u32* arena_top = nullptr;
  u32 arena_cap = 0;
  u32* cnt = nullptr;       // scratch counter
  void free_all() {
    void* ps[] = {fstart, splice, line_start, line_file, line_hi, line_no, line_st, line_scan,
                  line_info, line_mask, line_ntok, line_tok, line_err, line_err_col, line_err_pos,
                  fline, dir_line, fdir, dir_live, stk, fp, toks, arena, arena_top, cnt,
                  foff, cfg};
    for (void* p : ps) dfree(p);
  }
};

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

inline void run_lex(LexState& S, const WalkBufs& WB, Scratch& sc, cudaStream_t st) {
  const u32 N = S.N, F = S.F;
  const u32 W = N / 32 + 1;
  S.fstart = dalloc<u32>(W);
  S.splice = dalloc<u32>(W);
  S.cnt = dalloc<u32>(4);
  dzero(S.fstart, W * 4, st);
  dzero(S.splice, W * 4, st);
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
    par_for(W, [=] EXS_HD (i64 w) {
      u32 bits = 0;
      u32 base = (u32)w * 32;
      for (u32 j = 0; j < 32 && base + j < N; j++) {
        u8 c = s[base + j];
        if ((c == '\\' || c == '\n') && compute_spliced(v, base + j)) bits |= 1u << j;
      }
      sp[w] = bits;
    }, st);
  }
  // logical line starts
  S.line_start = dalloc<u32>(N + 1);
  {
    const u32* fs = S.fstart; const u32* sp = S.splice; const u8* s = S.src;
    auto pred = [=] EXS_HD (u32 p) -> bool {
      if ((fs[p >> 5] >> (p & 31)) & 1u) return true;
      return p > 0 && s[p - 1] == '\n' && !((sp[(p - 1) >> 5] >> ((p - 1) & 31)) & 1u);
    };
    S.L = select_idx(N, pred, S.line_start, S.cnt, sc, st);
  }
  const u32 L = S.L;
  S.line_file = dalloc<u32>(L + 1);
  S.line_hi = dalloc<u32>(L + 1);
  S.line_no = dalloc<u32>(L + 1);
  S.line_st = dalloc<u8>(L + 1);
  S.line_scan = dalloc<u64>(L + 1);
  S.fline = dalloc<u32>(F + 1);
  {
    const u32* ls = S.line_start; u32* lf = S.line_file; u32* lh = S.line_hi; u64* sc_in = S.line_scan;
    const u32* fo = S.foff; const u8* s = S.src; const u32* sp = S.splice;
    EXS_TAG("lex_line_map");
    par_for(L, [=] EXS_HD (i64 i) {
      u32 lo = ls[i];
      u32 f = upper_file(fo, F, lo);
      lf[i] = f;
      u32 fend = fo[f + 1];
      u32 hi;
      bool term;
      if (i + 1 < L && ls[i + 1] < fend) { hi = ls[i + 1] - 1; term = true; }
      else if (fend > lo && s[fend - 1] == '\n' && !((sp[(fend - 1) >> 5] >> ((fend - 1) & 31)) & 1u)) { hi = fend - 1; term = true; }
      else { hi = fend; term = false; }
      lh[i] = hi;
      u64 nl = term ? 1 : 0;
      for (u32 q = lo; q < hi; q++) if (s[q] == '\n') nl++;
      u8 m = line_fsm_map(s, sp, lo, hi);
      bool first = (i == 0) || (lf[i] != upper_file(fo, F, ls[i - 1]));
      sc_in[i] = (nl << 8) | (first ? 4 : 0) | m;
    }, st);
  }
  {
    u64* tmp = dalloc<u64>(L + 1);
    incl_scan(S.line_scan, tmp, L, LineScanOp(), sc, st);
    const u64* inc = tmp; const u64* el = S.line_scan;
    u32* lno = S.line_no; u8* lst = S.line_st;
    par_for(L, [=] EXS_HD (i64 i) {
      bool first = (el[i] & 4) != 0;
      if (first) { lno[i] = 1; lst[i] = S_CODE; return; }
      u64 prev = inc[i - 1];
      lno[i] = 1 + (u32)(prev >> 8);
      lst[i] = (prev & 1) ? S_BLOCK : S_CODE;  // state from CODE at file start
    }, st);
    sync(st);
    dfree(tmp);
  }
  {
    // first line of each file
    const u32* lf = S.line_file; u32* fl = S.fline;
    par_for(F + 1, [=] EXS_HD (i64 f) {
      u32 lo = 0, hi = L;  // first line with file >= f
      while (lo < hi) { u32 mid = (lo + hi) / 2; if (lf[mid] < f) lo = mid + 1; else hi = mid; }
      fl[f] = lo;
    }, st);
  }
  // directives
  S.arena_cap = N + 65536;
  S.arena = dalloc<u8>(S.arena_cap);
  S.arena_top = dalloc<u32>(1);
  dzero(S.arena_top, 4, st);
  S.line_info = dalloc<LineInfo>(L + 1);
  S.line_ntok = dalloc<u32>(L + 1);
  S.line_tok = dalloc<u32>(L + 2);
  S.line_err = dalloc<u16>(L + 1);
  S.line_err_col = dalloc<u32>(L + 1);
  S.line_err_pos = dalloc<u32>(L + 1);
  {
    // one pass per logical line: directive detection + token count (the
    // count does not depend on pass activity: tokens of inactive lines are
    // emitted with an empty pass mask and ignored downstream)
    const u32* ls = S.line_start; const u32* lh = S.line_hi; const u8* lst = S.line_st;
    const u32* lno = S.line_no; const u32* lf = S.line_file;
    const u8* s = S.src; const u32* sp = S.splice; LineInfo* li = S.line_info;
    u8* ar = S.arena; u32* at = S.arena_top; u32 cap = S.arena_cap;
    u32* nt = S.line_ntok; u16* le = S.line_err; u32* lec = S.line_err_col; u32* lep = S.line_err_pos;
    EXS_TAG("lex_directive_count");
    par_for_walk(L + 1, [=] EXS_HD (i64 i) {
      if (i == L) { nt[i] = 0; return; }
      LineInfo x = scan_line_directive(s, sp, ls[i], lh[i], lst[i], ar, at, cap);
      li[i] = x;
      if (x.kind >= LK_IFDEF) { nt[i] = 0; le[i] = 0; return; }
      LexErr e;
      nt[i] = lex_line(s, sp, ls[i], lh[i], lst[i], lno[i], lf[i], 0, nullptr, &e);
      le[i] = e.msg;
      lec[i] = e.col;
      lep[i] = e.pos;
    }, st);
  }
  excl_scan_u32(S.line_ntok, S.line_tok, L + 1, sc, st);
  S.T = get1(S.line_tok + L, st);
  S.dir_line = dalloc<u32>(L + 1);
  {
    const LineInfo* li = S.line_info;
    auto pred = [=] EXS_HD (u32 i) -> bool { return li[i].kind >= LK_IFDEF; };
    S.D = select_idx(L, pred, S.dir_line, S.cnt, sc, st);
  }
  const u32 D = S.D;
  S.fdir = dalloc<u32>(F + 1);
  S.dir_live = dalloc<u8>(D + 1);
  S.stk = dalloc<u32>(D + 1);
  dzero(S.dir_live, D + 1, st);
  S.fp = dalloc<FP>(2 * (size_t)F + 2);
  {
    const u32* dl = S.dir_line; const u32* lf = S.line_file; u32* fd = S.fdir;
    par_for(F + 1, [=] EXS_HD (i64 f) {
      u32 lo = 0, hi = D;
      while (lo < hi) { u32 mid = (lo + hi) / 2; if (lf[dl[mid]] < f) lo = mid + 1; else hi = mid; }
      fd[f] = lo;
    }, st);
  }
  {
    // per-file conditional stack for both passes (preprocess.py:159-203)
    const u32* fd = S.fdir; const u32* dl = S.dir_line; const LineInfo* li = S.line_info;
    const u8* cf = S.cfg; u8* live_out = S.dir_live; u32* stk = S.stk; FP* fp = S.fp;
    par_for(F, [=] EXS_HD (i64 f) {
      u32 d0 = fd[f], d1 = fd[f + 1];
      u8 c = cf[f];
      u8 np = file_passes(c);
      for (u32 p = 0; p < 2; p++) {
        FP& r = fp[2 * f + p];
        r.pp_line = NONE; r.pp_msg = 0; r.pp_a0 = 0; r.pp_a1 = 0;
        r.lex_line = NONE; r.view = NONE; r.perr = 0; r.eof_line = 1; r.eof_col = 1;
        if (!((np >> p) & 1)) { r.pp_line = NONE - 1; continue; }  // pass does not exist
        u8 defined = 0;
        if (!(c & CFG_PLAIN)) {
          defined = MAC_CUDACC | ((c & CFG_RELAXED) ? MAC_RELAXED : 0) | (p ? MAC_CUDA_ARCH : 0);
        }
        bool live = true;
        u32 depth = 0;
        for (u32 d = d0; d < d1; d++) {
          const LineInfo& x = li[dl[d]];
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
          if (msg) { r.pp_line = dl[d]; r.pp_msg = msg; r.pp_a0 = a0; r.pp_a1 = a1; break; }
          if (live) live_out[d] |= (u8)(1u << p); else live_out[d] &= (u8)~(1u << p);
        }
        if (r.pp_line == NONE && depth) {
          r.pp_line = dl[stk[d0 + depth - 1] >> 3];
          r.pp_msg = M_PP_UNTERMINATED;
        }
      }
    }, st);
  }
  // per-line activity mask
  S.line_mask = dalloc<u8>(L + 1);
  {
    const u32* lf = S.line_file; const u32* fd = S.fdir; const u32* dl = S.dir_line;
    const u8* live = S.dir_live; const LineInfo* li = S.line_info; const u8* cf = S.cfg;
    const FP* fp = S.fp; u8* lm = S.line_mask;
    par_for(L, [=] EXS_HD (i64 i) {
      u32 f = lf[i];
      u8 m = file_passes(cf[f]);
      for (u32 p = 0; p < 2; p++)
        if (fp[2 * f + p].pp_line != NONE) m &= (u8)~(1u << p);
      if (li[i].kind >= LK_IFDEF) { lm[i] = 0; return; }
      u32 d0 = fd[f], d1 = fd[f + 1];
      if (d0 < d1 && dl[d0] < (u32)i) {
        // last directive before line i
        u32 lo = d0, hi = d1;
        while (hi - lo > 1) { u32 mid = (lo + hi) / 2; if (dl[mid] < (u32)i) lo = mid; else hi = mid; }
        m &= live[lo];
      }
      lm[i] = m;
    }, st);
  }
  // tokens: emit (counts and offsets come from the directive pass)
  S.toks = dalloc<Tok>((size_t)S.T + 1);
  {
    const u32* ls = S.line_start; const u32* lh = S.line_hi; const u8* lst = S.line_st;
    const u32* lno = S.line_no; const u32* lf = S.line_file; const u8* lm = S.line_mask;
    const u8* s = S.src; const u32* sp = S.splice; const u32* lt = S.line_tok; Tok* tk = S.toks;
    const u16* le = S.line_err; const u32* nt = S.line_ntok; FP* fp = S.fp;
    EXS_TAG("lex_emit");
    par_for_walk(L, [=] EXS_HD (i64 i) {
      if (!nt[i] && !le[i]) return;
      u8 m = lm[i];
      LexErr e;
      lex_line(s, sp, ls[i], lh[i], lst[i], lno[i], lf[i], m, tk + lt[i], &e);
      if (e.msg) {
        u32 f = lf[i];
        for (u32 p = 0; p < 2; p++)
          if ((m >> p) & 1) at_min(&fp[2 * f + p].lex_line, (u32)i);
      }
    }, st);
  }
  // EOF positions and first errors per (file, pass)
  {
    const u32* fl = S.fline; const u32* lno = S.line_no; const u32* lh = S.line_hi;
    const u32* ls = S.line_start; const u64* el = S.line_scan; const LineInfo* li = S.line_info;
    const u8* lm = S.line_mask; const u32* fo = S.foff; const u8* s = S.src; const u32* sp = S.splice;
    const u16* le = S.line_err; const u32* lec = S.line_err_col; const u32* lep = S.line_err_pos;
    FP* fp = S.fp;
    WalkBufs B = WB;
    par_for(F, [=] EXS_HD (i64 f) {
      u32 l0 = fl[f], l1 = fl[f + 1];
      u32 fend = fo[f + 1];
      for (u32 p = 0; p < 2; p++) {
        FP& r = fp[2 * f + p];
        if (r.pp_line == NONE - 1) continue;  // no such pass
        if (r.pp_line != NONE) {
          emit_diag(B, mkdiag((u32)f, lno[r.pp_line], 1, C_E0002, r.pp_msg, r.pp_a0, 0, 0, r.pp_a1));
          continue;
        }
        if (r.lex_line != NONE) {
          u32 L_ = r.lex_line;
          emit_diag(B, mkdiag((u32)f, lno[L_], lec[L_], C_E0001, le[L_], ((u64)lep[L_] << 32) | 1));
          continue;
        }
        if (l0 == l1) { r.eof_line = 1; r.eof_col = 1; continue; }
        u32 last = l1 - 1;
        u32 total_nl = lno[last] - 1 + (u32)(el[last] >> 8);
        r.eof_line = 1 + total_nl;
        bool ends_nl = fend > ls[l0] && s[fend - 1] == '\n' &&
                       !((sp[(fend - 1) >> 5] >> ((fend - 1) & 31)) & 1u);
        if (ends_nl || li[last].has_splice || li[last].kind >= LK_IFDEF || !((lm[last] >> p) & 1))
          r.eof_col = 1;
        else
          r.eof_col = 1 + li[last].cps;
        (void)lh;
      }
    }, st);
  }
  sync(st);
}

}  // namespace exs
