// exs_parse.cuh -- K4: recursive-descent MiniCU parser over one view's tokens,
// building the flat AST (reference: syntax/parser.py:56-659).  One thread runs
// parse_item() from each top-level item start found by the token-parallel
// segmentation; a view whose items do not chain exactly is re-parsed
// sequentially by one thread (same code).
#pragma once
#include "exs_common.cuh"

namespace exs {

// expectation strings of expect() (parser.py:77-82) -- rendered by messages.py
enum Expect : u8 {
  EX_NONE = 0, EX_ENUM, EX_CLASS, EX_HDC_NAME, EX_LBRACE, EX_COMMA, EX_ENUM_HST, EX_ENUM_DEV,
  EX_ENUM_HSTDEV, EX_RBRACE, EX_SEMI, EX_STATIC_ASSERT, EX_LPAREN, EX_RPAREN, EX_TEMPLATE,
  EX_LT, EX_GT, EX_REQUIRES, EX_FN_BODY, EX_FOR, EX_INT, EX_ASSIGN, EX_INC, EX_GGG,
};
// expect_ident() "what" strings
enum NameWhat : u8 {
  NW_NONE = 0, NW_TPARAM, NW_STRUCT, NW_MEMBER, NW_FUNCTION, NW_PARAM, NW_TYPE, NW_TARG,
  NW_VARIABLE, NW_LOOPVAR,
};

struct PView {
  const Tok* toks;
  const u32* vtok;  // view token list (global token indices)
  u32 vbase, n;     // view tokens are vtok[vbase .. vbase+n)
  u32 eof_line, eof_col;
  u8 spec_mode;     // 0 keep, 1 erase, 2 reject (spacecheck.py:697-699)
  const u16* vkid;  // kind << 8 | id per view token: the parser's hot reads,
                    // 2 bytes and one load instead of a 32-byte record via vtok
};

struct PErr {
  u32 line, col;
  u16 msg;
  u64 a0, a1;  // expectation / name-what ids, or token text spans
};

#define SPAN_EOF 0xFFFFFFFFFFFFFFFFull
#define MAX_PARSE_DEPTH 200

struct Parser {
  PView v;
  u32 pos;
  Node* nodes;
  u32 nbase, nused, ncap;
  bool failed;
  bool overflow;
  PErr e;
  int depth;

  u32 defer_open, defer_close;  // view positions of a body parsed separately (or NONE)
  bool deferred;
  u32 block_stmts;              // statements of the last block parsed

  EXS_HD void init(const PView& view, Node* nd, u32 base, u32 cap, u32 start) {
    v = view; nodes = nd; nbase = base; nused = 0; ncap = cap; pos = start;
    failed = false; overflow = false; depth = 0;
    defer_open = NONE; defer_close = NONE; deferred = false;
    e.line = e.col = 0; e.msg = 0; e.a0 = e.a1 = 0;
  }

  // ------------------------------------------------------------ tokens
  // view position -> global token index
  EXS_HD u32 tix(u32 i) const { return v.vtok[v.vbase + i]; }
  EXS_HD u32 gtok(u32 i) const { return i < v.n ? tix(i) : NONE; }
  EXS_HD u8 kind(u32 k = 0) const {
    u32 i = pos + k;
    return i < v.n ? (u8)(v.vkid[v.vbase + i] >> 8) : (u8)TK_EOF;
  }
  EXS_HD u8 tid(u32 k = 0) const {
    u32 i = pos + k;
    return i < v.n ? (u8)v.vkid[v.vbase + i] : (u8)0;
  }
  // at(text): kind in (ident, punct) and text equal (parser.py:67-69)
  EXS_HD bool at_w(u8 w, u32 k = 0) const { return kind(k) == TK_IDENT && tid(k) == w; }
  EXS_HD bool at_p(u8 p, u32 k = 0) const { return kind(k) == TK_PUNCT && tid(k) == p; }
  EXS_HD bool is_kw(u32 k = 0) const {
    return kind(k) == TK_IDENT && tid(k) >= 1 && tid(k) <= W_LAST_KEYWORD;
  }
  EXS_HD u32 take() {
    u32 g = gtok(pos);
    if (pos < v.n) pos++;
    return g;
  }
  EXS_HD void loc_of(u32 i, u32& line, u32& col) const {
    if (i < v.n) { const Tok& t = v.toks[tix(i)]; line = t.line; col = t.col; }
    else { line = v.eof_line; col = v.eof_col; }
  }
  EXS_HD u64 span_of(u32 i) const {
    if (i >= v.n) return SPAN_EOF;
    const Tok& t = v.toks[tix(i)];
    return ((u64)t.pos << 32) | (u64)(t.end - t.pos);
  }

  // ------------------------------------------------------------ errors
  // error paths are cold: out of line to keep the parse kernels' instruction
  // footprint small
  EXS_HD EXS_NOINLINE bool fail_at(u32 tokpos, u16 msg, u64 a0 = 0, u64 a1 = 0) {
    if (!failed) {
      failed = true;
      loc_of(tokpos, e.line, e.col);
      e.msg = msg; e.a0 = a0; e.a1 = a1;
    }
    return false;
  }
  EXS_HD EXS_NOINLINE bool fail_tok(u32 gt, u16 msg, u64 a0 = 0, u64 a1 = 0) {
    // error located at a global token (already consumed)
    if (!failed) {
      failed = true;
      const Tok& t = v.toks[gt];
      e.line = t.line; e.col = t.col; e.msg = msg; e.a0 = a0; e.a1 = a1;
    }
    return false;
  }
  EXS_HD u64 gspan(u32 gt) const {
    const Tok& t = v.toks[gt];
    return ((u64)t.pos << 32) | (u64)(t.end - t.pos);
  }
  // failure at the current token with its text span (out of line, cold)
  EXS_HD EXS_NOINLINE bool fail_here(u16 msg, u64 a0) { return fail_at(pos, msg, a0, span_of(pos)); }
  // expect(text[, what]) -- tokens of kind ident/punct with the given id
  EXS_HD bool need_p(u8 p, u8 ex) {
    if (at_p(p)) { take(); return true; }
    return fail_here(M_P_EXPECTED, ex);
  }
  EXS_HD bool need_w(u8 w, u8 ex) {
    if (at_w(w)) { take(); return true; }
    return fail_here(M_P_EXPECTED, ex);
  }
  EXS_HD bool need_name(u8 what, u32& gt) {
    if (kind() != TK_IDENT || is_kw()) return fail_here(M_P_EXPECTED_NAME, what);
    gt = take();
    return true;
  }

  // ------------------------------------------------------------ nodes
  EXS_HD u32 mk(u8 k, u32 tok) {
    if (nused >= ncap) { overflow = true; failed = true; e.msg = M_X_CONTRACT; return NONE; }
    u32 id = nbase + nused++;
    Node& n = nodes[id];
    n.kind = k; n.sub = 0; n.n = 0; n.tok = tok; n.c0 = n.c1 = n.c2 = NONE; n.next = NONE;
    n.hv = tok != NONE ? v.toks[tok].hv : 0;
    return id;
  }
  EXS_HD Node& N(u32 id) { return nodes[id]; }

  struct ListB {
    u32 head = NONE, tail = NONE, count = 0;
  };
  EXS_HD void push(ListB& l, u32 id) {
    if (l.tail == NONE) l.head = id; else nodes[l.tail].next = id;
    l.tail = id; l.count++;
  }

  EXS_HD bool enter() {
    if (++depth > MAX_PARSE_DEPTH) return fail_at(pos, M_P_DEPTH);
    return true;
  }

  // ------------------------------------------------------------ items
  // returns root node id, or NONE on failure
  EXS_HD bool pragma_opt(u8& pragma) {
    pragma = 0;
    if (kind() != TK_PRAGMA) return true;
    u32 t = take();
    u8 id = v.toks[t].id;
    if (id != W_HD_WARNING_DISABLE && id != W_NV_EXEC_CHECK_DISABLE)
      return fail_tok(t, M_P_UNKNOWN_PRAGMA, gspan(t));
    pragma = id == W_HD_WARNING_DISABLE ? 1 : 2;
    return true;
  }

  EXS_HD u32 item() {
    u8 pragma;
    if (!pragma_opt(pragma)) return NONE;
    if (at_w(W_ENUM) || at_w(W_STATIC_ASSERT)) {
      if (pragma) { fail_at(pos, M_P_PRAGMA_FN); return NONE; }
      return at_w(W_ENUM) ? enum_item() : assert_item();
    }
    u32 tps = NONE, req = NONE;
    if (at_w(W_TEMPLATE)) {
      if (!template_header(tps)) return NONE;
      if (at_w(W_REQUIRES) && !requires_clause(req)) return NONE;
    }
    u16 sflags = 0; u32 hp = NONE, dp = NONE;
    if (!specifiers(sflags, hp, dp)) return NONE;
    if (at_w(W_STRUCT) || at_w(W_CLASS)) {
      if (pragma) { fail_at(pos, M_P_PRAGMA_FN); return NONE; }
      if (req != NONE) { fail_at(pos, M_P_REQ_STRUCT); return NONE; }
      return struct_(tps, sflags, hp, dp);
    }
    return function(tps, req, sflags, hp, dp, pragma, false, NONE, false);
  }

  EXS_HD u32 enum_item() {
    u32 t = take();
    if (!need_w(W_CLASS, EX_CLASS) || !need_w(W_HDC, EX_HDC_NAME) || !need_p(P_LBRACE, EX_LBRACE)) return NONE;
    if (!need_w(W_HST, EX_ENUM_HST) || !need_p(P_COMMA, EX_COMMA) || !need_w(W_DEV, EX_ENUM_DEV) ||
        !need_p(P_COMMA, EX_COMMA) || !need_w(W_HSTDEV, EX_ENUM_HSTDEV))
      return NONE;
    if (!need_p(P_RBRACE, EX_RBRACE) || !need_p(P_SEMI, EX_SEMI)) return NONE;
    return mk(N_ENUM, t);
  }

  EXS_HD u32 assert_item() {
    u32 t = take();
    if (!need_p(P_LPAREN, EX_LPAREN)) return NONE;
    u32 ex = expr();
    if (ex == NONE) return NONE;
    if (!need_p(P_RPAREN, EX_RPAREN) || !need_p(P_SEMI, EX_SEMI)) return NONE;
    u32 id = mk(N_ASSERT, t);
    if (id != NONE) N(id).c0 = ex;
    return id;
  }

  EXS_HD bool template_header(u32& out) {
    take();  // template
    if (!need_p(P_LT, EX_LT)) return false;
    ListB l;
    int ntype = 0, nhdc = 0;
    u32 last_name = NONE;
    while (true) {
      u32 here = pos;
      if (at_w(W_TYPENAME)) {
        take();
        u32 nm;
        if (!need_name(NW_TPARAM, nm)) return false;
        u32 id = mk(N_TPARAM, nm);
        if (id == NONE) return false;
        N(id).sub = 0;  // type
        push(l, id);
        ntype++;
        last_name = nm;
      } else if (at_w(W_HDC)) {
        take();
        u32 nm;
        if (!need_name(NW_TPARAM, nm)) return false;
        u32 dflt = NONE;
        if (at_p(P_ASSIGN)) {
          take();
          dflt = expr();
          if (dflt == NONE) return false;
        }
        u32 id = mk(N_TPARAM, nm);
        if (id == NONE) return false;
        N(id).sub = 1;  // hdc
        N(id).c0 = dflt;
        push(l, id);
        nhdc++;
        last_name = nm;
      } else {
        return fail_at(here, M_P_TPARAM_KIND);
      }
      if (!at_p(P_COMMA)) break;
      take();
    }
    if (!need_p(P_GT, EX_GT)) return false;
    if (ntype > 1 || nhdc > 1) return fail_tok(last_name, M_P_TPARAM_LIMIT);
    out = l.head;
    return true;
  }

  EXS_HD bool requires_clause(u32& out) {
    take();
    if (!need_p(P_LPAREN, EX_LPAREN)) return false;
    out = expr();
    if (out == NONE) return false;
    return need_p(P_RPAREN, EX_RPAREN);
  }

  // parse_specifiers (parser.py:201-236); flags use FF_H/FF_D/FF_G/FF_CX
  EXS_HD bool specifiers(u16& flags, u32& hp, u32& dp) {
    flags = 0; hp = dp = NONE;
    u8 seen = 0;
    u32 last = pos;
    while (true) {
      last = pos;
      if (kind() == TK_IDENT && (tid() == W_HOST || tid() == W_DEVICE || tid() == W_GLOBAL)) {
        u8 w = tid();
        u32 t = gtok(pos);
        if (v.spec_mode == 2) return fail_at(pos, M_P_SPEC_REJECT, gspan(t));
        u8 bit = w == W_HOST ? 1 : (w == W_DEVICE ? 2 : 4);
        if (seen & bit) return fail_at(pos, M_P_SPEC_DUP, gspan(t));
        seen |= bit;
        take();
        u32 pred = NONE;
        if (w != W_GLOBAL && at_p(P_LPAREN)) {
          take();
          pred = expr();
          if (pred == NONE) return false;
          if (!need_p(P_RPAREN, EX_RPAREN)) return false;
        }
        if (v.spec_mode == 1) continue;
        if (w == W_HOST) { flags |= FF_H; hp = pred; }
        else if (w == W_DEVICE) { flags |= FF_D; dp = pred; }
        else flags |= FF_G;
      } else if (at_w(W_CONSTEXPR)) {
        take();
        flags |= FF_CX;
      } else {
        break;
      }
    }
    if ((flags & FF_G) && (flags & (FF_H | FF_D))) return fail_at(last, M_P_GLOBAL_EXCL);
    return true;
  }

  EXS_HD u32 struct_(u32 tps, u16 sflags, u32 hp, u32 dp) {
    u32 kw = take();
    (void)kw; (void)hp; (void)dp;
    u32 nm;
    if (!need_name(NW_STRUCT, nm)) return NONE;
    if (sflags & (FF_CX | FF_G)) { fail_tok(nm, M_P_STRUCT_SPEC); return NONE; }
    for (u32 tp = tps; tp != NONE; tp = N(tp).next)
      if (N(tp).sub != 1) { fail_tok(N(tp).tok, M_P_STRUCT_TPARAM); return NONE; }
    if (!need_p(P_LBRACE, EX_LBRACE)) return NONE;
    ListB mem;
    while (!at_p(P_RBRACE)) {
      u32 m = member();
      if (m == NONE) return NONE;
      push(mem, m);
    }
    if (!need_p(P_RBRACE, EX_RBRACE) || !need_p(P_SEMI, EX_SEMI)) return NONE;
    u32 id = mk(N_STRUCT, nm);
    if (id == NONE) return NONE;
    Node& s = N(id);
    s.c0 = tps; s.c1 = mem.head; s.n = (u16)(sflags & (FF_H | FF_D | FF_G | FF_CX));
    return id;
  }

  EXS_HD u32 member() {
    u8 pragma;
    if (!pragma_opt(pragma)) return NONE;
    u32 tps = NONE, req = NONE;
    if (at_w(W_TEMPLATE)) {
      if (!template_header(tps)) return NONE;
      if (at_w(W_REQUIRES) && !requires_clause(req)) return NONE;
    }
    u16 flags = 0; u32 hp = NONE, dp = NONE;
    bool is_static = false;
    while (true) {
      if (at_w(W_STATIC)) { take(); is_static = true; }
      else if (at_w(W_CONSTEXPR)) { take(); flags |= FF_CX; }
      else if (kind() == TK_IDENT && (tid() == W_HOST || tid() == W_DEVICE || tid() == W_GLOBAL)) {
        u16 sf; u32 shp, sdp;
        if (!specifiers(sf, shp, sdp)) return NONE;
        flags |= sf & (FF_H | FF_D | FF_CX);
        if (shp != NONE) hp = shp;
        if (sdp != NONE) dp = sdp;
        if (sf & FF_G) { fail_at(pos, M_P_MEMBER_GLOBAL); return NONE; }
      } else break;
    }
    u32 ty = type_();
    if (ty == NONE) return NONE;
    u32 nm;
    if (!need_name(NW_MEMBER, nm)) return NONE;
    if (at_p(P_ASSIGN)) {
      if (tps != NONE || req != NONE || pragma) { fail_tok(nm, M_P_MCONST_DECL); return NONE; }
      u8 bt = N(ty).sub;
      if (!(bt == BT_HDC || bt == BT_BOOL || bt == BT_INT) || N(ty).c0 != NONE) { fail_tok(nm, M_P_MCONST_TYPE); return NONE; }
      if (!(is_static && (flags & FF_CX))) { fail_tok(nm, M_P_MCONST_STATIC); return NONE; }
      if (flags & (FF_H | FF_D)) { fail_tok(nm, M_P_MCONST_SPEC); return NONE; }
      take();
      u32 val = expr();
      if (val == NONE) return NONE;
      if (!need_p(P_SEMI, EX_SEMI)) return NONE;
      u32 id = mk(N_MVAR, nm);
      if (id == NONE) return NONE;
      N(id).sub = bt; N(id).c0 = val;
      return id;
    }
    pos--;  // give the member name back to function()
    return function(tps, req, flags, hp, dp, pragma, true, ty, is_static);
  }

  EXS_HD u32 function(u32 tps, u32 req, u16 flags, u32 hp, u32 dp, u8 pragma, bool member,
                      u32 ret, bool is_static) {
    if (ret == NONE) {
      ret = type_();
      if (ret == NONE) return NONE;
    }
    u32 nm;
    if (!need_name(NW_FUNCTION, nm)) return NONE;
    if (!need_p(P_LPAREN, EX_LPAREN)) return NONE;
    ListB params;
    if (!at_p(P_RPAREN)) {
      while (true) {
        u32 pty = type_();
        if (pty == NONE) return NONE;
        u32 pn;
        if (!need_name(NW_PARAM, pn)) return NONE;
        u32 pid = mk(N_PARAM, pn);
        if (pid == NONE) return NONE;
        N(pid).c0 = pty;
        push(params, pid);
        if (!at_p(P_COMMA)) break;
        take();
      }
    }
    if (!need_p(P_RPAREN, EX_RPAREN)) return NONE;
    if (req != NONE && tps == NONE) { fail_tok(nm, M_P_REQ_TEMPLATE); return NONE; }
    u8 rbt = N(ret).sub;
    if (flags & FF_G) {
      if (rbt != BT_VOID) { fail_tok(nm, M_P_GLOBAL_VOID); return NONE; }
      if (member) { fail_tok(nm, M_P_GLOBAL_MEMBER); return NONE; }
    }
    if (!member && v.toks[nm].id == W_MAIN) {
      if (tps != NONE || (flags & (FF_H | FF_D | FF_G | FF_CX)) || is_static) { fail_tok(nm, M_P_MAIN_SPEC); return NONE; }
      if (rbt != BT_INT || params.count) { fail_tok(nm, M_P_MAIN_SIG); return NONE; }
    }
    u32 body = NONE;
    bool has_body = false;
    u32 nst = 0;
    if (at_p(P_LBRACE) && pos == defer_open) {
      // a large body: its statements are parsed in parallel afterwards and
      // linked under this FN node (run_parse step 4b)
      pos = defer_close + 1;
      has_body = true;
      deferred = true;
    } else if (at_p(P_LBRACE)) {
      if (!block(body)) return NONE;
      has_body = true;
      nst = block_stmts;
    } else if (!need_p(P_SEMI, EX_FN_BODY)) {
      return NONE;
    }
    u32 id = mk(N_FN, nm);
    u32 xid = mk(N_FNX, nm);
    if (id == NONE || xid == NONE) return NONE;
    Node& f = N(id);
    f.c0 = tps; f.c1 = params.head; f.c2 = body;
    u16 fl = flags & (FF_H | FF_D | FF_G | FF_CX);
    if (is_static) fl |= FF_STATIC;
    if (has_body) fl |= FF_BODY;
    if (pragma) fl |= FF_PRAGMA;
    if (member) fl |= FF_MEMBER;
    if (hp != NONE) fl |= FF_HPRED;
    if (dp != NONE) fl |= FF_DPRED;
    f.n = fl;
    f.sub = (u8)params.count;
    Node& x = N(xid);
    x.c0 = req; x.c1 = hp; x.c2 = dp; x.next = ret;
    x.hv = nst;  // top-level statements of the body (a deferred body: set when linked)
    return id;
  }

  // ------------------------------------------------------------ types
  EXS_HD u32 type_() {
    if (kind() == TK_IDENT && (tid() == W_VOID || tid() == W_INT || tid() == W_BOOL || tid() == W_HDC)) {
      u8 w = tid();
      u32 t = take();
      u32 id = mk(N_TYPE, t);
      if (id != NONE) N(id).sub = w == W_VOID ? BT_VOID : (w == W_INT ? BT_INT : (w == W_BOOL ? BT_BOOL : BT_HDC));
      return id;
    }
    u32 nm;
    if (!need_name(NW_TYPE, nm)) return NONE;
    u32 targs = NONE;
    if (at_p(P_LT) && !targ_list(targs)) return NONE;
    u32 id = mk(N_TYPE, nm);
    if (id != NONE) N(id).c0 = targs;
    return id;
  }

  EXS_HD bool targ_list(u32& out) {
    if (!enter()) return false;
    if (!need_p(P_LT, EX_LT)) return false;
    ListB l;
    u32 a = targ();
    if (a == NONE) return false;
    push(l, a);
    while (at_p(P_COMMA)) {
      take();
      a = targ();
      if (a == NONE) return false;
      push(l, a);
    }
    if (!need_p(P_GT, EX_GT)) return false;
    out = l.head;
    depth--;
    return true;
  }

  EXS_HD bool tok_text_is(u8 w_or_p, bool punct) const {
    // text-only comparison of the current token (any kind), parser.py:384
    u8 k = kind();
    if (k == TK_EOF) return false;
    if (punct) return (k == TK_PUNCT && tid() == w_or_p) || (k == TK_STRING && tid() == (w_or_p == P_BANG ? W_BANG_STR : W_LPAREN_STR));
    return (k == TK_IDENT || k == TK_STRING || k == TK_PRAGMA) && tid() == w_or_p;
  }

  EXS_HD u32 targ() {
    if (kind() == TK_IDENT && (tid() == W_INT || tid() == W_BOOL)) {
      u8 w = tid();
      u32 t = take();
      u32 id = mk(N_TYPE, t);
      if (id != NONE) N(id).sub = w == W_INT ? BT_INT : BT_BOOL;
      return id;
    }
    if ((at_w(W_HDC) && at_p(P_SCOPE, 1)) || (at_w(W_HDC_TRAIT) && at_p(P_LT, 1))) return expr();
    if (kind() == TK_INT || tok_text_is(W_TRUE, false) || tok_text_is(W_FALSE, false) ||
        tok_text_is(P_BANG, true) || tok_text_is(P_LPAREN, true))
      return expr();
    u32 nm;
    if (!need_name(NW_TARG, nm)) return NONE;
    u32 targs = NONE;
    if (at_p(P_LT) && !targ_list(targs)) return NONE;
    u32 id = mk(N_TYPE, nm);
    if (id != NONE) N(id).c0 = targs;
    return id;
  }

  // ------------------------------------------------------------ statements
  EXS_HD bool block(u32& out) {
    if (!enter()) return false;
    if (!need_p(P_LBRACE, EX_LBRACE)) return false;
    ListB l;
    u32 cnt = 0;
    while (!at_p(P_RBRACE)) {
      u32 s = stmt();
      if (s == NONE) return false;
      push(l, s);
      cnt++;
    }
    if (!need_p(P_RBRACE, EX_RBRACE)) return false;
    out = l.head;
    block_stmts = cnt;
    depth--;
    return true;
  }

  // TOP = 1: the copy inlined into the statement-parallel kernel (run_parse
  // step 4b); nested statements go through the out-of-line stmt()
  EXS_HD u32 stmt() { return stmt_t<0>(); }
  template <int TOP>
  EXS_HD EXS_FI u32 stmt_t() {
    u32 tpos = pos;
    u32 t = gtok(pos);
    if (at_w(W_RETURN)) {
      take();
      u32 ex = NONE;
      if (!at_p(P_SEMI)) {
        ex = expr_t<1>();
        if (ex == NONE) return NONE;
      }
      if (!need_p(P_SEMI, EX_SEMI)) return NONE;
      u32 id = mk(N_SRET, t);
      if (id != NONE) N(id).c0 = ex;
      return id;
    }
    if (at_w(W_IF)) {
      take();
      if (!need_p(P_LPAREN, EX_LPAREN)) return NONE;
      u32 c = expr();
      if (c == NONE) return NONE;
      if (!need_p(P_RPAREN, EX_RPAREN)) return NONE;
      u32 then = NONE, other = NONE;
      if (!block(then)) return NONE;
      bool has_else = false;
      if (at_w(W_ELSE)) {
        take();
        if (!block(other)) return NONE;
        has_else = true;
      }
      u32 id = mk(N_SIF, t);
      if (id != NONE) { N(id).c0 = c; N(id).c1 = then; N(id).c2 = other; N(id).sub = has_else; }
      return id;
    }
    if (at_w(W_FOR)) return for_();
    if (kind() == TK_IDENT && (tid() == W_INT || tid() == W_BOOL)) {
      u8 w = tid();
      take();
      u32 nm;
      if (!need_name(NW_VARIABLE, nm)) return NONE;
      if (!need_p(P_SEMI, EX_SEMI)) return NONE;
      u32 ty = mk(N_TYPE, t);
      u32 id = mk(N_SVAR, nm);
      if (ty == NONE || id == NONE) return NONE;
      N(ty).sub = w == W_INT ? BT_INT : BT_BOOL;
      N(id).c0 = ty;
      return id;
    }
    if (kind() == TK_IDENT && !is_kw()) {
      bool matched = false;
      u32 s = ident_stmt(matched);
      if (failed) return NONE;
      if (matched) return s;
    }
    (void)tpos;
    u32 ex = expr_t<1>();
    if (ex == NONE) return NONE;
    if (!need_p(P_SEMI, EX_SEMI)) return NONE;
    u32 id = mk(N_SEXPR, t);
    if (id != NONE) N(id).c0 = ex;
    return id;
  }

  EXS_HD u32 for_() {
    u32 ft = take();
    if (!need_p(P_LPAREN, EX_LPAREN) || !need_w(W_INT, EX_INT)) return NONE;
    u32 v1, v2, v3;
    if (!need_name(NW_LOOPVAR, v1)) return NONE;
    if (!need_p(P_ASSIGN, EX_ASSIGN)) return NONE;
    u32 init = expr();
    if (init == NONE) return NONE;
    if (!need_p(P_SEMI, EX_SEMI)) return NONE;
    if (!need_name(NW_LOOPVAR, v2)) return NONE;
    if (!need_p(P_LT, EX_LT)) return NONE;
    u32 bound = expr();
    if (bound == NONE) return NONE;
    if (!need_p(P_SEMI, EX_SEMI) || !need_p(P_INC, EX_INC)) return NONE;
    if (!need_name(NW_LOOPVAR, v3)) return NONE;
    if (v.toks[v2].hv != v.toks[v1].hv || v.toks[v3].hv != v.toks[v1].hv) { fail_tok(ft, M_P_FOR_VAR); return NONE; }
    if (!need_p(P_RPAREN, EX_RPAREN)) return NONE;
    u32 body = NONE;
    if (!block(body)) return NONE;
    u32 id = mk(N_SFOR, v1);
    if (id != NONE) { N(id).c0 = init; N(id).c1 = bound; N(id).c2 = body; }
    return id;
  }

  // launch / variable declaration, else back off (parser.py:460-489)
  EXS_HD u32 ident_stmt(bool& matched) {
    matched = false;
    u32 mark = pos;
    u32 save_used = nused;
    u32 nm = take();
    u32 targs = NONE;
    if (at_p(P_LT)) {
      // look ahead to the '>' closing the template arguments (their grammar
      // has no bare '<' or '>' besides nested lists): unless a launch '<<<' or a
      // declared name follows, the statement is an expression -- back off now
      // instead of parsing the list twice
      u32 q = pos, dep = 0;
      bool known = false;
      while (q < v.n) {
        const u16 kq = v.vkid[v.vbase + q];
        if ((kq >> 8) == TK_PUNCT) {
          const u8 pq = (u8)kq;
          if (pq == P_LT) dep++;
          else if (pq == P_GT) { if (--dep == 0) { known = true; break; } }
          else if (pq == P_LLL || pq == P_GGG || pq == P_SEMI || pq == P_LBRACE || pq == P_RBRACE) break;
        }
        q++;
      }
      if (known) {
        const u16 kn = q + 1 < v.n ? v.vkid[v.vbase + q + 1] : (u16)(TK_EOF << 8);
        const bool launch = kn == (u16)((TK_PUNCT << 8) | P_LLL);
        const bool decl = (kn >> 8) == TK_IDENT && !((u8)kn >= 1 && (u8)kn <= W_LAST_KEYWORD);
        if (!launch && !decl) { pos = mark; return NONE; }
      }
      int save_depth = depth;
      bool ok = targ_list(targs);
      if (!ok) {
        if (overflow) return NONE;
        failed = false;   // a ParseError inside the targ list backtracks
        pos = mark; nused = save_used; depth = save_depth;
        return NONE;
      }
    }
    if (at_p(P_LLL)) {
      matched = true;
      take();
      u32 grid = expr();
      if (grid == NONE) return NONE;
      if (!need_p(P_COMMA, EX_COMMA)) return NONE;
      u32 blk = expr();
      if (blk == NONE) return NONE;
      if (!need_p(P_GGG, EX_GGG) || !need_p(P_LPAREN, EX_LPAREN)) return NONE;
      u32 args;
      if (!call_args(args)) return NONE;
      if (!need_p(P_RPAREN, EX_RPAREN) || !need_p(P_SEMI, EX_SEMI)) return NONE;
      u32 id = mk(N_SLAUNCH, nm);
      if (id == NONE) return NONE;
      N(grid).next = blk;
      N(id).c0 = targs; N(id).c1 = grid; N(id).c2 = args;
      return id;
    }
    if (kind() == TK_IDENT && !is_kw()) {
      matched = true;
      u32 var = take();
      if (!need_p(P_SEMI, EX_SEMI)) return NONE;
      u32 ty = mk(N_TYPE, nm);
      u32 id = mk(N_SVAR, var);
      if (ty == NONE || id == NONE) return NONE;
      N(ty).c0 = targs;
      N(id).c0 = ty;
      return id;
    }
    pos = mark;
    nused = save_used;
    return NONE;
  }

  // ------------------------------------------------------------ expressions
  // expression grammar; TOP = 1 is the copy inlined into stmt() (its own
  // recursion goes through the out-of-line expr()/unary(), TOP = 0)
  EXS_HD u32 expr() { return expr_t<0>(); }
  EXS_HD u32 unary() { return unary_t<0>(); }
  template <int TOP>
  EXS_HD EXS_FI u32 expr_t() {
    if (!enter()) return NONE;
    u32 lhs = conj<TOP>();
    while (lhs != NONE && at_p(P_OR)) {
      u32 op = take();
      u32 rhs = conj<TOP>();
      if (rhs == NONE) return NONE;
      u32 id = mk(N_BIN, op);
      if (id == NONE) return NONE;
      N(id).sub = OP_OR; N(id).c0 = lhs; N(id).c1 = rhs;
      lhs = id;
    }
    depth--;
    return lhs;
  }
  template <int TOP>
  EXS_HD EXS_FI u32 conj() {
    u32 lhs = cmp<TOP>();
    while (lhs != NONE && at_p(P_AND)) {
      u32 op = take();
      u32 rhs = cmp<TOP>();
      if (rhs == NONE) return NONE;
      u32 id = mk(N_BIN, op);
      if (id == NONE) return NONE;
      N(id).sub = OP_AND; N(id).c0 = lhs; N(id).c1 = rhs;
      lhs = id;
    }
    return lhs;
  }
  template <int TOP>
  EXS_HD EXS_FI u32 cmp() {
    u32 lhs = unary_t<TOP>();
    if (lhs == NONE) return NONE;
    if (at_p(P_EQ) || at_p(P_NE)) {
      u8 o = tid();
      u32 op = take();
      u32 rhs = unary_t<TOP>();
      if (rhs == NONE) return NONE;
      u32 id = mk(N_BIN, op);
      if (id == NONE) return NONE;
      N(id).sub = o == P_EQ ? OP_EQ : OP_NE; N(id).c0 = lhs; N(id).c1 = rhs;
      return id;
    }
    return lhs;
  }
  template <int TOP>
  EXS_HD EXS_FI u32 unary_t() {
    if (at_p(P_BANG)) {
      if (!enter()) return NONE;
      u32 op = take();
      u32 inner = unary();
      if (inner == NONE) return NONE;
      u32 id = mk(N_NOT, op);
      if (id != NONE) N(id).c0 = inner;
      depth--;
      return id;
    }
    return postfix();
  }
  EXS_HD EXS_FI bool call_args(u32& out) {
    ListB l;
    if (!at_p(P_RPAREN)) {
      while (true) {
        u32 a = expr();
        if (a == NONE) return false;
        push(l, a);
        if (!at_p(P_COMMA)) break;
        take();
      }
    }
    out = l.head;
    return true;
  }
  EXS_HD EXS_FI bool paren_args(u32& out, u32& count) {
    if (!need_p(P_LPAREN, EX_LPAREN)) return false;
    if (!call_args(out)) return false;
    count = 0;
    for (u32 a = out; a != NONE; a = N(a).next) count++;
    return need_p(P_RPAREN, EX_RPAREN);
  }
  EXS_HD u32 chain(u32 recv) {
    while (at_p(P_DOT)) {
      take();
      u32 nm;
      if (!need_name(NW_MEMBER, nm)) return NONE;
      u32 targs = NONE;
      if (at_p(P_LT) && !targ_list(targs)) return NONE;
      u32 args, cnt;
      if (!paren_args(args, cnt)) return NONE;
      u32 id = mk(N_MCALL, nm);
      if (id == NONE) return NONE;
      Node& m = N(id);
      m.c0 = recv; m.c1 = targs; m.c2 = args; m.n = (u16)cnt;
      recv = id;
    }
    return recv;
  }
  // printf / fixed-arity validation (parser.py:551-569); name = builtin word id
  EXS_HD bool check_builtin(u8 w, u32 args, u32 count, u32 loc_tok) {
    if (w == W_PRINTF) {
      if (args == NONE || N(args).kind != N_STR) return fail_tok(loc_tok, M_P_PRINTF_FMT);
      const Tok& st = v.toks[N(args).tok];
      // scan the format's logical text for % holes
      u32 holes = 0;
      const u8* src = v_src;
      u32 p = st.pos;
      while (p < st.end) {
        if (!spliced(p) && src[p] == '%') {
          u32 q = p + 1;
          while (q < st.end && spliced(q)) q++;
          if (!(q < st.end && src[q] == 'd')) return fail_tok(loc_tok, M_P_PRINTF_TEXT);
          holes++;
          p = q + 1;
          continue;
        }
        p++;
      }
      if (holes > 1) return fail_tok(loc_tok, M_P_PRINTF_ONE);
      if (count - 1 != holes) return fail_tok(loc_tok, M_P_PRINTF_COUNT);
      return true;
    }
    int ar = -1;
    if (w == W_RELEASE_ASSERT) ar = 1;
    else if (w == W_TRAP || w == W_ABORT || w == W_CUDASYNC) ar = 0;
    if (ar >= 0 && (int)count != ar) return fail_tok(loc_tok, M_P_ARITY, w);
    return true;
  }
  const u8* v_src = nullptr;
  const u32* v_splice = nullptr;
  EXS_HD bool spliced(u32 p) const { return (v_splice[p >> 5] >> (p & 31)) & 1u; }

  EXS_HD u32 postfix() {
    u32 tp = pos;
    u32 t = gtok(pos);
    u8 k = kind();
    if (k == TK_INT) { take(); return mk(N_INT, t); }
    if (k == TK_STRING) { take(); return mk(N_STR, t); }
    if (at_w(W_TRUE) || at_w(W_FALSE)) {
      u8 w = tid();
      take();
      u32 id = mk(N_BOOL, t);
      if (id != NONE) N(id).sub = w == W_TRUE;
      return id;
    }
    if (at_p(P_LPAREN)) {
      if (!enter()) return NONE;
      take();
      u32 inner = expr();
      if (inner == NONE) return NONE;
      if (!need_p(P_RPAREN, EX_RPAREN)) return NONE;
      depth--;
      return chain(inner);
    }
    if (at_w(W_CUDA_ARCH)) { take(); return mk(N_ARCH, t); }
    if (at_w(W_HDC) && at_p(P_SCOPE, 1)) {
      take(); take();
      u32 vpos = pos;
      u8 vk = kind(), vid = tid();
      take();
      bool ok = vk != TK_EOF && (vk == TK_IDENT || vk == TK_STRING || vk == TK_PRAGMA) &&
                (vid == W_HST || vid == W_DEV || vid == W_HSTDEV);
      if (!ok) { fail_at(vpos, M_P_HDC_VALUE, span_of(vpos)); return NONE; }
      u32 id = mk(N_HDCV, t);
      if (id != NONE) N(id).sub = vid == W_HST ? 1 : (vid == W_DEV ? 2 : 3);
      return id;
    }
    if (at_w(W_HDC_TRAIT) && at_p(P_LT, 1)) {
      take();
      if (!need_p(P_LT, EX_LT)) return NONE;
      u32 ty = type_();
      if (ty == NONE) return NONE;
      if (!need_p(P_GT, EX_GT)) return NONE;
      u32 id = mk(N_TRAIT, t);
      if (id != NONE) N(id).c0 = ty;
      return id;
    }
    if (at_w(W_STD) && at_p(P_SCOPE, 1)) {
      take(); take();
      u32 nm;
      if (!need_name(NW_FUNCTION, nm)) return NONE;
      u32 args, cnt;
      if (!paren_args(args, cnt)) return NONE;
      // std::NAME: the only fixed-arity std builtin is std::abort
      if (v.toks[nm].id == W_ABORT && cnt != 0) { fail_tok(t, M_P_ARITY, 0xFF); return NONE; }
      u32 id = mk(N_CALL, t);
      if (id == NONE) return NONE;
      Node& c = N(id);
      c.sub = CALL_STD; c.c0 = nm; c.c1 = NONE; c.c2 = args; c.n = (u16)cnt;
      return id;
    }
    if (k != TK_IDENT || is_kw()) { fail_at(tp, M_P_EXPR, span_of(tp)); return NONE; }
    take();
    u32 targs = NONE;
    if (at_p(P_LT) && !targ_list(targs)) return NONE;
    if (at_p(P_LBRACE)) {
      take();
      if (!need_p(P_RBRACE, EX_RBRACE)) return NONE;
      u32 ty = mk(N_TYPE, t);
      u32 id = mk(N_TMP, t);
      if (ty == NONE || id == NONE) return NONE;
      N(ty).c0 = targs;
      N(id).c0 = ty;
      return chain(id);
    }
    if (at_p(P_SCOPE)) {
      take();
      u32 mem;
      if (!need_name(NW_MEMBER, mem)) return NONE;
      u32 mtargs = NONE;
      if (at_p(P_LT) && !targ_list(mtargs)) return NONE;
      u32 ty = mk(N_TYPE, t);
      if (ty == NONE) return NONE;
      N(ty).c0 = targs;
      if (at_p(P_LPAREN)) {
        u32 args, cnt;
        if (!paren_args(args, cnt)) return NONE;
        u32 id = mk(N_SCALL, mem);
        if (id == NONE) return NONE;
        Node& s = N(id);
        s.c0 = ty; s.c1 = mtargs; s.c2 = args; s.n = (u16)cnt;
        return id;
      }
      u32 id = mk(N_MCONST, mem);
      if (id != NONE) N(id).c0 = ty;
      return id;
    }
    if (at_p(P_LPAREN)) {
      u32 args, cnt;
      if (!paren_args(args, cnt)) return NONE;
      u8 w = v.toks[t].id;
      if (w && !check_builtin(w, args, cnt, t)) return NONE;
      u32 id = mk(N_CALL, t);
      if (id == NONE) return NONE;
      Node& c = N(id);
      c.sub = CALL_PLAIN; c.c0 = NONE; c.c1 = targs; c.c2 = args; c.n = (u16)cnt;
      return chain(id);
    }
    if (targs != NONE) { fail_at(pos, M_P_TARGS, gspan(t)); return NONE; }
    return chain(mk(N_NAME, t));
  }
};

}  // namespace exs
