// exs_sema.cuh -- K5 tables + the evaluator used by the walk: type
// resolution, the hdc<T> trait, constant evaluation, SFINAE overload
// selection and effective execution spaces (reference: sema.py:329-703).
// Every function returns a status instead of raising: ST_SUBST mirrors
// SubstFailure (silent), ST_SEMA mirrors SemaError (diagnosed).
#pragma once
#include "exs_common.cuh"
#include "exs_parse.cuh"

namespace exs {

enum { ST_OK = 0, ST_SUBST = 1, ST_SEMA = 2 };
enum { V_NONE = 0, V_TYPE, V_HDC, V_BOOL, V_INT };
// name hashes of fixed words (NameHash: the lexer computes the same for tokens)
constexpr u64 H_INT = name_hash_c("int"), H_BOOL = name_hash_c("bool"), H_HDC_MEMBER = name_hash_c("hdc"),
              H_STD = name_hash_c("std::");

struct Val {
  u8 k;      // V_*
  u8 targ;   // type: 0 none, 1..3 HDC arg + 1 ... (Hst=1, Dev=2, HstDev=3)
  u8 bt;     // type: BT_* builtin code or BT_NONE for structs
  u8 pad;
  u32 rec;   // type: struct record (NONE for builtins)
  u64 x;     // type: name hash; hdc: 1..3; bool: 0/1; int: value
};
EXS_HD inline Val vnone() { Val v; v.k = V_NONE; v.targ = 0; v.bt = 0; v.pad = 0; v.rec = NONE; v.x = 0; return v; }
EXS_HD inline Val vhdc(u64 h) { Val v = vnone(); v.k = V_HDC; v.x = h; return v; }
EXS_HD inline Val vbool(bool b) { Val v = vnone(); v.k = V_BOOL; v.x = b; return v; }
EXS_HD inline Val vint(u64 i) { Val v = vnone(); v.k = V_INT; v.x = i; return v; }
EXS_HD inline bool val_eq(const Val& a, const Val& b) {
  return a.k == b.k && a.x == b.x && (a.k != V_TYPE || a.targ == b.targ);
}

// Struct and function records (one per declaration, view-local order)
// FR_BODY: an instance has something to walk (statements or parameters);
// FR_MAIN: the free function main (instances read both without the node/token)
enum { FR_DUP = 1, FR_OWNER = 2, FR_MEMBER = 4, FR_VARDECL = 8, FR_BODY = 16, FR_MAIN = 32 };
struct FnRec {
  u32 node, view, rec, order;  // rec: containing struct record (NONE for free)
  u64 sig, name;               // signature hash (sema.py:144-149), name hash
  u32 sig_rep;                 // first decl of the view with this signature
  u32 ncalls;                  // call sites in the body (edges/s unit)
  u8 flags, pad[3];
  u32 nstmts;                  // top-level statements of the body
  u32 stmt_base, pad2;         // first entry in the per-statement tables
};
struct RecRec {
  u32 node, view, order, dup;
  u64 name;
};

// open-addressing u64 -> u32 map (keys never 0); key and value share one
// 16-byte entry, so a probe touches one line
struct alignas(16) MapEnt {
  u64 k;
  u32 v, pad;
};
struct Map {
  MapEnt* e;
  u32 mask;
  EXS_HD u32 find(u64 k) const {
    if (!e) return NONE;
    u32 h = (u32)mix64(k) & mask;
    while (true) {
      const MapEnt x = e[h];
      if (x.k == k) return x.v;
      if (x.k == 0) return NONE;
      h = (h + 1) & mask;
    }
  }
};
EXS_HD inline u64 nz(u64 k) { return k ? k : 0x9E3779B97F4A7C15ull; }
EXS_HD inline u64 vkey(u32 view, u64 h) { return nz(hcombine((u64)view + 0x51ED27ull, h)); }

// the slot holding key k (inserted if absent; its value is left alone)
EXS_HD inline u32 map_insert_slot(MapEnt* e, u32 mask, u64 k) {
  u32 h = (u32)mix64(k) & mask;
  while (true) {
    unsigned long long prev = at_cas64((unsigned long long*)&e[h].k, 0ull, (unsigned long long)k);
    if (prev == 0ull || prev == k) return h;
    h = (h + 1) & mask;
  }
}
EXS_HD inline void map_insert_min(MapEnt* e, u32 mask, u64 k, u32 v) {
  u32 h = (u32)mix64(k) & mask;
  while (true) {
    unsigned long long prev = at_cas64((unsigned long long*)&e[h].k, 0ull, (unsigned long long)k);
    if (prev == 0ull || prev == k) { at_min(&e[h].v, v); return; }
    h = (h + 1) & mask;
  }
}

// ---------------------------------------------------------------------------
// evaluation context and errors

struct EErr {
  u16 code, msg;   // SemaError: C_* + M_*; SubstFailure: msg = SF_* (code 0)
  u32 line, col;
  u64 a0, a1, a2;
};

#define MAX_EVAL_DEPTH 96

struct Env {
  u8 n, nbase;
  u64 names[4];
  Val vals[4];
  u32 mv_rec;            // member-variable layer (sema.py:477-488), NONE if absent
  const Env* mv_env;     // env the member variables are evaluated in
  EXS_HD void clear() { n = 0; nbase = 0; mv_rec = NONE; mv_env = nullptr; }
  EXS_HD void add(u64 name, const Val& v) {
    if (n < 4) { names[n] = name; vals[n] = v; n++; }
  }
};

struct Tables {
  const Node* nodes;
  const Tok* toks;
  const FnRec* fns;
  const RecRec* recs;
  Map smap;        // (view, struct name) -> first struct record
  Map fmap;        // (view, fn name) -> start in fcand
  const u32* fcand;      // candidate decl indices grouped by name
  const u32* fcand_cnt;  // run length at each run start
  const u8* src;
  const u32* splice;
};

struct Sema {
  const Tables* T;
  u32 view;
  u8 mode, plain, relaxed, fund;
  EErr err;
  int depth;
  bool contract;   // recursion bound exceeded (out of contract)

  EXS_HD void init(const Tables* t, u32 v, u8 cfg) {
    T = t; view = v;
    mode = cfg & CFG_MODE_MASK; plain = (cfg & CFG_PLAIN) != 0;
    relaxed = (cfg & CFG_RELAXED) != 0; fund = (cfg & CFG_FUND) != 0;
    depth = 0; contract = false;
    err.code = err.msg = 0;
  }
  EXS_HD const Node& N(u32 id) const { return T->nodes[id]; }
  EXS_HD const Tok& K(u32 t) const { return T->toks[t]; }
  EXS_HD u64 span(u32 t) const { const Tok& k = K(t); return ((u64)k.pos << 32) | (u64)(k.end - k.pos); }

  // error setters are cold paths: out of line so the (large) walk kernel's
  // instruction footprint stays small (profiles/r01_walk: ~30% of stalls were
  // instruction-cache misses)
  EXS_HD EXS_NOINLINE u8 subst(u16 sf, u64 a0 = 0, u64 a1 = 0, u64 a2 = 0) {
    err.code = 0; err.msg = sf; err.a0 = a0; err.a1 = a1; err.a2 = a2;
    return ST_SUBST;
  }
  EXS_HD EXS_NOINLINE u8 sema(u16 code, u16 msg, u32 tok, u64 a0 = 0, u64 a1 = 0, u64 a2 = 0) {
    err.code = code; err.msg = msg; err.line = K(tok).line; err.col = K(tok).col;
    err.a0 = a0; err.a1 = a1; err.a2 = a2;
    return ST_SEMA;
  }

  // type-name argument for messages: struct name span, or marker for builtins
  EXS_HD u64 type_name_arg(const Val& t) const {
    if (t.rec != NONE) return span(N(T->recs[t.rec].node).tok);
    return 0xFFFFFFFF00000000ull | t.bt;
  }
  // loc of a node (the reference's .loc)
  EXS_HD u32 loc_tok(u32 id) const {
    while (true) {
      const Node& n = N(id);
      if (n.kind == N_MCALL) { id = n.c0; continue; }
      if (n.kind == N_SCALL || n.kind == N_MCONST) return N(n.c0).tok;
      return n.tok;
    }
  }

  // ------------------------------------------------------------- lookups
  EXS_HD u32 struct_of(u64 name) const { return T->smap.find(vkey(view, name)); }
  EXS_HD u32 first_mvar(u32 rec, u64 name) const {
    for (u32 m = N(T->recs[rec].node).c1; m != NONE; m = N(m).next)
      if (N(m).kind == N_MVAR && N(m).hv == name) return m;
    return NONE;
  }
  EXS_HD u64 type_name_hash(u32 tnode) const { return N(tnode).hv; }

  // env lookup with dict layering; returns false if absent
  EXS_HD bool env_get(const Env& env, u64 name, Val& out) {
    for (int i = env.n - 1; i >= env.nbase; i--)
      if (env.names[i] == name) { out = env.vals[i]; return true; }
    if (env.mv_rec != NONE) return env_get_mv(env, name, out);
    for (int i = env.nbase - 1; i >= 0; i--)
      if (env.names[i] == name) { out = env.vals[i]; return true; }
    return false;
  }
  // env_get through the member-variable layer (rare): out of line
  EXS_HD EXS_NOINLINE bool env_get_mv(const Env& env, u64 name, Val& out) {
    {
      // last member variable with this name whose value evaluates wins
      u32 last_ok = NONE;
      Val lv = vnone();
      EErr save = err;
      for (u32 m = N(T->recs[env.mv_rec].node).c1; m != NONE; m = N(m).next) {
        if (N(m).kind != N_MVAR || N(m).hv != name) continue;
        Val v;
        u8 st = eval(N(m).c0, *env.mv_env, false, v);
        if (contract) return false;
        if (st == ST_OK) { last_ok = m; lv = v; }
      }
      err = save;
      if (last_ok != NONE) { out = lv; return true; }
    }
    for (int i = env.nbase - 1; i >= 0; i--)
      if (env.names[i] == name) { out = env.vals[i]; return true; }
    return false;
  }

  EXS_HD void struct_env(u32 rec, const Val& t, Env& out) const {
    out.clear();
    u32 tp = N(T->recs[rec].node).c0;
    if (tp != NONE && t.targ) out.add(N(tp).hv, vhdc(t.targ));
    out.nbase = out.n;
  }

  EXS_HD bool enter() {
    if (++depth > MAX_EVAL_DEPTH) { contract = true; return false; }
    return true;
  }

  // ------------------------------------------------------------- types
  // resolve_type (sema.py:333-363)
  EXS_HD u8 type_of(u32 tr, const Env& env, Val& out) {
    const Node& t = N(tr);
    u8 bt = t.sub;
    u64 name = t.hv;
    if (bt == BT_INT || bt == BT_BOOL || bt == BT_VOID) {
      if (t.c0 != NONE) return sema(C_E0001, M_S_NO_TARGS_BUILTIN, t.tok, bt);
      out = vnone(); out.k = V_TYPE; out.bt = bt; out.x = name; out.rec = NONE;
      return ST_OK;
    }
    Val b;
    if (env_get(env, name, b)) {
      if (contract) return ST_SUBST;
      if (b.k == V_TYPE) {
        if (t.c0 != NONE) return subst(SF_NOT_TEMPLATE, span(t.tok));
        out = b;
        return ST_OK;
      }
      return subst(SF_NOT_TYPE_NAME, span(t.tok));
    }
    if (contract) return ST_SUBST;
    u32 rec = struct_of(name);
    if (rec == NONE) return sema(C_E0101, M_S_UNDEF_TYPE, t.tok, span(t.tok));
    if (!enter()) return ST_SUBST;
    const Node& sn = N(T->recs[rec].node);
    u32 ta = t.c0;
    u8 targ = 0;
    bool non_hdc = false;
    u32 ntp = 0;
    for (u32 tp = sn.c0; tp != NONE; tp = N(tp).next, ntp++) {
      Val v;
      u8 st;
      if (ta != NONE) {
        st = as_hdc(ta, env, v);
        ta = N(ta).next;
      } else if (N(tp).c0 != NONE) {
        st = eval(N(tp).c0, env, false, v);
      } else {
        depth--;
        return sema(C_E0001, M_S_MISSING_TARGS, t.tok, span(t.tok));
      }
      if (st != ST_OK) { depth--; return st; }
      if (v.k != V_HDC) non_hdc = true;
      else targ = (u8)v.x;
    }
    depth--;
    if (ta != NONE) return sema(C_E0001, M_S_TOO_MANY_TARGS, t.tok, span(t.tok));
    if (non_hdc) return subst(SF_STRUCT_TARGS_HDC);
    out = vnone(); out.k = V_TYPE; out.bt = BT_NONE; out.rec = rec; out.x = name; out.targ = ntp ? targ : 0;
    return ST_OK;
  }

  // _targ_as_hdc (sema.py:366-376)
  EXS_HD u8 as_hdc(u32 ta, const Env& env, Val& out) {
    const Node& t = N(ta);
    if (t.kind == N_TYPE) {
      if (t.c0 != NONE) return subst(SF_EXPECTED_HDC);
      Val b;
      if (env_get(env, t.hv, b)) {
        if (b.k == V_HDC) { out = b; return ST_OK; }
        return subst(SF_EXPECTED_HDC);
      }
      if (contract) return ST_SUBST;
      return subst(SF_NOT_HDC_CONST, span(t.tok));
    }
    return eval(ta, env, false, out);
  }

  // compute_hdc (sema.py:385-404)
  EXS_HD u8 trait(const Val& t, bool f, Val& out) {
    if (t.bt == BT_INT || t.bt == BT_BOOL) { out = vhdc(f ? 3 : 1); return ST_OK; }
    if (t.rec == NONE) return subst(SF_NO_COMPAT, type_name_arg(t));
    u32 mv = first_mvar(t.rec, H_HDC_MEMBER);
    if (mv == NONE) { out = vhdc(1); return ST_OK; }
    if (N(mv).sub != BT_HDC) return sema(C_E0103, M_S_HDC_MEMBER, N(mv).tok, type_name_arg(t));
    Env se;
    struct_env(t.rec, t, se);
    if (!enter()) return ST_SUBST;
    u8 st = eval(N(mv).c0, se, f, out);
    depth--;
    if (st != ST_OK) return st;
    if (out.k != V_HDC) return sema(C_E0103, M_S_HDC_MEMBER, N(mv).tok, type_name_arg(t));
    return ST_OK;
  }

  // eval_const_expr (sema.py:407-463)
  EXS_HD u8 eval(u32 e, const Env& env, bool f, Val& out) {
    if (!enter()) return ST_SUBST;
    u8 st = eval_(e, env, f, out);
    depth--;
    return st;
  }
  // T::member constant (sema.py:431-442); out of line so eval's frame stays small
  EXS_HD EXS_NOINLINE u8 eval_mconst(const Node& n, const Env& env, bool f, Val& out) {
    Val t;
    u8 st = type_of(n.c0, env, t);
    if (st != ST_OK) return st;
    if (t.rec == NONE) return subst(SF_NO_MEMBERS, type_name_arg(t));
    u32 mv = first_mvar(t.rec, n.hv);
    if (mv == NONE) return subst(SF_NO_MEMBER, type_name_arg(t), span(n.tok));
    Env se;
    struct_env(t.rec, t, se);
    st = eval(N(mv).c0, se, f, out);
    if (st != ST_OK) return st;
    if (N(mv).sub == BT_HDC && out.k != V_HDC)
      return sema(C_E0103, M_S_HDC_MEMBER, N(mv).tok, type_name_arg(t));
    return ST_OK;
  }

  EXS_HD EXS_FI u8 eval_(u32 e, const Env& env, bool f, Val& out) {
    const Node& n = N(e);
    switch (n.kind) {
      case N_INT: out = vint(n.hv); return ST_OK;
      case N_BOOL: out = vbool(n.sub != 0); return ST_OK;
      case N_HDCV: out = vhdc(n.sub); return ST_OK;
      case N_ARCH: return subst(SF_ARCH);
      case N_NAME: {
        Val b;
        if (!env_get(env, n.hv, b)) {
          if (contract) return ST_SUBST;
          return subst(SF_UNBOUND, span(n.tok));
        }
        if (b.k == V_TYPE) return subst(SF_IS_TYPE, span(n.tok));
        out = b;
        return ST_OK;
      }
      case N_TRAIT: {
        Val t;
        u8 st = type_of(n.c0, env, t);
        if (st != ST_OK) return st;
        return trait(t, f, out);
      }
      case N_MCONST: return eval_mconst(n, env, f, out);
      case N_NOT: {
        Val v;
        u8 st = eval(n.c0, env, f, v);
        if (st != ST_OK) return st;
        if (v.k != V_BOOL) return subst(SF_NOT_BOOL_OPERAND);
        out = vbool(!v.x);
        return ST_OK;
      }
      case N_BIN: {
        Val a, b;
        u8 st = eval(n.c0, env, f, a);
        if (st != ST_OK) return st;
        st = eval(n.c1, env, f, b);
        if (st != ST_OK) return st;
        if (n.sub == OP_EQ || n.sub == OP_NE) {
          if (a.k != b.k) return subst(SF_UNRELATED);
          bool eq = a.x == b.x && (a.k != V_TYPE || a.targ == b.targ);
          out = vbool(eq == (n.sub == OP_EQ));
          return ST_OK;
        }
        if (a.k != V_BOOL || b.k != V_BOOL) return subst(SF_LOGICAL);
        out = vbool(n.sub == OP_AND ? (a.x && b.x) : (a.x || b.x));
        return ST_OK;
      }
      default:
        return subst(SF_NOT_CONST, n.kind);
    }
  }

  // ------------------------------------------------------------- overloads
  struct Binds {
    u8 n;
    u64 names[2];
    Val vals[2];
    EXS_HD void clear() { n = 0; }
    EXS_HD bool get(u64 name, Val& v) const {
      for (int i = n - 1; i >= 0; i--) if (names[i] == name) { v = vals[i]; return true; }
      return false;
    }
    EXS_HD void set(u64 name, const Val& v) {
      for (int i = 0; i < n; i++) if (names[i] == name) { vals[i] = v; return; }
      if (n < 2) { names[n] = name; vals[n] = v; n++; }
    }
  };

  // the candidate env (sema.py:477-488): owner bindings, member vars, bindings
  EXS_HD void cand_env(const Binds& b, u32 orec, const Env& obinds, Env& out, Env& mv_env) const {
    mv_env = obinds;
    out = obinds;
    out.nbase = out.n;
    out.mv_rec = orec;
    out.mv_env = &mv_env;
    for (int i = 0; i < b.n; i++) out.add(b.names[i], b.vals[i]);
  }

  // _try_candidate (sema.py:545-607)
  EXS_HD EXS_FI u8 try_cand(u32 fi, u32 targs, const Val* argtys, u32 nargs, const Env& env, u32 orec,
                     const Env& obinds, Binds& b) {
    const FnRec& fr = T->fns[fi];
    const Node& fn = N(fr.node);
    b.clear();
    u32 ntp = 0;
    for (u32 tp = fn.c0; tp != NONE; tp = N(tp).next) ntp++;
    u32 nex = 0;
    for (u32 a = targs; a != NONE; a = N(a).next) nex++;
    if (nex > ntp) return subst(SF_OTHER);
    u32 ta = targs;
    for (u32 tp = fn.c0; tp != NONE && ta != NONE; tp = N(tp).next, ta = N(ta).next) {
      Val v;
      u8 st;
      if (N(tp).sub == 0) {
        if (N(ta).kind != N_TYPE) return subst(SF_OTHER);
        st = type_of(ta, env, v);
      } else {
        st = as_hdc(ta, env, v);
        if (st == ST_OK && v.k != V_HDC) return subst(SF_OTHER);
      }
      if (st != ST_OK) return st;
      b.set(N(tp).hv, v);
    }
    if (nargs != fn.sub) return subst(SF_OTHER);
    for (u32 tp = fn.c0; tp != NONE; tp = N(tp).next) {
      u64 tn = N(tp).hv;
      Val dummy;
      if (N(tp).sub != 0 || b.get(tn, dummy)) continue;
      u32 i = 0;
      for (u32 p = fn.c1; p != NONE; p = N(p).next, i++) {
        const Node& pty = N(N(p).c0);
        if (pty.sub == BT_NONE || pty.sub == BT_HDC) {
          if (pty.hv == tn && pty.c0 == NONE && argtys[i].k != V_NONE) { b.set(tn, argtys[i]); break; }
        }
      }
    }
    // common case: everything bound, no argument types to check, no requires
    bool pending = N(fr.node + 1).c0 != NONE;
    for (u32 i = 0; i < nargs && !pending; i++) pending = argtys[i].k != V_NONE;
    for (u32 tp = fn.c0; tp != NONE && !pending; tp = N(tp).next) {
      Val dummy;
      pending = !b.get(N(tp).hv, dummy);
    }
    if (!pending) return ST_OK;
    return cand_finish(fi, argtys, nargs, orec, obinds, b);
  }

  // defaults, argument types and requires of one candidate (sema.py:577-607);
  // out of line: the candidate and full environments live only here
  EXS_HD EXS_NOINLINE u8 cand_finish(u32 fi, const Val* argtys, u32 nargs, u32 orec,
                                     const Env& obinds, Binds& b) {
    const FnRec& fr = T->fns[fi];
    const Node& fn = N(fr.node);
    // the candidate env is materialised only when a default or the requires
    // clause is evaluated; the full env only when an argument type is known
    Env mv_env, cenv;
    bool have_cenv = false;
    for (u32 tp = fn.c0; tp != NONE; tp = N(tp).next) {
      u64 tn = N(tp).hv;
      Val dummy;
      if (b.get(tn, dummy)) continue;
      if (N(tp).sub == 1 && N(tp).c0 != NONE) {
        if (!have_cenv) { cand_env(b, orec, obinds, cenv, mv_env); have_cenv = true; }
        Val v;
        u8 st = eval(N(tp).c0, cenv, fund, v);
        if (st != ST_OK) return st;
        if (v.k != V_HDC) return subst(SF_OTHER);
        b.set(tn, v);
        cenv.add(tn, v);
      } else {
        return subst(SF_OTHER);
      }
    }
    bool any_arg = false;
    for (u32 i = 0; i < nargs; i++) any_arg |= argtys[i].k != V_NONE;
    if (any_arg) {
      Env full = obinds;
      full.nbase = full.n;
      for (int i = 0; i < b.n; i++) full.add(b.names[i], b.vals[i]);
      full.nbase = full.n;
      u32 i = 0;
      for (u32 p = fn.c1; p != NONE; p = N(p).next, i++) {
        if (argtys[i].k == V_NONE) continue;
        Val want;
        u8 st = type_of(N(p).c0, full, want);
        if (contract) return ST_SUBST;
        if (st != ST_OK) return subst(SF_OTHER);
        if (!val_eq(want, argtys[i])) return subst(SF_OTHER);
      }
    }
    u32 req = N(fr.node + 1).c0;
    if (req != NONE) {
      if (!have_cenv) { cand_env(b, orec, obinds, cenv, mv_env); have_cenv = true; }
      Val ok;
      u8 st = eval(req, cenv, fund, ok);
      if (st != ST_OK) return st;
      if (ok.k != V_BOOL || !ok.x) return subst(SF_OTHER);
    }
    return ST_OK;
  }

  EXS_HD bool declared(u16 fl, u8& sp) const {
    sp = 0;
    if (fl & FF_H) sp |= 1;
    if (fl & FF_D) sp |= 2;
    if (!sp) sp = 1;
    return true;
  }
  EXS_HD bool compatible(u32 fi, u8 side, u32 orec) const {
    u16 fl = N(T->fns[fi].node).n;
    bool undec = !(fl & (FF_H | FF_D | FF_G));
    if (undec && orec != NONE) {
      u16 sf = N(T->recs[orec].node).n;
      if (sf & (SF_H | SF_D | SF_G)) { fl = sf; undec = false; }
    }
    if (undec || (fl & FF_G)) return true;
    u8 d;
    declared(fl, d);
    return (d & (1u << side)) || d == 3;
  }

  // effective_spaces (sema.py:670-703): returns 1=H 2=D 3=HD 4=GLOBAL, or error status
  // merged = owner bindings + (tb, hb) bound to the decl's template params; it
  // is only materialised for conditional specifiers under proposal1
  EXS_HD EXS_FI u8 spaces(u32 fi, const Env* obinds, const Val& tb, const Val& hb, u8 side, u32 at_tok,
                   u32 orec, u8& out) {
    const FnRec& fr = T->fns[fi];
    const Node& fn = N(fr.node);
    u16 fl = fn.n;
    if (fl & FF_G) { out = 4; return ST_OK; }
    bool cond = (fl & (FF_HPRED | FF_DPRED)) != 0;
    if (mode == MODE_P1 && cond) return spaces_p1(fi, obinds, tb, hb, at_tok, orec, out);
    if (mode == MODE_P2) {
      if (K(fn.tok).id == W_MAIN && !(fr.flags & FR_OWNER)) { out = 1; return ST_OK; }
      if (!(fl & (FF_H | FF_D | FF_G))) {
        if (orec != NONE) {
          u16 sf = N(T->recs[orec].node).n;
          if (sf & (SF_H | SF_D | SF_G)) { declared(sf, out); return ST_OK; }
        }
        out = (u8)(1u << side);
        return ST_OK;
      }
    }
    declared(fl, out);
    return ST_OK;
  }

  // proposal1 conditional specifiers (sema.py:638-667), out of line
  EXS_HD EXS_NOINLINE u8 spaces_p1(u32 fi, const Env* obinds, const Val& tb, const Val& hb,
                                   u32 at_tok, u32 orec, u8& out) {
    const FnRec& fr = T->fns[fi];
    const Node& fn = N(fr.node);
    u16 fl = fn.n;
    {
      Env merged;
      if (obinds) merged = *obinds; else merged.clear();
      merged.nbase = merged.n;
      for (u32 tp = fn.c0; tp != NONE; tp = N(tp).next) {
        const Val& v = N(tp).sub == 0 ? tb : hb;
        if (v.k != V_NONE) merged.add(N(tp).hv, v);
      }
      merged.nbase = merged.n;
      Env mv_env = merged, env = merged;
      env.nbase = env.n;
      env.mv_rec = orec;
      env.mv_env = &mv_env;
      for (int i = 0; i < merged.n; i++) env.add(merged.names[i], merged.vals[i]);
      u8 r = 0;
      if (fl & FF_H) {
        bool t;
        u8 st = pred(N(fr.node + 1).c1, env, t);
        if (st != ST_OK) return st;
        if (t) r |= 1;
      }
      if (fl & FF_D) {
        bool t;
        u8 st = pred(N(fr.node + 1).c2, env, t);
        if (st != ST_OK) return st;
        if (t) r |= 2;
      }
      if (!r)
        return sema(C_E1401, M_S_EMPTY_SPACES, at_tok, span(fn.tok),
                    (fr.flags & FR_OWNER) ? span(N(T->recs[fr.rec].node).tok) : 0);
      out = r;
      return ST_OK;
    }
  }
  EXS_HD u8 pred(u32 p, const Env& env, bool& t) {
    if (p == NONE) { t = true; return ST_OK; }
    Val v;
    u8 st = eval(p, env, fund, v);
    if (st != ST_OK) return st;
    if (v.k != V_BOOL) return subst(SF_OTHER);
    t = v.x != 0;
    return ST_OK;
  }
};

}  // namespace exs
