// exs_walk.cuh -- K6: walk of one instance's body (reference: spacecheck.py
// _Walk._walk_instance .. _report_stray, lines 312-613).  One thread walks one
// frontier instance of a level-synchronous BFS; the FIFO order of the
// reference is reproduced by creation keys (level, parent rank, local index)
// kept with atomicMin, so "first creator" data (the E1201 location) matches.
#pragma once
#include "exs_common.cuh"
#include "exs_sema.cuh"

namespace exs {

// 128-bit instance key: a = sig_rep<<32 | tcode(type binding),
//                       b = 1<<63 | tcode(owner)<<32 | walk<<3 | hdc<<1 | side
struct alignas(16) IKey {
  u64 a, b;
};

// one slot of the instance hash table: key (128-bit CAS), published id and
// the creation-key minimum of the current level share one 32-byte sector, so
// a creator's probe, id read and atomicMin touch one line
struct alignas(32) Slot {
  IKey k;
  u32 sid, pad;
  unsigned long long sck;
};

// Creation key (the reference's FIFO position, spacecheck.py:312-351):
//   level << CK_LEVEL_SHIFT | parent rank << CK_RANK_SHIFT | local
// level: BFS level of the created instance (roots 0); parent rank: the
// creator's position among its walk's frontier of the previous level, by
// creation key (roots: decl order within the view); local: the creator's
// instantiation ordinal within its body, 2 x (call sites of the earlier
// top-level statements) + ordinal within the statement (a call site
// instantiates at most twice, spacecheck.py:585-596).  A field beyond its
// width marks the unit out of contract (X9999) instead of wrapping.
#define CK_LEVEL_SHIFT 52
#define CK_RANK_SHIFT 26
#define CK_FIELD_MAX ((1u << 26) - 1u)
#define CK_LEVEL_MAX ((1u << 12) - 1u)
EXS_HD inline unsigned long long make_ckey(u32 level, u64 rank, u32 local) {
  return ((unsigned long long)level << CK_LEVEL_SHIFT) | ((unsigned long long)rank << CK_RANK_SHIFT) | local;
}

struct Inst {
  u64 ka, kb;
  unsigned long long ckey;  // min creation key (make_ckey)
  u32 fn, orec, walk, at;   // creating decl, owner struct, walk, at_loc token
  u32 ebase, ecnt;          // legal edges (callee instance ids)
  Val tb, hb, ot;           // type binding, hdc binding, owner type
  u8 side, spaces, pad, flags;
  u32 slot;                 // hash slot of the key (creation key lives in sck[slot] during its level)
};
enum { IF_BODY = 1, IF_MAIN = 2 };

struct Pending {
  u32 walk, caller, line, col;
  u8 callee, pad[3];
};
struct CreateLog {
  unsigned long long ckey;
  u32 inst, at, fn, pad;
};

struct WalkBufs {
  // instance table
  Slot* slots;              // key, published id, min creation key of the current level
  u32 mask;
  Inst* inst;
  u32* n_inst;
  u32 cap_inst;
  u32 lvl_base;             // ids >= lvl_base were created in the level being walked
  u32 clevel;               // level of the instances the walkers of this launch create
  // outputs
  u32* edges;
  Pending* pend;
  u32* n_pend;
  u32 cap_pend;
  u32* seeds;   // (walk, inst) pairs
  u32* n_seeds;
  u32 cap_seeds;
  CreateLog* log;
  u32* n_log;
  u32 cap_log;
  u32* main_inst;               // per walk: instance of main with the max creation key
  unsigned long long* main_key; // per walk
  u32* mains;                   // ids of main's instances as created (n_mains may pass cap_mains)
  u32* n_mains;
  u32 cap_mains;
  // diagnostics
  Diag* diags;
  u32* n_diags;
  u32 cap_diags;
  u64* dset;      // dedup set of diag hashes
  u32 dmask;
  u32* overflow;  // bit0 instances, bit1 diags, bit2 log/pend/seeds
  u32* contract;  // units that exceeded a recursion bound (per file flag array)
};

EXS_HD inline u32 tcode(const Val& t) {
  if (t.k != V_TYPE) return 0;
  if (t.rec == NONE) return t.bt;  // BT_VOID/INT/BOOL are 1..3
  return 4u + t.rec * 4u + t.targ;
}

// ---------------------------------------------------------------------------
// diagnostics emission with on-the-fly dedup (diagnostics.py:116-121)

EXS_HD inline u64 diag_hash(const Diag& d) {
  u64 h = hcombine(d.file, ((u64)d.line << 32) | d.col);
  h = hcombine(h, ((u64)d.code << 16) | d.msg);
  h = hcombine(h, d.a0);
  h = hcombine(h, d.a1);
  h = hcombine(h, d.a2);
  h = hcombine(h, d.a3);
  return nz(h);
}

EXS_HD inline bool set_insert(u64* set, u32 mask, u64 k) {
  u32 h = (u32)mix64(k) & mask;
  for (u32 probes = 0; probes <= mask; probes++) {
    unsigned long long prev = at_cas64((unsigned long long*)&set[h], 0ull, (unsigned long long)k);
    if (prev == 0ull) return true;
    if (prev == k) return false;
    h = (h + 1) & mask;
  }
  return false;
}

// out of line: called from many sites, executed at a small fraction of them
EXS_HD EXS_NOINLINE void emit_diag(const WalkBufs& B, Diag d) {
  // a full buffer means the batch is re-run with a larger one: stop early
  // instead of probing an ever fuller dedup set
  if (ld_volatile(B.n_diags) >= B.cap_diags) { at_or(B.overflow, 2); return; }
  u64 h = diag_hash(d);
  if (!set_insert(B.dset, B.dmask, h)) return;
  u32 i = at_inc_agg(B.n_diags);
  if (i < B.cap_diags) B.diags[i] = d;
  else at_or(B.overflow, 2);
}
EXS_HD inline Diag mkdiag(u32 file, u32 line, u32 col, u16 code, u16 msg, u64 a0 = 0, u64 a1 = 0,
                          u64 a2 = 0, u32 a3 = 0, u8 sup = 0) {
  Diag d;
  d.file = file; d.line = line; d.col = col; d.code = code; d.msg = msg;
  d.a0 = a0; d.a1 = a1; d.a2 = a2; d.a3 = a3; d.suppressed = sup; d.pad0 = d.pad1 = d.pad2 = 0;
  return d;
}

// ---------------------------------------------------------------------------
// instance table

EXS_HD inline bool ikey_cas(IKey* slot, const IKey& k, IKey& old) {
#if EXS_DEV_PATH
  IKey empty; empty.a = 0; empty.b = 0;
  old = atomicCAS(slot, empty, k);
#else
  old = *slot;
  if (old.a == 0 && old.b == 0) *slot = k;
#endif
  return old.a == 0 && old.b == 0;
}
// Lookup-or-insert of an instance key.  The inserter allocates the id and
// publishes it in sid[slot]; the record itself is only read by later kernels
// (kernel boundaries order it), so no fence is needed -- other creators of
// the same level need the id alone, and "created in this level" is
// id >= lvl_base (ids are allocated monotonically).
EXS_HD inline u32 inst_lookup_or_insert(const WalkBufs& B, const IKey& k, bool& inserted, u32& slot) {
  u32 h = (u32)mix64(k.a ^ mix64(k.b)) & B.mask;
  inserted = false;
  // the table holds 2x the id capacity, so probing stays short even past an
  // overflow (then every insert fails to get an id and the walk is re-run)
  for (u32 probes = 0; probes <= B.mask; probes++) {
    IKey old;
    if (ikey_cas(&B.slots[h].k, k, old)) {
      u32 id = at_inc_agg(B.n_inst);
      if (id >= B.cap_inst) { at_or(B.overflow, 1u); id = NONE; }
      inserted = true;
      slot = h;
      return id;  // caller initialises the record, then publishes sid[slot]
    }
    if (old.a == k.a && old.b == k.b) {
      u32 id;
      while ((id = ld_volatile(&B.slots[h].sid)) == NONE) {
        if (ld_volatile(B.overflow) & 1u) return NONE;
      }
      slot = h;
      return id;
    }
    h = (h + 1) & B.mask;
  }
  at_or(B.overflow, 1u);
  return NONE;
}
EXS_HD inline void inst_publish(const WalkBufs& B, u32 slot, u32 id) {
  *(volatile u32*)&B.slots[slot].sid = id;
}

// instance key and record (spacecheck.py:325-341)
EXS_HD inline IKey make_ikey(u32 sig_rep, const Val& tb, const Val& hb, const Val& ot, u32 walk, u8 side) {
  IKey k;
  k.a = ((u64)sig_rep << 32) | tcode(tb);
  k.b = (1ull << 63) | ((u64)tcode(ot) << 32) | ((u64)walk << 3) |
        ((u64)(hb.k == V_HDC ? hb.x : 0) << 1) | side;
  return k;
}
EXS_HD inline void fill_instance(Inst& I, const Tables* T, const IKey& k, u32 fi, const Val& tb, const Val& hb,
                                 u8 side, u32 orec, const Val& ot, u32 at_tok, u32 walk, u8 sp, u32 slot) {
  const FnRec& fr = T->fns[fi];
  I.ka = k.a; I.kb = k.b;
  I.ckey = ~0ull; I.fn = fi; I.orec = orec; I.walk = walk; I.at = at_tok;
  I.ebase = 0; I.ecnt = 0;
  I.tb = tb; I.hb = hb; I.ot = ot;
  I.side = side; I.spaces = sp; I.pad = 0; I.slot = slot;
  // IF_BODY: a body to walk -- statements or parameter types to resolve (an
  // empty, parameterless body creates nothing and reports nothing)
  I.flags = (fr.flags & FR_BODY) ? IF_BODY : 0;
  if (fr.flags & FR_MAIN) I.flags |= IF_MAIN;
}
// an instance of main (the per-walk main is picked from these after the walk)
EXS_HD inline void note_main(const WalkBufs& B, u32 id) {
  const u32 k = at_add(B.n_mains, 1u);
  if (k < B.cap_mains) B.mains[k] = id;
}
// key insertion without an id (the level-0 roots allocate ids by a scan
// afterwards instead of one shared counter): the slot, NONE if the table is full
EXS_HD inline u32 slot_insert(const WalkBufs& B, const IKey& k, bool& inserted) {
  u32 h = (u32)mix64(k.a ^ mix64(k.b)) & B.mask;
  inserted = false;
  for (u32 probes = 0; probes <= B.mask; probes++) {
    IKey old;
    if (ikey_cas(&B.slots[h].k, k, old)) { inserted = true; return h; }
    if (old.a == k.a && old.b == k.b) return h;
    h = (h + 1) & B.mask;
  }
  at_or(B.overflow, 1u);
  return NONE;
}

// The part of _instantiate (spacecheck.py:312-351) after effective_spaces:
// look up or insert the key, fill a new record, and keep the minimum creation
// key of this level (with a log entry for a non-inserting creator that lowered
// it; the post-level fixup applies the entry whose key equals the minimum).
EXS_HD EXS_FI u32 create_instance(const WalkBufs& B, const Tables* T, u32 fi, const Val& tb, const Val& hb,
                                  u8 want_side, u32 orec, const Val& ot, u32 at_tok, u32 walk, u8 sp,
                                  unsigned long long ck) {
  const FnRec& fr = T->fns[fi];
  const IKey k = make_ikey(fr.sig_rep, tb, hb, ot, walk, want_side);
  bool inserted;
  u32 slot;
  u32 id = inst_lookup_or_insert(B, k, inserted, slot);
  if (id == NONE) return NONE;
  if (inserted) {
    fill_instance(B.inst[id], T, k, fi, tb, hb, want_side, orec, ot, at_tok, walk, sp, slot);
    inst_publish(B, slot, id);
    if (fr.flags & FR_MAIN) note_main(B, id);
  }
  if (id >= B.lvl_base) {
    // a creator in this level: the minimum creation key wins.  A creator
    // logs (ckey, location, decl) only if it lowered the minimum when it
    // arrived -- the final winner always did -- and not if it inserted (the
    // record already holds its data).  The post-level fixup applies the log
    // entry whose key equals the final minimum; none matches when the
    // inserter holds it.
    const unsigned long long old = at_min64(&B.slots[slot].sck, ck);
    if (inserted || old < ck) return id;
    u32 li = at_inc_agg(B.n_log);
    if (li < B.cap_log) {
      CreateLog& L = B.log[li];
      L.ckey = ck; L.inst = id; L.at = at_tok; L.fn = fi;
    } else {
      at_or(B.overflow, 4);
    }
  }
  return id;
}

// effective_spaces (sema.py:670-703) of a declaration whose specifiers need no
// evaluation (everything but proposal1 conditional specifiers): 1 H 2 D 3 HD 4 G.
// sf: specifier bits of the owning struct (0 for free functions).
EXS_HD inline u8 static_spaces(u16 fl, bool free_main, u16 sf, u8 mode, u8 side) {
  if (fl & FF_G) return 4;
  if (mode == MODE_P2) {
    if (free_main) return 1;
    if (!(fl & (FF_H | FF_D | FF_G))) {
      if (sf & (SF_H | SF_D | SF_G)) fl = sf;
      else return (u8)(1u << side);
    }
  }
  u8 sp = 0;
  if (fl & FF_H) sp |= 1;
  if (fl & FF_D) sp |= 2;
  return sp ? sp : 1;
}

// ---------------------------------------------------------------------------

// verdict table (spacecheck.py:86-132) for direct calls; callee 1=H 2=D
// returns a code or 0 (legal)
EXS_HD inline u16 verdict(u8 side, u8 callee, bool from_hd, u8 mode, bool reachable) {
  if (callee == 3 || callee == (1u << side)) return 0;
  bool host_only = callee == 1;
  if (!from_hd) {
    if (mode == MODE_P2) return C_E1501;
    return side == 0 ? C_E1001 : C_E1002;
  }
  if (mode == MODE_FIDELITY && !host_only) return 0;
  if (mode == MODE_SOUND && reachable) return host_only ? C_E1101 : C_E1102;
  if (mode == MODE_P2) return reachable ? C_E1501 : C_W1502;
  return host_only ? C_W1101 : C_W1102;
}
EXS_HD inline bool hard_code(u16 c) {
  return c == C_E0001 || c == C_E0002 || c == C_E0101 || c == C_E0102 || c == C_E0103 ||
         c == C_E0104 || c == C_E1301 || c == C_E1302;
}

// per-thread bounds; a unit beyond them is reported as out of contract (X9999)
#define MAX_LOCALS 16
#define MAX_WALK_DEPTH 160
#define MAX_ARGS 16
// call dispatch inline (C2 1 GB: walk_chunks 29.9 -> 25.8 ms against out of
// line: the call frames' register saves were local-memory traffic);
// EXS_DISPATCH_OUTLINE restores the smaller kernel
#ifdef EXS_DISPATCH_OUTLINE
#define EXS_DISPATCH EXS_NOINLINE
#else
#define EXS_DISPATCH EXS_FI
#endif

struct Walker {
  Sema S;
  const WalkBufs* B;
  const Tables* T;
  u32 file, walk, inst_id;
  u8 native, side, spaces;   // side 0 host 1 device; spaces bits 1 H 2 D 4 G
  u32 clevel;                // level of the instances this walker creates
  u32 fn;                    // decl of the instance
  bool pragma, from_hd, fidelity_host;
  u64 parent_rank;           // dense rank of this instance within its level
  u32 stmt_k, stmt_ord;      // top-level statement, instantiations in it so far
  u32 stmt_ord_max;          // 2 x call sites of the statement (bound of stmt_ord)
  u32 ebase, ecnt;           // edge slots of this instance, legal edges written
  u32 stmt_cs_base, cs_ord;  // edge slot of the current statement, edges in it so far
  bool silent;               // replaying declarations of earlier chunks: no side effects
  bool contract;
  int wdepth;
  u32 nloc;                  // locals in scope
  u32 asp;                   // argument-stack depth
  Env env;                   // owner bindings + bindings
  // the arrays last: a statement without locals or arguments (most of them)
  // touches only the lines above (the walker lives in local memory)
  u64 lname[MAX_LOCALS];     // locals (scoped dict)
  Val lval[MAX_LOCALS];
  Val astk[MAX_ARGS];        // argument types of the calls being walked (shared by all frames)

  EXS_HD const Node& N(u32 id) const { return T->nodes[id]; }
  EXS_HD const Tok& K(u32 t) const { return T->toks[t]; }
  EXS_HD u64 span(u32 t) const { return S.span(t); }

  EXS_HD void emit(u16 code, u32 line, u32 col, u16 msg, u64 a0 = 0, u64 a1 = 0, u64 a2 = 0,
                   u32 a3 = 0) {
    if (silent || (fidelity_host && !hard_code(code))) return;
    emit_diag(*B, mkdiag(file, line, col, code, msg, a0, a1, a2, a3));
  }
  EXS_HD void emit_tok(u16 code, u32 tok, u16 msg, u64 a0 = 0, u64 a1 = 0, u64 a2 = 0, u32 a3 = 0) {
    emit(code, K(tok).line, K(tok).col, msg, a0, a1, a2, a3);
  }
  EXS_HD void emit_err() {  // a SemaError from the evaluator
    emit(S.err.code, S.err.line, S.err.col, S.err.msg, S.err.a0, S.err.a1, S.err.a2);
  }

  // display-name arguments of a decl: (name span, owner span or 0)
  EXS_HD u64 owner_span(u32 fi) const {
    const FnRec& fr = T->fns[fi];
    return (fr.flags & FR_OWNER) ? span(N(T->recs[fr.rec].node).tok) : 0;
  }

  // ------------------------------------------------------------- locals
  EXS_HD bool local_get(u64 name, Val& v) const {
    for (int i = (int)nloc - 1; i >= 0; i--)
      if (lname[i] == name) { v = lval[i]; return true; }
    return false;
  }
  EXS_HD void local_set(u64 name, const Val& v) {
    if (nloc < MAX_LOCALS) { lname[nloc] = name; lval[nloc] = v; nloc++; }
    else contract = true;
  }

  // _resolve_type_soft (spacecheck.py:363-370)
  EXS_HD EXS_FI Val soft_type(u32 tr, u32 loc_tok) {
    Val t;
    S.depth = 0;
    u8 st = S.type_of(tr, env, t);
    if (S.contract) { contract = true; return vnone(); }
    if (st == ST_OK) return t;
    if (st == ST_SEMA) emit_err();
    else emit_tok(C_E0101, loc_tok, M_W_NOT_TYPE, span(N(tr).tok));
    return vnone();
  }

  // ------------------------------------------------------------- instantiate
  // _instantiate (spacecheck.py:312-351); returns instance id or NONE
  EXS_HD EXS_FI u32 instantiate(u32 fi, const Val& tb, const Val& hb, u8 want_side, u32 orec,
                         const Env& obinds, const Val& ot, u32 at_tok) {
    // creation order (make_ckey): a field past its width is out of contract
    const u32 ord = stmt_ord++;
    const u64 my_local = 2ull * stmt_cs_base + ord;
    if (ord >= stmt_ord_max || my_local > CK_FIELD_MAX || parent_rank > CK_FIELD_MAX || clevel > CK_LEVEL_MAX) {
      contract = true;
      return NONE;
    }
    u8 sp;
    S.depth = 0;
    u8 st = S.spaces(fi, &obinds, tb, hb, want_side, at_tok, orec, sp);
    if (S.contract) { contract = true; return NONE; }
    if (st == ST_SEMA) { emit_err(); return NONE; }
    if (st == ST_SUBST) { emit_tok(C_E0001, at_tok, M_W_PRED_CONST); return NONE; }
    const unsigned long long ck = make_ckey(clevel, parent_rank, (u32)my_local);
    return create_instance(*B, T, fi, tb, hb, want_side, orec, ot, at_tok, walk, sp, ck);
  }

  EXS_HD void add_binds(const Node& fnn, const Val& tb, const Val& hb, Env& e) const {
    for (u32 tp = fnn.c0; tp != NONE; tp = N(tp).next) {
      const Val& v = N(tp).sub == 0 ? tb : hb;
      if (v.k != V_NONE) e.add(N(tp).hv, v);
    }
  }

  // ------------------------------------------------------------- dispatch
  // _report_stray (spacecheck.py:604-613); callee 1=H 2=D
  EXS_HD EXS_FI void stray(u8 callee, u32 loc_tok) {
    if (from_hd) {
      u32 i = at_inc_agg(B->n_pend);
      if (i < B->cap_pend) {
        Pending& p = B->pend[i];
        p.walk = walk; p.caller = inst_id; p.line = K(loc_tok).line; p.col = K(loc_tok).col;
        p.callee = callee;
      } else {
        at_or(B->overflow, 4);
      }
      return;
    }
    u16 code = verdict(side, callee, false, S.mode, true);
    emit_tok(code, loc_tok, M_W_STRAY, callee, side, 0);
  }

  // _dispatch (spacecheck.py:554-596)
  EXS_HD EXS_FI void dispatch(u32 fi, const Val& tb, const Val& hb, u32 loc_tok, u32 orec,
                       const Env& obinds, const Val& ot) {
    const Node& fnn = N(T->fns[fi].node);
    u8 sp;
    S.depth = 0;
    u8 st = S.spaces(fi, &obinds, tb, hb, side, loc_tok, orec, sp);
    if (S.contract) { contract = true; return; }
    if (st == ST_SEMA) { emit_err(); return; }
    if (st == ST_SUBST) { emit_tok(C_E0001, loc_tok, M_W_PRED_CONST); return; }
    if (sp == 4) { emit_tok(C_E1004, loc_tok, M_W_GLOBAL_CALL); return; }
    bool relaxed_ok = S.relaxed && (fnn.n & FF_CX);
    bool legal = relaxed_ok || (sp & (1u << side));
    u8 want = legal ? side : ((sp & 1) ? 0 : 1);
    u32 callee = instantiate(fi, tb, hb, want, orec, obinds, ot, loc_tok);
    if (legal && callee != NONE) {
      // slot: post-order position inside the statement, statements in order
      B->edges[ebase + stmt_cs_base + cs_ord] = callee;
      cs_ord++;
      ecnt++;
    }
    if (!legal) stray(sp == 1 ? 1 : 2, loc_tok);
    bool tmpl = fnn.c0 != NONE;
    if ((S.mode == MODE_CLASSIC || S.mode == MODE_FIDELITY || S.mode == MODE_P1) && sp == 3 &&
        (tmpl || ot.k != V_NONE))
      instantiate(fi, tb, hb, native, orec, obinds, ot, loc_tok);
  }

  // _select + overload resolution (sema.py:491-542); cand list given as
  // (free: fcand run) or (member: struct rec).  Returns false on failure.
  EXS_HD EXS_FI bool select(bool member, u32 first, u32 count, u32 rec, u64 mname, u32 targs,
                     const Val* argtys, u32 nargs, u32 loc_tok, u8 ctx_side, const Env& obinds,
                     u64 name_a0, u64 name_a1, u32& out_fi, Val& out_tb, Val& out_hb,
                     u32 name_targ = 0) {
    u32 nviable = 0;
    u32 vfi[8];
    Val ftb = vnone(), fhb = vnone();  // bindings of the first viable candidate
    u32 i = 0;
    u32 m = member ? N(T->recs[rec].node).c1 : NONE;
    while (true) {
      u32 fi;
      if (member) {
        // member functions with this name, in member order (dups were removed)
        while (m != NONE) {
          const Node& mn = N(m);
          if (mn.kind == N_FN && mn.hv == mname) {
            u32 fx = N(m + 1).tok;  // FNX.tok holds the decl record index
            if (!(T->fns[fx].flags & FR_DUP)) break;
          }
          m = mn.next;
        }
        if (m == NONE) break;
        fi = N(m + 1).tok;
        m = N(m).next;
      } else {
        if (i >= count) break;
        fi = T->fcand[first + i];
        i++;
      }
      Sema::Binds b;
      S.depth = 0;
      u8 st = S.try_cand(fi, targs, argtys, nargs, env, member ? rec : NONE, obinds, b);
      if (S.contract) { contract = true; return false; }
      if (st == ST_SEMA) { emit_err(); return false; }
      if (st == ST_SUBST) continue;
      if (nviable < 8) vfi[nviable] = fi;
      if (nviable == 0) split_binds(fi, b, ftb, fhb);
      nviable++;
    }
    u32 first_ok = nviable ? vfi[0] : NONE;
    // the proposal2 space filter keeps the first 8 survivors: more is out of contract
    if (S.mode == MODE_P2 && nviable > 8) { contract = true; return false; }
    if (S.mode == MODE_P2 && nviable > 1) {
      u32 nc = 0;
      for (u32 j = 0; j < nviable; j++)
        if (S.compatible(vfi[j], ctx_side, member ? rec : NONE)) vfi[nc++] = vfi[j];
      if (nc) nviable = nc;
    }
    if (nviable == 0) { emit_tok(C_E1301, loc_tok, M_S_NO_VIABLE, name_a0, name_a1, 0, name_targ); return false; }
    if (nviable > 1) { emit_tok(C_E1302, loc_tok, M_S_AMBIGUOUS, name_a0, name_a1, nviable, name_targ); return false; }
    out_fi = vfi[0];
    if (out_fi == first_ok) { out_tb = ftb; out_hb = fhb; return true; }
    // the space filter chose a later candidate: re-derive its bindings
    Sema::Binds b;
    S.depth = 0;
    S.try_cand(out_fi, targs, argtys, nargs, env, member ? rec : NONE, obinds, b);
    split_binds(out_fi, b, out_tb, out_hb);
    return true;
  }
  EXS_HD void split_binds(u32 fi, const Sema::Binds& b, Val& tb, Val& hb) const {
    tb = vnone(); hb = vnone();
    const Node& fnn = N(T->fns[fi].node);
    for (u32 tp = fnn.c0; tp != NONE; tp = N(tp).next) {
      Val v;
      if (b.get(N(tp).hv, v)) {
        if (N(tp).sub == 0) tb = v; else hb = v;
      }
    }
  }

  // ------------------------------------------------------------- expressions
  EXS_HD u32 count_list(u32 l) const {
    u32 c = 0;
    for (; l != NONE; l = N(l).next) c++;
    return c;
  }

  // walk args (post-order) pushing their types on the argument stack; the
  // caller pops with asp = base after dispatching
  EXS_HD EXS_FI u32 walk_args(u32 args, u32& base) {
    base = asp;
    u32 n = 0;
    for (u32 a = args; a != NONE; a = N(a).next) {
      Val t = expr(a);
      if (asp < MAX_ARGS) astk[asp++] = t;
      else contract = true;
      n++;
    }
    return n;
  }

  // a work item's top-level statement: its expression root is walked inline
  // (no call frame for stmt/expr); nested statements and sub-expressions recurse
  EXS_HD EXS_FI void stmt_top(u32 s) {
    const Node& n = N(s);
    if (n.kind == N_SEXPR || (n.kind == N_SRET && n.c0 != NONE)) {
      if (++wdepth > MAX_WALK_DEPTH) { contract = true; wdepth--; return; }
      expr_<1>(n.c0);
      wdepth--;
    } else if (n.kind != N_SRET) {
      stmt(s);
    }
  }

  EXS_HD Val expr(u32 e) {
    if (++wdepth > MAX_WALK_DEPTH) { contract = true; wdepth--; return vnone(); }
    Val r = expr_<0>(e);
    wdepth--;
    return r;
  }

  // TOP = 1: the copy inlined into a work item's top-level statement (not
  // recursive itself: sub-expressions go through expr); TOP = 0: expr's body
  template <int TOP>
  EXS_HD EXS_FI Val expr_(u32 e) {
    const Node& n = N(e);
    switch (n.kind) {
      case N_INT: { Val t = vnone(); t.k = V_TYPE; t.bt = BT_INT; t.x = H_INT; return t; }
      case N_BOOL:
      case N_ARCH: { Val t = vnone(); t.k = V_TYPE; t.bt = BT_BOOL; t.x = H_BOOL; return t; }
      case N_STR:
      case N_HDCV: return vnone();
      case N_NAME: {
        u64 nm = n.hv;
        Val v;
        if (local_get(nm, v)) return v;
        for (int i = 0; i < env.n; i++)
          if (env.names[i] == nm) return vnone();
        emit_tok(C_E0101, n.tok, M_S_UNDEF_NAME, span(n.tok));
        return vnone();
      }
      case N_TMP: return soft_type(n.c0, n.tok);
      case N_TRAIT: {
        Val t;
        S.depth = 0;
        u8 st = S.type_of(n.c0, env, t);
        if (st == ST_OK) {
          Val h;
          st = S.trait(t, S.fund, h);
        }
        if (S.contract) { contract = true; return vnone(); }
        if (st == ST_SEMA) emit_err();
        return vnone();
      }
      case N_MCONST: {
        Val v;
        S.depth = 0;
        u8 st = S.eval(e, env, S.fund, v);
        if (S.contract) { contract = true; return vnone(); }
        if (st == ST_SEMA) emit_err();
        else if (st == ST_SUBST)
          emit_tok(C_E0101, N(n.c0).tok, M_W_SUBST, S.err.a0, S.err.a1, S.err.a2, S.err.msg);
        return vnone();
      }
      case N_NOT: {
        expr(n.c0);
        Val t = vnone(); t.k = V_TYPE; t.bt = BT_BOOL; t.x = H_BOOL;
        return t;
      }
      case N_BIN: {
        expr(n.c0);
        expr(n.c1);
        Val t = vnone(); t.k = V_TYPE; t.bt = BT_BOOL; t.x = H_BOOL;
        return t;
      }
      case N_CALL: return free_call(e);
      case N_MCALL: {
        u32 recv = n.c0;
        // a temporary receiver (T{}.f()) is typed in place, without a call frame
        Val rt;
        if (N(recv).kind == N_TMP && wdepth < MAX_WALK_DEPTH) rt = soft_type(N(recv).c0, N(recv).tok);
        else rt = expr(recv);
        u8 rk = N(recv).kind;
        if (rt.k == V_NONE && rk != N_TMP && rk != N_NAME)
          emit_tok(C_E0001, S.loc_tok(recv), M_W_RECEIVER);
        u32 base;
        u32 na = walk_args(n.c2, base);
        if (rt.k != V_NONE && !contract) member_dispatch(rt, n.tok, n.c1, astk + base, na, S.loc_tok(e));
        asp = base;
        return vnone();
      }
      case N_SCALL: {
        u32 base;
        u32 na = walk_args(n.c2, base);
        Val t = soft_type(n.c0, N(n.c0).tok);
        if (t.k != V_NONE && !contract) member_dispatch(t, n.tok, n.c1, astk + base, na, N(n.c0).tok);
        asp = base;
        return vnone();
      }
      default:
        return vnone();
    }
  }

  EXS_HD EXS_FI Val free_call(u32 e) {
    const Node& n = N(e);
    u32 base;
    u32 na = walk_args(n.c2, base);
    Val r = contract ? vnone() : free_call_(n, astk + base, na);
    asp = base;
    return r;
  }
  EXS_HD EXS_DISPATCH Val free_call_(const Node& n, const Val* tys, u32 na) {
    bool is_std = n.sub == CALL_STD;
    u64 nm = is_std ? hcombine(H_STD, K(n.c0).hv) : n.hv;
    u32 run = is_std ? NONE : T->fmap.find(vkey(S.view, nm));
    if (run == NONE) {
      // builtin_spaces (sema.py:99-102)
      u8 w = is_std ? (K(n.c0).id == W_ABORT ? (u8)0xFE : (u8)0) : K(n.tok).id;
      u8 sp = 0;
      if (w == W_PRINTF || w == W_RELEASE_ASSERT) sp = 3;
      else if (w == W_TRAP) sp = S.plain ? 0 : 2;
      else if (w == W_ABORT || w == 0xFE) sp = 1;
      else if (w == W_CUDASYNC) sp = S.plain ? 0 : 1;
      if (sp) {
        if (!(sp & (1u << side))) stray(sp == 1 ? 1 : 2, n.tok);
        if (w == W_CUDASYNC) { Val t = vnone(); t.k = V_TYPE; t.bt = BT_INT; t.x = H_INT; return t; }
      }
      return vnone();
    }
    u32 fi; Val tb, hb;
    Env none; none.clear();
    if (select(false, run, T->fcand_cnt[run], NONE, 0, n.c1, tys, na, n.tok, side, none,
               span(n.tok), 0, fi, tb, hb))
      dispatch(fi, tb, hb, n.tok, NONE, none, vnone());
    return vnone();
  }

  // _member_dispatch (spacecheck.py:529-550)
  EXS_HD EXS_DISPATCH void member_dispatch(const Val& rt, u32 name_tok, u32 targs, const Val* tys, u32 na,
                              u32 loc_tok) {
    u64 mname = K(name_tok).hv;
    u64 tname = S.type_name_arg(rt);
    u64 targ_arg = rt.targ;
    bool any = false;
    if (rt.rec != NONE) {
      for (u32 m = N(T->recs[rt.rec].node).c1; m != NONE; m = N(m).next) {
        const Node& mn = N(m);
        if (mn.kind == N_FN && mn.hv == mname && !(T->fns[N(m + 1).tok].flags & FR_DUP)) { any = true; break; }
      }
    }
    if (!any) {
      emit_tok(C_E0101, loc_tok, M_W_NO_MEMBER, tname, span(name_tok), targ_arg);
      return;
    }
    Env ob;
    S.struct_env(rt.rec, rt, ob);
    u32 fi; Val tb, hb;
    // name for messages: "{type display}::{name}"
    if (select(true, 0, 0, rt.rec, mname, targs, tys, na, loc_tok, side, ob,
               span(name_tok), tname, fi, tb, hb, rt.targ))
      dispatch(fi, tb, hb, loc_tok, rt.rec, ob, rt);
  }

  // ------------------------------------------------------------- statements
  EXS_HD void stmts(u32 s) {
    for (; s != NONE; s = N(s).next) {
      if (contract) return;
      stmt(s);
    }
  }
  EXS_HD void stmt(u32 s) {
    const Node& n = N(s);
    switch (n.kind) {
      case N_SEXPR: expr(n.c0); break;
      case N_SRET: if (n.c0 != NONE) expr(n.c0); break;
      case N_SVAR: {
        Val t = soft_type(n.c0, N(n.c0).tok);
        local_set(n.hv, t);
        break;
      }
      case N_SIF: {
        expr(n.c0);
        u32 mark = nloc;
        stmts(n.c1);
        nloc = mark;
        if (n.sub) { stmts(n.c2); nloc = mark; }
        break;
      }
      case N_SFOR: {
        expr(n.c0);
        expr(n.c1);
        u32 mark = nloc;
        Val t = vnone(); t.k = V_TYPE; t.bt = BT_INT; t.x = H_INT;
        local_set(n.hv, t);
        stmts(n.c2);
        nloc = mark;
        break;
      }
      case N_SLAUNCH: launch(s); break;
      default: break;
    }
  }

  // _walk_launch (spacecheck.py:395-415)
  EXS_HD void launch(u32 s) {
    const Node& n = N(s);
    u32 grid = n.c1;
    expr(grid);
    expr(N(grid).next);
    u32 base;
    u32 na = walk_args(n.c2, base);
    if (side == 1) emit_tok(C_E1003, n.tok, M_W_LAUNCH_DEVICE);
    if (!contract) launch_dispatch(n, astk + base, na);
    asp = base;
  }
  EXS_HD EXS_DISPATCH void launch_dispatch(const Node& n, const Val* tys, u32 na) {
    u32 run = T->fmap.find(vkey(S.view, n.hv));
    if (run == NONE) return;
    u32 fi; Val tb, hb;
    Env none; none.clear();
    bool ok = select(false, run, T->fcand_cnt[run], NONE, 0, n.c0, tys, na, n.tok, 1, none,
                     span(n.tok), 0, fi, tb, hb);
    if (!ok) return;
    if (!(N(T->fns[fi].node).n & FF_G)) { emit_tok(C_E1004, n.tok, M_W_LAUNCH_NONGLOBAL); return; }
    u32 tgt = instantiate(fi, tb, hb, 1, NONE, none, vnone(), n.tok);
    if (tgt != NONE && side == 0) {
      u32 i = at_inc_agg(B->n_seeds);
      if (i < B->cap_seeds) { B->seeds[2 * i] = walk; B->seeds[2 * i + 1] = tgt; }
      else at_or(B->overflow, 4);
    }
  }

  // _walk_instance (spacecheck.py:355-361) over top-level statements
  // [k0, k1) of the body.  A chunk that does not start the body first
  // replays, silently, the parameter and top-level declarations before it
  // (only those reach later statements: nested blocks are scoped).
  EXS_HD void run_chunk(const u32* stmt_node, const u32* stmt_cs, u32 sbase, u32 k0, u32 k1) {
    const Node& fnn = N(T->fns[fn].node);
    nloc = 0;
    wdepth = 0;
    asp = 0;
    silent = k0 != 0;
    for (u32 p = fnn.c1; p != NONE; p = N(p).next) {
      Val t = soft_type(N(p).c0, N(p).tok);
      local_set(N(p).hv, t);
    }
    if (T->fns[fn].flags & FR_VARDECL) {
      for (u32 k = 0; k < k0; k++) {
        const Node& s = N(stmt_node[sbase + k]);
        if (s.kind == N_SVAR) local_set(s.hv, soft_type(s.c0, N(s.c0).tok));
      }
    }
    silent = false;
    const FnRec& fr = T->fns[fn];
    for (u32 k = k0; k < k1 && !contract; k++) {
      stmt_k = k;
      stmt_ord = 0;
      stmt_cs_base = stmt_cs[sbase + k];
      stmt_ord_max = 2u * ((k + 1 < fr.nstmts ? stmt_cs[sbase + k + 1] : fr.ncalls) - stmt_cs_base);
      cs_ord = 0;
      stmt_top(stmt_node[sbase + k]);
    }
  }
};

}  // namespace exs
