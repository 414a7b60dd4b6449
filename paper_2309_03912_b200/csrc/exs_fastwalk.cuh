// exs_fastwalk.cuh -- K6 fast path: one top-level statement of the common
// shapes walked with register-resident state.
//
// The general walker (exs_walk.cuh Walker) is recursive: its state, its call
// frames and the evaluator's frames live in local memory, which at ~1K
// resident threads per SM is the walk kernel's DRAM traffic (profiles/r01_*).
// Nearly every statement of the measured corpora has one of four shapes:
//   name< targs >();          free call, no arguments      (spacecheck.py:420-447)
//   T{}.name< targs >();      member call on a temporary   (spacecheck.py:449-550)
//   builtin();                cudaDeviceSynchronize/__trap/abort (sema.py:99-102)
//   k<<< lit, lit >>>();      kernel launch, no arguments  (spacecheck.py:395-415)
// with candidates that bind every template parameter from explicit type
// arguments, no requires clause and no conditional specifier.  Those are
// walked here, inline, with the same steps in the same order as the general
// walker (overload selection, _dispatch, _instantiate with its creation key,
// the edge slot, _report_stray); everything else -- and any step that would
// raise a diagnostic other than the verdicts -- is left to the general walker
// BEFORE any side effect, so the result never depends on which path ran.
#pragma once
#include "exs_walk.cuh"

namespace exs {

struct FastEnv {  // walker env: owner HDC binding + the instance's bindings (<= 3)
  u32 n;
  u64 names[3];
  Val vals[3];
  // constant indices only (unrolled): the env stays in registers
  EXS_HD EXS_FI void add(u64 name, const Val& v) {
#pragma unroll
    for (int i = 0; i < 3; i++)
      if ((u32)i == n) { names[i] = name; vals[i] = v; }
    if (n < 3) n++;
  }
  EXS_HD EXS_FI bool get(u64 name, Val& out) const {
    bool hit = false;
#pragma unroll
    for (int i = 2; i >= 0; i--)
      if (!hit && (u32)i < n && names[i] == name) { out = vals[i]; hit = true; }
    return hit;
  }
};

struct FastWalk {
  const Tables* T;
  const WalkBufs* B;
  u32 view, file, walk, inst_id, ebase;
  u32 clevel;
  u64 parent_rank;
  u8 side, native, mode, plain, relaxed;
  bool from_hd, fidelity_host;
  u32 stmt_cs_base, stmt_ord, stmt_ord_max, cs_ord, ecnt;
  bool contract;
  FastEnv env;

  EXS_HD EXS_FI const Node& N(u32 id) const { return T->nodes[id]; }
  EXS_HD EXS_FI const Tok& K(u32 t) const { return T->toks[t]; }

  EXS_HD EXS_FI void emit(u16 code, u32 tok, u16 msg, u64 a0 = 0, u64 a1 = 0, u64 a2 = 0) {
    if (fidelity_host && !hard_code(code)) return;
    emit_diag(*B, mkdiag(file, K(tok).line, K(tok).col, code, msg, a0, a1, a2, 0));
  }

  // resolve_type of a type argument or temporary (sema.py:333-363), the cases
  // without a diagnostic or substitution failure: false = not handled here
  EXS_HD EXS_FI bool type_of(u32 tr, Val& out) const {
    const Node& t = N(tr);
    const u8 bt = t.sub;
    if (bt == BT_INT || bt == BT_BOOL || bt == BT_VOID) {
      if (t.c0 != NONE) return false;
      out = vnone(); out.k = V_TYPE; out.bt = bt; out.x = t.hv; out.rec = NONE;
      return true;
    }
    if (bt == BT_HDC) return false;
    Val b;
    if (env.get(t.hv, b)) {
      if (b.k != V_TYPE || t.c0 != NONE) return false;
      out = b;
      return true;
    }
    const u32 rec = T->smap.find(vkey(view, t.hv));
    if (rec == NONE || t.c0 != NONE) return false;
    if (N(T->recs[rec].node).c0 != NONE) return false;  // struct template: evaluated by the general walker
    out = vnone(); out.k = V_TYPE; out.bt = BT_NONE; out.rec = rec; out.x = t.hv; out.targ = 0;
    return true;
  }

  // _try_candidate (sema.py:545-607) for a call without arguments: 1 viable
  // (tb bound), 0 not viable, -1 not handled here
  EXS_HD EXS_FI int try_cand(u32 fi, u32 targs, Val& tb) const {
    const FnRec& fr = T->fns[fi];
    const Node& fn = N(fr.node);
    u32 ntp = 0, nex = 0;
    for (u32 tp = fn.c0; tp != NONE; tp = N(tp).next) ntp++;
    for (u32 a = targs; a != NONE; a = N(a).next) nex++;
    if (nex > ntp) return 0;  // too many template arguments
    tb = vnone();
    u32 ta = targs;
    for (u32 tp = fn.c0; tp != NONE; tp = N(tp).next) {
      if (ta == NONE) return -1;               // a default or a deduction: general walker
      if (N(tp).sub != 0) return -1;           // HDC parameter: general walker
      if (N(ta).kind != N_TYPE) return 0;      // substitution failure
      if (!type_of(ta, tb)) return -1;
      ta = N(ta).next;
    }
    if (fn.sub != 0) return 0;                  // argument count mismatch
    if (N(fr.node + 1).c0 != NONE) return -1;   // requires clause: general walker
    return 1;
  }

  // free-call candidates (member == false) or the members named mname of
  // struct rec: exactly one viable candidate -> fi/tb, else false
  EXS_HD EXS_FI bool select(bool member, u32 run, u32 count, u32 rec, u64 mname, u32 targs, u32& fi_out,
                            Val& tb_out) const {
    u32 nviable = 0;
    u32 m = member ? N(T->recs[rec].node).c1 : NONE;
    u32 i = 0;
    while (true) {
      u32 fi;
      if (member) {
        while (m != NONE) {
          const Node& mn = N(m);
          if (mn.kind == N_FN && mn.hv == mname && !(T->fns[N(m + 1).tok].flags & FR_DUP)) break;
          m = mn.next;
        }
        if (m == NONE) break;
        fi = N(m + 1).tok;
        m = N(m).next;
      } else {
        if (i >= count) break;
        fi = T->fcand[run + i];
        i++;
      }
      Val tb;
      const int r = try_cand(fi, targs, tb);
      if (r < 0) return false;
      if (r == 0) continue;
      if (++nviable > 1) return false;  // ambiguity (or the proposal2 space filter): general walker
      fi_out = fi;
      tb_out = tb;
    }
    return nviable == 1;
  }

  // effective_spaces (sema.py:670-703) without conditional specifiers
  EXS_HD EXS_FI u8 spaces(u32 fi, u8 sd, u32 orec) const {
    const FnRec& fr = T->fns[fi];
    const Node& fn = N(fr.node);
    const u16 sf = orec != NONE ? N(T->recs[orec].node).n : 0;
    return static_spaces(fn.n, K(fn.tok).id == W_MAIN && !(fr.flags & FR_OWNER), sf, mode, sd);
  }

  // _instantiate (spacecheck.py:312-351)
  EXS_HD EXS_FI u32 instantiate(u32 fi, const Val& tb, u8 want_side, u32 orec, const Val& ot, u32 at_tok) {
    const u32 ord = stmt_ord++;
    const u64 my_local = 2ull * stmt_cs_base + ord;
    if (ord >= stmt_ord_max || my_local > CK_FIELD_MAX || parent_rank > CK_FIELD_MAX || clevel > CK_LEVEL_MAX) {
      contract = true;
      return NONE;
    }
    const u8 sp = spaces(fi, want_side, orec);
    const unsigned long long ck = make_ckey(clevel, parent_rank, (u32)my_local);
    return create_instance(*B, T, fi, tb, vnone(), want_side, orec, ot, at_tok, walk, sp, ck);
  }

  // _report_stray (spacecheck.py:604-613); callee 1 = H, 2 = D
  EXS_HD EXS_FI void stray(u8 callee, u32 loc_tok) {
    if (from_hd) {
      const u32 i = at_inc_agg(B->n_pend);
      if (i < B->cap_pend) {
        Pending& p = B->pend[i];
        p.walk = walk; p.caller = inst_id; p.line = K(loc_tok).line; p.col = K(loc_tok).col;
        p.callee = callee;
      } else {
        at_or(B->overflow, 4);
      }
      return;
    }
    emit(verdict(side, callee, false, mode, true), loc_tok, M_W_STRAY, callee, side, 0);
  }

  // _dispatch (spacecheck.py:554-596)
  EXS_HD EXS_FI void dispatch(u32 fi, const Val& tb, u32 loc_tok, u32 orec, const Val& ot) {
    const Node& fnn = N(T->fns[fi].node);
    const u8 sp = spaces(fi, side, orec);
    if (sp == 4) { emit(C_E1004, loc_tok, M_W_GLOBAL_CALL); return; }
    const bool legal = (relaxed && (fnn.n & FF_CX)) || (sp & (1u << side));
    const u8 want = legal ? side : ((sp & 1) ? 0 : 1);
    const u32 callee = instantiate(fi, tb, want, orec, ot, loc_tok);
    if (legal && callee != NONE) {
      B->edges[ebase + stmt_cs_base + cs_ord] = callee;
      cs_ord++;
      ecnt++;
    }
    if (!legal) stray(sp == 1 ? 1 : 2, loc_tok);
    if ((mode == MODE_CLASSIC || mode == MODE_FIDELITY || mode == MODE_P1) && sp == 3 &&
        (fnn.c0 != NONE || ot.k != V_NONE))
      instantiate(fi, tb, native, orec, ot, loc_tok);
  }

  // does the proposal1 conditional-specifier path apply to a candidate?
  EXS_HD EXS_FI bool cond_spec(u32 fi) const {
    return mode == MODE_P1 && (N(T->fns[fi].node).n & (FF_HPRED | FF_DPRED));
  }

  // one top-level statement; false = not handled (nothing was done)
  EXS_HD EXS_FI bool stmt(u32 s) {
    const Node& st = N(s);
    if (st.kind == N_SRET && st.c0 == NONE) return true;
    if (st.kind == N_SLAUNCH) return launch(st);
    if (st.kind != N_SEXPR && st.kind != N_SRET) return false;
    const u32 e = st.c0;
    const Node& n = N(e);
    if (n.c2 != NONE) return false;  // arguments: general walker
    if (n.kind == N_CALL) {
      if (n.sub == CALL_STD) return false;
      const u32 run = T->fmap.find(vkey(view, n.hv));
      if (run == NONE) {
        // builtin_spaces (sema.py:99-102); an unknown name was reported by resolve
        const u8 w = K(n.tok).id;
        u8 sp = 0;
        if (w == W_PRINTF || w == W_RELEASE_ASSERT) sp = 3;
        else if (w == W_TRAP) sp = plain ? 0 : 2;
        else if (w == W_ABORT) sp = 1;
        else if (w == W_CUDASYNC) sp = plain ? 0 : 1;
        if (sp && !(sp & (1u << side))) stray(sp == 1 ? 1 : 2, n.tok);
        return true;
      }
      u32 fi;
      Val tb;
      if (!select(false, run, T->fcand_cnt[run], NONE, 0, n.c1, fi, tb) || cond_spec(fi)) return false;
      dispatch(fi, tb, n.tok, NONE, vnone());
      return true;
    }
    if (n.kind == N_MCALL) {
      const Node& r = N(n.c0);
      if (r.kind != N_TMP) return false;
      Val rt;
      if (!type_of(r.c0, rt) || rt.rec == NONE) return false;
      u32 fi;
      Val tb;
      if (!select(true, 0, 0, rt.rec, K(n.tok).hv, n.c1, fi, tb) || cond_spec(fi)) return false;
      dispatch(fi, tb, r.tok, rt.rec, rt);  // loc: the receiver's (parser.py:548)
      return true;
    }
    return false;
  }

  EXS_HD EXS_FI bool literal(u32 e) const {
    const u8 k = N(e).kind;
    return k == N_INT || k == N_BOOL || k == N_STR || k == N_HDCV;
  }

  // _walk_launch (spacecheck.py:395-415)
  EXS_HD EXS_FI bool launch(const Node& n) {
    if (n.c2 != NONE || !literal(n.c1) || !literal(N(n.c1).next)) return false;
    const u32 run = T->fmap.find(vkey(view, n.hv));
    u32 fi = NONE;
    Val tb = vnone();
    if (run != NONE && (!select(false, run, T->fcand_cnt[run], NONE, 0, n.c0, fi, tb) || cond_spec(fi)))
      return false;
    if (side == 1) emit(C_E1003, n.tok, M_W_LAUNCH_DEVICE);
    if (run == NONE) return true;
    if (!(N(T->fns[fi].node).n & FF_G)) { emit(C_E1004, n.tok, M_W_LAUNCH_NONGLOBAL); return true; }
    const u32 tgt = instantiate(fi, tb, 1, NONE, vnone(), n.tok);
    if (tgt != NONE && side == 0) {
      const u32 i = at_inc_agg(B->n_seeds);
      if (i < B->cap_seeds) { B->seeds[2 * i] = walk; B->seeds[2 * i + 1] = tgt; }
      else at_or(B->overflow, 4);
    }
    return true;
  }
};

}  // namespace exs
