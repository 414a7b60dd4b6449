// exs_stage_sema.cuh -- driver for K5: declaration records, the GPU hash-table
// symbol join (structs, overload sets, signature duplicates) and the
// unit-level checks of resolve() (reference: sema.py:152-320).
#pragma once
#include "exs_stage_parse.cuh"
#include "exs_sema.cuh"

namespace exs {

struct SemaState {
  u32 NF = 0, NR = 0, NC = 0;
  FnRec* fns = nullptr;
  RecRec* recs = nullptr;
  u32* item_fn = nullptr;   // FI+1 exclusive scan of fn counts per item
  u32* item_rec = nullptr;
  MapEnt* smap = nullptr; u32 smap_mask = 0;
  MapEnt* fmap = nullptr; u32 fmap_mask = 0;
  MapEnt* sigm = nullptr; u32 sig_mask = 0;    // resolve duplicates
  MapEnt* sigam = nullptr; u32 siga_mask = 0;  // walk-visible sig reps
  u32* fcand = nullptr, *fcand_cnt = nullptr;
  u32 NS = 0;                                  // top-level statements of all bodies
  u64 NCS = 0;                                 // call sites of all bodies
  u32* stmt_node = nullptr, *stmt_cs = nullptr;  // per statement: node, call sites before it
  Tables tab;
  void free_all() {
    void* ps[] = {fns, recs, item_fn, item_rec, smap, fmap, sigm, sigam, fcand, fcand_cnt, stmt_node,
                  stmt_cs};
    for (void* p : ps) dfree(p);
  }
};

// ---------------------------------------------------------------------------
// an empty map of mask + 1 entries (keys 0, values NONE)
inline MapEnt* alloc_map(u32 mask, cudaStream_t st) {
  MapEnt* e = dalloc<MapEnt>((u64)mask + 1);
  par_for((i64)mask + 1, [=] EXS_HD (i64 h) { MapEnt x; x.k = 0; x.v = NONE; x.pad = 0; e[h] = x; }, st);
  return e;
}

// canonical printer as a hash stream (nodes.py:336-383)

struct HashPrinter {
  const Node* nodes;
  const Tok* toks;
  u64 h;
  int depth;
  EXS_HD void s(const char* t) { while (*t) h = fnv_step(h, (u8)*t++); }
  EXS_HD void c(u8 ch) { h = fnv_step(h, ch); }
  // a name or string token: its NameHash stands for its text (one load, not
  // a byte loop over the source with the splice bitmap)
  EXS_HD void tok_text(u32 t) {
    const u64 v = toks[t].hv;
    h = nh_mix(nh_mix(h, (u32)v), (u32)(v >> 32));
  }
  EXS_HD void u64dec(u64 v) {
    char b[24]; int n = 0;
    do { b[n++] = (char)('0' + v % 10); v /= 10; } while (v);
    while (n) c((u8)b[--n]);
  }
  EXS_HD void targs(u32 l) {
    if (l == NONE) return;
    s("< ");
    bool first = true;
    for (; l != NONE; l = nodes[l].next) {
      if (!first) s(", ");
      first = false;
      if (nodes[l].kind == N_TYPE) type(l); else expr(l);
    }
    s(" >");
  }
  EXS_HD void type(u32 t) {
    tok_text(nodes[t].tok);
    targs(nodes[t].c0);
  }
  EXS_HD void args(u32 l) {
    bool first = true;
    for (; l != NONE; l = nodes[l].next) {
      if (!first) s(", ");
      first = false;
      expr(l);
    }
  }
  EXS_HD void expr(u32 e) {
    if (++depth > 400) { depth--; return; }
    const Node& n = nodes[e];
    switch (n.kind) {
      case N_INT: u64dec(toks[n.tok].hv); break;
      case N_STR: c('"'); tok_text(n.tok); c('"'); break;
      case N_BOOL: s(n.sub ? "true" : "false"); break;
      case N_HDCV: s(n.sub == 1 ? "HDC::Hst" : (n.sub == 2 ? "HDC::Dev" : "HDC::HstDev")); break;
      case N_ARCH: s("cuda_arch"); break;
      case N_NAME: tok_text(n.tok); break;
      case N_TMP: type(n.c0); s("{}"); break;
      case N_TRAIT: s("hdc< "); type(n.c0); s(" >"); break;
      case N_MCONST: type(n.c0); s("::"); tok_text(n.tok); break;
      case N_CALL:
        if (n.sub == CALL_STD) { s("std::"); tok_text(n.c0); }
        else { tok_text(n.tok); targs(n.c1); }
        c('('); args(n.c2); c(')');
        break;
      case N_MCALL: expr(n.c0); c('.'); tok_text(n.tok); targs(n.c1); c('('); args(n.c2); c(')'); break;
      case N_SCALL: type(n.c0); s("::"); tok_text(n.tok); targs(n.c1); c('('); args(n.c2); c(')'); break;
      case N_NOT: c('!'); expr(n.c0); break;
      case N_BIN:
        c('('); expr(n.c0);
        s(n.sub == OP_OR ? " || " : (n.sub == OP_AND ? " && " : (n.sub == OP_EQ ? " == " : " != ")));
        expr(n.c1); c(')');
        break;
      default: break;
    }
    depth--;
  }
};

// signature_key hash (sema.py:144-149) with the spaces string under P2 (133-141)
EXS_HD inline u64 sig_hash(const Node* nodes, const Tok* toks, u32 fn_node, u32 owner_name_tok, bool p2) {
  HashPrinter hp{nodes, toks, fnv_init(), 0};
  const Node& f = nodes[fn_node];
  const Node& x = nodes[fn_node + 1];
  if (owner_name_tok != NONE) hp.tok_text(owner_name_tok);
  hp.c(0x1f);
  hp.tok_text(f.tok);
  hp.c(0x1f);
  for (u32 p = f.c1; p != NONE; p = nodes[p].next) { hp.type(nodes[p].c0); hp.c(0x1e); }
  hp.c(0x1f);
  if (x.c0 != NONE) hp.expr(x.c0);
  hp.c(0x1f);
  if (p2) {
    if (f.n & FF_H) { hp.c('H'); if (x.c1 != NONE) { hp.c('('); hp.expr(x.c1); hp.c(')'); } }
    if (f.n & FF_D) { hp.c('D'); if (x.c2 != NONE) { hp.c('('); hp.expr(x.c2); hp.c(')'); } }
    if (f.n & FF_G) hp.c('G');
  }
  return nz(hp.h);
}

// call sites + E0101 checks over one body (sema.py:251-320)
struct BodyScan {
  const Node* nodes;
  const Tok* toks;
  const Tables* T;
  u32 view;
  bool plain;
  u32 ncalls;
  // emit
  const WalkBufs* B;
  u32 file;
  int depth;
  EXS_HD void expr(u32 e) {
    if (++depth > 400) { depth--; return; }
    const Node& n = nodes[e];
    switch (n.kind) {
      case N_CALL: {
        ncalls++;
        bool known;
        if (n.sub == CALL_STD) {
          known = toks[n.c0].id == W_ABORT;  // std::abort is the only std builtin
        } else {
          known = T->fmap.find(vkey(view, toks[n.tok].hv)) != NONE;
          if (!known) {
            u8 w = toks[n.tok].id;
            known = w == W_PRINTF || w == W_RELEASE_ASSERT || w == W_ABORT ||
                    ((w == W_TRAP || w == W_CUDASYNC) && !plain);
          }
        }
        if (!known && B) {
          const Tok& k = toks[n.tok];
          u64 a1 = n.sub == CALL_STD ? (((u64)toks[n.c0].pos << 32) | (toks[n.c0].end - toks[n.c0].pos)) : 0;
          emit_diag(*B, mkdiag(file, k.line, k.col, C_E0101, M_S_UNDEF_NAME,
                               ((u64)k.pos << 32) | (k.end - k.pos), a1, 0, n.sub == CALL_STD));
        }
        for (u32 a = n.c2; a != NONE; a = nodes[a].next) expr(a);
        break;
      }
      case N_SCALL:
        ncalls++;
        for (u32 a = n.c2; a != NONE; a = nodes[a].next) expr(a);
        break;
      case N_MCALL:
        ncalls++;
        expr(n.c0);
        for (u32 a = n.c2; a != NONE; a = nodes[a].next) expr(a);
        break;
      case N_NOT: expr(n.c0); break;
      case N_BIN: expr(n.c0); expr(n.c1); break;
      default: break;
    }
    depth--;
  }
  EXS_HD void stmts(u32 s) {
    for (; s != NONE; s = nodes[s].next) one(s);
  }
  EXS_HD void one(u32 s) {
    {
      const Node& n = nodes[s];
      switch (n.kind) {
        case N_SEXPR: expr(n.c0); break;
        case N_SRET: if (n.c0 != NONE) expr(n.c0); break;
        case N_SIF: expr(n.c0); stmts(n.c1); if (n.sub) stmts(n.c2); break;
        case N_SFOR: expr(n.c0); expr(n.c1); stmts(n.c2); break;
        case N_SLAUNCH: {
          expr(n.c1);
          expr(nodes[n.c1].next);
          for (u32 a = n.c2; a != NONE; a = nodes[a].next) expr(a);
          ncalls++;
          if (B && T->fmap.find(vkey(view, toks[n.tok].hv)) == NONE) {
            const Tok& k = toks[n.tok];
            emit_diag(*B, mkdiag(file, k.line, k.col, C_E0101, M_S_UNDEF_NAME,
                                 ((u64)k.pos << 32) | (k.end - k.pos)));
          }
          break;
        }
        default: break;
      }
    }
  }
};

inline u32 pow2_at_least(u64 n) {
  u32 c = 1024;
  while (c < n) c <<= 1;
  return c;
}

inline void run_sema(LexState& L, ParseState& P, SemaState& S, const WalkBufs& WB, Scratch& sc,
                     cudaStream_t st) {
  const u32 FI = P.FI, V = P.V;
  // 1. declaration records in _all_decls order (spacecheck.py:264-270)
  u32* cf = dalloc<u32>(FI + 1);
  u32* cr = dalloc<u32>(FI + 1);
  {
    const Node* nd = P.nodes; const u32* fit = P.fitems;
    par_for(FI + 1, [=] EXS_HD (i64 i) {
      if (i == FI) { cf[i] = cr[i] = 0; return; }
      const Node& n = nd[fit[i]];
      u32 nf = 0, nr = 0;
      if (n.kind == N_FN) nf = 1;
      else if (n.kind == N_STRUCT) {
        nr = 1;
        for (u32 m = n.c1; m != NONE; m = nd[m].next) if (nd[m].kind == N_FN) nf++;
      }
      cf[i] = nf; cr[i] = nr;
    }, st);
  }
  S.item_fn = dalloc<u32>(FI + 1);
  S.item_rec = dalloc<u32>(FI + 1);
  excl_scan_u32(cf, S.item_fn, FI + 1, sc, st);
  excl_scan_u32(cr, S.item_rec, FI + 1, sc, st);
  S.NF = get1(S.item_fn + FI, st);
  S.NR = get1(S.item_rec + FI, st);
  dfree(cf);
  dfree(cr);
  const u32 NF = S.NF, NR = S.NR;
  S.fns = dalloc<FnRec>(NF + 1);
  S.recs = dalloc<RecRec>(NR + 1);
  {
    Node* nd = P.nodes; const u32* fit = P.fitems; const u32* fiv = P.fitem_view;
    const u32* ifn = S.item_fn; const u32* irc = S.item_rec; FnRec* fr = S.fns; RecRec* rr = S.recs;
    const Tok* tk = L.toks;
    EXS_TAG("sema_decl_records");
    par_for(FI, [=] EXS_HD (i64 i) {
      Node& n = nd[fit[i]];
      u32 v = fiv[i];
      u32 f = ifn[i];
      auto put = [&](u32 node, u32 rec) {
        FnRec& r = fr[f];
        r.node = node; r.view = v; r.rec = rec; r.order = f;
        r.name = nd[node].hv; r.sig = 0; r.sig_rep = f; r.ncalls = 0;
        r.nstmts = (nd[node].n & FF_BODY) ? (u32)(nd[node + 1].hv & 0xFFFFFFFFu) : 0;  // counted by the parser
        r.flags = rec == NONE ? 0 : FR_MEMBER;
        if ((nd[node].n & FF_BODY) && (r.nstmts || nd[node].c1 != NONE)) r.flags |= FR_BODY;
        nd[node + 1].tok = f;  // FNX.tok -> decl record
        f++;
      };
      if (n.kind == N_FN) put(fit[i], NONE);
      else if (n.kind == N_STRUCT) {
        u32 r = irc[i];
        RecRec& q = rr[r];
        q.node = fit[i]; q.view = v; q.order = r; q.dup = 0; q.name = n.hv;
        n.c2 = r;
        for (u32 m = n.c1; m != NONE; m = nd[m].next) if (nd[m].kind == N_FN) put(m, r);
      }
    }, st);
  }
  // 2. struct table: first definition wins (sema.py:176-184)
  S.smap_mask = pow2_at_least(2ull * NR + 2) - 1;
  S.smap = alloc_map(S.smap_mask, st);
  {
    MapEnt* me = S.smap; u32 mask = S.smap_mask; RecRec* rr = S.recs;
    par_for(NR, [=] EXS_D (i64 r) { map_insert_min(me, mask, vkey(rr[r].view, rr[r].name), (u32)r); }, st);
    Map m{me, mask};
    const Node* nd = P.nodes; const Tok* tk = L.toks; const u32* vf = P.vfile; WalkBufs B = WB;
    par_for(NR, [=] EXS_HD (i64 r) {
      RecRec& q = rr[r];
      q.dup = m.find(vkey(q.view, q.name)) != (u32)r;
      if (q.dup) {
        const Tok& t = tk[nd[q.node].tok];
        emit_diag(B, mkdiag(vf[q.view], t.line, t.col, C_E0102, M_S_DUP, ((u64)t.pos << 32) | (t.end - t.pos)));
      }
    }, st);
  }
  // 3. owner flags, signature hashes
  {
    FnRec* fr = S.fns; const RecRec* rr = S.recs; const Node* nd = P.nodes; const Tok* tk = L.toks;
    const u32* vf = P.vfile; const u8* cfgs = L.cfg;
    EXS_TAG("sema_sig_hash");
    par_for(NF, [=] EXS_HD (i64 i) {
      FnRec& r = fr[i];
      u32 owner_tok = NONE;
      if (r.rec != NONE && !rr[r.rec].dup) { r.flags |= FR_OWNER; owner_tok = nd[rr[r.rec].node].tok; }
      if (tk[nd[r.node].tok].id == W_MAIN && !(r.flags & FR_OWNER)) r.flags |= FR_MAIN;
      bool p2 = (cfgs[vf[r.view]] & CFG_MODE_MASK) == MODE_P2;
      r.sig = sig_hash(nd, tk, r.node, owner_tok, p2);
    }, st);
  }
  // 4. duplicates among free functions and members of kept structs (sema.py:161-195)
  S.sig_mask = pow2_at_least(2ull * NF + 2) - 1;
  S.sigm = alloc_map(S.sig_mask, st);
  S.siga_mask = S.sig_mask;
  S.sigam = alloc_map(S.sig_mask, st);
  {
    FnRec* fr = S.fns; const RecRec* rr = S.recs;
    MapEnt* me = S.sigm; u32 mask = S.sig_mask;
    par_for(NF, [=] EXS_D (i64 i) {
      const FnRec& r = fr[i];
      if (r.rec != NONE && rr[r.rec].dup) return;  // members of duplicate structs are never checked
      map_insert_min(me, mask, vkey(r.view, r.sig), (u32)i);
    }, st);
    Map m{me, mask};
    const Node* nd = P.nodes; const Tok* tk = L.toks; const u32* vf = P.vfile; WalkBufs B = WB;
    par_for(NF, [=] EXS_HD (i64 i) {
      FnRec& r = fr[i];
      if (r.rec != NONE && rr[r.rec].dup) return;
      if (m.find(vkey(r.view, r.sig)) != (u32)i) {
        r.flags |= FR_DUP;
        const Tok& t = tk[nd[r.node].tok];
        u64 osp = 0;
        if (r.flags & FR_OWNER) { const Tok& o = tk[nd[rr[r.rec].node].tok]; osp = ((u64)o.pos << 32) | (o.end - o.pos); }
        emit_diag(B, mkdiag(vf[r.view], t.line, t.col, C_E0102, M_S_DUP, ((u64)t.pos << 32) | (t.end - t.pos), osp));
      }
    }, st);
    MapEnt* mea = S.sigam;
    par_for(NF, [=] EXS_D (i64 i) {
      const FnRec& r = fr[i];
      if ((r.flags & FR_DUP) && (r.flags & FR_OWNER)) return;  // removed from the struct
      map_insert_min(mea, mask, vkey(r.view, r.sig), (u32)i);
    }, st);
    Map ma{mea, mask};
    const u8* cfgs = L.cfg;
    par_for(NF, [=] EXS_HD (i64 i) {
      FnRec& r = fr[i];
      u32 rep = ma.find(vkey(r.view, r.sig));
      r.sig_rep = rep == NONE ? (u32)i : rep;
      if ((r.flags & FR_DUP) && (r.flags & FR_OWNER)) { r.nstmts = 0; return; }  // not in the struct any more
      const Node& n = nd[r.node];
      if ((n.n & (FF_HPRED | FF_DPRED)) && (cfgs[vf[r.view]] & CFG_MODE_MASK) != MODE_P1) {
        const Tok& t = tk[n.tok];
        emit_diag(B, mkdiag(vf[r.view], t.line, t.col, C_E0001, M_S_COND_SPEC_MODE));
      }
    }, st);
  }
  // 5. overload sets of free functions, in item order
  {
    u32* idx = dalloc<u32>(NF + 1);
    FnRec* fr = S.fns;
    S.NC = select_idx(NF, [=] EXS_HD (u32 i) -> bool { return fr[i].rec == NONE && !(fr[i].flags & FR_DUP); },
                      idx, L.cnt, sc, st);
    const u32 NC = S.NC;
    // group by the (view, name) key's slot in the name map: a stable radix sort
    // of 32-bit slot numbers (as many bits as the table) keeps item order inside
    // a group; the slot's value is then set to its group's start
    S.fmap_mask = pow2_at_least(2ull * NC + 2) - 1;
    S.fmap = alloc_map(S.fmap_mask, st);
    MapEnt* fme = S.fmap; const u32 mask = S.fmap_mask;
    u32* keys = dalloc<u32>(NC + 1);
    par_for(NC, [=] EXS_D (i64 i) { keys[i] = map_insert_slot(fme, mask, vkey(fr[idx[i]].view, fr[idx[i]].name)); }, st);
    int kb = 1;
    while (kb < 32 && (mask >> kb)) kb++;
    sort_pairs(keys, idx, NC, sc, st, kb);
    S.fcand = idx;
    S.fcand_cnt = dalloc<u32>(NC + 1);
    u32* cnt = S.fcand_cnt;
    par_for(NC, [=] EXS_HD (i64 i) {
      if (i > 0 && keys[i - 1] == keys[i]) return;
      u32 j = (u32)i;
      while (j < NC && keys[j] == keys[i]) j++;
      cnt[i] = j - (u32)i;
      fme[keys[i]].v = (u32)i;
    }, st);
    dfree(keys);
  }
  // tables for the evaluator
  S.tab.nodes = P.nodes; S.tab.toks = L.toks; S.tab.fns = S.fns; S.tab.recs = S.recs;
  S.tab.smap = Map{S.smap, S.smap_mask};
  S.tab.fmap = Map{S.fmap, S.fmap_mask};
  S.tab.fcand = S.fcand; S.tab.fcand_cnt = S.fcand_cnt;
  S.tab.src = L.src; S.tab.splice = L.splice;
  // 6. mode-gated syntax (sema.py:221-248), call sites, undefined names
  {
    const Tables tab = S.tab;
    const RecRec* rr = S.recs; const Node* nd = P.nodes; const Tok* tk = L.toks;
    const u32* vf = P.vfile; const u8* cfgs = L.cfg; WalkBufs B = WB;
    par_for(NR, [=] EXS_HD (i64 r) {
      const RecRec& q = rr[r];
      u8 mode = cfgs[vf[q.view]] & CFG_MODE_MASK;
      const Node& n = nd[q.node];
      if (mode != MODE_P2 && (n.n & (SF_H | SF_D | SF_G))) {
        const Tok& t = tk[n.tok];
        emit_diag(B, mkdiag(vf[q.view], t.line, t.col, C_E0001, M_S_STRUCT_SPEC_MODE));
      }
    }, st);
    FnRec* fr = S.fns;
    // bodies are scanned statement-parallel (BodyScan carries no state across
    // top-level statements): count, tabulate, scan each statement once
    // statement counts: set with the decl records (the parser counted them);
    // removed members were zeroed and conditional specifiers outside proposal1
    // reported with the signature representatives (step 4)
    // per-statement tables: statements of a body are walked in parallel (K6)
    u32* ns = dalloc<u32>(NF + 1);
    u32* sb = dalloc<u32>(NF + 1);
    par_for(NF + 1, [=] EXS_HD (i64 i) { ns[i] = i < NF ? fr[i].nstmts : 0; }, st);
    excl_scan_u32(ns, sb, NF + 1, sc, st);
    S.NS = get1(sb + NF, st);
    const u32 NSt = S.NS;
    S.stmt_node = dalloc<u32>(NSt + 1);
    S.stmt_cs = dalloc<u32>(NSt + 1);
    u32* sfn = dalloc<u32>(NSt + 1);
    u32* scnt = dalloc<u32>(NSt + 1);
    u32* cpre = dalloc<u32>(NSt + 1);
    u32* sn = S.stmt_node; u32* scs = S.stmt_cs;
    const u32* sroot = P.seg_root;
    // split bodies of many statements are tabulated by a 256-lane group each
    // (a main of 5,150 statements, C3), the rest by one thread per body
    constexpr u32 HEAVY = 64;
    u32* hn = dalloc<u32>(1);
    u32* hl = dalloc<u32>((u64)NSt / HEAVY + 2);
    dzero(hn, 4, st);
    EXS_TAG("sema_body_table");
    par_for(NF, [=] EXS_HD (i64 i) {
      FnRec& r = fr[i];
      r.stmt_base = sb[i];
      if (!r.nstmts) return;
      u32 k = sb[i];
      bool var = false;
      const u64 x = nd[r.node + 1].hv;
      if (x >> 32) {
        if (r.nstmts > HEAVY) { hl[at_inc_agg(hn)] = (u32)i; return; }
        // a split body: its statements are listed by segment (no list walk)
        const u32* sg = sroot + ((x >> 32) - 1);
        for (u32 t = 0; t < r.nstmts; t++) {
          const u32 s = sg[t];
          sn[k + t] = s;
          sfn[k + t] = (u32)i;
          var |= nd[s].kind == N_SVAR;
        }
      } else {
        for (u32 s = nd[r.node].c2; s != NONE; s = nd[s].next, k++) {
          sn[k] = s;
          sfn[k] = (u32)i;
          var |= nd[s].kind == N_SVAR;
        }
      }
      if (var) r.flags |= FR_VARDECL;
    }, st);
    {
      const i64 G = grid_threads();
      u32* hv = dalloc<u32>((u64)NSt / HEAVY + 2);
      dzero(hv, 4ull * (NSt / HEAVY + 2), st);
      EXS_TAG("sema_body_table_heavy");
      par_for(G, [=] EXS_HD (i64 t) {
        const i64 nh = *hn;
        for (i64 h = t >> 8; h < nh; h += G >> 8) {
          const u32 i = hl[h];
          const FnRec& r = fr[i];
          const u32* sg = sroot + ((nd[r.node + 1].hv >> 32) - 1);
          const u32 k = r.stmt_base;
          for (u32 q = (u32)(t & 255); q < r.nstmts; q += 256) {
            const u32 s = sg[q];
            sn[k + q] = s;
            sfn[k + q] = i;
            if (nd[s].kind == N_SVAR) hv[h] = 1;  // same value from every writer
          }
        }
      }, st);
      par_for(G, [=] EXS_HD (i64 t) {
        const i64 nh = *hn;
        for (i64 h = t; h < nh; h += G)
          if (hv[h]) fr[hl[h]].flags |= FR_VARDECL;
      }, st);
      dfree(hv);
    }
    dfree(hn);
    dfree(hl);
    EXS_TAG("sema_bodyscan");
    par_for_walk(NSt + 1, [=] EXS_HD (i64 k) {
      if (k == NSt) { scnt[k] = 0; return; }
      const FnRec& r = fr[sfn[k]];
      u8 c = cfgs[vf[r.view]];
      BodyScan bs{nd, tk, &tab, r.view, (c & CFG_PLAIN) != 0, 0, &B, vf[r.view], 0};
      bs.one(sn[k]);
      scnt[k] = bs.ncalls;
    }, st);
    excl_scan_u32(scnt, cpre, NSt + 1, sc, st);
    par_for(NSt, [=] EXS_HD (i64 k) { scs[k] = cpre[k] - cpre[fr[sfn[k]].stmt_base]; }, st);
    par_for(NF, [=] EXS_HD (i64 i) {
      FnRec& r = fr[i];
      if (r.nstmts) r.ncalls = cpre[r.stmt_base + r.nstmts] - cpre[r.stmt_base];
    }, st);
    S.NCS = get1(cpre + NSt, st);
    dfree(ns);
    dfree(sb);
    dfree(sfn);
    dfree(scnt);
    dfree(cpre);
  }
  // 7. static assertions (sema.py:200-217)
  {
    const Tables* tabp = nullptr;
    Tables* dt = dalloc<Tables>(1);
    h2d(dt, &S.tab, sizeof(Tables), st);
    tabp = dt;
    const u32* fit = P.fitems; const u32* fiv = P.fitem_view; const Node* nd = P.nodes;
    const u32* vf = P.vfile; const u8* cfgs = L.cfg; WalkBufs B = WB;
    par_for(FI, [=] EXS_HD (i64 i) {
      const Node& n = nd[fit[i]];
      if (n.kind != N_ASSERT) return;
      u32 v = fiv[i];
      Sema S2;
      S2.init(tabp, v, cfgs[vf[v]]);
      Env e; e.clear();
      Val out;
      u8 stt = S2.eval(n.c0, e, false, out);
      const Tok& t = S2.K(n.tok);
      if (S2.contract) { emit_diag(B, mkdiag(vf[v], t.line, t.col, C_X9999, M_X_CONTRACT)); return; }
      if (stt == ST_SUBST) emit_diag(B, mkdiag(vf[v], t.line, t.col, C_E0104, M_S_ASSERT_EVAL));
      else if (stt == ST_SEMA) emit_diag(B, mkdiag(vf[v], S2.err.line, S2.err.col, S2.err.code, S2.err.msg, S2.err.a0, S2.err.a1, S2.err.a2));
      else if (!(out.k == V_BOOL && out.x == 1)) emit_diag(B, mkdiag(vf[v], t.line, t.col, C_E0104, M_S_ASSERT_FAIL));
    }, st);
    dfree(dt);
  }
}

}  // namespace exs
