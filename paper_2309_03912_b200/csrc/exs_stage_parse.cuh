// exs_stage_parse.cuh -- driver for K4: views, token-parallel item
// segmentation, item-parallel parsing, sequential repair of views whose items
// do not chain, final ordered item lists.
#pragma once
#include "exs_stage_lex.cuh"
#include "exs_parse.cuh"

namespace exs {

struct ParseState {
  u32 V = 0, VT = 0, I = 0, FI = 0;
  u32* vbase = nullptr;   // V+1
  u32* vdirect = nullptr; // first token when the view is the file's whole token range
  u32* vfile = nullptr;
  u8* vpass = nullptr;    // passes served (bit0 host, bit1 device)
  u32* veof = nullptr;    // 2V (line, col)
  u32* vtok = nullptr;    // VT
  u32* vview = nullptr;   // VT
  u16* vkid = nullptr;    // VT kind << 8 | id
  u32* item_start = nullptr, *item_view = nullptr, *item_root = nullptr, *item_end = nullptr;
  u8* item_stat = nullptr;
  PErr* item_err = nullptr;
  u32* vfirst = nullptr;  // V+1 first segment item of each view
  u32* vbad = nullptr;    // V
  u8* vstat = nullptr;    // 0 ok, 1 failed, 2 fallback ok
  u32* vfb_base = nullptr, *vfb_cnt = nullptr;
  u32* fb_items = nullptr;
  u32* vfi = nullptr;     // V+1 final item range
  u32* fitems = nullptr;  // FI root nodes
  u32* fitem_view = nullptr;
  Node* nodes = nullptr;
  u64 n_nodes = 0;
  u32* seg_root = nullptr;  // statement node of each split-body segment (FNX.hv >> 32 - 1 indexes it)
  void free_all() {
    void* ps[] = {vbase, vfile, vpass, veof, vtok, vview, item_start, item_view, item_root,
                  item_end, item_stat, item_err, vfirst, vbad, vstat, vfb_base, vfb_cnt,
                  fb_items, vfi, fitems, fitem_view, nodes, vdirect, vkid, seg_root};
    for (void* p : ps) dfree(p);
  }
};

struct MaxU32Op {
  EXS_HD u32 operator()(u32 a, u32 b) const { return a > b ? a : b; }
};

EXS_HD inline u64 node_base(const u32* item_start, u32 j) { return 2ull * item_start[j] + 4ull * j; }

// split_min: items at least this many tokens long have their function body
// parsed statement-parallel (step 4b); exs_set_option(3, n)
inline void run_parse(LexState& L, ParseState& P, const WalkBufs& WB, Scratch& sc, cudaStream_t st,
                      u32 split_min = 16) {
  const u32 F = L.F, T = L.T;
  // 1. files whose passes see different token sets
  // the lexer's emit passes wrote, per token, the file and kind/id arrays of
  // the common one-view-per-file layout (dropped otherwise) and the per-file
  // pass-split flags; split[F] (irregular) is also set below when a pass failed
  u32* split = L.tsplit;
  u32* irr = split + F;  // some token is not live in all its file's passes, or a pass failed
  u32* tview = L.tfile;
  u16* tkid = L.tkid;
  L.tsplit = nullptr; L.tfile = nullptr; L.tkid = nullptr;  // owned here from now on
  // 2. views per file
  u32* fvc = dalloc<u32>(F + 1);
  u32* fvb = dalloc<u32>(F + 1);
  {
    const FP* fp = L.fp; const u8* cf = L.cfg;
    par_for(F + 1, [=] EXS_HD (i64 f) {
      if (f == F) { fvc[f] = 0; return; }
      bool ok[2];
      for (int p = 0; p < 2; p++) ok[p] = fp[2 * f + p].pp_line == NONE && fp[2 * f + p].lex_pos == NONE;
      u32 c;
      if (cf[f] & CFG_PLAIN) c = ok[0];
      else if (ok[0] && ok[1] && !split[f]) c = 1;
      else c = (u32)ok[0] + (u32)ok[1];
      fvc[f] = c;
      if (!ok[0] || (!(cf[f] & CFG_PLAIN) && !ok[1])) at_or(irr, 1u);
    }, st);
  }
  u32 V = 0, VT = 0;
  if (!get1(irr, st)) {
    // every token is live in all its file's passes and no pass failed (the
    // common case): one view per file, view positions are token indices
    V = P.V = F;
    VT = P.VT = T;
    P.vbase = dalloc<u32>(V + 1);
    P.vfile = dalloc<u32>(V + 1);
    P.vpass = dalloc<u8>(V + 1);
    P.veof = dalloc<u32>(2 * (size_t)V + 2);
    P.vdirect = dalloc<u32>(V + 1);
    {
      FP* fp = L.fp; const u8* cf = L.cfg; const u32* ft = L.ftok;
      u32* vb = P.vbase; u32* vf = P.vfile; u8* vp = P.vpass; u32* ve = P.veof; u32* vd = P.vdirect;
      par_for(F + 1, [=] EXS_HD (i64 f) {
        vb[f] = ft[f];
        if (f == F) return;
        const bool plain = (cf[f] & CFG_PLAIN) != 0;
        vf[f] = (u32)f; vp[f] = plain ? 1 : 3; vd[f] = ft[f];
        fp[2 * f].view = (u32)f;
        if (!plain) fp[2 * f + 1].view = (u32)f;
        ve[2 * f] = fp[2 * f].eof_line; ve[2 * f + 1] = fp[2 * f].eof_col;
      }, st);
    }
    P.vtok = dalloc<u32>(VT + 1);
    P.vview = tview;
    P.vkid = tkid;
    {
      u32* vt = P.vtok;
      par_for(T, [=] EXS_HD (i64 t) { vt[t] = (u32)t; }, st);
    }
    dfree(fvc); dfree(fvb); dfree(split);
  } else {
    dfree(tview);
    dfree(tkid);
    prof_mark(st);
    excl_scan_u32(fvc, fvb, F + 1, sc, st);
    P.V = get1(fvb + F, st);
    V = P.V;
    P.vbase = dalloc<u32>(V + 1);
    P.vfile = dalloc<u32>(V + 1);
    P.vpass = dalloc<u8>(V + 1);
    P.veof = dalloc<u32>(2 * (size_t)V + 2);
    P.vdirect = dalloc<u32>(V + 1);
    u32* vcnt = dalloc<u32>(V + 1);
    // token pass flags and their scans
    u32* s0 = dalloc<u32>(T + 1);
    u32* s1 = dalloc<u32>(T + 1);
    {
      u32* f0 = dalloc<u32>(T + 1);
      u32* f1 = dalloc<u32>(T + 1);
      const Tok* tk = L.toks;
      par_for(T + 1, [=] EXS_HD (i64 t) {
        if (t == T) { f0[t] = f1[t] = 0; return; }
        f0[t] = tk[t].mask & 1;
        f1[t] = (tk[t].mask >> 1) & 1;
      }, st);
      prof_mark(st);
      excl_scan_u32(f0, s0, T + 1, sc, st);
      excl_scan_u32(f1, s1, T + 1, sc, st);
      sync(st);
      prof_mark(st);
      dfree(f0);
      dfree(f1);
    }
    {
      FP* fp = L.fp; const u8* cf = L.cfg; const u32* ft = L.ftok;
      u32* vf = P.vfile; u8* vp = P.vpass; u32* ve = P.veof; u32* vd = P.vdirect;
      par_for(F, [=] EXS_HD (i64 f) {
        u32 v = fvb[f];
        u32 c = fvc[f];
        if (!c) return;
        u32 tf0 = ft[f], tf1 = ft[f + 1];
        bool ok0 = fp[2 * f].pp_line == NONE && fp[2 * f].lex_pos == NONE;
        bool ok1 = !(cf[f] & CFG_PLAIN) && fp[2 * f + 1].pp_line == NONE && fp[2 * f + 1].lex_pos == NONE;
        if (c == 1 && ok0 && ok1) {
          vf[v] = (u32)f; vp[v] = 3;
          fp[2 * f].view = v; fp[2 * f + 1].view = v;
          ve[2 * v] = fp[2 * f].eof_line; ve[2 * v + 1] = fp[2 * f].eof_col;
          vcnt[v] = s0[tf1] - s0[tf0];
          vd[v] = vcnt[v] == tf1 - tf0 ? tf0 : NONE;
          return;
        }
        for (u32 p = 0; p < 2; p++) {
          bool okp = p ? ok1 : ok0;
          if (!okp) continue;
          vf[v] = (u32)f; vp[v] = (u8)(1u << p);
          fp[2 * f + p].view = v;
          ve[2 * v] = fp[2 * f + p].eof_line; ve[2 * v + 1] = fp[2 * f + p].eof_col;
          vcnt[v] = p ? (s1[tf1] - s1[tf0]) : (s0[tf1] - s0[tf0]);
          vd[v] = vcnt[v] == tf1 - tf0 ? tf0 : NONE;
          v++;
        }
      }, st);
    }
    h2d(vcnt + V, "\0\0\0\0", 4, st);
    excl_scan_u32(vcnt, P.vbase, V + 1, sc, st);
    P.VT = get1(P.vbase + V, st);
    VT = P.VT;
    P.vtok = dalloc<u32>(VT + 1);
    P.vview = dalloc<u32>(VT + 1);
    P.vkid = dalloc<u16>(VT + 1);
    {
      const Tok* tk = L.toks; const FP* fp = L.fp; const u32* ft = L.ftok;
      const u32* vb = P.vbase; const u8* vp = P.vpass; u32* vt = P.vtok; u32* vv = P.vview;
      u16* vkd = P.vkid;
      par_for(T, [=] EXS_HD (i64 t) {
        u32 f = tk[t].file;
        u8 m = tk[t].mask;
        u32 tf0 = ft[f];
        for (u32 p = 0; p < 2; p++) {
          u32 v = fp[2 * f + p].view;
          if (v == NONE) continue;
          if (p == 1 && vp[v] == 3) continue;
          if (!((m >> p) & 1)) continue;
          u32 i = vb[v] + (p ? (s1[t] - s1[tf0]) : (s0[t] - s0[tf0]));
          vt[i] = (u32)t;
          vv[i] = v;
          vkd[i] = (u16)(((u32)tk[t].kind << 8) | tk[t].id);
        }
      }, st);
    }
    dfree(s0); dfree(s1); dfree(vcnt); dfree(fvc); dfree(fvb); dfree(split);
  }
  // 3. segmentation: depth scan and item starts (depth over ( ) { })
  u32* depth_after = nullptr;
  {
    u32* inc = dalloc<u32>(VT + 1);
    const u32* vv = P.vview; const u32* vb = P.vbase;
    const u16* vk = P.vkid;  // 2-byte kind/id per view position (not the 32-byte token)
    // depth delta of every view position, with the view-head reset flag: the
    // scan's input, computed inside the scan
    auto delta = [=] EXS_HD (u32 i) -> u32 {
      const u16 t = vk[i];
      u32 d = 0;
      if ((t >> 8) == TK_PUNCT) {
        const u8 id = (u8)t;
        if (id == P_LPAREN || id == P_LBRACE) d = 1;
        else if (id == P_RPAREN || id == P_RBRACE) d = 0x7FFFFFFFu;  // -1 mod 2^31
      }
      return d | (vb[vv[i]] == i ? 0x80000000u : 0u);
    };
    prof_mark(st);
    incl_scan_fn<u32>(delta, inc, VT, DepthOp(), sc, st);
    prof_mark(st);
    // item starts: a view's first token, or a token after one that ends an item
    // (a depth-0 ';', or a depth-0 '}' not followed by ';') -- evaluated in the
    // selection's own flag pass, no end-flag array
    P.item_start = dalloc<u32>(VT + 1);
    const u32* dep = inc;
    auto pred = [=] EXS_HD (u32 i) -> bool {
      if (vb[vv[i]] == i) return true;
      const u32 e = i - 1;
      if (vv[e] != vv[i] || depth_of(dep[e]) != 0) return false;
      const u16 t = vk[e];
      if ((t >> 8) != TK_PUNCT) return false;
      if ((u8)t == P_SEMI) return true;
      if ((u8)t != P_RBRACE) return false;
      return !(i < vb[vv[e] + 1] && vk[i] == (u16)((TK_PUNCT << 8) | P_SEMI));
    };
    prof_mark(st);
    P.I = select_idx(VT, pred, P.item_start, L.cnt, sc, st);
    prof_mark(st);
    h2d(P.item_start + P.I, &VT, 4, st);  // sentinel: node_base(is, I) bounds the last view's arena
    sync(st);
    depth_after = inc;  // kept for the statement segmentation of large bodies
  }
  const u32 I = P.I;
  P.item_view = dalloc<u32>(I + 1);
  P.item_root = dalloc<u32>(I + 1);
  P.item_end = dalloc<u32>(I + 1);
  P.item_stat = dalloc<u8>(I + 1);
  P.item_err = dalloc<PErr>(I + 1);
  P.vfirst = dalloc<u32>(V + 1);
  P.vbad = dalloc<u32>(V + 1);
  P.vstat = dalloc<u8>(V + 1);
  P.n_nodes = 2ull * VT + 4ull * I + 64;
  P.nodes = dalloc<Node>(P.n_nodes);
  {
    const u32* is = P.item_start; const u32* vv = P.vview; u32* iv = P.item_view;
    par_for(I, [=] EXS_HD (i64 j) { iv[j] = vv[is[j]]; }, st);
    const u32* ivc = P.item_view; u32* vfst = P.vfirst; u32* vbad = P.vbad;
    par_for(V + 1, [=] EXS_HD (i64 v) {
      u32 lo = 0, hi = I;
      while (lo < hi) { u32 mid = (lo + hi) / 2; if (ivc[mid] < v) lo = mid + 1; else hi = mid; }
      vfst[v] = lo;
      if (v < V) vbad[v] = NONE;
    }, st);
  }
  // 3b. large function bodies: statements are split at depth 1 so that one
  //     giant body (a main calling every module, C2/C3) is not parsed by a
  //     single thread.  Boundaries: ';' at depth 1, or a '}' returning to
  //     depth 1 that is not followed by 'else' (parser.py:397-438).
  const u32 BIG = split_min;
  u32* ibody = dalloc<u32>(I + 1);  // body '{' of a split item (global view position) or NONE
  u32 NSS = 0;
  u32* ss = nullptr;                // statement-segment starts
  u32* titem = nullptr;             // item of every view position (kept through step 4b)
  {
    const u32* vb = P.vbase; const u16* vk = P.vkid;
    const u32* is = P.item_start; const u32* iv = P.item_view; const u32* da = depth_after;
    par_for(I, [=] EXS_HD (i64 j) {
      u32 v = iv[j];
      u32 next = (j + 1 < I && iv[j + 1] == v) ? is[j + 1] : vb[v + 1];
      ibody[j] = NONE;
      if (next - is[j] < BIG) return;
      // last token must be the body's '}' returning to depth 0
      if (!(vk[next - 1] == (u16)((TK_PUNCT << 8) | P_RBRACE) && depth_of(da[next - 1]) == 0)) return;
      for (u32 i = is[j]; i < next; i++) {
        const u16 t = vk[i];
        const u32 dep_before = i == vb[v] ? 0 : depth_of(da[i - 1]);
        if (dep_before != 0) continue;
        const u8 kind = (u8)(t >> 8), id = (u8)t;
        if (kind == TK_IDENT && (id == W_STRUCT || id == W_CLASS || id == W_ENUM || id == W_STATIC_ASSERT)) return;
        if (kind == TK_PUNCT && id == P_LBRACE) { ibody[j] = i; return; }
      }
    }, st);
    ss = dalloc<u32>(VT + 1);
    // the item of every view position: item index scattered at its start,
    // max-scanned (O(1) per token instead of a search for the enclosing item)
    u32* tit0 = dalloc<u32>(VT + 1);
    titem = dalloc<u32>(VT + 1);
    dzero(tit0, 4ull * (VT + 1), st);
    par_for(I, [=] EXS_HD (i64 j) { tit0[is[j]] = (u32)j; }, st);
    incl_scan(tit0, titem, VT, MaxU32Op(), sc, st);
    const u32* ti = titem;
    const u32 Ic = I;
    auto pred = [=] EXS_HD (u32 i) -> bool {
      const u32 lo = ti[i];
      u32 bo = ibody[lo];
      if (bo == NONE || i <= bo) return false;
      u32 v = iv[lo];
      u32 next = (lo + 1 < Ic && iv[lo + 1] == v) ? is[lo + 1] : vb[v + 1];
      if (i >= next - 1) return false;  // the closing '}'
      if (i == bo + 1) return true;
      const u16 pt = vk[i - 1];
      if (depth_of(da[i - 1]) != 1 || (pt >> 8) != TK_PUNCT) return false;
      if ((u8)pt == P_SEMI) return true;
      if ((u8)pt == P_RBRACE) {
        // a block ends a statement unless 'else' or an operator follows (a
        // brace-initialised temporary: D{}.call(), D{} == x, f(D{}, ...))
        const u16 t = vk[i];
        const u8 kind = (u8)(t >> 8), id = (u8)t;
        if (kind == TK_IDENT) return id != W_ELSE;
        if (kind == TK_PUNCT) return id == P_LBRACE || id == P_RBRACE || id == P_LPAREN || id == P_BANG;
        return true;
      }
      return false;
    };
    prof_mark(st);
    NSS = select_idx(VT, pred, ss, L.cnt, sc, st);
    prof_mark(st);
    dfree(tit0);
  }
  dfree(depth_after);
  // 4. item-parallel parse
  {
    const Tok* tk = L.toks; const u32* vt = P.vtok; const u32* vb = P.vbase; const u32* ve = P.veof;
    const u16* vk = P.vkid;
    const u32* vdr = P.vdirect;
    const u32* is = P.item_start; const u32* iv = P.item_view; const u32* vf = P.vfile;
    const u8* cf = L.cfg; const u8* s = L.src; const u32* sp = L.splice;
    Node* nd = P.nodes; u32* ir = P.item_root; u32* ie = P.item_end; u8* ist = P.item_stat;
    PErr* ier = P.item_err; u32* vbad = P.vbad;
    // items in (header length bucket, first token) order: similar items per warp
    u32* iperm = dalloc<u32>(I + 1);
    {
      u32* key = dalloc<u32>(I + 1);
      const u32* ib = ibody;
      par_for(I, [=] EXS_HD (i64 j) {
        u32 v = iv[j];
        u32 next = (j + 1 < I && iv[j + 1] == v) ? is[j + 1] : vb[v + 1];
        u32 len = (ib[j] != NONE ? ib[j] + 1 : next) - is[j];  // tokens this thread parses
        u32 lb = 0;
        while ((1u << lb) < len && lb < 31) lb++;
        key[j] = (lb << 16) | vk[is[j]];
        iperm[j] = (u32)j;
      }, st);
      prof_mark(st);
      sort_pairs(key, iperm, I, sc, st, 24);
      prof_mark(st);
      dfree(key);
    }
    const u32* ipm = iperm;
    EXS_TAG("parse_items");
    par_for_parse(I, [=] EXS_HD (i64 jj) {
      const u32 j = ipm[jj];
      u32 v = iv[j];
      u32 next = (j + 1 < I && iv[j + 1] == v) ? is[j + 1] : vb[v + 1];
      u8 c = cf[vf[v]];
      PView pv{tk, vt, vb[v], vb[v + 1] - vb[v], ve[2 * v], ve[2 * v + 1],
               (u8)((c & CFG_PLAIN) ? ((c & CFG_ERASE) ? 1 : 2) : 0), vk};
      Parser p;
      u64 base = node_base(is, (u32)j);
      // a split item's header owns only the node slots below its body's
      // first statement (step 4b uses the rest)
      u32 bo = ibody[j];
      p.init(pv, nd, (u32)base, bo != NONE ? 2 * (bo + 1 - is[j]) : 2 * (next - is[j]) + 4, is[j] - vb[v]);
      p.v_src = s; p.v_splice = sp;
      if (bo != NONE) { p.defer_open = bo - vb[v]; p.defer_close = next - 1 - vb[v]; }
      u32 root = p.item();
      ir[j] = root;
      ie[j] = vb[v] + p.pos;
      u8 stt = 0;
      if (p.failed) stt = p.overflow ? 2 : 1;
      // a deferred body must have been taken by the item's FN node
      if (!p.failed && bo != NONE && (!p.deferred || root == NONE || nd[root].kind != N_FN)) stt = 2;
      ist[j] = stt;
      ier[j] = p.e;
      if (stt || vb[v] + p.pos != next) at_min(&vbad[v], (u32)j);
    }, st);
    dfree(iperm);
  }
  // 4b. statements of the split bodies, in parallel; merged into item status
  if (NSS) {
    const Tok* tk = L.toks; const u32* vt = P.vtok; const u32* vb = P.vbase; const u32* ve = P.veof;
    const u16* vk = P.vkid;
    const u32* is = P.item_start; const u32* iv = P.item_view; const u32* vf = P.vfile;
    const u8* cf = L.cfg; const u8* s = L.src; const u32* sp = L.splice;
    Node* nd = P.nodes; u8* ist = P.item_stat; PErr* ier = P.item_err; u32* vbad = P.vbad;
    const u32* ssc = ss;
    u32* sroot = dalloc<u32>(NSS + 1);
    u32* sbad = dalloc<u32>(I + 1);
    u8* sstat = dalloc<u8>(NSS + 1);
    PErr* serr = dalloc<PErr>(NSS + 1);
    dfill_ff(sbad, 4ull * (I + 1), st);
    const u32 Ic = I, NSSc = NSS;
    const u32* titm = titem;
    // segments in first-token order: warps parse statements of the same shape
    u32* sperm = dalloc<u32>(NSS + 1);
    {
      u32* key = dalloc<u32>(NSS + 1);
      par_for(NSS, [=] EXS_HD (i64 k) {
        key[k] = vk[ssc[k]];
        sperm[k] = (u32)k;
      }, st);
      sort_pairs(key, sperm, NSS, sc, st, 16);
      sync(st);
      dfree(key);
    }
    const u32* spm = sperm;
    EXS_TAG("parse_body_stmts");
    par_for_parse(NSS, [=] EXS_HD (i64 kk) {
      const u32 k = spm[kk];
      u32 i0 = ssc[k];
      u32 lo = titm[i0];  // the item holding segment start i0
      u32 j = lo, v = iv[j];
      u32 inext = (j + 1 < Ic && iv[j + 1] == v) ? is[j + 1] : vb[v + 1];
      bool last = !(k + 1 < NSSc && ssc[k + 1] < inext);
      u32 stop = last ? inext - 1 : ssc[k + 1];  // next segment, or the body's '}'
      u8 c = cf[vf[v]];
      PView pv{tk, vt, vb[v], vb[v + 1] - vb[v], ve[2 * v], ve[2 * v + 1],
               (u8)((c & CFG_PLAIN) ? ((c & CFG_ERASE) ? 1 : 2) : 0), vk};
      Parser p;
      p.init(pv, nd, (u32)(2ull * i0 + 4ull * j), 2 * (stop - i0), i0 - vb[v]);
      p.v_src = s; p.v_splice = sp;
      p.depth = 1;  // inside the body's block (parser depth limit)
      u32 r = p.stmt_t<1>();
      sroot[k] = r;
      u8 stt = p.failed ? (p.overflow ? 2 : 1) : 0;
      if (!stt && vb[v] + p.pos != stop) stt = 3;  // statements do not chain: sequential repair
      sstat[k] = stt;
      serr[k] = p.e;
      if (stt) at_min(&sbad[j], (u32)k);
    }, st);
    par_for(I, [=] EXS_HD (i64 j) {
      u32 k = sbad[j];
      if (k == NONE || ist[j]) return;  // an error before the body wins
      ist[j] = sstat[k] == 1 ? 1 : 2;
      ier[j] = serr[k];
      at_min(&vbad[iv[j]], (u32)j);
    }, st);
    // link the statements under their FN nodes
    const u32* ir = P.item_root;
    par_for(NSS, [=] EXS_HD (i64 k) {
      u32 i0 = ssc[k];
      u32 lo = titm[i0];  // the item holding segment start i0
      u32 j = lo;
      if (ist[j] || sroot[k] == NONE) return;
      u32 v = iv[j];
      u32 inext = (j + 1 < Ic && iv[j + 1] == v) ? is[j + 1] : vb[v + 1];
      bool first = k == 0 || ssc[k - 1] < is[j];
      bool last = !(k + 1 < NSSc && ssc[k + 1] < inext);
      nd[sroot[k]].next = last ? NONE : sroot[k + 1];
      if (first) {
        nd[ir[j]].c2 = sroot[k];
        u32 lo2 = k, hi2 = NSSc;  // the body's statements: segments [k, first segment >= inext)
        while (lo2 < hi2) { u32 mid = (lo2 + hi2) / 2; if (ssc[mid] < inext) lo2 = mid + 1; else hi2 = mid; }
        // FNX: statement count, and (first segment + 1) << 32: the statement
        // list of this body is seg_root[k, k + count)
        nd[ir[j] + 1].hv = ((u64)(k + 1) << 32) | (lo2 - (u32)k);
      }
    }, st);
    sync(st);
    P.seg_root = sroot;
    dfree(sbad); dfree(sstat); dfree(serr); dfree(sperm);
  }
  dfree(ss);
  dfree(titem);
  dfree(ibody);
  // 5. per view: parse error, ok, or sequential repair
  u32 nfb = 0;
  std::vector<u32> fb_views;
  {
    u8* vs = P.vstat; const u32* vbad = P.vbad; const u8* ist = P.item_stat; const PErr* ier = P.item_err;
    const u32* vf = P.vfile; const u8* vp = P.vpass; FP* fp = L.fp; WalkBufs B = WB;
    u32* fbflag = dalloc<u32>(V + 1);
    par_for(V, [=] EXS_HD (i64 v) {
      u32 j = vbad[v];
      fbflag[v] = 0;
      if (j == NONE) { vs[v] = 0; return; }
      if (ist[j] == 1) {
        vs[v] = 1;
        const PErr& e = ier[j];
        emit_diag(B, mkdiag(vf[v], e.line, e.col, C_E0001, e.msg, e.a0, e.a1));
        for (u32 p = 0; p < 2; p++) if ((vp[v] >> p) & 1) fp[2 * vf[v] + p].perr = 1;
        return;
      }
      vs[v] = 3;  // needs repair
      fbflag[v] = 1;
    }, st);
    u32* fbl = dalloc<u32>(V + 1);
    nfb = select_idx(V, [=] EXS_HD (u32 v) -> bool { return fbflag[v] != 0; }, fbl, L.cnt, sc, st);
    fb_views.resize(nfb);
    if (nfb) d2h(fb_views.data(), fbl, nfb * 4, st);
    sync(st);
    dfree(fbl);
    dfree(fbflag);
  }
  P.vfb_base = dalloc<u32>(V + 1);
  P.vfb_cnt = dalloc<u32>(V + 1);
  dzero(P.vfb_cnt, (V + 1) * 4, st);
  if (nfb) {
    // capacity: items consume >= 5 tokens
    std::vector<u32> vbh(V + 1);
    d2h(vbh.data(), P.vbase, (V + 1) * 4, st);
    sync(st);
    std::vector<u32> fbb(V + 1, 0);
    u32 tot = 0;
    for (u32 v : fb_views) { fbb[v] = tot; tot += (vbh[v + 1] - vbh[v]) / 5 + 2; }
    h2d(P.vfb_base, fbb.data(), (V + 1) * 4, st);
    P.fb_items = dalloc<u32>(tot + 1);
    u32* fbl = dalloc<u32>(nfb);
    h2d(fbl, fb_views.data(), nfb * 4, st);
    const Tok* tk = L.toks; const u32* vt = P.vtok; const u32* vb = P.vbase; const u32* ve = P.veof;
    const u16* vk = P.vkid;
    const u32* vdr = P.vdirect;
    const u32* is = P.item_start; const u32* vfst = P.vfirst; const u32* vf = P.vfile;
    const u8* cf = L.cfg; const u8* s = L.src; const u32* sp = L.splice; Node* nd = P.nodes;
    u32* fbi = P.fb_items; u32* fbase = P.vfb_base; u32* fcnt = P.vfb_cnt; u8* vs = P.vstat;
    const u8* vp = P.vpass; FP* fp = L.fp; WalkBufs B = WB;
    par_for(nfb, [=] EXS_HD (i64 k) {
      u32 v = fbl[k];
      u8 c = cf[vf[v]];
      PView pv{tk, vt, vb[v], vb[v + 1] - vb[v], ve[2 * v], ve[2 * v + 1],
               (u8)((c & CFG_PLAIN) ? ((c & CFG_ERASE) ? 1 : 2) : 0), vk};
      u64 base = node_base(is, vfst[v]);
      u64 lim = node_base(is, vfst[v + 1]);
      Parser p;
      p.init(pv, nd, (u32)base, (u32)(lim - base), 0);
      p.v_src = s; p.v_splice = sp;
      u32 n = 0;
      while (p.pos < pv.n) {
        u32 root = p.item();
        if (p.failed) break;
        fbi[fbase[v] + n++] = root;
      }
      if (p.failed) {
        vs[v] = 1;
        if (p.overflow) {
          emit_diag(B, mkdiag(vf[v], 1, 1, C_X9999, M_X_CONTRACT));
        } else {
          emit_diag(B, mkdiag(vf[v], p.e.line, p.e.col, C_E0001, p.e.msg, p.e.a0, p.e.a1));
        }
        for (u32 q = 0; q < 2; q++) if ((vp[v] >> q) & 1) fp[2 * vf[v] + q].perr = 1;
        return;
      }
      fcnt[v] = n;
      vs[v] = 2;
    }, st);
    dfree(fbl);
  }
  // 6. final ordered item lists
  {
    u32* cnt = dalloc<u32>(V + 1);
    const u8* vs = P.vstat; const u32* vfst = P.vfirst; const u32* fcnt = P.vfb_cnt;
    par_for(V + 1, [=] EXS_HD (i64 v) {
      if (v == V) { cnt[v] = 0; return; }
      cnt[v] = vs[v] == 0 ? vfst[v + 1] - vfst[v] : (vs[v] == 2 ? fcnt[v] : 0);
    }, st);
    P.vfi = dalloc<u32>(V + 1);
    excl_scan_u32(cnt, P.vfi, V + 1, sc, st);
    P.FI = get1(P.vfi + V, st);
    P.fitems = dalloc<u32>(P.FI + 1);
    P.fitem_view = dalloc<u32>(P.FI + 1);
    const u32* vfi = P.vfi; const u32* ir = P.item_root; const u32* fbi = P.fb_items;
    const u32* fbase = P.vfb_base; u32* fit = P.fitems; u32* fiv = P.fitem_view;
    const u32 Vv = V;
    par_for(P.FI, [=] EXS_HD (i64 i) {
      u32 lo = 0, hi = Vv;  // last view with vfi[v] <= i
      while (hi - lo > 1) { u32 mid = (lo + hi) / 2; if (vfi[mid] <= (u32)i) lo = mid; else hi = mid; }
      u32 v = lo, k = (u32)i - vfi[v];
      fit[i] = vs[v] == 0 ? ir[vfst[v] + k] : fbi[fbase[v] + k];
      fiv[i] = v;
    }, st);
    dfree(cnt);
  }
}

}  // namespace exs
