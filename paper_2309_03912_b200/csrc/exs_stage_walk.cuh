// exs_stage_walk.cuh -- driver for K6..K8: root seeding, the level-synchronous
// instantiation fixpoint, reachability, pending-stray verdicts and
// __CUDA_ARCH__ divergence (reference: spacecheck.py:254-767).
#pragma once
#include "exs_stage_sema.cuh"
#include "exs_walk.cuh"

namespace exs {

#ifndef EXS_WALK_SORT
#define EXS_WALK_SORT 1  // order walk work items by statement shape (C2 1 GB: walk 137 -> 76 us/MB)
#endif
#ifndef EXS_WALK_SORT_MIN
#define EXS_WALK_SORT_MIN (1u << 16)  // levels with fewer work items walk unsorted
#endif
#ifndef EXS_KCH
#define EXS_KCH 1  // top-level statements per walk_chunks thread (measured: 1 beats 2 and 4 at 1 GB)
#endif

// walk counters, each on its own 128-byte line (hot atomics must not share one)
enum { CNT_INST = 0, CNT_PEND = 1, CNT_SEEDS = 2, CNT_LOG = 3, CNT_OVF = 4, CNT_MAINS = 5, CNT_N = 6 };
constexpr u32 CNT_STRIDE = 32;

// The collective of one unit walked across GPUs: an
// all-gather of variable-size device buffers, supplied by the host (NCCL
// through torch.distributed on GPUs; gloo in the CPU tests).  recv receives
// every rank's buffer in rank order, sizes[r] bytes from rank r.
typedef int (*CollFn)(void* ctx, const void* send, u64 send_bytes, void* recv, const u64* sizes);
struct Coll {
  int rank = 0, world = 1;
  CollFn fn = nullptr;
  void* ctx = nullptr;
  bool on() const { return world > 1 && fn != nullptr; }
};
// all-gather of this rank's bytes: the concatenation (dalloc'd) and per-rank sizes
inline u8* coll_allgatherv(const Coll& c, const void* send, u64 bytes, std::vector<u64>& sizes, u64& total,
                           cudaStream_t st) {
  sync(st);
  u64* mine = dalloc<u64>(1);
  u64* all = dalloc<u64>(c.world);
  h2d(mine, &bytes, 8, st);
  sync(st);
  std::vector<u64> eight(c.world, 8);
  if (c.fn(c.ctx, mine, 8, all, eight.data())) throw Err("collective (sizes) failed");
  sizes.assign(c.world, 0);
  d2h(sizes.data(), all, 8ull * c.world, st);
  sync(st);
  total = 0;
  for (u64 v : sizes) total += v;
  u8* recv = dalloc<u8>(total + 1);
  if (c.fn(c.ctx, send, bytes, recv, sizes.data())) throw Err("collective failed");
  dfree(mine);
  dfree(all);
  return recv;
}
// OR of a flag word over the ranks
inline u32 coll_or(const Coll& c, u32 v, cudaStream_t st) {
  u32* d = dalloc<u32>(1);
  h2d(d, &v, 4, st);
  std::vector<u64> sz;
  u64 tot;
  u8* r = coll_allgatherv(c, d, 4, sz, tot, st);
  std::vector<u32> h(c.world);
  d2h(h.data(), r, 4ull * c.world, st);
  sync(st);
  dfree(d);
  dfree(r);
  u32 o = 0;
  for (u32 x : h) o |= x;
  return o;
}

struct WalkState {
  u32 cap_inst = 0, n_inst = 0, levels = 0;
  u32 buf_scale = 1;  // multiplier of the creation-log estimate (grows on overflow)
  Coll coll;          // one unit across GPUs: work items split by rank, exchanges per level
  u64 n_edges = 0, edge_cap = 0, callsites = 0;
  Slot* slots = nullptr;
  u32 mask = 0;
  Inst* inst = nullptr;
  u32* edges = nullptr;
  Pending* pend = nullptr;
  u32 cap_pend = 0;
  u32* seeds = nullptr;
  u32 cap_seeds = 0;
  CreateLog* log = nullptr;
  u32 cap_log = 0;
  u32* main_inst = nullptr;
  unsigned long long* main_key = nullptr;
  u32* mains = nullptr;     // ids of the instances of main (few), in creation order
  u32 cap_mains = 0;
  u32* counters = nullptr;  // [n_inst, n_pend, n_seeds, n_log, overflow, n_mains]
  u8* visited = nullptr;
  // per walk statistics
  std::vector<u32> w_inst, w_edges, w_demands;
  u32* ctr(u32 k) const { return counters + k * CNT_STRIDE; }
  std::vector<u32> read_counters(cudaStream_t st) const {
    std::vector<u32> raw(CNT_N * CNT_STRIDE), out(8, 0);
    d2h(raw.data(), counters, 4ull * CNT_N * CNT_STRIDE, st);
    sync(st);
    for (u32 k = 0; k < CNT_N; k++) out[k] = raw[k * CNT_STRIDE];
    return out;
  }
  void free_all() {
    void* ps[] = {slots, inst, edges, pend, seeds, log, main_inst, main_key, mains, counters, visited};
    for (void* p : ps) dfree(p);
    slots = nullptr; inst = nullptr; edges = nullptr; pend = nullptr; seeds = nullptr;
    log = nullptr; main_inst = nullptr; main_key = nullptr; mains = nullptr; counters = nullptr; visited = nullptr;
  }
};

struct WalkCfg {
  const Tables* tab;  // device copy
  const FnRec* fns;
  const RecRec* recs;
  const Node* nodes;
  const Tok* toks;
  const u32* vfile;
  const u8* cfg;      // per file
  const FP* fp;
};

// a root candidate (run_walk roots): decl, walk, owner type, specifier inputs
struct RootCand {
  u32 i, p, file, walk;
  u8 mode, cfg;
  bool fast, free_main;  // fast: no specifier needs evaluation
  u16 sf;                // specifier bits of the owning struct
  Val ot;
};
// what step 2 of the roots needs of a fast candidate, written by step 1 (one
// coalesced record instead of re-reading the decl, node, token and struct)
struct RootStash {
  u64 otx;          // owner type name (ot.x) when rec != NONE
  u32 walk, at;     // walk, declaration token
  u32 rec, otrec;   // owner struct record, canonical owner record (ot.rec)
  u8 sp[2];         // static spaces per side
  u8 iflags, pad;   // IF_BODY / IF_MAIN
  u32 pad2;
};

// build a walker for an existing instance
EXS_HD inline void walker_for(Walker& w, const WalkCfg& C, const WalkBufs& B, u32 id, u64 rank) {
  const Inst& I = B.inst[id];
  const FnRec& fr = C.fns[I.fn];
  u32 file = C.vfile[fr.view];
  u8 c = C.cfg[file];
  w.S.init(C.tab, fr.view, c);
  w.B = &B;
  w.T = C.tab;
  w.file = file;
  w.walk = I.walk;
  w.inst_id = id;
  w.native = (u8)(I.walk & 1);
  w.side = I.side;
  w.spaces = I.spaces;
  w.clevel = B.clevel;
  w.fn = I.fn;
  const Node& fn = C.nodes[fr.node];
  w.pragma = (fn.n & FF_PRAGMA) != 0;
  w.from_hd = I.spaces == 3;
  w.fidelity_host = (c & CFG_MODE_MASK) == MODE_FIDELITY && w.native == 0;
  w.parent_rank = rank;
  w.stmt_k = 0; w.stmt_ord = 0; w.stmt_ord_max = 0; w.stmt_cs_base = 0; w.cs_ord = 0;
  w.silent = false; w.asp = 0; w.nloc = 0; w.wdepth = 0;
  w.ebase = I.ebase;
  w.ecnt = 0;
  w.contract = false;
  w.env.clear();
  if (I.orec != NONE && I.ot.k == V_TYPE) w.S.struct_env(I.orec, I.ot, w.env);
  w.env.nbase = w.env.n;
  w.add_binds(fn, I.tb, I.hb, w.env);
  w.env.nbase = w.env.n;
}

inline WalkBufs make_bufs(WalkState& W, u32* n_diags, Diag* diags, u32 cap_diags, u64* dset,
                          u32 dmask, u32* contract) {
  WalkBufs B;
  B.slots = W.slots; B.mask = W.mask; B.inst = W.inst;
  B.n_inst = W.ctr(CNT_INST); B.cap_inst = W.cap_inst; B.lvl_base = 0; B.clevel = 0;
  B.edges = W.edges;
  B.pend = W.pend; B.n_pend = W.ctr(CNT_PEND); B.cap_pend = W.cap_pend;
  B.seeds = W.seeds; B.n_seeds = W.ctr(CNT_SEEDS); B.cap_seeds = W.cap_seeds;
  B.log = W.log; B.n_log = W.ctr(CNT_LOG); B.cap_log = W.cap_log;
  B.main_inst = W.main_inst; B.main_key = W.main_key;
  B.mains = W.mains; B.n_mains = W.ctr(CNT_MAINS); B.cap_mains = W.cap_mains;
  B.diags = diags; B.n_diags = n_diags; B.cap_diags = cap_diags; B.dset = dset; B.dmask = dmask;
  B.overflow = W.ctr(CNT_OVF);
  B.contract = contract;
  return B;
}

template <class T>
void grow(T*& p, u64& cap_or_dummy, u64 need, u64 used, cudaStream_t st) {
  if (need <= cap_or_dummy) return;
  u64 nc = need + need / 2 + 1024;
  T* q = dalloc<T>(nc);
  if (p && used) d2d(q, p, used * sizeof(T), st);
  dfree(p);
  p = q;
  cap_or_dummy = nc;
}

// Grow the instance store to hold `need` ids and rehash the keys of the n
// existing instances (between levels only: no creator is running).  A level
// creates at most two instances per call site (spacecheck.py:591-596) and
// usually at most one; growing before each level replaces the overflow-and-
// rerun of the whole walk.
// an empty instance hash table (mask + 1 slots)
inline Slot* alloc_slots(u32 mask, cudaStream_t st) {
  Slot* sl = dalloc<Slot>((u64)mask + 1);
  par_for((i64)mask + 1, [=] EXS_HD (i64 h) {
    Slot e;
    e.k.a = 0; e.k.b = 0; e.sid = NONE; e.pad = 0; e.sck = ~0ull;
    sl[h] = e;
  }, st);
  return sl;
}

inline void grow_inst(WalkState& W, u64 need, u32 n, cudaStream_t st) {
  if (need <= W.cap_inst) return;
  const u32 cap = (u32)std::min<u64>(std::max<u64>(need + need / 2, 2ull * W.cap_inst), 0x7FFFFFFFull);
  Inst* in = dalloc<Inst>(cap);
  if (n) d2d(in, W.inst, sizeof(Inst) * (u64)n, st);
  const u32 mask = (u32)(pow2_at_least(2ull * cap) - 1);
  Slot* slots = alloc_slots(mask, st);
  par_for(n, [=] EXS_HD (i64 i) {
    Inst& I = in[i];
    IKey k; k.a = I.ka; k.b = I.kb;
    u32 h = (u32)mix64(k.a ^ mix64(k.b)) & mask;
    IKey old;
    while (!ikey_cas(&slots[h].k, k, old)) h = (h + 1) & mask;
    slots[h].sid = (u32)i;
    I.slot = h;
  }, st);
  sync(st);
  dfree(W.inst); dfree(W.slots);
  W.inst = in; W.slots = slots;
  W.cap_inst = cap; W.mask = mask;
}

// a reference to an instance across ranks: (walk, creation key) -- creation
// keys are unique within a walk -- plus a position (edge slot) or the seed's walk
struct XRef {
  unsigned long long key;
  u32 walk, a;
};

// One level's exchange of a sharded walk: every rank's new instance records
// (the ones its work items created, [prev_n, n_now) here) are merged into
// every rank's table -- a key seen for the first time is inserted, and the
// minimum creation key over all creators wins, with its location and decl
// (spacecheck.py:331-337) -- so every rank continues with the same instance
// set and the same frontier order.  Ids stay rank-local: references across
// ranks go by creation key, which is unique per instance.  Returns the OR of
// the ranks' overflow flags; n_now becomes the merged instance count.
inline u32 merge_level(WalkState& W, u32 prev_n, u32& n_now, bool ovf_local, cudaStream_t st) {
  const Coll& c = W.coll;
  const u64 nrec = ovf_local ? 0 : (u64)(n_now - prev_n);
  const u64 bytes = 8 + nrec * sizeof(Inst);
  u8* send = dalloc<u8>(bytes);
  const u64 hdr = ovf_local ? 1 : 0;
  h2d(send, &hdr, 8, st);
  if (nrec) d2d(send + 8, W.inst + prev_n, nrec * sizeof(Inst), st);
  std::vector<u64> sizes;
  u64 total = 0;
  u8* recv = coll_allgatherv(c, send, bytes, sizes, total, st);
  dfree(send);
  std::vector<u64> offs(c.world, 0);
  u32 any = 0;
  u64 incoming = 0;
  for (int r = 0; r < c.world; r++) {
    offs[r] = r ? offs[r - 1] + sizes[r - 1] : 0;
    u64 h = 0;
    d2h(&h, recv + offs[r], 8, st);
    sync(st);
    any |= (u32)h;
    if (r != c.rank) incoming += (sizes[r] - 8) / sizeof(Inst);
  }
  if (any) { dfree(recv); return 1; }
  grow_inst(W, (u64)n_now + incoming + 1024, n_now, st);  // ids and slots for the incoming records
  WalkBufs B{};
  B.slots = W.slots; B.mask = W.mask; B.inst = W.inst; B.n_inst = W.ctr(CNT_INST); B.cap_inst = W.cap_inst;
  B.overflow = W.ctr(CNT_OVF);
  {
    // this rank's level minimum back into the slots (a rehash dropped it)
    Inst* in = W.inst; Slot* sl = W.slots; const u32 base = prev_n;
    par_for(n_now - prev_n, [=] EXS_HD (i64 j) { const Inst& I = in[base + j]; sl[I.slot].sck = I.ckey; }, st);
  }
  for (int r = 0; r < c.world; r++) {
    if (r == c.rank) continue;
    const u64 cnt = (sizes[r] - 8) / sizeof(Inst);
    const Inst* rr = reinterpret_cast<const Inst*>(recv + offs[r] + 8);
    // insert or find, and keep the minimum creation key per slot
    par_for(cnt, [=] EXS_HD (i64 k) {
      const Inst R = rr[k];
      IKey key;
      key.a = R.ka; key.b = R.kb;
      bool ins;
      u32 slot;
      const u32 id = inst_lookup_or_insert(B, key, ins, slot);
      if (id == NONE) return;
      if (ins) {
        Inst I = R;
        I.slot = slot; I.ebase = 0; I.ecnt = 0;
        B.inst[id] = I;
        inst_publish(B, slot, id);
      }
      at_min64(&B.slots[slot].sck, R.ckey);
    }, st);
  }
  for (int r = 0; r < c.world; r++) {
    if (r == c.rank) continue;
    const u64 cnt = (sizes[r] - 8) / sizeof(Inst);
    const Inst* rr = reinterpret_cast<const Inst*>(recv + offs[r] + 8);
    // the winning creator's data (one record per minimum)
    par_for(cnt, [=] EXS_HD (i64 k) {
      const Inst& R = rr[k];
      IKey key;
      key.a = R.ka; key.b = R.kb;
      bool ins;
      const u32 slot = slot_insert(B, key, ins);
      if (slot == NONE || B.slots[slot].sck != R.ckey) return;
      Inst& I = B.inst[B.slots[slot].sid];
      I.ckey = R.ckey; I.at = R.at; I.fn = R.fn;
    }, st);
  }
  sync(st);
  dfree(recv);
  n_now = get1(W.ctr(CNT_INST), st);
  return get1(W.ctr(CNT_OVF), st) ? 1u : 0u;
}

// returns false if a buffer overflowed (caller grows and retries)
inline bool run_walk(LexState& L, ParseState& P, SemaState& S, WalkState& W, WalkBufs& B0,
                     Scratch& sc, cudaStream_t st, u32 diag_cap) {
  const u32 F = L.F, NF = S.NF;
  const u32 NW = 2 * F;
  Tables* dtab = dalloc<Tables>(1);
  h2d(dtab, &S.tab, sizeof(Tables), st);
  WalkCfg C{dtab, S.fns, S.recs, P.nodes, L.toks, P.vfile, L.cfg, L.fp};
  // buffers
  W.mask = pow2_at_least(2ull * W.cap_inst) - 1;
  W.slots = alloc_slots(W.mask, st);
  W.inst = dalloc<Inst>(W.cap_inst);
  W.counters = dalloc<u32>(CNT_N * CNT_STRIDE);
  dzero(W.counters, 4ull * CNT_N * CNT_STRIDE, st);
  W.main_inst = dalloc<u32>(NW + 1);
  W.main_key = dalloc<unsigned long long>(NW + 1);
  dfill_ff(W.main_inst, 4ull * (NW + 1), st);
  dzero(W.main_key, 8ull * (NW + 1), st);
  W.cap_mains = 4 * NW + 1024;
  W.mains = dalloc<u32>(W.cap_mains);
  u64 edge_cap = 0, pend_cap = 0, seed_cap = 0, log_cap = 0;
  W.edges = nullptr; W.pend = nullptr; W.seeds = nullptr; W.log = nullptr;
  // roots log only their non-inserting creators (duplicate decls): few
  grow(W.log, log_cap, std::min<u64>(4ull * NF, ((u64)NF / 8 + 65536) * W.buf_scale) + 64, 0, st);
  grow(W.pend, pend_cap, 1024, 0, st);
  grow(W.seeds, seed_cap, 2048, 0, st);
  grow(W.edges, edge_cap, 1024, 0, st);
  auto bufs = [&]() {
    W.cap_log = (u32)log_cap; W.cap_pend = (u32)pend_cap; W.cap_seeds = (u32)(seed_cap / 2);
    WalkBufs B = make_bufs(W, B0.n_diags, B0.diags, diag_cap, B0.dset, B0.dmask, B0.contract);
    return B;
  };
  WalkBufs B = bufs();
  prof_mark(st);
  // ---- roots (spacecheck.py:272-308)
  bool roots_keyed = false;  // every root's creation key already in its record (no step 3)
  {
    const FnRec* fr = S.fns; const RecRec* rr = S.recs; const Node* nd = P.nodes; const Tok* tk = L.toks;
    const FP* fp = L.fp; const u32* vf = P.vfile; const u8* cfgs = L.cfg;
    const Tables* tab = dtab;
    // root candidates (spacecheck.py:272-283 filters), compacted and ordered by
    // declaration shape so warps evaluate the same specifier paths
    auto is_root = [=] EXS_HD (u32 x) -> bool {
      u32 i = x >> 1, p = x & 1;
      const FnRec& r = fr[i];
      u32 file = vf[r.view];
      u32 walk = 2 * file + p;
      if (fp[walk].view != r.view || fp[walk].perr) return false;
      if ((r.flags & FR_DUP) && (r.flags & FR_OWNER)) return false;
      const Node& fn = nd[r.node];
      if (fn.c0 != NONE || !(fn.n & FF_BODY)) return false;
      if (r.rec != NONE && nd[rr[r.rec].node].c0 != NONE) return false;
      u8 mode = cfgs[file] & CFG_MODE_MASK;
      if (mode == MODE_P2) {
        bool undec = !(fn.n & (FF_H | FF_D | FF_G));
        return (tk[fn.tok].id == W_MAIN && r.rec == NONE) || !undec ||
               (r.rec != NONE && (nd[rr[r.rec].node].n & (SF_H | SF_D | SF_G)));
      }
      return true;
    };
    u32* rcand = dalloc<u32>(2ull * NF + 1);
    const u32 NRC = select_idx(2ull * NF, is_root, rcand, L.cnt, sc, st);
    // root ranks (make_ckey) are batch decl indices while they fit the rank
    // field, else decl indices relative to the view's first decl
    u32* vd0 = nullptr;
    if (NF > CK_FIELD_MAX) {
      const u32 NV = P.V;
      vd0 = dalloc<u32>((u64)NV + 1);
      dfill_ff(vd0, 4ull * (NV + 1), st);
      u32* v0 = vd0;
      par_for(NF, [=] EXS_HD (i64 i) { at_min(&v0[fr[i].view], (u32)i); }, st);
    }
    if (NRC) {
      u32* key = dalloc<u32>(NRC);
      const u32* rcc = rcand;
      par_for(NRC, [=] EXS_HD (i64 k) {
        const FnRec& r = fr[rcc[k] >> 1];
        const Node& fn = nd[r.node];
        key[k] = (u32)(fn.n & (FF_H | FF_D | FF_G | FF_HPRED | FF_DPRED | FF_CX)) |
                 ((u32)(r.rec != NONE) << 16) | ((u32)(cfgs[vf[r.view]] & CFG_MODE_MASK) << 17);
      }, st);
      sort_pairs(key, rcand, NRC, sc, st, 20);
      sync(st);
      dfree(key);
    }
    const u32* rcc = rcand;
    // a root candidate: its decl, walk, owner type and (when no specifier
    // needs evaluation) its sides
    // rot: the canonical owner record per candidate, found once (step 1)
    u32* rot = dalloc<u32>((u64)NRC + 1);
    const u32* rotc = rot;
    auto cand = [=] EXS_HD (u32 x, u32 kk, bool find_owner) -> RootCand {
      RootCand q;
      q.i = x >> 1; q.p = x & 1;
      const FnRec& r = fr[q.i];
      q.file = vf[r.view];
      q.walk = 2 * q.file + q.p;
      const Node& fn = nd[r.node];
      q.cfg = cfgs[q.file];
      q.mode = q.cfg & CFG_MODE_MASK;
      q.ot = vnone();
      if (r.rec != NONE) {
        q.ot.k = V_TYPE; q.ot.x = rr[r.rec].name;
        q.ot.rec = find_owner ? tab->smap.find(vkey(r.view, rr[r.rec].name)) : rotc[kk];
        q.ot.bt = BT_NONE; q.ot.targ = 0;
      }
      q.fast = !(q.mode == MODE_P1 && (fn.n & (FF_HPRED | FF_DPRED)));
      q.free_main = tk[fn.tok].id == W_MAIN && r.rec == NONE;
      q.sf = r.rec != NONE ? nd[rr[r.rec].node].n : 0;
      return q;
    };
    // 1. candidates whose specifiers need no evaluation: insert the keys, keep
    // the minimum creation key (decl order x side order, spacecheck.py:272-283)
    // and log lowering non-inserters by SLOT; ids come from a scan (no shared
    // counter: at this rate one counter serialises the kernel)
    u32* rslot = dalloc<u32>(2ull * NRC + 1);
    RootStash* rstash = dalloc<RootStash>((u64)NRC + 1);
    u32* nslow = dalloc<u32>(2);  // [0] candidates left to step 3, [1] step 2's id count
    dzero(nslow, 8, st);
    const u32 nlog0 = get1(B.n_log, st);
    {
      u32* rs = rslot;
      RootStash* rst = rstash;
      EXS_TAG("walk_roots");
      u32* ro = rot;
      par_for_walk(NRC, [=] EXS_HD (i64 kk) {
        rs[2 * kk] = rs[2 * kk + 1] = NONE;
        const RootCand q = cand(rcc[kk], (u32)kk, true);
        ro[kk] = q.ot.rec;
        if (!q.fast) { rs[2 * kk] = NONE - 1; at_inc_agg(nslow); return; }  // evaluated in step 3
        const FnRec& r = fr[q.i];
        const u16 fl = nd[r.node].n;
        const u8 sides = (fl & FF_G) ? 2 : (static_spaces(fl, q.free_main, q.sf, q.mode, 0) & 3);
        {
          RootStash z;
          z.otx = q.ot.x; z.walk = q.walk; z.at = nd[r.node].tok; z.rec = r.rec; z.otrec = q.ot.rec;
          z.sp[0] = static_spaces(fl, q.free_main, q.sf, q.mode, 0);
          z.sp[1] = static_spaces(fl, q.free_main, q.sf, q.mode, 1);
          z.iflags = (u8)(((r.flags & FR_BODY) ? IF_BODY : 0) | ((r.flags & FR_MAIN) ? IF_MAIN : 0));
          z.pad = 0; z.pad2 = 0;
          rst[kk] = z;
        }
        u32 k = 0;
        for (u8 sd = 0; sd < 2; sd++) {
          if (!((sides >> sd) & 1)) continue;
          const u32 rank = vd0 ? q.i - vd0[r.view] : q.i;  // decl order within the view
          if (rank > CK_FIELD_MAX) { at_or(&B.contract[q.file], 1); return; }
          const unsigned long long ck = make_ckey(0, rank, k++);
          const IKey key = make_ikey(r.sig_rep, vnone(), vnone(), q.ot, q.walk, sd);
          bool inserted;
          const u32 slot = slot_insert(B, key, inserted);
          if (slot == NONE) return;
          if (inserted) rs[2 * kk + sd] = slot;
          const unsigned long long old = at_min64(&B.slots[slot].sck, ck);
          if (inserted || old < ck) continue;
          const u32 li = at_inc_agg(B.n_log);
          if (li < B.cap_log) {
            CreateLog& L = B.log[li];
            L.ckey = ck; L.inst = slot; L.at = nd[r.node].tok; L.fn = q.i;
          } else {
            at_or(B.overflow, 4);
          }
        }
      }, st);
    }
    // 2. ids in candidate order, records, published ids
    {
      const u32 NS2 = 2 * NRC;
      u32* ins = dalloc<u32>(NS2 + 1);
      u32* ids = dalloc<u32>(NS2 + 1);
      const u32* rs = rslot;
      par_for(NS2 + 1, [=] EXS_HD (i64 j) { ins[j] = j < NS2 && rs[j] < NONE - 1; }, st);
      excl_scan_u32(ins, ids, NS2 + 1, sc, st);
      {
        const u32* idl = ids + NS2; u32* ns_ = nslow;
        par_for(1, [=] EXS_HD (i64) { ns_[1] = *idl; }, st);
      }
      u32 two[2];
      d2h(two, nslow, 8, st);
      sync(st);
      const u32 total = two[1];
      roots_keyed = two[0] == 0;
      const u32* id_of = ids;
      const RootStash* rst = rstash;
      par_for(NS2, [=] EXS_HD (i64 j) {
        const u32 slot = rs[j];
        if (slot >= NONE - 1) return;
        const u32 id = id_of[j];
        if (id >= B.cap_inst) { at_or(B.overflow, 1u); return; }
        const RootStash z = rst[j >> 1];
        const u8 sd = (u8)(j & 1);
        Val ot = vnone();
        if (z.rec != NONE) { ot.k = V_TYPE; ot.x = z.otx; ot.rec = z.otrec; ot.bt = BT_NONE; ot.targ = 0; }
        Slot& S_ = B.slots[slot];
        Inst& I = B.inst[id];
        I.ka = S_.k.a; I.kb = S_.k.b;  // the key step 1 inserted (make_ikey of the decl, owner, walk, side)
        I.ckey = ~0ull; I.fn = rcc[j >> 1] >> 1; I.orec = z.rec; I.walk = z.walk; I.at = z.at;
        I.ebase = 0; I.ecnt = 0;
        I.tb = vnone(); I.hb = vnone(); I.ot = ot;
        I.side = sd; I.spaces = z.sp[sd]; I.pad = 0; I.slot = slot;
        I.flags = z.iflags;  // fill_instance's flags, from the decl record
        I.ckey = S_.sck;     // final: every root creator ran in step 1 (step 3 redoes it otherwise)
        S_.sid = id;
        if (z.iflags & IF_MAIN) note_main(B, id);
      }, st);
      u32* ni = B.n_inst;
      par_for(1, [=] EXS_HD (i64) { *ni = total; }, st);
      // log entries of step 1 hold slots: resolve them to ids
      const u32 nlog1 = get1(B.n_log, st);
      const u32 lo = nlog0, hi = nlog1 < B.cap_log ? nlog1 : B.cap_log;
      if (hi > lo) {
        CreateLog* lg = B.log; const Slot* sl = B.slots;
        par_for(hi - lo, [=] EXS_HD (i64 j) { lg[lo + j].inst = sl[lg[lo + j].inst].sid; }, st);
      }
      sync(st);
      dfree(ins);
      dfree(ids);
    }
    // 3. proposal1 conditional specifiers: evaluated by a walker
    const u32* rs3 = rslot;
    par_for_walk(NRC, [=] EXS_HD (i64 kk) {
      if (rs3[2 * kk] != NONE - 1) return;
      const RootCand q = cand(rcc[kk], (u32)kk, false);
      const u32 i = q.i, p = q.p, file = q.file, walk = q.walk;
      const FnRec& r = fr[i];
      const Node& fn = nd[r.node];
      const u8 c = q.cfg, mode = q.mode;
      const Val ot = q.ot;
      Walker w;
      w.S.init(tab, r.view, c);
      w.B = &B; w.T = tab; w.file = file; w.walk = walk; w.inst_id = NONE;
      w.native = (u8)p; w.side = 0; w.clevel = 0;  // roots are created at level 0
      w.fn = i; w.pragma = false; w.from_hd = false;
      w.fidelity_host = mode == MODE_FIDELITY && p == 0;
      w.parent_rank = vd0 ? i - vd0[r.view] : i; w.contract = false;
      w.stmt_k = 0; w.stmt_ord = 0; w.stmt_ord_max = 2; w.stmt_cs_base = 0; w.cs_ord = 0;
      w.silent = false; w.asp = 0; w.nloc = 0; w.wdepth = 0; w.ebase = 0; w.ecnt = 0;
      Env none; none.clear();
      u8 sides;
      if (fn.n & FF_G) sides = 2;
      else {
        u8 sp;
        w.S.depth = 0;
        u8 stt = w.S.spaces(i, nullptr, vnone(), vnone(), 0, fn.tok, r.rec, sp);
        if (w.S.contract) { at_or(&B.contract[file], 1); return; }
        if (stt == ST_SEMA) { w.emit_err(); return; }
        if (stt == ST_SUBST) { w.emit_tok(C_E0001, fn.tok, M_W_PRED_CONST); return; }
        sides = sp & 3;
      }
      u32 k = 0;
      for (u8 sd = 0; sd < 2; sd++) {
        if (!((sides >> sd) & 1)) continue;
        w.stmt_ord = k++;  // roots: decl order x side order (spacecheck.py:272-283)
        w.instantiate(i, vnone(), vnone(), sd, r.rec, none, ot, fn.tok);
      }
      if (w.contract) at_or(&B.contract[file], 1);
    }, st);
    sync(st);
    dfree(rcand);
    dfree(rslot);
    dfree(rstash);
    dfree(nslow);
    dfree(rot);
    dfree(vd0);
  }
  prof_mark(st);
  // ---- levels
  u32 prev_n = 0;
  u32 level = 0;
  // bounds on the parent ranks and locals of the next frontier's creation
  // keys; the roots': decl indices and the side order
  u64 rank_lim = std::min<u64>(std::max<u64>(NF, 1), (u64)CK_FIELD_MAX + 1);
  u64 local_lim = 2;
  u32* front = nullptr;
  u64 front_cap = 0;
  u64 edges_used = 0;
  W.callsites = 0;
  while (true) {
    std::vector<u32> cnt = W.read_counters(st);
    const bool ovf_local = cnt[CNT_OVF] != 0;
    if (ovf_local && !W.coll.on()) { dfree(dtab); dfree(front); return false; }
    u32 n_now = cnt[CNT_INST];
    prof_mark(st);
    if (!ovf_local) {
      // creation keys of this level's instances (min over creators), then the
      // first creator's location (spacecheck.py:331-337)
      if (level > 0 || !roots_keyed) {  // the roots' keys were written with their records
        Inst* in = W.inst; const Slot* sl = W.slots; const u32 base = prev_n;
        par_for(n_now - prev_n, [=] EXS_HD (i64 j) { Inst& I = in[base + j]; I.ckey = sl[I.slot].sck; }, st);
      }
      {
        const CreateLog* lg = W.log; Inst* in = W.inst;
        par_for(cnt[CNT_LOG], [=] EXS_HD (i64 j) {
          const CreateLog& e = lg[j];
          Inst& I = in[e.inst];
          if (I.ckey == e.ckey) { I.at = e.at; I.fn = e.fn; }
        }, st);
      }
    }
    dzero(W.ctr(CNT_LOG), 4, st);
    // a sharded walk: the ranks' new instances of the level just walked are
    // merged everywhere (the roots, level 0, are built alike on every rank)
    if (W.coll.on() && level > 0 && merge_level(W, prev_n, n_now, ovf_local, st)) {
      dfree(dtab); dfree(front); return false;
    }
    B = bufs();
    u32 nnew = n_now - prev_n;
    if (!nnew) break;
    prof_mark(st);
    // frontier: new instances with a body to walk (IF_BODY: an empty,
    // parameterless body is left out -- creation keys only order the creators
    // among themselves, so dropping non-creators keeps them), by creation key
    // (no host round trip: body instances sort first, the count stays on the
    // device until the totals below are read)
    grow(front, front_cap, nnew + 1, 0, st);
    u32* tot = dalloc<u32>(4);  // edge slots, work items, frontier size, most call sites of a body
    dzero(tot, 16, st);
    {
      const Inst* in = W.inst;
      u32 base = prev_n;
      u32* fr_tmp = dalloc<u32>(nnew + 1);
      // sort keys: (parent rank, local) of the creation key -- the level bits
      // are equal in a frontier, parent ranks are below the previous frontier's
      // size and locals below twice its largest body's call sites -- with the
      // non-body instances last; 32-bit keys when they fit (fewer radix passes)
      auto nbits = [](u64 lim) { int b = 0; while (b < 26 && (lim - 1) >> b) b++; return b; };
      const int rbits = nbits(rank_lim), lbits = nbits(local_lim);
      // non-body instances: the all-ones key when no body key reaches it
      // (a bound below its field's power of two), else a flag bit above
      const bool spare = rank_lim < (1ull << rbits) || local_lim < (1ull << lbits);
      const int kbits = rbits + lbits + (spare ? 0 : 1);
      const u64 last = spare ? (1ull << (rbits + lbits)) - 1 : 1ull << (rbits + lbits);
      u32* nfd = tot + 2;
      auto key_of = [=] EXS_HD (const Inst& I) -> u64 {
        if (!(I.flags & IF_BODY)) return last;
        const u64 rank = (I.ckey >> CK_RANK_SHIFT) & CK_FIELD_MAX, local = I.ckey & CK_FIELD_MAX;
        return (rank << lbits) | local;
      };
      if (kbits <= 32) {
        u32* keys = dalloc<u32>(nnew + 1);
        par_for(nnew, [=] EXS_D (i64 j) {
          const Inst& I = in[base + j];
          keys[j] = (u32)key_of(I);
          fr_tmp[j] = base + (u32)j;
          if (I.flags & IF_BODY) at_inc_agg(nfd);
        }, st);
        sort_pairs(keys, fr_tmp, nnew, sc, st, kbits);
        dfree(keys);  // blocks are reused in stream order (cache_alloc): no wait
      } else {
        u64* keys = dalloc<u64>(nnew + 1);
        par_for(nnew, [=] EXS_D (i64 j) {
          const Inst& I = in[base + j];
          keys[j] = key_of(I);
          fr_tmp[j] = base + (u32)j;
          if (I.flags & IF_BODY) at_inc_agg(nfd);
        }, st);
        sort_pairs(keys, fr_tmp, nnew, sc, st, kbits);
        dfree(keys);
      }
      d2d(front, fr_tmp, 4ull * nnew, st);
      dfree(fr_tmp);
    }
    prev_n = n_now;
    const u32 nnew_prev = nnew;  // new instances per level track the next level's
    prof_mark(st);
    // edge bases (scan of call-site counts) and work items (scan of statement
    // chunks) over the frontier; the three totals come back in one round trip
    const u32 KCH = EXS_KCH;
    u32* ec = dalloc<u32>(nnew + 1);
    u32* eb = dalloc<u32>(nnew + 1);
    u32* wc = dalloc<u32>(nnew + 1);
    u32* wb = dalloc<u32>(nnew + 1);
    {
      const Inst* in = W.inst; const FnRec* fr = S.fns; const u32* fl = front; const u32* nfd = tot + 2;
      par_for(nnew + 1, [=] EXS_HD (i64 j) {
        if (j < *nfd) {
          const FnRec& r = fr[in[fl[j]].fn];
          ec[j] = r.ncalls;
          wc[j] = r.nstmts ? (r.nstmts + KCH - 1) / KCH : 1;
          at_max_agg(tot + 3, r.ncalls);
        } else {
          ec[j] = 0;
          wc[j] = 0;
        }
      }, st);
    }
    excl_scan_u32(ec, eb, nnew + 1, sc, st);
    excl_scan_u32(wc, wb, nnew + 1, sc, st);
    par_for(1, [=] EXS_HD (i64) { tot[0] = eb[nnew]; tot[1] = wb[nnew]; }, st);
    u32 tot_h[4];
    d2h(tot_h, tot, sizeof tot_h, st);
    sync(st);
    dfree(tot);
    const u32 nf = tot_h[2];
    if (!nf) { dfree(ec); dfree(eb); dfree(wc); dfree(wb); break; }
    u64 S_level = tot_h[0];
    const u32 nwi = tot_h[1];
    W.callsites += S_level;
    grow(W.edges, edge_cap, edges_used + S_level + 1, edges_used, st);
    // the creation log holds the creators that did not insert (several creators
    // of one instance in one level) -- few; it grows on overflow (buf_scale)
    grow(W.log, log_cap, std::min<u64>(2ull * S_level, ((u64)S_level / 8 + 65536) * W.buf_scale) + 64, 0, st);
    u32 npend = cnt[CNT_PEND], nseeds = cnt[CNT_SEEDS];
    grow(W.pend, pend_cap, (u64)npend + S_level + 64, npend, st);
    grow(W.seeds, seed_cap, 2ull * (nseeds + S_level) + 64, 2ull * nseeds, st);
    // a level creates at most ~one new instance per call site (exact for deep
    // chains, C3) and about as many as the previous level did (C4: calls hit
    // existing roots); an overflow is handled by the caller's walk-only retry
    grow_inst(W, (u64)n_now + std::min<u64>(S_level, 2ull * nnew_prev) + S_level / 8 + 65536, n_now, st);
    B = bufs();
    B.lvl_base = n_now;
    B.clevel = level + 1;
    {
      Inst* in = W.inst; const u32* fl = front; u64 eu = edges_used;
      par_for(nf, [=] EXS_HD (i64 j) { in[fl[j]].ebase = (u32)(eu + eb[j]); }, st);
    }
    dfill_ff(W.edges + edges_used, 4ull * S_level, st);  // empty edge slots
    edges_used += S_level;
    prof_mark(st);
    // walk the frontier: one thread per (instance, chunk of top-level statements)
    {
      const Inst* in = W.inst; const FnRec* fr = S.fns; const u32* fl = front;
      WalkCfg Cc = C;
      u32* ct = B.contract;
      const u32* sn = S.stmt_node; const u32* scs = S.stmt_cs;
      // the (frontier instance, chunk) of every work item, materialised once
      // (no per-thread binary search over the chunk prefix)
      u32* itj = dalloc<u32>(nwi + 1);
      u32* itc = dalloc<u32>(nwi + 1);
      par_for(nf, [=] EXS_HD (i64 j) {
        const u32 b0 = wb[j], n = wc[j];
        for (u32 c = 0; c < n; c++) { itj[b0 + c] = (u32)j; itc[b0 + c] = c; }
      }, st);
      // work items in statement-shape order (statement kind, expression kind):
      // warps then run similar code paths.  Results do not depend on the order
      // (creation keys and edge slots are order-free).
      u32* perm = nullptr;
#if EXS_WALK_SORT
      if (nwi >= EXS_WALK_SORT_MIN) {  // a small level: the sort costs more than it saves
        perm = dalloc<u32>(nwi + 1);
        u32* key = dalloc<u32>(nwi + 1);
        const Node* nd = P.nodes;
        par_for(nwi, [=] EXS_HD (i64 i) {
          const FnRec& r = fr[in[fl[itj[i]]].fn];
          u32 k = itc[i] * KCH;
          u32 shape = 0;
          if (k < r.nstmts) {
            const Node& s = nd[sn[r.stmt_base + k]];
            u32 sub = s.c0 != NONE ? nd[s.c0].kind : 0;
            shape = ((u32)s.kind << 8) | sub;
          }
          key[i] = shape;
          perm[i] = (u32)i;
        }, st);
        sort_pairs(key, perm, nwi, sc, st, 16);
        dfree(key);
      }
#endif
      // parent ranks (make_ckey): frontier positions while they fit the rank
      // field, else positions among the frontier entries of the same walk
      // (creation keys are only compared within a walk)
      u32* frank = nullptr;
      if (nf > CK_FIELD_MAX) {
        frank = dalloc<u32>(nf + 1);
        u64* wk = dalloc<u64>(nf + 1);
        u32* pos = dalloc<u32>(nf + 1);
        u32* wfirst = dalloc<u32>((u64)NW + 1);
        par_for(nf, [=] EXS_HD (i64 j) { wk[j] = in[fl[j]].walk; pos[j] = (u32)j; }, st);
        int wbits = 1;
        while (wbits < 32 && (NW >> wbits)) wbits++;
        sort_pairs(wk, pos, nf, sc, st, wbits);  // stable: frontier order within a walk
        par_for(nf, [=] EXS_HD (i64 p) { if (p == 0 || wk[p - 1] != wk[p]) wfirst[wk[p]] = (u32)p; }, st);
        u32* fk = frank;
        par_for(nf, [=] EXS_HD (i64 p) { fk[pos[p]] = (u32)p - wfirst[wk[p]]; }, st);
        sync(st);
        dfree(wk); dfree(pos); dfree(wfirst);
      }
      const u32* frk = frank;
      const u32* pm = perm;
      // a sharded walk: this rank's contiguous share of the (shape-ordered) items
      u64 it_lo = 0, it_hi = nwi;
      if (W.coll.on()) {
        it_lo = (u64)nwi * (u64)W.coll.rank / (u64)W.coll.world;
        it_hi = (u64)nwi * (u64)(W.coll.rank + 1) / (u64)W.coll.world;
      }
      EXS_TAG("walk_chunks");
      par_for_walk((i64)(it_hi - it_lo), [=] EXS_HD (i64 ii0) {
        const i64 ii = ii0 + (i64)it_lo;
        const u32 i = pm ? pm[ii] : (u32)ii;
        const u32 j = itj[i], c = itc[i];
        Walker w;
        walker_for(w, Cc, B, fl[j], frk ? (u64)frk[j] : (u64)j);
        const FnRec& r = fr[w.fn];
        u32 k0 = c * KCH, k1 = k0 + KCH < r.nstmts ? k0 + KCH : r.nstmts;
#ifdef EXS_EXP_NOWALK  // timing experiment only: walker set-up without the statements
        if (w.ecnt == 12345) w.run_chunk(sn, scs, r.stmt_base, k0, k1);
#else
        w.run_chunk(sn, scs, r.stmt_base, k0, k1);
#endif
        if (w.ecnt) at_add(&B.inst[fl[j]].ecnt, w.ecnt);
        if (w.contract) at_or(&ct[w.file], 1);
      }, st);
      dfree(perm);
      dfree(frank);
      dfree(itj);
      dfree(itc);
    }
    dfree(ec);
    dfree(eb);
    dfree(wc);
    dfree(wb);
    rank_lim = std::min<u64>(nf, (u64)CK_FIELD_MAX + 1);
    local_lim = std::min<u64>(std::max<u64>(2ull * tot_h[3], 1), (u64)CK_FIELD_MAX + 1);
    prof_mark(st);
    level++;
  }
  W.levels = level;
  dfree(front);
  W.n_inst = prev_n;
  W.n_edges = edges_used;
  if (W.coll.on()) {
    // a sharded walk: the edge slots and launch seeds each rank wrote for its
    // work items go to every rank (edge positions agree across ranks; callees
    // travel as creation keys and come back as local ids), then every
    // instance's legal-edge count is recounted from the merged slots
    const Coll& c = W.coll;
    const u32 n = W.n_inst;
    // instances ordered by (walk, creation key): two stable radix sorts
    u64* ck = dalloc<u64>((u64)n + 1);
    u64* wk = dalloc<u64>((u64)n + 1);
    u32* cid = dalloc<u32>((u64)n + 1);
    {
      const Inst* in = W.inst;
      par_for(n, [=] EXS_HD (i64 i) { ck[i] = in[i].ckey; cid[i] = (u32)i; }, st);
      sort_pairs(ck, cid, n, sc, st);
      const u32* ci = cid;
      par_for(n, [=] EXS_HD (i64 i) { wk[i] = in[ci[i]].walk; }, st);
      sort_pairs(wk, cid, n, sc, st, 32);
      par_for(n, [=] EXS_HD (i64 i) { ck[i] = in[ci[i]].ckey; }, st);
    }
    auto id_of = [=] EXS_HD (u32 walk, u64 key) -> u32 {  // binary search of (walk, creation key)
      u32 lo = 0, hi = n;
      while (lo < hi) {
        const u32 mid = (lo + hi) / 2;
        if (wk[mid] < walk || (wk[mid] == walk && ck[mid] < key)) lo = mid + 1; else hi = mid;
      }
      return lo < n && wk[lo] == walk && ck[lo] == key ? cid[lo] : NONE;
    };
    {
      // edges: (position, callee creation key)
      u32* pos = dalloc<u32>(edges_used + 1);
      const u32* ed = W.edges;
      const u32 ne = select_idx((i64)edges_used, [=] EXS_HD (u32 p) -> bool { return ed[p] != NONE; }, pos, L.cnt,
                                sc, st);
      XRef* xs = dalloc<XRef>((u64)ne + 1);
      const Inst* in = W.inst; const u32* ps = pos;
      par_for(ne, [=] EXS_HD (i64 k) {
        const Inst& I = in[ed[ps[k]]];
        XRef x; x.key = I.ckey; x.walk = I.walk; x.a = ps[k]; xs[k] = x;
      }, st);
      std::vector<u64> sizes;
      u64 total = 0;
      u8* recv = coll_allgatherv(c, xs, sizeof(XRef) * (u64)ne, sizes, total, st);
      u64 off = 0;
      u32* edw = W.edges;
      for (int r = 0; r < c.world; off += sizes[r], r++) {
        if (r == c.rank) continue;
        const XRef* rx = reinterpret_cast<const XRef*>(recv + off);
        par_for(sizes[r] / sizeof(XRef), [=] EXS_HD (i64 k) { edw[rx[k].a] = id_of(rx[k].walk, rx[k].key); }, st);
      }
      sync(st);
      dfree(recv); dfree(xs); dfree(pos);
    }
    {
      // launch seeds: (walk, target creation key)
      std::vector<u32> cnt = W.read_counters(st);
      const u32 ns = std::min<u32>(cnt[CNT_SEEDS], W.cap_seeds);
      XRef* xs = dalloc<XRef>((u64)ns + 1);
      const Inst* in = W.inst; const u32* sd = W.seeds;
      par_for(ns, [=] EXS_HD (i64 k) {
        const Inst& I = in[sd[2 * k + 1]];
        XRef x; x.key = I.ckey; x.walk = I.walk; x.a = sd[2 * k]; xs[k] = x;
      }, st);
      std::vector<u64> sizes;
      u64 total = 0;
      u8* recv = coll_allgatherv(c, xs, sizeof(XRef) * (u64)ns, sizes, total, st);
      const u64 all = total / sizeof(XRef);
      grow(W.seeds, seed_cap, 2ull * all + 64, 2ull * ns, st);
      W.cap_seeds = (u32)(seed_cap / 2);
      u64 off = 0, at = ns;
      u32* sw = W.seeds;
      for (int r = 0; r < c.world; off += sizes[r], r++) {
        if (r == c.rank) continue;
        const XRef* rx = reinterpret_cast<const XRef*>(recv + off);
        const u64 m = sizes[r] / sizeof(XRef), a0 = at;
        par_for(m, [=] EXS_HD (i64 k) {
          sw[2 * (a0 + k)] = rx[k].a;
          sw[2 * (a0 + k) + 1] = id_of(rx[k].walk, rx[k].key);
        }, st);
        at += m;
      }
      const u32 nsn = (u32)at;
      h2d(W.ctr(CNT_SEEDS), &nsn, 4, st);
      sync(st);
      dfree(recv); dfree(xs);
    }
    {
      Inst* in = W.inst; const FnRec* fr = S.fns; const u32* ed = W.edges;
      par_for(n, [=] EXS_HD (i64 i) {
        Inst& I = in[i];
        if (!(I.flags & IF_BODY)) return;
        const u32 ns = fr[I.fn].ncalls;
        u32 k = 0;
        for (u32 e = 0; e < ns; e++) k += ed[I.ebase + e] != NONE;
        I.ecnt = k;
      }, st);
    }
    sync(st);
    dfree(ck); dfree(wk); dfree(cid);
  }
  prof_mark(st);
  // ---- main instance per walk: the last created (max creation key), over the
  // list kept at creation (every instance in a sharded walk, whose merged
  // instances were created on other ranks, or past the list's capacity)
  {
    const Inst* in = W.inst; unsigned long long* mk = W.main_key; u32* mi = W.main_inst;
    const u32 nm = W.read_counters(st)[CNT_MAINS];
    const bool listed = !W.coll.on() && nm <= W.cap_mains;
    const u32 n = listed ? nm : W.n_inst;
    const u32* ml = listed ? W.mains : nullptr;
    par_for(n, [=] EXS_D (i64 j) {
      const u32 i = ml ? ml[j] : (u32)j;
      if (in[i].flags & IF_MAIN) {
#ifndef EXS_EMU
        atomicMax(&mk[in[i].walk], in[i].ckey + 1);
#else
        if (in[i].ckey + 1 > mk[in[i].walk]) mk[in[i].walk] = in[i].ckey + 1;
#endif
      }
    }, st);
    par_for(n, [=] EXS_HD (i64 j) {
      const u32 i = ml ? ml[j] : (u32)j;
      if ((in[i].flags & IF_MAIN) && mk[in[i].walk] == in[i].ckey + 1) mi[in[i].walk] = i;
    }, st);
  }
  prof_mark(st);
  // ---- reachability (spacecheck.py:617-632)
  W.visited = dalloc<u8>((u64)W.n_inst + 8);
  dzero(W.visited, (u64)W.n_inst + 8, st);
  {
    u32 n = W.n_inst;
    u32* q0 = dalloc<u32>((u64)n + 1);
    u32* q1 = dalloc<u32>((u64)n + 1);
    u32* qn = dalloc<u32>(2);
    dzero(qn, 8, st);
    u8* vis = W.visited; const u32* mi = W.main_inst; const u32* sd = W.seeds; const Inst* in = W.inst;
    std::vector<u32> cnt = W.read_counters(st);
    u32 nseeds = cnt[CNT_SEEDS];
    // host walks: main; device walks: launch seeds
    par_for(NW, [=] EXS_D (i64 w) {
      if (w & 1) return;
      u32 m = mi[w];
      if (m == NONE) return;
      vis[m] = 1;  // one main per walk
      u32 k = at_add(&qn[0], 1);
      q0[k] = m;
    }, st);
    par_for(nseeds, [=] EXS_D (i64 k) {
      u32 w = sd[2 * k], t = sd[2 * k + 1];
      if (!(w & 1)) return;
#ifndef EXS_EMU
      u32* wp = (u32*)(vis + (t & ~3u));
      u32 sh = (t & 3u) * 8;
      u32 old = atomicOr(wp, 1u << sh);
      if ((old >> sh) & 0xFF) return;
#else
      if (vis[t]) return;
      vis[t] = 1;
#endif
      u32 j = at_add(&qn[0], 1);
      q0[j] = t;
    }, st);
    // BFS steps in rounds of RS launches with the queue lengths on the device:
    // one host round trip per round, not per step (C3: 66 steps); a step past
    // the end reads a zero length and returns
    const u32* ed = W.edges;
    const FnRec* fr_ = S.fns;
    // instances with many call sites (a main calling every chain head, C3) are
    // expanded by a 256-lane group each, not by one thread
    constexpr int RS = 8;
    constexpr u32 HEAVY = 64;
    const i64 G = grid_threads();
    u32* qc = dalloc<u32>(2 * RS + 1);  // queue lengths per step, then heavy-list lengths
    u32* hq = dalloc<u32>((u64)n + 1);
    d2d(qc, qn, 4, st);  // the seeds' queue length
    for (;;) {
      dzero(qc + 1, 4 * 2 * RS, st);
      for (int r = 0; r < RS; r++) {
        const u32* qa = q0; u32* qb = q1;
        const u32* cin = qc + r; u32* cout = qc + r + 1; u32* hn = qc + RS + 1 + r;
        // the newly reached callees of one instance, from edge slot e0 in steps of de
        auto expand = [=] EXS_D (const Inst& I, u32 e0, u32 de) {
          const u8 native = (u8)(I.walk & 1);
          const u32 ns = fr_[I.fn].ncalls;
          for (u32 e = e0; e < ns; e += de) {
            u32 c = ed[I.ebase + e];
            if (c == NONE || in[c].side != native) continue;
#ifndef EXS_EMU
            u32* wp = (u32*)(vis + (c & ~3u));
            u32 sh = (c & 3u) * 8;
            u32 old = atomicOr(wp, 1u << sh);
            if ((old >> sh) & 0xFF) continue;
#else
            if (vis[c]) continue;
            vis[c] = 1;
#endif
            u32 k = at_inc_agg(cout);  // warp-aggregated: one atomic per warp
            qb[k] = c;
          }
        };
        EXS_TAG("walk_reach");
        par_for(G, [=] EXS_D (i64 t) {
          const i64 nq = *cin;
          for (i64 j = t; j < nq; j += G) {
            const Inst& I = in[qa[j]];
            if (fr_[I.fn].ncalls > HEAVY) { hq[at_inc_agg(hn)] = qa[j]; continue; }
            expand(I, 0, 1);
          }
        }, st);
        EXS_TAG("walk_reach_heavy");
        par_for(G, [=] EXS_D (i64 t) {
          const i64 nh = *hn;
          for (i64 h = t >> 8; h < nh; h += G >> 8) expand(in[hq[h]], (u32)(t & 255), 256);
        }, st);
        std::swap(q0, q1);
      }
      if (!get1(qc + RS, st)) break;
      d2d(qc, qc + RS, 4, st);
    }
    dfree(qc);
    dfree(hq);
    sync(st);
    dfree(q0); dfree(q1); dfree(qn);
  }
  prof_mark(st);
  // ---- pending verdicts (spacecheck.py:634-655)
  {
    std::vector<u32> cnt = W.read_counters(st);
    const Pending* pd = W.pend; const Inst* in = W.inst; const u8* vis = W.visited;
    const FnRec* fr = S.fns; const Node* nd = P.nodes; const u32* vf = P.vfile; const u8* cfgs = L.cfg;
    WalkBufs Bc = B;
    EXS_TAG("walk_pending");
    par_for(cnt[CNT_PEND], [=] EXS_HD (i64 j) {
      const Pending& p = pd[j];
      const Inst& I = in[p.caller];
      u8 native = (u8)(p.walk & 1);
      if (I.side != native) return;
      u32 file = vf[fr[I.fn].view];
      u8 c = cfgs[file];
      u8 mode = c & CFG_MODE_MASK;
      u16 code = verdict(I.side, p.callee, true, mode, vis[p.caller] != 0);
      if (!code) return;
      if (mode == MODE_FIDELITY && native == 0 && !hard_code(code)) return;
      bool warn = code == C_W1101 || code == C_W1102 || code == C_W1502;
      u8 sup = warn && (nd[fr[I.fn].node].n & FF_PRAGMA) ? 1 : 0;
      emit_diag(Bc, mkdiag(file, p.line, p.col, code, M_W_STRAY, p.callee, I.side, 1, 0, sup));
    }, st);
  }
  sync(st);
  dfree(dtab);
  return true;
}

}  // namespace exs
