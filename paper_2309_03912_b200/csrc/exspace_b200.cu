// exspace_b200.cu -- pipeline driver and C ABI (include/exspace_b200.h).
//
// One exs_run() = one batch of units:
//   K1-K3 lex (exs_stage_lex.cuh) -> K4 parse (exs_stage_parse.cuh) ->
//   K5 symbol join + resolve checks (exs_stage_sema.cuh) ->
//   K6-K8 instantiation fixpoint, reachability, verdicts (exs_stage_walk.cuh) ->
//   divergence (E1201) and the ordered diagnostic set (this file).
#include "exs_stage_walk.cuh"
#include "../../include/exspace_b200.h"
#include <chrono>
#include <map>
#include <mutex>

namespace exs {
#ifndef EXS_EMU
int g_sm_count = 148;
u64 g_launches = 0;
thread_local cudaStream_t g_alloc_stream = 0;
bool g_profile = getenv("EXS_PROFILE") != nullptr;
std::vector<ProfRec> g_prof;
thread_local const char* g_tag = nullptr;
thread_local i64 g_select_flagged_min = EXS_SELECT_FLAGGED_MIN;
static std::string g_prof_text;

// size-exact block cache (see exs_par.cuh); keyed per stream so handles on
// different streams never share a block
struct BlockCache {
  std::mutex mu;
  std::multimap<std::pair<cudaStream_t, size_t>, void*> free_;
  std::map<void*, std::pair<cudaStream_t, size_t>> live;
  size_t cached = 0;
  size_t live_bytes = 0, peak_bytes = 0;
};
static BlockCache g_cache;

void* cache_alloc(size_t bytes) {
  bytes = (bytes + 255) & ~size_t(255);
  std::lock_guard<std::mutex> g(g_cache.mu);
  auto it = g_cache.free_.find({g_alloc_stream, bytes});
  void* p = nullptr;
  if (it != g_cache.free_.end()) {
    p = it->second;
    g_cache.free_.erase(it);
    g_cache.cached -= bytes;
  } else {
    cudaError_t e = cudaMallocAsync(&p, bytes, g_alloc_stream);
    if (e != cudaSuccess) {
      // release cached blocks of this stream and retry once
      cudaGetLastError();
      for (auto i = g_cache.free_.begin(); i != g_cache.free_.end();) {
        if (i->first.first == g_alloc_stream) {
          cudaFreeAsync(i->second, g_alloc_stream);
          g_cache.cached -= i->first.second;
          i = g_cache.free_.erase(i);
        } else {
          ++i;
        }
      }
      cudaStreamSynchronize(g_alloc_stream);
      e = cudaMallocAsync(&p, bytes, g_alloc_stream);
      if (e != cudaSuccess) {
        cudaGetLastError();
        char msg[256];
        snprintf(msg, sizeof msg,
                 "device out of memory: %.1f MiB requested with %.1f MiB live (peak %.1f MiB) in this "
                 "process's pipelines; split the batch",
                 bytes / 1048576.0, g_cache.live_bytes / 1048576.0, g_cache.peak_bytes / 1048576.0);
        throw std::runtime_error(msg);
      }
    }
  }
  g_cache.live[p] = {g_alloc_stream, bytes};
  g_cache.live_bytes += bytes;
  if (g_cache.live_bytes > g_cache.peak_bytes) g_cache.peak_bytes = g_cache.live_bytes;
  return p;
}

void cache_free(void* p) {
  std::lock_guard<std::mutex> g(g_cache.mu);
  auto it = g_cache.live.find(p);
  if (it == g_cache.live.end()) { cudaFreeAsync(p, g_alloc_stream); return; }
  g_cache.free_.insert({it->second, p});
  g_cache.cached += it->second.second;
  g_cache.live_bytes -= it->second.second;
  g_cache.live.erase(it);
}

// drop every cached block of a stream (handle destruction)
static void cache_release(cudaStream_t s) {
  std::lock_guard<std::mutex> g(g_cache.mu);
  for (auto i = g_cache.free_.begin(); i != g_cache.free_.end();) {
    if (i->first.first == s) {
      cudaFreeAsync(i->second, s);
      g_cache.cached -= i->first.second;
      i = g_cache.free_.erase(i);
    } else {
      ++i;
    }
  }
}

// fold the recorded launch events into "site ms count" lines
static void collect_profile() {
  if (!g_profile) return;
  cudaDeviceSynchronize();
  std::vector<std::pair<std::string, std::pair<double, int>>> acc;
  cudaEvent_t last_mark = nullptr;
  std::string last_name;
  for (auto& p : g_prof) {
    float ms = 0;
    std::string k;
    if (p.line < 0) {  // a timeline mark: interval since the previous mark
      if (last_mark) cudaEventElapsedTime(&ms, last_mark, p.a);
      k = "[" + last_name + " .. " + std::to_string(-p.line) + "]";
      last_name = std::string(p.fn) + ":" + std::to_string(-p.line);
      if (last_mark) cudaEventDestroy(last_mark);
      last_mark = p.a;
      if (k == "[ .. " + std::to_string(-p.line) + "]") continue;
    } else {
      cudaEventElapsedTime(&ms, p.a, p.b);
      cudaEventDestroy(p.a);
      cudaEventDestroy(p.b);
      k = p.line ? std::string(p.fn) + ":" + std::to_string(p.line) : std::string(p.fn);
    }
    bool found = false;
    for (auto& e : acc)
      if (e.first == k) { e.second.first += ms; e.second.second++; found = true; break; }
    if (!found) acc.push_back({k, {ms, 1}});
  }
  g_prof.clear();
  g_prof_text.clear();
  for (auto& e : acc) {
    char b[256];
    snprintf(b, sizeof b, "%-40s %9.3f ms x%d\n", e.first.c_str(), e.second.first, e.second.second);
    g_prof_text += b;
  }
}
#else
u64 g_launches = 0;
#endif

static thread_local std::string g_err;

struct Handle {
  int device = 0;
  cudaStream_t st = 0;
  Scratch sc;
  LexState L;
  ParseState P;
  SemaState S;
  WalkState W;
  // diagnostics
  Diag* d_diags = nullptr;
  u32 cap_diags = 0;
  u64* d_dset = nullptr;
  u32 dmask = 0;
  u32* d_ndiags = nullptr;
  u32* d_contract = nullptr;
  u8* d_src_owned = nullptr;
  // ordered diagnostics on the host: pinned, so the D2H runs at full PCIe
  // speed and exs_diags_view can hand them out without a copy
  Diag* diags = nullptr;
  u64 n_diags_host = 0, diags_host_cap = 0;
  std::vector<u32> walk_inst, walk_edges, walk_dem;
  exs_stats stats{};
  float t_stage[4] = {0, 0, 0, 0};
  bool want_demands = false;
  u32 split_min = 16;  // statement-parallel body parsing threshold (tokens; C2 1 GB best)
  long long select_flagged_min = EXS_SELECT_FLAGGED_MIN;  // select_idx flag-pass threshold (indices)
  bool diag_sort_two_pass = false;  // force the two-key diagnostic sort (parity tests)

  void reset() {
    L.free_all(); L = LexState();
    P.free_all(); P = ParseState();
    S.free_all(); S = SemaState();
    W.free_all(); W = WalkState();
    dfree(d_diags); d_diags = nullptr;
    dfree(d_dset); d_dset = nullptr;
    dfree(d_ndiags); d_ndiags = nullptr;
    dfree(d_contract); d_contract = nullptr;
  }
  ~Handle() {
    reset();
#ifndef EXS_EMU
    if (diags) cudaFreeHost(diags);
#else
    free(diags);
#endif
    dfree(d_src_owned);
    dfree(sc.p);
    sc.p = nullptr;
    sc.cap = 0;
#ifndef EXS_EMU
    cache_release(st);
    if (st) { cudaStreamSynchronize(st); cudaStreamDestroy(st); }
#endif
  }
};

inline void bind_stream(Handle& H) {
#ifndef EXS_EMU
  g_alloc_stream = H.st;
  cudaSetDevice(H.device);
#else
  (void)H;
#endif
}

struct Timer {
#ifndef EXS_EMU
  cudaEvent_t a, b;
  cudaStream_t s;
  explicit Timer(cudaStream_t s_) : s(s_) {
    cudaEventCreate(&a); cudaEventCreate(&b); cudaEventRecord(a, s);
  }
  float stop() {
    cudaEventRecord(b, s); cudaEventSynchronize(b);
    float ms = 0; cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a); cudaEventDestroy(b);
    return ms;
  }
#else
  std::chrono::steady_clock::time_point t0;
  explicit Timer(cudaStream_t) : t0(std::chrono::steady_clock::now()) {}
  float stop() {
    return std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
#endif
};

// ---------------------------------------------------------------------------
// demands and __CUDA_ARCH__ divergence (spacecheck.py:255-257,345-346,753-767)

struct DemEnt {
  u64 key, rank;
  u32 id, walk;
  u8 kind, pad[7];
};

static void run_demands(Handle& H, bool emit_e1201) {
  LexState& L = H.L; ParseState& P = H.P; SemaState& S = H.S; WalkState& W = H.W;
  cudaStream_t st = H.st;
  const u32 NF = S.NF, NI = W.n_inst, F = L.F;
  const u64 NE = 2ull * NF + NI;
  DemEnt* ent = dalloc<DemEnt>(NE + 1);
  u64* keys = dalloc<u64>(NE + 1);
  u32* idx = dalloc<u32>(NE + 1);
  const FnRec* fr = S.fns; const Node* nd = P.nodes; const FP* fp = L.fp; const u32* vf = P.vfile;
  const Tok* tk = L.toks;
  par_for(2ull * NF, [=] EXS_HD (i64 x) {
    u32 i = (u32)(x >> 1), p = (u32)(x & 1);
    const FnRec& r = fr[i];
    u32 file = vf[r.view];
    u32 walk = 2 * file + p;
    DemEnt& e = ent[x];
    idx[x] = (u32)x;
    if (fp[walk].view != r.view || fp[walk].perr || ((r.flags & FR_DUP) && (r.flags & FR_OWNER))) {
      keys[x] = ~0ull; e.key = ~0ull; return;
    }
    e.key = hcombine(0xDEC1ull, r.sig);
    e.rank = r.order;
    e.id = i; e.walk = walk; e.kind = 1;
    keys[x] = nz(hcombine(file, e.key));
  }, st);
  const Inst* in = W.inst;
  par_for(NI, [=] EXS_HD (i64 j) {
    const Inst& I = in[j];
    u64 x = 2ull * NF + j;
    DemEnt& e = ent[x];
    idx[x] = (u32)x;
    const FnRec& r = fr[I.fn];
    const Node& fn = nd[r.node];
    if (fn.c0 == NONE && I.ot.k == V_NONE) { keys[x] = ~0ull; e.key = ~0ull; return; }
    u64 b = 0;
    for (u32 tp = fn.c0; tp != NONE; tp = nd[tp].next) {
      const Val& v = nd[tp].sub == 0 ? I.tb : I.hb;
      if (v.k == V_NONE) continue;
      u64 vc = v.k == V_TYPE ? hcombine(v.x, v.targ) : hcombine(0x4DC0ull, v.x);
      b += hcombine(tk[nd[tp].tok].hv, vc);
    }
    u64 oc = I.ot.k == V_TYPE ? hcombine(I.ot.x, I.ot.targ) : 0;
    e.key = hcombine(hcombine(0x1257ull, r.sig), hcombine(b, oc));
    e.rank = I.ckey;
    e.id = (u32)j; e.walk = I.walk; e.kind = 2;
    keys[x] = nz(hcombine(vf[r.view], e.key));
  }, st);
  sort_pairs(keys, idx, NE, H.sc, st);
  u32* dem = dalloc<u32>(2ull * F + 1);
  dzero(dem, 4ull * (2 * F + 1), st);
  WalkBufs B{};
  B.diags = H.d_diags; B.n_diags = H.d_ndiags; B.cap_diags = H.cap_diags; B.dset = H.d_dset;
  B.dmask = H.dmask; B.overflow = W.ctr(CNT_OVF);
  const u8* cfgs = L.cfg;
  par_for(NE, [=] EXS_HD (i64 i) {
    if (keys[i] == ~0ull) return;
    if (i > 0 && keys[i - 1] == keys[i]) return;
    u32 sides = 0;
    u64 best[2] = {~0ull, ~0ull};
    u32 besti[2] = {0, 0};
    u32 walks[2] = {NONE, NONE};
    for (u64 j = i; j < NE && keys[j] == keys[i]; j++) {
      const DemEnt& e = ent[idx[j]];
      u32 s = e.walk & 1;
      sides |= 1u << s;
      walks[s] = e.walk;
      if (e.rank < best[s]) { best[s] = e.rank; besti[s] = idx[j]; }
    }
    for (u32 s = 0; s < 2; s++) if (walks[s] != NONE) at_add(&dem[walks[s]], 1);
    if (!emit_e1201 || sides == 3) return;
    u32 s = sides == 1 ? 0 : 1;
    const DemEnt& e = ent[besti[s]];
    u32 file = e.walk >> 1;
    u8 mode = cfgs[file] & CFG_MODE_MASK;
    if (!(mode == MODE_SOUND || mode == MODE_P1 || mode == MODE_P2)) return;
    // both walks of the file must exist
    if (fp[2 * file].view == NONE || fp[2 * file].perr || fp[2 * file + 1].view == NONE || fp[2 * file + 1].perr) return;
    u32 loc_tok = e.kind == 1 ? nd[fr[e.id].node].tok : in[e.id].at;
    const Tok& t = tk[loc_tok];
    emit_diag(B, mkdiag(file, t.line, t.col, C_E1201, M_W_E1201, e.id, 0, 0, e.kind));
  }, st);
  H.walk_dem.assign(2 * F, 0);
  if (F) d2h(H.walk_dem.data(), dem, 8ull * F, st);
  sync(st);
  dfree(dem); dfree(ent); dfree(keys); dfree(idx);
}

// ---------------------------------------------------------------------------

static void run_batch(Handle& H, const u8* d_src, u64 n_bytes, const u64* foff, u32 n_files,
                      const u8* cfg) {
  if (n_bytes >= (1ull << 31)) throw Err("batch larger than 2 GiB; split into batches");
  cudaStream_t st = H.st;
  H.reset();
#ifndef EXS_EMU
  g_select_flagged_min = H.select_flagged_min;
#endif
  u64 launches0 = g_launches;
  Timer total(st);
  bool any_div = false;
  for (u32 f = 0; f < n_files; f++) {
    u8 m = cfg[f] & CFG_MODE_MASK;
    if (m == MODE_SOUND || m == MODE_P1 || m == MODE_P2) any_div = true;
  }
  u32 retries = 0;
  u32 cap_diags = (u32)std::max<u64>(65536, 64ull * n_files + n_bytes / 64);
  u32 cap_inst = 0;
  while (true) {
    H.reset();
    LexState& L = H.L;
    L.N = (u32)n_bytes;
    L.F = n_files;
    L.src = (u8*)d_src;
    std::vector<u32> fo(n_files + 1);
    for (u32 f = 0; f <= n_files; f++) fo[f] = (u32)foff[f];
    L.foff = dalloc<u32>(n_files + 1);
    h2d(L.foff, fo.data(), 4ull * (n_files + 1), st);
    L.cfg = dalloc<u8>(n_files + 1);
    if (n_files) h2d(L.cfg, cfg, n_files, st);
    // diagnostics buffers
    // n_files slots past the capacity the stages use: the out-of-contract
    // markers written after the last retry always fit
    H.cap_diags = cap_diags;
    H.d_diags = dalloc<Diag>((u64)cap_diags + n_files);
    H.dmask = pow2_at_least(2ull * cap_diags) - 1;
    H.d_dset = dalloc<u64>((u64)H.dmask + 1);
    dzero(H.d_dset, 8ull * (H.dmask + 1), st);
    H.d_ndiags = dalloc<u32>(1);
    dzero(H.d_ndiags, 4, st);
    H.d_contract = dalloc<u32>(n_files + 1);
    dzero(H.d_contract, 4ull * (n_files + 1), st);
    u32* ovf = dalloc<u32>(1);
    dzero(ovf, 4, st);
    WalkBufs B0{};
    B0.diags = H.d_diags; B0.n_diags = H.d_ndiags; B0.cap_diags = cap_diags; B0.dset = H.d_dset;
    B0.dmask = H.dmask; B0.overflow = ovf; B0.contract = H.d_contract;

    prof_mark(st);
    Timer t0(st);
    run_lex(L, B0, H.sc, st);
    H.t_stage[0] = t0.stop();
    prof_mark(st);
    Timer t1(st);
    run_parse(L, H.P, B0, H.sc, st, H.split_min);
    H.t_stage[1] = t1.stop();
    prof_mark(st);
    Timer t2(st);
    run_sema(L, H.P, H.S, B0, H.sc, st);
    H.t_stage[2] = t2.stop();
    // roots (<= 2 per decl) plus the first level's growth bound of run_walk
    // (one instance per call site, at most twice the roots): the table is not
    // rehashed on the common two-level corpora
    if (!cap_inst) {
      const u64 nf4 = 4ull * H.S.NF;
      cap_inst = (u32)std::min<u64>(std::max<u64>(65536, nf4 + std::min<u64>(H.S.NCS, nf4) + H.S.NCS / 8 + 65536 + 1024),
                                    0x7FFFFFFFull);
    }
    // the walk is retried alone (bigger instance table) after restoring the
    // diagnostics emitted by the earlier stages
    u32 nd0 = get1(H.d_ndiags, st);
    u64* dset_snap = dalloc<u64>((u64)H.dmask + 1);
    u32* ct_snap = dalloc<u32>(n_files + 1);
    d2d(dset_snap, H.d_dset, 8ull * (H.dmask + 1), st);
    d2d(ct_snap, H.d_contract, 4ull * (n_files + 1), st);
    prof_mark(st);
    Timer t3(st);
    u32 walk_ovf = 0;
    u32 buf_scale = 1;
    while (true) {
      H.W.free_all();
      H.W = WalkState();
      H.W.cap_inst = cap_inst;
      H.W.buf_scale = buf_scale;
      bool ok = run_walk(L, H.P, H.S, H.W, B0, H.sc, st, cap_diags);
      if (ok && (any_div || H.want_demands)) run_demands(H, any_div);
      walk_ovf = get1(H.W.ctr(CNT_OVF), st);
      (void)ok;
      if (!(walk_ovf & 7)) break;
      if ((walk_ovf & 2) && !(get1(ovf, st) & 2) && nd0 <= cap_diags) {
        // diagnostics overflowed inside the walk: grow the buffer and its dedup
        // set, keep the diagnostics of the earlier stages, re-run the walk only
        const u32 nd_now = get1(H.d_ndiags, st);
        const u32 ncap = (u32)std::min<u64>(4ull * std::max(nd_now, cap_diags), 0x7FFFFFFFull);
        Diag* ndg = dalloc<Diag>((u64)ncap + n_files);
        if (nd0) d2d(ndg, H.d_diags, sizeof(Diag) * (u64)nd0, st);
        const u32 nmask = pow2_at_least(2ull * ncap) - 1;
        u64* nset = dalloc<u64>((u64)nmask + 1);
        dzero(nset, 8ull * ((u64)nmask + 1), st);
        par_for(nd0, [=] EXS_HD (i64 i) { set_insert(nset, nmask, diag_hash(ndg[i])); }, st);
        dfree(H.d_diags); dfree(H.d_dset); dfree(dset_snap);
        H.d_diags = ndg; H.d_dset = nset; H.dmask = nmask; H.cap_diags = ncap; cap_diags = ncap;
        B0.diags = ndg; B0.cap_diags = ncap; B0.dset = nset; B0.dmask = nmask;
        dset_snap = dalloc<u64>((u64)nmask + 1);
        d2d(dset_snap, nset, 8ull * ((u64)nmask + 1), st);
      } else if (walk_ovf & 2) {
        break;  // the earlier stages overflowed too: outer loop
      }
      if (walk_ovf & 4) buf_scale = std::min<u32>(buf_scale * 4, 1u << 20);  // creation log
      if (walk_ovf & 1) {
        u32 n_now = get1(H.W.ctr(CNT_INST), st);
        cap_inst = (u32)std::min<u64>(std::max<u64>(8ull * cap_inst, 2ull * n_now), 0x7FFFFFFFull);
      }
      h2d(H.d_ndiags, &nd0, 4, st);
      d2d(H.d_dset, dset_snap, 8ull * (H.dmask + 1), st);
      d2d(H.d_contract, ct_snap, 4ull * (n_files + 1), st);
      retries++;
    }
    H.t_stage[3] = t3.stop();
    dfree(dset_snap);
    dfree(ct_snap);
    u32 ovf_h = get1(ovf, st);
    u32 nd = get1(H.d_ndiags, st);
    dfree(ovf);
    if (nd > cap_diags || (ovf_h & 2) || (walk_ovf & 2)) {
      cap_diags = (u32)std::min<u64>(4ull * std::max(nd, cap_diags), 0x7FFFFFFFull);
      retries++;
      continue;
    }
    break;
  }
  // out-of-contract units get one marker record
  {
    u32* ct = H.d_contract;
    WalkBufs B{};
    B.diags = H.d_diags; B.n_diags = H.d_ndiags; B.cap_diags = H.cap_diags + n_files; B.dset = H.d_dset;
    B.dmask = H.dmask; B.overflow = H.W.ctr(CNT_OVF);
    par_for(n_files, [=] EXS_HD (i64 f) {
      if (ct[f]) emit_diag(B, mkdiag((u32)f, 1, 1, C_X9999, M_X_CONTRACT));
    }, st);
  }
  // order diagnostics by (file, line, col, code) with two stable radix passes
  u32 nd = std::min(get1(H.d_ndiags, st), H.cap_diags + n_files);
  {
    u64* k = dalloc<u64>(nd + 1);
    u32* ix = dalloc<u32>(nd + 1);
    const Diag* dd = H.d_diags;
    // field widths (OR of every value: its top bit is the maximum's)
    u32* wor = dalloc<u32>(4);
    dzero(wor, 16, st);
    const i64 T = std::min<i64>((i64)nd, 1 << 16);
    par_for(T, [=] EXS_HD (i64 t) {
      u32 o[4] = {0, 0, 0, 0};
      for (i64 i = t; i < (i64)nd; i += T) {
        o[0] |= dd[i].file; o[1] |= dd[i].line; o[2] |= dd[i].col; o[3] |= dd[i].code;
      }
      for (int q = 0; q < 4; q++) {
#if defined(__CUDA_ARCH__) && !defined(EXS_EMU)
        o[q] = __reduce_or_sync(__activemask(), o[q]);
        if ((threadIdx.x & 31) != (__ffs(__activemask()) - 1)) continue;
#endif
        if (o[q]) at_or(&wor[q], o[q]);
      }
    }, st);
    u32 wo[4] = {0, 0, 0, 0};
    if (nd) { d2h(wo, wor, 16, st); sync(st); }
    dfree(wor);
    auto bits = [](u32 v) { int b = 0; while (v) { b++; v >>= 1; } return b; };
    const int bf = bits(wo[0]), bl = bits(wo[1]), bc = bits(wo[2]), bk = bits(wo[3]);
    if (bf + bl + bc + bk <= 64 && !H.diag_sort_two_pass) {
      // (file, line, col, code) in one key: one stable radix sort of bf+bl+bc+bk bits
      const int sl = bk + bc, sf = bk + bc + bl;
      par_for(nd, [=] EXS_HD (i64 i) {
        ix[i] = (u32)i;
        k[i] = (sf < 64 ? (u64)dd[i].file << sf : 0) | ((u64)dd[i].line << sl) | ((u64)dd[i].col << bk) | dd[i].code;
      }, st);
      sort_pairs(k, ix, nd, H.sc, st, std::max(1, bf + bl + bc + bk));
    } else {
      par_for(nd, [=] EXS_HD (i64 i) { ix[i] = (u32)i; k[i] = ((u64)dd[i].col << 16) | dd[i].code; }, st);
      sort_pairs(k, ix, nd, H.sc, st, 48);
      par_for(nd, [=] EXS_HD (i64 i) { k[i] = ((u64)dd[ix[i]].file << 32) | dd[ix[i]].line; }, st);
      sort_pairs(k, ix, nd, H.sc, st);
    }
    Diag* out = dalloc<Diag>(nd + 1);
    par_for(nd, [=] EXS_HD (i64 i) { out[i] = dd[ix[i]]; }, st);
    if ((u64)nd > H.diags_host_cap) {
      u64 cap = (u64)nd + nd / 4 + 1024;
#ifndef EXS_EMU
      if (H.diags) cudaFreeHost(H.diags);
      CK(cudaHostAlloc((void**)&H.diags, cap * sizeof(Diag), cudaHostAllocDefault));
#else
      free(H.diags);
      H.diags = (Diag*)malloc(cap * sizeof(Diag));
#endif
      H.diags_host_cap = cap;
    }
    H.n_diags_host = nd;
    Timer td(st);
    if (nd) d2h(H.diags, out, sizeof(Diag) * (u64)nd, st);
    sync(st);
    H.stats.ms_d2h = td.stop();
    dfree(out); dfree(k); dfree(ix);
  }
  // per-walk statistics
  {
    u32 F = n_files;
    H.walk_inst.assign(2 * F, 0);
    H.walk_edges.assign(2 * F, 0);
    u32* wi = dalloc<u32>(2ull * F + 1);
    u32* we = dalloc<u32>(2ull * F + 1);
    dzero(wi, 4ull * (2 * F + 1), st);
    dzero(we, 4ull * (2 * F + 1), st);
    const Inst* in = H.W.inst;
    par_for(H.W.n_inst, [=] EXS_HD (i64 i) {
      at_add(&wi[in[i].walk], 1);
      at_add(&we[in[i].walk], in[i].ecnt);
    }, st);
    if (F) {
      d2h(H.walk_inst.data(), wi, 8ull * F, st);
      d2h(H.walk_edges.data(), we, 8ull * F, st);
    }
    sync(st);
    dfree(wi); dfree(we);
    if (H.walk_dem.size() != 2 * F) H.walk_dem.assign(2 * F, 0);
  }
  exs_stats& s = H.stats;
  s.bytes = n_bytes; s.files = n_files; s.lines = H.L.L; s.directives = H.L.D; s.tokens = H.L.T;
  s.views = H.P.V; s.view_tokens = H.P.VT; s.items = H.P.FI; s.functions = H.S.NF;
  s.structs = H.S.NR; s.instances = H.W.n_inst; s.edges = H.W.n_edges; s.callsites = H.W.callsites;
  s.levels = H.W.levels; s.diagnostics = nd; s.retries = retries;
  s.ms_lex = H.t_stage[0]; s.ms_parse = H.t_stage[1]; s.ms_sema = H.t_stage[2]; s.ms_walk = H.t_stage[3];
  s.ms_total = total.stop();
  s.gpu_launches = g_launches - launches0;
#ifndef EXS_EMU
  collect_profile();
#endif
}

}  // namespace exs

using namespace exs;

struct exs_handle_s {
  Handle h;
};

#define API_TRY try {
#define API_END                      \
  }                                  \
  catch (const std::exception& e) {  \
    g_err = e.what();                \
    return -1;                       \
  }                                  \
  return 0;

extern "C" {

const char* exs_last_error(void) { return g_err.c_str(); }

int exs_create(int device, exs_handle* out) {
  API_TRY
  auto* x = new exs_handle_s();
  x->h.device = device;
#ifndef EXS_EMU
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n <= 0) { delete x; throw Err("no CUDA device visible"); }
  CK(cudaSetDevice(device));
  cudaDeviceProp pr;
  CK(cudaGetDeviceProperties(&pr, device));
  g_sm_count = pr.multiProcessorCount;
  CK(cudaDeviceSetLimit(cudaLimitStackSize, 16384));
  CK(cudaStreamCreateWithFlags(&x->h.st, cudaStreamNonBlocking));
  // keep freed pool memory cached across stages and runs (no cudaFree syncs)
  cudaMemPool_t pool;
  CK(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t thr = ~0ull;
  CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  g_alloc_stream = x->h.st;
#endif
  *out = x;
  API_END
}

int exs_destroy(exs_handle h) {
  API_TRY
  bind_stream(h->h);
  delete h;
  API_END
}

int exs_run(exs_handle x, const uint8_t* bytes, uint64_t n_bytes, const uint64_t* file_off,
            uint32_t n_files, const uint8_t* file_cfg) {
  API_TRY
  Handle& H = x->h;
  bind_stream(H);
#ifndef EXS_EMU
  CK(cudaSetDevice(H.device));
#endif
  Timer th(H.st);
  // size-exact block cache: a repeated batch size gets its block back
  dfree(H.d_src_owned);
  H.d_src_owned = dalloc<u8>(n_bytes + 64);
  h2d(H.d_src_owned, bytes, n_bytes, H.st);
  dzero(H.d_src_owned + n_bytes, 64, H.st);
  sync(H.st);
  float ms_h2d = th.stop();
  run_batch(H, H.d_src_owned, n_bytes, file_off, n_files, file_cfg);
  H.stats.ms_h2d = ms_h2d;
  API_END
}

int exs_run_device(exs_handle x, const uint8_t* d_bytes, uint64_t n_bytes, const uint64_t* file_off,
                   uint32_t n_files, const uint8_t* file_cfg) {
  API_TRY
  Handle& H = x->h;
  bind_stream(H);
#ifndef EXS_EMU
  CK(cudaSetDevice(H.device));
#endif
  run_batch(H, d_bytes, n_bytes, file_off, n_files, file_cfg);
  H.stats.ms_h2d = 0;
  API_END
}

int exs_get_stats(exs_handle x, exs_stats* out) {
  API_TRY
  *out = x->h.stats;
  API_END
}

int exs_set_option(exs_handle x, int key, int value) {
  API_TRY
  if (key == 1) x->h.want_demands = value != 0;
#ifndef EXS_EMU
  else if (key == 2) g_profile = value != 0;  // per-launch device timing of later runs
#endif
  else if (key == 3) x->h.split_min = value < 4 ? 4u : (u32)value;  // statement-split threshold (tokens)
  else if (key == 4) x->h.select_flagged_min = value < 0 ? 0 : value;  // flag-pass selection threshold
  else if (key == 5) x->h.diag_sort_two_pass = value != 0;  // diagnostic order by two sorts
  else throw Err("unknown option");
  API_END
}

const char* exs_profile_text(void) {
#ifndef EXS_EMU
  return g_prof_text.c_str();
#else
  return "";
#endif
}

int exs_stage_times(exs_handle x, float* out4) {
  API_TRY
  for (int i = 0; i < 4; i++) out4[i] = x->h.t_stage[i];
  API_END
}

int exs_get_diags(exs_handle x, exs_diag* out, uint64_t cap, uint64_t* n) {
  API_TRY
  const Handle& H = x->h;
  *n = H.n_diags_host;
  u64 m = std::min<u64>(cap, H.n_diags_host);
  if (m) memcpy(out, H.diags, m * sizeof(Diag));
  API_END
}

int exs_diags_view(exs_handle x, const exs_diag** out, uint64_t* n) {
  API_TRY
  const Handle& H = x->h;
  *n = H.n_diags_host;
  *out = reinterpret_cast<const exs_diag*>(H.diags);
  API_END
}

int exs_get_arena(exs_handle x, uint8_t* out, uint64_t cap, uint64_t* n) {
  API_TRY
  Handle& H = x->h;
  bind_stream(H);
  u32 top = H.L.arena_top ? get1(H.L.arena_top, H.st) : 0;
  top = std::min(top, H.L.arena_cap);
  *n = top;
  u64 m = std::min<u64>(cap, top);
  if (m) { d2h(out, H.L.arena, m, H.st); sync(H.st); }
  API_END
}

int exs_get_pass_status(exs_handle x, exs_pass_status* out, uint64_t cap) {
  API_TRY
  Handle& H = x->h;
  bind_stream(H);
  u32 F = H.L.F;
  std::vector<FP> fp(2 * F);
  if (F) d2h(fp.data(), H.L.fp, sizeof(FP) * 2 * F, H.st);
  sync(H.st);
  for (u64 i = 0; i < std::min<u64>(cap, 2ull * F); i++) {
    exs_pass_status& o = out[i];
    memset(&o, 0, sizeof(o));
    const FP& r = fp[i];
    o.exists = r.pp_line != NONE - 1;
    if (!o.exists) continue;
    if (r.pp_line != NONE) { o.pp_line = r.pp_line; o.pp_msg = r.pp_msg; }
    if (r.lex_pos != NONE) { o.lex_line = r.lex_line; o.lex_col = r.lex_col; o.lex_msg = r.lex_msg; }
    o.eof_line = r.eof_line; o.eof_col = r.eof_col; o.view = r.view; o.parse_failed = r.perr;
  }
  API_END
}

int exs_get_tokens(exs_handle x, uint32_t file, exs_token* out, uint64_t cap, uint64_t* n) {
  API_TRY
  Handle& H = x->h;
  bind_stream(H);
  if (file >= H.L.F) throw Err("file index out of range");
  u32 lt[2];
  d2h(lt, H.L.ftok + file, 8, H.st);
  sync(H.st);
  u64 cnt = lt[1] - lt[0];
  *n = cnt;
  u64 m = std::min<u64>(cap, cnt);
  if (m) { d2h(out, H.L.toks + lt[0], m * sizeof(Tok), H.st); sync(H.st); }
  API_END
}

int exs_get_walk_stats(exs_handle x, exs_walk_stats* out, uint64_t cap) {
  API_TRY
  Handle& H = x->h;
  bind_stream(H);
  u32 F = H.L.F;
  std::vector<FP> fp(2 * F);
  if (F) d2h(fp.data(), H.L.fp, sizeof(FP) * 2 * F, H.st);
  sync(H.st);
  for (u64 i = 0; i < std::min<u64>(cap, 2ull * F); i++) {
    out[i].instances = H.walk_inst[i];
    out[i].edges = H.walk_edges[i];
    out[i].demands = H.walk_dem.size() > i ? H.walk_dem[i] : 0;
    out[i].exists = fp[i].view != NONE && !fp[i].perr;
  }
  API_END
}

// ---- walk materialisation (the arrays behind Analysis.walks)
static_assert(sizeof(exs_val) == sizeof(Val), "exs_val mirrors Val");
static_assert(sizeof(exs_node) == sizeof(Node), "exs_node mirrors Node");
static_assert(sizeof(exs_token) == sizeof(Tok), "exs_token mirrors Tok");

int exs_get_decls(exs_handle x, exs_decl* out, uint64_t cap, uint64_t* n) {
  API_TRY
  Handle& H = x->h;
  bind_stream(H);
  const u32 NF = H.S.fns ? H.S.NF : 0;
  *n = NF;
  const u64 m = std::min<u64>(cap, NF);
  if (out && m) {
    std::vector<FnRec> fr(m);
    d2h(fr.data(), H.S.fns, sizeof(FnRec) * m, H.st);
    sync(H.st);
    for (u64 i = 0; i < m; i++) {
      out[i].node = fr[i].node; out[i].view = fr[i].view; out[i].rec = fr[i].rec;
      out[i].order = fr[i].order; out[i].ncalls = fr[i].ncalls;
      out[i].flags = fr[i].flags & (FR_DUP | FR_OWNER | FR_MEMBER);
    }
  }
  API_END
}

int exs_get_structs(exs_handle x, exs_struct* out, uint64_t cap, uint64_t* n) {
  API_TRY
  Handle& H = x->h;
  bind_stream(H);
  const u32 NR = H.S.recs ? H.S.NR : 0;
  *n = NR;
  const u64 m = std::min<u64>(cap, NR);
  if (out && m) {
    std::vector<RecRec> rr(m);
    d2h(rr.data(), H.S.recs, sizeof(RecRec) * m, H.st);
    sync(H.st);
    for (u64 i = 0; i < m; i++) { out[i].node = rr[i].node; out[i].view = rr[i].view; }
  }
  API_END
}

int exs_get_instances(exs_handle x, exs_inst* out, uint64_t cap, uint64_t* n) {
  API_TRY
  Handle& H = x->h;
  bind_stream(H);
  const u32 NI = H.W.inst ? H.W.n_inst : 0;
  *n = NI;
  const u64 m = std::min<u64>(cap, NI);
  if (out && m) {
    std::vector<Inst> in(m);
    d2h(in.data(), H.W.inst, sizeof(Inst) * m, H.st);
    sync(H.st);
    for (u64 i = 0; i < m; i++) {
      exs_inst& o = out[i];
      o.decl = in[i].fn; o.walk = in[i].walk; o.side = in[i].side; o.at = in[i].at;
      o.ebase = in[i].ebase; o.ecnt = in[i].ecnt; o.flags = in[i].flags; o.spaces = in[i].spaces;
      o.ckey = in[i].ckey;
      memcpy(&o.tb, &in[i].tb, sizeof(Val));
      memcpy(&o.hb, &in[i].hb, sizeof(Val));
      memcpy(&o.ot, &in[i].ot, sizeof(Val));
    }
  }
  API_END
}

int exs_get_edges(exs_handle x, uint32_t* out, uint64_t cap, uint64_t* n) {
  API_TRY
  Handle& H = x->h;
  bind_stream(H);
  const u64 NE = H.W.edges ? H.W.n_edges : 0;
  *n = NE;
  const u64 m = std::min<u64>(cap, NE);
  if (out && m) { d2h(out, H.W.edges, 4ull * m, H.st); sync(H.st); }
  API_END
}

int exs_get_nodes(exs_handle x, exs_node* out, uint64_t cap, uint64_t* n) {
  API_TRY
  Handle& H = x->h;
  bind_stream(H);
  const u64 NN = H.P.nodes ? H.P.n_nodes : 0;
  *n = NN;
  const u64 m = std::min<u64>(cap, NN);
  if (out && m) { d2h(out, H.P.nodes, sizeof(Node) * m, H.st); sync(H.st); }
  API_END
}

int exs_get_token_range(exs_handle x, uint64_t first, uint64_t count, exs_token* out) {
  API_TRY
  Handle& H = x->h;
  bind_stream(H);
  if (first > H.L.T || count > H.L.T - first) throw Err("token range out of bounds");
  if (count) { d2h(out, H.L.toks + first, sizeof(Tok) * count, H.st); sync(H.st); }
  API_END
}

int exs_describe(exs_handle x, const uint32_t* ids, const uint8_t* kinds, uint32_t n, exs_desc* out) {
  API_TRY
  Handle& H = x->h;
  bind_stream(H);
  if (!n) return 0;
  u32* d_ids = dalloc<u32>(n);
  u8* d_k = dalloc<u8>(n);
  exs_desc* d_out = dalloc<exs_desc>(n);
  h2d(d_ids, ids, 4ull * n, H.st);
  h2d(d_k, kinds, n, H.st);
  const FnRec* fr = H.S.fns; const RecRec* rr = H.S.recs; const Node* nd = H.P.nodes;
  const Tok* tk = H.L.toks; const Inst* in = H.W.inst;
  par_for(n, [=] EXS_HD (i64 i) {
    exs_desc o;
    memset(&o, 0, sizeof(o));
    auto span = [&](u32 t) -> u64 { return ((u64)tk[t].pos << 32) | (tk[t].end - tk[t].pos); };
    u32 fi = d_k[i] == 1 ? d_ids[i] : in[d_ids[i]].fn;
    const FnRec& r = fr[fi];
    o.name = span(nd[r.node].tok);
    if (r.flags & FR_OWNER) o.owner = span(nd[rr[r.rec].node].tok);
    if (d_k[i] == 2) {
      const Inst& I = in[d_ids[i]];
      if (I.ot.k == V_TYPE && I.ot.targ && I.ot.rec != NONE) { o.otype = span(nd[rr[I.ot.rec].node].tok); o.otarg = I.ot.targ; }
      u32 k = 0;
      for (u32 tp = nd[r.node].c0; tp != NONE && k < 2; tp = nd[tp].next) {
        const Val& v = nd[tp].sub == 0 ? I.tb : I.hb;
        if (v.k == V_NONE) continue;
        o.bname[k] = span(nd[tp].tok);
        if (v.k == V_TYPE) {
          o.bkind[k] = 1;
          o.bval[k] = v.rec != NONE ? span(nd[rr[v.rec].node].tok) : (0xFFFFFFFF00000000ull | v.bt);
          o.bvx[k] = v.targ;
        } else {
          o.bkind[k] = 2;
          o.bvx[k] = (u8)v.x;
        }
        k++;
      }
      o.nb = (u8)k;
    }
    d_out[i] = o;
  }, H.st);
  d2h(out, d_out, sizeof(exs_desc) * (u64)n, H.st);
  sync(H.st);
  dfree(d_ids); dfree(d_k); dfree(d_out);
  API_END
}

}  // extern "C"
