// exspace_b200.cu -- pipeline driver and C ABI (include/exspace_b200.h).
//
// One exs_run() = one batch of units:
//   K1-K3 lex (exs_stage_lex.cuh) -> K4 parse (exs_stage_parse.cuh) ->
//   K5 symbol join + resolve checks (exs_stage_sema.cuh) ->
//   K6-K8 instantiation fixpoint, reachability, verdicts (exs_stage_walk.cuh) ->
//   divergence (E1201) and the ordered diagnostic set (this file).
#include "exs_render.cuh"
#include "../../include/exspace_b200.h"
#include <chrono>
#include <map>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <thread>

namespace exs {
#ifndef EXS_EMU
int g_sm_count = 148;
thread_local u64 g_launches = 0;
thread_local cudaStream_t g_alloc_stream = 0;
int g_profile = getenv("EXS_PROFILE") != nullptr ? 2 : 0;
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
  u64 hits = 0, misses = 0, trims = 0, oom_retries = 0;
};
static BlockCache g_cache;
// idle blocks are given back past this bound (half the device by default, set
// at exs_create; EXS_CACHE_GB overrides): below it, blocks are reused -- a C4
// run with a 32 GiB bound kept trimming and re-allocating (337 -> 600 ms from
// run to run), with the device's half it reuses 94% of its blocks
static size_t g_cache_bound = 64ull << 30;

// give back every idle block (of every stream when s is null)
static void cache_trim_locked(cudaStream_t s) {
  for (auto i = g_cache.free_.begin(); i != g_cache.free_.end();) {
    if (!s || i->first.first == s) {
      cudaFreeAsync(i->second, i->first.first);
      g_cache.cached -= i->first.second;
      i = g_cache.free_.erase(i);
    } else {
      ++i;
    }
  }
}

void* cache_alloc(size_t bytes) {
  bytes = (bytes + 255) & ~size_t(255);
  // size classes above 1 MiB (three significant bits, <= 12.5% slack): the
  // batches of a stream differ in size, and exact sizes would never be reused
  if (bytes > (1u << 20)) {
    int hb = 63 - __builtin_clzll(bytes);
    const size_t q = size_t(1) << (hb - 3);
    bytes = (bytes + q - 1) & ~(q - 1);
  }
  std::lock_guard<std::mutex> g(g_cache.mu);
  // keep the cache bounded: past the bound of idle blocks, give this stream's back
  if (g_cache.cached > g_cache_bound) { cache_trim_locked(g_alloc_stream); g_cache.trims++; }
  // best fit among this stream's idle blocks, up to 25% larger than asked
  auto it = g_cache.free_.lower_bound({g_alloc_stream, bytes});
  void* p = nullptr;
  if (it != g_cache.free_.end() && it->first.first == g_alloc_stream && it->first.second <= bytes + bytes / 4) {
    p = it->second;
    bytes = it->first.second;
    g_cache.free_.erase(it);
    g_cache.cached -= bytes;
    g_cache.hits++;
  } else {
    g_cache.misses++;
    cudaError_t e = cudaMallocAsync(&p, bytes, g_alloc_stream);
    if (e != cudaSuccess) {
      // give back every idle block, wait for the frees, retry once
      cudaGetLastError();
      g_cache.oom_retries++;
      cache_trim_locked(nullptr);
      cudaDeviceSynchronize();
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

static std::vector<cudaEvent_t> g_prof_pool;
static size_t g_prof_used = 0;
cudaEvent_t prof_event() {
  if (g_prof_used == g_prof_pool.size()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    g_prof_pool.push_back(e);
  }
  return g_prof_pool[g_prof_used++];
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
      last_mark = p.a;
      if (k == "[ .. " + std::to_string(-p.line) + "]") continue;
    } else {
      cudaEventElapsedTime(&ms, p.a, p.b);
      k = p.line ? std::string(p.fn) + ":" + std::to_string(p.line) : std::string(p.fn);
    }
    bool found = false;
    for (auto& e : acc)
      if (e.first == k) { e.second.first += ms; e.second.second++; found = true; break; }
    if (!found) acc.push_back({k, {ms, 1}});
  }
  g_prof.clear();
  g_prof_used = 0;  // the pool's events are recorded again by the next run
  g_prof_text.clear();
  for (auto& e : acc) {
    char b[256];
    snprintf(b, sizeof b, "%-40s %9.3f ms x%d\n", e.first.c_str(), e.second.first, e.second.second);
    g_prof_text += b;
  }
}
#else
thread_local u64 g_launches = 0;
#endif

static thread_local std::string g_err;

// page-locked host buffer that grows geometrically, keeping its contents
struct PinnedBuf {
  u8* p = nullptr;
  u64 cap = 0;
  void ensure(u64 need, u64 keep) {
    if (need <= cap) return;
    const u64 ncap = std::max<u64>(need, cap + cap / 2) + 4096;
    u8* q = nullptr;
#ifndef EXS_EMU
    CK(cudaHostAlloc((void**)&q, ncap, cudaHostAllocDefault));
#else
    q = (u8*)malloc(ncap);
    if (!q) throw Err("out of host memory");
#endif
    if (keep) memcpy(q, p, keep);
    release();
    p = q;
    cap = ncap;
  }
  void release() {
#ifndef EXS_EMU
    if (p) cudaFreeHost(p);
#else
    free(p);
#endif
    p = nullptr;
    cap = 0;
  }
  ~PinnedBuf() { release(); }
};

// one rendered, finished diagnostic (include/exspace_b200.h exs_result)
struct ResRec {
  u32 unit, line, col, msg_len;
  u64 msg_off;
  u16 code;
  u8 suppressed, pad[5];
};
static_assert(sizeof(ResRec) == 32, "result record is 32 bytes");

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
  bool keep_records = false;        // also keep the raw records (exs_get_diags / exs_diags_view)
  Coll coll;                        // one batch walked across ranks (exs_set_collective)
  // rendered results of a run (all its batches), in unit order.  A run fills
  // a free set; a caller may lease the current one (zero-copy views that stay
  // valid until it releases them) and later runs then use another
  struct ResultSet {
    PinnedBuf res, text;
    u64 n_res = 0, text_bytes = 0;
    std::vector<u64> unit_first;    // n_units + 1
    bool leased = false;
  };
  std::vector<std::unique_ptr<ResultSet>> sets;
  ResultSet* cur = nullptr;
  std::string static_txt;           // the static message section (start of every text arena)
  u64 static_bytes = 0;
  u32* d_static = nullptr;          // per static message key: (offset, length)
  // results sink: the handle whose result buffers render_results appends to
  // (this one, or the owner of a pipeline), batch by batch in batch order
  Handle* sink = this;
  u64 cur_batch = 0;
  struct Turn {
    std::mutex mu;
    std::condition_variable cv;
    u64 next = 0;
    bool on = false;
    bool abort = false;  // a pipeline failed: the others stop waiting
  } turn;
  // streaming driver (exs_run_units): two host staging slots, two device slots;
  // with pipelines = P > 1, P - 1 more handles (own stream, own buffers)
  // analyse batches concurrently on the same device
  std::vector<std::unique_ptr<Handle>> peers;
  int pipelines = 2;
  u64 batch_cap = 1ull << 30;
  int pack_threads = 0;             // 0: hardware threads (<= 16)
  PinnedBuf stage[2];
  u8* d_slot[2] = {nullptr, nullptr};
  u64 d_slot_cap[2] = {0, 0};
#ifndef EXS_EMU
  cudaStream_t cst = 0;             // host-to-device copies of the next batch
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr};
#endif

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
    dfree(d_static);
    for (int k = 0; k < 2; k++) {
      dfree(d_slot[k]);
#ifndef EXS_EMU
      if (ev_h2d[k]) cudaEventDestroy(ev_h2d[k]);
#endif
    }
#ifndef EXS_EMU
    if (cst) { cudaStreamSynchronize(cst); cudaStreamDestroy(cst); }
#endif
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
    for (u32 s = 0; s < 2; s++) if (walks[s] != NONE) at_add_agg(&dem[walks[s]], 1);
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
// K9: messages and finish_diagnostics (diagnostics.py:116-121), results

// results of a new run: the static message section first
static void static_init(Handle& H) {
  if (!H.d_static) {
    // static messages rendered once per handle, on the host, by the same code
    std::vector<u32> tab(2 * EXS_STATIC_KEYS, 0);
    std::string txt;
    RenderCtx none{};
    for (int k = 0; k < EXS_STATIC_KEYS; k++) {
      Diag d;
      if (!static_diag(k, d)) continue;
      Out cnt{nullptr, 0};
      render_message(none, d, cnt);
      std::string m(cnt.n, '\0');
      Out w{&m[0], 0};
      render_message(none, d, w);
      tab[2 * k] = (u32)txt.size();
      tab[2 * k + 1] = (u32)m.size();
      txt += m;
    }
    H.static_bytes = txt.size();
    H.static_txt = txt;
    H.d_static = dalloc<u32>(2 * EXS_STATIC_KEYS);
    h2d(H.d_static, tab.data(), 8ull * EXS_STATIC_KEYS, H.st);
    sync(H.st);
  }
}
static void results_reset(Handle& H, u64 n_units) {
  static_init(H);
  Handle::ResultSet* rs = nullptr;
  for (auto& x : H.sets)
    if (!x->leased) { rs = x.get(); break; }
  if (!rs) {
    H.sets.emplace_back(new Handle::ResultSet());
    rs = H.sets.back().get();
  }
  H.cur = rs;
  rs->n_res = 0;
  rs->text.ensure(H.static_bytes, 0);
  memcpy(rs->text.p, H.static_txt.data(), H.static_bytes);
  rs->text_bytes = H.static_bytes;
  rs->unit_first.assign(n_units + 1, 0);
}

// Render the ordered records dd[0, nd) of one batch (units unit_base ..),
// finish them and append them to the handle's results.
static void render_results(Handle& H, const Diag* dd, u32 nd, const u8* d_src, u64 n_bytes, u32 n_files,
                           u64 unit_base) {
  cudaStream_t st = H.st;
  if (!nd) {
    Handle& R = *H.sink;
    if (R.turn.on) {
      std::unique_lock<std::mutex> lk(R.turn.mu);
      R.turn.cv.wait(lk, [&] { return R.turn.next == H.cur_batch || R.turn.abort; });
      if (R.turn.abort) throw Err("another pipeline failed");
      R.turn.next++;
      lk.unlock();
      R.turn.cv.notify_all();
    }
    return;
  }
  const RenderCtx RC{d_src, H.L.splice, H.L.arena, H.S.fns, H.S.recs, H.P.nodes, H.L.toks, H.W.inst,
                     (u32)n_bytes};
  const u32* stab = H.d_static;
  u64* len = dalloc<u64>((u64)nd + 1);
  u64* off = dalloc<u64>((u64)nd + 1);
  EXS_TAG("render_len");
  par_for((i64)nd + 1, [=] EXS_HD (i64 i) {
    if (i == nd) { len[i] = 0; return; }
    if (static_key(dd[i]) >= 0) { len[i] = 0; return; }
    Out o{nullptr, 0};
    render_message(RC, dd[i], o);
    len[i] = o.n;
  }, st);
  excl_scan_u64(len, off, (i64)nd + 1, H.sc, st);
  const u64 total = get1(off + nd, st);
  char* txt = dalloc<char>(total + 1);
  EXS_TAG("render_text");
  par_for(nd, [=] EXS_HD (i64 i) {
    if (!len[i]) return;
    Out o{txt + off[i], 0};
    render_message(RC, dd[i], o);
  }, st);
  // appended in batch order: wait for this batch's turn (pipelines), then the
  // offsets of its records are known
  Handle& R = *H.sink;
  std::unique_lock<std::mutex> turn_lock(R.turn.mu, std::defer_lock);
  if (R.turn.on) {
    turn_lock.lock();
    R.turn.cv.wait(turn_lock, [&] { return R.turn.next == H.cur_batch || R.turn.abort; });
    if (R.turn.abort) throw Err("another pipeline failed");
  }
  // message bytes of record i, wherever they live
  Handle::ResultSet& RS = *R.cur;
  const u64 tbase = RS.text_bytes;
  auto msg_of = [=] EXS_HD (u32 i, const char*& p, u32& n, u64& glob) {
    const int k = static_key(dd[i]);
    if (k >= 0) { glob = stab[2 * k]; n = stab[2 * k + 1]; p = nullptr; }
    else { glob = tbase + off[i]; n = (u32)len[i]; p = txt + off[i]; }
  };
  // runs of equal (file, line, col, code): order by message text (then by
  // record order) and drop repeated messages, keeping the first
  u32* ord = dalloc<u32>((u64)nd + 1);
  u8* keep = dalloc<u8>((u64)nd + 1);
  char* stxt = nullptr;  // the static section on the device (for comparisons)
  stxt = dalloc<char>(H.static_bytes + 1);
  h2d(stxt, H.static_txt.data(), H.static_bytes, st);
  const char* sx = stxt;
  EXS_TAG("finish_runs");
  par_for(nd, [=] EXS_HD (i64 i) {
    auto same = [&](i64 a, i64 b) {
      return dd[a].file == dd[b].file && dd[a].line == dd[b].line && dd[a].col == dd[b].col &&
             dd[a].code == dd[b].code;
    };
    if (i > 0 && same(i - 1, i)) return;  // not the head of its run
    i64 e = i + 1;
    while (e < (i64)nd && same(i, e)) e++;
    for (i64 k = i; k < e; k++) ord[k] = (u32)k;
    auto text = [&](u32 r, const char*& p, u32& n) {
      u64 g;
      msg_of(r, p, n, g);
      if (!p) p = sx + g;
    };
    auto less = [&](u32 a, u32 b) {
      const char* pa; const char* pb; u32 na, nb;
      text(a, pa, na); text(b, pb, nb);
      const int c = msg_cmp(pa, na, pb, nb);
      return c ? c < 0 : a < b;
    };
    const i64 n = e - i;
    if (n > 1) {
      // shell sort (runs are short; no scratch)
      for (i64 gap = n / 2; gap > 0; gap /= 2)
        for (i64 k = gap; k < n; k++) {
          const u32 v = ord[i + k];
          i64 j = k;
          while (j >= gap && less(v, ord[i + j - gap])) { ord[i + j] = ord[i + j - gap]; j -= gap; }
          ord[i + j] = v;
        }
    }
    keep[i] = 1;
    for (i64 k = i + 1; k < e; k++) {
      const char* pa; const char* pb; u32 na, nb;
      text(ord[k - 1], pa, na); text(ord[k], pb, nb);
      keep[k] = msg_cmp(pa, na, pb, nb) != 0;
    }
  }, st);
  u32* kidx = dalloc<u32>((u64)nd + 1);
  const u8* kp = keep;
  const u32 nk = select_idx(nd, [=] EXS_HD (u32 k) -> bool { return kp[k] != 0; }, kidx, H.L.cnt, H.sc, st);
  ResRec* rr = dalloc<ResRec>((u64)nk + 1);
  u32* fcnt = dalloc<u32>(2ull * n_files + 1);  // per file: first record, end
  dzero(fcnt, 8ull * n_files + 4, st);
  EXS_TAG("results");
  par_for(nk, [=] EXS_HD (i64 j) {
    const u32 x = ord[kidx[j]];
    const Diag& d = dd[x];
    ResRec r;
    const char* p; u32 n; u64 g;
    msg_of(x, p, n, g);
    r.unit = (u32)(unit_base + d.file); r.line = d.line; r.col = d.col; r.msg_len = n; r.msg_off = g;
    r.code = d.code; r.suppressed = d.suppressed;
    for (int q = 0; q < 5; q++) r.pad[q] = 0;
    rr[j] = r;
  }, st);
  // records are in file order: per-file ranges from the boundaries (no
  // counter shared by all records of a huge unit)
  {
    const ResRec* rc = rr;
    const u64 ub = unit_base;
    par_for(nk, [=] EXS_HD (i64 j) {
      const u32 f = (u32)(rc[j].unit - ub);
      if (j == 0 || rc[j - 1].unit != rc[j].unit) fcnt[2 * f] = (u32)j;
      if (j + 1 == (i64)nk || rc[j + 1].unit != rc[j].unit) fcnt[2 * f + 1] = (u32)j + 1;
    }, st);
  }
  RS.res.ensure((RS.n_res + nk) * sizeof(ResRec), RS.n_res * sizeof(ResRec));
  RS.text.ensure(RS.text_bytes + total, RS.text_bytes);
  std::vector<u32> fc(2ull * n_files);
  d2h(RS.res.p + RS.n_res * sizeof(ResRec), rr, (u64)nk * sizeof(ResRec), st);
  if (total) d2h(RS.text.p + RS.text_bytes, txt, total, st);
  d2h(fc.data(), fcnt, 8ull * n_files, st);
  sync(st);
  for (u32 f = 0; f < n_files; f++) RS.unit_first[unit_base + f + 1] = fc[2 * f + 1] - fc[2 * f];
  RS.n_res += nk;
  RS.text_bytes += total;
  if (R.turn.on) {
    R.turn.next++;
    turn_lock.unlock();
    R.turn.cv.notify_all();
  }
  dfree(len); dfree(off); dfree(txt); dfree(ord); dfree(keep); dfree(stxt); dfree(kidx); dfree(rr); dfree(fcnt);
}

// unit_first: per-unit counts -> first result index per unit
static void results_close(Handle& H) {
  std::vector<u64>& uf = H.cur->unit_first;
  for (u64 u = 0; u + 1 < uf.size(); u++) uf[u + 1] += uf[u];
}

static void run_batch(Handle& H, const u8* d_src, u64 n_bytes, const u64* foff, u32 n_files,
                      const u8* cfg, u64 unit_base) {
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
    if (H.coll.on() && H.coll.rank != 0) {
      // a sharded walk: the replicated front end's diagnostics come from rank 0
      nd0 = 0;
      h2d(H.d_ndiags, &nd0, 4, st);
    }
    // grow the diagnostics buffer and its dedup set, keeping the nd0
    // diagnostics of the earlier stages
    auto regrow = [&](u32 ncap) {
      Diag* ndg = dalloc<Diag>((u64)ncap + n_files);
      if (nd0) d2d(ndg, H.d_diags, sizeof(Diag) * (u64)nd0, st);
      const u32 nmask = pow2_at_least(2ull * ncap) - 1;
      u64* nset = dalloc<u64>((u64)nmask + 1);
      dzero(nset, 8ull * ((u64)nmask + 1), st);
      par_for(nd0, [=] EXS_HD (i64 i) { set_insert(nset, nmask, diag_hash(ndg[i])); }, st);
      dfree(H.d_diags); dfree(H.d_dset);
      H.d_diags = ndg; H.d_dset = nset; H.dmask = nmask; H.cap_diags = ncap; cap_diags = ncap;
      B0.diags = ndg; B0.cap_diags = ncap; B0.dset = nset; B0.dmask = nmask;
    };
    // size it for the walk from the (static) call sites up front: the walks
    // emit at most about one diagnostic per two of them on the measured
    // corpora (C4: 43.7 M from 100 M, both sides walked), and an overflow
    // costs a second walk
    {
      const u64 want = std::min<u64>((u64)nd0 + H.S.NCS / 2 + 65536, 0x7FFFFFFFull);
      if (want > cap_diags && nd0 <= cap_diags) regrow((u32)want);
    }
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
      H.W.coll = H.coll;
      bool ok = run_walk(L, H.P, H.S, H.W, B0, H.sc, st, cap_diags);
      // E1201 of a sharded walk from rank 0 only (every rank holds every instance)
      if (ok && (any_div || H.want_demands)) run_demands(H, any_div && H.coll.rank == 0);
      walk_ovf = get1(H.W.ctr(CNT_OVF), st);
      if (H.coll.on()) walk_ovf = coll_or(H.coll, walk_ovf, st);  // every rank retries together
      (void)ok;
      if (!(walk_ovf & 7)) break;
      if (getenv("EXS_TRACE_UNITS"))
        fprintf(stderr, "[run_batch] walk retry: overflow bits %u (1 instances, 2 diagnostics, 4 log/pending/seeds), "
                "%u diagnostics of %u, %u before the walk, %llu call sites\n", walk_ovf, get1(H.d_ndiags, st),
                cap_diags, nd0, (unsigned long long)H.S.NCS);
      if ((walk_ovf & 2) && !(get1(ovf, st) & 2) && nd0 <= cap_diags) {
        // diagnostics overflowed inside the walk: grow the buffer and its dedup
        // set, keep the diagnostics of the earlier stages, re-run the walk only
        const u32 nd_now = get1(H.d_ndiags, st);
        regrow((u32)std::min<u64>(4ull * std::max(nd_now, cap_diags), 0x7FFFFFFFull));
        dfree(dset_snap);
        dset_snap = dalloc<u64>((u64)H.dmask + 1);
        d2d(dset_snap, H.d_dset, 8ull * ((u64)H.dmask + 1), st);
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
    bool redo = nd > cap_diags || (ovf_h & 2) || (walk_ovf & 2);
    if (H.coll.on()) redo = coll_or(H.coll, redo ? 1u : 0u, st) != 0;
    if (redo) {
      if (getenv("EXS_TRACE_UNITS"))
        fprintf(stderr, "[run_batch] batch retry: %u diagnostics, capacity %u, overflow %u/%u\n", nd, cap_diags,
                ovf_h, walk_ovf);
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
  // a sharded walk: every rank's diagnostic records to every rank (the
  // ordering and finish_diagnostics below drop the repeats)
  if (H.coll.on()) {
    const u32 nl = std::min(get1(H.d_ndiags, st), H.cap_diags + n_files);
    std::vector<u64> sizes;
    u64 total = 0;
    u8* all = coll_allgatherv(H.coll, H.d_diags, sizeof(Diag) * (u64)nl, sizes, total, st);
    const u32 nt = (u32)(total / sizeof(Diag));
    dfree(H.d_diags);
    H.d_diags = reinterpret_cast<Diag*>(all);
    H.cap_diags = std::max(H.cap_diags, nt);
    h2d(H.d_ndiags, &nt, 4, st);
  }
  // order diagnostics by (file, line, col, code string) -- one radix sort of a
  // packed key, or two stable passes when the fields exceed 64 bits
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
        o[0] |= dd[i].file; o[1] |= dd[i].line; o[2] |= dd[i].col; o[3] |= code_rank(dd[i].code);
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
        k[i] = (sf < 64 ? (u64)dd[i].file << sf : 0) | ((u64)dd[i].line << sl) | ((u64)dd[i].col << bk) | code_rank(dd[i].code);
      }, st);
      sort_pairs(k, ix, nd, H.sc, st, std::max(1, bf + bl + bc + bk));
    } else {
      par_for(nd, [=] EXS_HD (i64 i) { ix[i] = (u32)i; k[i] = ((u64)dd[i].col << 16) | code_rank(dd[i].code); }, st);
      sort_pairs(k, ix, nd, H.sc, st, 48);
      par_for(nd, [=] EXS_HD (i64 i) { k[i] = ((u64)dd[ix[i]].file << 32) | dd[ix[i]].line; }, st);
      sort_pairs(k, ix, nd, H.sc, st);
    }
    Diag* out = dalloc<Diag>(nd + 1);
    par_for(nd, [=] EXS_HD (i64 i) { out[i] = dd[ix[i]]; }, st);
    Timer td(st);
    render_results(H, out, nd, d_src, n_bytes, n_files, unit_base);
    H.n_diags_host = 0;
    if (H.keep_records && (u64)nd > H.diags_host_cap) {
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
    if (H.keep_records) {
      H.n_diags_host = nd;
      if (nd) d2h(H.diags, out, sizeof(Diag) * (u64)nd, st);
    }
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
      at_add_agg(&wi[in[i].walk], 1);
      at_add_agg(&we[in[i].walk], in[i].ecnt);
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
  s.ms_wall = s.ms_total;
  s.batches = 1;
#ifndef EXS_EMU
  if (getenv("EXS_TRACE_UNITS")) {
    std::lock_guard<std::mutex> g(g_cache.mu);
    fprintf(stderr, "[cache] hits %llu misses %llu trims %llu oom retries %llu, idle %.1f GiB, live %.1f GiB, peak %.1f GiB\n",
            (unsigned long long)g_cache.hits, (unsigned long long)g_cache.misses, (unsigned long long)g_cache.trims,
            (unsigned long long)g_cache.oom_retries, g_cache.cached / 1073741824.0, g_cache.live_bytes / 1073741824.0,
            g_cache.peak_bytes / 1073741824.0);
  }
#endif
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
  g_cache_bound = getenv("EXS_CACHE_GB") ? (size_t)(atof(getenv("EXS_CACHE_GB")) * 1073741824.0)
                                         : (size_t)(pr.totalGlobalMem / 2);
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
  results_reset(H, n_files);
  run_batch(H, H.d_src_owned, n_bytes, file_off, n_files, file_cfg, 0);
  results_close(H);
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
  results_reset(H, n_files);
  run_batch(H, d_bytes, n_bytes, file_off, n_files, file_cfg, 0);
  results_close(H);
  H.stats.ms_h2d = 0;
  API_END
}

// ---- streaming driver: any number of units in batches of <= batch_cap bytes;
// batch k+1 is packed into page-locked memory and copied to the device while
// batch k is analysed

static void pack_units(const char* const* texts, const uint64_t* lens, u64 u0, u64 u1, const u64* uoff,
                       u8* dst, int nthreads) {
  // byte-balanced ranges over the concatenation of units [u0, u1)
  const u64 total = uoff[u1 - u0];
  const u64 per = (total + nthreads - 1) / std::max(1, nthreads);
  auto work = [=](u64 lo, u64 hi) {
    if (lo >= hi) return;
    // first unit overlapping lo
    u64 a = 0, b = u1 - u0;
    while (b - a > 1) { const u64 m = (a + b) / 2; if (uoff[m] <= lo) a = m; else b = m; }
    for (u64 k = a; k < u1 - u0 && uoff[k] < hi; k++) {
      const u64 s0 = std::max(lo, uoff[k]), s1 = std::min(hi, uoff[k + 1]);
      if (s1 > s0) memcpy(dst + s0, texts[u0 + k] + (s0 - uoff[k]), s1 - s0);
    }
  };
  if (nthreads <= 1 || total < (8u << 20)) { work(0, total); return; }
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; t++) th.emplace_back(work, (u64)t * per, std::min(total, (u64)(t + 1) * per));
  for (auto& t : th) t.join();
}

// device slots come from the stream-ordered pool like every other buffer (a
// plain cudaMalloc would fail while the pool holds the memory of earlier runs)
static void ensure_slot(Handle& H, int k, u64 bytes) {
  if (H.d_slot_cap[k] >= bytes) return;
#ifndef EXS_EMU
  if (H.cst) CK(cudaStreamSynchronize(H.cst));
#endif
  sync(H.st);
  dfree(H.d_slot[k]);
  H.d_slot[k] = dalloc<u8>(bytes);
  H.d_slot_cap[k] = bytes;
  sync(H.st);  // the copy stream uses it next
}

struct BatchPlan {
  u64 u0, u1, bytes;
  std::vector<u64> off;  // unit offsets within the batch (u1 - u0 + 1)
};

static void add_stats(exs_stats& acc, const exs_stats& s) {
  acc.bytes += s.bytes; acc.files += s.files; acc.lines += s.lines; acc.directives += s.directives;
  acc.tokens += s.tokens; acc.views += s.views; acc.view_tokens += s.view_tokens; acc.items += s.items;
  acc.functions += s.functions; acc.structs += s.structs; acc.instances += s.instances;
  acc.edges += s.edges; acc.callsites += s.callsites; acc.levels = std::max(acc.levels, s.levels);
  acc.diagnostics += s.diagnostics; acc.retries += s.retries; acc.gpu_launches += s.gpu_launches;
  acc.ms_lex += s.ms_lex; acc.ms_parse += s.ms_parse; acc.ms_sema += s.ms_sema; acc.ms_walk += s.ms_walk;
  acc.ms_total += s.ms_total; acc.ms_d2h += s.ms_d2h;
}

#ifndef EXS_EMU
// P pipelines on one device: this handle and P - 1 peer handles (own stream,
// own device buffers), each in its own host thread: pack -> copy -> analyse.  The device runs one pipeline's kernels in
// the other's host round trips and low-occupancy phases (sorts, scans, small
// grids); results are appended in batch order (Handle::turn).
static void run_units_pipelined(Handle& H, const char* const* texts, const uint64_t* lens, u64 n_units,
                                const u8* cfg, const std::vector<BatchPlan>& plan, u64 maxb) {
  const int np = std::max(2, H.pipelines);
  while ((int)H.peers.size() < np - 1) {
    H.peers.emplace_back(new Handle());
    Handle& Q = *H.peers.back();
    Q.device = H.device;
    CK(cudaStreamCreateWithFlags(&Q.st, cudaStreamNonBlocking));
  }
  for (int q = 0; q < np - 1; q++) {
    Handle& Q = *H.peers[q];
    Q.want_demands = H.want_demands; Q.split_min = H.split_min; Q.select_flagged_min = H.select_flagged_min;
    Q.diag_sort_two_pass = H.diag_sort_two_pass; Q.keep_records = false;
  }
  const int nthreads = H.pack_threads > 0 ? H.pack_threads
                                          : (int)std::min<unsigned>(8, std::max(1u, std::thread::hardware_concurrency() / 2));
  results_reset(H, n_units);
  {
    std::lock_guard<std::mutex> g(H.turn.mu);
    H.turn.next = 0; H.turn.on = true; H.turn.abort = false;
  }
  std::mutex acc_mu;
  exs_stats acc{};
  float t_stage[4] = {0, 0, 0, 0};
  auto t0 = std::chrono::steady_clock::now();
  static const bool trace = getenv("EXS_TRACE_UNITS") != nullptr;
  auto ms_since = [t0]() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  };
  // batches are claimed from a shared counter (a pipeline that finishes early
  // takes the next one) and a pipeline packs its next batch into its second
  // staging buffer while the device analyses the current one; results are
  // appended in batch order (turn counter)
  std::atomic<size_t> next_batch{0};
  auto worker = [&](Handle& P, int id, std::string& err) {
    try {
      bind_stream(P);
      static_init(P);
      P.sink = &H;
      P.stage[0].ensure(maxb + 64, 0);
      P.stage[1].ensure(maxb + 64, 0);
      ensure_slot(P, 0, maxb + 64);
      double a0 = 0, a1 = 0;
      auto pack = [&](size_t b, int k) {
        const BatchPlan& B = plan[b];
        pack_units(texts, lens, B.u0, B.u1, B.off.data(), P.stage[k].p, nthreads);
        memset(P.stage[k].p + B.bytes, 0, 64);
      };
      size_t b = next_batch.fetch_add(1);
      int k = 0;
      if (b < plan.size()) { a0 = ms_since(); pack(b, k); a1 = ms_since(); }
      while (b < plan.size()) {
        const BatchPlan& B = plan[b];
        h2d(P.d_slot[0], P.stage[k].p, B.bytes + 64, P.st);  // same stream as the analysis
        const size_t nb = next_batch.fetch_add(1);
        std::thread ahead;
        std::string ahead_err;
        double n0 = 0, n1 = 0;
        if (nb < plan.size())
          ahead = std::thread([&, nb, k]() {
            try { n0 = ms_since(); pack(nb, 1 - k); n1 = ms_since(); } catch (const std::exception& e) { ahead_err = e.what(); }
          });
        try {
          P.cur_batch = b;
          run_batch(P, P.d_slot[0], B.bytes, B.off.data(), (u32)(B.u1 - B.u0), cfg + B.u0, B.u0);
        } catch (...) {
          if (ahead.joinable()) ahead.join();
          throw;
        }
        if (ahead.joinable()) ahead.join();
        if (!ahead_err.empty()) throw Err(ahead_err);
        if (trace)
          fprintf(stderr, "[run_units] pipeline %d batch %zu (%.1f MB): packed %.1f..%.1f, analysed by %.1f ms (device %.1f)\n",
                  id, b, B.bytes / 1e6, a0, a1, ms_since(), P.stats.ms_total);
        {
          std::lock_guard<std::mutex> g(acc_mu);
          add_stats(acc, P.stats);
          for (int q = 0; q < 4; q++) t_stage[q] += P.t_stage[q];
        }
        b = nb; k = 1 - k; a0 = n0; a1 = n1;
      }
    } catch (const std::exception& e) {
      err = e.what();
      std::lock_guard<std::mutex> g(H.turn.mu);
      H.turn.abort = true;
      H.turn.cv.notify_all();
    }
  };
  std::vector<std::string> errs(np);
  std::vector<std::thread> others;
  for (int q = 1; q < np; q++) others.emplace_back([&, q]() { worker(*H.peers[q - 1], q, errs[q]); });
  worker(H, 0, errs[0]);
  for (auto& t : others) t.join();
  bind_stream(H);
  for (int q = 0; q < np - 1; q++) H.peers[q]->sink = H.peers[q].get();
  H.sink = &H;
  H.turn.on = false;
  // the first real error (a pipeline that saw another fail reports that)
  const std::string aborted = "another pipeline failed";
  std::string err;
  for (auto& e : errs)
    if (!e.empty() && (err.empty() || err == aborted)) err = e;
  if (!err.empty()) throw Err(err);
  results_close(H);
  acc.batches = plan.size();
  acc.ms_wall = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
  H.stats = acc;
  for (int q = 0; q < 4; q++) H.t_stage[q] = t_stage[q];
}
#endif

static void run_units(Handle& H, const char* const* texts, const uint64_t* lens, u64 n_units, const u8* cfg) {
  if (n_units >= 0xFFFFFFFFull) throw Err("too many units");
  // plan
  std::vector<BatchPlan> plan;
  {
    u64 total = 0;
    for (u64 u = 0; u < n_units; u++) total += lens[u];
    // the first batch's packing and copy are not hidden behind an earlier
    // batch: a smaller first batch starts the device sooner
    const u64 cap0 = total > H.batch_cap ? std::min<u64>(H.batch_cap, std::max<u64>(H.batch_cap / 4, 16ull << 20))
                                         : H.batch_cap;
    BatchPlan cur{0, 0, 0, {0}};
    for (u64 u = 0; u < n_units; u++) {
      const u64 n = lens[u];
      if (n >= (1ull << 31) - 64) throw Err("a unit larger than 2 GiB is outside the contract");
      const u64 cap = plan.empty() ? cap0 : H.batch_cap;
      if (cur.u1 > cur.u0 && (cur.bytes + n > cap || cur.u1 - cur.u0 >= (1u << 26))) {
        plan.push_back(cur);
        cur = BatchPlan{u, u, 0, {0}};
      }
      cur.bytes += n;
      cur.off.push_back(cur.bytes);
      cur.u1 = u + 1;
    }
    if (cur.u1 > cur.u0 || plan.empty()) plan.push_back(cur);
  }
  u64 maxb = 0;
  for (auto& b : plan) maxb = std::max(maxb, b.bytes);
#ifndef EXS_EMU
  if (H.pipelines >= 2 && plan.size() >= 2 && !g_profile && !H.keep_records && !H.coll.on()) {
    run_units_pipelined(H, texts, lens, n_units, cfg, plan, maxb);
    return;
  }
#endif
  const int nslots = plan.size() > 1 ? 2 : 1;
  for (int k = 0; k < nslots; k++) {
    H.stage[k].ensure(maxb + 64, 0);
    ensure_slot(H, k, maxb + 64);
  }
#ifndef EXS_EMU
  if (!H.cst) CK(cudaStreamCreateWithFlags(&H.cst, cudaStreamNonBlocking));
  for (int k = 0; k < 2; k++)
    if (!H.ev_h2d[k]) CK(cudaEventCreateWithFlags(&H.ev_h2d[k], cudaEventDisableTiming));
#endif
  const int nthreads = H.pack_threads > 0 ? H.pack_threads
                                          : (int)std::min<unsigned>(16, std::max(1u, std::thread::hardware_concurrency()));
  const int dev = H.device;
  // pack batch b into slot k and queue its copy (any thread)
  static const bool trace = getenv("EXS_TRACE_UNITS") != nullptr;
  const auto tz = std::chrono::steady_clock::now();
  auto ms_since = [tz]() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tz).count();
  };
  auto prep = [&H, &plan, texts, lens, nthreads, dev, ms_since](size_t b, int k) {
    const BatchPlan& P = plan[b];
    const double a0 = ms_since();
    pack_units(texts, lens, P.u0, P.u1, P.off.data(), H.stage[k].p, nthreads);
    if (trace) fprintf(stderr, "[run_units] batch %zu packed %.1f MB at %.1f..%.1f ms\n", b, P.bytes / 1e6, a0, ms_since());
    memset(H.stage[k].p + P.bytes, 0, 64);
#ifndef EXS_EMU
    CK(cudaSetDevice(dev));
    CK(cudaMemcpyAsync(H.d_slot[k], H.stage[k].p, P.bytes + 64, cudaMemcpyHostToDevice, H.cst));
    CK(cudaEventRecord(H.ev_h2d[k], H.cst));
#else
    (void)dev;
    memcpy(H.d_slot[k], H.stage[k].p, P.bytes + 64);
#endif
  };
  results_reset(H, n_units);
  exs_stats acc{};
  float t_stage[4] = {0, 0, 0, 0};
  auto t0 = std::chrono::steady_clock::now();
  prep(0, 0);
  for (size_t b = 0; b < plan.size(); b++) {
    const int k = (int)(b & 1);
    std::thread next;
    std::string next_err;
    if (b + 1 < plan.size()) {
      next = std::thread([&, b]() {
        try { prep(b + 1, (int)((b + 1) & 1)); } catch (const std::exception& e) { next_err = e.what(); }
      });
    }
    try {
#ifndef EXS_EMU
      CK(cudaStreamWaitEvent(H.st, H.ev_h2d[k], 0));
#endif
      const BatchPlan& P = plan[b];
      const double r0 = ms_since();
      run_batch(H, H.d_slot[k], P.bytes, P.off.data(), (u32)(P.u1 - P.u0), cfg + P.u0, P.u0);
      if (trace) fprintf(stderr, "[run_units] batch %zu analysed at %.1f..%.1f ms (device %.1f ms)\n", b, r0,
                         ms_since(), H.stats.ms_total);
    } catch (...) {
      if (next.joinable()) next.join();
      throw;
    }
    if (next.joinable()) next.join();
    if (!next_err.empty()) throw Err(next_err);
    add_stats(acc, H.stats);
    for (int q = 0; q < 4; q++) t_stage[q] += H.t_stage[q];
  }
  results_close(H);
  acc.batches = plan.size();
  acc.ms_wall = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
  H.stats = acc;
  for (int q = 0; q < 4; q++) H.t_stage[q] = t_stage[q];
}

int exs_set_collective(exs_handle x, int rank, int world, exs_allgather_fn fn, void* ctx) {
  API_TRY
  if (world < 1 || rank < 0 || rank >= world) throw Err("bad rank / world");
  if (world > 1 && !fn) throw Err("a collective needs an all-gather function");
  Handle& H = x->h;
  H.coll.rank = rank;
  H.coll.world = world;
  H.coll.fn = reinterpret_cast<CollFn>(fn);
  H.coll.ctx = ctx;
  API_END
}

int exs_run_units(exs_handle x, const char* const* texts, const uint64_t* lens, uint64_t n_units,
                  const uint8_t* unit_cfg) {
  API_TRY
  Handle& H = x->h;
  bind_stream(H);
#ifndef EXS_EMU
  CK(cudaSetDevice(H.device));
#endif
  run_units(H, texts, lens, n_units, unit_cfg);
  API_END
}

// parallel copy of [src, src + n) to dst (first touch of fresh pages included)
static void copy_threads(void* dst, const void* src, u64 n, int nthreads) {
  if (nthreads <= 1 || n < (4u << 20)) { if (n) memcpy(dst, src, n); return; }
  const u64 per = ((n + nthreads - 1) / nthreads + 4095) & ~4095ull;
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; t++) {
    const u64 lo = (u64)t * per, hi = std::min(n, lo + per);
    if (lo >= hi) break;
    th.emplace_back([=]() { memcpy((u8*)dst + lo, (const u8*)src + lo, hi - lo); });
  }
  for (auto& x : th) x.join();
}

int exs_results_copy(exs_handle x, exs_result* recs, char* text, uint64_t* unit_first) {
  API_TRY
  const Handle& H = x->h;
  const int nt = H.pack_threads > 0 ? H.pack_threads
                                    : (int)std::min<unsigned>(16, std::max(1u, std::thread::hardware_concurrency()));
  if (!H.cur) throw Err("no results: nothing was run");
  const Handle::ResultSet& RS = *H.cur;
  if (recs) copy_threads(recs, RS.res.p, RS.n_res * sizeof(ResRec), nt);
  if (text) copy_threads(text, RS.text.p, RS.text_bytes, nt);
  if (unit_first && !RS.unit_first.empty()) memcpy(unit_first, RS.unit_first.data(), 8 * RS.unit_first.size());
  API_END
}

int exs_results_view(exs_handle x, const exs_result** recs, uint64_t* n, const char** text,
                     uint64_t* text_bytes, const uint64_t** unit_first, uint64_t* n_units) {
  API_TRY
  const Handle& H = x->h;
  if (!H.cur) throw Err("no results: nothing was run");
  const Handle::ResultSet& RS = *H.cur;
  *recs = reinterpret_cast<const exs_result*>(RS.res.p);
  *n = RS.n_res;
  *text = reinterpret_cast<const char*>(RS.text.p);
  *text_bytes = RS.text_bytes;
  *unit_first = RS.unit_first.data();
  *n_units = RS.unit_first.empty() ? 0 : RS.unit_first.size() - 1;
  API_END
}

int exs_results_lease(exs_handle x, uint64_t* lease) {
  API_TRY
  Handle& H = x->h;
  if (!H.cur) throw Err("no results: nothing was run");
  H.cur->leased = true;
  u64 k = 0;
  while (H.sets[k].get() != H.cur) k++;
  *lease = k + 1;
  API_END
}

int exs_results_release(exs_handle x, uint64_t lease) {
  API_TRY
  Handle& H = x->h;
  if (lease == 0 || lease > H.sets.size()) throw Err("unknown results lease");
  H.sets[lease - 1]->leased = false;
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
  else if (key == 2) g_profile = value <= 0 ? 0 : (value >= 2 ? 2 : 1);  // device timing of later runs: 1 named launches, 2 all
#endif
  else if (key == 3) x->h.split_min = value < 4 ? 4u : (u32)value;  // statement-split threshold (tokens)
  else if (key == 4) x->h.select_flagged_min = value < 0 ? 0 : value;  // flag-pass selection threshold
  else if (key == 5) x->h.diag_sort_two_pass = value != 0;  // diagnostic order by two sorts
  else if (key == 6) x->h.keep_records = value != 0;        // keep raw records (exs_get_diags)
  else if (key == 7) x->h.batch_cap = (u64)std::min(2047, std::max(1, value)) << 20;  // batch MiB
  else if (key == 8) x->h.pack_threads = value;               // host packing threads (0 = auto)
  else if (key == 9) x->h.pipelines = value < 2 ? 1 : (value > 4 ? 4 : value);  // concurrent batch pipelines
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
