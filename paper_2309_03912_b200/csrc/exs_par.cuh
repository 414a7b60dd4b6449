// exs_par.cuh -- parallel primitives used by the pipeline driver.
// Device build: grid-stride kernels + CUB.  EXS_EMU: sequential host loops.
#pragma once
#include "exs_common.cuh"
#include <vector>
#include <algorithm>
#include <stdexcept>
#include <string>

// select_idx flag-pass threshold default (both builds)
#ifndef EXS_SELECT_FLAGGED_MIN
#define EXS_SELECT_FLAGGED_MIN (1ll << 22)
#endif
#ifndef EXS_EMU
#include <cub/cub.cuh>
#include <nvtx3/nvToolsExt.h>
#endif

namespace exs {

struct Err : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#ifndef EXS_EMU
#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e__ = (x);                                                           \
    if (e__ != cudaSuccess)                                                          \
      throw exs::Err(std::string("CUDA error ") + cudaGetErrorString(e__) + " at " + \
                     __FILE__ + ":" + std::to_string(__LINE__));                     \
  } while (0)
#else
#define CK(x) (void)0
#endif

// ----------------------------------------------------------------- memory
#ifndef EXS_EMU
extern thread_local cudaStream_t g_alloc_stream;
#endif
#ifndef EXS_EMU
// Size-exact block cache over the stream-ordered pool: a repeated batch shape
// (the steady state of a corpus service) allocates nothing.  All work is on
// one stream per handle, so a block freed in stream order is safe to reuse.
void* cache_alloc(size_t bytes);
void cache_free(void* p);
#endif
template <class T>
T* dalloc(size_t n) {
  if (n == 0) n = 1;
  void* p = nullptr;
#ifndef EXS_EMU
  p = cache_alloc(n * sizeof(T));
#else
  p = calloc(n, sizeof(T));
  if (!p) throw Err("out of host memory");
#endif
  return (T*)p;
}
inline void dfree(void* p) {
  if (!p) return;
#ifndef EXS_EMU
  cache_free(p);
#else
  free(p);
#endif
}
inline void dzero(void* p, size_t bytes, cudaStream_t s) {
#ifndef EXS_EMU
  CK(cudaMemsetAsync(p, 0, bytes, s));
#else
  (void)s;
  memset(p, 0, bytes);
#endif
}
inline void dfill_ff(void* p, size_t bytes, cudaStream_t s) {
#ifndef EXS_EMU
  CK(cudaMemsetAsync(p, 0xFF, bytes, s));
#else
  (void)s;
  memset(p, 0xFF, bytes);
#endif
}
inline void h2d(void* d, const void* h, size_t bytes, cudaStream_t s) {
#ifndef EXS_EMU
  CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s));
#else
  (void)s;
  memcpy(d, h, bytes);
#endif
}
inline void d2h(void* h, const void* d, size_t bytes, cudaStream_t s) {
#ifndef EXS_EMU
  CK(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s));
#else
  (void)s;
  memcpy(h, d, bytes);
#endif
}
inline void d2d(void* d, const void* s_, size_t bytes, cudaStream_t s) {
#ifndef EXS_EMU
  CK(cudaMemcpyAsync(d, s_, bytes, cudaMemcpyDeviceToDevice, s));
#else
  (void)s;
  memcpy(d, s_, bytes);
#endif
}
inline void sync(cudaStream_t s) {
#ifndef EXS_EMU
  CK(cudaStreamSynchronize(s));
#else
  (void)s;
#endif
}
template <class T>
T get1(const T* d, cudaStream_t s) {
  T v;
  d2h(&v, d, sizeof(T), s);
  sync(s);
  return v;
}

// ------------------------------------------------------------------ for
#ifndef EXS_EMU
template <class F>
__global__ void __launch_bounds__(256) k_for(F f, i64 n) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) f(i);
}
// latency-bound walkers: cap registers so enough warps fit per SM
// (EXS_WALK_MINB blocks of 128 threads: 8 -> 64 regs, 6 -> 80, 4 -> 128)
#ifndef EXS_WALK_MINB
#define EXS_WALK_MINB 8  // C2 1 GB after the shape sort: 16/12/8/4 -> 76.3/73.4/72.5/74.6 us/MB walk
#endif
template <class F>
__global__ void __launch_bounds__(128, EXS_WALK_MINB) k_for_walk(F f, i64 n) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) f(i);
}
// the recursive parser: its per-thread state lives in local memory, so the
// resident thread count sets the L1/L2 footprint of that state
#ifndef EXS_PARSE_MINB
#define EXS_PARSE_MINB 6  // C2 1 GB: parse_items 6.3 ms at 6 (80 registers), 6.8 at 8; 8 beat 16, 4, 2
#endif
template <class F>
__global__ void __launch_bounds__(128, EXS_PARSE_MINB) k_for_parse(F f, i64 n) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) f(i);
}
extern int g_sm_count;
extern thread_local u64 g_launches;  // per host thread (pipelines run on several)
// optional per-launch device timing (EXS_PROFILE=1): (site, start, stop) events
struct ProfRec { const char* fn; int line; cudaEvent_t a, b; };
extern int g_profile;  // 0 off, 1 named launches (EXS_TAG), 2 every launch and timeline mark
extern std::vector<ProfRec> g_prof;
cudaEvent_t prof_event();  // from a reused pool (no create/destroy per launch)
extern thread_local const char* g_tag;  // name of the next launch (EXS_TAG)
// select_idx switches to a flag pass + DeviceSelect::Flagged at this many indices
// (set per run from the handle: exs_set_option key 4)
extern thread_local i64 g_select_flagged_min;
#define EXS_TAG(name) (::exs::g_tag = (name))
#endif

// threads of one full par_for grid (one index per thread): kernels whose work
// count is on the device loop over it in strides of this, 256-lane groups
// (t >> 8) taking the heavy items
#ifndef EXS_EMU
inline i64 grid_threads() { return (i64)g_sm_count * 16 * 256; }
#else
inline i64 grid_threads() { return 256; }
#endif

template <class F>
void par_for(i64 n, F f, cudaStream_t s, int block = 256, const char* fn = __builtin_FUNCTION(),
             int line = __builtin_LINE()) {
  if (n <= 0) return;
#ifndef EXS_EMU
  i64 want = (n + block - 1) / block;
  i64 cap = (i64)g_sm_count * 16;
  int grid = (int)(want < cap ? want : cap);
  ProfRec pr{g_tag ? g_tag : fn, g_tag ? 0 : line, nullptr, nullptr};
  g_tag = nullptr;
  const bool timed = g_profile > 1 || (g_profile && pr.line == 0);
  if (timed) {
    pr.a = prof_event(); pr.b = prof_event();
    cudaEventRecord(pr.a, s);
  }
  if (pr.line == 0) nvtxRangePushA(pr.fn);
  k_for<<<grid, block, 0, s>>>(f, n);
  if (pr.line == 0) nvtxRangePop();
  CK(cudaGetLastError());
  if (timed) { cudaEventRecord(pr.b, s); g_prof.push_back(pr); }
  g_launches++;
#else
  (void)fn; (void)line;
  (void)s; (void)block;
  for (i64 i = 0; i < n; i++) f(i);
#endif
}

// launch for the heavy walker kernels (128 threads, register-capped)
template <class F>
void par_for_walk(i64 n, F f, cudaStream_t s, const char* fn = __builtin_FUNCTION(),
                  int line = __builtin_LINE()) {
  if (n <= 0) return;
#ifndef EXS_EMU
  i64 want = (n + 127) / 128;
  i64 cap = (i64)g_sm_count * 64;
  int grid = (int)(want < cap ? want : cap);
  ProfRec pr{g_tag ? g_tag : fn, g_tag ? 0 : line, nullptr, nullptr};
  g_tag = nullptr;
  const bool timed = g_profile > 1 || (g_profile && pr.line == 0);
  if (timed) {
    pr.a = prof_event(); pr.b = prof_event();
    cudaEventRecord(pr.a, s);
  }
  if (pr.line == 0) nvtxRangePushA(pr.fn);  // named launches are NVTX ranges (ncu --nvtx-include)
#ifdef EXS_WALK_CARVEOUT
  static bool carve = false;  // per kernel instance: prefer L1 over shared memory
  if (!carve) {
    CK(cudaFuncSetAttribute(k_for_walk<F>, cudaFuncAttributePreferredSharedMemoryCarveout, EXS_WALK_CARVEOUT));
    carve = true;
  }
#endif
  k_for_walk<<<grid, 128, 0, s>>>(f, n);
  if (pr.line == 0) nvtxRangePop();
  CK(cudaGetLastError());
  if (timed) { cudaEventRecord(pr.b, s); g_prof.push_back(pr); }
  g_launches++;
#else
  (void)s; (void)fn; (void)line;
  for (i64 i = 0; i < n; i++) f(i);
#endif
}

template <class F>
void par_for_parse(i64 n, F f, cudaStream_t s, const char* fn = __builtin_FUNCTION(),
                   int line = __builtin_LINE()) {
  if (n <= 0) return;
#ifndef EXS_EMU
  i64 want = (n + 127) / 128;
  i64 cap = (i64)g_sm_count * EXS_PARSE_MINB * 4;
  int grid = (int)(want < cap ? want : cap);
  ProfRec pr{g_tag ? g_tag : fn, g_tag ? 0 : line, nullptr, nullptr};
  g_tag = nullptr;
  const bool timed = g_profile > 1 || (g_profile && pr.line == 0);
  if (timed) {
    pr.a = prof_event(); pr.b = prof_event();
    cudaEventRecord(pr.a, s);
  }
  if (pr.line == 0) nvtxRangePushA(pr.fn);
  k_for_parse<<<grid, 128, 0, s>>>(f, n);
  if (pr.line == 0) nvtxRangePop();
  CK(cudaGetLastError());
  if (timed) { cudaEventRecord(pr.b, s); g_prof.push_back(pr); }
  g_launches++;
#else
  (void)s; (void)fn; (void)line;
  for (i64 i = 0; i < n; i++) f(i);
#endif
}

// profiling marks on the stream timeline: the interval between consecutive
// marks includes host-side gaps (allocation, synchronisation, launch latency)
inline void prof_mark(cudaStream_t s, const char* fn = __builtin_FUNCTION(), int line = __builtin_LINE()) {
#ifndef EXS_EMU
  if (g_profile < 2) return;
  ProfRec pr{fn, -line, nullptr, nullptr};
  pr.a = prof_event();
  cudaEventRecord(pr.a, s);
  g_prof.push_back(pr);
#else
  (void)s; (void)fn; (void)line;
#endif
}

// ------------------------------------------------------------ scratch
struct Scratch {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes) {
    if (bytes > cap) {
      dfree(p);
      cap = bytes + (bytes >> 2) + 1024;
      p = dalloc<u8>(cap);
    }
    return p;
  }
  ~Scratch() { dfree(p); }
};

// exclusive scan of u32 in place-able; returns nothing (total = last+count)
inline void excl_scan_u32(const u32* in, u32* out, i64 n, Scratch& sc, cudaStream_t s) {
  if (n <= 0) return;
#ifndef EXS_EMU
  size_t tb = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, (int)n, s));
  CK(cub::DeviceScan::ExclusiveSum(sc.get(tb), tb, in, out, (int)n, s));
  g_launches += 2;
#else
  (void)sc; (void)s;
  u32 acc = 0;
  for (i64 i = 0; i < n; i++) { u32 v = in[i]; out[i] = acc; acc += v; }
#endif
}

inline void excl_scan_u64(const u64* in, u64* out, i64 n, Scratch& sc, cudaStream_t s) {
  if (n <= 0) return;
#ifndef EXS_EMU
  size_t tb = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, (int)n, s));
  CK(cub::DeviceScan::ExclusiveSum(sc.get(tb), tb, in, out, (int)n, s));
  g_launches += 2;
#else
  (void)sc; (void)s;
  u64 acc = 0;
  for (i64 i = 0; i < n; i++) { u64 v = in[i]; out[i] = acc; acc += v; }
#endif
}

template <class T, class Op>
void incl_scan(const T* in, T* out, i64 n, Op op, Scratch& sc, cudaStream_t s) {
  if (n <= 0) return;
#ifndef EXS_EMU
  size_t tb = 0;
  CK(cub::DeviceScan::InclusiveScan(nullptr, tb, in, out, op, (int)n, s));
  CK(cub::DeviceScan::InclusiveScan(sc.get(tb), tb, in, out, op, (int)n, s));
  g_launches += 2;
#else
  (void)sc; (void)s;
  T acc = in[0];
  out[0] = acc;
  for (i64 i = 1; i < n; i++) { acc = op(acc, in[i]); out[i] = acc; }
#endif
}

// inclusive scan of f(0), f(1), ..., f(n-1): the input is computed inside the
// scan (no array written and read back)
template <class T, class F, class Op>
void incl_scan_fn(F f, T* out, i64 n, Op op, Scratch& sc, cudaStream_t s) {
  if (n <= 0) return;
#ifndef EXS_EMU
  cub::CountingInputIterator<u32> c(0);
  cub::TransformInputIterator<T, F, cub::CountingInputIterator<u32>> it(c, f);
  size_t tb = 0;
  CK(cub::DeviceScan::InclusiveScan(nullptr, tb, it, out, op, (int)n, s));
  CK(cub::DeviceScan::InclusiveScan(sc.get(tb), tb, it, out, op, (int)n, s));
  g_launches += 2;
#else
  (void)sc; (void)s;
  T acc = f(0);
  out[0] = acc;
  for (i64 i = 1; i < n; i++) { acc = op(acc, f((u32)i)); out[i] = acc; }
#endif
}

// indices i in [0,n) with pred(i) -> out (ordered); returns count
template <class P>
u32 select_idx(i64 n, P pred, u32* out, u32* d_count, Scratch& sc, cudaStream_t s) {
  if (n <= 0) return 0;
#ifndef EXS_EMU
  cub::CountingInputIterator<u32> it(0);
  size_t tb = 0;
  if (n >= g_select_flagged_min) {
    // large selections: the predicate runs once in a coalesced pass (one
    // thread per index, 1-byte flag out) and the compaction reads only the
    // flags; inside DeviceSelect::If each thread evaluates a run of
    // consecutive indices, so a predicate that gathers strides its loads
    u8* fl = dalloc<u8>((size_t)n);
    par_for(n, [=] EXS_HD (i64 i) { fl[i] = pred((u32)i) ? 1 : 0; }, s, 256, "select_flags", 1);
    CK(cub::DeviceSelect::Flagged(nullptr, tb, it, fl, out, d_count, (int)n, s));
    CK(cub::DeviceSelect::Flagged(sc.get(tb), tb, it, fl, out, d_count, (int)n, s));
    g_launches += 2;
    const u32 c = get1(d_count, s);
    dfree(fl);
    return c;
  }
  CK(cub::DeviceSelect::If(nullptr, tb, it, out, d_count, (int)n, pred, s));
  CK(cub::DeviceSelect::If(sc.get(tb), tb, it, out, d_count, (int)n, pred, s));
  g_launches += 2;
  return get1(d_count, s);
#else
  (void)d_count; (void)sc; (void)s;
  u32 c = 0;
  for (i64 i = 0; i < n; i++)
    if (pred((u32)i)) out[c++] = (u32)i;
  return c;
#endif
}

// stable sort of (u64 or u32 key, u32 value) pairs; results written back in place
template <class K>
void sort_pairs(K* keys, u32* vals, i64 n, Scratch& sc, cudaStream_t s, int end_bit = 8 * sizeof(K)) {
  if (n <= 1) return;
#ifndef EXS_EMU
  K* k2 = dalloc<K>(n);
  u32* v2 = dalloc<u32>(n);
  // double-buffered: the passes ping-pong between the two buffers and the
  // result is copied back only when it ends in the scratch pair
  cub::DoubleBuffer<K> dk(keys, k2);
  cub::DoubleBuffer<u32> dv(vals, v2);
  size_t tb = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, (int)n, 0, end_bit, s));
  CK(cub::DeviceRadixSort::SortPairs(sc.get(tb), tb, dk, dv, (int)n, 0, end_bit, s));
  if (dk.Current() != keys) CK(cudaMemcpyAsync(keys, dk.Current(), n * sizeof(K), cudaMemcpyDeviceToDevice, s));
  if (dv.Current() != vals) CK(cudaMemcpyAsync(vals, dv.Current(), n * 4, cudaMemcpyDeviceToDevice, s));
  dfree(k2);  // reused in stream order (cache_alloc)
  dfree(v2);
  g_launches += 2;
#else
  (void)sc; (void)s;
  // like CUB, order by bits [0, end_bit) only: a key with higher bits set
  // sorts by its truncated value here too, so the emulation catches it
  const u64 m = end_bit >= 64 ? ~0ull : ((1ull << end_bit) - 1);
  std::vector<std::pair<u64, u32>> v(n);
  static_assert(sizeof(K) <= 8, "key type");
  for (i64 i = 0; i < n; i++) v[i] = {keys[i], vals[i]};
  std::stable_sort(v.begin(), v.end(), [m](auto& a, auto& b) { return (a.first & m) < (b.first & m); });
  for (i64 i = 0; i < n; i++) { keys[i] = (K)v[i].first; vals[i] = v[i].second; }
#endif
}

}  // namespace exs
