// exs_common.cuh -- shared types, vocabulary, hashing and parallel primitives
// for the B200 stray-call analyser (sm_100a).
//
// The semantic core (lexer line scanner, parser, evaluator, body walker) is
// written once as __host__ __device__ code -- the paper's own generic pattern
// (PAPER.md: "__host__ __device__ -- Generic programming in Cuda") -- and run
// by the kernels in exs_*.cu.  EXS_EMU builds the same orchestration as plain
// host loops for the developer harness under tests/emu (never shipped, never
// loaded by the package).
#pragma once
#include <cstdint>
#include <cstring>
#include <cstdio>
#include <cstdlib>

#ifndef EXS_EMU
#include <cuda_runtime.h>
#define EXS_HD __host__ __device__
#define EXS_D __device__
#else
#include <cuda_runtime.h>  // types only; no device code is generated or launched
#define EXS_HD __host__
#define EXS_D __host__
#endif

#ifdef EXS_EMU
#define EXS_TAG(name) ((void)0)
#define EXS_FI inline
#define EXS_NOINLINE
#else
// Stack discipline for the recursive walkers (local-memory traffic dominated
// DRAM traffic, profiles/r01_*): keep the frames of the recursive functions
// small by inlining only light steps into them (EXS_FI) and moving heavy,
// non-recursive leaf work (overload selection, dispatch, instantiation) into
// separate functions (EXS_NOINLINE) whose big frames exist only while they run.
#define EXS_FI __forceinline__
#define EXS_NOINLINE __noinline__
#endif

typedef uint8_t u8;
typedef uint16_t u16;
typedef uint32_t u32;
typedef uint64_t u64;
typedef int64_t i64;

#define NONE 0xFFFFFFFFu

// ---------------------------------------------------------------------------
// tokens (reference: syntax/lexer.py:16-20)

enum TokKind : u8 { TK_IDENT = 1, TK_INT, TK_STRING, TK_PUNCT, TK_PRAGMA, TK_EOF };

// punctuator ids in the reference's greedy order (lexer.py:23-43)
enum Punct : u8 {
  P_LLL = 1, P_GGG, P_SCOPE, P_EQ, P_NE, P_AND, P_OR, P_INC,
  P_LBRACE, P_RBRACE, P_LPAREN, P_RPAREN, P_LT, P_GT, P_COMMA, P_SEMI, P_DOT,
  P_BANG, P_ASSIGN, P_COUNT
};

// vocabulary ids for identifiers / string contents / pragma names.
// 1..22 are the parser KEYWORDS (parser.py:8-31).
enum Word : u8 {
  W_NONE = 0,
  W_STRUCT = 1, W_CLASS, W_ENUM, W_TEMPLATE, W_TYPENAME, W_REQUIRES, W_RETURN,
  W_IF, W_ELSE, W_FOR, W_VOID, W_INT, W_BOOL, W_TRUE, W_FALSE, W_CONSTEXPR,
  W_STATIC, W_STATIC_ASSERT, W_HDC, W_HOST, W_DEVICE, W_GLOBAL,  // 22
  W_MAIN, W_CUDA_ARCH, W_HDC_TRAIT, W_STD, W_HST, W_DEV, W_HSTDEV, W_PRINTF,
  W_RELEASE_ASSERT, W_TRAP, W_ABORT, W_CUDASYNC, W_HD_WARNING_DISABLE,
  W_NV_EXEC_CHECK_DISABLE, W_BANG_STR, W_LPAREN_STR, W_COUNT
};
#define W_LAST_KEYWORD W_GLOBAL

struct Tok {
  u32 pos;    // raw byte offset of the token text (pragma: of its NAME word)
  u32 end;    // raw end (exclusive); may include spliced bytes
  u32 line, col;  // reference SrcLoc (1-based, code points)
  u64 hv;     // ident/string/pragma: NameHash of the logical text; int: value
  u8 kind, id, mask, flags;  // mask: bit0 host pass, bit1 device pass
  u32 file;
};
static_assert(sizeof(Tok) == 32, "token record is 32 bytes");
#define TF_INT_OVERFLOW 1
#define TF_HAS_SPLICE 2

// ---------------------------------------------------------------------------
// AST nodes (reference: syntax/nodes.py) -- flat, first-child/next-sibling

enum NodeKind : u8 {
  N_NONE = 0,
  // expressions
  N_INT, N_STR, N_BOOL, N_HDCV, N_ARCH, N_NAME, N_TMP, N_TRAIT, N_MCONST,
  N_CALL, N_MCALL, N_SCALL, N_NOT, N_BIN,
  // types / decl parts
  N_TYPE, N_TPARAM, N_PARAM, N_MVAR,
  // statements
  N_SEXPR, N_SRET, N_SVAR, N_SIF, N_SFOR, N_SLAUNCH,
  // items
  N_FN, N_FNX, N_STRUCT, N_ENUM, N_ASSERT,
};

// N_TYPE.sub: builtin code
enum { BT_NONE = 0, BT_VOID, BT_INT, BT_BOOL, BT_HDC };
// N_BIN.sub
enum { OP_OR = 1, OP_AND, OP_EQ, OP_NE };
// N_FN.n flags
enum {
  FF_H = 1, FF_D = 2, FF_G = 4, FF_CX = 8, FF_STATIC = 16, FF_BODY = 32,
  FF_PRAGMA = 64, FF_MEMBER = 128, FF_HPRED = 256, FF_DPRED = 512,
};
// N_STRUCT.n flags
enum { SF_H = 1, SF_D = 2, SF_G = 4, SF_CX = 8 };
// N_CALL.sub
enum { CALL_PLAIN = 0, CALL_STD = 1 };

struct Node {
  u8 kind, sub;
  u16 n;
  u32 tok;          // main token (global index)
  u32 c0, c1, c2;   // children / misc
  u32 next;         // sibling link
  u64 hv;           // the main token's text hash / int value, copied at parse time:
                    // sema and the walk read names without the 32-byte token record
};
static_assert(sizeof(Node) == 32, "node record is 32 bytes (one sector)");

// ---------------------------------------------------------------------------
// diagnostics (reference: diagnostics.py:15-37)

enum Code : u16 {
  C_E0001 = 1, C_E0002, C_E0101, C_E0102, C_E0103, C_E0104, C_E1001, C_E1002,
  C_E1003, C_E1004, C_W1101, C_W1102, C_E1101, C_E1102, C_E1201, C_E1301,
  C_E1302, C_E1401, C_E1501, C_W1502, C_X9999
};

// Position of a code in the reference's order, which compares the code
// STRINGS (Diagnostic.sort_key, diagnostics.py:73-74): every E code sorts
// before W1101/W1102/W1502, so the enum value is not the order.
EXS_HD inline u32 code_rank(u32 c) {
  // E0001..E1004 keep their values; E1101..E1501 follow; then W1101, W1102, W1502, X9999
  return c <= C_E1004 ? c : (c >= C_E1101 && c <= C_E1501) ? c - 2 : (c == C_W1101 || c == C_W1102) ? c + 7 : c;
}

// message templates; rendered on the GPU by exs_render.cuh (and by
// paper_2309_03912_b200/messages.py for the walk-key renderer)
enum Msg : u16 {
  M_NONE = 0,
  // preprocessor (preprocess.py:177-202) -- a0: text-arena span
  M_PP_EXPECTS_ONE, M_PP_UNKNOWN_MACRO, M_PP_ELSE_NOMATCH, M_PP_SECOND_ELSE,
  M_PP_ENDIF_NOMATCH, M_PP_ERROR, M_PP_UNKNOWN_DIRECTIVE, M_PP_UNTERMINATED,
  // lexer (lexer.py:75,86,116)
  M_LEX_PRAGMA, M_LEX_STRING, M_LEX_CHAR,
  // parser (parser.py) -- see messages.py for argument layouts
  M_P_EXPECTED, M_P_EXPECTED_NAME, M_P_UNKNOWN_PRAGMA, M_P_PRAGMA_FN,
  M_P_REQ_STRUCT, M_P_TPARAM_KIND, M_P_TPARAM_LIMIT, M_P_SPEC_REJECT,
  M_P_SPEC_DUP, M_P_GLOBAL_EXCL, M_P_STRUCT_SPEC, M_P_STRUCT_TPARAM,
  M_P_MEMBER_GLOBAL, M_P_MCONST_DECL, M_P_MCONST_TYPE, M_P_MCONST_STATIC,
  M_P_MCONST_SPEC, M_P_REQ_TEMPLATE, M_P_GLOBAL_VOID, M_P_GLOBAL_MEMBER,
  M_P_MAIN_SPEC, M_P_MAIN_SIG, M_P_FOR_VAR, M_P_PRINTF_FMT, M_P_PRINTF_TEXT,
  M_P_PRINTF_ONE, M_P_PRINTF_COUNT, M_P_ARITY, M_P_HDC_VALUE, M_P_EXPR,
  M_P_TARGS, M_P_DEPTH,
  // sema (sema.py)
  M_S_DUP, M_S_STRUCT_SPEC_MODE, M_S_COND_SPEC_MODE, M_S_UNDEF_NAME,
  M_S_ASSERT_EVAL, M_S_ASSERT_FAIL, M_S_NO_TARGS_BUILTIN, M_S_UNDEF_TYPE,
  M_S_MISSING_TARGS, M_S_TOO_MANY_TARGS, M_S_HDC_MEMBER, M_S_NO_VIABLE,
  M_S_AMBIGUOUS, M_S_EMPTY_SPACES,
  // walk (spacecheck.py)
  M_W_PRED_CONST, M_W_NOT_TYPE, M_W_LAUNCH_DEVICE, M_W_LAUNCH_NONGLOBAL,
  M_W_RECEIVER, M_W_NO_MEMBER, M_W_GLOBAL_CALL, M_W_STRAY, M_W_E1201,
  M_W_SUBST,  // E0101 carrying a SubstFailure text (spacecheck.py:469-470)
  M_X_CONTRACT,
};

// SubstFailure texts (sema.py) used by M_W_SUBST
enum Subst : u16 {
  SF_NONE = 0, SF_NOT_TEMPLATE, SF_NOT_TYPE_NAME, SF_STRUCT_TARGS_HDC, SF_EXPECTED_HDC,
  SF_NOT_HDC_CONST, SF_NO_MEMBERS, SF_NO_MEMBER, SF_ARCH, SF_UNBOUND, SF_IS_TYPE,
  SF_NOT_BOOL_OPERAND, SF_UNRELATED, SF_LOGICAL, SF_NOT_CONST, SF_NO_COMPAT,
  SF_OTHER,
};

// Diagnostic record produced on the GPU.  Arguments are typed per template:
// text spans are (raw pos << 32 | raw len) "span" values, types are
// (name span, targ) pairs, small enums are plain integers.
struct Diag {
  u32 file, line, col;
  u16 code, msg;
  u64 a0, a1, a2;
  u32 a3;
  u8 suppressed, pad0, pad1, pad2;
};
static_assert(sizeof(Diag) == 48, "diag record is 48 bytes");

// ---------------------------------------------------------------------------
// hashing

EXS_HD inline u64 fnv_init() { return 1469598103934665603ull; }
EXS_HD inline u64 fnv_step(u64 h, u8 c) { return (h ^ c) * 1099511628211ull; }

// Name hash of a token's text (identifiers, string contents, pragma names):
// FNV-1a steps over 4-byte little-endian chunks of the text (the last one
// zero-padded), then the length, then a final avalanche.  Every step is a
// bijection of the state, so two different texts of the same length never
// share a hash.  The word-parallel lexer feeds whole chunks from registers
// (four bytes per step); the line lexer streams bytes into the same chunks.
EXS_HD constexpr u64 nh_mix(u64 h, u32 x) { return (h ^ x) * 1099511628211ull; }
EXS_HD constexpr u64 nh_fin(u64 h, u32 len) {
  h = nh_mix(h, len);
  h ^= h >> 33; h *= 0xff51afd7ed558ccdull; h ^= h >> 33;
  return h;
}
// NameHash of a NUL-terminated word at compile time (vocabulary, builtin types)
EXS_HD constexpr u64 name_hash_c(const char* w) {
  u32 n = 0;
  while (w[n]) n++;
  u64 h = 1469598103934665603ull;
  for (u32 q = 0; q < n; q += 4) {
    u32 x = 0;
    for (u32 k = 0; k < 4 && q + k < n; k++) x |= (u32)(u8)w[q + k] << (8 * k);
    h = nh_mix(h, x);
  }
  return nh_fin(h, n);
}
struct NameHash {
  u64 h = 1469598103934665603ull;
  u32 acc = 0, n = 0;
  EXS_HD void step(u8 c) {
    acc |= (u32)c << (8 * (n & 3));
    if ((++n & 3) == 0) { h = nh_mix(h, acc); acc = 0; }
  }
  EXS_HD u64 done() const { return nh_fin((n & 3) ? nh_mix(h, acc) : h, n); }
};
EXS_HD inline u64 mix64(u64 x) {
  x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27; x *= 0x94d049bb133111ebull;
  x ^= x >> 31; return x;
}
EXS_HD inline u64 hcombine(u64 a, u64 b) { return mix64(a * 0x9E3779B97F4A7C15ull + b + 0x632BE59BD9B4E019ull); }

// ---------------------------------------------------------------------------
// atomics (device) / plain ops (emulation)

// body-only __CUDA_ARCH__ switch: device atomics on the GPU,
// plain operations in the host instantiation (used by the EXS_EMU harness only)
#if defined(__CUDA_ARCH__) && !defined(EXS_EMU)
#define EXS_DEV_PATH 1
#else
#define EXS_DEV_PATH 0
#endif
EXS_HD inline u32 at_add(u32* p, u32 v) {
#if EXS_DEV_PATH
  return atomicAdd(p, v);
#else
  u32 o = *p; *p = o + v; return o;
#endif
}
// Warp-aggregated "allocate one slot" on a shared counter: the lanes that are
// active together issue a single atomicAdd (the counters of the walk are hit
// by every thread: instance ids, creation log, pending list, diagnostics).
EXS_HD inline u32 at_inc_agg(u32* p) {
#if EXS_DEV_PATH
  u32 mask = __activemask();
  u32 lane = threadIdx.x & 31;
  // group lanes by counter address (different counters may be in flight)
  u32 peers = __match_any_sync(mask, (unsigned long long)p);
  u32 leader = __ffs(peers) - 1;
  u32 base = 0;
  if (lane == leader) base = atomicAdd(p, (u32)__popc(peers));
  base = __shfl_sync(peers, base, leader);
  return base + __popc(peers & ((1u << lane) - 1));
#else
  u32 o = *p; *p = o + 1; return o;
#endif
}
// Warp-aggregated add: the active lanes that add to the same counter issue
// one atomicAdd of their sum (per-walk statistics: every instance of a huge
// unit adds to the same two counters)
EXS_HD inline void at_add_agg(u32* p, u32 v) {
#if EXS_DEV_PATH
  const u32 mask = __activemask();
  const u32 peers = __match_any_sync(mask, (unsigned long long)p);
  const u32 sum = __reduce_add_sync(peers, v);
  if ((threadIdx.x & 31) == (u32)(__ffs(peers) - 1) && sum) atomicAdd(p, sum);
#else
  *p += v;
#endif
}
// Warp-aggregated max into one counter (all active lanes name the same p)
EXS_HD inline void at_max_agg(u32* p, u32 v) {
#if EXS_DEV_PATH
  const u32 mask = __activemask();
  const u32 m = __reduce_max_sync(mask, v);
  if ((threadIdx.x & 31) == (u32)(__ffs(mask) - 1) && m) atomicMax(p, m);
#else
  if (v > *p) *p = v;
#endif
}
EXS_HD inline u32 at_min(u32* p, u32 v) {
#if EXS_DEV_PATH
  return atomicMin(p, v);
#else
  u32 o = *p; if (v < o) *p = v; return o;
#endif
}
EXS_HD inline unsigned long long at_min64(unsigned long long* p, unsigned long long v) {
#if EXS_DEV_PATH
  return atomicMin(p, v);
#else
  auto o = *p; if (v < o) *p = v; return o;
#endif
}
EXS_HD inline u32 at_or(u32* p, u32 v) {
#if EXS_DEV_PATH
  return atomicOr(p, v);
#else
  u32 o = *p; *p = o | v; return o;
#endif
}
EXS_HD inline u32 at_cas(u32* p, u32 c, u32 v) {
#if EXS_DEV_PATH
  return atomicCAS(p, c, v);
#else
  u32 o = *p; if (o == c) *p = v; return o;
#endif
}
EXS_HD inline unsigned long long at_cas64(unsigned long long* p, unsigned long long c, unsigned long long v) {
#if EXS_DEV_PATH
  return atomicCAS(p, c, v);
#else
  auto o = *p; if (o == c) *p = v; return o;
#endif
}
EXS_HD inline u32 ld_volatile(const u32* p) { return *(volatile const u32*)p; }
EXS_HD inline void fence_gpu() {
#if EXS_DEV_PATH
  __threadfence();
#endif
}

// ---------------------------------------------------------------------------
// small helpers

EXS_HD inline bool is_digit(u8 c) { return c >= '0' && c <= '9'; }
EXS_HD inline bool is_alpha(u8 c) { return (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z'); }
EXS_HD inline bool is_ident_start(u8 c) { return is_alpha(c) || c == '_'; }
EXS_HD inline bool is_ident_char(u8 c) { return is_alpha(c) || is_digit(c) || c == '_'; }
// Python str.isspace() over ASCII (used by str.strip/split in preprocess.py:164,169)
EXS_HD inline bool is_pyspace(u8 c) { return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f); }
EXS_HD inline bool is_cont_byte(u8 c) { return (c & 0xC0) == 0x80; }

// file configuration byte
enum {
  CFG_MODE_MASK = 7,      // 0 classic 1 fidelity 2 sound 3 proposal1 4 proposal2
  CFG_PLAIN = 8, CFG_RELAXED = 16, CFG_ERASE = 32, CFG_FUND = 64,
};
enum { MODE_CLASSIC = 0, MODE_FIDELITY, MODE_SOUND, MODE_P1, MODE_P2 };
