/* exspace_b200.h -- C ABI of the B200 stray-call analyser.
 *
 * Drop-in boundary for the reference's hot path.  The reference has no FFI:
 * its boundary is the Python API
 *     exspace.spacecheck.analyze(text, path, profile, mode, cfg)      spacecheck.py:687-739
 *     exspace.spacecheck.check_unit(text, path, profile, mode, cfg)   spacecheck.py:742-750
 * applied one unit at a time (cli.py:82-91, corpus.py:123-175).  This ABI is
 * the batch form of that call: one exs_run() analyses many units; the
 * Python mirror (paper_2309_03912_b200.exspace) rebuilds Diagnostic objects,
 * messages and ordering exactly as the reference does.
 * for the ctypes binding the reference-side shim uses.
 *
 * Plain pointers and sizes only; no torch types.  All entry points return 0
 * on success and a negative code on error (exs_last_error() has the text);
 * they never abort the process.
 */
#ifndef EXSPACE_B200_H
#define EXSPACE_B200_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct exs_handle_s* exs_handle;

/* per-unit configuration byte (replaces CompileProfile/Mode/TraitConfig,
 * preprocess.py:46-63, spacecheck.py:53-58, sema.py:54-62) */
#define EXS_MODE_CLASSIC 0
#define EXS_MODE_FIDELITY 1
#define EXS_MODE_SOUND 2
#define EXS_MODE_PROPOSAL1 3
#define EXS_MODE_PROPOSAL2 4
#define EXS_CFG_PLAIN 8        /* CompileProfile(compiler="plain")      */
#define EXS_CFG_RELAXED 16     /* relaxed_constexpr=True                */
#define EXS_CFG_ERASE 32       /* erase_specifiers=True                 */
#define EXS_CFG_FUND_HSTDEV 64 /* TraitConfig(fundamentals_hstdev=True) */

/* One diagnostic (diagnostics.py:56-62).  code: 1=E0001 .. 20=W1502, 21 =
 * out-of-contract marker.  msg + a0..a3: message template and arguments
 * (spans are raw-byte (pos<<32 | len) into the batch; bit 63 marks the
 * directive-text arena). */
typedef struct {
  uint32_t file, line, col;
  uint16_t code, msg;
  uint64_t a0, a1, a2;
  uint32_t a3;
  uint8_t suppressed, pad0, pad1, pad2;
} exs_diag;

typedef struct {
  uint64_t bytes, files, lines, directives, tokens, views, view_tokens, items;
  uint64_t functions, structs, instances, edges, callsites, levels, diagnostics;
  uint64_t retries, gpu_launches;
  float ms_lex, ms_parse, ms_sema, ms_walk, ms_total, ms_h2d, ms_d2h;
  float ms_wall;      /* exs_run_units: host wall time of the whole call     */
  uint32_t batches;   /* exs_run_units: batches the units were analysed in   */
} exs_stats;

/* per (file, pass) preprocessing / lexing status, pass 0 host, 1 device */
typedef struct {
  uint32_t pp_line; /* 0 = no E0002 */
  uint16_t pp_msg, exists;
  uint32_t lex_line, lex_col; /* 0 = no lexical error */
  uint16_t lex_msg, pad;
  uint32_t eof_line, eof_col, view, parse_failed;
} exs_pass_status;

/* a token record (lexer.py:16-20): kind 1 ident 2 int 3 string 4 punct 5 pragma */
typedef struct {
  uint32_t pos, end, line, col;
  uint64_t hv;
  uint8_t kind, id, mask, flags;
  uint32_t file;
} exs_token;

/* per walk (2*file + pass) counts, as exposed by Analysis.walks */
typedef struct {
  uint32_t instances, edges, demands, exists;
} exs_walk_stats;

/* description of a declaration or instance (for E1201 display names) */
typedef struct {
  uint64_t name, owner, otype;  /* spans; 0 = none */
  uint8_t otarg, nb, pad[6];
  uint64_t bname[2], bval[2];   /* binding names (spans) and values (type spans) */
  uint8_t bkind[2], bvx[2], pad2[4]; /* bkind 1 type 2 hdc; bvx: type targ / hdc */
} exs_desc;

/* ---- walk materialisation: the arrays behind Analysis.walks[side].instances /
 * .demands / .edges (spacecheck.py:183-221,239-346,585).  All refer to the last
 * run on the handle; a host renders the reference's canonical keys from them. */

/* one function declaration (sema.py FunctionDecl; order = _all_decls order) */
typedef struct {
  uint32_t node, view, rec, order;  /* FN node; struct record (0xFFFFFFFF free) */
  uint32_t ncalls, flags;           /* call-site slots of an instance's edges; 1 DUP 2 OWNER 4 MEMBER */
} exs_decl;

/* one struct declaration */
typedef struct {
  uint32_t node, view;
} exs_struct;

/* a value bound in an instance key: k 1 = type (struct record rec, or builtin
 * bt 1 void 2 int 3 bool 4 HDC; targ 1..3 = HDC argument Hst/Dev/HstDev),
 * k 2 = HDC value (x = 1 Hst, 2 Dev, 3 HstDev), k 0 = none */
typedef struct {
  uint8_t k, targ, bt, pad;
  uint32_t rec;
  uint64_t x;
} exs_val;

/* one instance (spacecheck.py Instance): creating decl, walk (2*file + pass),
 * side (0 host 1 device), first-creation token, bindings and owner type,
 * legal edges: slots [ebase, ebase + decl.ncalls) of the edge array;
 * spaces = the instance's execution spaces, bits 1 host 2 device 4 global
 * (spacecheck.py Instance.spaces, GLOBAL = {__global__}) */
typedef struct {
  uint32_t decl, walk, side, at;
  uint32_t ebase, ecnt, flags, spaces;
  uint64_t ckey;                    /* creation order (level, parent rank, statement, ordinal) */
  exs_val tb, hb, ot;
} exs_inst;

/* AST node (32 bytes, csrc/exs_common.cuh Node) */
typedef struct {
  uint8_t kind, sub;
  uint16_t n;
  uint32_t tok, c0, c1, c2, next;
  uint64_t hv;
} exs_node;

int exs_get_decls(exs_handle h, exs_decl* out, uint64_t cap, uint64_t* n);
int exs_get_structs(exs_handle h, exs_struct* out, uint64_t cap, uint64_t* n);
int exs_get_instances(exs_handle h, exs_inst* out, uint64_t cap, uint64_t* n);
int exs_get_edges(exs_handle h, uint32_t* out, uint64_t cap, uint64_t* n);   /* callee ids, 0xFFFFFFFF empty */
int exs_get_nodes(exs_handle h, exs_node* out, uint64_t cap, uint64_t* n);
int exs_get_token_range(exs_handle h, uint64_t first, uint64_t count, exs_token* out);

int exs_create(int device, exs_handle* out);
int exs_destroy(exs_handle h);
const char* exs_last_error(void);

/* Analyse a batch of units held in HOST memory (copied to HBM inside). */
int exs_run(exs_handle h, const uint8_t* bytes, uint64_t n_bytes, const uint64_t* file_off,
            uint32_t n_files, const uint8_t* file_cfg);
/* Same with the bytes already in device memory (d_bytes is not modified). */
int exs_run_device(exs_handle h, const uint8_t* d_bytes, uint64_t n_bytes,
                   const uint64_t* file_off, uint32_t n_files, const uint8_t* file_cfg);

/* Analyse n_units units given as (text, length) pairs in HOST memory -- the
 * reference's analyze(text, path, profile, mode, cfg) (spacecheck.py:687-739)
 * over a corpus (corpus.py:163-175, cli.py:82-91), unit_cfg[u] the
 * configuration byte of unit u.  Any total size: units are cut into batches
 * of <= the batch capacity (option 7); batch k+1 is packed into page-locked
 * memory and copied to the device while batch k is analysed.  One unit must
 * be smaller than 2 GiB.  Results: exs_results_view. */
int exs_run_units(exs_handle h, const char* const* texts, const uint64_t* lens, uint64_t n_units,
                  const uint8_t* unit_cfg);

/* One finished diagnostic (diagnostics.py:40-62 Diagnostic): unit index,
 * 1-based line and column, code (1=E0001 .. 20=W1502, 21 = out-of-contract
 * marker X9999), suppressed flag, and its message: msg_len bytes of UTF-8
 * (surrogateescape for invalid input bytes) at text + msg_off. */
typedef struct {
  uint32_t unit, line, col, msg_len;
  uint64_t msg_off;
  uint16_t code;
  uint8_t suppressed, pad[5];
} exs_result;

/* Results of the last run (exs_run_units, exs_run or exs_run_device): the
 * ordered, de-duplicated diagnostics of every unit (finish_diagnostics,
 * diagnostics.py:116-121: unit, then (line, col, code, message)), suppressed
 * ones included.  Unit u owns records [unit_first[u], unit_first[u+1]).  All
 * pointers are owned by the handle (page-locked) and valid until its next
 * run or exs_destroy. */
int exs_results_view(exs_handle h, const exs_result** recs, uint64_t* n, const char** text,
                     uint64_t* text_bytes, const uint64_t** unit_first, uint64_t* n_units);

/* Keep the current results: their buffers are not reused by later runs (which
 * fill another set) until exs_results_release(lease); the views of
 * exs_results_view stay valid that long.  For zero-copy consumers. */
int exs_results_lease(exs_handle h, uint64_t* lease);
int exs_results_release(exs_handle h, uint64_t lease);

/* Copy the results of the last run into caller memory (sizes from
 * exs_results_view; any pointer may be null), with several host threads. */
int exs_results_copy(exs_handle h, exs_result* recs, char* text, uint64_t* unit_first);

/* One batch walked across ranks (one huge unit, C4): every
 * rank runs the front end on the same batch, walks its share of every level's
 * work items, and the ranks exchange the level's new instances, then the edge
 * slots, launch seeds and diagnostics -- all through fn, an all-gather of
 * variable-size DEVICE buffers (recv gets every rank's bytes in rank order,
 * recv_sizes[r] from rank r; return 0 on success).  The host supplies it:
 * NCCL through torch.distributed (paper_2309_03912_b200/shard.py).  Every
 * rank ends with the same results.  world = 1 (the default) walks alone. */
typedef int (*exs_allgather_fn)(void* ctx, const void* send, uint64_t send_bytes, void* recv,
                                const uint64_t* recv_sizes);
int exs_set_collective(exs_handle h, int rank, int world, exs_allgather_fn fn, void* ctx);

int exs_get_stats(exs_handle h, exs_stats* out);
/* raw records ordered by (file, line, col, code), duplicates removed (only
 * kept with option 6; the rendered form is exs_results_view) */
int exs_get_diags(exs_handle h, exs_diag* out, uint64_t cap, uint64_t* n);
/* Zero-copy view of the ordered diagnostics of the last run: *out points to
 * *n records in page-locked host memory owned by the handle, valid until the
 * next exs_run / exs_run_device / exs_destroy on it. */
int exs_diags_view(exs_handle h, const exs_diag** out, uint64_t* n);
int exs_get_arena(exs_handle h, uint8_t* out, uint64_t cap, uint64_t* n);
int exs_get_pass_status(exs_handle h, exs_pass_status* out, uint64_t cap);
int exs_get_tokens(exs_handle h, uint32_t file, exs_token* out, uint64_t cap, uint64_t* n);
int exs_get_walk_stats(exs_handle h, exs_walk_stats* out, uint64_t cap);
int exs_describe(exs_handle h, const uint32_t* ids, const uint8_t* kinds, uint32_t n,
                 exs_desc* out);
/* options: 1 = also compute per-walk demand counts (Analysis.walks parity);
 * 2 = device timing of later runs (exs_profile_text): 1 the named launches
 *     (CUDA events around each), 2 every launch and the timeline marks, 0 off;
 * 3 = statement-parallel body parsing threshold (tokens, >= 4);
 * 4 = ordered selections of at least this many indices use a flag pass +
 *     flagged compaction (default 4M; 0 forces it, for the parity tests);
 * 5 = nonzero: order diagnostics by two radix sorts ((col, code) then (file, line))
 *     instead of one packed (file, line, col, code) key (for the parity tests);
 * 6 = nonzero: also keep the raw records (exs_get_diags / exs_diags_view);
 * 7 = exs_run_units batch capacity in MiB (default 1024, at most 2047);
 * 8 = host threads packing a batch into page-locked memory (0 = automatic);
 * 9 = exs_run_units pipelines, 1-4: P > 1 analyses P batches concurrently, each
 *     on its own stream with its own buffers (default 2); 1 runs the batches one
 *     after the other */
int exs_set_option(exs_handle h, int key, int value);
/* with option 2 (or EXS_PROFILE=1 in the environment: level 2): per-launch-site
 * device times of the last run, one "site ms xcount" line each */
const char* exs_profile_text(void);
/* per-stage device time of the last run (ms): lex, parse, sema, walk */
int exs_stage_times(exs_handle h, float* out4);

#ifdef __cplusplus
}
#endif
#endif
