/*
 * ct.h -- C ABI of the B200-native Compact-Table (CT) propagation library
 * (paper_2507_18413_b200/libct_b200.so).
 *
 * What it computes: GAC propagation of ONE positive table constraint
 * (PAPER.md L46-55 problem statement; Algorithms 1-3, L131-244):
 *   given the current domains D of x_1..x_n and the values the caller removes,
 *   V = { tuples tau_j : tau_j[i] in D'(x_i) for all i }  (currTable, L189-193)
 *   where D' = D minus the removed values;  FAIL iff V is empty (Alg. 1 L5);
 *   else every value with no valid tuple is pruned (Alg. 3): the new domain of
 *   x_i is { tau_j[i] : j in V }.
 * It gets there the CT way, on the device: static per-(x,a) support bitsets
 * (L188), an RSparseBitSet-style currTable with a compacted index of non-zero
 * words, updateTable with the Delta- or dom-branch (Alg. 2), and filterDomains
 * with residues (L220).  Everything is integer/bitwise; results are exact.
 *
 * Conventions used by every entry point:
 *   - Domains of a table with n variables are "domain bitmaps": uint64 words,
 *     variable i owns ceil(d_i/64) consecutive words starting at word
 *     ct_dom_word_offset(t, i); value v of x_i is bit (v - lo_i) % 64 of word
 *     offset_i + (v - lo_i) / 64 (LSB-first).  Total words: ct_dom_words(t)
 *     ("Wd").  Bits >= d_i in a variable's last word are ignored on input and
 *     written as 0 on output.
 *   - The initial domain of x_i is the interval [lo_i, lo_i + d_i) minus the
 *     holes given by `init_dom` (_variablesOffsets = lo_i).
 *   - currTable is a bitset over tuples: tuple j -> word j/64, bit j%64.
 *   - Status: CT_OK (=0) GAC fixpoint reached; CT_FAIL (=1) no valid tuple
 *     (a normal result that drives backtracking);
 *     negative values are errors; ct_last_error() describes the last one
 *     raised on the calling thread.
 *   - Ownership: the caller owns every buffer it passes; the library copies
 *     what it keeps.  The library owns handles and the device memory behind
 *     them until the matching *_destroy.  Host pointers are plain pageable
 *     memory unless stated; "device pointer" means memory on cfg.device.
 *   - Streams: all device work of a table and its states is ordered on one
 *     CUDA stream (cfg.stream, or a library stream if NULL).  *_async calls
 *     only enqueue work; synchronous calls return after it completed.
 *   - Thread safety: distinct states/batches may be driven from distinct host
 *     threads only if they use distinct streams (ct_state_set_stream); one
 *     state must not be used concurrently.
 *   - A state that returned CT_FAIL is dead: later propagations return
 *     CT_ESTATE without touching the outputs until ct_state_copy() restores it
 *     (SURVEY Q19).
 */
#ifndef CT_B200_H
#define CT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum ct_status {
  CT_OK = 0,        /* GAC fixpoint reached; outputs written                        */
  CT_FAIL = 1,      /* no valid tuple (currTable = 0); outputs not written          */
  CT_PENDING = 2,   /* ct_create of a caller-combined shard: the root's local phase  */
                    /* ran; combine its flags, then ct_propagate_apply_async(root)   */
  CT_EINVAL = -1,   /* invalid argument (message in ct_last_error)                   */
  CT_ENOMEM = -2,   /* device or pinned-host allocation failed                      */
  CT_ECUDA = -3,    /* a CUDA runtime call failed                                   */
  CT_ENCCL = -4,    /* an NCCL call failed                                          */
  CT_ESTATE = -5    /* state is dead (after CT_FAIL) or belongs to another table    */
} ct_status;

typedef struct ct_table ct_table;   /* immutable: geometry + device supports (this shard) */
typedef struct ct_state ct_state;   /* mutable: domains, currTable, index, residues      */
typedef struct ct_batch ct_batch;   /* S independent states of one table, one device pool */

/* Device-memory provider.  alloc returns a device pointer (NULL on failure);
 * `stream` is the cudaStream_t the memory will be used on.  The Python binding
 * passes PyTorch's caching allocator here. */
typedef struct ct_allocator {
  void *(*alloc)(size_t bytes, void *stream, void *ctx);
  void (*free)(void *ptr, size_t bytes, void *stream, void *ctx);
  void *ctx;
} ct_allocator;

/* update_policy: which branch of Alg. 2 each changed
 * variable uses.  Results are identical for all three. */
enum { CT_POLICY_AUTO = 0,   /* Delta-branch iff |Delta_x| < |dom(x)| (L163), else dom   */
       CT_POLICY_DOM = 1,    /* dom-branch only: the paper's implementations (L269-271)  */
       CT_POLICY_DELTA = 2 };/* Delta-branch only                                        */

typedef struct ct_config {
  int32_t device;             /* CUDA device ordinal                                     */
  void *stream;               /* cudaStream_t; NULL -> a library-owned stream           */
  const ct_allocator *alloc;  /* NULL -> cudaMalloc/cudaFree                             */
  int32_t n_shards;           /* tuple-range sharding: 1 = off                           */
  int32_t shard_rank;         /* this process's shard in [0, n_shards)                  */
  const void *nccl_unique_id; /* 128-byte ncclUniqueId shared by all shards, or NULL:   */
                              /*  NULL with n_shards > 1 -> caller combines the flags    */
                              /*  (ct_propagate_local_async / ct_propagate_apply_async)  */
  int32_t update_policy;      /* CT_POLICY_*                                             */
  int32_t use_residues;       /* 1: probe residue word first in filter (L220)            */
  int32_t use_index;          /* 1: keep the compacted non-zero-word index (RSparseBitSet)*/
  int32_t use_graph;          /* 1: synchronous calls replay a captured CUDA graph      */
  int32_t use_fused;          /* 1: a single-state call is one kernel: one CTA for      */
                              /*    tables of <= 8192 16-byte blocks, else a cooperative */
                              /*    persistent grid with software barriers; 0: one      */
                              /*    kernel per phase                                     */
  int32_t use_gather;         /* 1: the k_fast filter may resolve its residue misses by  */
                              /*    gathering the valid tuples' values (device copy of   */
                              /*    the tuples as 8/16-bit value offsets, t x n cells)   */
                              /*    instead of scanning supports rows (Alg. 3), when that */
                              /*    reads fewer bytes; 0: always scan.  Same results.    */
  /* Launch-shape controls (tests and ablations; results never change):        */
  int32_t launch_shape;       /* CT_SHAPE_*: force the single-state launch shape; a    */
                              /*    table that does not fit it gets the automatic one   */
                              /*    (ct_table_info.kernel_path tells which runs)         */
  int32_t grid_override;      /* > 0: CTAs of the cooperative single-state kernels and  */
                              /*    of the model kernels (fewer CTAs than tiles/tables) */
  int32_t batch_per_state;    /* 1: ct_propagate_many runs the per-state phase kernels  */
                              /*    instead of the tile-major batch update              */
  int32_t search_levels;      /* > 0: trail depth of the device-resident DFS (models);  */
                              /*    a deeper search falls back to the host driver       */
  int32_t batch_cells;        /* 1 (default): the tile-major batch update may check the  */
                              /*    few valid tuples of a sparse (state, tile) against  */
                              /*    the new domains instead of OR-ing*/
                              /*    support rows (needs the t x n cells of use_gather); */
                              /*    0: rows only.  Same results.                         */
} ct_config;
enum { CT_SHAPE_AUTO = 0, CT_SHAPE_PHASES = 1, CT_SHAPE_FUSED = 2, CT_SHAPE_FAST = 3, CT_SHAPE_SMALL = 4,
       CT_SHAPE_WIDE = 5 };

/* Fill *cfg with defaults: device 0, NULL stream, default allocator, 1 shard,
 * CT_POLICY_AUTO, residues, index, graphs and the fused kernel on. */
void ct_config_init(ct_config *cfg);

/* ---------------------------------------------------------------- creation */
/* Build the table (supports bitsets) and its root state, and run
 * the root propagation ("checks if each variable ... is supported by at least
 * one tuple, otherwise unsatisfiability is reported", L305-306).
 *   n_vars      >= 1
 *   scope       n_vars distinct variable ids (only checked for duplicates and
 *               kept for the caller; PAPER.md L48 var(c) is a set); may be NULL
 *   dom_lo      int32[n_vars]  lo_i
 *   dom_size    int32[n_vars]  d_i >= 1
 *   init_dom    uint64[Wd] domain bitmap of the initial domains, or NULL = the
 *               full intervals
 *   n_tuples    t >= 0 (t = 0 gives a root CT_FAIL)
 *   tuples      int32[t][n_vars] row-major host array; values outside
 *               [lo_i, lo_i + d_i) are legal and make the tuple never valid.
 *               With n_shards > 1 every rank passes the FULL array and keeps
 *               its own range of 64-tuple words.
 *   cfg         may be NULL (defaults)
 *   out_table, out_root   receive the handles (also on CT_FAIL)
 *   out_dom     host uint64[Wd]: root domains on CT_OK; may be NULL
 * Returns CT_OK, CT_FAIL (root wipe-out; the root state is dead) or an error
 * (no handles are returned on error).
 * Caller-combined shards (n_shards > 1, nccl_unique_id NULL): the root's GAC
 * needs every shard's flags, so ct_create runs only the root's LOCAL phase
 * and returns CT_PENDING without writing out_dom.  The caller then ORs the
 * root's flags across shards (ct_state_flags) and calls
 * ct_propagate_apply_async(root, ...), whose out_status is the root verdict
 * (CT_OK / CT_FAIL) and whose out_dom are the root domains.  Until that apply
 * is enqueued the root cannot be propagated, cloned or copied (CT_ESTATE). */
ct_status ct_create(int32_t n_vars, const int32_t *scope, const int32_t *dom_lo,
                    const int32_t *dom_size, const uint64_t *init_dom, int64_t n_tuples,
                    const int32_t *tuples, const ct_config *cfg, ct_table **out_table,
                    ct_state **out_root, uint64_t *out_dom);

/* ---------------------------------------------------------------- f4: short and negative tables
 * PAPER.md L66-68 and its footnote: "A table c is positive if its tuples list
 * the allowed values for var(c).  A table explicitly listing the disallowed
 * tuples is said negative.  A table is short if more than one domain value can
 * be specified in each cell."  The paper evaluates positive tables only; these
 * kinds are the extensions it names, with GAC still defined
 * by L52-55 on the relation the table denotes.
 *   CT_TABLE_POSITIVE  ct_create's table.
 *   CT_TABLE_SHORT     a cell equal to CT_STAR matches every value of its
 *                      variable (the tuple denotes the product of its cells);
 *                      any other cell is one value as for a positive table.
 *                      Same state, batch, sharding and async calls as positive
 *                      tables; a column holding a star always takes Alg. 2's
 *                      dom-branch (the Δ-branch would drop star tuples).
 *   CT_TABLE_NEGATIVE  the tuples are the FORBIDDEN assignments: rel(c) is the
 *                      product of the initial domains minus the list.  Value a
 *                      of x is pruned iff every assignment of the current
 *                      domains with x = a is listed (a count of valid listed
 *                      tuples per (x,a) against prod_{y != x} |D_y|); CT_FAIL
 *                      iff every assignment is listed.  Duplicate tuples are
 *                      merged at creation (ct_state_read_table then addresses
 *                      the distinct tuples in order of first occurrence).
 *                      Single-state calls only (ct_propagate, _async, clone,
 *                      copy): ct_batch_create, n_shards > 1 and the
 *                      local/apply calls return CT_EINVAL.
 * ct_create_table(kind, ...) takes ct_create's arguments; ct_create(...) is
 * ct_create_table(CT_TABLE_POSITIVE, ...).  CT_STAR is an ordinary
 * out-of-range value for the other kinds. */
enum { CT_TABLE_POSITIVE = 0, CT_TABLE_SHORT = 1, CT_TABLE_NEGATIVE = 2 };
#define CT_STAR INT32_MIN
ct_status ct_create_table(int32_t kind, int32_t n_vars, const int32_t *scope, const int32_t *dom_lo,
                          const int32_t *dom_size, const uint64_t *init_dom, int64_t n_tuples,
                          const int32_t *tuples, const ct_config *cfg, ct_table **out_table,
                          ct_state **out_root, uint64_t *out_dom);

typedef struct ct_table_info {
  int32_t n_vars, n_rows;       /* n, R = sum d_i (support rows)          */
  int32_t dom_words;            /* Wd                                                    */
  int32_t n_shards, shard_rank;
  int64_t n_tuples;             /* t (whole table)                                       */
  int64_t words_total;          /* ceil(t / 64)                                          */
  int64_t word_begin, words;    /* this shard's currTable words [begin, begin + words)   */
  int64_t row_stride_words;     /* padded words per support row on the device            */
  int64_t device_bytes;         /* supports + table metadata on the device               */
  int64_t state_bytes;          /* device bytes of one state                             */
  int32_t kernel_path;          /* single-state launch shape: 0 one kernel per phase,      */
                                /* 1 k_fused (grid barrier per phase), 2 k_fast (per-CTA   */
                                /* ingest, 1-2 grid barriers), 3 k_small (one CTA),        */
                                /* 4 k_wide (one CTA + a thread-per-item filter grid: many */
                                /* support rows over few words, e.g. the paper's LIN sets), */
                                /* 5 negative table (ingest, update, plan, count, finalize) */
  int32_t grid;                 /* CTAs of the single-state launch                       */
  int32_t batch_tile;           /* ct_propagate_many: 16-byte blocks per shared-memory    */
                                /* support tile of the tile-major update (32, 16 or 8), or */
                                /* 0 = one pass per state (R too large for the tile)      */
  int32_t gather_cell_bits;     /* bits per cell of the gather filter's tuple copy, 0 = off */
  int32_t kind;                 /* CT_TABLE_*                                             */
  int32_t batch_cells;          /* 1: the batch update's cell route and sparse-state route */
                                /* are on (ct_config.batch_cells and 8-bit tuple cells)   */
} ct_table_info;

ct_status ct_table_info_get(const ct_table *t, ct_table_info *out);
int32_t ct_dom_words(const ct_table *t);                    /* Wd                         */
int32_t ct_dom_word_offset(const ct_table *t, int32_t i);   /* first word of var i; -1 if bad */

/* ---------------------------------------------------------------- propagation */
/* Synchronous, host buffers (the user-facing call; Alg. 1).
 *   removed     host uint64[Wd]: values to remove (bit set = remove); values
 *               already absent and bits >= d_i are ignored.  May
 *               be NULL = remove nothing.
 *   out_dom     host uint64[Wd]: domains after GAC (written on CT_OK only)
 *   out_pruned  host uint64[Wd] or NULL: values pruned by this call's
 *               filtering, i.e. (domain after the removal) AND NOT out_dom.
 * Copies removed in, runs the whole path on the device (one CUDA graph when
 * cfg.use_graph), copies the result out, and waits for it. */
ct_status ct_propagate(ct_state *s, const uint64_t *removed, uint64_t *out_dom,
                       uint64_t *out_pruned);

/* Asynchronous, device-accessible buffers, enqueued on the state's stream; the
 * call does not wait.  The buffers may be device memory or pinned host memory
 * (cudaHostAlloc / cudaMallocHost).  A host `removed` is read at enqueue and
 * passed with the launch on the k_fast shape (ct_table_info.kernel_path 2,
 * Wd <= 16); otherwise it is DMA'd into one of the state's two device slots on
 * the state's copy stream, overlapping the previous call (pageable memory is
 * accepted but the copy then blocks).  On the k_fast shape the host buffer
 * may be reused as soon as the call returns; otherwise only after the call
 * has run (the DMA is asynchronous).  Host outputs are written in place
 * by the kernel (zero-copy).  So a caller can keep many host-buffer calls in
 * flight.
 *   removed     device uint64[Wd] (NULL = nothing removed)
 *   out_dom     device uint64[Wd] or NULL
 *   out_pruned  device uint64[Wd] or NULL
 *   out_status  device int32[1] or NULL: CT_OK / CT_FAIL / CT_ESTATE
 * Returns CT_OK if the work was enqueued (the propagation's own status lands
 * in *out_status), or an error. */
ct_status ct_propagate_async(ct_state *s, const uint64_t *removed, uint64_t *out_dom,
                             uint64_t *out_pruned, int32_t *out_status);

/* The same call with the input taken from another state of the table: dst
 * becomes the result of propagating `removed` from src (src is only read), as
 * ct_state_copy(dst, src) + ct_propagate_async(dst, ...) would produce, in
 * one pass: on the k_fast launch shape (ct_table_info.kernel_path 2) the
 * update reads src's currTable and index and writes dst's, so the restore of a
 * search node costs no separate copy (the solver's trail, PAPER.md L276,
 * L312); other shapes copy first.  dst == src is ct_propagate_async.  Buffers
 * and status as ct_propagate_async; dst's stream waits for src's earlier
 * work, src's stream waits for the call. */
ct_status ct_propagate_from_async(ct_state *dst, const ct_state *src, const uint64_t *removed,
                                  uint64_t *out_dom, uint64_t *out_pruned, int32_t *out_status);

/* Tuple-range sharding with a caller-side combine (n_shards > 1 and no NCCL id,
 * or for testing several shards on one device).  local: phases a2-a6 on this
 * shard's words, leaving R+1 flag bytes (per support row: "supported by a valid
 * tuple of my slice"; last byte: "my slice has a valid tuple") at the device
 * pointer returned by ct_state_flags.  The caller ORs the flag arrays of all
 * shards element-wise (e.g. an all-reduce with MAX over uint8) into every
 * shard's flags, then calls apply, which finishes the call exactly as the
 * unsharded path would.  The root of a caller-combined shard table goes through
 * the same combine + apply once after ct_create (CT_PENDING above). */
ct_status ct_propagate_local_async(ct_state *s, const uint64_t *removed);
ct_status ct_state_flags(ct_state *s, uint8_t **flags_dev, int32_t *n_bytes);
ct_status ct_propagate_apply_async(ct_state *s, uint64_t *out_dom, uint64_t *out_pruned,
                                   int32_t *out_status);

/* ---------------------------------------------------------------- states */
ct_status ct_state_clone(const ct_state *src, ct_state **out);       /* new state = src      */
ct_status ct_state_copy(ct_state *dst, const ct_state *src);         /* dst := src (async,   */
                                                                    /* device to device);   */
/* with distinct streams, dst's stream first waits for src's earlier work and
 * src's stream then waits for the copy, so either state may be used next on
 * its own stream.  Batch copies (ct_batch_copy*, ct_batch_restore_dead,
 * ct_batch_create) order src's stream after the copy the same way. */
ct_status ct_state_set_stream(ct_state *s, void *stream);            /* cudaStream_t          */
void *ct_state_stream(const ct_state *s);
ct_status ct_synchronize(ct_state *s);                               /* wait for its stream   */
void ct_state_destroy(ct_state *s);
void ct_table_destroy(ct_table *t);   /* destroy all states and batches of t first */

/* ---------------------------------------------------------------- batches */
/* S independent states of one table in one device pool (BASELINE config 4:
 * independent search states).  Each slot starts as a copy of `init`. */
ct_status ct_batch_create(ct_table *t, int32_t n_states, const ct_state *init, ct_batch **out);
int32_t ct_batch_size(const ct_batch *b);
ct_status ct_batch_copy(ct_batch *b, int32_t dst_index, const ct_state *src);   /* async */
ct_status ct_batch_copy_all(ct_batch *b, const ct_state *src);                  /* async */
/* Device-side restart: every state of the batch that is dead (returned CT_FAIL)
 * becomes a copy of `src` (typically the root) -- one kernel, no host round
 * trip, so a search driver can keep S states busy (async, batch stream). */
ct_status ct_batch_restore_dead(ct_batch *b, const ct_state *src);
/* Synchronous, host buffers: removed/out_dom are [S][Wd] row-major (removed may
 * be NULL); out_status int32[S] receives CT_OK / CT_FAIL / CT_ESTATE per state.
 * Returns CT_OK unless an error occurred. */
ct_status ct_propagate_many(ct_batch *b, const uint64_t *removed, uint64_t *out_dom,
                            int32_t *out_status);
/* Asynchronous, device buffers of the same shapes (out_dom, out_status nullable). */
ct_status ct_propagate_many_async(ct_batch *b, const uint64_t *removed, uint64_t *out_dom,
                                  int32_t *out_status);
void ct_batch_destroy(ct_batch *b);

/* ---------------------------------------------------------------- models (several tables) */
/* A CSP of table constraints over shared variables (PAPER.md
 * L46-51 CSP <X, D, C>; L312-316 the engine alternates search and propagation).
 * Every table is a ct_table on the same device; propagation to the common
 * fixpoint runs in ONE cooperative kernel per call (Jacobi iterations over the
 * tables: all tables' CT phases at once, shared domains ANDed after each
 * round, until no table sees a change or one fails).
 *   n_vars, var_lo[n_vars], var_size[n_vars]   the variables X and initial D
 *   n_tables                                    <= 64
 *   arity[n_tables], scopes = concatenated scope var ids (sum arity entries)
 *   n_tuples[n_tables], tuples[k] = int32[n_tuples[k]][arity[k]] host arrays
 *   out_dom (nullable): uint64[ct_model_dom_words] shared domains after the
 *   root fixpoint (CT_OK) -- layout as the table domain bitmaps, one
 *   word-aligned run per variable.
 * Returns CT_OK, CT_FAIL (root wipe-out; the model is dead until
 * ct_model_pop) or an error. */
typedef struct ct_model ct_model;
ct_status ct_model_create(int32_t n_vars, const int32_t *var_lo, const int32_t *var_size, int32_t n_tables,
                          const int32_t *arity, const int32_t *scopes, const int64_t *n_tuples,
                          const int32_t *const *tuples, const ct_config *cfg, ct_model **out,
                          uint64_t *out_dom);
int32_t ct_model_dom_words(const ct_model *m);
int32_t ct_model_dom_word_offset(const ct_model *m, int32_t v);
/* Synchronous.  dom_in (nullable, host uint64[Wg]): restrict the shared domains
 * to dom_in (a search decision; values absent now stay absent), then propagate
 * all tables to the common fixpoint.  out_dom (nullable) receives the shared
 * domains on CT_OK.  On CT_FAIL the model is dead until ct_model_pop. */
ct_status ct_model_fixpoint(ct_model *m, const uint64_t *dom_in, uint64_t *out_dom);
ct_status ct_model_push(ct_model *m);   /* save the whole model state (trail level) */
ct_status ct_model_pop(ct_model *m);    /* restore and drop the last saved state     */
typedef struct ct_search_stats {
  int64_t nodes;          /* fixpoint calls: the root plus every branch            */
  int64_t failures;       /* of those, CT_FAIL                                      */
  int64_t solutions;
  int64_t table_calls;    /* non-no-op table propagations inside the fixpoints      */
  int64_t iterations;     /* Jacobi rounds summed over the fixpoints                */
  int64_t max_depth;
  double device_ms;       /* kernel time summed over the fixpoints (%globaltimer)   */
  uint64_t trace_hash;    /* FNV-1a over (depth, var, value, branch, status) per node */
} ct_search_stats;
/* Depth-first search with binary branching x = v / x != v,
 * variable order input_order (lowest-index unbound variable), value order
 * indomain_max (value_order = 0) or indomain_min (1), the paper's strategy
 * (PAPER.md L469-477).  Stops after max_solutions solutions (<= 0: all) or
 * max_nodes nodes (<= 0: no limit).  out_solution (nullable): int32[n_vars],
 * the last solution found.  Returns CT_OK if a solution was found, CT_FAIL if
 * the (explored part of the) tree has none, or an error.  The model's state is
 * restored to what it was before the call. */
ct_status ct_model_search(ct_model *m, int32_t value_order, int64_t max_nodes, int64_t max_solutions,
                          int32_t *out_solution, ct_search_stats *out_stats);
/* The same search with an explicit driver: 0 = device-resident (the whole DFS
 * in one cooperative kernel: decisions, trail snapshots of all table states,
 * fixpoints and backtracking stay on the GPU; falls back to the host driver if
 * the trail would exceed 512 levels or the model has a push pending), 1 =
 * host-driven (one fixpoint launch per node).  Identical results and node
 * traces; ct_model_search uses driver 0.
 * device_ms is then the whole kernel's time. */
ct_status ct_model_search_ex(ct_model *m, int32_t value_order, int64_t max_nodes, int64_t max_solutions,
                             int32_t driver, int32_t *out_solution, ct_search_stats *out_stats);
/* Measurement only: ns the last device-resident search spent in each phase,
 * out6 = {ingest, update, probe, scan, finalize, trail copies} (block 0's
 * clock, barriers included); -1 if no device search ran. */
ct_status ct_model_search_phases(const ct_model *m, int64_t *out6);
void ct_model_destroy(ct_model *m);

/* ---------------------------------------------------------------- introspection */
/* Test/measurement only.  currTable of this shard: host uint64[words]. */
ct_status ct_state_read_table(const ct_state *s, uint64_t *out_bits);
/* currTable of state i of a batch: host uint64[words]. */
ct_status ct_batch_read_table(const ct_batch *b, int32_t i, uint64_t *out_bits);
/* One support row (row = rowbase_i + v - lo_i) of this shard: host uint64[words]. */
ct_status ct_table_read_supports(const ct_table *t, int32_t row, uint64_t *out_bits);
/* Current domains of a state (its last fixpoint): host uint64[Wd]. */
ct_status ct_state_read_dom(const ct_state *s, uint64_t *out_dom);

typedef struct ct_stats {
  int64_t calls;            /* propagations run on this state (copies carry it over)  */
  int32_t last_status;      /* CT_OK / CT_FAIL / CT_ESTATE of the last call            */
  int32_t noop;             /* last call had no changed variable                       */
  int32_t n_changed;        /* |s_val|                                 */
  int32_t n_update_rows;    /* support rows OR-ed by updateTable                       */
  int32_t n_filter_items;   /* (x,a) checked by filterDomains (x in s_sup, L201)       */
  int32_t n_residue_miss;   /* of those, residue probe misses -> index scans           */
  int64_t words_in;         /* index entries before the update (L_in); an entry is a   */
                            /* 16-byte block (2 currTable words) with a valid tuple    */
  int64_t words_out;        /* index entries after the update (L_out)                  */
  int64_t update_support_words;  /* 64-bit support words loaded by updateTable          */
  int64_t update_table_writes;   /* 16-byte currTable blocks rewritten by updateTable   */
  int64_t filter_support_words;  /* support words loaded by the filter's index scans    */
  int64_t phase_ns[7];      /* single-state kernels only (%globaltimer of block 0, and of */
                            /* the finishing CTA for k_fast); k_fused / k_small: ingest,  */
                            /* update, probe, scan, finalize, 0, 0; k_fast: ingest,        */
                            /* update (+ barrier), probe, barrier, scan, completion wait,   */
                            /* finalize.  Not written by the per-phase kernels.            */
  int64_t filter_gathered_tuples; /* k_fast gather filter: valid tuples whose values it read  */
                                  /* (0 when the misses were scanned, ct_config.use_gather)  */
} ct_stats;
ct_status ct_state_stats(const ct_state *s, ct_stats *out);
/* The same counters for every state of a batch (last ct_propagate_many call):
 * out = host ct_stats[ct_batch_size(b)], caller-owned.  Waits for the table's
 * stream.  phase_ns is 0 (the batch kernels do not stamp phases); with the
 * tile-major update (ct_table_info.batch_tile > 0) update_support_words and
 * update_table_writes are per batch only, see ct_batch_work. */
ct_status ct_batch_stats(const ct_batch *b, ct_stats *out);
/* Work counters of the tile-major batch path (measurement only): [0] 64-bit support words the update OR-ed (from shared memory),
 * [1] 16-byte currTable blocks it read, [2] blocks it rewrote, [3] support
 * (and tuple-cell) bytes staged from global into shared memory, [6] valid
 * tuples the update's cell routes checked, [7] state updates that took the
 * sparse-state route, [8] the updating states' input active 16-byte blocks
 * (sum of L_in: the currTable traffic the algorithm needs) -- [0..3] and
 * [6..8] summed over all calls since the last reset (reset != 0 zeroes them
 * after the read); [4] support words the filter scans loaded and [5]
 * residue-probe misses, both of the last call; [9] 0.  out10 = host int64[10].
 * All -1 on the per-state path (batch_tile = 0).  Waits for the stream. */
ct_status ct_batch_work(ct_batch *b, int64_t *out10, int32_t reset);

/* Served calls (latency-bound tables, BASELINE config 2).  on != 0: the
 * state's synchronous ct_propagate calls are served by a persistent
 * single-CTA kernel on the state's own server stream that polls a doorbell in
 * mapped host memory, instead of one graph launch per call: the call writes
 * the removal and rings; the kernel (k_small's body) writes domains, pruned
 * values and the status word straight to mapped host memory.  The server starts
 * with the first call, stops after ct_debug_serve_idle (default 200 ms)
 * without a request (the next call restarts it), and is stopped by on = 0,
 * ct_state_destroy and by every call that writes the state or reads it on a
 * stream (clones, async / sharded calls, batches from it); ct_state_copy
 * INTO a running served state (a search's restore) is served in place.
 * Results are those of ct_propagate.  Requires the single-CTA launch shape
 * (ct_table_info.kernel_path 3), one shard and Wd <= 14, else CT_EINVAL; the
 * state must be used from one host thread.  It occupies one SM while running. */
ct_status ct_state_serve(ct_state *s, int32_t on);
/* The served kernel's idle limit (ns, > 0), all states of the process. */
ct_status ct_debug_serve_idle(int64_t ns);
/* Experiment builds (-DCT_SERVE_TRACE) only: %globaltimer stamps of the last
 * served call (out16 = host int64[16]; zeros otherwise). */
ct_status ct_debug_serve_trace(const ct_state *s, int64_t *out16);

/* ---- a10 over NVLink peer memory.
 * Instead of an NCCL all-reduce between two kernels, the k_fast finalizer of a
 * tuple-range shard stores its R+1 flag bytes into every rank's inbox over
 * NVLink (CUDA IPC peer pointers), publishes them with a system-scope release,
 * waits for every rank's flags of the same call and ORs them itself: one
 * kernel per sharded call.  Collective protocol, every rank in the same order:
 *   ct_peer_export(table, handle)        -> this rank's inbox as a
 *                                           CT_PEER_HANDLE_BYTES-byte IPC handle
 *   (exchange the handles, e.g. torch.distributed.all_gather_object)
 *   ct_peer_attach(table, n_shards, all) -> handles[n_shards][CT_PEER_HANDLE_BYTES],
 *                                           rank order; opens the others' inboxes
 * After attach every sharded call on the table combines in-kernel (the NCCL
 * communicator, if any, is no longer used by k_fast).  Requirements: the
 * table runs the k_fast launch shape (ct_table_info.kernel_path 2; CT_EINVAL
 * otherwise), all ranks on one node with peer access, and a table's sharded
 * calls issued in the same order on every rank and one at a time (its states
 * on one stream): the calls are matched by a per-table epoch counter.  With
 * n_shards = 1 the table exchanges with itself (tests the protocol on one GPU).
 * Errors: CT_EINVAL (NULL, wrong count, not exported, already attached,
 * launch shape), CT_ENOMEM, CT_ECUDA (IPC).  A rank that does not arrive
 * within 120 s makes the others' kernels trap (CT_ECUDA). */
#define CT_PEER_HANDLE_BYTES 64
ct_status ct_peer_export(ct_table *t, void *out_handle);
ct_status ct_peer_attach(ct_table *t, int32_t n_shards, const void *handles);

/* Per-kernel device timing (measurement only).  While enabled, every
 * *_async / ct_propagate_many call on this table's states and batches records a
 * CUDA event pair around each of its kernels on the launching stream (not inside
 * captured graphs).  read() waits for the stream, returns the summed durations
 * and launch counts since the last reset, and resets them if `reset`.
 * Kernel slots: 0 ingest, 1 update, 2 probe, 3 scan, 4 combine (NCCL), 5 finalize,
 * 6 fused (all phases of a single-state call in one kernel), 7 small (the same in
 * one CTA, for tables of at most 8192 16-byte blocks; also k_wide + k_wide_filter). */
typedef struct ct_kernel_times {
  int64_t launches[8];
  double ms[8];
} ct_kernel_times;
ct_status ct_table_profile(ct_table *t, int32_t enable);
ct_status ct_table_profile_read(ct_table *t, ct_kernel_times *out, int32_t reset);

/* ---------------------------------------------------------------- placement ablation
 * The paper's serial CT propagator and its GPU-offloaded derivatives
 * (§4), for the placement ablation only -- a separate,
 * explicitly selected engine; ct_propagate never routes through it:
 *   CT_PLACE_HOST  serial CT on the host: Alg. 1-3, RSparseBitSet currTable,
 *                  residues
 *   CT_PLACE_U     CT^u: currTable + s_val + domains to the device, the mask
 *                  (dom-branch OR per changed variable, AND over them) built
 *                  by a kernel and copied back, ANDed on the host; host filter
 *
 *   CT_PLACE_F     CT^f: host update; currTable + domains to the device, a
 *                  kernel returns the removal bitmap
 *   CT_PLACE_UF    CT^uf: both kernels with the paper's per-call transfers
 *
 * Semantics are ct_create / ct_propagate's (same domain-bitmap layout, same
 * results; CT_FAIL kills the state until ct_host_copy).  Host buffers only;
 * every call is synchronous.  cfg: device, stream, update_policy are used. */
enum { CT_PLACE_HOST = 0, CT_PLACE_U = 1, CT_PLACE_F = 2, CT_PLACE_UF = 3 };
typedef struct ct_host_table ct_host_table;
typedef struct ct_host_state ct_host_state;
ct_status ct_host_create(int32_t n_vars, const int32_t *dom_lo, const int32_t *dom_size, const uint64_t *init_dom,
                         int64_t n_tuples, const int32_t *tuples, int32_t placement, const ct_config *cfg,
                         ct_host_table **out_table, ct_host_state **out_root, uint64_t *out_dom);
ct_status ct_host_propagate(ct_host_state *s, const uint64_t *removed, uint64_t *out_dom, uint64_t *out_pruned);
ct_status ct_host_clone(const ct_host_state *src, ct_host_state **out);
ct_status ct_host_copy(ct_host_state *dst, const ct_host_state *src);
int32_t ct_host_dom_words(const ct_host_table *t);
/* Per-table accounting since the last reset: host time of the propagator's own
 * work, CUDA-event times of the copies and kernels, bytes moved. */
typedef struct ct_place_stats {
  int64_t calls, noops, kernel_launches;
  int64_t h2d_bytes, d2h_bytes;
  double host_ms, h2d_ms, kernel_ms, d2h_ms;
} ct_place_stats;
ct_status ct_host_stats(ct_host_table *t, ct_place_stats *out, int32_t reset);
void ct_host_state_destroy(ct_host_state *s);
void ct_host_table_destroy(ct_host_table *t);   /* destroy its states first */

/* Tuple-range partition used by sharded tables (host-only, no device needed):
 * shard `rank` of `n_shards` owns currTable words [*word_begin, *word_begin +
 * *words) of the ceil(n_tuples/64) words, i.e. tuples [64*begin, min(64*(begin
 * + words), n_tuples)).  Boundaries are floor(g * words_total / n_shards)
 * rounded down to a multiple of 16 words (128-byte rows); the shards tile the
 * table exactly.  Returns CT_EINVAL on bad arguments. */
ct_status ct_shard_range(int64_t n_tuples, int32_t n_shards, int32_t rank, int64_t *word_begin,
                         int64_t *words);

/* Spin watchdog (diagnostics).  Every software grid barrier and chained-scan
 * look-back of the kernels traps after waiting 4 s (the call then fails with
 * CT_ECUDA instead of hanging the GPU).  attach: give `device`'s kernels a
 * host-mapped buffer to record, before trapping, which CTA waited where (its
 * kind, polled words, location marker, barrier count) and every CTA's location
 * and barrier count.  read: copy up to n_words of that buffer (no CUDA call, so
 * it works while a kernel spins); word 0 == 0xD1A6D1A6 once a report is
 * complete.  Returns the words copied. */
ct_status ct_debug_diag_attach(int32_t device);
/* The watchdog's limit for `device` (default 4 s; e.g. raised under
 * compute-sanitizer, which slows every CTA). */
ct_status ct_debug_spin_limit(int32_t device, double seconds);
int64_t ct_debug_diag_read(uint64_t *out, int64_t n_words);

/* NCCL bootstrap helper: writes a fresh 128-byte ncclUniqueId (rank 0 calls it
 * and broadcasts the bytes, e.g. with torch.distributed). */
ct_status ct_nccl_unique_id(void *out128);

const char *ct_last_error(void);
const char *ct_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CT_B200_H */
