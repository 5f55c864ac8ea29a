/*
 * gfx.h -- C ABI of libgfx.so, the B200 (sm_100a) frontier core that backs the
 * graphfx-compatible Python package `paper_1701_01170_b200`.
 *
 * The reference (`graphfx`, /root/reference/pkg/src/graphfx) is pure Python;
 * its boundary is the Python API re-exported in graphfx/__init__.py:8-72.
 * Each entry point below replaces the device work behind one reference
 * function (cited per function).  The Python layer (`_native.py`) binds these
 * with ctypes and keeps the reference's argument meaning and error behaviour.
 *
 * Conventions
 *   - Every function returns an int status: GFX_OK (0), GFX_EINVAL (1, ->
 *     ValueError), GFX_ECUDA (2, -> RuntimeError), GFX_ENOMEM (3, ->
 *     MemoryError), GFX_ENCCL (4).  gfx_last_error() returns a thread-local
 *     message for the last failure on the calling thread.
 *   - Pointers suffixed _d are DEVICE pointers (borrowed; caller keeps them
 *     alive, e.g. torch tensors).  Pointers without the suffix are host.
 *   - Device vertex ids / labels are int32; row offsets are int64.  Unreached
 *     labels are GFX_UNVISITED (INT32_MAX), missing predecessors are -1.  The
 *     Python layer widens to the reference's int64 layout (graph.py:15-22).
 *   - One ctx per device; calls on a ctx are stream-ordered on the ctx stream
 *     and synchronise that stream before returning (bulk-synchronous
 *     visibility, reference operators.py:10-15).  Not re-entrant.
 *   - Scratch (queues, bitmaps, scan temporaries) is owned by the graph handle.
 */
#ifndef GFX_H
#define GFX_H

#include <stdint.h>

#if defined(GFX_BUILD)
#define GFX_API __attribute__((visibility("default")))
#else
#define GFX_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define GFX_OK 0
#define GFX_EINVAL 1
#define GFX_ECUDA 2
#define GFX_ENOMEM 3
#define GFX_ENCCL 4

#define GFX_UNVISITED 2147483647

/* graph flags */
#define GFX_GRAPH_UNDIRECTED 1 /* CSR is symmetric: reverse adjacency == CSR */

/* traversal direction (reference primitives/bfs.py:42-68) */
#define GFX_DIR_PUSH 0
#define GFX_DIR_PULL 1
#define GFX_DIR_AUTO 2

/* filter modes (reference operators.py:61-63) */
#define GFX_FILTER_EXACT 0
#define GFX_FILTER_INEXACT 1

/* BFS run modes */
#define GFX_LOOP_HOST 0   /* host decides direction each level (exact Python replica) */
#define GFX_LOOP_DEVICE 1 /* device-resident level loop, decision on device */

typedef struct gfx_ctx gfx_ctx;
typedef struct gfx_graph gfx_graph;

/* One record per BFS/SSSP/BC iteration; mirrors RunStats.per_iteration and
 * RunStats.direction_trace (reference stats.py:33-59, bfs.py:104-107). */
typedef struct gfx_iter_rec {
  int64_t iteration;
  int64_t frontier_in;  /* n_f */
  int64_t frontier_out;
  int64_t n_u;          /* unvisited estimate after subtracting n_f */
  int64_t edges;        /* plan.total_output of this iteration */
  double m_f;
  double m_u;
  int32_t mode_before;  /* GFX_DIR_PUSH / GFX_DIR_PULL */
  int32_t decision;
  float ms;             /* device time of the iteration (0 unless timing is on) */
  int32_t pad;
  int64_t candidates;   /* pull: |U| with in-degree > 0 */
  int64_t work;         /* push: expansion slots; pull: early-exit probes S(U) */
  int64_t bytes_alg;    /* algorithmic HBM bytes of the iteration */
} gfx_iter_rec;

typedef struct gfx_stats {
  int64_t iterations;
  int64_t edges_traversed;
  int64_t direction_switches;
  int64_t reached;        /* vertices with a finite label */
  int64_t edges_reached;  /* sum of out-degrees of reached vertices (E_r) */
  int64_t work_slots;     /* kernel-counted expansion slots (SSSP inflation) */
  int64_t bytes_alg;      /* algorithmic HBM bytes (DESIGN.md formulas) */
  double device_ms;       /* CUDA-event time of the device loop */
  int64_t num_records;    /* records written (<= rec_cap) */
  int64_t init_ns;        /* device-resident BFS: output/state initialisation */
  int64_t loop_ns;        /* device-resident BFS: level loop */
} gfx_stats;

/* ---- library / context ------------------------------------------------ */
GFX_API int gfx_version(void);
/* number of kernels libgfx has launched in this process (monotonic) */
GFX_API int64_t gfx_launch_count(void);
/* per-iteration CUDA-event timing of the level loops (records' ms field) */
GFX_API int gfx_ctx_set_timing(gfx_ctx* ctx, int enabled);
/* 1 (default): full RunStats (E_r, pull-level edges via a degree post-pass);
 * 0: skip the statistics post-passes (labels/preds/trace unaffected) */
GFX_API int gfx_ctx_set_stats(gfx_ctx* ctx, int detail);
GFX_API const char* gfx_last_error(void);
/* stream: a cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream); NULL
 * selects the legacy default stream */
GFX_API int gfx_ctx_create(int device, void* stream, gfx_ctx** out);
GFX_API int gfx_ctx_destroy(gfx_ctx* ctx);
GFX_API int gfx_ctx_sync(gfx_ctx* ctx);
GFX_API int gfx_ctx_sm_count(gfx_ctx* ctx);

/* ---- graph (reference graph.py:61-155 CsrGraph) ------------------------ */
/* row_d int64[n+1], col_d int32[m], w_d int32[m] or NULL.  For directed graphs
 * the reverse adjacency (graph.py:113-126 CsrGraph.csc) is attached with
 * gfx_graph_set_reverse before any pull traversal. */
GFX_API int gfx_graph_create(gfx_ctx* ctx, int64_t n, int64_t m, const int64_t* row_d,
                     const int32_t* col_d, const int32_t* w_d, int flags,
                     gfx_graph** out);
GFX_API int gfx_graph_set_reverse(gfx_graph* g, const int64_t* rrow_d, const int32_t* rcol_d);
GFX_API int gfx_graph_destroy(gfx_graph* g);
/* max out-degree (host value, computed at create) */
GFX_API int64_t gfx_graph_max_degree(gfx_graph* g);
/* release scratch buffers (they are re-allocated lazily) */
GFX_API int gfx_graph_trim(gfx_graph* g);
/* The caller rewrote the borrowed row/col (/weights/reverse) arrays in place,
 * same n and m (e.g. a new graph uploaded into the same device buffers):
 * recompute the graph constants derived from them (max degree, nonzero
 * bitmaps, pull heads, TC orientation), keeping every scratch allocation.
 * Replaces building a fresh CsrGraph device copy (reference graph.py:61-155). */
GFX_API int gfx_graph_refresh(gfx_graph* g);

/* ---- BFS (reference primitives/bfs.py:42-159) ---------------------------
 * labels_d/preds_d int32[n] (outputs).  recs: host array of rec_cap records
 * (may be NULL).  loop: GFX_LOOP_HOST or GFX_LOOP_DEVICE. */
GFX_API int gfx_bfs(gfx_graph* g, int64_t source, int direction, int idempotent,
            int filter_mode, double do_a, double do_b, int mu_edge_based,
            int loop, int32_t* labels_d, int32_t* preds_d, gfx_iter_rec* recs,
            int64_t rec_cap, gfx_stats* stats);

/* count BFS runs from sources[0..count) back to back on the device-resident
 * loop (one launch each, one synchronisation): *ms = device time of all runs.
 * labels_d/preds_d receive the last run.  Used to measure device throughput
 * without per-call host round trips. */
GFX_API int gfx_bfs_batch(gfx_graph* g, const int64_t* sources, int64_t count, int direction,
                          double do_a, double do_b, int mu_edge_based, int32_t* labels_d,
                          int32_t* preds_d, float* ms);

/* Host-only replica of reference direction.py:52-61 estimate_mf_mu with the
 * same correctly rounded integer divisions CPython performs (no GPU needed). */
GFX_API int gfx_estimate_mf_mu(int64_t n, int64_t m, int64_t n_f, int64_t n_u, int mu_edge_based,
                               double* m_f, double* m_u);

/* ---- SSSP near/far (reference primitives/sssp.py:41-121, near_far.py) ---
 * delta: bucket width (<= 0 or +inf: no priority queue).  dist_d int32[n]
 * (INT32_MAX = unreached), preds_d int32[n]. */
GFX_API int gfx_sssp(gfx_graph* g, int64_t source, double delta, int32_t* dist_d,
             int32_t* preds_d, gfx_iter_rec* recs, int64_t rec_cap, gfx_stats* stats);

/* ---- BC (reference primitives/bc.py:32-116) ----------------------------
 * Accumulates into bc_d (float64[n], caller zero-initialises). */
GFX_API int gfx_bc(gfx_graph* g, const int64_t* sources, int64_t num_sources, double* bc_d,
           gfx_stats* stats);

/* ---- CC (reference primitives/cc.py:23-98) -----------------------------
 * comp_d int32[n] receives canonical min-id labels. */
GFX_API int gfx_cc(gfx_graph* g, int32_t* comp_d, int64_t* num_components, gfx_stats* stats);

/* ---- PageRank (reference primitives/pagerank.py:30-91) ------------------ */
GFX_API int gfx_pagerank(gfx_graph* g, double damping, double epsilon, int64_t max_iters,
                 double* rank_d, gfx_stats* stats);

/* ---- TC (reference primitives/tc.py:27-86, operators.py:485-525) --------
 * Phase 1 orients and returns the oriented edge count; phase 2 fills the
 * caller-allocated outputs (int32[m_oriented] each, osrc/odst in the
 * oriented CSR order of tc.py:53-56) and the int64 total. */
GFX_API int gfx_tc_orient(gfx_graph* g, int64_t* m_oriented);
GFX_API int gfx_tc_count(gfx_graph* g, int32_t* osrc_d, int32_t* odst_d, int32_t* counts_d,
                 int64_t* total, gfx_stats* stats);

/* ---- segmented intersection (reference operators.py:485-525) ------------
 * counts_d int32[num_pairs]; total out. */
GFX_API int gfx_segmented_intersect(gfx_graph* g, const int32_t* u_d, const int32_t* v_d,
                            int64_t num_pairs, int32_t* counts_d, int64_t* total);

/* ---- generic advance / filter with the closed device-functor registry ---
 * (reference operators.py:218-266, 360-384; SURVEY 8(b) functor table).
 * Registry functors run fused inside the load-balanced expansion; arbitrary
 * Python callables run staged on device tensors through the building blocks
 * further below (gfx_scan_offsets / gfx_gather / gfx_select_i64 ...). */
#define GFX_FN_NONE 0
#define GFX_FN_BFS_CLAIM 1     /* bfs.py:118-121 compare_and_swap claim + preds[d] = s */
#define GFX_FN_BFS_IDEMP 2     /* bfs.py:113-116 labels[d] == UNVISITED; _set_depth */
#define GFX_FN_SSSP_RELAX 3    /* sssp.py:95-103 atomic_min winners + set_pred */
#define GFX_FN_TC_ORIENT 4     /* tc.py:57-59 */
#define GFX_FN_LABEL_EQ 5      /* cond / vertex_cond labels[x] == value */
#define GFX_FN_LABEL_NE 6      /* cond / vertex_cond labels[x] != value */
#define GFX_FN_SET_LABEL 7     /* compute: labels[v] = value */
#define GFX_FN_ADD_I64 8       /* compute: acc[v] += value (atomic_add, operators.py:127-128) */
#define GFX_FN_BFS_PULL 9      /* bfs.py:142-145 pull cond labels[s] == value-1; _set_depth */
#define GFX_FN_BC_CLAIM 10     /* bc.py:80-84 compare_and_swap(labels, d, UNVISITED, depth) */
#define GFX_FN_BC_SIGMA 11     /* bc.py:87-92 labels[d] == value; sigma[d] += sigma[s] */
#define GFX_FN_BC_DELTA 12     /* bc.py:104-109 labels[d] == value;
                                  delta[s] += sigma[s]/sigma[d]*(1+delta[d]) */
#define GFX_FN_PR_SCATTER 13   /* pagerank.py:71-75 rank_next[d] += scalar*rank[s]/outdeg[s] */
#define GFX_FN_PR_MOVED 14     /* pagerank.py:81-85 vertex_cond |rank_next-rank| >= scalar */
#define GFX_FN_CC_SAME_COMP 15 /* cc.py:55-58 edge vertex_cond comp[src(e)] != comp[col[e]] */
#define GFX_FN_SSSP_STAMP 16   /* sssp.py:112-115 vertex_cond stamps[v] == value */
#define GFX_FN_COUNT 17

typedef struct gfx_functor_args {
  int32_t* labels_d;   /* int32 labels / distances / comp / stamps */
  int32_t* preds_d;    /* int32 preds (may be NULL) */
  int64_t value;       /* depth / compared value */
  double* f0_d;        /* BC sigma / PR rank */
  double* f1_d;        /* BC delta / PR rank_next */
  double scalar;       /* PR damping (scatter) / epsilon (moved) */
} gfx_functor_args;

#define GFX_KIND_V2V 0
#define GFX_KIND_V2E 1
#define GFX_KIND_E2V 2
#define GFX_KIND_E2E 3

/* Push advance over fin_d[0..nin) (vertex or edge ids by kind).  Output ids
 * (cond-true images) are written to fout_d (capacity fout_cap); *nout gets
 * the count.  Returns GFX_EINVAL if the output would overflow. */
GFX_API int gfx_advance(gfx_graph* g, const int32_t* fin_d, int64_t nin, int kind,
                int functor_id, const gfx_functor_args* args, int32_t* fout_d,
                int64_t fout_cap, int64_t* nout, int64_t* edges);
/* advance_filter_fused (operators.py:392-456): ONE load-balanced expansion
 * that evaluates the registry cond, the registry vertex_cond on the image and
 * culls re-occurrences against a bitmap over the output domain (n or m), so
 * every survivor is emitted once and no middle frontier exists. */
GFX_API int gfx_advance_fused(gfx_graph* g, const int32_t* fin_d, int64_t nin, int kind,
                              int cond_id, const gfx_functor_args* cond_args, int vcond_id,
                              const gfx_functor_args* vcond_args, int32_t* fout_d,
                              int64_t fout_cap, int64_t* nout, int64_t* edges);
/* pull_expand with a registry functor (operators.py:269-307, direction.py:73-89):
 * for each unvisited u in fin_d (in order), probe its in-neighbours s in
 * reverse-adjacency order and stop at the first cond-true triple; for
 * GFX_FN_BFS_PULL the hit commits labels[u] = value, preds[u] = s.  The input
 * is split stably into active_d (a hit) and rest_d (no hit); *edges gets the
 * probes made (the early-exit count S(U)). */
GFX_API int gfx_pull_advance(gfx_graph* g, const int32_t* fin_d, int64_t nin, int functor_id,
                             const gfx_functor_args* args, int32_t* active_d, int64_t* nactive,
                             int32_t* rest_d, int64_t* nrest, int64_t* edges);
/* Filter: keep items satisfying vertex functor, then (EXACT) dedup to the
 * sorted unique set of survivors (np.unique semantics) or (INEXACT) cull. */
GFX_API int gfx_filter(gfx_graph* g, const int32_t* fin_d, int64_t nin, int mode,
               int functor_id, const gfx_functor_args* args, int64_t domain,
               int32_t* fout_d, int64_t* nout);
/* mask_d[i] = registry vertex_cond(fin_d[i]) (INEXACT filtering runs the
 * culling stages over the survivors) */
GFX_API int gfx_vertex_mask(gfx_graph* g, const int32_t* fin_d, int64_t nin, int functor_id,
                            const gfx_functor_args* args, uint8_t* mask_d);
/* compute (operators.py:528-533): apply a registry functor to every item,
 * multiplicity included (acc_d: int64 array for GFX_FN_ADD_I64) */
GFX_API int gfx_compute(gfx_graph* g, const int32_t* fin_d, int64_t nin, int functor_id,
                        const gfx_functor_args* args, int64_t* acc_d);

/* ---- building blocks of the staged operator path (Python callables as
 * functors, evaluated on device tensors between these calls) ------------- */
/* compute_scan_offsets (load_balance.py:94-113): scan_d int64[nin+1] is the
 * exclusive prefix sum of the expansion degrees of fin_d (vertex ids, or edge
 * ids whose head col[e] expands when edge_input); reverse: in-degrees. */
GFX_API int gfx_scan_offsets(gfx_graph* g, const int32_t* fin_d, int64_t nin, int edge_input,
                             int reverse, int64_t* scan_d, int64_t* total);
/* _gather (operators.py:161-197): every expansion slot k in slot order.  Item
 * i owns slots [scan[i], scan[i+1]); its vertex v expands slot j = row[v] +
 * k - scan[i]: a_d[k] = v, b_d[k] = col[j], e_d[k] = j.  reverse: the reverse
 * adjacency (gfx_graph_build_csc), e_d[k] = the forward slot of the in-edge.
 * rep_d[k] = i (nullable). */
GFX_API int gfx_gather(gfx_graph* g, const int32_t* fin_d, int64_t nin, int edge_input,
                       int reverse, const int64_t* scan_d, int64_t total, int64_t* a_d,
                       int64_t* b_d, int64_t* e_d, int32_t* rep_d);
/* CsrGraph.csc (graph.py:113-126) on the device: rrow_d int64[n+1], rcol_d
 * int32[m] (sources, ascending within a row) and reid_d int64[m] (forward
 * slot of each in-edge), from a stable radix sort of the column ids; the
 * result is attached to the graph as its reverse adjacency. */
GFX_API int gfx_graph_build_csc(gfx_graph* g, int64_t* rrow_d, int32_t* rcol_d, int64_t* reid_d);
/* stable stream compaction: out_d = in_d[flags_d != invert] (order kept) */
GFX_API int gfx_select_i64(gfx_ctx* ctx, const int64_t* in_d, const uint8_t* flags_d, int64_t n,
                           int invert, int64_t* out_d, int64_t* nout);
/* StatusBitmap.test_and_set (frontier.py:70-94): fresh_d[i] = bit ids[i]
 * clear before the call (reads precede writes), then every bit is set */
GFX_API int gfx_bitmap_test_and_set(gfx_ctx* ctx, uint32_t* words_d, const int64_t* ids_d,
                                    int64_t k, uint8_t* fresh_d);
/* generate_unvisited_frontier (frontier.py:97-100): ascending ids with
 * labels[v] == sentinel (dtype 0 int32, 1 int64) */
GFX_API int gfx_unvisited(gfx_ctx* ctx, int dtype, const void* labels_d, int64_t n,
                          int64_t sentinel, int64_t* out_d, int64_t* nout);
/* hits_d[rep_d[k]] = 1 for every k with mask_d[k] (pull_expand hit marking) */
GFX_API int gfx_mark_items(gfx_ctx* ctx, const uint8_t* mask_d, const int32_t* rep_d, int64_t k,
                           uint8_t* hits_d);
/* INEXACT culling (operators.py:315-357), reproduced exactly: keep_d[i] = 0
 * for items the reference heuristics drop.  Bitmask: an item is kept iff no
 * earlier batch of bitmask_batch items held its id; history tables: within
 * each batch an item is dropped when the previous item of the batch hashing
 * to its slot (id mod table) carried the same id.  Pass table 0 to skip a
 * stage.  Stages run in the reference order, each over the survivors of the
 * previous one, so the caller compacts between stages (stage = 0, 1, 2). */
GFX_API int gfx_cull_stage(gfx_ctx* ctx, const int64_t* items_d, int64_t n, int stage,
                           int64_t domain, int64_t table_or_batch, int64_t batch,
                           uint8_t* keep_d);

/* ---- batched atomic helpers (operators.py:111-153) on device arrays -----
 * dtype: 0 int32, 1 int64, 2 float32, 3 float64.  idx_d int64[k]. */
/* scatter-min; won_d[i] = vals[i] < pre[idx[i]] && vals[i] == post[idx[i]] */
GFX_API int gfx_atomic_min(gfx_ctx* ctx, int dtype, void* arr_d, const int64_t* idx_d,
                           const void* vals_d, int64_t k, uint8_t* won_d, void* pre_d);
/* scatter-add (np.add.at); vals_d NULL adds the scalar */
GFX_API int gfx_atomic_add(gfx_ctx* ctx, int dtype, void* arr_d, const int64_t* idx_d,
                           const void* vals_d, double scalar, int64_t k);
/* first-claim-wins conditional store: among entries with arr[idx] ==
 * expected (pre-call state) the earliest occurrence of each index wins and
 * stores vals[i] (or the scalar when vals_d is NULL); pos_d: int64 scratch
 * over the array (n entries) */
GFX_API int gfx_compare_and_swap(gfx_ctx* ctx, int dtype, void* arr_d, const int64_t* idx_d,
                                 int64_t k, int64_t expected, const void* vals_d, int64_t scalar,
                                 uint8_t* won_d, int64_t* pos_d);

/* intersection elements per pair, in pair order, ascending within a pair
 * (IntersectResult.intersections); offsets_d = exclusive scan of counts */
GFX_API int gfx_segmented_intersect_list(gfx_graph* g, const int32_t* u_d, const int32_t* v_d,
                                         int64_t num_pairs, const int64_t* offsets_d,
                                         int32_t* out_d);

/* ---- compressed CSR columns for host<->device transfer ------------------
 * (the PCIe-bound end-to-end path; no reference counterpart -- the
 * reference's GFXCSR cache, io.py:121-159, stores int64 columns).  Zigzag
 * deltas to the previous slot in a StreamVByte-like layout: ctrl_d holds a
 * 2-bit length code per slot ((m+3)/4 bytes), data_d the 1..4 low bytes of
 * each delta, boff_d[b] the data offset of slot block b (1024 slots per
 * block, (m+1023)/1024 + 1 entries).  vals_d: int32 column ids (elem_bytes
 * 4) or int64 row offsets (elem_bytes 8; differences = degrees < 2^31).
 * pack_size fills boff_d and returns the data size; unpack decodes into
 * vals_d; sync = 0 leaves the work enqueued on the ctx stream. */
GFX_API int gfx_csr_pack_size(gfx_ctx* ctx, const void* vals_d, int elem_bytes, int64_t m,
                              int64_t* boff_d, int64_t* data_bytes);
GFX_API int gfx_csr_pack(gfx_ctx* ctx, const void* vals_d, int elem_bytes, int64_t m,
                         const int64_t* boff_d, uint8_t* ctrl_d, uint8_t* data_d);
GFX_API int gfx_csr_unpack(gfx_ctx* ctx, const uint8_t* ctrl_d, const uint8_t* data_d,
                           const int64_t* boff_d, int64_t m, void* vals_d, int elem_bytes,
                           int sync);
/* Rebuild an undirected graph's columns from its upper triangle (each
 * edge once, as the reference's COO input holds it before coo_to_csr
 * symmetrises it, graph.py:158-203): g->row must already hold the full row
 * offsets; urow_d int64[n+1] / ucol_d int32[mu] are the upper triangle's CSR
 * (entries > the row id), mu = m/2.  Writes the full sorted g->col (lower
 * parts by a stable radix-sort transpose); enqueued on the ctx stream, call
 * gfx_graph_refresh after it. */
GFX_API int gfx_graph_rebuild_upper(gfx_graph* g, const int64_t* urow_d, const int32_t* ucol_d,
                                    int64_t mu);

/* ---- bit-exact R-MAT + canonical CSR builder ----------------------------
 * (reference generators.py:22-52, graph.py:158-203, graph.py:227-246)
 * pcg_state/pcg_inc: the numpy PCG64 state of default_rng(seed) as (hi, lo)
 * 64-bit halves.  Phase 1 writes the symmetrised, sorted, unique keys
 * (src<<scale | dst) to keys_d (capacity 2*edge_factor*2^scale) and returns
 * their count; phase 2 turns them into row_d int64[n+1] and col_d int32[m]. */
GFX_API int gfx_rmat_keys(gfx_ctx* ctx, int scale, int edge_factor, const double* cum3,
                  uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                  uint64_t inc_lo, int make_undirected, uint64_t* keys_d,
                  int64_t* num_keys);
GFX_API int gfx_keys_to_csr(gfx_ctx* ctx, const uint64_t* keys_d, int64_t num_keys, int scale,
                    int64_t* row_d, int32_t* col_d);
/* assign_random_weights(g, lo, hi, seed) for a canonical undirected CSR:
 * per undirected pair (u<v) in sorted order, w = lo + bounded(u32 stream). */
GFX_API int gfx_assign_weights(gfx_graph* g, int64_t lo, int64_t hi, uint64_t state_hi,
                       uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                       int32_t* w_d);

/* ---- partitioned multi-GPU BFS (1D cyclic partition) -------
 * Rank r of P owns vertices v = l*P + r (local id l); its local CSR holds
 * the owned rows with GLOBAL column ids.  The host drives the levels and the
 * collectives (allreduce of the level counters, all_to_all of (dst, src)
 * pairs for push levels, all_gather of local frontier bitmaps for pull
 * levels) on buffers it owns and binds here; the direction decision is the
 * reference formula on the global counts (direction.py:52-70).  Undirected
 * graphs only.  Every level entry point only ENQUEUES work on the context
 * stream (no host synchronisation): per-level counts land in the bound
 * device arrays, the host reduces / reads them once per level and hands the
 * rank's new frontier size back with gfx_dbfs_commit. */
typedef struct gfx_dbfs gfx_dbfs;
GFX_API int gfx_dist_partition_sizes(gfx_graph* g, int P, int r, int64_t* n_local,
                                     int64_t* m_local);
GFX_API int gfx_dist_partition(gfx_graph* g, int P, int r, int64_t* lrow_d, int32_t* lcol_d);
GFX_API int gfx_dbfs_create(gfx_ctx* ctx, int64_t n, int64_t m, int P, int r,
                            const int64_t* lrow_d, const int32_t* lcol_d, int64_t n_local,
                            int64_t m_local, gfx_dbfs** out);
GFX_API int gfx_dbfs_destroy(gfx_dbfs* db);
GFX_API int gfx_dbfs_words(gfx_dbfs* db, int64_t* words_local, int64_t* words_max);
/* labels/preds: int32[n_local]; send/recv: uint64 pairs (dst << 32 | src);
 * front_local: uint32[words_max]; gathered: uint32[P * words_max];
 * send_counts: int64[2P]: [0, P) pairs per destination rank (own rank 0),
 * [P, 2P) the counts received from each rank (written by the exchange);
 * stats: int64[8] = {local new frontier, local slots expanded, pull probes,
 * pull candidates} of the last level, written twice (stats[4..7] is the copy
 * the host allreduces in place) */
GFX_API int gfx_dbfs_bind(gfx_dbfs* db, int32_t* labels_d, int32_t* preds_d, void* send_d,
                          int64_t send_cap, void* recv_d, int64_t recv_cap,
                          uint32_t* front_local_d, uint32_t* gathered_d,
                          int64_t* send_counts_d, int64_t* stats_d);
/* *nf_local = 1 if this rank owns the source, else 0 (known on the host) */
GFX_API int gfx_dbfs_reset(gfx_dbfs* db, int64_t source, int64_t* nf_local);
/* push level: expand, claim owned targets, bucket remote (dst, src) pairs
 * into send (grouped by destination rank) and their counts into send_counts */
GFX_API int gfx_dbfs_push_expand(gfx_dbfs* db, int32_t depth);
/* push level, after the all_to_all: claim the nrecv received pairs */
GFX_API int gfx_dbfs_push_claim(gfx_dbfs* db, int64_t nrecv, int32_t depth);
/* pull level: local frontier -> front_local (before the all_gather) */
GFX_API int gfx_dbfs_pull_prepare(gfx_dbfs* db);
/* pull level, after the all_gather into gathered */
GFX_API int gfx_dbfs_pull(gfx_dbfs* db, int32_t depth);
/* end of level: the rank's new frontier size (stats[0] as read by the host) */
GFX_API int gfx_dbfs_commit(gfx_dbfs* db, int64_t nf_local);

/* Native level loop: one whole partitioned BFS from `source` with the
 * per-level protocol above, NCCL called from C++ on the context stream (one
 * host synchronisation per pull level, two per push level).  `comm` may be
 * NULL only when P == 1.  recs (rec_cap records) receives the direction
 * trace; stats the totals (edges_traversed = push slots, bytes_alg,
 * device_ms = CUDA-event time of the whole BFS on this rank). */
typedef struct gfx_nccl gfx_nccl;
/* ---- partitioned near/far SSSP (reference sssp.py:41-121,
 * near_far.py:20-85) --------------------------------------------------------
 * Same 1D cyclic partition as the BFS engine.  Per iteration the host calls
 * relax (expand the local near queue; owned targets relaxed in place, remote
 * ones bucketed as (d, dist<<32|pred) messages of 2 words, send_counts in
 * words), exchanges counts then messages (all_to_all), apply (owners relax
 * the received offers), split (touched -> near / far at the GLOBAL
 * threshold; stats[0..3] = near, far, slots, touched, copied to stats[4..7]
 * for the allreduce).  When the global near count is 0 and far is not,
 * every rank calls refar(threshold + delta, 1, far_local).  Nothing
 * synchronises the host inside relax / apply / split / refar. */
typedef struct gfx_dsssp gfx_dsssp;
GFX_API int gfx_dist_partition_weights(gfx_graph* g, int P, int r, const int64_t* lrow_d,
                                       int32_t* lw_d);
GFX_API int gfx_dsssp_create(gfx_ctx* ctx, int64_t n, int P, int r, const int64_t* lrow_d,
                             const int32_t* lcol_d, const int32_t* lw_d, int64_t n_local,
                             int64_t m_local, gfx_dsssp** out);
GFX_API int gfx_dsssp_destroy(gfx_dsssp* ds);
GFX_API int gfx_dsssp_bind(gfx_dsssp* ds, void* send_d, int64_t send_cap_words, void* recv_d,
                           int64_t recv_cap_words, int64_t* send_counts_d, int64_t* stats_d);
GFX_API int gfx_dsssp_reset(gfx_dsssp* ds, int64_t source, int64_t* near_local);
GFX_API int gfx_dsssp_relax(gfx_dsssp* ds);
GFX_API int gfx_dsssp_apply(gfx_dsssp* ds, int64_t nrecv_words);
GFX_API int gfx_dsssp_split(gfx_dsssp* ds, double threshold);
GFX_API int gfx_dsssp_refar(gfx_dsssp* ds, double threshold, int split, int64_t far_local);
/* local distances (INT32_MAX unreached) and global preds of the owned vertices */
GFX_API int gfx_dsssp_result(gfx_dsssp* ds, int32_t* dist_d, int32_t* preds_d);

/* resolve NCCL from the library already loaded in the process (path: its
 * file, e.g. torch's nvidia/nccl/lib/libnccl.so.2; NULL: by soname) */
GFX_API int gfx_nccl_load(const char* path);
GFX_API int gfx_nccl_unique_id(uint8_t* id_out /* 128 bytes */);
GFX_API int gfx_nccl_comm_create(gfx_ctx* ctx, int nranks, int rank, const uint8_t* id,
                                 gfx_nccl** out);
GFX_API int gfx_nccl_comm_destroy(gfx_nccl* comm);
GFX_API int gfx_dbfs_run(gfx_dbfs* db, gfx_nccl* comm, int64_t source, int direction,
                         double do_a, double do_b, int mu_edge_based, gfx_iter_rec* recs,
                         int64_t rec_cap, gfx_stats* stats);
/* The same loop over a caller-supplied collective table (the NCCL one above
 * is one implementation).  Each callback acts on the buffers bound with
 * gfx_dbfs_bind, ordered on the context stream, and returns 0 on success:
 * exchange_counts fills send_counts[P..2P) from every rank's [0..P);
 * exchange_pairs moves each rank's send buckets (host counts sc[P], rc[P],
 * own rank 0) into the receivers' recv arrays in rank order;
 * allgather_frontier fills gathered from every rank's front_local;
 * allreduce_stats sums stats[4..8) over the ranks in place. */
typedef struct gfx_dbfs_comm {
  void* user;
  int (*exchange_counts)(void* user);
  int (*exchange_pairs)(void* user, const int64_t* send_counts, const int64_t* recv_counts);
  int (*allgather_frontier)(void* user);
  int (*allreduce_stats)(void* user);
} gfx_dbfs_comm;
GFX_API int gfx_dbfs_run_comm(gfx_dbfs* db, const gfx_dbfs_comm* comm, int64_t source,
                              int direction, double do_a, double do_b, int mu_edge_based,
                              gfx_iter_rec* recs, int64_t rec_cap, gfx_stats* stats);

/* ---- device-resident partitioned BFS (SURVEY 8(e) low-latency path) -----
 * Replaces the host-driven level loop of the partitioned BFS (gfx_dbfs_run:
 * one host-launched collective per level) with ONE cooperative launch per
 * rank; ranks exchange frontier slices, (dst, src) claim pairs and level
 * counters through peer memory and device flags.  Same partition (owner(v) =
 * v mod P, local id v / P), same results as gfx_dbfs_run / the reference
 * bfs (primitives/bfs.py:42-159, direction.py:52-70).
 * Virtual ranks: all P ranks run inside one launch on this GPU (CTA b runs
 * rank b mod P) -- the complete multi-rank protocol on one device.
 * lrow / lcol / n_local / m_local: P entries (gfx_dist_partition output). */
typedef struct gfx_pdbfs gfx_pdbfs;
GFX_API int gfx_pdbfs_create_virtual(gfx_ctx* ctx, int64_t n, int64_t m, int P,
                                     const int64_t* const* lrow, const int32_t* const* lcol,
                                     const int64_t* n_local, const int64_t* m_local,
                                     gfx_pdbfs** out);
GFX_API int gfx_pdbfs_destroy(gfx_pdbfs* e);
/* Real ranks, one process per GPU: rank r's engine over its partition.  Its
 * exchange block is shared through CUDA IPC: gfx_pdbfs_export writes 5
 * cudaIpcMemHandle_t (320 bytes); the caller all-gathers them (P x 320
 * bytes, rank-major) and the sum over ranks of gfx_pdbfs_local_nnz
 * (vertices with degree > 0), and every rank calls gfx_pdbfs_import before
 * its first run (at P = 1: with its own handles and count). */
GFX_API int gfx_pdbfs_create_rank(gfx_ctx* ctx, int64_t n, int64_t m, int P, int r,
                                  const int64_t* lrow, const int32_t* lcol, int64_t n_local,
                                  int64_t m_local, gfx_pdbfs** out);
GFX_API int gfx_pdbfs_local_nnz(gfx_pdbfs* e, int64_t* nnz);
GFX_API int gfx_pdbfs_export(gfx_pdbfs* e, void* handles);
GFX_API int gfx_pdbfs_import(gfx_pdbfs* e, const void* all_handles, int64_t nnz_global);

/* One BFS; labels_d[q] / preds_d[q] (optional, int32 device, n_local[q]
 * entries) receive rank q's labels (local ids) and preds (global ids). */
GFX_API int gfx_pdbfs_run(gfx_pdbfs* e, int64_t source, int direction, double do_a, double do_b,
                          int mu_edge_based, int32_t* const* labels_d, int32_t* const* preds_d,
                          gfx_iter_rec* recs, int64_t rec_cap, gfx_stats* stats);
/* count BFS runs back to back (one cooperative launch each); device ms. */
GFX_API int gfx_pdbfs_batch(gfx_pdbfs* e, int64_t source, int64_t count, int direction,
                            double do_a, double do_b, int mu_edge_based, float* ms);

/* ---- device-resident partitioned near/far SSSP (gfx_pdsssp.cu) ----------
 * The low-latency form of the partitioned SSSP (gfx_dsssp: host-driven, one
 * host-launched collective per step): one cooperative launch per rank;
 * (d, dist << 32 | pred) offers stored into the owners' inboxes, level
 * counters into every rank's table, flag barriers.  Reference sssp.py:41-121,
 * near_far.py:20-85.  lw: the ranks' weights aligned with their local rows
 * (gfx_dist_partition_weights).  Virtual ranks: all P inside one launch on
 * this GPU; real ranks: one process per GPU, exchange block shared through
 * CUDA IPC (export: 4 handles, 256 bytes; import: P x 256 bytes). */
typedef struct gfx_pdsssp gfx_pdsssp;
GFX_API int gfx_pdsssp_create_virtual(gfx_ctx* ctx, int64_t n, int P, const int64_t* const* lrow,
                                      const int32_t* const* lcol, const int32_t* const* lw,
                                      const int64_t* n_local, const int64_t* m_local,
                                      gfx_pdsssp** out);
GFX_API int gfx_pdsssp_create_rank(gfx_ctx* ctx, int64_t n, int P, int r, const int64_t* lrow,
                                   const int32_t* lcol, const int32_t* lw, int64_t n_local,
                                   int64_t m_local, gfx_pdsssp** out);
GFX_API int gfx_pdsssp_export(gfx_pdsssp* e, void* handles);
GFX_API int gfx_pdsssp_import(gfx_pdsssp* e, const void* all_handles);
GFX_API int gfx_pdsssp_destroy(gfx_pdsssp* e);
/* delta <= 0: one bucket (infinite width).  dist_d[k] / preds_d[k]: rank k's
 * (virtual) or this rank's (real: k = 0) int32 outputs over local ids. */
GFX_API int gfx_pdsssp_run(gfx_pdsssp* e, int64_t source, double delta, int32_t* const* dist_d,
                           int32_t* const* preds_d, gfx_iter_rec* recs, int64_t rec_cap,
                           gfx_stats* stats);
GFX_API int gfx_pdsssp_batch(gfx_pdsssp* e, int64_t source, int64_t count, double delta,
                             float* ms);

/* ---- kernel experiments (tools/expand_lab.py; not a product path) -------
 * One LB expansion of F_d with functor variant 0 (stream only), 1 (stream +
 * visited probe) or 2 (full claim); visited = {labels < depth}. */
/* Diagnostics: microseconds per grid-wide barrier (variant 0: cooperative
 * groups grid sync, 1: flag barrier, 2: grid sync + every thread reads four
 * counters on one line, 3: grid sync + one read per CTA) for a cooperative
 * grid of blocks x threads. */
GFX_API int gfx_debug_gridsync(gfx_ctx* ctx, int variant, int blocks, int threads, int iters,
                               float* us_per_sync);
/* Diagnostic: ns per same-address atomic (variant 0 returned, 1 RED, 2 own
 * line per warp), one atomic per warp per iteration over blocks x 256. */
GFX_API int gfx_debug_atomics(gfx_ctx* ctx, int variant, int blocks, int iters,
                              double* ns_per_atomic);
/* Diagnostics: clock cycles per dependent load, chasing next = buf[next]
 * (uint32 words, device buffer prepared by the caller) from `start`. */
GFX_API int gfx_debug_chase(gfx_ctx* ctx, const uint32_t* buf_d, int iters, uint32_t start,
                            double* cycles_per_load);
GFX_API int gfx_debug_expand(gfx_graph* g, const int32_t* F_d, int64_t nf, int variant,
                             int32_t* labels_d, int32_t depth, float* ms, int64_t* out_count);

#ifdef __cplusplus
}
#endif
#endif /* GFX_H */
