/*
 * nextdoor_b200.h — C-ABI of the B200 transit-parallel sampling engine.
 *
 * The drop-in boundary for the reference `trawl` sampling path
 * (/root/reference/pkg/src/trawl).  Two nested levels, as in the reference:
 *
 *  Level 1 — the kernel-backend ABI that `trawl.kernels` exposes
 *  (kernels/__init__.py:29-44) and that _kernel_pairs / _kernel_exec / _batch
 *  call (transit_parallel.py:111-120, sample_parallel.py:43-53, chain.py:43-61):
 *      nd_individual_batch      <- individual_batch   (_ckernels.pyx:136-271)
 *      nd_segmented_prefix_sum  <- segmented_prefix_sum (_ckernels.pyx:103-116)
 *      nd_segment_max           <- segment_max        (_ckernels.pyx:119-133)
 *      nd_keyed_u64             <- keyed_u64          (_pykernels.py:61-68)
 *
 *  Level 2 — the engine entry `tp_run/sp_run(app, graph, samples, config)`
 *  (transit_parallel.py:249-257, sample_parallel.py:102-110), split into
 *      nd_graph_*               <- Graph / from_edges (graph.py:36-129)
 *      nd_run_walk              <- run_chain          (chain.py:64-164)
 *      nd_run_individual        <- run_loop + tp_step (driver.py:203-235,
 *                                  transit_parallel.py:185-230)
 *      nd_run_collective        <- tp_step collective branch +
 *                                  build_combined/collective_select
 *                                  (transit_parallel.py:187-198, collective.py:39-141)
 *      nd_transit_schedule      <- build_transit_map + partition_work_classes
 *                                  (transit_parallel.py:71-101)
 *      nd_result_*              <- SampleSetOutput fields (output.py:43-69)
 *
 * Conventions: plain pointers and sizes only.  Pointers are DEVICE pointers
 * unless a name says `host_`.  `stream` is a cudaStream_t passed as void*
 * (NULL = legacy default stream).  Every entry returns an int status; the
 * Python shim maps them onto the reference's exceptions:
 *      ND_ERR_STALL -> SamplerStallError (_ckernels.pyx:263-269)
 *      ND_ERR_APP   -> ValueError("unknown app code") (_ckernels.pyx:270-271)
 *      ND_ERR_ARG   -> ValueError, ND_ERR_CUDA -> DeviceError
 * Calls are re-entrant; a graph handle is read-only after creation and may
 * be shared by concurrent runs on different streams.
 */
#ifndef NEXTDOOR_B200_H
#define NEXTDOOR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ND_OK 0
#define ND_ERR_STALL 1
#define ND_ERR_APP 2
#define ND_ERR_ARG 3
#define ND_ERR_CUDA 4
#define ND_ERR_NOMEM 5
#define ND_ERR_EMPTY 6 /* no edges (EmptyGraphError, graph.py:178-179) */

/* individual app codes (kernels/_pykernels.py:32-36) */
#define ND_DEEPWALK 0
#define ND_PPR 1
#define ND_NODE2VEC 2
#define ND_KHOP 3
#define ND_MULTIRW 4

/* collective app kinds (apps.py:247-386) */
#define ND_LAYER 0
#define ND_IMPORTANCE 1 /* fastgcn / ladies */
#define ND_MVS 2
#define ND_CLUSTERGCN 3

/* paradigms (bench.py:91-96 --paradigm) */
#define ND_SP 0
#define ND_TP 1

typedef struct nd_graph nd_graph;
typedef struct nd_result nd_result;
typedef struct nd_ooc_graph nd_ooc_graph;
typedef struct nd_khop_plan nd_khop_plan;

/* last error text of this thread (for the Python shim) */
const char *nd_last_error(void);
int nd_version(void);
/* cudaMemcpyDefault copy helper for bindings without a CUDA runtime of their
 * own (synchronous when stream is NULL) */
int nd_copy(void *dst, const void *src, int64_t bytes, void *stream);

/* ---- level 1: kernel backend (_ckernels.pyx:103-271) --------------------- */
/* Sequential per-segment inclusive f64 prefix (bit-identical to the Cython
 * loop; one thread owns a segment). */
int nd_segmented_prefix_sum(const double *values, const int64_t *offsets,
                            int64_t n_segments, double *out, void *stream);
/* Per-segment max, 0.0 for empty segments. */
int nd_segment_max(const double *values, const int64_t *offsets,
                   int64_t n_segments, double *out, void *stream);
/* individual_batch over the reference's own array layout (int64 CSR, f64
 * weights/prefix/max, int64 item arrays).  seed is the reference's
 * `seed & (2^64-1)`.  Writes out[i] or -1.  Returns ND_ERR_APP for an unknown
 * code (before any work), ND_ERR_STALL on a node2vec cap hit. */
int nd_individual_batch(int app_code, const double *host_params, int64_t n_params,
                        const int64_t *row_offsets, const int64_t *col_indices,
                        const double *weights, const double *weight_prefix,
                        const double *max_weight, const int64_t *transits,
                        const int64_t *t_prev, const int64_t *sample_ids,
                        const int64_t *transit_idxs, const int64_t *slots, int64_t n,
                        uint64_t seed, int64_t step, int64_t *out, void *stream);
/* out[i] = u[i] % d[i] with the engine's exact fp64-assisted modulo (fuzz hook) */
int nd_mod_u64(const uint64_t *u, const uint64_t *d, int64_t n, uint64_t *out, void *stream);
/* keyed_u64 over id arrays (transit_idxs/slots may be NULL = zeros). */
int nd_keyed_u64(uint64_t seed, const int64_t *sample_ids, int64_t step,
                 const int64_t *transit_idxs, const int64_t *slots, int64_t domain,
                 int64_t draw, int64_t n, uint64_t *out, void *stream);

/* ---- level 2: graph residency (graph.py:36-129) ------------------------------ */
/* Device CSR from reference-layout arrays (host or device pointers, flag
 * `arrays_on_host`).  weights may be NULL (unit).  prefix/max are computed on
 * device when NULL.  Columns are stored int32 (requires V < 2^31). */
int nd_graph_create(const int64_t *row_offsets, const int64_t *col_indices,
                    const double *weights, const double *weight_prefix,
                    const double *max_weight, int64_t n_vertices, int64_t n_edges,
                    int arrays_on_host, void *stream, nd_graph **out);
/* Build on device from an edge list (from_edges semantics: stable lexsort
 * by (src, dst); parallel edges stay in input order). */
int nd_graph_from_edges(const int64_t *src, const int64_t *dst, const double *weights,
                        int64_t n_edges, int64_t n_vertices, void *stream,
                        nd_graph **out);
/* Edge-list ingestion on device (load_edge_list, graph.py:132-188), in three
 * calls.  nd_text_parse uploads the file's bytes and parses every line on
 * device (universal newlines, '#' comments, 2 or 3 whitespace-separated
 * fields, int/float with Python's grammar, keyed default weights).
 * host_info[4] = {n_lines, first malformed line (1-based, 0 = none), its error
 * code (1 fields, 2 id, 3 negative id, 4 weight, 5 negative weight), number
 * of lines left to the host}.  Lines left to the host (non-ASCII bytes, or
 * numbers the device cannot convert bit-exactly) are listed by
 * nd_text_host_lines (0-based line indexes, ascending; byte bounds via
 * nd_text_line_bounds); the caller parses them with the reference rules and
 * passes the results to nd_text_finish (kind 0 skip / 1 edge), which builds
 * the device CSR with ids compacted onto [0, n) (nd_text_remap: the original
 * ids).  ND_ERR_EMPTY when no line holds an edge. */
typedef struct nd_text nd_text;
int nd_text_parse(const char *host_text, int64_t n_bytes, int weighted, double lo_w, double hi_w,
                  uint64_t seed, void *stream, nd_text **out, int64_t *host_info);
/* the same over bytes already in device memory (caller-owned, read-only) */
int nd_text_parse_device(const char *dev_text, int64_t n_bytes, int weighted, double lo_w,
                         double hi_w, uint64_t seed, void *stream, nd_text **out,
                         int64_t *host_info);
int nd_text_host_lines(const nd_text *t, int64_t *host_lines);
int nd_text_line_bounds(const nd_text *t, int64_t line_index, int64_t *host_lo_hi);
int nd_text_finish(nd_text *t, const int64_t *host_line, const int64_t *host_src,
                   const int64_t *host_dst, const double *host_w, const uint8_t *host_kind,
                   int64_t n_patch, int undirected, void *stream, nd_graph **out,
                   int64_t *n_vertices);
int nd_text_remap(const nd_text *t, int64_t *host_remap);
int nd_text_destroy(nd_text *t);
/* Keyed RMAT graph generated and built on device. */
int nd_graph_rmat(int scale, int64_t n_edges, uint32_t ta, uint32_t tab, uint32_t tabc,
                  uint64_t seed, int undirected, int weighted, void *stream,
                  nd_graph **out);
int nd_graph_destroy(nd_graph *g);
/* A graph whose column / weight / prefix arrays stay in (page-locked) host
 * memory and are read in place over the host link (zero copy); row offsets
 * and per-row maxima are device-resident and no index is built.  The
 * out-of-core path for apps the partition shuttle does not run (node2vec,
 * MultiRW, the collective apps): rows identical to a resident graph's.
 * weights / prefix both NULL for unit weights.  Host arrays stay owned by
 * the caller and alive until nd_graph_destroy. */
int nd_graph_create_mapped(const int64_t *row_offsets, const int32_t *col, const double *weights,
                           const double *prefix, int64_t n_vertices, int64_t n_edges,
                           void *stream, nd_graph **out);
/* Build the exact search indexes (flags: 1 = node2vec membership hash sets,
 * 2 = weighted-pick guide tables).  nd_run_walk builds what it needs on first
 * use; answers are identical to the reference's binary searches. */
int nd_graph_build_index(nd_graph *g, int flags, void *stream);
/* sizes and device pointers (read-only views) */
int nd_graph_info(const nd_graph *g, int64_t *n_vertices, int64_t *n_edges, int *unit_weights,
                  int64_t *bytes);
/* HBM footprint: CSR bytes at creation, bytes of the lazily built indexes and
 * records, host time spent building them (ms), and bit sets of the structures
 * built / left out for lack of room (1 vrec, 2 nbw, 4 nbp, 8 nbu, 16 guide,
 * 32 hset, 64 pick lines).  A left-out structure means the kernels read the
 * plain CSR instead: same answers, more dependent reads. */
int nd_graph_footprint(const nd_graph *g, int64_t *csr_bytes, int64_t *index_bytes,
                       double *prep_ms, int *built, int *skipped);
int nd_graph_arrays(const nd_graph *g, const int64_t **row_offsets, const int32_t **col,
                    const double **weights, const double **prefix, const double **max_w);

/* ---- level 2: engine runs ------------------------------------------------------ */
/* Keyed roots (apps.py:83-103): count per sample, distinct when V >= count. */
int nd_uniform_roots(const nd_graph *g, int64_t count, uint64_t seed, int64_t sample_lo,
                     int64_t n_samples, int64_t *roots, void *stream);

/* Chain walks: DeepWalk / PPR / node2vec / MultiRW (chain.py:64-179).
 * roots: device int64 [n_samples * roots_per_sample] or NULL for the keyed
 * default roots.  steps < 0 means INF (capped at step_cap). */
int nd_run_walk(const nd_graph *g, int app_code, const double *host_params, int64_t n_params,
                int64_t sample_lo, int64_t n_samples, const int64_t *roots,
                int64_t roots_per_sample, uint64_t seed, int64_t steps, int64_t step_cap,
                int paradigm, void *stream, nd_result **out);

/* Multi-slot individual apps (k-hop) through the run loop: fanouts[n_steps]
 * (host array).  roots: device int64 [n_samples * roots_per_sample] or NULL.
 * host_unique[s] != 0 marks unique() steps (finish_step dedup, driver.py:
 * 165-172; steps >= n_unique repeat the last flag; NULL = none). */
int nd_run_individual(const nd_graph *g, int app_code, const double *host_params,
                      int64_t n_params, const int64_t *host_fanouts, int64_t n_fanouts,
                      int64_t sample_lo, int64_t n_samples, const int64_t *roots,
                      int64_t roots_per_sample, uint64_t seed, int64_t step_cap,
                      int paradigm, const uint8_t *host_unique, int64_t n_unique,
                      void *stream, nd_result **out);

/* Collective apps (layer / fastgcn / ladies / mvs / clustergcn).
 * roots_off[n+1] / roots (device, ragged) or NULL for the app's keyed default
 * roots (batch_size roots, or ClusterGCN clusters). */
int nd_run_collective(const nd_graph *g, int kind, int64_t step_size, int64_t max_size,
                      int distribution, int64_t steps, int64_t batch_size,
                      int64_t clusters_per_sample, int64_t num_clusters,
                      int64_t sample_lo, int64_t n_samples, const int64_t *roots_off,
                      const int64_t *roots, uint64_t seed, int64_t step_cap,
                      const uint8_t *host_unique, int64_t n_unique, void *stream,
                      nd_result **out);

/* build_transit_map + partition_work_classes for one step's pairs (device
 * int64 pair_transit[n], sample-major).  Outputs (device, caller-allocated,
 * size n / n+1): order (member pair ids, group-major), group_start[G+1],
 * group_transit[G], group_class[G] (0 small,1 medium,2 large),
 * sched_index[G] (rank within class, transit-ascending); *n_groups = G. */
int nd_transit_schedule(const int64_t *pair_transit, int64_t n_pairs, int64_t m,
                        int64_t *order, int64_t *group_start, int64_t *group_transit,
                        int32_t *group_class, int64_t *sched_index, int64_t *n_groups,
                        void *stream);

/* ---- results (output.py:43-69) ----------------------------------------------------
 * A result owns device buffers.  Field ids for nd_result_field: */
#define ND_F_FINAL_OFF 0   /* int64 [n+1] final-layout row offsets          */
#define ND_F_FINAL_IDS 1   /* int64 [total] roots + non-NULL sampled ids
                           (derived from ND_F_FINAL_IDS32 on first request) */
#define ND_F_ROOTS 2       /* int64 [n*R] (walks) / ragged (others) roots  */
#define ND_F_ROOTS_OFF 3   /* int64 [n+1]                                  */
#define ND_F_CHAIN_LEN 4   /* int64 [n] walk chain lengths (NULL included) */
#define ND_F_STEP_COUNTS 5 /* int64 [S*n] slots per sample per step        */
#define ND_F_STEP_VALS 6   /* int64 step-major slot values (NULLs kept)    */
#define ND_F_REC_COUNTS 7  /* int64 [S*n] recorded edges per sample/step   */
#define ND_F_REC_T 8       /* int64 recorded edge sources (step-major)     */
#define ND_F_REC_V 9       /* int64 recorded edge targets                  */
#define ND_F_STATS 10      /* int64 [S*4] {small, medium, large, fetches}  */
#define ND_F_CHAIN_VALS 11 /* int64 walk chains incl. NULL (multirw)       */
#define ND_F_FINAL_IDS32 12 /* int32 [total] the final ids as every run writes them */
#define ND_F_STEP_VALS32 13 /* int32 step-major slot values (k-hop runs write these;
                               ND_F_STEP_VALS is derived from them on request) */
int nd_result_info(const nd_result *r, int64_t *n_samples, int64_t *n_steps,
                   int64_t *total_sampled, int64_t *total_recorded);
/* device pointer + element count of one field (ptr NULL if absent) */
int nd_result_field(const nd_result *r, int field, const void **ptr, int64_t *count);
/* counters: {items, pairs, n2v_tries, n2v_probes, search, pair_bytes,
 * slot_bytes (SURVEY 8(d) model bytes), steps, launches, rand_sectors (random
 * 32-byte sector reads the walk kernels issued), tp_staged (TP walks: hub
 * members stepped from a row staged in shared memory), tp_inplace (TP walks:
 * small-class and grid-tier walkers stepped from global rows)} */
int nd_result_counters(const nd_result *r, int64_t *host_counters, int64_t n);
/* Ensure ND_F_FINAL_IDS32 (int32 final ids; vertex ids < 2^31, the device
 * CSR's column width).  Every run now writes it directly, so this is a no-op
 * kept for callers of the round-1 ABI. */
int nd_result_narrow_ids(nd_result *r, void *stream);
/* copy a field into caller memory (host or device; cudaMemcpyDefault) on
 * `stream`; synchronous when stream is NULL */
int nd_result_copy(const nd_result *r, int field, void *dst, void *stream);
/* event-timed phases when nd_set_profiling(1): {schedule_ms, sample_ms,
 * compaction_ms, 0} */
int nd_result_profile(const nd_result *r, double *ms, int64_t n);
/* Per-step event times when nd_set_profiling(1) was on during the run
 * (StepTiming.build_s / sample_s, driver.py:42-48, transit_parallel.py:204-228):
 * build = the step's transit->sample inversion / scheduling index, sample =
 * its sampling kernels.  *n_out = the number of timed steps (0 for the
 * walker-major SP walk kernel, which has no step boundaries); up to n_max are
 * written. */
int nd_result_step_times(const nd_result *r, double *build_ms, double *sample_ms, int64_t n_max,
                         int64_t *n_out);
int nd_set_profiling(int on);
/* Runs started by the calling host thread share the GPU with k-1 concurrent
 * runs (one host thread per job): persistent walk kernels launch 1/k of every
 * SM's CTA slots, so the jobs run side by side instead of queueing behind
 * each other's persistent grids.  Thread-local; k = 1 (default): whole GPU. */
int nd_set_concurrency(int k);
/* Text rows (output.py:72-92 render_text, remap output.py:145-150) printed
 * on the device: one line "<sample id>: <v0> <v1> ..." per row of the CSR
 * (off [n+1], ids int32 or int64 by id_bytes, sample_ids [n], remap
 * [max id + 1] or NULL), all device pointers.  host_out NULL: only the text's
 * byte length in *text_len; else the text (no terminating NUL) into host_out
 * of cap >= *text_len bytes. */
int nd_format_rows(const int64_t *off, const void *ids, int id_bytes, const int64_t *sample_ids,
                   int64_t n, const int64_t *remap, void *stream, char *host_out, int64_t cap,
                   int64_t *text_len);
/* Return the stream-ordered allocation pool's unused memory beyond `keep`
 * bytes to the device (between large jobs). */
int nd_pool_trim(int64_t keep);
/* Measured ceiling of dependent random 32-byte sector reads (sectors/s): one
 * pointer-chasing chain per thread, ctas_per_sm x 256 threads per SM, over a
 * `bytes` buffer (rounded down to a power of two).  The roofline a
 * gather-bound walk kernel actually faces (nd_probe.cu). */
int nd_gather_ceiling(int64_t bytes, int ctas_per_sm, int iters, double *sectors_per_s,
                      void *stream);
/* Dense final rows, the frontend's getFinalSamples (frontend/src/index.ts:
 * 160-171): out[n * width] int32 (device), row i = roots then sampled
 * vertices, padded with -1.  nd_result_max_row gives the natural width. */
int nd_result_max_row(const nd_result *r, int64_t *host_width);
int nd_result_dense(const nd_result *r, int64_t width, int32_t *out, void *stream);
int nd_result_destroy(nd_result *r);

/* ---- out-of-core sub-graph shuttling ------
 * A graph that does not fit the device stays in host memory (caller-owned
 * arrays, kept alive until destroy): int64 row offsets [V+1], int32 columns
 * [E], and the f64 inclusive per-row prefix [E] (NULL: unit weights).  Its
 * vertices are cut into contiguous partitions whose slices fit half of
 * `device_budget_bytes` after the resident row offsets; register_host
 * page-locks the column / prefix arrays for async uploads.  ND_ERR_NOMEM when
 * the budget cannot hold two slices of the largest row. */
int nd_ooc_graph_create(const int64_t *row_offsets, const int32_t *col, const double *prefix,
                        int64_t n_vertices, int64_t n_edges, int64_t device_budget_bytes,
                        int register_host, void *stream, nd_ooc_graph **out);
int nd_ooc_graph_destroy(nd_ooc_graph *g);
/* partitions, edges per slice buffer, device bytes held, host->device slice
 * bytes shuttled so far, slice uploads so far */
int nd_ooc_graph_info(const nd_ooc_graph *g, int64_t *n_parts, int64_t *slice_edges,
                      int64_t *device_bytes, int64_t *bytes_shuttled, int64_t *uploads);
/* vertex cut points [n_parts + 1] */
int nd_ooc_graph_parts(const nd_ooc_graph *g, int64_t *vcut, int64_t n_max);
/* DeepWalk (steps = walk length) or PPR (steps = the step cap; host_params =
 * {termination probability}) over a shuttled graph (others ND_ERR_APP): same
 * rows as nd_run_walk.  roots: device int64 [n] or NULL (keyed roots). */
int nd_run_walk_ooc(nd_ooc_graph *g, int app_code, const double *host_params, int64_t n_params,
                    int64_t sample_lo, int64_t n_samples, const int64_t *roots, uint64_t seed,
                    int64_t steps, void *stream, nd_result **out);
/* k-hop (ND_KHOP; others ND_ERR_APP) over a shuttled graph: same rows as
 * nd_run_individual. */
int nd_run_individual_ooc(nd_ooc_graph *g, int app_code, const int64_t *host_fanouts,
                          int64_t n_fanouts, int64_t sample_lo, int64_t n_samples,
                          const int64_t *roots, uint64_t seed, void *stream, nd_result **out);

/* ---- k-hop minibatch plans (CUDA graphs) -------------------------------------
 * GraphSAGE-style sampling of many equal-size batches (driver.py:203-235 per
 * batch, SURVEY §8(d) C3's 1,024-root batches): the fixed-layout SP k-hop run
 * for n samples captured once into a CUDA graph over preallocated buffers;
 * each batch is then a device parameter write, an optional roots copy and
 * one graph launch, with no allocation and no host synchronisation.  Rows
 * equal nd_run_individual's for the same roots and sample ids. */
int nd_khop_plan_create(const nd_graph *g, const int64_t *host_fanouts, int64_t n_fanouts,
                        int64_t n_samples, void *stream, nd_khop_plan **out);
/* roots: device int64 [n] copied into the plan (NULL: the plan's own roots
 * buffer, nd_khop_plan_outputs, was filled by the caller); asynchronous. */
int nd_khop_plan_run(nd_khop_plan *p, const int64_t *roots, int64_t sample_lo, uint64_t seed,
                     void *stream);
/* device views: the plan's roots buffer, final offsets [n+1] (total =
 * final_off[n]), final ids (capacity *cap), and each step's block
 * (int32 [n * B], NULL slots -1) with its size */
int nd_khop_plan_outputs(const nd_khop_plan *p, int64_t **roots, const int64_t **final_off,
                         const int32_t **final_ids, int64_t *cap, const int32_t **blocks,
                         int64_t *block_sizes, int64_t n_max);
int nd_khop_plan_destroy(nd_khop_plan *p);

#ifdef __cplusplus
}
#endif
#endif
