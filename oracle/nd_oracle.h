/*
 * nd_oracle.h — CPU oracle for the NextDoor/trawl sampling hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under paper_2009_06693_b200/ may link,
 * import or call this code; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg use it, and only as the
 * checker or the timed CPU baseline.  It is a plain-C restatement of the
 * reference algorithm (trawl, /root/reference/pkg/src/trawl), each function
 * citing the reference file:line it follows.  Parity is pinned against the
 * reference's own known-answer values and golden hashes (tests/golden/).
 */
#ifndef ND_ORACLE_H
#define ND_ORACLE_H
#include <stdint.h>

#define NDO_OK 0
#define NDO_ERR_STALL 1
#define NDO_ERR_APP 2
#define NDO_ERR_ARG 3
#define NDO_ERR_NOMEM 4

/* app codes: trawl/kernels/_pykernels.py:32-36 */
#define NDO_DEEPWALK 0
#define NDO_PPR 1
#define NDO_NODE2VEC 2
#define NDO_KHOP 3
#define NDO_MULTIRW 4

/* collective app kinds (apps.py:247-386) */
#define NDO_C_LAYER 0
#define NDO_C_IMPORTANCE 1
#define NDO_C_MVS 2
#define NDO_C_CLUSTERGCN 3

uint64_t ndo_key_u64(uint64_t seed, int64_t sample_id, int64_t step,
                     int64_t transit_idx, int64_t slot, int64_t domain,
                     int64_t draw);
double ndo_key_uniform(uint64_t seed, int64_t sample_id, int64_t step,
                       int64_t transit_idx, int64_t slot, int64_t domain,
                       int64_t draw);
void ndo_keyed_u64_batch(uint64_t seed, const int64_t *sample_ids, int64_t step,
                         const int64_t *transit_idxs, const int64_t *slots,
                         int64_t domain, int64_t draw, int64_t n, uint64_t *out);

void ndo_segmented_prefix_sum(const double *values, const int64_t *offsets,
                              int64_t n_segments, double *out);
void ndo_segment_max(const double *values, const int64_t *offsets,
                     int64_t n_segments, double *out);

int ndo_individual_batch(int app_code, const double *params, int64_t n_params,
                         const int64_t *row_offsets, const int64_t *col_indices,
                         const double *weights, const double *weight_prefix,
                         const double *max_weight, const int64_t *transits,
                         const int64_t *t_prev, const int64_t *sample_ids,
                         const int64_t *transit_idxs, const int64_t *slots,
                         int64_t n, uint64_t seed, int64_t step, int64_t *out);

void ndo_uniform_roots(int64_t n_vertices, int64_t count, uint64_t seed,
                       int64_t sample_lo, int64_t n_samples, int64_t *roots);

/* returns the number of roots written for one clustergcn sample; roots may
 * be NULL to query the count. */
int64_t ndo_cluster_roots(int64_t n_vertices, int64_t clusters_per_sample,
                          int64_t num_clusters, uint64_t seed, int64_t sample_id,
                          int64_t *roots);

void ndo_free(void *p);

/* chain walks (engine/chain.py:64-179).  roots is n*R (mutated in place for
 * root-pick apps).  chain output: chain_len[n], *chain_vals (malloc'd,
 * concatenated per sample, NULLs included).  stats: per step
 * {small, medium, large, fetches} (malloc'd, n_steps*4). */
int ndo_run_chain(const int64_t *row_offsets, const int64_t *col_indices,
                  const double *weights, const double *weight_prefix,
                  const double *max_weight, int64_t n_vertices, int app_code,
                  const double *params, int64_t n_params, int64_t sample_lo,
                  int64_t n, int64_t *roots, int64_t R, uint64_t seed,
                  int64_t steps, int64_t step_cap, int paradigm, int n_threads,
                  int64_t *chain_len, int64_t **chain_vals,
                  int64_t *n_steps_out, int64_t **stats_out);

/* generic individual run loop (engine/driver.py:203-235 + tp_step). */
int ndo_run_individual(const int64_t *row_offsets, const int64_t *col_indices,
                       const double *weights, const double *weight_prefix,
                       const double *max_weight, int64_t n_vertices, int app_code,
                       const double *params, int64_t n_params,
                       const int64_t *fanouts, int64_t n_fanouts,
                       int root_pick, int needs_prev2, int64_t sample_lo,
                       int64_t n, const int64_t *roots_off, int64_t *roots,
                       uint64_t seed, int64_t steps, int64_t step_cap,
                       int paradigm, const uint8_t *unique_mask, int64_t n_mask,
                       int64_t *n_steps_out,
                       int64_t **step_counts, int64_t **vals, int64_t *n_vals,
                       int64_t **stats_out);

/* collective run loop (transit_parallel.py:187-198, collective.py). */
int ndo_run_collective(const int64_t *row_offsets, const int64_t *col_indices,
                       int64_t n_vertices, int kind, int64_t step_size,
                       int64_t max_size, int distribution, int64_t sample_lo,
                       int64_t n, const int64_t *roots_off, const int64_t *roots,
                       uint64_t seed, int64_t steps, int64_t step_cap,
                       const uint8_t *unique_mask, int64_t n_mask,
                       int64_t *n_steps_out, int64_t **step_counts,
                       int64_t **vals, int64_t *n_vals, int64_t **rec_counts,
                       int64_t **rec_t, int64_t **rec_v, int64_t *n_rec,
                       int64_t **stats_out);

/* build_transit_map + partition_work_classes (transit_parallel.py:71-101). */
int64_t ndo_transit_schedule(const int64_t *pair_transit, int64_t n_pairs,
                             int64_t m, int64_t *order, int64_t *group_start,
                             int64_t *group_transit, int32_t *group_class,
                             int64_t *sched_index);

/* keyed RMAT edge generator + CSR build (from_edges semantics, graph.py:107-129) */
void ndo_rmat_edges(int scale, int64_t n_edges, uint32_t ta, uint32_t tab,
                    uint32_t tabc, uint64_t seed, int undirected, int weighted,
                    int64_t *src, int64_t *dst, double *w);
int ndo_from_edges(const int64_t *src, const int64_t *dst, const double *w,
                   int64_t n_edges, int64_t n_vertices, int64_t *row_offsets,
                   int64_t *col_indices, double *weights_out);

#endif
