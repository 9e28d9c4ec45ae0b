/*
 * nd_oracle.c — CPU oracle (TEST INFRASTRUCTURE; see nd_oracle.h).
 *
 * A plain-C restatement of the reference trawl sampling path.  Every
 * function cites the reference lines it restates.  This file is the checker
 * for the CUDA engine and the timed CPU baseline in bench.py; it is never
 * linked into the product library.
 */
#include "nd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* rng.py:22-30 */
#define K_SAMPLE 0x9E3779B97F4A7C15ull
#define K_STEP 0xC2B2AE3D27D4EB4Full
#define K_TRANSIT 0x165667B19E3779F9ull
#define K_SLOT 0x27D4EB2F165667C5ull
#define K_DOMAIN 0x85EBCA77C2B2AE63ull
#define K_DRAW 0xD6E8FEB86659FD93ull
#define K_MIXA 0xBF58476D1CE4E5B9ull
#define K_MIXB 0x94D049BB133111EBull
static const double TWO_M53 = 1.0 / 9007199254740992.0;

#define NULLV (-1)
#define N2V_MAX_TRIES 1000000L /* apps.py:35 */
#define SMALL_MAX_WORK 32      /* transit_parallel.py:37 */
#define LARGE_MIN_WORK 1024    /* transit_parallel.py:38 */

/* rng.py:43-49 (splitmix64 finalizer) */
static inline uint64_t fin64(uint64_t z) {
  z = (z ^ (z >> 30)) * K_MIXA;
  z = (z ^ (z >> 27)) * K_MIXB;
  return z ^ (z >> 31);
}

/* rng.py:52-71: Weyl sum of the key fields, finalised twice */
uint64_t ndo_key_u64(uint64_t seed, int64_t sample_id, int64_t step,
                     int64_t transit_idx, int64_t slot, int64_t domain,
                     int64_t draw) {
  uint64_t k = seed;
  k += K_SAMPLE * ((uint64_t)sample_id + 1u);
  k += K_STEP * ((uint64_t)step + 1u);
  k += K_TRANSIT * ((uint64_t)transit_idx + 1u);
  k += K_SLOT * ((uint64_t)slot + 1u);
  k += K_DOMAIN * ((uint64_t)domain + 1u);
  k += K_DRAW * ((uint64_t)draw + 1u);
  return fin64(fin64(k));
}

static inline double unit53(uint64_t u) { return (double)(u >> 11) * TWO_M53; }

/* rng.py:74-77 */
double ndo_key_uniform(uint64_t seed, int64_t sample_id, int64_t step,
                       int64_t transit_idx, int64_t slot, int64_t domain,
                       int64_t draw) {
  return unit53(ndo_key_u64(seed, sample_id, step, transit_idx, slot, domain, draw));
}

/* kernels/_pykernels.py:61-68 (keyed_u64 over id arrays) */
void ndo_keyed_u64_batch(uint64_t seed, const int64_t *sample_ids, int64_t step,
                         const int64_t *transit_idxs, const int64_t *slots,
                         int64_t domain, int64_t draw, int64_t n, uint64_t *out) {
  for (int64_t i = 0; i < n; i++)
    out[i] = ndo_key_u64(seed, sample_ids[i], step, transit_idxs ? transit_idxs[i] : 0,
                         slots ? slots[i] : 0, domain, draw);
}

/* _ckernels.pyx:103-116 — sequential accumulation per segment */
void ndo_segmented_prefix_sum(const double *values, const int64_t *offsets,
                              int64_t n_segments, double *out) {
  for (int64_t v = 0; v < n_segments; v++) {
    double acc = 0.0;
    for (int64_t i = offsets[v]; i < offsets[v + 1]; i++) {
      acc += values[i];
      out[i] = acc;
    }
  }
}

/* _ckernels.pyx:119-133 — 0.0 for an empty segment */
void ndo_segment_max(const double *values, const int64_t *offsets,
                     int64_t n_segments, double *out) {
  for (int64_t v = 0; v < n_segments; v++) {
    double best = 0.0;
    for (int64_t i = offsets[v]; i < offsets[v + 1]; i++)
      if (i == offsets[v] || values[i] > best) best = values[i];
    out[v] = best;
  }
}

/* _ckernels.pyx:65-74: first index in [lo,hi) with a[i] > x */
static inline int64_t first_greater(const double *a, int64_t lo, int64_t hi, double x) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

/* _ckernels.pyx:77-87 / graph.py:78-81: membership in a sorted segment */
static inline int sorted_has(const int64_t *a, int64_t lo, int64_t hi, int64_t t) {
  int64_t end = hi;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < t) lo = mid + 1; else hi = mid;
  }
  return lo < end && a[lo] == t;
}

typedef struct {
  const int64_t *row;
  const int64_t *col;
  const double *w;
  const double *pre;
  const double *mx;
  int64_t V;
} graph_t;

/* _ckernels.pyx:90-100 / graph.py:83-97: inverse-CDF pick over the prefix */
static inline int64_t pick_weighted(const graph_t *g, int64_t v, double r) {
  int64_t lo = g->row[v], hi = g->row[v + 1];
  double total = g->pre[hi - 1];
  int64_t idx = first_greater(g->pre, lo, hi, r * total);
  if (idx > hi - 1) idx = hi - 1;
  return g->col[idx];
}

typedef struct {
  int code;
  double term;                 /* ppr */
  double f_ret, f_adj, f_far;  /* node2vec */
  double f_max;
} app_t;

static int make_app(int code, const double *params, int64_t n_params, app_t *a) {
  memset(a, 0, sizeof(*a));
  a->code = code;
  if (code == NDO_PPR) {
    if (n_params < 1) return NDO_ERR_ARG;
    a->term = params[0];
  } else if (code == NDO_NODE2VEC) {
    if (n_params < 3) return NDO_ERR_ARG;
    double p = params[0], q = params[1];
    /* _ckernels.pyx:172-181 (apps.py:147-152 conventions) */
    if (params[2] == 0.0) { a->f_ret = 1.0 / p; a->f_adj = 1.0; a->f_far = 1.0 / q; }
    else { a->f_ret = p; a->f_adj = 1.0 / q; a->f_far = 1.0; }
    a->f_max = a->f_ret;
    if (a->f_adj > a->f_max) a->f_max = a->f_adj;
    if (a->f_far > a->f_max) a->f_max = a->f_far;
  } else if (code != NDO_DEEPWALK && code != NDO_KHOP && code != NDO_MULTIRW) {
    return NDO_ERR_APP;
  }
  return NDO_OK;
}

/* One work item of individual_batch (_ckernels.pyx:184-265, protocol
 * _pykernels.py:161-167).  Sets *stall on a node2vec cap hit. */
static int64_t run_item(const graph_t *g, const app_t *a, int64_t v, int64_t t,
                        int64_t sid, int64_t tix, int64_t slot, uint64_t seed,
                        int64_t step, int *stall) {
  int64_t base = g->row[v];
  int64_t deg = g->row[v + 1] - base;
  if (deg <= 0) return NULLV;
  switch (a->code) {
    case NDO_DEEPWALK:
      return pick_weighted(g, v, unit53(ndo_key_u64(seed, sid, step, tix, slot, 0, 0)));
    case NDO_PPR:
      if (unit53(ndo_key_u64(seed, sid, step, tix, slot, 0, 0)) < a->term) return NULLV;
      return pick_weighted(g, v, unit53(ndo_key_u64(seed, sid, step, tix, slot, 0, 1)));
    case NDO_KHOP:
    case NDO_MULTIRW: {
      uint64_t u = ndo_key_u64(seed, sid, step, tix, slot, 0, 0);
      return g->col[base + (int64_t)(u % (uint64_t)deg)];
    }
    case NDO_NODE2VEC: {
      if (t < 0)
        return pick_weighted(g, v, unit53(ndo_key_u64(seed, sid, step, tix, slot, 0, 0)));
      int64_t t_lo = g->row[t], t_hi = g->row[t + 1];
      double env = g->mx[v] * a->f_max;
      for (long j = 0; j < N2V_MAX_TRIES; j++) {
        uint64_t u = ndo_key_u64(seed, sid, step, tix, slot, 0, 2 * j);
        int64_t at = base + (int64_t)(u % (uint64_t)deg);
        int64_t nb = g->col[at];
        double w = g->w[at];
        double f;
        if (nb == t) f = a->f_ret;
        else if (sorted_has(g->col, t_lo, t_hi, nb)) f = a->f_adj;
        else f = a->f_far;
        double r = unit53(ndo_key_u64(seed, sid, step, tix, slot, 0, 2 * j + 1));
        if (env <= 0 || r * env < w * f) return nb;
      }
      *stall = 1;
      return NULLV;
    }
  }
  return NULLV;
}

/* _ckernels.pyx:136-271 */
int ndo_individual_batch(int app_code, const double *params, int64_t n_params,
                         const int64_t *row_offsets, const int64_t *col_indices,
                         const double *weights, const double *weight_prefix,
                         const double *max_weight, const int64_t *transits,
                         const int64_t *t_prev, const int64_t *sample_ids,
                         const int64_t *transit_idxs, const int64_t *slots,
                         int64_t n, uint64_t seed, int64_t step, int64_t *out) {
  app_t a;
  int rc = make_app(app_code, params, n_params, &a);
  if (rc) return rc;
  graph_t g = {row_offsets, col_indices, weights, weight_prefix, max_weight, 0};
  int stall = 0;
  for (int64_t i = 0; i < n; i++) {
    out[i] = run_item(&g, &a, transits[i], t_prev[i], sample_ids[i], transit_idxs[i],
                      slots[i], seed, step, &stall);
    if (stall) return NDO_ERR_STALL;
  }
  return NDO_OK;
}

/* apps.py:83-103: `count` keyed root draws, distinct when V >= count */
static void roots_one(int64_t V, int64_t count, uint64_t seed, int64_t sid, int64_t *out) {
  int distinct = V >= count;
  int64_t have = 0, draw = 0;
  while (have < count) {
    int64_t v = (int64_t)(ndo_key_u64(seed, sid, 0, 0, 0, 2, draw) % (uint64_t)V);
    draw++;
    if (distinct) {
      int dup = 0;
      for (int64_t k = 0; k < have; k++) if (out[k] == v) { dup = 1; break; }
      if (dup) continue;
    }
    out[have++] = v;
  }
}

void ndo_uniform_roots(int64_t n_vertices, int64_t count, uint64_t seed,
                       int64_t sample_lo, int64_t n_samples, int64_t *roots) {
  for (int64_t i = 0; i < n_samples; i++)
    roots_one(n_vertices, count, seed, sample_lo + i, roots + i * count);
}

/* apps.py:340-370: cluster assignment keyed on the vertex, chosen clusters
 * keyed on the sample; roots are the member vertices in ascending order. */
int64_t ndo_cluster_roots(int64_t n_vertices, int64_t clusters_per_sample,
                          int64_t num_clusters, uint64_t seed, int64_t sample_id,
                          int64_t *roots) {
  int64_t want = clusters_per_sample < num_clusters ? clusters_per_sample : num_clusters;
  char *chosen = calloc((size_t)num_clusters, 1);
  int64_t have = 0, draw = 0;
  while (have < want) {
    int64_t c = (int64_t)(ndo_key_u64(seed, sample_id, 0, 0, 0, 5, draw) % (uint64_t)num_clusters);
    draw++;
    if (!chosen[c]) { chosen[c] = 1; have++; }
  }
  int64_t cnt = 0;
  for (int64_t v = 0; v < n_vertices; v++) {
    int64_t c = (int64_t)(ndo_key_u64(seed, v, 0, 0, 0, 4, 0) % (uint64_t)num_clusters);
    if (chosen[c]) { if (roots) roots[cnt] = v; cnt++; }
  }
  free(chosen);
  return cnt;
}

void ndo_free(void *p) { free(p); }

/* ---------------------------------------------------------------------- */
/* stable argsort of int64 keys (the np.argsort(kind="stable") the engines
 * use, chain.py:113 / transit_parallel.py:76): merge sort on (key, index). */
static void stable_argsort(const int64_t *key, int64_t n, int64_t *idx, int64_t *tmp) {
  for (int64_t i = 0; i < n; i++) idx[i] = i;
  for (int64_t width = 1; width < n; width *= 2) {
    for (int64_t lo = 0; lo < n; lo += 2 * width) {
      int64_t mid = lo + width < n ? lo + width : n;
      int64_t hi = lo + 2 * width < n ? lo + 2 * width : n;
      int64_t i = lo, j = mid, k = lo;
      while (i < mid && j < hi) {
        if (key[idx[j]] < key[idx[i]]) tmp[k++] = idx[j++];
        else tmp[k++] = idx[i++];
      }
      while (i < mid) tmp[k++] = idx[i++];
      while (j < hi) tmp[k++] = idx[j++];
    }
    memcpy(idx, tmp, (size_t)n * sizeof(int64_t));
  }
}

/* work classes over sorted keys (chain.py:112-126 / transit_parallel.py:86-101) */
static void class_counts(const int64_t *sorted_keys, int64_t n, int64_t m, int64_t *st) {
  int64_t i = 0;
  while (i < n) {
    int64_t j = i + 1;
    while (j < n && sorted_keys[j] == sorted_keys[i]) j++;
    int64_t work = (j - i) * m;
    if (work < SMALL_MAX_WORK) st[0]++;
    else if (work <= LARGE_MIN_WORK) st[1]++;
    else st[2]++;
    st[3]++;
    i = j;
  }
}

typedef struct {
  int64_t *vals;
  int64_t len, cap;
} vec_t;

static int vec_push(vec_t *v, int64_t x) {
  if (v->len == v->cap) {
    int64_t nc = v->cap ? v->cap * 2 : 1024;
    int64_t *p = realloc(v->vals, (size_t)nc * sizeof(int64_t));
    if (!p) return NDO_ERR_NOMEM;
    v->vals = p; v->cap = nc;
  }
  v->vals[v->len++] = x;
  return NDO_OK;
}

/* One engine instance of run_chain (chain.py:64-164) over samples
 * [lo, hi).  Step records go to rec (pairs pos,value, step-major). */
typedef struct {
  int64_t *pos_rec;  /* local position per record */
  int64_t *val_rec;
  int64_t n_rec, cap_rec;
  int64_t n_steps;
  int64_t *stats;    /* 4 per step */
  int64_t stats_cap;
  int rc;
} chain_part_t;

static int grow2(int64_t **a, int64_t **b, int64_t *cap, int64_t need) {
  if (need <= *cap) return NDO_OK;
  int64_t nc = *cap ? *cap : 1024;
  while (nc < need) nc *= 2;
  int64_t *pa = realloc(*a, (size_t)nc * sizeof(int64_t));
  if (!pa) return NDO_ERR_NOMEM;
  *a = pa;
  int64_t *pb = realloc(*b, (size_t)nc * sizeof(int64_t));
  if (!pb) return NDO_ERR_NOMEM;
  *b = pb;
  *cap = nc;
  return NDO_OK;
}

static void chain_part(const graph_t *g, const app_t *a, int64_t sample_lo, int64_t lo,
                       int64_t hi, int64_t *roots, int64_t R, uint64_t seed,
                       int64_t steps, int64_t step_cap, int paradigm, chain_part_t *P) {
  int64_t n = hi - lo;
  int root_pick = a->code == NDO_MULTIRW;
  memset(P, 0, sizeof(*P));
  int64_t *cur = malloc((size_t)(n ? n : 1) * sizeof(int64_t));
  int64_t *prev = malloc((size_t)(n ? n : 1) * sizeof(int64_t));
  int64_t *alive = malloc((size_t)(n ? n : 1) * sizeof(int64_t));
  int64_t *trans = malloc((size_t)(n ? n : 1) * sizeof(int64_t));
  int64_t *order = malloc((size_t)(n ? n : 1) * sizeof(int64_t));
  int64_t *tmp = malloc((size_t)(n ? n : 1) * sizeof(int64_t));
  int64_t *skeys = malloc((size_t)(n ? n : 1) * sizeof(int64_t));
  int64_t *outv = malloc((size_t)(n ? n : 1) * sizeof(int64_t));
  int64_t n_alive = n;
  for (int64_t i = 0; i < n; i++) {
    alive[i] = i;
    prev[i] = NULLV;
    cur[i] = root_pick ? NULLV : roots[(lo + i) * R];
  }
  int64_t step = 0;
  int stall = 0;
  while (n_alive > 0) {
    if (steps >= 0 && step >= steps) break;
    if (step >= step_cap) break;
    if (step >= P->stats_cap) {
      int64_t nc = P->stats_cap ? 2 * P->stats_cap : 128;
      P->stats = realloc(P->stats, (size_t)nc * 4 * sizeof(int64_t));
      memset(P->stats + 4 * P->stats_cap, 0, (size_t)(nc - P->stats_cap) * 4 * sizeof(int64_t));
      P->stats_cap = nc;
    }
    int64_t *st = P->stats + 4 * step;
    for (int64_t k = 0; k < n_alive; k++) {
      int64_t i = alive[k];
      if (root_pick) {
        /* chain.py:102-108: per-step root pick, domain 1 */
        int64_t pick = (int64_t)(ndo_key_u64(seed, sample_lo + lo + i, step, 0, 0, 1, 0) % (uint64_t)R);
        trans[k] = roots[(lo + i) * R + pick];
      } else {
        trans[k] = cur[i];
      }
    }
    if (paradigm == 1) {
      stable_argsort(trans, n_alive, order, tmp);
      for (int64_t k = 0; k < n_alive; k++) skeys[k] = trans[order[k]];
      class_counts(skeys, n_alive, 1, st);
    } else {
      for (int64_t k = 0; k < n_alive; k++) order[k] = k;
      st[3] += n_alive;
    }
    for (int64_t q = 0; q < n_alive; q++) {
      int64_t k = order[q];
      int64_t i = alive[k];
      outv[k] = run_item(g, a, trans[k], prev[i], sample_lo + lo + i, 0, 0, seed, step, &stall);
      if (stall) { P->rc = NDO_ERR_STALL; goto done; }
    }
    if (grow2(&P->pos_rec, &P->val_rec, &P->cap_rec, P->n_rec + n_alive)) {
      P->rc = NDO_ERR_NOMEM; goto done;
    }
    for (int64_t k = 0; k < n_alive; k++) {
      P->pos_rec[P->n_rec] = alive[k];
      P->val_rec[P->n_rec] = outv[k];
      P->n_rec++;
    }
    if (root_pick) {
      /* chain.py:144-151: replace the first occurrence of the chosen root */
      for (int64_t k = 0; k < n_alive; k++) {
        if (outv[k] == NULLV) continue;
        int64_t *row = roots + (lo + alive[k]) * R;
        for (int64_t c = 0; c < R; c++)
          if (row[c] == trans[k]) { row[c] = outv[k]; break; }
      }
    } else {
      int64_t w = 0;
      for (int64_t k = 0; k < n_alive; k++) {
        int64_t i = alive[k];
        prev[i] = trans[k];
        cur[i] = outv[k];
        if (outv[k] != NULLV) alive[w++] = i;
      }
      n_alive = w;
    }
    step++;
  }
done:
  P->n_steps = step;
  free(cur); free(prev); free(alive); free(trans); free(order); free(tmp);
  free(skeys); free(outv);
}

int ndo_run_chain(const int64_t *row_offsets, const int64_t *col_indices,
                  const double *weights, const double *weight_prefix,
                  const double *max_weight, int64_t n_vertices, int app_code,
                  const double *params, int64_t n_params, int64_t sample_lo,
                  int64_t n, int64_t *roots, int64_t R, uint64_t seed,
                  int64_t steps, int64_t step_cap, int paradigm, int n_threads,
                  int64_t *chain_len, int64_t **chain_vals,
                  int64_t *n_steps_out, int64_t **stats_out) {
  app_t a;
  int rc = make_app(app_code, params, n_params, &a);
  if (rc) return rc;
  graph_t g = {row_offsets, col_indices, weights, weight_prefix, max_weight, n_vertices};
  if (n_threads < 1) n_threads = 1;
  /* driver.py:175-186 worker_ranges: contiguous, sizes differ by <= 1 */
  int64_t W = n_threads < n ? n_threads : (n ? n : 1);
  chain_part_t *parts = calloc((size_t)W, sizeof(chain_part_t));
  int64_t *bounds = malloc((size_t)(W + 1) * sizeof(int64_t));
  int64_t base = n / W, extra = n % W;
  bounds[0] = 0;
  for (int64_t w = 0; w < W; w++) bounds[w + 1] = bounds[w] + base + (w < extra ? 1 : 0);
#pragma omp parallel for schedule(dynamic, 1) num_threads(n_threads)
  for (int64_t w = 0; w < W; w++)
    chain_part(&g, &a, sample_lo, bounds[w], bounds[w + 1], roots, R, seed, steps, step_cap,
               paradigm, &parts[w]);
  /* _materialize (chain.py:167-179): per-sample chains in step order */
  int64_t total = 0, max_steps = 0, stats_steps = 0;
  for (int64_t w = 0; w < W; w++) {
    if (parts[w].rc) rc = parts[w].rc;
    total += parts[w].n_rec;
    if (parts[w].n_steps > max_steps) max_steps = parts[w].n_steps;
  }
  stats_steps = max_steps;
  int64_t *vals = malloc((size_t)(total ? total : 1) * sizeof(int64_t));
  int64_t *st = calloc((size_t)(stats_steps ? stats_steps : 1) * 4, sizeof(int64_t));
  memset(chain_len, 0, (size_t)n * sizeof(int64_t));
  for (int64_t w = 0; w < W; w++)
    for (int64_t r = 0; r < parts[w].n_rec; r++) chain_len[bounds[w] + parts[w].pos_rec[r]]++;
  int64_t *off = malloc((size_t)(n + 1) * sizeof(int64_t));
  off[0] = 0;
  for (int64_t i = 0; i < n; i++) off[i + 1] = off[i] + chain_len[i];
  int64_t *fill = calloc((size_t)(n ? n : 1), sizeof(int64_t));
  for (int64_t w = 0; w < W; w++) {
    for (int64_t r = 0; r < parts[w].n_rec; r++) {
      int64_t i = bounds[w] + parts[w].pos_rec[r];
      vals[off[i] + fill[i]++] = parts[w].val_rec[r];
    }
    for (int64_t s = 0; s < parts[w].n_steps; s++)
      for (int c = 0; c < 4; c++) st[4 * s + c] += parts[w].stats[4 * s + c];
    free(parts[w].pos_rec); free(parts[w].val_rec); free(parts[w].stats);
  }
  free(fill); free(off); free(parts); free(bounds);
  *chain_vals = vals;
  *n_steps_out = max_steps;
  *stats_out = st;
  return rc;
}

/* ---------------------------------------------------------------------- */
/* generic individual loop: driver.py:80-144 (StepPlan), 203-235 (run_loop),
 * core.py:168-203 (transits / liveness), transit_parallel.py:185-230.
 * Per step output: step_counts[s*n + i] slots for sample i (pairs*m, 0 when
 * not alive), vals step-major (sample-major inside a step, NULLs kept). */
static int cmp_i64(const void *a, const void *b) {
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  return x < y ? -1 : (x > y);
}

/* output.py:27-31 dedup_step: sorted distinct non-NULL values, in place;
 * returns the new length */
static int64_t dedup_inplace(int64_t *a, int64_t len) {
  int64_t w = 0;
  for (int64_t k = 0; k < len; k++) if (a[k] != NULLV) a[w++] = a[k];
  qsort(a, (size_t)w, sizeof(int64_t), cmp_i64);
  int64_t u = 0;
  for (int64_t k = 0; k < w; k++) if (u == 0 || a[k] != a[u - 1]) a[u++] = a[k];
  return u;
}

static int is_unique_step(const uint8_t *mask, int64_t n_mask, int64_t step) {
  if (!mask || n_mask <= 0) return 0;
  return mask[step < n_mask ? step : n_mask - 1] != 0;
}

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
                       int64_t **stats_out) {
  app_t a;
  int rc = make_app(app_code, params, n_params, &a);
  if (rc) return rc;
  graph_t g = {row_offsets, col_indices, weights, weight_prefix, max_weight, n_vertices};
  vec_t V = {0}, C = {0}, S = {0};
  /* per-sample index of each step's slice in V (for vertices_at) */
  int64_t cap_steps = 16;
  int64_t *slice_off = malloc((size_t)(cap_steps * n + 1) * sizeof(int64_t));
  int64_t *slice_len = malloc((size_t)(cap_steps * n + 1) * sizeof(int64_t));
  char *alive = malloc((size_t)(n ? n : 1));
  char *fallback = calloc((size_t)(n ? n : 1), 1);  /* driver.py:171 _sp_fallback */
  for (int64_t i = 0; i < n; i++) alive[i] = 1;
  vec_t pt = {0}, pp = {0}, pti = {0}, pprev = {0};
  int64_t step = 0;
  int stall = 0;
  for (;;) {
    if (steps >= 0 && step >= steps) break;
    if (step >= step_cap) break;
    if (step >= cap_steps) {
      cap_steps *= 2;
      slice_off = realloc(slice_off, (size_t)(cap_steps * n + 1) * sizeof(int64_t));
      slice_len = realloc(slice_len, (size_t)(cap_steps * n + 1) * sizeof(int64_t));
    }
    int64_t m = fanouts[step < n_fanouts ? step : n_fanouts - 1];
    pt.len = pp.len = pti.len = pprev.len = 0;
    int64_t any = 0;
    for (int64_t i = 0; i < n; i++) {
      slice_off[step * n + i] = 0;
      slice_len[step * n + i] = 0;
      if (!alive[i]) continue;
      const int64_t *rr = roots + roots_off[i];
      int64_t nr = roots_off[i + 1] - roots_off[i];
      /* core.py:168-203 */
      int64_t cnt = 0;
      if (root_pick) {
        if (nr > 0) {
          int64_t pick = (int64_t)(ndo_key_u64(seed, sample_lo + i, step, 0, 0, 1, 0) % (uint64_t)nr);
          vec_push(&pt, rr[pick]); vec_push(&pp, i); vec_push(&pti, 0); cnt = 1;
        }
      } else if (step == 0) {
        for (int64_t k = 0; k < nr; k++) { vec_push(&pt, rr[k]); vec_push(&pp, i); vec_push(&pti, cnt++); }
      } else {
        int64_t so = slice_off[(step - 1) * n + i], sl = slice_len[(step - 1) * n + i];
        for (int64_t k = 0; k < sl; k++)
          if (V.vals[so + k] != NULLV) { vec_push(&pt, V.vals[so + k]); vec_push(&pp, i); vec_push(&pti, cnt++); }
      }
      if (cnt == 0) { alive[i] = 0; continue; }
      any = 1;
      int64_t tprev = NULLV;
      if (needs_prev2 && step >= 1) {
        /* core.py:99-103 prev_vertex(2, 0): first non-NULL two steps back */
        if (step == 1) tprev = rr[0];
        else {
          int64_t so = slice_off[(step - 2) * n + i], sl = slice_len[(step - 2) * n + i];
          for (int64_t k = 0; k < sl; k++) if (V.vals[so + k] != NULLV) { tprev = V.vals[so + k]; break; }
        }
      }
      for (int64_t k = 0; k < cnt; k++) vec_push(&pprev, tprev);
    }
    if (!any) break;
    int64_t np_ = pt.len;
    int64_t st4[4] = {0, 0, 0, 0};
    if (paradigm == 1) {
      /* transit_parallel.py:200-231: samples flagged by the previous unique
       * step run sample-parallel (one fetch per pair, outside the groups) */
      int64_t *keep = malloc((size_t)(np_ ? np_ : 1) * sizeof(int64_t));
      int64_t nk = 0, nflag = 0;
      for (int64_t k = 0; k < np_; k++) {
        if (fallback[pp.vals[k]]) nflag++;
        else keep[nk++] = pt.vals[k];
      }
      int64_t *order = malloc((size_t)(nk ? nk : 1) * sizeof(int64_t)), *tmp = malloc((size_t)(nk ? nk : 1) * sizeof(int64_t));
      int64_t *sk = malloc((size_t)(nk ? nk : 1) * sizeof(int64_t));
      stable_argsort(keep, nk, order, tmp);
      for (int64_t k = 0; k < nk; k++) sk[k] = keep[order[k]];
      class_counts(sk, nk, m, st4);
      st4[3] += nflag;
      free(order); free(tmp); free(sk); free(keep);
    } else {
      st4[3] = np_;
    }
    for (int64_t i = 0; i < n; i++) fallback[i] = 0;
    for (int c = 0; c < 4; c++) vec_push(&S, st4[c]);
    /* outputs are order independent (keyed RNG): compute sample-major */
    int64_t base = V.len;
    for (int64_t p = 0; p < np_; p++) {
      int64_t i = pp.vals[p];
      for (int64_t sl = 0; sl < m; sl++) {
        int64_t o = run_item(&g, &a, pt.vals[p], pprev.vals[p], sample_lo + i, pti.vals[p], sl,
                             seed, step, &stall);
        if (stall) { rc = NDO_ERR_STALL; goto out; }
        vec_push(&V, o);
      }
    }
    for (int64_t p = 0; p < np_; p++) {
      int64_t i = pp.vals[p];
      if (slice_len[step * n + i] == 0) slice_off[step * n + i] = base + p * m;
      slice_len[step * n + i] += m;
    }
    if (is_unique_step(unique_mask, n_mask, step)) {
      /* driver.py:165-172 finish_step: dedup every alive sample's step, then
       * compact V (samples' slices are contiguous and sample-ordered) */
      int64_t wpos = base;
      for (int64_t i = 0; i < n; i++) {
        int64_t sl = slice_len[step * n + i];
        if (sl == 0) continue;
        int64_t so = slice_off[step * n + i];
        int64_t u = dedup_inplace(V.vals + so, sl);
        memmove(V.vals + wpos, V.vals + so, (size_t)u * sizeof(int64_t));
        slice_off[step * n + i] = wpos;
        slice_len[step * n + i] = u;
        fallback[i] = (0 < u && u < m);
        wpos += u;
      }
      V.len = wpos;
    }
    if (root_pick) {
      /* apps.py:228-235 multirw_post_step */
      for (int64_t p = 0; p < np_; p++) {
        int64_t i = pp.vals[p];
        int64_t v = V.vals[slice_off[step * n + i]];
        if (v == NULLV) continue;
        int64_t *rr = roots + roots_off[i];
        for (int64_t k = 0; k < roots_off[i + 1] - roots_off[i]; k++)
          if (rr[k] == pt.vals[p]) { rr[k] = v; break; }
      }
    }
    for (int64_t i = 0; i < n; i++) vec_push(&C, slice_len[step * n + i]);
    step++;
  }
out:
  *n_steps_out = step;
  *step_counts = C.vals ? C.vals : malloc(8);
  *vals = V.vals ? V.vals : malloc(8);
  *n_vals = V.len;
  *stats_out = S.vals ? S.vals : malloc(8);
  free(slice_off); free(slice_len); free(alive); free(fallback);
  free(pt.vals); free(pp.vals); free(pti.vals); free(pprev.vals);
  return rc;
}

/* ---------------------------------------------------------------------- */
/* collective loop: transit_parallel.py:187-198 -> collective.py:39-141 ->
 * apps.py:247-386.  kind: NDO_C_*; distribution 0 uniform / 1 degree_sq. */
int ndo_run_collective(const int64_t *row_offsets, const int64_t *col_indices,
                       int64_t n_vertices, int kind, int64_t step_size,
                       int64_t max_size, int distribution, int64_t sample_lo,
                       int64_t n, const int64_t *roots_off, const int64_t *roots,
                       uint64_t seed, int64_t steps, int64_t step_cap,
                       const uint8_t *unique_mask, int64_t n_mask,
                       int64_t *n_steps_out, int64_t **step_counts,
                       int64_t **vals, int64_t *n_vals, int64_t **rec_counts,
                       int64_t **rec_t, int64_t **rec_v, int64_t *n_rec,
                       int64_t **stats_out) {
  const int64_t *row = row_offsets, *col = col_indices;
  int64_t V_ = n_vertices;
  int rc = NDO_OK;
  vec_t V = {0}, C = {0}, RC = {0}, RT = {0}, RV = {0}, S = {0};
  double *cum = NULL;
  if (kind == NDO_C_IMPORTANCE && distribution == 1) {
    /* apps.py:291-296: cumsum(deg^2) in f64 */
    cum = malloc((size_t)V_ * sizeof(double));
    double acc = 0.0;
    for (int64_t v = 0; v < V_; v++) {
      double d = (double)(row[v + 1] - row[v]);
      acc += d * d;
      cum[v] = acc;
    }
  }
  int64_t *prev_off = calloc((size_t)(n ? n : 1), sizeof(int64_t));
  int64_t *prev_len = calloc((size_t)(n ? n : 1), sizeof(int64_t));
  int64_t *size_ = calloc((size_t)(n ? n : 1), sizeof(int64_t));
  char *alive = malloc((size_t)(n ? n : 1));
  for (int64_t i = 0; i < n; i++) { alive[i] = 1; size_[i] = roots_off[i + 1] - roots_off[i]; }
  vec_t tr = {0};
  int64_t step = 0;
  for (;;) {
    if (steps >= 0 && step >= steps) break;
    if (step >= step_cap) break;
    int64_t any = 0;
    int64_t m = step_size;
    int64_t st4[4] = {0, 0, 0, 0};
    /* TP build classes (collective.py:79-115): groups by transit over the
     * step's pairs, work = members * degree */
    vec_t allt = {0};
    int64_t *new_off = calloc((size_t)(n ? n : 1), sizeof(int64_t));
    int64_t *new_len = calloc((size_t)(n ? n : 1), sizeof(int64_t));
    int64_t *step_rec = calloc((size_t)(n ? n : 1), sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) {
      if (!alive[i]) continue;
      tr.len = 0;
      if (step == 0) {
        for (int64_t k = roots_off[i]; k < roots_off[i + 1]; k++) vec_push(&tr, roots[k]);
      } else {
        for (int64_t k = 0; k < prev_len[i]; k++) {
          int64_t v = V.vals[prev_off[i] + k];
          if (v != NULLV) vec_push(&tr, v);
        }
      }
      if (tr.len == 0) { alive[i] = 0; continue; }
      any = 1;
      for (int64_t k = 0; k < tr.len; k++) vec_push(&allt, tr.vals[k]);
      int64_t nt = tr.len;
      int64_t total = 0;
      for (int64_t k = 0; k < nt; k++) total += row[tr.vals[k] + 1] - row[tr.vals[k]];
      int64_t sid = sample_lo + i;
      new_off[i] = V.len;
      new_len[i] = m;
      int64_t rec_before = RT.len;
      if (kind == NDO_C_LAYER) {
        /* apps.py:261-277 */
        int64_t take = max_size - size_[i];
        if (take < 0) take = 0;
        if (take > m) take = m;
        if (total == 0) take = 0;
        for (int64_t sl = 0; sl < m; sl++) {
          int64_t o = NULLV;
          if (sl < take) {
            int64_t e = (int64_t)(ndo_key_u64(seed, sid, step, 0, sl, 0, 0) % (uint64_t)total);
            for (int64_t k = 0; k < nt; k++) {
              int64_t d = row[tr.vals[k] + 1] - row[tr.vals[k]];
              if (e < d) { o = col[row[tr.vals[k]] + e]; break; }
              e -= d;
            }
          }
          vec_push(&V, o);
        }
      } else if (kind == NDO_C_IMPORTANCE) {
        /* apps.py:286-312 */
        for (int64_t sl = 0; sl < m; sl++) {
          int64_t v;
          uint64_t u = ndo_key_u64(seed, sid, step, 0, sl, 0, 0);
          if (distribution == 0) v = (int64_t)(u % (uint64_t)V_);
          else {
            double x = unit53(u) * cum[V_ - 1];
            int64_t lo = 0, hi = V_;
            while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (cum[mid] <= x) lo = mid + 1; else hi = mid; }
            v = lo < V_ - 1 ? lo : V_ - 1;
          }
          for (int64_t k = 0; k < nt; k++) {
            int64_t t = tr.vals[k];
            if (sorted_has(col, row[t], row[t + 1], v)) { vec_push(&RT, t); vec_push(&RV, v); }
          }
          vec_push(&V, v);
        }
      } else if (kind == NDO_C_MVS) {
        /* apps.py:327-338 */
        for (int64_t sl = 0; sl < m; sl++) {
          int64_t o = NULLV;
          if (total > 0) {
            int64_t e = (int64_t)(ndo_key_u64(seed, sid, step, 0, sl, 0, 0) % (uint64_t)total);
            for (int64_t k = 0; k < nt; k++) {
              int64_t t = tr.vals[k], d = row[t + 1] - row[t];
              if (e < d) { o = col[row[t] + e]; vec_push(&RT, t); vec_push(&RV, o); break; }
              e -= d;
            }
          }
          vec_push(&V, o);
        }
      } else if (kind == NDO_C_CLUSTERGCN) {
        /* apps.py:372-379: record combined entries whose neighbour is a root
         * (np.isin against the root set; searched on a sorted copy) */
        int64_t nr = roots_off[i + 1] - roots_off[i];
        int64_t *rr = malloc((size_t)(nr ? nr : 1) * sizeof(int64_t));
        int64_t *rtmp = malloc((size_t)(nr ? nr : 1) * sizeof(int64_t));
        int64_t *ridx = malloc((size_t)(nr ? nr : 1) * sizeof(int64_t));
        stable_argsort(roots + roots_off[i], nr, ridx, rtmp);
        for (int64_t k = 0; k < nr; k++) rr[k] = roots[roots_off[i] + ridx[k]];
        free(rtmp); free(ridx);
        for (int64_t sl = 0; sl < m; sl++) {
          for (int64_t k = 0; k < nt; k++) {
            int64_t t = tr.vals[k];
            for (int64_t e = row[t]; e < row[t + 1]; e++) {
              int64_t v = col[e];
              int64_t lo = 0, hi = nr;  /* roots are ascending */
              while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (rr[mid] < v) lo = mid + 1; else hi = mid; }
              if (lo < nr && rr[lo] == v) { vec_push(&RT, t); vec_push(&RV, v); }
            }
          }
          vec_push(&V, NULLV);
        }
        free(rr);
      } else {
        rc = NDO_ERR_APP;
        goto out;
      }
      if (is_unique_step(unique_mask, n_mask, step)) {
        /* finish_step dedup (driver.py:165-172) of this sample's slots */
        int64_t u = dedup_inplace(V.vals + new_off[i], m);
        V.len = new_off[i] + u;
        new_len[i] = u;
        size_[i] += u;
      } else {
        for (int64_t sl = 0; sl < m; sl++) if (V.vals[new_off[i] + sl] != NULLV) size_[i]++;
      }
      step_rec[i] = RT.len - rec_before;
    }
    if (!any) { free(allt.vals); free(new_off); free(new_len); free(step_rec); break; }
    {
      int64_t np_ = allt.len;
      int64_t *order = malloc((size_t)np_ * sizeof(int64_t)), *tmp = malloc((size_t)np_ * sizeof(int64_t));
      stable_argsort(allt.vals, np_, order, tmp);
      int64_t q = 0;
      while (q < np_) {
        int64_t t = allt.vals[order[q]], r = q + 1;
        while (r < np_ && allt.vals[order[r]] == t) r++;
        int64_t work = (r - q) * (row[t + 1] - row[t]);
        if (work < SMALL_MAX_WORK) st4[0]++; else if (work <= LARGE_MIN_WORK) st4[1]++; else st4[2]++;
        st4[3]++;
        q = r;
      }
      free(order); free(tmp);
    }
    free(allt.vals);
    for (int c = 0; c < 4; c++) vec_push(&S, st4[c]);
    /* per sample slot counts and recorded-edge counts of this step */
    for (int64_t i = 0; i < n; i++) {
      vec_push(&C, alive[i] ? new_len[i] : 0);
      vec_push(&RC, step_rec[i]);
      prev_off[i] = new_off[i];
      prev_len[i] = alive[i] ? new_len[i] : 0;
    }
    free(new_off); free(new_len); free(step_rec);
    step++;
  }
out:
  *n_steps_out = step;
  *step_counts = C.vals ? C.vals : malloc(8);
  *vals = V.vals ? V.vals : malloc(8);
  *n_vals = V.len;
  *rec_counts = RC.vals ? RC.vals : malloc(8);
  *rec_t = RT.vals ? RT.vals : malloc(8);
  *rec_v = RV.vals ? RV.vals : malloc(8);
  *n_rec = RT.len;
  *stats_out = S.vals ? S.vals : malloc(8);
  free(cum); free(prev_off); free(prev_len); free(size_); free(alive); free(tr.vals);
  return rc;
}

/* ---------------------------------------------------------------------- */
/* transit_parallel.py:71-101: stable grouping by transit, classes by work =
 * members*m, dense per-class rank in ascending transit order. */
int64_t ndo_transit_schedule(const int64_t *pair_transit, int64_t n_pairs,
                             int64_t m, int64_t *order, int64_t *group_start,
                             int64_t *group_transit, int32_t *group_class,
                             int64_t *sched_index) {
  int64_t *tmp = malloc((size_t)(n_pairs ? n_pairs : 1) * sizeof(int64_t));
  stable_argsort(pair_transit, n_pairs, order, tmp);
  free(tmp);
  int64_t G = 0, rank[3] = {0, 0, 0};
  int64_t q = 0;
  while (q < n_pairs) {
    int64_t t = pair_transit[order[q]], r = q + 1;
    while (r < n_pairs && pair_transit[order[r]] == t) r++;
    int64_t work = (r - q) * m;
    int c = work < SMALL_MAX_WORK ? 0 : (work <= LARGE_MIN_WORK ? 1 : 2);
    group_start[G] = q;
    group_transit[G] = t;
    group_class[G] = c;
    sched_index[G] = rank[c]++;
    G++;
    q = r;
  }
  group_start[G] = n_pairs;
  return G;
}

/* ---------------------------------------------------------------------- */
/* Keyed RMAT generator (this build's input generator):
 * 16-bit quadrant draws, 4 levels per keyed u64 (domain 16), endpoints
 * permuted by a keyed bijection (domain 17), weights 1 + 4u keyed on the
 * edge index (domain 3, as graph.py:168-169).  Undirected emits (s,d),(d,s). */
static inline uint64_t bij(uint64_t x, int scale, uint64_t k1, uint64_t k2) {
  uint64_t mask = scale >= 64 ? ~0ull : ((1ull << scale) - 1);
  int sh = scale / 2 + 1;
  x = (x * (k1 | 1u)) & mask;
  x ^= x >> sh;
  x = (x * (k2 | 1u)) & mask;
  x ^= x >> sh;
  return x;
}

void ndo_rmat_edges(int scale, int64_t n_edges, uint32_t ta, uint32_t tab,
                    uint32_t tabc, uint64_t seed, int undirected, int weighted,
                    int64_t *src, int64_t *dst, double *w) {
  uint64_t k1 = ndo_key_u64(seed, 0, 0, 0, 0, 17, 0);
  uint64_t k2 = ndo_key_u64(seed, 0, 0, 0, 0, 17, 1);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < n_edges; e++) {
    uint64_t s = 0, d = 0, u = 0;
    for (int l = 0; l < scale; l++) {
      if ((l & 3) == 0) u = ndo_key_u64(seed, e, l >> 2, 0, 0, 16, 0);
      uint32_t r = (uint32_t)((u >> (16 * (l & 3))) & 0xFFFFu);
      uint64_t sb = r >= tab, db = (r >= ta && r < tab) || r >= tabc;
      s = (s << 1) | sb;
      d = (d << 1) | db;
    }
    s = bij(s, scale, k1, k2);
    d = bij(d, scale, k1, k2);
    double we = 1.0;
    if (weighted) {
      volatile double span = 4.0 * ndo_key_uniform(seed, e, 0, 0, 0, 3, 0);
      we = 1.0 + span;
    }
    if (undirected) {
      src[2 * e] = (int64_t)s; dst[2 * e] = (int64_t)d; w[2 * e] = we;
      src[2 * e + 1] = (int64_t)d; dst[2 * e + 1] = (int64_t)s; w[2 * e + 1] = we;
    } else {
      src[e] = (int64_t)s; dst[e] = (int64_t)d; w[e] = we;
    }
  }
}

/* graph.py:107-129: lexsort((dst, src)) — stable, rows dst-sorted, parallel
 * edges in input order.  Counting sort by src, then a stable sort by dst
 * inside each row. */
int ndo_from_edges(const int64_t *src, const int64_t *dst, const double *w,
                   int64_t n_edges, int64_t n_vertices, int64_t *row_offsets,
                   int64_t *col_indices, double *weights_out) {
  memset(row_offsets, 0, (size_t)(n_vertices + 1) * sizeof(int64_t));
  for (int64_t e = 0; e < n_edges; e++) {
    if (src[e] < 0 || src[e] >= n_vertices || dst[e] < 0 || dst[e] >= n_vertices) return NDO_ERR_ARG;
    row_offsets[src[e] + 1]++;
  }
  for (int64_t v = 0; v < n_vertices; v++) row_offsets[v + 1] += row_offsets[v];
  int64_t *fill = malloc((size_t)(n_vertices ? n_vertices : 1) * sizeof(int64_t));
  int64_t *eid = malloc((size_t)(n_edges ? n_edges : 1) * sizeof(int64_t));
  memcpy(fill, row_offsets, (size_t)n_vertices * sizeof(int64_t));
  for (int64_t e = 0; e < n_edges; e++) eid[fill[src[e]]++] = e;
  free(fill);
  int64_t maxdeg = 0;
  for (int64_t v = 0; v < n_vertices; v++) {
    int64_t d = row_offsets[v + 1] - row_offsets[v];
    if (d > maxdeg) maxdeg = d;
  }
  int64_t *keys = malloc((size_t)(maxdeg ? maxdeg : 1) * sizeof(int64_t));
  int64_t *idx = malloc((size_t)(maxdeg ? maxdeg : 1) * sizeof(int64_t));
  int64_t *tmp = malloc((size_t)(maxdeg ? maxdeg : 1) * sizeof(int64_t));
  for (int64_t v = 0; v < n_vertices; v++) {
    int64_t lo = row_offsets[v], d = row_offsets[v + 1] - lo;
    for (int64_t k = 0; k < d; k++) keys[k] = dst[eid[lo + k]];
    stable_argsort(keys, d, idx, tmp);
    for (int64_t k = 0; k < d; k++) {
      int64_t e = eid[lo + idx[k]];
      col_indices[lo + k] = dst[e];
      weights_out[lo + k] = w ? w[e] : 1.0;
    }
  }
  free(keys); free(idx); free(tmp); free(eid);
  return NDO_OK;
}
