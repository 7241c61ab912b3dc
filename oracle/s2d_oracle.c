/*
 * s2d_oracle.c -- CPU restatement of the reference 2D-sparse-parallel
 * embedding step.  TEST INFRASTRUCTURE ONLY: this file is the parity checker
 * for the CUDA path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it; the product library never links it.
 *
 * Parity status: PINNED.  tests/test_oracle.py checks every function here
 * against (a) the reference's own known-answer tests (restated from
 * proj/tests/test_embedding.cpp, test_optimizer.cpp, test_topology.cpp,
 * test_planner.cpp) and (b) golden vectors in tests/golden/ produced by
 * oracle/_ref (the reference sources under /root/reference/proj/src compiled
 * by oracle/Makefile and driven through their public API by
 * oracle/ref_harness.cpp; generator: tests/golden/make_golden.py).
 *
 * Numerics follow the reference bit for bit: fp32 storage, f64 accumulation,
 * no FMA contraction (compile with -ffp-contract=off, as the reference's
 * proj/CMakeLists.txt:11-14 does).
 *
 * Layout conventions (shared with the CUDA path):
 *   - a replica is the flat concatenation of all tables: weights at
 *     woff[f] = sum_{f'<f} rows[f']*dims[f'], moments at voff[f] = sum rows.
 *   - a rank's batch is sample-major bags (s, f): lengths[B*F] and the ids of
 *     all bags concatenated in (s, f) order.  ids are GLOBAL table rows.
 *   - pooled output / upstream gradient rows are [B][sum_f dims[f]] with
 *     feature column offset coff[f] = sum_{f'<f} dims[f'] (trainer.cpp:387-389).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL -1
#define OR_ERANGE -2   /* id outside every shard (embedding.cpp:61-63) */
#define OR_ENONFINITE -3 /* nonfinite row gradient (optimizer.cpp:69-72) */
#define OR_ENOMEM -4

/* ---- rng.hpp:11-49 ---------------------------------------------------- */

uint64_t or_mix64(uint64_t x) { /* rng.hpp:12-19 */
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ULL;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBULL;
  x ^= x >> 31;
  return x;
}

uint64_t or_make_key(const uint64_t* fields, uint32_t n) { /* rng.hpp:22-28 */
  uint64_t h = 0x8A5CD789635D2DFFULL;
  for (uint32_t i = 0; i < n; ++i) h = or_mix64(h + 0x9E3779B97F4A7C15ULL + fields[i]);
  return h;
}

/* embedding.cpp:17-37: w[r][j] = f32(lo + (hi-lo)*u_j), u_j = CounterRng draw
 * j+1 of key make_key({seed, table_id, r}); lo=-1/sqrt(D), hi=+1/sqrt(D). */
void or_init_rows(uint32_t table_id, uint32_t row_lo, uint32_t row_hi, uint32_t dim,
                  uint64_t seed, float* out) {
  const double bound = 1.0 / sqrt((double)dim);
  const double lo = -bound, hi = bound;
  for (uint32_t r = row_lo; r < row_hi; ++r) {
    const uint64_t f[3] = {seed, table_id, r};
    const uint64_t key = or_make_key(f, 3);
    float* row = out + (size_t)(r - row_lo) * dim;
    for (uint32_t j = 0; j < dim; ++j) {
      const uint64_t z = key + (uint64_t)(j + 1) * 0x9E3779B97F4A7C15ULL;
      const double u = (double)(or_mix64(z) >> 11) * 0x1.0p-53;
      row[j] = (float)(lo + (hi - lo) * u);
    }
  }
}

/* init_table rows for an arbitrary list of row ids (out: n x dim), for
 * tests that compact a big table to the rows a step touches. */
void or_init_rows_list(uint32_t table_id, const uint32_t* rows, uint64_t n, uint32_t dim, uint64_t seed, float* out) {
  for (uint64_t i = 0; i < n; ++i) or_init_rows(table_id, rows[i], rows[i] + 1, dim, seed, out + i * dim);
}

/* ---- optimizer.cpp:61-90 ------------------------------------------------ */

double or_effective_lr(double v, double eta, double eps, double c) {
  return eta / (sqrt(v / c) + eps); /* optimizer.cpp:61-63 */
}

/* optimizer.cpp:65-83. Returns lr, or NAN with *err set on nonfinite g. */
double or_adagrad_row_step(float* w, float* v, const double* g, uint32_t dim, double eta,
                           double eps, double c, int* err) {
  double norm_sq = 0.0;
  for (uint32_t j = 0; j < dim; ++j) {
    if (!isfinite(g[j])) {
      if (err) *err = OR_ENONFINITE;
      return NAN;
    }
    norm_sq += g[j] * g[j];
  }
  const float v_new = (float)((double)(*v) + norm_sq);
  *v = v_new;
  const double lr = or_effective_lr((double)v_new, eta, eps, c);
  for (uint32_t j = 0; j < dim; ++j) w[j] = (float)((double)w[j] - lr * g[j]);
  return lr;
}

void or_sgd_row_step(float* w, const double* g, uint32_t dim, double eta) { /* 85-90 */
  for (uint32_t j = 0; j < dim; ++j) w[j] = (float)((double)w[j] - eta * g[j]);
}

/* ---- embedding.cpp:39-92 pool_ids -------------------------------------- */
/* shards: n_shards x (row_lo,row_hi) over ONE table whose rows start at `w`
 * (row-major, dim floats).  Returns OR_ERANGE if an id is in no shard. */
int or_pool_ids(const float* w, uint32_t dim, uint32_t n_shards, const uint32_t* shard_lo_hi,
                const uint32_t* ids, uint32_t n_ids, float* out) {
  double pool[512], partial[512];
  if (n_shards == 0 || dim > 512) return OR_EINVAL;
  for (uint32_t j = 0; j < dim; ++j) out[j] = 0.0f;
  if (n_ids == 0) return OR_OK;
  for (uint32_t k = 0; k < n_ids; ++k) {
    int covered = 0;
    for (uint32_t s = 0; s < n_shards; ++s)
      if (ids[k] >= shard_lo_hi[2 * s] && ids[k] < shard_lo_hi[2 * s + 1]) covered = 1;
    if (!covered) return OR_ERANGE;
  }
  for (uint32_t j = 0; j < dim; ++j) pool[j] = 0.0;
  for (uint32_t s = 0; s < n_shards; ++s) {
    int hit = 0;
    for (uint32_t j = 0; j < dim; ++j) partial[j] = 0.0;
    for (uint32_t k = 0; k < n_ids; ++k) {
      if (ids[k] < shard_lo_hi[2 * s] || ids[k] >= shard_lo_hi[2 * s + 1]) continue;
      hit = 1;
      const float* row = w + (size_t)ids[k] * dim;
      for (uint32_t j = 0; j < dim; ++j) partial[j] += (double)row[j];
    }
    if (!hit) continue;
    for (uint32_t j = 0; j < dim; ++j) pool[j] += (double)(float)partial[j];
  }
  for (uint32_t j = 0; j < dim; ++j) out[j] = (float)pool[j];
  return OR_OK;
}

/* ---- embedding.cpp:108-129 apply_row_update ---------------------------- */
/* One call on a table of `dim`-float rows starting at `w`, shard [lo,hi).
 * OR_ERANGE outside the shard, OR_EINVAL for a negative / nonfinite moment
 * (checked in that order, nothing written on error). */
int or_apply_row_update(float* w, float* v, uint32_t lo, uint32_t hi, uint32_t dim, uint32_t row,
                        const double* delta, double new_moment) {
  if (row < lo || row >= hi) return OR_ERANGE;
  if (!(new_moment >= 0.0) || !isfinite(new_moment)) return OR_EINVAL;
  float* r = w + (size_t)row * dim;
  for (uint32_t j = 0; j < dim; ++j) r[j] = (float)((double)r[j] + delta[j]);
  v[row] = (float)new_moment;
  return OR_OK;
}

/* ---- planner.cpp:38-89 plan_greedy ------------------------------------- */
/* Writes up to F*N entries (table_id,row_lo,row_hi,local_rank) to out; returns
 * the count.  strategy 0 = table-wise (LPT), 1 = row-wise. */
typedef struct {
  uint32_t table_id;
  double load;
} or_lpt_item;

static int or_lpt_cmp(const void* a, const void* b) {
  const or_lpt_item* x = (const or_lpt_item*)a;
  const or_lpt_item* y = (const or_lpt_item*)b;
  if (x->load != y->load) return x->load > y->load ? -1 : 1;
  return x->table_id < y->table_id ? -1 : (x->table_id > y->table_id);
}

int or_plan_greedy(uint32_t n_tables, const uint32_t* table_ids, const double* lookups,
                   const uint64_t* num_rows, uint32_t n, int strategy, uint32_t* out) {
  if (n < 1 || n_tables == 0) return OR_EINVAL;
  int cnt = 0;
  if (strategy == 1) {
    for (uint32_t t = 0; t < n_tables; ++t) {
      for (uint32_t j = 0; j < n; ++j) {
        const uint32_t lo = (uint32_t)(num_rows[t] * j / n);
        const uint32_t hi = (uint32_t)(num_rows[t] * (j + 1) / n);
        if (hi > lo) {
          out[4 * cnt + 0] = table_ids[t];
          out[4 * cnt + 1] = lo;
          out[4 * cnt + 2] = hi;
          out[4 * cnt + 3] = j;
          ++cnt;
        }
      }
    }
    return cnt;
  }
  or_lpt_item* items = (or_lpt_item*)malloc(sizeof(or_lpt_item) * n_tables);
  double* load = (double*)calloc(n, sizeof(double));
  uint32_t* owner = (uint32_t*)malloc(sizeof(uint32_t) * n_tables);
  uint64_t* rows_of = (uint64_t*)malloc(sizeof(uint64_t) * n_tables);
  for (uint32_t t = 0; t < n_tables; ++t) {
    items[t].table_id = table_ids[t];
    items[t].load = lookups[t];
  }
  /* qsort is not stable, but the comparator is total over distinct ids */
  qsort(items, n_tables, sizeof(or_lpt_item), or_lpt_cmp);
  for (uint32_t i = 0; i < n_tables; ++i) {
    uint32_t best = 0;
    for (uint32_t r = 1; r < n; ++r)
      if (load[r] < load[best]) best = r;
    load[best] += items[i].load;
    owner[i] = best;
    for (uint32_t t = 0; t < n_tables; ++t)
      if (table_ids[t] == items[i].table_id) rows_of[i] = num_rows[t];
  }
  /* entries sorted by table_id (planner.cpp:80-84) */
  for (uint32_t i = 0; i < n_tables; ++i) {
    uint32_t k = 0;
    for (uint32_t j = 0; j < n_tables; ++j)
      if (items[j].table_id < items[i].table_id) ++k;
    out[4 * k + 0] = items[i].table_id;
    out[4 * k + 1] = 0;
    out[4 * k + 2] = (uint32_t)rows_of[i];
    out[4 * k + 3] = owner[i];
  }
  cnt = (int)n_tables;
  free(items);
  free(load);
  free(owner);
  free(rows_of);
  return cnt;
}

/* ---- the mesh step (trainer.cpp:283-611) -------------------------------- */

typedef struct {
  uint32_t F, N, B;
  const uint32_t* rows; /* [F] */
  const uint32_t* dims; /* [F] */
  uint32_t n_entries;
  const uint32_t* plan; /* [n_entries][4] table_id,row_lo,row_hi,local_rank */
  double eta, eps, c;
  int sgd; /* OptimizerVariant::Sgd */
  /* per-table pooling mode, NULL = all sum (the reference's only mode,
   * embedding.cpp:39-92).  Mean pooling is this build's extension (north
   * star K2 "sum/mean"); its definition, pinned here and mirrored by the
   * CUDA path:
   *   forward   out_j = f32( (sum_{o asc} f64(p_o,j)) * (1.0 / L) ), p_o the
   *             owners' f32 partial sums (the sum-pooling wire format), L
   *             the bag length; an empty bag pools to 0;
   *   backward  the gradient row sent for the bag is
   *             f32( f64(up_j) * (1.0 / L) ) (the f32 wire format of
   *             trainer.cpp:424-427 applied to d out / d row = 1/L); the
   *             owner then aggregates it exactly as for sum pooling. */
  const uint8_t* mean;
} or_cfg;

typedef struct {
  size_t* woff;
  size_t* voff;
  uint32_t* coff;
  uint32_t sum_dims;
  uint8_t** row_owner; /* [F][rows[f]] (trainer.cpp:203-214) */
} or_derived;

static int or_derive(const or_cfg* c, or_derived* d) {
  d->woff = (size_t*)malloc(sizeof(size_t) * (c->F + 1));
  d->voff = (size_t*)malloc(sizeof(size_t) * (c->F + 1));
  d->coff = (uint32_t*)malloc(sizeof(uint32_t) * (c->F + 1));
  d->row_owner = (uint8_t**)calloc(c->F, sizeof(uint8_t*));
  if (!d->woff || !d->voff || !d->coff || !d->row_owner) return OR_ENOMEM;
  d->woff[0] = 0;
  d->voff[0] = 0;
  d->coff[0] = 0;
  for (uint32_t f = 0; f < c->F; ++f) {
    d->woff[f + 1] = d->woff[f] + (size_t)c->rows[f] * c->dims[f];
    d->voff[f + 1] = d->voff[f] + c->rows[f];
    d->coff[f + 1] = d->coff[f] + c->dims[f];
    d->row_owner[f] = (uint8_t*)calloc(c->rows[f], 1);
    if (!d->row_owner[f]) return OR_ENOMEM;
    for (uint32_t e = 0; e < c->n_entries; ++e) {
      const uint32_t* pe = c->plan + 4 * e;
      if (pe[0] != f) continue;
      for (uint32_t r = pe[1]; r < pe[2] && r < c->rows[f]; ++r) d->row_owner[f][r] = (uint8_t)pe[3];
    }
  }
  d->sum_dims = d->coff[c->F];
  return OR_OK;
}

static void or_free_derived(const or_cfg* c, or_derived* d) {
  if (d->row_owner)
    for (uint32_t f = 0; f < c->F; ++f) free(d->row_owner[f]);
  free(d->row_owner);
  free(d->woff);
  free(d->voff);
  free(d->coff);
}

size_t or_replica_floats(uint32_t F, const uint32_t* rows, const uint32_t* dims) {
  size_t s = 0;
  for (uint32_t f = 0; f < F; ++f) s += (size_t)rows[f] * dims[f];
  return s;
}

size_t or_replica_rows(uint32_t F, const uint32_t* rows) {
  size_t s = 0;
  for (uint32_t f = 0; f < F; ++f) s += rows[f];
  return s;
}

/* Optional layout dumps for the bit-exact a2a layout checks.  Any pointer may
 * be NULL.  Capacities are the caller's responsibility (see oracle.py). */
typedef struct {
  uint32_t* dem_len;   /* [N owner][N requester][B*F]: ids of bag owned by o */
  uint32_t* dem_ids;   /* [N owner][cap_ids] canonical demand ids (global) */
  uint64_t* dem_nnz;   /* [N owner] */
  uint32_t* mask;      /* [N requester][B*F] owner bitmask */
  float* part;         /* [N owner][cap_floats]: send_lookup[o][n] concat over n */
  uint64_t* part_cnt;  /* [N owner][N requester] floats */
  float* grad;         /* [N requester][cap_floats]: send_grad[n][o] concat over o */
  uint64_t* grad_cnt;  /* [N requester][N owner] floats */
  uint64_t cap_ids, cap_floats;
} or_dump;

/* One MP group's step: build_demand (trainer.cpp:283-313), owner_lookup
 * (316-338), the lookup all-to-all (topology.cpp:57-118), requester combine
 * (366-390), grad payloads (440-457), grad all-to-all, owner_update
 * (459-505).  Updates the group's replica (w, v) in place and marks dirty
 * rows (trainer.cpp:502). */
int or_group_step(const or_cfg* c, const uint32_t* const* lengths, const uint32_t* const* ids,
                  const float* const* upstream, float* const* pooled, float* w, float* v,
                  uint8_t* dirty, or_dump* dump) {
  const uint32_t F = c->F, N = c->N, B = c->B, BF = c->B * c->F;
  or_derived d;
  memset(&d, 0, sizeof(d));
  int rc = or_derive(c, &d);
  if (rc) {
    or_free_derived(c, &d);
    return rc;
  }
  if (N > 32) {
    or_free_derived(c, &d);
    return OR_EINVAL;
  }
  uint64_t total_ids = 0;
  uint64_t** roff = (uint64_t**)calloc(N, sizeof(uint64_t*)); /* per requester bag offsets */
  for (uint32_t n = 0; n < N; ++n) {
    roff[n] = (uint64_t*)malloc(sizeof(uint64_t) * (BF + 1));
    roff[n][0] = 0;
    for (uint32_t b = 0; b < BF; ++b) roff[n][b + 1] = roff[n][b] + lengths[n][b];
    total_ids += roff[n][BF];
  }
  /* bounds check: the reference indexes row_owner[f][id] unchecked
   * (trainer.cpp:293-299); pool_ids reports out_of_range (embedding.cpp:61). */
  for (uint32_t n = 0; n < N; ++n)
    for (uint32_t b = 0; b < BF; ++b)
      for (uint64_t k = roff[n][b]; k < roff[n][b + 1]; ++k)
        if (ids[n][k] >= c->rows[b % F]) rc = OR_ERANGE;
  /* ---- build_demand ---- */
  uint32_t* mask = (uint32_t*)calloc((size_t)N * BF, sizeof(uint32_t));
  uint32_t* dlen = (uint32_t*)calloc((size_t)N * N * BF, sizeof(uint32_t)); /* [o][n][b] */
  uint32_t** dids = (uint32_t**)calloc(N, sizeof(uint32_t*));
  uint64_t* dnnz = (uint64_t*)calloc(N, sizeof(uint64_t));
  for (uint32_t o = 0; o < N; ++o) dids[o] = (uint32_t*)malloc(sizeof(uint32_t) * (total_ids + 1));
  if (rc) goto done;
  for (uint32_t n = 0; n < N; ++n) {
    for (uint32_t s = 0; s < B; ++s) {
      for (uint32_t f = 0; f < F; ++f) {
        const uint32_t b = s * F + f;
        uint32_t m = 0;
        for (uint32_t o = 0; o < N; ++o) {
          uint32_t cnt = 0;
          for (uint64_t k = roff[n][b]; k < roff[n][b + 1]; ++k) {
            const uint32_t id = ids[n][k];
            if (d.row_owner[f][id] == o) {
              dids[o][dnnz[o]++] = id;
              ++cnt;
            }
          }
          if (cnt) {
            dlen[((size_t)o * N + n) * BF + b] = cnt;
            m |= 1u << o;
          }
        }
        mask[(size_t)n * BF + b] = m;
      }
    }
  }
  /* ---- owner_lookup: send_lookup[o][n], entries in canonical order ---- */
  {
    uint64_t* pcnt = (uint64_t*)calloc((size_t)N * N, sizeof(uint64_t));
    for (uint32_t o = 0; o < N; ++o)
      for (uint32_t n = 0; n < N; ++n)
        for (uint32_t b = 0; b < BF; ++b)
          if (dlen[((size_t)o * N + n) * BF + b]) pcnt[o * N + n] += c->dims[b % F];
    float*** send = (float***)calloc(N, sizeof(float**)); /* [o][n] */
    for (uint32_t o = 0; o < N; ++o) {
      send[o] = (float**)calloc(N, sizeof(float*));
      for (uint32_t n = 0; n < N; ++n) send[o][n] = (float*)malloc(sizeof(float) * (pcnt[o * N + n] + 1));
    }
    double partial[512];
    for (uint32_t o = 0; o < N; ++o) {
      uint64_t cur = 0;
      uint64_t* fill = (uint64_t*)calloc(N, sizeof(uint64_t));
      for (uint32_t n = 0; n < N; ++n) {
        for (uint32_t b = 0; b < BF; ++b) {
          const uint32_t cnt = dlen[((size_t)o * N + n) * BF + b];
          if (!cnt) continue;
          const uint32_t f = b % F, D = c->dims[f];
          for (uint32_t j = 0; j < D; ++j) partial[j] = 0.0;
          for (uint32_t k = 0; k < cnt; ++k) {
            const float* row = w + d.woff[f] + (size_t)dids[o][cur + k] * D;
            for (uint32_t j = 0; j < D; ++j) partial[j] += (double)row[j];
          }
          cur += cnt;
          for (uint32_t j = 0; j < D; ++j) send[o][n][fill[n]++] = (float)partial[j];
        }
      }
      free(fill);
    }
    /* ---- route_all_to_all: delivered[n][o] = send[o][n] ---- */
    /* ---- pool_and_forward combine (trainer.cpp:372-390) ---- */
    for (uint32_t n = 0; n < N; ++n) {
      uint64_t cursor[32] = {0};
      for (uint32_t s = 0; s < B; ++s) {
        for (uint32_t f = 0; f < F; ++f) {
          const uint32_t b = s * F + f, D = c->dims[f];
          const uint32_t m = mask[(size_t)n * BF + b];
          double pool[512];
          for (uint32_t j = 0; j < D; ++j) pool[j] = 0.0;
          for (uint32_t o = 0; o < N; ++o) {
            if (!(m & (1u << o))) continue;
            const float* part = send[o][n] + cursor[o];
            for (uint32_t j = 0; j < D; ++j) pool[j] += (double)part[j];
            cursor[o] += D;
          }
          float* out = pooled[n] + (size_t)s * d.sum_dims + d.coff[f];
          const uint32_t L = lengths[n][b];
          if (c->mean && c->mean[f] && L) {
            const double inv = 1.0 / (double)L;
            for (uint32_t j = 0; j < D; ++j) out[j] = (float)(pool[j] * inv);
          } else {
            for (uint32_t j = 0; j < D; ++j) out[j] = (float)pool[j];
          }
        }
      }
    }
    if (dump && dump->part) {
      for (uint32_t o = 0; o < N; ++o) {
        uint64_t at = 0;
        for (uint32_t n = 0; n < N; ++n) {
          memcpy(dump->part + o * dump->cap_floats + at, send[o][n], sizeof(float) * pcnt[o * N + n]);
          at += pcnt[o * N + n];
          if (dump->part_cnt) dump->part_cnt[o * N + n] = pcnt[o * N + n];
        }
      }
    }
    for (uint32_t o = 0; o < N; ++o) {
      for (uint32_t n = 0; n < N; ++n) free(send[o][n]);
      free(send[o]);
    }
    free(send);
    free(pcnt);
  }
  /* ---- build_grad_payloads: send_grad[n][o] (trainer.cpp:440-457) ---- */
  {
    uint64_t* gcnt = (uint64_t*)calloc((size_t)N * N, sizeof(uint64_t));
    for (uint32_t n = 0; n < N; ++n)
      for (uint32_t b = 0; b < BF; ++b)
        for (uint32_t o = 0; o < N; ++o)
          if (mask[(size_t)n * BF + b] & (1u << o)) gcnt[n * N + o] += c->dims[b % F];
    float*** sg = (float***)calloc(N, sizeof(float**)); /* [n][o] */
    for (uint32_t n = 0; n < N; ++n) {
      sg[n] = (float**)calloc(N, sizeof(float*));
      uint64_t fill[32] = {0};
      for (uint32_t o = 0; o < N; ++o) sg[n][o] = (float*)malloc(sizeof(float) * (gcnt[n * N + o] + 1));
      for (uint32_t s = 0; s < B; ++s) {
        const float* up = upstream[n] + (size_t)s * d.sum_dims;
        for (uint32_t f = 0; f < F; ++f) {
          const uint32_t m = mask[(size_t)n * BF + s * F + f], D = c->dims[f];
          const uint32_t L = lengths[n][s * F + f];
          const int scale = c->mean && c->mean[f] && L;
          const double inv = scale ? 1.0 / (double)L : 1.0;
          for (uint32_t o = 0; o < N; ++o) {
            if (!(m & (1u << o))) continue;
            if (scale)
              for (uint32_t j = 0; j < D; ++j) sg[n][o][fill[o] + j] = (float)((double)up[d.coff[f] + j] * inv);
            else
              memcpy(sg[n][o] + fill[o], up + d.coff[f], sizeof(float) * D);
            fill[o] += D;
          }
        }
      }
    }
    if (dump && dump->grad) {
      for (uint32_t n = 0; n < N; ++n) {
        uint64_t at = 0;
        for (uint32_t o = 0; o < N; ++o) {
          memcpy(dump->grad + n * dump->cap_floats + at, sg[n][o], sizeof(float) * gcnt[n * N + o]);
          at += gcnt[n * N + o];
          if (dump->grad_cnt) dump->grad_cnt[n * N + o] = gcnt[n * N + o];
        }
      }
    }
    /* ---- owner_update (trainer.cpp:459-505) + aggregate_group_gradient
     * (optimizer.cpp:25-59): per feature, contributions in canonical arrival
     * order, stable-sorted by row, f64 sums, x 1/(N*B), then the row step. */
    const double inv_batch = 1.0 / (double)((uint64_t)N * B);
    for (uint32_t o = 0; o < N && rc == OR_OK; ++o) {
      /* contribution list per feature: (row, pointer to f32 grad row) */
      uint64_t ncontrib = dnnz[o];
      uint32_t* crow = (uint32_t*)malloc(sizeof(uint32_t) * (ncontrib + 1));
      const float** cgrad = (const float**)malloc(sizeof(float*) * (ncontrib + 1));
      uint32_t* cfeat = (uint32_t*)malloc(sizeof(uint32_t) * (ncontrib + 1));
      uint64_t cur = 0, k = 0;
      for (uint32_t n = 0; n < N; ++n) {
        uint64_t gcur = 0;
        for (uint32_t b = 0; b < BF; ++b) {
          const uint32_t cnt = dlen[((size_t)o * N + n) * BF + b];
          if (!cnt) continue;
          const uint32_t f = b % F;
          const float* g = sg[n][o] + gcur;
          gcur += c->dims[f];
          for (uint32_t q = 0; q < cnt; ++q, ++k) {
            crow[k] = dids[o][cur + q];
            cgrad[k] = g;
            cfeat[k] = f;
          }
          cur += cnt;
        }
      }
      /* per feature: stable counting by row via insertion into per-row lists
       * (equivalent to std::stable_sort by row, optimizer.cpp:31-35) */
      for (uint32_t f = 0; f < F && rc == OR_OK; ++f) {
        const uint32_t R = c->rows[f], D = c->dims[f];
        uint32_t* head_cnt = (uint32_t*)calloc((size_t)R + 1, sizeof(uint32_t));
        uint64_t nf = 0;
        for (uint64_t i = 0; i < ncontrib; ++i)
          if (cfeat[i] == f) {
            head_cnt[crow[i] + 1]++;
            ++nf;
          }
        if (nf == 0) {
          free(head_cnt);
          continue;
        }
        for (uint32_t r = 0; r < R; ++r) head_cnt[r + 1] += head_cnt[r];
        uint64_t* order = (uint64_t*)malloc(sizeof(uint64_t) * nf);
        uint32_t* fillp = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)R + 1));
        memcpy(fillp, head_cnt, sizeof(uint32_t) * ((size_t)R + 1));
        for (uint64_t i = 0; i < ncontrib; ++i)
          if (cfeat[i] == f) order[fillp[crow[i]]++] = i;
        double g[512];
        for (uint32_t r = 0; r < R && rc == OR_OK; ++r) {
          if (head_cnt[r] == head_cnt[r + 1]) continue;
          for (uint32_t j = 0; j < D; ++j) g[j] = 0.0;
          for (uint32_t q = head_cnt[r]; q < head_cnt[r + 1]; ++q) {
            const float* gr = cgrad[order[q]];
            for (uint32_t j = 0; j < D; ++j) g[j] += (double)gr[j];
          }
          for (uint32_t j = 0; j < D; ++j) g[j] *= inv_batch;
          float* wr = w + d.woff[f] + (size_t)r * D;
          if (c->sgd) {
            or_sgd_row_step(wr, g, D, c->eta);
          } else {
            int err = OR_OK;
            or_adagrad_row_step(wr, v + d.voff[f] + r, g, D, c->eta, c->eps, c->c, &err);
            if (err) rc = err;
          }
          if (dirty) dirty[d.voff[f] + r] = 1;
        }
        free(order);
        free(fillp);
        free(head_cnt);
      }
      free(crow);
      free(cgrad);
      free(cfeat);
    }
    for (uint32_t n = 0; n < N; ++n) {
      for (uint32_t o = 0; o < N; ++o) free(sg[n][o]);
      free(sg[n]);
    }
    free(sg);
    free(gcnt);
  }
  if (dump) {
    if (dump->dem_len) memcpy(dump->dem_len, dlen, sizeof(uint32_t) * (size_t)N * N * BF);
    if (dump->mask) memcpy(dump->mask, mask, sizeof(uint32_t) * (size_t)N * BF);
    for (uint32_t o = 0; o < N; ++o) {
      if (dump->dem_nnz) dump->dem_nnz[o] = dnnz[o];
      if (dump->dem_ids) memcpy(dump->dem_ids + o * dump->cap_ids, dids[o], sizeof(uint32_t) * dnnz[o]);
    }
  }
done:
  for (uint32_t n = 0; n < N; ++n) free(roff[n]);
  free(roff);
  for (uint32_t o = 0; o < N; ++o) free(dids[o]);
  free(dids);
  free(dnnz);
  free(dlen);
  free(mask);
  or_free_derived(c, &d);
  return rc;
}

/* sync_replicas (trainer.cpp:547-596): for every row dirty in any group,
 * x = f32((sum_{g ascending} f64(x_g)) * (1/M)), weights then moments (moments
 * skipped for SGD); dirty flags cleared. */
int or_sync(uint32_t M, uint32_t F, const uint32_t* rows, const uint32_t* dims, int sgd,
            float* const* w, float* const* v, uint8_t* const* dirty) {
  const double inv_m = 1.0 / (double)M;
  size_t woff = 0, voff = 0;
  for (uint32_t f = 0; f < F; ++f) {
    const uint32_t D = dims[f];
    for (uint32_t r = 0; r < rows[f]; ++r) {
      int is_dirty = 0;
      for (uint32_t g = 0; g < M; ++g) is_dirty |= dirty[g][voff + r];
      if (!is_dirty) continue;
      for (uint32_t j = 0; j < D; ++j) {
        double acc = 0.0;
        for (uint32_t g = 0; g < M; ++g) acc += (double)w[g][woff + (size_t)r * D + j];
        const float mean = (float)(acc * inv_m);
        for (uint32_t g = 0; g < M; ++g) w[g][woff + (size_t)r * D + j] = mean;
      }
      if (!sgd) {
        double acc = 0.0;
        for (uint32_t g = 0; g < M; ++g) acc += (double)v[g][voff + r];
        const float mean = (float)(acc * inv_m);
        for (uint32_t g = 0; g < M; ++g) v[g][voff + r] = mean;
      }
      for (uint32_t g = 0; g < M; ++g) dirty[g][voff + r] = 0;
    }
    woff += (size_t)rows[f] * D;
    voff += rows[f];
  }
  return OR_OK;
}

/* deterministic_mean_inplace (topology.cpp:150-163) */
void or_deterministic_mean(uint32_t m, float* const* reps, size_t len) {
  const double inv_m = 1.0 / (double)m;
  for (size_t i = 0; i < len; ++i) {
    double acc = 0.0;
    for (uint32_t g = 0; g < m; ++g) acc += (double)reps[g][i];
    const float mean = (float)(acc * inv_m);
    for (uint32_t g = 0; g < m; ++g) reps[g][i] = mean;
  }
}

/* ---- synthetic upstream gradient ------------------------
 * upstream[s][coff_f + j] = f32(1e-3 * N(0,1)) from CounterRng({seed, step,
 * rank, s, f}) Box-Muller pairs (rng.hpp:42-56). */
void or_synthetic_upstream(uint64_t seed, uint64_t step, uint32_t rank, uint32_t B, uint32_t F,
                           const uint32_t* dims, float* out) {
  uint32_t sum = 0;
  for (uint32_t f = 0; f < F; ++f) sum += dims[f];
  for (uint32_t s = 0; s < B; ++s) {
    uint32_t col = 0;
    for (uint32_t f = 0; f < F; ++f) {
      const uint64_t k[5] = {seed, step, rank, s, f};
      const uint64_t key = or_make_key(k, 5);
      uint64_t ctr = 0;
      double spare = 0.0;
      int have = 0;
      for (uint32_t j = 0; j < dims[f]; ++j) {
        double z;
        if (have) {
          z = spare;
          have = 0;
        } else {
          const double u1 = (double)((or_mix64(key + (++ctr) * 0x9E3779B97F4A7C15ULL) >> 11) + 1) * 0x1.0p-53;
          const double u2 = (double)(or_mix64(key + (++ctr) * 0x9E3779B97F4A7C15ULL) >> 11) * 0x1.0p-53;
          const double r = sqrt(-2.0 * log(u1));
          const double t = 2.0 * 3.141592653589793 * u2;
          spare = r * sin(t);
          have = 1;
          z = r * cos(t);
        }
        out[(size_t)s * sum + col + j] = (float)(1e-3 * z);
      }
      col += dims[f];
    }
  }
}

/* ---- S2DCKPT1 checkpoint writer (embedding.cpp:133-185) --------------------
 * "S2DCKPT1", u32 table count, then per table: u32 version (1), u32 table_id,
 * u64 rows, u64 dim, f32 weights[rows*dim], f32 moments[rows]; little-endian
 * host order; written to path.tmp and renamed.  Tables are the flat replica
 * (table f's rows at woff/voff), table_id = f.  Returns 0, or -1 on IO error. */
int or_save_checkpoint(const char* path, uint32_t F, const uint32_t* rows, const uint32_t* dims, const float* w,
                       const float* v) {
  char tmp[4096];
  if (strlen(path) + 5 >= sizeof(tmp)) return -1;
  strcpy(tmp, path);
  strcat(tmp, ".tmp");
  FILE* f = fopen(tmp, "wb");
  if (!f) return -1;
  int ok = fwrite("S2DCKPT1", 1, 8, f) == 8 && fwrite(&F, 4, 1, f) == 1;
  size_t woff = 0, voff = 0;
  for (uint32_t t = 0; ok && t < F; ++t) {
    const uint32_t version = 1;
    const uint64_t r = rows[t], d = dims[t];
    ok = fwrite(&version, 4, 1, f) == 1 && fwrite(&t, 4, 1, f) == 1 && fwrite(&r, 8, 1, f) == 1 &&
         fwrite(&d, 8, 1, f) == 1 && fwrite(w + woff, 4, r * d, f) == r * d && fwrite(v + voff, 4, r, f) == r;
    woff += r * d;
    voff += r;
  }
  if (fclose(f) != 0) ok = 0;
  if (!ok) return -1;
  return rename(tmp, path) == 0 ? 0 : -1;
}

/* ---- DataGenerator ids (data.cpp:85-98 Zipf CDF, 115-136 gen_batch_into) --
 * cdf_f[k] = (sum_{i<=k} (i+1)^-s_f) / total_f in sequential f64, last = 1.
 * Bag (s, f) draws L_f ids: u = CounterRng({seed, lane=0, step, rank, s,
 * tag=1, f}).next_uniform(); id = min(upper_bound(cdf_f, u), rows_f - 1).
 * Output: sample-major bags, ids in (s, f, draw) order.  Returns 0. */
static uint32_t or_upper_bound(const double* cdf, uint32_t n, double u) {
  uint32_t lo = 0, hi = n; /* first index with cdf[i] > u */
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo) / 2;
    if (cdf[mid] > u)
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

void or_zipf_cdf(uint32_t rows, double s, double* cdf) { /* data.cpp:88-97 */
  double total = 0.0;
  for (uint32_t k = 0; k < rows; ++k) {
    total += pow((double)(k + 1), -s);
    cdf[k] = total;
  }
  for (uint32_t k = 0; k < rows; ++k) cdf[k] /= total;
  cdf[rows - 1] = 1.0;
}

int or_gen_batch_ids(uint64_t seed, uint64_t step, uint32_t rank, uint32_t F, const uint32_t* rows,
                     const double* zipf, const uint32_t* L, uint32_t B, uint32_t* out_ids) {
  double** cdf = (double**)calloc(F, sizeof(double*));
  if (!cdf) return OR_ENOMEM;
  for (uint32_t f = 0; f < F; ++f) {
    cdf[f] = (double*)malloc(sizeof(double) * rows[f]);
    if (!cdf[f]) return OR_ENOMEM;
    or_zipf_cdf(rows[f], zipf[f], cdf[f]);
  }
  size_t k = 0;
  for (uint32_t s = 0; s < B; ++s)
    for (uint32_t f = 0; f < F; ++f) {
      const uint64_t fl[7] = {seed, 0, step, rank, s, 1, f};
      const uint64_t key = or_make_key(fl, 7);
      for (uint32_t j = 0; j < L[f]; ++j) {
        const uint64_t z = key + (uint64_t)(j + 1) * 0x9E3779B97F4A7C15ULL;
        const double u = (double)(or_mix64(z) >> 11) * 0x1.0p-53;
        const uint32_t i = or_upper_bound(cdf[f], rows[f], u);
        out_ids[k++] = i < rows[f] - 1 ? i : rows[f] - 1;
      }
    }
  for (uint32_t f = 0; f < F; ++f) free(cdf[f]);
  free(cdf);
  return OR_OK;
}

/* ---- MetricsRow moment columns (trainer.cpp:745-771) ------------------- */

static int or_cmp_f64(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* Over every row of the replica (v: n moments, tables in order):
 * lrs[i] = effective_lr(v[i]); out[0] = lrs at ascending index
 * ceil(0.5 n) - 1, out[1] = at ceil(0.99 n) - 1 (nth_element == the sorted
 * value), out[2] = v_sum / n with v_sum the sequential f64 sum. */
int or_metrics_row(const float* v, uint64_t n, double eta, double eps, double c, double* out) {
  if (n == 0) return OR_EINVAL;
  double* lrs = (double*)malloc(sizeof(double) * n);
  if (!lrs) return OR_ENOMEM;
  double v_sum = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    v_sum += (double)v[i];
    lrs[i] = or_effective_lr((double)v[i], eta, eps, c);
  }
  qsort(lrs, n, sizeof(double), or_cmp_f64);
  const uint64_t i50 = (uint64_t)ceil(0.50 * (double)n) - 1, i99 = (uint64_t)ceil(0.99 * (double)n) - 1;
  out[0] = lrs[i50];
  out[1] = lrs[i99];
  out[2] = v_sum / (double)n;
  free(lrs);
  return OR_OK;
}

/* The f64 row gradients of one rank's step at N = 1 (aggregate_group_gradient,
 * optimizer.cpp:25-59; owner_update, trainer.cpp:459-505): for every touched
 * (table, row) in ascending (table, row) order, g_j = (sum over the row's ids
 * in item order of f64(up[s][coff_f + j])) * (1.0 / B).  rows_out[u] =
 * (table << 32 | row); g_out: u x max_dim (row-major, zero-padded). Returns
 * the number of touched rows (or < 0 if a capacity is exceeded). */
int64_t or_row_gradients(uint32_t F, const uint32_t* rows, const uint32_t* dims, uint32_t B, const uint32_t* lengths,
                         const uint32_t* ids, const float* upstream, uint64_t cap, uint64_t* rows_out,
                         double* g_out) {
  uint32_t sum_dims = 0, max_dim = 0;
  for (uint32_t f = 0; f < F; ++f) {
    sum_dims += dims[f];
    if (dims[f] > max_dim) max_dim = dims[f];
  }
  uint32_t* coff = (uint32_t*)malloc(sizeof(uint32_t) * (F + 1));
  coff[0] = 0;
  for (uint32_t f = 0; f < F; ++f) coff[f + 1] = coff[f] + dims[f];
  const uint64_t BF = (uint64_t)B * F;
  uint64_t nnz = 0;
  for (uint64_t b = 0; b < BF; ++b) nnz += lengths[b];
  /* per table: counting sort of items by row (stable) */
  uint64_t* item_bag = (uint64_t*)malloc(sizeof(uint64_t) * (nnz + 1));
  uint64_t* item_table_off = (uint64_t*)calloc(F + 1, sizeof(uint64_t));
  {
    uint64_t k = 0;
    for (uint64_t b = 0; b < BF; ++b)
      for (uint32_t q = 0; q < lengths[b]; ++q) item_bag[k++] = b;
  }
  int64_t u = 0;
  const double inv_b = 1.0 / (double)B;
  for (uint32_t f = 0; f < F && u >= 0; ++f) {
    const uint32_t R = rows[f], D = dims[f];
    uint64_t* cnt = (uint64_t*)calloc((size_t)R + 1, sizeof(uint64_t));
    uint64_t nf = 0;
    for (uint64_t i = 0; i < nnz; ++i)
      if (item_bag[i] % F == f) {
        cnt[ids[i] + 1]++;
        ++nf;
      }
    for (uint32_t r = 0; r < R; ++r) cnt[r + 1] += cnt[r];
    uint64_t* order = (uint64_t*)malloc(sizeof(uint64_t) * (nf + 1));
    uint64_t* fill = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)R + 1));
    memcpy(fill, cnt, sizeof(uint64_t) * ((size_t)R + 1));
    for (uint64_t i = 0; i < nnz; ++i)
      if (item_bag[i] % F == f) order[fill[ids[i]]++] = i;
    for (uint32_t r = 0; r < R; ++r) {
      if (cnt[r] == cnt[r + 1]) continue;
      if ((uint64_t)u >= cap) {
        u = -1;
        break;
      }
      double* g = g_out + (uint64_t)u * max_dim;
      for (uint32_t j = 0; j < max_dim; ++j) g[j] = 0.0;
      for (uint64_t q = cnt[r]; q < cnt[r + 1]; ++q) {
        const uint64_t b = item_bag[order[q]];
        const float* up = upstream + (b / F) * sum_dims + coff[f];
        for (uint32_t j = 0; j < D; ++j) g[j] += (double)up[j];
      }
      for (uint32_t j = 0; j < D; ++j) g[j] *= inv_b;
      rows_out[u] = ((uint64_t)f << 32) | r;
      ++u;
    }
    free(order);
    free(fill);
    free(cnt);
  }
  free(item_bag);
  free(item_table_off);
  free(coff);
  return u;
}
