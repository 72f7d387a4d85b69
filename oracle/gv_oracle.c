/*
 * gv_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, serial C implementation of what the GraphVite GPU hot path
 * computes (Zhu et al., arXiv 1903.00757), written from PAPER.md and the
 * readings in DESIGN.md / SURVEY.md §8(c). It is the parity oracle for the
 * CUDA path in paper_1903_00757_b200/csrc and shares no code with it.
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
 * --impl reference legs) may load it. Build:
 *   gcc -O2 -std=gnu11 -ffp-contract=off -fPIC -shared gv_oracle.c -lm
 * (-ffp-contract=off: every float operation is rounded as written.)
 *
 * Pins (tests/test_oracle_*.py): Philox KATs; exact alias mass identity and
 * chi-square; zig-zag worked example; stable-sort and conservation
 * of bucketing vs numpy (and of the vertex-tile order, R-VTILE, vs numpy's
 * stable sort per block); the hand-derived 4-node SGD example and finite
 * differences of the objective; schedule coverage; AUC vs sklearn.
 * Parity unpinned against the paper itself: the paper prints no intermediate
 * values (SURVEY §8(c) "Against the paper").
 */
#include "gv_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ===================================================================== */
/* Philox4x32-10. Step 4. Multipliers and Weyl constants from Salmon et al.
 * (2011), Random123 philox.h. Round r uses the key bumped r times.         */
/* ===================================================================== */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; r++) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static void seed_to_key(uint64_t seed, uint32_t key[2]) {
  key[0] = (uint32_t)seed;
  key[1] = (uint32_t)(seed >> 32);
}

/* ===================================================================== */
/* Graph ingest. Step 1: drop self-loops, symmetrise, sum duplicate weights
 * (in input order, double), weighted degree summed in ascending neighbour
 * id. P:392 "We treat networks as undirected graphs".      */
/* ===================================================================== */
struct or_graph {
  uint32_t nv;
  uint64_t n_entries;
  uint64_t* off;
  uint32_t* nbr;
  double* w;
  double* deg;
};

/* The symmetrised entries (row, col, input index k) are put in (row, col,
 * k) order by two STABLE counting sorts — by col, then by row (an LSD radix
 * sort with one digit per node id) — over the entries generated in input
 * order (edge k gives (src,dst,k) then (dst,src,k)). That is the order a
 * comparison sort by (row, col, k) gives, in time linear in |E| (the
 * Friendster-sized graph has 3.6e9 entries). Runs of equal (row, col)
 * are then merged, summing their weights in input order. Inputs with
 * 2^32 or more edges are rejected (k is stored in 32 bits).               */
int or_graph_build(uint32_t nv, const uint32_t* src, const uint32_t* dst,
                   const float* w, uint64_t ne, or_graph** out) {
  *out = NULL;
  if (nv == 0) return OR_ERR_INVALID_ARG;
  if (ne >= ((uint64_t)1 << 32)) return OR_ERR_INVALID_ARG;
  for (uint64_t k = 0; k < ne; k++) {
    if (src[k] >= nv || dst[k] >= nv) return OR_ERR_OUT_OF_RANGE;
    if (w && (!isfinite(w[k]) || w[k] < 0.0f)) return OR_ERR_INVALID_ARG;
  }
  uint64_t* cnt_col = (uint64_t*)calloc((size_t)nv + 1, sizeof(uint64_t));
  uint64_t* cnt_row = (uint64_t*)calloc((size_t)nv + 1, sizeof(uint64_t));
  if (!cnt_col || !cnt_row) { free(cnt_col); free(cnt_row); return OR_ERR_NOMEM; }
  /* entry counts per column and per row (symmetric: the same numbers) */
  uint64_t n_dir = 0;
  for (uint64_t k = 0; k < ne; k++) {
    if (src[k] == dst[k]) continue;
    cnt_col[dst[k] + 1]++; cnt_col[src[k] + 1]++;
    cnt_row[src[k] + 1]++; cnt_row[dst[k] + 1]++;
    n_dir += 2;
  }
  if (n_dir == 0) { free(cnt_col); free(cnt_row); return OR_ERR_EMPTY; }
  for (uint32_t v = 0; v < nv; v++) {
    cnt_col[v + 1] += cnt_col[v];
    cnt_row[v + 1] += cnt_row[v];
  }
  /* pass 1: stable by col; by_col[] holds (row, k), its col is implied */
  uint32_t* by_col = (uint32_t*)malloc(n_dir * 2 * sizeof(uint32_t));
  uint64_t* fill = (uint64_t*)malloc(((size_t)nv + 1) * sizeof(uint64_t));
  if (!by_col || !fill) { free(by_col); free(fill); free(cnt_col); free(cnt_row); return OR_ERR_NOMEM; }
  memcpy(fill, cnt_col, ((size_t)nv + 1) * sizeof(uint64_t));
  for (uint64_t k = 0; k < ne; k++) {
    uint32_t a = src[k], b = dst[k];
    if (a == b) continue;
    uint64_t q = fill[b]++; by_col[2 * q] = a; by_col[2 * q + 1] = (uint32_t)k; /* (a, b, k) */
    q = fill[a]++;          by_col[2 * q] = b; by_col[2 * q + 1] = (uint32_t)k; /* (b, a, k) */
  }
  /* pass 2: stable by row; by_row[] holds (col, k) in (row, col, k) order */
  uint32_t* by_row = (uint32_t*)malloc(n_dir * 2 * sizeof(uint32_t));
  if (!by_row) { free(by_col); free(fill); free(cnt_col); free(cnt_row); return OR_ERR_NOMEM; }
  memcpy(fill, cnt_row, ((size_t)nv + 1) * sizeof(uint64_t));
  for (uint32_t col = 0; col < nv; col++) {
    for (uint64_t q = cnt_col[col]; q < cnt_col[col + 1]; q++) {
      uint64_t r = fill[by_col[2 * q]]++;
      by_row[2 * r] = col;
      by_row[2 * r + 1] = by_col[2 * q + 1];
    }
  }
  free(by_col);
  free(fill);
  free(cnt_col);
  /* merge runs of equal (row, col), summing weights in input order */
  uint64_t m = 0;
  for (uint32_t row = 0; row < nv; row++)
    for (uint64_t q = cnt_row[row]; q < cnt_row[row + 1]; q++)
      if (q == cnt_row[row] || by_row[2 * q] != by_row[2 * (q - 1)]) m++;
  or_graph* g = (or_graph*)calloc(1, sizeof(or_graph));
  if (!g) { free(by_row); free(cnt_row); return OR_ERR_NOMEM; }
  g->nv = nv;
  g->n_entries = m;
  g->off = (uint64_t*)calloc((size_t)nv + 1, sizeof(uint64_t));
  g->nbr = (uint32_t*)malloc(m * sizeof(uint32_t));
  g->w = (double*)malloc(m * sizeof(double));
  g->deg = (double*)calloc(nv, sizeof(double));
  if (!g->off || !g->nbr || !g->w || !g->deg) {
    free(by_row); free(cnt_row); or_graph_free(g); return OR_ERR_NOMEM;
  }
  uint64_t o = 0;
  for (uint32_t row = 0; row < nv; row++) {
    g->off[row] = o;
    for (uint64_t q = cnt_row[row]; q < cnt_row[row + 1]; q++) {
      double wk = w ? (double)w[by_row[2 * q + 1]] : 1.0;
      if (q == cnt_row[row] || by_row[2 * q] != by_row[2 * (q - 1)]) {
        g->nbr[o] = by_row[2 * q];
        g->w[o] = wk;
        o++;
      } else {
        g->w[o - 1] += wk;
      }
    }
  }
  g->off[nv] = o;
  for (uint32_t v = 0; v < nv; v++) {
    double s = 0.0;
    for (uint64_t q = g->off[v]; q < g->off[v + 1]; q++) s += g->w[q];
    g->deg[v] = s;
  }
  free(by_row);
  free(cnt_row);
  *out = g;
  return OR_OK;
}

void or_graph_free(or_graph* g) {
  if (!g) return;
  free(g->off); free(g->nbr); free(g->w); free(g->deg); free(g);
}
uint64_t or_graph_entries(const or_graph* g) { return g->n_entries; }
void or_graph_csr(const or_graph* g, uint64_t* off, uint32_t* nbr, double* w) {
  memcpy(off, g->off, ((size_t)g->nv + 1) * sizeof(uint64_t));
  memcpy(nbr, g->nbr, g->n_entries * sizeof(uint32_t));
  memcpy(w, g->w, g->n_entries * sizeof(double));
}
void or_graph_degree(const or_graph* g, double* deg) {
  memcpy(deg, g->deg, g->nv * sizeof(double));
}

/* ===================================================================== */
/* Zig-zag partition. Step 2: order nodes by (degree desc, id asc); the node
 * of rank r goes to part r mod n when floor(r/n) is even and to
 * n-1-(r mod n) when it is odd, with local index floor(r/n) ("sort
 * nodes by their degrees and then assign them into different partitions in
 * a zig-zag fashion"). new id = part_off[part] + local.       */
/* ===================================================================== */
static const double* g_sort_deg; /* qsort has no context argument */
static int cmp_rank(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  if (g_sort_deg[x] != g_sort_deg[y]) return g_sort_deg[x] > g_sort_deg[y] ? -1 : 1;
  return x < y ? -1 : (x > y ? 1 : 0);
}

int or_zigzag(uint32_t nv, const double* deg, uint32_t n, uint32_t* perm,
              uint32_t* inv_perm, uint64_t* part_off) {
  if (n == 0 || n > nv) return OR_ERR_INVALID_ARG;
  uint32_t* order = (uint32_t*)malloc((size_t)nv * sizeof(uint32_t));
  uint32_t* part = (uint32_t*)malloc((size_t)nv * sizeof(uint32_t));
  uint32_t* local = (uint32_t*)malloc((size_t)nv * sizeof(uint32_t));
  if (!order || !part || !local) { free(order); free(part); free(local); return OR_ERR_NOMEM; }
  for (uint32_t v = 0; v < nv; v++) order[v] = v;
  g_sort_deg = deg;
  qsort(order, nv, sizeof(uint32_t), cmp_rank);
  for (uint32_t p = 0; p <= n; p++) part_off[p] = 0;
  for (uint32_t r = 0; r < nv; r++) {
    uint32_t round = r / n, pos = r % n;
    uint32_t p = (round % 2 == 0) ? pos : n - 1 - pos;
    part[order[r]] = p;
    local[order[r]] = round;
    part_off[p + 1]++;
  }
  for (uint32_t p = 0; p < n; p++) part_off[p + 1] += part_off[p];
  for (uint32_t v = 0; v < nv; v++) {
    uint32_t nid = (uint32_t)(part_off[part[v]] + local[v]);
    perm[v] = nid;
    inv_perm[nid] = v;
  }
  free(order); free(part); free(local);
  return OR_OK;
}

/* ===================================================================== */
/* Integer alias table. Step 3 (reading R-ALIAS): a_i = trunc(w_i * m 2^32 /
 * W), the deficit m 2^32 - sum a_i added to the lowest-index argmax, FIFO
 * small/large worklists in ascending index order. Then every i has implied
 * mass exactly a_i / (m 2^32).                                             */
/* ===================================================================== */
int or_alias_build(const double* w, uint32_t m, uint32_t* prob, uint32_t* alias) {
  if (m == 0) return OR_ERR_EMPTY;
  double W = 0.0;
  for (uint32_t i = 0; i < m; i++) W += w[i];
  if (!(W > 0.0)) return OR_ERR_EMPTY;
  const uint64_t ONE = (uint64_t)1 << 32;
  double scale = (double)m * 4294967296.0 / W;
  uint64_t* a = (uint64_t*)malloc((size_t)m * sizeof(uint64_t));
  uint32_t* small = (uint32_t*)malloc((size_t)m * sizeof(uint32_t));
  uint32_t* large = (uint32_t*)malloc((size_t)m * sizeof(uint32_t));
  if (!a || !small || !large) { free(a); free(small); free(large); return OR_ERR_NOMEM; }
  uint64_t sum = 0;
  uint32_t argmax = 0;
  for (uint32_t i = 0; i < m; i++) {
    a[i] = (uint64_t)(w[i] * scale);
    sum += a[i];
    if (a[i] > a[argmax]) argmax = i;
  }
  a[argmax] += ((uint64_t)m << 32) - sum; /* modular: also handles a surplus */
  uint32_t sh = 0, st = 0, lh = 0, lt = 0; /* FIFO heads and tails */
  for (uint32_t i = 0; i < m; i++) {
    if (a[i] < ONE) small[st++] = i; else large[lt++] = i;
  }
  while (sh < st && lh < lt) {
    uint32_t s = small[sh++];
    uint32_t l = large[lh];
    prob[s] = (uint32_t)a[s];
    alias[s] = l;
    a[l] -= ONE - a[s];
    if (a[l] < ONE) { lh++; small[st++] = l; }
  }
  while (sh < st) { uint32_t s = small[sh++]; prob[s] = 0xFFFFFFFFu; alias[s] = s; }
  while (lh < lt) { uint32_t l = large[lh++]; prob[l] = 0xFFFFFFFFu; alias[l] = l; }
  free(a); free(small); free(large);
  return OR_OK;
}

/* Step 4: slot = floor(((r0 << 32) | r1) * m / 2^64); accept the slot when
 * r2 < prob[slot], else take its alias. */
uint32_t or_alias_draw(const uint32_t* prob, const uint32_t* alias, uint32_t m,
                       uint32_t r0, uint32_t r1, uint32_t r2) {
  uint64_t x = ((uint64_t)r0 << 32) | (uint64_t)r1;
  uint32_t slot = (uint32_t)(((unsigned __int128)x * (unsigned __int128)m) >> 64);
  return r2 < prob[slot] ? slot : alias[slot];
}

/* ===================================================================== */
/* Learning rate. Step 8.                                    */
/* ===================================================================== */
float or_lr(int kind, double lr0, double floor_ratio, uint64_t s_before, uint64_t s_total) {
  if (kind == 0 || s_total == 0) return (float)lr0;
  double r = 1.0 - (double)s_before / (double)s_total;
  if (r < floor_ratio) r = floor_ratio;
  return (float)(lr0 * r);
}

/* ===================================================================== */
/* One SGNS update, LINE convention (step 9; reading R-ORDER). The sample's
 * objective is  l = log s(U.C_v) + omega * sum_k log s(-U.C_{n_k})  (P:97,
 * P:392 "scale the gradient of the negative sample by 5"). For targets tau
 * in order: x = U.C_tau, p = s(x), g = (y - p) lr omega, err += g C_tau,
 * C_tau += g U; finally U += err. U is not changed while the sample runs.  */
/* ===================================================================== */
double or_sgd_sample(float* U, float* const* C, uint32_t n_targets, uint32_t d,
                     float lr, float neg_weight) {
  float err[1024];
  double loss = 0.0;
  for (uint32_t k = 0; k < d; k++) err[k] = 0.0f;
  for (uint32_t tau = 0; tau < n_targets; tau++) {
    float* Ct = C[tau];
    float y = (tau == 0) ? 1.0f : 0.0f;
    float omega = (tau == 0) ? 1.0f : neg_weight;
    float x = 0.0f;
    for (uint32_t k = 0; k < d; k++) x += U[k] * Ct[k];
    float p = 1.0f / (1.0f + expf(-x));
    float g = (y - p) * lr * omega;
    for (uint32_t k = 0; k < d; k++) err[k] += g * Ct[k];
    for (uint32_t k = 0; k < d; k++) Ct[k] += g * U[k];
    /* loss: -log s(x) for the positive, -log s(-x) for a negative */
    double z = (tau == 0) ? -(double)x : (double)x;
    loss += (z > 0 ? z : 0.0) + log1p(exp(-fabs(z)));
  }
  for (uint32_t k = 0; k < d; k++) U[k] += err[k];
  return loss;
}

/* ===================================================================== */
/* Bucketing. Step 6: stable counting sort by bin = part(u) n + part(v) of
 * the relabelled ids, emitting local ids; blocks row-major in (i, j).      */
/* ===================================================================== */
static uint32_t part_of(const uint64_t* part_off, uint32_t n, uint32_t nid) {
  uint32_t p = 0;
  while (p + 1 < n && part_off[p + 1] <= nid) p++;
  return p;
}

int or_bucket(const uint32_t* pairs, uint64_t count, uint32_t nv,
              const uint32_t* perm, const uint64_t* part_off, uint32_t n,
              uint32_t* out, uint64_t* block_off) {
  uint64_t nb = (uint64_t)n * n;
  for (uint64_t q = 0; q < count; q++)
    if (pairs[2 * q] >= nv || pairs[2 * q + 1] >= nv) return OR_ERR_OUT_OF_RANGE;
  uint32_t* bin = (uint32_t*)malloc((count ? count : 1) * sizeof(uint32_t));
  uint64_t* fill = (uint64_t*)calloc(nb, sizeof(uint64_t));
  if (!bin || !fill) { free(bin); free(fill); return OR_ERR_NOMEM; }
  for (uint64_t b = 0; b <= nb; b++) block_off[b] = 0;
  for (uint64_t q = 0; q < count; q++) {
    uint32_t pu = part_of(part_off, n, perm[pairs[2 * q]]);
    uint32_t pv = part_of(part_off, n, perm[pairs[2 * q + 1]]);
    bin[q] = pu * n + pv;
    block_off[bin[q] + 1]++;
  }
  for (uint64_t b = 0; b < nb; b++) block_off[b + 1] += block_off[b];
  for (uint64_t q = 0; q < count; q++) {
    uint32_t b = bin[q];
    uint32_t pu = b / n, pv = b % n;
    uint64_t pos = block_off[b] + fill[b]++;
    out[2 * pos] = perm[pairs[2 * q]] - (uint32_t)part_off[pu];
    out[2 * pos + 1] = perm[pairs[2 * q + 1]] - (uint32_t)part_off[pv];
  }
  free(bin); free(fill);
  return OR_OK;
}

/* Reading R-VTILE: within each block (i, j) of or_bucket's
 * output, a stable counting sort by the sample's vertex tile
 * floor(u_local / 2^tile_bits) — pool order inside a tile.               */
int or_bucket_tiled(const uint32_t* pairs, uint64_t count, uint32_t nv,
                    const uint32_t* perm, const uint64_t* part_off, uint32_t n,
                    uint32_t tile_bits, uint32_t* out, uint64_t* block_off) {
  if (tile_bits > 31) return OR_ERR_INVALID_ARG;
  if (tile_bits == 0) return or_bucket(pairs, count, nv, perm, part_off, n, out, block_off);
  uint32_t* lp = (uint32_t*)malloc((count ? count : 1) * 8);
  if (!lp) return OR_ERR_NOMEM;
  int rc = or_bucket(pairs, count, nv, perm, part_off, n, lp, block_off);
  if (rc) { free(lp); return rc; }
  for (uint64_t b = 0; b < (uint64_t)n * n; b++) {
    uint64_t beg = block_off[b], end = block_off[b + 1];
    uint32_t i = (uint32_t)(b / n);
    uint64_t rows = part_off[i + 1] - part_off[i];
    uint64_t tiles = (rows >> tile_bits) + 1;
    uint64_t* start = (uint64_t*)calloc(tiles + 1, sizeof(uint64_t));
    if (!start) { free(lp); return OR_ERR_NOMEM; }
    for (uint64_t q = beg; q < end; q++) start[(lp[2 * q] >> tile_bits) + 1]++;
    for (uint64_t t = 0; t < tiles; t++) start[t + 1] += start[t];
    for (uint64_t q = beg; q < end; q++) {
      uint64_t pos = beg + start[lp[2 * q] >> tile_bits]++;
      out[2 * pos] = lp[2 * q];
      out[2 * pos + 1] = lp[2 * q + 1];
    }
    free(start);
  }
  free(lp);
  return OR_OK;
}

/* Alg. 3: cid <- (i + offset) mod num_GPU. */
uint32_t or_schedule_cid(uint32_t n, uint32_t t, uint32_t i) { return (i + t) % n; }

/* ===================================================================== */
/* Initialisation. Step 5 (reading R-INIT): vertex[v][k] =
 * ((word_{k mod 4}(Philox({v, k/4, 0, 'INIT'}, seed)) >> 8) 2^-24 - 0.5)/d,
 * context = 0. Keyed by ORIGINAL id.                                      */
/* ===================================================================== */
void or_init_vertex(uint32_t nv, uint32_t d, uint64_t seed, float* vertex) {
  uint32_t key[2];
  seed_to_key(seed, key);
  for (uint32_t v = 0; v < nv; v++) {
    uint32_t r[4];
    for (uint32_t k = 0; k < d; k++) {
      if (k % 4 == 0) { /* one Philox block serves columns k .. k+3 */
        uint32_t ctr[4] = {v, k / 4, 0u, 0x494E4954u};
        or_philox4x32_10(ctr, key, r);
      }
      float u01 = (float)(r[k % 4] >> 8) * 0x1p-24f;
      vertex[(uint64_t)v * d + k] = (u01 - 0.5f) / (float)d;
    }
  }
}

/* ===================================================================== */
/* Trainer: steps 1-9 in one serial loop (Alg. 3 P:239-256 run with one
 * worker: for offset t, for i, train block (i, (i+t) mod n)).             */
/* ===================================================================== */
struct or_trainer {
  uint32_t nv, d, n, K;
  float lr0;
  int lr_kind;
  double floor_ratio;
  uint64_t total;
  uint32_t key[2];
  uint64_t seed_init;
  float neg_weight;
  or_graph* g;
  uint32_t* perm;
  uint32_t* inv_perm;
  uint64_t* part_off;
  uint32_t* nprob;  /* negative alias tables, partition p at part_off[p] */
  uint32_t* nalias;
  float* vertex;    /* ORIGINAL id order, nv x d */
  float* context;
  uint64_t samples_done;
  uint32_t pool_index;
  uint32_t vtile_bits;  /* R-VTILE: 0 = blocks in pool order (or_bucket) */
};

int or_trainer_set_vertex_tile(or_trainer* t, uint32_t tile_bits) {
  if (tile_bits > 31) return OR_ERR_INVALID_ARG;
  t->vtile_bits = tile_bits;
  return OR_OK;
}

int or_trainer_create(uint32_t nv, uint32_t d, uint32_t n, uint32_t K, float lr0,
                      int lr_kind, double floor_ratio, uint64_t total_samples,
                      uint64_t seed_neg, uint64_t seed_init, float neg_weight,
                      or_trainer** out) {
  *out = NULL;
  if (nv == 0 || d == 0 || d > 1024 || K == 0 || K > 8 || n == 0 || n > nv)
    return OR_ERR_INVALID_ARG;
  or_trainer* t = (or_trainer*)calloc(1, sizeof(or_trainer));
  t->nv = nv; t->d = d; t->n = n; t->K = K; t->lr0 = lr0;
  t->lr_kind = lr_kind; t->floor_ratio = floor_ratio; t->total = total_samples;
  seed_to_key(seed_neg, t->key);
  t->seed_init = seed_init;
  t->neg_weight = neg_weight;
  *out = t;
  return OR_OK;
}

int or_trainer_load_edges(or_trainer* t, const uint32_t* src, const uint32_t* dst,
                          const float* w, uint64_t ne) {
  int rc = or_graph_build(t->nv, src, dst, w, ne, &t->g);
  if (rc) return rc;
  uint32_t nv = t->nv, n = t->n;
  t->perm = (uint32_t*)malloc((size_t)nv * 4);
  t->inv_perm = (uint32_t*)malloc((size_t)nv * 4);
  t->part_off = (uint64_t*)malloc(((size_t)n + 1) * 8);
  t->nprob = (uint32_t*)malloc((size_t)nv * 4);
  t->nalias = (uint32_t*)malloc((size_t)nv * 4);
  t->vertex = (float*)malloc((size_t)nv * t->d * 4);
  t->context = (float*)calloc((size_t)nv * t->d, 4);
  if (!t->perm || !t->inv_perm || !t->part_off || !t->nprob || !t->nalias || !t->vertex ||
      !t->context)
    return OR_ERR_NOMEM;
  rc = or_zigzag(nv, t->g->deg, n, t->perm, t->inv_perm, t->part_off);
  if (rc) return rc;
  /* negatives: deg^0.75 over the members of each partition, local order
   * ("only ... from the context rows on the current GPU"). */
  double* wts = (double*)malloc((size_t)nv * sizeof(double));
  for (uint32_t p = 0; p < n; p++) {
    uint64_t b = t->part_off[p], e = t->part_off[p + 1];
    for (uint64_t q = b; q < e; q++) wts[q - b] = pow(t->g->deg[t->inv_perm[q]], 0.75);
    rc = or_alias_build(wts, (uint32_t)(e - b), t->nprob + b, t->nalias + b);
    if (rc) { free(wts); return rc; }
  }
  free(wts);
  or_init_vertex(nv, t->d, t->seed_init, t->vertex);
  return OR_OK;
}

static uint32_t negative_local(const or_trainer* t, uint32_t q, uint32_t i, uint32_t j,
                               uint32_t e, uint32_t k) {
  uint32_t ctr[4] = {q, (i << 16) | j, e, k}, r[4];
  or_philox4x32_10(ctr, t->key, r);
  uint64_t b = t->part_off[j];
  uint32_t m = (uint32_t)(t->part_off[j + 1] - b);
  return or_alias_draw(t->nprob + b, t->nalias + b, m, r[0], r[1], r[2]);
}

int or_trainer_negatives(const or_trainer* t, uint64_t count, uint32_t i, uint32_t j,
                         uint32_t e, uint32_t* out) {
  for (uint64_t q = 0; q < count; q++)
    for (uint32_t k = 0; k < t->K; k++)
      out[q * t->K + k] = negative_local(t, (uint32_t)q, i, j, e, k);
  return OR_OK;
}

uint32_t or_trainer_negative_at(const or_trainer* t, uint32_t q, uint32_t i, uint32_t j,
                                uint32_t e, uint32_t k) {
  return negative_local(t, q, i, j, e, k);
}

int or_trainer_train_block(or_trainer* t, const uint32_t* lp, uint64_t count, uint32_t i,
                           uint32_t j, uint32_t e, float lr, double* loss_out) {
  float* C[9];
  double loss = 0.0;
  uint32_t d = t->d;
  for (uint64_t q = 0; q < count; q++) {
    uint32_t u = t->inv_perm[t->part_off[i] + lp[2 * q]];
    uint32_t v = t->inv_perm[t->part_off[j] + lp[2 * q + 1]];
    C[0] = t->context + (uint64_t)v * d;
    for (uint32_t k = 0; k < t->K; k++) {
      uint32_t nl = negative_local(t, (uint32_t)q, i, j, e, k);
      C[1 + k] = t->context + (uint64_t)t->inv_perm[t->part_off[j] + nl] * d;
    }
    loss += or_sgd_sample(t->vertex + (uint64_t)u * d, C, 1 + t->K, d, lr, t->neg_weight);
  }
  if (loss_out) *loss_out += loss;
  return OR_OK;
}

int or_trainer_train_pool(or_trainer* t, const uint32_t* pairs, uint64_t count,
                          double* loss_out) {
  uint32_t n = t->n;
  uint64_t* block_off = (uint64_t*)malloc(((size_t)n * n + 1) * 8);
  uint32_t* lp = (uint32_t*)malloc((count ? count : 1) * 8);
  if (!block_off || !lp) { free(block_off); free(lp); return OR_ERR_NOMEM; }
  int rc = or_bucket_tiled(pairs, count, t->nv, t->perm, t->part_off, n, t->vtile_bits, lp, block_off);
  if (rc) { free(block_off); free(lp); return rc; }
  uint32_t e = t->pool_index;
  double loss = 0.0;
  for (uint32_t step = 0; step < n; step++) {
    float lr = or_lr(t->lr_kind, t->lr0, t->floor_ratio, t->samples_done, t->total);
    uint64_t step_samples = 0;
    for (uint32_t i = 0; i < n; i++) {
      uint32_t j = or_schedule_cid(n, step, i);
      uint64_t b = (uint64_t)i * n + j;
      uint64_t cnt = block_off[b + 1] - block_off[b];
      or_trainer_train_block(t, lp + 2 * block_off[b], cnt, i, j, e, lr, &loss);
      step_samples += cnt;
    }
    t->samples_done += step_samples;
  }
  t->pool_index++;
  if (loss_out) *loss_out = loss;
  free(block_off); free(lp);
  return OR_OK;
}

/* ---- CPU baseline class (bench.py's cpu_hogwild line only; NOT a parity
 * reference). The paper's CPU systems train with LINE-style asynchronous SGD
 * over all cores. This is or_trainer_train_pool with each block's
 * samples split over `threads` OpenMP threads that update the shared
 * matrices without locks (Hogwild): same bucketing, Philox negatives and lr
 * schedule; the result depends on the thread interleaving.                 */
int or_trainer_train_pool_hogwild(or_trainer* t, const uint32_t* pairs, uint64_t count,
                                  int threads, double* loss_out) {
  uint32_t n = t->n;
  uint64_t* block_off = (uint64_t*)malloc(((size_t)n * n + 1) * 8);
  uint32_t* lp = (uint32_t*)malloc((count ? count : 1) * 8);
  if (!block_off || !lp) { free(block_off); free(lp); return OR_ERR_NOMEM; }
  int rc = or_bucket_tiled(pairs, count, t->nv, t->perm, t->part_off, n, t->vtile_bits, lp, block_off);
  if (rc) { free(block_off); free(lp); return rc; }
  uint32_t e = t->pool_index, d = t->d;
  double loss = 0.0;
  for (uint32_t step = 0; step < n; step++) {
    float lr = or_lr(t->lr_kind, t->lr0, t->floor_ratio, t->samples_done, t->total);
    uint64_t step_samples = 0;
    for (uint32_t i = 0; i < n; i++) {
      uint32_t j = or_schedule_cid(n, step, i);
      uint64_t b = (uint64_t)i * n + j;
      uint64_t cnt = block_off[b + 1] - block_off[b];
      const uint32_t* blk = lp + 2 * block_off[b];
      double bl = 0.0;
#pragma omp parallel for num_threads(threads) schedule(static) reduction(+ : bl)
      for (int64_t q = 0; q < (int64_t)cnt; q++) {
        float* C[9];
        uint32_t u = t->inv_perm[t->part_off[i] + blk[2 * q]];
        uint32_t v = t->inv_perm[t->part_off[j] + blk[2 * q + 1]];
        C[0] = t->context + (uint64_t)v * d;
        for (uint32_t k = 0; k < t->K; k++) {
          uint32_t nl = negative_local(t, (uint32_t)q, i, j, e, k);
          C[1 + k] = t->context + (uint64_t)t->inv_perm[t->part_off[j] + nl] * d;
        }
        bl += or_sgd_sample(t->vertex + (uint64_t)u * d, C, 1 + t->K, d, lr, t->neg_weight);
      }
      loss += bl;
      step_samples += cnt;
    }
    t->samples_done += step_samples;
  }
  t->pool_index++;
  if (loss_out) *loss_out = loss;
  free(block_off); free(lp);
  return OR_OK;
}

int or_trainer_explicit(or_trainer* t, const uint32_t* u, const uint32_t* v,
                        const uint32_t* negs, uint64_t count, float lr) {
  float* C[9];
  uint32_t d = t->d;
  for (uint64_t q = 0; q < count; q++) {
    if (u[q] >= t->nv || v[q] >= t->nv) return OR_ERR_OUT_OF_RANGE;
    C[0] = t->context + (uint64_t)v[q] * d;
    for (uint32_t k = 0; k < t->K; k++) {
      uint32_t nk = negs[q * t->K + k];
      if (nk >= t->nv) return OR_ERR_OUT_OF_RANGE;
      C[1 + k] = t->context + (uint64_t)nk * d;
    }
    or_sgd_sample(t->vertex + (uint64_t)u[q] * d, C, 1 + t->K, d, lr, t->neg_weight);
  }
  return OR_OK;
}

void or_trainer_get(const or_trainer* t, int which, float* out) {
  memcpy(out, which ? t->context : t->vertex, (size_t)t->nv * t->d * 4);
}
void or_trainer_set(or_trainer* t, int which, const float* in) {
  memcpy(which ? t->context : t->vertex, in, (size_t)t->nv * t->d * 4);
}
void or_trainer_partition(const or_trainer* t, uint32_t* perm, uint64_t* part_off) {
  memcpy(perm, t->perm, (size_t)t->nv * 4);
  memcpy(part_off, t->part_off, ((size_t)t->n + 1) * 8);
}
int or_trainer_alias(const or_trainer* t, uint32_t p, uint32_t* prob, uint32_t* alias) {
  if (p >= t->n) return OR_ERR_INVALID_ARG;
  uint64_t b = t->part_off[p], e = t->part_off[p + 1];
  memcpy(prob, t->nprob + b, (e - b) * 4);
  memcpy(alias, t->nalias + b, (e - b) * 4);
  return OR_OK;
}
uint64_t or_trainer_samples_done(const or_trainer* t) { return t->samples_done; }
const or_graph* or_trainer_graph(const or_trainer* t) { return t->g; }
void or_trainer_free(or_trainer* t) {
  if (!t) return;
  or_graph_free(t->g);
  free(t->perm); free(t->inv_perm); free(t->part_off); free(t->nprob); free(t->nalias);
  free(t->vertex); free(t->context); free(t);
}

/* ===================================================================== */
/* Online augmentation (Alg. 2; "draw a departure node with
 * the probability proportional to the degree ... perform a random walk ...
 * pick node pairs within a specific augmentation distance s"; pseudo
 * shuffle P:198-199). Reading R-AUG fixes the random stream.              */
/* ===================================================================== */
struct or_sampler {
  const or_graph* g;
  uint32_t* dprob; uint32_t* dalias; /* departure, over nodes, weight deg */
  uint32_t* eprob; uint32_t* ealias; /* per-node neighbour tables, over CSR entries */
};

int or_sampler_create(const or_graph* g, or_sampler** out) {
  or_sampler* s = (or_sampler*)calloc(1, sizeof(or_sampler));
  s->g = g;
  s->dprob = (uint32_t*)malloc((size_t)g->nv * 4);
  s->dalias = (uint32_t*)malloc((size_t)g->nv * 4);
  s->eprob = (uint32_t*)malloc(g->n_entries * 4 + 4);
  s->ealias = (uint32_t*)malloc(g->n_entries * 4 + 4);
  int rc = or_alias_build(g->deg, g->nv, s->dprob, s->dalias);
  if (rc) { or_sampler_free(s); return rc; }
  for (uint32_t v = 0; v < g->nv; v++) {
    uint64_t b = g->off[v], e = g->off[v + 1];
    if (e == b || !(g->deg[v] > 0.0)) continue; /* never reached */
    rc = or_alias_build(g->w + b, (uint32_t)(e - b), s->eprob + b, s->ealias + b);
    if (rc) { or_sampler_free(s); return rc; }
  }
  *out = s;
  return OR_OK;
}

void or_sampler_free(or_sampler* s) {
  if (!s) return;
  free(s->dprob); free(s->dalias); free(s->eprob); free(s->ealias); free(s);
}

/* Walk `walk` of sampler thread `thread`: x_0 from the departure table with
 * Philox counter {walk, 0, thread, 'WALK'}, x_k a neighbour of x_{k-1}
 * drawn with counter {walk, k, thread, 'WALK'}, key = seed. */
int or_sampler_walk(const or_sampler* s, uint32_t thread, uint32_t walk,
                    uint32_t walk_len, uint64_t seed, uint32_t* nodes) {
  uint32_t key[2], r[4];
  seed_to_key(seed, key);
  const or_graph* g = s->g;
  uint32_t ctr[4] = {walk, 0u, thread, 0x57414C4Bu};
  or_philox4x32_10(ctr, key, r);
  nodes[0] = or_alias_draw(s->dprob, s->dalias, g->nv, r[0], r[1], r[2]);
  for (uint32_t k = 1; k <= walk_len; k++) {
    uint32_t x = nodes[k - 1];
    uint64_t b = g->off[x];
    uint32_t m = (uint32_t)(g->off[x + 1] - b);
    uint32_t c2[4] = {walk, k, thread, 0x57414C4Bu};
    or_philox4x32_10(c2, key, r);
    uint32_t slot = or_alias_draw(s->eprob + b, s->ealias + b, m, r[0], r[1], r[2]);
    nodes[k] = g->nbr[b + slot];
  }
  return OR_OK;
}

/* Pairs (walk[a], walk[b]), 0 < b - a <= s, walk[a] != walk[b], by
 * increasing a then b (reading R-PAIRS). len = walk_len + 1. */
uint64_t or_pairs_within(const uint32_t* walk, uint32_t len, uint32_t s, uint32_t* out) {
  uint64_t c = 0;
  for (uint32_t a = 0; a < len; a++)
    for (uint32_t b = a + 1; b < len && b <= a + s; b++)
      if (walk[a] != walk[b]) {
        out[2 * c] = walk[a];
        out[2 * c + 1] = walk[b];
        c++;
      }
  return c;
}

/* Pseudo shuffle ("divide the sample pool into s continuous
 * blocks, and scatter correlated samples into different blocks"): sample k
 * is appended to block k mod s; blocks are concatenated. */
void or_pseudo_shuffle(const uint32_t* in, uint64_t count, uint32_t s, uint32_t* out) {
  uint64_t pos = 0;
  for (uint32_t blk = 0; blk < s; blk++)
    for (uint64_t k = blk; k < count; k += s) {
      out[2 * pos] = in[2 * k];
      out[2 * pos + 1] = in[2 * k + 1];
      pos++;
    }
}

int or_augment(const or_sampler* s, uint32_t walk_len, uint32_t dist, uint32_t threads,
               uint64_t count, uint64_t seed, uint32_t* out) {
  if (walk_len == 0 || dist == 0 || dist > walk_len || threads == 0) return OR_ERR_INVALID_ARG;
  uint32_t* walk = (uint32_t*)malloc(((size_t)walk_len + 1) * 4);
  uint32_t* pr = (uint32_t*)malloc(((size_t)walk_len + 1) * dist * 8);
  for (uint32_t th = 0; th < threads; th++) {
    uint64_t b = (uint64_t)(((unsigned __int128)count * th) / threads);
    uint64_t e = (uint64_t)(((unsigned __int128)count * (th + 1)) / threads);
    uint64_t cap = e - b, filled = 0;
    uint32_t* seg = (uint32_t*)malloc((cap ? cap : 1) * 8);
    for (uint32_t w = 0; filled < cap; w++) {
      or_sampler_walk(s, th, w, walk_len, seed, walk);
      uint64_t np = or_pairs_within(walk, walk_len + 1, dist, pr);
      for (uint64_t q = 0; q < np && filled < cap; q++, filled++) {
        seg[2 * filled] = pr[2 * q];
        seg[2 * filled + 1] = pr[2 * q + 1];
      }
    }
    or_pseudo_shuffle(seg, cap, dist, out + 2 * b);
    free(seg);
  }
  free(walk); free(pr);
  return OR_OK;
}

/* ===================================================================== */
/* Evaluation: link-prediction AUC by cosine similarity.           */
/* ===================================================================== */
double or_cosine(const float* a, const float* b, uint32_t d) {
  double ab = 0, aa = 0, bb = 0;
  for (uint32_t k = 0; k < d; k++) {
    ab += (double)a[k] * b[k]; aa += (double)a[k] * a[k]; bb += (double)b[k] * b[k];
  }
  if (aa == 0.0 || bb == 0.0) return 0.0;
  return ab / (sqrt(aa) * sqrt(bb));
}

typedef struct { double s; int pos; } scored_t;
static int cmp_scored(const void* a, const void* b) {
  double x = ((const scored_t*)a)->s, y = ((const scored_t*)b)->s;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* Mann-Whitney: AUC = (sum of positive midranks - npos(npos+1)/2) / (npos nneg). */
double or_auc(const double* pos, uint64_t npos, const double* neg, uint64_t nneg) {
  uint64_t n = npos + nneg;
  if (npos == 0 || nneg == 0) return NAN;
  scored_t* a = (scored_t*)malloc(n * sizeof(scored_t));
  for (uint64_t q = 0; q < npos; q++) { a[q].s = pos[q]; a[q].pos = 1; }
  for (uint64_t q = 0; q < nneg; q++) { a[npos + q].s = neg[q]; a[npos + q].pos = 0; }
  qsort(a, n, sizeof(scored_t), cmp_scored);
  double rank_sum = 0.0;
  for (uint64_t i = 0; i < n;) {
    uint64_t j = i;
    while (j < n && a[j].s == a[i].s) j++;
    double mid = 0.5 * ((double)(i + 1) + (double)j); /* ranks i+1..j */
    for (uint64_t q = i; q < j; q++)
      if (a[q].pos) rank_sum += mid;
    i = j;
  }
  free(a);
  return (rank_sum - 0.5 * (double)npos * (double)(npos + 1)) / ((double)npos * (double)nneg);
}

double or_linkpred_auc(const float* emb, uint32_t d, const uint32_t* pp, uint64_t npos,
                       const uint32_t* np_, uint64_t nneg) {
  double* ps = (double*)malloc((npos ? npos : 1) * sizeof(double));
  double* ns = (double*)malloc((nneg ? nneg : 1) * sizeof(double));
  for (uint64_t q = 0; q < npos; q++)
    ps[q] = or_cosine(emb + (uint64_t)pp[2 * q] * d, emb + (uint64_t)pp[2 * q + 1] * d, d);
  for (uint64_t q = 0; q < nneg; q++)
    ns[q] = or_cosine(emb + (uint64_t)np_[2 * q] * d, emb + (uint64_t)np_[2 * q + 1] * d, d);
  double r = or_auc(ps, npos, ns, nneg);
  free(ps); free(ns);
  return r;
}
