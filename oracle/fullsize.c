/*
 * fullsize.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * The oracle at BASELINE.json's full sizes (C3 R-MAT-24, C4 WS(5e7),
 * C5 PA(1e8) ~ 2e9 edges): the same restatement as oracle.c, arranged so
 * that it fits a 62 GB host and finishes in minutes on its cores.
 *
 *  - the configs' seeded generators (the workload definitions): gen_pa
 *    restated from io.hpp:129-162 (identical mt19937_64 stream; the endpoint
 *    list is implicit), and the harness generators the reference lacks
 *    (G(n, m), R-MAT, Watts-Strogatz), bit-identical to the product's host
 *    harness (tests/test_oracle_full.py checks both);
 *  - build_graph (graph.hpp:58-85) as bucket-by-source + per-row sort +
 *    unique, in place (the pairs are consumed);
 *  - effective_adjacency (effective.hpp:37-52) over the ByDegree rank
 *    (order.hpp:95-104, orc_degree_rank), rows filled in parallel;
 *  - count_node_iterator_n (sequential.hpp:74-91) with the scalar merge of
 *    intersect.hpp:15-33 on every host thread (apex ranges claimed
 *    dynamically), recording per triangle (v, u, w), v the apex:
 *      * NodeTallySink T_v (sequential.hpp:24-33, per-thread arrays summed);
 *      * the AOP per-rank count = triangles whose apex v is in core i
 *        (engines.hpp:38-54 over partition.hpp:171-206);
 *      * the ANOP-surrogate per-rank count = triangles whose middle vertex u
 *        is in core i (engines.hpp:60-76, 146-198);
 *      * an order-independent digest of the ListSink triples
 *        (sequential.hpp:36-46: each triple sorted ascending), see
 *        orc_tri_hash below;
 *  - the surrogate engine's data_sent / data_recv (engines.hpp:173-187:
 *    one NeighborList per distinct remote owner of N_v, LastProc).
 *
 * The per-rank semantics above are the closed forms SURVEY App. A.5 verified
 * against run_engine; tests/test_oracle_full.py checks every function here
 * against oracle.c and oracle/_ref (the unmodified reference) on graphs
 * small enough for both.
 */
#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

/* ------------------------------------------------------------ threads */

typedef struct {
  void (*fn)(void* ctx, uint64_t chunk, int tid);
  void* ctx;
  uint64_t chunks;
  atomic_uint_fast64_t next;
} pool_t;

typedef struct {
  pool_t* pool;
  int tid;
} worker_t;

static void* pool_worker(void* arg) {
  worker_t* w = (worker_t*)arg;
  pool_t* p = w->pool;
  for (;;) {
    uint64_t c = atomic_fetch_add(&p->next, 1);
    if (c >= p->chunks) break;
    p->fn(p->ctx, c, w->tid);
  }
  return NULL;
}

/* Run fn(ctx, c, tid) for c in [0, chunks) on `threads` threads (tid in
 * [0, threads)), chunks claimed dynamically. */
static void parallel_for(int threads, uint64_t chunks, void (*fn)(void*, uint64_t, int),
                         void* ctx) {
  if (threads < 1) threads = 1;
  if ((uint64_t)threads > chunks) threads = chunks ? (int)chunks : 1;
  pool_t p;
  p.fn = fn;
  p.ctx = ctx;
  p.chunks = chunks;
  atomic_init(&p.next, 0);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  worker_t* ws = (worker_t*)malloc(sizeof(worker_t) * threads);
  for (int t = 0; t < threads; ++t) {
    ws[t].pool = &p;
    ws[t].tid = t;
  }
  for (int t = 1; t < threads; ++t) pthread_create(&th[t], NULL, pool_worker, &ws[t]);
  pool_worker(&ws[0]);
  for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
  free(ws);
  free(th);
}

/* ------------------------------------------------------------ generators */

static uint64_t splitmix64_next(uint64_t* x) {
  uint64_t z = (*x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

typedef struct {
  uint64_t s[4];
} xoshiro_t;

static void xo_seed(xoshiro_t* r, uint64_t seed) {
  uint64_t x = seed;
  for (int i = 0; i < 4; ++i) r->s[i] = splitmix64_next(&x);
}

static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* xoshiro256** */
static uint64_t xo_next(xoshiro_t* r) {
  uint64_t* s = r->s;
  const uint64_t res = rotl64(s[1] * 5, 7) * 9, t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return res;
}

static double xo_unit(xoshiro_t* r) { return (double)(xo_next(r) >> 11) * 0x1.0p-53; }

/* io.hpp:129-162 gen_pa(n, d, seed): clique on d/2+1 nodes (:139-145), then
 * each node v picks d/2 distinct targets t = endpoints[rng() % size]
 * (:147-154) and appends (v, t) (:155-159).  endpoints[] is never stored:
 * slot 2e / 2e+1 of the e-th non-clique edge are its new vertex (clique +
 * e / half) and its target, so only the targets are kept. */
uint64_t orc_gen_pa(uint64_t n, uint64_t d, uint64_t seed, uint32_t** pairs_out) {
  if (d < 2 || d % 2 != 0 || n <= d / 2) return UINT64_MAX;
  const uint64_t half = d / 2, clique = half + 1;
  const uint64_t cpairs = clique * (clique - 1) / 2;
  const uint64_t E = cpairs + (n - clique) * half;
  uint32_t* out = (uint32_t*)malloc((E ? E : 1) * 2 * sizeof(uint32_t));
  uint32_t* cl = (uint32_t*)malloc((2 * cpairs + 1) * sizeof(uint32_t));
  uint32_t* tgt = (uint32_t*)malloc(((n - clique) * half + 1) * sizeof(uint32_t));
  uint32_t* pk = (uint32_t*)malloc(half * sizeof(uint32_t));
  uint64_t w = 0, c0 = 0;
  for (uint32_t u = 0; u < clique; ++u)
    for (uint32_t v = u + 1; v < clique; ++v) {
      out[2 * w] = u;
      out[2 * w + 1] = v;
      ++w;
      cl[c0++] = u;
      cl[c0++] = v;
    }
  orc_mt64 rng;
  orc_mt64_seed(&rng, seed);
  uint64_t ne = 0;
  for (uint64_t v = clique; v < n; ++v) {
    const uint64_t size = c0 + 2 * ne;
    uint64_t c = 0;
    while (c < half) {
      const uint64_t r = orc_mt64_next(&rng) % size;
      uint32_t t;
      if (r < c0) t = cl[r];
      else if (((r - c0) & 1) == 0) t = (uint32_t)(clique + ((r - c0) >> 1) / half);
      else t = tgt[(r - c0) >> 1];
      int dup = 0;
      for (uint64_t i = 0; i < c; ++i)
        if (pk[i] == t) { dup = 1; break; }
      if (!dup) pk[c++] = t;
    }
    for (uint64_t i = 0; i < half; ++i) {
      out[2 * w] = (uint32_t)v;
      out[2 * w + 1] = pk[i];
      ++w;
      tgt[ne++] = pk[i];
    }
  }
  free(pk);
  free(tgt);
  free(cl);
  *pairs_out = out;
  return E;
}

/* G(n, m) (config 1): xoshiro256**(seed) draws u = next % n, v = next % n;
 * loops and repeats of an unordered pair are rejected; stored (min, max). */
uint64_t orc_gen_gnm(uint64_t n, uint64_t m, uint64_t seed, uint32_t** pairs_out) {
  if ((n < 2 && m > 0) || (n >= 2 && m > n * (n - 1) / 2)) return UINT64_MAX;
  uint32_t* out = (uint32_t*)malloc((m ? m : 1) * 2 * sizeof(uint32_t));
  uint64_t cap = 16;
  int lg = 4;
  while (cap < 4 * m) cap <<= 1, ++lg;
  uint64_t* set = (uint64_t*)malloc(cap * sizeof(uint64_t));
  memset(set, 0xff, cap * sizeof(uint64_t));
  xoshiro_t r;
  xo_seed(&r, seed);
  uint64_t w = 0;
  while (w < m) {
    uint64_t u = xo_next(&r) % n, v = xo_next(&r) % n;
    if (u == v) continue;
    if (u > v) { uint64_t x = u; u = v; v = x; }
    const uint64_t key = (u << 32) | v;
    uint64_t h = (key * 0x9E3779B97F4A7C15ull) >> (64 - lg);
    int seen = 0;
    while (set[h] != UINT64_MAX) {
      if (set[h] == key) { seen = 1; break; }
      h = (h + 1) & (cap - 1);
    }
    if (seen) continue;
    set[h] = key;
    out[2 * w] = (uint32_t)u;
    out[2 * w + 1] = (uint32_t)v;
    ++w;
  }
  free(set);
  *pairs_out = out;
  return m;
}

typedef struct {
  uint32_t scale;
  double a, ab, abc;
  uint64_t seed, E;
  uint32_t* out;
} rmat_ctx;

static void rmat_chunk(void* cv, uint64_t ci, int tid) {
  (void)tid;
  rmat_ctx* c = (rmat_ctx*)cv;
  xoshiro_t r;
  xo_seed(&r, c->seed * 0x9E3779B97F4A7C15ull + ci + 1);
  const uint64_t e0 = ci << 20, e1 = e0 + (1ull << 20) < c->E ? e0 + (1ull << 20) : c->E;
  for (uint64_t e = e0; e < e1; ++e) {
    uint32_t u = 0, v = 0;
    for (uint32_t l = 0; l < c->scale; ++l) {
      const double x = xo_unit(&r);
      uint32_t bu = 0, bv = 0;
      if (x < c->a) {
      } else if (x < c->ab) bv = 1;
      else if (x < c->abc) bu = 1;
      else bu = bv = 1;
      u = (u << 1) | bu;
      v = (v << 1) | bv;
    }
    c->out[2 * e] = u;
    c->out[2 * e + 1] = v;
  }
}

/* R-MAT (config 3): edge_factor << scale draws; draw e lives in chunk
 * e >> 20 whose stream is xoshiro256**(seed * 0x9E3779B97F4A7C15 + chunk + 1);
 * per level one unit double picks the quadrant (a | b | c | d). */
uint64_t orc_gen_rmat(uint32_t scale, uint64_t edge_factor, double a, double b, double c,
                      uint64_t seed, int threads, uint32_t** pairs_out) {
  if (scale == 0 || scale > 31 || a < 0 || b < 0 || c < 0 || a + b + c > 1.0) return UINT64_MAX;
  rmat_ctx x = {scale, a, a + b, a + b + c, seed, edge_factor << scale, NULL};
  x.out = (uint32_t*)malloc((x.E ? x.E : 1) * 2 * sizeof(uint32_t));
  parallel_for(threads, (x.E + (1ull << 20) - 1) >> 20, rmat_chunk, &x);
  *pairs_out = x.out;
  return x.E;
}

typedef struct {
  uint64_t n, half, seed;
  double beta;
  uint32_t* out;
} ws_ctx;

static void ws_chunk(void* cv, uint64_t ci, int tid) {
  (void)tid;
  ws_ctx* c = (ws_ctx*)cv;
  xoshiro_t r;
  xo_seed(&r, c->seed * 0xD1B54A32D192ED03ull + ci + 1);
  const uint64_t v0 = ci << 16, v1 = v0 + (1ull << 16) < c->n ? v0 + (1ull << 16) : c->n;
  for (uint64_t v = v0; v < v1; ++v)
    for (uint64_t j = 1; j <= c->half; ++j) {
      uint64_t t = (v + j) % c->n;
      if (xo_unit(&r) < c->beta) {
        uint64_t w;
        do w = xo_next(&r) % c->n; while (w == v);
        t = w;
      }
      const uint64_t e = v * c->half + (j - 1);
      c->out[2 * e] = (uint32_t)v;
      c->out[2 * e + 1] = (uint32_t)t;
    }
}

/* Watts-Strogatz (config 4): ring lattice, v joined to v+1..v+k/2 (mod n);
 * each edge's far end is rewired with probability beta to a uniform w != v.
 * Vertices in chunks of 2^16, chunk stream xoshiro256**(seed *
 * 0xD1B54A32D192ED03 + chunk + 1). */
uint64_t orc_gen_ws(uint64_t n, uint64_t k, double beta, uint64_t seed, int threads,
                    uint32_t** pairs_out) {
  if (k % 2 != 0 || k == 0 || k >= n || beta < 0 || beta > 1 || n > 0xFFFFFFFFull)
    return UINT64_MAX;
  ws_ctx x = {n, k / 2, seed, beta, NULL};
  const uint64_t E = n * x.half;
  x.out = (uint32_t*)malloc((E ? E : 1) * 2 * sizeof(uint32_t));
  parallel_for(threads, (n + (1ull << 16) - 1) >> 16, ws_chunk, &x);
  *pairs_out = x.out;
  return E;
}

/* ------------------------------------------------------------ build_graph */

typedef struct {
  const uint32_t* pairs;
  uint64_t E;
  uint64_t* pos; /* atomic fill cursors (n) */
  uint32_t* tmp;
  const uint64_t* cnt;
  uint64_t n;
  uint64_t* newlen;
  uint64_t* maxv; /* per-chunk max id */
} build_ctx;

#define BCHUNK (1ull << 22)

static void b_max(void* cv, uint64_t ci, int tid) {
  (void)tid;
  build_ctx* c = (build_ctx*)cv;
  const uint64_t e0 = ci * BCHUNK, e1 = e0 + BCHUNK < c->E ? e0 + BCHUNK : c->E;
  uint64_t m = 0;
  for (uint64_t e = e0; e < e1; ++e) {
    if (c->pairs[2 * e] + 1ull > m) m = c->pairs[2 * e] + 1ull;
    if (c->pairs[2 * e + 1] + 1ull > m) m = c->pairs[2 * e + 1] + 1ull;
  }
  c->maxv[ci] = m;
}

static void b_count(void* cv, uint64_t ci, int tid) {
  (void)tid;
  build_ctx* c = (build_ctx*)cv;
  const uint64_t e0 = ci * BCHUNK, e1 = e0 + BCHUNK < c->E ? e0 + BCHUNK : c->E;
  for (uint64_t e = e0; e < e1; ++e) {
    const uint32_t u = c->pairs[2 * e], v = c->pairs[2 * e + 1];
    if (u == v) continue;
    __atomic_fetch_add(&c->pos[u], 1, __ATOMIC_RELAXED);
    __atomic_fetch_add(&c->pos[v], 1, __ATOMIC_RELAXED);
  }
}

static void b_fill(void* cv, uint64_t ci, int tid) {
  (void)tid;
  build_ctx* c = (build_ctx*)cv;
  const uint64_t e0 = ci * BCHUNK, e1 = e0 + BCHUNK < c->E ? e0 + BCHUNK : c->E;
  for (uint64_t e = e0; e < e1; ++e) {
    const uint32_t u = c->pairs[2 * e], v = c->pairs[2 * e + 1];
    if (u == v) continue;
    c->tmp[__atomic_fetch_add(&c->pos[u], 1, __ATOMIC_RELAXED)] = v;
    c->tmp[__atomic_fetch_add(&c->pos[v], 1, __ATOMIC_RELAXED)] = u;
  }
}

static int cmp_u32f(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

static void sort_u32(uint32_t* a, uint64_t n) {
  if (n <= 24) {
    for (uint64_t i = 1; i < n; ++i) {
      uint32_t x = a[i];
      uint64_t j = i;
      while (j > 0 && a[j - 1] > x) { a[j] = a[j - 1]; --j; }
      a[j] = x;
    }
  } else {
    qsort(a, n, sizeof(uint32_t), cmp_u32f);
  }
}

#define VCHUNK (1ull << 16)

/* sort + unique each row in place (graph.hpp:73-74 per source bucket) */
static void b_rows(void* cv, uint64_t ci, int tid) {
  (void)tid;
  build_ctx* c = (build_ctx*)cv;
  const uint64_t v0 = ci * VCHUNK, v1 = v0 + VCHUNK < c->n ? v0 + VCHUNK : c->n;
  for (uint64_t v = v0; v < v1; ++v) {
    uint32_t* r = c->tmp + c->cnt[v];
    const uint64_t len = c->cnt[v + 1] - c->cnt[v];
    sort_u32(r, len);
    uint64_t w = 0;
    for (uint64_t k = 0; k < len; ++k)
      if (k == 0 || r[k] != r[w - 1]) r[w++] = r[k];
    c->newlen[v] = w;
  }
}

/* graph.hpp:58-85 build_graph(pairs, n_override).  Takes ownership of
 * `pairs` (malloc'ed, freed once the adjacency is filled).  n = max(
 * n_override, 1 + max id over all pairs, loops included) (:60-64); loops
 * dropped and both directions kept (:66-72); sort + unique (:73-74) per
 * source row, which gives the identical CSR (:76-84). */
uint64_t orc_build_graph_lean(uint32_t* pairs, uint64_t E, uint64_t n_override, int threads,
                              uint64_t** off_out, uint32_t** adj_out) {
  build_ctx c;
  memset(&c, 0, sizeof c);
  c.pairs = pairs;
  c.E = E;
  const uint64_t echunks = (E + BCHUNK - 1) / BCHUNK;
  c.maxv = (uint64_t*)calloc(echunks + 1, sizeof(uint64_t));
  parallel_for(threads, echunks, b_max, &c);
  uint64_t n = n_override;
  for (uint64_t i = 0; i < echunks; ++i)
    if (c.maxv[i] > n) n = c.maxv[i];
  free(c.maxv);
  c.n = n;
  c.pos = (uint64_t*)calloc(n + 1, sizeof(uint64_t));
  parallel_for(threads, echunks, b_count, &c);
  uint64_t* cnt = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
  uint64_t acc = 0;
  for (uint64_t v = 0; v < n; ++v) {
    cnt[v] = acc;
    acc += c.pos[v];
    c.pos[v] = cnt[v];
  }
  cnt[n] = acc;
  c.cnt = cnt;
  c.tmp = (uint32_t*)malloc((acc ? acc : 1) * sizeof(uint32_t));
  parallel_for(threads, echunks, b_fill, &c);
  free(pairs);
  free(c.pos);
  c.newlen = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
  parallel_for(threads, (n + VCHUNK - 1) / VCHUNK, b_rows, &c);
  /* compact in place, rows in ascending order (each row moves left) */
  uint64_t* off = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
  uint64_t w = 0;
  for (uint64_t v = 0; v < n; ++v) {
    off[v] = w;
    if (w != cnt[v]) memmove(c.tmp + w, c.tmp + cnt[v], c.newlen[v] * sizeof(uint32_t));
    w += c.newlen[v];
  }
  off[n] = w;
  free(c.newlen);
  free(cnt);
  uint32_t* adj = (uint32_t*)realloc(c.tmp, (w ? w : 1) * sizeof(uint32_t));
  *off_out = off;
  *adj_out = adj ? adj : c.tmp;
  return n;
}

/* ------------------------------------------------------------ effective */

typedef struct {
  uint64_t n;
  const uint64_t* off;
  const uint32_t* adj;
  const uint32_t* rank;
  uint64_t* eoff;
  uint32_t* eff;
} eff_ctx;

static void e_count(void* cv, uint64_t ci, int tid) {
  (void)tid;
  eff_ctx* c = (eff_ctx*)cv;
  const uint64_t v0 = ci * VCHUNK, v1 = v0 + VCHUNK < c->n ? v0 + VCHUNK : c->n;
  for (uint64_t v = v0; v < v1; ++v) {
    uint64_t h = 0;
    for (uint64_t k = c->off[v]; k < c->off[v + 1]; ++k) h += c->rank[v] < c->rank[c->adj[k]];
    c->eoff[v + 1] = h;
  }
}

static void e_fill(void* cv, uint64_t ci, int tid) {
  (void)tid;
  eff_ctx* c = (eff_ctx*)cv;
  const uint64_t v0 = ci * VCHUNK, v1 = v0 + VCHUNK < c->n ? v0 + VCHUNK : c->n;
  for (uint64_t v = v0; v < v1; ++v) {
    uint64_t w = c->eoff[v];
    for (uint64_t k = c->off[v]; k < c->off[v + 1]; ++k)
      if (c->rank[v] < c->rank[c->adj[k]]) c->eff[w++] = c->adj[k];
  }
}

/* effective.hpp:37-52 under the rank array (ByDegree: orc_degree_rank,
 * order.hpp:95-104): N_v = {u in adj(v) : rank[v] < rank[u]}, ID-sorted. */
uint64_t orc_effective_mt(uint64_t n, const uint64_t* off, const uint32_t* adj,
                          const uint32_t* rank, int threads, uint64_t* eoff, uint32_t** eff_out) {
  eff_ctx c = {n, off, adj, rank, eoff, NULL};
  eoff[0] = 0;
  parallel_for(threads, (n + VCHUNK - 1) / VCHUNK, e_count, &c);
  for (uint64_t v = 0; v < n; ++v) eoff[v + 1] += eoff[v];
  c.eff = (uint32_t*)malloc((eoff[n] ? eoff[n] : 1) * sizeof(uint32_t));
  parallel_for(threads, (n + VCHUNK - 1) / VCHUNK, e_fill, &c);
  *eff_out = c.eff;
  return eoff[n];
}

/* ------------------------------------------------------------ counting */

/* Digest of one ListSink triple a < b < c (sequential.hpp:39-44
 * normalisation): h = mix(mix(mix(a) ^ b) ^ c), mix = the SplitMix64
 * finaliser of sparsify.hpp:37-45.  The listing digest is the pair
 * (sum h, sum mix(h)) mod 2^64 -- independent of emission order. */
static inline uint64_t fmix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return x;
}

uint64_t orc_tri_hash(uint32_t a, uint32_t b, uint32_t c) {
  return fmix(fmix(fmix((uint64_t)a) ^ (uint64_t)b) ^ (uint64_t)c);
}

#define MAXSLOTS 256

typedef struct {
  uint64_t n;
  const uint64_t* eoff;
  const uint32_t* eff;
  const uint32_t* b;
  uint64_t p;
  uint64_t vchunk;
  int want_tally, want_digest;
  uint64_t* tally[MAXSLOTS];
  uint64_t* apex[MAXSLOTS];
  uint64_t* mid[MAXSLOTS];
  uint64_t total[MAXSLOTS];
  uint64_t d0[MAXSLOTS], d1[MAXSLOTS];
} cnt_ctx;

static void c_chunk(void* cv, uint64_t ci, int tid) {
  (void)tid;
  cnt_ctx* c = (cnt_ctx*)cv;
  const int s = tid;
  uint64_t* tally = c->tally[s];
  uint64_t* apex = c->apex[s];
  uint64_t* mid = c->mid[s];
  uint64_t total = 0, d0 = 0, d1 = 0;
  const uint64_t v0 = ci * c->vchunk, v1 = v0 + c->vchunk < c->n ? v0 + c->vchunk : c->n;
  for (uint64_t v = v0; v < v1; ++v) {
    const uint32_t* nv = c->eff + c->eoff[v];
    const uint64_t hv = c->eoff[v + 1] - c->eoff[v];
    uint64_t tv = 0;
    for (uint64_t k = 0; k < hv; ++k) {
      const uint32_t u = nv[k];
      const uint32_t* nu = c->eff + c->eoff[u];
      const uint64_t hu = c->eoff[u + 1] - c->eoff[u];
      uint64_t i = 0, j = 0, tu = 0; /* intersect.hpp:15-33 */
      while (i < hv && j < hu) {
        if (nv[i] < nu[j]) ++i;
        else if (nu[j] < nv[i]) ++j;
        else {
          const uint32_t w = nv[i];
          ++tu;
          if (tally) tally[w]++;
          if (c->want_digest) {
            uint32_t t0 = (uint32_t)v, t1 = u, t2 = w, x;
            if (t0 > t1) { x = t0; t0 = t1; t1 = x; }
            if (t1 > t2) { x = t1; t1 = t2; t2 = x; }
            if (t0 > t1) { x = t0; t0 = t1; t1 = x; }
            const uint64_t h = orc_tri_hash(t0, t1, t2);
            d0 += h;
            d1 += fmix(h);
          }
          ++i;
          ++j;
        }
      }
      if (tu) {
        tv += tu;
        if (tally) tally[u] += tu;
        if (mid) mid[orc_owner(c->b, c->p, u)] += tu;
      }
    }
    if (tv) {
      total += tv;
      if (tally) tally[v] += tv;
      if (apex) apex[orc_owner(c->b, c->p, (uint32_t)v)] += tv;
    }
  }
  c->total[s] += total;
  c->d0[s] += d0;
  c->d1[s] += d1;
}

typedef struct {
  cnt_ctx* c;
  int slots;
  uint64_t* out;
} sum_ctx;

static void s_chunk(void* cv, uint64_t ci, int tid) {
  (void)tid;
  sum_ctx* s = (sum_ctx*)cv;
  const uint64_t v0 = ci * VCHUNK, v1 = v0 + VCHUNK < s->c->n ? v0 + VCHUNK : s->c->n;
  for (uint64_t v = v0; v < v1; ++v) {
    uint64_t a = 0;
    for (int t = 0; t < s->slots; ++t) a += s->c->tally[t][v];
    s->out[v] = a;
  }
}

/* count_node_iterator_n (sequential.hpp:74-91) over the oriented CSR on
 * `threads` threads.  Optional outputs (NULL = skip):
 *   tally[n]    NodeTallySink T_v (sequential.hpp:24-33);
 *   apex_tri[p] triangles whose apex v lies in core i of plan b (p+1 ids)
 *               -- AOP per-rank counts (engines.hpp:38-54);
 *   mid_tri[p]  triangles whose middle vertex u lies in core i --
 *               ANOP-surrogate per-rank counts (engines.hpp:60-76);
 *   digest2     the ListSink digest (orc_tri_hash sums).
 * Returns the global count. */
uint64_t orc_count_full(uint64_t n, const uint64_t* eoff, const uint32_t* eff,
                        const uint32_t* b, uint64_t p, int threads, uint64_t* tally,
                        uint64_t* apex_tri, uint64_t* mid_tri, uint64_t* digest2) {
  if (threads < 1) threads = 1;
  if (threads > MAXSLOTS) threads = MAXSLOTS;
  cnt_ctx* c = (cnt_ctx*)calloc(1, sizeof(cnt_ctx));
  c->n = n;
  c->eoff = eoff;
  c->eff = eff;
  c->b = b;
  c->p = p;
  c->vchunk = 1024;
  c->want_tally = tally != NULL;
  c->want_digest = digest2 != NULL;
  for (int t = 0; t < threads; ++t) {
    if (tally) c->tally[t] = (uint64_t*)calloc(n ? n : 1, sizeof(uint64_t));
    if (apex_tri && b) c->apex[t] = (uint64_t*)calloc(p, sizeof(uint64_t));
    if (mid_tri && b) c->mid[t] = (uint64_t*)calloc(p, sizeof(uint64_t));
  }
  parallel_for(threads, (n + c->vchunk - 1) / c->vchunk, c_chunk, c);
  uint64_t total = 0, d0 = 0, d1 = 0;
  for (int t = 0; t < threads; ++t) {
    total += c->total[t];
    d0 += c->d0[t];
    d1 += c->d1[t];
  }
  if (digest2) {
    digest2[0] = d0;
    digest2[1] = d1;
  }
  if (apex_tri && b) {
    memset(apex_tri, 0, p * sizeof(uint64_t));
    for (int t = 0; t < threads; ++t)
      for (uint64_t i = 0; i < p; ++i) apex_tri[i] += c->apex[t][i];
  }
  if (mid_tri && b) {
    memset(mid_tri, 0, p * sizeof(uint64_t));
    for (int t = 0; t < threads; ++t)
      for (uint64_t i = 0; i < p; ++i) mid_tri[i] += c->mid[t][i];
  }
  if (tally) {
    sum_ctx s = {c, threads, tally};
    parallel_for(threads, (n + VCHUNK - 1) / VCHUNK, s_chunk, &s);
  }
  for (int t = 0; t < threads; ++t) {
    free(c->tally[t]);
    free(c->apex[t]);
    free(c->mid[t]);
  }
  free(c);
  return total;
}

/* engines.hpp:173-187 (surrogate LastProc): core-i apex v sends N_v once to
 * every distinct owner j != i of an entry of N_v (owners are nondecreasing
 * along the ID-sorted list).  sent[i] / recv[j] count those NeighborList
 * messages (RankStats data_sent / data_recv). */
void orc_surrogate_messages(uint64_t n, const uint64_t* eoff, const uint32_t* eff,
                            const uint32_t* b, uint64_t p, uint64_t* sent, uint64_t* recv) {
  memset(sent, 0, p * sizeof(uint64_t));
  memset(recv, 0, p * sizeof(uint64_t));
  for (uint64_t i = 0; i < p; ++i)
    for (uint64_t v = b[i]; v < b[i + 1] && v < n; ++v) {
      int64_t last = -1;
      for (uint64_t k = eoff[v]; k < eoff[v + 1]; ++k) {
        const uint64_t j = orc_owner(b, p, eff[k]);
        if (j == i) continue;
        if ((int64_t)j != last) {
          sent[i]++;
          recv[j]++;
          last = (int64_t)j;
        }
      }
    }
}
