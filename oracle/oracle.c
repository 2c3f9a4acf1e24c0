/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Plain-C restatement of the reference trigraph hot path.  Each function
 * cites the reference file:line it follows (paths relative to
 * /root/reference/proj/include/trigraph/ unless stated).  Written for
 * clarity over speed, but O(m log d) so it finishes the parity sizes in
 * seconds.
 */
#include "oracle.h"

#include <stdlib.h>
#include <string.h>

void orc_free(void* p) { free(p); }

static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

/* graph.hpp:58-85.  n = max(n_override, 1 + max id over ALL pairs, self-loops
 * included) (:60-64); self-loops dropped, both directions emitted (:66-72);
 * sort + unique of directed pairs (:73-74) is restated as bucket-by-source +
 * per-bucket sort + unique, which yields the identical CSR (:76-84). */
uint64_t orc_build_graph(const uint32_t* pairs, uint64_t E, uint64_t n_override,
                         uint64_t** off_out, uint32_t** adj_out) {
  uint64_t n = n_override;
  for (uint64_t e = 0; e < E; ++e) {
    uint64_t u = pairs[2 * e], v = pairs[2 * e + 1];
    if (u + 1 > n) n = u + 1;
    if (v + 1 > n) n = v + 1;
  }
  uint64_t* cnt = (uint64_t*)calloc(n + 1, sizeof(uint64_t));
  for (uint64_t e = 0; e < E; ++e) {
    uint32_t u = pairs[2 * e], v = pairs[2 * e + 1];
    if (u == v) continue;
    cnt[u + 1]++;
    cnt[v + 1]++;
  }
  for (uint64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  uint32_t* tmp = (uint32_t*)malloc((cnt[n] ? cnt[n] : 1) * sizeof(uint32_t));
  uint64_t* pos = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
  memcpy(pos, cnt, (n + 1) * sizeof(uint64_t));
  for (uint64_t e = 0; e < E; ++e) {
    uint32_t u = pairs[2 * e], v = pairs[2 * e + 1];
    if (u == v) continue;
    tmp[pos[u]++] = v;
    tmp[pos[v]++] = u;
  }
  uint64_t* off = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
  uint32_t* adj = (uint32_t*)malloc((cnt[n] ? cnt[n] : 1) * sizeof(uint32_t));
  uint64_t w = 0;
  off[0] = 0;
  for (uint64_t v = 0; v < n; ++v) {
    uint32_t* b = tmp + cnt[v];
    uint64_t len = cnt[v + 1] - cnt[v];
    qsort(b, len, sizeof(uint32_t), cmp_u32);
    for (uint64_t k = 0; k < len; ++k)
      if (k == 0 || b[k] != b[k - 1]) adj[w++] = b[k];
    off[v + 1] = w;
  }
  free(tmp);
  free(pos);
  free(cnt);
  *off_out = off;
  *adj_out = adj;
  return n;
}

/* order.hpp:95-104: std::sort of ids by (degree, id), rank[nodes[i]] = i.
 * Restated as a counting sort on degree, stable in id (same total order). */
void orc_degree_rank(uint64_t n, const uint64_t* off, uint32_t* rank) {
  uint64_t maxd = 0;
  for (uint64_t v = 0; v < n; ++v) {
    uint64_t d = off[v + 1] - off[v];
    if (d > maxd) maxd = d;
  }
  uint64_t* start = (uint64_t*)calloc(maxd + 2, sizeof(uint64_t));
  for (uint64_t v = 0; v < n; ++v) start[off[v + 1] - off[v] + 1]++;
  for (uint64_t d = 0; d <= maxd; ++d) start[d + 1] += start[d];
  for (uint64_t v = 0; v < n; ++v) rank[v] = (uint32_t)start[off[v + 1] - off[v]]++;
  free(start);
}

/* order.hpp:39-83 coreness: the Batagelj-Zaversnik bucket peeling.  Nodes
 * are processed in ascending current degree; core[v] = deg[v] at removal and
 * every neighbour u with deg[u] > deg[v] moves down one bucket (:66-79). */
void orc_coreness(uint64_t n, const uint64_t* off, const uint32_t* adj, uint64_t* core) {
  uint64_t maxd = 0;
  uint64_t* deg = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  for (uint64_t v = 0; v < n; ++v) {
    deg[v] = off[v + 1] - off[v];
    if (deg[v] > maxd) maxd = deg[v];
    core[v] = 0;
  }
  uint64_t* bin = (uint64_t*)calloc(maxd + 2, sizeof(uint64_t));
  for (uint64_t v = 0; v < n; ++v) bin[deg[v] + 1]++;
  for (uint64_t d = 0; d <= maxd; ++d) bin[d + 1] += bin[d];
  uint32_t* order = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  uint64_t* pos = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  uint64_t* start = (uint64_t*)malloc((maxd + 2) * sizeof(uint64_t));
  memcpy(start, bin, (maxd + 2) * sizeof(uint64_t));
  for (uint64_t v = 0; v < n; ++v) {
    pos[v] = start[deg[v]]++;
    order[pos[v]] = (uint32_t)v;
  }
  memcpy(start, bin, (maxd + 1) * sizeof(uint64_t));
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t v = order[i];
    core[v] = deg[v];
    for (uint64_t k = off[v]; k < off[v + 1]; ++k) {
      const uint32_t u = adj[k];
      if (deg[u] > deg[v]) {
        const uint64_t du = deg[u], pu = pos[u], pw = start[du];
        const uint32_t w = order[pw];
        if (u != w) {
          order[pu] = w;
          order[pw] = u;
          pos[u] = pw;
          pos[w] = pu;
        }
        ++start[du];
        --deg[u];
      }
    }
  }
  free(start);
  free(pos);
  free(order);
  free(bin);
  free(deg);
}

typedef struct {
  uint64_t a, b, c;
} key3_t;
static const key3_t* g_sort_keys;
static int cmp_key3_idx(const void* x, const void* y) {
  const key3_t* p = &g_sort_keys[*(const uint32_t*)x];
  const key3_t* q = &g_sort_keys[*(const uint32_t*)y];
  if (p->a != q->a) return p->a < q->a ? -1 : 1;
  if (p->b != q->b) return p->b < q->b ? -1 : 1;
  return (p->c > q->c) - (p->c < q->c);
}

/* order.hpp:85-128 compute_order for every OrderKind::Tag (order.hpp:19):
 * ById = identity (:90-93); ByDegree (:94-102); ByRandom = Fisher-Yates over
 * mt19937_64(seed) with a modulo draw, i from n down to 2 (:104-113);
 * ByCoreness = ascending (core, degree, id) (:114-124).  Returns -1 for an
 * unknown kind. */
int orc_compute_order(uint64_t n, const uint64_t* off, const uint32_t* adj, int kind,
                      uint64_t seed, uint32_t* rank) {
  if (kind == ORC_ORDER_BY_DEGREE) {
    orc_degree_rank(n, off, rank);
    return 0;
  }
  if (kind == ORC_ORDER_BY_ID) {
    for (uint64_t v = 0; v < n; ++v) rank[v] = (uint32_t)v;
    return 0;
  }
  uint32_t* nodes = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  for (uint64_t v = 0; v < n; ++v) nodes[v] = (uint32_t)v;
  if (kind == ORC_ORDER_BY_RANDOM) {
    orc_mt64 s;
    orc_mt64_seed(&s, seed);
    for (uint64_t i = n; i > 1; --i) {
      const uint64_t j = orc_mt64_next(&s) % i;
      const uint32_t x = nodes[i - 1];
      nodes[i - 1] = nodes[j];
      nodes[j] = x;
    }
  } else if (kind == ORC_ORDER_BY_CORENESS) {
    uint64_t* core = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    orc_coreness(n, off, adj, core);
    key3_t* keys = (key3_t*)malloc((n ? n : 1) * sizeof(key3_t));
    for (uint64_t v = 0; v < n; ++v) {
      keys[v].a = core[v];
      keys[v].b = off[v + 1] - off[v];
      keys[v].c = v;
    }
    g_sort_keys = keys;
    qsort(nodes, n, sizeof(uint32_t), cmp_key3_idx);
    free(keys);
    free(core);
  } else {
    free(nodes);
    return -1;
  }
  for (uint64_t i = 0; i < n; ++i) rank[nodes[i]] = (uint32_t)i;
  free(nodes);
  return 0;
}

/* effective.hpp:37-52: N_v = {u in adj(v) : rank[v] < rank[u]}, ID-sorted. */
uint64_t orc_effective(uint64_t n, const uint64_t* off, const uint32_t* adj,
                       const uint32_t* rank, uint64_t* eoff, uint32_t** eff_out) {
  eoff[0] = 0;
  for (uint64_t v = 0; v < n; ++v) {
    uint64_t c = 0;
    for (uint64_t k = off[v]; k < off[v + 1]; ++k)
      if (rank[v] < rank[adj[k]]) ++c;
    eoff[v + 1] = eoff[v] + c;
  }
  uint32_t* eff = (uint32_t*)malloc((eoff[n] ? eoff[n] : 1) * sizeof(uint32_t));
  uint64_t w = 0;
  for (uint64_t v = 0; v < n; ++v)
    for (uint64_t k = off[v]; k < off[v + 1]; ++k)
      if (rank[v] < rank[adj[k]]) eff[w++] = adj[k];
  *eff_out = eff;
  return w;
}

/* Sink state shared by the counting loops: sequential.hpp:24-46 and
 * engines.hpp:303-321 (RankSink). */
typedef struct {
  uint64_t* tally;
  uint32_t* tri;
  uint64_t cap;
  uint64_t written;
} sink_t;

static void sink_emit(sink_t* s, uint32_t v, uint32_t u, uint32_t w) {
  if (s->tally) {
    s->tally[v]++;
    s->tally[u]++;
    s->tally[w]++;
  }
  if (s->tri) {
    uint32_t t0 = v, t1 = u, t2 = w, x;
    if (t0 > t1) { x = t0; t0 = t1; t1 = x; }
    if (t1 > t2) { x = t1; t1 = t2; t2 = x; }
    if (t0 > t1) { x = t0; t0 = t1; t1 = x; }
    if (s->written < s->cap) {
      s->tri[3 * s->written + 0] = t0;
      s->tri[3 * s->written + 1] = t1;
      s->tri[3 * s->written + 2] = t2;
    }
    s->written++;
  }
}

/* intersect.hpp:15-33 intersect_visit: scalar merge; emits (v,u,w) for each
 * common w.  Returns the number of common elements. */
static uint64_t merge_emit(const uint32_t* a, uint64_t na, const uint32_t* b,
                           uint64_t nb, sink_t* s, uint32_t v, uint32_t u) {
  uint64_t i = 0, j = 0, c = 0;
  while (i < na && j < nb) {
    if (a[i] < b[j]) ++i;
    else if (b[j] < a[i]) ++j;
    else {
      if (s) sink_emit(s, v, u, a[i]);
      ++c;
      ++i;
      ++j;
    }
  }
  return c;
}

/* sequential.hpp:74-91 count_node_iterator_n. */
uint64_t orc_count(uint64_t n, const uint64_t* eoff, const uint32_t* eff,
                   uint64_t* tally, uint32_t* tri, uint64_t tri_cap) {
  sink_t s = {tally, tri, tri_cap, 0};
  sink_t* sp = (tally || tri) ? &s : NULL;
  uint64_t total = 0;
  for (uint64_t v = 0; v < n; ++v) {
    const uint32_t* nv = eff + eoff[v];
    uint64_t hv = eoff[v + 1] - eoff[v];
    for (uint64_t k = 0; k < hv; ++k) {
      uint32_t u = nv[k];
      total += merge_emit(nv, hv, eff + eoff[u], eoff[u + 1] - eoff[u], sp,
                          (uint32_t)v, u);
    }
  }
  return total;
}

/* NodeIteratorN restricted to apexes [vlo, vhi) (the AOP rank body's loop,
 * engines.hpp:38-54, over the full oriented lists). */
uint64_t orc_count_range(uint64_t n, const uint64_t* eoff, const uint32_t* eff,
                         uint64_t vlo, uint64_t vhi) {
  (void)n;
  uint64_t total = 0;
  for (uint64_t v = vlo; v < vhi; ++v) {
    const uint32_t* nv = eff + eoff[v];
    uint64_t hv = eoff[v + 1] - eoff[v];
    for (uint64_t k = 0; k < hv; ++k) {
      uint32_t u = nv[k];
      total += merge_emit(nv, hv, eff + eoff[u], eoff[u + 1] - eoff[u], NULL, (uint32_t)v, u);
    }
  }
  return total;
}

/* sequential.hpp:95-104 ordering_cost = sum_v d_v * effdeg_v. */
uint64_t orc_ordering_cost(uint64_t n, const uint64_t* off, const uint32_t* adj,
                           const uint32_t* rank) {
  uint64_t cost = 0;
  for (uint64_t v = 0; v < n; ++v) {
    uint64_t h = 0;
    for (uint64_t k = off[v]; k < off[v + 1]; ++k)
      if (rank[v] < rank[adj[k]]) ++h;
    cost += (off[v + 1] - off[v]) * h;
  }
  return cost;
}

static int bsearch_u32(const uint32_t* a, uint64_t n, uint32_t x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo < n && a[lo] == x;
}

static uint64_t lower_bound_u32(const uint32_t* a, uint64_t n, uint32_t x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

/* partition.hpp:45-91 node_costs (DpdVariant::EffectiveOnly) + inclusive
 * prefix (:84-89). */
void orc_node_costs(uint64_t n, const uint64_t* off, const uint32_t* adj,
                    const uint64_t* eoff, const uint32_t* eff, int kind,
                    uint64_t* f, uint64_t* prefix) {
  for (uint64_t v = 0; v < n; ++v) {
    uint64_t dv = off[v + 1] - off[v];
    uint64_t hv = eoff[v + 1] - eoff[v];
    uint64_t s = 0;
    switch (kind) {
      case ORC_COST_N: s = 1; break;
      case ORC_COST_D: s = dv; break;
      case ORC_COST_DH: s = hv; break;
      case ORC_COST_DDH: s = dv * hv; break;
      case ORC_COST_DH2: s = hv * hv; break;
      case ORC_COST_DPD: /* :60-69 */
        for (uint64_t k = eoff[v]; k < eoff[v + 1]; ++k) {
          uint32_t u = eff[k];
          s += hv + (eoff[u + 1] - eoff[u]);
        }
        break;
      case ORC_COST_NOV: /* :70-81 predecessors: neighbours not in N_v */
        for (uint64_t k = off[v]; k < off[v + 1]; ++k) {
          uint32_t u = adj[k];
          if (!bsearch_u32(eff + eoff[v], hv, u)) s += hv + (eoff[u + 1] - eoff[u]);
        }
        break;
      default: s = 0;
    }
    f[v] = s;
  }
  uint64_t acc = 0;
  for (uint64_t i = 0; i < n; ++i) {
    acc += f[i];
    prefix[i] = acc;
  }
}

/* partition.hpp:116-141: boundary x_j = smallest x in [x_{j-1}, n] with
 * p * F(x-1) >= j * total, exact 128-bit comparison (:130-135). */
int orc_compute_boundaries(const uint64_t* prefix, uint64_t n, uint64_t p,
                           uint32_t* b) {
  if (p == 0) return -1;
  uint64_t total = n ? prefix[n - 1] : 0;
  b[0] = 0;
  for (uint64_t j = 1; j < p; ++j) {
    unsigned __int128 target = (unsigned __int128)j * total;
    uint32_t lo = b[j - 1], hi = (uint32_t)n;
    while (lo < hi) {
      uint32_t mid = lo + (hi - lo) / 2;
      uint64_t before = mid == 0 ? 0 : prefix[mid - 1];
      unsigned __int128 lhs = (unsigned __int128)p * before;
      if (lhs >= target) hi = mid;
      else lo = mid + 1;
    }
    b[j] = lo;
  }
  b[p] = (uint32_t)n;
  return 0;
}

/* partition.hpp:106-109: upper_bound over the inner boundaries b[1..p-1]. */
uint64_t orc_owner(const uint32_t* b, uint64_t p, uint32_t v) {
  uint64_t lo = 1, hi = p; /* search in [1, p) */
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (b[mid] <= v) lo = mid + 1;
    else hi = mid;
  }
  return lo - 1;
}

/* ---- engines --------------------------------------------------------- */

typedef struct {
  uint64_t n;
  const uint64_t* eoff;
  const uint32_t* eff;
} effadj_t;

#define LIST(E, v) ((E)->eff + (E)->eoff[(v)])
#define LEN(E, v) ((E)->eoff[(v) + 1] - (E)->eoff[(v)])

/* engines.hpp:38-54 aop_count over partition.hpp:171-206
 * build_overlap_partition.  The halo lists are trimmed to partition members
 * exactly as the reference does; *stored receives stored_entries(). */
static uint64_t aop_rank(const effadj_t* E, uint32_t cb, uint32_t ce, sink_t* s,
                         uint64_t* stored) {
  uint8_t* in_halo = (uint8_t*)calloc(E->n ? E->n : 1, 1);
  uint64_t st = 0;
  for (uint32_t v = cb; v < ce; ++v) {
    st += LEN(E, v);
    for (uint64_t k = 0; k < LEN(E, v); ++k) {
      uint32_t u = LIST(E, v)[k];
      if (u < cb || u >= ce) in_halo[u] = 1;
    }
  }
  /* trimmed halo lists (partition.hpp:192-204) */
  uint32_t** tl = (uint32_t**)calloc(E->n ? E->n : 1, sizeof(uint32_t*));
  uint64_t* tn = (uint64_t*)calloc(E->n ? E->n : 1, sizeof(uint64_t));
  for (uint64_t w = 0; w < E->n; ++w) {
    if (!in_halo[w]) continue;
    tl[w] = (uint32_t*)malloc((LEN(E, w) ? LEN(E, w) : 1) * sizeof(uint32_t));
    for (uint64_t k = 0; k < LEN(E, w); ++k) {
      uint32_t x = LIST(E, w)[k];
      if ((x >= cb && x < ce) || in_halo[x]) tl[w][tn[w]++] = x;
    }
    st += tn[w];
  }
  uint64_t total = 0;
  for (uint32_t v = cb; v < ce; ++v) {
    const uint32_t* nv = LIST(E, v);
    uint64_t hv = LEN(E, v);
    for (uint64_t k = 0; k < hv; ++k) {
      uint32_t u = nv[k];
      const uint32_t* lu;
      uint64_t nu;
      if (u >= cb && u < ce) {
        lu = LIST(E, u);
        nu = LEN(E, u);
      } else {
        lu = tl[u];
        nu = tn[u];
      }
      total += merge_emit(nv, hv, lu, nu, s, v, u);
    }
  }
  for (uint64_t w = 0; w < E->n; ++w) free(tl[w]);
  free(tl);
  free(tn);
  free(in_halo);
  *stored = st;
  return total;
}

/* engines.hpp:60-76 surrogate_handle: for u in X cap [cb, ce) (contiguous in
 * the ID-sorted X, found by lower_bound), add |N_u cap X|. */
static uint64_t surrogate_handle(const effadj_t* E, uint32_t v, const uint32_t* x,
                                 uint64_t nx, uint32_t cb, uint32_t ce, sink_t* s) {
  uint64_t lo = 0, hi = nx;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (x[mid] < cb) lo = mid + 1;
    else hi = mid;
  }
  uint64_t total = 0;
  for (uint64_t k = lo; k < nx && x[k] < ce; ++k) {
    uint32_t u = x[k];
    total += merge_emit(LIST(E, u), LEN(E, u), x, nx, s, v, u);
  }
  return total;
}

/* ---- sparsification (sparsify.hpp) ----------------------------------- */

/* sparsify.hpp:37-45 detail::mix64 (the SplitMix64 finaliser). */
static uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return x;
}

/* sparsify.hpp:48-54 entry_unit + :58-62 keep_entry, with the rank key
 * already resolved (0 in Global mode, rank + 1 in PerPartition mode). */
int orc_keep_entry(double q, uint64_t seed, uint64_t rank_key, uint32_t v, uint32_t u) {
  uint64_t h = mix64(seed);
  h = mix64(h ^ rank_key);
  h = mix64(h ^ ((uint64_t)v + 0x51ed270b684a1571ULL));
  h = mix64(h ^ (uint64_t)u);
  return (double)(h >> 11) * 0x1.0p-53 < q;
}

/* Sparsified copy of E (sparsify.hpp:68-75 sparsify_list per row): row v
 * keeps entry u iff keep_entry with key kc (b == NULL) or owner(v)+1 (the
 * non-overlapping partitions of a PerPartition run, sparsify.hpp:85-89). */
static void sparsify_rows(uint64_t n, const uint64_t* eoff, const uint32_t* eff, double q,
                          uint64_t seed, uint64_t kc, const uint32_t* b, uint64_t p,
                          uint64_t* eoff2, uint32_t** eff2) {
  uint32_t* out = (uint32_t*)malloc((eoff[n] ? eoff[n] : 1) * sizeof(uint32_t));
  uint64_t w = 0;
  eoff2[0] = 0;
  for (uint64_t v = 0; v < n; ++v) {
    const uint64_t key = b ? orc_owner(b, p, (uint32_t)v) + 1 : kc;
    for (uint64_t k = eoff[v]; k < eoff[v + 1]; ++k)
      if (orc_keep_entry(q, seed, key, (uint32_t)v, eff[k])) out[w++] = eff[k];
    eoff2[v + 1] = w;
  }
  *eff2 = out;
}

uint64_t orc_run_engine(uint64_t n, const uint64_t* off, const uint32_t* adj,
                        int engine, uint64_t p, int cost,
                        const uint32_t* boundaries_in, uint32_t* boundaries_out,
                        uint64_t* tri, uint64_t* sent, uint64_t* recv,
                        uint64_t* stored, uint64_t* tally, uint32_t* list,
                        uint64_t list_cap) {
  return orc_run_engine_ex(n, off, adj, engine, p, cost, boundaries_in, boundaries_out, tri,
                           sent, recv, stored, tally, list, list_cap, 0, 1.0, 0);
}

/* engines.hpp:335-418 with cfg.sparsify (smode 1 = Global, 2 =
 * PerPartition, 0 = none).  Sequential sparsifies the effective adjacency
 * as rank 0 (:362-365, sparsify.hpp:94-107); AOP sparsifies each rank's
 * overlap partition with that rank's draws (:367-371, sparsify.hpp:80-84) --
 * the count equals NodeIteratorN over the apex core on the whole
 * adjacency sparsified with that key, because N'_v lies inside core+halo;
 * ANOP sparsifies each rank's core lists with its own draws (:387-391).
 * stored[] is the partition storage as built (before sparsification). */
uint64_t orc_run_engine_ex(uint64_t n, const uint64_t* off, const uint32_t* adj,
                           int engine, uint64_t p, int cost,
                           const uint32_t* boundaries_in, uint32_t* boundaries_out,
                           uint64_t* tri, uint64_t* sent, uint64_t* recv,
                           uint64_t* stored, uint64_t* tally, uint32_t* list,
                           uint64_t list_cap, int smode, double q, uint64_t seed) {
  return orc_run_engine_ord(n, off, adj, engine, p, cost, boundaries_in, boundaries_out, tri,
                            sent, recv, stored, tally, list, list_cap, smode, q, seed,
                            ORC_ORDER_BY_DEGREE, 0);
}

/* engines.hpp:335-418 with cfg.order (:274, compute_order at :341). */
uint64_t orc_run_engine_ord(uint64_t n, const uint64_t* off, const uint32_t* adj,
                            int engine, uint64_t p, int cost,
                            const uint32_t* boundaries_in, uint32_t* boundaries_out,
                            uint64_t* tri, uint64_t* sent, uint64_t* recv,
                            uint64_t* stored, uint64_t* tally, uint32_t* list,
                            uint64_t list_cap, int smode, double q, uint64_t seed,
                            int order, uint64_t order_seed) {
  /* engines.hpp:337-338 */
  if (engine == ORC_ENGINE_SEQ) p = 1;
  if (p == 0) return UINT64_MAX;
  uint32_t* rank = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  if (orc_compute_order(n, off, adj, order, order_seed, rank) != 0) {
    free(rank);
    return UINT64_MAX;
  }
  uint64_t* eoff = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
  uint32_t* eff = NULL;
  orc_effective(n, off, adj, rank, eoff, &eff);
  uint64_t* f = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  uint64_t* prefix = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  orc_node_costs(n, off, adj, eoff, eff, cost, f, prefix);
  /* engines.hpp:343-344: boundary override */
  if (boundaries_in) memcpy(boundaries_out, boundaries_in, (p + 1) * sizeof(uint32_t));
  else orc_compute_boundaries(prefix, n, p, boundaries_out);
  const uint32_t* b = boundaries_out;

  effadj_t E = {n, eoff, eff};
  sink_t s = {tally, list, list_cap, 0};
  sink_t* sp = (tally || list) ? &s : NULL;
  for (uint64_t i = 0; i < p; ++i) tri[i] = sent[i] = recv[i] = stored[i] = 0;
  uint64_t* eoff2 = NULL;
  uint32_t* eff2 = NULL;
  if (smode) eoff2 = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));

  if (engine == ORC_ENGINE_SEQ) {
    /* engines.hpp:362-365 */
    stored[0] = eoff[n];
    if (smode) {
      sparsify_rows(n, eoff, eff, q, seed, smode == 2 ? 1 : 0, NULL, 0, eoff2, &eff2);
      tri[0] = orc_count(n, eoff2, eff2, tally, list, list_cap);
    } else {
      tri[0] = orc_count(n, eoff, eff, tally, list, list_cap);
    }
  } else if (engine == ORC_ENGINE_AOP) {
    for (uint64_t i = 0; i < p; ++i) {
      if (!smode) {
        tri[i] = aop_rank(&E, b[i], b[i + 1], sp, &stored[i]);
        continue;
      }
      uint64_t dummy = 0;
      aop_rank(&E, b[i], b[i + 1], NULL, &stored[i]);
      sparsify_rows(n, eoff, eff, q, seed, smode == 2 ? i + 1 : 0, NULL, 0, eoff2, &eff2);
      effadj_t Es = {n, eoff2, eff2};
      tri[i] = aop_rank(&Es, b[i], b[i + 1], sp, &dummy);
      free(eff2);
      eff2 = NULL;
    }
  } else {
    for (uint64_t i = 0; i < p; ++i) stored[i] = eoff[b[i + 1]] - eoff[b[i]];
    if (smode) {
      sparsify_rows(n, eoff, eff, q, seed, 0, smode == 2 ? b : NULL, p, eoff2, &eff2);
      E.eoff = eoff2;
      E.eff = eff2;
    }
    for (uint64_t i = 0; i < p; ++i) {
      uint32_t cb = b[i], ce = b[i + 1];
      for (uint32_t v = cb; v < ce; ++v) {
        const uint32_t* nv = LIST(&E, v);
        uint64_t hv = LEN(&E, v);
        int64_t last = -1;
        for (uint64_t k = 0; k < hv; ++k) {
          uint32_t u = nv[k];
          if (u >= cb && u < ce) { /* local intersection */
            tri[i] += merge_emit(nv, hv, LIST(&E, u), LEN(&E, u), sp, v, u);
            continue;
          }
          uint64_t j = orc_owner(b, p, u);
          if (engine == ORC_ENGINE_ANOP_DIRECT) {
            /* engines.hpp:97-111: request + reply per (v,u), no caching */
            sent[i]++;
            recv[j]++;
            sent[j]++;
            recv[i]++;
            tri[i] += merge_emit(nv, hv, LIST(&E, u), LEN(&E, u), sp, v, u);
          } else if ((int64_t)j != last) {
            /* engines.hpp:173-187: LastProc dedup, ship N_v to owner(u);
             * the owner runs surrogate_handle (:60-76) on arrival. */
            sent[i]++;
            recv[j]++;
            last = (int64_t)j;
            tri[j] += surrogate_handle(&E, v, nv, hv, b[j], b[j + 1], sp);
          }
        }
      }
    }
  }
  uint64_t total = 0;
  for (uint64_t i = 0; i < p; ++i) total += tri[i];
  free(rank);
  free(eoff);
  free(eff);
  free(eoff2);
  free(eff2);
  free(f);
  free(prefix);
  return total;
}

/* engines.hpp:440-457 approx_count: PerPartition draws for AOP, Global for
 * the others; T' / q^3.  Returns NaN on invalid arguments. */
double orc_approx_count(uint64_t n, const uint64_t* off, const uint32_t* adj, uint64_t p,
                        int engine, double q, uint64_t seed, const uint32_t* boundaries,
                        int cost) {
  if (!(q > 0.0 && q <= 1.0)) return 0.0 / 0.0; /* sparsify.hpp:28-31 */
  const uint64_t pp = engine == ORC_ENGINE_SEQ ? 1 : p;
  if (pp == 0) return 0.0 / 0.0;
  uint32_t* bo = (uint32_t*)malloc((pp + 1) * sizeof(uint32_t));
  uint64_t* a = (uint64_t*)malloc(4 * pp * sizeof(uint64_t));
  const uint64_t t = orc_run_engine_ex(n, off, adj, engine, p, cost, boundaries, bo, a, a + pp,
                                       a + 2 * pp, a + 3 * pp, NULL, NULL, 0,
                                       engine == ORC_ENGINE_AOP ? 2 : 1, q, seed);
  free(bo);
  free(a);
  return (double)t / (q * q * q);
}

/* sequential.hpp:108-122 per_edge_triangle_counts, in Graph::edges() order
 * (graph.hpp:40-46: u ascending, v ascending, u < v).  te has m entries. */
void orc_per_edge_counts(uint64_t n, const uint64_t* off, const uint32_t* adj, uint64_t* te) {
  uint32_t* rank = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  orc_degree_rank(n, off, rank);
  uint64_t* eoff = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
  uint32_t* eff = NULL;
  orc_effective(n, off, adj, rank, eoff, &eff);
  /* edge index of (a, b), a < b: upper-triangle position */
  uint64_t* up = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
  up[0] = 0;
  for (uint64_t v = 0; v < n; ++v) {
    uint64_t c = 0;
    for (uint64_t k = off[v]; k < off[v + 1]; ++k) c += adj[k] > v;
    up[v + 1] = up[v] + c;
  }
  memset(te, 0, up[n] * sizeof(uint64_t));
#define EIDX(a, b) (up[(a)] + lower_bound_u32(adj + off[(a)], off[(a) + 1] - off[(a)], (b)) \
                    - lower_bound_u32(adj + off[(a)], off[(a) + 1] - off[(a)], (a)))
  for (uint64_t v = 0; v < n; ++v) {
    const uint32_t* nv = eff + eoff[v];
    const uint64_t hv = eoff[v + 1] - eoff[v];
    for (uint64_t k = 0; k < hv; ++k) {
      const uint32_t u = nv[k];
      const uint32_t* nu = eff + eoff[u];
      const uint64_t hu = eoff[u + 1] - eoff[u];
      uint64_t i = 0, j = 0;
      while (i < hv && j < hu) {
        if (nv[i] < nu[j]) ++i;
        else if (nu[j] < nv[i]) ++j;
        else {
          const uint32_t w = nv[i], x = (uint32_t)v;
          te[x < u ? EIDX(x, u) : EIDX(u, x)]++;
          te[x < w ? EIDX(x, w) : EIDX(w, x)]++;
          te[u < w ? EIDX(u, w) : EIDX(w, u)]++;
          ++i;
          ++j;
        }
      }
    }
  }
#undef EIDX
  free(up);
  free(rank);
  free(eoff);
  free(eff);
}

/* sparsify.hpp:113-155 variance_report: k = pairs of triangles sharing an
 * edge, k' = those pairs whose apexes (order-smallest corners) have the same
 * owner under plan b; var = (1/q^3 - 1) T + 2 k (1/q - 1), var' with k'.
 * out3 = {T, k, k'}, var2 = {var, var'}. */
void orc_variance_report(uint64_t n, const uint64_t* off, const uint32_t* adj,
                         const uint32_t* b, uint64_t p, double q, uint64_t* out3,
                         double* var2) {
  uint32_t* rank = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  orc_degree_rank(n, off, rank);
  uint64_t* eoff = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
  uint32_t* eff = NULL;
  orc_effective(n, off, adj, rank, eoff, &eff);
  const uint64_t m = off[n] / 2;
  /* per edge: count of triangles, and per (edge, owner of apex) counts via
   * one pass per owner (apexes of core i only) */
  uint64_t* te = (uint64_t*)malloc((m ? m : 1) * sizeof(uint64_t));
  uint64_t* up = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
  up[0] = 0;
  for (uint64_t v = 0; v < n; ++v) {
    uint64_t c = 0;
    for (uint64_t k = off[v]; k < off[v + 1]; ++k) c += adj[k] > v;
    up[v + 1] = up[v] + c;
  }
#define EIDX(a, b) (up[(a)] + lower_bound_u32(adj + off[(a)], off[(a) + 1] - off[(a)], (b)) \
                    - lower_bound_u32(adj + off[(a)], off[(a) + 1] - off[(a)], (a)))
  uint64_t T = 0, kp = 0;
  uint64_t* tot = (uint64_t*)calloc(m ? m : 1, sizeof(uint64_t));
  for (uint64_t i = 0; i < p; ++i) {
    memset(te, 0, (m ? m : 1) * sizeof(uint64_t));
    for (uint64_t v = b[i]; v < b[i + 1]; ++v) {
      const uint32_t* nv = eff + eoff[v];
      const uint64_t hv = eoff[v + 1] - eoff[v];
      for (uint64_t k = 0; k < hv; ++k) {
        const uint32_t u = nv[k];
        const uint32_t* nu = eff + eoff[u];
        const uint64_t hu = eoff[u + 1] - eoff[u];
        uint64_t a = 0, c = 0;
        while (a < hv && c < hu) {
          if (nv[a] < nu[c]) ++a;
          else if (nu[c] < nv[a]) ++c;
          else {
            const uint32_t w = nv[a], x = (uint32_t)v;
            const uint64_t e1 = x < u ? EIDX(x, u) : EIDX(u, x);
            const uint64_t e2 = x < w ? EIDX(x, w) : EIDX(w, x);
            const uint64_t e3 = u < w ? EIDX(u, w) : EIDX(w, u);
            te[e1]++; te[e2]++; te[e3]++;
            tot[e1]++; tot[e2]++; tot[e3]++;
            ++T;
            ++a;
            ++c;
          }
        }
      }
    }
    for (uint64_t e = 0; e < m; ++e) kp += te[e] * (te[e] - (te[e] > 0)) / 2;
  }
  uint64_t k = 0;
  for (uint64_t e = 0; e < m; ++e) k += tot[e] * (tot[e] - (tot[e] > 0)) / 2;
#undef EIDX
  out3[0] = T;
  out3[1] = k;
  out3[2] = kp;
  const double q3 = q * q * q;
  var2[0] = (1.0 / q3 - 1.0) * (double)T + 2.0 * (double)k * (1.0 / q - 1.0);
  var2[1] = (1.0 / q3 - 1.0) * (double)T + 2.0 * (double)kp * (1.0 / q - 1.0);
  free(tot);
  free(te);
  free(up);
  free(rank);
  free(eoff);
  free(eff);
}

/* engines.hpp:428-433: C_v = 2 T_v / (d (d-1)) in fp64, 0 when d < 2. */
void orc_cc(uint64_t n, const uint64_t* off, const uint64_t* tally, double* c) {
  for (uint64_t v = 0; v < n; ++v) {
    uint64_t d = off[v + 1] - off[v];
    c[v] = d >= 2 ? 2.0 * (double)tally[v] / ((double)d * (double)(d - 1)) : 0.0;
  }
}

/* ---- edge-list text (io.hpp:18-64) ------------------------------------ */

/* std::isspace in the "C" locale (istream >> skips these). */
static int orc_isspace(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

/* istream >> unsigned long long, as libstdc++'s num_get extracts it: skip
 * whitespace, optional sign, one or more decimal digits; overflow fails;
 * '-' negates modulo 2^64.  Returns 1 on success. */
static int orc_extract_ull(const char* s, uint64_t n, uint64_t* i, uint64_t* out) {
  while (*i < n && orc_isspace((unsigned char)s[*i])) ++*i;
  if (*i >= n) return 0;
  int neg = 0;
  if (s[*i] == '+' || s[*i] == '-') {
    neg = s[*i] == '-';
    ++*i;
  }
  if (*i >= n || s[*i] < '0' || s[*i] > '9') return 0;
  uint64_t acc = 0;
  int over = 0;
  while (*i < n && s[*i] >= '0' && s[*i] <= '9') {
    const uint64_t d = (uint64_t)(s[*i] - '0');
    if (acc > (UINT64_MAX - d) / 10) over = 1;
    else acc = acc * 10 + d;
    ++*i;
  }
  if (over) return 0;
  *out = neg ? (uint64_t)0 - acc : acc;
  return 1;
}

/* io.hpp:24-50 parse_edge_list.  Lines split at '\n' (:29-35); a line whose
 * first byte outside " \t\r" is absent or '#' is skipped (:37-39); then two
 * unsigned extractions (:41-43) and no further token (:44-45); ids are the
 * values truncated to NodeId (:46).  Returns the pair count (pairs written
 * up to cap), or UINT64_MAX on a ParseError with *err_line (1-based),
 * *err_kind (1 = "expected two integer tokens", 2 = "trailing token") and,
 * for kind 2, the token's byte range [*tok_b, *tok_e). */
uint64_t orc_parse_edge_list(const char* text, uint64_t len, uint32_t* pairs, uint64_t cap,
                             uint64_t* err_line, int* err_kind, uint64_t* tok_b,
                             uint64_t* tok_e) {
  uint64_t count = 0, lineno = 0, pos = 0;
  while (pos < len) {
    uint64_t end = pos;
    while (end < len && text[end] != '\n') ++end;
    const uint64_t b = pos, e = end;
    pos = end + 1;
    ++lineno;
    uint64_t first = b;
    while (first < e && (text[first] == ' ' || text[first] == '\t' || text[first] == '\r'))
      ++first;
    if (first == e || text[first] == '#') continue;
    uint64_t i = b, u = 0, v = 0;
    if (!orc_extract_ull(text, e, &i, &u) || !orc_extract_ull(text, e, &i, &v)) {
      *err_line = lineno;
      *err_kind = 1;
      return UINT64_MAX;
    }
    while (i < e && orc_isspace((unsigned char)text[i])) ++i;
    if (i < e) {
      uint64_t j = i;
      while (j < e && !orc_isspace((unsigned char)text[j])) ++j;
      *err_line = lineno;
      *err_kind = 2;
      *tok_b = i;
      *tok_e = j;
      return UINT64_MAX;
    }
    if (count < cap) {
      pairs[2 * count] = (uint32_t)u;
      pairs[2 * count + 1] = (uint32_t)v;
    }
    ++count;
  }
  return count;
}

/* io.hpp:52-64 write_edge_list: "u v\n" for every edge with u < v, u then
 * neighbour order.  Writes up to cap bytes; returns the full length. */
uint64_t orc_write_edge_list(uint64_t n, const uint64_t* off, const uint32_t* adj, char* out,
                             uint64_t cap) {
  uint64_t w = 0;
  char buf[32];
  for (uint64_t u = 0; u < n; ++u)
    for (uint64_t k = off[u]; k < off[u + 1]; ++k) {
      if (u >= adj[k]) continue;
      int len = 0;
      uint64_t x = adj[k];
      char tmp[12];
      int t = 0;
      do { tmp[t++] = (char)('0' + x % 10); x /= 10; } while (x);
      uint64_t y = u;
      char tu[12];
      int tl = 0;
      do { tu[tl++] = (char)('0' + y % 10); y /= 10; } while (y);
      while (tl) buf[len++] = tu[--tl];
      buf[len++] = ' ';
      while (t) buf[len++] = tmp[--t];
      buf[len++] = '\n';
      for (int c = 0; c < len; ++c, ++w)
        if (w < cap) out[w] = buf[c];
    }
  return w;
}

/* ---- fixtures -------------------------------------------------------- */

/* std::mt19937_64 (the standard's 64-bit Mersenne Twister parameters). */
void orc_mt64_seed(orc_mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->mti = 312;
}

uint64_t orc_mt64_next(orc_mt64* s) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  const uint64_t A = 0xB5026F5AA96619E9ULL;
  if (s->mti >= 312) {
    int i;
    for (i = 0; i < 312 - 156; ++i) {
      uint64_t x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ ((x & 1) ? A : 0);
    }
    for (; i < 311; ++i) {
      uint64_t x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + 156 - 312] ^ (x >> 1) ^ ((x & 1) ? A : 0);
    }
    uint64_t x = (s->mt[311] & UM) | (s->mt[0] & LM);
    s->mt[311] = s->mt[155] ^ (x >> 1) ^ ((x & 1) ? A : 0);
    s->mti = 0;
  }
  uint64_t x = s->mt[s->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* std::uniform_real_distribution<double>(0,1) over mt19937_64 as libstdc++
 * implements it: generate_canonical<double,53> with one 64-bit draw,
 * (double)draw / 2^64, clamped below 1. */
static double unit_canonical(orc_mt64* s) {
  double r = (double)orc_mt64_next(s) / 18446744073709551616.0;
  if (r >= 1.0) r = 0x1.fffffffffffffp-1;
  return r;
}

/* proj/tests/oracles.hpp:49-57 */
uint64_t orc_random_graph_pairs(uint64_t n, double density, uint64_t seed,
                                uint32_t* out, uint64_t cap) {
  orc_mt64 s;
  orc_mt64_seed(&s, seed);
  uint64_t c = 0;
  for (uint64_t u = 0; u < n; ++u)
    for (uint64_t v = u + 1; v < n; ++v)
      if (unit_canonical(&s) < density) {
        if (c < cap) {
          out[2 * c] = (uint32_t)u;
          out[2 * c + 1] = (uint32_t)v;
        }
        ++c;
      }
  return c;
}
