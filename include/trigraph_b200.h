/*
 * trigraph_b200.h -- C ABI of the B200-native exact triangle counter.
 *
 * Drop-in boundary for the reference `trigraph` hot path
 * (/root/reference/proj/include/trigraph/).  The reference has no FFI: its
 * boundary is the header-only C++ API, so every entry point below names the
 * reference function it replaces (file:line, relative to proj/include/trigraph/).
 * The C++ mirror in include/trigraph_b200/trigraph.hpp wraps these calls
 * behind the reference's own names and types.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Node ids are uint32_t (NodeId,
 *    graph.hpp:14); offsets and counters are uint64_t (size_t/uint64_t in the
 *    reference).
 *  - Input arrays may live in host memory (pageable or pinned) or device
 *    memory; the library detects which (cudaPointerGetAttributes).  Output
 *    arrays are caller-allocated HOST buffers unless the name says `_device`.
 *  - Every call returns a tg_status; tg_last_error() gives the message of the
 *    last failure on the calling thread.  The C++ mirror maps
 *    TG_ERR_INVALID_ARGUMENT to std::invalid_argument (engines.hpp:338,
 *    partition.hpp:117) and everything else to std::runtime_error.
 *  - A tg_graph lives on one device and is not thread-safe; calls on
 *    distinct graphs may run concurrently.  There is no CPU fallback: without
 *    a CUDA device every compute call fails with TG_ERR_CUDA.
 */
#ifndef TRIGRAPH_B200_H
#define TRIGRAPH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TG_OK = 0,
  TG_ERR_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
  TG_ERR_CUDA = 2,
  TG_ERR_OOM = 3,
  TG_ERR_CAPACITY = 4, /* caller buffer too small; required size reported */
  TG_ERR_INTERNAL = 5,
  TG_ERR_PARSE = 6 /* reference: trigraph::ParseError (io.hpp:18-22) */
} tg_status;

/* engines.hpp:24 EngineKind (same order). */
typedef enum {
  TG_ENGINE_SEQ = 0,
  TG_ENGINE_AOP = 1,
  TG_ENGINE_ANOP_DIRECT = 2,
  TG_ENGINE_ANOP_SURROGATE = 3
} tg_engine;

/* partition.hpp:18 CostKind (same order). */
typedef enum {
  TG_COST_N = 0,
  TG_COST_D = 1,
  TG_COST_DH = 2,
  TG_COST_DDH = 3,
  TG_COST_DH2 = 4,
  TG_COST_DPD = 5,
  TG_COST_NOV = 6
} tg_cost;

/* order.hpp:19 OrderKind::Tag (same order). */
typedef enum {
  TG_ORDER_BY_ID = 0,
  TG_ORDER_BY_DEGREE = 1, /* the reference default and the hot path */
  TG_ORDER_BY_RANDOM = 2, /* seeded Fisher-Yates, mt19937_64 */
  TG_ORDER_BY_CORENESS = 3,
  TG_ORDER_RANK = 16 /* a caller-supplied OrderRank (tg_set_order_rank) */
} tg_order;

/* engines.hpp:270-280 EngineConfig.  ExecMode has no meaning on the device
 * (results are mode-independent, acceptance.cpp:438-468).  A zero-
 * initialised config keeps the graph's current order (ByDegree unless
 * tg_set_order changed it); order_set = 1 selects OrderKind{order,
 * order_seed} (EngineConfig::order, engines.hpp:274). */
typedef struct {
  int32_t engine;            /* tg_engine */
  int32_t cost;              /* tg_cost, default TG_COST_DPD */
  uint64_t ranks;            /* logical ranks (>= 1; ignored by SEQ) */
  const uint32_t* boundaries;/* optional override, ranks+1 entries, host memory */
  int32_t track_nodes;       /* fill per-node counts */
  int32_t collect_triangles; /* fill the triangle list */
  /* optional<SparsifyConfig> (engines.hpp:279, sparsify.hpp:22-33):
   * TG_SPARSIFY_NONE / _GLOBAL / _PER_PARTITION, retention q in (0, 1]. */
  int32_t sparsify;
  double sparsify_q;
  uint64_t sparsify_seed;
  int32_t order_set;         /* 0: the graph's current order */
  int32_t order;             /* tg_order (when order_set) */
  uint64_t order_seed;       /* ByRandom seed (OrderKind::seed) */
} tg_config;

/* sparsify.hpp:22-24 SparsifyConfig::Mode (0 = no sparsification). */
typedef enum { TG_SPARSIFY_NONE = 0, TG_SPARSIFY_GLOBAL = 1, TG_SPARSIFY_PER_PARTITION = 2 } tg_sparsify;

/* engines.hpp:282-287 RankStats.  realized_cost is reported as the
 * algorithmic work sum_{v->u in rank} (h_v + h_u) (the DPD cost of the rank's
 * apexes), not merge comparisons. stored_entries is the
 * rank's partition storage (partition.hpp:163-168 / :218-222). */
typedef struct {
  uint64_t triangles;
  uint64_t data_sent;
  uint64_t data_recv;
  uint64_t realized_cost;
  uint64_t stored_entries;
} tg_rank_stats;

typedef struct tg_graph tg_graph;

/* ---- graph construction (graph.hpp:58-85 build_graph; Graph ctor :22) ---- */

/* build_graph on the device: drop self-loops, symmetrise, sort, unique.
 * pairs = E interleaved (u,v); n = max(n_override, 1 + max id). */
tg_status tg_graph_from_edges(int device, const uint32_t* pairs, uint64_t num_pairs,
                              uint64_t n_override, tg_graph** out);
/* Adopt an already-built symmetric CSR (offsets n+1, adj offsets[n]).  Lists
 * must be ID-sorted, loop- and duplicate-free (the Graph invariant). */
tg_status tg_graph_from_csr(int device, uint64_t n, const uint64_t* offsets,
                            const uint32_t* adj, tg_graph** out);
tg_status tg_graph_free(tg_graph* g);
/* count_node_iterator_n(effective_adjacency(Graph(n, offsets, adj), by_degree))
 * in one call from a HOST CSR (graph.hpp:22, effective.hpp:37-52,
 * sequential.hpp:74-91): the adjacency is streamed to the device in vertex
 * chunks on a copy stream while the chunks that already arrived are oriented
 * and every apex whose lists are all resident is counted, so the transfer
 * hides the orientation and most of the intersection.  Overlap needs
 * page-locked host buffers (pageable ones work, serialised).  Device
 * pointers fall back to tg_graph_from_csr + tg_count. */
tg_status tg_count_from_csr(int device, uint64_t n, const uint64_t* offsets, const uint32_t* adj,
                            uint64_t* total);
/* The same, counting only the apexes in [vlo, vhi): one AOP rank's body
 * (engines.hpp:38-54) from a host CSR, e.g. core i of a DPD plan. */
tg_status tg_count_from_csr_range(int device, uint64_t n, const uint64_t* offsets,
                                  const uint32_t* adj, uint64_t vlo, uint64_t vhi,
                                  uint64_t* total);
/* build_graph(parse_edge_list(text), n_override) with both steps on the
 * device (the CLI's --input path, cli.hpp:81-88).  text: len bytes, host or
 * device.  On malformed input: TG_ERR_PARSE, *err_line (may be NULL) = the
 * 1-based line of the first bad line, tg_last_error() = "line N: ..." (the
 * ParseError message, io.hpp:18-22, 41-45). */
tg_status tg_graph_from_text(int device, const char* text, uint64_t len, uint64_t n_override,
                             tg_graph** out, uint64_t* err_line);
/* Graph::num_nodes / num_edges (graph.hpp:25-26). */
tg_status tg_graph_info(tg_graph* g, uint64_t* num_nodes, uint64_t* num_edges);
/* Copy the CSR back (offsets n+1, adj 2m). */
tg_status tg_graph_csr(tg_graph* g, uint64_t* offsets, uint32_t* adj);
/* Launch on this CUDA stream (cudaStream_t) from now on; 0 = the library's own. */
tg_status tg_set_stream(tg_graph* g, void* stream);

/* ---- preprocessing (order.hpp:95-104, effective.hpp:37-52) ---- */

/* Select the total order every later preprocessing and counting call on g
 * orients by: compute_order(g, OrderKind{kind, seed}) (order.hpp:85-128).
 * ByDegree (the default) keys on the degrees; ById, ByRandom(seed) and
 * ByCoreness build their rank array on the device (ByRandom's sequential
 * Fisher-Yates on the host).  Drops the cached oriented CSR when the order
 * changes.  TG_ERR_INVALID_ARGUMENT for an unknown kind. */
tg_status tg_set_order(tg_graph* g, int32_t kind, uint64_t seed);
/* Orient by a caller's OrderRank (order.hpp:31-35): precedes(u, v) iff
 * rank[u] < rank[v]; rank = n entries (host or device), a permutation of
 * [0, n) (checked for host input; TG_ERR_INVALID_ARGUMENT otherwise).  The
 * two-argument effective_adjacency(g, order) (effective.hpp:37-52) is
 * tg_set_order_rank + tg_effective_adjacency. */
tg_status tg_set_order_rank(tg_graph* g, const uint32_t* rank);
/* coreness(g) (order.hpp:39-83): core numbers, n entries (host). */
tg_status tg_coreness(tg_graph* g, uint64_t* core);
/* compute_order(g, <current order>).rank (n entries). */
tg_status tg_compute_order(tg_graph* g, uint32_t* rank);
/* effective_adjacency(g, <current order>): offsets (n+1) and lists (m),
 * either may be NULL.  Builds and caches the oriented CSR on the device. */
tg_status tg_effective_adjacency(tg_graph* g, uint64_t* offsets, uint32_t* eff);
/* ordering_cost(g, <current order>) (sequential.hpp:95-104) = W. */
tg_status tg_ordering_cost(tg_graph* g, uint64_t* cost);

/* ---- EffectiveAdjacency as a value (effective.hpp:17-35) ---- */

/* EffectiveAdjacency(offsets, eff) (effective.hpp:18-20) adopted on
 * `device`: offsets n+1, entries offsets[n]; each list ID-sorted, ids < n
 * (checked for host input).  The handle owns the device copy. */
typedef struct tg_eff tg_eff;
tg_status tg_eff_from_csr(int device, uint64_t n, const uint64_t* offsets,
                          const uint32_t* entries, tg_eff** out);
tg_status tg_eff_free(tg_eff* e);
/* count_node_iterator_n(eff, sink) (sequential.hpp:74-91) over an adopted
 * EffectiveAdjacency.  total: the count.  tally (n, host or device, may be
 * NULL): NodeTallySink counts (sequential.hpp:24-33).  triples (3*capacity
 * uint32, host or device, may be NULL): every triangle once, either
 * normalised ascending (raw = 0, ListSink, sequential.hpp:36-46) or as the
 * sink call's (v, u, w) -- apex v, u in N_v, w in N_v cap N_u (raw = 1) --
 * in unspecified order; sorting raw triples by (v, u, w) gives the
 * reference's emission order.  *num_triangles = total; TG_ERR_CAPACITY when
 * capacity < total. */
tg_status tg_eff_count(tg_eff* e, uint64_t* total, uint64_t* tally, uint32_t* triples,
                       uint64_t capacity, int32_t raw, uint64_t* num_triangles);

/* ---- partitioning (partition.hpp:45-141) ---- */

/* node_costs(g, eff, kind): f (n) and inclusive prefix (n); either may be NULL. */
tg_status tg_node_costs(tg_graph* g, int32_t kind, uint64_t* f, uint64_t* prefix);
/* compute_boundaries(node_costs(kind), p): p+1 boundaries. */
tg_status tg_compute_boundaries(tg_graph* g, int32_t kind, uint64_t p, uint32_t* boundaries);

/* ---- counting (sequential.hpp:74-91, engines.hpp:335-435) ---- */

/* count_node_iterator_n(effective_adjacency(g, <current order>)). */
tg_status tg_count(tg_graph* g, uint64_t* total);

/* count_node_iterator_pp(g, <current order>, use_intersection)
 * (sequential.hpp:48-70): the paper's NodeIterator++ baseline on the
 * symmetric adjacency -- for every v < u < w in the order with u, w in
 * adj(v), test (u, w).  Same count as tg_count; both reference variants
 * (binary-search membership / merge intersection) compute the same sum, and
 * the device runs membership searches for either. */
tg_status tg_count_node_iterator_pp(tg_graph* g, int32_t use_intersection, uint64_t* total);

/* run_engine(g, cfg).  per_rank: ranks entries (1 for SEQ); boundaries_out:
 * ranks+1 entries (may be NULL); node_counts: n entries, filled when
 * cfg->track_nodes; triangles: 3*capacity uint32, filled (ascending ids per
 * triple, unspecified triple order) when cfg->collect_triangles, with
 * *num_triangles = total; TG_ERR_CAPACITY if capacity < total.  A device
 * `triangles` buffer with capacity >= total is written in place by the
 * listing kernels (no staging copy). */
tg_status tg_run_engine(tg_graph* g, const tg_config* cfg, uint64_t* total,
                        tg_rank_stats* per_rank, uint32_t* boundaries_out,
                        uint64_t* node_counts, uint32_t* triangles, uint64_t capacity,
                        uint64_t* num_triangles);

/* clustering_coefficients(g, cfg) (engines.hpp:422-435): T_v (n) and C_v (n). */
tg_status tg_clustering_coefficients(tg_graph* g, const tg_config* cfg,
                                     uint64_t* triangles_per_node, double* coefficient);

/* ---- approximate counting and per-edge analytics ---- */

/* approx_count(g, p, engine, q, seed, boundaries, cost) (engines.hpp:440-457):
 * sparsify-then-count estimate T' / q^3, PerPartition draws for AOP and
 * Global draws otherwise, under the degree order (the EngineConfig it builds
 * keeps the default order).  boundaries: optional (p+1 entries, host). */
tg_status tg_approx_count(tg_graph* g, uint64_t p, int32_t engine, double q, uint64_t seed,
                          const uint32_t* boundaries, int32_t cost, double* estimate);
/* per_edge_triangle_counts(g, eff) (sequential.hpp:108-122): t_e for every
 * edge in Graph::edges() order (u < v, u then v ascending; graph.hpp:40-46);
 * te has num_edges entries (host or device memory). */
tg_status tg_per_edge_triangle_counts(tg_graph* g, uint64_t* te);
/* variance_report(g, plan, q) (sparsify.hpp:113-155; degree order, :123-124): out3 = {T, k, k'},
 * var2 = {var, var'} for the 1/q^3-scaled estimator under the plan given by
 * `boundaries` (p+1 entries, host). */
tg_status tg_variance_report(tg_graph* g, const uint32_t* boundaries, uint64_t p, double q,
                             uint64_t* out3, double* var2);

/* ---- edge-list text (io.hpp:24-64) ---- */

/* parse_edge_list(text) on `device`: pairs (2*capacity uint32, host or
 * device) get the (u, v) edges in file order, *num_pairs their count;
 * TG_ERR_CAPACITY if capacity is smaller (count reported); pairs = NULL
 * queries the count.  Errors as tg_graph_from_text. */
tg_status tg_parse_edge_list(int device, const char* text, uint64_t len, uint32_t* pairs,
                             uint64_t capacity, uint64_t* num_pairs, uint64_t* err_line);
/* write_edge_list(g): "u v\n" per edge with u < v (io.hpp:52-64) into out
 * (capacity bytes, host or device); *len = the full length;
 * TG_ERR_CAPACITY if capacity < *len.  out may be NULL to query the size. */
tg_status tg_write_edge_list(tg_graph* g, char* out, uint64_t capacity, uint64_t* len);

/* ---- device-resident hot path (bench / multi-process drivers) ---- */

/* One pass of the hot path on the current stream without a host sync:
 * orientation (effective_adjacency) + NodeIteratorN count over all apexes.
 * The count lands in *d_total (device memory, uint64).  Stream-ordered. */
tg_status tg_step_device(tg_graph* g, uint64_t* d_total);
/* The orientation half of the step alone (effective_adjacency, rebuilt). */
tg_status tg_orient_device(tg_graph* g);
/* Kernel-only variant: count over the cached oriented CSR (no re-orientation). */
tg_status tg_count_device(tg_graph* g, uint64_t* d_total);

/* Rank-local work for one process per GPU (engines.hpp:38-54, 60-76,
 * 146-198).  `boundaries` has p+1 entries (host).  Each call is
 * stream-ordered and returns without a host sync unless noted. */
/* AOP rank body: count triangles whose apex lies in core `rank`. */
tg_status tg_aop_rank_device(tg_graph* g, const uint32_t* boundaries, uint64_t p,
                             uint64_t rank, uint64_t* d_total);
/* The AOP rank body with the reference's sinks (engines.hpp:303-321
 * RankSink): d_tally (n uint64, device, accumulated; may be NULL) gets
 * T_v += 1 at the three corners of every triangle whose apex is in core
 * `rank`; d_tri (3*capacity uint32, device; may be NULL) the triples
 * (ascending ids) at positions claimed from *d_cursor (device uint64). */
tg_status tg_aop_rank_sinks_device(tg_graph* g, const uint32_t* boundaries, uint64_t p,
                                   uint64_t rank, uint64_t* d_total, uint64_t* d_tally,
                                   uint32_t* d_tri, uint64_t capacity, uint64_t* d_cursor);
/* clustering coefficients (engines.hpp:258-267) of device tallies (n uint64)
 * into d_cc (n fp64, device), IEEE-rounded like tg_clustering_coefficients. */
tg_status tg_cc_from_tally_device(tg_graph* g, const uint64_t* d_tally, double* d_cc);
/* Surrogate pack (engines.hpp:173-187): sizes first (host sync).
 * msgs_per_dest / words_per_dest: p entries each (host). */
tg_status tg_surrogate_pack_sizes(tg_graph* g, const uint32_t* boundaries, uint64_t p,
                                  uint64_t rank, uint64_t* msgs_per_dest,
                                  uint64_t* words_per_dest);
/* Writes headers (2 uint32 per message: v, len) and list data, destination-
 * major, into device buffers sized from tg_surrogate_pack_sizes. */
tg_status tg_surrogate_pack_device(tg_graph* g, const uint32_t* boundaries, uint64_t p,
                                   uint64_t rank, uint32_t* d_hdr, uint32_t* d_data);
/* Local intersections of core `rank` plus SurrogateCount over received
 * messages (d_hdr: 2*num_msgs, d_data: the lists, concatenated in header
 * order).  Adds to *d_total. */
tg_status tg_surrogate_count_device(tg_graph* g, const uint32_t* boundaries, uint64_t p,
                                    uint64_t rank, const uint32_t* d_hdr, uint64_t num_msgs,
                                    const uint32_t* d_data, uint64_t* d_total);

/* ---- across GPUs: one rank per GPU (comm.cu) ----
 *
 * The engines with their real exchange (engines.hpp:38-76, 146-198,
 * 211-268).  Every rank holds rows [lo, hi) of the symmetric CSR (the ranks'
 * ranges tile [0, n) in rank order) and the global degrees -- a graph from
 * tg_graph_from_rows -- or the whole graph (then its rows are an equal-
 * orientation-cost split: adjacency entries + 32 per row).  Each rank orients only its rows.  One C++ host
 * can drive N devices: create the communicators, then call each rank's
 * entry points from its own host thread.  NCCL is loaded at run time. */
typedef struct tg_comm tg_comm;
/* ncclGetUniqueId: 128 bytes for tg_comm_init, made on one rank and
 * shared with the others by the caller. */
tg_status tg_comm_unique_id(void* id128);
/* ncclCommInitRank on `device`. */
tg_status tg_comm_init(int device, int nranks, int rank, const void* id128, tg_comm** out);
/* nranks in-process ranks (one host thread each) on devices[r]: the
 * exchange is host-orchestrated device copies (tests; no NCCL needed). */
tg_status tg_comm_init_local(int nranks, const int* devices, tg_comm** comms);
tg_status tg_comm_free(tg_comm* c);
tg_status tg_comm_info(tg_comm* c, int32_t* nranks, int32_t* rank);
/* A rank-local Graph: rows [row_lo, row_hi) of the symmetric CSR of an
 * n-vertex graph (offsets: row_hi - row_lo + 1 entries, any base; adj: the
 * rows' entries) and every vertex's degree (n, host).  Counted only through
 * the tg_*_comm entry points (it cannot orient the rows it does not hold). */
tg_status tg_graph_from_rows(int device, uint64_t n, uint32_t row_lo, uint32_t row_hi,
                             const uint64_t* offsets, const uint32_t* adj,
                             const uint32_t* degrees, tg_graph** out);
/* run_engine (engines.hpp:335-418) across the communicator, Aop,
 * AnopDirect or AnopSurrogate, counts (no sinks, no sparsification, degree
 * order):
 *  Aop       -- own rows oriented, the oriented rows gathered (one broadcast
 *               per rank), the cfg->cost plan from the gathered costs, the
 *               rank's core counted, one all-reduce of T;
 *  Surrogate -- own rows oriented, list lengths gathered, the plan from
 *               distributed costs, oriented rows moved to their core owner
 *               (one all-to-allv: Σ stored = m), the (v, N_v) messages
 *               exchanged (all-to-allv), SurrogateCount;
 *  Direct    -- (engines.hpp:80-141) the same core partitions; every
 *               off-core pair (v, u) is one request to owner(u) and one reply
 *               carrying N_u (no caching, as in the reference), batched into
 *               three all-to-allv (ids, reply lengths, reply lists); the
 *               requester intersects N_v with each reply.  data_sent /
 *               data_recv = requests + replies.  Refused when a rank's reply
 *               lists would not fit its device.
 * Every rank returns the same total, per_rank (nranks) and boundaries
 * (nranks+1); cfg->ranks must be 0 or nranks; cfg->boundaries overrides
 * the plan. */
tg_status tg_run_engine_comm(tg_graph* g, tg_comm* c, const tg_config* cfg, uint64_t* total,
                             tg_rank_stats* per_rank, uint32_t* boundaries_out);
/* effective_adjacency for rows [row_lo, row_hi) alone (one rank's share of
 * the orientation; *entries = its oriented entries).  Used by the per-rank
 * projections (tools/scaling_projection.py). */
tg_status tg_orient_rows_device(tg_graph* g, uint32_t row_lo, uint32_t row_hi, uint64_t* entries);
/* One AOP step (the bench's N-GPU step): own rows oriented + gathered, the
 * rank's core of `boundaries` (nranks+1) counted, T all-reduced into
 * *d_total (device u64) on every rank. */
tg_status tg_aop_step_comm(tg_graph* g, tg_comm* c, const uint32_t* boundaries, uint64_t* d_total);
/* clustering_coefficients (engines.hpp:422-435) across the communicator:
 * AOP tallies of the rank's apexes at all three corners, each core range
 * summed at its owner (aggregate_clustering, engines.hpp:229-254), C_v
 * there.  tally_core / cc_core: this rank's core [b_r, b_r+1) (host or
 * device); boundaries_out: nranks+1. */
tg_status tg_clustering_comm(tg_graph* g, tg_comm* c, const tg_config* cfg,
                             uint32_t* boundaries_out, uint64_t* tally_core, double* cc_core);

/* ---- diagnostics ---- */
const char* tg_last_error(void);
const char* tg_status_string(tg_status s);
/* Number of library kernels launched so far in this process. */
uint64_t tg_kernel_launches(void);
/* Test hook: shared-memory capacity (entries) of the CTA-path apex staging;
 * lists longer than this are searched in global memory.  0 = default. */
void tg_debug_set_block_cap(uint32_t entries);
/* Test hook: adjacency entries per streamed chunk of tg_count_from_csr
 * (0 = default 2^24; at most 64 chunks). */
void tg_debug_set_chunk_entries(uint64_t entries);
/* Test hook: intersection kernels, 0 = automatic (apex groups when the mean
 * oriented list is <= 16 entries, else one apex per warp iteration; 16-byte
 * quad loads when list indices fit 32 bits), 1 = scalar one-apex-per-warp and
 * scalar CTA path, 2 = quad apex groups, 3 = quad one-apex-per-warp, 4 =
 * scalar apex groups.  All exact. */
void tg_debug_set_warp_variant(int32_t variant);
/* Test hook: the bitmap CTA path (apexes whose rank window, n - rank(v) - 1,
 * fits cap_bits of shared memory; ctab.cuh).  mode 0 = automatic (on when
 * lists longer than 64 hold > 1% of the oriented entries), 1 = on, 2 = off;
 * cap_bits 0 = 2^19.  All exact. */
void tg_debug_set_rank_bitmap(int32_t mode, uint32_t cap_bits);
/* Test hook: the large-graph code paths on small graphs.  orient_mode: 0
 * auto, 1 compact count/scan/fill orientation (taken above 2^34 list
 * slots), +4 = 1-byte degree codes as orientation keys (taken above 32M
 * vertices), +8 = 4-bit endpoint-quantile degree codes (taken above 64M
 * vertices); force_wide: 64-bit element indices in the scalar
 * intersection kernels (taken above 2^32 list slots).  All exact. */
void tg_debug_set_paths(int32_t orient_mode, int32_t force_wide);
/* Test hook: the id-window encoding of the count (window.cu): 0 = automatic
 * (when <= 10% of the oriented entries lie outside their row's 64-id
 * window), 1 = always, 2 = never.  All exact. */
void tg_debug_set_window(int32_t mode);
/* Test hook: the slab layout of the oriented lists (each list's first 32
 * entries in its own 128-byte-aligned slab, so the intersection reads a list
 * as one DRAM line without a descriptor; slab.cuh): 0 = automatic (mean
 * list > 16, <= 2% of the entries in lists longer than a slab), 1 = always,
 * 2 = never.  All exact. */
void tg_debug_set_slab(int32_t mode);
/* Device-side time (ms) of the last intersection pass (CUDA events on the
 * launching stream); 0 if none. */
double tg_last_intersect_ms(tg_graph* g);

/* ---- synthetic inputs (host harness; BASELINE.json configs) ----
 * Each returns a malloc'ed interleaved pair array (free with tg_free_host). */
/* io.hpp:129-162 gen_pa(n, d, seed), bit-identical edge stream. */
tg_status tg_gen_pa(uint64_t n, uint64_t d, uint64_t seed, uint32_t** pairs, uint64_t* num_pairs);
/* io.hpp:85-123 gen_gnp(n, d, seed), bit-identical edge stream. */
tg_status tg_gen_gnp(uint64_t n, double d, uint64_t seed, uint32_t** pairs, uint64_t* num_pairs);
/* G(n, m): m distinct non-loop pairs drawn uniformly (config 1). */
tg_status tg_gen_gnm(uint64_t n, uint64_t m, uint64_t seed, uint32_t** pairs, uint64_t* num_pairs);
/* R-MAT scale s, edge factor ef, (a,b,c) with d = 1-a-b-c (config 3). */
tg_status tg_gen_rmat(uint32_t scale, uint64_t edge_factor, double a, double b, double c,
                      uint64_t seed, uint32_t** pairs, uint64_t* num_pairs);
/* Watts-Strogatz ring n, k neighbours (k/2 per side), rewiring beta (config 4). */
tg_status tg_gen_ws(uint64_t n, uint64_t k, double beta, uint64_t seed, uint32_t** pairs,
                    uint64_t* num_pairs);
void tg_free_host(void* p);
/* The same R-MAT / Watts-Strogatz streams generated ON THE DEVICE (one
 * thread per xoshiro chunk, bit-identical pairs) and built into a graph
 * there (n = 2^scale / n): no host edge list. */
tg_status tg_graph_from_rmat(int device, uint32_t scale, uint64_t edge_factor, double a, double b,
                             double c, uint64_t seed, tg_graph** out);
tg_status tg_graph_from_ws(int device, uint64_t n, uint64_t k, double beta, uint64_t seed,
                           tg_graph** out);

#ifdef __cplusplus
}
#endif
#endif /* TRIGRAPH_B200_H */
