/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference `trigraph` hot path
 * (/root/reference/proj/include/trigraph/*.hpp), used as the parity checker
 * for the B200 library.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product path
 * (paper_1706_05151_b200/) never links or calls anything in this directory.
 *
 * Pinning: the restatement is checked against the reference itself, built
 * from its own headers into oracle/_ref/ (see oracle/Makefile, ref_shim.cpp),
 * and against the reference tests' golden vectors (tests/golden/).
 *
 * Conventions: NodeId = uint32_t, offsets are uint64_t (reference size_t),
 * counters are uint64_t (reference std::uint64_t).
 */
#ifndef TG_ORACLE_H
#define TG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* graph.hpp:58-85 build_graph.  pairs = E (u,v) pairs, interleaved.
 * Returns n; *off_out (n+1) and *adj_out (2m) are malloc'ed (orc_free). */
uint64_t orc_build_graph(const uint32_t* pairs, uint64_t E, uint64_t n_override,
                         uint64_t** off_out, uint32_t** adj_out);
void orc_free(void* p);

/* order.hpp:95-104 compute_order(ByDegree): rank[v] = position of v in the
 * (degree, id) ascending sort. */
void orc_degree_rank(uint64_t n, const uint64_t* off, uint32_t* rank);

/* order.hpp:19 OrderKind::Tag, in declaration order. */
enum { ORC_ORDER_BY_ID = 0, ORC_ORDER_BY_DEGREE, ORC_ORDER_BY_RANDOM, ORC_ORDER_BY_CORENESS };

/* order.hpp:39-83 coreness (core numbers, n entries). */
void orc_coreness(uint64_t n, const uint64_t* off, const uint32_t* adj, uint64_t* core);

/* order.hpp:85-128 compute_order(g, OrderKind{kind, seed}).rank.  Returns 0,
 * or -1 for an unknown kind. */
int orc_compute_order(uint64_t n, const uint64_t* off, const uint32_t* adj, int kind,
                      uint64_t seed, uint32_t* rank);

/* effective.hpp:37-52.  eoff has n+1 entries (caller-allocated);
 * *eff_out (m entries) malloc'ed.  Returns m. */
uint64_t orc_effective(uint64_t n, const uint64_t* off, const uint32_t* adj,
                       const uint32_t* rank, uint64_t* eoff, uint32_t** eff_out);

/* sequential.hpp:74-91 count_node_iterator_n, with NodeTallySink
 * (sequential.hpp:24-33, tally may be NULL) and ListSink (sequential.hpp:36-46,
 * tri may be NULL; at most tri_cap triples written, normalised ascending). */
uint64_t orc_count(uint64_t n, const uint64_t* eoff, const uint32_t* eff,
                   uint64_t* tally, uint32_t* tri, uint64_t tri_cap);

/* count_node_iterator_n restricted to apexes [vlo, vhi). */
uint64_t orc_count_range(uint64_t n, const uint64_t* eoff, const uint32_t* eff,
                         uint64_t vlo, uint64_t vhi);

/* sequential.hpp:95-104 ordering_cost under the order given by rank. */
uint64_t orc_ordering_cost(uint64_t n, const uint64_t* off, const uint32_t* adj,
                           const uint32_t* rank);

/* partition.hpp:18 CostKind, in declaration order. */
enum { ORC_COST_N = 0, ORC_COST_D, ORC_COST_DH, ORC_COST_DDH, ORC_COST_DH2,
       ORC_COST_DPD, ORC_COST_NOV };

/* partition.hpp:45-91 node_costs (EffectiveOnly DPD variant). */
void orc_node_costs(uint64_t n, const uint64_t* off, const uint32_t* adj,
                    const uint64_t* eoff, const uint32_t* eff, int kind,
                    uint64_t* f, uint64_t* prefix);

/* partition.hpp:116-141 compute_boundaries; b has p+1 entries.
 * Returns 0, or -1 when p == 0 (reference: std::invalid_argument). */
int orc_compute_boundaries(const uint64_t* prefix, uint64_t n, uint64_t p,
                           uint32_t* b);

/* partition.hpp:106-109 PartitionPlan::owner. */
uint64_t orc_owner(const uint32_t* b, uint64_t p, uint32_t v);

/* engines.hpp:24 EngineKind, in declaration order. */
enum { ORC_ENGINE_SEQ = 0, ORC_ENGINE_AOP, ORC_ENGINE_ANOP_DIRECT,
       ORC_ENGINE_ANOP_SURROGATE };

/* engines.hpp:335-418 run_engine (degree order).  boundaries_in may be NULL
 * (cost-based plan).  boundaries_out has p+1 entries; tri/sent/recv/stored
 * have p entries each (stored = partition stored_entries()).  tally (n) and
 * list (3*list_cap) may be NULL.  Returns the global total, or UINT64_MAX on
 * invalid arguments (ranks == 0). */
uint64_t orc_run_engine(uint64_t n, const uint64_t* off, const uint32_t* adj,
                        int engine, uint64_t p, int cost,
                        const uint32_t* boundaries_in, uint32_t* boundaries_out,
                        uint64_t* tri, uint64_t* sent, uint64_t* recv,
                        uint64_t* stored, uint64_t* tally, uint32_t* list,
                        uint64_t list_cap);

/* orc_run_engine with cfg.sparsify (engines.hpp:279, sparsify.hpp):
 * smode 0 = none, 1 = Global, 2 = PerPartition; q in (0, 1]. */
uint64_t orc_run_engine_ex(uint64_t n, const uint64_t* off, const uint32_t* adj,
                           int engine, uint64_t p, int cost,
                           const uint32_t* boundaries_in, uint32_t* boundaries_out,
                           uint64_t* tri, uint64_t* sent, uint64_t* recv,
                           uint64_t* stored, uint64_t* tally, uint32_t* list,
                           uint64_t list_cap, int smode, double q, uint64_t seed);

/* orc_run_engine_ex under EngineConfig::order = OrderKind{order, order_seed}
 * (engines.hpp:274, :341).  UINT64_MAX also for an unknown order. */
uint64_t orc_run_engine_ord(uint64_t n, const uint64_t* off, const uint32_t* adj,
                            int engine, uint64_t p, int cost,
                            const uint32_t* boundaries_in, uint32_t* boundaries_out,
                            uint64_t* tri, uint64_t* sent, uint64_t* recv,
                            uint64_t* stored, uint64_t* tally, uint32_t* list,
                            uint64_t list_cap, int smode, double q, uint64_t seed,
                            int order, uint64_t order_seed);

/* sparsify.hpp:58-62 keep_entry with a resolved rank key. */
int orc_keep_entry(double q, uint64_t seed, uint64_t rank_key, uint32_t v, uint32_t u);

/* engines.hpp:440-457 approx_count (T' / q^3). */
double orc_approx_count(uint64_t n, const uint64_t* off, const uint32_t* adj, uint64_t p,
                        int engine, double q, uint64_t seed, const uint32_t* boundaries,
                        int cost);

/* sequential.hpp:108-122 per_edge_triangle_counts in Graph::edges() order. */
void orc_per_edge_counts(uint64_t n, const uint64_t* off, const uint32_t* adj, uint64_t* te);

/* sparsify.hpp:113-155 variance_report: out3 = {T, k, k'}, var2 = {var, var'}. */
void orc_variance_report(uint64_t n, const uint64_t* off, const uint32_t* adj,
                         const uint32_t* b, uint64_t p, double q, uint64_t* out3,
                         double* var2);

/* io.hpp:24-50 parse_edge_list.  Returns the pair count (at most cap pairs
 * written, interleaved), or UINT64_MAX on ParseError: *err_line (1-based),
 * *err_kind 1 = "expected two integer tokens", 2 = "trailing token" (token
 * bytes [*tok_b, *tok_e) of text). */
uint64_t orc_parse_edge_list(const char* text, uint64_t len, uint32_t* pairs, uint64_t cap,
                             uint64_t* err_line, int* err_kind, uint64_t* tok_b,
                             uint64_t* tok_e);

/* io.hpp:52-64 write_edge_list; writes up to cap bytes, returns the length. */
uint64_t orc_write_edge_list(uint64_t n, const uint64_t* off, const uint32_t* adj, char* out,
                             uint64_t cap);

/* engines.hpp:422-435 clustering coefficient formula. */
void orc_cc(uint64_t n, const uint64_t* off, const uint64_t* tally, double* c);

/* proj/tests/oracles.hpp:49-57 random_graph(n, density, seed): writes the
 * accepted (u,v) pairs into out (2*cap uint32); returns the pair count
 * (which may exceed cap, in which case only cap pairs were written). */
uint64_t orc_random_graph_pairs(uint64_t n, double density, uint64_t seed,
                                uint32_t* out, uint64_t cap);

/* std::mt19937_64 restated (used by the fixture generators). */
typedef struct { uint64_t mt[312]; int mti; } orc_mt64;
void orc_mt64_seed(orc_mt64* s, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* s);


/* ---- full-size oracle (fullsize.c): the configs' generators and the
 * memory-lean multi-threaded pipeline used for the C3/C4/C5 goldens ---- */

/* io.hpp:129-162 gen_pa; harness G(n,m) / R-MAT / Watts-Strogatz (the
 * workload definitions of configs 1, 3, 4).  Return the pair count
 * (*pairs_out malloc'ed, E interleaved pairs) or UINT64_MAX on bad args. */
uint64_t orc_gen_pa(uint64_t n, uint64_t d, uint64_t seed, uint32_t** pairs_out);
uint64_t orc_gen_gnm(uint64_t n, uint64_t m, uint64_t seed, uint32_t** pairs_out);
uint64_t orc_gen_rmat(uint32_t scale, uint64_t edge_factor, double a, double b, double c,
                      uint64_t seed, int threads, uint32_t** pairs_out);
uint64_t orc_gen_ws(uint64_t n, uint64_t k, double beta, uint64_t seed, int threads,
                    uint32_t** pairs_out);

/* graph.hpp:58-85 build_graph; CONSUMES pairs (freed). Returns n. */
uint64_t orc_build_graph_lean(uint32_t* pairs, uint64_t E, uint64_t n_override, int threads,
                              uint64_t** off_out, uint32_t** adj_out);

/* effective.hpp:37-52 on `threads` threads; eoff (n+1) caller-allocated. */
uint64_t orc_effective_mt(uint64_t n, const uint64_t* off, const uint32_t* adj,
                          const uint32_t* rank, int threads, uint64_t* eoff, uint32_t** eff_out);

/* Digest term of one normalised triple a < b < c (ListSink order,
 * sequential.hpp:39-44): mix(mix(mix(a) ^ b) ^ c), mix = SplitMix64
 * finaliser (sparsify.hpp:37-45).  A listing's digest is
 * (sum h, sum mix(h)) mod 2^64. */
uint64_t orc_tri_hash(uint32_t a, uint32_t b, uint32_t c);

/* count_node_iterator_n on `threads` threads; optional tally[n] (T_v),
 * apex_tri[p] / mid_tri[p] (triangles by owner of apex / middle vertex under
 * plan b: AOP / ANOP-surrogate per-rank counts), digest2[2] (listing). */
uint64_t orc_count_full(uint64_t n, const uint64_t* eoff, const uint32_t* eff,
                        const uint32_t* b, uint64_t p, int threads, uint64_t* tally,
                        uint64_t* apex_tri, uint64_t* mid_tri, uint64_t* digest2);

/* engines.hpp:173-187 surrogate NeighborList messages per rank. */
void orc_surrogate_messages(uint64_t n, const uint64_t* eoff, const uint32_t* eff,
                            const uint32_t* b, uint64_t p, uint64_t* sent, uint64_t* recv);

#ifdef __cplusplus
}
#endif
#endif
