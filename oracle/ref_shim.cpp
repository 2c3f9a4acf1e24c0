// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/trigraph/*.hpp and proj/tests/oracles.hpp),
// compiled by oracle/Makefile into oracle/_ref/libtrigraph_ref.so.  Nothing
// from the reference is copied: the headers are used in place through -I.
//
// Uses: (1) pinning the C restatement in oracle.c and the B200 library
// against the reference itself; (2) generating tests/golden/ fixtures;
// (3) the CPU baseline / `bench.py --impl reference` arm, which times the
// reference's own NodeIteratorN and AOP rank bodies on the host cores.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <optional>
#include <stdexcept>
#include <thread>
#include <vector>

#include "oracles.hpp"
#include "trigraph/trigraph.hpp"

using namespace trigraph;

namespace {

struct RefGraph {
  Graph g;
  std::optional<OrderRank> order;
  std::optional<EffectiveAdjacency> eff;

  const EffectiveAdjacency& effective() {
    if (!eff) {
      order = compute_order(g, OrderKind::by_degree());
      eff = effective_adjacency(g, *order);
    }
    return *eff;
  }
};

RefGraph* wrap(Graph g) {
  auto* r = new RefGraph;
  r->g = std::move(g);
  return r;
}

double now_s() {
  return std::chrono::duration<double>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

}  // namespace

extern "C" {

void* ref_graph_from_pairs(const uint32_t* pairs, uint64_t E, uint64_t n_override) {
  std::vector<std::pair<NodeId, NodeId>> e(E);
  for (uint64_t i = 0; i < E; ++i) e[i] = {pairs[2 * i], pairs[2 * i + 1]};
  return wrap(build_graph(e, n_override));
}

void* ref_graph_from_csr(uint64_t n, const uint64_t* off, const uint32_t* adj) {
  std::vector<std::size_t> o(off, off + n + 1);
  std::vector<NodeId> a(adj, adj + off[n]);
  return wrap(Graph(n, std::move(o), std::move(a)));
}

void* ref_random_graph(uint64_t n, double density, uint64_t seed) {
  return wrap(oracles::random_graph(n, density, seed));
}
void* ref_complete(uint64_t n) { return wrap(oracles::complete(n)); }
void* ref_wheel(uint64_t rim) { return wrap(oracles::wheel(rim)); }
void* ref_complete_bipartite(uint64_t a, uint64_t b) {
  return wrap(oracles::complete_bipartite(a, b));
}
void* ref_g5() { return wrap(oracles::g5()); }
void* ref_gen_pa(uint64_t n, uint64_t d, uint64_t seed) { return wrap(gen_pa(n, d, seed)); }
void* ref_gen_gnp(uint64_t n, double d, uint64_t seed) { return wrap(gen_gnp(n, d, seed)); }

void ref_graph_free(void* h) { delete static_cast<RefGraph*>(h); }

uint64_t ref_num_nodes(void* h) { return static_cast<RefGraph*>(h)->g.num_nodes(); }
uint64_t ref_num_edges(void* h) { return static_cast<RefGraph*>(h)->g.num_edges(); }

void ref_graph_csr(void* h, uint64_t* off, uint32_t* adj) {
  const Graph& g = static_cast<RefGraph*>(h)->g;
  uint64_t k = 0;
  off[0] = 0;
  for (NodeId v = 0; v < g.num_nodes(); ++v) {
    for (NodeId u : g.neighbors(v)) adj[k++] = u;
    off[v + 1] = k;
  }
}

void ref_degree_rank(void* h, uint32_t* rank) {
  auto ord = compute_order(static_cast<RefGraph*>(h)->g, OrderKind::by_degree());
  std::memcpy(rank, ord.rank.data(), ord.rank.size() * sizeof(uint32_t));
}

OrderKind order_kind(int kind, uint64_t seed) {
  switch (kind) {
    case 0: return OrderKind::by_id();
    case 1: return OrderKind::by_degree();
    case 2: return OrderKind::by_random(seed);
    default: return OrderKind::by_coreness();
  }
}

// compute_order(g, OrderKind{kind, seed}) (order.hpp:85-128).
void ref_compute_order(void* h, int kind, uint64_t seed, uint32_t* rank) {
  auto ord = compute_order(static_cast<RefGraph*>(h)->g, order_kind(kind, seed));
  std::memcpy(rank, ord.rank.data(), ord.rank.size() * sizeof(uint32_t));
}

// coreness(g) (order.hpp:39-83).
void ref_coreness(void* h, uint64_t* core) {
  auto c = coreness(static_cast<RefGraph*>(h)->g);
  for (std::size_t v = 0; v < c.size(); ++v) core[v] = c[v];
}

// effective_adjacency(g, compute_order(g, kind)) + count_node_iterator_n +
// ordering_cost under that order.  eoff (n+1) / eff (m) may be NULL.
uint64_t ref_effective_order(void* h, int kind, uint64_t seed, uint64_t* eoff, uint32_t* eff,
                             uint64_t* count, uint64_t* cost) {
  const Graph& g = static_cast<RefGraph*>(h)->g;
  auto ord = compute_order(g, order_kind(kind, seed));
  auto e = effective_adjacency(g, ord);
  uint64_t k = 0;
  if (eoff) eoff[0] = 0;
  for (NodeId v = 0; v < e.num_nodes(); ++v) {
    for (NodeId u : e.eff(v)) {
      if (eff) eff[k] = u;
      ++k;
    }
    if (eoff) eoff[v + 1] = k;
  }
  if (count) *count = count_node_iterator_n(e);
  if (cost) *cost = ordering_cost(g, ord);
  return k;
}

uint64_t ref_effective(void* h, uint64_t* eoff, uint32_t* eff) {
  const auto& e = static_cast<RefGraph*>(h)->effective();
  const uint64_t n = e.num_nodes();
  uint64_t k = 0;
  if (eoff) eoff[0] = 0;
  for (NodeId v = 0; v < n; ++v) {
    for (NodeId u : e.eff(v)) {
      if (eff) eff[k] = u;
      ++k;
    }
    if (eoff) eoff[v + 1] = k;
  }
  return k;
}

uint64_t ref_count(void* h) {
  return count_node_iterator_n(static_cast<RefGraph*>(h)->effective());
}

uint64_t ref_ordering_cost(void* h) {
  const Graph& g = static_cast<RefGraph*>(h)->g;
  return ordering_cost(g, compute_order(g, OrderKind::by_degree()));
}

void ref_node_costs(void* h, int kind, uint64_t* f, uint64_t* prefix) {
  auto* r = static_cast<RefGraph*>(h);
  auto c = node_costs(r->g, r->effective(), static_cast<CostKind>(kind));
  std::memcpy(f, c.f.data(), c.f.size() * sizeof(uint64_t));
  std::memcpy(prefix, c.prefix.data(), c.prefix.size() * sizeof(uint64_t));
}

int ref_compute_boundaries(const uint64_t* f, uint64_t n, uint64_t p, uint32_t* b) {
  CostVector c;
  c.f.assign(f, f + n);
  c.prefix.resize(n);
  uint64_t acc = 0;
  for (uint64_t i = 0; i < n; ++i) c.prefix[i] = (acc += f[i]);
  try {
    auto plan = compute_boundaries(c, p);
    std::memcpy(b, plan.boundaries.data(), plan.boundaries.size() * sizeof(uint32_t));
    return 0;
  } catch (const std::invalid_argument&) {
    return -1;
  }
}

uint64_t ref_overlap_stored(void* h, const uint32_t* b, uint64_t p, uint64_t i) {
  auto* r = static_cast<RefGraph*>(h);
  PartitionPlan plan{std::vector<NodeId>(b, b + p + 1)};
  return build_overlap_partition(r->g, r->effective(), plan, i).stored_entries();
}

// run_engine (engines.hpp:335).  tally != NULL turns on track_nodes; list !=
// NULL turns on collect_triangles (sorted ascending, up to cap triples;
// *n_listed gets the full count).  Returns total, UINT64_MAX on
// std::invalid_argument.
uint64_t ref_run_engine(void* h, int engine, uint64_t p, int cost, const uint32_t* b_in,
                        uint32_t* b_out, uint64_t* tri, uint64_t* sent, uint64_t* recv,
                        uint64_t* tally, uint32_t* list, uint64_t cap, uint64_t* n_listed,
                        int concurrent) {
  auto* r = static_cast<RefGraph*>(h);
  EngineConfig cfg;
  cfg.engine = static_cast<EngineKind>(engine);
  cfg.ranks = p;
  cfg.cost = static_cast<CostKind>(cost);
  cfg.mode = concurrent ? runtime::ExecMode::Concurrent : runtime::ExecMode::Interleaved;
  cfg.track_nodes = tally != nullptr;
  cfg.collect_triangles = list != nullptr;
  uint64_t pp = cfg.engine == EngineKind::Sequential ? 1 : p;
  if (b_in) cfg.boundaries = std::vector<NodeId>(b_in, b_in + pp + 1);
  RunReport rep;
  try {
    rep = run_engine(r->g, cfg);
  } catch (const std::invalid_argument&) {
    return UINT64_MAX;
  }
  std::memcpy(b_out, rep.boundaries.data(), rep.boundaries.size() * sizeof(uint32_t));
  for (std::size_t i = 0; i < rep.per_rank.size(); ++i) {
    tri[i] = rep.per_rank[i].triangles;
    sent[i] = rep.per_rank[i].data_sent;
    recv[i] = rep.per_rank[i].data_recv;
  }
  if (tally)
    std::memcpy(tally, rep.node_counts.data(), rep.node_counts.size() * sizeof(uint64_t));
  if (list) {
    std::sort(rep.triangles_list.begin(), rep.triangles_list.end());
    *n_listed = rep.triangles_list.size();
    for (uint64_t k = 0; k < rep.triangles_list.size() && k < cap; ++k)
      for (int c = 0; c < 3; ++c) list[3 * k + c] = rep.triangles_list[k][c];
  }
  return rep.total;
}

// parse_edge_list (io.hpp:24-50).  Returns the pair count (up to cap pairs
// written) or UINT64_MAX on ParseError, with *err_line and the message
// (what()) copied into msg (msg_cap bytes, NUL-terminated).
uint64_t ref_parse_edge_list(const char* text, uint64_t len, uint32_t* pairs, uint64_t cap,
                             uint64_t* err_line, char* msg, uint64_t msg_cap) {
  try {
    auto e = parse_edge_list(std::string_view(text, len));
    for (uint64_t k = 0; k < e.size() && k < cap; ++k) {
      pairs[2 * k] = e[k].first;
      pairs[2 * k + 1] = e[k].second;
    }
    return e.size();
  } catch (const ParseError& err) {
    *err_line = err.line;
    std::snprintf(msg, msg_cap, "%s", err.what());
    return UINT64_MAX;
  }
}

// write_edge_list (io.hpp:52-64): up to cap bytes; returns the length.
uint64_t ref_write_edge_list(void* h, char* out, uint64_t cap) {
  auto s = write_edge_list(static_cast<RefGraph*>(h)->g);
  std::memcpy(out, s.data(), std::min<uint64_t>(cap, s.size()));
  return s.size();
}

// run_engine with cfg.order = OrderKind{order, order_seed} (engines.hpp:274).
uint64_t ref_run_engine_order(void* h, int engine, uint64_t p, int cost, int order,
                              uint64_t order_seed, uint32_t* b_out, uint64_t* tri,
                              uint64_t* sent, uint64_t* recv, uint64_t* tally, uint32_t* list,
                              uint64_t cap, uint64_t* n_listed) {
  auto* r = static_cast<RefGraph*>(h);
  EngineConfig cfg;
  cfg.engine = static_cast<EngineKind>(engine);
  cfg.ranks = p;
  cfg.cost = static_cast<CostKind>(cost);
  cfg.order = order_kind(order, order_seed);
  cfg.track_nodes = tally != nullptr;
  cfg.collect_triangles = list != nullptr;
  RunReport rep;
  try {
    rep = run_engine(r->g, cfg);
  } catch (const std::invalid_argument&) {
    return UINT64_MAX;
  }
  std::memcpy(b_out, rep.boundaries.data(), rep.boundaries.size() * sizeof(uint32_t));
  for (std::size_t i = 0; i < rep.per_rank.size(); ++i) {
    tri[i] = rep.per_rank[i].triangles;
    sent[i] = rep.per_rank[i].data_sent;
    recv[i] = rep.per_rank[i].data_recv;
  }
  if (tally)
    std::memcpy(tally, rep.node_counts.data(), rep.node_counts.size() * sizeof(uint64_t));
  if (list) {
    std::sort(rep.triangles_list.begin(), rep.triangles_list.end());
    *n_listed = rep.triangles_list.size();
    for (uint64_t k = 0; k < rep.triangles_list.size() && k < cap; ++k)
      for (int c = 0; c < 3; ++c) list[3 * k + c] = rep.triangles_list[k][c];
  }
  return rep.total;
}

// run_engine with cfg.sparsify (smode 1 = Global, 2 = PerPartition)
uint64_t ref_run_engine_sparse(void* h, int engine, uint64_t p, int cost, const uint32_t* b_in,
                               int smode, double q, uint64_t seed, uint32_t* b_out, uint64_t* tri,
                               uint64_t* sent, uint64_t* recv, uint64_t* tally, uint32_t* list,
                               uint64_t cap, uint64_t* n_listed) {
  auto* r = static_cast<RefGraph*>(h);
  EngineConfig cfg;
  cfg.engine = static_cast<EngineKind>(engine);
  cfg.ranks = p;
  cfg.cost = static_cast<CostKind>(cost);
  cfg.track_nodes = tally != nullptr;
  cfg.collect_triangles = list != nullptr;
  cfg.sparsify = SparsifyConfig{q, seed,
                                smode == 2 ? SparsifyConfig::Mode::PerPartition
                                           : SparsifyConfig::Mode::Global};
  uint64_t pp = cfg.engine == EngineKind::Sequential ? 1 : p;
  if (b_in) cfg.boundaries = std::vector<NodeId>(b_in, b_in + pp + 1);
  RunReport rep;
  try {
    rep = run_engine(r->g, cfg);
  } catch (const std::invalid_argument&) {
    return UINT64_MAX;
  }
  std::memcpy(b_out, rep.boundaries.data(), rep.boundaries.size() * sizeof(uint32_t));
  for (std::size_t i = 0; i < rep.per_rank.size(); ++i) {
    tri[i] = rep.per_rank[i].triangles;
    sent[i] = rep.per_rank[i].data_sent;
    recv[i] = rep.per_rank[i].data_recv;
  }
  if (tally)
    std::memcpy(tally, rep.node_counts.data(), rep.node_counts.size() * sizeof(uint64_t));
  if (list) {
    std::sort(rep.triangles_list.begin(), rep.triangles_list.end());
    *n_listed = rep.triangles_list.size();
    for (uint64_t k = 0; k < rep.triangles_list.size() && k < cap; ++k)
      for (int c = 0; c < 3; ++c) list[3 * k + c] = rep.triangles_list[k][c];
  }
  return rep.total;
}

double ref_approx_count(void* h, uint64_t p, int engine, double q, uint64_t seed,
                        const uint32_t* b_in, int cost) {
  auto* r = static_cast<RefGraph*>(h);
  std::optional<std::vector<NodeId>> b;
  uint64_t pp = static_cast<EngineKind>(engine) == EngineKind::Sequential ? 1 : p;
  if (b_in) b = std::vector<NodeId>(b_in, b_in + pp + 1);
  try {
    return approx_count(r->g, p, static_cast<EngineKind>(engine), q, seed,
                        runtime::ExecMode::Interleaved, b, static_cast<CostKind>(cost));
  } catch (const std::invalid_argument&) {
    return std::nan("");
  }
}

int ref_keep_entry(double q, uint64_t seed, int smode, uint64_t rank, uint32_t v, uint32_t u) {
  SparsifyConfig cfg{q, seed,
                     smode == 2 ? SparsifyConfig::Mode::PerPartition : SparsifyConfig::Mode::Global};
  return keep_entry(cfg, rank, v, u) ? 1 : 0;
}

// per_edge_triangle_counts (sequential.hpp:108-122) in Graph::edges() order
uint64_t ref_per_edge_counts(void* h, uint64_t* te) {
  auto* r = static_cast<RefGraph*>(h);
  auto& eff = r->effective();
  auto m = per_edge_triangle_counts(r->g, eff);
  uint64_t k = 0;
  for (auto [u, v] : r->g.edges()) te[k++] = m.at({u, v});
  return k;
}

void ref_variance_report(void* h, const uint32_t* b, uint64_t p, double q, uint64_t* out3,
                         double* var2) {
  auto* r = static_cast<RefGraph*>(h);
  PartitionPlan plan{std::vector<NodeId>(b, b + p + 1)};
  auto rep = variance_report(r->g, plan, q);
  out3[0] = rep.triangles;
  out3[1] = rep.k;
  out3[2] = rep.k_prime;
  var2[0] = rep.var;
  var2[1] = rep.var_prime;
}

int ref_clustering(void* h, int engine, uint64_t p, int cost, uint64_t* tally, double* c) {
  auto* r = static_cast<RefGraph*>(h);
  EngineConfig cfg;
  cfg.engine = static_cast<EngineKind>(engine);
  cfg.ranks = p;
  cfg.cost = static_cast<CostKind>(cost);
  try {
    auto cc = clustering_coefficients(r->g, cfg);
    std::memcpy(tally, cc.triangles_per_node.data(), cc.triangles_per_node.size() * 8);
    std::memcpy(c, cc.coefficient.data(), cc.coefficient.size() * 8);
  } catch (const std::invalid_argument&) {
    return -1;
  }
  return 0;
}

// ---- CPU baseline legs (bench.py cpu_baseline / --impl reference) -------
//
// (i) one thread, count_node_iterator_n's loop; (ii) all host
// cores, the reference AOP through its public API with p = nproc, partition
// building and counting timed separately.  The EffectiveAdjacency is built
// once from the oracle's arrays (pinned bit-exact against
// effective_adjacency, tests/test_oracle_full.py) -- setup, untimed.

// EffectiveAdjacency(offsets, eff) (effective.hpp:18-20), copied in.
void* ref_eff_from_arrays(uint64_t n, const uint64_t* eoff, const uint32_t* eff) {
  std::vector<std::size_t> o(eoff, eoff + n + 1);
  std::vector<NodeId> e(eff, eff + eoff[n]);
  return new EffectiveAdjacency(std::move(o), std::move(e));
}
void ref_eff_free(void* h) { delete static_cast<EffectiveAdjacency*>(h); }

// (i) sequential.hpp:74-91 count_node_iterator_n over the apexes of `nr`
// ID ranges [r[2k], r[2k+1]) on the calling thread, with the reference's
// intersect_visit (intersect.hpp:15-33) and NullSink.  Returns seconds.
double ref_seq_sample(void* h, const uint32_t* r, uint64_t nr, uint64_t* edges, uint64_t* tris) {
  const auto& eff = *static_cast<const EffectiveAdjacency*>(h);
  uint64_t total = 0, e = 0;
  NullSink sink;
  double t0 = now_s();
  for (uint64_t k = 0; k < nr; ++k)
    for (NodeId v = r[2 * k]; v < r[2 * k + 1]; ++v) {
      auto nv = eff.eff(v);
      e += nv.size();
      for (NodeId u : nv)
        intersect_visit(nv, eff.eff(u), [&](NodeId w) {
          ++total;
          sink(v, u, w);
        });
    }
  double dt = now_s() - t0;
  *edges = e;
  *tris = total;
  return dt;
}

// (ii) The reference AOP (engines.hpp:38-54 over partition.hpp:171-206) on
// one std::thread per sampled core.  `s` holds p sub-ranges [s[2i], s[2i+1])
// of the p = nproc cores of the DPD plan; they become the odd parts of a
// PartitionPlan (partition.hpp:95-110) whose boundaries are {0, s_i, e_i, n}.
// Phase 1 (timed: t_build): every thread runs build_overlap_partition for
// its sub-core; barrier; phase 2 (timed, the return value): aop_count.
// Reports sampled oriented edges, triangles and Σ stored_entries.
double ref_aop_threads(void* h, const uint32_t* s, uint64_t p, double* t_build,
                       uint64_t* edges, uint64_t* tris, uint64_t* stored) {
  const auto& eff = *static_cast<const EffectiveAdjacency*>(h);
  const NodeId n = static_cast<NodeId>(eff.num_nodes());
  PartitionPlan plan;
  plan.boundaries.push_back(0);
  std::vector<std::size_t> part_of(p, SIZE_MAX);
  for (uint64_t i = 0; i < p; ++i) {
    if (s[2 * i] >= s[2 * i + 1]) continue;
    if (plan.boundaries.back() != s[2 * i]) plan.boundaries.push_back(s[2 * i]);
    part_of[i] = plan.boundaries.size() - 1;
    plan.boundaries.push_back(s[2 * i + 1]);
  }
  if (plan.boundaries.back() != n) plan.boundaries.push_back(n);
  Graph g;  // build_overlap_partition ignores g (partition.hpp:174)
  std::vector<OverlapPartition> parts(p);
  std::vector<uint64_t> tt(p, 0), ee(p, 0);
  std::atomic<uint64_t> built{0};
  std::atomic<bool> go{false};
  double tb0 = now_s(), tb1 = 0;
  std::vector<std::thread> pool;
  for (uint64_t i = 0; i < p; ++i)
    pool.emplace_back([&, i] {
      if (part_of[i] != SIZE_MAX) parts[i] = build_overlap_partition(g, eff, plan, part_of[i]);
      if (built.fetch_add(1) + 1 == p) {  // last builder starts the count phase
        tb1 = now_s();
        go.store(true);
      }
      while (!go.load()) std::this_thread::yield();
      if (part_of[i] == SIZE_MAX) return;
      NullSink sink;
      tt[i] = aop_count(parts[i], sink);
      for (NodeId v = parts[i].core_begin; v < parts[i].core_end; ++v) ee[i] += eff.effdeg(v);
    });
  for (auto& th : pool) th.join();
  double tc1 = now_s();
  *t_build = tb1 - tb0;
  uint64_t e = 0, t = 0, st = 0;
  for (uint64_t i = 0; i < p; ++i) {
    e += ee[i];
    t += tt[i];
    st += parts[i].stored_entries();
  }
  *edges = e;
  *tris = t;
  *stored = st;
  return tc1 - tb1;
}

}  // extern "C"
