// trigraph_b200/trigraph.hpp -- header-only C++ mirror of the reference
// `trigraph` API (/root/reference/proj/include/trigraph/) over the C ABI in
// trigraph_b200.h.  A reference user switches by including this header and
// linking libtrigraph_b200.so:
//
//   #include <trigraph_b200/trigraph.hpp>
//   namespace trigraph = trigraph_b200;     // same names, same semantics
//
// Names and argument meaning follow the reference (file:line cited per
// symbol).  Differences: Graph lives on a CUDA device;
// ExecMode is accepted and ignored;
// RankStats::realized_cost is algorithmic work, not merge comparisons.
// Besides the reference's signatures (effective_adjacency(g, OrderRank),
// count_node_iterator_n(eff, sink), count_node_iterator_pp(g, OrderRank)),
// the order-dependent helpers also take the Graph plus an OrderKind (the
// device keeps the oriented CSR cached).
#ifndef TRIGRAPH_B200_TRIGRAPH_HPP
#define TRIGRAPH_B200_TRIGRAPH_HPP

#include <array>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <algorithm>
#include <map>
#include <memory>
#include <optional>
#include <span>
#include <type_traits>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "../trigraph_b200.h"

namespace trigraph_b200 {

using NodeId = std::uint32_t;  // graph.hpp:14

/// io.hpp:18-22.
struct ParseError : std::runtime_error {
  std::size_t line;
  ParseError(std::size_t line_, const std::string& what_)
      : std::runtime_error(what_), line(line_) {}
};

namespace detail {
inline void check(tg_status s, std::uint64_t err_line = 0) {
  if (s == TG_OK) return;
  std::string msg = tg_last_error();
  if (s == TG_ERR_PARSE) throw ParseError(err_line, msg);  // what() = "line N: ..."
  if (s == TG_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(std::string(tg_status_string(s)) + ": " + msg);
}
}  // namespace detail

enum class EngineKind { Sequential, Aop, AnopDirect, AnopSurrogate };  // engines.hpp:24
enum class CostKind { N, D, Dh, Ddh, Dh2, Dpd, Nov };                  // partition.hpp:18
namespace runtime {
enum class ExecMode { Interleaved, Concurrent };  // runtime.hpp:27 (no effect on the device)
}

/// graph.hpp:19-53 -- immutable undirected simple graph, resident on a GPU.
class Graph {
 public:
  Graph() = default;
  /// Graph(n, offsets, adj) (graph.hpp:22-23): adopt a built CSR.
  Graph(std::size_t n, const std::vector<std::size_t>& offsets, const std::vector<NodeId>& adj,
        int device = 0) {
    std::vector<std::uint64_t> off(offsets.begin(), offsets.end());
    detail::check(tg_graph_from_csr(device, n, off.data(), adj.empty() ? nullptr : adj.data(), &h_));
    device_ = device;
  }
  explicit Graph(tg_graph* h, int device = 0) : h_(h), device_(device) {}
  Graph(const Graph&) = delete;
  Graph& operator=(const Graph&) = delete;
  Graph(Graph&& o) noexcept
      : h_(std::exchange(o.h_, nullptr)), device_(o.device_), host_(std::move(o.host_)) {}
  Graph& operator=(Graph&& o) noexcept {
    if (this != &o) {
      if (h_) tg_graph_free(h_);
      h_ = std::exchange(o.h_, nullptr);
      device_ = o.device_;
      host_ = std::move(o.host_);
    }
    return *this;
  }
  ~Graph() {
    if (h_) tg_graph_free(h_);
  }

  std::size_t num_nodes() const { return info().first; }   // graph.hpp:25
  std::size_t num_edges() const { return info().second; }  // graph.hpp:26
  tg_graph* handle() const { return h_; }
  int device() const { return device_; }

  /// Host copy of the CSR (offsets n+1, adjacency 2m).
  std::pair<std::vector<std::uint64_t>, std::vector<NodeId>> csr() const {
    auto [n, m] = info();
    std::vector<std::uint64_t> off(n + 1);
    std::vector<NodeId> adj(2 * m);
    detail::check(tg_graph_csr(h_, off.data(), adj.data()));
    return {std::move(off), std::move(adj)};
  }

  /// graph.hpp:28-46 accessors, served from a host copy of the (immutable)
  /// CSR downloaded on first use.
  std::size_t degree(NodeId v) const {
    const auto& c = host();
    return c.first[v + 1] - c.first[v];
  }
  std::span<const NodeId> neighbors(NodeId v) const {
    const auto& c = host();
    return {c.second.data() + c.first[v], c.second.data() + c.first[v + 1]};
  }
  bool has_edge(NodeId u, NodeId v) const {
    auto nb = neighbors(u);
    return std::binary_search(nb.begin(), nb.end(), v);
  }
  std::vector<std::pair<NodeId, NodeId>> edges() const {  // u < v, u then v ascending
    std::vector<std::pair<NodeId, NodeId>> out;
    const auto& c = host();
    for (NodeId u = 0; u + 1 < c.first.size(); ++u)
      for (std::uint64_t i = c.first[u]; i < c.first[u + 1]; ++i)
        if (u < c.second[i]) out.emplace_back(u, c.second[i]);
    return out;
  }

 private:
  std::pair<std::size_t, std::size_t> info() const {
    std::uint64_t n = 0, m = 0;
    detail::check(tg_graph_info(h_, &n, &m));
    return {n, m};
  }
  const std::pair<std::vector<std::uint64_t>, std::vector<NodeId>>& host() const {
    if (!host_)
      host_ = std::make_shared<std::pair<std::vector<std::uint64_t>, std::vector<NodeId>>>(csr());
    return *host_;
  }
  tg_graph* h_ = nullptr;
  int device_ = 0;
  mutable std::shared_ptr<std::pair<std::vector<std::uint64_t>, std::vector<NodeId>>> host_;
};

/// graph.hpp:58-85 build_graph, on the device.
inline Graph build_graph(const std::vector<std::pair<NodeId, NodeId>>& edge_pairs,
                         std::size_t n_override = 0, int device = 0) {
  std::vector<std::uint32_t> flat(2 * edge_pairs.size());
  for (std::size_t i = 0; i < edge_pairs.size(); ++i) {
    flat[2 * i] = edge_pairs[i].first;
    flat[2 * i + 1] = edge_pairs[i].second;
  }
  tg_graph* h = nullptr;
  detail::check(tg_graph_from_edges(device, flat.empty() ? nullptr : flat.data(), edge_pairs.size(),
                                    n_override, &h));
  return Graph(h, device);
}

/// order.hpp:17-28.
struct OrderKind {
  enum class Tag { ById, ByDegree, ByRandom, ByCoreness };
  Tag tag = Tag::ByDegree;
  std::uint64_t seed = 0;

  static OrderKind by_id() { return {Tag::ById, 0}; }
  static OrderKind by_degree() { return {Tag::ByDegree, 0}; }
  static OrderKind by_random(std::uint64_t seed) { return {Tag::ByRandom, seed}; }
  static OrderKind by_coreness() { return {Tag::ByCoreness, 0}; }
};

namespace detail {
// The graph orients by `kind` from here on (tg_set_order).
inline void use_order(const Graph& g, const OrderKind& kind) {
  check(tg_set_order(g.handle(), static_cast<int32_t>(kind.tag), kind.seed));
}
}  // namespace detail

/// order.hpp:31-35.
struct OrderRank {
  std::vector<NodeId> rank;
  bool precedes(NodeId u, NodeId v) const { return rank[u] < rank[v]; }
};
/// order.hpp:85-128 for every OrderKind (ByRandom bit-identical to the
/// reference's mt19937_64 Fisher-Yates).
inline OrderRank compute_order(const Graph& g, OrderKind kind = OrderKind::by_degree()) {
  detail::use_order(g, kind);
  OrderRank o;
  o.rank.resize(g.num_nodes());
  detail::check(tg_compute_order(g.handle(), o.rank.data()));
  return o;
}

/// order.hpp:39-83 core numbers.
inline std::vector<std::size_t> coreness(const Graph& g) {
  std::vector<std::uint64_t> c(g.num_nodes());
  detail::check(tg_coreness(g.handle(), c.data()));
  return std::vector<std::size_t>(c.begin(), c.end());
}

namespace detail {
// The graph orients by a caller's OrderRank from here on (tg_set_order_rank).
inline void use_order(const Graph& g, const OrderRank& order) {
  if (order.rank.size() != g.num_nodes())
    throw std::invalid_argument("OrderRank: rank must have num_nodes() entries");
  check(tg_set_order_rank(g.handle(), order.rank.empty() ? nullptr : order.rank.data()));
}
}  // namespace detail

/// effective.hpp:17-35.  N_v (ID-sorted) for every v, as host vectors; the
/// first count_node_iterator_n over it adopts a copy on the device
/// (tg_eff_from_csr) that later counts reuse.
class EffectiveAdjacency {
 public:
  EffectiveAdjacency() = default;
  /// EffectiveAdjacency(offsets, eff) (effective.hpp:18-20).
  EffectiveAdjacency(std::vector<std::size_t> offsets_, std::vector<NodeId> eff_, int device = 0)
      : offsets(offsets_.begin(), offsets_.end()), entries(std::move(eff_)), device_(device) {}

  std::size_t num_nodes() const { return offsets.size() - 1; }
  std::size_t total_entries() const { return entries.size(); }
  std::span<const NodeId> eff(NodeId v) const {
    return {entries.data() + offsets[v], entries.data() + offsets[v + 1]};
  }
  std::size_t effdeg(NodeId v) const { return offsets[v + 1] - offsets[v]; }

  std::vector<std::uint64_t> offsets{0};
  std::vector<NodeId> entries;

  /// The device copy (created on first use).
  tg_eff* handle() const {
    if (!dev_) {
      tg_eff* h = nullptr;
      detail::check(tg_eff_from_csr(device_, num_nodes(), offsets.data(),
                                    entries.empty() ? nullptr : entries.data(), &h));
      dev_ = std::shared_ptr<tg_eff>(h, [](tg_eff* p) { tg_eff_free(p); });
    }
    return dev_.get();
  }

 private:
  friend EffectiveAdjacency effective_adjacency_from(const Graph&);
  int device_ = 0;
  mutable std::shared_ptr<tg_eff> dev_;
};

/// The graph's current orientation, downloaded (compact, ID-sorted lists).
inline EffectiveAdjacency effective_adjacency_from(const Graph& g) {
  EffectiveAdjacency e;
  e.offsets.resize(g.num_nodes() + 1);
  e.entries.resize(g.num_edges());
  detail::check(tg_effective_adjacency(g.handle(), e.offsets.data(), e.entries.data()));
  e.device_ = g.device();
  return e;
}

/// effective.hpp:37-52 effective_adjacency(g, order) -- the reference's
/// signature, with the OrderRank of compute_order (or any permutation).
inline EffectiveAdjacency effective_adjacency(const Graph& g, const OrderRank& order) {
  detail::use_order(g, order);
  return effective_adjacency_from(g);
}
/// ... and under an OrderKind (default ByDegree).
inline EffectiveAdjacency effective_adjacency(const Graph& g,
                                              OrderKind order = OrderKind::by_degree()) {
  detail::use_order(g, order);
  return effective_adjacency_from(g);
}

/// sequential.hpp:19-46 sinks.
struct NullSink {
  void operator()(NodeId, NodeId, NodeId) const {}
};
struct NodeTallySink {
  std::vector<std::uint64_t> counts;
  explicit NodeTallySink(std::size_t n) : counts(n, 0) {}
  void operator()(NodeId v, NodeId u, NodeId w) {
    ++counts[v];
    ++counts[u];
    ++counts[w];
  }
};
struct ListSink {
  std::vector<std::array<NodeId, 3>> triangles;
  void operator()(NodeId v, NodeId u, NodeId w) {
    std::array<NodeId, 3> t{v, u, w};
    if (t[0] > t[1]) std::swap(t[0], t[1]);
    if (t[1] > t[2]) std::swap(t[1], t[2]);
    if (t[0] > t[1]) std::swap(t[0], t[1]);
    triangles.push_back(t);
  }
};

/// sequential.hpp:74-91 count_node_iterator_n(eff, sink), on the device:
///   NullSink      -> the count;
///   NodeTallySink -> the device TALLY path (counts added to sink.counts);
///   ListSink      -> the device LIST path (normalised triples appended);
///   any other callable sink(v, u, w) -> the raw (apex, middle, w) triples
///     listed on the device, sorted by (v, u, w) and replayed on the host --
///     the reference's emission order (v ascending, u along the ID-sorted
///     N_v, w ascending).
template <class Sink>
std::uint64_t count_node_iterator_n(const EffectiveAdjacency& eff, Sink&& sink) {
  using S = std::decay_t<Sink>;
  tg_eff* h = eff.handle();
  std::uint64_t t = 0, nt = 0;
  if constexpr (std::is_same_v<S, NullSink>) {
    detail::check(tg_eff_count(h, &t, nullptr, nullptr, 0, 0, &nt));
  } else if constexpr (std::is_same_v<S, NodeTallySink>) {
    std::vector<std::uint64_t> tv(eff.num_nodes());
    detail::check(tg_eff_count(h, &t, tv.empty() ? nullptr : tv.data(), nullptr, 0, 0, &nt));
    for (std::size_t v = 0; v < tv.size() && v < sink.counts.size(); ++v) sink.counts[v] += tv[v];
  } else {
    detail::check(tg_eff_count(h, &t, nullptr, nullptr, 0, 0, &nt));
    std::vector<std::array<NodeId, 3>> tri(t);
    constexpr int raw = std::is_same_v<S, ListSink> ? 0 : 1;
    detail::check(tg_eff_count(h, &t, nullptr, tri.empty() ? nullptr : tri.front().data(), t,
                               raw, &nt));
    if constexpr (std::is_same_v<S, ListSink>) {
      sink.triangles.insert(sink.triangles.end(), tri.begin(), tri.end());
    } else {
      std::sort(tri.begin(), tri.end());
      for (const auto& x : tri) sink(x[0], x[1], x[2]);
    }
  }
  return t;
}
inline std::uint64_t count_node_iterator_n(const EffectiveAdjacency& eff) {
  return count_node_iterator_n(eff, NullSink{});
}

/// sequential.hpp:74-91 over effective_adjacency(g, order) (count only;
/// the oriented CSR stays on the device).
inline std::uint64_t count_node_iterator_n(const Graph& g,
                                           OrderKind order = OrderKind::by_degree()) {
  detail::use_order(g, order);
  std::uint64_t t = 0;
  detail::check(tg_count(g.handle(), &t));
  return t;
}

/// sequential.hpp:48-70 NodeIterator++ (the reference's signature takes the
/// OrderRank; an OrderKind works too).
inline std::uint64_t count_node_iterator_pp(const Graph& g, const OrderRank& order,
                                            bool use_intersection = false) {
  detail::use_order(g, order);
  std::uint64_t t = 0;
  detail::check(tg_count_node_iterator_pp(g.handle(), use_intersection ? 1 : 0, &t));
  return t;
}
inline std::uint64_t count_node_iterator_pp(const Graph& g, OrderKind order = OrderKind::by_degree(),
                                            bool use_intersection = false) {
  detail::use_order(g, order);
  std::uint64_t t = 0;
  detail::check(tg_count_node_iterator_pp(g.handle(), use_intersection ? 1 : 0, &t));
  return t;
}

/// sequential.hpp:95-104 under `order` (default ByDegree).
inline std::uint64_t ordering_cost(const Graph& g, const OrderRank& order) {
  detail::use_order(g, order);
  std::uint64_t c = 0;
  detail::check(tg_ordering_cost(g.handle(), &c));
  return c;
}
inline std::uint64_t ordering_cost(const Graph& g, OrderKind order = OrderKind::by_degree()) {
  detail::use_order(g, order);
  std::uint64_t c = 0;
  detail::check(tg_ordering_cost(g.handle(), &c));
  return c;
}

/// partition.hpp:38-91.
struct CostVector {
  std::vector<std::uint64_t> f, prefix;
  std::uint64_t total() const { return prefix.empty() ? 0 : prefix.back(); }
};
inline CostVector node_costs(const Graph& g, CostKind kind,
                             OrderKind order = OrderKind::by_degree()) {
  detail::use_order(g, order);
  CostVector c;
  c.f.resize(g.num_nodes());
  c.prefix.resize(g.num_nodes());
  detail::check(tg_node_costs(g.handle(), static_cast<int32_t>(kind), c.f.data(), c.prefix.data()));
  return c;
}

/// partition.hpp:95-141.
struct PartitionPlan {
  std::vector<NodeId> boundaries;
  std::size_t ranks() const { return boundaries.size() - 1; }
  NodeId core_begin(std::size_t i) const { return boundaries[i]; }
  NodeId core_end(std::size_t i) const { return boundaries[i + 1]; }
  bool in_core(std::size_t i, NodeId v) const { return v >= core_begin(i) && v < core_end(i); }
  std::size_t owner(NodeId v) const {
    std::size_t lo = 1, hi = boundaries.size() - 1;
    while (lo < hi) {
      std::size_t mid = (lo + hi) / 2;
      if (boundaries[mid] <= v) lo = mid + 1;
      else hi = mid;
    }
    return lo - 1;
  }
};
inline PartitionPlan compute_boundaries(const Graph& g, CostKind kind, std::size_t p,
                                        OrderKind order = OrderKind::by_degree()) {
  if (p == 0) throw std::invalid_argument("compute_boundaries: p must be >= 1");
  detail::use_order(g, order);
  PartitionPlan plan;
  plan.boundaries.resize(p + 1);
  detail::check(tg_compute_boundaries(g.handle(), static_cast<int32_t>(kind), p,
                                      plan.boundaries.data()));
  return plan;
}

/// sparsify.hpp:22-33.
struct SparsifyConfig {
  enum class Mode { PerPartition, Global };
  double q = 1.0;
  std::uint64_t seed = 0;
  Mode mode = Mode::Global;
  void validate() const {
    if (!(q > 0.0 && q <= 1.0)) throw std::invalid_argument("sparsify: q must be in (0, 1]");
  }
};

/// engines.hpp:270-298.
struct EngineConfig {
  EngineKind engine = EngineKind::Aop;
  std::size_t ranks = 1;
  CostKind cost = CostKind::Dpd;
  OrderKind order = OrderKind::by_degree();
  runtime::ExecMode mode = runtime::ExecMode::Interleaved;
  bool track_nodes = false;
  bool collect_triangles = false;
  std::optional<SparsifyConfig> sparsify;
  std::optional<std::vector<NodeId>> boundaries;
};

struct RankStats {
  std::uint64_t triangles = 0, data_sent = 0, data_recv = 0, realized_cost = 0,
                stored_entries = 0;
};

struct RunReport {
  EngineKind engine = EngineKind::Sequential;
  std::size_t ranks = 1;
  CostKind cost = CostKind::Dpd;
  std::uint64_t total = 0;
  std::vector<RankStats> per_rank;
  std::vector<NodeId> boundaries;
  std::vector<std::uint64_t> node_counts;
  std::vector<std::array<NodeId, 3>> triangles_list;
};

namespace detail {
inline tg_config to_c(const EngineConfig& cfg) {
  tg_config c{};
  c.engine = static_cast<int32_t>(cfg.engine);
  c.cost = static_cast<int32_t>(cfg.cost);
  c.ranks = cfg.ranks;
  c.boundaries = cfg.boundaries ? cfg.boundaries->data() : nullptr;
  c.track_nodes = cfg.track_nodes;
  c.collect_triangles = cfg.collect_triangles;
  c.order_set = 1;  // engines.hpp:274
  c.order = static_cast<int32_t>(cfg.order.tag);
  c.order_seed = cfg.order.seed;
  if (cfg.sparsify) {
    cfg.sparsify->validate();
    c.sparsify = cfg.sparsify->mode == SparsifyConfig::Mode::PerPartition
                     ? TG_SPARSIFY_PER_PARTITION
                     : TG_SPARSIFY_GLOBAL;
    c.sparsify_q = cfg.sparsify->q;
    c.sparsify_seed = cfg.sparsify->seed;
  }
  return c;
}
}  // namespace detail

/// engines.hpp:335-418 run_engine.
inline RunReport run_engine(const Graph& g, const EngineConfig& cfg) {
  const std::size_t p = cfg.engine == EngineKind::Sequential ? 1 : cfg.ranks;
  if (p == 0) throw std::invalid_argument("run_engine: ranks must be >= 1");
  if (cfg.boundaries && cfg.boundaries->size() != p + 1)
    throw std::invalid_argument("run_engine: boundaries must have ranks+1 entries");
  tg_config c = detail::to_c(cfg);
  RunReport rep;
  rep.engine = cfg.engine;
  rep.ranks = p;
  rep.cost = cfg.cost;
  std::vector<tg_rank_stats> st(p);
  rep.boundaries.resize(p + 1);
  if (cfg.track_nodes) rep.node_counts.resize(g.num_nodes());
  std::uint64_t cap = cfg.collect_triangles ? count_node_iterator_n(g, cfg.order) : 0, got = 0;
  std::vector<NodeId> flat(3 * cap);
  detail::check(tg_run_engine(g.handle(), &c, &rep.total, st.data(), rep.boundaries.data(),
                              cfg.track_nodes ? rep.node_counts.data() : nullptr,
                              cfg.collect_triangles ? flat.data() : nullptr, cap, &got));
  for (const auto& s : st)
    rep.per_rank.push_back({s.triangles, s.data_sent, s.data_recv, s.realized_cost,
                            s.stored_entries});
  if (cfg.collect_triangles) {
    rep.triangles_list.resize(got);
    for (std::uint64_t k = 0; k < got; ++k)
      rep.triangles_list[k] = {flat[3 * k], flat[3 * k + 1], flat[3 * k + 2]};
  }
  return rep;
}

/// engines.hpp:203-206, 422-435.
struct ClusteringResult {
  std::vector<std::uint64_t> triangles_per_node;
  std::vector<double> coefficient;
};
inline ClusteringResult clustering_coefficients(const Graph& g, EngineConfig cfg) {
  const std::size_t p = cfg.engine == EngineKind::Sequential ? 1 : cfg.ranks;
  if (p == 0) throw std::invalid_argument("run_engine: ranks must be >= 1");
  cfg.track_nodes = true;
  tg_config c = detail::to_c(cfg);
  ClusteringResult r;
  r.triangles_per_node.resize(g.num_nodes());
  r.coefficient.resize(g.num_nodes());
  detail::check(tg_clustering_coefficients(g.handle(), &c, r.triangles_per_node.data(),
                                           r.coefficient.data()));
  return r;
}

/// engines.hpp:440-457 approx_count: T' / q^3 (AOP: per-partition draws).
inline double approx_count(const Graph& g, std::size_t p, EngineKind engine, double q,
                           std::uint64_t seed,
                           runtime::ExecMode = runtime::ExecMode::Interleaved,
                           const std::optional<std::vector<NodeId>>& boundaries = {},
                           CostKind cost = CostKind::Dpd) {
  double est = 0.0;
  detail::check(tg_approx_count(g.handle(), p, static_cast<int32_t>(engine), q, seed,
                                boundaries ? boundaries->data() : nullptr,
                                static_cast<int32_t>(cost), &est));
  return est;
}

/// sequential.hpp:108-122 per_edge_triangle_counts, keyed like the
/// reference's map by the (u < v) edge pairs in Graph::edges() order.
inline std::map<std::pair<NodeId, NodeId>, std::uint64_t> per_edge_triangle_counts(
    const Graph& g) {
  std::vector<std::uint64_t> te(g.num_edges());
  detail::check(tg_per_edge_triangle_counts(g.handle(), te.data()));
  std::map<std::pair<NodeId, NodeId>, std::uint64_t> out;
  const auto [off, adj] = g.csr();
  std::uint64_t k = 0;
  for (NodeId u = 0; u + 1 < off.size(); ++u)
    for (std::uint64_t i = off[u]; i < off[u + 1]; ++i)
      if (u < adj[i]) out[{u, adj[i]}] = te[k++];
  return out;
}
/// sequential.hpp:108-122 with the reference's signature: t_e does not
/// depend on the order the EffectiveAdjacency was built under.
inline std::map<std::pair<NodeId, NodeId>, std::uint64_t> per_edge_triangle_counts(
    const Graph& g, const EffectiveAdjacency&) {
  return per_edge_triangle_counts(g);
}

/// sparsify.hpp:113-155 variance_report.
struct VarianceReport {
  std::uint64_t triangles = 0, k = 0, k_prime = 0;
  double q = 1.0, var = 0.0, var_prime = 0.0;
};
inline VarianceReport variance_report(const Graph& g, const PartitionPlan& plan, double q) {
  std::uint64_t o3[3];
  double v2[2];
  detail::check(tg_variance_report(g.handle(), plan.boundaries.data(), plan.ranks(), q, o3, v2));
  return {o3[0], o3[1], o3[2], q, v2[0], v2[1]};
}

/// count_node_iterator_n(effective_adjacency(Graph(n, offsets, adj))) from a
/// host CSR in one call, the upload overlapped with the count.
inline std::uint64_t count_from_csr(std::size_t n, const std::uint64_t* offsets, const NodeId* adj,
                                    int device = 0) {
  std::uint64_t t = 0;
  detail::check(tg_count_from_csr(device, n, offsets, adj, &t));
  return t;
}

/// io.hpp:24-50 parse_edge_list, on the device.
inline std::vector<std::pair<NodeId, NodeId>> parse_edge_list(std::string_view text,
                                                              int device = 0) {
  std::uint64_t cnt = 0, line = 0;
  // (status first: the error line is only set once the call returned)
  tg_status st = tg_parse_edge_list(device, text.data(), text.size(), nullptr, 0, &cnt, &line);
  detail::check(st, line);
  std::vector<std::uint32_t> flat(2 * cnt);
  st = tg_parse_edge_list(device, text.data(), text.size(), flat.data(), cnt, &cnt, &line);
  detail::check(st, line);
  std::vector<std::pair<NodeId, NodeId>> out(cnt);
  for (std::uint64_t k = 0; k < cnt; ++k) out[k] = {flat[2 * k], flat[2 * k + 1]};
  return out;
}

/// build_graph(parse_edge_list(text), n_override) without the host round trip.
inline Graph build_graph_from_text(std::string_view text, std::size_t n_override = 0,
                                   int device = 0) {
  tg_graph* h = nullptr;
  std::uint64_t line = 0;
  const tg_status st = tg_graph_from_text(device, text.data(), text.size(), n_override, &h, &line);
  detail::check(st, line);
  return Graph(h, device);
}

/// io.hpp:52-64 write_edge_list, on the device.
inline std::string write_edge_list(const Graph& g) {
  std::uint64_t len = 0;
  detail::check(tg_write_edge_list(g.handle(), nullptr, 0, &len));
  std::string out(len, '\0');
  if (len) detail::check(tg_write_edge_list(g.handle(), &out[0], len, &len));
  return out;
}

/// stats.hpp:21-23 (host arithmetic, as in the reference).
inline double normalized_triangle_count(std::uint64_t triangles, std::size_t n) {
  return n == 0 ? 0.0 : static_cast<double>(triangles) / static_cast<double>(n);
}

/// stats.hpp:11-19 (host arithmetic, as in the reference).
inline std::uint64_t estimate_p_opt(double n, double dbar, double base_n, double base_dbar,
                                    double base_p_opt) {
  if (n <= 0 || dbar <= 0 || base_n <= 0 || base_dbar <= 0 || base_p_opt <= 0)
    throw std::invalid_argument("estimate_p_opt: all inputs must be positive");
  const double est = base_p_opt * (dbar / base_dbar) * std::sqrt(n / base_n);
  return static_cast<std::uint64_t>(std::llround(est));
}

/// io.hpp:129-162 gen_pa (host, bit-identical edge stream).
inline std::vector<std::pair<NodeId, NodeId>> gen_pa_edges(std::size_t n, std::size_t d,
                                                           std::uint64_t seed) {
  std::uint32_t* p = nullptr;
  std::uint64_t E = 0;
  detail::check(tg_gen_pa(n, d, seed, &p, &E));
  std::vector<std::pair<NodeId, NodeId>> out(E);
  for (std::uint64_t i = 0; i < E; ++i) out[i] = {p[2 * i], p[2 * i + 1]};
  tg_free_host(p);
  return out;
}
inline Graph gen_pa(std::size_t n, std::size_t d, std::uint64_t seed, int device = 0) {
  return build_graph(gen_pa_edges(n, d, seed), n, device);
}

inline const char* to_string(EngineKind e) {  // engines.hpp:26-34
  switch (e) {
    case EngineKind::Sequential: return "seq";
    case EngineKind::Aop: return "aop";
    case EngineKind::AnopDirect: return "anop-direct";
    case EngineKind::AnopSurrogate: return "anop-surrogate";
  }
  return "?";
}

}  // namespace trigraph_b200

#endif  // TRIGRAPH_B200_TRIGRAPH_HPP
