// C++ drop-in check, run on the B200 by tests/test_gpu_cpp.py (compiled
// against include/ + libtrigraph_b200.so; tests/test_abi.py compiles it on
// CPU).
//
// Part 1 is the reference's own test cases, copied unchanged from
// proj/tests/test_sequential.cpp and proj/tests/test_engines.cpp (file:line
// above each): the only differences are the namespace alias below and the
// doctest stand-ins (TEST_CASE / CHECK / REQUIRE / CHECK_THROWS_AS /
// doctest::Approx) of the small harness here.  `oracles::` is the test
// fixture library of proj/tests/oracles.hpp, restated on the mirror API
// (same fixtures, same seeded random_graph stream, brute-force oracles on
// the host).  Part 2 holds further cases written against the mirror.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "trigraph_b200/trigraph.hpp"

namespace trigraph = trigraph_b200;
using namespace trigraph;

// ---- doctest stand-ins --------------------------------------------------

namespace harness {
int failures = 0;
struct Case {
  const char* name;
  void (*fn)();
};
std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}
struct Registrar {
  Registrar(const char* name, void (*fn)()) { cases().push_back({name, fn}); }
};
struct RequireFailed {};
}  // namespace harness

namespace doctest {
struct Approx {  // doctest's default: relative epsilon FLT_EPSILON * 100
  double v;
  explicit Approx(double x) : v(x) {}
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v) < 1.1920929e-05 * (1.0 + std::max(std::fabs(a), std::fabs(b.v)));
  }
};
}  // namespace doctest

#define TG_CAT2(a, b) a##b
#define TG_CAT(a, b) TG_CAT2(a, b)
#define TEST_CASE(name)                                                                  \
  static void TG_CAT(tg_case_, __LINE__)();                                               \
  static harness::Registrar TG_CAT(tg_reg_, __LINE__)(name, TG_CAT(tg_case_, __LINE__)); \
  static void TG_CAT(tg_case_, __LINE__)()
#define CHECK(...)                                               \
  do {                                                           \
    if (!(__VA_ARGS__)) {                                        \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #__VA_ARGS__); \
      ++harness::failures;                                       \
    }                                                            \
  } while (0)
#define REQUIRE(...)                                                     \
  do {                                                                   \
    if (!(__VA_ARGS__)) {                                                \
      std::printf("FAIL (REQUIRE) %s:%d: %s\n", __FILE__, __LINE__, #__VA_ARGS__); \
      ++harness::failures;                                               \
      throw harness::RequireFailed{};                                    \
    }                                                                    \
  } while (0)
#define CHECK_THROWS_AS(expr, E)                     \
  do {                                               \
    bool tg_threw = false;                           \
    try {                                            \
      (void)(expr);                                  \
    } catch (const E&) {                             \
      tg_threw = true;                               \
    }                                                \
    CHECK(tg_threw && #expr " throws " #E);          \
  } while (0)

// ---- proj/tests/oracles.hpp fixtures, restated on the mirror ------------

namespace oracles {
inline Graph g5() { return build_graph({{0, 1}, {0, 2}, {1, 2}, {1, 3}, {2, 3}, {3, 4}}); }
inline Graph complete(std::size_t n) {
  std::vector<std::pair<NodeId, NodeId>> e;
  for (NodeId u = 0; u < n; ++u)
    for (NodeId v = u + 1; v < n; ++v) e.emplace_back(u, v);
  return build_graph(e, n);
}
// oracles.hpp:49-57: seeded G(n, density), the same mt19937_64 draws
inline Graph random_graph(std::size_t n, double density, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  std::vector<std::pair<NodeId, NodeId>> e;
  for (NodeId u = 0; u < n; ++u)
    for (NodeId v = u + 1; v < n; ++v)
      if (unit(rng) < density) e.emplace_back(u, v);
  return build_graph(e, n);
}
inline std::vector<std::array<NodeId, 3>> brute_list(const Graph& g) {
  std::vector<std::array<NodeId, 3>> out;
  const std::size_t n = g.num_nodes();
  for (NodeId a = 0; a < n; ++a)
    for (NodeId b = a + 1; b < n; ++b) {
      if (!g.has_edge(a, b)) continue;
      for (NodeId c = b + 1; c < n; ++c)
        if (g.has_edge(a, c) && g.has_edge(b, c)) out.push_back({a, b, c});
    }
  return out;
}
inline std::uint64_t brute_count(const Graph& g) { return brute_list(g).size(); }
inline std::vector<std::uint64_t> brute_node_counts(const Graph& g) {
  std::vector<std::uint64_t> tv(g.num_nodes(), 0);
  for (const auto& t : brute_list(g))
    for (NodeId x : t) ++tv[x];
  return tv;
}
// oracles.hpp:95-104: random total order (Fisher-Yates, modulo draw)
inline OrderRank random_order(std::size_t n, std::mt19937_64& rng) {
  std::vector<NodeId> nodes(n);
  for (std::size_t i = 0; i < n; ++i) nodes[i] = static_cast<NodeId>(i);
  for (std::size_t i = n; i > 1; --i) std::swap(nodes[i - 1], nodes[rng() % i]);
  OrderRank out;
  out.rank.resize(n);
  for (std::size_t i = 0; i < n; ++i) out.rank[nodes[i]] = static_cast<NodeId>(i);
  return out;
}
// oracles.hpp:108-115: agreement of an order with the degree order on (x, y)
inline int agreement(const Graph& g, const OrderRank& degree_order, const OrderRank& k_order,
                     NodeId x, NodeId y) {
  if (!g.has_edge(x, y)) return 0;
  if (degree_order.precedes(x, y) && k_order.precedes(y, x)) return -1;
  if (degree_order.precedes(y, x) && k_order.precedes(x, y)) return 1;
  return 0;
}
}  // namespace oracles

// ======================= part 1: the reference's cases ===================

// ---- reference test cases, unchanged (proj/tests/test_sequential.cpp) ----

// test_sequential.cpp:19-31
TEST_CASE("NodeIterator++ counts") {
  auto g5 = oracles::g5();
  auto ord = compute_order(g5, OrderKind::by_degree());
  CHECK(count_node_iterator_pp(g5, ord) == 2);
  CHECK(count_node_iterator_pp(g5, ord, true) == 2);

  auto k4 = oracles::complete(4);
  for (auto kind : {OrderKind::by_id(), OrderKind::by_degree(), OrderKind::by_random(5)})
    CHECK(count_node_iterator_pp(k4, compute_order(k4, kind)) == 4);

  auto path = build_graph({{0, 1}, {1, 2}, {2, 3}});
  CHECK(count_node_iterator_pp(path, compute_order(path, OrderKind::by_degree())) == 0);
}

// test_sequential.cpp:33-43
TEST_CASE("NodeIteratorN finds each triangle once with the apex first") {
  auto g = oracles::g5();
  auto eff = effective_adjacency(g, compute_order(g, OrderKind::by_degree()));
  std::vector<std::array<NodeId, 3>> raw;
  auto total = count_node_iterator_n(
      eff, [&](NodeId v, NodeId u, NodeId w) { raw.push_back({v, u, w}); });
  CHECK(total == 2);
  REQUIRE(raw.size() == 2);
  CHECK(raw[0] == std::array<NodeId, 3>{0, 1, 2});
  CHECK(raw[1] == std::array<NodeId, 3>{1, 2, 3});
}

// test_sequential.cpp:45-51
TEST_CASE("NodeIteratorN on complete graphs") {
  for (std::size_t n = 3; n <= 8; ++n) {
    auto g = oracles::complete(n);
    auto eff = effective_adjacency(g, compute_order(g, OrderKind::by_degree()));
    CHECK(count_node_iterator_n(eff) == n * (n - 1) * (n - 2) / 6);
  }
}

// test_sequential.cpp:53-68
TEST_CASE("both kernels match brute force under every ordering") {
  std::mt19937_64 rng(77);
  for (int i = 0; i < 25; ++i) {
    std::size_t n = 5 + rng() % 50;
    double density = 0.05 + 0.9 * (i / 25.0);
    auto g = oracles::random_graph(n, density, rng());
    auto expected = oracles::brute_count(g);
    for (auto kind : {OrderKind::by_id(), OrderKind::by_degree(),
                      OrderKind::by_random(rng()), OrderKind::by_coreness()}) {
      auto ord = compute_order(g, kind);
      CHECK(count_node_iterator_pp(g, ord) == expected);
      CHECK(count_node_iterator_pp(g, ord, true) == expected);
      CHECK(count_node_iterator_n(effective_adjacency(g, ord)) == expected);
    }
  }
}

// test_sequential.cpp:70-81
TEST_CASE("listing matches brute force") {
  std::mt19937_64 rng(5);
  for (int i = 0; i < 10; ++i) {
    auto g = oracles::random_graph(30, 0.3, rng());
    auto eff = effective_adjacency(g, compute_order(g, OrderKind::by_degree()));
    ListSink sink;
    count_node_iterator_n(eff, sink);
    auto got = sink.triangles;
    std::sort(got.begin(), got.end());
    CHECK(got == oracles::brute_list(g));
  }
}

// test_sequential.cpp:83-87
TEST_CASE("ordering cost on G5") {
  auto g = oracles::g5();
  CHECK(ordering_cost(g, compute_order(g, OrderKind::by_degree())) == 14);
  CHECK(ordering_cost(g, compute_order(g, OrderKind::by_id())) == 16);
}

// test_sequential.cpp:89-97
TEST_CASE("degree ordering minimizes the cost (Theorem 3 shape)") {
  std::mt19937_64 rng(123);
  for (int i = 0; i < 10; ++i) {
    auto g = oracles::random_graph(6 + rng() % 40, 0.3, rng());
    auto base = ordering_cost(g, compute_order(g, OrderKind::by_degree()));
    for (int j = 0; j < 40; ++j)
      CHECK(base <= ordering_cost(g, oracles::random_order(g.num_nodes(), rng)));
  }
}

// test_sequential.cpp:99-115
TEST_CASE("agreement function sign property (Lemma 1 shape)") {
  std::mt19937_64 rng(321);
  for (int i = 0; i < 10; ++i) {
    auto g = oracles::random_graph(5 + rng() % 30, 0.4, rng());
    auto dord = compute_order(g, OrderKind::by_degree());
    for (int j = 0; j < 20; ++j) {
      auto kord = oracles::random_order(g.num_nodes(), rng);
      for (auto [x, y] : g.edges()) {
        int yxy = oracles::agreement(g, dord, kord, x, y);
        CHECK(yxy == -oracles::agreement(g, dord, kord, y, x));
        long long dx = static_cast<long long>(g.degree(x));
        long long dy = static_cast<long long>(g.degree(y));
        CHECK(yxy * (dx - dy) >= 0);
      }
    }
  }
}

// test_sequential.cpp:117-135
TEST_CASE("per-edge triangle counts") {
  auto g = oracles::g5();
  auto eff = effective_adjacency(g, compute_order(g, OrderKind::by_degree()));
  auto te = per_edge_triangle_counts(g, eff);
  CHECK(te.at({1, 2}) == 2);
  CHECK(te.at({0, 1}) == 1);
  CHECK(te.at({0, 2}) == 1);
  CHECK(te.at({1, 3}) == 1);
  CHECK(te.at({2, 3}) == 1);
  CHECK(te.at({3, 4}) == 0);

  auto k4 = oracles::complete(4);
  auto ek4 = effective_adjacency(k4, compute_order(k4, OrderKind::by_degree()));
  for (const auto& [e, c] : per_edge_triangle_counts(k4, ek4)) CHECK(c == 2);

  std::uint64_t sum = 0;
  for (const auto& [e, c] : te) sum += c;
  CHECK(sum == 3 * 2);
}

// ---- reference test cases, unchanged (proj/tests/test_engines.cpp) ----

// test_engines.cpp:10-26
namespace {

EngineConfig config(EngineKind engine, std::size_t p,
                    CostKind cost = CostKind::Dpd,
                    runtime::ExecMode mode = runtime::ExecMode::Interleaved) {
  EngineConfig cfg;
  cfg.engine = engine;
  cfg.ranks = p;
  cfg.cost = cost;
  cfg.mode = mode;
  return cfg;
}

const EngineKind kParallel[] = {EngineKind::Aop, EngineKind::AnopDirect,
                                EngineKind::AnopSurrogate};

}  // namespace

// test_engines.cpp:28-38
TEST_CASE("AOP on G5 with plan [0,2,5]: rank 0 counts both triangles") {
  auto g = oracles::g5();
  auto cfg = config(EngineKind::Aop, 2);
  cfg.boundaries = std::vector<NodeId>{0, 2, 5};
  auto report = run_engine(g, cfg);
  CHECK(report.total == 2);
  CHECK(report.per_rank[0].triangles == 2);
  CHECK(report.per_rank[1].triangles == 0);
  CHECK(report.per_rank[0].data_sent == 0);
  CHECK(report.per_rank[1].data_sent == 0);
}

// test_engines.cpp:40-52
TEST_CASE("ANOP-direct on G5 with plan [0,2,5]: 3 requests, 3 replies") {
  auto g = oracles::g5();
  auto cfg = config(EngineKind::AnopDirect, 2);
  cfg.boundaries = std::vector<NodeId>{0, 2, 5};
  auto report = run_engine(g, cfg);
  CHECK(report.total == 2);
  CHECK(report.per_rank[0].triangles == 2);
  CHECK(report.per_rank[1].triangles == 0);
  // Rank 0 sends 3 requests, rank 1 sends 3 replies.
  CHECK(report.per_rank[0].data_sent == 3);
  CHECK(report.per_rank[1].data_sent == 3);
  CHECK(report.per_rank[0].data_sent + report.per_rank[1].data_sent == 6);
}

// test_engines.cpp:54-64
TEST_CASE("ANOP-surrogate on G5 with plan [0,2,5]: 2 data messages") {
  auto g = oracles::g5();
  auto cfg = config(EngineKind::AnopSurrogate, 2);
  cfg.boundaries = std::vector<NodeId>{0, 2, 5};
  auto report = run_engine(g, cfg);
  CHECK(report.total == 2);
  CHECK(report.per_rank[0].triangles == 1);
  CHECK(report.per_rank[1].triangles == 1);
  CHECK(report.per_rank[0].data_sent == 2);
  CHECK(report.per_rank[1].data_sent == 0);
}

// test_engines.cpp:81-88
TEST_CASE("p=1 runs send nothing") {
  auto g = oracles::g5();
  for (auto engine : kParallel) {
    auto report = run_engine(g, config(engine, 1));
    CHECK(report.total == 2);
    CHECK(report.per_rank[0].data_sent == 0);
  }
}

// test_engines.cpp:90-94
TEST_CASE("K8 with ANOP-surrogate, NOV, p=3") {
  auto report = run_engine(oracles::complete(8),
                           config(EngineKind::AnopSurrogate, 3, CostKind::Nov));
  CHECK(report.total == 56);
}

// test_engines.cpp:96-108
TEST_CASE("engine agreement across p, cost kinds and modes") {
  std::mt19937_64 rng(900);
  for (int i = 0; i < 8; ++i) {
    auto g = oracles::random_graph(20 + rng() % 40, 0.05 + 0.1 * i, rng());
    auto expected = oracles::brute_count(g);
    CHECK(run_engine(g, config(EngineKind::Sequential, 1)).total == expected);
    for (auto engine : kParallel)
      for (std::size_t p : {1, 2, 4})
        for (auto cost : {CostKind::N, CostKind::Dpd, CostKind::Nov})
          for (auto mode : {runtime::ExecMode::Interleaved, runtime::ExecMode::Concurrent})
            CHECK(run_engine(g, config(engine, p, cost, mode)).total == expected);
  }
}

// test_engines.cpp:110-123
TEST_CASE("collected triangle lists match brute force") {
  std::mt19937_64 rng(31);
  for (int i = 0; i < 5; ++i) {
    auto g = oracles::random_graph(30, 0.3, rng());
    auto expected = oracles::brute_list(g);
    for (auto engine : kParallel) {
      auto cfg = config(engine, 3);
      cfg.collect_triangles = true;
      auto got = run_engine(g, cfg).triangles_list;
      std::sort(got.begin(), got.end());
      CHECK(got == expected);
    }
  }
}

// test_engines.cpp:125-139
TEST_CASE("clustering coefficients on G5") {
  auto g = oracles::g5();
  for (auto engine : {EngineKind::Sequential, EngineKind::Aop, EngineKind::AnopDirect,
                      EngineKind::AnopSurrogate}) {
    auto cc = clustering_coefficients(g, config(engine, 2));
    CHECK(cc.triangles_per_node ==
          std::vector<std::uint64_t>{1, 2, 2, 1, 0});
    REQUIRE(cc.coefficient.size() == 5);
    CHECK(cc.coefficient[0] == doctest::Approx(1.0));
    CHECK(cc.coefficient[1] == doctest::Approx(2.0 / 3.0));
    CHECK(cc.coefficient[2] == doctest::Approx(2.0 / 3.0));
    CHECK(cc.coefficient[3] == doctest::Approx(1.0 / 3.0));
    CHECK(cc.coefficient[4] == doctest::Approx(0.0));
  }
}

// test_engines.cpp:141-148
TEST_CASE("K4 and star clustering coefficients") {
  auto cc = clustering_coefficients(oracles::complete(4), config(EngineKind::Aop, 2));
  for (double c : cc.coefficient) CHECK(c == doctest::Approx(1.0));

  auto star = build_graph({{0, 1}, {0, 2}, {0, 3}, {0, 4}});
  auto sc = clustering_coefficients(star, config(EngineKind::AnopSurrogate, 2));
  for (double c : sc.coefficient) CHECK(c == doctest::Approx(0.0));
}

// test_engines.cpp:150-160
TEST_CASE("per-node tallies match brute force across engines") {
  std::mt19937_64 rng(404);
  for (int i = 0; i < 5; ++i) {
    auto g = oracles::random_graph(40, 0.2, rng());
    auto expected = oracles::brute_node_counts(g);
    for (auto engine : kParallel) {
      auto cc = clustering_coefficients(g, config(engine, 3));
      CHECK(cc.triangles_per_node == expected);
    }
  }
}

// test_engines.cpp:162-170
TEST_CASE("realized cost is reported for parallel engines") {
  auto g = oracles::complete(8);
  for (auto engine : kParallel) {
    auto report = run_engine(g, config(engine, 2));
    std::uint64_t cost = 0;
    for (const auto& rs : report.per_rank) cost += rs.realized_cost;
    CHECK(cost > 0);
  }
}

// test_engines.cpp:172-175
TEST_CASE("run_engine validates rank count") {
  auto g = oracles::g5();
  CHECK_THROWS_AS(run_engine(g, config(EngineKind::Aop, 0)), std::invalid_argument);
}


// ======================= part 2: further mirror cases ======================

TEST_CASE("mirror 1: test_graph.cpp:10-17") {
  auto g = build_graph({{0, 1}, {1, 0}, {2, 2}});
  CHECK(g.num_nodes() == 3);
  CHECK(g.num_edges() == 1);
}

TEST_CASE("mirror 2: test_graph.cpp:57-64") {
  auto g = oracles::g5();
  auto ord = compute_order(g);
  CHECK((ord.rank == std::vector<NodeId>{1, 2, 3, 4, 0}));
  CHECK(ord.precedes(4, 0));
  auto eff = effective_adjacency(g);
  CHECK(eff.total_entries() == 6);
  CHECK(count_node_iterator_n(g) == 2);
  CHECK(ordering_cost(g) == 14);
  CHECK((node_costs(g, CostKind::Dpd).f == std::vector<std::uint64_t>{7, 5, 1, 0, 1}));
  CHECK((node_costs(g, CostKind::Nov).f == std::vector<std::uint64_t>{0, 4, 6, 4, 0}));
}

TEST_CASE("mirror 3: test_engines.cpp:28-64") {
  auto g = oracles::g5();
  auto cfg = config(EngineKind::Aop, 2);
  cfg.boundaries = std::vector<NodeId>{0, 2, 5};
  auto r = run_engine(g, cfg);
  CHECK(r.total == 2 && r.per_rank[0].triangles == 2 && r.per_rank[1].triangles == 0);
  cfg.engine = EngineKind::AnopDirect;
  r = run_engine(g, cfg);
  CHECK(r.per_rank[0].data_sent == 3 && r.per_rank[1].data_sent == 3);
  cfg.engine = EngineKind::AnopSurrogate;
  r = run_engine(g, cfg);
  CHECK(r.per_rank[0].triangles == 1 && r.per_rank[1].triangles == 1);
  CHECK(r.per_rank[0].data_sent == 2 && r.per_rank[1].data_sent == 0);
}

TEST_CASE("mirror 4: test_engines.cpp:90-94, 125-139, 172-175") {
  std::vector<std::pair<NodeId, NodeId>> k8;
  for (NodeId u = 0; u < 8; ++u)
    for (NodeId v = u + 1; v < 8; ++v) k8.push_back({u, v});
  CHECK(run_engine(build_graph(k8, 8), config(EngineKind::AnopSurrogate, 3, CostKind::Nov)).total == 56);
  auto cc = clustering_coefficients(oracles::g5(), config(EngineKind::Aop, 2));
  CHECK((cc.triangles_per_node == std::vector<std::uint64_t>{1, 2, 2, 1, 0}));
  CHECK(cc.coefficient[0] == 1.0 && cc.coefficient[1] == 2.0 / 3.0 && cc.coefficient[4] == 0.0);
  bool threw = false;
  try {
    run_engine(oracles::g5(), config(EngineKind::Aop, 0));
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
}

TEST_CASE("mirror 5: 8(f) rows: per-edge counts, q = 1 sparsification, variance report") {
  // (sequential.hpp:108-122, engines.hpp:440-457, sparsify.hpp:113-155)
  auto te = per_edge_triangle_counts(oracles::g5());
  CHECK(te.size() == 6 && te.at({1, 2}) == 2 && te.at({0, 1}) == 1 && te.at({3, 4}) == 0);
  std::vector<std::pair<NodeId, NodeId>> k8;
  for (NodeId u = 0; u < 8; ++u)
    for (NodeId v = u + 1; v < 8; ++v) k8.push_back({u, v});
  auto gk = build_graph(k8, 8);
  CHECK(approx_count(gk, 3, EngineKind::Aop, 1.0, 7) == 56.0);
  EngineConfig sc = config(EngineKind::AnopSurrogate, 3);
  sc.sparsify = SparsifyConfig{0.5, 11, SparsifyConfig::Mode::Global};
  auto rs = run_engine(gk, sc);
  auto rq = run_engine(gk, config(EngineKind::Sequential, 1));
  CHECK(rs.total <= rq.total);
  PartitionPlan plan{{0, 2, 5}};
  auto vr = variance_report(oracles::g5(), plan, 0.5);
  CHECK(vr.triangles == 2 && vr.k == 1 && vr.k_prime == 1 && vr.var == 16.0);
}

TEST_CASE("mirror 6: test_io.cpp:12-24 parse_edge_list basics") {
  auto e = parse_edge_list("0 1\n1 2\n");
  CHECK(e.size() == 2 && e[0] == (std::pair<NodeId, NodeId>{0, 1}) &&
        e[1] == (std::pair<NodeId, NodeId>{1, 2}));
  auto c = parse_edge_list("# comment\n3 4\n");
  CHECK(c.size() == 1 && c[0] == (std::pair<NodeId, NodeId>{3, 4}));
  CHECK(parse_edge_list("").empty());
  CHECK(parse_edge_list("\n  \n# only comments\n").empty());
}

TEST_CASE("mirror 7: test_io.cpp:26-35 errors carry line numbers") {
  bool threw = false;
  try {
    parse_edge_list("0 x\n");
  } catch (const ParseError&) {
    threw = true;
  }
  CHECK(threw);
  std::size_t line = 0;
  try {
    parse_edge_list("0 1\n\n2 y\n");
  } catch (const ParseError& e) {
    line = e.line;
  }
  CHECK(line == 3);
  threw = false;
  try {
    parse_edge_list("1 2 3\n");
  } catch (const ParseError& e) {
    threw = std::string(e.what()) == "line 1: trailing token '3'";
  }
  CHECK(threw);
}

TEST_CASE("mirror 8: test_io.cpp:37-46 round trip") {
  auto g = oracles::g5();
  auto text = write_edge_list(g);
  std::size_t nl = 0;
  for (char ch : text) nl += ch == '\n';
  CHECK(nl == 6);
  auto g2 = build_graph(parse_edge_list(text));
  CHECK(g2.num_nodes() == g.num_nodes() && g2.num_edges() == g.num_edges());
  CHECK(write_edge_list(g2) == text);
  CHECK(write_edge_list(build_graph_from_text(text)) == text);
  CHECK(write_edge_list(build_graph({})).empty());
}

TEST_CASE("mirror 9: test_graph.cpp:51-55 coreness") {
  CHECK((coreness(build_graph({{0, 1}, {0, 2}, {1, 2}})) == std::vector<std::size_t>{2, 2, 2}));
  CHECK((coreness(build_graph({{0, 1}, {1, 2}})) == std::vector<std::size_t>{1, 1, 1}));
  CHECK((coreness(oracles::g5()) == std::vector<std::size_t>{2, 2, 2, 2, 1}));
}

TEST_CASE("mirror 10: test_graph.cpp:67-71, :79-91, :111-116; test_sequential.cpp:84-87") {
  auto g = oracles::g5();
  auto id = compute_order(g, OrderKind::by_id());
  for (NodeId v = 0; v < 5; ++v) CHECK(id.rank[v] == v);
  auto a = compute_order(g, OrderKind::by_random(42));
  auto b = compute_order(g, OrderKind::by_random(42));
  CHECK(a.rank == b.rank);
  auto eff = effective_adjacency(g, OrderKind::by_id());
  CHECK(eff.effdeg(3) == 1 && eff.entries[eff.offsets[3]] == 4 && eff.effdeg(4) == 0);
  CHECK(ordering_cost(g, OrderKind::by_id()) == 16);
  CHECK(ordering_cost(g) == 14);
  for (auto kind : {OrderKind::by_id(), OrderKind::by_degree(), OrderKind::by_random(3),
                    OrderKind::by_coreness()}) {
    CHECK(count_node_iterator_n(g, kind) == 2);
    CHECK(count_node_iterator_pp(g, kind) == 2);          // test_sequential.cpp:20-31
    CHECK(count_node_iterator_pp(g, kind, true) == 2);
    CHECK(effective_adjacency(g, kind).total_entries() == g.num_edges());
    auto cfg = config(EngineKind::AnopSurrogate, 3);
    cfg.order = kind;
    CHECK(run_engine(g, cfg).total == 2);
  }
}

TEST_CASE("mirror 11: a PA graph through every engine: totals and per-rank sums agree") {
  auto g = gen_pa(20000, 20, 3);
  std::uint64_t t = count_node_iterator_n(g);
  for (auto e : {EngineKind::Aop, EngineKind::AnopDirect, EngineKind::AnopSurrogate}) {
    auto r = run_engine(g, config(e, 8));
    std::uint64_t s = 0;
    for (auto& rs : r.per_rank) s += rs.triangles;
    CHECK(r.total == t && s == t);
  }
  std::printf("pa20000 count %llu\n", (unsigned long long)t);
}

int main() {
  int ran = 0;
  for (const auto& c : harness::cases()) {
    const int before = harness::failures;
    try {
      c.fn();
    } catch (const harness::RequireFailed&) {
    } catch (const std::exception& e) {
      std::printf("FAIL %s: exception %s\n", c.name, e.what());
      ++harness::failures;
    }
    std::printf("%s %s\n", harness::failures == before ? "ok  " : "FAIL", c.name);
    ++ran;
  }
  std::printf("%d cases, %s (%d failures)\n", ran, harness::failures ? "FAILED" : "PASSED",
              harness::failures);
  return harness::failures ? 1 : 0;
}
