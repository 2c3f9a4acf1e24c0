// C++ drop-in check: the reference's own test cases (test_engines.cpp,
// test_graph.cpp, test_sequential.cpp) written against the C++ mirror, with
// only the namespace alias changed.  Built by tests/test_abi.py (g++ against
// include/ + libtrigraph_b200.so) and run on the GPU by tests/test_gpu_cpp.py.
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

#include "trigraph_b200/trigraph.hpp"

namespace trigraph = trigraph_b200;
using namespace trigraph;

static int failures = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);     \
      ++failures;                                                  \
    }                                                              \
  } while (0)

static Graph g5() { return build_graph({{0, 1}, {0, 2}, {1, 2}, {1, 3}, {2, 3}, {3, 4}}); }

static EngineConfig config(EngineKind e, std::size_t p, CostKind c = CostKind::Dpd) {
  EngineConfig cfg;
  cfg.engine = e;
  cfg.ranks = p;
  cfg.cost = c;
  return cfg;
}

int main(int argc, char** argv) {
  {  // test_graph.cpp:10-17
    auto g = build_graph({{0, 1}, {1, 0}, {2, 2}});
    CHECK(g.num_nodes() == 3);
    CHECK(g.num_edges() == 1);
  }
  {  // test_graph.cpp:57-64
    auto g = g5();
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
  {  // test_engines.cpp:28-64
    auto g = g5();
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
  {  // test_engines.cpp:90-94, 125-139, 172-175
    std::vector<std::pair<NodeId, NodeId>> k8;
    for (NodeId u = 0; u < 8; ++u)
      for (NodeId v = u + 1; v < 8; ++v) k8.push_back({u, v});
    CHECK(run_engine(build_graph(k8, 8), config(EngineKind::AnopSurrogate, 3, CostKind::Nov)).total == 56);
    auto cc = clustering_coefficients(g5(), config(EngineKind::Aop, 2));
    CHECK((cc.triangles_per_node == std::vector<std::uint64_t>{1, 2, 2, 1, 0}));
    CHECK(cc.coefficient[0] == 1.0 && cc.coefficient[1] == 2.0 / 3.0 && cc.coefficient[4] == 0.0);
    bool threw = false;
    try {
      run_engine(g5(), config(EngineKind::Aop, 0));
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  {  // 8(f) rows: per-edge counts, q = 1 sparsification, variance report
    // (sequential.hpp:108-122, engines.hpp:440-457, sparsify.hpp:113-155)
    auto te = per_edge_triangle_counts(g5());
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
    auto vr = variance_report(g5(), plan, 0.5);
    CHECK(vr.triangles == 2 && vr.k == 1 && vr.k_prime == 1 && vr.var == 16.0);
  }
  {  // test_io.cpp:12-24 parse_edge_list basics
    auto e = parse_edge_list("0 1\n1 2\n");
    CHECK(e.size() == 2 && e[0] == (std::pair<NodeId, NodeId>{0, 1}) &&
          e[1] == (std::pair<NodeId, NodeId>{1, 2}));
    auto c = parse_edge_list("# comment\n3 4\n");
    CHECK(c.size() == 1 && c[0] == (std::pair<NodeId, NodeId>{3, 4}));
    CHECK(parse_edge_list("").empty());
    CHECK(parse_edge_list("\n  \n# only comments\n").empty());
  }
  {  // test_io.cpp:26-35 errors carry line numbers
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
  {  // test_io.cpp:37-46 round trip
    auto g = g5();
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
  {  // test_graph.cpp:51-55 coreness
    CHECK((coreness(build_graph({{0, 1}, {0, 2}, {1, 2}})) == std::vector<std::size_t>{2, 2, 2}));
    CHECK((coreness(build_graph({{0, 1}, {1, 2}})) == std::vector<std::size_t>{1, 1, 1}));
    CHECK((coreness(g5()) == std::vector<std::size_t>{2, 2, 2, 2, 1}));
  }
  {  // test_graph.cpp:67-71, :79-91, :111-116; test_sequential.cpp:84-87
    auto g = g5();
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
  {  // a PA graph through every engine: totals and per-rank sums agree
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
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "PASSED", failures);
  return failures ? 1 : 0;
}
