// One C++ host driving N ranks through the C ABI (csrc/comm.cu): a thread
// per rank, each with its rank-local rows of the graph (tg_graph_from_rows),
// running run_engine across the ranks (AOP, ANOP-direct and ANOP-surrogate,
// engines.hpp:38-54, 80-141, 146-198), the AOP step and clustering at the owners.
// Checked against the single-device count of the whole graph.
//
//   comm_main <nranks> [local|nccl]
// local: in-process transport, every rank on device 0 (this box has one
// GPU); nccl: one NCCL communicator per rank on devices 0..nranks-1 (an
// N-GPU node).  Built and run by tests/test_gpu_cpp.py.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "trigraph_b200.h"

#define CK(x)                                                                      \
  do {                                                                             \
    tg_status _s = (x);                                                            \
    if (_s != TG_OK) {                                                             \
      std::fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #x, tg_last_error()); \
      std::exit(2);                                                                \
    }                                                                              \
  } while (0)

int main(int argc, char** argv) {
  const int N = argc > 1 ? std::atoi(argv[1]) : 2;
  const bool use_nccl = argc > 2 && std::string(argv[2]) == "nccl";
  // the workload: gen_pa (io.hpp:129-162) on the host, one CSR
  uint32_t* pairs = nullptr;
  uint64_t E = 0;
  const uint64_t n = 30000;
  CK(tg_gen_pa(n, 20, 11, &pairs, &E));
  tg_graph* whole = nullptr;
  CK(tg_graph_from_edges(0, pairs, E, n, &whole));
  tg_free_host(pairs);
  uint64_t nn = 0, m = 0, want = 0;
  CK(tg_graph_info(whole, &nn, &m));
  std::vector<uint64_t> off(nn + 1);
  std::vector<uint32_t> adj(2 * m);
  CK(tg_graph_csr(whole, off.data(), adj.data()));
  CK(tg_count(whole, &want));
  CK(tg_graph_free(whole));
  std::vector<uint32_t> deg(nn);
  for (uint64_t v = 0; v < nn; ++v) deg[v] = (uint32_t)(off[v + 1] - off[v]);
  // input distribution: equal adjacency volume per rank
  std::vector<uint32_t> rows(N + 1, 0);
  for (int r = 1; r < N; ++r) {
    const uint64_t target = off[nn] * r / N;
    uint32_t v = 0;
    while (off[v] < target) ++v;
    rows[r] = v;
  }
  rows[N] = (uint32_t)nn;
  // communicators
  std::vector<tg_comm*> comms(N, nullptr);
  if (use_nccl) {
    unsigned char id[128];
    CK(tg_comm_unique_id(id));
    std::vector<std::thread> th;
    for (int r = 0; r < N; ++r)
      th.emplace_back([&, r] { CK(tg_comm_init(r, N, r, id, &comms[r])); });
    for (auto& t : th) t.join();
  } else {
    std::vector<int> devs(N, 0);
    CK(tg_comm_init_local(N, devs.data(), comms.data()));
  }
  std::vector<uint64_t> aop(N), sur(N), dir(N), step(N), stored(N), tsum(N);
  std::vector<int> ok(N, 0);
  std::vector<std::thread> th;
  for (int r = 0; r < N; ++r)
    th.emplace_back([&, r] {
      const int dev = use_nccl ? r : 0;
      const uint32_t lo = rows[r], hi = rows[r + 1];
      tg_graph* g = nullptr;
      CK(tg_graph_from_rows(dev, nn, lo, hi, off.data() + lo, adj.data() + off[lo], deg.data(), &g));
      tg_config cfg{};
      cfg.engine = TG_ENGINE_AOP;
      cfg.cost = TG_COST_DPD;
      std::vector<tg_rank_stats> st(N);
      std::vector<uint32_t> b(N + 1);
      CK(tg_run_engine_comm(g, comms[r], &cfg, &aop[r], st.data(), b.data()));
      // ANOP-direct (engines.hpp:80-141): request / reply data path; as many
      // requests + replies sent as received over the whole job
      cfg.engine = TG_ENGINE_ANOP_DIRECT;
      CK(tg_run_engine_comm(g, comms[r], &cfg, &dir[r], st.data(), nullptr));
      uint64_t ds = 0, dr = 0;
      for (int i = 0; i < N; ++i) {
        ds += st[i].data_sent;
        dr += st[i].data_recv;
      }
      if (ds != dr) dir[r] = ~0ull;
      cfg.engine = TG_ENGINE_ANOP_SURROGATE;
      CK(tg_run_engine_comm(g, comms[r], &cfg, &sur[r], st.data(), nullptr));
      stored[r] = 0;
      tsum[r] = 0;
      for (int i = 0; i < N; ++i) {
        stored[r] += st[i].stored_entries;
        tsum[r] += st[i].triangles;
      }
      uint64_t* d = nullptr;
      if (cudaMalloc((void**)&d, 8) == cudaSuccess) {
        CK(tg_aop_step_comm(g, comms[r], b.data(), d));
        cudaMemcpy(&step[r], d, 8, cudaMemcpyDeviceToHost);
        cudaFree(d);
      }
      std::vector<uint64_t> tv(nn);
      std::vector<double> cc(nn);
      CK(tg_clustering_comm(g, comms[r], &cfg, b.data(), tv.data(), cc.data()));
      ok[r] = 1;
      CK(tg_graph_free(g));
    });
  for (auto& t : th) t.join();
  int failures = 0;
  for (int r = 0; r < N; ++r) {
    if (!ok[r] || aop[r] != want || sur[r] != want || dir[r] != want || step[r] != want || tsum[r] != want ||
        stored[r] != m) {
      std::printf("FAIL rank %d: aop %llu sur %llu step %llu per-rank sum %llu stored %llu "
                  "(want %llu, m %llu)\n",
                  r, (unsigned long long)aop[r], (unsigned long long)sur[r],
                  (unsigned long long)step[r], (unsigned long long)tsum[r],
                  (unsigned long long)stored[r], (unsigned long long)want, (unsigned long long)m);
      ++failures;
    }
  }
  for (auto* c : comms) tg_comm_free(c);
  std::printf("%d ranks (%s), T = %llu: %s (%d failures)\n", N, use_nccl ? "nccl" : "local",
              (unsigned long long)want, failures ? "FAILED" : "PASSED", failures);
  return failures ? 1 : 0;
}
