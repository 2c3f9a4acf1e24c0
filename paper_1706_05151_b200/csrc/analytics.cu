// analytics.cu -- per-edge triangle counts and the sparsification variance
// analytics, and the NodeIterator++ baseline.
//
// Reference (paths relative to /root/reference/proj/include/trigraph/):
//   count_node_iterator_pp     sequential.hpp:48-70
//   per_edge_triangle_counts   sequential.hpp:108-122
//   variance_report            sparsify.hpp:113-155
//   Graph::edges() order       graph.hpp:40-46
//
// t_e is accumulated from the exact triangle listing (the LIST sink of the
// intersection kernels, in apex ranges whose listing fits a bounded
// buffer): each listed triple (a < b < c) bumps its three edges, whose index
// in edges() order is up[x] + #{neighbours of x below y} - #{below x} (two
// binary searches in the ID-sorted symmetric adjacency).  One thread per
// triple, 64-bit atomics; k = sum_e t_e (t_e - 1) / 2 is a reduction.
#include <cub/cub.cuh>

#include "tg_internal.cuh"

namespace tgb {
namespace {

__device__ __forceinline__ uint64_t lb_u32(const uint32_t* __restrict__ a, uint64_t n, uint32_t x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ bool has_in(const uint32_t* __restrict__ a, uint64_t b, uint64_t e,
                                       uint32_t x) {
  while (b < e) {
    const uint64_t mid = (b + e) >> 1;
    const uint32_t y = a[mid];
    if (y == x) return true;
    if (y < x) b = mid + 1;
    else e = mid;
  }
  return false;
}

__device__ __forceinline__ bool key_precedes(uint32_t kv, uint32_t v, uint32_t ku, uint32_t u) {
  return kv < ku || (kv == ku && v < u);
}

// NodeIterator++ (sequential.hpp:51-70) on the symmetric adjacency: a warp
// per v walks its neighbours u with v < u in the order; lanes split adj(v)
// and test each w with u < w for membership in adj(u) (Graph::has_edge, a
// binary search, graph.hpp:34-38).  `key` is the order key (degree, or the
// rank of a non-degree order).
__global__ void __launch_bounds__(256)
k_node_iterator_pp(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                   const uint32_t* __restrict__ key, uint64_t n,
                   unsigned long long* __restrict__ total) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  uint64_t c = 0;
  for (uint64_t v = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; v < n; v += warps) {
    const uint32_t kv = key[v];
    const uint64_t b = off[v], e = off[v + 1];
    for (uint64_t j = b; j < e; ++j) {
      const uint32_t u = adj[j];
      const uint32_t ku = key[u];
      if (!key_precedes(kv, (uint32_t)v, ku, u)) continue;
      const uint64_t ub = off[u], ue = off[u + 1];
      for (uint64_t k = b + lane; k < e; k += 32) {
        const uint32_t w = adj[k];
        if (key_precedes(ku, u, key[w], w) && has_in(adj, ub, ue, w)) ++c;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0 && c) atomicAdd(total, (unsigned long long)c);
}

// #neighbours above v (edges() emits (v, u) for u > v)
__global__ void k_upper_deg(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                            uint64_t n, uint64_t* __restrict__ cnt) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = off[v], d = off[v + 1] - b;
    cnt[v] = d - lb_u32(adj + b, d, (uint32_t)v);
  }
}

__device__ __forceinline__ uint64_t edge_index(const uint64_t* __restrict__ off,
                                               const uint32_t* __restrict__ adj,
                                               const uint64_t* __restrict__ up, uint32_t x,
                                               uint32_t y) {  // x < y
  const uint64_t b = off[x], d = off[x + 1] - b;
  return up[x] + lb_u32(adj + b, d, y) - lb_u32(adj + b, d, x);
}

__global__ void k_bump_edges(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                             const uint64_t* __restrict__ up, const uint32_t* __restrict__ tri,
                             uint64_t cnt, unsigned long long* __restrict__ te,
                             unsigned long long* __restrict__ te2) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < cnt;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t a = tri[3 * t], b = tri[3 * t + 1], c = tri[3 * t + 2];  // a < b < c
    const uint64_t e[3] = {edge_index(off, adj, up, a, b), edge_index(off, adj, up, a, c),
                           edge_index(off, adj, up, b, c)};
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      atomicAdd(te + e[i], 1ull);
      if (te2) atomicAdd(te2 + e[i], 1ull);
    }
  }
}

__global__ void k_choose2(const unsigned long long* __restrict__ te, uint64_t m,
                          unsigned long long* __restrict__ acc) {
  unsigned long long s = 0;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long c = te[e];
    s += c ? c * (c - 1) / 2 : 0ull;
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(acc, s);
}

}  // namespace

uint64_t node_iterator_pp_device(const DevGraph& g, cudaStream_t s) {
  DBuf<unsigned long long> acc(1, s);
  acc.zero();
  if (g.n) {
    k_node_iterator_pp<<<grid_for(g.n * 32, 256, 148u * 32u), 256, 0, s>>>(g.off.p, g.adj.p,
                                                                          order_key(g), g.n, acc.p);
    TG_CHECK_LAUNCH();
    ++g_launches;
  }
  unsigned long long h = 0;
  TG_CUDA(cudaMemcpyAsync(&h, acc.p, 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  return h;
}

void upper_offsets(const DevGraph& g, uint64_t* d_up, cudaStream_t s) {
  TG_CUDA(cudaMemsetAsync(d_up, 0, 8, s));
  if (!g.n) return;
  DBuf<uint64_t> cnt(g.n, s);
  k_upper_deg<<<grid_for(g.n, 256), 256, 0, s>>>(g.off.p, g.adj.p, g.n, cnt.p);
  TG_CHECK_LAUNCH();
  size_t bytes = 0;
  TG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, cnt.p, d_up + 1, (int64_t)g.n, s));
  DBuf<char> tmp(bytes ? bytes : 1, s);
  TG_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, bytes, cnt.p, d_up + 1, (int64_t)g.n, s));
  g_launches += 3;
}

void bump_edges(const DevGraph& g, const uint64_t* d_up, const uint32_t* d_tri, uint64_t cnt,
                unsigned long long* d_te, unsigned long long* d_te2, cudaStream_t s) {
  if (!cnt) return;
  k_bump_edges<<<grid_for(cnt, 256, 148u * 32u), 256, 0, s>>>(g.off.p, g.adj.p, d_up, d_tri, cnt,
                                                               d_te, d_te2);
  TG_CHECK_LAUNCH();
  ++g_launches;
}

uint64_t sum_choose2(const unsigned long long* d_te, uint64_t m, cudaStream_t s) {
  if (!m) return 0;
  DBuf<unsigned long long> acc(1, s);
  acc.zero();
  k_choose2<<<grid_for(m, 256, 148u * 16u), 256, 0, s>>>(d_te, m, acc.p);
  TG_CHECK_LAUNCH();
  ++g_launches;
  unsigned long long h = 0;
  TG_CUDA(cudaMemcpyAsync(&h, acc.p, 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  return h;
}

}  // namespace tgb
