// prep.cu -- device CSR build, degree-ordered orientation, node costs, plan.
//
// Reference algorithm (paths relative to /root/reference/proj/include/trigraph/):
//   build_graph            graph.hpp:58-85
//   compute_order(ByDegree) order.hpp:95-104
//   effective_adjacency    effective.hpp:37-52
//   node_costs             partition.hpp:45-91
//   compute_boundaries     partition.hpp:116-141
//   ordering_cost          sequential.hpp:95-104
//
// B200 design: everything is a streaming pass over HBM.  build_graph is one
// 64-bit radix sort + unique of directed keys (u<<32|v) (CUB onesweep); the
// degree order needs no sort at all on the hot path: "v precedes u" is the
// comparison (deg v, v) < (deg u, u), evaluated against a 4 B/vertex degree
// array that stays L2-resident (126 MB L2 holds 31M degrees).  Orientation is
// count -> scan -> ballot-compacted fill, which keeps each N_v ID-sorted
// (effective.hpp:13-16).
#include <cub/cub.cuh>

#include "tg_internal.cuh"

namespace tgb {

unsigned long long g_launches = 0;

namespace {

template <class F>
void cub_run(cudaStream_t s, F&& f) {
  size_t bytes = 0;
  TG_CUDA(f((void*)nullptr, bytes));
  DBuf<char> tmp(bytes ? bytes : 1, s);
  TG_CUDA(f((void*)tmp.p, bytes));
}

__device__ __forceinline__ bool precedes(uint32_t dv, uint32_t v, uint32_t du, uint32_t u) {
  // order.hpp:95-104: sort by (degree, id); rank[v] < rank[u]
  return dv < du || (dv == du && v < u);
}

unsigned bitlen(uint64_t x) {
  unsigned b = 0;
  while (x) {
    ++b;
    x >>= 1;
  }
  return b;
}

// ---------------------------------------------------------------- build_graph

__global__ void k_make_keys(const uint32_t* __restrict__ pairs, uint64_t E, uint64_t sentinel,
                            uint64_t* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < E;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint2 e = reinterpret_cast<const uint2*>(pairs)[i];
    uint64_t a = sentinel, b = sentinel;
    if (e.x != e.y) {  // graph.hpp:69 self-loops dropped
      a = ((uint64_t)e.x << 32) | e.y;
      b = ((uint64_t)e.y << 32) | e.x;
    }
    keys[2 * i] = a;
    keys[2 * i + 1] = b;
  }
}

__global__ void k_split_keys(const uint64_t* __restrict__ keys, uint64_t m2,
                             uint32_t* __restrict__ adj) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m2;
       i += (uint64_t)gridDim.x * blockDim.x)
    adj[i] = (uint32_t)keys[i];
}

// off[v] = #keys with src < v  (lower_bound of v<<32)
__global__ void k_offsets_from_keys(const uint64_t* __restrict__ keys, uint64_t m2, uint64_t n,
                                    uint64_t* __restrict__ off) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v <= n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t target = v << 32, lo = 0, hi = m2;
    while (lo < hi) {
      uint64_t mid = (lo + hi) >> 1;
      if (keys[mid] < target) lo = mid + 1;
      else hi = mid;
    }
    off[v] = lo;
  }
}

__global__ void k_degrees(const uint64_t* __restrict__ off, uint64_t n, uint32_t* __restrict__ deg) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x)
    deg[v] = (uint32_t)(off[v + 1] - off[v]);
}

// ---------------------------------------------------------------- orientation

// G lanes per vertex.  Pass 0 counts h_v; pass 1 writes the ID-sorted N_v
// (ballot prefix keeps adjacency order).
template <int G, bool FILL>
__global__ void __launch_bounds__(256)
k_orient(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
         const uint32_t* __restrict__ deg, uint32_t vlo, uint32_t vhi,
         uint64_t* __restrict__ cnt_or_off, uint32_t* __restrict__ eff) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned sub = lane & (G - 1);
  const unsigned gbase = lane & ~(G - 1);
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << gbase);
  const uint64_t groups = ((uint64_t)gridDim.x * blockDim.x) / G;
  for (uint64_t g = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / G;; g += groups) {
    // all lanes of a warp iterate together so __ballot_sync stays legal
    uint64_t vv = vlo + g;
    bool active = vv < vhi;
    if (__all_sync(0xffffffffu, !active)) break;
    uint32_t v = active ? (uint32_t)vv : 0;
    uint64_t b = active ? off[v] : 0, e = active ? off[v + 1] : 0;
    uint32_t dv = active ? deg[v] : 0;
    uint64_t wpos = FILL && active ? cnt_or_off[v - vlo] : 0;
    uint64_t c = 0;
    uint64_t len = e - b;
    // uniform trip count across the warp
    uint64_t mylen = len, maxlen = len;
    for (int o = 16; o > 0; o >>= 1) {
      uint64_t t = __shfl_xor_sync(0xffffffffu, maxlen, o);
      maxlen = t > maxlen ? t : maxlen;
    }
    for (uint64_t k0 = 0; k0 < maxlen; k0 += G) {
      uint64_t k = k0 + sub;
      bool keep = false;
      uint32_t u = 0;
      if (k < mylen) {
        u = adj[b + k];
        keep = precedes(dv, v, deg[u], u);
      }
      unsigned bal = __ballot_sync(0xffffffffu, keep) & gmask;
      if (FILL && keep) {
        unsigned before = __popc(bal & ((1u << lane) - 1u));
        eff[wpos + c + before] = u;
      }
      c += __popc(bal);
    }
    if (!FILL && active && sub == 0) cnt_or_off[v - vlo] = c;
  }
}

template <int G>
void launch_orient(const DevGraph& g, uint32_t vlo, uint32_t vhi, uint64_t* cnt, uint64_t* off_out,
                   uint32_t* eff, cudaStream_t s) {
  uint64_t rows = vhi - vlo;
  unsigned grid = grid_for(rows * G, 256, 148u * 32u);
  k_orient<G, false><<<grid, 256, 0, s>>>(g.off.p, g.adj.p, g.deg.p, vlo, vhi, cnt, nullptr);
  TG_CHECK_LAUNCH();
  ++g_launches;
  // exclusive scan into off_out[0..rows]
  TG_CUDA(cudaMemsetAsync(off_out, 0, sizeof(uint64_t), s));
  if (rows) {
    cub_run(s, [&](void* t, size_t& b) {
      return cub::DeviceScan::InclusiveSum(t, b, cnt, off_out + 1, (int64_t)rows, s);
    });
    g_launches += 2;  // CUB decoupled look-back scan: init + scan kernels
    k_orient<G, true><<<grid, 256, 0, s>>>(g.off.p, g.adj.p, g.deg.p, vlo, vhi, off_out, eff);
    TG_CHECK_LAUNCH();
    ++g_launches;
  }
}

// ---------------------------------------------------------------- costs

__global__ void k_cost_simple(const uint64_t* __restrict__ eoff, const uint32_t* __restrict__ deg,
                              uint64_t n, int kind, uint64_t* __restrict__ f) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t d = deg[v], h = eoff[v + 1] - eoff[v], r = 0;
    switch (kind) {
      case TG_COST_N: r = 1; break;
      case TG_COST_D: r = d; break;
      case TG_COST_DH: r = h; break;
      case TG_COST_DDH: r = d * h; break;
      case TG_COST_DH2: r = h * h; break;
      default: r = 0;
    }
    f[v] = r;
  }
}

// DPD (partition.hpp:60-69): sum_{u in N_v} (h_v + h_u)
// NOV (partition.hpp:70-81): sum_{u in adj(v), u precedes v} (h_v + h_u)
template <bool NOV>
__global__ void __launch_bounds__(256)
k_cost_sum(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
           const uint32_t* __restrict__ deg, const uint64_t* __restrict__ eoff,
           const uint32_t* __restrict__ eff, uint64_t n, uint64_t* __restrict__ f) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t v = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; v < n; v += warps) {
    uint64_t hv = eoff[v + 1] - eoff[v];
    uint64_t b, e;
    if (NOV) { b = off[v]; e = off[v + 1]; }
    else { b = eoff[v]; e = eoff[v + 1]; }
    uint32_t dv = deg[v];
    uint64_t s = 0;
    for (uint64_t k = b + lane; k < e; k += 32) {
      uint32_t u = NOV ? adj[k] : eff[k];
      if (!NOV || precedes(deg[u], u, dv, (uint32_t)v)) s += hv + (eoff[u + 1] - eoff[u]);
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) f[v] = s;
  }
}

__global__ void k_boundaries(const uint64_t* __restrict__ prefix, uint64_t n, uint64_t p,
                             uint32_t* __restrict__ b) {
  // partition.hpp:128-138, one thread per inner boundary.  Searching [0, n]
  // instead of [b_{j-1}, n] gives the same smallest x because the predicate
  // is monotone in x.
  uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (j == 0) b[0] = 0;
  if (j == 0) b[p] = (uint32_t)n;
  if (j == 0 || j >= p) return;
  uint64_t total = n ? prefix[n - 1] : 0;
  unsigned __int128 target = (unsigned __int128)j * total;
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    uint64_t before = mid == 0 ? 0 : prefix[mid - 1];
    if ((unsigned __int128)p * before >= target) hi = mid;
    else lo = mid + 1;
  }
  b[j] = (uint32_t)lo;
}

__global__ void k_ordering_cost(const uint32_t* __restrict__ deg, const uint64_t* __restrict__ eoff,
                                uint64_t n, unsigned long long* __restrict__ out) {
  uint64_t s = 0;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x)
    s += (uint64_t)deg[v] * (eoff[v + 1] - eoff[v]);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, (unsigned long long)s);
}

__global__ void k_rank_keys(const uint32_t* __restrict__ deg, uint64_t n, uint64_t* __restrict__ k) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x)
    k[v] = ((uint64_t)deg[v] << 32) | v;
}

__global__ void k_rank_scatter(const uint64_t* __restrict__ k, uint64_t n, uint32_t* __restrict__ rank) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    rank[(uint32_t)k[i]] = (uint32_t)i;
}

}  // namespace

// graph.hpp:58-85 on the device.
void build_graph_device(const uint32_t* d_pairs, uint64_t E, uint64_t n_override, DevGraph& g,
                        cudaStream_t s) {
  uint64_t n = n_override;
  if (E) {
    DBuf<uint32_t> mx(1, s);
    cub_run(s, [&](void* t, size_t& b) {
      return cub::DeviceReduce::Max(t, b, d_pairs, mx.p, (int64_t)(2 * E), s);
    });
    ++g_launches;
    uint32_t h = 0;
    TG_CUDA(cudaMemcpyAsync(&h, mx.p, 4, cudaMemcpyDeviceToHost, s));
    TG_CUDA(cudaStreamSynchronize(s));
    if ((uint64_t)h + 1 > n) n = (uint64_t)h + 1;
  }
  TG_REQUIRE(n <= 0xFFFFFFFFull, "build_graph: node ids must fit NodeId (uint32) with n < 2^32");
  g.n = n;
  uint64_t keys_n = 2 * E;
  uint64_t sentinel = n << 32;  // sorts after every real key (src < n)
  unsigned end_bit = 32 + bitlen(n);
  if (end_bit > 64) end_bit = 64;
  DBuf<uint64_t> k1(keys_n ? keys_n : 1, s), k2(keys_n ? keys_n : 1, s);
  uint64_t m2 = 0;
  if (E) {
    k_make_keys<<<grid_for(E, 256), 256, 0, s>>>(d_pairs, E, sentinel, k1.p);
    TG_CHECK_LAUNCH();
    ++g_launches;
    cub_run(s, [&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortKeys(t, b, k1.p, k2.p, (int64_t)keys_n, 0, (int)end_bit, s);
    });
    ++g_launches;
    DBuf<int64_t> nsel(1, s);
    cub_run(s, [&](void* t, size_t& b) {
      return cub::DeviceSelect::Unique(t, b, k2.p, k1.p, nsel.p, (int64_t)keys_n, s);
    });
    ++g_launches;
    int64_t u = 0;
    uint64_t last = 0;
    TG_CUDA(cudaMemcpyAsync(&u, nsel.p, 8, cudaMemcpyDeviceToHost, s));
    TG_CUDA(cudaStreamSynchronize(s));
    if (u > 0) {
      TG_CUDA(cudaMemcpyAsync(&last, k1.p + (u - 1), 8, cudaMemcpyDeviceToHost, s));
      TG_CUDA(cudaStreamSynchronize(s));
    }
    m2 = (uint64_t)u - ((u > 0 && last == sentinel) ? 1 : 0);
  }
  g.m2 = m2;
  g.off.alloc(n + 1, s);
  g.adj.alloc(m2 ? m2 : 1, s);
  if (m2) {
    k_split_keys<<<grid_for(m2, 256), 256, 0, s>>>(k1.p, m2, g.adj.p);
    TG_CHECK_LAUNCH();
    ++g_launches;
  }
  k_offsets_from_keys<<<grid_for(n + 1, 256), 256, 0, s>>>(k1.p, m2, n, g.off.p);
  TG_CHECK_LAUNCH();
  ++g_launches;
  compute_degrees(g, s);
}

void compute_degrees(DevGraph& g, cudaStream_t s) {
  g.deg.alloc(g.n ? g.n : 1, s);
  if (g.n) {
    k_degrees<<<grid_for(g.n, 256), 256, 0, s>>>(g.off.p, g.n, g.deg.p);
    TG_CHECK_LAUNCH();
    ++g_launches;
  }
}

// effective.hpp:37-52 for rows [vlo, vhi).  No host sync: sum of h over all
// rows is m when vlo = 0 and vhi = n; for a partial range the caller learns
// `entries` from the scanned offsets (one 8-byte D2H).
void orient_rows(const DevGraph& g, uint32_t vlo, uint32_t vhi, DevEff& out, cudaStream_t s) {
  uint64_t rows = vhi - vlo;
  out.rows = rows;
  out.base = vlo;
  out.off.alloc(rows + 1, s);
  DBuf<uint64_t> cnt(rows ? rows : 1, s);
  uint64_t entries;
  bool full = (vlo == 0 && vhi == g.n);
  // data buffer: exact size for the full graph (sum h = m), else bound by the
  // symmetric entries of the range
  uint64_t bound = full ? g.m2 / 2 : 0;
  if (!full) {
    uint64_t ob[2];
    TG_CUDA(cudaMemcpyAsync(&ob[0], g.off.p + vlo, 8, cudaMemcpyDeviceToHost, s));
    TG_CUDA(cudaMemcpyAsync(&ob[1], g.off.p + vhi, 8, cudaMemcpyDeviceToHost, s));
    TG_CUDA(cudaStreamSynchronize(s));
    bound = ob[1] - ob[0];
  }
  out.data.alloc(bound ? bound : 1, s);
  uint64_t avg = g.n ? g.m2 / g.n : 0;
  if (avg <= 12) launch_orient<8>(g, vlo, vhi, cnt.p, out.off.p, out.data.p, s);
  else if (avg <= 24) launch_orient<16>(g, vlo, vhi, cnt.p, out.off.p, out.data.p, s);
  else launch_orient<32>(g, vlo, vhi, cnt.p, out.off.p, out.data.p, s);
  if (full) {
    entries = g.m2 / 2;
  } else {
    TG_CUDA(cudaMemcpyAsync(&entries, out.off.p + rows, 8, cudaMemcpyDeviceToHost, s));
    TG_CUDA(cudaStreamSynchronize(s));
  }
  out.entries = entries;
}

// order.hpp:95-104: rank = position in the (degree, id) sort.
void degree_rank(const DevGraph& g, uint32_t* d_rank, cudaStream_t s) {
  if (!g.n) return;
  DBuf<uint64_t> k1(g.n, s), k2(g.n, s);
  k_rank_keys<<<grid_for(g.n, 256), 256, 0, s>>>(g.deg.p, g.n, k1.p);
  TG_CHECK_LAUNCH();
  ++g_launches;
  cub_run(s, [&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortKeys(t, b, k1.p, k2.p, (int64_t)g.n, 0, 64, s);
  });
  ++g_launches;
  k_rank_scatter<<<grid_for(g.n, 256), 256, 0, s>>>(k2.p, g.n, d_rank);
  TG_CHECK_LAUNCH();
  ++g_launches;
}

void node_costs_device(const DevGraph& g, const DevEff& eff, int kind, uint64_t* d_f,
                       uint64_t* d_prefix, cudaStream_t s) {
  TG_REQUIRE(kind >= TG_COST_N && kind <= TG_COST_NOV, "node_costs: unknown cost kind");
  if (!g.n) return;
  if (kind == TG_COST_DPD || kind == TG_COST_NOV) {
    unsigned grid = grid_for(g.n * 32, 256, 148u * 32u);
    if (kind == TG_COST_DPD)
      k_cost_sum<false><<<grid, 256, 0, s>>>(g.off.p, g.adj.p, g.deg.p, eff.off.p, eff.data.p, g.n, d_f);
    else
      k_cost_sum<true><<<grid, 256, 0, s>>>(g.off.p, g.adj.p, g.deg.p, eff.off.p, eff.data.p, g.n, d_f);
  } else {
    k_cost_simple<<<grid_for(g.n, 256), 256, 0, s>>>(eff.off.p, g.deg.p, g.n, kind, d_f);
  }
  TG_CHECK_LAUNCH();
  ++g_launches;
  cub_run(s, [&](void* t, size_t& b) {
    return cub::DeviceScan::InclusiveSum(t, b, d_f, d_prefix, (int64_t)g.n, s);
  });
  ++g_launches;
}

std::vector<uint32_t> boundaries_from_prefix(const uint64_t* d_prefix, uint64_t n, uint64_t p,
                                             cudaStream_t s) {
  TG_REQUIRE(p >= 1, "compute_boundaries: p must be >= 1");
  DBuf<uint32_t> b(p + 1, s);
  k_boundaries<<<grid_for(p, 128), 128, 0, s>>>(d_prefix, n, p, b.p);
  TG_CHECK_LAUNCH();
  ++g_launches;
  std::vector<uint32_t> h(p + 1);
  TG_CUDA(cudaMemcpyAsync(h.data(), b.p, (p + 1) * 4, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  return h;
}

uint64_t ordering_cost_device(const DevGraph& g, const DevEff& eff, cudaStream_t s) {
  DBuf<unsigned long long> acc(1, s);
  acc.zero();
  if (g.n) {
    k_ordering_cost<<<grid_for(g.n, 256, 148u * 8u), 256, 0, s>>>(g.deg.p, eff.off.p, g.n, acc.p);
    TG_CHECK_LAUNCH();
    ++g_launches;
  }
  unsigned long long h = 0;
  TG_CUDA(cudaMemcpyAsync(&h, acc.p, 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  return h;
}

}  // namespace tgb
