// order.cu -- the reference's non-degree total orders on the device
// (order.hpp:17-128): ById, ByRandom(seed), ByCoreness.
//
// The orientation kernels (prep.cu) test precedes(v, u) as
// (key_v, v) < (key_u, u).  ByDegree keys on the degree; every other order
// keys on its rank array (a permutation, so ties never reach the id), which
// the functions below build into DevGraph::okey.
//
//  * ById      (order.hpp:90-93)   rank = id.
//  * ByRandom  (order.hpp:104-113) Fisher-Yates over mt19937_64(seed) with a
//    modulo draw.  Inherently sequential (each swap depends on the previous
//    draws), so it runs on the host with the standard engine and the rank is
//    uploaded: O(n), ~0.1 s at n = 1e7.
//  * ByCoreness (order.hpp:39-83, :114-124) core numbers by parallel
//    peeling, then a stable CUB radix sort of ids by (core, degree).
//    Core numbers are unique, so the level-synchronous peel below gives the
//    same values as the reference's sequential bucket algorithm: at level k
//    every live vertex with current degree <= k gets core k and decrements
//    its live neighbours; a neighbour whose degree falls from k+1 to k joins
//    the next frontier (exactly one decrement sees that transition).  Levels
//    advance to the minimum live degree.
#include <cub/cub.cuh>

#include <algorithm>
#include <numeric>
#include <random>

#include "tg_internal.cuh"

namespace tgb {

namespace {

constexpr uint32_t kUnset = 0xffffffffu;

template <class F>
void cub_call(cudaStream_t s, F&& f) {
  size_t bytes = 0;
  TG_CUDA(f(nullptr, bytes));
  DBuf<unsigned char> tmp(bytes ? bytes : 1, s);
  TG_CUDA(f(tmp.p, bytes));
}

__global__ void k_iota(uint32_t* __restrict__ r, uint64_t n) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x)
    r[v] = (uint32_t)v;
}

__global__ void k_core_init(const uint32_t* __restrict__ deg, uint64_t n, uint32_t* __restrict__ cur,
                            uint32_t* __restrict__ core) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    cur[v] = deg[v];
    core[v] = kUnset;
  }
}

// minimum current degree over live vertices
__global__ void k_min_live(const uint32_t* __restrict__ cur, const uint32_t* __restrict__ core,
                           uint64_t n, unsigned* __restrict__ out) {
  uint32_t m = kUnset;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x)
    if (core[v] == kUnset) m = min(m, cur[v]);
  for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m != kUnset) atomicMin(out, m);
}

// live vertices with current degree <= k: core k, into the frontier
__global__ void k_frontier(const uint32_t* __restrict__ cur, uint32_t* __restrict__ core, uint64_t n,
                           uint32_t k, uint32_t* __restrict__ q, unsigned long long* __restrict__ qn) {
  const unsigned lane = threadIdx.x & 31;
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x + (threadIdx.x & ~31u); base < n;
       base += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = base + lane;
    const bool take = v < n && core[v] == kUnset && cur[v] <= k;
    const unsigned bal = __ballot_sync(0xffffffffu, take);
    if (!bal) continue;
    unsigned long long at = 0;
    if (lane == 0) at = atomicAdd(qn, (unsigned long long)__popc(bal));
    at = __shfl_sync(0xffffffffu, at, 0);
    if (take) {
      core[v] = k;
      q[at + __popc(bal & ((1u << lane) - 1u))] = (uint32_t)v;
    }
  }
}

// one warp per frontier vertex: decrement live neighbours; a k+1 -> k
// transition puts the neighbour in the next frontier with core k
__global__ void k_peel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                       const uint32_t* __restrict__ q, uint64_t qn, uint32_t* __restrict__ core,
                       uint32_t* __restrict__ cur, uint32_t k, uint32_t* __restrict__ q2,
                       unsigned long long* __restrict__ q2n) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < qn; i += warps) {
    const uint32_t v = q[i];
    const uint64_t b = off[v], e = off[v + 1];
    for (uint64_t j = b + lane; j < e; j += 32) {
      const uint32_t u = adj[j];
      if (__ldcg(core + u) != kUnset) continue;
      const uint32_t old = atomicSub(cur + u, 1u);
      if (old == k + 1) {
        core[u] = k;
        q2[atomicAdd(q2n, 1ull)] = u;
      }
    }
  }
}

__global__ void k_core_keys(const uint32_t* __restrict__ core, const uint32_t* __restrict__ deg,
                            uint64_t n, uint64_t* __restrict__ key, uint32_t* __restrict__ ids) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    key[v] = ((uint64_t)core[v] << 32) | deg[v];
    ids[v] = (uint32_t)v;
  }
}

__global__ void k_rank_from_sorted(const uint32_t* __restrict__ ids, uint64_t n,
                                   uint32_t* __restrict__ rank) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    rank[ids[i]] = (uint32_t)i;
}

uint64_t read_u64(const unsigned long long* d, cudaStream_t s) {
  unsigned long long h = 0;
  TG_CUDA(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  return h;
}

}  // namespace

void coreness_device(const DevGraph& g, uint32_t* d_core, cudaStream_t s) {
  const uint64_t n = g.n;
  if (!n) return;
  DBuf<uint32_t> cur(n, s), q0(n, s), q1(n, s);
  DBuf<unsigned long long> ctr(2, s);
  DBuf<unsigned> kmin(1, s);
  const unsigned grid = grid_for(n, 256);
  k_core_init<<<grid, 256, 0, s>>>(g.deg.p, n, cur.p, d_core);
  TG_CHECK_LAUNCH();
  ++g_launches;
  uint64_t remaining = n;
  uint32_t k = 0;
  while (remaining) {
    TG_CUDA(cudaMemsetAsync(kmin.p, 0xff, sizeof(unsigned), s));
    k_min_live<<<grid, 256, 0, s>>>(cur.p, d_core, n, kmin.p);
    TG_CHECK_LAUNCH();
    ++g_launches;
    unsigned km = 0;
    TG_CUDA(cudaMemcpyAsync(&km, kmin.p, 4, cudaMemcpyDeviceToHost, s));
    TG_CUDA(cudaStreamSynchronize(s));
    if (km == kUnset) throw Error(TG_ERR_INTERNAL, "coreness: live vertices without a degree");
    k = std::max(k, km);
    TG_CUDA(cudaMemsetAsync(ctr.p, 0, 8, s));
    k_frontier<<<grid, 256, 0, s>>>(cur.p, d_core, n, k, q0.p, ctr.p);
    TG_CHECK_LAUNCH();
    ++g_launches;
    uint64_t qn = read_u64(ctr.p, s);
    if (!qn) throw Error(TG_ERR_INTERNAL, "coreness: empty frontier at a live level");
    uint32_t* qa = q0.p;
    uint32_t* qb = q1.p;
    while (qn) {
      if (qn > remaining) throw Error(TG_ERR_INTERNAL, "coreness: frontier overflow");
      remaining -= qn;
      TG_CUDA(cudaMemsetAsync(ctr.p + 1, 0, 8, s));
      k_peel<<<grid_for(qn * 32, 256, 148u * 32u), 256, 0, s>>>(g.off.p, g.adj.p, qa, qn, d_core,
                                                               cur.p, k, qb, ctr.p + 1);
      TG_CHECK_LAUNCH();
      ++g_launches;
      qn = read_u64(ctr.p + 1, s);
      std::swap(qa, qb);
    }
  }
}

void set_order(DevGraph& g, int kind, uint64_t seed, cudaStream_t s) {
  TG_REQUIRE(kind >= TG_ORDER_BY_ID && kind <= TG_ORDER_BY_CORENESS, "unknown order kind");
  const uint64_t n = g.n;
  g.order = kind;
  g.order_seed = kind == TG_ORDER_BY_RANDOM ? seed : 0;
  if (kind == TG_ORDER_BY_DEGREE) {
    g.okey.release();
    return;
  }
  g.okey.alloc(n ? n : 1, s);
  if (!n) return;
  if (kind == TG_ORDER_BY_ID) {
    k_iota<<<grid_for(n, 256), 256, 0, s>>>(g.okey.p, n);
    TG_CHECK_LAUNCH();
    ++g_launches;
  } else if (kind == TG_ORDER_BY_RANDOM) {
    // order.hpp:104-113, bit-exact: the standard engine, modulo draw
    std::vector<uint32_t> nodes(n), rank(n);
    std::iota(nodes.begin(), nodes.end(), 0u);
    std::mt19937_64 rng(seed);
    for (uint64_t i = n; i > 1; --i) std::swap(nodes[i - 1], nodes[rng() % i]);
    for (uint64_t i = 0; i < n; ++i) rank[nodes[i]] = (uint32_t)i;
    TG_CUDA(cudaMemcpyAsync(g.okey.p, rank.data(), n * 4, cudaMemcpyHostToDevice, s));
    TG_CUDA(cudaStreamSynchronize(s));  // `rank` dies at scope exit
  } else {
    DBuf<uint32_t> core(n, s), ids(n, s), ids2(n, s);
    DBuf<uint64_t> key(n, s), key2(n, s);
    coreness_device(g, core.p, s);
    k_core_keys<<<grid_for(n, 256), 256, 0, s>>>(core.p, g.deg.p, n, key.p, ids.p);
    TG_CHECK_LAUNCH();
    // stable: equal (core, degree) keep ascending ids (order.hpp:118-122)
    cub_call(s, [&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, key.p, key2.p, ids.p, ids2.p, (int64_t)n, 0, 64, s);
    });
    k_rank_from_sorted<<<grid_for(n, 256), 256, 0, s>>>(ids2.p, n, g.okey.p);
    TG_CHECK_LAUNCH();
    g_launches += 3;
  }
}

void order_rank(const DevGraph& g, uint32_t* d_rank, cudaStream_t s) {
  if (!g.n) return;
  if (g.order == TG_ORDER_BY_DEGREE) return degree_rank(g, d_rank, s);
  TG_CUDA(cudaMemcpyAsync(d_rank, g.okey.p, g.n * 4, cudaMemcpyDeviceToDevice, s));
}

}  // namespace tgb
