// exchange.cu -- partition-side kernels: surrogate packing (ANOP), overlap
// storage accounting (AOP) and direct-engine message accounting.
//
// Reference: anop_surrogate_body (engines.hpp:146-198) ships N_v to owner(u)
// at most once per destination via LastProc (:173,182-187);
// build_overlap_partition (partition.hpp:171-206) stores core lists plus
// halo lists trimmed to partition members; anop_direct_body
// (engines.hpp:80-141) sends one request and one reply per (v,u) with an
// off-core u.
//
// B200 design: LastProc over an ID-sorted N_v with contiguous core ranges is
// "distinct owner values != self" (owners are monotone along N_v), so one
// warp per apex finds run starts with a ballot; messages are described by
// (dest << 32 | v) keys, stably radix-sorted by destination so every
// destination's headers and lists are contiguous -- exactly the send buffers
// of an all-to-allv over NVLink (ncclSend/ncclRecv or torch all_to_all_single).
#include <cub/cub.cuh>

#include "exchange.cuh"

namespace tgb {
namespace {

template <class F>
void cub_run(cudaStream_t s, F&& f) {
  size_t bytes = 0;
  TG_CUDA(f((void*)nullptr, bytes));
  DBuf<char> tmp(bytes ? bytes : 1, s);
  TG_CUDA(f((void*)tmp.p, bytes));
}

constexpr int kMaxP = 1024;

// owner(x) = upper_bound over inner boundaries b[1..p-1] (partition.hpp:106-109)
__device__ __forceinline__ uint32_t owner_of(const uint32_t* b, uint32_t p, uint32_t x) {
  uint32_t lo = 1, hi = p;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (b[mid] <= x) lo = mid + 1;
    else hi = mid;
  }
  return lo - 1;
}

// EMIT=false: r[v-cb] = #distinct remote owners in N_v.
// EMIT=true : desc[roff[v-cb] + t] = (owner << 32) | v for the t-th run.
template <bool EMIT>
__global__ void __launch_bounds__(256)
k_surr_runs(CsrView part, uint32_t cb, uint32_t ce, const uint32_t* __restrict__ gb, uint32_t p,
            uint32_t self, uint64_t* __restrict__ r_or_off, uint64_t* __restrict__ desc) {
  __shared__ uint32_t sb[kMaxP + 1];
  for (uint32_t i = threadIdx.x; i <= p; i += blockDim.x) sb[i] = gb[i];
  __syncthreads();
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < (uint64_t)(ce - cb);
       r += warps) {
    const uint32_t v = cb + (uint32_t)r;
    const uint64_t dsc = part.desc[v - part.base];
    const uint64_t a = desc_start(dsc), e = a + desc_len(dsc);
    uint64_t wpos = EMIT ? r_or_off[r] : 0;
    uint32_t prev = 0xffffffffu;  // owner of the previous element
    uint64_t c = 0;
    for (uint64_t k0 = a; k0 < e; k0 += 32) {
      const uint64_t k = k0 + lane;
      uint32_t o = 0xffffffffu;
      if (k < e) o = owner_of(sb, p, part.data[k]);
      uint32_t before = __shfl_up_sync(0xffffffffu, o, 1);
      if (lane == 0) before = prev;
      const bool start = k < e && o != self && o != before;
      const unsigned bal = __ballot_sync(0xffffffffu, start);
      if (EMIT && start)
        desc[wpos + c + __popc(bal & ((1u << lane) - 1u))] = ((uint64_t)o << 32) | v;
      c += __popc(bal);
      uint32_t last_lane = (uint32_t)min((uint64_t)31, e - 1 - k0);
      prev = __shfl_sync(0xffffffffu, o, last_lane);
    }
    if (!EMIT && lane == 0) r_or_off[r] = c;
  }
}

__global__ void k_desc_lens(const uint64_t* __restrict__ desc, uint64_t M, CsrView part,
                            uint64_t* __restrict__ lens, unsigned long long* __restrict__ per_dest_msgs,
                            unsigned long long* __restrict__ per_dest_words) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < M;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = (uint32_t)desc[k], j = (uint32_t)(desc[k] >> 32);
    const uint64_t h = desc_len(part.desc[v - part.base]);
    lens[k] = h;
    atomicAdd(&per_dest_msgs[j], 1ull);
    atomicAdd(&per_dest_words[j], (unsigned long long)h);
  }
}

__global__ void k_scatter(const uint64_t* __restrict__ desc, uint64_t M, CsrView part,
                          const uint64_t* __restrict__ doff, uint32_t* __restrict__ hdr,
                          uint32_t* __restrict__ data) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t k = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; k < M; k += warps) {
    const uint32_t v = (uint32_t)desc[k];
    const uint64_t dsc = part.desc[v - part.base];
    const uint64_t a = desc_start(dsc), e = a + desc_len(dsc);
    if (lane == 0) {
      hdr[2 * k] = v;
      hdr[2 * k + 1] = (uint32_t)(e - a);
    }
    const uint64_t o = doff[k];
    for (uint64_t i = a + lane; i < e; i += 32) data[o + (i - a)] = part.data[i];
  }
}

__global__ void k_hdr_lens(const uint32_t* __restrict__ hdr, uint64_t M, uint64_t* __restrict__ lens) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < M;
       k += (uint64_t)gridDim.x * blockDim.x)
    lens[k] = hdr[2 * k + 1];
}

// AOP storage: flag halo vertices (off-core members of core lists) ...
__global__ void k_mark_halo(CsrView eff, uint32_t cb, uint32_t ce, uint8_t* __restrict__ flag,
                            unsigned long long* __restrict__ core_entries) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < (uint64_t)(ce - cb);
       r += warps) {
    const uint32_t v = cb + (uint32_t)r;
    const uint64_t dsc = eff.desc[v], a = desc_start(dsc), e = a + desc_len(dsc);
    if (lane == 0 && e > a) atomicAdd(core_entries, (unsigned long long)(e - a));
    for (uint64_t k = a + lane; k < e; k += 32) {
      uint32_t u = eff.data[k];
      if (u < cb || u >= ce) flag[u] = 1;
    }
  }
}

// ... then count trimmed halo list entries (partition.hpp:192-204).
__global__ void k_count_trimmed(CsrView eff, uint64_t n, uint32_t cb, uint32_t ce,
                                const uint8_t* __restrict__ flag, unsigned long long* __restrict__ out) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  uint64_t s = 0;
  for (uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; w < n; w += warps) {
    if (!flag[w]) continue;
    const uint64_t dsc = eff.desc[w], a = desc_start(dsc), e = a + desc_len(dsc);
    for (uint64_t k = a + lane; k < e; k += 32) {
      uint32_t x = eff.data[k];
      if ((x >= cb && x < ce) || flag[x]) ++s;
    }
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0 && s) atomicAdd(out, (unsigned long long)s);
}

// Direct engine: per (v,u) with owner(u) != owner(v) one request (sender
// owner(v)) and one reply (sender owner(u)).
__global__ void __launch_bounds__(256)
k_direct_msgs(CsrView eff, uint64_t n, const uint32_t* __restrict__ gb, uint32_t p,
              unsigned long long* __restrict__ req, unsigned long long* __restrict__ rep) {
  __shared__ uint32_t sb[kMaxP + 1];
  for (uint32_t i = threadIdx.x; i <= p; i += blockDim.x) sb[i] = gb[i];
  __syncthreads();
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t v = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; v < n; v += warps) {
    const uint32_t ov = owner_of(sb, p, (uint32_t)v);
    unsigned long long mine = 0;
    const uint64_t dsc = eff.desc[v], a = desc_start(dsc), e = a + desc_len(dsc);
    for (uint64_t k = a + lane; k < e; k += 32) {
      uint32_t ou = owner_of(sb, p, eff.data[k]);
      if (ou != ov) {
        ++mine;
        atomicAdd(&rep[ou], 1ull);
      }
    }
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if (lane == 0 && mine) atomicAdd(&req[ov], mine);
  }
}

}  // namespace

void SurrogatePack::build(CsrView part, uint32_t cb, uint32_t ce, const std::vector<uint32_t>& b,
                          uint32_t self, cudaStream_t s) {
  const uint32_t p = (uint32_t)(b.size() - 1);
  TG_REQUIRE(p <= (uint32_t)kMaxP, "surrogate: at most 1024 ranks");
  this->part = part;
  DBuf<uint32_t> gb(p + 1, s);
  TG_CUDA(cudaMemcpyAsync(gb.p, b.data(), (p + 1) * 4, cudaMemcpyHostToDevice, s));
  const uint64_t rows = ce - cb;
  msgs_per_dest.assign(p, 0);
  words_per_dest.assign(p, 0);
  M = 0;
  if (!rows) return;
  DBuf<uint64_t> r(rows, s), roff(rows + 1, s);
  unsigned grid = grid_for(rows * 32, 256, 148u * 32u);
  k_surr_runs<false><<<grid, 256, 0, s>>>(part, cb, ce, gb.p, p, self, r.p, nullptr);
  TG_CHECK_LAUNCH();
  ++g_launches;
  TG_CUDA(cudaMemsetAsync(roff.p, 0, 8, s));
  cub_run(s, [&](void* t, size_t& bytes) {
    return cub::DeviceScan::InclusiveSum(t, bytes, r.p, roff.p + 1, (int64_t)rows, s);
  });
  ++g_launches;
  TG_CUDA(cudaMemcpyAsync(&M, roff.p + rows, 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  if (!M) return;
  DBuf<uint64_t> d1(M, s);
  desc.alloc(M, s);
  k_surr_runs<true><<<grid, 256, 0, s>>>(part, cb, ce, gb.p, p, self, roff.p, d1.p);
  TG_CHECK_LAUNCH();
  ++g_launches;
  unsigned bits = 1;
  while ((1u << bits) < p) ++bits;
  cub_run(s, [&](void* t, size_t& bytes) {
    return cub::DeviceRadixSort::SortKeys(t, bytes, d1.p, desc.p, (int64_t)M, 32, 32 + (int)bits, s);
  });
  ++g_launches;
  DBuf<uint64_t> lens(M, s);
  DBuf<unsigned long long> pm(p, s), pw(p, s);
  pm.zero();
  pw.zero();
  k_desc_lens<<<grid_for(M, 256), 256, 0, s>>>(desc.p, M, part, lens.p, pm.p, pw.p);
  TG_CHECK_LAUNCH();
  ++g_launches;
  doff.alloc(M + 1, s);
  TG_CUDA(cudaMemsetAsync(doff.p, 0, 8, s));
  cub_run(s, [&](void* t, size_t& bytes) {
    return cub::DeviceScan::InclusiveSum(t, bytes, lens.p, doff.p + 1, (int64_t)M, s);
  });
  ++g_launches;
  TG_CUDA(cudaMemcpyAsync(msgs_per_dest.data(), pm.p, p * 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaMemcpyAsync(words_per_dest.data(), pw.p, p * 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
}

void SurrogatePack::scatter(uint32_t* d_hdr, uint32_t* d_data, cudaStream_t s) const {
  if (!M) return;
  k_scatter<<<grid_for(M * 32, 256, 148u * 32u), 256, 0, s>>>(desc.p, M, part, doff.p, d_hdr, d_data);
  TG_CHECK_LAUNCH();
  ++g_launches;
}

void message_offsets(const uint32_t* d_hdr, uint64_t M, DBuf<uint64_t>& moff, cudaStream_t s) {
  moff.alloc(M + 1, s);
  TG_CUDA(cudaMemsetAsync(moff.p, 0, 8, s));
  if (!M) return;
  DBuf<uint64_t> lens(M, s);
  k_hdr_lens<<<grid_for(M, 256), 256, 0, s>>>(d_hdr, M, lens.p);
  TG_CHECK_LAUNCH();
  ++g_launches;
  cub_run(s, [&](void* t, size_t& bytes) {
    return cub::DeviceScan::InclusiveSum(t, bytes, lens.p, moff.p + 1, (int64_t)M, s);
  });
  ++g_launches;
}

uint64_t overlap_stored_entries(CsrView eff, uint64_t n, uint32_t cb, uint32_t ce, cudaStream_t s) {
  if (ce <= cb || !n) return 0;
  DBuf<uint8_t> flag(n, s);
  flag.zero();
  DBuf<unsigned long long> acc(1, s);
  acc.zero();
  k_mark_halo<<<grid_for((uint64_t)(ce - cb) * 32, 256, 148u * 32u), 256, 0, s>>>(eff, cb, ce, flag.p,
                                                                                 acc.p);
  TG_CHECK_LAUNCH();
  k_count_trimmed<<<grid_for(n * 32, 256, 148u * 32u), 256, 0, s>>>(eff, n, cb, ce, flag.p, acc.p);
  TG_CHECK_LAUNCH();
  g_launches += 2;
  unsigned long long h = 0;
  TG_CUDA(cudaMemcpyAsync(&h, acc.p, 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  return h;
}

void direct_messages(CsrView eff, uint64_t n, const std::vector<uint32_t>& b,
                     std::vector<uint64_t>& req, std::vector<uint64_t>& rep, cudaStream_t s) {
  const uint32_t p = (uint32_t)(b.size() - 1);
  TG_REQUIRE(p <= (uint32_t)kMaxP, "direct: at most 1024 ranks");
  DBuf<uint32_t> gb(p + 1, s);
  TG_CUDA(cudaMemcpyAsync(gb.p, b.data(), (p + 1) * 4, cudaMemcpyHostToDevice, s));
  DBuf<unsigned long long> dq(p, s), dp(p, s);
  dq.zero();
  dp.zero();
  if (n) {
    k_direct_msgs<<<grid_for(n * 32, 256, 148u * 32u), 256, 0, s>>>(eff, n, gb.p, p, dq.p, dp.p);
    TG_CHECK_LAUNCH();
    ++g_launches;
  }
  req.assign(p, 0);
  rep.assign(p, 0);
  TG_CUDA(cudaMemcpyAsync(req.data(), dq.p, p * 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaMemcpyAsync(rep.data(), dp.p, p * 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
}

}  // namespace tgb
