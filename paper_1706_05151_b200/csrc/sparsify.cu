// sparsify.cu -- edge-retention sampling of oriented lists.
//
// Reference (paths relative to /root/reference/proj/include/trigraph/):
//   detail::mix64, entry_unit, keep_entry   sparsify.hpp:37-62
//   sparsify_list / sparsify_partition      sparsify.hpp:68-90
//   sparsify_effective                      sparsify.hpp:94-107
//
// Entry u of N_v survives iff entry_unit(seed, key, v, u) < q, where
// entry_unit is four SplitMix64 finalisers and a 53-bit fraction; the fp64
// product (h >> 11) * 2^-53 and the comparison are exact, so the device
// draws are bit-identical to the reference's.  key = 0 (Global) or rank + 1
// (PerPartition); rows of a non-overlapping partition use their owner's key.
// One warp per row: the row-constant part of the hash is computed once, the
// lanes hash their entries, and a ballot keeps each list ID-sorted.
#include <cub/cub.cuh>

#include "tg_internal.cuh"

namespace tgb {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return x;
}

// partition.hpp:106-109 owner(): upper_bound over the inner boundaries
__device__ __forceinline__ uint64_t owner_of(const uint32_t* __restrict__ b, uint64_t p,
                                             uint32_t v) {
  uint64_t lo = 1, hi = p;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (b[mid] <= v) lo = mid + 1;
    else hi = mid;
  }
  return lo - 1;
}

template <bool FILL>
__global__ void __launch_bounds__(256)
k_sparsify(CsrView in, uint64_t rows, double q, uint64_t seed, uint64_t kc,
           const uint32_t* __restrict__ b, uint64_t p, uint64_t* __restrict__ lens_or_off,
           uint32_t* __restrict__ out) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t hs = mix64(seed);
  for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < rows; r += warps) {
    const uint32_t v = in.base + (uint32_t)r;
    const uint64_t key = b ? owner_of(b, p, v) + 1 : kc;
    const uint64_t hrow = mix64(mix64(hs ^ key) ^ ((uint64_t)v + 0x51ed270b684a1571ULL));
    const uint64_t d = in.desc[r];
    const uint32_t* L = in.data + desc_start(d);
    const uint32_t len = desc_len(d);
    uint64_t o = FILL ? lens_or_off[r] : 0;
    uint32_t kept = 0;
    for (uint32_t k0 = 0; k0 < len; k0 += 32) {
      const uint32_t k = k0 + lane;
      uint32_t u = 0;
      bool keep = false;
      if (k < len) {
        u = L[k];
        keep = (double)(mix64(hrow ^ (uint64_t)u) >> 11) * 0x1.0p-53 < q;
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (FILL && keep) out[o + kept + __popc(m & lt_mask)] = u;
      kept += __popc(m);
    }
    if (!FILL && lane == 0) lens_or_off[r] = kept;
  }
}

__global__ void k_desc_from_off2(const uint64_t* __restrict__ off, uint64_t rows,
                                 uint64_t* __restrict__ desc) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x)
    desc[r] = make_desc(off[r], off[r + 1] - off[r]);
}

}  // namespace

void sparsify_eff(const DevEff& in, DevEff& out, double q, uint64_t seed, uint64_t kc,
                  const uint32_t* d_b, uint64_t p, cudaStream_t s) {
  const uint64_t rows = in.rows;
  out.rows = rows;
  out.base = in.base;
  out.compact = true;
  out.off.alloc(rows + 1, s);
  out.desc.alloc(rows ? rows : 1, s);
  TG_CUDA(cudaMemsetAsync(out.off.p, 0, 8, s));
  const CsrView v{in.desc.p, in.data.p, in.base};
  const unsigned grid = grid_for(rows * 32, 256, 148u * 16u);
  DBuf<uint64_t> lens(rows ? rows : 1, s);
  if (rows) {
    k_sparsify<false><<<grid, 256, 0, s>>>(v, rows, q, seed, kc, d_b, p, lens.p, nullptr);
    TG_CHECK_LAUNCH();
    size_t bytes = 0;
    TG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, lens.p, out.off.p + 1, (int64_t)rows, s));
    DBuf<char> tmp(bytes ? bytes : 1, s);
    TG_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, bytes, lens.p, out.off.p + 1, (int64_t)rows, s));
  }
  uint64_t entries = 0;
  TG_CUDA(cudaMemcpyAsync(&entries, out.off.p + rows, 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  out.entries = entries;
  out.data.alloc(entries + kQuadPad, s);
  if (rows) {
    k_sparsify<true><<<grid, 256, 0, s>>>(v, rows, q, seed, kc, d_b, p, out.off.p, out.data.p);
    TG_CHECK_LAUNCH();
    k_desc_from_off2<<<grid_for(rows, 256), 256, 0, s>>>(out.off.p, rows, out.desc.p);
    TG_CHECK_LAUNCH();
    g_launches += 4;  // count, scan (2), fill, desc
  }
}

}  // namespace tgb
