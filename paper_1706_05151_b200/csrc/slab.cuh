// slab.cuh -- per-apex warp kernel over the slab layout of the oriented lists
// (included by intersect.cu; same reference semantics as k_intersect_quad:
// count_node_iterator_n, sequential.hpp:74-91, and aop_count, engines.hpp:38-54).
//
// Why a layout: on a PA graph the pass is a stream of RANDOM reads of ~80-byte
// lists N_u, and a B200 fetches DRAM in 128-byte lines.  Measured
// (tools/exp/slab_probe.cu, 4e8 reads over 1e8 lists): descriptor + unaligned
// list = 327 DRAM bytes per read, 2.1e10 reads/s -- exactly the rate of
// k_intersect_quad on C5 -- against 132 bytes and 4.4e10 reads/s when each list
// sits alone in one aligned 128-byte line and its address is 32 u (no
// descriptor).  So: list u = the kSlab = 32 slots at data + 32 u, padded with
// kNoEntry; a list longer than a slab keeps its first 32 entries there and is
// stored whole above the slabs (its descriptor points there), which a reader
// notices from a non-pad last slot.
//
// With the bytes halved the pass is bound by issue slots (ncu of the first
// slab kernel: 43 warp instructions per list read, issue 69%, DRAM 46%), so
// the membership test is as short as it gets: N_v goes into a per-warp
// direct-mapped table of 1024 words under a multiplier chosen PER APEX so
// that its <= 64 keys do not collide (a perfect hash: retry with the next
// multiplier on a collision, 17% of the tries at h_v = 20).  A probe is then
// IMAD, SHF, LOP3, LDS, ISETP -- exact, no filter, no second search.
// (C5: 70 -> 54 ms.  Measured and dropped afterwards: skipping a round's empty
// loads warp-uniformly, an all-pad slab for the lanes of a partial load and
// folded 64-bit addresses -- the same time at 4 resident blocks per SM, 6%
// slower at 5: the kernel now waits on DRAM lines, not on issue slots.)
//
// One warp per apex v (N_v = slab v, prefetched one apex ahead).  A warp load
// reads 4 whole slabs (8 lanes x 16 bytes each); a round of 6 loads covers 24
// lists, the whole apex on a PA graph.  No segment table, no head/tail slots:
// lane -> (list, quad) is a shift.
#pragma once

#ifndef TG_SLAB_U
#define TG_SLAB_U 6
#endif
#ifndef TG_SLAB_BLOCKS
#define TG_SLAB_BLOCKS 4
#endif
constexpr int kSlabU = TG_SLAB_U;            // warp loads per round (4 lists each)
constexpr int kSlabBlocks = TG_SLAB_BLOCKS;  // resident blocks per SM
constexpr uint32_t kPhWords = 1024;          // per-warp table (4 KB)
constexpr uint32_t kPhEmpty = 0xfffffffeu;   // empty slot: neither a NodeId nor the pad
constexpr int kPhTries = 16;
// shared memory of a block: the tables (4 KB-aligned), N_v, per-u tallies
constexpr size_t kSlabSmem = 4096 + kWarpsPerBlock * (kPhWords + 2 * kWCap) * sizeof(uint32_t);

__device__ __forceinline__ uint32_t ph_mul(int t) { return 0x2545F491u + 0x9E3779B2u * (uint32_t)t; }
// byte offset of x's slot in the table
__device__ __forceinline__ uint32_t ph_slot(uint32_t mul, uint32_t x) {
  return ((x * mul) >> 20) & ((kPhWords - 1) * 4u);
}
__device__ __forceinline__ bool ph_probe(uint32_t tb_s, uint32_t mul, uint32_t x) {
  return lds_u32(tb_s | ph_slot(mul, x)) == x;
}
__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

template <bool TALLY, bool LIST, bool FILTER, class Apex>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, kSlabBlocks)
k_intersect_slab(Apex A, CsrView nu, uint32_t ulo, uint32_t uhi, CountOut out,
                 uint32_t* __restrict__ big, unsigned long long* __restrict__ big_count,
                 uint64_t big_cap, unsigned long long* __restrict__ chunk_ctr, uint32_t chunk) {
  constexpr int U = kSlabU, R = 4 * U;  // lists per round
  constexpr int QS = kSlab / 4;         // quads per slab
  extern __shared__ uint32_t slab_smem[];
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu;
  const unsigned lt_mask = (1u << lane) - 1u;
  const unsigned jl = lane >> 3, q = lane & 7;  // list of the load, quad of the slab
  // carve: tables first (4 KB-aligned shared address), then N_v, then tallies
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(slab_smem);
  const uint32_t a0 = (s0 + 4095u) & ~4095u;
  uint32_t* base = slab_smem + ((a0 - s0) >> 2);
  const uint32_t tb_s = a0 + w * (kPhWords * 4u);
  uint32_t* Nv = base + kWarpsPerBlock * kPhWords + w * kWCap;
  uint32_t* CntU = base + kWarpsPerBlock * (kPhWords + kWCap) + w * kWCap;
  for (uint32_t i = lane; i < kPhWords; i += 32) sts_u32(tb_s + 4 * i, kPhEmpty);
  if (TALLY) {
    CntU[lane] = 0;
    CntU[lane + 32] = 0;
  }
  const uint64_t nitems = A.count();
  const uint4* __restrict__ Q4 = reinterpret_cast<const uint4*>(nu.data);
  unsigned long long acc = 0;
  __syncwarp();

  uint64_t k = 0, kend = 0;
  uint32_t nx = kNoEntry;  // slab word of the next apex (prefetched)
  bool have_nx = false;
  for (;;) {
    if (k == kend) {
      unsigned long long c = 0;
      if (lane == 0) c = atomicAdd(chunk_ctr, (unsigned long long)chunk);
      k = __shfl_sync(FULL, c, 0);
      if (k >= nitems) break;
      kend = min(nitems, k + chunk);
      have_nx = false;
    }
    const uint64_t kc = k++;
    const uint32_t v = A.vertex(kc);
    const uint32_t x = have_nx ? nx : __ldg(nu.data + ((uint64_t)(v - nu.base) * kSlab + lane));
    have_nx = k < kend;
    if (have_nx) nx = __ldg(nu.data + ((uint64_t)(A.vertex(k) - nu.base) * kSlab + lane));
    uint32_t hv = __popc(__ballot_sync(FULL, x != kNoEntry));
    if (hv < 2) continue;  // a triangle needs u, w ∈ N_v
    uint32_t x2 = kNoEntry;
    bool to_cta = false;
    if (hv == kSlab) {  // maybe longer than its slab: the descriptor knows
      const uint64_t d = nu.desc[v - nu.base];
      hv = desc_len(d);
      if (hv > kWCap) to_cta = true;
      else if (kSlab + lane < hv) x2 = nu.data[desc_start(d) + kSlab + lane];
    }
    // perfect hash of N_v: the first multiplier under which no two keys share a slot
    uint32_t mul = 0;
    if (!to_cta) {
      int t = 0;
      for (; t < kPhTries; ++t) {
        mul = ph_mul(t);
        if (x != kNoEntry) sts_u32(tb_s | ph_slot(mul, x), x);
        if (x2 != kNoEntry) sts_u32(tb_s | ph_slot(mul, x2), x2);
        __syncwarp();
        const bool ok = (x == kNoEntry || ph_probe(tb_s, mul, x)) &&
                        (x2 == kNoEntry || ph_probe(tb_s, mul, x2));
        if (__all_sync(FULL, ok)) break;
        if (x != kNoEntry) sts_u32(tb_s | ph_slot(mul, x), kPhEmpty);
        if (x2 != kNoEntry) sts_u32(tb_s | ph_slot(mul, x2), kPhEmpty);
        __syncwarp();
      }
      to_cta = t == kPhTries;  // (table left empty)
    }
    if (to_cta) {  // long or unhashable N_v: the CTA path
      if (lane == 0) {
        unsigned long long pos = atomicAdd(big_count, 1ull);
        if (pos < big_cap) big[pos] = (uint32_t)kc;
      }
      continue;
    }
    if (x != kNoEntry) Nv[lane] = x;
    if (x2 != kNoEntry) Nv[kSlab + lane] = x2;
    uint32_t jlo = 0, jhi = hv;
    if (FILTER) {  // (pads compare above every id)
      jlo = __popc(__ballot_sync(FULL, x < ulo)) + __popc(__ballot_sync(FULL, x2 < ulo));
      jhi = __popc(__ballot_sync(FULL, x != kNoEntry && x < uhi)) +
            __popc(__ballot_sync(FULL, x2 != kNoEntry && x2 < uhi));
    }
    __syncwarp();
    uint32_t apex_cnt = 0;  // per lane
    // a found element y of list j (warp-converged call)
    auto emit = [&](bool found, uint32_t j, uint32_t y) {
      apex_cnt += found;
      if (TALLY && found) {
        atomicAdd(&out.tally[y], 1ull);
        atomicAdd(&CntU[j], 1u);
      }
      if (LIST) {
        const unsigned m = __ballot_sync(FULL, found);
        if (m) {
          unsigned long long b0 = 0;
          if (lane == 0) b0 = atomicAdd(out.cursor, (unsigned long long)__popc(m));
          b0 = __shfl_sync(FULL, b0, 0);
          if (found) emit_triple(out, b0 + __popc(m & lt_mask), v, Nv[j], y);
        }
      }
    };
    for (uint32_t jb = jlo; jb < jhi; jb += R) {
      uint4 r[U];
#pragma unroll
      for (int b = 0; b < U; ++b) {
        const uint32_t j = jb + 4 * b + jl;
        r[b] = make_uint4(kNoEntry, kNoEntry, kNoEntry, kNoEntry);
        if (j < jhi) r[b] = ldg_stream4(Q4 + ((uint64_t)(Nv[j] - nu.base) * QS + q));
      }
      unsigned hm = 0;    // slots found in N_v (pads match nothing)
      unsigned more = 0;  // lists longer than their slab
#pragma unroll
      for (int b = 0; b < U; ++b) {
        hm |= (unsigned)ph_probe(tb_s, mul, r[b].x) << (4 * b);
        hm |= (unsigned)ph_probe(tb_s, mul, r[b].y) << (4 * b + 1);
        hm |= (unsigned)ph_probe(tb_s, mul, r[b].z) << (4 * b + 2);
        hm |= (unsigned)ph_probe(tb_s, mul, r[b].w) << (4 * b + 3);
        more |= (unsigned)(q == 7 && r[b].w != kNoEntry) << b;
      }
      if (!TALLY && !LIST) {
        apex_cnt += __popc(hm);
      } else if (__any_sync(FULL, hm != 0)) {
#pragma unroll
        for (int b = 0; b < U; ++b) {
          const uint32_t xq[4] = {r[b].x, r[b].y, r[b].z, r[b].w};
          const uint32_t j = min(jb + 4 * b + jl, hv - 1);
#pragma unroll
          for (int s2 = 0; s2 < 4; ++s2) emit((hm >> (4 * b + s2)) & 1u, j, xq[s2]);
        }
      }
      if (__any_sync(FULL, more != 0)) {
        // rare: entries [32, h_u) of the lists longer than a slab, 32 per step
#pragma unroll
        for (int b = 0; b < U; ++b) {
          unsigned mm = __ballot_sync(FULL, (more >> b) & 1u);
          while (mm) {
            const unsigned src = __ffs(mm) - 1;
            mm &= mm - 1;
            const uint32_t j = jb + 4 * b + (src >> 3);
            const uint64_t d = nu.desc[Nv[j] - nu.base];
            const uint32_t len = desc_len(d);
            const uint32_t* __restrict__ P = nu.data + desc_start(d);
            for (uint32_t i0 = kSlab; i0 < len; i0 += 32) {
              const uint32_t y = i0 + lane < len ? __ldg(P + i0 + lane) : kNoEntry;
              const bool found = ph_probe(tb_s, mul, y);
              if (__any_sync(FULL, found)) emit(found, j, y);
            }
          }
        }
      }
    }
    __syncwarp();
    if (TALLY) {
      const uint32_t tot = __reduce_add_sync(FULL, apex_cnt);
      if (lane == 0 && tot) atomicAdd(&out.tally[v], (unsigned long long)tot);
      for (uint32_t j = lane; j < hv; j += 32) {
        const unsigned cu = CntU[j];
        if (cu) {
          atomicAdd(&out.tally[Nv[j]], (unsigned long long)cu);
          CntU[j] = 0;
        }
      }
    }
    acc += apex_cnt;
    if (x != kNoEntry) sts_u32(tb_s | ph_slot(mul, x), kPhEmpty);
    if (x2 != kNoEntry) sts_u32(tb_s | ph_slot(mul, x2), kPhEmpty);
    __syncwarp();
  }
  unsigned long long a2 = acc;  // per-lane partials
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a2 += __shfl_xor_sync(FULL, a2, o);
  if (lane == 0 && a2) atomicAdd(out.total, a2);
}
