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
// One warp per apex v (N_v = slab v, prefetched one apex ahead so that the
// N_u reads are the only dependent DRAM hop per apex).  A warp load covers 4
// lists (8 lanes x 16 bytes each), 5 loads in flight = 20 lists.  No segment
// table, no head/tail slots: lane -> (list, quad) is a shift.  Membership as
// in the quad kernel: inverted blocked filter, exact search only on hits.
#pragma once

#ifndef TG_SLAB_U
#define TG_SLAB_U 5
#endif
#ifndef TG_SLAB_BLOCKS
#define TG_SLAB_BLOCKS 5
#endif
constexpr int kSlabU = TG_SLAB_U;            // warp loads in flight (4 lists each)
constexpr int kSlabBlocks = TG_SLAB_BLOCKS;  // resident blocks per SM

template <bool TALLY, bool LIST, bool FILTER, class Apex>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, kSlabBlocks)
k_intersect_slab(Apex A, CsrView nu, uint32_t ulo, uint32_t uhi, CountOut out,
                 uint32_t* __restrict__ big, unsigned long long* __restrict__ big_count,
                 uint64_t big_cap, unsigned long long* __restrict__ chunk_ctr, uint32_t chunk) {
  __shared__ uint32_t sNv[kWarpsPerBlock][kWCap];
  __shared__ __align__(1024) uint32_t sBm[kWarpsPerBlock][kBmWords];  // inverted filter
  __shared__ unsigned sCntU[TALLY ? kWarpsPerBlock : 1][kWCap];
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu;
  const unsigned lt_mask = (1u << lane) - 1u;
  const unsigned jl = lane >> 3, q = lane & 7;  // list of the load, quad of the slab
  const uint64_t nitems = A.count();
  const uint4* __restrict__ Q4 = reinterpret_cast<const uint4*>(nu.data);
  uint32_t* Nv = sNv[w];
  uint32_t* Bm = sBm[w];
  const uint32_t bm_s = (uint32_t)__cvta_generic_to_shared(Bm);  // 1 KB-aligned
#pragma unroll
  for (int i = 0; i < kBmWords / 32; ++i) Bm[lane + 32 * i] = 0xFFFFFFFFu;
  if (TALLY) {
    sCntU[w][lane] = 0;
    sCntU[w][lane + 32] = 0;
  }
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
    uint32_t x = have_nx ? nx : __ldg(nu.data + ((uint64_t)(v - nu.base) * kSlab + lane));
    have_nx = k < kend;
    if (have_nx) nx = __ldg(nu.data + ((uint64_t)(A.vertex(k) - nu.base) * kSlab + lane));
    uint32_t hv = __popc(__ballot_sync(FULL, x != kNoEntry));
    uint32_t jlo = 0, jhi = hv;
    if (hv < 2) continue;  // a triangle needs u, w ∈ N_v
    if (hv == kSlab) {     // maybe longer than its slab: the descriptor knows
      const uint64_t d = nu.desc[v - nu.base];
      hv = desc_len(d);
      if (hv > kWCap) {
        if (lane == 0) {
          unsigned long long pos = atomicAdd(big_count, 1ull);
          if (pos < big_cap) big[pos] = (uint32_t)kc;
        }
        continue;
      }
      Nv[lane] = x;
      atomicAnd(&Bm[bm_word(bm_hash(x))], ~qm_mask(bm_hash(x)));
      uint32_t x2 = kNoEntry;
      if (kSlab + lane < hv) {
        x2 = nu.data[desc_start(d) + kSlab + lane];
        Nv[kSlab + lane] = x2;
        atomicAnd(&Bm[bm_word(bm_hash(x2))], ~qm_mask(bm_hash(x2)));
      }
      jhi = hv;
      if (FILTER) {
        jlo = __popc(__ballot_sync(FULL, x < ulo)) + __popc(__ballot_sync(FULL, x2 < ulo));
        jhi = __popc(__ballot_sync(FULL, x < uhi)) + __popc(__ballot_sync(FULL, x2 != kNoEntry && x2 < uhi));
      }
    } else {
      if (lane < hv) {
        Nv[lane] = x;
        const uint32_t h = bm_hash(x);
        atomicAnd(&Bm[bm_word(h)], ~qm_mask(h));
      }
      if (FILTER) {
        jlo = __popc(__ballot_sync(FULL, x < ulo));  // (pads compare above every id)
        jhi = __popc(__ballot_sync(FULL, x < uhi && x != kNoEntry));
      }
    }
    __syncwarp();
    uint32_t apex_cnt = 0;  // per lane
    for (uint32_t jb = jlo; jb < jhi; jb += 4 * kSlabU) {
      uint4 r[kSlabU];
#pragma unroll
      for (int b = 0; b < kSlabU; ++b) {
        const uint32_t j = jb + 4 * b + jl;
        r[b] = make_uint4(kNoEntry, kNoEntry, kNoEntry, kNoEntry);
        if (j < jhi) r[b] = ldg_stream4(Q4 + ((uint64_t)(Nv[j] - nu.base) * (kSlab / 4) + q));
      }
      bool p = false;
      unsigned more = 0;  // lists that may continue past their slab
#pragma unroll
      for (int b = 0; b < kSlabU; ++b) {
        p |= qm_probe(bm_s, r[b].x) | qm_probe(bm_s, r[b].y) | qm_probe(bm_s, r[b].z) |
             qm_probe(bm_s, r[b].w);
        more |= (unsigned)(q == 7 && r[b].w != kNoEntry) << b;
      }
      if (__any_sync(FULL, p)) {
        // exact path: slots that pass the filter (pads are in no N_v)
        unsigned fnd = 0;
#pragma unroll
        for (int b = 0; b < kSlabU; ++b) {
          const uint32_t xq[4] = {r[b].x, r[b].y, r[b].z, r[b].w};
#pragma unroll
          for (int s2 = 0; s2 < 4; ++s2)
            if (qm_probe(bm_s, xq[s2]))
              fnd |= (unsigned)contains_small(Nv, hv, xq[s2]) << (4 * b + s2);
        }
        if (__any_sync(FULL, fnd != 0)) {
          apex_cnt += __popc(fnd);
          if (TALLY || LIST) {
#pragma unroll
            for (int b = 0; b < kSlabU; ++b) {
              const uint32_t xq[4] = {r[b].x, r[b].y, r[b].z, r[b].w};
              const uint32_t j = min(jb + 4 * b + jl, hv - 1);
#pragma unroll
              for (int s2 = 0; s2 < 4; ++s2) {
                const bool found = (fnd >> (4 * b + s2)) & 1u;
                if (TALLY && found) {
                  atomicAdd(&out.tally[xq[s2]], 1ull);
                  atomicAdd(&sCntU[w][j], 1u);
                }
                if (LIST) {
                  const unsigned m = __ballot_sync(FULL, found);
                  if (m) {
                    unsigned long long b0 = 0;
                    if (lane == 0) b0 = atomicAdd(out.cursor, (unsigned long long)__popc(m));
                    b0 = __shfl_sync(FULL, b0, 0);
                    if (found) emit_triple(out, b0 + __popc(m & lt_mask), v, Nv[j], xq[s2]);
                  }
                }
              }
            }
          }
        }
      }
      if (__any_sync(FULL, more != 0)) {
        // rare: entries [32, h_u) of the lists longer than a slab, 32 per step
#pragma unroll
        for (int b = 0; b < kSlabU; ++b) {
          unsigned mm = __ballot_sync(FULL, (more >> b) & 1u);
          while (mm) {
            const unsigned src = __ffs(mm) - 1;
            mm &= mm - 1;
            const uint32_t j = jb + 4 * b + (src >> 3);
            const uint32_t u = Nv[j];
            const uint64_t d = nu.desc[u - nu.base];
            const uint32_t len = desc_len(d);
            const uint32_t* __restrict__ P = nu.data + desc_start(d);
            for (uint32_t i0 = kSlab; i0 < len; i0 += 32) {
              const uint32_t y = i0 + lane < len ? __ldg(P + i0 + lane) : kNoEntry;
              const bool found = qm_probe(bm_s, y) && contains_small(Nv, hv, y);
              const unsigned m = __ballot_sync(FULL, found);
              if (!m) continue;
              apex_cnt += found;
              if (TALLY && found) {
                atomicAdd(&out.tally[y], 1ull);
                atomicAdd(&sCntU[w][j], 1u);
              }
              if (LIST) {
                unsigned long long b0 = 0;
                if (lane == 0) b0 = atomicAdd(out.cursor, (unsigned long long)__popc(m));
                b0 = __shfl_sync(FULL, b0, 0);
                if (found) emit_triple(out, b0 + __popc(m & lt_mask), v, u, y);
              }
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
        const unsigned c = sCntU[w][j];
        if (c) {
          atomicAdd(&out.tally[Nv[j]], (unsigned long long)c);
          sCntU[w][j] = 0;
        }
      }
    }
    acc += apex_cnt;
    for (uint32_t i0 = lane; i0 < hv; i0 += 32) Bm[bm_word(bm_hash(Nv[i0]))] = 0xFFFFFFFFu;
    __syncwarp();
  }
  unsigned long long a2 = acc;  // per-lane partials
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a2 += __shfl_xor_sync(FULL, a2, o);
  if (lane == 0 && a2) atomicAdd(out.total, a2);
}
