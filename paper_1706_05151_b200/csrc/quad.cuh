// quad.cuh -- per-apex warp kernel over 16-byte quads of the middle lists
// (included by intersect.cu; same reference semantics as k_intersect_warp:
// count_node_iterator_n, sequential.hpp:74-91, and the AOP / SurrogateCount
// bodies, engines.hpp:38-76).
//
// The oriented lists are unaligned and unpadded (tile layout or compact), so
// each N_u is read as the 16-byte-aligned quads that cover it: a lane loads
// one quad (LDG.128) and drops the slots outside [start, start+len) -- only a
// list's first quad (head slots) and last quad (tail slots) are partial.  One
// lane thus tests 4 elements per load, and the per-item bookkeeping (segment
// lookup, address, loop) is paid once per quad instead of once per element.
// The segment-start table, its windows and the filter + exact search are
// those of k_intersect_warp, in quad space.
#pragma once

#ifndef TG_QUNROLL
#define TG_QUNROLL 2
#endif
constexpr int kQUnroll = TG_QUNROLL;  // quad chunks (32 lanes x 16 B) in flight per warp

// N_u quads almost never hit L1 (ncu: 2.4% sector hit rate), so they are
// loaded without L1 allocation: C2 intersection 7.63 -> 7.30 ms (A/B of the
// two builds on one B200, two runs each; -DTG_QUAD_NO_L1=0 restores __ldg).
#ifndef TG_QUAD_NO_L1
#define TG_QUAD_NO_L1 1
#endif
// the same for the group / CTA quad kernels (ctaq, groupq, ctab): off -- on C3
// (R-MAT-24) it measured 225.0 vs 223.0 ms (two runs each), the hub lists
// those kernels re-read do hit L1
#ifndef TG_CQ_NO_L1
#define TG_CQ_NO_L1 0
#endif
// list descriptors DO hit L1: the no-allocate hint on them measured 7.79 vs
// 7.29 ms on C2, so it stays off (experiment macro only)
#ifndef TG_DESC_NO_L1
#define TG_DESC_NO_L1 0
#endif
template <bool NA>
__device__ __forceinline__ uint4 ldg_quad(const uint4* p) {
  if constexpr (NA) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
  } else {
    return __ldg(p);
  }
}
__device__ __forceinline__ uint4 ldg_stream4(const uint4* p) { return ldg_quad<TG_QUAD_NO_L1 != 0>(p); }
__device__ __forceinline__ uint4 ldg_cq4(const uint4* p) { return ldg_quad<TG_CQ_NO_L1 != 0>(p); }

template <bool TALLY, bool LIST, bool FILTER, class Apex>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, kWBlocks)
k_intersect_quad(Apex A, CsrView nu, uint32_t ulo, uint32_t uhi, CountOut out,
                 uint32_t* __restrict__ big, unsigned long long* __restrict__ big_count,
                 uint64_t big_cap, unsigned long long* __restrict__ chunk_ctr, uint32_t chunk) {
  __shared__ uint32_t sNv[kWarpsPerBlock][kWCap];
  __shared__ __align__(1024) uint32_t sBm[kWarpsPerBlock][kBmWords];  // inverted filter
  __shared__ uint32_t sTbl[kWarpsPerBlock][kTblWords + kQUnroll + 1];
  __shared__ uint32_t sQs[kWarpsPerBlock][32];  // segment: first quad - first item
  __shared__ uint32_t sHt[kWarpsPerBlock][32];  // segment: head | tail << 2 skipped slots
  __shared__ uint32_t sSt[kWarpsPerBlock][32];  // segment: first item (quad space)
  __shared__ uint32_t sU[kWarpsPerBlock][32];
  __shared__ unsigned sCntU[kWarpsPerBlock][32];
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu;
  const unsigned lt_mask = (1u << lane) - 1u;
  const unsigned le_mask = (2u << lane) - 1u;
  const uint64_t nitems = A.count();
  const uint4* __restrict__ Q4 = reinterpret_cast<const uint4*>(nu.data);
  uint32_t* Nv = sNv[w];
  uint32_t* Bm = sBm[w];
  const uint32_t bm_s = (uint32_t)__cvta_generic_to_shared(Bm);  // 1 KB-aligned
#pragma unroll
  for (int i = 0; i < kBmWords / 32; ++i) Bm[lane + 32 * i] = 0xFFFFFFFFu;
  uint32_t* Tbl = sTbl[w];
  unsigned long long acc = 0;
  __syncwarp();

  uint64_t k = 0, kend = 0;
  for (;;) {
    if (k == kend) {
      unsigned long long c = 0;
      if (lane == 0) c = atomicAdd(chunk_ctr, (unsigned long long)chunk);
      k = __shfl_sync(FULL, c, 0);
      if (k >= nitems) break;
      kend = min(nitems, k + chunk);
    }
    const uint64_t kc = k++;
    uint32_t v, hv;
    const uint32_t* L;
    A.get(kc, v, L, hv);
    if (hv < 2) continue;  // a triangle needs u, w ∈ N_v
    if (hv > kWCap) {
      if (lane == 0) {
        unsigned long long pos = atomicAdd(big_count, 1ull);
        if (pos < big_cap) big[pos] = (uint32_t)kc;
      }
      continue;
    }
    uint32_t jlo = 0, jhi = hv;
    if (FILTER) jhi = 0;
    for (uint32_t i0 = 0; i0 < hv; i0 += 32) {
      const bool in = i0 + lane < hv;
      uint32_t x = 0;
      if (in) {
        x = L[i0 + lane];
        Nv[i0 + lane] = x;
        const uint32_t h = bm_hash(x);
        atomicAnd(&Bm[bm_word(h)], ~qm_mask(h));
      }
      if (FILTER) {
        jlo += __popc(__ballot_sync(FULL, in && x < ulo));
        jhi += __popc(__ballot_sync(FULL, in && x < uhi));
      }
    }
    __syncwarp();
    uint32_t apex_cnt = 0;
    for (uint32_t jb = jlo; jb < jhi; jb += 32) {
      const uint32_t j = jb + lane;
      uint32_t nq = 0, u = 0, qs0 = 0, ht = 0;
      if (j < jhi) {
        u = Nv[j];
#if TG_DESC_NO_L1
        uint64_t d;
        asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(d) : "l"(nu.desc + (u - nu.base)));
#else
        const uint64_t d = nu.desc[u - nu.base];
#endif
        const uint32_t len = desc_len(d);
        const uint64_t lo = desc_start(d), end = lo + len;  // slots < 2^34
        qs0 = (uint32_t)(lo >> 2);
        nq = len ? (uint32_t)(((end + 3) >> 2) - (lo >> 2)) : 0u;
        ht = ((uint32_t)lo & 3u) | (((0u - (uint32_t)end) & 3u) << 2);
      }
      uint32_t incl = nq;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, incl, o);
        if ((int)lane >= o) incl += t;
      }
      const uint32_t S = __shfl_sync(FULL, incl, 31);  // quads of this batch
      if (jb == jlo && 4 * S > kWarpWork) {
        // heavy apex: the whole apex goes to the CTA path
        if (lane == 0) {
          unsigned long long pos = atomicAdd(big_count, 1ull);
          if (pos < big_cap) big[pos] = (uint32_t)kc;
        }
        break;
      }
      if (S == 0) continue;
      const unsigned ne = __ballot_sync(FULL, nq > 0);
      const uint32_t nseg = __popc(ne);
      if (nq > 0) {
        const uint32_t c = __popc(ne & lt_mask);
        sQs[w][c] = qs0 - (incl - nq);
        sHt[w][c] = ht;
        sSt[w][c] = incl - nq;
        if (TALLY || LIST) sU[w][c] = u;
      }
      if (TALLY) sCntU[w][lane] = 0;
      __syncwarp();
      const bool has = lane < nseg;
      const uint32_t my_qs = has ? sQs[w][lane] : 0u;
      const uint32_t my_ht = has ? sHt[w][lane] : 0u;
      const uint32_t my_st = has ? sSt[w][lane] : 0xffffffffu;
      uint32_t cnt = 0;  // segment starts before the current chunk
      for (uint32_t w0 = 0; w0 < S; w0 += 32 * kTblWords) {
        Tbl[lane] = 0;
        if (lane <= kQUnroll) Tbl[kTblWords + lane] = 0;
        __syncwarp();
        // segment starts of this window plus the first position after it
        // (a start or S, the end marker): bit idx+1 set <=> idx ends a segment
        if (has && my_st >= w0 && my_st <= w0 + 32 * kTblWords)
          atomicOr(&Tbl[(my_st - w0) >> 5], 1u << (my_st & 31));
        if (lane == 0 && S >= w0 && S <= w0 + 32 * kTblWords)
          atomicOr(&Tbl[(S - w0) >> 5], 1u << (S & 31));
        __syncwarp();
        const uint32_t wend = min(S, w0 + 32 * kTblWords);
        for (uint32_t base0 = w0; base0 < wend; base0 += 32 * kQUnroll) {
          uint4 r[kQUnroll];
          uint32_t jjs[kQUnroll];
#pragma unroll
          for (int q = 0; q < kQUnroll; ++q) {
            const uint32_t base = base0 + 32 * q;
            const uint32_t word = Tbl[(base - w0) >> 5];
            // segment of this slot; lanes past S count the end marker at S
            // (jj = nseg), so they are clamped to the last segment and below
            // re-read its last quad (qs + S - 1), which is in bounds
            const uint32_t jj = min(cnt + __popc(word & le_mask) - 1u, nseg - 1u);
            // only words inside the window: the next window's first segment start
            // (marked at word kTblWords) is counted there
            cnt += base < wend ? __popc(word) : 0u;
            jjs[q] = jj;
            const uint32_t qs = __shfl_sync(FULL, my_qs, jj);
            // validity (head/tail slots, lanes past S) is applied only on the
            // (rare) exact path below
            const uint32_t idx = min(base + lane, S - 1);
            r[q] = ldg_stream4(Q4 + (qs + idx));
          }
          // filter over all loaded slots (head/tail slots included)
          bool p = false;
#pragma unroll
          for (int q = 0; q < kQUnroll; ++q)
            p |= qm_probe(bm_s, r[q].x) | qm_probe(bm_s, r[q].y) | qm_probe(bm_s, r[q].z) |
                 qm_probe(bm_s, r[q].w);
          if (!__any_sync(FULL, p)) continue;
          // exact path: valid slots that pass the filter, branch-free search
          unsigned fnd = 0;
#pragma unroll
          for (int q = 0; q < kQUnroll; ++q) {
            const uint32_t base = base0 + 32 * q;
            const uint32_t word = Tbl[(base - w0) >> 5];
            const uint32_t nxt = Tbl[((base - w0) >> 5) + 1];
            const uint32_t hts = __shfl_sync(FULL, my_ht, jjs[q]);
            const bool first = (word >> lane) & 1u;
            const bool last = lane < 31 ? ((word >> (lane + 1)) & 1u) : (nxt & 1u);
            unsigned vm = base + lane < wend ? 0xFu : 0u;  // (this window only)
            if (first) vm &= (0xFu << (hts & 3u)) & 0xFu;
            if (last) vm &= 0xFu >> (hts >> 2);
            const uint32_t xq[4] = {r[q].x, r[q].y, r[q].z, r[q].w};
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2)
              if (((vm >> s2) & 1u) && qm_probe(bm_s, xq[s2]))
                fnd |= (unsigned)contains_small(Nv, hv, xq[s2]) << (4 * q + s2);
          }
          if (!__any_sync(FULL, fnd != 0)) continue;
          apex_cnt += __popc(fnd);  // per lane; reduced below
          if (TALLY || LIST) {
#pragma unroll
            for (int q = 0; q < kQUnroll; ++q) {
              const uint32_t xq[4] = {r[q].x, r[q].y, r[q].z, r[q].w};
#pragma unroll
              for (int s2 = 0; s2 < 4; ++s2) {
                const uint32_t x = xq[s2];
                const bool found = (fnd >> (4 * q + s2)) & 1u;
                if (TALLY && found) {
                  atomicAdd(&out.tally[x], 1ull);
                  atomicAdd(&sCntU[w][jjs[q]], 1u);
                }
                if (LIST) {
                  const unsigned m = __ballot_sync(FULL, found);
                  if (m) {
                    unsigned long long b0 = 0;
                    if (lane == 0) b0 = atomicAdd(out.cursor, (unsigned long long)__popc(m));
                    b0 = __shfl_sync(FULL, b0, 0);
                    if (found) emit_triple(out, b0 + __popc(m & lt_mask), v, sU[w][jjs[q]], x);
                  }
                }
              }
            }
          }
        }
        __syncwarp();
      }
      if (TALLY && has && sCntU[w][lane])
        atomicAdd(&out.tally[sU[w][lane]], (unsigned long long)sCntU[w][lane]);
      __syncwarp();
    }
    // apex_cnt is per lane here: reduce for the apex's own tally
    if (TALLY) {
      const uint32_t tot = __reduce_add_sync(FULL, apex_cnt);
      if (lane == 0 && tot) atomicAdd(&out.tally[v], (unsigned long long)tot);
    }
    acc += apex_cnt;
    __syncwarp();
    for (uint32_t i0 = lane; i0 < hv; i0 += 32) Bm[bm_word(bm_hash(Nv[i0]))] = 0xFFFFFFFFu;
    __syncwarp();
  }
  unsigned long long a2 = acc;  // per-lane partials
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a2 += __shfl_xor_sync(FULL, a2, o);
  if (lane == 0 && a2) atomicAdd(out.total, a2);
}
