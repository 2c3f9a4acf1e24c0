// ctab.cuh -- CTA path with an exact rank-window BITMAP (included by
// intersect.cu after ctaq.cuh; same apex queue and reference semantics:
// count_node_iterator_n, sequential.hpp:74-91).
//
// Every u in N_v and every w in N_u rank above v in the orientation order
// (effective.hpp:37-52: N_x = {y in adj(x) : rank x < rank y}), so all the
// ids an apex v ever tests lie in the rank window (rank v, n).  A heavy apex
// (the CTA path) has a high degree, hence a high rank and a short window:
// when n - rank(v) - 1 <= the bitmap capacity, N_v becomes a bitmap over the
// window in shared memory and each element of N_u is tested with ONE exact
// bit probe -- no filter, no hash set, no hit queue, no false positives.
// The middle lists are read as 16-byte quads of a RANK-labelled copy of the
// oriented lists (`rdata`: same slots as nu.data, rank instead of id), with
// the segment-start tables of ctaq.cuh; ids are read back (same slot of
// nu.data) only for the hits of the TALLY / LIST sinks.  Apexes whose window
// exceeds the capacity stay on k_intersect_ctaq.
#pragma once

#ifndef TG_CTAB_MINB
#define TG_CTAB_MINB 2
#endif

template <bool TALLY, bool LIST, bool FILTER, class Apex>
__global__ void __launch_bounds__(kCT, TG_CTAB_MINB)
k_intersect_ctab(Apex A, CsrView nu, uint32_t ulo, uint32_t uhi, CountOut out,
                 const uint32_t* __restrict__ big, const unsigned long long* __restrict__ big_count,
                 uint64_t big_cap, RankView rv, unsigned long long* __restrict__ work_ctr) {
  using Scan = cub::BlockScan<uint32_t, kCT>;
  extern __shared__ __align__(16) uint32_t sBits[];  // rv.cap_bits / 32 words
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ uint32_t sQs[kCT];  // segment: first quad - first item
  __shared__ uint32_t sHt2[kCT]; // segment: head | tail << 2
  __shared__ uint32_t sSt[kCT];  // segment: first item (quad space)
  __shared__ uint32_t sU[kCT];
  __shared__ unsigned sCntU[kCT];
  __shared__ uint32_t sTbl[kCTbl + 1];
  __shared__ uint32_t sPre[kCTbl];
  __shared__ uint32_t sJ[2];
  __shared__ unsigned long long sItem, sApex;
  const unsigned t = threadIdx.x, lane = t & 31;
  const unsigned FULL = 0xffffffffu;
  const unsigned le_mask = (2u << lane) - 1u, lt_mask = (1u << lane) - 1u;
  const uint4* __restrict__ R4 = reinterpret_cast<const uint4*>(rv.rdata);
  uint64_t nbig = *big_count;
  if (nbig > big_cap) nbig = big_cap;
  unsigned long long acc = 0;

  for (;;) {
    if (t == 0) sItem = atomicAdd(work_ctr, 1ull);
    __syncthreads();
    const uint64_t bi = sItem;
    if (bi >= nbig) break;
    uint32_t v, hv;
    const uint32_t* L;
    A.get(big[bi], v, L, hv);
    const uint32_t base = rv.rank[v] + 1u;  // window [base, n)
    const uint32_t W = rv.n - base;
    if (W > rv.cap_bits) {  // uniform: left to k_intersect_ctaq
      __syncthreads();          // sItem is rewritten at the loop top
      continue;
    }
    const uint32_t nw = (W + 31) / 32;
    for (uint32_t i = t; i < nw; i += kCT) sBits[i] = 0u;
    __syncthreads();
    const uint32_t* Lr = rv.rdata + (L - nu.data);  // N_v, rank-labelled
    for (uint32_t i = t; i < hv; i += kCT) {
      const uint32_t r = Lr[i] - base;
      atomicOr(&sBits[r >> 5], 1u << (r & 31));
    }
    if (t == 0) {
      sApex = 0;
      sJ[0] = FILTER ? lower_bound_u32(L, hv, ulo) : 0;
      sJ[1] = FILTER ? lower_bound_u32(L, hv, uhi) : hv;
    }
    __syncthreads();
    const uint32_t jlo = sJ[0], jhi = sJ[1];
    uint32_t apex_cnt = 0;  // per lane
    for (uint32_t jb = jlo; jb < jhi; jb += kCT) {
      const uint32_t j = jb + t;
      uint32_t nq = 0, u = 0, qs0 = 0, ht = 0;
      if (j < jhi) {
        u = L[j];
        const uint64_t d = nu.desc[u - nu.base];
        const uint32_t len = desc_len(d);
        const uint64_t lo = desc_start(d), end = lo + len;  // slots < 2^34
        qs0 = (uint32_t)(lo >> 2);
        nq = len ? (uint32_t)(((end + 3) >> 2) - (lo >> 2)) : 0u;
        ht = ((uint32_t)lo & 3u) | (((0u - (uint32_t)end) & 3u) << 2);
      }
      uint32_t excl, S;
      Scan(scan_tmp).ExclusiveSum(nq, excl, S);
      __syncthreads();
      uint32_t c, nseg;
      Scan(scan_tmp).ExclusiveSum(nq > 0 ? 1u : 0u, c, nseg);
      if (nq > 0) {
        sQs[c] = qs0 - excl;
        sHt2[c] = ht;
        sSt[c] = excl;
        if (TALLY || LIST) sU[c] = u;
        if (TALLY) sCntU[c] = 0;
      }
      __syncthreads();
      uint32_t cbase = 0;
      for (uint32_t w0 = 0; w0 < S; w0 += 32 * kCTbl) {
        for (uint32_t i = t; i <= (uint32_t)kCTbl; i += kCT) sTbl[i] = 0;
        __syncthreads();
        for (uint32_t cc = t; cc < nseg; cc += kCT) {
          const uint32_t st = sSt[cc];
          if (st >= w0 && st <= w0 + 32 * kCTbl) atomicOr(&sTbl[(st - w0) >> 5], 1u << (st & 31));
        }
        if (t == 0 && S <= w0 + 32 * kCTbl) atomicOr(&sTbl[(S - w0) >> 5], 1u << (S & 31));
        __syncthreads();
        const uint32_t a0 = __popc(sTbl[2 * t]), a1 = __popc(sTbl[2 * t + 1]);
        uint32_t e, wtot;
        Scan(scan_tmp).ExclusiveSum(a0 + a1, e, wtot);
        sPre[2 * t] = cbase + e;
        sPre[2 * t + 1] = cbase + e + a0;
        __syncthreads();
        const uint32_t wend = min(S, w0 + 32 * kCTbl);
        const uint32_t nch = (wend - w0 + 31) / 32;
        for (uint32_t ch0 = t >> 5; ch0 < nch; ch0 += kCWarps * kCQUnroll) {
          uint4 r[kCQUnroll];
          uint32_t jjs[kCQUnroll], vms[kCQUnroll], qix[kCQUnroll];
          unsigned full = 0;  // chunks with all 128 slots valid (warp-uniform bits)
#pragma unroll
          for (int q = 0; q < kCQUnroll; ++q) {
            const uint32_t ch = ch0 + q * kCWarps;
            r[q] = make_uint4(base, base, base, base);
            jjs[q] = 0;
            vms[q] = 0;
            qix[q] = 0;
            if (ch < nch) {  // warp-uniform
              const uint32_t word = sTbl[ch], nxt = sTbl[ch + 1];
              const uint32_t idx = w0 + 32 * ch + lane;
              if ((word | (nxt & 1u)) == 0u && w0 + 32 * ch + 32 <= wend) {
                // interior chunk (warp-uniform): 32 whole quads of ONE list, no
                // segment start or end inside -- the common case on the hub
                // lists this path reads (ncu on C3: the per-quad segment / mask
                // bookkeeping was 45% of the kernel's instructions)
                const uint32_t jj = sPre[ch] - 1u;
                jjs[q] = jj;
                qix[q] = sQs[jj] + idx;
                r[q] = ldg_cq4(R4 + qix[q]);
                vms[q] = 0xFu;
                full |= 1u << q;
                continue;
              }
              const uint32_t jj = sPre[ch] + __popc(word & le_mask) - 1u;
              jjs[q] = jj;
              if (idx < wend) {
                qix[q] = sQs[jj] + idx;
                r[q] = ldg_cq4(R4 + qix[q]);
                const uint32_t hts = sHt2[jj];
                const bool first = (word >> lane) & 1u;
                const bool last = lane < 31 ? ((word >> (lane + 1)) & 1u) : (nxt & 1u);
                unsigned vm = 0xFu;
                if (first) vm &= (0xFu << (hts & 3u)) & 0xFu;
                if (last) vm &= 0xFu >> (hts >> 2);
                vms[q] = vm;
              }
            }
          }
#pragma unroll
          for (int q = 0; q < kCQUnroll; ++q) {
            // head/tail slots of a quad may hold other lists' (or unwritten)
            // values: masked slots probe bit 0 instead
            const uint32_t xr[4] = {r[q].x, r[q].y, r[q].z, r[q].w};
            unsigned hb = 0;
            if ((full >> q) & 1u) {
#pragma unroll
              for (int s2 = 0; s2 < 4; ++s2) {
                const uint32_t xo = xr[s2] - base;
                hb |= ((sBits[xo >> 5] >> (xo & 31)) & 1u) << s2;
              }
            } else {
#pragma unroll
              for (int s2 = 0; s2 < 4; ++s2) {
                const uint32_t xo = ((vms[q] >> s2) & 1u) ? xr[s2] - base : 0u;
                hb |= ((sBits[xo >> 5] >> (xo & 31)) & 1u) << s2;
              }
              hb &= vms[q];
            }
            apex_cnt += __popc(hb);
            if (TALLY || LIST) {
#pragma unroll
              for (int s2 = 0; s2 < 4; ++s2) {
                const bool found = (hb >> s2) & 1u;
                const uint32_t x = found ? __ldg(nu.data + 4ull * qix[q] + s2) : 0u;  // the id
                if (TALLY && found) {
                  atomicAdd(&out.tally[x], 1ull);
                  atomicAdd(&sCntU[jjs[q]], 1u);
                }
                if (LIST) {
                  const unsigned m = __ballot_sync(FULL, found);
                  if (m) {
                    unsigned long long b0 = 0;
                    if (lane == 0) b0 = atomicAdd(out.cursor, (unsigned long long)__popc(m));
                    b0 = __shfl_sync(FULL, b0, 0);
                    if (found) emit_triple(out, b0 + __popc(m & lt_mask), v, sU[jjs[q]], x);
                  }
                }
              }
            }
          }
        }
        cbase += wtot;
        __syncthreads();
      }
      if (TALLY)
        for (uint32_t cc = t; cc < nseg; cc += kCT)
          if (sCntU[cc]) atomicAdd(&out.tally[sU[cc]], (unsigned long long)sCntU[cc]);
      __syncthreads();
    }
    const uint32_t wsum = __reduce_add_sync(FULL, apex_cnt);
    if (lane == 0 && wsum) atomicAdd(&sApex, (unsigned long long)wsum);
    __syncthreads();
    if (t == 0) {
      if (TALLY && sApex) atomicAdd(&out.tally[v], sApex);
      acc += sApex;
    }
    __syncthreads();
  }
  if (t == 0 && acc) atomicAdd(out.total, acc);
}
