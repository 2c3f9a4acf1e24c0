// ctaq.cuh -- CTA path over 16-byte quads of the middle lists (included by
// intersect.cu; the same apex queue and reference semantics as k_intersect_cta:
// count_node_iterator_n, sequential.hpp:74-91, aop_count / SurrogateCount,
// engines.hpp:38-76).
//
// One 512-thread CTA per long or heavy apex (claimed dynamically).  N_v goes
// into the two-choice bucketed hash set Ht4 behind an inverted blocked
// two-bit filter (16 bits per key).  The apex's items are the 16-byte-aligned
// quads covering each N_u (head/tail slots masked on the first/last quad of a
// list, as in quad.cuh), processed per 512-u batch in windows of 32K quads
// with a bit table of segment starts and per-word prefix counts; each lane
// loads one quad (LDG.128) per chunk and tests its 4 elements.  On skewed
// graphs most chunks hold filter hits (R-MAT: ~8% of elements are triangle
// closers), so there is no warp-wide skip: each element is probed, the hits
// of a chunk are compacted into a per-warp queue (ballot + popc), and the
// queue is checked exactly 32 at a time (Ht4, or binary search in HBM when
// the table would not fit) so that the hash probes run on full warps.
#pragma once

#ifndef TG_CQUNROLL
#define TG_CQUNROLL 4
#endif
constexpr int kCQUnroll = TG_CQUNROLL;  // quad chunks in flight per warp (ctaq, ctab)
#ifndef TG_CPH_MAX
#define TG_CPH_MAX 256
#endif
constexpr uint32_t kCPhMax = TG_CPH_MAX;  // longest N_v tried as a perfect hash (<= kCT)

template <bool TALLY, bool LIST, bool FILTER, class Apex>
__global__ void __launch_bounds__(kCT, 2)
k_intersect_ctaq(Apex A, CsrView nu, uint32_t ulo, uint32_t uhi, CountOut out,
                 const uint32_t* __restrict__ big, const unsigned long long* __restrict__ big_count,
                 uint64_t big_cap, uint32_t tcap_log2, unsigned long long* __restrict__ work_ctr,
                 RankView skip) {
  using Scan = cub::BlockScan<uint32_t, kCT>;
  extern __shared__ __align__(16) uint32_t sHt[];  // hash table (2^tcap_log2 slots) + filter
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ uint32_t sQs[kCT];  // segment: first quad - first item
  __shared__ uint32_t sHt2[kCT]; // segment: head | tail << 2
  __shared__ uint32_t sSt[kCT];  // segment: first item (quad space)
  __shared__ uint32_t sU[kCT];
  __shared__ unsigned sCntU[kCT];
  __shared__ uint32_t sTbl[kCTbl + 1];
  // per-warp queue of filter hits of one quad chunk (<= 128), checked exactly
  // 32 at a time so that the hash probes run on full warps
  __shared__ uint32_t sQx[kCWarps][128];
  __shared__ uint32_t sQj[(TALLY || LIST) ? kCWarps : 1][(TALLY || LIST) ? 128 : 1];
  __shared__ uint32_t sPre[kCTbl];
  __shared__ uint32_t sJ[2];
  __shared__ unsigned long long sItem, sApex;
  __shared__ int sOvf;
  const unsigned t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const unsigned FULL = 0xffffffffu;
  const unsigned lt_mask = (1u << lane) - 1u, le_mask = (2u << lane) - 1u;
  const uint4* __restrict__ Q4 = reinterpret_cast<const uint4*>(nu.data);
  uint64_t nbig = *big_count;
  if (nbig > big_cap) nbig = big_cap;
  const uint32_t tcap = 1u << tcap_log2;
  unsigned long long acc = 0;
  // Perfect-hash mode (round 2, as in slab.cuh): an N_v of <= kCPhMax keys goes
  // into the table region as a direct-mapped table under the first of 8
  // multipliers that maps its keys to distinct slots; a probe is then one
  // LDS + compare, exact -- no filter, no hit queue, no second search.  The
  // region is kept all-empty between apexes (`dirty` after a hash-set apex).
  bool dirty = true;

  for (;;) {
    if (t == 0) sItem = atomicAdd(work_ctr, 1ull);
    __syncthreads();
    const uint64_t bi = sItem;
    if (bi >= nbig) break;
    uint32_t v, hv;
    const uint32_t* L;
    A.get(big[bi], v, L, hv);
    // apexes whose rank window fits the bitmap path ran on k_intersect_ctab
    if (skip.rank && skip.n - (skip.rank[v] + 1u) <= skip.cap_bits) {
      __syncthreads();  // sItem is rewritten at the loop top
      continue;
    }
    bool use_ph = false;
    uint32_t pmul = 0, pslot = 0;
    const uint32_t psh = 32u - tcap_log2;
    if (hv <= kCPhMax && tcap >= 4096u) {
      if (dirty) {
        for (uint32_t i = t; i < tcap; i += kCT) sHt[i] = kCEmpty;
        dirty = false;
        __syncthreads();
      }
      const uint32_t x = t < hv ? L[t] : kCEmpty;  // one key per thread (kCPhMax <= kCT)
      for (int tr = 0; tr < 8; ++tr) {
        pmul = ph_mul(tr);
        pslot = (x * pmul) >> psh;
        if (t < hv) sHt[pslot] = x;
        __syncthreads();
        if (__syncthreads_and(t >= hv || sHt[pslot] == x)) {
          use_ph = true;
          break;
        }
        if (t < hv) sHt[pslot] = kCEmpty;
        __syncthreads();
      }
    }
    uint32_t bits = 3;
    while ((1u << bits) < hv) ++bits;
    bool in_ht = !use_ph && (4u << bits) <= tcap;
    const Ht4 H{sHt, 32u - bits};
    // inverted blocked filter, 16 bits per key (>= 32 words)
    uint32_t bmb = bits + 4;
    if (bmb < 10) bmb = 10;
    if ((1u << (bmb - 5)) > tcap / 8) bmb = 5 + 31 - __clz(tcap / 8);
    uint32_t* Bm = sHt + tcap;
    const uint32_t wshift = 32 - (bmb - 5), bwords = 1u << (bmb - 5);
    if (t == 0) sOvf = 0;
    if (!use_ph) {
      dirty = dirty || in_ht;
      for (uint32_t i = t; i < bwords; i += kCT) Bm[i] = 0xFFFFFFFFu;
      if (in_ht)
        for (uint32_t i = t; i < (4u << bits); i += kCT) sHt[i] = kCEmpty;
      __syncthreads();
      for (uint32_t i = t; i < hv; i += kCT) {
        const uint32_t x = L[i];
        if (in_ht && !H.insert(x)) sOvf = 1;
        const uint32_t h = bm_hash(x);
        atomicAnd(&Bm[h >> wshift], ~qm_mask(h));
      }
    }
    if (t == 0) {
      sApex = 0;
      sJ[0] = FILTER ? lower_bound_u32(L, hv, ulo) : 0;
      sJ[1] = FILTER ? lower_bound_u32(L, hv, uhi) : hv;
    }
    __syncthreads();
    if (sOvf) in_ht = false;  // an insertion found both buckets full
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
      uint32_t cbase = 0;  // segment starts before the window
      for (uint32_t w0 = 0; w0 < S; w0 += 32 * kCTbl) {
        for (uint32_t i = t; i <= (uint32_t)kCTbl; i += kCT) sTbl[i] = 0;
        __syncthreads();
        // segment starts of the window + the first position after it (a
        // start or S): bit idx+1 set <=> quad idx ends its segment
        for (uint32_t cc = t; cc < nseg; cc += kCT) {
          const uint32_t st = sSt[cc];
          if (st >= w0 && st <= w0 + 32 * kCTbl) atomicOr(&sTbl[(st - w0) >> 5], 1u << (st & 31));
        }
        if (t == 0 && S <= w0 + 32 * kCTbl) atomicOr(&sTbl[(S - w0) >> 5], 1u << (S & 31));
        __syncthreads();
        // per-word exclusive prefix of segment-start counts (2 words / thread)
        const uint32_t a0 = __popc(sTbl[2 * t]), a1 = __popc(sTbl[2 * t + 1]);
        uint32_t e, wtot;
        Scan(scan_tmp).ExclusiveSum(a0 + a1, e, wtot);
        sPre[2 * t] = cbase + e;
        sPre[2 * t + 1] = cbase + e + a0;
        __syncthreads();
        const uint32_t wend = min(S, w0 + 32 * kCTbl);
        const uint32_t nch = (wend - w0 + 31) / 32;
        for (uint32_t ch0 = wid; ch0 < nch; ch0 += kCWarps * kCQUnroll) {
          uint4 r[kCQUnroll];
          uint32_t jjs[kCQUnroll], vms[kCQUnroll];
#pragma unroll
          for (int q = 0; q < kCQUnroll; ++q) {
            const uint32_t ch = ch0 + q * kCWarps;
            r[q] = make_uint4(kNoItem, kNoItem, kNoItem, kNoItem);
            jjs[q] = 0;
            vms[q] = 0;
            if (ch < nch) {  // warp-uniform
              const uint32_t word = sTbl[ch], nxt = sTbl[ch + 1];
              const uint32_t idx = w0 + 32 * ch + lane;
              if ((word | (nxt & 1u)) == 0u && w0 + 32 * ch + 32 <= wend) {
                // interior chunk (warp-uniform): 32 whole quads of one list
                const uint32_t jj = sPre[ch] - 1u;
                jjs[q] = jj;
                r[q] = ldg_cq4(Q4 + (sQs[jj] + idx));
                vms[q] = 0xFu;
                continue;
              }
              const uint32_t jj = sPre[ch] + __popc(word & le_mask) - 1u;
              jjs[q] = jj;
              if (idx < wend) {
                r[q] = ldg_cq4(Q4 + (sQs[jj] + idx));
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
            const uint32_t xq[4] = {r[q].x, r[q].y, r[q].z, r[q].w};
            if (use_ph) {  // (block-uniform) exact probes, no queue
              unsigned fb = 0;
#pragma unroll
              for (int s2 = 0; s2 < 4; ++s2)
                fb |= (unsigned)(sHt[(xq[s2] * pmul) >> psh] == xq[s2]) << s2;
              fb &= vms[q];
              apex_cnt += __popc(fb);
              if (TALLY || LIST) {
#pragma unroll
                for (int s2 = 0; s2 < 4; ++s2) {
                  const bool found = (fb >> s2) & 1u;
                  if (TALLY && found) {
                    atomicAdd(&out.tally[xq[s2]], 1ull);
                    atomicAdd(&sCntU[jjs[q]], 1u);
                  }
                  if (LIST) {
                    const unsigned m = __ballot_sync(FULL, found);
                    if (m) {
                      unsigned long long b0 = 0;
                      if (lane == 0) b0 = atomicAdd(out.cursor, (unsigned long long)__popc(m));
                      b0 = __shfl_sync(FULL, b0, 0);
                      if (found) emit_triple(out, b0 + __popc(m & lt_mask), v, sU[jjs[q]], xq[s2]);
                    }
                  }
                }
              }
              continue;
            }
            // filter (branch-free), then enqueue the hits (warp-aggregated)
            unsigned hb = 0;
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) {
              const uint32_t h = bm_hash(xq[s2]);
              hb |= (unsigned)((qm_mask(h) & Bm[h >> wshift]) == 0u) << s2;
            }
            hb &= vms[q];
            uint32_t nh = 0;
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) {
              const bool hit = (hb >> s2) & 1u;
              const unsigned m = __ballot_sync(FULL, hit);
              const uint32_t pos = nh + __popc(m & lt_mask);
              if (hit) sQx[wid][pos] = xq[s2];
              if ((TALLY || LIST) && hit) sQj[wid][pos] = jjs[q];
              nh += __popc(m);
            }
            __syncwarp();
            for (uint32_t i0 = 0; i0 < nh; i0 += 32) {
              const bool in = i0 + lane < nh;
              const uint32_t x = in ? sQx[wid][i0 + lane] : kNoItem;
              const bool found = in && (in_ht ? H.contains(x) : contains_u32(L, hv, x));
              apex_cnt += found;
              if (TALLY && found) {
                atomicAdd(&out.tally[x], 1ull);
                atomicAdd(&sCntU[sQj[wid][i0 + lane]], 1u);
              }
              if (LIST) {
                const unsigned m = __ballot_sync(FULL, found);
                if (m) {
                  unsigned long long b0 = 0;
                  if (lane == 0) b0 = atomicAdd(out.cursor, (unsigned long long)__popc(m));
                  b0 = __shfl_sync(FULL, b0, 0);
                  if (found)
                    emit_triple(out, b0 + __popc(m & lt_mask), v, sU[sQj[wid][i0 + lane]], x);
                }
              }
            }
            __syncwarp();
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
    if (use_ph && t < hv) sHt[pslot] = kCEmpty;  // the table region stays all-empty
    __syncthreads();
  }
  if (t == 0 && acc) atomicAdd(out.total, acc);
}
