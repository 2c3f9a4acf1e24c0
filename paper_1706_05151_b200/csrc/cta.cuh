// cta.cuh -- CTA path of the intersection (apexes with h_v > kWCap), included
// by intersect.cu inside namespace tgb::{anon}.
//
// One 512-thread CTA per long apex (claimed dynamically; skewed graphs such
// as R-MAT have apexes with h_v in the thousands and sum_{u in N_v} h_u in
// the millions).  N_v is inserted into a shared-memory open-addressing hash
// table at load factor <= 1/4 (linear probing, ~1.4 probes per miss), so
// membership is exact without a sorted-array search.  The apex's items are
// processed per 512-u batch in windows of 32K items: a window-wide bit table
// of segment starts plus per-word prefix counts give every lane its middle
// vertex u with two broadcast LDS and two POPC; each warp streams 32-item
// chunks (kCUnroll in flight) of consecutive N_u elements.  Lists longer
// than the table capacity are probed by binary search in global memory.

constexpr int kCT = 512;
constexpr int kCWarps = kCT / 32;
constexpr int kCTbl = 1024;      // table words per window: 32768 items
constexpr int kCUnroll = 4;
constexpr uint32_t kCEmpty = 0xffffffffu;

__device__ __forceinline__ uint32_t ht_hash(uint32_t x, uint32_t shift) {
  return (x * 0x9E3779B1u) >> shift;
}

template <bool TALLY, bool LIST, bool FILTER, bool WIDE, class Apex>
__global__ void __launch_bounds__(kCT, 2)
k_intersect_cta(Apex A, CsrView nu, uint32_t ulo, uint32_t uhi, CountOut out,
                const uint32_t* __restrict__ big, const unsigned long long* __restrict__ big_count,
                uint64_t big_cap, uint32_t tcap_log2, unsigned long long* __restrict__ work_ctr) {
  using Adj = typename std::conditional<WIDE, long long, uint32_t>::type;
  using Scan = cub::BlockScan<uint32_t, kCT>;
  extern __shared__ uint32_t sHt[];  // hash table, 2^tcap_log2 slots
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ Adj sAdj[kCT];
  __shared__ uint32_t sSt[kCT];
  __shared__ uint32_t sU[kCT];
  __shared__ unsigned sCntU[kCT];
  __shared__ uint32_t sTbl[kCTbl];
  __shared__ uint32_t sPre[kCTbl];
  __shared__ uint32_t sJ[2];
  __shared__ unsigned long long sItem, sApex;
  const unsigned t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const unsigned FULL = 0xffffffffu;
  const unsigned lt_mask = (1u << lane) - 1u, le_mask = (2u << lane) - 1u;
  uint64_t nbig = *big_count;
  if (nbig > big_cap) nbig = big_cap;
  const uint32_t tcap = 1u << tcap_log2;
  unsigned long long acc = 0;

  for (;;) {
    if (t == 0) sItem = atomicAdd(work_ctr, 1ull);
    __syncthreads();
    const uint64_t bi = sItem;
    if (bi >= nbig) break;
    uint32_t v, hv;
    const uint32_t* L;
    A.get(big[bi], v, L, hv);
    // table of N_v at load factor <= 1/4 when it fits, else global search
    const bool in_ht = 4ull * hv <= tcap;
    uint32_t tl2 = 5;
    while ((1u << tl2) < 4u * hv && tl2 < tcap_log2) ++tl2;
    const uint32_t tsize = 1u << tl2, tshift = 32 - tl2, tmask = tsize - 1;
    if (in_ht) {
      for (uint32_t i = t; i < tsize; i += kCT) sHt[i] = kCEmpty;
      __syncthreads();
      for (uint32_t i = t; i < hv; i += kCT) {
        const uint32_t x = L[i];
        uint32_t s = ht_hash(x, tshift);
        while (atomicCAS(&sHt[s], kCEmpty, x) != kCEmpty) s = (s + 1) & tmask;
      }
    }
    if (t == 0) {
      sApex = 0;
      sJ[0] = FILTER ? lower_bound_u32(L, hv, ulo) : 0;
      sJ[1] = FILTER ? lower_bound_u32(L, hv, uhi) : hv;
    }
    __syncthreads();
    const uint32_t jlo = sJ[0], jhi = sJ[1];
    unsigned long long apex_cnt = 0;
    for (uint32_t jb = jlo; jb < jhi; jb += kCT) {
      const uint32_t j = jb + t;
      uint32_t len = 0, u = 0;
      uint64_t lo = 0;
      if (j < jhi) {
        u = L[j];
        const uint64_t d = nu.desc[u - nu.base];
        lo = desc_start(d);
        len = desc_len(d);
      }
      uint32_t excl, S;
      Scan(scan_tmp).ExclusiveSum(len, excl, S);
      __syncthreads();
      uint32_t c, nseg;
      Scan(scan_tmp).ExclusiveSum(len > 0 ? 1u : 0u, c, nseg);
      if (len > 0) {
        sAdj[c] = (Adj)((long long)lo - (long long)excl);
        sSt[c] = excl;
        if (TALLY || LIST) sU[c] = u;
        if (TALLY) sCntU[c] = 0;
      }
      __syncthreads();
      uint32_t cbase = 0;  // segment starts before the window
      for (uint32_t w0 = 0; w0 < S; w0 += 32 * kCTbl) {
        for (uint32_t i = t; i < (uint32_t)kCTbl; i += kCT) sTbl[i] = 0;
        __syncthreads();
        for (uint32_t cc = t; cc < nseg; cc += kCT) {
          const uint32_t st = sSt[cc];
          if (st >= w0 && st < w0 + 32 * kCTbl) atomicOr(&sTbl[(st - w0) >> 5], 1u << (st & 31));
        }
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
        for (uint32_t ch0 = wid; ch0 < nch; ch0 += kCWarps * kCUnroll) {
          uint32_t xs[kCUnroll], jjs[kCUnroll];
#pragma unroll
          for (int q = 0; q < kCUnroll; ++q) {
            const uint32_t ch = ch0 + q * kCWarps;
            xs[q] = kNoItem;
            jjs[q] = 0;
            if (ch < nch) {  // warp-uniform
              const uint32_t word = sTbl[ch];
              const uint32_t jj = sPre[ch] + __popc(word & le_mask) - 1u;
              const uint32_t idx = w0 + 32 * ch + lane;
              jjs[q] = jj;
              if (idx < wend) {
                const Adj a = sAdj[jj];
                xs[q] = WIDE ? __ldg(nu.data + ((long long)a + idx))
                             : __ldg(nu.data + (uint32_t)((uint32_t)a + idx));
              }
            }
          }
#pragma unroll
          for (int q = 0; q < kCUnroll; ++q) {
            const uint32_t x = xs[q];
            bool found = false;
            if (x != kNoItem) {
              if (in_ht) {
                uint32_t s = ht_hash(x, tshift);
                for (;;) {
                  const uint32_t k = sHt[s];
                  if (k == x) { found = true; break; }
                  if (k == kCEmpty) break;
                  s = (s + 1) & tmask;
                }
              } else {
                found = contains_u32(L, hv, x);
              }
            }
            const unsigned m = __ballot_sync(FULL, found);
            if (m) {
              apex_cnt += __popc(m);
              if (TALLY && found) {
                atomicAdd(&out.tally[x], 1ull);
                atomicAdd(&sCntU[jjs[q]], 1u);
              }
              if (LIST) {
                unsigned long long b0 = 0;
                if (lane == 0) b0 = atomicAdd(out.cursor, (unsigned long long)__popc(m));
                b0 = __shfl_sync(FULL, b0, 0);
                if (found) emit_triple(out, b0 + __popc(m & lt_mask), v, sU[jjs[q]], x);
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
    if (lane == 0 && apex_cnt) atomicAdd(&sApex, apex_cnt);  // per-warp (replicated) counts
    __syncthreads();
    if (t == 0) {
      if (TALLY && sApex) atomicAdd(&out.tally[v], sApex);
      acc += sApex;
    }
    __syncthreads();
  }
  if (t == 0 && acc) atomicAdd(out.total, acc);
}
