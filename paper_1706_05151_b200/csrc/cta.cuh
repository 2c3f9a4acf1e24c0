// cta.cuh -- CTA path of the intersection (apexes with h_v > kWCap), included
// by intersect.cu inside namespace tgb::{anon}.
//
// One 512-thread CTA per long or heavy apex (claimed dynamically; skewed
// graphs such as R-MAT have apexes with h_v in the thousands and
// sum_{u in N_v} h_u in the millions).  N_v is inserted into the two-choice
// bucketed hash set Ht4 in shared memory (<= 1 key per 4-slot bucket), so
// membership is two LDS.128 without a sorted-array search.  The apex's items are
// processed per 512-u batch in windows of 32K items: a window-wide bit table
// of segment starts plus per-word prefix counts give every lane its middle
// vertex u with two broadcast LDS and two POPC; each warp streams 32-item
// chunks (kCUnroll in flight) of consecutive N_u elements.  Lists longer
// than the table capacity are probed by binary search in global memory.

constexpr int kCT = 512;
constexpr int kCWarps = kCT / 32;
constexpr int kCTbl = 1024;      // table words per window: 32768 items
constexpr int kCUnroll = 4;
constexpr uint32_t kCEmpty = 0xffffffffu;  // == kNoItem

template <bool TALLY, bool LIST, bool FILTER, bool WIDE, class Apex>
__global__ void __launch_bounds__(kCT, 2)
k_intersect_cta(Apex A, CsrView nu, uint32_t ulo, uint32_t uhi, CountOut out,
                const uint32_t* __restrict__ big, const unsigned long long* __restrict__ big_count,
                uint64_t big_cap, uint32_t tcap_log2, unsigned long long* __restrict__ work_ctr) {
  using Adj = typename std::conditional<WIDE, long long, uint32_t>::type;
  using Scan = cub::BlockScan<uint32_t, kCT>;
  extern __shared__ __align__(16) uint32_t sHt[];  // hash table, 2^tcap_log2 slots
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ Adj sAdj[kCT];
  __shared__ uint32_t sSt[kCT];
  __shared__ uint32_t sU[kCT];
  __shared__ unsigned sCntU[kCT];
  __shared__ uint32_t sTbl[kCTbl];
  __shared__ uint32_t sPre[kCTbl];
  __shared__ uint32_t sJ[2];
  __shared__ unsigned long long sItem, sApex;
  __shared__ int sOvf;
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
    // two-choice bucketed table of N_v (<= 1 key per 4-slot bucket on
    // average) when it fits, else binary search of the sorted list in HBM
    uint32_t bits = 3;
    while ((1u << bits) < hv) ++bits;
    bool in_ht = (4u << bits) <= tcap;
    const Ht4 H{sHt, 32u - bits};
    // filter in front of the table: 16 bits per key (>= 1024 bits)
    uint32_t bmb = bits + 4;
    if (bmb < 10) bmb = 10;
    if ((1u << (bmb - 5)) > tcap / 8) bmb = 5 + 31 - __clz(tcap / 8);
    uint32_t* Bm = sHt + tcap;
    const uint32_t bshift = 32 - bmb, bwords = 1u << (bmb - 5);
    if (t == 0) sOvf = 0;
    for (uint32_t i = t; i < bwords; i += kCT) Bm[i] = 0;
    if (in_ht)
      for (uint32_t i = t; i < (4u << bits); i += kCT) sHt[i] = kCEmpty;
    __syncthreads();
    for (uint32_t i = t; i < hv; i += kCT) {
      const uint32_t x = L[i];
      if (in_ht && !H.insert(x)) sOvf = 1;
      const uint32_t h = (x * 0x2545F491u) >> bshift;
      atomicOr(&Bm[h >> 5], 1u << (h & 31));
    }
    if (t == 0) {
      sApex = 0;
      sJ[0] = FILTER ? lower_bound_u32(L, hv, ulo) : 0;
      sJ[1] = FILTER ? lower_bound_u32(L, hv, uhi) : hv;
    }
    __syncthreads();
    if (sOvf) in_ht = false;  // an insertion found both buckets full
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
            const uint32_t h = (x * 0x2545F491u) >> bshift;
            const bool hit = x != kNoItem && ((Bm[h >> 5] >> (h & 31)) & 1u);
            if (!__any_sync(FULL, hit)) continue;
            bool found = false;  // exact check of filter hits only
            if (hit) found = in_ht ? H.contains(x) : contains_u32(L, hv, x);
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
