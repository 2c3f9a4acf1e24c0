// lane.cuh -- lane-per-edge warp path for short oriented lists, included by
// intersect.cu inside namespace tgb::{anon} (after the helpers it uses).
//
// Watts-Strogatz-like graphs (h_v ~ 10, N_u ~ 10, a third of the elements
// closing a triangle) leave the flattened group kernel issue-bound (~60
// thread instructions per element: per-group scans and segment tables, a
// filter probe, then a binary search for every hit).  Here the group of
// apexes is formed the same way (consecutive apexes, 2 <= h_v <= 32, their
// oriented edges filling the 32 lanes), but then:
//   * the group's lists go into a per-warp open-addressing table keyed by
//     (apex slot, id) -- 128 slots for <= 32 keys, so a probe is one
//     LDS.64 and ~1.1 compares, exact (no filter + search);
//   * lane j owns edge j = (v_a, u_j) and walks N_{u_j} itself in 16-byte
//     quads (LDG.128, 4 elements per load), probing each element;
//   * N_u longer than kLLong is walked by the whole warp, 32 elements per
//     step, after the short lists, so a hub neighbour cannot stall 31 lanes.
// Apexes with h_v > 32 go to the CTA path's queue, as on the group path.

constexpr int kLWarps = 8;
constexpr uint32_t kLSlots = 128;  // table slots per warp (<= 32 keys)
constexpr uint32_t kLLong = 64;    // longer N_u: walked by the whole warp
constexpr unsigned long long kLEmpty = ~0ull;

__device__ __forceinline__ uint32_t lkey_slot(uint32_t x, uint32_t a) {
  return ((x ^ (a * 0x9E3779B9u)) * 0x2545F491u) >> 25;  // 7 bits
}

__device__ __forceinline__ bool lprobe(const unsigned long long* T, uint32_t a, uint32_t x) {
  const unsigned long long key = ((unsigned long long)a << 32) | x;
  uint32_t h = lkey_slot(x, a);
  for (;;) {
    const unsigned long long k = T[h];
    if (k == key) return true;
    if (k == kLEmpty) return false;
    h = (h + 1) & (kLSlots - 1);
  }
}

template <bool TALLY, bool LIST, bool FILTER, class Apex>
__global__ void __launch_bounds__(kLWarps * 32)
k_intersect_lane(Apex A, CsrView nu, uint32_t ulo, uint32_t uhi, CountOut out,
                 uint32_t* __restrict__ big, unsigned long long* __restrict__ big_count,
                 uint64_t big_cap, unsigned long long* __restrict__ chunk_ctr, uint32_t gchunk) {
  __shared__ unsigned long long sT[kLWarps][kLSlots];
  __shared__ uint32_t sAv[kLWarps][32], sAex[kLWarps][32];
  __shared__ const uint32_t* sAL[kLWarps][32];
  __shared__ unsigned sCntV[TALLY ? kLWarps : 1][32];
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu;
  const unsigned lt_mask = (1u << lane) - 1u, le_mask = (2u << lane) - 1u;
  unsigned long long* Tb = sT[w];
#pragma unroll
  for (uint32_t i = 0; i < kLSlots / 32; ++i) Tb[lane + 32 * i] = kLEmpty;
  __syncwarp();
  const uint64_t nitems = A.count();
  unsigned long long acc = 0;
  for (;;) {
    unsigned long long chunk = 0;
    if (lane == 0) chunk = atomicAdd(chunk_ctr, 1ull);
    chunk = __shfl_sync(FULL, chunk, 0);
    const uint64_t ka = chunk * gchunk;
    if (ka >= nitems) break;
    const uint64_t kb = ka + gchunk < nitems ? ka + gchunk : nitems;

    for (uint64_t cur = ka; cur < kb;) {
      // ---- a group: consecutive apexes whose oriented edges fill 32 lanes
      const uint64_t k = cur + lane;
      const bool valid = k < kb;
      uint32_t v = 0, hv = 0;
      const uint32_t* L = nullptr;
      if (valid) A.get(k, v, L, hv);
      const bool small = valid && hv >= 2 && hv <= 32u;
      const uint32_t hh = small ? hv : 0u;
      uint32_t incl = hh;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, incl, o);
        if ((int)lane >= o) incl += t;
      }
      uint32_t take = __popc(__ballot_sync(FULL, incl <= 32u));  // >= 1: hh <= 32
      if (take > kb - cur) take = (uint32_t)(kb - cur);
      const bool in_group = lane < take;
      if (in_group && valid && hv > 32u) {  // long apex -> CTA path
        const unsigned long long pos = atomicAdd(big_count, 1ull);
        if (pos < big_cap) big[pos] = (uint32_t)k;
      }
      const uint32_t E = __shfl_sync(FULL, incl, take - 1);
      cur += take;
      if (E == 0) continue;
      const bool member = in_group && hh > 0;
      const unsigned mm = __ballot_sync(FULL, member);
      const uint32_t excl = incl - hh;
      if (member) {
        const uint32_t c = __popc(mm & lt_mask);
        sAv[w][c] = v;
        sAL[w][c] = L;
        sAex[w][c] = excl;
        if (TALLY) sCntV[w][c] = 0;
      }
      const unsigned astarts = __reduce_or_sync(FULL, member ? (1u << excl) : 0u);
      __syncwarp();
      // ---- lane j: edge j = (v_a, u); the group's lists into the table
      const bool act = lane < E;
      const uint32_t a = act ? __popc(astarts & le_mask) - 1u : 0u;
      const uint32_t u = act ? sAL[w][a][lane - sAex[w][a]] : 0u;
      if (act) {
        const unsigned long long key = ((unsigned long long)a << 32) | u;
        uint32_t h = lkey_slot(u, a);
        while (atomicCAS(Tb + h, kLEmpty, key) != kLEmpty) h = (h + 1) & (kLSlots - 1);
      }
      __syncwarp();
      uint64_t lo = 0;
      uint32_t len = 0;
      if (act && (!FILTER || (u >= ulo && u < uhi))) {
        const uint64_t d = nu.desc[u - nu.base];
        lo = desc_start(d);
        len = desc_len(d);
      }
      const uint32_t va = (TALLY || LIST) && act ? sAv[w][a] : 0u;
      unsigned cu = 0;  // triangles through edge j (tally of u)
      // ---- short lists: each lane walks its own N_u in 16-byte quads
      const bool shortl = len <= kLLong;
      uint64_t q = lo & ~3ull;
      const uint64_t qe = shortl ? lo + len : 0;
      while (__any_sync(FULL, q < qe)) {
        const bool ok = q < qe;
        uint4 x4 = make_uint4(kNoItem, kNoItem, kNoItem, kNoItem);
        if (ok) x4 = __ldg(reinterpret_cast<const uint4*>(nu.data + q));
        const uint32_t xs[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const bool in = ok && q + t >= lo && q + t < qe;
          const bool found = in && lprobe(Tb, a, xs[t]);
          if (TALLY && found) {
            atomicAdd(&out.tally[xs[t]], 1ull);
            atomicAdd(&sCntV[w][a], 1u);
          }
          if (LIST) {
            const unsigned m = __ballot_sync(FULL, found);
            if (m) {
              unsigned long long b0 = 0;
              if (lane == 0) b0 = atomicAdd(out.cursor, (unsigned long long)__popc(m));
              b0 = __shfl_sync(FULL, b0, 0);
              if (found) emit_triple(out, b0 + __popc(m & lt_mask), va, u, xs[t]);
            }
          }
          cu += found;
        }
        q += 4;
      }
      acc += cu;
      // ---- long lists: the whole warp walks each, 32 elements a step
      unsigned lm = __ballot_sync(FULL, act && !shortl);
      while (lm) {
        const int src = __ffs(lm) - 1;
        lm &= lm - 1;
        const uint64_t lo_s = __shfl_sync(FULL, lo, src);
        const uint32_t len_s = __shfl_sync(FULL, len, src);
        const uint32_t a_s = __shfl_sync(FULL, a, src);
        const uint32_t u_s = __shfl_sync(FULL, u, src);
        const uint32_t v_s = __shfl_sync(FULL, va, src);
        unsigned got = 0;
        for (uint32_t k0 = 0; k0 < len_s; k0 += 32) {
          const bool ok = k0 + lane < len_s;
          const uint32_t x = ok ? __ldg(nu.data + lo_s + k0 + lane) : kNoItem;
          const bool found = ok && lprobe(Tb, a_s, x);
          const unsigned m = __ballot_sync(FULL, found);
          got += __popc(m);
          if (TALLY && found) atomicAdd(&out.tally[x], 1ull);
          if (LIST && m) {
            unsigned long long b0 = 0;
            if (lane == 0) b0 = atomicAdd(out.cursor, (unsigned long long)__popc(m));
            b0 = __shfl_sync(FULL, b0, 0);
            if (found) emit_triple(out, b0 + __popc(m & lt_mask), v_s, u_s, x);
          }
        }
        if (lane == src) cu += got;  // tally of u_s below
        if (lane == 0) {
          acc += got;
          if (TALLY && got) atomicAdd(&sCntV[w][a_s], got);
        }
      }
      if (TALLY && act && cu) atomicAdd(&out.tally[u], (unsigned long long)cu);
      __syncwarp();
      if (TALLY) {
        const uint32_t nslots = __popc(mm);
        if (lane < nslots && sCntV[w][lane])
          atomicAdd(&out.tally[sAv[w][lane]], (unsigned long long)sCntV[w][lane]);
      }
      // reset the table for the next group
#pragma unroll
      for (uint32_t i = 0; i < kLSlots / 32; ++i) Tb[lane + 32 * i] = kLEmpty;
      __syncwarp();
    }
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
  if (lane == 0 && acc) atomicAdd(out.total, acc);
}
