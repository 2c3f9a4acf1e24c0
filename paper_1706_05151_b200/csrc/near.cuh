// near.cuh -- locality-aware warp path (variant 6), included by intersect.cu
// inside namespace tgb::{anon} (after lane.cuh, whose constants it shares).
//
// On graphs whose ids carry locality (ring lattices such as Watts-Strogatz,
// meshes, locality-preserving orderings) most members of N_v lie within 32
// ids of v, and so do the elements of the N_u it is intersected with.  The
// apex groups of lane.cuh are kept (lane j owns edge j = (v_a, u_j) and
// walks N_{u_j} in 16-byte quads), but membership in N_{v_a} is one bit of a
// 64-bit REGISTER mask of the members in [v_a - 32, v_a + 32): a subtract, a
// compare, a shift.  Members outside the window ("far", e.g. rewired edges)
// sit in a per-warp list checked only by elements outside the window.  No
// shared-memory table, no filter, no search on the near path.
// Measured on C4 (Watts-Strogatz, ~90% of entries near their row): 25.5 ms
// against 18.2 ms for the flattened scalar group kernel -- per-lane list walks
// diverge and keep few loads in flight -- so it is not selected automatically
// (tg_debug_set_warp_variant(6) runs it; tested in every variant sweep).

constexpr int kNQ = 1;  // quads per lane in flight (4: 37.9 ms on C4, 64 registers)

// x in N_{v}: near x tests one bit of v's window mask; far x the group's far list
__device__ __forceinline__ bool near_member(uint32_t x, uint32_t v, unsigned long long mask,
                                            uint32_t a, uint32_t F, const uint32_t* farU,
                                            const uint32_t* farA) {
  const uint32_t d = x - v + 32u;
  if (d < 64u) return (mask >> d) & 1ull;
  bool f = false;
  for (uint32_t k = 0; k < F; ++k) f |= farU[k] == x && farA[k] == a;
  return f;
}

template <bool TALLY, bool LIST, bool FILTER, class Apex>
__global__ void __launch_bounds__(kLWarps * 32)
k_intersect_near(Apex A, CsrView nu, uint32_t ulo, uint32_t uhi, CountOut out,
                 uint32_t* __restrict__ big, unsigned long long* __restrict__ big_count,
                 uint64_t big_cap, unsigned long long* __restrict__ chunk_ctr, uint32_t gchunk) {
  __shared__ unsigned long long sMask[kLWarps][32];  // apex slot -> near members
  __shared__ uint32_t sFarU[kLWarps][32], sFarA[kLWarps][32];  // far members
  __shared__ uint32_t sAv[kLWarps][32], sAex[kLWarps][32];
  __shared__ const uint32_t* sAL[kLWarps][32];
  __shared__ unsigned sCntV[TALLY ? kLWarps : 1][32];
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu;
  const unsigned lt_mask = (1u << lane) - 1u, le_mask = (2u << lane) - 1u;
  unsigned long long* Mk = sMask[w];
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
        Mk[c] = 0ull;
        if (TALLY) sCntV[w][c] = 0;
      }
      const unsigned astarts = __reduce_or_sync(FULL, member ? (1u << excl) : 0u);
      __syncwarp();
      // ---- lane j: edge j = (v_a, u); the group's lists into the table
      const bool act = lane < E;
      const uint32_t a = act ? __popc(astarts & le_mask) - 1u : 0u;
      const uint32_t u = act ? sAL[w][a][lane - sAex[w][a]] : 0u;
      const uint32_t va0 = act ? sAv[w][a] : 0u;
      const uint32_t dn = u - va0 + 32u;  // window offset of u (near: < 64)
      const bool near_u = act && dn < 64u;
      if (near_u) atomicOr(Mk + a, 1ull << dn);
      const unsigned fm = __ballot_sync(FULL, act && !near_u);
      const uint32_t F = __popc(fm);
      if (act && !near_u) {
        const uint32_t fpos = __popc(fm & lt_mask);
        sFarU[w][fpos] = u;
        sFarA[w][fpos] = a;
      }
      __syncwarp();
      const unsigned long long mask = act ? Mk[a] : 0ull;
      uint64_t lo = 0;
      uint32_t len = 0;
      if (act && (!FILTER || (u >= ulo && u < uhi))) {
        const uint64_t d = nu.desc[u - nu.base];
        lo = desc_start(d);
        len = desc_len(d);
      }
      const uint32_t va = va0;
      unsigned cu = 0;  // triangles through edge j (tally of u)
      // ---- short lists: each lane walks its own N_u in 16-byte quads
      const bool shortl = len <= kLLong;
      uint64_t q = lo & ~3ull;
      const uint64_t qe = shortl ? lo + len : 0;
      // kNQ quads (16 elements) in flight per lane before any is tested
      while (__any_sync(FULL, q < qe)) {
        uint4 x4[kNQ];
#pragma unroll
        for (int j = 0; j < kNQ; ++j) {
          x4[j] = make_uint4(kNoItem, kNoItem, kNoItem, kNoItem);
          if (q + 4 * j < qe) x4[j] = __ldg(reinterpret_cast<const uint4*>(nu.data + q + 4 * j));
        }
#pragma unroll
        for (int j = 0; j < kNQ; ++j) {
          const uint32_t xs[4] = {x4[j].x, x4[j].y, x4[j].z, x4[j].w};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const uint64_t at = q + 4 * j + t;
            const bool in = at >= lo && at < qe;
            const bool found = in && near_member(xs[t], va0, mask, a, F, sFarU[w], sFarA[w]);
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
        }
        q += 4 * kNQ;
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
        const unsigned long long mask_s = __shfl_sync(FULL, mask, src);
        const uint32_t u_s = __shfl_sync(FULL, u, src);
        const uint32_t v_s = __shfl_sync(FULL, va, src);
        unsigned got = 0;
        for (uint32_t k0 = 0; k0 < len_s; k0 += 32) {
          const bool ok = k0 + lane < len_s;
          const uint32_t x = ok ? __ldg(nu.data + lo_s + k0 + lane) : kNoItem;
          const bool found = ok && near_member(x, v_s, mask_s, a_s, F, sFarU[w], sFarA[w]);
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
      __syncwarp();  // masks / far lists are rewritten by the next group
    }
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
  if (lane == 0 && acc) atomicAdd(out.total, acc);
}
