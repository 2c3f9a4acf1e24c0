// groupn.cuh -- locality variant of the flattened group kernel (group.cuh),
// included by intersect.cu after group.cuh.
//
// Same apex groups, staging and flattened 32-item chunks over the middle
// lists as k_intersect_group, but membership in N_{v_a} is exact and O(1)
// without a filter: the members of N_{v_a} within 32 ids of v_a are one bit
// each of a 64-bit per-slot mask in shared memory, the others ("far": e.g.
// rewired edges) sit in a per-group list.  An element x of N_u tests
// (x - v_a + 32) < 64 and one bit -- no hash, no hit queue, no binary search;
// only elements outside the window scan the far list.  Measured on C4
// (Watts-Strogatz, ~90% of entries within the window): 19.3 ms against 18.2
// ms for group.cuh -- the flattened chunk machinery, not the membership test,
// bounds that kernel -- so it is not chosen automatically
// (tg_debug_set_warp_variant(6); tested in every variant sweep).
#pragma once

template <bool TALLY, bool LIST, bool FILTER, bool WIDE, class Apex>
__global__ void __launch_bounds__(kGWarps * 32, 5)
k_intersect_groupn(Apex A, CsrView nu, uint32_t ulo, uint32_t uhi, CountOut out,
                  uint32_t* __restrict__ big, unsigned long long* __restrict__ big_count,
                  uint64_t big_cap, unsigned long long* __restrict__ chunk_ctr, uint32_t gchunk) {
  using Adj = typename std::conditional<WIDE, long long, uint32_t>::type;
  __shared__ uint32_t sN[kGWarps][2 * 32];               // group lists, back to back
  __shared__ unsigned long long sMk[kGWarps][32];         // apex slot -> near members
  __shared__ uint32_t sFarU[kGWarps][64], sFarA[kGWarps][64];  // far members
  __shared__ uint32_t sFarN[kGWarps];
  __shared__ uint32_t sTbl[kGWarps][kTblWords + kUnroll];  // segment starts
  __shared__ Adj sAdj[kGWarps][32];
  __shared__ uint32_t sSt[kGWarps][32];
  __shared__ uint32_t sSA[kGWarps][32];    // segment -> apex slot
  __shared__ uint32_t sU[kGWarps][32];     // segment -> u (tally / list)
  __shared__ unsigned sCntU[kGWarps][32];  // per-segment found (tally)
  __shared__ uint32_t sAv[kGWarps][32], sAex[kGWarps][32], sAh[kGWarps][32];  // apex slots
  __shared__ unsigned sCntV[kGWarps][32];  // per-apex found (tally)
  __shared__ const uint32_t* sAL[kGWarps][32];  // apex slot -> its list
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu;
  const unsigned lt_mask = (1u << lane) - 1u, le_mask = (2u << lane) - 1u;
  uint32_t* N = sN[w];
  unsigned long long* Mk = sMk[w];
  uint32_t* Tbl = sTbl[w];
  // warps claim chunks of `gchunk` consecutive apex items dynamically
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
    // ---- form a group from the next <= 32 apex items
    const uint64_t k = cur + lane;
    const bool valid = k < kb;
    uint32_t v = 0, hv = 0;
    const uint32_t* L = nullptr;
    if (valid) A.get(k, v, L, hv);
    const bool small = valid && hv >= 2 && hv <= (uint32_t)kWCap;
    const uint32_t hh = small ? hv : 0u;
    uint32_t incl = hh;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(FULL, incl, o);
      if ((int)lane >= o) incl += t;
    }
    uint32_t take = __popc(__ballot_sync(FULL, incl <= 32u));
    if (take == 0) take = 1;  // lane 0 alone: 33..64 edges
    if (take > kb - cur) take = (uint32_t)(kb - cur);
    const bool in_group = lane < take;
    if (in_group && valid && hv > (uint32_t)kWCap) {  // long apex -> CTA path
      const unsigned long long pos = atomicAdd(big_count, 1ull);
      if (pos < big_cap) big[pos] = (uint32_t)k;
    }
    const uint32_t E = __shfl_sync(FULL, incl, take - 1);  // edges of the group
    // search depth for the group's lists: largest power of two <= max h
    const uint32_t gmax = __reduce_max_sync(FULL, in_group ? hh : 0u);
    const uint32_t top = gmax ? 1u << (31 - __clz(gmax)) : 1u;
    const uint64_t gcur = cur;
    cur += take;
    if (E == 0) continue;
    // apex slots: compacted non-empty group members
    const bool member = in_group && hh > 0;
    const unsigned mm = __ballot_sync(FULL, member);
    const uint32_t excl = incl - hh;
    if (member) {
      const uint32_t c = __popc(mm & lt_mask);
      sAv[w][c] = v;
      sAL[w][c] = L;
      sAex[w][c] = excl;
      sAh[w][c] = hh;
      Mk[c] = 0ull;
      if (TALLY) sCntV[w][c] = 0;
    }
    if (lane == 0) sFarN[w] = 0;
    // edge j -> apex slot: bit table of apex starts (distinct: hh > 0)
    const unsigned astarts = __reduce_or_sync(FULL, (member && excl < 32) ? (1u << excl) : 0u);
    __syncwarp();
    // stage the group's lists and the filter
    for (uint32_t j0 = 0; j0 < E; j0 += 32) {
      const uint32_t j = j0 + lane;
      if (j < E) {
        const uint32_t a = j < 32 ? __popc(astarts & le_mask) - 1u : 0u;
        const uint32_t x = sAL[w][a][j - sAex[w][a]];
        N[j] = x;
        const uint32_t d = x - sAv[w][a] + 32u;  // window [v - 32, v + 32)
        if (d < 64u) {
          atomicOr(Mk + a, 1ull << d);
        } else {
          const uint32_t f = atomicAdd(&sFarN[w], 1u);
          sFarU[w][f] = x;
          sFarA[w][f] = a;
        }
      }
    }
    __syncwarp();
    const uint32_t F = sFarN[w];
    unsigned long long grp_cnt = 0;
    for (uint32_t jb = 0; jb < E; jb += 32) {
      const uint32_t j = jb + lane;
      uint32_t len = 0, u = 0, a = 0;
      uint64_t lo = 0;
      if (j < E) {
        u = N[j];
        a = j < 32 ? __popc(astarts & le_mask) - 1u : 0u;
        if (!FILTER || (u >= ulo && u < uhi)) {
          const uint64_t d = nu.desc[u - nu.base];
          lo = desc_start(d);
          len = desc_len(d);
        }
      }
      uint32_t inc2 = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, inc2, o);
        if ((int)lane >= o) inc2 += t;
      }
      const uint32_t S = __shfl_sync(FULL, inc2, 31);
      if (take == 1 && jb == 0 && S > kWarpWork) {
        // heavy apex (short N_v, hub neighbours): hand it to the CTA path
        if (lane == 0) {
          const unsigned long long pos = atomicAdd(big_count, 1ull);
          if (pos < big_cap) big[pos] = (uint32_t)gcur;
        }
        break;
      }
      if (S == 0) continue;
      const unsigned ne = __ballot_sync(FULL, len > 0);
      const uint32_t nseg = __popc(ne);
      if (len > 0) {
        const uint32_t c = __popc(ne & lt_mask);
        sAdj[w][c] = (Adj)((long long)lo - (long long)(inc2 - len));
        sSt[w][c] = inc2 - len;
        sSA[w][c] = a;
        if (TALLY || LIST) sU[w][c] = u;
        if (TALLY) sCntU[w][c] = 0;
      }
      __syncwarp();
      const bool has = lane < nseg;
      const Adj my_adj = has ? sAdj[w][lane] : (Adj)0;
      const uint32_t my_st = has ? sSt[w][lane] : 0xffffffffu;
      const uint32_t my_a = has ? sSA[w][lane] : 0u;
      uint32_t cnt = 0;
      for (uint32_t w0 = 0; w0 < S; w0 += 32 * kTblWords) {
        Tbl[lane] = 0;
        if (lane < kUnroll) Tbl[kTblWords + lane] = 0;
        __syncwarp();
        if (has && my_st >= w0 && my_st < w0 + 32 * kTblWords)
          atomicOr(&Tbl[(my_st - w0) >> 5], 1u << (my_st & 31));
        __syncwarp();
        const uint32_t wend = min(S, w0 + 32 * kTblWords);
        for (uint32_t base0 = w0; base0 < wend; base0 += 32 * kUnroll) {
          uint32_t xs[kUnroll], jjs[kUnroll], as[kUnroll];
#pragma unroll
          for (int q = 0; q < kUnroll; ++q) {
            const uint32_t base = base0 + 32 * q;
            const uint32_t word = Tbl[(base - w0) >> 5];  // padded: 0 past the window
            const uint32_t jj = cnt + __popc(word & le_mask) - 1u;
            cnt += __popc(word);
            const Adj ad = __shfl_sync(FULL, my_adj, jj);  // srcLane taken mod 32
            as[q] = __shfl_sync(FULL, my_a, jj);
            const uint32_t idx = base + lane;
            jjs[q] = jj;
            if (WIDE) xs[q] = idx < wend ? __ldg(nu.data + ((long long)ad + idx)) : kNoItem;
            else xs[q] = idx < wend ? __ldg(nu.data + (uint32_t)((uint32_t)ad + idx)) : kNoItem;
          }
#pragma unroll
          for (int q = 0; q < kUnroll; ++q) {
            const uint32_t x = xs[q], a = as[q];
            const uint32_t va = sAv[w][a];
            const uint32_t d = x - va + 32u;
            bool found = false;
            if (x != kNoItem) {
              if (d < 64u) {
                found = (Mk[a] >> d) & 1ull;
              } else {
                for (uint32_t k = 0; k < F; ++k) found |= sFarU[w][k] == x && sFarA[w][k] == a;
              }
            }
            grp_cnt += found;
            if (TALLY && found) {
              atomicAdd(&out.tally[x], 1ull);
              atomicAdd(&sCntU[w][jjs[q]], 1u);
              atomicAdd(&sCntV[w][a], 1u);
            }
            if (LIST) {
              const unsigned m = __ballot_sync(FULL, found);
              if (m) {
                unsigned long long b0 = 0;
                if (lane == 0) b0 = atomicAdd(out.cursor, (unsigned long long)__popc(m));
                b0 = __shfl_sync(FULL, b0, 0);
                if (found) emit_triple(out, b0 + __popc(m & lt_mask), va, sU[w][jjs[q]], x);
              }
            }
          }
          __syncwarp();
        }
        __syncwarp();
      }
      if (TALLY && has && sCntU[w][lane])
        atomicAdd(&out.tally[sU[w][lane]], (unsigned long long)sCntU[w][lane]);
      __syncwarp();
    }
    if (TALLY) {
      const uint32_t nslots = __popc(mm);
      if (lane < nslots && sCntV[w][lane])
        atomicAdd(&out.tally[sAv[w][lane]], (unsigned long long)sCntV[w][lane]);
    }
    acc += grp_cnt;
    __syncwarp();  // masks, far list and N are rewritten by the next group
  }
  }  // chunks
  // (counts are per lane here, not warp-uniform as in group.cuh)
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
  if (lane == 0 && acc) atomicAdd(out.total, acc);
}
