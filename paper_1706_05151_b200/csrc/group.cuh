// group.cuh -- warp path of the intersection, included by intersect.cu inside
// namespace tgb::{anon} (after the helpers it uses).
//
// One warp owns a contiguous range of apex items and processes them in
// GROUPS: consecutive apexes with 2 <= h_v <= kWCap are packed until their
// oriented edges fill the 32 lanes (an apex with 33..64 edges forms a group
// of its own).  Per group, in one pass:
//   * lane j holds oriented edge j = (v_a, u_j) of apex slot a; the group's
//     lists N_{v_a} are staged back to back in shared memory (ID-sorted per
//     apex) with a shared 8192-bit filter keyed by (apex slot, id);
//   * the group's work, sum_j h_{u_j} elements, is flattened over the lanes in
//     32-item chunks (kUnroll in flight); the bit table of segment starts gives
//     each lane its edge jj, hence its apex slot and its element x of N_u;
//   * x is rejected by one filter probe; chunks where some lane hits run the
//     exact branch-free search of the sorted N_{v_a}.
// Per-group setup (descriptor loads, scan, compaction, table) is thus paid
// once per ~32 oriented edges instead of once per apex (PA h_v ~ 20,
// Watts-Strogatz h_v ~ 10).  Longer apexes go to the CTA path's queue, and so
// do apexes whose first 32 middle vertices carry more than kWarpWork items.

constexpr int kGWarps = 8;
// apex items claimed per warp at a time: a launch parameter (32..256) sized so
// every warp gets several chunks

__device__ __forceinline__ uint32_t gkey_hash(uint32_t x, uint32_t a) {
  return ((x ^ (a * 0x9E3779B9u)) * 0x2545F491u) >> 19;  // 13 bits
}

// exact membership in the sorted sub-array a[0..n), n <= 64
__device__ __forceinline__ bool contains_sub(const uint32_t* a, uint32_t n, uint32_t x) {
  uint32_t pos = 0;
#pragma unroll
  for (uint32_t step = 32; step > 0; step >>= 1)
    if (pos + step <= n && a[pos + step - 1] < x) pos += step;
  return pos < n && a[pos] == x;
}
// the same search starting at step TOP (a power of two > n / 2): lists of a
// group of short apexes need fewer than 6 steps
template <uint32_t TOP>
__device__ __forceinline__ bool contains_top(const uint32_t* a, uint32_t n, uint32_t x) {
  uint32_t pos = 0;
#pragma unroll
  for (uint32_t step = TOP; step > 0; step >>= 1)
    if (pos + step <= n && a[pos + step - 1] < x) pos += step;
  return pos < n && a[pos] == x;
}
__device__ __forceinline__ bool contains_steps(const uint32_t* a, uint32_t n, uint32_t x,
                                               uint32_t top) {
  switch (top) {  // warp-uniform
    case 1: return contains_top<1>(a, n, x);
    case 2: return contains_top<2>(a, n, x);
    case 4: return contains_top<4>(a, n, x);
    case 8: return contains_top<8>(a, n, x);
    case 16: return contains_top<16>(a, n, x);
    default: return contains_top<32>(a, n, x);
  }
}

template <bool TALLY, bool LIST, bool FILTER, bool WIDE, class Apex>
__global__ void __launch_bounds__(kGWarps * 32, 5)
k_intersect_group(Apex A, CsrView nu, uint32_t ulo, uint32_t uhi, CountOut out,
                  uint32_t* __restrict__ big, unsigned long long* __restrict__ big_count,
                  uint64_t big_cap, unsigned long long* __restrict__ chunk_ctr, uint32_t gchunk) {
  using Adj = typename std::conditional<WIDE, long long, uint32_t>::type;
  __shared__ uint32_t sN[kGWarps][2 * 32];               // group lists, back to back
  __shared__ uint32_t sBm[kGWarps][kBmWords];             // filter
  __shared__ uint32_t sTbl[kGWarps][kTblWords + kUnroll];  // segment starts
  __shared__ Adj sAdj[kGWarps][32];
  __shared__ uint32_t sSt[kGWarps][32];
  __shared__ uint32_t sSA[kGWarps][32];    // segment -> apex slot
  __shared__ uint32_t sU[kGWarps][32];     // segment -> u (tally / list)
  __shared__ unsigned sCntU[kGWarps][32];  // per-segment found (tally)
  __shared__ uint32_t sAv[kGWarps][32], sAex[kGWarps][32], sAh[kGWarps][32];  // apex slots
  __shared__ unsigned sCntV[kGWarps][32];  // per-apex found (tally)
  __shared__ const uint32_t* sAL[kGWarps][32];  // apex slot -> its list
  // per-warp queue of one iteration's filter hits (<= 32 x kUnroll): the
  // exact searches then run on full warps (Watts-Strogatz: ~1/3 of the
  // elements close a triangle, so nearly every chunk has hits)
  __shared__ uint32_t sQx[kGWarps][32 * kUnroll], sQa[kGWarps][32 * kUnroll];
  __shared__ uint32_t sQj[(TALLY || LIST) ? kGWarps : 1][(TALLY || LIST) ? 32 * kUnroll : 1];
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu;
  const unsigned lt_mask = (1u << lane) - 1u, le_mask = (2u << lane) - 1u;
  uint32_t* N = sN[w];
  uint32_t* Bm = sBm[w];
  uint32_t* Tbl = sTbl[w];
#pragma unroll
  for (int i = 0; i < kBmWords / 32; ++i) Bm[lane + 32 * i] = 0;
  __syncwarp();
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
      if (TALLY) sCntV[w][c] = 0;
    }
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
        const uint32_t h = gkey_hash(x, a);
        atomicOr(&Bm[h >> 5], 1u << (h & 31));
      }
    }
    __syncwarp();
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
            // (idx < wend, not S: items past the window are the next window's)
            if (WIDE) xs[q] = idx < wend ? __ldg(nu.data + ((long long)ad + idx)) : kNoItem;
            else xs[q] = idx < wend ? __ldg(nu.data + (uint32_t)((uint32_t)ad + idx)) : kNoItem;
          }
          unsigned hits = 0;
#pragma unroll
          for (int q = 0; q < kUnroll; ++q) {
            const uint32_t h = gkey_hash(xs[q], as[q]);
            hits |= ((Bm[h >> 5] >> (h & 31)) & (unsigned)(xs[q] != kNoItem)) << q;
          }
          if (!__any_sync(FULL, hits != 0)) continue;
          // enqueue the hits, then search them 32 at a time
          uint32_t nh = 0;
#pragma unroll
          for (int q = 0; q < kUnroll; ++q) {
            const bool hit = (hits >> q) & 1u;
            const unsigned m = __ballot_sync(FULL, hit);
            const uint32_t pos = nh + __popc(m & lt_mask);
            if (hit) {
              sQx[w][pos] = xs[q];
              sQa[w][pos] = as[q];
              if (TALLY || LIST) sQj[w][pos] = jjs[q];
            }
            nh += __popc(m);
          }
          __syncwarp();
          for (uint32_t i0 = 0; i0 < nh; i0 += 32) {
            const bool in = i0 + lane < nh;
            const uint32_t x = in ? sQx[w][i0 + lane] : kNoItem;
            const uint32_t qa = in ? sQa[w][i0 + lane] : 0u;
            const bool found = in && contains_steps(N + sAex[w][qa], sAh[w][qa], x, top);
            const unsigned m = __ballot_sync(FULL, found);
            grp_cnt += __popc(m);
            if (TALLY && found) {
              atomicAdd(&out.tally[x], 1ull);
              atomicAdd(&sCntU[w][sQj[w][i0 + lane]], 1u);
              atomicAdd(&sCntV[w][qa], 1u);
            }
            if (LIST && m) {
              unsigned long long b0 = 0;
              if (lane == 0) b0 = atomicAdd(out.cursor, (unsigned long long)__popc(m));
              b0 = __shfl_sync(FULL, b0, 0);
              if (found)
                emit_triple(out, b0 + __popc(m & lt_mask), sAv[w][qa], sU[w][sQj[w][i0 + lane]],
                            x);
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
    // clear the filter words this group set
    __syncwarp();
    for (uint32_t j = lane; j < E; j += 32) {
      const uint32_t a = j < 32 ? __popc(astarts & ((2u << j) - 1u)) - 1u : 0u;
      Bm[gkey_hash(N[j], a) >> 5] = 0;
    }
    __syncwarp();
  }
  }  // chunks
  if (lane == 0 && acc) atomicAdd(out.total, acc);
}
