// groupq.cuh -- apex-group warp kernel over 16-byte quads of the middle
// lists (included by intersect.cu; the same groups, staging and reference
// semantics as group.cuh's k_intersect_group: count_node_iterator_n,
// sequential.hpp:74-91, aop_count / SurrogateCount, engines.hpp:38-76).
//
// Each N_u is read as the 16-byte-aligned quads that cover it (LDG.128, head
// and tail slots of a list's first and last quad dropped on the exact path,
// as in quad.cuh), so a lane tests 4 elements per load.  The group filter is
// the inverted blocked two-bit filter keyed by (apex slot, id): word from the
// top hash bits, bits from hash bits 0..4 and 5..9.
#pragma once

#ifndef TG_GQUNROLL
#define TG_GQUNROLL 2
#endif
constexpr int kGQUnroll = TG_GQUNROLL;

__device__ __forceinline__ uint32_t gq_hash(uint32_t x, uint32_t akey) {
  return (x ^ akey) * 0x2545F491u;  // akey = slot * 0x9E3779B9
}

template <bool TALLY, bool LIST, bool FILTER, class Apex>
__global__ void __launch_bounds__(kGWarps * 32, 5)
k_intersect_groupq(Apex A, CsrView nu, uint32_t ulo, uint32_t uhi, CountOut out,
                  uint32_t* __restrict__ big, unsigned long long* __restrict__ big_count,
                  uint64_t big_cap, unsigned long long* __restrict__ chunk_ctr, uint32_t gchunk) {
  __shared__ uint32_t sN[kGWarps][2 * 32];               // group lists, back to back
  __shared__ __align__(1024) uint32_t sBm[kGWarps][kBmWords];  // inverted filter
  __shared__ uint32_t sTbl[kGWarps][kTblWords + kGQUnroll + 1];  // segment starts
  __shared__ uint32_t sQs[kGWarps][32];  // segment: first quad - first item
  __shared__ uint32_t sHt[kGWarps][32];  // segment: head | tail << 2
  // per-warp queue of one quad chunk's filter hits (<= 128): element, apex
  // slot, segment -- checked exactly 32 at a time on full warps (graphs with
  // many triangles, e.g. Watts-Strogatz, hit on most chunks)
  __shared__ uint32_t sQx[kGWarps][128], sQa[kGWarps][128];
  __shared__ uint32_t sQj[(TALLY || LIST) ? kGWarps : 1][(TALLY || LIST) ? 128 : 1];
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
  uint32_t* Bm = sBm[w];
  uint32_t* Tbl = sTbl[w];
#pragma unroll
  for (int i = 0; i < kBmWords / 32; ++i) Bm[lane + 32 * i] = 0xFFFFFFFFu;
  const uint32_t bm_s = (uint32_t)__cvta_generic_to_shared(Bm);
  const uint4* __restrict__ Q4 = reinterpret_cast<const uint4*>(nu.data);
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
        const uint32_t h = gq_hash(x, a * 0x9E3779B9u);
        atomicAnd(&Bm[h >> 24], ~qm_mask(h));
      }
    }
    __syncwarp();
    unsigned long long grp_cnt = 0;
    for (uint32_t jb = 0; jb < E; jb += 32) {
      const uint32_t j = jb + lane;
      uint32_t len = 0, u = 0, a = 0, qs0 = 0, ht = 0;
      if (j < E) {
        u = N[j];
        a = j < 32 ? __popc(astarts & le_mask) - 1u : 0u;
        if (!FILTER || (u >= ulo && u < uhi)) {
          const uint64_t d = nu.desc[u - nu.base];
          const uint32_t l = desc_len(d);
          const uint64_t lo = desc_start(d), end = lo + l;  // slots < 2^34
          qs0 = (uint32_t)(lo >> 2);
          len = l ? (uint32_t)(((end + 3) >> 2) - (lo >> 2)) : 0u;  // quads
          ht = ((uint32_t)lo & 3u) | (((0u - (uint32_t)end) & 3u) << 2);
        }
      }
      uint32_t inc2 = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, inc2, o);
        if ((int)lane >= o) inc2 += t;
      }
      const uint32_t S = __shfl_sync(FULL, inc2, 31);
      if (take == 1 && jb == 0 && 4 * S > kWarpWork) {
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
        sQs[w][c] = qs0 - (inc2 - len);
        sHt[w][c] = ht;
        sSt[w][c] = inc2 - len;
        sSA[w][c] = a;
        if (TALLY || LIST) sU[w][c] = u;
        if (TALLY) sCntU[w][c] = 0;
      }
      __syncwarp();
      const bool has = lane < nseg;
      const uint32_t my_qs = has ? sQs[w][lane] : 0u;
      const uint32_t my_ht = has ? sHt[w][lane] : 0u;
      const uint32_t my_st = has ? sSt[w][lane] : 0xffffffffu;
      const uint32_t my_a = has ? sSA[w][lane] : 0u;
      uint32_t cnt = 0;
      for (uint32_t w0 = 0; w0 < S; w0 += 32 * kTblWords) {
        Tbl[lane] = 0;
        if (lane <= kGQUnroll) Tbl[kTblWords + lane] = 0;
        __syncwarp();
        // segment starts + the first position after the window (start or S)
        if (has && my_st >= w0 && my_st <= w0 + 32 * kTblWords)
          atomicOr(&Tbl[(my_st - w0) >> 5], 1u << (my_st & 31));
        if (lane == 0 && S >= w0 && S <= w0 + 32 * kTblWords)
          atomicOr(&Tbl[(S - w0) >> 5], 1u << (S & 31));
        __syncwarp();
        const uint32_t wend = min(S, w0 + 32 * kTblWords);
        for (uint32_t base0 = w0; base0 < wend; base0 += 32 * kGQUnroll) {
          uint4 r[kGQUnroll];
          uint32_t jjs[kGQUnroll], aks[kGQUnroll];
#pragma unroll
          for (int q = 0; q < kGQUnroll; ++q) {
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
            aks[q] = __shfl_sync(FULL, my_a, jj) * 0x9E3779B9u;
            const uint32_t idx = min(base + lane, S - 1);
            r[q] = ldg_cq4(Q4 + (qs + idx));
          }
          unsigned hb = 0;  // filter hits, 4 bits per chunk
#pragma unroll
          for (int q = 0; q < kGQUnroll; ++q) {
            const uint32_t xq[4] = {r[q].x, r[q].y, r[q].z, r[q].w};
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) {
              const uint32_t h = gq_hash(xq[s2], aks[q]);
              hb |= (unsigned)((qm_mask(h) & lds_u32(bm_s | ((h >> 22) & 0x3FCu))) == 0u)
                    << (4 * q + s2);
            }
          }
          if (!__any_sync(FULL, hb != 0)) continue;
#pragma unroll
          for (int q = 0; q < kGQUnroll; ++q) {
            // drop head/tail slots and lanes past S, then enqueue the hits
            const uint32_t base = base0 + 32 * q;
            const uint32_t word = Tbl[(base - w0) >> 5];
            const uint32_t nxt = Tbl[((base - w0) >> 5) + 1];
            const uint32_t hts = __shfl_sync(FULL, my_ht, jjs[q]);
            const uint32_t aa = __shfl_sync(FULL, my_a, jjs[q]);
            const bool first = (word >> lane) & 1u;
            const bool last = lane < 31 ? ((word >> (lane + 1)) & 1u) : (nxt & 1u);
            // items past this window belong to the next one (an unroll that
            // does not divide the window can reach them): not ours
            unsigned vm = base + lane < wend ? 0xFu : 0u;
            if (first) vm &= (0xFu << (hts & 3u)) & 0xFu;
            if (last) vm &= 0xFu >> (hts >> 2);
            const unsigned hq = (hb >> (4 * q)) & vm;
            if (!__any_sync(FULL, hq != 0)) continue;
            const uint32_t xq[4] = {r[q].x, r[q].y, r[q].z, r[q].w};
            uint32_t nh = 0;
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) {
              const bool hit = (hq >> s2) & 1u;
              const unsigned m = __ballot_sync(FULL, hit);
              const uint32_t pos = nh + __popc(m & lt_mask);
              if (hit) {
                sQx[w][pos] = xq[s2];
                sQa[w][pos] = aa;
                if (TALLY || LIST) sQj[w][pos] = jjs[q];
              }
              nh += __popc(m);
            }
            __syncwarp();
            for (uint32_t i0 = 0; i0 < nh; i0 += 32) {
              const bool in = i0 + lane < nh;
              const uint32_t x = in ? sQx[w][i0 + lane] : kNoItem;
              const uint32_t qa = in ? sQa[w][i0 + lane] : 0u;
              const bool found = in && contains_sub(N + sAex[w][qa], sAh[w][qa], x);
              grp_cnt += found;  // per lane; summed at the end
              if (TALLY && found) {
                const uint32_t qj = sQj[w][i0 + lane];
                atomicAdd(&out.tally[x], 1ull);
                atomicAdd(&sCntU[w][qj], 1u);
                atomicAdd(&sCntV[w][qa], 1u);
              }
              if (LIST) {
                const unsigned m = __ballot_sync(FULL, found);
                if (m) {
                  unsigned long long b0 = 0;
                  if (lane == 0) b0 = atomicAdd(out.cursor, (unsigned long long)__popc(m));
                  b0 = __shfl_sync(FULL, b0, 0);
                  if (found)
                    emit_triple(out, b0 + __popc(m & lt_mask), sAv[w][qa],
                                sU[w][sQj[w][i0 + lane]], x);
                }
              }
            }
            __syncwarp();
          }
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
      Bm[gq_hash(N[j], a * 0x9E3779B9u) >> 24] = 0xFFFFFFFFu;
    }
    __syncwarp();
  }
  }  // chunks
  unsigned long long a2 = acc;  // per-lane partials
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a2 += __shfl_xor_sync(FULL, a2, o);
  if (lane == 0 && a2) atomicAdd(out.total, a2);
}
