// intersect.cu -- the hot loop: |N_v ∩ N_u| over every oriented edge v -> u.
//
// Reference: count_node_iterator_n (sequential.hpp:74-91) over
// intersect_visit (intersect.hpp:15-33), the AOP rank body aop_count
// (engines.hpp:38-54) and SurrogateCount surrogate_handle (engines.hpp:60-76),
// with the sinks NodeTallySink (sequential.hpp:24-33) and ListSink
// (sequential.hpp:36-46) / RankSink (engines.hpp:303-321).
//
// B200 design (integer set intersection; no tensor cores):
//  * apex-centric: one warp (h_v <= 64) or one 512-thread CTA (longer N_v)
//    owns apex v and stages N_v in shared memory once (an 8192-bit filter +
//    sorted copy for the warp path, an exact hash table for the CTA path), so
//    N_v is read from HBM once per apex instead of once per oriented edge;
//  * the work of the apex, sum_{u in N_v} h_u elements, is flattened across
//    the lanes: each lane takes one element x of one N_u (consecutive lanes
//    read consecutive entries of the same list), finds its u from a bit table
//    of segment starts, and tests x ∈ N_v in shared memory.  A triangle
//    (v,u,x) is found exactly once (Theorem 1).
//  * counts are reduced with __ballot_sync/__popc and one 64-bit atomic per
//    warp per kernel; per-node tallies fold T_v per apex and T_u per edge
//    before touching global atomics; listing compacts found triples with one
//    atomicAdd per warp-iteration.
#include <cub/block/block_scan.cuh>
#include <type_traits>

#include "tg_internal.cuh"

namespace tgb {
namespace {

constexpr int kWarpsPerBlock = 8;  // warp path: 256 threads
constexpr int kWCap = 64;          // apex lists up to 64 entries on the warp path

struct RowsApex {
  CsrView view;
  uint32_t vlo, vhi;
  __device__ __forceinline__ uint64_t count() const { return vhi - vlo; }
  __device__ __forceinline__ uint32_t vertex(uint64_t k) const { return vlo + (uint32_t)k; }
  __device__ __forceinline__ void get(uint64_t k, uint32_t& v, const uint32_t*& L,
                                      uint32_t& hv) const {
    v = vlo + (uint32_t)k;
    const uint64_t d = view.desc[v - view.base];
    L = view.data + desc_start(d);
    hv = desc_len(d);
  }
};

// apexes given as an id list whose length is known only on the device
struct ListApex {
  CsrView view;
  const uint32_t* ids;
  const unsigned long long* n;
  __device__ __forceinline__ uint64_t count() const { return *n; }
  __device__ __forceinline__ uint32_t vertex(uint64_t k) const { return ids[k]; }
  __device__ __forceinline__ void get(uint64_t k, uint32_t& v, const uint32_t*& L,
                                      uint32_t& hv) const {
    v = ids[k];
    const uint64_t d = view.desc[v - view.base];
    L = view.data + desc_start(d);
    hv = desc_len(d);
  }
};

struct MsgApex {
  MsgView m;
  __device__ __forceinline__ uint64_t count() const { return m.count; }
  __device__ __forceinline__ void get(uint64_t k, uint32_t& v, const uint32_t*& L,
                                      uint32_t& hv) const {
    v = m.hdr[2 * k];
    hv = m.hdr[2 * k + 1];
    L = m.data + m.moff[k];
  }
};

// number of elements < x in ascending a[0..n)
__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* a, uint32_t n, uint32_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ bool contains_u32(const uint32_t* a, uint32_t n, uint32_t x) {
  uint32_t i = lower_bound_u32(a, n, x);
  return i < n && a[i] == x;
}

__device__ __forceinline__ void emit_triple(const CountOut& out, unsigned long long pos, uint32_t a,
                                            uint32_t b, uint32_t c) {
  // ListSink normalisation (sequential.hpp:39-44), unless the raw sink
  // order (v, u, w) is asked for
  if (!out.raw) {
    uint32_t t;
    if (a > b) { t = a; a = b; b = t; }
    if (b > c) { t = b; b = c; c = t; }
    if (a > b) { t = a; a = b; b = t; }
  }
  if (pos < out.cap) {
    out.tri[3 * pos + 0] = a;
    out.tri[3 * pos + 1] = b;
    out.tri[3 * pos + 2] = c;
  }
}

// ------------------------------------------------------------- warp path

constexpr int kBmWords = 256;   // per-warp membership filter: 8192 bits
// Blocked two-bit filter: key x sets two bits of ONE word (word = top 8 hash
// bits, bit positions from hash bits 14..23), so a probe is still one LDS.32
// but a non-member passes only if both of its bits are set: ~1/16 of the
// false positives of a one-bit filter of the same size at h_v ~ 30.
__device__ __forceinline__ uint32_t bm_hash(uint32_t x) { return x * 0x2545F491u; }
__device__ __forceinline__ uint32_t bm_word(uint32_t h) { return h >> 24; }
__device__ __forceinline__ uint32_t bm_mask(uint32_t h) {
  return (1u << ((h >> 14) & 31)) | (1u << ((h >> 19) & 31));
}
// Quad-kernel variant of the blocked filter, cheaper to probe: stored
// INVERTED (a cleared bit = present), bit positions from hash bits 0..4 and
// 5..9 (SHF.L.W takes the amount mod 32), word from the top 8 bits, and the
// per-warp filter 1 KB-aligned in shared memory so that the word address is
// base | byte offset.  A probe is IMAD, SHF, LOP3 (address), LDS, SHF, 2x
// SHF.L.W and one LOP3 that tests (b1 | b2) & word == 0.
__device__ __forceinline__ uint32_t qm_mask(uint32_t h) {
  return (1u << (h & 31)) | (1u << ((h >> 5) & 31));
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
// true iff both bits of x are present; bm = shared address of the filter
__device__ __forceinline__ bool qm_probe(uint32_t bm, uint32_t x) {
  const uint32_t h = bm_hash(x);
  return (qm_mask(h) & lds_u32(bm | ((h >> 22) & 0x3FCu))) == 0u;
}

// Branch-free membership in an ascending shared-memory array of n <= 64.
__device__ __forceinline__ bool contains_small(const uint32_t* a, uint32_t n, uint32_t x) {
  uint32_t pos = 0;
#pragma unroll
  for (uint32_t step = 32; step > 0; step >>= 1)
    if (pos + step <= n && a[pos + step - 1] < x) pos += step;
  return pos < n && a[pos] == x;
}
constexpr int kTblWords = 32;   // segment-start table window: 1024 items
#ifndef TG_UNROLL
#define TG_UNROLL 4
#endif
#ifndef TG_WBLOCKS
#define TG_WBLOCKS 6
#endif
#ifndef TG_GUNROLL
#define TG_GUNROLL 4
#endif
constexpr int kUnroll = TG_GUNROLL;  // chunks (of 32 items) in flight per warp (group kernel)
constexpr int kWUnroll = TG_UNROLL;  // ... in the per-apex warp kernel
constexpr int kWBlocks = TG_WBLOCKS; // resident blocks per SM of the per-apex warp kernel
constexpr uint32_t kWarpWork = 4096;  // items of the first u-batch above which
                                      // an apex moves to the CTA path
// Sentinel for "no item" / "empty slot": 0xffffffff is never a NodeId of an
// n < 2^32 graph.
constexpr uint32_t kNoItem = 0xffffffffu;

// Two-choice bucketed hash set of N_v in shared memory: 2^b buckets of 4
// slots (16 B).  A key lives in the less loaded of its two buckets, so a
// lookup is two LDS.128 and eight compares -- exact, branch-free, the same
// cost for members and non-members.  With <= 1 key per bucket on average the
// max load stays ~2-3; an insertion that finds both buckets full sets
// `overflow` and the apex falls back to searching the sorted list.
struct Ht4 {
  uint32_t* slots;  // 4 * 2^bits words, 16-byte aligned, kNoItem = empty
  uint32_t shift;   // 32 - bits
  __device__ __forceinline__ uint32_t b1(uint32_t x) const { return (x * 0x9E3779B1u) >> shift; }
  __device__ __forceinline__ uint32_t b2(uint32_t x) const {
    return ((x ^ 0x5BD1E995u) * 0x85EBCA6Bu) >> shift;
  }
  // x == kNoItem (an idle lane) matches empty slots, so it is excluded
  __device__ __forceinline__ bool contains(uint32_t x) const {
    const uint4 a = *reinterpret_cast<const uint4*>(slots + 4 * b1(x));
    const uint4 c = *reinterpret_cast<const uint4*>(slots + 4 * b2(x));
    return ((a.x == x) | (a.y == x) | (a.z == x) | (a.w == x) | (c.x == x) | (c.y == x) |
            (c.z == x) | (c.w == x)) &
           (x != kNoItem);
  }
  // concurrent insertion (atomicCAS); false when both buckets are full
  __device__ __forceinline__ bool insert(uint32_t x) const {
    const uint32_t ba = b1(x), bb = b2(x);
    const volatile uint32_t* vs = slots;
    for (;;) {
      int la = 0, lc = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        la += vs[4 * ba + i] != kNoItem;
        lc += vs[4 * bb + i] != kNoItem;
      }
      if (la == 4 && lc == 4) return false;
      const uint32_t bk = (la <= lc) ? ba : bb;
      const int l = (la <= lc) ? la : lc;
      if (atomicCAS(slots + 4 * bk + l, kNoItem, x) == kNoItem) return true;
    }
  }
};

// One warp per apex v (h_v <= kWCap).
//  * N_v is staged in shared memory, ID-sorted, with an 8192-bit hashed
//    filter.
//  * The apex's work, sum_{u in N_v} h_u elements, is flattened over the
//    lanes in 32-item chunks; kUnroll chunks are loaded before any is used.
//  * A lane finds the segment (middle vertex u) of its item from a per-window
//    bit table of segment starts: jj = #starts <= item - 1 (one broadcast LDS,
//    two POPCs), then fetches its element x of N_u (consecutive lanes read
//    consecutive addresses of the same list).
//  * x is rejected by one filter probe (one LDS.32 per lane); only chunks in
//    which some lane hits (members + ~0.3% false positives) run the exact
//    branch-free 6-step search of N_v; __ballot / __popc count the triangles.
// FILTER restricts the middle vertex to [ulo, uhi) (SurrogateCount's core
// range); WIDE selects 64-bit element indexing (> 2^32 list entries).
template <bool TALLY, bool LIST, bool FILTER, bool WIDE, class Apex>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, kWBlocks)
k_intersect_warp(Apex A, CsrView nu, uint32_t ulo, uint32_t uhi, CountOut out,
                 uint32_t* __restrict__ big, unsigned long long* __restrict__ big_count,
                 uint64_t big_cap, unsigned long long* __restrict__ chunk_ctr, uint32_t chunk) {
  using Adj = typename std::conditional<WIDE, long long, uint32_t>::type;
  __shared__ uint32_t sNv[kWarpsPerBlock][kWCap];
  __shared__ uint32_t sBm[kWarpsPerBlock][kBmWords];
  __shared__ uint32_t sTbl[kWarpsPerBlock][kTblWords + kWUnroll];
  __shared__ Adj sAdj[kWarpsPerBlock][32];
  __shared__ uint32_t sSt[kWarpsPerBlock][32];
  __shared__ uint32_t sU[kWarpsPerBlock][32];
  __shared__ unsigned sCntU[kWarpsPerBlock][32];
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu;
  const unsigned lt_mask = (1u << lane) - 1u;
  const unsigned le_mask = (2u << lane) - 1u;  // lane 31 -> 0xffffffff
  const uint64_t nitems = A.count();
  uint32_t* Nv = sNv[w];
  uint32_t* Bm = sBm[w];
#pragma unroll
  for (int i = 0; i < kBmWords / 32; ++i) Bm[lane + 32 * i] = 0;
  uint32_t* Tbl = sTbl[w];
  unsigned long long acc = 0;
  __syncwarp();

  // resident grid; warps claim runs of `chunk` consecutive apexes
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
    // stage N_v + filter; with FILTER count the middle-vertex range [jlo, jhi)
    uint32_t jlo = 0, jhi = hv;
    if (FILTER) jhi = 0;
    for (uint32_t i0 = 0; i0 < hv; i0 += 32) {
      const bool in = i0 + lane < hv;
      uint32_t x = 0;
      if (in) {
        x = L[i0 + lane];
        Nv[i0 + lane] = x;
        const uint32_t h = bm_hash(x);
        atomicOr(&Bm[bm_word(h)], bm_mask(h));
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
      uint32_t len = 0, u = 0;
      uint64_t lo = 0;
      if (j < jhi) {
        u = Nv[j];
        const uint64_t d = nu.desc[u - nu.base];
        lo = desc_start(d);
        len = desc_len(d);
      }
      uint32_t incl = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, incl, o);
        if ((int)lane >= o) incl += t;
      }
      const uint32_t S = __shfl_sync(FULL, incl, 31);
      if (jb == jlo && S > kWarpWork) {
        // heavy apex (short N_v but hub neighbours, e.g. R-MAT): hand the
        // whole apex to the CTA path so one warp cannot become a straggler
        if (lane == 0) {
          unsigned long long pos = atomicAdd(big_count, 1ull);
          if (pos < big_cap) big[pos] = (uint32_t)kc;
        }
        break;
      }
      if (S == 0) continue;
      // compact the non-empty segments: segment c lives in lane c
      const unsigned ne = __ballot_sync(FULL, len > 0);
      const uint32_t nseg = __popc(ne);
      if (len > 0) {
        const uint32_t c = __popc(ne & lt_mask);
        sAdj[w][c] = (Adj)((long long)lo - (long long)(incl - len));
        sSt[w][c] = incl - len;
        if (TALLY || LIST) sU[w][c] = u;
      }
      if (TALLY) sCntU[w][lane] = 0;
      __syncwarp();
      const bool has = lane < nseg;
      const Adj my_adj = has ? sAdj[w][lane] : (Adj)0;
      const uint32_t my_st = has ? sSt[w][lane] : 0xffffffffu;
      uint32_t cnt = 0;  // segment starts before the current chunk
      for (uint32_t w0 = 0; w0 < S; w0 += 32 * kTblWords) {
        Tbl[lane] = 0;
        if (lane < kWUnroll) Tbl[kTblWords + lane] = 0;
        __syncwarp();
        if (has && my_st >= w0 && my_st < w0 + 32 * kTblWords)
          atomicOr(&Tbl[(my_st - w0) >> 5], 1u << (my_st & 31));
        __syncwarp();
        const uint32_t wend = min(S, w0 + 32 * kTblWords);
        for (uint32_t base0 = w0; base0 < wend; base0 += 32 * kWUnroll) {
          uint32_t xs[kWUnroll], jjs[kWUnroll];
#pragma unroll
          for (int q = 0; q < kWUnroll; ++q) {
            const uint32_t base = base0 + 32 * q;
            const uint32_t word = Tbl[(base - w0) >> 5];  // padded: 0 past the window
            const uint32_t jj = cnt + __popc(word & le_mask) - 1u;
            cnt += __popc(word);
            const Adj a = __shfl_sync(FULL, my_adj, jj);  // srcLane is taken mod 32
            const uint32_t idx = base + lane;
            jjs[q] = jj;
            if (WIDE) xs[q] = idx < wend ? __ldg(nu.data + ((long long)a + idx)) : kNoItem;
            else xs[q] = idx < wend ? __ldg(nu.data + (uint32_t)((uint32_t)a + idx)) : kNoItem;
          }
          // filter: one conflict-light LDS.32 per item
          unsigned hits = 0;
#pragma unroll
          for (int q = 0; q < kWUnroll; ++q) {
            const uint32_t h = bm_hash(xs[q]), bm = bm_mask(h);
            hits |= (unsigned)(((Bm[bm_word(h)] & bm) == bm) & (xs[q] != kNoItem)) << q;
          }
          if (!__any_sync(FULL, hits != 0)) continue;
          // exact check of filter hits only: branch-free 6-step search of the
          // sorted N_v (cheaper than a bucket probe at PA/WS list lengths)
          unsigned fnd = 0;
#pragma unroll
          for (int q = 0; q < kWUnroll; ++q)
            if ((hits >> q) & 1u) fnd |= (unsigned)contains_small(Nv, hv, xs[q]) << q;
          if (!__any_sync(FULL, fnd != 0)) continue;
#pragma unroll
          for (int q = 0; q < kWUnroll; ++q) {
            const uint32_t x = xs[q];
            const bool found = (fnd >> q) & 1u;
            {
              const unsigned m = __ballot_sync(FULL, found);
              apex_cnt += __popc(m);
              if (TALLY && found) {
                atomicAdd(&out.tally[x], 1ull);
                atomicAdd(&sCntU[w][jjs[q]], 1u);
              }
              if (LIST && m) {
                unsigned long long b0 = 0;
                if (lane == 0) b0 = atomicAdd(out.cursor, (unsigned long long)__popc(m));
                b0 = __shfl_sync(FULL, b0, 0);
                if (found) emit_triple(out, b0 + __popc(m & lt_mask), v, sU[w][jjs[q]], x);
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
    if (TALLY && lane == 0 && apex_cnt) atomicAdd(&out.tally[v], (unsigned long long)apex_cnt);
    acc += apex_cnt;
    // clear the filter words this apex set
    __syncwarp();
    for (uint32_t i = lane; i < hv; i += 32) Bm[bm_word(bm_hash(Nv[i]))] = 0;
    __syncwarp();
  }
  if (lane == 0 && acc) atomicAdd(out.total, acc);
}

// ------------------------------------------------------------- CTA path

#include "cta.cuh"
#include "group.cuh"
#include "quad.cuh"
#include "slab.cuh"
#include "ctaq.cuh"
#include "groupq.cuh"
#include "ctab.cuh"

template <bool TALLY, bool LIST, bool FILTER, bool WIDE, class Apex>
void launch_warp(const Apex& A, uint64_t items, CsrView nu, uint32_t ulo, uint32_t uhi,
                 const CountOut& out, IntersectScratch& scr, cudaStream_t s) {
  // Apex groups pay off when oriented lists are short (they pack >= 2 apexes
  // per 32 lanes: Watts-Strogatz, G(n,m), R-MAT's tail); PA-like lists
  // (h ~ 20) rarely pair up, and the per-apex kernel is faster there.
  // g_warp_variant: 0 auto, 1 scalar per-apex, 2 groups, 3 quad per-apex,
  // 4 scalar groups (quads need 32-bit element indices: !WIDE)
  // Quads waste ~1.5 head/tail slots per list and quantise a group's short
  // tail; measured: scalar groups win on Watts-Strogatz (mean list 10), quad
  // groups on R-MAT (15.5), quad per-apex on PA (20).
  const int wv = g_warp_variant;
  // slab layout (apex lists = nu's own slabs): one DRAM line per N_u, no
  // descriptors -- the per-apex slab kernel whatever the list lengths
  if constexpr (!std::is_same<Apex, MsgApex>::value) {
    if (nu.slab && A.view.data == nu.data && A.view.desc == nu.desc && (wv == 0 || wv == 3)) {
      const unsigned wgrid = grid_for(items, kWarpsPerBlock, 148u * kSlabBlocks);  // resident
      uint64_t chunk = items / ((uint64_t)wgrid * kWarpsPerBlock * 16);
      chunk = chunk < 1 ? 1 : (chunk > 32 ? 32 : chunk);
      k_intersect_slab<TALLY, LIST, FILTER, Apex><<<wgrid, kWarpsPerBlock * 32, kSlabSmem, s>>>(
          A, nu, ulo, uhi, out, scr.big.p, scr.big_count.p, scr.big.n, scr.big_count.p + 2,
          (uint32_t)chunk);
      TG_CHECK_LAUNCH();
      ++g_launches;
      return;
    }
  }
  const bool groups = wv == 0 ? nu.avg_len <= 16.f : (wv == 2 || wv == 4);
  const bool quads = nu.quad_ok && (wv == 0 ? (!groups || nu.avg_len >= 14.f) : (wv == 2 || wv == 3));
  if (!groups && quads) {  // one apex per warp iteration, quad loads
    const unsigned wgrid = grid_for(items, kWarpsPerBlock, 148u * kWBlocks);  // resident
    uint64_t chunk = items / ((uint64_t)wgrid * kWarpsPerBlock * 16);
    chunk = chunk < 1 ? 1 : (chunk > 32 ? 32 : chunk);
    k_intersect_quad<TALLY, LIST, FILTER, Apex><<<wgrid, kWarpsPerBlock * 32, 0, s>>>(
        A, nu, ulo, uhi, out, scr.big.p, scr.big_count.p, scr.big.n, scr.big_count.p + 2,
        (uint32_t)chunk);
  } else if (!groups) {  // one apex per warp iteration
    const unsigned wgrid = grid_for(items, kWarpsPerBlock, 148u * kWBlocks);  // resident
    uint64_t chunk = items / ((uint64_t)wgrid * kWarpsPerBlock * 16);   // >= 16 runs per warp
    chunk = chunk < 1 ? 1 : (chunk > 32 ? 32 : chunk);
    k_intersect_warp<TALLY, LIST, FILTER, WIDE, Apex><<<wgrid, kWarpsPerBlock * 32, 0, s>>>(
        A, nu, ulo, uhi, out, scr.big.p, scr.big_count.p, scr.big.n, scr.big_count.p + 2,
        (uint32_t)chunk);
  } else {  // apex groups, contiguous item range per warp (resident grid)
    const unsigned ggrid = grid_for(items, kGWarps * 32, 148u * 5u);
    uint64_t chunk = items / ((uint64_t)ggrid * kGWarps * 8);  // >= 8 chunks per warp
    chunk = chunk < 32 ? 32 : (chunk > 256 ? 256 : chunk);
    if (quads)
      k_intersect_groupq<TALLY, LIST, FILTER, Apex><<<ggrid, kGWarps * 32, 0, s>>>(
          A, nu, ulo, uhi, out, scr.big.p, scr.big_count.p, scr.big.n, scr.big_count.p + 2,
          (uint32_t)chunk);
    else
      k_intersect_group<TALLY, LIST, FILTER, WIDE, Apex><<<ggrid, kGWarps * 32, 0, s>>>(
          A, nu, ulo, uhi, out, scr.big.p, scr.big_count.p, scr.big.n, scr.big_count.p + 2,
          (uint32_t)chunk);
  }
  TG_CHECK_LAUNCH();
  ++g_launches;
}

// CTA-path hash table: 2^14 slots (64 KB) holds N_v up to 4096 entries at load
// factor 1/4; g_block_cap (tests) lowers it to exercise the global fallback.
template <bool TALLY, bool LIST, bool FILTER, bool WIDE, class Apex>
void launch_cta(const Apex& A, CsrView nu, uint32_t ulo, uint32_t uhi, const CountOut& out,
                IntersectScratch& scr, cudaStream_t s, const RankView& rv) {
  uint32_t tl2 = 14;
  if (g_block_cap) {
    tl2 = 5;
    while ((1u << tl2) < 4u * g_block_cap) ++tl2;
  }
  const int dyn = (int)((1u << tl2) * 4 + (1u << tl2) / 2);  // table + filter (tcap/8 words)
  if (nu.quad_ok && g_warp_variant != 1) {  // quad loads
    if (rv.rank) {  // apexes whose rank window fits a bitmap (ctab.cuh) first
      const int bdyn = (int)(rv.cap_bits / 8);
      TG_CUDA(cudaFuncSetAttribute(k_intersect_ctab<TALLY, LIST, FILTER, Apex>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, bdyn));
      k_intersect_ctab<TALLY, LIST, FILTER, Apex><<<148 * 2, kCT, bdyn, s>>>(
          A, nu, ulo, uhi, out, scr.big.p, scr.big_count.p, scr.big.n, rv, scr.big_count.p + 3);
      TG_CHECK_LAUNCH();
      ++g_launches;
    }
    TG_CUDA(cudaFuncSetAttribute(k_intersect_ctaq<TALLY, LIST, FILTER, Apex>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
    k_intersect_ctaq<TALLY, LIST, FILTER, Apex><<<148 * 2, kCT, dyn, s>>>(
        A, nu, ulo, uhi, out, scr.big.p, scr.big_count.p, scr.big.n, tl2, scr.big_count.p + 1, rv);
  } else {
    TG_CUDA(cudaFuncSetAttribute(k_intersect_cta<TALLY, LIST, FILTER, WIDE, Apex>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
    k_intersect_cta<TALLY, LIST, FILTER, WIDE, Apex><<<148 * 2, kCT, dyn, s>>>(
        A, nu, ulo, uhi, out, scr.big.p, scr.big_count.p, scr.big.n, tl2, scr.big_count.p + 1);
  }
  TG_CHECK_LAUNCH();
  ++g_launches;
}

template <bool TALLY, bool LIST, class Apex>
void launch_pair(const Apex& A, uint64_t items, CsrView nu, uint32_t ulo, uint32_t uhi,
                 const CountOut& out, IntersectScratch& scr, cudaStream_t s, bool filter,
                 bool wide, const RankView& rv) {
  if (!items) return;
  scr.ensure(items, s);
  // [0]: long-apex queue size, [1]: CTA work counter, [2]: warp-path chunk
  // counter, [3]: bitmap-CTA work counter
  TG_CUDA(cudaMemsetAsync(scr.big_count.p, 0, 4 * sizeof(unsigned long long), s));
  if (filter) {
    if (wide) launch_warp<TALLY, LIST, true, true>(A, items, nu, ulo, uhi, out, scr, s);
    else launch_warp<TALLY, LIST, true, false>(A, items, nu, ulo, uhi, out, scr, s);
  } else {
    if (wide) launch_warp<TALLY, LIST, false, true>(A, items, nu, ulo, uhi, out, scr, s);
    else launch_warp<TALLY, LIST, false, false>(A, items, nu, ulo, uhi, out, scr, s);
  }
  if (filter) {
    if (wide) launch_cta<TALLY, LIST, true, true>(A, nu, ulo, uhi, out, scr, s, rv);
    else launch_cta<TALLY, LIST, true, false>(A, nu, ulo, uhi, out, scr, s, rv);
  } else {
    if (wide) launch_cta<TALLY, LIST, false, true>(A, nu, ulo, uhi, out, scr, s, rv);
    else launch_cta<TALLY, LIST, false, false>(A, nu, ulo, uhi, out, scr, s, rv);
  }
}

template <class Apex>
void dispatch(const Apex& A, uint64_t items, CsrView nu, uint32_t ulo, uint32_t uhi,
              const CountOut& out, IntersectScratch& scr, cudaStream_t s, bool filter,
              uint64_t data_entries, const RankView& rv = RankView{}) {
  const bool tally = out.tally != nullptr, list = out.tri != nullptr;
  const bool wide = data_entries >= (1ull << 32) || g_force_wide;
  nu.quad_ok = data_entries < (1ull << 34);  // quad indices fit 32 bits
  if (tally && list) launch_pair<true, true>(A, items, nu, ulo, uhi, out, scr, s, filter, wide, rv);
  else if (tally) launch_pair<true, false>(A, items, nu, ulo, uhi, out, scr, s, filter, wide, rv);
  else if (list) launch_pair<false, true>(A, items, nu, ulo, uhi, out, scr, s, filter, wide, rv);
  else launch_pair<false, false>(A, items, nu, ulo, uhi, out, scr, s, filter, wide, rv);
}

// rdata[slot] = rank[data[slot]] over every list (a warp per vertex)
__global__ void k_rank_lists(const uint64_t* __restrict__ desc, const uint32_t* __restrict__ data,
                             uint64_t rows, const uint32_t* __restrict__ rank,
                             uint32_t* __restrict__ rdata) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t v = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; v < rows; v += warps) {
    const uint64_t d = desc[v];
    const uint64_t b = desc_start(d);
    const uint32_t h = desc_len(d);
    for (uint32_t i = lane; i < h; i += 32) rdata[b + i] = __ldg(rank + __ldg(data + b + i));
  }
}

__global__ void k_cc(const uint64_t* __restrict__ off, uint64_t n,
                     const unsigned long long* __restrict__ tally, double* __restrict__ c) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t d = off[v + 1] - off[v];
    double r = 0.0;
    if (d >= 2)  // engines.hpp:428-433, IEEE-rounded mul/div, no contraction
      r = __ddiv_rn(__dmul_rn(2.0, (double)tally[v]), __dmul_rn((double)d, (double)(d - 1)));
    c[v] = r;
  }
}

}  // namespace

uint32_t g_block_cap = 0;
int g_warp_variant = 0;
bool g_force_wide = false;

void IntersectScratch::ensure(uint64_t cap, cudaStream_t s) {
  if (big.n < cap) big.alloc(cap, s);
  if (big_count.n < 4) big_count.alloc(4, s);
}

void rank_lists(const DevEff& e, const uint32_t* d_rank, uint32_t* rdata, cudaStream_t s) {
  if (!e.rows) return;
  k_rank_lists<<<grid_for(e.rows * 32, 256, 148u * 32u), 256, 0, s>>>(e.desc.p, e.data.p, e.rows,
                                                                    d_rank, rdata);
  TG_CHECK_LAUNCH();
  ++g_launches;
}

void intersect_rows(CsrView apex, uint32_t vlo, uint32_t vhi, CsrView nu, uint32_t ulo,
                    uint32_t uhi, const CountOut& out, IntersectScratch& scr, cudaStream_t s,
                    uint64_t nu_entries, bool unrestricted, const RankView& rv) {
  RowsApex A{apex, vlo, vhi};
  // the bitmap path reads N_v's rank labels at N_v's slots: apex lists must be nu's
  const RankView r = apex.data == nu.data && apex.desc == nu.desc ? rv : RankView{};
  dispatch(A, (uint64_t)(vhi - vlo), nu, ulo, uhi, out, scr, s, !unrestricted, nu_entries, r);
}

void intersect_list(CsrView apex, const uint32_t* ids, const unsigned long long* d_count,
                    uint64_t max_items, CsrView nu, const CountOut& out, IntersectScratch& scr,
                    cudaStream_t s, uint64_t nu_entries, const RankView& rv) {
  ListApex A{apex, ids, d_count};
  const RankView r = apex.data == nu.data && apex.desc == nu.desc ? rv : RankView{};
  dispatch(A, max_items, nu, 0, 0xffffffffu, out, scr, s, false, nu_entries, r);
}

void intersect_msgs(const MsgView& msgs, CsrView nu, uint32_t ulo, uint32_t uhi,
                    const CountOut& out, IntersectScratch& scr, cudaStream_t s,
                    uint64_t nu_entries) {
  MsgApex A{msgs};
  dispatch(A, msgs.count, nu, ulo, uhi, out, scr, s, true, nu_entries);
}

void clustering_device(const DevGraph& g, const unsigned long long* d_tally, double* d_c,
                       cudaStream_t s) {
  if (!g.n) return;
  k_cc<<<grid_for(g.n, 256), 256, 0, s>>>(g.off.p, g.n, d_tally, d_c);
  TG_CHECK_LAUNCH();
  ++g_launches;
}

}  // namespace tgb
