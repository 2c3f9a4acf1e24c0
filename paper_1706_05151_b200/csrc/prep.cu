// prep.cu -- device CSR build, degree-ordered orientation, node costs, plan.
//
// Reference algorithm (paths relative to /root/reference/proj/include/trigraph/):
//   build_graph            graph.hpp:58-85
//   compute_order(ByDegree) order.hpp:95-104
//   effective_adjacency    effective.hpp:37-52
//   node_costs             partition.hpp:45-91
//   compute_boundaries     partition.hpp:116-141
//   ordering_cost          sequential.hpp:95-104
//
// B200 design: everything is a streaming pass over HBM.  build_graph is one
// 64-bit radix sort + unique of directed keys (u<<32|v) (CUB onesweep); the
// degree order needs no sort at all on the hot path: "v precedes u" is the
// comparison (deg v, v) < (deg u, u), evaluated against a 4 B/vertex degree
// array that stays L2-resident (126 MB L2 holds 31M degrees); beyond ~32M
// vertices the comparison reads a monotone 1-byte degree code instead (exact
// degrees only on a bucket tie), which keeps the lookup table in L2.
// Orientation of the whole graph is tile-per-warp (32 vertices, dynamically
// claimed): COUNT writes a keep bitmask over the adjacency, a CUB scan gives
// the compact offsets, FILL streams the mask and writes each N_v ID-sorted
// (effective.hpp:13-16).  Vertices of degree > 256 go to a queue served by
// a CTA-per-vertex kernel so hub lists do not stall a tile.
#include <cub/cub.cuh>

#include "tg_internal.cuh"

namespace tgb {

unsigned long long g_launches = 0;
int g_orient_mode = 0;
int g_slab_mode = 0;

namespace {

template <class F>
void cub_run(cudaStream_t s, F&& f) {
  size_t bytes = 0;
  TG_CUDA(f((void*)nullptr, bytes));
  DBuf<char> tmp(bytes ? bytes : 1, s);
  TG_CUDA(f((void*)tmp.p, bytes));
}

__device__ __forceinline__ bool precedes(uint32_t dv, uint32_t v, uint32_t du, uint32_t u) {
  // order.hpp:95-104: sort by (degree, id); rank[v] < rank[u]
  return dv < du || (dv == du && v < u);
}

unsigned bitlen(uint64_t x) {
  unsigned b = 0;
  while (x) {
    ++b;
    x >>= 1;
  }
  return b;
}

// ---------------------------------------------------------------- build_graph

__global__ void k_make_keys(const uint32_t* __restrict__ pairs, uint64_t E, uint64_t sentinel,
                            uint64_t* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < E;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint2 e = reinterpret_cast<const uint2*>(pairs)[i];
    uint64_t a = sentinel, b = sentinel;
    if (e.x != e.y) {  // graph.hpp:69 self-loops dropped
      a = ((uint64_t)e.x << 32) | e.y;
      b = ((uint64_t)e.y << 32) | e.x;
    }
    keys[2 * i] = a;
    keys[2 * i + 1] = b;
  }
}

__global__ void k_split_keys(const uint64_t* __restrict__ keys, uint64_t m2,
                             uint32_t* __restrict__ adj) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m2;
       i += (uint64_t)gridDim.x * blockDim.x)
    adj[i] = (uint32_t)keys[i];
}

// off[v] = #keys with src < v  (lower_bound of v<<32)
__global__ void k_offsets_from_keys(const uint64_t* __restrict__ keys, uint64_t m2, uint64_t n,
                                    uint64_t* __restrict__ off) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v <= n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t target = v << 32, lo = 0, hi = m2;
    while (lo < hi) {
      uint64_t mid = (lo + hi) >> 1;
      if (keys[mid] < target) lo = mid + 1;
      else hi = mid;
    }
    off[v] = lo;
  }
}

// degrees, their 1-byte codes, and the sum of degrees above `big` (the
// orientation's hub threshold: size of its separate hub-list region)
__global__ void k_degrees(const uint64_t* __restrict__ off, uint64_t n, uint32_t* __restrict__ deg,
                          uint8_t* __restrict__ dcode, uint32_t big,
                          unsigned long long* __restrict__ big_sum) {
  unsigned long long bs = 0;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t d = (uint32_t)(off[v + 1] - off[v]);
    deg[v] = d;
    dcode[v] = degree_code(d);
    if (d > big) bs += d;
  }
  for (int o = 16; o > 0; o >>= 1) bs += __shfl_xor_sync(0xffffffffu, bs, o);
  if ((threadIdx.x & 31) == 0 && bs) atomicAdd(big_sum, bs);
}

// precedes(v, u) from the 1-byte codes, exact degrees only on a bucket tie
__device__ __forceinline__ bool precedes_coded(uint8_t cv, uint32_t v, uint8_t cu, uint32_t u,
                                               const uint32_t* __restrict__ deg) {
  if (cv != cu) return cv < cu;
  if (cv < 240) return v < u;  // equal exact degrees: tie broken by id
  const uint32_t dv = deg[v], du = deg[u];
  return dv < du || (dv == du && v < u);
}

// Order key of a vertex.  CODED 0: its degree; 1: its 1-byte code, when the
// degree array would not stay L2-resident (n beyond ~32M vertices); 2: a
// 4-bit code (two per byte) when even the 1-byte codes would not (n beyond
// ~64M: ncu of the C5 orientation showed 114 of its 131 GB of DRAM reads
// were 128-byte line fills for 1-byte lookups in the 100 MB code table).
// The 16 codes are degree buckets of equal ENDPOINT mass (build_nibble_codes),
// so a random edge's ends rarely share one; a tie inside a bucket that holds
// a single degree (bit of xmask) is decided by the ids, any other by the
// exact degrees.  The apex's own key packs (code << 28) | degree.
__device__ __forceinline__ uint32_t nibble_at(const uint8_t* __restrict__ t, uint32_t v) {
  return ((uint32_t)__ldg(t + (v >> 1)) >> ((v & 1u) * 4u)) & 15u;
}
template <int CODED>
__device__ __forceinline__ uint32_t okey(const uint32_t* __restrict__ deg,
                                         const uint8_t* __restrict__ dcode, uint32_t v) {
  if (CODED == 2) return (nibble_at(dcode, v) << 28) | __ldg(deg + v);
  return CODED ? (uint32_t)__ldg(dcode + v) : __ldg(deg + v);
}
// key of a neighbour (the random lookups)
template <int CODED>
__device__ __forceinline__ uint32_t okey_nb(const uint32_t* __restrict__ deg,
                                            const uint8_t* __restrict__ dcode, uint32_t u) {
  if (CODED == 2) return nibble_at(dcode, u);
  return okey<CODED>(deg, dcode, u);
}
template <int CODED>
__device__ __forceinline__ bool okey_precedes(uint32_t kv, uint32_t v, uint32_t ku, uint32_t u,
                                              const uint32_t* __restrict__ deg, uint32_t xmask = 0) {
  if (CODED == 2) {
    const uint32_t cv = kv >> 28;
    if (cv != ku) return cv < ku;
    if ((xmask >> cv) & 1u) return v < u;  // one degree in the bucket: tie broken by id
    const uint32_t dv = kv & 0x0FFFFFFFu, du = __ldg(deg + u);
    return dv < du || (dv == du && v < u);
  }
  return CODED ? precedes_coded((uint8_t)kv, v, (uint8_t)ku, u, deg) : precedes(kv, v, ku, u);
}

// ---------------------------------------------------------------- orientation

// G lanes per vertex.  MODE 0 counts h_v; MODE 1 writes the ID-sorted N_v
// compactly at cnt_or_off[v-vlo] (ballot prefix keeps adjacency order);
// MODE 2 (gappy, single pass) writes N_v into the first h_v slots of v's
// symmetric slot range and the packed descriptor (sym_off[v], h_v).
template <int G, int MODE>
__global__ void __launch_bounds__(256)
k_orient(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
         const uint32_t* __restrict__ deg, uint32_t vlo, uint32_t vhi,
         uint64_t* __restrict__ cnt_or_off, uint32_t* __restrict__ eff) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned sub = lane & (G - 1);
  const unsigned gbase = lane & ~(G - 1);
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << gbase);
  const unsigned lt = (1u << lane) - 1u;
  const uint64_t groups = ((uint64_t)gridDim.x * blockDim.x) / G;
  for (uint64_t g = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / G;; g += groups) {
    // all lanes of a warp iterate together so __ballot_sync stays legal
    const uint64_t vv = vlo + g;
    const bool active = vv < vhi;
    if (__all_sync(0xffffffffu, !active)) break;
    const uint32_t v = active ? (uint32_t)vv : 0;
    const uint64_t b = active ? off[v] : 0, e = active ? off[v + 1] : 0;
    const uint32_t dv = active ? deg[v] : 0;
    uint64_t wpos = 0;
    if (MODE == 1 && active) wpos = cnt_or_off[v - vlo];
    if (MODE == 2) wpos = b;
    uint64_t c = 0;
    const uint64_t len = e - b;
    uint64_t maxlen = len;  // uniform trip count across the warp
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t t = __shfl_xor_sync(0xffffffffu, maxlen, o);
      maxlen = t > maxlen ? t : maxlen;
    }
    for (uint64_t k0 = 0; k0 < maxlen; k0 += G) {
      const uint64_t k = k0 + sub;
      bool keep = false;
      uint32_t u = 0;
      if (k < len) {
        u = adj[b + k];
        keep = precedes(dv, v, deg[u], u);
      }
      const unsigned bal = __ballot_sync(0xffffffffu, keep) & gmask;
      if (MODE != 0 && keep) eff[wpos + c + __popc(bal & lt)] = u;
      c += __popc(bal);
    }
    if (active && sub == 0) {
      if (MODE == 0) cnt_or_off[v - vlo] = c;
      if (MODE == 2) cnt_or_off[v] = make_desc(b, c);
    }
  }
}

template <int G>
void launch_orient(const DevGraph& g, uint32_t vlo, uint32_t vhi, uint64_t* cnt, uint64_t* off_out,
                   uint32_t* eff, cudaStream_t s) {
  uint64_t rows = vhi - vlo;
  unsigned grid = grid_for(rows * G, 256, 148u * 32u);
  k_orient<G, 0><<<grid, 256, 0, s>>>(g.off.p, g.adj.p, order_key(g), vlo, vhi, cnt, nullptr);
  TG_CHECK_LAUNCH();
  ++g_launches;
  // exclusive scan into off_out[0..rows]
  TG_CUDA(cudaMemsetAsync(off_out, 0, sizeof(uint64_t), s));
  if (rows) {
    cub_run(s, [&](void* t, size_t& b) {
      return cub::DeviceScan::InclusiveSum(t, b, cnt, off_out + 1, (int64_t)rows, s);
    });
    g_launches += 2;  // CUB decoupled look-back scan: init + scan kernels
    k_orient<G, 1><<<grid, 256, 0, s>>>(g.off.p, g.adj.p, order_key(g), vlo, vhi, off_out, eff);
    TG_CHECK_LAUNCH();
    ++g_launches;
  }
}

template <int G>
void launch_orient_gappy(const DevGraph& g, uint64_t* desc, uint32_t* eff, cudaStream_t s) {
  unsigned grid = grid_for(g.n * G, 256, 148u * 32u);
  k_orient<G, 2><<<grid, 256, 0, s>>>(g.off.p, g.adj.p, order_key(g), 0, (uint32_t)g.n, desc, eff);
  TG_CHECK_LAUNCH();
  ++g_launches;
}

// ---- compact orientation, tile-streamed (the hot path) -------------------
//
// One warp per tile of 32 consecutive vertices.  The tile's adjacency
// [off[v0], off[v0+32]) is contiguous, so the warp streams it in coalesced
// 32-item chunks (kOUnroll chunks in flight), finds each item's source vertex
// from a bit table of segment starts, and tests precedes(v, u) against the
// L2-resident degree array.  Two modes, so tiles never wait on each other:
//   COUNT: h_v of each vertex (cumulative kept count at segment ends);
//   FILL : after a scan of h, kept item number k of the tile goes to
//          eff[eoff[v0] + k] -- stream order is vertex order and ID order
//          within a vertex, i.e. exactly the compact EffectiveAdjacency.
constexpr int kOWarps = 8;
constexpr int kOTbl = 32;       // table window: 1024 items
#ifndef TG_OUNROLL
#define TG_OUNROLL 4
#endif
#ifndef TG_OBLOCKS
#define TG_OBLOCKS 5
#endif
constexpr int kOUnroll = TG_OUNROLL;
constexpr int kOBlocks = TG_OBLOCKS;  // resident blocks per SM (launch bounds, grid)

constexpr uint32_t kOBig = 256;  // degree above which a vertex leaves its tile
constexpr uint32_t kOHub = 4096;  // ... and above which a whole CTA orients it (ONE mode)

// Tiles skip "big" vertices (degree > kOBig): their items are removed from the
// tile's item space (so a hub cannot stall one warp), and they are handled by
// k_orient_big (32 lanes per vertex) from a queue the COUNT pass fills.
// Tiles are claimed dynamically (tile_ctr).
//   ONE  : single pass (the hot path): kept item k of the tile goes to
//          eff[tile_b + k] -- each tile's lists back to back at the start of
//          the tile's own adjacency range (ID-sorted, vertex order), no mask,
//          no scan; big vertices write above m2 (k_orient_big1).
//   SLAB : ONE mode writing the slab layout instead: list v
//          in the 32-slot, 128-byte-aligned slab eff[32v, 32v+32), kNoEntry
//          padded; vertices with h_v > 32 are re-oriented by k_orient_big1
//          (full list above the slabs, its first 32 entries in the slab).
template <int MODE, int CODED, bool SLAB = false>
__global__ void __launch_bounds__(kOWarps * 32, kOBlocks)
k_orient_tiles(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
               const uint32_t* __restrict__ deg, const uint8_t* __restrict__ dcode, uint64_t n,
               uint64_t* __restrict__ cnt_or_eoff,
               uint64_t* __restrict__ edesc, uint32_t* __restrict__ eff,
               unsigned long long* __restrict__ tile_ctr, uint32_t* __restrict__ bigq,
               unsigned long long* __restrict__ bigq_n, uint32_t* __restrict__ kmask,
               const uint64_t* __restrict__ hcnt, uint64_t tile_lo = 0,
               uint64_t tile_hi = ~0ull, uint32_t xmask = 0) {
  __shared__ uint32_t sTbl[kOWarps][kOTbl + kOUnroll];
  __shared__ uint32_t sV[kOWarps][32], sDv[kOWarps][32], sSt[kOWarps][32], sSh[kOWarps][32];
  __shared__ uint32_t sCum[kOWarps][32], sAs[kOWarps][32];
  __shared__ uint32_t sHb[SLAB ? kOWarps : 1][32];  // kept entries of the tile before a segment
  constexpr bool FILL = MODE == 1, ONE = MODE == 2;
  static_assert(!SLAB || ONE, "the slab layout is written by the one-pass mode");
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu;
  const unsigned lt_mask = (1u << lane) - 1u, le_mask = (2u << lane) - 1u;
  uint32_t* Tbl = sTbl[w];
  const uint64_t ntiles = min((n + 31) / 32, tile_hi);  // tiles [tile_lo, ntiles)
  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = tile_lo + atomicAdd(tile_ctr, 1ull);
    t = __shfl_sync(FULL, t, 0);
    if (t >= ntiles) break;
    const uint64_t v0 = t * 32;
    const uint64_t v = v0 + lane;
    const bool valid = v < n;
    const uint64_t my_b = valid ? off[v] : 0, my_e = valid ? off[v + 1] : 0;
    const uint32_t my_dv = valid ? okey<CODED>(deg, dcode, (uint32_t)v) : 0;  // order key
    const uint64_t tile_b = __shfl_sync(FULL, my_b, 0);
    const uint32_t len = (uint32_t)(my_e - my_b);
    const bool big = len > kOBig;
    if (SLAB) {  // pad the tile's 32 slabs (4 KB, 8 coalesced 16-byte stores per lane)
      uint4* Q = reinterpret_cast<uint4*>(eff);
      const uint64_t qend = n * (kSlab / 4);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint64_t qi = v0 * (kSlab / 4) + 32 * j + lane;
        if (qi < qend) Q[qi] = make_uint4(kNoEntry, kNoEntry, kNoEntry, kNoEntry);
      }
      __syncwarp();  // ordered before the entries written below
    }
    if (!FILL && !ONE && big) bigq[atomicAdd(bigq_n, 1ull)] = (uint32_t)v;
    if (ONE && big) {  // hubs (> kOHub) from the back of the queue, one CTA each
      if (len > kOHub) bigq[n - 1 - atomicAdd(bigq_n + 2, 1ull)] = (uint32_t)v;
      else bigq[atomicAdd(bigq_n, 1ull)] = (uint32_t)v;
    }
    const uint32_t elen = big ? 0u : len;  // length in the tile's item space
    uint32_t est = elen;                   // -> exclusive prefix of elen
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(FULL, est, o);
      if ((int)lane >= o) est += x;
    }
    const uint32_t S = __shfl_sync(FULL, est, 31);  // tile items (big vertices excluded)
    est -= elen;
    if (S == 0) {
      if (valid && !big) {
        if (ONE) edesc[v] = make_desc(SLAB ? v * kSlab : 0, 0);
        else if (!FILL) cnt_or_eoff[v] = 0;
        else edesc[v] = make_desc(cnt_or_eoff[v], 0);
      }
      continue;
    }
    // FILL: tile-relative output base of each segment, minus its items before
    uint32_t obase = 0;
    uint64_t out_b = 0;
    if (FILL) {
      uint64_t my_o = valid ? cnt_or_eoff[v] : 0;
      out_b = __shfl_sync(FULL, my_o, 0);
      uint32_t hk = 0;  // kept entries of this (non-big) vertex (lists are padded)
      if (valid && !big) hk = (uint32_t)hcnt[v];
      uint32_t kst = hk;  // exclusive prefix of non-big kept counts
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(FULL, kst, o);
        if ((int)lane >= o) kst += x;
      }
      kst -= hk;
      obase = (uint32_t)(my_o - out_b) - kst;
      if (valid && !big) edesc[v] = make_desc(my_o, hk);
    }
    // compact the non-empty segments (non-big vertices with adjacency)
    const unsigned ne = __ballot_sync(FULL, elen > 0);
    const uint32_t nseg = __popc(ne);
    if (elen > 0) {
      const uint32_t c = __popc(ne & lt_mask);
      sV[w][c] = (uint32_t)v;
      sDv[w][c] = my_dv;
      sSt[w][c] = est;
      sAs[w][c] = (uint32_t)(my_b - tile_b) - est;  // item -> adjacency index shift
      if (FILL) sSh[w][c] = obase;                  // item's kept rank -> output shift
    }
    __syncwarp();
    const bool has = lane < nseg;
    const uint32_t c_v = has ? sV[w][lane] : 0, c_dv = has ? sDv[w][lane] : 0;
    const uint32_t c_st = has ? sSt[w][lane] : 0xffffffffu;
    const uint32_t c_sh = (FILL && has) ? sSh[w][lane] : 0;
    const uint32_t c_ash = has ? sAs[w][lane] : 0;
    uint32_t c_end = __shfl_down_sync(FULL, c_st, 1);  // end of compacted segment `lane`
    if (lane + 1 >= nseg) c_end = S;
    uint32_t kept = 0, cnt = 0;
    for (uint32_t w0 = 0; w0 < S; w0 += 32 * kOTbl) {
      Tbl[lane] = 0;
      if (lane < kOUnroll) Tbl[kOTbl + lane] = 0;
      __syncwarp();
      if (has && c_st >= w0 && c_st < w0 + 32 * kOTbl)
        atomicOr(&Tbl[(c_st - w0) >> 5], 1u << (c_st & 31));
      __syncwarp();
      const uint32_t wend = min(S, w0 + 32 * kOTbl);
      for (uint32_t base0 = w0; base0 < wend; base0 += 32 * kOUnroll) {
        uint32_t us[kOUnroll], jjs[kOUnroll], kms[kOUnroll];
#pragma unroll
        for (int q = 0; q < kOUnroll; ++q) {
          const uint32_t base = base0 + 32 * q;
          const uint32_t word = Tbl[(base - w0) >> 5];  // padded: 0 past the window
          const uint32_t jj = cnt + __popc(word & le_mask) - 1u;
          jjs[q] = jj;
          cnt += __popc(word);
          const uint32_t idx = base + lane;
          const uint32_t ash = __shfl_sync(FULL, c_ash, jj);
          if (FILL) {
            // keep decisions recorded by the COUNT pass: bits [tile_b+base, +32)
            const uint64_t pos = tile_b + base;
            const uint32_t sh = (uint32_t)(pos & 31);
            const uint32_t lo = kmask[pos >> 5], hi = sh ? kmask[(pos >> 5) + 1] : 0u;
            const uint32_t vm = base >= wend ? 0u
                                : (wend - base >= 32 ? FULL : ((1u << (wend - base)) - 1u));
            kms[q] = (sh ? ((lo >> sh) | (hi << (32 - sh))) : lo) & vm;
            us[q] = ((kms[q] >> lane) & 1u) ? __ldcs(adj + tile_b + ash + idx) : 0u;
          } else {
            us[q] = idx < wend ? __ldcs(adj + tile_b + ash + idx) : 0u;
          }
        }
        if (FILL) {
#pragma unroll
          for (int q = 0; q < kOUnroll; ++q) {
            const uint32_t km = kms[q];
            const uint32_t ob = __shfl_sync(FULL, c_sh, jjs[q]);
            if ((km >> lane) & 1u) eff[out_b + ob + kept + __popc(km & lt_mask)] = us[q];
            kept += __popc(km);
          }
        } else {
          uint32_t dus[kOUnroll];
#pragma unroll
          for (int q = 0; q < kOUnroll; ++q)
            dus[q] = (base0 + 32 * q + lane < wend) ? okey_nb<CODED>(deg, dcode, us[q]) : 0u;
#pragma unroll
          for (int q = 0; q < kOUnroll; ++q) {
            const uint32_t base = base0 + 32 * q;
            const uint32_t idx = base + lane;
            const uint32_t jj = jjs[q];
            const uint32_t sv = __shfl_sync(FULL, c_v, jj);
            const uint32_t sdv = __shfl_sync(FULL, c_dv, jj);
            const bool keep = idx < wend && okey_precedes<CODED>(sdv, sv, dus[q], us[q], deg, xmask);
            const unsigned km = __ballot_sync(FULL, keep);
            const uint32_t send = __shfl_sync(FULL, c_end, jj);
            if (idx < wend && idx + 1 == send) sCum[w][jj] = kept + __popc(km & le_mask);
            if (SLAB) {
              // rank of a kept entry in its own list = kept entries of the tile
              // before it - those before its segment's first item
              const uint32_t sst = __shfl_sync(FULL, c_st, jj);
              const uint32_t before = kept + __popc(km & lt_mask);
              if (idx < wend && idx == sst) sHb[w][jj] = before;
              __syncwarp();
              const uint32_t r = before - sHb[w][jj & 31u];  // (idle lanes: any slot)
              if (keep && r < kSlab) eff[(uint64_t)sv * kSlab + r] = us[q];
            } else if (ONE && keep) eff[tile_b + kept + __popc(km & lt_mask)] = us[q];
            if (!ONE && lane == 0 && km) {  // record the decisions for the FILL pass
              const uint64_t pos = tile_b + base;
              const uint32_t sh = (uint32_t)(pos & 31);
              atomicOr(&kmask[pos >> 5], km << sh);
              if (sh) atomicOr(&kmask[(pos >> 5) + 1], km >> (32 - sh));
            }
            kept += __popc(km);
          }
        }
      }
      __syncwarp();
    }
    __syncwarp();
    if (!FILL && valid && !big) {
      uint32_t h = 0, hb = 0;
      if (elen > 0) {
        const uint32_t c = __popc(ne & lt_mask);
        hb = c ? sCum[w][c - 1] : 0u;
        h = sCum[w][c] - hb;
      }
      if (SLAB) {
        edesc[v] = make_desc(v * kSlab, h);
        // longer than a slab: whole list above the slabs (k_orient_big1)
        if (h > kSlab) bigq[atomicAdd(bigq_n, 1ull)] = (uint32_t)v;
      } else if (ONE) edesc[v] = make_desc(tile_b + hb, h);
      else cnt_or_eoff[v] = h;
    }
    __syncwarp();
  }
}

// Big vertices: 32 lanes per vertex over a device-side queue.  COUNT writes
// h_v; FILL writes N_v at eoff[v] in adjacency order (ballot prefix).
template <bool FILL, int CODED>
__global__ void __launch_bounds__(256)
k_orient_big(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
             const uint32_t* __restrict__ deg, const uint8_t* __restrict__ dcode,
             const uint32_t* __restrict__ bigq,
             const unsigned long long* __restrict__ bigq_n, uint64_t* __restrict__ cnt_or_eoff,
             uint64_t* __restrict__ edesc, uint32_t* __restrict__ eff,
             uint32_t* __restrict__ kmask) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const uint64_t nq = *bigq_n;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  // keep bits at the real adjacency positions (a separate mask from the tiles')
  auto mask_at = [&](uint64_t pos, uint64_t e) -> uint32_t {
    const uint32_t sh = (uint32_t)(pos & 31);
    const uint32_t lo = kmask[pos >> 5], hi = sh ? kmask[(pos >> 5) + 1] : 0u;
    const uint32_t m = sh ? ((lo >> sh) | (hi << (32 - sh))) : lo;
    return e - pos >= 32 ? m : (m & ((1u << (e - pos)) - 1u));
  };
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < nq; i += warps) {
    const uint32_t v = bigq[i];
    const uint64_t b = off[v], e = off[v + 1];
    const uint32_t cv = okey<CODED>(deg, dcode, v);
    const uint64_t ob = FILL ? cnt_or_eoff[v] : 0;
    uint64_t c = 0;
    for (uint64_t k0 = b; k0 < e; k0 += 64) {
      const uint64_t k1 = k0 + lane, k2 = k0 + 32 + lane;
      unsigned m1, m2;
      uint32_t u1, u2;
      if (FILL) {
        m1 = mask_at(k0, e);
        m2 = k0 + 32 < e ? mask_at(k0 + 32, e) : 0u;
        u1 = ((m1 >> lane) & 1u) ? __ldcs(adj + k1) : 0u;
        u2 = ((m2 >> lane) & 1u) ? __ldcs(adj + k2) : 0u;
        if ((m1 >> lane) & 1u) eff[ob + c + __popc(m1 & lt_mask)] = u1;
        if ((m2 >> lane) & 1u) eff[ob + c + __popc(m1) + __popc(m2 & lt_mask)] = u2;
      } else {
        u1 = k1 < e ? __ldcs(adj + k1) : 0u;
        u2 = k2 < e ? __ldcs(adj + k2) : 0u;
        const uint32_t c1 = k1 < e ? okey_nb<CODED>(deg, dcode, u1) : 0, c2 = k2 < e ? okey_nb<CODED>(deg, dcode, u2) : 0;
        const bool p1 = k1 < e && okey_precedes<CODED>(cv, v, c1, u1, deg);
        const bool p2 = k2 < e && okey_precedes<CODED>(cv, v, c2, u2, deg);
        m1 = __ballot_sync(0xffffffffu, p1);
        m2 = __ballot_sync(0xffffffffu, p2);
        if (lane < 2) {
          const unsigned mm = lane ? m2 : m1;
          const uint64_t pos = k0 + 32 * lane;
          if (mm) {
            const uint32_t sh = (uint32_t)(pos & 31);
            atomicOr(&kmask[pos >> 5], mm << sh);
            if (sh) atomicOr(&kmask[(pos >> 5) + 1], mm >> (32 - sh));
          }
        }
      }
      c += __popc(m1) + __popc(m2);
    }
    if (lane == 0) {
      if (FILL) edesc[v] = make_desc(ob, c);
      else cnt_or_eoff[v] = c;
    }
  }
}

// Big vertices, single pass: v's list goes to a region above m2 reserved
// with one atomic per vertex (d_v slots, h_v used).
//  * hubs (d > kOHub, back of the queue): one 256-thread CTA per hub, in
//    8192-entry segments -- keep masks of the 256 32-entry chunks in shared
//    memory, a block scan of their popcounts, then the kept entries are
//    written (re-read from L1/L2) in adjacency order;
//  * the rest (kOBig < d <= kOHub): one warp per vertex, 32 x kBigU entries
//    per iteration so several loads and lookups are in flight.
// Counters: c[1] medium queue size, c[2] region cursor, c[3] hub queue size,
// c[4] hub claims, c[5] medium claims.
constexpr int kBigU = 4;
// SLAB: the first kSlab kept entries also go to v's slab (padded by the tile
// kernel), and the queue holds the non-big vertices with h_v > kSlab too.
template <int CODED, bool SLAB = false>
__global__ void __launch_bounds__(256)
k_orient_big1(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
              const uint32_t* __restrict__ deg, const uint8_t* __restrict__ dcode,
              const uint32_t* __restrict__ bigq, uint64_t n, unsigned long long* __restrict__ c,
              uint64_t m2, uint64_t* __restrict__ edesc, uint32_t* __restrict__ eff,
              uint32_t xmask = 0) {
  __shared__ uint32_t sM[256], sO[256], sW[8];
  __shared__ unsigned long long sI, sBase;
  const unsigned t = threadIdx.x, lane = t & 31, w = t >> 5;
  const unsigned FULL = 0xffffffffu, lt_mask = (1u << lane) - 1u;
  const uint64_t nh = c[3];
  for (;;) {  // hubs: one CTA each
    if (t == 0) sI = atomicAdd(c + 4, 1ull);
    __syncthreads();
    const uint64_t i = sI;
    if (i >= nh) break;
    const uint32_t v = bigq[n - 1 - i];
    const uint64_t b = off[v], e = off[v + 1];
    const uint32_t cv = okey<CODED>(deg, dcode, v);
    if (t == 0) sBase = m2 + atomicAdd(c + 2, (unsigned long long)(e - b));
    __syncthreads();
    const uint64_t ob = sBase;
    uint64_t kept = 0;
    for (uint64_t s0 = b; s0 < e; s0 += 8192) {
      const uint64_t wb = s0 + 1024 * w;  // this warp's 32 chunks
      for (int ch0 = 0; ch0 < 32; ch0 += kBigU) {
        uint32_t us[kBigU], ks[kBigU];
#pragma unroll
        for (int q = 0; q < kBigU; ++q) {
          const uint64_t k = wb + 32 * (ch0 + q) + lane;
          us[q] = k < e ? __ldg(adj + k) : 0u;
        }
#pragma unroll
        for (int q = 0; q < kBigU; ++q)
          ks[q] = (wb + 32 * (ch0 + q) + lane < e) ? okey_nb<CODED>(deg, dcode, us[q]) : 0u;
#pragma unroll
        for (int q = 0; q < kBigU; ++q) {
          const bool keep =
              wb + 32 * (ch0 + q) + lane < e && okey_precedes<CODED>(cv, v, ks[q], us[q], deg, xmask);
          const unsigned km = __ballot_sync(FULL, keep);
          if (lane == 0) sM[32 * w + ch0 + q] = km;
        }
      }
      __syncthreads();
      // exclusive scan of the chunk popcounts (chunk t)
      const uint32_t pc = __popc(sM[t]);
      uint32_t inc = pc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(FULL, inc, o);
        if ((int)lane >= o) inc += x;
      }
      if (lane == 31) sW[w] = inc;
      __syncthreads();
      uint32_t wpre = 0, tot = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t x = sW[j];
        wpre += (j < (int)w) ? x : 0u;
        tot += x;
      }
      sO[t] = wpre + inc - pc;
      __syncthreads();
      for (int ch = 0; ch < 32; ++ch) {
        const uint32_t km = sM[32 * w + ch];
        if ((km >> lane) & 1u) {
          const uint64_t r = kept + sO[32 * w + ch] + __popc(km & lt_mask);
          const uint32_t x = __ldg(adj + wb + 32 * ch + lane);
          eff[ob + r] = x;
          if (SLAB && r < kSlab) eff[(uint64_t)v * kSlab + r] = x;
        }
      }
      kept += tot;
      __syncthreads();  // sM / sO / sW reused by the next segment
    }
    if (t == 0) edesc[v] = (SLAB && kept <= kSlab) ? make_desc((uint64_t)v * kSlab, kept) : make_desc(ob, kept);
  }
  // medium big vertices: one warp each, claimed dynamically
  const uint64_t nq = c[1];
  for (;;) {
    unsigned long long i = 0;
    if (lane == 0) i = atomicAdd(c + 5, 1ull);
    i = __shfl_sync(FULL, i, 0);
    if (i >= nq) break;
    const uint32_t v = bigq[i];
    const uint64_t b = off[v], e = off[v + 1];
    const uint32_t cv = okey<CODED>(deg, dcode, v);
    unsigned long long ob = 0;
    if (lane == 0) ob = atomicAdd(c + 2, (unsigned long long)(e - b));
    ob = m2 + __shfl_sync(FULL, ob, 0);
    uint64_t kept = 0;
    for (uint64_t k0 = b; k0 < e; k0 += 32 * kBigU) {
      uint32_t us[kBigU], ks[kBigU];
#pragma unroll
      for (int q = 0; q < kBigU; ++q) {
        const uint64_t k = k0 + 32 * q + lane;
        us[q] = k < e ? __ldcs(adj + k) : 0u;
      }
#pragma unroll
      for (int q = 0; q < kBigU; ++q)
        ks[q] = (k0 + 32 * q + lane < e) ? okey_nb<CODED>(deg, dcode, us[q]) : 0u;
#pragma unroll
      for (int q = 0; q < kBigU; ++q) {
        const bool keep =
            k0 + 32 * q + lane < e && okey_precedes<CODED>(cv, v, ks[q], us[q], deg, xmask);
        const unsigned km = __ballot_sync(FULL, keep);
        if (keep) {
          const uint64_t r = kept + __popc(km & lt_mask);
          eff[ob + r] = us[q];
          if (SLAB && r < kSlab) eff[(uint64_t)v * kSlab + r] = us[q];
        }
        kept += __popc(km);
      }
    }
    // (SLAB: a big vertex whose list fits its slab is read from the slab)
    if (lane == 0) edesc[v] = (SLAB && kept <= kSlab) ? make_desc((uint64_t)v * kSlab, kept) : make_desc(ob, kept);
  }
}

__global__ void k_desc_from_off(const uint64_t* __restrict__ off, uint64_t rows,
                                uint64_t* __restrict__ desc) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x)
    desc[r] = make_desc(off[r], off[r + 1] - off[r]);
}

__global__ void k_desc_lens(const uint64_t* __restrict__ desc, uint64_t rows,
                            uint64_t* __restrict__ lens) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x)
    lens[r] = desc_len(desc[r]);
}

__global__ void k_gather_compact(CsrView in, uint64_t rows, const uint64_t* __restrict__ off,
                                 uint32_t* __restrict__ out) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < rows; r += warps) {
    const uint64_t d = in.desc[r];
    const uint64_t st = desc_start(d), o = off[r];
    for (uint32_t i = lane; i < desc_len(d); i += 32) out[o + i] = in.data[st + i];
  }
}

__global__ void k_sum_lens(const uint64_t* __restrict__ desc, uint64_t lo, uint64_t hi,
                           unsigned long long* __restrict__ acc) {
  uint64_t s = 0;
  for (uint64_t r = lo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < hi;
       r += (uint64_t)gridDim.x * blockDim.x)
    s += desc_len(desc[r]);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(acc, (unsigned long long)s);
}

// ---------------------------------------------------------------- costs

__global__ void k_cost_simple(const uint64_t* __restrict__ edesc, const uint32_t* __restrict__ deg,
                              uint64_t n, int kind, uint64_t* __restrict__ f) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t d = deg[v], h = desc_len(edesc[v]), r = 0;
    switch (kind) {
      case TG_COST_N: r = 1; break;
      case TG_COST_D: r = d; break;
      case TG_COST_DH: r = h; break;
      case TG_COST_DDH: r = d * h; break;
      case TG_COST_DH2: r = h * h; break;
      default: r = 0;
    }
    f[v] = r;
  }
}

// DPD (partition.hpp:60-69): sum_{u in N_v} (h_v + h_u)
// NOV (partition.hpp:70-81): sum_{u in adj(v), u precedes v} (h_v + h_u)
// `key` is the order key (degree, or the rank of a non-degree order).
template <bool NOV>
__global__ void __launch_bounds__(256)
k_cost_sum(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
           const uint32_t* __restrict__ deg, CsrView eff, uint64_t n, uint64_t* __restrict__ f) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t v = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; v < n; v += warps) {
    const uint64_t dsc = eff.desc[v];
    const uint64_t hv = desc_len(dsc);
    uint64_t b, e;
    if (NOV) { b = off[v]; e = off[v + 1]; }
    else { b = desc_start(dsc); e = b + hv; }
    const uint32_t dv = deg[v];
    uint64_t s = 0;
    for (uint64_t k = b + lane; k < e; k += 32) {
      const uint32_t u = NOV ? adj[k] : eff.data[k];
      if (!NOV || precedes(deg[u], u, dv, (uint32_t)v)) s += hv + desc_len(eff.desc[u]);
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) f[v] = s;
  }
}

__global__ void k_boundaries(const uint64_t* __restrict__ prefix, uint64_t n, uint64_t p,
                             uint32_t* __restrict__ b) {
  // partition.hpp:128-138, one thread per inner boundary.  Searching [0, n]
  // instead of [b_{j-1}, n] gives the same smallest x because the predicate
  // is monotone in x.
  uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (j == 0) b[0] = 0;
  if (j == 0) b[p] = (uint32_t)n;
  if (j == 0 || j >= p) return;
  uint64_t total = n ? prefix[n - 1] : 0;
  unsigned __int128 target = (unsigned __int128)j * total;
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    uint64_t before = mid == 0 ? 0 : prefix[mid - 1];
    if ((unsigned __int128)p * before >= target) hi = mid;
    else lo = mid + 1;
  }
  b[j] = (uint32_t)lo;
}

__global__ void k_ordering_cost(const uint32_t* __restrict__ deg, const uint64_t* __restrict__ edesc,
                                uint64_t n, unsigned long long* __restrict__ out) {
  uint64_t s = 0;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x)
    s += (uint64_t)deg[v] * desc_len(edesc[v]);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, (unsigned long long)s);
}

__global__ void k_rank_keys(const uint32_t* __restrict__ deg, uint64_t n, uint64_t* __restrict__ k) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x)
    k[v] = ((uint64_t)deg[v] << 32) | v;
}

__global__ void k_rank_scatter(const uint64_t* __restrict__ k, uint64_t n, uint32_t* __restrict__ rank) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    rank[(uint32_t)k[i]] = (uint32_t)i;
}

}  // namespace

// graph.hpp:58-85 on the device.
void build_graph_device(const uint32_t* d_pairs, uint64_t E, uint64_t n_override, DevGraph& g,
                        cudaStream_t s) {
  uint64_t n = n_override;
  if (E) {
    DBuf<uint32_t> mx(1, s);
    cub_run(s, [&](void* t, size_t& b) {
      return cub::DeviceReduce::Max(t, b, d_pairs, mx.p, (int64_t)(2 * E), s);
    });
    ++g_launches;
    uint32_t h = 0;
    TG_CUDA(cudaMemcpyAsync(&h, mx.p, 4, cudaMemcpyDeviceToHost, s));
    TG_CUDA(cudaStreamSynchronize(s));
    if ((uint64_t)h + 1 > n) n = (uint64_t)h + 1;
  }
  TG_REQUIRE(n <= 0xFFFFFFFFull, "build_graph: node ids must fit NodeId (uint32) with n < 2^32");
  g.n = n;
  uint64_t keys_n = 2 * E;
  uint64_t sentinel = n << 32;  // sorts after every real key (src < n)
  unsigned end_bit = 32 + bitlen(n);
  if (end_bit > 64) end_bit = 64;
  DBuf<uint64_t> k1(keys_n ? keys_n : 1, s), k2(keys_n ? keys_n : 1, s);
  uint64_t m2 = 0;
  if (E) {
    k_make_keys<<<grid_for(E, 256), 256, 0, s>>>(d_pairs, E, sentinel, k1.p);
    TG_CHECK_LAUNCH();
    ++g_launches;
    cub_run(s, [&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortKeys(t, b, k1.p, k2.p, (int64_t)keys_n, 0, (int)end_bit, s);
    });
    ++g_launches;
    DBuf<int64_t> nsel(1, s);
    cub_run(s, [&](void* t, size_t& b) {
      return cub::DeviceSelect::Unique(t, b, k2.p, k1.p, nsel.p, (int64_t)keys_n, s);
    });
    ++g_launches;
    int64_t u = 0;
    uint64_t last = 0;
    TG_CUDA(cudaMemcpyAsync(&u, nsel.p, 8, cudaMemcpyDeviceToHost, s));
    TG_CUDA(cudaStreamSynchronize(s));
    if (u > 0) {
      TG_CUDA(cudaMemcpyAsync(&last, k1.p + (u - 1), 8, cudaMemcpyDeviceToHost, s));
      TG_CUDA(cudaStreamSynchronize(s));
    }
    m2 = (uint64_t)u - ((u > 0 && last == sentinel) ? 1 : 0);
  }
  g.m2 = m2;
  g.off.alloc(n + 1, s);
  g.adj.alloc(m2 ? m2 : 1, s);
  if (m2) {
    k_split_keys<<<grid_for(m2, 256), 256, 0, s>>>(k1.p, m2, g.adj.p);
    TG_CHECK_LAUNCH();
    ++g_launches;
  }
  k_offsets_from_keys<<<grid_for(n + 1, 256), 256, 0, s>>>(k1.p, m2, n, g.off.p);
  TG_CHECK_LAUNCH();
  ++g_launches;
  compute_degrees(g, s);
}

void compute_degrees(DevGraph& g, cudaStream_t s) {
  g.deg.alloc(g.n ? g.n : 1, s);
  g.dcode.alloc(g.n ? g.n : 1, s);
  g.big_entries = 0;
  if (g.n) {
    DBuf<unsigned long long> bs(1, s);
    bs.zero();
    k_degrees<<<grid_for(g.n, 256), 256, 0, s>>>(g.off.p, g.n, g.deg.p, g.dcode.p, kOBig, bs.p);
    TG_CHECK_LAUNCH();
    ++g_launches;
    unsigned long long h = 0;
    TG_CUDA(cudaMemcpyAsync(&h, bs.p, 8, cudaMemcpyDeviceToHost, s));
    TG_CUDA(cudaStreamSynchronize(s));
    g.big_entries = h;
  }
}

// ---- 4-bit order codes (okey<2>) ----
// histogram of min(degree, 65535) (block-private for degrees < 2048), the
// degree mass of the clipped bin and the maximum degree
constexpr uint32_t kHistBins = 65536, kHistSmem = 2048;
__global__ void __launch_bounds__(256)
k_deg_hist(const uint32_t* __restrict__ deg, uint64_t n, unsigned long long* __restrict__ hist,
           unsigned long long* __restrict__ top /* [0] clipped mass, [1] max degree */) {
  __shared__ uint32_t sh[kHistSmem];
  for (uint32_t i = threadIdx.x; i < kHistSmem; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  unsigned long long mx = 0;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t d = deg[v];
    mx = d > mx ? d : mx;
    if (d < kHistSmem) atomicAdd(&sh[d], 1u);
    else if (d < kHistBins - 1) atomicAdd(&hist[d], 1ull);
    else {
      atomicAdd(&hist[kHistBins - 1], 1ull);
      atomicAdd(top, (unsigned long long)d);
    }
  }
  atomicMax(top + 1, mx);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < kHistSmem; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], (unsigned long long)sh[i]);
}

struct NibbleThr {
  uint32_t t[16];  // code(d) = #{c in 1..15 : d >= t[c]}
};
__global__ void k_nibble_codes(const uint32_t* __restrict__ deg, uint64_t n, NibbleThr thr,
                               uint32_t* __restrict__ words) {
  // a thread packs the codes of 8 consecutive vertices into one word
  for (uint64_t wi = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; wi * 8 < n;
       wi += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t word = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint64_t v = wi * 8 + i;
      uint32_t c = 0;
      if (v < n) {
        const uint32_t d = deg[v];
#pragma unroll
        for (int k = 1; k < 16; ++k) c += d >= thr.t[k];
      }
      word |= c << (4 * i);
    }
    words[wi] = word;
  }
}

void build_nibble_codes(DevGraph& g, cudaStream_t s) {
  g.nibble = -1;
  if (!g.n) return;
  DBuf<unsigned long long> hist(kHistBins + 2, s);
  hist.zero();
  k_deg_hist<<<148 * 8, 256, 0, s>>>(g.deg.p, g.n, hist.p, hist.p + kHistBins);
  TG_CHECK_LAUNCH();
  ++g_launches;
  std::vector<unsigned long long> h(kHistBins + 2);
  TG_CUDA(cudaMemcpyAsync(h.data(), hist.p, h.size() * 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  if (h[kHistBins + 1] >= (1ull << 28)) return;  // the packed apex key holds 28 degree bits
  // 16 buckets of equal endpoint mass: code(d) = floor(16 cum(d) / total)
  long double total = (long double)h[kHistBins];
  for (uint32_t d = 0; d + 1 < kHistBins; ++d) total += (long double)h[d] * d;
  if (total <= 0) return;
  NibbleThr thr;
  for (int k = 0; k < 16; ++k) thr.t[k] = 0xffffffffu;
  thr.t[0] = 0;
  long double cum = 0;
  uint32_t prev = 0;
  for (uint32_t d = 0; d < kHistBins; ++d) {
    cum += d + 1 < kHistBins ? (long double)h[d] * d : (long double)h[kHistBins];
    uint32_t c = (uint32_t)(16.0L * cum / total);
    c = c > 15 ? 15 : c;
    if (!h[d]) continue;
    for (uint32_t k = prev + 1; k <= c; ++k) thr.t[k] = d;  // first degree with code >= k
    prev = c > prev ? c : prev;
  }
  // buckets holding exactly one degree value (the clipped bin never does)
  uint32_t xmask = 0;
  for (uint32_t k = 0; k < 16; ++k) {
    const uint64_t lo = thr.t[k], hi = k < 15 ? thr.t[k + 1] : 0xffffffffull;
    if (lo == 0xffffffffu) continue;
    uint64_t distinct = 0;
    for (uint64_t d = lo; d < hi && d < kHistBins && distinct < 2; ++d) distinct += h[d] != 0;
    if (hi >= kHistBins - 1) distinct = 2;
    if (distinct <= 1) xmask |= 1u << k;
  }
  const uint64_t words = (g.n + 7) / 8;
  g.dcode4.alloc(words * 4, s);
  k_nibble_codes<<<grid_for(words, 256), 256, 0, s>>>(g.deg.p, g.n, thr, (uint32_t*)g.dcode4.p);
  TG_CHECK_LAUNCH();
  ++g_launches;
  g.xmask = xmask;
  g.nibble = 1;
}

// effective.hpp:37-52 for rows [vlo, vhi), compact layout (partitions, the
// exported EffectiveAdjacency).  One host sync for the entry count.
void orient_rows(const DevGraph& g, uint32_t vlo, uint32_t vhi, DevEff& out, cudaStream_t s) {
  const uint64_t rows = vhi - vlo;
  out.rows = rows;
  out.base = vlo;
  out.compact = true;
  out.off.alloc(rows + 1, s);
  out.desc.alloc(rows ? rows : 1, s);
  DBuf<uint64_t> cnt(rows ? rows : 1, s);
  uint64_t ob[2] = {0, 0};
  TG_CUDA(cudaMemcpyAsync(&ob[0], g.off.p + vlo, 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaMemcpyAsync(&ob[1], g.off.p + vhi, 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  const uint64_t bound = ob[1] - ob[0];  // symmetric entries of the range
  out.data.alloc(bound + kQuadPad, s);
  const uint64_t avg = g.n ? g.m2 / g.n : 0;
  if (avg <= 12) launch_orient<8>(g, vlo, vhi, cnt.p, out.off.p, out.data.p, s);
  else if (avg <= 24) launch_orient<16>(g, vlo, vhi, cnt.p, out.off.p, out.data.p, s);
  else launch_orient<32>(g, vlo, vhi, cnt.p, out.off.p, out.data.p, s);
  if (rows) {
    k_desc_from_off<<<grid_for(rows, 256), 256, 0, s>>>(out.off.p, rows, out.desc.p);
    TG_CHECK_LAUNCH();
    ++g_launches;
  }
  uint64_t entries = 0;
  TG_CUDA(cudaMemcpyAsync(&entries, out.off.p + rows, 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  out.entries = entries;
}

template <int CODED>
static void orient_tiles(const DevGraph& g, DevEff& out, cudaStream_t s) {
  const uint64_t ntiles = (g.n + 31) / 32;
  const unsigned grid = grid_for(ntiles, kOWarps, 148u * kOBlocks);  // resident
  DBuf<uint64_t> cnt(g.n, s);
  DBuf<uint32_t> bigq(g.n, s);
  DBuf<unsigned long long> ctr(3, s);  // tile counters (count, fill), big-queue size
  ctr.zero();
  // keep-decision bitmasks (tiles: compressed item space; big: real positions)
  const uint64_t mwords = g.m2 / 32 + 8;
  DBuf<uint32_t> kmask(2 * mwords, s);
  kmask.zero();
  k_orient_tiles<0, CODED><<<grid, kOWarps * 32, 0, s>>>(g.off.p, g.adj.p, order_key(g), g.dcode.p, g.n, cnt.p,
                                                      nullptr, nullptr, ctr.p, bigq.p, ctr.p + 2,
                                                      kmask.p, nullptr);
  TG_CHECK_LAUNCH();
  k_orient_big<false, CODED><<<148 * 8, 256, 0, s>>>(g.off.p, g.adj.p, order_key(g), g.dcode.p, bigq.p, ctr.p + 2, cnt.p,
                                              nullptr, nullptr, kmask.p + mwords);
  TG_CHECK_LAUNCH();
  TG_CUDA(cudaMemsetAsync(out.off.p, 0, 8, s));
  cub_run(s, [&](void* t, size_t& b) {
    return cub::DeviceScan::InclusiveSum(t, b, cnt.p, out.off.p + 1, (int64_t)g.n, s);
  });
  k_orient_tiles<1, CODED><<<grid, kOWarps * 32, 0, s>>>(g.off.p, g.adj.p, order_key(g), g.dcode.p, g.n, out.off.p,
                                                     out.desc.p, out.data.p, ctr.p + 1, nullptr,
                                                     nullptr, kmask.p, cnt.p);
  TG_CHECK_LAUNCH();
  k_orient_big<true, CODED><<<148 * 8, 256, 0, s>>>(g.off.p, g.adj.p, order_key(g), g.dcode.p, bigq.p, ctr.p + 2,
                                             out.off.p, out.desc.p, out.data.p, kmask.p + mwords);
  TG_CHECK_LAUNCH();
  g_launches += 6;  // count, big count, scan (init + sweep), fill, big fill
}

template <int CODED>
static void orient_onepass(const DevGraph& g, DevEff& out, cudaStream_t s) {
  const uint64_t ntiles = (g.n + 31) / 32;
  const unsigned grid = grid_for(ntiles, kOWarps, 148u * kOBlocks);  // resident
  DBuf<uint32_t> bigq(g.n, s);
  DBuf<unsigned long long> ctr(6, s);  // tile counter + k_orient_big1's counters
  ctr.zero();
  const uint8_t* codes = CODED == 2 ? g.dcode4.p : g.dcode.p;
  k_orient_tiles<2, CODED><<<grid, kOWarps * 32, 0, s>>>(g.off.p, g.adj.p, order_key(g), codes, g.n,
                                                         nullptr, out.desc.p, out.data.p, ctr.p,
                                                         bigq.p, ctr.p + 1, nullptr, nullptr, 0,
                                                         ~0ull, g.xmask);
  TG_CHECK_LAUNCH();
  k_orient_big1<CODED><<<148 * 6, 256, 0, s>>>(g.off.p, g.adj.p, order_key(g), codes, bigq.p, g.n,
                                               ctr.p, g.m2, out.desc.p, out.data.p, g.xmask);
  TG_CHECK_LAUNCH();
  g_launches += 2;
}

// One pass into the slab layout: n slabs of kSlab slots, then the region of
// the lists longer than a slab (big vertices and the g.slab_extra slots of
// the others, both sized by degree).
template <int CODED>
static void orient_slab(const DevGraph& g, DevEff& out, cudaStream_t s) {
  const uint64_t ntiles = (g.n + 31) / 32;
  const unsigned grid = grid_for(ntiles, kOWarps, 148u * kOBlocks);  // resident
  DBuf<uint32_t> bigq(g.n, s);
  DBuf<unsigned long long> ctr(6, s);
  ctr.zero();
  const uint8_t* codes = CODED == 2 ? g.dcode4.p : g.dcode.p;
  k_orient_tiles<2, CODED, true><<<grid, kOWarps * 32, 0, s>>>(g.off.p, g.adj.p, order_key(g), codes,
                                                               g.n, nullptr, out.desc.p, out.data.p,
                                                               ctr.p, bigq.p, ctr.p + 1, nullptr, nullptr,
                                                               0, ~0ull, g.xmask);
  TG_CHECK_LAUNCH();
  k_orient_big1<CODED, true><<<148 * 6, 256, 0, s>>>(g.off.p, g.adj.p, order_key(g), codes, bigq.p,
                                                     g.n, ctr.p, g.n * kSlab, out.desc.p, out.data.p,
                                                     g.xmask);
  TG_CHECK_LAUNCH();
  g_launches += 2;
}

// ---- chunked one-pass orientation (host CSR streamed in vertex chunks) ----
//
// The tile layout is position-independent (each tile writes inside its own
// adjacency range; hubs reserve slots above m2 with one atomic), so tiles can
// be oriented in any grouping: orient_chunk orients the tiles of vertices
// [vb, ve) (multiples of 32 except at n) as soon as their adjacency arrived.
// c[6] counters persist across chunks: [0] tile claims (reset per chunk),
// [1] medium-big queue size, [2] hub-region slots, [3] hubs, [4]/[5] hub /
// medium claim cursors (restarted at the previous chunk's queue ends).
__global__ void k_chunk_prep(unsigned long long* c) {
  c[0] = 0;
  c[4] = c[3];
  c[5] = c[1];
}

__device__ __forceinline__ uint32_t chunk_of(const uint32_t* __restrict__ cb, uint32_t K, uint32_t u) {
  uint32_t lo = 0, hi = K;  // first chunk whose end exceeds u
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (cb[mid + 1] <= u) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// ready chunk of each apex of chunk k: its lists and every N_u it intersects
// with are oriented once chunk max(k, chunk(max N_v)) is (lists ID-sorted);
// apexes with h_v < 2 close no triangle (0xff)
__global__ void k_ready_chunk(const uint64_t* __restrict__ edesc, const uint32_t* __restrict__ eff,
                              const uint32_t* __restrict__ cb, uint32_t K, uint32_t k, uint32_t vb,
                              uint32_t ve, uint8_t* __restrict__ ready) {
  for (uint64_t v = vb + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < ve;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t d = edesc[v];
    const uint32_t h = desc_len(d);
    uint8_t r = 0xff;
    if (h >= 2) r = (uint8_t)max(k, chunk_of(cb, K, eff[desc_start(d) + h - 1]));
    ready[v] = r;
  }
}

// apexes v < ve whose ready chunk is k (any order)
__global__ void k_select_ready(const uint8_t* __restrict__ ready, uint32_t vb, uint32_t ve, uint32_t k,
                               uint32_t* __restrict__ ids, unsigned long long* __restrict__ cnt) {
  const unsigned lane = threadIdx.x & 31;
  for (uint64_t base = vb + blockIdx.x * (uint64_t)blockDim.x + (threadIdx.x & ~31u); base < ve;
       base += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = base + lane;
    const bool take = v < ve && ready[v] == k;
    const unsigned bal = __ballot_sync(0xffffffffu, take);
    if (!bal) continue;
    unsigned long long at = 0;
    if (lane == 0) at = atomicAdd(cnt, (unsigned long long)__popc(bal));
    at = __shfl_sync(0xffffffffu, at, 0);
    if (take) ids[at + __popc(bal & ((1u << lane) - 1u))] = (uint32_t)v;
  }
}

void orient_chunk_begin(const DevGraph& g, DevEff& out, DBuf<uint32_t>& bigq,
                        DBuf<unsigned long long>& ctr, cudaStream_t s) {
  TG_REQUIRE(g.m2 + g.big_entries + kQuadPad < (1ull << 34), "graph too large for chunked orientation");
  out.rows = g.n;
  out.base = 0;
  out.compact = false;
  out.entries = g.m2 / 2;
  if (out.desc.n < (g.n ? g.n : 1)) out.desc.alloc(g.n ? g.n : 1, s);
  if (out.data.n < g.m2 + g.big_entries + kQuadPad) out.data.alloc(g.m2 + g.big_entries + kQuadPad, s);
  out.off.release();
  bigq.alloc(g.n ? g.n : 1, s);
  ctr.alloc(6, s);
  ctr.zero();
}

void orient_chunk(const DevGraph& g, DevEff& out, uint32_t vb, uint32_t ve, uint32_t* bigq,
                  unsigned long long* ctr, cudaStream_t s) {
  if (ve <= vb) return;
  const uint64_t t_lo = vb / 32, t_hi = ((uint64_t)ve + 31) / 32;
  const unsigned grid = grid_for(t_hi - t_lo, kOWarps, 148u * kOBlocks);
  k_chunk_prep<<<1, 1, 0, s>>>(ctr);
  TG_CHECK_LAUNCH();
  const bool coded = order_coded(g);
  if (coded)
    k_orient_tiles<2, true><<<grid, kOWarps * 32, 0, s>>>(
        g.off.p, g.adj.p, order_key(g), g.dcode.p, g.n, nullptr, out.desc.p, out.data.p, ctr,
        bigq, ctr + 1, nullptr, nullptr, t_lo, t_hi);
  else
    k_orient_tiles<2, false><<<grid, kOWarps * 32, 0, s>>>(
        g.off.p, g.adj.p, order_key(g), g.dcode.p, g.n, nullptr, out.desc.p, out.data.p, ctr,
        bigq, ctr + 1, nullptr, nullptr, t_lo, t_hi);
  TG_CHECK_LAUNCH();
  if (coded)
    k_orient_big1<true><<<148 * 6, 256, 0, s>>>(g.off.p, g.adj.p, order_key(g), g.dcode.p, bigq, g.n,
                                                ctr, g.m2, out.desc.p, out.data.p);
  else
    k_orient_big1<false><<<148 * 6, 256, 0, s>>>(g.off.p, g.adj.p, order_key(g), g.dcode.p, bigq,
                                                 g.n, ctr, g.m2, out.desc.p, out.data.p);
  TG_CHECK_LAUNCH();
  g_launches += 3;
}

// Rows [lo, hi) (lo a multiple of 32, hi too unless hi = n) with the
// one-pass tile kernel -- one rank's share of the orientation: the tiles of
// the range into a tile-layout scratch holding only the range's slots (the
// kernels address it through base pointers shifted by -off[lo] / -lo), big
// vertices above the range's slots, then one gather into the compact
// layout of orient_rows (off / desc / data, base lo).
void orient_rows_tiles(const DevGraph& g, uint32_t lo, uint32_t hi, DevEff& out, cudaStream_t s) {
  TG_REQUIRE(lo % 32 == 0 && (hi % 32 == 0 || hi == g.n) && lo <= hi && hi <= g.n,
             "orient_rows_tiles: rows must start on a 32-vertex tile");
  const uint64_t rows = hi - lo;
  uint64_t ob[2] = {0, 0};
  TG_CUDA(cudaMemcpyAsync(&ob[0], g.off.p + lo, 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaMemcpyAsync(&ob[1], g.off.p + hi, 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  const uint64_t span = ob[1] - ob[0];  // the range's symmetric slots
  // scratch: the range's slots + its big vertices' lists (<= span) + padding
  DevEff tile;
  tile.desc.alloc(rows ? rows : 1, s);
  tile.data.alloc(2 * span + kQuadPad, s);
  // big-vertex queue: medium ones from the front, hubs from index hi-1 down
  // (the kernels' convention with n = hi)
  DBuf<uint32_t> bigq(hi ? hi : 1, s);
  DBuf<unsigned long long> ctr(6, s);
  ctr.zero();
  uint64_t* desc_base = tile.desc.p - lo;
  uint32_t* data_base = tile.data.p - ob[0];
  if (rows) {
    const uint64_t t_lo = lo / 32, t_hi = ((uint64_t)hi + 31) / 32;
    const unsigned grid = grid_for(t_hi - t_lo, kOWarps, 148u * kOBlocks);
    const bool coded = order_coded(g);
    if (coded)
      k_orient_tiles<2, true><<<grid, kOWarps * 32, 0, s>>>(
          g.off.p, g.adj.p, order_key(g), g.dcode.p, hi, nullptr, desc_base, data_base, ctr.p,
          bigq.p, ctr.p + 1, nullptr, nullptr, t_lo, t_hi);
    else
      k_orient_tiles<2, false><<<grid, kOWarps * 32, 0, s>>>(
          g.off.p, g.adj.p, order_key(g), g.dcode.p, hi, nullptr, desc_base, data_base, ctr.p,
          bigq.p, ctr.p + 1, nullptr, nullptr, t_lo, t_hi);
    TG_CHECK_LAUNCH();
    // big vertices' lists above the range's slots (relative position span)
    if (coded)
      k_orient_big1<true><<<148 * 6, 256, 0, s>>>(g.off.p, g.adj.p, order_key(g), g.dcode.p,
                                                  bigq.p, hi, ctr.p, ob[1], desc_base, data_base);
    else
      k_orient_big1<false><<<148 * 6, 256, 0, s>>>(g.off.p, g.adj.p, order_key(g), g.dcode.p,
                                                   bigq.p, hi, ctr.p, ob[1], desc_base, data_base);
    TG_CHECK_LAUNCH();
    g_launches += 2;
  }
  // compact copy, base lo
  out.rows = rows;
  out.base = lo;
  out.compact = true;
  out.off.alloc(rows + 1, s);
  out.desc.alloc(rows ? rows : 1, s);
  TG_CUDA(cudaMemsetAsync(out.off.p, 0, 8, s));
  uint64_t entries = 0;
  if (rows) {
    DBuf<uint64_t> lens(rows, s);
    k_desc_lens<<<grid_for(rows, 256), 256, 0, s>>>(tile.desc.p, rows, lens.p);
    TG_CHECK_LAUNCH();
    cub_run(s, [&](void* t, size_t& b) {
      return cub::DeviceScan::InclusiveSum(t, b, lens.p, out.off.p + 1, (int64_t)rows, s);
    });
    TG_CUDA(cudaMemcpyAsync(&entries, out.off.p + rows, 8, cudaMemcpyDeviceToHost, s));
    TG_CUDA(cudaStreamSynchronize(s));
  }
  out.entries = entries;
  out.data.alloc(entries + kQuadPad, s);
  TG_CUDA(cudaMemsetAsync(out.data.p + entries, 0, kQuadPad * 4, s));
  if (rows) {
    CsrView v{tile.desc.p, data_base, 0};
    k_gather_compact<<<grid_for(rows * 32, 256, 148u * 32u), 256, 0, s>>>(v, rows, out.off.p,
                                                                        out.data.p);
    TG_CHECK_LAUNCH();
    k_desc_from_off<<<grid_for(rows, 256), 256, 0, s>>>(out.off.p, rows, out.desc.p);
    TG_CHECK_LAUNCH();
    g_launches += 4;
  }
}

void ready_chunks(const DevEff& e, const uint32_t* d_cb, uint32_t K, uint32_t k, uint32_t vb,
                  uint32_t ve, uint8_t* ready, cudaStream_t s) {
  if (ve <= vb) return;
  k_ready_chunk<<<grid_for(ve - vb, 256), 256, 0, s>>>(e.desc.p, e.data.p, d_cb, K, k, vb, ve, ready);
  TG_CHECK_LAUNCH();
  ++g_launches;
}

void select_ready(const uint8_t* ready, uint32_t vb, uint32_t ve, uint32_t k, uint32_t* ids,
                  unsigned long long* cnt, cudaStream_t s) {
  TG_CUDA(cudaMemsetAsync(cnt, 0, 8, s));
  if (ve <= vb) return;
  k_select_ready<<<grid_for(ve - vb, 256), 256, 0, s>>>(ready, vb, ve, k, ids, cnt);
  TG_CHECK_LAUNCH();
  ++g_launches;
}

// effective.hpp:37-52 for the whole graph (the hot path), no host sync.
//  * tile layout (default): ONE streaming pass; each tile's lists sit back
//    to back at the start of the tile's adjacency range, big vertices above
//    m2 -- list descriptors carry the positions;
//  * compact layout (when the tile layout would exceed 2^34 slots, where the
//    intersection's 32-bit quad indices end): count -> CUB scan -> fill,
//    lists back to back.
void orient_full(const DevGraph& g, DevEff& out, cudaStream_t s) {
  TG_REQUIRE(g.m2 < (1ull << 40), "graph too large for 40-bit list descriptors");
  const bool slab = g.slab && g.n && g.n * kSlab + g.big_entries + g.slab_extra + kQuadPad < (1ull << 34);
  const uint64_t slots = slab ? g.n * kSlab + g.big_entries + g.slab_extra : g.m2 + g.big_entries;
  out.slab = 0;
  if (!g.n || slots + kQuadPad >= (1ull << 34) || (!slab && (g_orient_mode & 3) == 1))
    return orient_full_compact(g, out, s);
  out.rows = g.n;
  out.base = 0;
  out.compact = false;
  out.entries = g.m2 / 2;
  if (out.desc.n < g.n) out.desc.alloc(g.n, s);
  if (out.data.n < slots + kQuadPad) out.data.alloc(slots + kQuadPad, s);
  out.off.release();
  if (slab) {
    out.slab = kSlab;
    if (order_nibble(g)) orient_slab<2>(g, out, s);
    else if (order_coded(g)) orient_slab<1>(g, out, s);
    else orient_slab<0>(g, out, s);
    return;
  }
  if (order_nibble(g)) orient_onepass<2>(g, out, s);
  else if (order_coded(g)) orient_onepass<1>(g, out, s);
  else orient_onepass<0>(g, out, s);
}

// count -> CUB scan -> fill, compact layout (sum h_v = m is known).
void orient_full_compact(const DevGraph& g, DevEff& out, cudaStream_t s) {
  TG_REQUIRE(g.m2 < (1ull << 40), "graph too large for 40-bit list descriptors");
  out.rows = g.n;
  out.base = 0;
  out.compact = true;
  out.entries = g.m2 / 2;
  const uint64_t m = g.m2 / 2;
  if (out.desc.n < (g.n ? g.n : 1)) out.desc.alloc(g.n ? g.n : 1, s);
  if (out.off.n < g.n + 1) out.off.alloc(g.n + 1, s);
  // (padding list starts to 32 B was measured: no gain on C2, so lists are
  // packed back to back)
  if (out.data.n < m + kQuadPad) out.data.alloc(m + kQuadPad, s);
  if (!g.n) {
    TG_CUDA(cudaMemsetAsync(out.off.p, 0, 8, s));
    return;
  }
  // 1-byte degree codes once the 4-byte degrees would not stay in L2
  if (order_coded(g)) orient_tiles<true>(g, out, s);
  else orient_tiles<false>(g, out, s);
}

// Gappy single-pass orientation (N_v in the first h_v slots of v's symmetric
// slot range); kept for comparison with the compact tile kernel.
void orient_full_gappy(const DevGraph& g, DevEff& out, cudaStream_t s) {
  TG_REQUIRE(g.m2 < (1ull << 40), "graph too large for 40-bit list descriptors");
  out.rows = g.n;
  out.base = 0;
  out.compact = false;
  out.entries = g.m2 / 2;
  if (out.desc.n < (g.n ? g.n : 1)) out.desc.alloc(g.n ? g.n : 1, s);
  if (out.data.n < g.m2 + kQuadPad) out.data.alloc(g.m2 + kQuadPad, s);
  out.off.release();
  if (!g.n) return;
  const uint64_t avg = g.m2 / g.n;
  if (avg <= 12) launch_orient_gappy<8>(g, out.desc.p, out.data.p, s);
  else if (avg <= 24) launch_orient_gappy<16>(g, out.desc.p, out.data.p, s);
  else launch_orient_gappy<32>(g, out.desc.p, out.data.p, s);
}

void eff_desc_from_off(DevEff& e, cudaStream_t s) {
  e.desc.alloc(e.rows ? e.rows : 1, s);
  if (!e.rows) return;
  k_desc_from_off<<<grid_for(e.rows, 256), 256, 0, s>>>(e.off.p, e.rows, e.desc.p);
  TG_CHECK_LAUNCH();
  ++g_launches;
}

void compact_eff(const DevEff& in, DevEff& out, cudaStream_t s) {
  const uint64_t rows = in.rows;
  out.rows = rows;
  out.base = in.base;
  out.compact = true;
  out.entries = in.entries;
  out.off.alloc(rows + 1, s);
  out.desc.alloc(rows ? rows : 1, s);
  out.data.alloc(in.entries + kQuadPad, s);
  TG_CUDA(cudaMemsetAsync(out.off.p, 0, 8, s));
  if (!rows) return;
  DBuf<uint64_t> lens(rows, s);
  k_desc_lens<<<grid_for(rows, 256), 256, 0, s>>>(in.desc.p, rows, lens.p);
  TG_CHECK_LAUNCH();
  cub_run(s, [&](void* t, size_t& b) {
    return cub::DeviceScan::InclusiveSum(t, b, lens.p, out.off.p + 1, (int64_t)rows, s);
  });
  CsrView v{in.desc.p, in.data.p, in.base};
  k_gather_compact<<<grid_for(rows * 32, 256, 148u * 32u), 256, 0, s>>>(v, rows, out.off.p, out.data.p);
  TG_CHECK_LAUNCH();
  k_desc_from_off<<<grid_for(rows, 256), 256, 0, s>>>(out.off.p, rows, out.desc.p);
  TG_CHECK_LAUNCH();
  g_launches += 5;
}

__global__ void k_heavy_lens(const uint64_t* __restrict__ desc, uint64_t rows, uint32_t thr,
                             unsigned long long* __restrict__ acc) {
  uint64_t s = 0;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t h = desc_len(desc[r]);
    if (h > thr) s += h;
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(acc, (unsigned long long)s);
}

uint64_t heavy_entries(const DevEff& e, uint32_t thr, cudaStream_t s) {
  DBuf<unsigned long long> acc(1, s);
  acc.zero();
  if (e.rows) {
    k_heavy_lens<<<grid_for(e.rows, 256, 148u * 8u), 256, 0, s>>>(e.desc.p, e.rows, thr, acc.p);
    TG_CHECK_LAUNCH();
    ++g_launches;
  }
  unsigned long long h = 0;
  TG_CUDA(cudaMemcpyAsync(&h, acc.p, 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  return h;
}

// acc[0] = entries of the lists longer than a slab, acc[1] = degrees of their
// vertices that the orientation does not treat as big, acc[2] = max h
__global__ void k_slab_stats(const uint64_t* __restrict__ desc, const uint32_t* __restrict__ deg,
                             uint64_t rows, unsigned long long* __restrict__ acc) {
  unsigned long long a = 0, b = 0, mx = 0;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t h = desc_len(desc[r]);
    if (h > kSlab) {
      a += h;
      if (deg[r] <= kOBig) b += deg[r];
    }
    mx = h > mx ? h : mx;
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = t > mx ? t : mx;
  }
  if ((threadIdx.x & 31) == 0) {
    if (a) atomicAdd(acc, a);
    if (b) atomicAdd(acc + 1, b);
    atomicMax(acc + 2, mx);
  }
}

SlabStats slab_stats(const DevGraph& g, const DevEff& e, cudaStream_t s) {
  DBuf<unsigned long long> acc(3, s);
  acc.zero();
  if (e.rows) {
    k_slab_stats<<<grid_for(e.rows, 256, 148u * 8u), 256, 0, s>>>(e.desc.p, g.deg.p, e.rows, acc.p);
    TG_CHECK_LAUNCH();
    ++g_launches;
  }
  unsigned long long h[3] = {0, 0, 0};
  TG_CUDA(cudaMemcpyAsync(h, acc.p, 24, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  return SlabStats{h[0], h[1], (uint32_t)h[2]};
}

// slabs of rows [vb, ve) from their lists (a warp per row: one coalesced
// 128-byte store, pads past h_v)
__global__ void __launch_bounds__(256)
k_slab_rows(const uint64_t* __restrict__ desc, uint32_t* __restrict__ data, uint64_t vb, uint64_t ve) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t v = vb + ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5); v < ve; v += warps) {
    const uint64_t d = desc[v];
    const uint32_t h = desc_len(d);
    const uint32_t x = lane < h ? __ldcs(data + desc_start(d) + lane) : kNoEntry;
    data[v * kSlab + lane] = x;
  }
}

void slab_rows(DevEff& e, uint32_t vb, uint32_t ve, cudaStream_t s) {
  if (ve <= vb) return;
  k_slab_rows<<<grid_for((uint64_t)(ve - vb) * 32, 256, 148u * 16u), 256, 0, s>>>(e.desc.p, e.data.p, vb, ve);
  TG_CHECK_LAUNCH();
  ++g_launches;
}

uint64_t sum_lens(const DevEff& e, uint32_t lo, uint32_t hi, cudaStream_t s) {
  DBuf<unsigned long long> acc(1, s);
  acc.zero();
  if (hi > lo) {
    k_sum_lens<<<grid_for(hi - lo, 256, 148u * 8u), 256, 0, s>>>(e.desc.p, lo - e.base, hi - e.base, acc.p);
    TG_CHECK_LAUNCH();
    ++g_launches;
  }
  unsigned long long h = 0;
  TG_CUDA(cudaMemcpyAsync(&h, acc.p, 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  return h;
}

// order.hpp:95-104: rank = position in the (degree, id) sort.
void degree_rank(const DevGraph& g, uint32_t* d_rank, cudaStream_t s) {
  if (!g.n) return;
  DBuf<uint64_t> k1(g.n, s), k2(g.n, s);
  k_rank_keys<<<grid_for(g.n, 256), 256, 0, s>>>(g.deg.p, g.n, k1.p);
  TG_CHECK_LAUNCH();
  ++g_launches;
  cub_run(s, [&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortKeys(t, b, k1.p, k2.p, (int64_t)g.n, 0, 64, s);
  });
  ++g_launches;
  k_rank_scatter<<<grid_for(g.n, 256), 256, 0, s>>>(k2.p, g.n, d_rank);
  TG_CHECK_LAUNCH();
  ++g_launches;
}

void node_costs_device(const DevGraph& g, const DevEff& eff, int kind, uint64_t* d_f,
                       uint64_t* d_prefix, cudaStream_t s) {
  TG_REQUIRE(kind >= TG_COST_N && kind <= TG_COST_NOV, "node_costs: unknown cost kind");
  if (!g.n) return;
  TG_REQUIRE(eff.base == 0 && eff.rows == g.n, "node_costs needs the full oriented CSR");
  const CsrView ev{eff.desc.p, eff.data.p, 0};
  if (kind == TG_COST_DPD || kind == TG_COST_NOV) {
    unsigned grid = grid_for(g.n * 32, 256, 148u * 32u);
    if (kind == TG_COST_DPD)
      k_cost_sum<false><<<grid, 256, 0, s>>>(g.off.p, g.adj.p, order_key(g), ev, g.n, d_f);
    else
      k_cost_sum<true><<<grid, 256, 0, s>>>(g.off.p, g.adj.p, order_key(g), ev, g.n, d_f);
  } else {
    k_cost_simple<<<grid_for(g.n, 256), 256, 0, s>>>(eff.desc.p, g.deg.p, g.n, kind, d_f);
  }
  TG_CHECK_LAUNCH();
  ++g_launches;
  cub_run(s, [&](void* t, size_t& b) {
    return cub::DeviceScan::InclusiveSum(t, b, d_f, d_prefix, (int64_t)g.n, s);
  });
  ++g_launches;
}

std::vector<uint32_t> boundaries_from_prefix(const uint64_t* d_prefix, uint64_t n, uint64_t p,
                                             cudaStream_t s) {
  TG_REQUIRE(p >= 1, "compute_boundaries: p must be >= 1");
  DBuf<uint32_t> b(p + 1, s);
  k_boundaries<<<grid_for(p, 128), 128, 0, s>>>(d_prefix, n, p, b.p);
  TG_CHECK_LAUNCH();
  ++g_launches;
  std::vector<uint32_t> h(p + 1);
  TG_CUDA(cudaMemcpyAsync(h.data(), b.p, (p + 1) * 4, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  return h;
}

uint64_t ordering_cost_device(const DevGraph& g, const DevEff& eff, cudaStream_t s) {
  DBuf<unsigned long long> acc(1, s);
  acc.zero();
  if (g.n) {
    k_ordering_cost<<<grid_for(g.n, 256, 148u * 8u), 256, 0, s>>>(g.deg.p, eff.desc.p, g.n, acc.p);
    TG_CHECK_LAUNCH();
    ++g_launches;
  }
  unsigned long long h = 0;
  TG_CUDA(cudaMemcpyAsync(&h, acc.p, 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  return h;
}

}  // namespace tgb
