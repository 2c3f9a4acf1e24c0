// window.cu -- NodeIteratorN for graphs whose oriented lists are local in
// id space (Watts-Strogatz, ring / lattice / banded graphs: config 4).
//
// Reference semantics: count_node_iterator_n (sequential.hpp:74-91) --
// |N_v ∩ N_u| over every oriented edge v -> u -- and the AOP rank body over an
// apex range (engines.hpp:38-54).  Same count, a different set encoding.
//
// Each oriented list is split by distance from its row:
//   W_v = [v-32, v+31]          the window of v;
//   L_v = N_v ∩ W_v             as ONE 64-bit mask (bit i <-> id v-32+i);
//   F_v = N_v \ W_v             the few "far" entries, a short sorted list.
// Then for an oriented edge v -> u:
//   |N_v ∩ N_u| = popc(align(mask_v, u - v) & mask_u)      L_v ∩ L_u
//               + #{x ∈ F_v : x ∈ W_u, bit of mask_u}       F_v ∩ L_u
//               + #{x ∈ F_u : x ∈ W_v ? bit of mask_v       L_v ∩ F_u
//                                     : x ∈ F_v}           F_v ∩ F_u
// (each common x is counted by exactly one term).
//
// Layout: one 32-byte record per row (one DRAM sector): the mask, |F_v| and
// up to kInline far entries inline; longer far lists live in far[] and the
// record holds their position.  An oriented edge then costs one record load
// of its middle vertex -- from a neighbouring row (L1/L2-resident) for the
// ~90% window edges of Watts-Strogatz, one sector for a rewired one -- one
// POPC and ~1-2 far tests, instead of a pass over the h_u entries of N_u.
// The middle vertices of an apex come from its own mask bits and far
// entries, so N_v itself is never re-read.
//
// The edges of 32 consecutive apexes are flattened over a warp's lanes (one
// edge per lane per round, apex from a per-round bit table of apex starts).
// Apexes with more than kFarMax far entries go to a queue that the generic
// kernels (intersect.cu, ListApex) count; the graph uses this path only when
// the far entries are a small fraction of m (engine.cu window_ready).
#include "tg_internal.cuh"

namespace tgb {
namespace {

constexpr uint32_t kFarMax = 16;  // an apex's far entries handled here
constexpr uint32_t kInline = 5;   // far entries stored in the record
constexpr int kWinWarps = 8;      // 256-thread blocks

// record = {mask.lo, mask.hi, nf, f0 | pos.lo} {f1 | pos.hi, f2, f3, f4}
struct Rec {
  uint64_t mask;
  uint32_t nf;
  uint32_t f[5];  // inline far entries, or f[0..1] = position in far[]
};

__device__ __forceinline__ Rec rec_from(uint4 a, uint4 b) {
  Rec r;
  r.mask = ((uint64_t)a.y << 32) | a.x;
  r.nf = a.z;
  r.f[0] = a.w;
  r.f[1] = b.x;
  r.f[2] = b.y;
  r.f[3] = b.z;
  r.f[4] = b.w;
  return r;
}

__device__ __forceinline__ Rec load_rec(const uint4* __restrict__ R, uint64_t v) {
  return rec_from(__ldg(R + 2 * v), __ldg(R + 2 * v + 1));
}

// k-th far entry of a record
__device__ __forceinline__ uint32_t far_at(const Rec& r, uint32_t k, const uint32_t* __restrict__ far) {
  if (r.nf <= kInline) {
    uint32_t x = r.f[0];
#pragma unroll
    for (uint32_t i = 1; i < kInline; ++i)
      if (k == i) x = r.f[i];
    return x;
  }
  const uint64_t pos = ((uint64_t)r.f[1] << 32) | r.f[0];
  return __ldg(far + pos + k);
}

// entries of the oriented lists outside their row's window (host result)
__global__ void k_window_far_count(CsrView e, uint64_t rows, unsigned long long* __restrict__ far) {
  unsigned long long c = 0;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < rows;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t d = e.desc[v];
    const uint32_t* L = e.data + desc_start(d);
    const uint32_t h = desc_len(d);
    const int64_t lo = (int64_t)v - 32;
    for (uint32_t i = 0; i < h; ++i) {
      const int64_t o = (int64_t)__ldg(L + i) - lo;
      c += (o < 0 || o >= 64);
    }
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(far, c);
}

// The records (and far[] for lists longer than kInline).  A thread per row
// reads its list as the 16-byte quads that cover it (4 entries per load);
// the overflow slots of a warp's 32 rows are claimed with one atomic.
__global__ void __launch_bounds__(256)
k_window_build(CsrView e, uint64_t rows, uint4* __restrict__ R, uint32_t* __restrict__ far,
               unsigned long long* __restrict__ cursor) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  const uint4* __restrict__ Q = reinterpret_cast<const uint4*>(e.data);
  for (uint64_t v0 = blockIdx.x * (uint64_t)blockDim.x; v0 < rows;
       v0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = v0 + threadIdx.x;
    const bool valid = v < rows;
    const uint64_t d = valid ? e.desc[v] : 0ull;
    const uint64_t st = desc_start(d), en = st + desc_len(d);
    const int64_t lo = (int64_t)v - 32;
    uint64_t mk = 0;
    uint32_t nf = 0, f[kInline] = {0, 0, 0, 0, 0};
    for (uint64_t q = st >> 2; q < ((en + 3) >> 2); ++q) {  // bits, far count, inline far
      const uint4 r = __ldg(Q + q);
      const uint32_t xs[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t slot = 4 * q + k;
        if (slot >= st && slot < en) {
          const int64_t o = (int64_t)xs[k] - lo;
          if (o >= 0 && o < 64) {
            mk |= 1ull << o;
          } else {
#pragma unroll
            for (uint32_t i = 0; i < kInline; ++i)
              if (nf == i) f[i] = xs[k];
            ++nf;
          }
        }
      }
    }
    const uint32_t over = nf > kInline ? nf : 0u;  // rows whose far list overflows
    uint32_t incl = over;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(FULL, incl, o);
      if ((int)lane >= o) incl += t;
    }
    const uint32_t tot = __shfl_sync(FULL, incl, 31);
    unsigned long long base = 0;
    if (lane == 31 && tot) base = atomicAdd(cursor, (unsigned long long)tot);
    base = __shfl_sync(FULL, base, 31);
    const uint64_t pos = base + (incl - over);
    if (over) {  // the full far list to far[] (the quads are L1-resident)
      f[0] = (uint32_t)pos;
      f[1] = (uint32_t)(pos >> 32);
      uint32_t wpos = 0;
      for (uint64_t q = st >> 2; q < ((en + 3) >> 2); ++q) {
        const uint4 r = __ldg(Q + q);
        const uint32_t xs[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t slot = 4 * q + k;
          const int64_t o = (int64_t)xs[k] - lo;
          if (slot >= st && slot < en && (o < 0 || o >= 64)) far[pos + wpos++] = xs[k];
        }
      }
    }
    if (valid) {
      R[2 * v] = make_uint4((uint32_t)mk, (uint32_t)(mk >> 32), nf, f[0]);
      R[2 * v + 1] = make_uint4(f[1], f[2], f[3], f[4]);
    }
  }
}

// index (0..63) of the k-th (0-based) set bit of x (k < popc(x))
__device__ __forceinline__ uint32_t select64(uint64_t x, uint32_t k) {
  uint32_t pos = 0;
  uint32_t w = (uint32_t)x;
  uint32_t c = __popc(w);
  if (k >= c) { k -= c; w = (uint32_t)(x >> 32); pos = 32; }
  c = __popc(w & 0xFFFFu);
  if (k >= c) { k -= c; w >>= 16; pos += 16; }
  c = __popc(w & 0xFFu);
  if (k >= c) { k -= c; w >>= 8; pos += 8; }
  c = __popc(w & 0xFu);
  if (k >= c) { k -= c; w >>= 4; pos += 4; }
  c = __popc(w & 0x3u);
  if (k >= c) { k -= c; w >>= 2; pos += 2; }
  if (k >= (w & 1u)) pos += 1;
  return pos;
}

// x ∈ F (ascending far entries of record r)
__device__ __forceinline__ bool far_contains(const Rec& r, uint32_t x, const uint32_t* __restrict__ far) {
  uint32_t lo = 0, hi = r.nf;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (far_at(r, mid, far) < x) lo = mid + 1;
    else hi = mid;
  }
  return lo < r.nf && far_at(r, lo, far) == x;
}

// mask of v's window shifted into u's window (d = u - v)
__device__ __forceinline__ uint64_t align_mask(uint64_t mv, int64_t d) {
  if (d >= 0) return d < 64 ? (mv >> d) : 0ull;
  return d > -64 ? (mv << (-d)) : 0ull;
}

// |N_v ∩ N_u| from the records of v and u (any far-list lengths; long ones
// are rare where the encoding is chosen)
__device__ __forceinline__ uint32_t edge_count(uint32_t v, const Rec& rv, uint32_t u,
                                               const uint4* __restrict__ R,
                                               const uint32_t* __restrict__ far) {
  const Rec ru = load_rec(R, u);
  const int64_t d = (int64_t)u - (int64_t)v;
  uint32_t c = __popcll(align_mask(rv.mask, d) & ru.mask);  // L_v ∩ L_u
  if (rv.nf <= kInline && ru.nf <= kInline) {
    // both far lists inline: fully unrolled and predicated (no divergent
    // loops, no dynamic register indexing)
    const int64_t ub = (int64_t)u - 32, vb = (int64_t)v - 32;
#pragma unroll
    for (uint32_t k = 0; k < kInline; ++k) {
      if (k < rv.nf) {  // F_v ∩ L_u
        const int64_t j = (int64_t)rv.f[k] - ub;
        c += (j >= 0 && j < 64) ? (uint32_t)((ru.mask >> j) & 1ull) : 0u;
      }
      if (k < ru.nf) {  // F_u ∩ (L_v ∪ F_v)
        const uint32_t x = ru.f[k];
        const int64_t i = (int64_t)x - vb;
        bool hit;
        if (i >= 0 && i < 64) {
          hit = (rv.mask >> i) & 1ull;
        } else {
          hit = false;
#pragma unroll
          for (uint32_t t = 0; t < kInline; ++t) hit |= (t < rv.nf) && rv.f[t] == x;
        }
        c += hit ? 1u : 0u;
      }
    }
    return c;
  }
  for (uint32_t k = 0; k < rv.nf; ++k) {                    // F_v ∩ L_u
    const int64_t j = (int64_t)far_at(rv, k, far) - ((int64_t)u - 32);
    if (j >= 0 && j < 64) c += (uint32_t)((ru.mask >> j) & 1ull);
  }
  for (uint32_t k = 0; k < ru.nf; ++k) {  // F_u ∩ (L_v ∪ F_v)
    const uint32_t x = far_at(ru, k, far);
    const int64_t i = (int64_t)x - ((int64_t)v - 32);
    if (i >= 0 && i < 64) c += (uint32_t)((rv.mask >> i) & 1ull);
    else c += far_contains(rv, x, far) ? 1u : 0u;
  }
  return c;
}

// NodeIteratorN over apexes [vlo, vhi): one warp per 32 consecutive apexes,
// their oriented edges (window bits, then far entries) flattened over the
// lanes so each lane does one edge per round.  A lane finds its apex from a
// per-round bit table of apex starts (one OR-reduction + one POPC) -- the
// segment-start scheme of the quad kernels.  Apexes with more than kFarMax
// far entries are appended to `defer` for the generic kernels.
__global__ void __launch_bounds__(kWinWarps * 32, 4)
k_window_count(const uint4* __restrict__ R, const uint32_t* __restrict__ far, uint32_t vlo,
               uint32_t vhi, unsigned long long* __restrict__ total,
               uint32_t* __restrict__ defer, unsigned long long* __restrict__ ndefer) {
  __shared__ uint4 sR[kWinWarps][32][2];
  __shared__ uint32_t sV[kWinWarps][32], sEx[kWinWarps][32];
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu, le = (2u << lane) - 1u;
  unsigned long long acc = 0;
  const uint64_t groups = ((uint64_t)(vhi - vlo) + 31) / 32;
  for (uint64_t gi = blockIdx.x * (uint64_t)kWinWarps + w; gi < groups;
       gi += (uint64_t)gridDim.x * kWinWarps) {
    const uint64_t v = vlo + gi * 32 + lane;
    const bool valid = v < vhi;
    uint4 a = make_uint4(0, 0, 0, 0), b = a;
    if (valid) {
      a = __ldg(R + 2 * v);
      b = __ldg(R + 2 * v + 1);
    }
    const uint64_t mv = ((uint64_t)a.y << 32) | a.x;
    const uint32_t nfv = a.z;
    const bool bad = valid && nfv > kFarMax;
    if (bad) defer[atomicAdd(ndefer, 1ull)] = (uint32_t)v;
    const uint32_t deg = (valid && !bad) ? (uint32_t)__popcll(mv) + nfv : 0u;
    // compact the apexes with edges; exclusive prefix of their degrees
    const unsigned has = __ballot_sync(FULL, deg > 0);
    uint32_t incl = deg;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(FULL, incl, o);
      if ((int)lane >= o) incl += t;
    }
    const uint32_t E = __shfl_sync(FULL, incl, 31);
    if (deg) {
      const uint32_t c = __popc(has & ((1u << lane) - 1u));
      sR[w][c][0] = a;
      sR[w][c][1] = b;
      sV[w][c] = (uint32_t)v;
      sEx[w][c] = incl - deg;
    }
    __syncwarp();
    const uint32_t my_ex = lane < (uint32_t)__popc(has) ? sEx[w][lane] : 0xffffffffu;
    uint32_t before = 0;  // apexes started before the current round
    for (uint32_t e0 = 0; e0 < E; e0 += 32) {
      // bit j of `starts`: an apex's first edge is item e0 + j
      const uint32_t rel = my_ex - e0;
      const unsigned starts = __reduce_or_sync(FULL, rel < 32u ? (1u << rel) : 0u);
      const uint32_t ei = e0 + lane;
      if (ei < E) {
        const uint32_t ai = before + __popc(starts & le) - 1u;
        const uint32_t k = ei - sEx[w][ai];
        const uint32_t va = sV[w][ai];
        const Rec rv = rec_from(sR[w][ai][0], sR[w][ai][1]);
        const uint32_t nb = (uint32_t)__popcll(rv.mask);
        const uint32_t u = k < nb ? (uint32_t)((int64_t)va - 32 + select64(rv.mask, k))
                                  : far_at(rv, k - nb, far);
        acc += edge_count(va, rv, u, R, far);
      }
      before += __popc(starts);
    }
    __syncwarp();
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(total, acc);
}

}  // namespace

int g_window_mode = 0;

uint64_t window_far_entries(const DevEff& e, cudaStream_t s) {
  if (!e.rows) return 0;
  DBuf<unsigned long long> c(1, s);
  c.zero();
  k_window_far_count<<<grid_for(e.rows, 256, 148u * 16u), 256, 0, s>>>(
      CsrView{e.desc.p, e.data.p, e.base}, e.rows, c.p);
  TG_CHECK_LAUNCH();
  ++g_launches;
  unsigned long long h = 0;
  TG_CUDA(cudaMemcpyAsync(&h, c.p, 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  return h;
}

void window_build(const DevEff& e, uint64_t far_cap, WindowEff& w, cudaStream_t s) {
  const uint64_t rows = e.rows;
  if (w.rec.n < 2 * rows) w.rec.alloc(2 * (rows ? rows : 1), s);
  if (w.far.n < far_cap + 1) w.far.alloc(far_cap + 1, s);
  if (w.ctr.n < 2) w.ctr.alloc(2, s);
  w.ctr.zero();
  w.rows = rows;
  if (!rows) return;
  k_window_build<<<grid_for(rows, 256, 148u * 8u), 256, 0, s>>>(
      CsrView{e.desc.p, e.data.p, e.base}, rows, w.rec.p, w.far.p, w.ctr.p);
  TG_CHECK_LAUNCH();
  ++g_launches;
}

void window_count(WindowEff& w, uint32_t vlo, uint32_t vhi, unsigned long long* d_total,
                  DBuf<uint32_t>& defer, cudaStream_t s) {
  if (vhi <= vlo) return;
  if (defer.n < (uint64_t)(vhi - vlo)) defer.alloc(vhi - vlo, s);
  TG_CUDA(cudaMemsetAsync(w.ctr.p + 1, 0, 8, s));
  k_window_count<<<grid_for(((uint64_t)(vhi - vlo) + 31) / 32, kWinWarps, 148u * 5u),
                   kWinWarps * 32, 0, s>>>(w.rec.p, w.far.p, vlo, vhi, d_total, defer.p,
                                           w.ctr.p + 1);
  TG_CHECK_LAUNCH();
  ++g_launches;
}

}  // namespace tgb
