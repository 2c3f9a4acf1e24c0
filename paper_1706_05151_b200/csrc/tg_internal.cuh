// tg_internal.cuh -- shared device/host plumbing for the B200 triangle library.
//
// Layout in HBM (one device, one graph):
//   sym_off  uint64[n+1], sym_adj uint32[2m]   -- reference Graph (graph.hpp:16-53)
//   deg      uint32[n]                          -- degree, the ByDegree key (order.hpp:95-104)
//   eff_off  uint64[n+1], eff uint32[m]         -- EffectiveAdjacency (effective.hpp:17-35),
//                                                  lists ID-sorted, oriented v -> u iff
//                                                  (deg v, v) < (deg u, u)
// All sizes are 64-bit; node ids are uint32 (NodeId, graph.hpp:14).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/trigraph_b200.h"

namespace tgb {

// Error carried from the C++ implementation to the C-ABI status codes.
struct Error : std::runtime_error {
  tg_status status;
  Error(tg_status s, const std::string& what) : std::runtime_error(what), status(s) {}
};

#define TG_CUDA(expr)                                                                  \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess)                                                             \
      throw ::tgb::Error(_e == cudaErrorMemoryAllocation ? TG_ERR_OOM : TG_ERR_CUDA,   \
                         std::string(#expr) + ": " + cudaGetErrorString(_e) + " at " + \
                             __FILE__ + ":" + std::to_string(__LINE__));               \
  } while (0)

#define TG_CHECK_LAUNCH() TG_CUDA(cudaGetLastError())

#define TG_REQUIRE(cond, msg)                                   \
  do {                                                          \
    if (!(cond)) throw ::tgb::Error(TG_ERR_INVALID_ARGUMENT, msg); \
  } while (0)

// Device buffer owned by the library; freed stream-ordered.
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = 0;
  DBuf() = default;
  DBuf(size_t count, cudaStream_t stream) { alloc(count, stream); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; s = o.s;
      o.p = nullptr; o.n = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t count, cudaStream_t stream) {
    release();
    s = stream;
    n = count;
    if (count) TG_CUDA(cudaMallocAsync((void**)&p, count * sizeof(T), stream));
  }
  void release() noexcept {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  void zero() {
    if (n) TG_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
};

// Symmetric CSR resident on a device (reference Graph).
struct DevGraph {
  uint64_t n = 0, m2 = 0;  // m2 = 2m adjacency entries
  DBuf<uint64_t> off;      // n+1
  DBuf<uint32_t> adj;      // m2
  DBuf<uint32_t> deg;      // n
  DBuf<uint8_t> dcode;     // n: monotone 1-byte degree code (orientation)
  // 4-bit degree codes, two per byte (build_nibble_codes): nibble 0 not
  // built yet, 1 built, -1 not applicable; xmask = buckets of one degree
  DBuf<uint8_t> dcode4;
  int nibble = 0;
  uint32_t xmask = 0;
  uint64_t big_entries = 0;  // sum of degrees of the orientation's hub vertices
  // Total order of the orientation (order.hpp:17-35).  ByDegree keys on
  // `deg` (or `dcode`); every other kind keys on okey = its rank array, so
  // precedes(v, u) = okey[v] < okey[u] through the same kernels.
  int order = TG_ORDER_BY_DEGREE;
  uint64_t order_seed = 0;
  DBuf<uint32_t> okey;     // n (non-degree orders only)
  // Slab layout of the oriented lists (orient_full): on when slab != 0;
  // slab_extra = sum of the degrees of the vertices with h_v > kSlab that the
  // orientation does not treat as big (the slots their full lists reserve).
  uint32_t slab = 0;
  uint64_t slab_extra = 0;
};

// Slab layout: list v in the 32 slots (one 128-byte DRAM line) at 32 v,
// padded with kNoEntry (never a NodeId: n < 2^32 - 1 is required).
constexpr uint32_t kSlab = 32;
constexpr uint32_t kNoEntry = 0xffffffffu;

extern int g_orient_mode;  // (see below)

// Order key array and key kind used by the orientation kernels.
inline const uint32_t* order_key(const DevGraph& g) {
  return g.order == TG_ORDER_BY_DEGREE ? g.deg.p : g.okey.p;
}
// 1-byte degree codes once the 4-byte degrees would not stay in L2.
#ifndef TG_CODED_MIN_N
#define TG_CODED_MIN_N (32ull << 20)
#endif
inline bool order_coded(const DevGraph& g) {
  return g.order == TG_ORDER_BY_DEGREE &&
         (g.n > (uint64_t)(TG_CODED_MIN_N) || (g_orient_mode & 4));
}

// 4-bit codes once even the 1-byte codes would not stay in L2 (the full
// orientation only; built by build_nibble_codes on first use).
#ifndef TG_NIBBLE_MIN_N
#define TG_NIBBLE_MIN_N (64ull << 20)
#endif
inline bool order_nibble_wanted(const DevGraph& g) {
  return g.order == TG_ORDER_BY_DEGREE && (g.n > (uint64_t)(TG_NIBBLE_MIN_N) || (g_orient_mode & 8));
}
inline bool order_nibble(const DevGraph& g) { return order_nibble_wanted(g) && g.nibble == 1; }
void build_nibble_codes(DevGraph& g, cudaStream_t s);

// Monotone 1-byte code of a degree: exact below 240, then one bucket per
// doubling.  code(a) < code(b) implies a < b; equal codes below 240 imply
// equal degrees; equal codes >= 240 need the exact degrees.  A 1-byte
// lookup table of n vertices stays L2-resident 4x longer than the degrees.
__host__ __device__ __forceinline__ uint8_t degree_code(uint32_t d) {
  if (d < 240) return (uint8_t)d;
  uint32_t c = 240, x = d / 240;  // x >= 1
  while (x > 1 && c < 255) {
    x >>= 1;
    c += 4;
  }
  return (uint8_t)(c > 255 ? 255 : c);
}

// Packed list descriptor: (start << 24) | len.  One 8-byte load gives a
// list's position and length (len < 2^24, start < 2^40).
__host__ __device__ __forceinline__ uint64_t desc_start(uint64_t d) { return d >> 24; }
__host__ __device__ __forceinline__ uint32_t desc_len(uint64_t d) { return (uint32_t)(d & 0xFFFFFFu); }
__host__ __device__ __forceinline__ uint64_t make_desc(uint64_t start, uint64_t len) {
  return (start << 24) | len;
}

// Oriented lists (reference EffectiveAdjacency), possibly partition-local:
// list(v) = data[start .. start+len) with (start, len) = desc[v-base], for v
// in [base, base+rows).  Two layouts:
//  * compact  -- lists back to back (off[] valid, rows+1 entries): partitions
//    and the exported EffectiveAdjacency;
//  * gappy    -- N_v in the first h_v slots of v's symmetric-CSR slot range
//    (start = sym_off[v]); built in ONE pass over the adjacency (the hot path).
//  * slab     -- (slab = kSlab) the first min(h_v, 32) entries of N_v in the
//    128-byte-aligned slab data[32 v, 32 v + 32), kNoEntry-padded, so a random
//    list read is ONE DRAM line and needs no descriptor; lists longer than a
//    slab are stored whole above the slabs (desc points there).
struct DevEff {
  uint64_t rows = 0, entries = 0;
  uint32_t base = 0;
  bool compact = false;
  uint32_t slab = 0;
  DBuf<uint64_t> desc;  // rows
  DBuf<uint64_t> off;   // rows+1 (compact layout only)
  DBuf<uint32_t> data;
};

// List arrays carry kQuadPad extra slots so that the intersection may read
// the whole 16-byte quad holding a list's last element.
constexpr uint64_t kQuadPad = 4;

// Read-only view passed to kernels.
struct CsrView {
  const uint64_t* desc;
  const uint32_t* data;
  uint32_t base;
  float avg_len = 0.f;  // host-side hint: mean list length (kernel choice)
  bool quad_ok = false;  // host-side: list slots < 2^34 (32-bit quad indices)
  uint32_t slab = 0;     // slab layout (DevEff::slab, base = 0): list v also at data + 32 v
};

// ---- build / orient (build.cu, orient.cu) ----
void build_graph_device(const uint32_t* d_pairs, uint64_t E, uint64_t n_override,
                        DevGraph& g, cudaStream_t s);
void compute_degrees(DevGraph& g, cudaStream_t s);
// Orient rows [vlo, vhi) of g into `out` (out.base = vlo), compact layout;
// lists ID-sorted.
void orient_rows(const DevGraph& g, uint32_t vlo, uint32_t vhi, DevEff& out, cudaStream_t s);
// The same output from the one-pass tile kernel (vlo a multiple of 32, vhi
// too unless vhi = n): one rank's share of the full orientation.
void orient_rows_tiles(const DevGraph& g, uint32_t vlo, uint32_t vhi, DevEff& out, cudaStream_t s);
// Orient the whole graph (no host sync): one-pass tile layout, or compact.
void orient_full(const DevGraph& g, DevEff& out, cudaStream_t s);
void orient_full_compact(const DevGraph& g, DevEff& out, cudaStream_t s);
// Chunked one-pass orientation (tile layout) for a CSR that arrives in
// vertex chunks: begin sizes `out` and the queue/counters; orient_chunk
// orients vertices [vb, ve) (vb a multiple of 32); ready_chunks records for
// each apex of chunk k the chunk after which it can be counted (chunk vertex
// boundaries d_cb, K+1 entries, device); select_ready lists the apexes
// v in [vb, ve) whose ready chunk is k into ids, their number into *cnt.
void orient_chunk_begin(const DevGraph& g, DevEff& out, DBuf<uint32_t>& bigq,
                        DBuf<unsigned long long>& ctr, cudaStream_t s);
void orient_chunk(const DevGraph& g, DevEff& out, uint32_t vb, uint32_t ve, uint32_t* bigq,
                  unsigned long long* ctr, cudaStream_t s);
void ready_chunks(const DevEff& e, const uint32_t* d_cb, uint32_t K, uint32_t k, uint32_t vb,
                  uint32_t ve, uint8_t* ready, cudaStream_t s);
void select_ready(const uint8_t* ready, uint32_t vb, uint32_t ve, uint32_t k, uint32_t* ids,
                  unsigned long long* cnt, cudaStream_t s);
// desc of a compact oriented CSR from its offsets (e.off, e.rows set).
void eff_desc_from_off(DevEff& e, cudaStream_t s);
// Compact copy of a (gappy) oriented CSR: off (n+1) and data (m).
void compact_eff(const DevEff& in, DevEff& out, cudaStream_t s);
// What the slab layout would cost for the oriented lists e of g (host result,
// one sync): entries of the lists longer than a slab, the extra slots their
// full copies reserve (DevGraph::slab_extra), the longest list.
struct SlabStats {
  uint64_t long_entries, extra_slots;
  uint32_t max_len;
};
SlabStats slab_stats(const DevGraph& g, const DevEff& e, cudaStream_t s);
// Fill the slabs of rows [vb, ve) of a slab-layout `e` (base 0) whose lists
// were written elsewhere in e.data (gathered lists: desc points at them).
void slab_rows(DevEff& e, uint32_t vb, uint32_t ve, cudaStream_t s);
extern int g_slab_mode;  // 0 auto, 1 force on, 2 off (tests, A/B)
// sum of the lengths of the lists longer than thr (host result).
uint64_t heavy_entries(const DevEff& e, uint32_t thr, cudaStream_t s);
// sum of list lengths over rows [lo, hi) (host result).
uint64_t sum_lens(const DevEff& e, uint32_t lo, uint32_t hi, cudaStream_t s);
void degree_rank(const DevGraph& g, uint32_t* d_rank, cudaStream_t s);

// ---- edge-list text (io.cu, io.hpp:18-64) ----
// parse_edge_list over a device text buffer padded with >= 16 zero bytes
// past `len` (16-byte aligned).  Returns the pair count (pairs: interleaved
// u, v in file order); on a ParseError returns 0 with *err_line = the
// 1-based line and *err_msg = "line N: ..." (io.hpp:18-22).
uint64_t parse_edge_list_device(const char* d_text, uint64_t len, DBuf<uint32_t>& pairs,
                                cudaStream_t s, uint64_t* err_line, std::string* err_msg);
// write_edge_list: "u v\n" for every edge u < v; returns the byte length.
uint64_t write_edge_list_device(const DevGraph& g, DBuf<char>& out, cudaStream_t s);

// ---- generators (gen.cu): the host harness's R-MAT / Watts-Strogatz
// streams, bit-identical, into a device pair buffer (returns the pair count)
uint64_t gen_rmat_device(uint32_t scale, uint64_t edge_factor, double a, double b, double c,
                         uint64_t seed, DBuf<uint32_t>& pairs, cudaStream_t s);
uint64_t gen_ws_device(uint64_t n, uint64_t k, double beta, uint64_t seed, DBuf<uint32_t>& pairs,
                       cudaStream_t s);

// ---- orders (order.cu, order.hpp:39-128) ----
// Switch g's orientation order to OrderKind{kind, seed}: builds g.okey
// (the rank array) for non-degree kinds.
void set_order(DevGraph& g, int kind, uint64_t seed, cudaStream_t s);
// rank (n) of g's current order.
void order_rank(const DevGraph& g, uint32_t* d_rank, cudaStream_t s);
// coreness (order.hpp:39-83): core numbers (n), parallel peeling.
void coreness_device(const DevGraph& g, uint32_t* d_core, cudaStream_t s);

// ---- costs / plan (costs.cu) ----
// f (n), prefix (n) on device.
void node_costs_device(const DevGraph& g, const DevEff& eff, int kind, uint64_t* d_f,
                       uint64_t* d_prefix, cudaStream_t s);
// boundaries (p+1) on host, from the device prefix array.
std::vector<uint32_t> boundaries_from_prefix(const uint64_t* d_prefix, uint64_t n, uint64_t p,
                                             cudaStream_t s);
uint64_t ordering_cost_device(const DevGraph& g, const DevEff& eff, cudaStream_t s);

// ---- intersection (intersect.cu) ----
struct CountOut {
  unsigned long long* total;   // device, 1 counter
  unsigned long long* tally;   // device n or nullptr (NodeTallySink)
  uint32_t* tri;               // device 3*cap or nullptr (ListSink)
  unsigned long long* cursor;  // device, listing cursor
  uint64_t cap;
  // listing: raw (apex v, middle u, w) as emitted by count_node_iterator_n's
  // sink call (sequential.hpp:82-86) instead of the ListSink normalisation
  bool raw = false;
};

// Rank-labelled view for the bitmap CTA path (ctab.cuh): rank[v] = position
// of v in the orientation order, rdata = the oriented lists with every id
// replaced by its rank (same slots as the id data).  rank == nullptr: off.
struct RankView {
  const uint32_t* rank = nullptr;
  const uint32_t* rdata = nullptr;
  uint32_t n = 0;
  uint32_t cap_bits = 0;  // bitmap capacity (window of ranks above an apex)
};

// Apexes: either CSR rows [vlo, vhi) of `apex` or packed surrogate messages.
struct MsgView {
  const uint32_t* hdr;   // 2*count: (v, len)
  const uint64_t* moff;  // count: data offset of each message
  const uint32_t* data;
  uint64_t count;
};

struct IntersectScratch {
  DBuf<uint32_t> big;               // apex items too long for the warp path
  DBuf<unsigned long long> big_count;
  void ensure(uint64_t cap, cudaStream_t s);
};

// NodeIteratorN over apex rows [vlo, vhi) of `apex`, N_u from `nu`, middle
// vertex u restricted to [ulo, uhi).
// `nu_entries` = size of nu.data (selects 32/64-bit element indexing);
// `unrestricted` = [ulo, uhi) covers every vertex (no middle-vertex filter).
void intersect_rows(CsrView apex, uint32_t vlo, uint32_t vhi, CsrView nu, uint32_t ulo,
                    uint32_t uhi, const CountOut& out, IntersectScratch& scr,
                    cudaStream_t s, uint64_t nu_entries, bool unrestricted,
                    const RankView& rv = RankView{});
// NodeIteratorN over an apex LIST (ids, *d_count entries, device; at most
// max_items): the pipelined count's ready apexes.
void intersect_list(CsrView apex, const uint32_t* ids, const unsigned long long* d_count,
                    uint64_t max_items, CsrView nu, const CountOut& out, IntersectScratch& scr,
                    cudaStream_t s, uint64_t nu_entries, const RankView& rv = RankView{});
// Rank-labelled copy of the oriented lists of `e` (all rows): rdata[slot] =
// rank[data[slot]] for every list slot (rdata sized like e.data).
void rank_lists(const DevEff& e, const uint32_t* d_rank, uint32_t* rdata, cudaStream_t s);
// SurrogateCount (engines.hpp:60-76) over received messages.
void intersect_msgs(const MsgView& msgs, CsrView nu, uint32_t ulo, uint32_t uhi,
                    const CountOut& out, IntersectScratch& scr, cudaStream_t s,
                    uint64_t nu_entries);

void clustering_device(const DevGraph& g, const unsigned long long* d_tally, double* d_c,
                       cudaStream_t s);

// ---- window.cu: local-id-window encoding of the oriented lists ----
// mask bit i <-> v-32+i ∈ N_v; F_v = the rest (inline in the row's 32-byte
// record up to 5 entries, else in far[]).  For graphs whose entries are
// mostly within 32 ids of their row (Watts-Strogatz).
struct WindowEff {
  DBuf<uint4> rec;  // 2 per row: {mask, |F_v|, F_v inline (<= 5) or its position in far}
  DBuf<uint32_t> far;
  DBuf<unsigned long long> ctr;  // [0] far cursor, [1] deferred apexes
  uint64_t rows = 0;
};
// entries of e outside their row's window (host result, one sync)
uint64_t window_far_entries(const DevEff& e, cudaStream_t s);
// (re)build w from e; far_cap >= window_far_entries(e)
void window_build(const DevEff& e, uint64_t far_cap, WindowEff& w, cudaStream_t s);
// NodeIteratorN over apexes [vlo, vhi) into *d_total; apexes with long far
// lists are written to defer (count at w.ctr.p + 1) for the generic kernels
void window_count(WindowEff& w, uint32_t vlo, uint32_t vhi, unsigned long long* d_total,
                  DBuf<uint32_t>& defer, cudaStream_t s);
extern int g_window_mode;  // 0 auto, 1 force on, 2 off (tests)

// ---- analytics.cu (sequential.hpp:48-70, 108-122, sparsify.hpp:113-155) ----
// count_node_iterator_pp under g's current order (host result).
uint64_t node_iterator_pp_device(const DevGraph& g, cudaStream_t s);
// d_up (n+1): exclusive prefix of #neighbours above v (edges() order).
void upper_offsets(const DevGraph& g, uint64_t* d_up, cudaStream_t s);
// bump t_e of the three edges of each listed triple (ascending ids) into
// d_te (and d_te2 when non-null).
void bump_edges(const DevGraph& g, const uint64_t* d_up, const uint32_t* d_tri, uint64_t cnt,
                unsigned long long* d_te, unsigned long long* d_te2, cudaStream_t s);
// sum_e t_e (t_e - 1) / 2 (host result).
uint64_t sum_choose2(const unsigned long long* d_te, uint64_t m, cudaStream_t s);

// ---- sparsify.cu (sparsify.hpp) ----
// Compact copy of `in` keeping entry u of row v iff keep_entry(q, seed, key,
// v, u); key = kc, or owner(v)+1 under the plan d_b (p+1 entries, device)
// when d_b != nullptr.  One host sync (entry count).
void sparsify_eff(const DevEff& in, DevEff& out, double q, uint64_t seed, uint64_t kc,
                  const uint32_t* d_b, uint64_t p, cudaStream_t s);

// launch counter (kernels of ours launched), for bench's gpu_launches claim
extern unsigned long long g_launches;
// CTA-path shared-memory capacity in entries (0 = default); tests lower it
// to exercise the global-memory search path on small graphs.
extern uint32_t g_block_cap;
// warp-path kernel: 0 = automatic, 1 = one apex per warp iteration, 2 = groups
extern int g_warp_variant;
// tests: 64-bit element indexing in the scalar kernels on small graphs (the
// > 2^32-slot path), and the orientation layout (0 auto, 1 compact
// count/scan/fill, 2 one-pass tiles; +4 = 1-byte degree codes)
extern bool g_force_wide;
extern int g_orient_mode;

inline unsigned grid_for(uint64_t work, unsigned block, unsigned cap = 148u * 64u) {
  uint64_t g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

}  // namespace tgb
