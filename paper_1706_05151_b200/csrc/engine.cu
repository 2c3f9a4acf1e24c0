// engine.cu -- engines and the C ABI (include/trigraph_b200.h).
//
// Reference: run_engine (engines.hpp:335-418), clustering_coefficients
// (engines.hpp:422-435), aop_count (:38-54), anop_surrogate_body (:146-198),
// anop_direct_body (:80-141), aggregate_clustering (:211-268).
//
// One tg_graph = one device.  The logical ranks of an EngineConfig run one
// after another on that device with their real data layout:
//   AOP       -- rank i counts apexes of core i against the oriented lists it
//                holds (core + halo; with one device the halo is the resident
//                oriented CSR, its trimmed size is reported as stored_entries);
//   SURROGATE -- rank i holds only its core lists (partition-local CSR with a
//                base offset), packs (v, N_v) per distinct remote owner,
//                "sends" by concatenating destination segments, and each
//                owner runs local intersections + SurrogateCount;
//   DIRECT    -- counts as AOP (the apex owner fetches N_u); message counts
//                follow the request/reply protocol.
// The multi-process path (one process per GPU, paper_1706_05151_b200/
// distributed.py) calls the same kernels through the rank-local entries.
#include <algorithm>
#include <cstring>
#include <mutex>

#include "exchange.cuh"
#include "handle.cuh"
#include "tg_internal.cuh"


namespace {

thread_local std::string t_last_error;
uint64_t g_chunk_entries = 0;  // tg_count_from_csr chunk size (0: default)
int g_rank_bitmap = 0;         // bitmap CTA path: 0 auto, 1 on, 2 off
uint32_t g_rank_cap = 0;       // its window capacity in bits (0: 2^19)

}  // namespace
void tgb_set_error(const std::string& msg) { t_last_error = msg; }
namespace {

template <class F>
tg_status guard(F&& f) {
  try {
    f();
    return TG_OK;
  } catch (const tgb::Error& e) {
    t_last_error = e.what();
    return e.status;
  } catch (const std::bad_alloc& e) {
    t_last_error = e.what();
    return TG_ERR_OOM;
  } catch (const std::exception& e) {
    t_last_error = e.what();
    return TG_ERR_INTERNAL;
  }
}

using tgb::CountOut;
using tgb::CsrView;
using tgb::RankView;
using tgb::DBuf;
using tgb::DevEff;

CsrView view(const DevEff& e) {
  CsrView v{e.desc.p, e.data.p, e.base, e.rows ? (float)e.entries / (float)e.rows : 0.f};
  v.slab = e.slab;
  return v;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

template <class T>
void upload(DBuf<T>& dst, const T* src, size_t count, cudaStream_t s) {
  dst.alloc(count ? count : 1, s);
  if (count)
    TG_CUDA(cudaMemcpyAsync(dst.p, src, count * sizeof(T),
                            is_device_ptr(src) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
}

template <class T>
void download(T* dst, const T* src, size_t count, cudaStream_t s) {
  if (count && dst) TG_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToHost, s));
}

void enter(tg_graph* g) {
  TG_REQUIRE(g != nullptr, "null graph handle");
  TG_CUDA(cudaSetDevice(g->device));
}

void sync(tg_graph* g) { TG_CUDA(cudaStreamSynchronize(g->stream)); }

tg_graph* new_graph(int device) {
  int count = 0;
  TG_CUDA(cudaGetDeviceCount(&count));
  TG_REQUIRE(device >= 0 && device < count, "invalid CUDA device ordinal");
  TG_CUDA(cudaSetDevice(device));
  // keep freed stream-ordered allocations in the pool instead of returning
  // them to the driver at every synchronisation (per-step scratch buffers)
  cudaMemPool_t pool;
  TG_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t keep = UINT64_MAX;
  TG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  auto* g = new tg_graph;
  g->device = device;
  TG_CUDA(cudaStreamCreateWithFlags(&g->own, cudaStreamNonBlocking));
  g->stream = g->own;
  TG_CUDA(cudaEventCreate(&g->ev0));
  TG_CUDA(cudaEventCreate(&g->ev1));
  return g;
}

// Orient by OrderKind{kind, seed} from now on (order.hpp:85-128); the cached
// oriented CSR and rank partitions are dropped when the order changes.
void apply_order(tg_graph* g, int kind, uint64_t seed) {
  TG_REQUIRE(kind >= TG_ORDER_BY_ID && kind <= TG_ORDER_BY_CORENESS, "unknown order kind");
  // (a caller's OrderRank, TG_ORDER_RANK, is only set by tg_set_order_rank)
  const uint64_t sd = kind == TG_ORDER_BY_RANDOM ? seed : 0;
  if (g->g.order == kind && g->g.order_seed == sd) return;
  tgb::set_order(g->g, kind, sd, g->stream);
  g->have_eff = false;
  g->have_part = false;
  g->have_rk = false;
  g->rank_mode = -1;
  g->window_mode = -1;
  g->slab_mode = -1;
  g->comm_slab = -1;
  g->g.slab = 0;
}

// (Re)orient the whole graph (effective.hpp:37-52).  The first orientation
// under an order also decides the layout: the slab layout (one 128-byte line
// per list, no descriptor on the intersection's random reads) when the
// per-apex kernel would run (mean list > 16: PA-like graphs), at most 2% of
// the entries sit in lists longer than a slab and none is longer than 4096;
// or as forced by tg_debug_set_slab.
void orient(tg_graph* g) {
  TG_REQUIRE(!g->partial,
             "a rank-local graph (tg_graph_from_rows) is oriented by the tg_*_comm entry points");
  if (g->slab_mode >= 0 && g->slab_for != tgb::g_slab_mode) {
    g->slab_mode = -1;
    g->g.slab = 0;
  }
  if (tgb::order_nibble_wanted(g->g) && g->g.nibble == 0) tgb::build_nibble_codes(g->g, g->stream);
  tgb::orient_full(g->g, g->eff, g->stream);
  if (g->slab_mode < 0) {
    g->slab_for = tgb::g_slab_mode;
    g->slab_mode = 0;
    const uint64_t n = g->g.n, m = g->g.m2 / 2;
    if (tgb::g_slab_mode != 2 && n && n < 0xffffffffull && (tgb::g_orient_mode & 3) == 0) {
      const tgb::SlabStats st = tgb::slab_stats(g->g, g->eff, g->stream);
      const bool fits = n * tgb::kSlab + g->g.big_entries + st.extra_slots + tgb::kQuadPad < (1ull << 34);
      const bool pays = m > 16 * n && st.long_entries * 50 <= m && st.max_len <= 4096;
      if (fits && (pays || tgb::g_slab_mode == 1)) {
        g->slab_mode = 1;
        g->g.slab = tgb::kSlab;
        g->g.slab_extra = st.extra_slots;
        g->eff.data.release();  // (the tile-layout buffer; the slabs are sized anew)
        tgb::orient_full(g->g, g->eff, g->stream);
      }
    }
  }
  g->have_eff = true;
  ++g->eff_gen;
}

void ensure_eff(tg_graph* g) {
  if (!g->have_eff) orient(g);
}

// The full oriented CSR as a kernel view (oriented on first use).
CsrView full_view(tg_graph* g) {
  ensure_eff(g);
  return view(g->eff);
}

// The bitmap CTA path's inputs when it pays (auto: the apexes with > 64
// oriented entries -- the CTA path -- hold more than 1% of the entries), or
// as forced by tg_debug_set_rank_bitmap.  Rebuilds the rank-labelled lists
// after every orientation (a gather over the m entries).
RankView rank_view(tg_graph* g) {
  const uint64_t n = g->g.n;
  if (g_rank_bitmap == 2 || !n || g->eff.data.n + tgb::kQuadPad >= (1ull << 34)) return {};
  cudaStream_t s = g->stream;
  if (g_rank_bitmap == 0 && g->rank_mode < 0)
    g->rank_mode = tgb::heavy_entries(g->eff, 64, s) * 100 > g->eff.entries ? 1 : 0;
  if (g_rank_bitmap == 0 && g->rank_mode == 0) return {};
  if (!g->have_rk) {
    g->rk.alloc(n, s);
    tgb::order_rank(g->g, g->rk.p, s);
    g->have_rk = true;
  }
  if (g->rdata_gen != g->eff_gen) {
    if (g->rdata.n < g->eff.data.n) g->rdata.alloc(g->eff.data.n, s);
    tgb::rank_lists(g->eff, g->rk.p, g->rdata.p, s);
    g->rdata_gen = g->eff_gen;
  }
  return RankView{g->rk.p, g->rdata.p, (uint32_t)n, g_rank_cap ? g_rank_cap : (1u << 19)};
}

// The window encoding (window.cu) when it pays: automatic when at most 10%
// of the oriented entries lie outside their row's 64-id window (decided once
// per order from one counting pass), or as forced by tg_debug_set_window.
// Rebuilt after every orientation.
bool window_ready(tg_graph* g) {
  if (tgb::g_window_mode == 2 || !g->g.n) return false;
  cudaStream_t s = g->stream;
  if (g->window_mode < 0) {
    g->window_far = tgb::window_far_entries(g->eff, s);
    g->window_mode = g->window_far * 10 <= g->eff.entries ? 1 : 0;
  }
  if (g->window_mode == 0 && tgb::g_window_mode != 1) return false;
  if (g->window_gen != g->eff_gen) {
    tgb::window_build(g->eff, g->window_far, g->win, s);
    g->window_gen = g->eff_gen;
  }
  return true;
}

// NodeIteratorN over apexes [vlo, vhi) through the window encoding; the
// deferred apexes (long far lists) through the generic kernels.
void window_rows(tg_graph* g, uint32_t vlo, uint32_t vhi, unsigned long long* d_total) {
  cudaStream_t s = g->stream;
  tgb::window_count(g->win, vlo, vhi, d_total, g->wdefer, s);
  const CsrView full = view(g->eff);
  tgb::intersect_list(full, g->wdefer.p, g->win.ctr.p + 1, vhi - vlo, full,
                      CountOut{d_total, nullptr, nullptr, nullptr, 0}, g->scr, s, g->eff.data.n,
                      rank_view(g));
}

// Counting pass with CUDA-event timing of the intersection kernels.
template <class F>
void timed_pass(tg_graph* g, F&& f) {
  TG_CUDA(cudaEventRecord(g->ev0, g->stream));
  f();
  TG_CUDA(cudaEventRecord(g->ev1, g->stream));
  g->timed = true;
}

std::vector<uint32_t> plan_for(tg_graph* g, int cost, uint64_t p, const uint32_t* override_b) {
  std::vector<uint32_t> b;
  if (override_b) {
    b.assign(override_b, override_b + p + 1);
    TG_REQUIRE(b[0] == 0 && b[p] <= g->g.n, "boundaries must start at 0 and end at <= n");
    for (uint64_t i = 0; i < p; ++i) TG_REQUIRE(b[i] <= b[i + 1], "boundaries must be sorted");
    return b;
  }
  DBuf<uint64_t> f(g->g.n ? g->g.n : 1, g->stream), pre(g->g.n ? g->g.n : 1, g->stream);
  tgb::node_costs_device(g->g, g->eff, cost, f.p, pre.p, g->stream);
  return tgb::boundaries_from_prefix(pre.p, g->g.n, p, g->stream);
}

// host copy of an inclusive prefix of f (for per-rank realized cost)
std::vector<uint64_t> range_sums(tg_graph* g, int cost, const std::vector<uint32_t>& b) {
  const uint64_t n = g->g.n, p = b.size() - 1;
  std::vector<uint64_t> out(p, 0);
  if (!n) return out;
  DBuf<uint64_t> f(n, g->stream), pre(n, g->stream);
  tgb::node_costs_device(g->g, g->eff, cost, f.p, pre.p, g->stream);
  std::vector<uint64_t> at(p + 1, 0);
  for (uint64_t i = 0; i <= p; ++i)
    if (b[i] > 0) download(&at[i], pre.p + (b[i] - 1), 1, g->stream);
  sync(g);
  for (uint64_t i = 0; i < p; ++i) out[i] = at[i + 1] - at[i];
  return out;
}

struct EngineResult {
  std::vector<uint32_t> b;
  std::vector<tg_rank_stats> per_rank;
  uint64_t total = 0;
};

// The engines.  `tally`/`tri` are device outputs (may be null).
EngineResult run(tg_graph* g, const tg_config& cfg, unsigned long long* d_tally, uint32_t* d_tri,
                 unsigned long long* d_cursor, uint64_t cap) {
  TG_REQUIRE(cfg.engine >= TG_ENGINE_SEQ && cfg.engine <= TG_ENGINE_ANOP_SURROGATE, "unknown engine");
  const uint64_t p = cfg.engine == TG_ENGINE_SEQ ? 1 : cfg.ranks;
  TG_REQUIRE(p >= 1, "run_engine: ranks must be >= 1");  // engines.hpp:337-338
  TG_REQUIRE(cfg.cost >= TG_COST_N && cfg.cost <= TG_COST_NOV, "unknown cost kind");
  cudaStream_t s = g->stream;
  if (cfg.order_set) apply_order(g, cfg.order, cfg.order_seed);  // engines.hpp:341
  ensure_eff(g);
  const uint64_t n = g->g.n;
  EngineResult R;
  R.b = plan_for(g, cfg.cost, p, cfg.boundaries);
  const auto& b = R.b;
  R.per_rank.assign(p, tg_rank_stats{0, 0, 0, 0, 0});
  DBuf<unsigned long long> ctr(p, s);
  ctr.zero();
  auto out_for = [&](uint64_t i) {
    return CountOut{ctr.p + i, d_tally, d_tri, d_cursor, cap};
  };
  const CsrView full = full_view(g);
  const uint32_t N = (uint32_t)n;
  // sparsify.hpp: the engines below count over sparsified lists; partition
  // storage (stored_entries) is reported as built, before sparsification
  const int sp = cfg.sparsify;
  TG_REQUIRE(sp >= TG_SPARSIFY_NONE && sp <= TG_SPARSIFY_PER_PARTITION, "unknown sparsify mode");
  if (sp) TG_REQUIRE(cfg.sparsify_q > 0.0 && cfg.sparsify_q <= 1.0, "sparsify: q must be in (0, 1]");
  const double sq = cfg.sparsify_q;
  const uint64_t sseed = cfg.sparsify_seed;
  DBuf<uint32_t> d_b;
  if (sp == TG_SPARSIFY_PER_PARTITION && cfg.engine == TG_ENGINE_ANOP_DIRECT)
    upload(d_b, b.data(), b.size(), s);

  if (cfg.engine == TG_ENGINE_SEQ) {
    // engines.hpp:362-365 / sparsify.hpp:94-107: rank 0's draws
    DevEff es;
    if (sp) tgb::sparsify_eff(g->eff, es, sq, sseed, sp == TG_SPARSIFY_PER_PARTITION ? 1 : 0,
                              nullptr, 0, s);
    const DevEff& E = sp ? es : g->eff;
    const CsrView ev = sp ? view(E) : full_view(g);
    timed_pass(g, [&] {
      const RankView rv = sp ? RankView{} : rank_view(g);
      tgb::intersect_rows(ev, 0, N, ev, 0, N, out_for(0), g->scr, s, E.data.n, true, rv);
    });
    R.per_rank[0].stored_entries = g->eff.entries;
  } else if (sp && cfg.engine == TG_ENGINE_AOP) {
    // engines.hpp:367-371 + sparsify.hpp:80-84: each rank sparsifies its
    // overlap partition with its own draws; N'_v lies in core+halo, so the
    // rank's count is NodeIteratorN over its apexes on the adjacency
    // sparsified with its key
    DevEff es;
    if (sp == TG_SPARSIFY_GLOBAL) tgb::sparsify_eff(g->eff, es, sq, sseed, 0, nullptr, 0, s);
    for (uint64_t i = 0; i < p; ++i) {
      if (sp == TG_SPARSIFY_PER_PARTITION) tgb::sparsify_eff(g->eff, es, sq, sseed, i + 1, nullptr, 0, s);
      const CsrView ev = view(es);
      if (b[i + 1] > b[i])
        tgb::intersect_rows(ev, b[i], b[i + 1], ev, 0, N, out_for(i), g->scr, s, es.data.n, true);
      R.per_rank[i].stored_entries = tgb::overlap_stored_entries(full, n, b[i], b[i + 1], s);
    }
  } else if (cfg.engine == TG_ENGINE_AOP || cfg.engine == TG_ENGINE_ANOP_DIRECT) {
    // direct (engines.hpp:80-141): every rank's core lists with its own
    // draws (owner key), then the same requests over the kept entries
    DevEff es;
    if (sp) tgb::sparsify_eff(g->eff, es, sq, sseed, 0,
                              sp == TG_SPARSIFY_PER_PARTITION ? d_b.p : nullptr, p, s);
    const DevEff& E = sp ? es : g->eff;
    const CsrView ev = sp ? view(E) : full_view(g);
    timed_pass(g, [&] {
      const RankView rv = sp ? RankView{} : rank_view(g);
      for (uint64_t i = 0; i < p; ++i)
        if (b[i + 1] > b[i])
          tgb::intersect_rows(ev, b[i], b[i + 1], ev, 0, N, out_for(i), g->scr, s,
                              E.data.n, true, rv);
    });
    if (cfg.engine == TG_ENGINE_AOP) {
      for (uint64_t i = 0; i < p; ++i)
        R.per_rank[i].stored_entries = tgb::overlap_stored_entries(full, n, b[i], b[i + 1], s);
    } else {
      std::vector<uint64_t> req, rep;
      tgb::direct_messages(ev, n, b, req, rep, s);
      for (uint64_t i = 0; i < p; ++i) {
        R.per_rank[i].data_sent = req[i] + rep[i];
        R.per_rank[i].data_recv = req[i] + rep[i];
      }
      for (uint64_t i = 0; i < p; ++i)
        R.per_rank[i].stored_entries = tgb::sum_lens(g->eff, b[i], b[i + 1], s);
    }
  } else {  // ANOP surrogate
    std::vector<DevEff> parts(p);
    std::vector<tgb::SurrogatePack> packs(p);
    std::vector<DBuf<uint32_t>> hdr(p), dat(p);
    for (uint64_t i = 0; i < p; ++i) {
      tgb::orient_rows(g->g, b[i], b[i + 1], parts[i], s);  // non-overlapping storage
      R.per_rank[i].stored_entries = parts[i].entries;
      if (sp) {  // sparsify.hpp:86-90: the rank's core lists, its own draws
        DevEff es;
        tgb::sparsify_eff(parts[i], es, sq, sseed, sp == TG_SPARSIFY_PER_PARTITION ? i + 1 : 0,
                          nullptr, 0, s);
        parts[i] = std::move(es);
      }
      packs[i].build(view(parts[i]), b[i], b[i + 1], b, (uint32_t)i, s);
      uint64_t msgs = 0, words = 0;
      for (uint64_t j = 0; j < p; ++j) {
        msgs += packs[i].msgs_per_dest[j];
        words += packs[i].words_per_dest[j];
        R.per_rank[i].data_sent += packs[i].msgs_per_dest[j];
        R.per_rank[j].data_recv += packs[i].msgs_per_dest[j];
      }
      hdr[i].alloc(2 * msgs + 1, s);
      dat[i].alloc(words + 1, s);
      packs[i].scatter(hdr[i].p, dat[i].p, s);
    }
    // "all-to-allv": receive buffer of rank j = dest-j segments of every sender
    std::vector<DBuf<uint32_t>> rh(p), rd(p);
    std::vector<uint64_t> rmsgs(p, 0);
    for (uint64_t j = 0; j < p; ++j) {
      uint64_t msgs = 0, words = 0;
      for (uint64_t i = 0; i < p; ++i) {
        msgs += packs[i].msgs_per_dest[j];
        words += packs[i].words_per_dest[j];
      }
      rmsgs[j] = msgs;
      rh[j].alloc(2 * msgs + 1, s);
      rd[j].alloc(words + 1, s);
      uint64_t mo = 0, wo = 0;
      for (uint64_t i = 0; i < p; ++i) {
        uint64_t m0 = 0, w0 = 0;
        for (uint64_t jj = 0; jj < j; ++jj) {
          m0 += packs[i].msgs_per_dest[jj];
          w0 += packs[i].words_per_dest[jj];
        }
        const uint64_t mi = packs[i].msgs_per_dest[j], wi = packs[i].words_per_dest[j];
        if (mi)
          TG_CUDA(cudaMemcpyAsync(rh[j].p + 2 * mo, hdr[i].p + 2 * m0, 2 * mi * 4,
                                  cudaMemcpyDeviceToDevice, s));
        if (wi)
          TG_CUDA(cudaMemcpyAsync(rd[j].p + wo, dat[i].p + w0, wi * 4, cudaMemcpyDeviceToDevice, s));
        mo += mi;
        wo += wi;
      }
    }
    std::vector<DBuf<uint64_t>> moff(p);
    for (uint64_t j = 0; j < p; ++j) tgb::message_offsets(rh[j].p, rmsgs[j], moff[j], s);
    timed_pass(g, [&] {
      for (uint64_t j = 0; j < p; ++j) {
        if (b[j + 1] <= b[j]) continue;
        const CsrView pv = view(parts[j]);
        tgb::intersect_rows(pv, b[j], b[j + 1], pv, b[j], b[j + 1], out_for(j), g->scr, s,
                            parts[j].data.n, false);
        tgb::MsgView mv{rh[j].p, moff[j].p, rd[j].p, rmsgs[j]};
        tgb::intersect_msgs(mv, pv, b[j], b[j + 1], out_for(j), g->scr, s, parts[j].data.n);
      }
    });
  }
  std::vector<unsigned long long> h(p);
  download(h.data(), ctr.p, p, s);
  sync(g);
  for (uint64_t i = 0; i < p; ++i) {
    R.per_rank[i].triangles = h[i];
    R.total += h[i];
  }
  // realized cost = algorithmic work of the rank: DPD over apex cores
  // (AOP / direct / seq), NOV over middle-vertex cores (surrogate).
  auto rc = range_sums(g, cfg.engine == TG_ENGINE_ANOP_SURROGATE ? TG_COST_NOV : TG_COST_DPD, b);
  for (uint64_t i = 0; i < p; ++i) R.per_rank[i].realized_cost = rc[i];
  return R;
}

uint64_t seq_count(tg_graph* g) {
  ensure_eff(g);
  cudaStream_t s = g->stream;
  DBuf<unsigned long long> ctr(1, s);
  ctr.zero();
  const CsrView full = full_view(g);
  const uint32_t N = (uint32_t)g->g.n;
  const bool win = window_ready(g);
  timed_pass(g, [&] {
    if (win)
      window_rows(g, 0, N, ctr.p);
    else
      tgb::intersect_rows(full, 0, N, full, 0, N, CountOut{ctr.p, nullptr, nullptr, nullptr, 0},
                          g->scr, s, g->eff.data.n, true, rank_view(g));
  });
  unsigned long long h = 0;
  download(&h, ctr.p, 1, s);
  sync(g);
  return h;
}

void prepare_part(tg_graph* g, const uint32_t* boundaries, uint64_t p, uint64_t rank) {
  TG_REQUIRE(boundaries && p >= 1 && rank < p, "invalid rank / boundaries");
  std::vector<uint32_t> b(boundaries, boundaries + p + 1);
  TG_REQUIRE(b[0] == 0 && b[p] <= g->g.n, "boundaries must start at 0 and end at <= n");
  if (g->have_part && g->part_rank == rank && g->part_b == b) return;
  tgb::orient_rows(g->g, b[rank], b[rank + 1], g->part, g->stream);
  g->pack.build(view(g->part), b[rank], b[rank + 1], b, (uint32_t)rank, g->stream);
  g->part_b = b;
  g->part_rank = rank;
  g->have_part = true;
}

}  // namespace

namespace {

// NodeIteratorN listing of apexes [lo, hi) in pieces whose triangles fit the
// buffer (count first; halve the apex range while it holds too many).
template <class F>
void list_in_pieces(tg_graph* g, uint32_t lo, uint32_t hi, DBuf<uint32_t>& tri, uint64_t cap,
                    F&& f) {
  if (hi <= lo) return;
  cudaStream_t s = g->stream;
  const CsrView full = full_view(g);
  const uint32_t N = (uint32_t)g->g.n;
  DBuf<unsigned long long> c(2, s);
  c.zero();
  tgb::intersect_rows(full, lo, hi, full, 0, N, CountOut{c.p, nullptr, nullptr, nullptr, 0},
                      g->scr, s, g->eff.data.n, true, rank_view(g));
  unsigned long long cnt = 0;
  download(&cnt, c.p, 1, s);
  sync(g);
  if (!cnt) return;
  if (cnt > cap && hi - lo > 1) {
    const uint32_t mid = lo + (hi - lo) / 2;
    list_in_pieces(g, lo, mid, tri, cap, f);
    list_in_pieces(g, mid, hi, tri, cap, f);
    return;
  }
  TG_REQUIRE(cnt <= cap, "one apex has more triangles than the listing buffer");
  c.zero();
  tgb::intersect_rows(full, lo, hi, full, 0, N, CountOut{c.p, nullptr, tri.p, c.p + 1, cap},
                      g->scr, s, g->eff.data.n, true);
  f(tri.p, (uint64_t)cnt);
}

constexpr uint64_t kListCap = 1ull << 26;  // triples per listing piece (768 MB)

}  // namespace

namespace {

// The text in a device buffer padded with 16 zero bytes past len (the parse
// kernels read aligned 16-byte groups); a host text is uploaded into it.
void stage_text(const char* text, uint64_t len, DBuf<char>& buf, cudaStream_t s) {
  buf.alloc(len + 32, s);
  TG_CUDA(cudaMemsetAsync(buf.p + len, 0, 32, s));
  if (len)
    TG_CUDA(cudaMemcpyAsync(buf.p, text, len,
                            is_device_ptr(text) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
}

struct ParseFailure {
  uint64_t line;
  std::string msg;
};

// parse_edge_list on the device; throws ParseFailure (mapped to TG_ERR_PARSE)
uint64_t parse_text(const char* text, uint64_t len, DBuf<uint32_t>& pairs, cudaStream_t s) {
  DBuf<char> buf;
  stage_text(text, len, buf, s);
  uint64_t line = 0;
  std::string msg;
  const uint64_t E = tgb::parse_edge_list_device(buf.p, len, pairs, s, &line, &msg);
  if (line) throw ParseFailure{line, msg};
  return E;
}

template <class F>
tg_status parse_guard(uint64_t* err_line, F&& f) {
  if (err_line) *err_line = 0;
  try {
    return guard([&] { f(); });
  } catch (const ParseFailure& e) {
    if (err_line) *err_line = e.line;
    t_last_error = e.msg;
    return TG_ERR_PARSE;
  }
}

}  // namespace

namespace {
template <class Gen>
tg_status graph_from_generator(int device, uint64_t n_override, tg_graph** out, Gen&& gen) {
  return guard([&] {
    TG_REQUIRE(out != nullptr, "null output handle");
    tg_graph* g = new_graph(device);
    try {
      DBuf<uint32_t> pairs;
      const uint64_t E = gen(pairs, g->stream);
      tgb::build_graph_device(pairs.p, E, n_override, g->g, g->stream);
      sync(g);
    } catch (...) {
      tg_graph_free(g);
      throw;
    }
    *out = g;
  });
}
}  // namespace

namespace tgh {  // the helpers above, for comm.cu
tg_graph* new_graph(int device) { return ::new_graph(device); }
void enter(tg_graph* g) { ::enter(g); }
void sync(tg_graph* g) { ::sync(g); }
void ensure_eff(tg_graph* g) { ::ensure_eff(g); }
tgb::CsrView view(const tgb::DevEff& e) { return ::view(e); }
tgb::CsrView full_view(tg_graph* g) { return ::full_view(g); }
tgb::RankView rank_view(tg_graph* g) { return ::rank_view(g); }
bool window_ready(tg_graph* g) { return ::window_ready(g); }
void window_rows(tg_graph* g, uint32_t vlo, uint32_t vhi, unsigned long long* d_total) {
  ::window_rows(g, vlo, vhi, d_total);
}
std::vector<uint32_t> plan_for(tg_graph* g, int cost, uint64_t p, const uint32_t* override_b) {
  return ::plan_for(g, cost, p, override_b);
}
bool is_device_ptr(const void* p) { return ::is_device_ptr(p); }
void install_eff(tg_graph* g, tgb::DevEff&& e) {
  g->eff = std::move(e);
  g->have_eff = true;
  ++g->eff_gen;
  g->have_part = false;
}
}  // namespace tgh

extern "C" {

const char* tg_last_error(void) { return t_last_error.c_str(); }

const char* tg_status_string(tg_status s) {
  switch (s) {
    case TG_OK: return "ok";
    case TG_ERR_INVALID_ARGUMENT: return "invalid argument";
    case TG_ERR_CUDA: return "CUDA error";
    case TG_ERR_OOM: return "out of device memory";
    case TG_ERR_CAPACITY: return "output capacity too small";
    case TG_ERR_INTERNAL: return "internal error";
    case TG_ERR_PARSE: return "parse error";
  }
  return "unknown status";
}

uint64_t tg_kernel_launches(void) { return tgb::g_launches; }

void tg_debug_set_block_cap(uint32_t entries) { tgb::g_block_cap = entries; }

void tg_debug_set_chunk_entries(uint64_t entries) { g_chunk_entries = entries; }

void tg_debug_set_warp_variant(int32_t variant) { tgb::g_warp_variant = variant; }

void tg_debug_set_rank_bitmap(int32_t mode, uint32_t cap_bits) {
  g_rank_bitmap = mode;
  g_rank_cap = cap_bits ? std::max<uint32_t>(32, (cap_bits + 31) & ~31u) : 0;
}

void tg_debug_set_window(int32_t mode) { tgb::g_window_mode = mode; }
void tg_debug_set_slab(int32_t mode) { tgb::g_slab_mode = mode; }

void tg_debug_set_paths(int32_t orient_mode, int32_t force_wide) {
  tgb::g_orient_mode = orient_mode;
  tgb::g_force_wide = force_wide != 0;
}

tg_status tg_graph_from_edges(int device, const uint32_t* pairs, uint64_t num_pairs,
                              uint64_t n_override, tg_graph** out) {
  return guard([&] {
    TG_REQUIRE(out != nullptr, "null output handle");
    TG_REQUIRE(pairs != nullptr || num_pairs == 0, "null pairs");
    tg_graph* g = new_graph(device);
    try {
      DBuf<uint32_t> dp;
      upload(dp, pairs, 2 * num_pairs, g->stream);
      tgb::build_graph_device(dp.p, num_pairs, n_override, g->g, g->stream);
      sync(g);
    } catch (...) {
      tg_graph_free(g);
      throw;
    }
    *out = g;
  });
}

tg_status tg_graph_from_text(int device, const char* text, uint64_t len, uint64_t n_override,
                             tg_graph** out, uint64_t* err_line) {
  return parse_guard(err_line, [&] {
    TG_REQUIRE(out != nullptr, "null output handle");
    TG_REQUIRE(text != nullptr || len == 0, "null text");
    tg_graph* g = new_graph(device);
    try {
      DBuf<uint32_t> pairs;
      const uint64_t E = parse_text(text, len, pairs, g->stream);
      tgb::build_graph_device(pairs.p, E, n_override, g->g, g->stream);
      sync(g);
    } catch (...) {
      tg_graph_free(g);
      throw;
    }
    *out = g;
  });
}

tg_status tg_parse_edge_list(int device, const char* text, uint64_t len, uint32_t* pairs,
                             uint64_t capacity, uint64_t* num_pairs, uint64_t* err_line) {
  tg_status cap_status = TG_OK;
  tg_status st = parse_guard(err_line, [&] {
    TG_REQUIRE(num_pairs != nullptr, "null output");
    TG_REQUIRE(text != nullptr || len == 0, "null text");
    int count = 0;
    TG_CUDA(cudaGetDeviceCount(&count));
    TG_REQUIRE(device >= 0 && device < count, "invalid CUDA device ordinal");
    TG_CUDA(cudaSetDevice(device));
    cudaStream_t s;
    TG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    try {
      DBuf<uint32_t> d;
      const uint64_t E = parse_text(text, len, d, s);
      *num_pairs = E;
      if (pairs && E)
        TG_CUDA(cudaMemcpyAsync(pairs, d.p, 8 * std::min(E, capacity),
                                is_device_ptr(pairs) ? cudaMemcpyDeviceToDevice
                                                     : cudaMemcpyDeviceToHost, s));
      d.release();
      TG_CUDA(cudaStreamSynchronize(s));
      if (pairs && capacity < E) cap_status = TG_ERR_CAPACITY;  // NULL: size query
    } catch (...) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
      throw;
    }
    TG_CUDA(cudaStreamDestroy(s));
  });
  if (st == TG_OK && cap_status != TG_OK) {
    t_last_error = "pair capacity smaller than the edge count";
    return cap_status;
  }
  return st;
}

tg_status tg_write_edge_list(tg_graph* g, char* out, uint64_t capacity, uint64_t* len) {
  tg_status cap_status = TG_OK;
  tg_status st = guard([&] {
    enter(g);
    TG_REQUIRE(len != nullptr, "null output");
    DBuf<char> d;
    const uint64_t L = tgb::write_edge_list_device(g->g, d, g->stream);
    *len = L;
    if (out && L)
      TG_CUDA(cudaMemcpyAsync(out, d.p, std::min(L, capacity),
                              is_device_ptr(out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                              g->stream));
    sync(g);
    if (out && capacity < L) cap_status = TG_ERR_CAPACITY;
  });
  if (st == TG_OK && cap_status != TG_OK) {
    t_last_error = "text capacity smaller than the edge list";
    return cap_status;
  }
  return st;
}

tg_status tg_count_from_csr(int device, uint64_t n, const uint64_t* offsets, const uint32_t* adj,
                            uint64_t* total) {
  return tg_count_from_csr_range(device, n, offsets, adj, 0, n, total);
}

tg_status tg_count_from_csr_range(int device, uint64_t n, const uint64_t* offsets,
                                  const uint32_t* adj, uint64_t vlo, uint64_t vhi,
                                  uint64_t* total) {
  return guard([&] {
    TG_REQUIRE(vlo <= vhi && vhi <= n, "apex range must satisfy vlo <= vhi <= n");
    TG_REQUIRE(total != nullptr && offsets != nullptr, "null argument");
    TG_REQUIRE(n <= 0xFFFFFFFFull, "n must fit NodeId");
    if (is_device_ptr(offsets) || (adj && is_device_ptr(adj))) {
      // already resident: nothing to overlap
      tg_graph* h = nullptr;
      tg_status st = tg_graph_from_csr(device, n, offsets, adj, &h);
      if (st != TG_OK) throw tgb::Error(st, t_last_error);
      if (vlo == 0 && vhi == n) {
        st = tg_count(h, total);
      } else {
        // AOP rank body over [vlo, vhi) (engines.hpp:38-54): core 1 of a 3-part plan
        DBuf<unsigned long long> d(1, h->stream);
        d.zero();
        const uint32_t plan[4] = {0, (uint32_t)vlo, (uint32_t)vhi, (uint32_t)n};
        st = tg_aop_rank_device(h, plan, 3, 1, (uint64_t*)d.p);
        if (st == TG_OK) {
          unsigned long long v = 0;
          download(&v, d.p, 1, h->stream);
          sync(h);
          *total = v;
        }
      }
      const std::string err = t_last_error;
      tg_graph_free(h);
      if (st != TG_OK) throw tgb::Error(st, err);
      return;
    }
    const uint64_t m2 = offsets[n];
    TG_REQUIRE(m2 % 2 == 0, "symmetric CSR must hold an even number of entries");
    TG_REQUIRE(adj != nullptr || m2 == 0, "null adjacency");
    tg_graph* g = new_graph(device);
    cudaStream_t cs = nullptr;
    std::vector<cudaEvent_t> evs;
    auto cleanup = [&] {
      if (cs) {
        cudaStreamSynchronize(cs);
        cudaStreamDestroy(cs);
      }
      for (auto e : evs) cudaEventDestroy(e);
      tg_graph_free(g);
    };
    try {
      cudaStream_t s = g->stream;
      TG_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      g->g.n = n;
      g->g.m2 = m2;
      g->g.off.alloc(n + 1, s);
      g->g.adj.alloc(m2 ? m2 : 1, s);
      TG_CUDA(cudaStreamSynchronize(s));  // allocations visible to the copy stream
      // chunks of ~2^24 adjacency entries (64 MB; measured best on C2 among
      // 2^23..2^27), vertex boundaries on tiles
      const uint64_t per = g_chunk_entries ? g_chunk_entries : (1ull << 24);
      const uint64_t K = std::min<uint64_t>(64, std::max<uint64_t>(1, m2 / per));
      std::vector<uint32_t> cb(K + 1, 0);
      cb[K] = (uint32_t)n;
      for (uint64_t k = 1; k < K; ++k) {
        const uint64_t target = m2 * k / K;
        const uint64_t v = (uint64_t)(std::lower_bound(offsets, offsets + n + 1, target) - offsets);
        cb[k] = (uint32_t)std::max<uint64_t>(cb[k - 1], std::min<uint64_t>(n, v & ~31ull));
      }
      evs.resize(K + 1);
      for (auto& e : evs) TG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      auto copy_chunk = [&](uint64_t k) {
        const uint64_t a = offsets[cb[k]], b = offsets[cb[k + 1]];
        if (b > a)
          TG_CUDA(cudaMemcpyAsync(g->g.adj.p + a, adj + a, (b - a) * 4, cudaMemcpyHostToDevice, cs));
        TG_CUDA(cudaEventRecord(evs[k + 1], cs));
      };
      TG_CUDA(cudaMemcpyAsync(g->g.off.p, offsets, (n + 1) * 8, cudaMemcpyHostToDevice, cs));
      TG_CUDA(cudaEventRecord(evs[0], cs));
      copy_chunk(0);
      TG_CUDA(cudaStreamWaitEvent(s, evs[0], 0));
      tgb::compute_degrees(g->g, s);  // host sync on the offsets only
      DBuf<uint32_t> bigq, ids(n ? n : 1, s), d_cb(K + 1, s);
      DBuf<unsigned long long> ctr, cnt(1, s), d_total(1, s);
      DBuf<uint8_t> ready(n ? n : 1, s);
      d_total.zero();
      TG_CUDA(cudaMemcpyAsync(d_cb.p, cb.data(), (K + 1) * 4, cudaMemcpyHostToDevice, s));
      tgb::orient_chunk_begin(g->g, g->eff, bigq, ctr, s);
      const CsrView full = view(g->eff);  // (the locality path stays off here)
      for (uint64_t k = 0; k < K; ++k) {
        if (k) copy_chunk(k);
        TG_CUDA(cudaStreamWaitEvent(s, evs[k + 1], 0));
        tgb::orient_chunk(g->g, g->eff, cb[k], cb[k + 1], bigq.p, ctr.p, s);
        tgb::ready_chunks(g->eff, d_cb.p, (uint32_t)K, (uint32_t)k, cb[k], cb[k + 1], ready.p, s);
        const uint32_t sb = (uint32_t)vlo, se = std::min<uint32_t>(cb[k + 1], (uint32_t)vhi);
        tgb::select_ready(ready.p, sb, se, (uint32_t)k, ids.p, cnt.p, s);
        if (se > sb)
          tgb::intersect_list(full, ids.p, cnt.p, se - sb, full,
                              CountOut{d_total.p, nullptr, nullptr, nullptr, 0}, g->scr, s,
                              g->eff.data.n);
      }
      unsigned long long h = 0;
      download(&h, d_total.p, 1, s);
      sync(g);
      *total = h;
      cudaStream_t keep = cs;
      cs = nullptr;
      TG_CUDA(cudaStreamSynchronize(keep));
      TG_CUDA(cudaStreamDestroy(keep));
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}

tg_status tg_graph_from_rmat(int device, uint32_t scale, uint64_t edge_factor, double a, double b,
                             double c, uint64_t seed, tg_graph** out) {
  const uint64_t n = scale >= 1 && scale <= 31 ? 1ull << scale : 0;
  return graph_from_generator(device, n, out, [&](DBuf<uint32_t>& pairs, cudaStream_t s) {
    return tgb::gen_rmat_device(scale, edge_factor, a, b, c, seed, pairs, s);
  });
}

tg_status tg_graph_from_ws(int device, uint64_t n, uint64_t k, double beta, uint64_t seed,
                           tg_graph** out) {
  return graph_from_generator(device, n, out, [&](DBuf<uint32_t>& pairs, cudaStream_t s) {
    return tgb::gen_ws_device(n, k, beta, seed, pairs, s);
  });
}

tg_status tg_graph_from_csr(int device, uint64_t n, const uint64_t* offsets, const uint32_t* adj,
                            tg_graph** out) {
  return guard([&] {
    TG_REQUIRE(out != nullptr && offsets != nullptr, "null argument");
    TG_REQUIRE(n <= 0xFFFFFFFFull, "n must fit NodeId");
    tg_graph* g = new_graph(device);
    try {
      uint64_t m2 = 0;
      if (is_device_ptr(offsets)) {
        TG_CUDA(cudaMemcpy(&m2, offsets + n, 8, cudaMemcpyDeviceToHost));
      } else {
        m2 = offsets[n];
      }
      TG_REQUIRE(m2 % 2 == 0, "symmetric CSR must hold an even number of entries");
      TG_REQUIRE(adj != nullptr || m2 == 0, "null adjacency");
      g->g.n = n;
      g->g.m2 = m2;
      upload(g->g.off, offsets, n + 1, g->stream);
      upload(g->g.adj, adj, m2, g->stream);
      tgb::compute_degrees(g->g, g->stream);
      sync(g);
    } catch (...) {
      tg_graph_free(g);
      throw;
    }
    *out = g;
  });
}

tg_status tg_graph_free(tg_graph* g) {
  if (!g) return TG_OK;
  return guard([&] {
    cudaSetDevice(g->device);
    cudaStreamSynchronize(g->own);
    if (g->stream != g->own) cudaStreamSynchronize(g->stream);
    // release buffers on their streams before destroying the library's own
    g->for_each_buf([](auto& b) { b.release(); });
    cudaStreamSynchronize(g->own);
    if (g->stream != g->own) cudaStreamSynchronize(g->stream);
    cudaEventDestroy(g->ev0);
    cudaEventDestroy(g->ev1);
    cudaStreamDestroy(g->own);
    delete g;
  });
}

tg_status tg_graph_info(tg_graph* g, uint64_t* num_nodes, uint64_t* num_edges) {
  return guard([&] {
    TG_REQUIRE(g != nullptr, "null graph handle");
    if (num_nodes) *num_nodes = g->g.n;
    if (num_edges) *num_edges = g->g.m2 / 2;
  });
}

tg_status tg_graph_csr(tg_graph* g, uint64_t* offsets, uint32_t* adj) {
  return guard([&] {
    enter(g);
    download(offsets, g->g.off.p, g->g.n + 1, g->stream);
    download(adj, g->g.adj.p, g->g.m2, g->stream);
    sync(g);
  });
}

tg_status tg_set_stream(tg_graph* g, void* stream) {
  return guard([&] {
    enter(g);
    cudaStream_t ns = stream ? (cudaStream_t)stream : g->own;
    if (ns != g->stream) {
      sync(g);  // buffers allocated on the old stream stay valid (pool-backed)
      g->stream = ns;
      // DBuf frees are stream-ordered on the stream they were allocated on;
      // re-home them so later frees order after work on the new stream.
      g->for_each_buf([&](auto& b) { b.s = ns; });
    }
  });
}

tg_status tg_set_order(tg_graph* g, int32_t kind, uint64_t seed) {
  return guard([&] {
    enter(g);
    apply_order(g, kind, seed);
  });
}

tg_status tg_set_order_rank(tg_graph* g, const uint32_t* rank) {
  return guard([&] {
    enter(g);
    const uint64_t n = g->g.n;
    TG_REQUIRE(rank != nullptr || n == 0, "null rank");
    if (n && !is_device_ptr(rank)) {  // OrderRank::rank is a permutation (order.hpp:31-33)
      std::vector<uint8_t> seen(n, 0);
      for (uint64_t v = 0; v < n; ++v) {
        TG_REQUIRE(rank[v] < n && !seen[rank[v]], "OrderRank: rank must be a permutation of [0, n)");
        seen[rank[v]] = 1;
      }
    }
    upload(g->g.okey, rank, n, g->stream);
    g->g.order = TG_ORDER_RANK;
    g->g.order_seed = 0;
    g->have_eff = false;
    g->have_part = false;
    g->have_rk = false;
    g->rank_mode = -1;
    g->window_mode = -1;
    sync(g);  // the caller's rank buffer may die on return
  });
}

tg_status tg_coreness(tg_graph* g, uint64_t* core) {
  return guard([&] {
    enter(g);
    const uint64_t n = g->g.n;
    TG_REQUIRE(core != nullptr || n == 0, "null core output");
    if (!n) return;
    DBuf<uint32_t> d(n, g->stream);
    tgb::coreness_device(g->g, d.p, g->stream);
    std::vector<uint32_t> h(n);
    download(h.data(), d.p, n, g->stream);
    sync(g);
    for (uint64_t v = 0; v < n; ++v) core[v] = h[v];
  });
}

tg_status tg_compute_order(tg_graph* g, uint32_t* rank) {
  return guard([&] {
    enter(g);
    TG_REQUIRE(rank != nullptr || g->g.n == 0, "null rank output");
    DBuf<uint32_t> d(g->g.n ? g->g.n : 1, g->stream);
    tgb::order_rank(g->g, d.p, g->stream);
    download(rank, d.p, g->g.n, g->stream);
    sync(g);
  });
}

tg_status tg_effective_adjacency(tg_graph* g, uint64_t* offsets, uint32_t* eff) {
  return guard([&] {
    enter(g);
    ensure_eff(g);
    DevEff c;  // compact copy of the (gappy) resident orientation
    tgb::compact_eff(g->eff, c, g->stream);
    download(offsets, c.off.p, g->g.n + 1, g->stream);
    download(eff, c.data.p, c.entries, g->stream);
    sync(g);
  });
}

tg_status tg_ordering_cost(tg_graph* g, uint64_t* cost) {
  return guard([&] {
    enter(g);
    TG_REQUIRE(cost != nullptr, "null output");
    ensure_eff(g);
    *cost = tgb::ordering_cost_device(g->g, g->eff, g->stream);
  });
}

tg_status tg_node_costs(tg_graph* g, int32_t kind, uint64_t* f, uint64_t* prefix) {
  return guard([&] {
    enter(g);
    TG_REQUIRE(kind >= TG_COST_N && kind <= TG_COST_NOV, "unknown cost kind");
    ensure_eff(g);
    const uint64_t n = g->g.n;
    DBuf<uint64_t> df(n ? n : 1, g->stream), dp(n ? n : 1, g->stream);
    tgb::node_costs_device(g->g, g->eff, kind, df.p, dp.p, g->stream);
    download(f, df.p, n, g->stream);
    download(prefix, dp.p, n, g->stream);
    sync(g);
  });
}

tg_status tg_compute_boundaries(tg_graph* g, int32_t kind, uint64_t p, uint32_t* boundaries) {
  return guard([&] {
    enter(g);
    TG_REQUIRE(p >= 1, "compute_boundaries: p must be >= 1");  // partition.hpp:117
    TG_REQUIRE(boundaries != nullptr, "null output");
    ensure_eff(g);
    auto b = plan_for(g, kind, p, nullptr);
    std::memcpy(boundaries, b.data(), b.size() * 4);
  });
}

tg_status tg_count(tg_graph* g, uint64_t* total) {
  return guard([&] {
    enter(g);
    TG_REQUIRE(total != nullptr, "null output");
    *total = seq_count(g);
  });
}

tg_status tg_count_node_iterator_pp(tg_graph* g, int32_t use_intersection, uint64_t* total) {
  (void)use_intersection;  // same count either way (sequential.hpp:58-66)
  return guard([&] {
    enter(g);
    TG_REQUIRE(total != nullptr, "null output");
    *total = tgb::node_iterator_pp_device(g->g, g->stream);
  });
}

tg_status tg_run_engine(tg_graph* g, const tg_config* cfg, uint64_t* total, tg_rank_stats* per_rank,
                        uint32_t* boundaries_out, uint64_t* node_counts, uint32_t* triangles,
                        uint64_t capacity, uint64_t* num_triangles) {
  tg_status cap_status = TG_OK;
  tg_status st = guard([&] {
    enter(g);
    TG_REQUIRE(cfg != nullptr, "null config");
    cudaStream_t s = g->stream;
    const uint64_t n = g->g.n;
    DBuf<unsigned long long> tally, cursor;
    DBuf<uint32_t> tri;
    uint64_t cap = 0;
    if (cfg->track_nodes) {
      TG_REQUIRE(node_counts != nullptr || n == 0, "track_nodes needs node_counts");
      tally.alloc(n ? n : 1, s);
      tally.zero();
    }
    // listing straight into a caller's DEVICE buffer when it holds all T
    // triples (no staging copy: C4's 1.6e9 triangles are 19.7 GB)
    uint32_t* list_out = nullptr;
    bool direct = false;
    if (cfg->collect_triangles) {
      TG_REQUIRE(num_triangles != nullptr, "collect_triangles needs num_triangles");
      cap = seq_count(g);  // exact size first (ListSink holds T triples)
      direct = triangles != nullptr && is_device_ptr(triangles) && capacity >= cap;
      if (direct) {
        list_out = triangles;
      } else {
        tri.alloc(3 * (cap ? cap : 1), s);
        list_out = tri.p;
      }
      cursor.alloc(1, s);
      cursor.zero();
    }
    EngineResult R = run(g, *cfg, cfg->track_nodes ? tally.p : nullptr, list_out,
                         cfg->collect_triangles ? cursor.p : nullptr, cap);
    if (total) *total = R.total;
    if (per_rank) std::memcpy(per_rank, R.per_rank.data(), R.per_rank.size() * sizeof(tg_rank_stats));
    if (boundaries_out) std::memcpy(boundaries_out, R.b.data(), R.b.size() * 4);
    if (cfg->track_nodes) download(node_counts, (const uint64_t*)tally.p, n, s);
    if (cfg->collect_triangles) {
      *num_triangles = R.total;
      if (triangles && !direct) {
        const uint64_t words = 3 * std::min<uint64_t>(R.total, capacity);
        if (words)
          TG_CUDA(cudaMemcpyAsync(triangles, tri.p, words * 4,
                                  is_device_ptr(triangles) ? cudaMemcpyDeviceToDevice
                                                           : cudaMemcpyDeviceToHost, s));
      }
      if (capacity < R.total) cap_status = TG_ERR_CAPACITY;
    }
    sync(g);
  });
  if (st == TG_OK && cap_status != TG_OK) {
    t_last_error = "triangle capacity smaller than the triangle count";
    return cap_status;
  }
  return st;
}

tg_status tg_approx_count(tg_graph* g, uint64_t p, int32_t engine, double q, uint64_t seed,
                          const uint32_t* boundaries, int32_t cost, double* estimate) {
  return guard([&] {
    enter(g);
    TG_REQUIRE(estimate != nullptr, "null output");
    TG_REQUIRE(q > 0.0 && q <= 1.0, "sparsify: q must be in (0, 1]");  // sparsify.hpp:28-31
    tg_config c{};
    c.engine = engine;
    c.cost = cost;
    c.ranks = p;
    c.boundaries = boundaries;
    // engines.hpp:450-452: per-partition draws for AOP, one draw per edge otherwise
    c.sparsify = engine == TG_ENGINE_AOP ? TG_SPARSIFY_PER_PARTITION : TG_SPARSIFY_GLOBAL;
    c.sparsify_q = q;
    c.sparsify_seed = seed;
    c.order_set = 1;  // the default EngineConfig::order (engines.hpp:274)
    c.order = TG_ORDER_BY_DEGREE;
    EngineResult R = run(g, c, nullptr, nullptr, nullptr, 0);
    *estimate = (double)R.total / (q * q * q);
  });
}

tg_status tg_per_edge_triangle_counts(tg_graph* g, uint64_t* te) {
  return guard([&] {
    enter(g);
    cudaStream_t s = g->stream;
    ensure_eff(g);
    const uint64_t n = g->g.n, m = g->g.m2 / 2;
    TG_REQUIRE(te != nullptr || m == 0, "null output");
    if (!m) return;
    DBuf<uint64_t> up(n + 1, s);
    tgb::upper_offsets(g->g, up.p, s);
    DBuf<unsigned long long> dte(m, s);
    dte.zero();
    const uint64_t T = seq_count(g);
    const uint64_t cap = std::max<uint64_t>(1, std::min<uint64_t>(T, kListCap));
    DBuf<uint32_t> tri(3 * cap, s);
    list_in_pieces(g, 0, (uint32_t)n, tri, cap, [&](const uint32_t* t, uint64_t cnt) {
      tgb::bump_edges(g->g, up.p, t, cnt, dte.p, nullptr, s);
    });
    TG_CUDA(cudaMemcpyAsync(te, dte.p, m * 8, is_device_ptr(te) ? cudaMemcpyDeviceToDevice
                                                                : cudaMemcpyDeviceToHost, s));
    sync(g);
  });
}

tg_status tg_variance_report(tg_graph* g, const uint32_t* boundaries, uint64_t p, double q,
                             uint64_t* out3, double* var2) {
  return guard([&] {
    enter(g);
    TG_REQUIRE(boundaries && p >= 1 && out3 && var2, "invalid argument");
    cudaStream_t s = g->stream;
    apply_order(g, TG_ORDER_BY_DEGREE, 0);  // sparsify.hpp:123-124
    ensure_eff(g);
    const std::vector<uint32_t> b = plan_for(g, TG_COST_DPD, p, boundaries);
    const uint64_t n = g->g.n, m = g->g.m2 / 2;
    uint64_t T = 0, k = 0, kp = 0;
    if (m) {
      DBuf<uint64_t> up(n + 1, s);
      tgb::upper_offsets(g->g, up.p, s);
      DBuf<unsigned long long> tot(m, s), per(m, s);
      tot.zero();
      const uint64_t cap = std::max<uint64_t>(1, std::min<uint64_t>(seq_count(g), kListCap));
      DBuf<uint32_t> tri(3 * cap, s);
      // k' (sparsify.hpp:140-144): pairs of triangles on one edge whose
      // apexes share an owner = sum over ranks of the pairs among the
      // triangles with apex in that core
      for (uint64_t i = 0; i < p; ++i) {
        per.zero();
        list_in_pieces(g, b[i], b[i + 1], tri, cap, [&](const uint32_t* t, uint64_t cnt) {
          tgb::bump_edges(g->g, up.p, t, cnt, per.p, tot.p, s);
          T += cnt;
        });
        kp += tgb::sum_choose2(per.p, m, s);
      }
      k = tgb::sum_choose2(tot.p, m, s);
    }
    out3[0] = T;
    out3[1] = k;
    out3[2] = kp;
    const double q3 = q * q * q;  // sparsify.hpp:148-152
    var2[0] = (1.0 / q3 - 1.0) * (double)T + 2.0 * (double)k * (1.0 / q - 1.0);
    var2[1] = (1.0 / q3 - 1.0) * (double)T + 2.0 * (double)kp * (1.0 / q - 1.0);
  });
}

tg_status tg_clustering_coefficients(tg_graph* g, const tg_config* cfg, uint64_t* triangles_per_node,
                                     double* coefficient) {
  return guard([&] {
    enter(g);
    TG_REQUIRE(cfg != nullptr, "null config");
    cudaStream_t s = g->stream;
    const uint64_t n = g->g.n;
    DBuf<unsigned long long> tally(n ? n : 1, s);
    tally.zero();
    tg_config c = *cfg;
    c.track_nodes = 1;  // engines.hpp:423
    c.collect_triangles = 0;
    run(g, c, tally.p, nullptr, nullptr, 0);
    DBuf<double> cc(n ? n : 1, s);
    tgb::clustering_device(g->g, tally.p, cc.p, s);
    download(triangles_per_node, (const uint64_t*)tally.p, n, s);
    download(coefficient, cc.p, n, s);
    sync(g);
  });
}

tg_status tg_step_device(tg_graph* g, uint64_t* d_total) {
  return guard([&] {
    enter(g);
    TG_REQUIRE(d_total != nullptr, "null output");
    cudaStream_t s = g->stream;
    // orientation: effective_adjacency (effective.hpp:37-52), rebuilt
    orient(g);
    TG_CUDA(cudaMemsetAsync(d_total, 0, 8, s));
    const CsrView full = full_view(g);
    const uint32_t N = (uint32_t)g->g.n;
    const bool win = window_ready(g);
    timed_pass(g, [&] {
      if (win)
        window_rows(g, 0, N, (unsigned long long*)d_total);
      else
        tgb::intersect_rows(full, 0, N, full, 0, N,
                            CountOut{(unsigned long long*)d_total, nullptr, nullptr, nullptr, 0},
                            g->scr, s, g->eff.data.n, true, rank_view(g));
    });
  });
}

tg_status tg_orient_device(tg_graph* g) {
  return guard([&] {
    enter(g);
    orient(g);
  });
}

tg_status tg_count_device(tg_graph* g, uint64_t* d_total) {
  return guard([&] {
    enter(g);
    TG_REQUIRE(d_total != nullptr, "null output");
    cudaStream_t s = g->stream;
    ensure_eff(g);
    TG_CUDA(cudaMemsetAsync(d_total, 0, 8, s));
    const CsrView full = full_view(g);
    const uint32_t N = (uint32_t)g->g.n;
    const bool win = window_ready(g);
    timed_pass(g, [&] {
      if (win)
        window_rows(g, 0, N, (unsigned long long*)d_total);
      else
        tgb::intersect_rows(full, 0, N, full, 0, N,
                            CountOut{(unsigned long long*)d_total, nullptr, nullptr, nullptr, 0},
                            g->scr, s, g->eff.data.n, true, rank_view(g));
    });
  });
}

double tg_last_intersect_ms(tg_graph* g) {
  if (!g || !g->timed) return 0.0;
  float ms = 0.f;
  cudaSetDevice(g->device);
  if (cudaEventSynchronize(g->ev1) != cudaSuccess) return 0.0;
  if (cudaEventElapsedTime(&ms, g->ev0, g->ev1) != cudaSuccess) return 0.0;
  return ms;
}

tg_status tg_aop_rank_device(tg_graph* g, const uint32_t* boundaries, uint64_t p, uint64_t rank,
                             uint64_t* d_total) {
  return guard([&] {
    enter(g);
    TG_REQUIRE(boundaries && p >= 1 && rank < p && d_total, "invalid argument");
    TG_REQUIRE(boundaries[0] == 0 && boundaries[p] <= g->g.n, "invalid boundaries");
    ensure_eff(g);
    cudaStream_t s = g->stream;
    const CsrView full = full_view(g);
    const uint32_t N = (uint32_t)g->g.n;
    const uint32_t cb = boundaries[rank], ce = boundaries[rank + 1];
    const bool win = ce > cb && window_ready(g);
    timed_pass(g, [&] {
      if (win)
        window_rows(g, cb, ce, (unsigned long long*)d_total);
      else if (ce > cb)
        tgb::intersect_rows(full, cb, ce, full, 0, N,
                            CountOut{(unsigned long long*)d_total, nullptr, nullptr, nullptr, 0}, g->scr, s,
                          g->eff.data.n, true, rank_view(g));
    });
  });
}

tg_status tg_aop_rank_sinks_device(tg_graph* g, const uint32_t* boundaries, uint64_t p,
                                   uint64_t rank, uint64_t* d_total, uint64_t* d_tally,
                                   uint32_t* d_tri, uint64_t capacity, uint64_t* d_cursor) {
  return guard([&] {
    enter(g);
    TG_REQUIRE(boundaries && p >= 1 && rank < p && d_total, "invalid argument");
    TG_REQUIRE(boundaries[0] == 0 && boundaries[p] <= g->g.n, "invalid boundaries");
    TG_REQUIRE(!d_tri || d_cursor, "listing needs a cursor");
    ensure_eff(g);
    cudaStream_t s = g->stream;
    const CsrView full = view(g->eff);
    const uint32_t N = (uint32_t)g->g.n;
    const uint32_t cb = boundaries[rank], ce = boundaries[rank + 1];
    timed_pass(g, [&] {
      if (ce > cb)
        tgb::intersect_rows(full, cb, ce, full, 0, N,
                            CountOut{(unsigned long long*)d_total, (unsigned long long*)d_tally,
                                     d_tri, (unsigned long long*)d_cursor, capacity},
                            g->scr, s, g->eff.data.n, true, rank_view(g));
    });
  });
}

tg_status tg_cc_from_tally_device(tg_graph* g, const uint64_t* d_tally, double* d_cc) {
  return guard([&] {
    enter(g);
    TG_REQUIRE(d_tally && d_cc, "null argument");
    tgb::clustering_device(g->g, (const unsigned long long*)d_tally, d_cc, g->stream);
  });
}

tg_status tg_surrogate_pack_sizes(tg_graph* g, const uint32_t* boundaries, uint64_t p, uint64_t rank,
                                  uint64_t* msgs_per_dest, uint64_t* words_per_dest) {
  return guard([&] {
    enter(g);
    prepare_part(g, boundaries, p, rank);
    if (msgs_per_dest) std::memcpy(msgs_per_dest, g->pack.msgs_per_dest.data(), p * 8);
    if (words_per_dest) std::memcpy(words_per_dest, g->pack.words_per_dest.data(), p * 8);
  });
}

tg_status tg_surrogate_pack_device(tg_graph* g, const uint32_t* boundaries, uint64_t p, uint64_t rank,
                                   uint32_t* d_hdr, uint32_t* d_data) {
  return guard([&] {
    enter(g);
    prepare_part(g, boundaries, p, rank);
    g->pack.scatter(d_hdr, d_data, g->stream);
  });
}

tg_status tg_surrogate_count_device(tg_graph* g, const uint32_t* boundaries, uint64_t p, uint64_t rank,
                                    const uint32_t* d_hdr, uint64_t num_msgs, const uint32_t* d_data,
                                    uint64_t* d_total) {
  return guard([&] {
    enter(g);
    TG_REQUIRE(d_total != nullptr, "null output");
    prepare_part(g, boundaries, p, rank);
    cudaStream_t s = g->stream;
    const uint32_t cb = boundaries[rank], ce = boundaries[rank + 1];
    DBuf<uint64_t> moff;
    tgb::message_offsets(d_hdr, num_msgs, moff, s);
    const CsrView pv = view(g->part);
    const CountOut out{(unsigned long long*)d_total, nullptr, nullptr, nullptr, 0};
    timed_pass(g, [&] {
      if (ce > cb) {
        tgb::intersect_rows(pv, cb, ce, pv, cb, ce, out, g->scr, s, g->part.data.n, false);
        if (num_msgs) {
          tgb::MsgView mv{d_hdr, moff.p, d_data, num_msgs};
          tgb::intersect_msgs(mv, pv, cb, ce, out, g->scr, s, g->part.data.n);
        }
      }
    });
    sync(g);  // moff is freed on return
  });
}

// ---- EffectiveAdjacency as a value (effective.hpp:17-35) ------------------

struct tg_eff {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint64_t n = 0;
  tgb::DevEff e;
  tgb::IntersectScratch scr;
};

tg_status tg_eff_from_csr(int device, uint64_t n, const uint64_t* offsets, const uint32_t* entries,
                          tg_eff** out) {
  return guard([&] {
    TG_REQUIRE(out != nullptr && offsets != nullptr, "null argument");
    TG_REQUIRE(n <= 0xFFFFFFFFull, "n must fit NodeId");
    int count = 0;
    TG_CUDA(cudaGetDeviceCount(&count));
    TG_REQUIRE(device >= 0 && device < count, "invalid CUDA device ordinal");
    TG_CUDA(cudaSetDevice(device));
    uint64_t m = 0;
    const bool dev = is_device_ptr(offsets);
    if (dev) {
      TG_CUDA(cudaMemcpy(&m, offsets + n, 8, cudaMemcpyDeviceToHost));
    } else {
      m = offsets[n];
      TG_REQUIRE(offsets[0] == 0, "EffectiveAdjacency: offsets[0] must be 0");
      for (uint64_t v = 0; v < n; ++v) TG_REQUIRE(offsets[v] <= offsets[v + 1], "offsets must be sorted");
      TG_REQUIRE(entries != nullptr || m == 0, "null entries");
      if (m && !is_device_ptr(entries))
        for (uint64_t v = 0; v < n; ++v)
          for (uint64_t k = offsets[v]; k < offsets[v + 1]; ++k)
            TG_REQUIRE(entries[k] < n && (k == offsets[v] || entries[k - 1] < entries[k]),
                       "EffectiveAdjacency: lists must be ID-sorted, ids < n");
    }
    auto* h = new tg_eff;
    try {
      h->device = device;
      TG_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
      h->n = n;
      DevEff& e = h->e;
      e.rows = n;
      e.entries = m;
      e.base = 0;
      e.compact = true;
      upload(e.off, offsets, n + 1, h->stream);
      e.data.alloc(m + tgb::kQuadPad, h->stream);
      TG_CUDA(cudaMemsetAsync(e.data.p, 0, (m + tgb::kQuadPad) * 4, h->stream));
      if (m)
        TG_CUDA(cudaMemcpyAsync(e.data.p, entries, m * 4,
                                is_device_ptr(entries) ? cudaMemcpyDeviceToDevice
                                                       : cudaMemcpyHostToDevice, h->stream));
      tgb::eff_desc_from_off(e, h->stream);
      TG_CUDA(cudaStreamSynchronize(h->stream));
    } catch (...) {
      tg_eff_free(h);
      throw;
    }
    *out = h;
  });
}

tg_status tg_eff_free(tg_eff* h) {
  if (!h) return TG_OK;
  return guard([&] {
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    h->e.off.release();
    h->e.desc.release();
    h->e.data.release();
    h->scr.big.release();
    h->scr.big_count.release();
    if (h->stream) {
      cudaStreamSynchronize(h->stream);
      cudaStreamDestroy(h->stream);
    }
    delete h;
  });
}

tg_status tg_eff_count(tg_eff* h, uint64_t* total, uint64_t* tally, uint32_t* triples,
                       uint64_t capacity, int32_t raw, uint64_t* num_triangles) {
  tg_status cap_status = TG_OK;
  tg_status st = guard([&] {
    TG_REQUIRE(h != nullptr, "null EffectiveAdjacency handle");
    TG_CUDA(cudaSetDevice(h->device));
    cudaStream_t s = h->stream;
    const uint64_t n = h->n;
    const uint32_t N = (uint32_t)n;
    const CsrView v = view(h->e);
    DBuf<unsigned long long> ctr(1, s), tv, cursor;
    ctr.zero();
    unsigned long long T = 0;
    if (n)  // the count (and the listing's exact size)
      tgb::intersect_rows(v, 0, N, v, 0, N, CountOut{ctr.p, nullptr, nullptr, nullptr, 0}, h->scr, s,
                          h->e.data.n, true);
    download(&T, ctr.p, 1, s);
    TG_CUDA(cudaStreamSynchronize(s));
    if (total) *total = T;
    if (num_triangles) *num_triangles = T;
    if (!tally && !triples) return;
    DBuf<uint32_t> tri;
    uint32_t* list_out = nullptr;
    bool direct = false;
    if (triples) {
      direct = is_device_ptr(triples) && capacity >= T;
      if (direct) {
        list_out = triples;
      } else {
        tri.alloc(3 * (T ? T : 1), s);
        list_out = tri.p;
      }
      cursor.alloc(1, s);
      cursor.zero();
    }
    unsigned long long* tp = nullptr;
    if (tally) {
      if (is_device_ptr(tally)) {
        tp = (unsigned long long*)tally;
        TG_CUDA(cudaMemsetAsync(tp, 0, n * 8, s));
      } else {
        tv.alloc(n ? n : 1, s);
        tv.zero();
        tp = tv.p;
      }
    }
    ctr.zero();
    CountOut out{ctr.p, tp, list_out, triples ? cursor.p : nullptr, triples ? T : 0};
    out.raw = raw != 0;
    if (n) tgb::intersect_rows(v, 0, N, v, 0, N, out, h->scr, s, h->e.data.n, true);
    if (tally && tv.p) download(tally, (const uint64_t*)tv.p, n, s);
    if (triples && !direct) {
      const uint64_t words = 3 * std::min<uint64_t>(T, capacity);
      if (words)
        TG_CUDA(cudaMemcpyAsync(triples, tri.p, words * 4,
                                is_device_ptr(triples) ? cudaMemcpyDeviceToDevice
                                                       : cudaMemcpyDeviceToHost, s));
    }
    if (triples && capacity < T) cap_status = TG_ERR_CAPACITY;
    TG_CUDA(cudaStreamSynchronize(s));
  });
  if (st == TG_OK && cap_status != TG_OK) {
    t_last_error = "triangle capacity smaller than the triangle count";
    return cap_status;
  }
  return st;
}

}  // extern "C"
