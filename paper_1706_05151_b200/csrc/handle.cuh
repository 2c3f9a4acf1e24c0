// handle.cuh -- the tg_graph handle behind the C ABI and the internal
// helpers the engines share (engine.cu, comm.cu).
#pragma once

#include <string>
#include <vector>

#include "exchange.cuh"
#include "tg_internal.cuh"

struct tg_graph {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  tgb::DevGraph g;
  bool have_eff = false;
  tgb::DevEff eff;
  uint64_t eff_gen = 0;          // bumped by every (re)orientation
  // bitmap CTA path (ctab.cuh): order rank + rank-labelled lists
  int rank_mode = -1;            // -1 undecided, 0 off, 1 on (per order)
  bool have_rk = false;
  uint64_t rdata_gen = ~0ull;    // rdata matches eff iff rdata_gen == eff_gen
  tgb::DBuf<uint32_t> rk, rdata;
  // slab layout of the oriented lists: -1 undecided, 0 off, 1 on (per order;
  // decided under slab_for = the g_slab_mode in force)
  int slab_mode = -1, slab_for = 0;
  int comm_slab = -1;  // the same choice for the gathered lists of tg_aop_step_comm
  // window encoding (window.cu): -1 undecided, 0 off, 1 on (per order)
  int window_mode = -1;
  uint64_t window_far = 0;
  uint64_t window_gen = ~0ull;   // win matches eff iff window_gen == eff_gen
  tgb::WindowEff win;
  tgb::DBuf<uint32_t> wdefer;
  tgb::IntersectScratch scr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  bool timed = false;
  // rank-local caches (multi-process surrogate)
  bool have_part = false;
  uint64_t part_rank = 0;
  std::vector<uint32_t> part_b;
  tgb::DevEff part;
  tgb::SurrogatePack pack;
  // rank-local input (tg_graph_from_rows): only rows [row_lo, row_hi) of
  // the symmetric CSR are resident, with the global degree vector; oriented
  // through the tg_*_comm entry points only
  bool partial = false;
  uint32_t row_lo = 0, row_hi = 0;

  // every device buffer the handle owns (release before the stream dies;
  // re-home stream-ordered frees when the caller switches streams)
  template <class F>
  void for_each_buf(F&& f) {
    f(g.off); f(g.adj); f(g.deg); f(g.dcode); f(g.dcode4); f(g.okey);
    f(eff.off); f(eff.data); f(eff.desc); f(rk); f(rdata);
    f(win.rec); f(win.far); f(win.ctr); f(wdefer);
    f(scr.big); f(scr.big_count);
    f(part.off); f(part.data); f(part.desc);
    f(pack.desc); f(pack.doff);
  }
};

void tgb_set_error(const std::string& msg);

namespace tgh {
tg_graph* new_graph(int device);
void enter(tg_graph* g);
void sync(tg_graph* g);
void ensure_eff(tg_graph* g);
tgb::CsrView view(const tgb::DevEff& e);
tgb::CsrView full_view(tg_graph* g);
tgb::RankView rank_view(tg_graph* g);
bool window_ready(tg_graph* g);
void window_rows(tg_graph* g, uint32_t vlo, uint32_t vhi, unsigned long long* d_total);
std::vector<uint32_t> plan_for(tg_graph* g, int cost, uint64_t p, const uint32_t* override_b);
bool is_device_ptr(const void* p);
// install a complete oriented CSR (compact) as g's current orientation
void install_eff(tg_graph* g, tgb::DevEff&& e);
}  // namespace tgh
