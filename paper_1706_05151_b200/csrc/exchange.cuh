// exchange.cuh -- partition-side helpers (see exchange.cu).
#pragma once

#include "tg_internal.cuh"

namespace tgb {

// Surrogate send buffers of one rank (engines.hpp:173-187): messages sorted
// by destination; message k = header (v, h_v) + N_v at data offset doff[k].
struct SurrogatePack {
  CsrView part{};
  uint64_t M = 0;                      // messages
  DBuf<uint64_t> desc;                 // (dest << 32 | v), dest-major, v ascending
  DBuf<uint64_t> doff;                 // M+1 data offsets
  std::vector<uint64_t> msgs_per_dest;   // p
  std::vector<uint64_t> words_per_dest;  // p
  void build(CsrView part, uint32_t cb, uint32_t ce, const std::vector<uint32_t>& b,
             uint32_t self, cudaStream_t s);
  void scatter(uint32_t* d_hdr, uint32_t* d_data, cudaStream_t s) const;
};

// moff[k] = data offset of received message k (exclusive scan of lengths).
void message_offsets(const uint32_t* d_hdr, uint64_t M, DBuf<uint64_t>& moff, cudaStream_t s);

// build_overlap_partition(...).stored_entries() (partition.hpp:163-168).
uint64_t overlap_stored_entries(CsrView eff, uint64_t n, uint32_t cb, uint32_t ce, cudaStream_t s);

// ANOP-direct message counts per rank: req[i] requests sent by i, rep[j]
// replies sent by j (engines.hpp:97-111).
void direct_messages(CsrView eff, uint64_t n, const std::vector<uint32_t>& b,
                     std::vector<uint64_t>& req, std::vector<uint64_t>& rep, cudaStream_t s);

}  // namespace tgb
