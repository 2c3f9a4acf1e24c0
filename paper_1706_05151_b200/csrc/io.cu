// io.cu -- edge-list text on the device (io.hpp:18-64): parse_edge_list and
// write_edge_list as HBM-streaming byte kernels.
//
// parse (io.hpp:24-50), two passes of one CTA per 16 KB of text:
//   1. k_parse_chunks<false>: stage the chunk (+512 B halo) in bank-padded
//      shared memory; each thread parses the lines starting in its 64-byte
//      segment with istream semantics; edges per chunk, and an atomic
//      minimum of the first bad line's byte position;
//   CUB scan of the chunk counts (file order = chunk order, thread order);
//   2. k_parse_chunks<true>: the same parse, writing (u | v << 32) at the
//      chunk offset plus the thread's block prefix.
// On a bad line its number is 1 + the newlines before it (k_count_nl over the
// prefix), and the ParseError message is formatted on the host from that one
// line (same rules as the kernel).
//
// write (io.hpp:52-64): a warp per vertex sums the byte lengths of its
// "u v\n" lines (v > u), CUB scan to row offsets, then lanes write their
// lines at their warp-scan positions.
#include <cub/cub.cuh>

#include <cstring>
#include <string>
#include <vector>

#include "tg_internal.cuh"

namespace tgb {

namespace {

template <class F>
void cub_call(cudaStream_t s, F&& f) {
  size_t bytes = 0;
  TG_CUDA(f(nullptr, bytes));
  DBuf<unsigned char> tmp(bytes ? bytes : 1, s);
  TG_CUDA(f(tmp.p, bytes));
}

constexpr uint64_t kChunk = 1ull << 16;  // bytes per newline-count chunk

// 0x80 in each byte of w that equals '\n' (exact: the per-byte add of 0x7f
// to a value <= 0x7f never carries into the next byte)
__device__ __forceinline__ uint32_t nl_hi_bits(uint32_t w) {
  const uint32_t x = w ^ 0x0a0a0a0au;
  return ~(((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x | 0x7f7f7f7fu);
}

__device__ __forceinline__ unsigned nl_in_word(uint32_t w) { return __popc(nl_hi_bits(w)); }

// bit k set iff byte k of w is '\n'
__device__ __forceinline__ uint32_t nl_mask_word(uint32_t w) {
  const uint32_t h = nl_hi_bits(w);
  return ((h >> 7) & 1u) | ((h >> 14) & 2u) | ((h >> 21) & 4u) | ((h >> 28) & 8u);
}

// pass 1: newlines per chunk (text padded with zeros to a 16-byte multiple)
__global__ void __launch_bounds__(256)
k_count_nl(const uint4* __restrict__ text, uint64_t len, uint64_t* __restrict__ cnt) {
  const uint64_t c = blockIdx.x;
  const uint64_t b = c * kChunk, e = min(len, b + kChunk);
  unsigned s = 0;
  for (uint64_t q = b / 16 + threadIdx.x; q * 16 < e; q += blockDim.x) {
    const uint4 w = __ldcs(text + q);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t at = q * 16 + 4 * k;
      if (at + 4 <= e) s += nl_in_word(ws[k]);
      else if (at < e) s += __popc(nl_mask_word(ws[k]) & ((1u << (e - at)) - 1u));
    }
  }
  typedef cub::BlockReduce<unsigned, 256> R;
  __shared__ typename R::TempStorage tmp;
  const unsigned t = R(tmp).Sum(s);
  if (threadIdx.x == 0) cnt[c] = t;
}

// ---- chunk parser: a CTA per 16 KB of text, a thread per 64-byte segment.
// The chunk (+ a 512-byte halo for lines that cross its end) is staged in
// shared memory with one pad word per 16 words, so the 32 threads of a warp
// reading byte k of their own segments (stride 64 B) hit 32 distinct banks.
// Each thread parses the lines that START in its segment; bytes past the
// halo (a line longer than 512 B) come from global memory.
constexpr int kPT = 256;                          // threads per CTA
constexpr uint32_t kSeg = 64;                     // bytes per thread
constexpr uint32_t kPChunk = kPT * kSeg;          // 16 KB per CTA
constexpr uint32_t kHalo = 512;
constexpr uint32_t kStage = kPChunk + kHalo;      // staged bytes
constexpr uint32_t kStageWords = kStage / 4 + kStage / 64;  // + 1 pad word / 16

struct ChunkText {
  const uint32_t* sw;   // padded shared words
  const char* g;        // global text
  uint64_t base, len;   // chunk start, text length
  uint32_t staged;      // bytes of the chunk staged (from base)
  __device__ __forceinline__ int at(uint64_t i) const {  // -1 past the text
    if (i < staged) {
      const uint32_t w = (uint32_t)(i >> 2);
      return (sw[w + (w >> 4)] >> (8 * (i & 3))) & 0xff;
    }
    return base + i < len ? (int)(unsigned char)__ldg(g + base + i) : -1;
  }
};

// sequential reader over one line: one shared-memory word per 4 bytes
struct Cursor {
  const ChunkText& T;
  uint64_t i;
  uint32_t wi = 0xffffffffu, w = 0;
  __device__ __forceinline__ int peek() {
    if (i < T.staged) {
      const uint32_t q = (uint32_t)(i >> 2);
      if (q != wi) {
        wi = q;
        w = T.sw[q + (q >> 4)];
      }
      return (w >> (8 * (i & 3))) & 0xff;
    }
    return T.at(i);
  }
};

__device__ __forceinline__ bool is_space(int c) {  // std::isspace, "C" locale: \t \n \v \f \r ' '
  return (unsigned)c <= 32u && ((0x100003E00ull >> c) & 1ull);
}

// istream >> unsigned long long on one line (libstdc++ num_get): skip
// spaces, sign, digits; overflow fails; '-' negates modulo 2^64.  The line
// ends at '\n' or at the end of the text (c < 0).
__device__ __forceinline__ bool extract_ull(Cursor& R, uint64_t& out) {
  int c;
  while ((c = R.peek()) >= 0 && c != '\n' && is_space(c)) ++R.i;
  if (c < 0 || c == '\n') return false;
  bool neg = false;
  if (c == '+' || c == '-') {
    neg = c == '-';
    ++R.i;
    c = R.peek();
  }
  if (c < '0' || c > '9') return false;
  // the first 9 digits accumulate in 32 bits (no overflow possible); the
  // 64-bit multiply with the overflow test only runs for longer numbers
  uint32_t a32 = 0, nd = 0;
  uint64_t acc = 0;
  bool over = false;
  while ((c = R.peek()) >= '0' && c <= '9') {
    const uint32_t d = (uint32_t)(c - '0');
    if (nd < 9) {
      a32 = a32 * 10u + d;
    } else {
      if (nd == 9) acc = a32;
      const uint64_t lo = acc * 10, sum = lo + d;
      over |= (__umul64hi(acc, 10) != 0) | (sum < lo);  // acc * 10 + d >= 2^64
      acc = sum;
    }
    ++nd;
    ++R.i;
  }
  if (nd <= 9) acc = a32;
  if (over) return false;
  out = neg ? 0ull - acc : acc;
  return true;
}

// io.hpp:37-46 for the line starting at chunk offset p: 0 skip, 1 edge, 2 error
__device__ __forceinline__ int parse_line(const ChunkText& T, uint64_t p, uint64_t& pair) {
  Cursor R{T, p};
  int c;
  while ((c = R.peek()) == ' ' || c == '\t' || c == '\r') ++R.i;
  if (c < 0 || c == '\n' || c == '#') return 0;
  uint64_t u = 0, v = 0;
  if (!extract_ull(R, u) || !extract_ull(R, v)) return 2;
  while ((c = R.peek()) >= 0 && c != '\n' && is_space(c)) ++R.i;
  if (c >= 0 && c != '\n') return 2;
  pair = (uint64_t)(uint32_t)u | ((uint64_t)(uint32_t)v << 32);  // static_cast<NodeId>
  return 1;
}

// WRITE = false: edges of each thread's segment (tcnt) and the first bad
// line start (bad); WRITE = true: pairs from the thread's scanned offset.
template <bool WRITE>
__global__ void __launch_bounds__(kPT)
k_parse_chunks(const char* __restrict__ text, uint64_t len, uint32_t* __restrict__ tcnt,
               const uint64_t* __restrict__ toff, uint64_t* __restrict__ pairs,
               unsigned long long* __restrict__ bad) {
  __shared__ uint32_t sw[kStageWords];
  const uint64_t base = (uint64_t)blockIdx.x * kPChunk;
  const uint32_t staged = (uint32_t)min((uint64_t)kStage, len - base);
  const uint4* g4 = reinterpret_cast<const uint4*>(text + base);  // base % 16 == 0
  for (uint32_t j = threadIdx.x; j * 16 < staged; j += kPT) {
    const uint4 x = __ldcs(g4 + j);  // the text buffer is padded past len
    const uint32_t w = 4 * j, pw = w + (w >> 4);
    sw[pw] = x.x;
    sw[pw + 1] = x.y;
    sw[pw + 2] = x.z;
    sw[pw + 3] = x.w;
  }
  __syncthreads();
  const ChunkText T{sw, text, base, len, staged};
  const uint32_t chunk_len = (uint32_t)min((uint64_t)kPChunk, len - base);
  const uint32_t sb = threadIdx.x * kSeg, se = min(chunk_len, sb + kSeg);
  const uint64_t gt = (uint64_t)blockIdx.x * kPT + threadIdx.x;
  // line starts in the segment: p with byte(p-1) == '\n' (one bit each, from
  // the staged words), so every thread runs its ~4 line parses back to back
  // and the warp stays converged (a byte-by-byte walk diverges at every byte)
  const int prev = sb == 0 ? (base == 0 ? '\n' : (int)(unsigned char)__ldg(text + base - 1))
                           : (sb < chunk_len ? T.at(sb - 1) : 0);
  uint64_t starts = 0;
  if (sb < se) {
    uint64_t nl = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const uint32_t w = (sb >> 2) + q;
      nl |= (uint64_t)nl_mask_word(sw[w + (w >> 4)]) << (4 * q);
    }
    const uint32_t nb = se - sb;  // <= 64
    starts = (nl << 1) | (prev == '\n' ? 1ull : 0ull);
    if (nb < 64) starts &= (1ull << nb) - 1ull;
  }
  uint32_t edges = 0;
  uint64_t out = WRITE ? toff[gt] : 0;
  while (starts) {
    const uint32_t p = sb + (uint32_t)(__ffsll((long long)starts) - 1);
    starts &= starts - 1;
    uint64_t pr = 0;
    const int r = parse_line(T, p, pr);
    if (r == 1) {
      if (WRITE) pairs[out++] = pr;
      ++edges;
    } else if (r == 2 && !WRITE) {
      atomicMin(bad, (unsigned long long)(base + p));
    }
  }
  if (!WRITE) tcnt[gt] = edges;
}

// ---- write_edge_list

__device__ __forceinline__ unsigned ndigits(uint32_t x) {
  unsigned d = 1;
  while (x >= 10) {
    x /= 10;
    ++d;
  }
  return d;
}

// first index in adj[b, e) whose id exceeds u (lists are ID-sorted)
__device__ __forceinline__ uint64_t upper_start(const uint32_t* adj, uint64_t b, uint64_t e, uint32_t u) {
  while (b < e) {
    const uint64_t mid = b + (e - b) / 2;
    if (adj[mid] <= u) b = mid + 1;
    else e = mid;
  }
  return b;
}

__global__ void __launch_bounds__(256)
k_row_bytes(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj, uint64_t n,
            uint64_t* __restrict__ rb) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t u = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; u < n; u += warps) {
    const uint64_t e = off[u + 1];
    const uint64_t s = upper_start(adj, off[u], e, (uint32_t)u);
    const unsigned du = ndigits((uint32_t)u);
    uint64_t t = 0;
    for (uint64_t j = s + lane; j < e; j += 32) t += du + ndigits(adj[j]) + 2;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) rb[u] = t;
  }
}

// lines of 32 neighbours are formatted into a per-warp shared buffer, then
// the warp's contiguous output range is stored as aligned 32-bit words
constexpr uint32_t kLineMax = 22;  // "4294967295 4294967295\n"

__device__ __forceinline__ void put_digits(char* p, uint32_t x, unsigned d) {
  for (int k = (int)d - 1; k >= 0; --k) {
    p[k] = (char)('0' + x % 10);
    x /= 10;
  }
}

__global__ void __launch_bounds__(256)
k_write_rows(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj, uint64_t n,
             const uint64_t* __restrict__ roff, char* __restrict__ out) {
  __shared__ __align__(4) char sbuf[8][32 * kLineMax + 4];
  const unsigned lane = threadIdx.x & 31;
  char* B = sbuf[threadIdx.x >> 5];
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t u = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; u < n; u += warps) {
    const uint64_t e = off[u + 1];
    const uint64_t s = upper_start(adj, off[u], e, (uint32_t)u);
    const unsigned du = ndigits((uint32_t)u);
    uint64_t base = roff[u];
    for (uint64_t j0 = s; j0 < e; j0 += 32) {
      const uint64_t j = j0 + lane;
      const bool has = j < e;
      const uint32_t v = has ? adj[j] : 0;
      const unsigned dv = ndigits(v);
      const unsigned l = has ? du + dv + 2 : 0;
      unsigned incl = l;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned x = __shfl_up_sync(0xffffffffu, incl, o);
        if ((int)lane >= o) incl += x;
      }
      const unsigned tot = __shfl_sync(0xffffffffu, incl, 31);
      if (has) {
        char* p = B + incl - l;
        put_digits(p, (uint32_t)u, du);
        p[du] = ' ';
        put_digits(p + du + 1, v, dv);
        p[du + 1 + dv] = '\n';
      }
      __syncwarp();
      // store B[0, tot) at out[base, base + tot): unaligned head, words, tail
      const unsigned head = min(tot, (unsigned)((4 - (base & 3)) & 3));
      if (lane < head) out[base + lane] = B[lane];
      const unsigned nw = (tot - head) >> 2;
      uint32_t* ow = reinterpret_cast<uint32_t*>(out + base + head);
      for (unsigned i = lane; i < nw; i += 32) {
        const char* q = B + head + 4 * i;
        ow[i] = (uint32_t)(unsigned char)q[0] | ((uint32_t)(unsigned char)q[1] << 8) |
                ((uint32_t)(unsigned char)q[2] << 16) | ((uint32_t)(unsigned char)q[3] << 24);
      }
      const unsigned t0 = head + 4 * nw;
      if (lane < tot - t0) out[base + t0 + lane] = B[t0 + lane];
      __syncwarp();
      base += tot;
    }
  }
}

struct Widen {
  __host__ __device__ __forceinline__ uint64_t operator()(uint32_t x) const { return x; }
};

bool host_space(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// The ParseError message of one bad line (io.hpp:42-45), host side.
std::string line_error(const std::string& line) {
  size_t i = 0;
  auto ull = [&]() {
    while (i < line.size() && host_space((unsigned char)line[i])) ++i;
    if (i >= line.size()) return false;
    if (line[i] == '+' || line[i] == '-') ++i;
    if (i >= line.size() || line[i] < '0' || line[i] > '9') return false;
    uint64_t acc = 0;
    bool over = false;
    while (i < line.size() && line[i] >= '0' && line[i] <= '9') {
      const uint64_t d = (uint64_t)(line[i] - '0');
      if (acc > (~0ull - d) / 10) over = true;
      else acc = acc * 10 + d;
      ++i;
    }
    return !over;
  };
  if (!ull() || !ull()) return "expected two integer tokens";
  while (i < line.size() && host_space((unsigned char)line[i])) ++i;
  size_t j = i;
  while (j < line.size() && !host_space((unsigned char)line[j])) ++j;
  return "trailing token '" + line.substr(i, j - i) + "'";
}

}  // namespace

uint64_t parse_edge_list_device(const char* d_text, uint64_t len, DBuf<uint32_t>& pairs,
                                cudaStream_t s, uint64_t* err_line, std::string* err_msg) {
  *err_line = 0;
  if (!len) {
    pairs.alloc(2, s);
    return 0;
  }
  const uint64_t chunks = (len + kPChunk - 1) / kPChunk;
  TG_REQUIRE(chunks < (1ull << 31), "text too large");
  const uint64_t nt = chunks * kPT;  // one count per 64-byte segment
  DBuf<uint32_t> tcnt(nt, s);
  DBuf<uint64_t> toff(nt + 1, s);
  DBuf<unsigned long long> bad(1, s);
  TG_CUDA(cudaMemsetAsync(bad.p, 0xff, 8, s));
  k_parse_chunks<false><<<(unsigned)chunks, kPT, 0, s>>>(d_text, len, tcnt.p, nullptr, nullptr, bad.p);
  TG_CHECK_LAUNCH();
  TG_CUDA(cudaMemsetAsync(toff.p, 0, 8, s));
  // 64-bit accumulation (a text may hold more than 2^32 lines)
  cub::TransformInputIterator<uint64_t, Widen, const uint32_t*> wide(tcnt.p, Widen());
  cub_call(s, [&](void* t, size_t& b) {
    return cub::DeviceScan::InclusiveSum(t, b, wide, toff.p + 1, (int64_t)nt, s);
  });
  uint64_t E = 0;
  unsigned long long h_bad = 0;
  TG_CUDA(cudaMemcpyAsync(&E, toff.p + nt, 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaMemcpyAsync(&h_bad, bad.p, 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  g_launches += 3;
  if (h_bad != ~0ull) {
    // line number: 1 + newlines in [0, bad); the line: [bad, next '\n')
    uint64_t nl = 0;
    if (h_bad) {
      const uint64_t nc = (h_bad + kChunk - 1) / kChunk;
      DBuf<uint64_t> c2(nc, s), tot(1, s);
      k_count_nl<<<(unsigned)nc, 256, 0, s>>>((const uint4*)d_text, h_bad, c2.p);
      TG_CHECK_LAUNCH();
      cub_call(s, [&](void* t, size_t& b) {
        return cub::DeviceReduce::Sum(t, b, c2.p, tot.p, (int64_t)nc, s);
      });
      TG_CUDA(cudaMemcpyAsync(&nl, tot.p, 8, cudaMemcpyDeviceToHost, s));
      TG_CUDA(cudaStreamSynchronize(s));
      g_launches += 2;
    }
    std::string line;
    for (uint64_t p = h_bad; p < len;) {  // the bad line, 4 KB at a time
      char buf[4096];
      const uint64_t k = std::min<uint64_t>(sizeof(buf), len - p);
      TG_CUDA(cudaMemcpy(buf, d_text + p, k, cudaMemcpyDeviceToHost));
      const char* e = static_cast<const char*>(memchr(buf, '\n', k));
      line.append(buf, e ? (size_t)(e - buf) : k);
      if (e) break;
      p += k;
    }
    *err_line = nl + 1;
    *err_msg = "line " + std::to_string(nl + 1) + ": " + line_error(line);
    return 0;
  }
  pairs.alloc(2 * (E ? E : 1), s);
  if (E) {
    k_parse_chunks<true><<<(unsigned)chunks, kPT, 0, s>>>(d_text, len, nullptr, toff.p,
                                                          (uint64_t*)pairs.p, nullptr);
    TG_CHECK_LAUNCH();
    ++g_launches;
  }
  return E;
}

uint64_t write_edge_list_device(const DevGraph& g, DBuf<char>& out, cudaStream_t s) {
  const uint64_t n = g.n;
  if (!n || !g.m2) {
    out.alloc(1, s);
    return 0;
  }
  DBuf<uint64_t> rb(n, s), roff(n + 1, s);
  const unsigned grid = grid_for(n * 32, 256, 148u * 32u);
  k_row_bytes<<<grid, 256, 0, s>>>(g.off.p, g.adj.p, n, rb.p);
  TG_CHECK_LAUNCH();
  TG_CUDA(cudaMemsetAsync(roff.p, 0, 8, s));
  cub_call(s, [&](void* t, size_t& b) {
    return cub::DeviceScan::InclusiveSum(t, b, rb.p, roff.p + 1, (int64_t)n, s);
  });
  uint64_t total = 0;
  TG_CUDA(cudaMemcpyAsync(&total, roff.p + n, 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  out.alloc(total ? total : 1, s);
  k_write_rows<<<grid, 256, 0, s>>>(g.off.p, g.adj.p, n, roff.p, out.p);
  TG_CHECK_LAUNCH();
  g_launches += 4;
  return total;
}

}  // namespace tgb
