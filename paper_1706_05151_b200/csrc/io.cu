// io.cu -- edge-list text on the device (io.hpp:18-64): parse_edge_list and
// write_edge_list as HBM-streaming byte kernels.
//
// parse (io.hpp:24-50), three passes over the text:
//   1. k_count_nl   : '\n' count per 64 KB chunk (16-byte loads, popc of a
//                     byte-compare mask)            -> CUB scan per chunk
//   2. k_line_ends  : positions of the newlines, ballot-compacted in file order
//   3. k_parse_lines: one thread per line (consecutive lines in consecutive
//                     lanes, so a warp reads ~0.5 KB of contiguous text),
//                     bytes read through an aligned 32-bit window; writes the
//                     pair (u | v << 32) and a keep flag; a malformed line
//                     lowers an atomic minimum of the failing line index.
//   CUB DeviceSelect::Flagged drops blank/comment lines (file order kept).
// Line i = bytes (end[i-1], end[i]) with end[-1] = -1, so its 1-based line
// number is i + 1 exactly as the reference counts (io.hpp:30-35).  The
// ParseError message of the first bad line is formatted on the host from
// that one line (same rules as the kernel).
//
// write (io.hpp:52-64): a warp per vertex sums the byte lengths of its
// "u v\n" lines (v > u), CUB scan to row offsets, then lanes write their
// lines at their warp-scan positions.
#include <cub/cub.cuh>

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

// pass 2: newline positions, in file order within each chunk
__global__ void __launch_bounds__(256)
k_line_ends(const uint32_t* __restrict__ text, uint64_t len, const uint64_t* __restrict__ base,
            uint64_t* __restrict__ ends) {
  const uint64_t c = blockIdx.x;
  const uint64_t b = c * kChunk, e = min(len, b + kChunk);
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __shared__ unsigned s_warp[8];
  __shared__ uint64_t s_base;
  if (threadIdx.x == 0) s_base = base[c];
  __syncthreads();
  // the block walks the chunk in 1 KB steps (one 4-byte word per thread)
  for (uint64_t p0 = b; p0 < e; p0 += 1024) {
    const uint64_t at = p0 + 4 * threadIdx.x;
    uint32_t m = 0;
    if (at < e) {
      m = nl_mask_word(__ldcs(text + at / 4));
      if (at + 4 > e) m &= (1u << (e - at)) - 1u;
    }
    const unsigned k = __popc(m);
    // block exclusive scan of k in thread order
    unsigned incl = k;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned x = __shfl_up_sync(0xffffffffu, incl, o);
      if ((int)lane >= o) incl += x;
    }
    if (lane == 31) s_warp[w] = incl;
    __syncthreads();
    unsigned wbase = 0, tot = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      wbase += (i < (int)w) ? s_warp[i] : 0u;
      tot += s_warp[i];
    }
    unsigned pos = wbase + incl - k;
    const uint64_t ob = s_base;
    while (m) {
      const int bit = __ffs(m) - 1;
      ends[ob + pos++] = at + bit;
      m &= m - 1;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base = ob + tot;
    __syncthreads();
  }
}

struct ByteWin {
  const uint32_t* t;
  uint64_t wi = ~0ull;
  uint32_t w = 0;
  __device__ __forceinline__ unsigned at(uint64_t p) {
    const uint64_t q = p >> 2;
    if (q != wi) {
      wi = q;
      w = __ldg(t + q);
    }
    return (w >> (8 * (p & 3))) & 0xffu;
  }
};

__device__ __forceinline__ bool is_space(unsigned c) {  // std::isspace, "C" locale
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// istream >> unsigned long long (libstdc++ num_get): skip spaces, sign,
// digits; overflow fails; '-' negates modulo 2^64
__device__ __forceinline__ bool extract_ull(ByteWin& bw, uint64_t& i, uint64_t e, uint64_t& out) {
  unsigned c = 0;
  while (i < e && is_space(c = bw.at(i))) ++i;
  if (i >= e) return false;
  bool neg = false;
  if (c == '+' || c == '-') {
    neg = c == '-';
    if (++i >= e) return false;
    c = bw.at(i);
  }
  if (c < '0' || c > '9') return false;
  uint64_t acc = 0;
  bool over = false;
  while (i < e && (c = bw.at(i)) >= '0' && c <= '9') {
    const uint64_t d = c - '0';
    if (acc > (~0ull - d) / 10) over = true;
    else acc = acc * 10 + d;
    ++i;
  }
  if (over) return false;
  out = neg ? 0ull - acc : acc;
  return true;
}

// pass 3: one thread per line
__global__ void __launch_bounds__(256)
k_parse_lines(const uint32_t* __restrict__ text, uint64_t len, const uint64_t* __restrict__ ends,
              uint64_t nlines, uint64_t* __restrict__ val, uint8_t* __restrict__ keep,
              unsigned long long* __restrict__ bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nlines;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = i ? ends[i - 1] + 1 : 0;
    const uint64_t e = ends[i];  // (the last line ends at len)
    ByteWin bw{text};
    uint64_t first = b;
    unsigned c = 0;
    while (first < e && ((c = bw.at(first)) == ' ' || c == '\t' || c == '\r')) ++first;
    uint8_t k = 0;
    uint64_t out = 0;
    if (first < e && c != '#') {
      uint64_t p = b, u = 0, v = 0;
      bool ok = extract_ull(bw, p, e, u) && extract_ull(bw, p, e, v);
      if (ok) {
        while (p < e && is_space(bw.at(p))) ++p;
        ok = p == e;
      }
      if (ok) {
        out = (uint64_t)(uint32_t)u | ((uint64_t)(uint32_t)v << 32);  // static_cast<NodeId>
        k = 1;
      } else {
        atomicMin(bad, (unsigned long long)i);
      }
    }
    val[i] = out;
    keep[i] = k;
  }
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

__global__ void __launch_bounds__(256)
k_write_rows(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj, uint64_t n,
             const uint64_t* __restrict__ roff, char* __restrict__ out) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t u = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; u < n; u += warps) {
    const uint64_t e = off[u + 1];
    const uint64_t s = upper_start(adj, off[u], e, (uint32_t)u);
    const unsigned du = ndigits((uint32_t)u);
    char ud[10];
    {
      uint32_t x = (uint32_t)u;
      for (int k = (int)du - 1; k >= 0; --k) {
        ud[k] = (char)('0' + x % 10);
        x /= 10;
      }
    }
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
      if (has) {
        char* p = out + base + incl - l;
        for (unsigned k = 0; k < du; ++k) p[k] = ud[k];
        p[du] = ' ';
        uint32_t x = v;
        for (int k = (int)dv - 1; k >= 0; --k) {
          p[du + 1 + k] = (char)('0' + x % 10);
          x /= 10;
        }
        p[du + 1 + dv] = '\n';
      }
      base += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
}

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
  const uint64_t chunks = (len + kChunk - 1) / kChunk;
  if (!len) {
    pairs.alloc(2, s);
    return 0;
  }
  DBuf<uint64_t> cnt(chunks, s), base(chunks + 1, s);
  k_count_nl<<<(unsigned)chunks, 256, 0, s>>>((const uint4*)d_text, len, cnt.p);
  TG_CHECK_LAUNCH();
  TG_CUDA(cudaMemsetAsync(base.p, 0, 8, s));
  cub_call(s, [&](void* t, size_t& b) {
    return cub::DeviceScan::InclusiveSum(t, b, cnt.p, base.p + 1, (int64_t)chunks, s);
  });
  uint64_t nl = 0;
  char last = 0;
  TG_CUDA(cudaMemcpyAsync(&nl, base.p + chunks, 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaMemcpyAsync(&last, d_text + len - 1, 1, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  // io.hpp:30-35: a final line without '\n' still counts
  const uint64_t nlines = nl + (last != '\n' ? 1 : 0);
  DBuf<uint64_t> ends(nlines ? nlines : 1, s);
  k_line_ends<<<(unsigned)chunks, 256, 0, s>>>((const uint32_t*)d_text, len, base.p, ends.p);
  TG_CHECK_LAUNCH();
  if (nlines > nl) TG_CUDA(cudaMemcpyAsync(ends.p + nl, &len, 8, cudaMemcpyHostToDevice, s));
  DBuf<uint64_t> val(nlines ? nlines : 1, s);
  DBuf<uint8_t> keep(nlines ? nlines : 1, s);
  DBuf<unsigned long long> bad(1, s);
  TG_CUDA(cudaMemsetAsync(bad.p, 0xff, 8, s));
  if (nlines) {
    k_parse_lines<<<grid_for(nlines, 256, 148u * 16u), 256, 0, s>>>(
        (const uint32_t*)d_text, len, ends.p, nlines, val.p, keep.p, bad.p);
    TG_CHECK_LAUNCH();
  }
  g_launches += 5;
  unsigned long long h_bad = 0;
  TG_CUDA(cudaMemcpyAsync(&h_bad, bad.p, 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  if (h_bad != ~0ull) {
    uint64_t be[2] = {0, 0};
    if (h_bad) TG_CUDA(cudaMemcpyAsync(&be[0], ends.p + h_bad - 1, 8, cudaMemcpyDeviceToHost, s));
    TG_CUDA(cudaMemcpyAsync(&be[1], ends.p + h_bad, 8, cudaMemcpyDeviceToHost, s));
    TG_CUDA(cudaStreamSynchronize(s));
    const uint64_t b = h_bad ? be[0] + 1 : 0;
    std::string line(be[1] - b, '\0');
    if (!line.empty())
      TG_CUDA(cudaMemcpy(&line[0], d_text + b, line.size(), cudaMemcpyDeviceToHost));
    *err_line = h_bad + 1;
    *err_msg = "line " + std::to_string(h_bad + 1) + ": " + line_error(line);
    return 0;
  }
  // drop blank / comment lines, keeping file order
  pairs.alloc(2 * (nlines ? nlines : 1), s);
  DBuf<int64_t> nsel(1, s);
  cub_call(s, [&](void* t, size_t& b) {
    return cub::DeviceSelect::Flagged(t, b, val.p, keep.p, (uint64_t*)pairs.p, nsel.p,
                                      (int64_t)nlines, s);
  });
  ++g_launches;
  int64_t E = 0;
  TG_CUDA(cudaMemcpyAsync(&E, nsel.p, 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  return (uint64_t)E;
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
