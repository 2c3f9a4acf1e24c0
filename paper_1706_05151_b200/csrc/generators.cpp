// generators.cpp -- seeded synthetic inputs for BASELINE.json's five configs
// (host harness; not on the measured path).
//
//  tg_gen_pa   -- io.hpp:129-162 gen_pa, bit-identical edge stream
//                 (std::mt19937_64, rng() % endpoints.size(), repeat until
//                 distinct).  The endpoint list is never materialised: slot
//                 2e of a non-clique edge e is its new vertex (known from e),
//                 slot 2e+1 its target, so only targets are stored and looked
//                 up (with prefetch over a window of pre-drawn numbers).
//  tg_gen_gnp  -- io.hpp:85-123 gen_gnp, bit-identical (geometric skipping).
//  tg_gen_gnm  -- G(n, m): m distinct non-loop pairs, uniform (config 1).
//  tg_gen_rmat -- R-MAT (config 3); chunked xoshiro streams, thread-count
//                 independent output.
//  tg_gen_ws   -- Watts-Strogatz ring + rewiring (config 4); chunked streams.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "../../include/trigraph_b200.h"

void tgb_set_error(const std::string& msg);  // engine.cu
namespace {

uint32_t* alloc_pairs(uint64_t E) {
  auto* p = static_cast<uint32_t*>(std::malloc((E ? E : 1) * 2 * sizeof(uint32_t)));
  if (!p) throw std::bad_alloc();
  return p;
}

template <class F>
tg_status guard(F&& f) {
  try {
    f();
    return TG_OK;
  } catch (const std::invalid_argument& e) {
    tgb_set_error(e.what());
    return TG_ERR_INVALID_ARGUMENT;
  } catch (const std::bad_alloc&) {
    tgb_set_error("host allocation failed");
    return TG_ERR_OOM;
  } catch (const std::exception& e) {
    tgb_set_error(e.what());
    return TG_ERR_INTERNAL;
  }
}

uint64_t splitmix64(uint64_t& x) {
  uint64_t z = (x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct Xoshiro {
  uint64_t s[4];
  explicit Xoshiro(uint64_t seed) {
    uint64_t x = seed;
    for (auto& v : s) v = splitmix64(x);
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    const uint64_t r = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3];
    s[2] ^= t; s[3] = rotl(s[3], 45);
    return r;
  }
  double unit() { return (double)(next() >> 11) * 0x1.0p-53; }
};

unsigned hw_threads() {
  unsigned t = std::thread::hardware_concurrency();
  return t ? t : 1;
}

template <class F>
void parallel_chunks(uint64_t chunks, F&& f) {
  unsigned T = std::min<uint64_t>(hw_threads(), chunks ? chunks : 1);
  std::vector<std::thread> pool;
  std::atomic<uint64_t> next{0};
  for (unsigned t = 0; t < T; ++t)
    pool.emplace_back([&] {
      for (;;) {
        uint64_t c = next.fetch_add(1);
        if (c >= chunks) break;
        f(c);
      }
    });
  for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

void tg_free_host(void* p) { std::free(p); }

tg_status tg_gen_pa(uint64_t n, uint64_t d, uint64_t seed, uint32_t** pairs, uint64_t* num_pairs) {
  return guard([&] {
    if (d < 2 || d % 2 != 0 || n <= d / 2)  // io.hpp:130-131
      throw std::invalid_argument("gen_pa: need d even, d >= 2, n > d/2");
    const uint64_t half = d / 2, clique = half + 1;
    const uint64_t cpairs = clique * (clique - 1) / 2;
    const uint64_t E = cpairs + (n - clique) * half;
    uint32_t* out = alloc_pairs(E);
    std::vector<uint32_t> cl;  // clique endpoint slots (io.hpp:140-145)
    cl.reserve(2 * cpairs);
    uint64_t w = 0;
    for (uint32_t u = 0; u < clique; ++u)
      for (uint32_t v = u + 1; v < clique; ++v) {
        out[2 * w] = u;
        out[2 * w + 1] = v;
        ++w;
        cl.push_back(u);
        cl.push_back(v);
      }
    const uint64_t C0 = 2 * cpairs;
    std::vector<uint32_t> tgt((n - clique) * half);  // targets of non-clique edges
    std::mt19937_64 rng(seed);
    constexpr int kWin = 128;
    uint64_t buf[kWin];
    uint64_t head = 0, tail = 0;  // buf holds draws [head, tail)
    auto refill = [&] {
      while (tail - head < (uint64_t)kWin) {
        buf[tail % kWin] = rng();
        ++tail;
      }
    };
    auto slot = [&](uint64_t r) -> uint32_t {
      if (r < C0) return cl[r];
      uint64_t e = (r - C0) >> 1;
      if (((r - C0) & 1) == 0) return (uint32_t)(clique + e / half);
      return tgt[e];
    };
    uint32_t picked[64];
    std::vector<uint32_t> pickv;
    uint32_t* pk = half <= 64 ? picked : (pickv.resize(half), pickv.data());
    uint64_t ne = 0;  // non-clique edges so far
    for (uint64_t v = clique; v < n; ++v) {
      const uint64_t size = C0 + 2 * ne;  // endpoints.size() (io.hpp:151)
      refill();
      // prefetch the next vertices' likely target slots
      {
        const uint64_t size2 = size + 2 * half;
        for (uint64_t q = head + half; q < tail && q < head + 3 * half; ++q) {
          uint64_t r = buf[q % kWin] % (q < head + 2 * half ? size2 : size2 + 2 * half);
          if (r >= C0 && ((r - C0) & 1)) __builtin_prefetch(&tgt[(r - C0) >> 1]);
        }
      }
      uint64_t c = 0;
      while (c < half) {  // io.hpp:150-154
        if (head == tail) refill();
        uint64_t x = buf[head % kWin];
        ++head;
        uint32_t t = slot(x % size);
        bool dup = false;
        for (uint64_t i = 0; i < c; ++i)
          if (pk[i] == t) { dup = true; break; }
        if (!dup) pk[c++] = t;
      }
      for (uint64_t i = 0; i < half; ++i) {  // io.hpp:155-159
        out[2 * w] = (uint32_t)v;
        out[2 * w + 1] = pk[i];
        ++w;
        tgt[ne++] = pk[i];
      }
    }
    *pairs = out;
    *num_pairs = E;
  });
}

tg_status tg_gen_gnp(uint64_t n, double d, uint64_t seed, uint32_t** pairs, uint64_t* num_pairs) {
  return guard([&] {
    std::vector<uint32_t> e;
    if (n == 0) {
      *pairs = alloc_pairs(0);
      *num_pairs = 0;
      return;
    }
    if (d < 0 || (n > 1 && d > (double)(n - 1)) || (n == 1 && d > 0))
      throw std::invalid_argument("gen_gnp: need 0 <= d <= n-1");  // io.hpp:87-88
    const double q = (n > 1) ? d / (double)(n - 1) : 0.0;
    if (q >= 1.0) {
      for (uint64_t u = 0; u < n; ++u)
        for (uint64_t v = u + 1; v < n; ++v) {
          e.push_back((uint32_t)u);
          e.push_back((uint32_t)v);
        }
    } else if (q > 0.0) {  // io.hpp:97-121
      std::mt19937_64 rng(seed);
      const double log1q = std::log1p(-q);
      const uint64_t total = n * (n - 1) / 2;
      uint64_t idx = 0;
      while (true) {
        double r = (double)(rng() >> 11) * 0x1.0p-53;
        double skip = std::floor(std::log1p(-r) / log1q);
        idx += (uint64_t)skip;
        if (idx >= total) break;
        uint64_t lo = 0, hi = n - 1;
        while (lo < hi) {
          uint64_t mid = (lo + hi) / 2;
          uint64_t cum = (mid + 1) * (2 * n - mid - 2) / 2;
          if (cum > idx) hi = mid;
          else lo = mid + 1;
        }
        uint64_t u = lo, before = u * (2 * n - u - 1) / 2;
        uint64_t v = u + 1 + (idx - before);
        e.push_back((uint32_t)u);
        e.push_back((uint32_t)v);
        ++idx;
      }
    }
    uint64_t E = e.size() / 2;
    uint32_t* out = alloc_pairs(E);
    std::memcpy(out, e.data(), e.size() * 4);
    *pairs = out;
    *num_pairs = E;
  });
}

tg_status tg_gen_gnm(uint64_t n, uint64_t m, uint64_t seed, uint32_t** pairs, uint64_t* num_pairs) {
  return guard([&] {
    if (n < 2 && m > 0) throw std::invalid_argument("gen_gnm: need n >= 2");
    if (n >= 2 && m > n * (n - 1) / 2) throw std::invalid_argument("gen_gnm: m > n(n-1)/2");
    uint32_t* out = alloc_pairs(m);
    std::unordered_set<uint64_t> seen;
    seen.reserve(m * 2);
    Xoshiro rng(seed);
    uint64_t w = 0;
    while (w < m) {
      uint64_t u = rng.next() % n, v = rng.next() % n;
      if (u == v) continue;
      if (u > v) std::swap(u, v);
      if (!seen.insert((u << 32) | v).second) continue;
      out[2 * w] = (uint32_t)u;
      out[2 * w + 1] = (uint32_t)v;
      ++w;
    }
    *pairs = out;
    *num_pairs = m;
  });
}

tg_status tg_gen_rmat(uint32_t scale, uint64_t edge_factor, double a, double b, double c,
                      uint64_t seed, uint32_t** pairs, uint64_t* num_pairs) {
  return guard([&] {
    if (scale == 0 || scale > 31) throw std::invalid_argument("gen_rmat: scale in [1, 31]");
    if (a < 0 || b < 0 || c < 0 || a + b + c > 1.0)
      throw std::invalid_argument("gen_rmat: need a,b,c >= 0 and a+b+c <= 1");
    const uint64_t E = edge_factor << scale;
    uint32_t* out = alloc_pairs(E);
    const double ab = a + b, abc = a + b + c;
    const uint64_t chunk = 1ull << 20, chunks = (E + chunk - 1) / chunk;
    parallel_chunks(chunks, [&](uint64_t ci) {
      Xoshiro rng(seed * 0x9E3779B97F4A7C15ull + ci + 1);
      const uint64_t e0 = ci * chunk, e1 = std::min(E, e0 + chunk);
      for (uint64_t e = e0; e < e1; ++e) {
        uint32_t u = 0, v = 0;
        for (uint32_t l = 0; l < scale; ++l) {
          double r = rng.unit();
          uint32_t bu = 0, bv = 0;
          if (r < a) {
          } else if (r < ab) bv = 1;
          else if (r < abc) bu = 1;
          else bu = bv = 1;
          u = (u << 1) | bu;
          v = (v << 1) | bv;
        }
        out[2 * e] = u;
        out[2 * e + 1] = v;
      }
    });
    *pairs = out;
    *num_pairs = E;
  });
}

tg_status tg_gen_ws(uint64_t n, uint64_t k, double beta, uint64_t seed, uint32_t** pairs,
                    uint64_t* num_pairs) {
  return guard([&] {
    if (k % 2 != 0 || k == 0 || k >= n) throw std::invalid_argument("gen_ws: need even 0 < k < n");
    if (beta < 0 || beta > 1) throw std::invalid_argument("gen_ws: beta in [0, 1]");
    if (n > 0xFFFFFFFFull) throw std::invalid_argument("gen_ws: n must fit NodeId");
    const uint64_t half = k / 2, E = n * half;
    uint32_t* out = alloc_pairs(E);
    const uint64_t chunk = 1ull << 16, chunks = (n + chunk - 1) / chunk;
    parallel_chunks(chunks, [&](uint64_t ci) {
      Xoshiro rng(seed * 0xD1B54A32D192ED03ull + ci + 1);
      const uint64_t v0 = ci * chunk, v1 = std::min(n, v0 + chunk);
      for (uint64_t v = v0; v < v1; ++v)
        for (uint64_t j = 1; j <= half; ++j) {
          uint64_t t = (v + j) % n;
          if (rng.unit() < beta) {  // rewire the far end uniformly, no self-loop
            uint64_t w;
            do w = rng.next() % n; while (w == v);
            t = w;
          }
          const uint64_t e = v * half + (j - 1);
          out[2 * e] = (uint32_t)v;
          out[2 * e + 1] = (uint32_t)t;
        }
    });
    *pairs = out;
    *num_pairs = E;
  });
}

}  // extern "C"
