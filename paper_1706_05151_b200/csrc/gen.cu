// gen.cu -- the parallel synthetic generators on the device (SURVEY 8(f) #3,
// BASELINE.json configs 3 and 4), bit-identical to the host harness in
// generators.cpp, followed by build_graph on the device -- no host round trip
// for the 2-4 GB edge lists.
//
// Both host generators are chunked: chunk c of R-MAT (2^20 edges) and of
// Watts-Strogatz (2^16 ring vertices) draws from its own xoshiro256** stream
// seeded by splitmix64 of a chunk-derived seed, so the device runs one thread
// per chunk with the same arithmetic (the unit draw (x >> 11) * 2^-53 is
// exact, the comparisons are IEEE, the rest is integer) and writes the same
// pairs at the same positions.  gen_pa / gen_gnp (the reference's io.hpp
// generators) are one sequential mt19937_64 stream with data-dependent
// rejection and stay on the host; G(n, m) needs a global dedup and stays there
// too.
#include <cstdint>

#include "tg_internal.cuh"

namespace tgb {
namespace {

__device__ __forceinline__ uint64_t d_splitmix64(uint64_t& x) {
  uint64_t z = (x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct DXoshiro {
  uint64_t s[4];
  __device__ explicit DXoshiro(uint64_t seed) {
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) s[i] = d_splitmix64(x);
  }
  __device__ static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  __device__ uint64_t next() {
    const uint64_t r = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3];
    s[2] ^= t; s[3] = rotl(s[3], 45);
    return r;
  }
  __device__ double unit() { return (double)(next() >> 11) * 0x1.0p-53; }
};

// generators.cpp tg_gen_rmat: chunk ci of 2^20 edges, one thread each
__global__ void k_gen_rmat(uint32_t scale, uint64_t E, double a, double ab, double abc,
                           uint64_t seed, uint32_t* __restrict__ out) {
  const uint64_t chunk = 1ull << 20, chunks = (E + chunk - 1) / chunk;
  for (uint64_t ci = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; ci < chunks;
       ci += (uint64_t)gridDim.x * blockDim.x) {
    DXoshiro rng(seed * 0x9E3779B97F4A7C15ull + ci + 1);
    const uint64_t e0 = ci * chunk, e1 = min(E, e0 + chunk);
    for (uint64_t e = e0; e < e1; ++e) {
      uint32_t u = 0, v = 0;
      for (uint32_t l = 0; l < scale; ++l) {
        const double r = rng.unit();
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
  }
}

// generators.cpp tg_gen_ws: chunk ci of 2^16 ring vertices, one thread each
__global__ void k_gen_ws(uint64_t n, uint64_t half, double beta, uint64_t seed,
                         uint32_t* __restrict__ out) {
  const uint64_t chunk = 1ull << 16, chunks = (n + chunk - 1) / chunk;
  for (uint64_t ci = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; ci < chunks;
       ci += (uint64_t)gridDim.x * blockDim.x) {
    DXoshiro rng(seed * 0xD1B54A32D192ED03ull + ci + 1);
    const uint64_t v0 = ci * chunk, v1 = min(n, v0 + chunk);
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
  }
}

}  // namespace

uint64_t gen_rmat_device(uint32_t scale, uint64_t edge_factor, double a, double b, double c,
                         uint64_t seed, DBuf<uint32_t>& pairs, cudaStream_t s) {
  TG_REQUIRE(scale >= 1 && scale <= 31, "gen_rmat: scale in [1, 31]");
  TG_REQUIRE(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0,
             "gen_rmat: need a,b,c >= 0 and a+b+c <= 1");
  const uint64_t E = edge_factor << scale;
  pairs.alloc(2 * (E ? E : 1), s);
  const uint64_t chunks = (E + (1ull << 20) - 1) >> 20;
  if (chunks) {
    k_gen_rmat<<<grid_for(chunks, 64, 148u * 16u), 64, 0, s>>>(scale, E, a, a + b, a + b + c, seed,
                                                               pairs.p);
    TG_CHECK_LAUNCH();
    ++g_launches;
  }
  return E;
}

uint64_t gen_ws_device(uint64_t n, uint64_t k, double beta, uint64_t seed, DBuf<uint32_t>& pairs,
                       cudaStream_t s) {
  TG_REQUIRE(k % 2 == 0 && k > 0 && k < n, "gen_ws: need even 0 < k < n");
  TG_REQUIRE(beta >= 0 && beta <= 1, "gen_ws: beta in [0, 1]");
  TG_REQUIRE(n <= 0xFFFFFFFFull, "gen_ws: n must fit NodeId");
  const uint64_t half = k / 2, E = n * half;
  pairs.alloc(2 * (E ? E : 1), s);
  const uint64_t chunks = (n + (1ull << 16) - 1) >> 16;
  k_gen_ws<<<grid_for(chunks, 64, 148u * 16u), 64, 0, s>>>(n, half, beta, seed, pairs.p);
  TG_CHECK_LAUNCH();
  ++g_launches;
  return E;
}

}  // namespace tgb
