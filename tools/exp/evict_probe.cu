// evict_probe.cu -- do L2 eviction-priority hints keep a hot set of slabs
// resident under a stream of cold random slab reads?  4e8 reads of 128-byte
// slabs over 1e8 slabs; a fraction HOT of them goes to the first 375K slabs
// (48 MB).  Variants: no hint / hot reads evict_last + cold reads evict_first.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o evict_probe evict_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)
__device__ __forceinline__ uint32_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return (uint32_t)x;
}
__global__ void k_ids(uint32_t* ids, uint64_t M, uint32_t n, uint32_t hot, uint32_t hot_per_1024) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < M; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t a = mix(i * 2654435761ULL + 12345), b = mix(i * 0x9E3779B97F4A7C15ULL + 7);
    const bool h = (b & 1023u) < hot_per_1024;
    ids[i] = (uint32_t)(((uint64_t)a * (h ? hot : n)) >> 32);
  }
}
template <int MODE> __device__ __forceinline__ uint4 ldq(const uint4* p, bool hot, uint64_t pol_last, uint64_t pol_first) {
  uint4 r;
  if (MODE == 0) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  } else {
    const uint64_t pol = hot ? pol_last : pol_first;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
  }
  return r;
}
template <int MODE>
__global__ void __launch_bounds__(256, 6)
k_fetch(const uint32_t* __restrict__ ids, uint64_t apexes, const uint4* __restrict__ data, uint32_t hot,
        unsigned long long* out, unsigned long long* ctr) {
  constexpr int H = 20, NB = 5;
  __shared__ uint32_t sU[8][32];
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5, j0 = lane >> 3, q = lane & 7;
  unsigned acc = 0;
  uint64_t pol_last = 0, pol_first = 0;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
  for (;;) {
    unsigned long long a = 0;
    if (lane == 0) a = atomicAdd(ctr, 8ull);
    a = __shfl_sync(0xffffffffu, a, 0);
    if (a >= apexes) break;
    for (unsigned long long k = a; k < a + 8 && k < apexes; ++k) {
      if (lane < H) sU[w][lane] = ids[k * H + lane];
      __syncwarp();
      uint4 r[NB];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const uint32_t u = sU[w][b * 4 + j0];
        r[b] = ldq<MODE>(data + (uint64_t)u * 8 + q, u < hot, pol_last, pol_first);
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) acc += (r[b].x == 7u) + (r[b].y == 7u) + (r[b].z == 7u) + (r[b].w == 7u);
      __syncwarp();
    }
  }
  if (acc) atomicAdd(out, (unsigned long long)acc);
}
int main(int argc, char** argv) {
  const uint32_t n = 100000000u, hot = 375000u;
  const uint64_t apexes = 20000000ull, M = apexes * 20;
  uint32_t* ids; uint4* data; unsigned long long* out;
  CK(cudaMalloc(&ids, M * 4)); CK(cudaMalloc(&data, (uint64_t)n * 128)); CK(cudaMalloc(&out, 16));
  CK(cudaMemset(data, 0xFF, (uint64_t)n * 128));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const uint32_t fr[3] = {0, 102, 154};  // hot share of the reads: 0, 10%, 15%
  for (int f = 0; f < 3; ++f) {
    k_ids<<<148 * 8, 256>>>(ids, M, n, hot, fr[f]);
    CK(cudaDeviceSynchronize());
    for (int mode = 0; mode < 2; ++mode) {
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        CK(cudaMemset(out, 0, 16));
        cudaEventRecord(e0);
        if (mode == 0) k_fetch<0><<<148 * 6, 256>>>(ids, apexes, data, hot, out, out + 1);
        else k_fetch<1><<<148 * 6, 256>>>(ids, apexes, data, hot, out, out + 1);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep && ms < best) best = ms;
      }
      printf("{\"hot_share\": %.3f, \"hints\": %d, \"ms\": %.3f, \"reads_per_s\": %.4g}\n", fr[f] / 1024.0, mode, best, M / (best * 1e-3));
    }
  }
  return 0;
}
