// slab_probe.cu -- how fast can a B200 fetch ~80-byte lists at random?
//
// Experiment behind the slab layout of the oriented lists: the
// intersection pass of a PA graph is a stream of random reads of N_u, h_u ~ 20.
// Variants (n lists, M random list reads, 20 reads per "apex"):
//   desc  : 8-byte descriptor at desc[u], then the 6 quads covering an
//           unaligned 20-entry list (stride 21 slots) -- today's layout;
//   slabK : list u in a K-slot slab at u*K (K = 24, 32): no descriptor, sector
//           aligned, 32/(K/4) lists per warp load.
// Each under cudaLimitMaxL2FetchGranularity = 32 / 64 / 128.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o slab_probe slab_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return (uint32_t)x;
}
__global__ void k_ids(uint32_t* ids, uint64_t M, uint32_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < M; i += (uint64_t)gridDim.x * blockDim.x)
    ids[i] = (uint32_t)(((uint64_t)mix(i * 2654435761ULL + 12345) * n) >> 32);
}
__global__ void k_desc(uint64_t* desc, uint32_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    desc[i] = ((i * 21) << 24) | 20;
}
__device__ __forceinline__ uint4 ldq(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// QK quads per list, G = 32 / QK lists per warp load, H = 20 lists per apex
template <int QK, bool DESC>
__global__ void __launch_bounds__(256, 6)
k_fetch(const uint32_t* __restrict__ ids, uint64_t apexes, const uint4* __restrict__ data,
        const uint64_t* __restrict__ desc, unsigned long long* out, unsigned long long* ctr) {
  constexpr int G = 32 / QK, H = 20, NB = (H + G - 1) / G;
  __shared__ uint32_t sU[8][32];
  __shared__ uint32_t sQ[8][32];
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned j0 = lane / QK, q = lane % QK;
  unsigned acc = 0;
  for (;;) {
    unsigned long long a = 0;
    if (lane == 0) a = atomicAdd(ctr, 8ull);
    a = __shfl_sync(0xffffffffu, a, 0);
    if (a >= apexes) break;
    for (unsigned long long k = a; k < a + 8 && k < apexes; ++k) {
      if (lane < H) {
        const uint32_t u = ids[k * H + lane];
        sU[w][lane] = u;
        if (DESC) sQ[w][lane] = (uint32_t)((desc[u] >> 24) >> 2);
      }
      __syncwarp();
      uint4 r[NB];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const unsigned j = b * G + j0;
        const bool ok = j < H && j0 < G;
        const unsigned jj = ok ? j : 0;
        const uint64_t qi = DESC ? (uint64_t)sQ[w][jj] + q : (uint64_t)sU[w][jj] * QK + q;
        r[b] = ok ? ldq(data + qi) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) acc += (r[b].x == 7u) + (r[b].y == 7u) + (r[b].z == 7u) + (r[b].w == 7u);
      __syncwarp();
    }
  }
  if (acc) atomicAdd(out, (unsigned long long)acc);
}

int main(int argc, char** argv) {
  const uint32_t n = argc > 1 ? (uint32_t)atof(argv[1]) : 100000000u;
  const uint64_t apexes = argc > 2 ? (uint64_t)atof(argv[2]) : 20000000ull;
  const uint64_t M = apexes * 20;
  uint32_t* ids; uint4* data; uint64_t* desc; unsigned long long* out;
  CK(cudaMalloc(&ids, M * 4));
  CK(cudaMalloc(&data, (uint64_t)n * 32 * 4 + 64));
  CK(cudaMalloc(&desc, (uint64_t)n * 8));
  CK(cudaMalloc(&out, 16));
  CK(cudaMemset(data, 0xFF, (uint64_t)n * 32 * 4 + 64));
  k_ids<<<148 * 8, 256>>>(ids, M, n);
  k_desc<<<148 * 8, 256>>>(desc, n);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int fs[3] = {32, 64, 128};
  for (int fi = 0; fi < 3; ++fi) {
    CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, fs[fi]));
    size_t got = 0;
    cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
    for (int variant = 0; variant < 4; ++variant) {
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        CK(cudaMemset(out, 0, 16));
        cudaEventRecord(e0);
        if (variant == 0) k_fetch<6, true><<<148 * 6, 256>>>(ids, apexes, data, desc, out, out + 1);
        if (variant == 1) k_fetch<6, false><<<148 * 6, 256>>>(ids, apexes, data, desc, out, out + 1);
        if (variant == 2) k_fetch<8, false><<<148 * 6, 256>>>(ids, apexes, data, desc, out, out + 1);
        if (variant == 3) k_fetch<5, false><<<148 * 6, 256>>>(ids, apexes, data, desc, out, out + 1);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep && ms < best) best = ms;
      }
      const char* nm[4] = {"desc+unaligned(6q)", "slab24", "slab32", "slab20"};
      printf("{\"fetch\": %zu, \"variant\": \"%s\", \"ms\": %.3f, \"lists_per_s\": %.4g, \"useful_GBs\": %.1f}\n", got,
             nm[variant], best, M / (best * 1e-3), M * 80.0 / (best * 1e-3) / 1e9);
    }
  }
  return 0;
}
