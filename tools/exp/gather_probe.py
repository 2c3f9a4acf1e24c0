#!/usr/bin/env python
"""Experiment: throughput of the orientation's key gather alone (keys[i] =
key(adj[i]) over the whole adjacency) on C2, 4-byte degrees vs 1-byte codes,
to decide whether a two-phase orientation (gather, then a streaming pass)
could beat the fused tile pass.  Not part of the library."""
import os
import sys

import torch
from torch.utils.cpp_extension import load_inline

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

src = r"""
#include <torch/extension.h>
#include <cstdint>
template <class K, int U>
__global__ void k_gather(const uint32_t* __restrict__ adj, long long m2, const K* __restrict__ key,
                         K* __restrict__ out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < m2; i0 += stride * U) {
    uint32_t u[U];
#pragma unroll
    for (int q = 0; q < U; ++q) u[q] = i0 + q * stride < m2 ? __ldcs(adj + i0 + q * stride) : 0u;
#pragma unroll
    for (int q = 0; q < U; ++q)
      if (i0 + q * stride < m2) __stcs(out + i0 + q * stride, __ldg(key + u[q]));
  }
}
void gather4(torch::Tensor adj, torch::Tensor key, torch::Tensor out, int blocks) {
  k_gather<uint32_t, 8><<<blocks, 256>>>((const uint32_t*)adj.data_ptr(), adj.numel(),
      (const uint32_t*)key.data_ptr(), (uint32_t*)out.data_ptr());
}
void gather1(torch::Tensor adj, torch::Tensor key, torch::Tensor out, int blocks) {
  k_gather<uint8_t, 8><<<blocks, 256>>>((const uint32_t*)adj.data_ptr(), adj.numel(),
      (const uint8_t*)key.data_ptr(), (uint8_t*)out.data_ptr());
}
"""
cpp = "void gather4(torch::Tensor, torch::Tensor, torch::Tensor, int);\nvoid gather1(torch::Tensor, torch::Tensor, torch::Tensor, int);"
mod = load_inline("gather_probe", cpp_sources=cpp, cuda_sources=src, functions=["gather4", "gather1"],
                  extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a", "-O3"],
                  build_directory="/tmp", verbose=False)

from paper_1706_05151_b200 import trigraph as T  # noqa: E402
import numpy as np  # noqa: E402

pairs = T.gen_pa(10_000_000, 40, 7)
g = T.build_graph(pairs, 10_000_000)
off, adj = g.csr()
deg = np.diff(off).astype(np.uint32)
code = np.minimum(deg, 255).astype(np.uint8)
adj_t = torch.from_numpy(adj.view(np.int32)).cuda()
deg_t = torch.from_numpy(deg.view(np.int32)).cuda()
code_t = torch.from_numpy(code).cuda()
o4 = torch.empty_like(adj_t)
o1 = torch.empty(adj_t.numel(), dtype=torch.uint8, device="cuda")
for blocks in (148 * 8, 148 * 16, 148 * 32):
    for name, f, k, o in (("deg4", mod.gather4, deg_t, o4), ("code1", mod.gather1, code_t, o1)):
        for _ in range(2):
            f(adj_t, k, o, blocks)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            f(adj_t, k, o, blocks)
        e.record()
        torch.cuda.synchronize()
        print(name, blocks, "%.3f ms" % (s.elapsed_time(e) / 5), flush=True)
