// comm.cu -- the paper's engines across GPUs: one rank per GPU (one process
// each, or one host thread each), NCCL over NVLink/NVSwitch for the exchange.
//
// Reference semantics (engines.hpp): AOP (:38-54, run_engine :367-381) --
// rank i counts the triangles whose apex lies in core i of the cost plan
// (partition.hpp:116-141) with no data-path messages; ANOP-surrogate
// (:146-198) -- rank i stores only its core lists (partition.hpp:210-239),
// ships (v, N_v) once per distinct remote owner of N_v's entries (LastProc)
// and every owner runs SurrogateCount (:60-76); aggregate_clustering
// (:211-268) -- off-core tallies summed at the owner, C_v computed there.
//
// Input distribution: every rank holds rows [lo, hi) of the symmetric CSR
// (tg_graph_from_rows; the ranks' row ranges tile [0, n) in rank order) plus
// the global degree vector -- or the whole graph (replicated input; then the
// rank's rows are an equal-adjacency-volume split).  Each rank orients ONLY
// its rows (1/N of the orientation work), then:
//   AOP       -- the oriented rows of all ranks are gathered (one broadcast
//                per rank over NVLink; list lengths first, so every rank
//                builds the same compact CSR), the plan is computed from the
//                gathered costs, and the rank counts its core;
//   SURROGATE -- list lengths are gathered (4 B per vertex), the plan is
//                computed from distributed costs, each rank's oriented rows
//                move to their core owner with one all-to-allv (Σ stored = m),
//                then the surrogate all-to-allv and the counts;
//   DIRECT    -- (engines.hpp:80-141) the same core partitions; one request
//                per off-core pair (v, u) to owner(u), one reply carrying
//                N_u, batched into three all-to-allv;
//   tallies   -- per-rank n-vectors reduced to their owner's core range
//                (one NCCL reduce per owner in a group), C_v at the owner.
// The global count is one all-reduce of a u64; per-rank stats are gathered
// so every rank returns the same RunReport.
//
// Transport: NCCL (loaded at run time with dlopen, so the library loads
// without it), or an in-process group of host threads (tests: N ranks on one
// GPU; the exchange is host-orchestrated device copies, so no kernel ever
// waits on another rank's kernel).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>

#include <cub/device/device_scan.cuh>

#include "handle.cuh"

namespace tgb {
namespace {

// ------------------------------------------------------------------ NCCL

struct Nccl {
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclBroadcast) Broadcast = nullptr;
  decltype(&ncclReduce) Reduce = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
};

Nccl& nccl() {
  static Nccl api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = "libnccl.so.2 not found";
      return;
    }
#define TG_SYM(name) api.name = (decltype(api.name))dlsym(h, "nccl" #name)
    TG_SYM(GetUniqueId);
    TG_SYM(CommInitRank);
    TG_SYM(CommDestroy);
    TG_SYM(AllReduce);
    TG_SYM(Broadcast);
    TG_SYM(Reduce);
    TG_SYM(Send);
    TG_SYM(Recv);
    TG_SYM(GroupStart);
    TG_SYM(GroupEnd);
    TG_SYM(GetErrorString);
#undef TG_SYM
    if (!api.CommInitRank || !api.AllReduce || !api.Send) err = "incomplete NCCL library";
  });
  if (!err.empty()) throw Error(TG_ERR_INTERNAL, "NCCL: " + err);
  return api;
}

#define TG_NCCL(expr)                                                                  \
  do {                                                                                 \
    ncclResult_t _r = (expr);                                                          \
    if (_r != ncclSuccess)                                                             \
      throw ::tgb::Error(TG_ERR_INTERNAL,                                              \
                         std::string("NCCL ") + #expr + ": " + ::tgb::nccl().GetErrorString(_r)); \
  } while (0)

// ------------------------------------------------------------------ transport

struct Transport {
  int rank = 0, size = 1;
  virtual ~Transport() = default;
  // element-wise sum over ranks, in place
  virtual void all_reduce_u64(uint64_t* d, size_t count, cudaStream_t s) = 0;
  // root's bytes to every rank, in place
  virtual void broadcast(void* d, size_t bytes, int root, cudaStream_t s) = 0;
  // sum over ranks into root's buffer (others' buffers unspecified after)
  virtual void reduce_u64(uint64_t* d, size_t count, int root, cudaStream_t s) = 0;
  // segment j of d_send (sbytes[j]) to rank j; segment i of d_recv from rank i
  virtual void all_to_allv(const void* d_send, const std::vector<size_t>& sbytes, void* d_recv,
                           const std::vector<size_t>& rbytes, cudaStream_t s) = 0;
};

struct NcclTransport : Transport {
  ncclComm_t comm = nullptr;
  ~NcclTransport() override {
    if (comm) nccl().CommDestroy(comm);
  }
  void all_reduce_u64(uint64_t* d, size_t count, cudaStream_t s) override {
    if (count) TG_NCCL(nccl().AllReduce(d, d, count, ncclUint64, ncclSum, comm, s));
  }
  void broadcast(void* d, size_t bytes, int root, cudaStream_t s) override {
    if (bytes) TG_NCCL(nccl().Broadcast(d, d, bytes, ncclChar, root, comm, s));
  }
  void reduce_u64(uint64_t* d, size_t count, int root, cudaStream_t s) override {
    if (count) TG_NCCL(nccl().Reduce(d, d, count, ncclUint64, ncclSum, root, comm, s));
  }
  void all_to_allv(const void* d_send, const std::vector<size_t>& sbytes, void* d_recv,
                   const std::vector<size_t>& rbytes, cudaStream_t s) override {
    size_t so = 0, ro = 0;
    std::vector<size_t> soff(size), roff(size);
    for (int j = 0; j < size; ++j) {
      soff[j] = so;
      roff[j] = ro;
      so += sbytes[j];
      ro += rbytes[j];
    }
    if (sbytes[rank])
      TG_CUDA(cudaMemcpyAsync((char*)d_recv + roff[rank], (const char*)d_send + soff[rank],
                              sbytes[rank], cudaMemcpyDeviceToDevice, s));
    TG_NCCL(nccl().GroupStart());
    for (int j = 0; j < size; ++j) {
      if (j == rank) continue;
      if (sbytes[j])
        TG_NCCL(nccl().Send((const char*)d_send + soff[j], sbytes[j], ncclChar, j, comm, s));
      if (rbytes[j]) TG_NCCL(nccl().Recv((char*)d_recv + roff[j], rbytes[j], ncclChar, j, comm, s));
    }
    TG_NCCL(nccl().GroupEnd());
  }
};

// N ranks in one process (host threads), host-orchestrated device copies.
struct LocalGroup {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<const void*> ptr;
  std::vector<std::vector<size_t>> sizes;
  std::vector<uint64_t> acc;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct LocalTransport : Transport {
  std::shared_ptr<LocalGroup> grp;
  void all_reduce_u64(uint64_t* d, size_t count, cudaStream_t s) override {
    std::vector<uint64_t> h(count);
    if (count) TG_CUDA(cudaMemcpyAsync(h.data(), d, count * 8, cudaMemcpyDeviceToHost, s));
    TG_CUDA(cudaStreamSynchronize(s));
    grp->barrier();
    if (rank == 0) grp->acc.assign(count, 0);
    grp->barrier();
    {
      std::lock_guard<std::mutex> lk(grp->mu);
      for (size_t i = 0; i < count; ++i) grp->acc[i] += h[i];
    }
    grp->barrier();
    if (count) TG_CUDA(cudaMemcpy(d, grp->acc.data(), count * 8, cudaMemcpyHostToDevice));
    grp->barrier();
  }
  void broadcast(void* d, size_t bytes, int root, cudaStream_t s) override {
    TG_CUDA(cudaStreamSynchronize(s));
    grp->ptr[rank] = d;
    grp->barrier();
    if (rank != root && bytes) TG_CUDA(cudaMemcpy(d, grp->ptr[root], bytes, cudaMemcpyDefault));
    grp->barrier();
  }
  void reduce_u64(uint64_t* d, size_t count, int root, cudaStream_t s) override {
    (void)root;
    all_reduce_u64(d, count, s);
  }
  void all_to_allv(const void* d_send, const std::vector<size_t>& sbytes, void* d_recv,
                   const std::vector<size_t>& rbytes, cudaStream_t s) override {
    TG_CUDA(cudaStreamSynchronize(s));
    grp->ptr[rank] = d_send;
    grp->sizes[rank] = sbytes;
    grp->barrier();
    size_t ro = 0;
    for (int i = 0; i < size; ++i) {
      size_t so = 0;
      for (int j = 0; j < rank; ++j) so += grp->sizes[i][j];
      TG_REQUIRE(grp->sizes[i][rank] == rbytes[i], "all_to_allv: send / receive sizes differ");
      if (rbytes[i])
        TG_CUDA(cudaMemcpy((char*)d_recv + ro, (const char*)grp->ptr[i] + so, rbytes[i],
                           cudaMemcpyDefault));
      ro += rbytes[i];
    }
    grp->barrier();
  }
};

// ------------------------------------------------------------------ kernels

constexpr uint64_t kRowCost = 32;
__global__ void k_volume_split(const uint64_t* __restrict__ off, uint64_t n, uint32_t parts,
                               uint32_t* __restrict__ a) {
  // Equal ORIENTATION COST: c(v) = off[v] + kRowCost v -- a row costs what ~32
  // adjacency entries do (fit of the per-rank orientation times of C5 at
  // N = 8, profiles/r02h_scaling.jsonl: 6.05e-9 ms per entry + 1.91e-7 ms per
  // row; an equal-adjacency split left the last rank at 2.1x the first).
  // a[j] = smallest v with c(v) >= j * c(n) / parts (a[0] = 0, a[parts] = n),
  // rounded down to whole 32-vertex tiles (the tile kernel's unit)
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j > parts) return;
  if (j == 0) { a[0] = 0; return; }
  if (j == parts) { a[parts] = (uint32_t)n; return; }
  const unsigned __int128 target = (unsigned __int128)(off[n] + kRowCost * n) * j;
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if ((unsigned __int128)(off[mid] + kRowCost * mid) * parts >= target) hi = mid;
    else lo = mid + 1;
  }
  a[j] = (uint32_t)(lo & ~31ull);
}

__global__ void k_lens_from_off(const uint64_t* __restrict__ off, uint64_t rows,
                                uint32_t* __restrict__ lens) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x)
    lens[r] = (uint32_t)(off[r + 1] - off[r]);
}

__global__ void k_u32_to_u64(const uint32_t* __restrict__ a, uint64_t n, uint64_t* __restrict__ b) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
       r += (uint64_t)gridDim.x * blockDim.x)
    b[r] = a[r];
}

__global__ void k_desc_from_off2(const uint64_t* __restrict__ off, uint64_t rows,
                                 uint64_t* __restrict__ desc, uint64_t shift = 0) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x)
    desc[r] = make_desc(shift + off[r], off[r + 1] - off[r]);
}

__global__ void k_dcode(const uint32_t* __restrict__ deg, uint64_t n, uint8_t* __restrict__ dcode) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x)
    dcode[v] = degree_code(deg[v]);
}

// partition.hpp:45-91 node_costs for rows [lo, hi): part = their oriented
// lists (compact, base lo), lens = every vertex's h, deg = every degree;
// the symmetric rows (off / adj, indexed by global id) for NOV.
__global__ void k_costs_rows(CsrView part, uint32_t lo, uint32_t hi, const uint32_t* __restrict__ lens,
                             const uint32_t* __restrict__ deg, const uint64_t* __restrict__ off,
                             const uint32_t* __restrict__ adj, int kind, uint64_t* __restrict__ f) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; w < hi - lo; w += warps) {
    const uint32_t v = lo + (uint32_t)w;
    const uint64_t hv = lens[v], dv = deg[v];
    uint64_t s = 0;
    if (kind == TG_COST_DPD) {  // :60-69
      const uint64_t d = part.desc[w];
      const uint32_t* L = part.data + desc_start(d);
      for (uint32_t i = lane; i < desc_len(d); i += 32) s += hv + lens[L[i]];
    } else if (kind == TG_COST_NOV) {  // :70-81, predecessors: neighbours not in N_v
      const uint64_t d = part.desc[w];
      const uint32_t* L = part.data + desc_start(d);
      const uint32_t h = desc_len(d);
      for (uint64_t k = off[v] + lane; k < off[v + 1]; k += 32) {
        const uint32_t u = adj[k];
        uint32_t a = 0, b = h;  // u in N_v?
        while (a < b) {
          const uint32_t mid = (a + b) >> 1;
          if (L[mid] < u) a = mid + 1;
          else b = mid;
        }
        if (!(a < h && L[a] == u)) s += hv + lens[u];
      }
    } else if (lane == 0) {
      s = kind == TG_COST_N ? 1 : kind == TG_COST_D ? dv : kind == TG_COST_DH ? hv
          : kind == TG_COST_DDH ? dv * hv : hv * hv;
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) f[v] = s;
  }
}

__global__ void k_cc_range(const uint32_t* __restrict__ deg, const unsigned long long* __restrict__ t,
                           uint32_t lo, uint32_t hi, double* __restrict__ c) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < hi - lo;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t d = deg[lo + i];
    double r = 0.0;
    if (d >= 2)  // engines.hpp:258-267, IEEE-rounded, no contraction
      r = __ddiv_rn(__dmul_rn(2.0, (double)t[i]), __dmul_rn((double)d, (double)(d - 1)));
    c[i] = r;
  }
}

// ---- ANOP-direct (engines.hpp:80-141): request / reply kernels ----
__device__ __forceinline__ uint32_t owner_dev(const uint32_t* __restrict__ gb, uint32_t p, uint32_t u) {
  uint32_t lo = 0, hi = p;  // the i with gb[i] <= u < gb[i+1] (partition.hpp:104-109)
  while (lo + 1 < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (gb[mid] <= u) lo = mid;
    else hi = mid;
  }
  return lo;
}

// One request per off-core entry u of a core list N_v (the reference sends
// one per (v, u) pair and never caches): FILL = false counts them per owner,
// FILL = true writes (u, v) destination-major at the cursors.
template <bool FILL>
__global__ void __launch_bounds__(256)
k_direct_requests(CsrView part, uint32_t cb, uint32_t ce, const uint32_t* __restrict__ gb, uint32_t p,
                  uint32_t self, unsigned long long* __restrict__ cnt_or_cur,
                  uint32_t* __restrict__ req_u, uint32_t* __restrict__ req_v) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; w < ce - cb; w += warps) {
    const uint64_t d = part.desc[w];
    const uint32_t* L = part.data + desc_start(d);
    for (uint32_t i = lane; i < desc_len(d); i += 32) {
      const uint32_t u = L[i], ou = owner_dev(gb, p, u);
      if (ou == self) continue;
      const unsigned long long pos = atomicAdd(&cnt_or_cur[ou], 1ull);
      if (FILL) {
        req_u[pos] = u;
        req_v[pos] = cb + (uint32_t)w;
      }
    }
  }
}

// serve_request (engines.hpp:93-99): the length of each requested core list
__global__ void k_reply_lens(CsrView part, const uint32_t* __restrict__ got_u, uint64_t R,
                             uint32_t* __restrict__ lens) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < R;
       i += (uint64_t)gridDim.x * blockDim.x)
    lens[i] = desc_len(part.desc[got_u[i] - part.base]);
}

// ... and the lists themselves, back to back in request order
__global__ void __launch_bounds__(256)
k_reply_fill(CsrView part, const uint32_t* __restrict__ got_u, uint64_t R,
             const uint64_t* __restrict__ off, uint32_t* __restrict__ payload) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < R; i += warps) {
    const uint64_t d = part.desc[got_u[i] - part.base];
    const uint32_t* L = part.data + desc_start(d);
    for (uint32_t k = lane; k < desc_len(d); k += 32) payload[off[i] + k] = L[k];
  }
}

// the requester's intersect_visit(N_v, reply) (engines.hpp:121-126): a warp
// per reply, each element searched in the sorted core list N_v
__global__ void __launch_bounds__(256)
k_direct_count(CsrView part, const uint32_t* __restrict__ req_v, uint64_t R,
               const uint64_t* __restrict__ off, const uint32_t* __restrict__ payload,
               unsigned long long* __restrict__ total) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long acc = 0;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < R; i += warps) {
    const uint64_t d = part.desc[req_v[i] - part.base];
    const uint32_t* Nv = part.data + desc_start(d);
    const uint32_t hv = desc_len(d);
    for (uint64_t k = off[i] + lane; k < off[i + 1]; k += 32) {
      const uint32_t x = payload[k];
      uint32_t a = 0, b = hv;
      while (a < b) {
        const uint32_t mid = (a + b) >> 1;
        if (Nv[mid] < x) a = mid + 1;
        else b = mid;
      }
      acc += a < hv && Nv[a] == x;
    }
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0 && acc) atomicAdd(total, acc);
}

template <class F>
void cub_run(cudaStream_t s, F&& f) {
  size_t bytes = 0;
  TG_CUDA(f(nullptr, bytes));
  DBuf<char> tmp(bytes ? bytes : 1, s);
  TG_CUDA(f(tmp.p, bytes));
}

uint64_t read_u64(const uint64_t* d, cudaStream_t s) {
  uint64_t h = 0;
  TG_CUDA(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  return h;
}

}  // namespace
}  // namespace tgb

struct tg_comm {
  int device = 0;
  std::unique_ptr<tgb::Transport> t;
};

namespace {

using tgb::CountOut;
using tgb::CsrView;
using tgb::DBuf;
using tgb::DevEff;
using tgb::Transport;

template <class F>
tg_status guard(F&& f) {
  try {
    f();
    return TG_OK;
  } catch (const tgb::Error& e) {
    tgb_set_error(e.what());
    return e.status;
  } catch (const std::bad_alloc& e) {
    tgb_set_error(e.what());
    return TG_ERR_OOM;
  } catch (const std::exception& e) {
    tgb_set_error(e.what());
    return TG_ERR_INTERNAL;
  }
}

// every rank's u64 value on every rank (an all-reduce of a one-hot vector)
std::vector<uint64_t> all_gather_host(Transport& T, const std::vector<uint64_t>& mine,
                                      cudaStream_t s) {
  const size_t k = mine.size(), N = T.size;
  std::vector<uint64_t> h(N * k, 0);
  std::copy(mine.begin(), mine.end(), h.begin() + T.rank * k);
  DBuf<uint64_t> d(N * k, s);
  TG_CUDA(cudaMemcpyAsync(d.p, h.data(), N * k * 8, cudaMemcpyHostToDevice, s));
  T.all_reduce_u64(d.p, N * k, s);
  TG_CUDA(cudaMemcpyAsync(h.data(), d.p, N * k * 8, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  return h;
}

// The rows this rank orients: its own rows (rank-local graph; the ranks'
// ranges must tile [0, n) in rank order) or an equal-orientation-cost split.
std::vector<uint32_t> row_split(tg_graph* g, Transport& T) {
  const uint32_t N = (uint32_t)T.size;
  cudaStream_t s = g->stream;
  std::vector<uint32_t> a(N + 1);
  if (g->partial) {
    auto r = all_gather_host(T, {g->row_lo, g->row_hi}, s);
    for (uint32_t i = 0; i < N; ++i) {
      TG_REQUIRE(r[2 * i] == (i ? r[2 * i - 1] : 0), "rank rows must tile [0, n) in rank order");
      a[i] = (uint32_t)r[2 * i];
    }
    TG_REQUIRE(r[2 * N - 1] == g->g.n, "rank rows must tile [0, n) in rank order");
    a[N] = (uint32_t)g->g.n;
    return a;
  }
  DBuf<uint32_t> d(N + 1, s);
  tgb::k_volume_split<<<1, 128 * ((N + 128) / 128), 0, s>>>(g->g.off.p, g->g.n, N, d.p);
  TG_CHECK_LAUNCH();
  ++tgb::g_launches;
  TG_CUDA(cudaMemcpyAsync(a.data(), d.p, (N + 1) * 4, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  return a;
}

// This rank's rows oriented (effective.hpp:37-52, compact, base lo) and the
// list length of every vertex gathered on every rank (one broadcast per rank).
struct Oriented {
  std::vector<uint32_t> a;    // N+1 row ranges
  std::vector<uint64_t> cnt;  // oriented entries per rank
  DevEff slice;
  DBuf<uint32_t> lens;        // n
};

void orient_mine(tg_graph* g, Transport& T, Oriented& o) {
  cudaStream_t s = g->stream;
  const uint64_t n = g->g.n;
  o.a = row_split(g, T);
  const uint32_t lo = o.a[T.rank], hi = o.a[T.rank + 1];
  if (lo % 32 == 0 && (hi % 32 == 0 || hi == n))
    tgb::orient_rows_tiles(g->g, lo, hi, o.slice, s);  // the one-pass tile kernel
  else
    tgb::orient_rows(g->g, lo, hi, o.slice, s);
  o.cnt = all_gather_host(T, {o.slice.entries}, s);
  o.lens.alloc(n ? n : 1, s);
  if (hi > lo) {
    tgb::k_lens_from_off<<<tgb::grid_for(hi - lo, 256), 256, 0, s>>>(o.slice.off.p, hi - lo,
                                                                     o.lens.p + lo);
    TG_CHECK_LAUNCH();
    ++tgb::g_launches;
  }
  for (int r = 0; r < T.size; ++r)
    T.broadcast(o.lens.p + o.a[r], (size_t)(o.a[r + 1] - o.a[r]) * 4, r, s);
}

// exclusive prefix of the gathered lengths (n+1) -> desc of a compact CSR
void offsets_from_lens(const DBuf<uint32_t>& lens, uint64_t n, DBuf<uint64_t>& off,
                       cudaStream_t s) {
  off.alloc(n + 1, s);
  TG_CUDA(cudaMemsetAsync(off.p, 0, 8, s));
  if (!n) return;
  DBuf<uint64_t> l64(n, s);
  tgb::k_u32_to_u64<<<tgb::grid_for(n, 256), 256, 0, s>>>(lens.p, n, l64.p);
  TG_CHECK_LAUNCH();
  tgb::cub_run(s, [&](void* t, size_t& b) {
    return cub::DeviceScan::InclusiveSum(t, b, l64.p, off.p + 1, (int64_t)n, s);
  });
  tgb::g_launches += 2;
}

// AOP input: the full oriented CSR on every rank -- the slices broadcast in
// rank order into one compact array (same layout everywhere).
void gather_full(tg_graph* g, Transport& T, Oriented& o, DevEff& full) {
  cudaStream_t s = g->stream;
  const uint64_t n = g->g.n;
  uint64_t m = 0;
  std::vector<uint64_t> base(T.size);
  for (int r = 0; r < T.size; ++r) {
    base[r] = m;
    m += o.cnt[r];
  }
  full.rows = n;
  full.base = 0;
  full.compact = true;
  full.entries = m;
  full.data.alloc(m + tgb::kQuadPad, s);
  TG_CUDA(cudaMemsetAsync(full.data.p + m, 0, tgb::kQuadPad * 4, s));
  if (o.slice.entries)
    TG_CUDA(cudaMemcpyAsync(full.data.p + base[T.rank], o.slice.data.p, o.slice.entries * 4,
                            cudaMemcpyDeviceToDevice, s));
  for (int r = 0; r < T.size; ++r) T.broadcast(full.data.p + base[r], o.cnt[r] * 4, r, s);
  offsets_from_lens(o.lens, n, full.off, s);
  full.desc.alloc(n ? n : 1, s);
  if (n) {
    tgb::k_desc_from_off2<<<tgb::grid_for(n, 256), 256, 0, s>>>(full.off.p, n, full.desc.p);
    TG_CHECK_LAUNCH();
    ++tgb::g_launches;
  }
}

// costs of every vertex (partition.hpp:45-91), each rank computing its rows
// from its oriented slice and the gathered lengths, then gathered
void gather_costs(tg_graph* g, Transport& T, const Oriented& o, int kind, DBuf<uint64_t>& f,
                  cudaStream_t s) {
  const uint64_t n = g->g.n;
  const uint32_t lo = o.a[T.rank], hi = o.a[T.rank + 1];
  f.alloc(n ? n : 1, s);
  if (hi > lo) {
    const CsrView pv = tgh::view(o.slice);
    tgb::k_costs_rows<<<tgb::grid_for((uint64_t)(hi - lo) * 32, 256, 148u * 32u), 256, 0, s>>>(
        pv, lo, hi, o.lens.p, g->g.deg.p, g->g.off.p, g->g.adj.p, kind, f.p);
    TG_CHECK_LAUNCH();
    ++tgb::g_launches;
  }
  for (int r = 0; r < T.size; ++r)
    T.broadcast(f.p + o.a[r], (size_t)(o.a[r + 1] - o.a[r]) * 8, r, s);
}

// compute_boundaries(node_costs(kind), p = N) (partition.hpp:116-141)
std::vector<uint32_t> plan_from_costs(const DBuf<uint64_t>& f, uint64_t n, uint64_t p,
                                      cudaStream_t s) {
  if (!n) return std::vector<uint32_t>(p + 1, 0);
  DBuf<uint64_t> pre(n, s);
  tgb::cub_run(s, [&](void* t, size_t& b) {
    return cub::DeviceScan::InclusiveSum(t, b, f.p, pre.p, (int64_t)n, s);
  });
  ++tgb::g_launches;
  return tgb::boundaries_from_prefix(pre.p, n, p, s);
}

// Σ f over [b_i, b_{i+1}) for every core i (every rank has all of f)
std::vector<uint64_t> core_sums(const DBuf<uint64_t>& f, uint64_t n,
                                const std::vector<uint32_t>& b, cudaStream_t s) {
  const size_t p = b.size() - 1;
  std::vector<uint64_t> out(p, 0);
  if (!n) return out;
  DBuf<uint64_t> pre(n, s);
  tgb::cub_run(s, [&](void* t, size_t& bb) {
    return cub::DeviceScan::InclusiveSum(t, bb, f.p, pre.p, (int64_t)n, s);
  });
  for (size_t i = 0; i < p; ++i) {
    const uint64_t hi = b[i + 1] ? tgb::read_u64(pre.p + (b[i + 1] - 1), s) : 0;
    const uint64_t lo = b[i] ? tgb::read_u64(pre.p + (b[i] - 1), s) : 0;
    out[i] = hi - lo;
  }
  return out;
}

std::vector<uint32_t> checked_boundaries(const uint32_t* b_in, uint64_t p, uint64_t n) {
  std::vector<uint32_t> b(b_in, b_in + p + 1);
  TG_REQUIRE(b[0] == 0 && b[p] <= n, "boundaries must start at 0 and end at <= n");
  for (uint64_t i = 0; i < p; ++i) TG_REQUIRE(b[i] <= b[i + 1], "boundaries must be sorted");
  return b;
}

// AOP (engines.hpp:38-54) of this rank over the installed full orientation
void count_core(tg_graph* g, uint32_t cb, uint32_t ce, unsigned long long* d_total,
                unsigned long long* d_tally = nullptr) {
  if (ce <= cb) return;
  const CsrView full = tgh::full_view(g);
  const uint32_t N = (uint32_t)g->g.n;
  if (!d_tally && tgh::window_ready(g)) {
    tgh::window_rows(g, cb, ce, d_total);
  } else {
    tgb::intersect_rows(full, cb, ce, full, 0, N, CountOut{d_total, d_tally, nullptr, nullptr, 0},
                        g->scr, g->stream, g->eff.data.n, true, tgh::rank_view(g));
  }
}

// orientation split + gather + install (AOP input on every rank)
void aop_prepare(tg_graph* g, Transport& T, Oriented& o) {
  orient_mine(g, T, o);
  DevEff full;
  gather_full(g, T, o, full);
  tgh::install_eff(g, std::move(full));
}

}  // namespace

extern "C" {

tg_status tg_comm_unique_id(void* id) {
  return guard([&] {
    TG_REQUIRE(id != nullptr, "null id");
    ncclUniqueId u;
    TG_NCCL(tgb::nccl().GetUniqueId(&u));
    std::memcpy(id, &u, sizeof(u));
  });
}

tg_status tg_comm_init(int device, int nranks, int rank, const void* id, tg_comm** out) {
  return guard([&] {
    TG_REQUIRE(out && id && nranks >= 1 && rank >= 0 && rank < nranks, "invalid argument");
    TG_CUDA(cudaSetDevice(device));
    auto t = std::make_unique<tgb::NcclTransport>();
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    TG_NCCL(tgb::nccl().CommInitRank(&t->comm, nranks, u, rank));
    t->rank = rank;
    t->size = nranks;
    auto* c = new tg_comm;
    c->device = device;
    c->t = std::move(t);
    *out = c;
  });
}

tg_status tg_comm_init_local(int nranks, const int* devices, tg_comm** comms) {
  return guard([&] {
    TG_REQUIRE(nranks >= 1 && devices && comms, "invalid argument");
    auto grp = std::make_shared<tgb::LocalGroup>();
    grp->n = nranks;
    grp->ptr.assign(nranks, nullptr);
    grp->sizes.assign(nranks, std::vector<size_t>(nranks, 0));
    for (int r = 0; r < nranks; ++r) {
      auto t = std::make_unique<tgb::LocalTransport>();
      t->grp = grp;
      t->rank = r;
      t->size = nranks;
      auto* c = new tg_comm;
      c->device = devices[r];
      c->t = std::move(t);
      comms[r] = c;
    }
  });
}

tg_status tg_comm_free(tg_comm* c) {
  if (!c) return TG_OK;
  return guard([&] {
    cudaSetDevice(c->device);
    delete c;
  });
}

tg_status tg_comm_info(tg_comm* c, int32_t* nranks, int32_t* rank) {
  return guard([&] {
    TG_REQUIRE(c != nullptr, "null communicator");
    if (nranks) *nranks = c->t->size;
    if (rank) *rank = c->t->rank;
  });
}

tg_status tg_graph_from_rows(int device, uint64_t n, uint32_t row_lo, uint32_t row_hi,
                             const uint64_t* offsets, const uint32_t* adj,
                             const uint32_t* degrees, tg_graph** out) {
  return guard([&] {
    TG_REQUIRE(out && degrees && (offsets || row_hi == row_lo), "null argument");
    TG_REQUIRE(n <= 0xFFFFFFFFull && row_lo <= row_hi && row_hi <= n, "invalid row range");
    TG_REQUIRE(!tgh::is_device_ptr(offsets) && !tgh::is_device_ptr(degrees),
               "tg_graph_from_rows takes host offsets / degrees");
    const uint64_t rows = row_hi - row_lo;
    for (uint64_t r = 0; r < rows; ++r) {
      TG_REQUIRE(offsets[r] <= offsets[r + 1], "offsets must be sorted");
      TG_REQUIRE(offsets[r + 1] - offsets[r] == degrees[row_lo + r],
                 "degrees must match the rows' lengths");
    }
    const uint64_t o0 = rows ? offsets[0] : 0;
    const uint64_t E = rows ? offsets[rows] - o0 : 0;
    TG_REQUIRE(adj != nullptr || E == 0, "null adjacency");
    // offsets over all n vertices: rows outside [row_lo, row_hi) are empty
    std::vector<uint64_t> off(n + 1, 0);
    for (uint64_t v = 0; v <= n; ++v)
      off[v] = v <= row_lo ? 0 : (v <= row_hi ? offsets[v - row_lo] - o0 : E);
    tg_graph* h = tgh::new_graph(device);
    try {
      cudaStream_t s = h->stream;
      h->g.n = n;
      h->g.m2 = E;
      h->g.off.alloc(n + 1, s);
      TG_CUDA(cudaMemcpyAsync(h->g.off.p, off.data(), (n + 1) * 8, cudaMemcpyHostToDevice, s));
      h->g.adj.alloc(E ? E : 1, s);
      if (E) TG_CUDA(cudaMemcpyAsync(h->g.adj.p, adj, E * 4, cudaMemcpyDefault, s));
      // the GLOBAL degrees: the orientation keys of rows held elsewhere
      h->g.deg.alloc(n ? n : 1, s);
      h->g.dcode.alloc(n ? n : 1, s);
      if (n) {
        TG_CUDA(cudaMemcpyAsync(h->g.deg.p, degrees, n * 4, cudaMemcpyHostToDevice, s));
        tgb::k_dcode<<<tgb::grid_for(n, 256), 256, 0, s>>>(h->g.deg.p, n, h->g.dcode.p);
        TG_CHECK_LAUNCH();
        ++tgb::g_launches;
      }
      h->partial = true;
      h->row_lo = row_lo;
      h->row_hi = row_hi;
      TG_CUDA(cudaStreamSynchronize(s));  // the host buffers die on return
    } catch (...) {
      tg_graph_free(h);
      throw;
    }
    *out = h;
  });
}

tg_status tg_orient_rows_device(tg_graph* g, uint32_t row_lo, uint32_t row_hi, uint64_t* entries) {
  return guard([&] {
    tgh::enter(g);
    TG_REQUIRE(row_lo <= row_hi && row_hi <= g->g.n, "invalid row range");
    TG_REQUIRE(!g->partial || (row_lo >= g->row_lo && row_hi <= g->row_hi),
               "rows outside the rank-local graph");
    DevEff slice;
    if (row_lo % 32 == 0 && (row_hi % 32 == 0 || row_hi == g->g.n))
      tgb::orient_rows_tiles(g->g, row_lo, row_hi, slice, g->stream);
    else
      tgb::orient_rows(g->g, row_lo, row_hi, slice, g->stream);
    if (entries) *entries = slice.entries;
  });
}

tg_status tg_aop_step_comm(tg_graph* g, tg_comm* c, const uint32_t* boundaries, uint64_t* d_total) {
  return guard([&] {
    tgh::enter(g);
    TG_REQUIRE(c && boundaries && d_total, "null argument");
    Transport& T = *c->t;
    const int N = T.size, r = T.rank;
    const uint64_t n = g->g.n;
    const auto b = checked_boundaries(boundaries, N, n);
    cudaStream_t s = g->stream;
    // own rows oriented, every list length gathered: the compact layout of
    // the full oriented CSR (offsets, descriptors) is fixed before any list
    // arrives
    Oriented o;
    orient_mine(g, T, o);
    uint64_t m = 0;
    std::vector<uint64_t> base(N);
    for (int k = 0; k < N; ++k) {
      base[k] = m;
      m += o.cnt[k];
    }
    DevEff full;
    full.rows = n;
    full.base = 0;
    full.compact = true;
    full.entries = m;
    offsets_from_lens(o.lens, n, full.off, s);
    full.desc.alloc(n ? n : 1, s);
    if (n) {
      tgb::k_desc_from_off2<<<tgb::grid_for(n, 256), 256, 0, s>>>(full.off.p, n, full.desc.p);
      TG_CHECK_LAUNCH();
      ++tgb::g_launches;
    }
    // Slab layout for the count (slab.cuh) when the gathered lists suit it
    // (the rule of engine.cu orient, decided once per order): the lists are
    // received behind the n slabs and each slice's slabs are filled on
    // arrival (one streaming pass over the slice, under the next transfer).
    if (g->comm_slab < 0) {
      g->comm_slab = 0;
      const int mode = tgb::g_slab_mode & 255;
      if (mode != 2 && n && n < 0xffffffffull) {
        const tgb::SlabStats st = tgb::slab_stats(g->g, full, s);
        const bool fits = n * tgb::kSlab + m + tgb::kQuadPad < (1ull << 34);
        const bool pays = m > 16 * n && st.long_entries * 50 <= m && st.max_len <= 4096;
        if (fits && (pays || mode == 1)) g->comm_slab = 1;
      }
    }
    const uint64_t lb = g->comm_slab == 1 ? n * tgb::kSlab : 0;  // first list slot
    if (lb) {
      full.slab = tgb::kSlab;
      tgb::k_desc_from_off2<<<tgb::grid_for(n, 256), 256, 0, s>>>(full.off.p, n, full.desc.p, lb);
      TG_CHECK_LAUNCH();
      ++tgb::g_launches;
    }
    full.data.alloc(lb + m + tgb::kQuadPad, s);
    TG_CUDA(cudaMemsetAsync(full.data.p + lb + m, 0, tgb::kQuadPad * 4, s));
    if (o.slice.entries)
      TG_CUDA(cudaMemcpyAsync(full.data.p + lb + base[r], o.slice.data.p, o.slice.entries * 4,
                              cudaMemcpyDeviceToDevice, s));
    // the slices arrive in rank order (= id order) on a transfer stream; after
    // slice k, every apex of this rank's core whose lists all arrived --
    // ready chunk max(chunk(v), chunk(last of N_v)), lists being ID-sorted --
    // is counted on the compute stream while slice k+1 is in flight
    const uint32_t cb = b[r], ce = b[r + 1];
    DBuf<uint32_t> d_a(N + 1, s), ids(ce > cb ? ce - cb : 1, s);
    DBuf<uint8_t> ready(n ? n : 1, s);
    DBuf<unsigned long long> cnt(1, s);
    TG_CUDA(cudaMemcpyAsync(d_a.p, o.a.data(), (N + 1) * 4, cudaMemcpyHostToDevice, s));
    TG_CUDA(cudaMemsetAsync(ready.p, 0xff, n ? n : 1, s));
    TG_CUDA(cudaMemsetAsync(d_total, 0, 8, s));
    cudaStream_t xs;
    cudaEvent_t ev_c, ev_x;
    TG_CUDA(cudaStreamCreateWithFlags(&xs, cudaStreamNonBlocking));
    TG_CUDA(cudaEventCreateWithFlags(&ev_c, cudaEventDisableTiming));
    TG_CUDA(cudaEventCreateWithFlags(&ev_x, cudaEventDisableTiming));
    TG_CUDA(cudaEventRecord(ev_c, s));  // own slice in place
    TG_CUDA(cudaStreamWaitEvent(xs, ev_c, 0));
    const CsrView fv = tgh::view(full);
    try {
      for (int k = 0; k < N; ++k) {
        T.broadcast(full.data.p + lb + base[k], o.cnt[k] * 4, k, xs);
        TG_CUDA(cudaEventRecord(ev_x, xs));
        TG_CUDA(cudaStreamWaitEvent(s, ev_x, 0));
        if (lb) tgb::slab_rows(full, o.a[k], o.a[k + 1], s);
        const uint32_t vb = std::max(o.a[k], cb), ve = std::min(o.a[k + 1], ce);
        tgb::ready_chunks(full, d_a.p, (uint32_t)N, (uint32_t)k, vb, ve, ready.p, s);
        if (ce > cb) {
          tgb::select_ready(ready.p, cb, ce, (uint32_t)k, ids.p, cnt.p, s);
          tgb::intersect_list(fv, ids.p, cnt.p, ce - cb, fv,
                              CountOut{(unsigned long long*)d_total, nullptr, nullptr, nullptr, 0},
                              g->scr, s, full.data.n);
        }
      }
    } catch (...) {
      cudaStreamSynchronize(xs);
      cudaStreamDestroy(xs);
      cudaEventDestroy(ev_c);
      cudaEventDestroy(ev_x);
      throw;
    }
    TG_CUDA(cudaStreamSynchronize(xs));
    TG_CUDA(cudaStreamDestroy(xs));
    TG_CUDA(cudaEventDestroy(ev_c));
    TG_CUDA(cudaEventDestroy(ev_x));
    T.all_reduce_u64(d_total, 1, s);
    tgh::install_eff(g, std::move(full));
  });
}

tg_status tg_run_engine_comm(tg_graph* g, tg_comm* c, const tg_config* cfg, uint64_t* total,
                             tg_rank_stats* per_rank, uint32_t* boundaries_out) {
  return guard([&] {
    tgh::enter(g);
    TG_REQUIRE(c && cfg, "null argument");
    TG_REQUIRE(cfg->engine == TG_ENGINE_AOP || cfg->engine == TG_ENGINE_ANOP_SURROGATE ||
                   cfg->engine == TG_ENGINE_ANOP_DIRECT,
               "across ranks: Aop, AnopDirect and AnopSurrogate");
    TG_REQUIRE(cfg->cost >= TG_COST_N && cfg->cost <= TG_COST_NOV, "unknown cost kind");
    TG_REQUIRE(!cfg->sparsify && !cfg->track_nodes && !cfg->collect_triangles,
               "across ranks: counts only (tallies via tg_clustering_comm)");
    TG_REQUIRE(cfg->ranks == 0 || cfg->ranks == (uint64_t)c->t->size,
               "cfg->ranks must equal the communicator size");
    TG_REQUIRE(!cfg->order_set || cfg->order == TG_ORDER_BY_DEGREE,
               "across ranks: the degree order");
    Transport& T = *c->t;
    const int N = T.size, r = T.rank;
    const uint64_t n = g->g.n;
    cudaStream_t s = g->stream;
    Oriented o;
    std::vector<uint32_t> b;
    DBuf<unsigned long long> ctr(1, s);
    ctr.zero();
    tg_rank_stats mine{0, 0, 0, 0, 0};
    if (cfg->engine == TG_ENGINE_AOP) {
      aop_prepare(g, T, o);  // every rank: the full orientation
      DBuf<uint64_t> fc;
      if (cfg->boundaries) {
        b = checked_boundaries(cfg->boundaries, N, n);
      } else {
        gather_costs(g, T, o, cfg->cost, fc, s);
        b = plan_from_costs(fc, n, N, s);
      }
      count_core(g, b[r], b[r + 1], ctr.p);
      mine.triangles = tgb::read_u64((const uint64_t*)ctr.p, s);
      mine.stored_entries =
          b[r + 1] > b[r] ? tgb::overlap_stored_entries(tgh::full_view(g), n, b[r], b[r + 1], s) : 0;
      DBuf<uint64_t> f;
      gather_costs(g, T, o, TG_COST_DPD, f, s);
      mine.realized_cost = core_sums(f, n, b, s)[r];
    } else {
      // ANOP (direct or surrogate): lengths + distributed costs -> plan;
      // oriented rows to their core owner (partition.hpp:210-239); then the
      // engine's exchange
      orient_mine(g, T, o);
      DBuf<uint64_t> f;
      if (cfg->boundaries) {
        b = checked_boundaries(cfg->boundaries, N, n);
      } else {
        gather_costs(g, T, o, cfg->cost, f, s);
        b = plan_from_costs(f, n, N, s);
      }
      DBuf<uint64_t> goff;
      offsets_from_lens(o.lens, n, goff, s);
      auto at = [&](uint32_t v) { return tgb::read_u64(goff.p + v, s); };
      const uint32_t lo = o.a[r], hi = o.a[r + 1], cb = b[r], ce = b[r + 1];
      // rows of rank i's slice that lie in core j move from i to j
      std::vector<size_t> sb(N, 0), rb(N, 0);
      for (int j = 0; j < N; ++j) {
        const uint32_t x0 = std::max(lo, b[j]), x1 = std::min(hi, b[j + 1]);
        if (x1 > x0) sb[j] = (at(x1) - at(x0)) * 4;
        const uint32_t y0 = std::max(o.a[j], cb), y1 = std::min(o.a[j + 1], ce);
        if (y1 > y0) rb[j] = (at(y1) - at(y0)) * 4;
      }
      DevEff part;
      part.rows = ce - cb;
      part.base = cb;
      part.compact = true;
      part.entries = ce > cb ? at(ce) - at(cb) : 0;
      part.data.alloc(part.entries + tgb::kQuadPad, s);
      TG_CUDA(cudaMemsetAsync(part.data.p + part.entries, 0, tgb::kQuadPad * 4, s));
      // the slice's rows are ID-ordered, so its segment for core j (rows
      // [max(lo, b_j), min(hi, b_{j+1}))) follows the one for core j-1; the
      // received segments arrive in rank order = core rows in ID order
      T.all_to_allv(o.slice.data.p, sb, part.data.p, rb, s);
      part.off.alloc(part.rows + 1, s);
      TG_CUDA(cudaMemsetAsync(part.off.p, 0, 8, s));
      if (part.rows) {
        DBuf<uint64_t> l64(part.rows, s);
        tgb::k_u32_to_u64<<<tgb::grid_for(part.rows, 256), 256, 0, s>>>(o.lens.p + cb, part.rows, l64.p);
        TG_CHECK_LAUNCH();
        tgb::cub_run(s, [&](void* t, size_t& bb) {
          return cub::DeviceScan::InclusiveSum(t, bb, l64.p, part.off.p + 1, (int64_t)part.rows, s);
        });
        part.desc.alloc(part.rows, s);
        tgb::k_desc_from_off2<<<tgb::grid_for(part.rows, 256), 256, 0, s>>>(part.off.p, part.rows,
                                                                           part.desc.p);
        TG_CHECK_LAUNCH();
        tgb::g_launches += 3;
      } else {
        part.desc.alloc(1, s);
      }
      mine.stored_entries = part.entries;
      if (cfg->engine == TG_ENGINE_ANOP_DIRECT) {
        // anop_direct_body (engines.hpp:80-141), batched: every off-core pair
        // (v, u) is one request to owner(u) and one reply carrying N_u; the
        // requester intersects N_v with each reply.  Three exchanges: the
        // requested ids, the reply lengths, the reply lists.
        const CsrView pv = tgh::view(part);
        const CountOut out{ctr.p, nullptr, nullptr, nullptr, 0};
        DBuf<uint32_t> gb(N + 1, s);
        TG_CUDA(cudaMemcpyAsync(gb.p, b.data(), (N + 1) * 4, cudaMemcpyHostToDevice, s));
        DBuf<unsigned long long> cur(N, s);
        cur.zero();
        const unsigned grid = tgb::grid_for((uint64_t)(ce - cb) * 32, 256, 148u * 16u);
        if (ce > cb) {
          tgb::k_direct_requests<false><<<grid, 256, 0, s>>>(pv, cb, ce, gb.p, (uint32_t)N,
                                                             (uint32_t)r, cur.p, nullptr, nullptr);
          TG_CHECK_LAUNCH();
          ++tgb::g_launches;
        }
        std::vector<uint64_t> cnt(N, 0);
        TG_CUDA(cudaMemcpyAsync(cnt.data(), cur.p, N * 8, cudaMemcpyDeviceToHost, s));
        TG_CUDA(cudaStreamSynchronize(s));
        auto all_cnt = all_gather_host(T, cnt, s);  // [i][j] = requests from i to j
        std::vector<uint64_t> start(N + 1, 0), rstart(N + 1, 0);
        std::vector<size_t> sq(N), rq(N);
        for (int j = 0; j < N; ++j) {
          start[j + 1] = start[j] + cnt[j];
          rstart[j + 1] = rstart[j] + all_cnt[(size_t)j * N + r];
          sq[j] = cnt[j] * 4;
          rq[j] = all_cnt[(size_t)j * N + r] * 4;
        }
        const uint64_t Rs = start[N], Rr = rstart[N];  // requests sent / received
        DBuf<uint32_t> req_u(Rs + 1, s), req_v(Rs + 1, s), got_u(Rr + 1, s);
        TG_CUDA(cudaMemcpyAsync(cur.p, start.data(), N * 8, cudaMemcpyHostToDevice, s));
        if (ce > cb) {
          tgb::k_direct_requests<true><<<grid, 256, 0, s>>>(pv, cb, ce, gb.p, (uint32_t)N,
                                                            (uint32_t)r, cur.p, req_u.p, req_v.p);
          TG_CHECK_LAUNCH();
          ++tgb::g_launches;
        }
        T.all_to_allv(req_u.p, sq, got_u.p, rq, s);
        // replies: lengths first (their sizes are the request counts, reversed)
        DBuf<uint32_t> my_lens(Rr + 1, s), rl(Rs + 1, s);
        if (Rr) {
          tgb::k_reply_lens<<<tgb::grid_for(Rr, 256), 256, 0, s>>>(pv, got_u.p, Rr, my_lens.p);
          TG_CHECK_LAUNCH();
          ++tgb::g_launches;
        }
        T.all_to_allv(my_lens.p, rq, rl.p, sq, s);
        auto scan = [&](const DBuf<uint32_t>& l, uint64_t cntl, DBuf<uint64_t>& off) {
          off.alloc(cntl + 1, s);
          TG_CUDA(cudaMemsetAsync(off.p, 0, 8, s));
          if (!cntl) return;
          DBuf<uint64_t> l64(cntl, s);
          tgb::k_u32_to_u64<<<tgb::grid_for(cntl, 256), 256, 0, s>>>(l.p, cntl, l64.p);
          TG_CHECK_LAUNCH();
          tgb::cub_run(s, [&](void* t, size_t& bb) {
            return cub::DeviceScan::InclusiveSum(t, bb, l64.p, off.p + 1, (int64_t)cntl, s);
          });
          tgb::g_launches += 2;
        };
        DBuf<uint64_t> soff, roff;  // reply offsets: the ones I serve, the ones I receive
        scan(my_lens, Rr, soff);
        scan(rl, Rs, roff);
        std::vector<size_t> sp(N), rp(N);
        for (int j = 0; j < N; ++j) {
          sp[j] = (tgb::read_u64(soff.p + rstart[j + 1], s) - tgb::read_u64(soff.p + rstart[j], s)) * 4;
          rp[j] = (tgb::read_u64(roff.p + start[j + 1], s) - tgb::read_u64(roff.p + start[j], s)) * 4;
        }
        const uint64_t sw = tgb::read_u64(soff.p + Rr, s), rw = tgb::read_u64(roff.p + Rs, s);
        size_t mfree = 0, mtot = 0;
        TG_CUDA(cudaMemGetInfo(&mfree, &mtot));
        TG_REQUIRE((sw + rw) * 4 + (64ull << 20) < mfree,
                   "AnopDirect: the reply lists of this rank do not fit the device (one list per "
                   "off-core pair, engines.hpp:80-141); use AnopSurrogate");
        DBuf<uint32_t> pay(sw + 1, s), rpay(rw + 1, s);
        if (Rr) {
          tgb::k_reply_fill<<<tgb::grid_for(Rr * 32, 256, 148u * 16u), 256, 0, s>>>(pv, got_u.p, Rr,
                                                                                  soff.p, pay.p);
          TG_CHECK_LAUNCH();
          ++tgb::g_launches;
        }
        T.all_to_allv(pay.p, sp, rpay.p, rp, s);
        if (ce > cb) {
          // in-core pairs locally, off-core pairs against their replies
          tgb::intersect_rows(pv, cb, ce, pv, cb, ce, out, g->scr, s, part.data.n, false);
          if (Rs) {
            tgb::k_direct_count<<<tgb::grid_for(Rs * 32, 256, 148u * 16u), 256, 0, s>>>(
                pv, req_v.p, Rs, roff.p, rpay.p, ctr.p);
            TG_CHECK_LAUNCH();
            ++tgb::g_launches;
          }
        }
        mine.triangles = tgb::read_u64((const uint64_t*)ctr.p, s);
        mine.data_sent = Rs + Rr;  // requests sent + replies sent
        mine.data_recv = Rr + Rs;  // requests received + replies received
        DBuf<uint64_t> fd;
        gather_costs(g, T, o, TG_COST_DPD, fd, s);
        mine.realized_cost = core_sums(fd, n, b, s)[r];
      } else {
      // SurrogatePack (engines.hpp:173-187) + the exchange of (v, N_v)
      tgb::SurrogatePack pack;
      pack.build(tgh::view(part), cb, ce, b, (uint32_t)r, s);
      std::vector<uint64_t> mw(2 * N);
      for (int j = 0; j < N; ++j) {
        mw[2 * j] = pack.msgs_per_dest[j];
        mw[2 * j + 1] = pack.words_per_dest[j];
      }
      auto all_mw = all_gather_host(T, mw, s);  // [i][j] = (msgs, words) from i to j
      std::vector<size_t> sh(N), sd(N), rh(N), rd(N);
      uint64_t msgs = 0, words = 0, rmsgs = 0, rwords = 0;
      for (int j = 0; j < N; ++j) {
        sh[j] = pack.msgs_per_dest[j] * 8;
        sd[j] = pack.words_per_dest[j] * 4;
        msgs += pack.msgs_per_dest[j];
        words += pack.words_per_dest[j];
        rh[j] = all_mw[(size_t)j * 2 * N + 2 * r] * 8;
        rd[j] = all_mw[(size_t)j * 2 * N + 2 * r + 1] * 4;
        rmsgs += all_mw[(size_t)j * 2 * N + 2 * r];
        rwords += all_mw[(size_t)j * 2 * N + 2 * r + 1];
      }
      DBuf<uint32_t> hdr(2 * msgs + 1, s), dat(words + 1, s), rhdr(2 * rmsgs + 1, s),
          rdat(rwords + 1, s);
      pack.scatter(hdr.p, dat.p, s);
      T.all_to_allv(hdr.p, sh, rhdr.p, rh, s);
      T.all_to_allv(dat.p, sd, rdat.p, rd, s);
      mine.data_sent = msgs - pack.msgs_per_dest[r];
      mine.data_recv = rmsgs - all_mw[(size_t)r * 2 * N + 2 * r];
      DBuf<uint64_t> moff;
      tgb::message_offsets(rhdr.p, rmsgs, moff, s);
      const CsrView pv = tgh::view(part);
      const CountOut out{ctr.p, nullptr, nullptr, nullptr, 0};
      if (ce > cb) {
        tgb::intersect_rows(pv, cb, ce, pv, cb, ce, out, g->scr, s, part.data.n, false);
        if (rmsgs) {
          tgb::MsgView mv{rhdr.p, moff.p, rdat.p, rmsgs};
          tgb::intersect_msgs(mv, pv, cb, ce, out, g->scr, s, part.data.n);
        }
      }
      mine.triangles = tgb::read_u64((const uint64_t*)ctr.p, s);
      DBuf<uint64_t> fn;
      gather_costs(g, T, o, TG_COST_NOV, fn, s);
      mine.realized_cost = core_sums(fn, n, b, s)[r];
      }
    }
    auto st = all_gather_host(
        T, {mine.triangles, mine.data_sent, mine.data_recv, mine.realized_cost, mine.stored_entries},
        s);
    uint64_t tot = 0;
    for (int i = 0; i < N; ++i) {
      tot += st[5 * i];
      if (per_rank)
        per_rank[i] = tg_rank_stats{st[5 * i], st[5 * i + 1], st[5 * i + 2], st[5 * i + 3],
                                    st[5 * i + 4]};
    }
    if (total) *total = tot;
    if (boundaries_out) std::memcpy(boundaries_out, b.data(), b.size() * 4);
  });
}

tg_status tg_clustering_comm(tg_graph* g, tg_comm* c, const tg_config* cfg,
                             uint32_t* boundaries_out, uint64_t* tally_core, double* cc_core) {
  return guard([&] {
    tgh::enter(g);
    TG_REQUIRE(c && cfg, "null argument");
    TG_REQUIRE(cfg->cost >= TG_COST_N && cfg->cost <= TG_COST_NOV, "unknown cost kind");
    Transport& T = *c->t;
    const int N = T.size, r = T.rank;
    const uint64_t n = g->g.n;
    cudaStream_t s = g->stream;
    Oriented o;
    aop_prepare(g, T, o);
    std::vector<uint32_t> b;
    if (cfg->boundaries) {
      b = checked_boundaries(cfg->boundaries, N, n);
    } else {
      DBuf<uint64_t> fc;
      gather_costs(g, T, o, cfg->cost, fc, s);
      b = plan_from_costs(fc, n, N, s);
    }
    DBuf<unsigned long long> ctr(1, s), tv(n ? n : 1, s);
    ctr.zero();
    tv.zero();
    // RankSink tallies of this rank's apexes at all three corners
    // (engines.hpp:303-321), then each core range summed at its owner
    // (aggregate_clustering's Tally messages, engines.hpp:229-254)
    count_core(g, b[r], b[r + 1], ctr.p, tv.p);
    for (int j = 0; j < N; ++j)
      T.reduce_u64((uint64_t*)tv.p + b[j], b[j + 1] - b[j], j, s);
    const uint32_t cb = b[r], ce = b[r + 1];
    if (ce > cb) {
      DBuf<double> cc(ce - cb, s);
      tgb::k_cc_range<<<tgb::grid_for(ce - cb, 256), 256, 0, s>>>(g->g.deg.p, tv.p + cb, cb, ce, cc.p);
      TG_CHECK_LAUNCH();
      ++tgb::g_launches;
      if (tally_core)
        TG_CUDA(cudaMemcpyAsync(tally_core, tv.p + cb, (ce - cb) * 8, cudaMemcpyDefault, s));
      if (cc_core) TG_CUDA(cudaMemcpyAsync(cc_core, cc.p, (ce - cb) * 8, cudaMemcpyDefault, s));
      TG_CUDA(cudaStreamSynchronize(s));
    }
    if (boundaries_out) std::memcpy(boundaries_out, b.data(), b.size() * 4);
  });
}

}  // extern "C"
