// bc.cu -- batched Brandes betweenness (algo/betweenness.cpp:11-86).
//
// The reference keeps ns x n matrices P (path counts), one boolean pattern per
// BFS level and B = 1 + dependency, and runs Gustavson mxm per level forward
// (F<!s(P)> = F plus.first A) and backward (W<s(S[i-1])> = W plus.first AT)
// (betweenness.cpp:27-72).  On the device the batch rows become lanes of a
// vertex-major layout -- level[v][b] (int32), sigma[v][b] and delta[v][b]
// (fp64) -- so one gather of a vertex fetches all sources' state in one
// sector, and every level of the batch is ONE kernel over the union frontier:
//   forward: push over A from the (vertex, <=1024-edge chunk) entries of the
//     previous level; a lane claims an unvisited vertex with atomicCAS on its
//     level word and adds its sigma with fp64 atomicAdd (path counts are
//     integers < 2^53, so the sum is exact and order-independent);
//   backward, level d = D-1..1: for u on level d, acc_b = sum over out-
//     neighbours v on level d+1 of coef_b(v) = (1 + delta_b(v)) / sigma_b(v);
//     then delta_b(u) = sigma_b(u) * acc_b, centrality(u) += delta_b(u), and
//     coef_b(u) replaces delta_b(u) for the next level down.
// centrality(j) = sum_b (B(b,j) - 1) = sum_b delta_b(j) (betweenness.cpp:74-79);
// sources and unreached vertices contribute 0, undirected pairs not halved.
// Algorithmic bytes per batch: E_r*(8 + 16*ns) + V_r*(16 + 24*ns).
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "plans.cuh"
#include "warpqueue.cuh"

namespace gbx {

constexpr int kBcLanes = 4;
constexpr int64_t kBcChunk = 1024;
constexpr unsigned kAll = 0xffffffffu;

__device__ __forceinline__ int bc_chunks(int64_t deg) {
  return deg <= kBcChunk ? 1 : static_cast<int>((deg + kBcChunk - 1) / kBcChunk);
}

struct BcArgs {
  const int64_t* rp;
  const int32_t* col;
  int32_t* level;    // [n][4]
  double* sigma;     // [n][4]
  double* delta;     // [n][4]: coef (1 + delta) / sigma once final
  double* acc;       // [n][4]: backward accumulator
  int32_t* mark;     // [n]: last level that listed the vertex
  int32_t* list_out; // vertices of the level being built
  const int64_t* ent_in;
  int64_t* ent_out;
  int* cnt;          // [0] list size [1] entries size
  int n_ent;
  int d;
  int lanes;
};

__global__ void __launch_bounds__(256) k_bc_forward(BcArgs a) {
  __shared__ int32_t s_buf[8][256];
  FrontierQueue<256> fq;
  fq.buf = s_buf[threadIdx.x >> 5];
  fq.rp = a.rp;
  fq.chunk = kBcChunk;
  fq.reset(a.ent_out, &a.cnt[1], &a.cnt[0], nullptr, a.list_out);
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int d = a.d;
  for (int64_t e = gwarp; e < a.n_ent; e += nwarps) {
    const int64_t ent = a.ent_in[e];
    const int32_t u = static_cast<int32_t>(ent & 0xffffffff);
    const int64_t c = ent >> 32;
    const int4 lu = *reinterpret_cast<const int4*>(a.level + static_cast<int64_t>(u) * 4);
    const int lv_u[4] = {lu.x, lu.y, lu.z, lu.w};
    double su[4];
    unsigned m = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      su[b] = a.sigma[static_cast<int64_t>(u) * 4 + b];
      if (b < a.lanes && lv_u[b] == d - 1) m |= 1u << b;
    }
    const int64_t b0 = a.rp[u] + c * kBcChunk;
    const int64_t e0 = min(a.rp[u + 1], b0 + kBcChunk);
    for (int64_t base = b0; base < e0; base += 32) {
      const int64_t p = base + lane;
      bool claimed = false;
      int32_t v = 0;
      if (p < e0 && m) {
        v = __ldg(a.col + p);
        int32_t* lvp = a.level + static_cast<int64_t>(v) * 4;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          if (!(m & (1u << b))) continue;
          int lv = *(volatile int32_t*)&lvp[b];
          if (lv == -1) {
            lv = atomicCAS(&lvp[b], -1, d);
            if (lv == -1) { claimed = true; lv = d; }
          }
          if (lv == d) atomicAdd(&a.sigma[static_cast<int64_t>(v) * 4 + b], su[b]);
        }
      }
      const bool has = claimed && atomicExch(&a.mark[v], d) != d;
      fq.push(has, v);
    }
  }
  fq.flush();
}

// backward accumulation for the entries of level d
__global__ void k_bc_backward(BcArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int d = a.d;
  for (int64_t e = gwarp; e < a.n_ent; e += nwarps) {
    const int64_t ent = a.ent_in[e];
    const int32_t u = static_cast<int32_t>(ent & 0xffffffff);
    const int64_t c = ent >> 32;
    const int4 lu = *reinterpret_cast<const int4*>(a.level + static_cast<int64_t>(u) * 4);
    const int lv_u[4] = {lu.x, lu.y, lu.z, lu.w};
    unsigned m = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b)
      if (b < a.lanes && lv_u[b] == d) m |= 1u << b;
    const int64_t b0 = a.rp[u] + c * kBcChunk;
    const int64_t e0 = min(a.rp[u + 1], b0 + kBcChunk);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t p = b0 + lane; p < e0; p += 32) {
      const int32_t v = __ldg(a.col + p);
      const int4 lvv = *reinterpret_cast<const int4*>(a.level + static_cast<int64_t>(v) * 4);
      const int lv[4] = {lvv.x, lvv.y, lvv.z, lvv.w};
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if ((m & (1u << b)) && lv[b] == d + 1) acc[b] += a.delta[static_cast<int64_t>(v) * 4 + b];
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[b] += __shfl_xor_sync(kAll, acc[b], o);
    }
    if (lane == 0) {
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if ((m & (1u << b)) && acc[b] != 0.0)
          atomicAdd(&a.acc[static_cast<int64_t>(u) * 4 + b], acc[b]);
    }
  }
}

// finalize level d: delta = sigma * acc; centrality += delta; coef replaces delta
__global__ void k_bc_finalize(const int32_t* list, int nlist, int d, int lanes,
                              const int32_t* level, const double* sigma, double* delta,
                              const double* acc, double* cent) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= nlist) return;
  const int64_t u = list[i];
  double c = 0.0;
  for (int b = 0; b < lanes; ++b) {
    if (level[u * 4 + b] != d) continue;
    const double s = sigma[u * 4 + b];
    const double dl = s * acc[u * 4 + b];
    c += dl;
    delta[u * 4 + b] = (1.0 + dl) / s;
  }
  cent[u] += c;
}

// deepest level: delta = 0, coef = 1 / sigma
__global__ void k_bc_leaf(const int32_t* list, int nlist, int d, int lanes, const int32_t* level,
                          const double* sigma, double* delta) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= nlist) return;
  const int64_t u = list[i];
  for (int b = 0; b < lanes; ++b)
    if (level[u * 4 + b] == d) delta[u * 4 + b] = 1.0 / sigma[u * 4 + b];
}

// rebuild the chunk entries of a level list
__global__ void k_bc_entries(const int32_t* list, int nlist, const int64_t* rp, int64_t* ent,
                             int* cnt) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= nlist) return;
  const int32_t v = list[i];
  const int k = bc_chunks(rp[v + 1] - rp[v]);
  const int off = atomicAdd(cnt, k);
  for (int c = 0; c < k; ++c) ent[off + c] = (static_cast<int64_t>(c) << 32) | v;
}

__global__ void k_bc_init(int32_t* level, double* sigma, double* delta, int32_t* mark,
                          double* acc, int64_t n) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n * 4) { level[i] = -1; sigma[i] = 0.0; delta[i] = 0.0; acc[i] = 0.0; }
  if (i < n) mark[i] = -1;
}

__global__ void k_bc_seed(const int32_t* src, int ns, int32_t* level, double* sigma,
                          int32_t* mark, int32_t* list, int64_t* ent, int* cnt, const int64_t* rp) {
  int nl = 0, ne = 0;
  for (int b = 0; b < ns; ++b) {
    const int64_t s = src[b];
    level[s * 4 + b] = 0;
    sigma[s * 4 + b] = 1.0;
    if (mark[s] != 0) {
      mark[s] = 0;
      list[nl++] = static_cast<int32_t>(s);
      const int k = bc_chunks(rp[s + 1] - rp[s]);
      for (int c = 0; c < k; ++c) ent[ne++] = (static_cast<int64_t>(c) << 32) | s;
    }
  }
  cnt[0] = nl;
  cnt[1] = ne;
}

void bc_run(gbx_graph* g, const uint64_t* sources, uint64_t ns, double* centrality) {
  const int64_t n = g->A.n;
  for (uint64_t b = 0; b < ns; ++b)
    if (sources[b] >= static_cast<uint64_t>(n))
      fail(GBX_SOURCE_OUT_OF_RANGE, "source " + std::to_string(sources[b]));
  if (!g->bc) g->bc = std::make_unique<BcWork>();
  BcWork& W = *g->bc;
  cudaStream_t s = g->stream;
  const Csr& A = g->A;
  const int64_t n1 = std::max<int64_t>(n, 1);
  if (W.n != n || !W.level.p) {
    W.n = n;
    W.lanes = kBcLanes;
    W.level.alloc(n1 * 4);
    W.sigma.alloc(n1 * 4);
    W.delta.alloc(n1 * 4);
    W.order.alloc(n1 * 4 + 8);
    W.cent.alloc(n1);
    W.ctl.alloc(4);
  }
  DevArray<int32_t> mark(n1);
  DevArray<double> acc(n1 * 4);
  const int64_t ecap = n + A.nnz / kBcChunk + 64;
  DevArray<int64_t> ent[2];
  ent[0].alloc(ecap);
  ent[1].alloc(ecap);
  DevArray<int32_t> dsrc(4);
  GBX_CUDA(cudaMemsetAsync(W.cent.p, 0, n1 * 8, s));
  const int grid = device_sms() * 16;
  int64_t launches = 1, edges = 0;
  int max_levels = 0;
  for (uint64_t b0 = 0; b0 < ns; b0 += kBcLanes) {
    const int nb = static_cast<int>(std::min<uint64_t>(kBcLanes, ns - b0));
    int32_t hs[4];
    for (int b = 0; b < nb; ++b) hs[b] = static_cast<int32_t>(sources[b0 + b]);
    GBX_CUDA(cudaMemcpyAsync(dsrc.p, hs, nb * 4, cudaMemcpyHostToDevice, s));
    k_bc_init<<<ceil_div(n * 4, 256), 256, 0, s>>>(W.level.p, W.sigma.p, W.delta.p, mark.p,
                                                    acc.p, n);
    k_bc_seed<<<1, 1, 0, s>>>(dsrc.p, nb, W.level.p, W.sigma.p, mark.p, W.order.p, ent[0].p,
                              W.ctl.p, A.rp.p);
    GBX_LAUNCHED();
    launches += 2;
    // ---- forward sweep
    std::vector<int64_t> off = {0};
    int hc[2];
    GBX_CUDA(cudaMemcpyAsync(hc, W.ctl.p, 8, cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaStreamSynchronize(s));
    off.push_back(hc[0]);
    int n_ent = hc[1];
    int cur = 0;
    for (int d = 1; static_cast<int64_t>(d) <= n; ++d) {
      if (off.back() == off[off.size() - 2]) break;
      GBX_CUDA(cudaMemsetAsync(W.ctl.p, 0, 8, s));
      BcArgs a{};
      a.rp = A.rp.p;
      a.col = A.col.p;
      a.level = W.level.p;
      a.sigma = W.sigma.p;
      a.delta = W.delta.p;
      a.mark = mark.p;
      a.list_out = W.order.p + off.back();
      a.ent_in = ent[cur].p;
      a.ent_out = ent[cur ^ 1].p;
      a.cnt = W.ctl.p;
      a.n_ent = n_ent;
      a.d = d;
      a.lanes = nb;
      k_bc_forward<<<grid, 256, 0, s>>>(a);
      GBX_LAUNCHED();
      ++launches;
      GBX_CUDA(cudaMemcpyAsync(hc, W.ctl.p, 8, cudaMemcpyDeviceToHost, s));
      GBX_CUDA(cudaStreamSynchronize(s));
      off.push_back(off.back() + hc[0]);
      n_ent = hc[1];
      cur ^= 1;
    }
    // levels: off[d]..off[d+1] lists vertices with some lane at depth d
    const int D = static_cast<int>(off.size()) - 1;  // depths 0..D-1 (last list may be empty)
    max_levels = std::max(max_levels, D);
    int deepest = D - 1;
    while (deepest > 0 && off[deepest + 1] == off[deepest]) --deepest;
    if (deepest >= 1) {
      const int nl = static_cast<int>(off[deepest + 1] - off[deepest]);
      k_bc_leaf<<<ceil_div(nl, 256), 256, 0, s>>>(W.order.p + off[deepest], nl, deepest, nb,
                                                   W.level.p, W.sigma.p, W.delta.p);
      GBX_LAUNCHED();
      ++launches;
      // the deepest level has delta = 0: nothing to add to the centrality
    }
    for (int d = deepest - 1; d >= 1; --d) {
      const int nl = static_cast<int>(off[d + 1] - off[d]);
      if (nl == 0) continue;
      const int32_t* list = W.order.p + off[d];
      GBX_CUDA(cudaMemsetAsync(W.ctl.p, 0, 4, s));
      k_bc_entries<<<ceil_div(nl, 256), 256, 0, s>>>(list, nl, A.rp.p, ent[0].p, W.ctl.p);
      GBX_LAUNCHED();
      int ne = 0;
      GBX_CUDA(cudaMemcpyAsync(&ne, W.ctl.p, 4, cudaMemcpyDeviceToHost, s));
      GBX_CUDA(cudaStreamSynchronize(s));
      BcArgs a{};
      a.rp = A.rp.p;
      a.col = A.col.p;
      a.level = W.level.p;
      a.sigma = W.sigma.p;
      a.delta = W.delta.p;
      a.ent_in = ent[0].p;
      a.acc = acc.p;
      a.n_ent = ne;
      a.d = d;
      a.lanes = nb;
      k_bc_backward<<<grid, 256, 0, s>>>(a);
      k_bc_finalize<<<ceil_div(nl, 256), 256, 0, s>>>(list, nl, d, nb, W.level.p, W.sigma.p,
                                                       W.delta.p, acc.p, W.cent.p);
      GBX_LAUNCHED();
      launches += 3;
    }
    edges += A.nnz;
  }
  if (centrality) {
    GBX_CUDA(cudaMemcpyAsync(centrality, W.cent.p, n * 8, cudaMemcpyDeviceToHost, s));
  }
  GBX_CUDA(cudaStreamSynchronize(s));
  g->stats = gbx_stats{};
  g->stats.launches = launches;
  g->stats.iterations = max_levels;
  g->stats.work_units = edges;
}

}  // namespace gbx
