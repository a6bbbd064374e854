// pagerank.cu -- GAP PageRank (algo/pagerank.cpp:8-81) as one fused pull-SpMV
// kernel per iteration, looped on the device by a CUDA-graph WHILE node.
//
// Reference per iteration: contrib = prior ./ (deg/damping) (:55-56), rank =
// teleport (:58), rank += AT plus.second contrib (:59-61), L1 = sum|prior -
// rank| (:65-73), stop when L1 < tol (:74).  Here one kernel does all of it:
//   * work is split into merge-path tiles of kPrItems (row-ends + nonzeros) so
//     every CTA does the same amount of work regardless of the in-degree skew
//     (R-MAT hubs have 10^5 in-edges);
//   * a tile stages its AT columns (streamed, evict-first) and the gathered
//     x = contrib values (read-only path, L2-resident: 4n bytes) in shared
//     memory, then each thread consumes kPrIpt merge items sequentially, a
//     block reduce-by-key scan fixes up rows split between threads;
//   * rows split between tiles are finished by the last tile to arrive
//     (per-row epoch counter, parts summed in tile order);
//   * the epilogue is fused: r_new = teleport + sum (fp64), L1 partial
//     |r_prev - r_new| (fp64), x_next = r_new / (deg / damping) (fp32, 0 for
//     dangling vertices -- their mass is lost exactly as in the reference);
//   * the last CTA reduces the per-CTA L1 partials in a fixed order, stores
//     the iteration count and clears the graph's WHILE condition on
//     convergence, so the whole run is one graph launch with no host syncs.
// Algorithmic bytes per iteration: 4*nnz (col) + 4*nnz (gathered
// x) + 8*(n+1) (row_ptr) + 16*n (read r_prev, read deg, write r, write x).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "plans.cuh"

namespace gbx {

constexpr int kPrThreads = 256;
constexpr int kPrIpt = 8;
constexpr int kPrItems = kPrThreads * kPrIpt;

PrPlan::~PrPlan() {
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
}

template <typename V>
struct PrArgs {
  const int64_t* trp;
  const int32_t* tcol;
  const int32_t* outdeg;   // indexed by global row
  const int64_t* tile_row;
  const int64_t* tile_nz;
  const int32_t* head_split;
  const int32_t* tail_split;
  const int32_t* split_first;
  const int32_t* split_parts;
  const int64_t* split_row;
  const int64_t* split_slot;
  double* split_part;
  unsigned* split_cnt;
  V* r0;
  V* r1;
  V* x0;   // x0/x1: contribution vectors indexed by global vertex
  V* x1;
  double* l1_block;
  double* l1_hist;
  int* ctl;
  unsigned* blk_cnt;
  int64_t ntiles;
  int64_t out_base;   // output row r is stored at r - out_base
  double damping, teleport, tol;
  int itermax;
  int fixed;          // 1: single step, r0/x0 are inputs, r1/x1 outputs
  cudaGraphConditionalHandle cond;
};

struct KeyVal {
  int key;
  double val;
};
struct ReduceBySeg {
  __device__ __forceinline__ KeyVal operator()(const KeyVal& a, const KeyVal& b) const {
    KeyVal r;
    r.key = b.key;
    r.val = (a.key == b.key) ? a.val + b.val : b.val;
    return r;
  }
};

template <typename V>
__device__ __forceinline__ double pr_epilogue(const PrArgs<V>& a, const V* r_cur, V* r_nxt,
                                              V* x_nxt, int64_t row, double s) {
  double rn = a.teleport + s;
  int64_t o = row - a.out_base;
  double d = fabs(static_cast<double>(r_cur[o]) - rn);
  r_nxt[o] = static_cast<V>(rn);
  int dg = a.outdeg[row];
  x_nxt[row] = dg > 0 ? static_cast<V>(rn / (static_cast<double>(dg) / a.damping)) : V(0);
  return d;
}

// One part of a row split between tiles; the last part to arrive finishes it.
template <typename V>
__device__ __forceinline__ double pr_split_part(const PrArgs<V>& a, const V* r_cur,
                                                V* r_nxt, V* x_nxt, int id, int64_t t,
                                                double v, unsigned epoch) {
  int64_t base = a.split_slot[id];
  int parts = a.split_parts[id];
  a.split_part[base + (t - a.split_first[id])] = v;
  __threadfence();
  unsigned prev = atomicAdd(&a.split_cnt[id], 1u);
  if (prev == epoch * static_cast<unsigned>(parts) - 1u) {
    __threadfence();
    double s = 0.0;
    for (int q = 0; q < parts; ++q) s += __ldcg(&a.split_part[base + q]);
    return pr_epilogue(a, r_cur, r_nxt, x_nxt, a.split_row[id], s);
  }
  return 0.0;
}

template <typename V, bool kGraph>
__global__ void __launch_bounds__(kPrThreads) k_pr_iter(PrArgs<V> a) {
  using BlockScan = cub::BlockScan<KeyVal, kPrThreads>;
  using BlockReduce = cub::BlockReduce<double, kPrThreads>;
  __shared__ int s_rowend[kPrItems];
  __shared__ V s_val[kPrItems];
  __shared__ double s_sum[kPrItems];
  __shared__ union {
    typename BlockScan::TempStorage scan;
    typename BlockReduce::TempStorage red;
  } tmp;
  __shared__ int s_last;

  if (!a.fixed && *(volatile int*)&a.ctl[1]) return;  // converged (host-looped path)
  const int k = *(volatile int*)&a.ctl[0];
  const unsigned epoch = static_cast<unsigned>(k) + 1u;
  const bool odd = !a.fixed && (k & 1);
  const V* x_cur = odd ? a.x1 : a.x0;
  const V* r_cur = odd ? a.r1 : a.r0;
  V* x_nxt = odd ? a.x0 : a.x1;
  V* r_nxt = odd ? a.r0 : a.r1;
  const int tid = threadIdx.x;
  double l1 = 0.0;

  for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
    const int64_t rs = a.tile_row[t], js = a.tile_nz[t];
    const int nrows = static_cast<int>(a.tile_row[t + 1] - rs);
    const int nnz = static_cast<int>(a.tile_nz[t + 1] - js);
    // ---- stage: row ends (local offsets) and gathered contributions
    {
      int c[kPrIpt];
#pragma unroll
      for (int q = 0; q < kPrIpt; ++q) {
        int i = tid + q * kPrThreads;
        c[q] = i < nnz ? __ldcs(a.tcol + js + i) : -1;
      }
#pragma unroll
      for (int q = 0; q < kPrIpt; ++q) {
        int i = tid + q * kPrThreads;
        if (i < nrows) s_rowend[i] = static_cast<int>(a.trp[rs + 1 + i] - js);
      }
#pragma unroll
      for (int q = 0; q < kPrIpt; ++q) {
        int i = tid + q * kPrThreads;
        if (c[q] >= 0) s_val[i] = __ldg(x_cur + c[q]);
      }
    }
    __syncthreads();
    // ---- merge-path consume
    const int total = nrows + nnz;
    const int diag = min(tid * kPrIpt, total);
    int lo = max(diag - nnz, 0), hi = min(diag, nrows);
    while (lo < hi) {
      int piv = (lo + hi) >> 1;
      if (s_rowend[piv] <= diag - piv - 1) lo = piv + 1; else hi = piv;
    }
    int x = lo, y = diag - lo;
    const int dend = min(diag + kPrIpt, total);
    double sum = 0.0, first_val = 0.0;
    int first_row = -1;
    for (int it = diag; it < dend; ++it) {
      if (x < nrows && s_rowend[x] <= y) {
        if (first_row < 0) { first_row = x; first_val = sum; } else { s_sum[x] = sum; }
        sum = 0.0;
        ++x;
      } else {
        sum += static_cast<double>(s_val[y]);
        ++y;
      }
    }
    KeyVal in{x, sum}, pre, agg;
    BlockScan(tmp.scan).ExclusiveScan(in, pre, KeyVal{-1, 0.0}, ReduceBySeg(), agg);
    if (first_row >= 0) s_sum[first_row] = first_val + (pre.key == first_row ? pre.val : 0.0);
    __syncthreads();
    // ---- fused epilogue over the rows completed in this tile
    const int hs = a.head_split[t];
    for (int i = tid; i < nrows; i += kPrThreads) {
      double s = s_sum[i];
      if (i == 0 && hs >= 0) {
        l1 += pr_split_part(a, r_cur, r_nxt, x_nxt, hs, t, s, epoch);
      } else {
        l1 += pr_epilogue(a, r_cur, r_nxt, x_nxt, rs + i, s);
      }
    }
    if (tid == 0) {
      const int ts = a.tail_split[t];
      if (ts >= 0) l1 += pr_split_part(a, r_cur, r_nxt, x_nxt, ts, t, agg.val, epoch);
    }
    __syncthreads();
  }
  // ---- L1: per-CTA partial, the last CTA reduces in a fixed order
  double blk = BlockReduce(tmp.red).Sum(l1);
  if (tid == 0) {
    a.l1_block[blockIdx.x] = blk;
    __threadfence();
    unsigned prev = atomicAdd(a.blk_cnt, 1u);
    s_last = (prev == epoch * gridDim.x - 1u) ? 1 : 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double part = 0.0;
  for (int b = tid; b < static_cast<int>(gridDim.x); b += kPrThreads) part += __ldcg(&a.l1_block[b]);
  double tot = BlockReduce(tmp.red).Sum(part);
  if (tid == 0) {
    a.l1_hist[k] = tot;
    a.ctl[0] = k + 1;
    bool stop = a.fixed || !(tot >= a.tol) || (k + 1 >= a.itermax);
    if (stop) a.ctl[1] = 1;
    if constexpr (kGraph) cudaGraphSetConditional(a.cond, stop ? 0u : 1u);
  }
}

template <typename V>
__global__ void k_pr_init(V* r, V* x, const int32_t* outdeg, int64_t n, double damping) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  double r0 = 1.0 / static_cast<double>(n);
  r[i] = static_cast<V>(r0);
  int dg = outdeg[i];
  x[i] = dg > 0 ? static_cast<V>(r0 / (static_cast<double>(dg) / damping)) : V(0);
}

// ---- plan construction (host; once per graph) -------------------------------

static void build_tiles(cudaStream_t s, PrPlan& P, const std::vector<int64_t>& trp) {
  const int64_t row0 = P.row0, row1 = P.row1;
  const int64_t nrows = row1 - row0;
  const int64_t nz0 = trp[row0], nz1 = trp[row1];
  const int64_t nnz = nz1 - nz0;
  const int64_t total = nrows + nnz;
  const int64_t ntiles = std::max<int64_t>(1, (total + kPrItems - 1) / kPrItems);
  std::vector<int64_t> trow(ntiles + 1), tnz(ntiles + 1);
  for (int64_t t = 0; t <= ntiles; ++t) {
    int64_t d = std::min(t * kPrItems, total);
    // merge path over row ends a[i] = trp[row0+i+1]-nz0 and nonzeros b[j] = j
    int64_t lo = std::max<int64_t>(d - nnz, 0), hi = std::min(d, nrows);
    while (lo < hi) {
      int64_t piv = (lo + hi) >> 1;
      if (trp[row0 + piv + 1] - nz0 <= d - piv - 1) lo = piv + 1; else hi = piv;
    }
    trow[t] = row0 + lo;
    tnz[t] = nz0 + (d - lo);
  }
  std::vector<int32_t> head(ntiles, -1), tail(ntiles, -1), sfirst, sparts;
  std::vector<int64_t> srow, sslot;
  int64_t slots = 0;
  for (int64_t t = 0; t < ntiles; ++t) {
    int64_t rs = trow[t], js = tnz[t];
    if (rs < row1 && js > trp[rs]) head[t] = static_cast<int32_t>(srow.size()) - 1;
    int64_t re = trow[t + 1], je = tnz[t + 1];
    if (re < row1 && je > trp[re]) {
      if (head[t] >= 0 && srow.back() == re) {
        tail[t] = head[t];
      } else {
        tail[t] = static_cast<int32_t>(srow.size());
        srow.push_back(re);
        sfirst.push_back(static_cast<int32_t>(t));
        sparts.push_back(0);
        sslot.push_back(0);
      }
    }
  }
  // parts = last tile containing the row end - first tile + 1
  for (int64_t t = 0; t < ntiles; ++t) {
    if (head[t] >= 0 && trow[t + 1] > trow[t]) {
      int id = head[t];
      sparts[id] = static_cast<int32_t>(t - sfirst[id] + 1);
    }
  }
  for (size_t id = 0; id < srow.size(); ++id) {
    sslot[id] = slots;
    slots += sparts[id];
  }
  P.ntiles = ntiles;
  P.nsplit = static_cast<int64_t>(srow.size());
  P.tile_row.alloc(ntiles + 1);
  P.tile_nz.alloc(ntiles + 1);
  P.head_split.alloc(ntiles);
  P.tail_split.alloc(ntiles);
  size_t ns = std::max<size_t>(srow.size(), 1);
  P.split_first.alloc(ns);
  P.split_parts.alloc(ns);
  P.split_row.alloc(ns);
  P.split_slot.alloc(ns);
  P.split_part.alloc(std::max<int64_t>(slots, 1));
  P.split_cnt.alloc(ns);
  GBX_CUDA(cudaMemcpyAsync(P.tile_row.p, trow.data(), (ntiles + 1) * 8, cudaMemcpyHostToDevice, s));
  GBX_CUDA(cudaMemcpyAsync(P.tile_nz.p, tnz.data(), (ntiles + 1) * 8, cudaMemcpyHostToDevice, s));
  GBX_CUDA(cudaMemcpyAsync(P.head_split.p, head.data(), ntiles * 4, cudaMemcpyHostToDevice, s));
  GBX_CUDA(cudaMemcpyAsync(P.tail_split.p, tail.data(), ntiles * 4, cudaMemcpyHostToDevice, s));
  if (!srow.empty()) {
    GBX_CUDA(cudaMemcpyAsync(P.split_first.p, sfirst.data(), srow.size() * 4, cudaMemcpyHostToDevice, s));
    GBX_CUDA(cudaMemcpyAsync(P.split_parts.p, sparts.data(), srow.size() * 4, cudaMemcpyHostToDevice, s));
    GBX_CUDA(cudaMemcpyAsync(P.split_row.p, srow.data(), srow.size() * 8, cudaMemcpyHostToDevice, s));
    GBX_CUDA(cudaMemcpyAsync(P.split_slot.p, sslot.data(), srow.size() * 8, cudaMemcpyHostToDevice, s));
  }
  GBX_CUDA(cudaStreamSynchronize(s));
}

static int pr_grid(int64_t ntiles) {
  int per_sm = 0;
  GBX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pr_iter<double, true>, kPrThreads, 0));
  per_sm = std::max(per_sm, 1);
  int64_t g = static_cast<int64_t>(device_sms()) * per_sm;
  return static_cast<int>(std::min<int64_t>(g, ntiles));
}

static void plan_rows(gbx_graph* g, PrPlan& P, int64_t row0, int64_t row1) {
  const Csr& AT = g->AT();
  cudaStream_t s = g->stream;
  P.n = AT.n;
  P.nnz = AT.nnz;
  P.row0 = row0;
  P.row1 = row1;
  std::vector<int64_t> trp(AT.n + 1);
  GBX_CUDA(cudaMemcpyAsync(trp.data(), AT.rp.p, (AT.n + 1) * 8, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  build_tiles(s, P, trp);
  P.grid = pr_grid(P.ntiles);
  P.l1_block.alloc(P.grid);
  P.l1_hist.alloc(128);
  P.ctl.alloc(2);
  P.blk_cnt.alloc(1);
}

void pagerank_prepare(gbx_graph* g) {
  require_at(g, "pagerank_gap");
  require_rowdeg(g, "pagerank_gap");
  if (g->pr) return;
  auto P = std::make_unique<PrPlan>();
  plan_rows(g, *P, 0, g->A.n);
  for (int b = 0; b < 2; ++b) {
    P->r[b].alloc(std::max<int64_t>(g->A.n, 1));
    P->x[b].alloc(std::max<int64_t>(g->A.n, 1));
  }
  g->pr = std::move(P);
}

// fp32 storage unless tol is within 16x of its rounding floor (~6e-8 * mass):
// the reference's own fixtures use tol = 1e-8 (test_pr.cpp:24-38).
static bool use_fp64(double tol) { return tol < 1e-6; }

template <typename V> V* buf_r(PrPlan& P, int b);
template <typename V> V* buf_x(PrPlan& P, int b);
template <> float* buf_r<float>(PrPlan& P, int b) { return P.r[b].p; }
template <> float* buf_x<float>(PrPlan& P, int b) { return P.x[b].p; }
template <> double* buf_r<double>(PrPlan& P, int b) {
  if (!P.rd[b].p) P.rd[b].alloc(P.r[b].n);
  return P.rd[b].p;
}
template <> double* buf_x<double>(PrPlan& P, int b) {
  if (!P.xd[b].p) P.xd[b].alloc(P.x[b].n);
  return P.xd[b].p;
}

template <typename V>
static PrArgs<V> make_args(gbx_graph* g, PrPlan& P, double damping, double tol, int itermax) {
  const Csr& AT = g->AT();
  PrArgs<V> a{};
  a.trp = AT.rp.p;
  a.tcol = AT.col.p;
  a.outdeg = g->rowdeg.p;
  a.tile_row = P.tile_row.p;
  a.tile_nz = P.tile_nz.p;
  a.head_split = P.head_split.p;
  a.tail_split = P.tail_split.p;
  a.split_first = P.split_first.p;
  a.split_parts = P.split_parts.p;
  a.split_row = P.split_row.p;
  a.split_slot = P.split_slot.p;
  a.split_part = P.split_part.p;
  a.split_cnt = P.split_cnt.p;
  if (P.r[0].p) {
    a.r0 = buf_r<V>(P, 0);
    a.r1 = buf_r<V>(P, 1);
    a.x0 = buf_x<V>(P, 0);
    a.x1 = buf_x<V>(P, 1);
  }
  a.l1_block = P.l1_block.p;
  a.l1_hist = P.l1_hist.p;
  a.ctl = P.ctl.p;
  a.blk_cnt = P.blk_cnt.p;
  a.ntiles = P.ntiles;
  a.out_base = 0;
  a.damping = damping;
  a.teleport = (1.0 - damping) / static_cast<double>(P.n);
  a.tol = tol;
  a.itermax = itermax;
  a.fixed = 0;
  return a;
}

static void reset_state(cudaStream_t s, PrPlan& P) {
  GBX_CUDA(cudaMemsetAsync(P.ctl.p, 0, 2 * sizeof(int), s));
  GBX_CUDA(cudaMemsetAsync(P.blk_cnt.p, 0, sizeof(unsigned), s));
  GBX_CUDA(cudaMemsetAsync(P.split_cnt.p, 0, P.split_cnt.bytes(), s));
}

template <typename V>
static bool build_graph(gbx_graph* g, PrPlan& P, double damping, double tol, int itermax) {
  const int prec = sizeof(V) == 8 ? 64 : 32;
  if (P.exec && P.g_damping == damping && P.g_tol == tol && P.g_itermax == itermax &&
      P.g_prec == prec)
    return true;
  if (P.graph_failed) return false;
  if (P.exec) { cudaGraphExecDestroy(P.exec); P.exec = nullptr; }
  if (P.graph) { cudaGraphDestroy(P.graph); P.graph = nullptr; }
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphConditionalHandle cond;
  cudaGraphNode_t node;
  cudaGraph_t body = nullptr;
  bool ok = cudaGraphCreate(&graph, 0) == cudaSuccess &&
            cudaGraphConditionalHandleCreate(&cond, graph, 1, cudaGraphCondAssignDefault) ==
                cudaSuccess;
  if (ok) {
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    ok = cudaGraphAddNode(&node, graph, nullptr, 0, &cp) == cudaSuccess;
    if (ok) body = cp.conditional.phGraph_out[0];
  }
  if (ok) {
    PrArgs<V> a = make_args<V>(g, P, damping, tol, itermax);
    a.cond = cond;
    void* params[] = {&a};
    cudaKernelNodeParams kp = {};
    kp.func = reinterpret_cast<void*>(k_pr_iter<V, true>);
    kp.gridDim = dim3(P.grid);
    kp.blockDim = dim3(kPrThreads);
    kp.sharedMemBytes = 0;
    kp.kernelParams = params;
    cudaGraphNode_t kn;
    ok = cudaGraphAddKernelNode(&kn, body, nullptr, 0, &kp) == cudaSuccess;
  }
  if (ok) ok = cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
  if (!ok) {
    (void)cudaGetLastError();
    if (graph) cudaGraphDestroy(graph);
    P.graph_failed = true;
    return false;
  }
  P.graph = graph;
  P.exec = exec;
  P.g_damping = damping;
  P.g_tol = tol;
  P.g_itermax = itermax;
  P.g_prec = prec;
  return true;
}

template <typename V>
static int pagerank_loop(gbx_graph* g, PrPlan& P, double damping, double tol, int itermax,
                         double* rank, int* iters) {
  const int64_t n = g->A.n;
  cudaStream_t s = g->stream;
  reset_state(s, P);
  k_pr_init<V><<<ceil_div(n, 256), 256, 0, s>>>(buf_r<V>(P, 0), buf_x<V>(P, 0), g->rowdeg.p, n,
                                                damping);
  GBX_LAUNCHED();
  if (build_graph<V>(g, P, damping, tol, itermax)) {
    GBX_CUDA(cudaGraphLaunch(P.exec, s));
  } else {
    // host-looped fallback: chunks of launches, each exits early once done
    PrArgs<V> a = make_args<V>(g, P, damping, tol, itermax);
    int done = 0, launched = 0;
    while (!done && launched < itermax) {
      int chunk = std::min(4, itermax - launched);
      for (int c = 0; c < chunk; ++c) {
        k_pr_iter<V, false><<<P.grid, kPrThreads, 0, s>>>(a);
        GBX_LAUNCHED();
      }
      launched += chunk;
      GBX_CUDA(cudaMemcpyAsync(&done, P.ctl.p + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
      GBX_CUDA(cudaStreamSynchronize(s));
    }
  }
  int it = 0;
  if (rank != nullptr || iters != nullptr) {
    GBX_CUDA(cudaMemcpyAsync(&it, P.ctl.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaStreamSynchronize(s));
    P.last_iters = it;
    if (iters) *iters = it;
    if (rank) {
      std::vector<V> r(n);
      GBX_CUDA(cudaMemcpyAsync(r.data(), buf_r<V>(P, it & 1), n * sizeof(V),
                               cudaMemcpyDeviceToHost, s));
      GBX_CUDA(cudaStreamSynchronize(s));
      for (int64_t i = 0; i < n; ++i) rank[i] = r[i];
    }
  }
  return it;
}

void pagerank_run(gbx_graph* g, double damping, double tol, int itermax, double* rank,
                  int* iters) {
  require_at(g, "pagerank_gap");
  require_rowdeg(g, "pagerank_gap");
  if (!(damping > 0.0)) fail(GBX_NON_POSITIVE_DAMPING, "damping must be positive");
  const int64_t n = g->A.n;
  g->stats = gbx_stats{};
  if (n == 0 || itermax <= 0) {
    if (iters) *iters = itermax <= 0 ? std::max(itermax, 0) : 0;
    if (n > 0 && rank) {
      for (int64_t i = 0; i < n; ++i) rank[i] = 1.0 / static_cast<double>(n);
    }
    return;
  }
  pagerank_prepare(g);
  PrPlan& P = *g->pr;
  const bool f64 = use_fp64(tol);
  P.last_prec = f64 ? 64 : 32;
  int it = f64 ? pagerank_loop<double>(g, P, damping, tol, itermax, rank, iters)
               : pagerank_loop<float>(g, P, damping, tol, itermax, rank, iters);
  const double vb = f64 ? 8.0 : 4.0;
  g->stats.launches = 1 + it;
  g->stats.hot_launches = it;
  g->stats.iterations = it;
  g->stats.work_units = g->AT().nnz;
  // col (4) + gathered x (vb) per edge; row_ptr (8) + r_prev, r, x (vb each) + deg (4)
  g->stats.hot_bytes_per_launch = (4.0 + vb) * static_cast<double>(g->AT().nnz) +
                                  8.0 * static_cast<double>(n + 1) + (3.0 * vb + 4.0) * n;
}

// ---- sharded step (multi-GPU driver) ----------------------------------------------

void pr_shard_prepare(gbx_graph* g, int64_t rb, int64_t re) {
  require_at(g, "pr_shard");
  require_rowdeg(g, "pr_shard");
  if (rb < 0 || re > g->A.n || rb > re) fail(GBX_INDEX_OUT_OF_BOUNDS, "pr_shard: bad row range");
  auto S = std::make_unique<PrShard>();
  plan_rows(g, S->plan, rb, re);
  g->prs = std::move(S);
}

void pr_shard_step(gbx_graph* g, const float* x_full, float* r, float* x_new, double* l1,
                   double damping) {
  if (!g->prs) fail(GBX_MISSING_PROPERTY, "pr_shard_step needs gbx_pr_shard_prepare");
  PrPlan& P = g->prs->plan;
  cudaStream_t s = g->stream;
  PrArgs<float> a = make_args<float>(g, P, damping, 0.0, 1 << 30);
  a.fixed = 1;
  a.x0 = const_cast<float*>(x_full);
  a.x1 = x_new;       // written at global row ids
  a.r0 = r;           // r_prev (local rows), overwritten in place by r_new
  a.r1 = r;
  a.out_base = P.row0;
  GBX_CUDA(cudaMemsetAsync(P.ctl.p, 0, 2 * sizeof(int), s));
  GBX_CUDA(cudaMemsetAsync(P.blk_cnt.p, 0, sizeof(unsigned), s));
  GBX_CUDA(cudaMemsetAsync(P.split_cnt.p, 0, P.split_cnt.bytes(), s));
  k_pr_iter<float, false><<<P.grid, kPrThreads, 0, s>>>(a);
  GBX_LAUNCHED();
  GBX_CUDA(cudaMemcpyAsync(l1, P.l1_hist.p, sizeof(double), cudaMemcpyDeviceToDevice, s));
  g->prs->steps++;
}

}  // namespace gbx
