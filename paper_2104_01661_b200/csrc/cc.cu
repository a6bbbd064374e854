// cc.cu -- connected components with canonical minimum-id labels.
//
// The reference's FastSV (algo/components.cpp:35-106) converges to the
// component minimum (components.cpp:27-30); any exact method with min-id roots
// is bit-exact.  Here: edge-parallel min-hooking of roots (the larger root is
// hooked under the smaller with atomicMin) alternated with pointer jumping,
// until no hook changes anything -- each round is two memory-bound sweeps.
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "plans.cuh"

namespace gbx {

__global__ void k_cc_init(int32_t* p, int64_t n) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) p[i] = static_cast<int32_t>(i);
}

__device__ __forceinline__ int32_t cc_find(const int32_t* p, int32_t x) {
  const volatile int32_t* vp = p;
  int32_t y = vp[x];
  while (y != x) { x = y; y = vp[x]; }
  return x;
}

// one warp per row: hook the roots of every edge endpoint pair
__global__ void k_cc_hook(const int64_t* rp, const int32_t* col, int64_t n, int32_t* p,
                          int* changed) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = w; i < n; i += nw) {
    const int64_t b = rp[i], e = rp[i + 1];
    for (int64_t q = b + lane; q < e; q += 32) {
      int32_t j = col[q];
      int32_t ri = static_cast<int32_t>(i), rj = j;
      // lock-free union: only a root may be re-hooked, always under the
      // smaller root, so every tree's root is its minimum id
      for (;;) {
        ri = cc_find(p, ri);
        rj = cc_find(p, rj);
        if (ri == rj) break;
        int32_t hi = max(ri, rj), lo = min(ri, rj);
        if (atomicCAS(&p[hi], hi, lo) == hi) { *changed = 1; break; }
      }
    }
  }
}

__global__ void k_cc_jump(int32_t* p, int64_t n) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) {
    int32_t x = static_cast<int32_t>(i);
    int32_t r = cc_find(p, x);
    p[i] = r;
  }
}

__global__ void k_cc_out(const int32_t* p, int64_t n, int64_t* out) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = p[i];
}

void cc_run(gbx_graph* g, int64_t* label, int* iters) {
  NvtxRange nvtx_("gbx.connected_components");
  const int64_t n = g->A.n;
  if (!g->cc) g->cc = std::make_unique<CcWork>();
  CcWork& W = *g->cc;
  if (W.n != n) {
    W.n = n;
    W.parent.alloc(std::max<int64_t>(n, 1));
    W.ctl.alloc(1);
  }
  cudaStream_t s = g->stream;
  g->stats = gbx_stats{};
  g->pending_iters = nullptr;
  if (n == 0) { if (iters) *iters = 0; return; }
  k_cc_init<<<ceil_div(n, 256), 256, 0, s>>>(W.parent.p, n);
  GBX_LAUNCHED();
  int rounds = 0, changed = 1;
  const int grid = device_sms() * 8;
  int launches = 1;
  while (changed) {
    GBX_CUDA(cudaMemsetAsync(W.ctl.p, 0, sizeof(int), s));
    k_cc_hook<<<grid, 256, 0, s>>>(g->A.rp.p, g->A.col.p, n, W.parent.p, W.ctl.p);
    k_cc_jump<<<ceil_div(n, 256), 256, 0, s>>>(W.parent.p, n);
    GBX_LAUNCHED();
    launches += 2;
    GBX_CUDA(cudaMemcpyAsync(&changed, W.ctl.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaStreamSynchronize(s));
    ++rounds;
  }
  if (label) {
    int64_t* tmp = nullptr;
    GBX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tmp), n * 8, s));
    k_cc_out<<<ceil_div(n, 256), 256, 0, s>>>(W.parent.p, n, tmp);
    cudaError_t le = cudaGetLastError();
    if (le == cudaSuccess) le = cudaMemcpyAsync(label, tmp, n * 8, cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(tmp, s);
    GBX_CUDA(le);
    GBX_CUDA(cudaStreamSynchronize(s));
    ++launches;
  }
  if (iters) *iters = rounds;
  g->stats.launches = launches;
  g->stats.hot_launches = rounds;
  g->stats.iterations = rounds;
  g->stats.work_units = g->A.nnz;
  g->stats.hot_bytes_per_launch = 4.0 * g->A.nnz + 8.0 * (n + 1) + 8.0 * n;
}

}  // namespace gbx
