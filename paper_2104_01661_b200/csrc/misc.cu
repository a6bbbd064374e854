// misc.cu -- row partitioning for the multi-GPU drivers and device result access.
#include <algorithm>
#include <string>
#include <vector>

#include "common.cuh"
#include "plans.cuh"

namespace gbx {

// Split rows into `parts` contiguous blocks with balanced (rows + nnz) work --
// the merge-path diagonal split, so a hub row never unbalances a shard by more
// than its own length ("split by nnz, not row count").
void partition_rows(const gbx_graph* g, int parts, bool transposed, int64_t* bounds) {
  if (parts < 1) fail(GBX_INVALID_VALUE, "partition_rows: parts must be >= 1");
  if (transposed && !g->has_at) fail(GBX_MISSING_PROPERTY, "partition_rows needs G.AT");
  const Csr& M = transposed ? g->AT() : g->A;
  std::vector<int64_t> rp(M.n + 1);
  GBX_CUDA(cudaMemcpyAsync(rp.data(), M.rp.p, (M.n + 1) * 8, cudaMemcpyDeviceToHost, g->stream));
  GBX_CUDA(cudaStreamSynchronize(g->stream));
  const int64_t total = M.n + M.nnz;
  bounds[0] = 0;
  for (int p = 1; p < parts; ++p) {
    int64_t target = total * p / parts;
    // smallest row r with r + rp[r] >= target
    int64_t lo = 0, hi = M.n;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (mid + rp[mid] < target) lo = mid + 1; else hi = mid;
    }
    bounds[p] = std::max(lo, bounds[p - 1]);
  }
  bounds[parts] = M.n;
}

void result_device(const gbx_graph* g, const std::string& w, void** ptr, int64_t* count) {
  *ptr = nullptr;
  *count = 0;
  if (w == "pagerank" && g->pr) {
    *ptr = g->pr->out.p;  // fp64 ranks, original vertex order
    *count = g->A.n;
  } else if (w == "bfs" && g->bfs) {
    *ptr = g->bfs->parent.p;
    *count = g->A.n;
  } else if (w == "bfs_batch" && g->bfs) {
    *ptr = g->bfs->mparent.p;
    *count = g->A.n * 64;
  } else if (w == "cc" && g->cc) {
    *ptr = g->cc->parent.p;
    *count = g->A.n;
  } else if (w == "sssp" && g->sssp) {
    *ptr = g->sssp->integral ? static_cast<void*>(g->sssp->lanes[0]->dist32.p)
                             : static_cast<void*>(g->sssp->lanes[0]->dist64.p);
    *count = g->A.n;
  } else if (w == "bc" && g->bc) {
    *ptr = g->bc->cent.p;
    *count = g->A.n;
  } else {
    fail(GBX_NO_VALUE, "no device result for '" + w + "'");
  }
}

}  // namespace gbx
