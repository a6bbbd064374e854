// mg.cu -- the multi-GPU algorithms over a distributed graph,
// host orchestration in C++ over gbx_comm (NCCL, or in-process ranks on one
// GPU), device work in the same shard kernels as the single-GPU library.
//
//   PageRank (config 2)  1D row blocks of the in-degree-relabeled AT; per
//                        iteration the exchange is FUSED into the iteration
//                        kernel (peer stores over NVLink into every rank's x,
//                        device-side signal barrier) or, as the fallback, one
//                        NCCL all-gather of the padded x slices + L1 partials.
//   Triangle count (3)   U replicated (all-gather of every rank's upper keys),
//                        middle vertices split by probe work, one u64
//                        all-reduce (triangle.cpp:55-62: mxm + reduce_scalar).
//   BFS (scale >= 22)    pull levels on the owned rows against the global
//                        frontier bitmap, one bitmap all-gather per level.
//   Betweenness (5)      row-partitioned Brandes: per BFS level the settled
//                        vertices' records are all-gathered; one fp64
//                        all-reduce of the centrality (betweenness.cpp:74-79).
// Every rank returns the same full result (the reference's outputs).
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>

#include "comm.cuh"
#include "plans.cuh"

namespace gbx {

namespace {

__global__ void k_row_len(const int64_t* rp, int64_t n, int32_t* len) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) len[i] = static_cast<int32_t>(rp[i + 1] - rp[i]);
}
__global__ void k_gather32(const int32_t* src, const int32_t* idx, int64_t n, int32_t* dst) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}
__global__ void k_gather32_to64(const int32_t* src, const int32_t* idx, int64_t n, int64_t* dst) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}
__global__ void k_invert(const int32_t* new2old, int64_t n, int32_t* old2new) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) old2new[new2old[i]] = static_cast<int32_t>(i);
}
// owned rows of a block CSR -> relabeled (new row << bits | new col) keys
__global__ void k_relabel_block(const int64_t* rp, const int32_t* col, int64_t rb, int64_t re,
                                const int32_t* old2new, int bits, uint64_t* keys) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t base = rp[rb];
  for (int64_t r = rb + w; r < re; r += nw) {
    const uint64_t nr = static_cast<uint64_t>(old2new[r]);
    for (int64_t p = rp[r] + lane; p < rp[r + 1]; p += 32)
      keys[p - base] = (nr << bits) | static_cast<uint64_t>(old2new[col[p]]);
  }
}
__global__ void k_axpy1(double* acc, const double* x, int64_t n) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) acc[i] += x[i];
}

struct CommLock {
  std::lock_guard<std::mutex> lk;
  explicit CommLock(gbx_comm* c) : lk(c->mu) { GBX_CUDA(cudaSetDevice(c->device)); }
};

void sync_shards(gbx_dgraph* D) {
  for (gbx_graph* g : D->shard) GBX_CUDA(cudaStreamSynchronize(g->stream));
}

// every rank's variable-length records (rec bytes each) in rank order, on
// every local rank: out[l] (device), total count returned
int64_t gather_records(gbx_comm* c, const std::vector<const void*>& recs,
                       const std::vector<int64_t>& nrec, size_t rec,
                       std::vector<DevArray<uint8_t>>& out) {
  const std::vector<int64_t> cnt = c_allgather_host(c, nrec);
  int64_t mx = 0, total = 0;
  for (int64_t x : cnt) {
    mx = std::max(mx, x);
    total += x;
  }
  const int L = c->nlocal, P = c->nranks;
  out.resize(L);
  if (total == 0) return 0;
  std::vector<DevArray<uint8_t>> send(L), recv(L);
  std::vector<const void*> sp(L);
  std::vector<void*> rp(L);
  for (int l = 0; l < L; ++l) {
    send[l].alloc(mx * rec);
    recv[l].alloc(mx * rec * P);
    if (nrec[l])
      GBX_CUDA(cudaMemcpyAsync(send[l].p, recs[l], nrec[l] * rec, cudaMemcpyDeviceToDevice, c->stream));
    sp[l] = send[l].p;
    rp[l] = recv[l].p;
  }
  comm_sync(c);
  c_allgather(c, sp.data(), rp.data(), mx * rec);
  for (int l = 0; l < L; ++l) {
    out[l].ensure(std::max<int64_t>(total, 1) * rec);
    int64_t off = 0;
    for (int q = 0; q < P; ++q) {
      if (cnt[q])
        GBX_CUDA(cudaMemcpyAsync(out[l].p + off * rec, recv[l].p + q * mx * rec, cnt[q] * rec,
                                 cudaMemcpyDeviceToDevice, c->stream));
      off += cnt[q];
    }
  }
  comm_sync(c);
  return total;
}

// ---- PageRank ---------------------------------------------------------------------

// the relabeled AT row blocks and the shard plans (cached on the shards)
void pr_mg_prepare(gbx_dgraph* D) {
  NvtxRange nvtx_("gbx.pagerank_mg.prepare");
  gbx_comm* c = D->comm;
  const int L = c->nlocal, P = c->nranks;
  bool ready = true;
  for (gbx_graph* g : D->shard) ready = ready && g->prs && g->prs->nranks == P;
  if (ready) return;
  const int64_t n = D->n;
  const int64_t n1 = std::max<int64_t>(n, 1);
  cudaStream_t s = c->stream;
  // 1. in- and out-degree of every vertex: the owned rows' lengths, all-reduced
  std::vector<DevArray<int32_t>> indeg(L), outdeg(L);
  std::vector<void*> pin(L), pout(L);
  for (int l = 0; l < L; ++l) {
    gbx_graph* g = D->shard[l];
    indeg[l].alloc(n1);
    outdeg[l].alloc(n1);
    if (n) {
      k_row_len<<<ceil_div(n, 256), 256, 0, s>>>(g->AT().rp.p, n, indeg[l].p);
      k_row_len<<<ceil_div(n, 256), 256, 0, s>>>(g->A.rp.p, n, outdeg[l].p);
      GBX_LAUNCHED();
    }
    pin[l] = indeg[l].p;
    pout[l] = outdeg[l].p;
  }
  comm_sync(c);
  c_allreduce(c, pin.data(), n, CollType::I32, CollOp::Sum);
  if (D->kind == GBX_UNDIRECTED) {
    for (int l = 0; l < L; ++l)
      GBX_CUDA(cudaMemcpyAsync(outdeg[l].p, indeg[l].p, n * 4, cudaMemcpyDeviceToDevice, s));
    comm_sync(c);
  } else {
    c_allreduce(c, pout.data(), n, CollType::I32, CollOp::Sum);
  }
  // 2. the relabeling (stable, descending in-degree -- the single-GPU plan's)
  //    and the balanced bounds over its row-pointer prefix: identical everywhere
  std::vector<DevArray<int32_t>> new2old(L), old2new(L), deg_new(L);
  for (int l = 0; l < L; ++l) {
    sort_ids_by_key(s, indeg[l].p, n, false, new2old[l]);
    old2new[l].alloc(n1);
    deg_new[l].alloc(n1);
    if (n) {
      k_invert<<<ceil_div(n, 256), 256, 0, s>>>(new2old[l].p, n, old2new[l].p);
      k_gather32<<<ceil_div(n, 256), 256, 0, s>>>(outdeg[l].p, new2old[l].p, n, deg_new[l].p);
      GBX_LAUNCHED();
    }
  }
  std::vector<int64_t> rp(n + 1, 0);
  {
    DevArray<int64_t> len(n1);
    if (n) {
      k_gather32_to64<<<ceil_div(n, 256), 256, 0, s>>>(indeg[0].p, new2old[0].p, n, len.p);
      GBX_LAUNCHED();
    }
    std::vector<int64_t> hl(n);
    GBX_CUDA(cudaMemcpyAsync(hl.data(), len.p, n * 8, cudaMemcpyDeviceToHost, s));
    comm_sync(c);
    for (int64_t i = 0; i < n; ++i) rp[i + 1] = rp[i] + hl[i];
  }
  const std::vector<int64_t> nb = pr_bounds(rp.data(), n, rp[n], P);
  // 3. every rank's AT entries relabeled and shuffled to their new owners
  const int bits = bits_for(std::max<int64_t>(n, 2));
  std::vector<KeyBlock> keys(L);
  for (int l = 0; l < L; ++l) {
    gbx_graph* g = D->shard[l];
    const Csr& AT = g->AT();
    int64_t rb, re;
    dgraph_block(D, l, &rb, &re);
    keys[l].m = AT.nnz;
    keys[l].k.alloc(std::max<int64_t>(AT.nnz, 1));
    if (AT.nnz) {
      k_relabel_block<<<device_sms() * 8, 256, 0, s>>>(AT.rp.p, AT.col.p, rb, re, old2new[l].p, bits,
                                                       keys[l].k.p);
      GBX_LAUNCHED();
    }
    comm_sync(c);
    sort_in_place(s, keys[l], bits);
  }
  std::vector<Csr> blocks(L);
  std::vector<Csr*> bp(L);
  for (int l = 0; l < L; ++l) bp[l] = &blocks[l];
  shuffle_to_blocks(c, keys, nb, n, bits, bp);
  // 4. the shard plans over the owned relabeled rows
  for (int l = 0; l < L; ++l)
    pr_shard_from_block(D->shard[l], c->global_rank(l), P, blocks[l], deg_new[l], new2old[l], nb);
}

// every rank's flag min-reduced (a barrier as well: no rank returns before
// every rank arrived); one persistent word, no allocation per call
int agree(gbx_comm* c, PrMgState& S, int ok) {
  if (!c->nccl) return ok;  // in-process ranks: one host thread, nothing to agree on
  if (!S.flag.p) S.flag.alloc(1);
  GBX_CUDA(cudaMemcpyAsync(S.flag.p, &ok, 4, cudaMemcpyHostToDevice, c->stream));
  void* fp = S.flag.p;
  c_allreduce(c, &fp, 1, CollType::I32, CollOp::Min);
  GBX_CUDA(cudaMemcpy(&ok, S.flag.p, 4, cudaMemcpyDeviceToHost));
  return ok;
}

// the fused run (peer stores + device barrier); false when any rank failed
bool pr_mg_p2p(gbx_dgraph* D, PrMgState& S, double damping, double tol, int itermax, int* iters) {
  NvtxRange nvtx_("gbx.pagerank_mg.fused_run");
  gbx_comm* c = D->comm;
  const int L = c->nlocal, P = c->nranks;
  int ok = 1;
  try {
    if (S.x0.local.empty()) {
      peer_alloc(c, P * S.chunk * sizeof(float), S.x0);
      peer_alloc(c, P * S.chunk * sizeof(float), S.x1);
      peer_alloc(c, 2 * P * sizeof(double), S.l1);
      peer_alloc(c, 16, S.sig);
    }
    for (int l = 0; l < L; ++l) {
      GBX_CUDA(cudaMemsetAsync(S.sig.local[l], 0, 16, c->stream));
      GBX_CUDA(cudaMemsetAsync(S.l1.local[l], 0, 2 * P * sizeof(double), c->stream));
      pr_shard_init(D->shard[l], static_cast<float*>(S.x0.local[l]), S.r0[l].p, damping);
    }
    comm_sync(c);
    sync_shards(D);
  } catch (const Error&) {
    ok = 0;
  }
  // every rank zeroed its words before any rank signals; agree on the setup
  ok = agree(c, S, ok);
  if (!ok) return false;
  int it = 0;
  try {
    if (c->nccl) {
      pr_shard_run_p2p(D->shard[0], S.x0.peer[0].data(), S.x1.peer[0].data(), S.l1.peer[0].data(),
                       S.sig.peer[0].data(), S.r0[0].p, S.r1[0].p, damping, tol, itermax, &it);
    } else {
      std::vector<float*> r0(L), r1(L);
      for (int l = 0; l < L; ++l) {
        r0[l] = S.r0[l].p;
        r1[l] = S.r1[l].p;
      }
      pr_shard_run_p2p_multi(D->shard.data(), L, S.x0.peer[0].data(), S.x1.peer[0].data(),
                             S.l1.peer[0].data(), S.sig.peer[0].data(), r0.data(), r1.data(),
                             damping, tol, itermax, &it);
    }
  } catch (const Error&) {
    ok = 0;  // e.g. a peer timeout: the words are re-zeroed by the next setup
  }
  ok = agree(c, S, ok);
  *iters = it;
  return ok != 0;
}

// one NCCL all-gather of the padded x slices (+ L1 partials) per iteration
void pr_mg_nccl(gbx_dgraph* D, PrMgState& S, double damping, double tol, int itermax, int* iters) {
  NvtxRange nvtx_("gbx.pagerank_mg.nccl_run");
  gbx_comm* c = D->comm;
  const int L = c->nlocal, P = c->nranks;
  const int64_t chunk = S.chunk;
  if (S.xfull.size() != static_cast<size_t>(L)) {
    S.xfull.resize(L);
    S.xs.resize(L);
    for (int l = 0; l < L; ++l) {
      S.xfull[l].alloc(P * chunk);
      S.xs[l].alloc(chunk);
    }
  }
  for (int l = 0; l < L; ++l) {
    GBX_CUDA(cudaMemsetAsync(S.xs[l].p, 0, chunk * 4, c->stream));
    pr_shard_init(D->shard[l], S.xfull[l].p, S.r0[l].p, damping);
  }
  comm_sync(c);
  sync_shards(D);
  std::vector<const void*> sp(L);
  std::vector<void*> rp(L);
  for (int l = 0; l < L; ++l) {
    sp[l] = S.xs[l].p;
    rp[l] = S.xfull[l].p;
  }
  std::vector<double> tails(P);
  int done_at = itermax;
  for (int k = 1; k <= itermax; ++k) {
    for (int l = 0; l < L; ++l) {
      float* rprev = (k - 1) & 1 ? S.r1[l].p : S.r0[l].p;
      float* rnew = k & 1 ? S.r1[l].p : S.r0[l].p;
      pr_shard_step(D->shard[l], S.xfull[l].p, rprev, rnew, S.xs[l].p,
                    reinterpret_cast<double*>(S.xs[l].p + chunk - 2), damping);
    }
    sync_shards(D);
    c_allgather(c, sp.data(), rp.data(), chunk * sizeof(float));
    // every rank's L1 partial sits in its slot's last 8 bytes: sum in rank order
    GBX_CUDA(cudaMemcpy2D(tails.data(), 8, S.xfull[0].p + chunk - 2, chunk * sizeof(float), 8, P,
                          cudaMemcpyDeviceToHost));
    double tot = 0.0;
    for (int q = 0; q < P; ++q) tot += tails[q];
    if (!(tot >= tol)) {  // pagerank.cpp:74
      done_at = k;
      break;
    }
  }
  *iters = done_at;
}

}  // namespace

void pagerank_mg(gbx_dgraph* D, double damping, double tol, int itermax, int exchange,
                 double* rank, int* iters) {
  NvtxRange nvtx_("gbx.pagerank_mg");
  gbx_comm* c = D->comm;
  CommLock lk(c);
  if (!(damping > 0.0)) fail(GBX_NON_POSITIVE_DAMPING, "damping must be positive");
  if (exchange < GBX_MG_AUTO || exchange > GBX_MG_P2P) fail(GBX_INVALID_VALUE, "pagerank_mg: unknown exchange");
  const int64_t n = D->n;
  D->stats = gbx_stats{};
  if (n == 0 || itermax <= 0) {  // pagerank.cpp:52-75, as pagerank_run
    if (iters) *iters = n == 0 ? 0 : itermax;
    if (rank)
      for (int64_t i = 0; i < n; ++i) rank[i] = 1.0 / static_cast<double>(n);
    return;
  }
  pr_mg_prepare(D);
  const int L = c->nlocal, P = c->nranks;
  if (!D->pr) D->pr = std::make_unique<PrMgState>();
  PrMgState& S = *D->pr;
  const int64_t chunk = D->shard[0]->prs->chunk;
  if (S.chunk != chunk) {
    S = PrMgState{};
    S.chunk = chunk;
    S.r0.resize(L);
    S.r1.resize(L);
    for (int l = 0; l < L; ++l) {
      S.r0[l].alloc(chunk);
      S.r1[l].alloc(chunk);
    }
  }
  int it = 0;
  S.p2p_failed = false;
  bool done = false;
  if (exchange != GBX_MG_NCCL && P <= kMaxRanks) {
    done = pr_mg_p2p(D, S, damping, tol, itermax, &it);
    if (!done) {
      S.p2p_failed = true;
      if (exchange == GBX_MG_P2P) fail(GBX_COMM_ERROR, "pagerank_mg: the fused exchange failed");
    }
  }
  if (!done) pr_mg_nccl(D, S, damping, tol, itermax, &it);
  D->stats.iterations = it;
  D->stats.launches = done ? 3 * L : (2 * it + 2) * L;
  D->stats.hot_launches = done ? L : it * L;
  D->stats.work_units = D->nnz;
  D->stats.hot_ms = D->shard[0]->prs->plan.last_rows_ms;
  if (iters) *iters = it;
  if (rank) {
    // every rank's r slice (padded layout) -> the full rank vector, original ids
    std::vector<const void*> sp(L);
    std::vector<void*> rp(L);
    std::vector<DevArray<float>> full(L);
    for (int l = 0; l < L; ++l) {
      sp[l] = (it & 1 ? S.r1[l] : S.r0[l]).p;
      full[l].alloc(P * chunk);
      rp[l] = full[l].p;
    }
    c_allgather(c, sp.data(), rp.data(), chunk * sizeof(float));
    pr_shard_unpermute(D->shard[0], full[0].p, rank);
  }
}

// ---- triangle count ------------------------------------------------------------------

uint64_t triangle_count_mg(gbx_dgraph* D) {
  NvtxRange nvtx_("gbx.triangle_count_mg");
  gbx_comm* c = D->comm;
  CommLock lk(c);
  if (D->kind != GBX_UNDIRECTED)
    fail(GBX_INVALID_GRAPH, "triangle_count needs an undirected graph (triangle.cpp:15-25)");
  const int L = c->nlocal, P = c->nranks;
  const int64_t n = D->n;
  const int64_t n1 = std::max<int64_t>(n, 1);
  cudaStream_t s = c->stream;
  D->stats = gbx_stats{};
  bool ready = true;
  for (gbx_graph* g : D->shard) ready = ready && g->tc;
  if (!ready) {
    const int bits = bits_for(std::max<int64_t>(n, 2));
    // degrees of every vertex (the rank order), then this rank's U keys
    std::vector<DevArray<int32_t>> deg(L);
    std::vector<void*> dp(L);
    for (int l = 0; l < L; ++l) {
      deg[l].alloc(n1);
      if (n) {
        k_row_len<<<ceil_div(n, 256), 256, 0, s>>>(D->shard[l]->A.rp.p, n, deg[l].p);
        GBX_LAUNCHED();
      }
      dp[l] = deg[l].p;
    }
    comm_sync(c);
    c_allreduce(c, dp.data(), n, CollType::I32, CollOp::Sum);
    std::vector<KeyBlock> up(L);
    std::vector<int64_t> cnt(L, 0);
    std::vector<const void*> src(L);
    for (int l = 0; l < L; ++l) {
      const Csr& A = D->shard[l]->A;
      up[l].m = A.nnz;
      up[l].k.alloc(std::max<int64_t>(A.nnz, 1));
      tc_upper_keys(s, A, deg[l].p, n, bits, up[l].k.p);
      sort_in_place(s, up[l], bits);
      // valid keys: the prefix before the first drop key
      const uint64_t drop = uint64_t(1) << (2 * bits);
      std::vector<uint64_t> hk;
      int64_t lo = 0, hi = up[l].m;
      while (lo < hi) {  // host binary search over device keys (log m copies)
        const int64_t mid = (lo + hi) >> 1;
        uint64_t v;
        GBX_CUDA(cudaMemcpy(&v, up[l].k.p + mid, 8, cudaMemcpyDeviceToHost));
        if (v < drop) lo = mid + 1; else hi = mid;
      }
      cnt[l] = lo;
      src[l] = up[l].k.p;
    }
    // U replicated: every rank's upper keys, all-gathered
    std::vector<DevArray<uint8_t>> all;
    const int64_t unnz = gather_records(c, src, cnt, 8, all);
    for (int l = 0; l < L; ++l) {
      up[l].k.release();
      KeyBlock u;
      u.m = unnz;
      u.k.alloc(std::max<int64_t>(unnz, 1));
      if (unnz)
        GBX_CUDA(cudaMemcpyAsync(u.k.p, all[l].p, unnz * 8, cudaMemcpyDeviceToDevice, s));
      all[l].release();
      sort_in_place(s, u, bits);
      DevArray<uint64_t> scratch(std::max<int64_t>(unnz, 1));
      tc_plan_from_upper(D->shard[l], n, bits, u.k.p, unnz, scratch.p, u.k.p);
      GBX_CUDA(cudaStreamSynchronize(D->shard[l]->stream));
    }
  }
  // middle vertices split by probe work: the same split on every rank (the
  // replicated U is identical everywhere; computed once per graph)
  if (static_cast<int>(D->tc_bounds.size()) != P + 1) {
    D->tc_bounds.assign(P + 1, 0);
    tc_partition(D->shard[0], P, D->tc_bounds.data());
  }
  const std::vector<int64_t>& b = D->tc_bounds;
  std::vector<DevArray<unsigned long long>> part(L);
  std::vector<void*> pp(L);
  for (int l = 0; l < L; ++l) {
    const int q = c->global_rank(l);
    const unsigned long long mine = tc_run(D->shard[l], b[q], b[q + 1]);
    D->stats.launches += D->shard[l]->stats.launches;
    part[l].alloc(1);
    GBX_CUDA(cudaMemcpy(part[l].p, &mine, 8, cudaMemcpyHostToDevice));
    pp[l] = part[l].p;
  }
  c_allreduce(c, pp.data(), 1, CollType::U64, CollOp::Sum);
  unsigned long long tot = 0;
  GBX_CUDA(cudaMemcpy(&tot, part[0].p, 8, cudaMemcpyDeviceToHost));
  D->stats.hot_launches = L;
  D->stats.work_units = D->nnz;
  return tot;
}

// ---- BFS ------------------------------------------------------------------------------

namespace {

__global__ void k_pack_rows(const int32_t* lev, const int32_t* par, int64_t rb, int64_t re,
                            int32_t* out) {  // out[2][mx]: level then parent of the owned rows
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (rb + i >= re) return;
  out[i] = lev[rb + i];
  out[(re - rb) + i] = par[rb + i];
}

__global__ void k_unpack_rows(const int32_t* in, int64_t mx, const int64_t* bounds, int P,
                              int64_t n, int64_t* lev, int64_t* par) {
  const int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (v >= n) return;
  int q = 0;
  while (q + 1 < P && v >= bounds[q + 1]) ++q;
  const int64_t m = bounds[q + 1] - bounds[q];
  const int32_t* blk = in + q * 2 * mx;
  const int32_t L = blk[v - bounds[q]], Pa = blk[m + (v - bounds[q])];
  lev[v] = L;
  par[v] = L < 0 ? -1 : Pa;
}

void gather_bfs_result(gbx_dgraph* D, int64_t* parent, int64_t* level) {
  gbx_comm* c = D->comm;
  const int L = c->nlocal, P = c->nranks;
  const int64_t n = D->n;
  int64_t mx = 1;
  for (int q = 0; q < P; ++q) mx = std::max(mx, D->bounds[q + 1] - D->bounds[q]);
  std::vector<DevArray<int32_t>> send(L), recv(L);
  std::vector<const void*> sp(L);
  std::vector<void*> rp(L);
  for (int l = 0; l < L; ++l) {
    int64_t rb, re;
    dgraph_block(D, l, &rb, &re);
    const int32_t *lev, *par;
    bfs_shard_result_device(D->shard[l], &lev, &par);
    send[l].alloc(2 * mx);
    recv[l].alloc(2 * mx * P);
    if (re > rb) {
      k_pack_rows<<<ceil_div(re - rb, 256), 256, 0, c->stream>>>(lev, par, rb, re, send[l].p);
      GBX_LAUNCHED();
    }
    sp[l] = send[l].p;
    rp[l] = recv[l].p;
  }
  sync_shards(D);
  comm_sync(c);
  c_allgather(c, sp.data(), rp.data(), 2 * mx * sizeof(int32_t));
  DevArray<int64_t> db(P + 1), out(2 * std::max<int64_t>(n, 1));
  GBX_CUDA(cudaMemcpyAsync(db.p, D->bounds.data(), (P + 1) * 8, cudaMemcpyHostToDevice, c->stream));
  if (n) {
    k_unpack_rows<<<ceil_div(n, 256), 256, 0, c->stream>>>(recv[0].p, mx, db.p, P, n, out.p,
                                                           out.p + n);
    GBX_LAUNCHED();
  }
  if (level) GBX_CUDA(cudaMemcpyAsync(level, out.p, n * 8, cudaMemcpyDeviceToHost, c->stream));
  if (parent) GBX_CUDA(cudaMemcpyAsync(parent, out.p + n, n * 8, cudaMemcpyDeviceToHost, c->stream));
  comm_sync(c);
}

}  // namespace

void bfs_mg(gbx_dgraph* D, uint64_t source, int64_t* parent, int64_t* level) {
  NvtxRange nvtx_("gbx.bfs_mg");
  gbx_comm* c = D->comm;
  CommLock lk(c);
  const int L = c->nlocal, P = c->nranks;
  const int64_t n = D->n;
  if (source >= static_cast<uint64_t>(n)) fail(GBX_SOURCE_OUT_OF_RANGE, "source " + std::to_string(source));
  D->stats = gbx_stats{};
  for (int l = 0; l < L; ++l)
    bfs_shard_begin(D->shard[l], source, c->global_rank(l), P, nullptr, nullptr, D->bounds.data());
  const int64_t words = (n + 31) / 32;
  std::vector<int64_t> wb(P + 1);
  for (int q = 0; q < P; ++q) wb[q] = D->bounds[q] / 32;
  wb[P] = words;
  int64_t mw = 1;
  for (int q = 0; q < P; ++q) mw = std::max(mw, wb[q + 1] - wb[q]);
  std::vector<DevArray<uint32_t>> front(L), nxt(L), gat(L);
  std::vector<const void*> sp(L);
  std::vector<void*> rp(L);
  for (int l = 0; l < L; ++l) {
    front[l].alloc(std::max<int64_t>(words, 1));
    nxt[l].alloc(mw);
    gat[l].alloc(mw * P);
    GBX_CUDA(cudaMemsetAsync(front[l].p, 0, front[l].bytes(), c->stream));
    const uint32_t bit = 1u << (source & 31);
    GBX_CUDA(cudaMemcpyAsync(front[l].p + (source >> 5), &bit, 4, cudaMemcpyHostToDevice, c->stream));
    sp[l] = nxt[l].p;
    rp[l] = gat[l].p;
  }
  comm_sync(c);
  int levels = 0, pushes = 0;
  int64_t fcount = 1;  // frontier vertices (all ranks)
  std::vector<DevArray<uint8_t>> cand(L);
  std::vector<void*> cp(L);
  // direction: Beamer's edge rule as in gbx_bfs (push while the frontier's
  // edges are under nnz/alpha, option bfs.alpha), or bfs.cpp:77-78's vertex
  // rule (push while the frontier has fewer than n/div vertices) when the
  // option bfs_mg.push_div is set
  const int64_t div = option(kOptBfsMgPushDiv);
  const int64_t alpha = option(kOptBfsAlpha);
  const bool trace = option(kOptBfsTrace) != 0;
  for (;;) {
    const auto t0 = std::chrono::steady_clock::now();
    bool pushed = false;
    std::vector<int64_t> found(L, 0);
    bool push;
    if (div > 0 || alpha <= 0) {
      push = fcount * (div > 0 ? div : 16) < n;
    } else {
      std::vector<int64_t> fe(L, 0);
      for (int l = 0; l < L; ++l) fe[l] = bfs_shard_front_edges(D->shard[l], front[l].p);
      int64_t tot_e = 0;
      for (int64_t x : c_allgather_host(c, fe)) tot_e += x;  // the same sum on every rank
      push = tot_e * alpha < D->nnz;
    }
    if (push) {
      for (int l = 0; l < L; ++l) {
        if (!cand[l].p) cand[l].alloc(std::max<int64_t>(n, 1));
        GBX_CUDA(cudaMemsetAsync(cand[l].p, 0, n, c->stream));
        cp[l] = cand[l].p;
      }
      comm_sync(c);
      for (int l = 0; l < L; ++l) bfs_shard_push_mark(D->shard[l], front[l].p, cand[l].p);
      c_allreduce(c, cp.data(), n, CollType::U8, CollOp::Max);  // the OR of every rank's marks
      for (int l = 0; l < L; ++l)
        bfs_shard_push_level(D->shard[l], cand[l].p, front[l].p, nxt[l].p, &found[l]);
      ++pushes;
      pushed = true;
    } else {
      for (int l = 0; l < L; ++l) bfs_shard_level(D->shard[l], front[l].p, nxt[l].p, &found[l]);
    }
    const std::vector<int64_t> all = c_allgather_host(c, found);
    int64_t tot = 0;
    for (int64_t x : all) tot += x;
    ++levels;
    if (trace)
      std::fprintf(stderr, "bfs_mg level %d %s frontier %lld -> found %lld  %.1f us\n", levels,
                   pushed ? "push" : "pull", static_cast<long long>(fcount),
                   static_cast<long long>(tot),
                   std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
    if (tot == 0) break;
    fcount = tot;
    // the frontier-bitmap all-gather (north_star): every rank's slice in place
    c_allgather(c, sp.data(), rp.data(), mw * 4);
    for (int l = 0; l < L; ++l)
      for (int q = 0; q < P; ++q)
        if (wb[q + 1] > wb[q])
          GBX_CUDA(cudaMemcpyAsync(front[l].p + wb[q], gat[l].p + q * mw, (wb[q + 1] - wb[q]) * 4,
                                   cudaMemcpyDeviceToDevice, c->stream));
    comm_sync(c);
  }
  D->stats.iterations = levels;
  D->stats.launches = (2 * levels + 3 * pushes) * L;
  D->stats.hot_launches = levels * L;
  if (!parent && !level) return;  // the result stays distributed over the ranks
  // every rank's owned slice of level / parent, gathered on the device
  gather_bfs_result(D, parent, level);
}

// ---- betweenness -------------------------------------------------------------------

void betweenness_mg(gbx_dgraph* D, const uint64_t* sources, uint64_t ns, double* centrality) {
  NvtxRange nvtx_("gbx.betweenness_mg");
  gbx_comm* c = D->comm;
  CommLock lk(c);
  const int L = c->nlocal, P = c->nranks;
  const int64_t n = D->n;
  if (ns == 0) fail(GBX_EMPTY_BATCH, "empty source batch");
  if (!sources) fail(GBX_NULL_ARGUMENT, "sources is NULL");
  for (uint64_t b = 0; b < ns; ++b)
    if (sources[b] >= static_cast<uint64_t>(n)) fail(GBX_SOURCE_OUT_OF_RANGE, "source " + std::to_string(sources[b]));
  D->stats = gbx_stats{};
  constexpr size_t kRec = 40;  // BcRec (bc.cu)
  std::vector<DevArray<double>> acc(L);
  for (int l = 0; l < L; ++l) {
    acc[l].alloc(std::max<int64_t>(n, 1));
    GBX_CUDA(cudaMemsetAsync(acc[l].p, 0, acc[l].bytes(), c->stream));
  }
  comm_sync(c);
  int levels = 0, cand_levels = 0;
  std::vector<DevArray<uint8_t>> all, cand(L);
  std::vector<void*> cp(L);
  const int64_t alpha = option(kOptBcAlpha);
  for (uint64_t b0 = 0; b0 < ns; b0 += 4) {  // batches of 4 (the lane width)
    const uint64_t nb = std::min<uint64_t>(4, ns - b0);
    for (int l = 0; l < L; ++l)
      bc_shard_begin(D->shard[l], sources + b0, nb, c->global_rank(l), P, nullptr, nullptr,
                     D->bounds.data());
    for (;;) {  // forward: one record exchange per depth
      std::vector<const void*> recs(L);
      std::vector<int64_t> nrec(L);
      // direction: while the settled depth's edges are under nnz/alpha (the
      // single-GPU push rule) the ranks pull only the marked candidates
      std::vector<int64_t> fe(L, 0);
      for (int l = 0; l < L; ++l) fe[l] = bc_shard_mark(D->shard[l], nullptr);
      int64_t tot_e = 0;
      for (int64_t x : c_allgather_host(c, fe)) tot_e += x;
      const bool candidates = alpha > 0 && tot_e * alpha < D->nnz;
      if (candidates) {
        for (int l = 0; l < L; ++l) {
          if (!cand[l].p) cand[l].alloc(std::max<int64_t>(n, 1));
          GBX_CUDA(cudaMemsetAsync(cand[l].p, 0, n, c->stream));
          cp[l] = cand[l].p;
        }
        comm_sync(c);
        for (int l = 0; l < L; ++l) bc_shard_mark(D->shard[l], cand[l].p);
        c_allreduce(c, cp.data(), n, CollType::U8, CollOp::Max);
        ++cand_levels;
      }
      for (int l = 0; l < L; ++l) {
        void* p = nullptr;
        bc_shard_forward(D->shard[l], &p, &nrec[l], candidates ? cand[l].p : nullptr);
        recs[l] = p;
      }
      const int64_t tot = gather_records(c, recs, nrec, kRec, all);
      int done = 0;
      for (int l = 0; l < L; ++l) bc_shard_forward_apply(D->shard[l], tot ? all[l].p : nullptr, tot, &done);
      ++levels;
      D->stats.launches += 4 * L;  // pull (+ hub passes), pack, apply
      if (done) break;
    }
    for (;;) {  // backward
      std::vector<const void*> recs(L);
      std::vector<int64_t> nrec(L);
      int done = 0;
      for (int l = 0; l < L; ++l) {
        void* p = nullptr;
        bc_shard_backward(D->shard[l], &p, &nrec[l], &done);
        recs[l] = p;
      }
      if (done) break;
      const int64_t tot = gather_records(c, recs, nrec, kRec, all);
      for (int l = 0; l < L; ++l) bc_shard_backward_apply(D->shard[l], tot ? all[l].p : nullptr, tot);
      ++levels;
      D->stats.launches += 6 * L;  // map, filter, bins, back (+ hub passes), pack, apply
    }
    for (int l = 0; l < L; ++l) {
      double* cent = nullptr;
      bc_shard_centrality(D->shard[l], &cent);
      if (n) {
        k_axpy1<<<ceil_div(n, 256), 256, 0, c->stream>>>(acc[l].p, cent, n);
        GBX_LAUNCHED();
      }
    }
    comm_sync(c);
  }
  std::vector<void*> ap(L);
  for (int l = 0; l < L; ++l) ap[l] = acc[l].p;
  c_allreduce(c, ap.data(), n, CollType::F64, CollOp::Sum);
  D->stats.iterations = levels;
  D->stats.hot_launches = cand_levels;
  D->stats.work_units = D->nnz;
  if (centrality && n) GBX_CUDA(cudaMemcpy(centrality, acc[0].p, n * 8, cudaMemcpyDeviceToHost));
}

}  // namespace gbx
