// dgraph.cu -- distributed graph construction: every rank builds ONLY its own
// row block of A (and of AT for a directed graph), SURVEY.md §2.2 "shards are
// built locally".
//
// The reference builds one matrix (build_matrix, containers.cpp:128-169: sort
// the tuples, combine duplicates) and the graph caches it (graph.cpp:16-41).
// Distributed, the same three steps run per rank:
//   1. keys: each rank produces (row << bits | col) keys for its SLICE of the
//      input -- generated edges [e0, e1) of the seeded R-MAT stream, or the
//      rows of a CSR block the caller holds -- symmetrised for an undirected
//      graph, self-loops as the drop key (sorts last);
//   2. layout: a histogram of rows per 32-row bucket, all-reduced, gives every
//      rank the same ownership bounds (32-aligned, balanced by rows + entries);
//   3. shuffle: the sorted keys are cut at the bounds and exchanged (NCCL
//      grouped send/recv = all-to-all-v); the received runs are sorted and
//      de-duplicated into the owner's CSR block.
// A directed graph repeats 3 with transposed keys for the AT block.
// Memory per rank: its slice of the keys + its block -- no full replica.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>

#include "comm.cuh"
#include "plans.cuh"

gbx_dgraph::~gbx_dgraph() {
  for (gbx_graph* g : shard) delete g;
}

namespace gbx {

namespace {

__global__ void k_bucket_hist(const uint64_t* keys, int64_t m, int bits, unsigned long long* hist) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < m) atomicAdd(&hist[(keys[i] >> bits) >> 5], 1ull);
}

// pos[q] = first sorted key with row >= bounds[q] (q = 0..P; bounds[P] = n,
// so pos[P] = the first drop key = the number of valid keys)
__global__ void k_key_cuts(const uint64_t* keys, int64_t m, const int64_t* bounds, int P, int bits,
                           int64_t* pos) {
  const int q = threadIdx.x;
  if (q > P) return;
  const uint64_t target = static_cast<uint64_t>(bounds[q]) << bits;
  int64_t lo = 0, hi = m;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < target) lo = mid + 1; else hi = mid;
  }
  pos[q] = lo;
}

__global__ void k_transpose_keys(uint64_t* keys, int64_t m, int bits) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= m) return;
  const uint64_t k = keys[i];
  const uint64_t drop = uint64_t(1) << (2 * bits);
  if (k == drop) return;
  const uint64_t mask = (uint64_t(1) << bits) - 1;
  keys[i] = ((k & mask) << bits) | (k >> bits);
}

// CSR block rows [rb, re) (host row_ptr of re - rb + 1, global cols) -> keys
__global__ void k_block_keys(const int64_t* rp, const int32_t* col, int64_t rb, int64_t rows,
                             int bits, int sym, int64_t n, uint64_t* keys, int* bad) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const uint64_t drop = uint64_t(1) << (2 * bits);
  for (int64_t r = w; r < rows; r += nw) {
    const uint64_t u = static_cast<uint64_t>(rb + r);
    for (int64_t p = rp[r] - rp[0] + lane; p < rp[r + 1] - rp[0]; p += 32) {
      const int32_t c = col[p];
      if (c < 0 || c >= n) { atomicExch(bad, 1); continue; }
      const uint64_t v = static_cast<uint64_t>(c);
      if (sym) {
        keys[2 * p] = u == v ? drop : ((u << bits) | v);
        keys[2 * p + 1] = u == v ? drop : ((v << bits) | u);
      } else {
        keys[p] = u == v ? drop : ((u << bits) | v);
      }
    }
  }
}

}  // namespace

void sort_in_place(cudaStream_t s, KeyBlock& K, int bits) {
  if (K.m <= 1) return;
  DevArray<uint64_t> alt(K.m);
  uint64_t* r = sort_keys(s, K.k.p, alt.p, K.m, 2 * bits + 1);
  if (r != K.k.p) K.k = std::move(alt);
  GBX_CUDA(cudaStreamSynchronize(s));
}

namespace {

// ownership bounds from the all-reduced 32-row bucket histogram
std::vector<int64_t> layout(gbx_comm* c, const std::vector<KeyBlock>& keys, int64_t n, int bits) {
  const int64_t nb = (n + 31) / 32;
  std::vector<DevArray<unsigned long long>> hist(c->nlocal);
  std::vector<void*> hp(c->nlocal);
  for (int l = 0; l < c->nlocal; ++l) {
    hist[l].alloc(std::max<int64_t>(nb, 1));
    GBX_CUDA(cudaMemsetAsync(hist[l].p, 0, hist[l].bytes(), c->stream));
    // drop keys are row n (past the last bucket): count only the valid prefix
    if (keys[l].m) {
      Tmp<int64_t> pos(2, c->stream);
      Tmp<int64_t> b(2, c->stream);
      const int64_t hb[2] = {0, n};
      GBX_CUDA(cudaMemcpyAsync(b.p, hb, sizeof hb, cudaMemcpyHostToDevice, c->stream));
      k_key_cuts<<<1, 32, 0, c->stream>>>(keys[l].k.p, keys[l].m, b.p, 1, bits, pos.p);
      int64_t hpos[2];
      GBX_CUDA(cudaMemcpyAsync(hpos, pos.p, sizeof hpos, cudaMemcpyDeviceToHost, c->stream));
      GBX_CUDA(cudaStreamSynchronize(c->stream));
      if (hpos[1])
        k_bucket_hist<<<ceil_div(hpos[1], 256), 256, 0, c->stream>>>(keys[l].k.p, hpos[1], bits,
                                                                     hist[l].p);
      GBX_LAUNCHED();
    }
    hp[l] = hist[l].p;
  }
  comm_sync(c);
  c_allreduce(c, hp.data(), nb, CollType::U64, CollOp::Sum);
  std::vector<unsigned long long> h(std::max<int64_t>(nb, 1));
  GBX_CUDA(cudaMemcpy(h.data(), hist[0].p, nb * 8, cudaMemcpyDeviceToHost));
  unsigned long long total = 0;
  for (int64_t i = 0; i < nb; ++i) total += h[i];
  const int P = c->nranks;
  std::vector<int64_t> bounds(P + 1, n);
  bounds[0] = 0;
  // every rank runs this on the same data: identical bounds everywhere
  int64_t acc = 0, b = 0;
  for (int q = 1; q < P; ++q) {
    const double target = (static_cast<double>(n) + static_cast<double>(total)) * q / P;
    while (b < nb && static_cast<double>(acc) < target) {
      acc += std::min<int64_t>(32, n - b * 32) + static_cast<int64_t>(h[b]);
      ++b;
    }
    bounds[q] = std::max(bounds[q - 1], std::min(n, b * 32));
  }
  return bounds;
}

}  // namespace

// sorted keys of every local rank -> the owner's sorted, de-duplicated CSR block
void shuffle_to_blocks(gbx_comm* c, std::vector<KeyBlock>& keys, const std::vector<int64_t>& bounds,
                       int64_t n, int bits, std::vector<Csr*>& out) {
  NvtxRange nvtx_("gbx.dgraph.shuffle");
  const int P = c->nranks, L = c->nlocal;
  std::vector<std::vector<int64_t>> cnt(L, std::vector<int64_t>(P, 0));
  std::vector<std::vector<int64_t>> soff(L, std::vector<int64_t>(P + 1, 0));
  Tmp<int64_t> db(P + 1, c->stream);
  GBX_CUDA(cudaMemcpyAsync(db.p, bounds.data(), (P + 1) * 8, cudaMemcpyHostToDevice, c->stream));
  for (int l = 0; l < L; ++l) {
    std::vector<int64_t> pos(P + 1, 0);
    if (keys[l].m) {
      Tmp<int64_t> dpos(P + 1, c->stream);
      k_key_cuts<<<1, 32, 0, c->stream>>>(keys[l].k.p, keys[l].m, db.p, P, bits, dpos.p);
      GBX_LAUNCHED();
      GBX_CUDA(cudaMemcpyAsync(pos.data(), dpos.p, (P + 1) * 8, cudaMemcpyDeviceToHost, c->stream));
      GBX_CUDA(cudaStreamSynchronize(c->stream));
    }
    for (int q = 0; q < P; ++q) {
      cnt[l][q] = pos[q + 1] - pos[q];
      soff[l][q] = pos[q] * 8;
    }
    soff[l][P] = pos[P] * 8;
  }
  const std::vector<std::vector<int64_t>> rcnt = c_exchange_counts(c, cnt);
  std::vector<std::vector<int64_t>> roff(L, std::vector<int64_t>(P + 1, 0));
  std::vector<KeyBlock> recv(L);
  std::vector<const void*> sp(L);
  std::vector<void*> rp(L);
  for (int l = 0; l < L; ++l) {
    for (int q = 0; q < P; ++q) roff[l][q + 1] = roff[l][q] + rcnt[l][q] * 8;
    recv[l].m = roff[l][P] / 8;
    recv[l].k.alloc(std::max<int64_t>(recv[l].m, 1));
    sp[l] = keys[l].k.p;
    rp[l] = recv[l].k.p;
  }
  c_alltoallv(c, sp.data(), soff, rp.data(), roff);
  for (int l = 0; l < L; ++l) {
    keys[l].k.release();
    keys[l].m = 0;
    sort_in_place(c->stream, recv[l], bits);
    csr_from_keys_unique(c->stream, n, bits, recv[l].k.p, recv[l].m, *out[l]);
  }
}

namespace {

gbx_dgraph* dgraph_from_keys(gbx_comm* c, int64_t n, int bits, int kind, std::vector<KeyBlock>& keys) {
  auto D = std::make_unique<gbx_dgraph>();
  D->comm = c;
  D->device = c->device;
  D->n = n;
  D->kind = kind;
  for (int l = 0; l < c->nlocal; ++l) sort_in_place(c->stream, keys[l], bits);
  D->bounds = layout(c, keys, n, bits);
  D->shard.assign(c->nlocal, nullptr);
  for (int l = 0; l < c->nlocal; ++l) {
    D->shard[l] = graph_handle();
    D->shard[l]->kind = kind;
  }
  // the AT block first (a directed graph needs the transposed keys)
  if (kind == GBX_DIRECTED) {
    std::vector<KeyBlock> tk(c->nlocal);
    for (int l = 0; l < c->nlocal; ++l) {
      tk[l].m = keys[l].m;
      tk[l].k.alloc(std::max<int64_t>(keys[l].m, 1));
      if (keys[l].m) {
        GBX_CUDA(cudaMemcpyAsync(tk[l].k.p, keys[l].k.p, keys[l].m * 8, cudaMemcpyDeviceToDevice,
                                 c->stream));
        k_transpose_keys<<<ceil_div(keys[l].m, 256), 256, 0, c->stream>>>(tk[l].k.p, keys[l].m, bits);
        GBX_LAUNCHED();
      }
      sort_in_place(c->stream, tk[l], bits);
    }
    std::vector<Csr*> at(c->nlocal);
    for (int l = 0; l < c->nlocal; ++l) at[l] = &D->shard[l]->at_own;
    shuffle_to_blocks(c, tk, D->bounds, n, bits, at);
  }
  std::vector<Csr*> a(c->nlocal);
  for (int l = 0; l < c->nlocal; ++l) a[l] = &D->shard[l]->A;
  shuffle_to_blocks(c, keys, D->bounds, n, bits, a);
  D->local_nnz.resize(c->nlocal);
  for (int l = 0; l < c->nlocal; ++l) {
    D->shard[l]->has_at = true;  // owned rows of AT: at_own (directed) / A itself (undirected)
    D->local_nnz[l] = D->shard[l]->A.nnz;
  }
  const std::vector<int64_t> all = c_allgather_host(c, D->local_nnz);
  D->nnz = 0;
  for (int64_t x : all) D->nnz += x;
  return D.release();
}

}  // namespace

gbx_dgraph* dgraph_generate_rmat(gbx_comm* c, int scale, int ef, double a, double b, double cc,
                                 uint64_t seed, int scramble, int kind) {
  NvtxRange nvtx_("gbx.dgraph.generate_rmat");
  if (kind != GBX_DIRECTED && kind != GBX_UNDIRECTED) fail(GBX_INVALID_VALUE, "rmat: unknown kind");
  if (scale < 1 || scale > 30) fail(GBX_INVALID_VALUE, "rmat: scale must be in [1,30]");
  if (ef < 1) fail(GBX_INVALID_VALUE, "rmat: edge factor must be >= 1");
  GBX_CUDA(cudaSetDevice(c->device));
  const int64_t n = int64_t(1) << scale;
  const int64_t m = int64_t(ef) << scale;
  const bool sym = kind == GBX_UNDIRECTED;
  std::vector<KeyBlock> keys(c->nlocal);
  for (int l = 0; l < c->nlocal; ++l) {
    // this rank's slice of the edge stream
    const int q = c->global_rank(l);
    const int64_t e0 = m * q / c->nranks, e1 = m * (q + 1) / c->nranks;
    keys[l].m = (e1 - e0) * (sym ? 2 : 1);
    keys[l].k.alloc(std::max<int64_t>(keys[l].m, 1));
    rmat_keys(c->stream, scale, ef, a, b, cc, seed, scramble, sym, e0, e1, keys[l].k.p);
  }
  comm_sync(c);
  return dgraph_from_keys(c, n, scale, kind, keys);
}

gbx_dgraph* dgraph_from_blocks(gbx_comm* c, int64_t n, const int64_t* row_begin,
                               const int64_t* row_end, const int64_t* const* row_ptr,
                               const int32_t* const* col, int kind) {
  NvtxRange nvtx_("gbx.dgraph.from_blocks");
  if (kind != GBX_DIRECTED && kind != GBX_UNDIRECTED) fail(GBX_INVALID_VALUE, "dgraph: unknown kind");
  if (n < 0 || n >= (int64_t(1) << 31)) fail(GBX_INVALID_VALUE, "dgraph: n out of range");
  if (!row_begin || !row_end || !row_ptr || !col) fail(GBX_NULL_ARGUMENT, "dgraph: NULL block array");
  GBX_CUDA(cudaSetDevice(c->device));
  const int bits = bits_for(std::max<int64_t>(n, 2));
  const bool sym = kind == GBX_UNDIRECTED;
  std::vector<KeyBlock> keys(c->nlocal);
  for (int l = 0; l < c->nlocal; ++l) {
    const int64_t rb = row_begin[l], re = row_end[l];
    if (rb < 0 || re < rb || re > n) fail(GBX_INDEX_OUT_OF_BOUNDS, "dgraph: block rows out of range");
    const int64_t rows = re - rb;
    if (rows && !row_ptr[l]) fail(GBX_NULL_ARGUMENT, "dgraph: NULL row_ptr");
    const int64_t nnz = rows ? row_ptr[l][rows] - row_ptr[l][0] : 0;
    for (int64_t r = 0; r < rows; ++r)
      if (row_ptr[l][r + 1] < row_ptr[l][r]) fail(GBX_INVALID_MATRIX, "dgraph: row_ptr not monotone");
    keys[l].m = nnz * (sym ? 2 : 1);
    keys[l].k.alloc(std::max<int64_t>(keys[l].m, 1));
    if (nnz) {
      Tmp<int64_t> drp(rows + 1, c->stream);
      Tmp<int32_t> dcol(nnz, c->stream);
      Tmp<int> bad(1, c->stream);
      GBX_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), c->stream));
      GBX_CUDA(cudaMemcpyAsync(drp.p, row_ptr[l], (rows + 1) * 8, cudaMemcpyHostToDevice, c->stream));
      GBX_CUDA(cudaMemcpyAsync(dcol.p, col[l], nnz * 4, cudaMemcpyHostToDevice, c->stream));
      k_block_keys<<<device_sms() * 8, 256, 0, c->stream>>>(drp.p, dcol.p, rb, rows, bits,
                                                            sym ? 1 : 0, n, keys[l].k.p, bad.p);
      GBX_LAUNCHED();
      int hb = 0;
      GBX_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      GBX_CUDA(cudaStreamSynchronize(c->stream));
      if (hb) fail(GBX_INDEX_OUT_OF_BOUNDS, "dgraph: column index out of range");
    }
  }
  comm_sync(c);
  return dgraph_from_keys(c, n, bits, kind, keys);
}

// the owned row range of local rank l
void dgraph_block(const gbx_dgraph* D, int l, int64_t* rb, int64_t* re) {
  const int q = D->comm->global_rank(l);
  *rb = D->bounds[q];
  *re = D->bounds[q + 1];
}

}  // namespace gbx
