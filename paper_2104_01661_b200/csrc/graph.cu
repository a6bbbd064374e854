// graph.cu -- the device CSR store and the Graph-object caches.
//
// Restates gblite's graph layer (graph.cpp:16-110, containers.cpp:104-169,
// core.cpp:237-256, util.cpp:35-44) for HBM: CSR with int64 row_ptr and int32
// columns, transpose / dedup / symmetrise by CUB radix sort instead of the
// reference's counting sort and std::stable_sort, degrees by one pass over
// row_ptr (rows) or one atomic histogram (columns).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstring>

#include "common.cuh"
#include "sort.cuh"

namespace gbx {

void cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  (void)cudaGetLastError();
  char buf[256];
  std::snprintf(buf, sizeof buf, "CUDA error %s (%s) at %s:%d", cudaGetErrorName(e), what,
                file, line);
  fail(e == cudaErrorMemoryAllocation ? GBX_OUT_OF_MEMORY : GBX_CUDA_ERROR, buf);
}

int device_sms() {
  int dev = 0, sms = 0;
  GBX_CUDA(cudaGetDevice(&dev));
  GBX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  return sms;
}

size_t domain_size(int d) {
  switch (d) {
    case GBX_BOOL: return 1;
    case GBX_INT32: return 4;
    case GBX_INT64:
    case GBX_UINT64:
    case GBX_FP64: return 8;
  }
  fail(GBX_DOMAIN_MISMATCH, "unknown value domain " + std::to_string(d));
}

Scope::Scope(gbx_graph* g) : lock(g->mu) {
  GBX_CUDA(cudaSetDevice(g->device));
  // keep freed stream-ordered temporaries cached in the device pool (the default
  // threshold returns them to the driver at every synchronisation)
  static bool pooled[64] = {false};
  if (g->device >= 0 && g->device < 64 && !pooled[g->device]) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, g->device) == cudaSuccess) {
      uint64_t thr = ~uint64_t(0);
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    (void)cudaGetLastError();
    pooled[g->device] = true;
  }
}

void sync(gbx_graph* g) { GBX_CUDA(cudaStreamSynchronize(g->stream)); }

}  // namespace gbx

// the deferred transpose of property_at (the handle's calls are serialised by
// its Scope lock, so materialising inside a const accessor is race-free)
void gbx_graph::materialize_at() const {
  gbx::NvtxRange nvtx_("gbx.property_at.transpose");
  gbx_graph* g = const_cast<gbx_graph*>(this);
  gbx::compute_transpose(g->stream, g->A, g->at_own);
  GBX_CUDA(cudaStreamSynchronize(g->stream));
  g->at_pending = false;
}

namespace gbx {

void require_at(const gbx_graph* g, const char* who) {
  if (!g->has_at) fail(GBX_MISSING_PROPERTY, std::string(who) + " needs G.AT");
}
void require_rowdeg(const gbx_graph* g, const char* who) {
  if (!g->has_rowdeg) fail(GBX_MISSING_PROPERTY, std::string(who) + " needs G.row_degree");
}

int bits_for(int64_t n) {
  int b = 1;
  while ((int64_t(1) << b) < n) ++b;
  return b;
}

// ---- validation (containers.cpp:104-124) -------------------------------------

__global__ void k_validate_rows(const int64_t* rp, int64_t n, int64_t nnz, uint8_t* head,
                                int* bad) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  int64_t b = rp[i], e = rp[i + 1];
  if (b > e || b < 0 || e > nnz) { atomicOr(bad, 1); return; }
  if (b < e) head[b] = 1;
}

__global__ void k_convert_cols(const int64_t* c64, int32_t* c32, int64_t nnz, int64_t n,
                               int* bad) {
  int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p >= nnz) return;
  int64_t c = c64[p];
  if (c < 0 || c >= n) { atomicOr(bad, 2); c = 0; }
  c32[p] = static_cast<int32_t>(c);
}

// entries [p0, p1): range and strictly-ascending-within-row checks; count != 0
// also counts the columns (in-degrees)
__global__ void k_validate_cols(const int32_t* col, const uint8_t* head, int64_t p0, int64_t p1,
                                int64_t nnz, int64_t n, int* bad, int32_t* count) {
  const int64_t p = p0 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p >= p1) return;
  const int32_t c = col[p];
  if (c < 0 || c >= n) {
    atomicOr(bad, 2);
  } else if (count) {
    atomicAdd(&count[c], 1);
  }
  if (p > 0 && !head[p] && col[p - 1] >= c) atomicOr(bad, 4);
}

void build_from_host(gbx_graph* g, int64_t n, const int64_t* rp, const int64_t* col64,
                     const int32_t* col32, const void* vals, int domain, int kind) {
  NvtxRange nvtx_("gbx.graph_new");
  if (n < 0) fail(GBX_INVALID_MATRIX, "graph_new: negative dimension");
  if (n >= (int64_t(1) << 31) - 1)
    fail(GBX_UNSUPPORTED, "graph_new: n >= 2^31 is not supported by the int32 column layout");
  if (kind != GBX_DIRECTED && kind != GBX_UNDIRECTED)
    fail(GBX_INVALID_VALUE, "graph_new: unknown kind");
  if (vals) (void)domain_size(domain);
  else domain = GBX_BOOL;
  if (!rp) fail(GBX_NULL_ARGUMENT, "graph_new: row_ptr is NULL");
  if (rp[0] != 0) fail(GBX_INVALID_MATRIX, "graph_new: row_ptr[0] is not 0");
  int64_t nnz = rp[n];
  if (nnz < 0) fail(GBX_INVALID_MATRIX, "graph_new: row_ptr[nrows] is negative");
  if (nnz > 0 && !col64 && !col32) fail(GBX_NULL_ARGUMENT, "graph_new: col_idx is NULL");
  cudaStream_t s = g->stream;
  Csr& A = g->A;
  A.n = n;
  A.nnz = nnz;
  A.domain = domain;
  A.rp.alloc(n + 1);
  A.col.alloc(std::max<int64_t>(nnz, 1));
  GBX_CUDA(cudaMemcpyAsync(A.rp.p, rp, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  Tmp<int> bad(1, s);
  GBX_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
  if (nnz > 0) {
    if (col64) {
      Tmp<int64_t> c64(nnz, s);
      GBX_CUDA(cudaMemcpyAsync(c64.p, col64, nnz * sizeof(int64_t), cudaMemcpyHostToDevice, s));
      k_convert_cols<<<ceil_div(nnz, 256), 256, 0, s>>>(c64.p, A.col.p, nnz, n, bad.p);
      GBX_LAUNCHED();
    }
  }
  if (vals && nnz > 0) {
    size_t es = domain_size(domain);
    A.val.alloc(nnz * es);
    GBX_CUDA(cudaMemcpyAsync(A.val.p, vals, nnz * es, cudaMemcpyHostToDevice, s));
  }
  if (n > 0) {
    Tmp<uint8_t> head(std::max<int64_t>(nnz, 1), s);
    GBX_CUDA(cudaMemsetAsync(head.p, 0, std::max<int64_t>(nnz, 1), s));
    k_validate_rows<<<ceil_div(n, 256), 256, 0, s>>>(A.rp.p, n, nnz, head.p, bad.p);
    GBX_LAUNCHED();
    if (nnz > 0 && col64) {
      k_validate_cols<<<ceil_div(nnz, 256), 256, 0, s>>>(A.col.p, head.p, 0, nnz, nnz, n, bad.p,
                                                         nullptr);
      GBX_LAUNCHED();
    } else if (nnz > 0) {
      // int32 columns: the stream goes up in chunks on a copy stream while the
      // graph's stream validates the chunks that have arrived and counts the
      // columns (= in-degrees, kept for the PageRank plan) -- both hide behind
      // the PCIe transfer instead of following it
      g->colcount.alloc(n);
      GBX_CUDA(cudaMemsetAsync(g->colcount.p, 0, n * sizeof(int32_t), s));
      cudaStream_t cs = nullptr;
      GBX_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      const int64_t chunk = int64_t(8) << 20;  // entries (32 MB)
      std::vector<cudaEvent_t> ev;
      cudaError_t err = cudaSuccess;
      for (int64_t off = 0; off < nnz && err == cudaSuccess; off += chunk) {
        const int64_t len = std::min(chunk, nnz - off);
        cudaEvent_t e = nullptr;
        err = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        if (err != cudaSuccess) break;
        ev.push_back(e);
        err = cudaMemcpyAsync(A.col.p + off, col32 + off, len * sizeof(int32_t),
                              cudaMemcpyHostToDevice, cs);
        if (err == cudaSuccess) err = cudaEventRecord(e, cs);
        if (err == cudaSuccess) err = cudaStreamWaitEvent(s, e, 0);
        if (err != cudaSuccess) break;
        // the chunk's first entry is compared with its predecessor, which an
        // earlier chunk brought (stream order)
        k_validate_cols<<<ceil_div(len, 256), 256, 0, s>>>(A.col.p, head.p, off, off + len, nnz, n,
                                                         bad.p, g->colcount.p);
        err = cudaGetLastError();
      }
      if (err == cudaSuccess) err = cudaStreamSynchronize(s);
      (void)cudaStreamSynchronize(cs);
      for (cudaEvent_t e : ev) (void)cudaEventDestroy(e);
      (void)cudaStreamDestroy(cs);
      GBX_CUDA(err);
      g->has_colcount = true;
    }
  }
  int hbad = 0;
  GBX_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  if (hbad & 1) fail(GBX_INVALID_MATRIX, "graph_new: row_ptr not nondecreasing");
  if (hbad & 2) fail(GBX_INVALID_MATRIX, "graph_new: column index out of range");
  if (hbad & 4) fail(GBX_INVALID_MATRIX, "graph_new: row columns not strictly increasing");
  g->kind = kind;
}

// ---- row expansion, degrees, transpose ---------------------------------------

__global__ void k_mark_row_starts(const int64_t* rp, int64_t n, int32_t* rowid) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  if (rp[i] < rp[i + 1]) rowid[rp[i]] = static_cast<int32_t>(i);
}

struct MaxOp {
  __device__ __forceinline__ int32_t operator()(int32_t a, int32_t b) const { return a > b ? a : b; }
};

// Sorted (row<<bits|col) keys -> col and row_ptr, fully parallel and without
// atomics: the LAST entry of each row's run writes end[row + 1] = p + 1 (into a
// zeroed array), then row_ptr = inclusive max-scan of end (empty rows inherit
// the previous end).  Replaces a per-row atomic count (same-address
// serialisation: 7 ms at 65M keys) and a boundary fill whose final thread
// wrote every trailing empty row (8 ms when half the rows are empty).
struct MaxOp64 {
  __device__ __forceinline__ int64_t operator()(int64_t a, int64_t b) const { return a > b ? a : b; }
};

__global__ void k_row_ends64(const uint64_t* keys, int64_t nnz, int bits, int32_t* col,
                             int64_t* end) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p >= nnz) return;
  const uint64_t k = keys[p];
  if (col) col[p] = static_cast<int32_t>(k & ((uint64_t(1) << bits) - 1));
  const uint64_t r = k >> bits;
  if (p == nnz - 1 || (keys[p + 1] >> bits) != r) end[r + 1] = p + 1;
}

__global__ void k_row_ends32(const uint32_t* rows, int64_t nnz, int64_t* end) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p >= nnz) return;
  const uint32_t r = rows[p];
  if (p == nnz - 1 || rows[p + 1] != r) end[static_cast<int64_t>(r) + 1] = p + 1;
}

static void max_scan_rowptr(cudaStream_t s, int64_t* rp, int64_t n) {
  size_t tb = 0;
  GBX_CUDA(cub::DeviceScan::InclusiveScan(nullptr, tb, rp, rp, MaxOp64(), n + 1, s));
  Tmp<uint8_t> t(tb, s);
  GBX_CUDA(cub::DeviceScan::InclusiveScan(t.p, tb, rp, rp, MaxOp64(), n + 1, s));
}

void expand_rows_into(cudaStream_t s, const Csr& A, int32_t* rowid) {
  if (A.nnz == 0) return;
  GBX_CUDA(cudaMemsetAsync(rowid, 0, A.nnz * sizeof(int32_t), s));
  k_mark_row_starts<<<ceil_div(A.n, 256), 256, 0, s>>>(A.rp.p, A.n, rowid);
  GBX_LAUNCHED();
  size_t tb = 0;
  GBX_CUDA(cub::DeviceScan::InclusiveScan(nullptr, tb, rowid, rowid, MaxOp(), A.nnz, s));
  Tmp<uint8_t> t(tb, s);
  GBX_CUDA(cub::DeviceScan::InclusiveScan(t.p, tb, rowid, rowid, MaxOp(), A.nnz, s));
}

void expand_rows(cudaStream_t s, const Csr& A, DevArray<int32_t>& rowid) {
  rowid.alloc(std::max<int64_t>(A.nnz, 1));
  expand_rows_into(s, A, rowid.p);
}

__global__ void k_row_degree(const int64_t* rp, int64_t n, int32_t* deg) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) deg[i] = static_cast<int32_t>(rp[i + 1] - rp[i]);
}

__global__ void k_col_count(const int32_t* col, int64_t nnz, int32_t* cnt) {
  int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p < nnz) atomicAdd(&cnt[col[p]], 1);
}

void compute_degrees(cudaStream_t s, const Csr& A, DevArray<int32_t>& out, bool by_row) {
  out.alloc(std::max<int64_t>(A.n, 1));
  if (A.n == 0) return;
  if (by_row) {
    k_row_degree<<<ceil_div(A.n, 256), 256, 0, s>>>(A.rp.p, A.n, out.p);
  } else {
    GBX_CUDA(cudaMemsetAsync(out.p, 0, A.n * sizeof(int32_t), s));
    if (A.nnz) k_col_count<<<ceil_div(A.nnz, 256), 256, 0, s>>>(A.col.p, A.nnz, out.p);
  }
  GBX_LAUNCHED();
}

// row_ptr from a count array (exclusive scan into int64)

__global__ void k_iota64(int64_t* x, int64_t n) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) x[i] = i;
}

// T(q) <- A(p) for the sorted order p = perm[q]: T.col = row of p, values copied
template <int ES>
__global__ void k_gather_transpose(const int64_t* perm, const int32_t* rowid, int64_t nnz,
                                   int32_t* tcol, const uint8_t* val, uint8_t* tval) {
  const int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (q >= nnz) return;
  const int64_t p = perm[q];
  tcol[q] = rowid[p];
  const uint8_t* src = val + p * ES;
  uint8_t* dst = tval + q * ES;
#pragma unroll
  for (int b = 0; b < ES; ++b) dst[b] = src[b];
}

// T = transpose(A): plain_transpose (core.cpp:237-256) as ONE stable radix
// sort of the column ids (bits_for(n) bits, 32-bit keys) carrying the row id:
// A is row-major with ascending rows, so the stable sort leaves every row of T
// strictly ascending.  Row pointers come from the sorted keys' boundaries.
void compute_transpose(cudaStream_t s, const Csr& A, Csr& T) {
  gbx::NvtxRange nvtx_("gbx.property_at.transpose");
  T.n = A.n;
  T.nnz = A.nnz;
  T.domain = A.domain;
  T.rp.alloc(A.n + 1);
  T.col.alloc(std::max<int64_t>(A.nnz, 1));
  if (A.nnz == 0) {
    GBX_CUDA(cudaMemsetAsync(T.rp.p, 0, (A.n + 1) * sizeof(int64_t), s));
    return;
  }
  Tmp<int32_t> rowid(A.nnz, s);
  expand_rows_into(s, A, rowid.p);
  const int bits = bits_for(A.n);
  const bool has_val = A.val.p != nullptr;
  const size_t es = has_val ? domain_size(A.domain) : 0;
  const uint32_t* kin = reinterpret_cast<const uint32_t*>(A.col.p);
  Tmp<uint32_t> kout(A.nnz, s);
  if (!has_val) {
    radix_sort_pairs<uint32_t, int32_t>(s, kin, kout.p, rowid.p, T.col.p, A.nnz, 0, bits);
  } else {
    Tmp<int64_t> pin(A.nnz, s), pout(A.nnz, s);
    k_iota64<<<ceil_div(A.nnz, 256), 256, 0, s>>>(pin.p, A.nnz);
    GBX_LAUNCHED();
    radix_sort_pairs<uint32_t, int64_t>(s, kin, kout.p, pin.p, pout.p, A.nnz, 0, bits);
    T.val.alloc(A.nnz * es);
    const int g = ceil_div(A.nnz, 256);
    switch (es) {
      case 1: k_gather_transpose<1><<<g, 256, 0, s>>>(pout.p, rowid.p, A.nnz, T.col.p, A.val.p, T.val.p); break;
      case 4: k_gather_transpose<4><<<g, 256, 0, s>>>(pout.p, rowid.p, A.nnz, T.col.p, A.val.p, T.val.p); break;
      default: k_gather_transpose<8><<<g, 256, 0, s>>>(pout.p, rowid.p, A.nnz, T.col.p, A.val.p, T.val.p); break;
    }
    GBX_LAUNCHED();
  }
  GBX_CUDA(cudaMemsetAsync(T.rp.p, 0, (A.n + 1) * sizeof(int64_t), s));
  k_row_ends32<<<ceil_div(A.nnz, 256), 256, 0, s>>>(kout.p, A.nnz, T.rp.p);
  GBX_LAUNCHED();
  max_scan_rowptr(s, T.rp.p, A.n);
}

// ---- ndiag / equality ----------------------------------------------------------------

__global__ void k_ndiag(const int64_t* rp, const int32_t* col, int64_t n,
                        unsigned long long* cnt) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  int hit = 0;
  if (i < n) {
    int64_t lo = rp[i], hi = rp[i + 1];
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (col[mid] < i) lo = mid + 1; else hi = mid;
    }
    hit = (lo < rp[i + 1] && col[lo] == i) ? 1 : 0;
  }
  unsigned b = __ballot_sync(0xffffffffu, hit);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(cnt, static_cast<unsigned long long>(__popc(b)));
}

int64_t count_ndiag(cudaStream_t s, const Csr& A) {
  if (A.n == 0) return 0;
  Tmp<unsigned long long> c(1, s);
  GBX_CUDA(cudaMemsetAsync(c.p, 0, sizeof(unsigned long long), s));
  k_ndiag<<<ceil_div(A.n, 256), 256, 0, s>>>(A.rp.p, A.col.p, A.n, c.p);
  GBX_LAUNCHED();
  unsigned long long h = 0;
  GBX_CUDA(cudaMemcpyAsync(&h, c.p, sizeof h, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  return static_cast<int64_t>(h);
}

template <typename T>
__global__ void k_neq(const T* a, const T* b, int64_t n, int* flag) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n && a[i] != b[i]) *flag = 1;
}

bool csr_equal(cudaStream_t s, const Csr& X, const Csr& Y) {
  if (X.n != Y.n || X.nnz != Y.nnz) return false;
  Tmp<int> f(1, s);
  GBX_CUDA(cudaMemsetAsync(f.p, 0, sizeof(int), s));
  k_neq<int64_t><<<ceil_div(X.n + 1, 256), 256, 0, s>>>(X.rp.p, Y.rp.p, X.n + 1, f.p);
  if (X.nnz) k_neq<int32_t><<<ceil_div(X.nnz, 256), 256, 0, s>>>(X.col.p, Y.col.p, X.nnz, f.p);
  GBX_LAUNCHED();
  int h = 0;
  GBX_CUDA(cudaMemcpyAsync(&h, f.p, sizeof h, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  return h == 0;
}

// ---- stable sort of ids by a key (util.cpp:35-44) -----------------------------------

__global__ void k_iota(int32_t* p, int64_t n) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) p[i] = static_cast<int32_t>(i);
}
__global__ void k_flip_keys(const int32_t* key, uint32_t* out, int64_t n, bool asc) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = asc ? static_cast<uint32_t>(key[i]) : ~static_cast<uint32_t>(key[i]);
}

void sort_ids_by_key(cudaStream_t s, const int32_t* key, int64_t n, bool ascending,
                     DevArray<int32_t>& perm) {
  perm.alloc(std::max<int64_t>(n, 1));
  if (n == 0) return;
  Tmp<uint32_t> k0(n, s), k1(n, s);
  Tmp<int32_t> v0(n, s);
  k_flip_keys<<<ceil_div(n, 256), 256, 0, s>>>(key, k0.p, n, ascending);
  k_iota<<<ceil_div(n, 256), 256, 0, s>>>(v0.p, n);
  GBX_LAUNCHED();
  radix_sort_pairs<uint32_t, int32_t>(s, k0.p, k1.p, v0.p, perm.p, n, 0, 32);
}

// ---- seeded generators (bit-identical to oracle/oracle.c) -------------------------

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}
__host__ __device__ __forceinline__ uint64_t gen_stream(uint64_t seed, uint64_t stream) {
  return mix64(seed ^ mix64(stream + 0x632BE59BD9B4E019ull));
}
__host__ __device__ __forceinline__ uint64_t gen_draw(uint64_t s, uint64_t i) {
  return mix64(s + (i + 1) * 0x9E3779B97F4A7C15ull);
}
__device__ __forceinline__ uint32_t gen_scramble(uint32_t x, int scale, uint64_t add) {
  uint64_t mask = (scale >= 32) ? 0xFFFFFFFFull : ((1ull << scale) - 1);
  int sh = scale / 2 + 1;
  uint64_t y = x;
  y = (y * 0x9E3779B97F4A7C15ull) & mask;
  y ^= y >> sh;
  y = (y + add) & mask;
  y = (y * 0xBF58476D1CE4E5B9ull) & mask;
  y ^= y >> sh;
  return static_cast<uint32_t>(y);
}


// edges [e0, e0 + m) of the seeded stream; key slot i = e - e0
__global__ void k_rmat(int scale, int64_t m, uint32_t ta, uint32_t tab, uint32_t tabc,
                       uint64_t s, int scramble, uint64_t add, int sym, uint64_t* keys,
                       int64_t e0) {
  const uint64_t kDropKey = uint64_t(1) << (2 * scale);
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= m) return;
  const int64_t e = e0 + i;
  int per = (scale + 1) / 2;
  uint32_t uu = 0, vv = 0;
  uint64_t r = 0;
  for (int l = 0; l < scale; ++l) {
    if ((l & 1) == 0) r = gen_draw(s, static_cast<uint64_t>(e) * per + (l >> 1));
    uint32_t x = (l & 1) ? static_cast<uint32_t>(r >> 32) : static_cast<uint32_t>(r);
    uint32_t ub, vb;
    if (x < ta) { ub = 0; vb = 0; }
    else if (x < tab) { ub = 0; vb = 1; }
    else if (x < tabc) { ub = 1; vb = 0; }
    else { ub = 1; vb = 1; }
    uu = (uu << 1) | ub;
    vv = (vv << 1) | vb;
  }
  if (scramble) {
    uu = gen_scramble(uu, scale, add);
    vv = gen_scramble(vv, scale, add);
  }
  bool loop = uu == vv;
  if (sym) {
    keys[2 * i] = loop ? kDropKey : ((uint64_t(uu) << scale) | vv);
    keys[2 * i + 1] = loop ? kDropKey : ((uint64_t(vv) << scale) | uu);
  } else {
    keys[i] = loop ? kDropKey : ((uint64_t(uu) << scale) | vv);
  }
}

__global__ void k_er(int logn, int64_t m, uint64_t s, uint64_t* keys, int32_t* w) {
  const uint64_t kDropKey = uint64_t(1) << (2 * logn);
  int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (e >= m) return;
  uint64_t r1 = gen_draw(s, 2 * static_cast<uint64_t>(e));
  uint64_t r2 = gen_draw(s, 2 * static_cast<uint64_t>(e) + 1);
  uint32_t u = static_cast<uint32_t>(r1 >> (64 - logn));
  uint32_t v = static_cast<uint32_t>(r2 >> (64 - logn));
  keys[e] = (u == v) ? kDropKey : ((uint64_t(u) << logn) | v);
  if (w) w[e] = 1 + static_cast<int32_t>(((r1 & 0xFFFFFFFFull) * 255ull) >> 32);
}

// keep the first key of every run (and the minimum weight of the run)
__global__ void k_run_heads(const uint64_t* keys, const int32_t* w, int64_t m,
                            uint64_t kDropKey, uint8_t* flag, int32_t* wmin) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= m) return;
  uint64_t k = keys[i];
  bool head = k != kDropKey && (i == 0 || keys[i - 1] != k);
  flag[i] = head ? 1 : 0;
  if (head && w) {
    int32_t best = w[i];
    for (int64_t j = i + 1; j < m && keys[j] == k; ++j) best = min(best, w[j]);
    wmin[i] = best;
  }
}


// sort 64-bit keys in place (double buffer); returns the buffer holding the result
uint64_t* sort_keys(cudaStream_t s, uint64_t* keys, uint64_t* alt, int64_t m, int end_bit) {
  cub::DoubleBuffer<uint64_t> kb(keys, alt);
  radix_sort_keys(s, kb, m, 0, end_bit);
  return kb.Current();
}

void rowptr_from_sorted_keys(cudaStream_t s, int64_t n, int bits, const uint64_t* keys,
                             int64_t nnz, int64_t* rp, int32_t* col) {
  GBX_CUDA(cudaMemsetAsync(rp, 0, (n + 1) * sizeof(int64_t), s));
  if (nnz == 0) return;
  k_row_ends64<<<ceil_div(nnz, 256), 256, 0, s>>>(keys, nnz, bits, col, rp);
  GBX_LAUNCHED();
  max_scan_rowptr(s, rp, n);
}

// row pointers (n+1) from a row-sorted 32-bit row-id array
void rowptr_from_sorted_rows32(cudaStream_t s, int64_t n, const uint32_t* rows, int64_t nnz,
                               int64_t* rp) {
  GBX_CUDA(cudaMemsetAsync(rp, 0, (n + 1) * sizeof(int64_t), s));
  if (nnz == 0) return;
  k_row_ends32<<<ceil_div(nnz, 256), 256, 0, s>>>(rows, nnz, rp);
  GBX_LAUNCHED();
  max_scan_rowptr(s, rp, n);
}

// the first nnz sorted (row<<bits|col) keys -> CSR arrays
void csr_from_sorted_keys(cudaStream_t s, int64_t n, int bits, const uint64_t* keys,
                          int64_t nnz, DevArray<int64_t>& rp, DevArray<int32_t>& col) {
  rp.alloc(n + 1);
  col.alloc(std::max<int64_t>(nnz, 1));
  rowptr_from_sorted_keys(s, n, bits, keys, nnz, rp.p, col.p);
}

// sorted (u<<bits|v) keys (+ weights) -> CSR in g->A
static void keys_to_graph(gbx_graph* g, int64_t n, int bits, uint64_t* keys, int32_t* w,
                          int64_t m, int kind) {
  cudaStream_t s = g->stream;
  // sort
  Tmp<uint64_t> kalt(m, s);
  Tmp<int32_t> walt(w ? m : 0, s);
  cub::DoubleBuffer<uint64_t> kb(keys, kalt.p);
  cub::DoubleBuffer<int32_t> wb(w, walt.p);
  // drop keys (self-loops) are 1 << 2*bits: they sort after every edge
  const int end_bit = 2 * bits + 1;
  const uint64_t drop = uint64_t(1) << (2 * bits);
  if (w) radix_sort_pairs(s, kb, wb, m, 0, end_bit);
  else radix_sort_keys(s, kb, m, 0, end_bit);
  Tmp<uint8_t> flag(m, s);
  Tmp<int32_t> wmin(w ? m : 0, s);
  k_run_heads<<<ceil_div(m, 256), 256, 0, s>>>(kb.Current(), w ? wb.Current() : nullptr, m,
                                                drop, flag.p, wmin.p);
  GBX_LAUNCHED();
  Tmp<uint64_t> uk(m, s);
  Tmp<int64_t> nsel(1, s);
  size_t tb = 0;
  GBX_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, kb.Current(), flag.p, uk.p, nsel.p, m, s));
  int64_t nnz = 0;
  {
    Tmp<uint8_t> t(tb, s);
    GBX_CUDA(cub::DeviceSelect::Flagged(t.p, tb, kb.Current(), flag.p, uk.p, nsel.p, m, s));
    GBX_CUDA(cudaMemcpyAsync(&nnz, nsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaStreamSynchronize(s));
  }
  Csr& A = g->A;
  A.n = n;
  A.nnz = nnz;
  A.domain = w ? GBX_INT32 : GBX_BOOL;
  A.rp.alloc(n + 1);
  A.col.alloc(std::max<int64_t>(nnz, 1));
  rowptr_from_sorted_keys(s, n, bits, uk.p, nnz, A.rp.p, A.col.p);
  if (w) {
    A.val.alloc(std::max<int64_t>(nnz, 1) * sizeof(int32_t));
    tb = 0;
    GBX_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, wmin.p, flag.p,
                                        reinterpret_cast<int32_t*>(A.val.p), nsel.p, m, s));
    Tmp<uint8_t> t(tb, s);
    GBX_CUDA(cub::DeviceSelect::Flagged(t.p, tb, wmin.p, flag.p,
                                        reinterpret_cast<int32_t*>(A.val.p), nsel.p, m, s));
  }
  GBX_CUDA(cudaStreamSynchronize(s));
  g->kind = kind;
}

static void rmat_check(int scale, int ef, double a, double b, double c) {
  if (scale < 1 || scale > 30) fail(GBX_INVALID_VALUE, "rmat: scale must be in [1,30]");
  if (ef < 1) fail(GBX_INVALID_VALUE, "rmat: edge factor must be >= 1");
  if (!(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0))
    fail(GBX_INVALID_VALUE, "rmat: need a,b,c >= 0 and a+b+c <= 1");
}

// keys (u << scale | v) of edges [e0, e1) of the seeded R-MAT stream (both
// directions when sym: 2 keys per edge); self-loops are the drop key 1 << 2*scale
void rmat_keys(cudaStream_t s, int scale, int ef, double a, double b, double c, uint64_t seed,
               int scramble, bool sym, int64_t e0, int64_t e1, uint64_t* keys) {
  rmat_check(scale, ef, a, b, c);
  const int64_t m = e1 - e0;
  if (m <= 0) return;
  uint32_t ta = static_cast<uint32_t>(a * 4294967296.0);
  uint32_t tab = static_cast<uint32_t>((a + b) * 4294967296.0);
  double abc = a + b + c;
  uint32_t tabc = abc >= 1.0 ? 0xFFFFFFFFu : static_cast<uint32_t>(abc * 4294967296.0);
  uint64_t st = gen_stream(seed, 0);
  uint64_t mask = (1ull << scale) - 1;
  uint64_t add = gen_stream(seed, 1) & mask;
  k_rmat<<<ceil_div(m, 256), 256, 0, s>>>(scale, m, ta, tab, tabc, st, scramble, add,
                                           sym ? 1 : 0, keys, e0);
  GBX_LAUNCHED();
}

void generate_rmat(gbx_graph* g, int scale, int ef, double a, double b, double c,
                   uint64_t seed, int scramble, int kind) {
  NvtxRange nvtx_("gbx.generate_rmat");
  rmat_check(scale, ef, a, b, c);
  cudaStream_t s = g->stream;
  int64_t n = int64_t(1) << scale;
  int64_t m = int64_t(ef) << scale;
  bool sym = kind == GBX_UNDIRECTED;
  int64_t mk = sym ? 2 * m : m;
  Tmp<uint64_t> keys(mk, s);
  rmat_keys(s, scale, ef, a, b, c, seed, scramble, sym, 0, m, keys.p);
  keys_to_graph(g, n, scale, keys.p, nullptr, mk, kind);
}

// sorted (row << bits | col) keys, drop keys (1 << 2*bits) last -> CSR over n
// rows with duplicates removed (pattern)
void csr_from_keys_unique(cudaStream_t s, int64_t n, int bits, const uint64_t* sorted, int64_t m,
                          Csr& A) {
  const uint64_t drop = uint64_t(1) << (2 * bits);
  int64_t nnz = 0;
  Tmp<uint64_t> uk(std::max<int64_t>(m, 1), s);
  if (m > 0) {
    Tmp<uint8_t> flag(m, s);
    k_run_heads<<<ceil_div(m, 256), 256, 0, s>>>(sorted, nullptr, m, drop, flag.p, nullptr);
    GBX_LAUNCHED();
    Tmp<int64_t> nsel(1, s);
    size_t tb = 0;
    GBX_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, sorted, flag.p, uk.p, nsel.p, m, s));
    Tmp<uint8_t> t(tb, s);
    GBX_CUDA(cub::DeviceSelect::Flagged(t.p, tb, sorted, flag.p, uk.p, nsel.p, m, s));
    GBX_CUDA(cudaMemcpyAsync(&nnz, nsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaStreamSynchronize(s));
  }
  A.n = n;
  A.nnz = nnz;
  A.domain = GBX_BOOL;
  A.rp.alloc(n + 1);
  A.col.alloc(std::max<int64_t>(nnz, 1));
  A.val.release();
  rowptr_from_sorted_keys(s, n, bits, uk.p, nnz, A.rp.p, A.col.p);
  GBX_CUDA(cudaStreamSynchronize(s));
}

void generate_er(gbx_graph* g, int logn, int degree, uint64_t seed, int weighted) {
  NvtxRange nvtx_("gbx.generate_er");
  if (logn < 1 || logn > 30) fail(GBX_INVALID_VALUE, "er: logn must be in [1,30]");
  if (degree < 1) fail(GBX_INVALID_VALUE, "er: degree must be >= 1");
  cudaStream_t s = g->stream;
  int64_t n = int64_t(1) << logn;
  int64_t m = int64_t(degree) << logn;
  Tmp<uint64_t> keys(m, s);
  Tmp<int32_t> w(weighted ? m : 0, s);
  k_er<<<ceil_div(m, 256), 256, 0, s>>>(logn, m, gen_stream(seed, 2), keys.p,
                                         weighted ? w.p : nullptr);
  GBX_LAUNCHED();
  keys_to_graph(g, n, logn, keys.p, weighted ? w.p : nullptr, m, GBX_DIRECTED);
}

}  // namespace gbx
