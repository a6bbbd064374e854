// io.cu -- graph ingest and export: the reference's gblite::io readers/writers
// (io.hpp, io.cpp) and build_matrix (containers.cpp:128-169), landing the
// matrix directly in HBM as a graph handle.
//
//   * LAGK v1 binary (io.cpp:224-334): the header is checked on the host
//     (BadMagic / UnsupportedVersion / InvalidValue / TruncatedStream exactly
//     as bin_read), then row_ptr and the u64 column stream are copied to the
//     device through two pinned staging buffers (the fread of chunk i+1
//     overlaps the H2D copy and the u64 -> int32 narrowing of chunk i), and
//     the matrix is validated on the device (containers.cpp:104-124; a bad
//     matrix is ParseError, io.cpp:325-331).
//   * Matrix Market coordinate (io.cpp:35-160): the banner, comment and size
//     lines are parsed on the host; the entry lines are tokenised by
//     host threads over newline-aligned slices of the file (line numbers
//     recovered by prefix sums so errors name the same line as the
//     reference); the tuples are then built into CSR on the device.
//   * build_matrix on the device: one stable radix sort of (row<<bits | col)
//     keys carrying the tuple index, run heads, the duplicate policy folded
//     over each run in input order (the reference combines duplicates in
//     input order, containers.cpp:139-158), CSR from the unique keys.
//   * writers (io.cpp:162-222, 261-280): D2H export, then byte-identical
//     output to mm_write / bin_write (same header lines, %.17g reals).
#include <cub/cub.cuh>

#include <algorithm>
#include <cerrno>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "sort.cuh"

namespace gbx {

void rowptr_from_sorted_keys(cudaStream_t s, int64_t n, int bits, const uint64_t* keys,
                             int64_t nnz, int64_t* rp, int32_t* col);

namespace {

// ---- device build (build_matrix, containers.cpp:128-169) --------------------

__global__ void k_coo_keys(const int64_t* rows, const int64_t* cols, int64_t m, int64_t nrows,
                           int64_t ncols, int bits, uint64_t* keys, int64_t* idx,
                           unsigned long long* bad) {
  const int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k >= m) return;
  const int64_t r = rows[k], c = cols[k];
  if (r < 0 || r >= nrows || c < 0 || c >= ncols) {
    atomicMin(bad, static_cast<unsigned long long>(k));  // first offending tuple
    keys[k] = 0;
  } else {
    keys[k] = (static_cast<uint64_t>(r) << bits) | static_cast<uint64_t>(c);
  }
  idx[k] = k;
}

__global__ void k_run_heads(const uint64_t* keys, int64_t m, int32_t* head) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p < m) head[p] = (p == 0 || keys[p] != keys[p - 1]) ? 1 : 0;
}

// unique key + run start per run (seg = inclusive head scan - 1)
__global__ void k_run_compact(const uint64_t* keys, const int32_t* head, const int64_t* seg,
                              int64_t m, uint64_t* ukeys, int64_t* start) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p >= m || !head[p]) return;
  const int64_t u = seg[p] - 1;
  ukeys[u] = keys[p];
  start[u] = p;
}

template <typename T>
__device__ __forceinline__ T dup_fold(int dup, T acc, T v) {
  switch (dup) {
    case GBX_DUP_SECOND: return v;
    case GBX_DUP_MIN: return v < acc ? v : acc;
    case GBX_DUP_MAX: return v > acc ? v : acc;
    case GBX_DUP_PLUS: return acc + v;
    default: return acc;  // FIRST (ERROR never folds)
  }
}

// one thread per run: fold the run's values in input order (stable sort)
template <typename T>
__global__ void k_run_fold(const T* vals, const int64_t* idx, const int64_t* start, int64_t nu,
                           int64_t m, int dup, T* out) {
  const int64_t u = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (u >= nu) return;
  const int64_t b = start[u], e = u + 1 < nu ? start[u + 1] : m;
  T acc = vals[idx[b]];
  for (int64_t p = b + 1; p < e; ++p) acc = dup_fold<T>(dup, acc, vals[idx[p]]);
  out[u] = acc;
}

// bool: plus/max = lor, min = land (ops.cpp monoids on Bool)
__global__ void k_run_fold_bool(const uint8_t* vals, const int64_t* idx, const int64_t* start,
                                int64_t nu, int64_t m, int dup, uint8_t* out) {
  const int64_t u = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (u >= nu) return;
  const int64_t b = start[u], e = u + 1 < nu ? start[u + 1] : m;
  uint8_t acc = vals[idx[b]] != 0;
  for (int64_t p = b + 1; p < e; ++p) {
    const uint8_t v = vals[idx[p]] != 0;
    switch (dup) {
      case GBX_DUP_SECOND: acc = v; break;
      case GBX_DUP_MIN: acc = acc & v; break;
      case GBX_DUP_MAX:
      case GBX_DUP_PLUS: acc = acc | v; break;
      default: break;
    }
  }
  out[u] = acc;
}

__global__ void k_narrow_cols(const uint64_t* c64, int32_t* c32, int64_t m, uint64_t ncols,
                              int* bad) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p >= m) return;
  const uint64_t c = c64[p];
  if (c >= ncols) { atomicOr(bad, 2); c32[p] = 0; return; }
  c32[p] = static_cast<int32_t>(c);
}

__global__ void k_bool_normalise(uint8_t* v, int64_t m) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p < m) v[p] = v[p] != 0;
}

__global__ void k_validate_rp(const int64_t* rp, int64_t n, int64_t nnz, int* bad) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i > n) return;
  if (i == 0 && rp[0] != 0) atomicOr(bad, 1);
  if (i == n && rp[n] != nnz) atomicOr(bad, 1);
  if (i < n && rp[i] > rp[i + 1]) atomicOr(bad, 1);
}

__global__ void k_validate_sorted(const int64_t* rp, const int32_t* col, int64_t n, int* bad) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  for (int64_t p = rp[i] + 1; p < rp[i + 1]; ++p)
    if (col[p - 1] >= col[p]) { atomicOr(bad, 4); return; }
}

// ---- host helpers -------------------------------------------------------------

const char* domain_name(int d) {
  switch (d) {
    case GBX_BOOL: return "bool";
    case GBX_INT64: return "int64";
    case GBX_UINT64: return "uint64";
    case GBX_FP64: return "fp64";
  }
  return "?";
}

struct File {
  FILE* f = nullptr;
  File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
  ~File() { if (f) std::fclose(f); }
};

struct Pinned {
  void* p = nullptr;
  explicit Pinned(size_t n) {
    if (n && cudaMallocHost(&p, n) != cudaSuccess) {
      (void)cudaGetLastError();
      fail(GBX_OUT_OF_MEMORY, "pinned staging allocation failed");
    }
  }
  ~Pinned() { if (p) cudaFreeHost(p); }
};

void check_square(int64_t nrows, int64_t ncols) {
  if (nrows != ncols) fail(GBX_INVALID_MATRIX, "graph_new: adjacency matrix must be square");
}

void check_n(int64_t n) {
  if (n >= (int64_t(1) << 31) - 1)
    fail(GBX_UNSUPPORTED, "graph: n >= 2^31 is not supported by the int32 column layout");
}

}  // namespace

// tuples (device or host arrays) -> g->A.  Mirrors build_matrix's checks:
// IndexOutOfBounds (first offending tuple), then the duplicate policy.
void build_from_coo(gbx_graph* g, int64_t nrows, int64_t ncols, int64_t m, const int64_t* rows,
                    const int64_t* cols, const void* vals, int domain, int dup, int kind,
                    bool host_ptrs) {
  if (nrows < 0 || ncols < 0 || m < 0) fail(GBX_INVALID_VALUE, "build: negative size");
  if (kind != GBX_DIRECTED && kind != GBX_UNDIRECTED) fail(GBX_INVALID_VALUE, "build: unknown kind");
  if (dup < GBX_DUP_ERROR || dup > GBX_DUP_PLUS) fail(GBX_INVALID_VALUE, "build: unknown dup policy");
  if (m > 0 && (!rows || !cols)) fail(GBX_NULL_ARGUMENT, "build: tuple arrays are NULL");
  if (vals && domain != GBX_BOOL && domain != GBX_INT64 && domain != GBX_UINT64 && domain != GBX_FP64)
    fail(GBX_DOMAIN_MISMATCH, "build: unknown value domain " + std::to_string(domain));
  const int64_t nd = std::max(nrows, ncols);
  check_n(nd);
  cudaStream_t s = g->stream;
  const int bits = bits_for(std::max<int64_t>(nd, 2));
  const size_t es = vals ? domain_size(domain) : 0;
  Csr& A = g->A;
  A = Csr();
  A.n = nrows;
  A.domain = vals ? domain : GBX_BOOL;
  if (m == 0) {
    check_square(nrows, ncols);
    A.rp.alloc(nrows + 1);
    A.col.alloc(1);
    GBX_CUDA(cudaMemsetAsync(A.rp.p, 0, (nrows + 1) * 8, s));
    GBX_CUDA(cudaStreamSynchronize(s));
    g->kind = kind;
    return;
  }
  Tmp<int64_t> drow(host_ptrs ? m : 0, s), dcol(host_ptrs ? m : 0, s);
  Tmp<uint8_t> dval(host_ptrs && vals ? m * es : 0, s);
  const int64_t* R = rows;
  const int64_t* Cc = cols;
  const uint8_t* V = static_cast<const uint8_t*>(vals);
  if (host_ptrs) {
    GBX_CUDA(cudaMemcpyAsync(drow.p, rows, m * 8, cudaMemcpyHostToDevice, s));
    GBX_CUDA(cudaMemcpyAsync(dcol.p, cols, m * 8, cudaMemcpyHostToDevice, s));
    if (vals) GBX_CUDA(cudaMemcpyAsync(dval.p, vals, m * es, cudaMemcpyHostToDevice, s));
    R = drow.p;
    Cc = dcol.p;
    V = dval.p;
  }
  Tmp<uint64_t> k0(m, s), k1(m, s);
  Tmp<int64_t> i0(m, s), i1(m, s);
  Tmp<unsigned long long> bad(1, s);
  GBX_CUDA(cudaMemsetAsync(bad.p, 0xff, 8, s));
  k_coo_keys<<<ceil_div(m, 256), 256, 0, s>>>(R, Cc, m, nrows, ncols, bits, k0.p, i0.p, bad.p);
  GBX_LAUNCHED();
  unsigned long long hbad = 0;
  GBX_CUDA(cudaMemcpyAsync(&hbad, bad.p, 8, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  if (hbad != ~0ull) fail(GBX_INDEX_OUT_OF_BOUNDS, "build_matrix tuple " + std::to_string(hbad));
  // stable sort of the keys carrying the tuple index
  cub::DoubleBuffer<uint64_t> kb(k0.p, k1.p);
  cub::DoubleBuffer<int64_t> ib(i0.p, i1.p);
  radix_sort_pairs(s, kb, ib, m, 0, 2 * bits);
  const uint64_t* keys = kb.Current();
  const int64_t* idx = ib.Current();
  Tmp<int32_t> head(m, s);
  Tmp<int64_t> seg(m, s);
  k_run_heads<<<ceil_div(m, 256), 256, 0, s>>>(keys, m, head.p);
  GBX_LAUNCHED();
  size_t tb = 0;
  GBX_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, head.p, seg.p, m, s));
  {
    Tmp<uint8_t> t(tb, s);
    GBX_CUDA(cub::DeviceScan::InclusiveSum(t.p, tb, head.p, seg.p, m, s));
  }
  int64_t nu = 0;
  GBX_CUDA(cudaMemcpyAsync(&nu, seg.p + m - 1, 8, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  if (dup == GBX_DUP_ERROR && nu != m)
    fail(GBX_DUPLICATE_ENTRY, "duplicate coordinates in the tuple list");
  Tmp<uint64_t> uk(nu, s);
  Tmp<int64_t> st(nu, s);
  k_run_compact<<<ceil_div(m, 256), 256, 0, s>>>(keys, head.p, seg.p, m, uk.p, st.p);
  GBX_LAUNCHED();
  if (vals) {
    A.val.alloc(nu * es);
    const int fdup = dup == GBX_DUP_ERROR ? GBX_DUP_FIRST : dup;
    switch (domain) {
      case GBX_BOOL:
        k_run_fold_bool<<<ceil_div(nu, 256), 256, 0, s>>>(V, idx, st.p, nu, m, fdup, A.val.p);
        break;
      case GBX_INT64:
        k_run_fold<long long><<<ceil_div(nu, 256), 256, 0, s>>>(
            reinterpret_cast<const long long*>(V), idx, st.p, nu, m, fdup,
            reinterpret_cast<long long*>(A.val.p));
        break;
      case GBX_UINT64:
        k_run_fold<unsigned long long><<<ceil_div(nu, 256), 256, 0, s>>>(
            reinterpret_cast<const unsigned long long*>(V), idx, st.p, nu, m, fdup,
            reinterpret_cast<unsigned long long*>(A.val.p));
        break;
      case GBX_FP64:
        k_run_fold<double><<<ceil_div(nu, 256), 256, 0, s>>>(
            reinterpret_cast<const double*>(V), idx, st.p, nu, m, fdup,
            reinterpret_cast<double*>(A.val.p));
        break;
    }
    GBX_LAUNCHED();
  }
  check_square(nrows, ncols);
  A.nnz = nu;
  A.rp.alloc(nrows + 1);
  A.col.alloc(std::max<int64_t>(nu, 1));
  rowptr_from_sorted_keys(s, nrows, bits, uk.p, nu, A.rp.p, A.col.p);
  GBX_CUDA(cudaStreamSynchronize(s));
  g->kind = kind;
}

// ---- LAGK v1 (io.cpp:224-334) -------------------------------------------------

namespace {

constexpr char kMagic[4] = {'L', 'A', 'G', 'K'};
constexpr uint32_t kVersion = 1;
constexpr size_t kStage = size_t(64) << 20;  // bytes per pinned staging buffer

struct Reader {  // a byte source: a FILE or a memory buffer
  FILE* f = nullptr;
  const uint8_t* buf = nullptr;
  size_t len = 0, pos = 0;
  size_t read(void* dst, size_t n) {
    if (f) return std::fread(dst, 1, n, f);
    const size_t k = std::min(n, len - pos);
    std::memcpy(dst, buf + pos, k);
    pos += k;
    return k;
  }
  void get(void* dst, size_t n) {
    if (read(dst, n) != n) fail(GBX_TRUNCATED_STREAM, "binary stream ended early");
  }
  uint64_t u64() { uint64_t v; get(&v, 8); return v; }
  uint32_t u32() { uint32_t v; get(&v, 4); return v; }
};

// stream `bytes` from the reader to device memory through two pinned buffers;
// each landed chunk is handed to on_chunk(device ptr, offset, size) on stream s
template <typename F>
void stream_to_device(Reader& rd, size_t bytes, uint8_t* dst_dev, cudaStream_t s, F&& on_chunk) {
  if (bytes == 0) return;
  Pinned st(2 * std::min(bytes, kStage));
  uint8_t* stage[2] = {static_cast<uint8_t*>(st.p),
                       static_cast<uint8_t*>(st.p) + std::min(bytes, kStage)};
  cudaEvent_t done[2];
  GBX_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
  GBX_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
  struct Ev {
    cudaEvent_t* e;
    ~Ev() { cudaEventDestroy(e[0]); cudaEventDestroy(e[1]); }
  } guard{done};
  bool used[2] = {false, false};
  size_t off = 0;
  int b = 0;
  while (off < bytes) {
    const size_t k = std::min(kStage, bytes - off);
    if (used[b]) GBX_CUDA(cudaEventSynchronize(done[b]));  // the buffer's last copy has landed
    if (rd.read(stage[b], k) != k) {
      GBX_CUDA(cudaStreamSynchronize(s));
      fail(GBX_TRUNCATED_STREAM, "binary stream ended early");
    }
    GBX_CUDA(cudaMemcpyAsync(dst_dev + off, stage[b], k, cudaMemcpyHostToDevice, s));
    GBX_CUDA(cudaEventRecord(done[b], s));
    used[b] = true;
    on_chunk(dst_dev + off, off, k);
    off += k;
    b ^= 1;
  }
  GBX_CUDA(cudaStreamSynchronize(s));
}

void read_lagk(gbx_graph* g, Reader& rd, int kind) {
  char magic[4];
  rd.get(magic, 4);
  if (std::memcmp(magic, kMagic, 4) != 0) fail(GBX_BAD_MAGIC, "not a gblite binary matrix");
  const uint32_t version = rd.u32();
  if (version != kVersion)
    fail(GBX_UNSUPPORTED_VERSION, "binary format version " + std::to_string(version));
  uint8_t tag;
  rd.get(&tag, 1);
  if (tag > 3) fail(GBX_INVALID_VALUE, "bad domain tag in binary stream");
  const uint64_t nrows = rd.u64(), ncols = rd.u64(), nvals = rd.u64();
  if (kind != GBX_DIRECTED && kind != GBX_UNDIRECTED) fail(GBX_INVALID_VALUE, "read: unknown kind");
  // a stream announcing more than it can hold is truncated before any allocation
  if (!rd.f) {
    const unsigned __int128 need = (unsigned __int128)(nrows + 1) * 8 + (unsigned __int128)nvals * 8 +
                                   (unsigned __int128)nvals * (tag == 0 ? 1 : 8);
    if (nrows == UINT64_MAX || need > rd.len - rd.pos)
      fail(GBX_TRUNCATED_STREAM, "binary stream ended early");
  } else {
    const long here = std::ftell(rd.f);
    if (here >= 0 && std::fseek(rd.f, 0, SEEK_END) == 0) {
      const long end = std::ftell(rd.f);
      std::fseek(rd.f, here, SEEK_SET);
      const unsigned __int128 need = (unsigned __int128)(nrows + 1) * 8 +
                                     (unsigned __int128)nvals * (8 + (tag == 0 ? 1 : 8));
      if (nrows == UINT64_MAX || need > static_cast<unsigned __int128>(end - here))
        fail(GBX_TRUNCATED_STREAM, "binary stream ended early");
    }
  }
  check_n(static_cast<int64_t>(std::max(nrows, ncols)));
  cudaStream_t s = g->stream;
  const int64_t n = static_cast<int64_t>(nrows), m = static_cast<int64_t>(nvals);
  Csr& A = g->A;
  A = Csr();
  A.n = n;
  A.nnz = m;
  A.domain = static_cast<int>(tag);
  A.rp.alloc(n + 1);
  A.col.alloc(std::max<int64_t>(m, 1));
  Tmp<int> bad(1, s);
  GBX_CUDA(cudaMemsetAsync(bad.p, 0, 4, s));
  stream_to_device(rd, (n + 1) * 8, reinterpret_cast<uint8_t*>(A.rp.p), s,
                   [](uint8_t*, size_t, size_t) {});
  // u64 columns: staged in 64 MB chunks, narrowed to int32 on the device
  if (m > 0) {
    Tmp<uint8_t> c64(std::min<size_t>(m * 8, 2 * kStage), s);
    // reuse a two-slot device ring: chunk i lands in slot i&1
    Pinned st(2 * std::min<size_t>(m * 8, kStage));
    uint8_t* stage[2] = {static_cast<uint8_t*>(st.p),
                         static_cast<uint8_t*>(st.p) + std::min<size_t>(m * 8, kStage)};
    cudaEvent_t done[2];
    GBX_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
    GBX_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
    struct Ev {
      cudaEvent_t* e;
      ~Ev() { cudaEventDestroy(e[0]); cudaEventDestroy(e[1]); }
    } guard{done};
    bool used[2] = {false, false};
    const size_t bytes = static_cast<size_t>(m) * 8;
    size_t off = 0;
    int b = 0;
    while (off < bytes) {
      const size_t k = std::min(kStage, bytes - off);
      if (used[b]) GBX_CUDA(cudaEventSynchronize(done[b]));
      if (rd.read(stage[b], k) != k) {
        GBX_CUDA(cudaStreamSynchronize(s));
        fail(GBX_TRUNCATED_STREAM, "binary stream ended early");
      }
      uint8_t* slot = c64.p + (b ? std::min<size_t>(bytes, kStage) : 0);
      GBX_CUDA(cudaMemcpyAsync(slot, stage[b], k, cudaMemcpyHostToDevice, s));
      const int64_t cnt = static_cast<int64_t>(k / 8);
      k_narrow_cols<<<ceil_div(cnt, 256), 256, 0, s>>>(reinterpret_cast<const uint64_t*>(slot),
                                                        A.col.p + off / 8, cnt, ncols, bad.p);
      GBX_LAUNCHED();
      GBX_CUDA(cudaEventRecord(done[b], s));
      used[b] = true;
      off += k;
      b ^= 1;
    }
    GBX_CUDA(cudaStreamSynchronize(s));
    const size_t es = tag == 0 ? 1 : 8;
    A.val.alloc(m * es);
    stream_to_device(rd, m * es, A.val.p, s, [](uint8_t*, size_t, size_t) {});
    if (tag == 0) {
      k_bool_normalise<<<ceil_div(m, 256), 256, 0, s>>>(A.val.p, m);
      GBX_LAUNCHED();
    }
  }
  // validate (containers.cpp:104-124): a bad matrix is ParseError (io.cpp:325-331)
  k_validate_rp<<<ceil_div(n + 1, 256), 256, 0, s>>>(A.rp.p, n, m, bad.p);
  GBX_LAUNCHED();
  int hb = 0;
  GBX_CUDA(cudaMemcpyAsync(&hb, bad.p, 4, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  if (!(hb & 1) && n > 0 && m > 0) {
    k_validate_sorted<<<ceil_div(n, 256), 256, 0, s>>>(A.rp.p, A.col.p, n, bad.p);
    GBX_LAUNCHED();
    GBX_CUDA(cudaMemcpyAsync(&hb, bad.p, 4, cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaStreamSynchronize(s));
  }
  if (hb & 1) fail(GBX_PARSE_ERROR, "binary stream holds an invalid matrix: bad row_ptr");
  if (hb & 2) fail(GBX_PARSE_ERROR, "binary stream holds an invalid matrix: column out of range");
  if (hb & 4) fail(GBX_PARSE_ERROR, "binary stream holds an invalid matrix: columns not sorted");
  check_square(n, static_cast<int64_t>(ncols));
  g->kind = kind;
}

// ---- Matrix Market (io.cpp:35-160) --------------------------------------------

[[noreturn]] void parse_fail(size_t line_no, const std::string& why) {
  fail(GBX_PARSE_ERROR, "line " + std::to_string(line_no) + ": " + why);
}

struct Text {
  const char* p;
  const char* end;
  // next line [b, e) without the newline; false at end of input
  bool line(const char*& b, const char*& e) {
    if (p >= end) return false;
    b = p;
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', end - p));
    e = nl ? nl : end;
    p = nl ? nl + 1 : end;
    return true;
  }
};

std::vector<std::string> words(const char* b, const char* e, size_t maxw) {
  std::vector<std::string> w;
  const char* q = b;
  while (q < e && w.size() < maxw) {
    while (q < e && std::isspace(static_cast<unsigned char>(*q))) ++q;
    const char* t = q;
    while (q < e && !std::isspace(static_cast<unsigned char>(*q))) ++q;
    if (q > t) w.emplace_back(t, q);
  }
  return w;
}

inline const char* skip_ws(const char* q, const char* e) {
  while (q < e && (*q == ' ' || *q == '\t' || *q == '\r' || *q == '\v' || *q == '\f')) ++q;
  return q;
}

// istream >> uint64: optional '+' / '-' (negated modulo 2^64), digits
inline bool parse_u64(const char*& q, const char* e, uint64_t& v) {
  q = skip_ws(q, e);
  bool neg = false;
  if (q < e && (*q == '+' || *q == '-')) { neg = *q == '-'; ++q; }
  if (q >= e || *q < '0' || *q > '9') return false;
  unsigned __int128 acc = 0;
  while (q < e && *q >= '0' && *q <= '9') {
    acc = acc * 10 + (*q - '0');
    if (acc > UINT64_MAX) return false;  // istream sets failbit on overflow
    ++q;
  }
  v = static_cast<uint64_t>(acc);
  if (neg) v = 0 - v;
  return true;
}

inline bool parse_i64(const char*& q, const char* e, int64_t& v) {
  q = skip_ws(q, e);
  bool neg = false;
  if (q < e && (*q == '+' || *q == '-')) { neg = *q == '-'; ++q; }
  if (q >= e || *q < '0' || *q > '9') return false;
  unsigned __int128 acc = 0;
  while (q < e && *q >= '0' && *q <= '9') {
    acc = acc * 10 + (*q - '0');
    if (acc > (unsigned __int128)INT64_MAX + 1) return false;
    ++q;
  }
  if (!neg && acc > INT64_MAX) return false;
  v = neg ? static_cast<int64_t>(0 - static_cast<uint64_t>(acc)) : static_cast<int64_t>(acc);
  return true;
}

inline bool parse_f64(const char*& q, const char* e, double& v) {
  q = skip_ws(q, e);
  if (q >= e) return false;
  char buf[128];
  size_t k = 0;
  while (q + k < e && k < sizeof buf - 1 && !std::isspace(static_cast<unsigned char>(q[k]))) {
    buf[k] = q[k];
    ++k;
  }
  buf[k] = '\0';
  char* stop = nullptr;
  errno = 0;
  v = std::strtod(buf, &stop);
  if (stop == buf) return false;
  q += stop - buf;
  return true;
}

struct MmError {
  int code = 0;
  size_t line = 0;  // 1-based line number within the file
  std::string why;
};

struct MmSlice {
  std::vector<int64_t> r, c;
  std::vector<uint8_t> v;  // values, es bytes each
  size_t lines = 0;
  MmError err;  // first error in the slice (line index relative to the slice)
  size_t err_idx = 0;
};

void read_mm(gbx_graph* g, const char* data, size_t len, int kind) {
  if (kind != GBX_DIRECTED && kind != GBX_UNDIRECTED) fail(GBX_INVALID_VALUE, "read: unknown kind");
  Text t{data, data + len};
  const char *b, *e;
  size_t line_no = 0;
  if (!t.line(b, e)) parse_fail(1, "empty stream");
  ++line_no;
  const auto ban = words(b, e, 5);
  auto w = [&](size_t i) { return i < ban.size() ? ban[i] : std::string(); };
  if (w(0) != "%%MatrixMarket") parse_fail(line_no, "missing MatrixMarket banner");
  if (w(1) != "matrix") parse_fail(line_no, "unsupported object '" + w(1) + "'");
  if (w(2) != "coordinate") parse_fail(line_no, "unsupported format '" + w(2) + "'");
  int domain;
  bool pattern = false;
  if (w(3) == "pattern") { domain = GBX_BOOL; pattern = true; }
  else if (w(3) == "integer") domain = GBX_INT64;
  else if (w(3) == "real") domain = GBX_FP64;
  else parse_fail(line_no, "unsupported field '" + w(3) + "'");
  bool symmetric = false;
  if (w(4) == "symmetric") symmetric = true;
  else if (w(4) != "general") parse_fail(line_no, "unsupported symmetry '" + w(4) + "'");
  // comments; "%%domain <name>" overrides the value domain
  int override_domain = -1;
  bool have_size = false;
  while (t.line(b, e)) {
    ++line_no;
    if (b == e) continue;
    if (*b != '%') { have_size = true; break; }
    const auto c = words(b, e, 2);
    if (!c.empty() && c[0] == "%%domain") {
      const std::string nm = c.size() > 1 ? c[1] : std::string();
      if (nm == "bool") override_domain = GBX_BOOL;
      else if (nm == "int64") override_domain = GBX_INT64;
      else if (nm == "uint64") override_domain = GBX_UINT64;
      else if (nm == "fp64") override_domain = GBX_FP64;
      else parse_fail(line_no, "unknown domain '" + nm + "'");
    }
  }
  if (override_domain >= 0 && !pattern) domain = override_domain;
  uint64_t nrows = 0, ncols = 0, nnz = 0;
  {
    if (!have_size) { b = e = t.end; }
    const char* q = b;
    if (!(parse_u64(q, e, nrows) && parse_u64(q, e, ncols) && parse_u64(q, e, nnz)))
      parse_fail(line_no, "bad size line");
  }
  // entry lines: slices of the remaining text at newline boundaries, one per thread
  const char* body = t.p;
  const char* bend = t.end;
  const size_t blen = bend - body;
  unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (blen < (size_t(1) << 20)) nt = 1;
  std::vector<const char*> cut(nt + 1);
  cut[0] = body;
  cut[nt] = bend;
  for (unsigned i = 1; i < nt; ++i) {
    const char* q = body + blen * i / nt;
    if (q < cut[i - 1]) q = cut[i - 1];
    const char* nl = static_cast<const char*>(std::memchr(q, '\n', bend - q));
    cut[i] = nl ? nl + 1 : bend;
  }
  const size_t es = pattern ? 0 : domain_size(domain);
  std::vector<MmSlice> sl(nt);
  auto work = [&](unsigned i) {
    MmSlice& S = sl[i];
    Text tt{cut[i], cut[i + 1]};
    const char *lb, *le;
    while (tt.line(lb, le)) {
      const size_t li = S.lines++;
      if (S.err.code) continue;  // keep counting lines after the first error
      const char* q = lb;
      uint64_t i1 = 0, j1 = 0;
      if (!(parse_u64(q, le, i1) && parse_u64(q, le, j1))) {
        S.err = {GBX_PARSE_ERROR, 0, "bad entry indices"};
        S.err_idx = li;
        continue;
      }
      if (i1 == 0 || j1 == 0 || i1 > nrows || j1 > ncols) {
        S.err = {GBX_INDEX_OUT_OF_BOUNDS, 0,
                 "entry (" + std::to_string(i1) + ", " + std::to_string(j1) + ") outside " +
                     std::to_string(nrows) + " x " + std::to_string(ncols)};
        S.err_idx = li;
        continue;
      }
      uint8_t vb[8] = {0};
      if (!pattern) {
        bool ok = true;
        switch (domain) {
          case GBX_BOOL: {
            int64_t raw = 0;
            ok = parse_i64(q, le, raw);
            vb[0] = raw != 0;
            break;
          }
          case GBX_INT64: {
            int64_t raw = 0;
            ok = parse_i64(q, le, raw);
            std::memcpy(vb, &raw, 8);
            break;
          }
          case GBX_UINT64: {
            int64_t raw = 0;
            ok = parse_i64(q, le, raw);
            if (ok && raw < 0) {
              S.err = {GBX_PARSE_ERROR, 0, "negative value in a uint64 matrix"};
              S.err_idx = li;
              continue;
            }
            std::memcpy(vb, &raw, 8);
            break;
          }
          case GBX_FP64: {
            double raw = 0.0;
            ok = parse_f64(q, le, raw);
            std::memcpy(vb, &raw, 8);
            break;
          }
        }
        if (!ok) {
          S.err = {GBX_PARSE_ERROR, 0, "missing value"};
          S.err_idx = li;
          continue;
        }
      }
      S.r.push_back(static_cast<int64_t>(i1 - 1));
      S.c.push_back(static_cast<int64_t>(j1 - 1));
      S.v.insert(S.v.end(), vb, vb + es);
      if (symmetric && i1 != j1) {
        S.r.push_back(static_cast<int64_t>(j1 - 1));
        S.c.push_back(static_cast<int64_t>(i1 - 1));
        S.v.insert(S.v.end(), vb, vb + es);
      }
    }
  };
  {
    std::vector<std::thread> th;
    for (unsigned i = 1; i < nt; ++i) th.emplace_back(work, i);
    work(0);
    for (auto& x : th) x.join();
  }
  // only the first nnz entry lines count (the reader stops there); report
  // the first error among them, or a short file
  size_t before = 0;
  size_t tuples = 0;
  std::vector<size_t> keep_tuples(nt, 0);
  for (unsigned i = 0; i < nt; ++i) {
    MmSlice& S = sl[i];
    const size_t want = nnz > before ? std::min<size_t>(S.lines, nnz - before) : 0;
    if (S.err.code && S.err_idx < want) {
      const size_t ln = line_no + before + S.err_idx + 1;
      if (S.err.code == GBX_INDEX_OUT_OF_BOUNDS)
        fail(GBX_INDEX_OUT_OF_BOUNDS, "line " + std::to_string(ln) + ": " + S.err.why);
      parse_fail(ln, S.err.why);
    }
    if (want < S.lines) {
      // trailing lines beyond the announced count: drop their tuples (the
      // slice's tuples are in line order; count those of the kept lines)
      Text tt{cut[i], cut[i + 1]};
      const char *lb, *le;
      size_t kept = 0;
      for (size_t li = 0; li < want && tt.line(lb, le); ++li) {
        const char* q = lb;
        uint64_t i1 = 0, j1 = 0;
        parse_u64(q, le, i1);
        parse_u64(q, le, j1);
        kept += (symmetric && i1 != j1) ? 2 : 1;
      }
      keep_tuples[i] = kept;
    } else {
      keep_tuples[i] = S.r.size();
    }
    tuples += keep_tuples[i];
    before += S.lines;
  }
  if (before < nnz) parse_fail(line_no + before + 1, "unexpected end of entries");
  std::vector<int64_t> R, C;
  std::vector<uint8_t> V;
  R.reserve(tuples);
  C.reserve(tuples);
  V.reserve(tuples * es);
  for (unsigned i = 0; i < nt; ++i) {
    const size_t k = keep_tuples[i];
    R.insert(R.end(), sl[i].r.begin(), sl[i].r.begin() + k);
    C.insert(C.end(), sl[i].c.begin(), sl[i].c.begin() + k);
    V.insert(V.end(), sl[i].v.begin(), sl[i].v.begin() + k * es);
    sl[i] = MmSlice();
  }
  check_n(static_cast<int64_t>(std::max(nrows, ncols)));
  static const uint64_t no_values = 0;  // a valued domain with zero entries keeps its domain
  const void* vp = pattern ? nullptr : (V.empty() ? static_cast<const void*>(&no_values) : V.data());
  build_from_coo(g, static_cast<int64_t>(nrows), static_cast<int64_t>(ncols),
                 static_cast<int64_t>(R.size()), R.data(), C.data(), vp, domain, GBX_DUP_ERROR,
                 kind, true);
  if (pattern) g->A.domain = GBX_BOOL;
}

std::vector<char> slurp(const char* path) {
  File f(path, "rb");
  if (!f.f) fail(GBX_IO_FAILURE, std::string("cannot open ") + path);
  std::vector<char> d;
  if (std::fseek(f.f, 0, SEEK_END) == 0) {
    const long n = std::ftell(f.f);
    if (n > 0) d.reserve(static_cast<size_t>(n));
    std::fseek(f.f, 0, SEEK_SET);
  }
  char buf[1 << 16];
  size_t k;
  while ((k = std::fread(buf, 1, sizeof buf, f.f)) > 0) d.insert(d.end(), buf, buf + k);
  return d;
}

// ---- writers (io.cpp:162-222, 261-280) -----------------------------------------

struct HostCsr {
  int64_t n = 0, nnz = 0;
  int domain = GBX_BOOL;
  bool has_vals = false;
  std::vector<int64_t> rp;
  std::vector<int32_t> col;
  std::vector<uint8_t> val;
  size_t es() const { return has_vals ? domain_size(domain) : 0; }
  bool truthy(int64_t p) const { return !has_vals || val[p] != 0; }
};

HostCsr export_host(gbx_graph* g) {
  HostCsr h;
  h.n = g->A.n;
  h.nnz = g->A.nnz;
  h.domain = g->A.domain;
  h.has_vals = g->A.val.p != nullptr && h.nnz > 0;
  h.rp.resize(h.n + 1);
  h.col.resize(h.nnz);
  cudaStream_t s = g->stream;
  GBX_CUDA(cudaMemcpyAsync(h.rp.data(), g->A.rp.p, (h.n + 1) * 8, cudaMemcpyDeviceToHost, s));
  if (h.nnz) GBX_CUDA(cudaMemcpyAsync(h.col.data(), g->A.col.p, h.nnz * 4, cudaMemcpyDeviceToHost, s));
  if (h.has_vals) {
    h.val.resize(h.nnz * h.es());
    GBX_CUDA(cudaMemcpyAsync(h.val.data(), g->A.val.p, h.val.size(), cudaMemcpyDeviceToHost, s));
  }
  GBX_CUDA(cudaStreamSynchronize(s));
  return h;
}

struct Out {
  FILE* f;
  void put(const void* p, size_t n) {
    if (n && std::fwrite(p, 1, n, f) != n) fail(GBX_IO_FAILURE, "stream write failed");
  }
};

void write_lagk(const HostCsr& h, Out& o) {
  o.put(kMagic, 4);
  o.put(&kVersion, 4);
  const uint8_t tag = static_cast<uint8_t>(h.domain);
  if (h.domain < 0 || h.domain > 3) fail(GBX_DOMAIN_MISMATCH, "LAGK holds bool/int64/uint64/fp64 only");
  o.put(&tag, 1);
  const uint64_t nr = h.n, nc = h.n, nv = h.nnz;
  o.put(&nr, 8);
  o.put(&nc, 8);
  o.put(&nv, 8);
  o.put(h.rp.data(), (h.n + 1) * 8);
  std::vector<uint64_t> buf;
  const int64_t kB = 1 << 20;
  for (int64_t p0 = 0; p0 < h.nnz; p0 += kB) {
    const int64_t p1 = std::min(h.nnz, p0 + kB);
    buf.assign(h.col.begin() + p0, h.col.begin() + p1);
    o.put(buf.data(), (p1 - p0) * 8);
  }
  if (h.domain == GBX_BOOL) {
    std::vector<uint8_t> b(h.nnz);
    for (int64_t p = 0; p < h.nnz; ++p) b[p] = h.truthy(p) ? 1 : 0;
    o.put(b.data(), b.size());
  } else if (h.nnz) {
    if (!h.has_vals) fail(GBX_INVALID_VALUE, "valued domain without values");
    o.put(h.val.data(), h.val.size());
  }
}

void format_value(const HostCsr& h, int64_t p, std::string& out) {
  char buf[64];
  switch (h.domain) {
    case GBX_BOOL: out += h.truthy(p) ? "1" : "0"; return;
    case GBX_INT64: {
      long long v;
      std::memcpy(&v, &h.val[p * 8], 8);
      std::snprintf(buf, sizeof buf, "%lld", v);
      break;
    }
    case GBX_UINT64: {
      unsigned long long v;
      std::memcpy(&v, &h.val[p * 8], 8);
      std::snprintf(buf, sizeof buf, "%llu", v);
      break;
    }
    case GBX_FP64: {
      double v;
      std::memcpy(&v, &h.val[p * 8], 8);
      std::snprintf(buf, sizeof buf, "%.17g", v);
      break;
    }
    default: fail(GBX_DOMAIN_MISMATCH, "Matrix Market holds bool/int64/uint64/fp64 only");
  }
  out += buf;
}

bool value_eq(const HostCsr& h, int64_t p, int64_t q) {
  if (!h.has_vals) return true;
  if (h.domain == GBX_BOOL) return h.truthy(p) == h.truthy(q);
  if (h.domain == GBX_FP64) {
    double a, b;
    std::memcpy(&a, &h.val[p * 8], 8);
    std::memcpy(&b, &h.val[q * 8], 8);
    return a == b;
  }
  return std::memcmp(&h.val[p * 8], &h.val[q * 8], 8) == 0;
}

void write_mm(const HostCsr& h, Out& o, bool symmetric) {
  if (h.domain < 0 || h.domain > 3) fail(GBX_DOMAIN_MISMATCH, "Matrix Market holds bool/int64/uint64/fp64 only");
  bool pattern = false;
  const char* field = "real";
  if (h.domain == GBX_BOOL) {
    bool all_true = true;
    for (int64_t p = 0; p < h.nnz && all_true; ++p) all_true = h.truthy(p);
    pattern = all_true;
    field = all_true ? "pattern" : "integer";
  } else if (h.domain == GBX_INT64 || h.domain == GBX_UINT64) {
    field = "integer";
  }
  if (symmetric) {
    // every stored (i, j) needs its mirror with an equal value (io.cpp:190-203)
    for (int64_t i = 0; i < h.n; ++i)
      for (int64_t p = h.rp[i]; p < h.rp[i + 1]; ++p) {
        const int64_t j = h.col[p];
        const int32_t* b = h.col.data() + h.rp[j];
        const int32_t* e = h.col.data() + h.rp[j + 1];
        const int32_t* f = std::lower_bound(b, e, static_cast<int32_t>(i));
        if (f == e || *f != i || !value_eq(h, p, f - h.col.data()))
          fail(GBX_INVALID_VALUE, "symmetric write requires a symmetric matrix");
      }
  }
  // body rows formatted by host threads over row ranges, written in order
  unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (h.nnz < (1 << 16)) nt = 1;
  std::vector<std::string> part(nt);
  std::vector<uint64_t> cnt(nt, 0);
  auto work = [&](unsigned t) {
    const int64_t r0 = h.n * t / nt, r1 = h.n * (t + 1) / nt;
    std::string& s = part[t];
    char buf[48];
    for (int64_t i = r0; i < r1; ++i)
      for (int64_t p = h.rp[i]; p < h.rp[i + 1]; ++p) {
        const int64_t j = h.col[p];
        if (symmetric && j > i) continue;
        const int k = std::snprintf(buf, sizeof buf, "%lld %lld", static_cast<long long>(i + 1),
                                    static_cast<long long>(j + 1));
        s.append(buf, k);
        if (!pattern) {
          s += ' ';
          format_value(h, p, s);
        }
        s += '\n';
        ++cnt[t];
      }
  };
  {
    std::vector<std::thread> th;
    for (unsigned t = 1; t < nt; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
  }
  uint64_t emitted = 0;
  for (auto c : cnt) emitted += c;
  std::string head = std::string("%%MatrixMarket matrix coordinate ") + field + ' ' +
                     (symmetric ? "symmetric" : "general") + "\n%%domain " +
                     domain_name(h.domain) + "\n" + std::to_string(h.n) + ' ' +
                     std::to_string(h.n) + ' ' + std::to_string(emitted) + "\n";
  o.put(head.data(), head.size());
  for (auto& s : part) o.put(s.data(), s.size());
}

}  // namespace

void graph_read(gbx_graph* g, const char* path, const void* data, size_t len, const char* format,
                int kind) {
  NvtxRange nvtx_("gbx.graph_read");
  if (!format) fail(GBX_NULL_ARGUMENT, "format is NULL");
  const std::string fmt(format);
  if (fmt != "bin" && fmt != "mm") fail(GBX_INVALID_VALUE, "unknown format '" + fmt + "'");
  if (fmt == "bin") {
    Reader rd;
    File f(path ? path : "", "rb");
    if (path) {
      if (!f.f) fail(GBX_IO_FAILURE, std::string("cannot open ") + path);
      rd.f = f.f;
    } else {
      rd.buf = static_cast<const uint8_t*>(data);
      rd.len = len;
    }
    read_lagk(g, rd, kind);
  } else if (path) {
    const std::vector<char> d = slurp(path);
    read_mm(g, d.data(), d.size(), kind);
  } else {
    read_mm(g, static_cast<const char*>(data), len, kind);
  }
}

void graph_write(gbx_graph* g, const char* path, const char* format, int symmetric) {
  if (!format || !path) fail(GBX_NULL_ARGUMENT, "path / format is NULL");
  const std::string fmt(format);
  if (fmt != "bin" && fmt != "mm") fail(GBX_INVALID_VALUE, "unknown format '" + fmt + "'");
  const HostCsr h = export_host(g);
  File f(path, "wb");
  if (!f.f) fail(GBX_IO_FAILURE, std::string("cannot open ") + path);
  Out o{f.f};
  if (fmt == "bin") write_lagk(h, o);
  else write_mm(h, o, symmetric != 0);
  if (std::fflush(f.f) != 0) fail(GBX_IO_FAILURE, "stream write failed");
}

}  // namespace gbx
