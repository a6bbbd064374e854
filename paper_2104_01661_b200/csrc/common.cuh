// common.cuh -- shared internals of libgbx.so (B200 / sm_100a).
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "gbx.h"

namespace gbx {

// Internal error: carries a gblite::ErrCode-compatible code (error.hpp:13-41).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& m) { throw Error(code, m); }

[[noreturn]] void cuda_fail(cudaError_t e, const char* what, const char* file, int line);
#define GBX_CUDA(x)                                                     \
  do {                                                                  \
    cudaError_t e_ = (x);                                               \
    if (e_ != cudaSuccess) ::gbx::cuda_fail(e_, #x, __FILE__, __LINE__); \
  } while (0)
#define GBX_LAUNCHED() GBX_CUDA(cudaGetLastError())

// Device checks (GBX_DEVICE_CHECKS builds, tools/build_variant.sh): bounds of
// every column-derived gather index in the hot kernels.  compute-sanitizer is
// closed on this GPU pool, so the GPU test suite runs against such a build
// instead (profiles/r02/device_checks.txt).  Compiled out otherwise.
#ifdef GBX_DEVICE_CHECKS
#define GBX_DCHECK(cond, what, val_)                                                       \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      printf("gbx device check failed: %s (%lld) at %s:%d block %d thread %d\n", what,      \
             static_cast<long long>(val_), __FILE__, __LINE__, blockIdx.x, threadIdx.x);    \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define GBX_DCHECK(cond, what, val_) \
  do {                               \
  } while (0)
#endif

// Coherent weak global load for data another CTA rewrites inside the same
// persistent launch (frontier bitmaps, contribution vectors): NOT the .nc
// path (__ldg), which is only defined for data read-only for the whole launch.
// The grid barrier between levels orders it after the writes.
template <typename T>
__device__ __forceinline__ T ld_weak(const T* p) {
  return *p;  // a plain LDG (pointers are not __restrict__, so never promoted to .nc)
}

// Tuning / diagnostics options (options.cu): ONE documented registry set
// through gbx_set_option (include/gbx.h) instead of per-knob environment
// variables.  Read at call time; defaults are the measured optimum.
enum Opt : int {
  kOptPrL1WindowKb = 0,  // "pagerank.l1_window_kb": bytes of x gathered L1 evict_last
  kOptPrCarveout,        // "pagerank.carveout": % shared-memory carveout of the row kernels
  kOptPrHostLoop,        // "pagerank.host_loop": per-iteration launches (ncu captures)
  kOptPrTrace,           // "pagerank.trace": per-phase %globaltimer means on stderr
  kOptP2pTimeoutMs,      // "p2p.timeout_ms": bound of the fused exchange's cross-rank spin
  kOptBfsAlpha,          // "bfs.alpha": push while frontier edges < nnz / alpha (0: reference rule)
  kOptBfs64PullDiv,      // "bfs64.pull_div"
  kOptBfsTrace,          // "bfs.trace": per-level %globaltimer log to stderr
  kOptBfsMgPushDiv,      // "bfs_mg.push_div": multi-GPU BFS pushes while the frontier < n/div
  kOptBcAlpha,           // "bc.alpha"
  kOptBcTrace,           // "bc.trace": per-depth host timing on stderr
  kOptBcBackPush,        // "bc.back_push": backward depth in push form when its children hold <= 1/this of the parents' edges (0: never)
  kOptBcBackPushMinDepth,  // "bc.back_push_min_depth"
  kOptBcRelabelMinN,     // "bc.relabel_min_n": graphs of at least this many vertices run Brandes on a degree-sorted copy (-1: never)
  kOptSsspTrace,         // "sssp.trace": per-phase %globaltimer log to stderr (2: + device printf)
  kOptSsspPullPct,       // "sssp.pull_pct": heavy pass by pull when pops*100 > pct*unpopped (0: never)
  kOptCount
};
int64_t option(Opt o);

// NVTX range over a library call / phase (header-only NVTX 3: a no-op unless a
// tool such as nsys or ncu --nvtx is attached), so a whole-process timeline
// attributes device time to the algorithm phases.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

constexpr int kSMs = 148;  // B200; the runtime value is queried in device_sms()
int device_sms();

// Owning device array.  Persistent graph data and per-plan workspaces, taken
// from the device's stream-ordered pool (kept cached: see Scope) so building
// and freeing graphs does not remap hundreds of MB through cudaMalloc/cudaFree
// each time; allocation and release both synchronise, like cudaMalloc/cudaFree.
// While a ReleaseScope is alive on this thread the device has been
// synchronised and nothing new is launched: DevArray::release skips its own
// cudaDeviceSynchronize (a graph handle owns ~30 arrays).
inline int& release_scope_depth() {
  static thread_local int depth = 0;
  return depth;
}
struct ReleaseScope {
  ReleaseScope() {
    cudaDeviceSynchronize();
    ++release_scope_depth();
  }
  ~ReleaseScope() { --release_scope_depth(); }
  ReleaseScope(const ReleaseScope&) = delete;
  ReleaseScope& operator=(const ReleaseScope&) = delete;
};

template <typename T>
struct DevArray {
  T* p = nullptr;
  size_t n = 0;
  DevArray() = default;
  explicit DevArray(size_t count) { alloc(count); }
  DevArray(const DevArray&) = delete;
  DevArray& operator=(const DevArray&) = delete;
  DevArray(DevArray&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DevArray& operator=(DevArray&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DevArray() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) {
      cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), 0);
      if (e == cudaSuccess) e = cudaStreamSynchronize(0);
      if (e != cudaSuccess) {
        p = nullptr;
        n = 0;
        (void)cudaGetLastError();
        fail(GBX_OUT_OF_MEMORY, "device allocation of " + std::to_string(count * sizeof(T)) +
                                    " bytes failed: " + cudaGetErrorString(e));
      }
    }
  }
  void ensure(size_t count) { if (n < count) alloc(count); }
  void release() {
    if (p) {
      // every stream's work on p is done (a handle's destructor synchronises
      // the device once for all of its arrays: ReleaseScope)
      if (!release_scope_depth()) cudaDeviceSynchronize();
      cudaFreeAsync(p, 0);
    }
    p = nullptr;
    n = 0;
  }
  T* get() const { return p; }
  size_t bytes() const { return n * sizeof(T); }
};

// Device CSR: row_ptr int64[n+1], col int32[nnz] strictly ascending per row
// (SparseMatrix invariant, containers.cpp:104-124), optional values in `domain`.
struct Csr {
  int64_t n = 0;
  int64_t nnz = 0;
  int domain = GBX_BOOL;
  DevArray<int64_t> rp;
  DevArray<int32_t> col;
  DevArray<uint8_t> val;  // raw bytes, element type given by domain
};

size_t domain_size(int domain);

struct PrPlan;
struct TcPlan;
struct SsspPlan;
struct BfsWork;
struct BcWork;
struct CcWork;
struct PrShard;

}  // namespace gbx

// The graph handle (graph.hpp:27-39 restated on the device).
struct gbx_graph {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  int kind = GBX_DIRECTED;
  gbx::Csr A;
  // caches
  bool has_at = false;
  gbx::Csr at_own;  // directed: the transpose; undirected graphs alias A
  // property_at (graph.cpp:30-41) on a directed graph records the cache and
  // builds it on first read: PageRank's plan needs only the in-degrees (from
  // A's columns), so a basic-mode PageRank never pays for a transpose it does
  // not read; BFS pulls, BC, check_graph ... materialise it through AT()
  bool at_pending = false;
  bool has_rowdeg = false, has_coldeg = false;
  gbx::DevArray<int32_t> rowdeg, coldeg;
  // column counts of A taken while the host CSR was uploaded (graph.cu); not a
  // property cache: the PageRank plan reads them instead of recounting
  bool has_colcount = false;
  gbx::DevArray<int32_t> colcount;
  int symmetric = GBX_UNKNOWN;
  int64_t ndiag = -1;
  // derived device layouts (plans), rebuilt after delete_properties
  std::unique_ptr<gbx::PrPlan> pr;
  std::unique_ptr<gbx::TcPlan> tc;
  std::unique_ptr<gbx::SsspPlan> sssp;
  std::unique_ptr<gbx::BfsWork> bfs;
  std::unique_ptr<gbx::BcWork> bc;
  std::unique_ptr<gbx::CcWork> cc;
  std::unique_ptr<gbx::PrShard> prs;
  gbx_stats stats{};
  const int* pending_iters = nullptr;  // device word holding stats.iterations of an async call

  const gbx::Csr& AT() const {
    if (kind == GBX_UNDIRECTED) return A;
    if (at_pending) materialize_at();
    return at_own;
  }
  void materialize_at() const;
  ~gbx_graph();
};

// operand matrix of the GraphBLAS operation layer (ops.cu)
struct gbx_mat {
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t nrows = 0, ncols = 0, nnz = 0;
  int domain = GBX_BOOL;
  gbx::DevArray<int64_t> rp;
  gbx::DevArray<int32_t> col;
  gbx::DevArray<uint64_t> val;  // 8-byte lanes
  // cached transpose (vxm / transpose flags)
  gbx::DevArray<int64_t> trp;
  gbx::DevArray<int32_t> tcol;
  gbx::DevArray<uint64_t> tval;
  bool has_t = false;
  ~gbx_mat() {
    if (stream) {
      cudaSetDevice(device);
      cudaStreamSynchronize(stream);
      cudaStreamDestroy(stream);
    }
  }
};

namespace gbx {

// Warp-aggregated list append: the threads that call it together (coalesced)
// reserve their slots with ONE atomic on the shared counter -- per-thread
// atomics on a single address serialise in L2 (10^5-10^6 per pass).
__device__ __forceinline__ int agg_append(int* cnt) {
  namespace cg = cooperative_groups;
  cg::coalesced_group g = cg::coalesced_threads();
  int base = 0;
  if (g.thread_rank() == 0) base = atomicAdd(cnt, static_cast<int>(g.size()));
  return g.shfl(base, 0) + static_cast<int>(g.thread_rank());
}

}  // namespace gbx

namespace gbx {

// RAII device guard + handle lock for every ABI entry.
struct Scope {
  std::unique_lock<std::mutex> lock;
  explicit Scope(gbx_graph* g);
};

// ---- graph-level primitives (graph.cu) ------------------------------------
void build_from_host(gbx_graph* g, int64_t n, const int64_t* rp, const int64_t* col64,
                     const int32_t* col32, const void* vals, int domain, int kind);
void build_from_coo(gbx_graph* g, int64_t nrows, int64_t ncols, int64_t m, const int64_t* rows,
                    const int64_t* cols, const void* vals, int domain, int dup, int kind,
                    bool host_ptrs);
void graph_read(gbx_graph* g, const char* path, const void* data, size_t len, const char* format,
                int kind);
void graph_write(gbx_graph* g, const char* path, const char* format, int symmetric);
gbx_mat* mat_alloc();
void mat_from_host(gbx_mat* M, int64_t nrows, int64_t ncols, const int64_t* rp, const int64_t* col,
                   const void* vals, int domain);
void mat_from_graph(gbx_mat* M, gbx_graph* g, int which);
void mat_export(gbx_mat* M, int64_t* rp, int64_t* col, void* vals);
void mxv_op(int64_t* w_idx, void* w_vals, int64_t* w_nvals, const gbx_vec* w, const gbx_desc* d,
            int sr, int sdom, gbx_mat* A, const gbx_vec* u);
void vxm_op(int64_t* w_idx, void* w_vals, int64_t* w_nvals, const gbx_vec* w, const gbx_desc* d,
            int sr, int sdom, const gbx_vec* u, gbx_mat* A);
void mxm_op(gbx_mat* out, gbx_mat* C, const gbx_desc* desc, int sr, int sdom, gbx_mat* A,
            gbx_mat* B);
void compute_transpose(cudaStream_t s, const Csr& A, Csr& T);
void rowptr_from_sorted_rows32(cudaStream_t s, int64_t n, const uint32_t* rows, int64_t nnz,
                               int64_t* rp);
void compute_degrees(cudaStream_t s, const Csr& A, DevArray<int32_t>& out, bool by_row);
void require_at(const gbx_graph* g, const char* who);
void require_rowdeg(const gbx_graph* g, const char* who);
void reset_plans(gbx_graph* g);
void set_option(const char* name, int64_t v);
void reset_option(const char* name);
int64_t get_option(const char* name);
const char* option_name(int i);
// stable ascending/descending permutation of ids by key (cub radix, LSD = stable)
void sort_ids_by_key(cudaStream_t s, const int32_t* key, int64_t n, bool ascending,
                     DevArray<int32_t>& perm);
// row ids per nonzero (max-scan over row starts)
void expand_rows(cudaStream_t s, const Csr& A, DevArray<int32_t>& rowid);
void expand_rows_into(cudaStream_t s, const Csr& A, int32_t* rowid);  // nnz entries
// transpose of A under a relabeling, rows ascending in the new ids (pagerank.cu)
void relabeled_transpose(cudaStream_t s, const Csr& A, const int32_t* new2old,
                         const int32_t* old2new, const int32_t* colcount, int64_t* trp,
                         int32_t* tcol);

// Stream-ordered temporary from the device pool (freed on the stream when it
// goes out of scope).
template <typename T>
struct Tmp {
  T* p = nullptr;
  cudaStream_t s;
  Tmp(size_t n, cudaStream_t st) : s(st) {
    if (n) {
      cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&p), n * sizeof(T), s);
      if (e != cudaSuccess) {
        (void)cudaGetLastError();
        fail(GBX_OUT_OF_MEMORY, "cudaMallocAsync of " + std::to_string(n * sizeof(T)) +
                                    " bytes failed");
      }
    }
  }
  ~Tmp() { if (p) cudaFreeAsync(p, s); }
  Tmp(const Tmp&) = delete;
  Tmp& operator=(const Tmp&) = delete;
};
void generate_rmat(gbx_graph* g, int scale, int ef, double a, double b, double c,
                   uint64_t seed, int scramble, int kind);
void generate_er(gbx_graph* g, int logn, int degree, uint64_t seed, int weighted);
void rmat_keys(cudaStream_t s, int scale, int ef, double a, double b, double c, uint64_t seed,
               int scramble, bool sym, int64_t e0, int64_t e1, uint64_t* keys);
void csr_from_keys_unique(cudaStream_t s, int64_t n, int bits, const uint64_t* sorted, int64_t m,
                          Csr& A);
gbx_graph* graph_handle();  // a new empty graph handle on the current device
int64_t count_ndiag(cudaStream_t s, const Csr& A);
bool csr_equal(cudaStream_t s, const Csr& X, const Csr& Y);
void sync(gbx_graph* g);
int bits_for(int64_t n);
uint64_t* sort_keys(cudaStream_t s, uint64_t* keys, uint64_t* alt, int64_t m, int end_bit);
void csr_from_sorted_keys(cudaStream_t s, int64_t n, int bits, const uint64_t* keys,
                          int64_t nnz, DevArray<int64_t>& rp, DevArray<int32_t>& col);

// ---- algorithms ----------------------------------------------------------------
void pagerank_run(gbx_graph* g, double damping, double tol, int itermax, double* rank,
                  int* iters);
void pagerank_prepare(gbx_graph* g);
void bfs_run(gbx_graph* g, uint64_t source, int direction, uint64_t push_divisor,
             bool use_at, int64_t* parent, int64_t* level);
void bfs_batch_run(gbx_graph* g, const uint64_t* sources, uint64_t ns, int64_t* parent,
                   int64_t* level);
void bfs_prepare(gbx_graph* g);
void bfs_shard_begin(gbx_graph* g, uint64_t source, int rank, int nranks, int64_t* rb_out,
                     int64_t* re_out, const int64_t* bounds = nullptr);
void bfs_shard_level(gbx_graph* g, const uint32_t* front, uint32_t* next_slice, int64_t* found);
void bfs_shard_result(gbx_graph* g, int64_t* parent, int64_t* level);
void bfs_shard_push_mark(gbx_graph* g, const uint32_t* front, uint8_t* cand);
int64_t bfs_shard_front_edges(gbx_graph* g, const uint32_t* front);
void bfs_shard_result_device(gbx_graph* g, const int32_t** level, const int32_t** parent);
void bfs_shard_push_level(gbx_graph* g, const uint8_t* cand, const uint32_t* front,
                          uint32_t* next_slice, int64_t* found);
uint64_t tc_run(gbx_graph* g, int64_t row_begin, int64_t row_end);
void tc_prepare(gbx_graph* g);
void tc_partition(gbx_graph* g, int parts, int64_t* bounds);
void tc_upper_keys(cudaStream_t s, const Csr& A, const int32_t* deg, int64_t n, int bits,
                   uint64_t* keys);
void tc_plan_from_upper(gbx_graph* g, int64_t n, int bits, const uint64_t* sorted, int64_t unnz,
                        uint64_t* scratch, uint64_t* scratch2);
void sssp_run(gbx_graph* g, uint64_t source, double delta, double* dist);
void sssp_batch_run(gbx_graph* g, const uint64_t* sources, uint64_t ns, double delta,
                    double* out);
double sssp_default_delta(gbx_graph* g);
void sssp_prepare(gbx_graph* g);
void bc_run(gbx_graph* g, const uint64_t* sources, uint64_t ns, double* centrality);
void bc_shard_begin(gbx_graph* g, const uint64_t* sources, uint64_t ns, int rank, int nranks,
                    int64_t* rb_out, int64_t* re_out, const int64_t* bounds = nullptr);
void bc_shard_forward(gbx_graph* g, void** recs, int64_t* nrec, const uint8_t* cand = nullptr);
int64_t bc_shard_mark(gbx_graph* g, uint8_t* cand);
void bc_shard_forward_apply(gbx_graph* g, const void* recs, int64_t nrec, int* done);
void bc_shard_backward(gbx_graph* g, void** recs, int64_t* nrec, int* done);
void bc_shard_backward_apply(gbx_graph* g, const void* recs, int64_t nrec);
void bc_shard_centrality(gbx_graph* g, double** cent);
void cc_run(gbx_graph* g, int64_t* label, int* iters);
void pr_shard_prepare(gbx_graph* g, int rank, int nranks, int64_t* rb, int64_t* re);
void pr_shard_init(gbx_graph* g, float* x_full, float* r_local, double damping);
void pr_shard_unpermute(gbx_graph* g, const float* r_full, double* out_host);
void pr_shard_step(gbx_graph* g, const float* x_full, const float* r_prev, float* r_new,
                   float* x_slice, double* l1, double damping);
void pr_shard_layout(gbx_graph* g, int64_t* chunk, int64_t* bounds);
std::vector<int64_t> pr_bounds(const int64_t* rp, int64_t n, int64_t nnz, int nranks);
void pr_shard_from_block(gbx_graph* g, int rank, int nranks, Csr& block, DevArray<int32_t>& deg,
                         DevArray<int32_t>& new2old, const std::vector<int64_t>& bounds);
void pr_shard_run_p2p_multi(gbx_graph* const* gs, int nv, const uint64_t* x0_peers,
                            const uint64_t* x1_peers, const uint64_t* l1_peers,
                            const uint64_t* sig_peers, float* const* r0s, float* const* r1s,
                            double damping, double tol, int itermax, int* iters);
void pr_shard_run_p2p(gbx_graph* g, const uint64_t* x0_peers, const uint64_t* x1_peers,
                      const uint64_t* l1_peers, const uint64_t* sig_peers, float* r0, float* r1,
                      double damping, double tol, int itermax, int* iters);
void partition_rows(const gbx_graph* g, int parts, bool transposed, int64_t* bounds);
void result_device(const gbx_graph* g, const std::string& which, void** ptr, int64_t* count);

// ---- device helpers ---------------------------------------------------------------
inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace gbx
