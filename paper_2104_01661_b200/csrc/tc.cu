// tc.cu -- triangle counting (algo/triangle.cpp:30-64).
//
// The reference computes C<s(L)> = L plus.pair U' with an unmasked Gustavson
// product and reduces it (triangle.cpp:49-62).  The count is invariant under
// vertex relabeling (test_tc.cpp:43-55, 75-85), so the device path always
// orients every edge from the lower to the higher (degree, id) rank -- the
// reference's ascending-degree presort (util.cpp:35-44) -- and never
// materialises C: for every row i of the oriented U and every j in U(i) it
// counts |U(i) n U(j)|, fusing the mask, the plus.pair product and the
// reduction (the fusion the paper asks for).
//
// Kernel: one warp per row (dU(i) <= 1024): U(i) goes into a shared-memory
// open-addressing hash table, then the concatenated lists U(j), j in U(i), are
// streamed with all 32 lanes (a warp-level prefix sum over dU(j) assigns
// elements to lanes, so short lists do not idle lanes) and probed in the
// table.  Rows with longer U(i) use a whole CTA and a larger table; beyond
// that, a binary search in global memory.  Counts are u64, reduced per warp.
// Algorithmic bytes: 4*W (streamed U(j) elements) + 4*nnz(U) +
// 8*(n+1), W = sum_i sum_{j in U(i)} dU(j).
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "plans.cuh"

namespace gbx {

constexpr int kTcWarpCap = 512;         // max dU(i) for the warp kernel
constexpr int kTcWarpSlots = 1024;      // hash slots per warp: 256 buckets x 4 (load <= 0.5)
constexpr int kTcWarpsPerCta = 8;
constexpr int kTcCtaCap = 16384;        // max dU(i) for the CTA kernel
constexpr int kTcCtaSlots = 32768;      // 128 KB dynamic shared memory
constexpr int kTcRowChunk = 8;
constexpr unsigned kFullMask = 0xffffffffu;

// Shared-memory hash set of U(i): buckets of 4 int32 slots (one 16-byte load
// per probe, no divergent probe chains), bucket = Fibonacci hash of the key,
// linear probing at bucket granularity only when a bucket is full (rare at a
// load factor <= 1/2).  log_slots counts slots (>= 2).
__device__ __forceinline__ uint32_t tc_bucket(int32_t k, int log_buckets) {
  return (static_cast<uint32_t>(k) * 0x9E3779B1u) >> (32 - log_buckets);
}

__device__ __forceinline__ void tc_insert(int* table, int log_slots, int32_t k) {
  const int lb = log_slots - 2;
  const uint32_t bmask = (1u << lb) - 1;
  uint32_t b = tc_bucket(k, lb);
  for (;;) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int prev = atomicCAS(&table[4 * b + q], -1, k);
      if (prev == -1 || prev == k) return;
    }
    b = (b + 1) & bmask;
  }
}

__device__ __forceinline__ bool tc_lookup(const int* table, int log_slots, int32_t k) {
  const int lb = log_slots - 2;
  const uint32_t bmask = (1u << lb) - 1;
  uint32_t b = tc_bucket(k, lb);
  for (;;) {
    const int4 v = *reinterpret_cast<const int4*>(table + 4 * b);
    if (v.x == k || v.y == k || v.z == k || v.w == k) return true;
    if (v.x == -1 || v.y == -1 || v.z == -1 || v.w == -1) return false;
    b = (b + 1) & bmask;
  }
}

// Stream the concatenation of U(j) for j in U(i)[jb, je) over a warp group,
// probing every element in the table.  Each round takes 32 j's, prefix-sums
// their lengths and spreads the elements over the lanes (32-bit offsets:
// nnz(U) < 2^31 is checked by tc_prepare).
template <int kWarps>
__device__ __forceinline__ unsigned long long tc_stream_row(
    const int64_t* __restrict__ urp, const int32_t* __restrict__ ucol, int jb, int je,
    const int* table, int log_slots, int lane, int warp_in_group, int* s_incl, int* s_sx) {
  unsigned long long cnt = 0;
  // each warp of the group takes every kWarps-th block of 32 j's
  for (int base = jb + 32 * warp_in_group; base < je; base += 32 * kWarps) {
    const int p = base + lane;
    int s = 0, len = 0;
    if (p < je) {
      const int32_t j = __ldg(ucol + p);
      s = static_cast<int>(__ldg(urp + j));
      len = static_cast<int>(__ldg(urp + j + 1)) - s;
    }
    int incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(kFullMask, incl, o);
      if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(kFullMask, incl, 31);
    // element e of lane l's list is ucol[sx[l] + e]; owners found in shared memory
    s_incl[lane] = incl;
    s_sx[lane] = s - (incl - len);
    __syncwarp();
    for (int e = lane; e < total; e += 32) {
      int lo = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1)
        if (s_incl[lo + step - 1] <= e) lo += step;
      cnt += tc_lookup(table, log_slots, __ldg(ucol + s_sx[lo] + e)) ? 1ull : 0ull;
    }
    __syncwarp();
  }
  return cnt;
}

struct TcArgs {
  const int64_t* urp;
  const int32_t* ucol;
  int64_t row_begin, row_end;
  unsigned* next_row;
  unsigned long long* count;
};

__global__ void __launch_bounds__(32 * kTcWarpsPerCta) k_tc_warp(TcArgs a) {
  __shared__ __align__(16) int tables[kTcWarpsPerCta][kTcWarpSlots];
  __shared__ int owners[kTcWarpsPerCta][64];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  int* table = tables[wid];
  unsigned long long cnt = 0;
  const int64_t nrows = a.row_end - a.row_begin;
  for (;;) {
    unsigned chunk = 0;
    if (lane == 0) chunk = atomicAdd(a.next_row, static_cast<unsigned>(kTcRowChunk));
    chunk = __shfl_sync(kFullMask, chunk, 0);
    if (static_cast<int64_t>(chunk) >= nrows) break;
    const int64_t cend = static_cast<int64_t>(chunk) + kTcRowChunk;
    const int64_t rend = cend < nrows ? cend : nrows;
    for (int64_t r = chunk; r < rend; ++r) {
      const int64_t i = a.row_begin + r;
      const int64_t b = __ldg(a.urp + i), e = __ldg(a.urp + i + 1);
      const int64_t du = e - b;
      if (du < 2 || du > kTcWarpCap) continue;
      int log_slots = 5;
      while ((1 << log_slots) < 2 * du) ++log_slots;
      const int slots = 1 << log_slots;
      for (int t = lane; t < slots; t += 32) table[t] = -1;
      __syncwarp();
      for (int64_t q = b + lane; q < e; q += 32) tc_insert(table, log_slots, __ldg(a.ucol + q));
      __syncwarp();
      cnt += tc_stream_row<1>(a.urp, a.ucol, static_cast<int>(b), static_cast<int>(e), table,
                              log_slots, lane, 0, owners[wid], owners[wid] + 32);
      __syncwarp();
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(kFullMask, cnt, o);
  if (lane == 0 && cnt) atomicAdd(a.count, cnt);
}

// one CTA per heavy row (kTcWarpCap < dU(i) <= kTcCtaCap)
__global__ void __launch_bounds__(512) k_tc_cta(const int64_t* urp, const int32_t* ucol,
                                                const int32_t* rows, int64_t nrows,
                                                unsigned long long* count) {
  extern __shared__ __align__(16) int table[];
  __shared__ int owners[16][64];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  constexpr int kW = 16;
  unsigned long long cnt = 0;
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int64_t i = rows[r];
    const int64_t b = urp[i], e = urp[i + 1];
    const int64_t du = e - b;
    int log_slots = 5;
    while ((1 << log_slots) < 2 * du) ++log_slots;
    const int slots = 1 << log_slots;
    for (int t = threadIdx.x; t < slots; t += blockDim.x) table[t] = -1;
    __syncthreads();
    for (int64_t q = b + threadIdx.x; q < e; q += blockDim.x) tc_insert(table, log_slots, ucol[q]);
    __syncthreads();
    cnt += tc_stream_row<kW>(urp, ucol, static_cast<int>(b), static_cast<int>(e), table,
                             log_slots, lane, wid, owners[wid], owners[wid] + 32);
    __syncthreads();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(kFullMask, cnt, o);
  if (lane == 0 && cnt) atomicAdd(count, cnt);
}

// fallback for rows too long for shared memory: binary search in global U(i)
__global__ void k_tc_global(const int64_t* urp, const int32_t* ucol, const int32_t* rows,
                            int64_t nrows, unsigned long long* count) {
  unsigned long long cnt = 0;
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int64_t i = rows[r];
    const int64_t b = urp[i], e = urp[i + 1];
    for (int64_t p = b; p < e; ++p) {
      const int32_t j = ucol[p];
      for (int64_t q = urp[j] + threadIdx.x; q < urp[j + 1]; q += blockDim.x) {
        const int32_t k = ucol[q];
        int64_t lo = b, hi = e;
        while (lo < hi) {
          int64_t mid = (lo + hi) >> 1;
          if (ucol[mid] < k) lo = mid + 1; else hi = mid;
        }
        if (lo < e && ucol[lo] == k) ++cnt;
      }
    }
  }
  atomicAdd(count, cnt);
}

// ---- plan: rank by (degree, id), keep the edges pointing up in rank --------

__global__ void k_scatter_rank(const int32_t* perm, int64_t n, int32_t* rank) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) rank[perm[i]] = static_cast<int32_t>(i);
}

__global__ void k_upper_keys(const int32_t* rowid, const int32_t* col, const int32_t* rank,
                             int64_t nnz, int bits, uint64_t* keys) {
  int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p >= nnz) return;
  const int32_t rv = rank[rowid[p]], rw = rank[col[p]];
  keys[p] = rw > rv ? ((static_cast<uint64_t>(rv) << bits) | static_cast<uint64_t>(rw))
                    : (uint64_t(1) << (2 * bits));
}

__global__ void k_row_work(const int64_t* urp, const int32_t* ucol, int64_t n, int64_t* work) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = w; i < n; i += nw) {
    int64_t s = 0;
    for (int64_t p = urp[i] + lane; p < urp[i + 1]; p += 32) {
      int32_t j = ucol[p];
      s += urp[j + 1] - urp[j];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFullMask, s, o);
    if (lane == 0) work[i] = s + (urp[i + 1] - urp[i]);
  }
}

void tc_prepare(gbx_graph* g) {
  if (g->tc) return;
  cudaStream_t s = g->stream;
  const Csr& A = g->A;
  const int64_t n = A.n;
  auto P = std::make_unique<TcPlan>();
  P->n = n;
  DevArray<int32_t> deg_tmp;
  const int32_t* deg = g->has_rowdeg ? g->rowdeg.p : nullptr;
  if (!deg) {
    compute_degrees(s, A, deg_tmp, true);
    deg = deg_tmp.p;
  }
  DevArray<int32_t> perm, rank, rowid;
  sort_ids_by_key(s, deg, n, true, perm);
  rank.alloc(std::max<int64_t>(n, 1));
  if (n) {
    k_scatter_rank<<<ceil_div(n, 256), 256, 0, s>>>(perm.p, n, rank.p);
    GBX_LAUNCHED();
  }
  perm.release();
  const int bits = bits_for(std::max<int64_t>(n, 2));
  int64_t m = A.nnz;
  DevArray<uint64_t> k0(std::max<int64_t>(m, 1)), k1(std::max<int64_t>(m, 1));
  if (m) {
    expand_rows(s, A, rowid);
    k_upper_keys<<<ceil_div(m, 256), 256, 0, s>>>(rowid.p, A.col.p, rank.p, m, bits, k0.p);
    GBX_LAUNCHED();
    rowid.release();
  }
  uint64_t* sorted = m ? sort_keys(s, k0.p, k1.p, m, 2 * bits + 1) : k0.p;
  // the graph is symmetric and loop-free (checked by the caller): exactly half
  // of the entries point up in rank
  const int64_t unnz = m / 2;
  if (unnz >= (int64_t(1) << 31) - 1)
    fail(GBX_UNSUPPORTED, "triangle_count: nnz(U) >= 2^31 is not supported (32-bit offsets)");
  csr_from_sorted_keys(s, n, bits, sorted, unnz, P->urp, P->ucol);
  P->nnz = unnz;
  P->count.alloc(1);
  P->next_row.alloc(1);
  GBX_CUDA(cudaStreamSynchronize(s));
  g->tc = std::move(P);
}

static void tc_heavy_rows(gbx_graph* g, int64_t rb, int64_t re, std::vector<int32_t>& heavy,
                          std::vector<int32_t>& huge) {
  TcPlan& P = *g->tc;
  std::vector<int64_t> rp(re - rb + 1);
  if (re > rb)
    GBX_CUDA(cudaMemcpyAsync(rp.data(), P.urp.p + rb, (re - rb + 1) * 8, cudaMemcpyDeviceToHost,
                             g->stream));
  GBX_CUDA(cudaStreamSynchronize(g->stream));
  for (int64_t i = rb; i < re; ++i) {
    int64_t du = rp[i - rb + 1] - rp[i - rb];
    if (du > kTcCtaCap) huge.push_back(static_cast<int32_t>(i));
    else if (du > kTcWarpCap) heavy.push_back(static_cast<int32_t>(i));
  }
}

uint64_t tc_run(gbx_graph* g, int64_t rb, int64_t re) {
  tc_prepare(g);
  TcPlan& P = *g->tc;
  cudaStream_t s = g->stream;
  if (re < 0 || re > P.n) re = P.n;
  if (rb < 0) rb = 0;
  g->stats = gbx_stats{};
  if (re <= rb) return 0;
  GBX_CUDA(cudaMemsetAsync(P.count.p, 0, sizeof(unsigned long long), s));
  GBX_CUDA(cudaMemsetAsync(P.next_row.p, 0, sizeof(unsigned), s));
  TcArgs a{P.urp.p, P.ucol.p, rb, re, P.next_row.p, P.count.p};
  int per_sm = 0;
  GBX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tc_warp, 32 * kTcWarpsPerCta, 0));
  const int grid = device_sms() * std::max(per_sm, 1);
  k_tc_warp<<<grid, 32 * kTcWarpsPerCta, 0, s>>>(a);
  GBX_LAUNCHED();
  int launches = 1;
  std::vector<int32_t> heavy, huge;
  tc_heavy_rows(g, rb, re, heavy, huge);
  int32_t* drows = nullptr;
  const size_t nr = std::max(heavy.size(), huge.size());
  if (nr) {
    GBX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&drows), nr * 4, s));
  }
  if (!heavy.empty()) {
    GBX_CUDA(cudaMemcpyAsync(drows, heavy.data(), heavy.size() * 4, cudaMemcpyHostToDevice, s));
    const size_t smem = kTcCtaSlots * sizeof(int);
    GBX_CUDA(cudaFuncSetAttribute(k_tc_cta, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    k_tc_cta<<<std::min<int64_t>(heavy.size(), 4 * device_sms()), 512, smem, s>>>(
        P.urp.p, P.ucol.p, drows, static_cast<int64_t>(heavy.size()), P.count.p);
    GBX_LAUNCHED();
    ++launches;
  }
  if (!huge.empty()) {
    GBX_CUDA(cudaStreamSynchronize(s));
    GBX_CUDA(cudaMemcpyAsync(drows, huge.data(), huge.size() * 4, cudaMemcpyHostToDevice, s));
    k_tc_global<<<std::min<int64_t>(huge.size(), 4 * device_sms()), 256, 0, s>>>(
        P.urp.p, P.ucol.p, drows, static_cast<int64_t>(huge.size()), P.count.p);
    GBX_LAUNCHED();
    ++launches;
  }
  if (drows) cudaFreeAsync(drows, s);
  unsigned long long h = 0;
  GBX_CUDA(cudaMemcpyAsync(&h, P.count.p, sizeof h, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  g->stats.launches = launches;
  g->stats.hot_launches = 1;
  g->stats.work_units = P.nnz;
  return h;
}

// Wedge-balanced contiguous split of the oriented rows (multi-GPU TC, §8e).
void tc_partition(gbx_graph* g, int parts, int64_t* bounds) {
  if (parts < 1) fail(GBX_INVALID_VALUE, "tc_partition: parts must be >= 1");
  tc_prepare(g);
  TcPlan& P = *g->tc;
  cudaStream_t s = g->stream;
  const int64_t n = P.n;
  DevArray<int64_t> work(std::max<int64_t>(n, 1));
  if (n) {
    k_row_work<<<device_sms() * 8, 256, 0, s>>>(P.urp.p, P.ucol.p, n, work.p);
    GBX_LAUNCHED();
  }
  std::vector<int64_t> w(n);
  if (n) GBX_CUDA(cudaMemcpyAsync(w.data(), work.p, n * 8, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  int64_t total = 0;
  for (int64_t x : w) total += x;
  bounds[0] = 0;
  int64_t acc = 0, i = 0;
  for (int p = 1; p < parts; ++p) {
    const int64_t target = total / parts * p;
    while (i < n && acc + w[i] <= target) acc += w[i++];
    bounds[p] = i;
  }
  bounds[parts] = n;
}

}  // namespace gbx
