// tc.cu -- triangle counting (algo/triangle.cpp:30-64).
//
// The reference computes C<s(L)> = L plus.pair U' with an unmasked Gustavson
// product and reduces it (triangle.cpp:49-62).  The count is invariant under
// vertex relabeling (test_tc.cpp:43-55, 75-85), so the device path always
// orients every edge from the lower to the higher (degree, id) rank -- the
// reference's ascending-degree presort (util.cpp:35-44) -- and never
// materialises C (the fusion the paper asks for).
//
// Every triangle i < j < k (rank order) is counted once, at its MIDDLE vertex
// j: for each in-neighbour i of j (j in U(i)), the tail of U(i) after j is
// probed against U(j).  The probes are the wedges i -> (j, k) with j < k both
// in U(i): sum_i C(dU(i), 2), 3.6x fewer than the sum_{j in U(i)} dU(j) of
// probing U(j) against U(i) at R-MAT scale 20 (measured on the generator).
//
// Plan (built once per graph): U in rank space, and L = its transpose as
// (tail start, tail end) pairs into U -- entry (i, p) of L(j), p the position
// of j in U(i), stores [p+1, urp[i+1]).  Work items are <= kTcItem in-
// neighbours of one j; a warp keeps U(j) in a shared-memory hash across the
// consecutive items of the same j.  Rows with dU(j) > kTcWarpCap use a CTA and
// a larger table; beyond kTcCtaCap a binary search in global memory.
// Algorithmic bytes: 4*W2 (streamed tail elements) + 8*nnz(U)
// (tails) + 4*nnz(U) (hashed rows) + 8*(n+1), W2 = sum_i C(dU(i), 2).
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "plans.cuh"

namespace gbx {

constexpr int kTcWarpCap = 512;         // max dU(j) for the warp kernel's hash
constexpr int64_t kTcSpan = 32 * 1024;  // max rank span of U(j) for the warp kernel's bitmap
constexpr int kTcWarpSlots = 1024;      // hash slots per warp: 256 buckets x 4 (load <= 0.5)
constexpr int kTcWarpsPerCta = 8;
constexpr int kTcCtaCap = 16384;        // max dU(i) for the CTA kernel
constexpr int kTcCtaSlots = 32768;      // 128 KB dynamic shared memory
constexpr int kTcRowChunk = 8;            // work items per atomic grab
constexpr int64_t kTcItem = 64;           // in-neighbours (tails) per work item
#ifndef GBX_TC_LONG
#define GBX_TC_LONG 32
#endif
#ifndef GBX_TC_VEC
#define GBX_TC_VEC 0  // 16-byte loads on the long-tail walks (measured slower: masking)
#endif
#ifndef GBX_TC_UNROLL
#define GBX_TC_UNROLL 4
#endif
constexpr int kTcLong = GBX_TC_LONG;      // tails this long are walked by the whole warp
constexpr int kTcUnroll = GBX_TC_UNROLL;  // loads in flight per lane on those walks
constexpr int64_t kTcCtaItem = 1024;      // ... per CTA work item (heavy middle vertices)
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

// The probed set U(j) in shared memory: a bitmap over [base, base + span)
// when U(j)'s rank span is at most kTcSpan (97% of the probe work at R-MAT
// scale 20: in rank space the neighbours of a high-rank vertex are close),
// else the bucketed hash.
struct TcSet {
  const int* mem;
  int log_slots;
  int32_t base;
  uint32_t span;  // 0: hash
  __device__ __forceinline__ bool has(int32_t k) const {
    if (span) {
      const uint32_t o = static_cast<uint32_t>(k - base);
      return o < span && ((static_cast<uint32_t>(mem[o >> 5]) >> (o & 31)) & 1u);
    }
    return tc_lookup(mem, log_slots, k);
  }
};

// Build the set for U(j) = ucol[b, e) with `nthreads` cooperating threads
// (index t); the caller synchronises before and after.
__device__ __forceinline__ TcSet tc_build(int* mem, const int32_t* __restrict__ ucol, int64_t b,
                                          int64_t e, int t, int nthreads, bool clear_only) {
  TcSet S;
  S.mem = mem;
  const int64_t du = e - b;
  const int32_t lo = __ldg(ucol + b), hi = __ldg(ucol + e - 1);
  const int64_t span = static_cast<int64_t>(hi) - lo + 1;
  if (span < kTcSpan) {
    S.span = static_cast<uint32_t>(span);
    S.base = lo;
    S.log_slots = 0;
    if (clear_only) {
      // words [0, span/32]: bit `span` stays 0, the clamp target of tc_has
      for (int w = t; w <= span / 32; w += nthreads) mem[w] = 0;
    } else {
      for (int64_t q = b + t; q < e; q += nthreads) {
        const uint32_t o = static_cast<uint32_t>(__ldg(ucol + q) - lo);
        atomicOr(&mem[o >> 5], 1 << (o & 31));
      }
    }
  } else {
    S.span = 0;
    S.base = 0;
    int ls = 5;
    while ((1 << ls) < 2 * du) ++ls;
    S.log_slots = ls;
    if (clear_only) {
      for (int w = t; w < (1 << ls); w += nthreads) mem[w] = -1;
    } else {
      for (int64_t q = b + t; q < e; q += nthreads) tc_insert(mem, ls, __ldg(ucol + q));
    }
  }
  return S;
}

// membership test with the set's kind fixed at compile time (the probe loop
// is issue-bound: no per-probe branch on the kind)
template <bool kBm>
__device__ __forceinline__ unsigned tc_has(const TcSet& S, int32_t k) {
  if constexpr (kBm) {
    // branch-free: an offset outside the span is clamped onto bit `span`,
    // which the build keeps 0
    const uint32_t o = min(static_cast<uint32_t>(k - S.base), S.span);
    return (static_cast<uint32_t>(S.mem[o >> 5]) >> (o & 31)) & 1u;
  } else {
    return tc_lookup(S.mem, S.log_slots, k) ? 1u : 0u;
  }
}

// Stream the tails L(j)[qb, qe) over a warp group, probing every element in
// the set.  Each round takes 32 tails: tails of >= 32 elements are walked by
// the whole warp one at a time with 16-byte loads (4 probes per load, from the
// 4-aligned element at or below the tail start; out-of-tail lanes masked),
// shorter ones are concatenated and spread over the lanes (owner of an
// element by binary search in shared memory over the prefix sums).  32-bit
// counts per call (a call probes < 2^32 elements).
template <int kWarps, bool kBm>
__device__ __forceinline__ unsigned long long tc_stream_tails_k(
    const int2* __restrict__ tails, const int32_t* __restrict__ ucol, int qb, int qe,
    const TcSet& S, int lane, int warp_in_group, int* s_incl, int* s_sx) {
  unsigned cnt = 0;
  for (int base = qb + 32 * warp_in_group; base < qe; base += 32 * kWarps) {
    const int q = base + lane;
    int s = 0, len = 0;
    if (q < qe) {
      const int2 t = __ldg(tails + q);
      s = t.x;
      len = t.y - t.x;
    }
    unsigned longs = __ballot_sync(kFullMask, len >= kTcLong);
    while (longs) {
      const int src = __ffs(longs) - 1;
      longs &= longs - 1;
      const int ls = __shfl_sync(kFullMask, s, src);
      const int le = ls + __shfl_sync(kFullMask, len, src);
#if GBX_TC_VEC
      const int a0 = ls & ~3;  // ucol is 256-byte aligned: int4 at multiples of 4
      for (int e = a0 + 4 * lane; e < le; e += 128 * kTcUnroll) {
        int4 v[kTcUnroll];
#pragma unroll
        for (int u = 0; u < kTcUnroll; ++u)
          v[u] = e + 128 * u < le ? __ldg(reinterpret_cast<const int4*>(ucol + e + 128 * u))
                                  : make_int4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < kTcUnroll; ++u) {
          const int x = e + 128 * u;
          if (x < le) {
            const int k4[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
            for (int c = 0; c < 4; ++c)
              if (x + c >= ls && x + c < le) cnt += tc_has<kBm>(S, k4[c]);
          }
        }
      }
#else
      for (int e = ls + lane; e < le; e += 32 * kTcUnroll) {
        int32_t k[kTcUnroll];
        if (e - lane + 32 * kTcUnroll <= le) {
          // a full round (warp-uniform): no per-probe bounds
#pragma unroll
          for (int u = 0; u < kTcUnroll; ++u) k[u] = __ldg(ucol + e + 32 * u);
#pragma unroll
          for (int u = 0; u < kTcUnroll; ++u) cnt += tc_has<kBm>(S, k[u]);
        } else {
#pragma unroll
          for (int u = 0; u < kTcUnroll; ++u) k[u] = e + 32 * u < le ? __ldg(ucol + e + 32 * u) : 0;
#pragma unroll
          for (int u = 0; u < kTcUnroll; ++u)
            if (e + 32 * u < le) cnt += tc_has<kBm>(S, k[u]);
        }
      }
#endif
    }
    if (len >= kTcLong) len = 0;
    int incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(kFullMask, incl, o);
      if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(kFullMask, incl, 31);
    s_incl[lane] = incl;
    s_sx[lane] = s - (incl - len);
    __syncwarp();
    for (int e = lane; e < total; e += 32) {
      int lo = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1)
        if (s_incl[lo + step - 1] <= e) lo += step;
      cnt += tc_has<kBm>(S, __ldg(ucol + s_sx[lo] + e));
    }
    __syncwarp();
  }
  return cnt;
}

template <int kWarps>
__device__ __forceinline__ unsigned long long tc_stream_tails(
    const int2* __restrict__ tails, const int32_t* __restrict__ ucol, int qb, int qe,
    const TcSet& S, int lane, int warp_in_group, int* s_incl, int* s_sx) {
  return S.span ? tc_stream_tails_k<kWarps, true>(tails, ucol, qb, qe, S, lane, warp_in_group,
                                                  s_incl, s_sx)
                : tc_stream_tails_k<kWarps, false>(tails, ucol, qb, qe, S, lane, warp_in_group,
                                                   s_incl, s_sx);
}

struct TcArgs {
  const int64_t* urp;
  const int32_t* ucol;
  const int64_t* lrp;
  const int2* tails;
  const int64_t* items;  // j << 32 | chunk
  int64_t item_begin, item_end;
  unsigned* next_item;
  unsigned long long* count;
};

__global__ void __launch_bounds__(32 * kTcWarpsPerCta) k_tc_warp(TcArgs a) {
  __shared__ __align__(16) int tables[kTcWarpsPerCta][kTcWarpSlots];
  __shared__ int owners[kTcWarpsPerCta][64];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  int* table = tables[wid];
  unsigned long long cnt = 0;
  const int64_t nitems = a.item_end - a.item_begin;
  int64_t cur = -1;
  TcSet S{};
  for (;;) {
    unsigned chunk = 0;
    if (lane == 0) chunk = atomicAdd(a.next_item, static_cast<unsigned>(kTcRowChunk));
    chunk = __shfl_sync(kFullMask, chunk, 0);
    if (static_cast<int64_t>(chunk) >= nitems) break;
    const int64_t cend = static_cast<int64_t>(chunk) + kTcRowChunk;
    const int64_t rend = cend < nitems ? cend : nitems;
    for (int64_t r = chunk; r < rend; ++r) {
      const int64_t it = __ldg(a.items + a.item_begin + r);
      const int64_t j = it >> 32;
      const int64_t c = it & 0xffffffff;
      const int64_t lb = __ldg(a.lrp + j), le = __ldg(a.lrp + j + 1);
      const int qb = static_cast<int>(lb + c * kTcItem);
      const int qe = static_cast<int>(min(le, lb + (c + 1) * kTcItem));
      if (j != cur) {  // U(j) into the set (kept for the next items of j)
        const int64_t b = __ldg(a.urp + j), e = __ldg(a.urp + j + 1);
        __syncwarp();
        tc_build(table, a.ucol, b, e, lane, 32, true);
        __syncwarp();
        S = tc_build(table, a.ucol, b, e, lane, 32, false);
        __syncwarp();
        cur = j;
      }
      cnt += tc_stream_tails<1>(a.tails, a.ucol, qb, qe, S, lane, 0, owners[wid], owners[wid] + 32);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(kFullMask, cnt, o);
  if (lane == 0 && cnt) atomicAdd(a.count, cnt);
}

// heavy middle vertices (kTcWarpCap < dU(j) <= kTcCtaCap): CTA work items of
// <= kTcCtaItem in-neighbours; a CTA keeps U(j) hashed across consecutive items
__global__ void __launch_bounds__(512) k_tc_cta(const int64_t* urp, const int32_t* ucol,
                                                const int64_t* lrp, const int2* tails,
                                                const int64_t* items, int64_t nitems,
                                                unsigned* next_item, unsigned long long* count) {
  extern __shared__ __align__(16) int table[];
  __shared__ int owners[16][64];
  __shared__ unsigned s_item;
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  constexpr int kW = 16;
  unsigned long long cnt = 0;
  int64_t cur = -1;
  TcSet S{};
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_item = atomicAdd(next_item, 1u);
    __syncthreads();
    const int64_t r = s_item;
    if (r >= nitems) break;
    const int64_t it = items[r];
    const int64_t j = it >> 32, c = it & 0xffffffff;
    if (j != cur) {
      const int64_t b = urp[j], e = urp[j + 1];
      tc_build(table, ucol, b, e, threadIdx.x, blockDim.x, true);
      __syncthreads();
      S = tc_build(table, ucol, b, e, threadIdx.x, blockDim.x, false);
      __syncthreads();
      cur = j;
    }
    const int64_t lb = lrp[j], le = lrp[j + 1];
    const int qb = static_cast<int>(lb + c * kTcCtaItem);
    const int qe = static_cast<int>(min(le, lb + (c + 1) * kTcCtaItem));
    cnt += tc_stream_tails<kW>(tails, ucol, qb, qe, S, lane, wid, owners[wid], owners[wid] + 32);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(kFullMask, cnt, o);
  if (lane == 0 && cnt) atomicAdd(count, cnt);
}

// fallback for middle vertices with U(j) too long for shared memory: binary
// search of every tail element in the global U(j)
__global__ void k_tc_global(const int64_t* urp, const int32_t* ucol, const int64_t* lrp,
                            const int2* tails, const int32_t* rows, int64_t nrows,
                            unsigned long long* count) {
  unsigned long long cnt = 0;
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int64_t j = rows[r];
    const int64_t b = urp[j], e = urp[j + 1];
    for (int64_t q = lrp[j]; q < lrp[j + 1]; ++q) {
      const int2 t = tails[q];
      for (int64_t p = t.x + threadIdx.x; p < t.y; p += blockDim.x) {
        const int32_t k = ucol[p];
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

// per middle vertex j: probe work = sum of its in-neighbours' tails + dU(j)
__global__ void k_row_work(const int64_t* urp, const int64_t* lrp, const int2* tails, int64_t n,
                           int64_t* work) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = w; j < n; j += nw) {
    const int64_t du = urp[j + 1] - urp[j];
    int64_t s = 0;
    if (du > 0)
      for (int64_t q = lrp[j] + lane; q < lrp[j + 1]; q += 32) s += tails[q].y - tails[q].x;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFullMask, s, o);
    if (lane == 0) work[j] = du > 0 ? s + du : 0;
  }
}

// row id of every U entry (warp per row)
__global__ void k_u_rows(const int64_t* urp, int64_t n, int32_t* rowu) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = w; i < n; i += nw)
    for (int64_t p = urp[i] + lane; p < urp[i + 1]; p += 32) rowu[p] = static_cast<int32_t>(i);
}

// L keys: (j = ucol[p]) << 31 | p
__global__ void k_l_keys(const int32_t* ucol, int64_t m, uint64_t* keys) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p < m) keys[p] = (static_cast<uint64_t>(ucol[p]) << 31) | static_cast<uint64_t>(p);
}

// tails[q] = [p + 1, urp[i + 1]) for L entry q = (i, p)
__global__ void k_l_tails(const int32_t* lcol, const int32_t* rowu, const int64_t* urp, int64_t m,
                          int2* tails) {
  const int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (q >= m) return;
  const int32_t p = lcol[q];
  tails[q] = make_int2(p + 1, static_cast<int>(urp[rowu[p] + 1]));
}

// work items per middle vertex j handled by the warp kernel: ceil(|L(j)| / kTcItem)
// when 1 <= dU(j) <= kTcWarpCap; class[j] = 1 (CTA) / 2 (global) for longer U(j)
__global__ void k_item_counts(const int64_t* urp, const int32_t* ucol, const int64_t* lrp,
                              int64_t n, int64_t* cnt, int8_t* cls) {
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (j >= n) return;
  const int64_t du = urp[j + 1] - urp[j], nl = lrp[j + 1] - lrp[j];
  int64_t k = 0;
  int8_t c = 0;
  if (du > 0 && nl > 0) {
    const int64_t span = static_cast<int64_t>(ucol[urp[j + 1] - 1]) - ucol[urp[j]] + 1;
    if (span < kTcSpan || du <= kTcWarpCap) k = (nl + kTcItem - 1) / kTcItem;
    else c = du <= kTcCtaCap ? 1 : 2;
  }
  cnt[j] = k;
  cls[j] = c;
}

__global__ void k_item_fill(const int64_t* off, int64_t n, int64_t* items) {
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (j >= n) return;
  for (int64_t c = 0; c < off[j + 1] - off[j]; ++c) items[off[j] + c] = (j << 32) | c;
}

// U keys (rank(i) << bits | rank(j)) for every entry pointing up in rank
// (the rest: drop keys); rank = stable ascending (degree, id) order
void tc_upper_keys(cudaStream_t s, const Csr& A, const int32_t* deg, int64_t n, int bits,
                   uint64_t* keys) {
  DevArray<int32_t> perm, rank, rowid;
  sort_ids_by_key(s, deg, n, true, perm);
  rank.alloc(std::max<int64_t>(n, 1));
  if (n) {
    k_scatter_rank<<<ceil_div(n, 256), 256, 0, s>>>(perm.p, n, rank.p);
    GBX_LAUNCHED();
  }
  perm.release();
  const int64_t m = A.nnz;
  if (m) {
    expand_rows(s, A, rowid);
    k_upper_keys<<<ceil_div(m, 256), 256, 0, s>>>(rowid.p, A.col.p, rank.p, m, bits, keys);
    GBX_LAUNCHED();
  }
  GBX_CUDA(cudaStreamSynchronize(s));
}

void tc_plan_from_upper(gbx_graph* g, int64_t n, int bits, const uint64_t* sorted, int64_t unnz,
                        uint64_t* scratch, uint64_t* scratch2);

void tc_prepare(gbx_graph* g) {
  NvtxRange nvtx_("gbx.triangle_count.prepare");
  if (g->tc) return;
  cudaStream_t s = g->stream;
  const Csr& A = g->A;
  const int64_t n = A.n;
  DevArray<int32_t> deg_tmp;
  const int32_t* deg = g->has_rowdeg ? g->rowdeg.p : nullptr;
  if (!deg) {
    compute_degrees(s, A, deg_tmp, true);
    deg = deg_tmp.p;
  }
  const int bits = bits_for(std::max<int64_t>(n, 2));
  int64_t m = A.nnz;
  DevArray<uint64_t> k0(std::max<int64_t>(m, 1)), k1(std::max<int64_t>(m, 1));
  tc_upper_keys(s, A, deg, n, bits, k0.p);
  uint64_t* sorted = m ? sort_keys(s, k0.p, k1.p, m, 2 * bits + 1) : k0.p;
  // the graph is symmetric and loop-free (checked by the caller): exactly half
  // of the entries point up in rank
  tc_plan_from_upper(g, n, bits, sorted, m / 2, sorted == k0.p ? k1.p : k0.p,
                     const_cast<uint64_t*>(sorted));
}

// the plan from U's sorted keys (unnz of them); scratch, scratch2: buffers of
// >= unnz keys (scratch2 may be `sorted` itself: it is consumed first)
void tc_plan_from_upper(gbx_graph* g, int64_t n, int bits, const uint64_t* sorted, int64_t unnz,
                        uint64_t* scratch, uint64_t* scratch2) {
  cudaStream_t s = g->stream;
  auto P = std::make_unique<TcPlan>();
  P->n = n;
  if (unnz >= (int64_t(1) << 31) - 1)
    fail(GBX_UNSUPPORTED, "triangle_count: nnz(U) >= 2^31 is not supported (32-bit offsets)");
  csr_from_sorted_keys(s, n, bits, sorted, unnz, P->urp, P->ucol);
  P->nnz = unnz;
  // L = U' as tails into U, sorted by middle vertex j
  {
    DevArray<int32_t> rowu(std::max<int64_t>(unnz, 1)), lcol;
    uint64_t* lk = scratch;
    if (unnz) {
      k_u_rows<<<device_sms() * 8, 256, 0, s>>>(P->urp.p, n, rowu.p);
      k_l_keys<<<ceil_div(unnz, 256), 256, 0, s>>>(P->ucol.p, unnz, lk);
      GBX_LAUNCHED();
    }
    uint64_t* ls = unnz ? sort_keys(s, lk, scratch2, unnz, bits + 31) : lk;
    csr_from_sorted_keys(s, n, 31, ls, unnz, P->lrp, lcol);
    P->tails.alloc(std::max<int64_t>(unnz, 1));
    if (unnz) {
      k_l_tails<<<ceil_div(unnz, 256), 256, 0, s>>>(lcol.p, rowu.p, P->urp.p, unnz, P->tails.p);
      GBX_LAUNCHED();
    }
  }
  // work items (warp kernel) and the CTA / global middle vertices
  {
    const int64_t n1 = std::max<int64_t>(n, 1);
    DevArray<int64_t> cnt(n1);
    DevArray<int8_t> cls(n1);
    P->item_off.alloc(n + 1);
    GBX_CUDA(cudaMemsetAsync(P->item_off.p, 0, sizeof(int64_t), s));
    if (n) {
      k_item_counts<<<ceil_div(n, 256), 256, 0, s>>>(P->urp.p, P->ucol.p, P->lrp.p, n, cnt.p, cls.p);
      GBX_LAUNCHED();
      size_t tb = 0;
      GBX_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, cnt.p, P->item_off.p + 1, n, s));
      DevArray<uint8_t> t(tb + 1);
      GBX_CUDA(cub::DeviceScan::InclusiveSum(t.p, tb, cnt.p, P->item_off.p + 1, n, s));
    }
    int64_t nitems = 0;
    GBX_CUDA(cudaMemcpyAsync(&nitems, P->item_off.p + n, 8, cudaMemcpyDeviceToHost, s));
    std::vector<int8_t> hc(n);
    if (n) GBX_CUDA(cudaMemcpyAsync(hc.data(), cls.p, n, cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaStreamSynchronize(s));
    P->nitems = nitems;
    P->items.alloc(std::max<int64_t>(nitems, 1));
    if (n) {
      k_item_fill<<<ceil_div(n, 256), 256, 0, s>>>(P->item_off.p, n, P->items.p);
      GBX_LAUNCHED();
    }
    for (int64_t j = 0; j < n; ++j) {
      if (hc[j] == 1) P->heavy_h.push_back(static_cast<int32_t>(j));
      else if (hc[j] == 2) P->huge_h.push_back(static_cast<int32_t>(j));
    }
    // heavy middle vertices: CTA items of kTcCtaItem in-neighbours (ascending j)
    P->heavy_item_off_h.assign(1, 0);
    std::vector<int64_t> hitems;
    for (int32_t j : P->heavy_h) {
      int64_t l[2];
      GBX_CUDA(cudaMemcpyAsync(l, P->lrp.p + j, 16, cudaMemcpyDeviceToHost, s));
      GBX_CUDA(cudaStreamSynchronize(s));
      const int64_t k = (l[1] - l[0] + kTcCtaItem - 1) / kTcCtaItem;
      for (int64_t c = 0; c < k; ++c) hitems.push_back((static_cast<int64_t>(j) << 32) | c);
      P->heavy_item_off_h.push_back(static_cast<int64_t>(hitems.size()));
    }
    P->heavy_items.alloc(std::max<size_t>(hitems.size(), 1));
    if (!hitems.empty())
      GBX_CUDA(cudaMemcpyAsync(P->heavy_items.p, hitems.data(), hitems.size() * 8,
                               cudaMemcpyHostToDevice, s));
    P->huge.alloc(std::max<size_t>(P->huge_h.size(), 1));
    if (!P->huge_h.empty())
      GBX_CUDA(cudaMemcpyAsync(P->huge.p, P->huge_h.data(), P->huge_h.size() * 4,
                               cudaMemcpyHostToDevice, s));
  }
  P->count.alloc(1);
  P->next_row.alloc(2);
  GBX_CUDA(cudaStreamSynchronize(s));
  g->tc = std::move(P);
}

// [lo, hi) of a sorted id list restricted to [rb, re)
static void id_range(const std::vector<int32_t>& v, int64_t rb, int64_t re, size_t& lo,
                     size_t& hi) {
  lo = std::lower_bound(v.begin(), v.end(), rb) - v.begin();
  hi = std::lower_bound(v.begin(), v.end(), re) - v.begin();
}

// triangles whose middle vertex (rank space) lies in [rb, re)
uint64_t tc_run(gbx_graph* g, int64_t rb, int64_t re) {
  NvtxRange nvtx_("gbx.triangle_count");
  tc_prepare(g);
  TcPlan& P = *g->tc;
  cudaStream_t s = g->stream;
  if (re < 0 || re > P.n) re = P.n;
  if (rb < 0) rb = 0;
  g->stats = gbx_stats{};
  g->pending_iters = nullptr;
  if (re <= rb) return 0;
  // the long-tail walks read U with 16-byte loads from 4-aligned element ids
  if (reinterpret_cast<uintptr_t>(P.ucol.p) % 16 != 0)
    fail(GBX_CUDA_ERROR, "triangle_count: U column array is not 16-byte aligned");
  int64_t ib = 0, ie = P.nitems;
  if (rb > 0 || re < P.n) {
    GBX_CUDA(cudaMemcpyAsync(&ib, P.item_off.p + rb, 8, cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaMemcpyAsync(&ie, P.item_off.p + re, 8, cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaStreamSynchronize(s));
  }
  GBX_CUDA(cudaMemsetAsync(P.count.p, 0, sizeof(unsigned long long), s));
  GBX_CUDA(cudaMemsetAsync(P.next_row.p, 0, sizeof(unsigned), s));
  int launches = 0;
  if (ie > ib) {
    TcArgs a{P.urp.p, P.ucol.p, P.lrp.p, P.tails.p, P.items.p, ib, ie, P.next_row.p, P.count.p};
    static int per_sm = 0;
    if (!per_sm)
      GBX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tc_warp,
                                                             32 * kTcWarpsPerCta, 0));
    const int grid = device_sms() * std::max(per_sm, 1);
    k_tc_warp<<<grid, 32 * kTcWarpsPerCta, 0, s>>>(a);
    GBX_LAUNCHED();
    ++launches;
  }
  size_t lo, hi;
  id_range(P.heavy_h, rb, re, lo, hi);
  const int64_t hib = P.heavy_item_off_h[lo], hie = P.heavy_item_off_h[hi];
  if (hie > hib) {
    const size_t smem = kTcCtaSlots * sizeof(int);
    GBX_CUDA(cudaFuncSetAttribute(k_tc_cta, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    GBX_CUDA(cudaMemsetAsync(P.next_row.p + 1, 0, sizeof(unsigned), s));
    k_tc_cta<<<std::min<int64_t>(hie - hib, device_sms()), 512, smem, s>>>(
        P.urp.p, P.ucol.p, P.lrp.p, P.tails.p, P.heavy_items.p + hib, hie - hib,
        P.next_row.p + 1, P.count.p);
    GBX_LAUNCHED();
    ++launches;
  }
  id_range(P.huge_h, rb, re, lo, hi);
  if (hi > lo) {
    k_tc_global<<<std::min<int64_t>(hi - lo, 4 * device_sms()), 256, 0, s>>>(
        P.urp.p, P.ucol.p, P.lrp.p, P.tails.p, P.huge.p + lo, static_cast<int64_t>(hi - lo),
        P.count.p);
    GBX_LAUNCHED();
    ++launches;
  }
  unsigned long long h = 0;
  GBX_CUDA(cudaMemcpyAsync(&h, P.count.p, sizeof h, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  g->stats.launches = launches;
  g->stats.hot_launches = 1;
  g->stats.work_units = P.nnz;
  return h;
}

// Work-balanced contiguous split of the middle vertices (multi-GPU TC, §8e).
void tc_partition(gbx_graph* g, int parts, int64_t* bounds) {
  if (parts < 1) fail(GBX_INVALID_VALUE, "tc_partition: parts must be >= 1");
  tc_prepare(g);
  TcPlan& P = *g->tc;
  cudaStream_t s = g->stream;
  const int64_t n = P.n;
  DevArray<int64_t> work(std::max<int64_t>(n, 1));
  if (n) {
    k_row_work<<<device_sms() * 8, 256, 0, s>>>(P.urp.p, P.lrp.p, P.tails.p, n, work.p);
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
