// pagerank.cu -- GAP PageRank (algo/pagerank.cpp:8-81) as a fused pull SpMV,
// looped on the device by a CUDA-graph WHILE node.
//
// Reference per iteration: contrib = prior ./ (deg/damping) (:55-56), rank =
// teleport (:58), rank += AT plus.second contrib (:59-61), L1 = sum|prior -
// rank| (:65-73), stop when L1 < tol (:74).
//
// Device layout (the PageRank plan, built once per graph):
//   * vertices are relabeled by descending in-degree (stable).  R-MAT in- and
//     out-degree skews coincide, so the hot contribution entries x[k] gathered
//     by most edges land in a compact prefix of x that stays L1/L2 resident;
//   * rows are therefore sorted by length and binned: a row of length in
//     (G/2, G] is summed by a group of G lanes (G = 1..32, 32/G rows per warp),
//     rows longer than kPrLong are cut into kPrChunk-nonzero chunks whose
//     partial sums go to fixed slots -- every warp gets a similar amount of
//     work and no block barrier sits in the hot loop.
// Per iteration two kernels run inside the graph body:
//   k_pr_rows   -- every warp unit: coalesced AT column loads (streamed,
//                  evict-first), gathered x (read-only path), fp64 sums, and
//                  the fused epilogue r = teleport + sum, |r_prev - r| (fp64),
//                  x_next = r / (deg / damping) (0 for dangling vertices --
//                  their mass is lost exactly as in the reference);
//   k_pr_finish -- sums the chunk slots of the long rows (warp per row, fixed
//                  lane-strided + shuffle-tree order), their
//                  epilogue, then the last CTA reduces every L1 partial in a
//                  fixed order, counts the iteration and clears the WHILE
//                  condition on convergence.  Deterministic end to end.
// Algorithmic bytes per iteration: (4 + sizeof x) * nnz + 8 * (n+1)
// + (3 * sizeof x + 4) * n.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "plans.cuh"

namespace gbx {

constexpr int kPrThreads = 256;
#ifndef GBX_PR_MINB
#define GBX_PR_MINB 6  // resident CTAs per SM the rows kernel is compiled for
#endif
#ifndef GBX_PR_IPL
#define GBX_PR_IPL 16  // measured: 4 / 8 / 16 -> 219.1 / 215.8 / 215.0 us per iteration
#endif
constexpr int kPrIpl = GBX_PR_IPL;  // chunk walks: independent gathers in flight per lane
#ifndef GBX_PR_B0IPL
#define GBX_PR_B0IPL 2  // measured: 2 and 4 within 1%, 8 slower (registers)
#endif
constexpr int kPrB0Ipl = GBX_PR_B0IPL;  // gathers per lane per step in warp-per-row units
constexpr int64_t kPrLong = 1024;   // rows longer than this are chunked
constexpr int64_t kPrShort = 32;    // rows up to this length: thread per row, exact-length bins
constexpr int64_t kPrChunk = 2048;  // nonzeros per chunk unit
// default shared-memory hot prefix of x (override: GBX_PR_HOT_KB)
constexpr int kPrHotKbDefault = 0;
constexpr unsigned kWarp = 0xffffffffu;
constexpr int kPrMaxPeers = 8;     // ranks of the fused P2P exchange (one NVSwitch box)

PrPlan::~PrPlan() {
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
}

template <typename V>
struct PrArgs {
  const int64_t* trp;      // relabeled AT
  const int32_t* tcol;
  const int32_t* outdeg;   // relabeled out-degree
  const V* inv;            // damping / outdeg (0 for dangling vertices), relabeled
  const PrBin* bins;       // warp units by bin (staged in shared memory)
  int nbins;
  int64_t nunits;
  const int64_t* chunk_p;  // chunk units: nonzero range [p0, p1) -> slot
  int64_t nchunks;
  const int32_t* long_row;     // rows finished by k_pr_finish
  const int64_t* long_slot;    // [nlong+1] slot ranges
  int64_t nlong;
  double* slot;
  V* r0;
  V* r1;
  V* x0;
  V* x1;
  double* l1_rows;     // [gridA] per-CTA partials of k_pr_rows
  double* l1_fin;      // [gridB]
  double* l1_hist;
  int* ctl;            // [0] completed iterations [1] done
  unsigned long long* ktime;  // [128][2]: per iteration, min CTA start / max CTA end (%globaltimer)
  unsigned* fin_cnt;
  int64_t hot;         // x[0, hot) is staged in shared memory by k_pr_rows
  int64_t l1hot;       // x[hot, l1hot) gathered with L1 evict_last, the rest no_allocate
  int64_t row0;        // first row of this plan (shards); outputs indexed row - row0
  int grid_rows;
  double damping, teleport, tol;
  int itermax;
  int fixed;           // single step: r0/x0 inputs, r1/x1 outputs, no convergence
  cudaGraphConditionalHandle cond;
  // fused multi-GPU run (k_pr_persist_p2p): x_next is stored straight into
  // every rank's x buffer over NVLink.  xp[b][q] = rank q's x_b, pre-offset so
  // that xp[b][q][row] is this rank's padded slot entry for relabeled row
  int npeer;
  V* xp[2][kPrMaxPeers];
};

template <typename V>
__device__ __forceinline__ void pr_buffers(const PrArgs<V>& a, int k, const V*& x_cur,
                                           const V*& r_cur, V*& x_nxt, V*& r_nxt) {
  const bool odd = !a.fixed && (k & 1);
  x_cur = odd ? a.x1 : a.x0;
  r_cur = odd ? a.r1 : a.r0;
  x_nxt = odd ? a.x0 : a.x1;
  r_nxt = odd ? a.r0 : a.r1;
}

// Cache-policy loads (PTX): the AT column stream is read once -> no L1
// allocation, evict-first in L2; gathers of the hot prefix of x (the highest-
// degree vertices after relabeling, ~58% of all gathers on R-MAT in the first
// 48K ids) are kept in L1 (evict_last); cold gathers bypass L1 so they do not
// evict the hot lines.
__device__ __forceinline__ int ld_stream(const int32_t* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_hot(const float* p) {
  float v;
  asm("ld.global.nc.L1::evict_last.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_hot(const double* p) {
  double v;
  asm("ld.global.nc.L1::evict_last.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_cold(const float* p) {
  float v;
  asm("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_cold(const double* p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// device clock for the live launch-duration measurement of k_pr_rows (the
// iterations run inside one CUDA graph, where events cannot bracket a node)
__device__ __forceinline__ unsigned long long pr_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// gather x[c]: optional shared-memory prefix [0, hot), L1-resident prefix
// [hot, l1hot), the rest from L2 without L1 allocation
template <typename V>
__device__ __forceinline__ V pr_x(const V* s_x, int64_t hot, const V* x, int c) {
  return c < hot ? s_x[c] : ld_hot(x + c);
}
template <typename V>
__device__ __forceinline__ V pr_xg(const V* s_x, int64_t hot, int64_t l1hot, const V* x, int c) {
  if (c < hot) return s_x[c];
  return c < l1hot ? ld_hot(x + c) : ld_cold(x + c);
}

// fused epilogue of one row with prefetched r_prev / out-degree
template <typename V>
__device__ __forceinline__ double pr_finish_row(const PrArgs<V>& a, V* r_nxt, V* x_nxt,
                                                int64_t row, double s, V rprev, V inv) {
  const double rn = a.teleport + s;
  r_nxt[row - a.row0] = static_cast<V>(rn);
  const V xv = static_cast<V>(rn * static_cast<double>(inv));
  if (a.npeer == 0) {
    x_nxt[row] = xv;
  } else {
    // fused exchange: the contribution goes to every rank's copy of x (peer
    // stores over NVLink; consecutive rows of a warp -> coalesced 128 B writes)
    V* const* xp = a.xp[x_nxt == a.x1 ? 1 : 0];
    for (int q = 0; q < a.npeer; ++q) xp[q][row] = xv;
  }
  return fabs(static_cast<double>(rprev) - rn);
}

// BS = 256: several CTAs per SM, hot prefix in L1 only.  BS = 1024: two CTAs
// per SM, each with a shared-memory copy of the hot prefix of x (random
// gathers are L1TEX-tag bound -- one 32-byte sector per cycle per SM; from
// shared memory they are bank-parallel).
// one iteration's row work for this CTA (every unit of the grid-stride walk);
// returns the CTA's fp64 L1 partial (valid in thread 0)
template <typename V, int BS>
__device__ __forceinline__ double pr_rows_phase(const PrArgs<V>& a, int k,
                                                typename cub::BlockReduce<double, BS>::TempStorage& red,
                                                PrBin* s_bins, V* s_x) {
  using BlockReduce = cub::BlockReduce<double, BS>;
  // the shared-memory prefix exists only in the 1024-thread variant: for 256
  // threads the bound is a compile-time 0 and the per-gather test folds away
  const int64_t hot = BS == 1024 ? a.hot : 0;
  const V *x_cur, *r_cur;
  V *x_nxt, *r_nxt;
  pr_buffers(a, k, x_cur, r_cur, x_nxt, r_nxt);
  {
    // stage the hot prefix of x (16-byte vector loads; hot is a multiple of 16 B)
    constexpr int kVec = 16 / sizeof(V);
    const int4* src = reinterpret_cast<const int4*>(x_cur);
    int4* dst = reinterpret_cast<int4*>(s_x);
    for (int64_t i = threadIdx.x; i < a.hot / kVec; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  for (int i = threadIdx.x; i < a.nbins; i += blockDim.x) s_bins[i] = a.bins[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  double l1 = 0.0;
  // 1) long-row chunks: 32 lanes, kPrIpl independent gathers in flight per lane
  for (int64_t u = gwarp; u < a.nchunks; u += nwarps) {
    const int64_t p0 = a.chunk_p[2 * u], p1 = a.chunk_p[2 * u + 1];
    double s = 0.0;
    for (int64_t base = p0 + lane; base < p1; base += 32 * kPrIpl) {
      int c[kPrIpl];
#pragma unroll
      for (int j = 0; j < kPrIpl; ++j) {
        const int64_t p = base + 32 * j;
        c[j] = p < p1 ? ld_stream(a.tcol + p) : -1;
      }
#pragma unroll
      for (int j = 0; j < kPrIpl; ++j)
        if (c[j] >= 0) s += static_cast<double>(pr_xg(s_x, hot, a.l1hot, x_cur, c[j]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kWarp, s, o);
    if (lane == 0) a.slot[u] = s;
  }
  // 2) warp units in bin order.  Bin 0: rows kPrShort < len <= kPrLong, one
  //    warp per row through row_ptr.  Bins 1..: rows of one exact length L <=
  //    kPrShort, 32 rows per unit, thread per row, nonzeros at p0 + i*L and a
  //    warp-uniform L-trip loop.  The grid-stride walk visits units in
  //    increasing order, so the bin cursor only moves forward.
  int bk = 0;
  for (int64_t u = gwarp; u < a.nunits; u += nwarps) {
    while (bk + 1 < a.nbins && u >= s_bins[bk + 1].unit0) ++bk;
    const PrBin& B = s_bins[bk];
    if (B.len < 0) {
      // one warp per row (kPrShort < len <= kPrLong): coalesced column loads,
      // kPrB0Ipl gathers in flight per lane; the next group of columns is
      // loaded while the current gathers are outstanding
      const int64_t row = B.row0 + (u - B.unit0);
      const int64_t b = a.trp[row], e = a.trp[row + 1];
      const V rprev = r_cur[row - a.row0];
      const V inv = a.inv[row];
      double s = 0.0;
      int c[kPrB0Ipl];
#pragma unroll
      for (int q = 0; q < kPrB0Ipl; ++q) {
        const int64_t p = b + lane + 32 * q;
        c[q] = p < e ? ld_stream(a.tcol + p) : -1;
      }
      for (int64_t base = b + lane; base < e; base += 32 * kPrB0Ipl) {
        int nx[kPrB0Ipl];
#pragma unroll
        for (int q = 0; q < kPrB0Ipl; ++q) {
          const int64_t p = base + 32 * (kPrB0Ipl + q);
          nx[q] = p < e ? ld_stream(a.tcol + p) : -1;
        }
#pragma unroll
        for (int q = 0; q < kPrB0Ipl; ++q)
          if (c[q] >= 0) s += static_cast<double>(pr_xg(s_x, hot, a.l1hot, x_cur, c[q]));
#pragma unroll
        for (int q = 0; q < kPrB0Ipl; ++q) c[q] = nx[q];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kWarp, s, o);
      if (lane == 0) l1 += pr_finish_row(a, r_nxt, x_nxt, row, s, rprev, inv);
    } else {
      // exact-length bin, unit-interleaved columns: element j of the unit's
      // lane-l row sits at unit base + j * m + l (m = rows in the unit), so
      // every column load of the warp is one coalesced 4-sector request
      // instead of 32 scattered sectors.  The next four columns are loaded
      // while the current four gathers are in flight.
      const int64_t iu = u - B.unit0;
      const int64_t row = B.row0 + iu * 32 + lane;
      if (row < B.row1) {
        const V rprev = r_cur[row - a.row0];
        const V inv = a.inv[row];
        const int L = B.len;
        const int m = static_cast<int>(min(int64_t(32), B.row1 - B.row0 - iu * 32));
        const int32_t* cp = a.tcol + B.p0 + iu * 32 * L + lane;
        int c[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) c[q] = q < L ? ld_stream(cp + q * m) : -1;
        double s = 0.0;
        for (int j = 0; j < L; j += 4) {
          int nx[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) nx[q] = j + 4 + q < L ? ld_stream(cp + (j + 4 + q) * m) : -1;
          V t[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) t[q] = c[q] >= 0 ? pr_xg(s_x, hot, a.l1hot, x_cur, c[q]) : V(0);
          s += (static_cast<double>(t[0]) + static_cast<double>(t[1])) +
               (static_cast<double>(t[2]) + static_cast<double>(t[3]));
#pragma unroll
          for (int q = 0; q < 4; ++q) c[q] = nx[q];
        }
        l1 += pr_finish_row(a, r_nxt, x_nxt, row, s, rprev, inv);
      }
    }
  }
  __syncthreads();  // red may still be in use by a previous reduction
  return BlockReduce(red).Sum(l1);
}

template <typename V, int BS>
__global__ void __launch_bounds__(BS, BS == 1024 ? 2 : GBX_PR_MINB) k_pr_rows(PrArgs<V> a) {
  using BlockReduce = cub::BlockReduce<double, BS>;
  __shared__ typename BlockReduce::TempStorage red;
  __shared__ PrBin s_bins[kPrBinsMax];
  extern __shared__ __align__(16) unsigned char s_raw[];
  V* s_x = reinterpret_cast<V*>(s_raw);
  if (!a.fixed && *(volatile int*)&a.ctl[1]) return;  // converged (host-looped path)
  const int k = *(volatile int*)&a.ctl[0];
  if (a.ktime && threadIdx.x == 0) atomicMin(&a.ktime[(k % 128) * 2], pr_gtimer());
  const double blk = pr_rows_phase<V, BS>(a, k, red, s_bins, s_x);
  if (threadIdx.x == 0) {
    a.l1_rows[blockIdx.x] = blk;
    if (a.ktime) atomicMax(&a.ktime[(k % 128) * 2 + 1], pr_gtimer());
  }
}

// The whole iteration loop in ONE cooperative launch: per iteration the row
// phase, a grid barrier, the long-row finish (warp per long row), a grid
// barrier, then every CTA folds all L1 partials in the same fixed order and
// reaches the same convergence decision (pagerank.cpp:65-74).  Replaces the
// graph's two kernel nodes + conditional per iteration (~20 us of launch gaps
// per iteration against ~200 us of row work) with two grid barriers.
// BS = kPrThreads: several CTAs per SM, the hot prefix of x in L1 only.  BS =
// 1024: ONE CTA per SM (64 registers per thread) holding x[0, hot) in shared
// memory, restaged after every grid barrier -- the hot gathers leave the
// L1 -> L2 request path (one sector request per cycle per SM, the measured
// limiter of the L1 variant).
template <typename V, int BS>
__global__ void __launch_bounds__(BS, BS == 1024 ? 1 : GBX_PR_MINB) k_pr_persist(PrArgs<V> a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  using BlockReduce = cub::BlockReduce<double, BS>;
  __shared__ typename BlockReduce::TempStorage red;
  __shared__ PrBin s_bins[kPrBinsMax];
  __shared__ int s_stop;
  extern __shared__ __align__(16) unsigned char s_raw[];
  V* s_x = reinterpret_cast<V*>(s_raw);  // a.hot entries (0: unused)
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int k = 0;; ++k) {
    if (a.ktime && threadIdx.x == 0) atomicMin(&a.ktime[(k % 128) * 2], pr_gtimer());
    const double blk = pr_rows_phase<V, BS>(a, k, red, s_bins, s_x);
    if (threadIdx.x == 0) {
      a.l1_rows[blockIdx.x] = blk;
      if (a.ktime) atomicMax(&a.ktime[(k % 128) * 2 + 1], pr_gtimer());
    }
    grid.sync();
    // long rows: the chunk slots summed (lane-strided, fixed shuffle tree)
    const V *x_cur, *r_cur;
    V *x_nxt, *r_nxt;
    pr_buffers(a, k, x_cur, r_cur, x_nxt, r_nxt);
    double l1 = 0.0;
    for (int64_t i = gwarp; i < a.nlong; i += nwarps) {
      const int64_t q0 = a.long_slot[i], q1 = a.long_slot[i + 1];
      double s = 0.0;
      for (int64_t q = q0 + lane; q < q1; q += 32) s += __ldcg(a.slot + q);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kWarp, s, o);
      if (lane == 0) {
        const int64_t row = a.long_row[i];
        l1 += pr_finish_row(a, r_nxt, x_nxt, row, s, r_cur[row - a.row0], a.inv[row]);
      }
    }
    __syncthreads();
    const double blk2 = BlockReduce(red).Sum(l1);
    if (threadIdx.x == 0) a.l1_fin[blockIdx.x] = blk2;
    grid.sync();
    // every CTA: all partials in a fixed order -> the same total everywhere
    double part = 0.0;
    for (int b = threadIdx.x; b < static_cast<int>(gridDim.x); b += BS)
      part += __ldcg(&a.l1_rows[b]) + __ldcg(&a.l1_fin[b]);
    __syncthreads();
    const double tot = BlockReduce(red).Sum(part);
    if (threadIdx.x == 0) {
      const bool stop = !(tot >= a.tol) || (k + 1 >= a.itermax);
      s_stop = stop;
      if (blockIdx.x == 0) {
        a.l1_hist[k % 128] = tot;
        a.ctl[0] = k + 1;
        if (stop) a.ctl[1] = 1;
      }
    }
    __syncthreads();
    if (s_stop) break;
  }
}

// Sharded PageRank with the exchange fused into the iteration kernel (one
// cooperative launch per rank for the whole run).  Per iteration: the row
// phase and the long-row finish store x_next into EVERY rank's x (peer
// pointers, e.g. torch symmetric memory over NVLink/NVSwitch); the rank's fp64
// L1 total goes to slot [k&1][rank] of every rank's table; then a cross-rank
// barrier -- system-scope fence per CTA, grid barrier, one signal increment
// per peer, spin on the own signal word, grid barrier -- and every CTA sums
// the table in rank order: the same decision on every rank (pagerank.cpp:74).
// x and the slot table are double-buffered by iteration parity, so a rank one
// iteration ahead never overwrites what a slower rank still reads.
struct PrP2p {
  double* l1p[kPrMaxPeers];     // rank q's slot table [2][nranks]
  unsigned* sigp[kPrMaxPeers];  // rank q's signal word
  double* l1_own;               // this rank's table
  unsigned* sig_own;            // this rank's signal word
  int rank, nranks;
};

__global__ void __launch_bounds__(kPrThreads, GBX_PR_MINB) k_pr_persist_p2p(PrArgs<float> a,
                                                                            PrP2p m) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  using BlockReduce = cub::BlockReduce<double, kPrThreads>;
  __shared__ typename BlockReduce::TempStorage red;
  __shared__ PrBin s_bins[kPrBinsMax];
  __shared__ int s_stop;
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int k = 0;; ++k) {
    if (a.ktime && threadIdx.x == 0) atomicMin(&a.ktime[(k % 128) * 2], pr_gtimer());
    const double blk = pr_rows_phase<float, kPrThreads>(a, k, red, s_bins, nullptr);
    if (threadIdx.x == 0) {
      a.l1_rows[blockIdx.x] = blk;
      if (a.ktime) atomicMax(&a.ktime[(k % 128) * 2 + 1], pr_gtimer());
    }
    grid.sync();
    const float *x_cur, *r_cur;
    float *x_nxt, *r_nxt;
    pr_buffers(a, k, x_cur, r_cur, x_nxt, r_nxt);
    double l1 = 0.0;
    for (int64_t i = gwarp; i < a.nlong; i += nwarps) {
      const int64_t q0 = a.long_slot[i], q1 = a.long_slot[i + 1];
      double s = 0.0;
      for (int64_t q = q0 + lane; q < q1; q += 32) s += __ldcg(a.slot + q);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kWarp, s, o);
      if (lane == 0) {
        const int64_t row = a.long_row[i];
        l1 += pr_finish_row(a, r_nxt, x_nxt, row, s, r_cur[row - a.row0], a.inv[row]);
      }
    }
    __syncthreads();
    const double blk2 = BlockReduce(red).Sum(l1);
    if (threadIdx.x == 0) a.l1_fin[blockIdx.x] = blk2;
    __threadfence_system();  // this CTA's peer stores before the signal below
    grid.sync();
    if (blockIdx.x == 0) {
      double part = 0.0;
      for (int b = threadIdx.x; b < static_cast<int>(gridDim.x); b += kPrThreads)
        part += __ldcg(&a.l1_rows[b]) + __ldcg(&a.l1_fin[b]);
      __syncthreads();
      const double mine = BlockReduce(red).Sum(part);
      if (threadIdx.x == 0) {
        const int par = k & 1;
        for (int q = 0; q < m.nranks; ++q)
          m.l1p[q][par * m.nranks + m.rank] = mine;
        __threadfence_system();
        for (int q = 0; q < m.nranks; ++q) atomicAdd_system(m.sigp[q], 1u);
        // every rank signals every rank once per iteration
        // (the caller zeroes the signal words and barriers before the run)
        const unsigned want = static_cast<unsigned>(m.nranks) * (k + 1);
        for (;;) {
          unsigned v;
          asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(m.sig_own) : "memory");
          if (static_cast<int>(v - want) >= 0) break;
          __nanosleep(64);
        }
        __threadfence_system();
      }
    }
    grid.sync();
    if (threadIdx.x == 0) {
      const int par = k & 1;
      double tot = 0.0;
      for (int q = 0; q < m.nranks; ++q)  // rank order: identical on every rank
        tot += *(volatile double*)&m.l1_own[par * m.nranks + q];
      const bool stop = !(tot >= a.tol) || (k + 1 >= a.itermax);
      s_stop = stop;
      if (blockIdx.x == 0) {
        a.l1_hist[k % 128] = tot;
        a.ctl[0] = k + 1;
        if (stop) a.ctl[1] = 1;
      }
    }
    __syncthreads();
    if (s_stop) break;
  }
}

template <typename V, bool kGraph>
__global__ void __launch_bounds__(kPrThreads) k_pr_finish(PrArgs<V> a) {
  using BlockReduce = cub::BlockReduce<double, kPrThreads>;
  __shared__ typename BlockReduce::TempStorage red;
  __shared__ int s_last;
  if (!a.fixed && *(volatile int*)&a.ctl[1]) return;
  const int k = *(volatile int*)&a.ctl[0];
  const unsigned epoch = static_cast<unsigned>(k) + 1u;
  const V *x_cur, *r_cur;
  V *x_nxt, *r_nxt;
  pr_buffers(a, k, x_cur, r_cur, x_nxt, r_nxt);
  double l1 = 0.0;
  // one warp per long row: lane-strided slot sums, fixed shuffle tree
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; i < a.nlong; i += nw) {
    const int64_t q0 = a.long_slot[i], q1 = a.long_slot[i + 1];
    double s = 0.0;
    for (int64_t q = q0 + lane; q < q1; q += 32) s += a.slot[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kWarp, s, o);
    if (lane == 0) {
      const int64_t row = a.long_row[i];
      l1 += pr_finish_row(a, r_nxt, x_nxt, row, s, r_cur[row - a.row0], a.inv[row]);
    }
  }
  double blk = BlockReduce(red).Sum(l1);
  if (threadIdx.x == 0) {
    a.l1_fin[blockIdx.x] = blk;
    __threadfence();
    const unsigned prev = atomicAdd(a.fin_cnt, 1u);
    s_last = prev == epoch * gridDim.x - 1u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double part = 0.0;
  for (int b = threadIdx.x; b < a.grid_rows; b += kPrThreads) part += __ldcg(&a.l1_rows[b]);
  for (int b = threadIdx.x; b < static_cast<int>(gridDim.x); b += kPrThreads)
    part += __ldcg(&a.l1_fin[b]);
  __syncthreads();
  const double tot = BlockReduce(red).Sum(part);
  if (threadIdx.x == 0) {
    a.l1_hist[k % 128] = tot;
    a.ctl[0] = k + 1;
    const bool stop = a.fixed || !(tot >= a.tol) || (k + 1 >= a.itermax);
    if (stop) a.ctl[1] = 1;
    if constexpr (kGraph) cudaGraphSetConditional(a.cond, stop ? 0u : 1u);
  }
}

__global__ void k_pr_inv(float* inv, const int32_t* outdeg, int64_t n, double damping) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) inv[i] = outdeg[i] > 0 ? static_cast<float>(damping / static_cast<double>(outdeg[i])) : 0.f;
}

template <typename V>
__global__ void k_pr_init(V* r, V* x, V* inv, const int32_t* outdeg, int64_t n, double damping) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double r0 = 1.0 / static_cast<double>(n);
  r[i] = static_cast<V>(r0);
  const int dg = outdeg[i];
  // contrib = prior ./ (deg / damping) (pagerank.cpp:30-40, 55-56); the
  // iterations use the precomputed damping / deg (0: dangling, mass lost)
  x[i] = dg > 0 ? static_cast<V>(r0 / (static_cast<double>(dg) / damping)) : V(0);
  inv[i] = dg > 0 ? static_cast<V>(damping / static_cast<double>(dg)) : V(0);
}

// relabeled rank -> original ids (fp64 for the host copy)
template <typename V>
__global__ void k_pr_unpermute(const V* r, const int32_t* new2old, int64_t n, double* out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) out[new2old[i]] = static_cast<double>(r[i]);
}

// ---- plan -------------------------------------------------------------------------

__global__ void k_neg_len(const int64_t* rp, int64_t n, int32_t* key) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) key[i] = static_cast<int32_t>(rp[i + 1] - rp[i]);
}
__global__ void k_inverse_perm(const int32_t* new2old, int64_t n, int32_t* old2new) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) old2new[new2old[i]] = static_cast<int32_t>(i);
}
__global__ void k_relabel_pairs(const int32_t* rowid, const int32_t* col, const int32_t* old2new,
                                int64_t nnz, uint32_t* new_col, uint32_t* new_row) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p < nnz) {
    new_col[p] = static_cast<uint32_t>(old2new[col[p]]);
    new_row[p] = static_cast<uint32_t>(old2new[rowid[p]]);
  }
}
__global__ void k_gather_i32(const int32_t* src, const int32_t* idx, int64_t n, int32_t* dst) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

// exact-length bin [row0, row0 + nrows) of length L, row-major -> unit-
// interleaved (32-row units; element j of unit row l at unit*32*L + j*m + l)
__global__ void k_pr_interleave(const int32_t* src, int32_t* dst, int64_t nrows, int L) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p >= nrows * L) return;
  const int64_t i = p / L;
  const int j = static_cast<int>(p - i * L);
  const int64_t u = i >> 5;
  const int m = static_cast<int>(min(int64_t(32), nrows - u * 32));
  dst[u * 32 * L + int64_t(j) * m + (i & 31)] = src[p];
}

// first row r in [row0, row1) with length(r) <= thr[t] (lengths are
// non-increasing: binary search), and its row pointer
__global__ void k_pr_bounds(const int64_t* rp, int64_t row0, int64_t row1, const int64_t* thr,
                            int nt, int64_t* out_row, int64_t* out_p) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  int64_t lo = row0, hi = row1;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (rp[mid + 1] - rp[mid] <= thr[t]) hi = mid; else lo = mid + 1;
  }
  out_row[t] = lo;
  out_p[t] = rp[lo];
}

// work units over relabeled rows [row0, row1) (lengths non-increasing): long
// rows become chunk units; rows up to kPrLong are binned by G = lanes per row
// (G*kPrIpl >= length); rows up to kPrShort get one bin per distinct length so
// the kernel computes their nonzero offsets instead of loading row_ptr.  The
// bin boundaries come from device binary searches (no O(n) host pass).
static void build_units(PrPlan& P, int64_t row0, int64_t row1, cudaStream_t s) {
  // thresholds: kPrLong, then kPrShort, kPrShort-1, ..., 0
  std::vector<int64_t> thr = {kPrLong};
  for (int64_t L = kPrShort; L >= 0; --L) thr.push_back(L);
  const int nt = static_cast<int>(thr.size());
  std::vector<int64_t> brow(nt), bp(nt);
  {
    DevArray<int64_t> dthr(nt), drow(nt), dp(nt);
    GBX_CUDA(cudaMemcpyAsync(dthr.p, thr.data(), nt * 8, cudaMemcpyHostToDevice, s));
    k_pr_bounds<<<1, 64, 0, s>>>(P.trp.p, row0, row1, dthr.p, nt, drow.p, dp.p);
    GBX_LAUNCHED();
    GBX_CUDA(cudaMemcpyAsync(brow.data(), drow.p, nt * 8, cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaMemcpyAsync(bp.data(), dp.p, nt * 8, cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaStreamSynchronize(s));
  }
  // long rows [row0, brow[0]): their row pointers, cut into chunks
  const int64_t rlong = brow[0];
  std::vector<int64_t> lrp(rlong - row0 + 1);
  if (rlong > row0) {
    GBX_CUDA(cudaMemcpyAsync(lrp.data(), P.trp.p + row0, lrp.size() * 8, cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaStreamSynchronize(s));
  }
  std::vector<int64_t> chunks, lslot;
  std::vector<int32_t> lrow;
  for (int64_t r = row0; r < rlong; ++r) {
    const int64_t b = lrp[r - row0], e = lrp[r - row0 + 1];
    lrow.push_back(static_cast<int32_t>(r));
    lslot.push_back(static_cast<int64_t>(chunks.size() / 2));
    for (int64_t p = b; p < e; p += kPrChunk) {
      chunks.push_back(p);
      chunks.push_back(std::min(e, p + kPrChunk));
    }
  }
  lslot.push_back(static_cast<int64_t>(chunks.size() / 2));
  std::vector<PrBin> bins;
  int64_t units = 0;
  {
    // bin 0: kPrShort < len <= kPrLong, one warp (unit) per row
    PrBin b{};
    b.unit0 = units;
    b.row0 = rlong;
    b.row1 = brow[1];
    b.p0 = bp[0];
    b.len = -1;
    bins.push_back(b);
    units += b.row1 - b.row0;
  }
  // bins 1..: one per exact length (non-increasing), 32 rows per unit
  for (int t = 1; t < nt; ++t) {
    const int64_t len = thr[t];
    const int64_t r0 = brow[t], r1 = t + 1 < nt ? brow[t + 1] : row1;
    if (r1 <= r0) continue;
    PrBin b{};
    b.unit0 = units;
    b.row0 = r0;
    b.row1 = r1;
    b.p0 = bp[t];
    b.len = static_cast<int32_t>(len);
    bins.push_back(b);
    units += (r1 - r0 + 31) / 32;
  }
  if (bins.size() > static_cast<size_t>(kPrBinsMax)) fail(GBX_CUDA_ERROR, "pagerank: too many bins");
  // exact-length bins: columns to the unit-interleaved layout k_pr_rows reads
  {
    int64_t q0 = -1, q1 = -1;
    for (const PrBin& b : bins)
      if (b.len > 0) {
        if (q0 < 0) q0 = b.p0;
        q1 = b.p0 + (b.row1 - b.row0) * b.len;
      }
    if (q0 >= 0 && q1 > q0) {
      Tmp<int32_t> cp(q1 - q0, s);
      GBX_CUDA(cudaMemcpyAsync(cp.p, P.tcol.p + q0, (q1 - q0) * 4, cudaMemcpyDeviceToDevice, s));
      for (const PrBin& b : bins) {
        const int64_t cnt = (b.row1 - b.row0) * b.len;
        if (b.len <= 0 || cnt == 0) continue;
        k_pr_interleave<<<ceil_div(cnt, 256), 256, 0, s>>>(cp.p + (b.p0 - q0), P.tcol.p + b.p0,
                                                           b.row1 - b.row0, b.len);
        GBX_LAUNCHED();
      }
    }
  }
  P.nbins = static_cast<int>(bins.size());
  P.bins.alloc(std::max<size_t>(bins.size(), 1));
  if (!bins.empty())
    GBX_CUDA(cudaMemcpyAsync(P.bins.p, bins.data(), bins.size() * sizeof(PrBin),
                             cudaMemcpyHostToDevice, s));
  P.nunits = units;
  P.nchunks = static_cast<int64_t>(chunks.size() / 2);
  P.nlong = static_cast<int64_t>(lrow.size());
  P.chunk_p.alloc(std::max<int64_t>(2 * P.nchunks, 2));
  P.long_row.alloc(std::max<int64_t>(P.nlong, 1));
  P.long_slot.alloc(P.nlong + 1);
  P.slot.alloc(std::max<int64_t>(P.nchunks, 1));
  if (P.nchunks)
    GBX_CUDA(cudaMemcpyAsync(P.chunk_p.p, chunks.data(), chunks.size() * 8, cudaMemcpyHostToDevice, s));
  if (P.nlong)
    GBX_CUDA(cudaMemcpyAsync(P.long_row.p, lrow.data(), lrow.size() * 4, cudaMemcpyHostToDevice, s));
  GBX_CUDA(cudaMemcpyAsync(P.long_slot.p, lslot.data(), lslot.size() * 8, cudaMemcpyHostToDevice, s));
  GBX_CUDA(cudaStreamSynchronize(s));
}

// row-permutation relabel: new row r = AT row new2old[r] with every column
// mapped through old2new (no sort: the rows move as whole segments)
__global__ void k_pr_newlen(const int64_t* atrp, const int32_t* new2old, int64_t n, int64_t* len) {
  const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (r < n) {
    const int32_t o = new2old[r];
    len[r] = atrp[o + 1] - atrp[o];
  } else if (r == n) {
    len[r] = 0;
  }
}
constexpr int64_t kPrGatherLong = 256;
// rows longer than kPrGatherLong (a prefix: rows are in descending length): a CTA each
__global__ void k_pr_gather_long(const int64_t* atrp, const int32_t* atcol, const int32_t* new2old,
                                 const int32_t* old2new, const int64_t* trp, int64_t n,
                                 int32_t* tcol) {
  for (int64_t r = blockIdx.x; r < n; r += gridDim.x) {
    const int64_t d = trp[r], len = trp[r + 1] - d;
    if (len <= kPrGatherLong) return;
    const int64_t src = atrp[new2old[r]];
    for (int64_t p = threadIdx.x; p < len; p += blockDim.x) tcol[d + p] = old2new[atcol[src + p]];
  }
}
// the rest: 8 lanes per row
__global__ void k_pr_gather_short(const int64_t* atrp, const int32_t* atcol,
                                  const int32_t* new2old, const int32_t* old2new,
                                  const int64_t* trp, int64_t n, int32_t* tcol) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = gw * 4 + (lane >> 3); r < n; r += nw * 4) {
    const int64_t d = trp[r], len = trp[r + 1] - d;
    if (len > kPrGatherLong) continue;
    const int64_t src = atrp[new2old[r]];
    for (int64_t p = lane & 7; p < len; p += 8) tcol[d + p] = old2new[atcol[src + p]];
  }
}

// rows of A in the new order, as (new column, new row) pairs: the pairs come
// out ordered by new row, so ONE stable sort by new column yields the
// relabeled AT with every row's columns ascending in the new ids
// (A's rows are not in length order here: the long ones are listed first)
__global__ void k_pr_list_long(const int64_t* prp, int64_t n, int32_t* list, int* cnt) {
  const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (r < n && prp[r + 1] - prp[r] > kPrGatherLong) list[agg_append(cnt)] = static_cast<int32_t>(r);
}
// long rows cut into kPrGatherChunk-element items (one hub row per CTA left
// a single CTA looping over 10^5 elements at the end of the launch)
constexpr int64_t kPrGatherChunk = 2048;
__global__ void k_pr_long_chunks(const int64_t* prp, const int32_t* list, int m, int64_t* nch) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) {
    const int64_t r = list[i];
    nch[i] = (prp[r + 1] - prp[r] + kPrGatherChunk - 1) / kPrGatherChunk;
  }
}
__global__ void k_pr_gather_a_long(const int64_t* arp, const int32_t* acol, const int32_t* new2old,
                                   const int32_t* old2new, const int64_t* prp,
                                   const int32_t* list, const int64_t* cincl, int m,
                                   uint32_t* key, uint32_t* val) {
  const int64_t total = cincl[m - 1];
  for (int64_t c = blockIdx.x; c < total; c += gridDim.x) {
    int lo = 0, hi = m - 1;  // first i with cincl[i] > c
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (cincl[mid] > c) hi = mid; else lo = mid + 1;
    }
    const int64_t r = list[lo];
    const int64_t k = c - (lo ? cincl[lo - 1] : 0);
    const int64_t d = prp[r], len = prp[r + 1] - d;
    const int64_t src = arp[new2old[r]];
    const int64_t p1 = min(len, (k + 1) * kPrGatherChunk);
    for (int64_t p = k * kPrGatherChunk + threadIdx.x; p < p1; p += blockDim.x) {
      key[d + p] = static_cast<uint32_t>(old2new[acol[src + p]]);
      val[d + p] = static_cast<uint32_t>(r);
    }
  }
}
__global__ void k_pr_gather_a_short(const int64_t* arp, const int32_t* acol,
                                    const int32_t* new2old, const int32_t* old2new,
                                    const int64_t* prp, int64_t n, uint32_t* key, uint32_t* val) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = gw * 4 + (lane >> 3); r < n; r += nw * 4) {
    const int64_t d = prp[r], len = prp[r + 1] - d;
    if (len > kPrGatherLong) continue;
    const int64_t src = arp[new2old[r]];
    for (int64_t p = lane & 7; p < len; p += 8) {
      key[d + p] = static_cast<uint32_t>(old2new[acol[src + p]]);
      val[d + p] = static_cast<uint32_t>(r);
    }
  }
}

// relabel mode: 0 = two stable radix sorts (rows and columns in new-id order),
// 1 = row permutation (columns in the original ascending order, mapped),
// 2 = row permutation + segmented sort of every row (new-id order),
// 3 (default) = A's rows permuted into the new order + ONE stable radix sort
// by new column (new-id order; scale 22: 4.4 -> ~2.4 ms, same SpMV time)
static int relabel_mode() {
  static const int m = [] {
    const char* e = std::getenv("GBX_PR_RELABEL");
    if (!e) return 3;
    if (!std::strcmp(e, "gather")) return 1;
    if (!std::strcmp(e, "gather_seg")) return 2;
    if (!std::strcmp(e, "sort2")) return 0;
    return 3;
  }();
  return m;
}

// relabeled AT (rows by descending in-degree) + relabeled out-degree
static void build_relabeled(gbx_graph* g, PrPlan& P) {
  const Csr& AT = g->AT();
  cudaStream_t s = g->stream;
  const int64_t n = AT.n, nnz = AT.nnz;
  P.n = n;
  P.nnz = nnz;
  DevArray<int32_t> len(std::max<int64_t>(n, 1));
  if (n) {
    k_neg_len<<<ceil_div(n, 256), 256, 0, s>>>(AT.rp.p, n, len.p);
    GBX_LAUNCHED();
  }
  sort_ids_by_key(s, len.p, n, false, P.new2old);
  P.old2new.alloc(std::max<int64_t>(n, 1));
  P.deg.alloc(std::max<int64_t>(n, 1));
  if (n) {
    k_inverse_perm<<<ceil_div(n, 256), 256, 0, s>>>(P.new2old.p, n, P.old2new.p);
    k_gather_i32<<<ceil_div(n, 256), 256, 0, s>>>(g->rowdeg.p, P.new2old.p, n, P.deg.p);
    GBX_LAUNCHED();
  }
  // relabeled AT, every row's columns ascending in the new ids (the thread-
  // per-row bins then read the hub end of x together at each step): two
  // stable 32-bit radix sorts -- by new column carrying the new row, then by
  // new row carrying the column -- instead of one sort of 64-bit (row, col)
  // keys (2*bits digits): 5.1 -> ~1.5 ms at scale 22
  const int bits = bits_for(std::max<int64_t>(n, 2));
  P.trp.alloc(n + 1);
  P.tcol.alloc(std::max<int64_t>(nnz, 1));
  if (nnz && relabel_mode() == 3) {
    const Csr& A = g->A;
    DevArray<int64_t> prp(n + 1);
    k_pr_newlen<<<ceil_div(n + 1, 256), 256, 0, s>>>(A.rp.p, P.new2old.p, n, prp.p);
    GBX_LAUNCHED();
    {
      size_t tb = 0;
      GBX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, prp.p, prp.p, n + 1, s));
      Tmp<uint8_t> t(tb, s);
      GBX_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tb, prp.p, prp.p, n + 1, s));
    }
    Tmp<uint32_t> kc(nnz, s), kc2(nnz, s), vr(nnz, s);
    {
      Tmp<int32_t> list(n, s);
      Tmp<int> cnt(1, s);
      GBX_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int), s));
      k_pr_list_long<<<ceil_div(n, 256), 256, 0, s>>>(prp.p, n, list.p, cnt.p);
      GBX_LAUNCHED();
      int m = 0;
      GBX_CUDA(cudaMemcpyAsync(&m, cnt.p, sizeof(int), cudaMemcpyDeviceToHost, s));
      GBX_CUDA(cudaStreamSynchronize(s));
      if (m > 0) {
        Tmp<int64_t> nch(m, s);
        k_pr_long_chunks<<<ceil_div(m, 256), 256, 0, s>>>(prp.p, list.p, m, nch.p);
        size_t tb2 = 0;
        GBX_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb2, nch.p, nch.p, m, s));
        {
          Tmp<uint8_t> t(tb2, s);
          GBX_CUDA(cub::DeviceScan::InclusiveSum(t.p, tb2, nch.p, nch.p, m, s));
        }
        k_pr_gather_a_long<<<device_sms() * 8, 256, 0, s>>>(A.rp.p, A.col.p, P.new2old.p,
                                                             P.old2new.p, prp.p, list.p, nch.p, m,
                                                             kc.p, vr.p);
      }
    }
    k_pr_gather_a_short<<<device_sms() * 8, 256, 0, s>>>(A.rp.p, A.col.p, P.new2old.p,
                                                          P.old2new.p, prp.p, n, kc.p, vr.p);
    GBX_LAUNCHED();
    size_t tb = 0;
    GBX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kc.p, kc2.p, vr.p,
                                             reinterpret_cast<uint32_t*>(P.tcol.p), nnz, 0, bits,
                                             s));
    {
      Tmp<uint8_t> t(tb, s);
      GBX_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tb, kc.p, kc2.p, vr.p,
                                               reinterpret_cast<uint32_t*>(P.tcol.p), nnz, 0,
                                               bits, s));
    }
    rowptr_from_sorted_rows32(s, n, kc2.p, nnz, P.trp.p);
  } else if (nnz && relabel_mode() > 0) {
    k_pr_newlen<<<ceil_div(n + 1, 256), 256, 0, s>>>(AT.rp.p, P.new2old.p, n, P.trp.p);
    GBX_LAUNCHED();
    {
      size_t tb = 0;
      GBX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, P.trp.p, P.trp.p, n + 1, s));
      Tmp<uint8_t> t(tb, s);
      GBX_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tb, P.trp.p, P.trp.p, n + 1, s));
    }
    const int grid = device_sms() * 8;
    k_pr_gather_long<<<device_sms() * 4, 256, 0, s>>>(AT.rp.p, AT.col.p, P.new2old.p, P.old2new.p,
                                                       P.trp.p, n, P.tcol.p);
    k_pr_gather_short<<<grid, 256, 0, s>>>(AT.rp.p, AT.col.p, P.new2old.p, P.old2new.p, P.trp.p, n,
                                           P.tcol.p);
    GBX_LAUNCHED();
    if (relabel_mode() == 2) {
      Tmp<int32_t> out(nnz, s);
      size_t tb = 0;
      GBX_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, tb, P.tcol.p, out.p, nnz, n, P.trp.p,
                                                  P.trp.p + 1, s));
      Tmp<uint8_t> t(tb, s);
      GBX_CUDA(cub::DeviceSegmentedSort::SortKeys(t.p, tb, P.tcol.p, out.p, nnz, n, P.trp.p,
                                                  P.trp.p + 1, s));
      GBX_CUDA(cudaMemcpyAsync(P.tcol.p, out.p, nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    }
  } else if (nnz) {
    Tmp<uint32_t> kc(nnz, s), kc2(nnz, s), vr(nnz, s), vr2(nnz, s);
    {
      Tmp<int32_t> rowid(nnz, s);
      expand_rows_into(s, AT, rowid.p);
      k_relabel_pairs<<<ceil_div(nnz, 256), 256, 0, s>>>(rowid.p, AT.col.p, P.old2new.p, nnz,
                                                         kc.p, vr.p);
      GBX_LAUNCHED();
    }
    size_t tb = 0;
    GBX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kc.p, kc2.p, vr.p, vr2.p, nnz, 0, bits, s));
    {
      Tmp<uint8_t> t(tb, s);
      GBX_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tb, kc.p, kc2.p, vr.p, vr2.p, nnz, 0, bits, s));
      // by new row (stable): (row, col) order; the columns land in tcol
      GBX_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tb, vr2.p, vr.p, kc2.p,
                                               reinterpret_cast<uint32_t*>(P.tcol.p), nnz, 0, bits,
                                               s));
    }
    rowptr_from_sorted_rows32(s, n, vr.p, nnz, P.trp.p);
  } else {
    GBX_CUDA(cudaMemsetAsync(P.trp.p, 0, (n + 1) * sizeof(int64_t), s));
  }
  GBX_CUDA(cudaStreamSynchronize(s));
}

static void plan_rows(gbx_graph* g, PrPlan& P, int64_t row0, int64_t row1) {
  cudaStream_t s = g->stream;
  P.row0 = row0;
  P.row1 = row1;
  build_units(P, row0, row1, s);
  P.grid = 0;  // set per precision by rows_grid() (depends on the shared-memory footprint)
  P.grid_fin = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(
      (P.nlong * 32 + kPrThreads - 1) / kPrThreads, 4 * device_sms())));
  P.l1_block.alloc(static_cast<size_t>(device_sms()) * 32);
  P.l1_fin.alloc(std::max<int64_t>(P.grid_fin, static_cast<int64_t>(device_sms()) * 32));
  P.l1_hist.alloc(128);
  P.ktime.alloc(256);
  P.ctl.alloc(2);
  P.blk_cnt.alloc(1);
}

void pagerank_prepare(gbx_graph* g) {
  require_at(g, "pagerank_gap");
  require_rowdeg(g, "pagerank_gap");
  if (g->pr) return;
  static const bool timing = std::getenv("GBX_PLAN_TIMING") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!timing) return;
    GBX_CUDA(cudaStreamSynchronize(g->stream));
    auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "pagerank_prepare %s %.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  auto P = std::make_unique<PrPlan>();
  build_relabeled(g, *P);
  mark("relabel");
  plan_rows(g, *P, 0, P->n);
  mark("plan_rows");
  for (int b = 0; b < 2; ++b) {
    P->r[b].alloc(std::max<int64_t>(g->A.n, 1));
    P->x[b].alloc(std::max<int64_t>(g->A.n, 1));
  }
  P->out.alloc(std::max<int64_t>(g->A.n, 1));
  mark("vectors");
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
template <typename V> V* buf_inv(PrPlan& P);
template <> float* buf_inv<float>(PrPlan& P) {
  if (!P.invf.p) P.invf.alloc(P.r[0].n);
  return P.invf.p;
}
template <> double* buf_inv<double>(PrPlan& P) {
  if (!P.invd.p) P.invd.alloc(P.r[0].n);
  return P.invd.p;
}

static int64_t hot_bytes() {
  static const int64_t hb = [] {
    const char* e = std::getenv("GBX_PR_HOT_KB");
    return static_cast<int64_t>(e ? std::atoi(e) : kPrHotKbDefault) * 1024;
  }();
  return hb;
}

// bytes of x kept L1-resident (override: GBX_PR_L1_KB)
static int64_t l1_hot_bytes() {
  static const int64_t hb = [] {
    const char* e = std::getenv("GBX_PR_L1_KB");
    return static_cast<int64_t>(e ? std::atoi(e) : 144) * 1024;  // measured at the 32 KB carveout: 64 / 96 / 112 / 128 / 144 / 160 / 176 / 192 KB -> 221.6 / 216.1 / 209.9 / 209.0 / 205.9 / 207.0 / 208.4 / 209.7 us/iter
  }();
  return hb;
}

#ifndef GBX_PR_PERSIST_CARVEOUT
#define GBX_PR_PERSIST_CARVEOUT 10  // 32 KB of shared memory, 224 KB of L1: 214.0 -> 207.1 us/iter (A/B)
#endif
static int persist_carveout() {
  static const int c = [] {
    const char* cv = std::getenv("GBX_PR_CARVEOUT");
    return cv ? std::atoi(cv) : GBX_PR_PERSIST_CARVEOUT;
  }();
  return c;
}

template <typename V>
static size_t rows_smem(const PrArgs<V>& a) {
  static bool attr = false;
  if (!attr) {
    const int mx = static_cast<int>(std::min<int64_t>(hot_bytes(), 200 * 1024));
    GBX_CUDA(cudaFuncSetAttribute(k_pr_rows<float, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  std::max(mx, 1)));
    GBX_CUDA(cudaFuncSetAttribute(k_pr_rows<double, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  std::max(mx, 1)));
    // (measured: the default carveout is best; GBX_PR_CARVEOUT overrides)
    if (const char* cv = std::getenv("GBX_PR_CARVEOUT")) {
      const int carve = std::atoi(cv);
      GBX_CUDA(cudaFuncSetAttribute(k_pr_rows<float, 1024>,
                                    cudaFuncAttributePreferredSharedMemoryCarveout, carve));
      GBX_CUDA(cudaFuncSetAttribute(k_pr_rows<double, 1024>,
                                    cudaFuncAttributePreferredSharedMemoryCarveout, carve));
      GBX_CUDA(cudaFuncSetAttribute(k_pr_rows<float, kPrThreads>,
                                    cudaFuncAttributePreferredSharedMemoryCarveout, carve));
      GBX_CUDA(cudaFuncSetAttribute(k_pr_rows<double, kPrThreads>,
                                    cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    }
    // the 256-thread row kernels (host-looped path) share the persistent
    // kernel's carveout
    if (const int carve = persist_carveout(); carve >= 0) {
      GBX_CUDA(cudaFuncSetAttribute(k_pr_rows<float, kPrThreads>,
                                    cudaFuncAttributePreferredSharedMemoryCarveout, carve));
      GBX_CUDA(cudaFuncSetAttribute(k_pr_rows<double, kPrThreads>,
                                    cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    }
    attr = true;
  }
  return static_cast<size_t>(a.hot) * sizeof(V);
}

template <typename V>
static int rows_block(const PrArgs<V>& a) {
  return a.hot > 0 ? 1024 : kPrThreads;
}
template <typename V>
static void* rows_fn(const PrArgs<V>& a) {
  return a.hot > 0 ? reinterpret_cast<void*>(k_pr_rows<V, 1024>)
                   : reinterpret_cast<void*>(k_pr_rows<V, kPrThreads>);
}

// persistent grid: SMs x resident CTAs for this shared-memory footprint
template <typename V>
static int rows_grid(const PrArgs<V>& a) {
  int per_sm = 0;
  GBX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rows_fn<V>(a), rows_block<V>(a),
                                                         rows_smem<V>(a)));
  return device_sms() * std::max(per_sm, 1);
}

template <typename V>
static void launch_rows(const PrArgs<V>& a, cudaStream_t s) {
  if (a.hot > 0)
    k_pr_rows<V, 1024><<<a.grid_rows, 1024, rows_smem<V>(a), s>>>(a);
  else
    k_pr_rows<V, kPrThreads><<<a.grid_rows, kPrThreads, 0, s>>>(a);
}

template <typename V>
static PrArgs<V> make_args(PrPlan& P, double damping, double tol, int itermax) {
  PrArgs<V> a{};
  a.trp = P.trp.p;
  a.tcol = P.tcol.p;
  a.outdeg = P.deg.p;
  if (P.r[0].p) a.inv = buf_inv<V>(P);
  a.bins = P.bins.p;
  a.nbins = P.nbins;
  a.nunits = P.nunits;
  a.chunk_p = P.chunk_p.p;
  a.nchunks = P.nchunks;
  a.long_row = P.long_row.p;
  a.long_slot = P.long_slot.p;
  a.nlong = P.nlong;
  a.slot = P.slot.p;
  if (P.r[0].p) {
    a.r0 = buf_r<V>(P, 0);
    a.r1 = buf_r<V>(P, 1);
    a.x0 = buf_x<V>(P, 0);
    a.x1 = buf_x<V>(P, 1);
  }
  a.l1_rows = P.l1_block.p;
  a.l1_fin = P.l1_fin.p;
  a.l1_hist = P.l1_hist.p;
  a.ctl = P.ctl.p;
  a.ktime = P.ktime.p;
  a.fin_cnt = P.blk_cnt.p;
  a.row0 = 0;
  a.hot = std::min<int64_t>(P.n, hot_bytes() / static_cast<int64_t>(sizeof(V))) & ~int64_t(3);
  // with a shared-memory prefix, the L1 evict_last window follows it
  // (GBX_PR_L1X_KB bytes of x past the prefix)
  static const int64_t l1x = [] {
    const char* e = std::getenv("GBX_PR_L1X_KB");
    return static_cast<int64_t>(e ? std::atoi(e) : 48) * 1024;
  }();
  a.l1hot = a.hot > 0 ? std::min<int64_t>(P.n, a.hot + l1x / static_cast<int64_t>(sizeof(V)))
                      : std::min<int64_t>(P.n, l1_hot_bytes() / static_cast<int64_t>(sizeof(V)));
  a.grid_rows = rows_grid<V>(a);
  a.damping = damping;
  a.teleport = (1.0 - damping) / static_cast<double>(P.n);
  a.tol = tol;
  a.itermax = itermax;
  a.fixed = 0;
  return a;
}

__global__ void k_pr_ktime_reset(unsigned long long* t) {
  const int i = threadIdx.x;
  if (i < 256) t[i] = (i & 1) ? 0ull : ~0ull;
}

static void reset_state(cudaStream_t s, PrPlan& P) {
  GBX_CUDA(cudaMemsetAsync(P.ctl.p, 0, 2 * sizeof(int), s));
  GBX_CUDA(cudaMemsetAsync(P.blk_cnt.p, 0, sizeof(unsigned), s));
  if (P.ktime.p) k_pr_ktime_reset<<<1, 256, 0, s>>>(P.ktime.p);
}

template <typename V>
static bool build_graph(PrPlan& P, double damping, double tol, int itermax) {
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
  PrArgs<V> a = make_args<V>(P, damping, tol, itermax);
  a.cond = cond;
  void* params[] = {&a};
  cudaGraphNode_t kn_rows = nullptr, kn_fin = nullptr;
  if (ok) {
    cudaKernelNodeParams kp = {};
    kp.func = rows_fn<V>(a);
    kp.gridDim = dim3(a.grid_rows);
    kp.blockDim = dim3(rows_block<V>(a));
    kp.sharedMemBytes = static_cast<unsigned>(rows_smem<V>(a));
    kp.kernelParams = params;
    ok = cudaGraphAddKernelNode(&kn_rows, body, nullptr, 0, &kp) == cudaSuccess;
  }
  if (ok) {
    cudaKernelNodeParams kp = {};
    kp.func = reinterpret_cast<void*>(k_pr_finish<V, true>);
    kp.gridDim = dim3(P.grid_fin);
    kp.blockDim = dim3(kPrThreads);
    kp.kernelParams = params;
    ok = cudaGraphAddKernelNode(&kn_fin, body, &kn_rows, 1, &kp) == cudaSuccess;
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

// the persistent variant needs every CTA resident (cooperative launch): one
// CTA per SM with the shared-memory hot prefix (a.hot > 0), else as many
// kPrThreads CTAs as fit
template <typename V>
static void* persist_fn(const PrArgs<V>& a) {
  return a.hot > 0 ? reinterpret_cast<void*>(k_pr_persist<V, 1024>)
                   : reinterpret_cast<void*>(k_pr_persist<V, kPrThreads>);
}

template <typename V>
static bool persist_args(PrPlan& P, double damping, double tol, int itermax, PrArgs<V>& a,
                         int& block, size_t& smem) {
  a = make_args<V>(P, damping, tol, itermax);
  block = a.hot > 0 ? 1024 : kPrThreads;
  smem = static_cast<size_t>(a.hot) * sizeof(V);
  if (a.hot > 0) {
    if (smem > 200 * 1024) return false;
    if (cudaFuncSetAttribute(persist_fn<V>(a), cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem)) != cudaSuccess) {
      (void)cudaGetLastError();
      return false;
    }
  }
  // shared-memory carveout of the persistent kernel (percent of the maximum;
  // GBX_PR_CARVEOUT overrides, < 0 leaves the driver's choice)
  if (const int carve = persist_carveout(); carve >= 0)
    (void)cudaFuncSetAttribute(persist_fn<V>(a), cudaFuncAttributePreferredSharedMemoryCarveout,
                               carve);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, persist_fn<V>(a), block, smem) !=
          cudaSuccess || per_sm < 1) {
    (void)cudaGetLastError();
    return false;
  }
  a.grid_rows = device_sms() * per_sm;
  return static_cast<int64_t>(P.l1_fin.n) >= a.grid_rows &&
         static_cast<int64_t>(P.l1_block.n) >= a.grid_rows;
}

template <typename V>
static int pagerank_loop(gbx_graph* g, PrPlan& P, double damping, double tol, int itermax,
                         double* rank, int* iters) {
  const int64_t n = g->A.n;
  cudaStream_t s = g->stream;
  reset_state(s, P);
  P.last_persist = false;
  k_pr_init<V><<<ceil_div(n, 256), 256, 0, s>>>(buf_r<V>(P, 0), buf_x<V>(P, 0), buf_inv<V>(P),
                                                P.deg.p, n, damping);
  GBX_LAUNCHED();
  // GBX_PR_NO_GRAPH=1 forces the host-looped path (ncu cannot profile kernel
  // nodes of a graph that holds conditional nodes)
  static const bool no_graph = std::getenv("GBX_PR_NO_GRAPH") != nullptr;
  static const bool use_graph = std::getenv("GBX_PR_GRAPH") != nullptr;
  PrArgs<V> pa{};
  int pblock = 0;
  size_t psmem = 0;
  if (!no_graph && !use_graph && persist_args<V>(P, damping, tol, itermax, pa, pblock, psmem)) {
    void* args[] = {&pa};
    GBX_CUDA(cudaLaunchCooperativeKernel(persist_fn<V>(pa), dim3(pa.grid_rows), dim3(pblock), args,
                                         psmem, s));
    P.last_persist = true;
  } else if (!no_graph && build_graph<V>(P, damping, tol, itermax)) {
    GBX_CUDA(cudaGraphLaunch(P.exec, s));
  } else {
    PrArgs<V> a = make_args<V>(P, damping, tol, itermax);
    int done = 0, launched = 0;
    while (!done && launched < itermax) {
      const int chunk = std::min(4, itermax - launched);
      for (int c = 0; c < chunk; ++c) {
        launch_rows<V>(a, s);
        k_pr_finish<V, false><<<P.grid_fin, kPrThreads, 0, s>>>(a);
        GBX_LAUNCHED();
      }
      launched += chunk;
      GBX_CUDA(cudaMemcpyAsync(&done, P.ctl.p + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
      GBX_CUDA(cudaStreamSynchronize(s));
    }
  }
  int it = 0;
  unsigned long long kt[256];
  GBX_CUDA(cudaMemcpyAsync(&it, P.ctl.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaMemcpyAsync(kt, P.ktime.p, sizeof kt, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  P.last_iters = it;
  {
    // mean k_pr_rows launch duration over this run's iterations (first CTA
    // start to last CTA end, %globaltimer)
    double sum = 0.0;
    int cnt = 0;
    for (int k = 0; k < std::min(it, 128); ++k)
      if (kt[2 * k + 1] > kt[2 * k] && kt[2 * k] != ~0ull) {
        sum += static_cast<double>(kt[2 * k + 1] - kt[2 * k]);
        ++cnt;
      }
    P.last_rows_ms = cnt ? sum / cnt * 1e-6 : 0.0;
  }
  if (iters) *iters = it;
  // ranks back in original vertex order (device-resident result; fp64)
  k_pr_unpermute<V><<<ceil_div(n, 256), 256, 0, s>>>(buf_r<V>(P, it & 1), P.new2old.p, n,
                                                       P.out.p);
  GBX_LAUNCHED();
  if (rank) {
    GBX_CUDA(cudaMemcpyAsync(rank, P.out.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaStreamSynchronize(s));
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
  g->pending_iters = nullptr;
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
  const int it = f64 ? pagerank_loop<double>(g, P, damping, tol, itermax, rank, iters)
                     : pagerank_loop<float>(g, P, damping, tol, itermax, rank, iters);
  const double vb = f64 ? 8.0 : 4.0;
  g->stats.launches = P.last_persist ? 4 : 3 + 2 * it;  // (+ the ktime reset)
  g->stats.hot_launches = it;
  g->stats.iterations = it;
  g->stats.hot_ms = P.last_rows_ms;
  g->stats.work_units = P.nnz;
  // col (4) + gathered x (vb) per edge; row_ptr (8) + r_prev, r, x (vb each) + deg (4)
  g->stats.hot_bytes_per_launch = (4.0 + vb) * static_cast<double>(P.nnz) +
                                  8.0 * static_cast<double>(n + 1) + (3.0 * vb + 4.0) * n;
}

// ---- sharded step (multi-GPU driver) ----------------------------------------------
// Shards own contiguous blocks of the RELABELED rows, balanced by rows + nnz
// (merge-path split).  The exchange layout is padded: rank q's rows keep their
// contributions at x_full[q * chunk + (row - bounds[q])] (chunk = the longest
// block), so the driver's one equal-size all-gather (NCCL
// all_gather_into_tensor) lands every slice in place with no unpacking copies;
// the shard's column indices are remapped to that layout once, at prepare.

__device__ __forceinline__ int64_t pr_pad_index(const int64_t* bounds, int nranks, int64_t chunk,
                                                int64_t i) {
  int q = 0;
  while (q + 1 < nranks && i >= bounds[q + 1]) ++q;
  return static_cast<int64_t>(q) * chunk + (i - bounds[q]);
}

__global__ void k_pr_pad_cols(int32_t* col, int64_t nnz, const int64_t* bounds, int nranks,
                              int64_t chunk) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p < nnz) col[p] = static_cast<int32_t>(pr_pad_index(bounds, nranks, chunk, col[p]));
}

void pr_shard_prepare(gbx_graph* g, int rank, int nranks, int64_t* rb_out, int64_t* re_out) {
  require_at(g, "pr_shard");
  require_rowdeg(g, "pr_shard");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    fail(GBX_INVALID_VALUE, "pr_shard: bad rank / nranks");
  auto S = std::make_unique<PrShard>();
  PrPlan& P = S->plan;
  build_relabeled(g, P);
  std::vector<int64_t> rp(P.n + 1);
  GBX_CUDA(cudaMemcpyAsync(rp.data(), P.trp.p, (P.n + 1) * 8, cudaMemcpyDeviceToHost, g->stream));
  GBX_CUDA(cudaStreamSynchronize(g->stream));
  auto split = [&](int q) -> int64_t {
    if (q <= 0) return 0;
    if (q >= nranks) return P.n;
    const int64_t target = (P.n + P.nnz) * q / nranks;
    int64_t lo = 0, hi = P.n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (mid + rp[mid] < target) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  // every rank computes the same bounds from the same relabeled AT
  S->bounds.assign(nranks + 1, 0);
  for (int q = 1; q <= nranks; ++q) S->bounds[q] = std::max(S->bounds[q - 1], split(q));
  // slot = the longest block rounded up to even + 2 floats: the slot's last
  // 8 bytes carry the rank's fp64 L1 partial, so ONE all-gather per
  // iteration moves both the contributions and every partial
  int64_t longest = 1;
  for (int q = 0; q < nranks; ++q) longest = std::max(longest, S->bounds[q + 1] - S->bounds[q]);
  S->chunk = ((longest + 1) & ~int64_t(1)) + 2;
  if (S->chunk * nranks >= (int64_t(1) << 31))
    fail(GBX_INVALID_VALUE, "pr_shard: padded exchange layout exceeds int32 column ids");
  const int64_t rb = S->bounds[rank], re = S->bounds[rank + 1];
  plan_rows(g, P, rb, re);
  S->dbounds.alloc(nranks + 1);
  GBX_CUDA(cudaMemcpyAsync(S->dbounds.p, S->bounds.data(), (nranks + 1) * 8,
                           cudaMemcpyHostToDevice, g->stream));
  if (P.nnz) {
    k_pr_pad_cols<<<ceil_div(P.nnz, 256), 256, 0, g->stream>>>(P.tcol.p, P.nnz, S->dbounds.p,
                                                                 nranks, S->chunk);
    GBX_LAUNCHED();
  }
  P.invf.alloc(std::max<int64_t>(P.n, 1));
  GBX_CUDA(cudaStreamSynchronize(g->stream));
  S->nranks = nranks;
  S->rank = rank;
  g->prs = std::move(S);
  if (rb_out) *rb_out = rb;
  if (re_out) *re_out = re;
}

void pr_shard_layout(gbx_graph* g, int64_t* chunk, int64_t* bounds) {
  if (!g->prs) fail(GBX_MISSING_PROPERTY, "pr_shard_layout needs gbx_pr_shard_prepare");
  if (chunk) *chunk = g->prs->chunk;
  if (bounds) std::copy(g->prs->bounds.begin(), g->prs->bounds.end(), bounds);
}

__global__ void k_pr_shard_init(float* x, float* r_local, float* inv, const int32_t* outdeg,
                                int64_t n, int64_t rb, int64_t re, double damping,
                                const int64_t* bounds, int nranks, int64_t chunk) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double r0 = 1.0 / static_cast<double>(n);
  const int dg = outdeg[i];
  x[pr_pad_index(bounds, nranks, chunk, i)] =
      dg > 0 ? static_cast<float>(r0 / (static_cast<double>(dg) / damping)) : 0.f;
  inv[i] = dg > 0 ? static_cast<float>(damping / static_cast<double>(dg)) : 0.f;
  if (i >= rb && i < re) r_local[i - rb] = static_cast<float>(r0);
}

void pr_shard_init(gbx_graph* g, float* x_full, float* r_local, double damping) {
  if (!g->prs) fail(GBX_MISSING_PROPERTY, "pr_shard_init needs gbx_pr_shard_prepare");
  PrShard& S = *g->prs;
  PrPlan& P = S.plan;
  GBX_CUDA(cudaMemsetAsync(x_full, 0, S.chunk * S.nranks * sizeof(float), g->stream));
  k_pr_shard_init<<<ceil_div(std::max<int64_t>(P.n, 1), 256), 256, 0, g->stream>>>(
      x_full, r_local, P.invf.p, P.deg.p, P.n, P.row0, P.row1, damping, S.dbounds.p, S.nranks,
      S.chunk);
  GBX_LAUNCHED();
  P.g_damping = damping;
}

void pr_shard_step(gbx_graph* g, const float* x_full, const float* r_prev, float* r_new,
                   float* x_slice, double* l1, double damping) {
  if (!g->prs) fail(GBX_MISSING_PROPERTY, "pr_shard_step needs gbx_pr_shard_prepare");
  PrPlan& P = g->prs->plan;
  cudaStream_t s = g->stream;
  if (P.g_damping != damping) {
    k_pr_inv<<<ceil_div(std::max<int64_t>(P.n, 1), 256), 256, 0, s>>>(P.invf.p, P.deg.p, P.n,
                                                                      damping);
    GBX_LAUNCHED();
    P.g_damping = damping;
  }
  PrArgs<float> a = make_args<float>(P, damping, 0.0, 1 << 30);
  a.inv = P.invf.p;
  a.fixed = 1;
  a.x0 = const_cast<float*>(x_full);  // padded layout (tcol remapped to it)
  a.x1 = x_slice - P.row0;            // x_nxt[row] -> x_slice[row - row0]
  a.r0 = const_cast<float*>(r_prev);  // local rows; may alias r_new
  a.r1 = r_new;
  a.row0 = P.row0;
  a.hot = 0;
  a.grid_rows = rows_grid<float>(a);
  GBX_CUDA(cudaMemsetAsync(P.ctl.p, 0, 2 * sizeof(int), s));
  GBX_CUDA(cudaMemsetAsync(P.blk_cnt.p, 0, sizeof(unsigned), s));
  launch_rows<float>(a, s);
  k_pr_finish<float, false><<<P.grid_fin, kPrThreads, 0, s>>>(a);
  GBX_LAUNCHED();
  GBX_CUDA(cudaMemcpyAsync(l1, P.l1_hist.p, sizeof(double), cudaMemcpyDeviceToDevice, s));
  g->prs->steps++;
}

void pr_shard_run_p2p(gbx_graph* g, const uint64_t* x0_peers, const uint64_t* x1_peers,
                      const uint64_t* l1_peers, const uint64_t* sig_peers, float* r0, float* r1,
                      double damping, double tol, int itermax, int* iters) {
  if (!g->prs) fail(GBX_MISSING_PROPERTY, "pr_shard_run_p2p needs gbx_pr_shard_prepare");
  PrShard& S = *g->prs;
  PrPlan& P = S.plan;
  if (S.nranks > kPrMaxPeers) fail(GBX_INVALID_VALUE, "pr_shard_run_p2p: more than 8 ranks");
  if (!x0_peers || !x1_peers || !l1_peers || !sig_peers || !r0 || !r1)
    fail(GBX_NULL_ARGUMENT, "pr_shard_run_p2p: NULL buffer");
  cudaStream_t s = g->stream;
  if (P.g_damping != damping) {
    k_pr_inv<<<ceil_div(std::max<int64_t>(P.n, 1), 256), 256, 0, s>>>(P.invf.p, P.deg.p, P.n,
                                                                      damping);
    GBX_LAUNCHED();
    P.g_damping = damping;
  }
  if (itermax <= 0 || P.n == 0) {  // as pagerank_run: nothing to iterate
    if (iters) *iters = itermax <= 0 ? std::max(itermax, 0) : 0;
    return;
  }
  PrArgs<float> a = make_args<float>(P, damping, tol, itermax);
  a.inv = P.invf.p;
  a.fixed = 0;
  a.row0 = P.row0;
  a.hot = 0;
  a.x0 = reinterpret_cast<float*>(x0_peers[S.rank]);
  a.x1 = reinterpret_cast<float*>(x1_peers[S.rank]);
  a.r0 = r0;
  a.r1 = r1;
  a.npeer = S.nranks;
  const int64_t off = static_cast<int64_t>(S.rank) * S.chunk - P.row0;
  for (int q = 0; q < S.nranks; ++q) {
    a.xp[0][q] = reinterpret_cast<float*>(x0_peers[q]) + off;
    a.xp[1][q] = reinterpret_cast<float*>(x1_peers[q]) + off;
  }
  // the gathers read the local padded copy; x_nxt only selects the parity
  a.x0 = reinterpret_cast<float*>(x0_peers[S.rank]);
  a.x1 = reinterpret_cast<float*>(x1_peers[S.rank]);
  PrP2p m{};
  for (int q = 0; q < S.nranks; ++q) {
    m.l1p[q] = reinterpret_cast<double*>(l1_peers[q]);
    m.sigp[q] = reinterpret_cast<unsigned*>(sig_peers[q]);
  }
  m.l1_own = m.l1p[S.rank];
  m.sig_own = m.sigp[S.rank];
  m.rank = S.rank;
  m.nranks = S.nranks;
  int per_sm = 0;
  if (const int carve = persist_carveout(); carve >= 0)  // same L1 split as k_pr_persist
    (void)cudaFuncSetAttribute(k_pr_persist_p2p, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
  GBX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pr_persist_p2p, kPrThreads, 0));
  a.grid_rows = device_sms() * std::max(per_sm, 1);
  if (static_cast<int64_t>(P.l1_fin.n) < a.grid_rows || static_cast<int64_t>(P.l1_block.n) < a.grid_rows)
    fail(GBX_CUDA_ERROR, "pr_shard_run_p2p: partial buffers too small");
  reset_state(s, P);
  void* args[] = {&a, &m};
  GBX_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_pr_persist_p2p),
                                       dim3(a.grid_rows), dim3(kPrThreads), args, 0, s));
  GBX_LAUNCHED();
  int it = 0;
  GBX_CUDA(cudaMemcpyAsync(&it, P.ctl.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  P.last_iters = it;
  if (iters) *iters = it;
}

__global__ void k_pr_unpermute_f(const float* r, const int32_t* new2old, int64_t n, double* out,
                                 const int64_t* bounds, int nranks, int64_t chunk) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) out[new2old[i]] = static_cast<double>(r[pr_pad_index(bounds, nranks, chunk, i)]);
}

void pr_shard_unpermute(gbx_graph* g, const float* r_full, double* out_host) {
  if (!g->prs) fail(GBX_MISSING_PROPERTY, "pr_shard_unpermute needs gbx_pr_shard_prepare");
  PrShard& S = *g->prs;
  PrPlan& P = S.plan;
  cudaStream_t s = g->stream;
  double* tmp = nullptr;
  GBX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tmp), std::max<int64_t>(P.n, 1) * 8, s));
  k_pr_unpermute_f<<<ceil_div(std::max<int64_t>(P.n, 1), 256), 256, 0, s>>>(
      r_full, P.new2old.p, P.n, tmp, S.dbounds.p, S.nranks, S.chunk);
  cudaError_t le = cudaGetLastError();
  if (le == cudaSuccess) le = cudaMemcpyAsync(out_host, tmp, P.n * 8, cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(tmp, s);
  GBX_CUDA(le);
  GBX_CUDA(cudaStreamSynchronize(s));
}

}  // namespace gbx
