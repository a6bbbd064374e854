// pagerank.cu -- GAP PageRank (algo/pagerank.cpp:8-81) as a fused pull SpMV,
// every iteration inside ONE persistent cooperative launch.
//
// Reference per iteration: contrib = prior ./ (deg/damping) (:55-56), rank =
// teleport (:58), rank += AT plus.second contrib (:59-61), L1 = sum|prior -
// rank| (:65-73), stop when L1 < tol (:74).
//
// Device layout (the PageRank plan, built once per graph):
//   * vertices are relabeled by descending in-degree (stable).  R-MAT in- and
//     out-degree skews coincide, so the hot contribution entries x[k] gathered
//     by most edges land in a compact prefix of x that stays L1/L2 resident;
//   * rows are therefore sorted by length and binned: rows of one exact length
//     <= kPrShort are summed thread-per-row (32 rows per warp unit, columns
//     unit-interleaved), rows up to kPrLong warp-per-row, longer rows are cut
//     into kPrChunk-nonzero chunks whose partial sums go to fixed slots --
//     every warp gets a similar amount of work and no block barrier sits in
//     the hot loop.
// Per iteration (k_pr_persist): the row phase -- coalesced AT column loads
// (streamed, no L1 allocation), gathered x (coherent loads, hot prefix
// evict_last in L1), fp64 sums and the fused epilogue r = teleport + sum,
// |r_prev - r| (fp64), x_next = r * (damping / deg) (0 for dangling vertices
// -- their mass is lost exactly as in the reference) -- a grid barrier, the
// long-row finish (chunk slots summed in a fixed lane-strided + shuffle-tree
// order), a grid barrier, and every CTA folds all L1 partials in the same fixed
// order: the same stop decision everywhere, no host round trip.
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
#include "sort.cuh"
#include "plans.cuh"

namespace gbx {

constexpr int kPrThreads = 256;
#ifndef GBX_PR_MINB
#define GBX_PR_MINB 6  // resident CTAs per SM the rows kernel is compiled for
#endif
#ifndef GBX_PR_IPL
#define GBX_PR_IPL 8  // round 1 (2048-nonzero chunks): 4 / 8 / 16 -> 219.1 / 215.8 / 215.0; with 1024-nonzero chunks: 8 / 16 -> 172.9 / 173.5 us per iteration
#endif
constexpr int kPrIpl = GBX_PR_IPL;  // chunk walks: independent gathers in flight per lane
#ifndef GBX_PR_B0IPL
#define GBX_PR_B0IPL 6  // with the 80-nonzero bins and kPrLong 2048: 2 / 3 / 4 / 6 / 8 -> 180.7 / 178.5 / 178.4 / 176.5 / 185.3 us per iteration
#endif
constexpr int kPrB0Ipl = GBX_PR_B0IPL;  // gathers per lane per step in warp-per-row units
#ifndef GBX_PR_LONG
#define GBX_PR_LONG 2048  // at B0IPL 6: 1024 / 2048 / 3072 / 4096 / 8192 -> 176.5 / 175.6 / 175.9 / 175.6 / 244.2 us per iteration
#endif
constexpr int64_t kPrLong = GBX_PR_LONG;  // rows longer than this are chunked
#ifndef GBX_PR_SHORT
// measured: 32 / 48 / 64 / 66 / 72 / 80 / 96 / 128 / 158 -> 204.6 / 194.0 / 192.3 / 185.7 /
// 183.6 / 183.8 / 183.9 / 189.6 / 191.8 us per iteration
#define GBX_PR_SHORT 80
#endif
constexpr int64_t kPrShort = GBX_PR_SHORT;  // rows up to this length: thread per row, exact-length bins
#ifndef GBX_PR_ZBLK
#define GBX_PR_ZBLK 1024
#endif
constexpr int64_t kPrZeroBlk = GBX_PR_ZBLK;  // rows without in-edges: rows per dynamically claimed block
static_assert(GBX_PR_SHORT + 2 <= kPrBinsMax, "one bin per exact length + the warp-per-row bin");
#ifndef GBX_PR_CHUNK
#define GBX_PR_CHUNK 1024  // 512 / 768 / 1024 / 1280 / 2048 / 3072 / 4096 -> 176.2 / 174.0 / 173.5 / 178.9 / 175.8 / 181.9 / 194.1 us per iteration
#endif
constexpr int64_t kPrChunk = GBX_PR_CHUNK;  // nonzeros per chunk unit
constexpr unsigned kWarp = 0xffffffffu;
constexpr int kPrMaxPeers = 8;     // ranks of the fused P2P exchange (one NVSwitch box)

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
  double* l1_rows;     // [2][grid] per-CTA row-phase partials (by iteration parity)
  double* l1_fin;      // [gridB]
  double* l1_hist;
  int* ctl;            // [0] completed iterations [1] done [2] peer timeout (fused exchange)
  unsigned long long* ktime;  // [128][8]: per iteration, min CTA start / max CTA end of the row phase (%globaltimer); trace: [2] min after barrier 1, [3] max finish end, [4] min after barrier 2, [5] max fold end
  int trace;
  unsigned long long* cta_end;  // trace: every CTA's row-phase end in iteration 5
  unsigned* fin_cnt;
  unsigned* dyn_cnt;   // [4] block counters of the rows without in-edges, by iteration & 3
  unsigned long long* l1_acc;  // [4] the iteration's L1 norm in 2^-60 fixed point, by iteration & 3
  int64_t zrow0, zrow1;  // rows without in-edges, claimed in blocks of kPrZeroBlk
  int64_t l1hot;       // x[0, l1hot) gathered with L1 evict_last, the rest no_allocate
  int64_t nx;          // entries of x (device checks)
  int64_t row0;        // first row of this plan (shards); outputs indexed row - row0
  int grid_rows;
  double damping, teleport, tol;
  int itermax;
  int fixed;           // single step: r0/x0 inputs, r1/x1 outputs, no convergence
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

// Cache-policy loads (PTX).  The AT column stream is read-only for the whole
// launch: non-coherent path, no L1 allocation.  x is rewritten every
// iteration inside the same persistent launch (and by peer GPUs in the fused
// multi-GPU kernel), so its gathers are COHERENT weak loads (no .nc) that keep
// the eviction hints: the hot prefix (the highest-degree vertices after
// relabeling) stays in L1 (evict_last) within an iteration, the cold gathers
// bypass L1; the grid barrier between iterations orders them after the writes
// (PTX memory model: release/acquire at gpu scope).  volatile: never merged or
// moved across the barriers by the compiler.
__device__ __forceinline__ int ld_stream(const int32_t* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_hot(const float* p) {
  float v;
  asm volatile("ld.global.L1::evict_last.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_hot(const double* p) {
  double v;
  asm volatile("ld.global.L1::evict_last.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_cold(const float* p) {
  float v;
  asm volatile("ld.global.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_cold(const double* p) {
  double v;
  asm volatile("ld.global.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// device clock for the live launch-duration measurement of k_pr_rows (the
// iterations run inside one CUDA graph, where events cannot bracket a node)
__device__ __forceinline__ unsigned long long pr_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// gather x[c]: the L1-resident prefix [0, l1hot) (evict_last), the rest from
// L2 without L1 allocation
template <typename V>
__device__ __forceinline__ V pr_xg(int64_t l1hot, const V* x, int c) {
  return c < l1hot ? ld_hot(x + c) : ld_cold(x + c);
}
#define PR_CHECK_COL(a, c) GBX_DCHECK((c) < (a).nx, "pagerank column", (c))

// fused epilogue of one row with prefetched r_prev / out-degree
template <typename V>
__device__ __forceinline__ double pr_finish_row(const PrArgs<V>& a, V* r_nxt, V* x_nxt,
                                                int64_t row, double s, V rprev, V inv) {
  const double rn = a.teleport + s;
  GBX_DCHECK(row >= a.row0 && row < a.nx, "pagerank row", row);
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

// One iteration's row work for CTA `cta` of `ncta` (every unit of the grid-
// stride walk); returns the CTA's fp64 L1 partial (valid in thread 0).
template <typename V>
__device__ __forceinline__ double pr_rows_phase(const PrArgs<V>& a, int k, int cta, int ncta,
                                                typename cub::BlockReduce<double, kPrThreads>::TempStorage& red,
                                                PrBinS* s_bins) {
  using BlockReduce = cub::BlockReduce<double, kPrThreads>;
  const V *x_cur, *r_cur;
  V *x_nxt, *r_nxt;
  pr_buffers(a, k, x_cur, r_cur, x_nxt, r_nxt);
  for (int i = threadIdx.x; i < a.nbins; i += blockDim.x) {
    const PrBin b = a.bins[i];
    s_bins[i] = PrBinS{b.p0, static_cast<int32_t>(b.unit0), static_cast<int32_t>(b.row0),
                       static_cast<int32_t>(b.row1), b.len};
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (cta * int64_t(kPrThreads) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(ncta) * kPrThreads) >> 5;
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
        if (c[j] >= 0) {
          PR_CHECK_COL(a, c[j]);
          s += static_cast<double>(pr_xg(a.l1hot, x_cur, c[j]));
        }
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
    const PrBinS& B = s_bins[bk];
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
          if (c[q] >= 0) {
            PR_CHECK_COL(a, c[q]);
            s += static_cast<double>(pr_xg(a.l1hot, x_cur, c[q]));
          }
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
          for (int q = 0; q < 4; ++q) {
            if (c[q] >= 0) PR_CHECK_COL(a, c[q]);
            t[q] = c[q] >= 0 ? pr_xg(a.l1hot, x_cur, c[q]) : V(0);
          }
          s += (static_cast<double>(t[0]) + static_cast<double>(t[1])) +
               (static_cast<double>(t[2]) + static_cast<double>(t[3]));
#pragma unroll
          for (int q = 0; q < 4; ++q) c[q] = nx[q];
        }
        l1 += pr_finish_row(a, r_nxt, x_nxt, row, s, rprev, inv);
      }
    }
  }
  // 3) rows without in-edges (r = teleport; the same arithmetic as an exact-
  //    length unit of length 0), claimed in blocks from the iteration's
  //    counter: the CTAs' static shares end up to ~7% apart (measured), and
  //    whoever is done first takes more of this cheap tail (row phase 171 ->
  //    165 us; blocks of 256 / 1024 / 4096 rows: 166 / 165 / 190 us).  Claiming
  //    the shortest exact-length bins the same way costs the main loops
  //    registers (spills) and lost: 168 us.
  if (a.zrow1 > a.zrow0) {
    unsigned* const dyn = a.dyn_cnt + (k & 3);
    for (;;) {
      unsigned blk = 0;
      if (lane == 0) blk = atomicAdd(dyn, 1u);
      blk = __shfl_sync(kWarp, blk, 0);
      const int64_t z0 = a.zrow0 + int64_t(blk) * kPrZeroBlk;
      if (z0 >= a.zrow1) break;
      const int64_t z1 = min(z0 + kPrZeroBlk, a.zrow1);
      for (int64_t row = z0 + lane; row < z1; row += 32)
        l1 += pr_finish_row(a, r_nxt, x_nxt, row, 0.0, r_cur[row - a.row0], a.inv[row]);
    }
  }
  __syncthreads();  // red may still be in use by a previous reduction
  return BlockReduce(red).Sum(l1);
}

// long rows: the chunk slots of every long row summed by one warp each
// (lane-strided, fixed shuffle tree) and the row's epilogue; returns the
// CTA's fp64 L1 partial (valid in thread 0)
template <typename V>
__device__ __forceinline__ double pr_long_phase(const PrArgs<V>& a, int k, int cta, int ncta,
                                                typename cub::BlockReduce<double, kPrThreads>::TempStorage& red) {
  using BlockReduce = cub::BlockReduce<double, kPrThreads>;
  const V *x_cur, *r_cur;
  V *x_nxt, *r_nxt;
  pr_buffers(a, k, x_cur, r_cur, x_nxt, r_nxt);
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (cta * int64_t(kPrThreads) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(ncta) * kPrThreads) >> 5;
  double l1 = 0.0;
  // the zero-row block counter iteration k + 2 will use (last read in k - 2)
  if (cta == 0 && threadIdx.x == 0) {
    a.dyn_cnt[(k + 2) & 3] = 0u;
    a.l1_acc[(k + 2) & 3] = 0ull;
  }
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
  return BlockReduce(red).Sum(l1);
}

// host-looped row kernel (pr_shard_step, and the per-iteration path kept for
// ncu captures: option pagerank.host_loop)
template <typename V>
__global__ void __launch_bounds__(kPrThreads, GBX_PR_MINB) k_pr_rows(PrArgs<V> a) {
  using BlockReduce = cub::BlockReduce<double, kPrThreads>;
  __shared__ typename BlockReduce::TempStorage red;
  __shared__ PrBinS s_bins[kPrBinsMax];
  if (!a.fixed && *(volatile int*)&a.ctl[1]) return;  // converged (host-looped path)
  const int k = *(volatile int*)&a.ctl[0];
  if (a.ktime && threadIdx.x == 0) atomicMin(&a.ktime[(k % 128) * 8], pr_gtimer());
  const double blk = pr_rows_phase<V>(a, k, blockIdx.x, gridDim.x, red, s_bins);
  if (threadIdx.x == 0) {
    a.l1_rows[blockIdx.x] = blk;
    if (a.ktime) atomicMax(&a.ktime[(k % 128) * 8 + 1], pr_gtimer());
  }
}

// The whole iteration loop in ONE cooperative launch: per iteration the row
// phase, a grid barrier, the long-row finish (warp per long row), a grid
// barrier, then every CTA folds all L1 partials in the same fixed order and
// reaches the same convergence decision (pagerank.cpp:65-74).  Replaces a
// graph's two kernel nodes + conditional per iteration (~20 us of launch gaps
// per iteration against ~200 us of row work) with two grid barriers.
// The row partials are double-buffered by iteration parity: a CTA that has
// folded iteration k's partials races ahead into iteration k+1's row phase
// while slower CTAs still fold k -- it writes the other half (the next write
// of this half, at k+2, comes after barrier #1 of k+1, which every CTA passes
// only after its fold of k).
template <typename V>
__global__ void __launch_bounds__(kPrThreads, GBX_PR_MINB) k_pr_persist(PrArgs<V> a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  using BlockReduce = cub::BlockReduce<double, kPrThreads>;
  __shared__ typename BlockReduce::TempStorage red;
  __shared__ PrBinS s_bins[kPrBinsMax];
  __shared__ int s_stop;
  const int ncta = gridDim.x;
  for (int k = 0;; ++k) {
    // the CTA's L1 partial (rows + long rows) of iteration k, by parity
    double* l1_part = a.l1_rows + (k & 1) * ncta;
    if (a.ktime && threadIdx.x == 0) atomicMin(&a.ktime[(k % 128) * 8], pr_gtimer());
    const double blk = pr_rows_phase<V>(a, k, blockIdx.x, ncta, red, s_bins);
    if (threadIdx.x == 0 && a.ktime) atomicMax(&a.ktime[(k % 128) * 8 + 1], pr_gtimer());
    if (a.trace && k == 5 && threadIdx.x == 0) a.cta_end[blockIdx.x] = pr_gtimer();
    grid.sync();
    unsigned long long* kt = a.ktime + (k % 128) * 8;
    if (a.trace && threadIdx.x == 0) atomicMin(kt + 2, pr_gtimer());
    const double blk2 = pr_long_phase<V>(a, k, blockIdx.x, ncta, red);
    if (threadIdx.x == 0) {
      // the CTAs' partials meet in ONE integer accumulator (2^-60 fixed point:
      // the sum does not depend on the order of the atomics, every CTA reads
      // the same total after the barrier) instead of every CTA re-reading and
      // folding all of them: 2.1 -> 0.7 us per iteration
      l1_part[blockIdx.x] = blk + blk2;
      const double p = fmin(blk + blk2, 8.0);
      atomicAdd(&a.l1_acc[k & 3], static_cast<unsigned long long>(__double2ll_rn(p * 0x1p60)));
      if (a.trace) atomicMax(kt + 3, pr_gtimer());
    }
    grid.sync();
    if (a.trace && threadIdx.x == 0) atomicMin(kt + 4, pr_gtimer());
    if (a.trace && threadIdx.x == 0) atomicMax(kt + 5, pr_gtimer());
    if (threadIdx.x == 0) {
      const double tot =
          static_cast<double>(*(volatile unsigned long long*)&a.l1_acc[k & 3]) * 0x1p-60;
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
// cooperative launch per GPU for the whole run).  Per iteration: the row
// phase and the long-row finish store x_next into EVERY rank's x (peer
// pointers over NVLink / NVSwitch); the rank's fp64 L1 total goes to slot
// [k&1][rank] of every rank's table; then a cross-rank barrier -- system-scope
// fence per CTA, grid barrier, one signal increment per peer, a BOUNDED spin on
// the own signal word, grid barrier -- and every CTA sums the table in rank
// order: the same decision on every rank (pagerank.cpp:74).  x and the slot
// table are double-buffered by iteration parity, so a rank one iteration ahead
// never overwrites what a slower rank still reads.
//
// The spin gives up after timeout_ns (%globaltimer): a peer that never
// launched, crashed or was handed other arguments then surfaces as an error
// word (ctl[2] = 1) on every waiting rank -- the host turns it into
// GBX_CUDA_ERROR and the driver falls back to the NCCL exchange -- instead of
// a cooperative grid spinning forever.
//
// `nvirt` ranks may share ONE launch on one GPU (blocks [v*per, (v+1)*per)
// are rank v; each rank's arguments in device memory): the emulation of a
// multi-GPU run that the tests use -- every rank's CTAs are co-resident
// (cooperative launch), so the ranks' spins always see each other's signals.
// On a real multi-GPU run nvirt = 1 and the arguments come by value.
struct PrP2p {
  double* l1p[kPrMaxPeers];     // rank q's slot table [2][nranks]
  unsigned* sigp[kPrMaxPeers];  // rank q's signal word
  double* l1_own;               // this rank's table
  unsigned* sig_own;            // this rank's signal word
  int rank, nranks;
  unsigned long long timeout_ns;
};

__device__ __forceinline__ void pr_p2p_body(const PrArgs<float>& a, const PrP2p& m, int cta,
                                            int ncta, cooperative_groups::grid_group& grid,
                                            cub::BlockReduce<double, kPrThreads>::TempStorage& red,
                                            PrBinS* s_bins, int& s_stop) {
  using BlockReduce = cub::BlockReduce<double, kPrThreads>;
  for (int k = 0;; ++k) {
    if (a.ktime && threadIdx.x == 0) atomicMin(&a.ktime[(k % 128) * 8], pr_gtimer());
    const double blk = pr_rows_phase<float>(a, k, cta, ncta, red, s_bins);
    if (threadIdx.x == 0) {
      a.l1_rows[cta] = blk;
      if (a.ktime) atomicMax(&a.ktime[(k % 128) * 8 + 1], pr_gtimer());
    }
    grid.sync();
    const double blk2 = pr_long_phase<float>(a, k, cta, ncta, red);
    if (threadIdx.x == 0) a.l1_fin[cta] = blk2;
    __threadfence_system();  // this CTA's peer stores before the signal below
    grid.sync();
    if (cta == 0) {
      double part = 0.0;
      for (int b = threadIdx.x; b < ncta; b += kPrThreads)
        part += __ldcg(&a.l1_rows[b]) + __ldcg(&a.l1_fin[b]);
      __syncthreads();
      const double mine = BlockReduce(red).Sum(part);
      if (threadIdx.x == 0) {
        const int par = k & 1;
        for (int q = 0; q < m.nranks; ++q) m.l1p[q][par * m.nranks + m.rank] = mine;
        __threadfence_system();
        for (int q = 0; q < m.nranks; ++q) atomicAdd_system(m.sigp[q], 1u);
        // every rank signals every rank once per iteration
        // (the caller zeroes the signal words and barriers before the run)
        const unsigned want = static_cast<unsigned>(m.nranks) * (k + 1);
        const unsigned long long t0 = pr_gtimer();
        for (;;) {
          unsigned v;
          asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(m.sig_own) : "memory");
          if (static_cast<int>(v - want) >= 0) break;
          if (pr_gtimer() - t0 > m.timeout_ns) {
            atomicExch(&a.ctl[2], 1);  // a peer never arrived: every CTA leaves below
            break;
          }
          __nanosleep(256);
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
      const bool failed = *(volatile int*)&a.ctl[2] != 0;
      const bool stop = failed || !(tot >= a.tol) || (k + 1 >= a.itermax);
      s_stop = stop;
      if (cta == 0) {
        a.l1_hist[k % 128] = tot;
        a.ctl[0] = k + 1;
        if (stop) a.ctl[1] = 1;
      }
    }
    __syncthreads();
    if (s_stop) break;
  }
}

__global__ void __launch_bounds__(kPrThreads, GBX_PR_MINB) k_pr_persist_p2p(PrArgs<float> a,
                                                                            PrP2p m) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ cub::BlockReduce<double, kPrThreads>::TempStorage red;
  __shared__ PrBinS s_bins[kPrBinsMax];
  __shared__ int s_stop;
  pr_p2p_body(a, m, blockIdx.x, gridDim.x, grid, red, s_bins, s_stop);
}

// nvirt emulated ranks in one launch (arguments per rank in device memory,
// staged in shared memory per CTA)
__global__ void __launch_bounds__(kPrThreads, GBX_PR_MINB) k_pr_persist_p2p_virt(
    const PrArgs<float>* va, const PrP2p* vm, int nvirt) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ cub::BlockReduce<double, kPrThreads>::TempStorage red;
  __shared__ PrBinS s_bins[kPrBinsMax];
  __shared__ int s_stop;
  __shared__ PrArgs<float> sa;
  __shared__ PrP2p sm;
  const int per = gridDim.x / nvirt;
  const int v = blockIdx.x / per;
  if (threadIdx.x == 0) {
    sa = va[v];
    sm = vm[v];
  }
  __syncthreads();
  pr_p2p_body(sa, sm, blockIdx.x - v * per, per, grid, red, s_bins, s_stop);
}

template <typename V>
__global__ void __launch_bounds__(kPrThreads) k_pr_finish(PrArgs<V> a) {
  using BlockReduce = cub::BlockReduce<double, kPrThreads>;
  __shared__ typename BlockReduce::TempStorage red;
  __shared__ int s_last;
  if (!a.fixed && *(volatile int*)&a.ctl[1]) return;
  const int k = *(volatile int*)&a.ctl[0];
  const unsigned epoch = static_cast<unsigned>(k) + 1u;
  const double blk = pr_long_phase<V>(a, k, blockIdx.x, gridDim.x, red);
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
  }
}

__global__ void k_pr_inv(float* inv, const int32_t* outdeg, int64_t n, double damping) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) inv[i] = outdeg[i] > 0 ? static_cast<float>(damping / static_cast<double>(outdeg[i])) : 0.f;
}

template <typename V>
__global__ void k_pr_init(V* r, V* x, V* inv, const int32_t* outdeg, int64_t n, double damping,
                          int* ctl, unsigned* fin_cnt, unsigned long long* ktime) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  // the run's control words and launch-span table (one kernel instead of
  // three memsets / resets before the persistent launch)
  if (i < 4) ctl[i] = 0;
  if (i < 16) fin_cnt[i] = 0;  // the finish counter, the zero-row block counters, the L1 accumulators
  if (ktime && i < 128 * 8) ktime[i] = (i & 1) ? 0ull : ~0ull;
  if (i >= n) return;
  const double r0 = 1.0 / static_cast<double>(n);
  r[i] = static_cast<V>(r0);
  const int dg = outdeg[i];
  // contrib = prior ./ (deg / damping) (pagerank.cpp:30-40, 55-56); the
  // iterations use the precomputed damping / deg (0: dangling, mass lost)
  x[i] = dg > 0 ? static_cast<V>(r0 / (static_cast<double>(dg) / damping)) : V(0);
  inv[i] = dg > 0 ? static_cast<V>(damping / static_cast<double>(dg)) : V(0);
}

// relabeled rank -> original ids (fp64 for the host copy); the buffer holding
// the last iterate is chosen on the device from the completed-iteration count,
// so the launch is queued before the host reads anything back
template <typename V>
__global__ void k_pr_unpermute(const V* r0, const V* r1, const int* ctl, const int32_t* new2old,
                               int64_t n, double* out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) out[new2old[i]] = static_cast<double>((ctl[0] & 1) ? r1[i] : r0[i]);
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
__global__ void k_gather_i32(const int32_t* src, const int32_t* idx, int64_t n, int32_t* dst) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

// exact-length bins (bins[b0..nbins), ascending p0), row-major -> unit-
// interleaved (32-row units; element j of unit row l at unit*32*L + j*m + l):
// one launch over the bins' whole nonzero range [q0, q1)
__global__ void k_pr_interleave(const int32_t* src, int32_t* dst, const PrBin* bins, int b0,
                                int nbins, int64_t q0, int64_t q1) {
  __shared__ int64_t s_p0[kPrBinsMax + 1];
  for (int i = threadIdx.x; i < nbins - b0; i += blockDim.x) s_p0[i] = bins[b0 + i].p0;
  __syncthreads();
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t p = q0 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < q1; p += stride) {
    int lo = 0, hi = nbins - b0 - 1;  // last bin with p0 <= p
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_p0[mid] <= p) lo = mid; else hi = mid - 1;
    }
    const PrBin& B = bins[b0 + lo];
    const int L = B.len;
    if (L <= 0) continue;
    const int64_t nrows = B.row1 - B.row0;
    const int64_t q = p - B.p0;
    const int64_t i = q / L;
    const int j = static_cast<int>(q - i * L);
    const int64_t u = i >> 5;
    const int m = static_cast<int>(min(int64_t(32), nrows - u * 32));
    dst[B.p0 + u * 32 * L + int64_t(j) * m + (i & 31)] = src[q + (B.p0 - q0)];
  }
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
    k_pr_bounds<<<(nt + 63) / 64, 64, 0, s>>>(P.trp.p, row0, row1, dthr.p, nt, drow.p, dp.p);
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
  P.zrow0 = P.zrow1 = 0;
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
    if (len == 0) {
      // the rows without in-edges are not warp units: claimed in blocks
      P.zrow0 = r0;
      P.zrow1 = r1;
      continue;
    }
    bins.push_back(b);
    units += (r1 - r0 + 31) / 32;
  }
  if (bins.size() > static_cast<size_t>(kPrBinsMax)) fail(GBX_CUDA_ERROR, "pagerank: too many bins");
  P.nbins = static_cast<int>(bins.size());
  P.bins.alloc(std::max<size_t>(bins.size(), 1));
  if (!bins.empty())
    GBX_CUDA(cudaMemcpyAsync(P.bins.p, bins.data(), bins.size() * sizeof(PrBin),
                             cudaMemcpyHostToDevice, s));
  // exact-length bins: columns to the unit-interleaved layout k_pr_rows reads
  // (the bins with len > 0 are contiguous in the bin list and in tcol)
  {
    int64_t q0 = -1, q1 = -1;
    int b0 = -1;
    for (size_t i = 0; i < bins.size(); ++i) {
      const PrBin& b = bins[i];
      if (b.len > 0) {
        if (q0 < 0) {
          q0 = b.p0;
          b0 = static_cast<int>(i);
        }
        q1 = b.p0 + (b.row1 - b.row0) * b.len;
      }
    }
    if (q0 >= 0 && q1 > q0) {
      Tmp<int32_t> cp(q1 - q0, s);
      GBX_CUDA(cudaMemcpyAsync(cp.p, P.tcol.p + q0, (q1 - q0) * 4, cudaMemcpyDeviceToDevice, s));
      // bins after the last positive length (len 0) hold no nonzeros
      int b1 = b0;
      while (b1 < static_cast<int>(bins.size()) && bins[b1].len > 0) ++b1;
      k_pr_interleave<<<device_sms() * 8, 256, 0, s>>>(cp.p, P.tcol.p, P.bins.p, b0, b1, q0, q1);
      GBX_LAUNCHED();
    }
  }
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
__global__ void k_pr_gather_len(const int32_t* len, const int32_t* new2old, int64_t n, int64_t* out) {
  const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (r <= n) out[r] = r < n ? len[new2old[r]] : 0;
}
constexpr int64_t kPrGatherLong = 256;
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
// rows of up to kPrGatherLong entries: a warp takes 32 consecutive new rows
// (lane l holds row l's source pointer, destination and length), then walks
// the concatenation of their entries one per lane -- the owner row of an
// entry by a shuffle binary search over the lanes' prefix sums -- four
// entries per lane in flight (column, then its new id), coalesced stores
__global__ void __launch_bounds__(256) k_pr_gather_a_short(const int64_t* arp, const int32_t* acol,
                                    const int32_t* new2old, const int32_t* old2new,
                                    const int64_t* prp, int64_t n, uint32_t* key, uint32_t* val) {
  constexpr unsigned kAllW = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r0 = gw * 32; r0 < n; r0 += nw * 32) {
    const int64_t r = r0 + lane;
    int64_t d = 0, src = 0;
    int len = 0;
    if (r < n) {
      d = prp[r];
      const int64_t l = prp[r + 1] - d;
      if (l <= kPrGatherLong) {
        len = static_cast<int>(l);
        src = arp[new2old[r]];
      }
    }
    int inc = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(kAllW, inc, o);
      if (lane >= o) inc += t;
    }
    const int total = __shfl_sync(kAllW, inc, 31);
    const int exc = inc - len;
    for (int base = 0; base < total; base += 128) {
      int64_t at[4], to[4];
      int row[4];
      bool ok[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int q = base + 32 * k + lane;
        ok[k] = q < total;
        int lo = 0;  // last lane whose exclusive prefix is <= q (an empty row never wins: the
                     // next lane has the same prefix)
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
          const int e = __shfl_sync(kAllW, exc, (lo + step) & 31);
          if (lo + step < 32 && e <= q) lo += step;
        }
        const int e = __shfl_sync(kAllW, exc, lo);
        const int64_t sj = __shfl_sync(kAllW, src, lo);
        const int64_t dj = __shfl_sync(kAllW, d, lo);
        at[k] = sj + (q - e);
        to[k] = dj + (q - e);
        row[k] = lo;
      }
      int32_t c[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) c[k] = ok[k] ? __ldg(acol + at[k]) : 0;
      int32_t nc[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) nc[k] = ok[k] ? __ldg(old2new + c[k]) : 0;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (ok[k]) {
          key[to[k]] = static_cast<uint32_t>(nc[k]);
          val[to[k]] = static_cast<uint32_t>(r0 + row[k]);
        }
    }
  }
}

// plan phases on stderr (option pagerank.trace; synchronises per phase)
struct PlanTimer {
  cudaStream_t s;
  bool on;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    GBX_CUDA(cudaStreamSynchronize(s));
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "pagerank plan: %-28s %8.1f us\n", what,
                 std::chrono::duration<double, std::micro>(t1 - t0).count());
    t0 = t1;
  }
};

// The transpose of A under a relabeling (plans.cuh / common.cuh): row r of the
// result holds the new ids of the rows of A that have (old) column new2old[r],
// ascending.  A's rows are gathered in the new order as (new column, new row)
// pairs -- ordered by new row -- then ONE stable 32-bit radix sort by new column
// (two sorts took 4.4 ms at scale 22, this ~2.4 ms); the row pointers are the
// scan of A's column counts in the new order.  trp: n + 1, tcol: nnz entries.
void relabeled_transpose(cudaStream_t s, const Csr& A, const int32_t* new2old,
                         const int32_t* old2new, const int32_t* colcount, int64_t* trp,
                         int32_t* tcol) {
  PlanTimer tm{s, option(kOptPrTrace) != 0};
  const int64_t n = A.n, nnz = A.nnz;
  // relabeled AT, every row's columns ascending in the new ids (the thread-
  // per-row bins then read the hub end of x together at each step): A's rows
  // gathered in the new order as (new column, new row) pairs -- ordered by new
  // row -- then ONE stable 32-bit radix sort by new column (two sorts took
  // 4.4 ms at scale 22, this ~2.4 ms)
  const int bits = bits_for(std::max<int64_t>(n, 2));
  if (nnz) {
    DevArray<int64_t> prp(n + 1);
    k_pr_newlen<<<ceil_div(n + 1, 256), 256, 0, s>>>(A.rp.p, new2old, n, prp.p);
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
        k_pr_gather_a_long<<<device_sms() * 8, 256, 0, s>>>(A.rp.p, A.col.p, new2old,
                                                             old2new, prp.p, list.p, nch.p, m,
                                                             kc.p, vr.p);
      }
    }
    k_pr_gather_a_short<<<device_sms() * 8, 256, 0, s>>>(A.rp.p, A.col.p, new2old,
                                                          old2new, prp.p, n, kc.p, vr.p);
    GBX_LAUNCHED();
    tm.mark("gather A rows (new order)");
    // double buffers (the value alternate is the plan's own tcol) and a 32-bit item count
    cub::DoubleBuffer<uint32_t> kb(kc.p, kc2.p);
    cub::DoubleBuffer<uint32_t> vb(vr.p, reinterpret_cast<uint32_t*>(tcol));
    radix_sort_pairs(s, kb, vb, nnz, 0, bits);
    if (vb.Current() != reinterpret_cast<uint32_t*>(tcol))
      GBX_CUDA(cudaMemcpyAsync(tcol, vb.Current(), nnz * 4, cudaMemcpyDeviceToDevice, s));
    tm.mark("radix sort by new column");
    // row pointers of the relabeled AT: the exclusive scan of the in-degrees in
    // the new order (no pass over the sorted keys)
    k_pr_gather_len<<<ceil_div(n + 1, 256), 256, 0, s>>>(colcount, new2old, n, trp);
    GBX_LAUNCHED();
    {
      size_t tb = 0;
      GBX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, trp, trp, n + 1, s));
      Tmp<uint8_t> t(tb, s);
      GBX_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tb, trp, trp, n + 1, s));
    }
    tm.mark("row pointers");
  } else {
    GBX_CUDA(cudaMemsetAsync(trp, 0, (n + 1) * sizeof(int64_t), s));
  }
}

// relabeled AT (rows by descending in-degree) + relabeled out-degree
static void build_relabeled(gbx_graph* g, PrPlan& P) {
  PlanTimer tm{g->stream, option(kOptPrTrace) != 0};
  cudaStream_t s = g->stream;
  const Csr& A = g->A;
  const int64_t n = A.n, nnz = A.nnz;
  P.n = n;
  P.nnz = nnz;
  // in-degree = AT's row lengths = A's column counts: the plan is built from
  // A alone (the relabeled AT below is gathered from A's rows), so a pending
  // transpose is never materialised for PageRank
  DevArray<int32_t> len;
  if (g->kind == GBX_UNDIRECTED) {
    len.alloc(std::max<int64_t>(n, 1));
    if (n) {
      k_neg_len<<<ceil_div(n, 256), 256, 0, s>>>(A.rp.p, n, len.p);
      GBX_LAUNCHED();
    }
  } else if (g->has_colcount) {
    len = std::move(g->colcount);  // counted while the host CSR was uploaded
    g->has_colcount = false;
  } else {
    compute_degrees(s, A, len, false);
  }
  tm.mark("in-degrees");
  sort_ids_by_key(s, len.p, n, false, P.new2old);
  tm.mark("relabel sort");
  P.old2new.alloc(std::max<int64_t>(n, 1));
  P.deg.alloc(std::max<int64_t>(n, 1));
  if (n) {
    k_inverse_perm<<<ceil_div(n, 256), 256, 0, s>>>(P.new2old.p, n, P.old2new.p);
    k_gather_i32<<<ceil_div(n, 256), 256, 0, s>>>(g->rowdeg.p, P.new2old.p, n, P.deg.p);
    GBX_LAUNCHED();
  }
  // relabeled AT, every row's columns ascending in the new ids (the thread-
  // per-row bins then read the hub end of x together at each step)
  P.trp.alloc(n + 1);
  P.tcol.alloc(std::max<int64_t>(nnz, 1));
  relabeled_transpose(s, A, P.new2old.p, P.old2new.p, len.p, P.trp.p, P.tcol.p);
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
  P.ktime.alloc(128 * 8);
  P.ctl.alloc(4);
  P.blk_cnt.alloc(16);  // [0] finish counter, [4..7] zero-row block counters, [8..15] four u64 L1 accumulators
}

void pagerank_prepare(gbx_graph* g) {
  NvtxRange nvtx_("gbx.pagerank.prepare");
  require_at(g, "pagerank_gap");
  require_rowdeg(g, "pagerank_gap");
  if (g->pr) return;
  auto P = std::make_unique<PrPlan>();
  PlanTimer tm{g->stream, option(kOptPrTrace) != 0};
  build_relabeled(g, *P);
  tm.mark("relabeled AT (total)");
  plan_rows(g, *P, 0, P->n);
  tm.mark("work units / bins");
  for (int b = 0; b < 2; ++b) {
    P->r[b].alloc(std::max<int64_t>(g->A.n, 1));
    P->x[b].alloc(std::max<int64_t>(g->A.n, 1));
  }
  P->out.alloc(std::max<int64_t>(g->A.n, 1));
  tm.mark("vectors");
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

// bytes of x kept L1-resident (option pagerank.l1_window_kb; measured at the
// 32 KB carveout: 64 / 96 / 112 / 128 / 144 / 160 / 176 / 192 KB -> 221.6 /
// 216.1 / 209.9 / 209.0 / 205.9 / 207.0 / 208.4 / 209.7 us/iter)
static int64_t l1_hot_bytes() { return option(kOptPrL1WindowKb) * 1024; }

// shared-memory carveout of the row kernels: 10% -> 32 KB of shared memory,
// 224 KB of L1 (214.0 -> 207.1 us/iter, A/B); < 0 leaves the driver's choice
static void set_carveout(const void* fn) {
  const int carve = static_cast<int>(option(kOptPrCarveout));
  if (carve >= 0) (void)cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
  (void)cudaGetLastError();
}

// resident CTAs per SM x SMs for a row kernel
static int resident_grid(const void* fn) {
  set_carveout(fn);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kPrThreads, 0) != cudaSuccess) {
    (void)cudaGetLastError();
    per_sm = 1;
  }
  return device_sms() * std::max(per_sm, 1);
}

template <typename V>
static void launch_rows(const PrArgs<V>& a, cudaStream_t s) {
  k_pr_rows<V><<<a.grid_rows, kPrThreads, 0, s>>>(a);
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
  a.trace = static_cast<int>(option(kOptPrTrace));
  if (a.trace && !P.cta_end.p) P.cta_end.alloc(static_cast<size_t>(device_sms()) * 32);
  a.cta_end = P.cta_end.p;
  a.fin_cnt = P.blk_cnt.p;
  a.dyn_cnt = P.blk_cnt.p + 4;
  a.l1_acc = reinterpret_cast<unsigned long long*>(P.blk_cnt.p + 8);
  a.zrow0 = P.zrow0;
  a.zrow1 = P.zrow1;
  a.row0 = 0;
  a.l1hot = std::min<int64_t>(P.n, l1_hot_bytes() / static_cast<int64_t>(sizeof(V)));
  a.nx = P.n;
  a.grid_rows = resident_grid(reinterpret_cast<const void*>(k_pr_rows<V>));
  a.damping = damping;
  a.teleport = (1.0 - damping) / static_cast<double>(P.n);
  a.tol = tol;
  a.itermax = itermax;
  a.fixed = 0;
  return a;
}

__global__ void k_pr_ktime_reset(unsigned long long* t) {
  const int i = threadIdx.x;
  for (int j = i; j < 128 * 8; j += blockDim.x) t[j] = (j & 1) ? 0ull : ~0ull;
}

static void reset_state(cudaStream_t s, PrPlan& P) {
  GBX_CUDA(cudaMemsetAsync(P.ctl.p, 0, P.ctl.n * sizeof(int), s));
  GBX_CUDA(cudaMemsetAsync(P.blk_cnt.p, 0, 16 * sizeof(unsigned), s));
  if (P.ktime.p) k_pr_ktime_reset<<<1, 256, 0, s>>>(P.ktime.p);
}

// the persistent kernel needs every CTA resident (cooperative launch); its
// row partials are double-buffered (2 * grid entries)
template <typename V>
static bool persist_args(PrPlan& P, double damping, double tol, int itermax, PrArgs<V>& a) {
  a = make_args<V>(P, damping, tol, itermax);
  a.grid_rows = resident_grid(reinterpret_cast<const void*>(k_pr_persist<V>));
  return static_cast<int64_t>(P.l1_fin.n) >= a.grid_rows &&
         static_cast<int64_t>(P.l1_block.n) >= 2 * static_cast<int64_t>(a.grid_rows);
}

template <typename V>
static int pagerank_loop(gbx_graph* g, PrPlan& P, double damping, double tol, int itermax,
                         double* rank, int* iters) {
  const int64_t n = g->A.n;
  cudaStream_t s = g->stream;
  P.last_persist = false;
  k_pr_init<V><<<ceil_div(std::max<int64_t>(n, 128 * 8), 256), 256, 0, s>>>(
      buf_r<V>(P, 0), buf_x<V>(P, 0), buf_inv<V>(P), P.deg.p, n, damping, P.ctl.p, P.blk_cnt.p,
      P.ktime.p);
  GBX_LAUNCHED();
  PrArgs<V> pa{};
  if (!option(kOptPrHostLoop) && persist_args<V>(P, damping, tol, itermax, pa)) {
    void* args[] = {&pa};
    GBX_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_pr_persist<V>),
                                         dim3(pa.grid_rows), dim3(kPrThreads), args, 0, s));
    P.last_persist = true;
    P.grid = pa.grid_rows;
  } else {
    // one row launch + one finish launch per iteration, checked on the host
    // every 4 iterations (the finish kernels of a converged run return at once)
    PrArgs<V> a = make_args<V>(P, damping, tol, itermax);
    int done = 0, launched = 0;
    while (!done && launched < itermax) {
      const int chunk = std::min(4, itermax - launched);
      for (int c = 0; c < chunk; ++c) {
        launch_rows<V>(a, s);
        k_pr_finish<V><<<P.grid_fin, kPrThreads, 0, s>>>(a);
        GBX_LAUNCHED();
      }
      launched += chunk;
      GBX_CUDA(cudaMemcpyAsync(&done, P.ctl.p + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
      GBX_CUDA(cudaStreamSynchronize(s));
    }
  }
  // ranks back in original vertex order (device-resident result; fp64),
  // queued behind the run before the host reads the counters back
  k_pr_unpermute<V><<<ceil_div(n, 256), 256, 0, s>>>(buf_r<V>(P, 0), buf_r<V>(P, 1), P.ctl.p,
                                                       P.new2old.p, n, P.out.p);
  GBX_LAUNCHED();
  int it = 0;
  std::vector<unsigned long long> kt(128 * 8);
  GBX_CUDA(cudaMemcpyAsync(&it, P.ctl.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaMemcpyAsync(kt.data(), P.ktime.p, kt.size() * 8, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  P.last_iters = it;
  {
    // mean row-phase duration over this run's iterations (first CTA start to
    // last CTA end, %globaltimer)
    double sum = 0.0;
    int cnt = 0;
    double ph[4] = {0, 0, 0, 0};
    for (int k = 0; k < std::min(it, 128); ++k) {
      const unsigned long long* t = &kt[8 * k];
      if (t[1] > t[0] && t[0] != ~0ull) {
        sum += static_cast<double>(t[1] - t[0]);
        ++cnt;
      }
      if (option(kOptPrTrace) && P.last_persist && t[2] != ~0ull && t[4] != ~0ull) {
        ph[0] += static_cast<double>(t[2] - t[1]);  // last row-phase CTA -> first past barrier 1
        ph[1] += static_cast<double>(t[3] - t[2]);  // long-row finish
        ph[2] += static_cast<double>(t[4] - t[3]);  // barrier 2
        ph[3] += static_cast<double>(t[5] - t[4]);  // L1 fold
      }
    }
    P.last_rows_ms = cnt ? sum / cnt * 1e-6 : 0.0;
    if (option(kOptPrTrace) && cnt && P.last_persist && it > 5 && P.cta_end.p) {
      // spread of the CTAs' row-phase end times in iteration 5 (static unit assignment)
      std::vector<unsigned long long> ce(P.grid);
      GBX_CUDA(cudaMemcpy(ce.data(), P.cta_end.p, ce.size() * 8, cudaMemcpyDeviceToHost));
      std::vector<double> d;
      for (unsigned long long t : ce) d.push_back(static_cast<double>(t - kt[8 * 5]) * 1e-3);
      std::sort(d.begin(), d.end());
      std::fprintf(stderr, "pagerank trace: CTA row-phase ends (iteration 5): min %.1f p10 %.1f p50 %.1f "
                           "p90 %.1f max %.1f us\n",
                   d.front(), d[d.size() / 10], d[d.size() / 2], d[d.size() * 9 / 10], d.back());
    }
    if (option(kOptPrTrace) && cnt)
      std::fprintf(stderr, "pagerank trace: grid %d, %d iterations, rows %.2f us, barrier1 %.2f us, finish "
                           "%.2f us, barrier2 %.2f us, fold %.2f us (means)\n",
                   P.grid, it, sum / cnt * 1e-3, ph[0] / cnt * 1e-3, ph[1] / cnt * 1e-3,
                   ph[2] / cnt * 1e-3, ph[3] / cnt * 1e-3);
  }
  if (iters) *iters = it;
  if (rank) {
    GBX_CUDA(cudaMemcpyAsync(rank, P.out.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaStreamSynchronize(s));
  }
  return it;
}

void pagerank_run(gbx_graph* g, double damping, double tol, int itermax, double* rank,
                  int* iters) {
  NvtxRange nvtx_("gbx.pagerank");
  require_at(g, "pagerank_gap");
  require_rowdeg(g, "pagerank_gap");
  if (!(damping > 0.0)) fail(GBX_NON_POSITIVE_DAMPING, "damping must be positive");
  const int64_t n = g->A.n;
  g->stats = gbx_stats{};
  g->pending_iters = nullptr;
  if (n == 0 || itermax <= 0) {
    // pagerank.cpp:52-75: iterations = min(k, itermax) with k = 1 when the loop
    // never runs, so a non-positive itermax comes back unchanged; n = 0 -> 0
    if (iters) *iters = n == 0 ? 0 : itermax;
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

// row blocks of the relabeled AT balanced by rows + nnz (merge-path split of
// the row-pointer prefix rp[0..n]); every rank computes the same bounds
std::vector<int64_t> pr_bounds(const int64_t* rp, int64_t n, int64_t nnz, int nranks) {
  auto split = [&](int q) -> int64_t {
    if (q <= 0) return 0;
    if (q >= nranks) return n;
    const int64_t target = (n + nnz) * q / nranks;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (mid + rp[mid] < target) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  std::vector<int64_t> bounds(nranks + 1, 0);
  for (int q = 1; q <= nranks; ++q) bounds[q] = std::max(bounds[q - 1], split(q));
  return bounds;
}

// the padded exchange layout + this rank's plan over its rows
static void pr_shard_finish(gbx_graph* g, std::unique_ptr<PrShard> S, int rank, int nranks,
                            const std::vector<int64_t>& bounds, int64_t* rb_out,
                            int64_t* re_out) {
  PrPlan& P = S->plan;
  S->bounds = bounds;
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
  // every rank computes the same bounds from the same relabeled AT
  const std::vector<int64_t> bounds = pr_bounds(rp.data(), P.n, P.nnz, nranks);
  pr_shard_finish(g, std::move(S), rank, nranks, bounds, rb_out, re_out);
}

// A shard from this rank's block of the RELABELED AT built by the distributed
// graph (mg.cu): rows [bounds[rank], bounds[rank+1]) of an n-row CSR whose
// other rows are empty, columns in new ids; deg = relabeled out-degree (n),
// new2old = the relabeling -- both identical on every rank.
void pr_shard_from_block(gbx_graph* g, int rank, int nranks, Csr& block, DevArray<int32_t>& deg,
                         DevArray<int32_t>& new2old, const std::vector<int64_t>& bounds) {
  auto S = std::make_unique<PrShard>();
  PrPlan& P = S->plan;
  P.n = block.n;
  P.nnz = block.nnz;
  P.trp = std::move(block.rp);
  P.tcol = std::move(block.col);
  P.deg = std::move(deg);
  P.new2old = std::move(new2old);
  pr_shard_finish(g, std::move(S), rank, nranks, bounds, nullptr, nullptr);
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
  NvtxRange nvtx_("gbx.pagerank.shard_step");
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
  a.nx = g->prs->chunk * g->prs->nranks;
  a.x1 = x_slice - P.row0;            // x_nxt[row] -> x_slice[row - row0]
  a.r0 = const_cast<float*>(r_prev);  // local rows; may alias r_new
  a.r1 = r_new;
  a.row0 = P.row0;
  a.grid_rows = resident_grid(reinterpret_cast<const void*>(k_pr_rows<float>));
  GBX_CUDA(cudaMemsetAsync(P.ctl.p, 0, 2 * sizeof(int), s));
  GBX_CUDA(cudaMemsetAsync(P.blk_cnt.p, 0, 16 * sizeof(unsigned), s));
  launch_rows<float>(a, s);
  k_pr_finish<float><<<P.grid_fin, kPrThreads, 0, s>>>(a);
  GBX_LAUNCHED();
  GBX_CUDA(cudaMemcpyAsync(l1, P.l1_hist.p, sizeof(double), cudaMemcpyDeviceToDevice, s));
  g->prs->steps++;
}

// per-rank arguments of the fused run: peers[q] = rank q's buffers
static void p2p_rank_args(gbx_graph* g, const uint64_t* x0_peers, const uint64_t* x1_peers,
                          const uint64_t* l1_peers, const uint64_t* sig_peers, float* r0,
                          float* r1, double damping, double tol, int itermax, PrArgs<float>& a,
                          PrP2p& m) {
  if (!g->prs) fail(GBX_MISSING_PROPERTY, "pr_shard_run_p2p needs gbx_pr_shard_prepare");
  PrShard& S = *g->prs;
  PrPlan& P = S.plan;
  if (S.nranks > kPrMaxPeers) fail(GBX_INVALID_VALUE, "pr_shard_run_p2p: more than 8 ranks");
  if (!x0_peers || !x1_peers || !l1_peers || !sig_peers || !r0 || !r1)
    fail(GBX_NULL_ARGUMENT, "pr_shard_run_p2p: NULL buffer");
  if (P.g_damping != damping) {
    k_pr_inv<<<ceil_div(std::max<int64_t>(P.n, 1), 256), 256, 0, g->stream>>>(P.invf.p, P.deg.p,
                                                                              P.n, damping);
    GBX_LAUNCHED();
    P.g_damping = damping;
  }
  a = make_args<float>(P, damping, tol, itermax);
  a.inv = P.invf.p;
  a.fixed = 0;
  a.row0 = P.row0;
  a.r0 = r0;
  a.r1 = r1;
  a.npeer = S.nranks;
  a.nx = S.chunk * S.nranks;
  const int64_t off = static_cast<int64_t>(S.rank) * S.chunk - P.row0;
  for (int q = 0; q < S.nranks; ++q) {
    a.xp[0][q] = reinterpret_cast<float*>(x0_peers[q]) + off;
    a.xp[1][q] = reinterpret_cast<float*>(x1_peers[q]) + off;
  }
  // the gathers read the local padded copy; x_nxt only selects the parity
  a.x0 = reinterpret_cast<float*>(x0_peers[S.rank]);
  a.x1 = reinterpret_cast<float*>(x1_peers[S.rank]);
  m = PrP2p{};
  for (int q = 0; q < S.nranks; ++q) {
    m.l1p[q] = reinterpret_cast<double*>(l1_peers[q]);
    m.sigp[q] = reinterpret_cast<unsigned*>(sig_peers[q]);
  }
  m.l1_own = m.l1p[S.rank];
  m.sig_own = m.sigp[S.rank];
  m.rank = S.rank;
  m.nranks = S.nranks;
  m.timeout_ns = static_cast<unsigned long long>(option(kOptP2pTimeoutMs)) * 1000000ull;
}

// after the run: iterations, or GBX_CUDA_ERROR when a peer never arrived
static int p2p_finish(gbx_graph* g) {
  PrPlan& P = g->prs->plan;
  int ctl[3] = {0, 0, 0};
  GBX_CUDA(cudaMemcpyAsync(ctl, P.ctl.p, sizeof ctl, cudaMemcpyDeviceToHost, g->stream));
  GBX_CUDA(cudaStreamSynchronize(g->stream));
  P.last_iters = ctl[0];
  if (ctl[2])
    fail(GBX_CUDA_ERROR, "pr_shard_run_p2p: a peer rank did not reach iteration " +
                             std::to_string(ctl[0]) + " within p2p.timeout_ms");
  return ctl[0];
}

void pr_shard_run_p2p(gbx_graph* g, const uint64_t* x0_peers, const uint64_t* x1_peers,
                      const uint64_t* l1_peers, const uint64_t* sig_peers, float* r0, float* r1,
                      double damping, double tol, int itermax, int* iters) {
  NvtxRange nvtx_("gbx.pagerank.fused_run");
  PrArgs<float> a{};
  PrP2p m{};
  p2p_rank_args(g, x0_peers, x1_peers, l1_peers, sig_peers, r0, r1, damping, tol, itermax, a, m);
  PrPlan& P = g->prs->plan;
  if (itermax <= 0 || P.n == 0) {  // as pagerank_run: nothing to iterate
    if (iters) *iters = P.n == 0 ? 0 : itermax;
    return;
  }
  a.grid_rows = resident_grid(reinterpret_cast<const void*>(k_pr_persist_p2p));
  if (static_cast<int64_t>(P.l1_fin.n) < a.grid_rows || static_cast<int64_t>(P.l1_block.n) < a.grid_rows)
    fail(GBX_CUDA_ERROR, "pr_shard_run_p2p: partial buffers too small");
  reset_state(g->stream, P);
  void* args[] = {&a, &m};
  GBX_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_pr_persist_p2p),
                                       dim3(a.grid_rows), dim3(kPrThreads), args, 0, g->stream));
  GBX_LAUNCHED();
  const int it = p2p_finish(g);
  if (iters) *iters = it;
}

// nv ranks emulated in ONE cooperative launch on one GPU (every shard's graph
// handle lives on this device): the multi-rank protocol -- peer stores, slot
// tables, signal counts, the cross-rank stop agreement -- with ranks that can
// never wait on a rank that is not running.  peers arrays are [nv] as above;
// r0s / r1s per rank.
void pr_shard_run_p2p_multi(gbx_graph* const* gs, int nv, const uint64_t* x0_peers,
                            const uint64_t* x1_peers, const uint64_t* l1_peers,
                            const uint64_t* sig_peers, float* const* r0s, float* const* r1s,
                            double damping, double tol, int itermax, int* iters) {
  NvtxRange nvtx_("gbx.pagerank.fused_run_multi");
  if (nv < 1 || nv > kPrMaxPeers) fail(GBX_INVALID_VALUE, "pr_shard_run_p2p_multi: 1..8 ranks");
  std::vector<PrArgs<float>> va(nv);
  std::vector<PrP2p> vm(nv);
  for (int v = 0; v < nv; ++v) {
    if (!gs[v] || !gs[v]->prs || gs[v]->prs->rank != v || gs[v]->prs->nranks != nv)
      fail(GBX_INVALID_VALUE, "pr_shard_run_p2p_multi: shard v must be rank v of nv");
    p2p_rank_args(gs[v], x0_peers, x1_peers, l1_peers, sig_peers, r0s[v], r1s[v], damping, tol,
                  itermax, va[v], vm[v]);
    GBX_CUDA(cudaStreamSynchronize(gs[v]->stream));
  }
  const int64_t n = gs[0]->prs->plan.n;
  if (itermax <= 0 || n == 0) {
    if (iters) *iters = n == 0 ? 0 : itermax;
    return;
  }
  const int per = resident_grid(reinterpret_cast<const void*>(k_pr_persist_p2p_virt)) / nv;
  if (per < 1) fail(GBX_CUDA_ERROR, "pr_shard_run_p2p_multi: too many ranks for one launch");
  for (int v = 0; v < nv; ++v) {
    PrPlan& P = gs[v]->prs->plan;
    va[v].grid_rows = per;
    if (static_cast<int64_t>(P.l1_fin.n) < per || static_cast<int64_t>(P.l1_block.n) < per)
      fail(GBX_CUDA_ERROR, "pr_shard_run_p2p_multi: partial buffers too small");
    reset_state(gs[0]->stream, P);
  }
  cudaStream_t s = gs[0]->stream;
  Tmp<PrArgs<float>> da(nv, s);
  Tmp<PrP2p> dm(nv, s);
  GBX_CUDA(cudaMemcpyAsync(da.p, va.data(), nv * sizeof(PrArgs<float>), cudaMemcpyHostToDevice, s));
  GBX_CUDA(cudaMemcpyAsync(dm.p, vm.data(), nv * sizeof(PrP2p), cudaMemcpyHostToDevice, s));
  const PrArgs<float>* pa = da.p;
  const PrP2p* pm = dm.p;
  void* args[] = {&pa, &pm, &nv};
  GBX_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_pr_persist_p2p_virt),
                                       dim3(per * nv), dim3(kPrThreads), args, 0, s));
  GBX_LAUNCHED();
  GBX_CUDA(cudaStreamSynchronize(s));
  int it0 = -1;
  for (int v = 0; v < nv; ++v) {
    const int it = p2p_finish(gs[v]);
    if (it0 >= 0 && it != it0) fail(GBX_CUDA_ERROR, "pr_shard_run_p2p_multi: ranks disagree on the iteration count");
    it0 = it;
  }
  if (iters) *iters = it0;
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
