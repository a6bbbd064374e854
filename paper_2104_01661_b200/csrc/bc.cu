// bc.cu -- batched Brandes betweenness (algo/betweenness.cpp:11-86).
//
// The reference keeps ns x n matrices P (path counts), one boolean pattern per
// BFS level and B = 1 + dependency, and runs Gustavson mxm per level forward
// (F<!s(P)> = F plus.first A) and backward (W<s(S[i-1])> = W plus.first AT)
// (betweenness.cpp:27-72).  On the device the batch rows become 4 lanes of a
// vertex-major layout:
//   level[v][4]  int32 exact BFS depth per lane (-1 unreached)
//   lv8[v]       uint32, one byte per lane = min(depth, 254), 0xFF unreached
//   map[v/8]     level map: 4 bits per vertex = membership of ONE depth; the
//                word every edge gathers (8 MB at scale 24, L2-resident) --
//                depth d-1 in the forward pull, depth d+1 in the backward
//   sigma[v][4]  fp64 path counts (integers < 2^53: sums are exact in any order)
//   coef[v][4]   fp64 (1 + delta) / sigma once v's level is final
// Forward, level d (direction-optimizing like the BFS, results identical):
//   push (small frontier): (vertex, <=kBcChunk-edge) entries of level d-1; a
//     lane claims an unreached neighbour with atomicCAS on its level word and
//     adds sigma with fp64 atomicAdd;
//   pull (frontier edges >= nnz/alpha): every vertex still unreached in a live
//     lane sums sigma over its in-neighbours on level d-1 (AT rows, no atomics);
//     only vertices a previous pull left unreached are rescanned; rows longer
//     than kBcHeavy are split into chunks summed with atomics by a side pass.
// Backward, level d = D-1..1: for u on level d, acc_b = sum over out-neighbours
//   v on level d+1 of coef_b(v); delta_b(u) = sigma_b(u) * acc_b, centrality(u)
//   += delta_b(u), coef_b(u) = (1 + delta_b(u)) / sigma_b(u) -- finalised in the
//   same pass for ordinary rows, by a side pass for chunked hub rows.
// centrality(j) = sum_b (B(b,j) - 1) = sum_b delta_b(j) (betweenness.cpp:74-79);
// sources and unreached vertices contribute 0, undirected pairs not halved.
// Algorithmic bytes per batch: E_r*(8 + 16*ns) + V_r*(16 + 24*ns).
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "plans.cuh"
#include "warpqueue.cuh"

namespace gbx {

constexpr int kBcLanes = 4;
constexpr int64_t kBcChunk = 256;    // push entries: edges per warp
#ifndef GBX_BC_HEAVY
#define GBX_BC_HEAVY 2048
#endif
#ifndef GBX_BC_HCHUNK
#define GBX_BC_HCHUNK 1024
#endif
constexpr int64_t kBcHeavy = GBX_BC_HEAVY;    // rows longer than this are chunked
constexpr int64_t kBcHChunk = GBX_BC_HCHUNK;  // edges per hub-row chunk
constexpr int kBcBuf = 256;
constexpr unsigned kAll = 0xffffffffu;

__device__ __forceinline__ int bc_chunks(int64_t deg) {
  return deg <= kBcChunk ? 1 : static_cast<int>((deg + kBcChunk - 1) / kBcChunk);
}

// lane b of lv8 word x is on depth L (exact: depths >= 254 share byte 254)
__device__ __forceinline__ bool on_level(uint32_t x, int b, int L, const int32_t* level,
                                         int64_t v) {
  const uint32_t byte = (x >> (8 * b)) & 0xFFu;
  if (L < 254) return byte == static_cast<uint32_t>(L);
  return byte == 254u && level[v * 4 + b] == L;
}

__device__ __forceinline__ unsigned lanes_on(uint32_t x, int L, unsigned lanes,
                                             const int32_t* level, int64_t v) {
  unsigned m = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b)
    if (((lanes >> b) & 1u) && on_level(x, b, L, level, v)) m |= 1u << b;
  return m;
}

__device__ __forceinline__ unsigned lanes_unreached(uint32_t x, unsigned lanes) {
  unsigned m = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b)
    if (((x >> (8 * b)) & 0xFFu) == 0xFFu) m |= 1u << b;
  return m & lanes;
}

__device__ __forceinline__ uint32_t lv8_byte(int d) { return d < 254 ? d : 254; }

// Level maps: 4 bits per vertex (one per lane), 8 vertices per word -- the
// membership of ONE depth (8 MB at scale 24, L2-resident), gathered per edge
// in place of the 64 MB lv8 array.
__device__ __forceinline__ unsigned nib(const uint32_t* map, int64_t v) {
  return (__ldg(map + (v >> 3)) >> ((v & 7) * 4)) & 0xFu;
}
__device__ __forceinline__ void nib_or(uint32_t* map, int64_t v, unsigned m) {
  atomicOr(map + (v >> 3), m << ((v & 7) * 4));
}

// streamed column index (no L1 allocation: L1 is kept for the map words)
__device__ __forceinline__ int32_t ld_col(const int32_t* p) {
  int32_t v;
  asm("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// val[v][0..3] (32 bytes, sector-aligned) in one 256-bit read-only load
__device__ __forceinline__ void ld_sector(const double* p, double x[4]) {
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(x[0]), "=d"(x[1]), "=d"(x[2]), "=d"(x[3])
      : "l"(p));
}

// s[b] += val[u][b] over the row entries p, p+st, ... < e whose map nibble is
// in m; U independent column loads, then U map gathers, per step (the chain
// col -> map -> val is latency-bound, so each lane keeps U in flight)
template <int U>
__device__ __forceinline__ void row_sum(const int32_t* col, int64_t n, int64_t p, int64_t e, int st,
                                        const uint32_t* map, const double* val, unsigned m,
                                        double s[4]) {
  for (; p < e; p += U * st) {
    int32_t u[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      u[k] = p + k * st < e ? ld_col(col + p + k * st) : -1;
      GBX_DCHECK(u[k] < n, "bc column", u[k]);
    }
    unsigned h[U];
#pragma unroll
    for (int k = 0; k < U; ++k) h[k] = u[k] >= 0 ? (nib(map, u[k]) & m) : 0u;
#pragma unroll
    for (int k = 0; k < U; ++k)
      if (h[k]) {
        // the vertex's 4 lanes are one 32-byte sector: one 256-bit load
        double x[4];
        ld_sector(val + static_cast<int64_t>(u[k]) * 4, x);
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if ((h[k] >> b) & 1u) s[b] += x[b];
      }
  }
}

__device__ __forceinline__ void group_reduce(double s[4]) {
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    s[b] += __shfl_xor_sync(0xffffffffu, s[b], 4);
    s[b] += __shfl_xor_sync(0xffffffffu, s[b], 2);
    s[b] += __shfl_xor_sync(0xffffffffu, s[b], 1);
  }
}

__device__ __forceinline__ void warp_reduce(double s[4]) {
#pragma unroll
  for (int b = 0; b < 4; ++b)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s[b] += __shfl_xor_sync(0xffffffffu, s[b], o);
}

#ifndef GBX_BC_UNROLL
#define GBX_BC_UNROLL 8  // on the degree-sorted copy, 4 CTAs/SM: 4 / 6 / 8 / 10 / 12 / 16 -> 10.03 / 9.98 / 9.69 / 9.92 / 10.17 / 10.47 ms (scale 24, batch of 4)
#endif
constexpr int kBcUnroll = GBX_BC_UNROLL;  // loads in flight per lane, group/hub rows
#ifndef GBX_BC_MINB
#define GBX_BC_MINB 4  // on the degree-sorted copy: 3 / 4 / 5 / 6 -> 10.7 / 10.03 / 10.3 / 11.2 ms
#endif
constexpr int kBcMinBlocks = GBX_BC_MINB;  // resident 256-thread blocks per SM asked of ptxas

// Row-length bins: rows of a list are partitioned (2-bit radix sort, stable)
// so a warp step handles rows of one shape -- bin 0 (<= kBin0 edges): one
// row per lane; bin 1 (<= kBin1): 8-lane groups, 4 rows per warp; bin 2
// (<= kBcHeavy): one row per warp; bin 3 (hubs): the chunked side passes.
#ifndef GBX_BC_BIN0
#define GBX_BC_BIN0 16  // on the degree-sorted copy (scale 24): 4 / 8 / 16 -> 8.38 / 8.13 / 8.03 ms
#endif
#ifndef GBX_BC_BIN1
#define GBX_BC_BIN1 256  // 32 / 64 / 128 / 256 / 512 -> 8.17 / 8.13 / 7.77 / 7.61 / 7.60 ms; with bin 0 <= 16 and 1024-edge hub chunks: 7.52
#endif
constexpr int64_t kBin0 = GBX_BC_BIN0, kBin1 = GBX_BC_BIN1;
__device__ __forceinline__ uint8_t deg_bin(int64_t deg) {
  return deg <= kBin0 ? 0 : deg <= kBin1 ? 1 : deg <= kBcHeavy ? 2 : 3;
}
struct BcBins {
  const int32_t* list;  // [bin 0 | bin 1 | bin 2 | bin 3]
  const int* cnt;       // device: sizes of bins 0..3
};

struct BcArgs {
  const int64_t* rp;   // A
  const int32_t* col;
  const int64_t* trp;  // AT
  const int32_t* tcol;
  int64_t n;
  int32_t* level;
  uint32_t* lv8;
  double* sigma;
  double* coef;
  double* cent;
  double* hacc;          // [nheavy][4] hub-row partial sums (zero between uses)
  double* bacc;          // [n][4] backward push sums (zero between uses)
  int32_t* mark;         // push: last level that listed the vertex
  int32_t* list_out;     // vertices of the level being built
  const int32_t* list_in;
  int n_list;
  const int64_t* ent_in;
  int64_t* ent_out;
  int n_ent;
  const int32_t* ul_in;  // pull: vertices still unreached (-1 count: all)
  int32_t* ul_out;
  int ul_cnt;
  const int32_t* hv;     // hub rows (slot -> vertex) and their chunks (chunk<<32|slot)
  const int64_t* hent;
  int nhv, nhent;
  BcBins bins;             // pull: still-unreached vertices / back: level-d list
  const uint32_t* map_in;  // level map of depth d-1 (forward) / d+1 (backward)
  uint32_t* map_out;       // forward: level map of depth d being built
  int* cnt;  // [0] list [1] entries [2] unreached list [3] lanes discovered
  unsigned long long* edges;  // frontier edges of the level being built
  int d;
  unsigned lanes;  // lanes still live (their previous level was non-empty)
  int64_t own0, own1;  // vertices this rank finalises (sharded BC; else [0, n))
  const uint8_t* cand;  // candidate levels of the sharded forward: only these hubs (else NULL)
};

// forward push over A from the entries of level d-1
__global__ void __launch_bounds__(256) k_bc_push(BcArgs a) {
  __shared__ int32_t s_buf[8][kBcBuf];
  __shared__ int32_t s_kbuf[8][kBcBuf];
  __shared__ __align__(8) int s_red[8];
  FrontierQueue<kBcBuf> fq;
  fq.buf = s_buf[threadIdx.x >> 5];
  fq.rp = a.rp;
  fq.chunk = kBcChunk;
  fq.reset(a.ent_out, &a.cnt[1], &a.cnt[0], a.edges, a.list_out);
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int d = a.d;
  unsigned found = 0;
  // small queues: every entry split over S warps (S a power of two <= 8)
  int S = 1;
  while (S < 8 && static_cast<int64_t>(a.n_ent) * S * 2 <= nwarps) S <<= 1;
  const int64_t sub = kBcChunk / S;
  for (int64_t e2 = gwarp; e2 < static_cast<int64_t>(a.n_ent) * S; e2 += nwarps) {
    const int64_t e = e2 / S;
    const int part = static_cast<int>(e2 - e * S);
    const int64_t ent = a.ent_in[e];
    const int32_t u = static_cast<int32_t>(ent & 0xffffffff);
    const int64_t c = ent >> 32;
    const unsigned m = lanes_on(a.lv8[u], d - 1, a.lanes, a.level, u);
    double su[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) su[b] = (m >> b) & 1u ? a.sigma[static_cast<int64_t>(u) * 4 + b] : 0.0;
    const int64_t cb = a.rp[u] + c * kBcChunk;
    const int64_t ce = min(a.rp[u + 1], cb + kBcChunk);
    const int64_t b0 = cb + part * sub;
    const int64_t e0 = min(ce, b0 + sub);
    for (int64_t base = b0; base < e0; base += 32) {
      const int64_t p = base + lane;
      bool claimed = false;
      int32_t v = 0;
      if (p < e0 && m) {
        v = __ldg(a.col + p);
        GBX_DCHECK(v >= 0 && v < a.n, "bc push column", v);
        int32_t* lvp = a.level + static_cast<int64_t>(v) * 4;
        // the lv8 word (L2-resident) filters out the lanes where v is already
        // settled on an earlier depth before touching the int32 level words
        const uint32_t x = *(volatile uint32_t*)&a.lv8[v];
        const uint32_t db = lv8_byte(d);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          if (!((m >> b) & 1u)) continue;
          const uint32_t xb = (x >> (8 * b)) & 0xFFu;
          if (xb != 0xFFu && xb != db) continue;
          int lv = *(volatile int32_t*)&lvp[b];
          if (lv == -1) {
            lv = atomicCAS(&lvp[b], -1, d);
            if (lv == -1) {
              claimed = true;
              lv = d;
              found |= 1u << b;
              atomicAnd(&a.lv8[v], ~((0xFFu ^ lv8_byte(d)) << (8 * b)));
              nib_or(a.map_out, v, 1u << b);
            }
          }
          if (lv == d) atomicAdd(&a.sigma[static_cast<int64_t>(v) * 4 + b], su[b]);
        }
      }
      const bool has = claimed && atomicExch(&a.mark[v], d) != d;
      fq.push(has, v);
    }
  }
  fq.flush_block(s_kbuf[threadIdx.x >> 5], s_red);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) found |= __shfl_xor_sync(kAll, found, o);
  if (lane == 0 && found) atomicOr(&a.cnt[3], static_cast<int>(found));
}

// forward pull over AT for the vertices still unreached in a live lane
// settle vertex v with path-count sums s for the unreached live lanes um
__device__ __forceinline__ unsigned bc_settle(const BcArgs& a, int64_t v, unsigned um,
                                              const double s[4]) {
  unsigned nm = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b)
    if (((um >> b) & 1u) && s[b] > 0.0) nm |= 1u << b;
  if (nm) {
    uint32_t x = a.lv8[v];
#pragma unroll
    for (int b = 0; b < 4; ++b)
      if ((nm >> b) & 1u) {
        a.level[v * 4 + b] = a.d;
        a.sigma[v * 4 + b] = s[b];
        x = (x & ~(0xFFu << (8 * b))) | (lv8_byte(a.d) << (8 * b));
      }
    a.lv8[v] = x;
    nib_or(a.map_out, v, nm);
  }
  return nm;
}

__global__ void __launch_bounds__(256, kBcMinBlocks) k_bc_pull(BcArgs a) {
  __shared__ int32_t s_buf[8][kBcBuf];
  __shared__ int32_t s_ubuf[8][kBcBuf];
  __shared__ int32_t s_kbuf[8][kBcBuf];
  __shared__ __align__(8) int s_red[8];
  FrontierQueue<kBcBuf> fq;
  fq.buf = s_buf[threadIdx.x >> 5];
  fq.rp = a.rp;
  fq.chunk = kBcChunk;
  fq.reset(a.ent_out, &a.cnt[1], &a.cnt[0], a.edges, a.list_out);
  WarpQueue<int32_t, kBcBuf> uq;
  uq.buf = s_ubuf[threadIdx.x >> 5];
  uq.reset(a.ul_out, &a.cnt[2]);
  const int lane = threadIdx.x & 31;
  const int grp = lane >> 3, sub = lane & 7;
  const int64_t gwarp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int32_t* L = a.bins.list;
  const int n0 = a.bins.cnt[0], n1 = a.bins.cnt[1], n2 = a.bins.cnt[2];
  const int64_t s0 = (n0 + 31) / 32, s1 = (n1 + 3) / 4, tot = s0 + s1 + n2;
  unsigned found = 0;
  for (int64_t t = gwarp; t < tot; t += nwarps) {
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    if (t < s0) {  // bin 0: a row per lane
      const int64_t i = t * 32 + lane;
      const int64_t v = i < n0 ? L[i] : -1;
      unsigned um = 0, nm = 0;
      int64_t pp = 0, pe = 0;
      if (v >= 0) {
        um = lanes_unreached(a.lv8[v], a.lanes);
        if (um) {
          pp = a.trp[v];
          pe = a.trp[v + 1];
          row_sum<4>(a.tcol, a.n, pp, pe, 1, a.map_in, a.sigma, um, s);
          nm = bc_settle(a, v, um, s);
          found |= nm;
        }
      }
      fq.push(nm != 0, static_cast<int32_t>(v));
      uq.push(pe > pp && (um & ~nm) != 0, static_cast<int32_t>(v));
    } else if (t < s0 + s1) {  // bin 1: 8 lanes per row
      const int64_t i = n0 + (t - s0) * 4 + grp;
      const int64_t v = i < n0 + n1 ? L[i] : -1;
      const unsigned um = v >= 0 ? lanes_unreached(a.lv8[v], a.lanes) : 0u;
      if (um) row_sum<kBcUnroll>(a.tcol, a.n, a.trp[v] + sub, a.trp[v + 1], 8, a.map_in, a.sigma, um, s);
      group_reduce(s);
      unsigned nm = 0;
      if (sub == 0 && um) {
        nm = bc_settle(a, v, um, s);
        found |= nm;
      }
      fq.push(nm != 0, static_cast<int32_t>(v));
      uq.push(sub == 0 && (um & ~nm) != 0, static_cast<int32_t>(v));
    } else {  // bin 2: a warp per row
      const int64_t v = L[n0 + n1 + (t - s0 - s1)];
      const unsigned um = lanes_unreached(a.lv8[v], a.lanes);
      if (um) row_sum<kBcUnroll>(a.tcol, a.n, a.trp[v] + lane, a.trp[v + 1], 32, a.map_in, a.sigma, um, s);
      warp_reduce(s);
      unsigned nm = 0;
      if (lane == 0 && um) {
        nm = bc_settle(a, v, um, s);
        found |= nm;
      }
      fq.push(nm != 0, static_cast<int32_t>(v));
      uq.push(lane == 0 && (um & ~nm) != 0, static_cast<int32_t>(v));
    }
  }
  fq.flush_block(s_kbuf[threadIdx.x >> 5], s_red);
  uq.flush();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) found |= __shfl_xor_sync(kAll, found, o);
  if (lane == 0 && found) atomicOr(&a.cnt[3], static_cast<int>(found));
}

// forward pull, hub rows: one warp per chunk, partial sums into hacc[slot]
__global__ void __launch_bounds__(256, kBcMinBlocks) k_bc_pull_hub(BcArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t e = gwarp; e < a.nhent; e += nwarps) {
    const int64_t ent = a.hent[e];
    const int slot = static_cast<int>(ent & 0xffffffff);
    const int64_t c = ent >> 32;
    const int32_t v = a.hv[slot];
    if (a.cand && !a.cand[v]) continue;  // no frontier in-neighbour: nothing to sum
    const unsigned um = lanes_unreached(a.lv8[v], a.lanes);
    if (!um) continue;
    const int64_t b0 = a.trp[v] + c * kBcHChunk;
    const int64_t e0 = min(a.trp[v + 1], b0 + kBcHChunk);
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    row_sum<kBcUnroll>(a.tcol, a.n, b0 + lane, e0, 32, a.map_in, a.sigma, um, s);
    warp_reduce(s);
    if (lane < 4 && ((um >> lane) & 1u)) {
      const double mine = lane == 0 ? s[0] : lane == 1 ? s[1] : lane == 2 ? s[2] : s[3];
      if (mine != 0.0) atomicAdd(&a.hacc[slot * 4 + lane], mine);
    }
  }
}

// forward pull, hub rows: settle the summed hubs, one warp per 32 slots
__global__ void __launch_bounds__(256) k_bc_pull_hub_fin(BcArgs a) {
  __shared__ int32_t s_buf[8][kBcBuf];
  FrontierQueue<kBcBuf> fq;
  fq.buf = s_buf[threadIdx.x >> 5];
  fq.rp = a.rp;
  fq.chunk = kBcChunk;
  fq.reset(a.ent_out, &a.cnt[1], &a.cnt[0], a.edges, a.list_out);
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int d = a.d;
  unsigned found = 0;
  for (int64_t base = gwarp * 32; base < a.nhv; base += nwarps * 32) {
    const int64_t slot = base + lane;
    bool has = false, still = false;
    int32_t v = 0;
    if (slot < a.nhv) {
      v = a.hv[slot];
      uint32_t x = a.lv8[v];
      const unsigned um = lanes_unreached(x, a.lanes);
      unsigned nm = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const double sb = a.hacc[slot * 4 + b];
        if (((um >> b) & 1u) && sb > 0.0) {
          nm |= 1u << b;
          a.level[static_cast<int64_t>(v) * 4 + b] = d;
          a.sigma[static_cast<int64_t>(v) * 4 + b] = sb;
          x = (x & ~(0xFFu << (8 * b))) | (lv8_byte(d) << (8 * b));
        }
        if (sb != 0.0) a.hacc[slot * 4 + b] = 0.0;
      }
      if (nm) {
        a.lv8[v] = x;
        nib_or(a.map_out, v, nm);
        found |= nm;
        has = true;
      }
      still = (um & ~nm) != 0;
    }
    fq.push(has, v);
    // hubs still unreached in a live lane: while there are none, the next
    // pulls skip the hub passes (a walk over every hub chunk otherwise)
    const unsigned sb = __ballot_sync(kAll, still);
    if (lane == 0 && sb) atomicAdd(&a.cnt[6], __popc(sb));
  }
  fq.flush();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) found |= __shfl_xor_sync(kAll, found, o);
  if (lane == 0 && found) atomicOr(&a.cnt[3], static_cast<int>(found));
}

// backward for the level-d list over A rows (hub rows skipped), finalised inline
__device__ __forceinline__ void bc_final(const BcArgs& a, int64_t u, unsigned m,
                                         const double acc[4]) {
  double c = 0.0;
#pragma unroll
  for (int b = 0; b < 4; ++b)
    if ((m >> b) & 1u) {
      const double sg = a.sigma[u * 4 + b];
      const double dl = sg * acc[b];
      c += dl;
      a.coef[u * 4 + b] = (1.0 + dl) / sg;
    }
  a.cent[u] += c;
}

__global__ void __launch_bounds__(256, kBcMinBlocks) k_bc_back(BcArgs a) {
  const int lane = threadIdx.x & 31;
  const int grp = lane >> 3, sub = lane & 7;
  const int64_t gwarp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int32_t* L = a.bins.list;
  const int n0 = a.bins.cnt[0], n1 = a.bins.cnt[1], n2 = a.bins.cnt[2];
  const int64_t s0 = (n0 + 31) / 32, s1 = (n1 + 3) / 4, tot = s0 + s1 + n2;
  for (int64_t t = gwarp; t < tot; t += nwarps) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    if (t < s0) {  // bin 0: a row per lane
      const int64_t i = t * 32 + lane;
      if (i < n0) {
        const int64_t u = L[i];
        const unsigned m = lanes_on(a.lv8[u], a.d, a.lanes, a.level, u);
        if (m) {
          row_sum<4>(a.col, a.n, a.rp[u], a.rp[u + 1], 1, a.map_in, a.coef, m, acc);
          bc_final(a, u, m, acc);
        }
      }
    } else if (t < s0 + s1) {  // bin 1: 8 lanes per row
      const int64_t i = n0 + (t - s0) * 4 + grp;
      const int64_t u = i < n0 + n1 ? L[i] : -1;
      const unsigned m = u >= 0 ? lanes_on(a.lv8[u], a.d, a.lanes, a.level, u) : 0u;
      if (m) row_sum<kBcUnroll>(a.col, a.n, a.rp[u] + sub, a.rp[u + 1], 8, a.map_in, a.coef, m, acc);
      group_reduce(acc);
      if (sub == 0 && m) bc_final(a, u, m, acc);
    } else {  // bin 2: a warp per row
      const int64_t u = L[n0 + n1 + (t - s0 - s1)];
      const unsigned m = lanes_on(a.lv8[u], a.d, a.lanes, a.level, u);
      if (m) row_sum<kBcUnroll>(a.col, a.n, a.rp[u] + lane, a.rp[u + 1], 32, a.map_in, a.coef, m, acc);
      warp_reduce(acc);
      if (lane == 0 && m) bc_final(a, u, m, acc);
    }
  }
}

// backward, hub rows of A: one warp per chunk, partial sums into hacc[slot]
__global__ void __launch_bounds__(256, kBcMinBlocks) k_bc_back_hub(BcArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int d = a.d;
  for (int64_t e = gwarp; e < a.nhent; e += nwarps) {
    const int64_t ent = a.hent[e];
    const int slot = static_cast<int>(ent & 0xffffffff);
    const int64_t c = ent >> 32;
    const int32_t u = a.hv[slot];
    const unsigned m = lanes_on(a.lv8[u], d, a.lanes, a.level, u);
    if (!m) continue;
    const int64_t b0 = a.rp[u] + c * kBcHChunk;
    const int64_t e0 = min(a.rp[u + 1], b0 + kBcHChunk);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    row_sum<kBcUnroll>(a.col, a.n, b0 + lane, e0, 32, a.map_in, a.coef, m, acc);
    warp_reduce(acc);
    if (lane < 4 && ((m >> lane) & 1u)) {
      const double mine = lane == 0 ? acc[0] : lane == 1 ? acc[1] : lane == 2 ? acc[2] : acc[3];
      if (mine != 0.0) atomicAdd(&a.hacc[slot * 4 + lane], mine);
    }
  }
}

__global__ void k_bc_back_hub_fin(BcArgs a) {
  const int64_t slot = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (slot >= a.nhv) return;
  const int64_t u = a.hv[slot];
  if (u < a.own0 || u >= a.own1) return;  // another rank's hub
  const unsigned m = lanes_on(a.lv8[u], a.d, a.lanes, a.level, u);
  double c = 0.0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const double ab = a.hacc[slot * 4 + b];
    if ((m >> b) & 1u) {
      const double sg = a.sigma[u * 4 + b];
      const double dl = sg * ab;
      c += dl;
      a.coef[u * 4 + b] = (1.0 + dl) / sg;
    }
    if (ab != 0.0) a.hacc[slot * 4 + b] = 0.0;
  }
  if (m) a.cent[u] += c;
}

// Backward in PUSH form (depth d from depth d+1): the children list (depth
// d+1, binned by in-degree) adds every child's finished coefficient into
// bacc[v] of its depth-d in-neighbours v (fp64 atomics, map_in = level map of
// depth d); k_bc_back_fin then finalises the depth-d list from bacc and
// re-zeroes it.  The children's rows hold far fewer edges than the parents'
// once the BFS is past its hub levels (scale 24: depth 4 has 25 M edges, depth
// 3 has 100 M), so this scans less than the pull form above.
__device__ __forceinline__ void push_row(const BcArgs& a, int64_t p, int64_t e, int st, unsigned mw,
                                         const double cw[4]) {
  for (; p < e; p += kBcUnroll * st) {
    int32_t v[kBcUnroll];
#pragma unroll
    for (int k = 0; k < kBcUnroll; ++k) {
      v[k] = p + k * st < e ? ld_col(a.tcol + p + k * st) : -1;
      GBX_DCHECK(v[k] < a.n, "bc back-push column", v[k]);
    }
    unsigned h[kBcUnroll];
#pragma unroll
    for (int k = 0; k < kBcUnroll; ++k) h[k] = v[k] >= 0 ? (nib(a.map_in, v[k]) & mw) : 0u;
#pragma unroll
    for (int k = 0; k < kBcUnroll; ++k)
      if (h[k]) {
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if ((h[k] >> b) & 1u) atomicAdd(&a.bacc[static_cast<int64_t>(v[k]) * 4 + b], cw[b]);
      }
  }
}

__global__ void __launch_bounds__(256, kBcMinBlocks) k_bc_back_push(BcArgs a) {
  const int lane = threadIdx.x & 31;
  const int grp = lane >> 3, sub = lane & 7;
  const int64_t gwarp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int32_t* L = a.bins.list;
  const int n0 = a.bins.cnt[0], n1 = a.bins.cnt[1], n23 = a.bins.cnt[2] + a.bins.cnt[3];
  const int64_t s0 = (n0 + 31) / 32, s1 = (n1 + 3) / 4, tot = s0 + s1 + n23;
  const int dc = a.d + 1;  // the children's depth
  for (int64_t t = gwarp; t < tot; t += nwarps) {
    int64_t w = -1;
    int64_t p = 0, e = 0;
    int st = 1;
    if (t < s0) {  // a row per lane
      const int64_t i = t * 32 + lane;
      if (i < n0) w = L[i];
      if (w >= 0) { p = a.trp[w]; e = a.trp[w + 1]; }
    } else if (t < s0 + s1) {  // 8 lanes per row
      const int64_t i = n0 + (t - s0) * 4 + grp;
      if (i < n0 + n1) w = L[i];
      if (w >= 0) { p = a.trp[w] + sub; e = a.trp[w + 1]; }
      st = 8;
    } else {  // a warp per row (hub rows too: few children are hubs)
      w = L[n0 + n1 + (t - s0 - s1)];
      p = a.trp[w] + lane;
      e = a.trp[w + 1];
      st = 32;
    }
    if (w < 0) continue;
    const unsigned mw = lanes_on(a.lv8[w], dc, a.lanes, a.level, w);
    if (!mw) continue;
    double cw[4];
    ld_sector(a.coef + w * 4, cw);
    push_row(a, p, e, st, mw, cw);
  }
}

__global__ void k_bc_back_fin(BcArgs a) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= a.n_list) return;
  const int64_t u = a.list_in[i];
  const unsigned m = lanes_on(a.lv8[u], a.d, a.lanes, a.level, u);
  double acc[4];
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    acc[b] = a.bacc[u * 4 + b];
    if (acc[b] != 0.0) a.bacc[u * 4 + b] = 0.0;
  }
  if (m) bc_final(a, u, m, acc);
}

// level map of depth d from its list (backward)
__global__ void k_bc_map(const int32_t* list, int nlist, int d, unsigned lanes,
                         const int32_t* level, const uint32_t* lv8, uint32_t* map) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= nlist) return;
  const int64_t v = list[i];
  const unsigned m = lanes_on(lv8[v], d, lanes, level, v);
  if (m) nib_or(map, v, m);
}

// deepest level: delta = 0, coef = 1 / sigma
__global__ void k_bc_leaf(const int32_t* list, int nlist, int d, unsigned lanes,
                          const int32_t* level, const uint32_t* lv8, const double* sigma,
                          double* coef) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= nlist) return;
  const int64_t u = list[i];
  const unsigned m = lanes_on(lv8[u], d, lanes, level, u);
  for (int b = 0; b < 4; ++b)
    if ((m >> b) & 1u) coef[u * 4 + b] = 1.0 / sigma[u * 4 + b];
}

__global__ void k_bc_init(int32_t* level, uint32_t* lv8, double* sigma, int32_t* mark,
                          int64_t n) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n * 4) { level[i] = -1; sigma[i] = 0.0; }
  if (i < n) { mark[i] = -1; lv8[i] = 0xFFFFFFFFu; }
}

__global__ void k_bc_seed(const int32_t* src, int ns, int32_t* level, uint32_t* lv8,
                          double* sigma, int32_t* mark, int32_t* list, int64_t* ent, int* cnt,
                          unsigned long long* edges, const int64_t* rp, uint32_t* map) {
  int nl = 0, ne = 0;
  unsigned long long fe = 0;
  for (int b = 0; b < ns; ++b) {
    const int64_t s = src[b];
    level[s * 4 + b] = 0;
    sigma[s * 4 + b] = 1.0;
    lv8[s] &= ~(0xFFu << (8 * b));
    map[s >> 3] |= (1u << b) << ((s & 7) * 4);
    if (mark[s] != 0) {
      mark[s] = 0;
      list[nl++] = static_cast<int32_t>(s);
      const int64_t deg = rp[s + 1] - rp[s];
      fe += static_cast<unsigned long long>(deg);
      const int k = bc_chunks(deg);
      for (int c = 0; c < k; ++c) ent[ne++] = (static_cast<int64_t>(c) << 32) | s;
    }
  }
  cnt[0] = nl;
  cnt[1] = ne;
  cnt[2] = 0;
  cnt[3] = (1 << ns) - 1;
  *edges = fe;
}

// hub rows (degree > kBcHeavy) of a CSR and their kBcHChunk-edge chunks
__global__ void k_bc_hubs(const int64_t* rp, int64_t n, int32_t* hv, int64_t* hent, int* cnt) {
  int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (v >= n) return;
  const int64_t deg = rp[v + 1] - rp[v];
  if (deg <= kBcHeavy) return;
  const int slot = atomicAdd(&cnt[0], 1);
  hv[slot] = static_cast<int32_t>(v);
  const int k = static_cast<int>((deg + kBcHChunk - 1) / kBcHChunk);
  const int off = atomicAdd(&cnt[1], k);
  for (int c = 0; c < k; ++c) hent[off + c] = (static_cast<int64_t>(c) << 32) | slot;
}

// keys = row-length bin of each listed vertex (list == nullptr: 0..n-1, also
// written to iota); cnt[0..3] += bin sizes (block-aggregated: one atomic per
// bin per block)
__global__ void __launch_bounds__(256) k_bc_bin_keys(const int32_t* list, int64_t n,
                                                     const int64_t* rp, uint8_t* keys,
                                                     int32_t* iota, int* cnt) {
  __shared__ int s_cnt[4];
  if (threadIdx.x < 4) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = blockIdx.x * int64_t(blockDim.x); i0 < n; i0 += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    int k = -1;
    if (i < n) {
      const int64_t v = list ? list[i] : i;
      if (!list) iota[i] = static_cast<int32_t>(i);
      k = deg_bin(rp[v + 1] - rp[v]);
      keys[i] = static_cast<uint8_t>(k);
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const unsigned bal = __ballot_sync(kAll, k == b);
      if (lane == 0 && bal) atomicAdd(&s_cnt[b], __popc(bal));
    }
  }
  __syncthreads();
  if (threadIdx.x < 4 && s_cnt[threadIdx.x]) atomicAdd(&cnt[threadIdx.x], s_cnt[threadIdx.x]);
}

// stable partition of list[0, n) by row-length bin of M into out; sizes to cnt
static void bin_list(cudaStream_t s, BcWork& W, const int32_t* list, int64_t n, const Csr& M,
                     int32_t* out, int* cnt) {
  GBX_CUDA(cudaMemsetAsync(cnt, 0, 4 * sizeof(int), s));
  if (n == 0) return;
  const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(n, 256), device_sms() * 8));
  k_bc_bin_keys<<<blocks, 256, 0, s>>>(list, n, M.rp.p, W.bkeys[0].p, W.iota.p, cnt);
  GBX_LAUNCHED();
  size_t tb = W.btemp.bytes();
  GBX_CUDA(cub::DeviceRadixSort::SortPairs(W.btemp.p, tb, W.bkeys[0].p, W.bkeys[1].p,
                                           list ? list : W.iota.p, out, static_cast<int>(n), 0,
                                           2, s));
}

static void build_hubs(cudaStream_t s, const Csr& M, BcHubs& H) {
  if (H.key == M.rp.p && H.nnz == M.nnz && H.hv.p) return;
  const int64_t n1 = std::max<int64_t>(M.n, 1);
  DevArray<int> cnt(2);
  GBX_CUDA(cudaMemsetAsync(cnt.p, 0, 2 * sizeof(int), s));
  // hubs have > kBcHeavy edges each: at most nnz / kBcHeavy of them
  const int64_t cap_v = std::min<int64_t>(n1, M.nnz / kBcHeavy + 1);
  const int64_t cap_e = M.nnz / kBcHChunk + cap_v + 1;
  H.hv.alloc(cap_v);
  H.hent.alloc(cap_e);
  H.hacc.alloc(cap_v * 4);
  GBX_CUDA(cudaMemsetAsync(H.hacc.p, 0, H.hacc.bytes(), s));
  k_bc_hubs<<<ceil_div(n1, 256), 256, 0, s>>>(M.rp.p, M.n, H.hv.p, H.hent.p, cnt.p);
  GBX_LAUNCHED();
  int hc[2];
  GBX_CUDA(cudaMemcpyAsync(hc, cnt.p, sizeof hc, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  H.nhv = hc[0];
  H.nhent = hc[1];
  H.key = M.rp.p;
  H.nnz = M.nnz;
}

// per-graph BC workspaces (allocated once per vertex count)
static BcWork& ensure_work(gbx_graph* g) {
  if (!g->bc) g->bc = std::make_unique<BcWork>();
  BcWork& W = *g->bc;
  cudaStream_t s = g->stream;
  const Csr& A = g->A;
  const int64_t n = A.n;
  const int64_t n1 = std::max<int64_t>(n, 1);
  const int64_t ecap = n + A.nnz / kBcChunk + 64;
  if (W.n != n || !W.level.p) {
    W.n = n;
    W.lanes = kBcLanes;
    W.level.alloc(n1 * 4);
    W.lv8.alloc(n1);
    W.sigma.alloc(n1 * 4);
    W.delta.alloc(n1 * 4);
    W.order.alloc(n1 * 4 + 8);
    W.border.alloc(n1 * 4 + 8);
    W.cent.alloc(n1);
    W.mark.alloc(n1);
    W.ulist[0].alloc(n1);
    W.ulist[1].alloc(n1);
    W.ent[0].alloc(ecap);
    W.ent[1].alloc(ecap);
    W.ctl.alloc(8);
    W.src.alloc(4);
    W.map[0].alloc(n1 / 8 + 1);
    W.map[1].alloc(n1 / 8 + 1);
    W.bkeys[0].alloc(n1);
    W.bkeys[1].alloc(n1);
    W.iota.alloc(n1);
    W.ucnt.alloc(4);
    W.allcnt.alloc(4);
    W.allbin.alloc(n1);
    size_t tb = 0;
    GBX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, W.bkeys[0].p, W.bkeys[1].p, W.iota.p,
                                             W.order.p, static_cast<int>(n1), 0, 2, s));
    W.btemp.alloc(tb + 256);
    W.allbin_key = nullptr;
  }
  return W;
}

__global__ void k_bc_degree_key(const int64_t* rp, const int32_t* colcount, int64_t n, int32_t* key) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) key[i] = static_cast<int32_t>(rp[i + 1] - rp[i]) + (colcount ? colcount[i] : 0);
}
__global__ void k_bc_count_nonzero(const int32_t* key, int64_t n, int* cnt) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const bool nz = i < n && key[i] > 0;
  const unsigned bal = __ballot_sync(0xffffffffu, nz);
  if ((threadIdx.x & 31) == 0 && bal) atomicAdd(cnt, __popc(bal));
}
__global__ void k_bc_inverse(const int32_t* new2old, int64_t n, int32_t* old2new) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) old2new[new2old[i]] = static_cast<int32_t>(i);
}
__global__ void k_bc_map_sources(int32_t* src, int ns, const int32_t* old2new) {
  if (threadIdx.x < ns) src[threadIdx.x] = old2new[src[threadIdx.x]];
}
__global__ void k_bc_unpermute(const double* cent_new, const int32_t* old2new, int64_t n, double* cent) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) cent[i] = cent_new[old2new[i]];
}

// the degree-sorted copy (BcWork::ra / rat), built once per graph
static void ensure_relabel(gbx_graph* g, BcWork& W) {
  const Csr& A = g->A;
  if (W.relabel_key == A.rp.p && W.relabel_nnz == A.nnz && W.rat.rp.p) return;
  cudaStream_t s = g->stream;
  const int64_t n = A.n, nnz = A.nnz;
  const bool directed = g->kind != GBX_UNDIRECTED;
  DevArray<int32_t> rowlen, colcount, key(std::max<int64_t>(n, 1));
  compute_degrees(s, A, rowlen, true);
  if (directed) compute_degrees(s, A, colcount, false);
  k_bc_degree_key<<<ceil_div(std::max<int64_t>(n, 1), 256), 256, 0, s>>>(
      A.rp.p, directed ? colcount.p : nullptr, n, key.p);
  GBX_LAUNCHED();
  sort_ids_by_key(s, key.p, n, false, W.new2old);
  // vertices with edges come first in the new order: the first pull's work
  // list stops there (45% of an R-MAT graph's vertices are isolated)
  {
    Tmp<int> nz(1, s);
    GBX_CUDA(cudaMemsetAsync(nz.p, 0, sizeof(int), s));
    k_bc_count_nonzero<<<ceil_div(std::max<int64_t>(n, 1), 256), 256, 0, s>>>(key.p, n, nz.p);
    GBX_LAUNCHED();
    int h = 0;
    GBX_CUDA(cudaMemcpyAsync(&h, nz.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaStreamSynchronize(s));
    W.relabel_nz = h;
  }
  W.old2new.alloc(std::max<int64_t>(n, 1));
  k_bc_inverse<<<ceil_div(std::max<int64_t>(n, 1), 256), 256, 0, s>>>(W.new2old.p, n, W.old2new.p);
  GBX_LAUNCHED();
  // relabeled AT = the transpose of A under the relabeling; an undirected
  // graph's relabeled A is the same matrix
  W.rat.n = n;
  W.rat.nnz = nnz;
  W.rat.rp.alloc(n + 1);
  W.rat.col.alloc(std::max<int64_t>(nnz, 1));
  relabeled_transpose(s, A, W.new2old.p, W.old2new.p, directed ? colcount.p : rowlen.p,
                      W.rat.rp.p, W.rat.col.p);
  if (directed) {
    const Csr& AT = g->AT();
    W.ra.n = n;
    W.ra.nnz = nnz;
    W.ra.rp.alloc(n + 1);
    W.ra.col.alloc(std::max<int64_t>(nnz, 1));
    relabeled_transpose(s, AT, W.new2old.p, W.old2new.p, rowlen.p, W.ra.rp.p, W.ra.col.p);
  }
  W.cent_new.alloc(std::max<int64_t>(n, 1));
  GBX_CUDA(cudaStreamSynchronize(s));
  W.relabel_key = A.rp.p;
  W.relabel_nnz = nnz;
}

void bc_run(gbx_graph* g, const uint64_t* sources, uint64_t ns, double* centrality) {
  NvtxRange nvtx_("gbx.bc");
  const int64_t n = g->A.n;
  for (uint64_t b = 0; b < ns; ++b)
    if (sources[b] >= static_cast<uint64_t>(n))
      fail(GBX_SOURCE_OUT_OF_RANGE, "source " + std::to_string(sources[b]));
  BcWork& W = ensure_work(g);
  cudaStream_t s = g->stream;
  // large graphs run on the degree-sorted copy: sources mapped in, the
  // centrality mapped back at the end (same sums, another fp64 rounding order)
  const int64_t rmin = option(kOptBcRelabelMinN);
  const bool relabeled = rmin >= 0 && n >= rmin && g->A.nnz > 0;
  if (relabeled) ensure_relabel(g, W);
  const Csr& AT = relabeled ? W.rat : g->AT();
  const Csr& A = relabeled ? (g->kind == GBX_UNDIRECTED ? W.rat : W.ra) : g->A;
  double* const cent_acc = relabeled ? W.cent_new.p : W.cent.p;
  const int64_t n1 = std::max<int64_t>(n, 1);
  const size_t map_bytes = (n1 / 8 + 1) * sizeof(uint32_t);
  build_hubs(s, A, W.hub_a);
  const bool same = &AT == &A;
  if (!same) build_hubs(s, AT, W.hub_t);
  BcHubs& HT = same ? W.hub_a : W.hub_t;
  // every vertex, binned by in-degree: the first pull's work list
  if (W.allbin_key != AT.rp.p || W.allbin_nnz != AT.nnz) {
    bin_list(s, W, nullptr, relabeled ? W.relabel_nz : n, AT, W.allbin.p, W.allcnt.p);
    W.allbin_key = AT.rp.p;
    W.allbin_nnz = AT.nnz;
  }
  GBX_CUDA(cudaMemsetAsync(cent_acc, 0, n1 * 8, s));
  const int grid = device_sms() * 8;
  const int alpha = static_cast<int>(option(kOptBcAlpha));
  int* ctl = W.ctl.p;
  unsigned long long* dedges = reinterpret_cast<unsigned long long*>(W.ctl.p + 4);
  int64_t launches = 1, edges = 0;
  int max_levels = 0;
  for (uint64_t b0 = 0; b0 < ns; b0 += kBcLanes) {
    const int nb = static_cast<int>(std::min<uint64_t>(kBcLanes, ns - b0));
    int32_t hs[4];
    for (int b = 0; b < nb; ++b) hs[b] = static_cast<int32_t>(sources[b0 + b]);
    GBX_CUDA(cudaMemcpyAsync(W.src.p, hs, nb * 4, cudaMemcpyHostToDevice, s));
    if (relabeled) k_bc_map_sources<<<1, 32, 0, s>>>(W.src.p, nb, W.old2new.p);
    k_bc_init<<<ceil_div(n1 * 4, 256), 256, 0, s>>>(W.level.p, W.lv8.p, W.sigma.p, W.mark.p, n);
    GBX_CUDA(cudaMemsetAsync(W.map[0].p, 0, map_bytes, s));
    GBX_CUDA(cudaMemsetAsync(W.map[1].p, 0, map_bytes, s));
    k_bc_seed<<<1, 1, 0, s>>>(W.src.p, nb, W.level.p, W.lv8.p, W.sigma.p, W.mark.p, W.order.p,
                              W.ent[0].p, ctl, dedges, A.rp.p, W.map[0].p);
    GBX_LAUNCHED();
    launches += 2;
    // ---- forward sweep
    std::vector<int64_t> off = {0};
    std::vector<unsigned long long> lev_edges;  // out-edges of the vertices of each depth
    struct Hc { int c[4]; unsigned long long e; int hubs_left; int pad; } hc;
    bool hubs_left = true;  // some hub row is unreached in a live lane (unknown before a pull)
    GBX_CUDA(cudaMemcpyAsync(&hc, W.ctl.p, sizeof hc, cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaStreamSynchronize(s));
    off.push_back(hc.c[0]);
    lev_edges.push_back(hc.e);
    int n_ent = hc.c[1];
    unsigned long long fe = hc.e;
    unsigned live = static_cast<unsigned>(hc.c[3]);
    int cur = 0, ucnt = -1;
    const bool trace = option(kOptBcTrace) != 0;
    auto tnow = [] { return std::chrono::steady_clock::now(); };
    auto us = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
      return std::chrono::duration<double, std::micro>(b - a).count();
    };
    for (int d = 1; static_cast<int64_t>(d) <= n; ++d) {
      if (off.back() == off[off.size() - 2]) break;
      const auto t0 = tnow();
      GBX_CUDA(cudaMemsetAsync(W.ctl.p, 0, sizeof hc, s));
      bool pulled_hubs = false;
      BcArgs a{};
      a.own0 = 0;
      a.own1 = n;
      a.rp = A.rp.p;
      a.col = A.col.p;
      a.trp = AT.rp.p;
      a.tcol = AT.col.p;
      a.n = n;
      a.level = W.level.p;
      a.lv8 = W.lv8.p;
      a.sigma = W.sigma.p;
      a.mark = W.mark.p;
      a.list_out = W.order.p + off.back();
      a.ent_in = W.ent[cur].p;
      a.ent_out = W.ent[cur ^ 1].p;
      a.n_ent = n_ent;
      a.cnt = ctl;
      a.edges = dedges;
      a.d = d;
      a.lanes = live;
      a.map_in = W.map[cur].p;
      a.map_out = W.map[cur ^ 1].p;
      // push while the frontier's edges are under nnz/alpha -- and, once a pull
      // has listed the still-unreached vertices, only while the frontier's
      // edges are under those vertices' (estimated) in-edges
      const double unreached_edges =
          ucnt < 0 ? 1e300 : static_cast<double>(ucnt) * A.nnz / std::max<int64_t>(n, 1);
      const bool push = alpha <= 0 || (fe * static_cast<unsigned long long>(alpha) <
                                           static_cast<unsigned long long>(A.nnz) &&
                                       static_cast<double>(fe) < unreached_edges);
      if (push) {
        k_bc_push<<<grid, 256, 0, s>>>(a);
        GBX_LAUNCHED();
        ++launches;
      } else {
        // work list: every vertex (first pull) or the survivors of the last
        // pull, binned by in-degree; survivors of this pull go to ulist[0]
        if (ucnt < 0) {
          a.bins = BcBins{W.allbin.p, W.allcnt.p};
        } else {
          bin_list(s, W, W.ulist[0].p, ucnt, AT, W.ulist[1].p, W.ucnt.p);
          a.bins = BcBins{W.ulist[1].p, W.ucnt.p};
          launches += 2;
        }
        a.ul_out = W.ulist[0].p;
        a.hv = HT.hv.p;
        a.hent = HT.hent.p;
        a.nhv = HT.nhv;
        a.nhent = HT.nhent;
        a.hacc = HT.hacc.p;
        k_bc_pull<<<grid, 256, 0, s>>>(a);
        GBX_LAUNCHED();
        ++launches;
        pulled_hubs = HT.nhv && hubs_left;
        if (pulled_hubs) {
          k_bc_pull_hub<<<grid, 256, 0, s>>>(a);
          k_bc_pull_hub_fin<<<ceil_div(HT.nhv, 256), 256, 0, s>>>(a);
          GBX_LAUNCHED();
          launches += 2;
        }
      }
      GBX_CUDA(cudaMemcpyAsync(&hc, W.ctl.p, sizeof hc, cudaMemcpyDeviceToHost, s));
      GBX_CUDA(cudaStreamSynchronize(s));
      off.push_back(off.back() + hc.c[0]);
      lev_edges.push_back(hc.e);
      n_ent = hc.c[1];
      fe = hc.e;
      live = static_cast<unsigned>(hc.c[3]);
      if (!push) ucnt = hc.c[2];
      if (pulled_hubs) hubs_left = hc.hubs_left > 0;
      GBX_CUDA(cudaMemsetAsync(W.map[cur].p, 0, map_bytes, s));  // depth d-1 map retired
      cur ^= 1;
      if (trace)
        std::fprintf(stderr, "bc forward depth %d %s: %d settled, %.1f us\n", d, push ? "push" : "pull",
                     hc.c[0], us(t0, tnow()));
    }
    // levels: off[d]..off[d+1] lists vertices with some lane at depth d
    const int D = static_cast<int>(off.size()) - 1;  // depths 0..D-1 (last list may be empty)
    max_levels = std::max(max_levels, D);
    int deepest = D - 1;
    while (deepest > 0 && off[deepest + 1] == off[deepest]) --deepest;
    const unsigned all = (1u << nb) - 1;
    if (deepest >= 1) {
      const int nl = static_cast<int>(off[deepest + 1] - off[deepest]);
      k_bc_leaf<<<ceil_div(nl, 256), 256, 0, s>>>(W.order.p + off[deepest], nl, deepest, all,
                                                   W.level.p, W.lv8.p, W.sigma.p, W.delta.p);
      GBX_LAUNCHED();
      ++launches;
      // the deepest level has delta = 0: nothing to add to the centrality
    }
    if (static_cast<int64_t>(W.lcnt.n) < 4 * static_cast<int64_t>(D + 1)) W.lcnt.alloc(4 * (D + 1));
    for (int d = deepest - 1; d >= 1; --d) {
      const int nl = static_cast<int>(off[d + 1] - off[d]);
      if (nl == 0) continue;
      const auto t0 = tnow();
      BcArgs a{};
      a.own0 = 0;
      a.own1 = n;
      a.rp = A.rp.p;
      a.col = A.col.p;
      a.n = n;
      a.level = W.level.p;
      a.lv8 = W.lv8.p;
      a.sigma = W.sigma.p;
      a.coef = W.delta.p;
      a.cent = cent_acc;
      a.hv = W.hub_a.hv.p;
      a.hent = W.hub_a.hent.p;
      a.nhv = W.hub_a.nhv;
      a.nhent = W.hub_a.nhent;
      a.hacc = W.hub_a.hacc.p;
      a.d = d;
      a.lanes = all;
      const int nl1 = static_cast<int>(off[d + 2] - off[d + 1]);
      // push form when the children's rows hold at most 1/bc.back_push of the
      // parents' edges (and the depth is past the hub levels, whose parents
      // would serialise the atomics)
      const int64_t bp = option(kOptBcBackPush);
      const bool push_back = bp > 0 && d >= option(kOptBcBackPushMinDepth) && nl1 > 0 &&
                             lev_edges[d + 1] * static_cast<unsigned long long>(bp) <= lev_edges[d];
      GBX_CUDA(cudaMemsetAsync(W.map[0].p, 0, map_bytes, s));
      a.map_in = W.map[0].p;
      if (push_back) {
        // level map of depth d (the parents'), children binned by in-degree
        k_bc_map<<<ceil_div(nl, 256), 256, 0, s>>>(W.order.p + off[d], nl, d, all, W.level.p,
                                                   W.lv8.p, W.map[0].p);
        bin_list(s, W, W.order.p + off[d + 1], nl1, AT, W.border.p + off[d + 1],
                 W.lcnt.p + 4 * (d + 1));
        a.bins = BcBins{W.border.p + off[d + 1], W.lcnt.p + 4 * (d + 1)};
        a.trp = AT.rp.p;
        a.tcol = AT.col.p;
        if (!W.bacc.p) {
          W.bacc.alloc(n1 * 4);
          GBX_CUDA(cudaMemsetAsync(W.bacc.p, 0, W.bacc.bytes(), s));
        }
        a.bacc = W.bacc.p;
        a.list_in = W.order.p + off[d];
        a.n_list = nl;
        k_bc_back_push<<<grid, 256, 0, s>>>(a);
        k_bc_back_fin<<<ceil_div(nl, 256), 256, 0, s>>>(a);
        GBX_LAUNCHED();
        launches += 5;
      } else {
        // level map of depth d+1 (the successors' depth) from its list
        k_bc_map<<<ceil_div(std::max(nl1, 1), 256), 256, 0, s>>>(W.order.p + off[d + 1], nl1, d + 1,
                                                                 all, W.level.p, W.lv8.p, W.map[0].p);
        // the level-d list binned by out-degree
        bin_list(s, W, W.order.p + off[d], nl, A, W.border.p + off[d], W.lcnt.p + 4 * d);
        a.bins = BcBins{W.border.p + off[d], W.lcnt.p + 4 * d};
        k_bc_back<<<grid, 256, 0, s>>>(a);
        GBX_LAUNCHED();
        launches += 4;
        if (W.hub_a.nhv) {
          k_bc_back_hub<<<grid, 256, 0, s>>>(a);
          k_bc_back_hub_fin<<<ceil_div(W.hub_a.nhv, 256), 256, 0, s>>>(a);
          GBX_LAUNCHED();
          launches += 2;
        }
      }
      if (trace) {
        GBX_CUDA(cudaStreamSynchronize(s));
        std::fprintf(stderr, "bc backward depth %d %s: %d vertices (%llu edges; %llu below), %.1f us\n",
                     d, push_back ? "push" : "pull", nl, lev_edges[d], lev_edges[d + 1],
                     us(t0, tnow()));
      }
    }
    edges += A.nnz;
  }
  if (relabeled) {
    k_bc_unpermute<<<ceil_div(n1, 256), 256, 0, s>>>(W.cent_new.p, W.old2new.p, n, W.cent.p);
    GBX_LAUNCHED();
    ++launches;
  }
  if (centrality) {
    GBX_CUDA(cudaMemcpyAsync(centrality, W.cent.p, n * 8, cudaMemcpyDeviceToHost, s));
  }
  GBX_CUDA(cudaStreamSynchronize(s));
  g->stats = gbx_stats{};
  g->pending_iters = nullptr;
  g->stats.launches = launches;
  g->stats.iterations = max_levels;
  g->stats.work_units = edges;
}


// ---------------------------------------------------------------------------
// Row-partitioned batched Brandes for the multi-GPU driver (1D row
// blocks, one exchange per BFS level).  Every rank holds the graph and the
// replicated per-vertex state; rank r owns vertices [rb, re) (nnz-balanced):
//   forward, depth d: pull over AT for the OWNED still-unreached vertices (the
//     same k_bc_pull / hub passes, work lists restricted to owned rows); the
//     rank packs (v, new lanes, sigma[4]) for the vertices it settled; the
//     driver all-gathers every rank's records (rank order) and each rank
//     applies the others' and appends all of them to the global level list
//     -- so the level lists, maps and sigma are identical on every rank;
//   backward, depth d: the owned part of the level-d list runs k_bc_back (and
//     the owned hub chunks); (v, coef[4]) records are exchanged the same way;
//   the centrality partials (owned vertices only) are summed by one
//     all-reduce at the end (betweenness.cpp:74-79).
// The per-vertex sums are computed by the same kernels as the single-GPU run
// (push levels become pulls: path counts are integers, exact in any order),
// so the result equals gbx_betweenness up to the rounding order of the hub
// rows' fp64 atomics (measured: <= 1e-15 relative).
// Record layout (40 bytes): int32 v, uint32 lanes, double x[4].
// ---------------------------------------------------------------------------

struct BcRec {
  int32_t v;
  uint32_t lanes;
  double x[4];
};
static_assert(sizeof(BcRec) == 40, "BcRec layout");

__global__ void k_bc_iota_range(int32_t* out, int64_t b, int64_t e) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (b + i < e) out[i] = static_cast<int32_t>(b + i);
}

// first row r with r + rp[r] >= target (nnz + rows balanced split)
__global__ void k_bc_split(const int64_t* rp, int64_t n, int parts, int64_t* bounds) {
  const int q = threadIdx.x;
  if (q > parts) return;
  const int64_t target = (n + rp[n]) * q / parts;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (mid + rp[mid] < target) lo = mid + 1; else hi = mid;
  }
  bounds[q] = q == 0 ? 0 : q == parts ? n : lo;
}

__global__ void k_bc_own_hubs(const int64_t* hent, int nhent, const int32_t* hv, int64_t rb,
                              int64_t re, int64_t* out, int* cnt) {
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (e >= nhent) return;
  const int64_t ent = hent[e];
  const int32_t v = hv[static_cast<int>(ent & 0xffffffff)];
  if (v >= rb && v < re) out[agg_append(cnt)] = ent;
}

__global__ void k_bc_pack_fwd(const int32_t* list, int nl, int d, const int32_t* level,
                              const double* sigma, BcRec* out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= nl) return;
  const int64_t v = list[i];
  BcRec r;
  r.v = static_cast<int32_t>(v);
  r.lanes = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    if (level[v * 4 + b] == d) r.lanes |= 1u << b;
    r.x[b] = sigma[v * 4 + b];
  }
  out[i] = r;
}

// apply every rank's records of depth d: others' vertices get level / lv8 /
// sigma / map bits; all of them are appended (rank order) to the level list
__global__ void k_bc_apply_fwd(const BcRec* recs, int64_t nrec, int d, int64_t rb, int64_t re,
                               int32_t* level, uint32_t* lv8, double* sigma, uint32_t* map,
                               int32_t* order_out, int* live) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  unsigned m = 0;
  if (i < nrec) {
    const BcRec r = recs[i];
    const int64_t v = r.v;
    order_out[i] = r.v;
    m = r.lanes;
    if (v < rb || v >= re) {
      uint32_t x = lv8[v];
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if ((r.lanes >> b) & 1u) {
          level[v * 4 + b] = d;
          sigma[v * 4 + b] = r.x[b];
          x = (x & ~(0xFFu << (8 * b))) | (lv8_byte(d) << (8 * b));
        }
      lv8[v] = x;
      nib_or(map, v, r.lanes);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m |= __shfl_xor_sync(kAll, m, o);
  if ((threadIdx.x & 31) == 0 && m) atomicOr(live, static_cast<int>(m));
}

__global__ void k_bc_own_filter(const int32_t* list, int64_t nl, int64_t rb, int64_t re,
                                int32_t* out, int* cnt) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= nl) return;
  const int32_t v = list[i];
  if (v >= rb && v < re) out[agg_append(cnt)] = v;
}

__global__ void k_bc_pack_back(const int32_t* list, int nl, const double* coef, BcRec* out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= nl) return;
  const int64_t v = list[i];
  BcRec r;
  r.v = static_cast<int32_t>(v);
  r.lanes = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) r.x[b] = coef[v * 4 + b];
  out[i] = r;
}

__global__ void k_bc_apply_back(const BcRec* recs, int64_t nrec, int d, int64_t rb, int64_t re,
                                const int32_t* level, double* coef) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= nrec) return;
  const BcRec r = recs[i];
  const int64_t v = r.v;
  if (v >= rb && v < re) return;
#pragma unroll
  for (int b = 0; b < 4; ++b)
    if (level[v * 4 + b] == d) coef[v * 4 + b] = r.x[b];
}

// ---- candidate levels of the sharded forward sweep (small frontiers): the
// owned depth-(d-1) vertices mark their out-neighbours (a byte per vertex,
// max-reduced over the ranks by the driver); each rank pulls only its owned
// marked vertices -- the same sums as a full pull (a vertex without a
// frontier in-neighbour sums to nothing), at the frontier's edge count.
constexpr int64_t kBcMarkHeavy = 2048;

__global__ void k_bc_front_split(const int32_t* list, int64_t nl, int64_t rb, int64_t re,
                                 const int64_t* rp, int32_t* light, int* nlight, int32_t* heavy,
                                 int* nheavy, unsigned long long* edges) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  unsigned long long e = 0;
  if (i < nl) {
    const int32_t v = list[i];
    if (v >= rb && v < re) {
      const int64_t deg = rp[v + 1] - rp[v];
      e = static_cast<unsigned long long>(deg);
      if (deg > kBcMarkHeavy) heavy[agg_append(nheavy)] = v;
      else light[agg_append(nlight)] = v;
    }
  }
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(kAll, e, o);
  if ((threadIdx.x & 31) == 0 && e) atomicAdd(edges, e);
}

__global__ void __launch_bounds__(256) k_bc_mark(const int64_t* rp, const int32_t* col, int64_t n,
                                                 const int32_t* light, const int* nlight,
                                                 const int32_t* heavy, const int* nheavy,
                                                 uint8_t* cand) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int m = *nlight;
  for (int64_t i = gw; i < m; i += nw) {
    const int32_t u = light[i];
    for (int64_t p = rp[u] + lane; p < rp[u + 1]; p += 32) {
      const int32_t v = __ldg(col + p);
      GBX_DCHECK(v >= 0 && v < n, "bc mark column", v);
      cand[v] = 1;
    }
  }
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t nt = int64_t(gridDim.x) * blockDim.x;
  const int mh = *nheavy;
  for (int h = 0; h < mh; ++h) {
    const int32_t u = heavy[h];
    for (int64_t p = rp[u] + t; p < rp[u + 1]; p += nt) {
      const int32_t v = __ldg(col + p);
      GBX_DCHECK(v >= 0 && v < n, "bc mark column", v);
      cand[v] = 1;
    }
  }
}

__global__ void k_bc_cand_list(const uint8_t* cand, int64_t rb, int64_t re, int32_t* out, int* cnt) {
  const int64_t v = rb + blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (v < re && cand[v]) out[agg_append(cnt)] = static_cast<int32_t>(v);
}

static BcShard& need_shard(gbx_graph* g) {
  if (!g->bc || !g->bc->shard) fail(GBX_MISSING_PROPERTY, "bc shard protocol needs gbx_bc_shard_begin");
  return *g->bc->shard;
}

void bc_shard_begin(gbx_graph* g, const uint64_t* sources, uint64_t ns, int rank, int nranks,
                    int64_t* rb_out, int64_t* re_out, const int64_t* bounds) {
  require_at(g, "bc_shard");
  const int64_t n = g->A.n;
  if (ns == 0) fail(GBX_EMPTY_BATCH, "empty source batch");
  if (ns > static_cast<uint64_t>(kBcLanes))
    fail(GBX_INVALID_VALUE, "bc_shard: one batch of at most 4 sources per protocol run");
  if (nranks < 1 || rank < 0 || rank >= nranks) fail(GBX_INVALID_VALUE, "bc_shard: bad rank / nranks");
  for (uint64_t b = 0; b < ns; ++b)
    if (sources[b] >= static_cast<uint64_t>(n))
      fail(GBX_SOURCE_OUT_OF_RANGE, "source " + std::to_string(sources[b]));
  BcWork& W = ensure_work(g);
  cudaStream_t s = g->stream;
  const Csr& A = g->A;
  const Csr& AT = g->AT();
  const int64_t n1 = std::max<int64_t>(n, 1);
  auto S = std::make_unique<BcShard>();
  S->rank = rank;
  S->nranks = nranks;
  S->ns = static_cast<int>(ns);
  if (bounds) {
    S->rb = bounds[rank];
    S->re = std::max(bounds[rank], bounds[rank + 1]);
  } else {
    DevArray<int64_t> bnd(nranks + 1);
    k_bc_split<<<1, std::max(32, ((nranks + 32) / 32) * 32), 0, s>>>(A.rp.p, n, nranks, bnd.p);
    GBX_LAUNCHED();
    std::vector<int64_t> hb(nranks + 1);
    GBX_CUDA(cudaMemcpyAsync(hb.data(), bnd.p, (nranks + 1) * 8, cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaStreamSynchronize(s));
    S->rb = hb[rank];
    S->re = std::max(hb[rank], hb[rank + 1]);
  }
  // hub rows and the owned chunks of them
  build_hubs(s, A, W.hub_a);
  const bool same = &AT == &A;
  if (!same) build_hubs(s, AT, W.hub_t);
  BcHubs& HT = same ? W.hub_a : W.hub_t;
  DevArray<int> c(2);
  GBX_CUDA(cudaMemsetAsync(c.p, 0, 2 * sizeof(int), s));
  S->hent_a.alloc(std::max(W.hub_a.nhent, 1));
  S->hent_t.alloc(std::max(HT.nhent, 1));
  if (W.hub_a.nhent)
    k_bc_own_hubs<<<ceil_div(W.hub_a.nhent, 256), 256, 0, s>>>(W.hub_a.hent.p, W.hub_a.nhent,
                                                               W.hub_a.hv.p, S->rb, S->re,
                                                               S->hent_a.p, c.p);
  if (HT.nhent)
    k_bc_own_hubs<<<ceil_div(HT.nhent, 256), 256, 0, s>>>(HT.hent.p, HT.nhent, HT.hv.p, S->rb,
                                                          S->re, S->hent_t.p, c.p + 1);
  GBX_LAUNCHED();
  int hc[2];
  GBX_CUDA(cudaMemcpyAsync(hc, c.p, sizeof hc, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  S->nhent_a = hc[0];
  S->nhent_t = hc[1];
  // the owned rows binned by in-degree: the first pull's work list
  const int64_t own = S->re - S->rb;
  S->ownbin.alloc(std::max<int64_t>(own, 1));
  S->owncnt.alloc(4);
  S->snew.alloc(n1);
  S->slist.alloc(n1);
  S->scnt.alloc(4);
  S->recs.alloc(n1 * sizeof(BcRec));
  {
    DevArray<int32_t> ids(std::max<int64_t>(own, 1));
    if (own) {
      k_bc_iota_range<<<ceil_div(own, 256), 256, 0, s>>>(ids.p, S->rb, S->re);
      GBX_LAUNCHED();
    }
    bin_list(s, W, ids.p, own, AT, S->ownbin.p, S->owncnt.p);
    GBX_CUDA(cudaStreamSynchronize(s));
  }
  // replicated initial state (betweenness.cpp:27-35)
  int32_t hs[4];
  for (uint64_t b = 0; b < ns; ++b) hs[b] = static_cast<int32_t>(sources[b]);
  GBX_CUDA(cudaMemcpyAsync(W.src.p, hs, ns * 4, cudaMemcpyHostToDevice, s));
  const size_t map_bytes = (n1 / 8 + 1) * sizeof(uint32_t);
  k_bc_init<<<ceil_div(n1 * 4, 256), 256, 0, s>>>(W.level.p, W.lv8.p, W.sigma.p, W.mark.p, n);
  GBX_CUDA(cudaMemsetAsync(W.map[0].p, 0, map_bytes, s));
  GBX_CUDA(cudaMemsetAsync(W.map[1].p, 0, map_bytes, s));
  GBX_CUDA(cudaMemsetAsync(W.cent.p, 0, n1 * 8, s));
  k_bc_seed<<<1, 1, 0, s>>>(W.src.p, static_cast<int>(ns), W.level.p, W.lv8.p, W.sigma.p, W.mark.p,
                            W.order.p, W.ent[0].p, W.ctl.p,
                            reinterpret_cast<unsigned long long*>(W.ctl.p + 4), A.rp.p, W.map[0].p);
  GBX_LAUNCHED();
  int hseed[4];
  GBX_CUDA(cudaMemcpyAsync(hseed, W.ctl.p, sizeof hseed, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  S->off = {0, hseed[0]};
  S->live = static_cast<unsigned>(hseed[3]);
  S->cur = 0;
  S->ucnt = -1;
  W.shard = std::move(S);
  if (rb_out) *rb_out = W.shard->rb;
  if (re_out) *re_out = W.shard->re;
}

// edges of the owned vertices of the last settled depth (the direction rule's
// measure) and, with cand != NULL (n bytes, zeroed by the caller), the marks
// of their out-neighbours
int64_t bc_shard_mark(gbx_graph* g, uint8_t* cand) {
  NvtxRange nvtx_("gbx.bc.shard_mark");
  BcShard& S = need_shard(g);
  BcWork& W = *g->bc;
  if (S.fwd_done) return 0;
  cudaStream_t s = g->stream;
  const Csr& A = g->A;
  const int64_t n1 = std::max<int64_t>(A.n, 1);
  const int d = static_cast<int>(S.off.size()) - 1;  // the depth being built; d-1 settled
  const int64_t b = S.off[d - 1], nl = S.off[d] - S.off[d - 1];
  if (!S.ccnt.p) {
    S.ccnt.alloc(4);
    S.flight.alloc(n1);
    S.fheavy.alloc(n1);
  }
  Tmp<unsigned long long> e(1, s);
  GBX_CUDA(cudaMemsetAsync(e.p, 0, 8, s));
  GBX_CUDA(cudaMemsetAsync(S.ccnt.p, 0, 4 * sizeof(int), s));
  if (nl > 0) {
    k_bc_front_split<<<ceil_div(nl, 256), 256, 0, s>>>(W.order.p + b, nl, S.rb, S.re, A.rp.p,
                                                       S.flight.p, S.ccnt.p, S.fheavy.p,
                                                       S.ccnt.p + 1, e.p);
    GBX_LAUNCHED();
    if (cand) {
      k_bc_mark<<<device_sms() * 8, 256, 0, s>>>(A.rp.p, A.col.p, A.n, S.flight.p, S.ccnt.p,
                                                 S.fheavy.p, S.ccnt.p + 1, cand);
      GBX_LAUNCHED();
    }
  }
  unsigned long long h = 0;
  GBX_CUDA(cudaMemcpyAsync(&h, e.p, 8, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  return static_cast<int64_t>(h);
}

// one forward depth on the owned rows; *recs = device records of the owned
// vertices it settled (valid until the next protocol call)
void bc_shard_forward(gbx_graph* g, void** recs, int64_t* nrec, const uint8_t* cand) {
  NvtxRange nvtx_("gbx.bc.shard_forward");
  BcShard& S = need_shard(g);
  BcWork& W = *g->bc;
  *recs = S.recs.p;
  *nrec = 0;
  if (S.fwd_done) return;
  cudaStream_t s = g->stream;
  const Csr& A = g->A;
  const Csr& AT = g->AT();
  const bool same = &AT == &A;
  BcHubs& HT = same ? W.hub_a : W.hub_t;
  const int d = static_cast<int>(S.off.size()) - 1;
  GBX_CUDA(cudaMemsetAsync(W.ctl.p, 0, 8 * sizeof(int), s));
  BcArgs a{};
  a.rp = A.rp.p;
  a.col = A.col.p;
  a.trp = AT.rp.p;
  a.tcol = AT.col.p;
  a.n = A.n;
  a.level = W.level.p;
  a.lv8 = W.lv8.p;
  a.sigma = W.sigma.p;
  a.mark = W.mark.p;
  a.list_out = S.snew.p;
  a.ent_out = W.ent[1].p;
  a.cnt = W.ctl.p;
  a.edges = reinterpret_cast<unsigned long long*>(W.ctl.p + 4);
  a.d = d;
  a.lanes = S.live;
  a.map_in = W.map[S.cur].p;
  a.map_out = W.map[S.cur ^ 1].p;
  a.own0 = S.rb;
  a.own1 = S.re;
  a.cand = cand;
  const int64_t n1 = std::max<int64_t>(A.n, 1);
  if (cand) {
    // candidate level: the owned marked vertices only; their survivors go to
    // scratch (the owned still-unreached list of the pull levels stays as it
    // is: the pull skips vertices settled since)
    if (!S.clist.p) {
      S.clist.alloc(n1);
      S.cbin.alloc(n1);
      S.cscr.alloc(n1);
    }
    if (!S.ccnt.p) S.ccnt.alloc(4);
    GBX_CUDA(cudaMemsetAsync(S.ccnt.p + 2, 0, sizeof(int), s));
    if (S.re > S.rb)
      k_bc_cand_list<<<ceil_div(S.re - S.rb, 256), 256, 0, s>>>(cand, S.rb, S.re, S.clist.p,
                                                                S.ccnt.p + 2);
    GBX_LAUNCHED();
    int nc = 0;
    GBX_CUDA(cudaMemcpyAsync(&nc, S.ccnt.p + 2, sizeof(int), cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaStreamSynchronize(s));
    bin_list(s, W, S.clist.p, nc, AT, S.cbin.p, W.ucnt.p);
    a.bins = BcBins{S.cbin.p, W.ucnt.p};
    a.ul_out = S.cscr.p;
  } else if (S.ucnt < 0) {
    a.bins = BcBins{S.ownbin.p, S.owncnt.p};
    a.ul_out = W.ulist[0].p;
  } else {
    bin_list(s, W, W.ulist[0].p, S.ucnt, AT, W.ulist[1].p, W.ucnt.p);
    a.bins = BcBins{W.ulist[1].p, W.ucnt.p};
    a.ul_out = W.ulist[0].p;
  }
  a.hv = HT.hv.p;
  a.hent = S.hent_t.p;
  a.nhv = HT.nhv;
  a.nhent = S.nhent_t;
  a.hacc = HT.hacc.p;
  const int grid = device_sms() * 8;
  k_bc_pull<<<grid, 256, 0, s>>>(a);
  GBX_LAUNCHED();
  if (HT.nhv) {
    if (S.nhent_t) k_bc_pull_hub<<<grid, 256, 0, s>>>(a);
    k_bc_pull_hub_fin<<<ceil_div(HT.nhv, 256), 256, 0, s>>>(a);
    GBX_LAUNCHED();
  }
  int hc[4];
  GBX_CUDA(cudaMemcpyAsync(hc, W.ctl.p, sizeof hc, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  if (!cand) S.ucnt = hc[2];
  if (hc[0]) {
    k_bc_pack_fwd<<<ceil_div(hc[0], 256), 256, 0, s>>>(S.snew.p, hc[0], d, W.level.p, W.sigma.p,
                                                       reinterpret_cast<BcRec*>(S.recs.p));
    GBX_LAUNCHED();
    GBX_CUDA(cudaStreamSynchronize(s));
  }
  *nrec = hc[0];
}

// every rank's records of the depth just computed, concatenated in rank order
void bc_shard_forward_apply(gbx_graph* g, const void* recs, int64_t nrec, int* done) {
  BcShard& S = need_shard(g);
  BcWork& W = *g->bc;
  cudaStream_t s = g->stream;
  const int64_t n1 = std::max<int64_t>(g->A.n, 1);
  const size_t map_bytes = (n1 / 8 + 1) * sizeof(uint32_t);
  if (S.fwd_done) { if (done) *done = 1; return; }
  const int d = static_cast<int>(S.off.size()) - 1;
  GBX_CUDA(cudaMemsetAsync(W.ctl.p + 3, 0, sizeof(int), s));
  if (nrec > 0) {
    k_bc_apply_fwd<<<ceil_div(nrec, 256), 256, 0, s>>>(
        reinterpret_cast<const BcRec*>(recs), nrec, d, S.rb, S.re, W.level.p, W.lv8.p, W.sigma.p,
        W.map[S.cur ^ 1].p, W.order.p + S.off.back(), W.ctl.p + 3);
    GBX_LAUNCHED();
  }
  int live = 0;
  GBX_CUDA(cudaMemcpyAsync(&live, W.ctl.p + 3, sizeof(int), cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaMemsetAsync(W.map[S.cur].p, 0, map_bytes, s));  // depth d-1 map retired
  GBX_CUDA(cudaStreamSynchronize(s));
  S.off.push_back(S.off.back() + nrec);
  S.live = static_cast<unsigned>(live);
  S.cur ^= 1;
  if (nrec == 0 || S.off.size() > static_cast<size_t>(g->A.n) + 1) S.fwd_done = true;
  if (done) *done = S.fwd_done ? 1 : 0;
}

// one backward depth on the owned part of the level list; *done = 1 (and no
// records) once depth 1 has been processed
void bc_shard_backward(gbx_graph* g, void** recs, int64_t* nrec, int* done) {
  NvtxRange nvtx_("gbx.bc.shard_backward");
  BcShard& S = need_shard(g);
  BcWork& W = *g->bc;
  if (!S.fwd_done) fail(GBX_PRECONDITION_VIOLATED, "bc_shard_backward before the forward sweep ended");
  cudaStream_t s = g->stream;
  const Csr& A = g->A;
  const int64_t n1 = std::max<int64_t>(A.n, 1);
  const size_t map_bytes = (n1 / 8 + 1) * sizeof(uint32_t);
  const unsigned all = (1u << S.ns) - 1;
  const std::vector<int64_t>& off = S.off;
  const int D = static_cast<int>(off.size()) - 1;
  *recs = S.recs.p;
  *nrec = 0;
  if (S.bd < 0) {
    // the deepest non-empty level: delta = 0, coef = 1 / sigma (replicated)
    int deepest = D - 1;
    while (deepest > 0 && off[deepest + 1] == off[deepest]) --deepest;
    if (deepest >= 1) {
      const int nl = static_cast<int>(off[deepest + 1] - off[deepest]);
      k_bc_leaf<<<ceil_div(nl, 256), 256, 0, s>>>(W.order.p + off[deepest], nl, deepest, all,
                                                   W.level.p, W.lv8.p, W.sigma.p, W.delta.p);
      GBX_LAUNCHED();
    }
    S.bd = deepest - 1;
  }
  while (S.bd >= 1 && off[S.bd + 1] == off[S.bd]) --S.bd;
  if (S.bd < 1) { *done = 1; return; }
  *done = 0;
  const int d = S.bd;
  const int nl = static_cast<int>(off[d + 1] - off[d]);
  const int nl1 = static_cast<int>(off[d + 2] - off[d + 1]);
  GBX_CUDA(cudaMemsetAsync(W.map[0].p, 0, map_bytes, s));
  if (nl1)
    k_bc_map<<<ceil_div(nl1, 256), 256, 0, s>>>(W.order.p + off[d + 1], nl1, d + 1, all, W.level.p,
                                                 W.lv8.p, W.map[0].p);
  GBX_CUDA(cudaMemsetAsync(S.scnt.p, 0, sizeof(int), s));
  k_bc_own_filter<<<ceil_div(nl, 256), 256, 0, s>>>(W.order.p + off[d], nl, S.rb, S.re, S.snew.p,
                                                    S.scnt.p);
  GBX_LAUNCHED();
  int own = 0;
  GBX_CUDA(cudaMemcpyAsync(&own, S.scnt.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  BcArgs a{};
  a.rp = A.rp.p;
  a.col = A.col.p;
  a.n = A.n;
  a.level = W.level.p;
  a.lv8 = W.lv8.p;
  a.sigma = W.sigma.p;
  a.coef = W.delta.p;
  a.cent = W.cent.p;
  a.hv = W.hub_a.hv.p;
  a.hent = S.hent_a.p;
  a.nhv = W.hub_a.nhv;
  a.nhent = S.nhent_a;
  a.hacc = W.hub_a.hacc.p;
  a.d = d;
  a.lanes = all;
  a.map_in = W.map[0].p;
  a.own0 = S.rb;
  a.own1 = S.re;
  bin_list(s, W, S.snew.p, own, A, S.slist.p, S.scnt.p);
  a.bins = BcBins{S.slist.p, S.scnt.p};
  const int grid = device_sms() * 8;
  if (own) {
    k_bc_back<<<grid, 256, 0, s>>>(a);
    GBX_LAUNCHED();
  }
  if (W.hub_a.nhv) {
    if (S.nhent_a) k_bc_back_hub<<<grid, 256, 0, s>>>(a);
    k_bc_back_hub_fin<<<ceil_div(W.hub_a.nhv, 256), 256, 0, s>>>(a);
    GBX_LAUNCHED();
  }
  if (own) {
    k_bc_pack_back<<<ceil_div(own, 256), 256, 0, s>>>(S.snew.p, own, W.delta.p,
                                                      reinterpret_cast<BcRec*>(S.recs.p));
    GBX_LAUNCHED();
  }
  GBX_CUDA(cudaStreamSynchronize(s));
  *nrec = own;
}

void bc_shard_backward_apply(gbx_graph* g, const void* recs, int64_t nrec) {
  BcShard& S = need_shard(g);
  BcWork& W = *g->bc;
  cudaStream_t s = g->stream;
  if (S.bd < 1) return;
  if (nrec > 0) {
    k_bc_apply_back<<<ceil_div(nrec, 256), 256, 0, s>>>(reinterpret_cast<const BcRec*>(recs), nrec,
                                                        S.bd, S.rb, S.re, W.level.p, W.delta.p);
    GBX_LAUNCHED();
  }
  GBX_CUDA(cudaStreamSynchronize(s));
  --S.bd;
}

// this rank's centrality partial (device, fp64, n entries; zero off its rows)
void bc_shard_centrality(gbx_graph* g, double** cent) {
  need_shard(g);
  GBX_CUDA(cudaStreamSynchronize(g->stream));
  *cent = g->bc->cent.p;
}

}  // namespace gbx
