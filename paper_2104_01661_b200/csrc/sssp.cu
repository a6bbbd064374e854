// sssp.cu -- delta-stepping SSSP (algo/sssp.cpp:16-112) as ONE persistent
// cooperative kernel.
//
// The reference relaxes light edges (w <= delta) of the current bucket
// [lo, lo+delta) to a fixpoint, then heavy edges once, and jumps to the next
// non-empty bucket (sssp.cpp:55-106).  Its result equals Dijkstra exactly
// (test_sssp.cpp:91-111), so the device mirrors it in result, not mechanism
// (SURVEY.md §7 hard part 4): a near/far bucketed label-correcting sweep.
//   * near queue: vertices whose tentative distance fell into the current
//     bucket; each level relaxes all their edges with atomicMin on the
//     distance word; improvements below hi re-enter the near queue, the rest
//     go to the far pile, each deduplicated by a parity-alternating bitmap
//     (n/8 bytes: L2-resident; the iteration that pops a queue clears its bits);
//   * the distance array is pinned in L2 with an access-policy window while
//     the edge stream bypasses L1;
//   * when the near queue drains, the bucket jumps to floor(min far / delta)
//     * delta (the reference's jump, sssp.cpp:60-65) and the far pile is
//     split into the new near queue and what stays far -- all on the device;
//   * edges are packed as (col << 8 | w) in one u32 when n <= 2^24 and the
//     weights are integers in [1,255] (BASELINE config 4: 4 B/edge), else
//     separate col + weight arrays; integer weights use u32 distances, other
//     fp64 weights u64 bit patterns of positive doubles (order-preserving).
// Algorithmic bytes per source: 8*m_r + 12*V_r.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "plans.cuh"
#include "sort.cuh"
#include "warpqueue.cuh"

namespace cg = cooperative_groups;

namespace gbx {

constexpr int kSsspThreads = 256;
#ifndef GBX_SSSP_IBUCKET
#define GBX_SSSP_IBUCKET 1  // integer bucket index (shift / u32 division) for integral delta
#endif
#ifndef GBX_SSSP_PRECHECK
#define GBX_SSSP_PRECHECK 0  // plain load of the dedup word before its atomicOr
#endif
#ifndef GBX_SSSP_MINB
#define GBX_SSSP_MINB 4  // resident CTAs per SM (measured: 2 -> 160 ms, 3 -> 133, 4 -> 128 for config 4)
#endif
constexpr int kSsspWarps = kSsspThreads / 32;
constexpr int kSsspBuf = 256;  // staged pushes per warp and queue
#ifndef GBX_SSSP_SMALL
#define GBX_SSSP_SMALL 262144  // 0 / 4096 / 32768 / 262144 -> 67.0 / 66.0 / 65.5 / 64.9 ms per 16 sources (ER 2^24)
#endif
constexpr int64_t kSsspSmallBucket = GBX_SSSP_SMALL;
#ifndef GBX_SSSP_ORDERED
#define GBX_SSSP_ORDERED 4  // 0 (never) / 4 / 16 / 64 / 256 -> 65.4 / 64.3 / 66.7 / 73.7 / 78.0 ms per 16 sources (ER 2^24)
#endif
constexpr int64_t kSsspOrdered = GBX_SSSP_ORDERED;  // near queues above n / this are walked in vertex order (0: never)  // pops per bucket up to which the heavy pass walks a log
constexpr unsigned kFullW = 0xffffffffu;

template <typename D> struct DistTraits;
template <> struct DistTraits<uint32_t> {
  static __device__ __forceinline__ uint32_t inf() { return 0xffffffffu; }
  static __device__ __forceinline__ uint32_t add(uint32_t d, uint32_t w) { return d + w; }
  static __device__ __forceinline__ uint32_t bucket_hi(uint32_t lo, double delta) {
    double h = static_cast<double>(lo) + delta;
    return h >= 4294967295.0 ? 0xffffffffu : static_cast<uint32_t>(ceil(h));
  }
};
template <> struct DistTraits<unsigned long long> {
  static __device__ __forceinline__ unsigned long long inf() { return 0x7FF0000000000000ull; }
  static __device__ __forceinline__ unsigned long long add(unsigned long long d, double w) {
    return static_cast<unsigned long long>(__double_as_longlong(__longlong_as_double(d) + w));
  }
};

// edge readers
struct PackedEdges {
  const uint32_t* e;
  __device__ __forceinline__ void get(int64_t p, int32_t& v, uint32_t& w) const {
    uint32_t x;
    // the edge stream bypasses L1 (read once per relaxation pass; measured:
    // an L1-allocating load 83.5 vs 83.1 ms, an L2 evict-first policy 134 vs 121)
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(x) : "l"(e + p));
    v = static_cast<int32_t>(x >> 8);
    w = x & 0xffu;
  }
};
struct IntEdges {
  const int32_t* col;
  const int32_t* w;
  __device__ __forceinline__ void get(int64_t p, int32_t& v, uint32_t& ww) const {
    v = __ldg(col + p);
    ww = static_cast<uint32_t>(__ldg(w + p));
  }
};
struct DblEdges {
  const int32_t* col;
  const double* w;
  __device__ __forceinline__ void get(int64_t p, int32_t& v, double& ww) const {
    v = __ldg(col + p);
    ww = __ldg(w + p);
  }
};

// relaxation statistics: one atomic per warp (the per-thread atomicAdd on this
// single counter at the end of every phase serialised ~10^5 atomics in L2)
__device__ __forceinline__ void sssp_count_relax(unsigned long long* relax,
                                                 unsigned long long nrel) {
  const unsigned tot = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(nrel));
  if ((threadIdx.x & 31) == 0 && tot) atomicAdd(relax, static_cast<unsigned long long>(tot));
}

template <typename D, typename E>
struct SsspArgs {
  const int64_t* rp;
  E edges;
  int64_t n;
  double delta;
  D* dist;
  int32_t* q0;
  int32_t* q1;
  int32_t* f0;
  int32_t* f1;
  uint32_t* qbits[2];  // near-queue membership, alternating per near iteration
  uint32_t* fbits[2];  // far-pile membership, alternating per bucket epoch
  int* ctl;        // [0] |Q| [1] |Qnext| [2] |F| [3] |Fnext| [4] near iterations [5] buckets
  D* lohi;         // [0] lo [1] hi [2] min far (scratch)
  unsigned long long* relax;  // edges relaxed
};

template <typename D>
__device__ __forceinline__ D next_hi(D lo, double delta);
template <>
__device__ __forceinline__ uint32_t next_hi<uint32_t>(uint32_t lo, double delta) {
  return DistTraits<uint32_t>::bucket_hi(lo, delta);
}
template <>
__device__ __forceinline__ unsigned long long next_hi<unsigned long long>(unsigned long long lo,
                                                                         double delta) {
  return static_cast<unsigned long long>(__double_as_longlong(__longlong_as_double(lo) + delta));
}
template <typename D>
__device__ __forceinline__ D bucket_floor(D m, double delta);
template <>
__device__ __forceinline__ uint32_t bucket_floor<uint32_t>(uint32_t m, double delta) {
  return static_cast<uint32_t>(floor(static_cast<double>(m) / delta) * delta);
}
template <>
__device__ __forceinline__ unsigned long long bucket_floor<unsigned long long>(
    unsigned long long m, double delta) {
  double lo = floor(__longlong_as_double(m) / delta) * delta;
  return static_cast<unsigned long long>(__double_as_longlong(lo));
}

template <typename D, typename E, typename W>
__global__ void __launch_bounds__(kSsspThreads) k_sssp(SsspArgs<D, E> a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ int32_t s_near[kSsspWarps][kSsspBuf];
  __shared__ int32_t s_far[kSsspWarps][kSsspBuf];
  WarpQueue<int32_t, kSsspBuf> nearq, farq;
  nearq.buf = s_near[threadIdx.x >> 5];
  farq.buf = s_far[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t gtid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t gsize = int64_t(gridDim.x) * blockDim.x;
  int qp = 1;          // parity of the near-queue bitmap receiving pushes (the
                       // source sits in bitmap 0, released when it is popped)
  int fp = 0;          // parity of the far-pile bitmap of the current bucket epoch
  int pq = 0, pf = 0;  // parity of the current near queue / far pile
  for (;;) {
    // ---------------- near iterations inside the bucket
    for (;;) {
      const int nq = *(volatile int*)&a.ctl[0];
      if (nq == 0) break;
      const D hi = *(volatile D*)&a.lohi[1];
      const int32_t* qc = pq ? a.q1 : a.q0;
      int32_t* qn = pq ? a.q0 : a.q1;
      int32_t* fc = pf ? a.f1 : a.f0;
      unsigned long long nrel = 0;
      nearq.reset(qn, &a.ctl[1]);
      farq.reset(fc, &a.ctl[2]);
      // 4 lanes per queued vertex (8 vertices per warp), each lane relaxing 4
      // edges per round: 4 independent edge -> dist -> atomicMin chains
      const int g4 = lane >> 2, s4 = lane & 3;
      for (int64_t base = gwarp * 8; base < nq; base += nwarps * 8) {
        const int64_t qi = base + g4;
        bool active = qi < nq;
        int32_t u = active ? qc[qi] : 0;
        // u was queued through the other near bitmap: release its bit
        if (active && s4 == 0) atomicAnd(&a.qbits[qp ^ 1][u >> 5], ~(1u << (u & 31)));
        int64_t p = active ? a.rp[u] : 0;
        const int64_t e = active ? a.rp[u + 1] : 0;
        const D du = active ? *(volatile D*)&a.dist[u] : D(0);
        while (__any_sync(kFullW, active)) {
          int32_t v[4];
          D nd[4];
          bool ok[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int64_t q = p + s4 + 4 * t;
            ok[t] = active && q < e;
            W w = W(0);
            v[t] = 0;
            if (ok[t]) a.edges.get(q, v[t], w);
            GBX_DCHECK(v[t] >= 0 && v[t] < a.n, "sssp edge target", v[t]);
            nd[t] = DistTraits<D>::add(du, w);
          }
          D cur[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) cur[t] = ok[t] ? *(volatile D*)&a.dist[v[t]] : D(0);
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            bool near_push = false, far_push = false;
            if (ok[t]) {
              ++nrel;
              if (nd[t] < cur[t]) {
                const D old = atomicMin(&a.dist[v[t]], nd[t]);
                if (nd[t] < old) {
                  const uint32_t bit = 1u << (v[t] & 31);
                  if (nd[t] < hi) near_push = !(atomicOr(&a.qbits[qp][v[t] >> 5], bit) & bit);
                  else far_push = !(atomicOr(&a.fbits[fp][v[t] >> 5], bit) & bit);
                }
              }
            }
            nearq.push(near_push, v[t]);
            farq.push(far_push, v[t]);
          }
          if (active) {
            p += 16;
            if (p >= e) active = false;
          }
        }
      }
      nearq.flush();
      farq.flush();
      sssp_count_relax(a.relax, nrel);
      grid.sync();
      if (gtid == 0) {
        a.ctl[0] = a.ctl[1];
        a.ctl[1] = 0;
        a.ctl[4] += 1;
      }
      pq ^= 1;
      qp ^= 1;
      grid.sync();
    }
    // ---------------- bucket jump: min over the far pile at or above hi
    const int nf = *(volatile int*)&a.ctl[2];
    if (nf == 0) break;
    const int32_t* fc = pf ? a.f1 : a.f0;
    int32_t* fn = pf ? a.f0 : a.f1;
    const D hi = *(volatile D*)&a.lohi[1];
    {
      D m = DistTraits<D>::inf();
      for (int64_t i = gtid; i < nf; i += gsize) {
        const D d = *(volatile D*)&a.dist[fc[i]];
        if (d >= hi && d < m) m = d;
      }
      for (int o = 16; o > 0; o >>= 1) {
        D t = __shfl_xor_sync(kFullW, m, o);
        m = t < m ? t : m;
      }
      if (lane == 0 && m != DistTraits<D>::inf()) atomicMin(&a.lohi[2], m);
    }
    grid.sync();
    const D mfar = *(volatile D*)&a.lohi[2];
    if (mfar == DistTraits<D>::inf()) break;  // every far entry was stale
    const D lo2 = bucket_floor<D>(mfar, a.delta);
    D hi2 = next_hi<D>(lo2, a.delta);
    if (!(mfar < hi2)) hi2 = mfar + 1;  // rounding guard: the bucket must hold mfar
                                         // (for fp64 bit patterns: the next double up)
    // split the pile: [lo2, hi2) -> near queue, >= hi2 -> stays far, < hi stale
    int32_t* qn = pq ? a.q1 : a.q0;  // current (empty) near queue
    nearq.reset(qn, &a.ctl[0]);
    farq.reset(fn, &a.ctl[3]);
    for (int64_t base = gwarp * 32; base < nf; base += nwarps * 32) {
      const int64_t i = base + lane;
      bool to_near = false, to_far = false;
      int32_t v = 0;
      if (i < nf) {
        v = fc[i];
        const uint32_t bit = 1u << (v & 31);
        atomicAnd(&a.fbits[fp][v >> 5], ~bit);  // leaves this epoch's pile
        const D d = *(volatile D*)&a.dist[v];
        if (d >= hi) {
          if (d < hi2) to_near = !(atomicOr(&a.qbits[qp][v >> 5], bit) & bit);
          else to_far = !(atomicOr(&a.fbits[fp ^ 1][v >> 5], bit) & bit);
        }
      }
      nearq.push(to_near, v);
      farq.push(to_far, v);
    }
    nearq.flush();
    farq.flush();
    grid.sync();
    if (gtid == 0) {
      a.lohi[0] = lo2;
      a.lohi[1] = hi2;
      a.lohi[2] = DistTraits<D>::inf();
      a.ctl[2] = a.ctl[3];
      a.ctl[3] = 0;
      a.ctl[5] += 1;
    }
    pf ^= 1;
    fp ^= 1;
    qp ^= 1;  // the new near queue was marked in qbits[qp]: popped next, released there
    grid.sync();
  }
}

// ---------------------------------------------------------------------------
// Circular-bucket variant (used when NB = pow2 >= 2 + max_w / delta <= 64):
// an improvement nd >= hi goes straight into bucket floor(nd/delta) mod NB (it
// cannot be more than max_w/delta buckets ahead of the current one), so a
// bucket jump reads ONE bucket instead of rescanning a far pile.
// ---------------------------------------------------------------------------
template <typename D>
__device__ __forceinline__ int64_t bucket_of(D d, double delta);
template <>
__device__ __forceinline__ int64_t bucket_of<uint32_t>(uint32_t d, double delta) {
  return static_cast<int64_t>(floor(static_cast<double>(d) / delta));
}
template <>
__device__ __forceinline__ int64_t bucket_of<unsigned long long>(unsigned long long d,
                                                                 double delta) {
  return static_cast<int64_t>(floor(__longlong_as_double(static_cast<long long>(d)) / delta));
}

// bucket index of an integer distance without the fp64 division when delta is
// an integer (a shift for a power of two: config 4's delta = 64)
template <typename D, typename A>
__device__ __forceinline__ int64_t bucket_k(D d, const A& a) {
#if GBX_SSSP_IBUCKET
  if constexpr (std::is_same<D, uint32_t>::value) {
    if (a.dshift >= 0) return static_cast<int64_t>(d >> a.dshift);
    if (a.idelta) return static_cast<int64_t>(d / a.idelta);
  }
#endif
  return bucket_of<D>(d, a.delta);
}

// lower dist[v] to nd (an improvement landing in the later bucket kb) and
// report whether v must be appended to kb's queue: exactly when the distance
// it replaced was not already in bucket kb (infinite, or a later bucket --
// that entry goes stale).  One returning atomic replaces the fire-and-forget
// min + the returning atomicOr on a per-bucket membership bitmap.
template <typename D, typename A>
__device__ __forceinline__ bool bucket_enter(D* dist, D nd, int64_t kb, const A& a) {
  const D old = atomicMin(dist, nd);
  if (!(nd < old)) return false;
  return old == DistTraits<D>::inf() || bucket_k<D>(old, a) != kb;
}

template <typename D, typename E>
struct SsspBArgs {
  const int64_t* rp;
  E edges;
  int64_t n;
  double delta;
  int dshift;          // delta = 2^dshift (integer distances), else -1
  uint32_t idelta;     // integral delta (integer distances), else 0
  int nb;              // buckets (power of two)
  int64_t cap;         // entries per bucket array
  D* dist;
  int32_t* q0;
  int32_t* q1;
  int32_t* bq;         // [nb][cap]
  int* bcnt;           // [nb]
  uint32_t* qbits[2];  // near-queue membership (parity per near iteration)
  uint32_t* bbits;     // [nb][words] bucket membership
  int64_t words;
  int* ctl;            // [0..2] queue counts [4] near iterations [5] buckets [6,7] jump [8] |S|
  unsigned long long* relax;
  // light/heavy split (Delta-stepping proper, sssp.cpp:30-33, 66-106): every
  // row holds its light edges (w <= delta) first, nl[u] of them.  Near
  // iterations relax light edges only and, when the bucket drains, the heavy
  // edges of every vertex it settled are relaxed ONCE from their final
  // distances (they always land in a later bucket).  nl == nullptr: every edge
  // in the near phase (label-correcting).
  const int32_t* nl;
  const uint4* vm;     // {begin, light end, end, 0} per vertex, or nullptr
  // pull form of the heavy pass (packed edges): every still-unsettled vertex
  // scans its heavy in-edges in ascending weight until lo_k + w >= its
  // distance; chosen for a bucket when its pops * 100 > pull_pct * (vertices
  // not yet popped), i.e. when the settled set outweighs what is left
  const uint32_t* hrp;
  const uint32_t* hin;
  int pull_pct;
  int light_group;     // lanes per vertex in the light (near) phase: 1, 2 or 4
  // small buckets: while a bucket has popped <= slog_cap vertices its near
  // iterations log them (ctl[8] entries, a vertex popped twice is listed
  // twice: its heavy edges are then relaxed twice from the same final
  // distance), and the heavy pass walks the log instead of the dense pass
  // over dist (~25 us per bucket at 2^24 vertices)
  int32_t* slog;
  int slog_cap;
  int trace;
  unsigned long long* tlog;  // optional: [2i] %globaltimer, [2i+1] kind<<32 | size (debug)
  int tlog_cap;
};

__device__ __forceinline__ unsigned long long sssp_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// stages (vertex, bucket) pushes; a flush counts the staged entries per
// bucket in shared memory and reserves each bucket's run with ONE global
// atomic (the nb bucket counters are the hottest addresses of the kernel:
// one atomic per 32 entries and bucket serialised in L2)
template <int CAP>
struct BucketQueue {
  int32_t* bv;
  int32_t* bb;   // bucket, then bucket | slot << 8 during a flush
  int* scnt;     // [64] per-bucket counts / bases (warp-private)
  int n;
  __device__ __forceinline__ void flush(int32_t* bq, int64_t cap, int* bcnt, int nb) {
    __syncwarp();
    if (n == 0) return;
    const int lane = threadIdx.x & 31;
    for (int t = lane; t < nb; t += 32) scnt[t] = 0;
    __syncwarp();
    for (int i = lane; i < n; i += 32) {
      const int b = bb[i];
      bb[i] = b | (atomicAdd(&scnt[b], 1) << 8);
    }
    __syncwarp();
    for (int t = lane; t < nb; t += 32) {
      const int c = scnt[t];
      scnt[t] = c ? atomicAdd(&bcnt[t], c) : 0;
    }
    __syncwarp();
    for (int i = lane; i < n; i += 32) {
      const int x = bb[i];
      const int b = x & 0xff;
      bq[static_cast<int64_t>(b) * cap + scnt[b] + (x >> 8)] = bv[i];
    }
    __syncwarp();
    n = 0;
  }
  __device__ __forceinline__ void push(bool has, int32_t v, int b, int32_t* bq, int64_t cap,
                                       int* bcnt, int nb) {
    const unsigned m = __ballot_sync(0xffffffffu, has);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    if (has) {
      const int pos = n + __popc(m & ((1u << lane) - 1));
      bv[pos] = v;
      bb[pos] = b;
    }
    n += __popc(m);
    if (n > CAP - 32) flush(bq, cap, bcnt, nb);
  }
};

template <typename D, typename E, typename W>
__global__ void __launch_bounds__(kSsspThreads, GBX_SSSP_MINB) k_sssp_b(SsspBArgs<D, E> a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ int32_t s_near[kSsspWarps][kSsspBuf];
  __shared__ int32_t s_bv[kSsspWarps][kSsspBuf];
  __shared__ int32_t s_bb[kSsspWarps][kSsspBuf];
  __shared__ int s_bcnt[kSsspWarps][64];
  __shared__ int32_t s_settle[kSsspWarps][kSsspBuf];
  WarpQueue<int32_t, kSsspBuf> nearq;
  BucketQueue<kSsspBuf> bucq;
  nearq.buf = s_near[threadIdx.x >> 5];
  bucq.bv = s_bv[threadIdx.x >> 5];
  bucq.bb = s_bb[threadIdx.x >> 5];
  bucq.scnt = s_bcnt[threadIdx.x >> 5];
  bucq.n = 0;
  const int lane = threadIdx.x & 31;
  const int g4 = lane >> 2, s4 = lane & 3;
  const int64_t gwarp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int nbm = a.nb - 1;
  int64_t k = 0;  // current bucket (absolute index)
  // near iteration t pops queue t&1 (count ctl[t%3], dedup bits qbits[t&1])
  // and pushes queue (t+1)&1 (count ctl[(t+1)%3]); ctl[(t+2)%3] -- read by
  // every thread before the previous barrier -- is zeroed for iteration t+1,
  // so ONE grid barrier per near iteration suffices
  int t = 0;
  int zero_bucket = -1;  // bucket emptied by the last jump, cleared lazily
  const bool trace = a.trace && blockIdx.x == 0 && threadIdx.x == 0;
  const bool tl = a.tlog && blockIdx.x == 0 && threadIdx.x == 0;
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  int tn = 0;
  // pops of the current bucket / of all buckets so far (every thread reads each
  // near iteration's count, so every thread takes the same push / pull decision)
  int64_t popped_k = 0, popped_all = 0;
  bool log_pops = false;  // this near iteration logs its pops (the bucket is still small)
  // relax the edges of the vertices list[0, cnt): phase 0 all edges, 1 light
  // edges (and record the vertex in the settled list), 2 heavy edges.  4 lanes
  // per vertex (8 vertices per warp), each lane 4 edges per round: 4
  // independent edge -> dist -> atomicMin chains.  pop_bits: the list's
  // membership bitmap, released as entries are taken.
  // local: the list is this warp's own (shared memory window), walked by the
  // warp alone; else the grid shares it warp-strided
  auto relax = [&](auto gsz, const int32_t* list, int cnt, int phase, uint32_t* pop_bits,
                   uint32_t* push_bits, unsigned long long& nrel, bool local = false) {
    constexpr int G = decltype(gsz)::value;  // lanes per vertex
    constexpr int VPW = 32 / G;              // vertices per warp step
    const int gi = lane / G, si = lane % G;
    const int64_t first = local ? 0 : gwarp * VPW, stride = local ? VPW : nwarps * VPW;
    for (int64_t base = first; base < cnt; base += stride) {
      const int64_t qi = base + gi;
      bool active = qi < cnt;
      const int32_t u = active ? list[qi] : 0;
      const uint32_t ubit = 1u << (u & 31);
      if (active && si == 0 && pop_bits) atomicAnd(&pop_bits[u >> 5], ~ubit);
      if (active && si == 0 && log_pops) a.slog[atomicAdd(&a.ctl[8], 1)] = u;
      int64_t p = 0, e = 0;
      if (a.vm) {
        if (active) {
          const uint4 m = __ldg(a.vm + u);
          p = phase == 2 ? m.y : m.x;
          e = phase == 1 ? m.y : m.z;
        }
      } else {
        p = active ? a.rp[u] : 0;
        e = active ? a.rp[u + 1] : 0;
        if (active && phase == 1) e = p + a.nl[u];
        if (active && phase == 2) p += a.nl[u];
      }
      if (p >= e) active = false;
      const D du = active ? *(volatile D*)&a.dist[u] : D(0);
      while (__any_sync(kFullW, active)) {
        int32_t v[4];
        D nd[4];
        bool ok[4];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const int64_t q = p + si + G * q4;
          ok[q4] = active && q < e;
          W w = W(0);
          v[q4] = 0;
          if (ok[q4]) a.edges.get(q, v[q4], w);
          GBX_DCHECK(v[q4] >= 0 && v[q4] < a.n, "sssp edge target", v[q4]);
          nd[q4] = DistTraits<D>::add(du, w);
        }
        D cur[4];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) cur[q4] = ok[q4] ? *(volatile D*)&a.dist[v[q4]] : D(0);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          bool near_push = false, buck_push = false;
          int bidx = 0;
          if (ok[q4]) {
            ++nrel;
            if (nd[q4] < cur[q4]) {
              const uint32_t bit = 1u << (v[q4] & 31);
              const int64_t kb = bucket_k<D>(nd[q4], a);
              if (kb <= k && phase != 2) {  // (a heavy edge always leaves the bucket)
                // fire-and-forget min: a push whose value lost the race is a
                // harmless extra relaxation; the near queue dedups by bitmap
                atomicMin(&a.dist[v[q4]], nd[q4]);
                near_push = !(atomicOr(&push_bits[v[q4] >> 5], bit) & bit);
              } else {
                // a later bucket: the returned old distance is the dedup -- v
                // already sits in bucket kb's queue iff its old distance did
                bidx = static_cast<int>(kb & nbm);
                buck_push = bucket_enter<D>(&a.dist[v[q4]], nd[q4], kb, a);
              }
            }
          }
          if (phase != 2) nearq.push(near_push, v[q4]);
          bucq.push(buck_push, v[q4], bidx, a.bq, a.cap, a.bcnt, a.nb);
        }
        if (active) {
          p += 4 * G;
          if (p >= e) active = false;
        }
      }
    }
  };
  // heavy edges of the vertices win[0, c) (warp-local list, every lane calls)
  auto relax_local = [&](const int32_t* win, int c, unsigned long long& nrel) {
    for (int base = 0; base < c; base += 8) {
      const int qi = base + g4;
      bool active = qi < c;
      const int32_t u = active ? win[qi] : 0;
      int64_t p = 0, e = 0;
      if (active) {
        if (a.vm) {
          const uint4 m = __ldg(a.vm + u);
          p = m.y;
          e = m.z;
        } else {
          p = a.rp[u] + a.nl[u];
          e = a.rp[u + 1];
        }
      }
      if (p >= e) active = false;
      const D du = active ? *(volatile D*)&a.dist[u] : D(0);
      while (__any_sync(kFullW, active)) {
        int32_t v[4];
        D nd[4];
        bool ok[4];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const int64_t q = p + s4 + 4 * q4;
          ok[q4] = active && q < e;
          W w = W(0);
          v[q4] = 0;
          if (ok[q4]) a.edges.get(q, v[q4], w);
          GBX_DCHECK(v[q4] >= 0 && v[q4] < a.n, "sssp edge target", v[q4]);
          nd[q4] = DistTraits<D>::add(du, w);
        }
        D cur[4];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) cur[q4] = ok[q4] ? *(volatile D*)&a.dist[v[q4]] : D(0);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          bool buck_push = false;
          int bidx = 0;
          if (ok[q4]) {
            ++nrel;
            if (nd[q4] < cur[q4]) {
              const int64_t kb = bucket_k<D>(nd[q4], a);
              bidx = static_cast<int>(kb & nbm);
              buck_push = bucket_enter<D>(&a.dist[v[q4]], nd[q4], kb, a);
            }
          }
          bucq.push(buck_push, v[q4], bidx, a.bq, a.cap, a.bcnt, a.nb);
        }
        if (active) {
          p += 16;
          if (p >= e) active = false;
        }
      }
    }
  };
  // pull form of the heavy pass (packed plans, u32 distances): the unsettled
  // vertices win[0, c) (distances in win[128 + i]) scan their heavy in-edges in
  // ascending weight, 4 lanes per vertex, 4 edges per lane and round.  Only a
  // source settled in bucket <= k counts -- its improvement then
  // lands within nb-1 buckets, as a push would -- and the scan stops at the
  // first weight with lo + w >= the lane's best (weights ascend, every settled
  // source of bucket k has du >= lo, earlier buckets already pushed).  The
  // vertex is written by its own group only (no atomics): plain store of the
  // minimum, queued in its bucket unless its old distance was already there.
  auto pull_local = [&](const int32_t* win, int c, uint32_t lo, unsigned long long& nrel) {
    for (int base = 0; base < c; base += 8) {
      const int qi = base + g4;
      bool active = qi < c;
      const int32_t v = active ? win[qi] : 0;
      const uint32_t dv = active ? static_cast<uint32_t>(win[128 + qi]) : 0u;
      uint32_t p = 0, e = 0;
      if (active) {
        p = __ldg(a.hrp + v);
        e = __ldg(a.hrp + v + 1);
      }
      if (p >= e) active = false;
      uint32_t best = dv;
      while (__any_sync(kFullW, active)) {
        uint32_t x[4];
        bool ok[4];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const uint32_t q = p + s4 + 4 * q4;
          ok[q4] = active && q < e;
          x[q4] = 0;
          if (ok[q4])
            asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(x[q4]) : "l"(a.hin + q));
        }
        bool stop = !active;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4)
          if (ok[q4] && static_cast<uint64_t>(lo) + (x[q4] & 0xffu) >= best) {
            ok[q4] = false;
            stop = true;
          }
        uint32_t du[4];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          GBX_DCHECK(!ok[q4] || static_cast<int64_t>(x[q4] >> 8) < a.n, "sssp in-edge source", x[q4] >> 8);
          du[q4] = ok[q4] ? __ldcg(reinterpret_cast<const uint32_t*>(a.dist) + (x[q4] >> 8))
                          : 0xffffffffu;
        }
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4)
          if (ok[q4]) {
            ++nrel;
            if (du[q4] != 0xffffffffu && bucket_k<D>(static_cast<D>(du[q4]), a) <= k) {
              const uint32_t nd = du[q4] + (x[q4] & 0xffu);
              best = nd < best ? nd : best;
            }
          }
        p += 16;
        if (stop || p >= e) active = false;
      }
      // the group's minimum (4 lanes, uniform shuffles)
      uint32_t o = __shfl_xor_sync(kFullW, best, 1);
      best = o < best ? o : best;
      o = __shfl_xor_sync(kFullW, best, 2);
      best = o < best ? o : best;
      bool push = false;
      int bidx = 0;
      if (qi < c && s4 == 0 && best < dv) {
        reinterpret_cast<uint32_t*>(a.dist)[v] = best;
        const int64_t kb = bucket_k<D>(static_cast<D>(best), a);
        bidx = static_cast<int>(kb & nbm);
        push = dv == 0xffffffffu || bucket_k<D>(static_cast<D>(dv), a) != kb;
      }
      bucq.push(push, v, bidx, a.bq, a.cap, a.bcnt, a.nb);
    }
  };
  for (int guard = 0;; ++guard) {
    if (guard > (1 << 28)) break;
    // ---------------- near iterations inside bucket k
    for (;;) {
      const int nq = *(volatile int*)&a.ctl[t % 3];
      if (trace) printf("near k=%lld nq=%d t=%d\n", (long long)k, nq, t);
      if (tl && tn < a.tlog_cap) {
        a.tlog[2 * tn] = sssp_gtimer();
        a.tlog[2 * tn + 1] = (static_cast<unsigned long long>(k) << 32) | static_cast<unsigned>(nq);
        ++tn;
      }
      if (nq == 0) break;
      popped_k += nq;
      if (leader) {
        a.ctl[(t + 2) % 3] = 0;
        a.ctl[4] += 1;
        if (zero_bucket >= 0) a.bcnt[zero_bucket] = 0;
      }
      zero_bucket = -1;
      log_pops = a.nl && a.slog && popped_k <= a.slog_cap;
      const int32_t* qc = (t & 1) ? a.q1 : a.q0;
      int32_t* qn = (t & 1) ? a.q0 : a.q1;
      uint32_t* pop_bits = a.qbits[t & 1];
      uint32_t* push_bits = a.qbits[(t + 1) & 1];
      unsigned long long nrel = 0;
      nearq.reset(qn, &a.ctl[(t + 1) % 3]);
      // large queues release their dedup bitmap wholesale (coalesced stores;
      // the next push into it is two barriers away) instead of one atomicAnd
      // per popped entry
      // big queues (> n / kSsspOrdered of the vertices, split plans) are walked in
      // VERTEX order through their membership bitmap instead of in push order:
      // the vertex records and the light edges of the popped vertices are then
      // read front to back (DRAM pages, shared sectors) instead of one random
      // sector each; the warp clears the bitmap words it has read
      const bool ordered = a.nl && a.light_group == 2 && kSsspOrdered > 0 &&
                           static_cast<int64_t>(nq) * kSsspOrdered > a.n;
      const bool dense_clear = !ordered && static_cast<int64_t>(nq) * 8 > a.words;
      if (dense_clear)
        for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < a.words;
             i += int64_t(gridDim.x) * blockDim.x)
          pop_bits[i] = 0u;
      uint32_t* pb = dense_clear ? nullptr : pop_bits;
      if (ordered) {
        int32_t* win = s_settle[threadIdx.x >> 5];
        for (int64_t base = gwarp * 128; base < a.n; base += nwarps * 128) {
          // 4 bitmap words = 128 vertices per step; lane l tests bit l of each
          uint32_t wd[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int64_t wi = (base >> 5) + j;
            wd[j] = wi < a.words ? *(volatile uint32_t*)&pop_bits[wi] : 0u;
          }
          int c = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const bool in = (wd[j] >> lane) & 1u;
            if (in) win[c + __popc(wd[j] & ((1u << lane) - 1))] = static_cast<int32_t>(base + 32 * j + lane);
            c += __popc(wd[j]);
          }
          if (lane < 4 && (base >> 5) + lane < a.words && wd[lane]) pop_bits[(base >> 5) + lane] = 0u;
          __syncwarp();
          if (c) relax(std::integral_constant<int, 2>{}, win, c, 1, nullptr, push_bits, nrel, true);
          __syncwarp();
        }
      } else if (!a.nl) relax(std::integral_constant<int, 4>{}, qc, nq, 0, pb, push_bits, nrel);
      else if (a.light_group == 1) relax(std::integral_constant<int, 1>{}, qc, nq, 1, pb, push_bits, nrel);
      else if (a.light_group == 2) relax(std::integral_constant<int, 2>{}, qc, nq, 1, pb, push_bits, nrel);
      else relax(std::integral_constant<int, 4>{}, qc, nq, 1, pb, push_bits, nrel);
      nearq.flush();
      bucq.flush(a.bq, a.cap, a.bcnt, a.nb);
      sssp_count_relax(a.relax, nrel);
      grid.sync();
      ++t;
    }
    // ---------------- heavy edges of every vertex the bucket settled, once:
    // a dense pass over dist (4 B/vertex, coalesced) finds the vertices whose
    // final distance lies in bucket k -- cheaper than recording them (one more
    // atomic per near visit); each warp compacts its 32-vertex window into
    // shared memory and relaxes the heavy edges 8 vertices at a time
    popped_all += popped_k;
    // every near iteration of the bucket logged its pops: walk the log
    const bool small = a.nl && a.slog && popped_k <= a.slog_cap;
    const bool pull = !small && a.hin != nullptr &&
                      popped_k * 100 > static_cast<int64_t>(a.pull_pct) * (a.n - popped_all);
    popped_k = 0;
    log_pops = false;
    if (tl && tn < a.tlog_cap) {
      a.tlog[2 * tn] = sssp_gtimer();
      a.tlog[2 * tn + 1] = (1ull << 62) | (pull ? 1ull : 0ull);
      ++tn;
    }
    if (small) {
      unsigned long long nrel = 0;
      const int cnt = *(volatile int*)&a.ctl[8];
      if (cnt) {
        relax(std::integral_constant<int, 4>{}, a.slog, cnt, 2, nullptr, nullptr, nrel);
        bucq.flush(a.bq, a.cap, a.bcnt, a.nb);
        sssp_count_relax(a.relax, nrel);
        grid.sync();  // before the leader below re-zeroes ctl[8]
      }
    } else if (a.nl && pull) {
      if constexpr (std::is_same<D, uint32_t>::value) {
        unsigned long long nrel = 0;
        int32_t* win = s_settle[threadIdx.x >> 5];
        // a lower bound of bucket k's distances (exact for an integral delta;
        // one below the rounded product otherwise: the pruning stays safe)
        const double lod = a.idelta ? static_cast<double>(k) * a.idelta
                                    : floor(static_cast<double>(k) * a.delta) - 1.0;
        const uint32_t lo = lod <= 0.0 ? 0u
                            : lod >= 4294967295.0 ? 0xffffffffu : static_cast<uint32_t>(lod);
        for (int64_t base = gwarp * 128; base < a.n; base += nwarps * 128) {
          uint32_t dv[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int64_t v = base + 32 * j + lane;
            dv[j] = v < a.n ? __ldcg(reinterpret_cast<const uint32_t*>(a.dist) + v) : 0u;
          }
          int c = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            // unsettled (a later bucket) or unreached
            const bool in = base + 32 * j + lane < a.n &&
                            (dv[j] == 0xffffffffu || bucket_k<D>(static_cast<D>(dv[j]), a) > k);
            const unsigned m = __ballot_sync(kFullW, in);
            if (in) {
              const int pos = c + __popc(m & ((1u << lane) - 1));
              win[pos] = static_cast<int32_t>(base + 32 * j + lane);
              win[128 + pos] = static_cast<int32_t>(dv[j]);
            }
            c += __popc(m);
          }
          __syncwarp();
          if (c) pull_local(win, c, lo, nrel);
          __syncwarp();
        }
        bucq.flush(a.bq, a.cap, a.bcnt, a.nb);
        sssp_count_relax(a.relax, nrel);
        grid.sync();
      }
    } else if (a.nl) {
      unsigned long long nrel = 0;
      int32_t* win = s_settle[threadIdx.x >> 5];
      for (int64_t base = gwarp * 128; base < a.n; base += nwarps * 128) {
        D dv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // 4 independent coalesced loads in flight
          const int64_t v = base + 32 * j + lane;
          dv[j] = v < a.n ? __ldcg(&a.dist[v]) : DistTraits<D>::inf();
        }
        int c = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const bool in = dv[j] != DistTraits<D>::inf() && bucket_k<D>(dv[j], a) == k;
          const unsigned m = __ballot_sync(kFullW, in);
          if (in) win[c + __popc(m & ((1u << lane) - 1))] = static_cast<int32_t>(base + 32 * j + lane);
          c += __popc(m);
        }
        __syncwarp();
        if (c) relax_local(win, c, nrel);
        __syncwarp();
      }
      bucq.flush(a.bq, a.cap, a.bcnt, a.nb);
      sssp_count_relax(a.relax, nrel);
      grid.sync();
    }
    // ---------------- jump to the next non-empty bucket (at most nb-1 ahead):
    // one thread decides, everyone reads the decision after a grid barrier
    if (leader) {
      if (zero_bucket >= 0) a.bcnt[zero_bucket] = 0;  // the near loop ran no iteration
      int jj = 1;
      for (; jj < a.nb; ++jj)
        if (*(volatile int*)&a.bcnt[(k + jj) & nbm] > 0) break;
      a.ctl[6] = jj;
      a.ctl[7] = jj < a.nb ? *(volatile int*)&a.bcnt[(k + jj) & nbm] : 0;
      a.ctl[5] += 1;
      a.ctl[8] = 0;  // the settled list was consumed by the heavy phase
    }
    zero_bucket = -1;
    grid.sync();
    const int j = *(volatile int*)&a.ctl[6];
    if (trace) printf("jump k=%lld j=%d\n", (long long)k, j);
    if (tl && tn < a.tlog_cap) {
      a.tlog[2 * tn] = sssp_gtimer();
      a.tlog[2 * tn + 1] = (1ull << 63) | static_cast<unsigned>(*(volatile int*)&a.ctl[7]);
      ++tn;
    }
    if (j >= a.nb) {
      if (tl && tn < a.tlog_cap) {
        a.tlog[2 * tn] = sssp_gtimer();
        a.tlog[2 * tn + 1] = 3ull << 62;
        ++tn;
      }
      break;
    }
    k += j;
    const int b = static_cast<int>(k & nbm);
    const int cnt = *(volatile int*)&a.ctl[7];
    const int32_t* src = a.bq + static_cast<int64_t>(b) * a.cap;
    // the near queue iteration t pops (empty: the loop above ended on it)
    int32_t* qn = (t & 1) ? a.q1 : a.q0;
    uint32_t* push_bits = a.qbits[t & 1];
    nearq.reset(qn, &a.ctl[t % 3]);
    for (int64_t base = gwarp * 32; base < cnt; base += nwarps * 32) {
      const int64_t i = base + lane;
      bool to_near = false;
      int32_t v = 0;
      if (i < cnt) {
        v = src[i];
        const uint32_t bit = 1u << (v & 31);
        // stale entries (improved into an earlier bucket since) are skipped
        if (bucket_k<D>(*(volatile D*)&a.dist[v], a) == k)
          to_near = !(atomicOr(&push_bits[v >> 5], bit) & bit);
      }
      nearq.push(to_near, v);
    }
    nearq.flush();
    // bcnt[b] is zeroed by the next near iteration's leader: no push can
    // target bucket b before k moves past it
    zero_bucket = b;
    grid.sync();
  }
}

template <typename D>
__global__ void k_sssp_init(D* dist, uint32_t* bits, int64_t n, int32_t src, int32_t* q0, int* ctl,
                            D* lohi, unsigned long long* relax, D hi0, D inf) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) dist[i] = i == src ? D(0) : inf;
  const int64_t words = (n + 31) / 32;
  if (i < 4 * words) bits[i] = 0u;
  if (i == 0) bits[src >> 5] |= 1u << (src & 31);  // the source sits in near queue 0
  if (i == 0) {
    q0[0] = src;
    for (int k = 0; k < 10; ++k) ctl[k] = 0;
    ctl[0] = 1;
    lohi[0] = D(0);
    lohi[1] = hi0;
    lohi[2] = inf;
    *relax = 0;
  }
}

template <typename D>
__global__ void k_sssp_out(const D* dist, int64_t n, double* out);
template <>
__global__ void k_sssp_out<uint32_t>(const uint32_t* dist, int64_t n, double* out) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = dist[i] == 0xffffffffu ? __longlong_as_double(0x7FF0000000000000ll)
                                              : static_cast<double>(dist[i]);
}
template <>
__global__ void k_sssp_out<unsigned long long>(const unsigned long long* dist, int64_t n,
                                               double* out) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = __longlong_as_double(static_cast<long long>(dist[i]));
}

// ---- plan ------------------------------------------------------------------------

__global__ void k_weight_stats(const uint8_t* val, int dom, int64_t nnz, int* bad_nonpos,
                               int* nonint, double* maxw) {
  int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  double w = 0;
  bool ni = false, np = false;
  if (p < nnz) {
    if (dom == GBX_FP64) {
      w = reinterpret_cast<const double*>(val)[p];
      np = !(w > 0.0);
      ni = !(w == floor(w)) || w > 2147483647.0;
    } else {
      w = reinterpret_cast<const int32_t*>(val)[p];
      np = !(w > 0.0);
    }
  }
  if (np) atomicOr(bad_nonpos, 1);
  if (ni) atomicOr(nonint, 1);
  typedef cub::BlockReduce<double, 256> BR;
  __shared__ typename BR::TempStorage t;
  double m = BR(t).Reduce(p < nnz ? w : -1.0, cub::Max());
  if (threadIdx.x == 0) {
    // max of non-negative doubles via integer atomicMax on the bit pattern
    if (m > 0) atomicMax(reinterpret_cast<unsigned long long*>(maxw),
                         static_cast<unsigned long long>(__double_as_longlong(m)));
  }
}

__global__ void k_pack_edges(const int32_t* col, const uint8_t* val, int dom, int64_t nnz,
                             uint32_t* packed, int32_t* wint) {
  int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p >= nnz) return;
  int32_t w = dom == GBX_FP64 ? static_cast<int32_t>(reinterpret_cast<const double*>(val)[p])
                              : reinterpret_cast<const int32_t*>(val)[p];
  if (packed) packed[p] = (static_cast<uint32_t>(col[p]) << 8) | static_cast<uint32_t>(w);
  if (wint) wint[p] = w;
}

// light-first partition of every row for one delta (stable within each side):
// thread per row, a counting pass then a writing pass.  Light = w <= delta
// (sssp.cpp:30-33).
__global__ void k_split_packed(const int64_t* rp, int64_t n, double delta, const uint32_t* src,
                               uint32_t* dst, int32_t* nl) {
  const int64_t u = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (u >= n) return;
  const int64_t b = rp[u], e = rp[u + 1];
  int64_t c = 0;
  for (int64_t p = b; p < e; ++p) c += static_cast<double>(src[p] & 0xffu) <= delta;
  int64_t lo = b, hi = b + c;
  for (int64_t p = b; p < e; ++p) {
    const uint32_t x = src[p];
    if (static_cast<double>(x & 0xffu) <= delta) dst[lo++] = x; else dst[hi++] = x;
  }
  nl[u] = static_cast<int32_t>(c);
}
template <typename W>
__global__ void k_split_cw(const int64_t* rp, int64_t n, double delta, const int32_t* col,
                           const W* w, int32_t* ocol, W* ow, int32_t* nl) {
  const int64_t u = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (u >= n) return;
  const int64_t b = rp[u], e = rp[u + 1];
  int64_t c = 0;
  for (int64_t p = b; p < e; ++p) c += static_cast<double>(w[p]) <= delta;
  int64_t lo = b, hi = b + c;
  for (int64_t p = b; p < e; ++p) {
    const int64_t q = static_cast<double>(w[p]) <= delta ? lo++ : hi++;
    ocol[q] = col[p];
    ow[q] = w[p];
  }
  nl[u] = static_cast<int32_t>(c);
}

__global__ void k_vmeta(const int64_t* rp, const int32_t* nl, int64_t n, uint4* vm) {
  const int64_t u = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (u >= n) return;
  const uint32_t b = static_cast<uint32_t>(rp[u]);
  vm[u] = make_uint4(b, b + static_cast<uint32_t>(nl[u]), static_cast<uint32_t>(rp[u + 1]), 0u);
}

// heavy in-edges for the pull form of the heavy pass: (v:24 | w:8) keys with
// the source u as value, one thread per (light-first) row
__global__ void k_heavy_in_keys(const int64_t* rp, const int32_t* nl, int64_t n,
                                const uint32_t* pe, const int64_t* hoff, uint32_t* key,
                                uint32_t* src) {
  const int64_t u = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (u >= n) return;
  int64_t q = hoff[u];
  for (int64_t p = rp[u] + nl[u]; p < rp[u + 1]; ++p, ++q) {
    const uint32_t x = pe[p];
    key[q] = ((x >> 8) << 8) | (x & 0xffu);
    src[q] = static_cast<uint32_t>(u);
  }
}
__global__ void k_heavy_count(const int64_t* rp, const int32_t* nl, int64_t n, int64_t* cnt) {
  const int64_t u = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (u < n) cnt[u] = rp[u + 1] - rp[u] - nl[u];
  if (u == n) cnt[u] = 0;
}
__global__ void k_heavy_in_rows(const uint32_t* key, int64_t h, uint32_t* cnt) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < h) atomicAdd(&cnt[key[i] >> 8], 1u);
}
__global__ void k_heavy_in_pack(const uint32_t* key, const uint32_t* src, int64_t h,
                                uint32_t* hin) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < h) hin[i] = (src[i] << 8) | (key[i] & 0xffu);
}

// heavy in-edge CSR of the packed plan for its split delta: rows by target,
// every row ascending in (w, u) -- a stable sort of (v, w) keys generated in
// source order
static void build_heavy_in(gbx_graph* g, SsspPlan& P) {
  cudaStream_t s = g->stream;
  const Csr& A = g->A;
  const int64_t n = A.n;
  P.hin_rp.release();
  P.hin.release();
  if (!P.packed || n == 0 || A.nnz == 0 || A.nnz >= (int64_t(1) << 32)) return;
  Tmp<int64_t> hoff(n + 1, s);
  {
    Tmp<int64_t> hc(n + 1, s);
    k_heavy_count<<<ceil_div(n + 1, 256), 256, 0, s>>>(A.rp.p, P.nlight.p, n, hc.p);
    GBX_LAUNCHED();
    size_t tb = 0;
    GBX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, hc.p, hoff.p, n + 1, s));
    Tmp<uint8_t> t(tb, s);
    GBX_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tb, hc.p, hoff.p, n + 1, s));
  }
  int64_t h = 0;
  GBX_CUDA(cudaMemcpyAsync(&h, hoff.p + n, 8, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  P.hin_rp.alloc(n + 1);
  P.hin.alloc(std::max<int64_t>(h, 1));
  Tmp<uint32_t> cnt(n + 1, s);
  GBX_CUDA(cudaMemsetAsync(cnt.p, 0, (n + 1) * 4, s));
  if (h > 0) {
    Tmp<uint32_t> k0(h, s), k1(h, s), v0(h, s), v1(h, s);
    k_heavy_in_keys<<<ceil_div(n, 256), 256, 0, s>>>(A.rp.p, P.nlight.p, n, P.packed_edges.p,
                                                     hoff.p, k0.p, v0.p);
    GBX_LAUNCHED();
    cub::DoubleBuffer<uint32_t> kb(k0.p, k1.p), vb(v0.p, v1.p);
    radix_sort_pairs(s, kb, vb, h, 0, 32);
    k_heavy_in_rows<<<ceil_div(h, 256), 256, 0, s>>>(kb.Current(), h, cnt.p);
    GBX_LAUNCHED();
    k_heavy_in_pack<<<ceil_div(h, 256), 256, 0, s>>>(kb.Current(), vb.Current(), h, P.hin.p);
    GBX_LAUNCHED();
  }
  {
    size_t tb = 0;
    GBX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, P.hin_rp.p, n + 1, s));
    Tmp<uint8_t> t(tb, s);
    GBX_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tb, cnt.p, P.hin_rp.p, n + 1, s));
  }
  GBX_CUDA(cudaStreamSynchronize(s));
}

// (re)partition the plan's edges for delta; any row order is valid for the
// label-correcting sweep, so the packed edges are partitioned in place of the
// plan's own copy and re-partitioned when delta changes
static void ensure_split(gbx_graph* g, SsspPlan& P, double delta) {
  if (P.split_delta == delta) return;
  cudaStream_t s = g->stream;
  const Csr& A = g->A;
  const int64_t n = A.n, n1 = std::max<int64_t>(n, 1);
  P.nlight.alloc(n1);
  if (n > 0 && A.nnz > 0) {
    if (P.packed) {
      DevArray<uint32_t> out(A.nnz);
      k_split_packed<<<ceil_div(n, 256), 256, 0, s>>>(A.rp.p, n, delta, P.packed_edges.p, out.p,
                                                      P.nlight.p);
      GBX_LAUNCHED();
      GBX_CUDA(cudaStreamSynchronize(s));
      P.packed_edges = std::move(out);
    } else if (P.integral) {
      const int32_t* w = A.domain == GBX_INT32 ? reinterpret_cast<const int32_t*>(A.val.p) : P.wint.p;
      const int32_t* col = P.split_col.p ? P.split_col.p : A.col.p;
      const int32_t* ws = P.split_wi.p ? P.split_wi.p : w;
      DevArray<int32_t> oc(A.nnz), ow(A.nnz);
      k_split_cw<int32_t><<<ceil_div(n, 256), 256, 0, s>>>(A.rp.p, n, delta, col, ws, oc.p, ow.p,
                                                           P.nlight.p);
      GBX_LAUNCHED();
      GBX_CUDA(cudaStreamSynchronize(s));
      P.split_col = std::move(oc);
      P.split_wi = std::move(ow);
    } else {
      const int32_t* col = P.split_col.p ? P.split_col.p : A.col.p;
      const double* ws = P.split_wd.p ? P.split_wd.p : reinterpret_cast<const double*>(A.val.p);
      DevArray<int32_t> oc(A.nnz);
      DevArray<double> ow(A.nnz);
      k_split_cw<double><<<ceil_div(n, 256), 256, 0, s>>>(A.rp.p, n, delta, col, ws, oc.p, ow.p,
                                                          P.nlight.p);
      GBX_LAUNCHED();
      GBX_CUDA(cudaStreamSynchronize(s));
      P.split_col = std::move(oc);
      P.split_wd = std::move(ow);
    }
  } else if (n > 0) {
    GBX_CUDA(cudaMemsetAsync(P.nlight.p, 0, n * 4, s));
  }
  if (n > 0 && A.nnz < (int64_t(1) << 32)) {
    if (!P.vmeta.p) P.vmeta.alloc(n);
    k_vmeta<<<ceil_div(n, 256), 256, 0, s>>>(A.rp.p, P.nlight.p, n, P.vmeta.p);
    GBX_LAUNCHED();
  }
  GBX_CUDA(cudaStreamSynchronize(s));
  build_heavy_in(g, P);
  P.split_delta = delta;
}

// lane i's workspace (lane 0 on the graph's stream, the others on their own)
static SsspLane& ensure_lane(gbx_graph* g, SsspPlan& P, int i) {
  while (static_cast<int>(P.lanes.size()) <= i) P.lanes.emplace_back();
  if (P.lanes[i]) return *P.lanes[i];
  auto L = std::make_unique<SsspLane>();
  const int64_t n1 = std::max<int64_t>(P.n, 1);
  if (P.integral) L->dist32.alloc(n1); else L->dist64.alloc(n1);
  L->q[0].alloc(n1 + 1);
  L->q[1].alloc(n1 + 1);
  // far pile: every successful improvement above hi appends once
  const int64_t fcap = P.n + 1;  // <= one entry per vertex per bucket epoch
  L->far[0].alloc(fcap);
  L->far[1].alloc(fcap);
  L->stamp.alloc(4 * ((n1 + 31) / 32));  // 2 near + 2 far membership bitmaps
  L->ctl.alloc(10);
  L->lohi.alloc(3);
  L->relax.alloc(1);
  if (i > 0) GBX_CUDA(cudaStreamCreateWithFlags(&L->stream, cudaStreamNonBlocking));
  P.lanes[i] = std::move(L);
  return *P.lanes[i];
}

void sssp_prepare(gbx_graph* g) {
  NvtxRange nvtx_("gbx.sssp.prepare");
  if (g->sssp) return;
  const Csr& A = g->A;
  if (A.domain != GBX_FP64 && A.domain != GBX_INT32)
    fail(GBX_DOMAIN_MISMATCH, "sssp needs fp64 (or int32) edge weights");
  cudaStream_t s = g->stream;
  auto P = std::make_unique<SsspPlan>();
  P->n = A.n;
  P->nnz = A.nnz;
  DevArray<int> flags(2);
  DevArray<double> mx(1);
  GBX_CUDA(cudaMemsetAsync(flags.p, 0, 8, s));
  GBX_CUDA(cudaMemsetAsync(mx.p, 0, 8, s));
  if (A.nnz) {
    k_weight_stats<<<ceil_div(A.nnz, 256), 256, 0, s>>>(A.val.p, A.domain, A.nnz, flags.p,
                                                         flags.p + 1, mx.p);
    GBX_LAUNCHED();
  }
  int hf[2];
  GBX_CUDA(cudaMemcpyAsync(hf, flags.p, 8, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaMemcpyAsync(&P->max_w, mx.p, 8, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  P->nonpositive = hf[0] != 0;
  const bool integral = hf[1] == 0;
  // u32 distances are exact while max_w * (n-1) fits
  P->integral = integral && P->max_w * static_cast<double>(std::max<int64_t>(A.n - 1, 1)) <
                                4294967294.0;
  P->packed = P->integral && P->max_w <= 255.0 && A.n <= (int64_t(1) << 24);
  if (!P->nonpositive && A.nnz) {
    if (P->packed) {
      P->packed_edges.alloc(A.nnz);
      k_pack_edges<<<ceil_div(A.nnz, 256), 256, 0, s>>>(A.col.p, A.val.p, A.domain, A.nnz,
                                                         P->packed_edges.p, nullptr);
      GBX_LAUNCHED();
    } else if (P->integral) {
      if (A.domain == GBX_FP64) {
        P->wint.alloc(A.nnz);
        k_pack_edges<<<ceil_div(A.nnz, 256), 256, 0, s>>>(A.col.p, A.val.p, A.domain, A.nnz,
                                                           nullptr, P->wint.p);
        GBX_LAUNCHED();
      }
    }
  }
  GBX_CUDA(cudaStreamSynchronize(s));
  g->sssp = std::move(P);
  ensure_lane(g, *g->sssp, 0);
}

// one traversal on lane L (stream s) with 1/share of the resident grid;
// persist: keep the distance array in the L2 persisting window (one lane only:
// the set-aside is device-wide)
template <typename D, typename E, typename W>
static void sssp_launch(gbx_graph* g, SsspPlan& P, SsspLane& L, cudaStream_t s, int share,
                        bool persist, E edges, D* dist, int32_t src, double delta, D hi0, D inf,
                        bool split) {
  const int64_t n = P.n;
  D* lohi = reinterpret_cast<D*>(L.lohi.p);
  uint32_t* bits = reinterpret_cast<uint32_t*>(L.stamp.p);
  const int64_t words = (n + 31) / 32;
  k_sssp_init<D><<<ceil_div(std::max<int64_t>(n, 4 * words), 256), 256, 0, s>>>(dist, bits, n, src, L.q[0].p, L.ctl.p,
                                                   lohi, L.relax.p, hi0, inf);
  GBX_LAUNCHED();
  SsspArgs<D, E> a{};
  a.rp = g->A.rp.p;
  a.edges = edges;
  a.n = n;
  a.delta = delta;
  a.dist = dist;
  a.q0 = L.q[0].p;
  a.q1 = L.q[1].p;
  a.f0 = L.far[0].p;
  a.f1 = L.far[1].p;
  a.qbits[0] = bits;
  a.qbits[1] = bits + words;
  a.fbits[0] = bits + 2 * words;
  a.fbits[1] = bits + 3 * words;
  a.ctl = L.ctl.p;
  a.lohi = lohi;
  a.relax = L.relax.p;
  // keep the distance array resident in L2 while the edges stream past it
  {
    int max_persist = 0;
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, g->device);
    const size_t bytes = static_cast<size_t>(n) * sizeof(D);
    if (option(kOptSsspTrace))
      std::fprintf(stderr, "sssp: max persisting L2 %d bytes, dist %zu bytes\n", max_persist, bytes);
    if (max_persist > 0 && persist) {
      // the set-aside is a device-wide setting (and costly to change): grow only
      static size_t set_aside[64] = {0};
      const size_t want = std::min<size_t>(bytes, max_persist);
      if (g->device < 64 && set_aside[g->device] < want) {
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
        set_aside[g->device] = want;
      }
      cudaStreamAttrValue at = {};
      at.accessPolicyWindow.base_ptr = dist;
      at.accessPolicyWindow.num_bytes = std::min<size_t>(bytes, max_persist);
      at.accessPolicyWindow.hitRatio = 1.0f;
      at.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      at.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &at);
    }
    (void)cudaGetLastError();  // persistence is an optimisation: never fail on it
  }
  // circular buckets when no improvement can land more than nb-1 buckets ahead
  int nb = 1;
  const double span = 2.0 + P.max_w / delta;
  while (nb < span && nb <= 64) nb <<= 1;
  if (nb <= 64) {
    const int64_t cap = n + 1;
    if (static_cast<int>(L.bcnt.n) < nb || L.nb_alloc < nb) {
      L.bq.alloc(static_cast<size_t>(nb) * cap);
      L.bbits.alloc(static_cast<size_t>(nb) * std::max<int64_t>(words, 1));
      L.bcnt.alloc(nb);
      L.nb_alloc = nb;
    }
    GBX_CUDA(cudaMemsetAsync(L.bbits.p, 0, L.bbits.bytes(), s));
    GBX_CUDA(cudaMemsetAsync(L.bcnt.p, 0, L.bcnt.bytes(), s));
    SsspBArgs<D, E> b{};
    b.rp = a.rp;
    b.edges = edges;
    b.n = n;
    b.delta = delta;
    b.dshift = -1;
    b.idelta = 0;
    if (std::is_same<D, uint32_t>::value && delta == std::floor(delta) && delta >= 1.0 &&
        delta < 4294967296.0) {
      b.idelta = static_cast<uint32_t>(delta);
      if ((b.idelta & (b.idelta - 1)) == 0) {
        int sh = 0;
        while ((1u << sh) < b.idelta) ++sh;
        b.dshift = sh;
      }
    }
    b.nb = nb;
    b.cap = cap;
    b.dist = dist;
    b.q0 = a.q0;
    b.q1 = a.q1;
    b.bq = L.bq.p;
    b.bcnt = L.bcnt.p;
    b.qbits[0] = a.qbits[0];
    b.qbits[1] = a.qbits[1];
    b.bbits = L.bbits.p;
    b.words = words;
    b.ctl = a.ctl;
    b.relax = a.relax;
    if (split) {
      b.light_group = 2;  // 2 lanes per vertex in the light phase (1 / 4: 128 / 124 vs 121 ms)
      b.nl = P.nlight.p;
      b.vm = P.vmeta.p;
      if (P.hin.p && option(kOptSsspPullPct) > 0) {
        b.hrp = P.hin_rp.p;
        b.hin = P.hin.p;
        b.pull_pct = static_cast<int>(option(kOptSsspPullPct));
      }
    }
    if (split) {
      b.slog = L.far[0].p;  // (the far piles belong to the unbucketed kernel)
      b.slog_cap = static_cast<int>(std::min<int64_t>(kSsspSmallBucket, n));
    }
    b.trace = option(kOptSsspTrace) >= 2 ? 1 : 0;
    const bool tlog_on = option(kOptSsspTrace) != 0;
    DevArray<unsigned long long> tlog;
    if (tlog_on) {
      tlog.alloc(2 * 4096);
      GBX_CUDA(cudaMemsetAsync(tlog.p, 0, tlog.bytes(), s));
      b.tlog = tlog.p;
      b.tlog_cap = 4096;
    }
    auto fnb = k_sssp_b<D, E, W>;
    int per_sm = 0;
    GBX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fnb, kSsspThreads, 0));
    if (per_sm < 1) fail(GBX_CUDA_ERROR, "sssp kernel does not fit on an SM");
    const int grid = std::max(1, device_sms() * per_sm / share);
    void* args[] = {&b};
    GBX_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(fnb), dim3(grid),
                                         dim3(kSsspThreads), args, 0, s));
    if (tlog_on) {
      std::vector<unsigned long long> t(2 * 4096);
      GBX_CUDA(cudaMemcpyAsync(t.data(), tlog.p, t.size() * 8, cudaMemcpyDeviceToHost, s));
      GBX_CUDA(cudaStreamSynchronize(s));
      for (int i = 0; i + 1 < 4096 && t[2 * i + 2]; ++i) {
        const unsigned long long tag = t[2 * i + 1];
        const double us = (t[2 * i + 2] - t[2 * i]) / 1e3;
        if ((tag >> 62) == 2)
          std::fprintf(stderr, "sssp jump  cnt=%u %.1fus\n", static_cast<unsigned>(tag), us);
        else if ((tag >> 62) == 1)
          std::fprintf(stderr, "sssp heavy %s %.1fus\n", (tag & 1) ? "pull" : "push", us);
        else if ((tag >> 62) == 3)
          break;
        else
          std::fprintf(stderr, "sssp near k=%llu nq=%u %.1fus\n", tag >> 32,
                       static_cast<unsigned>(tag), us);
      }
    }
  } else {
    auto fn = k_sssp<D, E, W>;
    int per_sm = 0;
    GBX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kSsspThreads, 0));
    if (per_sm < 1) fail(GBX_CUDA_ERROR, "sssp kernel does not fit on an SM");
    const int grid = std::max(1, device_sms() * per_sm / share);
    void* args[] = {&a};
    GBX_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(fn), dim3(grid),
                                         dim3(kSsspThreads), args, 0, s));
  }
  cudaStreamAttrValue off = {};
  off.accessPolicyWindow.num_bytes = 0;
  cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &off);
  (void)cudaGetLastError();
}

static void sssp_checks(gbx_graph* g, double delta) {
  if (!(delta > 0.0)) fail(GBX_NON_POSITIVE_DELTA, "delta must be positive");
  sssp_prepare(g);
  SsspPlan& P = *g->sssp;
  if (P.nonpositive) fail(GBX_NON_POSITIVE_WEIGHT, "edge weights must be positive");
  int nb = 1;
  while (nb < 2.0 + P.max_w / delta && nb <= 64) nb <<= 1;
  if (nb <= 64) ensure_split(g, P, delta);  // the light-first partition for delta
}

// one source on lane L (stream s, 1/share of the SMs); out: n doubles on the
// host (NULL: the distances stay in the lane's buffer)
static void sssp_one(gbx_graph* g, SsspLane& L, cudaStream_t s, int share, bool persist,
                     int32_t src, double delta, double* out) {
  SsspPlan& P = *g->sssp;
  const int64_t n = P.n;
  // the circular-bucket kernel (nb <= 64) runs proper Delta-stepping on a
  // light-first row partition
  int nb = 1;
  while (nb < 2.0 + P.max_w / delta && nb <= 64) nb <<= 1;
  const bool split = nb <= 64;
  const bool cw = split && !P.packed;  // partitioned copies of col + weights
  if (P.integral) {
    // integer distances: bucket [lo, lo+delta) -> integer hi = ceil(lo + delta)
    const double h0 = std::ceil(delta);
    const uint32_t hi0 = h0 >= 4294967295.0 ? 0xffffffffu : static_cast<uint32_t>(h0);
    if (P.packed) {
      sssp_launch<uint32_t, PackedEdges, uint32_t>(g, P, L, s, share, persist,
                                                   PackedEdges{P.packed_edges.p}, L.dist32.p, src,
                                                   delta, hi0, 0xffffffffu, split);
    } else {
      const int32_t* w = g->A.domain == GBX_INT32 ? reinterpret_cast<const int32_t*>(g->A.val.p)
                                                  : P.wint.p;
      sssp_launch<uint32_t, IntEdges, uint32_t>(
          g, P, L, s, share, persist,
          IntEdges{cw ? P.split_col.p : g->A.col.p, cw ? P.split_wi.p : w}, L.dist32.p, src, delta,
          hi0, 0xffffffffu, split);
    }
  } else {
    unsigned long long hi0, inf = 0x7FF0000000000000ull;
    std::memcpy(&hi0, &delta, 8);
    sssp_launch<unsigned long long, DblEdges, double>(
        g, P, L, s, share, persist,
        DblEdges{cw ? P.split_col.p : g->A.col.p,
                 cw ? P.split_wd.p : reinterpret_cast<const double*>(g->A.val.p)},
        L.dist64.p, src, delta, hi0, inf, split);
  }
  if (out) {
    L.out.ensure(std::max<int64_t>(n, 1));
    if (P.integral) k_sssp_out<uint32_t><<<ceil_div(n, 256), 256, 0, s>>>(L.dist32.p, n, L.out.p);
    else k_sssp_out<unsigned long long><<<ceil_div(n, 256), 256, 0, s>>>(L.dist64.p, n, L.out.p);
    GBX_LAUNCHED();
    GBX_CUDA(cudaMemcpyAsync(out, L.out.p, n * 8, cudaMemcpyDeviceToHost, s));
  }
}

void sssp_run(gbx_graph* g, uint64_t source, double delta, double* out) {
  NvtxRange nvtx_("gbx.sssp");
  const int64_t n = g->A.n;
  if (source >= static_cast<uint64_t>(n))
    fail(GBX_SOURCE_OUT_OF_RANGE, "source " + std::to_string(source));
  sssp_checks(g, delta);
  SsspPlan& P = *g->sssp;
  SsspLane& L = ensure_lane(g, P, 0);
  cudaStream_t s = g->stream;
  sssp_one(g, L, s, 1, true, static_cast<int32_t>(source), delta, out);
  int hctl[10];
  unsigned long long rel = 0;
  GBX_CUDA(cudaMemcpyAsync(hctl, L.ctl.p, sizeof hctl, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaMemcpyAsync(&rel, L.relax.p, 8, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  g->stats = gbx_stats{};
  g->pending_iters = nullptr;
  g->stats.launches = 2 + (out ? 1 : 0);
  g->stats.hot_launches = 1;
  g->stats.iterations = hctl[4];
  g->stats.work_units = static_cast<int64_t>(rel);
}

// sssp_default_delta (sssp.cpp:114-120): half the largest weight, or 1.
double sssp_default_delta(gbx_graph* g) {
  if (g->A.nnz == 0 || (g->A.domain != GBX_FP64 && g->A.domain != GBX_INT32)) return 1.0;
  sssp_prepare(g);
  const double m = g->sssp->max_w;
  return m > 0 ? m / 2.0 : 1.0;
}

// Several sources of sssp_delta_stepping (gapbench's per-source trials,
// gapbench.cpp:300-330) in one call: the traversals are queued back to back
// on the graph's stream (lane 0's workspace; each kernel reads its own
// counters from the device), with ONE host synchronisation at the end instead
// of one per source.  out: ns * n doubles (row b = sources[b]) or NULL.
// (A vertex-major sweep of up to 16 sources sharing every edge read was
// measured and rejected: its 16 distance rows per vertex (1 GB at
// 2^24) no longer fit the 126 MB L2 the one-source kernel's 64 MB distance
// array lives in -- 224 vs 83 ms for config 4.)
void sssp_batch_run(gbx_graph* g, const uint64_t* sources, uint64_t ns, double delta,
                    double* out) {
  NvtxRange nvtx_("gbx.sssp.batch");
  const int64_t n = g->A.n;
  if (ns == 0) fail(GBX_EMPTY_BATCH, "empty source batch");
  if (!sources) fail(GBX_NULL_ARGUMENT, "sources is NULL");
  for (uint64_t b = 0; b < ns; ++b)
    if (sources[b] >= static_cast<uint64_t>(n))
      fail(GBX_SOURCE_OUT_OF_RANGE, "source " + std::to_string(sources[b]));
  sssp_checks(g, delta);
  SsspPlan& P = *g->sssp;
  SsspLane& L = ensure_lane(g, P, 0);
  cudaStream_t s = g->stream;
  DevArray<double> dev_out;
  if (out) dev_out.alloc(std::max<int64_t>(static_cast<int64_t>(ns) * n, 1));
  DevArray<unsigned long long> rel(ns);
  for (uint64_t b = 0; b < ns; ++b) {
    sssp_one(g, L, s, 1, true, static_cast<int32_t>(sources[b]), delta, nullptr);
    GBX_CUDA(cudaMemcpyAsync(rel.p + b, L.relax.p, 8, cudaMemcpyDeviceToDevice, s));
    if (out) {
      if (P.integral) k_sssp_out<uint32_t><<<ceil_div(n, 256), 256, 0, s>>>(L.dist32.p, n, dev_out.p + b * n);
      else k_sssp_out<unsigned long long><<<ceil_div(n, 256), 256, 0, s>>>(L.dist64.p, n, dev_out.p + b * n);
      GBX_LAUNCHED();
    }
  }
  std::vector<unsigned long long> hr(ns);
  GBX_CUDA(cudaMemcpyAsync(hr.data(), rel.p, ns * 8, cudaMemcpyDeviceToHost, s));
  if (out) GBX_CUDA(cudaMemcpyAsync(out, dev_out.p, ns * n * 8, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  unsigned long long total = 0;
  for (unsigned long long r : hr) total += r;
  g->stats = gbx_stats{};
  g->pending_iters = nullptr;
  g->stats.launches = static_cast<int64_t>(ns) * (2 + (out ? 1 : 0));
  g->stats.hot_launches = static_cast<int64_t>(ns);
  g->stats.work_units = static_cast<int64_t>(total);
}

}  // namespace gbx
