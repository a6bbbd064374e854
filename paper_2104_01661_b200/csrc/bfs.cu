// bfs.cu -- direction-optimizing BFS (algo/bfs.cpp:18-85) and a 64-lane
// multi-source BFS, each as ONE persistent cooperative kernel: the level loop,
// the push/pull decision and the frontier swap all run on the device with
// grid-wide barriers, so a whole traversal costs one launch (scale-16 BFS is
// latency-bound: SURVEY.md §7 hard part 7).
//
// Parent semantics: the reference's any.secondi keeps the first contribution in
// ascending frontier order (core.cpp:214-222, ops.cpp:170-175), i.e. the
// minimum-id neighbour on the previous level.  Push reproduces it with
// atomicMin over every frontier edge into an unvisited vertex; pull scans the
// ascending AT row and keeps the first frontier hit.  Both are bit-exact.
//
// Frontier: queue of (vertex, chunk) entries (push: one warp per <= kChunk
// edges, so hubs are split) plus a bitmap (pull: 1 bit per vertex, L2/L1
// resident).  Compaction into the next queue is warp-aggregated (one atomic
// per warp).  Direction rule = the reference's (bfs.cpp:77-78): push iff the
// frontier has < n/push_divisor + 1 vertices and is growing.
#include <cooperative_groups.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "common.cuh"
#include "plans.cuh"
#include "warpqueue.cuh"

namespace cg = cooperative_groups;

namespace gbx {

constexpr int kBfsThreads = 256;
constexpr int kBfsBuf = 256;  // staged frontier vertices per warp
#ifndef GBX_BFS_CHUNK
#define GBX_BFS_CHUNK 256
#endif
constexpr int64_t kChunk = GBX_BFS_CHUNK;  // push: edges per warp entry (latency-bound steps)
constexpr unsigned kFull = 0xffffffffu;
// In-degree above which a pull row goes to a whole warp instead of 8 lanes.
// The 64-lane batch has to find a parent for every lane, so its hubs are
// scanned far (256); a single-source pull stops at the first frontier hit,
// which a hub meets within its first in-edges: a separate pass over them only
// costs (scale 22, 8 sources: 256 / 512 / 1024 / 2048 / 4096 / 8192 / none ->
// 2.16 / 1.91 / 1.86 / 1.85 / 1.83 / 1.83 / 1.82 ms; 8192 keeps a bound on what
// one lane group may have to walk).
#ifndef GBX_BFS_HEAVY
#define GBX_BFS_HEAVY 256
#endif
#ifndef GBX_BFS1_HEAVY
#define GBX_BFS1_HEAVY 8192
#endif
constexpr int64_t kBfsHeavy = GBX_BFS_HEAVY;
constexpr int64_t kBfs1Heavy = GBX_BFS1_HEAVY;
// Pull: 4-edge rounds a lane scans its own row before handing it to a group.
#ifndef GBX_BFS_ROUNDS
#define GBX_BFS_ROUNDS 2
#endif
constexpr int kThreadRounds = GBX_BFS_ROUNDS;

__device__ __forceinline__ int n_chunks(int64_t deg) {
  return deg <= kChunk ? 1 : static_cast<int>((deg + kChunk - 1) / kChunk);
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------------------
// single source
// ---------------------------------------------------------------------------
struct Bfs1Args {
  const int64_t* rp;
  const int32_t* col;
  const int64_t* trp;
  const int32_t* tcol;
  int64_t n, nnz;
  int mode;
  int64_t divisor;
  int alpha;         // AUTO also pulls once frontier edges * alpha >= nnz (0: off)
  int32_t* level;
  int32_t* parent;
  int64_t* q0;
  int64_t* q1;
  uint32_t* bm0;
  uint32_t* bm1;
  uint32_t* bm2;
  int32_t* ul0;      // still-unvisited vertices (pull levels only scan these)
  int32_t* ul1;
  const int32_t* heavy;  // in-degree > kBfsHeavy: pulled by whole warps, never listed
  int64_t nheavy;
  const int32_t* unz;    // vertices with in-edges, ascending: what the FIRST pull scans
  int64_t nunz;          // (vertices without in-edges can never be pulled)
  int* ctl;  // [5] levels done [6] push levels; slot j = ctl + 16 + 8 * (j & 3) describes
             // the frontier level j produced: [0] queue entries [1] vertices [2:4) u64
             // frontier edges [4] unvisited-list size (-1: not built) [5] list parity
  unsigned long long* tlog;  // optional: %globaltimer at phase boundaries (debug)
  int32_t source;
};

__global__ void __launch_bounds__(kBfsThreads) k_bfs1(Bfs1Args a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ int32_t s_buf[kBfsThreads / 32][kBfsBuf];
  __shared__ int32_t s_ubuf[kBfsThreads / 32][kBfsBuf];
  __shared__ int32_t s_kbuf[kBfsThreads / 32][kBfsBuf];
  __shared__ __align__(8) int s_red[6];
  FrontierQueue<kBfsBuf> fq;
  fq.buf = s_buf[threadIdx.x >> 5];
  fq.rp = a.rp;
  fq.chunk = kChunk;
  WarpQueue<int32_t, kBfsBuf> uq;
  uq.buf = s_ubuf[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t gtid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t gsize = int64_t(gridDim.x) * blockDim.x;
  const int64_t nwords = (a.n + 31) >> 5;
  // one grid barrier per level: the per-level counters live in a ring of 4
  // slots (level d reads slot d-1 and d-2, accumulates slot d and zeroes slot
  // d+1, last read at the start of level d-2) and the frontier bitmaps in a
  // ring of 3 (level d reads bm[d-1], writes bm[d], clears bm[d+1], which level
  // d-1 read) -- nothing a level touches is still in use by the previous one
  auto slot = [&](int j) { return a.ctl + 16 + 8 * (j & 3); };
  uint32_t* bms[3] = {a.bm0, a.bm1, a.bm2};
  if (a.tlog && gtid == 0) a.tlog[0] = gtimer();
  {
    // initial state, inside the persistent kernel (no init / seed launches):
    // every vertex unreached except the source, empty bitmaps but the
    // source's bit, and the source's level-1 queue entries (bfs.cpp:18-55)
    const int32_t src = a.source;
    for (int64_t i = gtid; i < a.n || i < nwords; i += gsize) {
      if (i < a.n) {
        a.level[i] = i == src ? 0 : -1;
        a.parent[i] = i == src ? src : INT_MAX;
      }
      if (i < nwords) {
        a.bm0[i] = i == (src >> 5) ? 1u << (src & 31) : 0u;
        a.bm1[i] = 0u;
      }
    }
    if (gtid == 0) {
      const int64_t deg = a.rp[src + 1] - a.rp[src];
      const int k = n_chunks(deg);
      for (int c = 0; c < k; ++c) a.q0[c] = (static_cast<int64_t>(c) << 32) | src;
      for (int i = 0; i < 48; ++i) a.ctl[i] = 0;
      int* s0 = slot(0);
      s0[0] = k;
      s0[1] = 1;
      *reinterpret_cast<unsigned long long*>(s0 + 2) = static_cast<unsigned long long>(deg);
      s0[4] = -1;
      s0[5] = 0;
    }
    grid.sync();
  }
  for (int d = 1; static_cast<int64_t>(d) + 1 <= a.n; ++d) {
    const int* sc = slot(d - 1);
    int* sn = slot(d);
    const int qe = *(volatile const int*)&sc[0];
    const int qv = *(volatile const int*)&sc[1];
    const int pv = d >= 2 ? *(volatile const int*)&slot(d - 2)[1] : 0;
    const unsigned long long fe = *(volatile const unsigned long long*)(sc + 2);
    if (qv == 0) break;
    // alpha == 0: the reference's rule (bfs.cpp:77-78), push while the frontier
    // has < n/divisor + 1 vertices and grows.  alpha > 0 (default): Beamer's
    // edge test replaces "grows" -- push while the frontier's edges are under
    // nnz/alpha, so a 1-vertex or shrinking frontier is pushed instead of paying
    // a scan of every unvisited row.  Results are identical either way (min-id
    // parents in both directions); only the work differs.
    const bool small = qv < a.n / a.divisor + 1;
    const bool push =
        a.mode == GBX_BFS_PUSH ||
        (a.mode == GBX_BFS_AUTO &&
         (a.alpha == 0 ? (small && qv > pv)
                       : (small && fe * static_cast<unsigned long long>(a.alpha) <
                                       static_cast<unsigned long long>(a.nnz))));
    if (a.tlog && gtid == 0) {
      a.tlog[4 * d] = gtimer();
      a.tlog[4 * d + 3] = (push ? 1ull : 0ull) | (static_cast<unsigned long long>(qv) << 8);
    }
    const int p = (d - 1) & 1;
    const int64_t* qc = p ? a.q1 : a.q0;
    int64_t* qn = p ? a.q0 : a.q1;
    const uint32_t* bc = bms[(d - 1) % 3];
    uint32_t* bn = bms[d % 3];
    {
      // the bitmap level d+1 writes (level d-1 read it) and slot d+1
      uint32_t* bclr = bms[(d + 1) % 3];
      for (int64_t i = gtid; i < nwords; i += gsize) bclr[i] = 0u;
      if (gtid == 0) {
        int* sz = slot(d + 1);
        for (int i = 0; i < 8; ++i) sz[i] = 0;
      }
    }
    const int ucnt = *(volatile const int*)&sc[4];
    const int upar = *(volatile const int*)&sc[5];
    if (gtid == 0) {
      // the unvisited list this level leaves behind: a pull builds the other
      // buffer (its size accumulates in sn[4], zeroed two levels ago), a push
      // keeps the current one
      if (push) sn[4] = ucnt;
      sn[5] = push ? upar : (upar ^ 1);
    }
    unsigned long long* edges_n = reinterpret_cast<unsigned long long*>(sn + 2);
    fq.reset(qn, &sn[0], &sn[1], edges_n, nullptr);
    if (push) {
      // a small queue (a hub or two) would leave most warps idle and walk each
      // kChunk-edge entry in kChunk/32 dependent steps: split every entry over
      // S warps (S = power of two up to 8, uniform over the grid)
      int S = 1;
      while (S < 8 && static_cast<int64_t>(qe) * S * 2 <= nwarps) S <<= 1;
      const int64_t sub = kChunk / S;
      // many entries with few edges each (the traversal's late levels: ~5 edges
      // per frontier vertex): four entries per warp step, 8 lanes each -- a warp
      // per entry leaves most lanes idle and walks the entries one dependent
      // chain after the other
      const bool grouped = S == 1 && fe < 16ull * static_cast<unsigned long long>(qe);
      if (grouped) {
        const int grp = lane >> 3, sl = lane & 7;
        for (int64_t e4 = gwarp * 4; e4 < qe; e4 += nwarps * 4) {
          const int64_t e = e4 + grp;
          int32_t v = 0;
          int64_t q = 0, e0 = 0;
          if (e < qe) {
            const int64_t ent = qc[e];
            v = static_cast<int32_t>(ent & 0xffffffff);
            const int64_t c = ent >> 32;
            const int64_t cb = a.rp[v] + c * kChunk;
            e0 = min(a.rp[v + 1], cb + kChunk);
            q = cb + sl;
          }
          bool active = q < e0;
          while (__any_sync(kFull, active)) {
            bool has = false;
            int32_t w = 0;
            if (active) {
              w = __ldg(a.col + q);
              GBX_DCHECK(w >= 0 && w < a.n, "bfs push column", w);
              const int lw = *(volatile int32_t*)&a.level[w];
              const int32_t pw = *(volatile int32_t*)&a.parent[w];
              if ((lw == -1 || lw == d) && v < pw) {
                atomicMin(&a.parent[w], v);
                if (lw == -1 && atomicCAS(&a.level[w], -1, d) == -1) {
                  has = true;
                  atomicOr(&bn[w >> 5], 1u << (w & 31));
                }
              }
              q += 8;
              if (q >= e0) active = false;
            }
            fq.push(has, w);
          }
        }
      } else
      for (int64_t e2 = gwarp; e2 < static_cast<int64_t>(qe) * S; e2 += nwarps) {
        const int64_t e = e2 / S;
        const int part = static_cast<int>(e2 - e * S);
        const int64_t ent = qc[e];
        const int32_t v = static_cast<int32_t>(ent & 0xffffffff);
        const int64_t c = ent >> 32;
        const int64_t cb = a.rp[v] + c * kChunk;
        const int64_t ce = min(a.rp[v + 1], cb + kChunk);
        const int64_t b0 = cb + part * sub;
        const int64_t e0 = min(ce, b0 + sub);
        for (int64_t base = b0; base < e0; base += 32) {
          const int64_t q = base + lane;
          bool has = false;
          int32_t w = 0;
          if (q < e0) {
            w = __ldg(a.col + q);
            GBX_DCHECK(w >= 0 && w < a.n, "bfs push column", w);
            // level and parent loads issued together; min-id parent: skip the
            // atomic when a smaller one already landed
            const int lw = *(volatile int32_t*)&a.level[w];
            const int32_t pw = *(volatile int32_t*)&a.parent[w];
            if ((lw == -1 || lw == d) && v < pw) {
              atomicMin(&a.parent[w], v);
              if (lw == -1 && atomicCAS(&a.level[w], -1, d) == -1) {
                has = true;
                atomicOr(&bn[w >> 5], 1u << (w & 31));
              }
            }
          }
          fq.push(has, w);
        }
      }
    } else {
      // scan every vertex the first time, afterwards only the ones a previous
      // pull left unvisited (vertices with no in-edges never enter the list)
      // the first pull scans the (per-graph) list of vertices WITH in-edges --
      // on an R-MAT graph 45% of the vertices have none and would cost a step
      // slot, a level word and two row pointers each in a latency-bound level
      const int32_t* ucur = ucnt < 0 ? a.unz : (upar ? a.ul1 : a.ul0);
      uq.reset(upar ? a.ul0 : a.ul1, &sn[4]);
      const int64_t range = ucnt < 0 ? a.nunz : ucnt;
      const int grp = lane >> 3, sub = lane & 7;
      // 32 vertices per warp step, one per lane: the level/row-pointer loads
      // coalesce and every lane scans its own row 4 edges per round (the 4
      // neighbour and 4 bitmap loads are independent); rows still unresolved
      // after kThreadRounds rounds go to 8-lane groups, 4 rows at a time.
      // (the next step's list entry is loaded a step ahead: one register, one
      //  round trip less per step)
      int32_t wnext = gwarp * 32 + lane < range ? ucur[gwarp * 32 + lane] : -1;
      for (int64_t vb = gwarp * 32; vb < range; vb += nwarps * 32) {
        const int64_t w = wnext >= 0 ? wnext : a.n;
        {
          const int64_t i = vb + nwarps * 32 + lane;
          wnext = i < range ? ucur[i] : -1;
        }
        // the row pointers are loaded together with the level (not behind its
        // test): one round trip less per 32-vertex step of a latency-bound level
        // (26 steps per warp at scale 22, each a chain vertex -> level / row
        // pointers -> neighbours -> bitmap words): 2.44 -> 2.38 ms per 8 sources.
        // Loading the NEXT step's vertex, level and row pointers one step ahead
        // as well costs 16 registers (3 CTAs per SM instead of 4): 2.47 ms.
        const bool inr = w < a.n;
        const int32_t lw0 = inr ? a.level[w] : 0;
        int64_t pp = inr ? a.trp[w] : 0, pe = inr ? a.trp[w + 1] : 0;
        bool active = inr && lw0 == -1;
        if (!active) pp = pe = 0;
        if (pe - pp > kBfs1Heavy) active = false;  // hub: the warp pass below
        const bool cand = active && pe > pp;
        active = cand;
        int32_t found = -1;
#pragma unroll 1
        for (int r = 0; r < kThreadRounds && __any_sync(kFull, active); ++r) {
          if (active) {
            int32_t u[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              u[k] = pp + k < pe ? __ldg(a.tcol + pp + k) : -1;
              GBX_DCHECK(u[k] < a.n, "bfs pull column", u[k]);
            }
            unsigned hits = 0u;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (u[k] >= 0 && ((ld_weak(bc + (u[k] >> 5)) >> (u[k] & 31)) & 1u)) hits |= 1u << k;
            if (hits) {
              const int k = __ffs(hits) - 1;
              found = k == 0 ? u[0] : k == 1 ? u[1] : k == 2 ? u[2] : u[3];
              active = false;
            } else {
              pp += 4;
              if (pp >= pe) active = false;
            }
          }
        }
        bool has = found >= 0;
        if (has) {
          a.level[w] = d;
          a.parent[w] = found;
          atomicOr(&bn[w >> 5], 1u << (w & 31));
        }
        fq.push(has, static_cast<int32_t>(w));
        uq.push(cand && !active && found < 0, static_cast<int32_t>(w));
        // long rows: 8-lane groups, 4 rows at a time, continuing at pp
        unsigned rest = __ballot_sync(kFull, active);
        while (rest) {
          int src = -1;
          unsigned m = rest;
          for (int k = 0; k < grp && m; ++k) m &= m - 1;
          if (m) src = __ffs(m) - 1;
          for (int k = 0; k < 4 && rest; ++k) rest &= rest - 1;
          const int64_t gw = __shfl_sync(kFull, w, src < 0 ? 0 : src);
          int64_t gp = __shfl_sync(kFull, pp, src < 0 ? 0 : src);
          const int64_t ge = __shfl_sync(kFull, pe, src < 0 ? 0 : src);
          bool gact = src >= 0;
          int32_t gfound = -1;
          while (__any_sync(kFull, gact)) {
            int32_t u = -1;
            bool hit = false;
            if (gact && gp + sub < ge) {
              u = __ldg(a.tcol + gp + sub);
              GBX_DCHECK(u >= 0 && u < a.n, "bfs pull column", u);
              hit = (ld_weak(bc + (u >> 5)) >> (u & 31)) & 1u;
            }
            const unsigned bal = __ballot_sync(kFull, hit);
            const unsigned gb = (bal >> (grp * 8)) & 0xffu;
            const int sl = grp * 8 + (gb ? __ffs(gb) - 1 : 0);
            const int32_t uu = __shfl_sync(kFull, u, sl);
            if (gact) {
              if (gb) { gfound = uu; gact = false; }
              else { gp += 8; if (gp >= ge) gact = false; }
            }
          }
          const bool ghas = sub == 0 && gfound >= 0;
          if (ghas) {
            a.level[gw] = d;
            a.parent[gw] = gfound;
            atomicOr(&bn[gw >> 5], 1u << (gw & 31));
          }
          fq.push(ghas, static_cast<int32_t>(gw));
          uq.push(sub == 0 && src >= 0 && gfound < 0, static_cast<int32_t>(gw));
        }
      }
      uq.flush();
      for (int64_t h = gwarp; h < a.nheavy; h += nwarps) {
        const int32_t w = a.heavy[h];
        if (a.level[w] != -1) continue;
        const int64_t pe = a.trp[w + 1];
        int32_t found = -1;
        for (int64_t pp = a.trp[w]; pp < pe; pp += 32) {
          int32_t u = -1;
          bool hit = false;
          if (pp + lane < pe) {
            u = __ldg(a.tcol + pp + lane);
            GBX_DCHECK(u >= 0 && u < a.n, "bfs pull column", u);
            hit = (ld_weak(bc + (u >> 5)) >> (u & 31)) & 1u;
          }
          const unsigned bal = __ballot_sync(kFull, hit);
          if (bal) {
            found = __shfl_sync(kFull, u, __ffs(bal) - 1);
            break;
          }
        }
        const bool has = lane == 0 && found >= 0;
        if (has) {
          a.level[w] = d;
          a.parent[w] = found;
          atomicOr(&bn[w >> 5], 1u << (w & 31));
        }
        fq.push(has, w);
      }
    }
    fq.flush_block(s_kbuf[threadIdx.x >> 5], s_red);
    if (a.tlog && gtid == 0) a.tlog[4 * d + 1] = gtimer();
    if (gtid == 0) {
      a.ctl[5] = d;
      if (push) a.ctl[6] += 1;
    }
    grid.sync();
    if (a.tlog && gtid == 0) a.tlog[4 * d + 2] = gtimer();
  }
  if (a.tlog && gtid == 0) a.tlog[1] = gtimer();
}

__global__ void k_i32_to_i64(const int32_t* in, int64_t* out, int64_t n, int32_t none) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = in[i] == none ? -1 : in[i];
}

// per-level trace written by the kernels when GBX_BFS_TLOG is set
static void dump_tlog(BfsWork& W, const char* tag) {
  std::vector<unsigned long long> t(4 * 256);
  GBX_CUDA(cudaMemcpy(t.data(), W.tlog.p, t.size() * 8, cudaMemcpyDeviceToHost));
  if (t[0] && t[1]) std::fprintf(stderr, "%s kernel %.1fus\n", tag, (t[1] - t[0]) / 1e3);
  if (t[0] && t[4]) std::fprintf(stderr, "%s initial state %.1fus\n", tag, (t[4] - t[0]) / 1e3);
  for (int d = 1; d < 256 && t[4 * d]; ++d)
    std::fprintf(stderr, "%s level %d %s qv=%llu work=%.1fus finalize=%.1fus\n", tag, d,
                 (t[4 * d + 3] & 1) ? "push" : "pull", t[4 * d + 3] >> 8,
                 (t[4 * d + 1] - t[4 * d]) / 1e3, (t[4 * d + 2] - t[4 * d + 1]) / 1e3);
}

static int coop_grid(const void* fn, int threads) {
  int per_sm = 0;
  GBX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0));
  if (per_sm < 1) fail(GBX_CUDA_ERROR, "cooperative kernel does not fit on an SM");
  return device_sms() * per_sm;
}

struct HasInEdges {
  const int64_t* trp;
  __device__ __forceinline__ bool operator()(int32_t v) const { return trp[v + 1] > trp[v]; }
};

__global__ void k_bfs_heavy(const int64_t* trp, int64_t n, int64_t thr, int32_t* out, int* cnt) {
  int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (v < n && trp[v + 1] - trp[v] > thr) out[atomicAdd(cnt, 1)] = static_cast<int32_t>(v);
}

// hub list for the pull passes, rebuilt when the transpose changes
static void ensure_heavy(gbx_graph* g, const Csr& AT) {
  BfsWork& W = *g->bfs;
  if (W.heavy_key == AT.rp.p && W.heavy_nnz == AT.nnz && W.heavy.p) return;
  const int64_t n = AT.n;
  cudaStream_t s = g->stream;
  if (!W.heavy_cnt.p) W.heavy_cnt.alloc(1);
  // two hub lists: the 64-lane batch's (kBfsHeavy) and the single source's (kBfs1Heavy)
  for (int which = 0; which < 2; ++which) {
    DevArray<int32_t>& list = which ? W.heavy1 : W.heavy;
    list.alloc(std::max<int64_t>(n, 1));
    GBX_CUDA(cudaMemsetAsync(W.heavy_cnt.p, 0, sizeof(int), s));
    k_bfs_heavy<<<ceil_div(std::max<int64_t>(n, 1), 256), 256, 0, s>>>(
        AT.rp.p, n, which ? kBfs1Heavy : kBfsHeavy, list.p, W.heavy_cnt.p);
    GBX_LAUNCHED();
    int c = 0;
    GBX_CUDA(cudaMemcpyAsync(&c, W.heavy_cnt.p, sizeof c, cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaStreamSynchronize(s));
    (which ? W.nheavy1 : W.nheavy) = c;
  }
  // vertices with in-edges, ascending (the first pull's work list)
  W.unz.alloc(std::max<int64_t>(n, 1));
  {
    Tmp<int64_t> nsel(1, s);
    size_t tb = 0;
    HasInEdges pred{AT.rp.p};
    thrust::counting_iterator<int32_t> ids(0);
    GBX_CUDA(cub::DeviceSelect::If(nullptr, tb, ids, W.unz.p, nsel.p, static_cast<int>(n), pred, s));
    Tmp<uint8_t> t(tb, s);
    GBX_CUDA(cub::DeviceSelect::If(t.p, tb, ids, W.unz.p, nsel.p, static_cast<int>(n), pred, s));
    int64_t h = 0;
    GBX_CUDA(cudaMemcpyAsync(&h, nsel.p, sizeof h, cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaStreamSynchronize(s));
    W.nunz = h;
  }
  W.heavy_key = AT.rp.p;
  W.heavy_nnz = AT.nnz;
}

static void ensure_bfs1(gbx_graph* g) {
  if (!g->bfs) g->bfs = std::make_unique<BfsWork>();
  BfsWork& W = *g->bfs;
  const int64_t n = g->A.n;
  if (W.n == n && W.level.p) return;
  W.n = n;
  W.level.alloc(std::max<int64_t>(n, 1));
  W.parent.alloc(std::max<int64_t>(n, 1));
  const int64_t qcap = n + g->A.nnz / kChunk + 64;
  W.queue[0].alloc(2 * qcap);  // int64 entries stored in int32 pairs
  W.queue[1].alloc(2 * qcap);
  W.bitmap[0].alloc((n + 31) / 32 + 1);
  W.bitmap[1].alloc((n + 31) / 32 + 1);
  W.bitmap[2].alloc((n + 31) / 32 + 1);
  W.ulist[0].alloc(std::max<int64_t>(n, 1));
  W.ulist[1].alloc(std::max<int64_t>(n, 1));
  W.ctl.alloc(64);
}

void bfs_prepare(gbx_graph* g) { ensure_bfs1(g); }

static void copy_out_i64(cudaStream_t s, const int32_t* dev, int64_t n, int32_t none,
                         int64_t* host) {
  int64_t* tmp = nullptr;
  GBX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tmp), std::max<int64_t>(n, 1) * 8, s));
  k_i32_to_i64<<<ceil_div(std::max<int64_t>(n, 1), 256), 256, 0, s>>>(dev, tmp, n, none);
  cudaError_t le = cudaGetLastError();
  if (le == cudaSuccess)
    le = cudaMemcpyAsync(host, tmp, n * sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(tmp, s);
  GBX_CUDA(le);
}

void bfs_run(gbx_graph* g, uint64_t source, int direction, uint64_t push_divisor,
             bool use_at, int64_t* parent, int64_t* level) {
  NvtxRange nvtx_("gbx.bfs");
  const int64_t n = g->A.n;
  if (source >= static_cast<uint64_t>(n))
    fail(GBX_SOURCE_OUT_OF_RANGE, "source " + std::to_string(source) + " with n = " +
                                      std::to_string(n));
  if (direction != GBX_BFS_AUTO && direction != GBX_BFS_PUSH && direction != GBX_BFS_PULL)
    fail(GBX_INVALID_VALUE, "bfs: unknown direction");
  ensure_bfs1(g);
  BfsWork& W = *g->bfs;
  cudaStream_t s = g->stream;
  const Csr& A = g->A;
  const Csr* AT = use_at ? &g->AT() : nullptr;
  if (AT) ensure_heavy(g, *AT);
  const bool tlog_on = option(kOptBfsTrace) != 0;
  cudaEvent_t ev[4];
  if (tlog_on) {
    for (auto& e : ev) GBX_CUDA(cudaEventCreate(&e));
    GBX_CUDA(cudaEventRecord(ev[0], s));
  }
  int64_t* q0 = reinterpret_cast<int64_t*>(W.queue[0].p);
  int64_t* q1 = reinterpret_cast<int64_t*>(W.queue[1].p);
  Bfs1Args a{};
  a.source = static_cast<int32_t>(source);
  a.rp = A.rp.p;
  a.col = A.col.p;
  a.trp = AT ? AT->rp.p : nullptr;
  a.tcol = AT ? AT->col.p : nullptr;
  a.n = n;
  a.nnz = A.nnz;
  a.mode = use_at ? direction : GBX_BFS_PUSH;
  const int alpha = static_cast<int>(option(kOptBfsAlpha));
  a.alpha = alpha;
  a.ul0 = W.ulist[0].p;
  a.ul1 = W.ulist[1].p;
  a.heavy = W.heavy1.p;
  a.nheavy = W.nheavy1;
  a.unz = AT ? W.unz.p : nullptr;
  a.nunz = AT ? W.nunz : 0;
  a.divisor = push_divisor == 0 ? 1 : static_cast<int64_t>(push_divisor);
  a.level = W.level.p;
  a.parent = W.parent.p;
  a.q0 = q0;
  a.q1 = q1;
  a.bm0 = W.bitmap[0].p;
  a.bm1 = W.bitmap[1].p;
  a.bm2 = W.bitmap[2].p;
  a.ctl = W.ctl.p;
  if (tlog_on) {
    if (!W.tlog.p) W.tlog.alloc(4 * 256);
    GBX_CUDA(cudaMemsetAsync(W.tlog.p, 0, W.tlog.bytes(), s));
    a.tlog = W.tlog.p;
    GBX_CUDA(cudaEventRecord(ev[1], s));
  }
  static int grid = 0;
  if (!grid) grid = coop_grid(reinterpret_cast<const void*>(k_bfs1), kBfsThreads);
  void* args[] = {&a};
  GBX_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_bfs1), dim3(grid),
                                       dim3(kBfsThreads), args, 0, s));
  if (tlog_on) GBX_CUDA(cudaEventRecord(ev[2], s));
  g->stats = gbx_stats{};
  g->pending_iters = nullptr;
  g->stats.launches = 1 + (parent ? 1 : 0) + (level ? 1 : 0);
  g->stats.hot_launches = 1;
  if (!parent && !level && !tlog_on) {
    // device-resident result (gbx_result_device): the call stays asynchronous
    // (gbx.h: synchronous unless every output pointer is NULL), so back-to-back
    // traversals queue on the stream without a host round trip between them
    g->pending_iters = W.ctl.p + 5;  // read by gbx_last_stats after a stream sync
    return;
  }
  if (parent) copy_out_i64(s, W.parent.p, n, INT_MAX, parent);
  if (level) copy_out_i64(s, W.level.p, n, -1, level);
  int hctl[8] = {0};
  GBX_CUDA(cudaMemcpyAsync(hctl, W.ctl.p, sizeof hctl, cudaMemcpyDeviceToHost, s));
  if (tlog_on) GBX_CUDA(cudaEventRecord(ev[3], s));
  GBX_CUDA(cudaStreamSynchronize(s));
  if (tlog_on) {
    float t01, t12, t23;
    cudaEventElapsedTime(&t01, ev[0], ev[1]);
    cudaEventElapsedTime(&t12, ev[1], ev[2]);
    cudaEventElapsedTime(&t23, ev[2], ev[3]);
    std::fprintf(stderr, "bfs1 events: setup %.1fus kernel %.1fus out %.1fus\n", t01 * 1e3,
                 t12 * 1e3, t23 * 1e3);
    for (auto& e : ev) cudaEventDestroy(e);
  }
  g->stats.iterations = hctl[5];
  if (tlog_on) dump_tlog(W, "bfs1");
}

// ---------------------------------------------------------------------------
// multi-source: 64 lanes, one bit per source in seen/frontier words
// ---------------------------------------------------------------------------
struct Bfs64Args {
  const int64_t* rp;
  const int32_t* col;
  const int64_t* trp;
  const int32_t* tcol;
  int64_t n, nnz;
  unsigned long long lanes;
  unsigned long long* seen;
  unsigned long long* f0;
  unsigned long long* f1;
  unsigned long long* f2;
  int32_t* mlevel;   // [n][64]
  int32_t* mparent;  // [n][64]
  int64_t* q0;
  int64_t* q1;
  int* ctl;  // [0] entries [1] vertices [2] next entries [3] next vertices [5] levels [6] push
  unsigned long long* edges;  // [0] frontier edges cur, [1] next
  unsigned long long* tlog;   // optional: %globaltimer at phase boundaries (debug)
  int pull_div;               // pull once frontier edges >= nnz / pull_div
  const int32_t* heavy;       // vertices with in-degree > kBfsHeavy
  int64_t nheavy;
  const int32_t* unz;         // vertices with in-edges, ascending: what a pull level scans
  int64_t nunz;
};


// k_bfs64 control words: triple-buffered queue counters (entries, vertices,
// frontier edges as u64 at ctl + 8), levels done, push levels
constexpr int kB64Ent = 0, kB64Vtx = 3, kB64Levels = 6, kB64Push = 7, kB64Words = 16;

__global__ void __launch_bounds__(kBfsThreads) k_bfs64(Bfs64Args a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ int32_t s_buf[kBfsThreads / 32][kBfsBuf];
  __shared__ int32_t s_kbuf[kBfsThreads / 32][kBfsBuf];
  __shared__ __align__(8) int s_red[6];
  FrontierQueue<kBfsBuf> fq;
  fq.buf = s_buf[threadIdx.x >> 5];
  fq.rp = a.rp;
  fq.chunk = kChunk;
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  // level d pops the queue counted in buffer d%3 and pushes into (d+1)%3;
  // buffer (d+2)%3 -- last read during level d-1, before its closing barrier
  // -- is zeroed by the leader for level d+1.  ONE grid barrier per level:
  // the frontier words are a ring of 3 (level d reads f[d-1], writes f[d],
  // clears f[d+1], which only level d-1 read) and "seen" lags one level --
  // level d folds level d-1's frontier into seen (and writes its level rows)
  // while testing visits against seen | f[d-1], which is exact either way
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long* fr[3] = {a.f0, a.f1, a.f2};
  // (depth <= n - 1, so level n always finds an empty frontier and stops)
  for (int d = 1; static_cast<int64_t>(d) <= a.n; ++d) {
    const int bc = d % 3, bn = (d + 1) % 3, bz = (d + 2) % 3;
    const int qe = *(volatile int*)&a.ctl[kB64Ent + bc];
    const int qv = *(volatile int*)&a.ctl[kB64Vtx + bc];
    const unsigned long long fe = *(volatile unsigned long long*)&a.edges[bc];
    if (qv == 0) break;
    if (leader) {
      a.ctl[kB64Ent + bz] = 0;
      a.ctl[kB64Vtx + bz] = 0;
      a.edges[bz] = 0ull;
    }
    // 64 lanes rarely satisfy every source bit early in a pull (and hub rows
    // straggle in one group), so push until the frontier edges reach nnz/2
    const bool push = fe * static_cast<unsigned long long>(a.pull_div) <
                      static_cast<unsigned long long>(a.nnz) + 1ull;
    if (a.tlog && blockIdx.x == 0 && threadIdx.x == 0) {
      a.tlog[4 * d] = gtimer();
      a.tlog[4 * d + 3] = (push ? 1ull : 0ull) | (static_cast<unsigned long long>(qv) << 8);
    }
    const int p = (d - 1) & 1;
    const int64_t* qc = p ? a.q1 : a.q0;
    int64_t* qn = p ? a.q0 : a.q1;
    unsigned long long* fc = fr[(d - 1) % 3];
    unsigned long long* fn = fr[d % 3];
    {
      unsigned long long* fz = fr[(d + 1) % 3];  // written by level d+1
      for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < a.n;
           i += int64_t(gridDim.x) * blockDim.x)
        fz[i] = 0ull;
    }
    // level d-1's frontier into seen + its level rows (a warp per vertex,
    // lanes b and b+32 write the vertex's 256-byte level row coalesced)
    for (int64_t e = gwarp; e < qe; e += nwarps) {
      const int64_t ent = qc[e];
      if ((ent >> 32) != 0) continue;
      const int32_t w = static_cast<int32_t>(ent & 0xffffffff);
      const unsigned long long nb = fc[w];
      if (lane == 0) a.seen[w] |= nb;
      int32_t* lv = a.mlevel + static_cast<int64_t>(w) * 64;
      if ((nb >> lane) & 1ull) lv[lane] = d - 1;
      if ((nb >> (lane + 32)) & 1ull) lv[lane + 32] = d - 1;
    }
    fq.reset(qn, &a.ctl[kB64Ent + bn], &a.ctl[kB64Vtx + bn], &a.edges[bn], nullptr);
    if (push) {
      // small queues: every entry split over S warps (as in k_bfs1)
      int S = 1;
      while (S < 8 && static_cast<int64_t>(qe) * S * 2 <= nwarps) S <<= 1;
      const int64_t sub = kChunk / S;
      for (int64_t e2 = gwarp; e2 < static_cast<int64_t>(qe) * S; e2 += nwarps) {
        const int64_t e = e2 / S;
        const int part = static_cast<int>(e2 - e * S);
        const int64_t ent = qc[e];
        const int32_t v = static_cast<int32_t>(ent & 0xffffffff);
        const int64_t c = ent >> 32;
        const unsigned long long f = fc[v];
        const int64_t cb = a.rp[v] + c * kChunk;
        const int64_t ce = min(a.rp[v + 1], cb + kChunk);
        const int64_t b0 = cb + part * sub;
        const int64_t e0 = min(ce, b0 + sub);
        for (int64_t base = b0; base < e0; base += 32) {
          const int64_t q = base + lane;
          bool has = false;
          int32_t w = 0;
          if (q < e0) {
            w = __ldg(a.col + q);
            GBX_DCHECK(w >= 0 && w < a.n, "bfs push column", w);
            unsigned long long bits = f & ~(a.seen[w] | fc[w]);
            if (bits) {
              unsigned long long old = atomicOr(&fn[w], bits);
              has = old == 0ull;
              while (bits) {
                int b = __ffsll(static_cast<long long>(bits)) - 1;
                bits &= bits - 1;
                atomicMin(&a.mparent[static_cast<int64_t>(w) * 64 + b], v);
              }
            }
          }
          fq.push(has, w);
        }
      }
    } else {
      const int grp = lane >> 3, sub = lane & 7;
      const unsigned gmask = 0xffu << (grp * 8);
      // (only the vertices with in-edges: the others can never be pulled)
      for (int64_t vb = gwarp * 4; vb < a.nunz; vb += nwarps * 4) {
        const int64_t w = vb + grp < a.nunz ? a.unz[vb + grp] : a.n;
        unsigned long long need = w < a.n ? (~(a.seen[w] | fc[w]) & a.lanes) : 0ull;
        bool active = need != 0ull;
        int64_t pp = active ? a.trp[w] : 0, pe = active ? a.trp[w + 1] : 0;
        if (pe - pp > kBfsHeavy) active = false;  // hub: the warp pass below
        unsigned long long found = 0ull;
        while (__any_sync(kFull, active)) {
          int32_t u = -1;
          unsigned long long hit = 0ull;
          if (active && pp + sub < pe) {
            u = __ldg(a.tcol + pp + sub);
            GBX_DCHECK(u >= 0 && u < a.n, "bfs pull column", u);
            hit = ld_weak(fc + u) & need;
          }
          // exclusive prefix-OR over the 8 lanes of the group: the lowest
          // lane (smallest neighbour id) claims each newly found source bit
          unsigned long long incl = hit;
#pragma unroll
          for (int o = 1; o < 8; o <<= 1) {
            unsigned long long t = __shfl_up_sync(kFull, incl, o);
            if (sub >= o) incl |= t;
          }
          unsigned long long excl = __shfl_up_sync(kFull, incl, 1);
          if (sub == 0) excl = 0ull;
          unsigned long long mine = hit & ~excl;
          const unsigned long long tot = __shfl_sync(kFull, incl, grp * 8 + 7);
          (void)gmask;
          while (mine) {
            int b = __ffsll(static_cast<long long>(mine)) - 1;
            mine &= mine - 1;
            a.mparent[w * 64 + b] = u;
          }
          if (active) {
            found |= tot;
            need &= ~tot;
            pp += 8;
            if (need == 0ull || pp >= pe) active = false;
          }
        }
        const bool has = sub == 0 && found != 0ull;
        if (has) fn[w] = found;
        fq.push(has, static_cast<int32_t>(w));
      }
      // hubs: one warp per vertex, 32 in-neighbours per step, lowest lane
      // (smallest neighbour id) claims each source bit as in the groups above
      for (int64_t h = gwarp; h < a.nheavy; h += nwarps) {
        const int32_t w = a.heavy[h];
        unsigned long long need = ~(a.seen[w] | fc[w]) & a.lanes;
        unsigned long long found = 0ull;
        if (need) {
          const int64_t pe = a.trp[w + 1];
          for (int64_t pp = a.trp[w]; pp < pe; pp += 32) {
            int32_t u = -1;
            unsigned long long hit = 0ull;
            if (pp + lane < pe) {
              u = __ldg(a.tcol + pp + lane);
              GBX_DCHECK(u >= 0 && u < a.n, "bfs pull column", u);
            GBX_DCHECK(u >= 0 && u < a.n, "bfs pull column", u);
              hit = ld_weak(fc + u) & need;
            }
            unsigned long long incl = hit;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              unsigned long long t = __shfl_up_sync(kFull, incl, o);
              if (lane >= o) incl |= t;
            }
            unsigned long long excl = __shfl_up_sync(kFull, incl, 1);
            if (lane == 0) excl = 0ull;
            unsigned long long mine = hit & ~excl;
            const unsigned long long tot = __shfl_sync(kFull, incl, 31);
            while (mine) {
              int b = __ffsll(static_cast<long long>(mine)) - 1;
              mine &= mine - 1;
              a.mparent[static_cast<int64_t>(w) * 64 + b] = u;
            }
            found |= tot;
            need &= ~tot;
            if (need == 0ull) break;
          }
        }
        const bool has = lane == 0 && found != 0ull;
        if (has) fn[w] = found;
        fq.push(has, w);
      }
    }
    fq.flush_block(s_kbuf[threadIdx.x >> 5], s_red);
    if (a.tlog && blockIdx.x == 0 && threadIdx.x == 0) a.tlog[4 * d + 1] = gtimer();
    if (leader) {
      a.ctl[kB64Levels] = d;
      if (push) a.ctl[kB64Push] += 1;
    }
    grid.sync();
    if (a.tlog && blockIdx.x == 0 && threadIdx.x == 0) a.tlog[4 * d + 2] = gtimer();
  }
}

__global__ void k_bfs64_init(unsigned long long* seen, unsigned long long* f0,
                             unsigned long long* f1, unsigned long long* f2, int32_t* mlevel,
                             int32_t* mparent, int64_t n) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) { seen[i] = 0ull; f0[i] = 0ull; f1[i] = 0ull; f2[i] = 0ull; }
  if (i < n * 64) { mlevel[i] = -1; mparent[i] = INT_MAX; }
}

// One warp per distinct source: set its lane bits, then emit its degree chunks
// into the level-1 queue (counter buffer 1: entries, vertices, frontier edges).
// src[0..ns) are the batch lanes, src[ns..ns+nu) the distinct sources.
__global__ void k_bfs64_seed(const int32_t* src, int ns, int nu, const int64_t* rp,
                             unsigned long long* seen, unsigned long long* f0, int32_t* mlevel,
                             int32_t* mparent, int64_t* q, int* ctl,
                             unsigned long long* edges) {
  const int u = blockIdx.x;
  const int lane = threadIdx.x;
  const int32_t v = src[ns + u];
  if (lane == 0) {
    unsigned long long bits = 0ull;
    for (int b = 0; b < ns; ++b)
      if (src[b] == v) {
        bits |= 1ull << b;
        mlevel[static_cast<int64_t>(v) * 64 + b] = 0;
        mparent[static_cast<int64_t>(v) * 64 + b] = v;
      }
    seen[v] = bits;
    f0[v] = bits;
  }
  const int64_t deg = rp[v + 1] - rp[v];
  const int64_t k = deg <= kChunk ? 1 : (deg + kChunk - 1) / kChunk;
  int base = 0;
  if (lane == 0) {
    base = atomicAdd(&ctl[kB64Ent + 1], static_cast<int>(k));  // level 1 pops buffer 1
    atomicAdd(&ctl[kB64Vtx + 1], 1);
    atomicAdd(edges + 1, static_cast<unsigned long long>(deg));
  }
  base = __shfl_sync(0xffffffffu, base, 0);
  for (int64_t c = lane; c < k; c += 32) q[base + c] = (c << 32) | v;
}

// [n][64] int32 -> [ns][n] int64 (-1 for none)
__global__ void k_lanes_out(const int32_t* in, int64_t n, int ns, int32_t none, int64_t* out) {
  __shared__ int32_t tile[32][65];
  const int64_t v0 = blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    int64_t v = v0 + r;
    for (int b = threadIdx.x; b < 64; b += blockDim.x)
      tile[r][b] = v < n ? in[v * 64 + b] : none;
  }
  __syncthreads();
  for (int b = threadIdx.y; b < ns; b += blockDim.y) {
    int64_t v = v0 + threadIdx.x;
    if (v < n) {
      int32_t x = tile[threadIdx.x][b];
      out[static_cast<int64_t>(b) * n + v] = x == none ? -1 : x;
    }
  }
}

static void ensure_bfs64(gbx_graph* g) {
  if (!g->bfs) g->bfs = std::make_unique<BfsWork>();
  BfsWork& W = *g->bfs;
  const int64_t n = g->A.n;
  if (W.seen.p && W.seen.n >= static_cast<size_t>(std::max<int64_t>(n, 1))) return;
  W.seen.alloc(std::max<int64_t>(n, 1));
  W.front.alloc(std::max<int64_t>(n, 1));
  W.next.alloc(std::max<int64_t>(n, 1));
  W.third.alloc(std::max<int64_t>(n, 1));
  W.mlevel.alloc(std::max<int64_t>(n, 1) * 64);
  W.mparent.alloc(std::max<int64_t>(n, 1) * 64);
  const int64_t qcap = n + g->A.nnz / kChunk + 64;
  W.mqueue[0].alloc(2 * qcap);
  W.mqueue[1].alloc(2 * qcap);
  W.mctl.alloc(kB64Words);
  W.msrc.alloc(128);
}

void bfs_batch_run(gbx_graph* g, const uint64_t* sources, uint64_t ns, int64_t* parent,
                   int64_t* level) {
  NvtxRange nvtx_("gbx.bfs.batch64");
  require_at(g, "bfs_batch");
  const int64_t n = g->A.n;
  if (ns == 0) fail(GBX_EMPTY_BATCH, "empty source batch");
  for (uint64_t b = 0; b < ns; ++b)
    if (sources[b] >= static_cast<uint64_t>(n))
      fail(GBX_SOURCE_OUT_OF_RANGE, "source " + std::to_string(sources[b]));
  ensure_bfs64(g);
  BfsWork& W = *g->bfs;
  cudaStream_t s = g->stream;
  const Csr& A = g->A;
  const Csr& AT = g->AT();
  ensure_heavy(g, AT);
  static int grid = 0;
  if (!grid) grid = coop_grid(reinterpret_cast<const void*>(k_bfs64), kBfsThreads);
  int64_t total_launches = 0;
  g->pending_iters = nullptr;
  for (uint64_t b0 = 0; b0 < ns; b0 += 64) {
    const int nb = static_cast<int>(std::min<uint64_t>(64, ns - b0));
    k_bfs64_init<<<ceil_div(n * 64, 256), 256, 0, s>>>(W.seen.p, W.front.p, W.next.p,
                                                       W.third.p, W.mlevel.p, W.mparent.p, n);
    GBX_LAUNCHED();
    // lanes then distinct sources; the seed kernel builds the level-1 queue
    std::vector<int32_t> src(nb);
    for (int b = 0; b < nb; ++b) src[b] = static_cast<int32_t>(sources[b0 + b]);
    std::vector<int32_t> uniq(src);
    std::sort(uniq.begin(), uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    const int nu = static_cast<int>(uniq.size());
    src.insert(src.end(), uniq.begin(), uniq.end());
    int64_t* q0 = reinterpret_cast<int64_t*>(W.mqueue[0].p);
    int64_t* q1 = reinterpret_cast<int64_t*>(W.mqueue[1].p);
    GBX_CUDA(cudaMemsetAsync(W.mctl.p, 0, kB64Words * sizeof(int), s));
    GBX_CUDA(cudaMemcpyAsync(W.msrc.p, src.data(), src.size() * sizeof(int32_t),
                             cudaMemcpyHostToDevice, s));
    k_bfs64_seed<<<nu, 32, 0, s>>>(W.msrc.p, nb, nu, A.rp.p, W.seen.p, W.front.p, W.mlevel.p,
                                   W.mparent.p, q0, W.mctl.p,
                                   reinterpret_cast<unsigned long long*>(W.mctl.p + 8));
    GBX_LAUNCHED();
    Bfs64Args a{};
    a.rp = A.rp.p;
    a.col = A.col.p;
    a.trp = AT.rp.p;
    a.tcol = AT.col.p;
    a.n = n;
    a.nnz = A.nnz;
    a.lanes = nb == 64 ? ~0ull : ((1ull << nb) - 1);
    a.seen = W.seen.p;
    a.f0 = W.front.p;
    a.f1 = W.next.p;
    a.f2 = W.third.p;
    a.mlevel = W.mlevel.p;
    a.mparent = W.mparent.p;
    a.q0 = q0;
    a.q1 = q1;
    a.ctl = W.mctl.p;
    a.edges = reinterpret_cast<unsigned long long*>(W.mctl.p + 8);
    const int pull_div = static_cast<int>(option(kOptBfs64PullDiv));
    a.pull_div = pull_div;
    a.heavy = W.heavy.p;
    a.unz = W.unz.p;
    a.nunz = W.nunz;
    a.nheavy = W.nheavy;
    const bool tlog_on = option(kOptBfsTrace) != 0;
    if (tlog_on) {
      if (!W.tlog.p) W.tlog.alloc(4 * 256);
      GBX_CUDA(cudaMemsetAsync(W.tlog.p, 0, W.tlog.bytes(), s));
      a.tlog = W.tlog.p;
    }
    void* args[] = {&a};
    if (n > 1) {
      GBX_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_bfs64), dim3(grid),
                                           dim3(kBfsThreads), args, 0, s));
    }
    total_launches += 3;
    W.ms_ns = nb;
    if (parent || level) {
      int64_t* tmp = nullptr;
      GBX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tmp), std::max<int64_t>(n, 1) * nb * 8, s));
      dim3 blk(32, 8);
      if (parent) {
        k_lanes_out<<<ceil_div(n, 32), blk, 0, s>>>(W.mparent.p, n, nb, INT_MAX, tmp);
        GBX_LAUNCHED();
        GBX_CUDA(cudaMemcpyAsync(parent + b0 * n, tmp, n * nb * 8, cudaMemcpyDeviceToHost, s));
        total_launches++;
      }
      if (level) {
        k_lanes_out<<<ceil_div(n, 32), blk, 0, s>>>(W.mlevel.p, n, nb, -1, tmp);
        GBX_LAUNCHED();
        GBX_CUDA(cudaMemcpyAsync(level + b0 * n, tmp, n * nb * 8, cudaMemcpyDeviceToHost, s));
        total_launches++;
      }
      cudaFreeAsync(tmp, s);
    }
    int hctl[kB64Words];
    GBX_CUDA(cudaMemcpyAsync(hctl, W.mctl.p, sizeof hctl, cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaStreamSynchronize(s));
    g->stats.iterations = hctl[kB64Levels];
    if (tlog_on) dump_tlog(W, "bfs64");
  }
  g->stats.launches = total_launches;
  g->stats.hot_launches = (ns + 63) / 64;
}


// ---------------------------------------------------------------------------
// Row-sharded single-source BFS for the multi-GPU driver (scale >=
// 22): rank r owns the 32-aligned vertex block [rb, re) (balanced by AT nnz +
// rows).  Per level every rank pulls its still-unvisited owned vertices
// against the GLOBAL frontier bitmap (n bits) -- the first frontier
// in-neighbour in the ascending AT row is the parent, the minimum id exactly
// as in the single-GPU traversal -- and writes its slice of the next bitmap;
// the driver all-gathers the slices (the north_star's frontier-bitmap
// all-gather) and sums the found counts.  Pull-only: results are identical
// to gbx_bfs (parents are min-id in both directions).
// ---------------------------------------------------------------------------

// 8 lanes per vertex, 4 vertices per warp step: the group scans its AT row 8
// edges per step; the lowest lane with a frontier hit holds the min-id parent
__global__ void __launch_bounds__(256) k_bfs_shard_pull(const int64_t* trp, const int32_t* tcol,
                                                        int64_t rb, int64_t re,
                                                        const int32_t* ul_in, int ucnt,
                                                        const uint32_t* front, int d,
                                                        int32_t* level, int32_t* parent,
                                                        uint32_t* next_slice, int32_t* ul_out,
                                                        int* cnt) {
  const int lane = threadIdx.x & 31;
  const int grp = lane >> 3, sub = lane & 7;
  const unsigned gmask = 0xffu << (grp * 8);
  const int64_t gwarp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t range = ucnt < 0 ? re - rb : ucnt;
  int found = 0;
  for (int64_t base = gwarp * 4; base < range; base += nwarps * 4) {
    const int64_t i = base + grp;
    int64_t v = -1;
    if (i < range) v = ucnt < 0 ? rb + i : ul_in[i];
    bool active = v >= 0 && level[v] == -1;
    int64_t p = active ? trp[v] : 0;
    const int64_t e = active ? trp[v + 1] : 0;
    const bool nonempty = e > p;
    int32_t par = -1;
    while (__any_sync(kFull, active)) {
      bool hit = false;
      int32_t u = 0;
      if (active && p + sub < e) {
        u = __ldg(tcol + p + sub);
        hit = (__ldg(front + (u >> 5)) >> (u & 31)) & 1u;
      }
      const unsigned hb = __ballot_sync(kFull, hit) & gmask;
      if (active) {
        if (hb) {
          const int first = __ffs(hb) - 1;  // lowest lane = smallest neighbour id
          par = __shfl_sync(gmask, u, first, 32);
          active = false;
        } else {
          p += 8;
          if (p >= e) active = false;
        }
      } else {
        (void)__shfl_sync(gmask, u, grp * 8, 32);
      }
    }
    if (v >= 0 && sub == 0) {
      if (par >= 0) {
        level[v] = d;
        parent[v] = par;
        const int64_t w = (v >> 5) - (rb >> 5);
        atomicOr(next_slice + w, 1u << (v & 31));
        ++found;
      } else if (nonempty && level[v] == -1) {
        ul_out[agg_append(&cnt[1])] = static_cast<int32_t>(v);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) found += __shfl_xor_sync(kFull, found, o);
  if (lane == 0 && found) atomicAdd(&cnt[0], found);
}

__global__ void k_bfs_shard_init(int32_t* level, int32_t* parent, int64_t rb, int64_t re,
                                 int32_t src) {
  const int64_t v = rb + blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (v >= re) return;
  level[v] = v == src ? 0 : -1;
  parent[v] = v == src ? src : -1;
}

__global__ void k_bfs_shard_split(const int64_t* trp, int64_t n, int parts, int64_t* bounds) {
  const int q = threadIdx.x;
  if (q > parts) return;
  const int64_t target = (n + trp[n]) * q / parts;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (mid + trp[mid] < target) lo = mid + 1; else hi = mid;
  }
  // 32-aligned so every rank owns whole bitmap words
  bounds[q] = q == 0 ? 0 : q == parts ? n : min(n, (lo + 31) & ~int64_t(31));
}

static BfsShard& need_bfs_shard(gbx_graph* g) {
  if (!g->bfs || !g->bfs->shard) fail(GBX_MISSING_PROPERTY, "bfs shard protocol needs gbx_bfs_shard_begin");
  return *g->bfs->shard;
}

void bfs_shard_begin(gbx_graph* g, uint64_t source, int rank, int nranks, int64_t* rb_out,
                     int64_t* re_out, const int64_t* bounds) {
  require_at(g, "bfs_shard");
  const int64_t n = g->A.n;
  if (source >= static_cast<uint64_t>(n)) fail(GBX_SOURCE_OUT_OF_RANGE, "source " + std::to_string(source));
  if (nranks < 1 || rank < 0 || rank >= nranks) fail(GBX_INVALID_VALUE, "bfs_shard: bad rank / nranks");
  ensure_bfs1(g);
  BfsWork& W = *g->bfs;
  cudaStream_t s = g->stream;
  const Csr& AT = g->AT();
  auto S = std::make_unique<BfsShard>();
  S->rank = rank;
  S->nranks = nranks;
  S->source = static_cast<int32_t>(source);
  if (bounds) {
    // the distributed graph's ownership (32-aligned; its shard holds only these rows)
    S->rb = bounds[rank];
    S->re = bounds[rank + 1];
    if ((S->rb & 31) || (S->re < n && (S->re & 31)))
      fail(GBX_INVALID_VALUE, "bfs_shard: row blocks must be 32-aligned");
  } else {
    DevArray<int64_t> b(nranks + 1);
    k_bfs_shard_split<<<1, ((nranks + 32) / 32) * 32, 0, s>>>(AT.rp.p, n, nranks, b.p);
    GBX_LAUNCHED();
    std::vector<int64_t> hb(nranks + 1);
    GBX_CUDA(cudaMemcpyAsync(hb.data(), b.p, (nranks + 1) * 8, cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaStreamSynchronize(s));
    for (int q = 1; q <= nranks; ++q) hb[q] = std::max(hb[q], hb[q - 1]);
    S->rb = hb[rank];
    S->re = hb[rank + 1];
  }
  S->cnt.alloc(2);
  if (S->re > S->rb) {
    k_bfs_shard_init<<<ceil_div(S->re - S->rb, 256), 256, 0, s>>>(W.level.p, W.parent.p, S->rb,
                                                                   S->re, S->source);
    GBX_LAUNCHED();
  }
  GBX_CUDA(cudaStreamSynchronize(s));
  W.shard = std::move(S);
  if (rb_out) *rb_out = W.shard->rb;
  if (re_out) *re_out = W.shard->re;
}

// one level: pull the owned unvisited vertices against front (n bits, global);
// next_slice = this rank's words [rb/32, ceil(re/32)) of the next frontier
void bfs_shard_level(gbx_graph* g, const uint32_t* front, uint32_t* next_slice, int64_t* found) {
  NvtxRange nvtx_("gbx.bfs.shard_level");
  BfsShard& S = need_bfs_shard(g);
  BfsWork& W = *g->bfs;
  cudaStream_t s = g->stream;
  const Csr& AT = g->AT();
  const int64_t words = (S.re + 31) / 32 - S.rb / 32;
  if (words > 0) GBX_CUDA(cudaMemsetAsync(next_slice, 0, words * 4, s));
  GBX_CUDA(cudaMemsetAsync(S.cnt.p, 0, 2 * sizeof(int), s));
  const int d = S.d + 1;
  const int grid = device_sms() * 8;
  if (S.re > S.rb && S.ucnt != 0) {
    k_bfs_shard_pull<<<grid, 256, 0, s>>>(AT.rp.p, AT.col.p, S.rb, S.re, W.ulist[S.ul].p, S.ucnt,
                                          front, d, W.level.p, W.parent.p, next_slice,
                                          W.ulist[S.ul ^ 1].p, S.cnt.p);
    GBX_LAUNCHED();
  }
  int hc[2] = {0, 0};
  GBX_CUDA(cudaMemcpyAsync(hc, S.cnt.p, sizeof hc, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  if (S.re > S.rb && S.ucnt != 0) {
    S.ucnt = hc[1];
    S.ul ^= 1;
  }
  S.d = d;
  *found = hc[0];
}

// ---- push levels of the row-sharded BFS (small frontiers): the owned
// frontier vertices mark their out-neighbours as candidates (a byte per
// vertex, max-reduced over the ranks by the driver); each rank then pulls
// only its owned unvisited candidates -- the same min-id parent as a full
// pull (the first frontier hit in the ascending AT row), at the cost of the
// frontier's edges instead of every unvisited row.

// owned frontier vertices (bits of front in [rb, re)) -> light list (a warp
// each) and heavy list (rows longer than kBfsMarkHeavy: the whole grid)
constexpr int64_t kBfsMarkHeavy = 2048;
__global__ void k_bfs_owned_front(const uint32_t* front, const int64_t* rp, int64_t rb, int64_t re,
                                  int32_t* list, int* cnt, int32_t* heavy, int* hcnt) {
  const int64_t v = rb + blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const bool on = v < re && ((front[v >> 5] >> (v & 31)) & 1u);
  if (!on) return;
  if (rp[v + 1] - rp[v] > kBfsMarkHeavy) heavy[agg_append(hcnt)] = static_cast<int32_t>(v);
  else list[agg_append(cnt)] = static_cast<int32_t>(v);
}

// a warp per light frontier vertex, then every thread of the grid over the
// heavy ones' edges: every out-neighbour becomes a candidate
__global__ void __launch_bounds__(256) k_bfs_shard_mark(const int64_t* rp, const int32_t* col,
                                                        int64_t n, const int32_t* list,
                                                        const int* cnt, const int32_t* heavy,
                                                        const int* hcnt, uint8_t* cand) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int m = *cnt;
  for (int64_t i = gw; i < m; i += nw) {
    const int32_t u = list[i];
    for (int64_t p = rp[u] + lane; p < rp[u + 1]; p += 32) {
      const int32_t v = __ldg(col + p);
      GBX_DCHECK(v >= 0 && v < n, "bfs push column", v);
      cand[v] = 1;  // idempotent plain store
    }
  }
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t nt = int64_t(gridDim.x) * blockDim.x;
  const int mh = *hcnt;
  for (int h = 0; h < mh; ++h) {
    const int32_t u = heavy[h];
    for (int64_t p = rp[u] + t; p < rp[u + 1]; p += nt) {
      const int32_t v = __ldg(col + p);
      GBX_DCHECK(v >= 0 && v < n, "bfs push column", v);
      cand[v] = 1;
    }
  }
}

// owned unvisited candidates -> list
__global__ void k_bfs_cand_list(const uint8_t* cand, const int32_t* level, int64_t rb, int64_t re,
                                int32_t* list, int* cnt) {
  const int64_t v = rb + blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const bool on = v < re && cand[v] && level[v] == -1;
  if (on) list[agg_append(cnt)] = static_cast<int32_t>(v);
}

// edges of the owned frontier vertices (the direction rule's measure)
__global__ void k_bfs_front_edges(const uint32_t* front, const int64_t* rp, int64_t rb, int64_t re,
                                  unsigned long long* out) {
  const int64_t v = rb + blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  unsigned long long e = 0;
  if (v < re && ((front[v >> 5] >> (v & 31)) & 1u)) e = static_cast<unsigned long long>(rp[v + 1] - rp[v]);
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
  if ((threadIdx.x & 31) == 0 && e) atomicAdd(out, e);
}

int64_t bfs_shard_front_edges(gbx_graph* g, const uint32_t* front) {
  BfsShard& S = need_bfs_shard(g);
  cudaStream_t s = g->stream;
  if (S.re <= S.rb) return 0;
  Tmp<unsigned long long> e(1, s);
  GBX_CUDA(cudaMemsetAsync(e.p, 0, 8, s));
  k_bfs_front_edges<<<ceil_div(S.re - S.rb, 256), 256, 0, s>>>(front, g->A.rp.p, S.rb, S.re, e.p);
  GBX_LAUNCHED();
  unsigned long long h = 0;
  GBX_CUDA(cudaMemcpyAsync(&h, e.p, 8, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  return static_cast<int64_t>(h);
}

// this rank's level / parent words of its owned rows (device, int32; -1 =
// unreached): the driver gathers them on the device
void bfs_shard_result_device(gbx_graph* g, const int32_t** level, const int32_t** parent) {
  need_bfs_shard(g);
  *level = g->bfs->level.p;
  *parent = g->bfs->parent.p;
}

// mark phase: cand (n bytes, zeroed by the caller) gets this rank's owned
// frontier vertices' out-neighbours
void bfs_shard_push_mark(gbx_graph* g, const uint32_t* front, uint8_t* cand) {
  NvtxRange nvtx_("gbx.bfs.shard_push_mark");
  BfsShard& S = need_bfs_shard(g);
  BfsWork& W = *g->bfs;
  cudaStream_t s = g->stream;
  const Csr& A = g->A;
  if (S.re <= S.rb) return;
  int32_t* list = reinterpret_cast<int32_t*>(W.queue[0].p);
  int32_t* heavy = reinterpret_cast<int32_t*>(W.queue[1].p);
  GBX_CUDA(cudaMemsetAsync(S.cnt.p, 0, 2 * sizeof(int), s));
  k_bfs_owned_front<<<ceil_div(S.re - S.rb, 256), 256, 0, s>>>(front, A.rp.p, S.rb, S.re, list,
                                                               S.cnt.p, heavy, S.cnt.p + 1);
  k_bfs_shard_mark<<<device_sms() * 8, 256, 0, s>>>(A.rp.p, A.col.p, A.n, list, S.cnt.p, heavy,
                                                    S.cnt.p + 1, cand);
  GBX_LAUNCHED();
  GBX_CUDA(cudaStreamSynchronize(s));
}

// pull phase of a push level: only the owned unvisited candidates (every
// rank's marks max-reduced into cand); the owned still-unvisited list of the
// pull levels is left as it is (the pull kernel skips vertices visited since)
void bfs_shard_push_level(gbx_graph* g, const uint8_t* cand, const uint32_t* front,
                          uint32_t* next_slice, int64_t* found) {
  NvtxRange nvtx_("gbx.bfs.shard_push_level");
  BfsShard& S = need_bfs_shard(g);
  BfsWork& W = *g->bfs;
  cudaStream_t s = g->stream;
  const Csr& AT = g->AT();
  const int64_t words = (S.re + 31) / 32 - S.rb / 32;
  if (words > 0) GBX_CUDA(cudaMemsetAsync(next_slice, 0, words * 4, s));
  const int d = S.d + 1;
  int hc[2] = {0, 0};
  if (S.re > S.rb) {
    int32_t* clist = reinterpret_cast<int32_t*>(W.queue[0].p);
    int32_t* scratch = reinterpret_cast<int32_t*>(W.queue[1].p);
    GBX_CUDA(cudaMemsetAsync(S.cnt.p, 0, 2 * sizeof(int), s));
    k_bfs_cand_list<<<ceil_div(S.re - S.rb, 256), 256, 0, s>>>(cand, W.level.p, S.rb, S.re, clist,
                                                               S.cnt.p + 1);
    GBX_LAUNCHED();
    int nc = 0;
    GBX_CUDA(cudaMemcpyAsync(&nc, S.cnt.p + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaStreamSynchronize(s));
    GBX_CUDA(cudaMemsetAsync(S.cnt.p, 0, 2 * sizeof(int), s));
    if (nc > 0) {
      k_bfs_shard_pull<<<device_sms() * 8, 256, 0, s>>>(AT.rp.p, AT.col.p, S.rb, S.re, clist, nc,
                                                        front, d, W.level.p, W.parent.p,
                                                        next_slice, scratch, S.cnt.p);
      GBX_LAUNCHED();
    }
    GBX_CUDA(cudaMemcpyAsync(hc, S.cnt.p, sizeof hc, cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaStreamSynchronize(s));
  }
  S.d = d;
  *found = hc[0];
}

// owned rows [rb, re): parent / level (-1 = unreached), host arrays of re - rb
void bfs_shard_result(gbx_graph* g, int64_t* parent, int64_t* level) {
  BfsShard& S = need_bfs_shard(g);
  BfsWork& W = *g->bfs;
  cudaStream_t s = g->stream;
  const int64_t m = S.re - S.rb;
  if (m <= 0) return;
  std::vector<int32_t> tp(m), tl(m);
  GBX_CUDA(cudaMemcpyAsync(tp.data(), W.parent.p + S.rb, m * 4, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaMemcpyAsync(tl.data(), W.level.p + S.rb, m * 4, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  for (int64_t i = 0; i < m; ++i) {
    if (parent) parent[i] = tl[i] < 0 ? -1 : tp[i];
    if (level) level[i] = tl[i];
  }
}

}  // namespace gbx
