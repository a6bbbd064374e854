// plans.cuh -- per-algorithm device layouts and workspaces owned by a gbx_graph.
#pragma once

#include <vector>

#include "common.cuh"

namespace gbx {

// A PageRank work bin: warp units [unit0, next bin's unit0) cover rows
// [row0, row1), 32/2^lg rows per unit with 2^lg lanes per row.  len >= 0: every
// row has exactly len nonzeros starting at p0 + (row - row0) * len.
constexpr int kPrBinsMax = 160;
struct PrBin {
  int64_t unit0, row0, row1, p0;
  int32_t len;
  int32_t lg;
};
// the copy the row kernels stage in shared memory (24 bytes; units and rows fit
// 32 bits: column ids are int32)
struct PrBinS {
  int64_t p0;
  int32_t unit0, row0, row1, len;
};

// PageRank pull plan (pagerank.cu): AT relabeled by descending in-degree,
// rows binned into warp units (G lanes per row) and long-row chunks.
struct PrPlan {
  int64_t n = 0, nnz = 0, row0 = 0, row1 = 0;  // rows [row0,row1) of the relabeled AT
  DevArray<int64_t> trp;           // relabeled AT
  DevArray<int32_t> tcol;
  DevArray<int32_t> deg;           // relabeled out-degree
  DevArray<int32_t> new2old, old2new;
  DevArray<PrBin> bins;            // warp units by bin
  int nbins = 0;
  int64_t nunits = 0;
  int64_t zrow0 = 0, zrow1 = 0;    // rows without in-edges
  DevArray<int64_t> chunk_p;       // [2 * nchunks] nonzero ranges of long rows
  int64_t nchunks = 0;
  DevArray<int32_t> long_row;
  DevArray<int64_t> long_slot;     // [nlong + 1]
  int64_t nlong = 0;
  DevArray<double> slot;           // chunk partial sums
  int grid = 0, grid_fin = 1;
  DevArray<float> r[2], x[2];      // fp32 storage (tol >= 1e-6)
  DevArray<double> rd[2], xd[2];    // fp64 storage (tight tolerances)
  DevArray<double> out;            // ranks in original vertex order
  DevArray<float> invf;            // damping / out-degree (fp32 storage)
  DevArray<double> invd;           // damping / out-degree (fp64 storage)
  DevArray<double> l1_block, l1_fin, l1_hist;
  DevArray<int> ctl;            // [0] completed iterations, [1] done, [2] peer timeout
  DevArray<unsigned long long> ktime;  // k_pr_rows launch spans (%globaltimer)
  DevArray<unsigned long long> cta_end;  // trace: per-CTA row-phase end times
  double last_rows_ms = 0.0;
  bool last_persist = false;       // the last run used k_pr_persist
  DevArray<unsigned> blk_cnt;
  double g_damping = -1;           // damping the shard's inv vector was built for
  int last_prec = 32;
  int last_iters = 0;
};

// Sharded PageRank step (multi-GPU driver): a PrPlan over a row block.
struct PrShard {
  PrPlan plan;
  int64_t steps = 0;
  int rank = 0, nranks = 1;
  // padded exchange layout: rank q's rows [bounds[q], bounds[q+1]) keep their
  // contributions at x_full[q * chunk + (row - bounds[q])], so one equal-size
  // all-gather writes every slice in place (tcol is remapped to it)
  std::vector<int64_t> bounds;
  int64_t chunk = 1;
  DevArray<int64_t> dbounds;
};

// BFS workspaces (bfs.cu).
// Row-sharded single-source BFS (bfs.cu, multi-GPU driver): this rank owns
// vertices [rb, re) (32-aligned), pulls them against the global frontier
// bitmap each level and contributes its slice of the next bitmap.
struct BfsShard {
  int rank = 0, nranks = 1;
  int64_t rb = 0, re = 0;
  int32_t source = 0;
  int d = 0;             // levels done
  int ucnt = -1;         // owned still-unvisited list (-1: every owned vertex)
  int ul = 0;            // parity of the list being read
  DevArray<int> cnt;     // [0] found [1] next list size
};

struct BfsWork {
  int64_t n = 0;
  std::unique_ptr<BfsShard> shard;
  DevArray<int32_t> level, parent;          // single source
  DevArray<int32_t> queue[2];
  DevArray<uint32_t> bitmap[3];             // frontier bitmaps: read, write, clear per level
  DevArray<int32_t> ulist[2];               // unvisited vertices for pull levels
  DevArray<int> ctl;
  // multi-source (64 lanes)
  DevArray<unsigned long long> seen, front, next, third;  // seen + a ring of 3 frontiers
  DevArray<int32_t> mlevel, mparent;        // [n][64] vertex-major
  int64_t ms_ns = 0;
  DevArray<int32_t> mqueue[2];
  DevArray<int> mctl;
  DevArray<int32_t> msrc;                   // batch lanes + distinct sources
  DevArray<unsigned long long> tlog;
  // pull-mode hubs (in-degree > kBfsHeavy) handled warp-per-vertex
  DevArray<int32_t> heavy, heavy1;          // the 64-lane batch's hubs / the single source's
  DevArray<int> heavy_cnt;
  int64_t nheavy = 0, nheavy1 = 0;
  DevArray<int32_t> unz;                    // vertices with in-edges, ascending (first pull)
  int64_t nunz = 0;
  const void* heavy_key = nullptr;
  int64_t heavy_nnz = -1;
};

// Triangle counting plan (tc.cu): degree-ordered upper triangle U, its
// transpose as tails into U, and the per-middle-vertex work items.
struct TcPlan {
  int64_t n = 0, nnz = 0;
  DevArray<int64_t> urp;
  DevArray<int32_t> ucol;
  DevArray<int64_t> lrp;     // L = U' by middle vertex j
  DevArray<int2> tails;      // [p + 1, urp[i + 1]) for L entry (i, p)
  DevArray<int64_t> items;   // j << 32 | chunk of <= kTcItem in-neighbours
  DevArray<int64_t> item_off;  // [n + 1]: first item of each j
  int64_t nitems = 0;
  std::vector<int32_t> heavy_h, huge_h;  // middle vertices with long U(j)
  std::vector<int64_t> heavy_item_off_h;  // [heavy + 1]: first CTA item of each
  DevArray<int64_t> heavy_items;          // j << 32 | chunk (CTA kernel)
  DevArray<int32_t> huge;
  DevArray<unsigned long long> count;
  DevArray<unsigned> next_row;
};

// One SSSP traversal's workspace (sssp.cu): distances, near / far queues,
// membership bits, circular buckets, control words.  Lane 0 runs on the
// graph's stream; a batch (gbx_sssp_batch) runs several lanes concurrently,
// each on its own stream with its share of the SMs.
struct SsspLane {
  DevArray<uint32_t> dist32;
  DevArray<unsigned long long> dist64;
  DevArray<int32_t> q[2], far[2], stamp;
  DevArray<int> ctl;
  DevArray<unsigned long long> lohi, relax;
  // circular buckets (bucketed variant)
  DevArray<int32_t> bq;
  DevArray<uint32_t> bbits;
  DevArray<int> bcnt;
  int nb_alloc = 0;
  DevArray<double> out;            // fp64 copy of the distances for the host
  cudaStream_t stream = nullptr;   // owned (lanes > 0)
  ~SsspLane() {
    if (stream) {
      cudaStreamSynchronize(stream);
      cudaStreamDestroy(stream);
    }
  }
};

// SSSP plan (sssp.cu): packed (col:24 | w:8) edges when exact, else split.
struct SsspPlan {
  int64_t n = 0, nnz = 0;
  bool packed = false;     // uint32 col<<8|w, n <= 2^24, integer w in [1,255]
  bool integral = false;   // integer weights: uint32 distances
  bool nonpositive = false; // some weight <= 0 (NonPositiveWeight on every call)
  double max_w = 0;
  DevArray<uint32_t> packed_edges;
  DevArray<int32_t> wint;
  DevArray<double> wdbl;
  // light-first row partition for delta = split_delta (sssp.cu: k_split_*)
  double split_delta = -1.0;
  DevArray<int32_t> nlight, split_col, split_wi;
  DevArray<double> split_wd;
  // per-vertex edge ranges {begin, light end, end, 0} (nnz < 2^32): one 16-byte
  // load per popped vertex instead of row_ptr[u], row_ptr[u+1] and nlight[u]
  DevArray<uint4> vmeta;
  // heavy in-edges (w > split_delta) of every vertex, packed (u:24 | w:8) and
  // ascending in w within a row: the pull form of a bucket's heavy pass
  // (packed plans only; empty when nnz >= 2^32)
  DevArray<uint32_t> hin_rp, hin;
  std::vector<std::unique_ptr<SsspLane>> lanes;  // [0]: the single-source call's
};

// Row-partitioned batched Brandes (bc.cu, sharded protocol): this rank owns
// vertices [rb, re) -- it settles their path counts (forward pull) and their
// dependencies (backward) -- while level / sigma / coef stay replicated and are
// refreshed from the other ranks' records after every level.
struct BcShard {
  int rank = 0, nranks = 1, ns = 0;
  int64_t rb = 0, re = 0;
  std::vector<int64_t> off;      // global order offsets per depth
  int cur = 0;                   // forward map parity
  int ucnt = -1;                 // owned still-unreached list (-1: first pull)
  unsigned live = 0;
  bool fwd_done = false;
  int bd = -1;                   // next backward depth (-1: not started)
  DevArray<int32_t> ownbin;      // owned vertices binned by in-degree
  DevArray<int> owncnt;
  DevArray<int32_t> snew;        // owned vertices of the level at hand
  DevArray<int32_t> slist;       // its binned copy
  DevArray<int> scnt;
  DevArray<unsigned char> recs;  // packed 40-byte records
  DevArray<int64_t> hent_t, hent_a;  // chunks of the owned hub rows
  int nhent_t = 0, nhent_a = 0;
  // candidate levels (small frontiers): marked owned candidates, their binned
  // copy, the pull's survivor scratch, the frontier lists of the mark pass
  DevArray<int32_t> clist, cbin, cscr, flight, fheavy;
  DevArray<int> ccnt;
};

// Betweenness workspaces (bc.cu).
struct BcHubs {                // rows longer than kBcHeavy, split into chunks
  DevArray<int32_t> hv;        // slot -> vertex
  DevArray<int64_t> hent;      // chunk << 32 | slot
  DevArray<double> hacc;       // [slot][4] partial sums, zero between uses
  int nhv = 0, nhent = 0;
  const void* key = nullptr;
  int64_t nnz = -1;
};

struct BcWork {
  int64_t n = 0;
  int lanes = 0;
  DevArray<int32_t> level;   // [n][lanes]
  DevArray<uint32_t> lv8;    // [n]: byte per lane, min(depth, 254), 0xFF unreached
  DevArray<double> sigma;    // [n][lanes]
  DevArray<double> delta;    // [n][lanes]: (1 + delta) / sigma once final
  DevArray<int32_t> order;   // vertices by level (union over lanes)
  DevArray<int32_t> mark, ulist[2], src;
  DevArray<int64_t> ent[2];
  DevArray<uint32_t> map[2];  // level maps: 4 bits (lanes) per vertex
  // row-length binning (stable 2-bit radix partition of a vertex list)
  DevArray<int32_t> border;   // level lists binned by out-degree
  DevArray<int32_t> allbin;   // every vertex binned by in-degree (first pull)
  DevArray<int32_t> iota;
  DevArray<uint8_t> bkeys[2];
  DevArray<uint8_t> btemp;
  DevArray<int> ucnt, allcnt, lcnt;
  const void* allbin_key = nullptr;
  int64_t allbin_nnz = -1;
  DevArray<double> cent;
  DevArray<int> ctl;
  BcHubs hub_a, hub_t;       // hub rows of A (backward) and AT (forward pull)
  // degree-sorted copy of the graph (bc_run on large graphs): vertices
  // relabeled by descending degree, rows ascending in the new ids.  A BFS
  // depth is then (nearly) a contiguous id range: the sigma / coef sectors a
  // depth's edges gather are dense in L2 instead of one per 128-byte line, and
  // the rows of a degree bin are adjacent in memory.
  Csr ra, rat;               // relabeled A and AT (undirected: rat only, ra unused)
  DevArray<int32_t> new2old, old2new;
  DevArray<double> cent_new; // centrality in the new ids (cent: original ids)
  DevArray<double> bacc;     // [n][4] sums of the backward push form (zero between uses)
  const void* relabel_key = nullptr;
  int64_t relabel_nnz = -1;
  int64_t relabel_nz = 0;    // vertices with edges (ids [0, relabel_nz) of the copy)
  std::unique_ptr<BcShard> shard;
};

struct CcWork {
  int64_t n = 0;
  DevArray<int32_t> parent;
  DevArray<int> ctl;
};

}  // namespace gbx
