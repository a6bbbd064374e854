// plans.cuh -- per-algorithm device layouts and workspaces owned by a gbx_graph.
#pragma once

#include "common.cuh"

namespace gbx {

// PageRank pull plan over AT (pagerank.cu): merge-path tiles of
// kPrItems (row-ends + nonzeros) each, and the rows that straddle tiles.
struct PrPlan {
  int64_t n = 0, nnz = 0, row0 = 0, row1 = 0;  // rows [row0,row1) of AT
  int64_t ntiles = 0, nsplit = 0;
  int grid = 0;
  DevArray<int64_t> tile_row, tile_nz;      // [ntiles+1] merge-path coordinates
  DevArray<int32_t> head_split, tail_split; // [ntiles] split id or -1
  DevArray<int32_t> split_first, split_parts;
  DevArray<int64_t> split_row, split_slot;
  DevArray<double> split_part;
  DevArray<unsigned> split_cnt;
  DevArray<float> r[2], x[2];      // fp32 storage (tol >= 1e-6)
  DevArray<double> rd[2], xd[2];    // fp64 storage (tight tolerances)
  DevArray<double> l1_block, l1_hist;
  DevArray<int> ctl;            // [0] completed iterations, [1] done
  DevArray<unsigned> blk_cnt;
  // CUDA graph with a conditional WHILE node (one iteration kernel per trip)
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  double g_damping = -1, g_tol = -1;
  int g_itermax = -1;
  int g_prec = 0;
  int last_prec = 32;
  bool graph_failed = false;
  int last_iters = 0;
  ~PrPlan();
};

// Sharded PageRank step (multi-GPU driver): a PrPlan over a row block.
struct PrShard {
  PrPlan plan;
  int64_t steps = 0;
};

// BFS workspaces (bfs.cu).
struct BfsWork {
  int64_t n = 0;
  DevArray<int32_t> level, parent;          // single source
  DevArray<int32_t> queue[2];
  DevArray<uint32_t> bitmap[2];
  DevArray<int> ctl;
  // multi-source (64 lanes)
  DevArray<unsigned long long> seen, front, next;
  DevArray<int32_t> mlevel, mparent;        // [n][64] vertex-major
  int64_t ms_ns = 0;
  DevArray<int32_t> mqueue[2];
  DevArray<int> mctl;
};

// Triangle counting plan (tc.cu): degree-ordered upper triangle U.
struct TcPlan {
  int64_t n = 0, nnz = 0;
  DevArray<int64_t> urp;
  DevArray<int32_t> ucol;
  DevArray<int32_t> order;   // rows with >= 2 entries, heaviest first
  DevArray<int64_t> work;    // prefix of per-row wedge work (ordered rows)
  int64_t nrows_active = 0;
  DevArray<unsigned long long> count;
  DevArray<unsigned> next_row;
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
  DevArray<uint32_t> dist32;
  DevArray<unsigned long long> dist64;
  DevArray<int32_t> q[2], far[2], stamp;
  DevArray<int> ctl;
  DevArray<unsigned long long> lohi, relax;
};

// Betweenness workspaces (bc.cu).
struct BcWork {
  int64_t n = 0;
  int lanes = 0;
  DevArray<int32_t> level;   // [n][lanes]
  DevArray<double> sigma;    // [n][lanes]
  DevArray<double> delta;    // [n][lanes]
  DevArray<int32_t> order;   // vertices by level (union over lanes)
  DevArray<double> cent;
  DevArray<int> ctl;
};

struct CcWork {
  int64_t n = 0;
  DevArray<int32_t> parent;
  DevArray<int> ctl;
};

}  // namespace gbx
