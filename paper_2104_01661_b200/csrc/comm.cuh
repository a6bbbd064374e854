// comm.cuh -- communicator, collectives and the distributed graph of libgbx.so
// (comm.cu, dgraph.cu, mg.cu).
#pragma once

#include <memory>
#include <vector>

#include "common.cuh"

constexpr int kMaxRanks = 8;  // one NVSwitch node

// Communicator handle (include/gbx.h: gbx_comm_*): NCCL (one rank per process)
// or `nlocal` == nranks in-process ranks on one GPU.
struct gbx_comm {
  int nranks = 1;
  int rank = 0;      // NCCL: this process's rank; local: 0 (local rank l is rank l)
  int nlocal = 1;
  int device = 0;
  void* nccl = nullptr;  // ncclComm_t
  cudaStream_t stream = nullptr;
  std::mutex mu;
  int global_rank(int l) const { return nccl ? rank : l; }
  ~gbx_comm();
};

struct gbx_dgraph;

namespace gbx {

enum class CollType { U8, I32, U32, I64, U64, F64 };
enum class CollOp { Sum, Max, Min };

void comm_unique_id(void* id);
gbx_comm* comm_new_nccl(int nranks, int rank, const void* id, int device);
gbx_comm* comm_new_local(int nranks, int device);
void comm_sync(gbx_comm* c);
void comm_destroy_nccl(void* nc);

// all collectives take one buffer per LOCAL rank and are synchronous
// recv[l] = concat over ranks q of send[q] (bytes each)
void c_allgather(gbx_comm* c, const void* const* send, void* const* recv, size_t bytes);
// in place, every rank's buf[l] = op over ranks (fp64 sums in rank order in
// the local transport; NCCL's own order otherwise)
void c_allreduce(gbx_comm* c, void* const* buf, size_t count, CollType t, CollOp op);
// one host value per local rank -> the value of every rank (rank order)
std::vector<int64_t> c_allgather_host(gbx_comm* c, const std::vector<int64_t>& mine);
// cnt[l][q] = count local rank l sends to rank q -> out[l][q] = count l receives from q
std::vector<std::vector<int64_t>> c_exchange_counts(gbx_comm* c,
                                                    const std::vector<std::vector<int64_t>>& cnt);
// byte offsets [nlocal][nranks+1]
void c_alltoallv(gbx_comm* c, const void* const* send, const std::vector<std::vector<int64_t>>& soff,
                 void* const* recv, const std::vector<std::vector<int64_t>>& roff);

// Buffers every rank can address: local[l] (this process's), peer[l][q] = the
// address local rank l uses for rank q's buffer (IPC-mapped over NVLink with
// NCCL; the other local rank's buffer in the local transport).
struct PeerBuf {
  size_t bytes = 0;
  std::vector<void*> local;
  std::vector<std::vector<uint64_t>> peer;
  std::vector<void*> opened;  // IPC mappings to close
  void release();
  ~PeerBuf();
};
void peer_alloc(gbx_comm* c, size_t bytes, PeerBuf& b);

// PageRank exchange state of a distributed graph (mg.cu), kept between calls
struct PrMgState {
  int64_t chunk = 0;
  PeerBuf x0, x1, l1, sig;                   // fused exchange (peer stores)
  std::vector<DevArray<float>> r0, r1;       // [nlocal] local ranks, chunk each
  std::vector<DevArray<float>> xfull, xs;    // NCCL exchange: padded x, own slice
  bool p2p_failed = false;                   // the fused run fell back this call
  DevArray<int32_t> flag;                    // the ranks' agreement word
};

// (row << bits | col) keys of one local rank; drop keys (1 << 2*bits) sort last
struct KeyBlock {
  DevArray<uint64_t> k;
  int64_t m = 0;
};
void sort_in_place(cudaStream_t s, KeyBlock& K, int bits);
// SORTED keys of every local rank -> out[l] = the de-duplicated CSR block (n
// rows, only [bounds[q], bounds[q+1]) non-empty) of local rank l; keys released
void shuffle_to_blocks(gbx_comm* c, std::vector<KeyBlock>& keys, const std::vector<int64_t>& bounds,
                       int64_t n, int bits, std::vector<Csr*>& out);
gbx_dgraph* dgraph_generate_rmat(gbx_comm* c, int scale, int ef, double a, double b, double cc,
                                 uint64_t seed, int scramble, int kind);
gbx_dgraph* dgraph_from_blocks(gbx_comm* c, int64_t n, const int64_t* row_begin,
                               const int64_t* row_end, const int64_t* const* row_ptr,
                               const int32_t* const* col, int kind);
void dgraph_block(const gbx_dgraph* D, int l, int64_t* rb, int64_t* re);

// multi-GPU algorithms (mg.cu)
void pagerank_mg(gbx_dgraph* D, double damping, double tol, int itermax, int exchange,
                 double* rank, int* iters);
uint64_t triangle_count_mg(gbx_dgraph* D);
void bfs_mg(gbx_dgraph* D, uint64_t source, int64_t* parent, int64_t* level);
void betweenness_mg(gbx_dgraph* D, const uint64_t* sources, uint64_t ns, double* centrality);

}  // namespace gbx

// Distributed graph (include/gbx.h: gbx_dgraph_*): rank q owns the rows
// [bounds[q], bounds[q+1]) (32-aligned, balanced by rows + entries).  Each
// local rank's shard is a gbx_graph over ALL n vertices whose rows outside its
// block are empty (row_ptr is n+1 long, entries only for owned rows, global
// column ids): the single-GPU kernels run on it unchanged for owned rows, and
// no rank holds more than its block of A (and, for a directed graph, of AT).
struct gbx_dgraph {
  gbx_comm* comm = nullptr;
  int device = 0;
  int64_t n = 0;
  int64_t nnz = 0;  // global stored entries of A
  int kind = GBX_DIRECTED;
  std::vector<int64_t> bounds;     // [nranks + 1]
  std::vector<gbx_graph*> shard;   // [nlocal]
  std::vector<int64_t> local_nnz;  // [nlocal]
  std::unique_ptr<gbx::PrMgState> pr;  // PageRank exchange buffers (mg.cu)
  std::vector<int64_t> tc_bounds;      // triangle count: middle-vertex split (mg.cu)
  gbx_stats stats{};                   // the last multi-GPU call
  ~gbx_dgraph();
};
