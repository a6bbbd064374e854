// mg_nccl.cpp -- a C++ caller of the multi-GPU C ABI over the NCCL transport
// (1-rank communicator on the test GPU): every gbx_*_mg call against the
// oracle (oracle/oracle.h, the CPU restatement of the reference).  Built and
// run by tests/test_mg_cpp.py.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "gbx.h"
#include "../../oracle/oracle.h"

#define CHECK(x)                                                                   \
  do {                                                                             \
    char msg_[GBX_MSG_LEN];                                                        \
    int rc_ = (x);                                                                 \
    (void)msg_;                                                                    \
    if (rc_ < 0) {                                                                 \
      std::fprintf(stderr, "%s:%d: %s -> %d\n", __FILE__, __LINE__, #x, rc_);     \
      std::exit(1);                                                                \
    }                                                                              \
  } while (0)

static char msg[GBX_MSG_LEN];

static void require(bool ok, const char* what) {
  if (!ok) {
    std::fprintf(stderr, "FAILED: %s\n", what);
    std::exit(1);
  }
}

// the oracle's CSR of the seeded R-MAT graph (the generator both sides share)
static void oracle_graph(int scale, int ef, uint64_t seed, int sym, std::vector<int64_t>& rp,
                         std::vector<int32_t>& col) {
  const int64_t n = int64_t(1) << scale, m = int64_t(ef) << scale;
  std::vector<uint32_t> u(m), v(m);
  orc_rmat_edges(scale, ef, 0.57, 0.19, 0.19, seed, 1, u.data(), v.data());
  rp.assign(n + 1, 0);
  col.assign(sym ? 2 * m : m, 0);
  const int64_t nnz = orc_build_csr(n, m, u.data(), v.data(), nullptr, sym, rp.data(), col.data(), nullptr);
  col.resize(nnz);
}

int main() {
  CHECK(gbx_init(0, msg));
  unsigned char id[GBX_COMM_ID_BYTES];
  CHECK(gbx_comm_unique_id(id, msg));
  gbx_comm* comm = nullptr;
  CHECK(gbx_comm_init(&comm, 1, 0, id, 0, msg));
  const int scale = 12;
  const int64_t n = int64_t(1) << scale;

  // ---- directed: the distributed build equals the oracle's CSR; PageRank
  std::vector<int64_t> rp;
  std::vector<int32_t> col;
  oracle_graph(scale, 16, 1, 0, rp, col);
  gbx_dgraph* dg = nullptr;
  CHECK(gbx_dgraph_generate_rmat(&dg, comm, scale, 16, 0.57, 0.19, 0.19, 1, 1, GBX_DIRECTED, msg));
  {
    int64_t rb, re, nnz;
    CHECK(gbx_dgraph_block(dg, 0, &rb, &re, &nnz, msg));
    require(rb == 0 && re == n && nnz == static_cast<int64_t>(col.size()), "block shape");
    std::vector<int64_t> brp(n + 1);
    std::vector<int32_t> bcol(nnz);
    CHECK(gbx_dgraph_export_block(dg, 0, brp.data(), bcol.data(), msg));
    require(brp == rp && bcol == col, "distributed build == oracle CSR");
  }
  {
    std::vector<int64_t> trp(n + 1), odeg(n);
    std::vector<int32_t> tcol(col.size());
    orc_transpose(n, rp.data(), col.data(), nullptr, trp.data(), tcol.data(), nullptr);
    for (int64_t i = 0; i < n; ++i) odeg[i] = rp[i + 1] - rp[i];
    std::vector<double> want(n);
    int wit = 0;
    orc_pagerank(n, trp.data(), tcol.data(), odeg.data(), 0.85, 1e-4, 100, want.data(), &wit, nullptr);
    for (int ex : {GBX_MG_P2P, GBX_MG_NCCL, GBX_MG_AUTO}) {
      std::vector<double> got(n);
      int it = 0;
      CHECK(gbx_pagerank_mg(got.data(), &it, dg, 0.85, 1e-4, 100, ex, msg));
      double num = 0, den = 0;
      for (int64_t i = 0; i < n; ++i) {
        num += std::fabs(got[i] - want[i]);
        den += std::fabs(want[i]);
      }
      require(it == wit, "pagerank iterations == oracle");
      require(num <= 1e-4 * den, "pagerank rel L1 <= 1e-4");
    }
  }
  CHECK(gbx_dgraph_free(&dg, msg));

  // ---- undirected: triangle count, BFS, betweenness
  oracle_graph(scale, 16, 1, 1, rp, col);
  CHECK(gbx_dgraph_generate_rmat(&dg, comm, scale, 16, 0.57, 0.19, 0.19, 1, 1, GBX_UNDIRECTED, msg));
  uint64_t tc = 0;
  CHECK(gbx_triangle_count_mg(&tc, dg, msg));
  require(tc == orc_triangle_count(n, rp.data(), col.data()), "triangle count == oracle");
  int64_t src = 0;
  for (int64_t i = 0; i < n; ++i)
    if (rp[i + 1] - rp[i] > rp[src + 1] - rp[src]) src = i;
  {
    std::vector<int64_t> par(n), lev(n), wp(n), wl(n);
    CHECK(gbx_bfs_mg(par.data(), lev.data(), dg, static_cast<uint64_t>(src), msg));
    orc_bfs(n, rp.data(), col.data(), src, wp.data(), wl.data());
    require(par == wp && lev == wl, "bfs parents / levels == oracle");
  }
  {
    const uint64_t srcs[3] = {static_cast<uint64_t>(src), 1, 2};
    const int64_t isrcs[3] = {src, 1, 2};
    std::vector<double> got(n), want(n);
    CHECK(gbx_betweenness_mg(got.data(), dg, srcs, 3, msg));
    orc_bc(n, rp.data(), col.data(), rp.data(), col.data(), isrcs, 3, want.data());
    double num = 0, den = 0;
    for (int64_t i = 0; i < n; ++i) {
      num += std::fabs(got[i] - want[i]);
      den += std::fabs(want[i]);
    }
    require(num <= 1e-9 * (den > 0 ? den : 1), "betweenness rel L1 <= 1e-9");
  }
  CHECK(gbx_dgraph_free(&dg, msg));
  CHECK(gbx_comm_free(&comm, msg));
  std::printf("mg nccl ok: pagerank, triangle count %llu, bfs, betweenness\n",
              static_cast<unsigned long long>(tc));
  return 0;
}
