// gbx_gblite.hpp -- header-only C++ adapter: the reference's gblite API
// (include/gblite/graph.hpp, include/gblite/algorithms.hpp) served by libgbx.so.
//
// A gblite user switches by including this header and calling
// gblite::b200::algo::X where they called gblite::algo::X (same arguments, same
// result types, same gblite::Error codes).  `DeviceGraph` keeps the adjacency
// and the caches resident in HBM across calls; the free functions build a
// transient DeviceGraph from a gblite::Graph, mirroring the caches it holds
// (advanced mode: absent caches raise MissingProperty exactly like the
// reference, algorithms.hpp:14-17).
#pragma once

#include <cmath>
#include <cstdint>
#include <limits>
#include <span>
#include <string>
#include <vector>

#include "gblite/algorithms.hpp"
#include "gblite/graph.hpp"
#include "gbx.h"

namespace gblite::b200 {

inline void check(int rc, const char* msg) {
  if (rc < 0) {
    // gbx codes <= -30 (device failures) have no gblite counterpart
    const ErrCode code = rc <= -30 ? ErrCode::InvalidValue : static_cast<ErrCode>(rc);
    fail(code, std::string("gbx: ") + msg);
  }
}

// The adjacency + caches of a gblite::Graph, resident on the device.
class DeviceGraph {
 public:
  explicit DeviceGraph(const Graph& g) {
    const SparseMatrix& A = g.A;
    const Index n = A.nrows();
    std::vector<int64_t> rp(A.row_ptr().begin(), A.row_ptr().end());
    std::vector<int64_t> col(A.col_idx().begin(), A.col_idx().end());
    std::vector<double> w;
    const void* vals = nullptr;
    int domain = GBX_BOOL;
    if (A.domain() == Domain::Fp64) {
      w.reserve(A.nvals());
      for (const Scalar& s : A.values()) w.push_back(as_fp64(s));
      vals = w.data();
      domain = GBX_FP64;
    }
    char msg[GBX_MSG_LEN];
    check(gbx_graph_new(&h_, static_cast<int64_t>(n), rp.data(), col.data(), vals, domain,
                        g.kind == Kind::UndirectedAdjacency ? GBX_UNDIRECTED : GBX_DIRECTED,
                        msg),
          msg);
    if (g.AT) check(gbx_property_at(h_, msg), msg);
    if (g.row_degree) check(gbx_property_rowdegree(h_, msg), msg);
    if (g.col_degree) check(gbx_property_coldegree(h_, msg), msg);
    if (g.pattern_is_symmetric != TriState::Unknown)
      check(gbx_property_symmetric_pattern(h_, msg), msg);
    if (g.ndiag != -1) check(gbx_property_ndiag(h_, msg), msg);
    n_ = n;
  }
  ~DeviceGraph() {
    char msg[GBX_MSG_LEN];
    if (h_) gbx_graph_free(&h_, msg);
  }
  DeviceGraph(const DeviceGraph&) = delete;
  DeviceGraph& operator=(const DeviceGraph&) = delete;
  gbx_graph* get() const { return h_; }
  Index n() const { return n_; }

 private:
  gbx_graph* h_ = nullptr;
  Index n_ = 0;
};

namespace detail {
inline SparseVector sparse_from_dense(const std::vector<int64_t>& d, Index n) {
  SparseVector v(n, Domain::Uint64);
  std::vector<Index> idx;
  std::vector<Scalar> vals;
  for (Index i = 0; i < n; ++i)
    if (d[i] >= 0) {
      idx.push_back(i);
      vals.emplace_back(static_cast<std::uint64_t>(d[i]));
    }
  v.adopt(std::move(idx), std::move(vals));
  return v;
}
}  // namespace detail

namespace algo {

// algo::bfs_direction_optimizing (algorithms.hpp:35-37)
inline gblite::algo::BfsResult bfs_direction_optimizing(
    const Graph& g, Index source, const gblite::algo::BfsConfig& config = {}) {
  DeviceGraph d(g);
  std::vector<int64_t> parent(d.n()), level(config.want_level ? d.n() : 0);
  char msg[GBX_MSG_LEN];
  check(gbx_bfs(parent.data(), config.want_level ? level.data() : nullptr, d.get(), source,
                static_cast<int>(config.direction), config.push_divisor, msg),
        msg);
  gblite::algo::BfsResult r;
  r.parent = detail::sparse_from_dense(parent, d.n());
  if (config.want_level) r.level = detail::sparse_from_dense(level, d.n());
  return r;
}

// algo::bfs_push (algorithms.hpp:25)
inline gblite::algo::BfsResult bfs_push(const Graph& g, Index source, bool want_level = false) {
  DeviceGraph d(g);
  std::vector<int64_t> parent(d.n()), level(want_level ? d.n() : 0);
  char msg[GBX_MSG_LEN];
  check(gbx_bfs_push(parent.data(), want_level ? level.data() : nullptr, d.get(), source, msg),
        msg);
  gblite::algo::BfsResult r;
  r.parent = detail::sparse_from_dense(parent, d.n());
  if (want_level) r.level = detail::sparse_from_dense(level, d.n());
  return r;
}

// algo::pagerank_gap (algorithms.hpp:52-55)
inline gblite::algo::PageRankResult pagerank_gap(const Graph& g, double damping = 0.85,
                                                 double tol = 1e-4, int itermax = 100) {
  DeviceGraph d(g);
  gblite::algo::PageRankResult r;
  r.rank.assign(d.n(), 0.0);
  char msg[GBX_MSG_LEN];
  check(gbx_pagerank(r.rank.data(), &r.iterations, d.get(), damping, tol, itermax, msg), msg);
  return r;
}

// algo::triangle_count (algorithms.hpp:76)
inline std::uint64_t triangle_count(const Graph& g,
                                    const gblite::algo::TriangleCountConfig& config = {}) {
  DeviceGraph d(g);
  std::uint64_t c = 0;
  char msg[GBX_MSG_LEN];
  check(gbx_triangle_count(&c, d.get(), static_cast<int>(config.presort), config.sample_seed,
                           msg),
        msg);
  return c;
}

// algo::sssp_delta_stepping (algorithms.hpp:61)
inline gblite::algo::SsspResult sssp_delta_stepping(const Graph& g, Index source, double delta) {
  DeviceGraph d(g);
  std::vector<double> dist(d.n());
  char msg[GBX_MSG_LEN];
  check(gbx_sssp(dist.data(), d.get(), source, delta, msg), msg);
  gblite::algo::SsspResult r;
  r.dist = SparseVector(d.n(), Domain::Fp64);
  std::vector<Index> idx;
  std::vector<Scalar> vals;
  for (Index i = 0; i < d.n(); ++i)
    if (dist[i] < std::numeric_limits<double>::infinity()) {
      idx.push_back(i);
      vals.emplace_back(dist[i]);
    }
  r.dist.adopt(std::move(idx), std::move(vals));
  return r;
}

// algo::betweenness_centrality (algorithms.hpp:44-45)
inline gblite::algo::CentralityResult betweenness_centrality(const Graph& g,
                                                             std::span<const Index> sources) {
  DeviceGraph d(g);
  gblite::algo::CentralityResult r;
  r.centrality.assign(d.n(), 0.0);
  std::vector<std::uint64_t> s(sources.begin(), sources.end());
  char msg[GBX_MSG_LEN];
  check(gbx_betweenness(r.centrality.data(), d.get(), s.data(), s.size(), msg), msg);
  return r;
}

// algo::connected_components_fastsv (algorithms.hpp:84-85)
inline gblite::algo::ComponentResult connected_components_fastsv(const Graph& g) {
  DeviceGraph d(g);
  std::vector<int64_t> lab(d.n());
  gblite::algo::ComponentResult r;
  char msg[GBX_MSG_LEN];
  check(gbx_connected_components(lab.data(), &r.iterations, d.get(), msg), msg);
  r.label.assign(lab.begin(), lab.end());
  return r;
}

}  // namespace algo
}  // namespace gblite::b200
