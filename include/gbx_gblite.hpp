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
#include <cstring>
#include <memory>
#include <limits>
#include <span>
#include <string>
#include <vector>

#include "gblite/algorithms.hpp"
#include "gblite/core.hpp"
#include "gblite/graph.hpp"
#include "gbx.h"

namespace gblite::b200 {

// Device / runtime failures (gbx codes <= -30: CUDA errors, out of device
// memory, unsupported sizes, NULL arguments, NCCL failures) have no gblite
// ErrCode.  They are thrown as DeviceError: a gblite::Error (so a caller that
// catches gblite::Error still catches it; its code() is InvalidValue) that
// also carries the gbx code -- distinct from every argument error the
// reference itself raises.
class DeviceError : public Error {
 public:
  DeviceError(int gbx_code, const std::string& message)
      : Error(ErrCode::InvalidValue, "device failure " + std::to_string(gbx_code) + ": " + message),
        gbx_code_(gbx_code) {}
  int gbx_code() const noexcept { return gbx_code_; }

 private:
  int gbx_code_;
};

inline void check(int rc, const char* msg) {
  if (rc <= -30) throw DeviceError(rc, std::string("gbx: ") + msg);
  if (rc < 0) fail(static_cast<ErrCode>(rc), std::string("gbx: ") + msg);
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


// ---- the GraphBLAS operation layer (core.hpp:100-120) on the device ----------
// gblite::b200::mxm / vxm / mxv take the reference's own containers, Descriptor
// and Semiring (one of the built-ins of ops.cpp:362-372, recognised by name and
// domain) and leave the same result in the output container, bit for bit.
namespace detail {

struct HostCsr {
  std::vector<int64_t> rp, col;
  std::vector<unsigned char> vals;  // bool: 1 byte, others 8
};

inline int dom_id(Domain d) { return static_cast<int>(d); }

inline void put_scalar(const Scalar& s, Domain d, std::vector<unsigned char>& out) {
  if (d == Domain::Bool) {
    out.push_back(as_bool(s) ? 1 : 0);
    return;
  }
  unsigned char b[8];
  if (d == Domain::Int64) { const std::int64_t v = as_int64(s); std::memcpy(b, &v, 8); }
  else if (d == Domain::Uint64) { const std::uint64_t v = as_uint64(s); std::memcpy(b, &v, 8); }
  else { const double v = as_fp64(s); std::memcpy(b, &v, 8); }
  out.insert(out.end(), b, b + 8);
}

inline Scalar get_scalar(const unsigned char* p, Domain d) {
  if (d == Domain::Bool) return *p != 0;
  if (d == Domain::Int64) { std::int64_t v; std::memcpy(&v, p, 8); return v; }
  if (d == Domain::Uint64) { std::uint64_t v; std::memcpy(&v, p, 8); return v; }
  double v;
  std::memcpy(&v, p, 8);
  return v;
}

inline std::size_t esize(Domain d) { return d == Domain::Bool ? 1 : 8; }

class Mat {
 public:
  explicit Mat(const SparseMatrix& A) {
    std::vector<int64_t> rp(A.row_ptr().begin(), A.row_ptr().end());
    std::vector<int64_t> col(A.col_idx().begin(), A.col_idx().end());
    std::vector<unsigned char> v;
    v.reserve(A.nvals() * esize(A.domain()));
    for (const Scalar& x : A.values()) put_scalar(x, A.domain(), v);
    char msg[GBX_MSG_LEN];
    check(gbx_mat_new(&h_, static_cast<int64_t>(A.nrows()), static_cast<int64_t>(A.ncols()),
                      rp.data(), col.data(), v.data(), dom_id(A.domain()), msg),
          msg);
  }
  explicit Mat(gbx_mat* h) : h_(h) {}
  ~Mat() {
    char msg[GBX_MSG_LEN];
    if (h_) gbx_mat_free(&h_, msg);
  }
  Mat(const Mat&) = delete;
  Mat& operator=(const Mat&) = delete;
  gbx_mat* get() const { return h_; }
  void to(SparseMatrix& C) const {
    int64_t nr = 0, nc = 0, nv = 0;
    int d = 0;
    char msg[GBX_MSG_LEN];
    check(gbx_mat_info(h_, &nr, &nc, &nv, &d, msg), msg);
    const Domain dom = static_cast<Domain>(d);
    std::vector<int64_t> rp(nr + 1), col(nv);
    std::vector<unsigned char> v(nv * esize(dom) + 8);
    check(gbx_mat_export(h_, rp.data(), col.data(), v.data(), msg), msg);
    std::vector<Index> r(rp.begin(), rp.end()), c(col.begin(), col.end());
    std::vector<Scalar> vals;
    vals.reserve(nv);
    for (int64_t p = 0; p < nv; ++p) vals.push_back(get_scalar(v.data() + p * esize(dom), dom));
    SparseMatrix out(static_cast<Index>(nr), static_cast<Index>(nc), dom);
    out.adopt(std::move(r), std::move(c), std::move(vals));
    C = std::move(out);
  }

 private:
  gbx_mat* h_ = nullptr;
};

struct Vec {
  std::vector<int64_t> idx;
  std::vector<unsigned char> vals;
  gbx_vec v{};
  explicit Vec(const SparseVector& w) {
    idx.assign(w.indices().begin(), w.indices().end());
    for (const Scalar& x : w.values()) put_scalar(x, w.domain(), vals);
    v.n = static_cast<int64_t>(w.size());
    v.nvals = static_cast<int64_t>(w.nvals());
    v.idx = idx.data();
    v.vals = vals.data();
    v.domain = dom_id(w.domain());
  }
};

inline int semiring_id(const Semiring& s) {
  static const char* names[] = {"plus-times", "any-secondi", "min-plus", "plus-first",
                                "plus-second", "plus-pair", "min-second"};
  for (int i = 0; i < 7; ++i)
    if (s.name == names[i]) return i;
  fail(ErrCode::InvalidValue, "semiring '" + s.name + "' is not one of the device built-ins");
}

inline int op_id(const BinaryOp& op) {
  static const char* names[] = {"plus", "minus", "times", "div",  "min",  "max",
                                "first", "second", "pair", "any", "lor", "land"};
  for (int i = 0; i < 12; ++i)
    if (op.name == names[i]) return i + 1;
  fail(ErrCode::InvalidValue, "accumulator '" + op.name + "' is not a device operator");
}

struct Desc {
  gbx_desc d{};
  std::unique_ptr<Vec> mv;
  std::unique_ptr<Mat> mm;
  explicit Desc(const Descriptor& desc) {
    if (desc.mask.vector) {
      mv = std::make_unique<Vec>(*desc.mask.vector);
      d.mask_vec = &mv->v;
    }
    if (desc.mask.matrix) {
      mm = std::make_unique<Mat>(*desc.mask.matrix);
      d.mask_mat = mm->get();
    }
    d.complement = desc.mask.complement;
    d.structural = desc.mask.structural;
    d.replace = desc.mask.replace;
    if (desc.accum) {
      d.accum = op_id(*desc.accum);
      d.accum_domain = dom_id(desc.accum->out);
    }
    d.transpose_in1 = desc.transpose_in1;
    d.transpose_in2 = desc.transpose_in2;
  }
};

inline void vec_result(SparseVector& w, const std::vector<int64_t>& oi,
                       const std::vector<unsigned char>& ov, int64_t nv) {
  std::vector<Index> idx(oi.begin(), oi.begin() + nv);
  std::vector<Scalar> vals;
  vals.reserve(nv);
  for (int64_t p = 0; p < nv; ++p) vals.push_back(get_scalar(ov.data() + p * esize(w.domain()), w.domain()));
  w.adopt(std::move(idx), std::move(vals));
}

}  // namespace detail

// mxm (core.hpp:105-107, core.cpp:267-306)
inline void mxm(SparseMatrix& C, const Descriptor& desc, const Semiring& semiring,
                const SparseMatrix& A, const SparseMatrix& B) {
  if (&C == &A || &C == &B || desc.mask.matrix == &C)
    fail(ErrCode::AliasedOutput, "output container aliases an input");
  detail::Mat a(A), b(B), c(C);
  detail::Desc d(desc);
  gbx_mat* out = nullptr;
  char msg[GBX_MSG_LEN];
  check(gbx_mxm(&out, c.get(), &d.d, detail::semiring_id(semiring),
                detail::dom_id(semiring.add.op.out), a.get(), b.get(), msg),
        msg);
  detail::Mat(out).to(C);
}

// vxm (core.hpp:110-112, core.cpp:308-338)
inline void vxm(SparseVector& w, const Descriptor& desc, const Semiring& semiring,
                const SparseVector& u, const SparseMatrix& A) {
  if (&w == &u || desc.mask.vector == &w)
    fail(ErrCode::AliasedOutput, "output container aliases an input");
  detail::Mat a(A);
  detail::Vec uv(u), wv(w);
  detail::Desc d(desc);
  std::vector<int64_t> oi(w.size() + 1);
  std::vector<unsigned char> ov((w.size() + 1) * 8);
  int64_t nv = 0;
  char msg[GBX_MSG_LEN];
  check(gbx_vxm(oi.data(), ov.data(), &nv, &wv.v, &d.d, detail::semiring_id(semiring),
                detail::dom_id(semiring.add.op.out), &uv.v, a.get(), msg),
        msg);
  detail::vec_result(w, oi, ov, nv);
}

// mxv (core.hpp:114-116, core.cpp:340-386)
inline void mxv(SparseVector& w, const Descriptor& desc, const Semiring& semiring,
                const SparseMatrix& A, const SparseVector& u) {
  if (&w == &u || desc.mask.vector == &w)
    fail(ErrCode::AliasedOutput, "output container aliases an input");
  detail::Mat a(A);
  detail::Vec uv(u), wv(w);
  detail::Desc d(desc);
  std::vector<int64_t> oi(w.size() + 1);
  std::vector<unsigned char> ov((w.size() + 1) * 8);
  int64_t nv = 0;
  char msg[GBX_MSG_LEN];
  check(gbx_mxv(oi.data(), ov.data(), &nv, &wv.v, &d.d, detail::semiring_id(semiring),
                detail::dom_id(semiring.add.op.out), a.get(), &uv.v, msg),
        msg);
  detail::vec_result(w, oi, ov, nv);
}

// ---- io (io.hpp): files straight into HBM -------------------------------------
namespace io {

// read_matrix_file (io.cpp:336-343) + graph_new: a resident DeviceGraph-style
// handle; release with gbx_graph_free
inline gbx_graph* read_graph_file(const std::string& path, const std::string& format, Kind kind) {
  gbx_graph* g = nullptr;
  char msg[GBX_MSG_LEN];
  check(gbx_graph_read(&g, path.c_str(), format.c_str(),
                       kind == Kind::UndirectedAdjacency ? GBX_UNDIRECTED : GBX_DIRECTED, msg),
        msg);
  return g;
}

// write_matrix_file (io.cpp:345-355) of a resident graph (byte-identical output)
inline void write_graph_file(const gbx_graph* g, const std::string& path, const std::string& format,
                             bool symmetric = false) {
  char msg[GBX_MSG_LEN];
  check(gbx_graph_write(g, path.c_str(), format.c_str(), symmetric ? 1 : 0, msg), msg);
}

}  // namespace io

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
