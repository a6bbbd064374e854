// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" adapter over the UNMODIFIED reference library (gblite sources under
// /root/reference/proj/src, compiled by oracle/Makefile into oracle/_ref/).  It
// lets the Python test suite, oracle/make_golden.py and bench.py's reference arm
// call the reference's own public API (gblite::graph_new, property_*,
// algo::*) on CSR arrays.  Nothing here re-implements reference behaviour: every
// entry point converts arrays -> gblite containers, calls the reference, and
// converts the result back.  Error codes are gblite::ErrCode values
// (error.hpp:13-41).
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <limits>
#include <optional>
#include <string>
#include <vector>

#include "gblite/gblite.hpp"
#include "gblite/verify.hpp"

using namespace gblite;

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return 0;
  } catch (const Error& e) {
    g_last_error = e.what();
    return static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return -100;
  }
}

SparseMatrix csr_to_matrix(int64_t nrows, int64_t ncols, const int64_t* rp,
                           const int32_t* col, const double* w) {
  SparseMatrix m(nrows, ncols, w ? Domain::Fp64 : Domain::Bool);
  int64_t nnz = rp[nrows];
  std::vector<Index> row_ptr(rp, rp + nrows + 1);
  std::vector<Index> cols(col, col + nnz);
  std::vector<Scalar> vals;
  vals.reserve(nnz);
  for (int64_t p = 0; p < nnz; ++p) {
    if (w) vals.emplace_back(w[p]);
    else vals.emplace_back(true);
  }
  m.adopt(std::move(row_ptr), std::move(cols), std::move(vals));
  return m;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }

// graph_new (graph.cpp:16-28) with move semantics; kind 0 directed, 1 undirected.
int ref_graph_new(void** out, int64_t n, const int64_t* rp, const int32_t* col,
                  const double* w, int kind) {
  return guarded([&] {
    auto m = csr_to_matrix(n, n, rp, col, w);
    auto* g = new Graph(graph_new(std::move(m), kind ? Kind::UndirectedAdjacency
                                                     : Kind::DirectedAdjacency));
    *out = g;
  });
}

void ref_graph_free(void* g) { delete static_cast<Graph*>(g); }

int ref_property_at(void* g) { return guarded([&] { property_at(*static_cast<Graph*>(g)); }); }
int ref_property_rowdegree(void* g) {
  return guarded([&] { property_rowdegree(*static_cast<Graph*>(g)); });
}
int ref_property_ndiag(void* g) { return guarded([&] { property_ndiag(*static_cast<Graph*>(g)); }); }
int ref_property_symmetric(void* g) {
  return guarded([&] { property_symmetric_pattern(*static_cast<Graph*>(g)); });
}
int64_t ref_ndiag(void* g) { return static_cast<Graph*>(g)->ndiag; }
int ref_symmetric(void* g) {
  auto t = static_cast<Graph*>(g)->pattern_is_symmetric;
  return t == TriState::True ? 1 : (t == TriState::False ? 0 : -1);
}

// direction: 0 Auto, 1 ForcePush, 2 ForcePull (bfs_direction_optimizing),
// 3 = algo::bfs_push.  parent/level: -1 for unreached.
int ref_bfs(void* gp, int64_t src, int direction, int64_t push_divisor, int want_level,
            int64_t* parent, int64_t* level) {
  return guarded([&] {
    auto& g = *static_cast<Graph*>(gp);
    algo::BfsResult r;
    if (direction == 3) {
      r = algo::bfs_push(g, static_cast<Index>(src), want_level != 0);
    } else {
      algo::BfsConfig cfg;
      cfg.direction = direction == 1   ? algo::BfsConfig::Direction::ForcePush
                      : direction == 2 ? algo::BfsConfig::Direction::ForcePull
                                       : algo::BfsConfig::Direction::Auto;
      cfg.push_divisor = static_cast<Index>(push_divisor);
      cfg.want_level = want_level != 0;
      r = algo::bfs_direction_optimizing(g, static_cast<Index>(src), cfg);
    }
    Index n = g.n();
    for (Index i = 0; i < n; ++i) parent[i] = -1;
    for (std::size_t p = 0; p < r.parent.nvals(); ++p)
      parent[r.parent.indices()[p]] = static_cast<int64_t>(as_uint64(r.parent.values()[p]));
    if (level) {
      for (Index i = 0; i < n; ++i) level[i] = -1;
      if (r.level)
        for (std::size_t p = 0; p < r.level->nvals(); ++p)
          level[r.level->indices()[p]] = static_cast<int64_t>(as_uint64(r.level->values()[p]));
    }
  });
}

int ref_pagerank(void* gp, double damping, double tol, int itermax, double* rank,
                 int* iters, double* trace) {
  return guarded([&] {
    auto& g = *static_cast<Graph*>(gp);
    std::vector<std::vector<double>> tr;
    auto r = algo::pagerank_gap(g, damping, tol, itermax, trace ? &tr : nullptr);
    std::memcpy(rank, r.rank.data(), r.rank.size() * sizeof(double));
    *iters = r.iterations;
    if (trace)
      for (std::size_t k = 0; k < tr.size(); ++k)
        std::memcpy(trace + k * g.n(), tr[k].data(), g.n() * sizeof(double));
  });
}

// presort: 0 Auto, 1 Force, 2 Never.
int ref_triangle_count(void* gp, int presort, uint64_t seed, uint64_t* count) {
  return guarded([&] {
    algo::TriangleCountConfig cfg;
    cfg.presort = presort == 1   ? algo::TriangleCountConfig::Presort::Force
                  : presort == 2 ? algo::TriangleCountConfig::Presort::Never
                                 : algo::TriangleCountConfig::Presort::Auto;
    cfg.sample_seed = seed;
    *count = algo::triangle_count(*static_cast<Graph*>(gp), cfg);
  });
}

// dist: +inf for unreached.
int ref_sssp(void* gp, int64_t src, double delta, double* dist) {
  return guarded([&] {
    auto& g = *static_cast<Graph*>(gp);
    auto r = algo::sssp_delta_stepping(g, static_cast<Index>(src), delta);
    for (Index i = 0; i < g.n(); ++i) dist[i] = std::numeric_limits<double>::infinity();
    for (std::size_t p = 0; p < r.dist.nvals(); ++p)
      dist[r.dist.indices()[p]] = as_fp64(r.dist.values()[p]);
  });
}

double ref_sssp_default_delta(void* gp) {
  return algo::sssp_default_delta(*static_cast<Graph*>(gp));
}

int ref_bc(void* gp, const int64_t* sources, int64_t ns, double* centrality) {
  return guarded([&] {
    std::vector<Index> s(sources, sources + ns);
    auto r = algo::betweenness_centrality(*static_cast<Graph*>(gp), s);
    std::memcpy(centrality, r.centrality.data(), r.centrality.size() * sizeof(double));
  });
}

int ref_cc(void* gp, int64_t* label, int* iters) {
  return guarded([&] {
    auto r = algo::connected_components_fastsv(*static_cast<Graph*>(gp));
    for (std::size_t i = 0; i < r.label.size(); ++i) label[i] = static_cast<int64_t>(r.label[i]);
    *iters = r.iterations;
  });
}

// util::sort_by_degree (util.cpp:35-44) / util::sample_degree (util.cpp:46-67).
int ref_sort_by_degree(void* gp, int64_t* perm) {
  return guarded([&] {
    auto p = util::sort_by_degree(*static_cast<Graph*>(gp), true, true);
    for (std::size_t i = 0; i < p.size(); ++i) perm[i] = static_cast<int64_t>(p[i]);
  });
}
int ref_sample_degree(void* gp, int64_t sample, uint64_t seed, double* mean, double* median) {
  return guarded([&] {
    auto s = util::sample_degree(*static_cast<Graph*>(gp), static_cast<Index>(sample), seed);
    *mean = s.mean;
    *median = s.median;
  });
}

// Bounded sample of one PageRank iteration through the reference's own mxv
// (core.cpp:340-386): rows [r0, r1) of AT against the full contribution vector
// of a uniform iterate (pagerank.cpp:55-61).  Returns seconds of the mxv call.
int ref_pr_mxv_sample(int64_t n, const int64_t* at_rp, const int32_t* at_col,
                      const int64_t* outdeg, double damping, int64_t r0, int64_t r1,
                      double* seconds, double* checksum) {
  return guarded([&] {
    int64_t rows = r1 - r0;
    std::vector<int64_t> rp(rows + 1);
    for (int64_t i = 0; i <= rows; ++i) rp[i] = at_rp[r0 + i] - at_rp[r0];
    SparseMatrix sub = csr_to_matrix(rows, n, rp.data(), at_col + at_rp[r0], nullptr);
    SparseMatrix subf(rows, n, Domain::Fp64);
    {
      std::vector<Index> rpp(sub.row_ptr());
      std::vector<Index> cc(sub.col_idx());
      std::vector<Scalar> vv(cc.size(), Scalar(1.0));
      subf.adopt(std::move(rpp), std::move(cc), std::move(vv));
    }
    SparseVector contrib(n, Domain::Fp64);
    {
      std::vector<Index> idx;
      std::vector<Scalar> vals;
      for (int64_t k = 0; k < n; ++k)
        if (outdeg[k] > 0) {
          idx.push_back(k);
          vals.emplace_back((1.0 / n) / (static_cast<double>(outdeg[k]) / damping));
        }
      contrib.adopt(std::move(idx), std::move(vals));
    }
    SparseVector out(rows, Domain::Fp64);
    auto t0 = std::chrono::steady_clock::now();
    mxv(out, Descriptor{}, ops::plus_second(Domain::Fp64), subf, contrib);
    auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    double cs = 0;
    for (const auto& v : out.values()) cs += as_fp64(v);
    *checksum = cs;
  });
}

// verify:: checkers (verify.cpp) for completeness of the golden pins.
int ref_verify_bfs_parents(void* gp, int64_t src, const int64_t* parent, int* ok) {
  return guarded([&] {
    auto& g = *static_cast<Graph*>(gp);
    SparseVector pv(g.n(), Domain::Uint64);
    std::vector<Index> idx;
    std::vector<Scalar> vals;
    for (Index i = 0; i < g.n(); ++i)
      if (parent[i] >= 0) {
        idx.push_back(i);
        vals.emplace_back(static_cast<std::uint64_t>(parent[i]));
      }
    pv.adopt(std::move(idx), std::move(vals));
    *ok = verify::check_bfs_parents(g.A, static_cast<Index>(src), pv, nullptr) ? 1 : 0;
  });
}

// gblite::io round trip (io.cpp:336-355): read_matrix_file(in, in_fmt), then
// write_matrix_file(out, out_fmt) -- or mm_write(symmetric) for "mm_sym".
// Also graph_new's square check (graph.cpp:16-28) when check_graph != 0, so the
// code matches reading straight into a graph.
int ref_io_convert(const char* in_path, const char* in_fmt, const char* out_path,
                   const char* out_fmt, int check_graph) {
  return guarded([&] {
    SparseMatrix m = io::read_matrix_file(in_path, in_fmt);
    if (check_graph) {
      Graph g = graph_new(SparseMatrix(m), Kind::DirectedAdjacency);
      (void)g;
    }
    if (!out_path) return;
    if (std::string(out_fmt) == "mm_sym") {
      std::ofstream out(out_path, std::ios::binary);
      io::mm_write(m, out, true);
    } else {
      io::write_matrix_file(m, out_path, out_fmt);
    }
  });
}

}  // extern "C"

// ---- GraphBLAS operation layer (core.cpp:267-386) for the op-layer fixtures ----
namespace {

Scalar scalar_at(int dom, const void* vals, int64_t p) {
  switch (dom) {
    case 0: return static_cast<const uint8_t*>(vals)[p] != 0;
    case 1: return static_cast<const int64_t*>(vals)[p];
    case 2: return static_cast<const uint64_t*>(vals)[p];
    default: return static_cast<const double*>(vals)[p];
  }
}

void scalar_put(int dom, const Scalar& v, void* out, int64_t p) {
  switch (dom) {
    case 0: static_cast<uint8_t*>(out)[p] = as_bool(v) ? 1 : 0; break;
    case 1: static_cast<int64_t*>(out)[p] = as_int64(v); break;
    case 2: static_cast<uint64_t*>(out)[p] = as_uint64(v); break;
    default: static_cast<double*>(out)[p] = as_fp64(v); break;
  }
}

SparseMatrix mat_of(int64_t nr, int64_t nc, const int64_t* rp, const int64_t* col,
                    const void* vals, int dom) {
  SparseMatrix m(nr, nc, static_cast<Domain>(dom));
  const int64_t nnz = rp[nr];
  std::vector<Index> r(rp, rp + nr + 1), c(col, col + nnz);
  std::vector<Scalar> v;
  v.reserve(nnz);
  for (int64_t p = 0; p < nnz; ++p) v.push_back(scalar_at(dom, vals, p));
  m.adopt(std::move(r), std::move(c), std::move(v));
  return m;
}

SparseVector vec_of(int64_t n, int64_t nv, const int64_t* idx, const void* vals, int dom) {
  SparseVector w(n, static_cast<Domain>(dom));
  for (int64_t p = 0; p < nv; ++p) w.set_element(idx[p], scalar_at(dom, vals, p));
  return w;
}

Semiring semiring_of(int sr, int dom) {
  const Domain d = static_cast<Domain>(dom);
  switch (sr) {
    case 0: return ops::plus_times(d);
    case 1: return ops::any_secondi();
    case 2: return ops::min_plus(d);
    case 3: return ops::plus_first(d);
    case 4: return ops::plus_second(d);
    case 5: return ops::plus_pair(d);
    default: return ops::min_second(d);
  }
}

std::optional<BinaryOp> accum_of(int op, int dom) {
  const Domain d = static_cast<Domain>(dom);
  switch (op) {
    case 1: return ops::plus(d);
    case 2: return ops::minus(d);
    case 3: return ops::times(d);
    case 4: return ops::div(d);
    case 5: return ops::min(d);
    case 6: return ops::max(d);
    case 7: return ops::first(d);
    case 8: return ops::second(d);
    case 9: return ops::pair(d);
    case 10: return ops::any(d);
    case 11: return ops::lor();
    case 12: return ops::land();
    default: return std::nullopt;
  }
}

thread_local SparseMatrix g_last_mat;

}  // namespace

extern "C" {

// op: 0 mxv (A, u), 1 vxm (u, A); returns the post-step output vector
int ref_vec_op(int op, int sr, int sdom, int64_t anr, int64_t anc, const int64_t* arp,
               const int64_t* acol, const void* aval, int adom, int64_t un, int64_t unv,
               const int64_t* uidx, const void* uval, int udom, int64_t wn, int64_t wnv,
               const int64_t* widx, const void* wval, int wdom, int has_mask, int64_t mn,
               int64_t mnv, const int64_t* midx, const void* mval, int mdom, int comp, int structural,
               int replace, int accum, int accum_dom, int tr1, int tr2, int64_t* out_idx,
               void* out_val, int64_t* out_nv) {
  return guarded([&] {
    SparseMatrix A = mat_of(anr, anc, arp, acol, aval, adom);
    SparseVector u = vec_of(un, unv, uidx, uval, udom);
    SparseVector w = vec_of(wn, wnv, widx, wval, wdom);
    SparseVector M = has_mask ? vec_of(mn, mnv, midx, mval, mdom) : SparseVector();
    Descriptor d;
    if (has_mask) d.mask_of(M);
    d.mask.complement = comp != 0;
    d.mask.structural = structural != 0;
    d.mask.replace = replace != 0;
    d.accum = accum_of(accum, accum_dom);
    d.transpose_in1 = tr1 != 0;
    d.transpose_in2 = tr2 != 0;
    const Semiring s = semiring_of(sr, sdom);
    if (op == 0) mxv(w, d, s, A, u);
    else vxm(w, d, s, u, A);
    *out_nv = static_cast<int64_t>(w.nvals());
    for (int64_t p = 0; p < *out_nv; ++p) {
      out_idx[p] = static_cast<int64_t>(w.indices()[p]);
      scalar_put(wdom, w.values()[p], out_val, p);
    }
  });
}

int ref_mxm2(int sr, int sdom, int64_t anr, int64_t anc, const int64_t* arp, const int64_t* acol,
             const void* aval, int adom, int64_t bnr, int64_t bnc, const int64_t* brp,
             const int64_t* bcol, const void* bval, int bdom, int64_t cnr, int64_t cnc,
             const int64_t* crp, const int64_t* ccol, const void* cval, int cdom, int has_mask,
             int64_t mnr, int64_t mnc, const int64_t* mrp, const int64_t* mcol, const void* mval,
             int mdom, int comp, int structural, int replace, int accum, int accum_dom, int tr1,
             int tr2, int64_t* out_nnz) {
  return guarded([&] {
    SparseMatrix A = mat_of(anr, anc, arp, acol, aval, adom);
    SparseMatrix B = mat_of(bnr, bnc, brp, bcol, bval, bdom);
    SparseMatrix C = mat_of(cnr, cnc, crp, ccol, cval, cdom);
    SparseMatrix M = has_mask ? mat_of(mnr, mnc, mrp, mcol, mval, mdom) : SparseMatrix();
    Descriptor d;
    if (has_mask) d.mask_of(M);
    d.mask.complement = comp != 0;
    d.mask.structural = structural != 0;
    d.mask.replace = replace != 0;
    d.accum = accum_of(accum, accum_dom);
    d.transpose_in1 = tr1 != 0;
    d.transpose_in2 = tr2 != 0;
    mxm(C, d, semiring_of(sr, sdom), A, B);
    *out_nnz = static_cast<int64_t>(C.nvals());
    g_last_mat = std::move(C);
  });
}

int ref_mxm(int sr, int sdom, int64_t anr, int64_t anc, const int64_t* arp, const int64_t* acol,
            const void* aval, int adom, int64_t bnr, int64_t bnc, const int64_t* brp,
            const int64_t* bcol, const void* bval, int bdom, int64_t cnr, int64_t cnc,
            const int64_t* crp, const int64_t* ccol, const void* cval, int cdom, int has_mask,
            const int64_t* mrp, const int64_t* mcol, const void* mval, int mdom, int comp,
            int structural, int replace, int accum, int accum_dom, int tr1, int tr2,
            int64_t* out_nnz) {
  return ref_mxm2(sr, sdom, anr, anc, arp, acol, aval, adom, bnr, bnc, brp, bcol, bval, bdom, cnr,
                  cnc, crp, ccol, cval, cdom, has_mask, cnr, cnc, mrp, mcol, mval, mdom, comp,
                  structural, replace, accum, accum_dom, tr1, tr2, out_nnz);
}

void ref_mxm_fetch(int64_t* rp, int64_t* col, void* vals) {
  const SparseMatrix& C = g_last_mat;
  for (int64_t i = 0; i <= static_cast<int64_t>(C.nrows()); ++i) rp[i] = C.row_ptr()[i];
  for (int64_t p = 0; p < static_cast<int64_t>(C.nvals()); ++p) {
    col[p] = C.col_idx()[p];
    scalar_put(static_cast<int>(C.domain()), C.values()[p], vals, p);
  }
}

}  // extern "C"
