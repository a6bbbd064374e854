// Compile/link check of include/gbx_gblite.hpp against the reference's own
// headers and library (the drop-in path a gblite user would take).  Run on a
// GPU box it also checks one PageRank and one BFS against gblite itself.
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "gbx_gblite.hpp"
#include "gblite/util.hpp"

int main(int argc, char** argv) {
  using namespace gblite;
  SparseMatrix m(4, 4, Domain::Bool);
  m.set_element(0, 1, true);
  m.set_element(1, 2, true);
  m.set_element(2, 0, true);
  m.set_element(2, 3, true);
  auto g = graph_new(std::move(m), Kind::DirectedAdjacency);
  property_at(g);
  property_rowdegree(g);
  // device failures surface as DeviceError: still a gblite::Error, distinct type
  static_assert(std::is_base_of_v<Error, b200::DeviceError>);
  try {
    b200::check(GBX_NULL_ARGUMENT, "probe");
    return 3;
  } catch (const b200::DeviceError& e) {
    if (e.gbx_code() != GBX_NULL_ARGUMENT || e.code() != ErrCode::InvalidValue) return 4;
  }
  try {
    b200::check(GBX_SOURCE_OUT_OF_RANGE, "probe");
    return 5;
  } catch (const b200::DeviceError&) {
    return 6;  // an argument error must keep its gblite code, not become a device error
  } catch (const Error& e) {
    if (e.code() != ErrCode::SourceOutOfRange) return 7;
  }
  if (argc < 2) {  // link check only (no GPU)
    std::puts("adapter linked");
    return 0;
  }
  auto want = algo::pagerank_gap(g);
  auto got = b200::algo::pagerank_gap(g);
  double l1 = 0, tot = 0;
  for (Index i = 0; i < 4; ++i) {
    l1 += std::abs(want.rank[i] - got.rank[i]);
    tot += want.rank[i];
  }
  algo::BfsConfig cfg;
  cfg.want_level = true;
  auto bw = algo::bfs_direction_optimizing(g, 0, cfg);
  auto bg = b200::algo::bfs_direction_optimizing(g, 0, cfg);
  bool bfs_ok = util::is_equal(bw.parent, bg.parent) && util::is_equal(*bw.level, *bg.level);
  // the op layer through the reference's own containers: C<M> += A plus.times B
  SparseMatrix A(3, 4, Domain::Fp64), B(4, 2, Domain::Fp64), C(3, 2, Domain::Fp64),
      M(3, 2, Domain::Bool);
  A.set_element(0, 0, 1.5); A.set_element(0, 3, -2.0); A.set_element(2, 1, 0.25);
  B.set_element(0, 1, 4.0); B.set_element(3, 1, 0.5); B.set_element(1, 0, 8.0);
  C.set_element(0, 1, 1.0); C.set_element(1, 0, 7.0);
  M.set_element(0, 1, true); M.set_element(2, 0, true);
  Descriptor d;
  d.mask_of(M).accumulate(ops::plus(Domain::Fp64));
  SparseMatrix Cw = C.dup(), Cg = C.dup();
  mxm(Cw, d, ops::plus_times(Domain::Fp64), A, B);
  b200::mxm(Cg, d, ops::plus_times(Domain::Fp64), A, B);
  const bool mxm_ok = util::is_equal(Cw, Cg);
  SparseVector u(4, Domain::Fp64), w1(3, Domain::Fp64), w2(3, Domain::Fp64);
  u.set_element(0, 2.0); u.set_element(1, 3.0);
  mxv(w1, Descriptor{}, ops::min_plus(Domain::Fp64), A, u);
  b200::mxv(w2, Descriptor{}, ops::min_plus(Domain::Fp64), A, u);
  const bool mxv_ok = util::is_equal(w1, w2);
  std::printf("pagerank iters %d/%d relL1 %.3g bfs %s mxm %s mxv %s\n", want.iterations,
              got.iterations, l1 / tot, bfs_ok ? "ok" : "MISMATCH", mxm_ok ? "ok" : "MISMATCH",
              mxv_ok ? "ok" : "MISMATCH");
  return (want.iterations == got.iterations && l1 / tot < 1e-4 && bfs_ok && mxm_ok && mxv_ok)
             ? 0 : 1;
}
