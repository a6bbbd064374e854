// Compile/link check of include/gbx_gblite.hpp against the reference's own
// headers and library (the drop-in path a gblite user would take).  Run on a
// GPU box it also checks one PageRank and one BFS against gblite itself.
#include <cstdio>
#include <cstdlib>

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
  std::printf("pagerank iters %d/%d relL1 %.3g bfs %s\n", want.iterations, got.iterations,
              l1 / tot, bfs_ok ? "ok" : "MISMATCH");
  return (want.iterations == got.iterations && l1 / tot < 1e-4 && bfs_ok) ? 0 : 1;
}
