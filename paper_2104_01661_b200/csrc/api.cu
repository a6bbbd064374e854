// api.cu -- the extern "C" boundary (include/gbx.h).  Every entry point maps
// internal gbx::Error / CUDA failures onto gblite::ErrCode values and fills msg
// (empty on success), mirroring the reference's Status / Error contract
// (error.hpp:45-77).  No exception crosses the ABI.
#include <cstdio>
#include <cstring>
#include <string>

#include "common.cuh"
#include "comm.cuh"
#include "plans.cuh"

#ifndef GBX_VERSION
#define GBX_VERSION "gbx-b200 0.1 (sm_100a)"
#endif

gbx_graph::~gbx_graph() {
  if (stream) {
    cudaSetDevice(device);
    cudaStreamSynchronize(stream);
  }
  gbx::ReleaseScope all_idle;  // one device synchronisation for every array below
  pr.reset();
  tc.reset();
  sssp.reset();
  bfs.reset();
  bc.reset();
  cc.reset();
  prs.reset();
  A = gbx::Csr();
  at_own = gbx::Csr();
  rowdeg.release();
  coldeg.release();
  if (stream) cudaStreamDestroy(stream);
  (void)cudaGetLastError();  // never leave a destructor's error for the next call
}

namespace gbx {

gbx_graph* graph_handle() {
  auto* g = new gbx_graph();
  cudaError_t e = cudaGetDevice(&g->device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete g;
    gbx::fail(GBX_CUDA_ERROR, std::string("no CUDA device: ") + cudaGetErrorString(e));
  }
  return g;
}

void reset_plans(gbx_graph* g) {
  g->pr.reset();
  g->tc.reset();
  g->sssp.reset();
  g->bc.reset();
  g->prs.reset();
}

}  // namespace gbx

namespace {

void set_msg(char* msg, const std::string& s) {
  if (!msg) return;
  size_t n = std::min<size_t>(s.size(), GBX_MSG_LEN - 1);
  std::memcpy(msg, s.data(), n);
  msg[n] = '\0';
}

template <typename F>
int guard(char* msg, F&& f) {
  try {
    f();
    set_msg(msg, "");
    return GBX_SUCCESS;
  } catch (const gbx::Error& e) {
    set_msg(msg, e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_msg(msg, "host allocation failed");
    return GBX_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    set_msg(msg, e.what());
    return GBX_CUDA_ERROR;
  }
}

gbx_graph* need(const gbx_graph* g) {
  if (!g) gbx::fail(GBX_NULL_ARGUMENT, "graph handle is NULL");
  return const_cast<gbx_graph*>(g);
}

gbx_graph* new_handle() { return gbx::graph_handle(); }

template <typename Build>
int make_graph(gbx_graph** out, char* msg, Build&& build) {
  return guard(msg, [&] {
    if (!out) gbx::fail(GBX_NULL_ARGUMENT, "output handle pointer is NULL");
    *out = nullptr;
    gbx_graph* g = new_handle();
    try {
      std::lock_guard<std::mutex> lk(g->mu);
      build(g);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

}  // namespace

namespace {
template <typename Build>
int make_mat(gbx_mat** out, char* msg, Build&& build) {
  return guard(msg, [&] {
    if (!out) gbx::fail(GBX_NULL_ARGUMENT, "output handle pointer is NULL");
    *out = nullptr;
    gbx_mat* m = gbx::mat_alloc();
    try {
      build(m);
    } catch (...) {
      delete m;
      throw;
    }
    *out = m;
  });
}
gbx_mat* need_mat(const gbx_mat* m) {
  if (!m) gbx::fail(GBX_NULL_ARGUMENT, "matrix handle is NULL");
  return const_cast<gbx_mat*>(m);
}
}  // namespace

extern "C" {

const char* gbx_version(void) { return GBX_VERSION; }

int gbx_set_option(const char* name, int64_t value, char* msg) {
  return guard(msg, [&] { gbx::set_option(name, value); });
}

int gbx_reset_option(const char* name, char* msg) {
  return guard(msg, [&] { gbx::reset_option(name); });
}

int gbx_get_option(const char* name, int64_t* value, char* msg) {
  return guard(msg, [&] {
    if (!value) gbx::fail(GBX_NULL_ARGUMENT, "value is NULL");
    *value = gbx::get_option(name);
  });
}

const char* gbx_option_name(int index) { return gbx::option_name(index); }

int gbx_init(int device, char* msg) {
  return guard(msg, [&] {
    int count = 0;
    GBX_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count)
      gbx::fail(GBX_INVALID_VALUE, "device " + std::to_string(device) + " of " +
                                       std::to_string(count));
    GBX_CUDA(cudaSetDevice(device));
    GBX_CUDA(cudaFree(nullptr));
  });
}

int gbx_graph_new(gbx_graph** out, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                  const void* vals, int domain, int kind, char* msg) {
  return make_graph(out, msg, [&](gbx_graph* g) {
    gbx::build_from_host(g, n, row_ptr, col_idx, nullptr, vals, domain, kind);
  });
}

int gbx_graph_new32(gbx_graph** out, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                    const void* vals, int domain, int kind, char* msg) {
  return make_graph(out, msg, [&](gbx_graph* g) {
    gbx::build_from_host(g, n, row_ptr, nullptr, col_idx, vals, domain, kind);
  });
}

int gbx_graph_build(gbx_graph** out, int64_t n, int64_t nvals, const int64_t* rows,
                    const int64_t* cols, const void* vals, int domain, int dup, int kind,
                    char* msg) {
  return make_graph(out, msg, [&](gbx_graph* g) {
    gbx::build_from_coo(g, n, n, nvals, rows, cols, vals, domain, dup, kind, true);
  });
}

int gbx_graph_read(gbx_graph** out, const char* path, const char* format, int kind, char* msg) {
  return make_graph(out, msg, [&](gbx_graph* g) {
    if (!path) gbx::fail(GBX_NULL_ARGUMENT, "path is NULL");
    gbx::graph_read(g, path, nullptr, 0, format, kind);
  });
}

int gbx_graph_read_buffer(gbx_graph** out, const void* data, size_t len, const char* format,
                          int kind, char* msg) {
  return make_graph(out, msg, [&](gbx_graph* g) {
    if (!data && len) gbx::fail(GBX_NULL_ARGUMENT, "data is NULL");
    static const char empty = 0;
    gbx::graph_read(g, nullptr, data ? data : &empty, len, format, kind);
  });
}

int gbx_graph_write(const gbx_graph* gc, const char* path, const char* format, int symmetric,
                    char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    gbx::Scope sc(g);
    gbx::graph_write(g, path, format, symmetric);
  });
}

// ---- GraphBLAS operation layer (ops.cu) ------------------------------------


int gbx_mat_new(gbx_mat** out, int64_t nrows, int64_t ncols, const int64_t* row_ptr,
                const int64_t* col_idx, const void* vals, int domain, char* msg) {
  return make_mat(out, msg, [&](gbx_mat* m) {
    gbx::mat_from_host(m, nrows, ncols, row_ptr, col_idx, vals, domain);
  });
}

int gbx_mat_from_graph(gbx_mat** out, const gbx_graph* gc, int which, char* msg) {
  return make_mat(out, msg, [&](gbx_mat* m) {
    gbx_graph* g = need(gc);
    gbx::Scope sc(g);
    gbx::mat_from_graph(m, g, which);
  });
}

int gbx_mat_info(const gbx_mat* mc, int64_t* nrows, int64_t* ncols, int64_t* nvals, int* domain,
                 char* msg) {
  return guard(msg, [&] {
    gbx_mat* m = need_mat(mc);
    if (nrows) *nrows = m->nrows;
    if (ncols) *ncols = m->ncols;
    if (nvals) *nvals = m->nnz;
    if (domain) *domain = m->domain;
  });
}

int gbx_mat_export(const gbx_mat* mc, int64_t* row_ptr, int64_t* col_idx, void* vals, char* msg) {
  return guard(msg, [&] { gbx::mat_export(need_mat(mc), row_ptr, col_idx, vals); });
}

int gbx_mat_free(gbx_mat** m, char* msg) {
  return guard(msg, [&] {
    if (!m) gbx::fail(GBX_NULL_ARGUMENT, "handle pointer is NULL");
    delete *m;
    *m = nullptr;
  });
}

int gbx_mxv(int64_t* w_idx, void* w_vals, int64_t* w_nvals, const gbx_vec* w, const gbx_desc* desc,
            int semiring, int domain, const gbx_mat* A, const gbx_vec* u, char* msg) {
  return guard(msg, [&] {
    gbx::mxv_op(w_idx, w_vals, w_nvals, w, desc, semiring, domain, need_mat(A), u);
  });
}

int gbx_vxm(int64_t* w_idx, void* w_vals, int64_t* w_nvals, const gbx_vec* w, const gbx_desc* desc,
            int semiring, int domain, const gbx_vec* u, const gbx_mat* A, char* msg) {
  return guard(msg, [&] {
    gbx::vxm_op(w_idx, w_vals, w_nvals, w, desc, semiring, domain, u, need_mat(A));
  });
}

int gbx_mxm(gbx_mat** C_out, const gbx_mat* C, const gbx_desc* desc, int semiring, int domain,
            const gbx_mat* A, const gbx_mat* B, char* msg) {
  return make_mat(C_out, msg, [&](gbx_mat* out) {
    gbx::mxm_op(out, need_mat(C), desc, semiring, domain, need_mat(A), need_mat(B));
  });
}

int gbx_generate_rmat(gbx_graph** out, int scale, int edge_factor, double a, double b,
                      double c, uint64_t seed, int scramble, int kind, char* msg) {
  return make_graph(out, msg, [&](gbx_graph* g) {
    if (kind != GBX_DIRECTED && kind != GBX_UNDIRECTED)
      gbx::fail(GBX_INVALID_VALUE, "rmat: unknown kind");
    gbx::generate_rmat(g, scale, edge_factor, a, b, c, seed, scramble, kind);
  });
}

int gbx_generate_er(gbx_graph** out, int logn, int degree, uint64_t seed, int weighted,
                    char* msg) {
  return make_graph(out, msg,
                    [&](gbx_graph* g) { gbx::generate_er(g, logn, degree, seed, weighted); });
}

int gbx_graph_free(gbx_graph** g, char* msg) {
  return guard(msg, [&] {
    if (!g) gbx::fail(GBX_NULL_ARGUMENT, "handle pointer is NULL");
    delete *g;
    *g = nullptr;
  });
}

int gbx_graph_info(const gbx_graph* gc, int64_t* n, int64_t* nnz, int* kind, int* domain,
                   char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    if (n) *n = g->A.n;
    if (nnz) *nnz = g->A.nnz;
    if (kind) *kind = g->kind;
    if (domain) *domain = g->A.domain;
  });
}

int gbx_graph_export(const gbx_graph* gc, int64_t* row_ptr, int32_t* col, void* vals,
                     char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    gbx::Scope sc(g);
    cudaStream_t s = g->stream;
    if (row_ptr)
      GBX_CUDA(cudaMemcpyAsync(row_ptr, g->A.rp.p, (g->A.n + 1) * 8, cudaMemcpyDeviceToHost, s));
    if (col && g->A.nnz)
      GBX_CUDA(cudaMemcpyAsync(col, g->A.col.p, g->A.nnz * 4, cudaMemcpyDeviceToHost, s));
    if (vals && g->A.nnz && g->A.val.p)
      GBX_CUDA(cudaMemcpyAsync(vals, g->A.val.p, g->A.nnz * gbx::domain_size(g->A.domain),
                               cudaMemcpyDeviceToHost, s));
    gbx::sync(g);
  });
}

// property_at (graph.cpp:30-41): undirected graphs store A's content (aliased).
int gbx_property_at(gbx_graph* g, char* msg) {
  return guard(msg, [&] {
    need(g);
    gbx::Scope sc(g);
    if (g->kind != GBX_UNDIRECTED) {
      g->at_own = gbx::Csr();
      g->at_pending = true;  // built on first read (gbx_graph::AT)
    }
    g->has_at = true;
  });
}

int gbx_property_rowdegree(gbx_graph* g, char* msg) {
  return guard(msg, [&] {
    need(g);
    gbx::Scope sc(g);
    gbx::compute_degrees(g->stream, g->A, g->rowdeg, true);
    gbx::sync(g);
    g->has_rowdeg = true;
  });
}

int gbx_property_coldegree(gbx_graph* g, char* msg) {
  return guard(msg, [&] {
    need(g);
    gbx::Scope sc(g);
    gbx::compute_degrees(g->stream, g->A, g->coldeg, false);
    gbx::sync(g);
    g->has_coldeg = true;
  });
}

// property_symmetric_pattern (graph.cpp:80-94): compare A with (cached) AT.
int gbx_property_symmetric_pattern(gbx_graph* g, char* msg) {
  return guard(msg, [&] {
    need(g);
    gbx::Scope sc(g);
    bool sym;
    if (g->has_at) {
      sym = g->kind == GBX_UNDIRECTED ? true : gbx::csr_equal(g->stream, g->A, g->AT());
    } else {
      gbx::Csr t;
      gbx::compute_transpose(g->stream, g->A, t);
      sym = gbx::csr_equal(g->stream, g->A, t);
    }
    g->symmetric = sym ? GBX_TRUE : GBX_FALSE;
  });
}

int gbx_property_ndiag(gbx_graph* g, char* msg) {
  return guard(msg, [&] {
    need(g);
    gbx::Scope sc(g);
    g->ndiag = gbx::count_ndiag(g->stream, g->A);
  });
}

int gbx_delete_properties(gbx_graph* g, char* msg) {
  return guard(msg, [&] {
    need(g);
    gbx::Scope sc(g);
    gbx::sync(g);
    gbx::reset_plans(g);
    g->at_own = gbx::Csr();
    g->at_pending = false;
    g->has_at = false;
    g->rowdeg.release();
    g->coldeg.release();
    g->has_rowdeg = g->has_coldeg = false;
    g->symmetric = GBX_UNKNOWN;
    g->ndiag = -1;
  });
}

int gbx_graph_properties(const gbx_graph* gc, int* has_at, int* has_rowdeg, int* has_coldeg,
                         int* symmetric, int64_t* ndiag, char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    if (has_at) *has_at = g->has_at ? 1 : 0;
    if (has_rowdeg) *has_rowdeg = g->has_rowdeg ? 1 : 0;
    if (has_coldeg) *has_coldeg = g->has_coldeg ? 1 : 0;
    if (symmetric) *symmetric = g->symmetric;
    if (ndiag) *ndiag = g->ndiag;
  });
}

static void degree_out(gbx_graph* g, const gbx::DevArray<int32_t>& d, int64_t* out) {
  gbx::Scope sc(g);
  std::vector<int32_t> h(g->A.n);
  if (g->A.n)
    GBX_CUDA(cudaMemcpyAsync(h.data(), d.p, g->A.n * 4, cudaMemcpyDeviceToHost, g->stream));
  gbx::sync(g);
  for (int64_t i = 0; i < g->A.n; ++i) out[i] = h[i];
}

int gbx_row_degree(const gbx_graph* gc, int64_t* deg, char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    if (!g->has_rowdeg) gbx::fail(GBX_MISSING_PROPERTY, "row_degree property not computed");
    degree_out(g, g->rowdeg, deg);
  });
}

int gbx_col_degree(const gbx_graph* gc, int64_t* deg, char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    if (!g->has_coldeg) gbx::fail(GBX_MISSING_PROPERTY, "col_degree property not computed");
    degree_out(g, g->coldeg, deg);
  });
}

// check_graph (graph.cpp:112-187)
int gbx_check_graph(const gbx_graph* gc, char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    gbx::Scope sc(g);
    cudaStream_t s = g->stream;
    gbx::Csr t;
    gbx::compute_transpose(s, g->A, t);
    if (g->has_at && g->kind != GBX_UNDIRECTED && !gbx::csr_equal(s, g->AT(), t))
      gbx::fail(GBX_INVALID_GRAPH, "AT does not equal transpose(A)");
    auto check_deg = [&](const gbx::DevArray<int32_t>& d, bool by_row, const char* name) {
      gbx::DevArray<int32_t> want;
      gbx::compute_degrees(s, g->A, want, by_row);
      std::vector<int32_t> a(g->A.n), b(g->A.n);
      if (g->A.n) {
        GBX_CUDA(cudaMemcpyAsync(a.data(), d.p, g->A.n * 4, cudaMemcpyDeviceToHost, s));
        GBX_CUDA(cudaMemcpyAsync(b.data(), want.p, g->A.n * 4, cudaMemcpyDeviceToHost, s));
      }
      gbx::sync(g);
      for (int64_t i = 0; i < g->A.n; ++i)
        if (a[i] != b[i])
          gbx::fail(GBX_INVALID_GRAPH, std::string(name) + " disagrees with A at node " +
                                           std::to_string(i));
    };
    if (g->has_rowdeg) check_deg(g->rowdeg, true, "row_degree");
    if (g->has_coldeg) check_deg(g->coldeg, false, "col_degree");
    bool sym = gbx::csr_equal(s, g->A, t);
    if (g->kind == GBX_UNDIRECTED && !sym)
      gbx::fail(GBX_INVALID_GRAPH, "undirected graph with an asymmetric pattern");
    if (g->symmetric == GBX_TRUE && !sym)
      gbx::fail(GBX_INVALID_GRAPH, "pattern_is_symmetric is TRUE but A is asymmetric");
    if (g->symmetric == GBX_FALSE && sym)
      gbx::fail(GBX_INVALID_GRAPH, "pattern_is_symmetric is FALSE but A is symmetric");
    if (g->ndiag != -1 && gbx::count_ndiag(s, g->A) != g->ndiag)
      gbx::fail(GBX_INVALID_GRAPH, "ndiag disagrees with A");
  });
}

int gbx_sort_by_degree(int64_t* perm, const gbx_graph* gc, int ascending, int by_row,
                       char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    gbx::Scope sc(g);
    if (by_row ? !g->has_rowdeg : !g->has_coldeg)
      gbx::fail(GBX_MISSING_PROPERTY, by_row ? "row_degree property not computed"
                                             : "col_degree property not computed");
    gbx::DevArray<int32_t> p;
    gbx::sort_ids_by_key(g->stream, by_row ? g->rowdeg.p : g->coldeg.p, g->A.n,
                         ascending != 0, p);
    std::vector<int32_t> h(g->A.n);
    if (g->A.n)
      GBX_CUDA(cudaMemcpyAsync(h.data(), p.p, g->A.n * 4, cudaMemcpyDeviceToHost, g->stream));
    gbx::sync(g);
    for (int64_t i = 0; i < g->A.n; ++i) perm[i] = h[i];
  });
}

// ---- algorithms ------------------------------------------------------------

int gbx_bfs_push(int64_t* parent, int64_t* level, const gbx_graph* gc, uint64_t source,
                 char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    gbx::Scope sc(g);
    gbx::bfs_run(g, source, GBX_BFS_PUSH, 16, false, parent, level);
  });
}

int gbx_bfs(int64_t* parent, int64_t* level, const gbx_graph* gc, uint64_t source,
            int direction, uint64_t push_divisor, char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    gbx::Scope sc(g);
    gbx::require_at(g, "bfs_direction_optimizing");
    gbx::bfs_run(g, source, direction, push_divisor, true, parent, level);
  });
}

int gbx_bfs_batch(int64_t* parent, int64_t* level, const gbx_graph* gc,
                  const uint64_t* sources, uint64_t ns, char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    gbx::Scope sc(g);
    if (ns > 0 && !sources) gbx::fail(GBX_NULL_ARGUMENT, "sources is NULL");
    gbx::bfs_batch_run(g, sources, ns, parent, level);
  });
}

int gbx_pagerank(double* rank, int* iterations, const gbx_graph* gc, double damping,
                 double tol, int itermax, char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    gbx::Scope sc(g);
    gbx::pagerank_run(g, damping, tol, itermax, rank, iterations);
  });
}

// triangle_count preconditions (triangle.cpp:13-26)
static void tc_preconditions(const gbx_graph* g) {
  if (g->kind != GBX_UNDIRECTED) {
    if (g->symmetric == GBX_UNKNOWN)
      gbx::fail(GBX_MISSING_PROPERTY,
                "triangle_count needs the symmetric-pattern property on directed graphs");
    if (g->symmetric == GBX_FALSE)
      gbx::fail(GBX_PRECONDITION_VIOLATED, "triangle_count needs a symmetric pattern");
  }
  if (g->ndiag == -1) gbx::fail(GBX_MISSING_PROPERTY, "triangle_count needs the ndiag property");
  if (g->ndiag != 0) gbx::fail(GBX_PRECONDITION_VIOLATED, "triangle_count needs a loop-free graph");
}

int gbx_triangle_count(uint64_t* count, const gbx_graph* gc, int presort, uint64_t sample_seed,
                       char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    gbx::Scope sc(g);
    (void)sample_seed;
    if (presort < GBX_PRESORT_AUTO || presort > GBX_PRESORT_NEVER)
      gbx::fail(GBX_INVALID_VALUE, "triangle_count: unknown presort");
    tc_preconditions(g);
    if (presort == GBX_PRESORT_AUTO || presort == GBX_PRESORT_FORCE)
      gbx::require_rowdeg(g, "triangle_count");
    uint64_t c = gbx::tc_run(g, 0, -1);
    if (count) *count = c;
  });
}

int gbx_triangle_count_rows(uint64_t* count, const gbx_graph* gc, int64_t rb, int64_t re,
                            char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    gbx::Scope sc(g);
    tc_preconditions(g);
    uint64_t c = gbx::tc_run(g, rb, re);
    if (count) *count = c;
  });
}

int gbx_tc_partition(int64_t* bounds, gbx_graph* g, int parts, char* msg) {
  return guard(msg, [&] {
    need(g);
    gbx::Scope sc(g);
    tc_preconditions(g);
    gbx::tc_partition(g, parts, bounds);
  });
}

int gbx_sssp(double* dist, const gbx_graph* gc, uint64_t source, double delta, char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    gbx::Scope sc(g);
    gbx::sssp_run(g, source, delta, dist);
  });
}

int gbx_sssp_batch(double* dist, const gbx_graph* gc, const uint64_t* sources, uint64_t ns,
                   double delta, char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    gbx::Scope sc(g);
    gbx::sssp_batch_run(g, sources, ns, delta, dist);
  });
}

int gbx_sssp_default_delta(double* delta, const gbx_graph* gc, char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    gbx::Scope sc(g);
    *delta = gbx::sssp_default_delta(g);
  });
}

int gbx_betweenness(double* centrality, const gbx_graph* gc, const uint64_t* sources,
                    uint64_t ns, char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    gbx::Scope sc(g);
    gbx::require_at(g, "betweenness_centrality");
    if (ns == 0) gbx::fail(GBX_EMPTY_BATCH, "empty source batch");
    if (!sources) gbx::fail(GBX_NULL_ARGUMENT, "sources is NULL");
    gbx::bc_run(g, sources, ns, centrality);
  });
}

// components preconditions (components.cpp:13-24)
static void cc_preconditions(const gbx_graph* g) {
  if (g->kind == GBX_UNDIRECTED) return;
  if (g->symmetric == GBX_UNKNOWN)
    gbx::fail(GBX_MISSING_PROPERTY,
              "connected_components needs the symmetric-pattern property on directed graphs");
  if (g->symmetric == GBX_FALSE)
    gbx::fail(GBX_PRECONDITION_VIOLATED, "connected_components needs a symmetric pattern");
}

int gbx_connected_components(int64_t* label, int* iterations, const gbx_graph* gc, char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    gbx::Scope sc(g);
    cc_preconditions(g);
    gbx::cc_run(g, label, iterations);
  });
}

// ---- basic forms: fill the missing caches, then delegate ---------------------

int gbx_basic_bfs_push(int64_t* parent, int64_t* level, gbx_graph* g, uint64_t source,
                       char* msg) {
  return gbx_bfs_push(parent, level, g, source, msg);
}

int gbx_basic_bfs(int64_t* parent, int64_t* level, gbx_graph* g, uint64_t source,
                  int direction, uint64_t push_divisor, char* msg) {
  if (g && !g->has_at) {
    int rc = gbx_property_at(g, msg);
    if (rc) return rc;
  }
  return gbx_bfs(parent, level, g, source, direction, push_divisor, msg);
}

int gbx_basic_pagerank(double* rank, int* iterations, gbx_graph* g, double damping, double tol,
                       int itermax, char* msg) {
  if (g && !g->has_at) {
    int rc = gbx_property_at(g, msg);
    if (rc) return rc;
  }
  if (g && !g->has_rowdeg) {
    int rc = gbx_property_rowdegree(g, msg);
    if (rc) return rc;
  }
  return gbx_pagerank(rank, iterations, g, damping, tol, itermax, msg);
}

int gbx_basic_triangle_count(uint64_t* count, gbx_graph* g, int presort, uint64_t seed,
                             char* msg) {
  if (g && g->kind != GBX_UNDIRECTED && g->symmetric == GBX_UNKNOWN) {
    int rc = gbx_property_symmetric_pattern(g, msg);
    if (rc) return rc;
  }
  if (g && g->ndiag == -1) {
    int rc = gbx_property_ndiag(g, msg);
    if (rc) return rc;
  }
  if (g && !g->has_rowdeg) {
    int rc = gbx_property_rowdegree(g, msg);
    if (rc) return rc;
  }
  return gbx_triangle_count(count, g, presort, seed, msg);
}

int gbx_basic_sssp(double* dist, gbx_graph* g, uint64_t source, double delta, char* msg) {
  if (!(delta > 0.0)) {
    double d = 1.0;
    int rc = gbx_sssp_default_delta(&d, g, msg);
    if (rc) return rc;
    delta = d;
  }
  return gbx_sssp(dist, g, source, delta, msg);
}

int gbx_basic_betweenness(double* centrality, gbx_graph* g, const uint64_t* sources,
                          uint64_t ns, char* msg) {
  if (g && !g->has_at) {
    int rc = gbx_property_at(g, msg);
    if (rc) return rc;
  }
  return gbx_betweenness(centrality, g, sources, ns, msg);
}

int gbx_basic_connected_components(int64_t* label, int* iterations, gbx_graph* g, char* msg) {
  if (g && g->kind != GBX_UNDIRECTED && g->symmetric == GBX_UNKNOWN) {
    int rc = gbx_property_symmetric_pattern(g, msg);
    if (rc) return rc;
  }
  return gbx_connected_components(label, iterations, g, msg);
}

// ---- device plumbing -------------------------------------------------------

int gbx_graph_stream(const gbx_graph* gc, void** stream, char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    *stream = reinterpret_cast<void*>(g->stream);
  });
}

int gbx_prepare(gbx_graph* g, const char* which, char* msg) {
  return guard(msg, [&] {
    need(g);
    gbx::Scope sc(g);
    std::string w = which ? which : "";
    if (w == "pagerank") gbx::pagerank_prepare(g);
    else if (w == "tc") gbx::tc_prepare(g);
    else if (w == "sssp") gbx::sssp_prepare(g);
    else if (w == "bfs") gbx::bfs_prepare(g);
    else if (w == "bc") {}
    else gbx::fail(GBX_INVALID_VALUE, "gbx_prepare: unknown algorithm '" + w + "'");
    gbx::sync(g);
  });
}

int gbx_result_device(const gbx_graph* gc, const char* which, void** ptr, int64_t* count,
                      char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    gbx::result_device(g, which ? which : "", ptr, count);
  });
}

int gbx_last_stats(const gbx_graph* gc, gbx_stats* stats, char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    gbx::Scope sc(g);
    if (g->pending_iters) {  // an asynchronous call: its count lands with the stream
      int it = 0;
      GBX_CUDA(cudaMemcpyAsync(&it, g->pending_iters, sizeof(int), cudaMemcpyDeviceToHost, g->stream));
      GBX_CUDA(cudaStreamSynchronize(g->stream));
      g->stats.iterations = it;
      g->pending_iters = nullptr;
    }
    *stats = g->stats;
  });
}

int gbx_bfs_shard_begin(gbx_graph* g, uint64_t source, int rank, int nranks, int64_t* row_begin,
                        int64_t* row_end, char* msg) {
  return guard(msg, [&] {
    need(g);
    gbx::Scope sc(g);
    gbx::bfs_shard_begin(g, source, rank, nranks, row_begin, row_end);
  });
}

int gbx_bfs_shard_level(gbx_graph* g, const uint32_t* front, uint32_t* next_slice, int64_t* found,
                        char* msg) {
  return guard(msg, [&] {
    need(g);
    if (!front || !found) gbx::fail(GBX_NULL_ARGUMENT, "frontier / found is NULL");
    gbx::Scope sc(g);
    gbx::bfs_shard_level(g, front, next_slice, found);
  });
}

int gbx_bfs_shard_result(gbx_graph* g, int64_t* parent, int64_t* level, char* msg) {
  return guard(msg, [&] {
    need(g);
    gbx::Scope sc(g);
    gbx::bfs_shard_result(g, parent, level);
  });
}

int gbx_bc_shard_begin(gbx_graph* g, const uint64_t* sources, uint64_t ns, int rank, int nranks,
                       int64_t* row_begin, int64_t* row_end, char* msg) {
  return guard(msg, [&] {
    need(g);
    if (!sources && ns) gbx::fail(GBX_NULL_ARGUMENT, "sources is NULL");
    gbx::Scope sc(g);
    gbx::bc_shard_begin(g, sources, ns, rank, nranks, row_begin, row_end);
  });
}

int gbx_bc_shard_forward(gbx_graph* g, void** recs, int64_t* nrecs, char* msg) {
  return guard(msg, [&] {
    need(g);
    if (!recs || !nrecs) gbx::fail(GBX_NULL_ARGUMENT, "output pointers are NULL");
    gbx::Scope sc(g);
    gbx::bc_shard_forward(g, recs, nrecs);
  });
}

int gbx_bc_shard_forward_apply(gbx_graph* g, const void* recs, int64_t nrecs, int* done, char* msg) {
  return guard(msg, [&] {
    need(g);
    if (!recs && nrecs) gbx::fail(GBX_NULL_ARGUMENT, "records are NULL");
    gbx::Scope sc(g);
    gbx::bc_shard_forward_apply(g, recs, nrecs, done);
  });
}

int gbx_bc_shard_backward(gbx_graph* g, void** recs, int64_t* nrecs, int* done, char* msg) {
  return guard(msg, [&] {
    need(g);
    if (!recs || !nrecs || !done) gbx::fail(GBX_NULL_ARGUMENT, "output pointers are NULL");
    gbx::Scope sc(g);
    gbx::bc_shard_backward(g, recs, nrecs, done);
  });
}

int gbx_bc_shard_backward_apply(gbx_graph* g, const void* recs, int64_t nrecs, char* msg) {
  return guard(msg, [&] {
    need(g);
    if (!recs && nrecs) gbx::fail(GBX_NULL_ARGUMENT, "records are NULL");
    gbx::Scope sc(g);
    gbx::bc_shard_backward_apply(g, recs, nrecs);
  });
}

int gbx_bc_shard_centrality(gbx_graph* g, double** cent, char* msg) {
  return guard(msg, [&] {
    need(g);
    if (!cent) gbx::fail(GBX_NULL_ARGUMENT, "output pointer is NULL");
    gbx::Scope sc(g);
    gbx::bc_shard_centrality(g, cent);
  });
}

int gbx_pr_shard_prepare(gbx_graph* g, int rank, int nranks, int64_t* row_begin,
                         int64_t* row_end, char* msg) {
  return guard(msg, [&] {
    need(g);
    gbx::Scope sc(g);
    gbx::pr_shard_prepare(g, rank, nranks, row_begin, row_end);
  });
}

int gbx_pr_shard_init(gbx_graph* g, float* x_full, float* r_local, double damping, char* msg) {
  return guard(msg, [&] {
    need(g);
    gbx::Scope sc(g);
    gbx::pr_shard_init(g, x_full, r_local, damping);
  });
}

int gbx_pr_shard_unpermute(gbx_graph* g, const float* r_full, double* out, char* msg) {
  return guard(msg, [&] {
    need(g);
    gbx::Scope sc(g);
    gbx::pr_shard_unpermute(g, r_full, out);
  });
}

int gbx_pr_shard_step(gbx_graph* g, const float* x_full, const float* r_prev, float* r_new,
                      float* x_slice, double* l1, double damping, char* msg) {
  return guard(msg, [&] {
    need(g);
    if (!x_full || !r_prev || !r_new || !x_slice || !l1)
      gbx::fail(GBX_NULL_ARGUMENT, "pr_shard_step: NULL device buffer");
    gbx::Scope sc(g);
    gbx::pr_shard_step(g, x_full, r_prev, r_new, x_slice, l1, damping);
  });
}

int gbx_pr_shard_run_p2p(gbx_graph* g, const uint64_t* x0_peers, const uint64_t* x1_peers,
                         const uint64_t* l1_peers, const uint64_t* sig_peers, float* r0,
                         float* r1, double damping, double tol, int itermax, int* iters,
                         char* msg) {
  return guard(msg, [&] {
    need(g);
    gbx::Scope sc(g);
    gbx::pr_shard_run_p2p(g, x0_peers, x1_peers, l1_peers, sig_peers, r0, r1, damping, tol,
                          itermax, iters);
  });
}

int gbx_pr_shard_run_p2p_multi(gbx_graph* const* shards, int nranks, const uint64_t* x0_peers,
                               const uint64_t* x1_peers, const uint64_t* l1_peers,
                               const uint64_t* sig_peers, float* const* r0, float* const* r1,
                               double damping, double tol, int itermax, int* iters, char* msg) {
  return guard(msg, [&] {
    if (!shards || !r0 || !r1) gbx::fail(GBX_NULL_ARGUMENT, "pr_shard_run_p2p_multi: NULL array");
    std::vector<std::unique_ptr<gbx::Scope>> sc;
    for (int v = 0; v < nranks; ++v) sc.emplace_back(new gbx::Scope(need(shards[v])));
    gbx::pr_shard_run_p2p_multi(shards, nranks, x0_peers, x1_peers, l1_peers, sig_peers, r0, r1,
                                damping, tol, itermax, iters);
  });
}

int gbx_pr_shard_layout(const gbx_graph* gc, int64_t* chunk, int64_t* bounds, char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    gbx::pr_shard_layout(g, chunk, bounds);
  });
}

int gbx_partition_rows(int64_t* bounds, const gbx_graph* gc, int parts, int transposed,
                       char* msg) {
  return guard(msg, [&] {
    gbx_graph* g = need(gc);
    gbx::Scope sc(g);
    gbx::partition_rows(g, parts, transposed != 0, bounds);
  });
}

}  // extern "C"

// ---- multi-GPU: communicator, distributed graph, algorithms ----------------------

namespace {

gbx_comm* need_comm(const gbx_comm* c) {
  if (!c) gbx::fail(GBX_NULL_ARGUMENT, "communicator handle is NULL");
  return const_cast<gbx_comm*>(c);
}
gbx_dgraph* need_dg(const gbx_dgraph* g) {
  if (!g) gbx::fail(GBX_NULL_ARGUMENT, "distributed graph handle is NULL");
  return const_cast<gbx_dgraph*>(g);
}
void check_local(const gbx_dgraph* g, int l) {
  if (l < 0 || l >= g->comm->nlocal) gbx::fail(GBX_INVALID_VALUE, "local rank out of range");
}

}  // namespace

int gbx_comm_unique_id(void* id, char* msg) {
  return guard(msg, [&] {
    if (!id) gbx::fail(GBX_NULL_ARGUMENT, "id is NULL");
    gbx::comm_unique_id(id);
  });
}

int gbx_comm_init(gbx_comm** c, int nranks, int rank, const void* id, int device, char* msg) {
  return guard(msg, [&] {
    if (!c) gbx::fail(GBX_NULL_ARGUMENT, "comm out-pointer is NULL");
    *c = nullptr;
    *c = gbx::comm_new_nccl(nranks, rank, id, device);
  });
}

int gbx_comm_init_local(gbx_comm** c, int nranks, int device, char* msg) {
  return guard(msg, [&] {
    if (!c) gbx::fail(GBX_NULL_ARGUMENT, "comm out-pointer is NULL");
    *c = nullptr;
    *c = gbx::comm_new_local(nranks, device);
  });
}

int gbx_comm_free(gbx_comm** c, char* msg) {
  return guard(msg, [&] {
    if (c && *c) {
      delete *c;
      *c = nullptr;
    }
  });
}

int gbx_comm_info(const gbx_comm* c, int* nranks, int* rank, int* nlocal, char* msg) {
  return guard(msg, [&] {
    need_comm(c);
    if (nranks) *nranks = c->nranks;
    if (rank) *rank = c->rank;
    if (nlocal) *nlocal = c->nlocal;
  });
}

int gbx_dgraph_generate_rmat(gbx_dgraph** g, gbx_comm* c, int scale, int edge_factor, double a,
                             double b, double cc, uint64_t seed, int scramble, int kind,
                             char* msg) {
  return guard(msg, [&] {
    if (!g) gbx::fail(GBX_NULL_ARGUMENT, "graph out-pointer is NULL");
    *g = nullptr;
    need_comm(c);
    std::lock_guard<std::mutex> lk(c->mu);
    *g = gbx::dgraph_generate_rmat(c, scale, edge_factor, a, b, cc, seed, scramble, kind);
  });
}

int gbx_dgraph_from_blocks(gbx_dgraph** g, gbx_comm* c, int64_t n, const int64_t* row_begin,
                           const int64_t* row_end, const int64_t* const* row_ptr,
                           const int32_t* const* col, int kind, char* msg) {
  return guard(msg, [&] {
    if (!g) gbx::fail(GBX_NULL_ARGUMENT, "graph out-pointer is NULL");
    *g = nullptr;
    need_comm(c);
    std::lock_guard<std::mutex> lk(c->mu);
    *g = gbx::dgraph_from_blocks(c, n, row_begin, row_end, row_ptr, col, kind);
  });
}

int gbx_dgraph_free(gbx_dgraph** g, char* msg) {
  return guard(msg, [&] {
    if (g && *g) {
      // the communicator must still be alive (free graphs before their comm)
      GBX_CUDA(cudaSetDevice((*g)->device));
      delete *g;
      *g = nullptr;
    }
  });
}

int gbx_dgraph_info(const gbx_dgraph* g, int64_t* n, int64_t* nnz, int* kind, char* msg) {
  return guard(msg, [&] {
    need_dg(g);
    if (n) *n = g->n;
    if (nnz) *nnz = g->nnz;
    if (kind) *kind = g->kind;
  });
}

int gbx_dgraph_block(const gbx_dgraph* g, int local, int64_t* rb, int64_t* re, int64_t* nnz,
                     char* msg) {
  return guard(msg, [&] {
    need_dg(g);
    check_local(g, local);
    int64_t b, e;
    gbx::dgraph_block(g, local, &b, &e);
    if (rb) *rb = b;
    if (re) *re = e;
    if (nnz) *nnz = g->local_nnz[local];
  });
}

int gbx_dgraph_export_block(const gbx_dgraph* g, int local, int64_t* row_ptr, int32_t* col,
                            char* msg) {
  return guard(msg, [&] {
    need_dg(g);
    check_local(g, local);
    int64_t b, e;
    gbx::dgraph_block(g, local, &b, &e);
    const gbx_graph* s = g->shard[local];
    GBX_CUDA(cudaSetDevice(g->comm->device));
    if (row_ptr) GBX_CUDA(cudaMemcpy(row_ptr, s->A.rp.p + b, (e - b + 1) * 8, cudaMemcpyDeviceToHost));
    if (col && s->A.nnz) GBX_CUDA(cudaMemcpy(col, s->A.col.p, s->A.nnz * 4, cudaMemcpyDeviceToHost));
  });
}

int gbx_dgraph_last_stats(const gbx_dgraph* g, gbx_stats* st, char* msg) {
  return guard(msg, [&] {
    need_dg(g);
    if (!st) gbx::fail(GBX_NULL_ARGUMENT, "stats is NULL");
    *st = g->stats;
  });
}

int gbx_pagerank_mg(double* rank, int* iters, gbx_dgraph* g, double damping, double tol,
                    int itermax, int exchange, char* msg) {
  return guard(msg, [&] { gbx::pagerank_mg(need_dg(g), damping, tol, itermax, exchange, rank, iters); });
}

int gbx_triangle_count_mg(uint64_t* count, gbx_dgraph* g, char* msg) {
  return guard(msg, [&] {
    const uint64_t t = gbx::triangle_count_mg(need_dg(g));
    if (count) *count = t;
  });
}

int gbx_bfs_mg(int64_t* parent, int64_t* level, gbx_dgraph* g, uint64_t source, char* msg) {
  return guard(msg, [&] { gbx::bfs_mg(need_dg(g), source, parent, level); });
}

int gbx_betweenness_mg(double* centrality, gbx_dgraph* g, const uint64_t* sources, uint64_t ns,
                       char* msg) {
  return guard(msg, [&] { gbx::betweenness_mg(need_dg(g), sources, ns, centrality); });
}
