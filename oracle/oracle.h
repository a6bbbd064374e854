/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference ("gblite", /root/reference/proj) algorithms on
 * the hot path, used as the parity checker for the B200 library.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load it.  The product (libgbx.so) never links or calls anything here.
 *
 * Parity pinning: oracle/make_golden.py runs the reference library itself
 * (oracle/_ref, built from /root/reference sources by oracle/Makefile) on seeded
 * inputs and on the reference's own named fixtures; the resulting vectors are
 * committed under tests/golden/ and tests/test_oracle_golden.py checks this
 * restatement against every one of them.
 *
 * Layout conventions: row_ptr is int64[n+1], col is int32[nnz] sorted strictly
 * ascending per row (the reference's SparseMatrix invariant,
 * containers.cpp:104-124), unreached / absent entries are -1 (ints) or +inf.
 */
#ifndef GBX_ORACLE_H
#define GBX_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- seeded synthetic inputs (the same definition as csrc/gen.cu) -------- */
uint64_t orc_splitmix64(uint64_t state_plus_gamma_times_i);
uint64_t orc_stream(uint64_t seed, uint64_t stream);
uint64_t orc_draw(uint64_t stream_state, uint64_t i);
uint32_t orc_scramble(uint32_t x, int scale, uint64_t seed);

/* R-MAT edge list (ef * 2^scale directed draws). Returns m. */
int64_t orc_rmat_edges(int scale, int edge_factor, double a, double b, double c,
                       uint64_t seed, int scramble, uint32_t* u, uint32_t* v);
/* Erdos-Renyi edge list with weights uniform in [1,255]. Returns m. */
int64_t orc_er_edges(int logn, int degree, uint64_t seed, uint32_t* u,
                     uint32_t* v, int32_t* w);

/* Edge list -> CSR: optional symmetrize, self-loops dropped, duplicates
 * removed (keeping the minimum weight).  col/wout must hold 2m (sym) or m.
 * Returns nnz. */
int64_t orc_build_csr(int64_t n, int64_t m, const uint32_t* u, const uint32_t* v,
                      const int32_t* w, int symmetrize, int64_t* row_ptr,
                      int32_t* col, int32_t* wout);

void orc_transpose(int64_t n, const int64_t* rp, const int32_t* col,
                   const int32_t* w, int64_t* trp, int32_t* tcol, int32_t* tw);

/* ---- algorithms --------------------------------------------------------- */
int orc_bfs(int64_t n, const int64_t* rp, const int32_t* col, int64_t src,
            int64_t* parent, int64_t* level);
int orc_pagerank(int64_t n, const int64_t* at_rp, const int32_t* at_col,
                 const int64_t* outdeg, double damping, double tol, int itermax,
                 double* rank, int* iters, double* trace);
uint64_t orc_triangle_count(int64_t n, const int64_t* rp, const int32_t* col);
int orc_sssp_delta(int64_t n, const int64_t* rp, const int32_t* col,
                   const double* w, int64_t src, double delta, double* dist);
int orc_dijkstra(int64_t n, const int64_t* rp, const int32_t* col,
                 const double* w, int64_t src, double* dist);
int orc_bc(int64_t n, const int64_t* rp, const int32_t* col, const int64_t* at_rp,
           const int32_t* at_col, const int64_t* sources, int64_t ns,
           double* centrality);
int orc_cc(int64_t n, const int64_t* rp, const int32_t* col, int64_t* label);
void orc_sort_by_degree(int64_t n, const int64_t* deg, int64_t* perm);

/* threads used by the parallel parts (OpenMP); 0 = all */
void orc_set_threads(int t);
int orc_get_threads(void);

#ifdef __cplusplus
}
#endif
#endif
