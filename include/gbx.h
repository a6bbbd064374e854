/*
 * gbx.h -- C ABI of the B200-native hot path (libgbx.so).
 *
 * Drop-in boundary for the reference's (gblite, /root/reference/proj) graph
 * object and algorithm entry points.  The reference surface is a C++ namespace
 * API; this header is its C restatement in the LAGraph calling convention the
 * paper uses: outputs first, then inputs, then
 * char msg[GBX_MSG_LEN] last; int return 0 = success, < 0 error, > 0 warning.
 * Return codes are IDENTICAL to gblite::ErrCode (include/gblite/error.hpp:13-41);
 * codes <= -30 are new (device / runtime failures).  msg is "" on success
 * (Status::kMaxMessage = 256, error.hpp:67).  No exceptions cross this ABI.
 *
 * Ownership: a gbx_graph owns device copies of A and of every cached property
 * (graph.hpp:27-39).  Host arrays passed in are only read.  Outputs are
 * caller-allocated host arrays of length n (or ns*n).  Passing NULL for a
 * result array keeps the result on the device (see gbx_result_device), which
 * is how device-resident throughput is measured.
 *
 * Threading: every handle owns one CUDA stream; calls are synchronous from the
 * host's view unless every output pointer is NULL.  Calls on one handle are
 * serialised internally.
 *
 * Each entry point cites the reference interface it replaces.
 */
#ifndef GBX_H
#define GBX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GBX_MSG_LEN 256

/* ---- error codes: gblite::ErrCode (error.hpp:13-41) + device codes ------- */
enum {
  GBX_SUCCESS = 0,
  GBX_NO_VALUE = 1,
  GBX_DIMENSION_MISMATCH = -1,
  GBX_DOMAIN_MISMATCH = -2,
  GBX_INDEX_OUT_OF_BOUNDS = -3,
  GBX_INVALID_MATRIX = -4,
  GBX_INVALID_GRAPH = -5,
  GBX_MISSING_PROPERTY = -6,
  GBX_SOURCE_OUT_OF_RANGE = -7,
  GBX_EMPTY_BATCH = -8,
  GBX_NON_POSITIVE_DAMPING = -9,
  GBX_NON_POSITIVE_DELTA = -10,
  GBX_NON_POSITIVE_WEIGHT = -11,
  GBX_PRECONDITION_VIOLATED = -12,
  GBX_PARSE_ERROR = -13,
  GBX_DUPLICATE_ENTRY = -14,
  GBX_IO_FAILURE = -15,
  GBX_BAD_MAGIC = -16,
  GBX_UNSUPPORTED_VERSION = -17,
  GBX_TRUNCATED_STREAM = -18,
  GBX_LENGTH_MISMATCH = -19,
  GBX_ALIASED_OUTPUT = -20,
  GBX_INVALID_VALUE = -21,
  /* new: failures the CPU reference cannot have */
  GBX_CUDA_ERROR = -30,
  GBX_OUT_OF_MEMORY = -31,
  GBX_UNSUPPORTED = -32,
  GBX_NULL_ARGUMENT = -33,
  GBX_COMM_ERROR = -34  /* NCCL / peer-memory failure of a multi-GPU call */
};

/* value domains: gblite::Domain (value.hpp:18-23) + int32 weights */
enum { GBX_BOOL = 0, GBX_INT64 = 1, GBX_UINT64 = 2, GBX_FP64 = 3, GBX_INT32 = 4 };
/* gblite::Kind (graph.hpp:16-19) */
enum { GBX_DIRECTED = 0, GBX_UNDIRECTED = 1 };
/* gblite::TriState (graph.hpp:23) */
enum { GBX_FALSE = 0, GBX_TRUE = 1, GBX_UNKNOWN = -1 };
/* algo::BfsConfig::Direction (algorithms.hpp:28) */
enum { GBX_BFS_AUTO = 0, GBX_BFS_PUSH = 1, GBX_BFS_PULL = 2 };
/* algo::TriangleCountConfig::Presort (algorithms.hpp:69) */
enum { GBX_PRESORT_AUTO = 0, GBX_PRESORT_FORCE = 1, GBX_PRESORT_NEVER = 2 };

typedef struct gbx_graph gbx_graph;

/* Library / device.  Returns the library version string in msg. */
int gbx_init(int device, char msg[GBX_MSG_LEN]);
const char* gbx_version(void);

/* Tuning / diagnostics options (process-wide; no reference counterpart -- the
 * reference has no device knobs).  Unknown names and out-of-range values ->
 * GBX_INVALID_VALUE.  gbx_option_name(i) enumerates them (NULL past the end):
 *   pagerank.l1_window_kb  144    bytes of x gathered with L1 evict_last
 *   pagerank.carveout      10     % shared-memory carveout of the row kernels (-1: driver)
 *   pagerank.host_loop     0      1: one launch per iteration (for ncu captures)
 *   pagerank.trace         0      1: per-iteration phase means (%globaltimer) on stderr
 *   p2p.timeout_ms         10000  bound of the fused multi-GPU exchange's peer wait
 *   bfs.alpha              14     push while frontier edges < nnz/alpha (0: bfs.cpp:77-78 rule)
 *   bfs64.pull_div         2      64-lane batch: pull when frontier edges > nnz/div
 *   bfs_mg.push_div        0      gbx_bfs_mg: 0 = push while frontier edges < nnz/bfs.alpha,
 *                                 else push while the frontier < n/div (bfs.cpp:77-78)
 *   bfs.trace / sssp.trace 0      1: per-level %globaltimer log on stderr (sssp 2: + device printf)
  *   sssp.pull_pct          50     heavy pass of a bucket by pull (heavy in-edges, ascending
 *                                 weight, pruned) when its pops*100 > pct * vertices not yet
 *                                 popped; 0: always push
 *   bc.alpha               14     as bfs.alpha for the Brandes forward sweep
 *   bc.trace               0      1: per-depth host timing on stderr
 *   bc.back_push           2      a backward depth runs in push form (children add into
 *                                 their parents' sums, fp64 atomics) when its children's
 *                                 rows hold <= 1/this of the parents' edges; 0: always pull
 *   bc.back_push_min_depth 3      ... and the depth is at least this (hub levels pull)
 *   bc.relabel_min_n       262144 graphs of at least this many vertices run the batched
 *                                 Brandes on a degree-sorted copy built once per graph
 *                                 (sources mapped in, centrality mapped back); -1: never */
int gbx_set_option(const char* name, int64_t value, char msg[GBX_MSG_LEN]);
int gbx_reset_option(const char* name, char msg[GBX_MSG_LEN]);
int gbx_get_option(const char* name, int64_t* value, char msg[GBX_MSG_LEN]);
const char* gbx_option_name(int index);

/* ---- graph object (graph.hpp:27-60, graph.cpp:16-220) --------------------- */

/* graph_new(SparseMatrix&&, Kind) (graph.cpp:16-28): validates the CSR like
 * SparseMatrix::validate (containers.cpp:104-124) -> GBX_INVALID_MATRIX, square
 * only.  vals may be NULL for a Bool pattern; otherwise its element type is
 * domain (GBX_FP64 / GBX_INT64 / GBX_UINT64 / GBX_INT32 / GBX_BOOL as uint8). */
int gbx_graph_new(gbx_graph** g, int64_t n, const int64_t* row_ptr,
                  const int64_t* col_idx, const void* vals, int domain, int kind,
                  char msg[GBX_MSG_LEN]);
/* Same, with int32 column indices (saves the host-side widening). */
int gbx_graph_new32(gbx_graph** g, int64_t n, const int64_t* row_ptr,
                    const int32_t* col_idx, const void* vals, int domain, int kind,
                    char msg[GBX_MSG_LEN]);
int gbx_graph_free(gbx_graph** g, char msg[GBX_MSG_LEN]);

/* Seeded synthetic graphs built directly in HBM (the BASELINE configs):
 * R-MAT (edge_factor * 2^scale draws, quadrant probabilities a/b/c, optional id
 * scramble; kind GBX_UNDIRECTED symmetrises) and Erdos-Renyi (degree * 2^logn
 * uniform draws, int32 weights in [1,255] when weighted).  Self-loops and
 * duplicates are removed (duplicates keep the minimum weight).  Bit-identical
 * to oracle/oracle.c's generator. */
int gbx_generate_rmat(gbx_graph** g, int scale, int edge_factor, double a, double b,
                      double c, uint64_t seed, int scramble, int kind,
                      char msg[GBX_MSG_LEN]);
int gbx_generate_er(gbx_graph** g, int logn, int degree, uint64_t seed, int weighted,
                    char msg[GBX_MSG_LEN]);

/* build_matrix (containers.cpp:128-169) + graph_new on the device: n x n
 * tuples (rows[k], cols[k], vals[k]) -- host arrays -- sorted stably on the
 * device, duplicates combined in input order by dup (GBX_DUP_ERROR fails with
 * GBX_DUPLICATE_ENTRY, as mm_read's trap, io.cpp:143-153); a tuple outside
 * n x n is GBX_INDEX_OUT_OF_BOUNDS.  vals NULL = Bool pattern. */
enum { GBX_DUP_ERROR = 0, GBX_DUP_FIRST = 1, GBX_DUP_SECOND = 2, GBX_DUP_MIN = 3,
       GBX_DUP_MAX = 4, GBX_DUP_PLUS = 5 };
int gbx_graph_build(gbx_graph** g, int64_t n, int64_t nvals, const int64_t* rows,
                    const int64_t* cols, const void* vals, int domain, int dup, int kind,
                    char msg[GBX_MSG_LEN]);

/* gblite::io (io.hpp): read_matrix_file (io.cpp:336-343) + graph_new.
 * format "bin" = LAGK v1 (bin_read, io.cpp:282-334: GBX_BAD_MAGIC,
 * GBX_UNSUPPORTED_VERSION, GBX_TRUNCATED_STREAM, GBX_PARSE_ERROR for an invalid
 * matrix) streamed to HBM through pinned staging; "mm" = Matrix Market
 * coordinate (mm_read, io.cpp:35-160: pattern/integer/real, general/symmetric,
 * "%%domain", GBX_PARSE_ERROR / GBX_INDEX_OUT_OF_BOUNDS / GBX_DUPLICATE_ENTRY).
 * A non-square matrix is GBX_INVALID_MATRIX (graph_new).  GBX_IO_FAILURE when
 * the file cannot be opened.  The _buffer form parses len bytes in memory. */
int gbx_graph_read(gbx_graph** g, const char* path, const char* format, int kind,
                   char msg[GBX_MSG_LEN]);
int gbx_graph_read_buffer(gbx_graph** g, const void* data, size_t len, const char* format,
                          int kind, char msg[GBX_MSG_LEN]);
/* write_matrix_file (io.cpp:345-355): "bin" byte-identical to bin_write
 * (io.cpp:261-280); "mm" byte-identical to mm_write (io.cpp:162-222), symmetric
 * != 0 writes the lower triangle and requires a symmetric matrix
 * (GBX_INVALID_VALUE otherwise). */
int gbx_graph_write(const gbx_graph* g, const char* path, const char* format, int symmetric,
                    char msg[GBX_MSG_LEN]);

/* n, nnz, kind, value domain. */
int gbx_graph_info(const gbx_graph* g, int64_t* n, int64_t* nnz, int* kind, int* domain,
                   char msg[GBX_MSG_LEN]);
/* Copy A back to the host (row_ptr[n+1], col[nnz]; vals[nnz] in the graph's
 * domain, may be NULL). */
int gbx_graph_export(const gbx_graph* g, int64_t* row_ptr, int32_t* col, void* vals,
                     char msg[GBX_MSG_LEN]);

/* property_at / rowdegree / coldegree / symmetric_pattern / ndiag
 * (graph.cpp:30-102) and delete_properties (graph.cpp:104-110). */
int gbx_property_at(gbx_graph* g, char msg[GBX_MSG_LEN]);
int gbx_property_rowdegree(gbx_graph* g, char msg[GBX_MSG_LEN]);
int gbx_property_coldegree(gbx_graph* g, char msg[GBX_MSG_LEN]);
int gbx_property_symmetric_pattern(gbx_graph* g, char msg[GBX_MSG_LEN]);
int gbx_property_ndiag(gbx_graph* g, char msg[GBX_MSG_LEN]);
int gbx_delete_properties(gbx_graph* g, char msg[GBX_MSG_LEN]);
/* Cache status: has_at, has_rowdeg, has_coldeg (0/1), symmetric (TriState),
 * ndiag (-1 unknown). */
int gbx_graph_properties(const gbx_graph* g, int* has_at, int* has_rowdeg,
                         int* has_coldeg, int* symmetric, int64_t* ndiag,
                         char msg[GBX_MSG_LEN]);
/* Dense row/column degree (0 for empty rows); requires the cache. */
int gbx_row_degree(const gbx_graph* g, int64_t* deg, char msg[GBX_MSG_LEN]);
int gbx_col_degree(const gbx_graph* g, int64_t* deg, char msg[GBX_MSG_LEN]);
/* check_graph (graph.cpp:112-187): 0 iff every cache is consistent with A,
 * else GBX_INVALID_GRAPH naming the first violated invariant. */
int gbx_check_graph(const gbx_graph* g, char msg[GBX_MSG_LEN]);
/* util::sort_by_degree(g, ascending, by_row) (util.cpp:35-44): stable. */
int gbx_sort_by_degree(int64_t* perm, const gbx_graph* g, int ascending, int by_row,
                       char msg[GBX_MSG_LEN]);

/* ---- algorithms: advanced forms (algorithms.hpp:19-86) ---------------------
 * Advanced calls never touch the caches and fail with GBX_MISSING_PROPERTY when
 * one is absent; gbx_basic_* compute what is missing, then delegate
 * (algorithms.hpp:89-104). */

/* algo::bfs_push (bfs.cpp:56-62) / bfs_direction_optimizing (bfs.cpp:64-85).
 * parent[n]: parent id, parent(source) = source, -1 = unreached.
 * level[n] (nullable): hop count, -1 = unreached.  Parents are the minimum-id
 * neighbour on the previous level (the reference's any.secondi in ascending k). */
int gbx_bfs_push(int64_t* parent, int64_t* level, const gbx_graph* g, uint64_t source,
                 char msg[GBX_MSG_LEN]);
int gbx_bfs(int64_t* parent, int64_t* level, const gbx_graph* g, uint64_t source,
            int direction, uint64_t push_divisor, char msg[GBX_MSG_LEN]);
/* B200 extension: ns independent BFS runs in one multi-source sweep (64-bit
 * lanes).  parent/level are [ns][n] row-major. */
int gbx_bfs_batch(int64_t* parent, int64_t* level, const gbx_graph* g,
                  const uint64_t* sources, uint64_t ns, char msg[GBX_MSG_LEN]);

/* algo::pagerank_gap (pagerank.cpp:8-81): GAP PageRank, dangling mass lost.
 * rank[n] (nullable), iterations (nullable).  fp32 ranks, fp64 row sums and
 * fp64 L1 change (compared against tol exactly as pagerank.cpp:65-74). */
int gbx_pagerank(double* rank, int* iterations, const gbx_graph* g, double damping,
                 double tol, int itermax, char msg[GBX_MSG_LEN]);

/* algo::triangle_count (triangle.cpp:30-64).  The count is invariant under the
 * presort choice; presort/seed are validated and recorded but the device
 * kernel always orients edges by ascending degree. */
int gbx_triangle_count(uint64_t* count, const gbx_graph* g, int presort,
                       uint64_t sample_seed, char msg[GBX_MSG_LEN]);

/* algo::sssp_delta_stepping (sssp.cpp:16-112).  dist[n]: +inf = unreached.
 * Weights must be positive (GBX_FP64, GBX_INT32 or GBX_INT64 domain). */
int gbx_sssp(double* dist, const gbx_graph* g, uint64_t source, double delta,
             char msg[GBX_MSG_LEN]);
/* algo::sssp_default_delta (sssp.cpp:114-120): max weight / 2, or 1. */
/* Several sources of sssp_delta_stepping (gapbench runs one trial per source,
 * gapbench.cpp:300-330) in one call: the traversals are queued back to back
 * on the graph's stream with one host synchronisation at the end.
 * dist: ns * n doubles, row b = sources[b] (as gbx_sssp), or NULL. */
int gbx_sssp_batch(double* dist, const gbx_graph* g, const uint64_t* sources, uint64_t ns,
                   double delta, char msg[GBX_MSG_LEN]);
int gbx_sssp_default_delta(double* delta, const gbx_graph* g, char msg[GBX_MSG_LEN]);

/* algo::betweenness_centrality (betweenness.cpp:11-86): batched Brandes,
 * centrality[n] = sum over sources of the dependency (no halving). */
int gbx_betweenness(double* centrality, const gbx_graph* g, const uint64_t* sources,
                    uint64_t ns, char msg[GBX_MSG_LEN]);

/* algo::connected_components_fastsv (components.cpp:35-106): label[n] = the
 * minimum vertex id of the component. */
int gbx_connected_components(int64_t* label, int* iterations, const gbx_graph* g,
                             char msg[GBX_MSG_LEN]);

/* ---- basic forms (algorithms.hpp:89-104) ---------------------------------- */
int gbx_basic_bfs_push(int64_t* parent, int64_t* level, gbx_graph* g, uint64_t source,
                       char msg[GBX_MSG_LEN]);
int gbx_basic_bfs(int64_t* parent, int64_t* level, gbx_graph* g, uint64_t source,
                  int direction, uint64_t push_divisor, char msg[GBX_MSG_LEN]);
int gbx_basic_pagerank(double* rank, int* iterations, gbx_graph* g, double damping,
                       double tol, int itermax, char msg[GBX_MSG_LEN]);
int gbx_basic_triangle_count(uint64_t* count, gbx_graph* g, int presort,
                             uint64_t sample_seed, char msg[GBX_MSG_LEN]);
/* delta <= 0 means "use sssp_default_delta" (sssp.cpp:124-127). */
int gbx_basic_sssp(double* dist, gbx_graph* g, uint64_t source, double delta,
                   char msg[GBX_MSG_LEN]);
int gbx_basic_betweenness(double* centrality, gbx_graph* g, const uint64_t* sources,
                          uint64_t ns, char msg[GBX_MSG_LEN]);
int gbx_basic_connected_components(int64_t* label, int* iterations, gbx_graph* g,
                                   char msg[GBX_MSG_LEN]);

/* ---- GraphBLAS operation layer (core.hpp / core.cpp, ops.cpp) -------------
 * The operations the paper's algorithms are written in, on the device, with
 * the reference's semantics bit for bit (every fold in the reference's order):
 *   gbx_mxv  (core.cpp:340-386)  w<mask> accum= A ⊕.⊗ u
 *   gbx_vxm  (core.cpp:308-338)  w<mask> accum= u ⊕.⊗ A
 *   gbx_mxm  (core.cpp:267-306)  C<mask> accum= A ⊕.⊗ B
 * followed by the shared mask / accumulator / replace post-step
 * (merge_entries, core.cpp:131-175).  Matrices are gbx_mat handles (device
 * CSR, any shape, bool/int64/uint64/fp64 values); vectors are host sparse
 * vectors (ascending indices).  Vector results are written to caller arrays of
 * capacity w->n; matrix results are new gbx_mat handles.  Errors are the
 * reference's: DimensionMismatch, DomainMismatch, AliasedOutput,
 * InvalidMatrix, InvalidValue. */
typedef struct gbx_mat gbx_mat;
/* built-in semirings (ops.cpp:362-372); the domain argument is the operand /
 * result domain (any_secondi is always uint64) */
enum { GBX_SR_PLUS_TIMES = 0, GBX_SR_ANY_SECONDI = 1, GBX_SR_MIN_PLUS = 2, GBX_SR_PLUS_FIRST = 3,
       GBX_SR_PLUS_SECOND = 4, GBX_SR_PLUS_PAIR = 5, GBX_SR_MIN_SECOND = 6 };
/* binary operators (ops.cpp:52-203) for the accumulator; GBX_OP_SECONDI is
 * the positional multiply of any_secondi only */
enum { GBX_OP_NONE = 0, GBX_OP_PLUS = 1, GBX_OP_MINUS = 2, GBX_OP_TIMES = 3, GBX_OP_DIV = 4,
       GBX_OP_MIN = 5, GBX_OP_MAX = 6, GBX_OP_FIRST = 7, GBX_OP_SECOND = 8, GBX_OP_PAIR = 9,
       GBX_OP_ANY = 10, GBX_OP_LOR = 11, GBX_OP_LAND = 12, GBX_OP_SECONDI = 13 };
/* SparseVector (containers.hpp): n, nvals, idx[nvals] ascending, vals[nvals]
 * (bool as uint8, others 8 bytes) */
typedef struct {
  int64_t n;
  int64_t nvals;
  const int64_t* idx;
  const void* vals;
  int domain;
} gbx_vec;
/* Descriptor + MaskSpec (core.hpp:15-73); zero-initialised = no mask, merge,
 * no accumulator, no transposes */
typedef struct {
  const gbx_vec* mask_vec;
  const gbx_mat* mask_mat;
  int complement;
  int structural;
  int replace;
  int accum;         /* GBX_OP_*; GBX_OP_NONE = no accumulator */
  int accum_domain;  /* the accumulator operator's domain */
  int transpose_in1;
  int transpose_in2;
} gbx_desc;
/* SparseMatrix from host CSR (validated like containers.cpp:104-124) */
int gbx_mat_new(gbx_mat** m, int64_t nrows, int64_t ncols, const int64_t* row_ptr,
                const int64_t* col_idx, const void* vals, int domain, char msg[GBX_MSG_LEN]);
/* a graph's A (which = 0) or cached AT (which = 1) as an operand; pattern
 * graphs are bool true, int32 weights widen to int64 */
int gbx_mat_from_graph(gbx_mat** m, const gbx_graph* g, int which, char msg[GBX_MSG_LEN]);
int gbx_mat_info(const gbx_mat* m, int64_t* nrows, int64_t* ncols, int64_t* nvals, int* domain,
                 char msg[GBX_MSG_LEN]);
/* row_ptr[nrows+1], col[nvals] (int64), vals[nvals] (domain element size) */
int gbx_mat_export(const gbx_mat* m, int64_t* row_ptr, int64_t* col_idx, void* vals,
                   char msg[GBX_MSG_LEN]);
int gbx_mat_free(gbx_mat** m, char msg[GBX_MSG_LEN]);
/* w is the prior output (its entries merge / accumulate); the result replaces
 * it in (w_idx, w_vals, *w_nvals) */
int gbx_mxv(int64_t* w_idx, void* w_vals, int64_t* w_nvals, const gbx_vec* w,
            const gbx_desc* desc, int semiring, int domain, const gbx_mat* A, const gbx_vec* u,
            char msg[GBX_MSG_LEN]);
int gbx_vxm(int64_t* w_idx, void* w_vals, int64_t* w_nvals, const gbx_vec* w,
            const gbx_desc* desc, int semiring, int domain, const gbx_vec* u, const gbx_mat* A,
            char msg[GBX_MSG_LEN]);
/* *C_out = post_step(C, A ⊕.⊗ B); C is the prior output (not modified) */
int gbx_mxm(gbx_mat** C_out, const gbx_mat* C, const gbx_desc* desc, int semiring, int domain,
            const gbx_mat* A, const gbx_mat* B, char msg[GBX_MSG_LEN]);

/* ---- device plumbing (benchmarks, multi-GPU drivers) ---------------------- */

/* The handle's CUDA stream (cudaStream_t) -- record events on it to time calls. */
int gbx_graph_stream(const gbx_graph* g, void** stream, char msg[GBX_MSG_LEN]);
/* Build the per-algorithm device layouts ahead of time so the first call does
 * not pay for them: which = "pagerank" | "tc" | "sssp" | "bfs" | "bc". */
int gbx_prepare(gbx_graph* g, const char* which, char msg[GBX_MSG_LEN]);
/* Device pointer + element count of the last result of an algorithm
 * (which as above, plus "cc"); layout documented in DESIGN.md. */
int gbx_result_device(const gbx_graph* g, const char* which, void** ptr,
                      int64_t* count, char msg[GBX_MSG_LEN]);
/* Launch statistics of the last call: number of kernel launches, and for the
 * dominant kernel its launch count and algorithmic bytes per launch. */
typedef struct {
  int64_t launches;            /* our kernels launched by the last call   */
  int64_t hot_launches;        /* launches of the dominant kernel         */
  double hot_bytes_per_launch; /* algorithmic bytes per dominant launch   */
  int64_t work_units;          /* edges / wedges / relaxations processed  */
  int iterations;              /* levels / iterations                     */
  double hot_ms;               /* mean device duration of one dominant-kernel
                                  launch in the last call (ms; 0 = not measured) */
} gbx_stats;
int gbx_last_stats(const gbx_graph* g, gbx_stats* stats, char msg[GBX_MSG_LEN]);

/* ---- sharded PageRank for the multi-GPU driver (1D row blocks) -------------
 * pagerank.cpp:52-76 split over ranks.  Every rank holds the graph; rank r of
 * nranks owns rows [row_begin, row_end) of the in-degree-relabeled AT (balanced
 * by rows + nnz; every rank computes the same split).  Exchange layout: rank
 * q's contributions live at x_full[q * chunk + (row - bounds[q])], chunk = the
 * longest block rounded up to even + 2 (gbx_pr_shard_layout), so x_full has
 * nranks * chunk floats; the last 8 bytes of every slot are free for the rank's
 * fp64 L1 partial (pass l1_dev = (double*)(x_slice + chunk - 2)), so ONE
 * equal-size all-gather of the chunk-long slices (NCCL all_gather_into_tensor)
 * per iteration moves the contributions and every partial in place.
 *   gbx_pr_shard_init   x_full (padded) = initial contributions, r_local = 1/n;
 *   gbx_pr_shard_step   for its rows: r_new = teleport + sum x(k) (fp64),
 *                       x_slice[row - row_begin] = r_new * damping / outdeg,
 *                       *l1_dev = fp64 L1 partial |r_prev - r_new| (r_prev may
 *                       alias r_new); the caller all-gathers the slices and
 *                       sums the partials (pagerank.cpp:65-74 on the sum);
 *   gbx_pr_shard_unpermute maps a gathered (padded) rank vector back to the
 *                       original vertex order (fp64, host).
 * All vector arguments are device pointers. */
int gbx_pr_shard_prepare(gbx_graph* g, int rank, int nranks, int64_t* row_begin,
                         int64_t* row_end, char msg[GBX_MSG_LEN]);
/* The whole sharded run in ONE cooperative launch per rank, the exchange fused
 * into the iteration kernel (no NCCL per iteration): the row epilogue stores
 * x_next straight into every rank's padded x over NVLink (peer pointers, e.g.
 * torch symmetric memory); the rank's fp64 L1 total goes to slot
 * [k&1][rank] of every rank's table; a device-side barrier (one system-scope
 * signal increment per peer, spin on the own word) separates iterations and
 * every rank sums the table in rank order -> the same stop decision.
 *   x0_peers/x1_peers[q]  rank q's x buffers (nranks * chunk floats each); x0
 *                         holds the initial contributions (gbx_pr_shard_init)
 *   l1_peers[q]           rank q's slot table (2 * nranks doubles)
 *   sig_peers[q]          rank q's signal word (u32); every word must read 0
 *                         when the run starts (zero them, then barrier)
 *   r0 / r1               this rank's local rank buffers (chunk floats; r0 =
 *                         the initial 1/n); the result is in (iters & 1 ? r1 : r0)
 * At most 8 ranks; every rank must call it (the kernels wait on each other). */
int gbx_pr_shard_run_p2p(gbx_graph* g, const uint64_t* x0_peers, const uint64_t* x1_peers,
                         const uint64_t* l1_peers, const uint64_t* sig_peers, float* r0,
                         float* r1, double damping, double tol, int itermax, int* iters,
                         char msg[GBX_MSG_LEN]);
/* chunk (slot length of the padded layout) and, if non-NULL, bounds[nranks+1]. */
/* The same run for `nranks` shards that all live on THIS GPU, as ONE
 * cooperative launch (shard v = rank v; its CTAs are co-resident with every
 * other rank's, so no rank ever waits on a rank that is not running): the
 * single-GPU emulation of the multi-rank protocol (tests, gbx_comm_init_local).
 * Peer arrays as above, r0[v] / r1[v] per rank.  Fails with GBX_CUDA_ERROR if
 * the ranks disagree on the iteration count. */
int gbx_pr_shard_run_p2p_multi(gbx_graph* const* shards, int nranks, const uint64_t* x0_peers,
                               const uint64_t* x1_peers, const uint64_t* l1_peers,
                               const uint64_t* sig_peers, float* const* r0, float* const* r1,
                               double damping, double tol, int itermax, int* iters,
                               char msg[GBX_MSG_LEN]);
int gbx_pr_shard_layout(const gbx_graph* g, int64_t* chunk, int64_t* bounds,
                        char msg[GBX_MSG_LEN]);
int gbx_pr_shard_init(gbx_graph* g, float* x_full_dev, float* r_local_dev, double damping,
                      char msg[GBX_MSG_LEN]);
int gbx_pr_shard_step(gbx_graph* g, const float* x_full_dev, const float* r_prev_dev,
                      float* r_new_dev, float* x_slice_dev, double* l1_dev, double damping,
                      char msg[GBX_MSG_LEN]);
int gbx_pr_shard_unpermute(gbx_graph* g, const float* r_full_dev, double* rank_out,
                           char msg[GBX_MSG_LEN]);
/* Rows [row_begin,row_end) of a split with balanced nnz + rows (merge-path). */
int gbx_partition_rows(int64_t* bounds, const gbx_graph* g, int parts, int transposed,
                       char msg[GBX_MSG_LEN]);
/* Triangle count restricted to the triangles whose middle vertex, in the
 * degree-ordered rank space, lies in [row_begin, row_end) (for work-balanced
 * sharding; the sum over a partition of [0, n) = count). */
int gbx_triangle_count_rows(uint64_t* count, const gbx_graph* g, int64_t row_begin,
                            int64_t row_end, char msg[GBX_MSG_LEN]);
/* Wedge-balanced split of the oriented rows into parts. */
int gbx_tc_partition(int64_t* bounds, gbx_graph* g, int parts, char msg[GBX_MSG_LEN]);

/* ---- row-partitioned batched Brandes for the multi-GPU driver --------------
 * betweenness.cpp:11-86 over 1D row blocks (one exchange per BFS
 * level).  Every rank holds the graph (AT cached) and calls, in lockstep:
 *   gbx_bc_shard_begin          owned rows [row_begin, row_end) (nnz-balanced),
 *                               replicated initial state for <= 4 sources;
 *   repeat: gbx_bc_shard_forward -> device records of the owned vertices this
 *           depth settled (40 bytes each: int32 v, uint32 lanes, fp64 sigma[4]);
 *           the driver all-gathers every rank's records in rank order;
 *           gbx_bc_shard_forward_apply(all records) -> *done once a depth is empty;
 *   repeat: gbx_bc_shard_backward -> records (int32 v, pad, fp64 coef[4]) of the
 *           owned vertices of the next depth, *done after depth 1;
 *           gbx_bc_shard_backward_apply(all records);
 *   gbx_bc_shard_centrality     device fp64[n]: this rank's partial (zero off its
 *                               rows); the sum over ranks (all-reduce) equals
 *                               gbx_betweenness (to the rounding of the hub rows'
 *                               fp64 atomics, which both runs share).
 * Record pointers are device memory owned by the handle (valid until the next
 * protocol call); applied record buffers are the caller's device memory. */
int gbx_bc_shard_begin(gbx_graph* g, const uint64_t* sources, uint64_t ns, int rank, int nranks,
                       int64_t* row_begin, int64_t* row_end, char msg[GBX_MSG_LEN]);
int gbx_bc_shard_forward(gbx_graph* g, void** recs_dev, int64_t* nrecs, char msg[GBX_MSG_LEN]);
int gbx_bc_shard_forward_apply(gbx_graph* g, const void* recs_dev, int64_t nrecs, int* done,
                               char msg[GBX_MSG_LEN]);
int gbx_bc_shard_backward(gbx_graph* g, void** recs_dev, int64_t* nrecs, int* done,
                          char msg[GBX_MSG_LEN]);
int gbx_bc_shard_backward_apply(gbx_graph* g, const void* recs_dev, int64_t nrecs,
                                char msg[GBX_MSG_LEN]);
int gbx_bc_shard_centrality(gbx_graph* g, double** cent_dev, char msg[GBX_MSG_LEN]);

/* ---- row-sharded single-source BFS for the multi-GPU driver ---------------
 * bfs.cpp:18-85 over 1D row blocks (scale >= 22): rank r owns the
 * 32-aligned block [row_begin, row_end) (balanced by AT nnz + rows).  Per level
 * every rank calls gbx_bfs_shard_level with the GLOBAL frontier bitmap (n bits,
 * device) and receives its slice of the next bitmap (words [row_begin/32,
 * ceil(row_end/32)), device) and the number of owned vertices it reached; the
 * driver all-gathers the slices (NCCL) and stops when no rank found any.
 * Owned vertices are pulled against the frontier: the first frontier
 * in-neighbour in the ascending AT row is the parent -- the minimum id, as in
 * gbx_bfs, whose results these equal.  gbx_bfs_shard_result copies the owned
 * rows' parent / level (-1 = unreached) to host arrays of row_end - row_begin. */
int gbx_bfs_shard_begin(gbx_graph* g, uint64_t source, int rank, int nranks, int64_t* row_begin,
                        int64_t* row_end, char msg[GBX_MSG_LEN]);
int gbx_bfs_shard_level(gbx_graph* g, const uint32_t* frontier_dev, uint32_t* next_slice_dev,
                        int64_t* found, char msg[GBX_MSG_LEN]);
int gbx_bfs_shard_result(gbx_graph* g, int64_t* parent, int64_t* level, char msg[GBX_MSG_LEN]);

/* ---- multi-GPU: communicator, distributed graph, algorithms ---------------
 * SURVEY.md §8e.  The reference is single-threaded (no counterpart); the
 * entry points mirror its algorithm signatures (algorithms.hpp:19-104) with a
 * distributed graph in place of the Graph, and every rank receives the same
 * full result the reference returns.
 *
 * Communicator: one NCCL rank per process / GPU (gbx_comm_init, the unique id
 * from gbx_comm_unique_id on one rank, passed to the others by the caller), or
 * nranks in-process ranks on ONE GPU (gbx_comm_init_local: the same protocols,
 * the exchange as device copies -- used to test the multi-rank paths on one
 * B200).  NCCL is bound at run time (the copy already loaded in the process,
 * else the system libnccl.so.2).  NCCL failures -> GBX_COMM_ERROR. */
#define GBX_COMM_ID_BYTES 128
typedef struct gbx_comm gbx_comm;
typedef struct gbx_dgraph gbx_dgraph;
int gbx_comm_unique_id(void* id, char msg[GBX_MSG_LEN]);
int gbx_comm_init(gbx_comm** comm, int nranks, int rank, const void* id, int device,
                  char msg[GBX_MSG_LEN]);
int gbx_comm_init_local(gbx_comm** comm, int nranks, int device, char msg[GBX_MSG_LEN]);
int gbx_comm_free(gbx_comm** comm, char msg[GBX_MSG_LEN]);
int gbx_comm_info(const gbx_comm* comm, int* nranks, int* rank, int* nlocal,
                  char msg[GBX_MSG_LEN]);

/* Distributed graph: rank q owns rows [b_q, b_{q+1}) (32-aligned, balanced by
 * rows + entries) of A -- and of AT for a directed graph -- and nothing else;
 * every rank builds its block LOCALLY (graph_new, graph.cpp:16-41, split over
 * the ranks): generated edges [q*m/P, (q+1)*m/P) of the seeded R-MAT stream
 * (the same graph as gbx_generate_rmat), or the CSR rows each rank passes
 * (host arrays, global column ids, int32), shuffled to their owners with one
 * all-to-all; self-loops dropped, duplicates combined (Bool pattern).
 * With a local communicator the block arrays have nlocal entries (one per
 * in-process rank), with NCCL one.  gbx_dgraph_block / _export_block read back
 * local rank `local`'s block (row_ptr: re - rb + 1 entries). */
int gbx_dgraph_generate_rmat(gbx_dgraph** g, gbx_comm* comm, int scale, int edge_factor,
                             double a, double b, double c, uint64_t seed, int scramble, int kind,
                             char msg[GBX_MSG_LEN]);
int gbx_dgraph_from_blocks(gbx_dgraph** g, gbx_comm* comm, int64_t n, const int64_t* row_begin,
                           const int64_t* row_end, const int64_t* const* row_ptr,
                           const int32_t* const* col, int kind, char msg[GBX_MSG_LEN]);
int gbx_dgraph_free(gbx_dgraph** g, char msg[GBX_MSG_LEN]);
int gbx_dgraph_info(const gbx_dgraph* g, int64_t* n, int64_t* nnz, int* kind,
                    char msg[GBX_MSG_LEN]);
int gbx_dgraph_block(const gbx_dgraph* g, int local, int64_t* row_begin, int64_t* row_end,
                     int64_t* nnz, char msg[GBX_MSG_LEN]);
int gbx_dgraph_export_block(const gbx_dgraph* g, int local, int64_t* row_ptr, int32_t* col,
                            char msg[GBX_MSG_LEN]);
int gbx_dgraph_last_stats(const gbx_dgraph* g, gbx_stats* stats, char msg[GBX_MSG_LEN]);

/* pagerank_gap (pagerank.cpp:8-81) over the ranks: 1D row blocks of the
 * in-degree-relabeled AT; exchange GBX_MG_P2P = fused into the iteration
 * kernel (peer stores over NVLink, device-side barrier bounded by option
 * p2p.timeout_ms), GBX_MG_NCCL = one all-gather of the x slices per iteration,
 * GBX_MG_AUTO = fused, falling back to NCCL on every rank when any rank's
 * fused run fails.  rank: n doubles (NULL: keep on the device). */
enum { GBX_MG_AUTO = 0, GBX_MG_NCCL = 1, GBX_MG_P2P = 2 };
int gbx_pagerank_mg(double* rank, int* iterations, gbx_dgraph* g, double damping, double tol,
                    int itermax, int exchange, char msg[GBX_MSG_LEN]);
/* triangle_count (triangle.cpp:30-64), undirected: U replicated, middle
 * vertices split by probe work, one u64 all-reduce. */
int gbx_triangle_count_mg(uint64_t* count, gbx_dgraph* g, char msg[GBX_MSG_LEN]);
/* bfs (bfs.cpp:18-85): parents / levels as gbx_bfs (n each, -1 unreached,
 * NULL allowed), pull levels over the owned rows + one frontier-bitmap
 * all-gather per level. */
int gbx_bfs_mg(int64_t* parent, int64_t* level, gbx_dgraph* g, uint64_t source,
               char msg[GBX_MSG_LEN]);
/* betweenness_centrality (betweenness.cpp:11-86): row-partitioned Brandes
 * in batches of 4 sources, one record all-gather per BFS level, one fp64
 * all-reduce of the centrality (n doubles, NULL allowed). */
int gbx_betweenness_mg(double* centrality, gbx_dgraph* g, const uint64_t* sources, uint64_t ns,
                       char msg[GBX_MSG_LEN]);

#ifdef __cplusplus
}
#endif
#endif /* GBX_H */
