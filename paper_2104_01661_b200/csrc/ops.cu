// ops.cu -- the GraphBLAS operation layer the paper's algorithms are written
// in (gblite core.hpp / core.cpp): mxv, vxm and mxm over the built-in
// semirings (ops.cpp:362-372), with the shared mask / accumulator / replace
// post-step (core.cpp:131-204), on the device.
//
// Values travel as 8-byte lanes (Bool as 0/1) tagged with the gblite domain;
// every operator mirrors ops.cpp exactly (wrapping integer arithmetic, Bool
// plus = or / times = and / min = and / max = or, fmin / fmax for Fp64,
// integer division by zero = 0, the any monoid keeps the first contribution).
// Every fold runs in the reference's order, so results are bit-exact --
// including Fp64 sums:
//   * mxv  (core.cpp:340-386): one thread per output row folds A(i,:) ∩ u in
//     ascending k against a dense staging of u;
//   * vxm  (core.cpp:308-338): the reference's push order gives every output
//     j its contributions in ascending k, which is the pull fold over the
//     column j of A (a device transpose of A, cached per matrix);
//   * mxm  (core.cpp:267-306): masked by a non-complemented mask -> one thread
//     per mask entry folds A(i,:) ∩ B(:,j) (dot form, the masked-SpGEMM of
//     triangle counting); otherwise expand-sort-reduce: the products are
//     generated in (i, k, j) order and stably radix-sorted by (i, j), so each
//     output run holds its contributions in ascending k and one thread folds
//     it -- the Gustavson DenseAcc order;
//   * post-step (merge_entries, core.cpp:131-175): vectors on dense
//     n-arrays, matrices as a stable key sort of prior (C) and result (T)
//     entries with the mask row probed by binary search.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "sort.cuh"

namespace gbx {

int bits_for(int64_t n);
void rowptr_from_sorted_keys(cudaStream_t s, int64_t n, int bits, const uint64_t* keys,
                             int64_t nnz, int64_t* rp, int32_t* col);

namespace {

constexpr int kT = 256;

// ---- scalar semantics (ops.cpp) -------------------------------------------------

__host__ __device__ inline uint64_t one_of(int d) {
  if (d == GBX_FP64) {
    const double o = 1.0;
    uint64_t b;
    memcpy(&b, &o, 8);
    return b;
  }
  return 1;
}

__host__ __device__ inline uint64_t any_identity(int d) {
  switch (d) {
    case GBX_BOOL: return 0;
    case GBX_INT64: return 0x8000000000000000ull;
    case GBX_UINT64: return ~0ull;
    default: return 0xFFF0000000000000ull;  // -inf
  }
}

__device__ __forceinline__ double as_f(uint64_t b) { return __longlong_as_double(static_cast<long long>(b)); }
__device__ __forceinline__ uint64_t of_f(double v) { return static_cast<uint64_t>(__double_as_longlong(v)); }

__device__ inline bool scalar_eq(int d, uint64_t x, uint64_t y) {
  if (d == GBX_FP64) return as_f(x) == as_f(y);
  if (d == GBX_BOOL) return (x != 0) == (y != 0);
  return x == y;
}

__device__ inline bool nonzero(int d, uint64_t x) {
  if (d == GBX_FP64) return as_f(x) != 0.0;
  return x != 0;
}

// z = op(x, y) in domain d (ops.cpp:52-203)
__device__ inline uint64_t bop(int op, int d, uint64_t x, uint64_t y) {
  const bool bx = x != 0, by = y != 0;
  const int64_t ix = static_cast<int64_t>(x), iy = static_cast<int64_t>(y);
  switch (op) {
    case GBX_OP_PLUS:
      if (d == GBX_BOOL) return bx || by;
      if (d == GBX_FP64) return of_f(as_f(x) + as_f(y));
      return x + y;  // wrapping for Int64 and Uint64 alike
    case GBX_OP_MINUS:
      if (d == GBX_BOOL) return bx != by;
      if (d == GBX_FP64) return of_f(as_f(x) - as_f(y));
      return x - y;
    case GBX_OP_TIMES:
      if (d == GBX_BOOL) return bx && by;
      if (d == GBX_FP64) return of_f(as_f(x) * as_f(y));
      return x * y;
    case GBX_OP_DIV:
      if (d == GBX_BOOL) return bx;
      if (d == GBX_FP64) return of_f(as_f(x) / as_f(y));
      if (d == GBX_INT64) {
        if (iy == 0) return 0;
        if (ix == INT64_MIN && iy == -1) return x;
        return static_cast<uint64_t>(ix / iy);
      }
      return y == 0 ? 0 : x / y;
    case GBX_OP_MIN:
      if (d == GBX_BOOL) return bx && by;
      if (d == GBX_FP64) return of_f(fmin(as_f(x), as_f(y)));
      if (d == GBX_INT64) return ix < iy ? x : y;
      return x < y ? x : y;
    case GBX_OP_MAX:
      if (d == GBX_BOOL) return bx || by;
      if (d == GBX_FP64) return of_f(fmax(as_f(x), as_f(y)));
      if (d == GBX_INT64) return ix > iy ? x : y;
      return x > y ? x : y;
    case GBX_OP_FIRST: return x;
    case GBX_OP_SECOND: return y;
    case GBX_OP_PAIR: return one_of(d);
    case GBX_OP_ANY: return scalar_eq(d, x, any_identity(d)) ? y : x;
    case GBX_OP_LOR: return bx || by;
    case GBX_OP_LAND: return bx && by;
  }
  return x;
}

struct Sr {
  int add;   // monoid operator
  int mult;  // multiplicative operator (GBX_OP_SECONDI: positional)
  int dom;   // output (and operand) domain
  bool use1, use2;
};

Sr semiring_of(int sr, int dom) {
  switch (sr) {
    case GBX_SR_PLUS_TIMES: return {GBX_OP_PLUS, GBX_OP_TIMES, dom, true, true};
    case GBX_SR_ANY_SECONDI: return {GBX_OP_ANY, GBX_OP_SECONDI, GBX_UINT64, false, false};
    case GBX_SR_MIN_PLUS: return {GBX_OP_MIN, GBX_OP_PLUS, dom, true, true};
    case GBX_SR_PLUS_FIRST: return {GBX_OP_PLUS, GBX_OP_FIRST, dom, true, false};
    case GBX_SR_PLUS_SECOND: return {GBX_OP_PLUS, GBX_OP_SECOND, dom, false, true};
    case GBX_SR_PLUS_PAIR: return {GBX_OP_PLUS, GBX_OP_PAIR, dom, false, false};
    case GBX_SR_MIN_SECOND: return {GBX_OP_MIN, GBX_OP_SECOND, dom, false, true};
  }
  fail(GBX_INVALID_VALUE, "unknown semiring " + std::to_string(sr));
}

__device__ __forceinline__ uint64_t mult(const Sr& s, uint64_t x, uint64_t y, int64_t k) {
  return s.mult == GBX_OP_SECONDI ? static_cast<uint64_t>(k) : bop(s.mult, s.dom, x, y);
}

const char* dname(int d) {
  switch (d) {
    case GBX_BOOL: return "bool";
    case GBX_INT64: return "int64";
    case GBX_UINT64: return "uint64";
    case GBX_FP64: return "fp64";
  }
  return "?";
}

void check_domain(int d) {
  if (d < GBX_BOOL || d > GBX_FP64) fail(GBX_DOMAIN_MISMATCH, "unknown domain " + std::to_string(d));
}

// check_op_inputs (core.cpp:64-73)
void check_inputs(const Sr& s, int d1, int d2, const char* what) {
  if (s.use1 && s.dom != d1)
    fail(GBX_DOMAIN_MISMATCH, std::string(what) + ": first input is " + dname(d1) + ", expects " +
                                  dname(s.dom));
  if (s.use2 && s.dom != d2)
    fail(GBX_DOMAIN_MISMATCH, std::string(what) + ": second input is " + dname(d2) +
                                  ", expects " + dname(s.dom));
}

// check_accum (core.cpp:75-80): value operators over the target's domain
void check_accum(int accum, int accum_dom, int cdom) {
  if (accum == GBX_OP_NONE) return;
  if (accum < GBX_OP_PLUS || accum > GBX_OP_LAND) fail(GBX_INVALID_VALUE, "unknown accumulator");
  check_domain(accum_dom);
  const int ad = (accum == GBX_OP_LOR || accum == GBX_OP_LAND) ? GBX_BOOL : accum_dom;
  // every accumulator's output domain is its operand domain, which must be
  // the target's (the used inputs are checked against the same domain)
  if (ad != cdom) fail(GBX_DOMAIN_MISMATCH, "accumulator domain differs from the target");
}

// ---- host <-> device lanes -------------------------------------------------------

__global__ void k_widen(const uint8_t* src, int es, int64_t m, uint64_t* dst) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p >= m) return;
  if (es == 1) dst[p] = src[p] != 0;
  else dst[p] = reinterpret_cast<const uint64_t*>(src)[p];
}

__global__ void k_widen_i32(const int32_t* src, int64_t m, uint64_t* dst) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p < m) dst[p] = static_cast<uint64_t>(static_cast<int64_t>(src[p]));
}

__global__ void k_narrow(const uint64_t* src, int64_t m, uint8_t* dst) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p < m) dst[p] = src[p] != 0;
}

__global__ void k_fill(uint64_t* v, int64_t m, uint64_t x) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p < m) v[p] = x;
}

__global__ void k_cols64(const int64_t* c64, int64_t m, int64_t ncols, int32_t* c32, int* bad) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p >= m) return;
  const int64_t c = c64[p];
  if (c < 0 || c >= ncols) { atomicOr(bad, 2); c32[p] = 0; return; }
  c32[p] = static_cast<int32_t>(c);
}

__global__ void k_check_rows(const int64_t* rp, const int32_t* col, int64_t n, int64_t nnz, int* bad) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i > n) return;
  if (i == 0 && rp[0] != 0) atomicOr(bad, 1);
  if (i == n) { if (rp[n] != nnz) atomicOr(bad, 1); return; }
  const int64_t b = rp[i], e = rp[i + 1];
  if (b > e || b < 0 || e > nnz) { atomicOr(bad, 1); return; }
  for (int64_t p = b + 1; p < e; ++p)
    if (col[p - 1] >= col[p]) { atomicOr(bad, 4); return; }
}

size_t esize(int d) { return d == GBX_BOOL ? 1 : 8; }

// dense staging of a host sparse vector: present[n], val[n]
struct DenseVec {
  int64_t n = 0;
  int dom = GBX_BOOL;
  DevArray<uint8_t> has;
  DevArray<uint64_t> val;
};

__global__ void k_scatter_vec(const int64_t* idx, const uint64_t* v, int64_t m, int64_t n,
                              uint8_t* has, uint64_t* val, int* bad) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p >= m) return;
  const int64_t i = idx[p];
  if (i < 0 || i >= n || (p > 0 && idx[p - 1] >= i)) { atomicOr(bad, 1); return; }
  has[i] = 1;
  val[i] = v[p];
}

void stage_vec(cudaStream_t s, const gbx_vec* h, DenseVec& d) {
  d.n = h->n;
  d.dom = h->domain;
  check_domain(h->domain);
  if (h->nvals < 0 || h->nvals > h->n) fail(GBX_INVALID_MATRIX, "vector nvals out of range");
  if (h->nvals && (!h->idx || !h->vals)) fail(GBX_NULL_ARGUMENT, "vector arrays are NULL");
  const int64_t n1 = std::max<int64_t>(h->n, 1);
  d.has.alloc(n1);
  d.val.alloc(n1);
  GBX_CUDA(cudaMemsetAsync(d.has.p, 0, n1, s));
  if (h->nvals == 0) return;
  const int64_t m = h->nvals;
  Tmp<int64_t> ix(m, s);
  Tmp<uint8_t> raw(m * esize(h->domain), s);
  Tmp<uint64_t> v(m, s);
  Tmp<int> bad(1, s);
  GBX_CUDA(cudaMemsetAsync(bad.p, 0, 4, s));
  GBX_CUDA(cudaMemcpyAsync(ix.p, h->idx, m * 8, cudaMemcpyHostToDevice, s));
  GBX_CUDA(cudaMemcpyAsync(raw.p, h->vals, m * esize(h->domain), cudaMemcpyHostToDevice, s));
  k_widen<<<ceil_div(m, kT), kT, 0, s>>>(raw.p, static_cast<int>(esize(h->domain)), m, v.p);
  k_scatter_vec<<<ceil_div(m, kT), kT, 0, s>>>(ix.p, v.p, m, h->n, d.has.p, d.val.p, bad.p);
  GBX_LAUNCHED();
  int hb = 0;
  GBX_CUDA(cudaMemcpyAsync(&hb, bad.p, 4, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  if (hb) fail(GBX_INVALID_MATRIX, "vector indices out of range or not strictly increasing");
}

// ---- transpose with values (plain_transpose, core.cpp:237-256) ------------------

__global__ void k_tkeys(const int64_t* rp, const int32_t* col, int64_t nrows, int bits,
                        uint64_t* keys, int64_t* pos) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= nrows) return;
  for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
    keys[p] = (static_cast<uint64_t>(col[p]) << bits) | static_cast<uint64_t>(i);
    pos[p] = p;
  }
}

__global__ void k_gather_u64(const uint64_t* src, const int64_t* pos, int64_t m, uint64_t* dst) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p < m) dst[p] = src[pos[p]];
}

void ensure_transpose(gbx_mat* A) {
  if (A->has_t) return;
  cudaStream_t s = A->stream;
  const int64_t m = A->nnz;
  const int bits = bits_for(std::max<int64_t>(std::max(A->nrows, A->ncols), 2));
  A->trp.alloc(A->ncols + 1);
  A->tcol.alloc(std::max<int64_t>(m, 1));
  A->tval.alloc(std::max<int64_t>(m, 1));
  if (m == 0) {
    GBX_CUDA(cudaMemsetAsync(A->trp.p, 0, (A->ncols + 1) * 8, s));
  } else {
    Tmp<uint64_t> k0(m, s), k1(m, s);
    Tmp<int64_t> p0(m, s), p1(m, s);
    k_tkeys<<<ceil_div(A->nrows, kT), kT, 0, s>>>(A->rp.p, A->col.p, A->nrows, bits, k0.p, p0.p);
    GBX_LAUNCHED();
    cub::DoubleBuffer<uint64_t> kb(k0.p, k1.p);
    cub::DoubleBuffer<int64_t> pb(p0.p, p1.p);
    radix_sort_pairs(s, kb, pb, m, 0, 2 * bits);
    rowptr_from_sorted_keys(s, A->ncols, bits, kb.Current(), m, A->trp.p, A->tcol.p);
    k_gather_u64<<<ceil_div(m, kT), kT, 0, s>>>(A->val.p, pb.Current(), m, A->tval.p);
    GBX_LAUNCHED();
  }
  GBX_CUDA(cudaStreamSynchronize(s));
  A->has_t = true;
}

struct View {  // CSR operand (A or its transpose)
  int64_t nrows, ncols;
  const int64_t* rp;
  const int32_t* col;
  const uint64_t* val;
};

View view(gbx_mat* A, bool t) {
  if (!t) return {A->nrows, A->ncols, A->rp.p, A->col.p, A->val.p};
  ensure_transpose(A);
  return {A->ncols, A->nrows, A->trp.p, A->tcol.p, A->tval.p};
}

// ---- mxv / vxm ------------------------------------------------------------------

// T(i) = fold over A(i,:) ∩ u in ascending k.  swap: the multiply takes
// (u(k), A(k,i)) -- vxm through the transpose.
__global__ void k_pull(View A, const uint8_t* uh, const uint64_t* uv, Sr s, int swap,
                       uint8_t* th, uint64_t* tv) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= A.nrows) return;
  bool hit = false;
  uint64_t acc = 0;
  for (int64_t p = A.rp[i]; p < A.rp[i + 1]; ++p) {
    const int32_t k = A.col[p];
    if (!uh[k]) continue;
    const uint64_t v = swap ? mult(s, uv[k], A.val[p], k) : mult(s, A.val[p], uv[k], k);
    acc = hit ? bop(s.add, s.dom, acc, v) : v;
    hit = true;
  }
  th[i] = hit;
  if (hit) tv[i] = acc;
}

// merge_entries (core.cpp:131-175) for a vector, dense over n positions
__global__ void k_post_vec(int64_t n, const uint8_t* ch, const uint64_t* cv, const uint8_t* th,
                           const uint64_t* tv, const uint8_t* mh, const uint64_t* mv, int mdom,
                           int has_mask, int comp, int structural, int replace, int accum,
                           int cdom, uint8_t* oh, uint64_t* ov) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p >= n) return;
  bool in = true;
  if (has_mask) {
    in = mh[p] && (structural || nonzero(mdom, mv[p]));
    in = in != (comp != 0);
  }
  const bool hc = ch[p], ht = th[p];
  bool out = false;
  uint64_t v = 0;
  if (in) {
    if (ht) {
      out = true;
      v = (hc && accum != GBX_OP_NONE) ? bop(accum, cdom, cv[p], tv[p]) : tv[p];
    } else if (hc) {
      out = true;
      v = cv[p];
    }
  } else if (hc && !replace) {
    out = true;
    v = cv[p];
  }
  oh[p] = out;
  ov[p] = v;
}

__global__ void k_iota64(int64_t* a, int64_t n) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) a[i] = i;
}

void vec_op(int64_t* w_idx, void* w_vals, int64_t* w_nvals, const gbx_vec* w,
            const gbx_desc* desc, int sr, int sdom, gbx_mat* A, const gbx_vec* u, bool is_vxm) {
  if (!A || !u || !w || !w_nvals) fail(GBX_NULL_ARGUMENT, "vector op: NULL argument");
  check_domain(sdom);
  const Sr s = semiring_of(sr, sdom);
  const gbx_desc d0{};
  const gbx_desc& d = desc ? *desc : d0;
  // alias checks (core.cpp:36-40): the output may not be an input
  if (w == u || (d.mask_vec && d.mask_vec == w)) fail(GBX_ALIASED_OUTPUT, "output container aliases an input");
  const bool tr = is_vxm ? d.transpose_in2 != 0 : d.transpose_in1 != 0;
  // operand shapes: mxv T = A u (A: n x m, u: m); vxm T = u A (u: n, A: n x m)
  const int64_t arows = tr ? A->ncols : A->nrows, acols = tr ? A->nrows : A->ncols;
  if (is_vxm) {
    if (u->n != arows) fail(GBX_DIMENSION_MISMATCH, "vxm vector length does not match rows");
    if (w->n != acols) fail(GBX_DIMENSION_MISMATCH, "vxm output length");
    check_inputs(s, u->domain, A->domain, "vxm");
  } else {
    if (acols != u->n) fail(GBX_DIMENSION_MISMATCH, "mxv vector length does not match columns");
    if (w->n != arows) fail(GBX_DIMENSION_MISMATCH, "mxv output length");
    check_inputs(s, A->domain, u->domain, "mxv");
  }
  if (w->domain != s.dom)
    fail(GBX_DOMAIN_MISMATCH, std::string(is_vxm ? "vxm" : "mxv") + ": output container is " +
                                  dname(w->domain) + ", result is " + dname(s.dom));
  // post-step checks (core.cpp:177-179)
  if (d.mask_mat) fail(GBX_DIMENSION_MISMATCH, "vector operation given a matrix mask");
  if (d.mask_vec && d.mask_vec->n != w->n) fail(GBX_DIMENSION_MISMATCH, "mask length does not match output");
  check_accum(d.accum, d.accum_domain, w->domain);
  cudaStream_t st = A->stream;
  DenseVec U, C, M;
  stage_vec(st, u, U);
  stage_vec(st, w, C);
  if (d.mask_vec) stage_vec(st, d.mask_vec, M);
  // T: vxm pulls over the columns of A (rows of its transpose)
  const View V = view(A, is_vxm ? !tr : tr);
  const int64_t n = w->n, n1 = std::max<int64_t>(n, 1);
  Tmp<uint8_t> th(n1, st), oh(n1, st);
  Tmp<uint64_t> tv(n1, st), ov(n1, st);
  if (n > 0) {
    k_pull<<<ceil_div(n, kT), kT, 0, st>>>(V, U.has.p, U.val.p, s, is_vxm ? 1 : 0, th.p, tv.p);
    GBX_LAUNCHED();
    k_post_vec<<<ceil_div(n, kT), kT, 0, st>>>(
        n, C.has.p, C.val.p, th.p, tv.p, d.mask_vec ? M.has.p : nullptr,
        d.mask_vec ? M.val.p : nullptr, d.mask_vec ? d.mask_vec->domain : 0, d.mask_vec != nullptr,
        d.complement, d.structural, d.replace, d.accum, w->domain, oh.p, ov.p);
    GBX_LAUNCHED();
  }
  // compaction: ascending indices with their values
  Tmp<int64_t> iota(n1, st), oi(n1, st);
  Tmp<uint64_t> ovc(n1, st);
  Tmp<int64_t> cnt(1, st);
  int64_t nv = 0;
  if (n > 0) {
    k_iota64<<<ceil_div(n, kT), kT, 0, st>>>(iota.p, n);
    GBX_LAUNCHED();
    size_t tb = 0;
    GBX_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota.p, oh.p, oi.p, cnt.p, n, st));
    {
      Tmp<uint8_t> t(tb, st);
      GBX_CUDA(cub::DeviceSelect::Flagged(t.p, tb, iota.p, oh.p, oi.p, cnt.p, n, st));
    }
    tb = 0;
    GBX_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, ov.p, oh.p, ovc.p, cnt.p, n, st));
    {
      Tmp<uint8_t> t(tb, st);
      GBX_CUDA(cub::DeviceSelect::Flagged(t.p, tb, ov.p, oh.p, ovc.p, cnt.p, n, st));
    }
    GBX_CUDA(cudaMemcpyAsync(&nv, cnt.p, 8, cudaMemcpyDeviceToHost, st));
    GBX_CUDA(cudaStreamSynchronize(st));
  }
  *w_nvals = nv;
  if (nv > 0) {
    if (w_idx) GBX_CUDA(cudaMemcpyAsync(w_idx, oi.p, nv * 8, cudaMemcpyDeviceToHost, st));
    if (w_vals) {
      if (w->domain == GBX_BOOL) {
        Tmp<uint8_t> nb(nv, st);
        k_narrow<<<ceil_div(nv, kT), kT, 0, st>>>(ovc.p, nv, nb.p);
        GBX_LAUNCHED();
        GBX_CUDA(cudaMemcpyAsync(w_vals, nb.p, nv, cudaMemcpyDeviceToHost, st));
        GBX_CUDA(cudaStreamSynchronize(st));
      } else {
        GBX_CUDA(cudaMemcpyAsync(w_vals, ovc.p, nv * 8, cudaMemcpyDeviceToHost, st));
      }
    }
  }
  GBX_CUDA(cudaStreamSynchronize(st));
}

// ---- mxm -------------------------------------------------------------------------

// products per row of A: sum over k in A(i,:) of nnz(B(k,:))
__global__ void k_row_products(View A, View B, int64_t* cnt) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= A.nrows) return;
  int64_t c = 0;
  for (int64_t p = A.rp[i]; p < A.rp[i + 1]; ++p) {
    const int32_t k = A.col[p];
    c += B.rp[k + 1] - B.rp[k];
  }
  cnt[i] = c;
}

// expand row i's products in (k ascending, j ascending) order
__global__ void k_expand(View A, View B, const int64_t* off, Sr s, int bits, uint64_t* keys,
                         uint64_t* vals) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= A.nrows) return;
  int64_t q = off[i];
  for (int64_t p = A.rp[i]; p < A.rp[i + 1]; ++p) {
    const int32_t k = A.col[p];
    for (int64_t r = B.rp[k]; r < B.rp[k + 1]; ++r) {
      const int32_t j = B.col[r];
      keys[q] = (static_cast<uint64_t>(i) << bits) | static_cast<uint64_t>(j);
      vals[q] = mult(s, A.val[p], B.val[r], k);
      ++q;
    }
  }
}

__global__ void k_heads64(const uint64_t* keys, int64_t m, int32_t* head) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p < m) head[p] = (p == 0 || keys[p] != keys[p - 1]) ? 1 : 0;
}

__global__ void k_runs(const uint64_t* keys, const int32_t* head, const int64_t* seg, int64_t m,
                       uint64_t* ukeys, int64_t* start) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p >= m || !head[p]) return;
  ukeys[seg[p] - 1] = keys[p];
  start[seg[p] - 1] = p;
}

// fold each (i, j) run in generation (= ascending k) order
__global__ void k_fold_runs(const uint64_t* vals, const int64_t* start, int64_t nu, int64_t m,
                            Sr s, uint64_t* out) {
  const int64_t u = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (u >= nu) return;
  const int64_t b = start[u], e = u + 1 < nu ? start[u + 1] : m;
  uint64_t acc = vals[b];
  for (int64_t p = b + 1; p < e; ++p) acc = bop(s.add, s.dom, acc, vals[p]);
  out[u] = acc;
}

// masked dot form: one thread per mask entry (i, j) in the mask's structure;
// inactive entries (valued mask with a zero) produce nothing
__global__ void k_dot(View A, View BT, const int64_t* mrp, const int32_t* mcol, const uint64_t* mval,
                      int mdom, int structural, int64_t mrows, int bits, Sr s, uint64_t* keys,
                      uint64_t* vals, uint8_t* hit) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= mrows) return;
  for (int64_t q = mrp[i]; q < mrp[i + 1]; ++q) {
    const int32_t j = mcol[q];
    keys[q] = (static_cast<uint64_t>(i) << bits) | static_cast<uint64_t>(j);
    hit[q] = 0;
    if (!structural && !nonzero(mdom, mval[q])) continue;
    int64_t a = A.rp[i], ae = A.rp[i + 1], b = BT.rp[j], be = BT.rp[j + 1];
    bool h = false;
    uint64_t acc = 0;
    while (a < ae && b < be) {
      const int32_t ka = A.col[a], kb = BT.col[b];
      if (ka < kb) ++a;
      else if (ka > kb) ++b;
      else {
        const uint64_t v = mult(s, A.val[a], BT.val[b], ka);
        acc = h ? bop(s.add, s.dom, acc, v) : v;
        h = true;
        ++a;
        ++b;
      }
    }
    hit[q] = h;
    vals[q] = acc;
  }
}

// matrix post-step: merged (key, source) list of prior C (src 0) and T (src 1)
// entries, sorted by key with C first; one thread per distinct key
__global__ void k_mkeys(const int64_t* rp, const int32_t* col, int64_t nrows, int bits, int tag,
                        uint64_t* keys, int64_t* ref, int64_t base) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= nrows) return;
  for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
    keys[base + p] = (static_cast<uint64_t>(i) << bits) | static_cast<uint64_t>(col[p]);
    ref[base + p] = (p << 1) | tag;
  }
}

// T entry q of the merged list: reference (q << 1) | 1
__global__ void k_tref(int64_t* r, int64_t n) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) r[i] = (i << 1) | 1;
}

__device__ bool mask_member(const int64_t* mrp, const int32_t* mcol, const uint64_t* mval,
                            int mdom, int structural, int comp, int64_t i, int32_t j) {
  int64_t lo = mrp[i], hi = mrp[i + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (mcol[mid] < j) lo = mid + 1; else hi = mid;
  }
  bool in = lo < mrp[i + 1] && mcol[lo] == j && (structural || nonzero(mdom, mval[lo]));
  return in != (comp != 0);
}

__global__ void k_post_mat(const uint64_t* keys, const int64_t* ref, int64_t m, int bits,
                           const uint64_t* cval, const uint64_t* tval, const int64_t* mrp,
                           const int32_t* mcol, const uint64_t* mval, int mdom, int has_mask,
                           int structural, int comp, int replace, int accum, int cdom,
                           uint8_t* keep, uint64_t* outv) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p >= m) return;
  keep[p] = 0;
  if (p > 0 && keys[p - 1] == keys[p]) return;  // the run's first thread decides
  const bool two = p + 1 < m && keys[p + 1] == keys[p];
  bool hc = false, ht = false;
  int64_t pc = 0, pt = 0;
  for (int t = 0; t < (two ? 2 : 1); ++t) {
    const int64_t r = ref[p + t];
    if (r & 1) { ht = true; pt = r >> 1; } else { hc = true; pc = r >> 1; }
  }
  const int64_t i = static_cast<int64_t>(keys[p] >> bits);
  const int32_t j = static_cast<int32_t>(keys[p] & ((1ull << bits) - 1));
  const bool in = has_mask ? mask_member(mrp, mcol, mval, mdom, structural, comp, i, j) : true;
  bool out = false;
  uint64_t v = 0;
  if (in) {
    if (ht) {
      out = true;
      v = (hc && accum != GBX_OP_NONE) ? bop(accum, cdom, cval[pc], tval[pt]) : tval[pt];
    } else if (hc) {
      out = true;
      v = cval[pc];
    }
  } else if (hc && !replace) {
    out = true;
    v = cval[pc];
  }
  keep[p] = out;
  outv[p] = v;
}

}  // namespace

gbx_mat* mat_alloc() {
  auto* m = new gbx_mat();
  cudaError_t e = cudaGetDevice(&m->device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete m;
    fail(GBX_CUDA_ERROR, std::string("no CUDA device: ") + cudaGetErrorString(e));
  }
  return m;
}

// SparseMatrix + validate (containers.cpp:104-124) from host CSR
void mat_from_host(gbx_mat* M, int64_t nrows, int64_t ncols, const int64_t* rp, const int64_t* col,
                   const void* vals, int domain) {
  check_domain(domain);
  if (nrows < 0 || ncols < 0) fail(GBX_INVALID_MATRIX, "negative dimension");
  if (std::max(nrows, ncols) >= (int64_t(1) << 31) - 1)
    fail(GBX_UNSUPPORTED, "dimensions >= 2^31 are not supported by the int32 column layout");
  if (!rp) fail(GBX_NULL_ARGUMENT, "row_ptr is NULL");
  const int64_t m = rp[nrows];
  if (m < 0) fail(GBX_INVALID_MATRIX, "row_ptr[nrows] is negative");
  if (m && (!col || !vals)) fail(GBX_NULL_ARGUMENT, "col / vals is NULL");
  cudaStream_t s = M->stream;
  M->nrows = nrows;
  M->ncols = ncols;
  M->nnz = m;
  M->domain = domain;
  M->rp.alloc(nrows + 1);
  M->col.alloc(std::max<int64_t>(m, 1));
  M->val.alloc(std::max<int64_t>(m, 1));
  GBX_CUDA(cudaMemcpyAsync(M->rp.p, rp, (nrows + 1) * 8, cudaMemcpyHostToDevice, s));
  Tmp<int> bad(1, s);
  GBX_CUDA(cudaMemsetAsync(bad.p, 0, 4, s));
  if (m) {
    Tmp<int64_t> c64(m, s);
    Tmp<uint8_t> raw(m * esize(domain), s);
    GBX_CUDA(cudaMemcpyAsync(c64.p, col, m * 8, cudaMemcpyHostToDevice, s));
    GBX_CUDA(cudaMemcpyAsync(raw.p, vals, m * esize(domain), cudaMemcpyHostToDevice, s));
    k_cols64<<<ceil_div(m, kT), kT, 0, s>>>(c64.p, m, ncols, M->col.p, bad.p);
    k_widen<<<ceil_div(m, kT), kT, 0, s>>>(raw.p, static_cast<int>(esize(domain)), m, M->val.p);
    GBX_LAUNCHED();
  }
  k_check_rows<<<ceil_div(nrows + 1, kT), kT, 0, s>>>(M->rp.p, M->col.p, nrows, m, bad.p);
  GBX_LAUNCHED();
  int hb = 0;
  GBX_CUDA(cudaMemcpyAsync(&hb, bad.p, 4, cudaMemcpyDeviceToHost, s));
  GBX_CUDA(cudaStreamSynchronize(s));
  if (hb & 1) fail(GBX_INVALID_MATRIX, "row_ptr is not a valid prefix of nvals");
  if (hb & 2) fail(GBX_INVALID_MATRIX, "column index out of range");
  if (hb & 4) fail(GBX_INVALID_MATRIX, "row columns not strictly increasing");
}

// a graph's A (or cached AT) as an operand; pattern graphs are Bool true,
// int32 weights widen to Int64
void mat_from_graph(gbx_mat* M, gbx_graph* g, int which) {
  if (which == 1) require_at(g, "gbx_graph_mat");
  const Csr& A = which == 1 ? g->AT() : g->A;
  cudaStream_t s = M->stream;
  const int64_t m = A.nnz;
  M->nrows = M->ncols = A.n;
  M->nnz = m;
  M->domain = A.domain == GBX_INT32 ? GBX_INT64 : A.domain;
  M->rp.alloc(A.n + 1);
  M->col.alloc(std::max<int64_t>(m, 1));
  M->val.alloc(std::max<int64_t>(m, 1));
  GBX_CUDA(cudaStreamSynchronize(g->stream));
  GBX_CUDA(cudaMemcpyAsync(M->rp.p, A.rp.p, (A.n + 1) * 8, cudaMemcpyDeviceToDevice, s));
  if (m) {
    GBX_CUDA(cudaMemcpyAsync(M->col.p, A.col.p, m * 4, cudaMemcpyDeviceToDevice, s));
    if (!A.val.p) k_fill<<<ceil_div(m, kT), kT, 0, s>>>(M->val.p, m, 1);
    else if (A.domain == GBX_INT32)
      k_widen_i32<<<ceil_div(m, kT), kT, 0, s>>>(reinterpret_cast<const int32_t*>(A.val.p), m, M->val.p);
    else k_widen<<<ceil_div(m, kT), kT, 0, s>>>(A.val.p, static_cast<int>(esize(A.domain)), m, M->val.p);
    GBX_LAUNCHED();
  }
  GBX_CUDA(cudaStreamSynchronize(s));
}

void mat_export(gbx_mat* M, int64_t* rp, int64_t* col, void* vals) {
  cudaStream_t s = M->stream;
  if (rp) GBX_CUDA(cudaMemcpyAsync(rp, M->rp.p, (M->nrows + 1) * 8, cudaMemcpyDeviceToHost, s));
  if (M->nnz && col) {
    std::vector<int32_t> c(M->nnz);
    GBX_CUDA(cudaMemcpyAsync(c.data(), M->col.p, M->nnz * 4, cudaMemcpyDeviceToHost, s));
    GBX_CUDA(cudaStreamSynchronize(s));
    for (int64_t p = 0; p < M->nnz; ++p) col[p] = c[p];
  }
  if (M->nnz && vals) {
    if (M->domain == GBX_BOOL) {
      Tmp<uint8_t> nb(M->nnz, s);
      k_narrow<<<ceil_div(M->nnz, kT), kT, 0, s>>>(M->val.p, M->nnz, nb.p);
      GBX_LAUNCHED();
      GBX_CUDA(cudaMemcpyAsync(vals, nb.p, M->nnz, cudaMemcpyDeviceToHost, s));
      GBX_CUDA(cudaStreamSynchronize(s));
    } else {
      GBX_CUDA(cudaMemcpyAsync(vals, M->val.p, M->nnz * 8, cudaMemcpyDeviceToHost, s));
    }
  }
  GBX_CUDA(cudaStreamSynchronize(s));
}

void mxv_op(int64_t* w_idx, void* w_vals, int64_t* w_nvals, const gbx_vec* w, const gbx_desc* d,
            int sr, int sdom, gbx_mat* A, const gbx_vec* u) {
  NvtxRange nvtx_("gbx.mxv");
  vec_op(w_idx, w_vals, w_nvals, w, d, sr, sdom, A, u, false);
}
void vxm_op(int64_t* w_idx, void* w_vals, int64_t* w_nvals, const gbx_vec* w, const gbx_desc* d,
            int sr, int sdom, const gbx_vec* u, gbx_mat* A) {
  NvtxRange nvtx_("gbx.vxm");
  vec_op(w_idx, w_vals, w_nvals, w, d, sr, sdom, A, u, true);
}

// C_out = post_step(C, T = A ⊕.⊗ B) (mxm, core.cpp:267-306)
void mxm_op(gbx_mat* out, gbx_mat* C, const gbx_desc* desc, int sr, int sdom, gbx_mat* A,
            gbx_mat* B) {
  NvtxRange nvtx_("gbx.mxm");
  check_domain(sdom);
  const Sr s = semiring_of(sr, sdom);
  const gbx_desc d0{};
  const gbx_desc& d = desc ? *desc : d0;
  if (C == A || C == B || (d.mask_mat && d.mask_mat == C))
    fail(GBX_ALIASED_OUTPUT, "output container aliases an input");
  const View Av = view(A, d.transpose_in1 != 0);
  const View Bv = view(B, d.transpose_in2 != 0);
  if (Av.ncols != Bv.nrows) fail(GBX_DIMENSION_MISMATCH, "mxm inner dimensions disagree");
  if (C->nrows != Av.nrows || C->ncols != Bv.ncols) fail(GBX_DIMENSION_MISMATCH, "mxm output shape");
  check_inputs(s, A->domain, B->domain, "mxm");
  if (C->domain != s.dom)
    fail(GBX_DOMAIN_MISMATCH, std::string("mxm: output container is ") + dname(C->domain) +
                                  ", result is " + dname(s.dom));
  if (d.mask_vec) fail(GBX_DIMENSION_MISMATCH, "matrix operation given a vector mask");
  gbx_mat* Mk = const_cast<gbx_mat*>(d.mask_mat);
  if (Mk && (Mk->nrows != C->nrows || Mk->ncols != C->ncols))
    fail(GBX_DIMENSION_MISMATCH, "mask shape does not match output");
  check_accum(d.accum, d.accum_domain, C->domain);
  cudaStream_t st = A->stream;
  GBX_CUDA(cudaStreamSynchronize(B->stream));
  GBX_CUDA(cudaStreamSynchronize(C->stream));
  if (Mk) GBX_CUDA(cudaStreamSynchronize(Mk->stream));
  const int64_t nr = C->nrows, nc = C->ncols;
  const int bits = bits_for(std::max<int64_t>(std::max(nr, nc), 2));
  // ---- T as sorted unique (i, j) keys + values
  int64_t nt = 0;
  DevArray<uint64_t> tkeys, tvals;
  if (Mk && !d.complement) {
    // dot form over the mask's structure (entries outside it cannot be written)
    const View BT = view(B, d.transpose_in2 == 0);
    const int64_t mm = Mk->nnz;
    Tmp<uint64_t> k(std::max<int64_t>(mm, 1), st), v(std::max<int64_t>(mm, 1), st);
    Tmp<uint8_t> h(std::max<int64_t>(mm, 1), st);
    Tmp<int64_t> cnt(1, st);
    if (mm && nr) {
      k_dot<<<ceil_div(nr, kT), kT, 0, st>>>(Av, BT, Mk->rp.p, Mk->col.p, Mk->val.p, Mk->domain,
                                            d.structural, nr, bits, s, k.p, v.p, h.p);
      GBX_LAUNCHED();
      tkeys.alloc(mm);
      tvals.alloc(mm);
      size_t tb = 0;
      GBX_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, k.p, h.p, tkeys.p, cnt.p, mm, st));
      {
        Tmp<uint8_t> t(tb, st);
        GBX_CUDA(cub::DeviceSelect::Flagged(t.p, tb, k.p, h.p, tkeys.p, cnt.p, mm, st));
      }
      tb = 0;
      GBX_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, v.p, h.p, tvals.p, cnt.p, mm, st));
      {
        Tmp<uint8_t> t(tb, st);
        GBX_CUDA(cub::DeviceSelect::Flagged(t.p, tb, v.p, h.p, tvals.p, cnt.p, mm, st));
      }
      GBX_CUDA(cudaMemcpyAsync(&nt, cnt.p, 8, cudaMemcpyDeviceToHost, st));
      GBX_CUDA(cudaStreamSynchronize(st));
    }
  } else if (nr) {
    // expand-sort-reduce
    Tmp<int64_t> rc(nr, st), off(nr + 1, st);
    k_row_products<<<ceil_div(nr, kT), kT, 0, st>>>(Av, Bv, rc.p);
    GBX_LAUNCHED();
    GBX_CUDA(cudaMemsetAsync(off.p, 0, 8, st));
    size_t tb = 0;
    GBX_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, rc.p, off.p + 1, nr, st));
    {
      Tmp<uint8_t> t(tb, st);
      GBX_CUDA(cub::DeviceScan::InclusiveSum(t.p, tb, rc.p, off.p + 1, nr, st));
    }
    int64_t np = 0;
    GBX_CUDA(cudaMemcpyAsync(&np, off.p + nr, 8, cudaMemcpyDeviceToHost, st));
    GBX_CUDA(cudaStreamSynchronize(st));
    if (np > (int64_t(1) << 31)) fail(GBX_OUT_OF_MEMORY, "mxm: " + std::to_string(np) +
                                                            " products exceed the expansion budget");
    if (np) {
      Tmp<uint64_t> k0(np, st), k1(np, st), v0(np, st), v1(np, st);
      k_expand<<<ceil_div(nr, kT), kT, 0, st>>>(Av, Bv, off.p, s, bits, k0.p, v0.p);
      GBX_LAUNCHED();
      cub::DoubleBuffer<uint64_t> kb(k0.p, k1.p), vb(v0.p, v1.p);
      radix_sort_pairs(st, kb, vb, np, 0, 2 * bits);
      Tmp<int32_t> head(np, st);
      Tmp<int64_t> seg(np, st);
      k_heads64<<<ceil_div(np, kT), kT, 0, st>>>(kb.Current(), np, head.p);
      GBX_LAUNCHED();
      tb = 0;
      GBX_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, head.p, seg.p, np, st));
      {
        Tmp<uint8_t> t(tb, st);
        GBX_CUDA(cub::DeviceScan::InclusiveSum(t.p, tb, head.p, seg.p, np, st));
      }
      GBX_CUDA(cudaMemcpyAsync(&nt, seg.p + np - 1, 8, cudaMemcpyDeviceToHost, st));
      GBX_CUDA(cudaStreamSynchronize(st));
      tkeys.alloc(nt);
      tvals.alloc(nt);
      Tmp<int64_t> start(nt, st);
      k_runs<<<ceil_div(np, kT), kT, 0, st>>>(kb.Current(), head.p, seg.p, np, tkeys.p, start.p);
      k_fold_runs<<<ceil_div(nt, kT), kT, 0, st>>>(vb.Current(), start.p, nt, np, s, tvals.p);
      GBX_LAUNCHED();
      GBX_CUDA(cudaStreamSynchronize(st));
    }
  }
  // ---- post-step: merge prior C and T under the mask
  const int64_t mc = C->nnz, m = mc + nt;
  out->nrows = nr;
  out->ncols = nc;
  out->domain = C->domain;
  out->rp.alloc(nr + 1);
  if (m == 0) {
    out->nnz = 0;
    out->col.alloc(1);
    out->val.alloc(1);
    GBX_CUDA(cudaMemsetAsync(out->rp.p, 0, (nr + 1) * 8, out->stream));
    GBX_CUDA(cudaStreamSynchronize(out->stream));
    return;
  }
  Tmp<uint64_t> k0(m, st), k1(m, st);
  Tmp<int64_t> r0(m, st), r1(m, st);
  if (mc) {
    k_mkeys<<<ceil_div(nr, kT), kT, 0, st>>>(C->rp.p, C->col.p, nr, bits, 0, k0.p, r0.p, 0);
    GBX_LAUNCHED();
  }
  if (nt) {
    GBX_CUDA(cudaMemcpyAsync(k0.p + mc, tkeys.p, nt * 8, cudaMemcpyDeviceToDevice, st));
    k_tref<<<ceil_div(nt, kT), kT, 0, st>>>(r0.p + mc, nt);
    GBX_LAUNCHED();
  }
  cub::DoubleBuffer<uint64_t> kb(k0.p, k1.p);
  cub::DoubleBuffer<int64_t> rb(r0.p, r1.p);
  radix_sort_pairs(st, kb, rb, m, 0, 2 * bits);
  Tmp<uint8_t> keep(m, st);
  Tmp<uint64_t> ov(m, st);
  k_post_mat<<<ceil_div(m, kT), kT, 0, st>>>(
      kb.Current(), rb.Current(), m, bits, C->val.p, tvals.p, Mk ? Mk->rp.p : nullptr,
      Mk ? Mk->col.p : nullptr, Mk ? Mk->val.p : nullptr, Mk ? Mk->domain : 0, Mk != nullptr,
      d.structural, d.complement, d.replace, d.accum, C->domain, keep.p, ov.p);
  GBX_LAUNCHED();
  Tmp<uint64_t> ok(m, st);
  Tmp<int64_t> cnt(1, st);
  out->val.alloc(m);
  size_t tb = 0;
  GBX_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, kb.Current(), keep.p, ok.p, cnt.p, m, st));
  {
    Tmp<uint8_t> t(tb, st);
    GBX_CUDA(cub::DeviceSelect::Flagged(t.p, tb, kb.Current(), keep.p, ok.p, cnt.p, m, st));
  }
  tb = 0;
  GBX_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, ov.p, keep.p, out->val.p, cnt.p, m, st));
  {
    Tmp<uint8_t> t(tb, st);
    GBX_CUDA(cub::DeviceSelect::Flagged(t.p, tb, ov.p, keep.p, out->val.p, cnt.p, m, st));
  }
  int64_t no = 0;
  GBX_CUDA(cudaMemcpyAsync(&no, cnt.p, 8, cudaMemcpyDeviceToHost, st));
  GBX_CUDA(cudaStreamSynchronize(st));
  out->nnz = no;
  out->col.alloc(std::max<int64_t>(no, 1));
  rowptr_from_sorted_keys(st, nr, bits, ok.p, no, out->rp.p, out->col.p);
  GBX_CUDA(cudaStreamSynchronize(st));
}

}  // namespace gbx
