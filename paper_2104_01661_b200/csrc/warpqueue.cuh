// warpqueue.cuh -- warp-private append buffers in shared memory.
//
// Frontier/queue appends from every warp to one global counter serialise in the
// L2 atomic unit (one address): with ~10^7 warp iterations per traversal that
// alone costs tens of ms.  A warp instead stages its pushes in a private
// shared-memory buffer and flushes it with ONE global atomicAdd per ~CAP
// entries (coalesced copy-out).  All lanes of the warp must call push/flush
// together (warp-uniform control flow).
#pragma once

#include <cstdint>

namespace gbx {

template <typename T, int CAP>
struct WarpQueue {
  T* buf;     // shared memory, CAP entries, private to the warp
  int n;      // staged entries (warp-uniform)
  T* q;       // global queue
  int* cnt;   // global counter

  __device__ __forceinline__ void reset(T* out, int* counter) {
    q = out;
    cnt = counter;
    n = 0;
  }

  __device__ __forceinline__ void flush() {
    __syncwarp();
    if (n == 0) return;
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == 0) base = atomicAdd(cnt, n);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (int i = lane; i < n; i += 32) q[base + i] = buf[i];
    __syncwarp();
    n = 0;
  }

  __device__ __forceinline__ void push(bool has, T v) {
    const unsigned b = __ballot_sync(0xffffffffu, has);
    if (!b) return;
    const int lane = threadIdx.x & 31;
    if (has) buf[n + __popc(b & ((1u << lane) - 1))] = v;
    n += __popc(b);
    if (n > CAP - 32) flush();
  }
};

}  // namespace gbx

namespace gbx {

// Frontier variant: stages vertex ids; the flush expands each vertex into
// (vertex | chunk << 32) entries of <= chunk edges (so hub rows are split over
// warps) and updates the entry / vertex / frontier-edge counters with one
// atomic each.  Optionally also appends the vertex ids to a plain list.
template <int CAP>
struct FrontierQueue {
  int32_t* buf;
  int n;
  int64_t* q;                      // entries
  int* cnt_ent;
  int* cnt_vtx;
  unsigned long long* cnt_edges;   // nullable
  int32_t* list;                   // nullable: vertex list (shares cnt_vtx)
  const int64_t* rp;
  int64_t chunk;

  __device__ __forceinline__ static int nchunks(int64_t deg, int64_t chunk) {
    return deg <= chunk ? 1 : static_cast<int>((deg + chunk - 1) / chunk);
  }

  __device__ __forceinline__ void reset(int64_t* entries, int* ce, int* cv,
                                        unsigned long long* cedges, int32_t* vlist) {
    q = entries;
    cnt_ent = ce;
    cnt_vtx = cv;
    cnt_edges = cedges;
    list = vlist;
    n = 0;
  }

  __device__ __forceinline__ void flush() {
    __syncwarp();
    if (n == 0) return;
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    // pass 1: totals
    int ent = 0;
    unsigned long long edges = 0;
    for (int i = lane; i < n; i += 32) {
      const int32_t v = buf[i];
      const int64_t d = rp[v + 1] - rp[v];
      ent += nchunks(d, chunk);
      edges += static_cast<unsigned long long>(d);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ent += __shfl_xor_sync(full, ent, o);
      edges += __shfl_xor_sync(full, edges, o);
    }
    int ebase = 0, vbase = 0;
    if (lane == 0) {
      ebase = atomicAdd(cnt_ent, ent);
      vbase = atomicAdd(cnt_vtx, n);
      if (cnt_edges) atomicAdd(cnt_edges, edges);
    }
    ebase = __shfl_sync(full, ebase, 0);
    vbase = __shfl_sync(full, vbase, 0);
    // pass 2: write entries in rounds of 32 vertices
    int off = ebase;
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      int32_t v = 0;
      int k = 0;
      if (i < n) {
        v = buf[i];
        k = nchunks(rp[v + 1] - rp[v], chunk);
        if (list) list[vbase + i] = v;
      }
      int incl = k;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(full, incl, o);
        if (lane >= o) incl += t;
      }
      const int tot = __shfl_sync(full, incl, 31);
      for (int c = 0; c < k; ++c)
        q[off + incl - k + c] = (static_cast<int64_t>(c) << 32) | static_cast<uint32_t>(v);
      off += tot;
    }
    __syncwarp();
    n = 0;
  }

  __device__ __forceinline__ void push(bool has, int32_t v) {
    const unsigned b = __ballot_sync(0xffffffffu, has);
    if (!b) return;
    const int lane = threadIdx.x & 31;
    if (has) buf[n + __popc(b & ((1u << lane) - 1))] = v;
    n += __popc(b);
    if (n > CAP - 32) flush();
  }

  // End-of-level flush called by EVERY thread of the CTA (block-uniform): the
  // warps' totals meet in shared memory and ONE thread per CTA reserves the
  // CTA's runs with the global atomics (every warp flushing at the same moment
  // piled ~10^4 atomics onto the same three addresses at the end of a level).
  // The per-vertex chunk counts of pass 1 are kept in kbuf (CAP ints per
  // warp), so pass 2 re-reads no row pointers.  s_red: 6 ints of CTA shared
  // memory, 8-byte aligned.
  __device__ __forceinline__ void flush_block(int* kbuf, int* s_red) {
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    unsigned long long* s_edges = reinterpret_cast<unsigned long long*>(s_red + 4);
    if (threadIdx.x == 0) {
      s_red[0] = 0;
      s_red[1] = 0;
      *s_edges = 0ull;
    }
    __syncthreads();
    int ent = 0;
    unsigned long long edges = 0;
    for (int i = lane; i < n; i += 32) {
      const int32_t v = buf[i];
      const int64_t d = rp[v + 1] - rp[v];
      const int k = nchunks(d, chunk);
      kbuf[i] = k;
      ent += k;
      edges += static_cast<unsigned long long>(d);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ent += __shfl_xor_sync(full, ent, o);
      edges += __shfl_xor_sync(full, edges, o);
    }
    int eoff = 0, voff = 0;
    if (lane == 0 && n > 0) {
      eoff = atomicAdd(&s_red[0], ent);
      voff = atomicAdd(&s_red[1], n);
      if (cnt_edges) atomicAdd(s_edges, edges);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int te = s_red[0], tv = s_red[1];
      s_red[2] = te ? atomicAdd(cnt_ent, te) : 0;
      s_red[3] = tv ? atomicAdd(cnt_vtx, tv) : 0;
      if (cnt_edges && tv) atomicAdd(cnt_edges, *s_edges);
    }
    __syncthreads();
    const int ebase = s_red[2] + __shfl_sync(full, eoff, 0);
    const int vbase = s_red[3] + __shfl_sync(full, voff, 0);
    int off = ebase;
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      int32_t v = 0;
      int k = 0;
      if (i < n) {
        v = buf[i];
        k = kbuf[i];
        if (list) list[vbase + i] = v;
      }
      int incl = k;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(full, incl, o);
        if (lane >= o) incl += t;
      }
      const int tot = __shfl_sync(full, incl, 31);
      for (int c = 0; c < k; ++c)
        q[off + incl - k + c] = (static_cast<int64_t>(c) << 32) | static_cast<uint32_t>(v);
      off += tot;
    }
    __syncwarp();
    n = 0;
  }
};

}  // namespace gbx
