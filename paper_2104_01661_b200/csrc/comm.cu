// comm.cu -- the multi-GPU communicator of libgbx.so ("multi-GPU
// handles own one communicator (ncclComm_t per GPU)").
//
// Two transports behind one interface:
//   * NCCL: one process per GPU, gbx_comm_init(nranks, rank, unique id): every
//     collective is an NCCL call on the communicator's stream (NVLink /
//     NVSwitch inside one node).  libnccl.so.2 is bound at run time (dlopen):
//     inside a process that already loaded NCCL (PyTorch) the loaded copy is
//     reused, otherwise the system library is opened -- so libgbx.so never
//     forces an NCCL version on its host process.
//   * local: gbx_comm_init_local(nranks, device): all ranks live in THIS
//     process on ONE GPU (the "nlocal" ranks of the handle), and a collective
//     is a set of device copies / a reduction kernel.  It runs the identical
//     multi-rank protocols one rank after another between exchanges -- no rank
//     ever waits for a rank that is not running -- which is how the sharded
//     algorithms are tested on one B200.
// Every collective takes per-LOCAL-rank buffers (arrays of nlocal pointers);
// with NCCL nlocal = 1.  Calls are synchronous from the host's view.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>
#include <vector>

#include "comm.cuh"

namespace gbx {

// ---- NCCL, bound at run time ---------------------------------------------------
namespace {

struct NcclApi {
  bool loaded = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already in the process?
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      api.why = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) {
      void* p = dlsym(h, n);
      if (!p && api.why.empty()) api.why = std::string("NCCL symbol missing: ") + n;
      return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.CommAbort = reinterpret_cast<decltype(api.CommAbort)>(sym("ncclCommAbort"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.GetVersion = reinterpret_cast<decltype(api.GetVersion)>(sym("ncclGetVersion"));
    api.loaded = api.why.empty();
  });
  if (!api.loaded) fail(GBX_COMM_ERROR, "nccl: " + api.why);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(GBX_COMM_ERROR, std::string("nccl: ") + what + ": " + nccl().GetErrorString(r));
}

ncclDataType_t nccl_type(CollType t) {
  switch (t) {
    case CollType::F64: return ncclFloat64;
    case CollType::I64: return ncclInt64;
    case CollType::U64: return ncclUint64;
    case CollType::I32: return ncclInt32;
    case CollType::U32: return ncclUint32;
    default: return ncclUint8;
  }
}

size_t type_size(CollType t) {
  switch (t) {
    case CollType::F64: case CollType::I64: case CollType::U64: return 8;
    case CollType::I32: case CollType::U32: return 4;
    default: return 1;
  }
}

// local transport: dst[i] = op over the nl sources
template <typename T>
__global__ void k_reduce_local(const T* const* src, int nl, int64_t count, T* out, int op) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= count) return;
  T v = src[0][i];
  for (int q = 1; q < nl; ++q) {  // rank order: the same fp64 sums on every rank
    const T w = src[q][i];
    v = op == 0 ? T(v + w) : (op == 1 ? (w > v ? w : v) : (w < v ? w : v));
  }
  out[i] = v;
}

}  // namespace

void comm_unique_id(void* id) {
  ncclUniqueId u;
  nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
  std::memcpy(id, &u, sizeof u);
}

gbx_comm* comm_new_nccl(int nranks, int rank, const void* id, int device) {
  if (nranks < 1 || rank < 0 || rank >= nranks) fail(GBX_INVALID_VALUE, "comm: bad rank / nranks");
  if (!id) fail(GBX_NULL_ARGUMENT, "comm: unique id is NULL");
  auto c = std::make_unique<gbx_comm>();
  c->nranks = nranks;
  c->rank = rank;
  c->nlocal = 1;
  c->device = device;
  GBX_CUDA(cudaSetDevice(device));
  GBX_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof u);
  ncclComm_t nc = nullptr;
  nccl_check(nccl().CommInitRank(&nc, nranks, u, rank), "ncclCommInitRank");
  c->nccl = nc;
  return c.release();
}

gbx_comm* comm_new_local(int nranks, int device) {
  if (nranks < 1 || nranks > kMaxRanks) fail(GBX_INVALID_VALUE, "comm_local: 1..8 ranks");
  auto c = std::make_unique<gbx_comm>();
  c->nranks = nranks;
  c->rank = 0;
  c->nlocal = nranks;
  c->device = device;
  GBX_CUDA(cudaSetDevice(device));
  GBX_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  return c.release();
}

void comm_destroy_nccl(void* nc) {
  // never throws (destructor path): the communicator was created by this library
  if (nc) (void)nccl().CommDestroy(static_cast<ncclComm_t>(nc));
}

void comm_sync(gbx_comm* c) { GBX_CUDA(cudaStreamSynchronize(c->stream)); }

void c_allgather(gbx_comm* c, const void* const* send, void* const* recv, size_t bytes) {
  if (c->nccl) {
    nccl_check(nccl().AllGather(send[0], recv[0], bytes, ncclUint8,
                                static_cast<ncclComm_t>(c->nccl), c->stream),
               "ncclAllGather");
  } else {
    for (int l = 0; l < c->nlocal; ++l)
      for (int q = 0; q < c->nranks; ++q)
        if (bytes)
          GBX_CUDA(cudaMemcpyAsync(static_cast<char*>(recv[l]) + q * bytes, send[q], bytes,
                                   cudaMemcpyDeviceToDevice, c->stream));
  }
  comm_sync(c);
}

void c_allreduce(gbx_comm* c, void* const* buf, size_t count, CollType t, CollOp op) {
  if (count == 0) return;
  if (c->nccl) {
    const ncclRedOp_t o = op == CollOp::Sum ? ncclSum : op == CollOp::Max ? ncclMax : ncclMin;
    nccl_check(nccl().AllReduce(buf[0], buf[0], count, nccl_type(t), o,
                                static_cast<ncclComm_t>(c->nccl), c->stream),
               "ncclAllReduce");
    comm_sync(c);
    return;
  }
  if (c->nlocal == 1) return;
  const size_t es = type_size(t);
  Tmp<uint8_t> out(count * es, c->stream);
  Tmp<void*> src(c->nlocal, c->stream);
  GBX_CUDA(cudaMemcpyAsync(src.p, buf, c->nlocal * sizeof(void*), cudaMemcpyHostToDevice, c->stream));
  const int o = op == CollOp::Sum ? 0 : op == CollOp::Max ? 1 : 2;
  const int grid = ceil_div(static_cast<int64_t>(count), 256);
  switch (t) {
    case CollType::F64:
      k_reduce_local<double><<<grid, 256, 0, c->stream>>>(reinterpret_cast<const double* const*>(src.p),
                                                          c->nlocal, count, reinterpret_cast<double*>(out.p), o);
      break;
    case CollType::I64:
      k_reduce_local<int64_t><<<grid, 256, 0, c->stream>>>(reinterpret_cast<const int64_t* const*>(src.p),
                                                           c->nlocal, count, reinterpret_cast<int64_t*>(out.p), o);
      break;
    case CollType::U64:
      k_reduce_local<uint64_t><<<grid, 256, 0, c->stream>>>(reinterpret_cast<const uint64_t* const*>(src.p),
                                                            c->nlocal, count, reinterpret_cast<uint64_t*>(out.p), o);
      break;
    case CollType::I32:
      k_reduce_local<int32_t><<<grid, 256, 0, c->stream>>>(reinterpret_cast<const int32_t* const*>(src.p),
                                                           c->nlocal, count, reinterpret_cast<int32_t*>(out.p), o);
      break;
    case CollType::U32:
      k_reduce_local<uint32_t><<<grid, 256, 0, c->stream>>>(reinterpret_cast<const uint32_t* const*>(src.p),
                                                            c->nlocal, count, reinterpret_cast<uint32_t*>(out.p), o);
      break;
    case CollType::U8:
      k_reduce_local<uint8_t><<<grid, 256, 0, c->stream>>>(reinterpret_cast<const uint8_t* const*>(src.p),
                                                           c->nlocal, count, reinterpret_cast<uint8_t*>(out.p), o);
      break;
    default:
      fail(GBX_INVALID_VALUE, "allreduce: unsupported type");
  }
  GBX_LAUNCHED();
  for (int l = 0; l < c->nlocal; ++l)
    GBX_CUDA(cudaMemcpyAsync(buf[l], out.p, count * es, cudaMemcpyDeviceToDevice, c->stream));
  comm_sync(c);
}

std::vector<int64_t> c_allgather_host(gbx_comm* c, const std::vector<int64_t>& mine) {
  if (static_cast<int>(mine.size()) != c->nlocal) fail(GBX_INVALID_VALUE, "allgather_host: one value per local rank");
  if (!c->nccl) return mine;  // every rank is local: the values are already here
  Tmp<int64_t> d(1 + c->nranks, c->stream);
  GBX_CUDA(cudaMemcpyAsync(d.p, mine.data(), 8, cudaMemcpyHostToDevice, c->stream));
  nccl_check(nccl().AllGather(d.p, d.p + 1, 1, ncclInt64, static_cast<ncclComm_t>(c->nccl),
                              c->stream),
             "ncclAllGather");
  std::vector<int64_t> all(c->nranks);
  GBX_CUDA(cudaMemcpyAsync(all.data(), d.p + 1, c->nranks * 8, cudaMemcpyDeviceToHost, c->stream));
  comm_sync(c);
  return all;
}

void c_alltoallv(gbx_comm* c, const void* const* send, const std::vector<std::vector<int64_t>>& soff,
                 void* const* recv, const std::vector<std::vector<int64_t>>& roff) {
  // soff[l][q] .. soff[l][q+1]: bytes local rank l sends to rank q;
  // roff[l][q] .. roff[l][q+1]: bytes local rank l receives from rank q
  if (c->nccl) {
    const int me = c->rank;
    ncclComm_t nc = static_cast<ncclComm_t>(c->nccl);
    nccl_check(nccl().GroupStart(), "ncclGroupStart");
    for (int q = 0; q < c->nranks; ++q) {
      const int64_t sb = soff[0][q + 1] - soff[0][q], rb = roff[0][q + 1] - roff[0][q];
      if (q == me) {
        if (sb)
          GBX_CUDA(cudaMemcpyAsync(static_cast<char*>(recv[0]) + roff[0][q],
                                   static_cast<const char*>(send[0]) + soff[0][q], sb,
                                   cudaMemcpyDeviceToDevice, c->stream));
        continue;
      }
      if (sb) nccl_check(nccl().Send(static_cast<const char*>(send[0]) + soff[0][q], sb, ncclUint8, q, nc, c->stream), "ncclSend");
      if (rb) nccl_check(nccl().Recv(static_cast<char*>(recv[0]) + roff[0][q], rb, ncclUint8, q, nc, c->stream), "ncclRecv");
    }
    nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
  } else {
    for (int l = 0; l < c->nlocal; ++l)
      for (int q = 0; q < c->nranks; ++q) {
        const int64_t b = roff[l][q + 1] - roff[l][q];
        if (b)
          GBX_CUDA(cudaMemcpyAsync(static_cast<char*>(recv[l]) + roff[l][q],
                                   static_cast<const char*>(send[q]) + soff[q][l], b,
                                   cudaMemcpyDeviceToDevice, c->stream));
      }
  }
  comm_sync(c);
}

std::vector<std::vector<int64_t>> c_exchange_counts(gbx_comm* c,
                                                    const std::vector<std::vector<int64_t>>& cnt) {
  // cnt[l][q] = what local rank l sends to rank q -> out[l][q] = what l gets from q
  const int P = c->nranks;
  std::vector<std::vector<int64_t>> out(c->nlocal, std::vector<int64_t>(P, 0));
  if (!c->nccl) {
    for (int l = 0; l < c->nlocal; ++l)
      for (int q = 0; q < P; ++q) out[l][q] = cnt[q][l];
    return out;
  }
  Tmp<int64_t> d(P + P * P, c->stream);
  GBX_CUDA(cudaMemcpyAsync(d.p, cnt[0].data(), P * 8, cudaMemcpyHostToDevice, c->stream));
  nccl_check(nccl().AllGather(d.p, d.p + P, P, ncclInt64, static_cast<ncclComm_t>(c->nccl),
                              c->stream),
             "ncclAllGather");
  std::vector<int64_t> all(P * P);
  GBX_CUDA(cudaMemcpyAsync(all.data(), d.p + P, P * P * 8, cudaMemcpyDeviceToHost, c->stream));
  comm_sync(c);
  for (int q = 0; q < P; ++q) out[0][q] = all[q * P + c->rank];
  return out;
}

// ---- peer buffers (the fused exchange's x / slot tables / signal words) ----
PeerBuf::~PeerBuf() { release(); }

void PeerBuf::release() {
  for (size_t i = 0; i < opened.size(); ++i)
    if (opened[i]) cudaIpcCloseMemHandle(opened[i]);
  opened.clear();
  for (void* p : local)
    if (p) cudaFree(p);
  local.clear();
  peer.clear();
}

void peer_alloc(gbx_comm* c, size_t bytes, PeerBuf& b) {
  b.release();
  b.bytes = bytes;
  b.local.assign(c->nlocal, nullptr);
  for (int l = 0; l < c->nlocal; ++l) {
    // cudaMalloc (not the stream-ordered pool): legacy IPC handles need it
    GBX_CUDA(cudaMalloc(&b.local[l], std::max<size_t>(bytes, 16)));
    GBX_CUDA(cudaMemset(b.local[l], 0, std::max<size_t>(bytes, 16)));
  }
  b.peer.assign(c->nlocal, std::vector<uint64_t>(c->nranks, 0));
  if (!c->nccl) {
    for (int l = 0; l < c->nlocal; ++l)
      for (int q = 0; q < c->nranks; ++q) b.peer[l][q] = reinterpret_cast<uint64_t>(b.local[q]);
    return;
  }
  // NCCL: IPC handles all-gathered over the communicator itself
  cudaIpcMemHandle_t h;
  GBX_CUDA(cudaIpcGetMemHandle(&h, b.local[0]));
  Tmp<uint8_t> d(sizeof h * (1 + c->nranks), c->stream);
  GBX_CUDA(cudaMemcpyAsync(d.p, &h, sizeof h, cudaMemcpyHostToDevice, c->stream));
  nccl_check(nccl().AllGather(d.p, d.p + sizeof h, sizeof h, ncclUint8,
                              static_cast<ncclComm_t>(c->nccl), c->stream),
             "ncclAllGather(ipc handles)");
  std::vector<cudaIpcMemHandle_t> all(c->nranks);
  GBX_CUDA(cudaMemcpyAsync(all.data(), d.p + sizeof h, sizeof h * c->nranks, cudaMemcpyDeviceToHost,
                           c->stream));
  comm_sync(c);
  for (int q = 0; q < c->nranks; ++q) {
    if (q == c->rank) {
      b.peer[0][q] = reinterpret_cast<uint64_t>(b.local[0]);
      continue;
    }
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, all[q], cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      fail(GBX_COMM_ERROR, std::string("peer buffer of rank ") + std::to_string(q) +
                               " not mappable: " + cudaGetErrorString(e));
    }
    b.opened.push_back(p);
    b.peer[0][q] = reinterpret_cast<uint64_t>(p);
  }
}

}  // namespace gbx

gbx_comm::~gbx_comm() {
  cudaSetDevice(device);
  if (stream) cudaStreamSynchronize(stream);
  if (nccl) gbx::comm_destroy_nccl(nccl);
  if (stream) cudaStreamDestroy(stream);
  (void)cudaGetLastError();  // never leave a destructor's error for the next call
}
