// Cross-instance transports for H2 (and the H5 partial exchange):
//  * two-sided NCCL: gather -> ncclSend / ncclRecv -> scatter, all on the caller's stream.
//    NCCL is resolved at run time (dlopen "libnccl.so.2" -- the copy PyTorch already
//    loaded, or $BS_NCCL_LIBRARY), so the library loads and every non-NCCL entry point
//    works without it.
//  * CUDA IPC: export / import a device allocation so another process can describe a
//    peer GPU's pool as a remote view; bs_kv_migrate_layer then pushes chunks straight
//    into the peer pool over NVLink (P2P push, no staging).
// PAPER.md names only the fabrics (NVLink / InfiniBand); this is reading D6.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstring>

#include "internal.h"
#include "nccl.h"

namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi* nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = getenv("BS_NCCL_LIBRARY");
    void* h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
      return;
    }
#define BS_SYM(field, name)                                          \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name)); \
  if (!api.field) {                                                  \
    api.why = std::string("missing NCCL symbol ") + name;            \
    return;                                                          \
  }
    BS_SYM(GetUniqueId, "ncclGetUniqueId");
    BS_SYM(CommInitRank, "ncclCommInitRank");
    BS_SYM(CommDestroy, "ncclCommDestroy");
    BS_SYM(Send, "ncclSend");
    BS_SYM(Recv, "ncclRecv");
    BS_SYM(GroupStart, "ncclGroupStart");
    BS_SYM(GroupEnd, "ncclGroupEnd");
    BS_SYM(GetErrorString, "ncclGetErrorString");
#undef BS_SYM
    api.ok = true;
  });
  return &api;
}

bs_status nccl_err(const char* what, ncclResult_t r) {
  return bs::set_error(BS_ERR_NCCL, "%s: %s", what, nccl()->GetErrorString(r));
}

}  // namespace

struct bs_comm {
  ncclComm_t comm = nullptr;
  int32_t nranks = 0, rank = 0;
};

extern "C" {

size_t bs_nccl_unique_id_bytes(void) { return sizeof(ncclUniqueId); }

bs_status bs_nccl_get_unique_id(void* out) {
  BS_REQUIRE(out, "bs_nccl_get_unique_id: out is NULL");
  NcclApi* a = nccl();
  if (!a->ok) return bs::set_error(BS_ERR_NCCL, "%s", a->why.c_str());
  ncclUniqueId id;
  ncclResult_t r = a->GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_err("ncclGetUniqueId", r);
  memcpy(out, &id, sizeof id);
  return BS_OK;
}

bs_status bs_comm_init(const void* nccl_unique_id, int32_t nranks, int32_t rank, bs_comm** out) {
  BS_REQUIRE(out && nccl_unique_id, "bs_comm_init: NULL argument");
  *out = nullptr;
  BS_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "bs_comm_init: rank %d of %d", rank, nranks);
  NcclApi* a = nccl();
  if (!a->ok) return bs::set_error(BS_ERR_NCCL, "%s", a->why.c_str());
  ncclUniqueId id;
  memcpy(&id, nccl_unique_id, sizeof id);
  bs_comm* c = new bs_comm();
  ncclResult_t r = a->CommInitRank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_err("ncclCommInitRank", r);
  }
  c->nranks = nranks;
  c->rank = rank;
  *out = c;
  return BS_OK;
}

bs_status bs_comm_destroy(bs_comm* comm) {
  if (!comm) return BS_OK;
  if (comm->comm) nccl()->CommDestroy(comm->comm);
  delete comm;
  return BS_OK;
}

bs_status bs_sendrecv(bs_comm* comm, const void* sendbuf, size_t send_bytes, int32_t send_peer,
                      void* recvbuf, size_t recv_bytes, int32_t recv_peer, void* stream) {
  BS_REQUIRE(comm, "bs_sendrecv: NULL comm");
  BS_REQUIRE(send_peer < comm->nranks && recv_peer < comm->nranks, "bs_sendrecv: peer out of range");
  BS_REQUIRE(send_peer < 0 || send_bytes == 0 || sendbuf, "bs_sendrecv: NULL sendbuf");
  BS_REQUIRE(recv_peer < 0 || recv_bytes == 0 || recvbuf, "bs_sendrecv: NULL recvbuf");
  NcclApi* a = nccl();
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ncclResult_t r = a->GroupStart();
  if (r != ncclSuccess) return nccl_err("ncclGroupStart", r);
  if (send_peer >= 0 && send_bytes) {
    r = a->Send(sendbuf, send_bytes, ncclUint8, send_peer, comm->comm, s);
    if (r != ncclSuccess) {
      a->GroupEnd();
      return nccl_err("ncclSend", r);
    }
  }
  if (recv_peer >= 0 && recv_bytes) {
    r = a->Recv(recvbuf, recv_bytes, ncclUint8, recv_peer, comm->comm, s);
    if (r != ncclSuccess) {
      a->GroupEnd();
      return nccl_err("ncclRecv", r);
    }
  }
  r = a->GroupEnd();
  if (r != ncclSuccess) return nccl_err("ncclGroupEnd", r);
  return BS_OK;
}

bs_status bs_exchange(bs_comm* comm, int32_t n_send, const void* const* send_bufs,
                      const size_t* send_bytes, const int32_t* send_peers, int32_t n_recv,
                      void* const* recv_bufs, const size_t* recv_bytes, const int32_t* recv_peers,
                      void* stream) {
  BS_REQUIRE(comm, "bs_exchange: NULL comm");
  BS_REQUIRE(n_send >= 0 && n_recv >= 0, "bs_exchange: negative count");
  BS_REQUIRE(n_send == 0 || (send_bufs && send_bytes && send_peers), "bs_exchange: NULL send array");
  BS_REQUIRE(n_recv == 0 || (recv_bufs && recv_bytes && recv_peers), "bs_exchange: NULL recv array");
  for (int i = 0; i < n_send; ++i)
    BS_REQUIRE(send_peers[i] >= 0 && send_peers[i] < comm->nranks && (send_bytes[i] == 0 || send_bufs[i]),
               "bs_exchange: send %d: peer %d / buffer", i, send_peers[i]);
  for (int i = 0; i < n_recv; ++i)
    BS_REQUIRE(recv_peers[i] >= 0 && recv_peers[i] < comm->nranks && (recv_bytes[i] == 0 || recv_bufs[i]),
               "bs_exchange: recv %d: peer %d / buffer", i, recv_peers[i]);
  NcclApi* a = nccl();
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ncclResult_t r = a->GroupStart();
  if (r != ncclSuccess) return nccl_err("ncclGroupStart", r);
  for (int i = 0; i < n_send && r == ncclSuccess; ++i)
    if (send_bytes[i]) r = a->Send(send_bufs[i], send_bytes[i], ncclUint8, send_peers[i], comm->comm, s);
  for (int i = 0; i < n_recv && r == ncclSuccess; ++i)
    if (recv_bytes[i]) r = a->Recv(recv_bufs[i], recv_bytes[i], ncclUint8, recv_peers[i], comm->comm, s);
  const ncclResult_t r2 = a->GroupEnd();
  if (r != ncclSuccess) return nccl_err("ncclSend / ncclRecv", r);
  if (r2 != ncclSuccess) return nccl_err("ncclGroupEnd", r2);
  return BS_OK;
}

bs_status bs_kv_send_layer(const bs_kv_pool* src, int32_t layer, const int32_t* src_ids, int32_t n,
                           int32_t peer, bs_comm* comm, void* staging, void* stream) {
  bs_status st = bs_kv_gather_layer(src, layer, src_ids, n, staging, stream);
  if (st != BS_OK || n == 0) return st;
  return bs_sendrecv(comm, staging, (size_t)n * src->chunk_bytes, peer, nullptr, 0, -1, stream);
}

bs_status bs_kv_recv_layer(bs_kv_pool* dst, int32_t layer, const int32_t* dst_ids, int32_t n,
                           int32_t peer, bs_comm* comm, void* staging, void* stream) {
  BS_REQUIRE(dst, "bs_kv_recv_layer: NULL pool");
  if (n == 0) return BS_OK;
  bs_status st = bs_sendrecv(comm, nullptr, 0, -1, staging, (size_t)n * dst->chunk_bytes, peer, stream);
  if (st != BS_OK) return st;
  return bs_kv_scatter_layer(dst, layer, dst_ids, n, staging, stream);
}

bs_status bs_kv_sendrecv_layer(bs_comm* comm, const bs_kv_pool* src, const int32_t* src_ids,
                               int32_t n_send, int32_t send_peer, void* send_staging,
                               bs_kv_pool* dst, const int32_t* dst_ids, int32_t n_recv,
                               int32_t recv_peer, void* recv_staging, int32_t layer, void* stream) {
  BS_REQUIRE(comm, "bs_kv_sendrecv_layer: NULL comm");
  bs_status st = BS_OK;
  if (n_send > 0) {
    st = bs_kv_gather_layer(src, layer, src_ids, n_send, send_staging, stream);
    if (st != BS_OK) return st;
  }
  BS_REQUIRE(n_recv == 0 || dst, "bs_kv_sendrecv_layer: NULL dst pool");
  st = bs_sendrecv(comm, send_staging, n_send > 0 ? (size_t)n_send * src->chunk_bytes : 0,
                   n_send > 0 ? send_peer : -1, recv_staging,
                   n_recv > 0 ? (size_t)n_recv * dst->chunk_bytes : 0, n_recv > 0 ? recv_peer : -1,
                   stream);
  if (st != BS_OK || n_recv == 0) return st;
  return bs_kv_scatter_layer(dst, layer, dst_ids, n_recv, recv_staging, stream);
}

// ---- CUDA IPC ---------------------------------------------------------------------------

size_t bs_ipc_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

bs_status bs_ipc_export(const void* dev_ptr, void* handle_out, size_t* offset_out) {
  BS_REQUIRE(dev_ptr && handle_out && offset_out, "bs_ipc_export: NULL argument");
  // the IPC handle names the whole allocation; the caller's pointer may be interior
  using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static GetRange get_range = nullptr;
  if (!get_range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        !fn)
      return bs::set_error(BS_ERR_CUDA, "bs_ipc_export: cuMemGetAddressRange unavailable");
    get_range = reinterpret_cast<GetRange>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range(&base, &size, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS)
    return bs::set_error(BS_ERR_CUDA, "bs_ipc_export: pointer is not a device allocation");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return bs::set_error(BS_ERR_CUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  memcpy(handle_out, &h, sizeof h);
  *offset_out = (size_t)((CUdeviceptr)dev_ptr - base);
  return BS_OK;
}

bs_status bs_ipc_import(const void* handle, size_t offset, void** dev_ptr_out) {
  BS_REQUIRE(handle && dev_ptr_out, "bs_ipc_import: NULL argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  void* base = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return bs::set_error(BS_ERR_CUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
  *dev_ptr_out = static_cast<uint8_t*>(base) + offset;
  return BS_OK;
}

bs_status bs_ipc_close(void* dev_ptr, size_t offset) {
  BS_REQUIRE(dev_ptr, "bs_ipc_close: NULL pointer");
  cudaError_t e = cudaIpcCloseMemHandle(static_cast<uint8_t*>(dev_ptr) - offset);
  if (e != cudaSuccess) return bs::set_error(BS_ERR_CUDA, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
  return BS_OK;
}

}  // extern "C"
