// NCCL collectives of the sharded volume (the n x n Gram and
// the line-search scalars all-reduced, the (K-1)-plane halos exchanged),
// issued from the library on the caller's compute stream.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2: the copy PyTorch
// already mapped, or the system one), so the library still loads -- and its
// exports can be checked -- on hosts without NCCL.  One communicator per
// process (one GPU per rank); the 128-byte unique id is created on rank 0 and
// broadcast by the host (torch.distributed in parallel.NativeComm).
#include <dlfcn.h>
#include <nccl.h>

#include <stdio.h>
#include <string.h>

#include <mutex>

#include "common.cuh"

namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
    api.Send = (decltype(api.Send))dlsym(h, "ncclSend");
    api.Recv = (decltype(api.Recv))dlsym(h, "ncclRecv");
    api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.Send && api.Recv &&
             api.GroupStart && api.GroupEnd && api.GetErrorString;
  });
  return api;
}

int nccl_check(ncclResult_t r, const char* where) {
  if (r == ncclSuccess) return HICU_OK;
  static thread_local char msg[256];
  snprintf(msg, sizeof(msg), "%s: %s", where, nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error");
  return hicu_set_error(HICU_ERR_CUDA, msg);
}

}  // namespace

extern "C" int hicu_comm_available(void) { return nccl().ok ? 1 : 0; }

extern "C" int hicu_comm_unique_id(void* id_out) {
  if (!id_out) return hicu_set_error(HICU_ERR_PARAMETER, "comm_unique_id: null");
  if (!nccl().ok) return hicu_set_error(HICU_ERR_CUDA, "comm: libnccl.so.2 not loadable");
  ncclUniqueId id;
  const int s = nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  if (s) return s;
  memcpy(id_out, &id, sizeof(id));
  return HICU_OK;
}

extern "C" int hicu_comm_init(int nranks, int rank, const void* id, void** comm_out) {
  if (!id || !comm_out || nranks < 1 || rank < 0 || rank >= nranks)
    return hicu_set_error(HICU_ERR_PARAMETER, "comm_init: bad arguments");
  if (!nccl().ok) return hicu_set_error(HICU_ERR_CUDA, "comm: libnccl.so.2 not loadable");
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  const int s = nccl_check(nccl().CommInitRank(&c, nranks, uid, rank), "ncclCommInitRank");
  if (s) return s;
  *comm_out = (void*)c;
  return HICU_OK;
}

extern "C" int hicu_comm_destroy(void* comm) {
  if (!comm) return HICU_OK;
  if (!nccl().ok) return hicu_set_error(HICU_ERR_CUDA, "comm: libnccl.so.2 not loadable");
  return nccl_check(nccl().CommDestroy((ncclComm_t)comm), "ncclCommDestroy");
}

// In-place sum over the ranks of `count` doubles (the Gram as 2 n^2 doubles,
// the 7 step scalars), on `stream`.
extern "C" int hicu_allreduce(void* comm, double* buf, int64_t count, void* stream) {
  if (!comm || !buf || count < 0) return hicu_set_error(HICU_ERR_PARAMETER, "allreduce: bad arguments");
  if (!nccl().ok) return hicu_set_error(HICU_ERR_CUDA, "comm: libnccl.so.2 not loadable");
  if (count == 0) return HICU_OK;
  return nccl_check(nccl().AllReduce(buf, buf, (size_t)count, ncclFloat64, ncclSum, (ncclComm_t)comm,
                                     (cudaStream_t)stream),
                    "ncclAllReduce");
}

// One grouped round of point-to-point transfers (the halo accumulate or
// refresh pattern of parallel.HaloExchange: every rank posts its sends and
// receives together, so the round cannot deadlock).
extern "C" int hicu_halo_exchange(void* comm, int nops, const hicu_p2p_op* ops, void* stream) {
  if (!comm || nops < 0 || (nops > 0 && !ops)) return hicu_set_error(HICU_ERR_PARAMETER, "halo_exchange: bad arguments");
  if (!nccl().ok) return hicu_set_error(HICU_ERR_CUDA, "comm: libnccl.so.2 not loadable");
  if (nops == 0) return HICU_OK;
  const NcclApi& a = nccl();
  int s = nccl_check(a.GroupStart(), "ncclGroupStart");
  if (s) return s;
  int first_err = HICU_OK;
  for (int i = 0; i < nops; ++i) {
    const hicu_p2p_op& op = ops[i];
    ncclResult_t r;
    if (op.kind == HICU_P2P_SEND)
      r = a.Send(op.buf, (size_t)op.bytes, ncclUint8, op.peer, (ncclComm_t)comm, (cudaStream_t)stream);
    else
      r = a.Recv(op.buf, (size_t)op.bytes, ncclUint8, op.peer, (ncclComm_t)comm, (cudaStream_t)stream);
    if (r != ncclSuccess && !first_err) first_err = nccl_check(r, op.kind == HICU_P2P_SEND ? "ncclSend" : "ncclRecv");
  }
  s = nccl_check(a.GroupEnd(), "ncclGroupEnd");
  return first_err ? first_err : s;
}
