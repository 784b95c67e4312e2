// NCCL transport of the multi-rank exchange (world > 1, one process per GPU).
// libnccl is loaded at run time (dlopen): a single-GPU build and run never needs it, and in a
// PyTorch process the already-loaded libnccl.so.2 is the one bound.  Per step (sc_step): the
// packed values for every peer go out with ncclSend and the peers' values come in with
// ncclRecv inside one ncclGroupStart/End, on the context stream (NVLink / NVSwitch P2P).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>

#include "sc_internal.h"

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  if (a.h) return a;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* n : names)
    if ((a.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
  if (!a.h) throw ScError(SC_ERR_NCCL, "world > 1 needs libnccl.so.2 (dlopen failed)");
  auto sym = [&](const char* s) {
    void* f = dlsym(a.h, s);
    if (!f) throw ScError(SC_ERR_NCCL, std::string("libnccl lacks ") + s);
    return f;
  };
  a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
  a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
  a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
  a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
  a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
  a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
  a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
  a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
  a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
  return a;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw ScError(SC_ERR_NCCL, std::string(what) + ": " + api().GetErrorString(r));
}

}  // namespace

int nccl_unique_id(void* out128) {
  ncclUniqueId id;
  check(api().GetUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, sizeof(id));
  return 0;
}

void nccl_init(sc_ctx* c, const void* unique_id) {
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  ncclComm_t comm = nullptr;
  check(api().CommInitRank(&comm, c->world, id, c->rank), "ncclCommInitRank");
  c->nccl_comm = comm;
}

void nccl_exchange(sc_ctx* c) {
  NcclApi& a = api();
  ncclComm_t comm = static_cast<ncclComm_t>(c->nccl_comm);
  check(a.GroupStart(), "ncclGroupStart");
  for (int q = 0; q < c->world; ++q) {
    const size_t ns = (size_t)(c->xs_off[q + 1] - c->xs_off[q]);
    const size_t nr = (size_t)(c->xr_off[q + 1] - c->xr_off[q]);
    if (ns) check(a.Send(c->d_xs_buf + c->xs_off[q], ns, ncclFloat64, q, comm, c->stream), "ncclSend");
    if (nr) check(a.Recv(c->d_xr_buf + c->xr_off[q], nr, ncclFloat64, q, comm, c->stream), "ncclRecv");
  }
  check(a.GroupEnd(), "ncclGroupEnd");
}

void nccl_allreduce_sum(sc_ctx* c, double* buf, int64_t n) {
  check(api().AllReduce(buf, buf, (size_t)n, ncclFloat64, ncclSum, static_cast<ncclComm_t>(c->nccl_comm),
                        c->stream),
        "ncclAllReduce");
}

void nccl_destroy(sc_ctx* c) {
  if (c->nccl_comm) api().CommDestroy(static_cast<ncclComm_t>(c->nccl_comm));
  c->nccl_comm = nullptr;
}
