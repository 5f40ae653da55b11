// nccl.cu — the library's own NCCL transport of the partitioned evaluation
// (SURVEY §8(b) nccl_unique_id / TLFEA_E_NCCL, §8(e) steps 2-4: the packed
// boundary partials travel with NCCL point-to-point over NVLink on the
// context's communication stream while tlfea_eval_interior runs).
//
// libnccl.so.2 is loaded at run time (dlopen; in a PyTorch process the copy
// torch already mapped is reused), so the library has no link-time NCCL
// dependency and single-GPU use never touches NCCL. Only the types of nccl.h
// are used at compile time.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "common.cuh"

namespace tlfea {

namespace {
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
      return;
    }
#define TL_SYM(f)                                                     \
  a.f = reinterpret_cast<decltype(a.f)>(dlsym(h, "nccl" #f));         \
  if (!a.f) {                                                         \
    a.why = "libnccl: missing symbol nccl" #f;                        \
    return;                                                           \
  }
    TL_SYM(GetUniqueId)
    TL_SYM(CommInitRank)
    TL_SYM(CommDestroy)
    TL_SYM(GroupStart)
    TL_SYM(GroupEnd)
    TL_SYM(Send)
    TL_SYM(Recv)
    TL_SYM(GetErrorString)
#undef TL_SYM
    a.ok = true;
  });
  return a;
}

tlfea_status nccl_fail(ncclResult_t r, const char* what) {
  return fail(TLFEA_E_NCCL, std::string(what) + ": " + api().GetErrorString(r));
}
}  // namespace

tlfea_status nccl_get_unique_id(void* id_out) {
  const NcclApi& a = api();
  if (!a.ok) return fail(TLFEA_E_NCCL, a.why);
  ncclUniqueId id;
  const ncclResult_t r = a.GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == TLFEA_NCCL_ID_BYTES, "ncclUniqueId size");
  std::memcpy(id_out, &id, sizeof(id));
  return TLFEA_OK;
}

tlfea_status nccl_attach(Context* c, const void* id_in) {
  const NcclApi& a = api();
  if (!a.ok) return fail(TLFEA_E_NCCL, a.why);
  if (c->nccl_comm) return fail(TLFEA_E_INVALID, "tlfea_nccl_attach: the context already has a communicator");
  ncclUniqueId id;
  std::memcpy(&id, id_in, sizeof(id));
  ncclComm_t comm = nullptr;
  const ncclResult_t r = a.CommInitRank(&comm, c->nranks, id, c->rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  c->nccl_comm = comm;
  TL_CUDA(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
  TL_CUDA(cudaEventCreateWithFlags(&c->ev_packed, cudaEventDisableTiming));
  TL_CUDA(cudaEventCreateWithFlags(&c->ev_exchanged, cudaEventDisableTiming));
  return TLFEA_OK;
}

void nccl_detach(Context* c) {
  if (c->nccl_comm) api().CommDestroy(static_cast<ncclComm_t>(c->nccl_comm));
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->ev_packed) cudaEventDestroy(c->ev_packed);
  if (c->ev_exchanged) cudaEventDestroy(c->ev_exchanged);
  c->nccl_comm = nullptr;
  c->comm_stream = nullptr;
  c->ev_packed = c->ev_exchanged = nullptr;
}

// After tlfea_eval_begin on `s`: the transfer send_buf -> peers, recv_buf <-
// peers (the per-peer segments of tlfea_exchange_sizes, rank order) as one
// NCCL group on comm_stream, ordered after `s` by an event; the caller's next
// launches on `s` (tlfea_eval_interior) overlap it, and tlfea_eval_finish
// orders `s` after it.
tlfea_status nccl_exchange(Context* c, const double* send_buf, double* recv_buf, cudaStream_t s) {
  const NcclApi& a = api();
  if (!c->nccl_comm) return fail(TLFEA_E_INVALID, "tlfea_eval_exchange: call tlfea_nccl_attach first");
  ncclComm_t comm = static_cast<ncclComm_t>(c->nccl_comm);
  TL_CUDA(cudaEventRecord(c->ev_packed, s));
  TL_CUDA(cudaStreamWaitEvent(c->comm_stream, c->ev_packed, 0));
  ncclResult_t r = a.GroupStart();
  if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
  int64_t so = 0, ro = 0;
  for (int p = 0; p < c->nranks; ++p) {
    const int64_t ns = p < (int)c->send_counts.size() ? c->send_counts[p] : 0;
    const int64_t nr = p < (int)c->recv_counts.size() ? c->recv_counts[p] : 0;
    if (ns > 0 && (r = a.Send(send_buf + so, (size_t)ns, ncclFloat64, p, comm, c->comm_stream)) != ncclSuccess)
      break;
    if (nr > 0 && (r = a.Recv(recv_buf + ro, (size_t)nr, ncclFloat64, p, comm, c->comm_stream)) != ncclSuccess)
      break;
    so += ns;
    ro += nr;
  }
  const ncclResult_t r2 = a.GroupEnd();
  if (r != ncclSuccess) return nccl_fail(r, "ncclSend/ncclRecv");
  if (r2 != ncclSuccess) return nccl_fail(r2, "ncclGroupEnd");
  TL_CUDA(cudaEventRecord(c->ev_exchanged, c->comm_stream));
  c->exchange_pending = true;
  return TLFEA_OK;
}

// tlfea_eval_finish: order `s` after a pending library exchange.
tlfea_status nccl_wait(Context* c, cudaStream_t s) {
  if (!c->exchange_pending) return TLFEA_OK;
  TL_CUDA(cudaStreamWaitEvent(s, c->ev_exchanged, 0));
  c->exchange_pending = false;
  return TLFEA_OK;
}

}  // namespace tlfea
