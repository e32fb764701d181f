// exchange.cu -- the per-step spike-bitmap exchange of a recurrent network
// sharded over GPUs (BASELINE config 5), inside the C ABI.
//
// The reference steps one process over the whole network (cortex.py:273-310:
// every spike of step t is visible to every synapse row at once).  Sharded,
// each rank owns a 32-aligned neuron range and the synapses whose TARGET it
// owns, so after its HH step a rank must see the spike bitmap of every rank:
// one all-gather of words_per_rank uint32 words per rank per step (4.8 KB in
// total at 38,586 neurons), then the local fixed-point delivery.  That
// all-gather is ncclAllGather on the caller's stream (NVLink / NVSwitch
// between the GPUs of a node), so it is captured into the same CUDA graph as
// the step kernels; hhb_spk_step fuses it with the delivery launch.
//
// NCCL is bound at run time (dlopen "libnccl.so.2"): inside a torch process
// that resolves to the NCCL torch already loaded; no link-time dependency, so
// the library still loads (and every single-GPU entry point works) where NCCL
// is absent -- hhb_spk_exchange_available() reports it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>

#include "hh_host.cuh"

namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*comm_abort)(ncclComm_t) = nullptr;
  ncclResult_t (*async_error)(ncclComm_t, ncclResult_t*) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    // prefer the NCCL already in the process (torch's), else the system one
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
#define HHB_SYM(field, name)                                         \
  a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name));     \
  if (!a.field) {                                                    \
    a.why = std::string("libnccl.so.2 lacks ") + name;               \
    return;                                                          \
  }
    HHB_SYM(get_unique_id, "ncclGetUniqueId")
    HHB_SYM(comm_init_rank, "ncclCommInitRank")
    HHB_SYM(all_gather, "ncclAllGather")
    HHB_SYM(comm_destroy, "ncclCommDestroy")
    HHB_SYM(comm_abort, "ncclCommAbort")
    HHB_SYM(async_error, "ncclCommGetAsyncError")
    HHB_SYM(error_string, "ncclGetErrorString")
#undef HHB_SYM
    a.ok = true;
  });
  return a;
}

int nccl_fail(const char* what, ncclResult_t r) {
  return hhb::fail(HHB_ECOMM, std::string(what) + ": " + api().error_string(r));
}

}  // namespace

struct hhb_exchange {
  ncclComm_t comm;
  int32_t rank, world;
  int64_t words_per_rank;
};

extern "C" {

int hhb_spk_exchange_available(void) { return api().ok ? 1 : 0; }

int hhb_spk_exchange_unique_id(void* id, int64_t bytes) {
  NcclApi& a = api();
  if (!a.ok) return hhb::fail(HHB_ENOTSUP, a.why);
  if (!id || bytes < int64_t(sizeof(ncclUniqueId))) return hhb::fail(HHB_EINVAL, "unique id buffer < 128 bytes");
  ncclUniqueId u;
  const ncclResult_t r = a.get_unique_id(&u);
  if (r != ncclSuccess) return nccl_fail("ncclGetUniqueId", r);
  memcpy(id, &u, sizeof(u));
  return HHB_OK;
}

int hhb_spk_exchange_init(const void* id, int32_t rank, int32_t world, int64_t words_per_rank,
                          hhb_exchange_t** out) {
  NcclApi& a = api();
  if (!a.ok) return hhb::fail(HHB_ENOTSUP, a.why);
  if (!id || !out || world < 1 || rank < 0 || rank >= world || words_per_rank < 1)
    return hhb::fail(HHB_EINVAL, "bad spk_exchange_init arguments");
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  ncclComm_t comm;
  const ncclResult_t r = a.comm_init_rank(&comm, world, u, rank);
  if (r != ncclSuccess) return nccl_fail("ncclCommInitRank", r);
  *out = new hhb_exchange{comm, rank, world, words_per_rank};
  return HHB_OK;
}

int hhb_spk_exchange_allgather(hhb_exchange_t* ex, const uint32_t* local_words, uint32_t* global_words,
                               void* stream) {
  if (!ex || !local_words || !global_words) return hhb::fail(HHB_EINVAL, "bad spk_exchange_allgather arguments");
  const ncclResult_t r = api().all_gather(local_words, global_words, size_t(ex->words_per_rank), ncclUint32,
                                          ex->comm, static_cast<cudaStream_t>(stream));
  if (r != ncclSuccess) return nccl_fail("ncclAllGather", r);
  return HHB_OK;
}

int hhb_spk_step(hhb_exchange_t* ex, const uint32_t* local_words, uint32_t* global_words, int64_t words_global,
                 const int64_t* offsets, const int32_t* targets, const int32_t* weights_fx, const int32_t* delays,
                 int64_t t, const int64_t* t_dev, int64_t depth, int64_t n_local, int64_t* ring, int64_t* scratch,
                 void* stream) {
  if (!ex) return hhb::fail(HHB_EINVAL, "spk_step: no exchange");
  if (words_global > ex->words_per_rank * ex->world)
    return hhb::fail(HHB_EINVAL, "spk_step: words_global exceeds the gathered words");
  int rc = hhb_spk_exchange_allgather(ex, local_words, global_words, stream);
  if (rc) return rc;
  return hhb_spike_deliver_flat(words_global, global_words, offsets, targets, weights_fx, delays, t, t_dev, depth,
                                n_local, ring, scratch, stream);
}

int hhb_spk_exchange_status(hhb_exchange_t* ex) {
  if (!ex) return hhb::fail(HHB_EINVAL, "spk_exchange_status: no exchange");
  ncclResult_t st = ncclSuccess;
  const ncclResult_t r = api().async_error(ex->comm, &st);
  if (r != ncclSuccess) return nccl_fail("ncclCommGetAsyncError", r);
  if (st != ncclSuccess && st != ncclInProgress) return nccl_fail("NCCL asynchronous error", st);
  return HHB_OK;
}

int hhb_spk_exchange_abort(hhb_exchange_t* ex) {
  if (!ex) return HHB_OK;
  const ncclResult_t r = api().comm_abort(ex->comm);
  delete ex;
  return r == ncclSuccess ? HHB_OK : nccl_fail("ncclCommAbort", r);
}

int hhb_spk_exchange_destroy(hhb_exchange_t* ex) {
  if (!ex) return HHB_OK;
  const ncclResult_t r = api().comm_destroy(ex->comm);
  delete ex;
  return r == ncclSuccess ? HHB_OK : nccl_fail("ncclCommDestroy", r);
}

}  // extern "C"
