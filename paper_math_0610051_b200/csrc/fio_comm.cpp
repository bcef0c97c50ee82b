// fio_comm.cpp -- the cross-GPU sum of the wedge-sharded apply (SURVEY.md 8(a) A6,
// BASELINE.json north_star (3)): L = sum_l L_l, each rank holding the partial
// sum over its own wedges, summed by one NCCL reduce-scatter that leaves rank r with output rows
// [r N/R, (r+1) N/R).  NCCL is resolved at run time (dlopen of libnccl.so.2, so a process that
// already loaded NCCL -- e.g. through torch -- shares that copy; a single-GPU user needs no NCCL at
// all).  Only the types come from <nccl.h>.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>

#include "fio_comm.h"
#include "fio_internal.h"

namespace fio {

namespace {
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*reduce_scatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                 cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      a.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return;
    }
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.reduce_scatter = reinterpret_cast<decltype(a.reduce_scatter)>(dlsym(h, "ncclReduceScatter"));
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.reduce_scatter && a.all_gather && a.error_string;
    if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
  });
  return a;
}

fio_status nccl_fail(const char* what, ncclResult_t r) {
  set_error(std::string(what) + ": " + api().error_string(r));
  return FIO_ENCCL;
}
}  // namespace

fio_status comm_unique_id(void* id_out) {
  const NcclApi& a = api();
  if (!a.ok) {
    set_error("fio_nccl_unique_id: " + a.why);
    return FIO_ENCCL;
  }
  ncclUniqueId id;
  ncclResult_t r = a.get_unique_id(&id);
  if (r != ncclSuccess) return nccl_fail("ncclGetUniqueId", r);
  std::memcpy(id_out, id.internal, sizeof(id.internal));
  return FIO_OK;
}

fio_status comm_create(const void* id_bytes, int nranks, int rank, void** comm_out) {
  *comm_out = nullptr;
  const NcclApi& a = api();
  if (!a.ok) {
    set_error("fio_plan: " + a.why);
    return FIO_ENCCL;
  }
  ncclUniqueId id;
  std::memcpy(id.internal, id_bytes, sizeof(id.internal));
  ncclComm_t c = nullptr;
  ncclResult_t r = a.comm_init_rank(&c, nranks, id, rank);  // collective: every rank's fio_plan joins
  if (r != ncclSuccess) return nccl_fail("ncclCommInitRank", r);
  *comm_out = c;
  return FIO_OK;
}

void comm_destroy(void* comm) {
  if (comm && api().ok) api().comm_destroy(static_cast<ncclComm_t>(comm));
}

fio_status comm_reduce_scatter(void* comm, const void* part, void* slab, size_t slab_reals, bool c64,
                               cudaStream_t s) {
  ncclResult_t r = api().reduce_scatter(part, slab, slab_reals, c64 ? ncclFloat32 : ncclFloat64, ncclSum,
                                        static_cast<ncclComm_t>(comm), s);
  if (r != ncclSuccess) return nccl_fail("ncclReduceScatter", r);
  return FIO_OK;
}

fio_status comm_all_gather(void* comm, void* full, int rank, size_t slab_reals, bool c64, cudaStream_t s) {
  const size_t rb = c64 ? sizeof(float) : sizeof(double);
  const void* mine = static_cast<const char*>(full) + rb * slab_reals * (size_t)rank;  // in place (NCCL)
  ncclResult_t r = api().all_gather(mine, full, slab_reals, c64 ? ncclFloat32 : ncclFloat64,
                                    static_cast<ncclComm_t>(comm), s);
  if (r != ncclSuccess) return nccl_fail("ncclAllGather", r);
  return FIO_OK;
}

}  // namespace fio
