// COLL: the sharded fit's only exchange step -- an in-place SUM
// all-reduce of each device's packed fp64 statistics {sums | sumsq | counts}
// over NCCL (NVLink / NVSwitch on an 8 x B200 box).  The statistics are
// integer-valued doubles below 2^53, so any reduction order gives the same
// bits: the bundle is identical for 1, 2, 4 or 8 GPUs.
//
// NCCL is resolved at run time with dlopen("libnccl.so.2"): a process that
// already has NCCL (torch's) shares that copy, otherwise the system library is
// loaded.  libgnb.so itself has no link-time NCCL dependency, so importing it
// never changes which NCCL torch.distributed runs on.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <vector>

#include "gnb_internal.h"

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [h](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      return fn != nullptr;
    };
    api.ok = sym(api.get_unique_id, "ncclGetUniqueId") &&
             sym(api.comm_init_all, "ncclCommInitAll") &&
             sym(api.comm_init_rank, "ncclCommInitRank") &&
             sym(api.comm_destroy, "ncclCommDestroy") && sym(api.all_reduce, "ncclAllReduce") &&
             sym(api.group_start, "ncclGroupStart") && sym(api.group_end, "ncclGroupEnd") &&
             sym(api.error_string, "ncclGetErrorString");
  });
  return api;
}

int nccl_fail(const NcclApi& api, ncclResult_t r, const char* what) {
  char msg[256];
  snprintf(msg, sizeof(msg), "%s: %s", what, api.error_string ? api.error_string(r) : "nccl error");
  return gnb::set_error(GNB_ECUDA, msg);
}

int no_nccl() {
  return gnb::set_error(GNB_EUNSUPPORTED, "NCCL (libnccl.so.2) could not be loaded");
}

}  // namespace

struct gnb_comms {
  std::vector<ncclComm_t> comms;  // one per local device, in `devs` order
  std::vector<int> devs;
};

extern "C" {

int gnb_comms_unique_id(uint8_t* id) {
  const NcclApi& api = nccl();
  if (!api.ok) return no_nccl();
  if (!id) return gnb::set_error(GNB_EINVAL, "comms_unique_id: null buffer");
  static_assert(sizeof(ncclUniqueId) == GNB_COMMS_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId u;
  const ncclResult_t r = api.get_unique_id(&u);
  if (r != ncclSuccess) return nccl_fail(api, r, "ncclGetUniqueId");
  memcpy(id, &u, sizeof(u));
  return GNB_OK;
}

int gnb_comms_init(gnb_comms** out, int32_t ndev, const int32_t* devs) {
  if (!out || ndev < 1 || !devs) return gnb::set_error(GNB_EINVAL, "comms_init: bad arguments");
  *out = nullptr;
  const NcclApi& api = nccl();
  if (!api.ok) return no_nccl();
  auto* c = new gnb_comms();
  c->devs.assign(devs, devs + ndev);
  c->comms.resize(static_cast<size_t>(ndev));
  const ncclResult_t r = api.comm_init_all(c->comms.data(), ndev, c->devs.data());
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(api, r, "ncclCommInitAll");
  }
  *out = c;
  return GNB_OK;
}

int gnb_comms_init_rank(gnb_comms** out, int32_t nranks, int32_t rank, const uint8_t* id,
                        int32_t device) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks || !id)
    return gnb::set_error(GNB_EINVAL, "comms_init_rank: bad arguments");
  *out = nullptr;
  const NcclApi& api = nccl();
  if (!api.ok) return no_nccl();
  if (cudaSetDevice(device) != cudaSuccess)
    return gnb::set_error(GNB_ECUDA, "comms_init_rank: cudaSetDevice failed");
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  auto* c = new gnb_comms();
  c->devs.assign(1, device);
  c->comms.resize(1);
  const ncclResult_t r = api.comm_init_rank(&c->comms[0], nranks, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(api, r, "ncclCommInitRank");
  }
  *out = c;
  return GNB_OK;
}

void gnb_comms_destroy(gnb_comms* c) {
  if (!c) return;
  const NcclApi& api = nccl();
  if (api.ok)
    for (ncclComm_t m : c->comms) api.comm_destroy(m);
  delete c;
}

int gnb_fit_allreduce(gnb_comms* c, double* const* packed_stats, int64_t elems,
                      const uintptr_t* streams) {
  if (!c || !packed_stats || elems < 0 || !streams)
    return gnb::set_error(GNB_EINVAL, "fit_allreduce: bad arguments");
  const NcclApi& api = nccl();
  if (!api.ok) return no_nccl();
  const size_t n = c->comms.size();
  for (size_t i = 0; i < n; ++i)
    if (!packed_stats[i]) return gnb::set_error(GNB_EINVAL, "fit_allreduce: null buffer");
  ncclResult_t r = api.group_start();
  for (size_t i = 0; r == ncclSuccess && i < n; ++i)
    r = api.all_reduce(packed_stats[i], packed_stats[i], static_cast<size_t>(elems), ncclFloat64,
                       ncclSum, c->comms[i], reinterpret_cast<cudaStream_t>(streams[i]));
  const ncclResult_t r2 = api.group_end();
  if (r != ncclSuccess) return nccl_fail(api, r, "ncclAllReduce");
  if (r2 != ncclSuccess) return nccl_fail(api, r2, "ncclGroupEnd");
  return GNB_OK;
}

int32_t gnb_comms_size(const gnb_comms* c) { return c ? static_cast<int32_t>(c->comms.size()) : 0; }

}  // extern "C"
