// adg_comm.cu -- NCCL communicators for the multi-GPU exchange.
//
// libnccl.so.2 is loaded at run time (dlopen), so libadg.so has no link-time
// NCCL dependency and, inside a PyTorch process, shares the NCCL torch has
// already loaded.  An adg_collectives over NCCL enqueues every collective on
// the plan's stream: the exchange stays stream-ordered behind the screen.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "adg_internal.cuh"

namespace adg {
namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string error;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.error = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) api.error = std::string("libnccl.so.2 lacks ") + name;
    };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommInitAll, "ncclCommInitAll");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.AllReduce, "ncclAllReduce");
    sym(api.AllGather, "ncclAllGather");
    sym(api.GetErrorString, "ncclGetErrorString");
    api.ok = api.error.empty();
  });
  if (!api.ok) fail(ADG_ENCCL, api.error);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(ADG_ENCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

struct NcclComm {
  ncclComm_t comm = nullptr;
  int device = 0;
};

int nccl_all_reduce(void* user, void* buf, int64_t count, int32_t op, void* stream) {
  auto* c = static_cast<NcclComm*>(user);
  ncclDataType_t t = ncclUint64;
  ncclRedOp_t o = ncclSum;
  switch (op) {
    case ADG_SUM_U64: t = ncclUint64; o = ncclSum; break;
    case ADG_SUM_F64: t = ncclFloat64; o = ncclSum; break;
    case ADG_MAX_F32: t = ncclFloat32; o = ncclMax; break;
    case ADG_MAX_U64: t = ncclUint64; o = ncclMax; break;
    default: return 1;
  }
  if (count <= 0) return 0;
  return nccl().AllReduce(buf, buf, (size_t)count, t, o, c->comm, (cudaStream_t)stream) == ncclSuccess
             ? 0 : 2;
}

int nccl_all_gather(void* user, const void* send, void* recv, int64_t bytes, void* stream) {
  auto* c = static_cast<NcclComm*>(user);
  if (bytes <= 0) return 0;
  return nccl().AllGather(send, recv, (size_t)bytes, ncclUint8, c->comm, (cudaStream_t)stream) ==
                 ncclSuccess ? 0 : 2;
}

void fill(adg_collectives* out, NcclComm* c, int world, int rank) {
  out->world = world;
  out->rank = rank;
  out->user = c;
  out->all_reduce = nccl_all_reduce;
  out->all_gather = nccl_all_gather;
}

}  // namespace
}  // namespace adg

using namespace adg;

extern "C" {

adg_status adg_nccl_unique_id(uint8_t id_out[128]) {
  try {
    if (!id_out) fail(ADG_EINVAL, "nccl_unique_id: null out");
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(id_out, id.internal, sizeof(id.internal));
    return ADG_OK;
  } catch (const Error& e) {
    set_last_error(e.msg);
    return e.status;
  }
}

adg_status adg_comm_nccl_create(adg_ctx* ctx, int32_t world, int32_t rank, const uint8_t id[128],
                                adg_collectives* out) {
  try {
    if (!ctx || !id || !out || world < 1 || rank < 0 || rank >= world)
      fail(ADG_EINVAL, "comm_nccl_create: bad arguments");
    ADG_CUDA(cudaSetDevice(ctx->device));
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, sizeof(uid.internal));
    auto* c = new NcclComm();
    c->device = ctx->device;
    const ncclResult_t r = nccl().CommInitRank(&c->comm, world, uid, rank);
    if (r != ncclSuccess) {
      delete c;
      nccl_check(r, "ncclCommInitRank");
    }
    fill(out, c, world, rank);
    return ADG_OK;
  } catch (const Error& e) {
    set_last_error(e.msg);
    return e.status;
  }
}

adg_status adg_comm_nccl_create_all(int32_t ndev, const int32_t* devices, adg_collectives* comms) {
  try {
    if (ndev < 1 || !devices || !comms) fail(ADG_EINVAL, "comm_nccl_create_all: bad arguments");
    std::vector<ncclComm_t> cs((size_t)ndev);
    std::vector<int> devs(devices, devices + ndev);
    nccl_check(nccl().CommInitAll(cs.data(), ndev, devs.data()), "ncclCommInitAll");
    for (int r = 0; r < ndev; ++r) {
      auto* c = new NcclComm();
      c->comm = cs[(size_t)r];
      c->device = devs[(size_t)r];
      fill(&comms[r], c, ndev, r);
    }
    return ADG_OK;
  } catch (const Error& e) {
    set_last_error(e.msg);
    return e.status;
  }
}

adg_status adg_comm_nccl_destroy(adg_collectives* comm) {
  try {
    if (!comm || !comm->user) return ADG_OK;
    auto* c = static_cast<NcclComm*>(comm->user);
    if (c->comm) {
      cudaSetDevice(c->device);
      nccl_check(nccl().CommDestroy(c->comm), "ncclCommDestroy");
    }
    delete c;
    comm->user = nullptr;
    return ADG_OK;
  } catch (const Error& e) {
    set_last_error(e.msg);
    return e.status;
  }
}

}  // extern "C"
