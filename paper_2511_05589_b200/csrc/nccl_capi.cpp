// nccl_capi.cpp — the one collective of the sharded path:
// a SUM-allreduce of the four fp64 loss scalars after the kernels, plus the
// communicator helpers a C++ trainer without its own NCCL setup needs.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, preferring the copy the
// process already loaded, e.g. torch's), so the product library has no link-time
// NCCL dependency and a communicator created by the caller's NCCL is used by the
// same library. The resolved entry points are immutable after first use.
#include <dlfcn.h>
#include <nccl.h>  // types and prototypes only

#include <cstdint>
#include <cstring>
#include <string>

#include "../../include/copris_b200.h"
#include "internal.hpp"

using copris_b200::DeviceGuard;
using copris_b200::fail;

namespace {

struct Nccl {
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclCommInitAll) init_all = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclGetUniqueId) unique_id = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  bool ok = false;
};

template <typename F>
void sym(void* h, const char* name, F& f) {
  f = reinterpret_cast<F>(dlsym(h, name));
}

const Nccl& nccl() {
  static const Nccl n = [] {
    Nccl r;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) return r;
    sym(h, "ncclAllReduce", r.all_reduce);
    sym(h, "ncclCommInitAll", r.init_all);
    sym(h, "ncclCommInitRank", r.init_rank);
    sym(h, "ncclGetUniqueId", r.unique_id);
    sym(h, "ncclCommDestroy", r.destroy);
    sym(h, "ncclGetErrorString", r.error_string);
    r.ok = r.all_reduce && r.init_all && r.init_rank && r.unique_id && r.destroy && r.error_string;
    return r;
  }();
  return n;
}

int nccl_fail(const Nccl& n, ncclResult_t r, const char* where) {
  return fail(COPRIS_E_CUDA, std::string(where) + ": " + n.error_string(r));
}

}  // namespace

extern "C" {

int copris_allreduce_scalars(void* comm, double* d_buf4, void* stream) {
  copris_b200::NvtxRange nv("copris_allreduce_scalars");
  if (!comm || !d_buf4) return fail(COPRIS_E_INVALID, "null pointer");
  const Nccl& n = nccl();
  if (!n.ok) return fail(COPRIS_E_CUDA, "libnccl.so.2 not available");
  const ncclResult_t r = n.all_reduce(d_buf4, d_buf4, 4, ncclFloat64, ncclSum,
                                      static_cast<ncclComm_t>(comm),
                                      static_cast<cudaStream_t>(stream));
  return r == ncclSuccess ? COPRIS_OK : nccl_fail(n, r, "ncclAllReduce");
}

int copris_nccl_comm_init_all(int32_t n_dev, const int32_t* devices, void** out_comms) {
  if (n_dev < 1 || !devices || !out_comms) return fail(COPRIS_E_INVALID, "bad arguments");
  const Nccl& n = nccl();
  if (!n.ok) return fail(COPRIS_E_CUDA, "libnccl.so.2 not available");
  static_assert(sizeof(int) == sizeof(int32_t), "int");
  const ncclResult_t r = n.init_all(reinterpret_cast<ncclComm_t*>(out_comms), n_dev,
                                    reinterpret_cast<const int*>(devices));
  return r == ncclSuccess ? COPRIS_OK : nccl_fail(n, r, "ncclCommInitAll");
}

int copris_nccl_unique_id(uint8_t out_id[128]) {
  if (!out_id) return fail(COPRIS_E_INVALID, "null pointer");
  const Nccl& n = nccl();
  if (!n.ok) return fail(COPRIS_E_CUDA, "libnccl.so.2 not available");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId");
  ncclUniqueId id;
  const ncclResult_t r = n.unique_id(&id);
  if (r != ncclSuccess) return nccl_fail(n, r, "ncclGetUniqueId");
  std::memcpy(out_id, &id, sizeof(id));
  return COPRIS_OK;
}

int copris_nccl_comm_init_rank(int32_t device, int32_t n_ranks, const uint8_t id[128], int32_t rank,
                               void** out_comm) {
  if (!id || !out_comm || n_ranks < 1 || rank < 0 || rank >= n_ranks)
    return fail(COPRIS_E_INVALID, "bad arguments");
  const Nccl& n = nccl();
  if (!n.ok) return fail(COPRIS_E_CUDA, "libnccl.so.2 not available");
  DeviceGuard g(device);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  const ncclResult_t r = n.init_rank(&c, n_ranks, uid, rank);
  if (r != ncclSuccess) return nccl_fail(n, r, "ncclCommInitRank");
  *out_comm = c;
  return COPRIS_OK;
}

int copris_nccl_comm_destroy(void* comm) {
  if (!comm) return COPRIS_OK;
  const Nccl& n = nccl();
  if (!n.ok) return fail(COPRIS_E_CUDA, "libnccl.so.2 not available");
  const ncclResult_t r = n.destroy(static_cast<ncclComm_t>(comm));
  return r == ncclSuccess ? COPRIS_OK : nccl_fail(n, r, "ncclCommDestroy");
}

}  // extern "C"
