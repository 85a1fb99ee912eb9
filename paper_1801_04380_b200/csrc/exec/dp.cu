// Data-parallel plumbing of the executor: NCCL loaded at run
// time, the unique-id / communicator entry points of the C ABI.  The bucketed
// all-reduce itself is compiled into the executor's program (executor.cu).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "nccl_dl.hpp"
#include "superneurons.h"

namespace sndp {
namespace {
std::once_flag g_once;
Nccl g_nccl;
std::string g_err;
bool g_ok = false;

template <class F>
bool sym(void* h, const char* name, F* out) {
  *out = reinterpret_cast<F>(dlsym(h, name));
  if (!*out) g_err = std::string("libnccl lacks ") + name;
  return *out != nullptr;
}
}  // namespace

const Nccl* nccl(std::string* err) {
  std::call_once(g_once, [] {
    const char* env = std::getenv("SN_NCCL_LIB");
    void* h = dlopen(env && *env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      g_err = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return;
    }
    g_ok = sym(h, "ncclGetUniqueId", &g_nccl.GetUniqueId) && sym(h, "ncclCommInitRank", &g_nccl.CommInitRank) &&
           sym(h, "ncclCommDestroy", &g_nccl.CommDestroy) && sym(h, "ncclAllReduce", &g_nccl.AllReduce) &&
           sym(h, "ncclGetVersion", &g_nccl.GetVersion) && sym(h, "ncclGetErrorString", &g_nccl.GetErrorString);
  });
  if (!g_ok && err) *err = g_err;
  return g_ok ? &g_nccl : nullptr;
}

}  // namespace sndp

namespace {
thread_local std::string g_dp_err;
int dp_fail(const std::string& m, int code) {
  g_dp_err = m;
  return code;
}
}  // namespace

extern "C" {

const char* sn_dp_last_error(void) { return g_dp_err.c_str(); }

int sn_dp_nccl_version(int32_t* version) {
  std::string err;
  const sndp::Nccl* n = sndp::nccl(&err);
  if (!n) return dp_fail(err, SN_ERR_CUDA);
  int v = 0;
  if (n->GetVersion(&v) != ncclSuccess) return dp_fail("ncclGetVersion failed", SN_ERR_CUDA);
  if (version) *version = v;
  return SN_OK;
}

int sn_dp_unique_id(sn_dp_id* out) {
  if (!out) return dp_fail("null argument", SN_ERR_OTHER);
  std::string err;
  const sndp::Nccl* n = sndp::nccl(&err);
  if (!n) return dp_fail(err, SN_ERR_CUDA);
  static_assert(sizeof(ncclUniqueId) == sizeof(out->bytes), "ncclUniqueId size");
  ncclUniqueId id;
  const ncclResult_t r = n->GetUniqueId(&id);
  if (r != ncclSuccess) return dp_fail(std::string("ncclGetUniqueId: ") + n->GetErrorString(r), SN_ERR_CUDA);
  std::memcpy(out->bytes, id.internal, sizeof(out->bytes));
  return SN_OK;
}

int sn_dp_comm_create(const sn_dp_id* id, int32_t world, int32_t rank, int32_t device, void** comm_out) {
  if (!id || !comm_out || world < 1 || rank < 0 || rank >= world) return dp_fail("bad argument", SN_ERR_OTHER);
  std::string err;
  const sndp::Nccl* n = sndp::nccl(&err);
  if (!n) return dp_fail(err, SN_ERR_CUDA);
  if (cudaSetDevice(device) != cudaSuccess) return dp_fail("cudaSetDevice failed", SN_ERR_CUDA);
  ncclUniqueId uid;
  std::memcpy(uid.internal, id->bytes, sizeof(uid.internal));
  ncclComm_t c = nullptr;
  const ncclResult_t r = n->CommInitRank(&c, world, uid, rank);
  if (r != ncclSuccess) return dp_fail(std::string("ncclCommInitRank: ") + n->GetErrorString(r), SN_ERR_CUDA);
  *comm_out = c;
  return SN_OK;
}

void sn_dp_comm_destroy(void* comm) {
  const sndp::Nccl* n = sndp::nccl(nullptr);
  if (n && comm) n->CommDestroy(static_cast<ncclComm_t>(comm));
}

}  // extern "C"
