// nccl_dyn.cpp — resolve NCCL at run time from the copy torch already loaded
// (venv NCCL 2.28.9), so a borrowed ncclComm_t is always used by the library that
// created it (/usr's 2.27.3 is a mismatched copy).  No link-time
// dependency: libdsp.so also loads on hosts without NCCL (world == 1 works).
#include <dlfcn.h>

#include <cstdlib>

#include "dsp_internal.h"

namespace dsp {

template <typename F>
static bool sym(void* h, const char* name, F* out) {
  *out = reinterpret_cast<F>(dlsym(h, name));
  return *out != nullptr;
}

bool nccl_load(NcclApi* api, std::string* err) {
  if (api->ok) return true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) {
    const char* path = std::getenv("DSP_NCCL_LIBRARY");
    if (path) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
  }
  if (!h) {
    if (err) *err = "libnccl.so.2 is not loaded in this process (import torch.distributed first or set DSP_NCCL_LIBRARY)";
    return false;
  }
  bool ok = sym(h, "ncclAlltoAll", &api->AlltoAll) && sym(h, "ncclAllGather", &api->AllGather) &&
            sym(h, "ncclGroupStart", &api->GroupStart) && sym(h, "ncclGroupEnd", &api->GroupEnd) &&
            sym(h, "ncclSend", &api->Send) && sym(h, "ncclRecv", &api->Recv) &&
            sym(h, "ncclGetErrorString", &api->GetErrorString);
  if (!ok) {
    // ncclAlltoAll appeared in NCCL 2.28; older libraries get grouped send/recv.
    api->AlltoAll = nullptr;
    ok = sym(h, "ncclAllGather", &api->AllGather) && sym(h, "ncclGroupStart", &api->GroupStart) &&
         sym(h, "ncclGroupEnd", &api->GroupEnd) && sym(h, "ncclSend", &api->Send) && sym(h, "ncclRecv", &api->Recv) &&
         sym(h, "ncclGetErrorString", &api->GetErrorString);
  }
  if (ok) {
    sym(h, "ncclCommGetAsyncError", &api->CommGetAsyncError);  // optional: health check only
    sym(h, "ncclAllReduce", &api->AllReduce);                  // optional: gradient reduction only
    sym(h, "ncclReduceScatter", &api->ReduceScatter);
  }
  if (!ok && err) *err = "libnccl.so.2 lacks the collectives dsp needs";
  api->ok = ok;
  return ok;
}

}  // namespace dsp
