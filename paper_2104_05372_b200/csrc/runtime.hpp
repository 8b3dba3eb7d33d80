// Internal runtime types shared by the C-ABI and the program lowering.
#pragma once

#include <cuda.h>

#include <map>
#include <string>
#include <utility>
#include <vector>

#include "dexlet_cuda.h"

namespace dxrt {

void setError(const std::string& msg);
const std::string& lastError();
int check(CUresult r, const char* what);
int ensureInit();
// NVRTC: prepend the device runtime, compile for sm_100a, return the cubin.
int compileCubin(const std::string& source, std::string& cubin);
const char* deviceRuntimeSource();
const char* gemmSource();  // dx_gemm.cuh: tcgen05 contraction kernels
const char* gmmSource();   // dx_gmm.cuh: fused GMM objective + gradient
int loadNccl();

struct Ctx {
  int device = 0;
  CUdevice dev = 0;
  CUcontext ctx = nullptr;
  CUstream stream = nullptr;
  int smCount = 148;
  int maxSmemOptin = 227 * 1024;
  void* comm = nullptr;  // ncclComm_t
  int nranks = 1;
  int rank = 0;
  std::map<std::string, CUmodule> modules;
  CUdeviceptr scratch = 0;
  size_t scratchBytes = 0;

  static int create(int dev, Ctx** out);
  int makeCurrent();
  int loadModule(const std::string& source, CUmodule* out);
  int allreduceSum(CUdeviceptr p, size_t count, int dtype);
  // grouped all-gathers (one NCCL launch): recv_i = [nranks][count_i]
  int allgatherGroup(const std::vector<std::pair<CUdeviceptr, CUdeviceptr>>& sendRecv,
                     const std::vector<size_t>& counts, int dtype);
  ~Ctx();
};

}  // namespace dxrt

// The C-ABI context handle is the runtime context itself.
struct dxc_ctx : dxrt::Ctx {};
