// Lazy binding of the CUDA driver API (libcuda.so.1 is dlopen'ed on first
// use) so libdexlet_cuda.so loads on machines without a driver: lowering and
// NVRTC compilation work there; any device call returns CUDA_ERROR_NO_DEVICE.
#include <cuda.h>
#include <dlfcn.h>

#define DX_STR2(x) #x
#define DX_STR(x) DX_STR2(x)

static void* dxCudaLib() {
  static void* h = [] {
    void* p = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
    if (!p) p = dlopen("libcuda.so", RTLD_NOW | RTLD_GLOBAL);
    return p;
  }();
  return h;
}

static void* dxSym(const char* n) {
  void* h = dxCudaLib();
  return h ? dlsym(h, n) : nullptr;
}

#define SHIM(name, params, args)                                                    \
  extern "C" CUresult CUDAAPI name params {                                        \
    using Fn = CUresult(CUDAAPI*) params;                                          \
    static Fn fn = (Fn)dxSym(DX_STR(name));                                        \
    if (!fn) return CUDA_ERROR_NO_DEVICE;                                          \
    return fn args;                                                                \
  }

SHIM(cuInit, (unsigned int f), (f))
SHIM(cuGetErrorName, (CUresult e, const char** s), (e, s))
SHIM(cuGetErrorString, (CUresult e, const char** s), (e, s))
SHIM(cuDeviceGet, (CUdevice* d, int o), (d, o))
SHIM(cuDeviceGetCount, (int* c), (c))
SHIM(cuDeviceGetAttribute, (int* v, CUdevice_attribute a, CUdevice d), (v, a, d))
SHIM(cuDevicePrimaryCtxRetain, (CUcontext* c, CUdevice d), (c, d))
SHIM(cuDevicePrimaryCtxRelease, (CUdevice d), (d))
SHIM(cuCtxSetCurrent, (CUcontext c), (c))
SHIM(cuStreamCreate, (CUstream* s, unsigned int f), (s, f))
SHIM(cuStreamDestroy, (CUstream s), (s))
SHIM(cuStreamSynchronize, (CUstream s), (s))
SHIM(cuModuleLoadData, (CUmodule* m, const void* img), (m, img))
SHIM(cuModuleUnload, (CUmodule m), (m))
SHIM(cuModuleGetFunction, (CUfunction* f, CUmodule m, const char* n), (f, m, n))
SHIM(cuFuncSetAttribute, (CUfunction f, CUfunction_attribute a, int v), (f, a, v))
SHIM(cuLaunchKernel,
     (CUfunction f, unsigned gx, unsigned gy, unsigned gz, unsigned bx, unsigned by, unsigned bz,
      unsigned smem, CUstream s, void** params, void** extra),
     (f, gx, gy, gz, bx, by, bz, smem, s, params, extra))
SHIM(cuLaunchKernelEx, (const CUlaunchConfig* c, CUfunction f, void** params, void** extra), (c, f, params, extra))
SHIM(cuOccupancyMaxActiveBlocksPerMultiprocessor, (int* n, CUfunction f, int b, size_t smem), (n, f, b, smem))
SHIM(cuMemAlloc, (CUdeviceptr* p, size_t n), (p, n))
SHIM(cuMemFree, (CUdeviceptr p), (p))
SHIM(cuMemHostAlloc, (void** p, size_t n, unsigned int f), (p, n, f))
SHIM(cuMemFreeHost, (void* p), (p))
SHIM(cuMemcpyHtoD, (CUdeviceptr d, const void* s, size_t n), (d, s, n))
SHIM(cuMemcpyDtoH, (void* d, CUdeviceptr s, size_t n), (d, s, n))
SHIM(cuMemcpyHtoDAsync, (CUdeviceptr d, const void* s, size_t n, CUstream st), (d, s, n, st))
SHIM(cuMemcpyDtoHAsync, (void* d, CUdeviceptr s, size_t n, CUstream st), (d, s, n, st))
SHIM(cuMemcpyDtoDAsync, (CUdeviceptr d, CUdeviceptr s, size_t n, CUstream st), (d, s, n, st))
SHIM(cuMemsetD8, (CUdeviceptr d, unsigned char v, size_t n), (d, v, n))
SHIM(cuMemsetD8Async, (CUdeviceptr d, unsigned char v, size_t n, CUstream st), (d, v, n, st))
SHIM(cuEventCreate, (CUevent* e, unsigned int f), (e, f))
SHIM(cuEventRecord, (CUevent e, CUstream s), (e, s))
SHIM(cuEventRecordWithFlags, (CUevent e, CUstream s, unsigned int f), (e, s, f))
SHIM(cuEventSynchronize, (CUevent e), (e))
SHIM(cuEventElapsedTime, (float* ms, CUevent a, CUevent b), (ms, a, b))
SHIM(cuEventDestroy, (CUevent e), (e))
SHIM(cuStreamBeginCapture, (CUstream s, CUstreamCaptureMode m), (s, m))
SHIM(cuStreamEndCapture, (CUstream s, CUgraph* g), (s, g))
SHIM(cuStreamIsCapturing, (CUstream s, CUstreamCaptureStatus* st), (s, st))
SHIM(cuGraphInstantiate, (CUgraphExec* e, CUgraph g, unsigned long long f), (e, g, f))
SHIM(cuGraphLaunch, (CUgraphExec e, CUstream s), (e, s))
SHIM(cuGraphExecDestroy, (CUgraphExec e), (e))
SHIM(cuGraphDestroy, (CUgraph g), (g))
SHIM(cuTensorMapEncodeTiled,
     (CUtensorMap * m, CUtensorMapDataType dt, cuuint32_t rank, void* addr, const cuuint64_t* dims,
      const cuuint64_t* strides, const cuuint32_t* box, const cuuint32_t* estr, CUtensorMapInterleave il,
      CUtensorMapSwizzle sw, CUtensorMapL2promotion l2, CUtensorMapFloatOOBfill oob),
     (m, dt, rank, addr, dims, strides, box, estr, il, sw, l2, oob))
