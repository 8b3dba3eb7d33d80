// Device runtime behind the dxc_* C-ABI (include/dexlet_cuda.h).
//
// Replaces the reference's fork-join executor (Interp::parallelFor,
// reference proj/src/eval.cpp:310-369): instead of one std::thread per chunk
// with private overlays, each lowered nest is a kernel launched on one CUDA
// stream per GPU, and cross-GPU overlay merging becomes an NCCL all-reduce.
//
// CUDA driver API only (the primary context is shared with torch when both
// are loaded).  NVRTC compiles the per-program module for sm_100a; NCCL is
// dlopen'ed so the copy torch already mapped is reused.

#include "runtime.hpp"

#include <dlfcn.h>
#include <nvrtc.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <mutex>
#include <sstream>
#include <string>
#include <sys/stat.h>
#include <unistd.h>
#include <unordered_map>

#include "dx_device_src.inc"  // kDxDeviceSource: hand-written device runtime
#include "dx_gemm_src.inc"    // kDxGemmSource: tcgen05 GEMM for contraction nests
#include "dx_gmm_src.inc"     // kDxGmmSource: fused GMM objective + gradient

namespace dxrt {

thread_local std::string g_lastError;

void setError(const std::string& msg) { g_lastError = msg; }
const std::string& lastError() { return g_lastError; }

const char* deviceRuntimeSource() { return kDxDeviceSource; }
const char* gemmSource() { return kDxGemmSource; }
const char* gmmSource() { return kDxGmmSource; }

static bool g_cuInit = false;
static std::mutex g_mu;

int check(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return DXC_OK;
  const char* name = nullptr;
  const char* str = nullptr;
  cuGetErrorName(r, &name);
  cuGetErrorString(r, &str);
  if (!name) name = r == CUDA_ERROR_NO_DEVICE ? "CUDA_ERROR_NO_DEVICE (no driver/GPU)" : "?";
  setError(std::string(what) + ": " + name + " " + (str ? str : ""));
  return DXC_E_CUDA;
}

int ensureInit() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_cuInit) return DXC_OK;
  int rc = check(cuInit(0), "cuInit");
  if (rc) return rc;
  g_cuInit = true;
  return DXC_OK;
}

// ---------------------------------------------------------------------------
// NVRTC compile with an in-process cache keyed by the full source text and an
// optional on-disk cubin cache ($DEXLET_CACHE_DIR, default ~/.cache/dexlet).

static std::string hashHex(const std::string& s) {
  // FNV-1a 64 over the source, twice with different seeds (collision margin).
  uint64_t h1 = 1469598103934665603ull, h2 = 0x9e3779b97f4a7c15ull;
  for (unsigned char c : s) {
    h1 = (h1 ^ c) * 1099511628211ull;
    h2 = (h2 ^ c) * 0x100000001b3ull + 0x7f4a7c15;
  }
  char buf[40];
  std::snprintf(buf, sizeof buf, "%016llx%016llx", (unsigned long long)h1,
                (unsigned long long)h2);
  return buf;
}

static std::string cacheDir() {
  if (const char* d = std::getenv("DEXLET_CACHE_DIR")) return d;
  if (const char* h = std::getenv("HOME")) return std::string(h) + "/.cache/dexlet";
  return "";
}

static std::unordered_map<std::string, std::string> g_cubinCache;

int compileCubin(const std::string& source, std::string& cubin) {
  std::string full = std::string(kDxDeviceSource) + "\n" + source;
  std::string key = hashHex(full);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_cubinCache.find(key);
    if (it != g_cubinCache.end()) {
      cubin = it->second;
      return DXC_OK;
    }
  }
  std::string dir = cacheDir();
  std::string path = dir.empty() ? "" : dir + "/" + key + ".cubin";
  if (!path.empty() && !std::getenv("DEXLET_NO_DISK_CACHE")) {
    std::ifstream in(path, std::ios::binary);
    if (in) {
      std::stringstream ss;
      ss << in.rdbuf();
      cubin = ss.str();
      if (!cubin.empty()) {
        std::lock_guard<std::mutex> lk(g_mu);
        g_cubinCache[key] = cubin;
        return DXC_OK;
      }
    }
  }
  nvrtcProgram prog;
  nvrtcResult r = nvrtcCreateProgram(&prog, full.c_str(), "dexlet_nests.cu", 0,
                                     nullptr, nullptr);
  if (r != NVRTC_SUCCESS) {
    setError(std::string("nvrtcCreateProgram: ") + nvrtcGetErrorString(r));
    return DXC_E_CUDA;
  }
  const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17",
                        "-lineinfo", "--fmad=true", "-default-device",
                        "--extra-device-vectorization"};
  r = nvrtcCompileProgram(prog, sizeof(opts) / sizeof(opts[0]), opts);
  if (r != NVRTC_SUCCESS) {
    size_t logSize = 0;
    nvrtcGetProgramLogSize(prog, &logSize);
    std::string log(logSize, '\0');
    nvrtcGetProgramLog(prog, log.data());
    nvrtcDestroyProgram(&prog);
    if (log.size() > 6000) log = log.substr(0, 6000) + "\n...";
    setError(std::string("NVRTC compile failed: ") + nvrtcGetErrorString(r) + "\n" + log);
    return DXC_E_CUDA;
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  cubin.assign(n, '\0');
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    g_cubinCache[key] = cubin;
  }
  if (!path.empty() && !std::getenv("DEXLET_NO_DISK_CACHE")) {
    ::mkdir(dir.c_str(), 0755);
    std::string tmp = path + ".tmp" + std::to_string(::getpid());
    std::ofstream out(tmp, std::ios::binary);
    if (out) {
      out.write(cubin.data(), (std::streamsize)cubin.size());
      out.close();
      std::rename(tmp.c_str(), path.c_str());
    }
  }
  return DXC_OK;
}

// ---------------------------------------------------------------------------
// NCCL via dlopen.  Only the handful of entry points the allreduce needs.

typedef int ncclResult_t_;
// ncclUniqueId is a 128-byte struct passed BY VALUE to ncclCommInitRank (a
// `char[128]` parameter would decay to a pointer and break the call ABI)
struct NcclUniqueId_ {
  char internal[128];
};
struct NcclApi {
  void* lib = nullptr;
  ncclResult_t_ (*getUniqueId)(NcclUniqueId_*) = nullptr;
  ncclResult_t_ (*commInitRank)(void**, int, NcclUniqueId_, int) = nullptr;
  ncclResult_t_ (*allReduce)(const void*, void*, size_t, int, int, void*, CUstream) = nullptr;
  ncclResult_t_ (*allGather)(const void*, void*, size_t, int, void*, CUstream) = nullptr;
  ncclResult_t_ (*groupStart)() = nullptr;
  ncclResult_t_ (*groupEnd)() = nullptr;
  ncclResult_t_ (*commDestroy)(void*) = nullptr;
  const char* (*getErrorString)(ncclResult_t_) = nullptr;
};
static NcclApi g_nccl;

int loadNccl() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_nccl.lib) return DXC_OK;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  for (const char* n : names) {
    h = dlopen(n, RTLD_NOW | RTLD_NOLOAD);  // the copy torch mapped, if any
    if (h) break;
  }
  if (!h) {
    for (const char* n : names) {
      h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
  }
  if (!h) {
    setError(std::string("cannot load NCCL: ") + dlerror());
    return DXC_E_CUDA;
  }
  g_nccl.lib = h;
  g_nccl.getUniqueId = (decltype(g_nccl.getUniqueId))dlsym(h, "ncclGetUniqueId");
  g_nccl.commInitRank = (decltype(g_nccl.commInitRank))dlsym(h, "ncclCommInitRank");
  g_nccl.allReduce = (decltype(g_nccl.allReduce))dlsym(h, "ncclAllReduce");
  g_nccl.allGather = (decltype(g_nccl.allGather))dlsym(h, "ncclAllGather");
  g_nccl.groupStart = (decltype(g_nccl.groupStart))dlsym(h, "ncclGroupStart");
  g_nccl.groupEnd = (decltype(g_nccl.groupEnd))dlsym(h, "ncclGroupEnd");
  g_nccl.commDestroy = (decltype(g_nccl.commDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.getErrorString = (decltype(g_nccl.getErrorString))dlsym(h, "ncclGetErrorString");
  if (!g_nccl.getUniqueId || !g_nccl.commInitRank || !g_nccl.allReduce || !g_nccl.allGather ||
      !g_nccl.groupStart || !g_nccl.groupEnd) {
    setError("NCCL library lacks required symbols");
    g_nccl.lib = nullptr;
    return DXC_E_CUDA;
  }
  return DXC_OK;
}

static int ncclCheck(int r, const char* what) {
  if (r == 0) return DXC_OK;
  setError(std::string(what) + ": " +
           (g_nccl.getErrorString ? g_nccl.getErrorString(r) : "nccl error"));
  return DXC_E_CUDA;
}

int Ctx::allreduceSum(CUdeviceptr p, size_t count, int dtype) {
  if (!comm) return DXC_OK;
  // ncclDataType_t: ncclInt32=2, ncclUint32=3, ncclInt64=4, ncclFloat32=7, ncclFloat64=8
  int nd = 7;
  switch (dtype) {
    case DXC_F32: nd = 7; break;
    case DXC_F64: nd = 8; break;
    case DXC_I32: nd = 2; break;
    case DXC_U32: nd = 3; break;
    case DXC_I64: nd = 4; break;
    default: setError("allreduce: bad dtype"); return DXC_E_ARG;
  }
  return ncclCheck(g_nccl.allReduce((const void*)p, (void*)p, count, nd, /*ncclSum*/ 0,
                                    comm, stream),
                   "ncclAllReduce");
}

int Ctx::allgatherGroup(const std::vector<std::pair<CUdeviceptr, CUdeviceptr>>& sendRecv,
                        const std::vector<size_t>& counts, int dtype) {
  if (!comm) return DXC_OK;
  const int nd = dtype == DXC_F64 ? 8 : dtype == DXC_F32 ? 7 : dtype == DXC_I64 ? 4 : 2;
  int rc = ncclCheck(g_nccl.groupStart(), "ncclGroupStart");
  if (rc) return rc;
  for (size_t i = 0; i < sendRecv.size(); ++i) {
    rc = ncclCheck(g_nccl.allGather((const void*)sendRecv[i].first, (void*)sendRecv[i].second, counts[i], nd, comm,
                                    stream),
                   "ncclAllGather");
    if (rc) break;
  }
  const int rc2 = ncclCheck(g_nccl.groupEnd(), "ncclGroupEnd");
  return rc ? rc : rc2;
}

// ---------------------------------------------------------------------------

int Ctx::create(int dev, Ctx** out) {
  int rc = ensureInit();
  if (rc) return rc;
  auto* c = new Ctx();
  c->device = dev;
  if ((rc = check(cuDeviceGet(&c->dev, dev), "cuDeviceGet"))) { delete c; return rc; }
  if ((rc = check(cuDevicePrimaryCtxRetain(&c->ctx, c->dev), "cuDevicePrimaryCtxRetain"))) {
    delete c;
    return rc;
  }
  if ((rc = check(cuCtxSetCurrent(c->ctx), "cuCtxSetCurrent"))) { delete c; return rc; }
  if ((rc = check(cuStreamCreate(&c->stream, CU_STREAM_NON_BLOCKING), "cuStreamCreate"))) {
    delete c;
    return rc;
  }
  cuDeviceGetAttribute(&c->smCount, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, c->dev);
  cuDeviceGetAttribute(&c->maxSmemOptin,
                       CU_DEVICE_ATTRIBUTE_MAX_SHARED_MEMORY_PER_BLOCK_OPTIN, c->dev);
  *out = c;
  return DXC_OK;
}

int Ctx::makeCurrent() { return check(cuCtxSetCurrent(ctx), "cuCtxSetCurrent"); }

Ctx::~Ctx() {
  if (ctx) {
    cuCtxSetCurrent(ctx);
    for (auto& kv : modules) cuModuleUnload(kv.second);
    if (scratch) cuMemFree(scratch);
    if (stream) cuStreamDestroy(stream);
    if (comm && g_nccl.commDestroy) g_nccl.commDestroy(comm);
    cuDevicePrimaryCtxRelease(dev);
  }
}

int Ctx::loadModule(const std::string& source, CUmodule* out) {
  std::string key = hashHex(source);
  auto it = modules.find(key);
  if (it != modules.end()) {
    *out = it->second;
    return DXC_OK;
  }
  std::string cubin;
  int rc = compileCubin(source, cubin);
  if (rc) return rc;
  if ((rc = makeCurrent())) return rc;
  CUmodule m;
  if ((rc = check(cuModuleLoadData(&m, cubin.data()), "cuModuleLoadData"))) return rc;
  modules[key] = m;
  *out = m;
  return DXC_OK;
}

}  // namespace dxrt

// ===========================================================================
// C-ABI

using namespace dxrt;

struct dxc_buf {
  dxrt::Ctx* ctx;
  CUdeviceptr ptr;
  size_t bytes;
};
struct dxc_module {
  dxrt::Ctx* ctx;
  CUmodule mod;
};

extern "C" {

const char* dxc_last_error(void) { return g_lastError.c_str(); }

int dxc_device_count(int* out) {
  int rc = ensureInit();
  if (rc) return rc;
  return check(cuDeviceGetCount(out), "cuDeviceGetCount");
}

int dxc_init(int device, dxc_ctx** out) {
  Ctx* c = nullptr;
  int rc = Ctx::create(device, &c);
  if (rc) return rc;
  *out = static_cast<dxc_ctx*>(c);
  return DXC_OK;
}

int dxc_destroy(dxc_ctx* ctx) {
  delete static_cast<Ctx*>(ctx);
  return DXC_OK;
}

int dxc_sm_count(dxc_ctx* ctx, int* out) {
  *out = ctx->smCount;
  return DXC_OK;
}

void* dxc_stream(dxc_ctx* ctx) { return (void*)ctx->stream; }

int dxc_sync(dxc_ctx* ctx) {
  ctx->makeCurrent();
  return check(cuStreamSynchronize(ctx->stream), "cuStreamSynchronize");
}

int dxc_buf_alloc(dxc_ctx* ctx, size_t bytes, dxc_buf** out) {
  int rc = ctx->makeCurrent();
  if (rc) return rc;
  auto* b = new dxc_buf{ctx, 0, bytes};
  if ((rc = check(cuMemAlloc(&b->ptr, bytes ? bytes : 4), "cuMemAlloc"))) {
    delete b;
    return rc;
  }
  *out = b;
  return DXC_OK;
}

int dxc_buf_free(dxc_buf* b) {
  if (!b) return DXC_OK;
  b->ctx->makeCurrent();
  cuMemFree(b->ptr);
  delete b;
  return DXC_OK;
}

void* dxc_buf_ptr(dxc_buf* b) { return (void*)b->ptr; }

int dxc_buf_upload(dxc_buf* b, size_t off, const void* host, size_t bytes) {
  if (off + bytes > b->bytes) { setError("upload out of range"); return DXC_E_ARG; }
  b->ctx->makeCurrent();
  int rc = check(cuMemcpyHtoDAsync(b->ptr + off, host, bytes, b->ctx->stream), "cuMemcpyHtoD");
  if (rc) return rc;
  return check(cuStreamSynchronize(b->ctx->stream), "sync");
}

int dxc_buf_download(dxc_buf* b, size_t off, void* host, size_t bytes) {
  if (off + bytes > b->bytes) { setError("download out of range"); return DXC_E_ARG; }
  b->ctx->makeCurrent();
  int rc = check(cuMemcpyDtoHAsync(host, b->ptr + off, bytes, b->ctx->stream), "cuMemcpyDtoH");
  if (rc) return rc;
  return check(cuStreamSynchronize(b->ctx->stream), "sync");
}

int dxc_buf_zero(dxc_buf* b) {
  b->ctx->makeCurrent();
  return check(cuMemsetD8Async(b->ptr, 0, b->bytes, b->ctx->stream), "cuMemsetD8");
}

int dxc_host_alloc(size_t bytes, void** out) {
  int rc = ensureInit();
  if (rc) return rc;
  return check(cuMemHostAlloc(out, bytes ? bytes : 4, CU_MEMHOSTALLOC_PORTABLE), "cuMemHostAlloc");
}

int dxc_host_free(void* p) { return check(cuMemFreeHost(p), "cuMemFreeHost"); }

int dxc_module_compile(dxc_ctx* ctx, const char* source, dxc_module** out) {
  CUmodule m;
  int rc = ctx->loadModule(source, &m);
  if (rc) return rc;
  *out = new dxc_module{ctx, m};
  return DXC_OK;
}

int dxc_module_cubin(const char* source, void* out, size_t cap, size_t* size) {
  std::string cubin;
  int rc = compileCubin(source, cubin);
  if (rc) return rc;
  *size = cubin.size();
  if (out && cap >= cubin.size()) std::memcpy(out, cubin.data(), cubin.size());
  return DXC_OK;
}

int dxc_launch(dxc_ctx* ctx, dxc_module* mod, const char* kernel, unsigned grid,
               unsigned block, unsigned smem, void** args) {
  ctx->makeCurrent();
  CUfunction f;
  int rc = check(cuModuleGetFunction(&f, mod->mod, kernel), "cuModuleGetFunction");
  if (rc) return rc;
  if (smem > 48 * 1024) {
    rc = check(cuFuncSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem),
               "cuFuncSetAttribute");
    if (rc) return rc;
  }
  return check(cuLaunchKernel(f, grid, 1, 1, block, 1, 1, smem, ctx->stream, args, nullptr),
               "cuLaunchKernel");
}

int dxc_l2_flush(dxc_ctx* ctx, size_t bytes) {
  ctx->makeCurrent();
  if (ctx->scratchBytes < bytes) {
    if (ctx->scratch) cuMemFree(ctx->scratch);
    ctx->scratch = 0;
    ctx->scratchBytes = 0;
    int rc = check(cuMemAlloc(&ctx->scratch, bytes), "cuMemAlloc scratch");
    if (rc) return rc;
    ctx->scratchBytes = bytes;
  }
  static unsigned char flip = 0;
  flip ^= 0x5a;
  return check(cuMemsetD8Async(ctx->scratch, flip, bytes, ctx->stream), "l2 flush");
}

// Stream capture of a sequence of runs into one CUDA graph (bench / serving
// loops: K back-to-back evaluations launched without host work between them;
// programmatic-dependent-launch edges are kept in the graph).
int dxc_capture_begin(dxc_ctx* ctx) {
  ctx->makeCurrent();
  return check(cuStreamBeginCapture(ctx->stream, CU_STREAM_CAPTURE_MODE_THREAD_LOCAL), "cuStreamBeginCapture");
}

int dxc_capture_end(dxc_ctx* ctx, void** graph_exec) {
  ctx->makeCurrent();
  CUgraph g = nullptr;
  int rc = check(cuStreamEndCapture(ctx->stream, &g), "cuStreamEndCapture");
  if (rc) return rc;
  CUgraphExec e = nullptr;
  rc = check(cuGraphInstantiate(&e, g, 0), "cuGraphInstantiate");
  cuGraphDestroy(g);
  if (rc) return rc;
  *graph_exec = (void*)e;
  return DXC_OK;
}

int dxc_graph_launch(dxc_ctx* ctx, void* graph_exec) {
  ctx->makeCurrent();
  return check(cuGraphLaunch((CUgraphExec)graph_exec, ctx->stream), "cuGraphLaunch");
}

int dxc_graph_destroy(void* graph_exec) {
  return graph_exec ? check(cuGraphExecDestroy((CUgraphExec)graph_exec), "cuGraphExecDestroy") : DXC_OK;
}

int dxc_event_record(dxc_ctx* ctx, void** ev) {
  ctx->makeCurrent();
  CUevent e;
  int rc = check(cuEventCreate(&e, CU_EVENT_DEFAULT), "cuEventCreate");
  if (rc) return rc;
  rc = check(cuEventRecord(e, ctx->stream), "cuEventRecord");
  *ev = (void*)e;
  return rc;
}

int dxc_event_elapsed_ms(void* ev0, void* ev1, float* ms) {
  int rc = check(cuEventSynchronize((CUevent)ev1), "cuEventSynchronize");
  if (rc) return rc;
  return check(cuEventElapsedTime(ms, (CUevent)ev0, (CUevent)ev1), "cuEventElapsedTime");
}

int dxc_event_destroy(void* ev) { return check(cuEventDestroy((CUevent)ev), "cuEventDestroy"); }

int dxc_nccl_unique_id(void* out128) {
  int rc = loadNccl();
  if (rc) return rc;
  return ncclCheck(g_nccl.getUniqueId(static_cast<NcclUniqueId_*>(out128)), "ncclGetUniqueId");
}

int dxc_comm_init(dxc_ctx* ctx, const void* uid, int nranks, int rank) {
  int rc = loadNccl();
  if (rc) return rc;
  ctx->makeCurrent();
  NcclUniqueId_ id;
  std::memcpy(id.internal, uid, 128);
  void* comm = nullptr;
  rc = ncclCheck(g_nccl.commInitRank(&comm, nranks, id, rank), "ncclCommInitRank");
  if (rc) return rc;
  ctx->comm = comm;
  ctx->nranks = nranks;
  ctx->rank = rank;
  return DXC_OK;
}

int dxc_allreduce_sum(dxc_ctx* ctx, void* devptr, size_t count, int dtype) {
  ctx->makeCurrent();
  return ctx->allreduceSum((CUdeviceptr)devptr, count, dtype);
}

}  // extern "C"
