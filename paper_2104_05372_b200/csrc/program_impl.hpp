// Internal: a lowered program bound to a device context.
#pragma once

#include <cuda.h>

#include <map>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "lower.hpp"
#include "runtime.hpp"

struct dxg_gmm;

namespace dexlet {
namespace dev {

size_t storageBytes(SK k, bool f64);

ExprPtr buildEntryApplication(const std::string& src, const std::string& entry,
                              std::vector<std::pair<Name, ValuePtr>>& params, ExprPtr* optimized);

struct Program {
  dxrt::Ctx* ctx = nullptr;
  Plan plan;
  std::string optimizedIR;
  std::string planText;
  std::string planDump;
  CUmodule mod = nullptr;
  bool prepared = false;
  bool checkFlag = true;
  bool allowCommMismatch = false;  // DXL_F_TEST_COMM_MISMATCH (single-device tests only)
  std::vector<CUdeviceptr> devptr;
  std::vector<CUdeviceptr> owned;
  std::set<int> boundInputs;
  std::vector<int> grids;
  std::vector<CUfunction> funcs;
  std::vector<std::pair<long long, long long>> ranges;
  std::vector<std::vector<char>> staging;
  CUfunction finFn[4] = {};
  CUfunction addFn[3] = {};  // f32 += f32, f64 += f64, f64 += f32
  CUfunction finF32D = nullptr;
  CUfunction cvtFn[2] = {};
  CUfunction checkIdxFn = nullptr;
  CUfunction rankFoldFn = nullptr;
  CUdeviceptr upFlags = 0;  // one int per input leaf: E-bounds seen by the upload check
  int numLeafFlags = 0;
  int readFlags(int* any);  // synchronizes; *any = error flag or any upload flag
  int launches = 0;
  std::vector<CUtensorMap> tmaps;                  // TMA descriptors (kernel args)
  std::map<std::pair<int, int>, int> tmapOf;        // (step, arg) -> tmaps index
  bool tmapsDirty = true;
  int buildTensorMaps();
  CUgraphExec graphExec = nullptr;
  bool useGraph = true;
  bool pdlSingle = false;  // one-launch plan: direct launch with PDL, no graph
  bool capturing = false;  // issue() is being captured into the graph (external event nodes)
  bool timing = false;
  std::vector<std::pair<CUevent, CUevent>> kernelEvents;  // per kernel step
  std::vector<int> kernelEventStep;
  std::string kernelNames;

  // The canonical ADBench GMM program (programs.gmm_program, the source
  // text with its constants; see matchGmmProgram in program.cpp) dispatches
  // to the fused GMM kernel class: inputs x / alphas / means / icf are the
  // kernel class's own device buffers, the table inputs must be the
  // canonical ones (checked on upload), the stabilizers are not needed.
  struct GmmMode {
    dxg_gmm* g = nullptr;
    long long n = 0;
    int d = 0, K = 0, m = 0;
    double gamma = 1.0;
  };
  GmmMode* gmm = nullptr;
  std::vector<int> gmmBufs;  // x, alphas, means, icf input buffers (the kernel class's)
  std::string gmmNote;
  double gmmErr = 0.0;
  bool gmmErrValid = false;

  int prepare();
  int run();
  int issue();  // enqueue every plan step on the context stream
  int launch(CUfunction f, unsigned grid, unsigned block, unsigned smem, void** args);
  std::vector<char> convertInit(const BufDecl& d) const;
  ~Program();
};

}  // namespace dev
}  // namespace dexlet
