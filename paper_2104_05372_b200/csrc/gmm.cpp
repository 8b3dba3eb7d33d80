// gmm.cpp — host side of the fused GMM kernel class (include/dexlet_gmm.h).
//
// One plan per (d = 64, K, n): device buffers for the parameters, the points,
// the operand images and the per-point betas; seven launches per objective +
// gradient (dx_gmm.cuh): prep_q, prep_x, fwd, lse (+ sum), bwd, moments,
// finish, with an NCCL all-reduce of the fp64 moments and of the log-likelihood
// sum between moments and finish when the points are sharded over ranks.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dexlet_gmm.h"
#include "runtime.hpp"

using dxrt::check;
using dxrt::setError;

namespace {

constexpr int D = 64;
constexpr int ICF = D * (D + 1) / 2;
constexpr int GC = 8;      // DXG_GC
constexpr int FXS = 2;     // DXG_FXS
constexpr int TM = 128;
constexpr int BC = 64;
constexpr int BN = 64;
constexpr int WP = 2 * (1 + 64);  // DXG_WP
constexpr int FMAX = 8;
constexpr int NXS = 5;  // DXG_NXS
constexpr int MOM = D * D + D + 1;
constexpr int FWD_SMEM = 2 * GC * 64 * 128 + FXS * 2 * TM * 128 + 1024;
inline int bwd4Smem() { return NXS * 2 * (BN * 128) + 2 * BN * 128 * 8 + 1024; }
constexpr int FIN_SMEM = 2 * D * (D + 1) * 8;
enum { K_ABSMAX, K_PREPQ, K_PREPX, K_FWD, K_LSE, K_SUM, K_BWD, K_MOM, K_FIN, K_N };
const char* kNames[K_N] = {"dx_gmm_absmax", "dx_gmm_prep_q", "dx_gmm_prep_x", "dx_gmm_fwd", "dx_gmm_lse",
                           "dx_gmm_sum",    "dx_gmm_bwd",    "dx_gmm_moments", "dx_gmm_finish"};

// Work split of the forward: units = NG groups x P tile ranges, CTAs take
// units round-robin; pick P (<= T tiles, >= 4 tiles per unit when possible)
// that balances whole units over the grid.
int pickP(int NG, long long T, int grid) {
  int best = 1;
  double bestEff = -1;
  for (int P = 1; P <= 4096 && P <= T; ++P) {
    long long units = (long long)NG * P;
    long long per = (units + grid - 1) / grid;
    double eff = (double)units / (double)(per * grid);
    if (T / P < 4 && P > 1) break;
    if (eff > bestEff + 1e-9) { bestEff = eff; best = P; }
    if (eff > 0.995 && T / P >= 16) break;
  }
  return best;
}
// Backward: units = NP pairs x P2 chunk ranges dealt round-robin; each unit
// is one partial slot, so a CTA may take at most FMAX units.
int pickP2(int NP, long long C, int grid) {
  int best = 1;
  double bestEff = -1;
  for (int P2 = 1; P2 <= 4096 && P2 <= C; ++P2) {
    long long units = (long long)NP * P2;
    long long per = (units + grid - 1) / grid;
    if (per > FMAX) break;
    double eff = (double)units / (double)(per * grid);
    if (eff > bestEff + 1e-9) { bestEff = eff; best = P2; }
  }
  return best;
}

double logGammaDistrib(double a, int p) {
  double out = 0.25 * p * (p - 1) * std::log(M_PI);
  for (int j = 1; j <= p; ++j) out += std::lgamma(a + 0.5 * (1 - j));
  return out;
}

}  // namespace

struct dxg_gmm {
  dxrt::Ctx* ctx = nullptr;
  CUmodule mod = nullptr;
  CUfunction fn[K_N] = {};
  int K = 0, NG = 0, NP = 0, P = 1, P2 = 1, gridF = 1, gridB = 1, gridL = 1;
  long long n = 0, ng = 0, npad = 0, T = 0, C = 0;
  CUdeviceptr alphas = 0, means = 0, icf = 0, x = 0;
  CUdeviceptr xmax = 0, svec = 0, dvec = 0, qimg = 0, bvec = 0, cvec = 0, ximg = 0, xtimg = 0, beta = 0, lse = 0, lpart = 0, lsum = 0;
  CUdeviceptr dpart = 0, wpart = 0, ppart = 0, mom = 0, dal = 0, dmu = 0, dicf = 0, prior = 0;
  bool timing = false;
  CUevent ev[K_N + 1] = {};
  float ms[K_N] = {};
  double gamma = 1.0;
  int wm = 0;
  int dr = D;  // the caller's dimension (<= 64; the kernels run padded to 64)
  bool haveGrad = false;
  ~dxg_gmm();
};

dxg_gmm::~dxg_gmm() {
  if (!ctx) return;
  ctx->makeCurrent();
  for (CUdeviceptr p : {alphas, means, icf, x, xmax, svec, dvec, qimg, bvec, cvec, ximg, xtimg, beta, lse, lpart, lsum, dpart, wpart,
                        ppart, mom, dal, dmu, dicf, prior})
    if (p) cuMemFree(p);
  for (auto& e : ev)
    if (e) cuEventDestroy(e);
}

static int allocZ(CUdeviceptr* p, size_t bytes) {
  int rc = check(cuMemAlloc(p, bytes ? bytes : 16), "cuMemAlloc(gmm)");
  if (rc) return rc;
  return check(cuMemsetD8(*p, 0, bytes ? bytes : 16), "cuMemsetD8(gmm)");
}

static int launch(dxg_gmm* g, int k, unsigned grid, unsigned block, unsigned smem, void** args) {
  if (g->timing) cuEventRecord(g->ev[k], g->ctx->stream);
  int rc = check(cuLaunchKernel(g->fn[k], grid, 1, 1, block, 1, 1, smem, g->ctx->stream, args, nullptr), kNames[k]);
  return rc;
}

extern "C" {

int dxg_gmm_create(dxc_ctx* cx, int d, int k, int64_t n_local, int64_t n_global, dxg_gmm** out) {
  if (!cx || !out) { setError("dxg_gmm_create: null argument"); return DXC_E_ARG; }
  if (d < 1 || d > D) { setError("dxg_gmm_create: d must be in 1..64"); return DXC_E_ARG; }
  if (k < 1 || n_local < 1 || n_global < n_local) { setError("dxg_gmm_create: bad sizes"); return DXC_E_ARG; }
  dxrt::Ctx* ctx = cx;
  int rc = ctx->makeCurrent();
  if (rc) return rc;
  auto* g = new dxg_gmm();
  g->ctx = ctx;
  g->dr = d;
  g->K = k;
  g->n = n_local;
  g->ng = n_global;
  g->NG = (k + GC - 1) / GC;
  g->NP = (k + 1) / 2;
  g->npad = (n_local + TM - 1) / TM * TM;
  g->T = g->npad / TM;
  g->C = g->npad / BC;
  const int sms = ctx->smCount;
  g->P = pickP(g->NG, g->T, sms);
  g->gridF = (int)std::min<long long>(sms, (long long)g->NG * g->P);
  // dx_gmm_bwd feeds two component pairs (a quad) from each X^T chunk
  g->P2 = pickP2((k + 3) / 4, g->C, sms);
  g->gridB = (int)std::min<long long>(sms, (long long)((k + 3) / 4) * g->P2);
  g->gridL = (int)std::min<long long>(8 * sms, (g->n + 255) / 256);  // 2048 threads per SM: more loads in flight
  std::string src = std::string(dxrt::gemmSource()) + "\n" + dxrt::gmmSource();
  if ((rc = ctx->loadModule(src, &g->mod))) { delete g; return rc; }
  for (int i = 0; i < K_N; ++i)
    if ((rc = check(cuModuleGetFunction(&g->fn[i], g->mod, kNames[i]), kNames[i]))) { delete g; return rc; }
  if ((rc = check(cuFuncSetAttribute(g->fn[K_FWD], CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, FWD_SMEM), "smem fwd")) ||
      (rc = check(cuFuncSetAttribute(g->fn[K_BWD], CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, bwd4Smem()), "smem bwd")) ||
      (rc = check(cuFuncSetAttribute(g->fn[K_FIN], CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, FIN_SMEM), "smem fin"))) {
    delete g;
    return rc;
  }
  const long long Kq = (long long)g->NG * GC;
  struct { CUdeviceptr* p; size_t b; } al[] = {
      {&g->alphas, (size_t)k * 4},
      {&g->means, (size_t)k * D * 4},
      {&g->icf, (size_t)k * ICF * 4},
      {&g->x, (size_t)n_local * D * 4},
      {&g->qimg, (size_t)Kq * 2 * 64 * 128},
      {&g->bvec, (size_t)Kq * D * 4},
      {&g->cvec, (size_t)Kq * 4},
      {&g->svec, (size_t)Kq * 4},
      {&g->dvec, (size_t)Kq * D * 4},
      {&g->xmax, 16},
      {&g->ximg, (size_t)g->npad * 2 * 128},
      {&g->xtimg, (size_t)g->npad * 2 * 128},
      {&g->beta, (size_t)k * g->npad * 4},
      {&g->lse, (size_t)g->npad * 4},
      {&g->lpart, (size_t)g->gridL * 8},
      {&g->lsum, 8},
      {&g->dpart, (size_t)g->gridB * FMAX * 256 * BN * 8},
      {&g->wpart, (size_t)g->gridB * FMAX * 2 * WP * 8},
      {&g->ppart, (size_t)g->gridB * FMAX * 4},
      {&g->mom, (size_t)k * MOM * 8},
      {&g->dal, (size_t)k * 8},
      {&g->dmu, (size_t)k * D * 8},
      {&g->dicf, (size_t)k * ICF * 8},
      {&g->prior, (size_t)k * 8},
  };
  for (auto& a : al)
    if ((rc = allocZ(a.p, a.b))) { delete g; return rc; }
  for (auto& e : g->ev)
    if ((rc = check(cuEventCreate(&e, CU_EVENT_DEFAULT), "cuEventCreate"))) { delete g; return rc; }
  *out = g;
  return DXC_OK;
}

int dxg_gmm_destroy(dxg_gmm* g) {
  delete g;
  return DXC_OK;
}

// d < 64 runs the 64-wide kernels on an exactly equivalent padded problem:
// padded coordinates of x and the means are 0, padded log-diagonals of Q are 0
// (q = 1) and padded strictly-lower entries are 0, so every y = Q(x - mu) gains
// only zero coordinates and beta, the responsibilities and the real gradient
// entries are unchanged.  The padded dimensions' Wishart terms (1/2 gamma^2 q^2
// with q = 1) and the d-dependent constants are corrected on the host.
// Packed strictly-lower index of (row j, column i), i < j < dd (ADBench order).
static inline long long trilIndex(int dd, int j, int i) {
  return (long long)i * dd - (long long)i * (i + 1) / 2 + (j - i - 1);
}

int dxg_gmm_set_params(dxg_gmm* g, const float* alphas, const float* means, const float* icf) {
  if (!g || !alphas || !means || !icf) { setError("dxg_gmm_set_params: null argument"); return DXC_E_ARG; }
  int rc = g->ctx->makeCurrent();
  if (rc) return rc;
  CUstream s = g->ctx->stream;
  if (g->dr == D) {
    if ((rc = check(cuMemcpyHtoDAsync(g->alphas, alphas, (size_t)g->K * 4, s), "H2D alphas")) ||
        (rc = check(cuMemcpyHtoDAsync(g->means, means, (size_t)g->K * D * 4, s), "H2D means")) ||
        (rc = check(cuMemcpyHtoDAsync(g->icf, icf, (size_t)g->K * ICF * 4, s), "H2D icf")))
      return rc;
    return DXC_OK;
  }
  const int d = g->dr, K = g->K, icfd = d * (d + 1) / 2;
  std::vector<float> mu((size_t)K * D, 0.f), ic((size_t)K * ICF, 0.f);
  for (int k = 0; k < K; ++k) {
    for (int j = 0; j < d; ++j) {
      mu[(size_t)k * D + j] = means[(size_t)k * d + j];
      ic[(size_t)k * ICF + j] = icf[(size_t)k * icfd + j];
    }
    for (int i = 0; i < d; ++i)
      for (int j = i + 1; j < d; ++j)
        ic[(size_t)k * ICF + D + trilIndex(D, j, i)] = icf[(size_t)k * icfd + d + trilIndex(d, j, i)];
  }
  // synchronous copies: the staging vectors die with this call
  if ((rc = check(cuMemcpyHtoDAsync(g->alphas, alphas, (size_t)K * 4, s), "H2D alphas")) ||
      (rc = check(cuMemcpyHtoD(g->means, mu.data(), mu.size() * 4), "H2D means")) ||
      (rc = check(cuMemcpyHtoD(g->icf, ic.data(), ic.size() * 4), "H2D icf")))
    return rc;
  return DXC_OK;
}

int dxg_gmm_set_points(dxg_gmm* g, const float* x) {
  if (!g || !x) { setError("dxg_gmm_set_points: null argument"); return DXC_E_ARG; }
  int rc = g->ctx->makeCurrent();
  if (rc) return rc;
  if (g->dr == D) return check(cuMemcpyHtoDAsync(g->x, x, (size_t)g->n * D * 4, g->ctx->stream), "H2D x");
  const int d = g->dr;
  std::vector<float> xp((size_t)g->n * D, 0.f);
  for (long long i = 0; i < g->n; ++i) std::memcpy(&xp[(size_t)i * D], x + (size_t)i * d, (size_t)d * 4);
  return check(cuMemcpyHtoD(g->x, xp.data(), xp.size() * 4), "H2D x");
}

int dxg_gmm_input_device_ptrs(dxg_gmm* g, void** alphas, void** means, void** icf, void** x) {
  if (alphas) *alphas = (void*)g->alphas;
  if (means) *means = (void*)g->means;
  if (icf) *icf = (void*)g->icf;
  if (x) *x = (void*)g->x;
  return DXC_OK;
}

int dxg_gmm_grad_device_ptrs(dxg_gmm* g, void** d_alphas, void** d_means, void** d_icf) {
  // fp64 gradients of the last run, d = 64 layout (valid after the run's work completes)
  if (d_alphas) *d_alphas = (void*)g->dal;
  if (d_means) *d_means = (void*)g->dmu;
  if (d_icf) *d_icf = (void*)g->dicf;
  return DXC_OK;
}

int dxg_gmm_run(dxg_gmm* g, double gamma, int wm, int want_grad) {
  if (!g) { setError("dxg_gmm_run: null plan"); return DXC_E_ARG; }
  if (!(gamma > 0.0) || wm < 0) { setError("dxg_gmm_run: Wishart gamma must be > 0 and m >= 0"); return DXC_E_ARG; }
  int rc = g->ctx->makeCurrent();
  if (rc) return rc;
  if (g->ng != g->n) {
    // a shard of the points: the moments and the log-likelihood must be
    // summed over exactly the ranks that hold the other shards
    if (!g->ctx->comm) {
      setError("dxg_gmm_run: sharded plan (n_global > n_local) needs dxc_comm_init on the context first");
      return DXC_E_ARG;
    }
    if (g->ctx->nranks < 2) {
      setError("dxg_gmm_run: sharded plan (n_global > n_local) over a one-rank communicator");
      return DXC_E_ARG;
    }
  }
  g->gamma = gamma;
  g->wm = wm;
  g->haveGrad = want_grad != 0;
  CUstream s = g->ctx->stream;
  int K = g->K;
  long long n = g->n, npad = g->npad, ng = g->ng;
  const unsigned Kq = (unsigned)(g->NG * GC);
  {
    if ((rc = check(cuMemsetD8Async(g->xmax, 0, 4, s), "memset xmax"))) return rc;
    long long cnt = n * D;
    void* a[] = {&g->x, &cnt, &g->xmax};
    if ((rc = launch(g, K_ABSMAX, (unsigned)std::min<long long>(4LL * g->ctx->smCount, (cnt / 4 + 255) / 256), 256, 0, a)))
      return rc;
  }
  {
    void* a[] = {&g->alphas, &g->means, &g->icf, &K, &g->xmax, &g->qimg, &g->bvec, &g->cvec, &g->svec, &g->dvec};
    if ((rc = launch(g, K_PREPQ, Kq, 256, 0, a))) return rc;
  }
  {
    void* a[] = {&g->x, &n, &g->xmax, &g->ximg, &g->xtimg};
    if ((rc = launch(g, K_PREPX, (unsigned)g->T, 256, 0, a))) return rc;
  }
  {
    int P = g->P;
    void* a[] = {&g->qimg, &g->ximg, &g->bvec, &g->cvec, &g->svec, &g->dvec, &K, &n, &npad, &P, &g->beta};
    if ((rc = launch(g, K_FWD, (unsigned)g->gridF, 320, FWD_SMEM, a))) return rc;
  }
  {
    void* a[] = {&g->beta, &K, &n, &npad, &g->lse, &g->lpart};
    if ((rc = launch(g, K_LSE, (unsigned)g->gridL, 256, 0, a))) return rc;
    int nl = g->gridL;
    void* b[] = {&g->lpart, &nl, &g->lsum};
    if ((rc = launch(g, K_SUM, 1, 256, 0, b))) return rc;
  }
  if (want_grad) {
    if ((rc = check(cuMemsetD8Async(g->ppart, 0xff, (size_t)g->gridB * FMAX * 4, s), "memset ppart"))) return rc;
    int P2 = g->P2;
    void* a[] = {&g->xtimg, &g->beta, &g->lse, &g->means, &g->xmax, &K, &n, &npad, &P2, &g->dpart, &g->wpart, &g->ppart};
    if ((rc = launch(g, K_BWD, (unsigned)g->gridB, 576, bwd4Smem(), a))) return rc;
    int nslot = g->gridB * FMAX;
    int G = 4;
    void* b[] = {&g->dpart, &g->wpart, &g->ppart, &nslot, &g->xmax, &G, &g->mom};
    if ((rc = launch(g, K_MOM, (unsigned)K, 256, 0, b))) return rc;
  }
  if (g->ctx->comm) {
    if ((rc = g->ctx->allreduceSum(g->lsum, 1, DXC_F64))) return rc;
    if (want_grad && (rc = g->ctx->allreduceSum(g->mom, (size_t)K * MOM, DXC_F64))) return rc;
  }
  {
    void* a[] = {&g->alphas, &g->means, &g->icf, &K, &ng, &g->mom, &g->gamma, &g->wm, &g->dal, &g->dmu, &g->dicf, &g->prior};
    if ((rc = launch(g, K_FIN, (unsigned)K, 256, FIN_SMEM, a))) return rc;
  }
  if (g->timing) cuEventRecord(g->ev[K_N], s);
  return DXC_OK;
}

int dxg_gmm_get(dxg_gmm* g, double* err, double* d_alphas, double* d_means, double* d_icf) {
  int rc = g->ctx->makeCurrent();
  if (rc) return rc;
  CUstream s = g->ctx->stream;
  if ((rc = check(cuStreamSynchronize(s), "gmm run"))) return rc;
  if (g->timing) {
    // stage k spans ev[k] .. next recorded event
    int order[K_N] = {K_ABSMAX, K_PREPQ, K_PREPX, K_FWD, K_LSE, K_SUM, K_BWD, K_MOM, K_FIN};
    for (int i = 0; i < K_N; ++i) {
      int a = order[i];
      int b = K_N;
      for (int j = i + 1; j < K_N; ++j) {
        if (!g->haveGrad && (order[j] == K_BWD || order[j] == K_MOM)) continue;
        b = order[j];
        break;
      }
      if (!g->haveGrad && (a == K_BWD || a == K_MOM)) { g->ms[a] = 0.f; continue; }
      float t = 0.f;
      cuEventElapsedTime(&t, g->ev[a], g->ev[b]);
      g->ms[a] = t;
    }
  }
  const int K = g->K;
  std::vector<double> prior(K);
  double lsum = 0.0;
  if ((rc = check(cuMemcpyDtoH(&lsum, g->lsum, 8), "D2H lsum")) ||
      (rc = check(cuMemcpyDtoH(prior.data(), g->prior, (size_t)K * 8), "D2H prior")))
    return rc;
  if (err) {
    std::vector<float> al(K);
    if ((rc = check(cuMemcpyDtoH(al.data(), g->alphas, (size_t)K * 4), "D2H alphas"))) return rc;
    double m0 = -1e300;
    for (float a : al) m0 = std::max(m0, (double)a);
    double se = 0.0;
    for (float a : al) se += std::exp((double)a - m0);
    const double lse_a = m0 + std::log(se);
    const int d = g->dr;
    const double nn = (double)g->ng;
    const double CONST = -nn * d * 0.5 * std::log(2 * M_PI);
    const int nw = d + g->wm + 1;
    const double Cw = nw * d * (std::log(g->gamma) - 0.5 * std::log(2.0)) - logGammaDistrib(0.5 * nw, d);
    double pr = 0.0;
    for (double p : prior) pr += p;
    pr -= (double)K * 0.5 * g->gamma * g->gamma * (D - d);  // padded dimensions: q = 1, icf = 0
    *err = CONST + lsum - nn * lse_a + pr - K * Cw;
  }
  if (d_alphas && (rc = check(cuMemcpyDtoH(d_alphas, g->dal, (size_t)K * 8), "D2H dalphas"))) return rc;
  if (g->dr == D) {
    if (d_means && (rc = check(cuMemcpyDtoH(d_means, g->dmu, (size_t)K * D * 8), "D2H dmeans"))) return rc;
    if (d_icf && (rc = check(cuMemcpyDtoH(d_icf, g->dicf, (size_t)K * ICF * 8), "D2H dicf"))) return rc;
    return DXC_OK;
  }
  const int d = g->dr, icfd = d * (d + 1) / 2;
  if (d_means) {
    std::vector<double> m((size_t)K * D);
    if ((rc = check(cuMemcpyDtoH(m.data(), g->dmu, m.size() * 8), "D2H dmeans"))) return rc;
    for (int k = 0; k < K; ++k)
      for (int j = 0; j < d; ++j) d_means[(size_t)k * d + j] = m[(size_t)k * D + j];
  }
  if (d_icf) {
    std::vector<double> c((size_t)K * ICF);
    if ((rc = check(cuMemcpyDtoH(c.data(), g->dicf, c.size() * 8), "D2H dicf"))) return rc;
    for (int k = 0; k < K; ++k) {
      for (int j = 0; j < d; ++j) d_icf[(size_t)k * icfd + j] = c[(size_t)k * ICF + j];
      for (int i = 0; i < d; ++i)
        for (int j = i + 1; j < d; ++j)
          d_icf[(size_t)k * icfd + d + trilIndex(d, j, i)] = c[(size_t)k * ICF + D + trilIndex(D, j, i)];
    }
  }
  return DXC_OK;
}

int dxg_gmm_enable_timing(dxg_gmm* g, int on) {
  g->timing = on != 0;
  return DXC_OK;
}

int dxg_gmm_kernel_times(dxg_gmm* g, float* ms, int cap, int* n) {
  for (int i = 0; i < K_N && i < cap; ++i) ms[i] = g->ms[i];
  if (n) *n = K_N;
  return DXC_OK;
}

static int oneShot(dxc_ctx* ctx, int d, int k, int64_t n, const float* alphas, const float* means, const float* icf,
                   const float* x, double gamma, int wm, bool grad, double* err, double* out) {
  dxg_gmm* g = nullptr;
  int rc = dxg_gmm_create(ctx, d, k, n, n, &g);
  if (rc) return rc;
  if (!(rc = dxg_gmm_set_params(g, alphas, means, icf)) && !(rc = dxg_gmm_set_points(g, x)) &&
      !(rc = dxg_gmm_run(g, gamma, wm, grad ? 1 : 0)))
    rc = grad ? dxg_gmm_get(g, err, out, out + k, out + k + (size_t)k * d) : dxg_gmm_get(g, err, nullptr, nullptr, nullptr);
  dxg_gmm_destroy(g);
  return rc;
}

int dxg_gmm_objective(dxc_ctx* ctx, int d, int k, int64_t n, const float* alphas, const float* means,
                      const float* icf, const float* x, double gamma, int wm, double* err) {
  return oneShot(ctx, d, k, n, alphas, means, icf, x, gamma, wm, false, err, nullptr);
}

int dxg_gmm_objective_grad(dxc_ctx* ctx, int d, int k, int64_t n, const float* alphas, const float* means,
                           const float* icf, const float* x, double gamma, int wm, double* err, double* grad) {
  return oneShot(ctx, d, k, n, alphas, means, icf, x, gamma, wm, true, err, grad);
}

}  // extern "C"
