/* dexlet_gmm.h — C-ABI of the fused GMM objective + gradient kernel class
 * (BASELINE.json configs[2], SURVEY.md §7 kernel class 6).
 *
 * The reference language has no exp/log (reference
 * proj/include/dexlet/ir.hpp:121-124), so the ADBench GMM objective is not a
 * dexlet program and no reference interface exists for it.  These entry
 * points follow ADBench's own C++ interface (microsoft/ADBench
 * src/cpp/shared/gmm.h):
 *   void gmm_objective(int d, int k, int n, const double* alphas,
 *                      const double* means, const double* icf,
 *                      const double* x, Wishart wishart, double* err);
 * with the gradient laid out as ADBench's GMM Jacobian row
 * [d alphas (k) | d means (k*d) | d icf (k*d(d+1)/2)].
 * Parameters and points are fp32 on the device; err and the gradient are
 * fp64 (accumulated in fp64 from fp32 moments).  1 <= d <= 64: the kernels
 * are 64 wide, and d < 64 runs them on the exactly equivalent zero-padded
 * problem (padded coordinates 0, padded log-diagonal 0, padded lower entries
 * 0; the padded Wishart terms and d-dependent constants are removed on the
 * host).  ADBench's d = 128 sets are out of range.
 * Multi-GPU: each rank passes its own contiguous block of points (the
 * reference's chunk rule, eval.cpp:323-330) and the global n; the moments
 * and the log-likelihood sum are combined with NCCL (dxc_comm_init). */
#ifndef DEXLET_GMM_H
#define DEXLET_GMM_H

#include <stdint.h>

#include "dexlet_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dxg_gmm dxg_gmm;

/* Plan for dimension d (1..64), k components and n_local points of n_global on this rank
 * (n_local == n_global on one GPU).  Compiles the sm_100a module (NVRTC). */
int dxg_gmm_create(dxc_ctx* ctx, int d, int k, int64_t n_local, int64_t n_global, dxg_gmm** out);
int dxg_gmm_destroy(dxg_gmm* g);
/* Parameters (alphas [k], means [k][d], icf [k][d(d+1)/2]) and points
 * x [n_local][d], fp32, from host memory (pinned or pageable). */
int dxg_gmm_set_params(dxg_gmm* g, const float* alphas, const float* means, const float* icf);
int dxg_gmm_set_points(dxg_gmm* g, const float* x);
/* Device pointers of the input buffers (write them directly to skip the copy).
 * They hold the 64-wide layout: for d < 64, write padded data (see above). */
int dxg_gmm_input_device_ptrs(dxg_gmm* g, void** alphas, void** means, void** icf, void** x);
/* Objective and gradient, asynchronous on the context stream.  want_grad = 0
 * runs the objective only (prep + forward + log-sum-exp). */
int dxg_gmm_run(dxg_gmm* g, double wishart_gamma, int wishart_m, int want_grad);
/* Device pointers of the fp64 gradient buffers (64-wide layout; contents
 * valid once the run's work on the context stream completes). */
int dxg_gmm_grad_device_ptrs(dxg_gmm* g, void** d_alphas, void** d_means, void** d_icf);
/* Results of the last run (synchronizes).  Any output pointer may be NULL. */
int dxg_gmm_get(dxg_gmm* g, double* err, double* d_alphas, double* d_means, double* d_icf);
/* One-shot ADBench-shaped calls: set inputs, run, read back. */
int dxg_gmm_objective(dxc_ctx* ctx, int d, int k, int64_t n, const float* alphas, const float* means,
                      const float* icf, const float* x, double wishart_gamma, int wishart_m, double* err);
int dxg_gmm_objective_grad(dxc_ctx* ctx, int d, int k, int64_t n, const float* alphas, const float* means,
                           const float* icf, const float* x, double wishart_gamma, int wishart_m, double* err,
                           double* grad);
/* Per-kernel device time of the last run (absmax, prep_q, prep_x, fwd, lse, sum, bwd,
 * moments, finish) in ms when timing was enabled before the run. */
int dxg_gmm_enable_timing(dxg_gmm* g, int on);
int dxg_gmm_kernel_times(dxg_gmm* g, float* ms, int cap, int* n);

#ifdef __cplusplus
}
#endif

#endif /* DEXLET_GMM_H */
