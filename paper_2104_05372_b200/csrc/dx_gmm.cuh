// dx_gmm.cuh — fused GMM objective + gradient (BASELINE configs[2]; the
// "fused GMM" kernel class of SURVEY.md §7, item 6) on sm_100a tensor cores.
//
// Objective (ADBench gmm_objective, restated in oracle/gmm.py):
//   beta[k][i] = alpha_k + sum(q_k) - 0.5 || Q_k (x_i - mu_k) ||^2
//   err = CONST + sum_i logsumexp_k beta[k][i] - n lse(alpha) + wishart prior
// Gradient through the responsibilities g_ik = exp(beta[k][i] - lse_i):
//   W_k = sum_i g_ik and the centred moments sum_i g_ik (x_i - mu_k) and
//   sum_i g_ik (x_i - mu_k) x_i^T
// from which the per-component d alpha, d mu, d Q follow in closed form
// (dx_gmm_finish).  Both O(n K d^2) contractions run on tcgen05 (kind::f16,
// FP16 operands, FP32 accumulators in TMEM) in "fp16x3": every fp32 operand
// is a pair hi + lo of fp16 values (11-bit significands: the pair carries ~22
// bits) and the MMA accumulates hi*hi + hi*lo + lo*hi, an error of ~2^-22
// relative per product.  (bf16x3 carries only ~16 bits: its error in
// ||Q (x - mu)||^2 moves beta by ~1e-3 and the responsibilities with it.)
// fp16's range is handled by exact power-of-two scales: one for the points
// (from their max |x|, dx_gmm_absmax) and one per component for Q_k.
//
//   dx_gmm_absmax  max |x| over the points (their power-of-two scale)
//   dx_gmm_prep_q  per component: Q_k split into hi/lo SW128 K-major smem
//                  images (B operand), b_k = Q_k mu_k, c_k = alpha_k + sum q_k
//   dx_gmm_prep_x  points: X hi/lo images, 128-point tiles (forward A operand)
//                  and X^T hi/lo images, 64-point chunks (backward B operand)
//   dx_gmm_fwd     Y = X Q^T for 8 resident components per CTA; the epilogue
//                  reduces each 64-column block to beta (never stores Y);
//                  the MMAs carry the strictly lower L_k, the diagonal of Q_k
//                  is applied in fp32 in the epilogue
//   dx_gmm_lse     lse_i over the K betas of each point, sum_i lse_i
//   dx_gmm_bwd     per component pair: D[(k,b)][a] = sum_i z_ikb x_ia with
//                  z = g (x - mu_k), the A operand z^T produced by SIMT warps
//                  straight into tensor memory; W_k and m~_kb = sum_i z_ikb
//                  by the same warps in fp32/fp64
//   dx_gmm_finish  fp64 per component: moments -> gradients, prior, err
// The whole objective+gradient is deterministic: every reduction has a fixed
// order (per-CTA contiguous work ranges, partial slots folded in CTA order).
//
// Sizes: d = 64 is compiled in (DXG_D); n and K are runtime.

#define DXG_D 64
#define DXG_ICF (DXG_D * (DXG_D + 1) / 2)
#ifndef DXG_GC
#define DXG_GC 8                 // components resident per forward CTA (8; 4 measured slower: 5.4 vs 4.1 ms)
#endif
#define DXG_FXS (DXG_GC == 4 ? 4 : 2)  // forward X-tile stages
#define DXG_NH (DXG_GC / 4)          // N=256 MMA groups (TMEM halves) per tile
#define DXG_TM 128               // points per forward tile (MMA M)
#define DXG_BC 64                // points per backward chunk (MMA K extent)
#define DXG_BN 64                // backward MMA N: the 64 dims of X^T
#define DXG_WP (2 * (1 + DXG_D))  // backward per-slot sums: per component W and the centred m~
#ifndef DXG_PROMO
#define DXG_PROMO 1              // backward chunks per TMEM promotion (fp32 registers)
#endif
#define DXG_F64_EVERY 16         // promotions per fp64 spill (shared memory)
#define DXG_FMAX 8               // backward partial slots per CTA (= units per CTA)
#define DXG_FIN_SMEM (2 * DXG_D * (DXG_D + 1) * 8)
// Backward A operand (g * (x - mu)^T) in tensor memory (written by the SIMT
// producers with tcgen05.st, read by the MMA as [a-tmem]) instead of shared
// memory: takes its 32 KB/chunk of writes and 48 KB/chunk of MMA reads off
// the shared-memory pipe, which bounds the kernel otherwise.
#ifndef DXG_TMEM_A
#define DXG_TMEM_A 1
#endif
// TMEM columns of the backward kernel: D buffer b at 192 b with three
// independent accumulators (hi*hi, hi*lo, lo*hi at +0, +64, +128: the MMAs of
// a k-step do not wait on each other); A stage s (hi 32 columns, lo 32) at
// 384 + 64 s.
#define DXG_NXS 5                // X^T (+ beta, lse) stages of the backward TMA ring
#ifndef DXG_NACC
#define DXG_NACC 1               // TMEM accumulators per D buffer (1: merged, 3: hh / hl / lh)
#endif
#ifndef DXG_PN128  // pair kernel: one N=128 MMA over [X^T hi ; X^T lo] per A split
#define DXG_PN128 (DXG_TMEM_A && DXG_NACC == 1)
#endif
#define DXG_TD(b) ((b) * 128)  // D buffer b: 128 columns (products with x hi | x lo)
#define DXG_TACC(i) 0
#define DXG_NZS 4
#define DXG_TA(s) (256 + 64 * (s))

// ---- shared helpers ----------------------------------------------------------
// byte offset of element (row, col) of a bf16 K-major SWIZZLE_128B image whose
// rows are 128 bytes (64 bf16): 16-byte chunk index XOR (row & 7)
__device__ __forceinline__ unsigned dxg_sw(unsigned row, unsigned col) {
  return row * 128u + ((((col >> 3) ^ (row & 7u)) & 7u) << 4) + (col & 7u) * 2u;
}
// fp16 halves of a packed f16x2 word, as floats
__device__ __forceinline__ float dxg_h_lo(unsigned w) {
  float f;
  asm("{ .reg .b16 l, h; mov.b32 {l, h}, %1; cvt.f32.f16 %0, l; }" : "=f"(f) : "r"(w));
  return f;
}
__device__ __forceinline__ float dxg_h_hi(unsigned w) {
  float f;
  asm("{ .reg .b16 l, h; mov.b32 {l, h}, %1; cvt.f32.f16 %0, h; }" : "=f"(f) : "r"(w));
  return f;
}
// split two floats into packed f16x2 hi and lo words (x0 in the low half)
__device__ __forceinline__ void dxg_split2(float x0, float x1, unsigned& hi, unsigned& lo) {
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(hi) : "f"(x1), "f"(x0));
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(lo) : "f"(x1 - dxg_h_hi(hi)), "f"(x0 - dxg_h_lo(hi)));
}
__device__ __forceinline__ void dxg_split2v(float2 z, unsigned& hi, unsigned& lo) {  // f32x2 residual
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(hi) : "f"(z.y), "f"(z.x));
  const float2 r = dx_f2sub(z, make_float2(dxg_h_lo(hi), dxg_h_hi(hi)));
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(lo) : "f"(r.y), "f"(r.x));
}
// exact power-of-two scale s with max_abs * s < 2^14 (fp16 max is 65504)
__device__ __forceinline__ float dxg_scale_for(float max_abs) {
  if (!(max_abs > 0.f)) return 1.f;
  int e;
  frexpf(max_abs, &e);  // max_abs < 2^e
  return ldexpf(1.f, 14 - e);
}

template <int N>
__device__ __forceinline__ unsigned dxg_idesc_f16() {
  // c F32 (bit 4), a/b F16 (0 at bits 7, 10), both K-major, N>>3 at 17, M=128 (8 at 24)
  return (1u << 4) | ((unsigned)(N >> 3) << 17) | (8u << 24);
}
__device__ __forceinline__ void dxg_umma_f16(unsigned tmem, unsigned long long da, unsigned long long db,
                                              unsigned idesc, unsigned accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void dxg_umma_f16_ta(unsigned tmem, unsigned ta, unsigned long long db, unsigned idesc,
                                                unsigned accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
      "r"(ta), "l"(db), "r"(idesc), "r"(accumulate));
}
#define DXG_TMEM_ST16(taddr, v)                                                                                \
  asm volatile(                                                                                                \
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" \
      ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),      \
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])              \
      : "memory")
__device__ __forceinline__ void dxg_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void dxg_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void dxg_named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

#define DXG_TMEM_LD16(taddr, v)                                                                              \
  asm volatile(                                                                                              \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),      \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]) \
      : "r"(taddr))

#define DXG_TMEM_LD8(taddr, v)                                                                     \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"                   \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]) \
               : "r"(taddr))

// ---- max |x| (bit pattern of a non-negative float: atomicMax on u32 orders it)
extern "C" __global__ void __launch_bounds__(256) dx_gmm_absmax(const float* __restrict__ x, long long cnt,
                                                                unsigned* __restrict__ out) {
  float m = 0.f;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt / 4; i += (long long)gridDim.x * blockDim.x) {
    const float4 v = reinterpret_cast<const float4*>(x)[i];
    m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(DX_FULL, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

// ---- prep: per-component Q images, b_k = Q_k mu_k, c_k = alpha_k + sum q_k ----
// qimg layout: [Kpad/8 groups][split hi,lo][512 rows = 8 comps x 64][128 B];
// row j*64 + r of group g holds row r of sq_k Q_{8g+j} (zero for k >= K);
// bvec = sx sq_k Q_k mu_k, dvec = sq_k diag(Q_k), svec = (sx sq_k)^-2: the
// forward forms sx sq_k Q_k (x - mu_k) = MMA(L) + dvec * (sx x) - bvec.
extern "C" __global__ void __launch_bounds__(256) dx_gmm_prep_q(const float* alphas, const float* means,
                                                                const float* icf, int K, const unsigned* xmax,
                                                                unsigned char* qimg, float* bvec, float* cvec,
                                                                float* svec, float* dvec) {
  __shared__ double Q[DXG_D][DXG_D + 1];
  __shared__ float qmax[8];
  const int k = blockIdx.x;
  const bool live = k < K;
  for (int e = threadIdx.x; e < DXG_D * DXG_D; e += blockDim.x) {
    const int r = e / DXG_D, c = e % DXG_D;
    double v = 0.0;
    if (live) {
      const float* q = icf + (long long)k * DXG_ICF;
      if (r == c) v = exp((double)q[r]);
      else if (r > c) v = (double)q[DXG_D + c * (DXG_D - 1) - c * (c - 1) / 2 + (r - c - 1)];
    }
    Q[r][c] = v;
  }
  __syncthreads();
  float m = 0.f;
  for (int e = threadIdx.x; e < DXG_D * DXG_D; e += blockDim.x) m = fmaxf(m, fabsf((float)Q[e / DXG_D][e % DXG_D]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(DX_FULL, m, o));
  if ((threadIdx.x & 31) == 0) qmax[threadIdx.x >> 5] = m;
  __syncthreads();
  m = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, qmax[w]);
  const double sq = (double)dxg_scale_for(m), sx = (double)dxg_scale_for(__uint_as_float(*xmax));
  const int g = k / DXG_GC, j = k % DXG_GC;
  unsigned char* hi = qimg + (long long)g * 2 * (DXG_GC * 64 * 128);
  unsigned char* lo = hi + DXG_GC * 64 * 128;
  for (int e = threadIdx.x; e < DXG_D * DXG_D / 2; e += blockDim.x) {
    const int r = e / (DXG_D / 2), c = 2 * (e % (DXG_D / 2));
    unsigned h, l;
    // the tensor cores see only the strictly lower L_k; the diagonal is
    // applied exactly in the forward epilogue (dvec), which keeps the TMEM
    // accumulation small (~|L x|) and beta accurate to fp32 level
    dxg_split2(c == r ? 0.f : (float)(Q[r][c] * sq), c + 1 == r ? 0.f : (float)(Q[r][c + 1] * sq), h, l);
    const unsigned off = dxg_sw((unsigned)(j * 64 + r), (unsigned)c);
    *reinterpret_cast<unsigned*>(hi + off) = h;
    *reinterpret_cast<unsigned*>(lo + off) = l;
  }
  if (threadIdx.x < DXG_D) {
    const int r = threadIdx.x;
    double s = 0.0;
    if (live)
      for (int c = 0; c <= r; ++c) s += Q[r][c] * (double)means[(long long)k * DXG_D + c];
    bvec[(long long)k * DXG_D + r] = (float)(s * sq * sx);
  }
  if (threadIdx.x == 0) svec[k] = (float)(1.0 / (sq * sx * sq * sx));
  if (threadIdx.x < DXG_D) dvec[(long long)k * DXG_D + threadIdx.x] = (float)(Q[threadIdx.x][threadIdx.x] * sq);
  if (threadIdx.x == 0) {
    double s = 0.0;
    if (live) {
      s = alphas[k];
      for (int c = 0; c < DXG_D; ++c) s += (double)icf[(long long)k * DXG_ICF + c];
    }
    cvec[k] = (float)s;
  }
}

// ---- prep: point images ----------------------------------------------------------
// ximg:  [tiles of 128 points][hi 16 KB][lo 16 KB], row = point, col = dim
// xtimg: [chunks of 64 points][hi 8 KB][lo 8 KB], row = dim, col = point
// Rows past n are zero.  One block = one 128-point tile (two 64-point chunks).
extern "C" __global__ void __launch_bounds__(256) dx_gmm_prep_x(const float* x, long long n, const unsigned* xmax,
                                                                unsigned char* ximg, unsigned char* xtimg) {
  __shared__ float xs[DXG_TM][DXG_D + 1];
  const long long t = blockIdx.x;
  const float sx = dxg_scale_for(__uint_as_float(*xmax));
  for (int e = threadIdx.x; e < DXG_TM * DXG_D / 4; e += blockDim.x) {
    const int r = e / (DXG_D / 4), c4 = e % (DXG_D / 4);
    const long long p = t * DXG_TM + r;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (p < n) v = *reinterpret_cast<const float4*>(x + p * DXG_D + 4 * c4);
    v.x *= sx; v.y *= sx; v.z *= sx; v.w *= sx;  // exact (power of two)
    xs[r][4 * c4] = v.x;
    xs[r][4 * c4 + 1] = v.y;
    xs[r][4 * c4 + 2] = v.z;
    xs[r][4 * c4 + 3] = v.w;
  }
  __syncthreads();
  unsigned char* xh = ximg + t * 2 * (DXG_TM * 128);
  unsigned char* xl = xh + DXG_TM * 128;
  for (int e = threadIdx.x; e < DXG_TM * DXG_D / 2; e += blockDim.x) {
    const int r = e / (DXG_D / 2), c = 2 * (e % (DXG_D / 2));
    unsigned h, l;
    dxg_split2(xs[r][c], xs[r][c + 1], h, l);
    const unsigned off = dxg_sw((unsigned)r, (unsigned)c);
    *reinterpret_cast<unsigned*>(xh + off) = h;
    *reinterpret_cast<unsigned*>(xl + off) = l;
  }
  for (int e = threadIdx.x; e < 2 * DXG_D * (DXG_BC / 2); e += blockDim.x) {
    const int ch = e / (DXG_D * (DXG_BC / 2));
    const int rem = e % (DXG_D * (DXG_BC / 2));
    const int a = rem / (DXG_BC / 2), p = 2 * (rem % (DXG_BC / 2));
    unsigned h, l;
    dxg_split2(xs[ch * DXG_BC + p][a], xs[ch * DXG_BC + p + 1][a], h, l);
    unsigned char* th = xtimg + (t * 2 + ch) * 2 * (DXG_D * 128);
    const unsigned off = dxg_sw((unsigned)a, (unsigned)p);
    *reinterpret_cast<unsigned*>(th + off) = h;
    *reinterpret_cast<unsigned*>(th + DXG_D * 128 + off) = l;
  }
}

// ---- forward: beta[k][i] for every point and component ---------------------------
// Work unit = (component group g of 8, contiguous tile range p of the points);
// CTA c takes units c, c + grid, ...  Warp 0: bulk-copy producer (Q group once
// per unit, X tiles through a 2-stage ring); warp 1: MMA issuer; warps 2-9:
// epilogue (warp w drains TMEM lanes 32*(w%4)..+31 = tile rows, of one half).  TMEM: 512
// columns = 8 components x 64, in two halves of 4 components that alternate
// between MMA and epilogue.
#define DXG_FWD_SMEM (2 * DXG_GC * 64 * 128 + DXG_FXS * 2 * DXG_TM * 128 + 1024)
extern "C" __global__ void __launch_bounds__(320, 1)
    dx_gmm_fwd(const unsigned char* __restrict__ qimg, const unsigned char* __restrict__ ximg,
               const float* __restrict__ bvec, const float* __restrict__ cvec, const float* __restrict__ svec,
               const float* __restrict__ dvec, int K, long long n,
               long long npad, int P, float* __restrict__ beta) {
  extern __shared__ __align__(1024) unsigned char dxg_smem_raw[];
  unsigned char* smem = dxg_smem_raw + ((1024u - (dx_smem_addr(dxg_smem_raw) & 1023u)) & 1023u);
  unsigned char* qs = smem;                                // 128 KB: hi (64 KB) then lo
  unsigned char* xsm = smem + 2 * DXG_GC * 64 * 128;       // DXG_FXS stages x 32 KB
  __shared__ __align__(8) unsigned long long xfull[DXG_FXS], xempty[DXG_FXS], tfull[2], tempty[2], qfull, qempty;
  __shared__ __align__(16) float bsm[DXG_GC][DXG_D], dsm[DXG_GC][DXG_D];
  __shared__ float csm[DXG_GC], ssm[DXG_GC];
  __shared__ unsigned tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NG = (K + DXG_GC - 1) / DXG_GC;
  const long long T = npad / DXG_TM;
  const int units = NG * P;

  if (threadIdx.x == 0) {
    for (int s = 0; s < DXG_FXS; ++s) {
      dx_mbar_init(&xfull[s], 1);
      dx_mbar_init(&xempty[s], 9);  // MMA commit + the 8 epilogue warps (they read x)
    }
    for (int s = 0; s < 2; ++s) {
      dx_mbar_init(&tfull[s], 1);
      dx_mbar_init(&tempty[s], 32 / DXG_GC);  // epilogue warps per TMEM buffer
    }
    dx_mbar_init(&qfull, 1);
    dx_mbar_init(&qempty, 1);
    dx_fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dx_smem_addr(&tmem_base)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  dxg_fence_before();
  __syncthreads();
  dxg_fence_after();
  const unsigned tmem = tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0, qn = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++qn) {
        const int g = u / P, p = u % P;
        const long long t0 = (long long)p * T / P, t1 = (long long)(p + 1) * T / P;
        if (qn > 0) dx_mbar_wait_bounded(&qempty, (unsigned)((qn - 1) & 1));
        dx_mbar_expect_tx(&qfull, 2 * DXG_GC * 64 * 128);
        dx_bulk_g2s(qs, qimg + (long long)g * 2 * DXG_GC * 64 * 128, 2 * DXG_GC * 64 * 128, &qfull);
        for (long long t = t0; t < t1; ++t, ++it) {
          const int s = it % DXG_FXS;
          if (it >= DXG_FXS) dx_mbar_wait_bounded(&xempty[s], (unsigned)(((it / DXG_FXS) - 1) & 1));
          dx_mbar_expect_tx(&xfull[s], 2 * DXG_TM * 128);
          dx_bulk_g2s(xsm + s * 2 * DXG_TM * 128, ximg + t * 2 * DXG_TM * 128, 2 * DXG_TM * 128, &xfull[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const unsigned idesc = dxg_idesc_f16<256>();
      const unsigned qaddr = dx_smem_addr(qs), xaddr = dx_smem_addr(xsm);
      int it = 0, qn = 0, tt = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++qn) {
        const int p = u % P;
        const long long t0 = (long long)p * T / P, t1 = (long long)(p + 1) * T / P;
        dx_mbar_wait_bounded(&qfull, (unsigned)(qn & 1));
        dxg_fence_after();
        for (long long t = t0; t < t1; ++t, ++it) {
          const int s = it % DXG_FXS;
          dx_mbar_wait_bounded(&xfull[s], (unsigned)((it / DXG_FXS) & 1));
          dxg_fence_after();
          const unsigned xa = xaddr + (unsigned)(s * 2 * DXG_TM * 128);
          for (int h = 0; h < DXG_NH; ++h, ++tt) {
            const int bb = tt & 1;  // TMEM buffer (with DXG_GC = 4: alternates per tile)
            if (tt >= 2) dx_mbar_wait_bounded(&tempty[bb], (unsigned)(((tt >> 1) - 1) & 1));
            dxg_fence_after();
            const unsigned td = tmem + (unsigned)(bb * 256);
            const unsigned qh = qaddr + (unsigned)(h * 256 * 128), ql = qh + DXG_GC * 64 * 128;
#pragma unroll
            for (int kk = 0; kk < DXG_D / 16; ++kk) {
              const unsigned long long ah = dx_umma_desc_sw128(xa + kk * 32);
              const unsigned long long al = dx_umma_desc_sw128(xa + DXG_TM * 128 + kk * 32);
              const unsigned long long bh = dx_umma_desc_sw128(qh + kk * 32);
              const unsigned long long bl = dx_umma_desc_sw128(ql + kk * 32);
              dxg_umma_f16(td, ah, bh, idesc, kk > 0);
              dxg_umma_f16(td, ah, bl, idesc, 1u);
              dxg_umma_f16(td, al, bh, idesc, 1u);
            }
            dx_umma_commit(&tfull[bb]);
          }
          dx_umma_commit(&xempty[s]);
        }
        dx_umma_commit(&qempty);  // Q group free once every MMA of this unit retired
      }
    }
  } else {
    // epilogue: warps 2..9; warp w drains TMEM lane quarter w % 4 for the
    // components [hsel * GC/2, (hsel + 1) * GC/2) of the resident group
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int hsel = (warp - 2) >> 2;
    const int et = threadIdx.x - 64;  // 0..255
    const unsigned lanebase = tmem + ((unsigned)(q * 32) << 16);
    int tt = 0, it = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int g = u / P, p = u % P;
      const long long t0 = (long long)p * T / P, t1 = (long long)(p + 1) * T / P;
      dxg_named_sync(1, 256);  // previous unit's epilogue is done with bsm/csm
      for (int e = et; e < DXG_GC * DXG_D; e += 256) {
        const int j = e / DXG_D, c = e % DXG_D;
        const int k = g * DXG_GC + j;
        bsm[j][c] = k < K ? bvec[(long long)k * DXG_D + c] : 0.f;
        dsm[j][c] = k < K ? dvec[(long long)k * DXG_D + c] : 0.f;
      }
      if (et < DXG_GC) {
        csm[et] = g * DXG_GC + et < K ? cvec[g * DXG_GC + et] : 0.f;
        ssm[et] = g * DXG_GC + et < K ? svec[g * DXG_GC + et] : 0.f;
      }
      dxg_named_sync(1, 256);
      for (long long t = t0; t < t1; ++t, ++it) {
        const long long i = t * DXG_TM + row;
        // this row's scaled point sx*x from the A stage (fp16 hi + lo)
        float xr[DXG_D];
        {
          const int s = it % DXG_FXS;
          dx_mbar_wait_bounded(&xfull[s], (unsigned)((it / DXG_FXS) & 1));
          const unsigned char* xh = xsm + s * 2 * DXG_TM * 128;
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) {
            const unsigned off = dxg_sw((unsigned)row, (unsigned)(ch * 8));
            const uint4 hv = *reinterpret_cast<const uint4*>(xh + off);
            const uint4 lv = *reinterpret_cast<const uint4*>(xh + DXG_TM * 128 + off);
            const unsigned hw[4] = {hv.x, hv.y, hv.z, hv.w}, lw[4] = {lv.x, lv.y, lv.z, lv.w};
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              const float2 xv = dx_f2add(make_float2(dxg_h_lo(hw[w]), dxg_h_hi(hw[w])),
                                         make_float2(dxg_h_lo(lw[w]), dxg_h_hi(lw[w])));
              xr[ch * 8 + 2 * w] = xv.x;
              xr[ch * 8 + 2 * w + 1] = xv.y;
            }
          }
          __syncwarp();
          if (lane == 0) dx_mbar_arrive(&xempty[s]);
        }
        for (int h = 0; h < DXG_NH; ++h, ++tt) {
          const int bb = tt & 1;
          if (DXG_NH == 2 && h != hsel) continue;
          dx_mbar_wait_bounded(&tfull[bb], (unsigned)((tt >> 1) & 1));
          dxg_fence_after();
#pragma unroll 1
          for (int jj = 0; jj < DXG_GC / 2; ++jj) {
            const int j = hsel * (DXG_GC / 2) + jj;  // component within the group
            unsigned v0[16], v1[16], v2[16], v3[16];
            const unsigned ta = lanebase + (unsigned)(bb * 256 + (j % 4) * 64);
            DXG_TMEM_LD16(ta, v0);
            DXG_TMEM_LD16(ta + 16, v1);
            DXG_TMEM_LD16(ta + 32, v2);
            DXG_TMEM_LD16(ta + 48, v3);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            float2 s2 = make_float2(0.f, 0.f);  // even / odd columns
            // y~_c = MMA_c - bvec_c + dvec_c * x~_c  (= sx sq Q (x - mu))
            // (columns c, c+1 as one f32x2 pair: same per-lane rounding as the scalar form)
#define DXG_Y(V, c0)                                                                                        \
  {                                                                                                         \
    const float2 t = dx_f2sub(make_float2(__uint_as_float(V[c]), __uint_as_float(V[c + 1])),               \
                              *reinterpret_cast<const float2*>(&bsm[j][c0 + c]));                           \
    const float2 y = dx_f2fma(*reinterpret_cast<const float2*>(&dsm[j][c0 + c]),                            \
                              make_float2(xr[c0 + c], xr[c0 + c + 1]), t);                                  \
    s2 = dx_f2fma(y, y, s2);                                                                                \
  }
#pragma unroll
            for (int c = 0; c < 16; c += 2) {
              DXG_Y(v0, 0)
              DXG_Y(v1, 16)
              DXG_Y(v2, 32)
              DXG_Y(v3, 48)
            }
#undef DXG_Y
            const int k = g * DXG_GC + j;
            if (k < K && i < n) beta[(long long)k * npad + i] = csm[j] - 0.5f * ssm[j] * (s2.x + s2.y);
          }
          dxg_fence_before();
          __syncwarp();
          if (lane == 0) dx_mbar_arrive(&tempty[bb]);
        }
      }
    }
  }
  dxg_fence_before();
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

// ---- log-sum-exp over components per point; block partials of sum_i lse_i -------
extern "C" __global__ void __launch_bounds__(256) dx_gmm_lse(const float* __restrict__ beta, int K, long long n,
                                                             long long npad, float* __restrict__ lse,
                                                             double* __restrict__ part) {
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    // one pass, online max: s = sum exp(beta - m) rescaled when m grows
    float m = -3.0e38f, s = 0.f;
    for (int k0 = 0; k0 < K; k0 += 8) {
      float v[8];  // the 8 loads of a step are independent (issued together)
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = k0 + q < K ? beta[(long long)(k0 + q) * npad + i] : -3.0e38f;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (v[q] > m) {
          s = s * __expf(m - v[q]) + 1.f;
          m = v[q];
        } else {
          s += __expf(v[q] - m);
        }
      }
    }
    const float l = m + __logf(s);
    lse[i] = l;
    acc += (double)l;
  }
  __shared__ double scr[32];
  const double tot = dx_block_sum(acc, scr);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

// ---- backward moments -------------------------------------------------------------
// Work unit = (component pair pr, contiguous chunk range p); CTA c takes
// units c, c + grid, ... (chunk-range-major order) and flushes a partial slot
// per unit.  Warp 0: X^T chunk producer (bulk copies, 2-stage ring); warp 1: MMA
// issuer; warps 2-9: A-operand producers (g * (X - mu)^T, fp16x3 split, W sums);
// warps 10-13: TMEM promotion epilogue.  D (128 lanes x 80 columns, hi*hi and
// the small cross products in separate accumulators) is double buffered in
// TMEM and promoted every DXG_PROMO chunks into fp32 registers, which spill
// every DXG_F64_EVERY promotions into fp64 accumulators in shared memory
// (column-major, conflict-free).
#define DXG_XT_BYTES (2 * DXG_D * 128)          // hi + lo image of one chunk
#define DXG_XB_BYTES (DXG_BN * 128)             // one split of the B operand
#define DXG_Z_BYTES (2 * 128 * 128)             // hi + lo A operand of one chunk
#define DXG_BWD_SMEM (DXG_NXS * 2 * DXG_XB_BYTES + DXG_BN * 128 * 8 + 1024)
// ---- backward, two pairs (four components) per unit (default) ----------------------
// Same math as dx_gmm_bwd_pair, but each X^T chunk staged by the bulk-copy ring
// feeds the MMAs of two component pairs (the single-pair kernel is bound by
// re-streaming X^T once per pair).  TMEM: D[q][b] (pair q, buffer b, one merged
// accumulator) at (2q + b) * 64, A[q][s] (pair q, stage s: hi 32 + lo 32
// columns) at 256 + (2q + s) * 64.  Warps: 0 bulk copies, 1 MMA, 2-9
// producers (warps 2-5 pair 0, 6-9 pair 1; each thread one row (k, b) over all
// 64 points of the chunk), 10-17 epilogue (warps 10-13 pair 0, 14-17 pair 1:
// fp32 register accumulators promoted after every chunk, spilled to fp64
// shared memory every DXG_F64_EVERY chunks, one fp64 partial slot per unit).
// Promoting every chunk (64 points, 12 MMAs per TMEM accumulation) keeps the
// error of the tensor core's fp32 accumulation at the single-pair kernel's.
#define DXG_QWP (4 * (1 + DXG_D))
#define DXG_BWD4_SMEM (DXG_NXS * 2 * DXG_XB_BYTES + 2 * DXG_BN * 128 * 8 + 1024)
extern "C" __global__ void __launch_bounds__(576, 1)
    dx_gmm_bwd(const unsigned char* __restrict__ xtimg, const float* __restrict__ beta,
                const float* __restrict__ lse, const float* __restrict__ means, const unsigned* __restrict__ xmax,
                int K, long long n, long long npad, int P2, double* __restrict__ dpart, double* __restrict__ wpart,
                int* __restrict__ ppart) {
  extern __shared__ __align__(1024) unsigned char dxg_smem_raw[];
  unsigned char* smem = dxg_smem_raw + ((1024u - (dx_smem_addr(dxg_smem_raw) & 1023u)) & 1023u);
  unsigned char* bs = smem;                                                      // NXS x (hi 8 KB, lo 8 KB)
  double* dacc = reinterpret_cast<double*>(smem + DXG_NXS * 2 * DXG_XB_BYTES);  // [2][64][128]
  __shared__ __align__(16) float gin[DXG_NXS][5][DXG_BC];
  __shared__ __align__(16) float gw[8][64];
  __shared__ __align__(8) unsigned long long xfull[DXG_NXS], xempty[DXG_NXS], zfull[2][2], zempty[2][2],
      tfull[2][2], tempty[2][2];
  __shared__ unsigned tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NQ = (K + 3) / 4;
  const long long C = npad / DXG_BC;
  const long long units = (long long)NQ * P2;

  if (threadIdx.x == 0) {
    for (int q = 0; q < 2; ++q)
      for (int b = 0; b < 2; ++b) {
        dx_mbar_init(&zfull[q][b], 4);
        dx_mbar_init(&zempty[q][b], 1);
        dx_mbar_init(&tfull[q][b], 1);
        dx_mbar_init(&tempty[q][b], 4);
      }
    for (int s = 0; s < DXG_NXS; ++s) {
      dx_mbar_init(&xfull[s], 1);
      dx_mbar_init(&xempty[s], 1);
    }
    dx_fence_mbar_init();
  }
  for (int e = threadIdx.x; e < 2 * DXG_BN * 128; e += blockDim.x) dacc[e] = 0.0;
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dx_smem_addr(&tmem_base)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  dxg_fence_before();
  __syncthreads();
  dxg_fence_after();
  const unsigned tmem = tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (long long u = blockIdx.x; u < units; u += gridDim.x) {
        const long long qd = u % NQ, p = u / NQ;
        const long long c0 = p * C / P2, c1 = (p + 1) * C / P2;
        long long kr[4];
        for (int j = 0; j < 4; ++j) kr[j] = (4 * qd + j < K) ? 4 * qd + j : 0;
        for (long long c = c0; c < c1; ++c, ++it) {
          const int xs = it % DXG_NXS;
          if (it >= DXG_NXS) dx_mbar_wait_bounded(&xempty[xs], (unsigned)(((it / DXG_NXS) - 1) & 1));
          dx_mbar_expect_tx(&xfull[xs], DXG_XT_BYTES + 5 * DXG_BC * 4);
          const unsigned char* src = xtimg + c * DXG_XT_BYTES;
          dx_bulk_g2s(bs + (xs * 2) * DXG_XB_BYTES, src, DXG_D * 128, &xfull[xs]);
          dx_bulk_g2s(bs + (xs * 2 + 1) * DXG_XB_BYTES, src + DXG_D * 128, DXG_D * 128, &xfull[xs]);
          for (int j = 0; j < 4; ++j) dx_bulk_g2s(gin[xs][j], beta + kr[j] * npad + c * DXG_BC, DXG_BC * 4, &xfull[xs]);
          dx_bulk_g2s(gin[xs][4], lse + c * DXG_BC, DXG_BC * 4, &xfull[xs]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // B = [X^T hi ; X^T lo]: the two images of a chunk are contiguous SW128
      // row groups, i.e. one N=128 operand.  D[q] (128 columns: products with
      // x hi | x lo) = A_hi B + A_lo B over one chunk, drained every chunk.
      const unsigned idesc = dxg_idesc_f16<2 * DXG_BN>();
      const unsigned baddr = dx_smem_addr(bs);
      int it = 0;
      for (long long u = blockIdx.x; u < units; u += gridDim.x) {
        const long long p = u / NQ;
        const long long c0 = p * C / P2, c1 = (p + 1) * C / P2;
        for (long long c = c0; c < c1; ++c, ++it) {
          const int xs = it % DXG_NXS, s = it & 1;
          dx_mbar_wait_bounded(&xfull[xs], (unsigned)((it / DXG_NXS) & 1));
          const unsigned bh = baddr + (unsigned)(xs * 2 * DXG_XB_BYTES);
          for (int q = 0; q < 2; ++q) {
            if (it > 0) dx_mbar_wait_bounded(&tempty[q][0], (unsigned)((it - 1) & 1));
            dx_mbar_wait_bounded(&zfull[q][s], (unsigned)((it >> 1) & 1));
            dxg_fence_after();
            const unsigned td = tmem + (unsigned)(q * 128);
            const unsigned tah = tmem + (unsigned)(256 + (2 * q + s) * 64), tal = tah + 32;
#pragma unroll
            for (int kk = 0; kk < DXG_BC / 16; ++kk) {
              const unsigned long long db = dx_umma_desc_sw128(bh + kk * 32);
              dxg_umma_f16_ta(td, tah + kk * 8, db, idesc, kk > 0 ? 1u : 0u);
              dxg_umma_f16_ta(td, tal + kk * 8, db, idesc, 1u);
            }
            dx_umma_commit(&zempty[q][s]);
            dx_umma_commit(&tfull[q][0]);
          }
          dx_umma_commit(&xempty[xs]);
        }
      }
    }
  } else if (warp < 10) {
    const int pw = warp - 2, q = pw >> 2;           // pair of this producer warp
    const int r = (warp & 3) * 32 + lane;            // TMEM lane = row (k_local, b) of A[q]
    const int kl = r >> 6, b = r & 63;
    const bool wrow = (r & 32) == 0;                 // the warp with rows b < 32 sums W of comp kl
    const float sx = dxg_scale_for(__uint_as_float(*xmax));
    int it = 0, slot = 0;
    for (long long u = blockIdx.x; u < units; u += gridDim.x, ++slot) {
      const long long qd = u % NQ, p = u / NQ;
      const long long c0 = p * C / P2, c1 = (p + 1) * C / P2;
      const int kq = 2 * q + kl;                     // component within the quad
      const int k = (int)(4 * qd) + kq;
      const bool live = k < K;
      const float mub = live ? means[(long long)k * DXG_D + b] * sx : 0.f;
      float wacc = 0.f;
      double msum = 0.0;
      for (long long c = c0; c < c1; ++c, ++it) {
        const int xs = it % DXG_NXS, s = it & 1;
        if (it >= 2) dx_mbar_wait_bounded(&zempty[q][s], (unsigned)(((it >> 1) - 1) & 1));
        dx_mbar_wait_bounded(&xfull[xs], (unsigned)((it / DXG_NXS) & 1));
        {
          const long long i0 = c * DXG_BC + lane, i1 = i0 + 32;
          const float g0 = __expf(gin[xs][kq][lane] - gin[xs][4][lane]);
          const float g1 = __expf(gin[xs][kq][lane + 32] - gin[xs][4][lane + 32]);
          const float q0 = (live && i0 < n) ? g0 : 0.f, q1 = (live && i1 < n) ? g1 : 0.f;
          if (wrow) wacc += q0 + q1;
          gw[pw][lane] = q0;
          gw[pw][lane + 32] = q1;
          __syncwarp();
        }
        const unsigned char* xh = bs + (xs * 2) * DXG_XB_BYTES;
        const unsigned char* xl = xh + DXG_XB_BYTES;
        unsigned th[32], tl[32];
        float2 mchunk = make_float2(0.f, 0.f);  // even / odd points
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {  // 8 x 8 points
          const unsigned off_x = dxg_sw((unsigned)b, (unsigned)(cc * 8));
          const uint4 h4 = *reinterpret_cast<const uint4*>(xh + off_x);
          const uint4 l4 = *reinterpret_cast<const uint4*>(xl + off_x);
          const float4 ga = *reinterpret_cast<const float4*>(&gw[pw][cc * 8]);
          const float4 gb = *reinterpret_cast<const float4*>(&gw[pw][cc * 8 + 4]);
          const float gv[8] = {ga.x, ga.y, ga.z, ga.w, gb.x, gb.y, gb.z, gb.w};
          const unsigned hw[4] = {h4.x, h4.y, h4.z, h4.w}, lw[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
          for (int w = 0; w < 4; ++w) {  // points (2w, 2w+1) as one f32x2 pair
            const float2 xs = dx_f2add(make_float2(dxg_h_lo(hw[w]), dxg_h_hi(hw[w])),
                                       make_float2(dxg_h_lo(lw[w]), dxg_h_hi(lw[w])));
            const float2 z = dx_f2mul(make_float2(gv[2 * w], gv[2 * w + 1]), dx_f2sub(xs, make_float2(mub, mub)));
            mchunk = dx_f2add(mchunk, z);
            dxg_split2v(z, th[cc * 4 + w], tl[cc * 4 + w]);
          }
        }
        msum += (double)(mchunk.x + mchunk.y);
        {
          const unsigned ta = tmem + ((unsigned)((warp & 3) * 32) << 16) + (unsigned)(256 + (2 * q + s) * 64);
          DXG_TMEM_ST16(ta, th);
          DXG_TMEM_ST16(ta + 16, (th + 16));
          DXG_TMEM_ST16(ta + 32, tl);
          DXG_TMEM_ST16(ta + 48, (tl + 16));
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          dxg_fence_before();
        }
        __syncwarp();
        if (lane == 0) dx_mbar_arrive(&zfull[q][s]);
      }
      // unit done: W (warp sum) and m~ (per row) of this thread's component
      double* wp = wpart + ((long long)blockIdx.x * DXG_FMAX + slot) * DXG_QWP + kq * (1 + DXG_D);
      const float wsum = dx_warp_sum(wacc);
      if (wrow && lane == 0) wp[0] = (double)wsum;
      wp[1 + b] = msum;
    }
  } else {
    // epilogue: warps 10..17 -> pair q = (warp - 10) / 4, TMEM lane quarter warp & 3
    const int q = (warp - 10) >> 2, qr = warp & 3;
    const int row = qr * 32 + lane;
    const unsigned lanebase = tmem + ((unsigned)(qr * 32) << 16);
    double* dq = dacc + q * DXG_BN * 128 + row;
    float acc[DXG_BN];
#pragma unroll
    for (int j = 0; j < DXG_BN; ++j) acc[j] = 0.f;
    int pc = 0, slot = 0, nacc = 0;
    auto spill = [&]() {
#pragma unroll
      for (int j = 0; j < DXG_BN; ++j) {
        dq[j * 128] += (double)acc[j];
        acc[j] = 0.f;
        if ((j & 7) == 7) asm volatile("" ::: "memory");  // <= 8 fp64 loads in flight (registers)
      }
      nacc = 0;
    };
    for (long long u = blockIdx.x; u < units; u += gridDim.x, ++slot) {
      const int qd = (int)(u % NQ);
      const long long p = u / NQ;
      const int nch = (int)((p + 1) * C / P2 - p * C / P2);  // chunks of this unit (32-bit: registers)
      for (int c = 0; c < nch; ++c) {
        {
          dx_mbar_wait_bounded(&tfull[q][0], (unsigned)(pc & 1));
          dxg_fence_after();
#pragma unroll
          for (int j0 = 0; j0 < DXG_BN; j0 += 8) {  // x8 loads: acc[64] + 16 in flight (96 registers at 576 threads)
            unsigned v[8], w[8];
            DXG_TMEM_LD8(lanebase + (unsigned)(q * 128 + j0), v);
            DXG_TMEM_LD8(lanebase + (unsigned)(q * 128 + DXG_BN + j0), w);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 8; j += 2) {  // f32x2: acc += (hi-column + lo-column) products
              const float2 t = dx_f2add(make_float2(__uint_as_float(v[j]), __uint_as_float(v[j + 1])),
                                        make_float2(__uint_as_float(w[j]), __uint_as_float(w[j + 1])));
              const float2 a2 = dx_f2add(make_float2(acc[j0 + j], acc[j0 + j + 1]), t);
              acc[j0 + j] = a2.x;
              acc[j0 + j + 1] = a2.y;
            }
          }
          dxg_fence_before();
          __syncwarp();
          if (lane == 0) dx_mbar_arrive(&tempty[q][0]);
          ++pc;
          if (++nacc == DXG_F64_EVERY) spill();
        }
      }
      // flush this unit: rows (q, row) of the quad's D to an fp64 slot
      spill();
      double* dst = dpart + (((long long)blockIdx.x * DXG_FMAX + slot) * 256 + q * 128 + row) * DXG_BN;
#pragma unroll 4
      for (int j = 0; j < DXG_BN; ++j) {
        dst[j] = dq[j * 128];
        dq[j * 128] = 0.0;
      }
      if (threadIdx.x == 320) ppart[blockIdx.x * DXG_FMAX + slot] = qd;
    }
  }
  dxg_fence_before();
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

// ---- moments: fold the backward partial slots of each component's pair in CTA
// order into fp64 mom[k] = (P [64][64], m~ [64], W) with the centred moments
// P[b][a] = sum_i g (x - mu)_b x_a and m~ = sum_i g (x - mu) ----------------------
#define DXG_MOM (DXG_D * DXG_D + DXG_D + 1)
extern "C" __global__ void __launch_bounds__(256) dx_gmm_moments(const double* dpart, const double* wpart,
                                                                 const int* ppart, int nslot, const unsigned* xmax,
                                                                 int G, double* mom) {
  // G components per partial slot (4: dx_gmm_bwd, 2: dx_gmm_bwd_pair)
  // the operands were scaled by the points' scale sx: D = sx^2 P, m~ sums sx m~
  const double isx = 1.0 / (double)dxg_scale_for(__uint_as_float(*xmax));
  __shared__ int slots[2048];  // host guarantees nslot <= 2048
  __shared__ int nsl;
  const int k = blockIdx.x, pr = k / G, kl = k % G;
  if (threadIdx.x == 0) {
    int ns = 0;
    for (int e = 0; e < nslot && ns < 2048; ++e)
      if (ppart[e] == pr) slots[ns++] = e;
    nsl = ns;
  }
  __syncthreads();
  double* out = mom + (long long)k * DXG_MOM;
  // four entries per thread: four independent slot chains in flight (each
  // entry still sums its slots in slot order)
  for (int e0 = threadIdx.x; e0 < DXG_D * DXG_D; e0 += 4 * blockDim.x) {
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    for (int sl = 0; sl < nsl; ++sl) {
      const double* src = dpart + ((long long)slots[sl] * (G * 64) + kl * 64) * DXG_BN;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * blockDim.x;
        if (e < DXG_D * DXG_D) s[u] += src[(e / DXG_D) * DXG_BN + e % DXG_D];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e < DXG_D * DXG_D) out[e] = s[u] * isx * isx;
    }
  }
  if (threadIdx.x <= DXG_D) {
    double s = 0.0;  // threadIdx 0: W; 1 + b: m~_b
    for (int sl = 0; sl < nsl; ++sl) s += wpart[(long long)slots[sl] * (G * (1 + DXG_D)) + kl * (1 + DXG_D) + threadIdx.x];
    if (threadIdx.x == 0) out[DXG_D * DXG_D + DXG_D] = s;
    else out[DXG_D * DXG_D + threadIdx.x - 1] = s * isx;
  }
}

// fixed-order sum of the lse block partials
extern "C" __global__ void dx_gmm_sum(const double* part, int n, double* out) {
  __shared__ double scr[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  const double t = dx_block_sum(s, scr);
  if (threadIdx.x == 0) *out = t;
}

// ---- finish: per component, fp64 --------------------------------------------------
// From the fp64 moments of dx_gmm_moments (summed over ranks when sharded):
//   M   = P - m~ mu^T                              (= sum_i g (x-mu)(x-mu)^T)
//   dQ  = -Q M (lower triangle), v = Q m~, d mu = Q^T v
//   d alpha = W - n softmax(alpha), d icf = (diag: dQ_jj e^q_j + W + gamma^2 e^{2 q_j} - m;
//   L: dQ + gamma^2 L), and the prior term of the objective.
extern "C" __global__ void __launch_bounds__(256) dx_gmm_finish(
    const float* alphas, const float* means, const float* icf, int K, long long n, const double* mom,
    double gamma, int wm, double* d_alphas, double* d_means, double* d_icf, double* prior_k) {
  extern __shared__ double dxg_fin_smem[];  // Q, M: 2 x 64 x 65 doubles (dynamic)
  double(*Q)[DXG_D + 1] = reinterpret_cast<double(*)[DXG_D + 1]>(dxg_fin_smem);
  double(*M)[DXG_D + 1] = reinterpret_cast<double(*)[DXG_D + 1]>(dxg_fin_smem + DXG_D * (DXG_D + 1));
  __shared__ double mu[DXG_D], mm[DXG_D], v[DXG_D];
  __shared__ double Wk, lse_a;
  const int k = blockIdx.x;
  const float* q = icf + (long long)k * DXG_ICF;
  const double* mk = mom + (long long)k * DXG_MOM;
  for (int e = threadIdx.x; e < DXG_D * DXG_D; e += blockDim.x) {
    const int r = e / DXG_D, c = e % DXG_D;
    double val = 0.0;
    if (r == c) val = exp((double)q[r]);
    else if (r > c) val = (double)q[DXG_D + c * (DXG_D - 1) - c * (c - 1) / 2 + (r - c - 1)];
    Q[r][c] = val;
    M[r][c] = mk[r * DXG_D + c];
  }
  if (threadIdx.x < DXG_D) {
    const int b = threadIdx.x;
    mu[b] = (double)means[(long long)k * DXG_D + b];
    mm[b] = mk[DXG_D * DXG_D + b];
  }
  if (threadIdx.x == 0) {
    Wk = mk[DXG_D * DXG_D + DXG_D];
    double m0 = -1e300;
    for (int j = 0; j < K; ++j) m0 = fmax(m0, (double)alphas[j]);
    double se = 0.0;
    for (int j = 0; j < K; ++j) se += exp((double)alphas[j] - m0);
    lse_a = m0 + log(se);
  }
  __syncthreads();
  // M <- P - m~ mu^T
  for (int e = threadIdx.x; e < DXG_D * DXG_D; e += blockDim.x) {
    const int r = e / DXG_D, c = e % DXG_D;
    M[r][c] = M[r][c] - mm[r] * mu[c];
  }
  if (threadIdx.x < DXG_D) {
    const int r = threadIdx.x;
    double s = 0.0;
    for (int c = 0; c <= r; ++c) s += Q[r][c] * mm[c];
    v[r] = s;
  }
  __syncthreads();
  if (threadIdx.x < DXG_D) {
    const int a = threadIdx.x;
    double s = 0.0;
    for (int r = a; r < DXG_D; ++r) s += Q[r][a] * v[r];
    d_means[(long long)k * DXG_D + a] = s;
  }
  const double g2 = gamma * gamma;
  double* di = d_icf + (long long)k * DXG_ICF;
  for (int e = threadIdx.x; e < DXG_D * DXG_D; e += blockDim.x) {
    const int r = e / DXG_D, c = e % DXG_D;
    if (c > r) continue;
    double s = 0.0;
    for (int j = 0; j <= r; ++j) s += Q[r][j] * M[j][c];  // Q lower triangular
    const double dq = -s;
    if (r == c) di[r] = dq * Q[r][r] + Wk + g2 * Q[r][r] * Q[r][r] - (double)wm;
    else di[DXG_D + c * (DXG_D - 1) - c * (c - 1) / 2 + (r - c - 1)] = dq + g2 * Q[r][c];
  }
  if (threadIdx.x == 0) {
    d_alphas[k] = Wk - (double)n * exp((double)alphas[k] - lse_a);
    double frob = 0.0, sq = 0.0;
    for (int c = 0; c < DXG_D; ++c) {
      frob += Q[c][c] * Q[c][c];
      sq += (double)q[c];
    }
    for (int e = DXG_D; e < DXG_ICF; ++e) frob += (double)q[e] * (double)q[e];
    prior_k[k] = 0.5 * g2 * frob - (double)wm * sq;
  }
}
