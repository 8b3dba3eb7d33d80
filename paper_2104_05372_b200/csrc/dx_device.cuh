// dx_device.cuh — hand-written sm_100a device runtime for lowered dexlet nests.
//
// Prepended (as text) to every NVRTC module the lowering emits; the
// per-nest kernels call these primitives for everything except the body
// arithmetic.  Replaces, on the device, the reference's chunk overlays and
// their merge (proj/src/eval.cpp:233-256, 357-366):
//   * scalar Accum cells   -> per-thread register partials, warp xor-shuffle,
//                             block tree, one partial per block, then a
//                             fixed-order finalize (deterministic);
//   * small Accum tables   -> shared-memory privatized copies per block,
//                             flushed as per-block partials, same finalize;
//   * integer-valued `+= c` (histograms) -> u32 shared counters, exact;
//   * row scatters r!k!j over a contiguous inner axis -> warp-cooperative
//     conflict-free shared-memory row adds (no atomics);
//   * everything else      -> global red.add.
// No includes: NVRTC compiles this without the CUDA headers.

#define DX_FULL 0xffffffffu

template <class T>
__device__ __forceinline__ T dx_warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(DX_FULL, v, o);
  return v;
}

// Fixed-shape block tree: xor-shuffle inside each warp, then warp 0 folds
// the per-warp sums.  Result valid in thread 0.  `scratch` holds 32 slots.
template <class T>
__device__ __forceinline__ T dx_block_sum(T v, T* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = dx_warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  T r = (threadIdx.x < nw) ? scratch[threadIdx.x] : T(0);
  if (warp == 0) r = dx_warp_sum(r);
  return r;
}

__device__ __forceinline__ float dx_ld(const float* p) { return *p; }
__device__ __forceinline__ double dx_ld(const double* p) { return *p; }
__device__ __forceinline__ int dx_ld(const int* p) { return *p; }
__device__ __forceinline__ long long dx_ld(const long long* p) { return *p; }

// Fused E-bounds check for index leaves read from program inputs: the only
// runtime check of the reference (fromOrdinal, index_set.cpp:99-106).
// Pure (no memory side effect, so repeated loads still CSE): the per-thread
// flag is folded into dx_err once at kernel exit.
__device__ __forceinline__ int dx_chk_idx(int v, int n, int& bad) {
  const bool b = (unsigned)v >= (unsigned)n;
  bad |= (int)b;
  return b ? 0 : v;
}

__device__ __forceinline__ void dx_red_global(float* p, float v) { atomicAdd(p, v); }
__device__ __forceinline__ void dx_red_global(double* p, double v) { atomicAdd(p, v); }

// Shared-memory atomics.  f32/f64 adds are CAS loops on sm_100a; the lowering
// only uses them when no conflict-free strategy applies.
__device__ __forceinline__ void dx_red_smem(float* p, float v) { atomicAdd(p, v); }
__device__ __forceinline__ void dx_red_smem(double* p, double v) { atomicAdd(p, v); }
// Histogram counters: native shared-memory u32 atomics (ATOMS.ADD).
__device__ __forceinline__ void dx_count_smem(unsigned* bins, int k, unsigned active) {
  (void)active;
  atomicAdd(&bins[k], 1u);
}

// Warp-cooperative row scatter: every lane holds one row `v[0..D)` destined
// for row `key` (key < 0: nothing) of a warp-private table `tab[K][D]` in
// shared memory.  Rows are staged through `stage[32][D+1]` (+32 key slots) and
// then added by lanes-over-columns, 32/D rows per step.  Each shared word has
// exactly one writer per step: plain LDS/FADD/STS, no atomics.
//
// D == 16: two rows per step; the two keys are read by every lane, so the
// "same row" test is warp-uniform and the rare collision takes a shuffle.
// D == 32: one row per step, no collisions.  Other D: generic path.
template <class T, int D>
__device__ __forceinline__ void dx_row_flush(T* tab, T* stage, int key, const T (&v)[D]) {
  const int lane = threadIdx.x & 31;
  int* keys = reinterpret_cast<int*>(stage + 32 * (D + 1));
#pragma unroll
  for (int j = 0; j < D; ++j) stage[lane * (D + 1) + j] = v[j];
  keys[lane] = key;
  __syncwarp();
  if constexpr (D == 16) {
    const int g = lane >> 4, c = lane & 15;
#pragma unroll
    for (int r0 = 0; r0 < 32; r0 += 2) {
      const int k0 = keys[r0], k1 = keys[r0 + 1];
      const int kr = g ? k1 : k0;
      const T val = stage[(r0 + g) * (D + 1) + c];
      if (k0 == k1) {  // warp-uniform
        const T other = __shfl_xor_sync(DX_FULL, val, 16);
        if (g == 0 && kr >= 0) tab[kr * D + c] += val + other;
      } else if (kr >= 0) {
        tab[kr * D + c] += val;
      }
      __syncwarp();
    }
  } else if constexpr (D == 32) {
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const int kr = keys[r];
      const T val = stage[r * (D + 1) + lane];
      if (kr >= 0) tab[kr * D + lane] += val;
      __syncwarp();
    }
  } else if constexpr (D < 32) {
    constexpr int G = 32 / D;  // rows per step
    const int g = lane / D, c = lane % D;
#pragma unroll 1
    for (int r0 = 0; r0 < 32; r0 += G) {
      const int r = r0 + g;
      const int kr = (g < G && r < 32) ? keys[r] : -1;
      const T val0 = (g < G && r < 32) ? stage[r * (D + 1) + c] : T(0);
      T val = val0;
      // combine rows of this step that share a key, lowest group writes
      bool write = (g < G) && kr >= 0;
#pragma unroll
      for (int h = 1; h < G; ++h) {
        const int kh = __shfl_sync(DX_FULL, kr, (lane + h * D) & 31);
        const T vh = __shfl_sync(DX_FULL, val0, (lane + h * D) & 31);
        if (g + h < G && kh == kr) val += vh;
        const int kl = __shfl_sync(DX_FULL, kr, (lane - h * D + 32) & 31);
        if (g - h >= 0 && kl == kr) write = false;
      }
      if (write) tab[kr * D + c] += val;
      __syncwarp();
    }
  } else {
#pragma unroll 1
    for (int r = 0; r < 32; ++r) {
      const int kr = keys[r];
      if (kr >= 0)
        for (int c = lane; c < D; c += 32) tab[kr * D + c] += stage[r * (D + 1) + c];
      __syncwarp();
    }
  }
  __syncwarp();
}

// ---- finalize: fold per-block partials into the Accum cell, fixed order ----
// Block = 32 columns x 32 row-groups.  Thread (c, g) sums partial rows
// g, g+32, g+64, ... of column c in that order; the 32 row-group sums are then
// folded by a fixed-shape tree.  Deterministic for a given grid, and every
// partial row is in flight at once (no long dependent chains).
template <class T, class P>
__device__ __forceinline__ void dx_fin2(const P* part, int nblk, long long width, T scale, T* cell,
                                        bool counts) {
  __shared__ T red[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const long long c = (long long)blockIdx.x * 32 + tx;
  T s = T(0);
  if (c < width) {
    if (counts) {
      unsigned long long u = 0;
      for (int b = ty; b < nblk; b += 32) u += (unsigned long long)part[(long long)b * width + c];
      s = (T)u;
    } else {
      for (int b = ty; b < nblk; b += 32) s += (T)part[(long long)b * width + c];
    }
  }
  red[ty][tx] = s;
  __syncthreads();
#pragma unroll
  for (int h = 16; h > 0; h >>= 1) {
    if (ty < h) red[ty][tx] += red[ty + h][tx];
    __syncthreads();
  }
  if (ty == 0 && c < width) cell[c] += counts ? red[0][tx] * scale : red[0][tx];
}

extern "C" __global__ void __launch_bounds__(1024) dx_fin_f32(const float* p, int n, long long w, float* c) { dx_fin2<float, float>(p, n, w, 1.0f, c, false); }
extern "C" __global__ void __launch_bounds__(1024) dx_fin_f64(const double* p, int n, long long w, double* c) { dx_fin2<double, double>(p, n, w, 1.0, c, false); }
extern "C" __global__ void __launch_bounds__(1024) dx_fin_count_f32(const unsigned* p, int n, long long w, float s, float* c) { dx_fin2<float, unsigned>(p, n, w, s, c, true); }
extern "C" __global__ void __launch_bounds__(1024) dx_fin_count_f64(const unsigned* p, int n, long long w, double s, double* c) { dx_fin2<double, unsigned>(p, n, w, s, c, true); }

// Elementwise cell += src (host-level `r += table`), and fills.
extern "C" __global__ void dx_add_f32(float* c, const float* s, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) c[i] += s[i];
}
extern "C" __global__ void dx_add_f64(double* c, const double* s, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) c[i] += s[i];
}
// Bounds check of uploaded index leaves (fromOrdinal's check, index_set.cpp:99-106).
extern "C" __global__ void dx_check_index(const int* x, long long n, int size, int* bad) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int v = x[i];
    if (v < 0 || v >= size) atomicOr(bad, 1);
  }
}
