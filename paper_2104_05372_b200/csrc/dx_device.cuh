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

// ---- TMA bulk copies + mbarriers (streaming tiles into shared memory) ----
__device__ __forceinline__ unsigned dx_smem_addr(const void* p) {
  unsigned a;
  asm("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(a) : "l"(p));
  return a;
}
__device__ __forceinline__ void dx_mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(dx_smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void dx_fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void dx_fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void dx_mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(dx_smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void dx_mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(dx_smem_addr(bar)) : "memory");
}
// global -> shared bulk copy (TMA, 1-D), completion counted on `bar`.
// dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void dx_bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dx_smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(dx_smem_addr(bar))
      : "memory");
}
// 2-D TMA tensor tile load (CUtensorMap passed as a __grid_constant__
// kernel parameter); coordinates {c0 = column, c1 = row}.
struct __align__(64) dx_tmap {
  unsigned long long v[16];
};
__device__ __forceinline__ void dx_tma_2d(void* dst, const dx_tmap* map, int c0, int c1, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dx_smem_addr(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(dx_smem_addr(bar))
      : "memory");
}
// Byte address swizzle of TMA SWIZZLE_{32,64,128}B: 16-byte chunk bits XOR
// the 128-byte line bits (mask 1, 3, 7).
__device__ __forceinline__ unsigned dx_swz(unsigned a, unsigned mask) { return a ^ (((a >> 7) & mask) << 4); }

__device__ __forceinline__ void dx_mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n DX_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra DX_WAIT_%=;\n}" ::"r"(
          dx_smem_addr(bar)),
      "r"(parity)
      : "memory");
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

// Tile-sorted row reduction (block level, every thread must call it).
// Thread t of an NT-thread block holds one row v[0..D) for table row `key`
// (-1: none), already stored at etile[t*(D+1) ..].  The rows are bucketed by
// key with a stable counting sort (warp ranks from __match_any_sync, per-warp
// counts, per-key prefix over warps, prefix over keys), then thread t adds the
// rows of bucket k = e / D, column j = e % D into acc[i] for its entries
// e = t + i*NT, in ascending thread order: a deterministic segmented sum with
// the accumulators in registers across tiles (no atomics, no RMW).
template <class T, int D, int K, int NT, int NACC>
__device__ __forceinline__ void dx_tile_rows(const T* etile, int key, int* wcnt, int* start, int* perm,
                                             T (&acc)[NACC]) {
  constexpr int NW = NT / 32;
  constexpr int SUBS = (NT / K) < 32 ? (NT / K) : 32;  // threads per key in the warp scan
  constexpr int WPS = (NW + SUBS - 1) / SUBS;          // warps summarized per thread
  static_assert(SUBS >= 1 && (SUBS & (SUBS - 1)) == 0, "SUBS must be a power of two");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned peers = __match_any_sync(DX_FULL, key);
  const int rank = __popc(peers & ((1u << lane) - 1u));
  for (int i = tid; i < NW * K; i += NT) wcnt[i] = 0;
  __syncthreads();
  if (rank == 0 && key >= 0) wcnt[warp * K + key] = __popc(peers);
  __syncthreads();
  // per key: exclusive prefix over warps (SUBS threads per key, shuffles)
  if (tid < K * SUBS) {
    const int k = tid / SUBS, sub = tid % SUBS;
    int c[WPS];
    int loc = 0;
#pragma unroll
    for (int q = 0; q < WPS; ++q) {
      const int w = sub * WPS + q;
      c[q] = w < NW ? wcnt[w * K + k] : 0;
      loc += c[q];
    }
    int inc = loc;
#pragma unroll
    for (int o = 1; o < SUBS; o <<= 1) {
      const int y = __shfl_up_sync(DX_FULL, inc, o, SUBS);
      if (sub >= o) inc += y;
    }
    int run = inc - loc;
#pragma unroll
    for (int q = 0; q < WPS; ++q) {
      const int w = sub * WPS + q;
      if (w < NW) wcnt[w * K + k] = run;
      run += c[q];
    }
    if (sub == SUBS - 1) start[k + 1] = inc;  // bucket size
  }
  __syncthreads();
  // exclusive scan over the K bucket sizes (one warp)
  if (warp == 0) {
    constexpr int PER = (K + 31) / 32;
    int v[PER];
    int loc = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int k = lane * PER + q;
      v[q] = k < K ? start[k + 1] : 0;
      loc += v[q];
    }
    int inc = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(DX_FULL, inc, o);
      if (lane >= o) inc += y;
    }
    int run = inc - loc;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int k = lane * PER + q;
      if (k < K) start[k] = run;
      run += v[q];
    }
    if (lane == 31) start[K] = inc;
  }
  __syncthreads();
  if (key >= 0) perm[start[key] + wcnt[warp * K + key] + rank] = tid;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NACC; ++i) {
    const int e = tid + i * NT;
    if (e < K * D) {
      const int k = e / D, j = e - (e / D) * D;
      const int q1 = start[k + 1];
      T sum = acc[i];
      for (int q = start[k]; q < q1; ++q) sum += etile[perm[q] * (D + 1) + j];
      acc[i] = sum;
    }
  }
  __syncthreads();
}

// f32 rows with D % 4 == 0: rows live in etile as D/4 float4 blocks, block b
// of row t stored at slot b ^ ((t >> 1) & (D/4 - 1)) (conflict-free 128-bit
// stores: each 8-lane phase hits 8 distinct 16-byte bank groups).
template <int D>
__device__ __forceinline__ void dx_tile_store4(float* etile, int t, const float (&v)[D]) {
  constexpr int NB = D / 4;
  float4* row = reinterpret_cast<float4*>(etile + t * D);
#pragma unroll
  for (int b = 0; b < NB; ++b)
    row[b ^ ((t >> 1) & (NB - 1))] = make_float4(v[4 * b], v[4 * b + 1], v[4 * b + 2], v[4 * b + 3]);
}

// Vectorized variant of dx_tile_rows: thread tid owns (key k, column block jb)
// pair p = tid % P (P = K*D/4) and split s = tid / P of the bucket (elements
// q = start + s, s + NS, ...), accumulating a float4 in registers.
// Four block barriers per tile: [rows + warp counts] | [one warp: prefix over
// warps per key + scan over keys] | [scatter of row offsets] | [reduce; the
// warp counts are re-zeroed for the next tile].  wcnt must be zero on entry
// (zero it once before the first tile).
template <int D, int K, int NT>
__device__ __forceinline__ void dx_tile_rows4(const float* etile, int key, int* wcnt, int* start, int* perm,
                                              float4& acc) {
  constexpr int NB = D / 4, P = K * NB;
  constexpr int NS = P >= NT ? 1 : NT / P;
  constexpr int NW = NT / 32;
  constexpr int PER = (K + 31) / 32;
  static_assert(P <= NT, "one (key, block) pair per thread at most");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned peers = __match_any_sync(DX_FULL, key);
  const int rank = __popc(peers & ((1u << lane) - 1u));
  if (rank == 0 && key >= 0) wcnt[warp * K + key] = __popc(peers);
  __syncthreads();
  if (warp == 0) {
    // lane owns keys lane*PER .. lane*PER+PER-1: exclusive prefix over the
    // warps in place, bucket sizes, then a warp scan over the keys
    int tot[PER];
    int loc = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int k = lane * PER + q;
      int run = 0;
      if (k < K) {
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const int c = wcnt[w * K + k];
          wcnt[w * K + k] = run;
          run += c;
        }
      }
      tot[q] = run;
      loc += run;
    }
    int inc = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(DX_FULL, inc, o);
      if (lane >= o) inc += y;
    }
    int run = inc - loc;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int k = lane * PER + q;
      if (k < K) start[k] = run;
      run += tot[q];
    }
    if (lane == 31) start[K] = inc;
  }
  __syncthreads();
  // perm holds the swizzled byte offset of each row's block 0, so block jb is
  // one XOR away: (t*D*4 + 16*s(t)) ^ 16*jb  (see dx_tile_store4)
  if (key >= 0) perm[start[key] + wcnt[warp * K + key] + rank] = tid * (D * 4) + (((tid >> 1) & (NB - 1)) << 4);
  __syncthreads();
  for (int i = tid; i < NW * K; i += NT) wcnt[i] = 0;  // ready for the next tile
  if (tid < P * NS) {
    const int p = tid % P, sp = tid / P;
    const int k = p / NB, jb16 = (p % NB) << 4;
    const int q1 = start[k + 1];
    const char* base = reinterpret_cast<const char*>(etile);
    float4 a = acc;
#pragma unroll 4
    for (int q = start[k] + sp; q < q1; q += NS) {
      const float4 w = *reinterpret_cast<const float4*>(base + (perm[q] ^ jb16));
      a.x += w.x; a.y += w.y; a.z += w.z; a.w += w.w;
    }
    acc = a;
  }
  __syncthreads();
}

// Warp-private row table (WarpTab).  The warp's 32 rows were stored by
// dx_tile_store4 at etile rows 32*warp .. 32*warp+31; they are added, lanes
// over columns, G = 32/D rows per step, into a table of K+1 rows x 32 words
// holding G interleaved copies (copy g in columns g*D .. g*D+D-1; row K takes
// rows without a key).  Every step touches 32 distinct banks and each word has
// one writer, so the adds are plain LDS/FADD/STS with no atomics, no
// collisions and no block barrier.  Order is fixed: ascending row within the
// warp, copies folded in order by dx_warp_tab_flush.
template <int D, int K>
__device__ __forceinline__ void dx_warp_tab(const float* etile, int key, float* tab) {
  static_assert(D >= 4 && D <= 32 && (32 % D) == 0, "WarpTab row width");
  constexpr int G = 32 / D, NB = D / 4;
  const int lane = threadIdx.x & 31, wbase = threadIdx.x & ~31;
  const int g = lane / D, c = lane % D;
  const int k = key < 0 ? K : key;
  __syncwarp();
  {
  // Software-pipelined read-modify-write: the load of step s+1 is issued
  // before the store of step s (ordered volatile shared accesses), and when
  // both steps hit the same word the value just computed is forwarded.  Any
  // older step's store precedes the load in program order.
  constexpr int S = 32 / G;
  const unsigned base = dx_smem_addr(tab + g * D + c);
  float v[S];
  unsigned a[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int r = s * G + g;
    const int t = wbase + r;
    v[s] = etile[t * D + ((((c >> 2) ^ ((t >> 1) & (NB - 1)))) << 2) + (c & 3)];
    a[s] = base + (unsigned)__shfl_sync(DX_FULL, k, r) * 128u;
  }
  float cur;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(cur) : "r"(a[0]) : "memory");
#pragma unroll
  for (int s = 0; s < S; ++s) {
    float nxt = 0.f;
    if (s + 1 < S) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(nxt) : "r"(a[(s + 1) % S]) : "memory");
    const float val = cur + v[s];
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(a[s]), "f"(val) : "memory");
    if (s + 1 < S) cur = a[(s + 1) % S] == a[s] ? val : nxt;
  }
  }
}
// Block partial of NW warp tables: entry (k, j) = sum over warps, then copies,
// in that fixed order.
template <int D, int K, int NW>
__device__ __forceinline__ void dx_warp_tab_flush(const float* tabs, float* part) {
  // warp w folds rows w, w + NW, ...: lane l sums word l of the row over the
  // NW tables (conflict-free), then the G copies of a column are combined by
  // an xor tree; fixed order, every warp busy
  constexpr int G = 32 / D;
  static_assert(G >= 1, "row width");
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = warp; k < K; k += NW) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += tabs[(w * (K + 1) + k) * 32 + lane];
#pragma unroll
    for (int o = D; o < 32; o <<= 1) s += __shfl_xor_sync(DX_FULL, s, o);
    if (lane < D) part[k * D + lane] = s;
  }
}

// Block partial of a dx_tile_rows4 table: splits folded in fixed order.
template <int D, int K, int NT>
__device__ __forceinline__ void dx_tile_rows4_flush(float* scratch, const float4& acc, float* part) {
  constexpr int NB = D / 4, P = K * NB;
  constexpr int NS = P >= NT ? 1 : NT / P;
  const int tid = threadIdx.x;
  __syncthreads();
  if (tid < P * NS) reinterpret_cast<float4*>(scratch)[tid] = acc;
  __syncthreads();
  for (int p = tid; p < P; p += NT) {
    float4 s = reinterpret_cast<const float4*>(scratch)[p];
    for (int sp = 1; sp < NS; ++sp) {
      const float4 w = reinterpret_cast<const float4*>(scratch)[sp * P + p];
      s.x += w.x; s.y += w.y; s.z += w.z; s.w += w.w;
    }
    reinterpret_cast<float4*>(part)[p] = s;  // entry (k, 4*jb..4*jb+3) at p*4
  }
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

// ---- in-kernel finalize: last-block-done fold (no grid barrier) -----------
// Every block writes its partial row, then arrives on its group's ticket
// (groups of DX_LBD_GB consecutive blocks); the last block of a group folds
// the group's rows in block order into a group partial (f64 / u64), and the
// last group to finish folds the group partials in group order into the cell.
// The result is deterministic for a fixed grid, no block waits for another,
// and the tickets are reset by the block that consumed them, so they never
// wrap (any number of launches).  tick layout: [ngroups] group tickets, then
// DX_LBD_TOP (final ticket) and DX_LBD_ERR (E-bounds flags of this launch).
#define DX_LBD_GB 16
#define DX_LBD_TOP 1024
#define DX_LBD_ERR 1025
#define DX_LBD_WORDS 1026
__device__ __forceinline__ float dx_ldcg(const float* p) {
  float v;
  asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double dx_ldcg(const double* p) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned dx_ldcg(const unsigned* p) {
  unsigned v;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ long long dx_ldcg(const long long* p) {
  long long v;
  asm volatile("ld.global.cg.s64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
// Block-wide: true in exactly one block, the last of `expected` to arrive
// on tick[slot]; that block then sees every arriving block's writes.
__device__ __forceinline__ bool dx_lbd_arrive(unsigned* tick, int slot, unsigned expected) {
  __shared__ int dx_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    dx_last = atomicAdd(&tick[slot], 1u) == expected - 1u;
  }
  __syncthreads();
  const bool last = dx_last != 0;
  if (last) __threadfence();
  return last;
}
// Group fold: gpart[grp][c] = sum over blocks first .. first+cnt-1 (block
// order) of part[b][c]; all loads of a column are issued before the sum.
template <class P, class G>
__device__ __forceinline__ void dx_lbd_group(const P* part, long long width, G* gpart, int grp, int first, int cnt) {
  for (long long c = threadIdx.x; c < width; c += blockDim.x) {
    P v[DX_LBD_GB];
#pragma unroll
    for (int b = 0; b < DX_LBD_GB; ++b) v[b] = b < cnt ? dx_ldcg(&part[(long long)(first + b) * width + c]) : P(0);
    G s = G(0);
#pragma unroll
    for (int b = 0; b < DX_LBD_GB; ++b)
      if (b < cnt) s += (G)v[b];
    gpart[(long long)grp * width + c] = s;
  }
}
// Final fold of the group partials (group order) into the cell: store (the
// cell's zero-fill was folded into this kernel) or add.
template <class G, class T>
__device__ __forceinline__ void dx_lbd_final(const G* gpart, long long width, int ngrp, T scale, T* cell, bool counts,
                                             bool store) {
  for (long long c = threadIdx.x; c < width; c += blockDim.x) {
    G s = G(0);
    for (int g0 = 0; g0 < ngrp; g0 += 32) {
      G v[32];
#pragma unroll
      for (int b = 0; b < 32; ++b) v[b] = g0 + b < ngrp ? dx_ldcg(&gpart[(long long)(g0 + b) * width + c]) : G(0);
#pragma unroll
      for (int b = 0; b < 32; ++b)
        if (g0 + b < ngrp) s += v[b];
    }
    const T val = counts ? (T)s * scale : (T)s;
    if (store) cell[c] = val;
    else cell[c] += val;
  }
}

// ---- in-kernel finalize, cooperative form (every block resident) ---------
// Wrap-safe grid barrier: bar[0] counts arrivals, bar[1] is a generation that
// the last arriver bumps after resetting the count; waiters compare
// generations for equality, so the words never overflow into a hang.
__device__ __forceinline__ void dx_grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned gen;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(gen) : "l"(bar + 1) : "memory");
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1u) {
      bar[0] = 0u;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (true) {
        unsigned g;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
        if (g != gen) break;
        __nanosleep(20);
      }
    }
    __threadfence();
  }
  __syncthreads();
}
// Programmatic dependent launch: a kernel launched with the PDL attribute
// may start while its predecessor on the stream drains; it waits here before
// touching anything that predecessor may write.  No-ops without PDL.
__device__ __forceinline__ void dx_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void dx_pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Bulk L2 prefetch (TMA engine, no registers or shared memory): group mode
// asks for the rows of the chunk after next while the next one is loading.
// Needs a 16-byte aligned start (checked) and a size multiple of 16.
__device__ __forceinline__ void dx_l2_prefetch(const void* p, unsigned bytes) {
  if (((unsigned long long)p & 15ull) == 0ull)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Streaming (evict-first) loads for rows read once.
__device__ __forceinline__ float dx_ldcs(const float* p) {
  float v;
  asm volatile("ld.global.cs.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double dx_ldcs(const double* p) {
  double v;
  asm volatile("ld.global.cs.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int dx_ldcs(const int* p) {
  int v;
  asm volatile("ld.global.cs.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ long long dx_ldcs(const long long* p) {
  long long v;
  asm volatile("ld.global.cs.s64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

// Group sum over the G lanes sharing an ordinal (group mode): fixed xor tree.
template <int G, class T>
__device__ __forceinline__ T dx_grp_sum(T v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(DX_FULL, v, o);
  return v;
}

// ... the same over the active group only (the ragged chunk, where a group
// past the end skips its ordinal: the guard is uniform within a group).
template <int G, class T>
__device__ __forceinline__ T dx_grp_sum_m(T v) {
  const unsigned lane = threadIdx.x & 31u;
  const unsigned m = (G == 32) ? DX_FULL : (((1u << G) - 1u) << (lane & ~(unsigned)(G - 1)));
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(m, v, o);
  return v;
}

// Grid barrier on a 64-bit ticket counter (one atomic per block; never
// wraps in practice: 2^64 arrivals).  All launches of a kernel on one
// counter use the same grid, so the counter is a multiple of the grid at
// every launch start.  Requires every block to be resident.
// Spread grid barrier: the blocks arrive on DX_NCTR counters (block b on
// counter b mod DX_NCTR, each in its own 128-byte line), so same-address
// atomics at one L2 slice serialize DX_NCTR times fewer arrivals (measured on
// the k-means kernel, 148 blocks: 1.7 -> 1.1 us from the last arrival to the
// first exit).  The epoch is read from the block's own counter after
// griddepcontrol.wait (the previous launch has completed; this block has not
// arrived, so its counter holds a whole number of epochs plus fewer than its
// count of early arrivals).
#define DX_NCTR 8
__device__ __forceinline__ unsigned long long dx_bar_epoch(const unsigned long long* ctr) {
  const unsigned i = blockIdx.x % DX_NCTR;
  const unsigned long long cnt = (gridDim.x - i + DX_NCTR - 1) / DX_NCTR;
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr + i * 16) : "memory");
  return v / cnt;
}
// `epoch`: a shared variable thread 0 set from dx_bar_epoch (kept out of
// registers across the kernel's main loop)
__device__ __forceinline__ void dx_spread_barrier(unsigned long long* ctr, const unsigned long long& epoch_s) {
  __syncthreads();
  const unsigned long long epoch = epoch_s;
  if (threadIdx.x == 0)
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr + (blockIdx.x % DX_NCTR) * 16) : "memory");
  if (threadIdx.x < DX_NCTR && threadIdx.x < gridDim.x) {
    const unsigned long long target = (epoch + 1ull) * ((gridDim.x - threadIdx.x + DX_NCTR - 1) / DX_NCTR);
    unsigned long long v;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr + threadIdx.x * 16) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

__device__ __forceinline__ void dx_ticket_barrier(unsigned long long* ctr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long t = atomicAdd(ctr, 1ull);
    const unsigned long long target = (t / gridDim.x + 1ull) * gridDim.x;
    unsigned long long v;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// Block-per-column-group fold of per-block partials [nblk][width] into
// `cell`: block bk takes groups of 32 consecutive columns (lane = column, so
// every load is one coalesced 128-byte line); its warps split the partial
// rows (warp w sums rows w, w + NW, ... in order), then warp 0 adds the NW
// warp sums in order.  Groups of several cells share one index space
// (`first` = groups of the cells before).  Deterministic for a fixed grid.
template <class T, class P>
__device__ __forceinline__ void dx_coop_fold_b(const P* part, long long width, T scale, T* cell, bool counts,
                                               bool store, long long first) {
  __shared__ __align__(8) unsigned char fraw[32 * 33 * 8];
  T (*fred)[33] = reinterpret_cast<T (*)[33]>(fraw);
  unsigned long long (*fredu)[33] = reinterpret_cast<unsigned long long (*)[33]>(fraw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nblk = gridDim.x;
  const long long ng = (width + 31) / 32;
  for (long long gi = ((long long)blockIdx.x - first % nblk + nblk) % nblk; gi < ng; gi += nblk) {
    const long long c = gi * 32 + lane;
    const bool ok = c < width;
    T s = T(0);
    unsigned long long u = 0;
    for (int b0 = warp; b0 < nblk; b0 += 8 * nw) {
      P x[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int b = b0 + r * nw;
        x[r] = (ok && b < nblk) ? dx_ldcg(part + (long long)b * width + c) : P(0);
      }
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        if (counts) u += (unsigned long long)x[r];
        else s += (T)x[r];
      }
    }
    if (counts) fredu[warp][lane] = u;
    else fred[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && ok) {
      T v;
      if (counts) {
        unsigned long long t = 0;
        for (int w = 0; w < nw; ++w) t += fredu[w][lane];
        v = (T)t * scale;
      } else {
        T t = T(0);
        for (int w = 0; w < nw; ++w) t += fred[w][lane];
        v = t;
      }
      if (store) cell[c] = v;  // the cell's zero-fill was folded into this kernel
      else cell[c] += v;
    }
    __syncthreads();
  }
}

// Work counters (count mode, EvalCounters eval.hpp:60-65): per-thread
// counts summed per warp, one atomic per warp per counter.
__device__ __forceinline__ void dx_count_add(unsigned long long* c, unsigned long long ops, unsigned long long acc,
                                             unsigned long long cells) {
  if (ops) atomicAdd(c, ops);
  if (acc) atomicAdd(c + 1, acc);
  if (cells) atomicAdd(c + 2, cells);
}
__device__ __forceinline__ void dx_count_flush(unsigned long long* c, unsigned long long ops, unsigned long long acc,
                                               unsigned long long cells) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ops += __shfl_xor_sync(DX_FULL, ops, o);
    acc += __shfl_xor_sync(DX_FULL, acc, o);
    cells += __shfl_xor_sync(DX_FULL, cells, o);
  }
  if ((threadIdx.x & 31) == 0) dx_count_add(c, ops, acc, cells);
}

// Warp-per-column fold of per-block partials [nblk][width] into `cell`:
// global warp w folds columns w, w + W, ...; lanes take blocks lane, lane +
// 32, ... in order, then the fixed xor tree.  Deterministic for a fixed grid.
template <class T, class P>
__device__ __forceinline__ void dx_coop_fold_w(const P* part, long long width, T scale, T* cell, bool counts,
                                               bool store, long long first) {
  // columns of several cells share one index space: this cell's column c is
  // folded by global warp (first + c) mod (number of warps)
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  const int nblk = gridDim.x;
  const long long me = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  long long c0 = (me - first % nw + nw) % nw;
  for (long long c = c0; c < width; c += nw) {
    // eight loads in flight per lane (one L2 round trip for grids <= 256
    // blocks), then the lane's blocks in ascending order, then the xor tree
    T v;
    if (counts) {
      unsigned long long u = 0;
      for (int b0 = 0; b0 < nblk; b0 += 256) {
        P x[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int b = b0 + lane + 32 * r;
          x[r] = b < nblk ? dx_ldcg(part + (long long)b * width + c) : P(0);
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) u += (unsigned long long)x[r];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) u += __shfl_xor_sync(DX_FULL, u, o);
      v = (T)u * scale;
    } else {
      T s = T(0);
      for (int b0 = 0; b0 < nblk; b0 += 256) {
        P x[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int b = b0 + lane + 32 * r;
          x[r] = b < nblk ? dx_ldcg(part + (long long)b * width + c) : P(0);
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) s += (T)x[r];
      }
      v = dx_warp_sum(s);
    }
    if (lane == 0) {
      if (store) cell[c] = v;  // the cell's zero-fill was folded into this kernel
      else cell[c] += v;
    }
  }
}
// Cooperative fold of per-block partials [nblk][width] into `cell`: block b
// owns columns [8b, 8b+8); thread (c, g) sums rows g, g+R, ... in order, then a
// fixed tree over the R row groups.
// Deterministic for a fixed grid.
template <class T, class P>
__device__ __forceinline__ void dx_coop_fold(const P* part, long long width, T scale, T* cell, bool counts,
                                             bool store) {
  constexpr int C = 8;
  const int R = (blockDim.x / C) < 32 ? (blockDim.x / C) : 32;
  __shared__ T red[32][C];
  const int tx = threadIdx.x % C, ty = threadIdx.x / C;
  const int nblk = gridDim.x;
  for (long long c0 = (long long)blockIdx.x * C; c0 < width; c0 += (long long)gridDim.x * C) {  // block-uniform
    const long long c = c0 + tx;
    T s = T(0);
    if (c < width && ty < R) {
      if (counts) {
        unsigned long long u = 0;
        for (int b = ty; b < nblk; b += R) u += (unsigned long long)part[(long long)b * width + c];
        s = (T)u;
      } else {
        for (int b = ty; b < nblk; b += R) s += (T)part[(long long)b * width + c];
      }
    }
    if (ty < R) red[ty][tx] = s;
    __syncthreads();
    for (int h = 16; h > 0; h >>= 1) {
      if (ty < h && ty + h < R) red[ty][tx] += red[ty + h][tx];
      __syncthreads();
    }
    if (ty == 0 && c < width) {
      const T v = counts ? red[0][tx] * scale : red[0][tx];
      if (store) cell[c] = v;  // the cell's zero-fill was folded into this kernel
      else cell[c] += v;
    }
    __syncthreads();
  }
}
// Paired fp32 arithmetic (sm_100 FADD2 / FFMA2: two IEEE fp32 operations per
// instruction, each lane rounded exactly as the scalar op)
__device__ __forceinline__ float2 dx_f2sub(float2 a, float2 b) {
  float2 d;
  asm("{\n .reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " sub.rn.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 dx_f2add(float2 a, float2 b) {
  float2 d;
  asm("{\n .reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " add.rn.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 dx_f2mul(float2 a, float2 b) {
  float2 d;
  asm("{\n .reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " mul.rn.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 dx_f2fma(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n .reg .b64 ra, rb, rc, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " mov.b64 rc, {%6, %7};\n fma.rn.f32x2 rd, ra, rb, rc;\n mov.b64 {%0, %1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

extern "C" __global__ void __launch_bounds__(1024) dx_fin_f32(const float* p, int n, long long w, float* c) { dx_fin2<float, float>(p, n, w, 1.0f, c, false); }
extern "C" __global__ void __launch_bounds__(1024) dx_fin_f64(const double* p, int n, long long w, double* c) { dx_fin2<double, double>(p, n, w, 1.0, c, false); }
extern "C" __global__ void __launch_bounds__(1024) dx_fin_f32d(const float* p, int n, long long w, double* c) { dx_fin2<double, float>(p, n, w, 1.0, c, false); }
extern "C" __global__ void __launch_bounds__(1024) dx_fin_count_f32(const unsigned* p, int n, long long w, float s, float* c) { dx_fin2<float, unsigned>(p, n, w, s, c, true); }
extern "C" __global__ void __launch_bounds__(1024) dx_fin_count_f64(const unsigned* p, int n, long long w, double s, double* c) { dx_fin2<double, unsigned>(p, n, w, s, c, true); }

// Elementwise cell += src (host-level `r += table`), and fills.
extern "C" __global__ void dx_add_f32(float* c, const float* s, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) c[i] += s[i];
}
extern "C" __global__ void dx_add_f64(double* c, const double* s, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) c[i] += s[i];
}
extern "C" __global__ void dx_add_f64_f32(double* c, const float* s, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) c[i] += (double)s[i];
}
// Element-type conversion copies (f32 values into f64 cells and back).
extern "C" __global__ void dx_cvt_f32_f64(double* d, const float* s, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) d[i] = s[i];
}
extern "C" __global__ void dx_cvt_f64_f32(float* d, const double* s, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) d[i] = (float)s[i];
}
// Rank-ordered merge of gathered per-rank Accum deltas g[world][n] into the
// cell: cell = ((cell + d_0) + d_1) + ..., the left fold of the reference's
// chunk-overlay merge (eval.cpp:357-366) with ranks as chunks.  Every rank
// folds the same gathered data, so all ranks hold identical bits.
extern "C" __global__ void dx_rank_fold(const double* g, long long n, int world, double* cell) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double c = cell[i];
    for (int r = 0; r < world; ++r) c += g[(long long)r * n + i];
    cell[i] = c;
  }
}
// Bounds check of uploaded index leaves (fromOrdinal's check, index_set.cpp:99-106).
extern "C" __global__ void dx_check_index(const int* x, long long n, int size, int* bad) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int v = x[i];
    if (v < 0 || v >= size) atomicOr(bad, 1);
  }
}
