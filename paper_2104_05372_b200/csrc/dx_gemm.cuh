// dx_gemm.cuh — hand-written sm_100a tensor-core GEMM for dense contraction
// nests (`for i k. sum (for j. A.i.j * B.j.k)` recognized by the lowering).
//
//   C[m][n] (+)= isa_m isb_n sum_k A'[m][k] * B'[n][k]    (A', B' K-major fp16 pairs)
//
// tcgen05.mma kind::f16, cta_group::1, M = 128, N = BN, fp32 accumulators in
// TMEM.  fp32 parity with the f64 reference (<= 1e-4) uses fp16x3: every
// operand row r is scaled by a power of two s_r (its max |v| into [2^13,
// 2^14)) and arrives as a pair of fp16 images hi + lo (dx_f16_split: 11 + 11
// significand bits, the precision of a tf32 pair), written by the generated
// operand prologues of contract.inc; the MMA accumulates hi*hi + hi*lo +
// lo*hi and the epilogue multiplies by the exact inverse scales.  kind::f16
// runs twice the tf32 MMA rate on half the operand bytes (measured on the
// MLP's 8192x1024x1024 GEMMs: 121 -> 84 us).
// Operand tiles arrive by TMA (2-D tensor maps, SWIZZLE_128B, box 32 x rows)
// into a STAGES-deep mbarrier ring; one elected thread issues the MMAs and
// releases stages with tcgen05.commit; four epilogue warps drain TMEM with
// tcgen05.ld (warp w owns TMEM lanes 32w..32w+31 = tile rows) chunk by chunk.

#define DX_GEMM_BM 128
#define DX_GEMM_BK 64  // fp16 per 128-byte swizzle row

__device__ __forceinline__ unsigned long long dx_umma_desc_sw128(unsigned saddr) {
  // K-major, SWIZZLE_128B canonical layout: 8-row x 128 B atoms, SBO = 1024 B
  return (unsigned long long)((saddr & 0x3FFFFu) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

template <int BN>
__device__ __forceinline__ unsigned dx_idesc_f16() {
  // c_format F32 (bit 4), a/b format F16 (0 at bits 7, 10), K-major, N>>3 at 17, M>>4 at 24
  return (1u << 4) | ((unsigned)(BN >> 3) << 17) | ((unsigned)(DX_GEMM_BM >> 4) << 24);
}

__device__ __forceinline__ void dx_umma_f16(unsigned tmem, unsigned long long da, unsigned long long db,
                                            unsigned idesc, unsigned accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

// fp16x3 split of a scaled double (|x| < 2^14): x ~ hi + lo, hi and lo fp16
// (11-bit significands each: the pair carries ~22 bits, as a tf32 pair does)
__device__ __forceinline__ void dx_f16_split(double x, unsigned short& hi, unsigned short& lo) {
  float h;
  asm("cvt.rn.f16.f32 %0, %1;" : "=h"(hi) : "f"((float)x));
  asm("cvt.f32.f16 %0, %1;" : "=f"(h) : "h"(hi));
  asm("cvt.rn.f16.f32 %0, %1;" : "=h"(lo) : "f"((float)(x - (double)h)));
}
// the same split of an fp32 value: x - hi is exact in fp32 (hi is x rounded
// to 11 significand bits), so the images equal dx_f16_split's bit for bit
__device__ __forceinline__ void dx_f16_splitf(float x, unsigned short& hi, unsigned short& lo) {
  float h;
  asm("cvt.rn.f16.f32 %0, %1;" : "=h"(hi) : "f"(x));
  asm("cvt.f32.f16 %0, %1;" : "=f"(h) : "h"(hi));
  asm("cvt.rn.f16.f32 %0, %1;" : "=h"(lo) : "f"(__fsub_rn(x, h)));
}
// the scale as fp32 when it is a normal fp32 power of two (0 otherwise)
__device__ __forceinline__ float dx_f16_scale_f(double sc) {
  return sc >= 0x1p-126 && sc <= 0x1p126 ? (float)sc : 0.f;
}
// split x * sc: fp32 when the scale fits (x * scf is the exact product rounded
// once to fp32, as (float)((double)x * sc) is), fp64 otherwise
__device__ __forceinline__ void dx_f16_split_sc(float x, double sc, float scf, unsigned short& hi, unsigned short& lo) {
  if (scf != 0.f) dx_f16_splitf(__fmul_rn(x, scf), hi, lo);
  else dx_f16_split((double)x * sc, hi, lo);
}
// power-of-two scale putting a row's max |v| in [2^13, 2^14) (fp16 max 65504)
__device__ __forceinline__ double dx_f16_scale(double max_abs) {
  if (!(max_abs > 0.0) || !(max_abs < 1e300)) return 1.0;
  int e;
  frexp(max_abs, &e);  // max_abs < 2^e
  return ldexp(1.0, 14 - e);
}

__device__ __forceinline__ void dx_umma_commit(unsigned long long* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   dx_smem_addr(bar))
               : "memory");
}

// mbarrier wait with a bound: a descriptor/TMA fault traps (launch error)
// instead of spinning forever.
__device__ __forceinline__ void dx_mbar_wait_bounded(unsigned long long* bar, unsigned parity) {
  unsigned ok = 0;
  for (long long it = 0; it < (1LL << 26); ++it) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(dx_smem_addr(bar)), "r"(parity)
        : "memory");
    if (ok) return;
  }
  __trap();
}

#define DX_TMEM_LD32(taddr, v)                                                                                    \
  asm volatile(                                                                                                   \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"           \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                   \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),           \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),     \
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),   \
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])    \
      : "r"(taddr))

// Accumulation precision.  The tensor core adds into its fp32 accumulator
// with truncation, so a long K drifts (measured 1.5e-4 rel at K = 1024 with
// one accumulator, 3xTF32).  Two remedies, both free on TMEM: the large hi*hi
// products and the small residual products (hi*lo + lo*hi, ~2^-11 smaller)
// go to separate accumulators, and every DX_GEMM_CHUNK k-blocks the
// epilogue warps promote both into fp32 registers with round-to-nearest
// adds.  Accumulators are double-buffered in TMEM (4 x BN columns) so the
// promotion of chunk c overlaps the MMAs of chunk c+1.
#define DX_GEMM_CHUNK 1

// Warps 0..EW-1: epilogue (warp w owns TMEM lanes / tile rows 32(w%4)..+31 and
// accumulator columns [128(w/4), +128)); warp EW: TMA producer; warp EW+1:
// MMA issuer.  mode 0: C = acc, 1: C += acc.  MERGED: the three products
// share one accumulator (BN = 256 fits TMEM double-buffered; the promotion
// every 32 k keeps the truncation error at fp32 level).
// The row scales factor out of the k-sum: C[m][n] = isa_m isb_n sum_k
// (s_m A)(s_n B); the epilogue applies them before the store.
template <int BN, int STAGES, class CT, bool MERGED = false>
__device__ __forceinline__ void dx_gemm_f16x3(const dx_tmap* ta, const dx_tmap* tal, const dx_tmap* tb,
                                              const dx_tmap* tbl, long long M, long long N, long long K, CT* C,
                                              long long ldc, long long mode, long long ksplit, unsigned* tickets,
                                              const float* isa, const float* isb) {
  constexpr int BK = DX_GEMM_BK;  // K elements per 128-byte swizzle row
  constexpr unsigned A_BYTES = DX_GEMM_BM * 128, B_BYTES = BN * 128;
  constexpr unsigned STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  constexpr int NACC = MERGED ? 1 : 2;                   // accumulators per buffer
  constexpr unsigned TMEM_COLS = 2 * NACC * BN;
  constexpr int CW = BN < 128 ? BN : 128;                // accumulator columns per epilogue warp
  constexpr int EW = 4 * (BN / CW);                      // epilogue warps
  constexpr int TMA_W = EW, MMA_W = EW + 1;
  static_assert(TMEM_COLS == 128 || TMEM_COLS == 256 || TMEM_COLS == 512, "TMEM allocation");
  extern __shared__ __align__(1024) unsigned char dx_gemm_smem_raw[];
  unsigned char* smem = dx_gemm_smem_raw + ((1024u - (dx_smem_addr(dx_gemm_smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) unsigned long long full[STAGES], empty[STAGES], tfull[2], tempty[2];
  __shared__ unsigned tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NT = (int)((N + BN - 1) / BN);
  // split-K: CTA (tile, part) takes k-blocks [kb0, kb0 + KB); the parts of a
  // tile add into C one after another, in part order (ticket per tile), so the
  // result is deterministic
  const int S = (int)(ksplit > 1 ? ksplit : 1);
  const int tile = (int)(blockIdx.x / S), part = (int)(blockIdx.x % S);
  const int m0 = (int)(tile / NT) * DX_GEMM_BM, n0 = (int)(tile % NT) * BN;
  const int KBT = (int)((K + BK - 1) / BK);
  const int kb0 = (int)((long long)part * KBT / S);
  const int KB = (int)((long long)(part + 1) * KBT / S) - kb0;
  const int NC = (KB + DX_GEMM_CHUNK - 1) / DX_GEMM_CHUNK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      dx_mbar_init(&full[s], 1);
      dx_mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      dx_mbar_init(&tfull[b], 1);
      dx_mbar_init(&tempty[b], EW);
    }
    dx_fence_mbar_init();
  }
  if (warp == TMA_W) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dx_smem_addr(&tmem_base)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = tmem_base;

  if (warp == TMA_W) {
    if (lane == 0) {
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % STAGES;
        if (kb >= STAGES) dx_mbar_wait_bounded(&empty[s], (unsigned)(((kb / STAGES) - 1) & 1));
        unsigned char* st = smem + s * STAGE_BYTES;
        dx_mbar_expect_tx(&full[s], STAGE_BYTES);
        const int kc = (kb0 + kb) * BK;
        dx_tma_2d(st, ta, kc, m0, &full[s]);
        dx_tma_2d(st + A_BYTES, tal, kc, m0, &full[s]);
        dx_tma_2d(st + 2 * A_BYTES, tb, kc, n0, &full[s]);
        dx_tma_2d(st + 2 * A_BYTES + B_BYTES, tbl, kc, n0, &full[s]);
      }
    }
  } else if (warp == MMA_W) {
    if (lane == 0) {
      const unsigned idesc = dx_idesc_f16<BN>();
      for (int c = 0; c < NC; ++c) {
        const int b = c & 1;
        if (c >= 2) dx_mbar_wait_bounded(&tempty[b], (unsigned)(((c >> 1) - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const unsigned tbig = tmem + (unsigned)(b * NACC * BN), tsmall = MERGED ? tbig : tbig + BN;
        const int k1 = min(KB, (c + 1) * DX_GEMM_CHUNK);
        for (int kb = c * DX_GEMM_CHUNK; kb < k1; ++kb) {
          const int s = kb % STAGES;
          dx_mbar_wait_bounded(&full[s], (unsigned)((kb / STAGES) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const unsigned st = dx_smem_addr(smem + s * STAGE_BYTES);
          const unsigned first = kb == c * DX_GEMM_CHUNK;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {  // 16 fp16 (32 bytes) of K per MMA
            const unsigned long long ah = dx_umma_desc_sw128(st + kk * 32);
            const unsigned long long al = dx_umma_desc_sw128(st + A_BYTES + kk * 32);
            const unsigned long long bh = dx_umma_desc_sw128(st + 2 * A_BYTES + kk * 32);
            const unsigned long long bl = dx_umma_desc_sw128(st + 2 * A_BYTES + B_BYTES + kk * 32);
            const unsigned accum = !(first && kk == 0);
            if (!MERGED && BN <= 128) {
              // [B hi ; B lo] are contiguous SW128 row groups and [big | small]
              // contiguous TMEM columns: hi*hi and hi*lo as ONE N = 2 BN MMA
              // (same products, same accumulators, same order), so A hi is
              // read from shared memory once per k-step instead of twice --
              // the SS-mode MMAs are shared-memory-read bound (128 B/clk for
              // three N = 128 products, 107 B/clk this way)
              dx_umma_f16(tbig, ah, bh, dx_idesc_f16<2 * BN>(), accum);
            } else {
              dx_umma_f16(tbig, ah, bh, idesc, accum);
              dx_umma_f16(tsmall, ah, bl, idesc, MERGED ? 1u : accum);
            }
            dx_umma_f16(tsmall, al, bh, idesc, 1u);
          }
          dx_umma_commit(&empty[s]);  // frees the stage once these MMAs retire
        }
        dx_umma_commit(&tfull[b]);
      }
    }
  } else {
    // epilogue warps: promote each chunk into fp32 registers (RN adds)
    const int wq = warp & 3, cb = (warp >> 2) * CW;  // lane quarter, first column
    float acc[CW];
#pragma unroll
    for (int j = 0; j < CW; ++j) acc[j] = 0.f;
    const unsigned lanebase = tmem + ((unsigned)(wq * 32) << 16) + (unsigned)cb;
    for (int c = 0; c < NC; ++c) {
      const int b = c & 1;
      dx_mbar_wait_bounded(&tfull[b], (unsigned)((c >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (MERGED) {  // x16 loads: acc[128] + 16 in flight fit the 168 registers of 10 warps
#pragma unroll
        for (int q = 0; q < CW / 16; ++q) {
          unsigned v[16];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
              : "r"(lanebase + (unsigned)(b * NACC * BN + q * 16)));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 16; j += 2) {
            const float2 a2 = dx_f2add(make_float2(acc[q * 16 + j], acc[q * 16 + j + 1]),
                                       make_float2(__uint_as_float(v[j]), __uint_as_float(v[j + 1])));
            acc[q * 16 + j] = a2.x;
            acc[q * 16 + j + 1] = a2.y;
          }
        }
      } else {  // big (hi*hi) + small (hi*lo + lo*hi) accumulators
#pragma unroll
        for (int q = 0; q < CW / 32; ++q) {
          unsigned vb[32], vs[32];
          DX_TMEM_LD32(lanebase + (unsigned)(b * NACC * BN + q * 32), vb);
          DX_TMEM_LD32(lanebase + (unsigned)(b * NACC * BN + BN + q * 32), vs);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 32; j += 2) {  // f32x2 pairs, same per-lane rounding
            const float2 t = dx_f2add(make_float2(__uint_as_float(vb[j]), __uint_as_float(vb[j + 1])),
                                      make_float2(__uint_as_float(vs[j]), __uint_as_float(vs[j + 1])));
            const float2 a2 = dx_f2add(make_float2(acc[q * 32 + j], acc[q * 32 + j + 1]), t);
            acc[q * 32 + j] = a2.x;
            acc[q * 32 + j + 1] = a2.y;
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) dx_mbar_arrive(&tempty[b]);
    }
    if (S > 1) {  // wait for the previous parts of this tile
      if (threadIdx.x == 0) {
        while (true) {
          unsigned v;
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(tickets + tile) : "memory");
          if ((int)v == part) break;
          __nanosleep(64);
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(EW * 32) : "memory");
      if (part > 0) mode = 1;
    }
    const long long row = m0 + wq * 32 + lane;
    if (row < M) {  // undo the operand row scales (powers of two: exact)
      const float ra = isa[row];
      const int nc = n0 + cb;
#pragma unroll
      for (int j = 0; j < CW; ++j) acc[j] *= ra * (nc + j < N ? __ldg(isb + nc + j) : 0.f);
    }
    if (row < M) {
      const int nc = n0 + cb;  // this warp's first output column
      CT* out = C + row * ldc + nc;
      // MERGED (N = 256) kernels are only planned for full, 16-byte aligned
      // column tiles (contract.inc), so they carry no scalar fallback (whose
      // unrolled code would push acc[] out of the 168 registers of 10 warps)
      const bool vec = sizeof(CT) == 4 && (MERGED || (nc + CW <= N && ((ldc | nc) & 3) == 0 &&
                                                      ((reinterpret_cast<unsigned long long>(C) & 15) == 0)));
      const bool vecd = sizeof(CT) == 8 && (MERGED || (nc + CW <= N && ((ldc | nc) & 1) == 0 &&
                                                       ((reinterpret_cast<unsigned long long>(C) & 15) == 0)));
      if (vec && mode == 0) {
#pragma unroll
        for (int j = 0; j < CW; j += 4)
          *reinterpret_cast<float4*>(out + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
      } else if (vecd) {
        // f64 cells: 16-byte read-modify-writes, 16 loads in flight per batch
        // (the row-per-thread RMW is latency-bound when few tiles exist)
        double2* o2 = reinterpret_cast<double2*>(out);
        constexpr int QB = 16;  // 16-byte loads per batch
#pragma unroll
        for (int j0 = 0; j0 < CW; j0 += 2 * QB) {
          double2 cur[QB];
#pragma unroll
          for (int q = 0; q < QB; ++q) cur[q] = mode == 0 ? make_double2(0.0, 0.0) : o2[j0 / 2 + q];
#pragma unroll
          for (int q = 0; q < QB; ++q)
            o2[j0 / 2 + q] = make_double2(cur[q].x + (double)acc[j0 + 2 * q], cur[q].y + (double)acc[j0 + 2 * q + 1]);
        }
      } else if (!MERGED) {
#pragma unroll
        for (int j = 0; j < CW; ++j) {
          if (nc + j < N) {
            if (mode == 0) out[j] = (CT)acc[j];
            else out[j] += (CT)acc[j];
          }
        }
      } else {  // f32 cells with += (no 16-byte RMW path for them)
#pragma unroll
        for (int j = 0; j < CW; j += 4) {
          float4 o = *reinterpret_cast<float4*>(out + j);
          o.x += acc[j];
          o.y += acc[j + 1];
          o.z += acc[j + 2];
          o.w += acc[j + 3];
          *reinterpret_cast<float4*>(out + j) = o;
        }
      }
    }
    if (S > 1) {  // release the next part
      __threadfence();
      asm volatile("bar.sync 1, %0;" ::"n"(EW * 32) : "memory");
      // the last part resets the tile's ticket: it stays in [0, S) and never
      // wraps (S need not divide 2^32)
      if (threadIdx.x == 0) {
        if (part == S - 1) atomicExch(tickets + tile, 0u);
        else atomicAdd(tickets + tile, 1u);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == TMA_W) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
  }
}

#define DX_GEMM_SMEM(BN, STAGES) (STAGES * (2 * DX_GEMM_BM * 128 + 2 * (BN)*128) + 1024)

extern "C" __global__ void __launch_bounds__(192, 1)
    dx_gemm_f16x3_n128(const __grid_constant__ dx_tmap ta, const __grid_constant__ dx_tmap tal,
                       const __grid_constant__ dx_tmap tb, const __grid_constant__ dx_tmap tbl, long long M,
                       long long N, long long K, float* C, long long ldc, long long mode, long long ksplit,
                       unsigned* tickets, const float* isa, const float* isb) {
  dx_gemm_f16x3<128, 3, float>(&ta, &tal, &tb, &tbl, M, N, K, C, ldc, mode, ksplit, tickets, isa, isb);
}
extern "C" __global__ void __launch_bounds__(192, 1)
    dx_gemm_f16x3_n128_d(const __grid_constant__ dx_tmap ta, const __grid_constant__ dx_tmap tal,
                         const __grid_constant__ dx_tmap tb, const __grid_constant__ dx_tmap tbl, long long M,
                         long long N, long long K, double* C, long long ldc, long long mode, long long ksplit,
                         unsigned* tickets, const float* isa, const float* isb) {
  dx_gemm_f16x3<128, 3, double>(&ta, &tal, &tb, &tbl, M, N, K, C, ldc, mode, ksplit, tickets, isa, isb);
}
// f64 parity mode (dxl_options.float64): the same contraction class in
// binary64, as the reference evaluates it (eval.cpp:500-514).  SIMT f64 FMA,
// 64 x 64 output tile per 256-thread block (4 x 4 per thread), K in steps of
// 16 staged through shared memory; A and B are K-major f64 images written by
// the operand prologues.  C[m][n] (+)= sum_k A[m][k] * B[n][k], each output
// summed in ascending k (deterministic).
extern "C" __global__ void __launch_bounds__(256) dx_gemm_f64(const double* __restrict__ A, const double* __restrict__ B,
                                                              long long M, long long N, long long K, double* C,
                                                              long long ldc, long long mode) {
  __shared__ double As[16][64 + 1], Bs[16][64 + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const long long NTn = (N + 63) / 64;
  const long long m0 = (long long)(blockIdx.x / NTn) * 64, n0 = (long long)(blockIdx.x % NTn) * 64;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (long long k0 = 0; k0 < K; k0 += 16) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = threadIdx.x + 256 * i, r = idx >> 4, c = idx & 15;
      const long long k = k0 + c;
      As[c][r] = (m0 + r < M && k < K) ? A[(m0 + r) * K + k] : 0.0;
      Bs[c][r] = (n0 + r < N && k < K) ? B[(n0 + r) * K + k] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __fma_rn(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const long long m = m0 + ty + 16 * i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const long long n = n0 + tx + 16 * j;
      if (n >= N) continue;
      double* o = C + m * ldc + n;
      *o = mode ? *o + acc[i][j] : acc[i][j];
    }
  }
}
