// a7: the LU Schur update  A[k1:N, c0:c1] -= A[k1:N, k0:k1] * A[k0:k1, c0:c1]  (Alg. 2 P:236,
// P:260-261), persistent and TMA-fed, on the FP64 tensor cores (DMMA).
//
// B200 has no FP64 kind for tcgen05.mma, so the FP64 tensor path is the warp-level DMMA
// (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4).  What TMA adds here is the operand staging:
//   * one producer warp (one elected lane) streams 16-deep K slices of the L panel and of the U row
//     through a 4-stage shared-memory ring with cp.async.bulk.tensor (SWIZZLE_128B boxes), arming
//     full / empty mbarriers, and the next tile's C through its own buffer; the consumer warps never
//     issue a global load for A, B or C and never meet at a CTA-wide barrier in the main loop;
//   * 8 consumer warps (2 x 4 warp tiles of 32 x 16; 4 per scheduler across the SM's 2 CTAs, so a
//     warp at a barrier or in its epilogue leaves three others to feed the DMMA pipe);
//   * every CTA (2 per SM) walks TM_TILES_PER_CTA output tiles in grouped raster order, and the
//     producer runs ahead into the next tile's K slices while the consumers finish the previous
//     tile's epilogue (no per-tile prologue bubble); CTAs still retire often enough for the
//     lookahead's high-priority panel kernels to get SMs;
//   * 128-byte swizzle + a fragment row order chosen so every DMMA fragment load is
//     bank-conflict free: the A (L panel) box is {16 rows, 16 k, 4 row groups}; accumulator row g
//     of a fragment holds panel row (g & 3) + 8 (g >> 2) + 4 s of its 16-row group (s = the
//     fragment's half), which spreads the 32 lanes over all 16 8-byte slots of a 128-byte row.
// The accumulators start from C and the A operand is sign-flipped, so every tile accumulates
// A_ij - A_ik A_kj in the DMMAs' own order -- bit-identical to gemm.cu's kernel.  (Accumulating the
// product from zero and subtracting it afterwards, as "A_ij - (A_ik A_kj)" reads, measured 10x
// worse HPL3 at C3: the product of the large growth-inflated factors cancels against A_ij.)
// Epilogue: the tile written back with the fused a12 column abs-sums (colpart) when asked.
// Eligibility (else gemm.cu's cp.async kernel): lda even, A 16-byte aligned, N and nb multiples of
// 16 (every TMA box in bounds or zero-filled past the matrix).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "hlq_internal.cuh"

namespace hlq {

namespace {
constexpr int TM_BM = 64, TM_BN = 64, TM_BK = 16, TM_ST = 4;
// consumer warps per CTA: CONS = 4 (2 x 2 warp tiles of 32 x 32) or 8 (2 x 4 warp tiles of 32 x 16:
// twice the warps per scheduler to cover each other's barrier / epilogue gaps, 0.75 instead of 0.5
// fragment loads per DMMA); + the producer warp
constexpr int tm_threads(int cons) { return 32 * (cons + 1); }
constexpr int TM_A_BYTES = TM_BM * TM_BK * 8;    // 8 KB
constexpr int TM_B_BYTES = TM_BN * TM_BK * 8;    // 8 KB
constexpr int TM_STAGE = TM_A_BYTES + TM_B_BYTES;
constexpr int TM_C_BYTES = TM_BM * TM_BN * 8;    // 32 KB: the next tile's C, prefetched by TMA
constexpr int TM_SMEM = TM_ST * TM_STAGE + TM_C_BYTES + 1024 /*align*/ + 2 * TM_BN * 8 + 256;
constexpr int TM_CTAS_PER_SM = 2;
// output tiles per CTA: enough to amortise the pipeline fill, few enough that CTAs retire every
// ~50 us so the high-priority panel stream of the lookahead gets SMs (a fully persistent grid
// starved it: C3 GETRF stage 161 -> 797 ms of stream time, the step 905 -> 944 ms)
constexpr int TM_TILES_PER_CTA = 4;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void dmma_tm(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
// row within a 16-row group held by accumulator row g of a fragment half s (conflict-free A loads)
__device__ __forceinline__ int frag_row(int g, int s) { return (g & 3) + 8 * (g >> 2) + 4 * s; }
}  // namespace

struct TmaMaps {
  CUtensorMap a;  // 3D {16 rows, columns, row groups of 16} over the whole matrix: the L panel role
  CUtensorMap b;  // 2D {rows, columns} over the whole matrix: the U row-block role
  CUtensorMap c;  // 3D like a, box {16, 64, 4}: a 64 x 64 output tile
};

template <int TM_CONS>
__global__ void __launch_bounds__(tm_threads(TM_CONS), TM_CTAS_PER_SM)
    k_dgemm_tma(const __grid_constant__ TmaMaps maps, double* __restrict__ C, int64_t ldc,
                int64_t M, int64_t N, int K, int arow0, int kcol0, int bcol0,
                const uint8_t* __restrict__ dec, int k, int want, double* __restrict__ colpart,
                int64_t ldp, int64_t tpc) {
  if (dec != nullptr && dec[k] != want) return;  // predicated launch (the branch not taken)
  extern __shared__ __align__(1024) unsigned char tm_smem_raw[];
  // align the stage ring to 1024 bytes in the SHARED window (the swizzle atom), by pointer
  // arithmetic on the __shared__ array so the fragment loads stay LDS
  unsigned char* sm = tm_smem_raw + ((1024u - (smem_u32(tm_smem_raw) & 1023u)) & 1023u);
  double* Cs = (double*)(sm + TM_ST * TM_STAGE);  // the prefetched C tile (swizzled like A)
  uint64_t* full = (uint64_t*)(sm + TM_ST * TM_STAGE + TM_C_BYTES);
  uint64_t* empty = full + TM_ST;
  uint64_t* cfull = empty + TM_ST;
  uint64_t* cempty = cfull + 1;
  double* red = (double*)(cempty + 1);  // 2 x 64 column partials (a12 epilogue)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < TM_ST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, TM_CONS);
    }
    mbar_init(cfull, 1);
    mbar_init(cempty, TM_CONS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t ntm = (M + TM_BM - 1) / TM_BM, ntn = (N + TM_BN - 1) / TM_BN;
  const int64_t ntiles = ntm * ntn;
  const int KT = K / TM_BK;
  // this CTA's tiles: a contiguous run of the grouped raster order, so that the tiles in flight at
  // any time form one window of the matrix (L2 reuse of the L panel rows and U row columns)
  const int64_t t0 = (int64_t)blockIdx.x * tpc;
  const int64_t t1 = t0 + tpc < ntiles ? t0 + tpc : ntiles;
  auto tile_coords = [&](int64_t t, int64_t& tm, int64_t& tn) {  // grouped raster (8 tile rows)
    const int64_t per_group = 8 * ntn;
    const int64_t grp = t / per_group;
    const int64_t first_tm = grp * 8;
    const int64_t gsz = (ntm - first_tm < 8) ? (ntm - first_tm) : 8;
    tm = first_tm + (t % per_group) % gsz;
    tn = (t % per_group) / gsz;
  };

  if (warp == TM_CONS) {
    // ---------------- producer: one lane streams the K slices of every tile of this CTA
    if (lane == 0) {
      int s = 0;
      unsigned ph = 0, cph = 0;
      for (int64_t t = t0; t < t1; ++t) {
        int64_t tm, tn;
        tile_coords(t, tm, tn);
        const int rg = (int)((arow0 + tm * TM_BM) >> 4);   // row group of the panel rows
        const int bc = (int)(bcol0 + tn * TM_BN);          // first output column
        // the tile's C (issued after every K slice of the previous tile: a full tile of lead)
        mbar_wait(cempty, cph ^ 1);
        mbar_expect_tx(cfull, TM_C_BYTES);
        tma_load_3d(Cs, &maps.c, cfull, 0, bc, rg);
        cph ^= 1;
        for (int kt = 0; kt < KT; ++kt) {
          mbar_wait(empty + s, ph ^ 1);
          unsigned char* st = sm + s * TM_STAGE;
          mbar_expect_tx(full + s, TM_STAGE);
          tma_load_3d(st, &maps.a, full + s, 0, kcol0 + kt * TM_BK, rg);
          tma_load_2d(st + TM_A_BYTES, &maps.b, full + s, kcol0 + kt * TM_BK, bc);
          if (++s == TM_ST) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
    return;
  }
  // ---------------- consumers: TM_CONS warps, warp tile 32 x WTN (wm, wn)
  constexpr int WN = TM_CONS / 2, WTN = TM_BN / WN, NI = WTN / 8;
  const int g = lane >> 2, t4 = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;
  int s = 0;
  unsigned ph = 0, cph = 0;
  for (int64_t t = t0; t < t1; ++t) {
    int64_t tm, tn;
    tile_coords(t, tm, tn);
    // the accumulators start from C (prefetched by TMA into the swizzled C buffer): the update
    // accumulates into A_ij in the DMMAs' own order, bit-identical to gemm.cu's kernel
    const int64_t m0 = tm * TM_BM, n0 = tn * TM_BN;
    double acc[4][NI][2];
    mbar_wait(cfull, cph);
    __syncwarp();
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      const int mhi = wm * 2 + (mi >> 1), mlo = frag_row(g, mi & 1);
#pragma unroll
      for (int ni = 0; ni < NI; ++ni)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int nn = wn * WTN + ni * 8 + 2 * t4 + h;  // C box: 128-byte row = (mhi, column)
          acc[mi][ni][h] = Cs[(mhi * 64 + nn) * 16 + ((((mlo >> 1) ^ (nn & 7)) << 1) | (mlo & 1))];
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // (as for the K stages)
    __syncwarp();
    if (lane == 0) mbar_arrive(cempty);
    cph ^= 1;
    for (int kt = 0; kt < KT; ++kt) {
      mbar_wait(full + s, ph);
      // the lanes may leave the try_wait loop in different iterations: reconverge before the
      // warp-synchronous mma.sync (.aligned) -- without this, a few fragments were intermittently
      // corrupted (lanes executing the DMMAs apart)
      __syncwarp();
      const double* As = (const double*)(sm + s * TM_STAGE);
      const double* Bs = (const double*)(sm + s * TM_STAGE + TM_A_BYTES);
#pragma unroll
      for (int k4 = 0; k4 < TM_BK; k4 += 4) {
        const int kk = k4 + t4;
        double a[4], b[NI];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
          const int mhi = wm * 2 + (mi >> 1), mlo = frag_row(g, mi & 1);
          // C - A B: the A operand sign-flipped on the integer pipe
          a[mi] = neg_bits(As[(mhi * 16 + kk) * 16 + ((((mlo >> 1) ^ (kk & 7)) << 1) | (mlo & 1))]);
        }
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          const int nn = wn * WTN + ni * 8 + g;
          b[ni] = Bs[nn * 16 + ((((kk >> 1) ^ g) << 1) | (kk & 1))];
        }
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) dmma_tm(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
      }
      // release the stage: the fragment loads (generic proxy) must be complete and ordered before
      // the producer's next TMA write into it (async proxy) -- the cross-proxy WAR fence; without
      // it ptxas let the arrive overtake the last loads of the stage and a few fragments were
      // intermittently read after the next K slice had landed
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
      if (++s == TM_ST) {
        s = 0;
        ph ^= 1;
      }
    }
    // epilogue: the accumulators are the updated tile
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      const int64_t row = m0 + (wm * 2 + (mi >> 1)) * 16 + frag_row(g, mi & 1);
      if (row >= M) continue;
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) {
        const int64_t col = n0 + wn * WTN + ni * 8 + 2 * t4;
        if (col < N) C[col * ldc + row] = acc[mi][ni][0];
        if (col + 1 < N) C[(col + 1) * ldc + row] = acc[mi][ni][1];
      }
    }
    if (colpart != nullptr) {
      // fused a12: per-column |C_new| sums over the tile's 64 rows (rows >= M are exact zeros)
#pragma unroll
      for (int ni = 0; ni < NI; ++ni)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double v = 0.0;
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) v += fabs(acc[mi][ni][h]);
          v += __shfl_xor_sync(0xffffffffu, v, 4);
          v += __shfl_xor_sync(0xffffffffu, v, 8);
          v += __shfl_xor_sync(0xffffffffu, v, 16);
          if (g == 0) red[wm * TM_BN + wn * WTN + ni * 8 + 2 * t4 + h] = v;
        }
      asm volatile("bar.sync 1, %0;" ::"n"(32 * TM_CONS) : "memory");
      if (tid < TM_BN && n0 + tid < N) colpart[tm * ldp + n0 + tid] = red[tid] + red[TM_BN + tid];
      asm volatile("bar.sync 1, %0;" ::"n"(32 * TM_CONS) : "memory");
    }
  }
}

// ---- host side ---------------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    else
      cudaGetLastError();
  }
  return fn;
}

// Tensor maps of the whole N x N matrix (ld lda) for the TMA Schur update; returns nullptr when the
// matrix is not eligible (the caller keeps the cp.async kernel).  The maps live in the returned
// heap block (free with free_tma_maps).
void* make_tma_maps(const double* A, int64_t N, int64_t lda, int nb) {
  static int off = -1;
  if (off < 0) off = getenv("HLQ_DGEMM_TMA") ? (atoi(getenv("HLQ_DGEMM_TMA")) == 0) : 0;
  if (off) return nullptr;
  if ((lda & 1) || (((uintptr_t)A) & 15) || (N % 16) || (nb % 16) || N < 16) return nullptr;
  if (N > (int64_t)1 << 31) return nullptr;
  auto fn = encode_fn();
  if (!fn) return nullptr;
  TmaMaps* m = (TmaMaps*)aligned_alloc(64, sizeof(TmaMaps));
  if (!m) return nullptr;
  memset(m, 0, sizeof(*m));
  const cuuint32_t estr3[3] = {1, 1, 1}, estr2[2] = {1, 1};
  // A role: dims {16 (rows within a group), N (columns), N/16 (row groups)}
  const cuuint64_t gdA[3] = {16, (cuuint64_t)N, (cuuint64_t)(N / 16)};
  const cuuint64_t gsA[2] = {(cuuint64_t)lda * 8, 16 * 8};
  const cuuint32_t boxA[3] = {16, TM_BK, TM_BM / 16};
  CUresult r1 = fn(&m->a, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)A, gdA, gsA, boxA, estr3,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  // B role: dims {N (rows = k), N (columns)}
  const cuuint64_t gdB[2] = {(cuuint64_t)N, (cuuint64_t)N};
  const cuuint64_t gsB[1] = {(cuuint64_t)lda * 8};
  const cuuint32_t boxB[2] = {TM_BK, TM_BN};
  CUresult r2 = fn(&m->b, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)A, gdB, gsB, boxB, estr2,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const cuuint32_t boxC[3] = {16, TM_BN, TM_BM / 16};
  CUresult r3 = fn(&m->c, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)A, gdA, gsA, boxC, estr3,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r1 != CUDA_SUCCESS || r2 != CUDA_SUCCESS || r3 != CUDA_SUCCESS) {
    free(m);
    return nullptr;
  }
  return m;
}

void free_tma_maps(void* m) { free(m); }

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// A[k1 : k1+M, c0 : c0+nc] -= A[k1 : k1+M, k0 : k0+K] * A[k0 : k0+K, c0 : c0+nc] on the TMA path
// (maps from make_tma_maps for this matrix); false when K or the tile origin is not eligible.
bool launch_schur_tma(const void* maps, double* A, int64_t lda, int64_t k0, int64_t k1, int64_t c0,
                      int64_t M, int64_t nc, int K, const uint8_t* dec, int k, int want,
                      double* colpart, int64_t ldp, cudaStream_t st) {
  if (!maps || K % TM_BK || k1 % 16 || M <= 0 || nc <= 0) return false;
  static int cons = -1;
  // 8 consumer warps by default (C3 step-1 shape: 33.5 TF vs 32.9 with 4; cuBLAS DGEMM on the same
  // shape 33.0, profiles/r02/schur_vs_cublas.jsonl); HLQ_TMA_CONS=4 selects the 2 x 2 warp grid
  if (cons < 0) cons = (getenv("HLQ_TMA_CONS") && atoi(getenv("HLQ_TMA_CONS")) == 4) ? 4 : 8;
  static unsigned long long attr = 0;
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(k_dgemm_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, TM_SMEM);
    cudaFuncSetAttribute(k_dgemm_tma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, TM_SMEM);
  }
  const int64_t tiles = ((M + TM_BM - 1) / TM_BM) * ((nc + TM_BN - 1) / TM_BN);
  static int64_t tpc = -1;
  if (tpc < 0) tpc = getenv("HLQ_TMA_TPC") ? atoll(getenv("HLQ_TMA_TPC")) : TM_TILES_PER_CTA;
  const int64_t tpc_eff = std::max<int64_t>(
      1, std::min<int64_t>(tpc, tiles / ((int64_t)sm_count() * TM_CTAS_PER_SM)));
  const int64_t grid = (tiles + tpc_eff - 1) / tpc_eff;
  ::hlq::g_launches++;
  if (cons == 8)
    k_dgemm_tma<8><<<(unsigned)grid, tm_threads(8), TM_SMEM, st>>>(
        *(const TmaMaps*)maps, A + c0 * lda + k1, lda, M, nc, K, (int)k1, (int)k0, (int)c0, dec, k,
        want, colpart, ldp ? ldp : nc, tpc_eff);
  else
    k_dgemm_tma<4><<<(unsigned)grid, tm_threads(4), TM_SMEM, st>>>(
        *(const TmaMaps*)maps, A + c0 * lda + k1, lda, M, nc, K, (int)k1, (int)k0, (int)c0, dec, k,
        want, colpart, ldp ? ldp : nc, tpc_eff);
  return true;
}

}  // namespace hlq

// ---- test hook (include/hlq.h hlq_test_schur): one Schur update on a device matrix ------------
extern "C" int hlq_test_schur(double* A, int64_t N, int64_t lda, int64_t k0, int32_t K,
                              int32_t use_tma, void* stream) {
  using namespace hlq;
  if (!A) return -1;
  if (N <= 0) return -2;
  if (lda < N) return -3;
  if (k0 < 0 || K <= 0 || k0 + K > N) return -4;
  const int64_t k1 = k0 + K, M = N - k1;
  cudaStream_t st = (cudaStream_t)stream;
  void* maps = use_tma ? make_tma_maps(A, N, lda, K) : nullptr;
  bool done = false;
  if (maps)
    done = launch_schur_tma(maps, A, lda, k0, k1, k1, M, M, K, nullptr, 0, 0, nullptr, 0, st);
  if (!done)
    launch_dgemm(A + k1 * lda + k1, lda, A + k0 * lda + k1, lda, A + k1 * lda + k0, lda, M, M, K,
                 true, true, nullptr, 0, 0, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (maps) free_tma_maps(maps);
  if (e != cudaSuccess) return HLQ_ERR_CUDA;
  return done ? 1 : 0;
}
