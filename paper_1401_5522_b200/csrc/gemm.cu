// a7 (and a5/a6): FP64 tensor-core GEMM  C = beta*C + alpha*A*B  on sm_100a.
//
// B200 has no FP64 kind for tcgen05.mma, so the FP64 tensor path is the warp-level DMMA
// (mma.sync.aligned.m8n8k4.row.col.f64 -> SASS DMMA.884), measured at 37.2 TFLOP/s on this pool
// (profiles/r01/peak_dmma.jsonl).  Design:
//   * CTA tile 64 x 64, 4 warps as 2 (M) x 2 (N), warp tile 32 x 32 = 4 x 4 DMMA fragments,
//     64 FP64 accumulators per thread; 4 CTAs per SM so one CTA's C load/store and barriers
//     overlap the others' main loops (K = nb = 256 is short).  Other warp grids by template.
//   * K staged through shared memory in BK=16 slices by a 3-stage cp.async pipeline;
//     A slice stored [k][m] (ld 132), B slice [n][k] (ld 20): both paddings make every DMMA
//     fragment load (lane -> (row g, k t)) bank-conflict free.
//   * grouped rasterisation (8 tile-rows per group) for L2 reuse of the A panel / B row.
// The Schur update of the LU step (Alg. 2) is C = C - L_panel * U_row on the
// strided trailing submatrix; TRSM / SWPTRSM are C = X * U^-1 and C = L^-1 * (P X).
#include <stdlib.h>
#include <string.h>

#include "hlq_internal.cuh"

namespace hlq {

constexpr int BK = 16, STAGES = 3;
constexpr int LDB_S = BK + 4;
// warp grid WM x WN of 32 x 32 warp tiles: CTA tile (32 WM) x (32 WN)
template <int WM> __host__ __device__ constexpr int gemm_bm() { return 32 * WM; }
template <int WM> __host__ __device__ constexpr int gemm_lda_s() { return 32 * WM + 4; }
template <int WM> __host__ __device__ constexpr int gemm_a_stage() { return BK * gemm_lda_s<WM>(); }
template <int WN> __host__ __device__ constexpr int gemm_bn() { return 32 * WN; }
template <int WN> __host__ __device__ constexpr int gemm_b_stage() { return gemm_bn<WN>() * LDB_S; }
template <int WM, int WN> __host__ __device__ constexpr int gemm_smem() {
  return (gemm_a_stage<WM>() + gemm_b_stage<WN>()) * STAGES * (int)sizeof(double);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <bool V16, int WM, int WN>
__device__ __forceinline__ void load_stage(double* As, double* Bs, const double* __restrict__ A,
                                           int64_t lda, const double* __restrict__ B, int64_t ldb,
                                           int64_t M, int64_t N, int K, int64_t m0, int64_t n0,
                                           int k0, int tid) {
  constexpr int NT = 32 * WM * WN, BM = gemm_bm<WM>(), LDA_S = gemm_lda_s<WM>();
  if (V16) {
    // A: BK x BM doubles = BK * BM / 2 16-byte chunks
#pragma unroll
    for (int i = 0; i < BK * BM / 2 / NT; ++i) {
      int q = tid + NT * i;
      int kk = q / (BM / 2), mm = (q % (BM / 2)) * 2;
      bool ok = (k0 + kk < K) && (m0 + mm < M);
      const double* src = ok ? A + (int64_t)(k0 + kk) * lda + m0 + mm : A;
      cp_async16(As + kk * LDA_S + mm, src, ok);
    }
    // B: BN x BK doubles = BN * BK / 2 chunks
#pragma unroll
    for (int i = 0; i < gemm_bn<WN>() * BK / 2 / NT; ++i) {
      int q = tid + NT * i;
      int nn = q / (BK / 2), kk = (q % (BK / 2)) * 2;
      bool ok = (n0 + nn < N) && (k0 + kk < K);
      const double* src = ok ? B + (n0 + nn) * ldb + k0 + kk : B;
      cp_async16(Bs + nn * LDB_S + kk, src, ok);
    }
  } else {
#pragma unroll
    for (int i = 0; i < BK * BM / NT; ++i) {
      int q = tid + NT * i;
      int kk = q / BM, mm = q % BM;
      bool ok = (k0 + kk < K) && (m0 + mm < M);
      const double* src = ok ? A + (int64_t)(k0 + kk) * lda + m0 + mm : A;
      cp_async8(As + kk * LDA_S + mm, src, ok);
    }
#pragma unroll
    for (int i = 0; i < gemm_bn<WN>() * BK / NT; ++i) {
      int q = tid + NT * i;
      int nn = q / BK, kk = q % BK;
      bool ok = (n0 + nn < N) && (k0 + kk < K);
      const double* src = ok ? B + (n0 + nn) * ldb + k0 + kk : B;
      cp_async8(Bs + nn * LDB_S + kk, src, ok);
    }
  }
}

template <bool V16, int WM, int WN>
__global__ void __launch_bounds__(32 * WM * WN, 16 / (WM * WN) > 0 ? 16 / (WM * WN) : 1)
    k_dgemm(double* __restrict__ C, int64_t ldc, const double* __restrict__ A, int64_t lda,
            const double* __restrict__ B, int64_t ldb, int64_t M, int64_t N, int K, int neg,
            int beta, const uint8_t* __restrict__ dec, int k, int want,
            double* __restrict__ colpart, int64_t ldp) {
  if (dec != nullptr && dec[k] != want) return;  // predicated launch: the other branch was taken
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  constexpr int BM = gemm_bm<WM>(), BN = gemm_bn<WN>(), B_STAGE = gemm_b_stage<WN>();
  constexpr int LDA_S = gemm_lda_s<WM>(), A_STAGE = gemm_a_stage<WM>();
  double* Bs = smem + STAGES * A_STAGE;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % WM, wn = warp / WM;

  // grouped rasterisation
  const int64_t ntm = (M + BM - 1) / BM, ntn = (N + BN - 1) / BN;
  const int64_t bid = blockIdx.x;
  const int64_t per_group = 8 * ntn;
  const int64_t grp = bid / per_group;
  const int64_t first_tm = grp * 8;
  const int64_t gsz = (ntm - first_tm < 8) ? (ntm - first_tm) : 8;
  const int64_t tm = first_tm + (bid % per_group) % gsz;
  const int64_t tn = (bid % per_group) / gsz;
  const int64_t m0 = tm * BM, n0 = tn * BN;

  double acc[4][4][2];
  // rows / cols of this thread's accumulators
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      int64_t row = m0 + wm * 32 + mi * 8 + g;
      int64_t col = n0 + wn * 32 + ni * 8 + 2 * t;
      double c0 = 0.0, c1 = 0.0;
      if (beta && row < M) {
        if (col < N) c0 = C[col * ldc + row];
        if (col + 1 < N) c1 = C[(col + 1) * ldc + row];
      }
      acc[mi][ni][0] = c0;
      acc[mi][ni][1] = c1;
    }

  const int KT = (K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT)
      load_stage<V16, WM, WN>(As + s * A_STAGE, Bs + s * B_STAGE, A, lda, B, ldb, M, N, K, m0, n0, s * BK,
                      tid);
    cp_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    {
      int nk = kt + STAGES - 1;
      if (nk < KT) {
        int sl = nk % STAGES;
        load_stage<V16, WM, WN>(As + sl * A_STAGE, Bs + sl * B_STAGE, A, lda, B, ldb, M, N, K, m0, n0,
                        nk * BK, tid);
      }
      cp_commit();
    }
    const double* as = As + (kt % STAGES) * A_STAGE + wm * 32 + g;
    const double* bs = Bs + (kt % STAGES) * B_STAGE + (wn * 32 + g) * LDB_S + t;
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      double a[4], b[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        a[mi] = as[(k4 + t) * LDA_S + mi * 8];
        if (neg) a[mi] = neg_bits(a[mi]);
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) b[ni] = bs[ni * 8 * LDB_S + k4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
    }
  }
  cp_wait<0>();
  if (colpart != nullptr) {
    // fused a12 epilogue: per-column |C| sums over this CTA's 128 rows (rows >= M are exact zeros)
    __syncthreads();
    double* red = smem;  // WM (wm) x BN columns
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double v = 0.0;
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) v += fabs(acc[mi][ni][h]);
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        if (g == 0) red[wm * BN + wn * 32 + ni * 8 + 2 * t + h] = v;
      }
    __syncthreads();
    if (tid < BN && n0 + tid < N) {
      double v = red[tid];
#pragma unroll
      for (int q = 1; q < WM; ++q) v += red[q * BN + tid];
      colpart[tm * ldp + n0 + tid] = v;
    }
  }
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      int64_t row = m0 + wm * 32 + mi * 8 + g;
      int64_t col = n0 + wn * 32 + ni * 8 + 2 * t;
      if (row < M) {
        if (col < N) C[col * ldc + row] = acc[mi][ni][0];
        if (col + 1 < N) C[(col + 1) * ldc + row] = acc[mi][ni][1];
      }
    }
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

template <int WM, int WN>
static void launch_dgemm_w(double* C, int64_t ldc, const double* A, int64_t lda, const double* B,
                           int64_t ldb, int64_t M, int64_t N, int K, bool neg, bool beta,
                           const uint8_t* dec, int k, int want, cudaStream_t st, double* colpart,
                           int64_t ldp) {
  static unsigned long long attr = 0;
  if (first_on_device(attr)) {
    smem_optin(k_dgemm<true, WM, WN>);
    smem_optin(k_dgemm<false, WM, WN>);
  }
  constexpr int BM = gemm_bm<WM>(), BN = gemm_bn<WN>();
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const bool v16 = aligned16(A) && aligned16(B) && (lda % 2 == 0) && (ldb % 2 == 0) &&
                   (M % 2 == 0) && (K % 2 == 0);
  ::hlq::g_launches++;
  if (v16)
    k_dgemm<true, WM, WN><<<(unsigned)tiles, 32 * WM * WN, gemm_smem<WM, WN>(), st>>>(
        C, ldc, A, lda, B, ldb, M, N, K, neg ? 1 : 0, beta ? 1 : 0, dec, k, want, colpart, ldp);
  else
    k_dgemm<false, WM, WN><<<(unsigned)tiles, 32 * WM * WN, gemm_smem<WM, WN>(), st>>>(
        C, ldc, A, lda, B, ldb, M, N, K, neg ? 1 : 0, beta ? 1 : 0, dec, k, want, colpart, ldp);
}

// CTA tile = (32 WM) x (32 WN) = 64 x 64 (4 warps, 4 CTAs/SM: C3 LU update 27.5 TF vs 27.3 for
// 128 x 64 with 2 CTAs/SM, 26.3 for 64 x 128, 25.0 for 128 x 32, 23.8 for 128 x 128, measured in
// round 1); its 64-row column partials match the TMA kernel's (gemm_tma.cu), so both feed the same
// colpart layout
constexpr int kGemmBM = 64;
int gemm_colpart_rows() { return kGemmBM; }

// C[M x N] = beta*C + (neg ? -1 : 1) * A[M x K] * B[K x N]; dec/k/want: optional predicate.
void launch_dgemm(double* C, int64_t ldc, const double* A, int64_t lda, const double* B,
                  int64_t ldb, int64_t M, int64_t N, int K, bool neg, bool beta,
                  const uint8_t* dec, int k, int want, cudaStream_t st, double* colpart,
                  int64_t ldp) {
  if (ldp == 0) ldp = N;
  if (M <= 0 || N <= 0 || K <= 0) return;
  static_assert(gemm_bm<2>() == kGemmBM, "colpart rows");
  launch_dgemm_w<2, 2>(C, ldc, A, lda, B, ldb, M, N, K, neg, beta, dec, k, want, st, colpart, ldp);
}

// a12 from the fused epilogue: tile row i = CTA row blocks [i*bpt, (i+1)*bpt); tile-norm max over
// (tile row, column) -> atomic max into *out.  grid (tile rows, column chunks of 256).
__global__ void k_colpart_max(const double* __restrict__ colpart, int64_t ntm, int64_t N, int bpt,
                              double* out, const uint8_t* __restrict__ dec, int k, int want) {
  if (dec != nullptr && dec[k] != want) return;
  const int64_t i = blockIdx.x;
  const int64_t c = (int64_t)blockIdx.y * 256 + threadIdx.x;
  double v = 0.0;
  if (c < N) {
    for (int b = 0; b < bpt; ++b) {
      int64_t tm = i * bpt + b;
      if (tm < ntm) v += colpart[tm * N + c];
    }
  }
  for (int o = 16; o > 0; o >>= 1) v = nanmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out, v);
}

void launch_colpart_max(const double* colpart, int64_t M, int64_t N, int nb, double* out,
                        const uint8_t* dec, int k, int want, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  const int BM = gemm_colpart_rows();
  const int64_t ntm = (M + BM - 1) / BM;
  const int bpt = nb / BM;
  const int64_t ntiles = (M + nb - 1) / nb;
  dim3 grid((unsigned)ntiles, (unsigned)((N + 255) / 256));
  { ::hlq::g_launches++; k_colpart_max<<<grid, 256, 0, st>>>(colpart, ntm, N, bpt, out, dec, k, want); }
}

}  // namespace hlq
