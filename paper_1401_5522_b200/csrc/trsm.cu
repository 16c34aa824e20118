// a5 / a6: the LU step's two triangular solves, as blocked substitution on the FP64 tensor cores.
//   Eliminate (Alg. 2):  A_ik <- A_ik U_kk^-1 for all i > k   (right, upper, non-unit)
//   Apply     (Alg. 2):  A_kj <- L_kk^-1 P_kk A_kj for j > k   (left, unit lower)
// Both are written as ONE kernel solving T Z = B for a Z of (tile rows) x 32 per CTA:
//   Eliminate: Z = X^T (32 rows of the panel below the diagonal tile), T = U_kk^T (lower, non-unit);
//   Apply:     Z = 32 columns of row block k (rows gathered through P_kk), T = L_kk (unit lower).
// T (from the speculative LU W, ld nb) is cut into 32 x 32 chunks; for every 32-row block jb of Z
// the off-diagonal chunks update it on DMMA (Z[jb] -= T[jb, kb] Z[kb], kb < jb, left-looking),
// then the diagonal chunk is solved by substitution (division by the pivot for Eliminate).  This
// is the standard blocked triangular solve: backward stable, unlike multiplying by an explicit
// triangular inverse, whose error grows with kappa(U_kk) -- exactly the ill-conditioned diagonal
// tiles that pivoting inside the tile produces ("Triangular solves").
//   Shared memory: Z (tile rows x 32, layout chosen so the DMMA B fragments are conflict free) and a
//   cp.async double buffer of T chunks.  4 warps, each a 16 x 16 quadrant of the 32 x 32 update.
#include "hlq_internal.cuh"

namespace hlq {

namespace {
constexpr int TR_T = 128;   // threads per CTA
constexpr int SJ_E = 40;    // Eliminate: Zs[j * 40 + c]  (== 8 mod 16: conflict-free B fragments)
constexpr int LDT_E = 36;   // Eliminate T chunk: Ts[j * 36 + i]   (A fragments: == 4 mod 16)
constexpr int LDT_A = 40;   // Apply T chunk:     Ts[i * 40 + j]   (A fragments: == 8 mod 16)
constexpr int TCH = 32 * 40;  // doubles per T chunk buffer

__device__ __forceinline__ void dmma_t(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cpa8z(void* s, const void* g, bool valid) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(sz));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cpa_wait0() { asm volatile("cp.async.wait_group 0;\n" ::); }

__host__ __device__ inline int rup32(int x) { return (x + 31) / 32 * 32; }
}  // namespace

// Z index of (tile row j, owned column c)
template <bool ELIM>
__device__ __forceinline__ int zidx(int j, int c, int ldz) {
  return ELIM ? j * SJ_E + c : c * ldz + j;
}
// T chunk index of (row j, column i) within a 32 x 32 chunk
template <bool ELIM>
__device__ __forceinline__ int tidx(int j, int i) {
  return ELIM ? j * LDT_E + i : i * LDT_A + j;
}

// T chunk (jb, kb) -> Ts: T(j, i) = U(i, j) = W[j*ldw + i] (Eliminate) or L(j, i) = W[i*ldw + j]
// (Apply); entries outside the bk x bk tile are zero
template <bool ELIM>
__device__ __forceinline__ void load_tchunk(double* Ts, const double* W, int ldw, int bk, int jb,
                                            int kb, int tid) {
  const int j0 = jb * 32, i0 = kb * 32;
  for (int o = tid; o < 1024; o += TR_T) {
    // consecutive threads walk the global-contiguous index
    const int a = o >> 5, b = o & 31;  // a: outer, b: inner (contiguous in W)
    const int j = ELIM ? a : b, i = ELIM ? b : a;
    const bool ok = (j0 + j < bk) && (i0 + i < bk);
    const double* src = ELIM ? W + (int64_t)(j0 + j) * ldw + i0 + i : W + (int64_t)(i0 + i) * ldw + j0 + j;
    cpa8z(Ts + tidx<ELIM>(j, i), ok ? src : W, ok);
  }
}

template <bool ELIM>
__global__ void __launch_bounds__(TR_T) k_trsm(double* __restrict__ A, int64_t lda, int64_t rowA,
                                               int64_t colA, int64_t nz, int bk,
                                               const double* __restrict__ W, int ldw,
                                               const int* __restrict__ perm,
                                               const uint8_t* __restrict__ dec, int k, int want) {
  if (dec != nullptr && dec[k] != want) return;  // predicated launch (the branch not taken exits)
  extern __shared__ __align__(16) double sm[];
  const int BK32 = rup32(bk);
  const int ldz = BK32 + 4;  // Apply: == 4 mod 16
  double* Zs = sm;
  double* Ts = sm + (ELIM ? BK32 * SJ_E : 32 * ldz);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t cz0 = (int64_t)blockIdx.x * 32;
  const int ncv = (int)min((int64_t)32, nz - cz0);

  // ---- Z <- B (zero outside the tile rows / owned columns); Apply gathers rows through P_kk
  for (int o = tid; o < BK32 * 32; o += TR_T) {
    int j, c;
    if (ELIM) { j = o >> 5; c = o & 31; }       // contiguous in c = panel rows
    else { c = o / BK32; j = o - c * BK32; }    // contiguous in j = tile rows
    const bool ok = (j < bk) && (c < ncv);
    const double* src = ELIM ? A + (colA + j) * lda + rowA + cz0 + c
                             : A + (colA + cz0 + c) * lda + rowA + (ok ? perm[j] : 0);
    cpa8z(Zs + zidx<ELIM>(j, c, ldz), ok ? src : A, ok);
  }
  const int NBK = BK32 / 32;
  const int S = NBK * (NBK + 1) / 2;  // chunks (jb, kb), kb = 0..jb
  load_tchunk<ELIM>(Ts, W, ldw, bk, 0, 0, tid);
  cpa_commit();

  const int wm = warp & 1, wn = warp >> 1;  // 16 x 16 quadrant of the 32 x 32 block update
  int s = 0, jb = 0, kb = 0;
  double acc[2][2][2];
  for (; s < S; ++s) {
    cpa_wait0();
    __syncthreads();  // chunk s (and Z) landed; every warp is done with the other buffer
    {
      int nj = jb, nk = kb + 1;
      if (nk > nj) { ++nj; nk = 0; }
      if (s + 1 < S) load_tchunk<ELIM>(Ts + ((s + 1) & 1) * TCH, W, ldw, bk, nj, nk, tid);
      cpa_commit();
    }
    const double* T = Ts + (s & 1) * TCH;
    if (kb < jb) {
      if (kb == 0) {  // first update of block jb: accumulators <- Z[jb]
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int ni = 0; ni < 2; ++ni)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              acc[mi][ni][h] = Zs[zidx<ELIM>(jb * 32 + wm * 16 + mi * 8 + g,
                                             wn * 16 + ni * 8 + 2 * t + h, ldz)];
      }
      // Z[jb] -= T[jb, kb] Z[kb]
#pragma unroll
      for (int kk = 0; kk < 32; kk += 4) {
        double a[2], b[2];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) a[mi] = neg_bits(T[tidx<ELIM>(wm * 16 + mi * 8 + g, kk + t)]);
#pragma unroll
        for (int ni = 0; ni < 2; ++ni)
          b[ni] = Zs[zidx<ELIM>(kb * 32 + kk + t, wn * 16 + ni * 8 + g, ldz)];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) dmma_t(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
      }
      if (kb + 1 == jb) {  // block jb fully updated: accumulators -> Z[jb]
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int ni = 0; ni < 2; ++ni)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              Zs[zidx<ELIM>(jb * 32 + wm * 16 + mi * 8 + g, wn * 16 + ni * 8 + 2 * t + h, ldz)] =
                  acc[mi][ni][h];
      }
      ++kb;
    } else {
      // diagonal chunk: substitution on Z[jb], lane = owned column (warp 0)
      __syncthreads();  // the accumulators of every warp are in Z[jb]
      if (warp == 0) {
        double z[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) z[j] = Zs[zidx<ELIM>(jb * 32 + j, lane, ldz)];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          if (ELIM) {
            const double d = (jb * 32 + i < bk) ? T[tidx<ELIM>(i, i)] : 1.0;
            z[i] = z[i] / d;
          }
#pragma unroll
          for (int j = i + 1; j < 32; ++j) z[j] = fma(neg_bits(T[tidx<ELIM>(j, i)]), z[i], z[j]);
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) Zs[zidx<ELIM>(jb * 32 + j, lane, ldz)] = z[j];
      }
      ++jb;
      kb = 0;
    }
  }
  __syncthreads();
  // ---- Z -> A (in place; Apply writes the rows in their permuted order)
  for (int o = tid; o < BK32 * 32; o += TR_T) {
    int j, c;
    if (ELIM) { j = o >> 5; c = o & 31; }
    else { c = o / BK32; j = o - c * BK32; }
    if (j < bk && c < ncv) {
      double* dst = ELIM ? A + (colA + j) * lda + rowA + cz0 + c : A + (colA + cz0 + c) * lda + rowA + j;
      *dst = Zs[zidx<ELIM>(j, c, ldz)];
    }
  }
}

static size_t trsm_smem(bool elim, int bk) {
  const int BK32 = rup32(bk);
  return sizeof(double) * ((elim ? (size_t)BK32 * SJ_E : (size_t)32 * (BK32 + 4)) + 2 * TCH);
}

// Eliminate: A[r0 : r0+M, c0 : c0+bk] <- A[...] U^-1, U = the upper triangle of W (ld ldw)
void launch_trsm_eliminate(double* A, int64_t lda, int64_t r0, int64_t c0, int64_t M, int bk,
                           const double* W, int ldw, const uint8_t* dec, int k, int want,
                           cudaStream_t st) {
  if (M <= 0 || bk <= 0) return;
  static unsigned long long attr = 0;
  if (first_on_device(attr)) smem_optin(k_trsm<true>);
  ::hlq::g_launches++;
  k_trsm<true><<<(unsigned)((M + 31) / 32), TR_T, trsm_smem(true, bk), st>>>(
      A, lda, r0, c0, M, bk, W, ldw, nullptr, dec, k, want);
}

// Apply: A[r0 : r0+bk, c0 : c0+nc] <- L^-1 P A[...], L = the unit lower triangle of W (ld ldw),
// P: row r of the result is row perm[r] of the input
void launch_trsm_apply(double* A, int64_t lda, int64_t r0, int64_t c0, int64_t nc, int bk,
                       const double* W, int ldw, const int* perm, const uint8_t* dec, int k,
                       int want, cudaStream_t st) {
  if (nc <= 0 || bk <= 0) return;
  static unsigned long long attr = 0;
  if (first_on_device(attr)) smem_optin(k_trsm<false>);
  ::hlq::g_launches++;
  k_trsm<false><<<(unsigned)((nc + 31) / 32), TR_T, trsm_smem(false, bk), st>>>(
      A, lda, r0, c0, nc, bk, W, ldw, perm, dec, k, want);
}

}  // namespace hlq
