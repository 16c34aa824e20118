// LU step, variant A1 (Alg. 2), predicated on dec[k] == LU:
//   a5  commit: A_kk <- W (the speculative GETRF), ipiv_k stored;      Factor
//       eliminate: A_ik <- A_ik U_kk^-1 for all i > k                  Eliminate
//   a6  apply: A_kj <- L_kk^-1 P_kk A_kj for all j > k                 Apply
//   a7  update: A_ij <- A_ij - A_ik A_kj for all i, j > k              Update
// With the LAPACK layout the i (j) loops are one strided column (row) block, so Eliminate and Apply
// are two blocked triangular solves (trsm.cu: DMMA off-diagonal updates + substitution in 32 x 32
// diagonal blocks) and Update is one rank-b GEMM.  The swaps touch the columns right of the
// diagonal tile only (reading 23).  LU variant A2 applies Q_kk^T (an orthogonal matrix,
// formed explicitly by getrf.cu) with a GEMM.
#include "hlq_internal.cuh"

namespace hlq {

void launch_colpart_max(const double* colpart, int64_t M, int64_t N, int nb, double* out,
                        const uint8_t* dec, int k, int want, cudaStream_t st);

// A_kk <- W, ipiv[k*nb..] <- ipiv_ws, perm[r] = row of (P A_kk) r  (sequential swaps composed)
__global__ void k_lu_commit(double* __restrict__ A, Geo g, int k, const double* __restrict__ W,
                            const int* __restrict__ ipiv_ws, int* __restrict__ ipiv,
                            int* __restrict__ perm, const uint8_t* __restrict__ dec) {
  if (dec[k] != HLQ_DEC_LU) return;
  const int bk = g.bs(k);
  double* Akk = g.tile(A, k, k);
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < bk * bk;
       idx += gridDim.x * blockDim.x) {
    int c = idx / bk, r = idx - c * bk;
    Akk[(int64_t)c * g.lda + r] = W[(int64_t)c * g.nb + r];
  }
  if (blockIdx.x == 0) {
    // the bk sequential swaps composed in shared memory by one thread (the composition is a serial
    // chain of dependent loads: from global memory it was most of this kernel's 51 us)
    __shared__ int sperm[HLQ_MAX_NB], spiv[HLQ_MAX_NB];
    for (int r = threadIdx.x; r < bk; r += blockDim.x) {
      sperm[r] = r;
      spiv[r] = ipiv_ws[r];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int c = 0; c < bk; ++c) {
        const int p = spiv[c];
        const int t = sperm[c];
        sperm[c] = sperm[p];
        sperm[p] = t;
      }
    }
    __syncthreads();
    for (int r = threadIdx.x; r < bk; r += blockDim.x) {
      perm[r] = sperm[r];
      ipiv[(int64_t)k * g.nb + r] = spiv[r];
    }
  }
}

// dst <- src (rows x cols) when dec[k] == want (the speculative QR panel's copy-back)
__global__ void k_copy_block_if(double* __restrict__ dst, int64_t ldd, const double* __restrict__ src,
                                int64_t lds, int64_t rows, int64_t cols,
                                const uint8_t* __restrict__ dec, int k, int want) {
  if (dec[k] != want) return;
  const int64_t total = rows * cols;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t / rows, r = t - c * rows;
    dst[c * ldd + r] = src[c * lds + r];
  }
}

// dst (rows x cols, ld_dst) <- src (ld_src), optionally with rows gathered through perm
__global__ void k_copy_block(double* __restrict__ dst, int64_t ldd, const double* __restrict__ src,
                             int64_t lds, int64_t rows, int64_t cols,
                             const int* __restrict__ perm, const uint8_t* __restrict__ dec, int k) {
  if (dec != nullptr && dec[k] != HLQ_DEC_LU) return;
  int64_t total = rows * cols;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = t / rows, r = t - c * rows;
    int64_t sr = perm ? perm[r] : r;
    dst[c * ldd + r] = src[c * lds + sr];
  }
}

static unsigned grid_for(int64_t total) {
  int64_t b = (total + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)(b < 1 ? 1 : b);
}

void launch_lu_commit(double* A, Geo g, int k, const double* W, const int* ipiv_ws, int* ipiv,
                      int* perm, const uint8_t* dec, cudaStream_t st) {
  ::hlq::g_launches++;
  k_lu_commit<<<8, 256, 0, st>>>(A, g, k, W, ipiv_ws, ipiv, perm, dec);
}

void launch_copy_block_if(double* dst, int64_t ldd, const double* src, int64_t lds, int64_t rows,
                          int64_t cols, const uint8_t* dec, int k, int want, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  ::hlq::g_launches++;
  k_copy_block_if<<<grid_for(rows * cols), 256, 0, st>>>(dst, ldd, src, lds, rows, cols, dec, k,
                                                         want);
}

void launch_copy_block(double* dst, int64_t ldd, const double* src, int64_t lds, int64_t rows,
                       int64_t cols, const int* perm, const uint8_t* dec, int k, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  ::hlq::g_launches++;
  k_copy_block<<<grid_for(rows * cols), 256, 0, st>>>(dst, ldd, src, lds, rows, cols, perm, dec, k);
}

__global__ void k_copy_ints(int* __restrict__ dst, const int* __restrict__ src, int n,
                            const uint8_t* __restrict__ dec, int k) {
  if (dec != nullptr && dec[k] != HLQ_DEC_LU) return;
  for (int t = threadIdx.x; t < n; t += blockDim.x) dst[t] = src[t];
}

void launch_copy_ints(int* dst, const int* src, int n, const uint8_t* dec, int k, cudaStream_t st) {
  if (n <= 0) return;
  ::hlq::g_launches++;
  k_copy_ints<<<1, 256, 0, st>>>(dst, src, n, dec, k);
}

// Panel stage of an LU step (column block k only): Factor (commit W, ipiv) + Eliminate (TRSM).
void launch_lu_panel(double* A, Geo g, int k, const DevWork& w, cudaStream_t st, bool commit) {
  const int bk = g.bs(k);
  const int64_t k0 = g.r0(k), k1 = k0 + bk;
  const int64_t M = g.N - k1;  // rows below the diagonal tile
  const uint8_t* dec = w.dec;
  int* perm = reinterpret_cast<int*>(w.scratch + (size_t)2 * g.nb * g.nb);
  if (commit) { ::hlq::g_launches++; k_lu_commit<<<8, 256, 0, st>>>(A, g, k, w.W, w.ipiv_ws, w.ipiv, perm, dec); }
  if (M <= 0) return;
  // Eliminate: A[k1:N, k0:k1] <- A[k1:N, k0:k1] U^-1 (U: upper triangle of W; A2: R), in place
  launch_trsm_eliminate(A, g.lda, k1, k0, M, bk, w.W, g.nb, dec, k, HLQ_DEC_LU, st);
}

// Update stage of an LU step on the trailing columns [c0, c1) (absolute column indices >= k1):
// Apply (SWPTRSM on row block k) + Update (DGEMM on all trailing rows).  colpart != nullptr fuses
// the a12 column sums into the GEMM epilogue (leading dimension ldp = N - k1, column offset c0-k1).
void launch_lu_update(double* A, Geo g, int k, const DevWork& w, int64_t c0, int64_t c1,
                      double* colpart, cudaStream_t st, bool a2) {
  const int bk = g.bs(k);
  const int64_t k0 = g.r0(k), k1 = k0 + bk;
  const int64_t M = g.N - k1;
  const int64_t nc = c1 - c0;
  if (M <= 0 || nc <= 0) return;
  const uint8_t* dec = w.dec;
  const double* Li = w.scratch;
  const int* perm = reinterpret_cast<const int*>(w.scratch + (size_t)2 * g.nb * g.nb);
  if (a2) {
    // A2 Apply: A[k0:k1, c0:c1] <- Q_kk^T A[k0:k1, c0:c1] (Li slot = Q^T, perm = identity)
    double* ws = w.ws_row + (c0 - k1) * bk;  // disjoint per column range
    { ::hlq::g_launches++; k_copy_block<<<grid_for(nc * bk), 256, 0, st>>>(ws, bk, A + c0 * g.lda + k0, g.lda, bk, nc, perm, dec, k); }
    launch_dgemm(A + c0 * g.lda + k0, g.lda, Li, g.nb, ws, bk, bk, nc, bk, false, false, dec, k,
                 HLQ_DEC_LU, st);
  } else {
    // Apply: A[k0:k1, c0:c1] <- L^-1 P A[k0:k1, c0:c1] (L: unit lower triangle of W), in place
    launch_trsm_apply(A, g.lda, k0, c0, nc, bk, w.W, g.nb, perm, dec, k, HLQ_DEC_LU, st);
  }
  // Update: A[k1:N, c0:c1] -= A[k1:N, k0:k1] * A[k0:k1, c0:c1] (persistent TMA kernel when the
  // matrix is eligible, else the cp.async kernel)
  if (!launch_schur_tma(w.tma_maps, A, g.lda, k0, k1, c0, M, nc, bk, dec, k, HLQ_DEC_LU,
                        colpart ? colpart + (c0 - k1) : nullptr, M, st))
    launch_dgemm(A + c0 * g.lda + k1, g.lda, A + k0 * g.lda + k1, g.lda, A + c0 * g.lda + k0,
                 g.lda, M, nc, bk, true, true, dec, k, HLQ_DEC_LU, st,
                 colpart ? colpart + (c0 - k1) : nullptr, M);
}

void launch_lu_growth(const DevWork& w, Geo g, int k, cudaStream_t st) {
  const int64_t M = g.N - (g.r0(k) + g.bs(k));
  launch_colpart_max(w.colpart, M, M, g.nb, w.gstep + k + 1, w.dec, k, HLQ_DEC_LU, st);
}

}  // namespace hlq
