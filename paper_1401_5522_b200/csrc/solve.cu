// a13: solve by a second pass over b ("apply the transformations on b during a
// second pass") followed by the N x N block back substitution.  HBM-bound: every factor
// element is read once (the GEMV kernels are coalesced down the columns of the LAPACK layout).
// Also: the HPL3 residual pieces ||Ax-b||_inf, ||A||_inf, ||x||_inf and the final
// status scan (non-finite factors, exact zeros on the U/R diagonal).
#include <math.h>

#include "hlq_internal.cuh"

namespace hlq {

// LU step k forward: x_k <- L_kk^-1 P_kk x_k (one warp)
__global__ void k_solve_lu_diag(const double* __restrict__ A, Geo g, int k,
                                const int* __restrict__ ipiv, double* __restrict__ x) {
  const int bk = g.bs(k);
  const int lane = threadIdx.x;
  const double* Akk = g.tile(const_cast<double*>(A), k, k);
  double* xk = x + g.r0(k);
  if (lane == 0) {
    for (int c = 0; c < bk; ++c) {
      int p = ipiv[(int64_t)k * g.nb + c];
      if (p != c) {
        double t = xk[c];
        xk[c] = xk[p];
        xk[p] = t;
      }
    }
  }
  __syncwarp();
  for (int c = 0; c < bk; ++c) {
    double xc = xk[c];
    __syncwarp();
    for (int r = c + 1 + lane; r < bk; r += 32) xk[r] -= Akk[(int64_t)c * g.lda + r] * xc;
    __syncwarp();
  }
}

// back substitution on the diagonal tile: x_k <- U_kk^-1 x_k (one warp)
__global__ void k_solve_upper_diag(const double* __restrict__ A, Geo g, int k,
                                   double* __restrict__ x) {
  const int bk = g.bs(k);
  const int lane = threadIdx.x;
  const double* Akk = g.tile(const_cast<double*>(A), k, k);
  double* xk = x + g.r0(k);
  for (int c = bk - 1; c >= 0; --c) {
    double xc = xk[c] / Akk[(int64_t)c * g.lda + c];
    __syncwarp();
    if (lane == 0) xk[c] = xc;
    for (int r = lane; r < c; r += 32) xk[r] -= Akk[(int64_t)c * g.lda + r] * xc;
    __syncwarp();
  }
}

// y[0:M) -= B[0:M, 0:K) * v[0:K)   (B column-major, ldb): one thread per row
__global__ void k_gemv_sub(double* __restrict__ y, const double* __restrict__ B, int64_t ldb,
                           int64_t M, int K, const double* __restrict__ v) {
  extern __shared__ double vs[];
  for (int c = threadIdx.x; c < K; c += blockDim.x) vs[c] = v[c];
  __syncthreads();
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= M) return;
  double acc = 0.0;
  for (int c = 0; c < K; ++c) acc += B[(int64_t)c * ldb + r] * vs[c];
  y[r] -= acc;
}

void launch_gemv_sub(double* y, const double* B, int64_t ldb, int64_t M, int K, const double* v,
                     cudaStream_t st) {
  if (M <= 0 || K <= 0) return;
  { ::hlq::g_launches++; k_gemv_sub<<<(unsigned)((M + 255) / 256), 256, sizeof(double) * K, st>>>(y, B, ldb, M, K, v); }
}

void launch_solve_lu_fwd(const double* A, Geo g, int k, const int* ipiv, double* x,
                         cudaStream_t st) {
  { ::hlq::g_launches++; k_solve_lu_diag<<<1, 32, 0, st>>>(A, g, k, ipiv, x); }
  const int64_t k0 = g.r0(k), k1 = k0 + g.bs(k);
  launch_gemv_sub(x + k1, A + k0 * g.lda + k1, g.lda, g.N - k1, g.bs(k), x + k0, st);
}

void launch_solve_back(const double* A, Geo g, int k, double* x, cudaStream_t st) {
  { ::hlq::g_launches++; k_solve_upper_diag<<<1, 32, 0, st>>>(A, g, k, x); }
  const int64_t k0 = g.r0(k);
  launch_gemv_sub(x, A + k0 * g.lda, g.lda, k0, g.bs(k), x + k0, st);
}

// ---------------------------------------------------------------------------------------------
// HPL3 pieces: out[0] = ||A x - b||_inf, out[1] = ||A||_inf, out[2] = ||x||_inf (atomic max >= 0)
__global__ void k_residual(const double* __restrict__ A, int64_t N, int64_t lda,
                           const double* __restrict__ x, const double* __restrict__ b,
                           double* out) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
  double acc = 0.0, rs = 0.0;
  for (int64_t c = 0; c < N; ++c) {
    double a = A[c * lda + r];
    acc += a * x[c];
    rs += fabs(a);
  }
  atomic_max_nonneg(&out[0], fabs(acc - b[r]));
  atomic_max_nonneg(&out[1], rs);
  atomic_max_nonneg(&out[2], fabs(x[r]));
}

void launch_residual(const double* A, int64_t N, int64_t lda, const double* x, const double* b,
                     double* out3dev, cudaStream_t st) {
  cudaMemsetAsync(out3dev, 0, 3 * sizeof(double), st);
  { ::hlq::g_launches++; k_residual<<<(unsigned)((N + 127) / 128), 128, 0, st>>>(A, N, lda, x, b, out3dev); }
}

// final status: flag[0] |= any non-finite factor entry, flag[1] |= exact zero on the diagonal
__global__ void k_final_scan(const double* __restrict__ A, int64_t N, int64_t lda, int* flag) {
  int bad = 0, zero = 0;
  int64_t total = N * N;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = t / N, r = t - c * N;
    double a = A[c * lda + r];
    if (!isfinite(a)) bad = 1;
    if (r == c && a == 0.0) zero = 1;
  }
  bad = __syncthreads_or(bad);
  zero = __syncthreads_or(zero);
  if (threadIdx.x == 0) {
    if (bad) atomicOr(&flag[0], 1);
    if (zero) atomicOr(&flag[1], 1);
  }
}

void launch_final_scan(const double* A, int64_t N, int64_t lda, int* flag, cudaStream_t st) {
  cudaMemsetAsync(flag, 0, 2 * sizeof(int), st);
  { ::hlq::g_launches++; k_final_scan<<<148 * 8, 256, 0, st>>>(A, N, lda, flag); }
}

}  // namespace hlq
