// a2: speculative GETRF of the diagonal tile, pivoting local to the tile (Alg. 2),
//     out of place into the workspace W (the paper's "Backup Panel" P:634-640 becomes unnecessary:
//     a QR decision simply discards W).
// a3: explicit triangular inverses L^-1, U^-1 of W and ||A_kk^-1||_1 = ||U^-1 L^-1||_1 exactly
//     (reading 3).  The inverses are reused by the LU step: TRSM and SWPTRSM
//     become DMMA GEMMs with U^-1 and L^-1 (gemm.cu).
//
// GETRF is blocked right-looking with 32-column panels held in shared memory, ONE CTA.  Every
// element update is a separately rounded multiply and subtract applied in column order (the
// __dmul_rn/__dsub_rn intrinsics forbid FMA contraction), and the pivot is the first maximum of
// |column|, so W and ipiv are bit-identical to the unblocked elimination order of the oracle.
#include <math.h>

#include "hlq_internal.cuh"

namespace hlq {

constexpr int GPW = 32;       // panel width

// pivot order of numpy argmax(|x|): NaN beats everything, then larger value, then smaller index
__device__ __forceinline__ bool piv_better(double v, int i, double bv, int bi) {
  bool vn = v != v, bn = bv != bv;
  if (vn != bn) return vn;
  if (!vn && v != bv) return v > bv;
  return i < bi;
}
constexpr int GT = 512;       // threads

// smem: panel P[GPW][ldp] + U12 block U[GPW][ldu]
__global__ void __launch_bounds__(GT) k_getrf(const double* __restrict__ A, Geo g, int k,
                                              double* __restrict__ W, int* __restrict__ ipiv,
                                              int* __restrict__ zp_out) {
  extern __shared__ double sm[];
  const int bk = g.bs(k);
  const int ldw = g.nb;
  const int ldp = g.nb + 1;  // odd stride: conflict-free column-per-thread access
  double* P = sm;                    // GPW x ldp
  double* U = sm + GPW * ldp;        // GPW x ldp  (row c of U12 for trailing column j at U[c*ldp + j])
  __shared__ double rv[GT / 32];
  __shared__ int ri[GT / 32];
  __shared__ int piv_sh[GPW];
  __shared__ int zp_sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* Akk = g.tile(const_cast<double*>(A), k, k);
  for (int idx = tid; idx < bk * bk; idx += GT) {
    int c = idx / bk, r = idx - c * bk;
    W[(int64_t)c * ldw + r] = Akk[(int64_t)c * g.lda + r];
  }
  if (tid == 0) zp_sh = 0;
  __syncthreads();
  for (int p0 = 0; p0 < bk; p0 += GPW) {
    const int pw = min(GPW, bk - p0);
    const int rows = bk - p0;
    for (int idx = tid; idx < pw * rows; idx += GT) {
      int c = idx / rows, r = idx - c * rows;
      P[c * ldp + r] = W[(int64_t)(p0 + c) * ldw + p0 + r];
    }
    __syncthreads();
    for (int c = 0; c < pw; ++c) {
      // first maximum of |P[c][r]|, r in [c, rows)
      double best = -1.0;
      int bidx = 0x7fffffff;
      for (int r = c + tid; r < rows; r += GT) {
        double v = fabs(P[c * ldp + r]);
        if (piv_better(v, r, best, bidx)) {
          best = v;
          bidx = r;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, best, o);
        int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
        if (piv_better(ov, oi, best, bidx)) {
          best = ov;
          bidx = oi;
        }
      }
      if (lane == 0) {
        rv[warp] = best;
        ri[warp] = bidx;
      }
      __syncthreads();
      if (tid == 0) {
        double b = rv[0];
        int bi = ri[0];
        for (int w = 1; w < GT / 32; ++w)
          if (piv_better(rv[w], ri[w], b, bi)) {
            b = rv[w];
            bi = ri[w];
          }
        if (bi == 0x7fffffff || bi >= rows) bi = c;
        piv_sh[c] = bi;
        ipiv[p0 + c] = p0 + bi;
      }
      __syncthreads();
      const int pr = piv_sh[c];
      if (pr != c && tid < pw) {
        double t = P[tid * ldp + c];
        P[tid * ldp + c] = P[tid * ldp + pr];
        P[tid * ldp + pr] = t;
      }
      __syncthreads();
      const double d = P[c * ldp + c];
      if (d == 0.0) {
        if (tid == 0) zp_sh = 1;
        __syncthreads();
        continue;  // ledger 7: column left unscaled, no update
      }
      for (int r = c + 1 + tid; r < rows; r += GT) P[c * ldp + r] = P[c * ldp + r] / d;
      __syncthreads();
      // rank-1 update inside the panel: P[j][r] -= P[c][r] * P[j][c]
      const int nr = rows - c - 1, nj = pw - c - 1;
      for (int idx = tid; idx < nr * nj; idx += GT) {
        int j = c + 1 + idx / nr, r = c + 1 + idx % nr;
        P[j * ldp + r] = __dsub_rn(P[j * ldp + r], __dmul_rn(P[c * ldp + r], P[j * ldp + c]));
      }
      __syncthreads();
    }
    // write the panel back
    for (int idx = tid; idx < pw * rows; idx += GT) {
      int c = idx / rows, r = idx - c * rows;
      W[(int64_t)(p0 + c) * ldw + p0 + r] = P[c * ldp + r];
    }
    // apply the panel's swaps to every other column of the tile (left and right), in order:
    // one warp per column, the column segment rows [p0, bk) staged in the warp's smem buffer
    {
      const int nother = bk - pw;
      double* cb = sm + 2 * GPW * ldp + warp * ldp;
      for (int t = warp; t < nother; t += GT / 32) {
        int col = (t < p0) ? t : t + pw;
        double* wc = W + (int64_t)col * ldw + p0;
        for (int r = lane; r < rows; r += 32) cb[r] = wc[r];
        __syncwarp();
        if (lane == 0)
          for (int c = 0; c < pw; ++c) {
            int pr = piv_sh[c];
            if (pr != c) {
              double x = cb[c];
              cb[c] = cb[pr];
              cb[pr] = x;
            }
          }
        __syncwarp();
        for (int r = lane; r < rows; r += 32) wc[r] = cb[r];
        __syncwarp();
      }
    }
    __syncthreads();
    const int ntr = bk - p0 - pw;  // trailing columns
    if (ntr > 0) {
      // U12 = L11^-1 A12: forward substitution per column in elimination order
      for (int t = tid; t < ntr; t += GT) {
        int col = p0 + pw + t;
        double* wc = W + (int64_t)col * ldw + p0;
        for (int c = 0; c < pw; ++c) {
          double x = wc[c];
          for (int l = 0; l < c; ++l) x = __dsub_rn(x, __dmul_rn(P[l * ldp + c], U[l * ldp + t]));
          U[c * ldp + t] = x;
          wc[c] = x;
        }
      }
      __syncthreads();
      // trailing update: W[p0+pw+r][col] -= sum_c L21[r][c] U12[c][col], sequential in c.
      // 64 x 128 output blocks, 4 x 4 per thread (rows tr + 16 i, cols tc + 32 j): 8 shared loads
      // per 16 separately-rounded multiply/subtract pairs.
      const int nr = rows - pw;
      const int tr = tid & 15, tc = tid >> 4;
      for (int rb = 0; rb < nr; rb += 64)
        for (int cb0 = 0; cb0 < ntr; cb0 += 128) {
          double acc[4][4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              int r = rb + tr + 16 * i, t = cb0 + tc + 32 * j;
              acc[i][j] = (r < nr && t < ntr) ? W[(int64_t)(p0 + pw + t) * ldw + p0 + pw + r] : 0.0;
            }
          for (int c = 0; c < pw; ++c) {
            double l[4], u[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              int r = rb + tr + 16 * i;
              l[i] = (r < nr) ? P[c * ldp + pw + r] : 0.0;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              int t = cb0 + tc + 32 * j;
              u[j] = (t < ntr) ? U[c * ldp + t] : 0.0;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j) acc[i][j] = __dsub_rn(acc[i][j], __dmul_rn(l[i], u[j]));
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              int r = rb + tr + 16 * i, t = cb0 + tc + 32 * j;
              if (r < nr && t < ntr) W[(int64_t)(p0 + pw + t) * ldw + p0 + pw + r] = acc[i][j];
            }
        }
    }
    __syncthreads();
  }
  if (tid == 0) zp_out[0] = zp_sh;
}

void launch_getrf(const double* A, Geo g, int k, DevWork w, bool need, cudaStream_t st) {
  if (!need) return;
  size_t smem = sizeof(double) * (2 * GPW + GT / 32) * (g.nb + 1);
  static bool attr = false;
  if (!attr) {
    smem_optin(k_getrf);
    attr = true;
  }
  { ::hlq::g_launches++; k_getrf<<<1, GT, smem, st>>>(A, g, k, w.W, w.ipiv_ws, w.zp); }
}

// ---------------------------------------------------------------------------------------------
// Triangular inverses of the speculative LU: Li = L^-1 (unit lower), Ui = U^-1 (upper), ld = nb.
// One warp per column j: blockIdx.y = 0 -> Li, 1 -> Ui.  Column j of L^-1 solves L y = e_j
// (forward, rows >= j); column j of U^-1 solves U x = e_j (backward, rows <= j).
__global__ void __launch_bounds__(256) k_tri_inv(const double* __restrict__ W, int bk, int ldw,
                                                 double* __restrict__ Li, double* __restrict__ Ui) {
  extern __shared__ double ys[];  // 8 warps x bk
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * 8 + warp;
  if (j >= bk) return;
  double* y = ys + warp * bk;
  for (int r = lane; r < bk; r += 32) y[r] = (r == j) ? 1.0 : 0.0;
  __syncwarp();
  if (blockIdx.y == 0) {
    for (int c = j; c < bk; ++c) {
      double yc = y[c];
      __syncwarp();
      if (yc != 0.0)
        for (int r = c + 1 + lane; r < bk; r += 32) y[r] -= W[(int64_t)c * ldw + r] * yc;
      __syncwarp();
    }
    for (int r = lane; r < bk; r += 32) Li[(int64_t)j * ldw + r] = y[r];
  } else {
    for (int c = j; c >= 0; --c) {
      double xc = y[c] / W[(int64_t)c * ldw + c];
      __syncwarp();
      if (lane == 0) y[c] = xc;
      for (int r = lane; r < c; r += 32) y[r] -= W[(int64_t)c * ldw + r] * xc;
      __syncwarp();
    }
    for (int r = lane; r < bk; r += 32) Ui[(int64_t)j * ldw + r] = y[r];
  }
}

// ||U^-1 L^-1||_1: warp per column j of X = Ui * Li; column abs-sum; atomic max.
__global__ void __launch_bounds__(256) k_invnorm(const double* __restrict__ Li,
                                                 const double* __restrict__ Ui, int bk, int ldw,
                                                 double* inv_norm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * 8 + warp;
  if (j >= bk) return;
  const double* lj = Li + (int64_t)j * ldw;
  double colsum = 0.0;
  for (int r = lane; r < bk; r += 32) {
    double x = 0.0;
    for (int c = (r > j ? r : j); c < bk; ++c) x += Ui[(int64_t)c * ldw + r] * lj[c];
    colsum += fabs(x);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) colsum += __shfl_xor_sync(0xffffffffu, colsum, o);
  if (lane == 0) atomic_max_nonneg(inv_norm, colsum);
}

// NEXT f3: the Hager / Higham estimate of ||U^-1 L^-1||_1 in the order of LAPACK
// dlacn2 (the oracle's inv_norm1_estimate), one CTA.  B x = Ui (Li x) and B^T v = Li^T (Ui^T v) are
// triangular GEMVs with the explicit inverses of k_tri_inv; sums and the first-max argmax are CTA
// reductions in a fixed order.
__device__ double est_asum(const double* y, int n, double* red) {
  const int tid = threadIdx.x;
  double s = 0.0;
  for (int r = tid; r < n; r += 256) s += fabs(y[r]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __syncthreads();
  if ((tid & 31) == 0) red[tid >> 5] = s;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < 8; ++w) t += red[w];
  __syncthreads();
  return t;
}
__device__ int est_argmax(const double* z, int n, double* redv, int* redi) {
  const int tid = threadIdx.x;
  double bv = -1.0;
  int bi = 0x7fffffff;
  for (int r = tid; r < n; r += 256) {
    const double v = fabs(z[r]);
    if (v > bv) {
      bv = v;
      bi = r;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  __syncthreads();
  if ((tid & 31) == 0) {
    redv[tid >> 5] = bv;
    redi[tid >> 5] = bi;
  }
  __syncthreads();
  double v = redv[0];
  int i = redi[0];
  for (int w = 1; w < 8; ++w)
    if (redv[w] > v || (redv[w] == v && redi[w] < i)) {
      v = redv[w];
      i = redi[w];
    }
  __syncthreads();
  return i;
}

__global__ void __launch_bounds__(256) k_invnorm_est(const double* __restrict__ Li,
                                                     const double* __restrict__ Ui, int n, int ld,
                                                     double* out) {
  __shared__ double x[512], t[512], y[512], xi[512];
  __shared__ double red[8];
  __shared__ int redi[8];
  __shared__ int s_diff;
  const int tid = threadIdx.x;
  auto Bx = [&](const double* v, double* o) {  // o = Ui (Li v)
    for (int r = tid; r < n; r += 256) {
      double a = 0.0;
      for (int c = 0; c <= r; ++c) a += Li[(int64_t)c * ld + r] * v[c];
      t[r] = a;
    }
    __syncthreads();
    for (int r = tid; r < n; r += 256) {
      double a = 0.0;
      for (int c = r; c < n; ++c) a += Ui[(int64_t)c * ld + r] * t[c];
      o[r] = a;
    }
    __syncthreads();
  };
  auto BTx = [&](const double* v, double* o) {  // o = Li^T (Ui^T v)
    for (int r = tid; r < n; r += 256) {
      double a = 0.0;
      for (int c = 0; c <= r; ++c) a += Ui[(int64_t)r * ld + c] * v[c];
      t[r] = a;
    }
    __syncthreads();
    for (int r = tid; r < n; r += 256) {
      double a = 0.0;
      for (int c = r; c < n; ++c) a += Li[(int64_t)r * ld + c] * t[c];
      o[r] = a;
    }
    __syncthreads();
  };
  for (int r = tid; r < n; r += 256) x[r] = 1.0 / (double)n;
  __syncthreads();
  Bx(x, y);
  if (n == 1) {
    if (tid == 0) out[0] = fabs(y[0]);
    return;
  }
  double est = est_asum(y, n, red);
  for (int r = tid; r < n; r += 256) xi[r] = y[r] >= 0.0 ? 1.0 : -1.0;
  __syncthreads();
  BTx(xi, x);  // z in x
  int j = est_argmax(x, n, red, redi);
  for (int it = 2;; ) {
    for (int r = tid; r < n; r += 256) x[r] = (r == j) ? 1.0 : 0.0;
    __syncthreads();
    Bx(x, y);
    const double est_old = est;
    est = est_asum(y, n, red);
    if (tid == 0) s_diff = 0;
    __syncthreads();
    for (int r = tid; r < n; r += 256)
      if ((y[r] >= 0.0 ? 1.0 : -1.0) != xi[r]) s_diff = 1;
    __syncthreads();
    if (!s_diff || est <= est_old) break;
    for (int r = tid; r < n; r += 256) xi[r] = y[r] >= 0.0 ? 1.0 : -1.0;
    __syncthreads();
    BTx(xi, x);
    const int jl = j;
    j = est_argmax(x, n, red, redi);
    if (x[jl] != fabs(x[j]) && it < 5) {
      ++it;
      continue;
    }
    break;
  }
  for (int r = tid; r < n; r += 256)
    x[r] = ((r & 1) ? -1.0 : 1.0) * (1.0 + (double)r / (double)(n - 1));
  __syncthreads();
  Bx(x, y);
  const double tt = 2.0 * (est_asum(y, n, red) / (double)(3 * n));
  if (tid == 0) out[0] = tt > est ? tt : est;
}

void launch_tri_inv(Geo g, int k, const DevWork& w, double* Li, double* Ui, cudaStream_t st) {
  const int bk = g.bs(k);
  dim3 grid((bk + 7) / 8, 2);
  { ::hlq::g_launches++; k_tri_inv<<<grid, 256, sizeof(double) * 8 * bk, st>>>(w.W, bk, g.nb, Li, Ui); }
}

void launch_invnorm(Geo g, int k, DevWork w, cudaStream_t st, int estimate) {
  const int bk = g.bs(k);
  const double* Li = w.scratch;                       // filled by launch_tri_inv
  const double* Ui = w.scratch + (size_t)g.nb * g.nb;
  if (estimate) {
    ::hlq::g_launches++;
    k_invnorm_est<<<1, 256, 0, st>>>(Li, Ui, bk, g.nb, w.inv_norm);
    return;
  }
  cudaMemsetAsync(w.inv_norm, 0, sizeof(double), st);
  { ::hlq::g_launches++; k_invnorm<<<(bk + 7) / 8, 256, 0, st>>>(Li, Ui, bk, g.nb, w.inv_norm); }
}

}  // namespace hlq
