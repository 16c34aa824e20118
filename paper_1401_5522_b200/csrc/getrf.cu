// a2: speculative GETRF of the diagonal tile, pivoting local to the tile (Alg. 2),
//     out of place into the workspace W (the paper's "Backup Panel" P:634-640 becomes unnecessary:
//     a QR decision simply discards W).
// a3: explicit triangular inverses L^-1, U^-1 of W and ||A_kk^-1||_1 = ||U^-1 L^-1||_1 exactly
//     (reading 3).  The inverses are reused by the LU step: TRSM and SWPTRSM
//     become DMMA GEMMs with U^-1 and L^-1 (gemm.cu).
//
// GETRF is blocked right-looking with 32-column panels, ONE CTA of 512 threads.  Inside a panel
// every thread holds one row in registers (two barriers per column, pivot search by redux.sync);
// the panel's 32 row swaps are applied to the rest of the tile as one gathered permutation, U12
// is a register-blocked forward substitution and the trailing update a 4x4-per-thread blocked
// product from shared memory.  Every
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

// The same order as a 64-bit key: for |v| >= 0 the IEEE bits are monotone, every NaN maps to one
// key above +inf, and the "no candidate" sentinel (-1) maps to 0 with index INT_MAX, which loses
// every tie to a real zero.  A warp reduces (key desc, index asc) with three redux.sync.
__device__ __forceinline__ unsigned long long piv_key(double v) {
  if (v != v) return 0x7ff8000000000000ull;
  return v < 0.0 ? 0ull : (unsigned long long)__double_as_longlong(v);
}
__device__ __forceinline__ void warp_piv_reduce(unsigned long long& key, int& idx) {
  const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  const unsigned mi =
      __reduce_min_sync(0xffffffffu, (hi == mhi && lo == mlo) ? (unsigned)idx : 0x7fffffffu);
  key = ((unsigned long long)mhi << 32) | mlo;
  idx = (int)mi;
}


// W[r][t] -= sum_c L[c][r] * U[c][t] (c sequential, separately rounded), r < nr, t < ntr.
// Blocks of 16 RI x 32 CJ outputs, RI x CJ per thread (rows tr + 16 i, cols tc + 32 j): RI + CJ
// shared loads per RI CJ multiply/subtract pairs.
template <int RI, int CJ>
__device__ __forceinline__ void trail_update(double* __restrict__ Wt, int ldw, const double* L,
                                             const double* U, int ldp, int nr, int ntr, int kc,
                                             int tid) {
  const int tr = tid & 15, tc = tid >> 4;
  for (int rb = 0; rb < nr; rb += 16 * RI)
    for (int cb0 = 0; cb0 < ntr; cb0 += 32 * CJ) {
      double acc[RI][CJ];
#pragma unroll
      for (int i = 0; i < RI; ++i)
#pragma unroll
        for (int j = 0; j < CJ; ++j) {
          const int r = rb + tr + 16 * i, t = cb0 + tc + 32 * j;
          acc[i][j] = (r < nr && t < ntr) ? Wt[(int64_t)t * ldw + r] : 0.0;
        }
      for (int c = 0; c < kc; ++c) {
        double l[RI], u[CJ];
#pragma unroll
        for (int i = 0; i < RI; ++i) {
          const int r = rb + tr + 16 * i;
          l[i] = (r < nr) ? L[c * ldp + r] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < CJ; ++j) {
          const int t = cb0 + tc + 32 * j;
          u[j] = (t < ntr) ? U[c * ldp + t] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < RI; ++i)
#pragma unroll
          for (int j = 0; j < CJ; ++j) acc[i][j] = __dsub_rn(acc[i][j], __dmul_rn(l[i], u[j]));
      }
#pragma unroll
      for (int i = 0; i < RI; ++i)
#pragma unroll
        for (int j = 0; j < CJ; ++j) {
          const int r = rb + tr + 16 * i, t = cb0 + tc + 32 * j;
          if (r < nr && t < ntr) Wt[(int64_t)t * ldw + r] = acc[i][j];
        }
    }
}

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
  __shared__ unsigned long long rv[GT / 32];
  __shared__ int ri[GT / 32];
  __shared__ int piv_sh[GPW];
  __shared__ int zp_sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* Akk = g.tile(const_cast<double*>(A), k, k);
  for (int c0 = warp; c0 < bk; c0 += 4 * (GT / 32)) {  // one warp per column, 4 columns in flight
    double v[4][(HLQ_MAX_NB + 31) / 32];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int i = 0; i < (HLQ_MAX_NB + 31) / 32; ++i) {
        const int c = c0 + q * (GT / 32), r = lane + 32 * i;
        if (c < bk && r < bk) v[q][i] = Akk[(int64_t)c * g.lda + r];
      }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int i = 0; i < (HLQ_MAX_NB + 31) / 32; ++i) {
        const int c = c0 + q * (GT / 32), r = lane + 32 * i;
        if (c < bk && r < bk) W[(int64_t)c * ldw + r] = v[q][i];
      }
  }
  if (tid == 0) zp_sh = 0;
  __syncthreads();
  for (int p0 = 0; p0 < bk; p0 += GPW) {
    const int pw = min(GPW, bk - p0);
    const int rows = bk - p0;
    // The panel lives in registers: thread r owns panel row r (rows <= nb <= GT) for the whole
    // panel.  Per column two barriers: (B) every warp reduces the partial maxima (redundantly),
    // the pivot row's owner publishes it to X and the owner of row c its row to Y; (A) the two
    // exchange rows, every row below c is scaled by the pivot and updated with the pivot row
    // (broadcast from X), and each warp takes its partial first maximum of the NEXT column.
    double* X = U;             // pivot row (GPW doubles)
    double* Y = U + GPW;       // row c on its way to the pivot's position
    double pr_[GPW];
    const bool own = tid < rows;
#pragma unroll
    for (int j = 0; j < GPW; ++j)
      pr_[j] = (own && j < pw) ? W[(int64_t)(p0 + j) * ldw + p0 + tid] : 0.0;
    const int nwarp_rows = GT / 32;
    {
      unsigned long long key = own ? piv_key(fabs(pr_[0])) : 0ull;
      int bidx = own ? tid : 0x7fffffff;
      warp_piv_reduce(key, bidx);
      if (lane == 0) {
        rv[warp] = key;
        ri[warp] = bidx;
      }
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < GPW; ++c) {
      if (c < pw) {
        unsigned long long bk_ = lane < nwarp_rows ? rv[lane] : 0ull;
        int bi = lane < nwarp_rows ? ri[lane] : 0x7fffffff;
        warp_piv_reduce(bk_, bi);
        if (bi == 0x7fffffff || bi >= rows) bi = c;
        if (tid == 0) {
          piv_sh[c] = bi;
          ipiv[p0 + c] = p0 + bi;
        }
        if (tid == bi) {
#pragma unroll
          for (int j = 0; j < GPW; ++j) X[j] = pr_[j];
        }
        if (tid == c && bi != c) {
#pragma unroll
          for (int j = 0; j < GPW; ++j) Y[j] = pr_[j];
        }
        __syncthreads();
        if (bi != c) {
          if (tid == c) {
#pragma unroll
            for (int j = 0; j < GPW; ++j) pr_[j] = X[j];
          } else if (tid == bi) {
#pragma unroll
            for (int j = 0; j < GPW; ++j) pr_[j] = Y[j];
          }
        }
        const double d = X[c];
        if (d == 0.0 && tid == 0) zp_sh = 1;  // ledger 7: column left unscaled, no update
        const bool act = own && tid > c;
        if (act && d != 0.0) {
          const double l = pr_[c] / d;
          pr_[c] = l;
#pragma unroll
          for (int j = c + 1; j < GPW; ++j) pr_[j] = __dsub_rn(pr_[j], __dmul_rn(l, X[j]));
        }
        if (c + 1 < pw) {
          unsigned long long key = act ? piv_key(fabs(pr_[c + 1])) : 0ull;
          int bidx = act ? tid : 0x7fffffff;
          warp_piv_reduce(key, bidx);
          if (lane == 0) {
            rv[warp] = key;
            ri[warp] = bidx;
          }
        }
        __syncthreads();
      }
    }
    if (own) {  // the factored panel: to shared memory (L11, L21 below) and back to W
#pragma unroll
      for (int j = 0; j < GPW; ++j)
        if (j < pw) {
          P[j * ldp + tid] = pr_[j];
          W[(int64_t)(p0 + j) * ldw + p0 + tid] = pr_[j];
        }
    }
    // apply the panel's swaps to every other column of the tile (left and right): the 32 sequential
    // swaps compose into a permutation that moves at most 64 rows; gather those rows column by
    // column, one warp per column.
    {
      int* perm = reinterpret_cast<int*>(sm + 2 * GPW * ldp);      // rows ints
      int* mv = perm + ((rows + 1) & ~1);                           // <= 2*GPW moved rows
      __shared__ int nmv_sh;
      for (int r = tid; r < rows; r += GT) perm[r] = r;
      __syncthreads();
      if (tid == 0) {
        for (int c = 0; c < pw; ++c) {
          const int pr = piv_sh[c];
          if (pr != c) {
            const int t = perm[c];
            perm[c] = perm[pr];
            perm[pr] = t;
          }
        }
        nmv_sh = 0;
      }
      __syncthreads();
      // moved rows (order irrelevant: every one has its own destination)
      for (int r = tid; r < rows; r += GT)
        if (perm[r] != r) mv[atomicAdd(&nmv_sh, 1)] = r;
      __syncthreads();
      const int nmv = nmv_sh;
      const int nother = bk - pw;
      // one warp per column: lane owns moved rows lane and lane + 32 (nmv <= 64); all loads of a
      // column precede its stores (__syncwarp), four columns in flight per warp
      int du0 = -1, su0 = 0, du1 = -1, su1 = 0;
      if (lane < nmv) { du0 = mv[lane]; su0 = perm[du0]; }
      if (lane + 32 < nmv) { du1 = mv[lane + 32]; su1 = perm[du1]; }
      if (nmv > 0) {
        constexpr int NW = GT / 32, CF = 4;
        for (int t0 = warp; t0 < nother; t0 += NW * CF) {
          double v0[CF], v1[CF];
#pragma unroll
          for (int q = 0; q < CF; ++q) {
            const int t = t0 + NW * q;
            const int col = (t < p0) ? t : t + pw;
            const double* wc = W + (int64_t)col * ldw + p0;
            if (t < nother && du0 >= 0) v0[q] = wc[su0];
            if (t < nother && du1 >= 0) v1[q] = wc[su1];
          }
          __syncwarp();
#pragma unroll
          for (int q = 0; q < CF; ++q) {
            const int t = t0 + NW * q;
            const int col = (t < p0) ? t : t + pw;
            double* wc = W + (int64_t)col * ldw + p0;
            if (t < nother && du0 >= 0) wc[du0] = v0[q];
            if (t < nother && du1 >= 0) wc[du1] = v1[q];
          }
        }
      }
    }
    __syncthreads();
    const int ntr = bk - p0 - pw;  // trailing columns
    if (ntr > 0) {
      // U12 = L11^-1 A12: forward substitution per column in elimination order
      // (same rounding order per element as the column-by-column substitution, l increasing; the
      // 32 running sums of a column are independent chains held in registers)
      for (int t = tid; t < ntr; t += GT) {
        int col = p0 + pw + t;
        double* wc = W + (int64_t)col * ldw + p0;
        double acc[GPW];
#pragma unroll
        for (int c = 0; c < GPW; ++c) acc[c] = c < pw ? wc[c] : 0.0;
#pragma unroll
        for (int l = 0; l < GPW; ++l) {
          if (l < pw) {
            const double u = acc[l];
            U[l * ldp + t] = u;
            wc[l] = u;
#pragma unroll
            for (int c = l + 1; c < GPW; ++c) acc[c] = __dsub_rn(acc[c], __dmul_rn(P[l * ldp + c], u));
          }
        }
      }
      __syncthreads();
      // trailing update: W[p0+pw+r][col] -= sum_c L21[r][c] U12[c][col], sequential in c; the
      // per-thread block shrinks with the trailing matrix so that idle lanes stay few
      const int nr = rows - pw;
      double* Wt = W + (int64_t)(p0 + pw) * ldw + p0 + pw;
      if (ntr > 64 && nr > 32)
        trail_update<4, 4>(Wt, ldw, P + pw, U, ldp, nr, ntr, pw, tid);
      else if (nr > 32)
        trail_update<4, 2>(Wt, ldw, P + pw, U, ldp, nr, ntr, pw, tid);
      else
        trail_update<2, 2>(Wt, ldw, P + pw, U, ldp, nr, ntr, pw, tid);
    }
    __syncthreads();
  }
  if (tid == 0) zp_out[0] = zp_sh;
}

void launch_getrf(const double* A, Geo g, int k, DevWork w, bool need, cudaStream_t st) {
  if (!need) return;
  size_t smem = sizeof(double) * (2 * GPW + GT / 32) * (g.nb + 1);
  static unsigned long long attr = 0;
  if (first_on_device(attr)) {
    smem_optin(k_getrf);
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
                                                 double* inv_norm, int dense) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * 8 + warp;
  if (j >= bk) return;
  const double* lj = Li + (int64_t)j * ldw;
  double colsum = 0.0;
  for (int r = lane; r < bk; r += 32) {
    double x = 0.0;
    const int cb = dense ? r : (r > j ? r : j);  // dense Li (A2: Q^T) has no zero upper part
    for (int c = cb; c < bk; ++c) x += Ui[(int64_t)c * ldw + r] * lj[c];
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

// NEXT f4, variant A2: the diagonal tile is QR-factored in place; W <- the tile, zero
// pivot = an exact zero on R's diagonal, no row interchanges (identity ipiv / permutation), Li <- I.
__global__ void k_a2_prep(const double* __restrict__ A, Geo g, int k, double* __restrict__ W,
                          int* __restrict__ zp, int* __restrict__ ipiv_step, int* __restrict__ perm,
                          double* __restrict__ Li) {
  const int bk = g.bs(k);
  const double* Akk = g.tile(const_cast<double*>(A), k, k);
  __shared__ int zero;
  if (threadIdx.x == 0) zero = 0;
  __syncthreads();
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < bk * bk;
       idx += gridDim.x * blockDim.x) {
    const int c = idx / bk, r = idx - c * bk;
    const double v = Akk[(int64_t)c * g.lda + r];
    W[(int64_t)c * g.nb + r] = v;
    Li[(int64_t)c * g.nb + r] = (r == c) ? 1.0 : 0.0;
    if (r == c && v == 0.0) zero = 1;
  }
  __syncthreads();
  if (blockIdx.x == 0) {
    for (int c = threadIdx.x; c < bk; c += blockDim.x) {
      ipiv_step[c] = c;
      perm[c] = c;
    }
  }
  if (threadIdx.x == 0 && zero) atomicOr(zp, 1);
}

void launch_a2_prep(const double* A, Geo g, int k, DevWork w, cudaStream_t st) {
  cudaMemsetAsync(w.zp, 0, sizeof(int), st);
  int* perm = reinterpret_cast<int*>(w.scratch + (size_t)2 * g.nb * g.nb);
  ::hlq::g_launches++;
  k_a2_prep<<<8, 256, 0, st>>>(A, g, k, w.W, w.zp, w.ipiv + (size_t)k * g.nb, perm, w.scratch);
}

void launch_invnorm(Geo g, int k, DevWork w, cudaStream_t st, int estimate, int dense) {
  const int bk = g.bs(k);
  const double* Li = w.scratch;                       // filled by launch_tri_inv
  const double* Ui = w.scratch + (size_t)g.nb * g.nb;
  if (estimate) {
    ::hlq::g_launches++;
    k_invnorm_est<<<1, 256, 0, st>>>(Li, Ui, bk, g.nb, w.inv_norm);
    return;
  }
  cudaMemsetAsync(w.inv_norm, 0, sizeof(double), st);
  { ::hlq::g_launches++; k_invnorm<<<(bk + 7) / 8, 256, 0, st>>>(Li, Ui, bk, g.nb, w.inv_norm, dense); }
}

}  // namespace hlq
