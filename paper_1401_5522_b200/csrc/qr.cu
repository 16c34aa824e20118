// QR step on the HQR greedy tree (Alg. 3, Alg. 4b; tree: DESIGN.md reading 16),
// predicated on dec[k] == QR.  The paper's LU decomposition of the panel "is dropped, and the
// factorization of the panel starts over": W is simply discarded.
//   a8  GEQRT of every panel tile (i,k), i >= k, in parallel (one CTA per tile);
//       UNMQR: row block i <- Q_ik^T row block i for all columns right of the panel
//   a11 TT levels of the greedy tree: TTQRT(e, i) merges R_i into R_e (V upper triangular stored in
//       the upper triangle of tile (i,k)), TTMQR applies it to [row e; row i]
// Householder convention: LAPACK dlarfg (reading 14); T factors ib-blocked, forward column-wise
// (dlarft), block b of tile (i,k) in columns b*ib.. of an ib x nb array (reading 15).
// The UNMQR/TTMQR kernels take a generic column block (base, ldc, ncols) so the solve reuses them
// on the right-hand side (ncols = 1).
#include <math.h>

#include "hlq_internal.cuh"

namespace hlq {

constexpr int QT = 256;   // threads per CTA (8 warps)
constexpr int MAXIB = 32;
constexpr int TLD = 33;   // T block smem stride

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct QRSmem {
  double* Vs;    // MAXIB x ldv : reflector block (column l at Vs + l*ldv)
  double* Ts;    // MAXIB x TLD : T block, T(q,l) at Ts[l*TLD + q]
  double* xs;    // 8 warps x ldv : column buffers
  double* ys;    // 8 warps x MAXIB
  double* ws;    // 8 warps x MAXIB
  double* Rs;    // MAXIB x TLD : R_e block of a TT factorization
  int ldv;
};

__device__ __forceinline__ QRSmem carve(double* sm, int nb) {
  QRSmem s;
  s.ldv = nb + 1;
  s.Vs = sm;
  s.Ts = s.Vs + MAXIB * s.ldv;
  s.xs = s.Ts + MAXIB * TLD;
  s.ys = s.xs + 8 * s.ldv;
  s.ws = s.ys + 8 * MAXIB;
  s.Rs = s.ws + 8 * MAXIB;
  return s;
}
static size_t qr_smem_bytes(int nb) {
  return sizeof(double) * ((size_t)MAXIB * (nb + 1) + 2 * MAXIB * TLD + 8 * (nb + 1) + 16 * MAXIB);
}

// Apply H_b^T = (I - V T V^T)^T of a GEQRT block to one column x (rows R, local to the block start),
// V unit lower (implicit 1 at (l,l), stored below), warp-cooperative, x in the warp's smem buffer.
__device__ void apply_unit_col(double* x, int R, const QRSmem& s, int sb, double* w, int lane) {
  for (int l = 0; l < sb; ++l) {
    const double* v = s.Vs + l * s.ldv;
    double p = 0.0;
    for (int r = l + 1 + lane; r < R; r += 32) p += v[r] * x[r];
    p = wsum(p);
    if (lane == 0) w[l] = (l < R ? x[l] : 0.0) + p;
  }
  __syncwarp();
  double u = 0.0;
  if (lane < sb)
    for (int q = 0; q <= lane; ++q) u += s.Ts[lane * TLD + q] * w[q];
  __syncwarp();
  if (lane < sb) w[lane] = u;
  __syncwarp();
  for (int r = lane; r < R; r += 32) {
    double acc = 0.0;
    int lmax = r < sb ? r : sb - 1;
    for (int l = 0; l <= lmax; ++l) acc += ((l == r) ? 1.0 : s.Vs[l * s.ldv + r]) * w[l];
    x[r] -= acc;
  }
  __syncwarp();
}

// Apply a TS/TT block: [c1 (sb rows); c2 (R2 rows)] <- Q_b^T [c1; c2], V2 = Vs (zeros stored where
// the TT structure has zeros).
__device__ void apply_pair_col(double* c1, double* c2, int R2, const QRSmem& s, int sb, double* w,
                               int lane) {
  for (int l = 0; l < sb; ++l) {
    const double* v = s.Vs + l * s.ldv;
    double p = 0.0;
    for (int r = lane; r < R2; r += 32) p += v[r] * c2[r];
    p = wsum(p);
    if (lane == 0) w[l] = c1[l] + p;
  }
  __syncwarp();
  double u = 0.0;
  if (lane < sb)
    for (int q = 0; q <= lane; ++q) u += s.Ts[lane * TLD + q] * w[q];
  __syncwarp();
  if (lane < sb) {
    w[lane] = u;
    c1[lane] -= u;
  }
  __syncwarp();
  for (int r = lane; r < R2; r += 32) {
    double acc = 0.0;
    for (int l = 0; l < sb; ++l) acc += s.Vs[l * s.ldv + r] * w[l];
    c2[r] -= acc;
  }
  __syncwarp();
}

// dlarfg on (alpha = *a, x[0..n)) in place by one warp: returns tau; *a <- beta; x <- v.
__device__ double warp_larfg(double* a, double* x, int n, int lane) {
  double p = 0.0;
  for (int r = lane; r < n; r += 32) p += x[r] * x[r];
  double ssq = wsum(p);
  double alpha = *a;
  if (ssq == 0.0) {
    for (int r = lane; r < n; r += 32) x[r] = 0.0;
    __syncwarp();
    return 0.0;
  }
  double nrm = sqrt(alpha * alpha + ssq);
  double beta = alpha >= 0.0 ? -nrm : nrm;
  double tau = (beta - alpha) / beta;
  double sc = alpha - beta;
  for (int r = lane; r < n; r += 32) x[r] = x[r] / sc;
  __syncwarp();
  if (lane == 0) *a = beta;
  __syncwarp();
  return tau;
}

// ---------------------------------------------------------------------------------------------
// GEQRT of tiles (k + blockIdx.x, k)
__global__ void __launch_bounds__(QT) k_geqrt(double* __restrict__ A, Geo g, int k, int ib,
                                              double* __restrict__ Tg, const uint8_t* __restrict__ dec) {
  if (dec != nullptr && dec[k] != HLQ_DEC_QR) return;
  extern __shared__ double sm[];
  QRSmem s = carve(sm, g.nb);
  const int i = k + blockIdx.x;
  const int bi = g.bs(i), bk = g.cbs(k);
  double* tile = g.tile(A, i, k);
  double* T = Tg + tri_index(i, k, g.n) * (int64_t)ib * g.nb;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int t = tid; t < ib * g.nb; t += QT) T[t] = 0.0;
  for (int i0 = 0; i0 < bk; i0 += ib) {
    const int sb = min(ib, bk - i0);
    const int R = bi - i0;
    if (R <= 0) break;  // wide ragged tile: remaining reflectors are the identity
    for (int t = tid; t < sb * R; t += QT) {
      int l = t / R, r = t - l * R;
      s.Vs[l * s.ldv + r] = tile[(int64_t)(i0 + l) * g.lda + i0 + r];
    }
    for (int t = tid; t < MAXIB * TLD; t += QT) s.Ts[t] = 0.0;
    __syncthreads();
    if (warp == 0) {
      for (int l = 0; l < sb && l < R; ++l) {
        double* v = s.Vs + l * s.ldv;
        double tau = warp_larfg(&v[l], v + l + 1, R - l - 1, lane);
        if (tau != 0.0) {
          for (int c = l + 1; c < sb; ++c) {
            double* vc = s.Vs + c * s.ldv;
            double p = 0.0;
            for (int r = l + 1 + lane; r < R; r += 32) p += v[r] * vc[r];
            double wv = vc[l] + wsum(p);
            __syncwarp();
            for (int r = l + 1 + lane; r < R; r += 32) vc[r] -= tau * (v[r] * wv);
            if (lane == 0) vc[l] -= tau * wv;
            __syncwarp();
          }
        }
        // T column l: T(l,l) = tau, T(0:l,l) = -tau T(0:l,0:l) z, z_q = V_q . v_l
        double* wz = s.ws + warp * MAXIB;
        for (int q = 0; q < l; ++q) {
          const double* vq = s.Vs + q * s.ldv;
          double p = 0.0;
          for (int r = l + 1 + lane; r < R; r += 32) p += vq[r] * v[r];
          p = wsum(p);
          if (lane == 0) wz[q] = vq[l] + p;
        }
        __syncwarp();
        double tv = 0.0;
        if (lane < l)
          for (int p2 = lane; p2 < l; ++p2) tv += s.Ts[p2 * TLD + lane] * wz[p2];
        __syncwarp();
        if (lane < l) s.Ts[l * TLD + lane] = -tau * tv;
        if (lane == 0) s.Ts[l * TLD + l] = tau;
        __syncwarp();
      }
    }
    __syncthreads();
    for (int t = tid; t < sb * R; t += QT) {
      int l = t / R, r = t - l * R;
      tile[(int64_t)(i0 + l) * g.lda + i0 + r] = s.Vs[l * s.ldv + r];
    }
    for (int t = tid; t < sb * sb; t += QT) {
      int l = t / sb, q = t - l * sb;
      T[(int64_t)(i0 + l) * ib + q] = s.Ts[l * TLD + q];
    }
    // trailing columns of the tile
    double* xb = s.xs + warp * s.ldv;
    double* wb = s.ws + warp * MAXIB;
    for (int c = i0 + sb + warp; c < bk; c += 8) {
      double* col = tile + (int64_t)c * g.lda + i0;
      for (int r = lane; r < R; r += 32) xb[r] = col[r];
      __syncwarp();
      apply_unit_col(xb, R, s, sb, wb, lane);
      for (int r = lane; r < R; r += 32) col[r] = xb[r];
      __syncwarp();
    }
    __syncthreads();
  }
}

// UNMQR: for tile rows i = k + blockIdx.y, columns [c0 + 64*blockIdx.x, +64) of the block
// (base + r0(i), ldc): C_i <- Q_ik^T C_i
__global__ void __launch_bounds__(QT) k_unmqr(const double* __restrict__ A, Geo g, int k, int ib,
                                              const double* __restrict__ Tg, double* base,
                                              int64_t ldc, int64_t ncols,
                                              const uint8_t* __restrict__ dec) {
  if (dec != nullptr && dec[k] != HLQ_DEC_QR) return;
  extern __shared__ double sm[];
  QRSmem s = carve(sm, g.nb);
  const int i = k + blockIdx.y;
  const int bi = g.bs(i), bk = g.cbs(k);
  const double* tile = g.tile(const_cast<double*>(A), i, k);
  const double* T = Tg + tri_index(i, k, g.n) * (int64_t)ib * g.nb;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t c0 = (int64_t)blockIdx.x * 64;
  double* xb = s.xs + warp * s.ldv;
  double* wb = s.ws + warp * MAXIB;
  for (int i0 = 0; i0 < bk; i0 += ib) {
    const int sb = min(ib, bk - i0);
    const int R = bi - i0;
    if (R <= 0) break;
    __syncthreads();
    for (int t = tid; t < sb * R; t += QT) {
      int l = t / R, r = t - l * R;
      s.Vs[l * s.ldv + r] = tile[(int64_t)(i0 + l) * g.lda + i0 + r];
    }
    for (int t = tid; t < sb * sb; t += QT) {
      int l = t / sb, q = t - l * sb;
      s.Ts[l * TLD + q] = T[(int64_t)(i0 + l) * ib + q];
    }
    __syncthreads();
    for (int cc = warp; cc < 64; cc += 8) {
      int64_t c = c0 + cc;
      if (c >= ncols) break;
      double* col = base + c * ldc + g.r0(i) + i0;
      for (int r = lane; r < R; r += 32) xb[r] = col[r];
      __syncwarp();
      apply_unit_col(xb, R, s, sb, wb, lane);
      for (int r = lane; r < R; r += 32) col[r] = xb[r];
      __syncwarp();
    }
  }
}

// TTQRT on pairs (e, i) = pairs[blockIdx.x]: [R_e; R_i] (both upper triangular) -> R_e, V (upper
// triangle of tile (i,k)), T.
__global__ void __launch_bounds__(QT) k_ttqrt(double* __restrict__ A, Geo g, int k, int ib,
                                              double* __restrict__ Ttt, const int2* __restrict__ pairs,
                                              const uint8_t* __restrict__ dec) {
  if (dec != nullptr && dec[k] != HLQ_DEC_QR) return;
  extern __shared__ double sm[];
  QRSmem s = carve(sm, g.nb);
  const int2 pr = pairs[blockIdx.x];
  const int e = pr.x, i = pr.y;
  const int bi = g.bs(i), bk = g.cbs(k);
  double* Re = g.tile(A, e, k);
  double* Ri = g.tile(A, i, k);
  double* T = Ttt + tri_index(i, k, g.n) * (int64_t)ib * g.nb;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* Rs = s.Rs;  // MAXIB x TLD block of R_e (row q, col l at Rs[l*TLD + q])
  for (int t = tid; t < ib * g.nb; t += QT) T[t] = 0.0;
  for (int i0 = 0; i0 < bk; i0 += ib) {
    const int sb = min(ib, bk - i0);
    const int R2 = min(bi, i0 + sb);  // rows of V2 that can be nonzero
    __syncthreads();
    for (int t = tid; t < sb * R2; t += QT) {
      int l = t / R2, r = t - l * R2;
      s.Vs[l * s.ldv + r] = (r <= i0 + l) ? Ri[(int64_t)(i0 + l) * g.lda + r] : 0.0;
    }
    for (int t = tid; t < sb * sb; t += QT) {
      int l = t / sb, q = t - l * sb;
      Rs[l * TLD + q] = (q <= l) ? Re[(int64_t)(i0 + l) * g.lda + i0 + q] : 0.0;
    }
    for (int t = tid; t < MAXIB * TLD; t += QT) s.Ts[t] = 0.0;
    __syncthreads();
    if (warp == 0) {
      for (int l = 0; l < sb; ++l) {
        double* v = s.Vs + l * s.ldv;
        const int nr = min(R2, i0 + l + 1);
        double tau = warp_larfg(&Rs[l * TLD + l], v, nr, lane);
        if (tau != 0.0) {
          for (int c = l + 1; c < sb; ++c) {
            double* vc = s.Vs + c * s.ldv;
            double p = 0.0;
            for (int r = lane; r < nr; r += 32) p += v[r] * vc[r];
            double wv = Rs[c * TLD + l] + wsum(p);
            __syncwarp();
            for (int r = lane; r < nr; r += 32) vc[r] -= tau * (v[r] * wv);
            if (lane == 0) Rs[c * TLD + l] -= tau * wv;
            __syncwarp();
          }
        }
        double* wz = s.ws + warp * MAXIB;
        for (int q = 0; q < l; ++q) {
          const double* vq = s.Vs + q * s.ldv;
          double p = 0.0;
          for (int r = lane; r < nr; r += 32) p += vq[r] * v[r];
          p = wsum(p);
          if (lane == 0) wz[q] = p;
        }
        __syncwarp();
        double tv = 0.0;
        if (lane < l)
          for (int p2 = lane; p2 < l; ++p2) tv += s.Ts[p2 * TLD + lane] * wz[p2];
        __syncwarp();
        if (lane < l) s.Ts[l * TLD + lane] = -tau * tv;
        if (lane == 0) s.Ts[l * TLD + l] = tau;
        __syncwarp();
      }
    }
    __syncthreads();
    for (int t = tid; t < sb * R2; t += QT) {
      int l = t / R2, r = t - l * R2;
      if (r <= i0 + l) Ri[(int64_t)(i0 + l) * g.lda + r] = s.Vs[l * s.ldv + r];
    }
    for (int t = tid; t < sb * sb; t += QT) {
      int l = t / sb, q = t - l * sb;
      if (q <= l) Re[(int64_t)(i0 + l) * g.lda + i0 + q] = Rs[l * TLD + q];
      T[(int64_t)(i0 + l) * ib + q] = s.Ts[l * TLD + q];
    }
    __syncthreads();
    // trailing columns c >= i0+sb of the pair (R_e rows i0..i0+sb-1, R_i rows 0..R2-1)
    for (int c = i0 + sb + warp; c < bk; c += 8) {
      double* col1 = Re + (int64_t)c * g.lda + i0;
      double* col2 = Ri + (int64_t)c * g.lda;
      double* wb = s.ws + warp * MAXIB;
      double* c1b = s.ys + warp * MAXIB;
      for (int r = lane; r < sb; r += 32) c1b[r] = col1[r];
      __syncwarp();
      // c2 directly in global memory (rows < R2 <= c: upper part of tile (i,k))
      apply_pair_col(c1b, col2, R2, s, sb, wb, lane);
      for (int r = lane; r < sb; r += 32) col1[r] = c1b[r];
      __syncwarp();
    }
  }
}

// TTMQR on pairs[blockIdx.y] for columns [64*blockIdx.x, +64) of (base, ldc):
// [C_e; C_i] <- Q^T [C_e; C_i]
__global__ void __launch_bounds__(QT) k_ttmqr(const double* __restrict__ A, Geo g, int k, int ib,
                                              const double* __restrict__ Ttt,
                                              const int2* __restrict__ pairs, double* base,
                                              int64_t ldc, int64_t ncols,
                                              const uint8_t* __restrict__ dec) {
  if (dec != nullptr && dec[k] != HLQ_DEC_QR) return;
  extern __shared__ double sm[];
  QRSmem s = carve(sm, g.nb);
  const int2 pr = pairs[blockIdx.y];
  const int e = pr.x, i = pr.y;
  const int bi = g.bs(i), bk = g.cbs(k);
  const double* Vt = g.tile(const_cast<double*>(A), i, k);
  const double* T = Ttt + tri_index(i, k, g.n) * (int64_t)ib * g.nb;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t c0 = (int64_t)blockIdx.x * 64;
  double* xb = s.xs + warp * s.ldv;
  double* wb = s.ws + warp * MAXIB;
  double* c1b = s.ys + warp * MAXIB;
  for (int i0 = 0; i0 < bk; i0 += ib) {
    const int sb = min(ib, bk - i0);
    const int R2 = min(bi, i0 + sb);
    __syncthreads();
    for (int t = tid; t < sb * R2; t += QT) {
      int l = t / R2, r = t - l * R2;
      s.Vs[l * s.ldv + r] = (r <= i0 + l) ? Vt[(int64_t)(i0 + l) * g.lda + r] : 0.0;
    }
    for (int t = tid; t < sb * sb; t += QT) {
      int l = t / sb, q = t - l * sb;
      s.Ts[l * TLD + q] = T[(int64_t)(i0 + l) * ib + q];
    }
    __syncthreads();
    for (int cc = warp; cc < 64; cc += 8) {
      int64_t c = c0 + cc;
      if (c >= ncols) break;
      double* col1 = base + c * ldc + g.r0(e) + i0;
      double* col2 = base + c * ldc + g.r0(i);
      for (int r = lane; r < sb; r += 32) c1b[r] = col1[r];
      for (int r = lane; r < R2; r += 32) xb[r] = col2[r];
      __syncwarp();
      apply_pair_col(c1b, xb, R2, s, sb, wb, lane);
      for (int r = lane; r < sb; r += 32) col1[r] = c1b[r];
      for (int r = lane; r < R2; r += 32) col2[r] = xb[r];
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------------------------------------
// The solve's Q^T x (one column): every reflector block read once straight from global memory
// (coalesced down the columns), the vector segment in shared memory; one CTA per tile row (UNMQR)
// or per TT pair.  Per block b: W = [x_e(b) +] V_b^T x, U = T_b^T W, x -= V_b U [x_e(b) -= U].
// Dot products: warp w takes reflectors 4w..4w+3, lanes stride the rows, warp-shuffle reduction.
// The solve's Q^T x, register form: thread t owns rows t and t + 256 of the tile (nb <= 320) and,
// per reflector block, its rows of V_b (32 registers per row), so V is read once; W = V_b^T x is a
// transpose-butterfly reduction (31 shuffles per warp) plus a fixed-order sum of the 8 warp
// partials, U = T_b^T W by 32 threads, and x -= V_b U stays in registers.
template <bool TT>
__global__ void __launch_bounds__(256) k_qr_apply_vec2(const double* __restrict__ A, Geo g, int k,
                                                       int ib, const double* __restrict__ Tb,
                                                       const int2* __restrict__ pairs,
                                                       double* __restrict__ x) {
  __shared__ double red[8][33];
  __shared__ double Uv[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int e = 0, i;
  if (TT) {
    const int2 pr = pairs[blockIdx.x];
    e = pr.x;
    i = pr.y;
  } else {
    i = k + blockIdx.x;
  }
  const int bi = g.bs(i), bk = g.cbs(k);
  const double* V = g.tile(const_cast<double*>(A), i, k);
  const double* T = Tb + tri_index(i, k, g.n) * (int64_t)ib * g.nb;
  double* xi = x + g.r0(i);
  double* xe = x + g.r0(e);
  const int r0 = tid, r1 = tid + 256;
  double x0 = r0 < bi ? xi[r0] : 0.0, x1 = r1 < bi ? xi[r1] : 0.0;
  for (int i0 = 0; i0 < bk; i0 += 32) {
    const int sb = min(32, bk - i0);
    if (!TT && i0 >= bi) break;
    // this thread's rows of V_b with the reflector structure made explicit
    double v0[32], v1[32];
#pragma unroll
    for (int l = 0; l < 32; ++l) {
      const int c = i0 + l;
      const double* col = V + (int64_t)c * g.lda;
      if (TT) {
        v0[l] = (l < sb && r0 < bi && r0 <= c) ? col[r0] : 0.0;
        v1[l] = (l < sb && r1 < bi && r1 <= c) ? col[r1] : 0.0;
      } else {
        v0[l] = (l < sb && r0 < bi && r0 >= c) ? (r0 == c ? 1.0 : col[r0]) : 0.0;
        v1[l] = (l < sb && r1 < bi && r1 >= c) ? (r1 == c ? 1.0 : col[r1]) : 0.0;
      }
    }
    // W = [x_e(b) +] V_b^T x
    double p[32];
#pragma unroll
    for (int l = 0; l < 32; ++l) p[l] = v0[l] * x0 + v1[l] * x1;
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
      const bool upper = (lane & s) != 0;
#pragma unroll
      for (int c = 0; c < s; ++c) {
        const double send = upper ? p[c] : p[c + s];
        const double keep = upper ? p[c + s] : p[c];
        p[c] = keep + __shfl_xor_sync(0xffffffffu, send, s);
      }
    }
    red[warp][lane] = p[0];
    __syncthreads();
    if (warp == 0) {
      double w = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) w += red[q][lane];
      const double xo = (TT && lane < sb) ? xe[i0 + lane] : 0.0;  // x_e(b) before the block
      if (TT) w += xo;
      // U = T_b^T W: u_l = sum_{q <= l} T(q, l) W_q (T(q, l) at T[(i0 + l) * ib + q])
      double u = 0.0;
      for (int q = 0; q < 32; ++q) {
        const double wq = __shfl_sync(0xffffffffu, w, q);
        if (q <= lane && lane < sb) u += T[(int64_t)(i0 + lane) * ib + q] * wq;
      }
      Uv[lane] = u;
      if (TT && lane < sb) xe[i0 + lane] = xo - u;  // x_e(b) -= U
    }
    __syncthreads();
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int l = 0; l < 32; ++l) {
      a0 += v0[l] * Uv[l];
      a1 += v1[l] * Uv[l];
    }
    x0 -= a0;
    x1 -= a1;
    __syncthreads();
  }
  if (r0 < bi) xi[r0] = x0;
  if (r1 < bi) xi[r1] = x1;
}

template <bool TT>
__global__ void __launch_bounds__(256) k_qr_apply_vec(const double* __restrict__ A, Geo g, int k,
                                                      int ib, const double* __restrict__ Tb,
                                                      const int2* __restrict__ pairs,
                                                      double* __restrict__ x) {
  __shared__ double xs[512];
  __shared__ double xe[32];
  __shared__ double Wv[32], Uv[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int e = 0, i;
  if (TT) {
    const int2 pr = pairs[blockIdx.x];
    e = pr.x;
    i = pr.y;
  } else {
    i = k + blockIdx.x;
  }
  const int bi = g.bs(i), bk = g.cbs(k);
  const double* V = g.tile(const_cast<double*>(A), i, k);
  const double* T = Tb + tri_index(i, k, g.n) * (int64_t)ib * g.nb;
  double* xi = x + g.r0(i);
  for (int r = tid; r < bi; r += 256) xs[r] = xi[r];
  __syncthreads();
  for (int i0 = 0; i0 < bk; i0 += ib) {
    const int sb = min(ib, bk - i0);
    if (!TT && i0 >= bi) break;
    if (TT && tid < sb) xe[tid] = x[g.r0(e) + i0 + tid];
    // W
    for (int l = warp; l < sb; l += 8) {
      const double* v = V + (int64_t)(i0 + l) * g.lda;
      double p = 0.0;
      if (TT) {
        const int rhi = min(bi, i0 + l + 1);
        for (int r = lane; r < rhi; r += 32) p += v[r] * xs[r];
      } else {
        for (int r = i0 + l + 1 + lane; r < bi; r += 32) p += v[r] * xs[r];
      }
      p = wsum(p);
      if (lane == 0) Wv[l] = p;
    }
    __syncthreads();
    if (tid < sb) {
      const double w0 = TT ? xe[tid] : (i0 + tid < bi ? xs[i0 + tid] : 0.0);
      Wv[tid] += w0;
    }
    __syncthreads();
    // U = T^T W (T(q, l) at T[(i0 + l) * ib + q], upper triangular)
    if (tid < sb) {
      double u = 0.0;
      for (int q = 0; q <= tid; ++q) u += T[(int64_t)(i0 + tid) * ib + q] * Wv[q];
      Uv[tid] = u;
    }
    __syncthreads();
    // x -= V U
    if (TT) {
      for (int r = tid; r < min(bi, i0 + sb); r += 256) {
        double acc = 0.0;
        for (int l = (r > i0 ? r - i0 : 0); l < sb; ++l) acc += V[(int64_t)(i0 + l) * g.lda + r] * Uv[l];
        xs[r] -= acc;
      }
      if (tid < sb) x[g.r0(e) + i0 + tid] = xe[tid] - Uv[tid];
    } else {
      for (int r = i0 + tid; r < bi; r += 256) {
        const int lmax = min(r - i0, sb - 1);
        double acc = 0.0;
        for (int l = 0; l <= lmax; ++l)
          acc += ((i0 + l == r) ? 1.0 : V[(int64_t)(i0 + l) * g.lda + r]) * Uv[l];
        xs[r] -= acc;
      }
    }
    __syncthreads();
  }
  for (int r = tid; r < bi; r += 256) xi[r] = xs[r];
}

static void set_attr_once() {
  static bool done = false;
  if (done) return;
  done = true;
  smem_optin(k_geqrt);
  smem_optin(k_unmqr);
  smem_optin(k_ttqrt);
  smem_optin(k_ttmqr);
}

// Apply the stored QR step k to the column block (base rows 0..N-1, ldc, ncols): used by the
// factorization (columns right of the panel) and by the solve (the right-hand side).
void launch_qr_apply(const double* A, Geo g, int k, int ib, const double* Tg, const double* Ttt,
                     const int2* const* level_pairs, const int* level_count, int nlevels,
                     double* base, int64_t ldc, int64_t ncols, const uint8_t* dec,
                     cudaStream_t st) {
  set_attr_once();
  size_t smem = qr_smem_bytes(g.nb);
  if (ncols <= 0) return;
  if (ncols == 1 && dec == nullptr && ib == 32) {
    { ::hlq::g_launches++; k_qr_apply_vec2<false><<<g.n - k, 256, 0, st>>>(A, g, k, ib, Tg, nullptr, base); }
    for (int l = 0; l < nlevels; ++l)
      { ::hlq::g_launches++; k_qr_apply_vec2<true><<<level_count[l], 256, 0, st>>>(A, g, k, ib, Ttt, level_pairs[l], base); }
    return;
  }
  if (ncols == 1 && dec == nullptr && g.nb <= 512) {
    { ::hlq::g_launches++; k_qr_apply_vec<false><<<g.n - k, 256, 0, st>>>(A, g, k, ib, Tg, nullptr, base); }
    for (int l = 0; l < nlevels; ++l)
      { ::hlq::g_launches++; k_qr_apply_vec<true><<<level_count[l], 256, 0, st>>>(A, g, k, ib, Ttt, level_pairs[l], base); }
    return;
  }
  unsigned slabs = (unsigned)((ncols + 63) / 64);
  { ::hlq::g_launches++; k_unmqr<<<dim3(slabs, g.n - k), QT, smem, st>>>(A, g, k, ib, Tg, base, ldc, ncols, dec); }
  for (int l = 0; l < nlevels; ++l)
    { ::hlq::g_launches++; k_ttmqr<<<dim3(slabs, level_count[l]), QT, smem, st>>>(A, g, k, ib, Ttt, level_pairs[l], base,
                                                           ldc, ncols, dec); }
}

void launch_tt_apply(const double* A, Geo g, int k, int ib, const double* Ttt,
                     const int2* const* level_pairs, const int* level_count, int nlevels,
                     double* base, int64_t ldc, int64_t ncols, const uint8_t* dec,
                     cudaStream_t st) {
  set_attr_once();
  size_t smem = qr_smem_bytes(g.nb);
  if (ncols <= 0) return;
  if (ncols == 1 && dec == nullptr && ib == 32) {
    for (int l = 0; l < nlevels; ++l)
      { ::hlq::g_launches++; k_qr_apply_vec2<true><<<level_count[l], 256, 0, st>>>(A, g, k, ib, Ttt, level_pairs[l], base); }
    return;
  }
  if (ncols == 1 && dec == nullptr && g.nb <= 512) {
    for (int l = 0; l < nlevels; ++l)
      { ::hlq::g_launches++; k_qr_apply_vec<true><<<level_count[l], 256, 0, st>>>(A, g, k, ib, Ttt, level_pairs[l], base); }
    return;
  }
  unsigned slabs = (unsigned)((ncols + 63) / 64);
  for (int l = 0; l < nlevels; ++l)
    { ::hlq::g_launches++; k_ttmqr<<<dim3(slabs, level_count[l]), QT, smem, st>>>(A, g, k, ib, Ttt, level_pairs[l], base,
                                                           ldc, ncols, dec); }
}

// Panel stage of a QR step (column block k only): GEQRT of every panel tile, then the TTQRT of
// every level of the greedy tree (a TTQRT only touches panel tiles, so all levels run before any
// trailing update).  Predicated on dec[k] == QR.
void launch_qr_panel(double* A, Geo g, int k, int ib, const int2* const* level_pairs,
                     const int* level_count, int nlevels, const DevWork& w, cudaStream_t st,
                     bool diag_done) {
  set_attr_once();
  const size_t smem = qr_smem_bytes(g.nb);
  const uint8_t* dec = w.dec;
  const bool tc = (ib == 32);
  if (tc)
    launch_qr_panel_tc(A, g, k, ib, w.Tg, w.Ttt, nullptr, 0, dec, false, st,
                       diag_done ? k + 1 : k);
  else
    { ::hlq::g_launches++; k_geqrt<<<g.n - k, QT, smem, st>>>(A, g, k, ib, w.Tg, dec); }
  for (int l = 0; l < nlevels; ++l) {
    if (tc)
      launch_qr_panel_tc(A, g, k, ib, w.Tg, w.Ttt, level_pairs[l], level_count[l], dec, true, st);
    else
      { ::hlq::g_launches++; k_ttqrt<<<level_count[l], QT, smem, st>>>(A, g, k, ib, w.Ttt, level_pairs[l], dec); }
  }
}

// Update stage of a QR step on the trailing columns [c0, c1): UNMQR of every tile row, then the
// TTMQR of every level in order.  Predicated on dec[k] == QR.
bool launch_qr_update(double* A, Geo g, int k, int ib, const int2* const* level_pairs,
                      const int* level_count, int nlevels, const DevWork& w, int64_t c0,
                      int64_t c1, cudaStream_t st, double* gmax) {
  set_attr_once();
  const size_t smem = qr_smem_bytes(g.nb);
  const uint8_t* dec = w.dec;
  const int64_t ncols = c1 - c0;
  if (ncols <= 0) return true;
  bool fused = gmax != nullptr && nlevels > 0;
  double* base = A + c0 * g.lda;
  const unsigned slabs = (unsigned)((ncols + 63) / 64);
  const bool tc = (ib == 32);  // DMMA trailing updates (qr_dmma.cu) need 32-row reflector blocks
  if (tc)
    launch_qr_update_dmma(A, g, k, ib, w.Tg, w.Ttt, level_pairs, level_count, nlevels, base,
                          g.lda, ncols, dec, 0, st);
  else
    { ::hlq::g_launches++; k_unmqr<<<dim3(slabs, g.n - k), QT, smem, st>>>(A, g, k, ib, w.Tg, base, g.lda, ncols, dec); }
  for (int l = 0; l < nlevels; ++l) {
    if (tc) {
      fused &= launch_qr_update_dmma(A, g, k, ib, w.Tg, w.Ttt, level_pairs, level_count, nlevels,
                                     base, g.lda, ncols, dec, 1 + l, st, gmax);
    } else {
      fused = false;
      { ::hlq::g_launches++; k_ttmqr<<<dim3(slabs, level_count[l]), QT, smem, st>>>(A, g, k, ib, w.Ttt, level_pairs[l], base, g.lda, ncols, dec); }
    }
  }
  return fused;
}

}  // namespace hlq
