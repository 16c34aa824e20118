// a13: solve by a second pass over b ("apply the transformations on b during a
// second pass") followed by the N x N block back substitution.  HBM-bound: every factor
// element is read once (the GEMV kernels are coalesced down the columns of the LAPACK layout).
// Also: the HPL3 residual pieces ||Ax-b||_inf, ||A||_inf, ||x||_inf and the final
// status scan (non-finite factors, exact zeros on the U/R diagonal).
#include <math.h>

#include <algorithm>

#include "hlq_internal.cuh"

namespace hlq {

// Triangular solves on one diagonal tile with one CTA (256 threads): the tile is streamed through
// shared memory in 32-column panels (coalesced loads); x_k lives in shared memory.
constexpr int SP = 32;

// LU step k forward: x_k <- L_kk^-1 P_kk x_k  (unit lower, column-oriented)
__global__ void __launch_bounds__(256) k_solve_lu_diag(const double* __restrict__ A, Geo g, int k,
                                                       const int* __restrict__ ipiv,
                                                       double* __restrict__ x) {
  extern __shared__ double sm[];
  const int bk = g.bs(k);
  const int ld = bk + 1;
  double* Ps = sm;            // SP x ld
  double* xs = sm + SP * ld;  // bk
  const double* Akk = g.tile(const_cast<double*>(A), k, k);
  double* xk = x + g.r0(k);
  const int tid = threadIdx.x;
  for (int r = tid; r < bk; r += 256) xs[r] = xk[r];
  __syncthreads();
  if (tid == 0 && ipiv != nullptr)
    for (int c = 0; c < bk; ++c) {
      int p = ipiv[(int64_t)k * g.nb + c];
      if (p != c) {
        double t = xs[c];
        xs[c] = xs[p];
        xs[p] = t;
      }
    }
  for (int p0 = 0; p0 < bk; p0 += SP) {
    const int pw = min(SP, bk - p0);
    __syncthreads();
    for (int t = tid; t < pw * bk; t += 256) {
      int c = t / bk, r = t - c * bk;
      Ps[c * ld + r] = Akk[(int64_t)(p0 + c) * g.lda + r];
    }
    __syncthreads();
    // warp 0: the pw x pw unit-lower diagonal block
    if (tid < 32) {
      for (int c = 0; c < pw; ++c) {
        double xc = xs[p0 + c];
        __syncwarp();
        if (tid > c && tid < pw) xs[p0 + tid] -= Ps[c * ld + p0 + tid] * xc;
        __syncwarp();
      }
    }
    __syncthreads();
    // all threads: rows below the block
    for (int r = p0 + pw + tid; r < bk; r += 256) {
      double acc = 0.0;
      for (int c = 0; c < pw; ++c) acc += Ps[c * ld + r] * xs[p0 + c];
      xs[r] -= acc;
    }
  }
  __syncthreads();
  for (int r = tid; r < bk; r += 256) xk[r] = xs[r];
}

// back substitution on the diagonal tile: x_k <- U_kk^-1 x_k (panels from the right)
__global__ void __launch_bounds__(256) k_solve_upper_diag(const double* __restrict__ A, Geo g, int k,
                                                          double* __restrict__ x) {
  extern __shared__ double sm[];
  const int bk = g.bs(k);
  const int ld = bk + 1;
  double* Ps = sm;
  double* xs = sm + SP * ld;
  const double* Akk = g.tile(const_cast<double*>(A), k, k);
  double* xk = x + g.r0(k);
  const int tid = threadIdx.x;
  for (int r = tid; r < bk; r += 256) xs[r] = xk[r];
  const int npan = (bk + SP - 1) / SP;
  for (int pi = npan - 1; pi >= 0; --pi) {
    const int p0 = pi * SP, pw = min(SP, bk - p0);
    __syncthreads();
    for (int t = tid; t < pw * (p0 + pw); t += 256) {
      int c = t / (p0 + pw), r = t - c * (p0 + pw);
      Ps[c * ld + r] = Akk[(int64_t)(p0 + c) * g.lda + r];
    }
    __syncthreads();
    if (tid < 32) {
      for (int c = pw - 1; c >= 0; --c) {
        double xc = xs[p0 + c] / Ps[c * ld + p0 + c];
        __syncwarp();
        if (tid == c) xs[p0 + c] = xc;
        if (tid < c) xs[p0 + tid] -= Ps[c * ld + p0 + tid] * xc;
        __syncwarp();
      }
    }
    __syncthreads();
    for (int r = tid; r < p0; r += 256) {
      double acc = 0.0;
      for (int c = 0; c < pw; ++c) acc += Ps[c * ld + r] * xs[p0 + c];
      xs[r] -= acc;
    }
  }
  __syncthreads();
  for (int r = tid; r < bk; r += 256) xk[r] = xs[r];
}

// y[0:M) -= B[0:M, 0:K) * v[0:K)   (B column-major): CTA = 64 rows x all K, 4 threads per row
// each summing a quarter of the columns, partials combined in a fixed order (deterministic).
__global__ void __launch_bounds__(256) k_gemv_sub(double* __restrict__ y, const double* __restrict__ B,
                                                  int64_t ldb, int64_t M, int K,
                                                  const double* __restrict__ v) {
  extern __shared__ double vs[];  // K + 256
  double* part = vs + K;
  for (int c = threadIdx.x; c < K; c += blockDim.x) vs[c] = v[c];
  __syncthreads();
  const int rl = threadIdx.x & 63, q = threadIdx.x >> 6;
  const int64_t r = (int64_t)blockIdx.x * 64 + rl;
  double acc = 0.0;
  if (r < M)
    for (int c = q; c < K; c += 4) acc += B[(int64_t)c * ldb + r] * vs[c];
  part[q * 64 + rl] = acc;
  __syncthreads();
  if (q == 0 && r < M) y[r] -= ((part[rl] + part[64 + rl]) + part[128 + rl]) + part[192 + rl];
}

void launch_gemv_sub(double* y, const double* B, int64_t ldb, int64_t M, int K, const double* v,
                     cudaStream_t st) {
  if (M <= 0 || K <= 0) return;
  { ::hlq::g_launches++; k_gemv_sub<<<(unsigned)((M + 63) / 64), 256, sizeof(double) * (K + 256), st>>>(y, B, ldb, M, K, v); }
}

static void solve_attr_once() {
  static unsigned long long done = 0;
  if (!first_on_device(done)) return;
  smem_optin(k_solve_lu_diag);
  smem_optin(k_solve_upper_diag);
}

void launch_solve_lu_fwd(const double* A, Geo g, int k, const int* ipiv, double* x,
                         cudaStream_t st) {
  solve_attr_once();
  size_t smem = sizeof(double) * ((size_t)SP * (g.bs(k) + 1) + g.bs(k));
  { ::hlq::g_launches++; k_solve_lu_diag<<<1, 256, smem, st>>>(A, g, k, ipiv, x); }
  const int64_t k0 = g.r0(k), k1 = k0 + g.bs(k);
  launch_gemv_sub(x + k1, A + k0 * g.lda + k1, g.lda, g.N - k1, g.bs(k), x + k0, st);
}

void launch_solve_back(const double* A, Geo g, int k, double* x, cudaStream_t st) {
  solve_attr_once();
  size_t smem = sizeof(double) * ((size_t)SP * (g.bs(k) + 1) + g.bs(k));
  { ::hlq::g_launches++; k_solve_upper_diag<<<1, 256, smem, st>>>(A, g, k, x); }
  const int64_t k0 = g.r0(k);
  launch_gemv_sub(x, A + k0 * g.lda, g.lda, k0, g.bs(k), x + k0, st);
}

// ---------------------------------------------------------------------------------------------
// LU steps with the explicit triangular inverses kept by the factorization (L_kk^-1, U_kk^-1 are
// what Eliminate / Apply multiply by, Alg. 2): the diagonal solves become parallel GEMVs.
// t[r] = sum_c M[c*ld + r] * v(c) over the triangle (lower: c <= r, upper: c >= r) or the whole
// row (dense: the A2 variant's Q_kk^T), v(c) = x_k[perm[c]] or x_k[c]; one CTA per 32 rows, 8 warps
// splitting c, partials summed in a fixed order.
template <bool LOWER, bool DENSE = false>
__global__ void __launch_bounds__(256) k_tri_gemv(const double* __restrict__ M, int ld, int bk,
                                                  const int* __restrict__ perm,
                                                  const double* __restrict__ xk,
                                                  double* __restrict__ t) {
  __shared__ double v[512];
  __shared__ double part[8][33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = threadIdx.x; c < bk; c += 256) v[c] = xk[perm ? perm[c] : c];
  __syncthreads();
  const int r = blockIdx.x * 32 + lane;
  double acc = 0.0;
  if (r < bk) {
    const int c0 = (LOWER || DENSE) ? 0 : r, c1 = DENSE ? bk : (LOWER ? r + 1 : bk);
    for (int c = c0 + ((warp - c0) % 8 + 8) % 8; c < c1; c += 8) acc += M[(int64_t)c * ld + r] * v[c];
  }
  part[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && r < bk) {
    double s2 = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) s2 += part[w][lane];
    t[r] = s2;
  }
}

void launch_solve_lu_fwd_inv(const double* A, Geo g, int k, const double* Li, const int* perm,
                             double* x, double* t, cudaStream_t st, bool dense) {
  const int bk = g.bs(k);
  const int64_t k0 = g.r0(k), k1 = k0 + bk;
  ::hlq::g_launches++;
  if (dense)
    k_tri_gemv<true, true><<<(bk + 31) / 32, 256, 0, st>>>(Li, g.nb, bk, perm, x + k0, t);
  else
    k_tri_gemv<true><<<(bk + 31) / 32, 256, 0, st>>>(Li, g.nb, bk, perm, x + k0, t);
  cudaMemcpyAsync(x + k0, t, sizeof(double) * bk, cudaMemcpyDeviceToDevice, st);
  launch_gemv_sub(x + k1, A + k0 * g.lda + k1, g.lda, g.N - k1, bk, x + k0, st);
}

void launch_solve_back_inv(const double* A, Geo g, int k, const double* Ui, double* x, double* t,
                           cudaStream_t st) {
  const int bk = g.bs(k);
  const int64_t k0 = g.r0(k);
  { ::hlq::g_launches++; k_tri_gemv<false><<<(bk + 31) / 32, 256, 0, st>>>(Ui, g.nb, bk, nullptr, x + k0, t); }
  cudaMemcpyAsync(x + k0, t, sizeof(double) * bk, cudaMemcpyDeviceToDevice, st);
  launch_gemv_sub(x, A + k0 * g.lda, g.lda, k0, bk, x + k0, st);
}

// ---------------------------------------------------------------------------------------------
// Persistent block-row solves: one launch per pass over many block rows, so the n sequential
// dependencies of the solve do not each cost a kernel launch and the factor reads of independent
// tiles overlap the dependency chain.  Work unit (i, c): block row i, chunk c of G tiles of that
// row (left of the diagonal in the forward pass, right of it in the back substitution).  Units
// take tickets in start order (atomic counter) from a host-built table ordered so that a unit only
// ever waits for units with smaller tickets -- units that are already running -- so the spin waits
// cannot deadlock.  A chunk publishes its partial sums (pflag); the LAST chunk of row i (the
// finisher) adds them in chunk order (deterministic), then solves the diagonal tile by blocked
// substitution and publishes x_i (xflag).  Release/acquire at GPU scope order the data.
constexpr int PS_T = 256;

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// each flag on its own 128-byte line (kFlagStride ints) so the pollers of different flags do not
// share an L2 line; the poll backs off (up to 256 ns) to keep a thousand spinning CTAs off L2
constexpr int kFlagStride = 32;
__device__ __forceinline__ void wait_flag(const int* p, int want) {
  unsigned ns = 32;
  while (ld_acquire(p) != want) {
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
  }
}

// acc[s][e] += sum over columns c (c = h, h+2, ...) of T(row 2q+256s+e, c) * xs[c]; with V2 (even
// ld, 16-byte aligned tile) the two rows are one 16-byte load
template <bool V2>
__device__ __forceinline__ void gemv_tile(const double* __restrict__ T, int64_t lda, int rows,
                                          int cols, const double* xs, int q, int h,
                                          double (&acc)[2][2]) {
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int r = 2 * q + 256 * s;
    if (r >= rows) continue;
    const bool two = r + 1 < rows;
    double a0 = 0.0, a1 = 0.0;
    if (V2 && two) {
#pragma unroll 16
      for (int c = h; c < cols; c += 2) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(T + (int64_t)c * lda + r));
        const double xv = xs[c];
        a0 = fma(v.x, xv, a0);
        a1 = fma(v.y, xv, a1);
      }
    } else {
#pragma unroll 8
      for (int c = h; c < cols; c += 2) {
        const double* col = T + (int64_t)c * lda + r;
        const double xv = xs[c];
        a0 = fma(__ldg(col), xv, a0);
        if (two) a1 = fma(__ldg(col + 1), xv, a1);
      }
    }
    acc[s][0] += a0;
    acc[s][1] += a1;
  }
}

// L2 prefetch of a tile (rows x cols, column-major, ld lda): one bulk prefetch per column, issued
// while the unit still waits for the x segment it will multiply (the tile does not depend on it)
__device__ __forceinline__ void prefetch_tile_l2(const double* T, int64_t lda, int rows, int cols,
                                                 int tid) {
  const unsigned bytes = (unsigned)(rows * 8) & ~15u;
  if (bytes == 0) return;
  for (int c = tid; c < cols; c += PS_T) {
    const double* p = T + (int64_t)c * lda;
    if ((((uintptr_t)p) & 15) == 0)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
  }
}

// Diagonal-tile triangular solves of the persistent passes, latency-pipelined (the n tile solves
// of a pass are its sequential chain; every load below is independent of the right-hand side):
//   * two chain warps alternate over the 32 x 32 diagonal blocks (warp t & 1 runs the t-th block's
//     register/shuffle substitution) and load their next block's coefficients right after a chain,
//     so they land while the other warp chains; the first two blocks are loaded by preload(), which
//     the finisher calls BEFORE it waits for the other chunks' partial sums;
//   * warps 2..7 own the rows the block's solution updates and load their 32 coefficients before
//     the barrier that ends the chain, so after it the update is 32 FMAs from registers.
// The arithmetic (per-row FMA order, reciprocal pivots) is that of the unpipelined solves.
template <bool LOWER>
struct TileSolve {
  double reg[32];  // chain warps: the block's triangle coefficients; update warps: a row's 32
  double rd;       // upper: 1 / U_rr of the chain lane's row
  // block index of chain step t
  __device__ __forceinline__ static int blk(int t, int nblk) { return LOWER ? t : nblk - 1 - t; }
  __device__ __forceinline__ void load_chain(const double* __restrict__ D, int64_t lda, int bi,
                                             int base, int lane) {
    const int r = base + lane;
#pragma unroll
    for (int cc = 0; cc < 32; ++cc) {
      const bool ok = LOWER ? (cc < lane && r < bi) : (cc > lane && base + cc < bi);
      reg[cc] = ok ? __ldg(D + (int64_t)(base + cc) * lda + r) : 0.0;
    }
    if (!LOWER) {
      // 1 / U_rr for every lane at once: the substitution chain multiplies instead of dividing
      const double d = r < bi ? __ldg(D + (int64_t)r * lda + r) : 1.0;
      rd = 1.0 / d;
    }
  }
  __device__ __forceinline__ void preload(const double* __restrict__ D, int64_t lda, int bi,
                                          int tid) {
    const int lane = tid & 31, warp = tid >> 5, nblk = (bi + 31) / 32;
    if (warp < 2 && warp < nblk) load_chain(D, lda, bi, 32 * blk(warp, nblk), lane);
  }
  // ys (bi entries, shared) <- L^-1 ys (unit lower) or U^-1 ys (upper, non-unit); preload() first
  __device__ __forceinline__ void run(const double* __restrict__ D, int64_t lda, int bi,
                                      double* ys, int tid) {
    const int lane = tid & 31, warp = tid >> 5, nblk = (bi + 31) / 32;
    constexpr int UT = PS_T - 64;  // update threads (warps 2..)
    const int uidx = tid - 64;
    for (int t = 0; t < nblk; ++t) {
      const int base = 32 * blk(t, nblk);
      const int pw = min(32, bi - base);
      // rows this block's solution updates: below it (lower) / above it (upper)
      const int ulo = LOWER ? base + 32 : 0, uhi = LOWER ? bi : base;
      const int r0 = ulo + uidx;
      const bool upd = warp >= 2 && r0 < uhi;
      if (upd) {
#pragma unroll
        for (int cc = 0; cc < 32; ++cc)
          reg[cc] = cc < pw ? __ldg(D + (int64_t)(base + cc) * lda + r0) : 0.0;
      }
      if (warp == (t & 1)) {
        const int r = base + lane;
        double v = r < bi ? ys[r] : 0.0;
        if (LOWER) {
#pragma unroll
          for (int cc = 0; cc < 32; ++cc) {
            const double xc = __shfl_sync(0xffffffffu, v, cc);
            if (lane > cc) v = fma(-reg[cc], xc, v);
          }
        } else {
#pragma unroll
          for (int cc = 31; cc >= 0; --cc) {
            if (lane == cc) v = v * rd;
            const double xc = __shfl_sync(0xffffffffu, v, cc);
            if (lane < cc) v = fma(-reg[cc], xc, v);
          }
        }
        if (r < bi) ys[r] = v;
        if (t + 2 < nblk) load_chain(D, lda, bi, 32 * blk(t + 2, nblk), lane);
      }
      __syncthreads();
      if (warp >= 2) {
        if (upd) {
          double a = 0.0;
#pragma unroll
          for (int cc = 0; cc < 32; ++cc) a = fma(reg[cc], cc < pw ? ys[base + cc] : 0.0, a);
          ys[r0] -= a;
        }
        for (int r = r0 + UT; r < uhi; r += UT) {  // (more than UT rows left: nb > 256 or block 0)
#pragma unroll
          for (int cc = 0; cc < 32; ++cc)
            reg[cc] = cc < pw ? __ldg(D + (int64_t)(base + cc) * lda + r) : 0.0;
          double a = 0.0;
#pragma unroll
          for (int cc = 0; cc < 32; ++cc) a = fma(reg[cc], cc < pw ? ys[base + cc] : 0.0, a);
          ys[r] -= a;
        }
      }
      __syncthreads();
    }
  }
};

// FWD: forward pass of the LU steps [ka, kb) over block rows i >= ka (x_i -= sum_j L_ij x_j, then
// x_i <- L_ii^-1 P_i x_i for i < kb).  BACK: back substitution over all block rows
// (x_i <- U_ii^-1 (x_i - sum_{j>i} U_ij x_j)).
template <bool FWD>
__global__ void __launch_bounds__(PS_T) k_solve_rows(const double* __restrict__ A, Geo g, int ka,
                                                     int kb, int G, int cmax,
                                                     const int2* __restrict__ units,
                                                     const int* __restrict__ perm_all,
                                                     double* __restrict__ x, int* __restrict__ xflag,
                                                     double* __restrict__ part,
                                                     int* __restrict__ pflag,
                                                     unsigned* __restrict__ ticket) {
  __shared__ int2 s_u;
  __shared__ double xs[HLQ_MAX_NB];
  __shared__ double ys[HLQ_MAX_NB];
  __shared__ double red[2][HLQ_MAX_NB];
  const int tid = threadIdx.x, q = tid & 127, h = tid >> 7;
  if (tid == 0) s_u = units[atomicAdd(ticket, 1u)];
  __syncthreads();
  const int i = s_u.x, c = s_u.y;
  const int bi = g.bs(i), nb = g.nb;
  // tiles of this unit, in the order their x_j become available
  int jfirst, ntiles, cn;
  if (FWD) {
    const int jend = min(i, kb);
    cn = max(1, (jend - ka + G - 1) / G);
    jfirst = ka + c * G;
    ntiles = max(0, min(G, jend - jfirst));
  } else {
    cn = max(1, (g.n - 1 - i + G - 1) / G);
    jfirst = g.n - 1 - c * G;  // descending
    ntiles = max(0, min(G, jfirst - i));
  }
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  const bool v2 = ((g.lda & 1) == 0) && ((((uintptr_t)A) & 15) == 0) && ((g.nb & 1) == 0);
  // the factor tiles do not depend on x: pull the next tile into L2 while the x segment it
  // multiplies is still being solved -- one tile ahead only (prefetching every resident unit's
  // tiles at once overflowed L2 and evicted them before use), the diagonal tile with the last one
  const int cn0 = FWD ? max(1, (min(i, kb) - ka + G - 1) / G) : max(1, (g.n - 1 - i + G - 1) / G);
  const bool finisher = c + 1 == cn0 && (!FWD || i < kb);
  if (ntiles > 0) {
    prefetch_tile_l2(A + g.r0(jfirst) * g.lda + g.r0(i), g.lda, bi, g.bs(jfirst), tid);
  } else if (finisher) {
    prefetch_tile_l2(A + g.r0(i) * g.lda + g.r0(i), g.lda, bi, bi, tid);
  }
  for (int t = 0; t < ntiles; ++t) {
    const int j = FWD ? jfirst + t : jfirst - t;
    const int bj = g.bs(j);
    if (t + 1 < ntiles) {
      const int jn = FWD ? j + 1 : j - 1;
      prefetch_tile_l2(A + g.r0(jn) * g.lda + g.r0(i), g.lda, bi, g.bs(jn), tid);
    } else if (finisher) {
      prefetch_tile_l2(A + g.r0(i) * g.lda + g.r0(i), g.lda, bi, bi, tid);
    }
    if (tid == 0) wait_flag(xflag + (int64_t)j * kFlagStride, 1);
    __syncthreads();
    for (int cc = tid; cc < bj; cc += PS_T) xs[cc] = __ldcg(x + g.r0(j) + cc);
    __syncthreads();
    if (v2)
      gemv_tile<true>(A + g.r0(j) * g.lda + g.r0(i), g.lda, bi, bj, xs, q, h, acc);
    else
      gemv_tile<false>(A + g.r0(j) * g.lda + g.r0(i), g.lda, bi, bj, xs, q, h, acc);
    __syncthreads();
  }
  // the two column halves' partial sums, per row
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int r = 2 * q + 256 * s + e;
      if (r < bi) red[h][r] = acc[s][e];
    }
  __syncthreads();
  double* my_part = part + ((int64_t)i * cmax + c) * nb;
  if (c + 1 < cn) {  // not the finisher: publish the partial sums of this chunk
    for (int r = tid; r < bi; r += PS_T) __stcg(my_part + r, red[0][r] + red[1][r]);
    __threadfence();
    __syncthreads();
    if (tid == 0) st_release(pflag + ((int64_t)i * cmax + c) * kFlagStride, 1);
    return;
  }
  // finisher: r_i = x_i - (sum of the chunk partials in chunk order + own); thread cc waits for
  // chunk cc's flag (all polls in flight at once: a sequential poll of up to n/G already-set flags
  // cost an L2 round trip each on the critical path)
  const bool solves = !(FWD && i >= kb);
  const double* D = A + g.r0(i) * g.lda + g.r0(i);
  TileSolve<FWD> ts;
  int pr[(HLQ_MAX_NB + PS_T - 1) / PS_T];  // row r of P_i x = x[perm[r]] (forward pass)
  if (solves) {
    // everything the diagonal solve loads that does not depend on x, before the waits below
    ts.preload(D, g.lda, bi, tid);
    if (FWD) {
      const int* perm = perm_all + (int64_t)i * nb;
#pragma unroll
      for (int u = 0; u < (HLQ_MAX_NB + PS_T - 1) / PS_T; ++u)
        pr[u] = (tid + u * PS_T < bi) ? __ldg(perm + tid + u * PS_T) : 0;
    }
  }
  for (int cc = tid; cc < c; cc += PS_T) wait_flag(pflag + ((int64_t)i * cmax + cc) * kFlagStride, 1);
  __syncthreads();
  double* xi = x + g.r0(i);
  for (int r = tid; r < bi; r += PS_T) {
    // the partial sums in chunk order, eight loads in flight at a time (a load per dependent add
    // cost an L2 round trip per chunk on the critical path of every block row)
    const double* pp = part + (int64_t)i * cmax * nb + r;
    double sum = 0.0;
    int cc = 0;
    for (; cc + 8 <= c; cc += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcg(pp + (int64_t)(cc + u) * nb);
#pragma unroll
      for (int u = 0; u < 8; ++u) sum += v[u];
    }
    for (; cc < c; ++cc) sum += __ldcg(pp + (int64_t)cc * nb);
    sum += red[0][r] + red[1][r];
    xs[r] = __ldcg(xi + r) - sum;
  }
  __syncthreads();
  if (!solves) {  // a row below the run: only the update
    for (int r = tid; r < bi; r += PS_T) xi[r] = xs[r];
    return;
  }
  if (FWD) {
#pragma unroll
    for (int u = 0; u < (HLQ_MAX_NB + PS_T - 1) / PS_T; ++u)
      if (tid + u * PS_T < bi) ys[tid + u * PS_T] = xs[pr[u]];
  } else {
    for (int r = tid; r < bi; r += PS_T) ys[r] = xs[r];
  }
  __syncthreads();
  ts.run(D, g.lda, bi, ys, tid);
  for (int r = tid; r < bi; r += PS_T) __stcg(xi + r, ys[r]);
  __threadfence();
  __syncthreads();
  if (tid == 0) st_release(xflag + (int64_t)i * kFlagStride, 1);
}

// Host side: unit table (ticket order) for one pass; the device buffers come from the handle's
// solve workspace (xflag n flags, pflag n*cmax flags -- 128 bytes each --, part n*cmax*nb doubles,
// ticket, units).
int solve_rows_cmax(int n, int G) { return std::max(1, (n + G - 1) / G); }

size_t build_solve_units(bool fwd, int n, int ka, int kb, int G, int2* out) {
  size_t u = 0;
  if (fwd) {
    for (int i = ka; i < n; ++i) {
      const int jend = std::min(i, kb);
      const int cn = std::max(1, (jend - ka + G - 1) / G);
      for (int c = 0; c < cn; ++c) out[u++] = make_int2(i, c);
    }
  } else {
    for (int i = n - 1; i >= 0; --i) {
      const int cn = std::max(1, (n - 1 - i + G - 1) / G);
      for (int c = 0; c < cn; ++c) out[u++] = make_int2(i, c);
    }
  }
  return u;
}

void launch_solve_rows(bool fwd, const double* A, Geo g, int ka, int kb, int G, const int2* units,
                       size_t nunits, const int* perm_all, double* x, int* xflag, double* part,
                       int* pflag, unsigned* ticket, cudaStream_t st) {
  if (nunits == 0) return;
  const int cmax = solve_rows_cmax(g.n, G);
  cudaMemsetAsync(ticket, 0, sizeof(unsigned), st);
  cudaMemsetAsync(xflag, 0, sizeof(int) * kFlagStride * (size_t)g.n, st);
  cudaMemsetAsync(pflag, 0, sizeof(int) * kFlagStride * (size_t)g.n * cmax, st);
  ::hlq::g_launches++;
  if (fwd)
    k_solve_rows<true><<<(unsigned)nunits, PS_T, 0, st>>>(A, g, ka, kb, G, cmax, units, perm_all,
                                                          x, xflag, part, pflag, ticket);
  else
    k_solve_rows<false><<<(unsigned)nunits, PS_T, 0, st>>>(A, g, ka, kb, G, cmax, units, perm_all,
                                                           x, xflag, part, pflag, ticket);
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

// final status: flag[0] |= any non-finite factor entry, flag[1] |= exact zero on the diagonal.
// grid-stride over columns (blockIdx), threads over rows with 16-byte loads where aligned: no
// per-element 64-bit division
__global__ void k_final_scan(const double* __restrict__ A, int64_t N, int64_t lda, int* flag) {
  int bad = 0, zero = 0;
  const bool v2 = ((lda & 1) == 0) && ((((uintptr_t)A) & 15) == 0);
  for (int64_t c = blockIdx.x; c < N; c += gridDim.x) {
    const double* col = A + c * lda;
    if (v2) {
      for (int64_t r = 2 * (int64_t)threadIdx.x; r < N; r += 2 * (int64_t)blockDim.x) {
        if (r + 1 < N) {
          const double2 v = *reinterpret_cast<const double2*>(col + r);
          if (!isfinite(v.x) || !isfinite(v.y)) bad = 1;
        } else if (!isfinite(col[r])) {
          bad = 1;
        }
      }
    } else {
      for (int64_t r = threadIdx.x; r < N; r += blockDim.x)
        if (!isfinite(col[r])) bad = 1;
    }
    if (threadIdx.x == 0 && col[c] == 0.0) zero = 1;
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
