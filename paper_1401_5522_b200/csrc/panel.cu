// Panel statistics (a1), decision (a4), tile-norm growth tracking (a12), input generator.
//   a1  s_i = ||A_ik||_1 (i>k), local_max(j), away_max(j)      Eqs. 2-4
//   a4  device-side decision d_k, margin, flags                 Alg. 1
//   a12 max_{i,j>=k} ||A_ij||_1 of the active matrix
// These kernels are HBM/latency bound: one warp per column, coalesced column reads (a column of a
// tile is contiguous in the LAPACK layout), warp-shuffle reductions.
#include <math.h>

#include "hlq_internal.cuh"

namespace hlq {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_nanmax(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = nanmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// grid: (tile rows i in [k, n), column chunks of 32); 256 threads = 8 warps, each warp one column
// at a time with 16-byte loads of row pairs (all the column's loads issued before the reductions);
// the tile norm max over the chunks goes to s[i] with an order-independent atomic max (s zeroed by
// the launcher), so the result does not depend on the chunking
constexpr int PS_CHUNK = 32;
__global__ void __launch_bounds__(256) k_panel_stats(const double* __restrict__ A, Geo g, int k,
                                                     int diag, double* __restrict__ s,
                                                     double* __restrict__ local_max,
                                                     double* __restrict__ away_max, int D) {
  const int i = k + blockIdx.x;
  const int bi = g.bs(i), bk = g.cbs(k);
  const double* T = g.tile(const_cast<double*>(A), i, k);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool v2 = ((g.lda & 1) == 0) && ((((uintptr_t)T) & 15) == 0);
  __shared__ double red[8];
  double tile_norm = 0.0;
  const int cend = min(bk, (int)(blockIdx.y + 1) * PS_CHUNK);
  for (int c = blockIdx.y * PS_CHUNK + warp; c < cend; c += 8) {
    const double* col = T + (int64_t)c * g.lda;
    double sum = 0.0, mx = 0.0;
    if (v2) {
      double2 v[(HLQ_MAX_NB + 63) / 64];
#pragma unroll
      for (int u = 0; u < (HLQ_MAX_NB + 63) / 64; ++u) {
        const int r = 2 * lane + 64 * u;
        v[u] = r + 1 < bi ? *reinterpret_cast<const double2*>(col + r)
                          : make_double2(r < bi ? col[r] : 0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < (HLQ_MAX_NB + 63) / 64; ++u) {
        const double a = fabs(v[u].x), b = fabs(v[u].y);
        sum += a;
        sum += b;
        mx = nanmax(mx, nanmax(a, b));
      }
    } else {
      for (int r = lane; r < bi; r += 32) {
        double a = fabs(col[r]);
        sum += a;
        mx = nanmax(mx, a);
      }
    }
    sum = warp_sum(sum);
    mx = warp_nanmax(mx);
    tile_norm = nanmax(tile_norm, sum);
    if (lane == 0) {
      if (D > 0)  // diagonal-domain statistics (local_max zeroed by the launcher)
        atomic_max_nonneg((i - k) % D == 0 ? &local_max[c] : &away_max[c], mx);
      else if (diag && i == k)
        local_max[c] = mx;
      else
        atomic_max_nonneg(&away_max[c], mx);
    }
  }
  if (lane == 0) red[warp] = tile_norm;
  __syncthreads();
  if (threadIdx.x == 0 && !(diag && i == k) && !(D > 0 && (i - k) % D == 0)) {
    double v = red[0];  // (the domain's tiles are not in the rhs: their s_i stays 0)
    for (int w = 1; w < 8; ++w) v = nanmax(v, red[w]);
    atomic_max_nonneg(&s[i], v);
  }
}

void launch_panel_stats(const double* A, Geo g, int k, DevWork w, cudaStream_t st) {
  launch_panel_stats_to(A, g, k, 1, w.s, w.local_max, w.away_max, st);
}

void launch_panel_stats_to(const double* A, Geo g, int k, int diag, double* s, double* local_max,
                           double* away_max, cudaStream_t st) {
  cudaMemsetAsync(away_max, 0, sizeof(double) * g.nb, st);
  if (g.n - k <= 0) return;
  cudaMemsetAsync(s + k, 0, sizeof(double) * (g.n - k), st);
  const dim3 grid(g.n - k, (g.cbs(k) + PS_CHUNK - 1) / PS_CHUNK);
  { ::hlq::g_launches++; k_panel_stats<<<grid, 256, 0, st>>>(A, g, k, diag, s, local_max, away_max, 0); }
}

void launch_panel_stats_domain(const double* A, Geo g, int k, int D, DevWork w, cudaStream_t st) {
  launch_panel_stats_domain_to(A, g, k, D, w.s, w.local_max, w.away_max, st);
}

// the same into explicit outputs (the 2D grid's statistics record: the owner of the diagonal tile
// holds the whole diagonal domain, tiles k, k + D, ... of its local panel)
void launch_panel_stats_domain_to(const double* A, Geo g, int k, int D, double* s,
                                  double* local_max, double* away_max, cudaStream_t st) {
  cudaMemsetAsync(away_max, 0, sizeof(double) * g.nb, st);
  cudaMemsetAsync(local_max, 0, sizeof(double) * g.nb, st);
  if (g.n - k <= 0) return;
  cudaMemsetAsync(s + k, 0, sizeof(double) * (g.n - k), st);
  ::hlq::g_launches++;
  const dim3 grid(g.n - k, (g.cbs(k) + PS_CHUNK - 1) / PS_CHUNK);
  k_panel_stats<<<grid, 256, 0, st>>>(A, g, k, 1, s, local_max, away_max, D);
}

// ---------------------------------------------------------------------------------------------
// a12: max over tiles i,j >= k of the tile 1-norm = max over (tile row, column) of column-segment
// abs-sums.  grid (tile rows, column groups of 64), 256 threads; atomicMax into *out (>= 0).
__global__ void __launch_bounds__(256) k_tile_norm_max(const double* __restrict__ A, Geo g, int k,
                                                       double* out, const uint8_t* __restrict__ dec,
                                                       int step, int want, int64_t cb, int64_t ce) {
  if (dec != nullptr && dec[step] != want) return;
  const int i = k + blockIdx.x;
  const int bi = g.bs(i);
  const int64_t c0 = cb + (int64_t)blockIdx.y * 64;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double best = 0.0;
  for (int cc = warp; cc < 64; cc += 8) {
    int64_t c = c0 + cc;
    if (c >= ce) break;
    const double* col = A + c * g.lda + g.r0(i);
    double sum = 0.0;
    for (int r = lane; r < bi; r += 32) sum += fabs(col[r]);
    best = nanmax(best, warp_sum(sum));
  }
  if (lane == 0) atomic_max_nonneg(out, best);
}

void launch_tile_norm_max(const double* A, Geo g, int k, double* out, cudaStream_t st,
                          const uint8_t* dec, int step, int want, int64_t cb, int64_t ce) {
  if (cb < 0) cb = g.r0(k);
  if (ce < 0) ce = g.N;
  int64_t ncols = ce - cb;
  if (ncols <= 0) return;
  dim3 grid(g.n - k, (unsigned)((ncols + 63) / 64));
  { ::hlq::g_launches++; k_tile_norm_max<<<grid, 256, 0, st>>>(A, g, k, out, dec, step, want, cb, ce); }
}

// ---------------------------------------------------------------------------------------------
// a4: the decision.  One block of 256 threads.  Mirrors DESIGN.md readings 3,4,5,7,21,22 and the
// MUMPS readings (1, 2).  Writes dec[k], margin[k], flags[k]; status[0] |= nonfinite,
// status[1] |= zero pivot in a forced LU step.
// Counter-based uniform generator: SplitMix64 finalizer.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double rel_margin(double lhs, double rhs) {
  double den = fmax(lhs, rhs);
  if (den == 0.0) return 1.0;
  return (lhs - rhs) / den;
}

__global__ void __launch_bounds__(256) k_decide(Geo g, int k, int crit, double alpha, int reading,
                                                double tol, int has_forced, int has_ref,
                                                DevWork w) {
  const int bk = g.bs(k);
  const int tid = threadIdx.x;
  __shared__ double sh_growth[512];
  __shared__ double sh_min[256];
  __shared__ int sh_fail[256], sh_nan[256];
  __shared__ double sh_mlhs[256], sh_mrhs[256];
  __shared__ double sh_margin, sh_lhs, sh_rhs;
  __shared__ int sh_d, sh_flags;
  const int zp = w.zp[0];
  if (tid == 0) {
    sh_flags = zp ? HLQ_FLAG_ZERO_PIVOT : 0;
    sh_d = -1;
    sh_margin = __longlong_as_double(0x7ff8000000000000LL);  // NaN
    sh_lhs = sh_margin;
    sh_rhs = sh_margin;
    if (has_forced) {
      sh_d = w.forced[k] ? HLQ_DEC_QR : HLQ_DEC_LU;  // any nonzero entry = QR
      sh_flags |= HLQ_FLAG_FORCED;
      if (sh_d == HLQ_DEC_LU && zp) atomicOr(&w.status[1], 1);
    } else if (alpha == 0.0) {
      sh_d = HLQ_DEC_QR;
    } else if (zp) {
      sh_d = HLQ_DEC_QR;
    } else if (isinf(alpha)) {
      sh_d = HLQ_DEC_LU;
    }
  }
  __syncthreads();
  if (sh_d < 0) {
    if (crit == HLQ_CRIT_MAX || crit == HLQ_CRIT_SUM) {
      if (tid == 0) {
        double lhs = alpha / w.inv_norm[0];
        double rhs = 0.0;
        for (int i = k + 1; i < g.n; ++i) {  // ascending i (deterministic, as the oracle)
          double v = w.s[i];
          rhs = (crit == HLQ_CRIT_MAX) ? ((i == k + 1) ? v : nanmax(rhs, v)) : rhs + v;
        }
        sh_lhs = lhs;
        sh_rhs = rhs;
        if (isnan(lhs) || isnan(rhs)) {
          sh_d = HLQ_DEC_QR;
          sh_flags |= HLQ_FLAG_NONFINITE;
        } else {
          sh_d = (lhs >= rhs) ? HLQ_DEC_LU : HLQ_DEC_QR;
          sh_margin = rel_margin(lhs, rhs);
        }
      }
    } else if (crit == HLQ_CRIT_RANDOM) {
      // reading 35: LU iff 100 u_k < alpha, u_k = the counter generator's draw k of stream 31
      if (tid == 0) {
        const uint64_t GAMMA = 0x9E3779B97F4A7C15ULL;
        const uint64_t key = mix64(31ULL + GAMMA);
        const double u = (double)(mix64(key + ((uint64_t)k + 1ULL) * GAMMA) >> 11) * 0x1.0p-53;
        sh_lhs = alpha;
        sh_rhs = u * 100.0;
        sh_d = (u * 100.0 < alpha) ? HLQ_DEC_LU : HLQ_DEC_QR;
      }
    } else {  // MUMPS (Eq. 4)
      for (int j = tid; j < bk; j += 256) {
        double p = fabs(w.W[(int64_t)j * g.nb + j]);
        double lm = w.local_max[j];
        sh_growth[j] = (lm == 0.0) ? (p > 0.0 ? INFINITY : 0.0) : p / lm;
      }
      __syncthreads();
      double mn = INFINITY, mlhs = NAN, mrhs = NAN;
      int fail = 0, nn = 0;
      for (int j = tid; j < bk; j += 256) {
        double p = fabs(w.W[(int64_t)j * g.nb + j]);
        double est = w.away_max[j];
        if (reading == 0) {
          if (est != 0.0) est = est * sh_growth[j];
        } else {
          for (int i = 0; i < j; ++i)
            if (est != 0.0) est = est * sh_growth[i];
        }
        double lhs = alpha * p;
        if (isnan(lhs) || isnan(est)) {
          nn = 1;
          continue;
        }
        double mj = isinf(est) ? -1.0 : rel_margin(lhs, est);
        if (!(lhs >= est)) fail = 1;
        if (mj < mn) {
          mn = mj;
          mlhs = lhs;
          mrhs = est;
        }
      }
      sh_min[tid] = mn;
      sh_fail[tid] = fail;
      sh_nan[tid] = nn;
      sh_mlhs[tid] = mlhs;
      sh_mrhs[tid] = mrhs;
      __syncthreads();
      if (tid == 0) {
        double m = INFINITY;
        int f = 0, q = 0;
        for (int t = 0; t < 256; ++t) {
          if (sh_min[t] < m) {  // the binding column (first minimum in thread order)
            sh_lhs = sh_mlhs[t];
            sh_rhs = sh_mrhs[t];
          }
          m = fmin(m, sh_min[t]);
          f |= sh_fail[t];
          q |= sh_nan[t];
        }
        if (q) {
          sh_d = HLQ_DEC_QR;
          sh_flags |= HLQ_FLAG_NONFINITE;
        } else {
          sh_d = f ? HLQ_DEC_QR : HLQ_DEC_LU;
          sh_margin = (bk == 0) ? 1.0 : m;
        }
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    int d = sh_d;
    double mg = sh_margin;
    int fl = sh_flags;
    if (!has_forced && !isnan(mg)) {
      bool near = fabs(mg) < tol;
      if (near) fl |= HLQ_FLAG_NEAR_TIE;
      if (has_ref && (near || fabs(w.ref_margin[k]) < tol)) {
        d = w.ref_dec[k] ? HLQ_DEC_QR : HLQ_DEC_LU;
        fl |= HLQ_FLAG_HINTED;
      }
    }
    if (fl & HLQ_FLAG_NONFINITE) atomicOr(&w.status[0], 1);
    w.dec[k] = (uint8_t)d;
    w.margin[k] = mg;
    w.flags[k] = fl;
    if (w.steplog != nullptr) {  // the decision log: the binding inequality's two sides
      w.steplog[2 * k] = sh_lhs;
      w.steplog[2 * k + 1] = sh_rhs;
    }
  }
}

void launch_decide(Geo g, int k, int crit, double alpha, int mumps_reading, double tie_tol,
                   int has_forced, int has_ref, DevWork w, cudaStream_t st) {
  { ::hlq::g_launches++; k_decide<<<1, 256, 0, st>>>(g, k, crit, alpha, mumps_reading, tie_tol, has_forced, has_ref, w); }
}

// ---------------------------------------------------------------------------------------------

__global__ void k_generate(double* dst, int64_t rows, int64_t cols, int64_t ld, uint64_t key,
                           uint64_t idx0, int64_t idx_ld) {
  const uint64_t GAMMA = 0x9E3779B97F4A7C15ULL;
  int64_t total = rows * cols;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = t / rows, r = t - c * rows;
    uint64_t idx = idx0 + (uint64_t)c * (uint64_t)idx_ld + (uint64_t)r;
    uint64_t u = mix64(key + (idx + 1ULL) * GAMMA);
    dst[c * ld + r] = (double)(u >> 11) * 0x1.0p-53 - 0.5;
  }
}

void launch_generate(double* dst, int64_t rows, int64_t cols, int64_t ld, uint64_t seed,
                     uint64_t idx0, int64_t idx_ld, cudaStream_t st) {
  // key(seed) = mix64(seed + GAMMA) computed on the host with the same integer arithmetic
  uint64_t z = seed + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  uint64_t key = z ^ (z >> 31);
  int64_t total = rows * cols;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  if (blocks < 1) blocks = 1;
  { ::hlq::g_launches++; k_generate<<<(unsigned)blocks, 256, 0, st>>>(dst, rows, cols, ld, key, idx0, idx_ld); }
}

}  // namespace hlq
