// QR step on the HQR greedy tree (Alg. 3, Alg. 4b; tree: DESIGN.md reading 16),
// predicated on dec[k] == QR.  The paper's LU decomposition of the panel "is dropped, and the
// factorization of the panel starts over": W is simply discarded.
//   a8  GEQRT of every panel tile (i,k), i >= k, in parallel (one CTA per tile, qr_dmma.cu);
//       UNMQR: row block i <- Q_ik^T row block i for all columns right of the panel (qr_update.cu)
//   a11 TT levels of the greedy tree: TTQRT(e, i) merges R_i into R_e (V upper triangular stored in
//       the upper triangle of tile (i,k)), TTMQR applies it to [row e; row i]
// Householder convention: LAPACK dlarfg (reading 14); T factors ib-blocked (ib = 32), forward
// column-wise (dlarft), block b of tile (i,k) in columns b*ib.. of an ib x nb array (reading 15).
// This file holds the step's launch sequence and the solve's Q^T x replay (k_qr_apply_vec2).
#include <math.h>

#include "hlq_internal.cuh"

namespace hlq {

// The solve's Q^T x, register form: thread t owns rows t and t + 256 of the tile (nb <= 320) and,
// per reflector block, its rows of V_b (32 registers per row), so V is read once; W = V_b^T x is a
// transpose-butterfly reduction (31 shuffles per warp) plus a fixed-order sum of the 8 warp
// partials, U = T_b^T W by 32 threads, and x -= V_b U stays in registers.
// MODE 0: GEQRT reflectors of tile row i (unit lower); 1: TT reflectors of the pair (e, i)
// (upper triangular); 2: TS reflectors of the pair (e, i) (square)
template <int MODE, bool CG = false>
__device__ void qr_apply_vec_body(const double* __restrict__ A, Geo g, int k, int ib,
                                  const double* __restrict__ Tb, int e, int i,
                                  double* __restrict__ x, double (*red)[33], double* Uv) {
  // (CG: x is written by other CTAs of the same launch -- read it through L2 only)
  auto ldx = [](const double* p) { if constexpr (CG) return __ldcg(p); else return *p; };
  constexpr bool TT = MODE != 0, TS = MODE == 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bi = g.bs(i), bk = g.cbs(k);
  const double* V = g.tile(const_cast<double*>(A), i, k);
  const double* T = Tb + tri_index(i, k, g.n) * (int64_t)ib * g.nb;
  double* xi = x + g.r0(i);
  double* xe = x + g.r0(e);
  const int r0 = tid, r1 = tid + 256;
  double x0 = r0 < bi ? ldx(xi + r0) : 0.0, x1 = r1 < bi ? ldx(xi + r1) : 0.0;
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
        v0[l] = (l < sb && r0 < bi && (TS || r0 <= c)) ? col[r0] : 0.0;
        v1[l] = (l < sb && r1 < bi && (TS || r1 <= c)) ? col[r1] : 0.0;
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
      const double xo = (TT && lane < sb) ? ldx(xe + i0 + lane) : 0.0;  // x_e(b) before the block
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
__global__ void __launch_bounds__(256) k_qr_apply_vec2(const double* __restrict__ A, Geo g, int k,
                                                       int ib, const double* __restrict__ Tb,
                                                       const int2* __restrict__ pairs,
                                                       const int* __restrict__ rows,
                                                       double* __restrict__ x) {
  __shared__ double red[8][33];
  __shared__ double Uv[32];
  if (TT) {
    const int2 pr = pairs[blockIdx.x];
    qr_apply_vec_body<1>(A, g, k, ib, Tb, pr.x, pr.y, x, red, Uv);
  } else {
    qr_apply_vec_body<0>(A, g, k, ib, Tb, 0, rows != nullptr ? rows[blockIdx.x] : k + blockIdx.x,
                         x, red, Uv);
  }
}

// the TS chains of an HQR step on x: one CTA per group, its pairs in order
__global__ void __launch_bounds__(256) k_qr_apply_vec_ts(const double* __restrict__ A, Geo g, int k,
                                                         int ib, const double* __restrict__ Tb,
                                                         const int2* __restrict__ pairs,
                                                         const int* __restrict__ off,
                                                         double* __restrict__ x) {
  __shared__ double red[8][33];
  __shared__ double Uv[32];
  for (int p = off[blockIdx.x]; p < off[blockIdx.x + 1]; ++p) {
    const int2 pr = pairs[p];
    qr_apply_vec_body<2>(A, g, k, ib, Tb, pr.x, pr.y, x, red, Uv);
    __syncthreads();
  }
}

// The op body of the DAG replay below: qr_apply_vec_body's arithmetic (same products, same
// summation order: bit-identical x) with everything that does not depend on x taken off the
// dependency chain -- the op's T factor (ib x nb) goes to shared memory and the first reflector
// block's V rows to registers BEFORE the op waits for its predecessors; with one row per thread
// (!BIG: nb <= 256) block b + 1's V rows are loaded into a second register set while block b is
// computed; x_e(b) is loaded at the top of the block; U = T_b^T W reads W by shared-memory
// broadcast instead of 32 dependent shuffles.  (ib = 32.)
template <int MODE, bool BIG>
__device__ __forceinline__ void qr_apply_vec_dag(const double* __restrict__ A, Geo g, int k, int ib,
                                                 const double* __restrict__ Tb, int e, int i,
                                                 double* __restrict__ x, double (*red)[33],
                                                 double* Uv, double* Wsh, double* Ts,
                                                 const int* done, int pe, int pi) {
  constexpr bool TT = MODE != 0, TS = MODE == 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bi = g.bs(i), bk = g.cbs(k);
  const double* V = g.tile(const_cast<double*>(A), i, k);
  const double* T = Tb + tri_index(i, k, g.n) * (int64_t)ib * g.nb;
  double* xi = x + g.r0(i);
  double* xe = x + g.r0(e);
  const int r0 = tid, r1 = tid + 256;
  // row r of V_b with the reflector structure made explicit
  auto loadv = [&](int i0, double (&v)[32], int r) {
    const int sb = min(32, bk - i0);
#pragma unroll
    for (int l = 0; l < 32; ++l) {
      const int c = i0 + l;
      const double* col = V + (int64_t)c * g.lda;
      if (TT)
        v[l] = (l < sb && r < bi && (TS || r <= c)) ? col[r] : 0.0;
      else
        v[l] = (l < sb && r < bi && r >= c) ? (r == c ? 1.0 : col[r]) : 0.0;
    }
  };
  // ---- independent of x: T (column c at Ts[33 c ..], conflict-free) and V_0
  for (int o = tid; o < bk * 32; o += 256) Ts[(o >> 5) * 33 + (o & 31)] = T[o];
  double v0[32], v1[BIG ? 32 : 1];
  loadv(0, v0, r0);
  if constexpr (BIG) loadv(0, reinterpret_cast<double(&)[32]>(v1), r1);
  // ---- wait for the previous op on each of the op's rows
  if (tid == 0) {
    unsigned ns = 32;
    auto wait = [&](int q) {
      if (q < 0) return;
      for (;;) {
        int v;
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(done + 32 * q) : "memory");
        if (v) break;
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
      }
    };
    wait(pe);
    wait(pi);
  }
  __syncthreads();
  // (x is written by other CTAs of the same launch -- read it through L2 only)
  double x0 = r0 < bi ? __ldcg(xi + r0) : 0.0, x1 = (BIG && r1 < bi) ? __ldcg(xi + r1) : 0.0;
  for (int i0 = 0; i0 < bk; i0 += 32) {
    const int sb = min(32, bk - i0);
    if (!TT && i0 >= bi) break;
    const bool more = i0 + 32 < bk && (TT || i0 + 32 < bi);
    double vn[BIG ? 1 : 32];
    if constexpr (!BIG) {
      if (more) loadv(i0 + 32, reinterpret_cast<double(&)[32]>(vn), r0);
    }
    const double xo = (TT && warp == 0 && lane < sb) ? __ldcg(xe + i0 + lane) : 0.0;  // x_e(b)
    // W = [x_e(b) +] V_b^T x
    double p[32];
#pragma unroll
    for (int l = 0; l < 32; ++l) {
      if constexpr (BIG)
        p[l] = v0[l] * x0 + v1[l] * x1;
      else
        p[l] = v0[l] * x0;
    }
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
      if (TT) w += xo;
      Wsh[lane] = w;
      __syncwarp();
      // U = T_b^T W: u_l = sum_{q <= l} T(q, l) W_q
      double u = 0.0;
      const double* tc = Ts + (i0 + lane) * 33;
#pragma unroll
      for (int q = 0; q < 32; ++q)
        if (q <= lane && lane < sb) u += tc[q] * Wsh[q];
      Uv[lane] = u;
      if (TT && lane < sb) xe[i0 + lane] = xo - u;  // x_e(b) -= U
    }
    __syncthreads();
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int l = 0; l < 32; ++l) {
      a0 += v0[l] * Uv[l];
      if constexpr (BIG) a1 += v1[l] * Uv[l];
    }
    x0 -= a0;
    if constexpr (BIG) x1 -= a1;
    // (no barrier here: red / Uv / Wsh are rewritten only after the next block's first barrier,
    // which every thread reaches after this block's reads)
    if (more) {
      if constexpr (BIG) {
        loadv(i0 + 32, v0, r0);
        loadv(i0 + 32, reinterpret_cast<double(&)[32]>(v1), r1);
      } else {
#pragma unroll
        for (int l = 0; l < 32; ++l) v0[l] = vn[l];
      }
    }
  }
  if (r0 < bi) xi[r0] = x0;
  if (BIG && r1 < bi) xi[r1] = x1;
}

// The Q^T x replay of a run of consecutive QR steps as ONE launch: one CTA per op (6 ints: kind 0
// GEQRT rows / 1 TS pair / 2 TT pair, rows e and i, the previous op on row e and on row i -- across
// steps --, the step k), listed in dependency order; an op waits for its predecessors' completion
// flags (acquire), applies its reflectors to x_e / x_i and releases its own flag.  (Prefetching
// every resident op's V tile at launch measured slower: a thousand waiting CTAs' tiles overflow L2;
// the op body loads only its T factor and first reflector block ahead of the wait.)  Replaces ~6
// launches per step (each a handful of CTAs) by a single launch whose critical path is the chain of
// ops through the rows.
template <bool BIG, bool OLD = false>
__global__ void __launch_bounds__(256) k_qr_solve_dag(const double* __restrict__ A, Geo g, int ib,
                                                      const double* __restrict__ Tg,
                                                      const double* __restrict__ Ttt,
                                                      const int* __restrict__ ops,
                                                      int* __restrict__ done, double* x) {
  __shared__ double red[8][33];
  __shared__ double Uv[32];
  __shared__ double Wsh[32];
  extern __shared__ __align__(16) double Ts[];  // 33 x nb: the op's T factor
  const int* op = ops + 6 * blockIdx.x;
  const int kind = op[0], e = op[1], i = op[2], pe = op[3], pi = op[4], k = op[5];
  if constexpr (OLD) {  // HLQ_QR_SOLVE_DAG_BODY=0: wait first, then the step-by-step kernels' body
    if (threadIdx.x == 0) {
      unsigned ns = 32;
      auto wait = [&](int q) {
        if (q < 0) return;
        for (;;) {
          int v;
          asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(done + 32 * q) : "memory");
          if (v) break;
          __nanosleep(ns);
          if (ns < 256) ns <<= 1;
        }
      };
      wait(pe);
      wait(pi);
    }
    __syncthreads();
    if (kind == 0)
      qr_apply_vec_body<0, true>(A, g, k, ib, Tg, 0, i, x, red, Uv);
    else if (kind == 1)
      qr_apply_vec_body<2, true>(A, g, k, ib, Ttt, e, i, x, red, Uv);
    else
      qr_apply_vec_body<1, true>(A, g, k, ib, Ttt, e, i, x, red, Uv);
  } else {
    if (kind == 0)
      qr_apply_vec_dag<0, BIG>(A, g, k, ib, Tg, 0, i, x, red, Uv, Wsh, Ts, done, pe, pi);
    else if (kind == 1)
      qr_apply_vec_dag<2, BIG>(A, g, k, ib, Ttt, e, i, x, red, Uv, Wsh, Ts, done, pe, pi);
    else
      qr_apply_vec_dag<1, BIG>(A, g, k, ib, Ttt, e, i, x, red, Uv, Wsh, Ts, done, pe, pi);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(done + 32 * blockIdx.x), "r"(1)
                 : "memory");
  }
}

// done: 32 ints (one 128-byte line) per op, zeroed here
void launch_qr_solve_dag(const double* A, Geo g, int ib, const double* Tg, const double* Ttt,
                         const int* ops, int nops, int* done, double* x, cudaStream_t st) {
  if (nops <= 0) return;
  cudaMemsetAsync(done, 0, sizeof(int) * 32 * (size_t)nops, st);
  ::hlq::g_launches++;
  const size_t smem = sizeof(double) * 33 * (size_t)g.nb;
  static unsigned long long attr = 0;
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(k_qr_solve_dag<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(double) * 33 * HLQ_MAX_NB));
    cudaFuncSetAttribute(k_qr_solve_dag<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(double) * 33 * HLQ_MAX_NB));
  }
  static int body = -1;
  if (body < 0) body = getenv("HLQ_QR_SOLVE_DAG_BODY") ? atoi(getenv("HLQ_QR_SOLVE_DAG_BODY")) : 1;
  if (body == 0)
    k_qr_solve_dag<true, true><<<nops, 256, 0, st>>>(A, g, ib, Tg, Ttt, ops, done, x);
  else if (g.nb > 256)
    k_qr_solve_dag<true><<<nops, 256, smem, st>>>(A, g, ib, Tg, Ttt, ops, done, x);
  else
    k_qr_solve_dag<false><<<nops, 256, smem, st>>>(A, g, ib, Tg, Ttt, ops, done, x);
}

// Apply the stored QR step k to the solve's vector x (rows 0..N-1 of base): Q_ik^T of every
// GEQRT tile, then the TTMQR of every level (ncols must be 1, ib = 32).
void launch_qr_apply(const double* A, Geo g, int k, int ib, const double* Tg, const double* Ttt,
                     const int2* const* level_pairs, const int* level_count, int nlevels,
                     double* base, int64_t ldc, int64_t ncols, const uint8_t* dec,
                     cudaStream_t st, const QRTsPlan* ts) {
  (void)ldc;
  (void)dec;
  if (ncols <= 0) return;
  if (ts != nullptr && ts->ngroups > 0) {  // HQR: Q^T of the group heads, then the TS chains
    { ::hlq::g_launches++; k_qr_apply_vec2<false><<<ts->nheads, 256, 0, st>>>(A, g, k, ib, Tg, nullptr, ts->heads, base); }
    { ::hlq::g_launches++; k_qr_apply_vec_ts<<<ts->ngroups, 256, 0, st>>>(A, g, k, ib, Ttt, ts->pairs, ts->off, base); }
  } else {
    { ::hlq::g_launches++; k_qr_apply_vec2<false><<<g.n - k, 256, 0, st>>>(A, g, k, ib, Tg, nullptr, nullptr, base); }
  }
  for (int l = 0; l < nlevels; ++l)
    { ::hlq::g_launches++; k_qr_apply_vec2<true><<<level_count[l], 256, 0, st>>>(A, g, k, ib, Ttt, level_pairs[l], nullptr, base); }
}

// TTMQR levels only on the solve's vector (the distributed solve's cross-rank head merges)
void launch_tt_apply(const double* A, Geo g, int k, int ib, const double* Ttt,
                     const int2* const* level_pairs, const int* level_count, int nlevels,
                     double* base, int64_t ldc, int64_t ncols, const uint8_t* dec,
                     cudaStream_t st) {
  (void)ldc;
  (void)dec;
  if (ncols <= 0) return;
  for (int l = 0; l < nlevels; ++l)
    { ::hlq::g_launches++; k_qr_apply_vec2<true><<<level_count[l], 256, 0, st>>>(A, g, k, ib, Ttt, level_pairs[l], nullptr, base); }
}

// Panel stage of a QR step (column block k only): GEQRT of every panel tile, then the TTQRT of
// every level of the greedy tree (a TTQRT only touches panel tiles, so all levels run before any
// trailing update).  Predicated on dec[k] (speculative launches also run while it is undecided).
void launch_qr_panel(double* A, Geo g, int k, int ib, const int2* const* level_pairs,
                     const int* level_count, int nlevels, const DevWork& w, cudaStream_t st,
                     bool diag_done, bool spec, const QRTsPlan* ts, const QRDag* dag,
                     int* progress, int epoch) {
  const uint8_t* dec = w.dec;
  if (dag != nullptr && dag->nops > 0) {  // GEQRTs, TS chains and TT levels as one DAG launch
    launch_qr_panel_dag(A, g, k, ib, w.Tg, w.Ttt, dag->ops, dag->nops, progress, epoch, dec, st,
                        spec, diag_done);
    return;
  }
  if (ts != nullptr && ts->ngroups > 0) {
    // HQR: GEQRT of the group heads (A2: the head k is done), then every group's TSQRT chain
    const int skip = (diag_done && ts->nheads > 0) ? 1 : 0;  // heads[0] == k
    launch_geqrt_rows(A, g, k, ib, w.Tg, ts->heads + skip, ts->nheads - skip, dec, st, spec);
    launch_tsqrt_chains(A, g, k, ib, w.Ttt, ts->pairs, ts->off, ts->ngroups, dec, st, spec);
  } else {
    launch_qr_panel_tc(A, g, k, ib, w.Tg, w.Ttt, nullptr, 0, dec, false, st,
                       diag_done ? k + 1 : k, spec);
  }
  for (int l = 0; l < nlevels; ++l)
    launch_qr_panel_tc(A, g, k, ib, w.Tg, w.Ttt, level_pairs[l], level_count[l], dec, true, st, -1,
                       spec);
}

// Update stage of a QR step on the trailing columns [c0, c1): UNMQR of every tile row, then the
// TTMQR of every level in order.  Predicated on dec[k] == QR.
bool launch_qr_update(double* A, Geo g, int k, int ib, const int2* const* level_pairs,
                      const int* level_count, int nlevels, const DevWork& w, int64_t c0,
                      int64_t c1, cudaStream_t st, double* gmax, const QRTsPlan* ts) {
  const uint8_t* dec = w.dec;
  const int64_t ncols = c1 - c0;
  if (ncols <= 0) return true;
  const bool hqr = ts != nullptr && ts->ngroups > 0;
  bool fused = gmax != nullptr && (nlevels > 0 || hqr);
  double* base = A + c0 * g.lda;
  if (hqr) {
    // HQR: UNMQR of the group heads, then the TSMQR chains (a12 fused: every TS-eliminated row is
    // final after its pair, every head after its TT merge)
    launch_unmqr_rows(A, g, k, w.Tg, ts->heads, ts->nheads, base, g.lda, ncols, dec, st);
    launch_tsmqr_chains(A, g, k, w.Ttt, ts->pairs, ts->off, ts->ngroups, base, g.lda, ncols, dec,
                        st, gmax);
  } else {
    launch_qr_update_dmma(A, g, k, ib, w.Tg, w.Ttt, level_pairs, level_count, nlevels, base,
                          g.lda, ncols, dec, 0, st);
  }
  for (int l = 0; l < nlevels; ++l)
    fused &= launch_qr_update_dmma(A, g, k, ib, w.Tg, w.Ttt, level_pairs, level_count, nlevels,
                                   base, g.lda, ncols, dec, 1 + l, st, gmax);
  return fused;
}

}  // namespace hlq
