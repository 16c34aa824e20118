// FP64 tensor-core (DMMA) QR panel kernels: GEQRT (a8) and TTQRT (a11) of the panel tiles, one CTA
// per tile / TT pair (Alg. 4, Alg. 4b).  Per 32-column reflector block the CTA
// factors the block (panel_factor, registers + warp shuffles) and applies the block reflector to
// the tile's remaining columns in W-column slabs:
//     GEMM1 (DMMA)  Wb = [C1_b +] V_b^T C          32 x W,  K = rows of V_b
//     TRMM  (DFMA)  U  = T_b^T Wb                   32 x W,  T_b upper triangular
//     GEMM2 (DMMA)  C -= V_b U   (TT: C1_b -= U)     rows x W, K = 32
// V_b is staged in shared memory with its structure made explicit (unit diagonal / zeros above for
// GEQRT reflectors, zeros below the diagonal for the TT reflectors), so both GEMMs are dense.
// Fragments: mma.sync.m8n8k4.f64 (lane g=lane/4, t=lane%4: A(g,t), B(t,g), C(g,2t..2t+1)); every
// operand array has a leading dimension == 4 (mod 16) doubles, which makes all fragment loads
// bank-conflict free.
#include <stdlib.h>

#include <type_traits>

#include "hlq_internal.cuh"

namespace hlq {

constexpr int QD_T = 256;  // 8 warps
constexpr int LDU = 36;    // 32 (+4) leading dimension of the 32 x W work arrays

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cpa16(void* smem, const void* gmem) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cpa8(void* smem, const void* gmem) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cpa_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
}

// Block-granular dependencies of the panel DAG (k_qr_panel_dag below): an op publishes, after each
// 32-column reflector block, how many blocks it has finished (release); an op waits before block b
// until its predecessors on the same tile rows have finished block b (acquire).  NoSync: the
// level-by-level launches, where stream order is the dependency.
struct NoSync {
  static constexpr bool dag = false;
  __device__ void before(int) const {}
  __device__ void after(int) const {}
};
struct DagSync {
  static constexpr bool dag = true;
  int* progress;  // per op of this launch: base + finished blocks
  int me, pe, pi;  // this op, the previous op on the eliminator / head row, on the eliminated row
  int base;        // launch epoch << 8
  __device__ void before(int b) const {
    if (threadIdx.x == 0) {
      const int want = base + b + 1;
      if (pe >= 0)
        while (ld_acquire_i(progress + pe) < want) __nanosleep(64);
      if (pi >= 0)
        while (ld_acquire_i(progress + pi) < want) __nanosleep(64);
    }
    __syncthreads();
  }
  __device__ void after(int b) const {  // blocks 0..b are final (b >= 15: the op is complete)
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      st_release_i(progress + me, base + b + 1);
    }
  }
  __device__ static int ld_acquire_i(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
  }
  __device__ static void st_release_i(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  }
};
// data written by another CTA of the same launch is read through L2 only (L1 is not coherent)
template <bool CG>
__device__ __forceinline__ double ldg_dag(const double* p) {
  if constexpr (CG) return __ldcg(p);
  else return *p;
}

// Asynchronous copy of a column block into shared memory (many bytes in flight per thread):
// dst[j*ldd + r] = src[j*lds + r] for r < rows, j < cols_valid; zero for rows_pad > r >= rows and
// for cols_valid <= j < cols_total.  The caller waits (cpa_wait_all) and synchronises.
template <bool CG = false>
__device__ __forceinline__ void cp_cols(double* dst, int ldd, const double* src, int64_t lds,
                                        int rows, int rows_pad, int cols_valid, int cols_total,
                                        int tid, int nthr) {
  const bool v16 = (((uintptr_t)src & 15) == 0) && ((lds & 1) == 0) && ((ldd & 1) == 0) &&
                   (((uintptr_t)dst & 15) == 0) && ((rows_pad & 1) == 0);
  if (v16) {
    const int rp2 = rows_pad >> 1;
    for (int o = tid; o < cols_total * rp2; o += nthr) {
      const int j = o / rp2, r = 2 * (o - j * rp2);
      double* d = dst + j * ldd + r;
      if (j < cols_valid && r + 1 < rows) {
        cpa16(d, src + j * lds + r);
      } else if (j < cols_valid && r < rows) {
        d[0] = ldg_dag<CG>(src + j * lds + r);
        d[1] = 0.0;
      } else {
        d[0] = 0.0;
        d[1] = 0.0;
      }
    }
  } else {
    for (int o = tid; o < cols_total * rows_pad; o += nthr) {
      const int j = o / rows_pad, r = o - j * rows_pad;
      if (j < cols_valid && r < rows) {
        if constexpr (CG)
          dst[j * ldd + r] = __ldcg(src + j * lds + r);
        else
          cpa8(dst + j * ldd + r, src + j * lds + r);
      } else {
        dst[j * ldd + r] = 0.0;
      }
    }
  }
}

__host__ __device__ inline int qd_ldc(int nb) { return (nb + 31) / 32 * 32 + 4; }
// the C slab region; during a panel factorisation it holds the scratch (PF_WS) and R_e's block
__host__ __device__ inline int qd_cs(int W, int nb) {
  const int c = W * qd_ldc(nb);
  constexpr int panel = 2 * 8 * 33 + 64 + 32 * 33 + 32 + 8 * 40 + 32 * 33;  // PF_WS + 32 x 33
  return c > panel ? c : panel;
}

template <int W>
static size_t qd_smem(int nb) {
  const int ldc = qd_ldc(nb);
  // Cs (W x ldc) + Vs (32 x ldc) + Us (W x LDU) + Ts (32 x 33)
  return sizeof(double) * ((size_t)qd_cs(W, nb) + 32 * (size_t)ldc + (size_t)W * LDU + 32 * 33);
}

// GEMM1 + TRMM:  Wb (32 x W) = [C1_b +] Vs^T (32 x RK) * Cs[c_off : c_off + RK, 0:W];
//                U = T_b^T Wb  -> Us (W x LDU, U(l, col) at Us[col*LDU + l]).
// Each n-frag (8 columns) is owned by one warp for all 32 rows, so the triangular T_b^T product
// runs inside the warp (Us doubles as the warp's scratch).  W = 64: warp w owns n-frag w.
// W = 32: warps w and w+4 split K for n-frag w&3; the upper half adds its partial through Us.
// TT (c1 != nullptr): Wb starts from C1_b (read from global) and C1_b <- C1_b - U is written back.
template <int W, bool CG = false>
__device__ __forceinline__ void gemm1_trmm(const double* Vs, const double* Cs, int ldc, int c_off,
                                           int RK, const double* Ts, double* Us, double* c1,
                                           int64_t ldcg, int64_t c0, int64_t ncols, int sb,
                                           int warp, int lane) {
  const int g = lane >> 2, t = lane & 3;
  const int nf = warp & (W / 8 - 1);
  const int khalf = (W == 64) ? 0 : (warp >> 2);
  const int kbeg = (W == 64) ? 0 : khalf * (RK / 2);
  const int kend = (W == 64) ? RK : kbeg + RK / 2;
  double acc[4][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int l = mi * 8 + g;
      int64_t col = c0 + nf * 8 + 2 * t + h;
      acc[mi][h] = (c1 != nullptr && khalf == 0 && l < sb && col < ncols)
                       ? ldg_dag<CG>(c1 + col * ldcg + l) : 0.0;
    }
  const double* cb = Cs + (nf * 8 + g) * ldc + c_off + t;
  const double* vb = Vs + g * ldc + t;
#pragma unroll 4
  for (int kk = kbeg; kk < kend; kk += 4) {
    double b = cb[kk];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) dmma(acc[mi][0], acc[mi][1], vb[mi * 8 * ldc + kk], b);
  }
  if (W == 32) {
    if (khalf == 1)
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int h = 0; h < 2; ++h) Us[(nf * 8 + 2 * t + h) * LDU + mi * 8 + g] = acc[mi][h];
    __syncthreads();
    if (khalf == 1) return;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int h = 0; h < 2; ++h) acc[mi][h] += Us[(nf * 8 + 2 * t + h) * LDU + mi * 8 + g];
    __syncwarp();
  }
  // Wb of this warp's 8 columns -> Us (scratch), then U = T^T Wb in place
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int h = 0; h < 2; ++h) Us[(nf * 8 + 2 * t + h) * LDU + mi * 8 + g] = acc[mi][h];
  __syncwarp();
  // U = T^T Wb on the tensor cores: A = T^T (lower triangular: k-steps kk <= 8 mi + 7 only),
  // B = Wb (this warp's 8 columns from Us)
  double ua[4][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) ua[mi][0] = ua[mi][1] = 0.0;
#pragma unroll
  for (int kk = 0; kk < 32; kk += 4) {
    const double bw = Us[(nf * 8 + g) * LDU + kk + t];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
      if (kk <= 8 * mi + 7) dmma(ua[mi][0], ua[mi][1], Ts[(mi * 8 + g) * 33 + kk + t], bw);
  }
  __syncwarp();
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int h = 0; h < 2; ++h) Us[(nf * 8 + 2 * t + h) * LDU + mi * 8 + g] = ua[mi][h];
  __syncwarp();
  double u[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) u[j] = Us[(nf * 8 + j) * LDU + lane];
  if (c1 != nullptr && lane < sb) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      int64_t col = c0 + nf * 8 + j;
      if (col < ncols) c1[col * ldcg + lane] = ldg_dag<CG>(c1 + col * ldcg + lane) - u[j];
    }
  }
}

// GEMM2: Cs[c_off : c_off + RK, 0:W] -= Vs (RK x 32) * Us (32 x W); macro tiles 32 rows x 16 cols
template <int W>
__device__ __forceinline__ void gemm2(const double* Vs, const double* Us, double* Cs, int ldc,
                                      int c_off, int RK, int warp, int lane) {
  const int g = lane >> 2, t = lane & 3;
  const int nmt_r = RK / 32, nmt_c = W / 16;
  for (int mt = warp; mt < nmt_r * nmt_c; mt += 8) {
    const int r0 = (mt / nmt_c) * 32, n0 = (mt % nmt_c) * 16;
    double acc[4][2][2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          acc[mi][ni][h] = Cs[(n0 + ni * 8 + 2 * t + h) * ldc + c_off + r0 + mi * 8 + g];
#pragma unroll
    for (int kk = 0; kk < 32; kk += 4) {
      double a[4], b[2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = neg_bits(Vs[(kk + t) * ldc + r0 + mi * 8 + g]);
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) b[ni] = Us[(n0 + ni * 8 + g) * LDU + kk + t];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
    }
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          Cs[(n0 + ni * 8 + 2 * t + h) * ldc + c_off + r0 + mi * 8 + g] = acc[mi][ni][h];
  }
}

// ---------------------------------------------------------------------------------------------
// Panel factorisation of one 32-column reflector block by the whole CTA (8 warps): per column l a
// CTA-wide sum of squares (dlarfg, reading 14), the update of the block's remaining
// columns and the T column (dlarft, forward column-wise).  Reductions are warp shuffles followed
// by a fixed-order sum over the 8 warp partials (deterministic).
//   GE (GEQRT): Vs column l holds rows 0..R-1 of the block (local row l is the diagonal);
//               reflector l acts on local rows l..R-1, top element Vs[l][l].
//   TT (TTQRT): top elements in Rs (32 x 33, R(q,l) at Rs[l*33+q]); Vs column l holds rows
//               0..R2-1 of R_i (upper triangular: rows <= i0 + l), the reflector's bottom part.
__device__ __forceinline__ double block_sum(double v, double* red, int tid) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((tid & 31) == 0) red[tid >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < 8; ++w) s += red[w];
  return s;
}

// Register-resident layout: lane c owns column c of the 32-column block and warp w owns the NR
// rows w*NR .. w*NR+NR-1 (NR static), so thread (w, c) holds V[r][c] of its rows in registers and
// the column loop needs no register indexing by l.  Per column l ONE barrier: x_r = V[r][l] is a
// shuffle from lane l, thread (w, c) forms its warp's partial of g[c] = sum_r V[r][c] x_r over
// the reflector's rows, and (GE) the owner of row l publishes that row (the reflector's top
// elements); after the barrier every warp sums the 8 partials itself (fixed order: identical in
// every warp), lane c forms dlarfg and w_c / z_c, and each thread updates its own elements.  The
// T recurrence (dlarft, forward column-wise) runs in warp 0 right after z_l is formed.
// v = x (1 / (alpha - beta)) as LAPACK dlarfg scales.  Scratch ws:
// red [2][8][33] | top [2][32] | Z [32][33] | (unused) [32] | xs [8][40]  (PF_WS doubles).  Column l
// reaches the 32 lanes of a warp through xs (lane l stores its NR values, 16-byte broadcasts back).
constexpr int PF_WS = 2 * 8 * 33 + 64 + 32 * 33 + 32 + 8 * 40;

// FULL (TT only): the eliminated tile is square (TSQRT): every reflector spans all R rows
template <bool TT, int NR, bool FULL = false>
__device__ void panel_factor(double* Vs, int ldc, double* Rs, double* Ts, int R, int i0, int sb,
                             double* ws, int tid) {
  const int lane = tid & 31, warp = tid >> 5;
  double* red = ws;
  double* top = ws + 2 * 8 * 33;
  double* Z = top + 64;
  double* tauv = Z + 32 * 33;
  double* xs = tauv + 32 + warp * 40;  // this warp's copy of column l (16-byte aligned)
  const int rw = warp * NR;  // first row of this warp
  const int lmax = TT ? sb : min(sb, R);
  int pl = -1;  // TT, warp 0: the pending R_e row update
  double ptau = 0.0, pwz = 0.0, pbeta = 0.0;
  double a[NR];
#pragma unroll
  for (int i = 0; i < NR; ++i) a[i] = (rw + i < R && lane < sb) ? Vs[lane * ldc + rw + i] : 0.0;
#pragma unroll 1
  for (int l = 0; l < lmax; ++l) {
    const int bf = l & 1;
    // reflector rows: GE below the diagonal (l, R), TT the upper-triangle rows [0, min(R, i0+l+1)),
    // TS (FULL) all rows [0, R)
    const int rlo = TT ? 0 : l + 1;
    const int rhi = TT ? (FULL ? R : min(R, i0 + l + 1)) : R;
    // this warp's reflector rows are i in [ilo, ihi) (warp-uniform; empty for most warps early on)
    const int ilo = max(0, rlo - rw), ihi = min(NR, rhi - rw);
    const bool wact = ilo < ihi;
    double part = 0.0;
    if (wact) {
      __syncwarp();  // the previous column's reads of xs are done
      if (lane == l) {
#pragma unroll
        for (int i = 0; i < NR; i += 2)
          *reinterpret_cast<double2*>(xs + i) = make_double2(a[i], a[i + 1]);
      }
      __syncwarp();
      // four independent FMA chains (NR is a multiple of 4): the dot product's latency is on the
      // critical path of every column
      double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
      if (ilo == 0 && ihi == NR) {  // every row of the warp (no per-row predicates)
#pragma unroll
        for (int i = 0; i < NR; i += 4) {
          const double2 x = *reinterpret_cast<const double2*>(xs + i);
          const double2 y = *reinterpret_cast<const double2*>(xs + i + 2);
          p0 = fma(a[i], x.x, p0);
          p1 = fma(a[i + 1], x.y, p1);
          p2 = fma(a[i + 2], y.x, p2);
          p3 = fma(a[i + 3], y.y, p3);
        }
      } else {
#pragma unroll
        for (int i = 0; i < NR; i += 4) {
          const double2 x = *reinterpret_cast<const double2*>(xs + i);
          const double2 y = *reinterpret_cast<const double2*>(xs + i + 2);
          if (i >= ilo && i < ihi) p0 = fma(a[i], x.x, p0);
          if (i + 1 >= ilo && i + 1 < ihi) p1 = fma(a[i + 1], x.y, p1);
          if (i + 2 >= ilo && i + 2 < ihi) p2 = fma(a[i + 2], y.x, p2);
          if (i + 3 >= ilo && i + 3 < ihi) p3 = fma(a[i + 3], y.y, p3);
        }
      }
      part = (p0 + p1) + (p2 + p3);
    }
    red[(bf * 8 + warp) * 33 + lane] = part;
    if (!TT && l >= rw && l < rw + NR) {
#pragma unroll
      for (int i = 0; i < NR; ++i)
        if (rw + i == l) top[bf * 32 + lane] = a[i];
    }
    __syncthreads();
    // the 8 warp partials as a fixed tree (the same order in every warp: identical gsum)
    const double* rp = red + bf * 8 * 33 + lane;
    const double gsum = ((rp[0] + rp[33]) + (rp[2 * 33] + rp[3 * 33])) +
                        ((rp[4 * 33] + rp[5 * 33]) + (rp[6 * 33] + rp[7 * 33]));
    const double ssq = __shfl_sync(0xffffffffu, gsum, l);
    const double alpha = TT ? Rs[l * 33 + l] : top[bf * 32 + l];
    double tau = 0.0, beta = alpha, rsc = 0.0;
    if (ssq != 0.0) {
      const double nrm = sqrt(alpha * alpha + ssq);
      beta = alpha >= 0.0 ? -nrm : nrm;
      // two independent correctly rounded divisions (dlarfg's tau and 1 / (alpha - beta))
      tau = __ddiv_rn(beta - alpha, beta);
      rsc = __drcp_rn(alpha - beta);
    }
    // lane c: w_c = top_c + V_c . v (c > l), z_q = [V_q(l)] + V_q . v (q < l)
    double topc = 0.0;
    if (TT) {
      if (lane > l) topc = Rs[lane * 33 + l];
    } else {
      topc = top[bf * 32 + lane];
    }
    const double wz = topc + gsum * rsc;
    if (TT && warp == 0) {
      // R_e row l (Rs[c*33 + l], c >= l) is written one column late: every warp reads it in this
      // column (alpha, top_c) and the next barrier orders the write after those reads
      if (pl >= 0) {
        if (lane > pl && lane < sb && ptau != 0.0) Rs[lane * 33 + pl] -= ptau * pwz;
        if (lane == 0) Rs[pl * 33 + pl] = pbeta;
      }
      pl = l;
      ptau = tau;
      pwz = wz;
      pbeta = beta;
    }
    if (warp == 7) {  // the highest rows: idle for most TT columns
      if (lane < l) Z[l * 33 + lane] = wz;
      __syncwarp();
      // T(q, l) = -tau sum_{p = q}^{l-1} T(q, p) z_p (q < l), T(l, l) = tau: four FMA chains
      if (lane < l) {
        double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
        int p2 = lane;
        for (; p2 + 3 < l; p2 += 4) {
          t0 += Ts[p2 * 33 + lane] * Z[l * 33 + p2];
          t1 += Ts[(p2 + 1) * 33 + lane] * Z[l * 33 + p2 + 1];
          t2 += Ts[(p2 + 2) * 33 + lane] * Z[l * 33 + p2 + 2];
          t3 += Ts[(p2 + 3) * 33 + lane] * Z[l * 33 + p2 + 3];
        }
        for (; p2 < l; ++p2) t0 += Ts[p2 * 33 + lane] * Z[l * 33 + p2];
        Ts[l * 33 + lane] = -tau * ((t0 + t1) + (t2 + t3));
      }
      if (lane == 0) Ts[l * 33 + l] = tau;
    }
    const bool upd = lane > l && lane < sb && tau != 0.0;
    if (wact && (lane == l || upd)) {
      // lane l stores v = x / (alpha - beta) = fma(x, rsc, 0); lanes c > l apply
      // a -= tau (x / (alpha - beta)) w_c = fma(x, -c, a), c = tau w_c / (alpha - beta): one code path
      // for both (no divergent passes), a select feeding the addend
      const bool own = lane == l;
      const double co = own ? rsc : -(tau * wz * rsc);
      if (ilo == 0 && ihi == NR) {
#pragma unroll
        for (int i = 0; i < NR; ++i) a[i] = fma(xs[i], co, own ? 0.0 : a[i]);
      } else {
#pragma unroll
        for (int i = 0; i < NR; ++i)
          if (i >= ilo && i < ihi) a[i] = fma(xs[i], co, own ? 0.0 : a[i]);
      }
    }
    if (!TT && l >= rw && l < rw + NR) {  // row l: the R row of reflector l
#pragma unroll
      for (int i = 0; i < NR; ++i)
        if (rw + i == l) {
          if (lane == l) a[i] = beta;
          else if (upd) a[i] -= tau * wz;
        }
    }
  }
#pragma unroll
  for (int i = 0; i < NR; ++i)
    if (rw + i < R && lane < sb) Vs[lane * ldc + rw + i] = a[i];
  __syncthreads();
  if (TT && warp == 0 && pl >= 0) {
    if (lane > pl && lane < sb && ptau != 0.0) Rs[lane * 33 + pl] -= ptau * pwz;
    if (lane == 0) Rs[pl * 33 + pl] = pbeta;
  }
  if (TT) __syncthreads();
}

// rows per warp for a block of R <= nb rows (one kernel for every NR: measured faster than
// per-NR kernels, whose smaller register allocations throttle the DMMA block updates)
template <bool TT, bool FULL = false>
__device__ __forceinline__ void panel_factor_nb(int nb, double* Vs, int ldc, double* Rs,
                                                double* Ts, int R, int i0, int sb, double* ws,
                                                int tid) {
  if (nb <= 64) panel_factor<TT, 8, FULL>(Vs, ldc, Rs, Ts, R, i0, sb, ws, tid);
  else if (nb <= 128) panel_factor<TT, 16, FULL>(Vs, ldc, Rs, Ts, R, i0, sb, ws, tid);
  else if (nb <= 192) panel_factor<TT, 24, FULL>(Vs, ldc, Rs, Ts, R, i0, sb, ws, tid);
  else if (nb <= 256) panel_factor<TT, 32, FULL>(Vs, ldc, Rs, Ts, R, i0, sb, ws, tid);
  else panel_factor<TT, 40, FULL>(Vs, ldc, Rs, Ts, R, i0, sb, ws, tid);
}

// GEQRT of tiles (k + blockIdx.x, k) on tensor cores: per 32-column block, CTA-wide panel
// factorisation, then the block reflector is applied to the tile's remaining columns in W-column
// slabs with the same DMMA GEMM1+TRMM / GEMM2 as UNMQR.
template <int W, class SYNC>
__device__ void geqrt_tile(double* __restrict__ A, Geo g, int k, int ib, double* __restrict__ Tg,
                           int i, double* sm, const SYNC& sync) {
  constexpr bool CG = SYNC::dag;
  const int ldc = qd_ldc(g.nb);
  double* Cs = sm;
  double* Vs = Cs + qd_cs(W, g.nb);
  double* Us = Vs + 32 * ldc;
  double* Ts = Us + W * LDU;
  const int bi = g.bs(i), bk = g.cbs(k);
  double* tile = g.tile(A, i, k);
  double* T = Tg + tri_index(i, k, g.n) * (int64_t)ib * g.nb;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int t = tid; t < ib * g.nb; t += QD_T) T[t] = 0.0;
  for (int i0 = 0; i0 < bk; i0 += ib) {
    const int sb = min(ib, bk - i0);
    const int R = bi - i0;
    if (R <= 0) break;
    const int RK = (R + 31) / 32 * 32;
    __syncthreads();
    cp_cols<CG>(Vs, ldc, tile + (int64_t)i0 * g.lda + i0, g.lda, R, RK, sb, 32, tid, QD_T);
    for (int o = tid; o < 32 * 33; o += QD_T) Ts[o] = 0.0;
    cpa_wait_all();
    __syncthreads();
    panel_factor_nb<false>(g.nb, Vs, ldc, nullptr, Ts, R, i0, sb, Cs, tid);
    for (int o = tid; o < sb * R; o += QD_T) {
      int l = o / R, r = o - l * R;
      tile[(int64_t)(i0 + l) * g.lda + i0 + r] = Vs[l * ldc + r];
    }
    for (int o = tid; o < sb * sb; o += QD_T) {
      int l = o / sb, q = o - l * sb;
      T[(int64_t)(i0 + l) * ib + q] = Ts[l * 33 + q];
    }
    __syncthreads();
    if (i0 + sb >= bk) break;
    for (int o = tid; o < 32 * 32; o += QD_T) {  // explicit unit-lower structure for the GEMMs
      int l = o >> 5, r = o & 31;
      if (r <= l && r < RK) Vs[l * ldc + r] = (r == l && l < sb && r < R) ? 1.0 : 0.0;
    }
    for (int c0 = i0 + sb; c0 < bk; c0 += W) {
      const int cv = min(W, bk - c0);
      __syncthreads();
      cp_cols(Cs, ldc, tile + (int64_t)c0 * g.lda + i0, g.lda, R, RK, cv, W, tid, QD_T);
      cpa_wait_all();
      __syncthreads();
      gemm1_trmm<W>(Vs, Cs, ldc, 0, RK, Ts, Us, nullptr, 0, 0, 0, sb, warp, lane);
      __syncthreads();
      gemm2<W>(Vs, Us, Cs, ldc, 0, RK, warp, lane);
      __syncthreads();
      for (int o = tid; o < cv * R; o += QD_T) {
        int j = o / R, r = o - j * R;
        tile[(int64_t)(c0 + j) * g.lda + i0 + r] = Cs[j * ldc + r];
      }
    }
    // block-row i0 / ib is final: its reflectors' trailing update is written
    sync.after(i0 / ib);
  }
  sync.after(15);  // every block (also after an early exit of a ragged tile)
}

template <int W>
__global__ void __launch_bounds__(QD_T) k_geqrt_tc(double* __restrict__ A, Geo g, int k, int ib,
                                                   double* __restrict__ Tg,
                                                   const uint8_t* __restrict__ dec, int i_first,
                                                   int spec, const int* __restrict__ rows) {
  // predicated on d_k == QR; a speculative launch (spec) also runs while d_k is undecided
  if (dec != nullptr && (spec ? dec[k] == HLQ_DEC_LU : dec[k] != HLQ_DEC_QR)) return;
  extern __shared__ __align__(16) double sm[];
  const int i = rows != nullptr ? rows[blockIdx.x] : i_first + blockIdx.x;
  geqrt_tile<W>(A, g, k, ib, Tg, i, sm, NoSync{});
}

// TTQRT (TS = false) / TSQRT (TS = true) of the pair (e, i): [R_e; A_i] -> R_e, the
// reflectors V in tile (i,k) (TT: its upper triangle; TS: the whole square tile), T
template <int W, bool TS, class SYNC = NoSync>
__device__ void qrt_pair(double* __restrict__ A, Geo g, int k, int ib, double* __restrict__ Ttt,
                         int e, int i, double* sm, const SYNC& sync = SYNC{}) {
  constexpr bool CG = SYNC::dag;
  const int ldc = qd_ldc(g.nb);
  double* Cs = sm;
  double* Vs = Cs + qd_cs(W, g.nb);
  double* Us = Vs + 32 * ldc;
  double* Ts = Us + W * LDU;
  double* Rs = Cs + PF_WS;       // panel phase: Cs holds the panel scratch, then R_e's block
  const int bi = g.bs(i), bk = g.cbs(k);
  double* Re = g.tile(A, e, k);
  double* Ri = g.tile(A, i, k);
  double* T = Ttt + tri_index(i, k, g.n) * (int64_t)ib * g.nb;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int t = tid; t < ib * g.nb; t += QD_T) T[t] = 0.0;
  for (int i0 = 0; i0 < bk; i0 += ib) {
    const int sb = min(ib, bk - i0);
    const int R2 = TS ? bi : min(bi, i0 + sb);
    const int RK = (R2 + 31) / 32 * 32;
    sync.before(i0 / ib);  // the predecessors' block rows 0 .. i0 / ib are final
    __syncthreads();
    cp_cols<CG>(Vs, ldc, Ri + (int64_t)i0 * g.lda, g.lda, R2, RK, sb, 32, tid, QD_T);
    for (int o = tid; o < 32 * 33; o += QD_T) {
      Ts[o] = 0.0;
      int l = o / 33, q = o - l * 33;
      if (l < sb && q <= l) {  // R_e's block triangle, in flight with V's block
        if constexpr (CG)
          Rs[o] = __ldcg(Re + (int64_t)(i0 + l) * g.lda + i0 + q);
        else
          cpa8(Rs + o, Re + (int64_t)(i0 + l) * g.lda + i0 + q);
      } else {
        Rs[o] = 0.0;
      }
    }
    cpa_wait_all();
    __syncthreads();
    if (!TS) {
      for (int o = tid; o < 32 * RK; o += QD_T) {
        int l = o / RK, r = o - l * RK;
        if (r > i0 + l) Vs[l * ldc + r] = 0.0;
      }
      __syncthreads();
    }
    panel_factor_nb<true, TS>(g.nb, Vs, ldc, Rs, Ts, R2, i0, sb, Cs, tid);
    for (int o = tid; o < sb * R2; o += QD_T) {
      int l = o / R2, r = o - l * R2;
      if (TS || r <= i0 + l) Ri[(int64_t)(i0 + l) * g.lda + r] = Vs[l * ldc + r];
    }
    for (int o = tid; o < sb * sb; o += QD_T) {
      int l = o / sb, q = o - l * sb;
      if (q <= l) Re[(int64_t)(i0 + l) * g.lda + i0 + q] = Rs[l * 33 + q];
      T[(int64_t)(i0 + l) * ib + q] = Ts[l * 33 + q];
    }
    __syncthreads();
    if (i0 + sb >= bk) break;
    for (int c0 = i0 + sb; c0 < bk; c0 += W) {
      const int cv = min(W, bk - c0);
      __syncthreads();
      cp_cols<CG>(Cs, ldc, Ri + (int64_t)c0 * g.lda, g.lda, R2, RK, cv, W, tid, QD_T);
      cpa_wait_all();
      __syncthreads();
      // Wb = R_e(block rows, slab) + V2^T R_i(slab); U = T^T Wb; R_e(block rows) -= U
      gemm1_trmm<W, CG>(Vs, Cs, ldc, 0, RK, Ts, Us, Re + i0, g.lda, c0, bk, sb, warp, lane);
      __syncthreads();
      gemm2<W>(Vs, Us, Cs, ldc, 0, RK, warp, lane);
      __syncthreads();
      for (int o = tid; o < cv * R2; o += QD_T) {
        int j = o / R2, r = o - j * R2;
        Ri[(int64_t)(c0 + j) * g.lda + r] = Cs[j * ldc + r];
      }
    }
    __syncthreads();
    sync.after(i0 / ib);  // the eliminator's block row i0 / ib is final
  }
  sync.after(15);
}

// TTQRT on pairs (e, i) = pairs[blockIdx.x]: [R_e; R_i] -> R_e, V (upper triangle of tile (i,k)), T
template <int W>
__global__ void __launch_bounds__(QD_T) k_ttqrt_tc(double* __restrict__ A, Geo g, int k, int ib,
                                                   double* __restrict__ Ttt,
                                                   const int2* __restrict__ pairs,
                                                   const uint8_t* __restrict__ dec, int spec) {
  if (dec != nullptr && (spec ? dec[k] == HLQ_DEC_LU : dec[k] != HLQ_DEC_QR)) return;
  extern __shared__ __align__(16) double sm[];
  const int2 pr = pairs[blockIdx.x];
  qrt_pair<W, false>(A, g, k, ib, Ttt, pr.x, pr.y, sm);
}

// TSQRT chains (Alg. 4a): CTA = one group of the HQR tree; its pairs (head, i) =
// pairs[off[blockIdx.x] .. off[blockIdx.x + 1]) in order, each killing the square tile i with the
// head's R (the head's R row stays in L2 between the pairs of the chain)
template <int W>
__global__ void __launch_bounds__(QD_T) k_tsqrt_tc(double* __restrict__ A, Geo g, int k, int ib,
                                                   double* __restrict__ Tts,
                                                   const int2* __restrict__ pairs,
                                                   const int* __restrict__ off,
                                                   const uint8_t* __restrict__ dec, int spec) {
  if (dec != nullptr && (spec ? dec[k] == HLQ_DEC_LU : dec[k] != HLQ_DEC_QR)) return;
  extern __shared__ __align__(16) double sm[];
  for (int p = off[blockIdx.x]; p < off[blockIdx.x + 1]; ++p) {
    const int2 pr = pairs[p];
    qrt_pair<W, true>(A, g, k, ib, Tts, pr.x, pr.y, sm);
    __syncthreads();
  }
}

// The whole QR panel of a step as ONE launch (GEQRT of the listed tiles, every TS chain pair, every
// TT level pair): one CTA per op (ops = 5 ints each: kind 0 GEQRT / 1 TSQRT / 2 TTQRT, eliminator or
// head row e, row i, the previous op on row e and on row i, -1 = none), listed in an order where
// every predecessor precedes its successors.  An op starts block b once its predecessors have
// finished block b (DagSync), so a TS chain or the next TT level trails its predecessor by one
// 32-column block instead of one whole kernel: the panel's critical path becomes
// (blocks + chain length + levels) block times.  Waiting CTAs only wait for CTAs with smaller
// indices, which are dispatched first, so the spin waits cannot deadlock.
template <int W>
__global__ void __launch_bounds__(QD_T) k_qr_panel_dag(double* __restrict__ A, Geo g, int k, int ib,
                                                       double* __restrict__ Tg,
                                                       double* __restrict__ Ttt,
                                                       const int* __restrict__ ops,
                                                       int* __restrict__ progress, int base,
                                                       const uint8_t* __restrict__ dec, int spec,
                                                       int skip_first) {
  if (dec != nullptr && (spec ? dec[k] == HLQ_DEC_LU : dec[k] != HLQ_DEC_QR)) return;
  extern __shared__ __align__(16) double sm[];
  const int* op = ops + 5 * blockIdx.x;
  const DagSync sync{progress, (int)blockIdx.x, op[3], op[4], base};
  if (blockIdx.x == 0 && skip_first) {  // (A2) the caller already factored tile k
    sync.after(15);
    return;
  }
  if (op[0] == 0)
    geqrt_tile<W>(A, g, k, ib, Tg, op[2], sm, sync);
  else if (op[0] == 1)
    qrt_pair<W, true>(A, g, k, ib, Ttt, op[1], op[2], sm, sync);
  else
    qrt_pair<W, false>(A, g, k, ib, Ttt, op[1], op[2], sm, sync);
}

void launch_qr_panel_dag(double* A, Geo g, int k, int ib, double* Tg, double* Ttt, const int* ops,
                         int nops, int* progress, int epoch, const uint8_t* dec, cudaStream_t st,
                         bool spec, bool skip_first) {
  if (nops <= 0) return;
  auto go = [&](auto W_) {
    constexpr int W = decltype(W_)::value;
    static unsigned long long attr = 0;
    if (first_on_device(attr)) smem_optin(k_qr_panel_dag<W>);
    ::hlq::g_launches++;
    k_qr_panel_dag<W><<<nops, QD_T, qd_smem<W>(g.nb), st>>>(A, g, k, ib, Tg, Ttt, ops, progress,
                                                           epoch << 8, dec, spec ? 1 : 0,
                                                           skip_first ? 1 : 0);
  };
  if (qd_smem<64>(g.nb) <= 227 * 1024) go(std::integral_constant<int, 64>());
  else go(std::integral_constant<int, 32>());
}

template <int W>
static void launch_panel_w(double* A, Geo g, int k, int ib, double* Tg, double* Ttt,
                           const int2* pairs, int npairs, const uint8_t* dec, bool tt,
                           cudaStream_t st, int i_first, bool spec) {
  static unsigned long long attr = 0;
  if (first_on_device(attr)) {
    smem_optin(k_geqrt_tc<W>);
    smem_optin(k_ttqrt_tc<W>);
  }
  const size_t smem = qd_smem<W>(g.nb);
  if (!tt) {
    if (g.n - i_first <= 0) return;
    { ::hlq::g_launches++; k_geqrt_tc<W><<<g.n - i_first, QD_T, smem, st>>>(A, g, k, ib, Tg, dec, i_first, spec ? 1 : 0, nullptr); }
  } else {
    { ::hlq::g_launches++; k_ttqrt_tc<W><<<npairs, QD_T, smem, st>>>(A, g, k, ib, Ttt, pairs, dec, spec ? 1 : 0); }
  }
}

void launch_qr_panel_tc(double* A, Geo g, int k, int ib, double* Tg, double* Ttt,
                        const int2* pairs, int npairs, const uint8_t* dec, bool tt,
                        cudaStream_t st, int i_first, bool spec) {
  if (i_first < 0) i_first = k;
  if (qd_smem<64>(g.nb) <= 227 * 1024)
    launch_panel_w<64>(A, g, k, ib, Tg, Ttt, pairs, npairs, dec, tt, st, i_first, spec);
  else
    launch_panel_w<32>(A, g, k, ib, Tg, Ttt, pairs, npairs, dec, tt, st, i_first, spec);
}

// GEQRT of the listed tile rows (the HQR tree's group heads), predicated as launch_qr_panel_tc
void launch_geqrt_rows(double* A, Geo g, int k, int ib, double* Tg, const int* rows, int nrows,
                       const uint8_t* dec, cudaStream_t st, bool spec) {
  if (nrows <= 0) return;
  auto go = [&](auto W_) {
    constexpr int W = decltype(W_)::value;
    static unsigned long long attr = 0;
    if (first_on_device(attr)) smem_optin(k_geqrt_tc<W>);
    ::hlq::g_launches++;
    k_geqrt_tc<W><<<nrows, QD_T, qd_smem<W>(g.nb), st>>>(A, g, k, ib, Tg, dec, 0, spec ? 1 : 0,
                                                          rows);
  };
  if (qd_smem<64>(g.nb) <= 227 * 1024) go(std::integral_constant<int, 64>());
  else go(std::integral_constant<int, 32>());
}

// TSQRT chains of the HQR tree: one CTA per group (pairs[off[g] .. off[g+1]) in order)
void launch_tsqrt_chains(double* A, Geo g, int k, int ib, double* Tts, const int2* pairs,
                         const int* off, int ngroups, const uint8_t* dec, cudaStream_t st,
                         bool spec) {
  if (ngroups <= 0) return;
  auto go = [&](auto W_) {
    constexpr int W = decltype(W_)::value;
    static unsigned long long attr = 0;
    if (first_on_device(attr)) smem_optin(k_tsqrt_tc<W>);
    ::hlq::g_launches++;
    k_tsqrt_tc<W><<<ngroups, QD_T, qd_smem<W>(g.nb), st>>>(A, g, k, ib, Tts, pairs, off, dec,
                                                            spec ? 1 : 0);
  };
  if (qd_smem<64>(g.nb) <= 227 * 1024) go(std::integral_constant<int, 64>());
  else go(std::integral_constant<int, 32>());
}

// what = 0: UNMQR of all tile rows; what = 1 + l: TTMQR of level l (qr_update.cu, register-slab
// DMMA kernel; ib = 32).  Returns whether the a12 scan was fused (TTMQR levels with gmax).
bool launch_qr_update_dmma(const double* A, Geo g, int k, int ib, const double* Tg,
                           const double* Ttt, const int2* const* level_pairs,
                           const int* level_count, int nlevels, double* base, int64_t ldc,
                           int64_t ncols, const uint8_t* dec, int what, cudaStream_t st,
                           double* gmax) {
  (void)ib;
  (void)nlevels;
  if (ncols <= 0) return true;
  if (what == 0)
    return launch_qr_update2(A, g, k, Tg, nullptr, 0, false, base, ldc, ncols, dec, st);
  return launch_qr_update2(A, g, k, Ttt, level_pairs[what - 1], level_count[what - 1], true, base,
                           ldc, ncols, dec, st, gmax);
}

}  // namespace hlq
