// QR trailing update (a8 UNMQR, a10/a11 TTMQR): the bulk of a QR step's flops (Table I "update D"
// PAPER.md:166; Alg. 4b), on the FP64 tensor cores (DMMA).  One CTA owns a column slab of
// one tile row (UNMQR) or of the eliminated tile of one TT pair (TTMQR) for the whole step and
// keeps it in REGISTERS as C^T accumulator fragments (design below, "v3"); every C element is read
// and written once per launch.  Householder convention and T layout: DESIGN.md readings 14-15.
#include <stdio.h>
#include <stdlib.h>

#include "hlq_internal.cuh"

namespace hlq {

namespace {

__device__ __forceinline__ void dmma_(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp16(void* s, const void* g, bool v) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  int sz = v ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(sz));
}
__device__ __forceinline__ void cp8(void* s, const void* g, bool v) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  int sz = v ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(sz));
}
// the same with a 32-bit shared-window address (no generic -> shared conversion per copy)
__device__ __forceinline__ void cp16s(unsigned sa, const void* g, bool v) {
  int sz = v ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(sz));
}
__device__ __forceinline__ void cp8s(unsigned sa, const void* g, bool v) {
  int sz = v ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(sz));
}
__device__ __forceinline__ void commit_() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void wait_() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

}  // namespace

bool launch_qr_update3(const double* A, Geo g, int k, const double* T, const int2* pairs,
                       int npairs, int mode, const int* list, double* base, int64_t ldc,
                       int64_t ncols, const uint8_t* dec, cudaStream_t st, double* gmax);

// UNMQR of every tile row k..n-1 (tt = false, T = GEQRT factors) or TTMQR of one level (tt = true,
// T = TTQRT factors) on the column block (base, ldc, ncols); returns whether the a12 scan was fused
bool launch_qr_update2(const double* A, Geo g, int k, const double* T, const int2* pairs,
                       int npairs, bool tt, double* base, int64_t ldc, int64_t ncols,
                       const uint8_t* dec, cudaStream_t st, double* gmax) {
  if (ncols <= 0) return true;
  const bool ok = tt ? launch_qr_update3(A, g, k, T, pairs, npairs, 1, nullptr, base, ldc, ncols,
                                         dec, st, gmax)
                     : launch_qr_update3(A, g, k, T, nullptr, g.n - k, 0, nullptr, base, ldc,
                                         ncols, dec, st, nullptr);
  if (!ok) {
    fprintf(stderr, "[hlq] QR update: nb = %d has no register-slab instantiation\n", g.nb);
    abort();
  }
  return tt && gmax != nullptr;
}

// =============================================================================================
// v3: the slab lives in REGISTERS as C^T accumulator fragments.
//
// A DMMA accumulator fragment of an 8x8 block X holds X(g, 2t) and X(g, 2t+1) in lane (g, t); the
// two registers are exactly the A-operand fragments (lane (g,t) -> A(g,t)) of the 8x4 matrices
// X[:, even columns] and X[:, odd columns].  Holding C^T (slab columns x tile rows) as accumulators:
//     GEMM1  W^T  = C^T V_b        A = C^T from registers (even / odd rows), B = V_b from smem
//     TRMM   U^T  = W^T T_b        A = W^T from registers,                    B = T_b from smem
//     GEMM2  C^T -= U^T V_b^T      A = U^T from registers,                    B = V_b from smem
// so the only shared-memory traffic is the B operand (0.5 LDS per DMMA: every B fragment feeds the
// two 8-column halves of a warp's 16 slab columns) and C never round-trips through shared memory.
// 8 warps: column group cg = warp & 3 (16 columns), row parity rh = warp >> 2 (the 8-row blocks
// RB == rh mod 2 of the tile).  GEMM1 partials of the two row parities are pair-reduced (W = P0+P1,
// commutative, so both warps hold identical W) and both compute the (tiny) TRMM.  V_b row chunks
// (32 x 32) stream through a cp.async ring in a pass-specific permuted layout that makes every B
// fragment load bank-conflict free.
namespace {
constexpr int LD3 = 40;    // GEMM1 / T chunks: == 8 (mod 16): conflict-free 16-byte fragment pairs
constexpr int LD3B = 34;   // GEMM2 chunks: == 2 (mod 16): conflict-free 8-byte B fragments
constexpr int CH3 = 32 * LD3;
__device__ __forceinline__ double2 lds2(const double* p) {
  return *reinterpret_cast<const double2*>(p);
}
}  // namespace

// MODE 0: UNMQR of tile row i (GEQRT reflectors, unit lower); 1: TTMQR of the pair (e, i) (TT
// reflectors, upper triangular); 2: TSMQR of the pair (e, i) (TS reflectors, square)
template <int NB, int MODE, int RQ, int NCG, bool V16>
__device__ __forceinline__ void qr_update3_body(const double* __restrict__ A, Geo g, int k,
                                                const double* __restrict__ Tbase, int e, int i,
                                                double* __restrict__ base, int64_t ldcg,
                                                int64_t ncols, double* __restrict__ gmax) {
  constexpr bool TT = MODE != 0;  // pair modes: the eliminator's rows C_e are read-modify-written
  constexpr bool TS = MODE == 2;
  constexpr int NCH = NB / 32;       // 32-row chunks of a tile
  constexpr int NJ = NB / (8 * RQ);  // 8-row blocks owned by one row group
  constexpr int QPC = 4 / RQ;        // of those, per 32-row chunk
  constexpr int NT = 32 * RQ * NCG;
  constexpr int W = 16 * NCG;        // slab columns
  // ring depth: T_b and C_e(b) land in buffer b & 1 with block b's first chunk, issued up to
  // `ahead` chunks before it is consumed; safe when block b + 2's first chunk is issued after every
  // warp finished block b's TRMM, i.e. n0(b) + 2 n0(b+1) >= ahead (n0 = chunks per pass).  That holds
  // for ahead = RING - 1 = 4 except in a TT merge whose eliminated tile has <= 32 rows (every
  // block one chunk: 1 + 2 = 3), where the distance drops to 3 (see short3 below).
  constexpr int RING = 5;
  extern __shared__ __align__(16) double sm[];
  double* ring = sm;                     // RING x CH3: V chunks [l][r] (ld LD3 / LD3B by pass)
  double* Ts = ring + RING * CH3;        // 2 x CH3: T_b [l][q]
  double* Rb = Ts + 2 * CH3;             // RQ*NCG warps x 512: partial W^T
  double* CE = Rb + RQ * NCG * 512;      // TT: 2 x (W x LD3) rows i0.. of C_e, [col][row]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int cg = warp % NCG, rh = warp / NCG;  // column group, row group (RB == rh mod RQ)
  const int bi = g.bs(i), bk = g.cbs(k);
  const double* Vt = g.tile(const_cast<double*>(A), i, k);
  const double* T = Tbase + tri_index(i, k, g.n) * (int64_t)32 * g.nb;
  const int64_t c0 = (int64_t)blockIdx.x * W;
  const int cvalid = (int)((ncols - c0) < W ? (ncols - c0) : W);
  const int crows = (TT && !TS) ? (bi < bk ? bi : bk) : bi;
  double* Cg = base + c0 * ldcg + g.r0(i);
  const int wc = cg * 16;  // first slab column of this warp

  const int nblk = (bk + 31) / 32;
  const int nch_i = (crows + 31) / 32;
  auto chunk_lo = [&](int b) { return TT ? 0 : b; };
  auto chunk_hi = [&](int b) {
    return (TT && !TS) ? (b < nch_i - 1 ? b : nch_i - 1) : nch_i - 1;
  };
  // the chunk schedule (block, pass, chunk) of the whole CTA, built once: the producer is a table
  // lookup per chunk
  // (block, pass, chunk) entries: GEQRT / TT reflectors touch chunks up to their block, a square TS
  // reflector block all NCH chunks
  constexpr int MAXS = (TS ? 2 * NCH * NCH : 2 * NCH * (NCH + 1) / 2) + 2;
  int* sched = reinterpret_cast<int*>(CE + 2 * W * LD3);  // (dynamic shared memory, after C_e)
  // entries of block b start at 2 * (chunks of blocks < b); warp 0, one lane per block (nblk <= 10)
  auto nch_of = [&](int b) { return chunk_hi(b) >= chunk_lo(b) ? chunk_hi(b) - chunk_lo(b) + 1 : 0; };
  int S = 0;
  for (int b = 0; b < nblk; ++b) S += 2 * nch_of(b);  // (uniform, cheap: <= 10 terms)
  if (warp == 0 && lane < nblk) {
    const int b = lane;
    int n = 0;
    for (int b2 = 0; b2 < b; ++b2) n += 2 * nch_of(b2);
    const int lo = chunk_lo(b), hi = chunk_hi(b);
    for (int pass = 0; pass < 2; ++pass)
      for (int ch = lo; ch <= hi; ++ch) sched[n++] = (b << 16) | (pass << 8) | ch;
  }
  __syncthreads();
  // per-thread copy coordinates (16-byte copies: column l, rows r, r+1 of a 32 x 32 chunk)
  constexpr int CPT = 512 / NT;   // copies per thread per chunk
  const int cl0 = tid >> 4, cr = (tid & 15) * 2;
  int64_t goff[CPT];
#pragma unroll
  for (int u = 0; u < CPT; ++u) goff[u] = (int64_t)(cl0 + (NT / 16) * u) * g.lda + cr;
  int ps = 0;
  int pslot = 0;  // ring slot of the next chunk
  const unsigned ring_s = (unsigned)__cvta_generic_to_shared(ring);
  const unsigned ts_s = ring_s + (unsigned)(RING * CH3) * 8u;
  const unsigned ce_s = ts_s + (unsigned)(2 * CH3 + RQ * NCG * 512) * 8u;
  auto issue = [&]() {
    if (ps < S) {
      const int se = sched[ps];
      const int pb = se >> 16, pass = (se >> 8) & 1, ch = se & 255;
      const int i0 = 32 * pb;
      const int cmax = (bk - i0) < 32 ? (bk - i0) : 32;
      const double* src = Vt + (int64_t)i0 * g.lda + 32 * ch;
      const int rmax = crows - 32 * ch;  // valid rows in this chunk
      const int ld = pass == 0 ? LD3 : LD3B;
      const unsigned slot_s = ring_s + (unsigned)(pslot * CH3) * 8u;
      if (V16) {
        const bool rok = cr < rmax;
#pragma unroll
        for (int u = 0; u < CPT; ++u) {
          const int l = cl0 + (NT / 16) * u;
          const bool ok = rok && (l < cmax);
          cp16s(slot_s + (unsigned)(l * ld + cr) * 8u, ok ? src + goff[u] : src, ok);
        }
      } else {
        for (int o = tid; o < 1024; o += NT) {
          const int l = o >> 5, r = o & 31;
          const bool ok = (r < rmax) && (l < cmax);
          cp8s(slot_s + (unsigned)(l * ld + r) * 8u, ok ? src + (int64_t)l * g.lda + r : src, ok);
        }
      }
      if (pass == 0 && ch == chunk_lo(pb)) {
        const unsigned t_s = ts_s + (unsigned)((pb & 1) * CH3) * 8u;
#pragma unroll
        for (int u = 0; u < CPT; ++u) {
          const int l = cl0 + (NT / 16) * u;
          const bool ok = l < cmax;
          cp16s(t_s + (unsigned)(l * LD3 + cr) * 8u, ok ? T + (int64_t)(i0 + l) * 32 + cr : T, ok);
        }
        if (TT) {
          // rows i0.. of C_e for this block (W = C_e(b) + V^T C_i; C_e(b) -= U after the TRMM)
          const unsigned c_s = ce_s + (unsigned)((pb & 1) * W * LD3) * 8u;
          const double* cs = base + c0 * ldcg + g.r0(e) + i0;
          if (V16) {
            for (int o = tid; o < W * 16; o += NT) {
              const int j = o >> 4, r = (o & 15) * 2;
              const bool ok = (j < cvalid) && (r < cmax);
              cp16s(c_s + (unsigned)(j * LD3 + r) * 8u, ok ? cs + (int64_t)j * ldcg + r : cs, ok);
            }
          } else {
            for (int o = tid; o < W * 32; o += NT) {
              const int j = o >> 5, r = o & 31;
              const bool ok = (j < cvalid) && (r < cmax);
              cp8s(c_s + (unsigned)(j * LD3 + r) * 8u, ok ? cs + (int64_t)j * ldcg + r : cs, ok);
            }
          }
        }
      }
      pslot = pslot == RING - 1 ? 0 : pslot + 1;
      ++ps;
    }
    commit_();
  };
  // a TT / TS merge of a tile with <= 32 rows has one chunk per pass in every block: prefetch 3
  // chunks ahead instead of 4 so block b + 2's T / C_e never overwrite block b's before its TRMM
  const bool short3 = TT && nch_i == 1;
#pragma unroll 1
  for (int d = 0; d < (short3 ? RING - 2 : RING - 1); ++d) issue();
  // the slab's C^T fragments, loaded while the first chunks are in flight
  // ---- C^T fragments: cT[m][j][h] = C(row 8 RB + 2t + h, col wc + 8m + g), RB = RQ j + rh
  double cT[2][NJ][2];
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    const int col = wc + 8 * m + gq;
    const bool cok = col < cvalid;
    const double* cp = Cg + (int64_t)col * ldcg;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int r = 8 * (RQ * j + rh) + 2 * tq;
      if (V16 && cok && r + 1 < crows) {  // 16-byte aligned pair (even ld, even row)
        const double2 v = *reinterpret_cast<const double2*>(cp + r);
        cT[m][j][0] = v.x;
        cT[m][j][1] = v.y;
      } else {
        cT[m][j][0] = (cok && r < crows) ? cp[r] : 0.0;
        cT[m][j][1] = (cok && r + 1 < crows) ? cp[r + 1] : 0.0;
      }
    }
  }

  // explicit structure of the diagonal 32 x 32 block of V_b (GEQRT: unit diagonal, zeros above;
  // TT: zeros below the diagonal); element (r, l) at V[r * sr + l * sl]
  auto fix_diag = [&](double* V, int sr, int sl) {
    if constexpr (!TS) {  // a square TS reflector block has no structure
      for (int o = tid; o < 1024; o += NT) {
        const int l = o >> 5, r = o & 31;
        if (TT) {
          if (r > l) V[r * sr + l * sl] = 0.0;
        } else {
          if (r <= l) V[r * sr + l * sl] = (r == l) ? 1.0 : 0.0;
        }
      }
    }
  };

  const double* cslot = ring;
#pragma unroll 1
  for (int b = 0; b < nblk; ++b) {
    const int clo = chunk_lo(b), chi = chunk_hi(b);
    if (chi < clo) continue;
    const int i0 = 32 * b;
    const int sb = (bk - i0) < 32 ? (bk - i0) : 32;
    double* Ceb = TT ? base + c0 * ldcg + g.r0(e) + i0 : nullptr;
    // ---------------- GEMM1: W^T[m][nl] (16 cols x 32 refl), K = the warp's rows
    double wT[2][4][2];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int nl = 0; nl < 4; ++nl) wT[m][nl][0] = wT[m][nl][1] = 0.0;
    const double* ce = CE + (b & 1) * W * LD3;
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      if (ch < clo || ch > chi) continue;
      if (short3)
        wait_<RING - 3>();
      else
        wait_<RING - 2>();
      __syncthreads();
      issue();
      const double* V = cslot;
      cslot = (cslot == ring + (RING - 1) * CH3) ? ring : cslot + CH3;
      if (ch == b) {
        fix_diag(const_cast<double*>(V), 1, LD3);
        __syncthreads();
      }
      if (TT && ch == clo && rh == 0) {  // W starts from the C_e block rows (landed with chunk clo)
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
          for (int nl = 0; nl < 4; ++nl) {
            const double2 v = lds2(ce + (wc + 8 * m + gq) * LD3 + 8 * nl + 2 * tq);
            wT[m][nl][0] += v.x;
            wT[m][nl][1] += v.y;
          }
      }
#pragma unroll
      for (int q = 0; q < QPC; ++q) {
        const int rb = rh + RQ * q;  // 8-row block within the chunk
#pragma unroll
        for (int nl = 0; nl < 4; ++nl) {
          const double2 bv = lds2(V + (8 * nl + gq) * LD3 + 8 * rb + 2 * tq);
#pragma unroll
          for (int m = 0; m < 2; ++m) {
            dmma_(wT[m][nl][0], wT[m][nl][1], cT[m][QPC * ch + q][0], bv.x);
            dmma_(wT[m][nl][0], wT[m][nl][1], cT[m][QPC * ch + q][1], bv.y);
          }
        }      }
    }
    // ---------------- group reduction: W = P_0 + ... + P_{RQ-1} in the same order on every warp
    {
      double* mine = Rb + warp * 512;
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int nl = 0; nl < 4; ++nl)
#pragma unroll
          for (int h = 0; h < 2; ++h) mine[((m * 4 + nl) * 2 + h) * 32 + lane] = wT[m][nl][h];
      asm volatile("bar.sync %0, %1;\n" ::"r"(1 + cg), "n"(32 * RQ));
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int nl = 0; nl < 4; ++nl)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int o = ((m * 4 + nl) * 2 + h) * 32 + lane;
            double v = Rb[cg * 512 + o];
#pragma unroll
            for (int r2 = 1; r2 < RQ; ++r2) v += Rb[(cg + NCG * r2) * 512 + o];
            wT[m][nl][h] = v;
          }
      asm volatile("bar.sync %0, %1;\n" ::"r"(1 + cg), "n"(32 * RQ));
    }
    // ---------------- TRMM: U^T = W^T T_b (both warps of the pair; T_b is upper triangular, its
    // 8 x 8 blocks below the diagonal are zero and skipped), then -U^T.  (Splitting the blocks
    // between the two warps and exchanging them through shared memory measured slower.)
    double uT[2][4][2];
    {
      const double* ts = Ts + (b & 1) * CH3;
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int no = 0; no < 4; ++no) uT[m][no][0] = uT[m][no][1] = 0.0;
#pragma unroll
      for (int nl = 0; nl < 4; ++nl)
#pragma unroll
        for (int no = 0; no < 4; ++no) {
          if (nl > no) continue;
          const double2 tv = lds2(ts + (8 * no + gq) * LD3 + 8 * nl + 2 * tq);
#pragma unroll
          for (int m = 0; m < 2; ++m) {
            dmma_(uT[m][no][0], uT[m][no][1], wT[m][nl][0], tv.x);
            dmma_(uT[m][no][0], uT[m][no][1], wT[m][nl][1], tv.y);
          }
        }
    }
    if (TT && rh == 0) {
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int no = 0; no < 4; ++no)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int col = wc + 8 * m + gq, l = 8 * no + 2 * tq + h;
            if (col < cvalid && l < sb)
              Ceb[(int64_t)col * ldcg + l] = ce[col * LD3 + l] - uT[m][no][h];
          }
    }
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int no = 0; no < 4; ++no)
#pragma unroll
        for (int h = 0; h < 2; ++h) uT[m][no][h] = neg_bits(uT[m][no][h]);
    // ---------------- GEMM2: C^T[rows of the chunk] -= U^T V_b^T
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      if (ch < clo || ch > chi) continue;
      if (short3)
        wait_<RING - 3>();
      else
        wait_<RING - 2>();
      __syncthreads();
      issue();
      const double* V = cslot;
      cslot = (cslot == ring + (RING - 1) * CH3) ? ring : cslot + CH3;
      if (ch == b) {
        fix_diag(const_cast<double*>(V), 1, LD3B);
        __syncthreads();
      }
#pragma unroll
      for (int q = 0; q < QPC; ++q) {
        const int rb = rh + RQ * q;
#pragma unroll
        for (int nl = 0; nl < 4; ++nl) {
          const double bx = V[(8 * nl + 2 * tq) * LD3B + 8 * rb + gq];
          const double by = V[(8 * nl + 2 * tq + 1) * LD3B + 8 * rb + gq];
#pragma unroll
          for (int m = 0; m < 2; ++m) {
            dmma_(cT[m][QPC * ch + q][0], cT[m][QPC * ch + q][1], uT[m][nl][0], bx);
            dmma_(cT[m][QPC * ch + q][0], cT[m][QPC * ch + q][1], uT[m][nl][1], by);
          }
        }      }
    }
  }
  wait_<0>();
  // ---- store C^T back
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    const int col = wc + 8 * m + gq;
    if (col >= cvalid) continue;
    double* cp = Cg + (int64_t)col * ldcg;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int r = 8 * (RQ * j + rh) + 2 * tq;
      if (V16 && r + 1 < crows) {
        *reinterpret_cast<double2*>(cp + r) = make_double2(cT[m][j][0], cT[m][j][1]);
      } else {
        if (r < crows) cp[r] = cT[m][j][0];
        if (r + 1 < crows) cp[r + 1] = cT[m][j][1];
      }
    }
  }
  // a12 fused (TT): the eliminated tile's rows are final after its merge, so the slab's column
  // abs-sums over the tile give its share of max_{i,j>k} ||A_ij||_1 for the next step
  if (TT && gmax != nullptr) {
    double cs[2];
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      double a = 0.0;
#pragma unroll
      for (int j = 0; j < NJ; ++j) a += fabs(cT[m][j][0]) + fabs(cT[m][j][1]);
      a += __shfl_xor_sync(0xffffffffu, a, 1);
      a += __shfl_xor_sync(0xffffffffu, a, 2);
      cs[m] = a;
    }
    double* xr = Rb + cg * 512;  // the row groups' partial column sums (Rb is free here)
    __syncthreads();
    if (tq == 0) {
      xr[rh * 16 + gq] = cs[0];
      xr[rh * 16 + 8 + gq] = cs[1];
    }
    __syncthreads();
    if (rh == 0 && lane < 16) {
      double v = 0.0;
#pragma unroll
      for (int r2 = 0; r2 < RQ; ++r2) v += xr[r2 * 16 + lane];
      if (wc + lane < cvalid) atomic_max_nonneg(gmax, fabs(v));
    }
  }
}

// UNMQR of tile rows i = rows[blockIdx.y] (rows == nullptr: k + blockIdx.y)
template <int NB, int RQ, int NCG, bool V16>
__global__ void __launch_bounds__(32 * RQ * NCG, (8 / (RQ * NCG)) > 0 ? 8 / (RQ * NCG) : 1)
    k_unmqr3(const double* __restrict__ A, Geo g, int k, const double* __restrict__ Tbase,
             const int* __restrict__ rows, double* __restrict__ base, int64_t ldcg, int64_t ncols,
             const uint8_t* __restrict__ dec) {
  if (dec != nullptr && dec[k] != HLQ_DEC_QR) return;
  const int i = rows != nullptr ? rows[blockIdx.y] : k + (int)blockIdx.y;
  qr_update3_body<NB, 0, RQ, NCG, V16>(A, g, k, Tbase, 0, i, base, ldcg, ncols, nullptr);
}

// TTMQR of the pairs of one level (pair = blockIdx.y)
template <int NB, int RQ, int NCG, bool V16>
__global__ void __launch_bounds__(32 * RQ * NCG, (8 / (RQ * NCG)) > 0 ? 8 / (RQ * NCG) : 1)
    k_ttmqr3(const double* __restrict__ A, Geo g, int k, const double* __restrict__ Tbase,
             const int2* __restrict__ pairs, double* __restrict__ base, int64_t ldcg,
             int64_t ncols, const uint8_t* __restrict__ dec, double* __restrict__ gmax) {
  if (dec != nullptr && dec[k] != HLQ_DEC_QR) return;
  const int2 pr = pairs[blockIdx.y];
  qr_update3_body<NB, 1, RQ, NCG, V16>(A, g, k, Tbase, pr.x, pr.y, base, ldcg, ncols,
                                              gmax);
}

// TSMQR chains of the HQR tree (group = blockIdx.y): the group's pairs in order, each applying
// Q_i^T to [C_head; C_i] (the head's rows read-modify-written per reflector block, C_i in registers)
template <int NB, int RQ, int NCG, bool V16>
__global__ void __launch_bounds__(32 * RQ * NCG, (8 / (RQ * NCG)) > 0 ? 8 / (RQ * NCG) : 1)
    k_tsmqr3(const double* __restrict__ A, Geo g, int k, const double* __restrict__ Tbase,
             const int2* __restrict__ pairs, const int* __restrict__ off,
             double* __restrict__ base, int64_t ldcg, int64_t ncols,
             const uint8_t* __restrict__ dec, double* __restrict__ gmax) {
  if (dec != nullptr && dec[k] != HLQ_DEC_QR) return;
  for (int p = off[blockIdx.y]; p < off[blockIdx.y + 1]; ++p) {
    const int2 pr = pairs[p];
    qr_update3_body<NB, 2, RQ, NCG, V16>(A, g, k, Tbase, pr.x, pr.y, base, ldcg, ncols,
                                                gmax);
    __syncthreads();  // the head's rows and the ring are reused by the next pair
  }
}

static size_t upd3_smem(int warps, int W) {
  // ring + T ring (7 chunks), W partials, C_e rows (2 x W x LD3), the chunk schedule
  return sizeof(double) * ((size_t)7 * CH3 + (size_t)warps * 512 + (size_t)2 * W * LD3) +
         sizeof(int) * (size_t)(2 * 10 * 10 + 2);
}

template <int NB, int RQ, int NCG, bool V16>
static void launch3(const double* A, Geo g, int k, const double* T, const int2* pairs, int npairs,
                    int mode, const int* list, double* base, int64_t ldc, int64_t ncols,
                    const uint8_t* dec, cudaStream_t st, double* gmax) {
  static unsigned long long attr = 0;
  if (first_on_device(attr)) {
    smem_optin(k_unmqr3<NB, RQ, NCG, V16>);
    smem_optin(k_ttmqr3<NB, RQ, NCG, V16>);
    smem_optin(k_tsmqr3<NB, RQ, NCG, V16>);
  }
  const unsigned slabs = (unsigned)((ncols + 16 * NCG - 1) / (16 * NCG));
  const size_t smem = upd3_smem(RQ * NCG, 16 * NCG);
  if (npairs <= 0) return;
  ::hlq::g_launches++;
  if (mode == 0)  // npairs = number of tile rows (list: the rows, or nullptr for k..)
    k_unmqr3<NB, RQ, NCG, V16><<<dim3(slabs, npairs), 32 * RQ * NCG, smem, st>>>(
        A, g, k, T, list, base, ldc, ncols, dec);
  else if (mode == 1)
    k_ttmqr3<NB, RQ, NCG, V16><<<dim3(slabs, npairs), 32 * RQ * NCG, smem, st>>>(
        A, g, k, T, pairs, base, ldc, ncols, dec, gmax);
  else  // npairs = number of groups, list = their pair offsets
    k_tsmqr3<NB, RQ, NCG, V16><<<dim3(slabs, npairs), 32 * RQ * NCG, smem, st>>>(
        A, g, k, T, pairs, list, base, ldc, ncols, dec, gmax);
}

// register-slab kernels for every nb <= 320 (instantiated at 64, 128, 192, 256, 320: a smaller
// tile size is the next instantiation's ragged case, every row, column and reflector bound being a
// runtime mask, e.g. the paper's nb = 240 runs on NB = 256).  mode 0: UNMQR of npairs tile rows
// (list = the rows or nullptr for k..); 1: TTMQR of npairs pairs; 2: TSMQR chains of npairs groups
// (list = pair offsets).  false: nb has no instantiation.
bool launch_qr_update3(const double* A, Geo g, int k, const double* T, const int2* pairs,
                       int npairs, int mode, const int* list, double* base, int64_t ldc,
                       int64_t ncols, const uint8_t* dec, cudaStream_t st, double* gmax) {
  if (ncols <= 0) return true;
  // 16-byte V copies need an even leading dimension, a 16-byte aligned matrix and even tile heights
  const bool v16 = ((g.lda & 1) == 0) && ((((uintptr_t)A) & 15) == 0) && ((g.N & 1) == 0) &&
                   ((g.nb & 1) == 0) && ((ldc & 1) == 0) && ((((uintptr_t)base) & 15) == 0);
#define HLQ_L3(NBV)                                                                           \
  case NBV:                                                                                   \
    if (!v16)                                                                                 \
      launch3<NBV, 2, 2, false>(A, g, k, T, pairs, npairs, mode, list, base, ldc, ncols, dec, st, \
                                gmax);                                                        \
    else                                                                                      \
      launch3<NBV, 2, 2, true>(A, g, k, T, pairs, npairs, mode, list, base, ldc, ncols, dec, st,  \
                               gmax);                                                         \
    return true;
  const int nbi = g.nb <= 64 ? 64 : g.nb <= 128 ? 128 : g.nb <= 192 ? 192 : g.nb <= 256 ? 256 : 320;
  switch (nbi) {
    HLQ_L3(64)
    HLQ_L3(128)
    HLQ_L3(192)
    HLQ_L3(256)
    HLQ_L3(320)
    default: return false;
  }
#undef HLQ_L3
}

static void must(bool ok, int nb) {
  if (!ok) {
    fprintf(stderr, "[hlq] QR update: nb = %d has no register-slab instantiation\n", nb);
    abort();
  }
}

void launch_unmqr_rows(const double* A, Geo g, int k, const double* T, const int* rows, int nrows,
                       double* base, int64_t ldc, int64_t ncols, const uint8_t* dec,
                       cudaStream_t st) {
  must(launch_qr_update3(A, g, k, T, nullptr, nrows, 0, rows, base, ldc, ncols, dec, st, nullptr),
       g.nb);
}

void launch_tsmqr_chains(const double* A, Geo g, int k, const double* T, const int2* pairs,
                         const int* off, int ngroups, double* base, int64_t ldc, int64_t ncols,
                         const uint8_t* dec, cudaStream_t st, double* gmax) {
  must(launch_qr_update3(A, g, k, T, pairs, ngroups, 2, off, base, ldc, ncols, dec, st, gmax),
       g.nb);
}

}  // namespace hlq
