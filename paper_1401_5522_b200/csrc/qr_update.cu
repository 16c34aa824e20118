// QR trailing update (a8 UNMQR, a10/a11 TTMQR): the bulk of a QR step's flops (Table I "update D"
// PAPER.md:166; Alg. 4b), on the FP64 tensor cores (DMMA).  One CTA owns a column slab of
// one tile row (UNMQR) or of the eliminated tile of one TT pair (TTMQR) for the whole step and
// keeps it in REGISTERS as C^T accumulator fragments (design below, "v3"); every C element is read
// and written once per launch.  Householder convention and T layout: DESIGN.md readings 14-15.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

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
// TMA (tensor) loads into the ring and their mbarriers
__device__ __forceinline__ void mbar_init_(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx_(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma2d_(unsigned dst, const CUtensorMap* tm, unsigned bar, int c0,
                                       int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(dst),
      "l"(tm), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
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
constexpr int QU_RING = 5;     // V chunk ring depth
constexpr int QU_SCHED = 202;  // chunk schedule capacity (2 NCH^2 + 2 at NB = 320)
// TMA path: a 32 x 32 chunk is two 16-row x 32-column boxes with the 128-byte swizzle (each column's
// 16 rows one 128-byte line; 16-byte unit u of line l at u ^ (l & 7)); element (r, l) at
constexpr int QU_SLOT = 1024;  // doubles per chunk (8 KB)
__device__ __forceinline__ int swz(int r, int l) {
  return (r >> 4) * 512 + l * 16 + ((((r & 15) >> 1) ^ (l & 7)) << 1) + (r & 1);
}
// shared-memory layout of the TMA path (bytes from a 1024-aligned base): ring, T ring, C_e ring,
// W partials, schedule, mbarriers
__host__ __device__ constexpr size_t qu_tma_bars(int warps) {
  return (size_t)(QU_RING + 4) * QU_SLOT * 8 + (size_t)warps * 512 * 8 + sizeof(int) * QU_SCHED;
}
__host__ __device__ constexpr size_t qu_tma_smem(int warps) {
  return (qu_tma_bars(warps) + 7) / 8 * 8 + 8 * QU_RING + 1024 /* alignment slack */;
}
}  // namespace

// tensor maps of the TMA path: A (rows x columns, box 16 x 32), the GEQRT and the TT/TS T arrays
// (32 x (tiles * nb), box 16 x 32); one set per factorization (api.cu)
struct QuMaps {
  CUtensorMap a, tg, tt;
};
namespace {
struct QuCtx {  // the factorization whose update is being launched (qu_tma_begin / qu_tma_end)
  const QuMaps* maps = nullptr;
  const double* A = nullptr;
  const double* Tg = nullptr;
  const double* Ttt = nullptr;
  int64_t lda = 0;
};
thread_local QuCtx g_qu;
}  // namespace

// MODE 0: UNMQR of tile row i (GEQRT reflectors, unit lower); 1: TTMQR of the pair (e, i) (TT
// reflectors, upper triangular); 2: TSMQR of the pair (e, i) (TS reflectors, square)
template <int NB, int MODE, int RQ, int NCG, bool V16, bool TMA>
__device__ __forceinline__ void qr_update3_body(const double* __restrict__ A, Geo g, int k,
                                                const double* __restrict__ Tbase, int e, int i,
                                                double* __restrict__ base, int64_t ldcg,
                                                int64_t ncols, double* __restrict__ gmax,
                                                const QuMaps* maps, int tmode, int64_t bcol,
                                                unsigned& phase) {
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
  constexpr int RING = QU_RING;
  constexpr int SLOT = TMA ? QU_SLOT : CH3;  // doubles per ring slot / T buffer
  extern __shared__ __align__(16) double sm[];
  // TMA: every buffer on a 1024-byte boundary of the shared window (the 128-byte swizzle atom)
  double* const sm0 = TMA ? sm + ((1024u - ((unsigned)__cvta_generic_to_shared(sm) & 1023u)) & 1023u) / 8
                          : sm;
  double* ring = sm0;                    // RING x SLOT: V chunks (cp.async: [l][r], ld LD3 / LD3B
                                         // by pass; TMA: swizzled 16 x 32 box pairs, swz())
  double* Ts = ring + RING * SLOT;       // 2 x SLOT: T_b
  double* CE;                            // TT: 2 buffers of rows i0.. of C_e
  double* Rb;                            // RQ*NCG warps x 512: partial W^T
  if constexpr (TMA) {
    CE = Ts + 2 * SLOT;
    Rb = CE + 2 * SLOT;
  } else {
    Rb = Ts + 2 * SLOT;
    CE = Rb + RQ * NCG * 512;
  }
  // element (r, l) of a V chunk / T block / C_e block (row r, column l) in its buffer
  auto vix = [](int r, int l, int ld) { return TMA ? swz(r, l) : l * ld + r; };
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
  int* sched = TMA ? reinterpret_cast<int*>(Rb + RQ * NCG * 512)
                  : reinterpret_cast<int*>(CE + 2 * W * LD3);  // (dynamic shared memory)
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
  const unsigned bar_s = ring_s + (unsigned)((qu_tma_bars(RQ * NCG) + 7) / 8 * 8);
  // TMA: one thread issues the chunk's two boxes (+ T_b and C_e(b) with a block's first chunk), the
  // slot's mbarrier counts the bytes; the consumers never touch the producer's bookkeeping
  auto issue_tma = [&]() {
    if (ps < S) {
      if (tid == 0) {
        const int se = sched[ps];
        const int pb = se >> 16, pass = (se >> 8) & 1, ch = se & 255;
        const int i0 = 32 * pb;
        const bool first = pass == 0 && ch == chunk_lo(pb);
        const unsigned bar = bar_s + 8u * (unsigned)pslot;
        mbar_arrive_tx_(bar, 8192u + (first ? 8192u + (TT ? 8192u : 0u) : 0u));
        const unsigned dst = ring_s + (unsigned)(pslot * QU_SLOT) * 8u;
        const int vr = (int)g.r0(i) + 32 * ch, vc = (int)g.r0(k) + i0;
        tma2d_(dst, &maps->a, bar, vr, vc);
        tma2d_(dst + 4096u, &maps->a, bar, vr + 16, vc);
        if (first) {
          const CUtensorMap* tm = tmode ? &maps->tt : &maps->tg;
          const int tcol = (int)(tri_index(i, k, g.n) * g.nb) + i0;
          const unsigned tdst = ring_s + (unsigned)((RING + (pb & 1)) * QU_SLOT) * 8u;
          tma2d_(tdst, tm, bar, 0, tcol);
          tma2d_(tdst + 4096u, tm, bar, 16, tcol);
          if (TT) {
            const unsigned cdst = ring_s + (unsigned)((RING + 2 + (pb & 1)) * QU_SLOT) * 8u;
            const int er = (int)g.r0(e) + i0, ec = (int)(bcol + c0);
            tma2d_(cdst, &maps->a, bar, er, ec);
            tma2d_(cdst + 4096u, &maps->a, bar, er + 16, ec);
          }
        }
      }
      pslot = pslot == RING - 1 ? 0 : pslot + 1;
      ++ps;
    }
  };
  auto issue = [&]() {
    if constexpr (TMA) {
      issue_tma();
      return;
    }
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
  auto fix_diag = [&](double* V, int ld) {
    if constexpr (!TS) {  // a square TS reflector block has no structure
      for (int o = tid; o < 1024; o += NT) {
        const int l = o >> 5, r = o & 31;
        if (TT) {
          if (r > l) V[vix(r, l, ld)] = 0.0;
        } else {
          if (r <= l) V[vix(r, l, ld)] = (r == l) ? 1.0 : 0.0;
        }
      }
    }
  };

  const double* cslot = ring;
  int cidx = 0;  // ring slot of the chunk being consumed
  // the chunk in slot cidx has landed (TMA: its mbarrier phase; cp.async: the groups) and every warp
  // is done with the previous chunk, whose slot is refilled next
  auto next_chunk = [&]() {
    if constexpr (TMA) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // my reads before the refill
      __syncthreads();
      issue();
      mbar_wait_(bar_s + 8u * (unsigned)cidx, (phase >> cidx) & 1u);
      phase ^= 1u << cidx;
    } else {
      if (short3)
        wait_<RING - 3>();
      else
        wait_<RING - 2>();
      __syncthreads();
      issue();
    }
    cidx = cidx == RING - 1 ? 0 : cidx + 1;
  };
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
    const double* ce = CE + (b & 1) * (TMA ? QU_SLOT : W * LD3);
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      if (ch < clo || ch > chi) continue;
      next_chunk();
      const double* V = cslot;
      cslot = (cslot == ring + (RING - 1) * SLOT) ? ring : cslot + SLOT;
      if (ch == b) {
        fix_diag(const_cast<double*>(V), LD3);
        __syncthreads();
      }
      if (TT && ch == clo && rh == 0) {  // W starts from the C_e block rows (landed with chunk clo)
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
          for (int nl = 0; nl < 4; ++nl) {
            const double2 v = lds2(ce + vix(8 * nl + 2 * tq, wc + 8 * m + gq, LD3));
            wT[m][nl][0] += v.x;
            wT[m][nl][1] += v.y;
          }
      }
#pragma unroll
      for (int q = 0; q < QPC; ++q) {
        const int rb = rh + RQ * q;  // 8-row block within the chunk
#pragma unroll
        for (int nl = 0; nl < 4; ++nl) {
          const double2 bv = lds2(V + vix(8 * rb + 2 * tq, 8 * nl + gq, LD3));
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
      const double* ts = Ts + (b & 1) * SLOT;
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int no = 0; no < 4; ++no) uT[m][no][0] = uT[m][no][1] = 0.0;
#pragma unroll
      for (int nl = 0; nl < 4; ++nl)
#pragma unroll
        for (int no = 0; no < 4; ++no) {
          if (nl > no) continue;
          const double2 tv = lds2(ts + vix(8 * nl + 2 * tq, 8 * no + gq, LD3));
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
              Ceb[(int64_t)col * ldcg + l] = ce[vix(l, col, LD3)] - uT[m][no][h];
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
      next_chunk();
      const double* V = cslot;
      cslot = (cslot == ring + (RING - 1) * SLOT) ? ring : cslot + SLOT;
      if (ch == b) {
        fix_diag(const_cast<double*>(V), LD3B);
        __syncthreads();
      }
#pragma unroll
      for (int q = 0; q < QPC; ++q) {
        const int rb = rh + RQ * q;
#pragma unroll
        for (int nl = 0; nl < 4; ++nl) {
          const double bx = V[vix(8 * rb + gq, 8 * nl + 2 * tq, LD3B)];
          const double by = V[vix(8 * rb + gq, 8 * nl + 2 * tq + 1, LD3B)];
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

// the TMA ring's mbarriers, initialised once per CTA; returns the slots' phase bits
template <bool TMA>
__device__ __forceinline__ unsigned qu_init_bars(int warps) {
  if constexpr (TMA) {
    extern __shared__ __align__(16) double sm[];
    const unsigned base_s = (unsigned)__cvta_generic_to_shared(sm);
    const unsigned ring_s = base_s + ((1024u - (base_s & 1023u)) & 1023u);
    const unsigned bar_s = ring_s + (unsigned)((qu_tma_bars(warps) + 7) / 8 * 8);
    if (threadIdx.x == 0) {
      for (int s = 0; s < QU_RING; ++s) mbar_init_(bar_s + 8u * s, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  return 0u;
}

// UNMQR of tile rows i = rows[blockIdx.y] (rows == nullptr: k + blockIdx.y)
template <int NB, int RQ, int NCG, bool V16, bool TMA>
__global__ void __launch_bounds__(32 * RQ * NCG, (8 / (RQ * NCG)) > 0 ? 8 / (RQ * NCG) : 1)
    k_unmqr3(const double* __restrict__ A, Geo g, int k, const double* __restrict__ Tbase,
             const int* __restrict__ rows, double* __restrict__ base, int64_t ldcg, int64_t ncols,
             const uint8_t* __restrict__ dec, const __grid_constant__ QuMaps maps, int tmode,
             int64_t bcol) {
  if (dec != nullptr && dec[k] != HLQ_DEC_QR) return;
  const int i = rows != nullptr ? rows[blockIdx.y] : k + (int)blockIdx.y;
  unsigned phase = qu_init_bars<TMA>(RQ * NCG);
  qr_update3_body<NB, 0, RQ, NCG, V16, TMA>(A, g, k, Tbase, 0, i, base, ldcg, ncols, nullptr,
                                            &maps, tmode, bcol, phase);
}

// TTMQR of the pairs of one level (pair = blockIdx.y)
template <int NB, int RQ, int NCG, bool V16, bool TMA>
__global__ void __launch_bounds__(32 * RQ * NCG, (8 / (RQ * NCG)) > 0 ? 8 / (RQ * NCG) : 1)
    k_ttmqr3(const double* __restrict__ A, Geo g, int k, const double* __restrict__ Tbase,
             const int2* __restrict__ pairs, double* __restrict__ base, int64_t ldcg,
             int64_t ncols, const uint8_t* __restrict__ dec, double* __restrict__ gmax,
             const __grid_constant__ QuMaps maps, int tmode, int64_t bcol) {
  if (dec != nullptr && dec[k] != HLQ_DEC_QR) return;
  const int2 pr = pairs[blockIdx.y];
  unsigned phase = qu_init_bars<TMA>(RQ * NCG);
  qr_update3_body<NB, 1, RQ, NCG, V16, TMA>(A, g, k, Tbase, pr.x, pr.y, base, ldcg, ncols, gmax,
                                            &maps, tmode, bcol, phase);
}

// TSMQR chains of the HQR tree (group = blockIdx.y): the group's pairs in order, each applying
// Q_i^T to [C_head; C_i] (the head's rows read-modify-written per reflector block, C_i in registers)
template <int NB, int RQ, int NCG, bool V16, bool TMA>
__global__ void __launch_bounds__(32 * RQ * NCG, (8 / (RQ * NCG)) > 0 ? 8 / (RQ * NCG) : 1)
    k_tsmqr3(const double* __restrict__ A, Geo g, int k, const double* __restrict__ Tbase,
             const int2* __restrict__ pairs, const int* __restrict__ off,
             double* __restrict__ base, int64_t ldcg, int64_t ncols,
             const uint8_t* __restrict__ dec, double* __restrict__ gmax,
             const __grid_constant__ QuMaps maps, int tmode, int64_t bcol) {
  if (dec != nullptr && dec[k] != HLQ_DEC_QR) return;
  unsigned phase = qu_init_bars<TMA>(RQ * NCG);
  for (int p = off[blockIdx.y]; p < off[blockIdx.y + 1]; ++p) {
    const int2 pr = pairs[p];
    qr_update3_body<NB, 2, RQ, NCG, V16, TMA>(A, g, k, Tbase, pr.x, pr.y, base, ldcg, ncols, gmax,
                                              &maps, tmode, bcol, phase);
    // the head's rows and the ring are reused by the next pair (TMA: order this pair's reads of
    // the ring before the next pair's tensor loads into it)
    if (TMA) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
  }
}

static size_t upd3_smem(int warps, int W, bool tma) {
  if (tma) return qu_tma_smem(warps);
  // ring + T ring (7 chunks), W partials, C_e rows (2 x W x LD3), the chunk schedule
  return sizeof(double) * ((size_t)7 * CH3 + (size_t)warps * 512 + (size_t)2 * W * LD3) +
         sizeof(int) * (size_t)QU_SCHED;
}

template <int NB, int RQ, int NCG, bool V16, bool TMA>
static void launch3(const double* A, Geo g, int k, const double* T, const int2* pairs, int npairs,
                    int mode, const int* list, double* base, int64_t ldc, int64_t ncols,
                    const uint8_t* dec, cudaStream_t st, double* gmax, const QuMaps* maps,
                    int tmode, int64_t bcol) {
  static unsigned long long attr = 0;
  if (first_on_device(attr)) {
    smem_optin(k_unmqr3<NB, RQ, NCG, V16, TMA>);
    smem_optin(k_ttmqr3<NB, RQ, NCG, V16, TMA>);
    smem_optin(k_tsmqr3<NB, RQ, NCG, V16, TMA>);
  }
  const unsigned slabs = (unsigned)((ncols + 16 * NCG - 1) / (16 * NCG));
  const size_t smem = upd3_smem(RQ * NCG, 16 * NCG, TMA);
  if (npairs <= 0) return;
  static const QuMaps none{};
  const QuMaps& mp = maps ? *maps : none;
  ::hlq::g_launches++;
  if (mode == 0)  // npairs = number of tile rows (list: the rows, or nullptr for k..)
    k_unmqr3<NB, RQ, NCG, V16, TMA><<<dim3(slabs, npairs), 32 * RQ * NCG, smem, st>>>(
        A, g, k, T, list, base, ldc, ncols, dec, mp, tmode, bcol);
  else if (mode == 1)
    k_ttmqr3<NB, RQ, NCG, V16, TMA><<<dim3(slabs, npairs), 32 * RQ * NCG, smem, st>>>(
        A, g, k, T, pairs, base, ldc, ncols, dec, gmax, mp, tmode, bcol);
  else  // npairs = number of groups, list = their pair offsets
    k_tsmqr3<NB, RQ, NCG, V16, TMA><<<dim3(slabs, npairs), 32 * RQ * NCG, smem, st>>>(
        A, g, k, T, pairs, list, base, ldc, ncols, dec, gmax, mp, tmode, bcol);
}

// register-slab kernels for every nb <= 320 (instantiated at 64, 128, 192, 256, 320: a smaller
// tile size is the next instantiation's ragged case, every row, column and reflector bound being a
// runtime mask, e.g. the paper's nb = 240 runs on NB = 256).  mode 0: UNMQR of npairs tile rows
// (list = the rows or nullptr for k..); 1: TTMQR of npairs pairs; 2: TSMQR chains of npairs groups
// (list = pair offsets).  false: nb has no instantiation.  The TMA-fed ring is used when the
// update's V tiles, T factors and C_e rows are those of the factorization whose tensor maps are
// current (qu_tma_begin): A itself, base a column offset of A with the same leading dimension.
bool launch_qr_update3(const double* A, Geo g, int k, const double* T, const int2* pairs,
                       int npairs, int mode, const int* list, double* base, int64_t ldc,
                       int64_t ncols, const uint8_t* dec, cudaStream_t st, double* gmax) {
  if (ncols <= 0) return true;
  // 16-byte V copies need an even leading dimension, a 16-byte aligned matrix and even tile heights
  const bool v16 = ((g.lda & 1) == 0) && ((((uintptr_t)A) & 15) == 0) && ((g.N & 1) == 0) &&
                   ((g.nb & 1) == 0) && ((ldc & 1) == 0) && ((((uintptr_t)base) & 15) == 0);
  const QuCtx& q = g_qu;
  const bool tma = v16 && q.maps != nullptr && A == q.A && ldc == q.lda && g.lda == q.lda &&
                   base >= A && ((base - A) % q.lda) == 0 && (T == q.Tg || T == q.Ttt);
  const int tmode = (tma && T == q.Ttt) ? 1 : 0;
  const int64_t bcol = tma ? (int64_t)((base - A) / q.lda) : 0;
#define HLQ_L3(NBV)                                                                           \
  case NBV:                                                                                   \
    if (!v16)                                                                                 \
      launch3<NBV, 2, 2, false, false>(A, g, k, T, pairs, npairs, mode, list, base, ldc, ncols,   \
                                       dec, st, gmax, nullptr, 0, 0);                         \
    else if (tma)                                                                             \
      launch3<NBV, 2, 2, true, true>(A, g, k, T, pairs, npairs, mode, list, base, ldc, ncols,     \
                                     dec, st, gmax, q.maps, tmode, bcol);                     \
    else                                                                                      \
      launch3<NBV, 2, 2, true, false>(A, g, k, T, pairs, npairs, mode, list, base, ldc, ncols,    \
                                      dec, st, gmax, nullptr, 0, 0);                          \
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

// ---- host: tensor maps of the TMA-fed QR update (per factorization) --------------------------
static PFN_cuTensorMapEncodeTiled_v12000 qu_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult r;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &r) ==
            cudaSuccess &&
        r == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    else
      cudaGetLastError();
  }
  return fn;
}

// maps of A (N x N, ld lda) and of the T arrays (ntri tiles of 32 x nb each); nullptr when the
// matrix is not eligible (odd lda / N / nb, misaligned, HLQ_QR_TMA=0) -- the cp.async ring is used
void* make_qu_maps(const double* A, int64_t N, int64_t lda, int nb, const double* Tg,
                   const double* Ttt, int64_t ntri) {
  static int off = -1;
  if (off < 0) off = getenv("HLQ_QR_TMA") ? (atoi(getenv("HLQ_QR_TMA")) == 0) : 0;
  // nb a multiple of 32: every 32-row chunk and 32-reflector block lies inside its tile, or past
  // the matrix edge where the boxes are zero-filled (the paper's nb = 240 keeps the cp.async ring,
  // which zero-fills ragged chunks itself)
  if (off || (lda & 1) || (N & 1) || (nb % 32) || (((uintptr_t)A) & 15) || N >= ((int64_t)1 << 31) ||
      ntri * nb >= ((int64_t)1 << 31))
    return nullptr;
  auto fn = qu_encode();
  if (!fn) return nullptr;
  QuMaps* m = (QuMaps*)aligned_alloc(64, sizeof(QuMaps));
  if (!m) return nullptr;
  memset(m, 0, sizeof(*m));
  const cuuint32_t box[2] = {16, 32}, es[2] = {1, 1};
  const cuuint64_t gdA[2] = {(cuuint64_t)N, (cuuint64_t)N}, gsA[1] = {(cuuint64_t)lda * 8};
  const cuuint64_t gdT[2] = {32, (cuuint64_t)(ntri * nb)}, gsT[1] = {32 * 8};
  auto enc = [&](CUtensorMap* t, const double* p, const cuuint64_t* gd, const cuuint64_t* gs) {
    return fn(t, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)p, gd, gs, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  };
  if (enc(&m->a, A, gdA, gsA) != CUDA_SUCCESS || enc(&m->tg, Tg, gdT, gsT) != CUDA_SUCCESS ||
      enc(&m->tt, Ttt, gdT, gsT) != CUDA_SUCCESS) {
    free(m);
    return nullptr;
  }
  return m;
}
void free_qu_maps(void* m) { free(m); }

// the factorization whose QR updates are being launched on this host thread (its maps, matrix and
// T arrays), so launch_qr_update3 can pick the TMA ring; qu_tma_end clears it
void qu_tma_begin(const void* maps, const double* A, int64_t lda, const double* Tg,
                  const double* Ttt) {
  g_qu.maps = (const QuMaps*)maps;
  g_qu.A = A;
  g_qu.lda = lda;
  g_qu.Tg = Tg;
  g_qu.Ttt = Ttt;
}
void qu_tma_end() { g_qu = QuCtx{}; }

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
