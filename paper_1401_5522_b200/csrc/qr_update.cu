// QR trailing update, v2 (a8 UNMQR, a10/a11 TTMQR): the bulk of a QR step's flops (Table I
// "update D" PAPER.md:166; Alg. 4b), on the FP64 tensor cores (DMMA).
//
// One CTA owns a slab of W = 8*NW columns of one tile row (UNMQR) or of one TT pair (TTMQR, the
// slab of the eliminated tile i; rows of the surviving tile e are read-modify-written per block).
// The slab stays in shared memory for the whole step: every C element is read and written once.
// Warp w owns slab columns [8w, 8w+8) for ALL three products of a reflector block b (32 columns):
//     GEMM1  W  = [C_e(b) +] V_b^T C        32 x 8 per warp, K = rows of V_b   (DMMA)
//     TRMM   U  = T_b^T W                   32 x 8 per warp, K = 32            (DMMA)
//     GEMM2  C -= V_b U   [C_e(b) -= U]     rows x 8 per warp, K = 32          (DMMA)
// so a warp only ever touches its own columns of C: the only data shared by the CTA is the stream
// of V_b row chunks (32 x 32, cp.async, DEPTH-deep ring) and T_b.  V_b is streamed twice per block
// (GEMM1, GEMM2) from L2; its explicit structure (unit diagonal / zeros above for GEQRT reflectors,
// zeros below the diagonal for the TT reflectors) is applied when the diagonal chunk's fragments are
// loaded.  Fragments: mma.sync.m8n8k4.f64 (lane g = lane/4, t = lane%4: A(g,t), B(t,g),
// C(g, 2t..2t+1)); every shared array has a leading dimension == 4 (mod 16) doubles, which makes the
// fragment loads bank-conflict free.  Householder convention and T layout: DESIGN.md 14-15.
#include "hlq_internal.cuh"

namespace hlq {

namespace {
constexpr int LDV = 36;  // V chunk [l][r], T [col][row], W/U [col][l]
constexpr int DEPTH = 3;
constexpr int CH = 32 * LDV;  // doubles per ring slot

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
__device__ __forceinline__ void commit_() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void wait_() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__host__ __device__ inline int rup32(int x) { return (x + 31) / 32 * 32; }
}  // namespace

// rows [r0, r0+32) x cols [c0, c0+32) of a column-major source (ld) -> dst[l*LDV + r]; zero-fill rows
// >= rmax and columns >= cmax
template <bool V16>
__device__ __forceinline__ void load_chunk(double* dst, const double* src, int64_t ld, int r0,
                                           int rmax, int cmax, int tid, int nthr) {
  if (V16) {
    for (int o = tid; o < 32 * 16; o += nthr) {
      const int l = o >> 4, r = (o & 15) * 2;
      const bool ok = (r0 + r < rmax) && (l < cmax);  // rmax even on this path
      cp16(dst + l * LDV + r, ok ? src + (int64_t)l * ld + r0 + r : src, ok);
    }
  } else {
    for (int o = tid; o < 32 * 32; o += nthr) {
      const int l = o >> 5, r = o & 31;
      const bool ok = (r0 + r < rmax) && (l < cmax);
      cp8(dst + l * LDV + r, ok ? src + (int64_t)l * ld + r0 + r : src, ok);
    }
  }
}

template <int NW, bool TT, bool V16>
__global__ void __launch_bounds__(NW * 32) k_qr_update2(const double* __restrict__ A, Geo g,
                                                       int k, const double* __restrict__ Tbase,
                                                       const int2* __restrict__ pairs,
                                                       double* __restrict__ base, int64_t ldcg,
                                                       int64_t ncols,
                                                       const uint8_t* __restrict__ dec) {
  if (dec != nullptr && dec[k] != HLQ_DEC_QR) return;
  constexpr int W = 8 * NW, NT = 32 * NW;
  extern __shared__ __align__(16) double sm[];
  const int ldc = rup32(g.nb) + 4;
  double* Cs = sm;                        // W x ldc   slab of tile i (col-major)
  double* ring = Cs + W * ldc;            // DEPTH x 32 x LDV
  double* Ts = ring + DEPTH * CH;         // 2 x 32 x LDV (double-buffered per block)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  double* Ws = Ts + 2 * CH + warp * 8 * LDV;  // per warp 8 x LDV

  int e = 0, i;
  if (TT) {
    const int2 pr = pairs[blockIdx.y];
    e = pr.x;
    i = pr.y;
  } else {
    i = k + blockIdx.y;
  }
  const int bi = g.bs(i), bk = g.cbs(k);
  const double* Vt = g.tile(const_cast<double*>(A), i, k);
  const double* T = Tbase + tri_index(i, k, g.n) * (int64_t)32 * g.nb;
  const int64_t c0 = (int64_t)blockIdx.x * W;
  const int cvalid = (int)((ncols - c0) < W ? (ncols - c0) : W);
  // rows of the slab that any block touches
  const int crows = TT ? (bi < bk ? bi : bk) : bi;
  const int crows_pad = rup32(crows);
  double* Cg = base + c0 * ldcg + g.r0(i);

  // ---- C slab (its own commit group, ahead of the ring prologue)
  {
    const bool v16 = V16 && ((ldcg & 1) == 0) && ((((uintptr_t)Cg) & 15) == 0);
    if (v16) {
      const int rp2 = crows_pad >> 1;
      for (int o = tid; o < W * rp2; o += NT) {
        const int j = o / rp2, r = 2 * (o - j * rp2);
        const bool ok = (j < cvalid) && (r + 1 < crows);
        if (ok) {
          cp16(Cs + j * ldc + r, Cg + (int64_t)j * ldcg + r, true);
        } else {
          Cs[j * ldc + r] = (j < cvalid && r < crows) ? Cg[(int64_t)j * ldcg + r] : 0.0;
          Cs[j * ldc + r + 1] = 0.0;
        }
      }
    } else {
      for (int o = tid; o < W * crows_pad; o += NT) {
        const int j = o / crows_pad, r = o - j * crows_pad;
        const bool ok = (j < cvalid) && (r < crows);
        cp8(Cs + j * ldc + r, ok ? Cg + (int64_t)j * ldcg + r : Cg, ok);
      }
    }
    commit_();
  }

  // ---- chunk stream: for every block b: GEMM1 chunks, then GEMM2 chunks (same V_b rows)
  const int nblk = (bk + 31) / 32;
  auto blk_rows = [&](int b, int& rlo, int& rhi) {
    const int i0 = 32 * b;
    if (TT) {
      rlo = 0;
      rhi = bi < i0 + 32 ? bi : i0 + 32;
    } else {
      rlo = i0;
      rhi = bi;
    }
  };
  // producer state
  int pb = 0, ppass = 0, pc = 0, ps = 0;
  bool pdone = false;
  auto issue = [&]() {
    if (!pdone) {
      int rlo, rhi;
      blk_rows(pb, rlo, rhi);
      if (rhi <= rlo) {
        pdone = true;
      } else {
        const int i0 = 32 * pb;
        const int cmax = (bk - i0) < 32 ? (bk - i0) : 32;
        double* slot = ring + (ps % DEPTH) * CH;
        const bool v16 = V16 && ((g.lda & 1) == 0) && ((((uintptr_t)Vt) & 15) == 0) &&
                         ((rhi & 1) == 0);
        if (v16)
          load_chunk<true>(slot, Vt + (int64_t)i0 * g.lda, g.lda, rlo + 32 * pc, rhi, cmax, tid, NT);
        else
          load_chunk<false>(slot, Vt + (int64_t)i0 * g.lda, g.lda, rlo + 32 * pc, rhi, cmax, tid,
                            NT);
        if (ppass == 0 && pc == 0) {
          // T_b (32 x 32, stored T(q, l) at T[(i0 + l) * 32 + q], zeros below the diagonal)
          double* ts = Ts + (pb & 1) * CH;
          for (int o = tid; o < 32 * 16; o += NT) {
            const int l = o >> 4, q = (o & 15) * 2;
            const bool ok = l < cmax;
            cp16(ts + l * LDV + q, ok ? T + (int64_t)(i0 + l) * 32 + q : T, ok);
          }
        }
        ++ps;
        const int nch = (rhi - rlo + 31) / 32;
        if (++pc == nch) {
          pc = 0;
          if (++ppass == 2) {
            ppass = 0;
            if (++pb == nblk) pdone = true;
          }
        }
      }
    }
    commit_();
  };
#pragma unroll 1
  for (int d = 0; d < DEPTH - 1; ++d) issue();

  int s = 0;  // consumer chunk index
  const int wc = warp * 8;  // first slab column of this warp
#pragma unroll 1
  for (int b = 0; b < nblk; ++b) {
    int rlo, rhi;
    blk_rows(b, rlo, rhi);
    if (rhi <= rlo) break;
    const int i0 = 32 * b;
    const int sb = (bk - i0) < 32 ? (bk - i0) : 32;
    const int nch = (rhi - rlo + 31) / 32;
    // chunk index (within the block) that holds the diagonal 32 x 32 block of V_b
    const int cdiag = TT ? (i0 / 32) : 0;
    double* Ceb = TT ? base + c0 * ldcg + g.r0(e) + i0 : nullptr;  // C_e rows of block b

    // ---------------- GEMM1: W = [C_e(b) +] V_b^T C
    double acc[2][4][2];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) acc[u][mi][0] = acc[u][mi][1] = 0.0;
    if (TT) {
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int l = mi * 8 + gq, col = wc + 2 * tq + h;
          if (l < sb && col < cvalid) acc[0][mi][h] = Ceb[(int64_t)col * ldcg + l];
        }
    }
#pragma unroll 1
    for (int c = 0; c < nch; ++c, ++s) {
      wait_<DEPTH - 2>();
      __syncthreads();
      issue();
      const double* V = ring + (s % DEPTH) * CH;
      const double* Cb = Cs + (wc + gq) * ldc + rlo + 32 * c + tq;
      if (c == cdiag) {
#pragma unroll
        for (int kk = 0; kk < 32; kk += 4) {
          const double bv = Cb[kk];
          const int r = kk + tq;  // row within the diagonal chunk
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) {
            const int l = mi * 8 + gq;
            double a = V[l * LDV + r];
            if (TT) {
              if (r > l) a = 0.0;
            } else {
              a = (r < l) ? 0.0 : ((r == l) ? 1.0 : a);
            }
            dmma_(acc[(kk >> 2) & 1][mi][0], acc[(kk >> 2) & 1][mi][1], a, bv);
          }
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < 32; kk += 4) {
          const double bv = Cb[kk];
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
            dmma_(acc[(kk >> 2) & 1][mi][0], acc[(kk >> 2) & 1][mi][1],
                  V[(mi * 8 + gq) * LDV + kk + tq], bv);
        }
      }
    }
    // ---------------- TRMM: U = T_b^T W (this warp's 8 columns), then -U for GEMM2's B operand
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int h = 0; h < 2; ++h) Ws[(2 * tq + h) * LDV + mi * 8 + gq] = acc[0][mi][h] + acc[1][mi][h];
    __syncwarp();
    {
      const double* ts = Ts + (b & 1) * CH;
      double u[4][2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) u[mi][0] = u[mi][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < 32; kk += 4) {
        const double bv = Ws[gq * LDV + kk + tq];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
          dmma_(u[mi][0], u[mi][1], ts[(mi * 8 + gq) * LDV + kk + tq], bv);
      }
      __syncwarp();
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int l = mi * 8 + gq, col = wc + 2 * tq + h;
          Ws[(2 * tq + h) * LDV + l] = neg_bits(u[mi][h]);
          if (TT && l < sb && col < cvalid) Ceb[(int64_t)col * ldcg + l] -= u[mi][h];
        }
      __syncwarp();
    }
    // ---------------- GEMM2: C[rows] -= V_b U
#pragma unroll 1
    for (int c = 0; c < nch; ++c, ++s) {
      wait_<DEPTH - 2>();
      __syncthreads();
      issue();
      const double* V = ring + (s % DEPTH) * CH;
      const int r0 = rlo + 32 * c;
      double cc[4][2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int h = 0; h < 2; ++h) cc[mi][h] = Cs[(wc + 2 * tq + h) * ldc + r0 + mi * 8 + gq];
      const double* Ub = Ws + gq * LDV + tq;
      if (c == cdiag) {
#pragma unroll
        for (int kk = 0; kk < 32; kk += 4) {
          const double bv = Ub[kk];
          const int l = kk + tq;
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) {
            const int r = mi * 8 + gq;
            double a = V[l * LDV + r];
            if (TT) {
              if (r > l) a = 0.0;
            } else {
              a = (r < l) ? 0.0 : ((r == l) ? 1.0 : a);
            }
            dmma_(cc[mi][0], cc[mi][1], a, bv);
          }
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < 32; kk += 4) {
          const double bv = Ub[kk];
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
            dmma_(cc[mi][0], cc[mi][1], V[(kk + tq) * LDV + mi * 8 + gq], bv);
        }
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int h = 0; h < 2; ++h) Cs[(wc + 2 * tq + h) * ldc + r0 + mi * 8 + gq] = cc[mi][h];
    }
  }
  wait_<0>();
  __syncthreads();
  // ---- store the slab
  for (int o = tid; o < W * crows; o += NT) {
    const int j = o / crows, r = o - j * crows;
    if (j < cvalid) Cg[(int64_t)j * ldcg + r] = Cs[j * ldc + r];
  }
}

template <int NW>
static size_t upd_smem(int nb) {
  return sizeof(double) * ((size_t)8 * NW * (rup32(nb) + 4) + (size_t)(DEPTH + 2) * CH +
                           (size_t)NW * 8 * LDV);
}

template <int NW>
static bool launch_nw(const double* A, Geo g, int k, const double* T, const int2* pairs,
                      int npairs, bool tt, double* base, int64_t ldc, int64_t ncols,
                      const uint8_t* dec, cudaStream_t st) {
  const size_t smem = upd_smem<NW>(g.nb);
  if (smem > 227 * 1024) return false;
  static bool attr = false;
  if (!attr) {
    smem_optin(k_qr_update2<NW, false, true>);
    smem_optin(k_qr_update2<NW, true, true>);
    attr = true;
  }
  const unsigned slabs = (unsigned)((ncols + 8 * NW - 1) / (8 * NW));
  if (!tt) {
    ::hlq::g_launches++;
    k_qr_update2<NW, false, true><<<dim3(slabs, g.n - k), NW * 32, smem, st>>>(
        A, g, k, T, nullptr, base, ldc, ncols, dec);
  } else {
    if (npairs <= 0) return true;
    ::hlq::g_launches++;
    k_qr_update2<NW, true, true><<<dim3(slabs, npairs), NW * 32, smem, st>>>(
        A, g, k, T, pairs, base, ldc, ncols, dec);
  }
  return true;
}

// UNMQR of every tile row k..n-1 (tt = false, T = GEQRT factors) or TTMQR of one level (tt = true,
// T = TTQRT factors) on the column block (base, ldc, ncols).  Requires ib = 32 and nb <= 512.
void launch_qr_update2(const double* A, Geo g, int k, const double* T, const int2* pairs,
                       int npairs, bool tt, double* base, int64_t ldc, int64_t ncols,
                       const uint8_t* dec, cudaStream_t st) {
  if (ncols <= 0) return;
  if (launch_nw<8>(A, g, k, T, pairs, npairs, tt, base, ldc, ncols, dec, st)) return;
  if (launch_nw<7>(A, g, k, T, pairs, npairs, tt, base, ldc, ncols, dec, st)) return;
  if (launch_nw<6>(A, g, k, T, pairs, npairs, tt, base, ldc, ncols, dec, st)) return;
  launch_nw<4>(A, g, k, T, pairs, npairs, tt, base, ldc, ncols, dec, st);
}

}  // namespace hlq
