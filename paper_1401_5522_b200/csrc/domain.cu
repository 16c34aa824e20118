// NEXT f1: diagonal-domain pivoting (DESIGN reading 33).
// The diagonal domain of step k is the panel tiles i >= k with i = k (mod D), D = the QR tree's
// domains.  The speculative factorization runs over the stacked domain (R x b, tile k first, out of
// place in Wd, ld R): unblocked right-looking elimination with partial pivoting over all R rows,
// separately rounded multiply / subtract and the first maximum, so Wd and the pivots are
// bit-identical to the oracle's getrf_stack.  One launch per column: every CTA scales and updates its
// rows with the current pivot row and takes its partial first maximum of the next column; the last
// CTA to finish (threadfence reduction) picks the pivot and swaps the two rows, which the next launch
// then reads.  An LU decision scatters Wd back over the domain tiles; the update stage applies the
// domain's row interchanges to the trailing columns before the Apply / Update GEMMs.
#include <math.h>

#include <algorithm>

#include "hlq_internal.cuh"

namespace hlq {

static unsigned grid_for(int64_t total) {
  int64_t b = (total + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)(b < 1 ? 1 : b);
}

// stack row r -> global row: the domain tiles are k, k + D, k + 2D, ... (only the last can be short)
__device__ __forceinline__ int64_t dom_row(Geo g, int k, int D, int64_t r) {
  const int64_t t = r / g.nb;
  return g.r0(k + (int)t * D) + (r - t * g.nb);
}

int64_t dom_rows(Geo g, int k, int D) {
  int64_t R = 0;
  for (int i = k; i < g.n; i += D) R += g.bs(i);
  return R;
}

// dir 0: Wd <- the domain's panel columns; dir 1 (dec[k] == LU): the domain's panel <- Wd
__global__ void k_dom_copy(double* __restrict__ A, Geo g, int k, int D, double* __restrict__ Wd,
                           int64_t R, int dir, const uint8_t* __restrict__ dec) {
  if (dir == 1 && dec != nullptr && dec[k] != HLQ_DEC_LU) return;
  const int bk = g.cbs(k);
  const int64_t k0 = g.r0(k), total = R * bk;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = idx / R, r = idx - c * R;
    double* a = A + (k0 + c) * g.lda + dom_row(g, k, D, r);
    if (dir == 0)
      Wd[idx] = *a;
    else
      *a = Wd[idx];
  }
}

// the same (|value|, NaN-canonical) key order as the tile GETRF: larger key, then smaller index
__device__ __forceinline__ unsigned long long dkey(double v) {
  v = fabs(v);
  if (v != v) return 0x7ff8000000000000ull;
  return (unsigned long long)__double_as_longlong(v);
}
__device__ __forceinline__ bool dbetter(unsigned long long ka, int ia, unsigned long long kb,
                                        int ib) {
  return ka > kb || (ka == kb && ia < ib);
}

constexpr int DT = 256;

// Column c of the stack elimination (c = -1: none), updating the columns (c, cend) of its 32-column
// sub-panel, then the pivot search of column cn (-1: none) with the swap of the whole row.  grid
// = G CTAs owning contiguous row ranges; part_key / part_idx hold the G partial maxima, *counter the
// arrivals.
__global__ void __launch_bounds__(DT) k_dom_step(double* __restrict__ Wd, int64_t R, int bk, int c,
                                                 int cend, int cn, int* __restrict__ ipiv,
                                                 int* __restrict__ zp,
                                                 unsigned long long* __restrict__ part_key,
                                                 int* __restrict__ part_idx,
                                                 unsigned int* __restrict__ counter) {
  __shared__ double urow[HLQ_MAX_NB];
  __shared__ unsigned long long sk[DT / 32];
  __shared__ int si[DT / 32];
  __shared__ bool last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t rpb = (R + gridDim.x - 1) / gridDim.x;
  const int64_t rb = (int64_t)blockIdx.x * rpb, re = min(R, rb + rpb);
  if (c >= 0) {
    for (int j = c + tid; j < cend; j += DT) urow[j] = __ldcg(Wd + (int64_t)j * R + c);
    __syncthreads();
    const double d = urow[c];
    if (d != 0.0) {  // exact zero pivot: the column stays unscaled, no update (ledger 7)
      for (int64_t r = max(rb, (int64_t)c + 1) + tid; r < re; r += DT) {
        const double l = Wd[(int64_t)c * R + r] / d;
        Wd[(int64_t)c * R + r] = l;
        for (int j = c + 1; j < cend; ++j)  // the sub-panel's columns (the rest: k_dom_trail)
          Wd[(int64_t)j * R + r] = __dsub_rn(Wd[(int64_t)j * R + r], __dmul_rn(l, urow[j]));
      }
    }
  }
  if (cn < 0 || cn >= bk) return;
  // partial first maximum of column cn over this CTA's rows >= cn
  unsigned long long bkey = 0ull;
  int bidx = 0x7fffffff;
  for (int64_t r = max(rb, (int64_t)cn) + tid; r < re; r += DT) {
    const unsigned long long kk = dkey(Wd[(int64_t)cn * R + r]);
    if (dbetter(kk, (int)r, bkey, bidx)) {
      bkey = kk;
      bidx = (int)r;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long ok = __shfl_xor_sync(0xffffffffu, bkey, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (dbetter(ok, oi, bkey, bidx)) {
      bkey = ok;
      bidx = oi;
    }
  }
  if (lane == 0) {
    sk[warp] = bkey;
    si[warp] = bidx;
  }
  __threadfence();  // this CTA's updates of Wd are visible before its arrival is counted
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < DT / 32; ++w)
      if (dbetter(sk[w], si[w], bkey, bidx)) {
        bkey = sk[w];
        bidx = si[w];
      }
    part_key[blockIdx.x] = bkey;
    part_idx[blockIdx.x] = bidx;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  // the last CTA: global first maximum (fixed order over the partials), row swap, pivot record
  __shared__ int p_sh;
  if (tid == 0) {
    unsigned long long gk = 0ull;
    int gi = 0x7fffffff;
    for (unsigned b = 0; b < gridDim.x; ++b) {
      const unsigned long long kb = __ldcg(part_key + b);
      const int ib2 = __ldcg(part_idx + b);
      if (dbetter(kb, ib2, gk, gi)) {
        gk = kb;
        gi = ib2;
      }
    }
    if (gi == 0x7fffffff || gi >= R) gi = cn;
    p_sh = gi;
    ipiv[cn] = gi;
    *counter = 0u;
  }
  __syncthreads();
  const int p = p_sh;
  if (p != cn) {
    for (int j = tid; j < bk; j += DT) {
      const double a = __ldcg(Wd + (int64_t)j * R + cn), b = __ldcg(Wd + (int64_t)j * R + p);
      Wd[(int64_t)j * R + cn] = b;
      Wd[(int64_t)j * R + p] = a;
    }
  }
  __syncthreads();
  if (tid == 0 && __ldcg(Wd + (int64_t)cn * R + cn) == 0.0) atomicOr(zp, 1);
}

// After a 32-column sub-panel [c0, c0 + pw): U12 = L11^-1 A12 on the sub-panel's rows (one thread per
// column, right-looking with the running sums in registers: per element the same sequence of
// separately rounded multiply / subtract as the unblocked elimination, c ascending).
__global__ void __launch_bounds__(128) k_dom_u12(double* __restrict__ Wd, int64_t R, int bk, int c0,
                                                 int pw) {
  __shared__ double L11[32][33];
  for (int o = threadIdx.x; o < 32 * 32; o += blockDim.x) {
    const int c = o >> 5, r = o & 31;
    L11[c][r] = (c < pw && r < pw) ? Wd[(int64_t)(c0 + c) * R + c0 + r] : 0.0;
  }
  __syncthreads();
  const int j = c0 + pw + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= bk) return;
  double* col = Wd + (int64_t)j * R + c0;
  double acc[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) acc[c] = c < pw ? col[c] : 0.0;
#pragma unroll
  for (int l = 0; l < 32; ++l) {
    if (l < pw) {
      const double u = acc[l];
      col[l] = u;
#pragma unroll
      for (int c = l + 1; c < 32; ++c) acc[c] = __dsub_rn(acc[c], __dmul_rn(L11[l][c], u));
    }
  }
}

// Trailing update of the stack after a sub-panel: rows [c0 + pw, R) x columns [c0 + pw, bk):
// W[r][j] -= sum_{c = c0}^{c0+pw-1} L[r][c] U[c][j], c ascending, separately rounded (bit-identical
// to the unblocked order).  64 x 64 output tiles, 4 x 4 per thread, L21 / U12 blocks in shared memory.
__global__ void __launch_bounds__(256) k_dom_trail(double* __restrict__ Wd, int64_t R, int bk,
                                                   int c0, int pw) {
  __shared__ double Ls[32][65];
  __shared__ double Us[32][65];
  const int64_t rbase = c0 + pw + (int64_t)blockIdx.x * 64;
  const int jbase = c0 + pw + blockIdx.y * 64;
  const int tid = threadIdx.x;
  for (int o = tid; o < 32 * 64; o += 256) {
    const int c = o >> 6, x = o & 63;
    const int64_t r = rbase + x;
    const int j = jbase + x;
    Ls[c][x] = (c < pw && r < R) ? Wd[(int64_t)(c0 + c) * R + r] : 0.0;
    Us[c][x] = (c < pw && j < bk) ? Wd[(int64_t)j * R + c0 + c] : 0.0;
  }
  __syncthreads();
  const int tr = tid & 15, tc = tid >> 4;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t r = rbase + tr + 16 * i;
      const int j = jbase + tc + 16 * q;
      acc[i][q] = (r < R && j < bk) ? Wd[(int64_t)j * R + r] : 0.0;
    }
  for (int c = 0; c < pw; ++c) {
    double l[4], u[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) l[i] = Ls[c][tr + 16 * i];
#pragma unroll
    for (int q = 0; q < 4; ++q) u[q] = Us[c][tc + 16 * q];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[i][q] = __dsub_rn(acc[i][q], __dmul_rn(l[i], u[q]));
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t r = rbase + tr + 16 * i;
      const int j = jbase + tc + 16 * q;
      if (r < R && j < bk) Wd[(int64_t)j * R + r] = acc[i][q];
    }
}

// top b x b of the stack -> W (ld nb) for the inverse / criterion kernels; identity permutations
__global__ void k_dom_top(const double* __restrict__ Wd, int64_t R, int bk, int ldw,
                          double* __restrict__ W, int* __restrict__ perm,
                          int* __restrict__ ipiv_step, const int* __restrict__ ipiv_stack) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < bk * bk;
       idx += gridDim.x * blockDim.x) {
    const int c = idx / bk, r = idx - c * bk;
    W[(int64_t)c * ldw + r] = Wd[(int64_t)c * R + r];
  }
  if (blockIdx.x == 0)
    for (int c = threadIdx.x; c < bk; c += blockDim.x) {
      perm[c] = c;
      ipiv_step[c] = ipiv_stack[c];
    }
}

void launch_dom_factor(double* A, Geo g, int k, int D, DevWork w, cudaStream_t st) {
  const int bk = g.cbs(k);
  const int64_t R = dom_rows(g, k, D);
  const unsigned G = (unsigned)std::min<int64_t>(2 * 148, (R + DT - 1) / DT);
  cudaMemsetAsync(w.zp, 0, sizeof(int), st);
  ::hlq::g_launches++;
  k_dom_copy<<<grid_for(R * bk), 256, 0, st>>>(A, g, k, D, w.wdom, R, 0, nullptr);
  int* ipiv_stack = w.dipiv + (size_t)k * g.nb;
  // blocked right-looking over 32-column sub-panels: per column one k_dom_step inside the
  // sub-panel, then U12 and the trailing update of the sub-panel's remaining columns
  auto step = [&](int c, int cend, int cn) {
    ::hlq::g_launches++;
    k_dom_step<<<G, DT, 0, st>>>(w.wdom, R, bk, c, cend, cn, ipiv_stack, w.zp, w.dom_key,
                                  w.dom_idx, w.dom_counter);
  };
  step(-1, 0, 0);
  for (int c0 = 0; c0 < bk; c0 += 32) {
    const int pw = std::min(32, bk - c0);
    const int nrest = bk - c0 - pw;
    // the sub-panel's last column defers the next search until U12 / the trailing update are done
    for (int c = c0; c < c0 + pw; ++c) step(c, c0 + pw, c + 1 < c0 + pw ? c + 1 : -1);
    if (nrest > 0) {
      ::hlq::g_launches += 2;
      k_dom_u12<<<(nrest + 127) / 128, 128, 0, st>>>(w.wdom, R, bk, c0, pw);
      dim3 tg((unsigned)((R - c0 - pw + 63) / 64), (unsigned)((nrest + 63) / 64));
      k_dom_trail<<<tg, 256, 0, st>>>(w.wdom, R, bk, c0, pw);
      step(-1, 0, c0 + pw);
    }
  }
  int* perm = reinterpret_cast<int*>(w.scratch + (size_t)2 * g.nb * g.nb);
  ::hlq::g_launches++;
  k_dom_top<<<8, 256, 0, st>>>(w.wdom, R, bk, g.nb, w.W, perm, w.ipiv + (size_t)k * g.nb,
                               ipiv_stack);
}

void launch_dom_commit(double* A, Geo g, int k, int D, DevWork w, cudaStream_t st) {
  const int bk = g.cbs(k);
  const int64_t R = dom_rows(g, k, D);
  ::hlq::g_launches++;
  k_dom_copy<<<grid_for(R * bk), 256, 0, st>>>(A, g, k, D, w.wdom, R, 1, w.dec);
}

// the domain's row interchanges (stack coordinates, LAPACK sequential order) on columns [c0, c1):
// one thread per column applies the bk swaps in order
__global__ void k_dom_swap_cols(double* __restrict__ A, Geo g, int k, int D,
                                const int* __restrict__ ipiv_stack, int64_t c0, int64_t c1,
                                const uint8_t* __restrict__ dec) {
  if (dec != nullptr && dec[k] != HLQ_DEC_LU) return;
  __shared__ int piv[HLQ_MAX_NB];
  const int bk = g.bs(k);
  for (int c = threadIdx.x; c < bk; c += blockDim.x) piv[c] = ipiv_stack[c];
  __syncthreads();
  const int64_t j = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= c1) return;
  double* col = A + j * g.lda;
  const int64_t k0 = g.r0(k);
  for (int c = 0; c < bk; ++c) {
    const int p = piv[c];
    if (p != c) {
      const int64_t rc = k0 + c, rp = dom_row(g, k, D, p);
      const double a = col[rc];
      col[rc] = col[rp];
      col[rp] = a;
    }
  }
}

void launch_dom_swap_cols(double* A, Geo g, int k, int D, const int* ipiv_stack, int64_t c0,
                          int64_t c1, const uint8_t* dec, cudaStream_t st) {
  if (c1 <= c0) return;
  ::hlq::g_launches++;
  k_dom_swap_cols<<<(unsigned)((c1 - c0 + 127) / 128), 128, 0, st>>>(A, g, k, D, ipiv_stack, c0,
                                                                     c1, dec);
}

// the solve's forward pass: the same interchanges on x (one thread, sequential)
__global__ void k_dom_swap_vec(double* __restrict__ x, Geo g, int k, int D,
                               const int* __restrict__ ipiv_stack) {
  if (threadIdx.x != 0) return;
  const int bk = g.bs(k);
  const int64_t k0 = g.r0(k);
  for (int c = 0; c < bk; ++c) {
    const int p = ipiv_stack[c];
    if (p != c) {
      const int64_t rc = k0 + c, rp = dom_row(g, k, D, p);
      const double a = x[rc];
      x[rc] = x[rp];
      x[rp] = a;
    }
  }
}

void launch_dom_swap_vec(double* x, Geo g, int k, int D, const int* ipiv_stack, cudaStream_t st) {
  ::hlq::g_launches++;
  k_dom_swap_vec<<<1, 32, 0, st>>>(x, g, k, D, ipiv_stack);
}

}  // namespace hlq
