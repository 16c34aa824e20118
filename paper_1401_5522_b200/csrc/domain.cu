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

// Column c of the stack elimination (c = -1: only the pivot search of column 0).  grid = G CTAs
// owning contiguous row ranges; part_key / part_idx hold the G partial maxima, *counter the arrivals.
__global__ void __launch_bounds__(DT) k_dom_step(double* __restrict__ Wd, int64_t R, int bk, int c,
                                                 int* __restrict__ ipiv, int* __restrict__ zp,
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
    for (int j = c + tid; j < bk; j += DT) urow[j] = __ldcg(Wd + (int64_t)j * R + c);
    __syncthreads();
    const double d = urow[c];
    if (d != 0.0) {  // exact zero pivot: the column stays unscaled, no update (ledger 7)
      for (int64_t r = max(rb, (int64_t)c + 1) + tid; r < re; r += DT) {
        const double l = Wd[(int64_t)c * R + r] / d;
        Wd[(int64_t)c * R + r] = l;
        for (int j = c + 1; j < bk; ++j)
          Wd[(int64_t)j * R + r] = __dsub_rn(Wd[(int64_t)j * R + r], __dmul_rn(l, urow[j]));
      }
    }
  }
  const int cn = c + 1;
  if (cn >= bk) return;
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
  for (int c = -1; c < bk; ++c) {
    ::hlq::g_launches++;
    k_dom_step<<<G, DT, 0, st>>>(w.wdom, R, bk, c, ipiv_stack, w.zp, w.dom_key, w.dom_idx,
                                  w.dom_counter);
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
