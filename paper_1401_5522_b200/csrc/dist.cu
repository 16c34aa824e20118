// Row e: the hybrid LU-QR factorization and solve on a P x Q process grid, 2D block-cyclic
// ("tile (i,j) is mapped onto process ((i-1) mod p, (j-1) mod q)"; 0-based here),
// one process per GPU with NCCL over NVLink, or P*Q "virtual ranks" emulated inside one process on
// one GPU (the collectives become stream-ordered device copies; the kernels are the same).
//
// Per step k (pk = k mod P, qk = k mod Q; the panel column lives on process column qk):
//   A  column qk: panel statistics of the local panel tiles (a1); the owner of A_kk runs the
//      speculative GETRF, the triangular inverses and ||A_kk^-1||_1 (a2, a3)
//   X1 column allgather of the statistics records (+ the owner's W, ipiv): the paper's "all-reduce
//      of the criterion data"
//   B  column qk: every rank reduces the records in global order and takes the SAME decision d_k on
//      its device (a4); LU: owner commits W, every rank TRSMs its panel tiles (a5); QR: GEQRT of the
//      local panel tiles and the intra-domain TT levels (a8, a9), domains = tile rows mod D with
//      P | D, so a domain never spans process rows
//   X2 column allgather of the domain-head R tiles
//   C  column qk: the inter-domain TTQRT merges, computed redundantly by every rank of the column
//      (a11); pack the panel package (panel tiles, T factors, merge reflectors, L^-1, perm, d_k)
//   X3 row broadcast of the package from column qk (the decision piggybacks on the panel,
//      P:468-470)
//   D  every rank: LU: process row pk applies SWPTRSM to row k (a6); QR: UNMQR of every local tile
//      row + intra-domain TTMQR levels (a10)
//   X4 column allgather of the domain-head rows (LU: row k)
//   E  every rank: LU: the Schur DGEMM with the received row k (a7); QR: the inter-domain TTMQR
//      merges, redundantly, then each rank keeps its own head rows (a11); growth partials (a12)
// The NCCL call sequence is identical for both branches, so the host never waits for d_k: every
// branch kernel is predicated on d_k in device memory, exactly as on one GPU.
#include <dlfcn.h>
#include <math.h>
#include <nccl.h>
#include <string.h>

#include <algorithm>
#include <functional>
#include <new>
#include <vector>

#include "handle.cuh"

namespace hlq {
void launch_solve_lu_fwd(const double* A, Geo g, int k, const int* ipiv, double* x,
                         cudaStream_t st);
void launch_solve_back(const double* A, Geo g, int k, double* x, cudaStream_t st);
}  // namespace hlq

using namespace hlq;

// ---------------------------------------------------------------------------------------------
// NCCL, loaded at run time (the process normally already holds torch's libnccl.so.2)
namespace {
struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;

bool nccl_load() {
  if (g_nccl.tried) return g_nccl.ok;
  g_nccl.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return false;
#define HLQ_SYM(f)                                                     \
  *(void**)(&g_nccl.f) = dlsym(h, "nccl" #f);                          \
  if (!g_nccl.f) return false;
  HLQ_SYM(GetUniqueId)
  HLQ_SYM(CommInitRank)
  HLQ_SYM(CommSplit)
  HLQ_SYM(CommDestroy)
  HLQ_SYM(Broadcast)
  HLQ_SYM(AllGather)
  HLQ_SYM(AllReduce)
  HLQ_SYM(GetErrorString)
#undef HLQ_SYM
  g_nccl.ok = true;
  return true;
}

int nccl_err(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return 0;
  fprintf(stderr, "[hlq] NCCL %s: %s\n", what, g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?");
  return HLQ_ERR_NCCL;
}

int cuda_check(cudaError_t e) {
  if (e == cudaSuccess) return 0;
  fprintf(stderr, "[hlq] CUDA error: %s\n", cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? HLQ_ERR_NOMEM : HLQ_ERR_CUDA;
}
}  // namespace

struct hlq_grid_s {
  int P = 1, Q = 1;
  int local = 1;       // 1: all P*Q ranks emulated in this process
  int rank = 0;        // this process's world rank (p = rank / Q, q = rank % Q)
  ncclComm_t world = nullptr, row = nullptr, col = nullptr, colp = nullptr;  // colp: panel stream
  // host-staged backend (hlq_grid_create_host): the caller's collectives on host buffers
  bool host = false;
  hlq_host_comm ops{};
  double* stage = nullptr;  // pinned staging buffer (grows)
  size_t stage_n = 0;
};

// ---------------------------------------------------------------------------------------------
// the per-rank collectives of the 2D grid, one entry point per kind: NCCL on the communicator of
// `comm` (HLQ_COMM_*), or -- host-staged backend -- stream sync, device -> pinned host copy, the
// caller's host collective on the same communicator, host -> device copy
namespace {
ncclComm_t comm_of(hlq_grid_s* g, int comm) {
  return comm == HLQ_COMM_ROW ? g->row
         : comm == HLQ_COMM_COL ? g->col
         : comm == HLQ_COMM_COL_PANEL ? g->colp
                                      : g->world;
}
int comm_size(hlq_grid_s* g, int comm) {
  return comm == HLQ_COMM_ROW ? g->Q : (comm == HLQ_COMM_WORLD ? g->P * g->Q : g->P);
}
double* host_stage(hlq_grid_s* g, size_t n) {
  if (n > g->stage_n) {
    if (g->stage) cudaFreeHost(g->stage);
    g->stage = nullptr;
    g->stage_n = 0;
    if (cudaMallocHost((void**)&g->stage, sizeof(double) * n) != cudaSuccess) return nullptr;
    g->stage_n = n;
  }
  return g->stage;
}
int host_rc(int r, const char* what) {
  if (r == 0) return 0;
  fprintf(stderr, "[hlq] host collective %s failed: %d\n", what, r);
  return HLQ_ERR_NCCL;
}
int xc_allgather(hlq_grid_s* g, int comm, const double* send, double* recv, int64_t count,
                 cudaStream_t st) {
  if (count <= 0) return 0;
  if (!g->host)
    return nccl_err(g_nccl.AllGather(send, recv, (size_t)count, ncclDouble, comm_of(g, comm), st),
                    "allgather");
  const int sz = comm_size(g, comm);
  double* h = host_stage(g, (size_t)count * (sz + 1));
  if (!h) return HLQ_ERR_NOMEM;
  if (cudaMemcpyAsync(h, send, sizeof(double) * count, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return HLQ_ERR_CUDA;
  int rc = host_rc(g->ops.allgather(g->ops.ctx, comm, h, h + count, count), "allgather");
  if (rc) return rc;
  if (cudaMemcpyAsync(recv, h + count, sizeof(double) * count * sz, cudaMemcpyHostToDevice, st) !=
          cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return HLQ_ERR_CUDA;
  return 0;
}
int xc_bcast(hlq_grid_s* g, int comm, double* buf, int64_t count, int root, cudaStream_t st) {
  if (count <= 0) return 0;
  if (!g->host)
    return nccl_err(g_nccl.Broadcast(buf, buf, (size_t)count, ncclDouble, root, comm_of(g, comm),
                                     st),
                    "broadcast");
  double* h = host_stage(g, (size_t)count);
  if (!h) return HLQ_ERR_NOMEM;
  if (cudaMemcpyAsync(h, buf, sizeof(double) * count, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return HLQ_ERR_CUDA;
  int rc = host_rc(g->ops.broadcast(g->ops.ctx, comm, h, count, root), "broadcast");
  if (rc) return rc;
  if (cudaMemcpyAsync(buf, h, sizeof(double) * count, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return HLQ_ERR_CUDA;
  return 0;
}
// op: 0 = sum, 1 = max
int xc_allreduce(hlq_grid_s* g, int comm, double* buf, int64_t count, int op, cudaStream_t st) {
  if (count <= 0) return 0;
  if (!g->host)
    return nccl_err(g_nccl.AllReduce(buf, buf, (size_t)count, ncclDouble, op ? ncclMax : ncclSum,
                                     comm_of(g, comm), st),
                    "allreduce");
  double* h = host_stage(g, (size_t)count);
  if (!h) return HLQ_ERR_NOMEM;
  if (cudaMemcpyAsync(h, buf, sizeof(double) * count, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return HLQ_ERR_CUDA;
  int rc = host_rc(g->ops.allreduce(g->ops.ctx, comm, h, count, op), "allreduce");
  if (rc) return rc;
  if (cudaMemcpyAsync(buf, h, sizeof(double) * count, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return HLQ_ERR_CUDA;
  return 0;
}
}  // namespace

// ---------------------------------------------------------------------------------------------
// block-cyclic index arithmetic (host and device)
namespace hlq {
__host__ __device__ inline int cyc_count(int n, int P, int p) {  // #{i in [0,n) : i mod P == p}
  return (n - p + P - 1) / P > 0 ? (n - p + P - 1) / P : 0;
}
__host__ __device__ inline int cyc_below(int k, int P, int p) {  // #{i in [0,k) : i mod P == p}
  return (k + P - 1 - p) / P;
}
inline int64_t cyc_extent(int64_t N, int nb, int P, int p) {     // local rows (ScaLAPACK numroc)
  const int n = (int)((N + nb - 1) / nb);
  const int mt = cyc_count(n, P, p);
  int64_t rows = (int64_t)mt * nb;
  if (mt > 0 && (n - 1) % P == p) rows -= (int64_t)n * nb - N;   // ragged last tile lives here
  return rows;
}

// Greedy halving tree (reading 16): with r live entries the bottom floor(r/2) are
// eliminated by the top ceil(r/2) (entry t kills entry ceil(r/2)+t).
static void halving(std::vector<int> live, std::vector<std::vector<int2>>& out) {
  while (live.size() > 1) {
    size_t r = live.size(), h = (r + 1) / 2;
    std::vector<int2> lv;
    for (size_t t = 0; t < r - h; ++t) lv.push_back(make_int2(live[t], live[h + t]));
    out.push_back(lv);
    live.resize(h);
  }
}

// Plan of step k for process row p (host logic; exported through hlq_dist_plan for the tests).
struct StepPlan {
  int li0 = 0, ms = 0, diag = 0;
  std::vector<int> head_local;                 // per slot t < c: local panel index of the head of
  std::vector<int> head_global;                //   domain d = p + P t (-1: domain empty)
  std::vector<std::vector<int2>> intra;        // TT levels inside the local domains (panel indices)
};

static StepPlan plan_step(int n, int P, int D, int p, int k) {
  StepPlan s;
  const int c = D / P;
  s.li0 = cyc_below(k, P, p);
  s.ms = cyc_count(n, P, p) - s.li0;
  if (s.ms < 0) s.ms = 0;
  s.diag = (k % P == p) ? 1 : 0;
  std::vector<std::vector<std::vector<int2>>> per(c);
  size_t depth = 0;
  for (int t = 0; t < c; ++t) {
    const int d = p + P * t;
    const int i0 = k + ((d - k) % D + D) % D;
    std::vector<int> rows;
    for (int i = i0; i < n; i += D) rows.push_back(i / P - s.li0);
    s.head_global.push_back(i0 < n ? i0 : -1);
    s.head_local.push_back(i0 < n ? i0 / P - s.li0 : -1);
    halving(rows, per[t]);
    depth = std::max(depth, per[t].size());
  }
  for (size_t l = 0; l < depth; ++l) {
    std::vector<int2> lv;
    for (int t = 0; t < c; ++t)
      if (l < per[t].size()) lv.insert(lv.end(), per[t][l].begin(), per[t][l].end());
    s.intra.push_back(lv);
  }
  return s;
}

// the inter-domain merges of step k in slot indices s = (d mod P) * c + d / P (heads ascending)
static std::vector<std::vector<int2>> plan_inter(int n, int P, int D, int k) {
  const int c = D / P;
  std::vector<std::pair<int, int>> heads;  // (global head, slot)
  for (int d = 0; d < D; ++d) {
    const int i0 = k + ((d - k) % D + D) % D;
    if (i0 < n) heads.push_back({i0, (d % P) * c + d / P});
  }
  std::sort(heads.begin(), heads.end());
  std::vector<int> live;
  for (auto& h : heads) live.push_back(h.second);
  std::vector<std::vector<int2>> lv;
  halving(live, lv);
  return lv;
}

struct HeadIdx {
  int v[16];
};

// ---------------------------------------------------------------------------------------------
// kernels of the distributed path (data movement + record reduction; all arithmetic of the method
// stays in the shared single-GPU kernels)

// X1 record: [s (ms_max)][away_max (nb)][local_max (nb)][inv_norm][zp][W (nb*nb)][ipiv (nb)]
__global__ void k_pack_owner(double* rec, const double* inv_norm, const int* zp, const double* W,
                             const int* ipiv_ws, int nb, int bk) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  if (tid == 0) {
    rec[0] = inv_norm[0];
    rec[1] = (double)zp[0];
  }
  for (int t = tid; t < nb * nb; t += nth) rec[2 + t] = W[t];
  for (int t = tid; t < bk; t += nth) rec[2 + nb * nb + t] = (double)ipiv_ws[t];
}

// Reduce the P records of column qk in GLOBAL tile order into the single-GPU DevWork layout, so the
// unchanged k_decide sees exactly what it sees on one GPU.
__global__ void k_unpack_stats(const double* __restrict__ recs, int64_t rec_count, int ms_max,
                               int k, int n, int P, int pk, int nb, int bk, double* s,
                               double* away_max, double* local_max, double* inv_norm, int* zp,
                               double* W, int* ipiv_ws) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  for (int p = 0; p < P; ++p) {
    const double* r = recs + (int64_t)p * rec_count;
    const int li0 = cyc_below(k, P, p);
    const int ms = cyc_count(n, P, p) - li0;
    for (int j = tid; j < ms; j += nth) {
      const int i = (li0 + j) * P + p;  // global tile index
      if (i > k) s[i] = r[j];
    }
  }
  for (int c = tid; c < nb; c += nth) {
    double m = 0.0;
    for (int p = 0; p < P; ++p) m = nanmax(m, recs[(int64_t)p * rec_count + ms_max + c]);
    away_max[c] = m;
    local_max[c] = recs[(int64_t)pk * rec_count + ms_max + nb + c];
  }
  const double* o = recs + (int64_t)pk * rec_count + ms_max + 2 * nb;
  if (tid == 0) {
    inv_norm[0] = o[0];
    zp[0] = (int)o[1];
  }
  for (int t = tid; t < nb * nb; t += nth) W[t] = o[2 + t];
  for (int t = tid; t < bk; t += nth) ipiv_ws[t] = (int)o[2 + nb * nb + t];
}

// slots t < c of dst (slot stride nb*W, ld nb) <- rows of local panel tile idx.v[t] (rows valid =
// min(nb, prow - idx*nb)), columns [0, W) of src (ld lds); zero rows / empty slots.
__global__ void k_pack_rows(double* __restrict__ dst, int c, HeadIdx idx,
                            const double* __restrict__ src, int64_t lds, int64_t prow, int nb,
                            int64_t W, int64_t Wvalid) {
  const int64_t per = (int64_t)nb * W;
  const int64_t total = per * c;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int slot = (int)(t / per);
    const int64_t o = t - slot * per;
    const int64_t col = o / nb;
    const int r = (int)(o - col * nb);
    const int h = idx.v[slot];
    double v = 0.0;
    if (h >= 0 && col < Wvalid) {
      const int64_t row = (int64_t)h * nb + r;
      if (row < prow && r < nb) v = src[col * lds + row];
    }
    dst[t] = v;
  }
}

// stacked (S*nb x W, ld S*nb) <- gathered slots (slot s at s*nb*W, ld nb)
__global__ void k_stack(double* __restrict__ dst, const double* __restrict__ src, int S, int nb,
                        int64_t W) {
  const int64_t total = (int64_t)S * nb * W;
  const int64_t ldd = (int64_t)S * nb;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(t / ((int64_t)nb * W));
    const int64_t o = t - (int64_t)s * nb * W;
    const int64_t col = o / nb;
    const int r = (int)(o - col * nb);
    dst[col * ldd + (int64_t)s * nb + r] = src[t];
  }
}

// own slots s0 + t of a stacked buffer (ld lds) -> local rows of panel tile idx.v[t] (dst, ldd),
// columns [0, W); upper != 0: only r <= col (the R / TT-reflector triangle of a head tile).
// Predicated on dec[0] == want when dec != nullptr.
__global__ void k_unstack_rows(double* __restrict__ dst, int64_t ldd, int64_t prow, int c,
                               HeadIdx idx, int s0, const double* __restrict__ src, int64_t lds,
                               int nb, int64_t W, int upper, const uint8_t* __restrict__ dec,
                               int want) {
  if (dec != nullptr && dec[0] != want) return;
  const int64_t per = (int64_t)nb * W;
  const int64_t total = per * c;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int slot = (int)(t / per);
    const int h = idx.v[slot];
    if (h < 0) continue;
    const int64_t o = t - slot * per;
    const int64_t col = o / nb;
    const int r = (int)(o - col * nb);
    const int64_t row = (int64_t)h * nb + r;
    if (row >= prow || (upper && r > col)) continue;
    dst[col * ldd + row] = src[col * lds + (int64_t)(s0 + slot) * nb + r];
  }
}

// plain predicated copy of n doubles
__global__ void k_copy_vec(double* __restrict__ dst, const double* __restrict__ src, int64_t n,
                           const uint8_t* __restrict__ dec, int want) {
  if (dec != nullptr && dec[0] != want) return;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    dst[t] = src[t];
}

// meta: [d_k, margin_k, flags_k, -][perm (nb)][the diagonal domain's stacked pivots (nb)]
__global__ void k_meta_pack(double* meta, const uint8_t* dec, const double* margin,
                            const int* flags, const int* perm, const int* dipiv, int bk, int k,
                            int nb) {
  if (threadIdx.x == 0) {
    meta[0] = (double)dec[k];
    meta[1] = margin[k];
    meta[2] = (double)flags[k];
  }
  for (int t = threadIdx.x; t < bk; t += blockDim.x) {
    meta[4 + t] = (double)perm[t];
    meta[4 + nb + t] = dipiv != nullptr ? (double)dipiv[t] : 0.0;
  }
}
__global__ void k_meta_unpack(const double* meta, uint8_t* dec, double* margin, int* flags,
                              int* perm, int* dipiv, int bk, int k, int nb) {
  if (threadIdx.x == 0) {
    dec[k] = (uint8_t)meta[0];
    margin[k] = meta[1];
    flags[k] = (int)meta[2];
  }
  for (int t = threadIdx.x; t < bk; t += blockDim.x) {
    perm[t] = (int)meta[4 + t];
    if (dipiv != nullptr) dipiv[t] = (int)meta[4 + nb + t];
  }
}

// final status scan of one rank: non-finite entries, exact zeros on the diagonal of the global
// diagonal tiles it owns.  flag[0] |= non-finite, flag[1] |= zero diagonal.
__global__ void k_dist_scan(const double* __restrict__ A, int64_t lld, int64_t mloc, int64_t nloc,
                            int nb, int n, int64_t N, int p, int q, int P, int Q, int* flag) {
  int bad = 0, zero = 0;
  const int64_t total = mloc * nloc;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t / mloc, r = t - c * mloc;
    const double a = A[c * lld + r];
    if (!isfinite(a)) bad = 1;
    const int li = (int)(r / nb), lj = (int)(c / nb);
    const int gi = li * P + p, gj = lj * Q + q;
    if (gi == gj && (r - (int64_t)li * nb) == (c - (int64_t)lj * nb) && a == 0.0) zero = 1;
  }
  bad = __syncthreads_or(bad);
  zero = __syncthreads_or(zero);
  if (threadIdx.x == 0) {
    if (bad) atomicOr(&flag[0], 1);
    if (zero) atomicOr(&flag[1], 1);
  }
  (void)n;
  (void)N;
}

// reductions at the end: dst[0..n] = gstep with NaN -> +inf; dst[n+1+j] = status[j] (j < 4)
__global__ void k_pack_final(double* dst, const double* gstep, const int* status, int n1) {
  for (int t = threadIdx.x; t < n1; t += blockDim.x) {
    double v = gstep[t];
    dst[t] = (v != v) ? INFINITY : v;
  }
  if (threadIdx.x < 4) dst[n1 + threadIdx.x] = (double)status[threadIdx.x];
}

// x segments: local tile rows of process row p <-> global vector
__global__ void k_gather_seg(double* __restrict__ seg, const double* __restrict__ x, int64_t mloc,
                             int nb, int P, int p) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < mloc;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t li = r / nb;
    seg[r] = x[(li * P + p) * nb + (r - li * nb)];
  }
}
__global__ void k_scatter_segs(double* __restrict__ x, const double* __restrict__ segs,
                               int64_t seg_cap, int64_t N, int nb, int P) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < N;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = g / nb;
    const int p = (int)(i % P);
    const int64_t li = i / P;
    x[g] = segs[p * seg_cap + li * nb + (g - i * nb)];
  }
}

// counter-based uniform generator on a rank's block-cyclic local array (the same G_u(seed, j*N + i)
// as hlq_generate_uniform on the global matrix; DESIGN.md input recipe)
__device__ __forceinline__ uint64_t dmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__global__ void k_generate_cyclic(double* __restrict__ A, int64_t lld, int64_t mloc, int64_t nloc,
                                  int64_t N, int nb, int P, int Q, int p, int q, uint64_t key) {
  const uint64_t GAMMA = 0x9E3779B97F4A7C15ULL;
  const int64_t total = mloc * nloc;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t / mloc, r = t - c * mloc;
    const int64_t li = r / nb, lj = c / nb;
    const int64_t gi = (li * P + p) * nb + (r - li * nb);
    const int64_t gj = (lj * Q + q) * nb + (c - lj * nb);
    const uint64_t idx = (uint64_t)gj * (uint64_t)N + (uint64_t)gi;
    const uint64_t u = dmix64(key + (idx + 1ULL) * GAMMA);
    A[c * lld + r] = (double)(u >> 11) * 0x1.0p-53 - 0.5;
  }
}

// HPL3 pieces on a rank: part[r] = sum_{local c} A(r,c) x[gcol(c)], part[mloc + r] = sum |A(r,c)|
// (columns in ascending local order; the row reduction over process columns follows)
__global__ void k_residual_part(const double* __restrict__ A, int64_t lld, int64_t mloc,
                                int64_t nloc, int nb, int Q, int q, const double* __restrict__ x,
                                double* __restrict__ part) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= mloc) return;
  double acc = 0.0, rs = 0.0;
  for (int64_t c = 0; c < nloc; ++c) {
    const int64_t lj = c / nb;
    const double a = A[c * lld + r];
    acc += a * x[(lj * Q + q) * nb + (c - lj * nb)];
    rs += fabs(a);
  }
  part[r] = acc;
  part[mloc + r] = rs;
}
__global__ void k_add_vec(double* __restrict__ dst, const double* __restrict__ src, int64_t n) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    dst[t] += src[t];
}
// out[0] = max_r |part[r] - b[grow(r)]|, out[1] = max_r part[mloc + r], out[2] = max |x| (atomic)
__global__ void k_residual_max(const double* __restrict__ part, int64_t mloc, int nb, int P, int p,
                               const double* __restrict__ b, const double* __restrict__ x,
                               int64_t N, double* out) {
  double r0 = 0.0, r1 = 0.0, r2 = 0.0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < mloc;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t li = r / nb;
    const int64_t g = (li * P + p) * nb + (r - li * nb);
    r0 = nanmax(r0, fabs(part[r] - b[g]));
    r1 = nanmax(r1, part[mloc + r]);
  }
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < N;
       g += (int64_t)gridDim.x * blockDim.x)
    r2 = nanmax(r2, fabs(x[g]));
  atomic_max_nonneg(&out[0], r0);
  atomic_max_nonneg(&out[1], r1);
  atomic_max_nonneg(&out[2], r2);
}

static unsigned blocks_for(int64_t total) {
  int64_t b = (total + 255) / 256;
  if (b > 148 * 8) b = 148 * 8;
  return (unsigned)(b < 1 ? 1 : b);
}

// ---------------------------------------------------------------------------------------------
// per-rank state
struct Ctx {
  int p = 0, q = 0;
  double* A = nullptr;
  int64_t lld = 1, mloc = 0, nloc = 0;
  int mt = 0, nt = 0;
  void* block = nullptr;
  DevWork w{};
  int* ipiv = nullptr;
  int* dipiv = nullptr;  // diagonal-domain pivoting: per step the stacked pivots (n x nb)
  double *Tg = nullptr, *Ttt = nullptr, *mstore = nullptr;
  double *rec_send = nullptr, *rec_recv = nullptr, *head_send = nullptr, *head_recv = nullptr;
  double *pkg = nullptr, *hr_send = nullptr, *hr_recv = nullptr, *HR = nullptr;
  double *pkgs[2] = {nullptr, nullptr}, *scrs[2] = {nullptr, nullptr};  // per step parity
  double *xseg = nullptr, *xk = nullptr, *hx_send = nullptr, *hx_recv = nullptr, *HX = nullptr;
  double *xg = nullptr, *fin = nullptr;
  int2* pairs = nullptr;
  std::vector<StepPlan> plan;                          // per step
  std::vector<std::vector<const int2*>> intra_ptr, inter_ptr;
  std::vector<std::vector<int>> intra_cnt, inter_cnt;
};

struct DistState {
  hlq_grid_s* gr = nullptr;
  int P = 1, Q = 1, D = 1, c = 1, S = 1, ib = 32, nb = 0, n = 0;
  bool dpiv = false;  // diagonal-domain pivoting (NEXT f1 on the grid, DESIGN reading 33)
  int64_t N = 0;
  int ms_max = 0, mt_max = 0;
  int64_t rec_count = 0, seg_cap = 0;
  cudaStream_t st = nullptr;
  cudaStream_t sp = nullptr;                    // high-priority panel stream (lookahead)
  cudaEvent_t ev_part0 = nullptr, ev_panel = nullptr;
  std::vector<Ctx> ctx;
  std::vector<std::vector<std::vector<int2>>> inter;  // per step
  // package layout (offsets in doubles) for a rank with `prow` panel rows and `ms` panel tiles
  int64_t off_Tg(int64_t prow) const { return prow * nb; }
  int64_t off_Ttt(int64_t prow, int ms) const { return off_Tg(prow) + (int64_t)ms * ib * nb; }
  int64_t off_HM(int64_t prow, int ms) const { return off_Ttt(prow, ms) + (int64_t)ms * ib * nb; }
  int64_t off_MT(int64_t prow, int ms) const { return off_HM(prow, ms) + (int64_t)S * nb * nb; }
  int64_t off_Li(int64_t prow, int ms) const { return off_MT(prow, ms) + (int64_t)S * ib * nb; }
  int64_t off_meta(int64_t prow, int ms) const { return off_Li(prow, ms) + (int64_t)nb * nb; }
  int64_t pkg_count(int64_t prow, int ms) const { return off_meta(prow, ms) + 4 + 2 * nb; }
  int64_t mstore_stride() const { return (int64_t)S * nb * nb + (int64_t)S * ib * nb; }
  ~DistState() {
    for (auto& c : ctx)
      if (c.block) cudaFree(c.block);
    if (ev_part0) cudaEventDestroy(ev_part0);
    if (ev_panel) cudaEventDestroy(ev_panel);
    if (sp) cudaStreamDestroy(sp);
  }
};
// Element counts (doubles) of the four per-step exchanges, as every rank computes them (host):
// [0] X1 statistics record (column qk allgather, per rank), [1] X2 head tiles (column qk allgather,
// per rank), [2] X3 panel package of process row p (row broadcast), [3] X4 head rows of process
// column q (column allgather, per rank).  Ranks of one communicator must agree (NCCL deadlocks
// otherwise): tests/test_dist_host.py checks it across gloo ranks.
inline void step_counts(int64_t N, int nb, int P, int Q, int D, int ib, int p, int q, int k,
                        int64_t out[4]) {
  const int n = (int)((N + nb - 1) / nb);
  const int c = D / P, S = D;
  const int ms_max = cyc_count(n, P, 0);
  out[0] = ms_max + 3 * (int64_t)nb + 2 + (int64_t)nb * nb;
  out[1] = (int64_t)c * nb * nb;
  const int li0 = cyc_below(k, P, p);
  const int ms = std::max(0, cyc_count(n, P, p) - li0);
  const int64_t prow = std::max<int64_t>(0, cyc_extent(N, nb, P, p) - (int64_t)li0 * nb);
  out[2] = prow * nb + 2 * (int64_t)ms * ib * nb + (int64_t)S * nb * nb + (int64_t)S * ib * nb +
           (int64_t)nb * nb + 4 + 2 * (int64_t)nb;
  const int lc1 = cyc_below(k + 1, Q, q);
  const int64_t ncl = std::max<int64_t>(0, cyc_extent(N, nb, Q, q) - (int64_t)lc1 * nb);
  out[3] = (int64_t)c * nb * ncl;
}
}  // namespace hlq

// ---------------------------------------------------------------------------------------------
// collectives over the contexts hosted by this process
namespace {
using Buf = std::function<double*(Ctx&)>;

// allgather inside process column q: member p's `count` doubles -> every member's recv at p*count
int col_allgather(DistState& ds, int q, const Buf& send, const Buf& recv, int64_t count,
                  cudaStream_t st, bool panel_comm) {
  if (count <= 0) return 0;
  if (!ds.gr->local) {
    for (auto& c : ds.ctx)
      if (c.q == q)
        return xc_allgather(ds.gr, panel_comm ? HLQ_COMM_COL_PANEL : HLQ_COMM_COL, send(c), recv(c),
                            count, st);
    return 0;
  }
  for (auto& dst : ds.ctx) {
    if (dst.q != q) continue;
    for (auto& src : ds.ctx) {
      if (src.q != q) continue;
      int rc = cuda_check(cudaMemcpyAsync(recv(dst) + (int64_t)src.p * count, send(src),
                                          sizeof(double) * count, cudaMemcpyDeviceToDevice, st));
      if (rc) return rc;
    }
  }
  return 0;
}

// broadcast inside every process row from process column root; count may depend on the row
int row_bcast(DistState& ds, int root, const Buf& buf, const std::function<int64_t(int)>& count,
              cudaStream_t st) {
  if (!ds.gr->local) {
    for (auto& c : ds.ctx) {
      int64_t n = count(c.p);
      if (n <= 0) return 0;
      return xc_bcast(ds.gr, HLQ_COMM_ROW, buf(c), n, root, st);
    }
    return 0;
  }
  for (auto& dst : ds.ctx) {
    if (dst.q == root) continue;
    for (auto& src : ds.ctx) {
      if (src.p != dst.p || src.q != root) continue;
      int64_t n = count(src.p);
      if (n <= 0) continue;
      int rc = cuda_check(cudaMemcpyAsync(buf(dst), buf(src), sizeof(double) * n,
                                          cudaMemcpyDeviceToDevice, st));
      if (rc) return rc;
    }
  }
  return 0;
}

// broadcast inside process column q from process row root
int col_bcast(DistState& ds, int q, int root, const Buf& buf, int64_t count) {
  if (count <= 0) return 0;
  if (!ds.gr->local) {
    for (auto& c : ds.ctx)
      if (c.q == q)
        return xc_bcast(ds.gr, HLQ_COMM_COL, buf(c), count, root, ds.st);
    return 0;
  }
  for (auto& src : ds.ctx) {
    if (src.q != q || src.p != root) continue;
    for (auto& dst : ds.ctx) {
      if (dst.q != q || dst.p == root) continue;
      int rc = cuda_check(cudaMemcpyAsync(buf(dst), buf(src), sizeof(double) * count,
                                          cudaMemcpyDeviceToDevice, ds.st));
      if (rc) return rc;
    }
  }
  return 0;
}
}  // namespace

// ---------------------------------------------------------------------------------------------
namespace hlq {

static HeadIdx head_idx(const StepPlan& sp) {
  HeadIdx h;
  for (int t = 0; t < 16; ++t) h.v[t] = t < (int)sp.head_local.size() ? sp.head_local[t] : -1;
  return h;
}

static int dist_alloc(DistState& ds, Ctx& c, const hlq_options& opt, bool has_ref) {
  const int nb = ds.nb, n = ds.n, ib = ds.ib, S = ds.S, P = ds.P, cc = ds.c;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) / 256 * 256 + 256;
    return o;
  };
  // pairs: count all levels of all steps
  size_t npairs = 0;
  for (int k = 0; k < n; ++k) {
    for (auto& lv : c.plan[k].intra) npairs += lv.size();
    for (auto& lv : ds.inter[k]) npairs += lv.size();
  }
  const int64_t mloc = std::max<int64_t>(c.mloc, 1), nloc = std::max<int64_t>(c.nloc, 1);
  const int mt = std::max(c.mt, 1), nt = std::max(c.nt, 1);
  size_t o_dec = take(n), o_mg = take(8 * n), o_fl = take(4 * n), o_st = take(16),
         o_gs = take(8 * (n + 1)), o_s = take(8 * n), o_lm = take(8 * nb), o_am = take(8 * nb),
         o_inv = take(8), o_zp = take(4), o_W = take(8 * (size_t)nb * nb), o_ipw = take(4 * nb),
         o_scr = take(8 * (2 * (size_t)nb * nb + nb)), o_wsp = take(8 * (size_t)mloc * nb),
         o_wsr = take(8 * (size_t)nb * nloc), o_fo = take(n), o_rd = take(n), o_rm = take(8 * n),
         o_ip = take(4 * (size_t)n * nb), o_Tg = take(8 * (size_t)mt * nt * ib * nb),
         o_Tt = take(8 * (size_t)mt * nt * ib * nb),
         o_ms = take(8 * (size_t)nt * ds.mstore_stride()), o_rs = take(8 * ds.rec_count),
         o_rr = take(8 * (size_t)P * ds.rec_count), o_hs = take(8 * (size_t)cc * nb * nb),
         o_hr = take(8 * (size_t)P * cc * nb * nb), o_pk = take(8 * (size_t)ds.pkg_count(mloc, mt)),
         o_pk2 = take(8 * (size_t)ds.pkg_count(mloc, mt)),
         o_scr2 = take(8 * (2 * (size_t)nb * nb + nb)),
         o_rws = take(8 * (size_t)cc * nb * nloc), o_rwr = take(8 * (size_t)P * cc * nb * nloc),
         o_HR = take(8 * (size_t)S * nb * nloc), o_xs = take(8 * (size_t)ds.seg_cap),
         o_xk = take(8 * (size_t)nb), o_hxs = take(8 * (size_t)cc * nb),
         o_hxr = take(8 * (size_t)P * cc * nb), o_HX = take(8 * (size_t)S * nb),
         o_xg = take(8 * (size_t)P * ds.seg_cap), o_fin = take(8 * (size_t)(n + 8)),
         o_pr = take(sizeof(int2) * (npairs + 1)),
         o_wd = take(ds.dpiv ? 8 * (size_t)mloc * nb : 8),
         o_dp = take(ds.dpiv ? 4 * (size_t)n * nb : 8), o_dk = take(8 * 2 * 148),
         o_di = take(4 * 2 * 148), o_dc = take(4);
  if (cudaMalloc(&c.block, off) != cudaSuccess) {
    cudaGetLastError();
    c.block = nullptr;
    return HLQ_ERR_NOMEM;
  }
  char* b = (char*)c.block;
  DevWork& w = c.w;
  w.dec = (uint8_t*)(b + o_dec);
  w.margin = (double*)(b + o_mg);
  w.flags = (int*)(b + o_fl);
  w.status = (int*)(b + o_st);
  w.gstep = (double*)(b + o_gs);
  w.s = (double*)(b + o_s);
  w.local_max = (double*)(b + o_lm);
  w.away_max = (double*)(b + o_am);
  w.inv_norm = (double*)(b + o_inv);
  w.zp = (int*)(b + o_zp);
  w.W = (double*)(b + o_W);
  w.ipiv_ws = (int*)(b + o_ipw);
  w.scratch = (double*)(b + o_scr);
  w.ws_panel = (double*)(b + o_wsp);
  w.ws_row = (double*)(b + o_wsr);
  w.forced = opt.forced ? (uint8_t*)(b + o_fo) : nullptr;
  w.ref_dec = has_ref ? (uint8_t*)(b + o_rd) : nullptr;
  w.ref_margin = has_ref ? (double*)(b + o_rm) : nullptr;
  w.ipiv = (int*)(b + o_ip);
  w.Tg = nullptr;
  w.Ttt = nullptr;
  w.pairs = nullptr;
  w.colpart = nullptr;
  w.wdom = ds.dpiv ? (double*)(b + o_wd) : nullptr;
  w.dipiv = ds.dpiv ? (int*)(b + o_dp) : nullptr;
  w.dom_key = (unsigned long long*)(b + o_dk);
  w.dom_idx = (int*)(b + o_di);
  w.dom_counter = (unsigned int*)(b + o_dc);
  c.ipiv = w.ipiv;
  c.dipiv = w.dipiv;
  c.Tg = (double*)(b + o_Tg);
  c.Ttt = (double*)(b + o_Tt);
  c.mstore = (double*)(b + o_ms);
  c.rec_send = (double*)(b + o_rs);
  c.rec_recv = (double*)(b + o_rr);
  c.head_send = (double*)(b + o_hs);
  c.head_recv = (double*)(b + o_hr);
  c.pkg = (double*)(b + o_pk);
  c.pkgs[0] = c.pkg;
  c.pkgs[1] = (double*)(b + o_pk2);
  c.scrs[0] = w.scratch;
  c.scrs[1] = (double*)(b + o_scr2);
  c.hr_send = (double*)(b + o_rws);
  c.hr_recv = (double*)(b + o_rwr);
  c.HR = (double*)(b + o_HR);
  c.xseg = (double*)(b + o_xs);
  c.xk = (double*)(b + o_xk);
  c.hx_send = (double*)(b + o_hxs);
  c.hx_recv = (double*)(b + o_hxr);
  c.HX = (double*)(b + o_HX);
  c.xg = (double*)(b + o_xg);
  c.fin = (double*)(b + o_fin);
  c.pairs = (int2*)(b + o_pr);
  // pair upload
  std::vector<int2> flat;
  flat.reserve(npairs);
  c.intra_ptr.assign(n, {});
  c.intra_cnt.assign(n, {});
  c.inter_ptr.assign(n, {});
  c.inter_cnt.assign(n, {});
  for (int k = 0; k < n; ++k) {
    for (auto& lv : c.plan[k].intra) {
      c.intra_ptr[k].push_back(c.pairs + flat.size());
      c.intra_cnt[k].push_back((int)lv.size());
      flat.insert(flat.end(), lv.begin(), lv.end());
    }
    for (auto& lv : ds.inter[k]) {
      c.inter_ptr[k].push_back(c.pairs + flat.size());
      c.inter_cnt[k].push_back((int)lv.size());
      flat.insert(flat.end(), lv.begin(), lv.end());
    }
  }
  int rc = 0;
  if (!flat.empty() &&
      (rc = cuda_check(cudaMemcpyAsync(c.pairs, flat.data(), sizeof(int2) * flat.size(),
                                       cudaMemcpyHostToDevice, ds.st))))
    return rc;
  if (w.forced && (rc = cuda_check(cudaMemcpyAsync(w.forced, opt.forced, n, cudaMemcpyHostToDevice,
                                                   ds.st))))
    return rc;
  if (has_ref) {
    if ((rc = cuda_check(cudaMemcpyAsync(w.ref_dec, opt.ref_dec, n, cudaMemcpyHostToDevice, ds.st))))
      return rc;
    if ((rc = cuda_check(cudaMemcpyAsync(w.ref_margin, opt.ref_margin, sizeof(double) * n,
                                         cudaMemcpyHostToDevice, ds.st))))
      return rc;
  }
  cudaMemsetAsync(w.status, 0, 16, ds.st);
  cudaMemsetAsync(w.gstep, 0, sizeof(double) * (n + 1), ds.st);
  cudaMemsetAsync(w.ipiv, 0, sizeof(int) * (size_t)n * nb, ds.st);
  cudaMemsetAsync(w.dec, 0, n, ds.st);
  cudaMemsetAsync(w.dom_counter, 0, sizeof(unsigned int), ds.st);
  if (c.dipiv) cudaMemsetAsync(c.dipiv, 0, sizeof(int) * (size_t)n * nb, ds.st);
  cudaMemsetAsync(c.xseg, 0, sizeof(double) * ds.seg_cap, ds.st);
  cudaMemsetAsync(w.scratch, 0, sizeof(double) * (2 * (size_t)nb * nb + nb), ds.st);
  cudaMemsetAsync(c.scrs[1], 0, sizeof(double) * (2 * (size_t)nb * nb + nb), ds.st);
  return cuda_check(cudaGetLastError());
}

// panel geometry of rank c at step k: local panel tiles li0.. of column lk
static Geo panel_geo(const DistState& ds, const Ctx& c, const StepPlan& sp, int64_t lda) {
  Geo g{};
  g.N = c.mloc - (int64_t)sp.li0 * ds.nb;
  if (g.N < 0) g.N = 0;
  g.lda = lda;
  g.nb = ds.nb;
  g.n = sp.ms;
  const int64_t bk = std::min<int64_t>(ds.nb, ds.N - (int64_t)0);
  (void)bk;
  g.Nc = 0;
  return g;
}

// the owner's DevWork for the domain kernels, which index step k of a local panel geometry as
// step 0: the step's stacked and tile pivots and its decision at offset 0
static DevWork dom_view(const Ctx& c, DevWork w, int k, int nb) {
  w.ipiv = c.ipiv + (int64_t)k * nb;
  w.dipiv = c.dipiv + (int64_t)k * nb;
  w.dec = w.dec + k;
  return w;
}

// The factorization schedule: panel stage P(k) (A, X1, B, X2, C, X3) on the high-priority panel
// stream, update stage U(k) (D, X4, E) on the caller's stream in two parts: part 0 = the local
// column tile k+1 (process column (k+1) mod Q only), part 1 = the rest.  P(k+1) starts as soon as
// U(k) part 0 is done and overlaps U(k) part 1 (lookahead depth 1, as on one GPU).  The panel
// package and the L^-1 / perm scratch are double-buffered by step parity; the panel stream uses its
// own column communicator (colp) so every NCCL communicator is driven by exactly one stream.
static int dist_factor(DistState& ds, int crit, double alpha, const hlq_options& opt, Prof& PR) {
  const int n = ds.n, nb = ds.nb, P = ds.P, Q = ds.Q, S = ds.S, cc = ds.c, ib = ds.ib;
  cudaStream_t st = ds.st, sp = ds.sp;
  const bool has_forced = opt.forced != nullptr;
  const bool has_ref = ds.ctx[0].w.ref_dec != nullptr;
  const bool criterion_needed = !has_forced && alpha > 0.0 && !isinf(alpha) &&
                                crit != HLQ_CRIT_RANDOM;
  auto known_of = [&](int k) {
    if (has_forced) return opt.forced[k] ? (int)HLQ_DEC_QR : (int)HLQ_DEC_LU;
    if (alpha == 0.0) return (int)HLQ_DEC_QR;
    return -1;
  };
  Geo gglob{};
  gglob.N = ds.N;
  gglob.Nc = ds.N;
  gglob.lda = ds.N;
  gglob.nb = nb;
  gglob.n = n;
  // per-parity views of the workspace (scratch = L^-1 | U^-1 | perm)
  auto wk = [&](Ctx& c, int k) {
    DevWork w = c.w;
    w.scratch = c.scrs[k & 1];
    return w;
  };

  // ======================================== panel stage P(k) on stream s
  auto panel = [&](int k, cudaStream_t s) -> int {
    int rc = 0;
    const int pk = k % P, qk = k % Q, lk = k / Q;
    const int bk = (int)std::min<int64_t>(nb, ds.N - (int64_t)k * nb);
    const int known = known_of(k);
    // ---- A: statistics, speculative GETRF on the owner
    for (auto& c : ds.ctx) {
      if (c.q != qk) continue;
      const StepPlan& sp_ = c.plan[k];
      DevWork w = wk(c, k);
      double* Apan = c.A + (int64_t)lk * nb * c.lld + (int64_t)sp_.li0 * nb;
      Geo gP = panel_geo(ds, c, sp_, c.lld);
      gP.Nc = bk;
      PR.begin(HLQ_PROF_CRITERION, s);
      cudaMemsetAsync(c.rec_send, 0, sizeof(double) * ds.rec_count, s);
      if (sp_.ms > 0 && criterion_needed) {
        if (ds.dpiv && sp_.diag)  // the whole diagonal domain is local: tiles 0, c, 2c, ...
          launch_panel_stats_domain_to(Apan, gP, 0, ds.c, c.rec_send,
                                       c.rec_send + ds.ms_max + nb, c.rec_send + ds.ms_max, s);
        else
          launch_panel_stats_to(Apan, gP, 0, sp_.diag, c.rec_send, c.rec_send + ds.ms_max + nb,
                                c.rec_send + ds.ms_max, s);
      }
      PR.end(s);
      if (sp_.diag) {
        PR.begin(HLQ_PROF_GETRF, s);
        cudaMemsetAsync(w.zp, 0, sizeof(int), s);
        cudaMemsetAsync(w.inv_norm, 0, sizeof(double), s);
        if (known != HLQ_DEC_QR) {
          if (ds.dpiv)  // partial pivoting over the stacked domain; W <- its pivoted top tile
            launch_dom_factor(Apan, gP, 0, ds.c, dom_view(c, w, k, nb), s);
          else
            launch_getrf(Apan, gP, 0, w, true, s);
          if (criterion_needed && crit != HLQ_CRIT_MUMPS) {  // the inverse norm only
            launch_tri_inv(gP, 0, w, w.scratch, w.scratch + (size_t)nb * nb, s);
            launch_invnorm(gP, 0, w, s, opt.invnorm_estimate);
          }
        }
        ::hlq::g_launches++;
        k_pack_owner<<<16, 256, 0, s>>>(c.rec_send + ds.ms_max + 2 * nb, w.inv_norm, w.zp, w.W,
                                        w.ipiv_ws, nb, bk);
        PR.end(s);
      }
    }
    PR.begin(HLQ_PROF_OTHER, s);
    if ((rc = col_allgather(ds, qk, [](Ctx& c) { return c.rec_send; },
                            [](Ctx& c) { return c.rec_recv; }, ds.rec_count, s, true)))
      return rc;
    PR.end(s);
    // ---- B: decision, LU panel / QR panel + intra-domain tree
    for (auto& c : ds.ctx) {
      if (c.q != qk) continue;
      const StepPlan& sp_ = c.plan[k];
      DevWork w = wk(c, k);
      double* Apan = c.A + (int64_t)lk * nb * c.lld + (int64_t)sp_.li0 * nb;
      Geo gP = panel_geo(ds, c, sp_, c.lld);
      gP.Nc = bk;
      const uint8_t* dk = w.dec + k;
      PR.begin(HLQ_PROF_CRITERION, s);
      ::hlq::g_launches++;
      k_unpack_stats<<<16, 256, 0, s>>>(c.rec_recv, ds.rec_count, ds.ms_max, k, n, P, pk, nb, bk,
                                        w.s, w.away_max, w.local_max, w.inv_norm, w.zp, w.W,
                                        w.ipiv_ws);
      launch_decide(gglob, k, crit, alpha, opt.mumps_reading, opt.tie_rel_tol, has_forced ? 1 : 0,
                    has_ref ? 1 : 0, w, s);
      PR.end(s);
      int* perm = reinterpret_cast<int*>(w.scratch + (size_t)2 * nb * nb);
      if (known != HLQ_DEC_QR) {
        PR.begin(HLQ_PROF_LU_TRSM, s);
        if (sp_.diag && !ds.dpiv)
          launch_lu_commit(Apan, gP, 0, w.W, w.ipiv_ws, c.ipiv + (int64_t)k * nb, perm, dk, s);
        const int64_t r0 = sp_.diag ? bk : 0;
        const int64_t M = gP.N - r0;
        // Eliminate with U_kk from the gathered speculative LU W (blocked substitution, trsm.cu)
        if (M > 0)
          launch_trsm_eliminate(Apan, c.lld, r0, 0, M, bk, w.W, nb, dk, 0, HLQ_DEC_LU, s);
        // domain pivoting: the stacked LU replaces the domain's tiles (the diagonal tile and
        // the local tiles c, 2c, ...; U_kk^-1 above applies to the tiles off the domain only)
        if (sp_.diag && ds.dpiv) launch_dom_commit(Apan, gP, 0, ds.c, dom_view(c, w, k, nb), s);
        PR.end(s);
      }
      if (known != HLQ_DEC_LU && sp_.ms > 0) {
        PR.begin(HLQ_PROF_QR_GEQRT, s);
        double* Tgk = c.Tg + ((int64_t)lk * c.mt + sp_.li0) * ib * nb;
        double* Ttk = c.Ttt + ((int64_t)lk * c.mt + sp_.li0) * ib * nb;
        launch_qr_panel_tc(Apan, gP, 0, ib, Tgk, Ttk, nullptr, 0, dk, false, s);
        for (size_t l = 0; l < c.intra_ptr[k].size(); ++l)
          launch_qr_panel_tc(Apan, gP, 0, ib, Tgk, Ttk, c.intra_ptr[k][l], c.intra_cnt[k][l], dk,
                             true, s);
        PR.end(s);
      }
      ::hlq::g_launches++;
      k_pack_rows<<<blocks_for((int64_t)cc * nb * nb), 256, 0, s>>>(
          c.head_send, cc, head_idx(sp_), Apan, c.lld, gP.N, nb, nb, bk);
    }
    PR.begin(HLQ_PROF_OTHER, s);
    if ((rc = col_allgather(ds, qk, [](Ctx& c) { return c.head_send; },
                            [](Ctx& c) { return c.head_recv; }, (int64_t)cc * nb * nb, s, true)))
      return rc;
    PR.end(s);
    // ---- C: inter-domain merges (redundant on the column), package
    for (auto& c : ds.ctx) {
      if (c.q != qk) continue;
      const StepPlan& sp_ = c.plan[k];
      DevWork w = wk(c, k);
      double* Apan = c.A + (int64_t)lk * nb * c.lld + (int64_t)sp_.li0 * nb;
      Geo gP = panel_geo(ds, c, sp_, c.lld);
      gP.Nc = bk;
      const uint8_t* dk = w.dec + k;
      const int64_t prow = gP.N;
      double* pk_ = c.pkgs[k & 1];
      double* HM = pk_ + ds.off_HM(prow, sp_.ms);
      double* MT = pk_ + ds.off_MT(prow, sp_.ms);
      Geo gH{};
      gH.N = (int64_t)S * nb;
      gH.lda = (int64_t)S * nb;
      gH.nb = nb;
      gH.n = S;
      gH.Nc = bk;
      ::hlq::g_launches++;
      k_stack<<<blocks_for((int64_t)S * nb * nb), 256, 0, s>>>(HM, c.head_recv, S, nb, nb);
      PR.begin(HLQ_PROF_QR_GEQRT, s);
      if (known != HLQ_DEC_LU) {
        for (size_t l = 0; l < c.inter_ptr[k].size(); ++l)
          launch_qr_panel_tc(HM, gH, 0, ib, nullptr, MT, c.inter_ptr[k][l], c.inter_cnt[k][l], dk,
                             true, s);
        // own heads: R / TT-reflector triangles back into A, merge T factors into the local store
        ::hlq::g_launches++;
        k_unstack_rows<<<blocks_for((int64_t)cc * nb * nb), 256, 0, s>>>(
            Apan, c.lld, prow, cc, head_idx(sp_), c.p * cc, HM, (int64_t)S * nb, nb, bk, 1, dk,
            HLQ_DEC_QR);
        for (int t = 0; t < cc; ++t) {
          const int hl = sp_.head_local[t], hg = sp_.head_global[t];
          if (hl < 0 || hg == k) continue;
          ::hlq::g_launches++;
          k_copy_vec<<<8, 256, 0, s>>>(c.Ttt + ((int64_t)lk * c.mt + sp_.li0 + hl) * ib * nb,
                                       MT + (int64_t)(c.p * cc + t) * ib * nb, (int64_t)ib * nb, dk,
                                       HLQ_DEC_QR);
        }
        // the solve replays the merges: keep HM + MT of this step
        double* ms_ = c.mstore + (int64_t)lk * ds.mstore_stride();
        cudaMemcpyAsync(ms_, HM, sizeof(double) * ds.mstore_stride(), cudaMemcpyDeviceToDevice, s);
      }
      // package: panel tiles, T factors, (HM, MT already in place), L^-1, perm, d_k
      if (prow > 0)
        cudaMemcpy2DAsync(pk_, sizeof(double) * prow, Apan, sizeof(double) * c.lld,
                          sizeof(double) * prow, bk, cudaMemcpyDeviceToDevice, s);
      if (sp_.ms > 0) {
        cudaMemcpyAsync(pk_ + ds.off_Tg(prow), c.Tg + ((int64_t)lk * c.mt + sp_.li0) * ib * nb,
                        sizeof(double) * sp_.ms * ib * nb, cudaMemcpyDeviceToDevice, s);
        cudaMemcpyAsync(pk_ + ds.off_Ttt(prow, sp_.ms),
                        c.Ttt + ((int64_t)lk * c.mt + sp_.li0) * ib * nb,
                        sizeof(double) * sp_.ms * ib * nb, cudaMemcpyDeviceToDevice, s);
      }
      // the package's L slot carries W (L_kk \\ U_kk): the row ranks' Apply solves with L_kk
      cudaMemcpyAsync(pk_ + ds.off_Li(prow, sp_.ms), w.W, sizeof(double) * nb * nb,
                      cudaMemcpyDeviceToDevice, s);
      ::hlq::g_launches++;
      k_meta_pack<<<1, 256, 0, s>>>(pk_ + ds.off_meta(prow, sp_.ms), w.dec, w.margin, w.flags,
                                    reinterpret_cast<int*>(w.scratch + (size_t)2 * nb * nb),
                                    ds.dpiv ? c.dipiv + (int64_t)k * nb : nullptr, bk, k, nb);
      PR.end(s);
    }
    auto pcount = [&](int p) {
      int64_t cnt[4];
      step_counts(ds.N, nb, P, Q, ds.D, ib, p, 0, k, cnt);
      return cnt[2];
    };
    PR.begin(HLQ_PROF_OTHER, s);
    const int par = k & 1;
    if ((rc = row_bcast(ds, qk, [par](Ctx& c) { return c.pkgs[par]; }, pcount, s))) return rc;
    PR.end(s);
    return cuda_check(cudaGetLastError());
  };

  // ======================================== update stage U(k), part 0 or 1, on stream s
  // local trailing columns [lc1*nb, nloc) split at the local column tile of global tile k+1
  auto part_range = [&](int k, int q, int64_t nloc, int part, int64_t& co, int64_t& w) {
    const int lc1 = cyc_below(k + 1, Q, q);
    const int64_t ncl = std::max<int64_t>(0, nloc - (int64_t)lc1 * nb);
    const int64_t w0 = (k + 1 < n && (k + 1) % Q == q) ? std::min<int64_t>(nb, ncl) : 0;
    co = part == 0 ? 0 : w0;
    w = part == 0 ? w0 : ncl - w0;
    return lc1;
  };
  auto update = [&](int k, int part, cudaStream_t s) -> int {
    int rc = 0;
    const int bk = (int)std::min<int64_t>(nb, ds.N - (int64_t)k * nb);
    const int known = known_of(k);
    const int par = k & 1;
    // ---- D: SWPTRSM / UNMQR + intra TTMQR, then pack the head rows
    for (auto& c : ds.ctx) {
      const StepPlan& sp_ = c.plan[k];
      DevWork w = wk(c, k);
      const int64_t prow = std::max<int64_t>(0, c.mloc - (int64_t)sp_.li0 * nb);
      double* pk_ = c.pkgs[par];
      const uint8_t* dk = w.dec + k;
      int* perm = reinterpret_cast<int*>(w.scratch + (size_t)2 * nb * nb);
      if (part == 0) {
        ::hlq::g_launches++;
        k_meta_unpack<<<1, 256, 0, s>>>(pk_ + ds.off_meta(prow, sp_.ms), w.dec, w.margin, w.flags,
                                        perm, ds.dpiv ? c.dipiv + (int64_t)k * nb : nullptr, bk,
                                        k, nb);
      }
      int64_t co, ncl;
      const int lc1 = part_range(k, c.q, c.nloc, part, co, ncl);
      if (ncl <= 0 || prow <= 0) continue;
      double* base = c.A + ((int64_t)lc1 * nb + co) * c.lld + (int64_t)sp_.li0 * nb;
      Geo gK{};
      gK.N = prow;
      gK.lda = prow;
      gK.nb = nb;
      gK.n = sp_.ms;
      gK.Nc = bk;
      if (known != HLQ_DEC_QR && sp_.diag) {
        PR.begin(HLQ_PROF_LU_UPDATE, s);
        if (ds.dpiv) {
          // the domain's row interchanges on this rank's trailing columns (the domain's rows are
          // all on process row pk), before the Apply (whose permutation is then the identity)
          Geo gS{};
          gS.N = prow;
          gS.lda = c.lld;
          gS.nb = nb;
          gS.n = sp_.ms;
          gS.Nc = bk;
          launch_dom_swap_cols(base, gS, 0, ds.c, c.dipiv + (int64_t)k * nb, 0, ncl, dk, s);
        }
        launch_trsm_apply(base, c.lld, 0, 0, ncl, bk, pk_ + ds.off_Li(prow, sp_.ms), nb, perm, dk,
                          0, HLQ_DEC_LU, s);
        PR.end(s);
      }
      if (known != HLQ_DEC_LU && sp_.ms > 0) {
        PR.begin(HLQ_PROF_QR_UNMQR, s);
        const int nl = (int)c.intra_ptr[k].size();
        launch_qr_update_dmma(pk_, gK, 0, ib, pk_ + ds.off_Tg(prow), pk_ + ds.off_Ttt(prow, sp_.ms),
                              c.intra_ptr[k].data(), c.intra_cnt[k].data(), nl, base, c.lld, ncl,
                              dk, 0, s);
        for (int l = 0; l < nl; ++l)
          launch_qr_update_dmma(pk_, gK, 0, ib, pk_ + ds.off_Tg(prow),
                                pk_ + ds.off_Ttt(prow, sp_.ms), c.intra_ptr[k].data(),
                                c.intra_cnt[k].data(), nl, base, c.lld, ncl, dk, 1 + l, s);
        PR.end(s);
      }
      ::hlq::g_launches++;
      k_pack_rows<<<blocks_for((int64_t)cc * nb * ncl), 256, 0, s>>>(
          c.hr_send, cc, head_idx(sp_), base, c.lld, prow, nb, ncl, ncl);
    }
    // ---- X4: head rows of this part's columns, every process column with a non-empty part
    PR.begin(HLQ_PROF_OTHER, s);
    for (int q = 0; q < Q; ++q) {
      int64_t co, ncl;
      part_range(k, q, cyc_extent(ds.N, nb, Q, q), part, co, ncl);
      if ((rc = col_allgather(ds, q, [](Ctx& c) { return c.hr_send; },
                              [](Ctx& c) { return c.hr_recv; }, (int64_t)cc * nb * ncl, s, false)))
        return rc;
    }
    PR.end(s);
    // ---- E: Schur DGEMM / inter-domain TTMQR; growth
    const int dk_dom = k % ds.D;
    const int slot_k = (dk_dom % P) * cc + dk_dom / P;
    for (auto& c : ds.ctx) {
      const StepPlan& sp_ = c.plan[k];
      DevWork w = wk(c, k);
      const int64_t prow = std::max<int64_t>(0, c.mloc - (int64_t)sp_.li0 * nb);
      int64_t co, ncl;
      const int lc1 = part_range(k, c.q, c.nloc, part, co, ncl);
      if (ncl <= 0) continue;
      double* pk_ = c.pkgs[par];
      const uint8_t* dk = w.dec + k;
      double* base = c.A + ((int64_t)lc1 * nb + co) * c.lld + (int64_t)sp_.li0 * nb;
      const int64_t ldh = (int64_t)S * nb;
      ::hlq::g_launches++;
      k_stack<<<blocks_for(ldh * ncl), 256, 0, s>>>(c.HR, c.hr_recv, S, nb, ncl);
      const int64_t r0 = sp_.diag ? bk : 0;
      if (known != HLQ_DEC_QR && prow - r0 > 0) {
        PR.begin(HLQ_PROF_LU_UPDATE, s);
        launch_dgemm(base + r0, c.lld, pk_ + r0, prow, c.HR + (int64_t)slot_k * nb, ldh, prow - r0,
                     ncl, bk, true, true, dk, 0, HLQ_DEC_LU, s);
        PR.end(s);
      }
      if (known != HLQ_DEC_LU) {
        PR.begin(HLQ_PROF_QR_UNMQR, s);
        Geo gH{};
        gH.N = ldh;
        gH.lda = ldh;
        gH.nb = nb;
        gH.n = S;
        gH.Nc = bk;
        const int nl = (int)c.inter_ptr[k].size();
        double* HM = pk_ + ds.off_HM(prow, sp_.ms);
        double* MT = pk_ + ds.off_MT(prow, sp_.ms);
        for (int l = 0; l < nl; ++l)
          launch_qr_update_dmma(HM, gH, 0, ib, nullptr, MT, c.inter_ptr[k].data(),
                                c.inter_cnt[k].data(), nl, c.HR, ldh, ncl, dk, 1 + l, s);
        if (prow > 0 && nl > 0) {
          ::hlq::g_launches++;
          k_unstack_rows<<<blocks_for((int64_t)cc * nb * ncl), 256, 0, s>>>(
              base, c.lld, prow, cc, head_idx(sp_), c.p * cc, c.HR, ldh, nb, ncl, 0, dk, HLQ_DEC_QR);
        }
        PR.end(s);
      }
      if (opt.track_growth && k + 1 < n && prow - r0 > 0) {
        PR.begin(HLQ_PROF_GROWTH, s);
        Geo gT{};
        gT.N = prow - r0;
        gT.Nc = c.nloc;
        gT.lda = c.lld;
        gT.nb = nb;
        gT.n = sp_.ms - sp_.diag;
        const int64_t cb = (int64_t)lc1 * nb + co;
        launch_tile_norm_max(c.A + (int64_t)sp_.li0 * nb + r0, gT, 0, w.gstep + k + 1, s, nullptr,
                             0, 0, cb, cb + ncl);
        PR.end(s);
      }
    }
    return cuda_check(cudaGetLastError());
  };

  // ======================================== driver
  int rc = 0;
  // a12 at k = 0: max tile norm of every local tile
  if (opt.track_growth)
    for (auto& c : ds.ctx) {
      if (c.mloc <= 0 || c.nloc <= 0) continue;
      Geo g{};
      g.N = c.mloc;
      g.Nc = c.nloc;
      g.lda = c.lld;
      g.nb = nb;
      g.n = c.mt;
      launch_tile_norm_max(c.A, g, 0, c.w.gstep, st, nullptr, 0, 0, 0, c.nloc);
    }
  cudaEventRecord(ds.ev_part0, st);
  cudaStreamWaitEvent(sp, ds.ev_part0, 0);
  if ((rc = panel(0, sp))) return rc;
  cudaEventRecord(ds.ev_panel, sp);
  for (int k = 0; k < n; ++k) {
    cudaStreamWaitEvent(st, ds.ev_panel, 0);
    if ((rc = update(k, 0, st))) return rc;
    if (k + 1 < n) {
      cudaEventRecord(ds.ev_part0, st);
      cudaStreamWaitEvent(sp, ds.ev_part0, 0);
      if ((rc = panel(k + 1, sp))) return rc;
      cudaEventRecord(ds.ev_panel, sp);
    }
    if ((rc = update(k, 1, st))) return rc;
  }
  // final scan + reductions
  for (auto& c : ds.ctx) {
    if (c.mloc > 0 && c.nloc > 0) {
      ::hlq::g_launches++;
      k_dist_scan<<<148 * 4, 256, 0, st>>>(c.A, c.lld, c.mloc, c.nloc, nb, n, ds.N, c.p, c.q, P, Q,
                                           c.w.status + 2);
    }
    ::hlq::g_launches++;
    k_pack_final<<<1, 256, 0, st>>>(c.fin, c.w.gstep, c.w.status, n + 1);
  }
  if (!ds.gr->local) {
    Ctx& c = ds.ctx[0];
    if ((rc = xc_allreduce(ds.gr, HLQ_COMM_WORLD, c.fin, n + 5, 1, st))) return rc;
  }
  return cuda_check(cudaGetLastError());
}

static int dist_solve(DistState& ds, const std::vector<uint8_t>& dec, const double* b, double* x) {
  const int n = ds.n, nb = ds.nb, P = ds.P, Q = ds.Q, S = ds.S, cc = ds.c, ib = ds.ib;
  cudaStream_t st = ds.st;
  int rc = 0;
  for (auto& c : ds.ctx) {
    cudaMemsetAsync(c.xseg, 0, sizeof(double) * ds.seg_cap, st);
    if (c.mloc > 0) {
      ::hlq::g_launches++;
      k_gather_seg<<<blocks_for(c.mloc), 256, 0, st>>>(c.xseg, b, c.mloc, nb, P, c.p);
    }
  }
  auto seg_count = [&](int p) { return cyc_extent(ds.N, nb, P, p); };
  Geo gH{};
  gH.N = (int64_t)S * nb;
  gH.lda = (int64_t)S * nb;
  gH.nb = nb;
  gH.n = S;
  for (int k = 0; k < n; ++k) {
    const int pk = k % P, qk = k % Q, lk = k / Q;
    const int bk = (int)std::min<int64_t>(nb, ds.N - (int64_t)k * nb);
    if (dec[k] == HLQ_DEC_LU) {
      for (auto& c : ds.ctx) {
        if (c.q != qk || c.p != pk) continue;
        const StepPlan& sp = c.plan[k];
        double* Apan = c.A + (int64_t)lk * nb * c.lld + (int64_t)sp.li0 * nb;
        Geo gP = panel_geo(ds, c, sp, c.lld);
        gP.Nc = bk;
        if (ds.dpiv) {  // the domain's interchanges on x (its rows are local), then L_kk^-1
          launch_dom_swap_vec(c.xseg + (int64_t)sp.li0 * nb, gP, 0, ds.c,
                              c.dipiv + (int64_t)k * nb, st);
          launch_solve_lu_fwd(Apan, gP, 0, nullptr, c.xseg + (int64_t)sp.li0 * nb, st);
        } else {
          launch_solve_lu_fwd(Apan, gP, 0, c.ipiv + (int64_t)k * nb,
                              c.xseg + (int64_t)sp.li0 * nb, st);
        }
        cudaMemcpyAsync(c.xk, c.xseg + (int64_t)sp.li0 * nb, sizeof(double) * bk,
                        cudaMemcpyDeviceToDevice, st);
      }
      if ((rc = col_bcast(ds, qk, pk, [](Ctx& c) { return c.xk; }, bk))) return rc;
      for (auto& c : ds.ctx) {
        if (c.q != qk || c.p == pk) continue;
        const StepPlan& sp = c.plan[k];
        const int64_t prow = std::max<int64_t>(0, c.mloc - (int64_t)sp.li0 * nb);
        double* Apan = c.A + (int64_t)lk * nb * c.lld + (int64_t)sp.li0 * nb;
        launch_gemv_sub(c.xseg + (int64_t)sp.li0 * nb, Apan, c.lld, prow, bk, c.xk, st);
      }
    } else {
      gH.Nc = bk;
      for (auto& c : ds.ctx) {
        if (c.q != qk) continue;
        const StepPlan& sp = c.plan[k];
        const int64_t prow = std::max<int64_t>(0, c.mloc - (int64_t)sp.li0 * nb);
        double* Apan = c.A + (int64_t)lk * nb * c.lld + (int64_t)sp.li0 * nb;
        Geo gP = panel_geo(ds, c, sp, c.lld);
        gP.Nc = bk;
        double* xs = c.xseg + (int64_t)sp.li0 * nb;
        if (sp.ms > 0)
          launch_qr_apply(Apan, gP, 0, ib, c.Tg + ((int64_t)lk * c.mt + sp.li0) * ib * nb,
                          c.Ttt + ((int64_t)lk * c.mt + sp.li0) * ib * nb, c.intra_ptr[k].data(),
                          c.intra_cnt[k].data(), (int)c.intra_ptr[k].size(), xs,
                          std::max<int64_t>(prow, 1), 1, nullptr, st);
        ::hlq::g_launches++;
        k_pack_rows<<<blocks_for((int64_t)cc * nb), 256, 0, st>>>(c.hx_send, cc, head_idx(sp), xs,
                                                                  std::max<int64_t>(prow, 1), prow,
                                                                  nb, 1, 1);
      }
      if ((rc = col_allgather(ds, qk, [](Ctx& c) { return c.hx_send; },
                              [](Ctx& c) { return c.hx_recv; }, (int64_t)cc * nb, st, false)))
        return rc;
      for (auto& c : ds.ctx) {
        if (c.q != qk) continue;
        const StepPlan& sp = c.plan[k];
        const int64_t prow = std::max<int64_t>(0, c.mloc - (int64_t)sp.li0 * nb);
        double* xs = c.xseg + (int64_t)sp.li0 * nb;
        ::hlq::g_launches++;
        k_stack<<<blocks_for((int64_t)S * nb), 256, 0, st>>>(c.HX, c.hx_recv, S, nb, 1);
        const double* ms_ = c.mstore + (int64_t)lk * ds.mstore_stride();
        const int nl = (int)c.inter_ptr[k].size();
        if (nl > 0) {
          launch_tt_apply(ms_, gH, 0, ib, ms_ + (int64_t)S * nb * nb, c.inter_ptr[k].data(),
                          c.inter_cnt[k].data(), nl, c.HX, (int64_t)S * nb, 1, nullptr, st);
          if (prow > 0) {
            ::hlq::g_launches++;
            k_unstack_rows<<<blocks_for((int64_t)cc * nb), 256, 0, st>>>(
                xs, std::max<int64_t>(prow, 1), prow, cc, head_idx(sp), c.p * cc, c.HX,
                (int64_t)S * nb, nb, 1, 0, nullptr, 0);
          }
        }
      }
    }
    if ((rc = row_bcast(ds, qk, [](Ctx& c) { return c.xseg; }, seg_count, st))) return rc;
  }
  for (int k = n - 1; k >= 0; --k) {
    const int pk = k % P, qk = k % Q, lk = k / Q;
    const int bk = (int)std::min<int64_t>(nb, ds.N - (int64_t)k * nb);
    for (auto& c : ds.ctx) {
      if (c.q != qk || c.p != pk) continue;
      const StepPlan& sp = c.plan[k];
      double* Apan = c.A + (int64_t)lk * nb * c.lld + (int64_t)sp.li0 * nb;
      Geo gP = panel_geo(ds, c, sp, c.lld);
      gP.Nc = bk;
      launch_solve_back(Apan, gP, 0, c.xseg + (int64_t)sp.li0 * nb, st);
      cudaMemcpyAsync(c.xk, c.xseg + (int64_t)sp.li0 * nb, sizeof(double) * bk,
                      cudaMemcpyDeviceToDevice, st);
    }
    if ((rc = col_bcast(ds, qk, pk, [](Ctx& c) { return c.xk; }, bk))) return rc;
    for (auto& c : ds.ctx) {
      if (c.q != qk) continue;
      const StepPlan& sp = c.plan[k];
      launch_gemv_sub(c.xseg, c.A + (int64_t)lk * nb * c.lld, c.lld, (int64_t)sp.li0 * nb, bk,
                      c.xk, st);
    }
    if ((rc = row_bcast(ds, qk, [](Ctx& c) { return c.xseg; }, seg_count, st))) return rc;
  }
  // full x on every rank: allgather of the segments in each process column
  for (int q = 0; q < Q; ++q)
    if ((rc = col_allgather(ds, q, [](Ctx& c) { return c.xseg; }, [](Ctx& c) { return c.xg; },
                            ds.seg_cap, st, false)))
      return rc;
  Ctx& c0 = ds.ctx[0];
  ::hlq::g_launches++;
  k_scatter_segs<<<blocks_for(ds.N), 256, 0, st>>>(x, c0.xg, ds.seg_cap, ds.N, nb, P);
  return cuda_check(cudaGetLastError());
}

int dist_solve_entry(hlq_factors_t f, const double* b, double* x) {
  DistState& ds = *f->dist;
  int rc = dist_solve(ds, f->dec, b, x);
  if (rc) return rc;
  if (f->blocking) return cuda_check(cudaStreamSynchronize(ds.st));
  return 0;
}

void dist_free(DistState* d) { delete d; }

}  // namespace hlq

// ---------------------------------------------------------------------------------------------
extern "C" {

int hlq_nccl_unique_id(void* id128) {
  if (!id128) return -1;
  if (!nccl_load()) return HLQ_ERR_NCCL;
  ncclUniqueId id;
  int rc = nccl_err(g_nccl.GetUniqueId(&id), "GetUniqueId");
  if (rc) return rc;
  memcpy(id128, &id, sizeof(id));
  return 0;
}

int hlq_grid_create_nccl(const void* id128, int32_t nranks, int32_t rank, int32_t P, int32_t Q,
                         hlq_grid_t* out) {
  if (!out) return -6;
  *out = nullptr;
  if (!id128) return -1;
  if (nranks < 1) return -2;
  if (rank < 0 || rank >= nranks) return -3;
  if (P < 1) return -4;
  if (Q < 1 || P * Q != nranks) return -5;
  if (!nccl_load()) return HLQ_ERR_NCCL;
  hlq_grid_s* g = new (std::nothrow) hlq_grid_s();
  if (!g) return HLQ_ERR_NOMEM;
  g->P = P;
  g->Q = Q;
  g->local = 0;
  g->rank = rank;
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  int rc = nccl_err(g_nccl.CommInitRank(&g->world, nranks, id, rank), "CommInitRank");
  const int p = rank / Q, q = rank % Q;
  if (!rc) rc = nccl_err(g_nccl.CommSplit(g->world, p, q, &g->row, nullptr), "CommSplit(row)");
  if (!rc) rc = nccl_err(g_nccl.CommSplit(g->world, q, p, &g->col, nullptr), "CommSplit(col)");
  if (!rc) rc = nccl_err(g_nccl.CommSplit(g->world, q, p, &g->colp, nullptr), "CommSplit(colp)");
  if (rc) {
    hlq_grid_free(g);
    return rc;
  }
  *out = g;
  return 0;
}

int hlq_grid_create_host(const hlq_host_comm* ops, int32_t nranks, int32_t rank, int32_t P,
                         int32_t Q, hlq_grid_t* out) {
  if (!out) return -6;
  *out = nullptr;
  if (!ops || ops->struct_size != (int32_t)sizeof(hlq_host_comm) || !ops->allgather ||
      !ops->broadcast || !ops->allreduce)
    return -1;
  if (nranks < 1) return -2;
  if (rank < 0 || rank >= nranks) return -3;
  if (P < 1 || P > 16) return -4;
  if (Q < 1 || Q > 16 || P * Q != nranks) return -5;
  hlq_grid_s* g = new (std::nothrow) hlq_grid_s();
  if (!g) return HLQ_ERR_NOMEM;
  g->P = P;
  g->Q = Q;
  g->local = 0;
  g->rank = rank;
  g->host = true;
  g->ops = *ops;
  *out = g;
  return 0;
}

int hlq_grid_create_local(int32_t P, int32_t Q, hlq_grid_t* out) {
  if (!out) return -3;
  *out = nullptr;
  if (P < 1 || P > 16) return -1;
  if (Q < 1 || Q > 16) return -2;
  hlq_grid_s* g = new (std::nothrow) hlq_grid_s();
  if (!g) return HLQ_ERR_NOMEM;
  g->P = P;
  g->Q = Q;
  g->local = 1;
  *out = g;
  return 0;
}

void hlq_grid_free(hlq_grid_t g) {
  if (!g) return;
  if (g->stage) cudaFreeHost(g->stage);
  if (g->row) g_nccl.CommDestroy(g->row);
  if (g->col) g_nccl.CommDestroy(g->col);
  if (g->colp) g_nccl.CommDestroy(g->colp);
  if (g->world) g_nccl.CommDestroy(g->world);
  delete g;
}

int hlq_grid_info(hlq_grid_t g, int32_t* P, int32_t* Q, int32_t* nlocal, int32_t* rank0) {
  if (!g) return -1;
  if (P) *P = g->P;
  if (Q) *Q = g->Q;
  if (nlocal) *nlocal = g->local ? g->P * g->Q : 1;
  if (rank0) *rank0 = g->local ? 0 : g->rank;
  return 0;
}

int hlq_grid_local_shape(int64_t N, int32_t nb, int32_t P, int32_t Q, int32_t p, int32_t q,
                         int64_t* mloc, int64_t* nloc) {
  if (N < 0) return -1;
  if (nb <= 0) return -2;
  if (P < 1) return -3;
  if (Q < 1) return -4;
  if (p < 0 || p >= P) return -5;
  if (q < 0 || q >= Q) return -6;
  if (mloc) *mloc = cyc_extent(N, nb, P, p);
  if (nloc) *nloc = cyc_extent(N, nb, Q, q);
  return 0;
}

int hlq_dist_plan(int32_t n, int32_t P, int32_t D, int32_t p, int32_t k, int32_t* out,
                  int32_t cap) {
  if (n < 1) return -1;
  if (P < 1) return -2;
  if (D < P || D % P != 0 || D / P > 16) return -3;
  if (p < 0 || p >= P) return -4;
  if (k < 0 || k >= n) return -5;
  StepPlan sp = plan_step(n, P, D, p, k);
  std::vector<std::vector<int2>> inter = plan_inter(n, P, D, k);
  std::vector<int32_t> v;
  v.push_back(sp.li0);
  v.push_back(sp.ms);
  v.push_back(sp.diag);
  v.push_back((int)sp.head_local.size());
  for (size_t t = 0; t < sp.head_local.size(); ++t) {
    v.push_back(sp.head_local[t]);
    v.push_back(sp.head_global[t]);
  }
  v.push_back((int)sp.intra.size());
  for (auto& lv : sp.intra) {
    v.push_back((int)lv.size());
    for (auto& pr : lv) {
      v.push_back(pr.x);
      v.push_back(pr.y);
    }
  }
  v.push_back((int)inter.size());
  for (auto& lv : inter) {
    v.push_back((int)lv.size());
    for (auto& pr : lv) {
      v.push_back(pr.x);
      v.push_back(pr.y);
    }
  }
  if (out && cap > 0) memcpy(out, v.data(), sizeof(int32_t) * std::min<size_t>(cap, v.size()));
  return (int)v.size();
}

int hlq_generate_uniform_cyclic(hlq_grid_t grid, double* const* A_local, const int64_t* lld,
                                int64_t N, int32_t nb, uint64_t seed, void* stream) {
  if (!grid) return -1;
  if (!A_local) return -2;
  if (N <= 0) return -4;
  if (nb <= 0) return -5;
  if (nb > N) nb = (int32_t)N;
  uint64_t z = seed + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  const uint64_t key = z ^ (z >> 31);
  const int nlocal = grid->local ? grid->P * grid->Q : 1;
  for (int t = 0; t < nlocal; ++t) {
    const int r = grid->local ? t : grid->rank;
    const int p = r / grid->Q, q = r % grid->Q;
    const int64_t mloc = cyc_extent(N, nb, grid->P, p), nloc = cyc_extent(N, nb, grid->Q, q);
    const int64_t ld = (lld && lld[t]) ? lld[t] : std::max<int64_t>(mloc, 1);
    if (mloc <= 0 || nloc <= 0) continue;
    if (!A_local[t]) return -2;
    if (ld < mloc) return -3;
    ::hlq::g_launches++;
    k_generate_cyclic<<<blocks_for(mloc * nloc), 256, 0, (cudaStream_t)stream>>>(
        A_local[t], ld, mloc, nloc, N, nb, grid->P, grid->Q, p, q, key);
  }
  return cuda_check(cudaGetLastError());
}

int hlq_residual_dist(hlq_grid_t grid, double* const* A_local, const int64_t* lld, int64_t N,
                      int32_t nb, const double* x, const double* b, double* out3, void* stream) {
  if (!grid) return -1;
  if (!A_local) return -2;
  if (N <= 0) return -4;
  if (nb <= 0) return -5;
  if (!x) return -6;
  if (!b) return -7;
  if (!out3) return -8;
  if (nb > N) nb = (int32_t)N;
  cudaStream_t st = (cudaStream_t)stream;
  const int P = grid->P, Q = grid->Q;
  const int nlocal = grid->local ? P * Q : 1;
  const int64_t mmax = cyc_extent(N, nb, P, 0);
  double* buf = nullptr;
  int rc;
  if ((rc = cuda_check(cudaMalloc(&buf, sizeof(double) * (nlocal * 2 * (mmax + 1) + 4 * nlocal)))))
    return rc;
  std::vector<int> ps(nlocal), qs(nlocal);
  std::vector<int64_t> ml(nlocal);
  for (int t = 0; t < nlocal; ++t) {
    const int r = grid->local ? t : grid->rank;
    ps[t] = r / Q;
    qs[t] = r % Q;
    ml[t] = cyc_extent(N, nb, P, ps[t]);
    const int64_t nloc = cyc_extent(N, nb, Q, qs[t]);
    const int64_t ld = (lld && lld[t]) ? lld[t] : std::max<int64_t>(ml[t], 1);
    double* part = buf + (int64_t)t * 2 * (mmax + 1);
    cudaMemsetAsync(part, 0, sizeof(double) * 2 * (mmax + 1), st);
    if (ml[t] > 0 && nloc > 0) {
      ::hlq::g_launches++;
      k_residual_part<<<(unsigned)((ml[t] + 127) / 128), 128, 0, st>>>(A_local[t], ld, ml[t], nloc,
                                                                       nb, Q, qs[t], x, part);
    }
  }
  // sum the partials over each process row (ascending q), then every rank takes its row's sum
  if (!grid->local) {
    if (ml[0] > 0 && (rc = xc_allreduce(grid, HLQ_COMM_ROW, buf, 2 * ml[0], 0, st))) {
      cudaFree(buf);
      return rc;
    }
  } else {
    // parts are laid out [mloc | mloc]: add q = 1.. into q = 0, then copy back
    for (int p = 0; p < P; ++p) {
      const int t0 = p * Q;
      double* dst = buf + (int64_t)t0 * 2 * (mmax + 1);
      for (int q = 1; q < Q; ++q) {
        ::hlq::g_launches++;
        k_add_vec<<<blocks_for(2 * ml[t0]), 256, 0, st>>>(
            dst, buf + (int64_t)(t0 + q) * 2 * (mmax + 1), 2 * ml[t0]);
      }
      for (int q = 1; q < Q; ++q)
        cudaMemcpyAsync(buf + (int64_t)(t0 + q) * 2 * (mmax + 1), dst,
                        sizeof(double) * 2 * ml[t0], cudaMemcpyDeviceToDevice, st);
    }
  }
  double* outs = buf + (int64_t)nlocal * 2 * (mmax + 1);
  cudaMemsetAsync(outs, 0, sizeof(double) * 4 * nlocal, st);
  for (int t = 0; t < nlocal; ++t) {
    ::hlq::g_launches++;
    k_residual_max<<<64, 256, 0, st>>>(buf + (int64_t)t * 2 * (mmax + 1), ml[t], nb, P, ps[t], b, x,
                                       N, outs + 4 * t);
  }
  if (!grid->local && (rc = xc_allreduce(grid, HLQ_COMM_WORLD, outs, 3, 1, st))) {
    cudaFree(buf);
    return rc;
  }
  std::vector<double> h(4 * nlocal);
  cudaMemcpyAsync(h.data(), outs, sizeof(double) * 4 * nlocal, cudaMemcpyDeviceToHost, st);
  rc = cuda_check(cudaStreamSynchronize(st));
  cudaFree(buf);
  if (rc) return rc;
  for (int j = 0; j < 3; ++j) {
    double m = 0.0;
    for (int t = 0; t < nlocal; ++t) m = std::max(m, h[4 * t + j]);
    out3[j] = m;
  }
  return 0;
}

int hlq_dist_counts(int64_t N, int32_t nb, int32_t P, int32_t Q, int32_t D, int32_t p, int32_t q,
                    int32_t k, int64_t* out4) {
  if (N <= 0) return -1;
  if (nb <= 0) return -2;
  if (P < 1) return -3;
  if (Q < 1) return -4;
  if (D < P || D % P != 0) return -5;
  if (p < 0 || p >= P) return -6;
  if (q < 0 || q >= Q) return -7;
  if (nb > N) nb = (int32_t)N;
  const int n = (int)((N + nb - 1) / nb);
  if (k < 0 || k >= n) return -8;
  if (!out4) return -9;
  step_counts(N, nb, P, Q, D, 32, p, q, k, out4);
  return 0;
}

int hlq_factor_dist(hlq_grid_t grid, double* const* A_local, const int64_t* lld, int64_t N,
                    int32_t nb, int32_t criterion, double alpha, const hlq_options* opt_in,
                    hlq_factors_t* out) {
  if (!out) return -10;
  *out = nullptr;
  if (!grid) return -1;
  if (!A_local) return -2;
  if (N <= 0) return -4;
  if (nb <= 0 || nb > HLQ_MAX_NB) return -5;
  if (criterion < 0 || criterion > 3) return -6;
  if (!(alpha >= 0.0)) return -7;
  hlq_options opt;
  hlq_default_options(&opt);
  if (opt_in) {
    if (opt_in->struct_size != (int32_t)sizeof(hlq_options)) return -8;
    opt = *opt_in;
  }
  if (nb > N) nb = (int32_t)N;
  const int P = grid->P, Q = grid->Q;
  const int D = opt.tree_domains ? opt.tree_domains : P;
  if (opt.ib == 0) opt.ib = 32;
  if (opt.tie_rel_tol == 0.0) opt.tie_rel_tol = 1e-10;
  if (opt.ib != 32 || D < P || D % P != 0 || D / P > 16 || opt.tree != HLQ_TREE_GREEDY ||
      opt.mumps_reading < 0 || opt.mumps_reading > 1 || opt.lu_variant != HLQ_LU_A1 ||
      opt.pivot_scope < HLQ_PIVOT_TILE || opt.pivot_scope > HLQ_PIVOT_DOMAIN)
    return -8;
  hlq_factors_t f = new (std::nothrow) hlq_factors_s();
  if (!f) return HLQ_ERR_NOMEM;
  DistState* ds = new (std::nothrow) DistState();
  if (!ds) {
    delete f;
    return HLQ_ERR_NOMEM;
  }
  f->dist = ds;
  *out = f;
  const int n = (int)((N + nb - 1) / nb);
  f->g.N = N;
  f->g.Nc = N;
  f->g.lda = N;
  f->g.nb = nb;
  f->g.n = n;
  f->ib = opt.ib;
  f->D = D;
  f->crit = criterion;
  f->alpha = alpha;
  f->st = (cudaStream_t)opt.stream;
  f->blocking = opt.blocking != 0;
  f->track_growth = opt.track_growth != 0;
  ds->gr = grid;
  ds->P = P;
  ds->Q = Q;
  ds->D = D;
  ds->c = D / P;
  ds->S = D;
  ds->dpiv = opt.pivot_scope == HLQ_PIVOT_DOMAIN;
  f->pivot_scope = opt.pivot_scope;
  ds->ib = opt.ib;
  ds->nb = nb;
  ds->n = n;
  ds->N = N;
  ds->st = f->st;
  {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&ds->sp, cudaStreamNonBlocking, hi);
    cudaEventCreateWithFlags(&ds->ev_part0, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ds->ev_panel, cudaEventDisableTiming);
  }
  ds->ms_max = cyc_count(n, P, 0);
  ds->mt_max = ds->ms_max;
  ds->rec_count = ds->ms_max + 3 * (int64_t)nb + 2 + (int64_t)nb * nb;
  ds->seg_cap = (int64_t)ds->mt_max * nb;
  ds->inter.resize(n);
  for (int k = 0; k < n; ++k) ds->inter[k] = plan_inter(n, P, D, k);
  const int nlocal = grid->local ? P * Q : 1;
  ds->ctx.resize(nlocal);
  const bool has_ref = opt.ref_dec && opt.ref_margin;
  for (int t = 0; t < nlocal; ++t) {
    Ctx& c = ds->ctx[t];
    const int r = grid->local ? t : grid->rank;
    c.p = r / Q;
    c.q = r % Q;
    c.A = A_local[t];
    c.mloc = cyc_extent(N, nb, P, c.p);
    c.nloc = cyc_extent(N, nb, Q, c.q);
    c.mt = cyc_count(n, P, c.p);
    c.nt = cyc_count(n, Q, c.q);
    c.lld = (lld && lld[t]) ? lld[t] : std::max<int64_t>(c.mloc, 1);
    if (c.lld < c.mloc) return -3;
    if (!c.A && c.mloc > 0 && c.nloc > 0) return -2;
    c.plan.resize(n);
    for (int k = 0; k < n; ++k) c.plan[k] = plan_step(n, P, D, c.p, k);
    int rc = dist_alloc(*ds, c, opt, has_ref);
    if (rc) return rc;
  }
  f->prof.on = opt.profile != 0;
  int rc = dist_factor(*ds, criterion, alpha, opt, f->prof);
  if (rc) return rc;
  Ctx& c0 = ds->ctx[0];
  f->dec.resize(n);
  f->margin.resize(n);
  f->flags.resize(n);
  f->gstep.assign(n + 1, 0.0);
  std::vector<double> fin(n + 5);
  cudaMemcpyAsync(f->dec.data(), c0.w.dec, n, cudaMemcpyDeviceToHost, ds->st);
  cudaMemcpyAsync(f->margin.data(), c0.w.margin, sizeof(double) * n, cudaMemcpyDeviceToHost, ds->st);
  cudaMemcpyAsync(f->flags.data(), c0.w.flags, sizeof(int) * n, cudaMemcpyDeviceToHost, ds->st);
  std::vector<std::vector<double>> fins(ds->ctx.size(), std::vector<double>(n + 5));
  for (size_t t = 0; t < ds->ctx.size(); ++t)
    cudaMemcpyAsync(fins[t].data(), ds->ctx[t].fin, sizeof(double) * (n + 5),
                    cudaMemcpyDeviceToHost, ds->st);
  if ((rc = cuda_check(cudaStreamSynchronize(ds->st)))) return rc;
  for (int j = 0; j < n + 5; ++j) {
    double m = fins[0][j];
    for (size_t t = 1; t < fins.size(); ++t) m = std::max(m, fins[t][j]);
    fin[j] = m;
  }
  for (int k = 0; k <= n; ++k) f->gstep[k] = fin[k];
  const double* stat = fin.data() + n + 1;
  if (stat[0] != 0.0 || stat[2] != 0.0)
    f->status = HLQ_ST_NONFINITE;
  else if (stat[1] != 0.0)
    f->status = HLQ_ST_ZERO_PIVOT_FORCED;
  else if (stat[3] != 0.0)
    f->status = HLQ_ST_SINGULAR;
  else
    f->status = HLQ_OK;
  if (f->track_growth) {
    double gmax = f->gstep[0];
    bool nonfinite = false;
    for (int k = 0; k <= n; ++k) {
      double v = f->gstep[k];
      if (v != v || isinf(v)) nonfinite = true;
      if (v > gmax) gmax = v;
    }
    f->growth = nonfinite ? INFINITY : (f->gstep[0] > 0 ? gmax / f->gstep[0] : NAN);
  } else {
    f->growth = NAN;
  }
  return f->status;
}

}  // extern "C"
