// C ABI of libhlq (include/hlq.h): the handle, the step scheduler of Alg. 1 and
// the solve.  The host only enqueues work: per step k it launches the criterion kernels, the decide
// kernel (which writes d_k to device memory) and BOTH branches' kernels, each predicated on d_k
// (a kernel of the branch not taken exits at its first instruction).  Decisions known on the host
// (a forced vector, alpha = 0) skip the other branch's launches.  No host round trip inside the
// factorization: this replaces the paper's Propagate / selection tasks.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <new>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "handle.cuh"

namespace hlq {
void launch_tri_inv(Geo g, int k, const DevWork& w, double* Li, double* Ui, cudaStream_t st);
void launch_final_scan(const double* A, int64_t N, int64_t lda, int* flag, cudaStream_t st);
}  // namespace hlq

namespace hlq {
int64_t g_launches = 0;
int dist_solve_entry(hlq_factors_t f, const double* b, double* x);
void dist_free(DistState* d);
}
using namespace hlq;

// ---------------------------------------------------------------------------------------------
// device-memory cache: big workspaces are reused across calls (like a cuBLAS workspace), so a
// repeated factorization of the same size does not pay cudaMalloc/cudaFree.  One entry per
// (device, slot); a taken block belongs to exactly one handle until it is put back.  Guarded by a
// mutex, so handles on different host threads (and devices) never share a block.
namespace {
struct CacheSlot {
  void* p = nullptr;
  size_t bytes = 0;
};
constexpr int kMaxDev = 64;
std::mutex g_cache_mu;
CacheSlot g_cache[kMaxDev][2];

int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < 0 ? 0 : (d >= kMaxDev ? kMaxDev - 1 : d);
}

void* cache_get(int slot, size_t bytes) {
  const int dev = cur_device();
  void* stale = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    CacheSlot& c = g_cache[dev][slot];
    if (c.p && c.bytes >= bytes) {
      void* p = c.p;
      c.p = nullptr;
      c.bytes = 0;
      return p;
    }
    stale = c.p;
    c.p = nullptr;
    c.bytes = 0;
  }
  if (stale) cudaFree(stale);
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}
// p was taken on device dev
void cache_put(int dev, int slot, void* p, size_t bytes) {
  if (!p) return;
  void* drop = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    CacheSlot& c = g_cache[dev][slot];
    if (c.p && c.bytes >= bytes) {
      drop = p;
    } else {
      drop = c.p;
      c.p = p;
      c.bytes = bytes;
    }
  }
  if (drop) {
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
    cudaFree(drop);
    if (prev != dev) cudaSetDevice(prev);
  }
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// tiles per work unit of the persistent solve (HLQ_SOLVE_G overrides, 1..64: measurement knob)
static int solve_g() {
  static int gval = -1;
  if (gval < 0) {
    const char* e = getenv("HLQ_SOLVE_G");
    const int v = e ? atoi(e) : 4;
    gval = v < 1 ? 1 : v > 64 ? 64 : v;
  }
  return gval;
}
constexpr size_t kFlagBytes = 128;  // one solve flag per cache line (solve.cu kFlagStride)
size_t solve_ws_bytes(int n, int nb, int cmax, size_t units) {
  return align_up(sizeof(int2) * units, 256) + align_up(kFlagBytes * n, 256) +
         align_up(kFlagBytes * (size_t)n * cmax, 256) + sizeof(double) * (size_t)n * cmax * nb +
         256;
}

}  // namespace

// the library's high-priority panel streams (lookahead), created once per device: sp runs the
// criterion (speculative LU) and the chosen branch, sq the speculative QR panel beside it.
// Concurrent factorizations on one device share them (their panel stages then serialise; every
// cross-stream dependency is an event of the handle itself, so correctness does not depend on it).
static cudaStream_t panel_stream(int which = 0) {
  static cudaStream_t s[kMaxDev][2] = {};
  const int dev = cur_device();
  std::lock_guard<std::mutex> lk(g_cache_mu);
  if (!s[dev][which]) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&s[dev][which], cudaStreamNonBlocking, hi);
  }
  return s[dev][which];
}


// NVTX ranges (factor, solve, every step) when HLQ_NVTX=1; no-ops without a tool attached
static bool nvtx_on() {
  static int on = -1;
  if (on < 0) on = getenv("HLQ_NVTX") ? atoi(getenv("HLQ_NVTX")) != 0 : 0;
  return on != 0;
}
struct NvtxScope {
  bool on;
  explicit NvtxScope(const char* name) : on(nvtx_on()) {
    if (on) nvtxRangePushA(name);
  }
  ~NvtxScope() {
    if (on) nvtxRangePop();
  }
};

static int cuda_err(cudaError_t e) {
  if (e == cudaSuccess) return 0;
  fprintf(stderr, "[hlq] CUDA error: %s\n", cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? HLQ_ERR_NOMEM : HLQ_ERR_CUDA;
}

// QR elimination plan of step k (readings 16 and 34): the rows of each domain (i mod D);
// tsa == 0: the greedy halving tree over all rows of a domain, then over the domain heads;
// tsa >= 1 (HQR): each domain's rows cut into consecutive groups of tsa tiles, flat TS inside a
// group onto its head, the halving tree over a domain's group heads, then over the domain heads.
struct StepPlanHost {
  std::vector<std::vector<int2>> levels;  // TT levels
  std::vector<int> heads;                 // GEQRT rows (HQR only; greedy: all rows k..n-1)
  std::vector<int2> ts_pairs;             // TS eliminations, group by group
  std::vector<int> ts_off;                // group offsets into ts_pairs (ngroups + 1)
};

static void plan_step(int k, int n, int D, int tsa, StepPlanHost& p) {
  p.levels.clear();
  p.heads.clear();
  p.ts_pairs.clear();
  p.ts_off.clear();
  std::vector<std::vector<int>> doms;
  for (int d = 0; d < D; ++d) {
    std::vector<int> rows;
    for (int i = k; i < n; ++i)
      if (i % D == d) rows.push_back(i);
    if (!rows.empty()) doms.push_back(rows);
  }
  std::sort(doms.begin(), doms.end(),
            [](const std::vector<int>& a, const std::vector<int>& b) { return a[0] < b[0]; });
  std::vector<int> dom_heads;
  for (auto& dm : doms) dom_heads.push_back(dm[0]);
  if (tsa >= 1) {
    p.ts_off.push_back(0);
    for (auto& dm : doms) {
      std::vector<int> gh;
      for (size_t s = 0; s < dm.size(); s += (size_t)tsa) {
        const size_t e = std::min(dm.size(), s + (size_t)tsa);
        gh.push_back(dm[s]);
        if (e - s > 1) {
          for (size_t t = s + 1; t < e; ++t) p.ts_pairs.push_back(make_int2(dm[s], dm[t]));
          p.ts_off.push_back((int)p.ts_pairs.size());
        }
      }
      dm = gh;  // the TT levels run over the group heads
    }
    for (auto& dm : doms) p.heads.insert(p.heads.end(), dm.begin(), dm.end());
    std::sort(p.heads.begin(), p.heads.end());
  }
  auto halving = [](std::vector<int> live, std::vector<std::vector<int2>>& out) {
    while (live.size() > 1) {
      size_t r = live.size(), h = (r + 1) / 2;
      std::vector<int2> lv;
      for (size_t t = 0; t < r - h; ++t) lv.push_back(make_int2(live[t], live[h + t]));
      out.push_back(lv);
      live.resize(h);
    }
  };
  std::vector<std::vector<std::vector<int2>>> per(doms.size());
  size_t depth = 0;
  for (size_t d = 0; d < doms.size(); ++d) {
    halving(doms[d], per[d]);
    depth = per[d].size() > depth ? per[d].size() : depth;
  }
  for (size_t l = 0; l < depth; ++l) {
    std::vector<int2> lv;
    for (size_t d = 0; d < per.size(); ++d)
      if (l < per[d].size()) lv.insert(lv.end(), per[d][l].begin(), per[d][l].end());
    p.levels.push_back(lv);
  }
  halving(dom_heads, p.levels);
}

// The QR panel of step k as a DAG (qr_dmma.cu k_qr_panel_dag): GEQRT of the factored rows (op 0
// is tile k), the TS chain pairs in chain order, the TT levels in order; each op records the
// previous op on its eliminator / head row and on its eliminated row (-1: none).
static void build_dag(int k, int n, int tsa, const StepPlanHost& p, std::vector<int>& ops) {
  std::vector<int> last(n, -1);
  auto add = [&](int kind, int e, int i, int pe, int pi) {
    const int id = (int)(ops.size() / 5);
    ops.insert(ops.end(), {kind, e, i, pe, pi});
    return id;
  };
  std::vector<int> geq;
  if (tsa >= 1 && p.ts_off.size() > 1)
    geq = p.heads;
  else
    for (int i = k; i < n; ++i) geq.push_back(i);
  for (int i : geq) last[i] = add(0, i, i, -1, -1);
  for (const int2& pr : p.ts_pairs) last[pr.x] = add(1, pr.x, pr.y, last[pr.x], -1);
  for (const auto& lv : p.levels)
    for (const int2& pr : lv) {
      const int id = add(2, pr.x, pr.y, last[pr.x], last[pr.y]);
      last[pr.x] = id;
    }
}

extern "C" {

int hlq_abi(int32_t* so, int32_t* si, int32_t* ver) {
  if (so) *so = (int32_t)sizeof(hlq_options);
  if (si) *si = (int32_t)sizeof(hlq_info);
  if (ver) *ver = 1;
  return 0;
}

int hlq_default_options(hlq_options* opt) {
  if (!opt) return -1;
  memset(opt, 0, sizeof(*opt));
  opt->struct_size = (int32_t)sizeof(hlq_options);
  opt->ib = 32;
  opt->tree_domains = 1;
  opt->tree = HLQ_TREE_GREEDY;
  opt->tie_rel_tol = 1e-10;
  opt->track_growth = 1;
  opt->blocking = 1;
  return 0;
}

const char* hlq_status_string(int code) {
  switch (code) {
    case HLQ_OK: return "ok";
    case HLQ_ST_NONFINITE: return "non-finite values encountered";
    case HLQ_ST_SINGULAR: return "exact zero on the final U/R diagonal";
    case HLQ_ST_ZERO_PIVOT_FORCED: return "forced LU step met an exact zero pivot";
    case HLQ_ERR_CUDA: return "CUDA error";
    case HLQ_ERR_NCCL: return "NCCL error";
    case HLQ_ERR_NOMEM: return "out of device memory";
    case HLQ_ERR_STATE: return "invalid handle state";
    default: return code < 0 ? "invalid argument" : "unknown";
  }
}

int hlq_factor_ex(double* A, int64_t N, int32_t nb, int32_t criterion, double alpha,
                  const hlq_options* opt_in, hlq_factors_t* out) {
  NvtxScope nvtx_scope("hlq_factor");
  if (!out) return -7;
  *out = nullptr;
  if (!A) return -1;
  if (N <= 0) return -2;
  if (nb <= 0 || nb > HLQ_MAX_NB) return -3;
  if (criterion < 0 || criterion > 3) return -4;
  if (!(alpha >= 0.0)) return -5;  // rejects NaN and negatives
  hlq_options opt;
  hlq_default_options(&opt);
  if (opt_in) {
    if (opt_in->struct_size != (int32_t)sizeof(hlq_options)) return -6;
    opt = *opt_in;
  }
  if (opt.ib == 0) opt.ib = 32;
  if (opt.tree_domains == 0) opt.tree_domains = 1;
  if (opt.tie_rel_tol == 0.0) opt.tie_rel_tol = 1e-10;
  if (opt.tree == HLQ_TREE_HQR && opt.ts_group == 0) opt.ts_group = 4;
  if (opt.ib != 32 || opt.tree_domains < 1 ||
      (opt.tree != HLQ_TREE_GREEDY && opt.tree != HLQ_TREE_HQR) ||
      (opt.tree == HLQ_TREE_HQR && opt.ts_group < 1) ||
      opt.mumps_reading < 0 || opt.mumps_reading > 1 || opt.invnorm_estimate < 0 ||
      opt.invnorm_estimate > 1 || opt.lu_variant < HLQ_LU_A1 || opt.lu_variant > HLQ_LU_A2 ||
      (opt.lu_variant == HLQ_LU_A2 && opt.invnorm_estimate != 0) ||
      opt.pivot_scope < HLQ_PIVOT_TILE || opt.pivot_scope > HLQ_PIVOT_DOMAIN ||
      (opt.pivot_scope == HLQ_PIVOT_DOMAIN && opt.lu_variant != HLQ_LU_A1))
    return -6;
  int64_t lda = opt.lda ? opt.lda : N;
  if (lda < N) return -6;
  if (nb > N) nb = (int32_t)N;

  hlq_factors_t f = new (std::nothrow) hlq_factors_s();
  if (!f) return HLQ_ERR_NOMEM;
  *out = f;
  for (int e = 0; e < 6; ++e) cudaEventCreateWithFlags(&f->ev[e], cudaEventDisableTiming);
  f->A = A;
  f->g.N = N;
  f->g.lda = lda;
  f->g.nb = nb;
  f->g.n = (int)((N + nb - 1) / nb);
  f->g.Nc = N;
  f->ib = opt.ib;
  f->D = opt.tree_domains;
  f->crit = criterion;
  f->lu_variant = opt.lu_variant;
  f->pivot_scope = opt.pivot_scope;
  f->alpha = alpha;
  f->st = (cudaStream_t)opt.stream;
  f->blocking = opt.blocking != 0;
  f->track_growth = opt.track_growth != 0;
  const int n = f->g.n, ib = f->ib;
  Geo g = f->g;

  // plans
  const int tsa = opt.tree == HLQ_TREE_HQR ? opt.ts_group : 0;
  std::vector<StepPlanHost> plans(n);
  size_t npairs = 0, nts = 0, nheads = 0, noff = 0;
  size_t qs_ops = 0;  // ops of the solve's Q^T replay DAG if every step is QR (hlq_solve)
  for (int k = 0; k < n; ++k) {
    plan_step(k, n, f->D, tsa, plans[k]);
    qs_ops += (tsa >= 1 && plans[k].ts_off.size() > 1)
                  ? plans[k].heads.size() + plans[k].ts_pairs.size()
                  : (size_t)(n - k);
    for (auto& lv : plans[k].levels) qs_ops += lv.size();
    for (auto& lv : plans[k].levels) npairs += lv.size();
    nts += plans[k].ts_pairs.size();
    nheads += plans[k].heads.size();
    noff += plans[k].ts_off.size();
  }
  f->tree = opt.tree;
  f->ts_group = tsa;
  // the QR panel as one DAG launch per step (HLQ_QR_DAG=0: the level-by-level launches)
  static int dag_env = -1;
  if (dag_env < 0) dag_env = getenv("HLQ_QR_DAG") ? atoi(getenv("HLQ_QR_DAG")) : 1;
  std::vector<std::vector<int>> dag_ops(n);
  size_t dag_total = 0, dag_max = 0;
  if (dag_env != 0 && ib == 32) {
    for (int k = 0; k < n; ++k) {
      build_dag(k, n, tsa, plans[k], dag_ops[k]);
      dag_total += dag_ops[k].size();
      dag_max = std::max(dag_max, dag_ops[k].size() / 5);
    }
  }

  // workspace layout (bytes, 256-aligned pieces)
  const size_t ntri = (size_t)n * (n + 1) / 2;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align_up(bytes ? bytes : 1, 256);
    return o;
  };
  const int cpr = gemm_colpart_rows();  // row granularity of the DGEMM's fused column partials
  const bool fuse_growth_any = f->track_growth && nb % cpr == 0;
  const size_t scr = (size_t)2 * nb * nb + align_up(nb, 64);
  size_t oW0 = take(sizeof(double) * nb * nb), oW1 = take(sizeof(double) * nb * nb),
         oIpw0 = take(sizeof(int) * nb), oIpw1 = take(sizeof(int) * nb),
         oIp = take(sizeof(int) * (size_t)n * nb), oTg = take(sizeof(double) * ntri * ib * nb),
         oTt = take(sizeof(double) * ntri * ib * nb), oS = take(sizeof(double) * n),
         oLm = take(sizeof(double) * nb), oAm = take(sizeof(double) * nb), oInv = take(8),
         oZp = take(sizeof(int)), oDec = take(n), oMg = take(sizeof(double) * n),
         oSl = take(sizeof(double) * 2 * n),
         oFl = take(sizeof(int) * n), oSt = take(sizeof(int) * 4), oFo = take(n), oRd = take(n),
         oRm = take(sizeof(double) * n), oGs = take(sizeof(double) * (n + 1)),
         oPr = take(sizeof(int2) * (npairs + nts + 1)), oHd = take(sizeof(int) * (nheads + noff + 1)), oSc0 = take(sizeof(double) * scr),
         oSc1 = take(sizeof(double) * scr), oWp = take(sizeof(double) * (size_t)N * nb),
         oWr = take(sizeof(double) * (size_t)N * nb),
         oCp = take(fuse_growth_any ? sizeof(double) * (size_t)((N + cpr - 1) / cpr) * N : 8),
         oLi = take(opt.lu_variant == HLQ_LU_A2 ? sizeof(double) * (size_t)n * 2 * nb * nb : 8),
         oLp = take(sizeof(int) * (size_t)n * nb), oSt2 = take(sizeof(double) * (size_t)nb);
  const bool dpiv = opt.pivot_scope == HLQ_PIVOT_DOMAIN;
  // speculative QR panel: with a criterion to evaluate, the QR branch's panel (GEQRT of every tile +
  // every TTQRT level) runs on a copy of the panel beside the speculative LU and the criterion, and
  // is copied back if the step is QR (A1, ib = 32; HLQ_SPEC_QR=0 disables it)
  static int spec_env = -1;
  if (spec_env < 0) spec_env = getenv("HLQ_SPEC_QR") ? atoi(getenv("HLQ_SPEC_QR")) : 1;
  const bool spec_qr = spec_env != 0 && !opt.forced && alpha > 0.0 && !isinf(alpha);
  size_t oWd = take(dpiv ? sizeof(double) * (size_t)N * nb : 8),
         oDp = take(dpiv ? sizeof(int) * (size_t)n * nb : 8),
         oDk = take(sizeof(unsigned long long) * 2 * 148), oDi = take(sizeof(int) * 2 * 148),
         oDc = take(sizeof(unsigned int)),
         oQp = take(spec_qr ? sizeof(double) * (size_t)N * nb : 8);
  // persistent-solve workspace (hlq_solve): unit tables (capacity 2 n cmax), flags, partials
  const int scmax = solve_rows_cmax(n, solve_g());
  const size_t solve_cap = (size_t)2 * n * scmax + 1;
  size_t oSv = take(solve_ws_bytes(n, nb, scmax, solve_cap));
  size_t oDag = take(sizeof(int) * (dag_total + 1)), oDagP = take(sizeof(int) * (dag_max + 1));
  // the solve's DAG: 6 ints per op + one 128-byte completion flag per op (no allocation, and so
  // no device synchronisation, inside the first hlq_solve)
  const size_t qs_tab = align_up(sizeof(int) * 6 * (qs_ops + 1), 256);
  size_t oQs = take(qs_tab + sizeof(int) * 32 * (qs_ops + 1));
  f->ws_bytes = off;
  f->dev = cur_device();
  f->ws_block = cache_get(0, off);
  if (!f->ws_block) return HLQ_ERR_NOMEM;
  char* base = (char*)f->ws_block;
  DevWork& w = f->w;
  w.W = (double*)(base + oW0);
  w.ipiv_ws = (int*)(base + oIpw0);
  w.ipiv = (int*)(base + oIp);
  w.Tg = (double*)(base + oTg);
  w.Ttt = (double*)(base + oTt);
  w.s = (double*)(base + oS);
  w.local_max = (double*)(base + oLm);
  w.away_max = (double*)(base + oAm);
  w.inv_norm = (double*)(base + oInv);
  w.zp = (int*)(base + oZp);
  w.dec = (uint8_t*)(base + oDec);
  w.margin = (double*)(base + oMg);
  w.steplog = (double*)(base + oSl);
  w.flags = (int*)(base + oFl);
  w.status = (int*)(base + oSt);
  w.forced = opt.forced ? (uint8_t*)(base + oFo) : nullptr;
  w.ref_dec = (opt.ref_dec && opt.ref_margin) ? (uint8_t*)(base + oRd) : nullptr;
  w.ref_margin = (opt.ref_dec && opt.ref_margin) ? (double*)(base + oRm) : nullptr;
  w.gstep = (double*)(base + oGs);
  w.pairs = (int2*)(base + oPr);
  w.scratch = (double*)(base + oSc0);
  w.ws_panel = (double*)(base + oWp);
  w.ws_row = (double*)(base + oWr);
  w.colpart = fuse_growth_any ? (double*)(base + oCp) : nullptr;
  w.luinv = (double*)(base + oLi);
  w.luperm = (int*)(base + oLp);
  w.solve_t = (double*)(base + oSt2);
  w.wdom = dpiv ? (double*)(base + oWd) : nullptr;
  w.qpan = spec_qr ? (double*)(base + oQp) : nullptr;
  w.dipiv = dpiv ? (int*)(base + oDp) : nullptr;
  w.dom_key = (unsigned long long*)(base + oDk);
  w.dom_idx = (int*)(base + oDi);
  w.dom_counter = (unsigned int*)(base + oDc);
  f->solve_ws_in = base + oSv;
  f->qsolve_ws_in = base + oQs;
  f->qsolve_cap = qs_ops;
  f->tma_maps = make_tma_maps(A, N, lda, nb);
  w.tma_maps = f->tma_maps;
  f->solve_cap = solve_cap;
  // per-parity views (lookahead: step k+1's panel runs while step k's update still reads step k's
  // W / ipiv / L^-1 / U^-1 / perm)
  DevWork wpar[2] = {w, w};
  wpar[1].W = (double*)(base + oW1);
  wpar[1].ipiv_ws = (int*)(base + oIpw1);
  wpar[1].scratch = (double*)(base + oSc1);
  cudaStream_t st = f->st;
  int rc = 0;

  // uploads (pairs flattened per step / level; HQR: heads, TS pairs and group offsets)
  std::vector<int2> flat;
  std::vector<int> iflat;
  flat.reserve(npairs + nts);
  iflat.reserve(nheads + noff);
  f->lvl_ptr.assign(n, {});
  f->lvl_cnt.assign(n, {});
  f->tsplan.assign(n, QRTsPlan{nullptr, 0, nullptr, nullptr, 0});
  int* hbase = (int*)(base + oHd);
  f->dag.assign(n, QRDag{nullptr, 0});
  f->dag_progress = (int*)(base + oDagP);
  f->dag_epoch = 0;
  if (dag_total > 0) {
    std::vector<int> dflat;
    dflat.reserve(dag_total);
    int* dbase = (int*)(base + oDag);
    for (int k = 0; k < n; ++k) {
      f->dag[k] = QRDag{dbase + dflat.size(), (int)(dag_ops[k].size() / 5)};
      dflat.insert(dflat.end(), dag_ops[k].begin(), dag_ops[k].end());
    }
    if ((rc = cuda_err(cudaMemcpyAsync(dbase, dflat.data(), sizeof(int) * dflat.size(),
                                       cudaMemcpyHostToDevice, st))))
      return rc;
    cudaMemsetAsync(f->dag_progress, 0, sizeof(int) * (dag_max + 1), st);
  }
  for (int k = 0; k < n; ++k) {
    for (auto& lv : plans[k].levels) {
      f->lvl_ptr[k].push_back(w.pairs + flat.size());
      f->lvl_cnt[k].push_back((int)lv.size());
      flat.insert(flat.end(), lv.begin(), lv.end());
    }
    const StepPlanHost& p = plans[k];
    if (tsa >= 1 && !p.ts_off.empty() && p.ts_off.size() > 1) {
      QRTsPlan& t = f->tsplan[k];
      t.pairs = w.pairs + flat.size();
      flat.insert(flat.end(), p.ts_pairs.begin(), p.ts_pairs.end());
      t.heads = hbase + iflat.size();
      t.nheads = (int)p.heads.size();
      iflat.insert(iflat.end(), p.heads.begin(), p.heads.end());
      t.off = hbase + iflat.size();
      t.ngroups = (int)p.ts_off.size() - 1;
      iflat.insert(iflat.end(), p.ts_off.begin(), p.ts_off.end());
    } else if (tsa >= 1) {
      // no TS pair in this step (every group a single tile): the greedy launches over the heads,
      // which are then all the rows k..n-1 (tsa = 1) -- or a one-row panel
      f->tsplan[k] = QRTsPlan{nullptr, 0, nullptr, nullptr, 0};
    }
  }
  if (!flat.empty() &&
      (rc = cuda_err(cudaMemcpyAsync(w.pairs, flat.data(), sizeof(int2) * flat.size(),
                                     cudaMemcpyHostToDevice, st))))
    return rc;
  if (!iflat.empty() &&
      (rc = cuda_err(cudaMemcpyAsync(hbase, iflat.data(), sizeof(int) * iflat.size(),
                                     cudaMemcpyHostToDevice, st))))
    return rc;
  if (w.forced &&
      (rc = cuda_err(cudaMemcpyAsync(w.forced, opt.forced, n, cudaMemcpyHostToDevice, st))))
    return rc;
  if (w.ref_dec) {
    if ((rc = cuda_err(cudaMemcpyAsync(w.ref_dec, opt.ref_dec, n, cudaMemcpyHostToDevice, st))))
      return rc;
    if ((rc = cuda_err(cudaMemcpyAsync(w.ref_margin, opt.ref_margin, sizeof(double) * n,
                                       cudaMemcpyHostToDevice, st))))
      return rc;
  }
  cudaMemsetAsync(w.status, 0, sizeof(int) * 4, st);
  cudaMemsetAsync(w.dom_counter, 0, sizeof(unsigned int), st);
  cudaMemsetAsync(w.gstep, 0, sizeof(double) * (n + 1), st);
  cudaMemsetAsync(w.ipiv, 0, sizeof(int) * (size_t)n * nb, st);
  // T factors of tiles without that factorization in a step (HQR: no GEQRT of a non-head row; no
  // TT/TS T for tile k itself; LU steps) read back as zeros, not as a previous call's workspace
  cudaMemsetAsync(w.Tg, 0, sizeof(double) * ntri * ib * nb, st);
  cudaMemsetAsync(w.Ttt, 0, sizeof(double) * ntri * ib * nb, st);
  // Two streams: st (the caller's) runs the trailing updates, sp (high priority) runs the panel
  // stage of step k+1 as soon as step k has updated column block k+1 (lookahead depth 1).
  cudaStream_t sp = panel_stream(0), sq = panel_stream(1);
  cudaEvent_t ev_ready = f->ev[0], ev_panel = f->ev[1], ev_qsrc = f->ev[2], ev_qdone = f->ev[3],
              ev_a2 = f->ev[4], ev_rest = f->ev[5];
  // Lookahead column on the panel stream (HLQ_LA_SP=0: on the update stream, before the rest): the
  // update of column block k+1 by step k is a narrow launch chain (a few hundred CTAs) that the
  // panel of step k+1 waits for; on sp it overlaps the rest of step k's update, which starts at once
  // on st, instead of running alone in front of it.  Step k+1's lookahead column waits for step
  // k's rest (ev_rest), exactly the order the single stream gave.
  static int la_env = -1;
  if (la_env < 0) la_env = getenv("HLQ_LA_SP") ? atoi(getenv("HLQ_LA_SP")) : 1;
  const bool la_sp = la_env != 0;
  f->la_sp = la_sp;
  if (f->track_growth) launch_tile_norm_max(A, g, 0, w.gstep, st);
  cudaEventRecord(ev_ready, st);

  const bool alpha_inf = isinf(alpha);
  Prof& P = f->prof;
  P.on = opt.profile != 0;
  if (P.on) {  // per-step times (hlq_get_step_times): events on the update stream
    f->step_ev.assign((size_t)n + 1, nullptr);
    for (auto& e : f->step_ev) cudaEventCreate(&e);
    cudaEventRecord(f->step_ev[0], st);
  }
  auto known_of = [&](int k) {
    if (opt.forced) return opt.forced[k] ? (int)HLQ_DEC_QR : (int)HLQ_DEC_LU;
    if (alpha == 0.0) return (int)HLQ_DEC_QR;
    return -1;
  };
  const bool criterion_needed = !opt.forced && alpha > 0.0 && !alpha_inf;
  // the statistics (a1) feed Max / Sum / MUMPS; the Random criterion (reading 35) draws instead
  const bool stats_needed = criterion_needed && criterion != HLQ_CRIT_RANDOM;
  const bool need_inv = stats_needed && criterion != HLQ_CRIT_MUMPS;  // ||A_kk^-1||_1 (Max, Sum)
  const bool a2 = opt.lu_variant == HLQ_LU_A2;
  const int Dp = f->D;  // diagonal-domain pivoting: the QR tree's domains
  for (int k = 0; k < n; ++k) {
    const DevWork& wk = wpar[k & 1];
    if (nvtx_on()) {
      char nm[32];
      snprintf(nm, sizeof nm, "hlq step %d", k);
      nvtxRangePushA(nm);
    }
    const int known = known_of(k);
    const int nl = (int)f->lvl_cnt[k].size();
    // ---- panel stage P(k) on sp: criterion, speculative GETRF, decision, the chosen branch's
    //      panel work (LU: commit + TRSM; QR: GEQRT + all TTQRT levels)
    cudaStreamWaitEvent(sp, ev_ready, 0);
    const bool spec = spec_qr && known == -1 && k + 1 < n;
    // the QR branch's panel on a copy of column block k (rows >= k0, global row indices, ld N),
    // started once the panel is in its pre-branch state (A2: after the diagonal GEQRT)
    auto start_spec = [&](cudaEvent_t after) {
      const int64_t k0 = g.r0(k);
      const int bk = g.cbs(k);
      cudaStreamWaitEvent(sq, after, 0);
      launch_copy_block(w.qpan + k0, N, A + k0 * lda + k0, lda, N - k0, bk, nullptr, nullptr, 0,
                        sq);
      cudaEventRecord(ev_qsrc, sq);  // (the LU branch may overwrite A's panel only after this)
      Geo gq = g;
      gq.lda = N;
      P.begin(HLQ_PROF_QR_GEQRT, sq);
      // predicated on d_k with "undecided" = run: once the criterion decides LU, the remaining
      // speculative launches exit at their first instruction
      launch_qr_panel(w.qpan - k0 * N, gq, k, ib, f->lvl_ptr[k].data(), f->lvl_cnt[k].data(), nl,
                      wk, sq, /*diag_done=*/a2, /*spec=*/true, &f->tsplan[k], &f->dag[k],
                      f->dag_progress, ++f->dag_epoch);
      P.end(sq);
      cudaEventRecord(ev_qdone, sq);
    };
    if (spec) {
      cudaMemsetAsync(w.dec + k, 0xff, 1, sp);  // d_k undecided until k_decide
      if (!a2) {
        cudaEventRecord(ev_a2, sp);
        start_spec(ev_a2);
      }
    }
    if (known != HLQ_DEC_QR) {
      if (stats_needed) {
        P.begin(HLQ_PROF_CRITERION, sp);
        if (dpiv)
          launch_panel_stats_domain(A, g, k, Dp, wk, sp);
        else
          launch_panel_stats(A, g, k, wk, sp);
        P.end(sp);
      }
      P.begin(HLQ_PROF_GETRF, sp);
      if (a2) {
        // A2 Factor: GEQRT of the diagonal tile in place (a one-tile view of A), then
        // W <- the tile, Li <- Q_kk^T (UNMQR applied to I), Ui <- U_kk^-1 (L^-1 is not needed)
        const int bk = g.bs(k);
        Geo gk = g;
        gk.N = bk;
        gk.Nc = bk;
        gk.n = 1;
        double* Akk = g.tile(A, k, k);
        const double* Tkk = w.Tg + tri_index(k, k, n) * (int64_t)ib * nb;
        launch_qr_panel_tc(Akk, gk, 0, ib, const_cast<double*>(Tkk), nullptr, nullptr, 0, nullptr,
                           false, sp);
        if (spec) {
          cudaEventRecord(ev_a2, sp);
          start_spec(ev_a2);
        }
        launch_a2_prep(A, g, k, wk, sp);
        launch_tri_inv(g, k, wk, wk.ws_panel, wk.scratch + (size_t)nb * nb, sp);
        launch_qr_update2(Akk, gk, 0, Tkk, nullptr, 0, false, wk.scratch, nb, bk, nullptr, sp);
      } else if (dpiv) {
        // NEXT f1: partial pivoting over the stacked diagonal domain; W <- its pivoted top tile
        launch_dom_factor(A, g, k, Dp, wk, sp);
        if (need_inv) launch_tri_inv(g, k, wk, wk.scratch, wk.scratch + (size_t)nb * nb, sp);
      } else {
        launch_getrf(A, g, k, wk, true, sp);
        // the explicit triangular inverses feed only the criterion's ||A_kk^-1||_1 (Eliminate and
        // Apply solve with W itself)
        if (need_inv) launch_tri_inv(g, k, wk, wk.scratch, wk.scratch + (size_t)nb * nb, sp);
      }
      P.end(sp);
      if (stats_needed && criterion != HLQ_CRIT_MUMPS) {
        P.begin(HLQ_PROF_CRITERION, sp);
        launch_invnorm(g, k, wk, sp, opt.invnorm_estimate, a2 ? 1 : 0);
        P.end(sp);
      }
    } else {
      cudaMemsetAsync(w.zp, 0, sizeof(int), sp);
    }
    P.begin(HLQ_PROF_CRITERION, sp);
    launch_decide(g, k, criterion, alpha, opt.mumps_reading, opt.tie_rel_tol, opt.forced != nullptr,
                  w.ref_dec != nullptr, wk, sp);
    P.end(sp);
    if (spec) cudaStreamWaitEvent(sp, ev_qsrc, 0);
    if (known != HLQ_DEC_QR) {
      P.begin(HLQ_PROF_LU_TRSM, sp);
      launch_lu_panel(A, g, k, wk, sp, /*commit=*/!a2 && !dpiv);
      // the domain's stacked LU replaces its panel tiles (after the Eliminate GEMM, which also
      // wrote them: U_kk^-1 applies to the tiles off the domain only)
      if (dpiv) launch_dom_commit(A, g, k, Dp, wk, sp);
      // keep the composed row permutation of P_kk for the solve (A2: identity) and, for A2,
      // Q_kk^T for its forward pass
      launch_copy_ints(w.luperm + (size_t)k * nb,
                       reinterpret_cast<const int*>(wk.scratch + (size_t)2 * nb * nb), nb, w.dec, k,
                       sp);
      if (a2)
        launch_copy_block(w.luinv + (size_t)k * 2 * nb * nb, nb, wk.scratch, nb, nb, nb, nullptr,
                          w.dec, k, sp);
      P.end(sp);
    }
    if (spec) {
      // QR decision: the speculative panel replaces A's column block k (rows >= k0)
      cudaStreamWaitEvent(sp, ev_qdone, 0);
      const int64_t k0 = g.r0(k);
      launch_copy_block_if(A + k0 * lda + k0, lda, w.qpan + k0, N, N - k0, g.cbs(k), w.dec, k,
                           HLQ_DEC_QR, sp);
    } else if (known != HLQ_DEC_LU) {
      P.begin(HLQ_PROF_QR_GEQRT, sp);
      launch_qr_panel(A, g, k, ib, f->lvl_ptr[k].data(), f->lvl_cnt[k].data(), nl, wk, sp,
                      /*diag_done=*/a2 && known != HLQ_DEC_QR, /*spec=*/false, &f->tsplan[k],
                      &f->dag[k], f->dag_progress, ++f->dag_epoch);
      P.end(sp);
    }
    cudaEventRecord(ev_panel, sp);
    // ---- update stage U(k) on st: column block k+1 first (then P(k+1) may start), then the rest
    cudaStreamWaitEvent(st, ev_panel, 0);
    const int64_t k1 = g.r0(k) + g.bs(k);
    const bool fuse = f->track_growth && k + 1 < n && nb % cpr == 0;
    for (int part = 0; part < 2; ++part) {
      const int64_t c0 = (part == 0) ? k1 : std::min(g.N, k1 + nb);
      const int64_t c1 = (part == 0) ? std::min(g.N, k1 + nb) : g.N;
      cudaStream_t const st_upd = st;
      cudaStream_t st = (part == 0 && la_sp) ? sp : st_upd;  // (shadows the update stream below)
      if (part == 0 && la_sp && k > 0) cudaStreamWaitEvent(sp, ev_rest, 0);
      if (c1 > c0) {
        // (profile: the lookahead column on the panel stream overlaps the rest of the update, so
        // its bracket is its own class and the dominant class times only the update stream)
        const bool la_cls = part == 0 && la_sp;
        if (known != HLQ_DEC_QR) {
          P.begin(la_cls ? HLQ_PROF_OTHER : HLQ_PROF_LU_UPDATE, st);
          if (dpiv) launch_dom_swap_cols(A, g, k, Dp, w.dipiv + (size_t)k * nb, c0, c1, w.dec, st);
          launch_lu_update(A, g, k, wk, c0, c1, fuse ? w.colpart : nullptr, st, a2);
          P.end(st);
        }
        bool qr_fused = false;
        if (known != HLQ_DEC_LU) {
          P.begin(la_cls ? HLQ_PROF_OTHER : HLQ_PROF_QR_UNMQR, st);
          // a12 fused into the TTMQR epilogues: every row i > k is final after its merge
          qr_fused = launch_qr_update(A, g, k, ib, f->lvl_ptr[k].data(), f->lvl_cnt[k].data(), nl,
                                      wk, c0, c1, st,
                                      (f->track_growth && k + 1 < n) ? w.gstep + k + 1 : nullptr,
                                      &f->tsplan[k]);
          P.end(st);
        }
        // a12 for whatever branch did not fuse it: the LU GEMM epilogue (fuse) and the TTMQR
        // epilogues (qr_fused) cover their own branch; the rest is scanned, predicated on d_k
        const bool lu_done = fuse || known == HLQ_DEC_QR;
        const bool qr_done = qr_fused || known == HLQ_DEC_LU;
        if (f->track_growth && k + 1 < n && !(lu_done && qr_done)) {
          P.begin(HLQ_PROF_GROWTH, st);
          if (lu_done)
            launch_tile_norm_max(A, g, k + 1, w.gstep + k + 1, st, w.dec, k, HLQ_DEC_QR, c0, c1);
          else if (qr_done)
            launch_tile_norm_max(A, g, k + 1, w.gstep + k + 1, st, w.dec, k, HLQ_DEC_LU, c0, c1);
          else
            launch_tile_norm_max(A, g, k + 1, w.gstep + k + 1, st, nullptr, 0, 0, c0, c1);
          P.end(st);
        }
      }
      if (part == 0) cudaEventRecord(ev_ready, st);
    }
    if (la_sp) cudaStreamWaitEvent(st, ev_ready, 0);  // the lookahead column (on sp) is done too
    if (fuse && known != HLQ_DEC_QR) {
      P.begin(HLQ_PROF_GROWTH, st);
      launch_lu_growth(w, g, k, st);
      P.end(st);
    }
    if (la_sp) cudaEventRecord(ev_rest, st);
    if (P.on) cudaEventRecord(f->step_ev[k + 1], st);  // step k's update stage is done
    if (nvtx_on()) nvtxRangePop();
  }
  int* scan = w.status + 2;
  launch_final_scan(A, N, lda, scan, st);
  if ((rc = cuda_err(cudaGetLastError()))) return rc;

  f->dec.resize(n);
  f->margin.resize(n);
  f->flags.resize(n);
  f->gstep.resize(n + 1);
  int stat[4];
  cudaMemcpyAsync(f->dec.data(), w.dec, n, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(f->margin.data(), w.margin, sizeof(double) * n, cudaMemcpyDeviceToHost, st);
  f->steplog.resize(2 * (size_t)n);
  cudaMemcpyAsync(f->steplog.data(), w.steplog, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(f->flags.data(), w.flags, sizeof(int) * n, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(f->gstep.data(), w.gstep, sizeof(double) * (n + 1), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(stat, w.status, sizeof(int) * 4, cudaMemcpyDeviceToHost, st);
  if ((rc = cuda_err(cudaStreamSynchronize(st)))) return rc;
  if (P.on) P.collect();
  // status priority: non-finite > zero pivot in a forced LU step > singular
  if (stat[0] || stat[2])
    f->status = HLQ_ST_NONFINITE;
  else if (stat[1])
    f->status = HLQ_ST_ZERO_PIVOT_FORCED;
  else if (stat[3])
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

int hlq_factor(double* A, int64_t N, int32_t nb, int32_t criterion, double alpha,
               hlq_factors_t* out) {
  return hlq_factor_ex(A, N, nb, criterion, alpha, nullptr, out);
}

int hlq_solve(hlq_factors_t f, const double* b, double* x) {
  NvtxScope nvtx_scope("hlq_solve");
  if (!f || f->dec.empty()) return -1;
  if (!b) return -2;
  if (!x) return -3;
  if (f->status == HLQ_ST_SINGULAR) return HLQ_ST_SINGULAR;
  if (f->dist) return hlq::dist_solve_entry(f, b, x);
  const Geo g = f->g;
  cudaStream_t st = f->st;
  int rc;
  f->prof.begin(HLQ_PROF_SOLVE, st);
  if (x != b &&
      (rc = cuda_err(cudaMemcpyAsync(x, b, sizeof(double) * g.N, cudaMemcpyDeviceToDevice, st))))
    return rc;
  // forward pass: replay every step on x (LU: P_kk, L_kk^-1 by substitution, x_i -= L_ik x_k;
  // A2: Q_kk^T; QR: the stored reflectors of the tree), then block back substitution with U_kk /
  // R_kk.  Runs of consecutive A1 LU steps and the back substitution are single persistent
  // launches (solve.cu k_solve_rows); QR, A2 and domain-pivoting steps replay step by step.
  const int n = g.n, G = solve_g(), cmax = solve_rows_cmax(n, G);
  if (!f->solve_ws) {
    auto eligible = [&](int k) {
      return f->dec[k] == HLQ_DEC_LU && f->lu_variant == HLQ_LU_A1 &&
             f->pivot_scope == HLQ_PIVOT_TILE;
    };
    std::vector<int2> table;
    f->solve_runs.clear();
    f->solve_unit_off.clear();
    f->solve_unit_cnt.clear();
    size_t used = 0;
    for (int k = 0; k < n;) {
      if (!eligible(k)) { ++k; continue; }
      int kb = k;
      while (kb < n && eligible(kb)) ++kb;
      f->solve_runs.push_back({k, kb});
      table.resize(used + (size_t)(n - k) * cmax);
      const size_t cnt = build_solve_units(true, n, k, kb, G, table.data() + used);
      f->solve_unit_off.push_back(used);
      f->solve_unit_cnt.push_back(cnt);
      used += cnt;
      k = kb;
    }
    table.resize(used + (size_t)n * cmax);
    const size_t cb = build_solve_units(false, n, 0, n, G, table.data() + used);
    f->solve_unit_off.push_back(used);
    f->solve_unit_cnt.push_back(cb);
    used += cb;
    if (used <= f->solve_cap) {
      f->solve_ws = f->solve_ws_in;  // the factorization's workspace piece
    } else {  // many alternating LU runs: a larger table
      if ((rc = cuda_err(cudaMalloc(&f->solve_ws_own, solve_ws_bytes(n, g.nb, cmax, used))))) {
        f->solve_ws_own = nullptr;
        return rc;
      }
      f->solve_ws = f->solve_ws_own;
    }
    f->solve_used = used;
    if ((rc = cuda_err(cudaMemcpyAsync(f->solve_ws, table.data(), sizeof(int2) * used,
                                       cudaMemcpyHostToDevice, st))))
      return rc;
  }
  if (!f->qsolve_built) {
    // runs of consecutive QR steps: one DAG of Q^T applies each (qr.cu k_qr_solve_dag); an op
    // waits for the previous op on each of its rows, across the run's steps
    f->qsolve_built = true;
    static int qenv = -1;
    if (qenv < 0) qenv = getenv("HLQ_QR_SOLVE_DAG") ? atoi(getenv("HLQ_QR_SOLVE_DAG")) : 1;
    std::vector<int> ops;
    size_t maxops = 0;
    for (int k = 0; k < n && qenv != 0;) {
      if (f->dec[k] != HLQ_DEC_QR) { ++k; continue; }
      int kb = k;
      while (kb < n && f->dec[kb] == HLQ_DEC_QR) ++kb;
      const size_t off = ops.size() / 6;
      std::vector<int> last(n, -1);
      auto add = [&](int kind, int e, int i, int step) {
        const int id = (int)(ops.size() / 6) - (int)off;
        ops.insert(ops.end(), {kind, e, i, kind == 0 ? -1 : last[e], last[i], step});
        last[i] = id;
        if (kind != 0) last[e] = id;
      };
      for (int s = k; s < kb; ++s) {
        StepPlanHost p;
        plan_step(s, n, f->D, f->ts_group, p);
        if (f->ts_group >= 1 && p.ts_off.size() > 1) {
          for (int h : p.heads) add(0, h, h, s);
          for (const int2& pr : p.ts_pairs) add(1, pr.x, pr.y, s);
        } else {
          for (int i = s; i < n; ++i) add(0, i, i, s);
        }
        for (const auto& lv : p.levels)
          for (const int2& pr : lv) add(2, pr.x, pr.y, s);
      }
      const size_t cnt = ops.size() / 6 - off;
      f->qsolve_runs.push_back({k, kb, (int)off, (int)cnt});
      maxops = std::max(maxops, cnt);
      k = kb;
    }
    if (!ops.empty()) {
      size_t ob = align_up(sizeof(int) * ops.size(), 256);
      if (ops.size() / 6 <= f->qsolve_cap && f->qsolve_ws_in) {
        f->qsolve_ops = f->qsolve_ws_in;  // the factorization's workspace piece
        ob = align_up(sizeof(int) * 6 * (f->qsolve_cap + 1), 256);
      } else {
        if ((rc = cuda_err(cudaMalloc(&f->qsolve_block, ob + sizeof(int) * 32 * maxops)))) {
          f->qsolve_block = nullptr;
          f->qsolve_runs.clear();
          return rc;
        }
        f->qsolve_ops = f->qsolve_block;
      }
      f->qsolve_done = (int*)((char*)f->qsolve_ops + ob);
      if ((rc = cuda_err(cudaMemcpyAsync(f->qsolve_ops, ops.data(), sizeof(int) * ops.size(),
                                         cudaMemcpyHostToDevice, st))))
        return rc;
    }
  }
  char* sw = (char*)f->solve_ws;
  const size_t used = f->solve_used > f->solve_cap ? f->solve_used : f->solve_cap;
  const int2* units = (const int2*)sw;
  int* xflag = (int*)(sw + align_up(sizeof(int2) * used, 256));
  int* pflag = (int*)((char*)xflag + align_up(kFlagBytes * n, 256));
  double* part = (double*)((char*)pflag + align_up(kFlagBytes * (size_t)n * cmax, 256));
  unsigned* ticket = (unsigned*)(part + (size_t)n * cmax * g.nb);
  size_t run = 0, qrun = 0;
  for (int k = 0; k < n; ++k) {
    if (qrun < f->qsolve_runs.size() && f->qsolve_runs[qrun][0] == k) {
      const auto& r = f->qsolve_runs[qrun++];
      launch_qr_solve_dag(f->A, g, f->ib, f->w.Tg, f->w.Ttt,
                          (const int*)f->qsolve_ops + (size_t)6 * r[2], r[3], f->qsolve_done, x,
                          st);
      k = r[1] - 1;
      continue;
    }
    if (run < f->solve_runs.size() && f->solve_runs[run].first == k) {
      const int kb = f->solve_runs[run].second;
      launch_solve_rows(true, f->A, g, k, kb, G, units + f->solve_unit_off[run],
                        f->solve_unit_cnt[run], f->w.luperm, x, xflag, part, pflag, ticket, st);
      ++run;
      k = kb - 1;
      continue;
    }
    if (f->dec[k] == HLQ_DEC_LU && f->pivot_scope == HLQ_PIVOT_DOMAIN)
      launch_dom_swap_vec(x, g, k, f->D, f->w.dipiv + (size_t)k * g.nb, st);
    if (f->dec[k] == HLQ_DEC_LU && f->lu_variant == HLQ_LU_A2)
      launch_solve_lu_fwd_inv(f->A, g, k, f->w.luinv + (size_t)k * 2 * g.nb * g.nb,
                              f->w.luperm + (size_t)k * g.nb, x, f->w.solve_t, st,
                              /*dense=*/true);
    else if (f->dec[k] == HLQ_DEC_LU)
      launch_solve_lu_fwd(f->A, g, k, nullptr, x, st);  // domain pivoting: rows already swapped
    else
      launch_qr_apply(f->A, g, k, f->ib, f->w.Tg, f->w.Ttt, f->lvl_ptr[k].data(),
                      f->lvl_cnt[k].data(), (int)f->lvl_cnt[k].size(), x, g.N, 1, nullptr, st,
                      &f->tsplan[k]);
  }
  launch_solve_rows(false, f->A, g, 0, n, G, units + f->solve_unit_off.back(),
                    f->solve_unit_cnt.back(), nullptr, x, xflag, part, pflag, ticket, st);
  f->prof.end(st);
  if ((rc = cuda_err(cudaGetLastError()))) return rc;
  if (f->blocking && (rc = cuda_err(cudaStreamSynchronize(st)))) return rc;
  if (f->prof.on && f->blocking) f->prof.collect();
  return 0;
}

int hlq_get_info(hlq_factors_t f, hlq_info* info) {
  if (!f || f->dec.empty()) return -1;
  if (!info) return -2;
  memset(info, 0, sizeof(*info));
  const Geo g = f->g;
  info->N = g.N;
  info->nb = g.nb;
  info->n = g.n;
  info->ib = f->ib;
  info->D = f->D;
  info->status = f->status;
  info->growth = f->growth;
  double Nd = (double)g.N;
  info->fake_flops = 2.0 / 3.0 * Nd * Nd * Nd;
  double tf = 0.0;
  for (int k = 0; k < g.n; ++k) {
    double b = g.bs(k), M = (double)(g.N - g.r0(k) - g.bs(k));
    double lu = 2.0 / 3.0 * b * b * b + 2.0 * M * b * b + 2.0 * M * M * b;  // Table I
    // A2: Factor and Apply cost twice A1's: 4/3 b^3 + M b^2 + 2 M b^2 + 2 M^2 b
    const double lu2 = 4.0 / 3.0 * b * b * b + 3.0 * M * b * b + 2.0 * M * M * b;
    tf += f->dec[k] == HLQ_DEC_QR ? 2.0 * lu : (f->lu_variant == HLQ_LU_A2 ? lu2 : lu);
    if (f->dec[k] == HLQ_DEC_QR) info->qr_steps++;
    if (f->flags[k] & HLQ_FLAG_NEAR_TIE) info->near_ties++;
    if (f->flags[k] & HLQ_FLAG_HINTED) info->hinted++;
  }
  info->true_flops = tf;
  return 0;
}

int hlq_get_profile(hlq_factors_t f, double* ms, double* flops, int64_t* launches) {
  if (!f || f->dec.empty()) return -1;
  if (!f->prof.on) return -2;
  cudaStreamSynchronize(f->st);
  f->prof.collect();
  const Geo g = f->g;
  double fl[HLQ_PROF_NCLASSES] = {0};
  for (int k = 0; k < g.n; ++k) {
    double b = g.bs(k), M = (double)(g.N - g.r0(k) - g.bs(k));
    // the update flops are proportional to the columns updated: the lookahead column block's
    // share is its own class when it ran on the panel stream
    const double la = (f->la_sp && M > 0) ? std::min((double)g.nb, M) / M : 0.0;
    if (f->dec[k] == HLQ_DEC_LU) {
      const bool a2 = f->lu_variant == HLQ_LU_A2;  // Factor and Apply cost twice
      fl[HLQ_PROF_GETRF] += (a2 ? 4.0 : 2.0) / 3.0 * b * b * b;
      fl[HLQ_PROF_LU_TRSM] += M * b * b;             // Table I: TRSM
      const double u = (a2 ? 2.0 : 1.0) * M * b * b + 2.0 * M * M * b;  // SWPTRSM + GEMM
      fl[HLQ_PROF_LU_UPDATE] += (1.0 - la) * u;
      fl[HLQ_PROF_OTHER] += la * u;
    } else {
      double m = M / b;                              // trailing tiles (fractional if ragged)
      fl[HLQ_PROF_QR_GEQRT] += (m + 1.0) * 4.0 / 3.0 * b * b * b + m * 2.0 / 3.0 * b * b * b;
      const double u = (m + 1.0) * 2.0 * b * b * M + m * 2.0 * b * b * M;
      fl[HLQ_PROF_QR_UNMQR] += (1.0 - la) * u;
      fl[HLQ_PROF_OTHER] += la * u;
    }
  }
  for (int c = 0; c < HLQ_PROF_NCLASSES; ++c) {
    if (ms) ms[c] = f->prof.ms[c];
    if (flops) flops[c] = fl[c];
    if (launches) launches[c] = f->prof.launches[c];
  }
  return 0;
}

int64_t hlq_launch_count(void) { return hlq::g_launches; }

int hlq_get_decisions(hlq_factors_t f, uint8_t* dec) {
  if (!f || f->dec.empty()) return -1;
  if (!dec) return -2;
  memcpy(dec, f->dec.data(), f->dec.size());
  return 0;
}
int hlq_get_margins(hlq_factors_t f, double* m) {
  if (!f || f->dec.empty()) return -1;
  if (!m) return -2;
  memcpy(m, f->margin.data(), sizeof(double) * f->margin.size());
  return 0;
}
int hlq_get_step_log(hlq_factors_t f, double* log2n) {
  if (!f || f->dec.empty()) return -1;
  if (!log2n) return -2;
  if (f->steplog.size() != 2 * f->dec.size()) return HLQ_ERR_STATE;
  memcpy(log2n, f->steplog.data(), sizeof(double) * f->steplog.size());
  return 0;
}
int hlq_get_step_times(hlq_factors_t f, double* ms) {
  if (!f || f->dec.empty()) return -1;
  if (!ms) return -2;
  if (!f->prof.on || f->step_ev.size() != f->dec.size() + 1) return HLQ_ERR_STATE;
  cudaStreamSynchronize(f->st);
  for (size_t k = 0; k + 1 < f->step_ev.size(); ++k) {
    float t = 0.f;
    cudaEventElapsedTime(&t, f->step_ev[k], f->step_ev[k + 1]);
    ms[k] = t;
  }
  return 0;
}
int hlq_get_step_flags(hlq_factors_t f, int32_t* fl) {
  if (!f || f->dec.empty()) return -1;
  if (!fl) return -2;
  memcpy(fl, f->flags.data(), sizeof(int) * f->flags.size());
  return 0;
}
int hlq_get_growth(hlq_factors_t f, double* gr) {
  if (!f || f->dec.empty()) return -1;
  if (!gr) return -2;
  *gr = f->growth;
  return 0;
}
int hlq_get_pivots(hlq_factors_t f, int32_t* ipiv) {
  if (!f || f->dec.empty()) return -1;
  if (!ipiv) return -2;
  if (f->dist) return HLQ_ERR_STATE;
  return cuda_err(cudaMemcpy(ipiv, f->w.ipiv, sizeof(int) * (size_t)f->g.n * f->g.nb,
                             cudaMemcpyDeviceToHost));
}
int hlq_get_T(hlq_factors_t f, int32_t i, int32_t k, int32_t kind, double* T) {
  if (!f || f->dec.empty()) return -1;
  if (k < 0 || k >= f->g.n) return -3;
  if (i < k || i >= f->g.n) return -2;
  if (kind < 0 || kind > 1) return -4;
  if (!T) return -5;
  if (f->dist) return HLQ_ERR_STATE;
  const double* src = (kind == 0 ? f->w.Tg : f->w.Ttt) + tri_index(i, k, f->g.n) * (int64_t)f->ib * f->g.nb;
  return cuda_err(cudaMemcpy(T, src, sizeof(double) * f->ib * f->g.nb, cudaMemcpyDeviceToHost));
}

void hlq_free(hlq_factors_t f) {
  if (!f) return;
  if (f->dist) {
    cudaStreamSynchronize(f->st);
    hlq::dist_free(f->dist);
    f->dist = nullptr;
  }
  if (f->ws_block) {
    cudaStreamSynchronize(f->st);
    cache_put(f->dev, 0, f->ws_block, f->ws_bytes);
  }
  if (f->tma_maps) free_tma_maps(f->tma_maps);
  if (f->qsolve_block) {
    cudaStreamSynchronize(f->st);
    cudaFree(f->qsolve_block);
  }
  if (f->solve_ws_own) {
    cudaStreamSynchronize(f->st);
    cudaFree(f->solve_ws_own);
  }
  f->prof.collect();
  for (auto e : f->ev)
    if (e) cudaEventDestroy(e);
  for (auto e : f->step_ev)
    if (e) cudaEventDestroy(e);
  delete f;
}

int hlq_gesv_host(const double* A_host, const double* b_host, double* x_host, int64_t N,
                  int32_t nb, int32_t criterion, double alpha, const hlq_options* opt,
                  hlq_info* info) {
  if (!A_host) return -1;
  if (!b_host) return -2;
  if (!x_host) return -3;
  if (N <= 0) return -4;
  hlq_options o;
  hlq_default_options(&o);
  if (opt) o = *opt;
  cudaStream_t st = (cudaStream_t)o.stream;
  size_t abytes = sizeof(double) * (size_t)N * N;
  const int dev = cur_device();
  char* buf = (char*)cache_get(1, abytes + 2 * sizeof(double) * (size_t)N + 512);
  if (!buf) return HLQ_ERR_NOMEM;
  double* dA = (double*)buf;
  double* db = (double*)(buf + align_up(abytes, 256));
  double* dx = db + align_up(N, 32);
  int rc;
  if ((rc = cuda_err(cudaMemcpyAsync(dA, A_host, abytes, cudaMemcpyHostToDevice, st))) ||
      (rc = cuda_err(cudaMemcpyAsync(db, b_host, sizeof(double) * N, cudaMemcpyHostToDevice, st)))) {
    cache_put(dev, 1, buf, abytes + 2 * sizeof(double) * (size_t)N + 512);
    return rc;
  }
  o.lda = N;
  hlq_factors_t f = nullptr;
  int st_f = hlq_factor_ex(dA, N, nb, criterion, alpha, &o, &f);
  if (st_f >= 0) {
    rc = hlq_solve(f, db, dx);
    if (rc == 0)
      rc = cuda_err(cudaMemcpyAsync(x_host, dx, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
    if (rc == 0) rc = cuda_err(cudaStreamSynchronize(st));
    if (info) hlq_get_info(f, info);
  } else {
    rc = st_f;
  }
  hlq_free(f);
  cache_put(dev, 1, buf, abytes + 2 * sizeof(double) * (size_t)N + 512);
  return rc != 0 ? rc : st_f;
}

int hlq_generate_uniform(double* dst, int64_t rows, int64_t cols, int64_t ld, uint64_t seed,
                         uint64_t idx0, int64_t idx_ld, void* stream) {
  if (!dst) return -1;
  if (rows < 0) return -2;
  if (cols < 0) return -3;
  if (ld < rows) return -4;
  launch_generate(dst, rows, cols, ld, seed, idx0, idx_ld, (cudaStream_t)stream);
  return cuda_err(cudaGetLastError());
}

int hlq_residual(const double* A, int64_t N, int64_t lda, const double* x, const double* b,
                 double* out3, void* stream) {
  if (!A) return -1;
  if (N <= 0) return -2;
  if (lda < N) return -3;
  if (!x) return -4;
  if (!b) return -5;
  if (!out3) return -6;
  cudaStream_t st = (cudaStream_t)stream;
  double* d = nullptr;
  int rc;
  if ((rc = cuda_err(cudaMallocAsync((void**)&d, 3 * sizeof(double), st)))) return rc;
  launch_residual(A, N, lda, x, b, d, st);
  rc = cuda_err(cudaMemcpyAsync(out3, d, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
  cudaFreeAsync(d, st);
  if (!rc) rc = cuda_err(cudaStreamSynchronize(st));
  return rc;
}

}  // extern "C"
