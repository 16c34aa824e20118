// The factorization handle behind hlq_factors_t and its CUDA-event profiler (shared by api.cu and
// the 2D block-cyclic path in dist.cu).
#pragma once
#include <stdlib.h>
#include <stdio.h>

#include <utility>
#include <array>
#include <vector>

#include "hlq_internal.cuh"

namespace hlq {
struct DistState;
}
using hlq::DevWork;
using hlq::Geo;

// CUDA-event profiler: begin/end pairs recorded on the factorization's stream, per kernel class.
struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> ev;  // pairs
  std::vector<int> cls;
  std::vector<int64_t> l0;      // launch counter at begin
  int64_t launches[HLQ_PROF_NCLASSES] = {0};
  double ms[HLQ_PROF_NCLASSES] = {0};
  int cur = -1;
  int debug = -1;
  void check(const char* where, int k) {
    if (debug < 0) debug = getenv("HLQ_DEBUG_SYNC") ? 1 : 0;
    if (!debug) return;
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) fprintf(stderr, "[hlq debug] %s (k=%d): %s\n", where, k, cudaGetErrorString(e));
  }
  void begin(int c, cudaStream_t st) {
    check("before stage", c);
    cur = c;
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    ev.push_back(e);
    cls.push_back(c);
    l0.push_back(hlq::g_launches);
  }
  void end(cudaStream_t st) {
    check("after stage", cur);
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    ev.push_back(e);
    launches[cls.back()] += hlq::g_launches - l0.back();
  }
  void collect() {  // after a stream synchronisation
    for (size_t i = 0; i + 1 < ev.size(); i += 2) {
      float t = 0.f;
      cudaEventElapsedTime(&t, ev[i], ev[i + 1]);
      ms[cls[i / 2]] += t;
    }
    for (auto e : ev) cudaEventDestroy(e);
    ev.clear();
    cls.clear();
    l0.clear();
  }
};

struct hlq_factors_s {
  Prof prof;
  bool la_sp = false;  // the lookahead column's update ran on the panel stream (class OTHER)
  cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  double* A = nullptr;
  Geo g{};
  int ib = 32, D = 1, crit = 0;
  int lu_variant = 0;  // HLQ_LU_A1 / HLQ_LU_A2
  int pivot_scope = 0;  // HLQ_PIVOT_TILE / HLQ_PIVOT_DOMAIN
  double alpha = 1.0;
  cudaStream_t st = nullptr;
  bool blocking = true;
  DevWork w{};
  void* ws_block = nullptr;
  int dev = 0;  // device of the workspace block
  size_t ws_bytes = 0;
  int tree = 0, ts_group = 0;  // HLQ_TREE_*, the HQR TS group size (0: greedy)
  std::vector<hlq::QRTsPlan> tsplan;  // per step: the HQR TS level (ngroups = 0: none)
  std::vector<hlq::QRDag> dag;        // per step: the QR panel as one DAG launch (empty: off)
  int* dag_progress = nullptr;        // device, per op of a DAG launch
  int dag_epoch = 0;                  // launches so far (progress values are epoch << 8 | blocks)
  // QR-tree plan: per step k, TT levels l: device pointer + count
  std::vector<std::vector<const int2*>> lvl_ptr;
  std::vector<std::vector<int>> lvl_cnt;
  // host results
  std::vector<uint8_t> dec;
  std::vector<double> margin;
  std::vector<int> flags;
  std::vector<double> gstep;
  std::vector<double> steplog;         // 2n: lhs, rhs of each step's binding criterion inequality
  std::vector<cudaEvent_t> step_ev;    // profiling: n+1 events on the update stream (step times)
  int status = 0;
  double growth = 0.0;
  bool track_growth = true;
  // persistent-solve workspace (allocated at the first hlq_solve): unit tables per forward LU run
  // and for the back substitution, flags, chunk partial sums
  void* tma_maps = nullptr;      // gemm_tma.cu tensor maps of A (host memory) or null
  void* solve_ws = nullptr;      // = solve_ws_in, or solve_ws_own when the tables outgrow it
  void* solve_ws_in = nullptr;   // piece of the factorization workspace (table capacity solve_cap)
  void* solve_ws_own = nullptr;  // own allocation (freed by hlq_free)
  size_t solve_cap = 0, solve_used = 0;
  std::vector<std::pair<int, int>> solve_runs;   // [ka, kb) of every forward LU run
  std::vector<size_t> solve_unit_off, solve_unit_cnt;  // per run (+1: back pass) in the table
  // the solve's Q^T replay of runs of consecutive QR steps as DAG launches (built at the first
  // hlq_solve): device ops (6 ints each) + completion flags in qsolve_block, per run {ka, kb, off,
  // count}
  void* qsolve_block = nullptr;   // own allocation (only when the workspace piece is too small)
  void* qsolve_ops = nullptr;     // the op table in use (workspace piece or qsolve_block)
  void* qsolve_ws_in = nullptr;   // the factorization workspace's piece: ops + flags
  size_t qsolve_cap = 0;          // ops it holds (every step QR)
  int* qsolve_done = nullptr;
  std::vector<std::array<int, 4>> qsolve_runs;
  bool qsolve_built = false;
  // 2D block-cyclic factorization state (dist.cu); nullptr on the single-GPU path
  hlq::DistState* dist = nullptr;
};

