// FP64 peak microbenchmark for B200 (sm_100a): measurement only, not product code.
// Measures sustained throughput of
//   (1) warp-level DMMA  mma.sync.aligned.m8n8k4.row.col.f64   (the FP64 tensor path)
//   (2) warp-level DMMA  mma.sync.aligned.m16n8k16.row.col.f64
//   (3) plain DFMA (fma.rn.f64) on the FP64 ALU pipe
// Each warp runs independent accumulator chains back to back on every SM, timed with CUDA events.
// Prints one JSON line per measurement.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_dmma884(double* out, long iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (long it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_dmma16816(double* out, long iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - (threadIdx.x + i) * 1e-9;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0.0;
  for (long it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_dfma(double* out, long iters) {
  double x = 1.0 + threadIdx.x * 1e-9, y = 1.0 - threadIdx.x * 1e-12;
  double c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] = i;
  for (long it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(c[i], y, x);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

template <typename K>
static int run(const char* name, K kern, int threads, int blocks_per_sm, long iters, double flop_per_warp_iter) {
  int dev = 0, sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* out; CK(cudaMalloc(&out, 8));
  int grid = sms * blocks_per_sm;
  kern<<<grid, threads>>>(out, iters / 10);  // warm-up
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f, total = 0.f; int reps = 5;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    kern<<<grid, threads>>>(out, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    total += ms; if (ms < best) best = ms;
  }
  double warps = (double)grid * threads / 32.0;
  double flops = warps * iters * flop_per_warp_iter;
  printf("{\"kernel\": \"%s\", \"sms\": %d, \"grid\": %d, \"threads\": %d, \"best_ms\": %.3f, \"mean_ms\": %.3f, "
         "\"tflops_best\": %.3f, \"tflops_mean\": %.3f, \"flop_per_clk_per_sm_at_1965MHz\": %.2f}\n",
         name, sms, grid, threads, best, total / reps, flops / best / 1e9, flops / (total / reps) / 1e9,
         flops / (best * 1e-3) / sms / 1.965e9);
  fflush(stdout);
  cudaFree(out);
  return 0;
}

int main() {
  // m8n8k4: 8*8*4 FMA = 256 FMA = 512 flop per instruction, 8 per iteration
  for (int bps : {1, 2, 4})
    run("dmma_m8n8k4", k_dmma884, 256, bps, 200000, 8 * 512.0);
  // m16n8k16: 16*8*16 = 2048 FMA = 4096 flop, 4 per iteration
  for (int bps : {1, 2, 4})
    run("dmma_m16n8k16", k_dmma16816, 256, bps, 50000, 4 * 4096.0);
  // DFMA: 32 lanes * 8 fma * 2 flop per warp-iteration
  for (int bps : {1, 2, 4})
    run("dfma", k_dfma, 256, bps, 200000, 32 * 8 * 2.0);
  return 0;
}
