// DMMA + shared-memory B-operand probe (measurement only): the v3 QR-update inner pattern
// (one LDS.128 feeding 4 DMMAs on 4 accumulators, A operands in registers), with and without a
// __syncthreads every SYNC_EVERY LDS groups, at several warps per SM.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma_(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int SYNC>
__global__ void k(double* out, long iters) {
  __shared__ __align__(16) double sm[32 * 40 * 2];
  for (int i = threadIdx.x; i < 32 * 40 * 2; i += blockDim.x) sm[i] = 1e-3 * i;
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double a[2][4][2], c[2][2][2];
  for (int m = 0; m < 2; ++m) for (int n = 0; n < 4; ++n) { a[m][n][0] = 1.0 + m; a[m][n][1] = 1.0 - n * 1e-3; }
  for (int m = 0; m < 2; ++m) for (int q = 0; q < 2; ++q) c[m][q][0] = c[m][q][1] = 0.0;
  for (long it = 0; it < iters; ++it) {
    const double* V = sm + (it & 1) * 1280;
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int nl = 0; nl < 4; ++nl) {
        const double2 bv = *reinterpret_cast<const double2*>(V + (8 * q + g) * 40 + 8 * nl + 2 * t);
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          dmma_(c[m][q][0], c[m][q][1], a[m][nl][0], bv.x);
          dmma_(c[m][q][0], c[m][q][1], a[m][nl][1], bv.y);
        }
      }
    if (SYNC) __syncthreads();
  }
  double s = 0;
  for (int m = 0; m < 2; ++m) for (int q = 0; q < 2; ++q) s += c[m][q][0] + c[m][q][1];
  if (s == 12345.678) out[0] = s;
}
template <int SYNC>
void run(int nw, int cps) {
  double* o;
  cudaMalloc(&o, 8);
  long iters = 20000;
  k<SYNC><<<148 * cps, nw * 32>>>(o, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<SYNC><<<148 * cps, nw * 32>>>(o, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = 148.0 * cps * nw * iters * 32 * 512.0;
  printf("{\"sync\": %d, \"warps_per_cta\": %d, \"ctas_per_sm\": %d, \"tflops\": %.2f}\n", SYNC, nw, cps, fl / ms / 1e9);
  cudaFree(o);
}
int main() {
  for (int nw : {4, 8, 16}) { run<0>(nw, 1); run<1>(nw, 1); }
  run<1>(4, 2); run<1>(8, 2);
  return 0;
}
