// DMMA chain-latency probe (measurement only): throughput of mma.sync m8n8k4.f64 with NCH
// independent accumulator chains per warp and NW warps per SM (one CTA per SM).
#include <cstdio>
#include <cuda_runtime.h>
template <int NCH>
__global__ void k(double* out, long iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NCH][2];
#pragma unroll
  for (int i = 0; i < NCH; ++i) c[i][0] = c[i][1] = 0.0;
  for (long it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
template <int NCH>
void run(int nw) {
  double* o;
  cudaMalloc(&o, 8);
  long iters = 20000 / NCH * 8;
  k<NCH><<<148, nw * 32>>>(o, 100);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<NCH><<<148, nw * 32>>>(o, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = 148.0 * nw * iters * NCH * 512.0;
  printf("{\"chains\": %d, \"warps_per_sm\": %d, \"tflops\": %.2f}\n", NCH, nw, fl / ms / 1e9);
  cudaFree(o);
}
int main() {
  for (int nw : {4, 8, 16}) {
    run<1>(nw); run<2>(nw); run<4>(nw); run<8>(nw);
  }
  return 0;
}
