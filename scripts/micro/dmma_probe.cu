// DMMA.8x8x4 latency / throughput probe (B200): one CTA per SM, `warps` warps,
// each issuing `chains` independent accumulator chains of `iters` DMMAs.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void probe(double *out, int iters, long long *cyc) {
  double d0[CH], d1[CH];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int c = 0; c < CH; ++c) d0[c] = d1[c] = c;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(d0[c], d1[c], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d0[c] + d1[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int CH>
void run(int warps, double *out, long long *cyc) {
  const int iters = 2000;
  probe<CH><<<148, 32 * warps>>>(out, iters, cyc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<CH><<<148, 32 * warps>>>(out, iters, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  double n = (double)iters * CH;  // DMMAs per warp
  printf("chains %2d warps %2d: %8.1f cycles per DMMA per warp (clock64), per-SMSP DMMA interval %.1f cycles, %.2f TFLOP/s\n",
         CH, warps, (double)c / n, (double)c / (n * warps / 4.0),
         148.0 * warps * n * 512.0 / (ms * 1e-3) / 1e12);
}
int main() {
  double *out; long long *cyc;
  cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&cyc, 8);
  for (int w : {1, 4, 8, 16}) { run<1>(w, out, cyc); run<2>(w, out, cyc); run<4>(w, out, cyc); run<8>(w, out, cyc); }
  return 0;
}
