// DFMA dependent-issue latency / throughput probe (B200): one CTA on one SM,
// `warps` warps, each thread runs `ilp` independent chains of dependent DFMAs.
// Prints cycles per DFMA per warp and the SM-wide DFMA rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dfma_probe dfma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void probe(double *out, long long *cyc, int iters, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-3 + i;
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int ILP>
void run(int warps) {
  double *out;
  long long *cyc, h;
  cudaMalloc(&out, sizeof(double) * 1024);
  cudaMalloc(&cyc, sizeof(long long));
  const int iters = 2000;
  probe<ILP><<<1, 32 * warps>>>(out, cyc, iters, 0.999999, 1e-9);
  probe<ILP><<<1, 32 * warps>>>(out, cyc, iters, 0.999999, 1e-9);
  cudaMemcpy(&h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  const double per = (double)h / (iters * 16.0 * ILP);
  printf("warps %2d ilp %d: %.2f cycles per DFMA per warp, %.1f DFMA lanes/clk/SM\n", warps, ILP, per,
         32.0 * warps / per);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {1, 4, 8, 16, 32}) {
    run<1>(w);
    run<2>(w);
    run<4>(w);
    run<8>(w);
  }
  return 0;
}
