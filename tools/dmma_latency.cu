// DMMA.8x8x4 issue interval and dependent latency on one SM sub-partition:
// one CTA of W warps per SM; every warp runs N mma.m8n8k4.f64 over ILP
// independent accumulators (ILP = 1: a fully dependent chain).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_latency tools/dmma_latency.cu && tools/dmma_latency
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int ILP>
__global__ void k(int iters, double* out, long long* clk) {
  double acc[ILP][2];
  for (int i = 0; i < ILP; ++i) acc[i][0] = acc[i][1] = 0.0;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) dmma(acc[i][0], acc[i][1], a, b);
  }
  const long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < ILP; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

template <int ILP>
void run(int warps) {
  double* out; long long* clk;
  cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&clk, 8);
  const int iters = 4096;
  k<ILP><<<148, warps * 32>>>(iters, out, clk);
  k<ILP><<<148, warps * 32>>>(iters, out, clk);
  long long h; cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
  const double per_warp = (double)h / ((double)iters * ILP);
  printf("warps/CTA %2d (per sub-partition %.1f) ILP %2d: %.2f clk per DMMA per warp, %.2f clk per DMMA per sub-partition\n",
         warps, warps / 4.0, ILP, per_warp, per_warp / (warps / 4.0));
  cudaFree(out); cudaFree(clk);
}

int main() {
  for (int w : {4, 8, 12, 16}) { run<1>(w); run<2>(w); run<4>(w); run<8>(w); run<13>(w); }
  return 0;
}
