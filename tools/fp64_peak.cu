// FP64 peak probe for B200 (sm_100a): DMMA (mma.sync .f64) vs DFMA.
// Register-only loops; reports TFLOP/s measured with CUDA events.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int NACC>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x, b = seed * 0.5 + threadIdx.x;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}

template <int NACC>
__global__ void dmma16_loop(double* out, int iters, double seed) {
  // m16n8k16: A 8 regs, B 4 regs, C 4 regs
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + i + threadIdx.x;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = seed * 0.25 + i;
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1.2345) out[0] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double x[NACC];
  double a = seed + threadIdx.x * 1e-9, b = 1.0 - 1e-12;
#pragma unroll
  for (int i = 0; i < NACC; ++i) x[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) x[i] = fma(x[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}

// Mixed probe: on every SM sub-partition half the warps run DMMA, half DFMA.
// If both rates add up past ~37 TF the two instruction kinds use separate pipes.
template <int NACC>
__global__ void mixed_loop(double* out, int iters, int dfma_iters, double seed) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  if (((warp >> 2) & 1) == 0) {  // warps 0-3, 8-11: DMMA; every SMSP (warp % 4) gets both kinds
    double a = seed + threadIdx.x, b = seed * 0.5 + threadIdx.x;
    double c[NACC][2];
#pragma unroll
    for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < NACC; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  } else {
    double x[NACC];
    double a = seed + threadIdx.x * 1e-9, b = 1.0 - 1e-12;
#pragma unroll
    for (int i = 0; i < NACC; ++i) x[i] = i;
    for (int it = 0; it < dfma_iters; ++it) {
#pragma unroll
      for (int i = 0; i < NACC; ++i) x[i] = fma(x[i], b, a);
    }
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += x[i];
  }
  if (s == 1.2345) out[0] = s;
}

int main() {
  double* d; CK(cudaMalloc(&d, 8));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  printf("device %s sms %d\n", prop.name, sms);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {4, 8, 16}) {
    for (int bpsm : {1, 2, 4}) {
      int threads = warps * 32, blocks = sms * bpsm;
      int iters = 20000;
      dmma_loop<16><<<blocks, threads>>>(d, 10, 1.0);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) dmma_loop<16><<<blocks, threads>>>(d, iters, 1.0);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 5.0 * blocks * warps * (double)iters * 16 * 512.0;
      printf("DMMA m8n8k4   warps/blk %2d blk/sm %d : %.2f TFLOP/s\n", warps, bpsm, flops / ms / 1e9);
    }
  }
  for (int warps : {4, 8, 16}) {
    int threads = warps * 32, blocks = sms * 2;
    int iters = 5000;
    dmma16_loop<4><<<blocks, threads>>>(d, 10, 1.0);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) dmma16_loop<4><<<blocks, threads>>>(d, iters, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 5.0 * blocks * warps * (double)iters * 4 * (16 * 8 * 16 * 2.0);
    printf("DMMA m16n8k16 warps/blk %2d blk/sm 2 : %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  for (int warps : {8, 16, 32}) {
    int threads = warps * 32, blocks = sms * 2;
    int iters = 20000;
    dfma_loop<16><<<blocks, threads>>>(d, 10, 1.0);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) dfma_loop<16><<<blocks, threads>>>(d, iters, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 5.0 * blocks * threads * (double)iters * 16 * 2.0;
    printf("DFMA          warps/blk %2d blk/sm 2 : %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  // mixed: half the warps DMMA, half DFMA; time each kind alone (the other
  // half idle) and together
  for (int ratio : {0, 8, 16, 32}) {
    int threads = 512, blocks = sms * 2, iters = 20000;
    int dfi = iters * ratio / 16;  // DFMA iterations (16 FMAs each) per DMMA iteration count
    mixed_loop<16><<<blocks, threads>>>(d, 10, 10, 1.0);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r) mixed_loop<16><<<blocks, threads>>>(d, iters, dfi, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fd = 3.0 * blocks * 8 * (double)iters * 16 * 512.0;
    double ff = 3.0 * blocks * 8 * 32 * (double)dfi * 16 * 2.0;
    printf("MIXED dfma/dmma iters %2d/16: DMMA %.2f + DFMA %.2f = %.2f TFLOP/s (%.3f ms)\n", ratio, fd / ms / 1e9,
           ff / ms / 1e9, (fd + ff) / ms / 1e9, ms / 3);
  }
  // sustained DMMA for ~4 s
  {
    int threads = 256, blocks = sms * 2, iters = 200000;
    cudaEventRecord(e0);
    int reps = 0; float ms = 0;
    while (ms < 4000.f) {
      dmma_loop<16><<<blocks, threads>>>(d, iters, 1.0); ++reps;
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    }
    double flops = (double)reps * blocks * 8 * (double)iters * 16 * 512.0;
    printf("DMMA sustained (%.1f s): %.2f TFLOP/s\n", ms / 1000, flops / ms / 1e9);
  }
  return 0;
}
