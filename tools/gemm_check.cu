// Standalone correctness probe for the NN/TN DMMA GEMM kernels on awkward
// shapes (partial tiles, K not a multiple of 16), output prefilled with NaN,
// compared against a CPU GEMM.  Debugging tool:  nvcc ... -o gemm_check && ./gemm_check
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2604_11558_b200/csrc/gemm.cuh"

using namespace cg;

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeFn enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return (EncodeFn)p;
}
static void mk(CUtensorMap* m, const void* base, int rank, const uint64_t* d, const uint64_t* s, const uint32_t* b,
               bool swz) {
  cuuint64_t gd[5], gs[4];
  cuuint32_t bx[5], es[5];
  for (int i = 0; i < rank; ++i) gd[i] = d[i], bx[i] = b[i], es[i] = 1;
  for (int i = 0; i < rank - 1; ++i) gs[i] = s[i];
  CUresult r = enc()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, (void*)base, gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) printf("encode failed %d\n", (int)r);
}

// NN middle mode: Y[f,s](M x N) = L(M x K) . X[f,s](K x N), L stored transposed [K][Mp]
template <int BM, int BN, int ST, int MINB, int EPI = EPI_STORE>
int run_nn(int M, int N, int K, int nslab, int nfield, int reps) {
  const int Mp = (M + 1) & ~1;
  std::vector<double> LT((size_t)K * Mp, 0.0), X((size_t)nfield * nslab * K * N), Y((size_t)nfield * nslab * M * N);
  srand(7);
  for (auto& v : LT) v = rand() / (double)RAND_MAX - 0.5;
  for (auto& v : X) v = rand() / (double)RAND_MAX - 0.5;
  double *dLT, *dX, *dY;
  cudaMalloc(&dLT, LT.size() * 8);
  cudaMalloc(&dX, X.size() * 8);
  cudaMalloc(&dY, Y.size() * 8);
  cudaMemcpy(dLT, LT.data(), LT.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dX, X.data(), X.size() * 8, cudaMemcpyHostToDevice);
  CUtensorMap ma, mb, mo;
  {
    uint64_t d[3] = {(uint64_t)M, (uint64_t)K, 1}, s[2] = {(uint64_t)Mp * 8, (uint64_t)K * Mp * 8};
    uint32_t b[3] = {16, 16, 1};
    mk(&ma, dLT, 3, d, s, b, true);
  }
  {
    uint64_t d[4] = {(uint64_t)N, (uint64_t)K, (uint64_t)nslab, (uint64_t)nfield};
    uint64_t s[3] = {(uint64_t)N * 8, (uint64_t)K * N * 8, (uint64_t)nslab * K * N * 8};
    uint32_t b[4] = {16, 16, 1, 1};
    mk(&mb, dX, 4, d, s, b, true);
  }
  {
    uint64_t d[4] = {(uint64_t)N, (uint64_t)M, (uint64_t)nslab, (uint64_t)nfield};
    uint64_t s[3] = {(uint64_t)N * 8, (uint64_t)M * N * 8, (uint64_t)nslab * M * N * 8};
    uint32_t b[4] = {(uint32_t)BN, (uint32_t)BM, 1, 1};
    mk(&mo, dY, 4, d, s, b, false);
  }
  GemmParams p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.nslab = nslab;
  p.ncomp = 1;
  p.nbatch = nfield * nslab;
  p.tiles_m = (M + BM - 1) / BM;
  p.tiles_n = (N + BN - 1) / BN;
  // phi1-like table Phi[f % ncomp][s][m][n] (ncomp = 1)
  std::vector<double> PH((size_t)nslab * M * N);
  for (auto& v : PH) v = 0.5 + rand() / (double)RAND_MAX;
  double* dPH;
  cudaMalloc(&dPH, PH.size() * 8);
  cudaMemcpy(dPH, PH.data(), PH.size() * 8, cudaMemcpyHostToDevice);
  p.phi = dPH;
  p.phi_c = (long long)nslab * M * N;
  p.phi_s = (long long)M * N;
  p.phi_m = N;
  p.phi_n = 1;
  p.phi_rdiv = 1;
  auto kern = gemm_f64_kernel<VAR_NN, BM, BN, 32, 32, ST, EPI, MINB>;
  constexpr int smem = gemm_smem_bytes<BM, BN, ST>();
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int per_sm = 0;
  constexpr int threads = (BM / 32) * (BN / 32) * 32 + 32;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  const int tiles = p.nbatch * p.tiles_m * p.tiles_n;
  const int grid = tiles < per_sm * 148 ? tiles : per_sm * 148;
  // CPU reference
  std::vector<double> ref(Y.size());
  for (int f = 0; f < nfield; ++f)
    for (int s = 0; s < nslab; ++s)
      for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
          double acc = 0;
          for (int k = 0; k < K; ++k) acc += LT[(size_t)k * Mp + m] * X[(((size_t)f * nslab + s) * K + k) * N + n];
          if (EPI == EPI_PHI) acc *= PH[((size_t)s * M + m) * N + n];
          ref[(((size_t)f * nslab + s) * M + m) * N + n] = acc;
        }
  int bad_reps = 0;
  for (int r = 0; r < reps; ++r) {
    std::vector<double> nanfill(Y.size(), NAN);
    cudaMemcpy(dY, nanfill.data(), Y.size() * 8, cudaMemcpyHostToDevice);
    kern<<<grid, threads, smem>>>(ma, mb, mo, mo, p);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) {
      printf("cuda error %s\n", cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(Y.data(), dY, Y.size() * 8, cudaMemcpyDeviceToHost);
    long bad = 0;
    int shown = 0;
    for (size_t i = 0; i < Y.size(); ++i) {
      const double err = fabs(Y[i] - ref[i]);
      if (!(err <= 1e-12 * (1 + fabs(ref[i])))) {
        ++bad;
        if (shown < 5) {
          size_t q = i;
          const int n = q % N;
          q /= N;
          const int m = q % M;
          q /= M;
          const int s = q % nslab;
          const int f = (int)(q / nslab);
          printf("   mismatch f=%d s=%d m=%d n=%d got %g want %g\n", f, s, m, n, Y[i], ref[i]);
          ++shown;
        }
      }
    }
    if (bad) {
      ++bad_reps;
      printf("  rep %d: %ld mismatches\n", r, bad);
    }
  }
  printf("EPI=%d NN BM=%d BN=%d ST=%d MINB=%d M=%d N=%d K=%d nslab=%d nfield=%d grid=%d tiles=%d: %d/%d bad reps\n", EPI, BM, BN,
         ST, MINB, M, N, K, nslab, nfield, grid, tiles, bad_reps, reps);
  cudaFree(dLT);
  cudaFree(dX);
  cudaFree(dY);
  return bad_reps;
}

// chain: Y = NN(X) then Z = NN(Y), both cfg 64x64x4 MINB2 vs CPU: catches a
// kernel reading what the previous kernel wrote through TMA stores
int chain(int M, int K, int N, int nslab, int nfield, int reps) {
  // square operators (M == K) so the chain composes: Z = L2 (L1 X)
  const int Mp = (M + 1) & ~1;
  std::vector<double> L1((size_t)K * Mp), L2((size_t)K * Mp), X((size_t)nfield * nslab * K * N);
  srand(11);
  for (auto& v : L1) v = rand() / (double)RAND_MAX - 0.5;
  for (auto& v : L2) v = rand() / (double)RAND_MAX - 0.5;
  for (auto& v : X) v = rand() / (double)RAND_MAX - 0.5;
  double *dL1, *dL2, *dX, *dY, *dZ;
  cudaMalloc(&dL1, L1.size() * 8);
  cudaMalloc(&dL2, L2.size() * 8);
  cudaMalloc(&dX, X.size() * 8);
  cudaMalloc(&dY, X.size() * 8);
  cudaMalloc(&dZ, X.size() * 8);
  cudaMemcpy(dL1, L1.data(), L1.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dL2, L2.data(), L2.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dX, X.data(), X.size() * 8, cudaMemcpyHostToDevice);
  auto mapsA = [&](CUtensorMap* m, double* L) {
    uint64_t d[3] = {(uint64_t)M, (uint64_t)K, 1}, s[2] = {(uint64_t)Mp * 8, (uint64_t)K * Mp * 8};
    uint32_t b[3] = {16, 16, 1};
    mk(m, L, 3, d, s, b, true);
  };
  auto mapsB = [&](CUtensorMap* m, double* src) {
    uint64_t d[4] = {(uint64_t)N, (uint64_t)K, (uint64_t)nslab, (uint64_t)nfield};
    uint64_t s[3] = {(uint64_t)N * 8, (uint64_t)K * N * 8, (uint64_t)nslab * K * N * 8};
    uint32_t b[4] = {16, 16, 1, 1};
    mk(m, src, 4, d, s, b, true);
  };
  auto mapsO = [&](CUtensorMap* m, double* dst) {
    uint64_t d[4] = {(uint64_t)N, (uint64_t)M, (uint64_t)nslab, (uint64_t)nfield};
    uint64_t s[3] = {(uint64_t)N * 8, (uint64_t)M * N * 8, (uint64_t)nslab * M * N * 8};
    uint32_t b[4] = {64, 64, 1, 1};
    mk(m, dst, 4, d, s, b, false);
  };
  CUtensorMap a1, a2, b1, b2, o1, o2;
  mapsA(&a1, dL1);
  mapsA(&a2, dL2);
  mapsB(&b1, dX);
  mapsB(&b2, dY);
  mapsO(&o1, dY);
  mapsO(&o2, dZ);
  GemmParams p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.nslab = nslab;
  p.ncomp = 1;
  p.nbatch = nfield * nslab;
  p.tiles_m = (M + 63) / 64;
  p.tiles_n = (N + 63) / 64;
  auto kern = gemm_f64_kernel<VAR_NN, 64, 64, 32, 32, 4, EPI_STORE, 2>;
  constexpr int smem = gemm_smem_bytes<64, 64, 4>();
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int tiles = p.nbatch * p.tiles_m * p.tiles_n;
  const int grid = tiles < 296 ? tiles : 296;
  // CPU
  std::vector<double> Y(X.size()), Z(X.size());
  auto cpu = [&](const std::vector<double>& L, const std::vector<double>& in, std::vector<double>& out) {
    for (int f = 0; f < nfield; ++f)
      for (int s = 0; s < nslab; ++s)
        for (int m = 0; m < M; ++m)
          for (int n = 0; n < N; ++n) {
            double acc = 0;
            for (int k = 0; k < K; ++k) acc += L[(size_t)k * Mp + m] * in[(((size_t)f * nslab + s) * K + k) * N + n];
            out[(((size_t)f * nslab + s) * M + m) * N + n] = acc;
          }
  };
  cpu(L1, X, Y);
  cpu(L2, Y, Z);
  int badreps = 0;
  std::vector<double> G(X.size());
  for (int r = 0; r < reps; ++r) {
    std::vector<double> nanfill(X.size(), NAN);
    cudaMemcpy(dY, nanfill.data(), X.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dZ, nanfill.data(), X.size() * 8, cudaMemcpyHostToDevice);
    kern<<<grid, 160, smem>>>(a1, b1, o1, o1, p);
    kern<<<grid, 160, smem>>>(a2, b2, o2, o2, p);
    cudaDeviceSynchronize();
    cudaMemcpy(G.data(), dZ, X.size() * 8, cudaMemcpyDeviceToHost);
    long bad = 0;
    for (size_t i = 0; i < G.size(); ++i)
      if (!(fabs(G[i] - Z[i]) <= 1e-11 * (1 + fabs(Z[i])))) ++bad;
    if (bad) ++badreps;
    if (bad) printf("  chain rep %d: %ld mismatches\n", r, bad);
  }
  printf("chain M=K=%d N=%d nslab=%d: %d/%d bad reps\n", M, N, nslab, badreps, reps);
  return badreps;
}

int main() {
  chain(96, 96, 100, 100, 2, 10);
  chain(100, 100, 100, 100, 2, 10);
  chain(128, 128, 128, 64, 2, 10);
  run_nn<64, 64, 4, 2, EPI_PHI>(96, 100, 96, 100, 2, 5);
  run_nn<64, 64, 4, 2, EPI_PHI>(100, 100, 100, 100, 2, 5);
  run_nn<64, 64, 6, 3, EPI_PHI>(96, 100, 96, 100, 2, 5);
  run_nn<128, 64, 4, 1, EPI_PHI>(96, 100, 96, 100, 2, 5);
  run_nn<64, 64, 4, 2, EPI_PHI>(128, 128, 128, 64, 2, 5);
  run_nn<64, 64, 4, 2>(96, 100, 96, 100, 2, 5);
  run_nn<64, 64, 6, 3>(96, 100, 96, 100, 2, 5);
  run_nn<128, 64, 4, 1>(96, 100, 96, 100, 2, 5);
  run_nn<64, 64, 4, 2>(96, 96, 96, 100, 2, 5);
  run_nn<64, 64, 4, 2>(100, 100, 100, 100, 2, 5);
  run_nn<64, 64, 4, 2>(128, 128, 128, 64, 2, 5);
  return 0;
}
