// libcurvigpu: plan construction, per-geometry step schedules, CUDA-graph
// time loop and the C ABI declared in include/curvigpu.h.
//
// One step of the reference (run_simulation loop body, integrators.py:413-427)
// becomes:
//   fbuild            F = coeff*M W + g(W+lift)      (HBM-bound stencil pass)
//   2..5 GEMM stages  the geometry's mu-mode chain    (DMMA, TMA-fed)
//                     (integrators.py:202-236), the last one fused with
//                     W + tau*T and the divergence guard
// and the whole sequence is captured once into a CUDA graph and replayed.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "curvigpu.h"
#include "errors.h"
#include "gemm.cuh"
#include "resident.cuh"
#include "stencil.cuh"
#include "thetafft.cuh"
#include "fused_disk.cuh"
#include "cluster_disk.cuh"
#include "coupling.cuh"
#include "diagnostics.cuh"

using namespace cg;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(x)                                                                         \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess)                                                                  \
      return fail(CG_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_) + " @" + \
                                std::to_string(__LINE__));                                  \
  } while (0)

}  // namespace

// other translation units (setup.cu) report through the same thread-local message
int cg_internal_fail(int code, const char* msg) { return fail(code, msg ? msg : ""); }

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// Launch a step-chain kernel with programmatic dependent launch (common.cuh:
// every such kernel calls pdl_wait() before touching step data), so its
// launch and prologue overlap the previous kernel's tail.  CURVIGPU_NO_PDL=1
// launches plainly (measurement).
bool pdl_enabled() {
  static const bool on = getenv("CURVIGPU_NO_PDL") == nullptr;
  return on;
}

template <typename... KArgs, typename... Args>
int launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
  return CG_OK;
}

// fp64 tensor map, 128B swizzle, zero fill; dims innermost first, strides in bytes.
int make_map(CUtensorMap* map, const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
             const uint32_t* box, bool swizzle = true) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(CG_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t gd[5], gs[4];
  cuuint32_t bx[5], es[5];
  for (int i = 0; i < rank; ++i) {
    gd[i] = dims[i];
    bx[i] = box[i];
    es[i] = 1;
  }
  for (int i = 0; i < rank - 1; ++i) gs[i] = strides_bytes[i];
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<void*>(base), gd, gs, bx, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CG_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return CG_OK;
}

// ---------------------------------------------------------------------------
// GEMM tile configurations and dispatch
// ---------------------------------------------------------------------------

struct TileCfg {
  int BM, BN;
};
constexpr int kNumCfg = 20;
constexpr int kChainCfg = 14;  // EPI_CHAIN only: 32 rows x all (<= 128) columns, 8 warps of 16x32
constexpr int kChainCfg16 = 15;  // EPI_CHAIN, 16-row tiles on 4 warps at 3 CTAs/SM (CURVIGPU_CHAIN_CFG=15)
constexpr int kRaggedCfg = 16;   // cfg 12 for NN stages with M or K off the tile grid (zero-block skips)
constexpr int kWideCfg = 17;     // 16 x 128 tiles (4 warps of 16x32, 3 CTAs/SM) for TN stages with N = 128
// NN stages whose operator has at most 112 rows (n = 100): one m tile of 112 x 32 on two consumer warps of
// 112 x 16 (up to 14 live 8-row blocks each: 16 fragment loads per 28 DMMAs instead of 4 per 4, no quarter-empty
// last m tile).  18: 4-stage ring, 2 CTAs/SM; 19: 2-stage ring, 3 CTAs/SM.
constexpr int kTallCfg = 18;
constexpr int kTallCfg3 = 19;
// 7, 8: the 64x64 configuration split-K over clusters of 2 / 4 CTAs
// 9, 10: 64x64 tiles on 8 consumer warps (32x16 / 16x32 warp tiles); 11: 10 split-K over 2-CTA clusters
// 12: 32x32 tiles on 4 warps of 16x16 (stages with very few 64x64 tiles); 13: 12 split-K over 2-CTA clusters
constexpr TileCfg kCfgs[kNumCfg] = {{128, 64}, {64, 128}, {64, 64}, {128, 64}, {64, 128}, {128, 128}, {64, 64},
                                    {64, 64}, {64, 64}, {64, 64}, {64, 64}, {64, 64},
                                    {32, 32}, {32, 32}, {32, 128}, {16, 128}, {32, 32}, {16, 128}, {112, 32}, {112, 32}};

// BM, BN, warp tile, stages; 32x32 warp tiles keep the accumulators +
// fragments under ~160 registers without spills.
// (BM, BN, warp tile WM x WN, stages, min CTAs per SM)
#define CFG0 128, 64, 32, 32, 4, 1
#define CFG1 64, 128, 32, 32, 4, 1
#define CFG2 64, 64, 32, 32, 4, 2
#define CFG3 128, 64, 32, 32, 4, 2
#define CFG4 64, 128, 32, 32, 4, 2
#define CFG5 128, 128, 32, 32, 3, 1
#define CFG6 64, 64, 32, 32, 6, 3
#define CFG9 64, 64, 32, 16, 4, 2
#define CFG10 64, 64, 16, 32, 4, 2
// 32x32 tiles: 4-stage ring at FIVE CTAs per SM (41 KB, 70 registers): 20 consumer warps per SM instead of 16 --
// ball rho 21.2 -> 19.9 us, its DMMA-theta stages 30.6 / 27.2 -> 28.7 / 25.4 us, cylinder rho 13.1 -> 12.9 us;
// six CTAs (3 stages, 64 registers) measured 21.4 us (profiles/r02_cfg12_occupancy.txt)
#ifndef CG_CFG12_ST
#define CG_CFG12_ST 4
#endif
#ifndef CG_CFG12_MINB
#define CG_CFG12_MINB 5
#endif
#define CFG12 32, 32, 16, 16, CG_CFG12_ST, CG_CFG12_MINB
#define CFG14 32, 128, 16, 32, 3, 2
#define CFG15 16, 128, 16, 32, 3, 3
#define CFG18 112, 32, 56, 16, 4, 2
#define CFG19 112, 32, 56, 16, 2, 3

// configure_only: set the dynamic shared memory opt-in (done at plan
// creation, never inside a stream capture).  KS > 1 launches clusters of KS
// CTAs that split each tile's k range (gemm.cuh).
template <int VAR, int BM, int BN, int WM, int WN, int ST, int MINB, int EPI, int KS = 1, bool RAG = false>
int launch_gemm_t(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mw, const CUtensorMap& mo,
                  const GemmParams& p, cudaStream_t stream, bool configure_only) {
  auto kern = gemm_f64_kernel<VAR, BM, BN, WM, WN, ST, EPI, MINB, KS, RAG>;
  constexpr int smem = gemm_smem_bytes<BM, BN, ST>();
  constexpr int threads = (BM / WM) * (BN / WN) * 32 + 32;
  static int resident = 0;  // CTAs (KS = 1) or clusters (KS > 1) of this instantiation that fit at once
  static int pad = 0;  // debugging: CURVIGPU_SMEM_PAD extra bytes per CTA (lowers occupancy)
  if (configure_only) {
    const char* ps = getenv("CURVIGPU_SMEM_PAD");
    pad = ps ? atoi(ps) : 0;
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem + pad));
    // Measurement knob only: CURVIGPU_MAX_CARVEOUT=1 requests the full
    // shared-memory carveout (tried for co-residing the front with the GEMM;
    // it made the stage-ring race of profiles/r01_partial_tile_race.md, since
    // fixed, far more frequent).
    if (getenv("CURVIGPU_MAX_CARVEOUT"))
      CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
    int dev = 0, sms = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (KS == 1) {
      int per_sm = 0;
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem + pad));
      if (const char* cap = getenv("CURVIGPU_GEMM_CPS")) per_sm = std::min(per_sm, std::max(1, atoi(cap)));
      resident = (per_sm > 0 ? per_sm : 1) * sms;
    } else {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = KS;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(KS * sms, 1, 1);
      cfg.blockDim = dim3(threads, 1, 1);
      cfg.dynamicSmemBytes = smem + pad;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int ncl = 0;
      CUDA_TRY(cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg));
      resident = ncl > 0 ? ncl : 1;
    }
    return CG_OK;
  }
  const long long tiles = (long long)p.nbatch * p.tiles_m * p.tiles_n;
  if (tiles <= 0) return CG_OK;
  if (tiles > INT_MAX) return fail(CG_EUNSUPPORTED, "grid too large");
  // persistent grid: at most one wave of resident CTAs (clusters), each looping over tiles
  long long units = (resident > 0 && tiles > resident) ? resident : tiles;
  if (getenv("CURVIGPU_NOPERSIST")) units = tiles;
  if (KS == 1) {
    int rc = launch_pdl(kern, dim3((unsigned)units), dim3(threads), smem + pad, stream, ma, mb, mw, mo, p);
    if (rc) return rc;
  } else {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = KS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3((unsigned)(units * KS), 1, 1);
    cfg.blockDim = dim3(threads, 1, 1);
    cfg.dynamicSmemBytes = smem + pad;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, ma, mb, mw, mo, p));
  }
  CUDA_TRY(cudaGetLastError());
  return CG_OK;
}

struct Maps {
  CUtensorMap a, b, w, o;
};

template <int VAR, int EPI>
int launch_gemm_cfg(int cfg, const Maps& m, const GemmParams& p, cudaStream_t stream, bool conf) {
  switch (cfg) {
    case 0: return launch_gemm_t<VAR, CFG0, EPI>(m.a, m.b, m.w, m.o, p, stream, conf);
    case 1: return launch_gemm_t<VAR, CFG1, EPI>(m.a, m.b, m.w, m.o, p, stream, conf);
    case 2: return launch_gemm_t<VAR, CFG2, EPI>(m.a, m.b, m.w, m.o, p, stream, conf);
    case 3: return launch_gemm_t<VAR, CFG3, EPI>(m.a, m.b, m.w, m.o, p, stream, conf);
    case 4: return launch_gemm_t<VAR, CFG4, EPI>(m.a, m.b, m.w, m.o, p, stream, conf);
    case 5: return launch_gemm_t<VAR, CFG5, EPI>(m.a, m.b, m.w, m.o, p, stream, conf);
    case 7: return launch_gemm_t<VAR, CFG2, EPI, 2>(m.a, m.b, m.w, m.o, p, stream, conf);
    case 8: return launch_gemm_t<VAR, CFG2, EPI, 4>(m.a, m.b, m.w, m.o, p, stream, conf);
    case 9: return launch_gemm_t<VAR, CFG9, EPI>(m.a, m.b, m.w, m.o, p, stream, conf);
    case 10: return launch_gemm_t<VAR, CFG10, EPI>(m.a, m.b, m.w, m.o, p, stream, conf);
    case 11: return launch_gemm_t<VAR, CFG10, EPI, 2>(m.a, m.b, m.w, m.o, p, stream, conf);
    case 12: return launch_gemm_t<VAR, CFG12, EPI>(m.a, m.b, m.w, m.o, p, stream, conf);
    case 13: return launch_gemm_t<VAR, CFG12, EPI, 2>(m.a, m.b, m.w, m.o, p, stream, conf);
    case 16: return launch_gemm_t<VAR, CFG12, EPI, 1, VAR == VAR_NN>(m.a, m.b, m.w, m.o, p, stream, conf);
    case 17: return launch_gemm_t<VAR, CFG15, EPI>(m.a, m.b, m.w, m.o, p, stream, conf);
    case kTallCfg:
      if constexpr (VAR == VAR_NN) return launch_gemm_t<VAR, CFG18, EPI, 1, true>(m.a, m.b, m.w, m.o, p, stream, conf);
      return fail(CG_EINVAL, "tall tiles are an NN configuration");
    case kTallCfg3:
      if constexpr (VAR == VAR_NN) return launch_gemm_t<VAR, CFG19, EPI, 1, true>(m.a, m.b, m.w, m.o, p, stream, conf);
      return fail(CG_EINVAL, "tall tiles are an NN configuration");
    default: return launch_gemm_t<VAR, CFG6, EPI>(m.a, m.b, m.w, m.o, p, stream, conf);
  }
}

int launch_gemm(int var, int epi, int cfg, const Maps& m, const GemmParams& p, cudaStream_t s, bool conf = false) {
  if (epi == EPI_CHAIN) {  // m.w carries the second operator's map
    if (var != VAR_TN || (cfg != kChainCfg && cfg != kChainCfg16))
      return fail(CG_EINVAL, "chained stage needs a TN chain tile");
    if (cfg == kChainCfg16) return launch_gemm_t<VAR_TN, CFG15, EPI_CHAIN>(m.a, m.b, m.w, m.o, p, s, conf);
    return launch_gemm_t<VAR_TN, CFG14, EPI_CHAIN>(m.a, m.b, m.w, m.o, p, s, conf);
  }
  if (var == VAR_TN) {
    if (epi == EPI_STORE) return launch_gemm_cfg<VAR_TN, EPI_STORE>(cfg, m, p, s, conf);
    if (epi == EPI_PHI) return launch_gemm_cfg<VAR_TN, EPI_PHI>(cfg, m, p, s, conf);
    return launch_gemm_cfg<VAR_TN, EPI_AXPY>(cfg, m, p, s, conf);
  }
  if (epi == EPI_STORE) return launch_gemm_cfg<VAR_NN, EPI_STORE>(cfg, m, p, s, conf);
  if (epi == EPI_PHI) return launch_gemm_cfg<VAR_NN, EPI_PHI>(cfg, m, p, s, conf);
  return launch_gemm_cfg<VAR_NN, EPI_AXPY>(cfg, m, p, s, conf);
}

__global__ void set_step_kernel(int* step, int value) { *step = value; }

__global__ void hadamard_kernel(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out,
                                long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = a[i] * b[i];
}

// rows of nl values from row stride lds to row stride ldd (padded <-> caller layout)
__global__ void repack_kernel(const double* __restrict__ src, int lds, double* __restrict__ dst, int ldd,
                              long long rows, int nl) {
  const long long total = rows * nl;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long r = t / nl;
    const int k = (int)(t - r * nl);
    dst[r * ldd + k] = src[r * lds + k];
  }
}

template <int GEOM, int KIN, int R2>
int launch_fbuild_r(const StencilParams& p, cudaStream_t s, bool configure_only) {
  using S = FbuildShape<GEOM, R2>;
  if (configure_only) {  // at plan creation, never under stream capture
    CUDA_TRY(cudaFuncSetAttribute(fbuild_rows_kernel<GEOM, KIN, R2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  200 * 1024));
    if constexpr (GEOM == 2)
      CUDA_TRY(cudaFuncSetAttribute(fbuild_rows_kernel<GEOM, KIN, R2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    200 * 1024));
    return CG_OK;
  }
  if (p.batch > 65535) return fail(CG_EUNSUPPORTED, "batch > 65535 runs per plan");
  const int nl = S::D3 ? p.n3 : p.n2;
  if (nl > 512) return fail(CG_EUNSUPPORTED, "contiguous axis longer than 512");
  const size_t smem = (size_t)(KIN == KIN_EXTERNAL ? 1 : 2) * S::ROWS * nl * sizeof(double);
  if (smem > 200 * 1024) return fail(CG_EUNSUPPORTED, "F-build tile exceeds shared memory");
  const dim3 grid((unsigned)((p.n1 + S::RB - 1) / S::RB), S::D3 ? (unsigned)((p.n2 + S::JB - 1) / S::JB) : 1u,
                  (unsigned)p.batch);
  const unsigned threads = (unsigned)((nl + 31) / 32 * 32);
  int rc;
  if (GEOM == 2 && threads <= 128)  // the cylinder measured 9.7 us wide, 9.8 us narrow
    rc = launch_pdl(fbuild_rows_kernel<GEOM, KIN, R2, GEOM == 2>, grid, dim3(threads), smem, s, p);
  else
    rc = launch_pdl(fbuild_rows_kernel<GEOM, KIN, R2, false>, grid, dim3(threads), smem, s, p);
  if (rc) return rc;
  CUDA_TRY(cudaGetLastError());
  return CG_OK;
}

// 2-D geometries: 4-row CTAs when the 8-row grid would not give every SM two CTAs
template <int GEOM, int KIN>
int launch_fbuild_t(const StencilParams& p, cudaStream_t s, bool configure_only) {
  if constexpr (GEOM >= 2) {
    return launch_fbuild_r<GEOM, KIN, 8>(p, s, configure_only);
  } else {
    if (configure_only) {
      if (int rc = launch_fbuild_r<GEOM, KIN, 4>(p, s, true)) return rc;
      return launch_fbuild_r<GEOM, KIN, 8>(p, s, true);
    }
    const long long ctas8 = (long long)((p.n1 + 7) / 8) * p.batch;
    if (ctas8 < 2LL * 148) return launch_fbuild_r<GEOM, KIN, 4>(p, s, false);
    return launch_fbuild_r<GEOM, KIN, 8>(p, s, false);
  }
}

template <int GEOM>
int launch_fbuild_g(int kin, const StencilParams& p, cudaStream_t s, bool conf) {
  switch (kin) {
    case KIN_SCHNAKENBERG: return launch_fbuild_t<GEOM, KIN_SCHNAKENBERG>(p, s, conf);
    case KIN_BRUSSELATOR: return launch_fbuild_t<GEOM, KIN_BRUSSELATOR>(p, s, conf);
    case KIN_GRAY_SCOTT: return launch_fbuild_t<GEOM, KIN_GRAY_SCOTT>(p, s, conf);
    case KIN_BVAM_ETA: return launch_fbuild_t<GEOM, KIN_BVAM_ETA>(p, s, conf);
    case KIN_BVAM: return launch_fbuild_t<GEOM, KIN_BVAM>(p, s, conf);
    case KIN_DIB: return launch_fbuild_t<GEOM, KIN_DIB>(p, s, conf);
    default: return launch_fbuild_t<GEOM, KIN_EXTERNAL>(p, s, conf);
  }
}

int launch_fbuild(int geom, int kin, const StencilParams& p, cudaStream_t s, bool conf = false) {
  switch (geom) {
    case CG_DISK: return launch_fbuild_g<0>(kin, p, s, conf);
    case CG_SPHERE: return launch_fbuild_g<1>(kin, p, s, conf);
    case CG_BALL: return launch_fbuild_g<2>(kin, p, s, conf);
    default: return launch_fbuild_g<3>(kin, p, s, conf);
  }
}

// ---------------------------------------------------------------------------
// plan
// ---------------------------------------------------------------------------

enum { BUF_X = 0, BUF_Y = 1, BUF_OUT = 2 };

constexpr int VAR_THETA = 2;  // FFT theta propagator (thetafft.cuh), not a GEMM

struct Stage {
  int var, epi, cfg;
  int M, N, K, nslab;
  int ldr;       // row stride of the contiguous dim of the state views (K for TN, N for NN and the output)
  int src, dst;  // BUF_X / BUF_Y / BUF_OUT
  const double* phi;
  long long phi_c, phi_s;
  int phi_m, phi_n, phi_rdiv;
  CUtensorMap opmap;  // operator operand (B for TN, A for NN)
  CUtensorMap opmap2;  // EPI_CHAIN: the second operator (B2, TN layout)
  // resident-operator kernel (resident.cuh): 8-row blocks of the operator
  // extent (0 = the tiled kernel runs this stage), k steps, padded operator copies
  int res_nb, res_ks;
  const double* rop;
  const double* rop2;
  // VAR_THETA: field = [A][N][Bc], W lines per CTA, Phi_j table, twiddles
  int tA, tBc, tW, tclass_mode, tnclass;
  const double* phif;
  const double* phis;  // pre-scaled, padded rows (ThetaParams::phis)
  int phis_ld;
  const double2* tw;
};

struct GraphEntry {
  double* state;
  int* first_bad;
  cudaGraphExec_t chunk;
};

constexpr int kChunk = 16;  // steps per captured graph (even)

}  // namespace

struct cg_plan {
  int geom, n1, n2, n3, B, C, kin, P;
  int NO = 0;  // operator sets: C (shared by the runs) or B * C (heterogeneous ensemble)
  double tau;
  // Storage layout: the contiguous (last) axis of logical extent nl is stored
  // with row stride ld = even(nl) so every TMA row stride is a multiple of 16
  // bytes.  npts / elems count storage elements, npts_u / elems_u the user's
  // unpadded arrays.  When padded, cg_run / cg_step repack the caller's
  // arrays into S0 (ghost column held at zero, never read by TMA: every map
  // declares the logical extent).
  int nl = 0, ld = 0;
  bool padded = false;
  long long npts, elems, npts_u = 0, elems_u = 0;
  double* S0 = nullptr;
  std::vector<void*> allocs;
  double *coeff = nullptr, *lift = nullptr, *kin_params = nullptr;
  double *rho_b = nullptr, *phi_b = nullptr, *z_b = nullptr, *th = nullptr, *d_rho = nullptr, *d_phi = nullptr;
  double *X = nullptr, *Y = nullptr, *S2 = nullptr;
  bool redzone = false;  // CURVIGPU_REDZONE: guard bands around the workspaces
  struct Guarded {
    uint8_t* raw;
    size_t bytes;  // payload; kRedzone bytes of guard band on each side
  };
  std::vector<Guarded> guarded;
  int* step_dev = nullptr;
  int* scratch_bad = nullptr;
  std::vector<Stage> stages;
  std::vector<GraphEntry> graphs;
  cudaStream_t cap_stream = nullptr;
  // disk + FFT theta + built-in kinetics: F-build and stages[0] (theta) run
  // as one persistent fused kernel (fused_disk.cuh) inside cg_run
  bool fused_front = false;
  int fused_m1 = 0, fused_m2 = 0, fused_nt = 256;
  // small disks (config 1): cg_run advances all its steps in one cluster
  // kernel with the state in the cluster's shared memory (cluster_disk.cuh)
  bool cluster_step = false;
  const double* cluster_rop = nullptr;
};

namespace {

int dev_alloc(cg_plan* p, size_t bytes, void** out) {
  CUDA_TRY(cudaMalloc(out, bytes == 0 ? 16 : bytes));
  p->allocs.push_back(*out);
  return CG_OK;
}

// X, Y, S2 (and S0 for padded storage), each the state's size: allocated by
// the first entry point that touches them.  Not capture-safe by design: the
// first call on a plan must not be made inside a caller's stream capture.
// With CURVIGPU_REDZONE=1 in the environment every workspace gets a
// kRedzone-byte guard band on both sides, filled with kRedzoneByte; a kernel
// writing past a buffer lands in a band and cg_plan_check_redzones reports it
// (our own bounds check: compute-sanitizer is not available on the GPU pool).
constexpr size_t kRedzone = 1 << 20;
constexpr unsigned char kRedzoneByte = 0xA5;

int ws_alloc(cg_plan* p, size_t bytes, double** out) {
  if (!p->redzone) return dev_alloc(p, bytes, reinterpret_cast<void**>(out));
  uint8_t* raw = nullptr;
  int rc = dev_alloc(p, bytes + 2 * kRedzone, reinterpret_cast<void**>(&raw));
  if (rc) return rc;
  CUDA_TRY(cudaMemset(raw, kRedzoneByte, bytes + 2 * kRedzone));
  CUDA_TRY(cudaMemset(raw + kRedzone, 0, bytes));
  *out = reinterpret_cast<double*>(raw + kRedzone);
  p->guarded.push_back({raw, bytes});
  return CG_OK;
}

int ensure_workspace(cg_plan* p) {
  if (p->X) return CG_OK;
  const size_t bytes = (size_t)p->elems * sizeof(double);
  int rc;
  double *X = nullptr, *Y = nullptr, *S2 = nullptr, *S0 = nullptr;
  if ((rc = ws_alloc(p, bytes, &X))) return rc;
  if ((rc = ws_alloc(p, bytes, &Y))) return rc;
  if ((rc = ws_alloc(p, bytes, &S2))) return rc;
  if (p->padded) {
    if ((rc = ws_alloc(p, bytes, &S0))) return rc;
    for (double* buf : {X, Y, S2, S0}) CUDA_TRY(cudaMemset(buf, 0, bytes));
  }
  if (p->padded || p->redzone) CUDA_TRY(cudaDeviceSynchronize());
  p->Y = Y;
  p->S2 = S2;
  p->S0 = S0;
  p->X = X;
  return CG_OK;
}

int upload(cg_plan* p, const double* host, size_t count, double** out) {
  if (!host) {
    *out = nullptr;
    return CG_OK;
  }
  int rc = dev_alloc(p, count * sizeof(double), reinterpret_cast<void**>(out));
  if (rc) return rc;
  CUDA_TRY(cudaMemcpy(*out, host, count * sizeof(double), cudaMemcpyHostToDevice));
  return CG_OK;
}

// Operator for a TN stage, stored [C][N][Kp] with Kp = even(K): op[c][n][k] = src(c, n, k).
// Operator for a NN stage, stored [C][K][Mp]: op[c][k][m] = L_c[m][k].
// `get(c, r, q)` returns L_c[r][q] (row r, col q) of the n x n left matrix.
template <typename Get>
int upload_operator(cg_plan* p, int var, int n, Get get, double** out, CUtensorMap* map, int box_rows) {
  const int np = (n + 1) & ~1;
  std::vector<double> h((size_t)p->NO * n * np, 0.0);
  for (int c = 0; c < p->NO; ++c)
    for (int r = 0; r < n; ++r)
      for (int q = 0; q < n; ++q) {
        // TN: B[n_out = r][k = q] = L[r][q];  NN: A^T[k = q][m = r] = L[r][q]
        if (var == VAR_TN)
          h[((size_t)c * n + r) * np + q] = get(c, r, q);
        else
          h[((size_t)c * n + q) * np + r] = get(c, r, q);
      }
  int rc = upload(p, h.data(), h.size(), out);
  if (rc) return rc;
  const uint64_t dims[3] = {(uint64_t)n, (uint64_t)n, (uint64_t)p->NO};
  const uint64_t strides[2] = {(uint64_t)np * 8, (uint64_t)n * np * 8};
  const uint32_t box[3] = {16, (uint32_t)box_rows, 1};
  return make_map(map, *out, 3, dims, strides, box);
}

// ---- resident-operator stages (resident.cuh) ----
template <int VAR, int EPI, int NB, int KSTEPS>
int launch_resident_t(const ResParams& rp, cudaStream_t s, bool conf) {
  auto kern = resident_gemm_kernel<VAR, EPI, NB, KSTEPS>;
  constexpr size_t smem = res_smem_bytes<EPI, NB, KSTEPS>();
  if (conf) {
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    return CG_OK;
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const long long units = (long long)rp.nitems * rp.upi;
  const unsigned blocks = (unsigned)std::min<long long>(sms, (units + kResGroups - 1) / kResGroups);
  return launch_pdl(kern, dim3(blocks), dim3(kResWarps * 32), smem, s, rp);
}

template <int VAR, int EPI>
int launch_resident_s(int nb, const ResParams& rp, cudaStream_t s, bool conf) {
  if (nb == 8) return launch_resident_t<VAR, EPI, 8, 16>(rp, s, conf);
  if (nb == 13) return launch_resident_t<VAR, EPI, 13, 25>(rp, s, conf);
  if constexpr (EPI != EPI_CHAIN) {
    if (nb == 16) return launch_resident_t<VAR, EPI, 16, 32>(rp, s, conf);
  }
  return fail(CG_EUNSUPPORTED, "no resident-operator instantiation for this extent");
}

int launch_resident(int var, int epi, int nb, const ResParams& rp, cudaStream_t s, bool conf = false) {
  if (var == VAR_TN) {
    if (epi == EPI_STORE) return launch_resident_s<VAR_TN, EPI_STORE>(nb, rp, s, conf);
    if (epi == EPI_PHI) return launch_resident_s<VAR_TN, EPI_PHI>(nb, rp, s, conf);
    if (epi == EPI_CHAIN) return launch_resident_s<VAR_TN, EPI_CHAIN>(nb, rp, s, conf);
  } else {
    if (epi == EPI_STORE) return launch_resident_s<VAR_NN, EPI_STORE>(nb, rp, s, conf);
    if (epi == EPI_PHI) return launch_resident_s<VAR_NN, EPI_PHI>(nb, rp, s, conf);
    if (epi == EPI_AXPY) return launch_resident_s<VAR_NN, EPI_AXPY>(nb, rp, s, conf);
  }
  return fail(CG_EUNSUPPORTED, "no resident-operator kernel for this stage");
}

// 8-row blocks of the resident instantiation that fits an n x n operator (0: none)
int resident_blocks(int epi, int n) {
  if (n <= 64) return 8;
  if (n <= 100) return 13;
  if (n <= 128 && epi != EPI_CHAIN) return 16;
  return 0;
}
int resident_ksteps(int nb) { return nb == 8 ? 16 : nb == 13 ? 25 : 32; }

// Should a stage run the resident-operator kernel?  Measured on B200
// (profiles/r02_resident_kernels.txt, tools/kernel_times.py): the ball's
// chained polar pair gains (45.7 -> 35.4 us: its two operators stay resident,
// the intermediate stays on chip and half-strip units balance n = 100), the
// single products do not (ball rho 22.4 vs 21.5 us tiled, cylinder phi1_z 21.4
// vs 21.0, cylinder rho 15.6 vs 13.0, config 5 rho 358 vs 277: one operator
// fragment load per DMMA and X loads that all warps of a sub-partition wait
// for at the same time hold the DMMA pipe at 66 %), so only chained stages take
// it by default.  CURVIGPU_RESIDENT=0 disables it, =1 takes every eligible
// stage (measurement; the parity suite runs in both modes).
bool want_resident(int var, int epi, long long nitems, int M, int N, int K, int n_op) {
  const char* env = getenv("CURVIGPU_RESIDENT");
  if (env && env[0] == '0') return false;
  if (K != n_op || (var == VAR_TN ? N != n_op : M != n_op)) return false;
  if (!resident_blocks(epi, n_op)) return false;
  // CURVIGPU_RESIDENT_CHAIN_ONLY=1 with =1: force the chained stages only (tests at small sizes)
  if (env && env[0] == '1') return epi == EPI_CHAIN || !getenv("CURVIGPU_RESIDENT_CHAIN_ONLY");
  const long long units = nitems * (((var == VAR_TN ? M : N) + 7) / 8);
  return epi == EPI_CHAIN && units >= 2LL * 4 * 148;
}

// zero-padded row-major copy [NO][8 nb][LDS] of the n x n operators L_c[r][q] = get(c, r, q)
template <typename Get>
int upload_resident_operator(cg_plan* p, int n, int nb, Get get, const double** out) {
  const int lds = res_lds(resident_ksteps(nb));
  std::vector<double> h((size_t)p->NO * nb * 8 * lds, 0.0);
  for (int c = 0; c < p->NO; ++c)
    for (int r = 0; r < n; ++r)
      for (int q = 0; q < n; ++q) h[((size_t)c * nb * 8 + r) * lds + q] = get(c, r, q);
  double* d = nullptr;
  int rc = upload(p, h.data(), h.size(), &d);
  *out = d;
  return rc;
}

int pick_cfg(int var, long long nbatch, int M, int N, int K, int stage_index) {
  // measurement override: CURVIGPU_TILE_CFG=<cfg> or "<s0>,<s1>,..." per stage
  if (const char* env = getenv("CURVIGPU_TILE_CFG")) {
    int vals[16], nv = 0;
    for (const char* q = env; *q && nv < 16;) {
      vals[nv++] = atoi(q);
      while (*q && *q != ',') ++q;
      if (*q == ',') ++q;
    }
    const int v = nv == 1 ? vals[0] : (stage_index < nv ? vals[stage_index] : -1);
    if ((v >= 0 && v < kChainCfg) || v == 17) return v;
    if ((v == kTallCfg || v == kTallCfg3) && var == VAR_NN && M <= 112) return v;
  }
  // Measured on B200 with the TMA epilogue (tools/sweep_tiles.py,
  // profiles/r01_tile_sweep_tmaepi.txt): 64x64 tiles, 4-stage ring, 2 CTAs/SM
  // is the best or within 2% of the best for every stage of every BASELINE
  // config (larger epilogue tiles cost occupancy).  Splitting the 64x64 tile
  // over 8 consumer warps (16x32 warp tiles, cfg 10) instead of 4 hides more
  // DMMA/fragment latency: config 5 rho stage 283 -> 277 us, ball stages
  // -7 to -10 %, config 1 5.7 -> 5.1 us (profiles/r01_warp8_sweep.txt).
  // Split-K (each tile's k range over a cluster of 2 CTAs) was the earlier
  // answer to stages with too few tiles (tools/small_gemm_sweep.py,
  // profiles/r01_splitk_sweep.jsonl: the sphere's 64-tile stages 13.7 -> 10.9
  // us; 4-CTA clusters and splits of short k ranges lose to the DSMEM
  // reduction and cluster handshakes; the split-K configurations 7, 8, 11, 13
  // stay selectable through CURVIGPU_TILE_CFG for measurement and are tested,
  // but the 32x32 tiles below now beat them).
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) !=
                                                  cudaSuccess)
      sms = 148;
  }
  // Stages with up to 8 x SMs 64x64 tiles (every stage of configs 1-4) run
  // 32x32 tiles at 4 CTAs/SM instead: 4x the CTAs to spread the work (config
  // 1 rho stage 4.98 -> 2.84 us, sphere stage 0 10.5 -> 7.05 us, faster than
  // the split-K clusters, 10.2 us), and no loss where the 64x64 grid already
  // has 2 waves (cylinder, ball: equal or 2-6 % faster).  Large stages keep
  // 64x64 (config 5: 277 vs 309 us) (profiles/r01_warp8_sweep.txt).
  (void)K;
  const long long tiles = nbatch * ((M + 63) / 64) * ((N + 63) / 64);
  if (tiles > 8LL * sms) return 10;
  // TN stages exactly 128 wide with many rows (the cylinder's phi1_z stage):
  // 16 x 128 tiles, 6 operand rows per 8 DMMAs instead of 4 per 4, 1024
  // tiles in balanced rounds: 21.6 -> 21.1 us.  (NN stages and the sphere's
  // 256-wide stage measured slower with it.)
  if (var == VAR_TN && N == 128 && K % 16 == 0 && M % 16 == 0 && nbatch * (M / 16) >= 2LL * sms) return kWideCfg;
  // NN stages with M or K off the 32 x 16 grid (n = 100) take the
  // zero-block-skipping instantiation: ball rho stage 23.2 -> 21.4 us
  return (var == VAR_NN && (M % 32 != 0 || K % 16 != 0)) ? kRaggedCfg : 12;
}

// Build one GEMM stage: operator L (n x n) via `get`, shapes, epilogue.
template <typename Get>
int add_stage(cg_plan* p, int var, int epi, int M, int N, int K, int nslab, int src, int dst, int n_op, Get get,
              int force_cfg = -1) {
  Stage st{};
  st.var = var;
  st.epi = epi;
  st.M = M;
  st.N = N;
  st.K = K;
  st.nslab = nslab;
  st.src = src;
  st.dst = dst;
  st.phi_rdiv = 1;
  st.ldr = p->ld;
  if (var == VAR_NN && p->n3 > 1 && nslab == 1 && N == p->n2 * p->n3) {
    // first-mode product over flattened (theta, last) columns: the padded
    // columns ride along (they hold zeros and only ever produce zeros)
    st.N = p->n2 * p->ld;
    st.ldr = st.N;
  }
  const long long nbatch = (long long)p->B * p->C * nslab;
  st.cfg = force_cfg >= 0 ? force_cfg : pick_cfg(var, nbatch, M, N, K, (int)p->stages.size());
  double* op = nullptr;
  const int box_rows = (var == VAR_TN) ? kCfgs[st.cfg].BN : 16;
  int rc = upload_operator(p, var, n_op, get, &op, &st.opmap, box_rows);
  if (rc) return rc;
  if (want_resident(var, epi, nbatch, st.M, st.N, st.K, n_op)) {
    st.res_nb = resident_blocks(epi, n_op);
    st.res_ks = resident_ksteps(st.res_nb);
    if ((rc = upload_resident_operator(p, n_op, st.res_nb, get, &st.rop))) return rc;
  }
  p->stages.push_back(st);
  return CG_OK;
}

double* buf_ptr(cg_plan* p, int id, double* out) { return id == BUF_X ? p->X : id == BUF_Y ? p->Y : out; }

bool pow2(int n) { return n >= 4 && (n & (n - 1)) == 0; }
// theta extents the FFT propagator handles: powers of two, and 100 (M = 5 x 10)
// (the 100-point kernel takes 20 lines per CTA: `span`, the extent the lines are
// spread over, must be a multiple of 20 -- other spans keep the GEMM pair)
bool fft_extent(int n, int span) { return pow2(n) || (n == 100 && span % 20 == 0); }

// row stride of the scaled Phi table: M + 1 rounded up to a multiple of 8
// doubles that is an odd multiple of 8 (two lines 64 bytes apart per half-warp)
int phis_stride(int M) {
  int ps = (M + 1 + 7) / 8 * 8;
  if (ps % 16 == 0) ps += 8;
  return ps;
}

// FFT theta-propagator stage over fields viewed as [A][N][Bc].  phi_at(c, cls,
// col) returns Phi for component c, line class cls and eigen-column col; the
// kernel takes Phi_j = Phi[col(j)] per frequency j = 0..N/2.
template <typename PhiAt>
int add_theta_stage(cg_plan* p, int epi, int src, int dst, int N, int A, int Bc, int class_mode, int nclass,
                    PhiAt phi_at) {
  Stage st{};
  st.var = VAR_THETA;
  st.epi = epi;
  st.N = N;
  st.src = src;
  st.dst = dst;
  st.tA = A;
  st.tBc = Bc;
  st.tclass_mode = class_mode;
  st.tnclass = nclass;
  const int M = N / 2;
  const int span = (Bc == 1) ? A : Bc;
  int W = 16;
  while (W > 1 && (span % W != 0 || theta_smem_bytes(N, W) > 96 * 1024)) W /= 2;
  st.tW = W;
  std::vector<double> h((size_t)p->NO * nclass * (M + 1));
  for (int c = 0; c < p->NO; ++c)
    for (int cls = 0; cls < nclass; ++cls)
      for (int j = 0; j <= M; ++j) {
        const int col = (j == 0) ? 0 : (j == M ? N - 1 : 2 * j - 1);
        h[((size_t)c * nclass + cls) * (M + 1) + j] = phi_at(c, cls, col);
      }
  double* phif = nullptr;
  int rc = upload(p, h.data(), h.size(), &phif);
  if (rc) return rc;
  // scaled copy for the register FFT kernels: exact power-of-two factors
  // (1/(2M) at j = 0, M; 1/(4M) otherwise), rows padded to an odd multiple of
  // 8; the pair (j, M - j) is stored as sum at j and difference at M - j, the
  // self-paired M/2 doubled (thetafft.cuh split_pair)
  const int ps = phis_stride(M);
  std::vector<double> hs((size_t)p->NO * nclass * ps, 0.0);
  for (size_t r = 0; r < (size_t)p->NO * nclass; ++r) {
    auto scaled = [&](int j) { return h[r * (M + 1) + j] * ((j == 0 || j == M) ? 0.5 : 0.25) / (double)M; };
    hs[r * ps] = scaled(0);
    hs[r * ps + M] = scaled(M);
    for (int j = 1; 2 * j <= M; ++j) {
      if (2 * j == M) {
        hs[r * ps + j] = 2.0 * scaled(j);
      } else {
        hs[r * ps + j] = scaled(j) + scaled(M - j);
        hs[r * ps + M - j] = scaled(j) - scaled(M - j);
      }
    }
  }
  double* phis = nullptr;
  if ((rc = upload(p, hs.data(), hs.size(), &phis))) return rc;
  st.phis = phis;
  st.phis_ld = ps;
  std::vector<double> tw(2 * (size_t)N);
  for (int t = 0; t < N; ++t) {
    const double ang = 2.0 * M_PI * (double)t / (double)N;
    tw[2 * t] = std::cos(ang);
    tw[2 * t + 1] = -std::sin(ang);
  }
  double* twd = nullptr;
  if ((rc = upload(p, tw.data(), tw.size(), &twd))) return rc;
  st.phif = phif;
  st.tw = reinterpret_cast<const double2*>(twd);
  p->stages.push_back(st);
  return CG_OK;
}

int launch_fstage(cg_plan* p, const double* Win, const double* Gext, bool fused_kin, bool count_step,
                  cudaStream_t s) {
  StencilParams sp{};
  sp.geometry = p->geom;
  sp.n1 = p->n1;
  sp.n2 = p->n2;
  sp.n3 = p->n3;
  sp.ncomp = p->C;
  sp.opb = p->NO == p->C ? 0 : p->C;
  sp.batch = p->B;
  sp.npts = p->npts;
  sp.rho_b = p->rho_b;
  sp.phi_b = p->phi_b;
  sp.z_b = p->z_b;
  sp.th = p->th;
  sp.d_rho = p->d_rho;
  sp.d_phi = p->d_phi;
  sp.coeff = p->coeff;
  sp.lift = p->lift;
  sp.kin = p->kin_params;
  sp.nparams = p->P;
  sp.ldw = sp.ldf = p->ld;
  sp.npw = sp.npf = p->npts;
  sp.W = Win;
  sp.G = Gext;
  sp.F = p->X;
  sp.with_diffusion = 1;
  sp.with_reaction = 1;
  sp.step = count_step ? p->step_dev : nullptr;
  return launch_fbuild(p->geom, fused_kin ? p->kin : KIN_EXTERNAL, sp, s);
}

int launch_theta(cg_plan* p, const Stage& st, const double* Win, double* Wout, int* first_bad, cudaStream_t s) {
  ThetaParams tp{};
  tp.N = st.N;
  tp.A = st.tA;
  tp.Bc = st.tBc;
  tp.nfield = p->B * p->C;
  tp.ncomp = p->NO;  // operator set of field f = f % NO
  tp.npts = p->npts;
  tp.W = st.tW;
  tp.phi_class_a = st.tclass_mode;
  tp.nclass = st.tnclass;
  tp.phif = st.phif;
  tp.phis = st.phis;
  tp.phis_ld = st.phis_ld;
  tp.tw = st.tw;
  tp.X = buf_ptr(p, st.src, Wout);
  tp.Y = buf_ptr(p, st.dst, Wout);
  tp.Wprev = Win;
  tp.tau = p->tau;
  tp.limit = 1e12;
  tp.first_bad = first_bad;
  tp.step = p->step_dev;
  const long long lines = (long long)tp.nfield * tp.A * tp.Bc;
  const int span = (tp.Bc == 1) ? tp.A : tp.Bc;
  const bool ax = st.epi == EPI_AXPY;
  // register-resident two-phase FFT when the split M = M1*M2 exists and the
  // lines tile the CTA; Stockham smem passes otherwise
  // 64-thread CTAs when 256-thread ones would leave SMs idle (the sphere's
  // 512 theta columns: 32 CTAs at 256 threads, 128 at 64)
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const bool small_cta = !getenv("CURVIGPU_NO_SMALL_CTA");
  // column kernels stage the N twiddles and their lines' Phi rows (one row when every line of a CTA
  // shares its class) behind the FFT tile; FastTheta::smem_cols is the opt-in maximum
  auto cols_smem = [&](size_t tile, int lpb, int ps) {
    return tile + (size_t)st.N * sizeof(double2) + (size_t)(tp.phi_class_a == 1 ? 1 : lpb) * ps * sizeof(double);
  };
#define TRY_FAST_R(M1, M2, R)                                                                        \
  {                                                                                                  \
    using F64 = FastTheta<M1, M2, 64>;                                                               \
    if (small_cta && lines / FastTheta<M1, M2>::LPB < sms && span % F64::LPB == 0) {                  \
      const unsigned nb = (unsigned)(lines / F64::LPB);                                              \
      if (ax)                                                                                        \
        return launch_pdl(theta_fast_kernel<M1, M2, true, 64, R>, dim3(nb), dim3(64), (R) ? F64::smem : cols_smem(F64::smem, F64::LPB, F64::PS), s, tp);  \
      return launch_pdl(theta_fast_kernel<M1, M2, false, 64, R>, dim3(nb), dim3(64), (R) ? F64::smem : cols_smem(F64::smem, F64::LPB, F64::PS), s, tp);   \
    }                                                                                                \
    const unsigned nb = (unsigned)(lines / FastTheta<M1, M2>::LPB);                                  \
    if (ax)                                                                                          \
      return launch_pdl(theta_fast_kernel<M1, M2, true, 256, R>, dim3(nb), dim3(256), (R) ? FastTheta<M1, M2>::smem : cols_smem(FastTheta<M1, M2>::smem, FastTheta<M1, M2>::LPB, FastTheta<M1, M2>::PS), s, tp); \
    return launch_pdl(theta_fast_kernel<M1, M2, false, 256, R>, dim3(nb), dim3(256), (R) ? FastTheta<M1, M2>::smem : cols_smem(FastTheta<M1, M2>::smem, FastTheta<M1, M2>::LPB, FastTheta<M1, M2>::PS), s, tp); \
  }
#define TRY_FAST(M1, M2)                                                                             \
  if (st.N / 2 == (M1) * (M2) && span % FastTheta<M1, M2>::LPB == 0) {                               \
    if (tp.Bc == 1) TRY_FAST_R(M1, M2, true)                                                         \
    TRY_FAST_R(M1, M2, false)                                                                        \
  }
  // M = 50 (n_theta = 100): 5 threads per line, 20 lines per 100-thread CTA
  if (st.N == 100 && span % 20 == 0) {
    using F5 = FastTheta<5, 10, 100>;
    const unsigned nb = (unsigned)(lines / F5::LPB);
    if (tp.Bc == 1) {
      if (ax) return launch_pdl(theta_fast_kernel<5, 10, true, 100, true>, dim3(nb), dim3(100), F5::smem, s, tp);
      return launch_pdl(theta_fast_kernel<5, 10, false, 100, true>, dim3(nb), dim3(100), F5::smem, s, tp);
    }
    if (ax) return launch_pdl(theta_fast_kernel<5, 10, true, 100>, dim3(nb), dim3(100), F5::smem, s, tp);
    return launch_pdl(theta_fast_kernel<5, 10, false, 100>, dim3(nb), dim3(100), F5::smem, s, tp);
  }
  TRY_FAST(4, 4)
  TRY_FAST(4, 8)
  TRY_FAST(8, 8)
  TRY_FAST(8, 16)
  TRY_FAST(16, 16)
#undef TRY_FAST
#undef TRY_FAST_R
  const unsigned blocks = (unsigned)(lines / tp.W);
  const size_t smem = theta_smem_bytes(st.N, st.tW);
  if (st.epi == EPI_AXPY) return launch_pdl(theta_prop_kernel<true>, dim3(blocks), dim3(256), smem, s, tp);
  return launch_pdl(theta_prop_kernel<false>, dim3(blocks), dim3(256), smem, s, tp);
}

int launch_stage(cg_plan* p, const Stage& st, const double* Win, double* Wout, int* first_bad, cudaStream_t s) {
  int rc;
  if (st.var == VAR_THETA) return launch_theta(p, st, Win, Wout, first_bad, s);
  if (st.res_nb) {
    ResParams rp{};
    rp.M = st.M;
    rp.N = st.N;
    rp.K = st.K;
    rp.nslab = st.nslab;
    rp.ncomp = p->NO;
    rp.nitems = p->B * p->C * st.nslab;
    rp.upi = ((st.var == VAR_TN ? st.M : st.N) + 7) / 8;
    rp.ldr = st.ldr;
    rp.fstride = p->npts;
    rp.sstride = st.var == VAR_NN ? (long long)st.K * st.ldr : 0;
    rp.X = buf_ptr(p, st.src, Wout);
    rp.out = buf_ptr(p, st.dst, Wout);
    rp.w = Win;
    rp.op = st.rop;
    rp.op2 = st.rop2;
    rp.phi = st.phi;
    rp.phi_c = st.phi_c;
    rp.phi_s = st.phi_s;
    rp.phi_m = st.phi_m;
    rp.phi_n = st.phi_n;
    rp.phi_rdiv = st.phi_rdiv;
    rp.tau = p->tau;
    rp.limit = 1e12;  // DIVERGENCE_LIMIT, integrators.py:33
    rp.first_bad = first_bad;
    rp.step = p->step_dev;
    return launch_resident(st.var, st.epi, st.res_nb, rp, s);
  }
  {
    const double* src = buf_ptr(p, st.src, Wout);
    double* dst = buf_ptr(p, st.dst, Wout);
    CUtensorMap smap;
    const TileCfg tc = kCfgs[st.cfg];
    const long long nfield = (long long)p->B * p->C;
    if (st.var == VAR_TN) {
      // state as (K, rows, field)
      const uint64_t dims[3] = {(uint64_t)st.K, (uint64_t)st.M, (uint64_t)nfield};
      const uint64_t strides[2] = {(uint64_t)st.ldr * 8, (uint64_t)p->npts * 8};
      const uint32_t box[3] = {16, (uint32_t)tc.BM, 1};
      rc = make_map(&smap, src, 3, dims, strides, box);
    } else {
      // state as (N, K, slab, field)
      const uint64_t dims[4] = {(uint64_t)st.N, (uint64_t)st.K, (uint64_t)st.nslab, (uint64_t)nfield};
      const uint64_t strides[3] = {(uint64_t)st.ldr * 8, (uint64_t)st.K * st.ldr * 8, (uint64_t)p->npts * 8};
      const uint32_t box[4] = {16, 16, 1, 1};
      rc = make_map(&smap, src, 4, dims, strides, box);
    }
    if (rc) return rc;
    GemmParams gp{};
    gp.M = st.M;
    gp.N = st.N;
    gp.K = st.K;
    gp.nslab = st.nslab;
    gp.ncomp = p->NO;  // operator set of field f = f % NO
    gp.nbatch = (int)(nfield * st.nslab);
    gp.tiles_m = (st.M + tc.BM - 1) / tc.BM;
    gp.tiles_n = (st.N + tc.BN - 1) / tc.BN;
    gp.out = dst;
    gp.out_f = p->npts;
    gp.out_s = (long long)st.K * st.ldr;  // slab stride (NN middle mode: K rows of ldr)
    gp.ldc = st.ldr;
    gp.w = Win;
    gp.phi = st.phi;
    gp.phi_c = st.phi_c;
    gp.phi_s = st.phi_s;
    gp.phi_m = st.phi_m;
    gp.phi_n = st.phi_n;
    gp.phi_rdiv = st.phi_rdiv;
    gp.tau = p->tau;
    gp.limit = 1e12;  // DIVERGENCE_LIMIT, integrators.py:33
    gp.first_bad = first_bad;
    gp.step = p->step_dev;
    const bool tma_partial = getenv("CURVIGPU_TMA_PARTIAL") != nullptr;  // measurement / test switch (profiles/r02_tma_partial.txt)
    gp.tma_partial = tma_partial ? 1 : 0;
    Maps mp;
    mp.a = (st.var == VAR_TN) ? smap : st.opmap;
    mp.b = (st.var == VAR_TN) ? st.opmap : smap;
    {
      // output (and, for the axpy epilogue, the previous state) as (N, M, slab, field), (BN, BM) boxes
      const uint64_t dims[4] = {(uint64_t)st.N, (uint64_t)st.M, (uint64_t)st.nslab, (uint64_t)nfield};
      const uint64_t slab = st.nslab > 1 ? (uint64_t)gp.out_s : (uint64_t)st.M * st.ldr;
      const uint64_t strides[3] = {(uint64_t)st.ldr * 8, slab * 8, (uint64_t)p->npts * 8};
      const uint32_t box[4] = {(uint32_t)tc.BN, (uint32_t)tc.BM, 1, 1};
      if ((rc = make_map(&mp.o, dst, 4, dims, strides, box, false))) return rc;
      if (st.epi == EPI_AXPY) {
        if ((rc = make_map(&mp.w, Win, 4, dims, strides, box, false))) return rc;
      } else if (st.epi == EPI_CHAIN) {
        mp.w = st.opmap2;
      } else {
        mp.w = mp.o;
      }
    }
    if ((rc = launch_gemm(st.var, st.epi, st.cfg, mp, gp, s))) return rc;
  }
  return CG_OK;
}

// Launch one full step: Win (+G) -> F -> stage chain -> Wout.
template <int M1, int M2, int KIN, int NBUF, int NT = 256>
int launch_fused_nb(const ThetaParams& tp, const StencilParams& sp, cudaStream_t s, bool configure_only) {
  using D = FusedDisk<M1, M2, NBUF, NT>;
  auto kern = disk_ftheta_kernel<M1, M2, KIN, NBUF, NT>;
  if (configure_only) {
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)D::smem));
    if (getenv("CURVIGPU_MAX_CARVEOUT"))
      CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
    return CG_OK;
  }
  // persistent: (3 - NBUF) CTAs per SM walk the (run, RPB-row block) items
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const long long items = (long long)sp.batch * (sp.n1 / D::RPB);
  static const int cps = getenv("CURVIGPU_FRONT_CPS") ? std::max(1, atoi(getenv("CURVIGPU_FRONT_CPS"))) : 3 - NBUF;
  static const int ctas_sm = getenv("CURVIGPU_FRONT_CTAS_PER_SM") ? atoi(getenv("CURVIGPU_FRONT_CTAS_PER_SM")) : 0;
  // 128-thread CTAs: three per SM (3 x 63 KB of shared memory; measured best for config 5)
  const long long per_sm = ctas_sm > 0 ? ctas_sm : (NT == 128 ? 3 : std::min(cps, 3 - NBUF) * (256 / NT));
  static const int grid_env = getenv("CURVIGPU_FRONT_GRID") ? atoi(getenv("CURVIGPU_FRONT_GRID")) : 0;
  const unsigned blocks = (unsigned)std::min<long long>(items, grid_env > 0 ? grid_env : (long long)num_sms * per_sm);
  int rc = launch_pdl(kern, dim3(blocks), dim3(NT), D::smem, s, tp, sp);
  if (rc) return rc;
  CUDA_TRY(cudaGetLastError());
  return CG_OK;
}

template <int M1, int M2, int KIN>
int launch_fused_t(const ThetaParams& tp, const StencilParams& sp, cudaStream_t s, bool configure_only, int nt) {
  static const int nbuf = getenv("CURVIGPU_FUSED_NBUF") ? atoi(getenv("CURVIGPU_FUSED_NBUF")) : 1;
  if (nt == 64) return launch_fused_nb<M1, M2, KIN, 1, 64>(tp, sp, s, configure_only);
  if (nt == 128) return launch_fused_nb<M1, M2, KIN, 1, 128>(tp, sp, s, configure_only);
  if (nbuf == 1) return launch_fused_nb<M1, M2, KIN, 1>(tp, sp, s, configure_only);
  return launch_fused_nb<M1, M2, KIN, 2>(tp, sp, s, configure_only);
}

template <int M1, int M2>
int launch_fused_k(int kin, const ThetaParams& tp, const StencilParams& sp, cudaStream_t s, bool conf, int nt) {
  switch (kin) {
    case KIN_SCHNAKENBERG: return launch_fused_t<M1, M2, KIN_SCHNAKENBERG>(tp, sp, s, conf, nt);
    case KIN_BRUSSELATOR: return launch_fused_t<M1, M2, KIN_BRUSSELATOR>(tp, sp, s, conf, nt);
    case KIN_GRAY_SCOTT: return launch_fused_t<M1, M2, KIN_GRAY_SCOTT>(tp, sp, s, conf, nt);
    case KIN_BVAM_ETA: return launch_fused_t<M1, M2, KIN_BVAM_ETA>(tp, sp, s, conf, nt);
    case KIN_BVAM: return launch_fused_t<M1, M2, KIN_BVAM>(tp, sp, s, conf, nt);
    default: return launch_fused_t<M1, M2, KIN_DIB>(tp, sp, s, conf, nt);
  }
}

void fill_front_params(cg_plan* p, const double* Win, bool count_step, ThetaParams& tp, StencilParams& sp) {
  const Stage& st = p->stages[0];
  tp = ThetaParams{};
  tp.N = st.N;
  tp.A = st.tA;
  tp.Bc = 1;
  tp.nfield = p->B * p->C;
  tp.ncomp = p->NO;  // operator set of field f = f % NO
  tp.npts = p->npts;
  tp.phi_class_a = st.tclass_mode;
  tp.nclass = st.tnclass;
  tp.phif = st.phif;
  tp.phis = st.phis;
  tp.phis_ld = st.phis_ld;
  tp.tw = st.tw;
  tp.Y = buf_ptr(p, st.dst, nullptr);
  sp = StencilParams{};
  sp.geometry = p->geom;
  sp.n1 = p->n1;
  sp.n2 = p->n2;
  sp.n3 = p->n3;
  sp.ncomp = p->C;
  sp.opb = p->NO == p->C ? 0 : p->C;
  sp.batch = p->B;
  sp.npts = p->npts;
  sp.rho_b = p->rho_b;
  sp.th = p->th;
  sp.d_rho = p->d_rho;
  sp.coeff = p->coeff;
  sp.lift = p->lift;
  sp.kin = p->kin_params;
  sp.nparams = p->P;
  sp.W = Win;
  sp.step = count_step ? p->step_dev : nullptr;
}

int launch_fused_front(cg_plan* p, const double* Win, bool count_step, cudaStream_t s, bool conf = false) {
  ThetaParams tp;
  StencilParams sp;
  fill_front_params(p, Win, count_step, tp, sp);
  if (p->fused_m1 == 8 && p->fused_m2 == 16) return launch_fused_k<8, 16>(p->kin, tp, sp, s, conf, p->fused_nt);
  if (p->fused_m1 == 8 && p->fused_m2 == 8) return launch_fused_k<8, 8>(p->kin, tp, sp, s, conf, p->fused_nt);
  return launch_fused_k<4, 8>(p->kin, tp, sp, s, conf, p->fused_nt);
}

// Launch one full step: Win (+G) -> F -> stage chain -> Wout.
int repack(const cg_plan* p, const double* src, int lds, double* dst, int ldd, cudaStream_t s) {
  const long long rows = p->elems_u / p->nl;
  const long long total = p->elems_u;
  const unsigned blocks = (unsigned)std::min<long long>((total + 255) / 256, 148LL * 16);
  repack_kernel<<<blocks, 256, 0, s>>>(src, lds, dst, ldd, rows, p->nl);
  CUDA_TRY(cudaGetLastError());
  return CG_OK;
}

int launch_step(cg_plan* p, const double* Win, double* Wout, const double* Gext, bool fused_kin, int* first_bad,
                bool count_step, cudaStream_t s) {
  int rc;
  size_t first = 0;
  if (p->fused_front && fused_kin) {
    if ((rc = launch_fused_front(p, Win, count_step, s))) return rc;
    first = 1;
  } else if ((rc = launch_fstage(p, Win, Gext, fused_kin, count_step, s))) {
    return rc;
  }
  for (size_t i = first; i < p->stages.size(); ++i)
    if ((rc = launch_stage(p, p->stages[i], Win, Wout, first_bad, s))) return rc;
  return CG_OK;
}

// Decide whether the disk front end runs fused (after build_stages): disk,
// built-in two-species kinetics, FFT theta with N in {64, 128, 256} and rho
// rows a multiple of the item height.  CURVIGPU_NO_FUSED_FRONT=1 keeps the
// two separate kernels (measurement / A-B comparison).
int setup_fused_front(cg_plan* p) {
  if (p->geom != CG_DISK || p->padded || p->kin == CG_KIN_EXTERNAL || p->C != 2 || p->stages.empty() ||
      p->stages[0].var != VAR_THETA || getenv("CURVIGPU_NO_FUSED_FRONT"))
    return CG_OK;
  const int M = p->n2 / 2;
  int m1 = 0, m2 = 0;
  if (M == 32) m1 = 4, m2 = 8;
  if (M == 64) m1 = 8, m2 = 8;
  if (M == 128) m1 = 8, m2 = 16;
  if (!m1) return CG_OK;
  const int lpb = 256 / (m1 < m2 ? m1 : m2);  // FastTheta::LPB
  if (p->n1 % (lpb / 2) != 0) return CG_OK;
  p->fused_m1 = m1;
  p->fused_m2 = m2;
  // fewer 256-thread items than SMs (config 1: 4): 64-thread items, a
  // quarter of the rows each
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long items256 = (long long)p->B * (p->n1 / (lpb / 2));
  if (items256 < sms && p->n1 % (lpb / 8) == 0 && (lpb / 8) % 2 == 0 && !getenv("CURVIGPU_NO_SMALL_CTA"))
    p->fused_nt = 64;
  // enough items for three 128-thread CTAs per SM (config 5: 8192 items of 8 rows): 128-thread CTAs,
  // front 163.2 -> 159.3 us against two 256-thread CTAs per SM (profiles/r01_front_variants.txt)
  const long long items128 = (long long)p->B * (p->n1 / (lpb / 4));
  if (p->fused_nt == 256 && items128 >= 3LL * sms && p->n1 % (lpb / 4) == 0 && (lpb / 4) % 2 == 0 &&
      !getenv("CURVIGPU_FRONT_NT256"))
    p->fused_nt = 128;
  if (getenv("CURVIGPU_FRONT_NT64") && p->n1 % (lpb / 8) == 0 && (lpb / 8) % 2 == 0) p->fused_nt = 64;  // measurement knob
  int rc = launch_fused_front(p, nullptr, false, nullptr, true);
  if (rc) return rc;
  p->fused_front = true;
  return CG_OK;
}

// ---- small disks: many steps in one cluster kernel (cluster_disk.cuh) ----
void fill_front_params(cg_plan* p, const double* Win, bool count_step, ThetaParams& tp, StencilParams& sp);

template <int M1, int M2, int KIN>
int launch_cluster_t(const ClusterDiskParams& cp, int batch, cudaStream_t s, bool conf) {
  using D = ClusterDisk<M1, M2>;
  auto kern = disk_cluster_kernel<M1, M2, KIN>;
  if (conf) {
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)D::smem));
    if (D::NC > 8) CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(batch * D::NC));
  cfg.blockDim = dim3(D::NT);
  cfg.dynamicSmemBytes = D::smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = D::NC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (conf) {
    // the cluster must be schedulable on this device (16 CTAs of ~115 KB on one GPC)
    int nclusters = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg);
    if (e != cudaSuccess || nclusters < 1) {
      cudaGetLastError();
      return fail(CG_EUNSUPPORTED, "cluster step kernel is not schedulable on this device");
    }
    return CG_OK;
  }
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, cp));
  return CG_OK;
}

template <int M1, int M2>
int launch_cluster_k(int kin, const ClusterDiskParams& cp, int batch, cudaStream_t s, bool conf) {
  switch (kin) {
    case KIN_SCHNAKENBERG: return launch_cluster_t<M1, M2, KIN_SCHNAKENBERG>(cp, batch, s, conf);
    case KIN_BRUSSELATOR: return launch_cluster_t<M1, M2, KIN_BRUSSELATOR>(cp, batch, s, conf);
    case KIN_GRAY_SCOTT: return launch_cluster_t<M1, M2, KIN_GRAY_SCOTT>(cp, batch, s, conf);
    case KIN_BVAM_ETA: return launch_cluster_t<M1, M2, KIN_BVAM_ETA>(cp, batch, s, conf);
    case KIN_BVAM: return launch_cluster_t<M1, M2, KIN_BVAM>(cp, batch, s, conf);
    default: return launch_cluster_t<M1, M2, KIN_DIB>(cp, batch, s, conf);
  }
}

int launch_cluster_steps(cg_plan* p, double* state, long long step0, long long nsteps, int* first_bad,
                         cudaStream_t s, bool conf = false) {
  ClusterDiskParams cp{};
  fill_front_params(p, state, false, cp.tp, cp.sp);
  cp.rop = p->cluster_rop;
  cp.state = state;
  cp.step0 = (int)step0;
  cp.nsteps = (int)nsteps;
  cp.tau = p->tau;
  cp.limit = 1e12;  // DIVERGENCE_LIMIT, integrators.py:33
  cp.first_bad = first_bad;
  if (p->n2 == 128) return launch_cluster_k<8, 8>(p->kin, cp, p->B, s, conf);
  return launch_cluster_k<4, 8>(p->kin, cp, p->B, s, conf);
}

// Eligible: the fused front applies (disk, two species, built-in kinetics, FFT
// theta), the grid is one of the cluster shapes (n_rho = 4 * n_theta / 8:
// 64 x 128 -- config 1 -- or 32 x 64) and every run gets its own cluster at
// once (B * NC <= SMs: a latency-bound plan; larger batches fill the chip
// through the batched kernels).  CURVIGPU_NO_CLUSTER_STEP=1 keeps the
// two-kernel step (measurement / A-B tests).
int setup_cluster_step(cg_plan* p, const cg_desc* d) {
  if (!p->fused_front || getenv("CURVIGPU_NO_CLUSTER_STEP") || !d->phi1_rho) return CG_OK;
  if (!((p->n1 == 64 && p->n2 == 128) || (p->n1 == 32 && p->n2 == 64))) return CG_OK;
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int nc = p->n2 / 8;
  if ((long long)p->B * nc > sms) return CG_OK;
  // phi1_rho in the resident row-major layout [NO][n1][LDS]
  const int n1 = p->n1, lds = res_lds(n1 / 4);
  std::vector<double> h((size_t)p->NO * n1 * lds, 0.0);
  for (int c = 0; c < p->NO; ++c)
    for (int r = 0; r < n1; ++r)
      for (int q = 0; q < n1; ++q) h[((size_t)c * n1 + r) * lds + q] = d->phi1_rho[((size_t)c * n1 + r) * n1 + q];
  double* dev_op = nullptr;
  int rc = upload(p, h.data(), h.size(), &dev_op);
  if (rc) return rc;
  p->cluster_rop = dev_op;
  rc = launch_cluster_steps(p, nullptr, 0, 0, nullptr, nullptr, true);
  if (rc == CG_EUNSUPPORTED) return CG_OK;  // not schedulable here: keep the two-kernel step
  if (rc) return rc;
  p->cluster_step = true;
  return CG_OK;
}

int build_stages(cg_plan* p, const cg_desc* d) {
  const int n1 = p->n1, n2 = p->n2, n3 = p->n3, C = p->NO;  // operator sets
  const double* Q = d->Q_theta;
  auto need = [&](const void* ptr, const char* name) -> int {
    if (!ptr) return fail(CG_EINVAL, std::string("missing operand ") + name);
    return CG_OK;
  };
  int rc = 0;
  // phi tables
  auto up_phi = [&](const double* h, size_t per, double** out) -> int { return upload(p, h, per * C, out); };
  // the FFT theta kernels address unpadded fields: padded plans keep the GEMM pair
  const bool fft = (d->options & CG_OPT_THETA_FFT) != 0 && !p->padded;
  if (p->geom == CG_DISK && fft && pow2(n2)) {
    if ((rc = need(d->phi1_rho, "phi1_rho")) || (rc = need(d->Phi, "Phi"))) return rc;
    const double *Ph = d->Phi, *P1 = d->phi1_rho;
    // T = Q (Phi_i o Q^T F) along theta for every rho row i, by FFT
    if ((rc = add_theta_stage(p, EPI_STORE, BUF_X, BUF_Y, n2, n1, 1, 1, n1,
                              [&](int c, int i, int col) { return Ph[((size_t)c * n1 + i) * n2 + col]; })))
      return rc;
    // W + tau * phi1_rho T
    return add_stage(p, VAR_NN, EPI_AXPY, n1, n2, n1, 1, BUF_Y, BUF_OUT, n1,
                     [&](int c, int r, int q) { return P1[((size_t)c * n1 + r) * n1 + q]; });
  }
  if (p->geom == CG_SPHERE && fft && pow2(n1)) {
    if ((rc = need(d->phi1_phi, "phi1_phi")) || (rc = need(d->Phi, "Phi"))) return rc;
    const double *Ph = d->Phi, *P1 = d->phi1_phi;
    // G = F phi1_phi^T, then W + tau * Q (Phi_j o Q^T G) along theta for every column j
    if ((rc = add_stage(p, VAR_TN, EPI_STORE, n1, n2, n2, 1, BUF_X, BUF_Y, n2,
                        [&](int c, int r, int q) { return P1[((size_t)c * n2 + r) * n2 + q]; })))
      return rc;
    return add_theta_stage(p, EPI_AXPY, BUF_Y, BUF_OUT, n1, 1, n2, 0, n2,
                           [&](int c, int j, int col) { return Ph[((size_t)c * n1 + col) * n2 + j]; });
  }
  if (p->geom == CG_CYLINDER && fft && pow2(n2)) {
    if ((rc = need(d->phi1_rho, "phi1_rho")) || (rc = need(d->Phi, "Phi")) || (rc = need(d->phi1_z, "phi1_z")))
      return rc;
    const double *Ph = d->Phi, *Pz = d->phi1_z, *P1 = d->phi1_rho;
    if ((rc = add_stage(p, VAR_TN, EPI_STORE, n1 * n2, n3, n3, 1, BUF_X, BUF_Y, n3,
                        [&](int c, int r, int q) { return Pz[((size_t)c * n3 + r) * n3 + q]; })))
      return rc;
    if ((rc = add_theta_stage(p, EPI_STORE, BUF_Y, BUF_X, n2, n1, n3, 1, n1,
                              [&](int c, int i, int col) { return Ph[((size_t)c * n1 + i) * n2 + col]; })))
      return rc;
    return add_stage(p, VAR_NN, EPI_AXPY, n1, n2 * n3, n1, 1, BUF_X, BUF_OUT, n1,
                     [&](int c, int r, int q) { return P1[((size_t)c * n1 + r) * n1 + q]; });
  }
  // Ball, polar (last) mode: T = (F x3 V^-1) o Phi_outer, T = T x3 V
  // (integrators.py:217-226).  Both products run in one chained kernel
  // (gemm.cuh EPI_CHAIN, the intermediate stays in shared memory) when the
  // mode fits one 128-column tile; CURVIGPU_NO_CHAIN keeps two stages
  // (bitwise-identical results, tests/test_gpu_parity.py).  Returns the
  // buffer holding T.
  auto ball_polar_mode = [&](double* phio, int* cur) -> int {
    const double *V = d->V_phi, *Vi = d->Vinv_phi;
    auto get_vi = [&](int c, int r, int q) { return Vi[((size_t)c * n3 + r) * n3 + q]; };
    auto get_v = [&](int c, int r, int q) { return V[((size_t)c * n3 + r) * n3 + q]; };
    const bool chain = n3 <= kCfgs[kChainCfg].BN && !getenv("CURVIGPU_NO_CHAIN");
    const char* ccfg = getenv("CURVIGPU_CHAIN_CFG");  // measurement knob
    const int chain_cfg = (ccfg && atoi(ccfg) == kChainCfg16) ? kChainCfg16 : kChainCfg;
    int r2 = chain ? add_stage(p, VAR_TN, EPI_CHAIN, n1 * n2, n3, n3, 1, BUF_X, BUF_Y, n3, get_vi, chain_cfg)
                   : add_stage(p, VAR_TN, EPI_PHI, n1 * n2, n3, n3, 1, BUF_X, BUF_Y, n3, get_vi);
    if (r2) return r2;
    Stage& s0 = p->stages.back();
    s0.phi = phio;
    s0.phi_c = (long long)n1 * n3;
    s0.phi_rdiv = n2;
    s0.phi_m = n3;
    s0.phi_n = 1;
    if (chain) {
      double* op2 = nullptr;
      *cur = BUF_Y;
      if (s0.res_nb) {
        int r3 = upload_resident_operator(p, n3, s0.res_nb, get_v, &s0.rop2);
        if (r3) return r3;
      }
      return upload_operator(p, VAR_TN, n3, get_v, &op2, &s0.opmap2, kCfgs[chain_cfg].BN);
    }
    *cur = BUF_X;
    return add_stage(p, VAR_TN, EPI_STORE, n1 * n2, n3, n3, 1, BUF_Y, BUF_X, n3, get_v);
  };
  auto other = [](int b) { return b == BUF_X ? BUF_Y : BUF_X; };
  if (p->geom == CG_BALL && fft && fft_extent(n2, n3)) {
    if ((rc = need(d->phi1_rho, "phi1_rho")) || (rc = need(d->Phi, "Phi")) ||
        (rc = need(d->Phi_outer, "Phi_outer")) || (rc = need(d->V_phi, "V_phi")) ||
        (rc = need(d->Vinv_phi, "Vinv_phi")))
      return rc;
    double* phio = nullptr;
    if ((rc = up_phi(d->Phi_outer, (size_t)n1 * n3, &phio))) return rc;
    const double *P1 = d->phi1_rho, *Ph = d->Phi;
    int cur = BUF_X;
    if ((rc = ball_polar_mode(phio, &cur))) return rc;
    if ((rc = add_theta_stage(p, EPI_STORE, cur, other(cur), n2, n1, n3, 2, n1 * n3, [&](int c, int cls, int col) {
           const int i = cls / n3, k = cls % n3;
           return Ph[(((size_t)c * n1 + i) * n2 + col) * n3 + k];
         })))
      return rc;
    return add_stage(p, VAR_NN, EPI_AXPY, n1, n2 * n3, n1, 1, other(cur), BUF_OUT, n1,
                     [&](int c, int r, int q) { return P1[((size_t)c * n1 + r) * n1 + q]; });
  }
  if (p->geom == CG_DISK) {
    const int nt = n2;
    if ((rc = need(Q, "Q_theta")) || (rc = need(d->phi1_rho, "phi1_rho")) || (rc = need(d->Phi, "Phi"))) return rc;
    double* phi = nullptr;
    if ((rc = up_phi(d->Phi, (size_t)n1 * n2, &phi))) return rc;
    // T = F Q  (L = Q^T: L[r][q] = Q[q][r]), epilogue *= Phi_c(i, j)
    if ((rc = add_stage(p, VAR_TN, EPI_PHI, n1, n2, n2, 1, BUF_X, BUF_Y, nt,
                        [&](int c, int r, int q) { return Q[((size_t)c * nt + q) * nt + r]; })))
      return rc;
    Stage& s0 = p->stages.back();
    s0.phi = phi;
    s0.phi_c = (long long)n1 * n2;
    s0.phi_m = n2;
    s0.phi_n = 1;
    // T = T Q^T  (L = Q)
    if ((rc = add_stage(p, VAR_TN, EPI_STORE, n1, n2, n2, 1, BUF_Y, BUF_X, nt,
                        [&](int c, int r, int q) { return Q[((size_t)c * nt + r) * nt + q]; })))
      return rc;
    // W + tau * phi1_rho T
    const double* P1 = d->phi1_rho;
    if ((rc = add_stage(p, VAR_NN, EPI_AXPY, n1, n2, n1, 1, BUF_X, BUF_OUT, n1,
                        [&](int c, int r, int q) { return P1[((size_t)c * n1 + r) * n1 + q]; })))
      return rc;
  } else if (p->geom == CG_SPHERE) {
    const int nt = n1, np_ = n2;
    if ((rc = need(Q, "Q_theta")) || (rc = need(d->phi1_phi, "phi1_phi")) || (rc = need(d->Phi, "Phi"))) return rc;
    double* phi = nullptr;
    if ((rc = up_phi(d->Phi, (size_t)n1 * n2, &phi))) return rc;
    // T = Q^T F
    if ((rc = add_stage(p, VAR_NN, EPI_STORE, n1, n2, n1, 1, BUF_X, BUF_Y, nt,
                        [&](int c, int r, int q) { return Q[((size_t)c * nt + q) * nt + r]; })))
      return rc;
    // T = T phi1_phi^T, epilogue *= Phi_c(i, j)
    const double* P1 = d->phi1_phi;
    if ((rc = add_stage(p, VAR_TN, EPI_PHI, n1, n2, n2, 1, BUF_Y, BUF_X, np_,
                        [&](int c, int r, int q) { return P1[((size_t)c * np_ + r) * np_ + q]; })))
      return rc;
    Stage& s1 = p->stages.back();
    s1.phi = phi;
    s1.phi_c = (long long)n1 * n2;
    s1.phi_m = n2;
    s1.phi_n = 1;
    // W + tau * Q T
    if ((rc = add_stage(p, VAR_NN, EPI_AXPY, n1, n2, n1, 1, BUF_X, BUF_OUT, nt,
                        [&](int c, int r, int q) { return Q[((size_t)c * nt + r) * nt + q]; })))
      return rc;
  } else if (p->geom == CG_BALL) {
    if ((rc = need(Q, "Q_theta")) || (rc = need(d->phi1_rho, "phi1_rho")) || (rc = need(d->Phi, "Phi")) ||
        (rc = need(d->Phi_outer, "Phi_outer")) || (rc = need(d->V_phi, "V_phi")) ||
        (rc = need(d->Vinv_phi, "Vinv_phi")))
      return rc;
    double *phi = nullptr, *phio = nullptr;
    if ((rc = up_phi(d->Phi, (size_t)n1 * n2 * n3, &phi))) return rc;
    if ((rc = up_phi(d->Phi_outer, (size_t)n1 * n3, &phio))) return rc;
    const double* P1 = d->phi1_rho;
    // T = (F x3 V^-1) o Phi_outer_c(i, k), T = T x3 V
    int cur = BUF_X;
    if ((rc = ball_polar_mode(phio, &cur))) return rc;
    const int b0 = cur, b1 = other(cur);
    // T = T x2 Q^T, epilogue *= Phi_c(i, j, k)
    if ((rc = add_stage(p, VAR_NN, EPI_PHI, n2, n3, n2, n1, b0, b1, n2,
                        [&](int c, int r, int q) { return Q[((size_t)c * n2 + q) * n2 + r]; })))
      return rc;
    Stage& s2 = p->stages.back();
    s2.phi = phi;
    s2.phi_c = (long long)n1 * n2 * n3;
    s2.phi_s = (long long)n2 * n3;
    s2.phi_m = n3;
    s2.phi_n = 1;
    // T = T x2 Q
    if ((rc = add_stage(p, VAR_NN, EPI_STORE, n2, n3, n2, n1, b1, b0, n2,
                        [&](int c, int r, int q) { return Q[((size_t)c * n2 + r) * n2 + q]; })))
      return rc;
    // W + tau * (T x1 phi1_rho)
    if ((rc = add_stage(p, VAR_NN, EPI_AXPY, n1, n2 * n3, n1, 1, b0, BUF_OUT, n1,
                        [&](int c, int r, int q) { return P1[((size_t)c * n1 + r) * n1 + q]; })))
      return rc;
  } else {  // cylinder
    if ((rc = need(Q, "Q_theta")) || (rc = need(d->phi1_rho, "phi1_rho")) || (rc = need(d->Phi, "Phi")) ||
        (rc = need(d->phi1_z, "phi1_z")))
      return rc;
    double* phi = nullptr;
    if ((rc = up_phi(d->Phi, (size_t)n1 * n2, &phi))) return rc;
    const double *Pz = d->phi1_z, *P1 = d->phi1_rho;
    // T = F x3 phi1_z
    if ((rc = add_stage(p, VAR_TN, EPI_STORE, n1 * n2, n3, n3, 1, BUF_X, BUF_Y, n3,
                        [&](int c, int r, int q) { return Pz[((size_t)c * n3 + r) * n3 + q]; })))
      return rc;
    // T = T x2 Q^T, epilogue *= Phi_c(i, j) (constant along z)
    if ((rc = add_stage(p, VAR_NN, EPI_PHI, n2, n3, n2, n1, BUF_Y, BUF_X, n2,
                        [&](int c, int r, int q) { return Q[((size_t)c * n2 + q) * n2 + r]; })))
      return rc;
    Stage& s1 = p->stages.back();
    s1.phi = phi;
    s1.phi_c = (long long)n1 * n2;
    s1.phi_s = n2;
    s1.phi_m = 1;
    s1.phi_n = 0;
    // T = T x2 Q
    if ((rc = add_stage(p, VAR_NN, EPI_STORE, n2, n3, n2, n1, BUF_X, BUF_Y, n2,
                        [&](int c, int r, int q) { return Q[((size_t)c * n2 + r) * n2 + q]; })))
      return rc;
    // W + tau * (T x1 phi1_rho)
    if ((rc = add_stage(p, VAR_NN, EPI_AXPY, n1, n2 * n3, n1, 1, BUF_Y, BUF_OUT, n1,
                        [&](int c, int r, int q) { return P1[((size_t)c * n1 + r) * n1 + q]; })))
      return rc;
  }
  return CG_OK;
}

int bands_upload(cg_plan* p, const double* h, int n, double** out) { return upload(p, h, (size_t)p->NO * 3 * n, out); }

}  // namespace

extern "C" {

const char* cg_last_error(void) { return g_err.c_str(); }
int cg_version(void) { return 1; }

long long cg_plan_state_elems(const cg_plan* plan) { return plan ? plan->elems_u : 0; }

void cg_plan_destroy(cg_plan* p) {
  if (!p) return;
  for (auto& g : p->graphs)
    if (g.chunk) cudaGraphExecDestroy(g.chunk);
  for (void* a : p->allocs) cudaFree(a);
  if (p->cap_stream) cudaStreamDestroy(p->cap_stream);
  delete p;
}

int cg_plan_create(const cg_desc* d, cg_plan** out) {
  if (!d || !out) return fail(CG_EINVAL, "null argument");
  *out = nullptr;
  if (d->geometry < CG_DISK || d->geometry > CG_CYLINDER) return fail(CG_EINVAL, "unknown geometry");
  const bool is3d = d->geometry == CG_BALL || d->geometry == CG_CYLINDER;
  if (d->n[0] < 2 || d->n[1] < 2 || (is3d && d->n[2] < 2)) return fail(CG_EINVAL, "grid extents must be >= 2");
  if (d->batch < 1 || d->ncomp < 1) return fail(CG_EINVAL, "batch and ncomp must be >= 1");
  if (d->kinetics != CG_KIN_EXTERNAL && d->ncomp != 2)
    return fail(CG_EUNSUPPORTED, "built-in kinetics kinds are two-species");
  if (d->kinetics < CG_KIN_EXTERNAL || d->kinetics > CG_KIN_DIB) return fail(CG_EUNSUPPORTED, "unknown kinetics");
  if (!(d->tau >= 0.0)) return fail(CG_EINVAL, "tau must be nonnegative");
  if (!d->coeff || !d->lift) return fail(CG_EINVAL, "coeff and lift are required");

  cg_plan* p = new cg_plan();
  p->geom = d->geometry;
  p->n1 = d->n[0];
  p->n2 = d->n[1];
  p->n3 = is3d ? d->n[2] : 1;
  p->B = d->batch;
  p->C = d->ncomp;
  p->kin = d->kinetics;
  p->P = d->nparams;
  p->tau = d->tau;
  p->nl = is3d ? p->n3 : p->n2;
  p->ld = (p->nl + 1) & ~1;
  p->padded = p->ld != p->nl;
  p->npts_u = (long long)p->n1 * p->n2 * p->n3;
  p->npts = p->npts_u / p->nl * p->ld;
  p->elems = p->npts * p->B * p->C;
  p->elems_u = p->npts_u * p->B * p->C;
  if (p->npts >= (1LL << 31)) {  // kernels index within a field with 32-bit offsets
    delete p;
    return fail(CG_EUNSUPPORTED, "a field of 2^31 or more points is not supported");
  }
  if (d->ops_per_run != 0 && d->ops_per_run != 1) return fail(CG_EINVAL, "ops_per_run must be 0 or 1");
  p->NO = d->ops_per_run ? p->B * p->C : p->C;
  {
    const char* rz = getenv("CURVIGPU_REDZONE");
    p->redzone = rz && rz[0] && rz[0] != '0';
  }

  int rc = CG_OK;
  auto bail = [&](int code) {
    cg_plan_destroy(p);
    return code;
  };
  const int C = p->C, NO = p->NO;
  if ((rc = upload(p, d->coeff, NO, &p->coeff))) return bail(rc);
  if ((rc = upload(p, d->lift, C, &p->lift))) return bail(rc);
  if (d->kin_params && d->nparams > 0) {
    if ((rc = upload(p, d->kin_params, (size_t)p->B * d->nparams, &p->kin_params))) return bail(rc);
  } else if (p->kin != CG_KIN_EXTERNAL) {
    return bail(fail(CG_EINVAL, "kinetics parameters missing"));
  }
  if (!d->theta_stencil) return bail(fail(CG_EINVAL, "theta stencil missing"));
  if ((rc = upload(p, d->theta_stencil, 2 * (size_t)NO, &p->th))) return bail(rc);
  int n_rho = 0, n_phi = 0, n_z = 0;
  if (p->geom == CG_DISK) n_rho = p->n1;
  if (p->geom == CG_SPHERE) n_phi = p->n2;
  if (p->geom == CG_BALL) {
    n_rho = p->n1;
    n_phi = p->n3;
  }
  if (p->geom == CG_CYLINDER) {
    n_rho = p->n1;
    n_z = p->n3;
  }
  if (n_rho) {
    if (!d->rho_bands || !d->d_rho) return bail(fail(CG_EINVAL, "rho operator missing"));
    if ((rc = bands_upload(p, d->rho_bands, n_rho, &p->rho_b))) return bail(rc);
    if ((rc = upload(p, d->d_rho, (size_t)NO * n_rho, &p->d_rho))) return bail(rc);
  }
  if (n_phi) {
    if (!d->phi_bands || !d->d_phi) return bail(fail(CG_EINVAL, "phi operator missing"));
    if ((rc = bands_upload(p, d->phi_bands, n_phi, &p->phi_b))) return bail(rc);
    if ((rc = upload(p, d->d_phi, (size_t)NO * n_phi, &p->d_phi))) return bail(rc);
  }
  if (n_z) {
    if (!d->z_bands) return bail(fail(CG_EINVAL, "z operator missing"));
    if ((rc = bands_upload(p, d->z_bands, n_z, &p->z_b))) return bail(rc);
  }
  if ((rc = build_stages(p, d))) return bail(rc);
  if ((rc = setup_fused_front(p))) return bail(rc);
  if ((rc = setup_cluster_step(p, d))) return bail(rc);
  for (const Stage& st : p->stages) {
    if (st.var == VAR_THETA) continue;
    if (st.res_nb) {
      ResParams rp{};
      if ((rc = launch_resident(st.var, st.epi, st.res_nb, rp, nullptr, true))) return bail(rc);
      continue;
    }
    Maps dummy{};
    GemmParams gp{};
    if ((rc = launch_gemm(st.var, st.epi, st.cfg, dummy, gp, nullptr, true))) return bail(rc);
  }
  {
    StencilParams sp{};
    if ((rc = launch_fbuild(p->geom, KIN_EXTERNAL, sp, nullptr, true))) return bail(rc);
    if ((rc = launch_fbuild(p->geom, p->kin, sp, nullptr, true))) return bail(rc);
  }
  {
    cudaError_t e1 = cudaFuncSetAttribute(theta_prop_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          100 * 1024);
    cudaError_t e2 = cudaFuncSetAttribute(theta_prop_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          100 * 1024);
    if (e1 != cudaSuccess || e2 != cudaSuccess) return bail(fail(CG_ECUDA, "theta kernel smem opt-in failed"));
#define OPT_IN_R(M1, M2, R)                                                                                   \
  e1 = cudaFuncSetAttribute(theta_fast_kernel<M1, M2, true, 256, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,\
                            (int)FastTheta<M1, M2>::smem_cols);                                               \
  e2 = cudaFuncSetAttribute(theta_fast_kernel<M1, M2, false, 256, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,\
                            (int)FastTheta<M1, M2>::smem_cols);                                               \
  if (e1 != cudaSuccess || e2 != cudaSuccess) return bail(fail(CG_ECUDA, "theta kernel smem opt-in failed"));  \
  e1 = cudaFuncSetAttribute(theta_fast_kernel<M1, M2, true, 64, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                            (int)FastTheta<M1, M2, 64>::smem_cols);                                           \
  e2 = cudaFuncSetAttribute(theta_fast_kernel<M1, M2, false, 64, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,\
                            (int)FastTheta<M1, M2, 64>::smem_cols);                                           \
  if (e1 != cudaSuccess || e2 != cudaSuccess) return bail(fail(CG_ECUDA, "theta kernel smem opt-in failed"));
#define OPT_IN(M1, M2) OPT_IN_R(M1, M2, false) OPT_IN_R(M1, M2, true)
    e1 = cudaFuncSetAttribute(theta_fast_kernel<5, 10, true, 100>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)FastTheta<5, 10, 100>::smem);
    e2 = cudaFuncSetAttribute(theta_fast_kernel<5, 10, false, 100>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)FastTheta<5, 10, 100>::smem);
    if (e1 != cudaSuccess || e2 != cudaSuccess) return bail(fail(CG_ECUDA, "theta kernel smem opt-in failed"));
    e1 = cudaFuncSetAttribute(theta_fast_kernel<5, 10, true, 100, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)FastTheta<5, 10, 100>::smem);
    e2 = cudaFuncSetAttribute(theta_fast_kernel<5, 10, false, 100, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)FastTheta<5, 10, 100>::smem);
    if (e1 != cudaSuccess || e2 != cudaSuccess) return bail(fail(CG_ECUDA, "theta kernel smem opt-in failed"));
    OPT_IN(4, 4)
    OPT_IN(4, 8)
    OPT_IN(8, 8)
    OPT_IN(8, 16)
    OPT_IN(16, 16)
#undef OPT_IN
#undef OPT_IN_R
  }
  // the state-sized workspaces (X, Y, S2, S0) are allocated on first use
  // (ensure_workspace): a plan used only as a descriptor -- the parent of a
  // laned SplitPlan, whose lanes step their own sub-plans -- never holds them
  if ((rc = dev_alloc(p, sizeof(int), reinterpret_cast<void**>(&p->step_dev)))) return bail(rc);
  if ((rc = dev_alloc(p, sizeof(int) * (size_t)p->B * C, reinterpret_cast<void**>(&p->scratch_bad))))
    return bail(rc);
  cudaError_t e = cudaMemset(p->step_dev, 0, sizeof(int));
  if (e != cudaSuccess) return bail(fail(CG_ECUDA, cudaGetErrorString(e)));
  e = cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) return bail(fail(CG_ECUDA, cudaGetErrorString(e)));
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return bail(fail(CG_ECUDA, cudaGetErrorString(e)));
  *out = p;
  return CG_OK;
}

int cg_plan_stage_count(const cg_plan* p) { return p ? (int)p->stages.size() : 0; }

long long cg_plan_check_redzones(cg_plan* p) {
  if (!p) return fail(CG_EINVAL, "null plan");
  if (!p->redzone) return fail(CG_EINVAL, "plan was created without CURVIGPU_REDZONE=1");
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return fail(CG_ECUDA, cudaGetErrorString(e));
  std::vector<unsigned char> h(kRedzone);
  long long bad = 0;
  for (const auto& g : p->guarded) {
    for (const uint8_t* band : {g.raw, g.raw + kRedzone + g.bytes}) {
      e = cudaMemcpy(h.data(), band, kRedzone, cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) return fail(CG_ECUDA, cudaGetErrorString(e));
      for (unsigned char c : h) bad += c != kRedzoneByte;
    }
  }
  return bad;
}

int cg_plan_copy_workspace(cg_plan* p, int which, double* dst, void* stream) {
  if (!p || !dst || which < 0 || which > 2) return fail(CG_EINVAL, "bad workspace request");
  int rc = ensure_workspace(p);
  if (rc) return rc;
  const double* src = which == 0 ? p->X : which == 1 ? p->Y : p->S2;
  if (p->padded) return repack(p, src, p->ld, dst, p->nl, static_cast<cudaStream_t>(stream));
  CUDA_TRY(cudaMemcpyAsync(dst, src, (size_t)p->elems * sizeof(double), cudaMemcpyDeviceToDevice,
                           static_cast<cudaStream_t>(stream)));
  return CG_OK;
}

int cg_plan_stage_info(const cg_plan* p, int stage, long long* flops, long long* bytes) {
  if (!p || stage < -2 || stage >= (int)p->stages.size()) return fail(CG_EINVAL, "bad stage index");
  if (stage < 0) {  // F-build, or the fused F-build + theta kernel: read W once, write F (T) once
    if (flops) *flops = 0;
    if (bytes) *bytes = 2LL * p->elems_u * (long long)sizeof(double);  // read W once, write F once
    return CG_OK;
  }
  const Stage& st = p->stages[stage];
  const long long items = (long long)p->B * p->C * st.nslab;
  if (flops) *flops = (st.epi == EPI_CHAIN ? 4LL : 2LL) * st.M * st.N * st.K * items;  // a chain is two products
  if (bytes) *bytes = (st.epi == EPI_AXPY ? 3LL : 2LL) * p->elems_u * (long long)sizeof(double);
  return CG_OK;
}

int cg_plan_step_kernels(const cg_plan* p, int* ids, int max_ids) {
  if (!p || !ids) return fail(CG_EINVAL, "null argument");
  int n = 0;
  auto push = [&](int v) {
    if (n < max_ids) ids[n] = v;
    ++n;
  };
  size_t first = 0;
  if (p->fused_front && p->kin != CG_KIN_EXTERNAL) {
    push(-2);
    first = 1;
  } else {
    push(-1);
  }
  for (size_t i = first; i < p->stages.size(); ++i) push((int)i);
  return n;
}

int cg_run_stage(cg_plan* p, int stage, const double* W, double* W_out, int* first_bad, void* stream) {
  if (!p || !W || !W_out) return fail(CG_EINVAL, "null argument");
  if (stage < -2 || stage >= (int)p->stages.size()) return fail(CG_EINVAL, "bad stage index");
  if (stage == -2 && !p->fused_front) return fail(CG_EINVAL, "plan has no fused front kernel");
  if (p->padded) return fail(CG_EUNSUPPORTED, "per-stage access needs an even contiguous axis");
  if (int rc = ensure_workspace(p)) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (stage == -2) return launch_fused_front(p, W, false, s);
  if (stage < 0) return launch_fstage(p, W, nullptr, p->kin != CG_KIN_EXTERNAL, false, s);
  return launch_stage(p, p->stages[stage], W, W_out, first_bad ? first_bad : p->scratch_bad, s);
}

int cg_apply_diffusion(cg_plan* p, const double* W, double* out, void* stream) {
  if (!p || !W || !out) return fail(CG_EINVAL, "null argument");
  StencilParams sp{};
  sp.geometry = p->geom;
  sp.n1 = p->n1;
  sp.n2 = p->n2;
  sp.n3 = p->n3;
  sp.ncomp = p->C;
  sp.opb = p->NO == p->C ? 0 : p->C;
  sp.batch = p->B;
  sp.npts = p->npts;
  sp.rho_b = p->rho_b;
  sp.phi_b = p->phi_b;
  sp.z_b = p->z_b;
  sp.th = p->th;
  sp.d_rho = p->d_rho;
  sp.d_phi = p->d_phi;
  sp.coeff = p->coeff;
  sp.lift = p->lift;
  sp.ldw = sp.ldf = p->nl;  // caller's unpadded arrays
  sp.npw = sp.npf = p->npts_u;
  sp.W = W;
  sp.F = out;
  sp.with_diffusion = 1;
  sp.with_reaction = 0;
  return launch_fbuild(p->geom, KIN_EXTERNAL, sp, static_cast<cudaStream_t>(stream));
}

int cg_kinetics(cg_plan* p, const double* W, double* G, void* stream) {
  if (!p || !W || !G) return fail(CG_EINVAL, "null argument");
  if (p->kin == CG_KIN_EXTERNAL) return fail(CG_EINVAL, "plan has no built-in kinetics");
  StencilParams sp{};
  sp.geometry = p->geom;
  sp.n1 = p->n1;
  sp.n2 = p->n2;
  sp.n3 = p->n3;
  sp.ncomp = p->C;
  sp.opb = p->NO == p->C ? 0 : p->C;
  sp.batch = p->B;
  sp.npts = p->npts;
  sp.lift = p->lift;
  sp.kin = p->kin_params;
  sp.nparams = p->P;
  sp.ldw = sp.ldf = p->nl;
  sp.npw = sp.npf = p->npts_u;
  sp.W = W;
  sp.F = G;
  sp.with_diffusion = 0;
  sp.with_reaction = 1;
  return launch_fbuild(p->geom, p->kin, sp, static_cast<cudaStream_t>(stream));
}

int cg_step(cg_plan* p, const double* W, const double* G, double* W_out, void* stream) {
  return cg_step_guarded(p, W, G, W_out, p ? p->scratch_bad : nullptr, stream);
}

int cg_step_guarded(cg_plan* p, const double* W, const double* G, double* W_out, int* first_bad, void* stream) {
  if (!p || !W || !G || !W_out || !first_bad) return fail(CG_EINVAL, "null argument");
  if (W == W_out) return fail(CG_EINVAL, "W_out must not alias W");
  if (int rc = ensure_workspace(p)) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool count = first_bad != p->scratch_bad;
  if (!p->padded) return launch_step(p, W, W_out, G, false, first_bad, count, s);
  // padded storage: W -> S0, G -> S2 (consumed by the F-build before the last stage writes S2)
  int rc;
  if ((rc = repack(p, W, p->nl, p->S0, p->ld, s)) || (rc = repack(p, G, p->nl, p->S2, p->ld, s))) return rc;
  if ((rc = launch_step(p, p->S0, p->S2, p->S2, false, first_bad, count, s))) return rc;
  return repack(p, p->S2, p->ld, W_out, p->nl, s);
}

int cg_plan_set_step(cg_plan* p, long long step, void* stream) {
  if (!p) return fail(CG_EINVAL, "null plan");
  if (step < 0 || step > INT_MAX) return fail(CG_EINVAL, "step out of range");
  set_step_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(p->step_dev, (int)step);
  CUDA_TRY(cudaGetLastError());
  return CG_OK;
}

// ---- standalone mu-mode product (tensor.mode_product, tensor.py:31-49) ----
// One GEMM stage of the plan machinery on its own: the field is the stage's
// source, the caller's output its destination.
struct cg_product {
  cg_plan* plan;
};

int cg_product_create(int mu, int ndim, const int* dims, const double* L, cg_product** out) {
  if (!dims || !L || !out) return fail(CG_EINVAL, "null argument");
  *out = nullptr;
  if (ndim < 2 || ndim > 3) return fail(CG_EINVAL, "fields of order 2 or 3");
  if (mu < 1 || mu > ndim) return fail(CG_EINVAL, "mode out of range for the field's order");
  for (int i = 0; i < ndim; ++i)
    if (dims[i] < 1) return fail(CG_EINVAL, "extents must be positive");
  if (dims[ndim - 1] % 2 != 0) return fail(CG_EUNSUPPORTED, "the contiguous (last) extent must be even");
  cg_plan* p = new cg_plan();
  p->geom = ndim == 3 ? CG_CYLINDER : CG_DISK;  // only names the order of the field here
  p->n1 = dims[0];
  p->n2 = dims[1];
  p->n3 = ndim == 3 ? dims[2] : 1;
  p->B = p->C = p->NO = 1;
  p->kin = CG_KIN_EXTERNAL;
  p->P = 0;
  p->tau = 0.0;
  p->nl = dims[ndim - 1];
  p->ld = p->nl;
  p->padded = false;
  p->npts = p->npts_u = (long long)p->n1 * p->n2 * p->n3;
  p->elems = p->elems_u = p->npts;
  const int n = dims[mu - 1];
  auto get = [&](int, int r, int q) { return L[(size_t)r * n + q]; };
  int rc;
  if (mu == ndim)  // last mode: Y = X L^T over contiguous rows
    rc = add_stage(p, VAR_TN, EPI_STORE, (int)(p->npts / n), n, n, 1, BUF_X, BUF_OUT, n, get);
  else if (mu == 1)  // first mode: Y = L X over the flattened trailing extents
    rc = add_stage(p, VAR_NN, EPI_STORE, n, (int)(p->npts / n), n, 1, BUF_X, BUF_OUT, n, get);
  else  // middle mode of an order-3 field: one slab per leading index
    rc = add_stage(p, VAR_NN, EPI_STORE, n, p->n3, n, p->n1, BUF_X, BUF_OUT, n, get);
  if (rc == CG_OK) {
    const Stage& st = p->stages[0];
    if (st.res_nb) {
      ResParams rp{};
      rc = launch_resident(st.var, st.epi, st.res_nb, rp, nullptr, true);
    } else {
      Maps dummy{};
      GemmParams gp{};
      rc = launch_gemm(st.var, st.epi, st.cfg, dummy, gp, nullptr, true);
    }
  }
  if (rc == CG_OK && cudaDeviceSynchronize() != cudaSuccess) rc = fail(CG_ECUDA, "operator upload failed");
  if (rc) {
    cg_plan_destroy(p);
    return rc;
  }
  *out = new cg_product{p};
  return CG_OK;
}

int cg_product_apply(cg_product* h, const double* T, double* out, void* stream) {
  if (!h || !T || !out) return fail(CG_EINVAL, "null argument");
  if (T == out) return fail(CG_EINVAL, "mode products are out of place");
  if ((reinterpret_cast<uintptr_t>(T) | reinterpret_cast<uintptr_t>(out)) & 15)
    return fail(CG_EINVAL, "fields must be 16-byte aligned");
  cg_plan* p = h->plan;
  p->X = const_cast<double*>(T);  // the stage's source buffer (read only)
  return launch_stage(p, p->stages[0], nullptr, out, nullptr, static_cast<cudaStream_t>(stream));
}

void cg_product_destroy(cg_product* h) {
  if (!h) return;
  h->plan->X = nullptr;
  cg_plan_destroy(h->plan);
  delete h;
}

// hadamard(A, B) (tensor.py:77-83): out = a * b elementwise
int cg_hadamard(const double* a, const double* b, double* out, long long n, void* stream) {
  if (!a || !b || !out) return fail(CG_EINVAL, "null argument");
  if (n < 1) return fail(CG_EINVAL, "n must be positive");
  const unsigned blocks = (unsigned)std::min<long long>((n + 255) / 256, 148LL * 16);
  hadamard_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(a, b, out, n);
  CUDA_TRY(cudaGetLastError());
  return CG_OK;
}

long long cg_weighted_sums_scratch(long long nfield, long long npts) {
  if (nfield <= 0 || npts <= 0) return 0;
  return nfield * wsum_segments(npts);
}

int cg_weighted_sums(const double* X, long long nfield, long long npts, const double* w, int ncls,
                     const double* off, double* out, double* scratch, long long scratch_len, void* stream) {
  if (!X || !w || !out || !scratch) return fail(CG_EINVAL, "null argument");
  if (nfield <= 0 || npts <= 0 || ncls <= 0) return fail(CG_EINVAL, "nfield, npts and ncls must be positive");
  if (nfield > 65535 || npts > (long long)INT_MAX * 2) return fail(CG_EUNSUPPORTED, "too many fields or points");
  const long long nseg = wsum_segments(npts);
  if (scratch_len < nfield * nseg) return fail(CG_EINVAL, "scratch too small (see cg_weighted_sums_scratch)");
  if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(w)) & 15)
    return fail(CG_EINVAL, "X and w must be 16-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  wsum_partial_kernel<<<dim3((unsigned)nseg, (unsigned)nfield), kWsThreads, 0, s>>>(X, npts, w, ncls, scratch,
                                                                                   (int)nseg);
  CUDA_TRY(cudaGetLastError());
  wsum_final_kernel<<<(unsigned)((nfield + 127) / 128), 128, 0, s>>>(scratch, (int)nseg, (int)nfield, ncls, off, out);
  CUDA_TRY(cudaGetLastError());
  return CG_OK;
}

struct CoupledGraph {
  const cg_plan* bulk;
  const cg_plan* surf;
  double* wb;
  double* ws;
  int* first_bad;
  cudaGraphExec_t chunk;
};

struct cg_coupling {
  CouplingParams cp;
  double* G = nullptr;  // [2][bulk] then [2][surface]
  cudaStream_t cap_stream = nullptr, side_stream = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  std::vector<CoupledGraph> graphs;
  ~cg_coupling() {
    for (auto& g : graphs) cudaGraphExecDestroy(g.chunk);
    if (G) cudaFree(G);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    if (side_stream) cudaStreamDestroy(side_stream);
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
  }
};

int cg_coupling_create(const cg_coupling_desc* d, cg_coupling** out) {
  if (!d || !out) return fail(CG_EINVAL, "null argument");
  *out = nullptr;
  if (d->kind != CG_BS_BALL && d->kind != CG_BS_CYLINDER) return fail(CG_EUNSUPPORTED, "unknown coupling kind");
  const int need = d->kind == CG_BS_BALL ? 8 : 16;
  if (!d->params || d->nparams < need) return fail(CG_EINVAL, "coupling parameters missing");
  for (int i = 0; i < 3; ++i)
    if (d->nb[i] < 2) return fail(CG_EINVAL, "bulk extents must be >= 2");
  const long long sb = d->kind == CG_BS_BALL ? (long long)d->nb[1] * d->nb[2] : (long long)d->nb[0] * d->nb[1];
  if ((long long)d->ns[0] * d->ns[1] != sb) return fail(CG_EINVAL, "surface grid does not match the bulk trace");
  cg_coupling* c = new cg_coupling();
  CouplingParams& cp = c->cp;
  cp.kind = d->kind;
  cp.nb1 = d->nb[0];
  cp.nb2 = d->nb[1];
  cp.nb3 = d->nb[2];
  cp.ns1 = d->ns[0];
  cp.ns2 = d->ns[1];
  cp.nbpts = (long long)d->nb[0] * d->nb[1] * d->nb[2];
  cp.nspts = sb;
  // caller layout (cg_coupled_kinetics); cg_coupled_run switches to the plans' storage
  cp.ldb = cp.nb3;
  cp.lds = cp.ns2;
  cp.fb = cp.nbpts;
  cp.fs = cp.nspts;
  if (d->kind == CG_BS_BALL ? (d->ns[0] != d->nb[1] || d->ns[1] != d->nb[2])
                            : (d->ns[0] != d->nb[0] || d->ns[1] != d->nb[1]))
    return fail(CG_EINVAL, "surface grid does not match the bulk trace");
  for (int i = 0; i < 16; ++i) cp.k[i] = i < d->nparams ? d->params[i] : 0.0;
  cp.h = d->geom[0];
  cp.rho_edge = d->geom[1];
  for (int i = 0; i < 4; ++i) cp.lift[i] = d->lift[i];
  auto bail = [&](cudaError_t e) {
    delete c;
    return fail(CG_ECUDA, std::string("cg_coupling_create: ") + cudaGetErrorString(e));
  };
  // reaction terms in the plans' storage layout (last axes padded to even)
  const long long fb_s = (long long)cp.nb1 * cp.nb2 * ((cp.nb3 + 1) & ~1);
  const long long fs_s = (long long)cp.ns1 * ((cp.ns2 + 1) & ~1);
  cudaError_t e = cudaMalloc(&c->G, (size_t)2 * (fb_s + fs_s) * sizeof(double));
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming);
  if (e != cudaSuccess) return bail(e);
  *out = c;
  return CG_OK;
}

void cg_coupling_destroy(cg_coupling* c) { delete c; }

int cg_coupled_kinetics(cg_coupling* c, const double* Wb, const double* Ws, double* Gb, double* Gs, void* stream) {
  if (!c || !Wb || !Ws || !Gb || !Gs) return fail(CG_EINVAL, "null argument");
  CouplingParams cp = c->cp;
  cp.Wb = Wb;
  cp.Ws = Ws;
  cp.Gb = Gb;
  cp.Gs = Gs;
  const long long total = cp.nbpts + cp.nspts;
  coupled_kinetics_kernel<<<(unsigned)((total + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(cp);
  CUDA_TRY(cudaGetLastError());
  return CG_OK;
}

}  // extern "C"

namespace {

// One coupled step: reaction terms from the common state, then the bulk pair
// on stream s and the surface pair on the coupling's side stream (the two
// step_split chains are independent once G is known), joined back on s.
int coupled_step(cg_coupling* c, cg_plan* bulk, cg_plan* surf, const double* wb, const double* ws, double* wb_out,
                 double* ws_out, int* first_bad, cudaStream_t s) {
  CouplingParams cp = c->cp;
  cp.ldb = bulk->ld;
  cp.lds = surf->ld;
  cp.fb = bulk->npts;
  cp.fs = surf->npts;
  cp.Wb = wb;
  cp.Ws = ws;
  cp.Gb = c->G;
  cp.Gs = c->G + 2 * cp.fb;
  const long long total = cp.nbpts + cp.nspts;
  coupled_kinetics_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(cp);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaEventRecord(c->fork, s));
  CUDA_TRY(cudaStreamWaitEvent(c->side_stream, c->fork, 0));
  int rc = launch_step(surf, ws, ws_out, cp.Gs, false, first_bad + 2, true, c->side_stream);
  if (rc) return rc;
  if ((rc = launch_step(bulk, wb, wb_out, cp.Gb, false, first_bad, true, s))) return rc;
  CUDA_TRY(cudaEventRecord(c->join, c->side_stream));
  CUDA_TRY(cudaStreamWaitEvent(s, c->join, 0));
  return CG_OK;
}

}  // namespace

extern "C" {

static int coupled_steps(cg_coupling* c, cg_plan* bulk, cg_plan* surf, double* Wb, double* Ws, long long step0,
                  long long nsteps, int* first_bad, cudaStream_t s);

int cg_coupled_run(cg_coupling* c, cg_plan* bulk, cg_plan* surf, double* Wb, double* Ws, long long step0,
                   long long nsteps, int* first_bad, void* stream) {
  if (!c || !bulk || !surf || !Wb || !Ws || !first_bad) return fail(CG_EINVAL, "null argument");
  if (nsteps < 0) return fail(CG_EINVAL, "nsteps must be >= 0");
  if (step0 < 0 || step0 + nsteps > INT_MAX) return fail(CG_EINVAL, "step index overflow");
  if (bulk->B != 1 || surf->B != 1 || bulk->C != 2 || surf->C != 2)
    return fail(CG_EINVAL, "coupled plans must hold one run of two components each");
  if (bulk->n1 != c->cp.nb1 || bulk->n2 != c->cp.nb2 || bulk->n3 != c->cp.nb3 || surf->n1 != c->cp.ns1 ||
      surf->n2 != c->cp.ns2)
    return fail(CG_EINVAL, "plan grids do not match the coupling");
  if (bulk->kin != CG_KIN_EXTERNAL || surf->kin != CG_KIN_EXTERNAL)
    return fail(CG_EINVAL, "coupled plans must be created with CG_KIN_EXTERNAL");
  const int want = c->cp.kind == CG_BS_BALL ? CG_BALL : CG_CYLINDER;
  const int want_s = c->cp.kind == CG_BS_BALL ? CG_SPHERE : CG_DISK;
  if (bulk->geom != want || surf->geom != want_s) return fail(CG_EINVAL, "plan geometries do not match the coupling");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (nsteps == 0) return CG_OK;
  if (int rc = ensure_workspace(bulk)) return rc;
  if (int rc = ensure_workspace(surf)) return rc;
  // padded plans step their storage copies (S0) of the caller's fields
  double* wb = bulk->padded ? bulk->S0 : Wb;
  double* ws = surf->padded ? surf->S0 : Ws;
  int rc;
  if (bulk->padded && (rc = repack(bulk, Wb, bulk->nl, wb, bulk->ld, s))) return rc;
  if (surf->padded && (rc = repack(surf, Ws, surf->nl, ws, surf->ld, s))) return rc;
  if ((rc = coupled_steps(c, bulk, surf, wb, ws, step0, nsteps, first_bad, s))) return rc;
  if (bulk->padded && (rc = repack(bulk, wb, bulk->ld, Wb, bulk->nl, s))) return rc;
  if (surf->padded && (rc = repack(surf, ws, surf->ld, Ws, surf->nl, s))) return rc;
  return CG_OK;
}

static int coupled_steps(cg_coupling* c, cg_plan* bulk, cg_plan* surf, double* Wb, double* Ws, long long step0,
                  long long nsteps, int* first_bad, cudaStream_t s) {
  set_step_kernel<<<1, 1, 0, s>>>(bulk->step_dev, (int)step0);
  set_step_kernel<<<1, 1, 0, s>>>(surf->step_dev, (int)step0);
  CUDA_TRY(cudaGetLastError());
  int rc;
  long long done = 0;
  if (nsteps >= kChunk) {
    CoupledGraph* ge = nullptr;
    for (auto& g : c->graphs)
      if (g.bulk == bulk && g.surf == surf && g.wb == Wb && g.ws == Ws && g.first_bad == first_bad) ge = &g;
    if (!ge) {
      CUDA_TRY(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
      int crc = CG_OK;
      for (int k = 0; k < kChunk && crc == CG_OK; ++k) {
        const bool even = (k % 2) == 0;
        crc = coupled_step(c, bulk, surf, even ? Wb : bulk->S2, even ? Ws : surf->S2, even ? bulk->S2 : Wb,
                           even ? surf->S2 : Ws, first_bad, c->cap_stream);
      }
      cudaGraph_t graph = nullptr;
      cudaError_t e = cudaStreamEndCapture(c->cap_stream, &graph);
      if (crc) {
        if (graph) cudaGraphDestroy(graph);
        return crc;
      }
      if (e != cudaSuccess) return fail(CG_ECUDA, std::string("capture: ") + cudaGetErrorString(e));
      cudaGraphExec_t exec = nullptr;
      e = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) return fail(CG_ECUDA, std::string("instantiate: ") + cudaGetErrorString(e));
      if (c->graphs.size() >= 4) {
        cudaGraphExecDestroy(c->graphs.front().chunk);
        c->graphs.erase(c->graphs.begin());
      }
      c->graphs.push_back(CoupledGraph{bulk, surf, Wb, Ws, first_bad, exec});
      ge = &c->graphs.back();
    }
    while (nsteps - done >= kChunk) {
      CUDA_TRY(cudaGraphLaunch(ge->chunk, s));
      done += kChunk;
    }
  }
  while (done < nsteps) {
    if ((rc = coupled_step(c, bulk, surf, Wb, Ws, bulk->S2, surf->S2, first_bad, s))) return rc;
    ++done;
    if (done < nsteps) {
      if ((rc = coupled_step(c, bulk, surf, bulk->S2, surf->S2, Wb, Ws, first_bad, s))) return rc;
      ++done;
    } else {
      CUDA_TRY(cudaMemcpyAsync(Wb, bulk->S2, (size_t)bulk->elems * sizeof(double), cudaMemcpyDeviceToDevice, s));
      CUDA_TRY(cudaMemcpyAsync(Ws, surf->S2, (size_t)surf->elems * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
  }
  return CG_OK;
}

}  // extern "C"

namespace {

int run_steps(cg_plan* p, double* state, long long step0, long long nsteps, int* first_bad, cudaStream_t s) {
  if (p->cluster_step) {
    // all steps in one kernel, the state resident in the cluster's shared memory
    int crc = launch_cluster_steps(p, state, step0, nsteps, first_bad, s);
    if (crc) return crc;
    set_step_kernel<<<1, 1, 0, s>>>(p->step_dev, (int)(step0 + nsteps));
    CUDA_TRY(cudaGetLastError());
    return CG_OK;
  }
  set_step_kernel<<<1, 1, 0, s>>>(p->step_dev, (int)step0);
  CUDA_TRY(cudaGetLastError());
  int rc;
  long long done = 0;
  if (nsteps >= kChunk) {
    GraphEntry* ge = nullptr;
    for (auto& g : p->graphs)
      if (g.state == state && g.first_bad == first_bad) ge = &g;
    if (!ge) {
      // capture kChunk steps state -> S2 -> state ... on a private stream
      CUDA_TRY(cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal));
      int crc = CG_OK;
      for (int k = 0; k < kChunk && crc == CG_OK; ++k) {
        const bool even = (k % 2) == 0;
        crc = launch_step(p, even ? state : p->S2, even ? p->S2 : state, nullptr, true, first_bad, true,
                          p->cap_stream);
      }
      cudaGraph_t graph = nullptr;
      cudaError_t e = cudaStreamEndCapture(p->cap_stream, &graph);
      if (crc) {
        if (graph) cudaGraphDestroy(graph);
        return crc;
      }
      if (e != cudaSuccess) return fail(CG_ECUDA, std::string("capture: ") + cudaGetErrorString(e));
      cudaGraphExec_t exec = nullptr;
      e = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) return fail(CG_ECUDA, std::string("instantiate: ") + cudaGetErrorString(e));
      if (p->graphs.size() >= 4) {
        cudaGraphExecDestroy(p->graphs.front().chunk);
        p->graphs.erase(p->graphs.begin());
      }
      p->graphs.push_back(GraphEntry{state, first_bad, exec});
      ge = &p->graphs.back();
    }
    while (nsteps - done >= kChunk) {
      CUDA_TRY(cudaGraphLaunch(ge->chunk, s));
      done += kChunk;
    }
  }
  // remainder eagerly, in pairs; an odd last step lands in S2 and is copied back
  while (done < nsteps) {
    if ((rc = launch_step(p, state, p->S2, nullptr, true, first_bad, true, s))) return rc;
    ++done;
    if (done < nsteps) {
      if ((rc = launch_step(p, p->S2, state, nullptr, true, first_bad, true, s))) return rc;
      ++done;
    } else {
      CUDA_TRY(cudaMemcpyAsync(state, p->S2, (size_t)p->elems * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
  }
  return CG_OK;
}

}  // namespace

extern "C" {

int cg_run(cg_plan* p, double* state, long long step0, long long nsteps, int* first_bad, void* stream) {
  if (!p || !state || !first_bad) return fail(CG_EINVAL, "null argument");
  if (nsteps < 0) return fail(CG_EINVAL, "nsteps must be >= 0");
  if (p->kin == CG_KIN_EXTERNAL) return fail(CG_EINVAL, "cg_run needs built-in kinetics");
  if (step0 < 0 || step0 + nsteps > INT_MAX) return fail(CG_EINVAL, "step index overflow");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (nsteps == 0) return CG_OK;
  if (int rc = ensure_workspace(p)) return rc;
  if (!p->padded) return run_steps(p, state, step0, nsteps, first_bad, s);
  int rc;
  if ((rc = repack(p, state, p->nl, p->S0, p->ld, s))) return rc;
  if ((rc = run_steps(p, p->S0, step0, nsteps, first_bad, s))) return rc;
  return repack(p, p->S0, p->ld, state, p->nl, s);
}

}  // extern "C"
