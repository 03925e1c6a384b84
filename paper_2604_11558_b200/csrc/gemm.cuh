// Batched fp64 mu-mode product kernels for sm_100a.
//
// Every mu-mode product of the split exponential Euler step
// (integrators.py:202-236, tensor.py:31-49) is one of two GEMM shapes over
// the C-contiguous [field][n1][n2](n3) state, so no tensor is ever permuted:
//
//   TN  ("right" product, last mode):  Y[f](rows x N) = X[f](rows x K) . B^T
//       A = state rows (K contiguous), B = operator stored [N][K].
//   NN  ("left" product, first/middle mode): Y[f,s](M x N) = L(M x K) . X[f,s](K x N)
//       A = operator stored transposed [K][M], B = state slab [K][N].
//
// fp64 has no tcgen05 kind (ptxas rejects .kind::f64), so the tensor-core
// path is warp-level DMMA (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4), measured
// at 37.05 TFLOP/s on B200 (profiles/r01_fp64_peak.txt).  Operand tiles are
// staged by TMA (cp.async.bulk.tensor, 128B swizzle, zero fill out of bounds
// so n = 100 needs no host padding) into a STAGES-deep mbarrier ring fed by
// one producer warp; consumer warps read register fragments with
// conflict-free 8-byte shared loads (the fragment-to-row map below is chosen
// against the swizzle so every half-warp touches 16 distinct bank pairs).
//
// Epilogues are fused: plain store, Hadamard with a phi1 tensor (the "T *=
// Phi" of the steppers), or the final "W + tau * T" with the divergence
// guard of run_simulation (integrators.py:422-427).
//
// EPI_CHAIN (TN only, N = K <= BN): two products along the same mode in one
// pass, Y = ((X . B1^T) o Phi) . B2^T -- the ball's "T = F x3 V^-1 o Phi;
// T = T x3 V" (integrators.py:217-226).  A tile covers all N columns: after
// the first k loop the Phi-scaled accumulators go into the shared-memory
// tile (in the 128B-swizzled k-slice layout the TMA gives the A operand),
// the producer streams B2 (passed as mapW) slices into the same ring and
// the second k loop reads A from that tile.  The intermediate never goes to
// HBM; DMMAs on column blocks >= N and k steps >= K are skipped (they only
// add zeros), so n = 100 costs 104 x 100 instead of 128 x 112 per row.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace cg {

enum { VAR_TN = 0, VAR_NN = 1 };
enum { EPI_STORE = 0, EPI_PHI = 1, EPI_AXPY = 2, EPI_CHAIN = 3 };

struct GemmParams {
  int M, N, K;
  int nslab;   // batch item t -> field f = t / nslab, slab s = t % nslab
  int ncomp;   // component c = f % ncomp
  int nbatch;  // nfield * nslab
  int tiles_m, tiles_n;
  double* out;
  long long out_f, out_s;  // element strides of field / slab in out (and w)
  int ldc;
  const double* w;  // EPI_AXPY: previous state, same indexing as out
  const double* phi;  // EPI_PHI: phi + c*phi_c + s*phi_s + (m/phi_rdiv)*phi_m + n*phi_n
  long long phi_c, phi_s;
  int phi_m, phi_n, phi_rdiv;
  double tau, limit;
  int* first_bad;   // [nfield] smallest diverged step (atomicMin)
  const int* step;  // current step number (device)
  int tma_partial;  // partial tiles leave by the (clipping) bulk tensor store too
};

template <int BM, int BN>
struct StageBytes {
  static constexpr int A = BM * 128;  // BM x 16 doubles (TN) == BM/16 boxes of 16x16 (NN)
  static constexpr int B = BN * 128;
  static constexpr int total = A + B;
  static constexpr int epi = BM * BN * 8;  // epilogue tile: W in (axpy) / result out
};

template <int BM, int BN, int STAGES>
constexpr int gemm_smem_bytes() {
  return STAGES * StageBytes<BM, BN>::total + StageBytes<BM, BN>::epi + (2 * STAGES + 5) * 8 + 1024;
}

// Row permutation within an 8-row group used by the TN fragments: rows of a
// half-warp land on distinct 128B-swizzle phases.
__device__ __forceinline__ int perm8(int g) { return ((g & 3) << 1) | (g >> 2); }
// Row -> 16-byte-chunk XOR of the EPI_CHAIN intermediate tile (bits 1 and 2 of
// the row swapped): the epilogue's 16-byte stores (quarter-warps = row pairs
// r, r^2) and the second k loop's 8-byte fragment loads (half-warps = rows
// {0,2,4,6} / {1,3,5,7}) both hit distinct bank groups.  The TMA 128B swizzle
// (XOR = row) gave the stores 2-way conflicts per quarter-warp.
__device__ __forceinline__ int chain_xor(int r) { return (r & 1) | ((r & 2) << 1) | ((r & 4) >> 1); }

// mapA / mapB: operand tensor maps (128B swizzle).  mapW: previous state,
// mapO: output, both viewed as (N, M, slab, field) with a (BN, BM) box; the
// epilogue tile goes through shared memory: W arrives by TMA during the
// mainloop, results leave by a bulk tensor store.
//
// KS > 1 (small problems, fewer tiles than SMs): split-K over a cluster of KS
// CTAs.  Cluster rank r runs k slices [r KT / KS, (r+1) KT / KS) of every tile
// of the cluster; ranks 1.. write their partial accumulators into their own
// etile, rank 0 pulls them over DSMEM (ld.shared::cluster) and adds them in
// rank order -- a fixed summation order, so results stay bitwise
// reproducible -- then runs the epilogue alone.  Handshakes are mbarriers
// armed across the cluster (red_full in rank 0, red_empty in each peer).
template <int VAR, int BM, int BN, int WM, int WN, int STAGES, int EPI, int MINB, int KS = 1, bool RAG = false>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32 + 32, MINB)
    gemm_f64_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                    const __grid_constant__ CUtensorMap mapW, const __grid_constant__ CUtensorMap mapO,
                    const GemmParams p) {
  constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  constexpr int NCW = WARPS_M * WARPS_N;  // consumer warps
  constexpr int MT = WM / 8, NT = WN / 8;
  constexpr int SA = StageBytes<BM, BN>::A, SB = StageBytes<BM, BN>::B;
  constexpr int STAGE = SA + SB;
  constexpr int EPIB = StageBytes<BM, BN>::epi;
  static_assert(EPI != EPI_CHAIN || (VAR == VAR_TN && KS == 1), "chained products: TN, one CTA per tile");

  extern __shared__ uint8_t smem_raw[];
  // align by pointer arithmetic on the shared array (an integer round trip
  // would hide the address space and turn every fragment load into a generic LD)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  double* etile = reinterpret_cast<double*>(smem + STAGES * STAGE);  // [BM][BN]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE + EPIB);
  uint64_t* empty = full + STAGES;
  uint64_t* epi_full = empty + STAGES;   // W tile landed (axpy)
  uint64_t* epi_empty = epi_full + 1;    // previous tile's store has read etile
  uint64_t* red_full = epi_empty + 1;    // KS > 1, rank 0: the peers' partials are in their etiles
  uint64_t* red_empty = red_full + 1;    // KS > 1, peers: rank 0 has read this CTA's partial
  uint64_t* epi_ready = red_empty + 1;   // consumers have written the tile's results into etile

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KT = (p.K + 15) >> 4;
  const int ntiles = p.nbatch * p.tiles_m * p.tiles_n;
  int rank = 0, cid = blockIdx.x, ncl = gridDim.x, kt_begin = 0, kt_end = KT;
  if constexpr (KS > 1) {
    rank = (int)cluster_ctarank();
    cid = blockIdx.x / KS;
    ncl = gridDim.x / KS;
    kt_begin = rank * KT / KS;
    kt_end = (rank + 1) * KT / KS;
  }

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NCW);
    }
    mbar_init(epi_full, 1);
    mbar_init(epi_empty, 1);
    mbar_init(epi_ready, 1);
    if constexpr (KS > 1) {
      mbar_init(red_full, (KS - 1) * NCW);
      mbar_init(red_empty, NCW);
    }
    fence_barrier_init();
  }
  if (KS > 1)
    cluster_sync_all();  // barrier inits visible to the peers before any remote arrive
  else
    __syncthreads();
  pdl_wait();     // the previous kernel's outputs (X / W / step counter) are complete

  // Persistent static schedule: CTA b takes tiles b, b + grid, ...; tile ->
  // (batch item, m tile, n tile) with n fastest so neighbouring CTAs share the
  // A rows in L2.  The stage ring runs continuously across tiles, so the
  // producer streams the next tile's operands while consumers run the
  // epilogue of the current one.
  if (warp == NCW) {
    // ---------------- TMA producer ----------------
    // The producer lane also issues each tile's result store: it waits until
    // the consumers have written tile t-1 into etile (epi_ready), stores it
    // while tile t's first k slices are already in flight, and waits for the
    // store to have read etile before it reuses etile (W tile of the axpy
    // epilogue) or releases it (epi_empty).  The consumer warps go straight
    // from one tile's epilogue into the next mainloop.
    if (lane == 0) {
      tma_prefetch_desc(&mapA);
      tma_prefetch_desc(&mapB);
      int it = 0, tc = 0;
      int pm0 = 0, pn0 = 0, ps = 0, pf = 0;  // previous tile (pending store)
      auto store_prev = [&](int ptc) {
        mbar_wait(epi_ready, ptc & 1);
        // partial tiles (and every CHAIN tile: etile holds its intermediate) were stored from registers
        if (EPI != EPI_CHAIN && (p.tma_partial || ((pm0 + BM <= p.M) && (pn0 + BN <= p.N)))) {
          tma_store_4d(&mapO, etile, pn0, pm0, ps, pf);
          bulk_commit();
        }
      };
      for (int tile = KS > 1 ? cid : (int)blockIdx.x; tile < ntiles; tile += KS > 1 ? ncl : (int)gridDim.x, ++tc) {
        int r = tile;
        const int tn = r % p.tiles_n;
        r /= p.tiles_n;
        const int tm = r % p.tiles_m;
        const int t = r / p.tiles_m;
        const int f = t / p.nslab, s = t - f * p.nslab;
        const int c = f % p.ncomp;
        const int m0 = tm * BM, n0 = tn * BN;
        const int kb = KS > 1 ? kt_begin : 0, ke = KS > 1 ? kt_end : KT;
        const int qe = EPI == EPI_CHAIN ? ke + (ke - kb) : ke;  // CHAIN: then the B2 slices
        const int kstore = kb + (qe - kb < STAGES ? qe - kb : STAGES);  // slices issued before the previous store
        for (int q = kb; q < qe; ++q, ++it) {
          if (rank == 0 && tc > 0 && q == kstore) store_prev(tc - 1);
          const int st = it % STAGES;
          if (it >= STAGES) mbar_wait(&empty[st], ((it / STAGES) - 1) & 1);
          uint8_t* sa = smem + st * STAGE;
          uint8_t* sb = sa + SA;
          if (EPI == EPI_CHAIN && q >= ke) {
            mbar_arrive_expect_tx(&full[st], SB);
            tma_load_3d(sb, &mapW, &full[st], (q - ke) * 16, n0, c);
            continue;
          }
          const int kt = q;
          mbar_arrive_expect_tx(&full[st], STAGE);
          if (VAR == VAR_TN) {
            tma_load_3d(sa, &mapA, &full[st], kt * 16, m0, f);
            tma_load_3d(sb, &mapB, &full[st], kt * 16, n0, c);
          } else {
#pragma unroll
            for (int q = 0; q < BM / 16; ++q) tma_load_3d(sa + q * 2048, &mapA, &full[st], m0 + 16 * q, kt * 16, c);
#pragma unroll
            for (int q = 0; q < BN / 16; ++q) tma_load_4d(sb + q * 2048, &mapB, &full[st], n0 + 16 * q, kt * 16, s, f);
          }
        }
        if (rank == 0) {
          if (tc > 0) {
            if (kstore == qe) store_prev(tc - 1);
            bulk_wait_read0();      // the previous tile's store has read etile
            mbar_arrive(epi_empty);
          }
          if (EPI == EPI_AXPY) {  // W tile for this tile's epilogue
            mbar_arrive_expect_tx(epi_full, EPIB);
            tma_load_4d(etile, &mapW, epi_full, n0, m0, s, f);
          }
        }
        pm0 = m0;
        pn0 = n0;
        ps = s;
        pf = f;
      }
      if (rank == 0 && tc > 0) {
        store_prev(tc - 1);
        bulk_wait0();
      }
    }
    if (KS > 1) {
      __syncwarp();
      cluster_sync_all();  // no CTA leaves while a peer may still touch its shared memory
    }
    return;
  }

  // ---------------- DMMA consumers ----------------
  const int wy = warp / WARPS_N, wx = warp % WARPS_N;
  const int wm0 = wy * WM, wn0 = wx * WN;
  const int g = lane >> 2, tq = lane & 3;
  int step_now = 0;
  if (EPI == EPI_AXPY) step_now = *p.step;
  int it = 0, tc = 0;

  // EPI_CHAIN: Phi for chain_mid, loaded when the tile starts (its L2 latency
  // hides under the first k loop)
  auto chain_phi = [&](double2 (&ph)[MT][NT], int cc, int ss, int mb, int wm, int wn, int gg, int tqq) {
    const int cin8 = ((tqq & 1) << 2) | (tqq & 2);
    const int rin8 = perm8(gg);
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int ml = wm + i * 8 + rin8;
      const int m = mb + ml < p.M ? mb + ml : 0;
      const double* phirow = p.phi + cc * p.phi_c + ss * p.phi_s + (long long)(m / p.phi_rdiv) * p.phi_m;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int n = wn + j * 8 + cin8;
        const int nlo = n < p.N ? n : 0;
        const int nhi = n + 1 < p.N ? n + 1 : nlo;
        ph[i][j].x = __ldg(phirow + (long long)nlo * p.phi_n);
        ph[i][j].y = __ldg(phirow + (long long)nhi * p.phi_n);
      }
    }
  };
  // EPI_CHAIN, between the two k loops: the first product's accumulators,
  // times Phi, become the second product's A operand in etile ([KT][BM][16]
  // k slices, rows XOR-swizzled by chain_xor); accumulators reset.
  auto chain_mid = [&](double (&ac)[MT][NT][2], const double2 (&ph)[MT][NT], int tcn, int wm, int wn, int gg,
                       int tqq) {
    // No epi_empty wait here: the producer only signals it after issuing all
    // 2 KT slices of this tile, which needs this tile's second loop to drain
    // the ring (deadlock).  Nothing async touches etile in CHAIN mode (every
    // tile is stored from registers, there is no W tile), and the previous
    // tile's second loop finished reading it before the closing named barrier.
    (void)tcn;
    const int cin8 = ((tqq & 1) << 2) | (tqq & 2);
    const int rin8 = perm8(gg);
    const int kcols = KT * 16;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int ml = wm + i * 8 + rin8;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        // TN fragments hold columns perm8(2t), perm8(2t+1): swap with lane^2 into adjacent pairs
        const bool hi = (tqq & 2) != 0;
        const double send = hi ? ac[i][j][0] : ac[i][j][1];
        const double recv = __shfl_xor_sync(0xffffffffu, send, 2);
        double v0 = hi ? recv : ac[i][j][0];
        double v1 = hi ? ac[i][j][1] : recv;
        ac[i][j][0] = ac[i][j][1] = 0.0;
        const int n = wn + j * 8 + cin8;
        if (n >= kcols) continue;
        v0 *= ph[i][j].x;
        v1 *= ph[i][j].y;
        double* slab = etile + (n >> 4) * (BM * 16) + ml * 16;
        *reinterpret_cast<double2*>(slab + (((((n & 15) >> 1) ^ chain_xor(ml & 7))) << 1)) = make_double2(v0, v1);
      }
    }
    named_bar(1, NCW * 32);  // the whole intermediate tile is written before any warp reads it
  };

  for (int tile = KS > 1 ? cid : (int)blockIdx.x; tile < ntiles; tile += KS > 1 ? ncl : (int)gridDim.x, ++tc) {
    int r = tile;
    const int tn = r % p.tiles_n;
    r /= p.tiles_n;
    const int tm = r % p.tiles_m;
    const int t = r / p.tiles_m;
    const int f = t / p.nslab, s = t - f * p.nslab;
    const int c = f % p.ncomp;
    const int m0 = tm * BM, n0 = tn * BN;

    double acc[MT][NT][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    double2 phc[MT][NT];
    if constexpr (EPI == EPI_CHAIN) chain_phi(phc, c, s, m0, wm0, wn0, g, tq);
    const int kend = KS > 1 ? kt_end : KT;
    const int qend = EPI == EPI_CHAIN ? 2 * KT : kend;
    for (int q = KS > 1 ? kt_begin : 0; q < qend; ++q, ++it) {
      if (EPI == EPI_CHAIN && q == KT) chain_mid(acc, phc, tc, wm0, wn0, g, tq);
      const int kt = (EPI == EPI_CHAIN && q >= KT) ? q - KT : q;
      const int st = it % STAGES;
      mbar_wait(&full[st], (it / STAGES) & 1);
      // mma.sync.aligned needs the whole warp converged: lanes leave the
      // try_wait poll independently, and lane 0 may still be in the
      // previous tile's store block
      __syncwarp();
      const double* sa = (EPI == EPI_CHAIN && q >= KT) ? etile + kt * BM * 16
                                                        : reinterpret_cast<const double*>(smem + st * STAGE);
      const double* sb = reinterpret_cast<const double*>(smem + st * STAGE + SA);
      if (VAR == VAR_TN) {
        const int pg = perm8(g);
        const int pga = (EPI == EPI_CHAIN && q >= KT) ? chain_xor(pg) : pg;  // A from the intermediate tile
        // CHAIN: k steps past K and column blocks past N only add zeros.  The
        // skips are warp-uniform branches to code with a compile-time count of
        // live column blocks NL (predicated-off DMMAs would still issue).
        const int kmax = EPI == EPI_CHAIN ? min(16, p.K - kt * 16) : 16;
        auto slice = [&](auto nlive) {
          constexpr int NL = decltype(nlive)::value;
#pragma unroll
          for (int kk = 0; kk < 16; kk += 4) {
            if (EPI == EPI_CHAIN && kk >= kmax) break;
            const int col = kk + tq;
            const int off = ((((col >> 1) ^ pg)) << 1) | (col & 1);
            const int offa = ((((col >> 1) ^ pga)) << 1) | (col & 1);
            double a[MT], b[NL];
#pragma unroll
            for (int i = 0; i < MT; ++i) a[i] = sa[(wm0 + i * 8 + pg) * 16 + offa];
#pragma unroll
            for (int j = 0; j < NL; ++j) b[j] = sb[(wn0 + j * 8 + pg) * 16 + off];
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
              for (int j = 0; j < NL; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
          }
        };
        if constexpr (EPI == EPI_CHAIN) {
          static_assert(NT == 4, "chain tile: four 8-column blocks per warp");
          const int nl = (p.N - wn0 + 7) >> 3;  // live column blocks of this warp
          if (nl >= 4)
            slice(std::integral_constant<int, 4>{});
          else if (nl == 3)
            slice(std::integral_constant<int, 3>{});
          else if (nl == 2)
            slice(std::integral_constant<int, 2>{});
          else if (nl == 1)
            slice(std::integral_constant<int, 1>{});
        } else {
          slice(std::integral_constant<int, NT>{});
        }
      } else {
        // RAG (a separate instantiation for NN stages whose M or K is not a
        // tile multiple, e.g. n = 100): skip what only adds zeros -- operator
        // rows past M (the last m tile) and the k8 half-slice past K -- by
        // warp-uniform branches to code with a compile-time count of live
        // 8-row blocks ML (predicated-off DMMAs would still issue).  Keeping it
        // out of the plain kernels keeps their code unchanged (measured: the
        // extra paths in one kernel cost the aligned stages 4-8 %).
        constexpr bool SKIP = RAG;
        auto slice = [&](auto mlive, auto kskip) {
          constexpr int ML = decltype(mlive)::value;
#pragma unroll
          for (int k8 = 0; k8 < 16; k8 += 8) {
            if (decltype(kskip)::value && kt * 16 + k8 >= p.K) break;
#pragma unroll
            for (int sub = 0; sub < 2; ++sub) {
              const int k = k8 + 2 * tq + sub;
              const int kx = k & 7;
              double a[ML > 0 ? ML : 1], b[NT];
#pragma unroll
              for (int i = 0; i < ML; ++i) {
                const int m = wm0 + i * 8 + g;
                const int mm = m & 15;
                a[i] = sa[(m >> 4) * 256 + k * 16 + ((((mm >> 1) ^ kx)) << 1) + (mm & 1)];
              }
#pragma unroll
              for (int j = 0; j < NT; ++j) {
                const int n = wn0 + j * 8 + g;
                const int nn = n & 15;
                b[j] = sb[(n >> 4) * 256 + k * 16 + ((((nn >> 1) ^ kx)) << 1) + (nn & 1)];
              }
#pragma unroll
              for (int i = 0; i < ML; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
            }
          }
        };
        using KS_ON = std::true_type;
        using KS_OFF = std::false_type;
        if constexpr (SKIP) {
          const int ml = (p.M - m0 - wm0 + 7) >> 3;  // live 8-row blocks of this warp
          // warp-uniform dispatch to the instantiation with min(ml, MT) live blocks
          auto pick = [&](auto self, auto live) -> void {
            constexpr int V = decltype(live)::value;
            if constexpr (V >= 1) {
              if (ml >= V)
                slice(std::integral_constant<int, V>{}, KS_ON{});
              else
                self(self, std::integral_constant<int, V - 1>{});
            }
          };
          pick(pick, std::integral_constant<int, MT>{});
        } else {
          slice(std::integral_constant<int, MT>{}, KS_OFF{});
        }
      }
      // Generic-proxy reads (the fragment LDS) of a stage followed by the
      // producer's async-proxy write (TMA refill) are a cross-proxy WAR: each
      // thread fences its reads into the async proxy before the release.
      // Without the fence the refill raced the slice's last fragment loads
      // (one 8x8 accumulator fragment of warp 0 differed in ~1 of 200 runs;
      // a register dependency on the last DMMA made it worse, delaying the
      // release by a slice hid it at a 3% cost; profiles/r01_partial_tile_race.md).
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }

    if (KS > 1) {
      // ---------------- split-K reduction over DSMEM (fixed rank order) ----------------
      // partial layout [warp][i][j][lane] (double2): lane-contiguous 16-byte accesses
      const uint32_t etile_s = smem_u32(etile);
      if (rank != 0) {
        if (tc > 0) mbar_wait_cluster(red_empty, (tc - 1) & 1);  // rank 0 has read the previous partial
        __syncwarp();
        double2* part = reinterpret_cast<double2*>(etile);
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j)
            part[((warp * MT + i) * NT + j) * 32 + lane] = make_double2(acc[i][j][0], acc[i][j][1]);
        fence_acq_rel_cluster();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(red_full), 0));
        continue;  // rank 0 runs the epilogue
      }
      mbar_wait_cluster(red_full, tc & 1);
      __syncwarp();
#pragma unroll 1
      for (int q = 1; q < KS; ++q) {
        const uint32_t peer = mapa_shared(etile_s, (uint32_t)q);
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const double2 v = ld_shared_cluster_f64x2(peer + 16u * (((warp * MT + i) * NT + j) * 32 + lane));
            acc[i][j][0] += v.x;
            acc[i][j][1] += v.y;
          }
      }
      fence_acq_rel_cluster();
      __syncwarp();
      if (lane == 0)
        for (int q = 1; q < KS; ++q) mbar_arrive_cluster(mapa_shared(smem_u32(red_empty), (uint32_t)q));
    }

    // ---------------- fused epilogue through the shared-memory tile ----------------
    int col_in8;
    if (VAR == VAR_TN) {
      // thread holds cols perm8(2t), perm8(2t+1) = {0,2},{4,6},{1,3},{5,7};
      // swap with lane^2 so each thread owns an adjacent pair.
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const bool hi = (tq & 2) != 0;
          const double send = hi ? acc[i][j][0] : acc[i][j][1];
          const double recv = __shfl_xor_sync(0xffffffffu, send, 2);
          if (hi)
            acc[i][j][0] = recv;
          else
            acc[i][j][1] = recv;
        }
      col_in8 = ((tq & 1) << 2) | (tq & 2);
    } else {
      col_in8 = 2 * tq;
    }
    const int row_in8 = (VAR == VAR_TN) ? perm8(g) : g;
    // Epilogue column rotation: odd row groups take fragment j^1 in step j, so
    // a quarter-warp's 16-byte accesses to the dense [BM][BN] tile cover all
    // eight bank groups (plain order: every row group hit the same banks,
    // 8-way conflicts on the W reads and the staging writes).
    static_assert(NT % 2 == 0, "epilogue rotation pairs fragments j and j^1");
    const bool rot = (g & 1) != 0;

    if (EPI == EPI_AXPY)
      mbar_wait(epi_full, tc & 1);  // W tile is in etile
    else if (EPI != EPI_CHAIN && tc > 0)
      mbar_wait(epi_empty, (tc - 1) & 1);  // previous tile's store has read etile
    bool bad = false;
    // Partial tiles (the last m or n tile of an extent that BM/BN do not
    // divide) are written straight from registers with bounds checks: the
    // clipped bulk tensor store of such tiles measured nondeterministic on
    // B200 with two CTAs per SM (tools/chain_dbg2.py); full tiles use TMA.
    // CHAIN: etile holds the intermediate other warps may still be reading
    const bool full_tile = EPI != EPI_CHAIN && (p.tma_partial || ((m0 + BM <= p.M) && (n0 + BN <= p.N)));
    // Phi1 operands for EPI_PHI (L2-resident table), all loads in flight per row group
    constexpr int EC = (MINB >= 2 && MT > 2 && MT % 2 == 0) ? MT / 2 : MT;
#pragma unroll
    for (int i0 = 0; i0 < MT; i0 += EC) {
      double2 ph[EC][NT];
      if (EPI == EPI_PHI) {
#pragma unroll
        for (int ii = 0; ii < EC; ++ii) {
          int m = m0 + wm0 + (i0 + ii) * 8 + row_in8;
          if (m >= p.M) m = 0;
          const double* phirow = p.phi + c * p.phi_c + s * p.phi_s + (long long)(m / p.phi_rdiv) * p.phi_m;
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            int n = n0 + wn0 + (j ^ (int)rot) * 8 + col_in8;
            if (n >= p.N) n = 0;
            const int n_hi = (n + 1 < p.N) ? n + 1 : n;  // odd N: the pair's second column is padding
            ph[ii][j].x = __ldg(phirow + (long long)n * p.phi_n);
            ph[ii][j].y = __ldg(phirow + (long long)n_hi * p.phi_n);
          }
        }
      }
#pragma unroll
      for (int ii = 0; ii < EC; ++ii) {
        const int i = i0 + ii;
        const int ml = wm0 + i * 8 + row_in8;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const int nl = wn0 + (j ^ (int)rot) * 8 + col_in8;
          double2* slot = reinterpret_cast<double2*>(etile + ml * BN + nl);
          double v0 = rot ? acc[i][j ^ 1][0] : acc[i][j][0];
          double v1 = rot ? acc[i][j ^ 1][1] : acc[i][j][1];
          if (EPI == EPI_PHI) {
            v0 *= ph[ii][j].x;
            v1 *= ph[ii][j].y;
          } else if (EPI == EPI_AXPY) {
            const double2 w2 = *slot;
            // W + tau*T rounded as the reference rounds it (no FMA contraction)
            v0 = __dadd_rn(w2.x, __dmul_rn(p.tau, v0));
            v1 = __dadd_rn(w2.y, __dmul_rn(p.tau, v1));
            bad |= !(fabs(v0) <= p.limit) || !(fabs(v1) <= p.limit);  // OOB entries are 0
          }
          if (full_tile) {
            *slot = make_double2(v0, v1);
          } else {
            const int m = m0 + ml, n = n0 + nl;
            if (m < p.M && n < p.N)
              *reinterpret_cast<double2*>(p.out + (long long)f * p.out_f + (long long)s * p.out_s +
                                          (long long)m * p.ldc + n) = make_double2(v0, v1);
          }
        }
      }
    }
    fence_proxy_async_smem();
    named_bar(1, NCW * 32);
    if (threadIdx.x == 0) mbar_arrive(epi_ready);  // the producer lane stores the tile
    __syncwarp();  // reconverge warp 0 before the next tile's MMAs
    if (EPI == EPI_AXPY) {
      if (__any_sync(0xffffffffu, bad) && lane == 0) atomicMin(p.first_bad + f, step_now);
    }
  }
  if (KS > 1) {
    __syncwarp();
    cluster_sync_all();
  }
}

}  // namespace cg
