// Small disks: the whole split exponential Euler step (step_split_disk,
// integrators.py:202-207, inside the loop of run_simulation, :413-427) for
// MANY steps in ONE kernel, the state resident in the shared memory of one
// thread-block cluster.
//
// A 64 x 128 two-species disk (BASELINE config 1) is 128 KB of state and
// ~4 MFLOP per step: as separate kernels (fused front + rho GEMM) a step costs
// two launches, two grid drains and two trips through L2 (6.5 us per step,
// graph-replayed with PDL).  Here one cluster of NC = n_theta / 8 CTAs owns a
// run; every step is two phases, each waiting for the bytes the other phase
// pushes into its shared memory (async DSMEM stores that complete transaction
// counts on the receiver's mbarriers; a cluster-wide barrier per phase measured
// ~1270 clocks each, 38 % of the step):
//   A  (rows)     CTA r owns rho rows [4r, 4r + 4) of both species: F-build
//                 (stencil + kinetics, disk_fpair: one warp per line) from the
//                 W rows in its shared memory, then the theta FFT propagator
//                 (thetafft.cuh) of its lines, exactly the fused front's
//                 arithmetic;
//   B  (columns)  CTA r owns theta columns [8r, 8r + 8): phase A pushed its
//                 column slab of T into its shared memory over DSMEM
//                 (st.async.shared::cluster); it multiplies by phi1_rho (DMMA
//                 m8n8k4, the operator's A fragments held in registers), applies
//                 W + tau * Y with the divergence guard on its column slab of
//                 W -- which lives in REGISTERS for the whole run (the C
//                 fragment positions never change) -- and pushes the new rows
//                 (and halo copies) back to the row owners
//                 (st.shared::cluster) for the next step's phase A.
// Global memory is touched at the start (state, operators, Phi rows) and at the
// end (state).  The reference's semantics are kept: kinetics from the common
// state at t_n (phase A reads both species' rows of step n), the guard names
// the first bad step per field.
#pragma once

#include "fused_disk.cuh"
#include "resident.cuh"

namespace cg {

struct ClusterDiskParams {
  ThetaParams tp;     // phis / phis_ld / nclass / tw of the plan's theta stage
  StencilParams sp;   // rho bands, d_rho, theta stencil, coeff, lift, kinetics parameters
  const double* rop;  // [NO][n1][res_lds(n1 / 4)] phi1_rho, row-major, zero padded (resident layout)
  double* state;      // [B][2][n1][N], advanced in place
  int step0, nsteps;
  double tau, limit;
  int* first_bad;     // [B][2]
};

// 16-byte store into another CTA of the cluster that completes 16 bytes of
// transaction count on an mbarrier of that CTA: the receiver waits for its
// bytes instead of the whole cluster meeting at a barrier
__device__ __forceinline__ void st_async_cluster_f64x2(uint32_t cluster_addr, double a, double b, uint32_t cluster_bar) {
  asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(
                   cluster_addr),
               "d"(a), "d"(b), "r"(cluster_bar)
               : "memory");
}

template <int M1, int M2>
struct ClusterDisk {
  static constexpr int M = M1 * M2, N = 2 * M;
  static constexpr int NC = N / 8;           // CTAs per cluster: 8 theta columns each
  static constexpr int R = 4;                // rho rows per CTA
  static constexpr int N1 = R * NC;          // rho extent
  static constexpr int TPL = M1 < M2 ? M1 : M2;
  static constexpr int LINES = 2 * R;        // FFT lines per CTA (both species)
  static constexpr int FT = LINES * TPL;     // threads of phase A
  static constexpr int NT = 256;
  static constexpr int KSTEPS = N1 / 4, NBM = N1 / 8;
  static constexpr int LDS = res_lds(KSTEPS);
  static constexpr int PAIRS = 2 * NBM;      // (species, 8-row block) pairs of phase B
  static constexpr int PW = PAIRS / 8;       // per warp
  using F = FastTheta<M1, M2, FT>;
  static constexpr int PS = ((M + 1 + 7) / 8 * 8) % 16 == 0 ? (M + 1 + 7) / 8 * 8 + 8 : (M + 1 + 7) / 8 * 8;
  // shared memory (doubles unless noted)
  static constexpr size_t ops_b = 0;  // phi1_rho fragments live in registers for the whole run
  static constexpr size_t wrows_b = (size_t)2 * (R + 2) * N * 8;
  static constexpr size_t trows_b = (size_t)2 * R * N * 8;  // F rows of the CTA's lines (phase A input)
  static constexpr size_t tslab_b = (size_t)2 * N1 * 8 * 8;
  static constexpr size_t s_b = (size_t)LINES * F::SL * 16;
  static constexpr size_t phi_b = (size_t)LINES * PS * 8;
  static constexpr size_t tw_b = (size_t)N * 16 + (size_t)M * 16;
  static constexpr size_t smem = 128 + ops_b + wrows_b + trows_b + tslab_b + s_b + phi_b + tw_b + 16;
  static constexpr uint32_t tslab_tx = (uint32_t)tslab_b;  // bytes of T a CTA receives per step
  static_assert(PAIRS % 8 == 0 && PW >= 1, "phase B spreads (species, row block) pairs over 8 warps");
  static_assert(TPL == M1 && (TPL & (TPL - 1)) == 0, "register split layout (thetafft.cuh RS)");
  static_assert(!kTailCtaSync, "phase A runs on a subset of the CTA's warps");
};

template <int M1, int M2, int KIN>
__global__ void __launch_bounds__(256, 1) disk_cluster_kernel(const ClusterDiskParams p) {
  using D = ClusterDisk<M1, M2>;
  using F = typename D::F;
  constexpr int N = D::N, M = D::M, NC = D::NC, R = D::R, N1 = D::N1, TPL = D::TPL, LDS = D::LDS, PS = D::PS;
  constexpr int KSTEPS = D::KSTEPS, NBM = D::NBM, PW = D::PW;
  extern __shared__ uint8_t cd_raw[];
  uint8_t* base = cd_raw + ((128u - (smem_u32(cd_raw) & 127u)) & 127u);
  double* wrows = reinterpret_cast<double*>(base + D::ops_b);                       // [2][R + 2][N]
  double* frows = reinterpret_cast<double*>(base + D::ops_b + D::wrows_b);          // [2][R][N]
  double* tslab = reinterpret_cast<double*>(base + D::ops_b + D::wrows_b + D::trows_b);  // [2][N1][8]
  double2* S = reinterpret_cast<double2*>(base + D::ops_b + D::wrows_b + D::trows_b + D::tslab_b);
  double* phs = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(S) + D::s_b);  // [LINES][PS]
  double2* tw_s = reinterpret_cast<double2*>(reinterpret_cast<uint8_t*>(phs) + D::phi_b);  // [N]
  double2* twa_s = tw_s + N;                                                        // [M1][M2]
  uint64_t* bars = reinterpret_cast<uint64_t*>(twa_s + M);  // [0] T slab complete, [1] W rows complete

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = (int)cluster_ctarank();
  const int b = blockIdx.x / NC;  // run
  const int i0 = rank * R;
  const StencilParams& sp = p.sp;
  double* st = p.state + (long long)b * 2 * N1 * N;

  // ---------------- set-up: operators, Phi rows, twiddles, W rows (with halos), W column slab
  for (int idx = tid; idx < D::LINES * PS; idx += D::NT) {
    const int ln = idx / PS, j = idx - ln * PS;
    const int c = ln / R, row = i0 + ln % R;
    phs[idx] = __ldg(p.tp.phis + ((long long)(b * sp.opb + c) * p.tp.nclass + row) * PS + j);
  }
  for (int i = tid; i < N; i += D::NT) tw_s[i] = __ldg(p.tp.tw + i);
  for (int idx = tid; idx < 2 * (R + 2) * N; idx += D::NT) {
    const int c = idx / ((R + 2) * N), rem = idx - c * (R + 2) * N;
    const int lr = rem / N, x = rem - lr * N;
    int row = i0 - 1 + lr;  // missing halo rows: clamped copies (their stencil coefficient is zero)
    row = row < 0 ? 0 : (row > N1 - 1 ? N1 - 1 : row);
    wrows[idx] = st[((long long)c * N1 + row) * N + x];
  }
  __syncthreads();
  for (int i = tid; i < M; i += D::NT) twa_s[i] = tw_s[2 * (i % M2) * (i / M2)];

  // phase-B ownership: warp -> PW (species, 8-row block) pairs; lane -> rows 8 mb + g, columns 8 rank + 2t, +1
  const int g = lane >> 2, t = lane & 3;
  int pc[PW], pmb[PW];
  double wreg[PW][2];
#pragma unroll
  for (int q = 0; q < PW; ++q) {
    const int pair = warp * PW + q;
    pc[q] = pair / NBM;
    pmb[q] = pair - pc[q] * NBM;
    const double2 v = *reinterpret_cast<const double2*>(st + ((long long)pc[q] * N1 + 8 * pmb[q] + g) * N + 8 * rank + 2 * t);
    wreg[q][0] = v.x;
    wreg[q][1] = v.y;
  }
  // phi1_rho as DMMA A fragments L[8 mb + g][4 ks + t]: the same for every step, kept in registers
  double lf[PW][KSTEPS];
#pragma unroll
  for (int q = 0; q < PW; ++q) {
    const double* lrow = p.rop + ((size_t)(b * sp.opb + pc[q]) * N1 + 8 * pmb[q] + g) * LDS + t;
#pragma unroll
    for (int ks = 0; ks < KSTEPS; ++ks) lf[q][ks] = __ldg(lrow + 4 * ks);
  }

  // F-build ownership: warp -> line (species, row), lane -> point pairs; per-line constants
  static_assert(D::LINES == D::NT / 32, "one warp per line in the F-build");
  constexpr int PPL = (N / 2) / 32;  // point pairs per lane
  static_assert(PPL >= 1, "a line has at least 32 point pairs");
  const int fcomp = warp / R, frr = warp - fcomp * R, frow = i0 + frr;
  double kin[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) kin[q] = (q < sp.nparams) ? __ldg(sp.kin + (long long)b * sp.nparams + q) : 0.0;
  DiskLine dl;
  {
    const int oc = b * sp.opb + fcomp;
    const CompCoef kc = comp_coef<0>(sp, oc, 0, N);
    const double* bands = sp.rho_b + (long long)oc * 3 * N1;
    RowCoef rc;
    rc.a = __ldg(bands + frow);
    rc.b = (frow < N1 - 1) ? __ldg(bands + N1 + frow) : 0.0;
    rc.c = (frow > 0) ? __ldg(bands + 2 * N1 + frow - 1) : 0.0;
    rc.d = __ldg(sp.d_rho + (long long)oc * N1 + frow);
    fold_disk_row(rc, kc, dl.fa, dl.fb, dl.fc, dl.fe);
    dl.lift0 = lift_addend(sp.lift[0]);
    dl.lift1 = lift_addend(sp.lift[1]);
    dl.rowc = wrows + ((size_t)fcomp * (R + 2) + frr + 1) * N;
    dl.rowo = wrows + ((size_t)(1 - fcomp) * (R + 2) + frr + 1) * N;
  }
  // FFT ownership: thread -> (line, slot) for the first FT threads
  const bool fthread = tid < D::FT;
  const int ln = fthread ? tid / TPL : 0, lt = tid - ln * TPL;
  ThetaParams tpl = p.tp;
  tpl.cl_slab = smem_u32(tslab);  // phase A pushes its lines into the column owners' slabs
  tpl.cl_bar = smem_u32(&bars[0]);
  const uint32_t wrows_s = smem_u32(wrows), wbar_s = smem_u32(&bars[1]);
  // Per step a CTA receives its whole T slab (phase A of every row owner) and
  // its W rows with the halo copies (phase B of every column owner): two
  // transaction-counting mbarriers, armed for the next delivery as soon as the
  // previous one has been consumed.  No cluster-wide barrier inside the loop:
  // a T push into a slab follows the pusher's receipt of every CTA's W rows of
  // the previous step, which each CTA sends after its last read of that slab
  // (and the same with the roles swapped), so buffers are never overwritten
  // while they are read.
  const uint32_t wrows_tx = (uint32_t)((2 * R + (rank > 0 ? 2 : 0) + (rank < NC - 1 ? 2 : 0)) * N * 8);
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
    mbar_arrive_expect_tx(&bars[0], D::tslab_tx);
    mbar_arrive_expect_tx(&bars[1], wrows_tx);
  }
  __syncthreads();
  cluster_sync_all();  // every CTA of the cluster is set up before any remote access

  bool bad[PW];
#pragma unroll
  for (int q = 0; q < PW; ++q) bad[q] = false;
  int bad_step[PW];
#pragma unroll
  for (int q = 0; q < PW; ++q) bad_step[q] = 0x7fffffff;

#ifdef CURVIGPU_CLUSTER_TIMING
  long long tacc[6] = {0, 0, 0, 0, 0, 0};
#define CT_STAMP(i) { const long long now_ = clock64(); tacc[i] += now_ - tlast; tlast = now_; }
  long long tlast = clock64();
#else
#define CT_STAMP(i)
#endif
  for (int s = 0; s < p.nsteps; ++s) {
    // ---------------- phase A: F rows by all warps (one line each), then the theta
    // propagator of the lines on the first FT threads; results go straight into
    // the column owners' slabs over DSMEM
    if (s > 0) {
      mbar_wait_cluster(&bars[1], (uint32_t)((s - 1) & 1));  // this step's W rows (and halos) have arrived
      if (tid == 0) mbar_arrive_expect_tx(&bars[1], wrows_tx);
    }
    {
      double* fr = frows + (size_t)warp * N;
#pragma unroll
      for (int j = 0; j < PPL; ++j) {
        const int kk = lane + 32 * j;
        const double2 v = fcomp == 0 ? disk_fpair<KIN, 0, N>(dl, kin, kk) : disk_fpair<KIN, 1, N>(dl, kin, kk);
        *reinterpret_cast<double2*>(fr + 2 * kk) = v;
      }
    }
    CT_STAMP(0)
    __syncthreads();
    if (fthread) {
      double2 keepa[M2 / TPL][M1];
      const double2* fl = reinterpret_cast<const double2*>(frows + (size_t)ln * N);
#pragma unroll
      for (int q = 0; q < M2 / TPL; ++q) {
        const int n2 = lt + q * TPL;
#pragma unroll
        for (int n1i = 0; n1i < M1; ++n1i) keepa[q][n1i] = fl[n2 + M2 * n1i];
      }
      double2* Sl = S + ln * F::SL;
#pragma unroll
      for (int q = 0; q < M2 / TPL; ++q) phase_a<M1, M2, false, true, true>(keepa[q], Sl, lt + q * TPL, twa_s);
      theta_tail<M1, M2, false, true, true, 1, true>(tpl, Sl, lt, phs + (size_t)ln * PS, tw_s, 0, (long long)ln * N, 1, 1,
                                                      twa_s);
    }
    CT_STAMP(1)
    mbar_wait_cluster(&bars[0], (uint32_t)(s & 1));  // this CTA's column slab of T is complete
    if (tid == 0) mbar_arrive_expect_tx(&bars[0], D::tslab_tx);
    CT_STAMP(2)

    // Y = phi1_rho T on the column slab, W + tau * Y, guard, push to the row owners
    const int step = p.step0 + s + 1;
    double a0[PW], a1[PW];
#pragma unroll
    for (int q = 0; q < PW; ++q) a0[q] = a1[q] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KSTEPS; ++ks) {
#pragma unroll
      for (int q = 0; q < PW; ++q) {  // the warp's pairs are independent accumulation chains
        const double* xfrag = tslab + ((size_t)pc[q] * N1 + t) * 8 + g;
        dmma_8x8x4(a0[q], a1[q], lf[q][ks], xfrag[4 * ks * 8]);
      }
    }
#pragma unroll
    for (int q = 0; q < PW; ++q) {
      const int c = pc[q], mb = pmb[q];
      // W + tau*T rounded as the reference rounds it (no FMA contraction)
      const double v0 = __dadd_rn(wreg[q][0], __dmul_rn(p.tau, a0[q]));
      const double v1 = __dadd_rn(wreg[q][1], __dmul_rn(p.tau, a1[q]));
      wreg[q][0] = v0;
      wreg[q][1] = v1;
      if (!(fabs(v0) <= p.limit) || !(fabs(v1) <= p.limit)) {
        if (!bad[q]) bad_step[q] = step;
        bad[q] = true;
      }
      const int i = 8 * mb + g, owner = i / R, lr = i - owner * R;
      const uint32_t col = (uint32_t)((8 * rank + 2 * t) * 8);
      st_async_cluster_f64x2(mapa_shared(wrows_s + (uint32_t)((c * (R + 2) + lr + 1) * N * 8) + col, (uint32_t)owner), v0,
                             v1, mapa_shared(wbar_s, (uint32_t)owner));
      if (lr == 0 && owner > 0)  // bottom halo of the rows above
        st_async_cluster_f64x2(mapa_shared(wrows_s + (uint32_t)((c * (R + 2) + R + 1) * N * 8) + col,
                                           (uint32_t)(owner - 1)), v0, v1, mapa_shared(wbar_s, (uint32_t)(owner - 1)));
      if (lr == R - 1 && owner < NC - 1)  // top halo of the rows below
        st_async_cluster_f64x2(mapa_shared(wrows_s + (uint32_t)((c * (R + 2)) * N * 8) + col, (uint32_t)(owner + 1)), v0,
                               v1, mapa_shared(wbar_s, (uint32_t)(owner + 1)));
    }
    CT_STAMP(3)
  }
  cluster_sync_all();  // no CTA leaves while stores into its shared memory are in flight
#ifdef CURVIGPU_CLUSTER_TIMING
  if (tid == 0 && blockIdx.x < 16 && p.first_bad) {
    printf("cta %d: wait W + F %lld  fft + push %lld  wait T %lld  dmma + push %lld  (clk per step)\n", (int)blockIdx.x,
           tacc[0] / p.nsteps, tacc[1] / p.nsteps, tacc[2] / p.nsteps, tacc[3] / p.nsteps);
  }
#endif

  // ---------------- state back to global memory, first bad step per field
#pragma unroll
  for (int q = 0; q < PW; ++q) {
    *reinterpret_cast<double2*>(st + ((long long)pc[q] * N1 + 8 * pmb[q] + g) * N + 8 * rank + 2 * t) =
        make_double2(wreg[q][0], wreg[q][1]);
    int bs = bad_step[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bs = min(bs, __shfl_xor_sync(0xffffffffu, bs, o));
    if (lane == 0 && bs != 0x7fffffff) atomicMin(p.first_bad + b * 2 + pc[q], bs);
  }
}

}  // namespace cg
