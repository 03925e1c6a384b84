// Disk front end fused into one persistent pass: F-build (stencil diffusion +
// kinetics) and the FFT theta propagator, W -> T = Q(Phi o Q^T F) row by row.
//
// For the disk the theta axis is the contiguous one, so a work item = RPB
// consecutive rho rows of BOTH species of one run (LPB = 2 RPB FFT lines).
// Its W rows i0-1 .. i0+RPB (both species) and its Phi rows arrive by 1-D
// bulk copies into one of two shared-memory buffers; the CTA evaluates F for
// its lines on the fly inside forward FFT phase A (F never goes to HBM) and
// runs the rest of the propagator (thetafft.cuh theta_tail) with Phi and the
// twiddles read from shared memory.  One CTA per SM walks the items
// persistently; item t+2's copies are issued as soon as item t has released
// its buffer, so HBM reads stay in flight under the FFT arithmetic.
// HBM traffic per step: read W (+2 halo rows per RPB) + write T, instead of
// read W + write F + read F + write T for fbuild_rows + theta_fast.
#pragma once

#include <type_traits>

#include "stencil.cuh"
#include "thetafft.cuh"

namespace cg {

#ifdef CURVIGPU_NO_REGSPLIT
constexpr bool kNoRegSplit = true;   // A/B build: split/merge through shared memory
#else
constexpr bool kNoRegSplit = false;
#endif

// One staged line of the disk front: pointers into shared-memory copies of
// the line's rho row (the rows above / below sit N doubles before / after it)
// and of the other species' row, plus the line's stencil coefficients.
struct DiskLine {
  const double* rowc;
  const double* rowo;
  double fa, fb, fc, fe;  // folded stencil row (fold_disk_row)
  double lift0, lift1;  // lift_addend() values
};

// The disk's diffusion row coeff * (a x0 + c x- + b x+ + d (off xl + diag x0 +
// off xr)) with the line's constants folded once per line: five FP64
// instructions per point instead of eight (the front is issue-bound).  The
// rounding differs from fbuild_rows_kernel's unfolded form by a few ulp of the
// largest term, as any reassociation of the reference's dense products does.
__device__ __forceinline__ void fold_disk_row(const RowCoef& rc, const CompCoef& kc, double& fa, double& fb, double& fc,
                                              double& fe) {
  fa = kc.coeff * (rc.a + rc.d * kc.th_diag);
  fb = kc.coeff * rc.b;
  fc = kc.coeff * rc.c;
  fe = kc.coeff * (rc.d * kc.th_off);
}

// F = coeff * (A_rho W + d_rho (W A_theta)) + g(W + lift) at the point pair
// (2kk, 2kk+1) of a line: one 16-byte load each for the row, the rows above
// and below and the other species, plus the two outer theta neighbours; the
// folded stencil row above plus the F-build kernel's reaction (bit for bit).
// CMP: the line's species (compile-time: the other species' reaction term is
// dead code).
template <int KIN, int CMP, int N>
__device__ __forceinline__ double2 disk_fpair(const DiskLine& L, const double (&kin)[9], int kk) {
  const int x = 2 * kk;
  const double* rowc = L.rowc;
  const double2 c2 = *reinterpret_cast<const double2*>(rowc + x);
  const double2 m2 = *reinterpret_cast<const double2*>(rowc - N + x);
  const double2 p2 = *reinterpret_cast<const double2*>(rowc + N + x);
  const double2 o2 = *reinterpret_cast<const double2*>(L.rowo + x);
  const double xl = rowc[x == 0 ? N - 1 : x - 1];
  const double xr = rowc[x + 2 == N ? 0 : x + 2];
  double2 out;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const double x0 = h ? c2.y : c2.x, xm = h ? m2.y : m2.x, xp = h ? p2.y : p2.x;
    const double left = h ? c2.x : xl, right = h ? xr : c2.y;
    double u = CMP == 0 ? x0 : (h ? o2.y : o2.x);
    double v = CMP == 0 ? (h ? o2.y : o2.x) : x0;
    u = __dadd_rn(u, L.lift0);  // lift_addend values: unconditional adds
    v = __dadd_rn(v, L.lift1);
    double g0, g1;
    reaction<KIN>(kin, u, v, g0, g1);
    // diffusion row accumulated onto the reaction term: four FMAs and one add
    const double val = fma(L.fa, x0, fma(L.fc, xm, fma(L.fb, xp, fma(L.fe, left + right, CMP == 0 ? g0 : g1))));
    if (h)
      out.y = val;
    else
      out.x = val;
  }
  return out;
}

template <int M1, int M2, int NBUF = 2, int NT = 256>
struct FusedDisk {
  using F = FastTheta<M1, M2, NT>;
  static constexpr int M = F::M;
  static constexpr int N = 2 * M;         // theta extent
  static constexpr int LPB = F::LPB;      // FFT lines per item
  static constexpr int RPB = LPB / 2;     // rho rows per item (2 species)
  static constexpr size_t wst = (size_t)2 * (RPB + 2) * N * sizeof(double);   // staged W rows
  static constexpr size_t sft = (size_t)LPB * F::SL * sizeof(double2);        // FFT tile (overlays W)
  static constexpr size_t reg_a = ((wst > sft ? wst : sft) + 127) / 128 * 128;
  static constexpr int PS = ((M + 1 + 7) / 8 * 8) % 16 == 0 ? (M + 1 + 7) / 8 * 8 + 8 : (M + 1 + 7) / 8 * 8;
  static constexpr size_t phib = (size_t)LPB * PS * sizeof(double);          // scaled Phi rows of the item
  static constexpr size_t buf = reg_a + (phib + 127) / 128 * 128;
  static constexpr size_t twb = (size_t)N * sizeof(double2);
  static constexpr size_t twab = (size_t)M * sizeof(double2);  // phase-A twiddles as [M1][M2]
  static constexpr size_t smem = 128 + twb + twab + NBUF * buf + 64;          // + alignment slack, barriers
  static_assert(RPB % 2 == 0, "Phi row blocks must stay 16-byte aligned");
};

// NBUF = 2: one CTA per SM, item t+2 prefetched into the buffer item t frees.
// NBUF = 1: two CTAs per SM (register-capped), each refilling its single
// buffer after its item; the other CTA's arithmetic covers the refill.
// NT = 64 (small grids): a quarter of the rows per item, four times the items
template <int M1, int M2, int KIN, int NBUF, int NT = 256>
__global__ void __launch_bounds__(NT, (3 - NBUF) * (256 / NT)) disk_ftheta_kernel(const ThetaParams tp, const StencilParams sp) {
  using F = FastTheta<M1, M2, NT>;
  using D = FusedDisk<M1, M2, NBUF, NT>;
  constexpr int M = F::M, TPL = F::TPL, RPB = D::RPB, N = D::N;
  extern __shared__ uint8_t fd_raw[];
  uint8_t* base_s = fd_raw + ((128u - (smem_u32(fd_raw) & 127u)) & 127u);  // stays a shared-space pointer
  double2* tw_s = reinterpret_cast<double2*>(base_s);
  double2* twa_s = reinterpret_cast<double2*>(base_s + D::twb);
  uint8_t* bufs = base_s + D::twb + D::twab;
  uint64_t* full = reinterpret_cast<uint64_t*>(bufs + NBUF * D::buf);  // [NBUF] item buffers, [2] twiddles

  const int n1 = sp.n1;
  const int per = n1 / RPB;
  const int items = sp.batch * per;
  const long long fsz = sp.npts;  // disk plans are never padded here
  const uint32_t row_bytes = N * sizeof(double);
  constexpr int PS = D::PS;  // == tp.phis_ld (checked at plan set-up)
  const uint32_t w_bytes = (uint32_t)(2 * (RPB + 2) * row_bytes);
  const uint32_t phi_bytes = (uint32_t)(2 * RPB * PS * sizeof(double));
  // Phi rows depend on (operator set, row block) only: with shared operators
  // (opb == 0) and a grid that is a multiple of the row blocks per run, a CTA
  // sees the same row block in every item, so each buffer copies them once
  int phi_rows[NBUF];
#pragma unroll
  for (int q = 0; q < NBUF; ++q) phi_rows[q] = -1;


  // copies of one item into buffer k (issued by one thread)
  auto issue = [&](int item, int k) {
    const int b = item / per;
    const int i0 = (item - b * per) * RPB;
    uint8_t* bb = bufs + k * D::buf;
    double* wst = reinterpret_cast<double*>(bb);
    double* phs = reinterpret_cast<double*>(bb + D::reg_a);
    const bool load_phi = !(sp.opb == 0 && phi_rows[k] == i0);
    phi_rows[k] = i0;
    mbar_arrive_expect_tx(&full[k], w_bytes + (load_phi ? phi_bytes : 0u));
    const int lo = i0 > 0 ? i0 - 1 : 0;
    const int hi = (i0 + RPB < n1) ? i0 + RPB : n1 - 1;
    for (int comp = 0; comp < 2; ++comp) {
      const double* src = sp.W + ((long long)b * 2 + comp) * fsz;
      double* dst = wst + (size_t)comp * (RPB + 2) * N;
      // staging row r <-> rho row i0 - 1 + r; missing halo rows are clamped
      // copies (their stencil coefficient is zero, they only need to be finite)
      bulk_load_1d(dst + (size_t)(lo - (i0 - 1)) * N, src + (long long)lo * N, (uint32_t)(hi - lo + 1) * row_bytes,
                   &full[k]);
      if (i0 == 0) bulk_load_1d(dst, src, row_bytes, &full[k]);
      if (i0 + RPB >= n1) bulk_load_1d(dst + (size_t)(RPB + 1) * N, src + (long long)(n1 - 1) * N, row_bytes, &full[k]);
      if (load_phi)
        bulk_load_1d(phs + (size_t)comp * RPB * PS, tp.phis + ((long long)(b * sp.opb + comp) * tp.nclass + i0) * PS,
                     (uint32_t)(RPB * PS * sizeof(double)), &full[k]);
    }
  };

  if (threadIdx.x == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(&full[2], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // twiddles are plan constants: loaded before waiting on the previous kernel
    mbar_arrive_expect_tx(&full[2], (uint32_t)D::twb);
    bulk_load_1d(tw_s, tp.tw, (uint32_t)D::twb, &full[2]);
  }
  pdl_wait();
  if (sp.step && blockIdx.x == 0 && threadIdx.x == 0) *sp.step += 1;
  if (threadIdx.x == 0) {
    if ((int)blockIdx.x < items) issue(blockIdx.x, 0);
    if (NBUF == 2 && (int)(blockIdx.x + gridDim.x) < items) issue(blockIdx.x + gridDim.x, 1);
  }

  const int tid = threadIdx.x;
  const int ln = tid / TPL, lt = tid - ln * TPL;
  const int comp = ln / RPB, rr = ln - comp * RPB;  // line = (species, interior row)
  const double lift0 = lift_addend(sp.lift[0]), lift1 = lift_addend(sp.lift[1]);
  mbar_wait(&full[2], 0);
  for (int i = threadIdx.x; i < M; i += blockDim.x) twa_s[i] = tw_s[2 * (i % M2) * (i / M2)];
  __syncthreads();

  int t = 0;
  for (int item = blockIdx.x; item < items; item += gridDim.x, ++t) {
    const int k = NBUF == 2 ? (t & 1) : 0;
    const int b = item / per;
    const int i0 = (item - b * per) * RPB;
    const int row = i0 + rr;
    const int f = b * 2 + comp;
    uint8_t* bb = bufs + k * D::buf;
    const double* Wst = reinterpret_cast<const double*>(bb);
    const double* phs = reinterpret_cast<const double*>(bb + D::reg_a);
    double kin[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) kin[q] = (q < sp.nparams) ? __ldg(sp.kin + (long long)b * sp.nparams + q) : 0.0;
    const int oc = b * sp.opb + comp;  // operator set of this (run, species)
    const CompCoef kc = comp_coef<0>(sp, oc, 0, N);
    RowCoef rc;
    {
      const double* bands = sp.rho_b + (long long)oc * 3 * n1;
      rc.a = __ldg(bands + row);
      rc.b = (row < n1 - 1) ? __ldg(bands + n1 + row) : 0.0;
      rc.c = (row > 0) ? __ldg(bands + 2 * n1 + row - 1) : 0.0;
      rc.d = __ldg(sp.d_rho + (long long)oc * n1 + row);
    }
    double fa, fb, fc, fe;
    fold_disk_row(rc, kc, fa, fb, fc, fe);
    mbar_wait(&full[k], NBUF == 2 ? ((t >> 1) & 1) : (t & 1));

    const double* Wc = Wst + (size_t)comp * (RPB + 2) * N;             // this species' staged rows
    const double* Wo = Wst + (size_t)(1 - comp) * (RPB + 2) * N;       // the other species'
    const double* rowc = Wc + (rr + 1) * N;
    // (this kernel keeps its own copy of disk_fpair's arithmetic as a lambda over
    // the item's locals: routing it through the DiskLine struct cost 4 % here,
    // 156.2 -> 162.3 us at config 5, profiles/r02_front_variants.txt)
    // F at the point pair (2kk, 2kk+1): one 16-byte load each for the row,
    // the rows above and below and the other species, plus the two outer
    // theta neighbours; the same arithmetic as disk_fpair, so the cluster step
    // kernel and this front produce the same F bit for bit.
    auto fpair = [&](auto compc, int kk) -> double2 {
      constexpr int CMP = decltype(compc)::value;  // species, compile-time: the other reaction term is dead code
      const int x = 2 * kk;
      const double2 c2 = *reinterpret_cast<const double2*>(rowc + x);
      const double2 m2 = *reinterpret_cast<const double2*>(rowc - N + x);
      const double2 p2 = *reinterpret_cast<const double2*>(rowc + N + x);
      const double2 o2 = *reinterpret_cast<const double2*>(Wo + (rr + 1) * N + x);
      const double xl = rowc[x == 0 ? N - 1 : x - 1];
      const double xr = rowc[x + 2 == N ? 0 : x + 2];
      double2 out;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double x0 = h ? c2.y : c2.x, xm = h ? m2.y : m2.x, xp = h ? p2.y : p2.x;
        const double left = h ? c2.x : xl, right = h ? xr : c2.y;
        double u = CMP == 0 ? x0 : (h ? o2.y : o2.x);
        double v = CMP == 0 ? (h ? o2.y : o2.x) : x0;
        u = __dadd_rn(u, lift0);
        v = __dadd_rn(v, lift1);
        double g0, g1;
        reaction<KIN>(kin, u, v, g0, g1);
        const double val = fma(fa, x0, fma(fc, xm, fma(fb, xp, fma(fe, left + right, CMP == 0 ? g0 : g1))));
        if (h)
          out.y = val;
        else
          out.x = val;
      }
      return out;
    };
    // ---- F on the fly, in forward phase A order (columns n2 = lt, lt + TPL, ...)
    double2 keepa[M2 / TPL][M1];
#pragma unroll
    for (int q = 0; q < M2 / TPL; ++q) {
      const int n2 = lt + q * TPL;
      if (comp == 0) {  // warp-uniform (a warp's lines share the species)
#pragma unroll
        for (int n1i = 0; n1i < M1; ++n1i) keepa[q][n1i] = fpair(std::integral_constant<int, 0>{}, n2 + M2 * n1i);
      } else {
#pragma unroll
        for (int n1i = 0; n1i < M1; ++n1i) keepa[q][n1i] = fpair(std::integral_constant<int, 1>{}, n2 + M2 * n1i);
      }
    }
    __syncthreads();  // every line's F is in registers: the W stage may be overwritten
    double2* S = reinterpret_cast<double2*>(bb) + ln * F::SL;
#pragma unroll
    for (int q = 0; q < M2 / TPL; ++q) phase_a<M1, M2, false, true, true>(keepa[q], S, lt + q * TPL, twa_s);
    const long long obase = (long long)f * fsz + (long long)row * N;
    theta_tail<M1, M2, false, true, !kNoRegSplit, 1>(tp, S, lt, phs + (size_t)ln * PS, tw_s, f, obase, 1, 1, twa_s);
    // release buffer k: generic-proxy accesses before the async-proxy refill
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0 && item + NBUF * (int)gridDim.x < items) issue(item + NBUF * gridDim.x, k);
  }
}

}  // namespace cg
