// Disk front end fused into one pass: F-build (stencil diffusion + kinetics)
// and the FFT theta propagator, W -> T = Q(Phi o Q^T F) row by row.
//
// For the disk the theta axis is the contiguous one, so a CTA that owns RPB
// consecutive rho rows of BOTH species of one run can stage W_u, W_v rows
// i0-1 .. i0+RPB in shared memory, evaluate F for its rows on the fly inside
// forward FFT phase A (F is never written to HBM), and run the rest of the
// propagator (thetafft.cuh theta_tail).  HBM traffic per step drops from
// read W + write F + read F + write T to read W + write T.
#pragma once

#include "stencil.cuh"
#include "thetafft.cuh"

namespace cg {

template <int M1, int M2>
struct FusedDisk {
  using F = FastTheta<M1, M2>;
  static constexpr int RPB = F::LPB / 2;  // rho rows per CTA (lines = 2 species x RPB rows)
  static constexpr int N = 2 * F::M;      // theta extent
  static constexpr size_t stage_bytes = (size_t)2 * (RPB + 2) * N * sizeof(double);
  static constexpr size_t smem = F::smem + stage_bytes;
};

template <int M1, int M2, int KIN>
__global__ void __launch_bounds__(256) disk_ftheta_kernel(const ThetaParams tp, const StencilParams sp) {
  using F = FastTheta<M1, M2>;
  using D = FusedDisk<M1, M2>;
  constexpr int M = F::M, TPL = F::TPL, RPB = D::RPB, N = D::N;
  extern __shared__ double2 fd_smem[];
  double2* Sbase = fd_smem;
  double* Wst = reinterpret_cast<double*>(fd_smem + F::LPB * F::SL);  // [2][RPB+2][N]

  if (sp.step && blockIdx.x == 0 && threadIdx.x == 0) *sp.step += 1;
  const int n1 = sp.n1;
  const int per = n1 / RPB;
  const int b = blockIdx.x / per;
  const int i0 = (blockIdx.x - b * per) * RPB;
  const long long run = (long long)b * 2 * sp.npts;

  // ---- stage W_u, W_v rows i0-1 .. i0+RPB (clamped rows are never used by the stencil)
  for (int idx = threadIdx.x; idx < 2 * (RPB + 2) * (N / 2); idx += blockDim.x) {
    const int comp = idx / ((RPB + 2) * (N / 2));
    const int rem = idx - comp * (RPB + 2) * (N / 2);
    const int r = rem / (N / 2), k = rem - r * (N / 2);
    const int i = min(max(i0 - 1 + r, 0), n1 - 1);
    const double2 v =
        __ldg(reinterpret_cast<const double2*>(sp.W + run + (long long)comp * sp.npts + (long long)i * N) + k);
    reinterpret_cast<double2*>(Wst + (comp * (RPB + 2) + r) * N)[k] = v;
  }
  __syncthreads();

  const int tid = threadIdx.x;
  const int ln = tid / TPL, lt = tid - ln * TPL;
  const int comp = ln / RPB, rr = ln - comp * RPB;  // line = (species, interior row)
  const int row = i0 + rr;
  const int f = b * 2 + comp;
  const long long base = (long long)f * sp.npts + (long long)row * N;
  double2* S = Sbase + ln * F::SL;
  const double* kin = sp.kin + (long long)b * sp.nparams;
  const double* Wc = Wst + comp * (RPB + 2) * N;
  const double* Wu = Wst;
  const double* Wv = Wst + (RPB + 2) * N;

  const CompCoef kc = comp_coef<0>(sp, comp, 0, N);
  RowCoef rc;
  {
    const double* bands = sp.rho_b + (long long)comp * 3 * n1;
    rc.a = bands[row];
    rc.b = (row < n1 - 1) ? bands[n1 + row] : 0.0;
    rc.c = (row > 0) ? bands[2 * n1 + row - 1] : 0.0;
    rc.d = sp.d_rho[comp * n1 + row];
  }
  auto fval = [&](int t) -> double {
    double u = Wu[(rr + 1) * N + t], v = Wv[(rr + 1) * N + t];
    if (sp.lift[0] != 0.0) u = __dadd_rn(u, sp.lift[0]);
    if (sp.lift[1] != 0.0) v = __dadd_rn(v, sp.lift[1]);
    double g0, g1;
    reaction<KIN>(kin, u, v, g0, g1);
    const double d = kc.coeff * diffusion_rows<0>(kc, rc, Wc, rr, t, N);
    return __dadd_rn(d, comp == 0 ? g0 : g1);
  };

  // ---- forward phase A with F evaluated on the fly (columns n2 = lt, lt + TPL, ...)
  double2 keepa[M2 / TPL][M1];
#pragma unroll
  for (int q = 0; q < M2 / TPL; ++q) {
    const int n2 = lt + q * TPL;
#pragma unroll
    for (int n1i = 0; n1i < M1; ++n1i) {
      const int k = n2 + M2 * n1i;
      keepa[q][n1i] = make_double2(fval(2 * k), fval(2 * k + 1));
    }
  }
#pragma unroll
  for (int q = 0; q < M2 / TPL; ++q) phase_a<M1, M2, false>(keepa[q], S, lt + q * TPL, tp.tw);
  theta_tail<M1, M2, false>(tp, S, lt, row, 0, comp, f, base, 1, 1);
}

}  // namespace cg
