// F-build kernel: F = coeff * M W + g(W + lift) for every field of every run.
//
// The reference forms the diffusion action with DENSE n x n matrices
// (apply_diffusion, integrators.py:176-199: A_rho @ W, W @ A_theta, ...) even
// though every 1-D operator is tridiagonal or circulant-tridiagonal
// (operators.py:37-88).  Here it is a 3-point stencil per axis - a single
// HBM-bound pass that reads each field once and writes F once - with the
// kinetics closure (models.py:284-319, :528-532 and the BASELINE custom
// closures) evaluated in the same pass from the common state, so all
// components see the state at t_n (integrators.py:414).
#pragma once

#include "common.cuh"

namespace cg {

enum { KIN_EXTERNAL = 0, KIN_SCHNAKENBERG = 1, KIN_BRUSSELATOR = 2, KIN_GRAY_SCOTT = 3,
       KIN_BVAM_ETA = 4, KIN_BVAM = 5, KIN_DIB = 6 };

struct StencilParams {
  int geometry;
  int n1, n2, n3;
  int ncomp, batch;
  long long npts;  // points per field
  const double* rho_b;  // [C][3][n_rho] a, b, c
  const double* phi_b;  // [C][3][n_phi]
  const double* z_b;    // [C][3][n_z]
  const double* th;     // [C][2] diag, off
  const double* d_rho;  // [C][n_rho]
  const double* d_phi;  // [C][n_phi]
  const double* coeff;  // [C]
  const double* lift;   // [C]
  const double* kin;    // [B][P]
  int nparams;
  const double* W;  // [B][C][pts]
  const double* G;  // external reaction terms (KIN_EXTERNAL) or nullptr
  double* F;        // [B][C][pts]
  int with_diffusion;  // 0: F = g only (cg_kinetics)
  int with_reaction;   // 0: F = coeff M W only (cg_apply_diffusion)
  int* step;           // incremented once per launch when non-null
};

// y = c_{i-1} x_{i-1} + a_i x_i + b_i x_{i+1} along one axis of extent n.
__device__ __forceinline__ double tri_axis(const double* bands, int n, int i, const double* x, long long stride) {
  const double* a = bands;
  const double* b = bands + n;
  const double* c = bands + 2 * n;
  double y = a[i] * x[0];
  if (i > 0) y += c[i - 1] * x[-stride];
  if (i < n - 1) y += b[i] * x[stride];
  return y;
}

// periodic: off x_{i-1} + diag x_i + off x_{i+1}
__device__ __forceinline__ double circ_axis(const double* th, int n, int i, const double* x, long long stride) {
  const long long dm = (i == 0) ? (long long)(n - 1) * stride : -stride;
  const long long dp = (i == n - 1) ? -(long long)(n - 1) * stride : stride;
  return th[1] * x[dm] + th[0] * x[0] + th[1] * x[dp];
}

template <int GEOM>
__device__ __forceinline__ double diffusion_at(const StencilParams& p, int c, const double* x, int i, int j, int l) {
  // x points at W[b][c][i][j][l]
  if (GEOM == 0) {  // disk (rho, theta)
    const double r = tri_axis(p.rho_b + (long long)c * 3 * p.n1, p.n1, i, x, p.n2);
    const double q = circ_axis(p.th + 2 * c, p.n2, j, x, 1);
    return r + p.d_rho[c * p.n1 + i] * q;
  } else if (GEOM == 1) {  // sphere (theta periodic, phi polar)
    const double q = circ_axis(p.th + 2 * c, p.n1, i, x, p.n2);
    const double r = tri_axis(p.phi_b + (long long)c * 3 * p.n2, p.n2, j, x, 1);
    return q * p.d_phi[c * p.n2 + j] + r;
  } else if (GEOM == 2) {  // ball (rho, theta periodic, phi polar)
    const long long s1 = (long long)p.n2 * p.n3;
    const double r = tri_axis(p.rho_b + (long long)c * 3 * p.n1, p.n1, i, x, s1);
    const double q = circ_axis(p.th + 2 * c, p.n2, j, x, p.n3);
    const double ph = tri_axis(p.phi_b + (long long)c * 3 * p.n3, p.n3, l, x, 1);
    const double dr = p.d_rho[c * p.n1 + i];
    return r + (dr * q) * p.d_phi[c * p.n3 + l] + dr * ph;
  } else {  // cylinder (rho, theta periodic, z)
    const long long s1 = (long long)p.n2 * p.n3;
    const double r = tri_axis(p.rho_b + (long long)c * 3 * p.n1, p.n1, i, x, s1);
    const double q = circ_axis(p.th + 2 * c, p.n2, j, x, p.n3);
    const double z = tri_axis(p.z_b + (long long)c * 3 * p.n3, p.n3, l, x, 1);
    return r + p.d_rho[c * p.n1 + i] * q + z;
  }
}

// Two-species reaction, rounded operation by operation in the reference's
// NumPy order (no FMA contraction), so g matches the oracle bit for bit.
template <int KIN>
__device__ __forceinline__ void reaction(const double* k, double u, double v, double& gu, double& gv) {
#define MUL __dmul_rn
#define ADD __dadd_rn
#define SUB __dsub_rn
  if (KIN == KIN_SCHNAKENBERG) {  // gamma, a, b
    const double uuv = MUL(MUL(u, u), v);
    gu = MUL(k[0], ADD(SUB(k[1], u), uuv));
    gv = MUL(k[0], SUB(k[2], uuv));
  } else if (KIN == KIN_BRUSSELATOR) {  // A, B
    const double uuv = MUL(MUL(u, u), v);
    gu = ADD(SUB(k[0], MUL(ADD(k[1], 1.0), u)), uuv);
    gv = SUB(MUL(k[1], u), uuv);
  } else if (KIN == KIN_GRAY_SCOTT) {  // F, k
    const double uvv = MUL(MUL(u, v), v);
    gu = ADD(-uvv, MUL(k[0], SUB(1.0, u)));
    gv = SUB(uvv, MUL(ADD(k[0], k[1]), v));
  } else if (KIN == KIN_BVAM_ETA) {  // eta, a, b, h, C
    const double uv = MUL(u, v);
    const double uvv = MUL(uv, v);
    gu = MUL(k[0], SUB(SUB(ADD(u, MUL(k[1], v)), MUL(k[4], uv)), uvv));
    gv = MUL(k[0], ADD(ADD(ADD(MUL(k[2], v), MUL(k[3], u)), MUL(k[4], uv)), uvv));
  } else if (KIN == KIN_BVAM) {  // alpha1, alpha2, alpha3, beta1, beta2 (models.py:284-290)
    const double a1 = k[0], a2 = k[1], a3 = k[2], b1 = k[3], b2 = k[4];
    gu = ADD(MUL(MUL(a1, u), SUB(1.0, MUL(a2, MUL(v, v)))), MUL(v, SUB(1.0, MUL(a3, u))));
    const double r = __ddiv_rn(MUL(a1, a2), b1);
    gv = ADD(MUL(MUL(b1, v), ADD(1.0, MUL(MUL(r, u), v))), MUL(u, ADD(b2, MUL(a3, v))));
  } else if (KIN == KIN_DIB) {  // zeta1..5, eta1, eta2, eta3, eta5 (models.py:299-319)
    const double z1 = k[0], z2 = k[1], z3 = k[2], z4 = k[3], z5 = k[4];
    const double e1 = k[5], e2 = k[6], e3 = k[7], e5 = k[8];
    // eta4 from the equilibrium constraint (models.py:299-308, beta2 absent)
    const double e4 = __ddiv_rn(MUL(MUL(e1, SUB(1.0, z5)), ADD(SUB(1.0, e3), MUL(e3, z5))),
                                MUL(z5, ADD(1.0, MUL(e3, z5))));
    const double r = u, s = v;
    const double pr = SUB(SUB(MUL(MUL(z2, SUB(1.0, s)), r), MUL(z3, MUL(MUL(r, r), r))), MUL(z4, SUB(s, z5)));
    const double one_s = SUB(1.0, s);
    const double q1 = MUL(MUL(MUL(e1, ADD(1.0, MUL(e2, r))), one_s), SUB(1.0, MUL(e3, one_s)));
    const double q2 = MUL(MUL(MUL(e4, s), ADD(1.0, MUL(e3, s))), ADD(1.0, MUL(e5, r)));
    gu = MUL(z1, pr);
    gv = MUL(z1, SUB(q1, q2));
  } else {
    gu = 0.0;
    gv = 0.0;
  }
#undef MUL
#undef ADD
#undef SUB
}

// ---------------------------------------------------------------------------
// Register-blocked F-build.  Lanes run along the contiguous axis (coalesced
// loads/stores; in-row neighbours come from warp shuffles), each thread walks
// RB consecutive points of the first axis with a 3-value sliding window, so
// every W value is read from memory about once (the naive one-thread-per-
// point kernel re-read 5-7 neighbours per point and was L1-bound).
//   grid = (ceil(n1 / RB), 3-D ? n2 : 1, batch), block = round32(n_last)
// ---------------------------------------------------------------------------

struct Win {
  double m, c, p;
};

// three-point tridiagonal row: c_{i-1} x_{i-1} + a_i x_i + b_i x_{i+1}
__device__ __forceinline__ double tri3(const double* bands, int n, int i, double xm, double x0, double xp) {
  double y = bands[i] * x0;
  if (i > 0) y += bands[2 * n + i - 1] * xm;
  if (i < n - 1) y += bands[n + i] * xp;
  return y;
}

__device__ __forceinline__ double circ3(const double* th, double xm, double x0, double xp) {
  return th[1] * xm + th[0] * x0 + th[1] * xp;
}

template <int GEOM, int KIN, int RB>
__global__ void __launch_bounds__(512) fbuild_rows_kernel(const StencilParams p) {
  constexpr bool D3 = GEOM >= 2;
  constexpr unsigned FULL = 0xffffffffu;
  if (p.step && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0) *p.step += 1;
  const int nl = D3 ? p.n3 : p.n2;  // contiguous extent
  const int n1 = p.n1;              // walked extent
  const int l = threadIdx.x;
  const int lane = l & 31;
  const bool act = l < nl;
  const int lc = act ? l : nl - 1;
  const int i0 = blockIdx.x * RB;
  const int j = D3 ? (int)blockIdx.y : 0;
  const int b = blockIdx.z;
  const long long rs = D3 ? (long long)p.n2 * p.n3 : (long long)p.n2;  // walked stride
  const long long run_base = (long long)b * p.ncomp * p.npts + (long long)j * (D3 ? p.n3 : 0);
  const bool periodic_walk = (GEOM == 1);
  const bool periodic_row = (GEOM == 0);
  const int nC = (KIN == KIN_EXTERNAL) ? p.ncomp : 2;
  if (i0 >= n1) return;
  const int iend = min(n1, i0 + RB);

  // contiguous-axis neighbours of the value x0 held at column l of row `rowp`
  auto row_nb = [&](const double* rowp, double x0, double& xl, double& xr) {
    const double up = __shfl_up_sync(FULL, x0, 1);
    const double dn = __shfl_down_sync(FULL, x0, 1);
    int li = lc - 1, ri = lc + 1;
    if (periodic_row) {
      if (li < 0) li = nl - 1;
      if (ri >= nl) ri = 0;
    }
    xl = (lane > 0 && li == lc - 1) ? up : ((li >= 0) ? __ldg(rowp + li) : 0.0);
    xr = (lane < 31 && ri == lc + 1 && ri < nl) ? dn : ((ri < nl) ? __ldg(rowp + ri) : 0.0);
  };

  auto diffusion = [&](int c, int i, const double* rowp, const Win& w) -> double {
    double xl, xr;
    row_nb(rowp, w.c, xl, xr);
    if (GEOM == 0) {
      const double r = tri3(p.rho_b + (long long)c * 3 * n1, n1, i, w.m, w.c, w.p);
      const double q = circ3(p.th + 2 * c, xl, w.c, xr);
      return r + p.d_rho[c * n1 + i] * q;
    } else if (GEOM == 1) {
      const double q = circ3(p.th + 2 * c, w.m, w.c, w.p);
      const double r = tri3(p.phi_b + (long long)c * 3 * nl, nl, lc, xl, w.c, xr);
      return q * p.d_phi[c * nl + lc] + r;
    } else {
      const int jm = (j == 0) ? p.n2 - 1 : j - 1;
      const int jp = (j == p.n2 - 1) ? 0 : j + 1;
      const double ym = __ldg(rowp + (long long)(jm - j) * nl + lc);
      const double yp = __ldg(rowp + (long long)(jp - j) * nl + lc);
      const double r = tri3(p.rho_b + (long long)c * 3 * n1, n1, i, w.m, w.c, w.p);
      const double q = circ3(p.th + 2 * c, ym, w.c, yp);
      const double dr = p.d_rho[c * n1 + i];
      if (GEOM == 2) {
        const double ph = tri3(p.phi_b + (long long)c * 3 * nl, nl, lc, xl, w.c, xr);
        return r + (dr * q) * p.d_phi[c * nl + lc] + dr * ph;
      } else {
        const double z = tri3(p.z_b + (long long)c * 3 * nl, nl, lc, xl, w.c, xr);
        return r + dr * q + z;
      }
    }
  };

  auto win_start = [&](const double* X) -> Win {
    Win w;
    const int im = (i0 > 0) ? i0 - 1 : (periodic_walk ? n1 - 1 : -1);
    w.m = (im >= 0) ? __ldg(X + (long long)im * rs + lc) : 0.0;
    w.c = __ldg(X + (long long)i0 * rs + lc);
    w.p = 0.0;
    return w;
  };
  auto win_next = [&](const double* X, int i) -> double {
    int ip = i + 1;
    if (ip >= n1) ip = periodic_walk ? 0 : -1;
    return (ip >= 0) ? __ldg(X + (long long)ip * rs + lc) : 0.0;
  };

  if (KIN == KIN_EXTERNAL) {
    for (int c = 0; c < nC; ++c) {
      const double* X = p.W + run_base + (long long)c * p.npts;
      Win w = win_start(X);
      for (int i = i0; i < iend; ++i) {
        w.p = win_next(X, i);
        const double* rowp = X + (long long)i * rs;
        double val = 0.0;
        if (p.with_diffusion) val = p.coeff[c] * diffusion(c, i, rowp, w);
        const long long idx = run_base + (long long)c * p.npts + (long long)i * rs + lc;
        if (p.with_reaction) val = p.with_diffusion ? __dadd_rn(val, __ldg(p.G + idx)) : __ldg(p.G + idx);
        if (act) p.F[idx] = val;
        w.m = w.c;
        w.c = w.p;
      }
    }
  } else {
    const double* __restrict__ U = p.W + run_base;
    const double* __restrict__ V = U + p.npts;
    double* __restrict__ Fo = p.F;
    const double* kin = p.kin + (long long)b * p.nparams;
    Win wu = win_start(U), wv = win_start(V);
#pragma unroll
    for (int ii = 0; ii < RB; ++ii) {
      const int i = i0 + ii;
      if (i >= iend) break;
      wu.p = win_next(U, i);
      wv.p = win_next(V, i);
      const long long off = (long long)i * rs + lc;
      double g0 = 0.0, g1 = 0.0;
      if (p.with_reaction) {
        double u = wu.c, v = wv.c;
        if (p.lift[0] != 0.0) u = __dadd_rn(u, p.lift[0]);
        if (p.lift[1] != 0.0) v = __dadd_rn(v, p.lift[1]);
        reaction<KIN>(kin, u, v, g0, g1);
      }
      double fu = g0, fv = g1;
      if (p.with_diffusion) {
        const double du = p.coeff[0] * diffusion(0, i, U + (long long)i * rs, wu);
        const double dv = p.coeff[1] * diffusion(1, i, V + (long long)i * rs, wv);
        fu = p.with_reaction ? __dadd_rn(du, g0) : du;
        fv = p.with_reaction ? __dadd_rn(dv, g1) : dv;
      }
      if (act) {
        Fo[run_base + off] = fu;
        Fo[run_base + p.npts + off] = fv;
      }
      wu.m = wu.c;
      wu.c = wu.p;
      wv.m = wv.c;
      wv.c = wv.p;
    }
  }
}

// grid = (ceil(npts / 256), batch): one thread per grid point of one run,
// consecutive threads along the contiguous axis; 32-bit index math only.
template <int GEOM, int KIN>
__global__ void __launch_bounds__(256) fbuild_kernel(const StencilParams p) {
  if (p.step && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *p.step += 1;
  const int npts = (int)p.npts;
  const int pt = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (pt < npts) {
    int i, j, l;
    if (GEOM == 0 || GEOM == 1) {
      i = pt / p.n2;
      j = pt - i * p.n2;
      l = 0;
    } else {
      const int r = pt / p.n3;
      l = pt - r * p.n3;
      i = r / p.n2;
      j = r - i * p.n2;
    }
    const long long fb = (long long)b * p.ncomp * p.npts;
    double g0 = 0.0, g1 = 0.0;
    if (KIN != KIN_EXTERNAL && p.with_reaction) {
      double u = __ldg(p.W + fb + pt);
      double v = __ldg(p.W + fb + p.npts + pt);
      if (p.lift[0] != 0.0) u = __dadd_rn(u, p.lift[0]);
      if (p.lift[1] != 0.0) v = __dadd_rn(v, p.lift[1]);
      reaction<KIN>(p.kin + b * p.nparams, u, v, g0, g1);
    }
    for (int c = 0; c < p.ncomp; ++c) {
      const long long idx = fb + (long long)c * p.npts + pt;
      double val = 0.0;
      if (p.with_diffusion) val = p.coeff[c] * diffusion_at<GEOM>(p, c, p.W + idx, i, j, l);
      if (p.with_reaction) {
        double gc;
        if (KIN == KIN_EXTERNAL)
          gc = __ldg(p.G + idx);
        else
          gc = (c == 0) ? g0 : g1;
        val = p.with_diffusion ? __dadd_rn(val, gc) : gc;
      }
      p.F[idx] = val;
    }
  }
}

}  // namespace cg
