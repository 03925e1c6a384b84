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
  int opb;              // operator-set stride per run: 0 (shared) or ncomp (heterogeneous ensemble)
  long long npts;  // points per field (storage)
  // storage layout of the F-build's input W and output F / external G: the
  // contiguous (last) axis has logical extent n_last and row stride ldw / ldf
  // (even, for TMA), a field holds npw / npf elements
  int ldw, ldf;
  long long npw, npf;
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

// The reference's kinetics closures add a component's lift only in lifted
// models (models.py:528-532; unlifted models pass the state through).
// x + (-0.0) == x bit for bit for every x (signed zeros included), so a zero
// lift becomes the addend -0.0 and the add is unconditional: no per-point
// select (256 FSEL in the fused disk front).
__device__ __forceinline__ double lift_addend(double lift) { return lift != 0.0 ? lift : -0.0; }

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
    const double pr = SUB(SUB(MUL(MUL(z2, SUB(1.0, s)), r), MUL(z3, cube_rn(r))), MUL(z4, SUB(s, z5)));
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
// F-build: one CTA stages RB+2 consecutive rows of the first axis (plus, for
// 3-D fields, the RB rows at theta-1 and theta+1) of every component into
// shared memory with all loads in flight at once, then each thread computes
// its column of the RB interior rows from shared memory.  Every W value is
// read from HBM about once; loads, compute and the coalesced F stores are
// separated so the kernel streams at HBM speed.
//   grid = (ceil(n1 / RB), 3-D ? n2 : 1, batch), block = round32(n_last),
//   dynamic smem = ncomp_staged * rows * n_last * 8 bytes
// ---------------------------------------------------------------------------

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

// R2: walked-axis rows per CTA of the 2-D geometries: 8 (two staged halo rows
// per 8), or 4 for small problems, where 8-row CTAs leave most SMs idle (the
// sphere's 512 rows: 64 CTAs; F-build 3.4 -> 2.4 us, config 2 step 17.6 -> 16.3 us)
template <int GEOM, int R2 = 8>
struct FbuildShape {
  static constexpr bool D3 = GEOM >= 2;
#ifndef CG_RB3
#define CG_RB3 4
#endif
#ifndef CG_JB3
#define CG_JB3 2
#endif
  // interior rows per CTA.  Ball: 5 (n_rho = 100: 20 x 50 = 1000 CTAs of 2.4
  // staged rows per output row; 4 rows: 1250 CTAs of 2.5), with the narrow
  // kernel's five CTAs per SM 12.5 -> 11.6 us (6 rows: 12.7 us)
  static constexpr int RB = D3 ? (GEOM == 2 ? 5 : CG_RB3) : R2;
  // 3-D: JB consecutive theta columns per CTA share their theta neighbours:
  // staged rows = JB (RB + 2) centre rows + 2 RB theta-halo rows.  JB = 2
  // (2.5 staged rows per output row instead of 3.5): cylinder F-build
  // 11.8 -> 10.9 us, ball 14.6 -> 13.8 us; JB = 4 (2.0, but a quarter of the
  // CTAs: ragged waves) measured 14.8 / 14.7 us
  static constexpr int JB = D3 ? CG_JB3 : 1;
  static constexpr int ROWS = D3 ? JB * (RB + 2) + 2 * RB : RB + 2;  // staged rows per component
};

// stage component X's rows for this CTA into s[ROWS][nl]
// 3-D: X points at column j0; centre block jj at rows jj (RB + 2) ..., the
// theta halo (columns j0 - 1 and j0 + jn, periodic) at JB (RB + 2) + [0, 2 RB)
// (offsets within one field are 32-bit: a field holds < 2^31 elements, checked
// at plan creation; 64-bit index arithmetic per load made the 3-D kernels
// issue-bound)
// One staged value.  ASYNC: an 8-byte cp.async (no register round trip; the
// cylinder's F-build 10.2 -> 9.7 us, no gain for the ball or the 2-D kernels,
// profiles/r02_fbuild_ab.txt), closed by stage_wait before the CTA barrier.
template <bool ASYNC>
__device__ __forceinline__ void stage_put(double* dst, const double* src) {
  if constexpr (ASYNC)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
  else
    *dst = __ldg(src);
}
template <bool ASYNC>
__device__ __forceinline__ void stage_wait() {
  if constexpr (ASYNC) asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
template <int GEOM>
constexpr bool kStageAsync = (GEOM == 3);

template <int GEOM, int R2 = 8>
__device__ __forceinline__ void stage_rows(double* s, const double* __restrict__ X, int i0, int j, int n1, int n2,
                                           int nl, int rs, int jst) {
  using S = FbuildShape<GEOM, R2>;
  const bool periodic_walk = (GEOM == 1);
  const int l = threadIdx.x;
  if (l >= nl) return;
  const int jn = S::D3 ? min(S::JB, n2 - j) : 1;  // valid columns of this CTA
#pragma unroll
  for (int jj = 0; jj < S::JB; ++jj) {
    const int jo = (jj < jn ? jj : jn - 1) * jst;
#pragma unroll
    for (int r = 0; r < S::RB + 2; ++r) {
      int i = i0 - 1 + r;
      if (i < 0) i = periodic_walk ? n1 - 1 : 0;
      if (i >= n1) i = periodic_walk ? i - n1 : n1 - 1;
      stage_put<kStageAsync<GEOM>>(&s[(jj * (S::RB + 2) + r) * nl + l], X + (i * rs + jo + l));
    }
  }
  if (S::D3) {
    const int jm = (j == 0) ? n2 - 1 : j - 1;
    const int jp = (j + jn == n2) ? 0 : j + jn;
    constexpr int H = S::JB * (S::RB + 2);
#pragma unroll
    for (int r = 0; r < S::RB; ++r) {
      const int i = min(i0 + r, n1 - 1);
      stage_put<kStageAsync<GEOM>>(&s[(H + r) * nl + l], X + (i * rs + (jm - j) * jst + l));
      stage_put<kStageAsync<GEOM>>(&s[(H + S::RB + r) * nl + l], X + (i * rs + (jp - j) * jst + l));
    }
  }
}

// Per-thread, per-component stencil coefficients, loaded once per CTA so the
// inner loop issues no global loads (the first version re-read the bands for
// every point and was LSU-bound).  Boundary terms carry a zero coefficient,
// which leaves every value bit-identical to the branchy three-point form.
struct CompCoef {
  double coeff;
  double th_diag, th_off;     // periodic theta stencil
  double la, lb, lc, ld;      // contiguous-axis tridiagonal row (a, b, c_prev) and its metric weight
};

struct RowCoef {              // walked-axis tridiagonal row (shared by the CTA, in smem)
  double a, b, c, d;          // a_i, b_i (0 at the last row), c_{i-1} (0 at the first), d_rho[i]
};

// c = operator set index (component, or run * ncomp + component)
template <int GEOM>
__device__ __forceinline__ CompCoef comp_coef(const StencilParams& p, int c, int l, int nl) {
  CompCoef k;
  k.coeff = p.coeff[c];
  k.th_diag = p.th[2 * c];
  k.th_off = p.th[2 * c + 1];
  k.la = k.lb = k.lc = k.ld = 0.0;
  if (GEOM != 0) {
    const double* bands = (GEOM == 3) ? p.z_b + (long long)c * 3 * nl : p.phi_b + (long long)c * 3 * nl;
    k.la = bands[l];
    k.lb = (l < nl - 1) ? bands[nl + l] : 0.0;
    k.lc = (l > 0) ? bands[2 * nl + l - 1] : 0.0;
    if (GEOM == 1 || GEOM == 2) k.ld = p.d_phi[c * nl + l];
  }
  return k;
}

// coeff-free diffusion action at interior row r (global row i), column l,
// from the shared-memory stage s (rows r, r+1, r+2 = i-1, i, i+1)
// (3-D: theta column jj of the CTA's jn; its theta neighbours are the adjacent
// centre blocks or the halo rows)
template <int GEOM, int R2 = 8>
__device__ __forceinline__ double diffusion_rows(const CompCoef& k, const RowCoef& rc, const double* s0, int r, int l,
                                                 int nl, int jj = 0, int jn = 1) {
  using S = FbuildShape<GEOM, R2>;
  const double* s = s0 + jj * (S::RB + 2) * nl;
  const double xm = s[r * nl + l], x0 = s[(r + 1) * nl + l], xp = s[(r + 2) * nl + l];
  int ll = l - 1, lr = l + 1;
  if (GEOM == 0) {  // periodic contiguous axis
    if (ll < 0) ll = nl - 1;
    if (lr >= nl) lr = 0;
  } else {
    if (ll < 0) ll = 0;  // coefficient is zero there
    if (lr >= nl) lr = nl - 1;
  }
  const double xl = s[(r + 1) * nl + ll];
  const double xr = s[(r + 1) * nl + lr];
  if (GEOM == 0) {  // disk: rho walked (tridiagonal), theta contiguous (periodic)
    const double rr = rc.a * x0 + rc.c * xm + rc.b * xp;
    const double q = k.th_off * xl + k.th_diag * x0 + k.th_off * xr;
    return rr + rc.d * q;
  } else if (GEOM == 1) {  // sphere: theta walked (periodic), phi contiguous (tridiagonal)
    const double q = k.th_off * xm + k.th_diag * x0 + k.th_off * xp;
    const double rr = k.la * x0 + k.lc * xl + k.lb * xr;
    return q * k.ld + rr;
  } else {
    constexpr int H = S::JB * (S::RB + 2);
    const double ym = jj > 0 ? s0[((jj - 1) * (S::RB + 2) + r + 1) * nl + l] : s0[(H + r) * nl + l];
    const double yp = jj + 1 < jn ? s0[((jj + 1) * (S::RB + 2) + r + 1) * nl + l] : s0[(H + S::RB + r) * nl + l];
    const double rr = rc.a * x0 + rc.c * xm + rc.b * xp;
    const double q = k.th_off * ym + k.th_diag * x0 + k.th_off * yp;
    const double dr = rc.d;
    const double t = k.la * x0 + k.lc * xl + k.lb * xr;
    if (GEOM == 2) return rr + (dr * q) * k.ld + dr * t;  // ball: phi contiguous
    return rr + dr * q + t;                                // cylinder: z contiguous
  }
}

// fill the CTA's walked-axis row coefficients for components [0, nc)
template <int GEOM, int R2 = 8>
__device__ __forceinline__ void row_coefs(RowCoef* rcs, const StencilParams& p, int i0, int nc, int ob) {
  using S = FbuildShape<GEOM, R2>;
  const int n1 = p.n1;
  for (int idx = threadIdx.x; idx < nc * S::RB; idx += blockDim.x) {
    const int c = idx / S::RB, r = idx - c * S::RB;
    const int i = min(i0 + r, n1 - 1);
    RowCoef rc{0.0, 0.0, 0.0, 0.0};
    if (GEOM != 1) {
      const double* bands = p.rho_b + (long long)(ob + c) * 3 * n1;
      rc.a = bands[i];
      rc.b = (i < n1 - 1) ? bands[n1 + i] : 0.0;
      rc.c = (i > 0) ? bands[2 * n1 + i - 1] : 0.0;
      rc.d = p.d_rho[(long long)(ob + c) * n1 + i];
    }
    rcs[idx] = rc;
  }
}

// NARROW (3-D fields whose contiguous axis fits 128 threads): capped at 96
// registers so five CTAs share an SM (ball 12.5 -> 11.8 us with 4-row CTAs)
template <int GEOM, int KIN, int R2 = 8, bool NARROW = false>
__global__ void __launch_bounds__(NARROW ? 128 : 512, NARROW ? 5 : 1) fbuild_rows_kernel(const StencilParams p) {
  using S = FbuildShape<GEOM, R2>;
  extern __shared__ double fb_smem[];
  __shared__ RowCoef rcs[8 * S::RB];  // up to 8 components
  pdl_wait();
  if (p.step && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0) *p.step += 1;
  const int nl = S::D3 ? p.n3 : p.n2;
  const int n1 = p.n1;
  const int l = threadIdx.x;
  const int lcl = l < nl ? l : nl - 1;
  const int i0 = blockIdx.x * S::RB;
  const int j = S::D3 ? (int)blockIdx.y * S::JB : 0;  // first theta column
  const int jn = S::D3 ? min(S::JB, p.n2 - j) : 1;
  const int b = blockIdx.z;
  const int rsw = S::D3 ? p.n2 * p.ldw : p.ldw;
  const int rsf = S::D3 ? p.n2 * p.ldf : p.ldf;
  const long long wbase = (long long)b * p.ncomp * p.npw + (long long)j * (S::D3 ? p.ldw : 0);
  const long long fbase = (long long)b * p.ncomp * p.npf + (long long)j * (S::D3 ? p.ldf : 0);
  const int plane = S::ROWS * nl;
  const int ob = b * p.opb;  // this run's operator sets

  if (KIN == KIN_EXTERNAL) {
    const int nc = p.ncomp < 8 ? p.ncomp : 8;
    row_coefs<GEOM, R2>(rcs, p, i0, nc, ob);
    for (int c = 0; c < p.ncomp; ++c) {
      const double* X = p.W + wbase + (long long)c * p.npw;
      if (c > 0) __syncthreads();
      stage_rows<GEOM, R2>(fb_smem, X, i0, j, n1, p.n2, nl, rsw, p.ldw);
      stage_wait<kStageAsync<GEOM>>();
      __syncthreads();
      if (l < nl) {
        const CompCoef k = comp_coef<GEOM>(p, ob + c, l, nl);
        for (int jj = 0; jj < jn; ++jj) {
#pragma unroll
          for (int r = 0; r < S::RB; ++r) {
            const int i = i0 + r;
            if (i >= n1) break;
            const long long idx = fbase + (long long)c * p.npf + (jj * p.ldf + i * rsf + l);
            double val = 0.0;
            if (p.with_diffusion)
              val = k.coeff * diffusion_rows<GEOM, R2>(k, rcs[(c < 8 ? c : 7) * S::RB + r], fb_smem, r, l, nl, jj, jn);
            if (p.with_reaction) val = p.with_diffusion ? __dadd_rn(val, __ldg(p.G + idx)) : __ldg(p.G + idx);
            p.F[idx] = val;
          }
        }
      }
    }
  } else {
    const bool with_d = p.with_diffusion;
    if (with_d) row_coefs<GEOM, R2>(rcs, p, i0, 2, ob);
    stage_rows<GEOM, R2>(fb_smem, p.W + wbase, i0, j, n1, p.n2, nl, rsw, p.ldw);
    stage_rows<GEOM, R2>(fb_smem + plane, p.W + wbase + p.npw, i0, j, n1, p.n2, nl, rsw, p.ldw);
    CompCoef k0{}, k1{};  // operator coefficients are only present when diffusing
    if (with_d) {
      k0 = comp_coef<GEOM>(p, ob, lcl, nl);
      k1 = comp_coef<GEOM>(p, ob + 1, lcl, nl);
    }
    double kin[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) kin[q] = (q < p.nparams) ? p.kin[(long long)b * p.nparams + q] : 0.0;
    const double lift0 = lift_addend(p.lift[0]), lift1 = lift_addend(p.lift[1]);
    const bool with_r = p.with_reaction;
    stage_wait<kStageAsync<GEOM>>();
    __syncthreads();
    if (l >= nl) return;
    double* __restrict__ Fo = p.F + fbase;       // species 0 of this CTA's run / theta column
    double* __restrict__ Fo1 = Fo + p.npf;       // species 1
    for (int jj = 0; jj < jn; ++jj) {
#pragma unroll
    for (int r = 0; r < S::RB; ++r) {
      const int i = i0 + r;
      if (i >= n1) break;
      const int off = jj * p.ldf + i * rsf + l;
      const int cs = (jj * (S::RB + 2) + r + 1) * nl + l;  // centre value in the stage
      double g0 = 0.0, g1 = 0.0;
      if (with_r) {
        double u = fb_smem[cs], v = fb_smem[plane + cs];
        u = __dadd_rn(u, lift0);
        v = __dadd_rn(v, lift1);
        reaction<KIN>(kin, u, v, g0, g1);
      }
      double fu = g0, fv = g1;
      if (with_d) {
        const double du = k0.coeff * diffusion_rows<GEOM, R2>(k0, rcs[r], fb_smem, r, l, nl, jj, jn);
        const double dv = k1.coeff * diffusion_rows<GEOM, R2>(k1, rcs[S::RB + r], fb_smem + plane, r, l, nl, jj, jn);
        fu = with_r ? __dadd_rn(du, g0) : du;
        fv = with_r ? __dadd_rn(dv, g1) : dv;
      }
      Fo[off] = fu;
      Fo1[off] = fv;
    }
    }
  }
}

}  // namespace cg
