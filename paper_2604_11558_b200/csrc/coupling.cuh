// Bulk-surface coupled kinetics: the reaction terms of
// the reference's two mixed-geometry models, evaluated from the common state
// in one pass over the bulk points and the surface points.
//
//   CG_BS_BALL      ball (u, v) + sphere surface (r, s):
//                   models.py:322-345 (bulk_surface_coupling_ball) and the
//                   closure of _build_ball, models.py:587-602
//   CG_BS_CYLINDER  cylinder (u, v, lifted) + bottom disk (r, s):
//                   models.py:348-369 (bs_cylinder_coupling) and the closure
//                   of _build_cylinder, models.py:633-649
//
// The trace the surface sees is the bulk's outermost radial slice (ball,
// rho index n1-1) or its bottom slice (cylinder, z index 0); the bulk
// receives the flux source on that same slice.  Operation order follows the
// reference expressions so results match the NumPy evaluation to rounding.
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace cg {

enum { BS_BALL = 1, BS_CYLINDER = 2 };

struct CouplingParams {
  int kind;
  int nb1, nb2, nb3;  // bulk extents
  int ns1, ns2;       // surface extents
  long long nbpts;    // logical bulk points per component
  long long nspts;    // logical surface points per component
  // storage of the state / reaction arrays: last-axis row stride and field stride
  int ldb, lds;
  long long fb, fs;
  double k[16];       // model parameters (order in curvigpu.h)
  double h, rho_edge; // ball: h_rho, rho_edge; cylinder: h_z
  double lift[4];     // u, v, r, s
  const double* Wb;   // [2][bulk]
  const double* Ws;   // [2][surface]
  double* Gb;
  double* Gs;
};

__device__ __forceinline__ void ball_flux(const CouplingParams& p, double ut, double vt, double r, double s,
                                          double& src_u, double& src_v, double& pr, double& qs) {
  // models.py:322-345 with alpha1, alpha2, beta1, zeta1, zeta2, zeta3, eta1, eta2 = k[0..7]
  const double a2 = p.k[1], b1 = p.k[2], z1 = p.k[3], z2 = p.k[4], z3 = p.k[5], e1 = p.k[6], e2 = p.k[7];
  const double ex_u = __dsub_rn(__dmul_rn(z2, r), __dmul_rn(z3, ut));
  const double ex_v = __dsub_rn(__dmul_rn(e1, s), __dmul_rn(e2, vt));
  const double flux_u = __dmul_rn(z1, ex_u), flux_v = __dmul_rn(z1, ex_v);
  const double ghost = __dadd_rn(__ddiv_rn(1.0, __dmul_rn(p.h, p.h)), __ddiv_rn(1.0, __dmul_rn(p.rho_edge, p.h)));
  const double pre = __dmul_rn(__dmul_rn(2.0, p.h), ghost);
  src_u = __dmul_rn(pre, flux_u);
  src_v = __dmul_rn(pre, flux_v);
  const double rrs = __dmul_rn(__dmul_rn(r, r), s);
  const double b = __dadd_rn(__dsub_rn(a2, r), rrs);
  const double c = __dsub_rn(b1, rrs);
  pr = __dsub_rn(b, ex_u);
  qs = __dsub_rn(c, ex_v);
}

__device__ __forceinline__ void cyl_flux(const CouplingParams& p, double ub, double vb, double r, double s,
                                         double& src_u, double& src_v, double& pr, double& qs) {
  // models.py:299-308, :348-369 with alpha1, alpha2, alpha3, beta1, beta2, beta3, delta,
  // zeta1..zeta5, eta1, eta2, eta3, eta5 = k[0..15]
  const double a3 = p.k[2], b2 = p.k[4], b3 = p.k[5], dl = p.k[6];
  const double z1 = p.k[7], z2 = p.k[8], z3 = p.k[9], z4 = p.k[10], z5 = p.k[11];
  const double e1 = p.k[12], e2 = p.k[13], e3 = p.k[14], e5 = p.k[15];
  const double eta4 = __ddiv_rn(__dmul_rn(__dmul_rn(__dmul_rn(b2, e1), __dsub_rn(1.0, z5)),
                                          __dadd_rn(__dsub_rn(1.0, e3), __dmul_rn(e3, z5))),
                                __dmul_rn(z5, __dadd_rn(1.0, __dmul_rn(e3, z5))));
  const double one_s = __dsub_rn(1.0, s);
  pr = __dsub_rn(__dsub_rn(__dmul_rn(__dmul_rn(__dmul_rn(z2, ub), one_s), r), __dmul_rn(z3, cube_rn(r))),
                 __dmul_rn(z4, __dsub_rn(s, z5)));
  const double q1 = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(e1, vb), __dadd_rn(1.0, __dmul_rn(e2, r))), one_s),
                              __dsub_rn(1.0, __dmul_rn(e3, one_s)));
  const double q2 = __dmul_rn(__dmul_rn(__dmul_rn(eta4, __dadd_rn(1.0, __dmul_rn(e5, r))), s),
                              __dadd_rn(1.0, __dmul_rn(e3, s)));
  qs = __dsub_rn(q1, q2);
  const double m2h = -__ddiv_rn(2.0, p.h);
  src_u = __dmul_rn(__dmul_rn(__dmul_rn(m2h, z1), a3), pr);
  src_v = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(m2h, z1), b3), dl), qs);
}

// one thread per (logical) bulk point, then one per surface point
__global__ void __launch_bounds__(256) coupled_kinetics_kernel(const CouplingParams p) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nb = p.nbpts, ns = p.nspts;
  auto phys = [&](const double* W, long long idx, int comp) {
    const double x = W[idx];
    return p.lift[comp] != 0.0 ? __dadd_rn(x, p.lift[comp]) : x;
  };
  // storage offsets
  auto bulk_at = [&](long long i, long long j, long long k) { return (i * p.nb2 + j) * p.ldb + k; };
  auto surf_at = [&](long long a, long long c) { return a * p.lds + c; };
  if (gid < nb) {
    const long long k = gid % p.nb3, ij = gid / p.nb3;
    const long long j = ij % p.nb2, i = ij / p.nb2;
    const long long bo = bulk_at(i, j, k);
    const double u = phys(p.Wb, bo, 0), v = phys(p.Wb + p.fb, bo, 1);
    double gu, gv;
    bool on_trace;
    long long so;
    if (p.kind == BS_BALL) {
      // gu = alpha1 * schnakenberg(u, v)
      const double a1 = p.k[0], a2 = p.k[1], b1 = p.k[2];
      const double uuv = __dmul_rn(__dmul_rn(u, u), v);
      gu = __dmul_rn(a1, __dadd_rn(__dsub_rn(a2, u), uuv));
      gv = __dmul_rn(a1, __dsub_rn(b1, uuv));
      on_trace = i == p.nb1 - 1;  // outermost rho slice
      so = surf_at(j, k);         // (theta, phi) on the sphere
    } else {
      const double a1 = p.k[0], a2 = p.k[1], b1 = p.k[3], b2 = p.k[4];
      gu = __dmul_rn(-a1, __dsub_rn(u, a2));
      gv = __dmul_rn(-b1, __dsub_rn(v, b2));
      on_trace = k == 0;   // z = 0 slice
      so = surf_at(i, j);  // (rho, theta) on the bottom disk
    }
    if (on_trace) {
      const double r = phys(p.Ws, so, 2), s = phys(p.Ws + p.fs, so, 3);
      double su, sv, pr, qs;
      if (p.kind == BS_BALL)
        ball_flux(p, u, v, r, s, su, sv, pr, qs);
      else
        cyl_flux(p, u, v, r, s, su, sv, pr, qs);
      gu = __dadd_rn(gu, su);
      gv = __dadd_rn(gv, sv);
    }
    p.Gb[bo] = gu;
    p.Gb[p.fb + bo] = gv;
  } else if (gid < nb + ns) {
    const long long sidx = gid - nb;
    const long long c2 = sidx % p.ns2, a2 = sidx / p.ns2;
    const long long so = surf_at(a2, c2);
    const long long bo = (p.kind == BS_BALL) ? bulk_at(p.nb1 - 1, a2, c2) : bulk_at(a2, c2, 0);
    const double u = phys(p.Wb, bo, 0), v = phys(p.Wb + p.fb, bo, 1);
    const double r = phys(p.Ws, so, 2), s = phys(p.Ws + p.fs, so, 3);
    double su, sv, pr, qs;
    double z1;
    if (p.kind == BS_BALL) {
      ball_flux(p, u, v, r, s, su, sv, pr, qs);
      z1 = p.k[3];
    } else {
      cyl_flux(p, u, v, r, s, su, sv, pr, qs);
      z1 = p.k[7];
    }
    p.Gs[so] = __dmul_rn(z1, pr);
    p.Gs[p.fs + so] = __dmul_rn(z1, qs);
  }
}

}  // namespace cg
