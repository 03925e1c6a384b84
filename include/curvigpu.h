/*
 * curvigpu.h — C ABI of libcurvigpu.so, the B200 (sm_100a) engine for the
 * split exponential Euler hot path of arXiv 2604.11558 (reference package
 * `curvipat`, pure Python; paths below are relative to
 * /root/reference/pkg/src/curvipat).
 *
 * The reference has no FFI: its seams are Python functions.  Each entry point
 * here replaces one of them; the Python drop-in (paper_2604_11558_b200/
 * integrators.py) binds these with ctypes under the reference's names.
 *
 *   cg_plan_create      replaces prepare()            integrators.py:130-173
 *                       (operands are computed on the host, as north_star
 *                        allows, and uploaded once)
 *   cg_apply_diffusion  replaces apply_diffusion()    integrators.py:176-199
 *   cg_kinetics         replaces CoupledSystem.kinetics closures
 *                                                     models.py:386-391,
 *                                                     :284-319, :528-532
 *   cg_step             replaces step_split()         integrators.py:247-249
 *                       (and the STEPPERS dispatch    integrators.py:239-244)
 *   cg_run              replaces the loop body of run_simulation()
 *                                                     integrators.py:413-427
 *                       (kinetics from the common state, step every
 *                        component, divergence guard DIVERGENCE_LIMIT :33)
 *   cg_coupled_*        replace the closures of the bulk-surface models
 *                       _build_ball / _build_cylinder   models.py:570-661
 *                       (coupling terms models.py:322-369) and their
 *                       run_simulation loop              integrators.py:413-427
 *   cg_rng_*            replaces Xoshiro256pp / Uniform / Normal
 *                                                     models.py:55-130
 *
 * Conventions
 *   - All field pointers are DEVICE pointers to fp64 arrays laid out
 *     C-contiguous as [batch][ncomp][n1][n2](n3), reference axis order.
 *   - `stream` is a cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream);
 *     all work is stream-ordered, nothing synchronises the host except
 *     cg_plan_create/destroy.
 *   - Return codes: 0 ok, CG_EINVAL bad argument, CG_ECUDA CUDA failure,
 *     CG_EUNSUPPORTED unsupported configuration.  cg_last_error() gives the
 *     thread-local message of the last failure.
 *   - A plan is not thread-safe; use one plan per host thread.
 */
#ifndef CURVIGPU_H
#define CURVIGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CG_OK 0
#define CG_EINVAL (-1)
#define CG_ECUDA (-2)
#define CG_EUNSUPPORTED (-3)

/* Geometry tags: Geometry enum, integrators.py:46-50 */
#define CG_DISK 0
#define CG_SPHERE 1
#define CG_BALL 2
#define CG_CYLINDER 3

/* Pointwise reaction kinds (two species, evaluated on physical = lifted + lift
 * values).  Parameter order per run in kin_params[b * nparams + i]:
 *   CG_KIN_EXTERNAL     0  no reaction in cg_run; cg_step takes G explicitly
 *   CG_KIN_SCHNAKENBERG 1  gamma, a, b:  gamma(a-u+u^2v), gamma(b-u^2v)
 *                          (models.py:293-296 scaled as in :528-532)
 *   CG_KIN_BRUSSELATOR  2  A, B:  A-(B+1)u+u^2v, Bu-u^2v
 *   CG_KIN_GRAY_SCOTT   3  F, k:  -uv^2+F(1-u), uv^2-(F+k)v
 *   CG_KIN_BVAM_ETA     4  eta, a, b, h, C:
 *                          eta(u+av-Cuv-uv^2), eta(bv+hu+Cuv+uv^2)
 *   CG_KIN_BVAM         5  alpha1, alpha2, alpha3, beta1, beta2 (models.py:284-290)
 *   CG_KIN_DIB          6  zeta1..zeta5, eta1, eta2, eta3, eta5 (models.py:299-319,
 *                          times zeta1 as in :555-557)
 */
#define CG_KIN_EXTERNAL 0
#define CG_KIN_SCHNAKENBERG 1
#define CG_KIN_BRUSSELATOR 2
#define CG_KIN_GRAY_SCOTT 3
#define CG_KIN_BVAM_ETA 4
#define CG_KIN_BVAM 5
#define CG_KIN_DIB 6

typedef struct cg_plan cg_plan;

/* Host-side description of a batched split-EE problem: `batch` independent
 * runs of the same `ncomp`-component system.  All pointers are HOST pointers;
 * cg_plan_create copies them into plan-owned device memory.  Operators may
 * differ per component (leading [ncomp] index), as ComponentOps allows
 * (integrators.py:53-84).  Arrays a geometry does not use may be NULL.
 * n_rho / n_theta / n_phi / n_z below mean the extent of that axis. */
typedef struct {
  int geometry;           /* CG_DISK .. CG_CYLINDER */
  int n[3];               /* reference axis order; n[2] = 1 for 2-D */
  int batch;              /* runs */
  int ncomp;              /* components (2 for every kinetics kind) */
  double tau;
  const double* coeff;    /* [ncomp] diffusion coefficients */
  /* stencils for the diffusion action (bands a, b, c of TridiagonalOperator,
   * operators.py:37-69; b and c have n-1 meaningful entries, stored in a
   * row of length n): [ncomp][3][n_axis] */
  const double* rho_bands;
  const double* phi_bands;
  const double* z_bands;
  const double* theta_stencil; /* [ncomp][2] = (diag, off) of PeriodicTridiagonal */
  const double* d_rho;    /* [ncomp][n_rho] rho weights (rho^-2 or rho^-(2+lambda)) */
  const double* d_phi;    /* [ncomp][n_phi] sin^-2(phi) */
  /* dense transforms as prepare() builds them */
  const double* Q_theta;  /* [ncomp][n_theta][n_theta] */
  const double* phi1_rho; /* [ncomp][n_rho][n_rho] */
  const double* phi1_phi; /* [ncomp][n_phi][n_phi]  (sphere) */
  const double* phi1_z;   /* [ncomp][n_z][n_z]      (cylinder) */
  const double* V_phi;    /* [ncomp][n_phi][n_phi]  (ball) */
  const double* Vinv_phi; /* [ncomp][n_phi][n_phi]  (ball) */
  /* phi1 tensors (PhiTensor.field, phifun.py:52-65), per component:
   *   disk [n_rho][n_theta]; sphere [n_theta][n_phi];
   *   ball Phi [n_rho][n_theta][n_phi] and Phi_outer [n_rho][n_phi]
   *        (constant along theta, stored 2-D);
   *   cylinder [n_rho][n_theta] (constant along z, stored 2-D) */
  const double* Phi;
  const double* Phi_outer;
  int kinetics;           /* CG_KIN_* */
  int nparams;
  const double* kin_params; /* [batch][nparams] */
  const double* lift;     /* [ncomp] constant lift restoring physical values */
  int options;            /* CG_OPT_* bit set */
  /* 0: one operator set per component, shared by every run (the arrays
   * above have a leading [ncomp] index).  1: heterogeneous ensemble -- one
   * operator set per (run, component), leading index [batch * ncomp] in
   * field order f = run * ncomp + component (coeff, bands, theta stencil,
   * d_rho, d_phi, the dense transforms and the Phi tensors; lift stays
   * [ncomp]).  Runs may then differ in diffusion coefficients and domain
   * sizes as long as the grid extents agree. */
  int ops_per_run;
} cg_desc;

/* options: apply the periodic-theta pair Q_theta diag(Phi) Q_theta^T as an
 * exact real-FFT propagator (power-of-two n_theta) instead of two dense DMMA
 * mu-mode products; same mathematics (integrators.py:204-206 etc.), O(n log n). */
#define CG_OPT_THETA_FFT 1

int cg_plan_create(const cg_desc* desc, cg_plan** out);
void cg_plan_destroy(cg_plan* plan);

/* Elements of one [batch][ncomp][...] state array. */
long long cg_plan_state_elems(const cg_plan* plan);

/* out = coeff * M W for every field (apply_diffusion, integrators.py:176-199). */
int cg_apply_diffusion(cg_plan* plan, const double* W, double* out, void* stream);

/* G = g(W + lift) for every run (the kinetics closure). */
int cg_kinetics(cg_plan* plan, const double* W, double* G, void* stream);

/* W_out = step_split(W, G) for every field; W_out must not alias W. */
int cg_step(cg_plan* plan, const double* W, const double* G, double* W_out, void* stream);

/* Advance `state` (in place) by nsteps split-EE steps with the plan's
 * kinetics, steps numbered step0+1 .. step0+nsteps.  first_bad ([batch*ncomp]
 * device ints) receives, per field, the smallest step whose result was
 * non-finite or exceeded 1e12 in magnitude (atomicMin; callers initialise it
 * to INT32_MAX).  The step sequence is replayed from CUDA graphs. */
int cg_run(cg_plan* plan, double* state, long long step0, long long nsteps,
           int* first_bad, void* stream);

/* Per-kernel access for measurement (bench.py roofline): stage -1 is the
 * F-build kernel (stencil + fused kinetics, reads W), stage -2 the fused disk
 * F-build + FFT theta kernel (when the plan uses it), stages 0..count-1 the
 * GEMM chain in order; each runs on the plan's workspaces exactly as inside
 * a step (the last stage writes W_out and reads W for the axpy).  Algorithmic
 * flops per launch count 2*M*N*K per batch item over the true extents. */
int cg_plan_stage_count(const cg_plan* plan);
/* Kernels one cg_run step launches, in order, as stage ids (-2 = the fused
 * disk F-build + FFT-theta kernel, -1 = F-build, >= 0 = stages); returns the
 * count (ids beyond max_ids are not written). */
int cg_plan_step_kernels(const cg_plan* plan, int* ids, int max_ids);
int cg_plan_stage_info(const cg_plan* plan, int stage, long long* flops, long long* bytes);
int cg_run_stage(cg_plan* plan, int stage, const double* W, double* W_out, int* first_bad, void* stream);
/* Copy a plan workspace (0 = X, 1 = Y, 2 = second state) to dst (debugging / tests). */
int cg_plan_copy_workspace(cg_plan* plan, int which, double* dst, void* stream);
/* Bounds check (testing): a plan created with CURVIGPU_REDZONE=1 in the
 * environment surrounds each workspace with a 1 MiB guard band of a fixed
 * byte pattern; returns the number of guard bytes that were overwritten so
 * far (0 = no out-of-bounds write), or < 0 on error.  Synchronises the device. */
long long cg_plan_check_redzones(cg_plan* plan);

/* step_split with external G plus the divergence guard: like cg_step, but the
 * guard records into first_bad with the plan's step counter, which this call
 * advances by one (building block of coupled time loops; graph-capturable). */
int cg_step_guarded(cg_plan* plan, const double* W, const double* G, double* W_out, int* first_bad,
                    void* stream);
/* Set the plan's device step counter (the next guarded step is step + 1). */
int cg_plan_set_step(cg_plan* plan, long long step, void* stream);

/* ---- on-device sampling ----
 * Replaces the per-sample host evaluation of mean_diagnostics()
 * (models.py:728-744: float(sum(W * weights)) + lift for every component,
 * weights from quadrature_weights() models.py:675-715, host setup):
 *   out[f] = sum_i X[f * npts + i] * w[(f % ncls) * npts + i] + (off ? off[f % ncls] : 0)
 * for nfield consecutive fields of npts values (a [B][C] state with ncls = C).
 * X, w, off, out, scratch are device pointers; X and w 16-byte aligned;
 * scratch holds cg_weighted_sums_scratch(nfield, npts) doubles.  Fixed
 * summation order: reruns are bitwise identical.  Graph-capturable. */
long long cg_weighted_sums_scratch(long long nfield, long long npts);
int cg_weighted_sums(const double* X, long long nfield, long long npts, const double* w, int ncls,
                     const double* off, double* out, double* scratch, long long scratch_len, void* stream);

/* ---- bulk-surface coupled models ----
 * Reaction terms of the reference's two mixed-geometry models from the common
 * state: bulk (u, v) on a ball or cylinder, surface (r, s) on the sphere or
 * the bottom disk, coupled through the bulk trace (outermost rho slice /
 * z = 0 slice) with Robin / flux sources (models.py:322-369, :570-661).
 *   CG_BS_BALL      params: alpha1 alpha2 beta1 zeta1 zeta2 zeta3 eta1 eta2;
 *                   geom = {h_rho, rho_edge}
 *   CG_BS_CYLINDER  params: alpha1 alpha2 alpha3 beta1 beta2 beta3 delta
 *                   zeta1 zeta2 zeta3 zeta4 zeta5 eta1 eta2 eta3 eta5;
 *                   geom = {h_z, 0}
 * Wb/Gb are [2][bulk] (u, v), Ws/Gs are [2][surface] (r, s) device arrays;
 * lift[] restores physical values (u, v, r, s). */
#define CG_BS_BALL 1
#define CG_BS_CYLINDER 2
typedef struct {
  int kind;
  int nb[3];
  int ns[2];
  const double* params;
  int nparams;
  double geom[2];
  double lift[4];
} cg_coupling_desc;
typedef struct cg_coupling cg_coupling;
int cg_coupling_create(const cg_coupling_desc* desc, cg_coupling** out);
void cg_coupling_destroy(cg_coupling* c);
int cg_coupled_kinetics(cg_coupling* c, const double* Wb, const double* Ws, double* Gb, double* Gs, void* stream);
/* The coupled time loop (run_simulation, integrators.py:413-427, for the
 * four-component bulk-surface systems): per step the coupled reaction terms
 * from the common state, then step_split of the bulk pair (plan `bulk`,
 * geometry ball / cylinder) and of the surface pair (plan `surf`, sphere /
 * disk), both created with batch 1, ncomp 2 and CG_KIN_EXTERNAL.  Wb / Ws
 * advance in place; first_bad[4] (u, v, r, s) as in cg_run.  Replayed from
 * CUDA graphs; the surface chain runs on a forked stream inside the graph. */
int cg_coupled_run(cg_coupling* c, cg_plan* bulk, cg_plan* surf, double* Wb, double* Ws, long long step0,
                   long long nsteps, int* first_bad, void* stream);

/* ---- standalone mu-mode product and Hadamard product ----
 * cg_product_*  replace tensor.mode_product(mu, L, field)   tensor.py:31-49
 *   (np.tensordot + moveaxis: one DGEMM over the matching unfolding): the
 *   batched DMMA GEMM of the step kernels on one field, the unfolding folded
 *   into the tensor maps.  dims: the field's extents in C order (ndim 2 or 3,
 *   the last one even), mu 1-based, L a HOST row-major n_mu x n_mu matrix
 *   (copied).  apply: T and out are device pointers (16-byte aligned, out of
 *   place); stream-ordered.
 * cg_hadamard   replaces tensor.hadamard(A, B)               tensor.py:77-83 */
typedef struct cg_product cg_product;
int cg_product_create(int mu, int ndim, const int* dims, const double* L, cg_product** out);
int cg_product_apply(cg_product* h, const double* T, double* out, void* stream);
void cg_product_destroy(cg_product* h);
int cg_hadamard(const double* a, const double* b, double* out, long long n, void* stream);

/* ---- on-device setup ----
 * Batched device replacements for the per-operator host work of prepare()
 * (integrators.py:130-173), for ensembles whose runs do not share operators.
 * All pointers are DEVICE pointers; calls are stream-ordered and
 * graph-capturable; nothing synchronises the host.
 *
 * cg_setup_eig_tridiag   replaces eig_tridiag()  operators.py:371-382 with the
 *   symmetriser symmetrize() operators.py:357-368 (scipy/LAPACK there): nmat
 *   operators with bands a [nmat][n], b, c [nmat][n-1] (b, c > 0) ->
 *   lam [nmat][n] ascending, Qt [nmat][n][n] with Qt[k][r] = Q[r][k]
 *   (eigenvector k contiguous, orthonormal), xi [nmat][n] the symmetriser
 *   (V = diag(xi) Q, V^-1 = Q^T diag(1/xi)).  work: nmat*n*n doubles of
 *   scratch (distinct from Qt).  status [nmat]: 0 ok, 1 the QL iteration did
 *   not converge (NumericalFailure, operators.py:381), 2 a nonpositive
 *   off-diagonal (ValueError, operators.py:362).
 * cg_setup_phi1_matrix   replaces phi1_matrix()  phifun.py:68-71:
 *   out[set] = V diag(phi1(s[set] * lam)) V^-1 for nset (operator, scale)
 *   pairs; mat_of_set[set] picks the operator (NULL: set itself).
 * cg_setup_phi1_outer    replaces phi1_outer()   phifun.py:52-65:
 *   out[set][i][j][k] = phi1(s[set] * ((f1[set][i] * f2[set][j]) * f3[set][k])),
 *   f3 NULL (n3 = 1) for two factors.
 * cg_setup_phi1          replaces phi1()         phifun.py:23-37, elementwise. */
int cg_setup_eig_tridiag(int nmat, int n, const double* a, const double* b, const double* c, double* lam, double* Qt,
                         double* xi, double* work, int* status, void* stream);
int cg_setup_phi1_matrix(int nset, int n, const double* lam, const double* Qt, const double* xi,
                         const int* mat_of_set, const double* s, double* out, void* stream);
int cg_setup_phi1_outer(int nset, int n1, int n2, int n3, const double* f1, const double* f2, const double* f3,
                        const double* s, double* out, void* stream);
int cg_setup_phi1(long long count, const double* x, double* out, void* stream);

/* Last error message of the calling thread. */
const char* cg_last_error(void);
int cg_version(void);

/* Host RNG: xoshiro256++ seeded through splitmix64 (models.py:43-104).
 * state is 4 uint64 words owned by the caller. */
void cg_rng_seed(uint64_t seed, uint64_t state[4]);
void cg_rng_next(uint64_t state[4], long long n, uint64_t* out);
/* lo + (hi - lo) * U[0,1) (models.py:107-119) */
void cg_rng_uniform(uint64_t state[4], long long n, double lo, double hi, double* out);
/* sigma * Box-Muller normal (models.py:93-104, :121-130) */
void cg_rng_normal(uint64_t state[4], long long n, double sigma, double* out);

#ifdef __cplusplus
}
#endif
#endif /* CURVIGPU_H */
