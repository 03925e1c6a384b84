// On-device setup: batched replacements for the per-operator
// host work of prepare() (integrators.py:130-173) --
//   eig_tridiag     symmetriser + symmetric tridiagonal eigenpairs
//                   (operators.py:357-382; LAPACK via scipy there)
//   phi1            (e^x - 1)/x with the reference's Taylor branch (phifun.py:23-37)
//   phi1_outer      phi1 over outer products of spectral factors (phifun.py:52-65)
//   phi1_matrix     V diag(phi1(s lambda)) V^-1 (phifun.py:68-71)
// for ensembles whose runs do not share operators (one operator set per run:
// 512 x 2 sets of 128 x 128 tables at the config-5 grid).  Everything is
// stream-ordered on device pointers; nothing here touches the host.
//
// Eigen-solver: one CTA per matrix runs the implicit-shift QL iteration
// (the classical tql2 recurrence: Wilkinson shift, one chase of plane
// rotations per iteration).  The scalar recurrence of a chase does not depend
// on the eigenvector matrix, so thread 0 produces the chase's rotations
// (c_i, s_i) into shared memory and then every thread applies the whole
// rotation sequence to its own rows of Q (rows are independent; the value
// carried between consecutive rotations stays in a register).  Q is held
// transposed (Zt[col][row]) so a rotation's two columns are contiguous
// across threads.  Products of plane rotations keep Q orthogonal to rounding,
// which phi1_matrix (Q^T as the inverse) relies on.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>

#include "curvigpu.h"
#include "errors.h"

namespace {

#define SETUP_TRY(x)                                                                                      \
  do {                                                                                                    \
    cudaError_t e_ = (x);                                                                                 \
    if (e_ != cudaSuccess)                                                                                \
      return cg_internal_fail(CG_ECUDA, (std::string(#x) + ": " + cudaGetErrorString(e_)).c_str());       \
  } while (0)

constexpr int kEigThreads = 256;
constexpr int kMaxQlIter = 60;  // per eigenvalue (tql2 allows 30; the polar operators need < 4)

// phi1 with the reference's branch: degree-6 Taylor (Horner) below 1e-5, else expm1(x)/x
__device__ __forceinline__ double phi1_dev(double x) {
  if (fabs(x) < 1e-5) {
    double acc = 1.0 / 5040.0;
    acc = __dadd_rn(__dmul_rn(acc, x), 1.0 / 720.0);
    acc = __dadd_rn(__dmul_rn(acc, x), 1.0 / 120.0);
    acc = __dadd_rn(__dmul_rn(acc, x), 1.0 / 24.0);
    acc = __dadd_rn(__dmul_rn(acc, x), 1.0 / 6.0);
    acc = __dadd_rn(__dmul_rn(acc, x), 1.0 / 2.0);
    acc = __dadd_rn(__dmul_rn(acc, x), 1.0);
    return acc;
  }
  return expm1(x) / x;
}

__device__ __forceinline__ double sign_of(double a, double b) { return b >= 0.0 ? fabs(a) : -fabs(a); }

// dynamic shared memory: d[n], e[n], cs[2n], sn[2n] (double-buffered chase), rank scratch
__global__ void __launch_bounds__(kEigThreads) eig_tridiag_kernel(int n, const double* __restrict__ a,
                                                                  const double* __restrict__ b,
                                                                  const double* __restrict__ c, double* __restrict__ lam,
                                                                  double* __restrict__ Qt, double* __restrict__ xi,
                                                                  double* __restrict__ work, int* __restrict__ status) {
  extern __shared__ double eg_smem[];
  double* d = eg_smem;
  double* e = d + n;
  double* cs = e + n;
  double* sn = cs + n;
  __shared__ int sh_l, sh_m, sh_state;  // chase range [l, m), 0 = go on, 1 = done, 2 = failed
  const int mat = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  const double* am = a + (size_t)mat * n;
  const double* bm = b + (size_t)mat * (n - 1);
  const double* cm = c + (size_t)mat * (n - 1);
  double* Zt = work + (size_t)mat * n * n;  // Zt[col][row]
  // ---- symmetriser (operators.py:357-368): xi_0 = 1, xi_i = exp(0.5 sum_{j<i} (log c_j - log b_j))
  bool bad = false;
  for (int i = tid; i < n - 1; i += nt) bad |= !(bm[i] > 0.0) || !(cm[i] > 0.0);
  if (__syncthreads_or(bad)) {
    if (tid == 0) status[mat] = 2;
    return;
  }
  if (tid == 0) {
    double acc = 0.0;
    xi[(size_t)mat * n] = 1.0;
    for (int i = 0; i < n - 1; ++i) {
      acc += log(cm[i]) - log(bm[i]);  // np.cumsum order
      xi[(size_t)mat * n + i + 1] = exp(0.5 * acc);
    }
  }
  for (int i = tid; i < n; i += nt) {
    d[i] = am[i];
    // tql2 keeps the sub-diagonal shifted down by one: e[i] couples i and i+1, e[n-1] = 0
    e[i] = (i < n - 1) ? sqrt(bm[i] * cm[i]) : 0.0;
  }
  for (size_t idx = tid; idx < (size_t)n * n; idx += nt) Zt[idx] = (idx / n == idx % n) ? 1.0 : 0.0;
  __syncthreads();

  // ---- QL iteration; thread 0 owns the scalar state
  double f = 0.0, tst1 = 0.0;
  int l = 0, iter = 0;
  bool fresh = true;  // first visit of this l
  while (true) {
    if (tid == 0) {
      int state = 0;
      // advance over converged eigenvalues, find the next unreduced block [l, m]
      while (true) {
        if (l >= n) {
          state = 1;
          break;
        }
        if (fresh) {
          const double h = fabs(d[l]) + fabs(e[l]);
          if (tst1 < h) tst1 = h;
          iter = 0;
          fresh = false;
        }
        int m = l;
        while (m < n - 1 && tst1 + fabs(e[m]) != tst1) ++m;
        if (m == l) {  // d[l] is an eigenvalue of the shifted matrix
          d[l] += f;
          ++l;
          fresh = true;
          continue;
        }
        if (++iter > kMaxQlIter) {
          state = 2;
          break;
        }
        // Wilkinson shift from the leading 2x2 of the block
        const int l1 = l + 1;
        double g = d[l];
        double p = (d[l1] - g) / (2.0 * e[l]);
        double r = hypot(p, 1.0);
        d[l] = e[l] / (p + sign_of(r, p));
        d[l1] = e[l] * (p + sign_of(r, p));
        const double dl1 = d[l1];
        double h = g - d[l];
        for (int i = l + 2; i < n; ++i) d[i] -= h;
        f += h;
        // the chase: rotations i = m-1 .. l
        p = d[m];
        double cc = 1.0, c2 = 1.0, c3 = 1.0, s = 0.0, s2 = 0.0;
        const double el1 = e[l1];
        for (int i = m - 1; i >= l; --i) {
          c3 = c2;
          c2 = cc;
          s2 = s;
          g = cc * e[i];
          h = cc * p;
          r = hypot(p, e[i]);
          e[i + 1] = s * r;
          s = e[i] / r;
          cc = p / r;
          p = cc * d[i] - s * g;
          d[i + 1] = h + s * (cc * g + s * d[i]);
          cs[i] = cc;
          sn[i] = s;
        }
        p = -s * s2 * c3 * el1 * e[l] / dl1;
        e[l] = s * p;
        d[l] = cc * p;
        sh_l = l;
        sh_m = m;
        break;
      }
      sh_state = state;
    }
    __syncthreads();
    const int state = sh_state;
    if (state != 0) {
      if (state == 2 && tid == 0) status[mat] = 1;
      if (state == 2) return;
      break;
    }
    // ---- apply the chase to the eigenvector rows: for i = m-1 .. l
    //      h = z[k][i+1]; z[k][i+1] = s z[k][i] + c h; z[k][i] = c z[k][i] - s h
    const int cl = sh_l, cm_ = sh_m;
    for (int k = tid; k < n; k += nt) {
      double hcar = Zt[(size_t)cm_ * n + k];
      for (int i = cm_ - 1; i >= cl; --i) {
        const double zi = Zt[(size_t)i * n + k];
        const double ci = cs[i], si = sn[i];
        Zt[(size_t)(i + 1) * n + k] = si * zi + ci * hcar;
        hcar = ci * zi - si * hcar;
      }
      Zt[(size_t)cl * n + k] = hcar;
    }
    __syncthreads();
  }
  // ---- ascending order (LAPACK's convention): rank by (value, index), scatter
  for (int k = tid; k < n; k += nt) {
    const double v = d[k];
    int rank = 0;
    for (int j = 0; j < n; ++j) rank += (d[j] < v) || (d[j] == v && j < k);
    lam[(size_t)mat * n + rank] = v;
    reinterpret_cast<int*>(cs)[k] = rank;
  }
  __syncthreads();
  const int* rk = reinterpret_cast<const int*>(cs);
  double* out = Qt + (size_t)mat * n * n;
  for (size_t idx = tid; idx < (size_t)n * n; idx += nt) {
    const int col = (int)(idx / n), row = (int)(idx % n);
    out[(size_t)rk[col] * n + row] = Zt[idx];
  }
  if (tid == 0) status[mat] = 0;
}

// out[set][r][q] = xi_r / xi_q * sum_k Q[r][k] phi1(s_set lambda_k) Q[q][k]
// (phi1_matrix: (V * f[None, :]) @ V_inv with V = diag(xi) Q, V_inv = Q^T diag(1/xi)).
// 32x32 output tile per CTA, k in slabs of 32 through shared memory.
__global__ void __launch_bounds__(256) phi1_matrix_kernel(int n, const double* __restrict__ lam,
                                                          const double* __restrict__ Qt,
                                                          const double* __restrict__ xi,
                                                          const int* __restrict__ mat_of_set,
                                                          const double* __restrict__ s, double* __restrict__ out) {
  __shared__ double As[32][33], Bs[32][33];  // As[k][r] = xi_r Q[r][k] f_k, Bs[k][q] = Q[q][k] / xi_q
  __shared__ double fs[32];                  // f_k = phi1(s lambda_k) of the slab
  const int set = blockIdx.z;
  const int mat = mat_of_set ? mat_of_set[set] : set;
  const double sc = s[set];
  const double* L = lam + (size_t)mat * n;
  const double* Z = Qt + (size_t)mat * n * n;  // Z[k][r] = Q[r][k]
  const double* X = xi + (size_t)mat * n;
  const int r0 = blockIdx.y * 32, q0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows of threads
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int k0 = 0; k0 < n; k0 += 32) {
    if (threadIdx.x < 32) fs[threadIdx.x] = (k0 + (int)threadIdx.x < n) ? phi1_dev(__dmul_rn(sc, L[k0 + threadIdx.x])) : 0.0;
    __syncthreads();
    for (int kk = ty; kk < 32; kk += 8) {
      const int k = k0 + kk;
      const int r = r0 + tx, q = q0 + tx;
      double va = 0.0, vb = 0.0;
      if (k < n) {
        if (r < n) va = __dmul_rn(__dmul_rn(X[r], Z[(size_t)k * n + r]), fs[kk]);
        if (q < n) vb = Z[(size_t)k * n + q] / X[q];
      }
      As[kk][tx] = va;
      Bs[kk][tx] = vb;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 32; ++kk) {
      const double bq = Bs[kk][tx];
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j] = fma(As[kk][ty + 8 * j], bq, acc[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int r = r0 + ty + 8 * j, q = q0 + tx;
    if (r < n && q < n) out[((size_t)set * n + r) * n + q] = acc[j];
  }
}

// out[set][i][j][k] = phi1(s_set * ((f1[set][i] * f2[set][j]) * f3[set][k]))  (f3 optional)
__global__ void __launch_bounds__(256) phi1_outer_kernel(int n1, int n2, int n3, const double* __restrict__ f1,
                                                         const double* __restrict__ f2,
                                                         const double* __restrict__ f3,
                                                         const double* __restrict__ s, double* __restrict__ out) {
  const int set = blockIdx.y;
  const size_t per = (size_t)n1 * n2 * n3;
  const double sc = s[set];
  const double* a = f1 + (size_t)set * n1;
  const double* bb = f2 + (size_t)set * n2;
  const double* cc = f3 ? f3 + (size_t)set * n3 : nullptr;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < per; idx += (size_t)gridDim.x * blockDim.x) {
    const int k = (int)(idx % n3);
    const size_t ij = idx / n3;
    const int j = (int)(ij % n2), i = (int)(ij / n2);
    double prod = __dmul_rn(a[i], bb[j]);
    if (cc) prod = __dmul_rn(prod, cc[k]);
    out[(size_t)set * per + idx] = phi1_dev(__dmul_rn(sc, prod));
  }
}

__global__ void phi1_kernel(long long count, const double* __restrict__ x, double* __restrict__ out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x)
    out[i] = phi1_dev(x[i]);
}

}  // namespace

extern "C" {

int cg_setup_eig_tridiag(int nmat, int n, const double* a, const double* b, const double* c, double* lam, double* Qt,
                         double* xi, double* work, int* status, void* stream) {
  if (!a || !b || !c || !lam || !Qt || !xi || !work || !status) return cg_internal_fail(CG_EINVAL, "null argument");
  if (nmat < 1 || n < 2) return cg_internal_fail(CG_EINVAL, "need nmat >= 1 and n >= 2");
  if (n > 4096) return cg_internal_fail(CG_EUNSUPPORTED, "operators above 4096 points are not supported");
  if (work == Qt) return cg_internal_fail(CG_EINVAL, "work and Qt must be distinct buffers");
  const size_t smem = (size_t)4 * n * sizeof(double);
  if (smem > 48 * 1024)
    SETUP_TRY(cudaFuncSetAttribute(eig_tridiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  eig_tridiag_kernel<<<(unsigned)nmat, kEigThreads, smem, static_cast<cudaStream_t>(stream)>>>(n, a, b, c, lam, Qt, xi,
                                                                                                work, status);
  SETUP_TRY(cudaGetLastError());
  return CG_OK;
}

int cg_setup_phi1_matrix(int nset, int n, const double* lam, const double* Qt, const double* xi,
                         const int* mat_of_set, const double* s, double* out, void* stream) {
  if (!lam || !Qt || !xi || !s || !out) return cg_internal_fail(CG_EINVAL, "null argument");
  if (nset < 1 || n < 1 || nset > 65535) return cg_internal_fail(CG_EINVAL, "need 1 <= nset <= 65535 and n >= 1");
  const unsigned t = (unsigned)((n + 31) / 32);
  phi1_matrix_kernel<<<dim3(t, t, (unsigned)nset), 256, 0, static_cast<cudaStream_t>(stream)>>>(n, lam, Qt, xi,
                                                                                                 mat_of_set, s, out);
  SETUP_TRY(cudaGetLastError());
  return CG_OK;
}

int cg_setup_phi1_outer(int nset, int n1, int n2, int n3, const double* f1, const double* f2, const double* f3,
                        const double* s, double* out, void* stream) {
  if (!f1 || !f2 || !s || !out) return cg_internal_fail(CG_EINVAL, "null argument");
  if (nset < 1 || nset > 65535 || n1 < 1 || n2 < 1 || n3 < 1)
    return cg_internal_fail(CG_EINVAL, "need 1 <= nset <= 65535 and positive extents");
  if (!f3 && n3 != 1) return cg_internal_fail(CG_EINVAL, "n3 must be 1 without a third factor");
  const size_t per = (size_t)n1 * n2 * n3;
  const unsigned blocks = (unsigned)std::min<size_t>((per + 255) / 256, 148 * 8);
  phi1_outer_kernel<<<dim3(blocks, (unsigned)nset), 256, 0, static_cast<cudaStream_t>(stream)>>>(n1, n2, n3, f1, f2,
                                                                                                  f3, s, out);
  SETUP_TRY(cudaGetLastError());
  return CG_OK;
}

int cg_setup_phi1(long long count, const double* x, double* out, void* stream) {
  if (!x || !out) return cg_internal_fail(CG_EINVAL, "null argument");
  if (count < 1) return cg_internal_fail(CG_EINVAL, "count must be positive");
  const unsigned blocks = (unsigned)std::min<long long>((count + 255) / 256, 148 * 8);
  phi1_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(count, x, out);
  SETUP_TRY(cudaGetLastError());
  return CG_OK;
}

}  // extern "C"
