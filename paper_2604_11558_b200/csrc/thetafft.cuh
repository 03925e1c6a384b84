// Fused theta propagator: y = Q_theta diag(Phi_line) Q_theta^T x along the
// periodic theta axis, by FFT.
//
// The reference applies phi1 of the theta summand as two dense mu-mode
// products with the real Fourier eigenbasis Q_theta (operators.py:142-169)
// around a Hadamard with a phi1 tensor (integrators.py:204-206, :211-214,
// :232-234): T = ((X Q) o Phi) Q^T.  Because Q's columns are the
// cos/sin pairs of frequency j with equal eigenvalues, Phi is equal on both
// columns of a pair and the triple product is exactly
//     y = IDFT_N( Phi_j * DFT_N(x) ),   Phi_j = Phi[col(j)],
//     col(0) = 0, col(j) = 2j - 1 (0 < j < N/2), col(N/2) = N - 1,
// i.e. a real circular convolution.  It is evaluated with a half-length
// complex FFT (z_k = x_2k + i x_2k+1, M = N/2 points), the real-FFT
// split/merge twiddles, the real Phi_j scaling, and the inverse, all in
// shared memory: O(N log N) work instead of 2 N^2 per line, one HBM read and
// one write per value.  N must be a power of two (radix-4 Stockham stages
// plus at most one radix-2 stage) for the Stockham kernel; the register
// two-phase kernel also takes M = 50 = 5 x 10 (the ball's n_theta = 100).
//
// A field is viewed as [A][N][Bc] (A = axes before theta, Bc = axes after);
// a CTA owns W lines: W consecutive a (Bc == 1, contiguous rows) or W
// consecutive bc (Bc > 1, lines are columns).  Epilogue: store, or
// W_out = W + tau * y with the divergence guard (sphere: theta is the last
// factor of its chain).
#pragma once

#include "common.cuh"

namespace cg {

struct ThetaParams {
  int N;             // theta extent (power of two)
  int A, Bc;         // field = [A][N][Bc]
  int nfield, ncomp;
  long long npts;    // A * N * Bc
  int W;             // lines per CTA
  int phi_class_a;   // Phi class of a line: 1 = a (disk, cylinder), 0 = bc (sphere), 2 = a*Bc + bc (ball)
  int nclass;        // classes per component
  const double* phif;  // [C][nclass][N/2 + 1] Phi_j
  // the same values pre-scaled for theta_tail (Phi_0, Phi_M by 1/(2M), the
  // rest by 1/(4M): exact powers of two that absorb the split/merge halves
  // and the inverse 1/M), rows padded to phis_ld (bank-conflict free in smem)
  const double* phis;
  int phis_ld;
  const double2* tw;   // [N] exp(-2 pi i t / N)
  const double* X;
  double* Y;
  const double* Wprev;  // AXPY: previous state
  double tau, limit;
  int* first_bad;
  const int* step;
  // cluster step kernel (cluster_disk.cuh): shared-space address of the
  // [2][N/2][8] column slab every CTA of the cluster holds at the same offset
  unsigned cl_slab;
  unsigned cl_bar;  // shared-space address of the mbarrier counting the slab's bytes (same offset in every CTA)
};

// dynamic shared memory: two [W][M+1] complex ping-pong buffers + N twiddles
inline size_t theta_smem_bytes(int N, int W) {
  return (size_t)(2 * W * (N / 2 + 1) + N) * sizeof(double2);
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

// One Stockham pass of radix R (4 or 2) over W lines of M points:
// src/dst are [W][M + 1] (padded rows).  INV selects the inverse sign.
template <int R, bool INV>
__device__ __forceinline__ void stockham_pass(const double2* src, double2* dst, int M, int W, int ns,
                                              const double2* tw, int twN) {
  const int q = M / R;  // butterflies per line
  const int ld = M + 1;
  for (int idx = threadIdx.x; idx < W * q; idx += blockDim.x) {
    const int w = idx / q;
    const int j = idx - w * q;
    const int k = j % ns;
    const double2* s = src + w * ld;
    double2* d = dst + w * ld;
    // twiddle exp(-+2 pi i k / (R ns)) from the length-twN table
    const int step = twN / (R * ns);
    if (R == 4) {
      double2 a0 = s[j], a1 = s[j + q], a2 = s[j + 2 * q], a3 = s[j + 3 * q];
      if (ns > 1) {
        double2 w1 = tw[k * step], w2 = tw[2 * k * step], w3 = tw[3 * k * step];
        if (INV) {
          w1 = cconj(w1);
          w2 = cconj(w2);
          w3 = cconj(w3);
        }
        a1 = cmul(a1, w1);
        a2 = cmul(a2, w2);
        a3 = cmul(a3, w3);
      }
      const double2 b0 = cadd(a0, a2), b1 = csub(a0, a2), b2 = cadd(a1, a3);
      const double2 t = csub(a1, a3);
      const double2 b3 = INV ? make_double2(-t.y, t.x) : make_double2(t.y, -t.x);  // +-i * (a1 - a3)
      const int base = (j / ns) * 4 * ns + k;
      d[base] = cadd(b0, b2);
      d[base + ns] = cadd(b1, b3);
      d[base + 2 * ns] = csub(b0, b2);
      d[base + 3 * ns] = csub(b1, b3);
    } else {
      double2 a0 = s[j], a1 = s[j + q];
      if (ns > 1) {
        double2 w1 = tw[k * step];
        if (INV) w1 = cconj(w1);
        a1 = cmul(a1, w1);
      }
      const int base = (j / ns) * 2 * ns + k;
      d[base] = cadd(a0, a1);
      d[base + ns] = csub(a0, a1);
    }
  }
}

// Complex FFT of length M on W lines, result returned in *cur (ping-pong).
template <bool INV>
__device__ __forceinline__ void fft_lines(double2*& cur, double2*& alt, int M, int W, const double2* tw, int twN) {
  int ns = 1;
  while (ns * 4 <= M) {
    stockham_pass<4, INV>(cur, alt, M, W, ns, tw, twN);
    __syncthreads();
    double2* t = cur;
    cur = alt;
    alt = t;
    ns *= 4;
  }
  if (ns < M) {
    stockham_pass<2, INV>(cur, alt, M, W, ns, tw, twN);
    __syncthreads();
    double2* t = cur;
    cur = alt;
    alt = t;
  }
}

template <bool AXPY>
__global__ void __launch_bounds__(256) theta_prop_kernel(const ThetaParams p) {
  pdl_wait();
  extern __shared__ double2 tp_smem[];
  const int N = p.N, M = N / 2, W = p.W, ld = M + 1;
  double2* bufA = tp_smem;
  double2* bufB = tp_smem + W * ld;
  double2* twS = tp_smem + 2 * W * ld;  // [N]

  // CTA -> (field, a0, bc0)
  const int Bc = p.Bc;
  int blk = blockIdx.x;
  int f, a0, bc0;
  if (Bc == 1) {
    const int per = p.A / W;
    f = blk / per;
    a0 = (blk - f * per) * W;
    bc0 = 0;
  } else {
    const int per = Bc / W;
    const int pa = blk / per;
    bc0 = (blk - pa * per) * W;
    f = pa / p.A;
    a0 = pa - f * p.A;
  }
  const int c = f % p.ncomp;
  const long long fbase = (long long)f * p.npts;
  const long long lstride = (long long)N * Bc;  // stride between consecutive a

  for (int t = threadIdx.x; t < N; t += blockDim.x) twS[t] = __ldg(p.tw + t);

  // ---- load: z_k = x_2k + i x_2k+1 for each of the W lines
  if (Bc == 1) {
    for (int idx = threadIdx.x; idx < W * M; idx += blockDim.x) {
      const int w = idx / M, k = idx - w * M;
      const double2 v = __ldg(reinterpret_cast<const double2*>(p.X + fbase + (long long)(a0 + w) * lstride) + k);
      bufA[w * ld + k] = v;
    }
  } else {
    const long long base = fbase + (long long)a0 * lstride + bc0;
    for (int idx = threadIdx.x; idx < W * M; idx += blockDim.x) {
      const int w = idx % W, k = idx / W;
      const double x0 = __ldg(p.X + base + (long long)(2 * k) * Bc + w);
      const double x1 = __ldg(p.X + base + (long long)(2 * k + 1) * Bc + w);
      bufA[w * ld + k] = make_double2(x0, x1);
    }
  }
  __syncthreads();

  double2* cur = bufA;
  double2* alt = bufB;
  fft_lines<false>(cur, alt, M, W, twS, N);

  // ---- split to the real spectrum X_j (j = 0..M), scale by Phi_j, merge
  //      back to the half-length spectrum Z'_j of the inverse (in place).
  const int half = M / 2;
  for (int idx = threadIdx.x; idx < W * (half + 1); idx += blockDim.x) {
    const int w = idx / (half + 1), j = idx - w * (half + 1);
    const int la = (Bc == 1) ? a0 + w : a0, lbc = (Bc == 1) ? 0 : bc0 + w;
    const int cls = p.phi_class_a == 1 ? la : (p.phi_class_a == 0 ? lbc : la * Bc + lbc);
    const double* ph = p.phif + ((long long)c * p.nclass + cls) * (M + 1);
    double2* z = cur + w * ld;
    if (j == 0) {
      const double2 z0 = z[0];
      const double x0 = (z0.x + z0.y) * ph[0];   // X_0 * Phi_0
      const double xm = (z0.x - z0.y) * ph[M];   // X_M * Phi_M
      // Z'_0 = (Y_0 + Y_M)/2 + i (Y_0 - Y_M)/2
      z[0] = make_double2(0.5 * (x0 + xm), 0.5 * (x0 - xm));
      continue;
    }
    const int jm = M - j;
    const double2 zj = z[j], zm = z[jm];
    // E_j = (Z_j + conj Z_{M-j})/2, O_j = (Z_j - conj Z_{M-j})/(2i)
    const double2 e = make_double2(0.5 * (zj.x + zm.x), 0.5 * (zj.y - zm.y));
    const double2 o = make_double2(0.5 * (zj.y + zm.y), -0.5 * (zj.x - zm.x));
    const double2 wj = twS[j];  // exp(-2 pi i j / N)
    const double2 wo = cmul(wj, o);
    // X_j = E + w^j O,  X_{M-j} = conj(E) - conj(w^j O)  (w^{M-j} = -conj(w^j))
    double2 xj = cadd(e, wo);
    double2 xmj = make_double2(e.x - wo.x, -(e.y - wo.y));
    xj.x *= ph[j];
    xj.y *= ph[j];
    xmj.x *= ph[jm];
    xmj.y *= ph[jm];
    // merge: Z'_j = (Y_j + conj Y_{M-j})/2 + i conj(w^j) (Y_j - conj Y_{M-j})/2
    const double2 s1 = make_double2(0.5 * (xj.x + xmj.x), 0.5 * (xj.y - xmj.y));
    const double2 d1 = make_double2(0.5 * (xj.x - xmj.x), 0.5 * (xj.y + xmj.y));
    const double2 wd = cmul(cconj(wj), d1);
    z[j] = make_double2(s1.x - wd.y, s1.y + wd.x);
    if (jm != j) {
      // Z'_{M-j} from the same pair (roles of j and M-j swapped)
      const double2 s2 = make_double2(0.5 * (xmj.x + xj.x), 0.5 * (xmj.y - xj.y));
      const double2 d2 = make_double2(0.5 * (xmj.x - xj.x), 0.5 * (xmj.y + xj.y));
      const double2 wmj = make_double2(-wj.x, wj.y);  // exp(-2 pi i (M-j)/N) = -conj(w^j)
      const double2 wd2 = cmul(cconj(wmj), d2);
      z[jm] = make_double2(s2.x - wd2.y, s2.y + wd2.x);
    }
  }
  __syncthreads();
  fft_lines<true>(cur, alt, M, W, twS, N);

  // ---- store y_2k = Re z'_k / M, y_2k+1 = Im z'_k / M (+ axpy / guard)
  const double scale = 1.0 / (double)M;
  bool bad = false;
  if (Bc == 1) {
    for (int idx = threadIdx.x; idx < W * M; idx += blockDim.x) {
      const int w = idx / M, k = idx - w * M;
      const double2 z = cur[w * ld + k];
      const long long o = fbase + (long long)(a0 + w) * lstride + 2 * k;
      double y0 = z.x * scale, y1 = z.y * scale;
      if (AXPY) {
        const double2 wv = __ldg(reinterpret_cast<const double2*>(p.Wprev + o));
        y0 = __dadd_rn(wv.x, __dmul_rn(p.tau, y0));
        y1 = __dadd_rn(wv.y, __dmul_rn(p.tau, y1));
        bad |= !(fabs(y0) <= p.limit) || !(fabs(y1) <= p.limit);
      }
      *reinterpret_cast<double2*>(p.Y + o) = make_double2(y0, y1);
    }
  } else {
    const long long base = fbase + (long long)a0 * lstride + bc0;
    for (int idx = threadIdx.x; idx < W * M; idx += blockDim.x) {
      const int w = idx % W, k = idx / W;
      const double2 z = cur[w * ld + k];
      const long long o0 = base + (long long)(2 * k) * Bc + w, o1 = o0 + Bc;
      double y0 = z.x * scale, y1 = z.y * scale;
      if (AXPY) {
        y0 = __dadd_rn(__ldg(p.Wprev + o0), __dmul_rn(p.tau, y0));
        y1 = __dadd_rn(__ldg(p.Wprev + o1), __dmul_rn(p.tau, y1));
        bad |= !(fabs(y0) <= p.limit) || !(fabs(y1) <= p.limit);
      }
      p.Y[o0] = y0;
      p.Y[o1] = y1;
    }
  }
  if (AXPY) {
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicMin(p.first_bad + f, *p.step);
  }
}

// ---------------------------------------------------------------------------
// Register-resident two-phase FFT (M = M1 * M2, M1, M2 <= 16).
// Phase A: thread n2 takes z[n2 + M2 n1], DFT_M1 over n1 in registers,
// twiddle w_M^(n2 k1); padded smem transpose; phase B: thread k1 takes the M2
// values of row k1, DFT_M2 in registers -> X[k1 + M1 k2].  One smem round
// trip per transform instead of log4(M) Stockham passes.
// ---------------------------------------------------------------------------

__host__ __device__ constexpr double cos16(int k) {
  // cos(2 pi k / 16), exact-symmetric correctly rounded values
  return k == 0 ? 1.0 : k == 1 ? 0.9238795325112867 : k == 2 ? 0.7071067811865476 : k == 3 ? 0.3826834323650898
       : k == 4 ? 0.0 : k == 5 ? -0.3826834323650898 : k == 6 ? -0.7071067811865476 : k == 7 ? -0.9238795325112867
       : k == 8 ? -1.0 : k == 9 ? -0.9238795325112867 : k == 10 ? -0.7071067811865476 : k == 11 ? -0.3826834323650898
       : k == 12 ? 0.0 : k == 13 ? 0.3826834323650898 : k == 14 ? 0.7071067811865476 : 0.9238795325112867;
}
__host__ __device__ constexpr double sin16(int k) { return cos16((k + 12) & 15); }  // sin x = cos(x - pi/2)

__host__ __device__ constexpr int bitrev(int i, int L) {
  int r = 0;
  for (int b = 1; b < L; b <<= 1) r = (r << 1) | ((i & b) ? 1 : 0);
  return r;
}

// One radix-2 DIT stage of sub-transform length LEN, then the next (template
// recursion so every index is a compile-time constant and `a` stays in
// registers; nested runtime-bounded loops left it in local memory).
template <int L, int LEN, bool INV>
__device__ __forceinline__ void dit_stage(double2* a) {
  constexpr int half = LEN / 2;
#pragma unroll
  for (int q = 0; q < L / 2; ++q) {
    const int st = (q / half) * LEN, j = q % half;
    const double2 u = a[st + j];
    double2 v = a[st + j + half];
    if (j != 0) {
      const int t = j * (16 / LEN);
      const double c = cos16(t), s = INV ? sin16(t) : -sin16(t);
      if (t == 4) {
        v = INV ? make_double2(-v.y, v.x) : make_double2(v.y, -v.x);  // w = +-i: free
      } else if (t == 2 || t == 6) {
        // |c| = |s| = sqrt(1/2): two adds and two multiplies
        const double h = 0.7071067811865476;
        const double re = (c > 0 ? v.x : -v.x) - (s > 0 ? v.y : -v.y);
        const double im = (s > 0 ? v.x : -v.x) + (c > 0 ? v.y : -v.y);
        v = make_double2(h * re, h * im);
      } else {
        v = make_double2(v.x * c - v.y * s, v.x * s + v.y * c);
      }
    }
    a[st + j] = make_double2(u.x + v.x, u.y + v.y);
    a[st + j + half] = make_double2(u.x - v.x, u.y - v.y);
  }
  if constexpr (LEN < L) dit_stage<L, LEN * 2, INV>(a);
}

// In-register DFT of length L (power of two <= 16), natural order in and out.
template <int L, bool INV>
__device__ __forceinline__ void dft_reg(double2* a) {
#pragma unroll
  for (int i = 0; i < L; ++i) {
    const int r = bitrev(i, L);
    if (r > i) {
      const double2 t = a[i];
      a[i] = a[r];
      a[r] = t;
    }
  }
  if constexpr (L > 1) dit_stage<L, 2, INV>(a);
}

// NT threads per CTA: 256, or 64 for problems with too few lines to give
// every SM a CTA at 256 (the sphere's 512 theta columns, config 1's disk)
// Odd-factor DFTs for theta extents that are not powers of two (the ball's
// n_theta = 100: M = 50 = 5 x 10).  5-point: the real-coefficient pair form
// (t1 = x1 + x4, t2 = x2 + x3, t3 = x1 - x4, t4 = x2 - x3); 10-point: one
// radix-2 step over two 5-point DFTs.
__device__ __forceinline__ double2 mul_mi(double2 v) { return make_double2(v.y, -v.x); }  // -i v
__device__ __forceinline__ double2 mul_pi(double2 v) { return make_double2(-v.y, v.x); }  // +i v

template <bool INV>
__device__ __forceinline__ void dft5(double2& x0, double2& x1, double2& x2, double2& x3, double2& x4) {
  constexpr double c1 = 0.30901699437494745, c2 = -0.8090169943749475;   // cos(2 pi/5), cos(4 pi/5)
  constexpr double s1 = 0.9510565162951535, s2 = 0.5877852522924731;     // sin(2 pi/5), sin(4 pi/5)
  const double2 t1 = cadd(x1, x4), t2 = cadd(x2, x3), t3 = csub(x1, x4), t4 = csub(x2, x3);
  const double2 a1 = make_double2(x0.x + c1 * t1.x + c2 * t2.x, x0.y + c1 * t1.y + c2 * t2.y);
  const double2 a2 = make_double2(x0.x + c2 * t1.x + c1 * t2.x, x0.y + c2 * t1.y + c1 * t2.y);
  const double2 b1 = make_double2(s1 * t3.x + s2 * t4.x, s1 * t3.y + s2 * t4.y);
  const double2 b2 = make_double2(s2 * t3.x - s1 * t4.x, s2 * t3.y - s1 * t4.y);
  x0 = cadd(x0, cadd(t1, t2));
  const double2 ib1 = INV ? mul_pi(b1) : mul_mi(b1), ib2 = INV ? mul_pi(b2) : mul_mi(b2);
  x1 = cadd(a1, ib1);
  x4 = csub(a1, ib1);
  x2 = cadd(a2, ib2);
  x3 = csub(a2, ib2);
}

template <bool INV>
__device__ __forceinline__ void dft10(double2* a) {
  double2 e[5] = {a[0], a[2], a[4], a[6], a[8]}, o[5] = {a[1], a[3], a[5], a[7], a[9]};
  dft5<INV>(e[0], e[1], e[2], e[3], e[4]);
  dft5<INV>(o[0], o[1], o[2], o[3], o[4]);
  constexpr double cs[5] = {1.0, 0.8090169943749475, 0.30901699437494745, -0.30901699437494745, -0.8090169943749475};
  constexpr double sn[5] = {0.0, 0.5877852522924731, 0.9510565162951535, 0.9510565162951535, 0.5877852522924731};
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const double s = INV ? sn[k] : -sn[k];  // w_10^k = cos - i sin (forward)
    const double2 w = make_double2(o[k].x * cs[k] - o[k].y * s, o[k].x * s + o[k].y * cs[k]);
    a[k] = cadd(e[k], w);
    a[k + 5] = csub(e[k], w);
  }
}

// DFT of length L in registers, natural order in and out
template <int L, bool INV>
__device__ __forceinline__ void dft_any(double2* a) {
  if constexpr ((L & (L - 1)) == 0) {
    dft_reg<L, INV>(a);
  } else if constexpr (L == 5) {
    dft5<INV>(a[0], a[1], a[2], a[3], a[4]);
  } else if constexpr (L == 10) {
    dft10<INV>(a);
  } else {
    static_assert(L == 0, "unsupported DFT length");
  }
}

#ifdef CURVIGPU_TAIL_CTA_SYNC
constexpr bool kTailCtaSync = true;   // A/B build: CTA barriers around the line transposes
#else
constexpr bool kTailCtaSync = false;
#endif

template <int M1, int M2, int NT = 256>
struct FastTheta {
  static constexpr int M = M1 * M2;
  // threads per line = min(M1, M2): in each phase every thread runs
  // max/min DFTs, so no lane idles during the heavy phase
  static constexpr int TPL = M1 < M2 ? M1 : M2;
  static constexpr int LPB = NT / TPL;           // lines per CTA
  static constexpr int LDT = M1 * (M2 + 1);      // padded transpose tile (complex)
  static constexpr int SL0 = LDT > M ? LDT : M;
  static constexpr int SL = (SL0 % 2 == 0) ? SL0 + 1 : SL0;  // odd line stride: lines land on distinct banks
  static constexpr size_t smem = (size_t)LPB * SL * sizeof(double2);
  // column kernels (theta_fast_kernel, !ROWS) also stage the N twiddles and
  // their lines' scaled Phi rows (row stride PS = plan.cu phis_stride(M))
  static constexpr int PS = ((M + 1 + 7) / 8 * 8) % 16 == 0 ? (M + 1 + 7) / 8 * 8 + 8 : (M + 1 + 7) / 8 * 8;
  static constexpr size_t smem_cols = smem + (size_t)2 * M * sizeof(double2) + (size_t)LPB * PS * sizeof(double);
};

// table read: read-only global path, or shared memory (TS) when a kernel
// stages the Phi rows and twiddles itself
template <bool TS, typename T>
__device__ __forceinline__ T ldt(const T* p) {
  if constexpr (TS)
    return *p;
  else
    return __ldg(p);
}

// forward phase A for column n2: M1 loaded values -> DFT_M1 -> twiddle -> S.
// tw: the length-2M table (w_M^(n2 k1) = tw[2 n2 k1]), or with TA a [M1][M2]
// table of exactly those values (shared memory: a quarter-warp's lanes then
// read consecutive entries instead of a stride of 2 k1, bank-conflict free)
template <int M1, int M2, bool INV, bool TS = false, bool TA = false>
__device__ __forceinline__ void phase_a(double2* r, double2* S, int n2, const double2* tw) {
  dft_any<M1, INV>(r);
#pragma unroll
  for (int k1 = 1; k1 < M1; ++k1) {
    const double2 w = ldt<TS>(TA ? tw + k1 * M2 + n2 : tw + 2 * n2 * k1);
    r[k1] = cmul(r[k1], INV ? cconj(w) : w);
  }
#pragma unroll
  for (int k1 = 0; k1 < M1; ++k1) S[k1 * (M2 + 1) + n2] = r[k1];
}

// Everything after forward phase A (every column's M1 twiddled values are in
// S's padded transpose layout, not yet synchronised): forward phase B, real
// split, Phi, merge, inverse FFT, scaled store (+ W + tau*y and the guard).
// ph = this line's Phi_j row (M + 1 values), tw = the N twiddles; both in
// global memory, or in shared memory when TS.
// Real split, Phi scaling and merge of one (j, M - j) pair: the textbook
// split/merge with every 1/2 and the inverse 1/M folded into the pre-scaled Phi
// row, which holds sg = Phi'_j + Phi'_{M-j} at j and dl = Phi'_j - Phi'_{M-j} at
// M - j (0 < j < M/2; 2 Phi'_{M/2} at M/2, paired with dl = 0): with e = 2 E_j,
// B = w^j 2 O_j the scaled spectrum values enter only as
//   s = X_j + conj(X_{M-j}) = sg e + dl B,   d = X_j - conj(X_{M-j}) = dl e + sg B,
// 24 FP64 instructions per pair instead of 28 with the two factors applied
// separately.  Returns Z'_j in zj_out and Z'_{M-j} in zm_out.
__device__ __forceinline__ void split_pair(double2 zj, double2 zm, double2 wj, double sg, double dl, double2& zj_out,
                                           double2& zm_out) {
  const double2 e = make_double2(zj.x + zm.x, zj.y - zm.y);    // 2 E_j
  const double2 o = make_double2(zj.y + zm.y, zm.x - zj.x);    // 2 O_j
  const double2 wo = cmul(wj, o);
  const double2 s1 = make_double2(sg * e.x + dl * wo.x, sg * e.y + dl * wo.y);
  const double2 d1 = make_double2(dl * e.x + sg * wo.x, dl * e.y + sg * wo.y);
  const double2 wd = cmul(cconj(wj), d1);
  zj_out = make_double2(s1.x - wd.y, s1.y + wd.x);
  zm_out = make_double2(s1.x + wd.y, wd.x - s1.y);
}

__device__ __forceinline__ double2 shfl_d2(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

// RS (register split): when a line's TPL = M1 threads are consecutive lanes of
// one warp, forward phase B leaves thread lt holding Z[lt + M1 k2] (k2 < M2),
// which are exactly the inputs of its inverse phase-A columns n2 = lt + q M1.
// The split/merge partner of index j = lt + M1 k2 is M - j = (M1 - lt) +
// M1 (M2 - 1 - k2), held by lane M1 - lt (lt = 0 pairs with itself: k2 <->
// M2 - k2).  Each thread computes the pairs of its lower half k2 < M2/2 (both
// outputs) from its partner's upper half received by shuffle, and sends the
// partner's outputs back: the phase-B store, the split's shared-memory round
// trip, the inverse phase-A load and two barriers disappear.  Same pairs,
// same formulas, so the results equal the shared-memory path bit for bit.
// BCM: 1 = lines are contiguous rows (Bc == 1), 2 = lines are columns
// (Bc > 1), 0 = decided at run time.  A compile-time layout keeps the layout
// branch out of the store loop, so its W loads are batched ahead of the stores.
// CLS (cluster step kernel): a line's results are pushed over DSMEM into the
// column slabs of the CTAs that own the columns -- base = line * N with lines
// ordered [species][4 rows of cluster rank r], column pair 2k goes to CTA k / 4
// at [species][rho row][2k % 8].
// TWA: with TS, twa holds the phase-A twiddles as a [M1][M2] table (the disk
// front); without it phase A reads them from the staged length-N table tw.
template <int M1, int M2, bool AXPY, bool TS = false, bool RS = false, int BCM = 0, bool CLS = false, bool TWA = TS>
__device__ __forceinline__ void theta_tail(const ThetaParams& p, double2* S, int lt, const double* ph,
                                           const double2* tw, int f, long long base, long long es, int Bc,
                                           const double2* twa = nullptr) {
  using F = FastTheta<M1, M2>;
  constexpr int M = F::M, TPL = F::TPL;
  constexpr int RMAX = M1 > M2 ? M1 : M2;
  double2 r[RMAX];
  // column lines with the axpy epilogue (the sphere: few, latency-bound CTAs)
  // issue their W loads before the whole tail, so they land under the FFT
  constexpr bool EARLY = AXPY && BCM == 2 && M1 / TPL == 1;
  double2 wearly[EARLY ? M2 : 1];
  if constexpr (EARLY) {
#pragma unroll
    for (int k2 = 0; k2 < M2; ++k2) {
      const long long o0 = base + (2LL * (lt + M1 * k2)) * es;
      wearly[k2] = make_double2(__ldg(p.Wprev + o0), __ldg(p.Wprev + o0 + es));
    }
  }
  // RS lines live in one warp and S is private to a line, so the transposes
  // only need warp-level ordering: the CTA's warps then drift apart and one
  // warp's shared-memory phases run under another's FP64 phases
  if constexpr (RS && !kTailCtaSync)
    __syncwarp();
  else
    __syncthreads();
  if constexpr (RS) {
    static_assert(TPL == M1 && (TPL & (TPL - 1)) == 0 && TPL <= 32 && M2 % 2 == 0, "register split layout");
    constexpr int H = M2 / 2;
    // ---------------- forward phase B: row k1 = lt -> keep[k2] = Z[lt + M1 k2]
    double2 keep[M2];
#pragma unroll
    for (int n2 = 0; n2 < M2; ++n2) keep[n2] = S[lt * (M2 + 1) + n2];
    dft_any<M2, false>(keep);
    // ---------------- split / Phi / merge in registers
    const int lane = threadIdx.x & 31;
    const int src = (lane & ~(TPL - 1)) | ((TPL - lt) & (TPL - 1));
    const bool z0 = lt == 0;
    double2 out_hi[H];  // outputs for the partner's slots M2 - 1 - h (lt = 0: own slots M2 - h)
    double2 selfm{};    // lt = 0: Z'_{M/2}
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const double2 zin = shfl_d2(keep[M2 - 1 - h], src);   // partner's Z[M - j]
      const double2 zm = z0 ? keep[(M2 - h) & (M2 - 1)] : zin;
      const int j = lt + M1 * h;
      const int jm = z0 ? ((M - M1 * h) & (M - 1)) : M - j;
      const double2 wj = ldt<TS>(tw + j);
      // (j = 0: the row holds Phi'_0 at 0 and Phi'_M at M, applied below)
      const double pj = ldt<TS>(ph + j), pm = ldt<TS>(ph + (h == 0 && z0 ? M : jm));
      double2 oj, om;
      split_pair(keep[h], zm, wj, pj, pm, oj, om);
      if (h == 0 && z0) {  // j = 0: DC and Nyquist packed in Z_0
        const double2 zz = keep[0];
        const double x0 = (zz.x + zz.y) * pj;
        const double xm = (zz.x - zz.y) * pm;
        oj = make_double2(x0 + xm, x0 - xm);
      }
      if (h == 0) {
        // lt = 0 also owns the self-paired j = M/2 (k2 = M2/2)
        const double2 zh = keep[H];
        double2 oh, unused;
        split_pair(zh, zh, ldt<TS>(tw + M / 2), ldt<TS>(ph + M / 2), 0.0, oh, unused);
        selfm = oh;
      }
      keep[h] = oj;
      out_hi[h] = om;
    }
    // partner's outputs for this thread's upper half
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const double2 back = shfl_d2(out_hi[h], src);
      // slot M2 - 1 - h: from the partner, or (lt = 0) own pair h + 1 / the M/2 self pair
      keep[M2 - 1 - h] = z0 ? (h + 1 < H ? out_hi[h + 1] : selfm) : back;
    }
    // every thread has read its S row (phase B) before phase A overwrites S
    if constexpr (kTailCtaSync)
      __syncthreads();
    else
      __syncwarp();
    // ---------------- inverse phase A from registers: column n2 = lt + q M1 holds k2 = q + (M2/M1) n1
#pragma unroll
    for (int q = 0; q < M2 / TPL; ++q) {
      double2 col[M1];
#pragma unroll
      for (int n1 = 0; n1 < M1; ++n1) col[n1] = keep[q + (M2 / M1) * n1];
      if constexpr (TWA)
        phase_a<M1, M2, true, true, true>(col, S, lt + q * TPL, twa);
      else
        phase_a<M1, M2, true, TS>(col, S, lt + q * TPL, tw);
    }
  } else {
  // ---------------- forward phase B: rows k1 = lt, lt + TPL, ...
  double2 keep[M1 / TPL][M2];
#pragma unroll
  for (int q = 0; q < M1 / TPL; ++q) {
    const int k1 = lt + q * TPL;
#pragma unroll
    for (int n2 = 0; n2 < M2; ++n2) keep[q][n2] = S[k1 * (M2 + 1) + n2];
    dft_any<M2, false>(keep[q]);
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < M1 / TPL; ++q) {
    const int k1 = lt + q * TPL;
#pragma unroll
    for (int k2 = 0; k2 < M2; ++k2) S[k1 + M1 * k2] = keep[q][k2];
  }
  __syncthreads();
  // ---------------- split to X_j, scale by Phi_j, merge to Z'_j (pairs j, M-j)
  // ph is the pre-scaled row (ThetaParams::phis): every 1/2 of the textbook
  // split/merge and the inverse 1/M are folded into it (exact powers of two),
  // and Z'_{M-j} = conj(s - i w^-j d) reuses the pair's s, d (both exact
  // identities), so the values equal the unscaled form's
  {
    for (int j = lt; j <= M / 2; j += TPL) {
      if (j == 0) {
        const double2 z0 = S[0];
        const double x0 = (z0.x + z0.y) * ldt<TS>(ph);
        const double xm = (z0.x - z0.y) * ldt<TS>(ph + M);
        S[0] = make_double2(x0 + xm, x0 - xm);
        continue;
      }
      const int jm = M - j;
      const double2 zj = S[j], zm = S[jm];
      const double2 e = make_double2(zj.x + zm.x, zj.y - zm.y);    // 2 E_j
      const double2 o = make_double2(zj.y + zm.y, zm.x - zj.x);    // 2 O_j
      const double2 wj = ldt<TS>(tw + j);
      const double2 wo = cmul(wj, o);
      const double sg = ldt<TS>(ph + j), dl = jm != j ? ldt<TS>(ph + jm) : 0.0;  // split_pair's form
      const double2 s1 = make_double2(sg * e.x + dl * wo.x, sg * e.y + dl * wo.y);
      const double2 d1 = make_double2(dl * e.x + sg * wo.x, dl * e.y + sg * wo.y);
      const double2 wd = cmul(cconj(wj), d1);
      S[j] = make_double2(s1.x - wd.y, s1.y + wd.x);
      if (jm != j) S[jm] = make_double2(s1.x + wd.y, wd.x - s1.y);
    }
  }
  __syncthreads();
  // ---------------- inverse phase A: columns n2 = lt, lt + TPL, ...
  double2 keepa[M2 / TPL][M1];
#pragma unroll
  for (int q = 0; q < M2 / TPL; ++q) {
    const int n2 = lt + q * TPL;
#pragma unroll
    for (int n1 = 0; n1 < M1; ++n1) keepa[q][n1] = S[n2 + M2 * n1];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < M2 / TPL; ++q) {
    if constexpr (TWA)
      phase_a<M1, M2, true, true, true>(keepa[q], S, lt + q * TPL, twa);
    else
      phase_a<M1, M2, true, TS>(keepa[q], S, lt + q * TPL, tw);
  }
  }  // RS
  if constexpr (RS && !kTailCtaSync)
    __syncwarp();
  else
    __syncthreads();
  // ---------------- inverse phase B + store (y_2k = Re z'_k / M, y_2k+1 = Im z'_k / M)
  // With a compile-time layout (BCM != 0) the axpy epilogue's W values are
  // loaded before the row's shared-memory loads and inverse DFT, so their L2
  // latency hides behind that arithmetic (the small-grid kernels are latency-bound).
  bool bad = false;
  const bool rows = BCM == 1 || (BCM == 0 && Bc == 1);
  constexpr bool PRE = AXPY && BCM != 0;
#pragma unroll
  for (int q = 0; q < M1 / TPL; ++q) {
    const int k1 = lt + q * TPL;
    double2 wpre[PRE ? M2 : 1];
    if constexpr (EARLY) {
#pragma unroll
      for (int k2 = 0; k2 < M2; ++k2) wpre[k2] = wearly[k2];
    } else if constexpr (PRE) {
#pragma unroll
      for (int k2 = 0; k2 < M2; ++k2) {
        const int k = k1 + M1 * k2;
        if (rows) {
          wpre[k2] = __ldg(reinterpret_cast<const double2*>(p.Wprev + base + 2LL * k));
        } else {
          const long long o0 = base + (2LL * k) * es;
          wpre[k2] = make_double2(__ldg(p.Wprev + o0), __ldg(p.Wprev + o0 + es));
        }
      }
    }
#pragma unroll
    for (int n2 = 0; n2 < M2; ++n2) r[n2] = S[k1 * (M2 + 1) + n2];
    dft_any<M2, true>(r);
#pragma unroll
    for (int k2 = 0; k2 < M2; ++k2) {
      const int k = k1 + M1 * k2;
      double y0 = r[k2].x, y1 = r[k2].y;  // 1/M is folded into phis
      if (rows) {
        const long long o = base + 2LL * k;
        if (AXPY) {
          const double2 wv = PRE ? wpre[PRE ? k2 : 0] : __ldg(reinterpret_cast<const double2*>(p.Wprev + o));
          y0 = __dadd_rn(wv.x, __dmul_rn(p.tau, y0));
          y1 = __dadd_rn(wv.y, __dmul_rn(p.tau, y1));
          bad |= !(fabs(y0) <= p.limit) || !(fabs(y1) <= p.limit);
        }
        if constexpr (CLS) {
          constexpr int N = 2 * M, N1 = M, R = 4;
          const int line = (int)(base / N);
          const int c = line / R, rho = (int)cluster_ctarank() * R + (line - c * R);
          const uint32_t dst = mapa_shared(p.cl_slab + (uint32_t)(((c * N1 + rho) * 8 + ((2 * k) & 7)) * 8),
                                           (uint32_t)(k >> 2));
          const uint32_t bar = mapa_shared(p.cl_bar, (uint32_t)(k >> 2));
          asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(dst),
                       "d"(y0), "d"(y1), "r"(bar)
                       : "memory");
        } else {
          *reinterpret_cast<double2*>(p.Y + o) = make_double2(y0, y1);
        }
      } else {
        const long long o0 = base + (2LL * k) * es, o1 = o0 + es;
        if (AXPY) {
          const double w0 = PRE ? wpre[PRE ? k2 : 0].x : __ldg(p.Wprev + o0);
          const double w1 = PRE ? wpre[PRE ? k2 : 0].y : __ldg(p.Wprev + o1);
          y0 = __dadd_rn(w0, __dmul_rn(p.tau, y0));
          y1 = __dadd_rn(w1, __dmul_rn(p.tau, y1));
          bad |= !(fabs(y0) <= p.limit) || !(fabs(y1) <= p.limit);
        }
        p.Y[o0] = y0;
        p.Y[o1] = y1;
      }
    }
  }
  if (AXPY) {
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicMin(p.first_bad + f, *p.step);
  }
}

// ROWS: lines are contiguous rows (Bc == 1), a compile-time split so the
// column kernels (Bc > 1) keep their own register allocation
// STG (column kernels): the N twiddles and the CTA's scaled Phi rows are plan
// constants, copied to shared memory by cp.async before the wait on the
// previous kernel, so the split / merge and both phase A passes read them at
// shared-memory latency instead of L2 latency in the middle of the dependent
// chain (ncu: long_scoreboard was 7.5 of 12 stall cycles per issue in the
// ball's kernel).  A CTA's lines have consecutive Phi classes (one class for
// phi_class_a == 1), so its rows are one contiguous block.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// Measured (profiles/r02_theta_staging.txt): sphere 6.28 -> 5.14 us, cylinder
// 10.85 -> 9.98 us; the ball's 100-point kernel (a Phi row per line, 9 KB per
// CTA) 12.2 -> 13.2 us, so the 5 x 10 kernels keep reading through L1.
template <int M1, int M2, bool AXPY, int NT = 256, bool ROWS = false, bool STG = !ROWS && (M1 != 5)>
__global__ void __launch_bounds__(NT) theta_fast_kernel(const ThetaParams p) {
  using F = FastTheta<M1, M2, NT>;
  constexpr int M = F::M, TPL = F::TPL, LPB = F::LPB;
  extern __shared__ double2 tf_smem[];
  const int N = 2 * M;
  // the dispatcher picks ROWS = (Bc == 1); the layout is compile-time for row
  // kernels and axpy column kernels (measured faster), run-time otherwise
  constexpr int MODE = ROWS ? 1 : (AXPY ? 2 : 0);
  const int Bc = ROWS ? 1 : p.Bc;
  const bool rows = MODE == 1 || (MODE == 0 && Bc == 1);
  const int tid = threadIdx.x;
  int ln, lt;  // line within CTA, thread within line
  if (rows) {
    ln = tid / TPL;
    lt = tid - ln * TPL;
  } else {
    ln = tid % LPB;
    lt = tid / LPB;
  }
  // CTA -> (field, a0, bc0) with W = LPB lines
  const int blk = blockIdx.x;
  int f, a0, bc0;
  if (rows) {
    const int per = p.A / LPB;
    f = blk / per;
    a0 = (blk - f * per) * LPB;
    bc0 = 0;
  } else {
    const int per = Bc / LPB;
    const int pa = blk / per;
    bc0 = (blk - pa * per) * LPB;
    f = pa / p.A;
    a0 = pa - f * p.A;
  }
  const int c = f % p.ncomp;
  const int la = rows ? a0 + ln : a0, lbc = rows ? 0 : bc0 + ln;
  const int cls = p.phi_class_a == 1 ? la : (p.phi_class_a == 0 ? lbc : la * Bc + lbc);
  const double* ph = p.phis + ((long long)c * p.nclass + cls) * p.phis_ld;
  const double2* tw = p.tw;
  if constexpr (STG) {
    double2* tw_s = tf_smem + LPB * F::SL;
    double* ph_s = reinterpret_cast<double*>(tw_s + N);
    const bool one = rows || p.phi_class_a == 1;  // every line of the CTA in one class (rows: never staged)
    const int cls0 = p.phi_class_a == 1 ? a0 : (p.phi_class_a == 0 ? bc0 : a0 * Bc + bc0);
    const double* src = p.phis + ((long long)c * p.nclass + cls0) * F::PS;  // PS == p.phis_ld (checked at plan set-up)
    const int chunks = (one ? 1 : LPB) * (F::PS / 2);
    for (int i = tid; i < N; i += NT) cp_async16(tw_s + i, p.tw + i);
    asm volatile("cp.async.commit_group;\n" ::: "memory");  // group 1: twiddles (needed by phase A)
    for (int i = tid; i < chunks; i += NT) cp_async16(ph_s + 2 * i, src + 2 * i);
    ph = ph_s + (one ? 0 : ln * F::PS);  // (unconditionally a shared-space pointer: a run-time choice
                                         // between the staged and the global row made every Phi load generic)
    asm volatile("cp.async.commit_group;\n" ::: "memory");  // group 2: Phi rows (needed by the split)
    tw = tw_s;
  }
  pdl_wait();
  const long long lstride = (long long)N * Bc;
  const long long base = (long long)f * p.npts + (long long)la * lstride + lbc;  // element t at base + t*es
  const long long es = Bc;
  double2* S = tf_smem + ln * F::SL;

  // forward phase A: columns n2 = lt, lt + TPL, ...; z_k = x_2k + i x_2k+1
  double2 keepa[M2 / TPL][M1];
#pragma unroll
  for (int q = 0; q < M2 / TPL; ++q) {
    const int n2 = lt + q * TPL;
#pragma unroll
    for (int n1 = 0; n1 < M1; ++n1) {
      const int k = n2 + M2 * n1;
      if (rows)
        keepa[q][n1] = __ldg(reinterpret_cast<const double2*>(p.X + base) + k);
      else
        keepa[q][n1] = make_double2(__ldg(p.X + base + (2LL * k) * es), __ldg(p.X + base + (2LL * k + 1) * es));
    }
  }
  if constexpr (STG) {
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    __syncthreads();  // the staged twiddles are visible to every thread
  }
#pragma unroll
  for (int q = 0; q < M2 / TPL; ++q) phase_a<M1, M2, false, STG>(keepa[q], S, lt + q * TPL, tw);
  // the Phi rows had phase A to land; theta_tail's first barrier publishes them
  if constexpr (STG) asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  // contiguous lines (Bc == 1) keep a line's threads in consecutive lanes: register split
  constexpr bool RS = ROWS && (TPL == M1) && ((TPL & (TPL - 1)) == 0) && TPL <= 32;
  theta_tail<M1, M2, AXPY, STG, RS, MODE, false, false>(p, S, lt, ph, tw, f, base, es, Bc);
}

}  // namespace cg
