// Resident-operator mode products: Y = X L^T (TN, last mode) or Y = L X (NN,
// first / middle mode) for operators of at most 128 x 128 (mode_product,
// tensor.py:31-49, through the steppers integrators.py:202-236).
//
// The tiled kernel (gemm.cuh) streams both operands through a TMA ring; for
// the 3-D configs (n = 64 .. 128) the operator is a few tens of KB that every
// tile reloads, tiles quantise badly (n = 100: 626 tiles of 32 rows on 296
// CTAs) and each tile pays ring fill, barriers and an epilogue hand-off.
// Here the operator (both operators of the ball's chained polar pair) is
// copied into shared memory ONCE per CTA by a bulk copy issued before
// griddepcontrol.wait, and warps work on 8-wide strips of the free dimension
// -- 8 rows of X (TN) or 8 columns (NN):
//   - a strip's fragments of X go straight from global memory into registers
//     (the mma.m8n8k4 fragment of X is one double per lane: 8 rows x 32 B (TN)
//     or 4 rows x 64 B (NN) per load, whole sectors);
//   - the operator fragment is an 8-byte shared-memory load per DMMA from a
//     row-major [n][LDS] copy with LDS = 4 (mod 16): conflict-free;
//   - a strip is split into NH = 2 parts over the operator extent (the 8x8
//     blocks of the output columns (TN) / rows (NN)), one warp each: half the
//     accumulators per warp, so 16 warps fit one SM (4 per sub-partition) and
//     the work unit is half a strip -- n = 100: 5000 units over 592
//     sub-partitions instead of 626 tiles over 296 CTAs;
//   - the epilogue (Phi, W + tau*Y + guard, store) runs from the C fragments
//     (adjacent column pairs: 16-byte stores);
//   - the chained pair (ball polar mode: (F x3 V^-1 o Phi) x3 V) exchanges the
//     Phi-scaled intermediate of a strip between its two warps through an
//     8-row shared-memory tile (two 64-thread named barriers per strip) and
//     reads it back as the second product's A fragments: the intermediate
//     never goes to HBM.
// One DMMA issues per 16 clocks per SM sub-partition and a dependent DMMA
// after 26 (tools/dmma_latency.cu), so a few warps per sub-partition keep the
// pipe full while others wait for their X loads or run an epilogue.  No ring
// or tensor map in the steady state.  Every output accumulates over k in
// sequential 4-blocks: for last-mode (TN) products that is the tiled kernel's
// order, so the chained pair is bitwise equal to it (tests/test_gpu_resident.py);
// the tiled first-mode (NN) fragments group k as {8q + 2t + s}, so NN stages
// agree to rounding.
#pragma once

#include "gemm.cuh"

namespace cg {

struct ResParams {
  int M, N, K;     // TN: M rows of X, N = K = operator extent; NN: M = K = operator extent, N columns
  int nslab, ncomp;
  int nitems;      // nfield * nslab
  int upi;         // 8-wide strips per item
  int ldr;         // row stride of X, out and w
  long long fstride, sstride;  // field / slab strides (elements)
  const double* X;
  double* out;
  const double* w;    // EPI_AXPY: previous state (indexed like out)
  const double* op;   // [ncomp][8 NB][LDS] row-major L, zero padded
  const double* op2;  // EPI_CHAIN: second operator, same layout
  const double* phi;  // EPI_PHI / EPI_CHAIN: phi + c*phi_c + s*phi_s + (m/phi_rdiv)*phi_m + n*phi_n
  long long phi_c, phi_s;
  int phi_m, phi_n, phi_rdiv;
  double tau, limit;
  int* first_bad;
  const int* step;
};

constexpr int kResWarps = 16;  // one CTA per SM, four warps per sub-partition
constexpr int kResParts = 2;   // warps per strip
constexpr int kResGroups = kResWarps / kResParts;
constexpr int kResTailMax = 2;  // last rounds of at most this many strips run one block per warp

// shared-memory row stride of the operator copy: >= 4 KSTEPS and 4 (mod 16)
__host__ __device__ constexpr int res_lds(int ksteps) {
  int l = 4 * ksteps;
  while (l % 16 != 4) ++l;
  return l;
}
template <int EPI, int NB, int KSTEPS>
constexpr size_t res_smem_bytes() {
  const size_t ops = (size_t)(EPI == EPI_CHAIN ? 2 : 1) * NB * 8 * res_lds(KSTEPS) * sizeof(double);
  const size_t xch = EPI == EPI_CHAIN ? (size_t)kResGroups * 8 * res_lds(KSTEPS) * sizeof(double) : 0;
  return ops + xch + 128 + 16;
}

// acc[j] += x (x) operator blocks j0 + j, j < NL (NL compile-time: no dead DMMAs)
template <int VAR, int NL, int NBH, int KSTEPS>
__device__ __forceinline__ void res_product(const double* o, int j0, int g, int t, const double (&x)[KSTEPS],
                                            double (&acc)[NBH][2]) {
  constexpr int LDS = res_lds(KSTEPS);
  const double* frag = o + (j0 * 8 + g) * LDS + t;
#pragma unroll
  for (int ks = 0; ks < KSTEPS; ++ks) {
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      const double l = frag[j * 8 * LDS + 4 * ks];
      if (VAR == VAR_TN)
        dmma_8x8x4(acc[j][0], acc[j][1], x[ks], l);  // A = X rows, B[k][n] = L[n][k]
      else
        dmma_8x8x4(acc[j][0], acc[j][1], l, x[ks]);  // A = L rows, B = X columns
    }
  }
}

// One strip part: blocks [j0, j0 + NL) of the operator extent for strip
// `strip` of (field f, slab s).  ops / ops2: the resident operator copies (ops2:
// the chain's second operator); tile_base: the strip's exchange tile and
// (bar_id, bar_threads) the named barrier of the warps sharing it (CHAIN).
template <int VAR, int EPI, int NL, int NBH, int KSTEPS>
__device__ __forceinline__ void res_strip_part(const ResParams& p, const double* ops, const double* ops2,
                                               double* tile_base, int bar_id, int bar_threads, int j0, int f, int s,
                                               int strip, int lane, int step_now, uint64_t* op2_bar = nullptr,
                                               uint32_t op2_phase = 0) {
  constexpr int LDS = res_lds(KSTEPS);
  const int g = lane >> 2, t = lane & 3;
  const int c = f % p.ncomp;
  double acc[NBH][2];
#pragma unroll
  for (int j = 0; j < NBH; ++j) acc[j][0] = acc[j][1] = 0.0;
  const long long obase = (long long)f * p.fstride + (long long)s * p.sstride;
  {
    // X fragments of the strip: TN x[ks] = X[row0 + g][4 ks + t]; NN x[ks] = X[4 ks + t][col0 + g]
    double x[KSTEPS];
    const int idx = strip * 8 + g;
    const double* src = p.X + obase;
    if (VAR == VAR_TN) {
      const bool ok = idx < p.M;
      src += (long long)idx * p.ldr + t;
#pragma unroll
      for (int ks = 0; ks < KSTEPS; ++ks) x[ks] = (ok && 4 * ks + t < p.K) ? __ldg(src + 4 * ks) : 0.0;
    } else {
      const bool ok = idx < p.N;
      src += idx + (long long)t * p.ldr;
#pragma unroll
      for (int ks = 0; ks < KSTEPS; ++ks)
        x[ks] = (ok && 4 * ks + t < p.K) ? __ldg(src + (long long)(4 * ks) * p.ldr) : 0.0;
    }
    res_product<VAR, NL, NBH, KSTEPS>(ops, j0, g, t, x, acc);
  }
  if constexpr (EPI == EPI_CHAIN) {
    // T = (X L1^T) o Phi: this warp's columns go into the strip's exchange
    // tile, the partner's come back with them as the A fragments
    // a2[ks] = T[g][4 ks + t] of the second product
    const int row = strip * 8 + g;
    const int m = row < p.M ? row : 0;
    const double* phirow = p.phi + c * p.phi_c + s * p.phi_s + (long long)(m / p.phi_rdiv) * p.phi_m;
    double* tile = tile_base + g * LDS;
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      const int n = 8 * (j0 + j) + 2 * t;
      const int nlo = n < p.N ? n : 0;
      const int nhi = n + 1 < p.N ? n + 1 : nlo;
      const double v0 = acc[j][0] * __ldg(phirow + (long long)nlo * p.phi_n);
      const double v1 = acc[j][1] * __ldg(phirow + (long long)nhi * p.phi_n);
      if (n < 4 * KSTEPS) *reinterpret_cast<double2*>(tile + n) = make_double2(v0, v1);
      acc[j][0] = acc[j][1] = 0.0;
    }
    named_bar(bar_id, bar_threads);  // every part of T is written
    double a2[KSTEPS];
#pragma unroll
    for (int ks = 0; ks < KSTEPS; ++ks) a2[ks] = tile[4 * ks + t];
    named_bar(bar_id, bar_threads);  // every warp of the strip holds T: the tile may be rewritten
    if (op2_bar) mbar_wait(op2_bar, op2_phase);  // first strip after an operator load: the second operator is in
    res_product<VAR, NL, NBH, KSTEPS>(ops2, j0, g, t, a2, acc);
    if (row < p.M) {
      double* orow = p.out + obase + (long long)row * p.ldr;
#pragma unroll
      for (int j = 0; j < NL; ++j) {
        const int n = 8 * (j0 + j) + 2 * t;
        if (n < p.N) *reinterpret_cast<double2*>(orow + n) = make_double2(acc[j][0], acc[j][1]);
      }
    }
  } else if constexpr (VAR == VAR_TN) {
    const int row = strip * 8 + g;
    if (row < p.M) {
      double* orow = p.out + obase + (long long)row * p.ldr;
      const double* phirow = nullptr;
      if (EPI == EPI_PHI) phirow = p.phi + c * p.phi_c + s * p.phi_s + (long long)(row / p.phi_rdiv) * p.phi_m;
#pragma unroll
      for (int j = 0; j < NL; ++j) {
        const int n = 8 * (j0 + j) + 2 * t;
        if (n >= p.N) continue;
        double v0 = acc[j][0], v1 = acc[j][1];
        if (EPI == EPI_PHI) {
          const int nhi = n + 1 < p.N ? n + 1 : n;
          v0 *= __ldg(phirow + (long long)n * p.phi_n);
          v1 *= __ldg(phirow + (long long)nhi * p.phi_n);
        }
        *reinterpret_cast<double2*>(orow + n) = make_double2(v0, v1);
      }
    }
  } else {
    const int n = strip * 8 + 2 * t;
    bool bad = false;
    if (n < p.N) {
      const int nhi = n + 1 < p.N ? n + 1 : n;
      double2 wv[NBH];
      if (EPI == EPI_AXPY) {
#pragma unroll
        for (int i = 0; i < NL; ++i) {
          const int m = 8 * (j0 + i) + g;
          wv[i] = m < p.M ? __ldg(reinterpret_cast<const double2*>(p.w + obase + (long long)m * p.ldr + n))
                          : make_double2(0.0, 0.0);
        }
      }
#pragma unroll
      for (int i = 0; i < NL; ++i) {
        const int m = 8 * (j0 + i) + g;
        if (m >= p.M) continue;
        double v0 = acc[i][0], v1 = acc[i][1];
        if (EPI == EPI_PHI) {
          const double* phirow = p.phi + c * p.phi_c + s * p.phi_s + (long long)(m / p.phi_rdiv) * p.phi_m;
          v0 *= __ldg(phirow + (long long)n * p.phi_n);
          v1 *= __ldg(phirow + (long long)nhi * p.phi_n);
        } else if (EPI == EPI_AXPY) {
          // W + tau*T rounded as the reference rounds it (no FMA contraction)
          v0 = __dadd_rn(wv[i].x, __dmul_rn(p.tau, v0));
          v1 = __dadd_rn(wv[i].y, __dmul_rn(p.tau, v1));
          bad |= !(fabs(v0) <= p.limit) || (n + 1 < p.N && !(fabs(v1) <= p.limit));
        }
        *reinterpret_cast<double2*>(p.out + obase + (long long)m * p.ldr + n) = make_double2(v0, v1);
      }
    }
    if (EPI == EPI_AXPY) {
      if (__any_sync(0xffffffffu, bad) && lane == 0) atomicMin(p.first_bad + f, step_now);
    }
  }
}

template <int VAR, int EPI, int NB, int KSTEPS>
__global__ void __launch_bounds__(kResWarps * 32, 1) resident_gemm_kernel(const ResParams p) {
  constexpr int LDS = res_lds(KSTEPS);
  constexpr int OPE = NB * 8 * LDS;  // doubles per operator copy
  constexpr int NOPS = EPI == EPI_CHAIN ? 2 : 1;
  constexpr int NBH = (NB + kResParts - 1) / kResParts;  // blocks of part 0; part 1 takes the rest
  constexpr int NBL = NB - NBH;
  static_assert(kResParts == 2 && NBL >= 1, "two parts per strip");
  static_assert(EPI != EPI_CHAIN || VAR == VAR_TN, "chained products are last-mode products");
  static_assert(EPI != EPI_CHAIN || 8 * NB >= 4 * KSTEPS, "the intermediate must cover the second product's k range");
  extern __shared__ uint8_t rs_raw[];
  uint8_t* base = rs_raw + ((128u - (smem_u32(rs_raw) & 127u)) & 127u);
  const double* ops = reinterpret_cast<const double*>(base);
  double* xch = reinterpret_cast<double*>(base + (size_t)NOPS * OPE * sizeof(double));  // CHAIN: [groups][8][LDS]
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + (size_t)NOPS * OPE * sizeof(double) +
                                              (EPI == EPI_CHAIN ? (size_t)kResGroups * 8 * LDS * sizeof(double) : 0));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = warp / kResParts, part = warp % kResParts;
  const long long U = (long long)p.nitems * p.upi;
  const long long lo = U * blockIdx.x / gridDim.x, hi = U * (blockIdx.x + 1) / gridDim.x;
  if (lo >= hi) return;

  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);  // CHAIN: the second operator lands while the first product runs
    fence_barrier_init();
  }
  __syncthreads();
  // operators are plan constants: their copy overlaps the previous kernel's tail
  int loaded = (int)(((lo / p.upi) / p.nslab) % p.ncomp);
  bool pending = true, first = true;
  uint32_t phase = 0;
  int step_now = 0;

  long long u = lo;
  while (u < hi) {
    const int c = (int)(((u / p.upi) / p.nslab) % p.ncomp);
    // a segment: this CTA's units of one field (every field when the operator set is shared)
    long long seg_end = hi;
    if (p.ncomp > 1) {
      const long long fend = ((u / p.upi) / p.nslab + 1) * (long long)p.nslab * p.upi;
      if (fend < seg_end) seg_end = fend;
    }
    if (first || c != loaded) {
      if (!first) {
        fence_proxy_async_smem();  // every warp's operator reads before the async-proxy overwrite
        __syncthreads();
      }
      if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(bar, (uint32_t)(OPE * sizeof(double)));
        bulk_load_1d(base, p.op + (size_t)c * OPE, (uint32_t)(OPE * sizeof(double)), bar);
        if (NOPS == 2) {
          mbar_arrive_expect_tx(bar + 1, (uint32_t)(OPE * sizeof(double)));
          bulk_load_1d(base + (size_t)OPE * sizeof(double), p.op2 + (size_t)c * OPE,
                       (uint32_t)(OPE * sizeof(double)), bar + 1);
        }
      }
      loaded = c;
      pending = true;
      if (first) {
        pdl_wait();  // the previous kernel's outputs (X / W / step counter) are complete
        if (EPI == EPI_AXPY) step_now = *p.step;
        first = false;
      }
    }
    uint64_t* bar2 = nullptr;  // CHAIN: waited for between the two products of the segment's first strip
    uint32_t phase2 = 0;
    if (pending) {
      mbar_wait(bar, phase);
      if (NOPS == 2) {
        bar2 = bar + 1;
        phase2 = phase;
      }
      phase ^= 1;
      pending = false;
    }
    // Full rounds: the strip's two warps walk the same strips (the chained pair
    // meets at named barriers).  A last round of only one or two strips would
    // leave them to one or two warp pairs running alone at the dependent-DMMA
    // rate (n = 100: 17 strips per CTA, the 17th cost 4 us of the chained
    // kernel's 35): such strips are spread over the whole CTA instead, one 8x8
    // output block per warp (NB <= 16 warps share the strip's exchange tile).
    const long long count = seg_end - u;
    const int tail = (int)(count % kResGroups);
    const long long round_end = tail > 0 && tail <= kResTailMax ? seg_end - tail : seg_end;
    for (long long mine = u + grp; mine < round_end; mine += kResGroups) {
      const long long item = mine / p.upi;
      const int strip = (int)(mine - item * p.upi);
      const int f = (int)(item / p.nslab), s = (int)(item - (long long)f * p.nslab);
      if (part == 0)
        res_strip_part<VAR, EPI, NBH, NBH, KSTEPS>(p, ops, ops + OPE, xch + (size_t)grp * 8 * LDS, 1 + grp,
                                                   kResParts * 32, 0, f, s, strip, lane, step_now, bar2, phase2);
      else
        res_strip_part<VAR, EPI, NBL, NBH, KSTEPS>(p, ops, ops + OPE, xch + (size_t)grp * 8 * LDS, 1 + grp,
                                                   kResParts * 32, NBH, f, s, strip, lane, step_now, bar2, phase2);
    }
    if (round_end < seg_end) {
      // the pairs' tiles are free once every pair is through its last strip
      if (EPI == EPI_CHAIN) __syncthreads();
      for (long long mine = round_end; mine < seg_end; ++mine) {
        const long long item = mine / p.upi;
        const int strip = (int)(mine - item * p.upi);
        const int f = (int)(item / p.nslab), s = (int)(item - (long long)f * p.nslab);
        if (warp < NB)
          res_strip_part<VAR, EPI, 1, NBH, KSTEPS>(p, ops, ops + OPE, xch, 1 + kResGroups, NB * 32, warp, f, s, strip,
                                                   lane, step_now, bar2, phase2);
      }
      if (EPI == EPI_CHAIN) __syncthreads();  // before a later segment's pairs reuse tile 0
    }
    u = seg_end;
  }
}

}  // namespace cg
