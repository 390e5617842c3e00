// rbns_newton_spec.cuh — K3 (default): register Gauss–Jordan with SPECULATIVE partial pivoting, verified.
//
// Newton iterations on one sample change J only a little, and the partial-pivoting row order rarely moves:
// on the BASELINE configs and the paper-form models the order is the identity at the first iteration and
// unchanged afterwards for every sample measured (tools/pivot_stability.py).  So the kernel takes the pivot
// order as a hint — the order chosen at this sample's previous Newton iteration, the identity at the first —
// and takes the search off the critical path:
//
//     barrier (+ OR-reduction of the verification flags)   column k and pivot row p_k = hint[k] are in
//                                                          shared memory (double-buffered by step parity)
//     update   every thread loads its multipliers l = column·(1/a_pk) and the pivot-row entries, and the
//              rank-1 DFMA update runs; the owners of column k+1 store it as soon as they updated it, the
//              owners of row p_{k+1} publish it at the end of the update.
//     verify   while loading its column entries each thread checks that none of its unpivoted rows beats
//              the hint under the partial-pivoting rule (|a_ik| > |a_pk|, or equal with i < p: LAPACK idamax's
//              tie rule) — a local predicate, folded into the next step's barrier (bar.red.or).
//
// One barrier and no reductions per column.  If any step's verification fails, the whole CTA abandons the
// speculative pass at that barrier and appends the sample to a miss list; the exact full-search kernel
// (rbns_newton2.cuh) then runs on the listed samples from the untouched J (same stream, launched right after,
// grid sized to the chunk, CTAs beyond the device-side count exit at once).  Results are therefore those of
// partial pivoting in every case, with identical arithmetic to gj2 whenever the hint was right.  The chosen
// order is written back as the next iteration's hint.
//
// Reference: SPEC.md:558 (LU with partial pivoting), SPEC.md:520-523 / :557-559 (Newton step and stop rule).
#pragma once

#include "rbns_common.cuh"
#include "rbns_newton.cuh"
#include "rbns_newton2.cuh"

namespace rbns {

template <int TGR, int TGC, int RS, int CS>
struct GJSShared : GJ2Shared<TGR, TGC, RS, CS> {
  static constexpr int NR = TGR * RS;
  double SP[2][CS][TGC];  // speculative pivot rows, double-buffered by step parity
  double spv[2], srp[2];  // pivot value and its reciprocal, from the thread holding a[p][k]
  int16_t hint[NR];
};

// Next pivot row, updated ahead of the bulk update and published: SP[s·TGC] = a[rp][s] − l1·pj[s] for
// s in [SB0, CS) (the same FMA the bulk update performs on that row: identical values), by the threads of the
// pivot's thread-row.  rp is CTA-uniform: the branches of the tree never diverge.  vk1 receives the entry in
// slot S1 (the next pivot value when the caller holds that column).
template <int RS, int CS, int SB0, int TGC, int LO = 0, int HI = RS>
__device__ __forceinline__ void gjs_publish_row(const double (&a)[RS][CS], int rp, double l1, const double (&pj)[CS],
                                                int s1, double* SP, double& vk1) {
  if constexpr (HI - LO == 1) {
#pragma unroll
    for (int s = SB0; s < CS; ++s) {
      const double v = fma(-l1, pj[s], a[LO][s]);
      SP[s * TGC] = v;
      if (s == s1) vk1 = v;
    }
  } else {
    constexpr int MID = (LO + HI) / 2;
    if (rp < MID)
      gjs_publish_row<RS, CS, SB0, TGC, LO, MID>(a, rp, l1, pj, s1, SP, vk1);
    else
      gjs_publish_row<RS, CS, SB0, TGC, MID, HI>(a, rp, l1, pj, s1, SP, vk1);
  }
}

__device__ __forceinline__ double gjs_rcp(double v) {
  return fabs(v) >= 2.2250738585072014e-308 ? rcp_nr(v) : 1.0 / v;
}

template <int TGR, int TGC, int RS, int CS, int SB>
__device__ __forceinline__ bool gjs_block(double (&a)[RS][CS], unsigned& pmask, bool& bad, const int N,
                                          const int tr, const int tc, GJSShared<TGR, TGC, RS, CS>& sh) {
  static_assert((TGR & (TGR - 1)) == 0, "TGR must be a power of two");
  constexpr int LG = TGR == 4 ? 2 : TGR == 8 ? 3 : TGR == 16 ? 4 : 5;
  if constexpr (SB < CS) {
#pragma unroll 1
    for (int kk = 0; kk < TGC; ++kk) {
      const int k = SB * TGC + kk;
      if (k >= N) return true;
      const int buf = k & 1;
      if (__syncthreads_or(bad)) return false;  // step barrier + verification of step k−1
      const unsigned p = static_cast<uint16_t>(sh.hint[k]);
      const double piv = sh.spv[buf], rpiv = sh.srp[buf];
      double pj[CS];
#pragma unroll
      for (int s = SB; s < CS; ++s) pj[s] = sh.SP[buf][s][tc];
      double l[RS];
#pragma unroll
      for (int r = 0; r < RS; ++r) l[r] = sh.col[buf][tr + TGR * r] * rpiv;  // row p stored as 0: l_p = 0
      const bool more = k + 1 < N;
      const unsigned p1 = more ? static_cast<uint16_t>(sh.hint[k + 1]) : 0u;
      const int kn = kk + 1;  // next column's thread-column (== TGC: slot SB+1 of thread-column 0)
      if (more && tr == int(p1 & (TGR - 1))) {
        const double l1 = sh.col[buf][p1] * rpiv;
        double vk1 = 0.0;
        gjs_publish_row<RS, CS, SB, TGC>(a, int(p1 >> LG), l1, pj, kn < TGC ? SB : SB + 1, &sh.SP[buf ^ 1][0][tc],
                                         vk1);
        if (tc == (kn < TGC ? kn : 0)) {
          sh.spv[buf ^ 1] = vk1;
          sh.srp[buf ^ 1] = gjs_rcp(vk1);
        }
      }
      // verification, one row slot per thread-column: no unpivoted row may beat the hint (idamax rule)
      const double apiv = fabs(piv);
#pragma unroll
      for (int r = tc; r < RS; r += TGC) {
        const int row = tr + TGR * r;
        const double ax = fabs(sh.col[buf][row]);
        const bool live = !((pmask >> r) & 1u);  // row p is stored as 0 and pivoted rows are masked
        bad |= live && (ax > apiv || (ax == apiv && row < int(p)));
      }
      if (!(apiv > 0.0) || !isfinite(piv)) bad = true;  // zero / non-finite pivot: the exact path decides
      if (tr == int(p & (TGR - 1))) pmask |= 1u << (p >> LG);
      if (threadIdx.x == 0) {
        sh.perm[k] = int(p);
        sh.piv[k] = piv;
      }
      // update; column k+1 first (its owners store it, with the next pivot's entry as 0)
#pragma unroll
      for (int r = 0; r < RS; ++r) a[r][SB] = fma(-l[r], pj[SB], a[r][SB]);
      if (kn < TGC && tc == kn) {
#pragma unroll
        for (int r = 0; r < RS; ++r) sh.col[buf ^ 1][tr + TGR * r] = a[r][SB];
        if (tr == int(p1 & (TGR - 1))) sh.col[buf ^ 1][p1] = 0.0;
      }
      if constexpr (SB + 1 < CS) {
#pragma unroll
        for (int r = 0; r < RS; ++r) a[r][SB + 1] = fma(-l[r], pj[SB + 1], a[r][SB + 1]);
        if (kn == TGC && tc == 0) {
#pragma unroll
          for (int r = 0; r < RS; ++r) sh.col[buf ^ 1][tr + TGR * r] = a[r][SB + 1];
          if (tr == int(p1 & (TGR - 1))) sh.col[buf ^ 1][p1] = 0.0;
        }
      }
#pragma unroll
      for (int s = SB + 2; s < CS; ++s)
#pragma unroll
        for (int r = 0; r < RS; ++r) a[r][s] = fma(-l[r], pj[s], a[r][s]);
    }
    return gjs_block<TGR, TGC, RS, CS, SB + 1>(a, pmask, bad, N, tr, tc, sh);
  } else {
    return true;
  }
}

template <int TGR, int TGC, int RS, int CS, int MINB = (TGR * TGC <= 128 ? 2 : 1)>
__global__ void __launch_bounds__(TGR * TGC, MINB) newton_gjs_kernel(const NewtonParams p) {
  using SH = GJSShared<TGR, TGC, RS, CS>;
  static_assert(RS <= 32 && TGR <= 32 && TGC <= 32 && (TGR * TGC) % 32 == 0, "shape");
  constexpr int NT = TGR * TGC, NR = TGR * RS;
  __shared__ SH sh;
  const int i_s = blockIdx.x;
  if (i_s >= p.n) return;
  const int b = p.act[i_s];
    RBNS_CHECK(i_s >= 0 && i_s < p.n && b >= 0 && (p.B == 0 || b < p.B));
  const int tid = threadIdx.x, tc = tid / TGR, tr = tid % TGR;
  const int N = p.N;
  for (int i = tid; i < NR; i += NT) {
    sh.hint[i] = int16_t((p.hint_in && i < N) ? p.hint_in[int64_t(b) * N + i] : i);
    sh.col[0][i] = sh.col[1][i] = 0.0;
  }
  double a[RS][CS];
  gj_load_system<TGR, TGC, RS, CS>(p, i_s, b, a, sh);
  {  // column 0 (pivot entry stored as 0) and pivot row hint[0]
    const int p0 = sh.hint[0];
    if (tc == 0) {
#pragma unroll
      for (int r = 0; r < RS; ++r) sh.col[0][tr + TGR * r] = a[r][0];
      if (tr == p0 % TGR) sh.col[0][p0] = 0.0;
    }
    if (tr == p0 % TGR) {
      double pj0[CS], v0 = 0.0;
#pragma unroll
      for (int s = 0; s < CS; ++s) pj0[s] = 0.0;
      gjs_publish_row<RS, CS, 0, TGC>(a, p0 / TGR, 0.0, pj0, 0, &sh.SP[0][0][tc], v0);
      if (tc == 0) {
        sh.spv[0] = v0;
        sh.srp[0] = gjs_rcp(v0);
      }
    }
  }
  unsigned pmask = 0;
  bool bad = false;
  bool ok = gjs_block<TGR, TGC, RS, CS, 0>(a, pmask, bad, N, tr, tc, sh);
  if (ok) ok = !__syncthreads_or(bad);  // the last step's verification
  if (!ok) {  // wrong hint somewhere: hand the sample to the exact full-search kernel (launched after this one)
    if (tid == 0) {
      p.miss_list[atomicAdd(p.miss_count, 1)] = i_s;
      if (p.spec_miss) atomicAdd(p.spec_miss, 1);
    }
    return;
  }
  gj_finish<TGR, TGC, RS, CS>(p, b, a, false, sh);
  if (p.hint_out) {
    for (int i = tid; i < N; i += NT) p.hint_out[int64_t(b) * N + i] = int16_t(sh.perm[i]);
  }
}

}  // namespace rbns
