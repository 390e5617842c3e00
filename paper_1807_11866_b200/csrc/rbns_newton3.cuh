// rbns_newton3.cuh — K3: register Gauss–Jordan with ONE CTA barrier per elimination step.
//
// Data distribution, prologue and epilogue as rbns_newton2.cuh (one CTA per μ sample, [J | −R] in registers,
// 2-D cyclic over a TGR×TGC thread grid, thread (tr, tc) owns rows tr + TGR·r and columns tc + TGC·s; column
// blocks left of the current one skipped statically).  Column-major thread numbering makes every warp hold
// complete thread-columns, so the part of the pivot row a warp needs lives inside that warp.  A step is
//
//     barrier   column k is in shared memory (its owners stored it inside the previous update)
//     search    EVERY warp reduces the whole column itself: lane ℓ takes rows RPL·ℓ … RPL·ℓ+RPL−1 (vector
//               loads), masks its pivoted rows with a per-lane bit mask (identical in all warps, no shared
//               flags), argmax by redux.sync on the (high, low) words; contiguous row blocks make the lowest
//               candidate lane the smallest row (LAPACK idamax tie rule)
//     row       the pivot row slot rp is CTA-uniform: a uniform branch tree selects a[rp][·] and a warp
//               shuffle from lane (tc mod 32/TGR)·TGR + tp hands each thread its pivot-row entries
//     update    l = column · (1/pivot) (pivot row's own multiplier zeroed by a second uniform tree), DFMA
//               rank-1 update; the owners of column k+1 update it first and store it for the next search
//
// — no candidate exchange and no pivot-row publication through shared memory, hence one barrier instead of
// gj2's three.  Partial pivoting semantics are unchanged.
//
// Reference: SPEC.md:558 (LU with partial pivoting), SPEC.md:520-523 / :557-559 (Newton step and stop rule).
#pragma once

#include "rbns_common.cuh"
#include "rbns_newton.cuh"
#include "rbns_newton2.cuh"

namespace rbns {

template <int TGR, int TGC, int RS, int CS>
struct GJ3Shared {
  static constexpr int NT = TGR * TGC;
  static constexpr int NW = (NT + 31) / 32;
  static constexpr int NR = TGR * RS;
  static constexpr int RPL = ((NR + 31) / 32 + 1) / 2 * 2;  // rows per search lane (even: double2 loads)
  NewtonWeights w;
  alignas(16) double col[2][32 * RPL];  // column k (row-indexed, zero-padded), double-buffered by step parity
  signed char pivoted[NR];              // unused by the kernel body (gj_load_system clears it)
  double piv[NR];
  int perm[NR];
  double rhs[NR];
  double rowred[NW][NR];
  double red[2][NW];
};

// out[s] = a[rp][s] for s in [SB, CS); rp is CTA-uniform, so the branches never diverge
template <int RS, int CS, int SB, int LO = 0, int HI = RS>
__device__ __forceinline__ void gj3_select_row(const double (&a)[RS][CS], int rp, double (&out)[CS]) {
  if constexpr (HI - LO == 1) {
#pragma unroll
    for (int s = SB; s < CS; ++s) out[s] = a[LO][s];
  } else {
    constexpr int MID = (LO + HI) / 2;
    if (rp < MID)
      gj3_select_row<RS, CS, SB, LO, MID>(a, rp, out);
    else
      gj3_select_row<RS, CS, SB, MID, HI>(a, rp, out);
  }
}

// l[rp] = 0 when `mine` (the pivot row keeps its values); uniform tree on rp
template <int RS, int LO = 0, int HI = RS>
__device__ __forceinline__ void gj3_zero_slot(double (&l)[RS], int rp, bool mine) {
  if constexpr (HI - LO == 1) {
    if (mine) l[LO] = 0.0;
  } else {
    constexpr int MID = (LO + HI) / 2;
    if (rp < MID)
      gj3_zero_slot<RS, LO, MID>(l, rp, mine);
    else
      gj3_zero_slot<RS, MID, HI>(l, rp, mine);
  }
}

template <int TGR, int TGC, int RS, int CS, int SB>
__device__ __forceinline__ void gj3_block(double (&a)[RS][CS], unsigned& pmask, bool& sing, const int N,
                                          const int tr, const int tc, GJ3Shared<TGR, TGC, RS, CS>& sh) {
  using SH = GJ3Shared<TGR, TGC, RS, CS>;
  constexpr int RPL = SH::RPL;
  constexpr int TPW = 32 / TGR;  // thread-columns per warp
  if constexpr (SB < CS) {
    if (sing) return;
    const int lane = threadIdx.x & 31;
    const int src_base = (tc % TPW) * TGR;
#pragma unroll 1
    for (int kk = 0; kk < TGC; ++kk) {
      const int k = SB * TGC + kk;
      if (k >= N) return;
      const int buf = k & 1;
      __syncthreads();  // column k stored; the previous update complete everywhere
      // ---- search (redundant per warp) ----
      double v[RPL];
#pragma unroll
      for (int i = 0; i < RPL; i += 2) {
        const double2 t = *reinterpret_cast<const double2*>(&sh.col[buf][RPL * lane + i]);
        v[i] = t.x;
        v[i + 1] = t.y;
      }
      unsigned bhi = 0, blo = 0;
      int bi = 0;
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const bool live = !((pmask >> i) & 1u);
        const unsigned hi = live ? (unsigned(__double2hiint(v[i])) & 0x7fffffffu) : 0u;
        const unsigned lo = live ? unsigned(__double2loint(v[i])) : 0u;
        const bool gt = hi > bhi || (hi == bhi && lo > blo);
        bhi = gt ? hi : bhi;
        blo = gt ? lo : blo;
        bi = gt ? i : bi;
      }
      const unsigned mhi = __reduce_max_sync(0xffffffffu, bhi);
      const bool eqhi = bhi == mhi;
      const unsigned mlo = __reduce_max_sync(0xffffffffu, eqhi ? blo : 0u);
      const unsigned cnd = __ballot_sync(0xffffffffu, eqhi && blo == mlo);
      const int src = __ffs(cnd) - 1;
      const int p = RPL * src + __shfl_sync(0xffffffffu, bi, src);
      if ((mhi | mlo) == 0u || (mhi & 0x7ff00000u) == 0x7ff00000u) {  // zero or non-finite: CTA-uniform
        sing = true;
        return;
      }
      double vb = v[0];
#pragma unroll
      for (int i = 1; i < RPL; ++i) vb = bi == i ? v[i] : vb;
      const double piv = __shfl_sync(0xffffffffu, vb, src);
      if (lane == src) pmask |= 1u << bi;
      if (threadIdx.x == 0) {
        sh.perm[k] = p;
        sh.piv[k] = piv;
      }
      // ---- pivot row through the warp ----
      const int tp = p % TGR, rp = p / TGR;
      double pr[CS];
      gj3_select_row<RS, CS, SB>(a, rp, pr);
      double pj[CS];
#pragma unroll
      for (int s = SB; s < CS; ++s) pj[s] = __shfl_sync(0xffffffffu, pr[s], src_base + tp);
      // ---- multipliers ----
      const double rpiv = fabs(piv) >= 2.2250738585072014e-308 ? rcp_nr(piv) : 1.0 / piv;
      double l[RS];
#pragma unroll
      for (int r = 0; r < RS; ++r) l[r] = sh.col[buf][tr + TGR * r] * rpiv;
      gj3_zero_slot<RS>(l, rp, tr == tp);
      // ---- update; column k+1 first, stored for the next search ----
#pragma unroll
      for (int r = 0; r < RS; ++r) a[r][SB] = fma(-l[r], pj[SB], a[r][SB]);
      if (kk + 1 < TGC && tc == kk + 1) {
#pragma unroll
        for (int r = 0; r < RS; ++r) sh.col[buf ^ 1][tr + TGR * r] = a[r][SB];
      }
      if constexpr (SB + 1 < CS) {
#pragma unroll
        for (int r = 0; r < RS; ++r) a[r][SB + 1] = fma(-l[r], pj[SB + 1], a[r][SB + 1]);
        if (kk + 1 == TGC && tc == 0) {
#pragma unroll
          for (int r = 0; r < RS; ++r) sh.col[buf ^ 1][tr + TGR * r] = a[r][SB + 1];
        }
      }
#pragma unroll
      for (int s = SB + 2; s < CS; ++s)
#pragma unroll
        for (int r = 0; r < RS; ++r) a[r][s] = fma(-l[r], pj[s], a[r][s]);
    }
    gj3_block<TGR, TGC, RS, CS, SB + 1>(a, pmask, sing, N, tr, tc, sh);
  }
}

template <int TGR, int TGC, int RS, int CS>
__global__ void __launch_bounds__(TGR * TGC, (TGR * TGC <= 128 ? 2 : 1)) newton_gj3_kernel(const NewtonParams p) {
  using SH = GJ3Shared<TGR, TGC, RS, CS>;
  static_assert(RS <= 32 && TGR <= 32 && TGC <= 32 && (TGR * TGC) % 32 == 0, "shape");
  static_assert(SH::RPL <= 32, "search lanes");
  __shared__ SH sh;
  const int i_s = blockIdx.x;
  if (i_s >= p.n) return;
  const int b = p.act[i_s];
  const int tid = threadIdx.x, tc = tid / TGR, tr = tid % TGR;
  double a[RS][CS];
  for (int i = tid; i < 2 * 32 * SH::RPL; i += TGR * TGC) (&sh.col[0][0])[i] = 0.0;  // padding rows stay 0
  gj_load_system<TGR, TGC, RS, CS>(p, i_s, b, a, sh);
  if (tc == 0) {  // column 0
#pragma unroll
    for (int r = 0; r < RS; ++r) sh.col[0][tr + TGR * r] = a[r][0];
  }
  // search lanes: rows ≥ N never win (masked as pivoted)
  const int lane = tid & 31;
  unsigned pmask = 0;
#pragma unroll
  for (int i = 0; i < SH::RPL; ++i)
    if (SH::RPL * lane + i >= p.N) pmask |= 1u << i;
  bool sing = false;
  gj3_block<TGR, TGC, RS, CS, 0>(a, pmask, sing, p.N, tr, tc, sh);
  gj_finish<TGR, TGC, RS, CS>(p, b, a, sing, sh);
}

}  // namespace rbns
