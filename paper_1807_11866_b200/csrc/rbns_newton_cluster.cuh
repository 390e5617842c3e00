// rbns_newton_cluster.cuh — K3 for large N (config 3, N = 200): the register Gauss–Jordan Newton update of
// rbns_newton.cuh spread over a 2-CTA thread-block cluster (two SMs), because [J | −R] (200×201 fp64,
// 322 KB) does not fit one SM's register file.
//
// Each CTA holds ALL rows and half of the columns: global thread-column tc_g = 16·rank + tc (32 in total),
// column j lives in CTA (j mod 32)/16, thread-column j mod 16, slot j/32; rows tr + 16·r as before.
// Per column step the owner half-warp (one CTA) publishes the pivot column and the pivot choice into BOTH
// CTAs' shared memory (DSMEM stores through the cluster window), one cluster barrier makes them visible,
// each CTA's pivot-row owners publish their half of the pivot row locally, one CTA barrier, register DFMA
// update.  The cluster barrier is the price of the second SM; partial pivoting is unchanged.
//
// The kernel first runs a speculative pass with the pivot order hinted by the sample's previous Newton
// iteration (identity at the first; see rbns_newton_spec.cuh): no search, one cluster barrier per column, the
// next column and pivot-row halves published ahead of the bulk update, each row verified under the idamax rule.
// If any check fails in either CTA, both reload J and run the exact search pass above; the order used is
// written back as the next iteration's hint.
#pragma once

#include <cooperative_groups.h>

#include "rbns_common.cuh"
#include "rbns_newton.cuh"

namespace rbns {

template <int TGR, int TGC, int RS, int CS>
struct GJCShared {
  static constexpr int NW = TGR * TGC / 32;
  static constexpr int CBS = RS | 1;
  NewtonWeights w;
  double pv[2];
  int pk[2];
  double colbuf[2][TGR][CBS];
  double P[CS][TGC];
  double piv[TGR * RS];
  int perm[TGR * RS];
  double rhs[TGR * RS];
  double rowred[NW][TGR * RS];
  double xred[2][TGR * RS];  // per-rank partial J·u row sums, collected in the RHS-owner CTA
  double red[2][NW];
  // speculative pass (hinted pivot order): this CTA's half of the pivot row, pivot value and reciprocal
  double SP[2][CS][TGC];
  double spv[2], srp[2];
  int16_t hint[TGR * RS];
  int bad_any[2];            // per-rank verification flags (written into both CTAs)
};

template <int TGR, int TGC, int RS, int CS, int SB>
__device__ __forceinline__ void gjc_block(double (&a)[RS][CS], unsigned& pmask, bool& sing, const int N,
                                          const int tr, const int tc, const int rank, GJCShared<TGR, TGC, RS, CS>& sh,
                                          GJCShared<TGR, TGC, RS, CS>* peer) {
  namespace cg = cooperative_groups;
  if constexpr (SB < CS) {
    if (sing) return;
#pragma unroll 1
    for (int kk = 0; kk < 2 * TGC; ++kk) {
      const int k = SB * 2 * TGC + kk;
      if (k >= N) return;
      const int buf = k & 1;
      const int oc = kk / TGC, otc = kk % TGC;
      if (rank == oc && tc == otc) {
        // owner half-warp: publish column k to both CTAs, argmax of |a| over unpivoted rows
        long long best = -1;
        double bsig = 0.0;
        int bi = -1;
#pragma unroll
        for (int r = 0; r < RS; ++r) {
          const double v = a[r][SB];
          sh.colbuf[buf][tr][r] = v;
          peer->colbuf[buf][tr][r] = v;
          const long long key =
              (((pmask >> r) & 1u) || tr + TGR * r >= N) ? -1LL : __double_as_longlong(fabs(v));
          if (key > best) {
            best = key;
            bsig = v;
            bi = tr + TGR * r;
          }
        }
        const unsigned gmask = ((1u << TGR) - 1u) << ((otc * TGR) & 31);
#pragma unroll
        for (int o = TGR / 2; o > 0; o >>= 1) {
          const long long k2 = __shfl_xor_sync(gmask, best, o);
          const double s2 = __shfl_xor_sync(gmask, bsig, o);
          const int i2 = __shfl_xor_sync(gmask, bi, o);
          if (k2 > best || (k2 == best && k2 >= 0 && i2 < bi)) {
            best = k2;
            bsig = s2;
            bi = i2;
          }
        }
        const bool ok = best > 0 && best < 0x7ff0000000000000LL;  // nonzero, finite
        __syncwarp(gmask);
        if (ok && tr == bi % TGR) {  // the pivot row itself is not updated
          sh.colbuf[buf][tr][bi / TGR] = 0.0;
          peer->colbuf[buf][tr][bi / TGR] = 0.0;
        }
        if (tr == 0) {
          sh.pk[buf] = ok ? bi : -1;
          sh.pv[buf] = bsig;
          peer->pk[buf] = ok ? bi : -1;
          peer->pv[buf] = bsig;
          sh.perm[k] = bi;
          sh.piv[k] = bsig;
          peer->perm[k] = bi;
          peer->piv[k] = bsig;
        }
      }
      cg::this_cluster().sync();
      const int p = sh.pk[buf];
      if (p < 0) {  // uniform across the cluster
        sing = true;
        return;
      }
      const double piv = sh.pv[buf];
      const int tp = p % TGR, rp = p / TGR;
      if (tr == tp) {
        publish_row<RS, CS, SB, TGC>(a, rp, &sh.P[0][tc]);
        pmask |= 1u << rp;
      }
      __syncthreads();
      const double rpiv = 1.0 / piv;
      double pj[CS];
#pragma unroll
      for (int s = SB; s < CS; ++s) pj[s] = sh.P[s][tc];
#pragma unroll
      for (int r = 0; r < RS; ++r) {
        const double l = sh.colbuf[buf][tr][r] * rpiv;
#pragma unroll
        for (int s = SB; s < CS; ++s) a[r][s] = fma(-l, pj[s], a[r][s]);
      }
    }
    gjc_block<TGR, TGC, RS, CS, SB + 1>(a, pmask, sing, N, tr, tc, rank, sh, peer);
  }
}

// a[rp][s] (slots ≥ SB0) after a rank-1 step with multiplier l and pivot row pj, stored to P (stride TGC);
// uniform tree on rp; vsel receives slot ssel's value
template <int RS, int CS, int SB0, int TGC, int LO = 0, int HI = RS>
__device__ __forceinline__ void gjcs_publish(const double (&a)[RS][CS], int rp, double l, const double (&pj)[CS],
                                             int ssel, double* P, double& vsel) {
  if constexpr (HI - LO == 1) {
#pragma unroll
    for (int s = SB0; s < CS; ++s) {
      const double v = fma(-l, pj[s], a[LO][s]);
      P[s * TGC] = v;
      if (s == ssel) vsel = v;
    }
  } else {
    constexpr int MID = (LO + HI) / 2;
    if (rp < MID)
      gjcs_publish<RS, CS, SB0, TGC, LO, MID>(a, rp, l, pj, ssel, P, vsel);
    else
      gjcs_publish<RS, CS, SB0, TGC, MID, HI>(a, rp, l, pj, ssel, P, vsel);
  }
}

// Speculative Gauss–Jordan over the cluster (pivot order = hint, verified under the idamax rule, see
// rbns_newton_spec.cuh): per column one cluster barrier; the column's owner writes it (pivot entry as 0) and
// the pivot value into both CTAs, each CTA's pivot-row owners publish their half locally, ahead of the bulk.
template <int TGR, int TGC, int RS, int CS, int SB>
__device__ __forceinline__ void gjcs_block(double (&a)[RS][CS], unsigned& pmask, bool& bad, const int N,
                                           const int tr, const int tc, const int rank,
                                           GJCShared<TGR, TGC, RS, CS>& sh, GJCShared<TGR, TGC, RS, CS>* peer) {
  namespace cg = cooperative_groups;
  if constexpr (SB < CS) {
#pragma unroll 1
    for (int kk = 0; kk < 2 * TGC; ++kk) {
      const int k = SB * 2 * TGC + kk;
      if (k >= N) return;
      const int buf = k & 1;
      cg::this_cluster().sync();  // column k, pivot value, this CTA's half of row p_k in place
      const int p = static_cast<uint16_t>(sh.hint[k]);
      const int tp = p % TGR, rp = p / TGR;
      const double piv = sh.spv[buf], rpiv = sh.srp[buf];
      double pj[CS];
#pragma unroll
      for (int s = SB; s < CS; ++s) pj[s] = sh.SP[buf][s][tc];
      double l[RS];
#pragma unroll
      for (int r = 0; r < RS; ++r) l[r] = sh.colbuf[buf][tr][r] * rpiv;  // row p stored as 0
      // next column k+1: owner rank / thread-column / slot
      const int k1 = k + 1, g1 = k1 % (2 * TGC), o1 = g1 / TGC, t1 = g1 % TGC, s1 = k1 / (2 * TGC);
      const bool more = k1 < N;
      const int p1 = more ? static_cast<uint16_t>(sh.hint[k1]) : 0;
      if (more && tr == p1 % TGR) {  // this CTA's half of row p_{k+1}, after this step
        const double l1 = sh.colbuf[buf][p1 % TGR][p1 / TGR] * rpiv;
        double v = 0.0;
        gjcs_publish<RS, CS, SB, TGC>(a, p1 / TGR, l1, pj, s1, &sh.SP[buf ^ 1][0][tc], v);
        if (rank == o1 && tc == t1) {
          const double r1 = fabs(v) >= 2.2250738585072014e-308 ? rcp_nr(v) : 1.0 / v;
          sh.spv[buf ^ 1] = v;
          sh.srp[buf ^ 1] = r1;
          peer->spv[buf ^ 1] = v;
          peer->srp[buf ^ 1] = r1;
        }
      }
      // verification (rank 0; one row slot per thread-column)
      if (rank == 0) {
        const double apiv = fabs(piv);
#pragma unroll
        for (int r = tc; r < RS; r += TGC) {
          const int row = tr + TGR * r;
          const double ax = fabs(sh.colbuf[buf][tr][r]);
          const bool live = !((pmask >> r) & 1u);
          bad |= live && (ax > apiv || (ax == apiv && row < p));
        }
        if (!(apiv > 0.0) || !isfinite(piv)) bad = true;
      }
      if (tr == tp) pmask |= 1u << rp;
      if (threadIdx.x == 0) {
        sh.perm[k] = p;
        sh.piv[k] = piv;
      }
      // update; the owner of column k+1 stores it into both CTAs (its pivot's entry as 0)
#pragma unroll
      for (int s = SB; s < CS; ++s) {
#pragma unroll
        for (int r = 0; r < RS; ++r) a[r][s] = fma(-l[r], pj[s], a[r][s]);
        if (more && s == s1 && rank == o1 && tc == t1) {
#pragma unroll
          for (int r = 0; r < RS; ++r) {
            const double v = (tr + TGR * r == p1) ? 0.0 : a[r][s];
            sh.colbuf[buf ^ 1][tr][r] = v;
            peer->colbuf[buf ^ 1][tr][r] = v;
          }
        }
      }
    }
    gjcs_block<TGR, TGC, RS, CS, SB + 1>(a, pmask, bad, N, tr, tc, rank, sh, peer);
  }
}

// One sample (chunk position i_s) on this cluster; the caller's loop keeps both CTAs on the same positions.
template <int TGR, int TGC, int RS, int CS>
__device__ __forceinline__ void gjc_sample(const NewtonParams& p, const int i_s, GJCShared<TGR, TGC, RS, CS>& sh,
                                           GJCShared<TGR, TGC, RS, CS>* peer, const int rank) {
  namespace cg = cooperative_groups;
  constexpr int NT = TGR * TGC;
  constexpr int NW = NT / 32;
  cg::cluster_group cluster = cg::this_cluster();
  const int b = p.act[i_s];
    RBNS_CHECK(i_s >= 0 && i_s < p.n && b >= 0 && (p.B == 0 || b < p.B));
  const int tid = threadIdx.x, tc = tid / TGR, tr = tid % TGR;
  const int N = p.N;
  const int rhs_rank = (N % (2 * TGC)) / TGC, rhs_tc = N % TGC, rhs_slot = N / (2 * TGC);
  auto gcol = [&](int s) { return s * 2 * TGC + rank * TGC + tc; };

  newton_weights(p, b, sh.w);
  __syncthreads();
  double a[RS][CS];
  const double* Jb = p.J + int64_t(i_s) * p.ldj;
  // J into registers and the right-hand side as column N (rank rhs_rank); called again by the exact path
  auto load_system = [&]() {
  #pragma unroll
    for (int r = 0; r < RS; ++r)
  #pragma unroll
      for (int s = 0; s < CS; ++s) {
        const int i = tr + TGR * r, j = gcol(s);
        a[r][s] = (i < N && j < N) ? __ldcs(&Jb[jidx(i, j, N, p.jl)]) : 0.0;
      }

    // right-hand side −R = f − ½ J u − ½ L(μ)u as column N (owned by CTA rhs_rank)
    {
      double uj[CS];
  #pragma unroll
      for (int s = 0; s < CS; ++s) {
        const int j = gcol(s);
        uj[s] = j < N ? p.u[int64_t(b) * N + j] : 0.0;
      }
      const int lane = tid & 31, warp = tid >> 5;
  #pragma unroll
      for (int r = 0; r < RS; ++r) {
        double part = 0.0;
  #pragma unroll
        for (int s = 0; s < CS; ++s) part = fma(a[r][s], uj[s], part);
  #pragma unroll
        for (int o = TGR; o < 32; o <<= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (lane < TGR) sh.rowred[warp][tr + TGR * r] = part;
      }
      __syncthreads();
      GJCShared<TGR, TGC, RS, CS>* own = rank == rhs_rank ? &sh : peer;
      for (int i = tid; i < TGR * RS; i += NT) {
        double s = 0.0;
  #pragma unroll
        for (int w = 0; w < NW; ++w) s += sh.rowred[w][i];
        own->xred[rank][i] = s;
      }
      cluster.sync();
      if (rank == rhs_rank) {
        for (int i = tid; i < TGR * RS; i += NT) {
          double rhs = 0.0;
          if (i < N) {
            const double ju = sh.xred[0][i] + sh.xred[1][i];
            rhs = newton_rhs(p, Jb, i, ju, sh.w);
          }
          sh.rhs[i] = rhs;
        }
        __syncthreads();
        if (tc == rhs_tc) {
  #pragma unroll
          for (int r = 0; r < RS; ++r)
  #pragma unroll
            for (int s = 0; s < CS; ++s)
              if (s == rhs_slot) a[r][s] = sh.rhs[tr + TGR * r];
        }
      }
    }


  };
  for (int i = tid; i < TGR * RS; i += NT)
    sh.hint[i] = int16_t((p.hint_in && i < N) ? p.hint_in[int64_t(b) * N + i] : i);
  load_system();
  // ---- speculative pass (pivot order = hint) ----
  unsigned pmask = 0;
  bool sing = false, bad = false;
  {
    const int p0 = static_cast<uint16_t>(sh.hint[0]);
    if (rank == 0 && tc == 0) {  // column 0 into both CTAs, the pivot's entry as 0
#pragma unroll
      for (int r = 0; r < RS; ++r) {
        const double v = (tr + TGR * r == p0) ? 0.0 : a[r][0];
        sh.colbuf[0][tr][r] = v;
        peer->colbuf[0][tr][r] = v;
      }
    }
    if (tr == p0 % TGR) {
      double z[CS], v = 0.0;
#pragma unroll
      for (int s = 0; s < CS; ++s) z[s] = 0.0;
      gjcs_publish<RS, CS, 0, TGC>(a, p0 / TGR, 0.0, z, 0, &sh.SP[0][0][tc], v);
      if (rank == 0 && tc == 0) {
        const double r0 = fabs(v) >= 2.2250738585072014e-308 ? rcp_nr(v) : 1.0 / v;
        sh.spv[0] = v;
        sh.srp[0] = r0;
        peer->spv[0] = v;
        peer->srp[0] = r0;
      }
    }
  }
  gjcs_block<TGR, TGC, RS, CS, 0>(a, pmask, bad, N, tr, tc, rank, sh, peer);
  {
    const int mine = __syncthreads_or(bad);
    if (tid == 0) {
      sh.bad_any[rank] = mine;
      peer->bad_any[rank] = mine;
    }
    cluster.sync();
  }
  if (sh.bad_any[0] || sh.bad_any[1]) {  // wrong hint: the exact full-search factorization from the original J
    if (rank == 0 && tid == 0 && p.spec_miss) atomicAdd(p.spec_miss, 1);
    load_system();
    pmask = 0;
    gjc_block<TGR, TGC, RS, CS, 0>(a, pmask, sing, N, tr, tc, rank, sh, peer);
  }


  if (rank == rhs_rank) {
    if (!sing && tc == rhs_tc) {
#pragma unroll
      for (int r = 0; r < RS; ++r)
#pragma unroll
        for (int s = 0; s < CS; ++s)
          if (s == rhs_slot) sh.rhs[tr + TGR * r] = a[r][s];
    }
    __syncthreads();
    double d2 = 0.0, un2 = 0.0, o2 = 0.0;  // o2: unknowns outside the stop norm
    if (!sing) {
      for (int k = tid; k < N; k += NT) {
        const double x = sh.rhs[sh.perm[k]] / sh.piv[k];
        const double unew = p.u[int64_t(b) * N + k] + x;
        if (k < p.n_stop) {
          d2 = fma(x, x, d2);
          un2 = fma(unew, unew, un2);
        } else {
          o2 = fma(x, x, fma(unew, unew, o2));
        }
      }
    }
    d2 = block_sum<NT>(d2, sh.red[0]);
    un2 = block_sum<NT>(un2, sh.red[1]);
    const bool finite = !__syncthreads_or(!isfinite(o2)) && isfinite(d2) && isfinite(un2);
    if (!sing && finite) {
      for (int k = tid; k < N; k += NT) {
        const double x = sh.rhs[sh.perm[k]] / sh.piv[k];
        p.u[int64_t(b) * N + k] += x;
      }
    }
    if (tid == 0) {
      int st;
      if (sing)
        st = RBNS_SINGULAR_SYSTEM;
      else if (!finite)
        st = RBNS_NONFINITE;
      else if (sqrt(d2) <= p.tol * (p.stop_abs ? 1.0 : sqrt(un2)))
        st = RBNS_CONVERGED;
      else if (p.iter >= p.max_iter)
        st = RBNS_NON_CONVERGED;
      else
        st = kStatusActive;
      p.status[b] = int8_t(st);
      p.iters[b] = p.iter;
      if (!sing && finite) p.last[b] = sqrt(d2);
    }
  }
  if (rank == 0 && p.hint_out && !sing) {  // the order used: the next Newton iteration's hint
    for (int i = tid; i < N; i += NT) p.hint_out[int64_t(b) * N + i] = int16_t(sh.perm[i]);
  }
  cluster.sync();  // the peer may still read this CTA's shared memory
}

// Grid: two CTAs per position.  p.sub == NULL: positions 0 .. n-1, one per cluster (grid 2n).  p.sub != NULL:
// the listed positions sub[0 .. *n_sub) (the samples a tiled kernel handed back), strided over the grid's
// clusters, so the grid need not know the device-side count.
template <int TGR, int TGC, int RS, int CS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TGR * TGC, 1)
    newton_gjc_kernel(const NewtonParams p) {
  namespace cg = cooperative_groups;
  static_assert(TGR == 16 && (TGR * TGC) % 32 == 0, "owner half-warp layout needs TGR = 16");
  __shared__ GJCShared<TGR, TGC, RS, CS> sh;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = int(cluster.block_rank());
  GJCShared<TGR, TGC, RS, CS>* peer = cluster.map_shared_rank(&sh, rank ^ 1);
  const int cnt = p.sub ? *p.n_sub : p.n;
#pragma unroll 1
  for (int k = int(blockIdx.x / 2); k < cnt; k += int(gridDim.x / 2))
    gjc_sample<TGR, TGC, RS, CS>(p, p.sub ? p.sub[k] : k, sh, peer, rank);
}

}  // namespace rbns
