// rbns_newton2.cuh — K3 (default): per-sample Newton update, register Gauss–Jordan with a CTA-parallel
// pivot search.
//
// Same data distribution as rbns_newton.cuh: one CTA per μ sample, [J | −R] in registers, 2-D cyclic over a
// TGR×TGC thread grid (thread (tr, tc) owns rows tr + TGR·r and columns tc + TGC·s), column blocks left of
// the current block skipped statically.  What changes is the critical path of one elimination step.  The
// rank-1 kernel let the TGR owners of the pivot column search it serially (RS values each, then a lane
// butterfly): a few hundred dependent instructions in one warp while the other warps idle.  Here every step is
//     A  owners write column k to shared memory                    (RS independent stores)      barrier
//     B  every thread takes one row: key |a|, warp argmax by redux.sync, per-warp winner         barrier
//     C  all threads reduce the NW winners (ties: smaller row), pivot-row owners publish the row,
//        1/pivot (MUFU + Newton)                                                                  barrier
//     D  register rank-1 update
// Three short barriers instead of one long serial chain.  Pivot = max |a| over unpivoted rows, ties to the
// smaller row (LAPACK idamax), i.e. unchanged partial pivoting.
//
// Reference: SPEC.md:558 (LU with partial pivoting), SPEC.md:520-523 / :557-559 (Newton step and stop rule);
// residual as in rbns_newton.cuh.
#pragma once

#include "rbns_common.cuh"
#include "rbns_newton.cuh"

namespace rbns {

template <int TGR, int TGC, int RS, int CS>
struct GJ2Shared {
  static constexpr int NT = TGR * TGC;
  static constexpr int NW = (NT + 31) / 32;
  static constexpr int NR = TGR * RS;
  NewtonWeights w;
  double col[2][NR];             // pivot column (row-indexed), double-buffered by step parity
  struct alignas(16) Cand {
    unsigned long long key;      // |a| bits (sign cleared): orders like |a|
    int row;
    int pad;
    double val;                  // signed value of the warp winner
    double pad2;
  } cand[NW];
  signed char pivoted[NR];
  double P[CS][TGC];             // pivot row, [slot][thread-column]
  double piv[NR];
  int perm[NR];
  double rhs[NR];
  double rowred[NW][NR];
  double red[2][NW];
  int sing;
};

// MODE (development ablations, tools/lu_probe.cu; results are wrong for MODE != 0): bit 0 skips the update
// FMAs, bit 1 skips the pivot search (p = k), bit 2 skips the pivot-row publication.
template <int TGR, int TGC, int RS, int CS, int SB, int MODE = 0>
__device__ __forceinline__ void gj2_block(double (&a)[RS][CS], bool& sing, const int N, const int tr, const int tc,
                                          GJ2Shared<TGR, TGC, RS, CS>& sh) {
  constexpr int NT = TGR * TGC;
  constexpr int NW = GJ2Shared<TGR, TGC, RS, CS>::NW;
  constexpr int NR = TGR * RS;
  constexpr int RPT = (NR + NT - 1) / NT;  // rows per thread in the search
  if constexpr (SB < CS) {
    if (sing) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll 1
    for (int kk = 0; kk < TGC; ++kk) {
      const int k = SB * TGC + kk;
      if (k >= N) return;
      const int buf = k & 1;
      // A: owners publish column k
      if (tc == kk) {
#pragma unroll
        for (int r = 0; r < RS; ++r) sh.col[buf][tr + TGR * r] = a[r][SB];
      }
      __syncthreads();
      // B: one row per thread, warp argmax on (high word, low word, row)
      if constexpr (!(MODE & 2)) {
        unsigned bhi = 0, blo = 0;
        int brow = 0x7fffffff;
        double bval = 0.0;
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
          const int row = tid + NT * j;
          if (row < N && !sh.pivoted[row]) {
            const double v = sh.col[buf][row];
            const unsigned hi = unsigned(__double2hiint(v)) & 0x7fffffffu, lo = unsigned(__double2loint(v));
            if (hi > bhi || (hi == bhi && lo > blo)) {
              bhi = hi;
              blo = lo;
              brow = row;
              bval = v;
            }
          }
        }
        const unsigned mhi = __reduce_max_sync(0xffffffffu, bhi);
        unsigned cnd = __ballot_sync(0xffffffffu, bhi == mhi);
        unsigned mlo = blo;
        if (__popc(cnd) > 1) {
          mlo = __reduce_max_sync(0xffffffffu, bhi == mhi ? blo : 0u);
          cnd = __ballot_sync(0xffffffffu, bhi == mhi && blo == mlo);
        }
        const int wrow =
            int(__reduce_min_sync(0xffffffffu, ((cnd >> lane) & 1u) ? unsigned(brow) : 0x7fffffffu));
        const int src = __ffs(cnd) - 1;
        const unsigned wlo = __shfl_sync(0xffffffffu, blo, src);
        const double wval = __shfl_sync(0xffffffffu, bval, src);
        if (lane == 0) {
          sh.cand[warp].key = (static_cast<unsigned long long>(mhi) << 32) | wlo;
          sh.cand[warp].row = wrow;
          sh.cand[warp].val = wval;
        }
      }
      if constexpr (!(MODE & 2)) __syncthreads();
      // C: reduce the warp winners, publish the pivot row
      unsigned long long bkey = 0;
      int p = 0x7fffffff;
      double piv = 0.0;
      if constexpr (MODE & 2) {
        p = k;
        piv = sh.col[buf][k];
        bkey = 1;
      } else
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const unsigned long long key = sh.cand[w].key;
        const int row = sh.cand[w].row;
        const double v = sh.cand[w].val;
        if (row < N && (key > bkey || (key == bkey && row < p))) {
          bkey = key;
          p = row;
          piv = v;
        }
      }
      if (p >= N || bkey == 0ull || (bkey >> 52) == 0x7ffull) {  // zero or non-finite: uniform
        sing = true;
        return;
      }
      const double rpiv = fabs(piv) >= 2.2250738585072014e-308 ? rcp_nr(piv) : 1.0 / piv;
      if (tid == p % NT) sh.col[buf][p] = 0.0;  // the row's searcher (it read row p in B): pivot row not updated
      const int tp = p % TGR, rp = p / TGR;
      if constexpr (!(MODE & 4))
        if (tr == tp) publish_row<RS, CS, SB, TGC>(a, rp, &sh.P[0][tc]);
      __syncthreads();
      // D: rank-1 update (the pivot row itself: l = 0)
      if (tid == 0) {
        sh.pivoted[p] = 1;
        sh.perm[k] = p;
        sh.piv[k] = piv;
      }
      double pj[CS];
#pragma unroll
      for (int s = SB; s < CS; ++s) pj[s] = sh.P[s][tc];
      if constexpr (!(MODE & 1)) {
#pragma unroll
        for (int r = 0; r < RS; ++r) {
          const double l = sh.col[buf][tr + TGR * r] * rpiv;
#pragma unroll
          for (int s = SB; s < CS; ++s) a[r][s] = fma(-l, pj[s], a[r][s]);
        }
      } else {
        a[0][SB] += pj[SB] * rpiv;  // keep the loads alive
      }
    }
    gj2_block<TGR, TGC, RS, CS, SB + 1, MODE>(a, sing, N, tr, tc, sh);
  }
}

// Kernel prologue shared by the register Gauss–Jordan variants: θ(μ), ν, the J tile into registers and the
// right-hand side −R = f − ½ J u − ½ L(μ)u as column N.  SH needs w, pivoted, rowred, rhs.
template <int TGR, int TGC, int RS, int CS, class SH>
__device__ __forceinline__ void gj_load_system(const NewtonParams& p, int i_s, int b, double (&a)[RS][CS], SH& sh) {
  constexpr int NT = TGR * TGC;
  constexpr int NW = (NT + 31) / 32;
  constexpr int NR = TGR * RS;
  const int tid = threadIdx.x, tc = tid / TGR, tr = tid % TGR;
  const int N = p.N;
  newton_weights(p, b, sh.w);
  for (int r = tid; r < NR; r += NT) sh.pivoted[r] = 0;
  __syncthreads();
  const double* Jb = p.J + int64_t(i_s) * p.ldj;
#pragma unroll
  for (int r = 0; r < RS; ++r)
#pragma unroll
    for (int s = 0; s < CS; ++s) {
      const int i = tr + TGR * r, j = tc + TGC * s;
      a[r][s] = (i < N && j < N) ? __ldcs(&Jb[jidx(i, j, N, p.jl)]) : 0.0;
    }
  double uj[CS];
#pragma unroll
  for (int s = 0; s < CS; ++s) {
    const int j = tc + TGC * s;
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
  for (int i = tid; i < NR; i += NT) {
    double rhs = 0.0;
    if (i < N) {
      double ju = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) ju += sh.rowred[w][i];
      rhs = newton_rhs(p, Jb, i, ju, sh.w);
    }
    sh.rhs[i] = rhs;
  }
  __syncthreads();
  if (tc == N % TGC) {
#pragma unroll
    for (int r = 0; r < RS; ++r)
#pragma unroll
      for (int s = 0; s < CS; ++s)
        if (tc + TGC * s == N) a[r][s] = sh.rhs[tr + TGR * r];
  }
}

// Kernel epilogue: x_k = rhs'[perm k] / piv_k, u += x, ‖δ‖ / ‖u‖ stop rule, per-sample status.
// SH needs rhs, perm, piv, red.
template <int TGR, int TGC, int RS, int CS, class SH>
__device__ __forceinline__ void gj_finish(const NewtonParams& p, int b, const double (&a)[RS][CS], bool sing, SH& sh) {
  constexpr int NT = TGR * TGC;
  const int tid = threadIdx.x, tc = tid / TGR, tr = tid % TGR;
  const int N = p.N;
  __syncthreads();
  if (!sing && tc == N % TGC) {
#pragma unroll
    for (int r = 0; r < RS; ++r)
#pragma unroll
      for (int s = 0; s < CS; ++s)
        if (tc + TGC * s == N) sh.rhs[tr + TGR * r] = a[r][s];
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

template <int TGR, int TGC, int RS, int CS, int MODE = 0>
__global__ void __launch_bounds__(TGR * TGC, (TGR * TGC <= 128 ? 2 : 1)) newton_gj2_kernel(const NewtonParams p) {
  static_assert(RS <= 32 && TGR <= 32 && TGC <= 32 && (TGR * TGC) % 32 == 0, "shape");
  __shared__ GJ2Shared<TGR, TGC, RS, CS> sh;
  // one sample per CTA, or (subset launch: the samples a speculative pass handed back, device-side count) a
  // grid-stride loop over the subset so the launch can be small
  const int n = p.sub ? *p.n_sub : p.n;
  const int tid = threadIdx.x, tc = tid / TGR, tr = tid % TGR;
#pragma unroll 1
  for (int j = blockIdx.x; j < n; j += gridDim.x) {
    const int i_s = p.sub ? p.sub[j] : j;
    const int b = p.act[i_s];
    RBNS_CHECK(i_s >= 0 && i_s < p.n && b >= 0 && (p.B == 0 || b < p.B));
    double a[RS][CS];
    gj_load_system<TGR, TGC, RS, CS>(p, i_s, b, a, sh);
    bool sing = false;
    gj2_block<TGR, TGC, RS, CS, 0, MODE>(a, sing, p.N, tr, tc, sh);
    gj_finish<TGR, TGC, RS, CS>(p, b, a, sing, sh);
    if (p.hint_out && !sing) {  // the order partial pivoting chose: the next iteration's speculation hint
      for (int i = tid; i < p.N; i += TGR * TGC) p.hint_out[int64_t(b) * p.N + i] = int16_t(sh.perm[i]);
    }
    __syncthreads();  // shared memory is reused by the next sample
  }
}

}  // namespace rbns
