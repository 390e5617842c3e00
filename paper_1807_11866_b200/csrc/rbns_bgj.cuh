// rbns_bgj.cuh — K3 (blocked): per-sample Newton update by blocked Gauss–Jordan elimination with partial
// pivoting, trailing updates on the FP64 tensor cores (DMMA.8x8x4).
//
// One CTA (NW warps) per μ sample.  The augmented matrix [J | −R] (N × (N+1), padded to RT×CT tiles of 8×8)
// lives in REGISTERS in the DMMA accumulator layout: warp w owns column tiles j ≡ w (mod NW), all row tiles;
// lane (g = lane/4, t = lane%4) holds entries (8i+g, 8j+2t) and (8i+g, 8j+2t+1) of tile (i, j).
//
// Panel P = the 8 columns of tile P.  Its owner warp copies the tile to shared memory and runs the scalar
// Gauss–Jordan steps with partial pivoting on it (pivot = max |a| over rows not yet pivoted, ties to the
// smaller row index; warp-wide argmax with redux.sync), recording for every row i the multipliers l_{i,c}
// (l = 0 on the step's own pivot row) and the pivot rows p_c.  The composite effect of the 8 steps on any
// other column v is v ← v − L·y with y = T⁻¹ v[Π], T[c][c'] = l_{p_c,c'} (c' < c, unit diagonal); so each
// warp updates its trailing tiles with two DMMAs per tile: acc(i,j) += (−L)(i) · (W · M_Π(j)), W = T⁻¹.
// This is exactly the scalar Gauss–Jordan sequence of the rank-1 kernel (rbns_newton.cuh) regrouped by 8
// columns, with one CTA barrier per panel instead of two per column.  Look-ahead: the owner of tile P+1 applies
// panel P to that tile first and factors panel P+1 while the other warps finish panel P; the owner's other
// tiles receive panel P one iteration later (three panel buffers), keeping the serial chain short.
//
// Speculative pivoting: the kernel first assumes partial pivoting never interchanges rows (the pivot of
// column k is row k) and verifies every column with a warp ballot (an unpivoted row with strictly larger |a|
// would be chosen by idamax; equal ones lose the tie to the smaller index).  On the first rejected column the
// sample is redone with the full pivot search, so the pivot sequence always equals partial pivoting's.
//
// Reference: dense LU with partial pivoting for the Newton systems, Newton step / stop rule
// (SPEC.md:520-523, :557-559); see rbns_newton.cuh for the residual formula.
#pragma once

#include "rbns_common.cuh"
#include "rbns_newton.cuh"

namespace rbns {



template <int RT, int CT, int NW>
struct BGJShared {
  static constexpr int NR = 8 * RT;
  static constexpr int PS = 9;                   // panel row stride (doubles): conflict-free column reads
  static constexpr int NB = 3;                   // panel buffers (P, P-1 pending, P+1 being factored)
  NewtonWeights w;
  int sing;
  int fail;                                      // speculative pass rejected: rerun with pivot search
  int nc[NB];                                    // columns factored in the panel of each buffer
  int prow[NB][8];                               // pivot rows of the panel
  signed char rowpos[NB][NR];                    // row -> step c within the panel (or -1)
  signed char pivoted[NR];                       // row already used as a pivot
  double panel[NR * PS];                         // the panel being factored
#ifndef RBNS_BGJ_LS
#define RBNS_BGJ_LS 8
#endif
#ifndef RBNS_BGJ_WS
#define RBNS_BGJ_WS 10  // 80-byte rows: the four T⁻¹ rows one warp reads per k-step sit in distinct banks
#endif
  static constexpr int LS = RBNS_BGJ_LS;         // multiplier row stride (doubles)
  static constexpr int WS = RBNS_BGJ_WS;         // T⁻¹ row stride (doubles)
  double L[NB][NR][LS];                          // −l_{i,c} (negated multipliers), A operand of the DMMA
  double W[NB][8][WS];                           // T⁻¹ (unit lower triangular)
  double Mpi[NW][8][8];                          // per-warp gathered pivot rows of one column tile
  double pivval[NR];
  int perm[NR];
  double rowred[NW][NR];
  double rhs[NR];
  double red[2][NW];
};

// ---- warp-wide argmax of a non-negative 64-bit key with a row tie-break (redux.sync on 32-bit halves) -----
__device__ __forceinline__ int warp_argmax_row(unsigned long long key, int row) {
  const unsigned hi = unsigned(key >> 32), lo = unsigned(key);
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  unsigned cand = __ballot_sync(0xffffffffu, hi == mhi);
  if (__popc(cand) > 1) {
    unsigned mlo = 0;
    if (hi == mhi) mlo = __reduce_max_sync(cand, lo);
    mlo = __shfl_sync(0xffffffffu, mlo, __ffs(cand) - 1);
    cand = __ballot_sync(0xffffffffu, hi == mhi && lo == mlo);
    if (__popc(cand) > 1) {  // exact tie on |a|: smallest row index (LAPACK idamax order)
      unsigned r = 0xffffffffu;
      if (hi == mhi && lo == mlo) r = __reduce_min_sync(cand, unsigned(row));
      r = __shfl_sync(0xffffffffu, r, __ffs(cand) - 1);
      return int(r);
    }
  }
  return __shfl_sync(0xffffffffu, row, __ffs(cand) - 1);
}

// W = T⁻¹ with T[c][c'] = l_{p_c, c'} = −L[p_c][c'] (c' < c), unit lower triangular; lane c' builds column c'.
template <int RT, int CT, int NW>
__device__ __forceinline__ void bgj_compute_w(int buf, int done, BGJShared<RT, CT, NW>& sh) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  if (lane < 8) {
    const int cp = lane;
    double w[8];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      double s = (cc == cp) ? 1.0 : 0.0;
      if (cc < done) {
        const int prr = sh.prow[buf][cc];
#pragma unroll
        for (int c2 = 0; c2 < cc; ++c2) s = fma(sh.L[buf][prr][c2], w[c2], s);
      }
      w[cc] = s;
    }
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) sh.W[buf][cc][cp] = w[cc];
  }
  __syncwarp();
}

// Speculative panel factorization (no interchanges), the serial critical path of the elimination.  The
// panel rows are held in registers rotated so that row 8P + c sits at (lane c, slot 0): the pivot of column
// c is lane c's pr[0][0].  Every lane computes the reciprocal of its own pr[0][0] right after the previous
// update (no broadcast before the reciprocal), then the pivot lane's values are shuffled out.  The register
// panel is rotated left after each column so the current column is always slot 0 (loop not unrolled).
// Verification compares the high words of |a| (sign-cleared IEEE bits: exponent + 20 mantissa bits); only
// an equal high word needs the exact 64-bit comparison.
template <int RT, int CT, int NW>
__device__ __forceinline__ void bgj_factor_spec(int P, int buf, int N, BGJShared<RT, CT, NW>& sh) {
  constexpr int NR = 8 * RT;
  constexpr int PS = BGJShared<RT, CT, NW>::PS;
  constexpr int RPL = (NR + 31) / 32;
  constexpr int NPOS = 32 * RPL;
  const int lane = threadIdx.x & 31;
  const int nc = min(8, N - 8 * P);
  if (nc < 8) {  // full panels overwrite every multiplier column
    for (int e = lane; e < NR * BGJShared<RT, CT, NW>::LS; e += 32) (&sh.L[buf][0][0])[e] = 0.0;
    __syncwarp();
  }
  int rr[RPL];
  double pr[RPL][8];
#pragma unroll
  for (int s = 0; s < RPL; ++s) {
    rr[s] = (lane + 32 * s + 8 * P) % NPOS;
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) pr[s][cc] = rr[s] < NR ? sh.panel[rr[s] * PS + cc] : 0.0;
  }
  int c = 0;
  bool bad = false;
#pragma unroll 1
  for (; c < nc; ++c) {
    const int k = 8 * P + c;
    const double myrcp = rcp_nr(pr[0][0]);
    const double piv = __shfl_sync(0xffffffffu, pr[0][0], c);
    const double rp = __shfl_sync(0xffffffffu, myrcp, c);
    double prow[8];
#pragma unroll
    for (int cc = 1; cc < 8; ++cc) prow[cc] = __shfl_sync(0xffffffffu, pr[0][cc], c);
    // verification: no row below k (not yet pivoted) may beat |piv|
    const int phi = __double2hiint(piv) & 0x7fffffff;
    int bh = 0;
#pragma unroll
    for (int s = 0; s < RPL; ++s) {
      const int h = (rr[s] > k && rr[s] < N) ? (__double2hiint(pr[s][0]) & 0x7fffffff) : 0;
      bh = max(bh, h);
    }
    unsigned gt = __ballot_sync(0xffffffffu, bh > phi);
    if (__ballot_sync(0xffffffffu, bh == phi)) {  // rare: equal high words, compare exactly
      bool g = false;
#pragma unroll
      for (int s = 0; s < RPL; ++s)
        g |= rr[s] > k && rr[s] < N && fabs(pr[s][0]) > fabs(piv);
      gt |= __ballot_sync(0xffffffffu, g);
    }
    // no early exit: the flags are collected and checked once after the panel (a rejected speculation reruns
    // the whole sample with the pivot search), so the branch never waits on the ballots inside the chain
    bad |= gt != 0u || !(fabs(piv) >= 2.2250738585072014e-308) || !isfinite(piv);
    double l[RPL];
#pragma unroll
    for (int s = 0; s < RPL; ++s) {  // next column first: it carries the next pivot (critical path)
      l[s] = (s == 0 && lane == c) ? 0.0 : pr[s][0] * rp;
      pr[s][0] = fma(-l[s], prow[1], pr[s][1]);
    }
#pragma unroll
    for (int s = 0; s < RPL; ++s) {
      if (rr[s] < NR) sh.L[buf][rr[s]][c] = -l[s];
#pragma unroll
      for (int cc = 1; cc < 7; ++cc) pr[s][cc] = fma(-l[s], prow[cc + 1], pr[s][cc + 1]);  // update + rotate
      pr[s][7] = 0.0;
    }
    if (lane == 0) sh.pivval[k] = piv;
  }
  if (lane < 8) {
    sh.prow[buf][lane] = 8 * P + lane;
    if (lane < c) sh.perm[8 * P + lane] = 8 * P + lane;
  }
  if (lane == 0) {
    sh.nc[buf] = c;
    if (bad) sh.fail = 1;  // an interchange (or a zero / non-finite pivot): redo with the pivot search
  }
  if (N / 8 == P) {  // the right-hand side column (index N - 8P = nc in this panel) is now pr[s][0]
#pragma unroll
    for (int s = 0; s < RPL; ++s)
      if (rr[s] < NR) sh.rhs[rr[s]] = pr[s][0];
  }
  __syncwarp();
  // W = T⁻¹, T[cc][c2] = l_{8P+cc, c2} = −L[8P+cc][c2] (pivot rows in natural order): all 28 entries are
  // loaded up front (independent loads), then each lane c' < 8 runs the short forward substitution
  if (lane < 8) {
    const int cp = lane;
    double T[8][8];
#pragma unroll
    for (int cc = 1; cc < 8; ++cc)
#pragma unroll
      for (int c2 = 0; c2 < cc; ++c2) T[cc][c2] = cc < c ? sh.L[buf][8 * P + cc][c2] : 0.0;
    double w[8];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      double sacc = (cc == cp) ? 1.0 : 0.0;
#pragma unroll
      for (int c2 = 0; c2 < cc; ++c2) sacc = fma(T[cc][c2], w[c2], sacc);
      w[cc] = sacc;
    }
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) sh.W[buf][cc][cp] = w[cc];
  }
  __syncwarp();
}

// Panel factorization with the full partial-pivoting search (warp argmax per column); rows in natural order.
template <int RT, int CT, int NW>
__device__ __forceinline__ void bgj_factor_pivot(int P, int buf, int N, BGJShared<RT, CT, NW>& sh) {
  constexpr int NR = 8 * RT;
  constexpr int PS = BGJShared<RT, CT, NW>::PS;
  constexpr int RPL = (NR + 31) / 32;
  const int lane = threadIdx.x & 31;
  for (int c = 0; c < sh.nc[buf]; ++c) sh.rowpos[buf][sh.prow[buf][c]] = -1;  // stale map of panel P-3
  const int nc = min(8, N - 8 * P);
  if (nc < 8) {
    for (int e = lane; e < NR * BGJShared<RT, CT, NW>::LS; e += 32) (&sh.L[buf][0][0])[e] = 0.0;
  }
  double pr[RPL][8];
  unsigned piv_mask = 0;  // bit s: row lane + 32 s already pivoted (or padding)
#pragma unroll
  for (int s = 0; s < RPL; ++s) {
    const int r = lane + 32 * s;
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) pr[s][cc] = r < NR ? sh.panel[r * PS + cc] : 0.0;
    if (r >= N || sh.pivoted[r]) piv_mask |= 1u << s;
  }
  __syncwarp();
  int c = 0;
#pragma unroll 1
  for (; c < nc; ++c) {
    const int k = 8 * P + c;
    unsigned long long best = 0;
    int brow = NR;
#pragma unroll
    for (int s = 0; s < RPL; ++s) {
      const unsigned long long key =
          ((piv_mask >> s) & 1u) ? 0ull : (unsigned long long)__double_as_longlong(fabs(pr[s][0]));
      if (key > best) {
        best = key;
        brow = lane + 32 * s;
      }
    }
    const int p = warp_argmax_row(best, brow);
    const int ol = p & 31, ps = p >> 5;
    double prow[8];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      double sel = pr[0][cc];
#pragma unroll
      for (int s = 1; s < RPL; ++s) sel = (ps == s) ? pr[s][cc] : sel;
      prow[cc] = __shfl_sync(0xffffffffu, sel, ol);
    }
    const double piv = prow[0];
    if (p >= N || !(fabs(piv) > 0.0) || !isfinite(piv)) {  // warp-uniform
      if (lane == 0) sh.sing = 1;
      break;
    }
    const double rp = fabs(piv) >= 2.2250738585072014e-308 ? rcp_nr(piv) : 1.0 / piv;
    double l[RPL];
#pragma unroll
    for (int s = 0; s < RPL; ++s) {
      l[s] = (lane + 32 * s == p) ? 0.0 : pr[s][0] * rp;
      pr[s][0] = fma(-l[s], prow[1], pr[s][1]);
    }
#pragma unroll
    for (int s = 0; s < RPL; ++s) {
      const int r = lane + 32 * s;
      if (r < NR) sh.L[buf][r][c] = -l[s];
#pragma unroll
      for (int cc = 1; cc < 7; ++cc) pr[s][cc] = fma(-l[s], prow[cc + 1], pr[s][cc + 1]);
      pr[s][7] = 0.0;
    }
    if (lane == ol) piv_mask |= 1u << ps;
    if (lane == 0) {
      sh.perm[k] = p;
      sh.pivval[k] = piv;
      sh.prow[buf][c] = p;
      sh.pivoted[p] = 1;
      sh.rowpos[buf][p] = (signed char)c;
    }
    __syncwarp();
  }
  if (lane == 0) sh.nc[buf] = c;
  if (N / 8 == P) {
#pragma unroll
    for (int s = 0; s < RPL; ++s)
      if (lane + 32 * s < NR) sh.rhs[lane + 32 * s] = pr[s][0];
  }
  bgj_compute_w<RT, CT, NW>(buf, c, sh);
}

// Apply panel P (buffer buf) to this warp's owned column tiles selected by `mask` (bit jj).
template <int RT, int CT, int NW, int J0>
__device__ __forceinline__ void bgj_update(double (&acc)[(CT - J0 + NW - 1) / NW][RT][2], unsigned mask, int buf,
                                           int P, bool spec, BGJShared<RT, CT, NW>& sh) {
  constexpr int JJ = (CT - J0 + NW - 1) / NW;
  const int warp = (threadIdx.x % (NW * 32)) >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  if (!mask) return;
  const int nc = sh.nc[buf];
  double b0[JJ], b1[JJ];
#pragma unroll
  for (int jj = 0; jj < JJ; ++jj) {
    b0[jj] = b1[jj] = 0.0;
    if (!((mask >> jj) & 1u)) continue;
    // gather the pivot rows of tile jj: M_pi[c][col]
    if (spec) {  // pivot rows are row tile P in natural order (rows beyond N are zero padding)
#pragma unroll
      for (int i = 0; i < RT; ++i)
        if (i == P) {
          sh.Mpi[warp][g][2 * t] = acc[jj][i][0];
          sh.Mpi[warp][g][2 * t + 1] = acc[jj][i][1];
        }
    } else {
#pragma unroll
      for (int e = lane; e < 64; e += 32) (&sh.Mpi[warp][0][0])[e] = 0.0;
      __syncwarp();
#pragma unroll
      for (int i = 0; i < RT; ++i) {
        const int pos = sh.rowpos[buf][8 * i + g];
        if (pos >= 0 && pos < nc) {
          sh.Mpi[warp][pos][2 * t] = acc[jj][i][0];
          sh.Mpi[warp][pos][2 * t + 1] = acc[jj][i][1];
        }
      }
    }
    __syncwarp();
    // B fragments of Y = W · M_pi: lane (g,t) needs Y[t][g] and Y[t+4][g]
    double y0 = 0.0, y1 = 0.0;
#pragma unroll
    for (int c2 = 0; c2 < 8; ++c2) {
      const double m = sh.Mpi[warp][c2][g];
      y0 = fma(sh.W[buf][t][c2], m, y0);
      y1 = fma(sh.W[buf][t + 4][c2], m, y1);
    }
    b0[jj] = y0;
    b1[jj] = y1;
    __syncwarp();
  }
#pragma unroll
  for (int i = 0; i < RT; ++i) {
    const double a0 = sh.L[buf][8 * i + g][t], a1 = sh.L[buf][8 * i + g][t + 4];
#pragma unroll
    for (int jj = 0; jj < JJ; ++jj) {
      if (!((mask >> jj) & 1u)) continue;
      dmma_8x8x4(acc[jj][i][0], acc[jj][i][1], a0, b0[jj]);
      dmma_8x8x4(acc[jj][i][0], acc[jj][i][1], a1, b1[jj]);
    }
  }
}

template <int RT, int CT, int NW, int J0>
__device__ __forceinline__ void bgj_copy_panel(const double (&acc)[(CT - J0 + NW - 1) / NW][RT][2], int jsel,
                                               BGJShared<RT, CT, NW>& sh) {
  constexpr int PS = BGJShared<RT, CT, NW>::PS;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int jj = 0; jj < (CT - J0 + NW - 1) / NW; ++jj) {
    if (jj != jsel) continue;
#pragma unroll
    for (int i = 0; i < RT; ++i) {
      sh.panel[(8 * i + g) * PS + 2 * t] = acc[jj][i][0];
      sh.panel[(8 * i + g) * PS + 2 * t + 1] = acc[jj][i][1];
    }
  }
  __syncwarp();
}

// One elimination pass: reset the shared state, load [J | −R] into the tiles, blocked Gauss–Jordan.
// J0 = 1: column tile 0 is never held in registers — it is only ever panel 0, loaded straight into the panel
// buffer (its columns are eliminated by their own factorization) — so 4 warps hold the 12 remaining tiles of a
// 13-tile (N ≤ 103) system 3 apiece: balanced registers, two CTAs per SM.
// i_s: chunk position of the sample (its J block).
template <int RT, int CT, int NW, int J0>
__device__ __forceinline__ void bgj_pass(const NewtonParams& p, int i_s, int b, bool spec,
                                         double (&acc)[(CT - J0 + NW - 1) / NW][RT][2], BGJShared<RT, CT, NW>& sh) {
  constexpr int JJ = (CT - J0 + NW - 1) / NW;
  constexpr int PS = BGJShared<RT, CT, NW>::PS;
  constexpr int NR = 8 * RT;
  constexpr int NT = NW * 32;
  constexpr int NB = BGJShared<RT, CT, NW>::NB;
  const int tid = threadIdx.x % NT, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int N = p.N;
  if (tid == 0) {
    sh.sing = 0;
    sh.fail = 0;
    for (int q = 0; q < NB; ++q) sh.nc[q] = 0;
  }
  for (int r = tid; r < NR; r += NT) {
    sh.pivoted[r] = 0;
    for (int q = 0; q < NB; ++q) sh.rowpos[q][r] = -1;
  }
  __syncthreads();
  const double* Jb = p.J + int64_t(i_s) * p.ldj;

  // ---- load the owned tiles of J ----
#pragma unroll
  for (int jj = 0; jj < JJ; ++jj) {
    const int j = J0 + warp + NW * jj;
#pragma unroll
    for (int i = 0; i < RT; ++i) {
      const int r = 8 * i + g;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = 8 * j + 2 * t + e;
        double v = 0.0;
        if (j < CT && r < N && col < N) v = __ldcs(&Jb[int64_t(r) * N + col]);
        acc[jj][i][e] = v;
      }
    }
  }
  if constexpr (J0 == 1) {  // column tile 0 goes straight to the panel buffer
    for (int e = tid; e < NR * 8; e += NT) {
      const int r = e >> 3, c = e & 7;
      sh.panel[r * PS + c] = (r < N && c < N) ? __ldcs(&Jb[int64_t(r) * N + c]) : 0.0;
    }
  }
  if (warp == 0) RBNS_TR(spec ? 1 : 101);

  // ---- right-hand side −R = f − ½ J u − ½ L(μ)u as column N ----
  {
    double part[RT];
#pragma unroll
    for (int i = 0; i < RT; ++i) part[i] = 0.0;
#pragma unroll
    for (int jj = 0; jj < JJ; ++jj) {
      const int c0 = 8 * (J0 + warp + NW * jj) + 2 * t;
      const double u0 = c0 < N ? p.u[int64_t(b) * N + c0] : 0.0;
      const double u1 = c0 + 1 < N ? p.u[int64_t(b) * N + c0 + 1] : 0.0;
#pragma unroll
      for (int i = 0; i < RT; ++i) part[i] = fma(acc[jj][i][0], u0, fma(acc[jj][i][1], u1, part[i]));
    }
#pragma unroll
    for (int i = 0; i < RT; ++i) {
      part[i] += __shfl_xor_sync(0xffffffffu, part[i], 1);
      part[i] += __shfl_xor_sync(0xffffffffu, part[i], 2);
      if (t == 0) sh.rowred[warp][8 * i + g] = part[i];
    }
    __syncthreads();
    for (int r = tid; r < NR; r += NT) {
      double rhs = 0.0;
      if (r < N) {
        double ju = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) ju += sh.rowred[w][r];
        if constexpr (J0 == 1) {
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if (c < N) ju = fma(sh.panel[r * PS + c], p.u[int64_t(b) * N + c], ju);
        }
        rhs = newton_rhs(p, Jb, r, ju, sh.w);
      }
      sh.rhs[r] = rhs;
    }
    __syncthreads();
    const int jr = N / 8;
    if (jr >= J0 && warp == (jr - J0) % NW && t == (N % 8) / 2) {
#pragma unroll
      for (int jj = 0; jj < JJ; ++jj)
        if (J0 + warp + NW * jj == jr) {
#pragma unroll
          for (int i = 0; i < RT; ++i) {
            if (N & 1)
              acc[jj][i][1] = sh.rhs[8 * i + g];
            else
              acc[jj][i][0] = sh.rhs[8 * i + g];
          }
        }
    }
  }
  if (warp == 0) RBNS_TR(spec ? 2 : 102);

  // ---- blocked Gauss–Jordan.  Iteration P: the owner of tile P+1 applies panel P to it and factors panel
  // P+1 (the critical path); every other warp applies its pending panel (if any) and panel P to its tiles.
  const int NP = (N + 7) / 8;  // panels
  int pend = -1;               // panel not yet applied to this warp's tiles beyond the look-ahead one
  auto tiles_above = [&](int q) {
    unsigned m = 0;
#pragma unroll
    for (int jj = 0; jj < JJ; ++jj)
      if (J0 + warp + NW * jj > q && J0 + warp + NW * jj < CT) m |= 1u << jj;
    return m;
  };
#pragma unroll 1
  for (int P = -1; P < NP; ++P) {
    if (sh.sing || sh.fail) break;
    const int nxt = P + 1;
    const bool owner = nxt < NP && (nxt < J0 ? warp == 0 : warp == (nxt - J0) % NW);
    // The owner shares its SM sub-partition (warp id mod 4) with one partner warp when NW == 8; DMMAs and
    // FP64 FMAs share that sub-partition's datapath, so the partner finishes its DMMA updates first and the
    // factorization then runs without competing tensor-core traffic (pair barrier, 64 threads).
    const int o = nxt % NW;
    const bool partner = J0 == 0 && NW == 8 && nxt < NP && warp == (o + 4) % NW;
    if (owner) {
      const int jn = (nxt - J0) / NW;
      if (warp == 0) RBNS_TR(8 + 4 * nxt);
      if (nxt >= J0) {  // (J0 = 1: panel 0 is already in the panel buffer)
        if (P >= 0) bgj_update<RT, CT, NW, J0>(acc, 1u << jn, P % NB, P, spec, sh);
        if (warp == 0) RBNS_TR(160 + nxt);
        bgj_copy_panel<RT, CT, NW, J0>(acc, jn, sh);
      }
      if (J0 == 0 && NW == 8) asm volatile("bar.sync %0, 64;" ::"r"(1 + (o & 3)) : "memory");
      if (warp == 0) RBNS_TR(9 + 4 * nxt);
      if (spec)
        bgj_factor_spec<RT, CT, NW>(nxt, nxt % NB, N, sh);
      else
        bgj_factor_pivot<RT, CT, NW>(nxt, nxt % NB, N, sh);
      if (warp == 0) RBNS_TR(10 + 4 * nxt);
      if (P >= 0) pend = P;
    } else {
      if (pend >= 0) {
        bgj_update<RT, CT, NW, J0>(acc, tiles_above(pend + 1), pend % NB, pend, spec, sh);
        pend = -1;
      }
      if (P >= 0) bgj_update<RT, CT, NW, J0>(acc, tiles_above(P), P % NB, P, spec, sh);
      if (partner) asm volatile("bar.sync %0, 64;" ::"r"(1 + (o & 3)) : "memory");
    }
    __syncthreads();
    if (warp == 0) RBNS_TR(11 + 4 * nxt);
  }
  if (pend >= 0 && !sh.sing && !sh.fail)
    bgj_update<RT, CT, NW, J0>(acc, tiles_above(pend + 1), pend % NB, pend, spec, sh);
}

constexpr int kBgjPrefetchAhead = 296;

template <int RT, int CT, int NW, int J0 = 0>
__global__ void __launch_bounds__(NW * 32, (NW <= 4 ? 2 : 1)) newton_bgj_kernel(const NewtonParams p) {
  constexpr int JJ = (CT - J0 + NW - 1) / NW;
  constexpr int NT = NW * 32;
  extern __shared__ __align__(16) unsigned char bgj_smem[];  // dynamic: sizeof(BGJShared) can exceed 48 KB
  BGJShared<RT, CT, NW>& sh = *reinterpret_cast<BGJShared<RT, CT, NW>*>(bgj_smem);
  const int i_s = blockIdx.x;
  if (i_s >= p.n) return;
  const int b = p.act[i_s];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int N = p.N;

  newton_weights(p, b, sh.w);
  // the CTA that takes this slot about one wave of resident CTAs later finds its J in L2 (bulk prefetch; the
  // distance is not critical: 148..592 measured alike, Newton update 79.4 -> 77.5 ms per cfg-2 step)
  if (tid == 0 && i_s + kBgjPrefetchAhead < p.n)
    bulk_prefetch_l2(p.J + int64_t(i_s + kBgjPrefetchAhead) * p.ldj, uint32_t(p.ldj * 8));
  __syncthreads();
  double acc[JJ][RT][2];
  if (warp == 0) RBNS_TR(0);
  // speculative pass (partial pivoting without interchanges); on a rejected speculation, the full pivot search.
  // A sample whose previous Newton iteration already needed interchanges (non-identity hint) goes straight to
  // the search pass.
  bool identity = true;
  if (p.hint_in)
    for (int k = tid; k < N; k += NT) identity &= p.hint_in[int64_t(b) * N + k] == k;
  const int first_pass = __syncthreads_and(identity) ? 0 : 1;
#pragma unroll 1
  for (int pass = first_pass; pass < 2; ++pass) {
    bgj_pass<RT, CT, NW, J0>(p, i_s, b, pass == 0, acc, sh);
    __syncthreads();
    if (!sh.fail) break;
    if (tid == 0 && p.spec_miss) atomicAdd(p.spec_miss, 1);
    __syncthreads();
  }
  if (warp == 0) RBNS_TR(sh.fail ? 201 : 200);

  // ---- solution: x_k = rhs[perm[k]] / piv[k] ----
  const bool sing = sh.sing != 0;
  if (!sing) {
    const int jr = N / 8, NP = (N + 7) / 8;
    if (jr >= NP && jr >= J0 && warp == (jr - J0) % NW && t == (N % 8) / 2) {  // RHS in its own tile
#pragma unroll
      for (int jj = 0; jj < JJ; ++jj)
        if (J0 + warp + NW * jj == jr) {
#pragma unroll
          for (int i = 0; i < RT; ++i) sh.rhs[8 * i + g] = (N & 1) ? acc[jj][i][1] : acc[jj][i][0];
        }
    }
  }
  __syncthreads();
  double d2 = 0.0, un2 = 0.0, o2 = 0.0;  // o2: unknowns outside the stop norm
  if (!sing) {
    for (int k = tid; k < N; k += NT) {
      const double x = sh.rhs[sh.perm[k]] / sh.pivval[k];
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
      const double x = sh.rhs[sh.perm[k]] / sh.pivval[k];
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
  if (p.hint_out && !sing) {  // the order used: the next Newton iteration's hint
    for (int k = tid; k < N; k += NT) p.hint_out[int64_t(b) * N + k] = int16_t(sh.perm[k]);
  }
  if (warp == 0) RBNS_TR(202);
}

}  // namespace rbns
