// rbns_newton.cuh — K3: per-sample Newton update.  One CTA per μ sample; the N×N Jacobian (plus the
// right-hand side as column N) lives in REGISTERS, distributed 2-D cyclically over a TGR×TGC thread grid:
// thread (tr, tc) owns rows tr + TGR·r (r < RS) and columns tc + TGC·s (s < CS); threads are numbered
// column-major (tid = tc·TGR + tr) so the TGR owners of a column are adjacent lanes of ONE warp, which finds
// the pivot with a lane butterfly while the other warps wait at the barrier.  J δ = −R is solved by
// Gauss–Jordan elimination with partial pivoting (pivot = max |a| over unpivoted rows, ties to the smaller
// row index as LAPACK's idamax).  Per elimination step only the pivot column and the pivot row cross threads
// (shared memory, two CTA barriers); the update a[i][j] −= (a[i][k]/piv)·a[p][j] is register-resident DFMA.
// Column blocks left of the current TGC-wide block are dead and skipped statically.
//
// Shapes (rbns_newton.cu): N ≤ 52 runs one warp per sample (4×8 grid); N ≤ 104 runs four warps (8×16 grid,
// 91 register doubles per thread, two CTAs per SM); N ≤ 127 runs eight warps (16×16).
//
// Reference: dense LU with partial pivoting; Newton step and stop rule (SPEC.md:520-523,
// SPEC.md:557-559); residual R = L(μ)u + Σθ_c C_c(u,u) − f(μ) evaluated as ½ J u + ½ L(μ)u − f(μ)
// (Euler identity for the quadratic term; J and the L(μ)u groups come from the contraction GEMM, which at
// u = 0 runs only its affine block: "η = 0 → Jacobian = linear blocks only").
#pragma once

#include "rbns_common.cuh"

namespace rbns {

struct NewtonParams {
  const int32_t* act;          // sample ids of this chunk
  int32_t n;
  const double* J;             // [n][ldj]: rows 0..N²-1 Jacobian (row-major l,m), then G groups of N rows h_g
  int64_t ldj;
  double* u;                   // [B][N] in/out
  const double* mu;            // [B][2]
  const double* f;             // [Qf][N] load terms
  const rbns_theta_term* thf;  // [Qf] their descriptors (device)
  int32_t N, Qf;
  int32_t G;                   // L(μ)u = Σ_g μ₁^{ge[g]} h_g   (G = 1, ge = −1: ν A(μ)u of the BASELINE configs)
  int32_t ge[RBNS_MAX_GROUPS];
  int32_t n_stop;              // leading unknowns in the stop norm (N: all; the velocity block of coupled systems)
  int32_t stop_abs;            // 1: ‖δ‖ ≤ tol (SPEC.md:513 coupled rule), 0: ‖δ‖ ≤ tol·‖u_new‖ (block rule)
  int32_t iter, max_iter;
  double tol;
  int32_t* iters;
  int8_t* status;
  double* last;
  const int16_t* hint_in;      // [B][N] pivot order hint (previous Newton iteration); NULL = identity
  int16_t* hint_out;           // [B][N] pivot order chosen (may alias hint_in); NULL = not recorded
  int32_t* spec_miss;          // count of CTAs whose hint failed verification (statistics), or NULL
  int32_t* miss_list;          // speculative kernel: chunk positions whose hint failed (appended), or NULL
  int32_t* miss_count;         //   … and their number (device counter, zeroed per chunk)
  const int32_t* sub;          // exact kernels: run only the chunk positions sub[0 .. *n_sub) (NULL: all n)
  const int32_t* n_sub;
  int32_t prefer_rank1;        // host policy: pivoting seen, use the hinted rank-1 kernel over the blocked one
  const double* wf;            // [B][Qf + G] precomputed residual weights (eval_load_weights), or NULL
  int32_t jl;                  // layout of the J block (jidx, rbns_common.cuh): 0 row-major, 1 tile layout
  int32_t num_sms;             // SMs of the model's device (persistent / subset grids)
};

// CTA → chunk position (and whether this CTA has work) for the exact kernels' optional subset launch
__device__ __forceinline__ int newton_position(const NewtonParams& p) {
  if (p.sub) return int(blockIdx.x) < *p.n_sub ? p.sub[blockIdx.x] : -1;
  return int(blockIdx.x) < p.n ? int(blockIdx.x) : -1;
}

// Per-sample residual weights, evaluated once per CTA into shared memory.
struct NewtonWeights {
  double th[RBNS_MAX_TERMS];  // θ_f(μ) of the load terms
  double gf[RBNS_MAX_GROUPS]; // μ₁^{ge[g]}
};

__device__ __forceinline__ void newton_weights(const NewtonParams& p, int b, NewtonWeights& w) {
  if (p.wf) {  // precomputed once per solve (eval_load_weights): [θ_f(μ_b) …, μ₁^{ge[g]} …]
    const double* wb = p.wf + int64_t(b) * (p.Qf + p.G);
    for (int q = threadIdx.x; q < p.Qf; q += blockDim.x) w.th[q] = wb[q];
    if (threadIdx.x < p.G) w.gf[threadIdx.x] = wb[p.Qf + threadIdx.x];
    return;
  }
  const double mu0 = p.mu[2 * b], mu1 = p.mu[2 * b + 1];
  for (int q = threadIdx.x; q < p.Qf; q += blockDim.x) w.th[q] = eval_theta(p.thf[q], mu0, mu1);
  if (threadIdx.x < p.G) w.gf[threadIdx.x] = mu1_pow(mu1, p.ge[threadIdx.x]);
}

// Newton right-hand side entry i: −R_i = f(μ)_i − ½ (J u)_i − ½ (L(μ) u)_i  (Euler identity J_c u = 2 C(u,u);
// J and the h groups come from the contraction kernel).  ju = (J u)_i.
__device__ __forceinline__ double newton_rhs(const NewtonParams& p, const double* Jb, int i, double ju,
                                             const NewtonWeights& w) {
  const int N = p.N;
  double fi = 0.0;
#pragma unroll 4
  for (int q = 0; q < p.Qf; ++q) fi = fma(w.th[q], __ldg(&p.f[q * N + i]), fi);
  double h = 0.0;
  for (int g = 0; g < p.G; ++g) h = fma(w.gf[g], Jb[int64_t(N) * N + int64_t(g) * N + i], h);
  return fi - 0.5 * ju - 0.5 * h;
}

template <int TGR, int TGC, int RS, int CS>
struct GJShared {
  static constexpr int NW = (TGR * TGC + 31) / 32;
  static constexpr int CBS = RS | 1;  // odd stride: conflict-free column reads by 8 thread-rows
  NewtonWeights w;
  double pv;                          // current pivot value (signed), from the owner warp
  int pk;                             // current pivot row (-1: singular)
  double colbuf[2][TGR][CBS];         // pivot column, thread-row major
  double P[CS][TGC];                  // pivot row, [slot][thread-column]
  double piv[TGR * RS];
  int perm[TGR * RS];
  double rhs[TGR * RS];
  double rowred[NW][TGR * RS];        // per-warp partial row sums (J u)
  double red[2][NW];
};

// Pivot-row publication: thread-row tp copies its slot rp (runtime) into P; the recursion keeps register
// indices static.
// Pivot-row publication: the thread-row holding row slot rp stores a[rp][SB..CS) to P (stride STRIDE).  rp is
// a runtime value and a[][] lives in registers, so select the slot by a binary search over [LO, HI) (static
// register indices in every leaf, ⌈log2 RS⌉ branches).
template <int RS, int CS, int SB, int STRIDE, int LO = 0, int HI = RS>
__device__ __forceinline__ void publish_row(const double (&a)[RS][CS], int rp, double* P) {
  if constexpr (HI - LO == 1) {
#pragma unroll
    for (int s = SB; s < CS; ++s) P[s * STRIDE] = a[LO][s];
  } else {
    constexpr int MID = (LO + HI) / 2;
    if (rp < MID)
      publish_row<RS, CS, SB, STRIDE, LO, MID>(a, rp, P);
    else
      publish_row<RS, CS, SB, STRIDE, MID, HI>(a, rp, P);
  }
}

template <int TGR, int TGC, int RS, int CS, int SB>
__device__ __forceinline__ void gj_block(double (&a)[RS][CS], unsigned& pmask, bool& sing, const int N,
                                         const int tr, const int tc, GJShared<TGR, TGC, RS, CS>& sh) {
  if constexpr (SB < CS) {
    if (sing) return;
    const int lane = threadIdx.x & 31;
#pragma unroll 1
    for (int kk = 0; kk < TGC; ++kk) {
      const int k = SB * TGC + kk;
      if (k >= N) return;
      const int buf = k & 1;
      if (tc == kk) {
        // owner lanes of column k (TGR adjacent lanes of one warp): publish the column, then argmax of
        // |a| over unpivoted rows.  Keys are the IEEE bits of |a| (order-preserving for non-negative
        // doubles); ties go to the smaller row index.
        long long best = -1;
        double bsig = 0.0;
        int bi = -1;
#pragma unroll
        for (int r = 0; r < RS; ++r) {
          const double v = a[r][SB];
          sh.colbuf[buf][tr][r] = v;
          const long long key =
              (((pmask >> r) & 1u) || tr + TGR * r >= N) ? -1LL : __double_as_longlong(fabs(v));
          if (key > best) {
            best = key;
            bsig = v;
            bi = tr + TGR * r;
          }
        }
        const unsigned gmask = ((TGR >= 32) ? 0xffffffffu : ((1u << TGR) - 1u)) << ((kk * TGR) & 31);
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
        if (tr == 0) {
          const bool ok = best > 0 && best < 0x7ff0000000000000LL;  // nonzero, finite
          sh.pk = ok ? bi : -1;
          sh.pv = bsig;
        }
      }
      __syncthreads();
      const int p = sh.pk;
      if (p < 0) {  // uniform across the CTA
        sing = true;
        return;
      }
      const double piv = sh.pv;
      const int tp = p % TGR, rp = p / TGR;
      if (tr == tp) {
        publish_row<RS, CS, SB, TGC>(a, rp, &sh.P[0][tc]);
        pmask |= 1u << rp;
        if (tc == kk) sh.colbuf[buf][tp][rp] = 0.0;  // the pivot row itself is not updated
      }
      if (threadIdx.x == 0) {
        sh.perm[k] = p;
        sh.piv[k] = piv;
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
    gj_block<TGR, TGC, RS, CS, SB + 1>(a, pmask, sing, N, tr, tc, sh);
  }
}

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if constexpr (NT > 32) {
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) s += red[i];
    return s;
  } else {
    return v;
  }
}

template <int TGR, int TGC, int RS, int CS>
__global__ void __launch_bounds__(TGR * TGC, (TGR * TGC <= 128 ? 2 : 1))
    newton_gj_kernel(const NewtonParams p) {
  constexpr int NT = TGR * TGC;
  static_assert(RS <= 32 && TGR <= 32 && TGC <= 32 && NT % 32 == 0, "shape");
  __shared__ GJShared<TGR, TGC, RS, CS> sh;
  const int i_s = blockIdx.x;
  if (i_s >= p.n) return;
  const int b = p.act[i_s];
  const int tid = threadIdx.x, tc = tid / TGR, tr = tid % TGR;
  const int N = p.N;

  newton_weights(p, b, sh.w);
  __syncthreads();

  double a[RS][CS];
  const double* Jb = p.J + int64_t(i_s) * p.ldj;
#pragma unroll
  for (int r = 0; r < RS; ++r)
#pragma unroll
    for (int s = 0; s < CS; ++s) {
      const int i = tr + TGR * r, j = tc + TGC * s;
      a[r][s] = (i < N && j < N) ? __ldcs(&Jb[int64_t(i) * N + j]) : 0.0;
    }

  // right-hand side −R = f − ½ J u − ½ L(μ)u, stored as column N.  J u: per-thread partial row sums,
  // lane shuffles across the thread-columns inside a warp, then a fixed-order sum over warps.
  {
    constexpr int NW = GJShared<TGR, TGC, RS, CS>::NW;
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
    for (int i = tid; i < TGR * RS; i += NT) {
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

  unsigned pmask = 0;
  bool sing = false;
  gj_block<TGR, TGC, RS, CS, 0>(a, pmask, sing, N, tr, tc, sh);

  if (!sing && tc == N % TGC) {
#pragma unroll
    for (int r = 0; r < RS; ++r)
#pragma unroll
      for (int s = 0; s < CS; ++s)
        if (tc + TGC * s == N) sh.rhs[tr + TGR * r] = a[r][s];
  }
  __syncthreads();

  // δ_k = rhs[perm[k]] / piv[k];  ‖δ‖², ‖u + δ‖² (fixed-order block reduction: deterministic)
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

}  // namespace rbns
