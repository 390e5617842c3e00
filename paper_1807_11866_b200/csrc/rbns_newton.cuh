// rbns_newton.cuh — K3 shared pieces: the Newton-update parameter block, per-sample residual weights and
// right-hand side, pivot-row publication and CTA reductions used by the Newton kernels (tiled Gauss–Jordan,
// rbns_tgj.cuh; speculative / exact rank-1 register kernels, rbns_newton_spec.cuh / rbns_newton2.cuh; 2-CTA
// cluster kernel, rbns_newton_cluster.cuh).
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
  int64_t B;                   // samples of the call (sample ids < B; checked builds)
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

}  // namespace rbns
