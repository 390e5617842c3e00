// rbns_aux.cuh — setup and bookkeeping kernels: GEMM-operand construction, active-set compaction (K5),
// pressure recovery triangular solves (K4), reduced-operator readout.
#pragma once

#include "rbns_common.cuh"
#include "rbns_newton.cuh"

namespace rbns {

// S[r][κ] for the contraction GEMM (layout documented in rbns_contract.cuh).  One-time, at model create.
// hb/hg/rho: for each linear term a, the block and group of its h rows and its factor ρ_a
// (θ_a = ρ_a · μ₁^{e_g} · θ_block, resolved on the host by rbns_model_create2).
__global__ void build_velocity_operator(double* __restrict__ S, int64_t rows, int kalloc,
                                        const double* __restrict__ C, int Qc, const double* __restrict__ A, int Ql,
                                        const int* __restrict__ hb, const int* __restrict__ hg,
                                        const double* __restrict__ rho, int N, int Ne, int Qb, int jl) {
  const int64_t total = rows * kalloc;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = idx / kalloc;
    const int kap = int(idx - r * kalloc);
    double v = 0.0;
    const int64_t nn = int64_t(N) * N;
    if (r < nn) {
      int l, m;  // S row r carries J[l][m] at its position in the model's J layout
      jpos(r, N, jl, l, m);
      if (kap < Qc * Ne) {
        const int q = kap / Ne, k = kap - q * Ne;
        if (k < N) {
          const int64_t base = int64_t(q) * N * nn;
          v = C[base + (int64_t(m) * N + k) * N + l] + C[base + (int64_t(k) * N + m) * N + l];
        }
      } else if (kap >= Qb * Ne && kap < Qb * Ne + Ql) {
        const int a = kap - Qb * Ne;
        v = A[(int64_t(a) * N + l) * N + m];
      }
    } else if (r < rows) {
      const int g = int((r - nn) / N), l = int(r - nn - int64_t(g) * N);
      if (kap < Qb * Ne) {
        const int j = kap / Ne, k = kap - j * Ne;
        if (k < N)
          for (int a = 0; a < Ql; ++a)
            if (hb[a] == j && hg[a] == g) v = fma(rho[a], A[(int64_t(a) * N + l) * N + k], v);
      }
    }
    S[idx] = v;
  }
}

// Sp[i][κ] = B_q[i][k] for κ = q·Ne + k: the recovery right-hand side Σ_q θ_q B_q u is the same GEMM
// (coupling family: Q blocks, no affine columns).
__global__ void build_pressure_operator(double* __restrict__ S, int np, int kalloc, const double* __restrict__ Bq,
                                        int N, int Ne, int Q) {
  const int64_t total = int64_t(np) * kalloc;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(idx / kalloc);
    const int kap = int(idx - int64_t(i) * kalloc);
    double v = 0.0;
    if (kap < Q * Ne) {
      const int q = kap / Ne, k = kap - q * Ne;
      if (k < N) v = Bq[(int64_t(q) * np + i) * N + k];
    }
    S[idx] = v;
  }
}

// out[b][i] = y[b][i], i < cols (the leading columns of a tile-padded contraction output)
__global__ void copy_leading(const double* __restrict__ y, int64_t ldy, int32_t n, int32_t cols, double* __restrict__ out) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < int64_t(n) * cols; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = e / cols;
    out[e] = y[b * ldy + (e - b * cols)];
  }
}

__global__ void init_solve(int32_t* act, int8_t* status, int32_t* iters, double* last, int64_t B) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < B; i += int64_t(gridDim.x) * blockDim.x) {
    act[i] = int32_t(i);
    status[i] = int8_t(kStatusActive);
    iters[i] = 0;
    last[i] = __longlong_as_double(0x7ff8000000000000ULL);
  }
}

// θ weights of the contraction's columns, once per solve (they depend on μ only; SPEC.md:360-368
// evaluate_weights): W[b][q] = θ_q(μ_b) for the Qb blocks, W[b][Qb + a] = [ν_b] θ_a(μ_b) for the Ql affine
// columns — the same expressions the contraction prologue evaluates when no table is given.
__global__ void eval_weights(const double* __restrict__ mu, int64_t B, const rbns_theta_term* __restrict__ thb,
                             int Qb, const rbns_theta_term* __restrict__ thl, int Ql, int nu_lin,
                             double* __restrict__ W) {
  const int ld = Qb + Ql;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < B * ld; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = i / ld;
    const int q = int(i - b * ld);
    const double mu0 = mu[2 * b], mu1 = mu[2 * b + 1];
    if (q < Qb) {
      W[i] = eval_theta(thb[q], mu0, mu1);
    } else {
      const double nu = nu_lin ? 1.0 / mu1 : 1.0;
      W[i] = nu * eval_theta(thl[q - Qb], mu0, mu1);
    }
  }
}

// The Newton kernels' residual weights, once per solve: W[b] = [θ_f(μ_b) for the Qf load terms, μ₁^{ge[g]} for
// the G groups] — newton_weights' expressions.
struct LoadWeightParams {
  int32_t G;
  int32_t ge[RBNS_MAX_GROUPS];
};
__global__ void eval_load_weights(const double* __restrict__ mu, int64_t B, const rbns_theta_term* __restrict__ thf,
                                  int Qf, LoadWeightParams gp, double* __restrict__ W) {
  const int ld = Qf + gp.G;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < B * ld; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = i / ld;
    const int q = int(i - b * ld);
    const double mu0 = mu[2 * b], mu1 = mu[2 * b + 1];
    W[i] = q < Qf ? eval_theta(thf[q], mu0, mu1) : mu1_pow(mu1, gp.ge[q - Qf]);
  }
}

__global__ void finalize_solve(int8_t* status, int64_t B) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < B; i += int64_t(gridDim.x) * blockDim.x)
    if (status[i] == int8_t(kStatusActive)) status[i] = int8_t(RBNS_NON_CONVERGED);
}

// K5: stable compaction of the still-active samples (deterministic order).  One CTA of 1024 threads; each
// pass covers 16384 consecutive positions, warp w a contiguous 512-position segment (16 coalesced loads per
// lane, issued together), ballots give the in-warp order, one shuffle scan the warp offsets.
constexpr int kCompactThreads = 1024;
__global__ void __launch_bounds__(kCompactThreads) compact_active(const int32_t* __restrict__ act_in, int32_t n_in,
                                                                   const int8_t* __restrict__ status,
                                                                   int32_t* __restrict__ act_out,
                                                                   int32_t* __restrict__ count) {
  constexpr int PER = 16, SEG = 32 * PER, TILE = kCompactThreads * PER;
  __shared__ int32_t wtot[kCompactThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  int running = 0;  // same value in every thread
  for (int t0 = 0; t0 < n_in; t0 += TILE) {
    const int s0 = t0 + w * SEG;
    int32_t id[PER];
    unsigned m[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int i = s0 + j * 32 + lane;
      id[j] = i < n_in ? act_in[i] : -1;
    }
    int cnt = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      m[j] = __ballot_sync(0xffffffffu, id[j] >= 0 && status[id[j]] == int8_t(kStatusActive));
      cnt += __popc(m[j]);
    }
    if (lane == 0) wtot[w] = cnt;
    __syncthreads();
    int v = wtot[lane];  // inclusive scan of the 32 warp counts, in every warp
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    int pos = running + __shfl_sync(0xffffffffu, v, w) - cnt;
    running += __shfl_sync(0xffffffffu, v, 31);
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      if ((m[j] >> lane) & 1u) {
        RBNS_CHECK(pos + __popc(m[j] & lt) < n_in);
        act_out[pos + __popc(m[j] & lt)] = id[j];
      }
      pos += __popc(m[j]);
    }
    __syncthreads();  // wtot is rewritten by the next pass
  }
  if (tid == 0) *count = running;
}

// K4 (second half): p = L^{-T} L^{-1} r per sample, one warp per sample, M_p = L Lᵀ factored once.
// Lt is Lᵀ row-major (column j of L contiguous) for the forward sweep, L row-major for the backward sweep.
template <int CP>
__global__ void __launch_bounds__(256) pressure_trisolve(const double* __restrict__ rbuf, int64_t ldr, int32_t n,
                                                        const double* __restrict__ L, const double* __restrict__ Lt,
                                                        int np, int ok, double* __restrict__ p,
                                                        int8_t* __restrict__ status, const int32_t* __restrict__ ids) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n) return;
  const int id = ids ? ids[warp] : warp;
  double r[CP];
#pragma unroll
  for (int c = 0; c < CP; ++c) {
    const int i = lane + 32 * c;
    r[c] = i < np ? rbuf[int64_t(warp) * ldr + i] : 0.0;
  }
  if (!ok) {
#pragma unroll
    for (int c = 0; c < CP; ++c) {
      const int i = lane + 32 * c;
      if (i < np) p[int64_t(id) * np + i] = __longlong_as_double(0x7ff8000000000000ULL);
    }
    if (lane == 0 && status && status[id] == RBNS_CONVERGED) status[id] = RBNS_SINGULAR_RECOVERY;
    return;
  }
  // forward: L y = r (y overwrites r)
  for (int j = 0; j < np; ++j) {
    double rj = 0.0;
#pragma unroll
    for (int c = 0; c < CP; ++c)
      if (c == (j >> 5)) rj = r[c];
    rj = __shfl_sync(0xffffffffu, rj, j & 31);
    const double yj = rj / __ldg(&Lt[int64_t(j) * np + j]);
#pragma unroll
    for (int c = 0; c < CP; ++c) {
      const int i = lane + 32 * c;
      if (i == j) r[c] = yj;
      else if (i > j && i < np) r[c] = fma(-__ldg(&Lt[int64_t(j) * np + i]), yj, r[c]);
    }
  }
  // backward: Lᵀ x = y
  for (int j = np - 1; j >= 0; --j) {
    double rj = 0.0;
#pragma unroll
    for (int c = 0; c < CP; ++c)
      if (c == (j >> 5)) rj = r[c];
    rj = __shfl_sync(0xffffffffu, rj, j & 31);
    const double xj = rj / __ldg(&L[int64_t(j) * np + j]);
#pragma unroll
    for (int c = 0; c < CP; ++c) {
      const int i = lane + 32 * c;
      if (i == j) r[c] = xj;
      else if (i < j) r[c] = fma(-__ldg(&L[int64_t(j) * np + i]), xj, r[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < CP; ++c) {
    const int i = lane + 32 * c;
    if (i < np) p[int64_t(id) * np + i] = r[c];
  }
}

// reduced_operator readout: R = ½ J η + ½ L(μ)η − f(μ) (the Newton right-hand side, negated), J copied out
// (debug / FD path).  p carries the load family and the h groups exactly as for the Newton kernel.
__global__ void operator_readout(const double* __restrict__ Y, int64_t ldy, const double* __restrict__ eta,
                                 const NewtonParams p, double* __restrict__ R, double* __restrict__ Jout) {
  const int b = blockIdx.x;
  if (b >= p.n) return;
  __shared__ NewtonWeights w;
  newton_weights(p, b, w);
  __syncthreads();
  const int N = p.N;
  const double* Yb = Y + int64_t(b) * ldy;
  for (int64_t e = threadIdx.x; e < int64_t(N) * N; e += blockDim.x) {
    const int l = int(e / N), m = int(e - int64_t(l) * N);
    Jout[int64_t(b) * N * N + e] = Yb[jidx(l, m, N, p.jl)];
  }
  for (int l = threadIdx.x; l < N; l += blockDim.x) {
    double ju = 0.0;
    for (int m = 0; m < N; ++m) ju = fma(Yb[jidx(l, m, N, p.jl)], eta[int64_t(b) * N + m], ju);
    R[int64_t(b) * N + l] = -newton_rhs(p, Yb, l, ju, w);
  }
}

}  // namespace rbns
