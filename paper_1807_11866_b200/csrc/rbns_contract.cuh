// rbns_contract.cuh — K1+K2: θ-weighted affine assembly fused into the convective contraction, as one
// FP64 tensor-core (DMMA) GEMM over the μ batch.
//
//   Y[b][r] = Σ_κ X[b][κ] · S[r][κ]
//     rows r < N²        : r = l·N + m    -> J[l][m] = L(μ)[l][m] + Σ_c θ_c Σ_k S_c[m,k,l] u_k
//     rows N² + g·N + l  : group g of G   -> h_g[l], with L(μ)u = Σ_g μ₁^{e_g} h_g   (residual helper)
//     cols κ = j·Ne + k  : block j < Qb   X = θ_j(μ_b) · u_b[k]     S = S_j[m,k,l] = C_j[m,k,l] + C_j[k,m,l]
//                                                                   (h rows: ρ_a A_a[l][k] of the linear terms
//                                                                    tied to block j; extra blocks: h only)
//     cols κ = Qb·Ne + a : linear term a  X = [ν_b] θ_a(μ_b)       S = A_a[l][m]
// (PAPER.md:797-805 affine sums; PAPER.md:821-844 tensor + Fréchet chain.)  The BASELINE
// configs have one θ list for every family: Qb = Qa = Q, G = 1, e = −1 (h = A(μ)u times ν).
//
// Dataflow (one CTA = BM samples × a range of BN-row tiles):
//   * S (the μ-independent operand, 56 MB at N=100/Q=7) is streamed from L2 by TMA (cp.async.bulk.tensor,
//     evict_last policy) through an mbarrier ring fed by one producer warp; a stage is 8 κ = two boxes of
//     BN rows × 4 κ (32-byte rows: the B-fragment loads of a half-warp cover 128 contiguous bytes).
//   * X is never materialised.  The GEMM is regrouped per affine term,
//         Y[b][r] = Σ_q θ_q(μ_b) · ( Σ_k u_b[k] S_q[r][k] )  +  Σ_q ν_b θ_q(μ_b) A_q[r],
//     so the A fragments are plain u values (resident smem tile, loaded once per CTA) and θ_q is applied
//     once per term to a partial accumulator (32 DFMA per thread per term) — no per-fragment scaling on the
//     FP64 pipe the DMMAs share.
//   * 8 consumer warps each own a 32-sample × 32-row tile (4×4 DMMA.8x8x4 fragments, two accumulator sets).
#pragma once

#include <cuda.h>

#include "rbns_common.cuh"

namespace rbns {

struct ContractParams {
  const int32_t* act;     // sample ids of this chunk (length n); NULL = identity
  int32_t n;              // samples in this chunk
  const double* u;        // [B][N] states, indexed by sample id
  const double* mu;       // [B][2]
  int32_t N, Ne;          // Ne = κ stride per block (N rounded up to a multiple of 4)
  int32_t Qb, Ql;         // contraction blocks (θ ⊗ u) and affine columns
  int32_t nu_lin;         // affine columns carry ν = 1/μ₁
  const rbns_theta_term* thb;  // [Qb] block descriptors (device)
  const rbns_theta_term* thl;  // [Ql] affine-column descriptors (device)
  int32_t nchunks;        // TMA stages per row tile (4·kKSub κ each)
  int32_t nsub;           // k4 sub-steps per row tile (= K / 4)
  int32_t sub_begin;      // first k4 sub-step (Qb·Ne/4 at u = 0: only the affine block is non-zero)
  int32_t row_tiles;      // ceil(R / BN)
  int32_t tiles_per_group;
  int32_t ldu_s;          // shared-memory row stride of the u tile (≡ 8 mod 16)
  int32_t stages;
  double* out;            // [n][ldo]
  int64_t ldo;
  const double* wts;      // [B][Qb + Ql] precomputed weights (eval_weights), indexed by sample id; NULL = evaluate
  int64_t B;              // samples of the call (sample ids < B; checked builds), 0 = n
};

#ifndef RBNS_BN
#define RBNS_BN 128
#endif
#ifndef RBNS_WN
#define RBNS_WN 4
#endif
#ifndef RBNS_WM
#define RBNS_WM 2
#endif
#ifndef RBNS_KSUB
#define RBNS_KSUB 2  // 4-κ k-steps per TMA stage (one full/empty mbarrier round trip per stage)
#endif
constexpr int kBM = 64, kBN = RBNS_BN, kWM = RBNS_WM, kWN = RBNS_WN, kKSub = RBNS_KSUB;
constexpr int kContractThreads = (kWM * kWN + 1) * 32;

// u-tile row stride ≡ 4 (mod 16) doubles: the 4 rows a half-warp touches land in distinct 32-byte bank groups
__host__ __device__ inline int contract_ldu(int ne) { return ne + ((4 - ne % 16) + 16) % 16; }

__host__ inline size_t contract_smem_bytes(int stages, int ldu, int qb, int ql) {
  return size_t(stages) * kKSub * kBN * 4 * sizeof(double) + size_t(kBM) * ldu * sizeof(double) +
         size_t(qb + ql) * kBM * sizeof(double) + 2 * size_t(stages) * sizeof(uint64_t);
}

// θ is applied once per term to a second accumulator set (168 registers, one CTA per SM).  Measured and not
// kept: θ applied to the A fragments (one accumulator set, fewer registers) with a co-resident Newton-update
// CTA on a second stream ran 273 vs 217 ms per config-2 step (the DMMAs and the Newton FP64 work share the FP64
// datapath), so the library runs one kernel at a time.
template <int BM, int BN, int WM, int WN, int MINB = 1>
__global__ void __launch_bounds__((WM * WN + 1) * 32, MINB)
    contract_kernel(const __grid_constant__ CUtensorMap tmap, const ContractParams p) {
  constexpr int NCW = WM * WN;
  constexpr int TM = BM / WM, TN = BN / WN;
  constexpr int MI = TM / 8, NI = TN / 8;
  constexpr int STAGE = kKSub * BN * 4;  // doubles per stage: kKSub [BN][4] boxes
  static_assert(TM % 8 == 0 && TN % 8 == 0, "warp tile must be a multiple of 8x8");

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  double* Sst = reinterpret_cast<double*>(smem_raw);
  double* Us = Sst + size_t(p.stages) * STAGE;
  double* thS = Us + size_t(BM) * p.ldu_s;
  double* thnuS = thS + p.Qb * BM;
  uint64_t* full = reinterpret_cast<uint64_t*>(thnuS + p.Ql * BM);
  uint64_t* empty = full + p.stages;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile0 = blockIdx.x * BM;
  const int rt_begin = blockIdx.y * p.tiles_per_group;
  const int rt_end = min(p.row_tiles, rt_begin + p.tiles_per_group);
  if (rt_begin >= rt_end) return;  // whole CTA, before any barrier

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_barrier_init();
  }
  if (warp == NCW && lane == 0) prefetch_tmap(&tmap);

  // resident u tile (zero-padded in k and beyond the chunk) and the block / affine weights of the tile's samples
  for (int idx = threadIdx.x; idx < BM * p.ldu_s; idx += blockDim.x) {
    const int b = idx / p.ldu_s, k = idx - b * p.ldu_s;
    const int i = tile0 + b;
    double v = 0.0;
    if (i < p.n && k < p.N && p.sub_begin == 0) v = p.u[int64_t(p.act ? p.act[i] : i) * p.N + k];
    Us[idx] = v;
  }
  for (int b = threadIdx.x; b < BM; b += blockDim.x) {
    const int i = tile0 + b;
    if (i < p.n) {
      const int id = p.act ? p.act[i] : i;
      RBNS_CHECK(id >= 0 && id < (p.B > 0 ? p.B : p.n));
      if (p.wts) {
        const double* w = p.wts + int64_t(id) * (p.Qb + p.Ql);
        for (int q = 0; q < p.Qb; ++q) thS[q * BM + b] = w[q];
        for (int q = 0; q < p.Ql; ++q) thnuS[q * BM + b] = w[p.Qb + q];
      } else {
        const double mu0 = p.mu ? p.mu[2 * id] : 0.0, mu1 = p.mu ? p.mu[2 * id + 1] : 1.0;  // NULL: μ-free operand
        const double nu = p.nu_lin ? 1.0 / mu1 : 1.0;
        for (int q = 0; q < p.Qb; ++q) thS[q * BM + b] = eval_theta(p.thb[q], mu0, mu1);
        for (int q = 0; q < p.Ql; ++q) thnuS[q * BM + b] = nu * eval_theta(p.thl[q], mu0, mu1);
      }
    } else {
      for (int q = 0; q < p.Qb; ++q) thS[q * BM + b] = 0.0;
      for (int q = 0; q < p.Ql; ++q) thnuS[q * BM + b] = 0.0;
    }
  }
  __syncthreads();

  if (warp == NCW) {
    // ---------------- TMA producer (one elected lane) ----------------
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int rt = rt_begin; rt < rt_end; ++rt) {
        for (int c = p.sub_begin / kKSub; c < p.nchunks; ++c) {
          // the producer lane sleeps between probes: spinning took issue slots from the consumer warps on its
          // SM sub-partition (contraction 126.0 → 124.7 ms per cfg-2 step; 32–256 ns measured alike)
          mbar_wait_backoff(&empty[stage], phase ^ 1u);
          mbar_arrive_expect_tx(&full[stage], STAGE * sizeof(double));
          double* dst = Sst + size_t(stage) * STAGE;
#pragma unroll
          for (int j = 0; j < kKSub; ++j)
            tma_load_2d(dst + j * BN * 4, &tmap, &full[stage], (c * kKSub + j) * 4, rt * BN, pol);
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
    return;
  }

  // ---------------- DMMA consumers ----------------
  const int wm = warp / WN, wn = warp % WN;
  const int g = lane >> 2, t = lane & 3;
  const int sb0 = wm * TM, rb0 = wn * TN;
  const int kterms = p.Qb * p.Ne;  // κ where the affine (linear) columns start
  int stage = 0;
  uint32_t phase = 0;

  for (int rt = rt_begin; rt < rt_end; ++rt) {
    double acc[MI][NI][2];
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
    double accq[MI][NI][2];
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) accq[mi][ni][0] = accq[mi][ni][1] = 0.0;

    int q = 0, k0 = 0;  // current term and k offset of the sub-step (uniform over the warp)
    for (int c = p.sub_begin / kKSub; c < p.nchunks; ++c) {
      mbar_wait(&full[stage], phase);  // (a sleeping consumer wait measured slower: 126.0 vs 124.7 ms)
      const double* st = Sst + size_t(stage) * STAGE;
#pragma unroll
      for (int j = 0; j < kKSub; ++j) {
        const int kap = 4 * kKSub * c + 4 * j;
        if (kap >= 4 * p.nsub) break;
        if (kap < 4 * p.sub_begin) continue;
        double af[MI], bf[NI];
        if (kap < kterms) {
#pragma unroll
          for (int mi = 0; mi < MI; ++mi) af[mi] = Us[(sb0 + mi * 8 + g) * p.ldu_s + k0 + t];
        } else {
          const int lin = kap - kterms + t;
#pragma unroll
          for (int mi = 0; mi < MI; ++mi) af[mi] = lin < p.Ql ? thnuS[lin * BM + sb0 + mi * 8 + g] : 0.0;
        }
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) bf[ni] = st[(j * BN + rb0 + ni * 8 + g) * 4 + t];
        if (kap < kterms) {
#pragma unroll
          for (int mi = 0; mi < MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) dmma_8x8x4(accq[mi][ni][0], accq[mi][ni][1], af[mi], bf[ni]);
          k0 += 4;
          if (k0 == p.Ne) {  // end of term q: acc += θ_q ∘ accq
#pragma unroll
            for (int mi = 0; mi < MI; ++mi) {
              const double th = thS[q * BM + sb0 + mi * 8 + g];
#pragma unroll
              for (int ni = 0; ni < NI; ++ni) {
                acc[mi][ni][0] = fma(th, accq[mi][ni][0], acc[mi][ni][0]);
                acc[mi][ni][1] = fma(th, accq[mi][ni][1], acc[mi][ni][1]);
                accq[mi][ni][0] = accq[mi][ni][1] = 0.0;
              }
            }
            k0 = 0;
            ++q;
          }
        } else {
#pragma unroll
          for (int mi = 0; mi < MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
        }
      }
      // release the stage once its fragments were consumed by the issued MMAs (register dependency)
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == p.stages) {
        stage = 0;
        phase ^= 1u;
      }
    }
    // epilogue: fragment (sample g, rows 2t..2t+1) -> out[sample][row] as 16-byte stores
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
      const int i = tile0 + sb0 + mi * 8 + g;
      if (i < p.n) {
        double* o = p.out + int64_t(i) * p.ldo + int64_t(rt) * BN + rb0 + 2 * t;
        RBNS_CHECK(int64_t(rt) * BN + rb0 + 2 * t + (NI - 1) * 8 + 1 < p.ldo);
#pragma unroll
        for (int ni = 0; ni < NI; ++ni)
          *reinterpret_cast<double2*>(o + ni * 8) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
      }
    }
  }
}

}  // namespace rbns
