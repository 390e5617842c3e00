// rbns_tgj.cuh — K3 (default where a shape is instantiated): tiled Gauss–Jordan Newton update with block
// pivots, FP64 tensor cores (DMMA.8x8x4) for every elimination, persistent CTAs fed by the TMA engine.
//
// Per μ sample the augmented system [J | −R] (N × (N+1)) is eliminated by blocked Gauss–Jordan over 8-column
// panels P.  Panel P's pivot block is its diagonal 8×8 tile J_PP; with W = J_PP⁻¹ every other column tile j
// is updated as
//         X_Pj = W J_Pj ,   J_ij ← J_ij − J_iP X_Pj  (i ≠ P),   J_Pj ← X_Pj
// which is exactly scalar Gauss–Jordan over the panel's 8 columns, regrouped (no per-row multipliers: the
// panel column itself is the left operand).  At the end the right-hand-side column holds δ = J⁻¹(−R).
//
// Layout.  The matrix lives in REGISTERS as transposed tiles: warp w owns column tiles j ≡ 1 + w (mod NW),
// and for each row tile i lane (g = lane/4, t = lane%4) holds J[8i+2t][8j+g], J[8i+2t+1][8j+g] — the DMMA
// accumulator fragment of (J_ij)ᵀ.  With the k index of each 8×8×8 product split as κ = 2t+s over the two
// m8n8k4 steps s, both products above take their operands straight from fragments already in place:
//     X_Pjᵀ = (J_Pj)ᵀ · Wᵀ          A = own fragment of tile (P, j), B = row g of W (shared memory)
//     (J_ij)ᵀ += X_Pjᵀ · M_iᵀ        A = the X fragment just computed, B = row g of M_i = −J_iP (shared)
// so no transposes or shuffles touch the bulk of the work.  Column tile 0 is never held in registers (it is
// only panel 0), which balances 12 tiles 3 per warp at N ≤ 103: 156 registers of matrix per thread, two CTAs
// (two samples) per SM.
//
// Panel chain.  The owner of tile P+1 applies panel P to that tile first, inverts its new diagonal tile
// (tgj_invert: 8 scalar Gauss–Jordan steps on one warp, ~100 cycles each) and publishes M_{P+1} (negated
// pivot column, transposed into shared memory) and W_{P+1} (double-buffered); every warp then applies panel P
// to its other live tiles; one CTA barrier per panel.
//
// Pivoting.  Partial pivoting keeps the natural row order for these systems (rbns_newton_spec.cuh), so the
// kernel eliminates without interchanges and VERIFIES that choice: inside the pivot tile at every step
// (|a_rc| ≤ |a_cc| for r > c), and for the rows below it through the panel's LU multipliers
// L_iP = J_iP U_PP⁻¹ (U_PP⁻¹ = W L_PP; two DMMAs per row tile, off the critical path): |l| ≤ 1 everywhere is
// exactly "idamax picks the diagonal" (ties go to the smaller row, as LAPACK).  A sample that fails — or has
// a zero / non-finite pivot, or needed interchanges at its previous Newton iteration — is appended to a miss
// list and solved by the exact full-search kernel (rbns_newton2.cuh) from its untouched J, so every result
// is that of partial pivoting.
//
// Data movement.  The contraction writes J in the tile layout (jidx_tile, rbns_common.cuh), so a sample's
// block is one contiguous 80 KB range: each CTA loops over samples and copies the NEXT sample's block into a
// shared-memory staging buffer with cp.async.bulk (TMA engine, mbarrier completion) while it eliminates the
// current one from registers; the register load is then one conflict-free 16-byte LDS per tile.
//
// Reference: dense LU with partial pivoting for the Newton systems, Newton step and stop rule
// (SPEC.md:520-523, :557-559); the residual −R = f − ½Ju − ½L(μ)u as in rbns_newton.cuh.
#pragma once

#include "rbns_common.cuh"
#include "rbns_newton.cuh"

namespace rbns {

// Shared-memory slot of entry (r, c) of an 8×8 tile.  Writers store transposed fragments (lane (g,t) writes
// rows 2t+s, column g: 8-byte stores) and readers load rows (lane (g,t) reads row g, columns 2t..2t+1: one
// 16-byte load); this row permutation + column XOR makes both patterns bank-conflict free.
__host__ __device__ constexpr int tgj_slot(int r, int c) {
  return ((r ^ ((r >> 1) & 1)) << 3) + (c ^ (((r >> 2) & 1) << 2));
}


#ifdef RBNS_TRACE  // clock64 trace of sample 0 (tools/trace_tgj.py)
#define TGJ_TR(slot)                                                   \
  do {                                                                 \
    if (i_s == 2960 && (threadIdx.x & 31) == 0) g_trace[(slot) & 255] = clock64(); /* a steady-state sample */ \
  } while (0)
#else
#define TGJ_TR(slot) \
  do {               \
  } while (0)
#endif

constexpr int kTgjSlots = 3;  // panel buffers in flight (published → consumed by every warp)

template <int RT, int NW>
struct TGJShared {
  static constexpr int NR = 8 * RT;
  static constexpr int NB = kTgjSlots;
  alignas(16) double M[NB][RT][64];  // panel P: M_i = −J_iP over the pivot columns, M_P = 0 (tgj_slot layout)
  alignas(16) double W[NB][64];      // W_P = J_PP⁻¹
  alignas(16) double L[NB][64];      // unit lower LU factor of J_PP (verification)
  alignas(16) double Wall[RT][64];   // every panel's W: final scaling of the (unscaled) pivot rows; the
                                     // prologue's per-warp row sums of J u alias it
  double rhs[NR];                    // right-hand side, then the unscaled solution column
  double red[2][NW];
  uint64_t full[NB], empty[NB];      // panel slot: every M_i published (one arrival) / consumed (one per warp)
  uint64_t bar;                      // staging buffer: the next sample's J block has landed
  int fail;                          // current sample: rejected speculation or unusable pivot
};

template <int RT, int NW>
__host__ __device__ constexpr size_t tgj_stage_offset() {
  return (sizeof(TGJShared<RT, NW>) + 127) & ~size_t(127);
}

// Pivot-tile factorization of one panel, in registers of one warp.
struct TgjPivot {
  double w0, w1;  // W = A⁻¹: W[2t][g], W[2t+1][g]
  double l0, l1;  // unit lower LU factor of A: L[2t][g], L[2t+1][g]
  bool bad;       // warp-uniform: interchange inside the tile, or a zero / denormal / non-finite pivot
};

// Inverse of a panel's 8×8 pivot tile A by Gauss–Jordan without interchanges, in the fragment layout
// (lane (g,t): a0 = A[2t][g], a1 = A[2t+1][g]).  Rows / columns ≥ nc (the last panel) are the identity.
// Partial pivoting would keep the diagonal iff |a_rc| ≤ |a_cc| for every r > c at step c (ties: smaller row).
template <bool FULL = false>  // FULL: nc == 8 known at compile time (straight-line code, no early exit)
__device__ __forceinline__ TgjPivot tgj_invert(double a0, double a1, int nc) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int r0 = 2 * t, r1 = r0 + 1;
  if (r0 >= nc || g >= nc) a0 = r0 == g ? 1.0 : 0.0;
  if (r1 >= nc || g >= nc) a1 = r1 == g ? 1.0 : 0.0;
  double e0 = r0 == g ? 1.0 : 0.0, e1 = r1 == g ? 1.0 : 0.0;
  double l0 = e0, l1 = e1;  // column g of L: recorded at step c = g (identity for padded columns)
  bool bad = false;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    if (!FULL && c >= nc) break;  // uniform
    const double ma0 = __shfl_sync(0xffffffffu, a0, 4 * c + t);                        // A[r0][c]
    const double ma1 = __shfl_sync(0xffffffffu, a1, 4 * c + t);                        // A[r1][c]
    const double pr = __shfl_sync(0xffffffffu, (c & 1) ? a1 : a0, 4 * g + (c >> 1));   // A[c][g]
    const double er = __shfl_sync(0xffffffffu, (c & 1) ? e1 : e0, 4 * g + (c >> 1));   // E[c][g]
    const double piv = __shfl_sync(0xffffffffu, (c & 1) ? a1 : a0, 4 * c + (c >> 1));  // A[c][c]
    const double ap = fabs(piv);
    bad |= !(ap >= 2.2250738585072014e-308 && ap <= 1.7976931348623157e308);
    bad |= (r0 > c && fabs(ma0) > ap) || (r1 > c && fabs(ma1) > ap);
    const double rp = rcp_cubic(piv);  // 3 dependent DFMAs after MUFU (rcp_nr: 4): 37.0 → 36.3 ms per cfg-2 step
    const double m0 = ma0 * rp, m1 = ma1 * rp;
    if (g == c) {
      if (r0 > c) l0 = m0;
      if (r1 > c) l1 = m1;
    }
    a0 = r0 == c ? pr * rp : fma(-m0, pr, a0);
    e0 = r0 == c ? er * rp : fma(-m0, er, e0);
    a1 = r1 == c ? pr * rp : fma(-m1, pr, a1);
    e1 = r1 == c ? er * rp : fma(-m1, er, e1);
  }
  return TgjPivot{e0, e1, l0, l1, __any_sync(0xffffffffu, bad) != 0};
}

// Row tile P of a register column tile: a branch-free select tree on the bits of P (CTA-uniform), static
// register indices, ⌈log2 RT⌉ levels of independent selects.
template <int RT>
__device__ __forceinline__ void tgj_pick(const double (&a)[RT][2], int P, double& p0, double& p1) {
  constexpr int NP2 = RT <= 2 ? 2 : RT <= 4 ? 4 : RT <= 8 ? 8 : 16;
  double v0[NP2], v1[NP2];
#pragma unroll
  for (int i = 0; i < NP2; ++i) {
    v0[i] = a[i < RT ? i : RT - 1][0];
    v1[i] = a[i < RT ? i : RT - 1][1];
  }
#pragma unroll
  for (int w = NP2 / 2, bit = 0; w >= 1; w >>= 1, ++bit) {
    const bool hi = (P >> bit) & 1;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      v0[i] = hi ? v0[2 * i + 1] : v0[2 * i];
      v1[i] = hi ? v1[2 * i + 1] : v1[2 * i];
    }
  }
  p0 = v0[0];
  p1 = v1[0];
}

// X_Pjᵀ = (J_Pj)ᵀ Wᵀ for one register column tile (W fragment wv = row g of W_P): the panel's scaled pivot
// row tile, k-permuted C fragment (k-step s of the next product uses element s).
template <int RT>
__device__ __forceinline__ void tgj_x(const double (&a)[RT][2], int P, const double2 wv, double& x0, double& x1) {
  double p0, p1;
  tgj_pick<RT>(a, P, p0, p1);
  x0 = x1 = 0.0;
  dmma_8x8x4(x0, x1, p0, wv.x);
  dmma_8x8x4(x0, x1, p1, wv.y);
}

// (J_ij)ᵀ += X M_iᵀ for every row tile i (unscaled Gauss–Jordan: M_P = 0 leaves the pivot row tile as it is).
template <int RT>
__device__ __forceinline__ void tgj_update(double (&a)[RT][2], double x0, double x1, const double (*M)[64]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int i = 0; i < RT; ++i) {
    const double2 m = *reinterpret_cast<const double2*>(&M[i][tgj_slot(g, 2 * t)]);
    dmma_8x8x4(a[i][0], a[i][1], x0, m.x);
    dmma_8x8x4(a[i][0], a[i][1], x1, m.y);
  }
}

// Panel P (W fragment wv, pivot column M) applied to one register column tile.
template <int RT>
__device__ __forceinline__ void tgj_apply(double (&a)[RT][2], int P, const double2 wv, const double (*M)[64]) {
  double x0, x1;
  tgj_x<RT>(a, P, wv, x0, x1);
  tgj_update<RT>(a, x0, x1, M);
}

// (row tile i of a) + X M_iᵀ into (q0, q1), a left unchanged
template <int RT>
__device__ __forceinline__ void tgj_row(const double (&a)[RT][2], int i, double x0, double x1, const double* Mi,
                                        double& q0, double& q1) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  tgj_pick<RT>(a, i, q0, q1);
  const double2 m = *reinterpret_cast<const double2*>(&Mi[tgj_slot(g, 2 * t)]);
  dmma_8x8x4(q0, q1, x0, m.x);
  dmma_8x8x4(q0, q1, x1, m.y);
}

// Verification of panel P for this warp's share of the rows below its pivot tile (row tiles i > P,
// i ≡ warp mod NW): L_iP = J_iP U⁻¹ = −M_i (W L), |l| ≤ 1.  Returns warp-uniform "rejected".
template <int NW>
__device__ __forceinline__ bool tgj_verify(int P, int NP, int N, const double2 wv, const double* Ls,
                                           const double (*M)[64]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int i0 = P + 1 + ((warp - (P + 1) % NW) + NW) % NW;
  if (i0 >= NP) return false;
  double ui0 = 0.0, ui1 = 0.0;  // U⁻ᵀ = Lᵀ Wᵀ: lane (g,t) gets U⁻¹[2t+s][g]
  dmma_8x8x4(ui0, ui1, Ls[tgj_slot(2 * t, g)], wv.x);
  dmma_8x8x4(ui0, ui1, Ls[tgj_slot(2 * t + 1, g)], wv.y);
  bool bad = false;
  constexpr int MAXI = (16 + NW - 1) / NW;
#pragma unroll
  for (int k = 0; k < MAXI; ++k) {
    const int i = i0 + k * NW;
    if (i < NP) {
      const double2 m = *reinterpret_cast<const double2*>(&M[i][tgj_slot(g, 2 * t)]);
      double l0 = 0.0, l1 = 0.0;
      dmma_8x8x4(l0, l1, m.x, ui0);
      dmma_8x8x4(l0, l1, m.y, ui1);
      bad |= 8 * i + g < N && (fabs(l0) > 1.0 || fabs(l1) > 1.0);
    }
  }
  return __any_sync(0xffffffffu, bad) != 0;
}

// load part of the residual, f(μ)_r, and the h-group weights μ₁^{e_g} (independent of J: evaluated while the
// sample's J block is still in flight); weights from the per-solve table (eval_load_weights) or evaluated here
__device__ __forceinline__ double tgj_load_term(const NewtonParams& p, int b, int r) {
  const double* wb = p.wf ? p.wf + int64_t(b) * (p.Qf + p.G) : nullptr;
  const double mu0 = p.mu[2 * b], mu1 = p.mu[2 * b + 1];
  double fi = 0.0;
#pragma unroll 4
  for (int q = 0; q < p.Qf; ++q)
    fi = fma(wb ? wb[q] : eval_theta(p.thf[q], mu0, mu1), __ldg(&p.f[q * p.N + r]), fi);
  return fi;
}

// resident CTAs per SM: two samples at N ≤ 103 (the register file holds two systems), four for small systems
template <int RT>
constexpr int tgj_min_blocks(int nw = 4) { return RT <= 8 ? (nw <= 3 ? 5 : 4) : 2; }

template <int RT, int CT, int NW>
__global__ void __launch_bounds__(NW * 32, tgj_min_blocks<RT>(NW)) newton_tgj_kernel(const NewtonParams p) {
  constexpr int JJ = (CT - 1 + NW - 1) / NW;  // register column tiles per warp (tile 0 stays in shared memory)
  constexpr int NT = NW * 32;
  constexpr int NR = 8 * RT;
  constexpr int NB = kTgjSlots;
  static_assert(RT <= 16 && CT >= 2 && CT <= RT + 1 && NW >= 3, "shape");
  using SH = TGJShared<RT, NW>;
  extern __shared__ __align__(128) unsigned char tgj_smem[];
  SH& sh = *reinterpret_cast<SH*>(tgj_smem);
  double* jst = reinterpret_cast<double*>(tgj_smem + tgj_stage_offset<RT, NW>());
  double (*rowred)[NR] = reinterpret_cast<double (*)[NR]>(&sh.Wall[0][0]);
  static_assert(NW * NR <= RT * 64, "row sums alias Wall");
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int N = p.N;
  const int NP = RT;                  // panels
  const int ncl = N - 8 * (NP - 1);   // pivot columns of the last panel
  const int jr = N >> 3, gr = N & 7;  // right-hand-side column: tile, column inside the tile
  const uint32_t jbytes = uint32_t(((int64_t(N) * N + int64_t(p.G) * N) * 8 + 15) & ~int64_t(15));
  if (tid == 0) {
    mbar_init(&sh.bar, 1);
    for (int s = 0; s < NB; ++s) {
      mbar_init(&sh.full[s], 1);
      mbar_init(&sh.empty[s], NW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  RBNS_CHECK(int64_t(jbytes) <= p.ldj * 8);  // the staging buffer holds ldj doubles
  auto issue = [&](int is) {  // thread 0: stage sample is's J block
    const uint64_t pol = l2_policy_evict_first();
    mbar_arrive_expect_tx(&sh.bar, jbytes);
    const char* src = reinterpret_cast<const char*>(p.J + int64_t(is) * p.ldj);
    for (uint32_t off = 0; off < jbytes; off += 32768u) {
      const uint32_t nb = jbytes - off < 32768u ? jbytes - off : 32768u;
      bulk_g2s(reinterpret_cast<char*>(jst) + off, src + off, nb, &sh.bar, pol);
    }
  };
  if (tid == 0 && int(blockIdx.x) < p.n) issue(blockIdx.x);
  uint32_t phase = 0;
  int pc0 = 0;  // panels published by this CTA so far (slot / parity bookkeeping)

#pragma unroll 1
  for (int i_s = blockIdx.x; i_s < p.n; i_s += gridDim.x) {
    const int b = p.act[i_s];
    RBNS_CHECK(i_s >= 0 && i_s < p.n && b >= 0 && (p.B == 0 || b < p.B));
    const int nxt_s = i_s + int(gridDim.x);
    // J-independent work first, while the block may still be in flight: pivot-order hint, f(μ), weights, u
    bool ident = true;
    if (p.hint_in)
      for (int k = tid; k < N; k += NT) ident &= p.hint_in[int64_t(b) * N + k] == k;
    static_assert(NR <= NT, "one row per thread");
    const double fr = tid < N ? tgj_load_term(p, b, tid) : 0.0;
    double hw[RBNS_MAX_GROUPS];
#pragma unroll
    for (int gg = 0; gg < RBNS_MAX_GROUPS; ++gg)
      hw[gg] = gg < p.G ? (p.wf ? p.wf[int64_t(b) * (p.Qf + p.G) + p.Qf + gg] : mu1_pow(p.mu[2 * b + 1], p.ge[gg]))
                        : 0.0;
    double u0[8];  // column tile 0 of u (every thread)
#pragma unroll
    for (int c = 0; c < 8; ++c) u0[c] = p.u[int64_t(b) * N + c];
    double uj[JJ];  // this lane's columns of u in its owned tiles
#pragma unroll
    for (int jj = 0; jj < JJ; ++jj) {
      const int col = 8 * (1 + warp + NW * jj) + g;
      uj[jj] = col < N ? p.u[int64_t(b) * N + col] : 0.0;
    }
    if (tid == 0) sh.fail = 0;
    TGJ_TR(0);
    mbar_wait(&sh.bar, phase);
    phase ^= 1u;
    TGJ_TR(1);
    if (!__syncthreads_and(ident)) {  // interchanges at the previous iteration: the exact kernel takes it
      if (tid == 0) {
        p.miss_list[atomicAdd(p.miss_count, 1)] = i_s;
        if (p.spec_miss) atomicAdd(p.spec_miss, 1);
        if (nxt_s < p.n) {
          fence_proxy_async_smem();
          issue(nxt_s);
        }
      }
      continue;
    }

    TGJ_TR(9);
    // ---- owned column tiles j = 1 + warp + NW·jj from the staging buffer ----
    double acc[JJ][RT][2];
#pragma unroll
    for (int jj = 0; jj < JJ; ++jj) {
      const int j = 1 + warp + NW * jj;
      const int cr = N - 8 * j < 8 ? N - 8 * j : 8;  // J columns in the tile (≤ 0: right-hand-side tile)
#pragma unroll
      for (int i = 0; i < RT; ++i) {
        const int rr = N - 8 * i < 8 ? N - 8 * i : 8;
        double v0 = 0.0, v1 = 0.0;
        if (j < CT && cr > 0) {
          const double* tb = jst + int64_t(8 * j) * N + 8 * i * cr;
          RBNS_CHECK(int64_t(8 * j) * N + 8 * i * cr + (cr - 1) * rr + rr <= int64_t(N) * N);
          if (cr == 8 && rr == 8) {
            const double2 v = *reinterpret_cast<const double2*>(tb + 2 * lane);
            v0 = v.x;
            v1 = v.y;
          } else if (g < cr) {
            if (2 * t < rr) v0 = tb[g * rr + 2 * t];
            if (2 * t + 1 < rr) v1 = tb[g * rr + 2 * t + 1];
          }
        }
        acc[jj][i][0] = v0;
        acc[jj][i][1] = v1;
      }
    }

    TGJ_TR(5);
    // ---- right-hand side −R = f − ½ J u − ½ L(μ)u: per-lane partial row sums over the warp's columns,
    //      reduced over the 8 column lanes g by a reduce-scatter (16 + 8 + 4 shuffles for 32 values) ----
    {
      double v[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) v[k] = 0.0;
#pragma unroll
      for (int i = 0; i < RT; ++i)
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
          for (int jj = 0; jj < JJ; ++jj) v[2 * i + s] = fma(acc[jj][i][s], uj[jj], v[2 * i + s]);
      const bool h4 = (lane >> 4) & 1, h2 = (lane >> 3) & 1, h1 = (lane >> 2) & 1;
#pragma unroll
      for (int k = 0; k < 16; ++k)
        v[k] = (h4 ? v[16 + k] : v[k]) + __shfl_xor_sync(0xffffffffu, h4 ? v[k] : v[16 + k], 16);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        v[k] = (h2 ? v[8 + k] : v[k]) + __shfl_xor_sync(0xffffffffu, h2 ? v[k] : v[8 + k], 8);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        v[k] = (h1 ? v[4 + k] : v[k]) + __shfl_xor_sync(0xffffffffu, h1 ? v[k] : v[4 + k], 4);
      const int kb = (h4 ? 16 : 0) + (h2 ? 8 : 0) + (h1 ? 4 : 0);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int kk = kb + k;  // = 2 i + s
        if (kk < 2 * RT) rowred[warp][8 * (kk >> 1) + 2 * t + (kk & 1)] = v[k];
      }
    }
    TGJ_TR(6);
    __syncthreads();
    TGJ_TR(7);
    if (tid < NR) {
      const int r = tid;
      double rhs = 0.0;
      if (r < N) {
        double ju = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) ju += rowred[w][r];
        const int i = r >> 3, rr = N - 8 * i < 8 ? N - 8 * i : 8;
        const double* tb = jst + 64 * i;  // column tile 0 (N > 8: 8 columns)
#pragma unroll
        for (int c = 0; c < 8; ++c) ju = fma(tb[c * rr + (r & 7)], u0[c], ju);
        double h = 0.0;
#pragma unroll
        for (int gg = 0; gg < RBNS_MAX_GROUPS; ++gg)
          if (gg < p.G) h = fma(hw[gg], jst[N * N + gg * N + r], h);
        rhs = fr - 0.5 * ju - 0.5 * h;
      }
      sh.rhs[r] = rhs;
    }
    TGJ_TR(8);
    // panel 0 (column tile 0, shared memory only): M_i = −J_i0, M_0 = 0, transposed into the slot layout
    const int s0 = pc0 % NB;
    for (int e = tid; e < RT * 64; e += NT) {
      const int i = e >> 6, r = (e >> 3) & 7, c = e & 7;
      const int rr = N - 8 * i < 8 ? N - 8 * i : 8;
      sh.M[s0][i][tgj_slot(r, c)] = (i > 0 && r < rr) ? -jst[64 * i + c * rr + r] : 0.0;
    }
    double d0 = 0.0, d1 = 0.0;  // warp 0: pivot tile of panel 0
    if (warp == 0) {
      const double2 v = *reinterpret_cast<const double2*>(jst + 2 * lane);
      d0 = v.x;
      d1 = v.y;
    }
    TGJ_TR(2);
    __syncthreads();  // the staging buffer is consumed: stage the next sample behind the elimination
    TGJ_TR(3);
    if (tid == 0 && nxt_s < p.n) {
      fence_proxy_async_smem();
      issue(nxt_s);
    }
    if (g == gr) {  // −R into column N
#pragma unroll
      for (int jj = 0; jj < JJ; ++jj)
        if (1 + warp + NW * jj == jr) {
#pragma unroll
          for (int i = 0; i < RT; ++i) {
            acc[jj][i][0] = sh.rhs[8 * i + 2 * t];
            acc[jj][i][1] = sh.rhs[8 * i + 2 * t + 1];
          }
        }
    }
    if (warp == 0) {
      const TgjPivot pv = tgj_invert(d0, d1, 8);
      mbar_wait(&sh.empty[s0], ((uint32_t(pc0) / NB) & 1u) ^ 1u);
      sh.W[s0][tgj_slot(2 * t, g)] = sh.Wall[0][tgj_slot(2 * t, g)] = pv.w0;
      sh.W[s0][tgj_slot(2 * t + 1, g)] = sh.Wall[0][tgj_slot(2 * t + 1, g)] = pv.w1;
      sh.L[s0][tgj_slot(2 * t, g)] = pv.l0;
      sh.L[s0][tgj_slot(2 * t + 1, g)] = pv.l1;
      __syncwarp();
      if (lane == 0) {
        if (pv.bad) sh.fail = 1;
        mbar_arrive(&sh.full[s0]);
      }
      TGJ_TR(4);
    }

    // ---- blocked Gauss–Jordan over the panels (dataflow through the panel slots) ----
    // Roles at panel P: the owner of tile P+1 (critical path: panel P into its tile, invert, publish P+1,
    // then its deferred work), the owner of tile P+2 (panel P into that tile only; the rest of panel P is
    // deferred to the next panel, where it is the owner), every other warp (panel P into all live tiles).
    int pend = -1;  // panel whose remaining work this warp deferred
    auto live = [&](int j, int P) { return j < CT && (j > P || (j == P && j == jr)); };
    auto finish_panel = [&](int P, int skip_jj) {  // panel P into the live tiles except skip_jj; verify; release
      const int s = (pc0 + P) % NB;
      const double2 wv = *reinterpret_cast<const double2*>(&sh.W[s][tgj_slot(g, 2 * t)]);
#pragma unroll
      for (int jj = 0; jj < JJ; ++jj)
        if (jj != skip_jj && live(1 + warp + NW * jj, P)) tgj_apply<RT>(acc[jj], P, wv, sh.M[s]);
      if (tgj_verify<NW>(P, NP, N, wv, sh.L[s], sh.M[s]) && lane == 0) sh.fail = 1;
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.empty[s]);
      TGJ_TR(64 + 4 * P + warp);
    };
#pragma unroll 1
    for (int P = 0; P < NP; ++P) {
      const int pc = pc0 + P, s = pc % NB;
      const uint32_t par = (uint32_t(pc) / NB) & 1u;
      const int nx = P + 1;
      const bool own1 = nx < NP && warp == (nx - 1) % NW;
      mbar_wait(&sh.full[s], par);  // (sleeping between probes here measured equal or slower)
      TGJ_TR(128 + 4 * P + warp);
      if (own1) {
        // critical path: panel P into tile nx, the inverse of its new pivot tile, publication of panel nx
        const int jn = (nx - 1) / NW;
        const double2 wv = *reinterpret_cast<const double2*>(&sh.W[s][tgj_slot(g, 2 * t)]);
        const int s1 = (pc + 1) % NB;
        const int nc = nx == NP - 1 ? ncl : 8;
        const bool live_col = g < nc;
#pragma unroll
        for (int jj = 0; jj < JJ; ++jj) {
          if (jj != jn) continue;
          // (ordering note: the inversion follows the tile update; with the inversion placed between X and the
          // update, ptxas -O1..-O3 produced wrong results for a later tile of this warp, -O0 did not)
          double x0, x1, q0, q1;
          tgj_x<RT>(acc[jj], P, wv, x0, x1);
          tgj_update<RT>(acc[jj], x0, x1, sh.M[s]);
          tgj_pick<RT>(acc[jj], nx, q0, q1);
          TGJ_TR(192 + nx);
          const TgjPivot pv = tgj_invert(q0, q1, nc);
          TGJ_TR(208 + nx);
          mbar_wait(&sh.empty[s1], ((uint32_t(pc + 1) / NB) & 1u) ^ 1u);
          sh.W[s1][tgj_slot(2 * t, g)] = sh.Wall[nx][tgj_slot(2 * t, g)] = pv.w0;
          sh.W[s1][tgj_slot(2 * t + 1, g)] = sh.Wall[nx][tgj_slot(2 * t + 1, g)] = pv.w1;
          sh.L[s1][tgj_slot(2 * t, g)] = pv.l0;
          sh.L[s1][tgj_slot(2 * t + 1, g)] = pv.l1;
#pragma unroll
          for (int i = 0; i < RT; ++i) {
            sh.M[s1][i][tgj_slot(2 * t, g)] = live_col ? -acc[jj][i][0] : 0.0;
            sh.M[s1][i][tgj_slot(2 * t + 1, g)] = live_col ? -acc[jj][i][1] : 0.0;
          }
          sh.M[s1][nx][tgj_slot(2 * t, g)] = 0.0;  // the pivot row tile is left unscaled
          sh.M[s1][nx][tgj_slot(2 * t + 1, g)] = 0.0;
          __syncwarp();
          if (lane == 0 && pv.bad) sh.fail = 1;
          TGJ_TR(224 + nx);
          if (lane == 0) mbar_arrive(&sh.full[s1]);
        }
        if (pend >= 0) {
          finish_panel(pend, jn);
          pend = -1;
        }
        finish_panel(P, jn);
      } else if (nx + 1 < NP && warp == nx % NW) {
        const int jn = nx / NW;  // tile P+2: panel P now, the rest at the next panel
        const double2 wv = *reinterpret_cast<const double2*>(&sh.W[s][tgj_slot(g, 2 * t)]);
#pragma unroll
        for (int jj = 0; jj < JJ; ++jj)
          if (jj == jn) tgj_apply<RT>(acc[jj], P, wv, sh.M[s]);
        pend = P;
      } else {
        finish_panel(P, -1);
      }
    }
    pc0 += NP;
    TGJ_TR(240 + warp);

    // ---- δ = W_i y_i per row tile from the unscaled column N; stop rule; status ----
    __syncthreads();
    if (g == gr) {
#pragma unroll
      for (int jj = 0; jj < JJ; ++jj)
        if (1 + warp + NW * jj == jr) {
#pragma unroll
          for (int i = 0; i < RT; ++i) {
            sh.rhs[8 * i + 2 * t] = acc[jj][i][0];
            sh.rhs[8 * i + 2 * t + 1] = acc[jj][i][1];
          }
        }
    }
    __syncthreads();
    if (sh.fail) {  // CTA-uniform: the exact kernel redoes this sample with the pivot search
      if (tid == 0) {
        p.miss_list[atomicAdd(p.miss_count, 1)] = i_s;
        if (p.spec_miss) atomicAdd(p.spec_miss, 1);
      }
      __syncthreads();
      continue;
    }
    double x = 0.0, d2 = 0.0, un2 = 0.0, o2 = 0.0;  // o2: unknowns outside the stop norm
    static_assert(NR <= NT, "one unknown per thread");
    if (tid < N) {
      const int i = tid >> 3, r = tid & 7;
#pragma unroll
      for (int c = 0; c < 8; ++c) x = fma(sh.Wall[i][tgj_slot(r, c)], sh.rhs[8 * i + c], x);
      const double unew = p.u[int64_t(b) * N + tid] + x;
      if (tid < p.n_stop) {
        d2 = x * x;
        un2 = unew * unew;
      } else {
        o2 = fma(x, x, unew * unew);
      }
    }
    d2 = block_sum<NT>(d2, sh.red[0]);
    un2 = block_sum<NT>(un2, sh.red[1]);
    const bool finite = !__syncthreads_or(!isfinite(o2)) && isfinite(d2) && isfinite(un2);
    if (finite && tid < N) p.u[int64_t(b) * N + tid] += x;
    if (tid == 0) {
      int st;
      if (!finite)
        st = RBNS_NONFINITE;
      else if (sqrt(d2) <= p.tol * (p.stop_abs ? 1.0 : sqrt(un2)))
        st = RBNS_CONVERGED;
      else if (p.iter >= p.max_iter)
        st = RBNS_NON_CONVERGED;
      else
        st = kStatusActive;
      p.status[b] = int8_t(st);
      p.iters[b] = p.iter;
      if (finite) p.last[b] = sqrt(d2);
    }
    if (p.hint_out)  // the row order used (identity): the next iteration's hint
      for (int k = tid; k < N; k += NT) p.hint_out[int64_t(b) * N + k] = int16_t(k);
    TGJ_TR(250);
    __syncthreads();  // shared state (rhs, red, Wall, fail) is rewritten by the next sample
  }
}

}  // namespace rbns
