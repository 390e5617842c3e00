// rbns_tgh.cuh — K3 for config 3 (N = 8·RT, RT = 25: N = 200): the tiled Gauss–Jordan Newton update of
// rbns_tgj.cuh for a system that does not fit one SM's register file, on ONE CTA per sample with the matrix
// split between registers and shared memory.
//
// [J | −R] at N = 200 is 200 × 201 fp64 = 322 KB; an SM has 256 KB of registers and 227 KB of shared memory
// per CTA.  Twelve warps (384 threads, ≤ 170 registers each) own the 25 column tiles j = 1..25 (tile 0 is only
// panel 0; tile 25 holds the right-hand side in its column 0) round-robin, warp w = (j−1) mod 12:
//     slot 0  j = 1 + w        shared memory   (dies at panel j, early)
//     slot 1  j = 13 + w       registers       (50 doubles per lane: the DMMA accumulator fragments of (J_ij)ᵀ)
//     slot 2  j = 25 (w = 0)   shared memory   (right-hand side, live at every panel)
// i.e. 12 column tiles in registers (154 KB) and 13 in shared memory (166 KB), each shared tile stored in the
// fragment order (lane (g,t) finds rows 8i+2t, 8i+2t+1 of column 8j+g at offset 64i + 2·lane: one conflict-free
// 16-byte access per lane), which is also the contraction's tile layout of J (jidx_tile, rbns_common.cuh) for
// N % 8 == 0 — so a sample's shared column tiles are copied straight from the J buffer by the TMA engine
// (cp.async.bulk), while the register tiles are loaded with coalesced 16-byte loads.  A shared tile's update is
// LDS.128 → 2 DMMA.8x8x4 → STS.128 per row tile; the pivot column M_i of the panel is loaded once per row tile
// and applied to every live tile of the warp.
//
// The panel algebra, the dataflow through the three panel slots (owner of tile P+1 on the critical path, owner
// of tile P+2 deferring), the speculative no-interchange pivoting verified through the LU multipliers, the
// right-hand side −R = f − ½Ju − ½L(μ)u and the stop rule are those of rbns_tgj.cuh.  A sample that fails
// verification (or needed interchanges at its previous iteration) is appended to the miss list and redone by
// the exact 2-CTA cluster kernel (rbns_newton_cluster.cuh) from its untouched J, so every result is that of
// partial pivoting.
#pragma once

#include "rbns_tgj.cuh"

namespace rbns {

template <int RT, int NW>
struct TGHShared {
  static constexpr int NR = 8 * RT;
  static constexpr int NB = kTgjSlots;
  static constexpr int NS = RT - NW;  // shared column tiles: slot 0 (NW tiles) + slot 2 (RT − 2NW tiles)
  alignas(16) double T[NS][RT][64];   // shared column tiles, fragment order
  alignas(16) double M[NB][RT][64];   // panel slots: M_i = −J_iP (tgj_slot layout); the prologue's per-warp
                                      // row sums of J u alias them
  alignas(16) double W[NB][64];       // W_P = J_PP⁻¹
  alignas(16) double L[NB][64];       // unit lower LU factor of J_PP (verification)
  alignas(16) double Wall[RT][64];    // every panel's W: final scaling of the unscaled pivot rows
  double rhs[NR];
  double red[2][NW];
  uint64_t full[NB], empty[NB];
  uint64_t bar;                       // this sample's shared column tiles have landed
  int fail;
};

template <int RT, int NW>
__host__ __device__ constexpr size_t tgh_smem_bytes() {
  return (sizeof(TGHShared<RT, NW>) + 127) & ~size_t(127);
}

// Row tile P of a register column tile by a chain of selects (static register indices; RT is too large for
// the select tree of tgj_pick to stay within the register budget).
template <int RT>
__device__ __forceinline__ void tgh_pick(const double (&a)[RT][2], int P, double& p0, double& p1) {
  p0 = a[0][0];
  p1 = a[0][1];
#pragma unroll
  for (int i = 1; i < RT; ++i) {
    p0 = P == i ? a[i][0] : p0;
    p1 = P == i ? a[i][1] : p1;
  }
}

// Verification of panel P for this warp's share of the rows below the pivot tile (rbns_tgj.cuh tgj_verify,
// any RT): L_iP = −M_i (W L), |l| ≤ 1.  Returns warp-uniform "rejected".
template <int RT, int NW>
__device__ __forceinline__ bool tgh_verify(int P, const double2 wv, const double* Ls, const double (*M)[64]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int i0 = P + 1 + ((warp - (P + 1) % NW) + NW) % NW;
  if (i0 >= RT) return false;
  double ui0 = 0.0, ui1 = 0.0;
  dmma_8x8x4(ui0, ui1, Ls[tgj_slot(2 * t, g)], wv.x);
  dmma_8x8x4(ui0, ui1, Ls[tgj_slot(2 * t + 1, g)], wv.y);
  bool bad = false;
  constexpr int MAXI = (RT + NW - 1) / NW;
#pragma unroll
  for (int k = 0; k < MAXI; ++k) {
    const int i = i0 + k * NW;
    if (i < RT) {
      const double2 m = *reinterpret_cast<const double2*>(&M[i][tgj_slot(g, 2 * t)]);
      double l0 = 0.0, l1 = 0.0;
      dmma_8x8x4(l0, l1, m.x, ui0);
      dmma_8x8x4(l0, l1, m.y, ui1);
      bad |= fabs(l0) > 1.0 || fabs(l1) > 1.0;
    }
  }
  return __any_sync(0xffffffffu, bad) != 0;
}

// Panel P (W_P = Ws, pivot column M) into this warp's selected tiles: shared tile T0 (A0), the register tile
// (A1), shared tile T2 (A2).  X_k = W_P J_Pk per tile, then one load of M_i per row tile for all of them.
template <int RT, int A0, int A1, int A2>
__device__ __forceinline__ void tgh_apply(double (&acc)[RT][2], double* T0, double* T2, const double* Ws,
                                          const double (*M)[64], int P) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const double2 wv = *reinterpret_cast<const double2*>(&Ws[tgj_slot(g, 2 * t)]);
  double x00 = 0.0, x01 = 0.0, x10 = 0.0, x11 = 0.0, x20 = 0.0, x21 = 0.0;
  if constexpr (A0 != 0) {
    const double2 pv = *reinterpret_cast<const double2*>(T0 + 64 * P + 2 * lane);
    dmma_8x8x4(x00, x01, pv.x, wv.x);
    dmma_8x8x4(x00, x01, pv.y, wv.y);
  }
  if constexpr (A1 != 0) {
    double q0, q1;
    tgh_pick<RT>(acc, P, q0, q1);
    dmma_8x8x4(x10, x11, q0, wv.x);
    dmma_8x8x4(x10, x11, q1, wv.y);
  }
  if constexpr (A2 != 0) {
    const double2 pv = *reinterpret_cast<const double2*>(T2 + 64 * P + 2 * lane);
    dmma_8x8x4(x20, x21, pv.x, wv.x);
    dmma_8x8x4(x20, x21, pv.y, wv.y);
  }
#pragma unroll
  for (int i = 0; i < RT; ++i) {
    const double2 m = *reinterpret_cast<const double2*>(&M[i][tgj_slot(g, 2 * t)]);
    if constexpr (A1 != 0) {
      dmma_8x8x4(acc[i][0], acc[i][1], x10, m.x);
      dmma_8x8x4(acc[i][0], acc[i][1], x11, m.y);
    }
    if constexpr (A0 != 0) {
      double2* c = reinterpret_cast<double2*>(T0 + 64 * i + 2 * lane);
      double2 v = *c;
      dmma_8x8x4(v.x, v.y, x00, m.x);
      dmma_8x8x4(v.x, v.y, x01, m.y);
      *c = v;
    }
    if constexpr (A2 != 0) {
      double2* c = reinterpret_cast<double2*>(T2 + 64 * i + 2 * lane);
      double2 v = *c;
      dmma_8x8x4(v.x, v.y, x20, m.x);
      dmma_8x8x4(v.x, v.y, x21, m.y);
      *c = v;
    }
  }
}

#ifdef RBNS_TGH_DUMP  // development: sample position 0's right-hand side, final y column and δ
__device__ double g_tgh_dump[4][256];
#endif

template <int RT, int NW>
__global__ void __launch_bounds__(NW * 32, 1) newton_tgh_kernel(const NewtonParams p) {
  constexpr int NT = NW * 32;
  constexpr int NR = 8 * RT;
  constexpr int NB = kTgjSlots;
  static_assert(RT > 2 * NW && RT <= 3 * NW, "slot layout: two shared slots + one register slot per warp");
  static_assert(NR <= NT, "one row per thread");
  using SH = TGHShared<RT, NW>;
  extern __shared__ __align__(128) unsigned char tgh_smem[];
  SH& sh = *reinterpret_cast<SH*>(tgh_smem);
  double (*rowred)[NR] = reinterpret_cast<double (*)[NR]>(&sh.M[0][0][0]);
  static_assert(NW * NR <= NB * RT * 64, "row sums alias the panel slots");
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int N = p.N;  // == NR (the host plan guarantees N % 8 == 0)
  constexpr int NP = RT;
  // this warp's tiles
  const int j0 = 1 + warp, j1 = 1 + NW + warp, j2 = 1 + 2 * NW + warp;
  const bool has2 = j2 <= RT;  // slot 2 exists (j2 == RT: the right-hand-side tile)
  double* T0 = &sh.T[j0 - 1][0][0];
  double* T2 = &sh.T[has2 ? j2 - 1 - NW : 0][0][0];
  constexpr int kRhsTile = RT - 1 - NW;  // shared index of tile RT (right-hand side, column 0)
  constexpr uint32_t kTileBytes = uint32_t(RT) * 64u * 8u;
  if (tid == 0) {
    mbar_init(&sh.bar, 1);
    for (int s = 0; s < NB; ++s) {
      mbar_init(&sh.full[s], 1);
      mbar_init(&sh.empty[s], NW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  uint32_t phase = 0;
  int pc0 = 0;

#pragma unroll 1
  for (int i_s = blockIdx.x; i_s < p.n; i_s += gridDim.x) {
    const int b = p.act[i_s];
    const double* Jb = p.J + int64_t(i_s) * p.ldj;
    if (tid == 0) {
      // shared column tiles 1..NW (slot 0) by the TMA engine, one bulk copy each (contiguous 8N-double blocks);
      // the next sample's block is prefetched into L2 behind this one
      fence_proxy_async_smem();
      const uint64_t pol = l2_policy_evict_first();
      mbar_arrive_expect_tx(&sh.bar, uint32_t(NW) * kTileBytes);
      for (int j = 1; j <= NW; ++j) bulk_g2s(&sh.T[j - 1][0][0], Jb + int64_t(8 * j) * N, kTileBytes, &sh.bar, pol);
      const int nxt = i_s + int(gridDim.x);
      if (nxt < p.n) bulk_prefetch_l2(p.J + int64_t(nxt) * p.ldj, uint32_t((int64_t(N) * N + int64_t(p.G) * N) * 8 + 15) & ~15u);
      sh.fail = 0;
    }
    // J-independent work and the register tile while the bulk copies are in flight
    bool ident = true;
    if (p.hint_in)
      for (int k = tid; k < N; k += NT) ident &= p.hint_in[int64_t(b) * N + k] == k;
    const double fr = tid < N ? tgj_load_term(p, b, tid) : 0.0;
    double hw[RBNS_MAX_GROUPS];
#pragma unroll
    for (int gg = 0; gg < RBNS_MAX_GROUPS; ++gg)
      hw[gg] = gg < p.G ? (p.wf ? p.wf[int64_t(b) * (p.Qf + p.G) + p.Qf + gg] : mu1_pow(p.mu[2 * b + 1], p.ge[gg]))
                        : 0.0;
    const double uc0 = p.u[int64_t(b) * N + 8 * j0 + g];
    const double uc1 = p.u[int64_t(b) * N + 8 * j1 + g];
    double acc[RT][2];
    {
      const double2* src = reinterpret_cast<const double2*>(Jb + int64_t(8 * j1) * N) + lane;
#pragma unroll
      for (int i = 0; i < RT; ++i) {
        const double2 v = __ldcs(src + 32 * i);
        acc[i][0] = v.x;
        acc[i][1] = v.y;
      }
    }
    // tile 0's share of J u (row r, thread r), read once from the J buffer
    double ju0 = 0.0;
    if (tid < N) {
      const double* t0 = Jb + 64 * (tid >> 3) + (tid & 7);
#pragma unroll
      for (int c = 0; c < 8; ++c) ju0 = fma(__ldcs(t0 + 8 * c), p.u[int64_t(b) * N + c], ju0);
    }
    mbar_wait(&sh.bar, phase);
    phase ^= 1u;
    if (!__syncthreads_and(ident)) {  // interchanges at the previous iteration: the exact kernel takes it
      if (tid == 0) {
        p.miss_list[atomicAdd(p.miss_count, 1)] = i_s;
        if (p.spec_miss) atomicAdd(p.spec_miss, 1);
      }
      __syncthreads();
      continue;
    }

    // ---- −R = f − ½ J u − ½ L(μ)u: per-warp row sums over the warp's J tiles, reduced over the 8 column lanes ----
    {
#pragma unroll
      for (int i = 0; i < RT; ++i) {
        const double2 s0 = *reinterpret_cast<const double2*>(T0 + 64 * i + 2 * lane);
        double v0 = fma(acc[i][0], uc1, s0.x * uc0);
        double v1 = fma(acc[i][1], uc1, s0.y * uc0);
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          v0 += __shfl_xor_sync(0xffffffffu, v0, o);
          v1 += __shfl_xor_sync(0xffffffffu, v1, o);
        }
        if (g == 0) {
          rowred[warp][8 * i + 2 * t] = v0;
          rowred[warp][8 * i + 2 * t + 1] = v1;
        }
      }
    }
    __syncthreads();
    if (tid < NR) {
      const int r = tid;
      double ju = ju0;
#pragma unroll
      for (int w = 0; w < NW; ++w) ju += rowred[w][r];
      double h = 0.0;
#pragma unroll
      for (int gg = 0; gg < RBNS_MAX_GROUPS; ++gg)
        if (gg < p.G) h = fma(hw[gg], Jb[int64_t(N) * N + gg * N + r], h);
      sh.rhs[r] = fr - 0.5 * ju - 0.5 * h;
    }
    __syncthreads();  // row sums consumed: the panel slots are free again
    // panel 0 (column tile 0): M_i = −J_i0 (M_0 = 0) into its slot; the right-hand-side tile: column 0 = −R
    const int s0 = pc0 % NB;
    for (int e = tid; e < RT * 64; e += NT) {
      const int i = e >> 6, r = (e >> 3) & 7, c = e & 7;
      sh.M[s0][i][tgj_slot(r, c)] = i > 0 ? -__ldcs(Jb + 64 * i + 8 * c + r) : 0.0;
      sh.T[kRhsTile][i][e & 63] = (e & 63) < 8 ? sh.rhs[8 * i + (e & 7)] : 0.0;
    }
    double d0 = 0.0, d1 = 0.0;
    if (warp == 0) {
      const double2 v = __ldcs(reinterpret_cast<const double2*>(Jb) + lane);
      d0 = v.x;
      d1 = v.y;
    }
    __syncthreads();
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
    }

    // ---- blocked Gauss–Jordan over the panels (rbns_tgj.cuh dataflow) ----
    // Panel P into the selected live tiles of this warp: X_k = W_P J_Pk per tile, then per row tile i one load
    // of M_i for all of them.  The pivot row tile (M_P = 0) is left as it is.
    auto apply = [&](int P, bool a0, bool a1, bool a2) {
      const int s = (pc0 + P) % NB;
      // compile-time tile selection: a runtime flag would be if-converted and the DMMAs of dead tiles issued
      const int sel = (a0 ? 1 : 0) | (a1 ? 2 : 0) | (a2 ? 4 : 0);
      switch (sel) {
        case 1: tgh_apply<RT, 1, 0, 0>(acc, T0, T2, sh.W[s], sh.M[s], P); break;
        case 2: tgh_apply<RT, 0, 1, 0>(acc, T0, T2, sh.W[s], sh.M[s], P); break;
        case 3: tgh_apply<RT, 1, 1, 0>(acc, T0, T2, sh.W[s], sh.M[s], P); break;
        case 4: tgh_apply<RT, 0, 0, 1>(acc, T0, T2, sh.W[s], sh.M[s], P); break;
        case 5: tgh_apply<RT, 1, 0, 1>(acc, T0, T2, sh.W[s], sh.M[s], P); break;
        case 6: tgh_apply<RT, 0, 1, 1>(acc, T0, T2, sh.W[s], sh.M[s], P); break;
        case 7: tgh_apply<RT, 1, 1, 1>(acc, T0, T2, sh.W[s], sh.M[s], P); break;
        default: break;
      }
    };
    // panel P into the live tiles other than slot `skip`, verification, release of the slot
    auto finish_panel = [&](int P, int skip) {
      apply(P, skip != 0 && j0 > P, skip != 1 && j1 > P, skip != 2 && has2);
      const int s = (pc0 + P) % NB;
      const double2 wv = *reinterpret_cast<const double2*>(&sh.W[s][tgj_slot(g, 2 * t)]);
      if (tgh_verify<RT, NW>(P, wv, sh.L[s], sh.M[s]) && lane == 0) sh.fail = 1;
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.empty[s]);
    };
    int pend = -1;
#pragma unroll 1
    for (int P = 0; P < NP; ++P) {
      const int pc = pc0 + P, s = pc % NB;
      const uint32_t par = (uint32_t(pc) / NB) & 1u;
      const int nx = P + 1;
      mbar_wait(&sh.full[s], par);
      if (nx < NP && warp == (nx - 1) % NW) {
        // critical path: panel P into tile nx, the inverse of its new pivot tile, publication of panel nx
        const int k = (nx - 1) / NW;  // slot of tile nx (0: shared, 1: registers)
        apply(P, k == 0, k == 1, false);
        double q0, q1;
        if (k == 0) {
          const double2 v = *reinterpret_cast<const double2*>(T0 + 64 * nx + 2 * lane);
          q0 = v.x;
          q1 = v.y;
        } else {
          tgh_pick<RT>(acc, nx, q0, q1);
        }
        const TgjPivot pv = tgj_invert(q0, q1, 8);
        const int s1 = (pc + 1) % NB;
        mbar_wait(&sh.empty[s1], ((uint32_t(pc + 1) / NB) & 1u) ^ 1u);
        sh.W[s1][tgj_slot(2 * t, g)] = sh.Wall[nx][tgj_slot(2 * t, g)] = pv.w0;
        sh.W[s1][tgj_slot(2 * t + 1, g)] = sh.Wall[nx][tgj_slot(2 * t + 1, g)] = pv.w1;
        sh.L[s1][tgj_slot(2 * t, g)] = pv.l0;
        sh.L[s1][tgj_slot(2 * t + 1, g)] = pv.l1;
        if (k == 0) {
#pragma unroll 5
          for (int i = 0; i < RT; ++i) {
            const double2 v = *reinterpret_cast<const double2*>(T0 + 64 * i + 2 * lane);
            sh.M[s1][i][tgj_slot(2 * t, g)] = i == nx ? 0.0 : -v.x;
            sh.M[s1][i][tgj_slot(2 * t + 1, g)] = i == nx ? 0.0 : -v.y;
          }
        } else {
#pragma unroll
          for (int i = 0; i < RT; ++i) {
            sh.M[s1][i][tgj_slot(2 * t, g)] = i == nx ? 0.0 : -acc[i][0];
            sh.M[s1][i][tgj_slot(2 * t + 1, g)] = i == nx ? 0.0 : -acc[i][1];
          }
        }
        __syncwarp();
        if (lane == 0) {
          if (pv.bad) sh.fail = 1;
          mbar_arrive(&sh.full[s1]);
        }
        if (pend >= 0) {
          finish_panel(pend, k);
          pend = -1;
        }
        finish_panel(P, k);
      } else if (nx + 1 < NP && warp == nx % NW) {
        const int k = nx / NW;  // tile nx+1: panel P now, the rest of panel P at the next panel
        apply(P, k == 0, k == 1, false);
        pend = P;
      } else {
        finish_panel(P, -1);
      }
    }
    pc0 += NP;

    // ---- δ = W_i y_i per row tile from the unscaled right-hand-side column; stop rule; status ----
    __syncthreads();
    if (sh.fail) {  // CTA-uniform: the exact kernel redoes this sample with the pivot search
      if (tid == 0) {
        p.miss_list[atomicAdd(p.miss_count, 1)] = i_s;
        if (p.spec_miss) atomicAdd(p.spec_miss, 1);
      }
      __syncthreads();
      continue;
    }
    double x = 0.0, d2 = 0.0, un2 = 0.0, o2 = 0.0;
    if (tid < N) {
      const int i = tid >> 3, r = tid & 7;
#pragma unroll
      for (int c = 0; c < 8; ++c) x = fma(sh.Wall[i][tgj_slot(r, c)], sh.T[kRhsTile][i][c], x);
#ifdef RBNS_TGH_DUMP
      if (i_s == 0) {
        g_tgh_dump[0][tid] = sh.rhs[tid];
        g_tgh_dump[1][tid] = sh.T[kRhsTile][i][r];
        g_tgh_dump[2][tid] = x;
        g_tgh_dump[3][tid] = sh.T[kRhsTile][i][8 + r];  // column 1 of the right-hand-side tile (must stay 0)
      }
#endif
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
    if (p.hint_out)
      for (int k = tid; k < N; k += NT) p.hint_out[int64_t(b) * N + k] = int16_t(k);
    __syncthreads();  // shared state (tiles, rhs, red, Wall, fail) is rewritten by the next sample
  }
}

}  // namespace rbns
