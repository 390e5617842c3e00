// rbns_tgh.cuh — K3 hybrid: the tiled Gauss–Jordan Newton update of rbns_tgj.cuh with each sample's matrix
// split between REGISTERS and SHARED MEMORY, one CTA per sample.  Two uses:
//
//  * config 3 (N = 200, <RT 25, CT 26, NW 12, REG 0b010>): [J | −R] is 200 × 201 fp64 = 322 KB, more than one
//    SM's 256 KB register file, so twelve warps (≤ 170 registers each) keep 12 column tiles in registers
//    (154 KB) and 13 in shared memory (166 KB), one CTA (one sample) per SM;
//  * config 2 (N = 97..103, <13, 13, 4, 0b110>): the 81 KB system fits registers (rbns_tgj.cuh holds two per
//    SM), but moving each warp's earliest-dying column tile to shared memory frees enough of the register file
//    for THREE samples per SM (4 warps × ≤ 168 registers × 3 CTAs), i.e. three independent panel chains.
//
// Column tiles j = 1 .. CT−1 (tile 0 is only panel 0; the right-hand side is column N, tile jr = N/8, column
// gr = N%8) are owned round-robin, warp w holding slot s = 0, 1, 2 → tile j = 1 + s·NW + w; bit s of REG says
// whether slot s lives in registers (the DMMA accumulator fragments of (J_ij)ᵀ, 2 doubles per lane per row
// tile) or in shared memory in the same fragment order (lane (g,t) at offset 64i + 2·lane: one conflict-free
// 16-byte access per lane; a shared tile's update is LDS.128 → 2 DMMA.8x8x4 → STS.128 per row tile).  The
// pivot column M_i of a panel is loaded once per row tile and applied to every live tile of the warp; the set
// of live tiles is a compile-time template argument of the update (a runtime flag is if-converted and issues
// the DMMAs of dead tiles).
//
// Loading: when N = 8·RT (CT = RT + 1) a shared column tile is one contiguous 8N-double block of the J buffer
// (the contraction's tile layout, jidx_tile) and is copied by the TMA engine (cp.async.bulk); otherwise the
// tiles are gathered element-wise (the last row / column tiles are packed).  Each CTA prefetches its next
// sample's J block into L2 (cp.async.bulk.prefetch.L2) so the gathers hit L2.
//
// The panel algebra, the dataflow through the three panel slots (owner of tile P+1 on the critical path, owner
// of tile P+2 deferring), the speculative no-interchange pivoting verified through the LU multipliers, the
// right-hand side −R = f − ½Ju − ½L(μ)u and the stop rule are those of rbns_tgj.cuh.  A sample that fails
// verification (or needed interchanges at its previous iteration) is appended to the miss list and redone by
// the exact kernel from its untouched J, so every result is that of partial pivoting.
#pragma once

#include "rbns_tgj.cuh"

namespace rbns {

// shared-memory tile index of slot s (a shared slot) of warp w, and the number of shared tiles
template <int CT, int NW, int REG>
__host__ __device__ constexpr int tgh_sidx(int s, int w) {
  int base = 0;
  for (int q = 0; q < s; ++q)
    if (!((REG >> q) & 1)) base += NW;
  return base + w;
}
template <int CT, int NW, int REG>
__host__ __device__ constexpr int tgh_nshared() {
  int n = 0;
  for (int s = 0; s < 3; ++s)
    if (!((REG >> s) & 1))
      for (int w = 0; w < NW; ++w)
        if (1 + s * NW + w < CT) n = tgh_sidx<CT, NW, REG>(s, w) + 1;
  return n;
}
template <int REG>
__host__ __device__ constexpr int tgh_nreg() { return (REG & 1) + ((REG >> 1) & 1) + ((REG >> 2) & 1); }
template <int REG>
__host__ __device__ constexpr int tgh_ridx(int s) { return s == 0 ? 0 : s == 1 ? (REG & 1) : (REG & 1) + ((REG >> 1) & 1); }

template <int RT, int CT, int NW, int REG>
struct TGHShared {
  static constexpr int NR = 8 * RT;
  static constexpr int NB = kTgjSlots;
  static constexpr int NS = tgh_nshared<CT, NW, REG>() > 0 ? tgh_nshared<CT, NW, REG>() : 1;
  alignas(16) double T[NS][RT][64];   // shared column tiles, fragment order
  alignas(16) double M[NB][RT][64];   // panel slots: M_i = −J_iP (tgj_slot layout); the prologue's per-warp
                                      // row sums of J u alias them
  alignas(16) double W[NB][64];       // W_P = J_PP⁻¹
  alignas(16) double L[NB][64];       // unit lower LU factor of J_PP (verification)
  alignas(16) double Wall[RT][64];    // every panel's W: final scaling of the unscaled pivot rows
  double rhs[NR];
  double red[2][NW];
  uint64_t full[NB], empty[NB];
  uint64_t bar;                       // this sample's TMA-copied shared tiles have landed (N = 8·RT)
  int fail;
};

template <int RT, int CT, int NW, int REG>
__host__ __device__ constexpr size_t tgh_smem_bytes() {
  return (sizeof(TGHShared<RT, CT, NW, REG>) + 127) & ~size_t(127);
}

// resident CTAs per SM the register file is budgeted for: 1 (≥ 8 warps: N > 127), 2 (5–7 warps: 103 < N ≤ 127),
// 3 (≤ 4 warps: the N ≤ 103 alternate)
template <int NW, int REG>
constexpr int tgh_min_blocks() { return NW >= 8 ? 1 : NW >= 5 ? 2 : 3; }

// Row tile P of a register column tile by a chain of selects (static register indices, 4 live registers).
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
// any RT): L_iP = −M_i (W L), |l| ≤ 1 on real rows.  Returns warp-uniform "rejected".
template <int RT, int NW>
__device__ __forceinline__ bool tgh_verify(int P, int N, const double2 wv, const double* Ls, const double (*M)[64]) {
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
      bad |= 8 * i + g < N && (fabs(l0) > 1.0 || fabs(l1) > 1.0);
    }
  }
  return __any_sync(0xffffffffu, bad) != 0;
}

// Panel P (W_P = Ws, pivot column M) into this warp's tiles selected by A (bit s: slot s).  X_s = W_P J_Ps per
// tile, then one load of M_i per row tile for all of them.
template <int RT, int REG, int A>
__device__ __forceinline__ void tgh_apply(double (&acc)[tgh_nreg<REG>() > 0 ? tgh_nreg<REG>() : 1][RT][2],
                                          double* const (&Ts)[3], const double* Ws, const double (*M)[64], int P) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const double2 wv = *reinterpret_cast<const double2*>(&Ws[tgj_slot(g, 2 * t)]);
  double x[3][2];
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    x[s][0] = x[s][1] = 0.0;
    if (((A >> s) & 1) == 0) continue;
    double q0, q1;
    if ((REG >> s) & 1) {
      tgh_pick<RT>(acc[tgh_ridx<REG>(s)], P, q0, q1);
    } else {
      const double2 v = *reinterpret_cast<const double2*>(Ts[s] + 64 * P + 2 * lane);
      q0 = v.x;
      q1 = v.y;
    }
    dmma_8x8x4(x[s][0], x[s][1], q0, wv.x);
    dmma_8x8x4(x[s][0], x[s][1], q1, wv.y);
  }
#pragma unroll
  for (int i = 0; i < RT; ++i) {
    const double2 m = *reinterpret_cast<const double2*>(&M[i][tgj_slot(g, 2 * t)]);
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      if (((A >> s) & 1) == 0) continue;
      if ((REG >> s) & 1) {
        double (&a)[RT][2] = acc[tgh_ridx<REG>(s)];
        dmma_8x8x4(a[i][0], a[i][1], x[s][0], m.x);
        dmma_8x8x4(a[i][0], a[i][1], x[s][1], m.y);
      } else {
        double2* c = reinterpret_cast<double2*>(Ts[s] + 64 * i + 2 * lane);
        double2 v = *c;
        dmma_8x8x4(v.x, v.y, x[s][0], m.x);
        dmma_8x8x4(v.x, v.y, x[s][1], m.y);
        *c = v;
      }
    }
  }
}

// runtime live mask → compile-time update (A = 0 does nothing)
template <int RT, int REG>
__device__ __forceinline__ void tgh_apply_mask(int a, double (&acc)[tgh_nreg<REG>() > 0 ? tgh_nreg<REG>() : 1][RT][2],
                                               double* const (&Ts)[3], const double* Ws, const double (*M)[64], int P) {
  switch (a) {
    case 1: tgh_apply<RT, REG, 1>(acc, Ts, Ws, M, P); break;
    case 2: tgh_apply<RT, REG, 2>(acc, Ts, Ws, M, P); break;
    case 3: tgh_apply<RT, REG, 3>(acc, Ts, Ws, M, P); break;
    case 4: tgh_apply<RT, REG, 4>(acc, Ts, Ws, M, P); break;
    case 5: tgh_apply<RT, REG, 5>(acc, Ts, Ws, M, P); break;
    case 6: tgh_apply<RT, REG, 6>(acc, Ts, Ws, M, P); break;
    case 7: tgh_apply<RT, REG, 7>(acc, Ts, Ws, M, P); break;
    default: break;
  }
}

#ifdef RBNS_TGH_DUMP  // development: sample position 0's load term, final y column and δ
__device__ double g_tgh_dump[4][256];
#endif

template <int RT, int CT, int NW, int REG>
__global__ void __launch_bounds__(NW * 32, tgh_min_blocks<NW, REG>()) newton_tgh_kernel(const NewtonParams p) {
  constexpr int NT = NW * 32;
  constexpr int NR = 8 * RT;
  constexpr int NB = kTgjSlots;
  constexpr int NRG = tgh_nreg<REG>() > 0 ? tgh_nreg<REG>() : 1;
  constexpr bool kFull = CT == RT + 1;  // N = 8·RT: full tiles, shared tiles by TMA bulk copies
  static_assert(CT - 1 <= 3 * NW && CT - 1 > NW, "three slots per warp cover the column tiles");
  static_assert(NR <= NT, "one row per thread");
  using SH = TGHShared<RT, CT, NW, REG>;
  extern __shared__ __align__(128) unsigned char tgh_smem[];
  SH& sh = *reinterpret_cast<SH*>(tgh_smem);
  double (*rowred)[NR] = reinterpret_cast<double (*)[NR]>(&sh.M[0][0][0]);
  static_assert(NW * NR <= NB * RT * 64, "row sums alias the panel slots");
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int N = p.N;
  constexpr int NP = RT;
  const int ncl = N - 8 * (NP - 1);   // pivot columns of the last panel
  const int jr = N >> 3, gr = N & 7;  // right-hand-side column: tile, column inside the tile
  // this warp's tiles: slot s → tile js[s] (absent when ≥ CT); shared slots point into sh.T
  int js[3];
  double* Ts[3];
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    js[s] = 1 + s * NW + warp;
    const bool sm = !((REG >> s) & 1) && js[s] < CT;
    Ts[s] = &sh.T[sm ? tgh_sidx<CT, NW, REG>(s, warp) : 0][0][0];
  }
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
  const uint32_t jbytes = uint32_t(((int64_t(N) * N + int64_t(p.G) * N) * 8 + 15) & ~int64_t(15));
  RBNS_CHECK(int64_t(jbytes) <= p.ldj * 8 && N <= NR && N > 8 * (RT - 1));

#pragma unroll 1
  for (int i_s = blockIdx.x; i_s < p.n; i_s += gridDim.x) {
    const int b = p.act[i_s];
    RBNS_CHECK(i_s >= 0 && i_s < p.n && b >= 0 && (p.B == 0 || b < p.B));
    const double* Jb = p.J + int64_t(i_s) * p.ldj;
    if (tid == 0) {
      if constexpr (kFull) {  // shared J tiles by the TMA engine (contiguous 8N-double column-tile blocks)
        constexpr uint32_t kTileBytes = uint32_t(RT) * 64u * 8u;
        fence_proxy_async_smem();
        const uint64_t pol = l2_policy_evict_first();
        uint32_t nb = 0;
        for (int s = 0; s < 3; ++s)
          if (!((REG >> s) & 1))
            for (int w = 0; w < NW; ++w) nb += (1 + s * NW + w < CT - 1) ? kTileBytes : 0u;
        mbar_arrive_expect_tx(&sh.bar, nb);
        for (int s = 0; s < 3; ++s)
          if (!((REG >> s) & 1))
            for (int w = 0; w < NW; ++w) {
              const int j = 1 + s * NW + w;
              RBNS_CHECK(j >= CT - 1 || int64_t(8 * j) * N + int64_t(RT) * 64 <= int64_t(N) * N);
              if (j < CT - 1)
                bulk_g2s(&sh.T[tgh_sidx<CT, NW, REG>(s, w)][0][0], Jb + int64_t(8 * j) * N, kTileBytes, &sh.bar, pol);
            }
      }
      const int nxt = i_s + int(gridDim.x);  // next sample's J block into L2 behind this one
      if (nxt < p.n) bulk_prefetch_l2(p.J + int64_t(nxt) * p.ldj, jbytes);
      sh.fail = 0;
    }
    // J-independent work first
    bool ident = true;
    if (p.hint_in)
      for (int k = tid; k < N; k += NT) ident &= p.hint_in[int64_t(b) * N + k] == k;
    const double fr = tid < N ? tgj_load_term(p, b, tid) : 0.0;
    double hw[RBNS_MAX_GROUPS];
#pragma unroll
    for (int gg = 0; gg < RBNS_MAX_GROUPS; ++gg)
      hw[gg] = gg < p.G ? (p.wf ? p.wf[int64_t(b) * (p.Qf + p.G) + p.Qf + gg] : mu1_pow(p.mu[2 * b + 1], p.ge[gg]))
                        : 0.0;
    double uc[3];  // this lane's column of u in each slot's tile (0 past the J columns: the right-hand side)
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const int col = 8 * js[s] + g;
      uc[s] = col < N ? p.u[int64_t(b) * N + col] : 0.0;
    }
    // register tiles (and, when gathered, shared tiles) from the J buffer; zero past the real rows / columns
    double acc[NRG][RT][2];
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const bool reg = (REG >> s) & 1;
      if (!reg && (kFull || js[s] >= CT)) continue;
      const int j = js[s];
      const int cr = N - 8 * j < 8 ? N - 8 * j : 8;  // J columns in the tile (≤ 0: right-hand-side tile)
#pragma unroll
      for (int i = 0; i < RT; ++i) {
        const int rr = N - 8 * i < 8 ? N - 8 * i : 8;
        double v0 = 0.0, v1 = 0.0;
        if constexpr (kFull) {  // every J tile full; the right-hand-side tile (cr = 0) starts at zero
          if (j < CT - 1) {
            const double2 v = __ldcs(reinterpret_cast<const double2*>(Jb + int64_t(8 * j) * N + 64 * i) + lane);
            v0 = v.x;
            v1 = v.y;
          }
        } else if (j < CT && cr > 0) {
          const double* tb = Jb + int64_t(8 * j) * N + 8 * i * cr;
          RBNS_CHECK(int64_t(8 * j) * N + 8 * i * cr + (cr - 1) * rr + rr <= int64_t(N) * N);
          if (cr == 8 && rr == 8) {
            const double2 v = __ldcs(reinterpret_cast<const double2*>(tb) + lane);
            v0 = v.x;
            v1 = v.y;
          } else if (g < cr) {
            if (2 * t < rr) v0 = __ldcs(tb + g * rr + 2 * t);
            if (2 * t + 1 < rr) v1 = __ldcs(tb + g * rr + 2 * t + 1);
          }
        }
        if (reg) {
          acc[tgh_ridx<REG>(s)][i][0] = v0;
          acc[tgh_ridx<REG>(s)][i][1] = v1;
        } else {
          *reinterpret_cast<double2*>(Ts[s] + 64 * i + 2 * lane) = make_double2(v0, v1);
        }
      }
    }
    if constexpr (kFull) {  // the right-hand-side tile (no J columns) starts at zero
#pragma unroll
      for (int s = 0; s < 3; ++s)
        if (!((REG >> s) & 1) && js[s] == CT - 1)
          for (int i = 0; i < RT; ++i) *reinterpret_cast<double2*>(Ts[s] + 64 * i + 2 * lane) = make_double2(0.0, 0.0);
    }
    // tile 0's share of J u (row r, thread r), read once from the J buffer
    double ju0 = 0.0;
    if (tid < N) {
      const int i = tid >> 3, rr = N - 8 * i < 8 ? N - 8 * i : 8;
      const double* t0 = Jb + 64 * i + (tid & 7);
#pragma unroll
      for (int c = 0; c < 8; ++c) ju0 = fma(__ldcs(t0 + c * rr), p.u[int64_t(b) * N + c], ju0);
    }
    if constexpr (kFull) {
      mbar_wait(&sh.bar, phase);
      phase ^= 1u;
    }
    if (!__syncthreads_and(ident)) {  // interchanges at the previous iteration: the exact kernel takes it
      if (tid == 0) {
        p.miss_list[atomicAdd(p.miss_count, 1)] = i_s;
        if (p.spec_miss) atomicAdd(p.spec_miss, 1);
      }
      __syncthreads();
      continue;
    }

    // ---- −R = f − ½ J u − ½ L(μ)u: per-warp row sums over the warp's J tiles, reduced over the 8 column lanes ----
#pragma unroll
    for (int i = 0; i < RT; ++i) {
      double v0 = 0.0, v1 = 0.0;
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        if (js[s] >= CT) continue;
        double a0, a1;
        if ((REG >> s) & 1) {
          a0 = acc[tgh_ridx<REG>(s)][i][0];
          a1 = acc[tgh_ridx<REG>(s)][i][1];
        } else {
          const double2 v = *reinterpret_cast<const double2*>(Ts[s] + 64 * i + 2 * lane);
          a0 = v.x;
          a1 = v.y;
        }
        v0 = fma(a0, uc[s], v0);
        v1 = fma(a1, uc[s], v1);
      }
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
    __syncthreads();
    if (tid < NR) {
      const int r = tid;
      double rhs = 0.0;
      if (r < N) {
        double ju = ju0;
#pragma unroll
        for (int w = 0; w < NW; ++w) ju += rowred[w][r];
        double h = 0.0;
#pragma unroll
        for (int gg = 0; gg < RBNS_MAX_GROUPS; ++gg)
          if (gg < p.G) h = fma(hw[gg], Jb[int64_t(N) * N + gg * N + r], h);
        rhs = fr - 0.5 * ju - 0.5 * h;
      }
      sh.rhs[r] = rhs;
    }
    __syncthreads();  // row sums consumed: the panel slots are free again
    // panel 0 (column tile 0): M_i = −J_i0 (M_0 = 0) into its slot
    const int s0 = pc0 % NB;
    for (int e = tid; e < RT * 64; e += NT) {
      const int i = e >> 6, r = (e >> 3) & 7, c = e & 7;
      const int rr = N - 8 * i < 8 ? N - 8 * i : 8;
      sh.M[s0][i][tgj_slot(r, c)] = (i > 0 && r < rr) ? -__ldcs(Jb + 64 * i + c * rr + r) : 0.0;
    }
    // −R into column N of tile jr (the owner's lanes g == gr)
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      if (js[s] != jr || g != gr) continue;
#pragma unroll
      for (int i = 0; i < RT; ++i) {
        const double r0 = sh.rhs[8 * i + 2 * t], r1 = sh.rhs[8 * i + 2 * t + 1];
        if ((REG >> s) & 1) {
          acc[tgh_ridx<REG>(s)][i][0] = r0;
          acc[tgh_ridx<REG>(s)][i][1] = r1;
        } else {
          *reinterpret_cast<double2*>(Ts[s] + 64 * i + 2 * lane) = make_double2(r0, r1);
        }
      }
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
    auto live = [&](int j, int P) { return j < CT && (j > P || (j == P && j == jr)); };
    auto live_mask = [&](int P, int skip) {
      int a = 0;
#pragma unroll
      for (int s = 0; s < 3; ++s)
        if (s != skip && live(js[s], P)) a |= 1 << s;
      return a;
    };
    auto finish_panel = [&](int P, int skip) {  // panel P into the live tiles except slot skip; verify; release
      const int s = (pc0 + P) % NB;
      tgh_apply_mask<RT, REG>(live_mask(P, skip), acc, Ts, sh.W[s], sh.M[s], P);
      const double2 wv = *reinterpret_cast<const double2*>(&sh.W[s][tgj_slot(g, 2 * t)]);
      if (tgh_verify<RT, NW>(P, N, wv, sh.L[s], sh.M[s]) && lane == 0) sh.fail = 1;
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
        const int k = (nx - 1) / NW;  // slot of tile nx
        tgh_apply_mask<RT, REG>(1 << k, acc, Ts, sh.W[s], sh.M[s], P);
        double q0 = 0.0, q1 = 0.0;
#pragma unroll
        for (int ss = 0; ss < 3; ++ss) {
          if (ss != k) continue;
          if ((REG >> ss) & 1) {
            tgh_pick<RT>(acc[tgh_ridx<REG>(ss)], nx, q0, q1);
          } else {
            const double2 v = *reinterpret_cast<const double2*>(Ts[ss] + 64 * nx + 2 * lane);
            q0 = v.x;
            q1 = v.y;
          }
        }
        const int nc = nx == NP - 1 ? ncl : 8;
        const TgjPivot pv = tgj_invert(q0, q1, nc);
        const int s1 = (pc + 1) % NB;
        mbar_wait(&sh.empty[s1], ((uint32_t(pc + 1) / NB) & 1u) ^ 1u);
        sh.W[s1][tgj_slot(2 * t, g)] = sh.Wall[nx][tgj_slot(2 * t, g)] = pv.w0;
        sh.W[s1][tgj_slot(2 * t + 1, g)] = sh.Wall[nx][tgj_slot(2 * t + 1, g)] = pv.w1;
        sh.L[s1][tgj_slot(2 * t, g)] = pv.l0;
        sh.L[s1][tgj_slot(2 * t + 1, g)] = pv.l1;
        const bool live_col = g < nc;
#pragma unroll
        for (int ss = 0; ss < 3; ++ss) {
          if (ss != k) continue;
#pragma unroll
          for (int i = 0; i < RT; ++i) {
            double a0, a1;
            if ((REG >> ss) & 1) {
              a0 = acc[tgh_ridx<REG>(ss)][i][0];
              a1 = acc[tgh_ridx<REG>(ss)][i][1];
            } else {
              const double2 v = *reinterpret_cast<const double2*>(Ts[ss] + 64 * i + 2 * lane);
              a0 = v.x;
              a1 = v.y;
            }
            const bool z = i == nx || !live_col;  // the pivot row tile is left unscaled
            sh.M[s1][i][tgj_slot(2 * t, g)] = z ? 0.0 : -a0;
            sh.M[s1][i][tgj_slot(2 * t + 1, g)] = z ? 0.0 : -a1;
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
        tgh_apply_mask<RT, REG>(1 << k, acc, Ts, sh.W[s], sh.M[s], P);
        pend = P;
      } else {
        finish_panel(P, -1);
      }
    }
    pc0 += NP;

    // ---- δ = W_i y_i per row tile from the unscaled right-hand-side column; stop rule; status ----
    __syncthreads();
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      if (js[s] != jr || g != gr) continue;
#pragma unroll
      for (int i = 0; i < RT; ++i) {
        double a0, a1;
        if ((REG >> s) & 1) {
          a0 = acc[tgh_ridx<REG>(s)][i][0];
          a1 = acc[tgh_ridx<REG>(s)][i][1];
        } else {
          const double2 v = *reinterpret_cast<const double2*>(Ts[s] + 64 * i + 2 * lane);
          a0 = v.x;
          a1 = v.y;
        }
        sh.rhs[8 * i + 2 * t] = a0;
        sh.rhs[8 * i + 2 * t + 1] = a1;
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
    double x = 0.0, d2 = 0.0, un2 = 0.0, o2 = 0.0;
    if (tid < N) {
      const int i = tid >> 3, r = tid & 7;
#pragma unroll
      for (int c = 0; c < 8; ++c) x = fma(sh.Wall[i][tgj_slot(r, c)], sh.rhs[8 * i + c], x);
#ifdef RBNS_TGH_DUMP
      if (i_s == 0) {
        g_tgh_dump[0][tid] = fr;
        g_tgh_dump[1][tid] = sh.rhs[tid];
        g_tgh_dump[2][tid] = x;
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
