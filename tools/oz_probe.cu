// oz_probe.cu — standalone check and timing of the INT8-sliced contraction GEMM (csrc/rbns_oz.cuh).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I include -I paper_1807_11866_b200/csrc \
//        tools/oz_probe.cu -o build/oz_probe
//   build/oz_probe [n_samples] [N] [Q] [reps]
// Checks: (1) the device result equals a host emulation of the same splitting bit for bit (validates the MMA
// descriptors, TMEM mapping and pipeline); (2) error against a long-double dot product, beside the error of a
// plain binary64 dot product, both relative to Σ|x||s|.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define RBNS_OZ_PROBE 1
#include "rbns_oz.cuh"

using namespace rbns;
using namespace rbns::oz;

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(2);                                                               \
    }                                                                             \
  } while (0)

// digits and scale of one row (values already column-equilibrated)
static double host_slice(const std::vector<double>& v, std::vector<int>& dig) {
  double m = 0.0;
  for (double x : v) m = std::fmax(m, std::fabs(x));
  dig.assign(v.size() * kS, 0);
  if (m == 0.0) return 0.0;
  const int E = std::ilogb(m) + 1;
  for (size_t k = 0; k < v.size(); ++k) {
    int d[kS];
    digits(std::ldexp(v[k], -(E + 1)), d);
    for (int i = 0; i < kS; ++i) dig[k * kS + i] = d[i];
  }
  return std::ldexp(1.0, E - 6);
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 4096;
  const int N = argc > 2 ? std::atoi(argv[2]) : 100;
  const int Q = argc > 3 ? std::atoi(argv[3]) : 7;
  const int reps = argc > 4 ? std::atoi(argv[4]) : 5;
  const int Ne = (N + 3) / 4 * 4;
  const int Qb = Q, Ql = Q;
  const int K = Qb * Ne + (Ql + 3) / 4 * 4;  // columns of S: blocks, then the affine columns
  const int kterms = Qb * Ne;
  const int k32 = (kterms + 31) / 32 * 32;
  const int64_t R = int64_t(N) * N + N;
  const int64_t row_tiles = (R + kTM - 1) / kTM, Rp = row_tiles * kTM;
  const int sample_tiles = (n + kTN - 1) / kTN;
  const int kchunks = k32 / kKC;
  std::printf("n=%d N=%d Q=%d K=%d k32=%d R=%lld row_tiles=%lld sample_tiles=%d slices=%d stages=%d smem=%zu\n", n, N, Q, K,
              k32, (long long)R, (long long)row_tiles, sample_tiles, kS, kStages, kSmemBytes);

  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd(0.0, 1.0);
  std::uniform_real_distribution<double> ud(-1.0, 1.0);
  std::vector<double> S(size_t(R) * K), u(size_t(n) * N), w(size_t(n) * (Qb + Ql));
  for (int64_t r = 0; r < R; ++r)
    for (int k = 0; k < K; ++k) {
      double v;
      if (k < Qb * Ne)
        v = (k % Ne) < N ? 1e-7 * nd(rng) : 0.0;
      else
        v = (k - Qb * Ne) < Ql ? 0.1 * nd(rng) : 0.0;
      S[size_t(r) * K + k] = v;
    }
  for (int b = 0; b < n; ++b) {
    for (int k = 0; k < N; ++k) u[size_t(b) * N + k] = nd(rng) * std::pow(0.9, k);
    for (int q = 0; q < Qb; ++q) w[size_t(b) * (Qb + Ql) + q] = ud(rng);
    for (int q = 0; q < Ql; ++q) w[size_t(b) * (Qb + Ql) + Qb + q] = 0.01 * ud(rng);
  }

  double *dS, *du, *dw, *dsa, *dsb, *dout, *daff;
  int32_t* dcexp;
  uint8_t *dA8, *dB8;
  const int64_t ldo = Rp;
  CK(cudaMalloc(&dS, S.size() * 8));
  CK(cudaMalloc(&du, u.size() * 8));
  CK(cudaMalloc(&dw, w.size() * 8));
  CK(cudaMalloc(&dsa, Rp * 8));
  CK(cudaMalloc(&daff, size_t(Ql) * Rp * 8));
  CK(cudaMalloc(&dsb, size_t(sample_tiles) * kTN * 8));
  CK(cudaMalloc(&dout, size_t(n) * ldo * 8));
  CK(cudaMalloc(&dcexp, k32 * 4));
  CK(cudaMalloc(&dA8, size_t(row_tiles) * kchunks * kAStage));
  CK(cudaMalloc(&dB8, size_t(sample_tiles) * kchunks * kBStage));
  CK(cudaMemcpy(dS, S.data(), S.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(du, u.data(), u.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dw, w.data(), w.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemset(dcexp, 0, k32 * 4));
  CK(cudaMemset(dout, 0xff, size_t(n) * ldo * 8));

  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float ms;

  CK(cudaEventRecord(e0));
  oz_col_exponents<<<kterms, 256>>>(dS, R, kterms, K, dcexp);
  oz_slice_S<<<unsigned((Rp + 7) / 8), 256>>>(dS, R, kterms, K, dcexp, k32, dA8, dsa, Rp);
  oz_gather_affine<<<unsigned((int64_t(Ql) * Rp + 255) / 256), 256>>>(dS, R, K, kterms, Ql, daff, Rp);
  CK(cudaEventRecord(e1));
  CK(cudaDeviceSynchronize());
  CK(cudaEventElapsedTime(&ms, e0, e1));
  std::printf("slice S: %.3f ms\n", ms);

  SliceXParams sp{};
  sp.act = nullptr;
  sp.n = n;
  sp.u = du;
  sp.wts = dw;
  sp.cexp = dcexp;
  sp.N = N;
  sp.Ne = Ne;
  sp.Qb = Qb;
  sp.Ql = Ql;
  sp.k32 = k32;
  sp.B8 = dB8;
  sp.sb = dsb;
  GemmParams gp{};
  gp.A8 = dA8;
  gp.B8 = dB8;
  gp.sa = dsa;
  gp.sb = dsb;
  gp.kchunks = kchunks;
  gp.kc_begin = 0;
  gp.row_tiles = int(row_tiles);
  gp.n = n;
  gp.out = dout;
  gp.ldo = ldo;
  gp.aff = daff;
  gp.aff_ld = Rp;
  gp.wts = dw;
  gp.act = nullptr;
  gp.Qb = Qb;
  gp.Ql = Ql;
  gp.ldw = Qb + Ql;
  int groups = std::max(1, (148 * 4 + sample_tiles - 1) / sample_tiles);
  groups = std::min<int>(groups, int(row_tiles));
  gp.tiles_per_group = int((row_tiles + groups - 1) / groups);
  groups = int((row_tiles + gp.tiles_per_group - 1) / gp.tiles_per_group);
  CK(cudaFuncSetAttribute(oz_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemBytes)));
  dim3 grid(sample_tiles, groups);
  std::printf("grid %d x %d, tiles_per_group %d\n", sample_tiles, groups, gp.tiles_per_group);

  long long* dtrace;
  CK(cudaMalloc(&dtrace, 64 * 8));
  CK(cudaMemset(dtrace, 0, 64 * 8));
  {
    GemmParams gd = gp;
    gd.trace = dtrace;
    oz_slice_X<<<sample_tiles * kTN / 8, 256>>>(sp);
    oz_gemm_kernel<<<grid, kThreads, kSmemBytes>>>(gd);
    CK(cudaDeviceSynchronize());
    long long tr[64];
    CK(cudaMemcpy(tr, dtrace, sizeof(tr), cudaMemcpyDeviceToHost));
    for (int t = 0; t < 4; ++t)
      std::printf("trace tile %d: start %lld | issue done +%lld | accum done +%lld | tmem drained +%lld | epilogue end +%lld\n", t,
                  tr[t * 8] - tr[0], tr[t * 8 + 1] - tr[t * 8], tr[t * 8 + 2] - tr[t * 8], tr[t * 8 + 3] - tr[t * 8],
                  tr[t * 8 + 4] - tr[t * 8]);
  }
  for (int dbg : {1, 2, 4, 8, 9}) {  // pipeline ablations (results are wrong by construction)
    GemmParams gd = gp;
    gd.dbg = dbg;
    oz_slice_X<<<sample_tiles * kTN / 8, 256>>>(sp);
    CK(cudaEventRecord(e0));
    oz_gemm_kernel<<<grid, kThreads, kSmemBytes>>>(gd);
    CK(cudaEventRecord(e1));
    CK(cudaDeviceSynchronize());
    CK(cudaEventElapsedTime(&ms, e0, e1));
    std::printf("ablation dbg=%d (1 no copies, 2 first A slice only, 4 no stores, 8 drain only): gemm %.3f ms\n", dbg, ms);
  }
  for (int it = 0; it < reps; ++it) {
    CK(cudaEventRecord(e0));
    oz_slice_X<<<sample_tiles * kTN / 8, 256>>>(sp);
    CK(cudaEventRecord(e1));
    CK(cudaDeviceSynchronize());
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const float ms_x = ms;
    CK(cudaEventRecord(e0));
    oz_gemm_kernel<<<grid, kThreads, kSmemBytes>>>(gp);
    CK(cudaEventRecord(e1));
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double flops = 2.0 * double(n) * double(R) * double(Qb) * double(N) * double(N) / double(N);  // 2·Q·N·R per sample
    const double macs = double(sample_tiles) * kTN * double(Rp) * k32 * (kS * (kS + 1) / 2);
    std::printf("rep %d: slice X %.3f ms, gemm %.3f ms  (%.1f FP64-equivalent TF/s, %.0f int8 TOPS)\n", it, ms_x, ms,
                flops / ms * 1e-9, 2.0 * macs / ms * 1e-9);
  }

  // ---- checks ----
  std::vector<double> out(size_t(n) * ldo);
  CK(cudaMemcpy(out.data(), dout, out.size() * 8, cudaMemcpyDeviceToHost));
  std::vector<int32_t> cexp(k32, 0);
  for (int k = 0; k < kterms; ++k) {
    double m = 0.0;
    for (int64_t r = 0; r < R; ++r) m = std::fmax(m, std::fabs(S[size_t(r) * K + k]));
    cexp[k] = m > 0.0 ? std::ilogb(m) + 1 : 0;
  }
  const int nb_chk = std::min(n, 96), nr_chk = 300;
  std::vector<int64_t> rows_chk;
  for (int i = 0; i < nr_chk; ++i) rows_chk.push_back((int64_t(i) * 7919 + (i % 3) * 127) % R);
  rows_chk.push_back(R - 1);
  rows_chk.push_back(0);
  long mism = 0;
  double max_oz = 0.0, max_dd = 0.0, max_vs_dd = 0.0;
  std::vector<std::vector<int>> xd(nb_chk);
  std::vector<double> xs(nb_chk);
  std::vector<std::vector<double>> xv(nb_chk);
  std::vector<int> bsel(nb_chk);
  for (int bi = 0; bi < nb_chk; ++bi) {
    const int b = bi < 70 ? bi : n - 1 - (bi - 70);
    bsel[bi] = b;
    std::vector<double> v(k32, 0.0);
    xv[bi].assign(K + 32, 0.0);
    for (int kap = 0; kap < K; ++kap) {
      double x = 0.0;
      if (kap < Qb * Ne) {
        const int j = kap / Ne, k = kap % Ne;
        if (k < N) x = w[size_t(b) * (Qb + Ql) + j] * u[size_t(b) * N + k];
      } else if (kap - Qb * Ne < Ql)
        x = w[size_t(b) * (Qb + Ql) + Qb + kap - Qb * Ne];
      xv[bi][kap] = x;
      if (kap < kterms) v[kap] = std::ldexp(x, cexp[kap]);
    }
    xs[bi] = host_slice(v, xd[bi]);
  }
  for (int64_t r : rows_chk) {
    std::vector<double> v(k32, 0.0);
    for (int k = 0; k < kterms; ++k) v[k] = std::ldexp(S[size_t(r) * K + k], -cexp[k]);
    std::vector<int> sd;
    const double ss = host_slice(v, sd);
    for (int bi = 0; bi < nb_chk; ++bi) {
      long long acc[kS] = {0};
      for (int k = 0; k < k32; ++k)
        for (int i = 0; i < kS; ++i)
          for (int j = 0; j < kS - i; ++j) acc[i + j] += (long long)sd[k * kS + i] * xd[bi][k * kS + j];
      int a32[kS];
      for (int g = 0; g < kS; ++g) a32[g] = int(acc[g]);
      double emu = combine_groups(a32) * ss * xs[bi];
      for (int a = 0; a < Ql; ++a) emu = std::fma(xv[bi][kterms + a], S[size_t(r) * K + kterms + a], emu);
      const double got = out[size_t(bsel[bi]) * ldo + r];
      if (!(emu == got)) {
        if (mism < 10) std::printf("MISMATCH b=%d r=%lld got %.17g emu %.17g\n", bsel[bi], (long long)r, got, emu);
        ++mism;
      }
      long double ref = 0.0L, mag = 0.0L;
      double dd = 0.0;
      for (int k = 0; k < K; ++k) {
        ref += (long double)xv[bi][k] * (long double)S[size_t(r) * K + k];
        mag += fabsl((long double)xv[bi][k] * (long double)S[size_t(r) * K + k]);
        dd = std::fma(xv[bi][k], S[size_t(r) * K + k], dd);
      }
      if (mag > 0) {
        max_oz = std::fmax(max_oz, double(fabsl(got - ref) / mag));
        max_dd = std::fmax(max_dd, double(fabsl(dd - ref) / mag));
        max_vs_dd = std::fmax(max_vs_dd, std::fabs(got - dd) / double(mag));
      }
    }
  }
  std::printf("checked %d samples x %zu rows: %ld mismatches vs host emulation\n", nb_chk, rows_chk.size(), mism);
  std::printf("max |err| / sum|x||s|: sliced %.3e, binary64 fma dot %.3e, sliced vs dot %.3e\n", max_oz, max_dd, max_vs_dd);
  std::printf(mism == 0 ? "OK\n" : "FAILED\n");
  return mism == 0 ? 0 : 1;
}
