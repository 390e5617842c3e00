// rbns.cu — C-ABI implementation (include/rbns.h): model upload, the batched Newton driver and the launch
// glue around the sm_100a kernels in rbns_contract.cuh / rbns_newton.cuh / rbns_aux.cuh.
//
// Driver per call: init → for it = 1..max_iter { [it ≥ 2: contraction GEMM (K1+K2)] →
// Gauss–Jordan Newton update (K3) → stable compaction of the active set (K5) } → pressure recovery (K4).
// Everything is stream-ordered on the caller's stream; the host reads back one int (the active count) per
// Newton round to size the next grids.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "rbns.h"
#include "rbns_aux.cuh"
#include "rbns_common.cuh"
#include "rbns_contract.cuh"
#include "rbns_launch.h"
#include "rbns_newton.cuh"

using namespace rbns;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define RBNS_CUDA(call)                                                                                  \
  do {                                                                                                   \
    cudaError_t e_ = (call);                                                                             \
    if (e_ != cudaSuccess) {                                                                             \
      return fail(e_ == cudaErrorMemoryAllocation ? RBNS_ERR_OUT_OF_MEMORY : RBNS_ERR_CUDA,              \
                  std::string(#call) + ": " + cudaGetErrorString(e_) + " (" + __FILE__ + ":" +           \
                      std::to_string(__LINE__) + ")");                                                    \
    }                                                                                                    \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int make_tensor_map(CUtensorMap* tm, const double* base, int64_t rows, int64_t cols) {
  auto enc = tensor_map_encoder();
  if (!enc) return fail(RBNS_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(cols) * sizeof(double)};
  cuuint32_t box[2] = {4, cuuint32_t(kBN)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(RBNS_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return RBNS_OK;
}

// Dense Cholesky M = L Lᵀ on the host (one-time, Np ≤ a few hundred).  Returns false if not SPD.
bool host_cholesky(const double* M, int n, std::vector<double>& L) {
  L.assign(size_t(n) * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double d = M[size_t(j) * n + j];
    for (int k = 0; k < j; ++k) d -= L[size_t(j) * n + k] * L[size_t(j) * n + k];
    if (!(d > 0.0) || !std::isfinite(d)) return false;
    const double ljj = std::sqrt(d);
    L[size_t(j) * n + j] = ljj;
    for (int i = j + 1; i < n; ++i) {
      double s = M[size_t(i) * n + j];
      for (int k = 0; k < j; ++k) s -= L[size_t(i) * n + k] * L[size_t(j) * n + k];
      L[size_t(i) * n + j] = s / ljj;
    }
  }
  return true;
}

int64_t env_int64(const char* name, int64_t dflt) {
  const char* v = std::getenv(name);
  if (!v || !*v) return dflt;
  return std::strtoll(v, nullptr, 10);
}

}  // namespace

struct rbns_model {
  int device = 0;
  int num_sms = 148;
  int N = 0, Q = 0, Np = 0, Ne = 0, kalloc = 0, nchunks = 0, nsub = 0;
  int64_t R = 0, row_tiles = 0, rp_tiles = 0;
  double* S = nullptr;   // [R][kalloc]
  double* A = nullptr;   // [Q][N][N]
  double* f = nullptr;   // [Q][N]
  double* Sp = nullptr;  // [Np][kalloc]
  double* L = nullptr;   // [Np][Np]
  double* Lt = nullptr;  // [Np][Np]
  int rec_ok = 0;
  CUtensorMap tmS{}, tmSp{};
  ThetaDesc th{};
  int stages = 0, ldu = 0;
  size_t smem = 0;
  int64_t bytes = 0;
  rbns_stats stats{};
  std::mutex stats_mu;
};

namespace {

// -------------------------------------------------------------------------------------------------------
// launch helpers
// -------------------------------------------------------------------------------------------------------
using ContractKernel = void (*)(const CUtensorMap, const ContractParams);
constexpr ContractKernel kContract = contract_kernel<kBM, kBN, kWM, kWN>;

int launch_contract(rbns_model* m, const CUtensorMap& tm, int64_t row_tiles, const int32_t* act, int n,
                    const double* u, const double* mu, double* out, int64_t ldo, cudaStream_t st,
                    bool linear_only = false) {
  if (n <= 0) return RBNS_OK;
  ContractParams p{};
  p.act = act;
  p.n = n;
  p.u = u;
  p.mu = mu;
  p.N = m->N;
  p.Ne = m->Ne;
  p.Q = m->Q;
  p.nchunks = m->nchunks;
  p.nsub = m->nsub;
  p.sub_begin = linear_only ? (m->Q * m->Ne) / 4 : 0;
  p.row_tiles = int(row_tiles);
  p.ldu_s = m->ldu;
  p.stages = m->stages;
  p.out = out;
  p.ldo = ldo;
  p.th = m->th;
  const int sample_tiles = (n + kBM - 1) / kBM;
  const int64_t want = 8LL * m->num_sms;
  int groups = int(std::max<int64_t>(1, (want + sample_tiles - 1) / sample_tiles));
  groups = int(std::min<int64_t>(groups, std::max<int64_t>(1, (row_tiles + 3) / 4)));
  p.tiles_per_group = int((row_tiles + groups - 1) / groups);
  groups = int((row_tiles + p.tiles_per_group - 1) / p.tiles_per_group);
  dim3 grid(sample_tiles, groups);
  kContract<<<grid, kContractThreads, m->smem, st>>>(tm, p);
  RBNS_CUDA(cudaGetLastError());
  return RBNS_OK;
}

int launch_newton(rbns_model* m, const int32_t* act, int n, const double* J, int64_t ldj, double* u,
                  const double* mu, int first, int iter, int max_iter, double tol, int32_t* iters, int8_t* status,
                  double* last, cudaStream_t st) {
  if (n <= 0) return RBNS_OK;
  NewtonParams p{};
  p.act = act;
  p.n = n;
  p.J = J;
  p.ldj = ldj;
  p.u = u;
  p.mu = mu;
  p.A = m->A;
  p.f = m->f;
  p.N = m->N;
  p.Q = m->Q;
  p.first = first;
  p.iter = iter;
  p.max_iter = max_iter;
  p.tol = tol;
  p.iters = iters;
  p.status = status;
  p.last = last;
  p.th = m->th;
  RBNS_CUDA(launch_newton_update(p, st));
  return RBNS_OK;
}

int grid_for(int64_t n, int threads) {
  return int(std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 65535)));
}

struct EventPair {
  cudaEvent_t a = nullptr, b = nullptr;
  int kind = 0;  // 0 gemm, 1 lu, 2 recovery
};

struct Timer {
  std::vector<EventPair> ev;
  cudaStream_t st;
  explicit Timer(cudaStream_t s) : st(s) {}
  ~Timer() {
    for (auto& e : ev) {
      cudaEventDestroy(e.a);
      cudaEventDestroy(e.b);
    }
  }
  int begin(int kind) {
    EventPair e;
    e.kind = kind;
    cudaEventCreate(&e.a);
    cudaEventCreate(&e.b);
    cudaEventRecord(e.a, st);
    ev.push_back(e);
    return int(ev.size()) - 1;
  }
  void end(int idx) { cudaEventRecord(ev[idx].b, st); }
  double total(int kind) const {
    double s = 0.0;
    for (auto& e : ev)
      if (e.kind == kind) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, e.a, e.b) == cudaSuccess) s += ms;
      }
    return s;
  }
};

int recover(rbns_model* m, const double* mu, const double* u, int64_t B, double* p, int8_t* status, cudaStream_t st,
            rbns_stats& stats) {
  if (!m->Np) return fail(RBNS_ERR_NO_PRESSURE, "model has no pressure-recovery operators");
  const int64_t ldr = m->rp_tiles * kBN;
  const int64_t budget = env_int64("RBNS_RBUF_BYTES", int64_t(1) << 30);
  const int64_t cap = std::max<int64_t>(kBM, std::min<int64_t>(B, budget / (ldr * 8)));
  double* rbuf = nullptr;
  RBNS_CUDA(cudaMallocAsync(&rbuf, size_t(cap) * ldr * sizeof(double), st));
  const int cp = (m->Np + 31) / 32;
  int rc = RBNS_OK;
  for (int64_t c0 = 0; c0 < B && rc == RBNS_OK; c0 += cap) {
    const int nc = int(std::min<int64_t>(cap, B - c0));
    // identity ids for this chunk: contraction reads u/mu by id = c0 + i via offset pointers
    rc = launch_contract(m, m->tmSp, m->rp_tiles, nullptr, nc, u + c0 * m->N, mu + 2 * c0, rbuf, ldr, st);
    if (rc) break;
    stats.kernel_launches += 1;
    const int threads = 256, blocks = int((int64_t(nc) * 32 + threads - 1) / threads);
    int8_t* stc = status ? status + c0 : nullptr;
    double* pc = p + c0 * m->Np;
#define RBNS_TRI(CP_)                                                                                        \
  case CP_:                                                                                                  \
    pressure_trisolve<CP_><<<blocks, threads, 0, st>>>(rbuf, ldr, nc, m->L, m->Lt, m->Np, m->rec_ok, pc, stc, \
                                                       nullptr);                                             \
    break;
    switch (cp) {
      RBNS_TRI(1) RBNS_TRI(2) RBNS_TRI(3) RBNS_TRI(4) RBNS_TRI(5) RBNS_TRI(6) RBNS_TRI(7) RBNS_TRI(8)
      default:
        rc = fail(RBNS_ERR_UNSUPPORTED, "pressure dimension > 256 not supported");
    }
#undef RBNS_TRI
    if (rc) break;
    stats.kernel_launches += 1;
    if (cudaGetLastError() != cudaSuccess) rc = fail(RBNS_ERR_CUDA, "pressure_trisolve launch failed");
  }
  cudaFreeAsync(rbuf, st);
  return rc;
}

int solve_device(rbns_model* m, const double* mu, int64_t B, double tol, int32_t max_iter, double* u, double* p,
                 int32_t* iters, int8_t* status, double* last, cudaStream_t st) {
  rbns_stats stats{};
  Timer timer(st);
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  cudaEventRecord(t0, st);

  const int64_t ldj = m->row_tiles * kBN;
  int32_t *act0 = nullptr, *act1 = nullptr, *dcount = nullptr;
  RBNS_CUDA(cudaMallocAsync(&act0, size_t(B) * sizeof(int32_t), st));
  RBNS_CUDA(cudaMallocAsync(&act1, size_t(B) * sizeof(int32_t), st));
  RBNS_CUDA(cudaMallocAsync(&dcount, sizeof(int32_t), st));
  const int64_t budget = env_int64("RBNS_JBUF_BYTES", int64_t(8) << 30);
  const int64_t cap = std::max<int64_t>(kBM, std::min<int64_t>(B, budget / (ldj * 8)));
  double* jbuf = nullptr;
  if (max_iter > 0) RBNS_CUDA(cudaMallocAsync(&jbuf, size_t(cap) * ldj * sizeof(double), st));
  static thread_local int32_t* hcount = nullptr;
  if (!hcount) RBNS_CUDA(cudaMallocHost(&hcount, sizeof(int32_t)));

  init_solve<<<grid_for(B, 256), 256, 0, st>>>(act0, status, iters, last, B);
  RBNS_CUDA(cudaMemsetAsync(u, 0, size_t(B) * m->N * sizeof(double), st));
  stats.kernel_launches += 1;

  int rc = RBNS_OK;
  int64_t n_act = B;
  for (int it = 1; it <= max_iter && n_act > 0 && rc == RBNS_OK; ++it) {
    const int first = it == 1;
    stats.sample_iterations += n_act;
    if (!first) stats.contraction_iterations += n_act;
    stats.newton_rounds = it;
    const int64_t nchunk = (n_act + cap - 1) / cap;
    const int64_t csz = (n_act + nchunk - 1) / nchunk;
    for (int64_t c0 = 0; c0 < n_act && rc == RBNS_OK; c0 += csz) {
      const int nc = int(std::min<int64_t>(csz, n_act - c0));
      {
        // u = 0 at the first step: the convective part vanishes, only the ν θ_q A_q block of the GEMM runs
        // (J = ν A(μ), h = 0); later steps run the full contraction
        const int e = timer.begin(first ? 3 : 0);
        rc = launch_contract(m, m->tmS, m->row_tiles, act0 + c0, nc, u, mu, jbuf, ldj, st, first);
        timer.end(e);
        if (rc) break;
        stats.gemm_launches += 1;
        stats.kernel_launches += 1;
      }
      const int e = timer.begin(1);
      rc = launch_newton(m, act0 + c0, nc, jbuf, ldj, u, mu, 0, it, max_iter, tol, iters, status, last, st);
      timer.end(e);
      if (rc) break;
      stats.lu_launches += 1;
      stats.kernel_launches += 1;
    }
    if (rc) break;
    compact_active<<<1, kCompactThreads, 0, st>>>(act0, int32_t(n_act), status, act1, dcount);
    stats.kernel_launches += 1;
    RBNS_CUDA(cudaGetLastError());
    RBNS_CUDA(cudaMemcpyAsync(hcount, dcount, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    RBNS_CUDA(cudaStreamSynchronize(st));
    n_act = *hcount;
    std::swap(act0, act1);
  }
  if (rc == RBNS_OK) {
    finalize_solve<<<grid_for(B, 256), 256, 0, st>>>(status, B);
    stats.kernel_launches += 1;
    if (p) {
      const int e = timer.begin(2);
      rc = recover(m, mu, u, B, p, status, st, stats);
      timer.end(e);
    }
  }
  cudaEventRecord(t1, st);
  cudaFreeAsync(act0, st);
  cudaFreeAsync(act1, st);
  cudaFreeAsync(dcount, st);
  if (jbuf) cudaFreeAsync(jbuf, st);
  cudaError_t se = cudaStreamSynchronize(st);
  if (rc == RBNS_OK && se != cudaSuccess) rc = fail(RBNS_ERR_CUDA, std::string("solve: ") + cudaGetErrorString(se));
  if (rc == RBNS_OK) {
    float tot = 0.f;
    cudaEventElapsedTime(&tot, t0, t1);
    stats.ms_total = tot;
    stats.ms_gemm = timer.total(0);
    stats.ms_lu = timer.total(1);
    stats.ms_recovery = timer.total(2);
    stats.ms_assembly = timer.total(3);
    std::lock_guard<std::mutex> lk(m->stats_mu);
    m->stats = stats;
  }
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  return rc;
}

int check_solve_args(const rbns_model* m, const double* mu, int64_t B, double tol, int32_t max_iter, const double* u,
                     const int32_t* iters, const int8_t* status, const double* last) {
  if (!m) return fail(RBNS_ERR_INVALID_ARGUMENT, "model is NULL");
  if (B < 0 || B > (int64_t(1) << 31) - 1) return fail(RBNS_ERR_INVALID_ARGUMENT, "batch out of range");
  if (B > 0 && (!mu || !u || !iters || !status || !last))
    return fail(RBNS_ERR_INVALID_ARGUMENT, "NULL output/input buffer");
  if (!(tol >= 0.0) || max_iter < 0) return fail(RBNS_ERR_INVALID_ARGUMENT, "tol must be >= 0, max_iter >= 0");
  return RBNS_OK;
}

}  // namespace

// =========================================================================================================
// C ABI
// =========================================================================================================
extern "C" {

int rbns_abi_version(void) { return RBNS_ABI_VERSION; }

const char* rbns_error_string(int code) {
  switch (code) {
    case RBNS_OK: return "ok";
    case RBNS_ERR_INVALID_ARGUMENT: return "invalid argument";
    case RBNS_ERR_CUDA: return "CUDA error";
    case RBNS_ERR_OUT_OF_MEMORY: return "out of device memory";
    case RBNS_ERR_UNSUPPORTED: return "unsupported configuration";
    case RBNS_ERR_NO_PRESSURE: return "model has no pressure-recovery operators";
    default: return "unknown error";
  }
}

const char* rbns_last_error_message(void) { return g_last_error.c_str(); }

int rbns_model_create(const rbns_model_desc* d, int device, rbns_model** out) {
  if (!d || !out) return fail(RBNS_ERR_INVALID_ARGUMENT, "NULL descriptor/out");
  *out = nullptr;
  if (d->n < 1 || d->q < 1 || d->q > RBNS_MAX_TERMS || d->n_p < 0)
    return fail(RBNS_ERR_INVALID_ARGUMENT, "need N >= 1, 1 <= Q <= 16, Np >= 0");
  if (!d->A || !d->C || !d->f || !d->theta) return fail(RBNS_ERR_INVALID_ARGUMENT, "NULL operator pointer");
  if (d->n_p > 0 && (!d->Mp || !d->Bq)) return fail(RBNS_ERR_INVALID_ARGUMENT, "Np > 0 needs Mp and Bq");
  if (d->n_p > 256) return fail(RBNS_ERR_UNSUPPORTED, "Np > 256");
  for (int q = 0; q < d->q; ++q) {
    const auto& t = d->theta[q];
    if (t.kind < RBNS_THETA_CONST || t.kind > RBNS_THETA_MONOMIAL || t.k < 0 || t.m < 0)
      return fail(RBNS_ERR_INVALID_ARGUMENT, "bad theta descriptor " + std::to_string(q));
  }
  if (!newton_supported(d->n))
    return fail(RBNS_ERR_UNSUPPORTED, "N=" + std::to_string(d->n) + " exceeds the register-resident Newton kernel");
  int ndev = 0;
  RBNS_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(RBNS_ERR_INVALID_ARGUMENT, "bad device index");
  DeviceGuard guard(device);

  auto m = new rbns_model();
  m->device = device;
  cudaDeviceGetAttribute(&m->num_sms, cudaDevAttrMultiProcessorCount, device);
  m->N = d->n;
  m->Q = d->q;
  m->Np = d->n_p;
  m->Ne = (m->N + 3) / 4 * 4;                      // κ stride per affine term (k4 sub-steps never straddle)
  const int K = m->Q * m->Ne + (m->Q + 3) / 4 * 4;  // + the ν θ_q block
  m->kalloc = K;
  m->nchunks = (K + 7) / 8;
  m->nsub = K / 4;
  m->R = int64_t(m->N) * m->N + m->N;
  m->row_tiles = (m->R + kBN - 1) / kBN;
  m->rp_tiles = (m->Np + kBN - 1) / kBN;
  m->th.q = m->Q;
  for (int q = 0; q < m->Q; ++q) {
    m->th.kind[q] = d->theta[q].kind;
    m->th.k[q] = d->theta[q].k;
    m->th.m[q] = d->theta[q].m;
    m->th.scale[q] = d->theta[q].scale;
  }
  m->ldu = contract_ldu(m->Ne);
  int max_smem = 0;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  m->stages = 16;
  while (m->stages > 2 && contract_smem_bytes(m->stages, m->ldu, m->Q) > size_t(max_smem)) --m->stages;
  m->smem = contract_smem_bytes(m->stages, m->ldu, m->Q);
  auto cleanup = [&](int rc) {
    rbns_model_destroy(m);
    return rc;
  };
  if (m->smem > size_t(max_smem))
    return cleanup(fail(RBNS_ERR_UNSUPPORTED, "u tile does not fit shared memory for N=" + std::to_string(m->N)));
  // a per-function cap shared by every model: set it to the device maximum (not this model's size), so a
  // model created later with a smaller tile cannot invalidate launches of an earlier one
  if (cudaFuncSetAttribute(kContract, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem) != cudaSuccess)
    return cleanup(fail(RBNS_ERR_CUDA, "cudaFuncSetAttribute(contract) failed"));

  // keep freed stream-ordered allocations pooled (no re-allocation between calls)
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = ~0ULL;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }

  const int64_t N = m->N, Q = m->Q;
  const size_t cbytes = size_t(Q) * N * N * N * sizeof(double);
  double* dC = nullptr;
  if (cudaMalloc(&dC, cbytes) != cudaSuccess) return cleanup(fail(RBNS_ERR_OUT_OF_MEMORY, "cudaMalloc(C)"));
  auto step = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
      fail(e == cudaErrorMemoryAllocation ? RBNS_ERR_OUT_OF_MEMORY : RBNS_ERR_CUDA,
           std::string(what) + ": " + cudaGetErrorString(e));
      return false;
    }
    return true;
  };
  bool ok = step(cudaMemcpy(dC, d->C, cbytes, cudaMemcpyHostToDevice), "upload C") &&
            step(cudaMalloc(&m->A, size_t(Q) * N * N * sizeof(double)), "cudaMalloc(A)") &&
            step(cudaMemcpy(m->A, d->A, size_t(Q) * N * N * sizeof(double), cudaMemcpyHostToDevice), "upload A") &&
            step(cudaMalloc(&m->f, size_t(Q) * N * sizeof(double)), "cudaMalloc(f)") &&
            step(cudaMemcpy(m->f, d->f, size_t(Q) * N * sizeof(double), cudaMemcpyHostToDevice), "upload f") &&
            step(cudaMalloc(&m->S, size_t(m->R) * m->kalloc * sizeof(double)), "cudaMalloc(S)");
  if (ok) {
    build_velocity_operator<<<4 * m->num_sms, 256>>>(m->S, m->R, m->kalloc, dC, m->A, m->N, m->Ne, m->Q);
    ok = step(cudaGetLastError(), "build_velocity_operator") && step(cudaDeviceSynchronize(), "build S");
  }
  cudaFree(dC);
  if (!ok) return cleanup(g_last_error.find("memory") != std::string::npos ? RBNS_ERR_OUT_OF_MEMORY : RBNS_ERR_CUDA);
  m->bytes = int64_t(m->R) * m->kalloc * 8 + Q * N * N * 8 + Q * N * 8;
  int rc = make_tensor_map(&m->tmS, m->S, m->R, m->kalloc);
  if (rc) return cleanup(rc);

  if (m->Np) {
    const int64_t np = m->Np;
    std::vector<double> L;
    m->rec_ok = host_cholesky(d->Mp, m->Np, L) ? 1 : 0;
    std::vector<double> Lt(size_t(np) * np, 0.0);
    if (m->rec_ok)
      for (int64_t i = 0; i < np; ++i)
        for (int64_t j = 0; j < np; ++j) Lt[size_t(j) * np + i] = L[size_t(i) * np + j];
    else
      L.assign(size_t(np) * np, 0.0);
    double* dB = nullptr;
    ok = step(cudaMalloc(&dB, size_t(Q) * np * N * sizeof(double)), "cudaMalloc(Bq)") &&
         step(cudaMemcpy(dB, d->Bq, size_t(Q) * np * N * sizeof(double), cudaMemcpyHostToDevice), "upload Bq") &&
         step(cudaMalloc(&m->Sp, size_t(np) * m->kalloc * sizeof(double)), "cudaMalloc(Sp)") &&
         step(cudaMalloc(&m->L, size_t(np) * np * sizeof(double)), "cudaMalloc(L)") &&
         step(cudaMalloc(&m->Lt, size_t(np) * np * sizeof(double)), "cudaMalloc(Lt)") &&
         step(cudaMemcpy(m->L, L.data(), size_t(np) * np * sizeof(double), cudaMemcpyHostToDevice), "upload L") &&
         step(cudaMemcpy(m->Lt, Lt.data(), size_t(np) * np * sizeof(double), cudaMemcpyHostToDevice), "upload Lt");
    if (ok) {
      build_pressure_operator<<<m->num_sms, 256>>>(m->Sp, m->Np, m->kalloc, dB, m->N, m->Ne, m->Q);
      ok = step(cudaGetLastError(), "build_pressure_operator") && step(cudaDeviceSynchronize(), "build Sp");
    }
    if (dB) cudaFree(dB);
    if (!ok) return cleanup(RBNS_ERR_CUDA);
    rc = make_tensor_map(&m->tmSp, m->Sp, m->Np, m->kalloc);
    if (rc) return cleanup(rc);
    m->bytes += np * m->kalloc * 8 + 2 * np * np * 8;
  }
  *out = m;
  return RBNS_OK;
}

int rbns_model_destroy(rbns_model* m) {
  if (!m) return RBNS_OK;
  DeviceGuard guard(m->device);
  for (double* p : {m->S, m->A, m->f, m->Sp, m->L, m->Lt})
    if (p) cudaFree(p);
  delete m;
  return RBNS_OK;
}

int rbns_model_info(const rbns_model* m, int32_t* n, int32_t* q, int32_t* n_p, int32_t* device) {
  if (!m) return fail(RBNS_ERR_INVALID_ARGUMENT, "model is NULL");
  if (n) *n = m->N;
  if (q) *q = m->Q;
  if (n_p) *n_p = m->Np;
  if (device) *device = m->device;
  return RBNS_OK;
}

int64_t rbns_model_device_bytes(const rbns_model* m) { return m ? m->bytes : 0; }

int rbns_get_stats(const rbns_model* m, rbns_stats* out) {
  if (!m || !out) return fail(RBNS_ERR_INVALID_ARGUMENT, "NULL argument");
  std::lock_guard<std::mutex> lk(const_cast<rbns_model*>(m)->stats_mu);
  *out = m->stats;
  return RBNS_OK;
}

int rbns_solve(rbns_model* m, const double* mu, int64_t B, double tol, int32_t max_iter, double* u, double* p,
               int32_t* iters, int8_t* status, double* last, void* stream) {
  int rc = check_solve_args(m, mu, B, tol, max_iter, u, iters, status, last);
  if (rc) return rc;
  if (p && !m->Np) return fail(RBNS_ERR_NO_PRESSURE, "pressure output requested but model has no Mp/Bq");
  if (B == 0) return RBNS_OK;
  DeviceGuard guard(m->device);
  return solve_device(m, mu, B, tol, max_iter, u, p, iters, status, last, static_cast<cudaStream_t>(stream));
}

int rbns_solve_host(rbns_model* m, const double* mu, int64_t B, double tol, int32_t max_iter, double* u, double* p,
                    int32_t* iters, int8_t* status, double* last, void* stream) {
  int rc = check_solve_args(m, mu, B, tol, max_iter, u, iters, status, last);
  if (rc) return rc;
  if (p && !m->Np) return fail(RBNS_ERR_NO_PRESSURE, "pressure output requested but model has no Mp/Bq");
  if (B == 0) return RBNS_OK;
  DeviceGuard guard(m->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double *dmu = nullptr, *du = nullptr, *dp = nullptr, *dl = nullptr;
  int32_t* di = nullptr;
  int8_t* ds = nullptr;
  const size_t N = m->N, np = m->Np;
  RBNS_CUDA(cudaMallocAsync(&dmu, B * 2 * sizeof(double), st));
  RBNS_CUDA(cudaMallocAsync(&du, B * N * sizeof(double), st));
  if (p) RBNS_CUDA(cudaMallocAsync(&dp, B * np * sizeof(double), st));
  RBNS_CUDA(cudaMallocAsync(&dl, B * sizeof(double), st));
  RBNS_CUDA(cudaMallocAsync(&di, B * sizeof(int32_t), st));
  RBNS_CUDA(cudaMallocAsync(&ds, B * sizeof(int8_t), st));
  RBNS_CUDA(cudaMemcpyAsync(dmu, mu, B * 2 * sizeof(double), cudaMemcpyHostToDevice, st));
  rc = solve_device(m, dmu, B, tol, max_iter, du, dp, di, ds, dl, st);
  if (rc == RBNS_OK) {
    RBNS_CUDA(cudaMemcpyAsync(u, du, B * N * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (p) RBNS_CUDA(cudaMemcpyAsync(p, dp, B * np * sizeof(double), cudaMemcpyDeviceToHost, st));
    RBNS_CUDA(cudaMemcpyAsync(iters, di, B * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    RBNS_CUDA(cudaMemcpyAsync(status, ds, B * sizeof(int8_t), cudaMemcpyDeviceToHost, st));
    RBNS_CUDA(cudaMemcpyAsync(last, dl, B * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  for (void* ptr : {static_cast<void*>(dmu), static_cast<void*>(du), static_cast<void*>(dp), static_cast<void*>(dl),
                    static_cast<void*>(di), static_cast<void*>(ds)})
    if (ptr) cudaFreeAsync(ptr, st);
  cudaError_t se = cudaStreamSynchronize(st);
  if (rc == RBNS_OK && se != cudaSuccess) rc = fail(RBNS_ERR_CUDA, std::string("solve_host: ") + cudaGetErrorString(se));
  return rc;
}

int rbns_reduced_operator(rbns_model* m, const double* mu, const double* eta, int64_t B, double* residual,
                          double* jacobian, void* stream) {
  if (!m || B < 0 || (B > 0 && (!mu || !eta || !residual || !jacobian)))
    return fail(RBNS_ERR_INVALID_ARGUMENT, "bad arguments to rbns_reduced_operator");
  if (B == 0) return RBNS_OK;
  DeviceGuard guard(m->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t ldy = m->row_tiles * kBN;
  double* y = nullptr;
  RBNS_CUDA(cudaMallocAsync(&y, size_t(B) * ldy * sizeof(double), st));
  int rc = launch_contract(m, m->tmS, m->row_tiles, nullptr, int(B), eta, mu, y, ldy, st);
  if (rc == RBNS_OK) {
    operator_readout<<<int(B), 128, 0, st>>>(y, ldy, int(B), eta, mu, m->f, m->N, m->Q, m->th, residual, jacobian);
    if (cudaGetLastError() != cudaSuccess) rc = fail(RBNS_ERR_CUDA, "operator_readout launch failed");
  }
  cudaFreeAsync(y, st);
  cudaError_t se = cudaStreamSynchronize(st);
  if (rc == RBNS_OK && se != cudaSuccess) rc = fail(RBNS_ERR_CUDA, std::string("reduced_operator: ") + cudaGetErrorString(se));
  return rc;
}

int rbns_recover_pressure(rbns_model* m, const double* mu, const double* u, int64_t B, double* p, int8_t* status,
                          void* stream) {
  if (!m || B < 0 || (B > 0 && (!mu || !u || !p))) return fail(RBNS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (!m->Np) return fail(RBNS_ERR_NO_PRESSURE, "model has no pressure-recovery operators");
  if (B == 0) return RBNS_OK;
  DeviceGuard guard(m->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  rbns_stats stats{};
  int rc = recover(m, mu, u, B, p, status, st, stats);
  cudaError_t se = cudaStreamSynchronize(st);
  if (rc == RBNS_OK && se != cudaSuccess) rc = fail(RBNS_ERR_CUDA, std::string("recover: ") + cudaGetErrorString(se));
  return rc;
}

}  // extern "C"
