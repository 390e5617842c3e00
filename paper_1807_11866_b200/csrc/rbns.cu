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
}  // namespace

int rbns::set_last_error(int code, const std::string& msg) { return fail(code, msg); }

namespace {

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

// One contraction operand: S (rows × kalloc, L2-resident, TMA-streamed) and its weight descriptors.
struct Operand {
  CUtensorMap tm{};
  double* S = nullptr;
  int64_t rows = 0, row_tiles = 0;
  int kalloc = 0, nchunks = 0, nsub = 0;
  int Qb = 0, Ql = 0;                      // θ ⊗ u blocks, affine columns
  const rbns_theta_term* thb = nullptr;    // device descriptors
  const rbns_theta_term* thl = nullptr;
  int stages = 0;
  size_t smem = 0;
  oz::OperandI8 i8;                        // sliced copy for the tcgen05 INT8 path (A8 == NULL: DMMA only)
};

// per-call buffers of the INT8 path: the sliced X of one launch
struct OzScratch {
  uint8_t* B8 = nullptr;
  double* sb = nullptr;
};

struct rbns_model {
  int device = 0;
  int num_sms = 148;
  int N = 0, Np = 0, Ne = 0, ldu = 0;
  int Qa = 0, Qc = 0, Qf = 0, Qp = 0;      // family sizes: linear, quadratic, load, coupling
  int G = 0, ge[RBNS_MAX_GROUPS] = {};     // h groups and their μ₁ exponents
  int nu_lin = 0;
  int jl = 0;                              // J block layout the Newton kernels read (jidx)
  int n_stop = 0, stop_abs = 0;            // stop norm over the leading n_stop unknowns; absolute or relative
  Operand vel, prs, att;                   // velocity contraction, pressure coupling, attached pressure modes
  int n_att = 0;                           // rows of P_att (combined-scheme reconstruction), 0 = none
  cudaMemPool_t pool = nullptr;            // private stream-ordered pool of the per-call workspaces
  double* f = nullptr;                     // [Qf][N]
  double* L = nullptr;                     // [Np][Np]
  double* Lt = nullptr;                    // [Np][Np]
  rbns_theta_term* dth = nullptr;          // device descriptors: blocks | linear | load | coupling
  const rbns_theta_term* thf = nullptr;
  int rec_ok = 0;
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

int launch_contract(rbns_model* m, const Operand& op, const int32_t* act, int n, const double* u, const double* mu,
                    double* out, int64_t ldo, cudaStream_t st, bool linear_only = false,
                    const double* wts = nullptr, int64_t B = 0, const OzScratch* ozs = nullptr, int* launches = nullptr) {
  if (n <= 0) return RBNS_OK;
  if (launches) *launches = 1;
  if (op.i8.A8 && wts && ozs && ozs->B8) {
    // INT8-sliced path on the tcgen05 tensor cores (rbns_oz.cuh): X slicing + GEMM
    RBNS_CUDA(oz::launch(op.i8, act, n, u, wts, m->N, m->Ne, op.Qb, op.Ql, linear_only, ozs->B8, ozs->sb, out, ldo,
                         m->num_sms, st, B));
    if (launches) *launches = linear_only ? 1 : 2;
    return RBNS_OK;
  }
  ContractParams p{};
  p.act = act;
  p.n = n;
  p.u = u;
  p.mu = mu;
  p.N = m->N;
  p.Ne = m->Ne;
  p.Qb = op.Qb;
  p.Ql = op.Ql;
  p.nu_lin = m->nu_lin;
  p.thb = op.thb;
  p.thl = op.thl;
  p.nchunks = op.nchunks;
  p.nsub = op.nsub;
  p.sub_begin = linear_only ? (op.Qb * m->Ne) / 4 : 0;
  p.row_tiles = int(op.row_tiles);
  p.ldu_s = m->ldu;
  p.stages = op.stages;
  p.out = out;
  p.ldo = ldo;
  p.wts = wts;
  p.B = B;
  const int sample_tiles = (n + kBM - 1) / kBM;
  // target CTAs per SM over the launch (16 measured best at configs 1 and 2: 4, 8, 12, 16, 24, 32, 64 tried)
  static const int64_t waves = env_int64("RBNS_CONTRACT_WAVES", 16);
  const int64_t want = waves * m->num_sms;
  int groups = int(std::max<int64_t>(1, (want + sample_tiles - 1) / sample_tiles));
  static const int64_t min_tiles = std::max<int64_t>(1, env_int64("RBNS_CONTRACT_MIN_TILES", 4));  // per CTA
  groups = int(std::min<int64_t>(groups, std::max<int64_t>(1, (op.row_tiles + min_tiles - 1) / min_tiles)));
  p.tiles_per_group = int((op.row_tiles + groups - 1) / groups);
  groups = int((op.row_tiles + p.tiles_per_group - 1) / p.tiles_per_group);
  dim3 grid(sample_tiles, groups);
  kContract<<<grid, kContractThreads, op.smem, st>>>(op.tm, p);
  RBNS_CUDA(cudaGetLastError());
  return RBNS_OK;
}

NewtonParams newton_params(const rbns_model* m) {
  NewtonParams p{};
  p.f = m->f;
  p.thf = m->thf;
  p.N = m->N;
  p.Qf = m->Qf;
  p.G = m->G;
  for (int g = 0; g < RBNS_MAX_GROUPS; ++g) p.ge[g] = m->ge[g];
  p.n_stop = m->n_stop;
  p.stop_abs = m->stop_abs;
  p.jl = m->jl;
  p.num_sms = m->num_sms;
  return p;
}

int launch_newton(rbns_model* m, const int32_t* act, int n, const double* J, int64_t ldj, double* u,
                  const double* mu, int iter, int max_iter, double tol, int32_t* iters, int8_t* status, double* last,
                  int16_t* hints, int32_t* spec_miss, int32_t* miss_list, int32_t* miss_count, int* launches,
                  bool prefer_rank1, cudaStream_t st, const double* wf = nullptr, int64_t B = 0) {
  if (n <= 0) return RBNS_OK;
  NewtonParams p = newton_params(m);
  p.act = act;
  p.n = n;
  p.J = J;
  p.ldj = ldj;
  p.u = u;
  p.mu = mu;
  p.iter = iter;
  p.max_iter = max_iter;
  p.tol = tol;
  p.iters = iters;
  p.status = status;
  p.last = last;
  p.hint_in = iter > 1 ? hints : nullptr;  // the first iteration starts from the identity order
  p.hint_out = hints;
  p.spec_miss = spec_miss;
  p.miss_list = miss_list;
  p.miss_count = miss_count;
  p.prefer_rank1 = prefer_rank1 ? 1 : 0;
  p.wf = wf;
  p.B = B;
  RBNS_CUDA(launch_newton_update(p, st, launches));
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

// Per-call workspace: stream-ordered allocations from the handle's private pool (kept pooled between calls,
// released with the handle; the device's default pool is never touched) and events, freed on every exit path.
struct SolveWorkspace {
  cudaStream_t st;
  cudaMemPool_t pool;
  std::vector<void*> bufs;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  SolveWorkspace(cudaStream_t s, cudaMemPool_t p) : st(s), pool(p) {}
  template <class T>
  cudaError_t alloc(T** p, size_t bytes) {
    cudaError_t e = cudaMallocFromPoolAsync(reinterpret_cast<void**>(p), bytes, pool, st);
    if (e == cudaSuccess) bufs.push_back(*p);
    return e;
  }
  ~SolveWorkspace() {
    for (void* b : bufs) cudaFreeAsync(b, st);
    if (t0) cudaEventDestroy(t0);
    if (t1) cudaEventDestroy(t1);
  }
};

int recover(rbns_model* m, const double* mu, const double* u, int64_t B, double* p, int8_t* status, cudaStream_t st,
            rbns_stats& stats) {
  if (!m->Np) return fail(RBNS_ERR_NO_PRESSURE, "model has no pressure-recovery operators");
  const int64_t ldr = m->prs.row_tiles * kBN;
  const int64_t budget = env_int64("RBNS_RBUF_BYTES", int64_t(1) << 30);
  const int64_t cap = std::max<int64_t>(kBM, std::min<int64_t>(B, budget / (ldr * 8)));
  double* rbuf = nullptr;
  SolveWorkspace ws(st, m->pool);
  RBNS_CUDA(ws.alloc(&rbuf, size_t(cap) * ldr * sizeof(double)));
  const int cp = (m->Np + 31) / 32;
  int rc = RBNS_OK;
  for (int64_t c0 = 0; c0 < B && rc == RBNS_OK; c0 += cap) {
    const int nc = int(std::min<int64_t>(cap, B - c0));
    // identity ids for this chunk: contraction reads u/mu by id = c0 + i via offset pointers
    rc = launch_contract(m, m->prs, nullptr, nc, u + c0 * m->N, mu + 2 * c0, rbuf, ldr, st);
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
  return rc;
}

// Combined-scheme reconstruction p = P_att u: the contraction kernel with the one-block operand S = P_att
// (θ ≡ 1) into a tile-padded buffer, then the n_att leading columns of each row into p.
int reconstruct(rbns_model* m, const double* u, int64_t B, double* p, cudaStream_t st) {
  const int64_t ldr = m->att.row_tiles * kBN;
  const int64_t budget = env_int64("RBNS_RBUF_BYTES", int64_t(1) << 30);
  const int64_t cap = std::max<int64_t>(kBM, std::min<int64_t>(B, budget / (ldr * 8)));
  double* rbuf = nullptr;
  SolveWorkspace ws(st, m->pool);
  RBNS_CUDA(ws.alloc(&rbuf, size_t(cap) * ldr * sizeof(double)));
  int rc = RBNS_OK;
  for (int64_t c0 = 0; c0 < B && rc == RBNS_OK; c0 += cap) {
    const int nc = int(std::min<int64_t>(cap, B - c0));
    rc = launch_contract(m, m->att, nullptr, nc, u + c0 * m->N, nullptr, rbuf, ldr, st);
    if (rc) break;
    copy_leading<<<grid_for(int64_t(nc) * m->n_att, 256), 256, 0, st>>>(rbuf, ldr, nc, m->n_att, p + c0 * m->n_att);
    if (cudaGetLastError() != cudaSuccess) rc = fail(RBNS_ERR_CUDA, "copy_leading launch failed");
  }
  return rc;
}

int solve_device(rbns_model* m, const double* mu, int64_t B, double tol, int32_t max_iter, double* u, double* p,
                 int32_t* iters, int8_t* status, double* last, cudaStream_t st, rbns_stats* stats_out) {
  rbns_stats stats{};
  Timer timer(st);
  SolveWorkspace ws(st, m->pool);
  RBNS_CUDA(cudaEventCreate(&ws.t0));
  RBNS_CUDA(cudaEventCreate(&ws.t1));
  RBNS_CUDA(cudaEventRecord(ws.t0, st));

  const int64_t ldj = m->vel.row_tiles * kBN;
  int32_t *act0 = nullptr, *act1 = nullptr, *dcount = nullptr;
  int16_t* hints = nullptr;  // per-sample pivot order of the previous Newton iteration (speculation hint)
  RBNS_CUDA(ws.alloc(&act0, size_t(B) * sizeof(int32_t)));
  RBNS_CUDA(ws.alloc(&act1, size_t(B) * sizeof(int32_t)));
  RBNS_CUDA(ws.alloc(&dcount, 3 * sizeof(int32_t)));  // active count, hint misses, chunk misses
  RBNS_CUDA(ws.alloc(&hints, size_t(B) * m->N * sizeof(int16_t)));
  RBNS_CUDA(cudaMemsetAsync(dcount, 0, 3 * sizeof(int32_t), st));
  const int64_t budget = env_int64("RBNS_JBUF_BYTES", int64_t(8) << 30);
  const int64_t cap = std::max<int64_t>(kBM, std::min<int64_t>(B, budget / (ldj * 8)));
  int32_t* miss_list = nullptr;  // chunk positions whose pivot hint failed (re-run by the exact kernel)
  RBNS_CUDA(ws.alloc(&miss_list, size_t(std::max<int64_t>(1, std::min<int64_t>(B, cap))) * sizeof(int32_t)));
  double* jbuf = nullptr;
  if (max_iter > 0) RBNS_CUDA(ws.alloc(&jbuf, size_t(cap) * ldj * sizeof(double)));
  OzScratch ozs;
  if (max_iter > 0 && m->vel.i8.A8) {
    RBNS_CUDA(ws.alloc(&ozs.B8, oz::scratch_b8_bytes(m->vel.i8, cap)));
    RBNS_CUDA(ws.alloc(&ozs.sb, oz::scratch_sb_bytes(cap)));
  }
  static thread_local int32_t* hcount = nullptr;  // pinned, one per host thread for the process lifetime
  if (!hcount) RBNS_CUDA(cudaMallocHost(&hcount, 2 * sizeof(int32_t)));

  init_solve<<<grid_for(B, 256), 256, 0, st>>>(act0, status, iters, last, B);
  RBNS_CUDA(cudaGetLastError());
  // the contraction's θ weights, once per solve
  double* wts = nullptr;
  const int ldw = m->vel.Qb + m->vel.Ql;
  if (max_iter > 0) {
    RBNS_CUDA(ws.alloc(&wts, size_t(B) * ldw * sizeof(double)));
    eval_weights<<<grid_for(B * ldw, 256), 256, 0, st>>>(mu, B, m->vel.thb, m->vel.Qb, m->vel.thl, m->vel.Ql,
                                                        m->nu_lin, wts);
    RBNS_CUDA(cudaGetLastError());
    stats.kernel_launches += 1;
  }
  // ... and the Newton kernels' residual weights (load terms, group powers)
  double* wf = nullptr;
  const int ldf = m->Qf + m->G;
  if (max_iter > 0) {
    RBNS_CUDA(ws.alloc(&wf, size_t(B) * ldf * sizeof(double)));
    LoadWeightParams gp{};
    gp.G = m->G;
    for (int g = 0; g < RBNS_MAX_GROUPS; ++g) gp.ge[g] = m->ge[g];
    eval_load_weights<<<grid_for(B * ldf, 256), 256, 0, st>>>(mu, B, m->thf, m->Qf, gp, wf);
    RBNS_CUDA(cudaGetLastError());
    stats.kernel_launches += 1;
  }
  RBNS_CUDA(cudaMemsetAsync(u, 0, size_t(B) * m->N * sizeof(double), st));
  stats.kernel_launches += 1;

  int rc = RBNS_OK;
  int64_t n_act = B;
  // The blocked Newton kernel speculates the identity pivot order; once a round shows samples that need row
  // interchanges, the remaining rounds use the rank-1 kernel, whose speculation follows each sample's own
  // previous order (hints are written by both).
  bool prefer_rank1 = false;
  int32_t misses_seen = 0;
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
        // u = 0 at the first step: the convective part vanishes, only the affine block of the GEMM runs
        // (J = L(μ), h = 0); later steps run the full contraction
        const int e = timer.begin(first ? 3 : 0);
        int nl = 1;
        rc = launch_contract(m, m->vel, act0 + c0, nc, u, mu, jbuf, ldj, st, first, wts, B, &ozs, &nl);
        timer.end(e);
        if (rc) break;
        stats.gemm_launches += 1;
        stats.kernel_launches += nl;
      }
      const int e = timer.begin(1);
      int nl = 0;
      rc = launch_newton(m, act0 + c0, nc, jbuf, ldj, u, mu, it, max_iter, tol, iters, status, last, hints,
                         dcount + 1, miss_list, dcount + 2, &nl, prefer_rank1, st, wf, B);
      timer.end(e);
      if (rc) break;
      stats.lu_launches += nl;
      stats.kernel_launches += nl;
    }
    if (rc) break;
    compact_active<<<1, kCompactThreads, 0, st>>>(act0, int32_t(n_act), status, act1, dcount);
    stats.kernel_launches += 1;
    RBNS_CUDA(cudaGetLastError());
    RBNS_CUDA(cudaMemcpyAsync(hcount, dcount, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    RBNS_CUDA(cudaStreamSynchronize(st));
    if (int64_t(hcount[1] - misses_seen) * 64 > n_act) prefer_rank1 = true;  // > 1/64 of the round missed
    misses_seen = hcount[1];
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
  cudaEventRecord(ws.t1, st);
  if (rc == RBNS_OK) RBNS_CUDA(cudaMemcpyAsync(hcount + 1, dcount + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  cudaError_t se = cudaStreamSynchronize(st);
  if (rc == RBNS_OK && se != cudaSuccess) rc = fail(RBNS_ERR_CUDA, std::string("solve: ") + cudaGetErrorString(se));
  if (rc == RBNS_OK) {
    float tot = 0.f;
    cudaEventElapsedTime(&tot, ws.t0, ws.t1);
    stats.ms_total = tot;
    stats.ms_gemm = timer.total(0);
    stats.ms_lu = timer.total(1);
    stats.ms_recovery = timer.total(2);
    stats.ms_assembly = timer.total(3);
    stats.pivot_fallbacks = hcount[1];
    if (stats_out) *stats_out = stats;
    std::lock_guard<std::mutex> lk(m->stats_mu);
    m->stats = stats;
  }
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
    case RBNS_ERR_NO_ATTACHED: return "model has no attached pressure modes";
    default: return "unknown error";
  }
}

const char* rbns_last_error_message(void) { return g_last_error.c_str(); }

int rbns_model_create(const rbns_model_desc* d, int device, rbns_model** out) {
  if (!d || !out) return fail(RBNS_ERR_INVALID_ARGUMENT, "NULL descriptor/out");
  rbns_model_desc2 d2{};
  d2.n = d->n;
  d2.n_p = d->n_p;
  d2.flags = RBNS_NU_LINEAR;
  d2.linear = {d->q, 0, d->A, d->theta};
  d2.quadratic = {d->q, 0, d->C, d->theta};
  d2.load = {d->q, 0, d->f, d->theta};
  d2.coupling = {d->n_p > 0 ? d->q : 0, 0, d->Bq, d->theta};
  d2.Mp = d->Mp;
  return rbns_model_create2(&d2, device, out);
}

namespace {

bool valid_terms(const rbns_term_family& fam, bool need_data, const char* name, std::string& why) {
  if (fam.count < 0 || fam.count > RBNS_MAX_TERMS) {
    why = std::string(name) + ": count outside [0, " + std::to_string(RBNS_MAX_TERMS) + "]";
    return false;
  }
  if (fam.count > 0 && ((need_data && !fam.data) || !fam.theta)) {
    why = std::string(name) + ": NULL data/theta";
    return false;
  }
  for (int q = 0; q < fam.count; ++q) {
    const auto& t = fam.theta[q];
    if (t.kind < RBNS_THETA_CONST || t.kind > RBNS_THETA_MONOMIAL || t.k < 0 || t.m < 0 || !std::isfinite(t.scale)) {
      why = std::string(name) + ": bad theta descriptor " + std::to_string(q);
      return false;
    }
  }
  return true;
}

// θ_a(μ) == rho · μ₁^e · θ_c(μ) for every μ?  (same base function up to a constant and a power of μ₁)
bool tie(const rbns_theta_term& a, const rbns_theta_term& c, int& e, double& rho) {
  if (a.kind != c.kind || c.scale == 0.0) return false;
  e = 0;
  switch (a.kind) {
    case RBNS_THETA_CONST: break;
    case RBNS_THETA_COS_K:
    case RBNS_THETA_SIN_K:
      if (a.k != c.k) return false;
      break;
    case RBNS_THETA_COS_SIN_POW:
      if (a.k != c.k || a.m != c.m) return false;
      break;
    default:  // monomial μ₀^k μ₁^m
      if (a.k != c.k) return false;
      e = a.m - c.m;
      break;
  }
  rho = a.scale / c.scale;
  return std::isfinite(rho);
}

}  // namespace

int rbns_model_create2(const rbns_model_desc2* d, int device, rbns_model** out) {
  if (!d || !out) return fail(RBNS_ERR_INVALID_ARGUMENT, "NULL descriptor/out");
  *out = nullptr;
  std::string why;
  if (d->n < 1 || d->n_p < 0) return fail(RBNS_ERR_INVALID_ARGUMENT, "need N >= 1, Np >= 0");
  if (d->n_stop < 0 || d->n_stop > d->n) return fail(RBNS_ERR_INVALID_ARGUMENT, "n_stop outside [0, N]");
  if (!valid_terms(d->linear, true, "linear", why) || !valid_terms(d->quadratic, true, "quadratic", why) ||
      !valid_terms(d->load, true, "load", why) || !valid_terms(d->coupling, true, "coupling", why))
    return fail(RBNS_ERR_INVALID_ARGUMENT, why);
  if (d->linear.count < 1) return fail(RBNS_ERR_INVALID_ARGUMENT, "the linear family needs >= 1 term");
  if (d->n_p > 0 && (!d->Mp || d->coupling.count < 1))
    return fail(RBNS_ERR_INVALID_ARGUMENT, "Np > 0 needs Mp and >= 1 coupling term");
  if (d->n_p > 256) return fail(RBNS_ERR_UNSUPPORTED, "Np > 256");
  if (d->n_att < 0 || (d->n_att > 0 && !d->P_att))
    return fail(RBNS_ERR_INVALID_ARGUMENT, "attached pressure modes: n_att < 0 or NULL P_att");
  if (!newton_supported(d->n))
    return fail(RBNS_ERR_UNSUPPORTED, "N=" + std::to_string(d->n) + " exceeds the register-resident Newton kernel");
  int ndev = 0;
  RBNS_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(RBNS_ERR_INVALID_ARGUMENT, "bad device index");
  DeviceGuard guard(device);

  // ---- host planning: tie each linear term's h rows to a contraction block ----
  const int Qa = d->linear.count, Qc = d->quadratic.count;
  std::vector<rbns_theta_term> blocks(d->quadratic.theta, d->quadratic.theta + Qc);
  std::vector<int> hb(Qa), hg(Qa);
  std::vector<double> rho(Qa);
  std::vector<int> ge;
  const int nu_lin = (d->flags & RBNS_NU_LINEAR) ? 1 : 0;
  for (int a = 0; a < Qa; ++a) {
    const rbns_theta_term& ta = d->linear.theta[a];
    int e = 0, j = -1;
    double r = 1.0;
    for (int c = 0; c < int(blocks.size()) && j < 0; ++c)
      if (tie(ta, blocks[c], e, r)) j = c;
    if (j < 0) {  // no block carries this base function: an extra, velocity-free block
      if (int(blocks.size()) >= RBNS_MAX_TERMS) return fail(RBNS_ERR_UNSUPPORTED, "too many contraction blocks");
      blocks.push_back(ta);
      j = int(blocks.size()) - 1;
      e = 0;
      r = 1.0;
    }
    e -= nu_lin;  // ν = μ₁⁻¹ on the whole linear family
    int g = int(std::find(ge.begin(), ge.end(), e) - ge.begin());
    if (g == int(ge.size())) {
      if (int(ge.size()) >= RBNS_MAX_GROUPS)
        return fail(RBNS_ERR_UNSUPPORTED, "linear terms need more than RBNS_MAX_GROUPS distinct mu1 powers");
      ge.push_back(e);
    }
    hb[a] = j;
    hg[a] = g;
    rho[a] = r;
  }

  auto m = new rbns_model();
  m->device = device;
  cudaDeviceGetAttribute(&m->num_sms, cudaDevAttrMultiProcessorCount, device);
  m->N = d->n;
  m->Np = d->n_p;
  m->Qa = Qa;
  m->Qc = Qc;
  m->Qf = d->load.count;
  m->Qp = d->n_p > 0 ? d->coupling.count : 0;
  m->nu_lin = nu_lin;
  m->n_stop = d->n_stop > 0 ? d->n_stop : d->n;
  m->stop_abs = (d->flags & RBNS_STOP_ABSOLUTE) ? 1 : 0;
  m->G = int(ge.size());
  for (int g = 0; g < m->G; ++g) m->ge[g] = ge[g];
  m->Ne = (m->N + 3) / 4 * 4;  // κ stride per block (k4 sub-steps never straddle)
  m->jl = newton_layout(m->N);
  m->ldu = contract_ldu(m->Ne);
  auto cleanup = [&](int rc) {
    rbns_model_destroy(m);
    return rc;
  };
  int max_smem = 0;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  auto plan = [&](Operand& op, int64_t rows, int qb, int ql) {
    op.rows = rows;
    op.row_tiles = (rows + kBN - 1) / kBN;
    op.Qb = qb;
    op.Ql = ql;
    op.kalloc = qb * m->Ne + (ql + 3) / 4 * 4;
    op.nchunks = (op.kalloc + 4 * kKSub - 1) / (4 * kKSub);
    op.nsub = op.kalloc / 4;
#ifndef RBNS_STAGES
#define RBNS_STAGES 16
#endif
    op.stages = RBNS_STAGES;  // TMA ring depth (reduced below if shared memory is short)
    while (op.stages > 2 && contract_smem_bytes(op.stages, m->ldu, qb, ql) > size_t(max_smem)) --op.stages;
    op.smem = contract_smem_bytes(op.stages, m->ldu, qb, ql);
    return op.smem <= size_t(max_smem);
  };
  const int Qb = int(blocks.size());
  m->n_att = d->n_att > 0 ? d->n_att : 0;
  if (!plan(m->vel, int64_t(m->N) * m->N + int64_t(m->G) * m->N, Qb, Qa) ||
      (m->Np && !plan(m->prs, m->Np, m->Qp, 0)) || (m->n_att && !plan(m->att, m->n_att, 1, 0)))
    return cleanup(fail(RBNS_ERR_UNSUPPORTED, "contraction tile does not fit shared memory for N=" +
                                                  std::to_string(m->N)));
  // a per-function cap shared by every model: set it to the device maximum (not this model's size), so a
  // model created later with a smaller tile cannot invalidate launches of an earlier one
  if (cudaFuncSetAttribute(kContract, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem) != cudaSuccess)
    return cleanup(fail(RBNS_ERR_CUDA, "cudaFuncSetAttribute(contract) failed"));
  if (newton_prepare(m->N) != cudaSuccess) return cleanup(fail(RBNS_ERR_CUDA, "Newton kernel attributes failed"));

  // private stream-ordered pool for the per-call workspaces: allocations stay pooled between calls (no
  // re-allocation on the hot path) and are returned to the device when the handle is destroyed
  {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    if (cudaMemPoolCreate(&m->pool, &props) != cudaSuccess)
      return cleanup(fail(RBNS_ERR_CUDA, "cudaMemPoolCreate failed"));
    uint64_t thr = ~0ULL;
    cudaMemPoolSetAttribute(m->pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }

  auto step = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
      fail(e == cudaErrorMemoryAllocation ? RBNS_ERR_OUT_OF_MEMORY : RBNS_ERR_CUDA,
           std::string(what) + ": " + cudaGetErrorString(e));
      return false;
    }
    return true;
  };
  auto bad = [&]() {
    return cleanup(g_last_error.find("memory") != std::string::npos ? RBNS_ERR_OUT_OF_MEMORY : RBNS_ERR_CUDA);
  };
  // descriptors on the device: blocks | linear | load | coupling
  std::vector<rbns_theta_term> th(blocks);
  th.insert(th.end(), d->linear.theta, d->linear.theta + Qa);
  if (m->Qf) th.insert(th.end(), d->load.theta, d->load.theta + m->Qf);
  if (m->Qp) th.insert(th.end(), d->coupling.theta, d->coupling.theta + m->Qp);
  const rbns_theta_term one{RBNS_THETA_CONST, 0, 0, 0, 1.0};
  if (d->n_att > 0) th.push_back(one);  // the attached-mode operand: one block, θ ≡ 1
  if (!step(cudaMalloc(&m->dth, th.size() * sizeof(rbns_theta_term)), "cudaMalloc(theta)") ||
      !step(cudaMemcpy(m->dth, th.data(), th.size() * sizeof(rbns_theta_term), cudaMemcpyHostToDevice),
            "upload theta"))
    return bad();
  m->vel.thb = m->dth;
  m->vel.thl = m->dth + Qb;
  m->thf = m->dth + Qb + Qa;
  m->prs.thb = m->dth + Qb + Qa + m->Qf;
  m->att.thb = m->dth + Qb + Qa + m->Qf + m->Qp;

  const int64_t N = m->N;
  double *dC = nullptr, *dA = nullptr, *drho = nullptr;
  int *dhb = nullptr, *dhg = nullptr;
  const size_t cbytes = size_t(std::max(Qc, 1)) * N * N * N * sizeof(double);
  bool ok = step(cudaMalloc(&dC, cbytes), "cudaMalloc(C)") &&
            (Qc == 0 || step(cudaMemcpy(dC, d->quadratic.data, size_t(Qc) * N * N * N * sizeof(double),
                                        cudaMemcpyHostToDevice), "upload C")) &&
            step(cudaMalloc(&dA, size_t(Qa) * N * N * sizeof(double)), "cudaMalloc(A)") &&
            step(cudaMemcpy(dA, d->linear.data, size_t(Qa) * N * N * sizeof(double), cudaMemcpyHostToDevice),
                 "upload A") &&
            step(cudaMalloc(&dhb, Qa * sizeof(int)), "cudaMalloc(hb)") &&
            step(cudaMalloc(&dhg, Qa * sizeof(int)), "cudaMalloc(hg)") &&
            step(cudaMalloc(&drho, Qa * sizeof(double)), "cudaMalloc(rho)") &&
            step(cudaMemcpy(dhb, hb.data(), Qa * sizeof(int), cudaMemcpyHostToDevice), "upload hb") &&
            step(cudaMemcpy(dhg, hg.data(), Qa * sizeof(int), cudaMemcpyHostToDevice), "upload hg") &&
            step(cudaMemcpy(drho, rho.data(), Qa * sizeof(double), cudaMemcpyHostToDevice), "upload rho") &&
            step(cudaMalloc(&m->f, size_t(std::max(m->Qf, 1)) * N * sizeof(double)), "cudaMalloc(f)") &&
            (m->Qf == 0 || step(cudaMemcpy(m->f, d->load.data, size_t(m->Qf) * N * sizeof(double),
                                           cudaMemcpyHostToDevice), "upload f")) &&
            step(cudaMalloc(&m->vel.S, size_t(m->vel.rows) * m->vel.kalloc * sizeof(double)), "cudaMalloc(S)");
  if (ok) {
    build_velocity_operator<<<4 * m->num_sms, 256>>>(m->vel.S, m->vel.rows, m->vel.kalloc, dC, Qc, dA, Qa, dhb, dhg,
                                                     drho, m->N, m->Ne, Qb, m->jl);
    ok = step(cudaGetLastError(), "build_velocity_operator") && step(cudaDeviceSynchronize(), "build S");
  }
  for (void* ptr : {static_cast<void*>(dC), static_cast<void*>(dA), static_cast<void*>(dhb),
                    static_cast<void*>(dhg), static_cast<void*>(drho)})
    if (ptr) cudaFree(ptr);
  if (!ok) return bad();
  m->bytes = m->vel.rows * m->vel.kalloc * 8 + int64_t(m->Qf) * N * 8 + int64_t(th.size()) * 24;
  int rc = make_tensor_map(&m->vel.tm, m->vel.S, m->vel.rows, m->vel.kalloc);
  if (rc) return cleanup(rc);
  {
    // The velocity contraction runs on the tcgen05 INT8 tensor cores over error-free slices of S and X
    // (rbns_oz.cuh) unless RBNS_CONTRACT=dmma asks for the FP64 DMMA kernel (read per model create).
    const char* mode = std::getenv("RBNS_CONTRACT");
    const bool want_i8 = !(mode && std::string(mode) == "dmma");
    const int kterms = m->vel.Qb * m->Ne;
    if (want_i8 && oz::supported(kterms, m->vel.Ql, max_smem)) {
      if (!step(oz::prepare(), "oz::prepare") ||
          !step(oz::build_operand(m->vel.S, m->vel.rows, kterms, m->vel.kalloc, m->vel.Ql, &m->vel.i8), "slice S"))
        return bad();
      m->bytes += oz::operand_bytes(m->vel.i8);
    }
  }

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
    const int Qp = m->Qp;
    ok = step(cudaMalloc(&dB, size_t(Qp) * np * N * sizeof(double)), "cudaMalloc(Bq)") &&
         step(cudaMemcpy(dB, d->coupling.data, size_t(Qp) * np * N * sizeof(double), cudaMemcpyHostToDevice),
              "upload Bq") &&
         step(cudaMalloc(&m->prs.S, size_t(np) * m->prs.kalloc * sizeof(double)), "cudaMalloc(Sp)") &&
         step(cudaMalloc(&m->L, size_t(np) * np * sizeof(double)), "cudaMalloc(L)") &&
         step(cudaMalloc(&m->Lt, size_t(np) * np * sizeof(double)), "cudaMalloc(Lt)") &&
         step(cudaMemcpy(m->L, L.data(), size_t(np) * np * sizeof(double), cudaMemcpyHostToDevice), "upload L") &&
         step(cudaMemcpy(m->Lt, Lt.data(), size_t(np) * np * sizeof(double), cudaMemcpyHostToDevice), "upload Lt");
    if (ok) {
      build_pressure_operator<<<m->num_sms, 256>>>(m->prs.S, m->Np, m->prs.kalloc, dB, m->N, m->Ne, Qp);
      ok = step(cudaGetLastError(), "build_pressure_operator") && step(cudaDeviceSynchronize(), "build Sp");
    }
    if (dB) cudaFree(dB);
    if (!ok) return bad();
    rc = make_tensor_map(&m->prs.tm, m->prs.S, m->Np, m->prs.kalloc);
    if (rc) return cleanup(rc);
    m->bytes += np * m->prs.kalloc * 8 + 2 * np * np * 8;
  }
  if (m->n_att) {  // attached pressure modes: S_att[i][k] = P_att[i][k] (one block, θ ≡ 1)
    const int64_t na = m->n_att;
    double* dPa = nullptr;
    ok = step(cudaMalloc(&dPa, size_t(na) * N * sizeof(double)), "cudaMalloc(P_att)") &&
         step(cudaMemcpy(dPa, d->P_att, size_t(na) * N * sizeof(double), cudaMemcpyHostToDevice), "upload P_att") &&
         step(cudaMalloc(&m->att.S, size_t(na) * m->att.kalloc * sizeof(double)), "cudaMalloc(Satt)");
    if (ok) {
      build_pressure_operator<<<m->num_sms, 256>>>(m->att.S, m->n_att, m->att.kalloc, dPa, m->N, m->Ne, 1);
      ok = step(cudaGetLastError(), "build attached operator") && step(cudaDeviceSynchronize(), "build Satt");
    }
    if (dPa) cudaFree(dPa);
    if (!ok) return bad();
    rc = make_tensor_map(&m->att.tm, m->att.S, m->n_att, m->att.kalloc);
    if (rc) return cleanup(rc);
    m->bytes += na * m->att.kalloc * 8;
  }
  *out = m;
  return RBNS_OK;
}

int rbns_model_destroy(rbns_model* m) {
  if (!m) return RBNS_OK;
  DeviceGuard guard(m->device);
  for (void* p : {static_cast<void*>(m->vel.S), static_cast<void*>(m->prs.S), static_cast<void*>(m->att.S),
                  static_cast<void*>(m->f), static_cast<void*>(m->L), static_cast<void*>(m->Lt),
                  static_cast<void*>(m->dth)})
    if (p) cudaFree(p);
  oz::free_operand(&m->vel.i8);
  if (m->pool) cudaMemPoolDestroy(m->pool);  // every call has synchronized and freed its workspace
  delete m;
  return RBNS_OK;
}

int rbns_model_info(const rbns_model* m, int32_t* n, int32_t* q, int32_t* n_p, int32_t* device) {
  if (!m) return fail(RBNS_ERR_INVALID_ARGUMENT, "model is NULL");
  if (n) *n = m->N;
  if (q) *q = m->Qc;
  if (n_p) *n_p = m->Np;
  if (device) *device = m->device;
  return RBNS_OK;
}

int rbns_model_terms(const rbns_model* m, int32_t counts[6]) {
  if (!m || !counts) return fail(RBNS_ERR_INVALID_ARGUMENT, "NULL argument");
  counts[0] = m->Qa;
  counts[1] = m->Qc;
  counts[2] = m->Qf;
  counts[3] = m->Qp;
  counts[4] = m->vel.Qb;
  counts[5] = m->G;
  return RBNS_OK;
}

int64_t rbns_model_device_bytes(const rbns_model* m) { return m ? m->bytes : 0; }

int rbns_model_contraction_slices(const rbns_model* m) { return (m && m->vel.i8.A8) ? oz::slices() : 0; }

int rbns_get_stats(const rbns_model* m, rbns_stats* out) {
  if (!m || !out) return fail(RBNS_ERR_INVALID_ARGUMENT, "NULL argument");
  std::lock_guard<std::mutex> lk(const_cast<rbns_model*>(m)->stats_mu);
  *out = m->stats;
  return RBNS_OK;
}

int rbns_solve_ex(rbns_model* m, const double* mu, int64_t B, double tol, int32_t max_iter, double* u, double* p,
                  int32_t* iters, int8_t* status, double* last, rbns_stats* stats, void* stream) {
  int rc = check_solve_args(m, mu, B, tol, max_iter, u, iters, status, last);
  if (rc) return rc;
  if (p && !m->Np) return fail(RBNS_ERR_NO_PRESSURE, "pressure output requested but model has no Mp/Bq");
  if (stats) *stats = rbns_stats{};
  if (B == 0) return RBNS_OK;
  DeviceGuard guard(m->device);
  return solve_device(m, mu, B, tol, max_iter, u, p, iters, status, last, static_cast<cudaStream_t>(stream), stats);
}

int rbns_solve(rbns_model* m, const double* mu, int64_t B, double tol, int32_t max_iter, double* u, double* p,
               int32_t* iters, int8_t* status, double* last, void* stream) {
  return rbns_solve_ex(m, mu, B, tol, max_iter, u, p, iters, status, last, nullptr, stream);
}

int rbns_solve_host_ex(rbns_model* m, const double* mu, int64_t B, double tol, int32_t max_iter, double* u,
                       double* p, int32_t* iters, int8_t* status, double* last, rbns_stats* stats, void* stream) {
  int rc = check_solve_args(m, mu, B, tol, max_iter, u, iters, status, last);
  if (rc) return rc;
  if (p && !m->Np) return fail(RBNS_ERR_NO_PRESSURE, "pressure output requested but model has no Mp/Bq");
  if (stats) *stats = rbns_stats{};
  if (B == 0) return RBNS_OK;
  DeviceGuard guard(m->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double *dmu = nullptr, *du = nullptr, *dp = nullptr, *dl = nullptr;
  int32_t* di = nullptr;
  int8_t* ds = nullptr;
  const size_t N = m->N, np = m->Np;
  SolveWorkspace ws(st, m->pool);
  RBNS_CUDA(ws.alloc(&dmu, B * 2 * sizeof(double)));
  RBNS_CUDA(ws.alloc(&du, B * N * sizeof(double)));
  if (p) RBNS_CUDA(ws.alloc(&dp, B * np * sizeof(double)));
  RBNS_CUDA(ws.alloc(&dl, B * sizeof(double)));
  RBNS_CUDA(ws.alloc(&di, B * sizeof(int32_t)));
  RBNS_CUDA(ws.alloc(&ds, B * sizeof(int8_t)));
  RBNS_CUDA(cudaMemcpyAsync(dmu, mu, B * 2 * sizeof(double), cudaMemcpyHostToDevice, st));
  rc = solve_device(m, dmu, B, tol, max_iter, du, dp, di, ds, dl, st, stats);
  if (rc == RBNS_OK) {
    RBNS_CUDA(cudaMemcpyAsync(u, du, B * N * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (p) RBNS_CUDA(cudaMemcpyAsync(p, dp, B * np * sizeof(double), cudaMemcpyDeviceToHost, st));
    RBNS_CUDA(cudaMemcpyAsync(iters, di, B * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    RBNS_CUDA(cudaMemcpyAsync(status, ds, B * sizeof(int8_t), cudaMemcpyDeviceToHost, st));
    RBNS_CUDA(cudaMemcpyAsync(last, dl, B * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  cudaError_t se = cudaStreamSynchronize(st);
  if (rc == RBNS_OK && se != cudaSuccess) rc = fail(RBNS_ERR_CUDA, std::string("solve_host: ") + cudaGetErrorString(se));
  return rc;
}

int rbns_solve_host(rbns_model* m, const double* mu, int64_t B, double tol, int32_t max_iter, double* u, double* p,
                    int32_t* iters, int8_t* status, double* last, void* stream) {
  return rbns_solve_host_ex(m, mu, B, tol, max_iter, u, p, iters, status, last, nullptr, stream);
}

int rbns_reduced_operator(rbns_model* m, const double* mu, const double* eta, int64_t B, double* residual,
                          double* jacobian, void* stream) {
  if (!m || B < 0 || (B > 0 && (!mu || !eta || !residual || !jacobian)))
    return fail(RBNS_ERR_INVALID_ARGUMENT, "bad arguments to rbns_reduced_operator");
  if (B > (int64_t(1) << 31) - 1) return fail(RBNS_ERR_INVALID_ARGUMENT, "batch out of range");
  if (B == 0) return RBNS_OK;
  DeviceGuard guard(m->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t ldy = m->vel.row_tiles * kBN;
  const int64_t budget = env_int64("RBNS_JBUF_BYTES", int64_t(8) << 30);
  const int64_t cap = std::max<int64_t>(kBM, std::min<int64_t>(B, budget / (ldy * 8)));
  double* y = nullptr;
  SolveWorkspace ws(st, m->pool);
  RBNS_CUDA(ws.alloc(&y, size_t(cap) * ldy * sizeof(double)));
  const int64_t N = m->N;
  int rc = RBNS_OK;
  for (int64_t c0 = 0; c0 < B && rc == RBNS_OK; c0 += cap) {  // chunks of the Y buffer
    const int nc = int(std::min<int64_t>(cap, B - c0));
    rc = launch_contract(m, m->vel, nullptr, nc, eta + c0 * N, mu + 2 * c0, y, ldy, st);
    if (rc) break;
    NewtonParams np = newton_params(m);
    np.n = nc;
    np.mu = mu + 2 * c0;
    operator_readout<<<nc, 128, 0, st>>>(y, ldy, eta + c0 * N, np, residual + c0 * N, jacobian + c0 * N * N);
    if (cudaGetLastError() != cudaSuccess) rc = fail(RBNS_ERR_CUDA, "operator_readout launch failed");
  }
  cudaError_t se = cudaStreamSynchronize(st);
  if (rc == RBNS_OK && se != cudaSuccess) rc = fail(RBNS_ERR_CUDA, std::string("reduced_operator: ") + cudaGetErrorString(se));
  return rc;
}

int rbns_reconstruct_pressure(rbns_model* m, const double* u, int64_t B, double* p, void* stream) {
  if (!m || B < 0 || (B > 0 && (!u || !p))) return fail(RBNS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (!m->n_att) return fail(RBNS_ERR_NO_ATTACHED, "model carries no attached pressure modes (combined scheme)");
  if (B > (int64_t(1) << 31) - 1) return fail(RBNS_ERR_INVALID_ARGUMENT, "batch out of range");
  if (B == 0) return RBNS_OK;
  DeviceGuard guard(m->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = reconstruct(m, u, B, p, st);
  cudaError_t se = cudaStreamSynchronize(st);
  if (rc == RBNS_OK && se != cudaSuccess) rc = fail(RBNS_ERR_CUDA, std::string("reconstruct: ") + cudaGetErrorString(se));
  return rc;
}

int rbns_model_attached(const rbns_model* m, int32_t* n_att) {
  if (!m || !n_att) return fail(RBNS_ERR_INVALID_ARGUMENT, "NULL argument");
  *n_att = m->n_att;
  return RBNS_OK;
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

// Checked builds: failed device-side checks of every translation unit (line of the first failure, total count);
// 0 / 0 in the product build, where the checks compile away.  Not part of the public ABI (include/rbns.h).
extern "C" int rbns_debug_checks(int* line_main, int* line_newton, unsigned long long* count) {
  int ln = 0;
  unsigned long long cn = 0;
  if (rbns::newton_debug_checks(&ln, &cn)) return 2;
  {
    int lo = 0;  // the INT8 contraction's translation unit: folded into the main line / total count
    unsigned long long co = 0;
    if (rbns::oz::debug_checks(&lo, &co)) return 2;
    if (ln == 0) ln = lo;
    cn += co;
  }
#ifdef RBNS_CHECKED
  int lm = 0;
  unsigned long long cm = 0;
  if (cudaMemcpyFromSymbol(&lm, rbns::g_chk_line, sizeof(int)) != cudaSuccess ||
      cudaMemcpyFromSymbol(&cm, rbns::g_chk_count, sizeof(unsigned long long)) != cudaSuccess)
    return 2;
  *line_main = lm;
  *count = cm + cn;
#else
  *line_main = 0;
  *count = cn;
#endif
  *line_newton = ln;
  return 0;
}
