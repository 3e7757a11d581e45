// ttg.cu — host orchestration of the TT-ICE / TT-ICE* per-increment sweep on
// B200 (sm_100a) and the C ABI declared in include/ttg.h.
//
// The sweep restates the reference's Algorithm 1 / 2 loops
//   tt_ice_update_with_tolerances  tt_ice.cpp:60-129
//   tt_ice_star_update             tt_ice_star.cpp:171-303
//   tt_svd (bootstrap)             tt_svd.cpp:9-66
// as a sequence of device passes over the increment:
//   norms      per-observation |y_o|^2 and |Y|^2, fused into the first kernel that
//              streams Y (k_tiles_to_obs; k_sumsq_obs when tiles straddle observations)
//   gram       raw Gram C of the unfolding on DMMA (k_syrk_kx / k_syrk_kp / k_syrk2 +
//              k_gram_reduce); the residual Gram P C P is never streamed from HBM
//   decide     rank rule + kept directions + appended core in one launch (k_decide,
//              ttg_decide.cuh); fallbacks: explicit P C P (k_pcp / k_build_q + GEMMs) ->
//              k_syev_top / k_syev (+ k_sytrd_grid, k_syev_bt), explicit residual
//              (k_gram_resid), TSQR factor + k_jacobi_eig, tall side (k_tall_u), k_append
//   project    cur_{i+1} = reshape(U_new^T cur_i) (k_project_kc / k_project_ws, TMA + DMMA)
//   pad        next core zero-padded to the new left rank (k_pad_core)
// An update sweep is speculative (sweep()): launches after a k_decide mode are sized
// with the rank that mode kept at the previous update, the kernel flags any
// disagreement, and the host reads flag + per-mode results once per update.
// Multi-GPU: the batch (observation) axis is sharded; the a_i x a_i Grams and
// a handful of scalars are all-reduced and the coefficient columns
// all-gathered with NCCL; every rank then runs the same deterministic eigen
// solve on identical bytes.
#include <cudaTypedefs.h>
#include <nccl.h>

#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ttg.h"
#include "ttg_eig.cuh"
#include "ttg_kernels.cuh"
#include "ttg_misc.cuh"
#include "ttg_syev.cuh"
#include "ttg_io.cuh"
#include "ttg_gemm.cuh"
#include "ttg_decide.cuh"

namespace {

struct TtgError {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw TtgError{code, msg}; }

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess)                                                                      \
      fail(e_ == cudaErrorMemoryAllocation ? TTG_E_RESOURCE : TTG_E_CUDA,                       \
           std::string(#x) + ": " + cudaGetErrorString(e_));                                    \
  } while (0)

#define NK(x)                                                                                   \
  do {                                                                                          \
    ncclResult_t r_ = (x);                                                                      \
    if (r_ != ncclSuccess) fail(TTG_E_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_));   \
  } while (0)

// Workspaces come from the device's stream-ordered memory pool on the
// calling context's stream (no device-wide sync on growth; freed blocks stay
// cached in the pool).  g_alloc_stream is set at every ABI entry.
thread_local cudaStream_t g_alloc_stream = nullptr;

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), cap(o.cap) { o.p = nullptr; o.cap = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      cap = o.cap;
      o.p = nullptr;
      o.cap = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (p) {
      if (g_alloc_stream) cudaFreeAsync(p, g_alloc_stream);
      else cudaFree(p);
    }
    p = nullptr;
    cap = 0;
  }
  // grow-only (x2 headroom); keep=true preserves the old contents (stream-ordered)
  void ensure(size_t bytes, bool keep = false, cudaStream_t s = nullptr) {
    if (bytes <= cap) return;
    if (!s) s = g_alloc_stream;
    const size_t nc = std::max(bytes + bytes / 4, 2 * cap);
    void* np = nullptr;
    if (std::getenv("TTG_TRACE")) std::fprintf(stderr, "[ttg-trace] alloc %zu bytes (had %zu)\n", nc, cap);
    CK(cudaMallocAsync(&np, nc, s));
    if (keep && p) CK(cudaMemcpyAsync(np, p, cap, cudaMemcpyDeviceToDevice, s));
    if (p) CK(cudaFreeAsync(p, s));
    p = np;
    cap = nc;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

}  // namespace

struct ttg_ctx {
  int device = 0;
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  // host collectives (ttg_ctx_create_hostcoll) instead of NCCL when set
  ttg_host_allreduce_fn host_ar = nullptr;
  ttg_host_allgather_fn host_ag = nullptr;
  void* host_user = nullptr;
  std::vector<uint8_t> host_coll_buf;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // side stream: the interface Gram Phi^T Phi (one small CTA) runs beside the
  // statistics pass instead of after it
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;  // ordering against caller streams
  // ttg_prefetch: two staging slots filled on the copy stream
  struct Prefetch {
    DevBuf buf;
    const double* src = nullptr;
    int64_t n = 0;
    cudaEvent_t ready = nullptr, freed = nullptr;
    bool valid = false, used = false;
  } pf[2];
  cudaStream_t copy = nullptr;
  int pf_next = 0, pf_inuse = -1;
  DevBuf trd;  // k_sytrd_grid p, [d | e | tau], barrier
  std::string err;
  int64_t launches = 0;
  int num_sms = 148;
  size_t smem_optin = 232448;
  // workspaces (grow-only)
  DevBuf ystage, cur[2], partials, G, W, UR, lam, UTf, UTt, Uf, Upad, scratch, eigres, on2, sumsq_part,
      scal, coeffs, coeffs_all, cn2, cmc, errs, rn2, sel, stats, M, Mtmp, iface[2], tsq, psif, wcomb, psi[2],
      spsi[2], scoeffs, matbuf, tmp, Craw, small[4], gcount, gemm_ws, gemm_ws_side, iface_T, tallR, tallRg, tallXt,
      UR2, specflag, eiglog;
  std::vector<DevBuf> corebak;    // speculative sweeps: the cores a sweep replaces, kept until it is verified
  std::vector<DevBuf> scur;       // TT-ICE* stats-chain intermediates (reused by the sweep)
  std::vector<bool> stat_has;
  ttg::EigResult* h_eig = nullptr;
  ttg::EigResult* h_eiglog = nullptr;  // pinned: per-mode results of a speculative sweep + its flag
  int64_t spec_sweeps = 0, spec_redone = 0;
  bool spec_active = false;  // a speculative sweep has k_decide modes in flight (fetch_eig_result polls their flag)
  double* h_scal = nullptr;
  ttg::StarStats* h_stats = nullptr;
  // per-kernel accounting (launches, algorithmic bytes/flops always; event
  // time only while profiling is on)
  struct KStat {
    std::string name;
    int64_t launches = 0;
    double ms = 0.0, bytes = 0.0, flops = 0.0;
  };
  struct Pending {
    int idx;
    cudaEvent_t e0, e1;
  };
  bool profiling = false;
  uint64_t iface_gen = 0;
  const double* iface_ptr = nullptr;
  bool pdl = true;  // programmatic dependent launch (launch_k); off under TTG_NO_PDL and on NCCL contexts
  // exchange steps active: every NCCL context (world 1 included, so the single-GPU
  // test exercises the NCCL transport) and host-collective contexts with world > 1
  bool coll = false;
  std::vector<KStat> kstats;
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> evpool;
  int cur_idx = -1;
  cudaEvent_t cur_e0 = nullptr;
  int64_t h2d = 0, d2h = 0;
  bool shard_check = false;  // shard sizes ride on the next |Y|^2 all-reduce (global_obs)
};

struct ttg_tt {
  int d = 0;                       // spatial modes
  std::vector<int64_t> modes;      // n_1..n_d
  std::vector<int64_t> ranks;      // r_0..r_d (r_0 = 1)
  std::vector<DevBuf> cores;       // compact (r_{i-1} n_i) x r_i
  DevBuf last;                     // r_d x n_obs, ld = rc
  int64_t rc = 0, oc = 0, n_obs = 0;
  int64_t ortho_count = 0;
  std::vector<int64_t> bounds;
  // rank kept per mode at the previous update of THIS train (eig block-attempt
  // hint; per train, so a train's results never depend on other trains' history)
  std::vector<int> mode_hint;
  // speculative sweeps (ttg.cu sweep()): sweeps to sit out after a rejected guess, and its growth
  int spec_wait = 0, spec_hold = 0;
  std::vector<int> decide_off;  // per mode: sweeps for which k_decide is not tried (it did not converge last time)
  std::vector<int> hint_prev;  // mode_hint after the sweep before the last one
  int hint_repeats = 0;        // consecutive sweeps whose per-mode ranks repeated
  uint64_t gen = next_gen();  // bumped whenever the cores may change (caches keyed on it)
  static uint64_t next_gen() {
    static std::atomic<uint64_t> g{0};
    return ++g;
  }
};

namespace {

using ttg::EigResult;

// TTG_TRACE=1: host-side timeline of the update (wall clock, for stall hunting)
struct Trace {
  bool on = std::getenv("TTG_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), last = t0;
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[ttg-trace] %-28s +%8.3f ms (t=%8.3f)\n", what,
                 std::chrono::duration<double, std::milli>(now - last).count(),
                 std::chrono::duration<double, std::milli>(now - t0).count());
    last = now;
  }
};
thread_local Trace* g_trace = nullptr;
void trace(const char* w) {
  if (g_trace) g_trace->mark(w);
}

cudaEvent_t get_event(ttg_ctx* c) {
  if (!c->evpool.empty()) {
    cudaEvent_t e = c->evpool.back();
    c->evpool.pop_back();
    return e;
  }
  cudaEvent_t e;
  CK(cudaEventCreate(&e));
  return e;
}

// Every library kernel launch: programmatic stream serialization (PDL, see
// ttg_pdl.cuh) when enabled on the context and no per-kernel timing events
// sit between launches; errors surface in post_launch.
template <typename... KArgs, typename... Args>
void launch_k(ttg_ctx* c, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (c->pdl && !c->profiling) ? 1 : 0;
  CK(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// Call before every kernel launch: accounts the launch under `name` with its
// algorithmic bytes / flops and opens a timing event.
void prof_begin(ttg_ctx* c, const char* name, double bytes, double flops) {
  int idx = -1;
  for (size_t i = 0; i < c->kstats.size(); ++i)
    if (c->kstats[i].name == name) { idx = (int)i; break; }
  if (idx < 0) {
    c->kstats.push_back({name});
    idx = (int)c->kstats.size() - 1;
  }
  auto& st = c->kstats[idx];
  st.launches++;
  st.bytes += bytes;
  st.flops += flops;
  c->cur_idx = idx;
  if (c->profiling) {
    c->cur_e0 = get_event(c);
    CK(cudaEventRecord(c->cur_e0, c->stream));
  }
}

void post_launch(ttg_ctx* c) {
  ++c->launches;
  CK(cudaGetLastError());
  if (c->profiling && c->cur_idx >= 0) {
    cudaEvent_t e1 = get_event(c);
    CK(cudaEventRecord(e1, c->stream));
    c->pending.push_back({c->cur_idx, c->cur_e0, e1});
  }
  c->cur_idx = -1;
}

void prof_flush(ttg_ctx* c) {
  if (c->pending.empty()) return;
  CK(cudaStreamSynchronize(c->stream));
  for (auto& p : c->pending) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, p.e0, p.e1));
    c->kstats[p.idx].ms += ms;
    c->evpool.push_back(p.e0);
    c->evpool.push_back(p.e1);
  }
  c->pending.clear();
}

// per-block shared-memory limit of the current device (opt-in)
int prop_smem_optin() {
  static int v = [] {
    int dev = 0, x = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&x, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return x;
  }();
  return v;
}

// dynamic shared memory a kernel may still request (opt-in limit minus its static shared memory)
size_t dyn_smem_cap(const void* kern) {
  static std::vector<std::pair<const void*, size_t>> cache;
  for (const auto& e : cache)
    if (e.first == kern) return e.second;
  cudaFuncAttributes fa{};
  CK(cudaFuncGetAttributes(&fa, kern));
  const size_t cap = (size_t)prop_smem_optin() - fa.sharedSizeBytes;
  cache.push_back({kern, cap});
  return cap;
}

// cudaFuncSetAttribute / occupancy queries are driver calls: cache them per
// (kernel, dynamic smem) so the per-increment host path stays short.
template <class K>
int kernel_occupancy(const void* key, K kern, int threads, size_t smem) {
  struct Entry {
    const void* k;
    size_t smem;
    int occ;
  };
  static std::vector<Entry> cache;
  static std::vector<std::pair<const void*, size_t>> attr;
  for (const auto& e : cache)
    if (e.k == key && e.smem == smem) return e.occ;
  size_t have = 0;
  for (const auto& a : attr)
    if (a.first == key) have = a.second;
  if (smem > have) {
    cudaFuncAttributes fa{};
    CK(cudaFuncGetAttributes(&fa, kern));
    if (fa.sharedSizeBytes + smem > (size_t)prop_smem_optin())
      fail(TTG_E_RESOURCE, "kernel shared memory plan exceeds the per-block limit: dynamic " + std::to_string(smem) +
                               " + static " + std::to_string(fa.sharedSizeBytes) + " > " +
                               std::to_string(prop_smem_optin()) + " (" + std::to_string(threads) + " threads)");
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    bool found = false;
    for (auto& a : attr)
      if (a.first == key) { a.second = smem; found = true; }
    if (!found) attr.push_back({key, smem});
  }
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
  cache.push_back({key, smem, occ});
  return occ;
}

int grid_for(long long n, int threads, int max_blocks) {
  long long b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (int)b;
}

void allreduce_sum(ttg_ctx* c, double* d, size_t n) {
  if (!c->coll) return;
  if (c->host_ar) {  // host transport: D2H, exchange, H2D (stream-ordered)
    c->host_coll_buf.resize(sizeof(double) * n);
    double* h = reinterpret_cast<double*>(c->host_coll_buf.data());
    CK(cudaMemcpyAsync(h, d, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (c->host_ar(c->host_user, h, (int64_t)n) != 0) fail(TTG_E_NCCL, "host all-reduce failed");
    CK(cudaMemcpyAsync(d, h, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return;
  }
  NK(ncclAllReduce(d, d, n, ncclDouble, ncclSum, c->comm, c->stream));
}

// recv (world x n doubles, rank order) <- send (n doubles) from every rank
void allgather(ttg_ctx* c, const double* send, double* recv, size_t n) {
  if (c->host_ag) {
    std::vector<double> hs(n), hr(n * (size_t)c->world);
    CK(cudaMemcpyAsync(hs.data(), send, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (c->host_ag(c->host_user, hs.data(), (int64_t)(sizeof(double) * n), hr.data()) != 0)
      fail(TTG_E_NCCL, "host all-gather failed");
    CK(cudaMemcpyAsync(recv, hr.data(), sizeof(double) * n * c->world, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return;
  }
  NK(ncclAllGather(send, recv, n, ncclDouble, c->comm, c->stream));
}

// ---- norms ---------------------------------------------------------------
// per-observation |y_o|^2 -> c->on2 (b), total -> c->scal[0] (global)
void obs_norms(ttg_ctx* c, const double* Y, long long S, int b) {
  // (16 K doubles per CTA at most, and enough CTAs to fill the device several times over:
  // with 64 K-double chunks a 100-observation batch of 0.8 MB slabs ran on 200 CTAs at 2.4 TB/s)
  int nchunk = (int)std::max<long long>(1, std::min<long long>((S + 16383) / 16384,
                                                                (long long)c->num_sms * 16 / std::max(1, b) + 1));
  c->sumsq_part.ensure(sizeof(double) * (size_t)nchunk * b);
  c->on2.ensure(sizeof(double) * b);
  c->scal.ensure(sizeof(double) * 16);
  dim3 grid(nchunk, b);
  prof_begin(c, "k_sumsq_obs", 8.0 * S * b, 2.0 * S * b);
  launch_k(c, ttg::k_sumsq_obs, grid, 256, 0, Y, S, nchunk, c->sumsq_part.as<double>());
  post_launch(c);
  prof_begin(c, "k_sumsq_finalize", 8.0 * nchunk * b, 0.0);
  launch_k(c, ttg::k_sumsq_finalize, 1, 256, 0, c->sumsq_part.as<double>(), nchunk, b,
                                                   c->on2.as<double>(), c->scal.as<double>());
  post_launch(c);
  allreduce_sum(c, c->scal.as<double>(), 3);  // |Y|^2 and the shard-size check (global_obs)
}

// |Y|^2 (c->scal[0], all-reduced) to the host; on a sharded context also the
// all-reduced shard sizes (scal[1..2], see global_obs), checked here.
double read_scalar(ttg_ctx* c, const double* d) {
  const int n = c->coll ? 3 : 1;
  c->d2h += sizeof(double) * n;
  CK(cudaMemcpyAsync(c->h_scal, d, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (c->shard_check) {
    c->shard_check = false;
    const double s = c->h_scal[1], s2 = c->h_scal[2];
    if (s * s != s2 * c->world) fail(TTG_E_DIMENSION, "multi-GPU update needs the same batch shard size on every rank");
  }
  return c->h_scal[0];
}

// ---- fragments -------------------------------------------------------------
void make_frags(ttg_ctx* c, const double* U, int a, int r, int ld, bool need_ut, bool need_u) {
  int a8 = ttg::round_up(a, 8), r8 = ttg::round_up(r, 8);
  size_t n1 = (size_t)(r8 / 8) * (a8 / 4) * 32, n2 = (size_t)(a8 / 8) * (r8 / 4) * 32;
  c->UTf.ensure(sizeof(double) * std::max<size_t>(n1, 1));
  c->Uf.ensure(sizeof(double) * std::max<size_t>(n2, 1));
  prof_begin(c, "k_make_frags", 8.0 * (n1 + n2), 0.0);
  launch_k(c, ttg::k_make_frags, grid_for(n1 + n2, 256, 1024), 256, 0, 
      U, a, r, ld, a8, r8, need_ut ? c->UTf.as<double>() : nullptr, need_u ? c->Uf.as<double>() : nullptr);
  post_launch(c);
}

// ---- generic GEMM (any size) ------------------------------------------------
// C = alpha op(A) op(B) + beta C (column-major) on the DMMA GEMM (ttg_gemm.cuh):
// every plain GEMM of the sweep, small or large.  Few output tiles with a long
// k (R^T R, append Grams) split k over grid z with a fixed-order reduction.
// ws: split-k workspace (default c->gemm_ws; GEMMs on the side stream pass their own)
template <bool TA, bool TB>
void gemm(ttg_ctx* c, const double* A, long long lda, const double* B, long long ldb, double* C, long long ldc,
          long long m, long long n, long long k, double alpha, double beta, DevBuf* ws = nullptr) {
  if (m == 0 || n == 0) return;
  ttg::DgemmArgs a{A, lda, B, ldb, C, ldc, m, n, k, alpha, beta, 0, nullptr};
  const bool big = m > 64;
  const int bm = big ? 128 : 64;
  const long long tiles_m = (m + bm - 1) / bm, tiles_n = (n + ttg::kGemmBN - 1) / ttg::kGemmBN;
  if (tiles_m > 65535) fail(TTG_E_RESOURCE, "gemm: m too large");
  const long long tiles = tiles_m * tiles_n;
  const long long ksteps = (k + ttg::kGemmBK - 1) / ttg::kGemmBK;
  int nz = 1;
  if (tiles < 2LL * c->num_sms && ksteps >= 16) {
    nz = (int)std::min<long long>({(2LL * c->num_sms + tiles - 1) / tiles, ksteps / 8, 64});
    nz = std::max(nz, 1);
  }
  a.kchunk = ((ksteps + nz - 1) / nz) * ttg::kGemmBK;
  nz = (int)std::max<long long>(1, (k + a.kchunk - 1) / std::max<long long>(a.kchunk, 1));
  if (k == 0) a.kchunk = ttg::kGemmBK;
  if (nz > 1) {
    DevBuf& w = ws ? *ws : c->gemm_ws;
    w.ensure(sizeof(double) * (size_t)nz * m * n);
    a.ws = w.as<double>();
  }
  auto kern = big ? ttg::k_dgemm<TA, TB, 128> : ttg::k_dgemm<TA, TB, 64>;
  const size_t smem = big ? ttg::dgemm_smem<128>() : ttg::dgemm_smem<64>();
  kernel_occupancy((const void*)kern, kern, bm * 2, smem);
  char nm[64];
  std::snprintf(nm, sizeof nm, "k_dgemm[%c%c]", TA ? 'T' : 'N', TB ? 'T' : 'N');
  prof_begin(c, nm, 8.0 * (m * k + k * n + m * n), 2.0 * m * n * k);
  launch_k(c, kern, dim3((unsigned)tiles_n, (unsigned)tiles_m, (unsigned)nz), bm * 2, smem, a);
  post_launch(c);
  if (nz > 1) {
    prof_begin(c, "k_dgemm_reduce", 8.0 * (nz + 2.0) * m * n, (double)nz * m * n);
    launch_k(c, ttg::k_dgemm_reduce, grid_for(m * n, 256, 4 * c->num_sms), 256, 0, (const double*)a.ws, nz, m, n, C,
             ldc, alpha, beta);
    post_launch(c);
  }
}

constexpr int kFastMax = 128;  // a8 / r8 limit of the fused DMMA tiles
constexpr int kFastSkip = 2048;    // a from which the block subspace attempt (G in global memory) is skipped

// ---- residual Gram -----------------------------------------------------------
constexpr int kFastMax1 = 256;  // a8 limit of the single-buffered DMMA tiles

// fixed-order two-stage reduction of nx per-CTA partials into c->G (a x a)
void gram_reduce(ttg_ctx* c, int nx, int layout, int ld, int a, double* G) {
  const long long n = (long long)a * a;
  const int xs = std::max(1, std::min(32, nx / 8));
  c->Mtmp.ensure(sizeof(double) * (size_t)(xs * n));
  const int gxb = (int)std::min<long long>((n + 255) / 256, 1024);
  prof_begin(c, "k_gram_reduce", 8.0 * (double)nx * n / 2, (double)nx * n / 2);
  launch_k(c, ttg::k_gram_reduce_s1, dim3(gxb, xs), 256, 0, c->partials.as<double>(), nx, layout, ld, a,
                                                               c->Mtmp.as<double>());
  post_launch(c);
  prof_begin(c, "k_gram_reduce", 8.0 * (double)xs * n / 2, (double)xs * n / 2);
  launch_k(c, ttg::k_gram_reduce_s2, gxb, 256, 0, c->Mtmp.as<double>(), xs, a, G);
  post_launch(c);
}

template <int WBR, int WBC, bool PRE, bool DB>
void launch_gram_t(ttg_ctx* c, const ttg::GramArgs& args, size_t smem, int npairs) {
  auto kern = ttg::k_gram_resid<WBR, WBC, PRE, DB>;
  const int occ = kernel_occupancy((const void*)kern, kern, ttg::kThreads, smem);
  if (occ < 1) fail(TTG_E_RESOURCE, "gram kernel does not fit on an SM");
  long long want = std::max<long long>(1, (long long)c->num_sms * occ / npairs);
  int gx = (int)std::min<long long>(want, std::max<long long>(1, args.n_tiles));
  if (args.tsumsq) gx = (int)std::min<long long>((long long)c->num_sms * occ, std::max<long long>(1, args.n_tiles));
  constexpr int SBD = 8 * 4 * WBR;
  c->partials.ensure(sizeof(double) * (size_t)npairs * gx * SBD * SBD);
  ttg::GramArgs a2 = args;
  a2.partials = c->partials.as<double>();
  {
    const double Ls = (double)args.src.L * args.sel_frac;
    const double a_ = args.a, r_ = args.r_old;
    char nm[64];
    std::snprintf(nm, sizeof nm, "%s[a=%d,r=%d]", PRE ? "k_gram_resid_pre" : "k_gram_resid", args.a, args.r_old);
    prof_begin(c, nm, 8.0 * args.src.a * Ls, Ls * (4.0 * r_ * a_ + a_ * a_));
  }
  launch_k(c, kern, dim3(gx, npairs), ttg::kThreads, smem, a2);
  post_launch(c);
  const int a = args.a;
  const long long n = (long long)a * a;
  (void)n;
  gram_reduce(c, gx, 0, SBD, a, c->G.as<double>());
}

// The current unfolding cur_i (a_i x L_i) over a stored buffer:
//   cur_i = (I_n (x) Psi^T) (S viewed as (As*n) x (Ls/n)),   a_i = r*n, L_i = Ls/n.
// Psi == nullptr means identity (r == As): cur_i is S itself.  Mode 1 is
// {Y, As = 1, Ls = N}.  Keeping Psi pending instead of materialising cur_i
// lets mode i be read straight from the buffer of an earlier mode.
struct Src {
  const double* S = nullptr;
  int64_t As = 1, Ls = 0;
  const double* Psi = nullptr;
  int64_t r = 1;
};

// per-tile sums of squares are only usable when tiles never straddle observations
bool tiles_align(int64_t rows, int64_t obs_elems) { return obs_elems % (rows * ttg::kTC) == 0; }

// Fused residual Gram of cur_i into c->G.  `tsq` (nullable): per-tile sums of
// squares of the source tiles (only when the fast path runs; returns whether
// they were produced).
bool gram_src(ttg_ctx* c, const Src& s, int64_t n, const double* U, int r_old, const uint8_t* sel, long long cpo,
              double sel_frac, double* tsq) {
  const int a = (int)(s.r * n);
  const long long L = s.Ls / n;
  const int a8 = ttg::round_up(a, 8);
  const int r8 = r_old > 0 ? ttg::round_up(r_old, 8) : 0;
  c->G.ensure(sizeof(double) * (size_t)a * a);
  ttg::GramArgs args{};
  args.a = a;
  args.a8 = a8;
  args.r8 = r8;
  args.r_old = r_old;
  args.sel_frac = sel_frac;
  args.ldt = ttg::smem_ld(a8);
  args.ldp = ttg::smem_ld(std::max(r8, 8));
  args.n_tiles = (L + ttg::kTC - 1) / ttg::kTC;
  args.tsumsq = tsq;
  if (s.Psi) {
    const int src_rows = (int)(s.As * n);
    if (src_rows > kFastMax || a8 > kFastMax || r8 > kFastMax)
      fail(TTG_E_RESOURCE, "internal: pre-projected Gram outside the fast path");
    if (r_old > 0) make_frags(c, U, a, r_old, a, true, true);
    // Psi^T fragments into their own buffer
    const int As8 = ttg::round_up((int)s.As, 8), rc8 = ttg::round_up((int)s.r, 8);
    const size_t nf = (size_t)(rc8 / 8) * (As8 / 4) * 32;
    c->psif.ensure(sizeof(double) * nf);
    prof_begin(c, "k_make_frags", 8.0 * nf, 0.0);
    launch_k(c, ttg::k_make_frags, grid_for((long long)nf, 256, 1024), 256, 0, 
        s.Psi, (int)s.As, (int)s.r, (int)s.As, As8, rc8, c->psif.as<double>(), nullptr);
    post_launch(c);
    args.src = ttg::TileSrc{s.S, src_rows, L, sel, cpo};
    args.lds = ttg::smem_ld(src_rows + (As8 - (int)s.As) + 4);
    args.As = (int)s.As;
    args.nblk = (int)n;
    args.rc = (int)s.r;
    args.MRC = rc8 / 8;
    args.KS = As8 / 4;
    args.PsiTf = c->psif.as<double>();
    args.UTf = c->UTf.as<double>();
    args.Uf = c->Uf.as<double>();
    size_t smem = sizeof(double) * ((size_t)args.lds * ttg::kTC + (size_t)args.ldt * ttg::kTC +
                                    (size_t)8 * args.ldp * 8);
    const size_t nfr = (size_t)(r8 / 8) * (a8 / 4) * 32 + (size_t)(a8 / 8) * (r8 / 4) * 32 + nf;
    if (smem + sizeof(double) * nfr <= 110 * 1024) {  // keep 2 CTAs / SM
      args.frag_smem = 1;
      smem += sizeof(double) * nfr;
    }
    const int nb = a8 / 8;
    if (nb <= 4) launch_gram_t<1, 2, true, true>(c, args, smem, 1);
    else if (nb <= 8) launch_gram_t<2, 4, true, true>(c, args, smem, 1);
    else if (nb <= 12) launch_gram_t<3, 6, true, true>(c, args, smem, 1);
    else launch_gram_t<4, 8, true, true>(c, args, smem, 1);
    allreduce_sum(c, c->G.as<double>(), (size_t)a * a);
    return tsq != nullptr;
  }
  const double* X = s.S;
  args.src = ttg::TileSrc{X, a, L, sel, cpo};
  if (a8 <= kFastMax1 && r8 <= kFastMax) {
    if (r_old > 0) make_frags(c, U, a, r_old, a, true, true);
    args.UTf = c->UTf.as<double>();
    args.Uf = c->Uf.as<double>();
    const int nb = a8 / 8;
    const size_t nfr = (size_t)(r8 / 8) * (a8 / 4) * 32 + (size_t)(a8 / 8) * (r8 / 4) * 32;
    if (a8 <= kFastMax) {
      size_t smem = sizeof(double) * ((size_t)2 * args.ldt * ttg::kTC + (size_t)8 * args.ldp * 8);
      if (smem + sizeof(double) * nfr <= 200 * 1024) {
        args.frag_smem = 1;
        smem += sizeof(double) * nfr;
      }
      if (nb <= 4) launch_gram_t<1, 2, false, true>(c, args, smem, 1);
      else if (nb <= 8) launch_gram_t<2, 4, false, true>(c, args, smem, 1);
      else if (nb <= 12) launch_gram_t<3, 6, false, true>(c, args, smem, 1);
      else launch_gram_t<4, 8, false, true>(c, args, smem, 1);
    } else {
      const int ns = (nb + 15) / 16;
      size_t smem = sizeof(double) * ((size_t)args.ldt * ttg::kTC + (size_t)8 * args.ldp * 8);
      if (smem + sizeof(double) * nfr <= 200 * 1024) {
        args.frag_smem = 1;
        smem += sizeof(double) * nfr;
      }
      launch_gram_t<4, 8, false, false>(c, args, smem, ns * (ns + 1) / 2);
    }
    allreduce_sum(c, c->G.as<double>(), (size_t)a * a);
    return tsq != nullptr;
  }
  // generic: R = X - U (U^T X) materialised, masked, then G = R R^T
  c->scratch.ensure(sizeof(double) * (size_t)a * L);
  double* R = c->scratch.as<double>();
  CK(cudaMemcpyAsync(R, X, sizeof(double) * (size_t)a * L, cudaMemcpyDeviceToDevice, c->stream));
  if (r_old > 0) {
    c->W.ensure(sizeof(double) * (size_t)r_old * L);
    double* P = c->W.as<double>();
    gemm<true, false>(c, U, a, X, a, P, r_old, r_old, L, a, 1.0, 0.0);
    gemm<false, false>(c, U, a, P, r_old, R, a, a, L, r_old, -1.0, 1.0);
  }
  if (sel) {
    prof_begin(c, "k_mask_cols", 16.0 * a * L, 0.0);
    launch_k(c, ttg::k_mask_cols, grid_for((long long)a * L, 256, 4096), 256, 0, R, a, L, sel, cpo);
    post_launch(c);
  }
  gemm<false, true>(c, R, a, R, a, c->G.as<double>(), a, a, a, L, 1.0, 0.0);
  allreduce_sum(c, c->G.as<double>(), (size_t)a * a);
  return false;
}


// ---- raw Gram (SYRK) ---------------------------------------------------------
template <int MAXT, int NCW = ttg::kConsumerWarps>
void launch_syrk_t(ttg_ctx* c, ttg::SyrkArgs args, int npairs, double sel_frac) {
  constexpr int SBD = 128;
  const bool two = npairs > 1;  // some pairs carry two slices
  const size_t slice = sizeof(double) * (size_t)args.ldt * ttg::kTC;
  const size_t stage = (two ? 2 : 1) * slice;
  int nst;  // per-column TMA issue needs >= 3 issuing CTAs / SM to stream (tools/probe/stream_probe.cu)
  if (3 * 2 * stage <= 220 * 1024) nst = 2;
  else if (2 * 3 * stage <= 220 * 1024) nst = 3;
  else nst = (int)std::max<size_t>(1, std::min<size_t>(ttg::kMaxStages, (216 * 1024) / stage));
  if (const char* e = std::getenv("TTG_SYRK_NST")) {  // tuning override (kept only when it fits)
    const int want = std::atoi(e);
    if (want >= 1 && want <= ttg::kMaxStages && want * stage <= 220 * 1024) nst = want;
  }
  args.nst = nst;
  const size_t smem = nst * stage;
  auto kern = ttg::k_syrk<MAXT, NCW>;
  constexpr int threads = (NCW + 1) * 32;
  const int occ = std::max(1, kernel_occupancy((const void*)kern, kern, threads, smem));
  long long want = std::max<long long>(1, (long long)c->num_sms * occ / npairs);
  int gx = (int)std::min<long long>(want, std::max<long long>(1, args.n_tiles));
  c->partials.ensure(sizeof(double) * (size_t)npairs * gx * SBD * SBD);
  args.partials = c->partials.as<double>();
  char nm[64];
  std::snprintf(nm, sizeof nm, "k_syrk[a=%d]", args.a);
  const double Ls = (double)args.L * sel_frac;
  prof_begin(c, nm, 8.0 * args.a * Ls, Ls * (double)args.a * args.a);
  launch_k(c, kern, dim3(gx, npairs), threads, smem, args);
  post_launch(c);
  const int a = args.a;
  const long long n = (long long)a * a;
  (void)n;
  gram_reduce(c, gx, 0, SBD, a, c->G.as<double>());
}

// 2-D tensor map of X (a x L, column-major) with 16 x 64 boxes and 128-byte
// swizzle (ttg_kernels.cuh, "Tensor-map TMA tiles").  The driver entry point
// is resolved once through the runtime (no -lcuda).  False when the operand
// does not qualify (odd a, misaligned base, L beyond int32 coordinates).
bool make_tmap(CUtensorMap* m, const double* X, int a, long long L, int box_cols = ttg::kTC) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  static bool resolved = false;
  if (!resolved) {
    resolved = true;
    cudaDriverEntryPointQueryResult q{};
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    else
      cudaGetLastError();
  }
  if (!enc || (a & 1) || a <= 0 || L <= 0 || L >= (1LL << 31) || (reinterpret_cast<uintptr_t>(X) & 15)) return false;
  cuuint64_t dims[2] = {(cuuint64_t)a, (cuuint64_t)L};
  cuuint64_t strides[1] = {(cuuint64_t)a * sizeof(double)};
  cuuint32_t box[2] = {16, (cuuint32_t)box_cols};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(X), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Tensor-map SYRK (k_syrk2) into c->G; false when the operand does not
// qualify (odd a, a > 256, selection not tile-aligned, fewer than two ring
// stages fit) and the caller takes the per-column path.
template <int MAXT>
void launch_syrk2_t(ttg_ctx* c, const CUtensorMap& tm, ttg::Syrk2Args args, int parts, size_t smem, double sel_frac) {
  auto kern = ttg::k_syrk2<MAXT>;
  const int occ = std::max(1, kernel_occupancy((const void*)kern, kern, ttg::kSyrkThreads, smem));
  const long long want = std::max<long long>(1, (long long)c->num_sms * occ / parts);
  const int gx = (int)std::min<long long>(want, std::max<long long>(1, args.n_tiles));
  c->partials.ensure(sizeof(double) * (size_t)gx * args.a8 * args.a8);
  args.partials = c->partials.as<double>();
  char nm[64];
  std::snprintf(nm, sizeof nm, "k_syrk[a=%d]", args.a);
  const double Ls = (double)args.L * sel_frac;
  prof_begin(c, nm, 8.0 * args.a * Ls, Ls * (double)args.a * args.a);
  launch_k(c, kern, dim3(gx, parts), ttg::kSyrkThreads, smem, tm, args);
  post_launch(c);
  const long long n = (long long)args.a * args.a;
  (void)n;
  gram_reduce(c, gx, 1, args.a8, args.a, c->G.as<double>());
}

// Warp-specialised m16n8k16 SYRK (k_syrk_ws16) for even a <= 128 into c->G.
template <int NCW, int MAXG>
void launch_syrk_ws16_t(ttg_ctx* c, const CUtensorMap& tm, ttg::Syrk2Args args, double sel_frac) {
  auto kern = ttg::k_syrk_ws16<NCW, MAXG>;
  constexpr int threads = (NCW + 1) * 32;
  const size_t stage = sizeof(double) * 1024 * args.nbox;
  const size_t cap = (size_t)c->smem_optin - 1024;
  // stages: as many as fit ~110 KB when two CTAs fit by registers, else up
  // to four in one CTA
  int regs_ok2 = 0;
  {
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, kern));
    regs_ok2 = (2 * threads * fa.numRegs <= 65536) ? 1 : 0;
  }
  const size_t per_cta = regs_ok2 ? 110 * 1024 : cap;
  int nst = 2;
  while (nst < ttg::kMaxStages && (nst + 1) * stage + 1024 <= per_cta) ++nst;
  if (std::getenv("TTG_SYRK16_NST")) {  // tuning override (ignored when it does not fit)
    const int want = std::atoi(std::getenv("TTG_SYRK16_NST"));
    if (want >= 2 && want <= ttg::kMaxStages + 4 && want * stage + 1024 <= cap) nst = want;
  }
  args.nst = nst;
  const size_t smem = nst * stage + 1024;
  const int occ = std::max(1, kernel_occupancy((const void*)kern, kern, threads, smem));
  const int gx = (int)std::min<long long>((long long)c->num_sms * occ, std::max<long long>(1, args.n_tiles));
  c->partials.ensure(sizeof(double) * (size_t)gx * args.a8 * args.a8);
  args.partials = c->partials.as<double>();
  char nm[64];
  std::snprintf(nm, sizeof nm, "k_syrk[a=%d]", args.a);
  const double Ls = (double)args.L * sel_frac;
  prof_begin(c, nm, 8.0 * args.a * Ls, Ls * (double)args.a * args.a);
  launch_k(c, kern, gx, threads, smem, tm, args);
  post_launch(c);
  const long long n = (long long)args.a * args.a;
  (void)n;
  gram_reduce(c, gx, 1, args.a8, args.a, c->G.as<double>());
}

bool syrk_ws16(ttg_ctx* c, const double* X, int a, long long L, const uint8_t* sel, long long cpo, double sel_frac,
               double* tsq) {
  // measured: the per-column super-tile kernel is faster up to a = 96 (a = 64:
  // 1.65 vs 1.74 ms per 4.3 GB), this one from a = 112 to 128
  if (std::getenv("TTG_NO_SYRK16") || (a & 1) || a <= 96 || a > 128 || (sel && cpo % ttg::kTC != 0)) return false;
  CUtensorMap tm;
  if (!make_tmap(&tm, X, a, L)) return false;
  const int nks = (a + 15) / 16;
  if (2 * sizeof(double) * 1024 * nks + 1024 > (size_t)c->smem_optin - 1024) return false;
  ttg::Syrk2Args args{};
  args.a = a;
  args.a8 = ttg::round_up(a, 8);
  args.nbox = nks;
  args.L = L;
  args.n_tiles = (L + ttg::kTC - 1) / ttg::kTC;
  args.sel = sel;
  args.cpo = cpo;
  args.tsumsq = tsq;
  // consumer warps x groups per warp = the nks (nks + 1) / 2 lower groups, balanced
  switch (nks) {
    case 1: launch_syrk_ws16_t<1, 1>(c, tm, args, sel_frac); break;
    case 2: launch_syrk_ws16_t<3, 1>(c, tm, args, sel_frac); break;
    case 3: launch_syrk_ws16_t<6, 1>(c, tm, args, sel_frac); break;
    case 4: launch_syrk_ws16_t<10, 1>(c, tm, args, sel_frac); break;
    case 5: launch_syrk_ws16_t<5, 3>(c, tm, args, sel_frac); break;
    case 6: launch_syrk_ws16_t<7, 3>(c, tm, args, sel_frac); break;
    case 7: launch_syrk_ws16_t<14, 2>(c, tm, args, sel_frac); break;
    default: launch_syrk_ws16_t<12, 3>(c, tm, args, sel_frac); break;
  }
  return true;
}

bool syrk2(ttg_ctx* c, const double* X, int a, long long L, const uint8_t* sel, long long cpo, double sel_frac,
           double* tsq) {
  // a <= 128: the per-column super-tile kernel (k_syrk) measures faster (one
  // super-tile, 3 CTAs / SM at a = 64); the tensor-map kernel wins above,
  // where k_syrk splits rows into super-tile pairs and re-reads them.
  if (std::getenv("TTG_NO_SYRK2") || (a & 1) || a <= 128 || a > 256 || (sel && cpo % ttg::kTC != 0)) return false;
  CUtensorMap tm;
  if (!make_tmap(&tm, X, a, L)) return false;
  const int a8 = ttg::round_up(a, 8), nb = a8 / 8, tI = (nb + 1) / 2;
  const int nbox = (a + 15) / 16;
  const size_t stage = sizeof(double) * 1024 * nbox;
  const size_t cap = (size_t)c->smem_optin - 1024;
  // ring: 4 stages when two CTAs fit, else as many as fit one CTA (>= 2)
  int nst = 4;
  while (nst > 2 && 2 * (nst * stage + 1024) > 220 * 1024) --nst;
  if (nst * stage + 1024 > cap) {
    nst = (int)std::min<size_t>(ttg::kMaxStages, (cap - 1024) / stage);
    if (nst < 2) return false;
  }
  ttg::Syrk2Args args{};
  args.a = a;
  args.a8 = a8;
  args.nbox = nbox;
  args.nst = nst;
  args.L = L;
  args.n_tiles = (L + ttg::kTC - 1) / ttg::kTC;
  args.sel = sel;
  args.cpo = cpo;
  args.ntiles2 = tI * (tI + 1) / 2;
  args.tsumsq = tsq;
  const size_t smem = nst * stage + 1024;
  const int nt = args.ntiles2;
  if (nt <= 8) launch_syrk2_t<1>(c, tm, args, 1, smem, sel_frac);
  else if (nt <= 16) launch_syrk2_t<2>(c, tm, args, 1, smem, sel_frac);
  else launch_syrk2_t<3>(c, tm, args, (nt + 23) / 24, smem, sel_frac);
  return true;
}

// k-split SYRK for 64 < a8 <= 160 (k_syrk_kp): parts P per NBK so that a warp
// holds at most 40 lower blocks
constexpr int kp_nbl(int nbk) { return nbk * (nbk + 1) / 2; }
// parts per CTA: a warp holds at most 40-44 lower blocks
constexpr int kp_parts(int nbk) {
  return kp_nbl(nbk) <= 40 ? 1 : (kp_nbl(nbk) + 1) / 2 <= 40 ? 2 : 4;
}
// CTAs per tile set
constexpr int kp_py(int nbk) {
  return kp_parts(nbk) < 4 ? 1 : (kp_nbl(nbk) + 4 * 44 - 1) / (4 * 44);
}
template <int NBK>
void* kp_kernel() {
  return (void*)ttg::k_syrk_kp<NBK, kp_parts(NBK), kp_py(NBK)>;
}
constexpr int kKpMaxNbk = 28;
template <int NBK>
void* kp_pick_t(int nbk) {
  if constexpr (NBK > kKpMaxNbk) {
    return nullptr;
  } else {
    return nbk == NBK ? kp_kernel<NBK>() : kp_pick_t<NBK + 1>(nbk);
  }
}
void* kp_pick(int nbk) { return nbk >= 7 ? kp_pick_t<7>(nbk) : nullptr; }

bool syrk_kp(ttg_ctx* c, const double* X, int a, long long L, const uint8_t* sel, long long cpo, double sel_frac,
             double* tsq) {
  const int a8 = ttg::round_up(a, 8), nbk = a8 / 8;
  // measured: 8 warp-parts per CTA re-load too many fragments per DMMA and
  // lose to k_syrk2; up to 4 parts win (a = 136: 0.16 vs 0.24 ms per 1.1 GB);
  // larger triangles add CTAs per tile set (kp_py) instead
  if (std::getenv("TTG_NO_KP") || tsq || (a & 1) || nbk < (std::getenv("TTG_KP8") ? 7 : 9) || nbk > kKpMaxNbk ||
      (sel && cpo % ttg::kTC != 0))
    return false;
  CUtensorMap tm;
  if (!make_tmap(&tm, X, a, L)) return false;
  const size_t stage = sizeof(double) * 1024 * (size_t)((nbk + 1) / 2);
  const size_t cap = (size_t)c->smem_optin - 1024;
  int nst = (int)std::min<size_t>(6, (cap - 1024) / stage);
  if (const char* e = std::getenv("TTG_KP_NST")) nst = std::min(nst, std::max(2, std::atoi(e)));
  if (nst < 2) return false;
  ttg::SyrkArgs args{};
  args.X = X;
  args.a = a;
  args.a8 = a8;
  args.L = L;
  args.sel = sel;
  args.cpo = cpo;
  args.nst = nst;
  args.n_tiles = (L + ttg::kTC - 1) / ttg::kTC;
  const size_t smem = nst * stage + 1024;
  auto kern = reinterpret_cast<void (*)(const CUtensorMap, ttg::SyrkArgs)>(kp_pick(nbk));
  constexpr int threads = ttg::kConsumerWarps * 32;
  const int occ = std::max(1, kernel_occupancy((const void*)kern, kern, threads, smem));
  int py = 1;
  switch (nbk) {  // CTAs per tile set of this instantiation
#define KP_PY(N) case N: py = kp_py(N); break;
    KP_PY(7) KP_PY(8) KP_PY(9) KP_PY(10) KP_PY(11) KP_PY(12) KP_PY(13) KP_PY(14) KP_PY(15) KP_PY(16) KP_PY(17)
    KP_PY(18) KP_PY(19) KP_PY(20) KP_PY(21) KP_PY(22) KP_PY(23) KP_PY(24) KP_PY(25) KP_PY(26) KP_PY(27) KP_PY(28)
#undef KP_PY
  }
  const int gx = (int)std::max<long long>(1, std::min<long long>((long long)c->num_sms * occ / py, args.n_tiles));
  c->partials.ensure(sizeof(double) * (size_t)gx * a8 * a8);
  args.partials = c->partials.as<double>();
  char nm[64];
  std::snprintf(nm, sizeof nm, "k_syrk[a=%d]", a);
  const double Ls = (double)L * sel_frac;
  prof_begin(c, nm, 8.0 * a * Ls, Ls * (double)a * a);
  launch_k(c, kern, dim3(gx, py), threads, smem, tm, args);
  post_launch(c);
  gram_reduce(c, gx, 1, a8, a, c->G.as<double>());
  return true;
}

// C = sum over selected columns x x^T -> c->G (a x a); returns whether per-tile
// sums of squares were produced
bool syrk(ttg_ctx* c, const double* X, int a, long long L, const uint8_t* sel, long long cpo, double sel_frac,
          double* tsq) {
  c->G.ensure(sizeof(double) * (size_t)a * a);
  const int a8 = ttg::round_up(a, 8), nb = a8 / 8;
  if (a & 1) {  // odd rows: no 16-byte TMA runs -> generic
    gram_src(c, Src{X, a, L, nullptr, a}, 1, nullptr, 0, sel, cpo, sel_frac, tsq);
    return tsq != nullptr && ttg::round_up(a, 8) <= kFastMax1;
  }
  if (syrk_kp(c, X, a, L, sel, cpo, sel_frac, tsq) || syrk_ws16(c, X, a, L, sel, cpo, sel_frac, tsq) ||
      syrk2(c, X, a, L, sel, cpo, sel_frac, tsq)) {
    allreduce_sum(c, c->G.as<double>(), (size_t)a * a);
    return tsq != nullptr;
  }
  ttg::SyrkArgs args{};
  args.X = X;
  args.a = a;
  args.a8 = a8;
  args.L = L;
  args.sel = sel;
  args.cpo = cpo;
  args.n_tiles = (L + ttg::kTC - 1) / ttg::kTC;
  // measured at a = 64: k_syrk_kx 1.17 ms, k_syrk_kp<8, 1> 1.32 ms per 4.3 GB
  if ((nb == 7 || nb == 8) && std::getenv("TTG_KP8") && syrk_kp(c, X, a, L, sel, cpo, sel_frac, tsq)) {
    allreduce_sum(c, c->G.as<double>(), (size_t)a * a);
    return false;
  }
  CUtensorMap tmk;
  if ((nb == 7 || nb == 8) && !std::getenv("TTG_NO_KX") && (!sel || cpo % ttg::kTC == 0) &&
      make_tmap(&tmk, X, a, L)) {  // k-split SYRK, one CTA / SM
    constexpr int SBD = 128;
    args.tsumsq = tsq;
    const size_t stage = sizeof(double) * 4 * 16 * ttg::kTC;
    int nst = 6;
    if (const char* e = std::getenv("TTG_KX_NST")) nst = std::max(2, std::min(ttg::kMaxStages + 4, std::atoi(e)));
    args.nst = nst;
    const size_t smem = nst * stage + 1024;
    auto kern = ttg::k_syrk_kx<8>;
    constexpr int threads = (ttg::kConsumerWarps + 1) * 32;
    const int occ = std::max(1, kernel_occupancy((const void*)kern, kern, threads, smem));
    const int gx = (int)std::min<long long>((long long)c->num_sms * occ, std::max<long long>(1, args.n_tiles));
    c->partials.ensure(sizeof(double) * (size_t)gx * SBD * SBD);
    args.partials = c->partials.as<double>();
    char nm[64];
    std::snprintf(nm, sizeof nm, "k_syrk[a=%d]", a);
    const double Ls = (double)L * sel_frac;
    prof_begin(c, nm, 8.0 * a * Ls, Ls * (double)a * a);
    launch_k(c, kern, gx, threads, smem, tmk, args);
    post_launch(c);
    gram_reduce(c, gx, 0, SBD, a, c->G.as<double>());
    allreduce_sum(c, c->G.as<double>(), (size_t)a * a);
    return tsq != nullptr;
  }
  // 2x2-block tiles per super-tile: T(T+1)/2 (diagonal) or T^2 (off-diagonal), T <= 8
  if (nb <= 16) {
    args.ldt = ttg::smem_ld(a8);
    args.tsumsq = tsq;
    const int T = (nb + 1) / 2, ntiles = T * (T + 1) / 2;
    if (ntiles <= 8) launch_syrk_t<1>(c, args, 1, sel_frac);
    else if (ntiles <= 16) launch_syrk_t<2>(c, args, 1, sel_frac);
    else if (ntiles <= 24) launch_syrk_t<3>(c, args, 1, sel_frac);
    else launch_syrk_t<5>(c, args, 1, sel_frac);
  } else {
    args.ldt = ttg::smem_ld(128);
    args.tsumsq = nullptr;
    const int ns = (nb + 15) / 16;
    launch_syrk_t<8>(c, args, ns * (ns + 1) / 2, sel_frac);
  }
  allreduce_sum(c, c->G.as<double>(), (size_t)a * a);
  return tsq != nullptr && nb <= 16;
}


// Residual Gram of a pre-projected unfolding from the RAW Gram of its source:
// cur_i = K s with K = I_n (x) Psi^T (orthonormal rows), so
//   G_i = P K C K^T P,   C = sum_{selected s} s s^T,   P = I - U U^T.
// The streaming kernel is then a plain SYRK of the source columns (no
// residual, no pre-projection); the rest is (a x a)-sized.  trace(C) is left
// in c->scal[4] for the accuracy guard (see sweep()).
bool pcp_from_c(ttg_ctx* c, const Src& s, int64_t n, const double* U, int r_old, bool did);
bool gram_raw_src(ttg_ctx* c, const Src& s, int64_t n, const double* U, int r_old, const uint8_t* sel,
                  long long cpo, double sel_frac, double* tsq) {
  const int64_t rows = s.Psi ? s.As * n : s.r * n;
  const long long L = s.Ls / n;
  const bool did = syrk(c, s.S, (int)rows, L, sel, cpo, sel_frac, tsq);  // C -> c->G (rows x rows)
  return pcp_from_c(c, s, n, U, r_old, did);
}
// c->G: raw Gram C of the source (rows x rows) -> residual Gram P K C K^T P (a x a)
bool pcp_from_c(ttg_ctx* c, const Src& s, int64_t n, const double* U, int r_old, bool did) {
  const int64_t rows = s.Psi ? s.As * n : s.r * n, a = s.r * n;
  c->scal.ensure(sizeof(double) * 16);
  const size_t pcp_smem = sizeof(double) * ttg::pcp_smem_doubles((int)a, r_old);
  // (Y = W - U M / 2 keeps <= 8 elements per thread in registers: a r <= 4096;
  // W = C U holds four 8-column accumulator blocks: r <= 32)
  if (!s.Psi && pcp_smem + 1024 <= (size_t)c->smem_optin && a * r_old <= 8 * ttg::kPcpThreads && r_old <= 32 &&
      !std::getenv("TTG_NO_PCP")) {
    // one CTA: G = P C P in place (rank-r form), trace(C) for the guard
    kernel_occupancy((const void*)ttg::k_pcp, ttg::k_pcp, ttg::kPcpThreads, pcp_smem);
    prof_begin(c, "k_pcp", 16.0 * a * a, 4.0 * a * a * std::max(r_old, 1));
    launch_k(c, ttg::k_pcp, 1, ttg::kPcpThreads, pcp_smem, (const double*)c->G.as<double>(), (int)a, U, r_old, c->G.as<double>(),
             c->scal.as<double>() + 4);
    post_launch(c);
    return did;
  }
  const size_t pcp_l2 = sizeof(double) * ttg::pcp_l2_smem_doubles((int)a, r_old);
  // (measured: one CTA streaming C from L2 twice is latency-bound, 88 us at a = 176,
  // vs ~35 us for the multi-CTA path below: opt-in only)
  if (std::getenv("TTG_PCP_L2") && !s.Psi && r_old <= 32 && ttg::round_up((int)a, 8) <= 256 &&
      pcp_l2 + 1024 <= (size_t)c->smem_optin && !std::getenv("TTG_NO_PCP")) {
    // one CTA, C from L2: G = P C P in place, trace(C) for the guard
    kernel_occupancy((const void*)ttg::k_pcp_l2, ttg::k_pcp_l2, ttg::kPcpThreads, pcp_l2);
    prof_begin(c, "k_pcp", 24.0 * a * a, 4.0 * a * a * std::max(r_old, 1));
    launch_k(c, ttg::k_pcp_l2, 1, ttg::kPcpThreads, pcp_l2, c->G.as<double>(), (int)a, U, r_old,
             c->scal.as<double>() + 4);
    post_launch(c);
    return did;
  }
  c->Craw.ensure(sizeof(double) * (size_t)(rows * rows));
  CK(cudaMemcpyAsync(c->Craw.p, c->G.p, sizeof(double) * rows * rows, cudaMemcpyDeviceToDevice, c->stream));
  // G = Q^T C Q with Q = K P (one element-wise kernel, two GEMMs): the same
  // P K^T C K P as before in 4 launches instead of 11
  c->wcomb.ensure(sizeof(double) * (size_t)(rows * a));
  double* Q = c->wcomb.as<double>();
  prof_begin(c, "k_build_q", 8.0 * rows * a, 2.0 * rows * a * std::max(r_old, 1) * (s.Psi ? s.r : 1));
  launch_k(c, ttg::k_build_q, grid_for(rows * a, 256, 1024), 256, 0, s.Psi, s.Psi ? (int)s.As : (int)s.r, (int)s.r,
                                                                        (int)n, U, r_old, Q);
  post_launch(c);
  c->small[0].ensure(sizeof(double) * (size_t)(rows * a));
  double* T1 = c->small[0].as<double>();
  gemm<false, false>(c, c->Craw.as<double>(), rows, Q, rows, T1, rows, rows, a, rows, 1.0, 0.0);  // C Q
  c->G.ensure(sizeof(double) * (size_t)(a * a));
  double* G = c->G.as<double>();
  gemm<true, false>(c, Q, rows, T1, rows, G, a, a, a, rows, 1.0, 0.0);  // Q^T (C Q)
  // trace(C) for the guard, then symmetrise G
  c->scal.ensure(sizeof(double) * 16);
  // (C is exactly symmetric: the SYRK reduction mirrors its lower triangle)
  prof_begin(c, "k_symmetrize_trace", 16.0 * a * a, 0.0);
  launch_k(c, ttg::k_symmetrize_trace, grid_for(a * a, 256, 64), 256, 0, G, (int)a, c->Craw.as<double>(), (int)rows,
                                                                          c->scal.as<double>() + 4);
  post_launch(c);
  return did;
}

// Thrown inside a speculative sweep (sweep()) once the device flag says a guess was wrong.
struct SpecRejected {};

// Eigen result + trace(C) to the host (one stream synchronisation).  Inside a
// speculative sweep the flag of the earlier k_decide modes rides along: a mode
// that reads its result on the host must not go on to its fallback solvers on
// operands a wrong guess has turned into garbage.
void fetch_eig_result(ttg_ctx* c) {
  c->d2h += sizeof(EigResult) + sizeof(double);
  CK(cudaMemcpyAsync(c->h_eig, c->eigres.p, sizeof(EigResult), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(c->h_scal + 8, c->scal.as<double>() + 4, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  int* hflag = reinterpret_cast<int*>(c->h_eiglog + TTG_MAX_CORES);
  if (c->spec_active)
    CK(cudaMemcpyAsync(hflag, c->specflag.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (c->spec_active && *hflag) throw SpecRejected{};
}

// ---- eigen-solve -------------------------------------------------------------
// factor == 0: G is the residual Gram -> tridiagonal solver (k_syev).
// factor == 1: G holds the TSQR factor T -> one-sided Jacobi on T^T (k_jacobi_eig).
// hint: the rank this mode kept at the previous increment (-1: unknown).  A
// block attempt whose Gram does not fit shared memory costs ~40 L2 passes of
// G when it fails, so it is skipped when the hint says the block is too small.
EigResult eig(ttg_ctx* c, int a, long long kmax, const double* delta_src, double delta_mult, int factor = 0,
              int hint = -1) {
  c->UR.ensure(sizeof(double) * (size_t)a * a);
  c->lam.ensure(sizeof(double) * a);
  c->eigres.ensure(sizeof(EigResult));
  c->scal.ensure(sizeof(double) * 16);
  bool fast_done = false;
  if (!factor) {
    ttg::SyevArgs args{};
    args.G = c->G.as<double>();
    args.a = a;
    args.kmax = kmax;
    args.delta_src = delta_src;
    args.delta_mult = delta_mult;
    args.UR = c->UR.as<double>();
    args.lam = c->lam.as<double>();
    c->Mtmp.ensure(sizeof(double) * (size_t)32 * 6 * a);
    args.zbuf = c->Mtmp.as<double>();
    args.res = c->eigres.as<EigResult>();
    // fast path: block subspace iteration for the few kept directions
    bool done = false;
    if (!std::getenv("TTG_FULL_EIG")) {
      // block of 4 first (the common case keeps 1-2 directions), then 8
      // a mode that kept at most one direction last time starts with a block of 2
      // (2 x 2 Rayleigh-Ritz: one rotation; CholQR of two columns)
      const std::vector<int> blocks = (hint == 0 || hint == 1) ? std::vector<int>{2, 4, 8} : std::vector<int>{4, 8};
      for (int K : blocks) {
        if (done || a >= kFastSkip) break;  // very large a: straight to the full decomposition
        const size_t sub_vec = sizeof(double) * (size_t)2 * a * K;
        size_t smem_s = sizeof(double) * (size_t)a * a + sub_vec;
        ttg::SyevArgs sa = args;
        auto kern = K == 2 ? ttg::k_syev_top<2> : K == 4 ? ttg::k_syev_top<4> : ttg::k_syev_top<8>;
        const size_t kcap = dyn_smem_cap((const void*)kern);
        if (sub_vec > kcap) break;  // even the block vectors do not fit: full solver
        const size_t packed_s = sizeof(double) * ((((size_t)a * (a + 1) / 2) + 1) & ~(size_t)1) + sub_vec;
        if (smem_s <= kcap) {
          sa.in_smem = 1;
        } else if (packed_s <= kcap) {  // the lower triangle fits: G stays on chip
          sa.in_smem = 2;
          smem_s = packed_s;
        } else {
          // G from L2: each failed iteration re-reads it, so only try when the
          // last solve of this mode kept fewer directions than the block holds
          // (and, above a = 512, only when that is known)
          if (hint >= K || (a > 512 && hint < 0)) continue;  // a block of K certifies rank <= K - 1
          sa.in_smem = 0;
          smem_s = sub_vec;
        }
        kernel_occupancy((const void*)kern, kern, ttg::kSubThreads, smem_s);
        char nm[64];
        std::snprintf(nm, sizeof nm, "k_syev_top[a=%d]", a);
        prof_begin(c, nm, 16.0 * a * a, 2.0 * a * a * K);
        launch_k(c, kern, 1, ttg::kSubThreads, smem_s, sa);
        post_launch(c);
        fetch_eig_result(c);
        done = c->h_eig->converged != 0;
        if (std::getenv("TTG_DEBUG"))
          std::fprintf(stderr, "[ttg] eig_top K=%d a=%d conv=%d iters=%d rank=%d jac=%lld cycles copy=%lld init=%lld qr=%lld iter=%lld gx=%lld h=%lld eig=%lld res=%lld\n",
                       K, a, c->h_eig->converged, c->h_eig->sweeps, c->h_eig->rank, c->h_eig->t_phase[1] >> 40,
                       c->h_eig->t_phase[0] & 0xfffff, (c->h_eig->t_phase[0] >> 20) & 0xfffff,
                       c->h_eig->t_phase[0] >> 40, c->h_eig->t_phase[1] & 0xffffffffffll,
                       c->h_eig->t_phase[2] & 0xffffffffll, c->h_eig->t_phase[2] >> 32,
                       c->h_eig->t_phase[3] & 0xffffffffll, c->h_eig->t_phase[3] >> 32);
      }
    }
    fast_done = done;
    if (!done) {
      size_t vec = sizeof(double) * (size_t)7 * a;
      size_t smem = sizeof(double) * (size_t)a * a + vec;
      if (smem <= dyn_smem_cap((const void*)ttg::k_syev)) {
        args.in_smem = 1;
      } else {
        // G does not fit one CTA: tridiagonalise on the multi-CTA kernel
        // (k_sytrd_grid, cooperative), then k_syev's eigenvalue / eigenvector
        // phases on the result (reflectors in W, tri = [d | e | tau])
        c->W.ensure(sizeof(double) * (size_t)a * a);
        CK(cudaMemcpyAsync(c->W.p, c->G.p, sizeof(double) * (size_t)a * a, cudaMemcpyDeviceToDevice, c->stream));
        c->trd.ensure(sizeof(double) * 4 * (size_t)a + 64);
        ttg::TrdArgs ta{};
        ta.A = c->W.as<double>();
        ta.a = a;
        ta.pbuf = c->trd.as<double>();
        ta.tri = ta.pbuf + a;
        ta.bar = reinterpret_cast<unsigned*>(ta.tri + 3 * (size_t)a);
        CK(cudaMemsetAsync(ta.bar, 0, 2 * sizeof(unsigned), c->stream));
        // panel width: the widest of 16 / 8 / 4 / 2 whose (3 + 2 nb) a doubles fit one CTA
        const size_t tcap = dyn_smem_cap((const void*)ttg::k_sytrd_grid);
        ta.nb = 16;
        while (ta.nb > 2 && sizeof(double) * (3 + 2 * (size_t)ta.nb) * a > tcap) ta.nb /= 2;
        const size_t tsm = sizeof(double) * (3 + 2 * (size_t)ta.nb) * a;
        if (tsm > tcap) fail(TTG_E_RESOURCE, "eigen-solve of a " + std::to_string(a) + "-row Gram exceeds the device solver");
        const int occ = kernel_occupancy((const void*)ttg::k_sytrd_grid, ttg::k_sytrd_grid, ttg::kTrdThreads, tsm);
        if (occ < 1) fail(TTG_E_RESOURCE, "tridiagonalisation kernel does not fit on an SM");
        const int want = std::getenv("TTG_TRD_CTAS") ? std::atoi(std::getenv("TTG_TRD_CTAS")) : c->num_sms;
        const int nblk = std::max(1, std::min({want, c->num_sms * occ, (a + 3) / 4}));
        char nm[64];
        std::snprintf(nm, sizeof nm, "k_sytrd_grid[a=%d]", a);
        prof_begin(c, nm, 24.0 * a * a, 4.0 / 3.0 * a * a * a);
        {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3((unsigned)nblk);
          cfg.blockDim = dim3(ttg::kTrdThreads);
          cfg.dynamicSmemBytes = tsm;
          cfg.stream = c->stream;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeCooperative;  // co-residency of the grid barrier
          at[0].val.cooperative = 1;
          cfg.attrs = at;
          cfg.numAttrs = 1;
          CK(cudaLaunchKernelEx(&cfg, ttg::k_sytrd_grid, ta));
        }
        post_launch(c);
        args.in_smem = 0;
        args.Ag = c->W.as<double>();
        args.tri = ta.tri;
        smem = vec;
      }
      kernel_occupancy((const void*)ttg::k_syev, ttg::k_syev, ttg::kSyevThreads, smem);
      char nm[64];
      std::snprintf(nm, sizeof nm, "k_syev[a=%d]", a);
      prof_begin(c, nm, 16.0 * a * a, args.tri ? 2.0 * a * a : 4.0 / 3.0 * a * a * a);
      launch_k(c, ttg::k_syev, 1, ttg::kSyevThreads, smem, args);
      post_launch(c);
      if (args.tri) {  // back-transform of the kept vectors, VB per CTA, over the grid
        const long long kcap = std::min<long long>(kmax, a);
        const bool wide = (size_t)8 * a * sizeof(double) <= (size_t)c->smem_optin - 4096;
        const int vb = wide ? 8 : 4;
        const size_t bsm = sizeof(double) * vb * (size_t)a;
        auto kbt = wide ? ttg::k_syev_bt<8> : ttg::k_syev_bt<4>;
        kernel_occupancy((const void*)kbt, kbt, ttg::kBtThreads, bsm);
        prof_begin(c, "k_syev_bt", 8.0 * a * a / 2, 4.0 * a * a / 2);
        launch_k(c, kbt, (unsigned)std::max<long long>(1, (kcap + vb - 1) / vb), ttg::kBtThreads, bsm,
                 (const double*)c->W.as<double>(), a, (const double*)(args.tri + 2 * (size_t)a),
                 (const ttg::EigResult*)c->eigres.as<EigResult>(), c->UR.as<double>());
        post_launch(c);
      }
    }
  } else {
    size_t need_smem = sizeof(double) * ((size_t)a * a + a) + sizeof(int) * a + 64;
    ttg::EigArgs args{};
    args.G = c->G.as<double>();
    args.a = a;
    args.factor = factor;
    args.kmax = kmax;
    args.delta_src = delta_src;
    args.delta_mult = delta_mult;
    args.tol = 2.220446049250313e-16 * std::max(8, a);
    args.max_sweeps = 60;
    args.UR = c->UR.as<double>();
    args.lam = c->lam.as<double>();
    args.res = c->eigres.as<EigResult>();
    size_t smem;
    if (need_smem <= dyn_smem_cap((const void*)ttg::k_jacobi_eig)) {
      args.in_smem = 1;
      args.Wg = nullptr;
      smem = need_smem;
    } else {
      args.in_smem = 0;
      c->W.ensure(sizeof(double) * (size_t)a * a);
      args.Wg = c->W.as<double>();
      smem = sizeof(double) * a + sizeof(int) * a + 64;
    }
    kernel_occupancy((const void*)ttg::k_jacobi_eig, ttg::k_jacobi_eig, ttg::kEigThreads, smem);
    prof_begin(c, "k_jacobi_eig", 16.0 * a * a, 0.0);
    launch_k(c, ttg::k_jacobi_eig, 1, ttg::kEigThreads, smem, args);
    post_launch(c);
  }
  if (!fast_done) {
    fetch_eig_result(c);
  }
  EigResult r = *c->h_eig;
  if (std::getenv("TTG_DEBUG"))
    std::fprintf(stderr,
                 "[ttg] eig a=%d factor=%d rank=%d sweeps=%d lam_max=%.3e lam_min_kept=%.3e delta=%.3e "
                 "cycles tri=%lld val=%lld vec=%lld n_lam=%lld\n",
                 a, factor, r.rank, r.sweeps, r.lam_max, r.lam_min_kept, r.delta, r.t_phase[0], r.t_phase[1],
                 r.t_phase[2], r.t_phase[3]);
  if (!r.converged) fail(TTG_E_NUMERIC, "svd_trunc: Jacobi eigen-solve failed to converge on " +
                                            std::to_string(a) + "x" + std::to_string(a) + " matrix");
  return r;
}

// ---- accurate path: TSQR factor + Jacobi on T^T ---------------------------------
bool accurate_supported(int a, int r_old) {
  return ttg::round_up(a, 8) <= kFastMax && (r_old == 0 || ttg::round_up(r_old, 8) <= kFastMax);
}

// Replaces c->G by the a x a R-factor T of the residual (T^T T = R R^T) and
// solves on T^T: singular values are resolved to eps_mach |R|.
EigResult accurate_eig(ttg_ctx* c, const double* X, int a, long long L, const double* U, int r_old, int ldu,
                       const uint8_t* sel, long long cpo, long long kmax, const double* dsrc, double dmult) {
  int a8 = ttg::round_up(a, 8);
  int r8 = r_old > 0 ? ttg::round_up(r_old, 8) : 0;
  if (r_old > 0) make_frags(c, U, a, r_old, ldu, true, true);
  ttg::TsqrArgs args{};
  args.src = ttg::TileSrc{X, a, L, sel, cpo};
  args.a8 = a8;
  args.ldt = ttg::smem_ld(a8);
  args.ldp = ttg::smem_ld(std::max(r8, 8));
  args.UTf = c->UTf.as<double>();
  args.Uf = c->Uf.as<double>();
  args.r8 = r8;
  args.n_tiles = (L + ttg::kTC - 1) / ttg::kTC;
  size_t smem = sizeof(double) * ((size_t)a * a + (size_t)args.ldt * ttg::kTC + (size_t)8 * args.ldp * 8);
  kernel_occupancy((const void*)ttg::k_tsqr_local, ttg::k_tsqr_local, ttg::kThreads, smem);
  int gx = (int)std::min<long long>(c->num_sms, std::max<long long>(1, args.n_tiles));
  c->partials.ensure(sizeof(double) * (size_t)gx * a * a);
  args.Tout = c->partials.as<double>();
  prof_begin(c, "k_tsqr_local", 8.0 * a * L, (double)L * (4.0 * r_old * a + 2.0 * a * a));
  launch_k(c, ttg::k_tsqr_local, gx, ttg::kThreads, smem, args);
  post_launch(c);
  c->scratch.ensure(sizeof(double) * (size_t)a * a);
  c->G.ensure(sizeof(double) * (size_t)a * a);
  size_t smem2 = sizeof(double) * (size_t)a * a;
  kernel_occupancy((const void*)ttg::k_tsqr_combine, ttg::k_tsqr_combine, 1024, smem2);
  prof_begin(c, "k_tsqr_combine", 16.0 * gx * a * a, 2.0 * gx * a * a * a);
  launch_k(c, ttg::k_tsqr_combine, 1, 1024, smem2, c->partials.as<double>(), gx, a, c->scratch.as<double>(),
                                                     c->G.as<double>());
  post_launch(c);
  if (c->coll) {
    c->partials.ensure(sizeof(double) * (size_t)c->world * a * a);
    allgather(c, c->G.as<double>(), c->partials.as<double>(), (size_t)a * a);
    prof_begin(c, "k_tsqr_combine", 16.0 * c->world * a * a, 2.0 * c->world * a * a * a);
    launch_k(c, ttg::k_tsqr_combine, 1, 1024, smem2, c->partials.as<double>(), c->world, a,
                                                       c->scratch.as<double>(), c->G.as<double>());
    post_launch(c);
  }
  return eig(c, a, kmax, dsrc, dmult, /*factor=*/1);
}

// The Gram floor resolves sigma only down to ~sqrt(eps_mach)|R|; fall back
// to the factor path when the decision or a kept direction gets near it.
bool needs_accurate(const EigResult& er) {
  if (!(er.lam_max > 0.0)) return false;
  if (er.delta * er.delta < 1e-9 * er.lam_max) return true;
  if (er.rank > 0 && er.lam_min_kept < 1e-6 * er.lam_max) return true;
  return false;
}

// [U_pad U_R] -> out (a x (r_old + r_R)) with the 1e-10 guard; returns guard flag
int append(ttg_ctx* c, const double* Upad, int a, int r_old, int r_R, double* out) {
  c->scratch.ensure(sizeof(double) * ((size_t)a * r_R + (size_t)(r_old + 1) * (r_R + 1) + 16));
  ttg::AppendArgs args{Upad, c->UR.as<double>(), a, r_old, r_R, out, c->scratch.as<double>(),
                       c->eigres.as<EigResult>(), c->gcount.as<int>(), 0};
  const int rn = r_old + r_R;
  if ((double)a * rn * rn >= 5e7) {
    // large block: [U_pad U_R] by copies, its Gram C^T C on the DMMA GEMM
    // (split-k, fixed order), the deviation by a grid reduction; k_append then
    // only runs the (rare) Householder correction when the guard fires
    if (Upad != out && r_old > 0)
      CK(cudaMemcpyAsync(out, Upad, sizeof(double) * (size_t)a * r_old, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(out + (size_t)a * r_old, c->UR.p, sizeof(double) * (size_t)a * r_R, cudaMemcpyDeviceToDevice,
                       c->stream));
    c->small[1].ensure(sizeof(double) * (size_t)rn * rn);
    double* S = c->small[1].as<double>();
    gemm<true, false>(c, out, a, out, a, S, rn, rn, rn, a, 1.0, 0.0);
    CK(cudaMemsetAsync(&c->eigres.as<EigResult>()->dev, 0, sizeof(double), c->stream));
    prof_begin(c, "k_gram_dev", 8.0 * rn * rn, 0.0);
    launch_k(c, ttg::k_gram_dev, grid_for((long long)rn * rn, 256, 2 * c->num_sms), 256, 0, (const double*)S, rn,
             c->eigres.as<EigResult>());
    post_launch(c);
    args.precomputed = 1;
  }
  prof_begin(c, "k_append", 8.0 * a * (2.0 * r_old + 2.0 * r_R), 2.0 * a * (r_old + r_R) * (r_old + r_R));
  launch_k(c, ttg::k_append, 1, 1024, 0, args);
  post_launch(c);
  return 0;  // the guard count is read once per update (guards_read), not per mode
}

// ---- one-launch mode decision (ttg_decide.cuh) -----------------------------------
// Applies when the unfolding is read directly (no pending pre-projection), the
// old basis is small and the previous update of this mode kept few directions.
int decide_block(int hint) { return hint <= 1 ? 2 : 4; }
bool decide_applies(const ttg_ctx* c, bool has_psi, int64_t a, int64_t r_old, int hint) {
  // (a mode that kept nothing last time most likely keeps nothing again: its whole cost is
  // trace(P C P), which the multi-CTA chain forms faster than one CTA computes C U)
  if (std::getenv("TTG_NO_DECIDE") || has_psi || hint < (std::getenv("TTG_DECIDE_ZERO") ? 0 : 1) || hint > 3) return false;
  const int K = decide_block(hint);
  if (r_old < 1 || r_old > ttg::kDecMaxR || a > ttg::kDecMaxA || a - r_old < K) return false;
  const void* kern = K == 2 ? (const void*)ttg::k_decide<2> : (const void*)ttg::k_decide<4>;
  return sizeof(double) * ttg::dec_smem_doubles((int)a, (int)r_old, K) <= dyn_smem_cap(kern);
}
// C in c->G (a x a raw Gram), old basis Upad (a x r_old) -> rank, U_R (c->UR) and the
// appended core in `out` (capacity a x (r_old + K - 1)); result in c->eigres, trace(C) in c->scal[4]
void decide_launch(ttg_ctx* c, int a, int r_old, const double* Upad, double* out, long long kmax, const double* dsrc,
                   double dmult, int hint, int expect, int* spec_flag, EigResult* log) {
  const int K = decide_block(hint);
  c->UR.ensure(sizeof(double) * (size_t)a * a);
  c->lam.ensure(sizeof(double) * a);
  c->eigres.ensure(sizeof(EigResult));
  c->scal.ensure(sizeof(double) * 16);
  ttg::DecideArgs da{};
  da.C = c->G.as<double>();
  da.a = a;
  da.U = Upad;
  da.r = r_old;
  da.kmax = kmax;
  da.delta_src = dsrc;
  da.delta_mult = dmult;
  da.UR = c->UR.as<double>();
  da.lam = c->lam.as<double>();
  da.out = out;
  da.res = c->eigres.as<EigResult>();
  da.trC = c->scal.as<double>() + 4;
  da.guard_count = c->gcount.as<int>();
  da.ldb = ttg::dec_ldb(a);
  const int best = (a + 63) / 64;  // k-range parts per 8-row block (dec_pass: 64 columns of C per task)
  da.ksplit = best;
  da.expect = expect;
  da.spec_flag = spec_flag;
  da.log = log;
  const size_t smem = sizeof(double) * ttg::dec_smem_doubles(a, r_old, K);
  char nm[64];
  std::snprintf(nm, sizeof nm, "k_decide[a=%d]", a);
  prof_begin(c, nm, 8.0 * a * a * 3, 2.0 * a * a * (r_old + 3.0 * K));
  if (K == 2) {
    kernel_occupancy((const void*)ttg::k_decide<2>, ttg::k_decide<2>, ttg::kDecThreads, smem);
    launch_k(c, ttg::k_decide<2>, 1, ttg::kDecThreads, smem, da);
  } else {
    kernel_occupancy((const void*)ttg::k_decide<4>, ttg::k_decide<4>, ttg::kDecThreads, smem);
    launch_k(c, ttg::k_decide<4>, 1, ttg::kDecThreads, smem, da);
  }
  post_launch(c);
}
EigResult eig_fetch(ttg_ctx* c) {
  fetch_eig_result(c);
  return *c->h_eig;
}

// Guard count of the last sweep: copied to the pinned slot after the sweep and
// valid after the caller's next stream synchronisation.
int* guards_slot(ttg_ctx* c) { return reinterpret_cast<int*>(c->h_scal + 12); }
void guards_fetch(ttg_ctx* c) {
  c->d2h += sizeof(int);
  CK(cudaMemcpyAsync(guards_slot(c), c->gcount.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
}

// ---- projection --------------------------------------------------------------
// out (r x L) = W^T X  (X: a x L, W: a x r with leading dimension ldw)
// Warp-specialised m16n8k16 projection (k_project_ws16) for r <= 32, even
// a <= 256: 4 consumer warps x 16 columns per 64-column tile; two CTAs / SM
// with two stages when they fit, else one CTA with up to four.  False when
// the operand does not qualify (the caller takes the other kernels).
bool project_ws16(ttg_ctx* c, const double* X, int a, long long L, const double* W, int r, int ldw, double* out,
                  double* tsq) {
  if (std::getenv("TTG_NO_WS16") || (a & 1) || a > 256 || r > 32) return false;
  CUtensorMap tm;
  if (!make_tmap(&tm, X, a, L, ttg::kTC)) return false;
  const int r8 = ttg::round_up(r, 8), NB = r8 / 8, nks = (a + 15) / 16;
  const size_t nfr = (size_t)nks * NB * 128;
  const size_t stage = sizeof(double) * (size_t)nks * 16 * ttg::kTC;
  const size_t fixed = 1024 + sizeof(double) * (nfr + (size_t)4 * 16 * r8);
  const size_t cap = (size_t)c->smem_optin - 1024;
  int nst = 2;
  if (fixed + 2 * stage > cap) return false;
  if (2 * (fixed + 2 * stage) > 220 * 1024) {  // one CTA / SM: deepen the ring
    while (nst < 4 && fixed + (nst + 1) * stage <= cap) ++nst;
  }
  if (std::getenv("TTG_WS16_NST")) nst = std::max(2, std::min(4, std::atoi(std::getenv("TTG_WS16_NST"))));
  const size_t smem = fixed + nst * stage;
  c->UTf.ensure(sizeof(double) * std::max<size_t>(nfr, 1));
  prof_begin(c, "k_make_frags", 8.0 * nfr, 0.0);
  launch_k(c, ttg::k_make_frags16, grid_for((long long)nfr, 256, 256), 256, 0, W, a, r, ldw, nks, NB,
                                                                                 c->UTf.as<double>());
  post_launch(c);
  ttg::ProjArgs args{};
  args.src = ttg::TileSrc{X, a, L, nullptr, 1};
  args.a8 = ttg::round_up(a, 8);
  args.WTf = c->UTf.as<double>();
  args.r = r;
  args.r8 = r8;
  args.out = out;
  args.tsumsq = tsq;
  args.n_tiles = (L + ttg::kTC - 1) / ttg::kTC;
  args.nst = nst;
  void (*kern)(const CUtensorMap, ttg::ProjArgs) = NB == 1   ? ttg::k_project_ws16<4, 1>
                                                   : NB == 2 ? ttg::k_project_ws16<4, 2>
                                                   : NB == 3 ? ttg::k_project_ws16<4, 3>
                                                             : ttg::k_project_ws16<4, 4>;
  constexpr int threads = 5 * 32;
  const int occ = std::max(kernel_occupancy((const void*)kern, kern, threads, smem), 1);
  const int gx = (int)std::min<long long>((long long)c->num_sms * occ, std::max<long long>(1, args.n_tiles));
  char nm[64];
  std::snprintf(nm, sizeof nm, "k_project[a=%d,r=%d]", a, r);
  prof_begin(c, nm, 8.0 * ((double)a + r) * L, 2.0 * a * r * (double)L);
  launch_k(c, kern, gx, threads, smem, tm, args);
  post_launch(c);
  return true;
}

// K-chunked projection (k_project_kc) for even a and r <= 34: n-blocks of 8
// rows by DMMA plus a DFMA tail of 1-2 rows when r = 8 NB + {1, 2}.  Tall
// sources (a > 64) stream in 64-row stages with the accumulators held in
// registers.  False when the operand does not qualify.
// DFMA tail rows of k_project_kc: r = 8 NB + T with T <= kKcMaxTail costs
// NB + T/8 n-blocks of FP64 work instead of NB + 1 (r = 19..20 no longer pay
// for 24 rows).
constexpr int kKcMaxTail = 3;  // measured: T = 4 (r = 20) runs slower than padding to NB + 1
template <int NCW, int NB, int T>
void* kc_kernel() {
  return (void*)ttg::k_project_kc<NCW, NB, T>;
}
template <int NCW, int NB, int T>
void* kc_pick_nb(int nb, int t) {
  if constexpr (NB > 4) {
    return nullptr;
  } else if constexpr (T > kKcMaxTail) {
    return kc_pick_nb<NCW, NB + 1, 0>(nb, t);
  } else {
    return (nb == NB && t == T) ? kc_kernel<NCW, NB, T>() : kc_pick_nb<NCW, NB, T + 1>(nb, t);
  }
}
template <int NCW>
void* kc_pick_t(int NB, int T) {
  return kc_pick_nb<NCW, 1, 0>(NB, T);
}
void* kc_pick(int ncw, int NB, int T) { return ncw == 8 ? kc_pick_t<8>(NB, T) : kc_pick_t<4>(NB, T); }

struct KcPlan {
  int NB = 0, T = 0, ncw = 0, kc = 0, nst = 0, nks = 0;
  size_t smem = 0, nfr = 0, ntl = 0;
};

// Shared-memory plan of k_project_kc for (a, r): 8 consumer warps (128-column
// tiles, two warps per SM sub-partition) for tall sources, 4 (64-column
// tiles, two CTAs / SM) when the whole tile fits a stage or the 8-warp ring
// does not fit next to the W fragments; false when neither fits.
bool kc_plan(const ttg_ctx* c, int a, int r, KcPlan& P) {
  if (std::getenv("TTG_NO_KC") || (a & 1) || r > 34 || r < 1) return false;
  P.NB = (r + 7) / 8;
  P.T = 0;
  const int max_tail = std::getenv("TTG_KC_TAIL") ? std::atoi(std::getenv("TTG_KC_TAIL")) : kKcMaxTail;
  if (r > 8 && r % 8 >= 1 && r % 8 <= std::min(max_tail, kKcMaxTail) && !std::getenv("TTG_NO_TAIL")) {
    P.NB = r / 8;
    P.T = r % 8;
  }
  if (P.NB > 4) return false;
  P.nks = (a + 15) / 16;
  P.nfr = (size_t)P.nks * P.NB * 128;
  P.ntl = (size_t)P.nks * P.T * 16;
  const size_t cap = (size_t)c->smem_optin - 1024;
  int order[2] = {P.nks > 4 ? 8 : 4, P.nks > 4 ? 4 : 8};
  if (const char* e = std::getenv("TTG_KC_NCW")) order[0] = order[1] = std::atoi(e) == 8 ? 8 : 4;
  for (int ncw : order) {
    for (int kcw : {4, 2}) {
      const int kc = std::min(P.nks, std::getenv("TTG_KC") ? std::max(1, std::atoi(std::getenv("TTG_KC"))) : kcw);
      const int tc = 16 * ncw;
      const size_t stage = sizeof(double) * (size_t)kc * 16 * tc;
      const size_t fixed = 1024 + sizeof(double) * (P.nfr + P.ntl + (size_t)ncw * 16 * (8 * P.NB + P.T));
      if (fixed + 2 * stage > cap) continue;
      int nst = 2;
      if (2 * (fixed + 2 * stage) > 220 * 1024) {  // one CTA / SM: deepen the ring
        while (nst < ttg::kProjStages && fixed + (nst + 1) * stage <= cap) ++nst;
      } else {
        while (nst < ttg::kProjStages && 2 * (fixed + (nst + 1) * stage) <= 220 * 1024) ++nst;
      }
      if (const char* e = std::getenv("TTG_KC_NST")) nst = std::max(2, std::min(ttg::kProjStages, std::atoi(e)));
      if (fixed + nst * stage > cap) continue;
      P.ncw = ncw;
      P.kc = kc;
      P.nst = nst;
      P.smem = fixed + nst * stage;
      return true;
    }
  }
  return false;
}

bool project_kc(ttg_ctx* c, const double* X, int a, long long L, const double* W, int r, int ldw, double* out,
                double* tsq) {
  KcPlan P;
  if (!kc_plan(c, a, r, P)) return false;
  const int NB = P.NB, T = P.T, ncw = P.ncw, nks = P.nks, kc = P.kc, nst = P.nst;
  const size_t nfr = P.nfr, ntl = P.ntl, smem = P.smem;
  const int tc = 16 * ncw;
  CUtensorMap tm;
  if (!make_tmap(&tm, X, a, L, tc)) return false;
  c->UTf.ensure(sizeof(double) * std::max<size_t>(nfr, 1));
  prof_begin(c, "k_make_frags16", 8.0 * nfr, 0.0);
  launch_k(c, ttg::k_make_frags16, grid_for((long long)nfr, 256, 256), 256, 0, W, a, r, ldw, nks, NB,
                                                                                 c->UTf.as<double>());
  post_launch(c);
  if (T) {
    c->UTt.ensure(sizeof(double) * std::max<size_t>(ntl, 1));
    prof_begin(c, "k_make_tail", 8.0 * ntl, 0.0);
    launch_k(c, ttg::k_make_tail, grid_for((long long)ntl, 256, 64), 256, 0, W, a, ldw, nks, 8 * NB, T,
                                                                               c->UTt.as<double>());
    post_launch(c);
  }
  ttg::ProjArgs args{};
  args.src = ttg::TileSrc{X, a, L, nullptr, 1};
  args.a8 = ttg::round_up(a, 8);
  args.WTf = c->UTf.as<double>();
  args.WTt = T ? c->UTt.as<double>() : nullptr;
  args.r = r;
  args.r8 = 8 * NB + T;
  args.out = out;
  args.tsumsq = tsq;
  args.n_tiles = (L + tc - 1) / tc;
  args.nst = nst;
  args.kc = kc;
  auto kern = reinterpret_cast<void (*)(const CUtensorMap, ttg::ProjArgs)>(kc_pick(ncw, NB, T));
  const int threads = (ncw + 1) * 32;
  const int occ = std::max(kernel_occupancy((const void*)kern, kern, threads, smem), 1);
  const int gx = (int)std::min<long long>((long long)c->num_sms * occ, std::max<long long>(1, args.n_tiles));
  char nm[64];
  std::snprintf(nm, sizeof nm, "k_project[a=%d,r=%d]", a, r);
  prof_begin(c, nm, 8.0 * ((double)a + r) * L, 2.0 * a * r * (double)L);
  launch_k(c, kern, gx, threads, smem, tm, args);
  post_launch(c);
  return true;
}

// High-rank projection (34 < r <= 128, even a): k_project_ws, W^T fragments
// streamed through the ring with the X boxes.  False when it does not apply.
template <int NCW, int NB>
void* ws_kernel() {
  return (void*)ttg::k_project_ws<NCW, NB>;
}
template <int NCW, int NB>
void* ws_pick_t(int nb) {
  if constexpr (NB > 16) {
    return nullptr;
  } else {
    return nb == NB ? ws_kernel<NCW, NB>() : ws_pick_t<NCW, NB + 1>(nb);
  }
}
void* ws_pick(int ncw, int nb) { return ncw == 8 ? ws_pick_t<8, 2>(nb) : ws_pick_t<4, 2>(nb); }

bool project_ws(ttg_ctx* c, const double* X, int a, long long L, const double* W, int r, int ldw, double* out,
                double* tsq) {
  if (std::getenv("TTG_NO_PWS") || (a & 1) || r <= 8 || r > 128) return false;
  const int NB = (r + 7) / 8, nks = (a + 15) / 16;
  const int ncw = nks > 4 ? 8 : 4, tc = 16 * ncw;
  const size_t cap = (size_t)c->smem_optin - 2048;
  const size_t box = sizeof(double) * 16 * tc, wch = sizeof(double) * 128 * NB;
  int kc = 0, nst = 0;
  for (int kcw : {2, 4, 1}) {  // deepest ring with >= 3 stages, else >= 2
    const int k_ = std::min(kcw, nks);
    const int n_ = (int)std::min<size_t>(ttg::kProjStages, cap / (k_ * (box + wch)));
    if (n_ >= 3 || (n_ >= 2 && kc == 0)) {
      kc = k_;
      nst = n_;
      if (n_ >= 3) break;
    }
  }
  if (const char* e = std::getenv("TTG_PWS_KC")) {  // tuning override: k16-steps per stage
    const int k_ = std::max(1, std::min(std::atoi(e), nks));
    const int n_ = (int)std::min<size_t>(ttg::kProjStages, cap / (k_ * (box + wch)));
    if (n_ >= 2) { kc = k_; nst = n_; }
  }
  if (kc == 0) return false;
  CUtensorMap tm;
  if (!make_tmap(&tm, X, a, L, tc)) return false;
  const size_t nfr = (size_t)nks * NB * 128;
  c->UTf.ensure(sizeof(double) * nfr);
  prof_begin(c, "k_make_frags16", 8.0 * nfr, 0.0);
  launch_k(c, ttg::k_make_frags16, grid_for((long long)nfr, 256, 512), 256, 0, W, a, r, ldw, nks, NB,
           c->UTf.as<double>());
  post_launch(c);
  ttg::ProjArgs args{};
  args.src = ttg::TileSrc{X, a, L, nullptr, 1};
  args.a8 = ttg::round_up(a, 8);
  args.WTf = c->UTf.as<double>();
  args.r = r;
  args.r8 = 8 * NB;
  args.out = out;
  args.tsumsq = tsq;
  args.n_tiles = (L + tc - 1) / tc;
  args.nst = nst;
  args.kc = kc;
  const size_t smem = 1024 + (size_t)nst * kc * (box + wch);
  auto kern = reinterpret_cast<void (*)(const CUtensorMap, ttg::ProjArgs)>(ws_pick(ncw, NB));
  const int threads = (ncw + 1) * 32;
  const int occ = std::max(kernel_occupancy((const void*)kern, kern, threads, smem), 1);
  const int gx = (int)std::min<long long>((long long)c->num_sms * occ, std::max<long long>(1, args.n_tiles));
  char nm[64];
  std::snprintf(nm, sizeof nm, "k_project[a=%d,r=%d]", a, r);
  prof_begin(c, nm, 8.0 * ((double)a + r) * L, 2.0 * a * r * (double)L);
  launch_k(c, kern, gx, threads, smem, tm, args);
  post_launch(c);
  return true;
}

bool project(ttg_ctx* c, const double* X, int a, long long L, const double* W, int r, int ldw, double* out,
             double* tsq = nullptr) {
  const int a8 = ttg::round_up(a, 8), r8 = ttg::round_up(r, 8);
  // tall sources (the a = 512 statistics pass) with r >= 20 (NB >= 3 n-blocks):
  // the streamed-W ring is measured faster than resident fragments, whose
  // 98 KB at NB = 3 leave room for only 3 x 32 KB stages (r = 24: 0.80 vs
  // 0.84 ms per 4.29 GB; r = 32: 1.03 vs 1.09 ms)
  if (!std::getenv("TTG_NO_PWS_MID") && r >= 20 && a >= 256 && project_ws(c, X, a, L, W, r, ldw, out, tsq))
    return tsq != nullptr;
  if (project_kc(c, X, a, L, W, r, ldw, out, tsq)) return tsq != nullptr;
  if (r > 34 && project_ws(c, X, a, L, W, r, ldw, out, tsq)) return tsq != nullptr;
  if (a8 > kFastMax1 || r8 > kFastMax) {
    gemm<true, false>(c, W, ldw, X, a, out, r, r, L, a, 1.0, 0.0);
    return false;
  }
  if (!(a & 1) && r8 <= 32 && (!(a8 <= 64 && r8 == 16) || std::getenv("TTG_WS16_ALL")) &&
      project_ws16(c, X, a, L, W, r, ldw, out, tsq))
    return tsq != nullptr;
  make_frags(c, W, a, r, ldw, true, false);
  ttg::ProjArgs args{};
  args.src = ttg::TileSrc{X, a, L, nullptr, 1};
  args.a8 = a8;
  args.ldt = ttg::smem_ld(a8);
  args.WTf = c->UTf.as<double>();
  args.r = r;
  args.r8 = r8;
  args.out = out;
  args.tsumsq = tsq;
  args.n_tiles = (L + ttg::kTC - 1) / ttg::kTC;
  if (a & 1) {  // odd rows: no 16-byte bulk runs -> cp.async single-buffered kernel
    const size_t nfr0 = (size_t)(r8 / 8) * (a8 / 4) * 32;
    size_t smem0 = sizeof(double) * (size_t)args.ldt * ttg::kTC;
    if (smem0 > c->smem_optin - 1024) {
      gemm<true, false>(c, W, ldw, X, a, out, r, r, L, a, 1.0, 0.0);
      return false;
    }
    if (smem0 + sizeof(double) * nfr0 <= 110 * 1024) {
      args.frag_smem = 1;
      smem0 += sizeof(double) * nfr0;
    }
    args.nst = 0;
    auto k0 = ttg::k_project<false, false>;
    const int occ0 = std::max(kernel_occupancy((const void*)k0, k0, ttg::kThreads, smem0), 1);
    const int gx0 = (int)std::min<long long>((long long)c->num_sms * occ0, std::max<long long>(1, args.n_tiles));
    char nm0[64];
    std::snprintf(nm0, sizeof nm0, "k_project[a=%d,r=%d]", a, r);
    prof_begin(c, nm0, 8.0 * ((double)a + r) * L, 2.0 * a * r * (double)L);
    launch_k(c, k0, gx0, ttg::kThreads, smem0, args);
    post_launch(c);
    return tsq != nullptr;
  }
  const bool db = a8 <= kFastMax;
  const size_t nfr = (size_t)(r8 / 8) * (a8 / 4) * 32;
  const size_t stage = sizeof(double) * (size_t)args.ldt * ttg::kTC;
  CUtensorMap tm;
  // 32-column tiles: keep 2 CTAs x 2 stages per SM for tall operands, and give
  // each warp half the k-steps so r8 <= 32 fits the register-resident W^T
  const bool narrow = r <= 32 && (a8 > 64 || r8 > 16);
  const int tc = narrow ? 32 : ttg::kTC;
  if (a8 <= 256 && !std::getenv("TTG_NO_TMAP") && make_tmap(&tm, X, a, L, tc)) {
    // tensor-map TMA ring: 2 stages at 2 CTAs / SM (the per-tile DMMA work of
    // one CTA hides behind the other's loads), deeper when only one CTA fits
    const size_t tstage = sizeof(double) * 16 * tc * (size_t)((a + 15) / 16);
    const size_t extra = 1024 + sizeof(double) * (r <= 32 ? (size_t)ttg::kConsumerWarps * 8 * 32 : 0);
    const bool regw = a8 <= 64 && r8 <= (narrow ? 32 : 16);
    const size_t fr = regw ? 0 : sizeof(double) * nfr;
    const size_t cap = (size_t)c->smem_optin - 1024;
    // two CTAs / SM, each with as many stages as fit ~110 KB (>= 64 KB in
    // flight per SM streams at HBM rate); one deeper CTA when two do not fit
    int nst = 2;
    size_t smem = nst * tstage + extra;
    if (fr && smem + fr <= std::min<size_t>(cap, 110 * 1024)) {
      args.frag_smem = 1;
      smem += fr;
    }
    const size_t per_cta = 2 * smem > 220 * 1024 ? cap : 110 * 1024;
    while (nst < ttg::kProjStages && smem + tstage <= per_cta) {
      ++nst;
      smem += tstage;
    }
    if (smem <= cap) {
      args.nst = nst;
      args.n_tiles = (L + tc - 1) / tc;
      auto kern = narrow ? (regw ? ttg::k_project_tma<true, 32> : ttg::k_project_tma<false, 32>)
                         : (regw ? ttg::k_project_tma<true, 64> : ttg::k_project_tma<false, 64>);
      const int occ = std::max(kernel_occupancy((const void*)kern, kern, ttg::kThreads, smem), 1);
      const int gx = (int)std::min<long long>((long long)c->num_sms * occ, std::max<long long>(1, args.n_tiles));
      char nm[64];
      std::snprintf(nm, sizeof nm, "k_project[a=%d,r=%d]", a, r);
      prof_begin(c, nm, 8.0 * ((double)a + r) * L, 2.0 * a * r * (double)L);
      launch_k(c, kern, gx, ttg::kThreads, smem, tm, args);
      post_launch(c);
      return tsq != nullptr;
    }
    args.frag_smem = 0;
    args.n_tiles = (L + ttg::kTC - 1) / ttg::kTC;
  }
  size_t smem = (db ? 2 : 1) * stage;
  if (smem > c->smem_optin - 1024) {  // does not fit the tile pipeline: generic path
    gemm<true, false>(c, W, ldw, X, a, out, r, r, L, a, 1.0, 0.0);
    return false;
  }
  if (smem + sizeof(double) * nfr <= std::min<size_t>(c->smem_optin - 1024, 110 * 1024)) {
    args.frag_smem = 1;
    smem += sizeof(double) * nfr;
  }
  const bool regw = db && a8 <= 64 && r8 <= 16;
  auto kern = regw ? ttg::k_project<true, true> : (db ? ttg::k_project<true, false> : ttg::k_project<false, false>);
  const int occ = std::max(kernel_occupancy((const void*)kern, kern, ttg::kThreads, smem), 1);
  const int gx = (int)std::min<long long>((long long)c->num_sms * occ, std::max<long long>(1, args.n_tiles));
  char nm[64];
  std::snprintf(nm, sizeof nm, "k_project[a=%d,r=%d]", a, r);
  prof_begin(c, nm, 8.0 * ((double)a + r) * L, 2.0 * a * r * (double)L);
  launch_k(c, kern, gx, ttg::kThreads, smem, args);
  post_launch(c);
  return tsq != nullptr;
}

// W' = (I_n (x) Psi) U : (As*n) x rn, the combined interface matrix of the
// pending pre-projection and U (a = r*n rows).  One small GEMM:
// Psi (As x r) * U viewed as r x (n*rn)  ->  As x (n*rn) == (As*n) x rn.
const double* combine_psi(ttg_ctx* c, const Src& s, int64_t n, const double* U, int64_t rn, DevBuf& dst) {
  dst.ensure(sizeof(double) * (size_t)(s.As * n * rn));
  gemm<false, false>(c, s.Psi, s.As, U, s.r, dst.as<double>(), s.As, s.As, n * rn, s.r, 1.0, 0.0);
  return dst.as<double>();
}

// out (rn x L_i) = U^T cur_i   (U: a_i x rn, ld a_i), through the pending Psi
bool project_src(ttg_ctx* c, const Src& s, int64_t n, const double* U, int64_t rn, double* out, double* tsq) {
  const long long L = s.Ls / n;
  if (!s.Psi) return project(c, s.S, (int)(s.As * n), L, U, (int)rn, (int)(s.As * n), out, tsq);
  const double* W = combine_psi(c, s, n, U, rn, c->wcomb);
  return project(c, s.S, (int)(s.As * n), L, W, (int)rn, (int)(s.As * n), out, tsq);
}

// materialise cur_i itself (accurate path on a pre-projected source)
const double* materialise(ttg_ctx* c, const Src& s, int64_t n, DevBuf& dst) {
  if (!s.Psi) return s.S;
  const int64_t rows = s.As * n, a = s.r * n;
  c->wcomb.ensure(sizeof(double) * (size_t)(rows * a));
  prof_begin(c, "k_kron_eye", 8.0 * rows * a, 0.0);
  launch_k(c, ttg::k_kron_eye, grid_for(rows * a, 256, 1024), 256, 0, s.Psi, (int)s.As, (int)s.r, (int)n,
                                                                         c->wcomb.as<double>());
  post_launch(c);
  const long long L = s.Ls / n;
  dst.ensure(sizeof(double) * (size_t)(a * L));
  project(c, s.S, (int)rows, L, c->wcomb.as<double>(), (int)a, (int)rows, dst.as<double>());
  return dst.as<double>();
}

// Collectives off while an already-gathered operand is processed (RAII).
struct NoColl {
  ttg_ctx* c;
  bool prev;
  explicit NoColl(ttg_ctx* cc) : c(cc), prev(cc->coll) { c->coll = false; }
  ~NoColl() { c->coll = prev; }
};

// Tall unfolding a > 2 L (the reference's QR branch, truncated_svd.cpp:51-59):
// R = cur - U (U^T cur) explicitly (a x L, selection applied; all-gathered
// across ranks, L is small), the eigen-problem on the L x L side -- R^T R, or
// the TSQR factor of R^T when the Gram cannot resolve the decision -- and
// u_j = R v_j / |R v_j| with the sign rule (k_tall_u) into c->UR.  a can be
// thousands (configs[2] modes 6-7: a ~ 3000, L = 96 / 32) at the cost of an
// L x L eigen-solve; the accurate path needs L <= 128, not a.
EigResult tall_eig(ttg_ctx* c, const Src& src, int64_t n_i, const double* U, int r_old, const uint8_t* sel,
                   long long cpo, long long kmax, const double* dsrc, double dmult, int hint, int& accurate,
                   int& unstable) {
  const int64_t a = src.r * n_i;
  const long long L = src.Ls / n_i;
  const double* X = materialise(c, src, n_i, c->matbuf);
  c->tallR.ensure(sizeof(double) * (size_t)std::max<long long>(a * L, 1));
  double* R = c->tallR.as<double>();
  CK(cudaMemcpyAsync(R, X, sizeof(double) * (size_t)(a * L), cudaMemcpyDeviceToDevice, c->stream));
  if (r_old > 0) {
    c->W.ensure(sizeof(double) * (size_t)std::max<long long>((long long)r_old * L, 1));
    double* P = c->W.as<double>();
    gemm<true, false>(c, U, a, X, a, P, r_old, r_old, L, a, 1.0, 0.0);   // P = U^T X
    gemm<false, false>(c, U, a, P, r_old, R, a, a, L, r_old, -1.0, 1.0);  // R = X - U P
  }
  if (sel) {
    prof_begin(c, "k_mask_cols", 16.0 * a * L, 0.0);
    launch_k(c, ttg::k_mask_cols, grid_for((long long)a * L, 256, 4096), 256, 0, R, (int)a, L, sel, cpo);
    post_launch(c);
  }
  const long long Lg = L * c->world;
  double* Rg = R;
  if (c->coll) {
    c->tallRg.ensure(sizeof(double) * (size_t)(a * Lg));
    Rg = c->tallRg.as<double>();
    allgather(c, R, Rg, (size_t)(a * L));
  }
  NoColl nc(c);  // every rank now holds the same Rg: local, identical solves
  c->G.ensure(sizeof(double) * (size_t)(Lg * Lg));
  gemm<true, false>(c, Rg, a, Rg, a, c->G.as<double>(), Lg, Lg, Lg, a, 1.0, 0.0);  // R^T R (exactly symmetric)
  EigResult er = eig(c, (int)Lg, kmax, dsrc, dmult, 0, hint);
  if (needs_accurate(er)) {
    if (accurate_supported((int)Lg, 0)) {
      c->tallXt.ensure(sizeof(double) * (size_t)(a * Lg));
      double* Xt = c->tallXt.as<double>();
      prof_begin(c, "k_transpose", 16.0 * a * Lg, 0.0);
      launch_k(c, ttg::k_transpose, dim3((unsigned)((Lg + 31) / 32), (unsigned)((a + 31) / 32)), dim3(32, 8), 0,
               (const double*)Rg, (int)a, Lg, Xt);
      post_launch(c);
      er = accurate_eig(c, Xt, (int)Lg, a, nullptr, 0, (int)Lg, nullptr, 1, kmax, dsrc, dmult);
      accurate++;
    } else {
      unstable++;
      if (std::getenv("TTG_STRICT"))
        fail(TTG_E_NUMERIC, "svd_trunc: threshold below the Gram eigen-solve's resolution on a tall " +
                                std::to_string(a) + " x " + std::to_string(Lg) + " residual");
    }
  }
  if (er.rank > 0) {
    c->UR2.ensure(sizeof(double) * (size_t)(a * er.rank));
    prof_begin(c, "k_tall_u", 8.0 * (a * Lg + a * er.rank), 2.0 * a * Lg * er.rank);
    launch_k(c, ttg::k_tall_u, (unsigned)er.rank, 256, 0, (const double*)Rg, (int)a, (int)Lg,
             (const double*)c->UR.as<double>(), c->UR2.as<double>());
    post_launch(c);
    std::swap(c->UR, c->UR2);
  }
  return er;
}

// ---- helpers -----------------------------------------------------------------
int64_t prod(const std::vector<int64_t>& v) {
  int64_t p = 1;
  for (auto x : v) p *= x;
  return p;
}

const double* stage_input(ttg_ctx* c, const double* y, int where, size_t n) {
  if (where == TTG_DEVICE) return y;
  if (where != TTG_HOST) fail(TTG_E_ARGUMENT, "where must be TTG_HOST or TTG_DEVICE");
  for (int i = 0; i < 2; ++i) {  // consumed a ttg_prefetch slot: wait for its copy, no transfer here
    auto& s = c->pf[i];
    if (s.valid && s.src == y && s.n == (int64_t)n) {
      CK(cudaStreamWaitEvent(c->stream, s.ready, 0));
      s.valid = false;
      c->pf_inuse = i;
      return s.buf.as<double>();
    }
  }
  c->ystage.ensure(sizeof(double) * n);
  CK(cudaMemcpyAsync(c->ystage.p, y, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  c->h2d += (int64_t)(sizeof(double) * n);
  return c->ystage.as<double>();
}

void check_shape_args(const int64_t* shape, int ndim) {
  if (!shape || ndim < 1) fail(TTG_E_ARGUMENT, "shape must be non-null with ndim >= 1");
  for (int i = 0; i < ndim; ++i)
    if (shape[i] < 1) fail(TTG_E_DIMENSION, "tensor extent must be >= 1");
}

// preconditions of tt_ice.cpp:16-30 / tt_project tensor_train.cpp:196-208
void check_train_vs_y(const ttg_tt* tt, const int64_t* shape, int ndim, bool state_first) {
  if (state_first && tt->ortho_count != tt->d)
    fail(TTG_E_STATE, "incremental update requires a fully orthonormal train");
  if (ndim != tt->d + 1) fail(TTG_E_DIMENSION, "increment must carry the spatial shape plus an observation mode");
  for (int i = 0; i < tt->d; ++i)
    if (shape[i] != tt->modes[i]) fail(TTG_E_DIMENSION, "increment spatial shape does not match the train");
}

// Sharded batch: every rank must carry the same number of observations.  The
// check rides on the first exchange of the update (the |Y|^2 all-reduce, which
// carries b and b^2 in scal[1..2]) and is evaluated where |Y|^2 reaches the
// host (read_scalar), before anything is mutated: no extra all-reduce or host
// synchronisation per call.
int64_t global_obs(ttg_ctx* c, int64_t b) {
  if (!c->coll) return b;
  c->scal.ensure(sizeof(double) * 16);
  c->h_scal[14] = (double)b;
  c->h_scal[15] = (double)b * (double)b;
  CK(cudaMemcpyAsync(c->scal.as<double>() + 1, c->h_scal + 14, 2 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  c->shard_check = true;
  return b * c->world;
}

// coefficients (r x b_local, compact) -> last core columns [n_obs, n_obs + b_global)
void append_last_core(ttg_ctx* c, ttg_tt* tt, const double* coeffs, int r, int64_t b_local) {
  int64_t bg = b_local * c->world;
  const double* src = coeffs;
  if (c->coll) {
    c->coeffs_all.ensure(sizeof(double) * (size_t)r * bg);
    allgather(c, coeffs, c->coeffs_all.as<double>(), (size_t)r * b_local);
    src = c->coeffs_all.as<double>();
  }
  int64_t need_rc = std::max<int64_t>(r, 1), need_oc = tt->n_obs + bg;
  if (need_rc > tt->rc || need_oc > tt->oc) {
    int64_t nrc = std::max(need_rc, tt->rc), noc = std::max(need_oc, tt->oc);
    if (need_rc > tt->rc) nrc = std::max<int64_t>(need_rc + 8, tt->rc * 3 / 2);
    if (need_oc > tt->oc) noc = std::max<int64_t>(need_oc, tt->oc * 2);
    DevBuf nb;
    nb.ensure(sizeof(double) * (size_t)nrc * noc);
    CK(cudaMemsetAsync(nb.p, 0, sizeof(double) * (size_t)nrc * noc, c->stream));
    if (tt->n_obs > 0)
      CK(cudaMemcpy2DAsync(nb.p, sizeof(double) * nrc, tt->last.p, sizeof(double) * tt->rc,
                           sizeof(double) * tt->rc, tt->n_obs, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    tt->last = std::move(nb);
    tt->rc = nrc;
    tt->oc = noc;
  }
  CK(cudaMemcpy2DAsync(tt->last.as<double>() + tt->rc * tt->n_obs, sizeof(double) * tt->rc, src,
                       sizeof(double) * r, sizeof(double) * r, bg, cudaMemcpyDeviceToDevice, c->stream));
  tt->n_obs += bg;
  tt->bounds.push_back(tt->n_obs);
}

void set_core(ttg_ctx* c, ttg_tt* tt, int i, const double* src, size_t n) {
  tt->cores[i].ensure(sizeof(double) * std::max<size_t>(n, 1), false, c->stream);
  if (src != tt->cores[i].p)
    CK(cudaMemcpyAsync(tt->cores[i].p, src, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
}

void fill_report_ranks(int64_t* dst, const ttg_tt* tt) {
  for (int i = 0; i <= tt->d; ++i) dst[i] = tt->ranks[i];
  dst[tt->d + 1] = 1;
}

// |x|^2 -> c->h_scal[0], valid after the caller's next stream synchronisation
void sumsq_device_async(ttg_ctx* c, const double* x, long long n) {
  // reuse the per-observation kernel with one "observation"
  c->sumsq_part.ensure(sizeof(double) * 64);
  c->scal.ensure(sizeof(double) * 16);
  dim3 grid(1, 1);
  prof_begin(c, "k_sumsq_obs", 8.0 * n, 2.0 * n);
  launch_k(c, ttg::k_sumsq_obs, grid, 256, 0, x, n, 1, c->sumsq_part.as<double>());
  post_launch(c);
  c->d2h += sizeof(double);
  CK(cudaMemcpyAsync(c->h_scal, c->sumsq_part.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
}

double sumsq_device(ttg_ctx* c, const double* x, long long n) {
  sumsq_device_async(c, x, n);
  CK(cudaStreamSynchronize(c->stream));
  return c->h_scal[0];
}

// ---- the TT-ICE / TT-ICE* sweep -----------------------------------------------
struct SweepOpts {
  bool star = false;
  double tau = 0.8;
  const uint8_t* sel = nullptr;   // TT-ICE*: selected observations (local)
  int64_t n_sel_global = 0;       // TT-ICE*: |D|
  bool bootstrap = false;
  const double* delta_src = nullptr;  // delta = mult * sqrt(*src) (uniform) ...
  double delta_mult = 0.0;
  const double* deltas = nullptr;     // ... or per-mode absolute deltas (host)
  double y_norm = 0.0;                // known only for the per-mode-delta API
  bool need_norms = false;            // fuse |y_o|^2 into the first pass over Y
  bool reuse_stats = false;           // TT-ICE*: intermediates of the stats chain are valid
  bool speculate = true;              // size the launches after a k_decide mode with the rank hint, verify once
};

struct SweepOut {
  double discarded_sq = 0.0;
  int guards = 0;
  int modes_updated = 0;
  int accurate_modes = 0;
  int raw_fallbacks = 0;
  int gram_only_unstable = 0;
  int tall_modes = 0;
  bool cores_changed = false;
  const double* coeffs = nullptr;  // r_d x b_local (compact)
  int r_d = 0;
};

// Norms of the increment: fused into the first kernel that streams Y (per-tile
// sums of squares, then a fixed-order per-observation reduction), or a
// separate pass when tiles would straddle observations.
struct Norms {
  bool pending = false;
  const double* Y = nullptr;
  int64_t S = 0, b = 0;
};

double* norms_tiles_for(ttg_ctx* c, Norms& nm, const double* src, int64_t rows, long long L) {
  if (!nm.pending || src != nm.Y) return nullptr;
  if (!tiles_align(rows, nm.S)) {
    obs_norms(c, nm.Y, nm.S, (int)nm.b);
    nm.pending = false;
    return nullptr;
  }
  const long long nt = (L + ttg::kTC - 1) / ttg::kTC;
  c->tsq.ensure(sizeof(double) * (size_t)nt * ttg::kConsumerWarps);
  return c->tsq.as<double>();
}

void norms_finish(ttg_ctx* c, Norms& nm, int64_t rows, bool produced) {
  if (!produced) {
    obs_norms(c, nm.Y, nm.S, (int)nm.b);
  } else {
    c->on2.ensure(sizeof(double) * nm.b);
    c->scal.ensure(sizeof(double) * 16);
    const long long tpo = nm.S / (rows * ttg::kTC);
    prof_begin(c, "k_tiles_to_obs", 8.0 * tpo * ttg::kConsumerWarps * nm.b, 0.0);
    launch_k(c, ttg::k_tiles_to_obs, (unsigned)nm.b, 256, 0, c->tsq.as<double>(), tpo, (int)nm.b,
                                                                 c->on2.as<double>(), nullptr);
    post_launch(c);
    prof_begin(c, "k_sum_vec", 8.0 * nm.b, 0.0);
    launch_k(c, ttg::k_sum_vec, 1, 256, 0, c->on2.as<double>(), (int)nm.b, c->scal.as<double>());
    post_launch(c);
    allreduce_sum(c, c->scal.as<double>(), 3);  // |Y|^2 and the shard-size check (global_obs)
  }
  nm.pending = false;
}

void check_finite_norm(double ysq) {
  if (!std::isfinite(ysq)) fail(TTG_E_NUMERIC, "non-finite element rejected at tensor construction");
}

// next-mode fusion rule: the next Gram / projection reads the same buffer
// through the combined pre-projection when its tile still fits the fast path
bool can_fuse(const Src& s, int64_t n_i, int64_t r_new, int64_t n_next, int64_t r_old_next) {
  return s.As * n_i * n_next <= kFastMax && ttg::round_up((int)(r_new * n_next), 8) <= kFastMax &&
         ttg::round_up((int)std::max<int64_t>(r_old_next, 1), 8) <= kFastMax;
}

// What a speculative sweep needs to be undone (owned by sweep(), filled by sweep_impl())
struct SpecState {
  bool any_spec = false;
  bool spec_on = false;  // replaced cores were kept aside (the train can be handed back as it was)
  std::vector<char> swapped;
  std::vector<int64_t> old_ranks;
  std::vector<int> hints_before;
};
SweepOut sweep_impl(ttg_ctx* c, ttg_tt* tt, const double* Y, int64_t b, const SweepOpts& o, Norms& nm, SpecState& st);

// Guesses are only worth making for a train whose per-mode ranks repeat: a wrong
// guess costs a second sweep.  hint_repeats counts the consecutive sweeps that
// kept the same number of directions in every mode as the sweep before.
void note_ranks(ttg_tt* tt) {
  if (tt->mode_hint == tt->hint_prev && !tt->mode_hint.empty()) ++tt->hint_repeats;
  else tt->hint_repeats = 0;
  tt->hint_prev = tt->mode_hint;
}

SweepOut sweep(ttg_ctx* c, ttg_tt* tt, const double* Y, int64_t b, const SweepOpts& o, Norms& nm) {
  SpecState st;
  auto undo = [&] {
    c->spec_redone++;
    for (size_t i = 0; i < st.swapped.size(); ++i)
      if (st.swapped[i]) std::swap(tt->cores[i], c->corebak[i]);
    tt->ranks = st.old_ranks;
    tt->mode_hint = st.hints_before;
    tt->spec_hold = std::min(8, 2 * tt->spec_hold + 1);
  };
  try {
    SweepOut out = sweep_impl(c, tt, Y, b, o, nm, st);
    c->spec_active = false;
    if (st.any_spec && tt->spec_hold > 0) --tt->spec_hold;  // (trust returns one verified sweep at a time)
    note_ranks(tt);
    return out;
  } catch (const SpecRejected&) {
    c->spec_active = false;
    undo();
  } catch (const TtgError&) {
    c->spec_active = false;
    // launches sized by a wrong guess may fail on their own (a solver that does
    // not converge on garbage): only a failure of the synchronous sweep counts
    if (!st.any_spec) {
      // a genuine failure: hand the kept-aside cores back before it propagates
      for (size_t i = 0; i < st.swapped.size(); ++i)
        if (st.swapped[i]) std::swap(tt->cores[i], c->corebak[i]);
      if (st.spec_on && !st.old_ranks.empty()) {
        tt->ranks = st.old_ranks;
        tt->mode_hint = st.hints_before;
      }
      throw;
    }
    undo();
  }
  tt->spec_wait = tt->spec_hold;
  SweepOpts o2 = o;
  o2.speculate = false;
  SpecState st2;
  SweepOut out = sweep_impl(c, tt, Y, b, o2, nm, st2);
  note_ranks(tt);
  return out;
}

SweepOut sweep_impl(ttg_ctx* c, ttg_tt* tt, const double* Y, int64_t b, const SweepOpts& o, Norms& nm, SpecState& st) {
  SweepOut out;
  tt->gen = ttg_tt::next_gen();  // the sweep rewrites the cores
  c->gcount.ensure(sizeof(int));
  CK(cudaMemsetAsync(c->gcount.p, 0, sizeof(int), c->stream));
  // Speculative sweep: a mode solved by k_decide does not wait for its rank --
  // the host sizes the following launches with the rank this mode kept at the
  // previous update, the kernel flags any disagreement, and flag + per-mode
  // results are read once at the end.  A flagged sweep is undone (the replaced
  // cores are kept aside until then) and repeated with a host read per mode.
  // A train whose last guesses were rejected sits out a growing number of sweeps
  // (1, 3, 7, 8 ...): alternating rank patterns must not pay for two sweeps every time.
  bool spec_on = o.speculate && !o.bootstrap && !std::getenv("TTG_NO_SPEC");
  if (spec_on && tt->hint_repeats < 1) spec_on = false;  // the last two sweeps did not agree: no guess
  if (spec_on) {
    // a guess saves one host read per k_decide mode and risks a second sweep: only
    // when (nearly) every mode of the train is one (judged on the current ranks)
    int eligible = 0;
    for (int i = 0; i < tt->d; ++i) {
      const int hint = i < (int)tt->mode_hint.size() ? tt->mode_hint[i] : -1;
      const int64_t a = tt->ranks[i] * tt->modes[i];
      if (!(a & 1) && decide_applies(c, false, a, tt->ranks[i + 1], hint)) ++eligible;
    }
    if (eligible + 2 < tt->d) spec_on = false;
  }
  if (spec_on && tt->spec_wait > 0) {
    --tt->spec_wait;
    spec_on = false;
  }
  st.spec_on = spec_on;
  std::vector<char> spec_mode(tt->d, 0);
  std::vector<char>& swapped = st.swapped;
  swapped.assign(tt->d, 0);
  std::vector<double> tails(tt->d, 0.0);
  st.hints_before = tt->mode_hint;
  bool& any_spec = st.any_spec;
  if (spec_on) {
    c->specflag.ensure(sizeof(int));
    c->eiglog.ensure(sizeof(EigResult) * (TTG_MAX_CORES + 1));
    CK(cudaMemsetAsync(c->specflag.p, 0, sizeof(int), c->stream));
    if ((int)c->corebak.size() < tt->d) c->corebak.resize(tt->d);
  }
  const int d = tt->d;
  const int64_t S = prod(tt->modes);
  std::vector<int64_t> old_ranks = tt->ranks;
  st.old_ranks = old_ranks;
  Src src{Y, 1, S * b, nullptr, 1};
  int flip = 0, pf = 0;
  bool unchanged = true;
  bool norm_checked = !o.need_norms;
  // U_pad of mode 0 is core 0 itself (r_left = 1 never grows)
  const double* Upad = tt->cores.empty() ? nullptr : tt->cores[0].as<double>();
  int64_t r_old = o.bootstrap ? 0 : old_ranks[1];
  for (int i = 0; i < d; ++i) {
    const int64_t n_i = tt->modes[i];
    const int64_t a = src.r * n_i;
    const long long L = src.Ls / n_i;
    const long long cpo = L / b;
    const bool was_unchanged = unchanged;
    const double* dsrc = o.deltas ? nullptr : o.delta_src;
    const double dmult = o.deltas ? o.deltas[i] : o.delta_mult;
    int64_t r_R = 0;
    bool run_svd = true;
    bool decided = false;  // k_decide solved the mode and wrote the appended core
    bool speculated = false;  // ... and the host did not wait for it (verified at the end of the sweep)
    if (o.star) {
      run_svd = (double)r_old / (double)a < o.tau;  // occupancy on the padded core, tt_ice_star.cpp:246-248
    } else if (!o.bootstrap && r_old == a) {
      // A square orthogonal basis leaves an identically zero residual; the
      // reference's SVD of its rounding noise returns rank 0 whenever
      // delta > 1e-12 |Y|; below that, run the full computation.
      const bool big = o.deltas ? (dmult > 1e-12 * o.y_norm) : (dmult > 1e-12);
      run_svd = !big;
    }
    const long long Lg = L * c->world;
    // tall: the reference's own QR branch (a > 2 L, truncated_svd.cpp:51-59), and
    // any a x L residual too large for one CTA's shared memory whose L x L side
    // is the smaller eigen-problem
    const bool tall = run_svd && a > kFastMax && !std::getenv("TTG_NO_TALL") &&
                      ((double)a > 2.0 * (double)Lg || (a > 256 && Lg < a));
    if (run_svd && !tall && a > 4096)
      fail(TTG_E_RESOURCE, "unfolding rows a_i = " + std::to_string(a) + " exceed the device solver limit");
    if (tall) {
      if (nm.pending && src.S == nm.Y) norms_finish(c, nm, 0, false);
      if (!norm_checked && !nm.pending) {
        check_finite_norm(read_scalar(c, c->scal.as<double>()));
        norm_checked = true;
      }
      const long long kmax = o.star ? o.n_sel_global * cpo : Lg;
      if ((int)tt->mode_hint.size() < d) tt->mode_hint.assign(d, -1);
      EigResult er = tall_eig(c, src, n_i, r_old > 0 ? Upad : nullptr, (int)r_old, o.star ? o.sel : nullptr, cpo,
                              kmax, dsrc, dmult, tt->mode_hint[i], out.accurate_modes, out.gram_only_unstable);
      r_R = er.rank;
      tails[i] = er.tail_sq;
      out.tall_modes++;
      tt->mode_hint[i] = (int)r_R;
    } else if (run_svd) {
      const uint8_t* sel = o.star ? o.sel : nullptr;
      const int64_t rows = src.Psi ? src.As * n_i : a;
      double* tsq = norms_tiles_for(c, nm, src.S, rows, L);
      const double sel_frac = o.star ? (double)o.n_sel_global / (double)(b * c->world) : 1.0;
      // raw Gram (SYRK + small-side projector) for every source; the explicit
      // residual kernel is the accuracy fallback below
      const bool raw = !std::getenv("TTG_NO_RAW_GRAM") && (src.Psi || ttg::round_up((int)a, 8) > 0);
      if ((int)tt->mode_hint.size() < d) tt->mode_hint.assign(d, -1);
      const int hint = tt->mode_hint[i];
      // one launch for P C P, the eigen-solve and the append (ttg_decide.cuh)
      if ((int)tt->decide_off.size() < d) tt->decide_off.assign(d, 0);
      const bool dec_held = tt->decide_off[i] > 0;
      if (dec_held) --tt->decide_off[i];
      const bool dec = raw && !o.bootstrap && !(a & 1) && !dec_held && decide_applies(c, src.Psi != nullptr, a, r_old, hint);
      bool did;
      if (dec) did = syrk(c, src.S, (int)a, L, sel, cpo, sel_frac, tsq);  // C -> c->G
      else did = raw ? gram_raw_src(c, src, n_i, r_old > 0 ? Upad : nullptr, (int)r_old, sel, cpo, sel_frac, tsq)
                     : gram_src(c, src, n_i, r_old > 0 ? Upad : nullptr, (int)r_old, sel, cpo, sel_frac, tsq);
      if (tsq) norms_finish(c, nm, rows, did);
      if (!norm_checked && !nm.pending) {  // reject non-finite input before anything is mutated
        check_finite_norm(read_scalar(c, c->scal.as<double>()));
        norm_checked = true;
      }
      const long long kmax = o.star ? o.n_sel_global * cpo : L * c->world;
      trace("sweep:gram launched");
      EigResult er;
      if (dec) {
        const bool alias = (Upad == tt->cores[i].p);
        if (spec_on && !alias) {  // the sweep replaces this core: keep the old one until verified
          std::swap(tt->cores[i], c->corebak[i]);
          swapped[i] = 1;
        }
        tt->cores[i].ensure(sizeof(double) * (size_t)a * (r_old + decide_block(hint) - 1), /*keep=*/alias, c->stream);
        if (alias) Upad = tt->cores[i].as<double>();
        decide_launch(c, (int)a, (int)r_old, Upad, tt->cores[i].as<double>(), kmax, dsrc, dmult, hint,
                      spec_on ? hint : -1, c->specflag.as<int>(), spec_on ? c->eiglog.as<EigResult>() + i : nullptr);
        if (spec_on) {
          er = EigResult{};
          er.rank = hint;
          er.converged = 1;
          spec_mode[i] = 1;
          any_spec = true;
          c->spec_active = true;
          speculated = true;
        } else {
          er = eig_fetch(c);
        }
        if (std::getenv("TTG_DEBUG"))
          std::fprintf(stderr, "[ttg] decide a=%d r=%d K=%d conv=%d iters=%d rank=%d lam_max=%.3e tail=%.3e dev=%.2e\n", (int)a,
                       (int)r_old, decide_block(hint), er.converged, er.sweeps, er.rank, er.lam_max, er.tail_sq, er.dev);
        if (std::getenv("TTG_DEBUG"))
          std::fprintf(stderr, "[ttg] decide cycles init=%lld pass1=%lld tgram=%lld zupd=%lld hs+rr=%lld rows+dec=%lld pass=%lld final=%lld\n",
                       er.t_phase[0] & 0xffffffffll, er.t_phase[0] >> 32, er.t_phase[1] & 0xffffffffll, er.t_phase[1] >> 32,
                       er.t_phase[2] & 0xffffffffll, er.t_phase[2] >> 32, er.t_phase[3] & 0xffffffffll, er.t_phase[3] >> 32);
        if (!er.converged && er.sweeps < ttg::kDecIters && decide_block(hint) == 2 && decide_applies(c, false, a, r_old, 2)) {
          // more directions than a block of 2 holds (not: no convergence): a block of 4 from the same C before the
          // explicit chain (whose block attempts re-read the a x a Gram from L2 per iteration)
          const bool alias4 = (Upad == tt->cores[i].p);
          tt->cores[i].ensure(sizeof(double) * (size_t)a * (r_old + 3), /*keep=*/alias4, c->stream);
          if (alias4) Upad = tt->cores[i].as<double>();
          decide_launch(c, (int)a, (int)r_old, Upad, tt->cores[i].as<double>(), kmax, dsrc, dmult, 2, -1,
                        c->specflag.as<int>(), nullptr);
          er = eig_fetch(c);
        }
        if (er.converged) {
          decided = true;
        } else {  // more directions than the block holds, or no gap: the explicit chain from the same C
          if (er.sweeps >= ttg::kDecIters) tt->decide_off[i] = 4;  // (a spectrum without a gap tends to stay one)
          pcp_from_c(c, src, n_i, Upad, (int)r_old, did);
          er = eig(c, (int)a, kmax, dsrc, dmult, 0, std::max(hint, decide_block(hint)));
        }
      } else {
        er = eig(c, (int)a, kmax, dsrc, dmult, 0, hint);
      }
      trace("sweep:eig done");
      if (!speculated && raw && er.rank > 0 && r_old > 0) {  // no projector (empty basis): C is G exactly
        // raw-Gram cancellation costs ~eps*tr(C)/gap in the kept vectors: keep
        // it only for directions carrying >= 1e-3 of the source energy
        const double trC = c->h_scal[8];  // trace(C), fetched with the eigen result
        if (er.lam_min_kept < 1e-3 * trC) {
          gram_src(c, src, n_i, r_old > 0 ? Upad : nullptr, (int)r_old, sel, cpo, sel_frac, nullptr);
          er = eig(c, (int)a, kmax, dsrc, dmult, 0, er.rank);
          out.raw_fallbacks++;
          decided = false;
        }
      }
      if (!speculated && needs_accurate(er)) {
        if (accurate_supported((int)a, (int)r_old)) {
          const double* X = materialise(c, src, n_i, c->matbuf);
          er = accurate_eig(c, X, (int)a, L, r_old > 0 ? Upad : nullptr, (int)r_old, (int)a, sel, cpo, kmax, dsrc,
                            dmult);
          out.accurate_modes++;
          decided = false;
        } else {
          out.gram_only_unstable++;  // surfaced in ttg_report; TTG_STRICT turns it into a NumericError
          if (std::getenv("TTG_STRICT"))
            fail(TTG_E_NUMERIC, "svd_trunc: threshold below the Gram eigen-solve's resolution on a " + std::to_string(a) +
                                    "-row unfolding and no factor path applies");
        }
      }
      r_R = er.rank;
      tails[i] = er.tail_sq;
      tt->mode_hint[i] = (int)r_R;
      if (decided && er.guard == 2) decided = false;  // Gram-deviation guard fired: k_append's correction
    }
    if (spec_on && !swapped[i] && Upad != tt->cores[i].p) {  // this mode's core is about to be replaced
      std::swap(tt->cores[i], c->corebak[i]);
      swapped[i] = 1;
    }
    int64_t r_new;
    bool zero_next = false;
    if (o.bootstrap) {
      if (r_R == 0) {  // tt_svd.cpp:42-47 unit-column placeholder, next carry = 0
        r_new = 1;
        std::vector<double> e1((size_t)a, 0.0);
        e1[0] = 1.0;
        tt->cores[i].ensure(sizeof(double) * a);
        CK(cudaMemcpyAsync(tt->cores[i].p, e1.data(), sizeof(double) * a, cudaMemcpyHostToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        zero_next = true;
      } else {
        r_new = r_R;
        set_core(c, tt, i, c->UR.as<double>(), (size_t)a * r_new);
      }
      out.cores_changed = true;
      unchanged = false;
    } else if (r_R > 0) {
      r_new = r_old + r_R;
      const bool alias = (Upad == tt->cores[i].p);
      tt->cores[i].ensure(sizeof(double) * (size_t)a * r_new, /*keep=*/alias, c->stream);
      if (alias) Upad = tt->cores[i].as<double>();  // keep aliasing valid after growth
      // (k_decide already wrote [U_pad U_R] unless its Gram-deviation guard fired)
      if (!decided)
        out.guards += append(c, Upad, (int)a, (int)r_old, (int)r_R, tt->cores[i].as<double>());
      out.cores_changed = true;
      out.modes_updated++;
      unchanged = false;
    } else {
      r_new = r_old;
      if (Upad != tt->cores[i].p) unchanged = false;  // padded core (an earlier mode grew)
      set_core(c, tt, i, Upad, (size_t)a * r_new);
    }
    const double* Ui = tt->cores[i].as<double>();
    if (i + 1 < d) {
      const int64_t n_next = tt->modes[i + 1];
      const int64_t rl_old = o.bootstrap ? 1 : old_ranks[i + 1];
      const int64_t rr_old = o.bootstrap ? 0 : old_ranks[i + 2];
      if (zero_next) {
        c->cur[flip].ensure(sizeof(double) * (size_t)std::max<long long>(L, 1));
        CK(cudaMemsetAsync(c->cur[flip].p, 0, sizeof(double) * L, c->stream));
        src = Src{c->cur[flip].as<double>(), 1, L, nullptr, 1};
        flip ^= 1;
      } else if (can_fuse(src, n_i, r_new, n_next, rr_old)) {
        const double* psi = src.Psi ? combine_psi(c, src, n_i, Ui, r_new, c->psi[pf]) : Ui;
        if (src.Psi) pf ^= 1;
        src = Src{src.S, src.As * n_i, L, psi, r_new};
      } else if (o.reuse_stats && unchanged && c->stat_has.size() > (size_t)(i + 1) && c->stat_has[i + 1]) {
        src = Src{c->scur[i + 1].as<double>(), r_new, L, nullptr, r_new};
      } else if (o.reuse_stats && was_unchanged && r_R > 0 && c->stat_has.size() > (size_t)(i + 1) &&
                 c->stat_has[i + 1] && r_old > 0) {
        // only mode i grew (appended columns): cur_{i+1} = [stats rows ; r_R new rows]
        c->tmp.ensure(sizeof(double) * (size_t)std::max<long long>(r_R * L, 1));
        project_src(c, src, n_i, Ui + (size_t)a * r_old, r_R, c->tmp.as<double>(), nullptr);
        c->cur[flip].ensure(sizeof(double) * (size_t)std::max<long long>(r_new * L, 1));
        const long long tot = r_new * L;
        prof_begin(c, "k_merge_rows", 8.0 * (double)(2 * r_new) * L, 0.0);
        launch_k(c, ttg::k_merge_rows, grid_for(tot, 256, 8 * c->num_sms), 256, 0, 
            c->scur[i + 1].as<double>(), (int)r_old, c->tmp.as<double>(), (int)r_new, L, c->cur[flip].as<double>());
        post_launch(c);
        src = Src{c->cur[flip].as<double>(), r_new, L, nullptr, r_new};
        flip ^= 1;
      } else {
        c->cur[flip].ensure(sizeof(double) * (size_t)std::max<long long>(r_new * L, 1));
        const int64_t rows = src.Psi ? src.As * n_i : a;
        double* tsq = norms_tiles_for(c, nm, src.S, rows, L);
        const bool did = project_src(c, src, n_i, Ui, r_new, c->cur[flip].as<double>(), tsq);
        if (tsq) norms_finish(c, nm, rows, did);
        src = Src{c->cur[flip].as<double>(), r_new, L, nullptr, r_new};
        flip ^= 1;
      }
      // pad the next core (Eq. 3.4) unless the left rank is unchanged
      if (o.bootstrap) {
        Upad = nullptr;
        r_old = 0;
      } else if (r_new != rl_old) {
        const int64_t tot = r_new * n_next * rr_old;
        c->Upad.ensure(sizeof(double) * (size_t)std::max<int64_t>(tot, 1));
        prof_begin(c, "k_pad_core", 16.0 * tot, 0.0);
        launch_k(c, ttg::k_pad_core, grid_for(tot, 256, 1024), 256, 0, 
            tt->cores[i + 1].as<double>(), (int)rl_old, (int)n_next, (int)rr_old, (int)r_new, c->Upad.as<double>());
        post_launch(c);
        Upad = c->Upad.as<double>();
        r_old = rr_old;
      } else {
        Upad = tt->cores[i + 1].as<double>();
        r_old = rr_old;
      }
    } else {
      c->coeffs.ensure(sizeof(double) * (size_t)std::max<long long>(r_new * L, 1));
      if (zero_next) {
        CK(cudaMemsetAsync(c->coeffs.p, 0, sizeof(double) * r_new * L, c->stream));
        out.coeffs = c->coeffs.as<double>();
      } else if (o.reuse_stats && unchanged) {
        out.coeffs = c->scoeffs.as<double>();  // projection through unchanged cores
      } else {
        const int64_t rows = src.Psi ? src.As * n_i : a;
        double* tsq = norms_tiles_for(c, nm, src.S, rows, L);
        const bool did = project_src(c, src, n_i, Ui, r_new, c->coeffs.as<double>(), tsq);
        if (tsq) norms_finish(c, nm, rows, did);
        out.coeffs = c->coeffs.as<double>();
      }
    }
    tt->ranks[i + 1] = r_new;
    if (i + 1 == d) out.r_d = (int)r_new;
    trace("sweep:mode advanced");
  }
  guards_fetch(c);
  if (any_spec) {
    c->spec_sweeps++;
    c->d2h += sizeof(EigResult) * d + sizeof(int);
    CK(cudaMemcpyAsync(c->h_eiglog, c->eiglog.p, sizeof(EigResult) * d, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(c->h_eiglog + TTG_MAX_CORES, c->specflag.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    const int flag = *reinterpret_cast<const int*>(c->h_eiglog + TTG_MAX_CORES);
    if (std::getenv("TTG_DEBUG")) std::fprintf(stderr, "[ttg] speculative sweep: flag=%d\n", flag);
    if (flag) throw SpecRejected{};  // sweep() undoes it and repeats with a host read per mode
    for (int i = 0; i < d; ++i)
      if (spec_mode[i]) tails[i] = c->h_eiglog[i].tail_sq;
  }
  for (int i = 0; i < d; ++i) out.discarded_sq += tails[i];
  return out;
}

// projection-only chains fuse further: the next projection reads the same
// buffer through the combined interface when k_project_kc takes it (even rows
// <= kProjFuseMax, r <= 34), so Y -> r_3 x L_3 at cfg3 is one pass (no cur_2).
constexpr int kProjFuseMax = 512;
// Without a k_project_kc plan (r > 34) the fused step is a plain GEMM; fuse
// when its per-column time max(F/P, B/BW) beats materialising cur_{i+1}
// (the projection at mode i plus the next one): at full-rank early modes
// (r_i = a_i) fusion removes a whole write + read of the increment.
bool can_fuse_proj(const ttg_ctx* c, const Src& s, int64_t n_i, int64_t r_i, int64_t n_next, int64_t r_next) {
  const int64_t rows = s.As * n_i * n_next;
  if (std::getenv("TTG_NO_PROJ_FUSE")) return rows <= kFastMax && r_next <= kFastMax;
  if (rows > kProjFuseMax) return false;
  KcPlan P;
  if (kc_plan(c, (int)rows, (int)r_next, P)) return true;
  const double Pf = 30e12, BW = 6e12;  // sustained FP64 / HBM rates (profiles/r01_box_probe.log)
  auto t = [&](double f, double b) { return std::max(f / Pf, b / BW); };
  const double src_rows = (double)s.As * n_i;  // rows of the current source per sub-column
  const double fused = t(2.0 * rows * r_next, 8.0 * rows);
  const double staged = t(2.0 * n_next * src_rows * r_i, 8.0 * (rows + r_i * n_next)) +
                        t(2.0 * r_i * n_next * r_next, 8.0 * r_i * n_next);
  return fused <= staged;
}

// Projection of Y through the train's current cores (projection-only fusion
// plan, can_fuse_proj).  cache=true keeps the materialised intermediates (c->scur) and the
// coefficients (c->scoeffs) for reuse by a following TT-ICE* sweep.
// The last modes of a chain in one launch (k_project_tail) once an observation's
// unfolding fits shared memory: returns the coefficient block, or null when the
// tail does not qualify at mode i (the per-mode kernels then carry on).
const double* project_tail(ttg_ctx* c, const ttg_tt* tt, const Src& src, int i, int64_t b, bool cache) {
  const int d = tt->d, nm = d - i;
  if (std::getenv("TTG_NO_TAIL") || src.Psi || nm < 2 || nm > ttg::kTailMaxModes || b <= 0) return nullptr;
  ttg::TailArgs ta{};
  ta.X = src.S;
  ta.nm = nm;
  long long cols = src.Ls / tt->modes[i] / b, rl = src.r;
  if (cols * b * tt->modes[i] != src.Ls) return nullptr;
  double fma_per_obs = 0.0;
  long long obuf = 1;
  for (int t = 0; t < nm; ++t) {
    const long long n = tt->modes[i + t], rr = tt->ranks[i + t + 1];
    if (t > 0) {
      if (cols % n) return nullptr;
      cols /= n;
    }
    if (rl * n > INT32_MAX || rr * cols > INT32_MAX) return nullptr;
    ta.core[t] = tt->cores[i + t].as<double>();
    ta.rows[t] = (int)(rl * n);
    ta.rr[t] = (int)rr;
    ta.cols[t] = (int)cols;
    fma_per_obs += (double)rl * n * rr * cols;
    obuf = std::max(obuf, rr * cols);
    rl = rr;
  }
  if (ta.cols[nm - 1] != 1 || fma_per_obs > 2e6) return nullptr;
  obuf = (obuf + 1) & ~1ll;
  ta.obuf = (int)obuf;
  long long ucap = 1;
  for (int t = 0; t < nm; ++t) ucap = std::max(ucap, (long long)ttg::tail_ld(ta.rows[t]) * ta.rr[t]);
  const size_t smem = sizeof(double) * ((size_t)ttg::tail_ld(ta.rows[0]) * ta.cols[0] + 2 * (size_t)obuf + (size_t)ucap + 8);
  if (smem > dyn_smem_cap((const void*)ttg::k_project_tail)) return nullptr;
  for (int t = 0; t < nm; ++t) {
    const size_t bytes = sizeof(double) * (size_t)std::max<long long>((long long)ta.rr[t] * ta.cols[t] * b, 1);
    if (t + 1 < nm) {
      if (cache) {
        c->scur[i + t + 1].ensure(bytes);
        ta.out[t] = c->scur[i + t + 1].as<double>();
        c->stat_has[i + t + 1] = true;
      } else {
        ta.out[t] = nullptr;
      }
    } else {
      DevBuf& dst = cache ? c->scoeffs : c->coeffs;
      dst.ensure(bytes);
      ta.out[t] = dst.as<double>();
    }
  }
  kernel_occupancy((const void*)ttg::k_project_tail, ttg::k_project_tail, ttg::kTailThreads, smem);
  prof_begin(c, "k_project_tail", 8.0 * ta.rows[0] * ta.cols[0] * b, 2.0 * fma_per_obs * b);
  launch_k(c, ttg::k_project_tail, (unsigned)b, ttg::kTailThreads, smem, ta);
  post_launch(c);
  return ta.out[nm - 1];
}

const double* project_chain(ttg_ctx* c, const ttg_tt* tt, const double* Y, int64_t b, bool cache, Norms& nm) {
  const int d = tt->d;
  const int64_t S = prod(tt->modes);
  Src src{Y, 1, S * b, nullptr, 1};
  int flip = 0, pf = 0;
  if (cache) {
    if ((int)c->scur.size() < d + 1) c->scur.resize(d + 1);
    c->stat_has.assign(d + 1, false);
  }
  for (int i = 0; i < d; ++i) {
    const int64_t n_i = tt->modes[i];
    const long long L = src.Ls / n_i;
    const int64_t r = tt->ranks[i + 1];
    const double* Ui = tt->cores[i].as<double>();
    const int64_t rows = src.Psi ? src.As * n_i : src.r * n_i;
    if (!(nm.pending && src.S == nm.Y))
      if (const double* cf = project_tail(c, tt, src, i, b, cache)) return cf;
    if (i + 1 < d) {
      const int64_t n_next = tt->modes[i + 1];
      const int64_t rr = tt->ranks[i + 2];
      if (can_fuse_proj(c, src, n_i, r, n_next, rr)) {
        const double* psi = src.Psi ? combine_psi(c, src, n_i, Ui, r, c->spsi[pf]) : Ui;
        if (src.Psi) pf ^= 1;
        src = Src{src.S, src.As * n_i, L, psi, r};
        continue;
      }
      DevBuf& dst = cache ? c->scur[i + 1] : c->cur[flip];
      dst.ensure(sizeof(double) * (size_t)std::max<long long>(r * L, 1));
      double* tsq = norms_tiles_for(c, nm, src.S, rows, L);
      const bool did = project_src(c, src, n_i, Ui, r, dst.as<double>(), tsq);
      if (tsq) norms_finish(c, nm, rows, did);
      if (cache) c->stat_has[i + 1] = true;
      trace("chain:materialised");
      src = Src{dst.as<double>(), r, L, nullptr, r};
      flip ^= 1;
    } else {
      trace("chain:last mode");
      DevBuf& dst = cache ? c->scoeffs : c->coeffs;
      dst.ensure(sizeof(double) * (size_t)std::max<long long>(r * L, 1));
      double* tsq = norms_tiles_for(c, nm, src.S, rows, L);
      const bool did = project_src(c, src, n_i, Ui, r, dst.as<double>(), tsq);
      if (tsq) norms_finish(c, nm, rows, did);
      return dst.as<double>();
    }
  }
  return nullptr;
}

// M = Phi^T Phi of the spatial chain -> returns device pointer (r_d x r_d)
const double* interface_gram_compute(ttg_ctx* c, const ttg_tt* tt);
// cached per train generation: a TT-ICE* skip step leaves the cores as they
// were, so the next increment's statistics reuse Phi^T Phi
const double* interface_gram(ttg_ctx* c, const ttg_tt* tt) {
  if (c->iface_gen == tt->gen && c->iface_ptr && !std::getenv("TTG_NO_IFACE_CACHE")) return c->iface_ptr;
  c->iface_ptr = interface_gram_compute(c, tt);
  c->iface_gen = tt->gen;
  return c->iface_ptr;
}
const double* interface_gram_compute(ttg_ctx* c, const ttg_tt* tt) {
  int64_t rmax = 1;
  for (auto r : tt->ranks) rmax = std::max(rmax, r);
  int64_t nmax = 1;
  for (auto n : tt->modes) nmax = std::max(nmax, n);
  c->iface[0].ensure(sizeof(double) * rmax * rmax);
  c->iface[1].ensure(sizeof(double) * rmax * rmax);
  c->Mtmp.ensure(sizeof(double) * rmax * nmax * rmax);
  size_t core_tot = 0;
  for (int i = 0; i < tt->d; ++i) core_tot += (size_t)((tt->ranks[i] * tt->modes[i] + 1) * tt->ranks[i + 1]);
  (void)core_tot;
  const size_t ismem = sizeof(double) * (size_t)(2 * rmax * rmax + 2 * (rmax * nmax + 1) * rmax);
  if (tt->d <= ttg::kIfaceMaxModes && ismem <= 200 * 1024) {  // one launch for the whole chain
    ttg::IfaceArgs ia{};
    ia.d = tt->d;
    double flops = 0.0;
    for (int i = 0; i < tt->d; ++i) {
      ia.cores[i] = tt->cores[i].as<double>();
      ia.rl[i] = (int)tt->ranks[i];
      ia.n[i] = (int)tt->modes[i];
      ia.rr[i] = (int)tt->ranks[i + 1];
      flops += 4.0 * ia.rl[i] * ia.n[i] * ia.rr[i] * (ia.rl[i] + ia.rr[i]);
    }
    ia.rmax = (int)rmax;
    ia.nmax = (int)nmax;
    ia.out = c->iface[0].as<double>();
    kernel_occupancy((const void*)ttg::k_iface_all, ttg::k_iface_all, 1024, ismem);
    prof_begin(c, "k_iface", 8.0 * core_tot, flops);
    launch_k(c, ttg::k_iface_all, 1, 1024, ismem, ia);
    post_launch(c);
    return c->iface[0].as<double>();
  }
  // large ranks: M_i = C_i^T (M_{i-1} C_i) per core on the DMMA GEMM, with C_i
  // viewed as r_{i-1} x (n r_i) for the first product and as (r_{i-1} n) x r_i
  // for the second (the same column-major buffer)
  // (may run on the side stream beside the statistics pass: its own buffers,
  // grown by star_stats before the fork)
  c->iface[0].ensure(sizeof(double) * rmax * rmax);
  c->iface_T.ensure(sizeof(double) * rmax * nmax * rmax);
  c->gemm_ws_side.ensure(sizeof(double) * 64 * rmax * rmax);
  const double one = 1.0;
  CK(cudaMemcpyAsync(c->iface[0].p, &one, sizeof(double), cudaMemcpyHostToDevice, c->stream));
  int f = 0;
  for (int i = 0; i < tt->d; ++i) {
    const long long rl = tt->ranks[i], n = tt->modes[i], rr = tt->ranks[i + 1];
    const double* C = tt->cores[i].as<double>();
    double* T = c->iface_T.as<double>();
    gemm<false, false>(c, c->iface[f].as<double>(), rl, C, rl, T, rl, rl, n * rr, rl, 1.0, 0.0, &c->gemm_ws_side);
    gemm<true, false>(c, C, rl * n, T, rl * n, c->iface[f ^ 1].as<double>(), rr, rr, rr, rl * n, 1.0, 0.0,
                      &c->gemm_ws_side);
    f ^= 1;
  }
  return c->iface[f].as<double>();
}

// TT-ICE* per-observation statistics: norms (fused) + projection through the
// current cores (cached for the sweep) + decisions' partial sums
void star_stats(ttg_ctx* c, const ttg_tt* tt, const double* Y, int64_t b, double eps) {
  Norms nm{true, Y, prod(tt->modes), b};
  // a stale Phi^T Phi (the cores changed in the previous update) is computed
  // on the side stream, concurrently with the statistics pass over Y
  const double* M = nullptr;
  const bool stale = !(c->iface_gen == tt->gen && c->iface_ptr) || std::getenv("TTG_NO_IFACE_CACHE");
  if (stale && !c->profiling && !std::getenv("TTG_NO_SIDE")) {
    // workspaces grow on the main stream (stream-ordered pool), before the fork
    int64_t rmax = 1, nmax = 1;
    for (auto r : tt->ranks) rmax = std::max(rmax, r);
    for (auto n : tt->modes) nmax = std::max(nmax, n);
    c->iface[0].ensure(sizeof(double) * rmax * rmax);
    c->iface[1].ensure(sizeof(double) * rmax * rmax);
    c->Mtmp.ensure(sizeof(double) * rmax * nmax * rmax);
    c->iface_T.ensure(sizeof(double) * rmax * nmax * rmax);
    c->gemm_ws_side.ensure(sizeof(double) * 64 * rmax * rmax);
    CK(cudaEventRecord(c->ev_fork, c->stream));
    CK(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    std::swap(c->stream, c->side);
    try {
      M = interface_gram(c, tt);
    } catch (...) {
      std::swap(c->stream, c->side);
      throw;
    }
    std::swap(c->stream, c->side);
    CK(cudaEventRecord(c->ev_join, c->side));
  }
  const double* coeffs = project_chain(c, tt, Y, b, /*cache=*/true, nm);
  if (nm.pending) norms_finish(c, nm, 0, false);
  if (M) CK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
  else M = interface_gram(c, tt);
  const int r = (int)tt->ranks[tt->d];
  c->cn2.ensure(sizeof(double) * b);
  c->cmc.ensure(sizeof(double) * b);
  c->errs.ensure(sizeof(double) * b);
  c->rn2.ensure(sizeof(double) * b);
  c->stats.ensure(sizeof(ttg::StarStats));
  if (r > 64) {  // c^T M c through T = M C on the DMMA GEMM
    c->small[2].ensure(sizeof(double) * (size_t)r * b);
    double* T = c->small[2].as<double>();
    gemm<false, false>(c, M, r, coeffs, r, T, r, r, b, r, 1.0, 0.0);
    prof_begin(c, "k_coef_stats", 16.0 * r * b, 4.0 * r * b);
    launch_k(c, ttg::k_coef_dots, grid_for(32 * b, 256, 1024), 256, 0, coeffs, (const double*)T, r, (int)b,
             c->cn2.as<double>(), c->cmc.as<double>());
    post_launch(c);
  } else {
    prof_begin(c, "k_coef_stats", 8.0 * r * b, 2.0 * r * r * b);
    launch_k(c, ttg::k_coef_stats, grid_for(32 * b, 256, 1024), 256, 0, coeffs, r, (int)b, M, c->cn2.as<double>(),
                                                                     c->cmc.as<double>());
    post_launch(c);
  }
  prof_begin(c, "k_star_local", 32.0 * b, 10.0 * b);
  launch_k(c, ttg::k_star_local, 1, 256, 0, c->on2.as<double>(), c->cn2.as<double>(), c->cmc.as<double>(),
                                             (int)b, eps, c->errs.as<double>(), c->rn2.as<double>(),
                                             c->stats.as<ttg::StarStats>());
  post_launch(c);
  allreduce_sum(c, c->stats.as<double>(), 9);
}

void fill_report_numerics(ttg_report* rep, const SweepOut& so) {
  rep->accurate_modes = so.accurate_modes;
  rep->raw_fallbacks = so.raw_fallbacks;
  rep->gram_only_unstable = so.gram_only_unstable;
}

struct Timer {
  ttg_ctx* c;
  explicit Timer(ttg_ctx* cc) : c(cc) { CK(cudaEventRecord(c->ev0, c->stream)); }
  double stop() {
    CK(cudaEventRecord(c->ev1, c->stream));
    CK(cudaEventSynchronize(c->ev1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    return ms * 1e-3;
  }
};

// ---- entry points (internal, throwing) ----------------------------------------

void do_update(ttg_ctx* c, ttg_tt* tt, const double* y, int where, const int64_t* shape, int ndim,
               const double* deltas, int n_deltas, double eps_des, bool uniform, ttg_report* rep) {
  if (!c || !tt || !y || !rep) fail(TTG_E_ARGUMENT, "null argument");
  check_shape_args(shape, ndim);
  if (uniform && !(eps_des > 0.0)) fail(TTG_E_NUMERIC, "eps_des must be positive");  // tt_ice.cpp:133-135
  check_train_vs_y(tt, shape, ndim, true);
  const int d = tt->d;
  if (!uniform && n_deltas != d) fail(TTG_E_DIMENSION, "need one SVD tolerance per spatial dimension");
  if (!uniform)
    for (int i = 0; i < d; ++i)
      if (deltas[i] < 0.0) fail(TTG_E_NUMERIC, "svd_trunc: negative truncation threshold");
  const int64_t b = shape[d];
  const int64_t S = prod(tt->modes);
  Timer tm(c);
  const double* Y = stage_input(c, y, where, (size_t)(S * b));
  const int64_t bg = global_obs(c, b);
  std::memset(rep, 0, sizeof(*rep));
  rep->increment_index = (int64_t)tt->bounds.size();
  rep->obs_in_batch = bg;
  rep->obs_used = bg;
  rep->n_ranks = d + 2;
  fill_report_ranks(rep->ranks_before, tt);
  SweepOpts o;
  Norms nm{true, Y, S, b};
  if (uniform) {
    o.delta_src = c->scal.as<double>();
    o.delta_mult = eps_des / std::sqrt((double)d);  // tt_ice.cpp:137-138
    o.need_norms = true;
  } else {
    obs_norms(c, Y, S, (int)b);  // per-mode thresholds are absolute: |Y| only for the shortcut and report
    nm.pending = false;
    const double ysq0 = read_scalar(c, c->scal.as<double>());
    check_finite_norm(ysq0);
    o.deltas = deltas;
    o.y_norm = std::sqrt(ysq0);
  }
  SweepOut so = sweep(c, tt, Y, b, o, nm);
  if (nm.pending) norms_finish(c, nm, 0, false);
  const double ysq = read_scalar(c, c->scal.as<double>());
  check_finite_norm(ysq);
  const double y_norm = std::sqrt(ysq);
  rep->eps_target = uniform ? eps_des * y_norm / std::sqrt((double)d) : (d > 0 ? deltas[0] : 0.0);
  append_last_core(c, tt, so.coeffs, so.r_d, b);
  fill_report_ranks(rep->ranks_after, tt);
  rep->batch_rel_error_estimate = (y_norm == 0.0) ? 0.0 : std::sqrt(so.discarded_sq) / y_norm;
  rep->guard_reorthogonalised = *guards_slot(c);  // fetched by the sweep, valid after read_scalar's sync
  rep->modes_updated = so.modes_updated;
  fill_report_numerics(rep, so);
  rep->seconds = tm.stop();
}

void do_star_update(ttg_ctx* c, ttg_tt* tt, const double* y, int where, const int64_t* shape, int ndim,
                    double eps_des, const ttg_heuristics* cfgp, ttg_report* rep) {
  if (!c || !tt || !y || !rep) fail(TTG_E_ARGUMENT, "null argument");
  ttg_heuristics cfg;
  ttg_heuristics_default(&cfg);
  if (cfgp) cfg = *cfgp;
  check_shape_args(shape, ndim);
  if (!(eps_des > 0.0)) fail(TTG_E_NUMERIC, "eps_des must be positive");  // tt_ice_star.cpp:175-177
  if (cfg.occupancy_threshold <= 0.0 || cfg.occupancy_threshold > 1.0)
    fail(TTG_E_CONFIG, "occupancy threshold must lie in (0, 1]");       // :178-180
  // per_obs_stats -> tt_project validates state and shape (tensor_train.cpp:196-208)
  if (tt->ortho_count != tt->d) fail(TTG_E_STATE, "projection requires a fully orthonormal train");
  check_train_vs_y(tt, shape, ndim, false);
  const int d = tt->d;
  const int64_t b = shape[d];
  const int64_t S = prod(tt->modes);
  Timer tm(c);
  const double* Y = stage_input(c, y, where, (size_t)(S * b));
  const int64_t bg = global_obs(c, b);
  std::memset(rep, 0, sizeof(*rep));
  rep->increment_index = (int64_t)tt->bounds.size();
  rep->obs_in_batch = bg;
  rep->n_ranks = d + 2;
  fill_report_ranks(rep->ranks_before, tt);

  Trace tr;
  g_trace = tr.on ? &tr : nullptr;
  trace("star:start");
  star_stats(c, tt, Y, b, eps_des);  // norms fused into the stats projection
  trace("star:stats launched");
  c->d2h += sizeof(ttg::StarStats);
  CK(cudaMemcpyAsync(c->h_stats, c->stats.p, sizeof(ttg::StarStats), cudaMemcpyDeviceToHost, c->stream));
  const double ysq = read_scalar(c, c->scal.as<double>());
  trace("star:stats synced");
  check_finite_norm(ysq);
  const double y_norm = std::sqrt(ysq);
  const double* s = c->h_stats->sums;
  // skip statistic (tt_ice_star.cpp:46-65)
  double skip_stat;
  if (cfg.skip_statistic == TTG_SKIP_MEAN) skip_stat = (s[1] == 0.0) ? 0.0 : s[0] / s[1];
  else skip_stat = (s[3] == 0.0) ? 0.0 : std::sqrt(s[2] / s[3]);
  int64_t n_sel = 0, n_rej = 0;
  if (cfg.skip_enabled && skip_stat <= eps_des) {
    n_sel = 0;
  } else if (cfg.subselect_enabled) {
    n_sel = (int64_t)s[6];
    n_rej = (int64_t)s[7];
  } else {
    n_sel = bg;
    n_rej = 0;
  }
  rep->obs_used = n_sel;
  SweepOut so;
  const double* coeffs = c->scoeffs.as<double>();  // stats projection = projection through unchanged cores
  int r_d = (int)tt->ranks[d];
  if (n_sel > 0) {
    double eps_upd = eps_des;
    if (n_rej > 0) {
      if (cfg.use_approx_tolerance) {  // Eq. 3.20, tt_ice_star.cpp:160-169
        const double mean_rej = s[8] / (double)n_rej;
        eps_upd = (eps_des * (double)bg - mean_rej * (double)n_rej) / (double)n_sel;
      } else {  // Eq. 3.19, tt_ice_star.cpp:121-158
        const double selected_sq = s[5];
        if (selected_sq == 0.0) fail(TTG_E_NUMERIC, "selected observations carry no energy");
        const double budget = eps_des * y_norm;
        double radicand = (budget * budget - s[4]) / selected_sq;
        if (radicand < 0.0) {
          radicand = 0.0;
          rep->tolerance_clamped = 1;
        }
        eps_upd = std::sqrt(radicand);
      }
    }
    const double d_sq = cfg.subselect_enabled ? s[5] : s[3];
    const double delta = eps_upd / std::sqrt((double)d) * std::sqrt(d_sq);  // :235-236
    rep->eps_target = delta;
    c->sel.ensure((size_t)b);
    prof_begin(c, "k_star_mask", 9.0 * b, 0.0);
    launch_k(c, ttg::k_star_mask, grid_for(b, 256, 64), 256, 0, c->errs.as<double>(), (int)b, eps_des,
                                                                    cfg.subselect_enabled, c->sel.as<uint8_t>());
    post_launch(c);
    SweepOpts o;
    o.star = true;
    o.tau = cfg.occupancy_threshold;
    o.sel = c->sel.as<uint8_t>();
    o.n_sel_global = n_sel;
    o.delta_mult = delta;
    o.reuse_stats = true;
    Norms nm;  // norms already known
    // the sweep mutates ranks/cores in place; TT-ICE* keeps the old cores when
    // nothing grew (tt_ice_star.cpp:276-277), which in-place is the same bytes
    so = sweep(c, tt, Y, b, o, nm);
    coeffs = so.coeffs;
    r_d = so.r_d;
    rep->modes_updated = so.modes_updated;
    fill_report_numerics(rep, so);
  }
  trace("star:sweep done");
  append_last_core(c, tt, coeffs, r_d, b);
  trace("star:append last core");
  fill_report_ranks(rep->ranks_after, tt);
  // estimate: Pythagoras on the appended coefficients (tt_ice_star.cpp:297-300)
  const double* csrc = c->coll ? c->coeffs_all.as<double>() : coeffs;
  // |c|^2 and the guard count ride on the timer's synchronisation (one host sync)
  sumsq_device_async(c, csrc, (long long)r_d * bg);
  rep->seconds = tm.stop();
  const double kept_sq = c->h_scal[0];
  if (n_sel > 0) rep->guard_reorthogonalised = *guards_slot(c);
  const double lost_sq = std::max(ysq - kept_sq, 0.0);
  rep->batch_rel_error_estimate = (y_norm == 0.0) ? 0.0 : std::sqrt(lost_sq) / y_norm;
  trace("star:end");
  g_trace = nullptr;
}

ttg_tt* do_bootstrap(ttg_ctx* c, const double* y, int where, const int64_t* shape, int ndim, double eps,
                     ttg_report* rep) {
  if (!c || !y || !rep) fail(TTG_E_ARGUMENT, "null argument");
  check_shape_args(shape, ndim);
  if (eps < 0.0 || eps > 1.0) fail(TTG_E_NUMERIC, "tt_svd tolerance must lie in [0, 1]");  // tt_svd.cpp:10-12
  if (ndim < 2) fail(TTG_E_DIMENSION, "bootstrap needs spatial modes plus an observation mode");
  if (ndim - 1 > TTG_MAX_CORES - 1) fail(TTG_E_DIMENSION, "too many modes");
  const int d = ndim - 1;
  auto tt = new ttg_tt();
  try {
    tt->d = d;
    tt->modes.assign(shape, shape + d);
    tt->ranks.assign(d + 1, 1);
    tt->cores.resize(d);
    const int64_t b = shape[d];
    const int64_t S = prod(tt->modes);
    Timer tm(c);
    const double* Y = stage_input(c, y, where, (size_t)(S * b));
    const int64_t bg = global_obs(c, b);
    SweepOpts o;
    o.bootstrap = true;
    o.delta_src = c->scal.as<double>();
    o.delta_mult = eps / std::sqrt((double)(ndim - 1));  // tt_svd.cpp:30
    o.need_norms = true;
    c->scal.ensure(sizeof(double) * 16);
    o.delta_src = c->scal.as<double>();
    Norms nm{true, Y, S, b};
    SweepOut so = sweep(c, tt, Y, b, o, nm);
    if (nm.pending) norms_finish(c, nm, 0, false);
    const double ysq = read_scalar(c, c->scal.as<double>());
    check_finite_norm(ysq);
    const double y_norm = std::sqrt(ysq);
    append_last_core(c, tt, so.coeffs, so.r_d, b);
    tt->ortho_count = d;
    std::memset(rep, 0, sizeof(*rep));
    rep->increment_index = 0;
    rep->obs_in_batch = bg;
    rep->obs_used = bg;
    rep->n_ranks = d + 2;
    fill_report_ranks(rep->ranks_after, tt);
    for (int i = 0; i <= d + 1; ++i) rep->ranks_before[i] = 1;
    fill_report_numerics(rep, so);
    rep->eps_target = eps * y_norm / std::sqrt((double)(ndim - 1));
    const double* src = c->coll ? c->coeffs_all.as<double>() : so.coeffs;
    const double kept_sq = sumsq_device(c, src, (long long)so.r_d * bg);  // tt_norm (tensor_train.cpp:383-386)
    const double lost_sq = std::max(ysq - kept_sq, 0.0);
    rep->batch_rel_error_estimate = (y_norm == 0.0) ? 0.0 : std::sqrt(lost_sq) / y_norm;
    rep->seconds = tm.stop();
  } catch (...) {
    delete tt;
    throw;
  }
  return tt;
}

int guard(ttg_ctx* c, auto&& fn) {
  struct StreamScope {
    cudaStream_t prev;
    explicit StreamScope(ttg_ctx* cc) : prev(g_alloc_stream) {
      if (cc && cc->stream) g_alloc_stream = cc->stream;
    }
    ~StreamScope() { g_alloc_stream = prev; }
  } scope(c);
  struct PrefetchRelease {  // the consumed staging slot is free once the call's stream work is done
    ttg_ctx* c;
    ~PrefetchRelease() {
      if (c && c->pf_inuse >= 0) {
        cudaEventRecord(c->pf[c->pf_inuse].freed, c->stream);
        c->pf[c->pf_inuse].used = true;
        c->pf_inuse = -1;
      }
    }
  } release{c};
  try {
    fn();
    return TTG_OK;
  } catch (const TtgError& e) {
    if (c) c->err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    if (c) c->err = "host allocation failed";
    return TTG_E_RESOURCE;
  } catch (const std::exception& e) {
    if (c) c->err = e.what();
    return TTG_E_CUDA;
  }
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

void ttg_heuristics_default(ttg_heuristics* h) {
  if (!h) return;
  h->occupancy_threshold = 0.8;
  h->skip_enabled = 1;
  h->subselect_enabled = 1;
  h->skip_statistic = TTG_SKIP_MEAN;
  h->use_approx_tolerance = 0;
}

static int ctx_init(ttg_ctx* c, int device) {
  CK(cudaSetDevice(device));
  c->device = device;
  c->pdl = std::getenv("TTG_NO_PDL") == nullptr;
  CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  CK(cudaEventCreate(&c->ev0));
  CK(cudaEventCreate(&c->ev1));
  CK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
  for (auto& s : c->pf) {
    CK(cudaEventCreateWithFlags(&s.ready, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&s.freed, cudaEventDisableTiming));
  }
  CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  c->num_sms = prop.multiProcessorCount;
  {
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  }
  c->smem_optin = prop.sharedMemPerBlockOptin;
  // eager-load every kernel variant (CUDA lazy loading would otherwise stall
  // the first increment that needs a new shape class, mid-stream)
  {
    cudaFuncAttributes fa;
    const void* ks[] = {
        (const void*)ttg::k_gram_resid<1, 2, false, true>, (const void*)ttg::k_gram_resid<2, 4, false, true>,
        (const void*)ttg::k_gram_resid<3, 6, false, true>, (const void*)ttg::k_gram_resid<4, 8, false, true>,
        (const void*)ttg::k_gram_resid<4, 8, false, false>, (const void*)ttg::k_gram_resid<1, 2, true, true>,
        (const void*)ttg::k_gram_resid<2, 4, true, true>, (const void*)ttg::k_gram_resid<3, 6, true, true>,
        (const void*)ttg::k_gram_resid<4, 8, true, true>, (const void*)ttg::k_project<true, true>,
        (const void*)ttg::k_project<true, false>, (const void*)ttg::k_project<false, false>,
        (const void*)ttg::k_syev, (const void*)ttg::k_sytrd_grid, (const void*)ttg::k_syev_bt<4>, (const void*)ttg::k_syev_bt<8>, (const void*)ttg::k_syev_top<2>, (const void*)ttg::k_syev_top<4>, (const void*)ttg::k_syev_top<8>, (const void*)ttg::k_decide<2>, (const void*)ttg::k_decide<4>, (const void*)ttg::k_project_tail,
        (const void*)ttg::k_jacobi_eig, (const void*)ttg::k_append, (const void*)ttg::k_tsqr_local,
        (const void*)ttg::k_tsqr_combine, (const void*)ttg::k_make_frags, (const void*)ttg::k_sumsq_obs,
        (const void*)ttg::k_sumsq_finalize, (const void*)ttg::k_tiles_to_obs, (const void*)ttg::k_pad_core,
        (const void*)ttg::k_iface_all, (const void*)ttg::k_build_q, (const void*)ttg::k_syrk_ws16<1, 1>, (const void*)ttg::k_syrk_ws16<3, 1>,
        (const void*)ttg::k_syrk_ws16<6, 1>, (const void*)ttg::k_syrk_ws16<10, 1>, (const void*)ttg::k_syrk_ws16<5, 3>,
        (const void*)ttg::k_syrk_ws16<7, 3>, (const void*)ttg::k_syrk_ws16<14, 2>, (const void*)ttg::k_syrk_ws16<12, 3>, (const void*)ttg::k_coef_stats, (const void*)ttg::k_coef_dots,
        (const void*)ttg::k_star_local, (const void*)ttg::k_star_mask, (const void*)ttg::k_mask_cols,
        (const void*)ttg::k_merge_rows, (const void*)ttg::k_kron_eye, (const void*)ttg::k_dgemm<false, false, 64>,
        (const void*)ttg::k_dgemm<true, false, 64>, (const void*)ttg::k_dgemm<false, true, 64>,
        (const void*)ttg::k_dgemm<true, true, 64>, (const void*)ttg::k_dgemm<false, false, 128>,
        (const void*)ttg::k_dgemm<true, false, 128>, (const void*)ttg::k_dgemm<false, true, 128>,
        (const void*)ttg::k_dgemm<true, true, 128>, (const void*)ttg::k_dgemm_reduce, (const void*)ttg::k_transpose, (const void*)ttg::k_tall_u,
        (const void*)ttg::k_syrk<1>,
        (const void*)ttg::k_syrk<2>, (const void*)ttg::k_syrk<3>, (const void*)ttg::k_syrk<5>,
        (const void*)ttg::k_syrk<8>, (const void*)ttg::k_syrk2<1>, (const void*)ttg::k_syrk2<2>,
        (const void*)ttg::k_syrk2<3>, (const void*)ttg::k_gram_reduce_s1, (const void*)ttg::k_gram_reduce_s2, (const void*)ttg::k_make_frags16,
        (const void*)ttg::k_project_ws16<4, 1>, (const void*)ttg::k_project_ws16<4, 2>,
        (const void*)ttg::k_project_ws16<4, 3>, (const void*)ttg::k_project_ws16<4, 4>, (const void*)ttg::k_project_tma<true, 64>, (const void*)ttg::k_project_tma<false, 64>,
        (const void*)ttg::k_project_tma<true, 32>, (const void*)ttg::k_project_tma<false, 32>,
        (const void*)ttg::k_sum_vec, (const void*)ttg::k_make_tail, (const void*)ttg::k_syrk_kx<8>, (const void*)ttg::k_pcp, (const void*)ttg::k_pcp_l2};
    for (int nbk = 7; nbk <= kKpMaxNbk; ++nbk) CK(cudaFuncGetAttributes(&fa, kp_pick(nbk)));
    for (int nb = 2; nb <= 16; ++nb) {
      CK(cudaFuncGetAttributes(&fa, ws_pick(4, nb)));
      CK(cudaFuncGetAttributes(&fa, ws_pick(8, nb)));
    }
    for (int nb = 1; nb <= 4; ++nb)
      for (int t = 0; t <= kKcMaxTail; ++t) {
        CK(cudaFuncGetAttributes(&fa, kc_pick(4, nb, t)));
        CK(cudaFuncGetAttributes(&fa, kc_pick(8, nb, t)));
      }
    for (const void* k : ks) CK(cudaFuncGetAttributes(&fa, k));
  }
  CK(cudaMallocHost((void**)&c->h_eig, sizeof(ttg::EigResult)));
  CK(cudaMallocHost((void**)&c->h_eiglog, sizeof(ttg::EigResult) * (TTG_MAX_CORES + 1)));
  CK(cudaMallocHost((void**)&c->h_scal, sizeof(double) * 16));
  CK(cudaMallocHost((void**)&c->h_stats, sizeof(ttg::StarStats)));
  return 0;
}

int ttg_ctx_create(int device, ttg_ctx** out) {
  if (!out) return TTG_E_ARGUMENT;
  auto c = new ttg_ctx();
  int rc = guard(c, [&] { ctx_init(c, device); });
  if (rc != TTG_OK) {
    fprintf(stderr, "ttg_ctx_create: %s\n", c->err.c_str());
    ttg_ctx_destroy(c);
    *out = nullptr;
    return rc;
  }
  *out = c;
  return TTG_OK;
}

int ttg_nccl_unique_id(uint8_t out[128]) {
  if (!out) return TTG_E_ARGUMENT;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return TTG_E_NCCL;
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  std::memcpy(out, &id, 128);
  return TTG_OK;
}

int ttg_ctx_create_dist(int device, int rank, int world, const uint8_t nccl_id[128], ttg_ctx** out) {
  if (!out || !nccl_id || world < 1 || rank < 0 || rank >= world) return TTG_E_ARGUMENT;
  auto c = new ttg_ctx();
  int rc = guard(c, [&] {
    ctx_init(c, device);
    c->rank = rank;
    c->world = world;
    // NCCL kernels interleave in the stream.  PDL stays on: our kernels never
    // trigger early, so a kernel behind an NCCL kernel launches at its exit
    // and every kernel's griddepcontrol.wait (tests/test_pdl_static.py) orders
    // its reads after the collective's writes; TTG_NCCL_NO_PDL turns it off.
    c->pdl = c->pdl && std::getenv("TTG_NCCL_NO_PDL") == nullptr;
    c->coll = true;
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, 128);
    NK(ncclCommInitRank(&c->comm, world, id, rank));
  });
  if (rc != TTG_OK) {
    fprintf(stderr, "ttg_ctx_create_dist: %s\n", c->err.c_str());
    ttg_ctx_destroy(c);
    *out = nullptr;
    return rc;
  }
  *out = c;
  return TTG_OK;
}

int ttg_ctx_create_hostcoll(int device, int rank, int world, ttg_host_allreduce_fn allreduce,
                            ttg_host_allgather_fn allgather_fn, void* user, ttg_ctx** out) {
  if (!out || world < 1 || rank < 0 || rank >= world || (world > 1 && (!allreduce || !allgather_fn)))
    return TTG_E_ARGUMENT;
  auto c = new ttg_ctx();
  int rc = guard(c, [&] {
    ctx_init(c, device);
    c->rank = rank;
    c->world = world;
    c->host_ar = allreduce;
    c->host_ag = allgather_fn;
    c->host_user = user;
    c->coll = world > 1;
  });
  if (rc != TTG_OK) {
    fprintf(stderr, "ttg_ctx_create_hostcoll: %s\n", c->err.c_str());
    ttg_ctx_destroy(c);
    *out = nullptr;
    return rc;
  }
  *out = c;
  return TTG_OK;
}

void ttg_ctx_destroy(ttg_ctx* c) {
  if (!c) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->h_eig) cudaFreeHost(c->h_eig);
  if (c->h_eiglog) cudaFreeHost(c->h_eiglog);
  if (c->h_scal) cudaFreeHost(c->h_scal);
  if (c->h_stats) cudaFreeHost(c->h_stats);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->side) {
    cudaStreamSynchronize(c->side);
    cudaStreamDestroy(c->side);
  }
  if (c->copy) {
    cudaStreamSynchronize(c->copy);
    cudaStreamDestroy(c->copy);
  }
  for (auto& s : c->pf) {
    if (s.ready) cudaEventDestroy(s.ready);
    if (s.freed) cudaEventDestroy(s.freed);
  }
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->ev_in) cudaEventDestroy(c->ev_in);
  if (c->ev_out) cudaEventDestroy(c->ev_out);
  for (auto& p : c->pending) {
    cudaEventDestroy(p.e0);
    cudaEventDestroy(p.e1);
  }
  for (auto e : c->evpool) cudaEventDestroy(e);
  cudaStream_t s = c->stream;
  g_alloc_stream = s;
  delete c;  // frees workspaces (stream-ordered)
  g_alloc_stream = nullptr;
  if (s) {
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  }
}

// context-free entry points (TTB1 read/write) leave their message per thread
thread_local std::string g_noctx_err = "no error";
const char* ttg_last_error(const ttg_ctx* c) { return c ? c->err.c_str() : g_noctx_err.c_str(); }
int ttg_ctx_rank(const ttg_ctx* c) { return c ? c->rank : -1; }
int ttg_ctx_world(const ttg_ctx* c) { return c ? c->world : -1; }
void* ttg_ctx_stream(const ttg_ctx* c) { return c ? (void*)c->stream : nullptr; }
int64_t ttg_ctx_launch_count(const ttg_ctx* c) { return c ? c->launches : -1; }
int ttg_ctx_set_profiling(ttg_ctx* c, int on) {
  if (!c) return TTG_E_ARGUMENT;
  return guard(c, [&] {
    prof_flush(c);
    c->profiling = on != 0;
  });
}

void ttg_ctx_reset_stats(ttg_ctx* c) {
  if (!c) return;
  try {
    prof_flush(c);
  } catch (...) {
  }
  c->kstats.clear();
  c->h2d = c->d2h = 0;
}

int ttg_ctx_num_kernel_stats(ttg_ctx* c) {
  if (!c) return -1;
  int rc = guard(c, [&] { prof_flush(c); });
  return rc == TTG_OK ? (int)c->kstats.size() : -rc;
}

int ttg_ctx_kernel_stat(ttg_ctx* c, int idx, char* name, int name_len, int64_t* launches, double* ms,
                        double* bytes, double* flops) {
  if (!c) return TTG_E_ARGUMENT;
  return guard(c, [&] {
    prof_flush(c);
    if (idx < 0 || idx >= (int)c->kstats.size()) fail(TTG_E_INDEX, "kernel stat index out of range");
    const auto& st = c->kstats[idx];
    if (name && name_len > 0) {
      std::snprintf(name, (size_t)name_len, "%s", st.name.c_str());
    }
    if (launches) *launches = st.launches;
    if (ms) *ms = st.ms;
    if (bytes) *bytes = st.bytes;
    if (flops) *flops = st.flops;
  });
}

int ttg_ctx_reserve(ttg_ctx* c, int64_t bytes) {
  if (!c || bytes < 0) return TTG_E_ARGUMENT;
  return guard(c, [&] {
    // map `bytes` into the stream-ordered pool now (release threshold is
    // unlimited, so the pages stay cached for later workspace growth)
    void* p = nullptr;
    CK(cudaMallocAsync(&p, (size_t)bytes, c->stream));
    CK(cudaFreeAsync(p, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int ttg_ctx_io_bytes(const ttg_ctx* c, int64_t* h2d, int64_t* d2h) {
  if (!c) return TTG_E_ARGUMENT;
  if (h2d) *h2d = c->h2d;
  if (d2h) *d2h = c->d2h;
  return TTG_OK;
}

int ttg_ctx_spec_stats(const ttg_ctx* c, int64_t* sweeps, int64_t* redone) {
  if (!c) return TTG_E_ARGUMENT;
  if (sweeps) *sweeps = c->spec_sweeps;
  if (redone) *redone = c->spec_redone;
  return TTG_OK;
}

int ttg_prefetch(ttg_ctx* c, const double* y, int64_t n) {
  if (!c || !y || n < 0) return TTG_E_ARGUMENT;
  return guard(c, [&] {
    const int i = c->pf_next;
    c->pf_next ^= 1;
    auto& s = c->pf[i];
    // an older, never consumed copy of the same host buffer is stale now (the
    // caller may have refilled it): only the newest prefetch may be consumed
    auto& o = c->pf[i ^ 1];
    if (o.valid && o.src == y && o.n == n) o.valid = false;
    if (s.used) CK(cudaStreamWaitEvent(c->copy, s.freed, 0));  // an earlier update may still read this slot
    s.buf.ensure(sizeof(double) * (size_t)std::max<int64_t>(n, 1), false, c->copy);
    CK(cudaMemcpyAsync(s.buf.p, y, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice, c->copy));
    CK(cudaEventRecord(s.ready, c->copy));
    s.src = y;
    s.n = n;
    s.valid = true;
    c->h2d += (int64_t)(sizeof(double) * n);
  });
}

int ttg_ctx_synchronize(ttg_ctx* c) {
  return guard(c, [&] { CK(cudaStreamSynchronize(c->stream)); });
}

int ttg_ctx_wait_stream(ttg_ctx* c, void* stream) {
  if (!c) return TTG_E_ARGUMENT;
  return guard(c, [&] {
    CK(cudaEventRecord(c->ev_in, (cudaStream_t)stream));
    CK(cudaStreamWaitEvent(c->stream, c->ev_in, 0));
  });
}

int ttg_ctx_join_stream(ttg_ctx* c, void* stream) {
  if (!c) return TTG_E_ARGUMENT;
  return guard(c, [&] {
    CK(cudaEventRecord(c->ev_out, c->stream));
    CK(cudaStreamWaitEvent((cudaStream_t)stream, c->ev_out, 0));
  });
}

int ttg_tt_upload(ttg_ctx* c, int n_cores, const int64_t* r_left, const int64_t* n, const int64_t* r_right,
                  const double* const* cores, int64_t ortho_count, const int64_t* bounds, int64_t n_bounds,
                  ttg_tt** out) {
  if (!c || !out || !r_left || !n || !r_right || !cores) return TTG_E_ARGUMENT;
  ttg_tt* tt = new ttg_tt();
  int rc = guard(c, [&] {
    // TensorTrain ctor validation (tensor_train.cpp:60-93)
    if (n_cores < 2) fail(TTG_E_DIMENSION, "a streamed train needs spatial cores plus the observation core");
    if (n_cores > TTG_MAX_CORES) fail(TTG_E_DIMENSION, "too many cores");
    if (r_left[0] != 1 || r_right[n_cores - 1] != 1) fail(TTG_E_DIMENSION, "boundary ranks must be 1");
    for (int i = 0; i < n_cores; ++i)
      if (r_left[i] < 1 || n[i] < 1 || r_right[i] < 1) fail(TTG_E_DIMENSION, "core extents must be >= 1");
    for (int i = 0; i + 1 < n_cores; ++i)
      if (r_right[i] != r_left[i + 1]) fail(TTG_E_DIMENSION, "bond rank mismatch between cores");
    if (ortho_count < 0 || ortho_count > n_cores - 1) fail(TTG_E_STATE, "ortho_count outside [0, D-1]");
    const int d = n_cores - 1;
    tt->d = d;
    tt->modes.assign(n, n + d);
    tt->ranks.resize(d + 1);
    tt->ranks[0] = 1;
    for (int i = 0; i < d; ++i) tt->ranks[i + 1] = r_right[i];
    tt->cores.resize(d);
    for (int i = 0; i < d; ++i) {
      size_t cnt = (size_t)(r_left[i] * n[i] * r_right[i]);
      tt->cores[i].ensure(sizeof(double) * cnt);
      CK(cudaMemcpyAsync(tt->cores[i].p, cores[i], sizeof(double) * cnt, cudaMemcpyHostToDevice, c->stream));
    }
    int64_t nobs = n[d];
    tt->rc = std::max<int64_t>(r_left[d] + 8, 16);
    tt->oc = std::max<int64_t>(nobs * 2, 1024);
    tt->last.ensure(sizeof(double) * (size_t)tt->rc * tt->oc);
    CK(cudaMemsetAsync(tt->last.p, 0, sizeof(double) * (size_t)tt->rc * tt->oc, c->stream));
    CK(cudaMemcpy2DAsync(tt->last.p, sizeof(double) * tt->rc, cores[d], sizeof(double) * r_left[d],
                         sizeof(double) * r_left[d], nobs, cudaMemcpyHostToDevice, c->stream));
    tt->n_obs = nobs;
    tt->ortho_count = ortho_count;
    if (n_bounds > 0 && bounds) tt->bounds.assign(bounds, bounds + n_bounds);
    else tt->bounds.push_back(nobs);
    int64_t prev = 0;
    for (auto bnd : tt->bounds) {
      if (bnd < prev) fail(TTG_E_DIMENSION, "batch boundaries must be nondecreasing");
      prev = bnd;
    }
    if (tt->bounds.back() != nobs) fail(TTG_E_DIMENSION, "batch boundaries must end at the observation count");
    CK(cudaStreamSynchronize(c->stream));
  });
  if (rc != TTG_OK) {
    delete tt;
    *out = nullptr;
    return rc;
  }
  *out = tt;
  return TTG_OK;
}

void ttg_tt_destroy(ttg_tt* tt) { delete tt; }
int ttg_tt_num_cores(const ttg_tt* tt) { return tt ? tt->d + 1 : -1; }

int ttg_tt_shape(const ttg_tt* tt, int64_t* ranks, int64_t* modes, int64_t* ortho_count, int64_t* n_bounds) {
  if (!tt) return TTG_E_ARGUMENT;
  if (ranks) {
    for (int i = 0; i <= tt->d; ++i) ranks[i] = tt->ranks[i];
    ranks[tt->d + 1] = 1;
  }
  if (modes) {
    for (int i = 0; i < tt->d; ++i) modes[i] = tt->modes[i];
    modes[tt->d] = tt->n_obs;
  }
  if (ortho_count) *ortho_count = tt->ortho_count;
  if (n_bounds) *n_bounds = (int64_t)tt->bounds.size();
  return TTG_OK;
}

int ttg_tt_bounds(const ttg_tt* tt, int64_t* bounds) {
  if (!tt || !bounds) return TTG_E_ARGUMENT;
  for (size_t i = 0; i < tt->bounds.size(); ++i) bounds[i] = tt->bounds[i];
  return TTG_OK;
}

int ttg_tt_download_core(ttg_ctx* c, const ttg_tt* tt, int i, double* out) {
  if (!c || !tt || !out) return TTG_E_ARGUMENT;
  return guard(c, [&] {
    if (i < 0 || i > tt->d) fail(TTG_E_INDEX, "core index out of range");
    if (i < tt->d) {
      size_t cnt = (size_t)(tt->ranks[i] * tt->modes[i] * tt->ranks[i + 1]);
      CK(cudaMemcpyAsync(out, tt->cores[i].p, sizeof(double) * cnt, cudaMemcpyDeviceToHost, c->stream));
    } else if (tt->n_obs > 0) {
      int64_t r = tt->ranks[tt->d];
      CK(cudaMemcpy2DAsync(out, sizeof(double) * r, tt->last.p, sizeof(double) * tt->rc, sizeof(double) * r,
                           tt->n_obs, cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
  });
}

int ttg_bootstrap(ttg_ctx* c, const double* y, int where, const int64_t* shape, int ndim, double eps_des,
                  ttg_tt** out, ttg_report* report) {
  if (!c || !out) return TTG_E_ARGUMENT;
  *out = nullptr;
  return guard(c, [&] { *out = do_bootstrap(c, y, where, shape, ndim, eps_des, report); });
}

int ttg_tt_ice_update(ttg_ctx* c, ttg_tt* tt, const double* y, int where, const int64_t* shape, int ndim,
                      double eps_des, ttg_report* report) {
  if (!c) return TTG_E_ARGUMENT;
  return guard(c, [&] { do_update(c, tt, y, where, shape, ndim, nullptr, 0, eps_des, true, report); });
}

int ttg_tt_ice_update_with_tolerances(ttg_ctx* c, ttg_tt* tt, const double* y, int where, const int64_t* shape,
                                      int ndim, const double* deltas, int n_deltas, ttg_report* report) {
  if (!c || !deltas) return TTG_E_ARGUMENT;
  return guard(c, [&] { do_update(c, tt, y, where, shape, ndim, deltas, n_deltas, 0.0, false, report); });
}

int ttg_tt_ice_star_update(ttg_ctx* c, ttg_tt* tt, const double* y, int where, const int64_t* shape, int ndim,
                           double eps_des, const ttg_heuristics* cfg, ttg_report* report) {
  if (!c) return TTG_E_ARGUMENT;
  return guard(c, [&] { do_star_update(c, tt, y, where, shape, ndim, eps_des, cfg, report); });
}

int ttg_per_obs_errors(ttg_ctx* c, const ttg_tt* tt, const double* y, int where, const int64_t* shape, int ndim,
                       double* errs) {
  if (!c || !tt || !y || !errs) return TTG_E_ARGUMENT;
  return guard(c, [&] {
    check_shape_args(shape, ndim);
    if (tt->ortho_count != tt->d) fail(TTG_E_STATE, "projection requires a fully orthonormal train");
    check_train_vs_y(tt, shape, ndim, false);
    const int64_t b = shape[tt->d];
    const int64_t S = prod(tt->modes);
    const double* Y = stage_input(c, y, where, (size_t)(S * b));
    star_stats(c, tt, Y, b, 0.0);
    CK(cudaMemcpyAsync(errs, c->errs.p, sizeof(double) * b, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int ttg_project(ttg_ctx* c, const ttg_tt* tt, const double* y, int where, const int64_t* shape, int ndim,
                double* coeffs) {
  if (!c || !tt || !y || !coeffs) return TTG_E_ARGUMENT;
  return guard(c, [&] {
    check_shape_args(shape, ndim);
    if (tt->ortho_count != tt->d) fail(TTG_E_STATE, "projection requires a fully orthonormal train");
    check_train_vs_y(tt, shape, ndim, false);
    const int64_t b = shape[tt->d];
    const int64_t S = prod(tt->modes);
    const double* Y = stage_input(c, y, where, (size_t)(S * b));
    Norms nm;  // not needed
    const double* cf = project_chain(c, tt, Y, b, /*cache=*/false, nm);
    CK(cudaMemcpyAsync(coeffs, cf, sizeof(double) * b * tt->ranks[tt->d], cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int ttg_reconstruct(ttg_ctx* c, const ttg_tt* tt, int64_t b0, int64_t e0, double* out, int where) {
  if (!c || !tt || !out) return TTG_E_ARGUMENT;
  return guard(c, [&] {
    if (b0 < 0 || e0 > tt->n_obs || b0 > e0) fail(TTG_E_INDEX, "observation range out of bounds");
    if (where != TTG_HOST && where != TTG_DEVICE) fail(TTG_E_ARGUMENT, "bad where");
    const int d = tt->d;
    const int64_t m = e0 - b0;
    const int64_t S = prod(tt->modes);
    if (m == 0) return;
    // spatial chain Phi (S x r_d), tensor_train.cpp:152-166
    int64_t rows = tt->modes[0];
    int64_t r = tt->ranks[1];
    c->cur[0].ensure(sizeof(double) * (size_t)(rows * r));
    CK(cudaMemcpyAsync(c->cur[0].p, tt->cores[0].p, sizeof(double) * rows * r, cudaMemcpyDeviceToDevice,
                       c->stream));
    int f = 0;
    for (int i = 1; i < d; ++i) {
      int64_t n_i = tt->modes[i], rr = tt->ranks[i + 1];
      c->cur[f ^ 1].ensure(sizeof(double) * (size_t)(rows * n_i * rr));
      gemm<false, false>(c, c->cur[f].as<double>(), rows, tt->cores[i].as<double>(), r, c->cur[f ^ 1].as<double>(),
                         rows, rows, n_i * rr, r, 1.0, 0.0);
      rows *= n_i;
      r = rr;
      f ^= 1;
    }
    double* dst;
    if (where == TTG_DEVICE) dst = out;
    else {
      c->cur[f ^ 1].ensure(sizeof(double) * (size_t)(S * m));
      dst = c->cur[f ^ 1].as<double>();
    }
    gemm<false, false>(c, c->cur[f].as<double>(), S, tt->last.as<double>() + tt->rc * b0, tt->rc, dst, S, S, m, r,
                       1.0, 0.0);
    if (where == TTG_HOST)
      CK(cudaMemcpyAsync(out, dst, sizeof(double) * S * m, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

}  // extern "C"

#include "ttg_io_abi.inc"
