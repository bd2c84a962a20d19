// glsgpu.cu -- host runtime + C-ABI of the B200-native SUR PCG-Aug solver (include/glsgpu.h).
//
// One glsgpu_sur handle = one SUR operator resident on one device: X, Q (the per-block thin QR
// factors, TSQR-built on the device), R, Y, Omega and the solver state.  The PCG-Aug iteration
// (proj/src/pcg.cpp:134-211) runs entirely on the device: three streaming passes per iteration
// (A: u update + Kronecker Sigma u + d; B: w/sw/r updates + Q'r; C: Pi r + c) with the scalar
// control in single-CTA kernels between them, captured into CUDA graphs of `graph_chunk`
// iterations; the host only checks the device's `active` flag between graph launches.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/glsgpu.h"
#include "kernels.cuh"
#include "ne.cuh"
#include "gemm.cuh"
#include "cqr.cuh"

using namespace glsgpu;

namespace {

thread_local std::string g_err = "";

struct GErr {
  int code;
  std::string msg;
  int block;
};

[[noreturn]] void fail(int code, const std::string& msg, int block = -1) { throw GErr{code, msg, block}; }

void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  cudaGetLastError();
  if (e == cudaErrorMemoryAllocation) fail(GLSGPU_ERR_OUT_OF_MEMORY, std::string(what) + ": out of device memory");
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
    fail(GLSGPU_ERR_NO_DEVICE, std::string(what) + ": " + cudaGetErrorString(e));
  fail(GLSGPU_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)
#define CKL(name) cuda_check(cudaGetLastError(), name)

int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

template <typename T>
T* dalloc(size_t count) {
  void* p = nullptr;
  CK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
  return static_cast<T*>(p);
}

constexpr int64_t QR_SMEM_BYTES = 200 * 1024;

// NCCL, resolved at run time: single-device use never needs it; row-sharded handles all-gather the
// per-rank partial sums over NVLink (dlopen of the libnccl.so.2 torch or the system already provides).
struct Nccl {
  void* so = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  static bool tried = false;
  if (!tried) {
    tried = true;
    n.so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!n.so) n.so = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (n.so) {
      n.GetUniqueId = (decltype(n.GetUniqueId))dlsym(n.so, "ncclGetUniqueId");
      n.CommInitRank = (decltype(n.CommInitRank))dlsym(n.so, "ncclCommInitRank");
      n.AllGather = (decltype(n.AllGather))dlsym(n.so, "ncclAllGather");
      n.CommDestroy = (decltype(n.CommDestroy))dlsym(n.so, "ncclCommDestroy");
      n.GetErrorString = (decltype(n.GetErrorString))dlsym(n.so, "ncclGetErrorString");
    }
  }
  if (!n.GetUniqueId || !n.CommInitRank || !n.AllGather || !n.CommDestroy)
    fail(GLSGPU_ERR_NCCL, "glsgpu: libnccl.so.2 not loadable (needed for row-sharded handles)");
  return n;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  const char* s = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
  fail(GLSGPU_ERR_NCCL, std::string(what) + ": " + s);
}

// cuSOLVER, resolved at run time like NCCL: only the sur_reduce pre-pass uses it, for the dense symmetric
// eigensolver of the n x n Gram (syevd; plus geqrf / orgqr for a basis wider than the TSQR kernels' 512 columns).
// The Gram, the basis and the rotations are this library's own DMMA GEMM (gemm.cuh), the basis QR its own TSQR.
struct Dla {
  void* sol = nullptr;
  decltype(&cusolverDnCreate) SolCreate = nullptr;
  decltype(&cusolverDnDestroy) SolDestroy = nullptr;
  decltype(&cusolverDnSetStream) SolSetStream = nullptr;
  decltype(&cusolverDnDsyevd_bufferSize) SyevdBuf = nullptr;
  decltype(&cusolverDnDsyevd) Syevd = nullptr;
  decltype(&cusolverDnDgeqrf_bufferSize) GeqrfBuf = nullptr;
  decltype(&cusolverDnDgeqrf) Geqrf = nullptr;
  decltype(&cusolverDnDorgqr_bufferSize) OrgqrBuf = nullptr;
  decltype(&cusolverDnDorgqr) Orgqr = nullptr;
};

Dla& dla() {
  static Dla d;
  static bool tried = false;
  if (!tried) {
    tried = true;
    d.sol = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_GLOBAL);
    if (!d.sol) d.sol = dlopen("libcusolver.so", RTLD_NOW | RTLD_GLOBAL);
    if (d.sol) {
      d.SolCreate = (decltype(d.SolCreate))dlsym(d.sol, "cusolverDnCreate");
      d.SolDestroy = (decltype(d.SolDestroy))dlsym(d.sol, "cusolverDnDestroy");
      d.SolSetStream = (decltype(d.SolSetStream))dlsym(d.sol, "cusolverDnSetStream");
      d.SyevdBuf = (decltype(d.SyevdBuf))dlsym(d.sol, "cusolverDnDsyevd_bufferSize");
      d.Syevd = (decltype(d.Syevd))dlsym(d.sol, "cusolverDnDsyevd");
      d.GeqrfBuf = (decltype(d.GeqrfBuf))dlsym(d.sol, "cusolverDnDgeqrf_bufferSize");
      d.Geqrf = (decltype(d.Geqrf))dlsym(d.sol, "cusolverDnDgeqrf");
      d.OrgqrBuf = (decltype(d.OrgqrBuf))dlsym(d.sol, "cusolverDnDorgqr_bufferSize");
      d.Orgqr = (decltype(d.Orgqr))dlsym(d.sol, "cusolverDnDorgqr");
    }
  }
  if (!d.SolCreate || !d.Syevd || !d.Geqrf || !d.Orgqr)
    fail(GLSGPU_ERR_UNSUPPORTED, "glsgpu: libcusolver not loadable (the symmetric eigensolver of glsgpu_sur_reduce)");
  return d;
}

void blas_check(int st, const char* what) {
  if (st != 0) fail(GLSGPU_ERR_CUDA, std::string(what) + ": status " + std::to_string(st));
}

}  // namespace

// In-process rank group (TEST-ONLY exchange, include/glsgpu.h glsgpu_local_group_create): P row-shard handles in
// ONE process on ONE device, each driven by its own host thread, exchange their all-gathers through device-to-device
// copies ordered by CUDA events and host barriers.  No kernel ever waits on another rank (the stream dependencies
// are resolved by the GPU front end), so the ranks cannot deadlock on one device; what runs is the library's real
// sharded decomposition -- cross-rank TSQR level (k_stack_r), rank-order sums (k_sum_ranks, k_reduce3) -- with the
// NCCL call replaced by these copies.  Graph capture is off for group handles (the copies cross streams).
struct glsgpu_local_group {
  int n = 0;
  int dev = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool aborted = false;
  std::vector<cudaEvent_t> ev_ready, ev_done;
  std::vector<const double*> send;
};

struct glsgpu_sur {
  int dev = 0;
  cudaStream_t s = nullptr;
  int G = 0;
  int64_t M = 0, ldm = 0, n = 0, CH = 0;
  int nch = 0, nmax = 0;
  std::vector<int> nb;
  std::vector<int64_t> p0, r0;
  std::vector<double> wts, wtc;
  int* d_nb = nullptr;
  int64_t *d_p0 = nullptr, *d_r0 = nullptr;
  double *d_wts = nullptr, *d_wtc = nullptr;
  // MVRGLM embedding (glsgpu_mvrglm_create): block b = [Z0 (M0 rows); C_b (k_b selector rows); 0], M = M0 + max k_b.
  // For SUR: msig = ldm (every row under Sigma), m_ref = M_global G, wtc = wts.
  bool mv = false;
  int64_t msig = 0;                 // rows of every block under Sigma
  int64_t m_ref = 0;                // rows of the reference's embedded GLM (host m-vectors)
  int64_t M0 = 0;                   // MVRGLM observation rows per equation
  std::vector<int64_t> kb, kofs;    // MVRGLM constraint rows of block b and their offset in the reference order
  std::vector<int64_t> rows_b;      // rows of block b in the reference's operator (cost model)
  double* Xqr = nullptr;            // pre-scaled QR source D^-1/2 X (two weights per block); null: X * w_b
  int rank_msg = 0;                 // 1: plain qr_thin (mv_reduce) wording of RankDeficient
  double* omegaInvT = nullptr;      // (unused since the device PCG-NE applies chol_solve; kept null)
  double *neLr = nullptr, *neLc = nullptr;  // PCG-NE: L = cholesky(Omega), row-major and column-major
  double* nebuf = nullptr;          // PCG-NE n-vectors: x, f, p, gp, x_best, v, h
  cudaGraphExec_t ne_graph = nullptr;
  int ne_chunk = 0;
  TraceRowD* ne_rows = nullptr;
  double* d_ones = nullptr;         // PCG-NE: unit row weights for the X' pass
  const double* X = nullptr;
  int64_t ldx = 0;
  double* X_own = nullptr;
  const double* Y = nullptr;
  int64_t ldy = 0;
  double* Y_own = nullptr;
  double *Q = nullptr, *R = nullptr, *omegaT = nullptr;
  std::vector<double> omega_h;
  // TSQR plan
  struct Level {
    int64_t first, count;  // generic item range (k_qr_factor / k_qr_formq)
    int smem_bytes;
    int64_t max_rows;
    bool any_global;
    int64_t ffirst = 0, fcount = 0;  // register-resident item range (n <= 32, rows <= 256)
    std::vector<int64_t> fblock;     // [G + 1]: fast items of block b are [ffirst + fblock[b], ffirst + fblock[b + 1])
  };
  std::vector<Level> qr_levels;
  QrItem* d_items = nullptr;
  double* qr_store = nullptr;
  double* qr_tau = nullptr;
  double* qr_scratch = nullptr;
  int64_t qr_slot = 0;
  int* d_rank_flags = nullptr;
  // width classes for the column passes
  int* d_blk_narrow = nullptr;
  int* d_blk_wide = nullptr;
  int n_narrow = 0, n_wide = 0;
  // solver buffers
  bool solver_ready = false;
  // the ten M x G iteration vectors live in one slab (column blocks of G columns, ld = ldm) so that one
  // 2-D tensor map reaches all of them: w[0..2], sw[0..2], r, u, su, pr (MV_* column-block indices)
  double* mvec = nullptr;
  CUtensorMap vmap;
  bool vmap_ok = false;
  CUtensorMap vmap64;               // 64-row boxes of the same slab (k_kron_mma)
  bool vmap64_ok = false;
  double *wb[3] = {nullptr, nullptr, nullptr}, *swb[3] = {nullptr, nullptr, nullptr};
  double *r = nullptr, *u = nullptr, *su = nullptr, *pr = nullptr;
  double *t = nullptr, *vs = nullptr, *est = nullptr, *t2 = nullptr, *xtw = nullptr, *zvec = nullptr,
         *beta_d = nullptr;
  double *tpart = nullptr, *rpart = nullptr, *partA = nullptr, *partC = nullptr, *scal = nullptr;
  int* d_stop = nullptr;
  SolveState* st = nullptr;
  SolveState* st_host = nullptr;  // pinned
  TraceRowD* rows_d = nullptr;
  int64_t rows_cap_d = 0;
  double frob_x = -1.0;
  glsgpu_counters_t counters{};
  uint64_t pi_cost = 0, xstar_t_cost = 0, xstar_cost = 0;
  std::vector<glsgpu_kernel_stat> kstats;
  // graphs
  cudaGraphExec_t graph = nullptr;
  int graph_chunk = 0, graph_xmode = -1, graph_diag = -2, graph_timing = -1, graph_fma = -1;
  int kron_fma = 0;  // glsgpu_pcg_config::kron_fma of the current solve
  int sw_direct = 0; // sw_mode 1 in effect for the current solve (k_kron_mma path)
  int graph_sw = -1;
  TraceRowD* graph_rows = nullptr;  // the trace buffer the captured k_scalar_c / k_diag_finalize write
  // staged upload (glsgpu_sur_stage / glsgpu_sur_update_staged): the next model's X goes into X_own on the
  // copy stream `cs` once the current factorisation has consumed it (ev_qr), Y into Y_next
  cudaStream_t cs = nullptr;
  cudaEvent_t ev_qr = nullptr, ev_stage = nullptr;
  bool staged = false;      // a staged upload awaits glsgpu_sur_update_staged
  bool x_released = false;  // X_own holds (or is receiving) the NEXT model's X: nothing may read it now
  double* Y_next = nullptr;
  double* t3 = nullptr;     // Q-side diagnostics: s = R est, then Q' w
  // diag_every = 1 folded into passes B / C (SMODE_BD / SMODE_CD): the second and third column-partial sets
  double *tpart2 = nullptr, *tpart3 = nullptr;
  int fold = 0, graph_fold = -1;
  bool factors_ok = false;          // false after a rank-deficient update / refactor until a good one
  int fused = 0;     // fused_c in effect: Sigma pr in pass C (k_pass_c_mma), element-wise pass A (k_pass_a_ew)
  int graph_fused = -1;
  double* spr = nullptr;            // Sigma pr (slab column block MV_SPR)
  CUtensorMap qmap;                 // tile-contiguous Q as [256 rows] x [columns], 64 x 32 boxes (k_pass_c_mma)
  bool qmap_ok = false;
  std::vector<cudaEvent_t> tev;  // timing events captured into the graph
  int64_t graph_kernels = 0;     // kernel nodes in the instantiated graph
  int64_t launches = 0;          // kernels launched by this handle (graph nodes counted per launch)
  bool capturing = false;
  // row sharding: this rank owns rows [row0, row0 + M) of M_global; Omega, R, n-vectors replicated
  int rank = 0, nranks = 1;
  bool coll = false;  // collective path (NCCL all-gathers, cross-rank TSQR level); also nranks == 1 + id
  bool use_stream = false;  // TMA-staged passes (n_i <= 128, 16-byte aligned X columns, ldx >= ldm)
  bool all_stream = false;  // use_stream on EVERY rank (a pass that changes the collective sequence needs it)
  bool qtiled = false;      // Q tile-contiguous: block b, rows [256 k, 256 k + 256) contiguous (n_i <= 32)
  bool no_qtile = false;    // keep Q column-major (ld ldm): a QR-only handle whose Q is read out as a matrix
  // wide blocks (some n_i > 32, all <= 128): the QR writes column-major Q; the streaming passes read a tiled copy
  // with 64-row tiles (one contiguous bulk copy per tile instead of n_i strided 512-byte segments)
  double* qt = nullptr;
  int64_t* d_qtoff = nullptr;
  int qt_rows = 0;          // rows per tile of the copy: the tile rows the streaming passes pick (<= 256)
  std::vector<int64_t> qoff;  // offset of Q_b
  int64_t* d_qoff = nullptr;
  int64_t qsize = 0;
  int64_t M_global = 0;
  ncclComm_t comm = nullptr;
  glsgpu_local_group* grp = nullptr;  // test-only in-process exchange instead of NCCL
  double *loc3 = nullptr, *all3 = nullptr, *t_loc = nullptr, *t_all = nullptr;
  double *rloc = nullptr, *rall = nullptr, *rstack = nullptr, *gtau = nullptr;  // TSQR across ranks
  int64_t* d_stack_off = nullptr;
  std::vector<QrItem> gitems;  // the cross-rank level (one item per block)
  QrItem* d_gitems = nullptr;
  int gsmem = 0;
  int64_t gmax_rows = 0;
  // CholeskyQR2 setup (cqr.cuh): the default factorisation of SUR handles on the TMA passes; TSQR is the fallback
  bool cq = false;
  int cq_nbp = 0, cq_tr = 0;
  CqItem* d_cq_items = nullptr;
  std::vector<int64_t> cq_first;      // [G + 1] first item of block b
  int64_t* d_cq_first = nullptr;
  int* d_cq_nsrc = nullptr;           // [G] items of block b
  int64_t* d_cq_xoff = nullptr;       // [G] p0[b] ldx
  double *cq_gpart = nullptr, *cq_r1 = nullptr, *cq_rinv = nullptr;
  int* d_cq_flags = nullptr;
  int64_t* d_cq_bidx = nullptr;       // sharded: source index b and count P of the all-gathered Grams
  int* d_cq_np = nullptr;
  double *cq_gloc = nullptr, *cq_gall = nullptr;
  int cq_fallbacks = 0;               // factorisations that fell back to the Householder TSQR
  bool cq_last = false;               // the current factors came from CholeskyQR2
};

namespace {

Geo geo_of(const glsgpu_sur* h) {
  Geo g;
  g.G = h->G;
  g.nch = h->nch;
  g.M = h->M;
  g.ldm = h->ldm;
  g.n = h->n;
  g.CH = h->CH;
  g.nb = h->d_nb;
  g.p0 = h->d_p0;
  g.r0 = h->d_r0;
  g.wts = h->d_wts;
  g.wtc = h->d_wtc;
  g.msig = h->msig;
  return g;
}

int kron_cpl(int G) {
  if (G <= 32) return 1;
  if (G <= 64) return 2;
  if (G <= 128) return 4;
  if (G <= 256) return 8;
  return 16;
}

WBuf wbuf_of(const glsgpu_sur* h) {
  WBuf b;
  for (int i = 0; i < 3; ++i) {
    b.w[i] = h->wb[i];
    b.sw[i] = h->swb[i];
  }
  return b;
}

// out = (Omega (x) I) x with the CTA partials; in_mode per k_kron.
void launch_kron(glsgpu_sur* h, const double* src, const double* prv, const double* div, double* u_io, double* out,
                 double* partials, int in_mode, const SolveState* st, int* grid_out) {
  const int cpl = kron_cpl(h->G);
  const int rw = cpl >= 16 ? 2 : 4;
  const int tr = 8 * rw;
  const int64_t ntiles = h->ldm / tr;
  const int grid = (int)std::min<int64_t>(ntiles, GRID_CAP);
  // G <= 128 (cpl <= 4): Omega behind the tile in shared memory
  const size_t smem = ((size_t)h->G * tr + (cpl <= 4 ? (size_t)h->G * h->G : 0)) * sizeof(double);
  if (grid_out) *grid_out = grid;
  {  // the dynamic shared memory bound of every k_kron instance (once; G <= 128 also stages Omega)
    static bool attrs = false;
    if (!attrs) {
      CK(cudaFuncSetAttribute(k_kron<1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (32 * 32 + 32 * 32) * 8));
      CK(cudaFuncSetAttribute(k_kron<2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (64 * 32 + 64 * 64) * 8));
      CK(cudaFuncSetAttribute(k_kron<4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (128 * 32 + 128 * 128) * 8));
      CK(cudaFuncSetAttribute(k_kron<8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * 32 * 8));
      CK(cudaFuncSetAttribute(k_kron<16, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 512 * 16 * 8));
      attrs = true;
    }
  }
#define KRON_CASE(C, RW)                                                                                       \
  k_kron<C, RW><<<grid, NT, smem, h->s>>>(h->G, h->ldm, ntiles, h->omegaT, src, prv, div, u_io, out, partials, \
                                          in_mode, st, wbuf_of(h), h->msig)
  switch (cpl) {
    case 1: KRON_CASE(1, 4); break;
    case 2: KRON_CASE(2, 4); break;
    case 4: KRON_CASE(4, 4); break;
    case 8: KRON_CASE(8, 4); break;
    default: KRON_CASE(16, 2); break;
  }
#undef KRON_CASE
  CKL("k_kron");
  if (!h->capturing) h->launches++;
  if (!h->capturing) h->launches++;
}

// the warp-specialised FP64 kernel serves the compute-bound shapes; the generic k_kron the rest
bool kron_gemm_ok(const glsgpu_sur* h) { return h->G > 128 && h->G <= 256 && h->G % 8 == 0 && h->vmap_ok; }

// the DMMA kernel serves the fused-multiply-add mode (bitwise the same FMA chain as k_kron_ws<true>)
bool kron_mma_ok(const glsgpu_sur* h) {
  static const bool off = std::getenv("GLSGPU_NO_DMMA") != nullptr;
  return !off && kron_gemm_ok(h) && h->kron_fma && h->vmap64_ok;
}

// GLSGPU_KRON_V1=1: the first tensor-core pass A (element warps feed the math warps through a U ring)
bool kron_mma_v1() {
  static const bool v = std::getenv("GLSGPU_KRON_V1") != nullptr;
  return v;
}
// GLSGPU_KRON_W16=1: sixteen math warps of 16 columns (four per scheduler) instead of eight of 32
bool kron_mma_w16() {
  static const bool v = std::getenv("GLSGPU_KRON_W16") != nullptr;
  return v;
}
// ring stages of k_kron_mma2 for nv vectors per stage: what fits beside its static shared memory
int km2_stages(int nv) {
  return (int)std::min<size_t>(KM2_MAXS, (size_t)(227 * 1024 - 1024) / km2_stage_bytes(nv));
}

constexpr int EW_GRID = 148 * 8;  // k_pass_a_ew: grid-stride element-wise pass

int kron_grid(const glsgpu_sur* h) {
  if (h->fused) return EW_GRID;
  if (kron_mma_ok(h)) return (int)std::min<int64_t>((h->ldm + KM_BM - 1) / KM_BM, 148);
  if (kron_gemm_ok(h)) return (int)std::min<int64_t>(h->ldm / KG_BM, 148);
  const int cpl = kron_cpl(h->G);
  const int tr = 8 * (cpl >= 16 ? 2 : 4);
  return (int)std::min<int64_t>(h->ldm / tr, GRID_CAP);
}

// pass A: u = pr + mu u, the deferred w / sw update, su = Sigma u with the (d, u.u) partials
void launch_pass_a(glsgpu_sur* h) {
  if (h->fused) {
    k_pass_a_ew<<<EW_GRID, NT, 0, h->s>>>(h->ldm * h->G, h->u, h->su, h->pr, h->spr, wbuf_of(h), h->partA, h->st);
    if (!h->capturing) h->launches++;
    CKL("k_pass_a_ew");
    return;
  }
  if (!kron_gemm_ok(h)) {
    launch_kron(h, nullptr, h->pr, nullptr, h->u, h->su, h->partA, 2, h->st, nullptr);
    return;
  }
  const int grid = kron_grid(h);
  if (kron_mma_ok(h) && !kron_mma_v1()) {
    const int nv = h->sw_direct ? 3 : 5, ns = km2_stages(nv);
    if (kron_mma_w16())
      k_kron_mma2<false, 16><<<grid, (16 + 1 + KM_EW) * 32, ns * km2_stage_bytes(nv), h->s>>>(
          h->mvec, h->G, h->ldm, (h->ldm + KM_BM - 1) / KM_BM, h->omegaT, h->u, h->su, h->partA, h->st, wbuf_of(h),
          h->msig, -1, ns, nv);
    else
      k_kron_mma2<false, 8><<<grid, KM_NT, ns * km2_stage_bytes(nv), h->s>>>(
          h->mvec, h->G, h->ldm, (h->ldm + KM_BM - 1) / KM_BM, h->omegaT, h->u, h->su, h->partA, h->st, wbuf_of(h),
          h->msig, -1, ns, nv);
    if (!h->capturing) h->launches++;
    CKL("k_kron_mma2");
    return;
  }
  if (kron_mma_ok(h)) {
    k_kron_mma<false><<<grid, KM_NT, km_smem_bytes(), h->s>>>(h->vmap64, h->G, h->ldm, (h->ldm + KM_BM - 1) / KM_BM,
                                                             h->omegaT, h->u, h->su, h->partA, h->st, wbuf_of(h),
                                                             h->msig, -1);
    if (!h->capturing) h->launches++;
    CKL("k_kron_mma");
    return;
  }
  if (h->kron_fma)
    k_kron_ws<true><<<grid, KW_NT, kw_smem_bytes(), h->s>>>(h->vmap, h->G, h->ldm, h->ldm / KG_BM, h->omegaT, h->u,
                                                            h->su, h->partA, h->st, wbuf_of(h), h->msig);
  else
    k_kron_ws<false><<<grid, KW_NT, kw_smem_bytes(), h->s>>>(h->vmap, h->G, h->ldm, h->ldm / KG_BM, h->omegaT, h->u,
                                                             h->su, h->partA, h->st, wbuf_of(h), h->msig);
  if (!h->capturing) h->launches++;
  CKL("k_kron_ws");
}

// Sigma x on the tensor-core kernel for a vector of the slab (column block `blk`, e.g. MV_W + k for w[k]), or
// (blk == -2) Sigma w_cur into sw_cur gated on the diagnostics row; false when that kernel does not serve
bool kron_mma_apply(glsgpu_sur* h, int blk, double* out) {
  // fused multiply-adds: only where the solve runs kron_fma (exact mode keeps the reference's mul / add sums)
  if (!(kron_gemm_ok(h) && h->vmap64_ok && h->kron_fma) || std::getenv("GLSGPU_NO_DMMA")) return false;
  const int grid = (int)std::min<int64_t>((h->ldm + KM_BM - 1) / KM_BM, 148);
  if (!kron_mma_v1()) {
    const int nv = 1, ns = km2_stages(nv);
    if (kron_mma_w16())
      k_kron_mma2<true, 16><<<grid, (16 + 1 + KM_EW) * 32, ns * km2_stage_bytes(nv), h->s>>>(
          h->mvec, h->G, h->ldm, (h->ldm + KM_BM - 1) / KM_BM, h->omegaT, h->u, out, nullptr, h->st, wbuf_of(h),
          h->msig, blk, ns, nv);
    else
      k_kron_mma2<true, 8><<<grid, KM_NT, ns * km2_stage_bytes(nv), h->s>>>(
          h->mvec, h->G, h->ldm, (h->ldm + KM_BM - 1) / KM_BM, h->omegaT, h->u, out, nullptr, h->st, wbuf_of(h),
          h->msig, blk, ns, nv);
    if (!h->capturing) h->launches++;
    CKL("k_kron_mma2 apply");
    return true;
  }
  k_kron_mma<true><<<grid, KM_NT, km_smem_bytes(), h->s>>>(h->vmap64, h->G, h->ldm, (h->ldm + KM_BM - 1) / KM_BM,
                                                          h->omegaT, h->u, out, nullptr, h->st, wbuf_of(h), h->msig, blk);
  if (!h->capturing) h->launches++;
  CKL("k_kron_mma apply");
  return true;
}

int rowpass_grid(const glsgpu_sur* h) { return (int)std::min<int64_t>((int64_t)h->G * h->nch, GRID_CAP); }

// gate: 0 none, 1 st->active, 2 st->diag_now
template <int MODE>
void launch_colpass(glsgpu_sur* h, ColArgs a, const SolveState* st) {
  Geo g = geo_of(h);
  if (h->n_narrow) {
    a.blocks = h->d_blk_narrow;
    k_colpass<MODE, true><<<h->n_narrow * h->nch, NT, 0, h->s>>>(g, a, st);
    if (!h->capturing) h->launches++;
    CKL("k_colpass fused");
  }
  if (h->n_wide) {
    a.blocks = h->d_blk_wide;
    k_colpass<MODE, false><<<h->n_wide * h->nch, NT, (size_t)h->CH * sizeof(double), h->s>>>(g, a, st);
    if (!h->capturing) h->launches++;
    CKL("k_colpass panels");
  }
}

void launch_reduce_t(glsgpu_sur* h, double* out, const SolveState* st, int gate, const double* tp = nullptr) {
  const int per = NT / 32;
  const int64_t grid = (h->n + per - 1) / per;
  k_reduce_t<<<(unsigned)grid, NT, 0, h->s>>>(tp ? tp : h->tpart, h->n, h->nch, out, st, gate);
  if (!h->capturing) h->launches++;
  CKL("k_reduce_t");
}

ColArgs base_args(glsgpu_sur* h) {
  ColArgs a;
  std::memset(&a, 0, sizeof(a));
  a.A = h->Q;
  a.lda = h->ldm;
  a.X = h->X;
  a.ldx = h->ldx;
  a.u = h->u;
  a.su = h->su;
  for (int i = 0; i < 3; ++i) {
    a.wb[i] = h->wb[i];
    a.swb[i] = h->swb[i];
  }
  a.r = h->r;
  a.y = h->Y;
  a.ldy = h->ldy;
  a.tpart = h->tpart;
  a.rpart = h->rpart;
  a.avalid = h->ldm;
  a.gate = 0;
  return a;
}

// ------------------------------------------------------------------------------------------ TMA passes
// k_stream tile geometry: T rows per tile (128 for narrow blocks), S = 3 ring stages.
struct StreamCfg {
  int T, S;
  int64_t stage_doubles;
  size_t smem;
  int grid;
};

StreamCfg stream_cfg(const glsgpu_sur* h, int nmat, int nv) {
  StreamCfg c;
  const int nmax = h->nmax;
  // largest tile (one row per thread at T = 256) whose ring of >= 2 stages fits in ~220 KB (the opt-in
  // 227 KB less the static buffers); a third stage when it still fits: with two stages only one tile
  // is in flight while the other is consumed, too little memory-level parallelism for HBM3e
  static const char* kb_env = std::getenv("GLSGPU_STREAM_KB");  // development knob
  const int64_t budget = (kb_env ? std::atoi(kb_env) : 220) * 1024;
  c.T = 32;
  c.S = 2;
  // narrow blocks (nmax <= 32, k_stream<MODE, true>) read 32 column slots per stage
  const int64_t slots = nmax <= 32 ? std::max<int64_t>(nmat * nmax + nv, 32) : nmat * nmax + nv;
  for (int T : {256, 128, 64, 32}) {
    if (h->qt_rows && T > h->qt_rows) continue;  // never more rows than a tile of the wide blocks' Q copy
    const int64_t stage = slots * T * 8;
    const int64_t extra = (int64_t)(T + nmax + std::max(nmax, 32)) * 8;
    if (2 * stage + extra <= budget) {
      c.T = T;
      c.S = (3 * stage + extra <= budget) ? 3 : 2;
      break;
    }
  }
  c.stage_doubles = slots * c.T;
  c.smem = (size_t)(c.S * c.stage_doubles + c.T + nmax + std::max(nmax, 32)) * sizeof(double);
  const int per_sm = std::max<int>(1, (int)((227 * 1024) / (c.smem + 2048)));
  const int64_t items = (int64_t)h->G * h->nch;
  c.grid = (int)std::min<int64_t>(items, (int64_t)148 * std::min(per_sm, 4));
  return c;
}

StreamArgs stream_args(glsgpu_sur* h) {
  StreamArgs a;
  std::memset(&a, 0, sizeof(a));
  a.Q = h->Q;
  a.X = h->X;
  a.ldx = h->ldx;
  a.u = h->u;
  a.su = h->su;
  for (int i = 0; i < 3; ++i) {
    a.wb[i] = h->wb[i];
    a.swb[i] = h->swb[i];
  }
  a.r = h->r;
  a.pr = h->pr;
  a.y = h->Y;
  a.ldy = h->ldy;
  a.tpart = h->tpart;
  a.nmax = h->nmax;
  a.qtiled = h->qtiled ? 1 : 0;
  a.qtile = 256;
  a.qoff = h->d_qoff;
  if (h->qt) {
    a.Q = h->qt;
    a.qtiled = 1;
    a.qtile = h->qt_rows;
    a.qoff = h->d_qtoff;
  }
  return a;
}

template <int MODE>
int stream_nmat_host(const StreamArgs& a) {
  return MODE == SMODE_B ? 1 + a.xv_from_x : 1;
}
template <int MODE>
int stream_nvec_host() {
  return stream_nvec<MODE>();
}

// returns the grid (= number of per-CTA partials written for SMODE_C / SMODE_DIAG)
template <int MODE>
int launch_stream(glsgpu_sur* h, StreamArgs a, const SolveState* st) {
  const StreamCfg c = stream_cfg(h, stream_nmat_host<MODE>(a), stream_nvec_host<MODE>());
  a.T = c.T;
  a.S = c.S;
  a.stage_doubles = c.stage_doubles;
  // narrow blocks: one register-resident row sweep, column partials accumulated in it (k_stream FUSE)
  if constexpr (MODE == SMODE_BD || MODE == SMODE_CD) {
    k_stream<MODE, true><<<c.grid, NT, c.smem, h->s>>>(geo_of(h), a, st);  // narrow blocks only (h->fold)
  } else {
    if (h->nmax <= 32)
      k_stream<MODE, true><<<c.grid, NT, c.smem, h->s>>>(geo_of(h), a, st);
    else
      k_stream<MODE, false><<<c.grid, NT, c.smem, h->s>>>(geo_of(h), a, st);
  }
  if (!h->capturing) h->launches++;
  CKL("k_stream");
  return c.grid;
}

// dynamic shared memory attributes of every streaming mode (set outside any graph capture)
void stream_attrs(glsgpu_sur* h) {
  // the tile choice depends on nmat (pass B: 1 or 2 matrices), so allow the full opt-in maximum
  auto set = [&](const void* fn, int, int) {
    int dev = 0, maxsm = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, fn));
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm - (int)fa.sharedSizeBytes));
  };
  set((const void*)k_kron_ws<false>, 0, 0);
  set((const void*)k_kron_ws<true>, 0, 0);
  set((const void*)k_kron_mma<false>, 0, 0);
  set((const void*)k_kron_mma<true>, 0, 0);
  set((const void*)k_kron_mma2<false, 8>, 0, 0);
  set((const void*)k_kron_mma2<true, 8>, 0, 0);
  set((const void*)k_kron_mma2<false, 16>, 0, 0);
  set((const void*)k_kron_mma2<true, 16>, 0, 0);
  set((const void*)k_pass_c_mma, 0, 0);
  set((const void*)k_stream<SMODE_B, false>, 0, 0);
  set((const void*)k_stream<SMODE_B, true>, 0, 0);
  set((const void*)k_stream<SMODE_C, false>, 0, 0);
  set((const void*)k_stream<SMODE_C, true>, 0, 0);
  set((const void*)k_stream<SMODE_XS, true>, 0, 0);
  set((const void*)k_stream<SMODE_QT_R, false>, 0, 0);
  set((const void*)k_stream<SMODE_QT_R, true>, 0, 0);
  set((const void*)k_stream<SMODE_QT_D, false>, 0, 0);
  set((const void*)k_stream<SMODE_QT_D, true>, 0, 0);
  set((const void*)k_stream<SMODE_QT_V, false>, 0, 0);
  set((const void*)k_stream<SMODE_QT_V, true>, 0, 0);
  set((const void*)k_stream<SMODE_DIAG, false>, 0, 0);
  set((const void*)k_stream<SMODE_DIAG, true>, 0, 0);
  set((const void*)k_stream<SMODE_XS, false>, 0, 0);
  set((const void*)k_stream<SMODE_BD, true>, 0, 0);
  set((const void*)k_stream<SMODE_CD, true>, 0, 0);
}

// ---- pass wrappers: TMA-staged k_stream when possible, the register kernels otherwise
// Q'(w x) column partials into tpart: mode MODE_QT_R (x = r), MODE_QT_D (x = y - sw[sel]), MODE_QT_V (x = vin)
void pass_qt(glsgpu_sur* h, int mode, const double* vin, const SolveState* st, int sel_best, int gate) {
  if (h->use_stream) {
    StreamArgs a = stream_args(h);
    a.vin = vin;
    a.sel_best = sel_best;
    a.gate = gate;
    if (mode == MODE_QT_R) launch_stream<SMODE_QT_R>(h, a, st);
    else if (mode == MODE_QT_D) launch_stream<SMODE_QT_D>(h, a, st);
    else launch_stream<SMODE_QT_V>(h, a, st);
    return;
  }
  ColArgs a = base_args(h);
  a.vin = vin;
  a.sel_best = sel_best;
  a.gate = gate;
  if (mode == MODE_QT_R) launch_colpass<MODE_QT_R>(h, a, st);
  else if (mode == MODE_QT_D) launch_colpass<MODE_QT_D>(h, a, st);
  else launch_colpass<MODE_QT_V>(h, a, st);
}

// pass B of an iteration (gated on st->active)
void pass_b(glsgpu_sur* h, int xv_from_x, const SolveState* st) {
  if (h->use_stream) {
    StreamArgs a = stream_args(h);
    a.vec = h->vs;
    a.xv_from_x = xv_from_x;
    a.gate = 1;
    launch_stream<SMODE_B>(h, a, st);
    return;
  }
  ColArgs a = base_args(h);
  a.vec = h->vs;
  a.xv_from_x = xv_from_x;
  a.gate = 1;
  launch_colpass<MODE_B>(h, a, st);
}

// pr = Pi r with the dot partials (r.pr, r.r, pr.pr) per CTA; returns the number of partial rows
int pass_c(glsgpu_sur* h, const double* t, const double* r_in, double* pr_out, double* partials, const SolveState* st,
           int gate) {
  if (h->fused && r_in == h->r && pr_out == h->pr) {  // the solve's pass C: Pi r and Sigma pr in one sweep
    const int64_t ntiles = (h->ldm + KM_BM - 1) / KM_BM;
    const int grid = (int)std::min<int64_t>(ntiles, 148);
    k_pass_c_mma<<<grid, KC_NT, kc_smem_bytes(), h->s>>>(h->qmap, h->vmap64, geo_of(h), ntiles, h->omegaT, t, h->d_qoff,
                                                        h->pr, h->spr, partials, st ? st : h->st, gate);
    if (!h->capturing) h->launches++;
    CKL("k_pass_c_mma");
    return grid;
  }
  if (h->use_stream) {
    StreamArgs a = stream_args(h);
    a.vec = t;
    a.r = const_cast<double*>(r_in);
    a.pr = pr_out;
    a.partials = partials;
    a.gate = gate;
    return launch_stream<SMODE_C>(h, a, st);
  }
  const int gC = rowpass_grid(h);
  k_rowpass<<<gC, NT, 0, h->s>>>(geo_of(h), h->Q, t, r_in, pr_out, partials, 0, gate ? st : nullptr);
  if (!h->capturing) h->launches++;
  CKL("k_rowpass");
  return gC;
}

// out = w_b Q t (xstar_impl row part)
void pass_xs(glsgpu_sur* h, const double* t, double* out) {
  if (h->use_stream) {
    StreamArgs a = stream_args(h);
    a.vec = t;
    a.out = out;
    launch_stream<SMODE_XS>(h, a, nullptr);
    return;
  }
  k_rowpass<<<rowpass_grid(h), NT, 0, h->s>>>(geo_of(h), h->Q, t, nullptr, out, nullptr, 1, nullptr);
  if (!h->capturing) h->launches++;
  CKL("k_rowpass xs");
}

// trace diagnostics pass over X: X'w partials (tpart) + residual partials; returns (pointer, rows)
std::pair<double*, int> pass_diag(glsgpu_sur* h, const double* est, const SolveState* st, int gate,
                                  const double* s_q = nullptr) {
  if (h->use_stream) {
    StreamArgs a = stream_args(h);
    a.vec = s_q ? s_q : est;  // Q source (xv_mode QR): X est = Q s / w with s = R est
    a.qdiag = s_q ? 1 : 0;
    a.partials = h->rpart;
    a.gate = gate;
    const int grid = launch_stream<SMODE_DIAG>(h, a, st);
    return {h->rpart, grid};
  }
  ColArgs x = base_args(h);
  if (s_q) {  // Q source (column-major Q on this path)
    x.qdiag = 1;
    x.vec = s_q;
  } else {
    x.A = h->X;
    x.lda = h->ldx;
    x.avalid = h->M;
    x.vec = est;
  }
  x.gate = gate;
  launch_colpass<MODE_DIAG>(h, x, st);
  return {h->rpart, h->G * h->nch};
}

// ------------------------------------------------------------------------------------------ ranks
void group_barrier(glsgpu_local_group* g) {
  std::unique_lock<std::mutex> lk(g->mu);
  if (g->aborted) fail(GLSGPU_ERR_INVALID, "glsgpu local group: another rank failed");
  const uint64_t my = g->gen;
  if (++g->arrived == g->n) {
    g->arrived = 0;
    ++g->gen;
    g->cv.notify_all();
    return;
  }
  if (!g->cv.wait_for(lk, std::chrono::seconds(300), [&] { return g->gen != my || g->aborted; })) {
    g->aborted = true;
    g->cv.notify_all();
    fail(GLSGPU_ERR_INVALID, "glsgpu local group: barrier timeout (a rank stopped calling)");
  }
  if (g->aborted) fail(GLSGPU_ERR_INVALID, "glsgpu local group: another rank failed");
}

void group_abort(glsgpu_local_group* g) {
  if (!g) return;
  std::lock_guard<std::mutex> lk(g->mu);
  g->aborted = true;
  g->cv.notify_all();
}

// a group rank that fails releases the others from their barriers
struct GroupGuard {
  glsgpu_local_group* g;
  bool ok = false;
  ~GroupGuard() {
    if (!ok) group_abort(g);
  }
};

// all-gather of `count` doubles per rank in rank order (recv: nranks x count)
void allgather(glsgpu_sur* h, const double* send, double* recv, size_t count) {
  if (!h->grp) {
    nccl_check(nccl().AllGather(send, recv, count, ncclFloat64, h->comm, h->s), "ncclAllGather");
    return;
  }
  glsgpu_local_group* g = h->grp;
  const int r = h->rank;
  g->send[(size_t)r] = send;
  CK(cudaEventRecord(g->ev_ready[(size_t)r], h->s));
  group_barrier(g);  // every rank's send buffer and ready event are published
  for (int q = 0; q < g->n; ++q) {
    CK(cudaStreamWaitEvent(h->s, g->ev_ready[(size_t)q], 0));
    CK(cudaMemcpyAsync(recv + (size_t)q * count, g->send[(size_t)q], count * sizeof(double), cudaMemcpyDeviceToDevice,
                       h->s));
  }
  CK(cudaEventRecord(g->ev_done[(size_t)r], h->s));
  group_barrier(g);  // every rank has enqueued its copies
  for (int q = 0; q < g->n; ++q) CK(cudaStreamWaitEvent(h->s, g->ev_done[(size_t)q], 0));  // send buffers reusable
}

// CTA partials (count x 3) -> (pointer, rows) that a scalar kernel sums in fixed order: the partials
// themselves on one rank; on several, every rank's local sum all-gathered in rank order, so every
// rank computes bitwise the same scalars and takes the same termination decisions.
std::pair<const double*, int> combine3(glsgpu_sur* h, const double* partials, int count) {
  if (!h->coll) return {partials, count};
  k_reduce3<<<1, NT, 0, h->s>>>(partials, count, h->loc3);
  if (!h->capturing) h->launches++;
  CKL("k_reduce3");
  allgather(h, h->loc3, h->all3, 3);
  return {h->all3, h->nranks};
}

std::pair<const double*, int> combine1(glsgpu_sur* h, const double* partials, int count) {
  if (!h->coll) return {partials, count};
  k_sum1<<<1, NT, 0, h->s>>>(partials, count, h->loc3);
  if (!h->capturing) h->launches++;
  CKL("k_sum1");
  allgather(h, h->loc3, h->all3, 1);
  return {h->all3, h->nranks};
}

// tpart -> out[n], summed over chunks and then over ranks (gate as k_reduce_t).
void reduce_t_global(glsgpu_sur* h, double* out, const SolveState* st, int gate, const double* tp = nullptr) {
  if (!h->coll) {
    launch_reduce_t(h, out, st, gate, tp);
    return;
  }
  launch_reduce_t(h, h->t_loc, st, gate, tp);
  allgather(h, h->t_loc, h->t_all, (size_t)h->n);
  k_sum_ranks<<<(unsigned)std::min<int64_t>((h->n + NT - 1) / NT, 148), NT, 0, h->s>>>(h->t_all, h->nranks, h->n,
                                                                                       out, st, gate);
  if (!h->capturing) h->launches++;
  CKL("k_sum_ranks");
}

// ------------------------------------------------------------------------------------------ setup
void build_geometry(glsgpu_sur* h, int G, int64_t M, const int64_t* n_i, const double* block_scale,
                    const double* c_scale = nullptr) {
  h->G = G;
  h->M = M;
  h->ldm = round_up(M, 32);
  if (!h->mv) {
    h->msig = h->ldm;
    h->m_ref = h->M_global * G;
    h->rows_b.assign(G, h->M_global);
  }
  h->nb.resize(G);
  h->p0.resize(G);
  h->r0.resize(G);
  h->wts.resize(G);
  h->wtc.resize(G);
  int64_t p = 0, r = 0;
  int nmax = 0;
  for (int b = 0; b < G; ++b) {
    h->nb[b] = (int)n_i[b];
    h->p0[b] = p;
    h->r0[b] = r;
    p += n_i[b];
    r += n_i[b] * n_i[b];
    nmax = std::max<int>(nmax, (int)n_i[b]);
    // w = 1/sqrt(scale) (structured.cpp:430)
    h->wts[b] = 1.0 / std::sqrt(block_scale ? block_scale[b] : 1.0);
    h->wtc[b] = c_scale ? 1.0 / std::sqrt(c_scale[b]) : h->wts[b];
  }
  h->n = p;
  h->nmax = nmax;
  // row chunk of the column passes (a work item = one chunk of one block): 256-row multiples, at most ~64 chunks
  // per block; small models take chunks of up to 2048 rows (8 tiles) as long as >= 4 items per SM remain, so the
  // per-item setup and column reductions are amortised over several tiles
  {
    const int64_t ch_large = round_up((h->ldm + 63) / 64, 256);
    const int64_t ch_cap = round_up((h->ldm + (592 + G - 1) / G - 1) / ((592 + G - 1) / G), 256);
    h->CH = std::min<int64_t>(16384, std::max<int64_t>(256, std::max(ch_large, std::min<int64_t>(2048, ch_cap))));
  }
  h->nch = (int)((h->ldm + h->CH - 1) / h->CH);
  h->d_nb = dalloc<int>(G);
  h->d_p0 = dalloc<int64_t>(G);
  h->d_r0 = dalloc<int64_t>(G);
  h->d_wts = dalloc<double>(G);
  h->d_wtc = dalloc<double>(G);
  CK(cudaMemcpy(h->d_nb, h->nb.data(), sizeof(int) * G, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(h->d_p0, h->p0.data(), sizeof(int64_t) * G, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(h->d_r0, h->r0.data(), sizeof(int64_t) * G, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(h->d_wts, h->wts.data(), sizeof(double) * G, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(h->d_wtc, h->wtc.data(), sizeof(double) * G, cudaMemcpyHostToDevice));
  std::vector<int> narrow, wide;
  for (int b = 0; b < G; ++b) (h->nb[b] <= 32 ? narrow : wide).push_back(b);
  h->n_narrow = (int)narrow.size();
  h->n_wide = (int)wide.size();
  h->d_blk_narrow = dalloc<int>(narrow.size());
  h->d_blk_wide = dalloc<int>(wide.size());
  if (!narrow.empty())
    CK(cudaMemcpy(h->d_blk_narrow, narrow.data(), sizeof(int) * narrow.size(), cudaMemcpyHostToDevice));
  if (!wide.empty()) CK(cudaMemcpy(h->d_blk_wide, wide.data(), sizeof(int) * wide.size(), cudaMemcpyHostToDevice));
  // pass cost model of finalize() (structured.cpp:296-305)
  h->pi_cost = h->xstar_t_cost = h->xstar_cost = 0;
  for (int b = 0; b < G; ++b) {
    const uint64_t rr = (uint64_t)h->rows_b[b], nn = (uint64_t)h->nb[b];
    h->pi_cost += 2 * rr * nn + 2 * rr;
    h->xstar_t_cost += rr * nn + nn * (nn + 1) / 2 + rr;
    h->xstar_cost += rr * nn + nn * (nn + 1) / 2 + rr;
  }
  h->counters = glsgpu_counters_t{};
  h->counters.factorizations = (uint64_t)G;
}

// narrow blocks (n <= 32): lane-per-column leaves of 256 rows (k_qr_factor_lc / k_qr_formq_lc), or the
// previous row-per-thread register leaves of 512 rows (GLSGPU_QR_REG=1, development comparison)
bool qr_lc() {
  static const bool lc = std::getenv("GLSGPU_QR_REG") == nullptr;
  return lc;
}
int64_t narrow_leaf_rows() { return qr_lc() ? QRC_ROWS : QRR_ROWS; }
bool qr_fast(int n, int64_t rows) { return n <= 32 && rows <= narrow_leaf_rows(); }

int64_t qr_leaf_rows(int n) {
  // narrow blocks: 256-row chunks, one row per thread in registers (k_qr_factor_reg / k_qr_formq_reg)
  if (n <= 32) return narrow_leaf_rows();
  // panel rows per chunk: the panel (rows x n doubles) in <= 200 KB of shared memory when possible,
  // at least 2n rows, at most 1024 (the register column of k_qr_formq).
  int64_t L = (QR_SMEM_BYTES / 8) / n;
  L = std::min<int64_t>(L, 1024);
  L = L / 32 * 32;
  if (L < 2 * n) L = std::min<int64_t>(1024, round_up(2 * n, 32));
  return L;
}

void build_qr_plan(glsgpu_sur* h) {
  struct BT {
    int64_t L;
    std::vector<int64_t> rows, nchs, tau_off, store_off;
  };
  std::vector<BT> trees(h->G);
  int64_t store_total = 0, tau_total = 0;
  int depth_max = 0;
  for (int b = 0; b < h->G; ++b) {
    BT& t = trees[b];
    const int n = h->nb[b];
    t.L = qr_leaf_rows(n);
    int64_t rows = h->ldm;
    for (int lvl = 0;; ++lvl) {
      const int64_t nchk = std::max<int64_t>(1, (rows + t.L - 1) / t.L);
      t.rows.push_back(rows);
      t.nchs.push_back(nchk);
      t.tau_off.push_back(tau_total);
      tau_total += nchk * n;
      if (lvl == 0) t.store_off.push_back(-1);
      else {
        t.store_off.push_back(store_total);
        store_total += rows * n;
      }
      if (nchk == 1) break;
      rows = nchk * n;
    }
    depth_max = std::max<int>(depth_max, (int)t.rows.size() - 1);
  }
  h->qr_store = dalloc<double>(store_total);
  h->qr_tau = dalloc<double>(tau_total);
  std::vector<QrItem> items;
  h->qr_levels.clear();
  int64_t slot = 0;
  bool any_global = false;
  for (int lvl = 0; lvl <= depth_max; ++lvl) {
    glsgpu_sur::Level L{0, 0, 0, 0, false};
    std::vector<QrItem> fast;
    const int64_t first = (int64_t)items.size();
    L.fblock.assign((size_t)h->G + 1, 0);
    for (int b = 0; b < h->G; ++b) {
      L.fblock[(size_t)b] = (int64_t)fast.size();
      const BT& t = trees[b];
      if ((int)t.rows.size() <= lvl) continue;
      const int n = h->nb[b];
      const int64_t rows = t.rows[lvl], nchk = t.nchs[lvl];
      const bool top = (lvl == (int)t.rows.size() - 1);
      double* store_l = lvl == 0 ? nullptr : h->qr_store + t.store_off[lvl];
      double* store_next = top ? nullptr : h->qr_store + t.store_off[lvl + 1];
      const int64_t rows_next = top ? 0 : t.rows[lvl + 1];
      for (int64_t c = 0; c < nchk; ++c) {
        QrItem it;
        std::memset(&it, 0, sizeof(it));
        it.r0 = c * rows / nchk;
        it.rows = (c + 1) * rows / nchk - it.r0;
        it.rr0 = it.r0;
        it.rhalf = QRR_NT;
        it.n = n;
        if (lvl == 0 && h->qtiled) {
          // tile-contiguous Q: leaf c = rows [256 c, 256 c + 256) (zero-padded) = Q tile c of block b
          it.r0 = c * narrow_leaf_rows();
          it.rows = std::min<int64_t>(narrow_leaf_rows(), rows - it.r0);
          it.src = h->Xqr ? h->Xqr + h->p0[b] * h->ldm : h->X + h->p0[b] * h->ldx;
          it.lds = h->Xqr ? h->ldm : h->ldx;
          it.valid = h->M;
          it.scale = h->Xqr ? 1.0 : h->wts[b];
          // leaf rows [r0, r0 + L) inside the 256-row Q tiles (L = 128: half a tile; 512: two tiles)
          it.refl = h->Q + h->qoff[b] + (it.r0 / QRR_NT) * QRR_NT * (int64_t)n + it.r0 % QRR_NT;
          it.ldr = QRR_NT;
          it.rr0 = 0;
          it.rhalf = (int64_t)QRR_NT * n;
        } else if (lvl == 0) {
          it.src = h->Xqr ? h->Xqr + h->p0[b] * h->ldm : h->X + h->p0[b] * h->ldx;
          it.lds = h->Xqr ? h->ldm : h->ldx;
          it.valid = h->M;
          it.scale = h->Xqr ? 1.0 : h->wts[b];
          it.refl = h->Q + h->p0[b] * h->ldm;
          it.ldr = h->ldm;
        } else {
          it.src = store_l;
          it.lds = rows;
          it.valid = rows;
          it.scale = 1.0;
          it.refl = store_l;
          it.ldr = rows;
        }
        it.tau = h->qr_tau + t.tau_off[lvl] + c * n;
        if (top && h->coll) {
          // this rank's R goes to the cross-rank level; its C slice comes back from that level's Q
          it.rout = h->rloc + h->r0[b];
          it.ldo = n;
          it.qpar = h->rstack + (int64_t)h->nranks * h->r0[b] + (int64_t)h->rank * n;
          it.ldp = (int64_t)h->nranks * n;
        } else if (top) {
          it.rout = h->R + h->r0[b];
          it.ldo = n;
          it.qpar = nullptr;
          it.ldp = 0;
        } else {
          it.rout = store_next + c * n;
          it.ldo = rows_next;
          it.qpar = store_next + c * n;
          it.ldp = rows_next;
        }
        if (qr_fast(n, it.rows)) {
          fast.push_back(it);
          continue;
        }
        const int64_t bytes = it.rows * n * (int64_t)sizeof(double);
        it.smem = bytes <= QR_SMEM_BYTES ? 1 : 0;
        if (it.smem) L.smem_bytes = std::max<int>(L.smem_bytes, (int)bytes);
        else {
          L.any_global = true;
          any_global = true;
          slot = std::max<int64_t>(slot, it.rows * n);
        }
        L.max_rows = std::max<int64_t>(L.max_rows, it.rows);
        items.push_back(it);
      }
    }
    L.fblock[(size_t)h->G] = (int64_t)fast.size();
    L.first = first;
    L.count = (int64_t)items.size() - first;
    L.ffirst = (int64_t)items.size();
    L.fcount = (int64_t)fast.size();
    items.insert(items.end(), fast.begin(), fast.end());
    h->qr_levels.push_back(L);
  }
  h->d_items = dalloc<QrItem>(items.size());
  CK(cudaMemcpy(h->d_items, items.data(), sizeof(QrItem) * items.size(), cudaMemcpyHostToDevice));
  h->qr_slot = slot;
  // cross-rank TSQR level: per block, one chunk = the stacked per-rank R's [R_0; ...; R_{P-1}]
  if (h->coll) {
    h->gitems.clear();
    h->gsmem = 0;
    h->gmax_rows = 0;
    std::vector<int64_t> soff(h->G);
    for (int b = 0; b < h->G; ++b) {
      const int n = h->nb[b];
      QrItem it;
      std::memset(&it, 0, sizeof(it));
      soff[b] = (int64_t)h->nranks * h->r0[b];
      it.src = it.refl = h->rstack + soff[b];
      it.lds = it.ldr = (int64_t)h->nranks * n;
      it.r0 = 0;
      it.rows = it.valid = (int64_t)h->nranks * n;
      it.scale = 1.0;
      it.tau = h->gtau + h->p0[b];
      it.rout = h->R + h->r0[b];
      it.ldo = n;
      it.n = n;
      const int64_t bytes = it.rows * n * (int64_t)sizeof(double);
      it.smem = bytes <= QR_SMEM_BYTES ? 1 : 0;
      if (it.smem) h->gsmem = std::max<int>(h->gsmem, (int)bytes);
      else {
        any_global = true;
        slot = std::max<int64_t>(slot, it.rows * n);
      }
      h->gmax_rows = std::max<int64_t>(h->gmax_rows, it.rows);
      h->gitems.push_back(it);
    }
    h->qr_slot = slot;
    h->d_gitems = dalloc<QrItem>(h->gitems.size());
    CK(cudaMemcpy(h->d_gitems, h->gitems.data(), sizeof(QrItem) * h->gitems.size(), cudaMemcpyHostToDevice));
    h->d_stack_off = dalloc<int64_t>(h->G);
    CK(cudaMemcpy(h->d_stack_off, soff.data(), sizeof(int64_t) * h->G, cudaMemcpyHostToDevice));
  }
  if (any_global) h->qr_scratch = dalloc<double>((size_t)h->qr_slot * 2 * 148);
  h->d_rank_flags = dalloc<int>(h->G);
}

void launch_formq(glsgpu_sur* h, int64_t max_rows, int grid, int smem, const QrItem* items, int count) {
  if (max_rows <= 256) {
    k_qr_formq<8><<<grid, QR_NT, smem, h->s>>>(items, count, h->qr_scratch, h->qr_slot);
  } else if (max_rows <= 512) {
    k_qr_formq<16><<<grid, QR_NT, smem, h->s>>>(items, count, h->qr_scratch, h->qr_slot);
  } else {
    k_qr_formq<32><<<grid, QR_NT, smem, h->s>>>(items, count, h->qr_scratch, h->qr_slot);
  }
  if (!h->capturing) h->launches++;
  CKL("k_qr_formq");
}

// lane-per-column leaf kernels: the two-CTA-per-SM forms (default) or the original one-CTA form (GLSGPU_QR_LC=1).
// (Measured and dropped in round 2: a four-warp / 64-rows-per-warp form, 335 vs 338 ms at c4 with one fewer CTA per
// SM, and a row-per-thread form with the 32 steps unrolled, 570 ms: its per-step transpose-reduce and shuffles cost
// more than the lane-per-column broadcast.)
bool qr_lc1() {
  static const bool v = [] {
    const char* e = std::getenv("GLSGPU_QR_LC");
    return e && std::atoi(e) == 1;
  }();
  return v;
}
const void* qrf_lc_fn() { return qr_lc1() ? (const void*)k_qr_factor_lc : (const void*)k_qr_factor_lc2; }
// explicit Q of the narrow leaves: the lane-per-column kernel (default) or compact WY on the DMMA
// (GLSGPU_QR_FORMQ=wy: the same time at c4, 343 vs 337 ms per setup -- both are bound by per-leaf latency)
bool qrq_wy() {
  static const bool v = [] {
    const char* e = std::getenv("GLSGPU_QR_FORMQ");
    return e && std::strcmp(e, "wy") == 0;
  }();
  return v && !qr_lc1();
}
const void* qrq_lc_fn() {
  return qr_lc1() ? (const void*)k_qr_formq_lc : qrq_wy() ? (const void*)k_qr_formq_wy : (const void*)k_qr_formq_lc2;
}
size_t qr_lc_smem() { return qr_lc1() ? qrc_smem_bytes() : qrc2_smem_bytes(); }
size_t qrq_lc_smem() { return qrq_wy() ? qw_smem_bytes() : qr_lc_smem(); }
void launch_qrf_lc(glsgpu_sur* h, const QrItem* items, int count, int grid) {
  if (qr_lc1()) k_qr_factor_lc<<<grid, QRC_NT, qrc_smem_bytes(), h->s>>>(items, count);
  else k_qr_factor_lc2<<<grid, QRC_NT, qrc2_smem_bytes(), h->s>>>(items, count);
  if (!h->capturing) h->launches++;
  CKL("k_qr_factor_lc");
}
void launch_qrq_lc(glsgpu_sur* h, const QrItem* items, int count, int grid) {
  if (qr_lc1()) k_qr_formq_lc<<<grid, QRC_NT, qrc_smem_bytes(), h->s>>>(items, count);
  else if (qrq_wy()) k_qr_formq_wy<<<grid, QW_NT, qw_smem_bytes(), h->s>>>(items, count);
  else k_qr_formq_lc2<<<grid, QRC_NT, qrc2_smem_bytes(), h->s>>>(items, count);
  if (!h->capturing) h->launches++;
  CKL("k_qr_formq_lc");
}
// resident CTAs of the lane-per-column leaves (the item loop strides by gridDim: a second wave would serialise)
void qr_lc_grids(glsgpu_sur* h, int* gf, int* gq) {
  CK(cudaFuncSetAttribute(qrf_lc_fn(), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qr_lc_smem()));
  CK(cudaFuncSetAttribute(qrq_lc_fn(), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qrq_lc_smem()));
  int occ_f = 1, occ_q = 1, nsm = 148;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_f, qrf_lc_fn(), QRC_NT, qr_lc_smem()));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_q, qrq_lc_fn(), QRC_NT, qrq_lc_smem()));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, h->dev));
  *gf = std::max(1, occ_f) * nsm;
  *gq = std::max(1, occ_q) * nsm;
}


// ---- CholeskyQR2 setup (cqr.cuh) ----------------------------------------------------------------------------
// GLSGPU_QR=tsqr keeps the Householder TSQR as the only factorisation (development comparison / fallback tests)
bool cqr_enabled() {  // read at every handle creation (the tests switch it)
  const char* e = std::getenv("GLSGPU_QR");
  return !(e && std::strcmp(e, "tsqr") == 0);
}

template <int NBP, int MODE>
void launch_cqr_pass_t(glsgpu_sur* h, const CqArgs& a) {
  static bool attr_done[8] = {false};  // per device ordinal (the attribute is per context)
  if (h->dev >= 8 || !attr_done[h->dev]) {
    CK(cudaFuncSetAttribute(k_cqr_pass<NBP, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)cq_smem_bytes<NBP, MODE>()));
    if (h->dev < 8) attr_done[h->dev] = true;
  }
  int nsm = 148;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, h->dev));
  const int grid = std::min(a.nitems, nsm);
  k_cqr_pass<NBP, MODE><<<grid, CQ_NT, cq_smem_bytes<NBP, MODE>(), h->s>>>(a);
  if (!h->capturing) h->launches++;
  CKL("k_cqr_pass");
}

template <int MODE>
void launch_cqr_pass(glsgpu_sur* h, const CqArgs& a) {
  if (h->cq_nbp == 32) launch_cqr_pass_t<32, MODE>(h, a);
  else if (h->cq_nbp == 64) launch_cqr_pass_t<64, MODE>(h, a);
  else launch_cqr_pass_t<128, MODE>(h, a);
}

void build_cqr_plan(glsgpu_sur* h) {
  // (a sharded handle: every rank must take the same factorisation -- its collectives differ -- so all ranks must
  // be on the TMA passes; GLSGPU_QR must agree across ranks)
  h->cq = cqr_enabled() && !h->mv && !h->no_qtile && (h->coll ? h->all_stream : h->use_stream) && h->nmax <= 128;
  if (!h->cq) return;
  h->cq_nbp = h->nmax <= 32 ? 32 : h->nmax <= 64 ? 64 : 128;
  h->cq_tr = h->cq_nbp == 32 ? CqCfg<32>::TR : h->cq_nbp == 64 ? CqCfg<64>::TR : CqCfg<128>::TR;
  const int64_t TR = h->cq_tr;
  // rows per item: ~4736 / G items per block (about 32 per SM in all), at least 16 tiles and 40 NBP rows (the
  // item's partial Gram stays below ~3% of its input)
  const int64_t target = std::max<int64_t>(1, (4736 + h->G - 1) / h->G);
  const int64_t rpi = round_up(std::max<int64_t>({(h->M + target - 1) / target, 16 * TR, 40 * (int64_t)h->cq_nbp}), TR);
  std::vector<CqItem> items;
  std::vector<int> nsrc((size_t)h->G);
  std::vector<int64_t> xoff((size_t)h->G);
  h->cq_first.assign((size_t)h->G + 1, 0);
  for (int b = 0; b < h->G; ++b) {
    h->cq_first[(size_t)b] = (int64_t)items.size();
    for (int64_t r = 0; r < h->M; r += rpi) {
      const int64_t rows = std::min(rpi, h->M - r);
      items.push_back(CqItem{b, (int)((rows + TR - 1) / TR), r});
    }
    nsrc[(size_t)b] = (int)((int64_t)items.size() - h->cq_first[(size_t)b]);
    xoff[(size_t)b] = h->p0[(size_t)b] * h->ldx;
  }
  h->cq_first[(size_t)h->G] = (int64_t)items.size();
  const int64_t nn = (int64_t)h->cq_nbp * h->cq_nbp;
  h->d_cq_items = dalloc<CqItem>(items.size());
  CK(cudaMemcpy(h->d_cq_items, items.data(), sizeof(CqItem) * items.size(), cudaMemcpyHostToDevice));
  h->d_cq_first = dalloc<int64_t>((size_t)h->G + 1);
  CK(cudaMemcpy(h->d_cq_first, h->cq_first.data(), sizeof(int64_t) * ((size_t)h->G + 1), cudaMemcpyHostToDevice));
  h->d_cq_nsrc = dalloc<int>((size_t)h->G);
  CK(cudaMemcpy(h->d_cq_nsrc, nsrc.data(), sizeof(int) * (size_t)h->G, cudaMemcpyHostToDevice));
  h->d_cq_xoff = dalloc<int64_t>((size_t)h->G);
  CK(cudaMemcpy(h->d_cq_xoff, xoff.data(), sizeof(int64_t) * (size_t)h->G, cudaMemcpyHostToDevice));
  h->cq_gpart = dalloc<double>((size_t)(items.size() * nn));
  int64_t rtot = 0;
  for (int b = 0; b < h->G; ++b) rtot += (int64_t)h->nb[b] * h->nb[b];
  h->cq_r1 = dalloc<double>((size_t)rtot);
  h->cq_rinv = dalloc<double>((size_t)h->G * h->cq_nbp * (h->cq_nbp + 4));
  h->d_cq_flags = dalloc<int>((size_t)h->G);
  if (h->coll) {
    std::vector<int64_t> bidx((size_t)h->G);
    for (int b = 0; b < h->G; ++b) bidx[(size_t)b] = b;
    std::vector<int> np((size_t)h->G, h->nranks);
    h->d_cq_bidx = dalloc<int64_t>((size_t)h->G);
    CK(cudaMemcpy(h->d_cq_bidx, bidx.data(), sizeof(int64_t) * (size_t)h->G, cudaMemcpyHostToDevice));
    h->d_cq_np = dalloc<int>((size_t)h->G);
    CK(cudaMemcpy(h->d_cq_np, np.data(), sizeof(int) * (size_t)h->G, cudaMemcpyHostToDevice));
    h->cq_gloc = dalloc<double>((size_t)(h->G * nn));
    h->cq_gall = dalloc<double>((size_t)(h->G * nn * h->nranks));
  }
}

template <bool FINAL>
void launch_cqr_chol(glsgpu_sur* h, int b0, int b1) {
  const size_t smem = (size_t)h->nmax * (h->nmax + 1) * sizeof(double);
  CK(cudaFuncSetAttribute(k_cqr_chol<FINAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (h->coll) {
    // this rank's Grams -> all ranks -> summed in rank order inside the Cholesky kernel
    const int64_t nn = (int64_t)h->cq_nbp * h->cq_nbp;
    k_cqr_sum<<<h->G, 256, 0, h->s>>>(h->cq_nbp, h->cq_gpart, h->d_cq_first, h->d_cq_nsrc, h->cq_gloc);
    if (!h->capturing) h->launches++;
    CKL("k_cqr_sum");
    allgather(h, h->cq_gloc, h->cq_gall, (size_t)(h->G * nn));
    k_cqr_chol<FINAL><<<h->G, 256, smem, h->s>>>(h->cq_nbp, 0, h->d_nb, h->d_r0, h->d_wts, h->cq_gall, h->d_cq_bidx,
                                                 h->d_cq_np, h->G, h->cq_r1, h->R, h->cq_rinv, h->d_cq_flags);
  } else {
    k_cqr_chol<FINAL><<<b1 - b0, 256, smem, h->s>>>(h->cq_nbp, b0, h->d_nb, h->d_r0, h->d_wts, h->cq_gpart,
                                                    h->d_cq_first, h->d_cq_nsrc, 1, h->cq_r1, h->R, h->cq_rinv,
                                                    h->d_cq_flags);
  }
  if (!h->capturing) h->launches++;
  CKL("k_cqr_chol");
}

// CholeskyQR2 of blocks [b0, b1): Q and R of the handle (flags in d_cq_flags, read by cqr_ok)
void run_cqr_blocks(glsgpu_sur* h, int b0, int b1) {
  const int64_t i0 = h->cq_first[(size_t)b0], cnt = h->cq_first[(size_t)b1] - i0;
  if (cnt <= 0) return;
  const int64_t nn = (int64_t)h->cq_nbp * h->cq_nbp;
  CK(cudaMemsetAsync(h->d_cq_flags + b0, 0, sizeof(int) * (size_t)(b1 - b0), h->s));
  CqArgs a{};
  a.items = h->d_cq_items + i0;
  a.nitems = (int)cnt;
  a.nb = h->d_nb;
  a.src = h->X;
  a.src_off = h->d_cq_xoff;
  a.src_cs = h->ldx;
  a.src_tiled = 0;
  a.src_valid = h->M;
  a.dst = h->Q;
  a.dst_off = h->d_qoff;
  a.dst_cs = h->qtiled ? h->cq_tr : h->ldm;
  a.dst_tiled = h->qtiled ? 1 : 0;
  a.dst_rows = h->qtiled ? round_up(h->ldm, QRR_NT) : h->ldm;
  a.rinv = h->cq_rinv;
  a.gpart = h->cq_gpart + i0 * nn;
  launch_cqr_pass<0>(h, a);
  launch_cqr_chol<false>(h, b0, b1);
  launch_cqr_pass<1>(h, a);
  launch_cqr_chol<true>(h, b0, b1);
  CqArgs c = a;  // in place on Q
  c.src = h->Q;
  c.src_off = h->d_qoff;
  c.src_cs = a.dst_cs;
  c.src_tiled = a.dst_tiled;
  c.src_valid = a.dst_rows;
  launch_cqr_pass<2>(h, c);
}

// did every block take the CholeskyQR2 factor?  (synchronises the solver stream)
bool cqr_ok(glsgpu_sur* h) {
  std::vector<int> flags((size_t)h->G);
  CK(cudaMemcpyAsync(flags.data(), h->d_cq_flags, sizeof(int) * (size_t)h->G, cudaMemcpyDeviceToHost, h->s));
  CK(cudaStreamSynchronize(h->s));
  for (int f : flags)
    if (f) return false;
  return true;
}

// The TSQR of blocks [b0, b1) only, every level, when every item is a lane-per-column leaf (narrow blocks):
// lets glsgpu_sur_create factor one group of blocks while the next group's columns are still in flight.
bool qr_groupable(const glsgpu_sur* h) {
  if (h->cq) return !h->coll;
  if (h->coll || !qr_lc()) return false;
  for (const auto& L : h->qr_levels)
    if (L.count) return false;
  return true;
}

void run_qr_blocks(glsgpu_sur* h, int b0, int b1, int lc_grid_f, int lc_grid_q) {
  if (h->cq) {
    run_cqr_blocks(h, b0, b1);
    return;
  }
  const int nl = (int)h->qr_levels.size();
  for (int l = 0; l < nl; ++l) {
    const auto& L = h->qr_levels[l];
    const int64_t f0 = L.fblock[(size_t)b0], cnt = L.fblock[(size_t)b1] - f0;
    if (cnt <= 0) continue;
    launch_qrf_lc(h, h->d_items + L.ffirst + f0, (int)cnt, (int)std::min<int64_t>(cnt, lc_grid_f));
  }
  for (int l = nl - 1; l >= 0; --l) {
    const auto& L = h->qr_levels[l];
    const int64_t f0 = L.fblock[(size_t)b0], cnt = L.fblock[(size_t)b1] - f0;
    if (cnt <= 0) continue;
    launch_qrq_lc(h, h->d_items + L.ffirst + f0, (int)cnt, (int)std::min<int64_t>(cnt, lc_grid_q));
  }
}

void rank_check(glsgpu_sur* h);
void run_tsqr(glsgpu_sur* h);

// group-pipelined setup from host X: group g's columns go up on a copy stream while the solver stream
// factors group g - 1 (the whole TSQR tree of its blocks), so the QR hides under the host-to-device copy
void upload_and_qr_pipelined(glsgpu_sur* h, const double* X_host, int groups) {
  int lc_grid_f = 148, lc_grid_q = 148;
  if (!h->cq) {
    qr_lc_grids(h, &lc_grid_f, &lc_grid_q);
    CK(cudaMemsetAsync(h->Q, 0, sizeof(double) * (size_t)h->qsize, h->s));  // CholeskyQR2 writes every row itself
  }
  cudaStream_t cs = nullptr;
  CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  std::vector<cudaEvent_t> ev((size_t)groups, nullptr);
  try {
    for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaEvent_t ready;  // the padding-row memsets on h->s precede every column copy
    CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    CK(cudaEventRecord(ready, h->s));
    CK(cudaStreamWaitEvent(cs, ready, 0));
    const int G = h->G;
    for (int g = 0; g < groups; ++g) {
      const int b0 = (int)((int64_t)g * G / groups), b1 = (int)((int64_t)(g + 1) * G / groups);
      const int64_t c0 = h->p0[(size_t)b0], c1 = b1 < G ? h->p0[(size_t)b1] : h->n;
      if (c1 > c0)
        CK(cudaMemcpy2DAsync(h->X_own + c0 * h->ldm, h->ldm * sizeof(double), X_host + c0 * h->M, h->M * sizeof(double),
                             h->M * sizeof(double), (size_t)(c1 - c0), cudaMemcpyHostToDevice, cs));
      CK(cudaEventRecord(ev[(size_t)g], cs));
    }
    for (int g = 0; g < groups; ++g) {
      const int b0 = (int)((int64_t)g * G / groups), b1 = (int)((int64_t)(g + 1) * G / groups);
      CK(cudaStreamWaitEvent(h->s, ev[(size_t)g], 0));
      run_qr_blocks(h, b0, b1, lc_grid_f, lc_grid_q);
    }
    CK(cudaStreamSynchronize(h->s));
    cudaEventDestroy(ready);
  } catch (...) {
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    cudaStreamSynchronize(cs);
    cudaStreamDestroy(cs);
    throw;
  }
  for (auto e : ev) cudaEventDestroy(e);
  cudaStreamDestroy(cs);
  h->cq_last = h->cq;
  if (h->cq && !cqr_ok(h)) {
    h->cq_fallbacks++;
    h->cq_last = false;
    run_tsqr(h);
    return;
  }
  rank_check(h);
}

// the factorisation of the handle's resident X: CholeskyQR2 where the handle takes it, Householder TSQR otherwise or
// when a block fails CholeskyQR2's own test (ill-conditioned or rank-deficient blocks)
void run_qr(glsgpu_sur* h) {
  if (h->cq) {
    run_cqr_blocks(h, 0, h->G);
    h->cq_last = cqr_ok(h);
    if (h->cq_last) {
      rank_check(h);
      return;
    }
    h->cq_fallbacks++;
  }
  run_tsqr(h);
}

void run_tsqr(glsgpu_sur* h) {
  CK(cudaFuncSetAttribute(k_qr_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)QR_SMEM_BYTES));
  CK(cudaFuncSetAttribute(k_qr_formq<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)QR_SMEM_BYTES));
  CK(cudaFuncSetAttribute(k_qr_formq<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)QR_SMEM_BYTES));
  CK(cudaFuncSetAttribute(k_qr_formq<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)QR_SMEM_BYTES));
  // zero Q (its padding rows stay zero) -- the level-0 reflectors overwrite the rest
  CK(cudaMemsetAsync(h->Q, 0, sizeof(double) * (size_t)h->qsize, h->s));
  const int nl = (int)h->qr_levels.size();
  CK(cudaFuncSetAttribute(k_qr_formq_reg<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, QRR_ROWS * 32 * 8));
  int lc_grid_f = 148, lc_grid_q = 148;
  qr_lc_grids(h, &lc_grid_f, &lc_grid_q);
  const int fgrid_cap = 2 * 148;  // register-resident leaves: 1-2 CTAs per SM
  for (int l = 0; l < nl; ++l) {
    const auto& L = h->qr_levels[l];
    if (L.count) {
      const int grid = (int)std::min<int64_t>(L.count, L.any_global ? 2 * 148 : 8 * 148);
      k_qr_factor<<<grid, QR_NT, L.smem_bytes, h->s>>>(h->d_items + L.first, (int)L.count, h->qr_scratch,
                                                      h->qr_slot);
      if (!h->capturing) h->launches++;
      CKL("k_qr_factor");
    }
    if (L.fcount) {
      if (qr_lc())
        launch_qrf_lc(h, h->d_items + L.ffirst, (int)L.fcount, (int)std::min<int64_t>(L.fcount, lc_grid_f));
      else {
        k_qr_factor_reg<32><<<(int)std::min<int64_t>(L.fcount, fgrid_cap), QRR_NT, 0, h->s>>>(h->d_items + L.ffirst,
                                                                                             (int)L.fcount);
        if (!h->capturing) h->launches++;
        CKL("k_qr_factor_reg");
      }
    }
  }
  if (h->coll) {
    // TSQR across ranks: gather every rank's top R, factor the stacks (redundantly, identically on
    // every rank), form their explicit Q; each rank's C slice then seeds its local top level
    int64_t rtot = 0;
    for (int b = 0; b < h->G; ++b) rtot += (int64_t)h->nb[b] * h->nb[b];
    allgather(h, h->rloc, h->rall, (size_t)rtot);
    int64_t* d_r0 = h->d_r0;
    k_stack_r<<<h->G, 256, 0, h->s>>>(h->rall, h->nranks, rtot, h->G, h->d_nb, d_r0, h->d_stack_off, h->rstack);
    if (!h->capturing) h->launches++;
    CKL("k_stack_r");
    const int grid = (int)std::min<int64_t>(h->G, 2 * 148);
    k_qr_factor<<<grid, QR_NT, h->gsmem, h->s>>>(h->d_gitems, h->G, h->qr_scratch, h->qr_slot);
    if (!h->capturing) h->launches++;
    CKL("k_qr_factor ranks");
    launch_formq(h, h->gmax_rows, grid, h->gsmem, h->d_gitems, h->G);
  }
  for (int l = nl - 1; l >= 0; --l) {
    const auto& L = h->qr_levels[l];
    if (L.count) {
      const int grid = (int)std::min<int64_t>(L.count, L.any_global ? 2 * 148 : 8 * 148);
      launch_formq(h, L.max_rows, grid, L.smem_bytes, h->d_items + L.first, (int)L.count);
    }
    if (L.fcount) {
      if (qr_lc())
        launch_qrq_lc(h, h->d_items + L.ffirst, (int)L.fcount, (int)std::min<int64_t>(L.fcount, lc_grid_q));
      else {
        k_qr_formq_reg<32><<<(int)std::min<int64_t>(L.fcount, fgrid_cap), QRR_NT, QRR_ROWS * 32 * 8, h->s>>>(
            h->d_items + L.ffirst, (int)L.fcount);
        if (!h->capturing) h->launches++;
      }
      CKL("k_qr_formq_reg");
    }
  }
  rank_check(h);
}

void rank_check(glsgpu_sur* h) {
  if (h->qt) {  // the streaming passes' tiled copy of the new Q
    const dim3 grid(64, (unsigned)h->G);
    k_q_relayout<<<grid, NT, 0, h->s>>>(h->Q, h->ldm, h->d_p0, h->d_nb, h->d_qtoff, h->qt_rows, h->G, h->qt);
    if (!h->capturing) h->launches++;
    CKL("k_q_relayout");
  }
  Geo g = geo_of(h);
  k_rank_check<<<(h->G + 127) / 128, 128, 0, h->s>>>(g, h->R, h->d_rank_flags);
  if (!h->capturing) h->launches++;
  CKL("k_rank_check");
  std::vector<int> flags(h->G);
  CK(cudaMemcpyAsync(flags.data(), h->d_rank_flags, sizeof(int) * h->G, cudaMemcpyDeviceToHost, h->s));
  CK(cudaStreamSynchronize(h->s));
  h->factors_ok = false;
  for (int b = 0; b < h->G; ++b)
    if (flags[b]) {
      if (h->rank_msg == 1) fail(GLSGPU_ERR_RANK_DEFICIENT, "qr: matrix is numerically rank deficient", b);
      fail(GLSGPU_ERR_RANK_DEFICIENT,
           std::string(h->mv ? "mvrglm_preconditioner: stacked block " : "sur_preconditioner: block ") +
               std::to_string(b) + " is rank deficient",
           b);
    }
  h->factors_ok = true;
}

// every operator apply / solve needs the factors of the handle's current X (a failed update or refactor
// leaves rank-deficient factors behind: the handle refuses work until a successful one)
void require_factors(const glsgpu_sur* h) {
  if (!h->factors_ok)
    fail(GLSGPU_ERR_RANK_DEFICIENT, "glsgpu: the handle's last factorisation failed (rank deficient); update or "
                                    "refactor it first");
}

void validate(int G, int64_t M, const int64_t* n_i, const double* block_scale, const double* omega,
              bool need_m_gt_n = true) {
  if (G < 1) fail(GLSGPU_ERR_DIMENSION_MISMATCH, "make_sur: need at least one block");
  if (!n_i || !omega) fail(GLSGPU_ERR_INVALID, "glsgpu_sur_create: null argument");
  if (M < 1) fail(GLSGPU_ERR_DIMENSION_MISMATCH, "make_sur: block row mismatch");
  if (G > 512) fail(GLSGPU_ERR_UNSUPPORTED, "glsgpu: G > 512 equations is outside this build's Kronecker kernel");
  for (int b = 0; b < G; ++b) {
    if (block_scale && !(block_scale[b] > 0.0))
      fail(GLSGPU_ERR_SINGULAR_D, "sur_preconditioner: scales must be positive", b);
    if (n_i[b] < 1 || M < n_i[b]) fail(GLSGPU_ERR_DIMENSION_MISMATCH, "qr: need rows >= cols >= 1", b);
    if (n_i[b] > 512) fail(GLSGPU_ERR_UNSUPPORTED, "glsgpu: block width > 512 is outside this build's kernels", b);
  }
  int64_t n = 0;
  for (int b = 0; b < G; ++b) n += n_i[b];
  if (need_m_gt_n && M * G <= n) fail(GLSGPU_ERR_DIMENSION_MISMATCH, "make_glm: need m > n >= 1");
}

void upload_omega(glsgpu_sur* h, const double* omega) {
  const int G = h->G;
  h->omega_h.assign(omega, omega + (size_t)G * G);
  std::vector<double> ot((size_t)G * G);
  for (int p = 0; p < G; ++p)
    for (int c = 0; c < G; ++c) ot[(size_t)p * G + c] = omega[p + (size_t)c * G];  // row p of Omega
  h->omegaT = dalloc<double>((size_t)G * G);
  CK(cudaMemcpy(h->omegaT, ot.data(), sizeof(double) * G * G, cudaMemcpyHostToDevice));
}

void alloc_common(glsgpu_sur* h) {
  // TMA-staged passes need 16-byte aligned column segments of X reaching every padded row
  h->use_stream = h->nmax <= 128 && h->ldx >= h->ldm && (h->ldx % 2) == 0 &&
                  (reinterpret_cast<uintptr_t>(h->X) % 16) == 0 && std::getenv("GLSGPU_NO_TMA") == nullptr;
  // tile-contiguous Q (256-row tiles per block) when every block takes the register-resident QR leaves
  h->qtiled = h->use_stream && h->nmax <= 32 && !h->no_qtile && std::getenv("GLSGPU_NO_QTILE") == nullptr;
  h->qoff.assign(h->G, 0);
  int64_t qsize = 0;
  for (int b = 0; b < h->G; ++b) {
    h->qoff[b] = h->qtiled ? qsize : h->p0[b] * h->ldm;
    qsize += (h->qtiled ? round_up(h->ldm, QRR_NT) : h->ldm) * h->nb[b];
  }
  h->qsize = qsize;
  h->Q = dalloc<double>((size_t)qsize);
  if (h->use_stream && !h->qtiled && !h->no_qtile && std::getenv("GLSGPU_NO_QTILE") == nullptr) {
    // tile rows = what pass C and pass B (QR mode) pick for these widths, so their tiles move as one bulk copy
    h->qt_rows = 0;
    h->qt_rows = (int)std::min(stream_cfg(h, 1, stream_nvec<SMODE_C>()).T, stream_cfg(h, 1, stream_nvec<SMODE_B>()).T);
    std::vector<int64_t> qto(h->G, 0);
    int64_t tot = 0;
    for (int b = 0; b < h->G; ++b) {
      qto[b] = tot;
      tot += round_up(h->ldm, h->qt_rows) * h->nb[b];
    }
    h->qt = dalloc<double>((size_t)tot);
    h->d_qtoff = dalloc<int64_t>(h->G);
    CK(cudaMemcpy(h->d_qtoff, qto.data(), sizeof(int64_t) * h->G, cudaMemcpyHostToDevice));
  }
  h->d_qoff = dalloc<int64_t>(h->G);
  CK(cudaMemcpy(h->d_qoff, h->qoff.data(), sizeof(int64_t) * h->G, cudaMemcpyHostToDevice));
  int64_t rtot = 0;
  for (int b = 0; b < h->G; ++b) rtot += (int64_t)h->nb[b] * h->nb[b];
  h->R = dalloc<double>((size_t)rtot);
  if (h->coll) {
    const int P = h->nranks;
    if ((int64_t)P * h->nmax > 1024)
      fail(GLSGPU_ERR_UNSUPPORTED, "glsgpu: nranks * max n_i > 1024 (cross-rank TSQR level)");
    h->rloc = dalloc<double>((size_t)rtot);
    h->rall = dalloc<double>((size_t)rtot * P);
    h->rstack = dalloc<double>((size_t)rtot * P);
    h->gtau = dalloc<double>((size_t)h->n);
    h->loc3 = dalloc<double>(4);
    h->all3 = dalloc<double>((size_t)4 * P);
    h->t_loc = dalloc<double>((size_t)h->n);
    h->t_all = dalloc<double>((size_t)h->n * P);
    // do all ranks take the TMA-staged passes?  (ranks with unaligned row counts do not)
    const double mine = h->use_stream ? 1.0 : 0.0;
    std::vector<double> all((size_t)P);
    CK(cudaMemcpyAsync(h->loc3, &mine, sizeof(double), cudaMemcpyHostToDevice, h->s));
    allgather(h, h->loc3, h->all3, 1);
    CK(cudaMemcpyAsync(all.data(), h->all3, sizeof(double) * P, cudaMemcpyDeviceToHost, h->s));
    CK(cudaStreamSynchronize(h->s));
    h->all_stream = true;
    for (double v : all) h->all_stream = h->all_stream && v != 0.0;
  } else {
    h->all_stream = h->use_stream;
  }
  build_qr_plan(h);
  build_cqr_plan(h);
}

void destroy_impl(glsgpu_sur* h) {
  if (!h) return;
  cudaSetDevice(h->dev);
  if (h->s) cudaStreamSynchronize(h->s);
  if (h->graph) cudaGraphExecDestroy(h->graph);
  if (h->ne_graph) cudaGraphExecDestroy(h->ne_graph);
  for (double* q : {h->neLr, h->neLc, h->nebuf})
    if (q) cudaFree(q);
  for (auto e : h->tev) cudaEventDestroy(e);
  void* ptrs[] = {h->d_nb, h->d_p0, h->d_r0, h->d_wts, h->d_wtc, h->Xqr, h->omegaInvT, h->d_ones, h->qt, h->d_qtoff,
                  h->X_own, h->Y_own, h->Q, h->R, h->omegaT, h->d_items,
                  h->qr_store, h->qr_tau, h->qr_scratch, h->d_rank_flags, h->d_blk_narrow, h->d_blk_wide,
                  h->mvec, h->t,
                  h->vs, h->est, h->t2, h->xtw, h->zvec, h->beta_d, h->tpart, h->rpart, h->partA, h->partC,
                  h->scal, h->d_stop, h->st, h->rows_d, h->loc3, h->all3, h->t_loc, h->t_all, h->rloc, h->rall,
                  h->rstack, h->gtau, h->d_stack_off, h->d_gitems, h->d_qoff, h->d_cq_items, h->d_cq_first,
                  h->d_cq_nsrc, h->d_cq_xoff, h->cq_gpart, h->cq_r1, h->cq_rinv, h->d_cq_flags, h->d_cq_bidx, h->d_cq_np,
                  h->cq_gloc, h->cq_gall};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (h->cs) {
    cudaStreamSynchronize(h->cs);
    cudaStreamDestroy(h->cs);
  }
  if (h->ev_qr) cudaEventDestroy(h->ev_qr);
  if (h->ev_stage) cudaEventDestroy(h->ev_stage);
  if (h->Y_next) cudaFree(h->Y_next);
  if (h->t3) cudaFree(h->t3);
  if (h->tpart2) cudaFree(h->tpart2);
  if (h->tpart3) cudaFree(h->tpart3);
  if (h->st_host) cudaFreeHost(h->st_host);
  if (h->comm) nccl().CommDestroy(h->comm);
  if (h->s) cudaStreamDestroy(h->s);
  delete h;
}

// MVRGLM embedding of glsgpu_mvrglm_create (set on the handle before the geometry is built)
struct MvDesc {
  int64_t M0 = 0, ktot = 0;
  std::vector<int64_t> kb, kofs;
  const double* c_scale = nullptr;
};

glsgpu_sur* create_common(int G, int64_t M, const int64_t* n_i, const double* omega, const double* block_scale,
                          int device, int64_t M_global = -1, int rank = 0, int nranks = 1,
                          const void* nccl_id = nullptr, const MvDesc* mvd = nullptr, bool qr_only = false,
                          glsgpu_local_group* grp = nullptr) {
  if (M_global < 0) M_global = M;
  validate(G, M_global, n_i, block_scale, omega, /*need_m_gt_n=*/!qr_only);
  if (nranks < 1 || rank < 0 || rank >= nranks) fail(GLSGPU_ERR_INVALID, "glsgpu: bad rank / nranks");
  if (grp && (grp->n != nranks || grp->dev != device))
    fail(GLSGPU_ERR_INVALID, "glsgpu: local group size / device differ from nranks / device");
  if (nranks > 1) {
    if (!nccl_id && !grp) fail(GLSGPU_ERR_INVALID, "glsgpu: sharded handle needs an NCCL unique id");
    for (int b = 0; b < G; ++b)
      if (M < n_i[b]) fail(GLSGPU_ERR_DIMENSION_MISMATCH, "glsgpu: every rank must own at least max n_i rows", b);
  }
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    fail(GLSGPU_ERR_NO_DEVICE, "glsgpu: no CUDA device available (there is no CPU fallback)");
  }
  if (device < 0 || device >= ndev) fail(GLSGPU_ERR_INVALID, "glsgpu: bad device ordinal");
  CK(cudaSetDevice(device));
  glsgpu_sur* h = new glsgpu_sur();
  h->dev = device;
  h->rank = rank;
  h->nranks = nranks;
  h->M_global = M_global;
  h->coll = nranks > 1 || nccl_id != nullptr || grp != nullptr;
  h->grp = grp;
  try {
    CK(cudaStreamCreateWithFlags(&h->s, cudaStreamNonBlocking));
    if (h->coll && !grp) {
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof(id));
      nccl_check(nccl().CommInitRank(&h->comm, nranks, id, rank), "ncclCommInitRank");
    }
    if (mvd) {
      h->mv = true;
      h->M0 = mvd->M0;
      h->kb = mvd->kb;
      h->kofs = mvd->kofs;
      h->msig = mvd->M0;
      h->m_ref = (int64_t)G * mvd->M0 + mvd->ktot;
      h->rows_b.resize(G);
      for (int b = 0; b < G; ++b) h->rows_b[b] = mvd->M0 + mvd->kb[b];
    }
    build_geometry(h, G, M, n_i, block_scale, mvd ? mvd->c_scale : nullptr);
    upload_omega(h, omega);
  } catch (...) {
    destroy_impl(h);
    throw;
  }
  return h;
}

// 2-D tensor map over the vector slab: rows = ldm (inner), columns = MV_COUNT * G; boxes of 32 rows x
// 8 columns (one pass-A element chunk of one vector).  cuTensorMapEncodeTiled comes from the driver
// through the runtime's entry-point query (no libcuda link).
bool make_vmap(glsgpu_sur* h, CUtensorMap* map, int box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {(cuuint64_t)h->ldm, (cuuint64_t)MV_COUNT * h->G};
  const cuuint64_t strides[1] = {(cuuint64_t)h->ldm * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)box_rows, (cuuint32_t)KG_BK};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult rc = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, h->mvec, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return rc == CUDA_SUCCESS;
}

// tile-contiguous Q as a 2-D tensor: inner = the 256 rows of a tile, outer = every tile column of every block
bool make_qmap(glsgpu_sur* h) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {(cuuint64_t)QRR_NT, (cuuint64_t)(h->qsize / QRR_NT)};
  const cuuint64_t strides[1] = {(cuuint64_t)QRR_NT * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)KM_BM, 32u};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult rc = encode(&h->qmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, h->Q, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return rc == CUDA_SUCCESS;
}

void ensure_solver(glsgpu_sur* h, int64_t rows_cap) {
  if (!h->solver_ready) {
    const size_t mv = (size_t)(h->ldm * h->G);
    h->mvec = dalloc<double>(mv * MV_COUNT);
    for (int i = 0; i < 3; ++i) {
      h->wb[i] = h->mvec + (MV_W + i) * mv;
      h->swb[i] = h->mvec + (MV_SW + i) * mv;
    }
    h->r = h->mvec + MV_R * mv;
    h->u = h->mvec + MV_U * mv;
    h->su = h->mvec + MV_SU * mv;
    h->pr = h->mvec + MV_PR * mv;
    h->spr = h->mvec + MV_SPR * mv;
    h->vmap_ok = make_vmap(h, &h->vmap, KG_BM);
    h->vmap64_ok = make_vmap(h, &h->vmap64, KM_BM);
    h->qmap_ok = h->qtiled && make_qmap(h);
    h->t = dalloc<double>(h->n);
    h->t3 = dalloc<double>(h->n);
    h->vs = dalloc<double>(h->n);
    h->est = dalloc<double>(h->n);
    h->t2 = dalloc<double>(h->n);
    h->xtw = dalloc<double>(h->n);
    h->zvec = dalloc<double>(h->n);
    h->beta_d = dalloc<double>(h->n);
    h->tpart = dalloc<double>((size_t)h->n * h->nch);
    h->tpart2 = dalloc<double>((size_t)h->n * h->nch);
    h->tpart3 = dalloc<double>((size_t)h->n * h->nch);
    h->rpart = dalloc<double>((size_t)std::max<int64_t>((int64_t)h->G * h->nch, 4 * GRID_CAP));
    h->partA = dalloc<double>(std::max(GRID_CAP, EW_GRID) * 3);  // k_pass_a_ew (fused_c) writes EW_GRID rows
    h->partC = dalloc<double>(GRID_CAP * 3);
    h->scal = dalloc<double>(64);
    h->d_stop = dalloc<int>(1);
    h->st = dalloc<SolveState>(1);
    CK(cudaMallocHost(&h->st_host, sizeof(SolveState)));
    for (int i = 0; i < 3; ++i) {
      CK(cudaMemsetAsync(h->wb[i], 0, mv * sizeof(double), h->s));
      CK(cudaMemsetAsync(h->swb[i], 0, mv * sizeof(double), h->s));
    }
    CK(cudaMemsetAsync(h->r, 0, mv * sizeof(double), h->s));
    CK(cudaMemsetAsync(h->u, 0, mv * sizeof(double), h->s));
    CK(cudaMemsetAsync(h->su, 0, mv * sizeof(double), h->s));
    CK(cudaMemsetAsync(h->pr, 0, mv * sizeof(double), h->s));
    h->solver_ready = true;
    stream_attrs(h);
    // kron kernels: >48 KB dynamic shared memory at large G
    CK(cudaFuncSetAttribute(k_kron<8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * 32 * 8));
    CK(cudaFuncSetAttribute(k_kron<16, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 512 * 16 * 8));
    CK(cudaFuncSetAttribute(k_kron<4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (128 * 32 + 128 * 128) * 8));
    CK(cudaFuncSetAttribute(k_kron<2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (64 * 32 + 64 * 64) * 8));
    CK(cudaFuncSetAttribute(k_colpass<MODE_B, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)(h->CH * 8)));
    CK(cudaFuncSetAttribute(k_colpass<MODE_QT_R, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)(h->CH * 8)));
    CK(cudaFuncSetAttribute(k_colpass<MODE_QT_D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)(h->CH * 8)));
    CK(cudaFuncSetAttribute(k_colpass<MODE_QT_V, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)(h->CH * 8)));
    CK(cudaFuncSetAttribute(k_colpass<MODE_DIAG, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)(h->CH * 8)));
  }
  if (rows_cap > h->rows_cap_d) {
    if (h->rows_d) CK(cudaFree(h->rows_d));
    h->rows_d = dalloc<TraceRowD>((size_t)rows_cap);
    h->rows_cap_d = rows_cap;
  }
}

// m-vector host (ld M per equation) <-> device (ld ldm)
// MVRGLM handles map the reference's embedded order (G M0 observation rows, then the k constraint rows,
// equation 0's first; structured.cpp:85-90) onto the padded per-block layout [obs; constraints; 0].
void h2d_mvec(glsgpu_sur* h, double* dst, const double* src) {
  if (!h->mv) {
    CK(cudaMemcpy2DAsync(dst, h->ldm * sizeof(double), src, h->M * sizeof(double), h->M * sizeof(double), h->G,
                         cudaMemcpyHostToDevice, h->s));
    return;
  }
  CK(cudaMemsetAsync(dst, 0, sizeof(double) * h->ldm * h->G, h->s));
  CK(cudaMemcpy2DAsync(dst, h->ldm * sizeof(double), src, h->M0 * sizeof(double), h->M0 * sizeof(double), h->G,
                       cudaMemcpyHostToDevice, h->s));
  for (int b = 0; b < h->G; ++b)
    if (h->kb[b])
      CK(cudaMemcpyAsync(dst + (int64_t)b * h->ldm + h->M0, src + (int64_t)h->G * h->M0 + h->kofs[b],
                         sizeof(double) * h->kb[b], cudaMemcpyHostToDevice, h->s));
}
void d2h_mvec(glsgpu_sur* h, double* dst, const double* src) {
  if (!h->mv) {
    CK(cudaMemcpy2DAsync(dst, h->M * sizeof(double), src, h->ldm * sizeof(double), h->M * sizeof(double), h->G,
                         cudaMemcpyDeviceToHost, h->s));
    return;
  }
  CK(cudaMemcpy2DAsync(dst, h->M0 * sizeof(double), src, h->ldm * sizeof(double), h->M0 * sizeof(double), h->G,
                       cudaMemcpyDeviceToHost, h->s));
  for (int b = 0; b < h->G; ++b)
    if (h->kb[b])
      CK(cudaMemcpyAsync(dst + (int64_t)h->G * h->M0 + h->kofs[b], src + (int64_t)b * h->ldm + h->M0,
                         sizeof(double) * h->kb[b], cudaMemcpyDeviceToHost, h->s));
}

// t_out = (Q' (w_b x))_b partials reduced: a Q'-apply of an m-vector already on the device.
void qt_apply(glsgpu_sur* h, int mode, const double* vin, double* out, const SolveState* st, int sel_best) {
  pass_qt(h, mode, vin, st, sel_best, 0);
  reduce_t_global(h, out, nullptr, 0);
}

double norm_probe(glsgpu_sur* h, int64_t iters) {
  // operator_norm_probe (pcg.cpp:233-244) starts from v = 1/sqrt(m) 1.  For Sigma = Omega (x) I_M every
  // row of reshape(v, M, G) then stays equal: v = 1_M x' and Sigma v = 1_M (x' Omega) (operators.cpp:45-50),
  // so the power iteration is exactly an iteration on the G-vector x with |v| = sqrt(M |x|^2).  Each
  // entry of Sigma v is the reference's own p-ascending sum; only the norm's summation order differs.
  // O(iters G^2) on the host instead of iters full Kronecker passes over M x G.
  // MVRGLM: Sigma = diag(Omega0 (x) I_M0, 0_k): the start vector has m = G M0 + k entries, the k constraint
  // entries vanish after the first apply and the rest stay row-constant per block over the M0 rows under Sigma
  const int G = h->G;
  const double Mg = static_cast<double>(h->mv ? h->M0 : h->M_global);
  const double m = static_cast<double>(h->m_ref);
  std::vector<double> x((size_t)G, 1.0 / std::sqrt(m)), y((size_t)G);
  double nrm = 0.0;
  for (int64_t it = 0; it < iters; ++it) {
    for (int j = 0; j < G; ++j) {
      double s = 0.0;
      for (int p = 0; p < G; ++p) {
        const double o = h->omega_h[(size_t)p + (size_t)j * G];
        if (o == 0.0) continue;
        s += x[(size_t)p] * o;
      }
      y[(size_t)j] = s;
    }
    double ss = 0.0;
    for (int j = 0; j < G; ++j) ss += y[(size_t)j] * y[(size_t)j];
    nrm = std::sqrt(Mg * ss);
    if (nrm == 0.0) return 0.0;
    for (int j = 0; j < G; ++j) x[(size_t)j] = y[(size_t)j] / nrm;
  }
  return nrm;
}

// ------------------------------------------------------------------------------------------ solve
// init scalars after the first pi apply: c = max(r.pr, 0), c1, threshold, pi_gain (pcg.cpp:72-86)
__global__ void k_init_scalars(const double* partials, int count, SolveState* st, TraceRowD* rows) {
  __shared__ double res[3];
  reduce_partials<3>(partials, count, res);
  if (threadIdx.x == 0) {
    double c = res[0];
    if (c < 0.0) c = 0.0;
    st->c = c;
    st->c1 = c;
    st->threshold = st->tol_rel * st->tol_rel * c;
    st->c_best = c;
    const double rr = res[1], prn = sqrt(res[2]);
    if (rr > 0.0) st->pi_gain = dmax_std(st->pi_gain, prn / sqrt(rr));
    if (st->rows_cap > 0) {
      rows[0].iter = 0;
      rows[0].c = c;
      rows[0].aug = __longlong_as_double(0x7ff8000000000000LL);
      rows[0].dual = rows[0].aug;
      rows[0].rmse = rows[0].aug;
      rows[0].elapsed_ns = (int64_t)(globaltimer() - st->t0);
    }
    if (c == 0.0) {
      st->term = T_CONVERGED;
      st->active = 0;
    }
  }
}

__global__ void k_set_t0(SolveState* st) { st->t0 = globaltimer(); }

// PCG-NE: out_b = X_b v_b (rows < M; padding rows 0), grid.y = block
__global__ void k_xapply(Geo g, const double* __restrict__ X, int64_t ldx, const double* __restrict__ v,
                         double* __restrict__ out, const SolveState* st = nullptr) {
  if (st && !st->active) return;
  const int b = blockIdx.y;
  const int nb = g.nb[b];
  const int64_t p0 = g.p0[b];
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < g.ldm; k += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    if (k < g.M)
      for (int j = 0; j < nb; ++j) s = s + X[(p0 + j) * ldx + k] * v[p0 + j];
    out[(int64_t)b * g.ldm + k] = s;
  }
}
// r = y - r over the M x G rows (padding rows stay 0)
__global__ void k_ysub(Geo g, const double* __restrict__ y, int64_t ldy, double* __restrict__ r) {
  const int b = blockIdx.y;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < g.ldm; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = (int64_t)b * g.ldm + k;
    r[o] = k < g.M ? y[(int64_t)b * ldy + k] - r[o] : 0.0;
  }
}

// MVRGLM embed: X[pos[i]] = 1 (the selector rows C_b(q, restr_b[q]) = 1, structured.cpp:83-84)
__global__ void k_set_ones(double* X, const int64_t* pos, int64_t count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    X[pos[i]] = 1.0;
}
// dst = D^-1/2 src per block of `per` columns: rows < msig times wz_b, the rest times wc_b (the stacked
// [Z0 w_z; C_i w_c] of MvRglmPreconditioner, structured.cpp:380-384)
__global__ void k_scale_rows(double* dst, const double* src, int64_t ld, int64_t ncols, int64_t per, int64_t msig,
                             const double* wz, const double* wc) {
  const int64_t total = ld * ncols;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = i / ld, k = i - col * ld;
    const int b = (int)(col / per);
    dst[i] = src[i] * (k < msig ? wz[b] : wc[b]);
  }
}

// X is the current factors' X (not overwritten by a staged upload of the next model)
void require_x(const glsgpu_sur* h, const char* what) {
  if (h->x_released)
    fail(GLSGPU_ERR_UNSUPPORTED, std::string(what) + ": X was released to the staged upload of the next model "
                                                     "(glsgpu_sur_stage); use xv_mode QR without w1 / z1, or "
                                                     "glsgpu_sur_update_staged first");
}

// One trace row's diagnostics (pcg.cpp:96-116): est = X*'(y - sw) (recover), |y - sw - X est|, |X' w| and the
// rmse.  gated: the per-iteration (captured) form, active on st->diag_now rows; otherwise trace row `row`.
// xv_mode QR never reads X: X est = Q s / w with s = Q'(w (y - sw)) = R est itself, and X' w = R' Q' w / w.
void diag_row(glsgpu_sur* h, int xv_mode, bool gated, int64_t row) {
  const int gate = gated ? 2 : 0;
  const SolveState* gst = gated ? h->st : nullptr;
  Geo g = geo_of(h);
  // the same on every rank (ranks may differ in use_stream): both pass kinds have a Q-source form
  const bool q = xv_mode == GLSGPU_XV_QR;
  if (!q) require_x(h, "trace diagnostics (xv_mode X)");
  pass_qt(h, MODE_QT_D, nullptr, h->st, 0, gate);
  reduce_t_global(h, h->t2, gst, gate);
  if (q) {
    k_copy_gated<<<(unsigned)std::min<int64_t>((h->n + NT - 1) / NT, 148), NT, 0, h->s>>>(h->t3, h->t2, h->n, gst);
    if (!h->capturing) h->launches++;
    CKL("k_copy_gated");
  }
  k_vupdate<<<(h->G + 63) / 64, 64, 0, h->s>>>(g, h->R, h->t2, nullptr, 1, 2, gst);
  if (!h->capturing) h->launches++;
  CKL("k_vupdate diag");
  const auto rp = pass_diag(h, h->t2, h->st, gate, q ? h->t3 : nullptr);
  reduce_t_global(h, q ? h->t3 : h->xtw, gst, gate);
  if (q) {
    k_rt_apply<<<dim3((unsigned)((h->nmax + 63) / 64), (unsigned)h->G), 64, 0, h->s>>>(g, h->R, h->t3, h->xtw, gst);
    if (!h->capturing) h->launches++;
    CKL("k_rt_apply");
  }
  const auto pr1 = combine1(h, rp.first, rp.second);
  k_diag_finalize<<<1, NT, 0, h->s>>>(pr1.first, pr1.second, h->xtw, h->n, h->t2, h->beta_d, h->st, h->rows_d,
                                      gated ? -1 : row);
  if (!h->capturing) h->launches++;
  CKL("k_diag_finalize");
}

void capture_iteration(glsgpu_sur* h, int xv_mode, int diag, int timing, int iter_idx) {
  Geo g = geo_of(h);
  const int gA = kron_grid(h);
  const int xfx = (xv_mode == GLSGPU_XV_X) ? 1 : 0;
  auto ev = [&](int k) {
    if (timing) CK(cudaEventRecordWithFlags(h->tev[(size_t)iter_idx * 6 + k], h->s, cudaEventRecordExternal));
  };
  // pass A: u = pr + mu u, su = Sigma u, d = u.su, uu = u.u
  ev(0);
  launch_pass_a(h);
  ev(1);
  const auto pa = combine3(h, h->partA, gA);
  k_scalar_a<<<1, NT, 0, h->s>>>(pa.first, pa.second, h->st);
  if (!h->capturing) h->launches++;
  CKL("k_scalar_a");
  if (h->fold) {
    // passes B and C with the row's diagnostics folded in (SMODE_BD / SMODE_CD)
    ev(2);
    StreamArgs ab = stream_args(h);
    ab.vec = h->vs;
    ab.gate = 1;
    ab.zbuf = h->spr;
    ab.tpart2 = h->tpart2;
    launch_stream<SMODE_BD>(h, ab, h->st);
    ev(3);
    reduce_t_global(h, h->t, h->st, 1);
    reduce_t_global(h, h->t2, h->st, 1, h->tpart2);  // s_est = Q'(w (y - sw_{i+1}))
    ev(4);
    StreamArgs ac = stream_args(h);
    ac.vec = h->t;
    ac.vec2 = h->t2;
    ac.zbuf = h->spr;
    ac.partials = h->partC;
    ac.partials2 = h->rpart;
    ac.tpart3 = h->tpart3;
    ac.gate = 1;
    const int gCD = launch_stream<SMODE_CD>(h, ac, h->st);
    ev(5);
    const auto pcd = combine3(h, h->partC, gCD);
    k_scalar_c<<<1, NT, 0, h->s>>>(pcd.first, pcd.second, h->st, h->rows_d);
    if (!h->capturing) h->launches++;
    CKL("k_scalar_c");
    k_vupdate<<<(h->G + 63) / 64, 64, 0, h->s>>>(g, h->R, h->t, h->vs, xfx, 0, h->st);
    if (!h->capturing) h->launches++;
    CKL("k_vupdate");
    // the row: est = R^-1 s_est, X'w = R' Q'w / w, |y - sw - X est|, rmse (gated on st->diag_now)
    reduce_t_global(h, h->t3, h->st, 2, h->tpart3);
    k_vupdate<<<(h->G + 63) / 64, 64, 0, h->s>>>(g, h->R, h->t2, nullptr, 1, 2, h->st);
    if (!h->capturing) h->launches++;
    k_rt_apply<<<dim3((unsigned)((h->nmax + 63) / 64), (unsigned)h->G), 64, 0, h->s>>>(g, h->R, h->t3, h->xtw, h->st);
    if (!h->capturing) h->launches++;
    const auto pr1 = combine1(h, h->rpart, gCD);
    k_diag_finalize<<<1, NT, 0, h->s>>>(pr1.first, pr1.second, h->xtw, h->n, h->t2, h->beta_d, h->st, h->rows_d, -1);
    if (!h->capturing) h->launches++;
    CKL("folded diagnostics");
    return;
  }
  // pass B: w, sw, r updates + Q'(w r) column partials
  ev(2);
  pass_b(h, xfx, h->st);
  ev(3);
  reduce_t_global(h, h->t, h->st, 1);
  // pass C: pr = Pi r, c = r.pr
  ev(4);
  const int gC = pass_c(h, h->t, h->r, h->pr, h->partC, h->st, 1);
  ev(5);
  const auto pcc = combine3(h, h->partC, gC);
  k_scalar_c<<<1, NT, 0, h->s>>>(pcc.first, pcc.second, h->st, h->rows_d);
  if (!h->capturing) h->launches++;
  CKL("k_scalar_c");
  k_vupdate<<<(h->G + 63) / 64, 64, 0, h->s>>>(g, h->R, h->t, h->vs, xfx, 0, h->st);
  if (!h->capturing) h->launches++;
  CKL("k_vupdate");
  if (diag >= 0) {
    // est = X*'(y - sw) and the row diagnostics, gated on st->diag_now
    if (h->sw_direct && !kron_mma_apply(h, -2, nullptr))
      launch_kron(h, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 3, h->st, nullptr);
    diag_row(h, xv_mode, true, -1);
  }
}

// the copy stream and events of the staged-upload path (created on first use)
void ensure_stage_objects(glsgpu_sur* h) {
  if (!h->cs) CK(cudaStreamCreateWithFlags(&h->cs, cudaStreamNonBlocking));
  if (!h->ev_qr) CK(cudaEventCreateWithFlags(&h->ev_qr, cudaEventDisableTiming));
  if (!h->ev_stage) CK(cudaEventCreateWithFlags(&h->ev_stage, cudaEventDisableTiming));
}

// a staged upload still in flight is finished (or dropped) before X / Y are written another way
void settle_staged(glsgpu_sur* h) {
  if (h->cs) CK(cudaStreamSynchronize(h->cs));
  h->staged = false;
}

// after a factorisation of X_own: the staged path may overwrite X_own once the QR has consumed it
void mark_factored(glsgpu_sur* h) {
  if (h->ev_qr) CK(cudaEventRecord(h->ev_qr, h->s));
  h->x_released = false;
  h->frob_x = -1.0;  // |X|_F of the new X (w1 projection) is recomputed on demand
}

// host X (M x n, ld M) and Y (M x G, ld M) -> X_own / Y_own, then the factorisation (pipelined by block groups
// with the H2D where the TSQR allows it; the cross-rank TSQR level of a sharded handle runs after the copy)
void upload_and_factor(glsgpu_sur* h, const double* X, const double* Y) {
  const int64_t M = h->M;
  CK(cudaMemcpy2DAsync(h->Y_own, h->ldm * sizeof(double), Y, M * sizeof(double), M * sizeof(double), h->G,
                       cudaMemcpyHostToDevice, h->s));
  static const bool no_overlap = std::getenv("GLSGPU_NO_OVERLAP") != nullptr;
  if (!no_overlap && qr_groupable(h) && h->G >= 2) {
    upload_and_qr_pipelined(h, X, std::min(h->G, 8));
  } else {
    CK(cudaMemcpy2DAsync(h->X_own, h->ldm * sizeof(double), X, M * sizeof(double), M * sizeof(double), h->n,
                         cudaMemcpyHostToDevice, h->s));
    run_qr(h);
  }
  mark_factored(h);
}

// handle that owns its X / Y (host inputs): glsgpu_sur_create (one rank) and glsgpu_sur_create_sharded_host
glsgpu_sur* create_host_owned(int G, int64_t M, int64_t M_global, const int64_t* n_i, const double* X, const double* Y,
                              const double* omega, const double* block_scale, int device, int rank, int nranks,
                              const void* nccl_id) {
  static const bool trace = std::getenv("GLSGPU_TRACE_CREATE") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
  };
  const auto t0 = now();
  glsgpu_sur* h = create_common(G, M, n_i, omega, block_scale, device, M_global, rank, nranks, nccl_id);
  try {
    h->X_own = dalloc<double>((size_t)(h->ldm * h->n));
    h->Y_own = dalloc<double>((size_t)(h->ldm * G));
    if (h->ldm > M)  // padding rows only: the copies write rows [0, M)
      CK(cudaMemset2DAsync(h->X_own + M, h->ldm * sizeof(double), 0, (h->ldm - M) * sizeof(double), h->n, h->s));
    CK(cudaMemsetAsync(h->Y_own, 0, sizeof(double) * h->ldm * G, h->s));
    h->X = h->X_own;
    h->ldx = h->ldm;
    h->Y = h->Y_own;
    h->ldy = h->ldm;
    alloc_common(h);
    CK(cudaStreamSynchronize(h->s));
    const auto t1 = now();
    upload_and_factor(h, X, Y);
    if (trace)
      std::fprintf(stderr, "glsgpu create: allocate + plan %.1f ms, upload + QR %.1f ms\n", ms(t0, t1), ms(t1, now()));
  } catch (...) {
    destroy_impl(h);
    throw;
  }
  return h;
}

// C = op(A) op(B) on the DMMA GEMM of gemm.cuh (column-major; split-K when the tile grid is smaller than the GPU);
// lower: only the lower-triangle tiles of a square C (the Gram for a lower-triangle eigensolver)
void dgemm_dev(cudaStream_t s, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, bool tA, const double* B,
               int64_t ldb, bool tB, double* C, int64_t ldc, bool lower, std::vector<void*>& bufs) {
  const int64_t tm = (m + GM_BM - 1) / GM_BM, tn = (n + GM_BN - 1) / GM_BN;
  const int64_t tiles = lower ? tm * (tm + 1) / 2 : tm * tn;
  int splits = (int)std::min<int64_t>(std::max<int64_t>(1, (2 * 148 + tiles - 1) / tiles), 64);
  splits = (int)std::max<int64_t>(1, std::min<int64_t>(splits, (k + 255) / 256));
  const dim3 grid((unsigned)tm, (unsigned)tn, (unsigned)splits);
  if (splits == 1) {
    k_gemm_dmma<<<grid, GM_NT, 0, s>>>(m, n, k, A, lda, tA ? 1 : 0, B, ldb, tB ? 1 : 0, C, ldc, 0, lower ? 1 : 0);
    CKL("k_gemm_dmma");
    return;
  }
  const int64_t stride = ldc * n;
  double* parts = dalloc<double>((size_t)(stride * splits));
  bufs.push_back(parts);
  CK(cudaMemsetAsync(parts, 0, sizeof(double) * stride * splits, s));
  k_gemm_dmma<<<grid, GM_NT, 0, s>>>(m, n, k, A, lda, tA ? 1 : 0, B, ldb, tB ? 1 : 0, parts, ldc, stride, lower ? 1 : 0);
  CKL("k_gemm_dmma split");
  k_gemm_reduce<<<(unsigned)std::min<int64_t>((m * n + 255) / 256, 148 * 8), 256, 0, s>>>(m, n, parts, stride, splits, C,
                                                                                         ldc);
  CKL("k_gemm_reduce");
}

}  // namespace

// ================================================================================ C ABI
extern "C" {

const char* glsgpu_last_error_message(void) { return g_err.c_str(); }
const char* glsgpu_version(void) { return "glsgpu 0.1 (sm_100a, fp64, no-FMA)"; }

int glsgpu_device_count(int* count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  if (count) *count = n;
  return n > 0 ? GLSGPU_OK : GLSGPU_ERR_NO_DEVICE;
}

void glsgpu_default_config(glsgpu_pcg_config* c) {
  std::memset(c, 0, sizeof(*c));
  c->tol_rel = 1e-10;
  c->max_iter = 0;
  c->breakdown_tol = 1e-14;
  c->stagnation_window = 5;
  c->growth_tol = 1e4;
  c->growth_window = 10;
  c->record_z_every = 1;
  c->diag_every = 1;
  c->xv_mode = GLSGPU_XV_X;
  c->graph_chunk = 0;
  c->kernel_timing = 0;
  c->kron_fma = 0;
  c->sw_mode = 0;
  c->fused_c = 0;
}

#define API_BEGIN try {
#define API_END(badp)                          \
  }                                            \
  catch (const GErr& e) {                      \
    g_err = e.msg;                             \
    if (badp && e.block >= 0) *(badp) = e.block; \
    return e.code;                             \
  }                                            \
  catch (const std::exception& e) {            \
    g_err = e.what();                          \
    return GLSGPU_ERR_CUDA;                    \
  }                                            \
  return GLSGPU_OK;

int glsgpu_sur_create(int G, int64_t M, const int64_t* n_i, const double* X, const double* Y, const double* omega,
                      const double* block_scale, int device, glsgpu_sur** out, int* bad_block) {
  API_BEGIN
  if (!out || !X || !Y) fail(GLSGPU_ERR_INVALID, "glsgpu_sur_create: null argument");
  *out = nullptr;
  *out = create_host_owned(G, M, M, n_i, X, Y, omega, block_scale, device, 0, 1, nullptr);
  API_END(bad_block)
}

int glsgpu_sur_create_sharded_host(int G, int64_t M_local, int64_t M_global, const int64_t* n_i, const double* X,
                                   const double* Y, const double* omega, const double* block_scale, int device,
                                   const void* nccl_id, int rank, int nranks, glsgpu_sur** out, int* bad_block) {
  API_BEGIN
  if (!out || !X || !Y || !nccl_id) fail(GLSGPU_ERR_INVALID, "glsgpu_sur_create_sharded_host: null argument");
  *out = nullptr;
  *out = create_host_owned(G, M_local, M_global, n_i, X, Y, omega, block_scale, device, rank, nranks, nccl_id);
  API_END(bad_block)
}

// New data for an existing host-created SUR handle (same G, M, widths; on a sharded handle this rank's rows):
// upload X and Y and refactor, reusing every allocation and the TSQR plan -- the per-solve cost of a "create
// once, solve many" caller.
int glsgpu_sur_update(glsgpu_sur* h, const double* X, const double* Y, int* bad_block) {
  API_BEGIN
  if (!h || !X || !Y) fail(GLSGPU_ERR_INVALID, "glsgpu_sur_update: null argument");
  if (!h->X_own || h->mv) fail(GLSGPU_ERR_UNSUPPORTED, "glsgpu_sur_update: needs a host-created SUR handle");
  CK(cudaSetDevice(h->dev));
  settle_staged(h);
  upload_and_factor(h, X, Y);
  API_END(bad_block)
}

// Stage the NEXT model's data (same shapes as glsgpu_sur_update): X and Y go up on the handle's copy stream as
// soon as the current factorisation has consumed X_own, overlapping whatever the solver stream runs meanwhile
// (a solve in xv_mode QR never reads X).  X and Y should be pinned host memory for the copy to be
// asynchronous, and must stay untouched until glsgpu_sur_update_staged returns.
int glsgpu_sur_stage(glsgpu_sur* h, const double* X, const double* Y) {
  API_BEGIN
  if (!h || !X || !Y) fail(GLSGPU_ERR_INVALID, "glsgpu_sur_stage: null argument");
  if (!h->X_own || h->mv) fail(GLSGPU_ERR_UNSUPPORTED, "glsgpu_sur_stage: needs a host-created SUR handle");
  CK(cudaSetDevice(h->dev));
  if (h->staged) fail(GLSGPU_ERR_INVALID, "glsgpu_sur_stage: an upload is already staged");
  ensure_stage_objects(h);
  if (!h->Y_next) h->Y_next = dalloc<double>((size_t)(h->ldm * h->G));
  const int64_t M = h->M;
  // X_own / the spare Y are free once everything enqueued so far on the solver stream (the last factorisation
  // among it) is done; the solve that follows runs concurrently with the copy
  CK(cudaEventRecord(h->ev_qr, h->s));
  CK(cudaStreamWaitEvent(h->cs, h->ev_qr, 0));
  if (h->ldm > M) CK(cudaMemsetAsync(h->Y_next, 0, sizeof(double) * h->ldm * h->G, h->cs));
  CK(cudaMemcpy2DAsync(h->Y_next, h->ldm * sizeof(double), Y, M * sizeof(double), M * sizeof(double), h->G,
                       cudaMemcpyHostToDevice, h->cs));
  CK(cudaMemcpy2DAsync(h->X_own, h->ldm * sizeof(double), X, M * sizeof(double), M * sizeof(double), h->n,
                       cudaMemcpyHostToDevice, h->cs));
  CK(cudaEventRecord(h->ev_stage, h->cs));
  h->staged = true;
  h->x_released = true;
  API_END((int*)nullptr)
}

// Make the staged model current: the solver stream waits for the staged copy, then refactors (glsgpu_sur_update
// without the copy).
int glsgpu_sur_update_staged(glsgpu_sur* h, int* bad_block) {
  API_BEGIN
  if (!h) fail(GLSGPU_ERR_INVALID, "glsgpu_sur_update_staged: null handle");
  if (!h->staged) fail(GLSGPU_ERR_INVALID, "glsgpu_sur_update_staged: nothing staged (glsgpu_sur_stage)");
  CK(cudaSetDevice(h->dev));
  CK(cudaStreamWaitEvent(h->s, h->ev_stage, 0));
  std::swap(h->Y_own, h->Y_next);
  h->Y = h->Y_own;
  h->staged = false;
  run_qr(h);
  mark_factored(h);
  API_END(bad_block)
}
int glsgpu_sur_create_device(int G, int64_t M, const int64_t* n_i, const double* X_dev, int64_t ldx,
                             const double* Y_dev, int64_t ldy, const double* omega, const double* block_scale,
                             int device, glsgpu_sur** out, int* bad_block) {
  API_BEGIN
  if (!out || !X_dev || !Y_dev) fail(GLSGPU_ERR_INVALID, "glsgpu_sur_create_device: null argument");
  if (ldx < M || ldy < M) fail(GLSGPU_ERR_DIMENSION_MISMATCH, "glsgpu_sur_create_device: leading dimension < M");
  *out = nullptr;
  glsgpu_sur* h = create_common(G, M, n_i, omega, block_scale, device);
  try {
    h->X = X_dev;
    h->ldx = ldx;
    h->Y = Y_dev;
    h->ldy = ldy;
    alloc_common(h);
    run_qr(h);
  } catch (...) {
    destroy_impl(h);
    throw;
  }
  *out = h;
  API_END(bad_block)
}

int glsgpu_sur_refactor(glsgpu_sur* h, int* bad_block) {
  API_BEGIN
  if (!h) fail(GLSGPU_ERR_INVALID, "null handle");
  CK(cudaSetDevice(h->dev));
  require_x(h, "glsgpu_sur_refactor");
  run_qr(h);
  mark_factored(h);  // also resets |X|_F: X may have been changed in place
  API_END(bad_block)
}

int glsgpu_sur_destroy(glsgpu_sur* h) {
  API_BEGIN
  destroy_impl(h);
  API_END((int*)nullptr)
}

int glsgpu_sur_dims(const glsgpu_sur* h, int* G, int64_t* M, int64_t* n) {
  if (!h) return GLSGPU_ERR_INVALID;
  if (G) *G = h->G;
  if (M) *M = h->M;
  if (n) *n = h->n;
  return GLSGPU_OK;
}

void* glsgpu_sur_stream(const glsgpu_sur* h) { return h ? (void*)h->s : nullptr; }

int glsgpu_counters(const glsgpu_sur* h, glsgpu_counters_t* out) {
  if (!h || !out) return GLSGPU_ERR_INVALID;
  *out = h->counters;
  return GLSGPU_OK;
}

int glsgpu_reset_apply_counters(glsgpu_sur* h) {
  if (!h) return GLSGPU_ERR_INVALID;
  h->counters.pi_applies = h->counters.xstar_t_applies = h->counters.xstar_applies = 0;
  h->counters.apply_multiplies = 0;
  return GLSGPU_OK;
}

int glsgpu_apply_pi(glsgpu_sur* h, const double* xi, double* out) {
  API_BEGIN
  if (!h || !xi || !out) fail(GLSGPU_ERR_INVALID, "apply_pi: null argument");
  CK(cudaSetDevice(h->dev));
  require_factors(h);
  ensure_solver(h, 1);
  h->counters.pi_applies++;
  h->counters.apply_multiplies += h->pi_cost;
  h2d_mvec(h, h->r, xi);
  qt_apply(h, MODE_QT_R, nullptr, h->t, nullptr, 0);
  pass_c(h, h->t, h->r, h->pr, h->partC, nullptr, 0);
  d2h_mvec(h, out, h->pr);
  CK(cudaStreamSynchronize(h->s));
  API_END((int*)nullptr)
}

int glsgpu_apply_xstar_t(glsgpu_sur* h, const double* xi, double* out) {
  API_BEGIN
  if (!h || !xi || !out) fail(GLSGPU_ERR_INVALID, "apply_xstar_t: null argument");
  CK(cudaSetDevice(h->dev));
  require_factors(h);
  ensure_solver(h, 1);
  h->counters.xstar_t_applies++;
  h->counters.apply_multiplies += h->xstar_t_cost;
  h2d_mvec(h, h->r, xi);
  qt_apply(h, MODE_QT_R, nullptr, h->t, nullptr, 0);
  Geo g = geo_of(h);
  k_vupdate<<<(h->G + 63) / 64, 64, 0, h->s>>>(g, h->R, h->t, nullptr, 1, 2, nullptr);
  if (!h->capturing) h->launches++;
  CKL("k_vupdate");
  CK(cudaMemcpyAsync(out, h->t, sizeof(double) * h->n, cudaMemcpyDeviceToHost, h->s));
  CK(cudaStreamSynchronize(h->s));
  API_END((int*)nullptr)
}

int glsgpu_apply_xstar(glsgpu_sur* h, const double* v, double* out) {
  API_BEGIN
  if (!h || !v || !out) fail(GLSGPU_ERR_INVALID, "apply_xstar: null argument");
  CK(cudaSetDevice(h->dev));
  require_factors(h);
  ensure_solver(h, 1);
  h->counters.xstar_applies++;
  h->counters.apply_multiplies += h->xstar_cost;
  CK(cudaMemcpyAsync(h->t, v, sizeof(double) * h->n, cudaMemcpyHostToDevice, h->s));
  Geo g = geo_of(h);
  k_vupdate<<<(h->G + 63) / 64, 64, 0, h->s>>>(g, h->R, h->t, nullptr, 1, 3, nullptr);
  if (!h->capturing) h->launches++;
  CKL("k_vupdate");
  pass_xs(h, h->t, h->pr);
  d2h_mvec(h, out, h->pr);
  CK(cudaStreamSynchronize(h->s));
  API_END((int*)nullptr)
}

int glsgpu_sigma_apply(glsgpu_sur* h, const double* x, double* out) {
  API_BEGIN
  if (!h || !x || !out) fail(GLSGPU_ERR_INVALID, "sigma_apply: null argument");
  CK(cudaSetDevice(h->dev));
  ensure_solver(h, 1);
  h2d_mvec(h, h->r, x);
  launch_kron(h, h->r, nullptr, nullptr, nullptr, h->su, h->partA, 0, nullptr, nullptr);
  d2h_mvec(h, out, h->su);
  CK(cudaStreamSynchronize(h->s));
  API_END((int*)nullptr)
}

int glsgpu_operator_norm_probe(glsgpu_sur* h, int64_t iters, double* norm) {
  API_BEGIN
  if (!h || !norm) fail(GLSGPU_ERR_INVALID, "operator_norm_probe: null argument");
  CK(cudaSetDevice(h->dev));
  *norm = norm_probe(h, iters);
  API_END((int*)nullptr)
}

int glsgpu_get_factors(const glsgpu_sur* h, double* Q, double* R) {
  API_BEGIN
  if (!h) fail(GLSGPU_ERR_INVALID, "null handle");
  CK(cudaSetDevice(h->dev));
  if (Q && !h->qtiled) {
    CK(cudaMemcpy2D(Q, h->M * sizeof(double), h->Q, h->ldm * sizeof(double), h->M * sizeof(double), h->n,
                    cudaMemcpyDeviceToHost));
  } else if (Q) {
    // tile-contiguous -> column-major M x n
    std::vector<double> qt((size_t)h->qsize);
    CK(cudaMemcpy(qt.data(), h->Q, sizeof(double) * h->qsize, cudaMemcpyDeviceToHost));
    for (int b = 0; b < h->G; ++b) {
      const int nb = h->nb[b];
      for (int j = 0; j < nb; ++j)
        for (int64_t k = 0; k < h->M; ++k)
          Q[(h->p0[b] + j) * h->M + k] = qt[h->qoff[b] + (k / QRR_NT) * QRR_NT * nb + (int64_t)j * QRR_NT + k % QRR_NT];
    }
  }
  if (R) {
    int64_t rtot = 0;
    for (int b = 0; b < h->G; ++b) rtot += (int64_t)h->nb[b] * h->nb[b];
    CK(cudaMemcpy(R, h->R, sizeof(double) * rtot, cudaMemcpyDeviceToHost));
  }
  API_END((int*)nullptr)
}

int glsgpu_factor_info(const glsgpu_sur* h, int* method, int* fallbacks) {
  if (!h) return GLSGPU_ERR_INVALID;
  if (method) *method = (h->cq && h->cq_last) ? 1 : 0;
  if (fallbacks) *fallbacks = h->cq_fallbacks;
  return GLSGPU_OK;
}

int glsgpu_launch_count(const glsgpu_sur* h, int64_t* count) {
  if (!h || !count) return GLSGPU_ERR_INVALID;
  *count = h->launches;
  return GLSGPU_OK;
}

int glsgpu_kernel_stats(const glsgpu_sur* h, glsgpu_kernel_stat* out, int cap) {
  if (!h) return 0;
  const int k = std::min<int>(cap, (int)h->kstats.size());
  for (int i = 0; i < k; ++i) out[i] = h->kstats[i];
  return k;
}

int glsgpu_sur_solve(glsgpu_sur* h, const glsgpu_pcg_config* cfg_in, const double* w1, const double* z1,
                     const double* beta_true, double* b_out, double* w_out, glsgpu_trace_row* rows,
                     int64_t rows_cap, glsgpu_result* res) {
  API_BEGIN
  if (!h || !b_out || !res) fail(GLSGPU_ERR_INVALID, "glsgpu_sur_solve: null argument");
  GroupGuard group_guard{h->grp};
  CK(cudaSetDevice(h->dev));
  glsgpu_pcg_config cfg;
  if (cfg_in) cfg = *cfg_in;
  else glsgpu_default_config(&cfg);
  const int64_t m = h->m_ref;  // rows of the reference's GLM (M G for SUR; G M0 + k for MVRGLM)
  const int64_t max_iter = cfg.max_iter ? cfg.max_iter : (m - h->n + 1);
  const int64_t cap_d = std::max<int64_t>(1, std::min<int64_t>(max_iter + 1, rows ? std::max<int64_t>(rows_cap, 1) : 1));
  require_factors(h);
  ensure_solver(h, cap_d);
  const int xv_mode = cfg.xv_mode == GLSGPU_XV_QR ? GLSGPU_XV_QR : GLSGPU_XV_X;
  const int diag = cfg.diag_every;
  h->kron_fma = cfg.kron_fma ? 1 : 0;
  Geo g = geo_of(h);
  cudaStream_t s = h->s;

  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, s));

  const double sigma_scale = norm_probe(h, 12);  // pcg.cpp:49

  SolveState hs;
  std::memset(&hs, 0, sizeof(hs));
  hs.tol_rel = cfg.tol_rel;
  hs.breakdown_tol = cfg.breakdown_tol;
  hs.growth_tol = cfg.growth_tol;
  hs.sigma_scale = sigma_scale;
  hs.i = 1;
  hs.max_iter = max_iter;
  hs.stride = cfg.record_z_every ? cfg.record_z_every : 1;
  hs.stagnation_window = cfg.stagnation_window;
  hs.growth_window = cfg.growth_window;
  hs.diag_every = diag;
  hs.rows_cap = cap_d;
  hs.breakdown_iter = -1;
  hs.active = 1;
  hs.term = T_MAXITER;
  hs.cur = 0;
  hs.best = 0;
  hs.nxt = 1;
  hs.mu_pending = 0;
  hs.have_beta = beta_true ? 1 : 0;
  // sw_mode 1: Sigma w formed where read (k_kron_mma path; diagnostics rows cost a Kronecker pass each, so
  // only with diag_every <= 0)
  h->sw_direct = (cfg.sw_mode == 1 && kron_mma_ok(h) && diag <= 0) ? 1 : 0;
  hs.sw_direct = h->sw_direct;
  // fused_c: needs Sigma w formed where read (the recurrence would need Sigma u_old in the element pass)
  h->fused = (cfg.fused_c == 1 && h->sw_direct && h->qmap_ok && std::getenv("GLSGPU_NO_FUSED") == nullptr) ? 1 : 0;
  // every row's diagnostics folded into passes B / C: narrow blocks, TMA passes, xv_mode QR, Sigma w by recurrence
  h->fold = (diag == 1 && xv_mode == GLSGPU_XV_QR && h->all_stream && h->nmax <= 32 && !h->sw_direct && !h->fused &&
             h->ldy >= h->ldm && (h->ldy % 2) == 0 && (reinterpret_cast<uintptr_t>(h->Y) % 16) == 0 &&
             std::getenv("GLSGPU_NO_FOLD") == nullptr) ? 1 : 0;
  CK(cudaMemcpyAsync(h->st, &hs, sizeof(hs), cudaMemcpyHostToDevice, s));
  k_set_t0<<<1, 1, 0, s>>>(h->st);
  if (!h->capturing) h->launches++;

  const size_t mvb = sizeof(double) * (size_t)(h->ldm * h->G);
  // w1 (pcg.cpp:55-66): enforce X'w1 = 0 by projecting along X*
  int w1_projected = 0;
  CK(cudaMemsetAsync(h->wb[0], 0, mvb, s));
  CK(cudaMemsetAsync(h->swb[0], 0, mvb, s));
  if (w1 && h->coll) fail(GLSGPU_ERR_UNSUPPORTED, "glsgpu: w1 on a row-sharded handle");
  if (w1) require_x(h, "w1");
  if (xv_mode == GLSGPU_XV_X) require_x(h, "xv_mode X");
  if (w1) {
    h2d_mvec(h, h->wb[0], w1);
    // X'w via the diagnostics pass with est = 0 (only its column part is used here)
    CK(cudaMemsetAsync(h->zvec, 0, sizeof(double) * h->n, s));
    pass_diag(h, h->zvec, h->st, 0);
    launch_reduce_t(h, h->xtw, nullptr, 0);
    std::vector<double> xtw((size_t)h->n), wv((size_t)m);
    CK(cudaMemcpyAsync(xtw.data(), h->xtw, sizeof(double) * h->n, cudaMemcpyDeviceToHost, s));
    if (h->frob_x < 0) {
      k_sumsq_cols<<<GRID_CAP, NT, 0, s>>>(h->X, h->ldx, h->M, h->n, h->partA);
      if (!h->capturing) h->launches++;
      k_sum1<<<1, NT, 0, s>>>(h->partA, GRID_CAP, h->scal + 8);
      if (!h->capturing) h->launches++;
      double ss = 0;
      CK(cudaMemcpyAsync(&ss, h->scal + 8, sizeof(double), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      h->frob_x = std::sqrt(ss);
    }
    CK(cudaStreamSynchronize(s));
    double feas = 0.0, wn = 0.0;
    for (double v : xtw) feas += v * v;
    feas = std::sqrt(feas);
    for (int64_t i = 0; i < m; ++i) wn += w1[i] * w1[i];
    wn = std::sqrt(wn);
    const double scale = h->frob_x * wn;
    if (feas > 1e-14 * scale && feas > 0.0) {
      // corr = X* xtw = Q R^-T xtw per block (xstar_impl); w -= corr
      CK(cudaMemcpyAsync(h->t, h->xtw, sizeof(double) * h->n, cudaMemcpyDeviceToDevice, s));
      k_vupdate<<<(h->G + 63) / 64, 64, 0, s>>>(g, h->R, h->t, nullptr, 1, 3, nullptr);
      if (!h->capturing) h->launches++;
      pass_xs(h, h->t, h->pr);
      k_axpy_sub<<<GRID_CAP, NT, 0, s>>>(h->wb[0], h->pr, h->ldm * h->G);
      if (!h->capturing) h->launches++;
      CKL("w1 projection");
      w1_projected = 1;
    }
  }
  if (z1) CK(cudaMemcpyAsync(h->zvec, z1, sizeof(double) * h->n, cudaMemcpyHostToDevice, s));
  else CK(cudaMemsetAsync(h->zvec, 0, sizeof(double) * h->n, s));
  if (beta_true) CK(cudaMemcpyAsync(h->beta_d, beta_true, sizeof(double) * h->n, cudaMemcpyHostToDevice, s));

  // sw = Sigma w (zero for w1 = 0: swb[0] was cleared above); r = (sw + X z) - y; pr = Pi r; c
  if (w1 && !kron_mma_apply(h, MV_W + 0, h->swb[0]))
    launch_kron(h, h->wb[0], nullptr, nullptr, nullptr, h->swb[0], h->partA, 0, nullptr, nullptr);
  {
    dim3 grid((unsigned)std::min<int64_t>((h->ldm + NT - 1) / NT, 64), (unsigned)h->G);
    if (z1) require_x(h, "z1");
    k_init_residual<<<grid, NT, 0, s>>>(g, z1 ? h->X : nullptr, h->ldx, h->zvec, h->swb[0], h->Y, h->ldy, h->r);
    if (!h->capturing) h->launches++;
    CKL("k_init_residual");
  }
  qt_apply(h, MODE_QT_R, nullptr, h->t, nullptr, 0);
  const int gC = pass_c(h, h->t, h->r, h->pr, h->partC, nullptr, 0);
  const auto pi0 = combine3(h, h->partC, gC);
  k_init_scalars<<<1, NT, 0, s>>>(pi0.first, pi0.second, h->st, h->rows_d);
  if (!h->capturing) h->launches++;
  CKL("k_init_scalars");
  // v = X*' r (X mode: R^-1 t; QR mode: s = t); u = pr
  k_vupdate<<<(h->G + 63) / 64, 64, 0, s>>>(g, h->R, h->t, h->vs, xv_mode == GLSGPU_XV_X ? 1 : 0, 1, nullptr);
  if (!h->capturing) h->launches++;
  CKL("k_vupdate init");
  CK(cudaMemcpyAsync(h->u, h->pr, mvb, cudaMemcpyDeviceToDevice, s));
  // row 0 diagnostics: est0 = recover(sw) (pcg.cpp:118-122)
  if (diag >= 0) diag_row(h, xv_mode, false, 0);

  // ---- the iteration loop: CUDA graphs of `chunk` iterations, device-side control
  int chunk = cfg.graph_chunk;
  if (chunk <= 0) {
    const double bytes_iter = 8.0 * (2.0 * (double)h->M * h->n + 14.0 * (double)h->M * h->G);
    const double t_iter_us = bytes_iter / 6.0e6 + 40.0;
    chunk = (int)std::clamp(2000.0 / t_iter_us, 2.0, 32.0);
  }
  const int timing = (cfg.kernel_timing && !h->grp) ? 1 : 0;
  // a local-group (test-only) handle runs the iterations eagerly: its exchange crosses streams, which a
  // captured graph cannot hold
  // diag_every = 0 (row 0 and the final row only): the captured iterations carry no diagnostics kernels -- nine
  // gated no-op launches per iteration, 8% of a config-1 iteration -- and the final row's run once after the loop
  const bool tail_diag = diag == 0 && !h->grp && !h->fold;
  const int gdiag = (diag >= 0 && !tail_diag) ? 1 : -1;
  const bool need_graph = !h->grp && (!h->graph || h->graph_chunk != chunk || h->graph_xmode != xv_mode ||
                          h->graph_diag != gdiag || h->graph_timing != timing ||
                          h->graph_fma != h->kron_fma || h->graph_sw != h->sw_direct || h->graph_fused != h->fused ||
                          h->graph_rows != h->rows_d || h->graph_fold != h->fold);
  if (need_graph) {
    if (h->graph) {
      CK(cudaGraphExecDestroy(h->graph));
      h->graph = nullptr;
    }
    for (auto e : h->tev) cudaEventDestroy(e);
    h->tev.clear();
    if (timing) {
      h->tev.resize((size_t)chunk * 6);
      for (auto& e : h->tev) CK(cudaEventCreate(&e));
    }
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    h->capturing = true;
    for (int k = 0; k < chunk; ++k) capture_iteration(h, xv_mode, gdiag, timing, k);
    h->capturing = false;
    CK(cudaStreamEndCapture(s, &graph));
    {
      size_t nn = 0;
      CK(cudaGraphGetNodes(graph, nullptr, &nn));
      std::vector<cudaGraphNode_t> nodes(nn);
      CK(cudaGraphGetNodes(graph, nodes.data(), &nn));
      int64_t kn = 0;
      for (auto nd : nodes) {
        cudaGraphNodeType ty;
        CK(cudaGraphNodeGetType(nd, &ty));
        if (ty == cudaGraphNodeTypeKernel) ++kn;
      }
      h->graph_kernels = kn;
    }
    CK(cudaGraphInstantiate(&h->graph, graph, 0));
    CK(cudaGraphDestroy(graph));
    h->graph_chunk = chunk;
    h->graph_xmode = xv_mode;
    h->graph_diag = gdiag;
    h->graph_timing = timing;
    h->graph_fma = h->kron_fma;
    h->graph_sw = h->sw_direct;
    h->graph_fused = h->fused;
    h->graph_rows = h->rows_d;
    h->graph_fold = h->fold;
  }
  std::vector<double> kt_ms(3, 0.0);
  std::vector<int64_t> kt_n(3, 0);
  int64_t prev_i = 1;
  for (;;) {
    CK(cudaMemcpyAsync(h->st_host, h->st, sizeof(SolveState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (!h->st_host->active) break;
    prev_i = h->st_host->i;
    if (h->grp) {
      for (int k = 0; k < chunk; ++k) capture_iteration(h, xv_mode, diag >= 0 ? 1 : -1, 0, k);
      continue;
    }
    CK(cudaGraphLaunch(h->graph, s));
    h->launches += h->graph_kernels;
    if (timing) {
      CK(cudaMemcpyAsync(h->st_host, h->st, sizeof(SolveState), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      // iterations that executed pass A: prev_i .. last (a pass-A breakdown adds done + 1)
      const SolveState& q = *h->st_host;
      const int64_t last = q.active ? q.i - 1 : (q.breakdown_iter == q.done + 1 ? q.done + 1 : q.done);
      const int64_t ran_a = std::max<int64_t>(0, last - prev_i + 1);
      const int64_t ran_bc = std::max<int64_t>(0, h->st_host->done - prev_i + 1);
      for (int64_t k = 0; k < std::min<int64_t>(ran_a, chunk); ++k) {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, h->tev[k * 6 + 0], h->tev[k * 6 + 1]));
        kt_ms[0] += ms;
        kt_n[0]++;
      }
      for (int64_t k = 0; k < std::min<int64_t>(ran_bc, chunk); ++k) {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, h->tev[k * 6 + 2], h->tev[k * 6 + 3]));
        kt_ms[1] += ms;
        CK(cudaEventElapsedTime(&ms, h->tev[k * 6 + 4], h->tev[k * 6 + 5]));
        kt_ms[2] += ms;
        kt_n[1]++;
        kt_n[2]++;
      }
    }
  }
  if (tail_diag) {
    // the final row's diagnostics (gated on st->diag_now, which k_scalar_c set on the terminating iteration; the
    // state is the one the in-graph kernels would have seen: the iterations captured after it did nothing)
    if (h->sw_direct && !kron_mma_apply(h, -2, nullptr))
      launch_kron(h, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 3, h->st, nullptr);
    diag_row(h, xv_mode, true, -1);
  }
  // a w / sw update still pending (the loop stopped in k_scalar_c) is materialized now
  k_apply_pending<<<GRID_CAP, NT, 0, s>>>(h->st, wbuf_of(h), h->u, h->su, h->ldm * h->G);
  k_finish_pending<<<1, 1, 0, s>>>(h->st);
  h->launches += 2;
  CKL("apply pending");
  CK(cudaMemcpyAsync(h->st_host, h->st, sizeof(SolveState), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  SolveState fin = *h->st_host;
  if (h->sw_direct) {  // Sigma w_sel for the recovery b = X*'(y - Sigma w_sel)
    const int sel = fin.term == T_CONVERGED ? fin.cur : fin.best;
    if (!kron_mma_apply(h, MV_W + sel, h->swb[sel]))
      launch_kron(h, h->wb[sel], nullptr, nullptr, nullptr, h->swb[sel], h->partA, 0, nullptr, nullptr);
  }

  // exit: b = X*'(y - sw_sel), sel = last if Converged else best (pcg.cpp:215-228)
  {
    pass_qt(h, MODE_QT_D, nullptr, h->st, 1, 0);
    reduce_t_global(h, h->t2, nullptr, 0);
    k_vupdate<<<(h->G + 63) / 64, 64, 0, s>>>(g, h->R, h->t2, nullptr, 1, 2, nullptr);
    if (!h->capturing) h->launches++;
    CKL("recover");
  }
  CK(cudaEventRecord(e1, s));
  CK(cudaMemcpyAsync(b_out, h->t2, sizeof(double) * h->n, cudaMemcpyDeviceToHost, s));
  const int wsel = fin.term == T_CONVERGED ? fin.cur : fin.best;
  if (w_out) d2h_mvec(h, w_out, h->wb[wsel]);
  const int64_t nrows = fin.done + 1;
  std::vector<TraceRowD> rd;
  if (rows && rows_cap > 0) {
    const int64_t k = std::min<int64_t>(std::min<int64_t>(nrows, rows_cap), cap_d);
    rd.resize((size_t)k);
    CK(cudaMemcpyAsync(rd.data(), h->rows_d, sizeof(TraceRowD) * k, cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  for (size_t i = 0; i < rd.size(); ++i) {
    rows[i].iter = rd[i].iter;
    rows[i].c = rd[i].c;
    rows[i].aug_residual_norm = rd[i].aug;
    rows[i].dual_feas_norm = rd[i].dual;
    rows[i].rmse = rd[i].rmse;
    rows[i].elapsed_ns = rd[i].elapsed_ns;
  }
  float solve_ms = 0;
  CK(cudaEventElapsedTime(&solve_ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);

  res->iterations = fin.done;
  res->termination = fin.term;
  res->w1_projected = w1_projected;
  res->breakdown_iteration = fin.term == T_BREAKDOWN ? fin.breakdown_iter : -1;
  res->residual_seminorm = fin.term == T_CONVERGED ? fin.c : fin.c_best;
  res->n_rows = nrows;
  res->sigma_scale = sigma_scale;
  res->solve_ms = solve_ms;

  // logical operator applies of run_aug (counters as the reference tallies them)
  {
    const uint64_t done = (uint64_t)fin.done;
    const bool c1zero = fin.c1 == 0.0;
    uint64_t pi = 1 + done;
    uint64_t xt = 1 /* v */ + 1 /* est0 */ + done /* est_i */ + 1 /* final recover */;
    // v updates happen after every iteration that passed all termination tests
    uint64_t cont = done;
    if (fin.term == T_CONVERGED || fin.term == T_STAGNATION ||
        (fin.term == T_BREAKDOWN && fin.breakdown_iter == fin.done))
      cont = done > 0 ? done - 1 : 0;
    if (c1zero) cont = 0;
    xt += cont;
    h->counters.pi_applies += pi;
    h->counters.xstar_t_applies += xt;
    h->counters.xstar_applies += (uint64_t)w1_projected;
    h->counters.apply_multiplies += pi * h->pi_cost + xt * h->xstar_t_cost + (uint64_t)w1_projected * h->xstar_cost;
  }
  h->kstats.clear();
  if (timing) {
    const double M = (double)h->M, G = (double)h->G, n = (double)h->n;
    // pass A: reads pr, u, su, w, sw; writes u, su, w, sw (the deferred update of pcg.cpp:151-152)
    // pass B: reads Q (+ X in xv_mode X), su, r; writes r.   pass C: reads Q, r; writes pr.
    // sw_mode 1: no sw / su(old) read, no sw write; fused_c: pass A is element-wise (reads u, pr, su, spr, w;
    // writes u, su, w) and pass C also writes Sigma pr
    const double bA = 8.0 * (h->fused ? 8.0 : h->sw_direct ? 6.0 : 9.0) * M * G;
    // fold (diag_every 1): B also reads sw and y, writes z; C also reads z, w, u
    const double bB = 8.0 * (M * n * (xv_mode == GLSGPU_XV_X ? 2.0 : 1.0) + (h->fold ? 6.0 : 3.0) * M * G);
    const double bC = 8.0 * (M * n + (h->fused ? 3.0 : h->fold ? 5.0 : 2.0) * M * G);
    const char* names[3] = {"passA_kron", h->fold ? "passB_update_qtr_diag" : "passB_update_qtr",
                            h->fold ? "passC_pi_diag" : "passC_pi"};
    const double bytes[3] = {bA, bB, bC};
    for (int k = 0; k < 3; ++k) {
      glsgpu_kernel_stat ks;
      std::memset(&ks, 0, sizeof(ks));
      std::snprintf(ks.name, sizeof(ks.name), "%s", names[k]);
      ks.launches = kt_n[k];
      ks.total_ms = kt_ms[k];
      ks.bytes_per_launch = bytes[k];
      h->kstats.push_back(ks);
    }
  }
  (void)prev_i;
  h->fused = 0;  // solve-scoped: probe-level applies after the solve take the plain passes
  group_guard.ok = true;
  API_END((int*)nullptr)
}

int glsgpu_synth_normal(double* dev, int64_t rows, int64_t cols, int64_t ld, int64_t row0, int64_t rows_total,
                        uint64_t seed, uint64_t stream, int device) {
  API_BEGIN
  if (!dev || ld < rows || row0 < 0 || row0 + rows > rows_total) fail(GLSGPU_ERR_INVALID, "synth_normal: bad shape");
  CK(cudaSetDevice(device));
  k_synth_normal<<<148 * 8, 256>>>(dev, rows, cols, ld, row0, rows_total, seed, stream);
  CKL("k_synth_normal");
  CK(cudaDeviceSynchronize());
  API_END((int*)nullptr)
}

int glsgpu_synth_response(int G, int64_t M, int64_t row0, int64_t M_total, const int64_t* n_i, const double* X_dev,
                          int64_t ldx, const double* beta, const double* omega_half, uint64_t seed, double* Y_dev,
                          int64_t ldy, int device) {
  API_BEGIN
  // Y = X beta + Z Omega^1/2, Z ~ N(0,1) from stream 3 of the M_total x G matrix (synth.py's recipe)
  glsgpu_sur* h = create_common(G, M, n_i, omega_half, nullptr, device);
  double *z = nullptr, *e = nullptr, *bd = nullptr;
  try {
    const size_t mv = (size_t)(h->ldm * G);
    z = dalloc<double>(mv);
    e = dalloc<double>(mv);
    h->partA = dalloc<double>(GRID_CAP * 3);
    CK(cudaMemsetAsync(z, 0, mv * sizeof(double), h->s));
    k_synth_normal<<<148 * 8, 256, 0, h->s>>>(z, M, G, h->ldm, row0, M_total, seed, 3);
    CKL("k_synth_normal");
    CK(cudaFuncSetAttribute(k_kron<8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * 32 * 8));
    CK(cudaFuncSetAttribute(k_kron<16, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 512 * 16 * 8));
    launch_kron(h, z, nullptr, nullptr, nullptr, e, h->partA, 0, nullptr, nullptr);
    CK(cudaMemcpy2DAsync(Y_dev, ldy * sizeof(double), e, h->ldm * sizeof(double), M * sizeof(double), G,
                         cudaMemcpyDeviceToDevice, h->s));
    bd = dalloc<double>(h->n);
    CK(cudaMemcpyAsync(bd, beta, sizeof(double) * h->n, cudaMemcpyHostToDevice, h->s));
    dim3 grid((unsigned)std::min<int64_t>((M + 255) / 256, 256), (unsigned)G);
    k_add_xbeta<<<grid, 256, 0, h->s>>>(G, M, h->d_nb, h->d_p0, X_dev, ldx, bd, Y_dev, ldy);
    CKL("k_add_xbeta");
    CK(cudaStreamSynchronize(h->s));
  } catch (...) {
    cudaFree(z);
    cudaFree(e);
    cudaFree(bd);
    destroy_impl(h);
    throw;
  }
  cudaFree(z);
  cudaFree(e);
  cudaFree(bd);
  destroy_impl(h);
  API_END((int*)nullptr)
}

int glsgpu_nccl_unique_id(void* id_out) {
  API_BEGIN
  if (!id_out) fail(GLSGPU_ERR_INVALID, "nccl_unique_id: null");
  ncclUniqueId id;
  nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(id_out, &id, sizeof(id));
  API_END((int*)nullptr)
}

int glsgpu_sur_create_sharded(int G, int64_t M_local, int64_t M_global, const int64_t* n_i, const double* X_dev,
                              int64_t ldx, const double* Y_dev, int64_t ldy, const double* omega,
                              const double* block_scale, int device, const void* nccl_id, int rank, int nranks,
                              glsgpu_sur** out, int* bad_block) {
  API_BEGIN
  if (!out || !X_dev || !Y_dev) fail(GLSGPU_ERR_INVALID, "glsgpu_sur_create_sharded: null argument");
  if (ldx < M_local || ldy < M_local) fail(GLSGPU_ERR_DIMENSION_MISMATCH, "glsgpu: leading dimension < M_local");
  *out = nullptr;
  glsgpu_sur* h = create_common(G, M_local, n_i, omega, block_scale, device, M_global, rank, nranks, nccl_id);
  try {
    h->X = X_dev;
    h->ldx = ldx;
    h->Y = Y_dev;
    h->ldy = ldy;
    alloc_common(h);
    run_qr(h);
  } catch (...) {
    destroy_impl(h);
    throw;
  }
  *out = h;
  API_END(bad_block)
}

int glsgpu_local_group_create(int nranks, int device, glsgpu_local_group** out) {
  API_BEGIN
  if (!out || nranks < 1) fail(GLSGPU_ERR_INVALID, "glsgpu_local_group_create: bad argument");
  *out = nullptr;
  CK(cudaSetDevice(device));
  glsgpu_local_group* g = new glsgpu_local_group();
  g->n = nranks;
  g->dev = device;
  g->ev_ready.assign((size_t)nranks, nullptr);
  g->ev_done.assign((size_t)nranks, nullptr);
  g->send.assign((size_t)nranks, nullptr);
  try {
    for (int r = 0; r < nranks; ++r) {
      CK(cudaEventCreateWithFlags(&g->ev_ready[(size_t)r], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&g->ev_done[(size_t)r], cudaEventDisableTiming));
    }
  } catch (...) {
    for (auto e : g->ev_ready)
      if (e) cudaEventDestroy(e);
    for (auto e : g->ev_done)
      if (e) cudaEventDestroy(e);
    delete g;
    throw;
  }
  *out = g;
  API_END((int*)nullptr)
}

int glsgpu_local_group_destroy(glsgpu_local_group* g) {
  if (!g) return GLSGPU_OK;
  cudaSetDevice(g->dev);
  for (auto e : g->ev_ready)
    if (e) cudaEventDestroy(e);
  for (auto e : g->ev_done)
    if (e) cudaEventDestroy(e);
  delete g;
  return GLSGPU_OK;
}

int glsgpu_sur_create_sharded_local(int G, int64_t M_local, int64_t M_global, const int64_t* n_i, const double* X_dev,
                                    int64_t ldx, const double* Y_dev, int64_t ldy, const double* omega,
                                    const double* block_scale, glsgpu_local_group* group, int rank, glsgpu_sur** out,
                                    int* bad_block) {
  API_BEGIN
  if (!out || !X_dev || !Y_dev || !group) fail(GLSGPU_ERR_INVALID, "glsgpu_sur_create_sharded_local: null argument");
  GroupGuard group_guard{group};
  if (ldx < M_local || ldy < M_local) fail(GLSGPU_ERR_DIMENSION_MISMATCH, "glsgpu: leading dimension < M_local");
  *out = nullptr;
  glsgpu_sur* h = create_common(G, M_local, n_i, omega, block_scale, group->dev, M_global, rank, group->n, nullptr,
                                nullptr, false, group);
  try {
    h->X = X_dev;
    h->ldx = ldx;
    h->Y = Y_dev;
    h->ldy = ldy;
    alloc_common(h);
    run_qr(h);
  } catch (...) {
    destroy_impl(h);
    throw;
  }
  *out = h;
  group_guard.ok = true;
  API_END(bad_block)
}

int glsgpu_sur_shard(const glsgpu_sur* h, int* rank, int* nranks, int64_t* M_global) {
  if (!h) return GLSGPU_ERR_INVALID;
  if (rank) *rank = h->rank;
  if (nranks) *nranks = h->nranks;
  if (M_global) *M_global = h->M_global;
  return GLSGPU_OK;
}

// ------------------------------------------------------------------------------------------ MVRGLM
// make_mvrglm + mvrglm_preconditioner (structured.cpp:63-74,365-414,468-477) on the device.  The embedded
// model (embed_mvrglm, structured.cpp:77-95) is laid out as G padded blocks of M = M0 + max k_b rows:
// block b = [Z0; C_b; 0] with C_b(q, restr_b[q]) = 1, its Y rows [Y_b; 0], and the Kronecker apply
// confined to the M0 observation rows (msig).  Host m-vectors keep the reference's order.
int glsgpu_mvrglm_create(int G, int64_t M0, int64_t N0, const double* Z0, const double* Y, const double* omega,
                         const int64_t* roff, const int64_t* ridx, const double* z_scale, const double* c_scale,
                         int device, glsgpu_sur** out, int* bad_block) {
  API_BEGIN
  if (!out || !Z0 || !Y || !omega || !roff) fail(GLSGPU_ERR_INVALID, "glsgpu_mvrglm_create: null argument");
  *out = nullptr;
  if (G < 1) fail(GLSGPU_ERR_DIMENSION_MISMATCH, "make_mvrglm: Omega0 must be G x G");
  if (N0 < 1 || M0 < N0) fail(GLSGPU_ERR_DIMENSION_MISMATCH, "make_mvrglm: Z0 must be tall");
  if (roff[0] != 0) fail(GLSGPU_ERR_DIMENSION_MISMATCH, "restrictions: need one list per equation");
  MvDesc d;
  d.M0 = M0;
  d.kb.resize(G);
  d.kofs.resize(G);
  int64_t kmax = 0;
  for (int i = 0; i < G; ++i) {  // check_restrictions (structured.cpp:13-24)
    if (roff[i + 1] < roff[i]) fail(GLSGPU_ERR_DIMENSION_MISMATCH, "restrictions: need one list per equation");
    for (int64_t q = roff[i]; q < roff[i + 1]; ++q) {
      if (!ridx || ridx[q] < 0 || ridx[q] >= N0) fail(GLSGPU_ERR_DIMENSION_MISMATCH, "restrictions: index out of range");
      if (q > roff[i] && ridx[q] <= ridx[q - 1])
        fail(GLSGPU_ERR_DIMENSION_MISMATCH, "restrictions: indices must be strictly increasing");
    }
    d.kb[i] = roff[i + 1] - roff[i];
    d.kofs[i] = roff[i];
    kmax = std::max(kmax, d.kb[i]);
  }
  d.ktot = roff[G];
  for (int i = 0; i < G; ++i)  // structured.cpp:372-374
    if ((z_scale && !(z_scale[i] > 0.0)) || (c_scale && !(c_scale[i] > 0.0)))
      fail(GLSGPU_ERR_SINGULAR_D, "mvrglm_preconditioner: scales must be positive", i);
  d.c_scale = c_scale;
  const int64_t Mp = M0 + kmax;
  std::vector<int64_t> n_i((size_t)G, N0);
  glsgpu_sur* h = create_common(G, Mp, n_i.data(), omega, z_scale, device, -1, 0, 1, nullptr, &d);
  try {
    const int64_t ld = h->ldm, n = h->n;
    h->X_own = dalloc<double>((size_t)(ld * n));
    h->Y_own = dalloc<double>((size_t)(ld * G));
    CK(cudaMemsetAsync(h->X_own, 0, sizeof(double) * ld * n, h->s));
    CK(cudaMemsetAsync(h->Y_own, 0, sizeof(double) * ld * G, h->s));
    // Z0 once, then device copies into every block's observation rows
    CK(cudaMemcpy2DAsync(h->X_own, ld * sizeof(double), Z0, M0 * sizeof(double), M0 * sizeof(double), N0,
                         cudaMemcpyHostToDevice, h->s));
    for (int b = 1; b < G; ++b)
      CK(cudaMemcpy2DAsync(h->X_own + (int64_t)b * N0 * ld, ld * sizeof(double), h->X_own, ld * sizeof(double),
                           M0 * sizeof(double), N0, cudaMemcpyDeviceToDevice, h->s));
    if (d.ktot > 0) {
      std::vector<int64_t> pos((size_t)d.ktot);
      for (int b = 0; b < G; ++b)
        for (int64_t q = 0; q < d.kb[b]; ++q)
          pos[(size_t)(roff[b] + q)] = ((int64_t)b * N0 + ridx[roff[b] + q]) * ld + M0 + q;
      int64_t* dpos = dalloc<int64_t>(pos.size());
      CK(cudaMemcpyAsync(dpos, pos.data(), sizeof(int64_t) * pos.size(), cudaMemcpyHostToDevice, h->s));
      k_set_ones<<<(unsigned)std::min<int64_t>((d.ktot + NT - 1) / NT, GRID_CAP), NT, 0, h->s>>>(h->X_own, dpos, d.ktot);
      h->launches++;
      CKL("k_set_ones");
      CK(cudaStreamSynchronize(h->s));
      CK(cudaFree(dpos));
    }
    CK(cudaMemcpy2DAsync(h->Y_own, ld * sizeof(double), Y, M0 * sizeof(double), M0 * sizeof(double), G,
                         cudaMemcpyHostToDevice, h->s));
    h->X = h->X_own;
    h->ldx = ld;
    h->Y = h->Y_own;
    h->ldy = ld;
    bool two = false;
    for (int b = 0; b < G; ++b) two = two || h->wts[b] != h->wtc[b];
    if (two) {
      h->Xqr = dalloc<double>((size_t)(ld * n));
      k_scale_rows<<<GRID_CAP, NT, 0, h->s>>>(h->Xqr, h->X_own, ld, n, N0, h->msig, h->d_wts, h->d_wtc);
      h->launches++;
      CKL("k_scale_rows");
    }
    alloc_common(h);
    run_qr(h);
  } catch (...) {
    destroy_impl(h);
    throw;
  }
  *out = h;
  API_END(bad_block)
}

// mv_reduce (structured.cpp:121-130): thin QR Z0 = Q0 R0 on the device (the TSQR tree), then Q0' Y.
int glsgpu_mv_reduce(int G, int64_t M0, int64_t N0, const double* Z0, const double* Y, double* R0, double* QtY,
                     int device) {
  API_BEGIN
  if (!Z0 || !Y || !R0 || !QtY) fail(GLSGPU_ERR_INVALID, "glsgpu_mv_reduce: null argument");
  if (G < 1 || N0 < 1 || M0 < N0) fail(GLSGPU_ERR_DIMENSION_MISMATCH, "qr: need rows >= cols >= 1");
  const int64_t nb = N0;
  const double one = 1.0;
  glsgpu_sur* h = create_common(1, M0, &nb, &one, nullptr, device, -1, 0, 1, nullptr, nullptr, /*qr_only=*/true);
  h->rank_msg = 1;
  try {
    const int64_t ld = h->ldm;
    h->X_own = dalloc<double>((size_t)(ld * N0));
    h->Y_own = dalloc<double>((size_t)ld);
    CK(cudaMemsetAsync(h->X_own, 0, sizeof(double) * ld * N0, h->s));
    CK(cudaMemsetAsync(h->Y_own, 0, sizeof(double) * ld, h->s));
    CK(cudaMemcpy2DAsync(h->X_own, ld * sizeof(double), Z0, M0 * sizeof(double), M0 * sizeof(double), N0,
                         cudaMemcpyHostToDevice, h->s));
    h->X = h->X_own;
    h->ldx = ld;
    h->Y = h->Y_own;
    h->ldy = ld;
    alloc_common(h);
    run_qr(h);
    ensure_solver(h, 1);
    for (int j = 0; j < G; ++j) {  // Q0' Y, one column per Q'-pass
      h2d_mvec(h, h->r, Y + (int64_t)j * M0);
      qt_apply(h, MODE_QT_R, nullptr, h->t, nullptr, 0);
      CK(cudaMemcpyAsync(QtY + (int64_t)j * N0, h->t, sizeof(double) * N0, cudaMemcpyDeviceToHost, h->s));
    }
    CK(cudaMemcpyAsync(R0, h->R, sizeof(double) * N0 * N0, cudaMemcpyDeviceToHost, h->s));
    CK(cudaStreamSynchronize(h->s));
  } catch (...) {
    destroy_impl(h);
    throw;
  }
  destroy_impl(h);
  API_END((int*)nullptr)
}

// Rows m (the reference's embedded GLM: M G for SUR, G M0 + k for MVRGLM) and parameters n of a handle.
int glsgpu_model_dims(const glsgpu_sur* h, int64_t* m, int64_t* n) {
  if (!h) return GLSGPU_ERR_INVALID;
  if (m) *m = h->m_ref;
  if (n) *n = h->n;
  return GLSGPU_OK;
}

// sur_reduce (structured.cpp:132-178, Remark 1 of the paper) on the device.  W = [X_1 ... X_G]; the numerical
// rank q counts the eigenvalues of W'W above max((rank_tol s_max)^2, 64 eps lambda_max); the basis of
// range(W) is W V_q Lambda_q^-1/2 re-orthonormalised by a Householder QR; every block and Y are rotated onto
// it.  The basis equals the reference's up to an orthogonal q x q factor (eigenvector signs / rotations inside
// clusters, QR signs), which the reduced model's GLS estimate and every Gram X_i'X_j, X_i'Y do not see.
int glsgpu_sur_reduce(int G, int64_t M, const int64_t* n_i, const double* X, const double* Y, double rank_tol,
                      int device, int64_t* q_out, double* X_red, double* Y_red, double* basis) {
  API_BEGIN
  if (!n_i || !X || !Y || !q_out || !X_red || !Y_red) fail(GLSGPU_ERR_INVALID, "glsgpu_sur_reduce: null argument");
  if (G < 1 || M < 1) fail(GLSGPU_ERR_DIMENSION_MISMATCH, "make_sur: need at least one block");
  int64_t n = 0;
  for (int b = 0; b < G; ++b) {
    if (n_i[b] < 1) fail(GLSGPU_ERR_DIMENSION_MISMATCH, "sur_reduce: empty block", b);
    n += n_i[b];
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    fail(GLSGPU_ERR_NO_DEVICE, "glsgpu: no CUDA device available (there is no CPU fallback)");
  }
  CK(cudaSetDevice(device));
  Dla& L = dla();
  cudaStream_t s = nullptr;
  cusolverDnHandle_t hs = nullptr;
  glsgpu_sur* qh = nullptr;  // the basis' TSQR (a one-block QR-only handle)
  std::vector<void*> bufs;
  auto alloc = [&](size_t count) {
    double* p = dalloc<double>(count);
    bufs.push_back(p);
    return p;
  };
  auto cleanup = [&]() {
    if (s) cudaStreamSynchronize(s);
    if (qh) destroy_impl(qh);
    qh = nullptr;
    for (void* p : bufs) cudaFree(p);
    if (hs) L.SolDestroy(hs);
    if (s) cudaStreamDestroy(s);
  };
  try {
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    blas_check(L.SolCreate(&hs), "cusolverDnCreate");
    blas_check(L.SolSetStream(hs, s), "cusolverDnSetStream");
    double* dX = alloc((size_t)(M * n));
    double* dY = alloc((size_t)(M * G));
    double* gram = alloc((size_t)(n * n));
    double* lam = alloc((size_t)n);
    int* info = reinterpret_cast<int*>(alloc(1));
    CK(cudaMemcpyAsync(dX, X, sizeof(double) * M * n, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dY, Y, sizeof(double) * M * G, cudaMemcpyHostToDevice, s));
    // W'W (lower triangle) on the DMMA GEMM, then its eigen-decomposition (sym_eig, linalg.cpp:376-400: ascending
    // eigenvalues).  The eigensolver is cuSOLVER's syevd: a dense symmetric n x n eigenproblem (tridiagonal
    // reduction + divide and conquer), O(n^3) once per model, off the iteration path; the reference's own tred2 /
    // tql2 is a different algorithm anyway, so the basis is pinned on what the reduction preserves
    dgemm_dev(s, n, n, M, dX, M, true, dX, M, false, gram, n, true, bufs);
    int lwork = 0;
    blas_check(L.SyevdBuf(hs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)n, gram, (int)n, lam, &lwork),
               "cusolverDnDsyevd_bufferSize");
    double* work = alloc((size_t)std::max(lwork, 1));
    blas_check(L.Syevd(hs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)n, gram, (int)n, lam, work, lwork, info),
               "cusolverDnDsyevd");
    std::vector<double> ev((size_t)n);
    int hinfo = 0;
    CK(cudaMemcpyAsync(ev.data(), lam, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hinfo != 0) fail(GLSGPU_ERR_CUDA, "sur_reduce: eigensolver did not converge (info " + std::to_string(hinfo) + ")");
    // numerical rank (structured.cpp:142-152)
    const double lam_max = std::max(ev[(size_t)n - 1], 0.0);
    const double smax = std::sqrt(lam_max);
    const double lam_floor = 64.0 * 2.220446049250313e-16 * lam_max;
    const double lam_cut = std::max(rank_tol * smax * (rank_tol * smax), lam_floor);
    int64_t q = 0;
    for (double l : ev)
      if (l > lam_cut) ++q;
    if (q >= M) {  // nothing to reduce: transform = I (structured.cpp:154-159)
      *q_out = M;
      std::memcpy(X_red, X, sizeof(double) * M * n);
      std::memcpy(Y_red, Y, sizeof(double) * M * G);
      if (basis) {
        std::memset(basis, 0, sizeof(double) * M * M);
        for (int64_t i = 0; i < M; ++i) basis[i + i * M] = 1.0;
      }
      cleanup();
      return GLSGPU_OK;
    }
    // V_q Lambda_q^-1/2, largest eigenvalue first (structured.cpp:161-169)
    std::vector<double> vh((size_t)(n * q));
    {
      std::vector<double> vfull((size_t)(n * n));
      CK(cudaMemcpyAsync(vfull.data(), gram, sizeof(double) * n * n, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      for (int64_t j = 0; j < q; ++j) {
        const int64_t idx = n - 1 - j;
        const double inv = 1.0 / std::sqrt(ev[(size_t)idx]);
        for (int64_t r = 0; r < n; ++r) vh[(size_t)(r + j * n)] = vfull[(size_t)(r + idx * n)] * inv;
      }
    }
    double* vq = alloc((size_t)(n * q));
    CK(cudaMemcpyAsync(vq, vh.data(), sizeof(double) * n * q, cudaMemcpyHostToDevice, s));
    double* B = alloc((size_t)(M * q));
    dgemm_dev(s, M, q, n, dX, M, false, vq, n, false, B, M, false, bufs);  // W V_q Lambda_q^-1/2
    // re-orthonormalise: basis = qr_thin(basis).q (structured.cpp:170): the library's TSQR as a one-block QR-only
    // handle (Householder leaves + tree, explicit Q); cuSOLVER geqrf / orgqr past the TSQR kernels' 512 columns
    double* Bq = B;
    if (q <= 512) {
      CK(cudaStreamSynchronize(s));
      const double one1 = 1.0;
      const int64_t nq[1] = {q};
      qh = create_common(1, M, nq, &one1, nullptr, device, -1, 0, 1, nullptr, nullptr, /*qr_only=*/true);
      qh->rank_msg = 1;  // qr_thin's wording of RankDeficient
      qh->no_qtile = true;
      qh->X = B;
      qh->ldx = M;
      qh->Y = dY;
      qh->ldy = M;
      alloc_common(qh);
      run_qr(qh);
      Bq = alloc((size_t)(M * q));
      CK(cudaMemcpy2DAsync(Bq, M * sizeof(double), qh->Q, qh->ldm * sizeof(double), M * sizeof(double), q,
                           cudaMemcpyDeviceToDevice, qh->s));
      CK(cudaStreamSynchronize(qh->s));
    } else {
      double* tau = alloc((size_t)q);
      int lw2 = 0, lw3 = 0;
      blas_check(L.GeqrfBuf(hs, (int)M, (int)q, B, (int)M, &lw2), "cusolverDnDgeqrf_bufferSize");
      blas_check(L.OrgqrBuf(hs, (int)M, (int)q, (int)q, B, (int)M, tau, &lw3), "cusolverDnDorgqr_bufferSize");
      double* w2 = alloc((size_t)std::max(std::max(lw2, lw3), 1));
      blas_check(L.Geqrf(hs, (int)M, (int)q, B, (int)M, tau, w2, std::max(lw2, lw3), info), "cusolverDnDgeqrf");
      blas_check(L.Orgqr(hs, (int)M, (int)q, (int)q, B, (int)M, tau, w2, std::max(lw2, lw3), info), "cusolverDnDorgqr");
    }
    // reduced blocks and responses: basis' X_i, basis' Y (structured.cpp:172-176)
    double* xr = alloc((size_t)(q * n));
    double* yr = alloc((size_t)(q * G));
    dgemm_dev(s, q, n, M, Bq, M, true, dX, M, false, xr, q, false, bufs);
    dgemm_dev(s, q, G, M, Bq, M, true, dY, M, false, yr, q, false, bufs);
    CK(cudaMemcpyAsync(X_red, xr, sizeof(double) * q * n, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(Y_red, yr, sizeof(double) * q * G, cudaMemcpyDeviceToHost, s));
    if (basis) CK(cudaMemcpyAsync(basis, Bq, sizeof(double) * M * q, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *q_out = q;
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
  API_END((int*)nullptr)
}

// pcg_normal_equations(embed_sur(sur), nullptr, cfg, true_beta) (pcg.cpp:364-511): CG on X' Sigma^-1 X b =
// X' Sigma^-1 y, the PCG-NE comparison solver of the harness (experiments.cpp:604-613,906-909).  The reference
// factors the dense m x m Sigma; Sigma^-1 = Omega^-1 (x) I_M is applied here as a Kronecker pass with Omega^-1
// (from cholesky(Omega), the reference's own pivot floor, so a singular Omega raises SingularCovariance as the
// dense factorisation does).  Per iteration: X p (k_xapply), Sigma^-1 (k_kron), X' (the column pass over X)
// on the device; the n-vector recurrences on the host.
int glsgpu_pcg_ne(glsgpu_sur* h, const glsgpu_pcg_config* cfg_in, const double* beta_true, double* b_out,
                  double* w_out, glsgpu_trace_row* rows, int64_t rows_cap, glsgpu_result* res) {
  API_BEGIN
  if (!h || !b_out || !res) fail(GLSGPU_ERR_INVALID, "glsgpu_pcg_ne: null argument");
  if (h->coll) fail(GLSGPU_ERR_UNSUPPORTED, "glsgpu_pcg_ne: row-sharded handles are not supported");
  require_x(h, "glsgpu_pcg_ne");
  if (h->mv && h->m_ref != (int64_t)h->G * h->M0)
    fail(GLSGPU_ERR_SINGULAR_COVARIANCE, "pcg_normal_equations: covariance is singular");
  CK(cudaSetDevice(h->dev));
  glsgpu_pcg_config cfg;
  if (cfg_in) cfg = *cfg_in;
  else glsgpu_default_config(&cfg);
  const int G = h->G;
  const int64_t n = h->n;
  // cholesky(Omega) (linalg.cpp:174-193): the factor of Sigma = Omega (x) I_M is L (x) I_M (pcg.cpp:369-373)
  if (!h->neLr) {
    std::vector<double> L((size_t)G * G, 0.0);
    double max_diag = 0.0;
    for (int i = 0; i < G; ++i) max_diag = std::max(max_diag, std::fabs(h->omega_h[(size_t)i * G + i]));
    const double floor_ = 64.0 * 2.220446049250313e-16 * max_diag;
    for (int j = 0; j < G; ++j) {
      double d = h->omega_h[(size_t)j * G + j];
      for (int k = 0; k < j; ++k) d -= L[j + (size_t)k * G] * L[j + (size_t)k * G];
      if (d <= floor_) fail(GLSGPU_ERR_SINGULAR_COVARIANCE, "pcg_normal_equations: covariance is singular");
      L[j + (size_t)j * G] = std::sqrt(d);
      for (int i = j + 1; i < G; ++i) {
        double v = h->omega_h[i + (size_t)j * G];
        for (int k = 0; k < j; ++k) v -= L[i + (size_t)k * G] * L[j + (size_t)k * G];
        L[i + (size_t)j * G] = v / L[j + (size_t)j * G];
      }
    }
    std::vector<double> Lr((size_t)G * G);
    for (int i = 0; i < G; ++i)
      for (int j = 0; j < G; ++j) Lr[(size_t)i * G + j] = L[i + (size_t)j * G];
    h->neLr = dalloc<double>((size_t)G * G);
    h->neLc = dalloc<double>((size_t)G * G);
    CK(cudaMemcpy(h->neLr, Lr.data(), sizeof(double) * G * G, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->neLc, L.data(), sizeof(double) * G * G, cudaMemcpyHostToDevice));
    std::vector<double> ones((size_t)G, 1.0);
    h->d_ones = dalloc<double>((size_t)G);
    CK(cudaMemcpy(h->d_ones, ones.data(), sizeof(double) * G, cudaMemcpyHostToDevice));
    h->nebuf = dalloc<double>((size_t)n * 7);
  }
  const int64_t max_iter = cfg.max_iter ? cfg.max_iter : 2 * n;
  const int64_t cap_d = std::max<int64_t>(1, std::min<int64_t>(max_iter + 1, rows ? std::max<int64_t>(rows_cap, 1) : 1));
  ensure_solver(h, cap_d);
  cudaStream_t s = h->s;
  Geo g = geo_of(h);
  double *x = h->nebuf, *f = x + n, *p = f + n, *gp = p + n, *xb = gp + n, *v = xb + n, *hv = v + n;
  const dim3 rgrid((unsigned)std::min<int64_t>((h->ldm + NT - 1) / NT, 64), (unsigned)G);
  // chol_solve tile: T rows x G columns of shared memory (<= 160 KB)
  const int cT = (int)std::max<int64_t>(32, std::min<int64_t>(128, (160 * 1024 / (8 * (int64_t)G)) / 32 * 32));
  const size_t csm = (size_t)cT * G * sizeof(double);
  CK(cudaFuncSetAttribute(k_chol_solve_kron, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm));
  const int cgrid = (int)std::min<int64_t>((h->M + cT - 1) / cT, 148 * 8);
  auto chol = [&](double* vec, const SolveState* gst) {
    k_chol_solve_kron<<<cgrid, cT, csm, s>>>(G, h->ldm, h->M, h->neLr, h->neLc, vec, gst);
    if (!h->capturing) h->launches++;
    CKL("k_chol_solve_kron");
  };
  // X' x over the user X (unit row weights), gated on st->active when gst is given
  auto xt = [&](const double* in, double* out, const SolveState* gst) {
    Geo gx = g;
    gx.wts = gx.wtc = h->d_ones;
    ColArgs a = base_args(h);
    a.A = h->X;
    a.lda = h->ldx;
    a.avalid = h->M;
    a.vin = in;
    a.gate = gst ? 1 : 0;
    if (h->n_narrow) {
      a.blocks = h->d_blk_narrow;
      k_colpass<MODE_QT_V, true><<<h->n_narrow * h->nch, NT, 0, s>>>(gx, a, gst);
      if (!h->capturing) h->launches++;
    }
    if (h->n_wide) {
      a.blocks = h->d_blk_wide;
      k_colpass<MODE_QT_V, false><<<h->n_wide * h->nch, NT, (size_t)h->CH * sizeof(double), s>>>(gx, a, gst);
      if (!h->capturing) h->launches++;
    }
    CKL("k_colpass X'");
    launch_reduce_t(h, out, gst, gst ? 1 : 0);
  };
  // gp = X' Sigma^-1 X v (pcg.cpp:378-380)
  auto apply_g = [&](const double* in, double* out, const SolveState* gst) {
    k_xapply<<<rgrid, NT, 0, s>>>(g, h->X, h->ldx, in, h->r, gst);
    if (!h->capturing) h->launches++;
    CKL("k_xapply");
    chol(h->r, gst);
    xt(h->r, out, gst);
  };
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, s));
  SolveState hs;
  std::memset(&hs, 0, sizeof(hs));
  hs.tol_rel = cfg.tol_rel;
  hs.breakdown_tol = cfg.breakdown_tol;
  hs.growth_tol = cfg.growth_tol;
  hs.max_iter = max_iter;
  hs.stride = cfg.record_z_every ? cfg.record_z_every : 1;
  hs.stagnation_window = cfg.stagnation_window;
  hs.growth_window = cfg.growth_window;
  hs.rows_cap = cap_d;
  hs.breakdown_iter = -1;
  hs.active = 1;
  hs.cont = 1;  // the norm probe runs while cont
  hs.term = T_MAXITER;
  hs.have_beta = beta_true ? 1 : 0;
  CK(cudaMemcpyAsync(h->st, &hs, sizeof(hs), cudaMemcpyHostToDevice, s));
  k_set_t0<<<1, 1, 0, s>>>(h->st);
  h->launches++;
  if (beta_true) CK(cudaMemcpyAsync(h->beta_d, beta_true, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  // crude norm probe for the breakdown scale (pcg.cpp:381-392): v = 1/sqrt(n)
  k_fill<<<(unsigned)std::min<int64_t>((n + NT - 1) / NT, 148), NT, 0, s>>>(v, 1.0 / std::sqrt((double)n), n);
  h->launches++;
  for (int it = 0; it < 12; ++it) {
    apply_g(v, gp, nullptr);
    k_ne_probe<<<1, NE_NT, 0, s>>>(h->st, gp, v, n);
    h->launches++;
    CKL("k_ne_probe");
  }
  // h = X' Sigma^-1 y; x = 0, f = -h, p = f, c, row 0 (pcg.cpp:396-421)
  CK(cudaMemsetAsync(h->r, 0, sizeof(double) * h->ldm * G, s));
  k_ysub<<<rgrid, NT, 0, s>>>(g, h->Y, h->ldy, h->r);
  h->launches++;
  chol(h->r, nullptr);
  xt(h->r, hv, nullptr);
  const double* bt = beta_true ? h->beta_d : nullptr;
  k_ne_init<<<1, NE_NT, 0, s>>>(h->st, hv, x, f, p, xb, bt, h->rows_d, n);
  h->launches++;
  CKL("k_ne_init");
  // the iteration: CUDA graphs of `chunk` steps, device-side control
  int chunk = cfg.graph_chunk > 0 ? cfg.graph_chunk : 16;
  if (!h->ne_graph || h->ne_chunk != chunk || h->ne_rows != h->rows_d) {
    if (h->ne_graph) CK(cudaGraphExecDestroy(h->ne_graph));
    h->ne_graph = nullptr;
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    h->capturing = true;
    for (int k = 0; k < chunk; ++k) {
      apply_g(p, gp, h->st);
      k_ne_step<<<1, NE_NT, 0, s>>>(h->st, gp, x, f, p, xb, h->beta_d, h->rows_d, n);
      CKL("k_ne_step");
    }
    h->capturing = false;
    CK(cudaStreamEndCapture(s, &graph));
    size_t nn = 0;
    CK(cudaGraphGetNodes(graph, nullptr, &nn));
    CK(cudaGraphInstantiate(&h->ne_graph, graph, 0));
    CK(cudaGraphDestroy(graph));
    h->ne_chunk = chunk;
    h->ne_rows = h->rows_d;
  }
  // have_beta gates the rmse: the captured step reads beta through h->beta_d only when st->have_beta
  for (;;) {
    CK(cudaMemcpyAsync(h->st_host, h->st, sizeof(SolveState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (!h->st_host->active) break;
    CK(cudaGraphLaunch(h->ne_graph, s));
    h->launches += (int64_t)chunk * (4 + (h->n_narrow ? 1 : 0) + (h->n_wide ? 1 : 0));
  }
  SolveState fin = *h->st_host;
  const bool keep_last = fin.term == T_CONVERGED;
  const double* bsel = keep_last ? x : xb;
  CK(cudaMemcpyAsync(b_out, bsel, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  if (w_out) {  // implied_w(b) = chol_solve(lower, y - X b) (pcg.cpp:414-416,503)
    k_xapply<<<rgrid, NT, 0, s>>>(g, h->X, h->ldx, bsel, h->r);
    k_ysub<<<rgrid, NT, 0, s>>>(g, h->Y, h->ldy, h->r);
    h->launches += 2;
    chol(h->r, nullptr);
    d2h_mvec(h, w_out, h->r);
  }
  const int64_t nrows = fin.done + 1;
  std::vector<TraceRowD> rd;
  if (rows && rows_cap > 0) {
    const int64_t k = std::min<int64_t>(std::min<int64_t>(nrows, rows_cap), cap_d);
    rd.resize((size_t)k);
    CK(cudaMemcpyAsync(rd.data(), h->rows_d, sizeof(TraceRowD) * k, cudaMemcpyDeviceToHost, s));
  }
  CK(cudaEventRecord(e1, s));
  CK(cudaStreamSynchronize(s));
  for (size_t i = 0; i < rd.size(); ++i) {
    rows[i].iter = rd[i].iter;
    rows[i].c = rd[i].c;
    rows[i].aug_residual_norm = rd[i].aug;
    rows[i].dual_feas_norm = rd[i].dual;
    rows[i].rmse = rd[i].rmse;
    rows[i].elapsed_ns = rd[i].elapsed_ns;
  }
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  res->iterations = fin.done;
  res->termination = fin.term;
  res->w1_projected = 0;
  res->breakdown_iteration = fin.term == T_BREAKDOWN ? fin.breakdown_iter : -1;
  res->residual_seminorm = keep_last ? fin.c : fin.c_best;
  res->n_rows = nrows;
  res->sigma_scale = fin.sigma_scale;
  res->solve_ms = ms;
  API_END((int*)nullptr)
}

}  // extern "C"
