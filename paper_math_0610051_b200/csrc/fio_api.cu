// fio_api.cu -- the C ABI (include/fio.h): plan construction (PAPER.md:981-1008,
// 1111-1250) and the apply orchestration.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <future>
#include <math.h>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "fio_comm.h"
#include "fio_internal.h"
#include "fio_kernels.h"

namespace fio {
const char* last_error_cstr();
}

using namespace fio;

namespace {

constexpr size_t kSmemBudgetDefault = 48 * 1024;  // per-CTA FFT pass target (FIO_FFT_SMEM_KB overrides)
constexpr size_t kSmemMax = 200 * 1024;     // opt-in maximum for one long sequence
constexpr int kCertSamples = 200;           // s of PAPER.md:1464-1477
constexpr double kEpsFloorC64 = 1e-6, kEpsFloorC128 = 1e-11;
constexpr double kGramEpsFloor = 1e-7;      // below: shifted CholeskyQR3 instead of the Gram eigen-decomposition

#define FIO_CUDA(expr)                                                                               \
  do {                                                                                               \
    cudaError_t e_ = (expr);                                                                         \
    if (e_ != cudaSuccess) {                                                                         \
      set_error(std::string("CUDA error at " #expr ": ") + cudaGetErrorString(e_));                  \
      return e_ == cudaErrorMemoryAllocation ? FIO_ENOMEM : FIO_ECUDA;                               \
    }                                                                                                \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  cudaError_t ensure(size_t b) {
    if (b <= bytes && p) return cudaSuccess;
    release();
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(b, 16));
    if (e == cudaSuccess) bytes = b;
    return e;
  }
  template <typename T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

// Selects `dev` for the lifetime of the guard and restores the caller's current device on every
// return path (the library never leaves the calling thread on another device).
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (dev >= 0 && dev != prev) err = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

#define FIO_GUARD(dev)                                                                      \
  DeviceGuard guard_(dev);                                                                  \
  if (guard_.err != cudaSuccess) {                                                          \
    set_error(std::string("cudaSetDevice: ") + cudaGetErrorString(guard_.err));            \
    return FIO_ECUDA;                                                                       \
  }

// [a, a + na) and [b, b + nb) overlap
static bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  const char* x = static_cast<const char*>(a);
  const char* y = static_cast<const char*>(b);
  return x < y + nb && y < x + na;
}

}  // namespace

// The separation of one wedge in compact form (plan save/load): skeleton columns C, Y = V S^{-1}
// (U = A(:, C) Y), skeleton rows R and Z = U_R^+ (beta = T = Z A(R, members)).
struct WedgeFactors {
  int l = 0, q = 0, r = 0;
  double err = 0;
  std::vector<int> C, R;
  std::vector<cplx> Y, Z;
};

struct fio_plan_s {
  int N = 0, W = 0, taps = 0, c64 = 0, device = 0, sms = 148;
  std::vector<WedgeFactors> factors;                 // per owned wedge, kept for fio_plan_save
  const std::vector<WedgeFactors>* load = nullptr;   // fio_plan_load: factors read from a file
  uint64_t input_hash = 0;                           // hash of the phase / amplitude arrays
  double eps = 0, es_beta = 0;
  int low_r2 = 0;  // reading R27: wedge members with |xi|^2 <= low_r2 are always skeleton columns
  fio_opts opts{};
  std::vector<WedgeGeom> geom;
  std::vector<int> owned;
  std::vector<WedgeDev> wd;
  std::vector<int> r_final;
  std::vector<double> sep_err;
  std::vector<void*> allocs;
  std::vector<void*> beta_ptrs;
  std::vector<InterpWedge> iw;
  OperatorDev op{};
  double2* a0 = nullptr;
  WedgeDev* d_wedges = nullptr;
  FftLen* d_ffts = nullptr;
  void* d_tw = nullptr;
  void** d_beta = nullptr;
  void *fhat = nullptr, *tmp = nullptr, *p1 = nullptr, *g = nullptr;
  std::vector<CUtensorMap> tmaps;  // per owned wedge: TMA map of its fine grids (K3 tiles)
  PFN_cuTensorMapEncodeTiled_v12000 encode_tmap = nullptr;  // driver entry point (null: no TMA tiles)
  FftJob *jobs_row = nullptr, *jobs_col = nullptr, *jobs_rowadj = nullptr;
  int njobs_rowadj = 0, smem_rowadj = 0;
  std::vector<void*> mask_ptrs;
  unsigned char** d_masks = nullptr;
  int njobs_row = 0, njobs_col = 0, smem_row = 0, smem_col = 0;
  int rows_per_cta_N = 1, cols_per_cta_N = 1, fft_N = 0;
  void *e2e_in = nullptr, *e2e_out = nullptr;
  // fio_apply_host_stream: double-buffered staging, its two copy streams and the pipeline's events
  void *hs_in[2] = {nullptr, nullptr}, *hs_out[2] = {nullptr, nullptr};
  cudaStream_t hs_h2d = nullptr, hs_d2h = nullptr;
  cudaEvent_t hs_fork = nullptr, hs_join = nullptr, hs_in_ready[2] = {}, hs_done[2] = {}, hs_out_free[2] = {};
  void* batch_ws = nullptr;  // (nrhs - 1) x (fhat + fine grids + K3 accumulator) for fio_apply_batch
  cudaStream_t side = nullptr;  // plan-owned side stream (skeleton-mode K3, adjoint spreads)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int batch_cap = 1;
  size_t alpha_bytes = 0, beta_bytes = 0, ws_bytes = 0, fine_elems = 0, p1_elems = 0, meta_bytes = 0;
  long long slots = 0;
  long long slot_terms = 0;  // sum over owned wedges of padded K3 slots x q_l
  long long max_tile_cap = 0;
  long long chunk_threads = 0;
  double balance = 1.0;  // predicted max/mean rank load of the wedge assignment
  std::vector<SkelWedge> skel;  // skeleton storage (opts.skeleton)
  size_t skel_bytes = 0, scratch_elems = 0;  // K3 thread slots (chunks x BLOCK): groups / this = thread fill
  double plan_seconds = 0, max_err = 0;
  EsPoly poly{};
  double poly_err = 0;
  int certified = 1;
  int launches = 0;
  void* comm = nullptr;        // NCCL communicator of the wedge-sharded apply (opts.nccl_id), or null
  void* part = nullptr;        // comm: the N x N partial(s) this rank reduce-scatters (part_cap RHS)
  int part_cap = 0;
  std::vector<cudaEvent_t> prof_ev;  // (kStages + 1) per recorded apply
  int prof_cap = 0, prof_n = 0;

  size_t elem_bytes() const { return c64 ? sizeof(float2) : sizeof(double2); }
  int out_rows() const { return comm && !opts.allgather ? N / opts.nranks : N; }  // rows fio_apply writes
  // A6: the sum over ranks of this rank's N x N partial into `out` -- its row slab (reduce-scatter),
  // or with opts.allgather the full N x N (reduce-scatter into this rank's rows of `out`, then an
  // in-place all-gather), both on stream s
  fio_status sum_ranks(const void* part_b, void* out, cudaStream_t s) const {
    const size_t slab = 2 * (size_t)(N / opts.nranks) * N;  // reals per rank
    if (!opts.allgather) return comm_reduce_scatter(comm, part_b, out, slab, c64, s);
    void* mine = static_cast<char*>(out) + (c64 ? sizeof(float) : sizeof(double)) * slab * (size_t)opts.rank;
    fio_status st = comm_reduce_scatter(comm, part_b, mine, slab, c64, s);
    return st != FIO_OK ? st : comm_all_gather(comm, out, opts.rank, slab, c64, s);
  }
  // comm: make room for nrhs N x N partials (synchronizes `s` before freeing a smaller buffer)
  cudaError_t ensure_part(int nrhs, cudaStream_t s) {
    if (nrhs <= part_cap) return cudaSuccess;
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return e;
    if (part) cudaFree(part);
    part = nullptr;
    part_cap = 0;
    e = cudaMalloc(&part, elem_bytes() * (size_t)N * N * nrhs);
    if (e == cudaSuccess) part_cap = nrhs;
    return e;
  }
  cudaError_t alloc(void** p, size_t bytes) {
    cudaError_t e = cudaMalloc(p, std::max<size_t>(bytes, 16));
    if (e == cudaSuccess) allocs.push_back(*p);
    return e;
  }
  template <typename T>
  cudaError_t upload(T** dst, const T* src, size_t n) {
    cudaError_t e = alloc(reinterpret_cast<void**>(dst), n * sizeof(T));
    if (e != cudaSuccess) return e;
    if (n) e = cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice);
    return e;
  }
  void free_events() {
    for (cudaEvent_t e : prof_ev) cudaEventDestroy(e);
    prof_ev.clear();
    prof_cap = prof_n = 0;
  }
  ~fio_plan_s() {
    free_events();
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (side) cudaStreamDestroy(side);
    for (cudaEvent_t e : {hs_fork, hs_join, hs_in_ready[0], hs_in_ready[1], hs_done[0], hs_done[1], hs_out_free[0],
                          hs_out_free[1]})
      if (e) cudaEventDestroy(e);
    if (hs_h2d) cudaStreamDestroy(hs_h2d);
    if (hs_d2h) cudaStreamDestroy(hs_d2h);
    if (batch_ws) cudaFree(batch_ws);
    if (part) cudaFree(part);
    comm_destroy(comm);
    for (void* p : allocs) cudaFree(p);
  }
};

extern "C" {

const char* fio_last_error(void) { return last_error_cstr(); }
const char* fio_version(void) { return "fio-b200 0.1 (sm_100a)"; }

void fio_default_opts(fio_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->dtype = FIO_C128;
  o->n_wedges = 0;
  o->nufft_w = 0;
  o->nufft_beta = 0.0;
  o->seed = 0x5EEDull;
  o->device = -1;
  o->rank = 0;
  o->nranks = 1;
  o->r_init = 32;
  o->r_max = 512;
  o->certify = 1;
}

fio_status fio_nccl_unique_id(void* id_out) {
  if (!id_out) {
    set_error("fio_nccl_unique_id: NULL argument");
    return FIO_EINVAL;
  }
  return comm_unique_id(id_out);
}

fio_status fio_geometry(int N, int W, int* wedge_of_out, int* M, int* xc, int* box) {
  if (N < 4 || N % 2 || W < 1) {
    set_error("fio_geometry: N must be even >= 4 and W >= 1");
    return FIO_EINVAL;
  }
  std::vector<WedgeGeom> g;
  build_geometry(N, W, g);
  if (wedge_of_out) {
    for (int k = 0; k < N * N; ++k) wedge_of_out[k] = -1;
    for (int l = 0; l < W; ++l)
      for (int k : g[l].members) wedge_of_out[k] = l;
  }
  for (int l = 0; l < W; ++l) {
    if (M) std::memcpy(M + 4 * l, g[l].M, 4 * sizeof(int));
    if (xc) { xc[2 * l] = g[l].xc1; xc[2 * l + 1] = g[l].xc2; }
    if (box) { box[4 * l] = g[l].n1; box[4 * l + 1] = g[l].n2; box[4 * l + 2] = g[l].n1f; box[4 * l + 3] = g[l].n2f; }
  }
  return FIO_OK;
}

fio_status fio_partition_weights(int W, double overlap, int xi1, int xi2, double* chi) {
  if (W < 1 || !chi || !(overlap >= 0.0 && overlap <= 1.0)) {
    set_error("fio_partition_weights: need W >= 1, overlap in [0, 1] and an output array");
    return FIO_EINVAL;
  }
  for (int l = 0; l < W; ++l) chi[l] = wedge_weight(W, overlap, l, xi1, xi2);
  return FIO_OK;
}

fio_status fio_assign_wedges(int W, const double* cost, int nranks, int* owner) {
  if (W < 1 || nranks < 1 || !cost || !owner) {
    set_error("fio_assign_wedges: bad arguments");
    return FIO_EINVAL;
  }
  lpt_assign(W, cost, nranks, owner);
  return FIO_OK;
}

}  // extern "C"

namespace {

// Randomized separation of the residual kernel of one wedge (PAPER.md:1111-1221,
// DESIGN.md reading R8: skeleton columns chosen by column pivoting on a random
// row sample, rows by pivoting on U; the paper's doubling of r and relative
// threshold eps are kept).  Produces U (m x q, device, FP64), beta (q x n,
// device, FP64), q, the final r and the sampled error.
// Rows sampled for the column pivoting of the separation, per skeleton column (reading R8): a wider row
// sample lets the pivoting see point classes a small sample misses.  FIO_SEP_ROWS overrides (experiments).
static int sep_row_oversample() {
  static const int v = [] {
    const char* e = std::getenv("FIO_SEP_ROWS");
    return e ? std::max(1, std::atoi(e)) : kSepRowOversample;
  }();
  return v;
}

fio_status separate_wedge(fio_plan_s& P, const WedgeGeom& g, Rng& rng, cudaStream_t s, DevBuf& dU, DevBuf& dBeta,
                          int& q_out, int& r_out, double& err_out, std::vector<int>& C_out,
                          std::vector<cplx>& Y_out, std::vector<int>& R_out, std::vector<cplx>& Z_out,
                          int r_start) {
  const int N = P.N;
  const int m = N * N;
  const int n = (int)g.members.size();
  const double eps = P.eps;
  DevBuf dMembers, dRows, dCols, dAC, dWork, dGram, dY, dAR, dZ, dTmp;
  FIO_CUDA(dMembers.ensure(sizeof(int) * n));
  FIO_CUDA(cudaMemcpy(dMembers.p, g.members.data(), sizeof(int) * n, cudaMemcpyHostToDevice));

  int r = std::min(std::max(r_start, 4), n);
  // reading R27: the members of the low-frequency disk |xi|^2 <= low_r2 (where the Bessel amplitude's
  // regularisation rho_e = max(rho, 1/2) makes the kernel non-smooth) are always skeleton columns and
  // always certified: a random column sample rarely contains these few frequencies
  std::vector<int> forced;  // member indices
  if (P.low_r2 > 0)
    for (int i = 0; i < n; ++i) {
      const int k = g.members[i], k1 = k / N, k2 = k - k1 * N;
      const long long x1 = k1 - (k1 >= N / 2 ? N : 0), x2 = k2 - (k2 >= N / 2 ? N : 0);
      if (x1 * x1 + x2 * x2 <= P.low_r2) forced.push_back(i);
    }
  std::vector<int> C;
  std::vector<cplx> V;
  std::vector<double> lam;
  int q = 0;
  for (;;) {
    // (1) random row sample R0, candidate columns, A(R0, cand) -> host
    std::vector<int> R0 = sample_distinct(rng, m, std::min(m, std::max(r, std::min(sep_row_oversample() * r, kSepRowCap))));
    std::vector<int> candIdx = sample_distinct(rng, n, std::min(n, 64 * r));
    std::vector<int> candCols(candIdx.size());
    for (size_t j = 0; j < candIdx.size(); ++j) candCols[j] = g.members[candIdx[j]];
    const int nr0 = (int)R0.size(), nc0 = (int)candCols.size();
    FIO_CUDA(dRows.ensure(sizeof(int) * nr0));
    FIO_CUDA(dCols.ensure(sizeof(int) * nc0));
    FIO_CUDA(cudaMemcpy(dRows.p, R0.data(), sizeof(int) * nr0, cudaMemcpyHostToDevice));
    FIO_CUDA(cudaMemcpy(dCols.p, candCols.data(), sizeof(int) * nc0, cudaMemcpyHostToDevice));
    FIO_CUDA(dTmp.ensure(sizeof(double2) * (size_t)nr0 * nc0));
    FIO_CUDA(launch_eval_entries(P.op, g.u1, g.u2, dRows.as<int>(), nr0, dCols.as<int>(), nc0, dTmp.as<double2>(), 1,
                                 nr0, s));
    std::vector<cplx> B((size_t)nr0 * nc0);
    FIO_CUDA(cudaMemcpyAsync(B.data(), dTmp.p, sizeof(cplx) * B.size(), cudaMemcpyDeviceToHost, s));
    FIO_CUDA(cudaStreamSynchronize(s));
    // (2) column pivoting -> skeleton columns C
    C.clear();
    if (P.opts.paper_accept) {  // the paper's step: r columns drawn uniformly
      for (int j = 0; j < std::min(r, nc0); ++j) C.push_back(candCols[j]);
    } else {
      std::vector<int> piv = pivoted_columns(nr0, nc0, B, r);
      for (int p : piv) C.push_back(candCols[p]);
    }
    for (int i : forced)
      if (std::find(C.begin(), C.end(), g.members[i]) == C.end()) C.push_back(g.members[i]);
    const int rc = (int)C.size();
    if (rc == 0) {
      q = 0;
      break;
    }
    // (3) A_C = A(all x, C) on the device, Gram = A_C^H A_C, eigen-decomposition
    FIO_CUDA(dCols.ensure(sizeof(int) * rc));
    FIO_CUDA(cudaMemcpy(dCols.p, C.data(), sizeof(int) * rc, cudaMemcpyHostToDevice));
    FIO_CUDA(dAC.ensure(sizeof(double2) * (size_t)m * rc));
    FIO_CUDA(launch_eval_entries(P.op, g.u1, g.u2, nullptr, m, dCols.as<int>(), rc, dAC.as<double2>(), 1, m, s));
    int nsplit = std::max(1, std::min(256, m / 8192));
    FIO_CUDA(dWork.ensure(sizeof(double2) * (size_t)nsplit * rc * rc));
    FIO_CUDA(dGram.ensure(sizeof(double2) * (size_t)rc * rc));
    auto gram = [&](const double2* A, std::vector<cplx>& G) -> fio_status {  // G = A^H A (m x rc)
      FIO_CUDA(launch_zgemm(rc, rc, m, A, m, 1, true, A, 1, m, dGram.as<double2>(), 1, rc, nsplit,
                            dWork.as<double2>(), s));
      G.resize((size_t)rc * rc);
      FIO_CUDA(cudaMemcpyAsync(G.data(), dGram.p, sizeof(cplx) * G.size(), cudaMemcpyDeviceToHost, s));
      FIO_CUDA(cudaStreamSynchronize(s));
      return FIO_OK;
    };
    std::vector<cplx> G;
    if (eps >= kGramEpsFloor) {
      // singular values of A_C from the eigen-decomposition of its Gram matrix: sigma_k / sigma_1
      // is resolved down to ~sqrt(machine eps), enough for eps >= kGramEpsFloor
      fio_status st = gram(dAC.as<double2>(), G);
      if (st != FIO_OK) return st;
      jacobi_svd(rc, rc, G, V, lam);  // G PSD: singular values = eigenvalues, V = eigenvectors
    } else {
      // high accuracy (eps below ~1e-7): shifted CholeskyQR3 of A_C = Q R (Q orthonormal to machine
      // precision even for numerically rank-deficient A_C), then the SVD of the small R, whose
      // singular values carry A_C's to ~1e-15 sigma_1 (a Gram eigen-decomposition would square the
      // condition number and lose everything below ~1e-8 sigma_1)
      FIO_CUDA(dY.ensure(sizeof(double2) * (size_t)rc * rc));
      DevBuf dQ[2];
      FIO_CUDA(dQ[0].ensure(sizeof(double2) * (size_t)m * rc));
      FIO_CUDA(dQ[1].ensure(sizeof(double2) * (size_t)m * rc));
      FIO_CUDA(cudaMemcpyAsync(dQ[0].p, dAC.p, sizeof(double2) * (size_t)m * rc, cudaMemcpyDeviceToDevice, s));
      std::vector<cplx> Rt((size_t)rc * rc, cplx{0, 0}), Rinv, tmp;
      for (int i = 0; i < rc; ++i) Rt[i + (size_t)i * rc] = {1.0, 0.0};
      int cur = 0;
      for (int pass = 0; pass < 3; ++pass) {
        fio_status st = gram(dQ[cur].as<double2>(), G);
        if (st != FIO_OK) return st;
        double shift = 0.0;
        if (pass == 0) {  // Fukaya et al.'s shift 11 (m n + n (n+1)) u ||A||_F^2
          double tr = 0;
          for (int i = 0; i < rc; ++i) tr += G[i + (size_t)i * rc].re;
          shift = 11.0 * ((double)m * rc + (double)rc * (rc + 1)) * 1.1102230246251565e-16 * tr;
        }
        std::vector<cplx> R = G;
        for (int i = 0; i < rc; ++i) R[i + (size_t)i * rc].re += shift;
        for (int tries = 0; !cholesky_upper(rc, R) && tries < 8; ++tries) {
          shift = shift > 0 ? 10.0 * shift : 1e-15 * G[0].re;
          R = G;
          for (int i = 0; i < rc; ++i) R[i + (size_t)i * rc].re += shift;
        }
        upper_inverse(rc, R, Rinv);
        FIO_CUDA(cudaMemcpy(dY.p, Rinv.data(), sizeof(cplx) * Rinv.size(), cudaMemcpyHostToDevice));
        FIO_CUDA(launch_zgemm(m, rc, rc, dQ[cur].as<double2>(), 1, m, false, dY.as<double2>(), 1, rc,
                              dQ[cur ^ 1].as<double2>(), 1, m, 1, nullptr, s));
        cur ^= 1;
        small_matmul(rc, R, Rt, tmp);  // R_total = R_pass R_total
        Rt.swap(tmp);
      }
      std::vector<double> sg;
      jacobi_svd(rc, rc, Rt, V, sg);  // R_total = U S V^H: A_C = (Q U) S V^H
      lam.resize(rc);
      for (int k = 0; k < rc; ++k) lam[k] = sg[k] * sg[k];
    }
    const double s1 = std::sqrt(std::max(lam[0], 0.0));
    q = 0;
    for (int k = 0; k < rc; ++k)
      if (std::sqrt(std::max(lam[k], 0.0)) > eps * s1) ++q;
    // accept when q is small against r, else double r and resample
    // paper_accept: uniform columns, accepted when q <= r/3; default: pivoted
    // columns, accepted when q <= 3r/4 or when the pivoting ran out of numerical rank (rc < r)
    const bool accepted = P.opts.paper_accept ? 3 * q <= rc : (4 * q <= 3 * rc || rc < r);
    if (accepted || r >= n || r >= P.opts.r_max) break;
    r = std::min(std::min(2 * r, n), P.opts.r_max);
  }
  r_out = r;
  q_out = q;
  if (q == 0) {
    err_out = 0.0;
    return FIO_OK;
  }
  const int rc = (int)C.size();
  // (4) U = A_C V_q S_q^{-1}
  std::vector<cplx> Y((size_t)rc * q);
  for (int t = 0; t < q; ++t) {
    double sg = std::sqrt(lam[t]);
    for (int i = 0; i < rc; ++i) Y[i + (size_t)t * rc] = {V[i + (size_t)t * rc].re / sg, V[i + (size_t)t * rc].im / sg};
  }
  FIO_CUDA(dY.ensure(sizeof(double2) * Y.size()));
  FIO_CUDA(cudaMemcpy(dY.p, Y.data(), sizeof(double2) * Y.size(), cudaMemcpyHostToDevice));
  FIO_CUDA(dU.ensure(sizeof(double2) * (size_t)m * q));
  FIO_CUDA(launch_zgemm(m, q, rc, dAC.as<double2>(), 1, m, false, dY.as<double2>(), 1, rc, dU.as<double2>(), 1, m, 1,
                        nullptr, s));
  dAC.release();
  C_out = C;  // skeleton storage keeps C and Y = V S^{-1}
  Y_out = Y;
  // (5) rows: pivoting on a random row sample of U, plus r uniform rows
  std::vector<int> R1 = sample_distinct(rng, m, std::min(m, 8 * r));
  const int n1r = (int)R1.size();
  FIO_CUDA(dRows.ensure(sizeof(int) * std::max(n1r, kCertSamples)));
  FIO_CUDA(cudaMemcpy(dRows.p, R1.data(), sizeof(int) * n1r, cudaMemcpyHostToDevice));
  FIO_CUDA(dTmp.ensure(sizeof(double2) * (size_t)std::max(n1r, kCertSamples) * q));
  FIO_CUDA(launch_gather_rows(dU.as<double2>(), m, q, dRows.as<int>(), n1r, dTmp.as<double2>(), s));
  std::vector<cplx> UR1((size_t)n1r * q);
  FIO_CUDA(cudaMemcpyAsync(UR1.data(), dTmp.p, sizeof(cplx) * UR1.size(), cudaMemcpyDeviceToHost, s));
  FIO_CUDA(cudaStreamSynchronize(s));
  std::vector<cplx> Bt((size_t)q * n1r);
  for (int i = 0; i < n1r; ++i)
    for (int t = 0; t < q; ++t) Bt[t + (size_t)i * q] = UR1[i + (size_t)t * n1r];
  std::vector<int> piv2 = pivoted_columns(q, n1r, Bt, q);
  std::vector<int> R;
  for (int p : piv2) R.push_back(R1[p]);
  for (int x : sample_distinct(rng, m, r)) R.push_back(x);
  std::sort(R.begin(), R.end());
  R.erase(std::unique(R.begin(), R.end()), R.end());
  const int nR = (int)R.size();
  // U_R and its pseudo-inverse (cutoff 1e-12 sigma_max, reading R8)
  std::vector<cplx> UR((size_t)nR * q);
  FIO_CUDA(dRows.ensure(sizeof(int) * std::max(nR, std::max(n1r, kCertSamples))));
  FIO_CUDA(cudaMemcpy(dRows.p, R.data(), sizeof(int) * nR, cudaMemcpyHostToDevice));
  FIO_CUDA(dTmp.ensure(sizeof(double2) * (size_t)std::max(nR, kCertSamples) * q));
  FIO_CUDA(launch_gather_rows(dU.as<double2>(), m, q, dRows.as<int>(), nR, dTmp.as<double2>(), s));
  FIO_CUDA(cudaMemcpyAsync(UR.data(), dTmp.p, sizeof(cplx) * UR.size(), cudaMemcpyDeviceToHost, s));
  FIO_CUDA(cudaStreamSynchronize(s));
  std::vector<cplx> Vr;
  std::vector<double> sr;
  jacobi_svd(nR, q, UR, Vr, sr);
  std::vector<cplx> Z((size_t)q * nR, cplx{0, 0});
  for (int k = 0; k < q; ++k) {
    if (!(sr[k] > 1e-12 * sr[0])) continue;
    const double inv2 = 1.0 / (sr[k] * sr[k]);
    for (int i = 0; i < nR; ++i) {
      cplx a = UR[i + (size_t)k * nR];  // = u_k sigma_k
      for (int t = 0; t < q; ++t) {
        cplx v = Vr[t + (size_t)k * q];
        // Z(t, i) += v_t conj(a_i) / sigma^2
        Z[t + (size_t)i * q].re += (v.re * a.re + v.im * a.im) * inv2;
        Z[t + (size_t)i * q].im += (v.im * a.re - v.re * a.im) * inv2;
      }
    }
  }
  // (6) beta = T = U_R^+ A_R
  FIO_CUDA(dAR.ensure(sizeof(double2) * (size_t)nR * n));
  FIO_CUDA(launch_eval_entries(P.op, g.u1, g.u2, dRows.as<int>(), nR, dMembers.as<int>(), n, dAR.as<double2>(), 1, nR,
                               s));
  R_out = R;
  Z_out = Z;
  FIO_CUDA(dZ.ensure(sizeof(double2) * Z.size()));
  FIO_CUDA(cudaMemcpy(dZ.p, Z.data(), sizeof(double2) * Z.size(), cudaMemcpyHostToDevice));
  FIO_CUDA(dBeta.ensure(sizeof(double2) * (size_t)q * n));
  FIO_CUDA(launch_zgemm(q, n, nR, dZ.as<double2>(), 1, q, false, dAR.as<double2>(), 1, nR, dBeta.as<double2>(), 1, q,
                        1, nullptr, s));
  dAR.release();
  // (7) certification: sampled relative Frobenius error on s x s entries
  err_out = 0.0;
  if (P.opts.certify) {
    std::vector<int> Gam = sample_distinct(rng, m, kCertSamples);
    std::vector<int> Del = sample_distinct(rng, n, kCertSamples);
    for (int i : forced)
      if (std::find(Del.begin(), Del.end(), i) == Del.end()) Del.push_back(i);
    const int ng = (int)Gam.size(), nd = (int)Del.size();
    std::vector<int> delCols(nd);
    for (int j = 0; j < nd; ++j) delCols[j] = g.members[Del[j]];
    FIO_CUDA(cudaMemcpy(dRows.p, Gam.data(), sizeof(int) * ng, cudaMemcpyHostToDevice));
    FIO_CUDA(dCols.ensure(sizeof(int) * nd));
    FIO_CUDA(cudaMemcpy(dCols.p, delCols.data(), sizeof(int) * nd, cudaMemcpyHostToDevice));
    DevBuf dA;
    FIO_CUDA(dA.ensure(sizeof(double2) * (size_t)ng * nd));
    FIO_CUDA(launch_eval_entries(P.op, g.u1, g.u2, dRows.as<int>(), ng, dCols.as<int>(), nd, dA.as<double2>(), 1, ng,
                                 s));
    std::vector<cplx> Aref((size_t)ng * nd), UG((size_t)ng * q), Bh((size_t)q * n);
    FIO_CUDA(cudaMemcpyAsync(Aref.data(), dA.p, sizeof(cplx) * Aref.size(), cudaMemcpyDeviceToHost, s));
    FIO_CUDA(launch_gather_rows(dU.as<double2>(), m, q, dRows.as<int>(), ng, dTmp.as<double2>(), s));
    FIO_CUDA(cudaMemcpyAsync(UG.data(), dTmp.p, sizeof(cplx) * UG.size(), cudaMemcpyDeviceToHost, s));
    FIO_CUDA(cudaMemcpyAsync(Bh.data(), dBeta.p, sizeof(cplx) * Bh.size(), cudaMemcpyDeviceToHost, s));
    FIO_CUDA(cudaStreamSynchronize(s));
    double num = 0, den = 0;
    for (int j = 0; j < nd; ++j)
      for (int i = 0; i < ng; ++i) {
        double ar = 0, ai = 0;
        for (int t = 0; t < q; ++t) {
          cplx u = UG[i + (size_t)t * ng], b = Bh[t + (size_t)Del[j] * q];
          ar += u.re * b.re - u.im * b.im;
          ai += u.re * b.im + u.im * b.re;
        }
        cplx e = Aref[i + (size_t)j * ng];
        num += (e.re - ar) * (e.re - ar) + (e.im - ai) * (e.im - ai);
        den += e.re * e.re + e.im * e.im;
      }
    err_out = den > 0 ? std::sqrt(num / den) : 0.0;
  }
  return FIO_OK;
}

// Cheap, rank-independent estimate of q_l for the wedge -> rank assignment: the number of
// column pivots of A(R, C) (64 random rows x <= 4096 random members) above eps x the largest.
// Its own RNG stream, so the separation's draws (and factors) do not depend on nranks.
fio_status estimate_rank(fio_plan_s& P, const WedgeGeom& g, cudaStream_t s, int& q_est) {
  const int m = P.N * P.N, n = (int)g.members.size();
  Rng rng(P.opts.seed ^ 0xA5A5A5A5DEADBEEFull ^ (0x9E3779B97F4A7C15ull * (uint64_t)(g.l + 7)));
  std::vector<int> R = sample_distinct(rng, m, 64);
  std::vector<int> ci = sample_distinct(rng, n, std::min(n, 4096));
  std::vector<int> C(ci.size());
  for (size_t j = 0; j < ci.size(); ++j) C[j] = g.members[ci[j]];
  const int nr = (int)R.size(), nc = (int)C.size();
  DevBuf dR, dC, dB;
  FIO_CUDA(dR.ensure(sizeof(int) * nr));
  FIO_CUDA(dC.ensure(sizeof(int) * nc));
  FIO_CUDA(dB.ensure(sizeof(double2) * (size_t)nr * nc));
  FIO_CUDA(cudaMemcpy(dR.p, R.data(), sizeof(int) * nr, cudaMemcpyHostToDevice));
  FIO_CUDA(cudaMemcpy(dC.p, C.data(), sizeof(int) * nc, cudaMemcpyHostToDevice));
  FIO_CUDA(launch_eval_entries(P.op, g.u1, g.u2, dR.as<int>(), nr, dC.as<int>(), nc, dB.as<double2>(), 1, nr, s));
  std::vector<cplx> B((size_t)nr * nc);
  FIO_CUDA(cudaMemcpyAsync(B.data(), dB.p, sizeof(cplx) * B.size(), cudaMemcpyDeviceToHost, s));
  FIO_CUDA(cudaStreamSynchronize(s));
  // modified Gram-Schmidt with pivoting over the nr sampled rows (vectors of length nc); the
  // eps-rank is the number of pivots whose residual norm exceeds eps x the largest row norm
  std::vector<cplx> Bt2((size_t)nc * nr);
  for (int j = 0; j < nc; ++j)
    for (int i = 0; i < nr; ++i) Bt2[j + (size_t)i * nc] = B[i + (size_t)j * nr];
  double mx = 0;
  for (int i = 0; i < nr; ++i) {
    double t = 0;
    for (int j = 0; j < nc; ++j) t += Bt2[j + (size_t)i * nc].re * Bt2[j + (size_t)i * nc].re + Bt2[j + (size_t)i * nc].im * Bt2[j + (size_t)i * nc].im;
    mx = std::max(mx, t);
  }
  q_est = 0;
  {
    std::vector<double> nr2(nr);
    std::vector<char> used(nr, 0);
    for (int i = 0; i < nr; ++i) {
      double t = 0;
      for (int j = 0; j < nc; ++j) t += Bt2[j + (size_t)i * nc].re * Bt2[j + (size_t)i * nc].re + Bt2[j + (size_t)i * nc].im * Bt2[j + (size_t)i * nc].im;
      nr2[i] = t;
    }
    for (int stp = 0; stp < nr; ++stp) {
      int p = -1;
      double best = -1;
      for (int i = 0; i < nr; ++i)
        if (!used[i] && nr2[i] > best) { best = nr2[i]; p = i; }
      if (p < 0 || best <= P.eps * P.eps * mx) break;
      used[p] = 1;
      ++q_est;
      const double inv = 1.0 / std::sqrt(best);
      cplx* qv = &Bt2[(size_t)p * nc];
      for (int j = 0; j < nc; ++j) { qv[j].re *= inv; qv[j].im *= inv; }
      for (int i = 0; i < nr; ++i) {
        if (used[i]) continue;
        cplx* b = &Bt2[(size_t)i * nc];
        double cr = 0, ci2 = 0;
        for (int j = 0; j < nc; ++j) {
          cr += qv[j].re * b[j].re + qv[j].im * b[j].im;
          ci2 += qv[j].re * b[j].im - qv[j].im * b[j].re;
        }
        double t = 0;
        for (int j = 0; j < nc; ++j) {
          b[j].re -= cr * qv[j].re - ci2 * qv[j].im;
          b[j].im -= cr * qv[j].im + ci2 * qv[j].re;
          t += b[j].re * b[j].re + b[j].im * b[j].im;
        }
        nr2[i] = t;
      }
    }
  }
  return FIO_OK;
}

int fft_index(std::map<int, int>& lens, std::vector<FftLen>& tab, int L) {
  auto it = lens.find(L);
  if (it != lens.end()) return it->second;
  FftLen f{};
  f.L = L;
  std::vector<int8_t> r = radix_plan(L);
  f.nst = (int)r.size();
  int ns = 1;
  for (int i = 0; i < f.nst; ++i) {
    f.radix[i] = r[i];
    f.div_nb[i] = make_fastdiv((uint32_t)(L / r[i]));
    f.div_ns[i] = make_fastdiv((uint32_t)ns);
    ns *= r[i];
  }
  int idx = (int)tab.size();
  tab.push_back(f);
  lens[L] = idx;
  return idx;
}

// K3 tables of one wedge (plan time, host only): group the points by supercell, cut the groups into
// chunks with bounded footprints and pad every chunk to BLOCK groups (see the K3 comment in
// fio_kernels.cu).  uh: fine coordinates (u1, u2) per x, consumed.
struct K3Tables {
  std::vector<int> anchor, slot_x, box;
  std::vector<double> off;   // c128 slot offsets
  std::vector<float> offf;   // c64 slot offsets
  long long cap = 0, real_groups = 0;
  int nchunks = 0;
};
// Bank-conflict-aware lane order inside one warp's share of a K3 chunk (blk lanes).  K3 reads every window row with 16-byte shared
// loads at (16-byte unit) offset u_g + const, u_g = ((a1 - r0) stride + (a2 - c0)) / epc for the group
// g a lane holds; a quarter-warp (8 lanes) takes one wavefront per distinct u among lanes with the
// same u mod 8 (equal u, i.e. the same anchor, is a broadcast).  Place the n groups on the blk lanes so
// that each quarter-warp holds at most one distinct u per residue where possible (greedy: largest
// same-anchor runs first, kept together); padding lanes repeat the anchor of a group of their
// quarter-warp.  lane_src[i] = group (0..n-1) on lane i, or -1 - g for a padding lane repeating group
// g's anchor.  Returns the extra wavefronts per window-row load summed over the quarter-warps.
// Pure reordering: every point's arithmetic is unchanged (K3 results are bit-identical).
static long long chunk_lane_order(const int* anc, int n, int blk, int r0, int c0, int stride, int epc,
                                  int* lane_src) {
  constexpr int kQ = 8;  // lanes per quarter-warp (16-byte loads)
  const int nq = blk / kQ;
  std::vector<long long> u(n);
  for (int g = 0; g < n; ++g) u[g] = ((long long)(anc[2 * g] - r0) * stride + (anc[2 * g + 1] - c0)) / epc;
  std::vector<std::pair<int, int>> runs;  // (first group, length) of equal-u runs, in group order
  for (int g = 0; g < n;) {
    int e = g + 1;
    while (e < n && u[e] == u[g]) ++e;
    runs.push_back({g, e - g});
    g = e;
  }
  std::stable_sort(runs.begin(), runs.end(), [](const auto& x, const auto& y) { return x.second > y.second; });
  std::vector<int> fill(nq, 0);
  std::vector<int> lanes((size_t)nq * kQ, 0);
  std::vector<std::vector<long long>> held((size_t)nq * kQ);  // per quarter-warp and residue: distinct u
  for (const auto& run : runs) {
    const long long ur = u[run.first];
    const int r = (int)(((ur % kQ) + kQ) % kQ);
    int left = run.second, g = run.first;
    while (left > 0) {
      auto holds = [&](int qw) {
        const auto& h = held[(size_t)qw * kQ + r];
        return std::find(h.begin(), h.end(), ur) != h.end();
      };
      int best = -1;
      for (int qw = 0; qw < nq && best < 0; ++qw)  // a quarter-warp already holding this u
        if (fill[qw] < kQ && holds(qw)) best = qw;
      for (int qw = 0; qw < nq && best < 0; ++qw)  // else one where the residue is free
        if (fill[qw] < kQ && held[(size_t)qw * kQ + r].empty()) best = qw;
      if (best < 0) {  // else the one with room whose residue holds the fewest (an unavoidable conflict)
        size_t fewest = SIZE_MAX;
        for (int qw = 0; qw < nq; ++qw)
          if (fill[qw] < kQ && held[(size_t)qw * kQ + r].size() < fewest) {
            fewest = held[(size_t)qw * kQ + r].size();
            best = qw;
          }
      }
      if (!holds(best)) held[(size_t)best * kQ + r].push_back(ur);
      const int take = std::min(left, kQ - fill[best]);
      for (int k = 0; k < take; ++k) lanes[(size_t)best * kQ + fill[best]++] = g++;
      left -= take;
    }
  }
  long long extra = 0;
  for (int qw = 0; qw < nq; ++qw) {
    size_t mx = 1;
    for (int r = 0; r < kQ; ++r) mx = std::max(mx, held[(size_t)qw * kQ + r].size());
    extra += (long long)mx - 1;
    const int rep = fill[qw] > 0 ? lanes[(size_t)qw * kQ] : 0;  // padding: a group of this quarter-warp
    for (int k = 0; k < kQ; ++k) lane_src[qw * kQ + k] = k < fill[qw] ? lanes[(size_t)qw * kQ + k] : -1 - rep;
  }
  return extra;
}

static K3Tables make_k3_tables(std::vector<double> uh, long long NN, int taps, bool c64, int n1f, int n2f) {
  K3Tables T;
#pragma omp parallel for schedule(static)
  for (long long x = 0; x < NN; ++x) std::swap(uh[2 * x], uh[2 * x + 1]);  // (K3 row, column) = (u2, u1)
  std::vector<int> anchor, slot_x;
  std::vector<double> off;
  group_points(uh.data(), NN, taps, group_p(c64, taps), n2f, n1f, super_rows(c64), super_cols(c64), anchor, slot_x, off);
  std::vector<double>().swap(uh);
  const int gp = group_p(c64, taps);
  T.real_groups = (long long)(anchor.size() / 2);
  const int blk = c64 ? kK3BlockC64 : kK3BlockC128;
  T.cap = chunk_boxes(anchor, blk, k3_window_rows(taps, c64), k3_window_cols(taps, c64),
                      c64 ? kK3TileCapC64 : kK3TileCapC128, T.box, c64 ? 8 : 16);
  T.nchunks = (int)(T.box.size() / 6);  // (chunk_boxes: 6 ints per chunk, widened to kBoxInts below)
  // pad every chunk to exactly blk groups, so that chunk c's groups are [c blk, (c+1) blk): K3 can then
  // prefetch a chunk's per-thread data without reading its box first.  Padding groups repeat the
  // anchor of a group of their quarter-warp (inside the box), have no points (slot -1) and alpha' = 0;
  // the groups' lane order and the tile's shared-memory row stride avoid bank conflicts
  // (chunk_lane_order).
  // Slots are stored in K3's physical layout (k3_slot: element-major inside each chunk), so that one
  // bulk copy moves a chunk's slot indices, offsets or alpha'(t) straight into its shared-memory image.
  T.anchor.assign((size_t)T.nchunks * blk * 2, 0);
  T.slot_x.assign((size_t)T.nchunks * blk * gp, -1);
  T.off.assign((size_t)T.nchunks * blk * gp * 2, 0.5 * taps);
  std::vector<int> box8((size_t)T.nchunks * kBoxInts, 0);  // per chunk: first group, r0, c0, rows, cols, groups,
                                                           // shared-memory row stride, 0
  std::vector<int> strides(T.nchunks), tmas(T.nchunks);
  const std::vector<int>& box = T.box;
#pragma omp parallel for schedule(static)
  for (int c = 0; c < T.nchunks; ++c) {
    const long long g0 = box[6 * c], n = box[6 * c + 5];
    // the tile's shared-memory row stride: the copied width or up to 7 (16-byte units) more, the one
    // whose best lane order leaves the fewest bank conflicts, inside the tile cap -- or, for a chunk
    // whose footprint fits the TMA box without wrapping, the box width (the TMA image is dense)
    const int epc = c64 ? 2 : 1, rows = box[6 * c + 3], cols = box[6 * c + 4];
    const int r0 = box[6 * c + 1], c0 = box[6 * c + 2];
    const int bxr = c64 ? kK3BoxRows64 : kK3BoxRows128, bxc = c64 ? kK3BoxCols64 : kK3BoxCols128;
    const bool tma = FIO_K3_TMA && rows <= bxr && cols <= bxc && r0 >= 0 && r0 + rows <= n2f && c0 + kHalo >= 0 &&
                     c0 + kHalo + bxc <= n1f + 2 * kHalo;
    tmas[c] = tma ? 1 : 0;
    const long long cap_c = c64 ? kK3TileCapC64 : kK3TileCapC128;
    std::vector<int> lane_src(blk), trial(blk);
    long long best = LLONG_MAX;
    int stride = cols;
    for (int st = tma ? bxc : cols; st <= (tma ? bxc : cols + 7 * epc); st += epc) {
      if (!tma && st > cols && (long long)rows * st > cap_c) break;
      // per warp: the lane order only permutes a warp's own groups, so every warp still covers the
      // same (serpentine-contiguous) groups -- the adjoint's spread keeps its atomics' locality
      long long ex = 0;
      for (int w0 = 0; w0 < blk; w0 += 32) {
        const int nw = (int)std::max<long long>(0, std::min<long long>(32, n - w0));
        if (nw == 0) {
          for (int i = 0; i < 32; ++i) trial[w0 + i] = -1;  // all padding: group 0's anchor
          continue;
        }
        ex += chunk_lane_order(&anchor[2 * (g0 + w0)], nw, 32, box[6 * c + 1], box[6 * c + 2], st, epc, &trial[w0]);
        for (int i = 0; i < 32; ++i) trial[w0 + i] += trial[w0 + i] >= 0 ? w0 : -w0;
      }
      if (ex < best) {
        best = ex;
        stride = st;
        lane_src.swap(trial);
        if (ex == 0) break;
      }
    }
    strides[c] = tma ? bxc : stride;
    for (long long i = 0; i < blk; ++i) {
      const bool real = lane_src[i] >= 0;
      const long long src = g0 + (real ? lane_src[i] : -1 - lane_src[i]), dst = (long long)c * blk + i;
      T.anchor[2 * dst] = anchor[2 * src];
      T.anchor[2 * dst + 1] = anchor[2 * src + 1];
      if (real)
        for (int k = 0; k < gp; ++k) {
          const long long ph = k3_slot(dst, k, gp, blk);
          T.slot_x[ph] = slot_x[src * gp + k];
          T.off[2 * ph] = off[2 * (src * gp + k)];
          T.off[2 * ph + 1] = off[2 * (src * gp + k) + 1];
        }
    }
    for (int e = 0; e < 6; ++e) box8[(size_t)kBoxInts * c + e] = box[6 * c + e];
    box8[(size_t)kBoxInts * c] = c * blk;
    box8[(size_t)kBoxInts * c + 6] = strides[c];
    box8[(size_t)kBoxInts * c + 7] = tmas[c];
  }
  T.box.swap(box8);
  for (int c = 0; c < T.nchunks; ++c)  // ring slot: the largest tile image (rows x stride, or the TMA box)
    T.cap = std::max(T.cap, tmas[c] ? (long long)(c64 ? kK3BoxRows64 * kK3BoxCols64 : kK3BoxRows128 * kK3BoxCols128)
                                    : (long long)T.box[(size_t)kBoxInts * c + 3] * strides[c]);
  T.cap = (T.cap + (c64 ? 15 : 7)) / (c64 ? 16 : 8) * (c64 ? 16 : 8);  // 128-byte slots (TMA destinations)
  if (c64) {
    T.offf.resize(T.off.size());
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < (long long)T.off.size(); ++i) T.offf[i] = (float)T.off[i];
    std::vector<double>().swap(T.off);
  }
  return T;
}

static WedgeDev geometry_wedgedev(const WedgeGeom& g) {
  WedgeDev w{};
  w.l = g.l;
  w.n1 = g.n1; w.n2 = g.n2; w.n1f = g.n1f; w.n2f = g.n2f;
  std::memcpy(w.M, g.M, sizeof(w.M));
  std::memcpy(w.Mi, g.Mi, sizeof(w.Mi));
  w.xc1 = g.xc1; w.xc2 = g.xc2;
  w.u1 = g.u1; w.u2 = g.u2;
  return w;
}

// A loaded wedge's factors must index inside this plan: skeleton columns C are members of the
// wedge (distinct), skeleton rows R are distinct output points in [0, N^2), and the factor shapes
// match q.  Anything else is a corrupted or foreign file (FIO_EINVAL, never an out-of-bounds read).
fio_status validate_factors(const WedgeFactors& F, const WedgeGeom& g, int N) {
  const long long m = (long long)N * N;
  const std::string w = " (wedge " + std::to_string(F.l) + ")";
  if (F.q < 0 || F.q > (int)F.C.size() || F.q > (int)F.R.size() || (F.q > 0 && F.C.empty())) {
    set_error("fio_plan_load: inconsistent rank q" + w);
    return FIO_EINVAL;
  }
  std::vector<int> mem(g.members);
  std::sort(mem.begin(), mem.end());
  std::vector<int> c(F.C);
  std::sort(c.begin(), c.end());
  if (std::adjacent_find(c.begin(), c.end()) != c.end()) {
    set_error("fio_plan_load: repeated skeleton column" + w);
    return FIO_EINVAL;
  }
  for (int k : c)
    if (!std::binary_search(mem.begin(), mem.end(), k)) {
      set_error("fio_plan_load: skeleton column outside the wedge" + w);
      return FIO_EINVAL;
    }
  std::vector<int> r(F.R);
  std::sort(r.begin(), r.end());
  if (std::adjacent_find(r.begin(), r.end()) != r.end() || (!r.empty() && (r.front() < 0 || r.back() >= m))) {
    set_error("fio_plan_load: skeleton rows out of range or repeated" + w);
    return FIO_EINVAL;
  }
  return FIO_OK;
}

// U = A(:, C) Y and beta = Z A(R, members) from saved factors: the same kernels and arguments as
// separate_wedge, so a loaded plan reproduces the saved one bit for bit.
fio_status expand_factors(fio_plan_s& P, const WedgeGeom& g, const WedgeFactors& F, cudaStream_t s, DevBuf& dU,
                          DevBuf& dBeta) {
  const int m = P.N * P.N;
  const int n = (int)g.members.size();
  const int q = F.q, rc = (int)F.C.size(), nR = (int)F.R.size();
  if (q == 0) return FIO_OK;
  if ((size_t)rc * q != F.Y.size() || (size_t)q * nR != F.Z.size()) {
    set_error("fio_plan_load: inconsistent factors for wedge " + std::to_string(F.l));
    return FIO_EINVAL;
  }
  DevBuf dMembers, dCols, dRows, dAC, dY, dAR, dZ;
  FIO_CUDA(dMembers.ensure(sizeof(int) * n));
  FIO_CUDA(cudaMemcpy(dMembers.p, g.members.data(), sizeof(int) * n, cudaMemcpyHostToDevice));
  FIO_CUDA(dCols.ensure(sizeof(int) * rc));
  FIO_CUDA(cudaMemcpy(dCols.p, F.C.data(), sizeof(int) * rc, cudaMemcpyHostToDevice));
  FIO_CUDA(dAC.ensure(sizeof(double2) * (size_t)m * rc));
  FIO_CUDA(launch_eval_entries(P.op, g.u1, g.u2, nullptr, m, dCols.as<int>(), rc, dAC.as<double2>(), 1, m, s));
  FIO_CUDA(dY.ensure(sizeof(double2) * F.Y.size()));
  FIO_CUDA(cudaMemcpy(dY.p, F.Y.data(), sizeof(double2) * F.Y.size(), cudaMemcpyHostToDevice));
  FIO_CUDA(dU.ensure(sizeof(double2) * (size_t)m * q));
  FIO_CUDA(launch_zgemm(m, q, rc, dAC.as<double2>(), 1, m, false, dY.as<double2>(), 1, rc, dU.as<double2>(), 1, m, 1,
                        nullptr, s));
  dAC.release();
  FIO_CUDA(dRows.ensure(sizeof(int) * nR));
  FIO_CUDA(cudaMemcpy(dRows.p, F.R.data(), sizeof(int) * nR, cudaMemcpyHostToDevice));
  FIO_CUDA(dAR.ensure(sizeof(double2) * (size_t)nR * n));
  FIO_CUDA(launch_eval_entries(P.op, g.u1, g.u2, dRows.as<int>(), nR, dMembers.as<int>(), n, dAR.as<double2>(), 1, nR,
                               s));
  FIO_CUDA(dZ.ensure(sizeof(double2) * F.Z.size()));
  FIO_CUDA(cudaMemcpy(dZ.p, F.Z.data(), sizeof(double2) * F.Z.size(), cudaMemcpyHostToDevice));
  FIO_CUDA(dBeta.ensure(sizeof(double2) * (size_t)q * n));
  FIO_CUDA(launch_zgemm(q, n, nR, dZ.as<double2>(), 1, q, false, dAR.as<double2>(), 1, nR, dBeta.as<double2>(), 1, q,
                        1, nullptr, s));
  return FIO_OK;
}

fio_status build_plan(fio_plan_s& P, const fio_phase* phase, const fio_amplitude* amp) {
  const int N = P.N;
  const long long NN = (long long)N * N;
  const bool c64 = P.c64;
  const size_t cs = c64 ? sizeof(float2) : sizeof(double2);
  cudaStream_t s = 0;
  // operator data on the device
  FIO_CUDA(P.upload(const_cast<double**>(&P.op.c1), phase->c1, NN));
  FIO_CUDA(P.upload(const_cast<double**>(&P.op.c2), phase->c2, NN));
  if (phase->b1) FIO_CUDA(P.upload(const_cast<double**>(&P.op.b1), phase->b1, NN));
  if (phase->b2) FIO_CUDA(P.upload(const_cast<double**>(&P.op.b2), phase->b2, NN));
  P.op.N = N;
  P.op.K = amp ? amp->K : 0;
  P.op.sign = phase->rho_sign < 0 ? -1 : 1;
  P.op.amp_kind = amp ? amp->kind : FIO_AMP_SEPARABLE;
  std::vector<double2> a0(NN);
  if (P.op.amp_kind == FIO_AMP_BESSEL_GRT) {
    // reading R27: the disk where rho_e = max(rho, 1/2) clamps, |xi| <= 1 / (2 min_x min(c1, c2)), plus one
    double cmin = 1e300;
    for (long long x = 0; x < NN; ++x) cmin = std::min(cmin, std::min(std::fabs(phase->c1[x]), std::fabs(phase->c2[x])));
    const int R = cmin > 1.0 / 30.0 ? (int)std::ceil(0.5 / cmin) + 1 : 16;
    P.low_r2 = std::min(R, 16) * std::min(R, 16);
  }
  if (P.op.amp_kind == FIO_AMP_BESSEL_GRT) {
    // a(x, 0) at rho_e = 1/2 (reading R22): (J0(pi) + s i Y0(pi)) e^{-s i pi} / (4 pi), x-independent
    const double PI = 3.14159265358979323846;
    const double J = ::j0(PI), Y = ::y0(PI), sg = P.op.sign;
    const double re = -J / (4.0 * PI), im = -sg * Y / (4.0 * PI);
    for (long long x = 0; x < NN; ++x) a0[x] = make_double2(re / N, im / N);
  } else if (P.op.K > 0) {
    const double2* px = reinterpret_cast<const double2*>(amp->px);
    const double2* pxi = reinterpret_cast<const double2*>(amp->pxi);
    FIO_CUDA(P.upload(const_cast<double2**>(&P.op.px), px, (size_t)P.op.K * NN));
    FIO_CUDA(P.upload(const_cast<double2**>(&P.op.pxi), pxi, (size_t)P.op.K * NN));
    for (long long x = 0; x < NN; ++x) {
      double re = 0, im = 0;
      for (int k = 0; k < P.op.K; ++k) {  // a(x, 0) = sum_k px_k(x) pxi_k(0)
        double2 u = px[k * NN + x], v = pxi[k * NN];
        re += u.x * v.x - u.y * v.y;
        im += u.x * v.y + u.y * v.x;
      }
      a0[x] = make_double2(re / N, im / N);
    }
  } else {
    for (long long x = 0; x < NN; ++x) a0[x] = make_double2(1.0 / N, 0.0);
  }
  FIO_CUDA(P.upload(&P.a0, a0.data(), NN));

  // geometry and ownership
  build_geometry(N, P.W, P.geom, P.opts.wedge_overlap);
  std::vector<int> owner(P.W, 0);
  if (P.opts.nranks > 1) {
    // per-wedge cost = q_l (estimated, identical on every rank) x (interpolation N^2 w^2 + FFT volume)
    std::vector<double> cost(P.W);
    for (int l = 0; l < P.W; ++l) {
      int qe = 1;
      if (!P.geom[l].members.empty()) {
        fio_status st = estimate_rank(P, P.geom[l], 0, qe);
        if (st != FIO_OK) return st;
      }
      cost[l] = (double)std::max(qe, 1) *
                ((double)NN * P.taps * P.taps +
                 8.0 * P.geom[l].n1f * P.geom[l].n2f * std::log2((double)P.geom[l].n1f * P.geom[l].n2f));
    }
    lpt_assign(P.W, cost.data(), P.opts.nranks, owner.data());
    std::vector<double> load(P.opts.nranks, 0.0);
    for (int l = 0; l < P.W; ++l) load[owner[l]] += cost[l];
    double mean = 0, mxl = 0;
    for (double v : load) { mean += v; mxl = std::max(mxl, v); }
    mean /= P.opts.nranks;
    P.balance = mean > 0 ? mxl / mean : 1.0;
  }
  for (int l = 0; l < P.W; ++l)
    if (owner[l] == P.opts.rank && !P.geom[l].members.empty()) P.owned.push_back(l);

  // FFT length table
  std::map<int, int> lens;
  std::vector<FftLen> ffts;
  P.fft_N = fft_index(lens, ffts, N);

  // per owned wedge: separation, folding of alpha' and beta'
  const bool prof = std::getenv("FIO_PLAN_PROFILE") != nullptr;  // per-phase plan timing to stderr
  double t_sep = 0, t_group = 0, t_fold = 0, t_gp = 0;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto secs = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
    return std::chrono::duration<double>(b - a).count();
  };
  // The host-side K3 grouping of wedge i+1.. runs on worker threads while wedge i is separated and
  // folded on the GPU (the grouping needs only the geometry and the fine coordinates).
  const size_t nown = P.owned.size();
  std::vector<std::future<K3Tables>> tables(nown);
  size_t next_prefetch = 0;
  auto prefetch = [&](size_t upto) -> fio_status {
    for (; next_prefetch < std::min(upto, nown); ++next_prefetch) {
      const WedgeGeom& gg = P.geom[P.owned[next_prefetch]];
      const WedgeDev wg = geometry_wedgedev(gg);
      DevBuf du;
      FIO_CUDA(du.ensure(sizeof(double2) * NN));
      FIO_CUDA(launch_fine_coords(P.op, wg, du.as<double2>(), s));
      std::vector<double> uh(2 * NN);
      FIO_CUDA(cudaMemcpyAsync(uh.data(), du.p, sizeof(double2) * NN, cudaMemcpyDeviceToHost, s));
      FIO_CUDA(cudaStreamSynchronize(s));
      tables[next_prefetch] = std::async(std::launch::async, make_k3_tables, std::move(uh), NN, P.taps, c64, gg.n1f,
                                         gg.n2f);
    }
    return FIO_OK;
  };
  constexpr size_t kLookahead = 3;
  for (size_t wi = 0; wi < P.owned.size(); ++wi) {
    const WedgeGeom& g = P.geom[P.owned[wi]];
    Rng rng(P.opts.seed ^ (0x9E3779B97F4A7C15ull * (uint64_t)(g.l + 1)));
    {
      fio_status pst = prefetch(wi + kLookahead);
      if (pst != FIO_OK) return pst;
    }
    auto tw0 = now();
    DevBuf dU, dBeta;
    int q = 0, r = 0;
    double err = 0;
    WedgeFactors F;
    fio_status st;
    if (P.load) {  // fio_plan_load: the saved separation of this wedge
      const WedgeFactors* src = nullptr;
      for (const WedgeFactors& f : *P.load)
        if (f.l == g.l) src = &f;
      if (!src) {
        set_error("fio_plan_load: the file has no factors for wedge " + std::to_string(g.l));
        return FIO_EINVAL;
      }
      F = *src;
      st = validate_factors(F, g, N);
      if (st == FIO_OK) st = expand_factors(P, g, F, s, dU, dBeta);
    } else {
      F.l = g.l;
      st = separate_wedge(P, g, rng, s, dU, dBeta, F.q, F.r, F.err, F.C, F.Y, F.R, F.Z, P.opts.r_init);
      // Certification-driven retry (reading R8): a random row sample can miss a rare kind
      // of output point (e.g. one region of a piecewise-smooth phase), so the skeleton -- and q --
      // miss a direction; the s = 200 sampled check sees it.  Redraw with a
      // doubled r (fresh draws from the wedge's stream) until certified or r_max.
      for (int r0 = 2 * P.opts.r_init; st == FIO_OK && P.opts.certify && F.err > 10.0 * P.eps && r0 <= P.opts.r_max;
           r0 *= 2) {
        WedgeFactors G2;
        G2.l = g.l;
        DevBuf dU2, dB2;
        st = separate_wedge(P, g, rng, s, dU2, dB2, G2.q, G2.r, G2.err, G2.C, G2.Y, G2.R, G2.Z, r0);
        if (st == FIO_OK && G2.err < F.err) {
          F = std::move(G2);
          std::swap(dU.p, dU2.p);
          std::swap(dU.bytes, dU2.bytes);
          std::swap(dBeta.p, dB2.p);
          std::swap(dBeta.bytes, dB2.bytes);
        }
      }
    }
    if (st != FIO_OK) return st;
    q = F.q;
    r = F.r;
    err = F.err;
    P.factors.push_back(std::move(F));
    if (prof) cudaDeviceSynchronize();
    auto tw1 = now();
    t_sep += secs(tw0, tw1);
    const std::vector<int>& Cs = P.factors.back().C;
    const std::vector<cplx>& Ys = P.factors.back().Y;
    WedgeDev w{};
    w.l = g.l;
    w.q = q;
    w.n1 = g.n1; w.n2 = g.n2; w.n1f = g.n1f; w.n2f = g.n2f;
    std::memcpy(w.M, g.M, sizeof(w.M));
    std::memcpy(w.Mi, g.Mi, sizeof(w.Mi));
    w.xc1 = g.xc1; w.xc2 = g.xc2;
    w.u1 = g.u1; w.u2 = g.u2;
    w.fft1 = fft_index(lens, ffts, g.n1f);
    w.fft2 = fft_index(lens, ffts, g.n2f);
    // K3 point groups (plan time): fine coordinates -> host grouping -> device tables
    InterpWedge iw{};
    iw.q = q;
    long long real_groups = 0;
    iw.nrow = g.n2f;                 // K3 rows = j2
    iw.ncol = g.n1f;                 // K3 columns = j1 (haloed)
    iw.ncolp = g.n1f + 2 * kHalo;
    {
      auto tg0 = now();
      K3Tables T;
      try {
        T = tables[wi].get();
      } catch (const std::exception& ex) {
        set_error(std::string("fio_plan: K3 grouping failed: ") + ex.what());
        return FIO_ENOMEM;
      }
      t_gp += secs(tg0, now());
      const int blk = c64 ? kK3BlockC64 : kK3BlockC128;
      real_groups = T.real_groups;
      iw.nchunks = T.nchunks;
      iw.ngroups = (int)(T.anchor.size() / 2);
      int* d_anchor = nullptr;
      int* d_slot = nullptr;
      FIO_CUDA(P.upload(&d_anchor, T.anchor.data(), T.anchor.size()));
      FIO_CUDA(P.upload(&d_slot, T.slot_x.data(), T.slot_x.size()));
      if (c64) {
        float* d_off = nullptr;
        FIO_CUDA(P.upload(&d_off, T.offf.data(), T.offf.size()));
        iw.slot_off = d_off;
      } else {
        double* d_off = nullptr;
        FIO_CUDA(P.upload(&d_off, T.off.data(), T.off.size()));
        iw.slot_off = d_off;
      }
      iw.anchor = d_anchor;
      iw.slot_x = d_slot;
      P.chunk_threads += (long long)iw.nchunks * blk;
      iw.tile_cap = (int)T.cap;
      int* d_box = nullptr;
      FIO_CUDA(P.upload(&d_box, T.box.data(), std::max<size_t>(T.box.size(), 4)));
      iw.box = d_box;
      P.max_tile_cap = std::max(P.max_tile_cap, T.cap);
      P.meta_bytes += T.anchor.size() * 4 + T.slot_x.size() * 4 + (c64 ? T.offf.size() * 4 : T.off.size() * 8);
    }
    auto tw2 = now();
    t_group += secs(tw1, tw2);
    const long long nslots = (long long)iw.ngroups * group_p(c64, P.taps);
    void* alpha = nullptr;
    void* betap = nullptr;
    SkelWedge sk{};
    if (P.opts.skeleton) {
      // alpha' is rebuilt before every K3 launch into one shared scratch (allocated below)
      if (q > 64) {
        set_error("fio_plan: skeleton storage supports separation ranks q <= 64 (wedge " + std::to_string(g.l) +
                  " has q = " + std::to_string(q) + ")");
        return FIO_EINVAL;
      }
      sk.rc = q > 0 ? (int)Cs.size() : 0;
      int* dC = nullptr;
      double2* dYs = nullptr;
      FIO_CUDA(P.upload(&dC, Cs.data(), std::max<size_t>(Cs.size(), 1)));
      FIO_CUDA(P.upload(&dYs, reinterpret_cast<const double2*>(Ys.data()), std::max<size_t>(Ys.size(), 1)));
      sk.C = dC;
      sk.Y = dYs;
      P.skel_bytes += Cs.size() * sizeof(int) + Ys.size() * sizeof(double2);
      P.scratch_elems = std::max<size_t>(P.scratch_elems, (size_t)q * (size_t)nslots);
    } else {
      FIO_CUDA(P.alloc(&alpha, cs * (size_t)q * nslots));
    }
    P.skel.push_back(sk);
    FIO_CUDA(P.alloc(&betap, cs * (size_t)q * g.n1 * g.n2));
    iw.alpha = alpha;
    if (q > 0) {
      if (!P.opts.skeleton) FIO_CUDA(launch_fold_alpha(P.op, w, dU.as<double2>(), q, iw.slot_x, nslots, alpha, c64, s));
      FIO_CUDA(cudaMemsetAsync(betap, 0, cs * (size_t)q * g.n1 * g.n2, s));
      std::vector<double> d1(g.n1), d2(g.n2);
      for (int i = 0; i < g.n1; ++i) d1[i] = 1.0 / es_fourier((double)(i - g.n1 / 2) / g.n1f, P.taps, P.es_beta);
      for (int i = 0; i < g.n2; ++i) d2[i] = 1.0 / es_fourier((double)(i - g.n2 / 2) / g.n2f, P.taps, P.es_beta);
      DevBuf dd1, dd2, dMem, dChi;
      FIO_CUDA(dd1.ensure(sizeof(double) * g.n1));
      FIO_CUDA(dd2.ensure(sizeof(double) * g.n2));
      FIO_CUDA(dMem.ensure(sizeof(int) * g.members.size()));
      FIO_CUDA(cudaMemcpy(dd1.p, d1.data(), sizeof(double) * g.n1, cudaMemcpyHostToDevice));
      FIO_CUDA(cudaMemcpy(dd2.p, d2.data(), sizeof(double) * g.n2, cudaMemcpyHostToDevice));
      FIO_CUDA(cudaMemcpy(dMem.p, g.members.data(), sizeof(int) * g.members.size(), cudaMemcpyHostToDevice));
      if (!g.chi.empty()) {  // smooth partition: chi_l folded into beta' with the deconvolution
        FIO_CUDA(dChi.ensure(sizeof(double) * g.chi.size()));
        FIO_CUDA(cudaMemcpy(dChi.p, g.chi.data(), sizeof(double) * g.chi.size(), cudaMemcpyHostToDevice));
      }
      FIO_CUDA(launch_fold_beta(N, w, dMem.as<int>(), (int)g.members.size(), dBeta.as<double2>(), q, dd1.as<double>(),
                                dd2.as<double>(), g.chi.empty() ? nullptr : dChi.as<double>(), betap, c64, s));
      FIO_CUDA(cudaStreamSynchronize(s));
    }
    if (prof) cudaDeviceSynchronize();
    t_fold += secs(tw2, now());
    if (!P.opts.skeleton) P.alpha_bytes += cs * (size_t)q * nslots;
    P.slots += real_groups * group_p(c64, P.taps);  // point slots before the chunk padding
    P.slot_terms += nslots * (long long)q;
    P.iw.push_back(iw);
    P.beta_bytes += cs * (size_t)q * g.n1 * g.n2;
    P.beta_ptrs.push_back(betap);
    {  // box mask of the wedge's members (adjoint K1* writes fhat* only there)
      std::vector<unsigned char> mask((size_t)g.n1 * g.n2, 0);
      for (int kf : g.members) {
        int k1 = kf / N, k2 = kf % N;
        int x1 = k1 >= N / 2 ? k1 - N : k1, x2 = k2 >= N / 2 ? k2 - N : k2;
        int i1 = g.M[0] * x1 + g.M[1] * x2 - g.xc1 + g.n1 / 2;
        int i2 = g.M[2] * x1 + g.M[3] * x2 - g.xc2 + g.n2 / 2;
        mask[(size_t)i1 * g.n2 + i2] = 1;
      }
      unsigned char* dm = nullptr;
      FIO_CUDA(P.upload(&dm, mask.data(), mask.size()));
      P.mask_ptrs.push_back(dm);
    }
    P.wd.push_back(w);
    P.r_final.push_back(r);
    P.sep_err.push_back(err);
    P.max_err = std::max(P.max_err, err);
    if (err > 10.0 * P.eps) P.certified = 0;  // reading R7: certify at the 10 eps apply budget
  }

  if (prof)
    std::fprintf(stderr,
                 "fio plan: separation %.2f s, K3 tables %.2f s (of which waiting for the grouping threads %.2f), "
                 "alpha'/beta' folding %.2f s (%zu wedges)\n",
                 t_sep, t_group, t_gp, t_fold, P.owned.size());
  if (P.opts.skeleton) {  // two alpha' scratches, alternating over the wedges (rebuilt per wedge per apply):
                          // wedge l's rebuild and K3 run on stream l mod 2, so they overlap the other's
    void* scratch[2] = {nullptr, nullptr};
    for (auto& sp : scratch) FIO_CUDA(P.alloc(&sp, cs * std::max<size_t>(P.scratch_elems, 1)));
    for (size_t wi = 0; wi < P.iw.size(); ++wi) P.iw[wi].alpha = scratch[wi & 1];
    P.alpha_bytes = 2 * cs * P.scratch_elems;
  }

  // twiddle tables
  std::vector<double2> twd;
  for (auto& f : ffts) {
    f.tw_off = (int)twd.size();
    for (int mm = 0; mm < f.L; ++mm) {
      const double ang = 6.283185307179586476925286766559 * (double)mm / (double)f.L;
      twd.push_back(make_double2(std::cos(ang), std::sin(ang)));
    }
    if (f.nst == 0 && f.L != 1) {
      set_error("internal: FFT length " + std::to_string(f.L) + " is not 5-smooth");
      return FIO_EINTERNAL;
    }
  }
  if (c64) {
    std::vector<float2> twf(twd.size());
    for (size_t i = 0; i < twd.size(); ++i) twf[i] = make_float2((float)twd[i].x, (float)twd[i].y);
    FIO_CUDA(P.upload(reinterpret_cast<float2**>(&P.d_tw), twf.data(), twf.size()));
  } else {
    FIO_CUDA(P.upload(reinterpret_cast<double2**>(&P.d_tw), twd.data(), twd.size()));
  }

  // workspace offsets and FFT job lists
  size_t kSmemBudget = kSmemBudgetDefault;
  if (const char* e = std::getenv("FIO_FFT_SMEM_KB")) kSmemBudget = (size_t)std::max(8, std::atoi(e)) * 1024;
  // K2 (column pass) budget: measured at N=1024, complex128 K2 48/64/80/96 KB = 1.49/1.36/1.59/1.53 ms,
  // complex64 0.45/0.49/0.60/0.59 ms
  size_t kSmemBudgetCol = std::getenv("FIO_FFT_SMEM_KB") ? kSmemBudget : (c64 ? 48 : 64) * 1024;
  if (const char* e = std::getenv("FIO_FFT_SMEM_KB_COL")) kSmemBudgetCol = (size_t)std::max(8, std::atoi(e)) * 1024;
  int max_rows = 32, max_cols = 16;
  if (const char* e = std::getenv("FIO_FFT_MAXSEQ")) max_rows = max_cols = std::min(32, std::max(1, std::atoi(e)));
  long long p1_off = 0, g_off = 0;
  std::vector<FftJob> jr, jc, jra;
  size_t smem_row = 0, smem_col = 0, smem_rowadj = 0;
  for (size_t wi = 0; wi < P.wd.size(); ++wi) {
    WedgeDev& w = P.wd[wi];
    w.p1_off = p1_off;
    w.g_off = g_off;
    P.iw[wi].g_off = g_off;
    p1_off += (long long)w.q * w.n1 * w.n2f;
    g_off += (long long)w.q * w.n2f * (w.n1f + 2 * kHalo);
    size_t sr = fft_seq_bytes(w.n2f, c64), sc = fft_seq_bytes(w.n1f, c64);
    int rows = (int)std::max<size_t>(1, std::min<size_t>(max_rows, kSmemBudget / sr));
    int cols = (int)std::max<size_t>(1, std::min<size_t>(max_cols, kSmemBudgetCol / sc));
    cols = std::min(cols, w.n2f);
    rows = std::min(rows, w.n1);
    for (int i = 0; i < w.n1; i += rows) {
      const int cnt = std::min(rows, w.n1 - i);
      jra.push_back({(int)wi, 0, i, cnt, w.fft2, {0, 0, 0}});
      smem_rowadj = std::max(smem_rowadj, sr * cnt + (size_t)cnt * w.n2 * (c64 ? sizeof(float2) : sizeof(double2)));
    }
    for (int t = 0; t < w.q; ++t) {
      for (int i = 0; i < w.n1; i += rows) {
        jr.push_back({(int)wi, t, i, std::min(rows, w.n1 - i), w.fft2, {0, 0, 0}});
        smem_row = std::max(smem_row, k1_row_bytes(w.n2f, c64) * std::min(rows, w.n1 - i));
      }
      for (int c = 0; c < w.n2f; c += cols) {
        jc.push_back({(int)wi, t, c, std::min(cols, w.n2f - c), w.fft1, {0, 0, 0}});
        smem_col = std::max(smem_col, sc * std::min(cols, w.n2f - c));
      }
    }
  }
  if (smem_row > kSmemMax || smem_col > kSmemMax || smem_rowadj > kSmemMax || fft_seq_bytes(N, c64) > kSmemMax) {
    set_error("fine grid too large for the shared-memory FFT (N too large for this dtype)");
    return FIO_EINVAL;
  }
  P.smem_row = (int)smem_row;
  P.smem_col = (int)smem_col;
  P.njobs_row = (int)jr.size();
  P.njobs_col = (int)jc.size();
  P.p1_elems = (size_t)p1_off;
  P.fine_elems = (size_t)g_off;
  P.rows_per_cta_N = (int)std::max<size_t>(1, kSmemBudget / fft_seq_bytes(N, c64));
  P.cols_per_cta_N = std::min(N, (int)std::max<size_t>(1, kSmemBudget / fft_seq_bytes(N, c64)));
  (void)kSmemBudgetDefault;
  FIO_CUDA(configure_kernels(kSmemMax));
  if (!P.iw.empty()) FIO_CUDA(configure_interp(P.taps, c64, P.max_tile_cap));
  if (P.opts.skeleton) {
    size_t rb = 0;
    for (size_t wi = 0; wi < P.skel.size(); ++wi) rb = std::max(rb, rebuild_smem_bytes(P.skel[wi].rc, P.wd[wi].q));
    FIO_CUDA(configure_rebuild(c64, rb));
  }
  FIO_CUDA(cudaDeviceGetAttribute(&P.sms, cudaDevAttrMultiProcessorCount, P.device));
  if (!jr.empty()) FIO_CUDA(P.upload(&P.jobs_row, jr.data(), jr.size()));
  if (!jc.empty()) FIO_CUDA(P.upload(&P.jobs_col, jc.data(), jc.size()));
  if (!jra.empty()) FIO_CUDA(P.upload(&P.jobs_rowadj, jra.data(), jra.size()));
  P.njobs_rowadj = (int)jra.size();
  P.smem_rowadj = (int)smem_rowadj;
  FIO_CUDA(P.upload(reinterpret_cast<void***>(&P.d_masks), P.mask_ptrs.data(), std::max<size_t>(P.mask_ptrs.size(), 1)));
  FIO_CUDA(P.upload(&P.d_ffts, ffts.data(), ffts.size()));
  FIO_CUDA(P.upload(&P.d_wedges, P.wd.data(), std::max<size_t>(P.wd.size(), 1)));
  FIO_CUDA(P.upload(&P.d_beta, P.beta_ptrs.data(), std::max<size_t>(P.beta_ptrs.size(), 1)));
  FIO_CUDA(P.alloc(&P.fhat, cs * NN));
  FIO_CUDA(P.alloc(&P.tmp, cs * NN));  // K0's scratch, then K3's second accumulator
  FIO_CUDA(cudaEventCreateWithFlags(&P.ev_fork, cudaEventDisableTiming));
  FIO_CUDA(cudaEventCreateWithFlags(&P.ev_join, cudaEventDisableTiming));
  FIO_CUDA(cudaStreamCreateWithFlags(&P.side, cudaStreamNonBlocking));
  FIO_CUDA(P.alloc(&P.p1, cs * std::max<size_t>(P.p1_elems, 1)));
  FIO_CUDA(P.alloc(&P.g, cs * std::max<size_t>(P.fine_elems, 1)));
  P.ws_bytes = cs * (2 * NN + P.p1_elems + P.fine_elems);
  // one TMA tensor map per owned wedge over its fine grids G_lt: 3-D [t][row][haloed column] in 8-byte
  // units (complex64: one element, complex128: two), box = the K3 TMA box (kK3BoxRows x kK3BoxCols)
  if (!P.encode_tmap) {  // the driver's encoder, through the runtime (no libcuda link dependency)
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult qr{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      P.encode_tmap = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    cudaGetLastError();
  }
  P.tmaps.assign(P.iw.size(), CUtensorMap{});
  for (size_t wi = 0; wi < P.iw.size(); ++wi) {
    InterpWedge& iw = P.iw[wi];
    iw.tma = 0;
    if (!FIO_K3_TMA || iw.q == 0 || !P.encode_tmap) continue;
    const cuuint64_t U = c64 ? 1 : 2;
    const cuuint64_t dims[3] = {U * (cuuint64_t)iw.ncolp, (cuuint64_t)iw.nrow, (cuuint64_t)iw.q};
    const cuuint64_t strides[2] = {(cuuint64_t)iw.ncolp * cs, (cuuint64_t)iw.nrow * iw.ncolp * cs};
    const cuuint32_t boxd[3] = {(cuuint32_t)(U * (c64 ? kK3BoxCols64 : kK3BoxCols128)),
                                (cuuint32_t)(c64 ? kK3BoxRows64 : kK3BoxRows128), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    void* base = static_cast<char*>(P.g) + (size_t)iw.g_off * cs;
    CUresult r = P.encode_tmap(&P.tmaps[wi], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, boxd, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    iw.tma = r == CUDA_SUCCESS ? 1 : 0;  // else this wedge keeps the cp.async tiles
  }
  FIO_CUDA(cudaDeviceSynchronize());
  return FIO_OK;
}

ApplyArgs make_args(const fio_plan_s& P) {
  ApplyArgs a{};
  a.N = P.N;
  a.nw = (int)P.wd.size();
  a.wedges = P.d_wedges;
  a.ffts = P.d_ffts;
  a.fft_N = P.fft_N;
  a.tw = P.d_tw;
  a.iw = P.iw.data();
  a.wd_host = P.wd.data();
  a.skel = P.opts.skeleton ? P.skel.data() : nullptr;
  a.beta = const_cast<const void* const*>(P.d_beta);
  a.op = P.op;
  a.a0 = P.a0;
  a.add_dc = P.opts.rank == 0 ? 1 : 0;
  a.taps = P.taps;
  a.es_beta = P.es_beta;
  a.poly = &P.poly;
  a.fhat = P.fhat;
  a.tmp = P.tmp;
  a.acc[0] = P.tmp;  // the second K3 accumulator is K0's scratch (free once K3 starts)
  a.side[0] = P.side;
  a.join[0] = P.ev_join;
  a.fork = P.ev_fork;
  a.tmaps = P.tmaps.empty() ? nullptr : P.tmaps.data();
  a.k3_rhs = std::getenv("FIO_K3_RHS") ? std::max(1, std::atoi(std::getenv("FIO_K3_RHS"))) : 2;
  a.p1 = P.p1;
  a.g = P.g;
  a.jobs_row = P.jobs_row;
  a.njobs_row = P.njobs_row;
  a.smem_row = P.smem_row;
  a.jobs_col = P.jobs_col;
  a.njobs_col = P.njobs_col;
  a.smem_col = P.smem_col;
  a.rows_per_cta_N = P.rows_per_cta_N;
  a.jobs_rowadj = P.jobs_rowadj;
  a.njobs_rowadj = P.njobs_rowadj;
  a.smem_rowadj = P.smem_rowadj;
  a.masks = const_cast<const unsigned char* const*>(P.d_masks);
  a.fine_elems = P.fine_elems;
  a.cols_per_cta_N = P.cols_per_cta_N;
  a.sms = P.sms;
  a.overlap = P.opts.wedge_overlap > 0.0 ? 1 : 0;
  return a;
}

}  // namespace

extern "C" {

// ------------------------------------------------------------------ plan save / load
struct SaveHeader {
  char magic[8];  // "FIOPLAN1"
  int32_t version, N, W, dtype, taps, rank, nranks, skeleton, n_owned;
  double eps, es_beta;
  uint64_t seed, input_hash;
  uint64_t body_hash;  // FNV-1a over every byte after the header (version 2)
};

// FNV-1a over the operator inputs the plan depends on (phase and amplitude arrays, kinds).
static uint64_t fnv1a(uint64_t h, const void* p, size_t n) {
  const unsigned char* b = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 1099511628211ull;
  }
  return h;
}
static uint64_t input_hash(int N, const fio_phase* phase, const fio_amplitude* amp) {
  const size_t NN = (size_t)N * N;
  uint64_t h = 1469598103934665603ull;
  h = fnv1a(h, phase->c1, sizeof(double) * NN);
  h = fnv1a(h, phase->c2, sizeof(double) * NN);
  const int flags[4] = {phase->b1 != nullptr, phase->b2 != nullptr, phase->rho_sign < 0 ? -1 : 1,
                        amp ? amp->kind : FIO_AMP_SEPARABLE};
  h = fnv1a(h, flags, sizeof(flags));
  if (phase->b1) h = fnv1a(h, phase->b1, sizeof(double) * NN);
  if (phase->b2) h = fnv1a(h, phase->b2, sizeof(double) * NN);
  if (amp && amp->K > 0) {
    h = fnv1a(h, &amp->K, sizeof(int));
    h = fnv1a(h, amp->px, 2 * sizeof(double) * NN * amp->K);
    h = fnv1a(h, amp->pxi, 2 * sizeof(double) * NN * amp->K);
  }
  return h;
}

static fio_status plan_impl(fio_handle* out, int N, const fio_phase* phase, const fio_amplitude* amp, double eps,
                            const fio_opts* opts, const std::vector<WedgeFactors>* load, const SaveHeader* hdr);

fio_status fio_plan(fio_handle* out, int N, const fio_phase* phase, const fio_amplitude* amp, double eps,
                    const fio_opts* opts) {
  return plan_impl(out, N, phase, amp, eps, opts, nullptr, nullptr);
}

fio_status fio_plan_save(fio_handle h, const char* path) {
  if (!h || !path) {
    set_error("fio_plan_save: NULL argument");
    return FIO_EINVAL;
  }
  FILE* fp = std::fopen(path, "wb");
  if (!fp) {
    set_error(std::string("fio_plan_save: cannot open ") + path);
    return FIO_EINVAL;
  }
  SaveHeader hd{};
  std::memcpy(hd.magic, "FIOPLAN1", 8);
  hd.version = 2;
  hd.N = h->N;
  hd.W = h->W;
  hd.dtype = h->opts.dtype;
  hd.taps = h->taps;
  hd.rank = h->opts.rank;
  hd.nranks = h->opts.nranks;
  hd.skeleton = h->opts.skeleton;
  hd.n_owned = (int)h->factors.size();
  hd.eps = h->eps;
  hd.es_beta = h->es_beta;
  hd.seed = h->opts.seed;
  hd.input_hash = h->input_hash;
  std::string body;  // serialized factors; hashed into the header, then written after it
  auto put = [&body](const void* p, size_t n) { body.append(static_cast<const char*>(p), n); };
  for (const WedgeFactors& F : h->factors) {
    const int32_t head[5] = {F.l, F.q, F.r, (int32_t)F.C.size(), (int32_t)F.R.size()};
    put(head, sizeof(head));
    put(&F.err, sizeof(double));
    put(F.C.data(), sizeof(int) * F.C.size());
    put(F.R.data(), sizeof(int) * F.R.size());
    put(F.Y.data(), sizeof(cplx) * F.Y.size());
    put(F.Z.data(), sizeof(cplx) * F.Z.size());
  }
  hd.body_hash = fnv1a(1469598103934665603ull, body.data(), body.size());
  bool ok = std::fwrite(&hd, sizeof(hd), 1, fp) == 1;
  ok = ok && std::fwrite(body.data(), 1, body.size(), fp) == body.size();
  ok = (std::fclose(fp) == 0) && ok;
  if (!ok) {
    set_error(std::string("fio_plan_save: write failed: ") + path);
    return FIO_EINVAL;
  }
  return FIO_OK;
}

fio_status fio_plan_load(fio_handle* out, const char* path, int N, const fio_phase* phase, const fio_amplitude* amp,
                         double eps, const fio_opts* opts) {
  if (!out || !path) {
    set_error("fio_plan_load: NULL argument");
    return FIO_EINVAL;
  }
  *out = nullptr;
  FILE* fp = std::fopen(path, "rb");
  if (!fp) {
    set_error(std::string("fio_plan_load: cannot open ") + path);
    return FIO_EINVAL;
  }
  SaveHeader hd{};
  bool ok = std::fread(&hd, sizeof(hd), 1, fp) == 1 && std::memcmp(hd.magic, "FIOPLAN1", 8) == 0 && hd.version == 2 &&
            hd.n_owned >= 0 && hd.n_owned <= 1 << 16;
  std::string body;  // the rest of the file, checked against the header's hash before it is parsed
  if (ok) {
    std::vector<char> buf(1 << 16);
    size_t got;
    while ((got = std::fread(buf.data(), 1, buf.size(), fp)) > 0) body.append(buf.data(), got);
    ok = fnv1a(1469598103934665603ull, body.data(), body.size()) == hd.body_hash;
  }
  std::fclose(fp);
  size_t pos = 0;
  auto take = [&](void* dst, size_t n) {
    if (pos + n > body.size()) return false;
    std::memcpy(dst, body.data() + pos, n);
    pos += n;
    return true;
  };
  std::vector<WedgeFactors> fs;
  std::vector<char> seen;
  for (int i = 0; ok && i < hd.n_owned; ++i) {
    WedgeFactors F;
    int32_t head[5];
    ok = take(head, sizeof(head)) && take(&F.err, sizeof(double));
    if (!ok) break;
    F.l = head[0];
    F.q = head[1];
    F.r = head[2];
    const long long nc = head[3], nr = head[4];
    ok = F.q >= 0 && nc >= 0 && nr >= 0 && nc <= (1 << 20) && nr <= (1 << 22) && F.q <= (1 << 16) && F.l >= 0 &&
         F.l < hd.W && F.l < (1 << 16);
    if (!ok) break;
    if ((int)seen.size() <= F.l) seen.resize(F.l + 1, 0);
    ok = !seen[F.l];  // each wedge at most once
    seen[F.l] = 1;
    if (!ok) break;
    F.C.resize(nc);
    F.R.resize(nr);
    F.Y.resize((size_t)nc * F.q);
    F.Z.resize((size_t)F.q * nr);
    ok = take(F.C.data(), sizeof(int) * F.C.size()) && take(F.R.data(), sizeof(int) * F.R.size()) &&
         take(F.Y.data(), sizeof(cplx) * F.Y.size()) && take(F.Z.data(), sizeof(cplx) * F.Z.size());
    fs.push_back(std::move(F));
  }
  ok = ok && pos == body.size();
  if (!ok) {
    set_error(std::string("fio_plan_load: not a valid plan file: ") + path);
    return FIO_EINVAL;
  }
  return plan_impl(out, N, phase, amp, eps, opts, &fs, &hd);
}

static fio_status plan_impl(fio_handle* out, int N, const fio_phase* phase, const fio_amplitude* amp, double eps,
                            const fio_opts* opts, const std::vector<WedgeFactors>* load, const SaveHeader* hdr) {
  if (!out) {
    set_error("fio_plan: out is NULL");
    return FIO_EINVAL;
  }
  *out = nullptr;
  if (N < 8 || N > 4096 || N % 2 != 0 || !is_smooth5(N)) {
    set_error("fio_plan: N must be even, 5-smooth and in [8, 4096] (got " + std::to_string(N) + ")");
    return FIO_EINVAL;
  }
  if (!(eps > 0.0 && eps < 1.0)) {
    set_error("fio_plan: eps must lie in (0, 1)");
    return FIO_EINVAL;
  }
  if (!phase || !phase->c1 || !phase->c2) {
    set_error("fio_plan: phase->c1 and phase->c2 are required");
    return FIO_EINVAL;
  }
  if (amp && amp->K < 0) {
    set_error("fio_plan: amplitude rank K must be >= 0");
    return FIO_EINVAL;
  }
  if (amp && amp->kind != FIO_AMP_SEPARABLE && amp->kind != FIO_AMP_BESSEL_GRT) {
    set_error("fio_plan: unknown amplitude kind");
    return FIO_EINVAL;
  }
  if (amp && amp->kind == FIO_AMP_BESSEL_GRT && amp->K != 0) {
    set_error("fio_plan: the Bessel amplitude takes K = 0");
    return FIO_EINVAL;
  }
  if (amp && amp->K > 0 && (!amp->px || !amp->pxi)) {
    set_error("fio_plan: amplitude K > 0 needs px and pxi");
    return FIO_EINVAL;
  }
  fio_opts o;
  fio_default_opts(&o);
  if (opts) o = *opts;
  if (o.dtype != FIO_C64 && o.dtype != FIO_C128) {
    set_error("fio_plan: dtype must be FIO_C64 or FIO_C128");
    return FIO_EINVAL;
  }
  // accuracy floors (reading R24): complex64 arithmetic cannot deliver 10 eps below ~1e-6;
  // complex128 is limited by the largest NUFFT window (kMaxTaps taps, ~1e-11)
  const double eps_floor = o.dtype == FIO_C64 ? kEpsFloorC64 : kEpsFloorC128;
  if (eps < eps_floor) {
    set_error("fio_plan: eps " + std::to_string(eps) + " is below the " +
              (o.dtype == FIO_C64 ? std::string("complex64") : std::string("complex128")) + " floor " +
              std::to_string(eps_floor));
    return FIO_EINVAL;
  }
  if (o.nranks < 1 || o.rank < 0 || o.rank >= o.nranks) {
    set_error("fio_plan: need 0 <= rank < nranks");
    return FIO_EINVAL;
  }
  if (o.nufft_w != 0 && (o.nufft_w < 3 || o.nufft_w > kMaxTaps)) {
    set_error("fio_plan: nufft_w must be 0 or in [3, 12]");
    return FIO_EINVAL;
  }
  if (o.paper_accept != 0 && o.paper_accept != 1) {
    set_error("fio_plan: paper_accept must be 0 or 1");
    return FIO_EINVAL;
  }
  if (!(o.wedge_overlap >= 0.0 && o.wedge_overlap <= 1.0)) {
    set_error("fio_plan: wedge_overlap must lie in [0, 1]");
    return FIO_EINVAL;
  }
  if (o.n_wedges < 0 || o.r_init < 0 || o.r_max < 0) {
    set_error("fio_plan: negative option");
    return FIO_EINVAL;
  }
  if (o.nranks > 1 && o.nccl_id && N % o.nranks != 0) {
    set_error("fio_plan: with a communicator nranks must divide N (row slabs)");
    return FIO_EINVAL;
  }
  if (o.allgather != 0 && o.allgather != 1) {
    set_error("fio_plan: allgather must be 0 or 1");
    return FIO_EINVAL;
  }
  if (o.allgather && !o.nccl_id) {
    set_error("fio_plan: allgather needs a communicator (nccl_id)");
    return FIO_EINVAL;
  }
  if (o.r_init == 0) o.r_init = 32;
  if (o.r_max == 0) o.r_max = 512;
  FIO_GUARD(o.device)
  auto t0 = std::chrono::steady_clock::now();
  fio_plan_s* P = new (std::nothrow) fio_plan_s();
  if (!P) {
    set_error("fio_plan: out of host memory");
    return FIO_ENOMEM;
  }
  cudaGetDevice(&P->device);
  P->N = N;
  P->eps = eps;
  P->opts = o;
  P->c64 = o.dtype == FIO_C64;
  P->W = o.n_wedges > 0 ? o.n_wedges : default_wedges(N);
  P->taps = o.nufft_w > 0 ? o.nufft_w : taps_for_eps(eps);
  P->es_beta = o.nufft_beta > 0 ? o.nufft_beta : 2.30 * P->taps;
  // polynomial kernel for the c128 K3 weights: error ~1.5 e^{-beta}, the kernel's own edge value
  P->poly_err = es_poly_fit(P->taps, P->es_beta, P->poly);
  P->input_hash = input_hash(N, phase, amp);
  if (o.wedge_overlap > 0.0) P->input_hash = fnv1a(P->input_hash, &o.wedge_overlap, sizeof(double));
  if (o.paper_accept) P->input_hash = fnv1a(P->input_hash, &o.paper_accept, sizeof(int));
  if (load) {  // fio_plan_load: the file must describe exactly this plan
    const bool same = hdr->N == N && hdr->W == P->W && hdr->dtype == o.dtype && hdr->taps == P->taps &&
                      hdr->rank == o.rank && hdr->nranks == o.nranks && hdr->eps == eps &&
                      hdr->es_beta == P->es_beta && hdr->seed == o.seed && hdr->input_hash == P->input_hash;
    if (!same) {
      delete P;
      set_error("fio_plan_load: the file was saved for a different operator, size, eps or options");
      return FIO_EINVAL;
    }
    P->load = load;
  }
  fio_status st = FIO_OK;
  if (o.nccl_id) {  // (nranks == 1 is allowed: a one-rank communicator, the reduce-scatter is a copy)
    // first, so that a rank whose plan fails later does not leave the others waiting in the init
    st = comm_create(o.nccl_id, o.nranks, o.rank, &P->comm);
    if (st != FIO_OK) {
      delete P;
      return st;
    }
  }
  P->opts.nccl_id = nullptr;  // not retained (the caller owns the id bytes)
  st = build_plan(*P, phase, amp);
  P->load = nullptr;
  if (st < 0) {
    delete P;
    return st;
  }
  P->plan_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  P->launches = 4 + std::max<int>(1, (int)P->wd.size()) * (o.skeleton ? 2 : 1);
  *out = P;
  return P->certified ? FIO_OK : FIO_WNOTCERT;
}

fio_status fio_apply(fio_handle h, const void* f_dev, void* Lf_dev, void* stream) {
  if (!h || !f_dev || !Lf_dev) {
    set_error("fio_apply: NULL argument");
    return FIO_EINVAL;
  }
  if (overlaps(f_dev, h->elem_bytes() * (size_t)h->N * h->N, Lf_dev, h->elem_bytes() * (size_t)h->out_rows() * h->N)) {
    set_error("fio_apply: f and Lf must not overlap");
    return FIO_EINVAL;
  }
  FIO_GUARD(h->device)
  ApplyArgs a = make_args(*h);
  int launches = 0;
  cudaEvent_t* ev = nullptr;
  if (h->prof_n < h->prof_cap) ev = &h->prof_ev[(size_t)h->prof_n++ * (kStages + 1)];
  cudaStream_t s = (cudaStream_t)stream;
  if (!h->comm) {
    FIO_CUDA(enqueue_apply(a, h->c64, f_dev, Lf_dev, s, &launches, ev));
    h->launches = launches;
    return FIO_OK;
  }
  // A6: this rank's partial over its wedges, then the sum over ranks into its row slab
  FIO_CUDA(h->ensure_part(1, s));
  FIO_CUDA(enqueue_apply(a, h->c64, f_dev, h->part, s, &launches, ev));
  h->launches = launches;
  return h->sum_ranks(h->part, Lf_dev, s);
}

fio_status fio_apply_batch(fio_handle h, int nrhs, const void* f_dev, void* Lf_dev, void* stream) {
  if (!h || !f_dev || !Lf_dev || nrhs < 1) {
    set_error("fio_apply_batch: bad arguments");
    return FIO_EINVAL;
  }
  if (overlaps(f_dev, h->elem_bytes() * (size_t)h->N * h->N * nrhs, Lf_dev,
               h->elem_bytes() * (size_t)h->out_rows() * h->N * nrhs)) {
    set_error("fio_apply_batch: f and Lf must not overlap");
    return FIO_EINVAL;
  }
  FIO_GUARD(h->device)
  const size_t cs = h->c64 ? sizeof(float2) : sizeof(double2);
  const size_t NN = (size_t)h->N * h->N;
  const size_t nacc = 1;  // K3's second accumulator
  const size_t per = NN + std::max<size_t>(h->fine_elems, 1) + nacc * NN;
  if (nrhs > h->batch_cap) {
    FIO_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    if (h->batch_ws) {
      cudaFree(h->batch_ws);
      h->batch_ws = nullptr;
    }
    FIO_CUDA(cudaMalloc(&h->batch_ws, cs * per * (size_t)(nrhs - 1)));
    h->batch_cap = nrhs;
  }
  std::vector<ApplyArgs> args(nrhs, make_args(*h));
  for (int b = 1; b < nrhs; ++b) {
    char* base = static_cast<char*>(h->batch_ws) + cs * per * (size_t)(b - 1);
    args[b].fhat = base;
    args[b].g = base + cs * NN;
    args[b].acc[0] = base + cs * (NN + std::max<size_t>(h->fine_elems, 1));
  }
  int launches = 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (!h->comm) {
    FIO_CUDA(enqueue_apply_batch(args.data(), nrhs, h->c64, f_dev, Lf_dev, s, &launches));
    return FIO_OK;
  }
  FIO_CUDA(h->ensure_part(nrhs, s));
  FIO_CUDA(enqueue_apply_batch(args.data(), nrhs, h->c64, f_dev, h->part, s, &launches));
  const size_t slab = (size_t)h->out_rows() * h->N;
  for (int b = 0; b < nrhs; ++b) {
    fio_status st = h->sum_ranks(static_cast<char*>(h->part) + cs * NN * b, static_cast<char*>(Lf_dev) + cs * slab * b, s);
    if (st != FIO_OK) return st;
  }
  return FIO_OK;
}

fio_status fio_apply_adjoint(fio_handle h, const void* g_dev, void* out_dev, void* stream) {
  if (!h || !g_dev || !out_dev) {
    set_error("fio_apply_adjoint: NULL argument");
    return FIO_EINVAL;
  }
  if (overlaps(g_dev, h->elem_bytes() * (size_t)h->N * h->N, out_dev, h->elem_bytes() * (size_t)h->out_rows() * h->N)) {
    set_error("fio_apply_adjoint: g and out must not overlap");
    return FIO_EINVAL;
  }
  FIO_GUARD(h->device)
  ApplyArgs a = make_args(*h);
  int launches = 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (!h->comm) {
    FIO_CUDA(enqueue_adjoint(a, h->c64, g_dev, out_dev, s, &launches));
    return FIO_OK;
  }
  FIO_CUDA(h->ensure_part(1, s));
  FIO_CUDA(enqueue_adjoint(a, h->c64, g_dev, h->part, s, &launches));
  return h->sum_ranks(h->part, out_dev, s);
}

fio_status fio_apply_host(fio_handle h, const void* f_host, void* Lf_host, void* stream) {
  if (!h || !f_host || !Lf_host) {
    set_error("fio_apply_host: NULL argument");
    return FIO_EINVAL;
  }
  const size_t bytes = (size_t)h->N * h->N * h->elem_bytes();
  const size_t out_bytes = (size_t)h->out_rows() * h->N * h->elem_bytes();
  FIO_GUARD(h->device)  // the staging buffers live on the plan's device
  if (!h->e2e_in) {
    FIO_CUDA(h->alloc(&h->e2e_in, bytes));
    FIO_CUDA(h->alloc(&h->e2e_out, bytes));
  }
  cudaStream_t s = (cudaStream_t)stream;
  FIO_CUDA(cudaMemcpyAsync(h->e2e_in, f_host, bytes, cudaMemcpyHostToDevice, s));
  fio_status st = fio_apply(h, h->e2e_in, h->e2e_out, stream);
  if (st != FIO_OK) return st;
  FIO_CUDA(cudaMemcpyAsync(Lf_host, h->e2e_out, out_bytes, cudaMemcpyDeviceToHost, s));
  FIO_CUDA(cudaStreamSynchronize(s));
  return FIO_OK;
}

fio_status fio_apply_host_stream(fio_handle h, int count, const void* f_host, void* Lf_host, void* stream) {
  if (!h || count < 0 || (count > 0 && (!f_host || !Lf_host))) {
    set_error("fio_apply_host_stream: bad arguments");
    return FIO_EINVAL;
  }
  if (count == 0) return FIO_OK;
  const size_t bytes = (size_t)h->N * h->N * h->elem_bytes();
  const size_t out_bytes = (size_t)h->out_rows() * h->N * h->elem_bytes();
  FIO_GUARD(h->device)
  if (!h->hs_in[0]) {
    for (int b = 0; b < 2; ++b) {
      FIO_CUDA(h->alloc(&h->hs_in[b], bytes));
      FIO_CUDA(h->alloc(&h->hs_out[b], bytes));
      FIO_CUDA(cudaEventCreateWithFlags(&h->hs_in_ready[b], cudaEventDisableTiming));
      FIO_CUDA(cudaEventCreateWithFlags(&h->hs_done[b], cudaEventDisableTiming));
      FIO_CUDA(cudaEventCreateWithFlags(&h->hs_out_free[b], cudaEventDisableTiming));
    }
    FIO_CUDA(cudaEventCreateWithFlags(&h->hs_fork, cudaEventDisableTiming));
    FIO_CUDA(cudaEventCreateWithFlags(&h->hs_join, cudaEventDisableTiming));
    FIO_CUDA(cudaStreamCreateWithFlags(&h->hs_h2d, cudaStreamNonBlocking));
    FIO_CUDA(cudaStreamCreateWithFlags(&h->hs_d2h, cudaStreamNonBlocking));
  }
  cudaStream_t s = (cudaStream_t)stream;
  // the copy streams start behind everything already enqueued on `stream`
  FIO_CUDA(cudaEventRecord(h->hs_fork, s));
  FIO_CUDA(cudaStreamWaitEvent(h->hs_h2d, h->hs_fork, 0));
  FIO_CUDA(cudaStreamWaitEvent(h->hs_d2h, h->hs_fork, 0));
  for (int i = 0; i < count; ++i) {
    const int b = i & 1;
    const char* in = static_cast<const char*>(f_host) + (size_t)i * bytes;
    char* out = static_cast<char*>(Lf_host) + (size_t)i * out_bytes;
    // input i into staging b once apply i-2 has consumed it
    if (i >= 2) FIO_CUDA(cudaStreamWaitEvent(h->hs_h2d, h->hs_done[b], 0));
    FIO_CUDA(cudaMemcpyAsync(h->hs_in[b], in, bytes, cudaMemcpyHostToDevice, h->hs_h2d));
    FIO_CUDA(cudaEventRecord(h->hs_in_ready[b], h->hs_h2d));
    // apply i once its input has landed and the read-back of output i-2 has left staging b
    FIO_CUDA(cudaStreamWaitEvent(s, h->hs_in_ready[b], 0));
    if (i >= 2) FIO_CUDA(cudaStreamWaitEvent(s, h->hs_out_free[b], 0));
    fio_status st = fio_apply(h, h->hs_in[b], h->hs_out[b], stream);
    if (st != FIO_OK) return st;
    FIO_CUDA(cudaEventRecord(h->hs_done[b], s));
    // read-back of output i on the second copy stream (both copy directions overlap the applies)
    FIO_CUDA(cudaStreamWaitEvent(h->hs_d2h, h->hs_done[b], 0));
    FIO_CUDA(cudaMemcpyAsync(out, h->hs_out[b], out_bytes, cudaMemcpyDeviceToHost, h->hs_d2h));
    FIO_CUDA(cudaEventRecord(h->hs_out_free[b], h->hs_d2h));
  }
  FIO_CUDA(cudaEventRecord(h->hs_join, h->hs_d2h));
  FIO_CUDA(cudaStreamWaitEvent(s, h->hs_join, 0));
  FIO_CUDA(cudaStreamSynchronize(s));
  return FIO_OK;
}

fio_status fio_profile_begin(fio_handle h, int max_applies) {
  if (!h || max_applies < 0) {
    set_error("fio_profile_begin: bad arguments");
    return FIO_EINVAL;
  }
  FIO_GUARD(h->device)
  h->free_events();
  h->prof_ev.resize((size_t)max_applies * (kStages + 1));
  for (auto& e : h->prof_ev) FIO_CUDA(cudaEventCreate(&e));
  h->prof_cap = max_applies;
  h->prof_n = 0;
  return FIO_OK;
}

fio_status fio_profile_end(fio_handle h, double* stage_ms, int* n_applies) {
  if (!h) {
    set_error("fio_profile_end: NULL handle");
    return FIO_EINVAL;
  }
  FIO_GUARD(h->device)
  std::vector<double> acc(kStages, 0.0);
  for (int i = 0; i < h->prof_n; ++i) {
    cudaEvent_t* ev = &h->prof_ev[(size_t)i * (kStages + 1)];
    FIO_CUDA(cudaEventSynchronize(ev[kStages]));
    for (int st = 0; st < kStages; ++st) {
      float ms = 0.f;
      FIO_CUDA(cudaEventElapsedTime(&ms, ev[st], ev[st + 1]));
      acc[st] += ms;
    }
  }
  if (stage_ms)
    for (int st = 0; st < kStages; ++st) stage_ms[st] = acc[st];
  if (n_applies) *n_applies = h->prof_n;
  h->free_events();
  return FIO_OK;
}

fio_status fio_destroy(fio_handle h) {
  if (!h) return FIO_OK;
  FIO_GUARD(h->device)  // streams, events and buffers are released on the plan's device
  delete h;
  return FIO_OK;
}

fio_status fio_plan_info(fio_handle h, fio_info* info) {
  if (!h || !info) {
    set_error("fio_plan_info: NULL argument");
    return FIO_EINVAL;
  }
  std::memset(info, 0, sizeof(*info));
  info->N = h->N;
  info->W = h->W;
  info->nufft_w = h->taps;
  info->dtype = h->c64 ? FIO_C64 : FIO_C128;
  info->rank = h->opts.rank;
  info->nranks = h->opts.nranks;
  info->n_owned = (int)h->wd.size();
  for (const auto& w : h->wd) info->sum_q += w.q;
  info->certified = h->certified;
  info->nufft_beta = h->es_beta;
  info->max_sep_err = h->max_err;
  info->plan_seconds = h->plan_seconds;
  info->alpha_bytes = h->alpha_bytes;
  info->meta_bytes = h->meta_bytes;
  info->slots = h->slots;
  info->max_tile_cap = h->max_tile_cap;
  info->k3_thread_slots = h->chunk_threads;
  info->rank_balance = h->balance;
  info->slot_terms = h->slot_terms;
  info->group_p = group_p(h->c64, h->taps);
  info->skeleton_bytes = h->skel_bytes;
  info->k3_window_cols = k3_window_cols(h->taps, h->c64);
  info->k3_streams = 2;  // K3 launches alternate between the caller's stream and the side stream
  info->k3_window_rows = k3_window_rows(h->taps, h->c64);
  info->beta_bytes = h->beta_bytes;
  info->workspace_bytes = h->ws_bytes;
  info->fine_elems = h->fine_elems;
  info->p1_elems = h->p1_elems;
  info->launches_per_apply = h->launches;
  info->has_comm = h->comm ? 1 : 0;
  info->wedge_overlap = h->opts.wedge_overlap;
  for (int l : h->owned) info->members += (long long)h->geom[l].members.size();
  info->out_rows = h->out_rows();
  return FIO_OK;
}

fio_status fio_plan_wedges(fio_handle h, int* l, int* q, int* box, int* M, int* xc, int* r, double* sep_err) {
  if (!h) {
    set_error("fio_plan_wedges: NULL handle");
    return FIO_EINVAL;
  }
  for (size_t i = 0; i < h->wd.size(); ++i) {
    const WedgeDev& w = h->wd[i];
    if (l) l[i] = w.l;
    if (q) q[i] = w.q;
    if (box) { box[4 * i] = w.n1; box[4 * i + 1] = w.n2; box[4 * i + 2] = w.n1f; box[4 * i + 3] = w.n2f; }
    if (M) std::memcpy(M + 4 * i, w.M, 4 * sizeof(int));
    if (xc) { xc[2 * i] = w.xc1; xc[2 * i + 1] = w.xc2; }
    if (r) r[i] = h->r_final[i];
    if (sep_err) sep_err[i] = h->sep_err[i];
  }
  return FIO_OK;
}

}  // extern "C"
