// fio_kernels.h -- launchers of the sm_100a kernels (fio_kernels.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "fio_internal.h"

namespace fio {

// Phase/amplitude data resident on the device (copied at plan time).
struct OperatorDev {
  int N;
  const double* c1;
  const double* c2;
  const double* b1;   // may be null
  const double* b2;   // may be null
  int K;
  const double2* px;  // K x N*N
  const double2* pxi; // K x N*N (FFT order)
  int sign;           // Phi = x.xi + b.xi + sign * rho
  int amp_kind;       // FIO_AMP_SEPARABLE / FIO_AMP_BESSEL_GRT
};

// ---- plan-time kernels (FP64) ----
// out[i*ldr + j*ldc] = a(x_i, xi_j) e^{2 pi i Phi_l(x_i, xi_j)} with the residual
// phase Phi_l = Phi - grad_xi Phi(x, xihat_l).xi.
cudaError_t launch_eval_entries(const OperatorDev& op, double u1, double u2, const int* rows, int nr,
                                const int* cols, int nc, double2* out, long long ldr, long long ldc,
                                cudaStream_t s);

// C(i,j) = sum_k opA(i,k) opB(k,j), complex FP64, strided operands; conjA
// conjugates A.  Split over K into `nsplit` partial products that are summed
// by a second kernel into C (work buffer of nsplit*p*s elements).
cudaError_t launch_zgemm(int p, int s, long long K, const double2* A, long long sai, long long sak, bool conjA,
                         const double2* B, long long sbk, long long sbj, double2* C, long long sci,
                         long long scj, int nsplit, double2* work, cudaStream_t st);

cudaError_t launch_gather_rows(const double2* U, long long m, int q, const int* rows, int nrows, double2* out,
                               cudaStream_t s);

// alpha'[t][x] = U[x + t m] e^{2 pi i y_l(x).xi_c} / N  (center phase of
// PAPER.md:1349-1356 and the 1/N of eq. dfio folded at plan time), in T2.
// in group-slot order: alpha'[t][s] for slot s with output point slot_x[s] (0 for padding)
cudaError_t launch_fold_alpha(const OperatorDev& op, const WedgeDev& w, const double2* U, int q, const int* slot_x,
                              long long nslots, void* alpha, bool c64, cudaStream_t s);

// u[x] = frac(y_l(x)) * (n1f, n2f), FP64 (plan-time input of the point grouping)
cudaError_t launch_fine_coords(const OperatorDev& op, const WedgeDev& w, double2* u, cudaStream_t s);

// beta'[t][i1][i2] = beta[t + j q] d1[i1] d2[i2] at the box cell of member j
// (zero elsewhere; chi_l, the relabeling xi' = M xi - xi_c and the NUFFT
// deconvolution folded).
cudaError_t launch_fold_beta(int N, const WedgeDev& w, const int* members, int n, const double2* beta, int q,
                             const double* d1, const double* d2, const double* chi, void* betap, bool c64,
                             cudaStream_t s);

// Skeleton storage: per owned wedge the skeleton columns C (member
// frequency indices) and Y = V S^{-1} (rc x q, column-major, FP64).
struct SkelWedge {
  int rc;
  const int* C;
  const double2* Y;
};

// alpha'[t][s] = e^{2 pi i y(x_s).xi_c} / N * sum_c A(x_s, C_c) Y[c + t rc]  (slot order; 0 for padding)
size_t rebuild_smem_bytes(int rc, int q);
cudaError_t configure_rebuild(bool c64, size_t smem);  // per device, at plan time
cudaError_t launch_rebuild_alpha(const OperatorDev& op, const WedgeDev& w, const SkelWedge& sk, int q,
                                 const int* slot_x, long long nslots, void* alpha, bool c64, cudaStream_t s);

// ---- apply-time kernels (the hot path) ----

struct ApplyArgs {
  int N;
  int nw;                   // owned wedges
  const WedgeDev* wedges;   // device table
  const FftLen* ffts;       // device table
  int fft_N;                // FftLen index of length N (input spectrum)
  const void* tw;           // twiddles (double2 or float2)
  const InterpWedge* iw;    // host array, one per owned wedge (passed by value to K3)
  const WedgeDev* wd_host;  // host copy of the wedge table
  const SkelWedge* skel;    // host array (skeleton mode) or nullptr: alpha' rebuilt before each K3
  const void* const* beta;  // per owned wedge
  OperatorDev op;
  const double2* a0;        // a(x,0)/N, N*N
  int add_dc;
  int taps;                 // w (K3 template), groups of group_p(dtype) points
  double es_beta;
  const EsPoly* poly;       // host pointer: piecewise-polynomial kernel (c128 K3 weights)
  void* fhat;               // N*N workspace
  void* tmp;                // N*N workspace
  void* p1;                 // row-pass buffer
  void* g;                  // fine grids
  const FftJob* jobs_row; int njobs_row; int smem_row;
  const FftJob* jobs_col; int njobs_col; int smem_col;
  const FftJob* jobs_rowadj; int njobs_rowadj; int smem_rowadj;  // K1* (all t per job)
  const unsigned char* const* masks;  // per owned wedge: n1 x n2 box mask (cell is a member)
  size_t fine_elems;        // elements of the fine-grid workspace (G, reused as G* by the adjoint)
  // second K3 accumulator (the side stream's wedges), N*N per RHS, the plan-owned side stream of K3
  // and of the adjoint's spreads, and the events that fork / join it
  void* acc[1];
  cudaStream_t side[1];
  cudaEvent_t fork, join[1];
  int rows_per_cta_N;       // K0 row pass
  int cols_per_cta_N;       // K0 column pass
  int sms;                  // multiprocessors of the plan's device (grid sizing)
  int overlap;              // smooth partition: wedges overlap, K1* accumulates fhat* atomically
  int k3_rhs;               // fio_apply_batch: right-hand sides per K3 launch (1 or 2; FIO_K3_RHS)
  const CUtensorMap* tmaps; // host array, per owned wedge: TMA map of its fine grids (iw.tma), or null
};

// Enqueue the whole apply (K0 row/column FFT, K1 window x beta + row FFT,
// K2 column FFT, K3 interpolation + alpha epilogue).  Returns the number of
// kernels launched in *launches.
// ev (optional): 6 events recorded before K0 and after each of the 5 stages.
cudaError_t enqueue_apply(const ApplyArgs& a, bool c64, const void* f, void* Lf, cudaStream_t s, int* launches,
                          cudaEvent_t* ev = nullptr);
constexpr int kStages = 5;

// Multi-RHS apply (NEXT-2): args[b] differ only in the per-RHS workspace (fhat, fine grids);
// f and Lf hold nrhs contiguous N x N arrays.  In skeleton mode alpha' is rebuilt once per wedge.
cudaError_t enqueue_apply_batch(const ApplyArgs* args, int nrhs, bool c64, const void* f, void* Lf, cudaStream_t s,
                                int* launches);

// Enqueue the exact adjoint of the fast operator: out = L~* g.
cudaError_t enqueue_adjoint(const ApplyArgs& a, bool c64, const void* g, void* out, cudaStream_t s, int* launches);

// Dynamic shared memory needed by the FFT passes for one sequence of length L.
size_t fft_seq_bytes(int L, bool c64);
size_t k1_row_bytes(int L, bool c64);  // K1 shared memory per row (two buffers of stride L + 1)
cudaError_t configure_kernels(size_t smem_bytes);
// Opt the K3 instance for (taps, dtype) into the dynamic shared memory of the plan's largest chunk
// footprint, on the current device (per device: every plan configures its own device).
cudaError_t configure_interp(int taps, bool c64, long long max_tile_cap);

}  // namespace fio
