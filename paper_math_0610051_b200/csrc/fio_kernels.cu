// fio_kernels.cu -- sm_100a CUDA kernels of the wedge-decomposed FIO apply
// (arXiv math/0610051) and of its plan.
//
// Hot path, per fio_apply:
//   K0  k_fft_rows / k_fft_cols   fhat = DFT(f)/N, eq. (dft)
//   K1  k_rowpass                 fhat * chi_l * beta_lt relabelled onto the box
//                                 (PAPER.md:1297-1298, 1327-1347), deconvolved,
//                                 zero-padded, FFT along axis 2, written transposed
//   K2  k_colpass                 zero-padded FFT along axis 1 -> fine grid G_lt, stored
//                                 [j2][j1] (the oversampled FFT of the NUFFT)
//   K3  k_interp                  interpolation of G_lt at the warped points
//                                 M^{-T} grad Phi(x, xihat_l) (PAPER.md:1299-1311,
//                                 1357-1363) fused with the alpha epilogue and the
//                                 sums over t and l, + DC term.
// No code here is shared with oracle/.
#include <vector>
#include <type_traits>
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <map>
#include <mutex>

#include "fio_kernels.h"

namespace fio {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per (kernel, device) and a later call with a
// smaller value would lower it under an existing plan: raise-only, per device, under a mutex.
static cudaError_t raise_smem_attr(const void* func, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = done[{func, dev}];
  if (smem <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) cur = smem;
  return e;
}

// ------------------------------------------------------------------ complex helpers
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }

template <typename T2> struct Real;
template <> struct Real<double2> { using type = double; };
template <> struct Real<float2> { using type = float; };

template <typename T2>
__device__ __forceinline__ T2 mk(typename Real<T2>::type x, typename Real<T2>::type y) {
  T2 r;
  r.x = x;
  r.y = y;
  return r;
}
template <typename T2>
__device__ __forceinline__ T2 to_t2(double2 v) {
  return mk<T2>((typename Real<T2>::type)v.x, (typename Real<T2>::type)v.y);
}

// ------------------------------------------------------------------ phase geometry
// grad_xi rho(x, u) for rho = sqrt(c1^2 xi1^2 + c2^2 xi2^2), u = xihat_l.
__device__ __forceinline__ void grad_rho(double c1, double c2, double u1, double u2, double& g1, double& g2) {
  double a = c1 * c1 * u1, b = c2 * c2 * u2;
  double den = sqrt(a * u1 + b * u2);
  if (den > 0.0) {
    g1 = a / den;
    g2 = b / den;
  } else {
    g1 = 0.0;
    g2 = 0.0;
  }
}

// y_l(x) = M^{-T} g_l(x), g_l(x) = x + b(x) + grad_xi rho(x, xihat_l)
__device__ __forceinline__ void warped_point(const OperatorDev& op, int n1, int n2, const WedgeDev& w, double& y1,
                                             double& y2) {
  const int N = op.N;
  const long long x = (long long)n1 * N + n2;
  double c1 = op.c1[x], c2 = op.c2[x];
  double gr1, gr2;
  grad_rho(c1, c2, w.u1, w.u2, gr1, gr2);
  double g1 = (double)n1 / N + op.sign * gr1, g2 = (double)n2 / N + op.sign * gr2;
  if (op.b1) g1 += op.b1[x];
  if (op.b2) g2 += op.b2[x];
  y1 = (double)w.Mi[0] * g1 + (double)w.Mi[2] * g2;
  y2 = (double)w.Mi[1] * g1 + (double)w.Mi[3] * g2;
}

// ------------------------------------------------------------------ plan kernels
// Residual kernel entry A(x, xi) = a(x, xi) e^{2 pi i (rho(x,xi) - grad rho(x,xihat).xi)}; the
// x-only quantities (c1, c2, grad rho(x, xihat)) are passed in.
__device__ double2 kernel_entry_x(const OperatorDev& op, int x, double c1, double c2, double g1, double g2, int kf) {
  const int N = op.N;
  int k1 = kf / N, k2 = kf - k1 * N;
  double xi1 = (double)(k1 >= N / 2 ? k1 - N : k1);
  double xi2 = (double)(k2 >= N / 2 ? k2 - N : k2);
  double rho = sqrt(c1 * c1 * xi1 * xi1 + c2 * c2 * xi2 * xi2);
  double ph = op.sign * (rho - g1 * xi1 - g2 * xi2);
  ph -= floor(ph);
  double s, c;
  sincospi(2.0 * ph, &s, &c);
  double2 e = make_double2(c, s);
  if (op.amp_kind == FIO_AMP_BESSEL_GRT) {
    // eq. ellipses_amp, rho_e = max(rho, 1/2) (reading R22)
    const double re = rho < 0.5 ? 0.5 : rho;
    const double J = j0(6.283185307179586476925286766559 * re), Y = y0(6.283185307179586476925286766559 * re);
    double fr = re - floor(re), sn, cs;
    sincospi(2.0 * fr, &sn, &cs);
    sn = -op.sign * sn;  // e^{-s 2 pi i rho_e}
    const double inv4pi = 0.079577471545947667884;
    const double2 a = make_double2((J * cs - op.sign * Y * sn) * inv4pi, (J * sn + op.sign * Y * cs) * inv4pi);
    e = cmul(a, e);
  } else if (op.K > 0) {
    double2 a = make_double2(0.0, 0.0);
    const long long NN = (long long)N * N;
    for (int k = 0; k < op.K; ++k) a = cadd(a, cmul(op.px[k * NN + x], op.pxi[k * NN + kf]));
    e = cmul(a, e);
  }
  return e;
}

__device__ double2 kernel_entry(const OperatorDev& op, int x, int kf, double u1, double u2) {
  const double c1 = op.c1[x], c2 = op.c2[x];
  double g1, g2;
  grad_rho(c1, c2, u1, u2, g1, g2);
  return kernel_entry_x(op, x, c1, c2, g1, g2, kf);
}

__global__ void k_eval_entries(OperatorDev op, double u1, double u2, const int* __restrict__ rows, int nr,
                               const int* __restrict__ cols, int nc, double2* __restrict__ out, long long ldr,
                               long long ldc) {
  long long total = (long long)nr * nc;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    int i = (int)(idx % nr), j = (int)(idx / nr);
    int x = rows ? rows[i] : i;
    out[i * ldr + j * ldc] = kernel_entry(op, x, cols[j], u1, u2);
  }
}

cudaError_t launch_eval_entries(const OperatorDev& op, double u1, double u2, const int* rows, int nr,
                                const int* cols, int nc, double2* out, long long ldr, long long ldc,
                                cudaStream_t s) {
  long long total = (long long)nr * nc;
  if (total == 0) return cudaSuccess;
  int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 64);
  k_eval_entries<<<blocks, 256, 0, s>>>(op, u1, u2, rows, nr, cols, nc, out, ldr, ldc);
  return cudaGetLastError();
}

// Tiled complex FP64 product (plan-time Gram matrix, factor expansion).
// loadA_i: A tile loaded with threadIdx.x along i (A contiguous in i) else along k.
__global__ void k_zgemm(int p, int s, long long K, long long kchunk, const double2* __restrict__ A, long long sai,
                        long long sak, int conjA, int loadA_i, const double2* __restrict__ B, long long sbk,
                        long long sbj, int loadB_k, double2* __restrict__ C, long long sci, long long scj,
                        long long split_stride) {
  __shared__ double2 As[16][17];  // [i][k]
  __shared__ double2 Bs[16][17];  // [k][j]
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int ib = blockIdx.x * 16, jb = blockIdx.y * 16;
  const long long k0 = (long long)blockIdx.z * kchunk;
  const long long k1 = min(K, k0 + kchunk);
  double2 acc = make_double2(0.0, 0.0);
  for (long long kk = k0; kk < k1; kk += 16) {
    {
      int ii = loadA_i ? tx : ty, kt = loadA_i ? ty : tx;
      int i = ib + ii;
      long long k = kk + kt;
      double2 v = make_double2(0.0, 0.0);
      if (i < p && k < k1) {
        v = A[i * sai + k * sak];
        if (conjA) v.y = -v.y;
      }
      As[ii][kt] = v;
    }
    {
      int kt = loadB_k ? tx : ty, jj = loadB_k ? ty : tx;
      int j = jb + jj;
      long long k = kk + kt;
      double2 v = make_double2(0.0, 0.0);
      if (j < s && k < k1) v = B[k * sbk + j * sbj];
      Bs[kt][jj] = v;
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      double2 a = As[ty][t], b = Bs[t][tx];
      acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
      acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
    }
    __syncthreads();
  }
  int i = ib + ty, j = jb + tx;
  if (i < p && j < s) C[blockIdx.z * split_stride + i * sci + j * scj] = acc;
}

__global__ void k_split_reduce(int p, int s, int nsplit, const double2* __restrict__ work, double2* __restrict__ C,
                               long long sci, long long scj) {
  long long total = (long long)p * s;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    int i = (int)(idx / s), j = (int)(idx % s);
    double2 acc = make_double2(0.0, 0.0);
    for (int z = 0; z < nsplit; ++z) acc = cadd(acc, work[z * total + idx]);
    C[i * sci + j * scj] = acc;
  }
}

cudaError_t launch_zgemm(int p, int s, long long K, const double2* A, long long sai, long long sak, bool conjA,
                         const double2* B, long long sbk, long long sbj, double2* C, long long sci,
                         long long scj, int nsplit, double2* work, cudaStream_t st) {
  if (p == 0 || s == 0) return cudaSuccess;
  if (nsplit < 1) nsplit = 1;
  long long kchunk = (K + nsplit - 1) / nsplit;
  kchunk = ((kchunk + 15) / 16) * 16;
  nsplit = (int)((K + kchunk - 1) / kchunk);
  if (nsplit < 1) nsplit = 1;
  dim3 grid((p + 15) / 16, (s + 15) / 16, nsplit), block(16, 16);
  int loadA_i = (sai == 1 && sak != 1) ? 1 : 0;
  int loadB_k = (sbk == 1 && sbj != 1) ? 1 : 0;
  if (nsplit == 1) {
    k_zgemm<<<grid, block, 0, st>>>(p, s, K, kchunk, A, sai, sak, conjA, loadA_i, B, sbk, sbj, loadB_k, C, sci, scj,
                                    0);
    return cudaGetLastError();
  }
  k_zgemm<<<grid, block, 0, st>>>(p, s, K, kchunk, A, sai, sak, conjA, loadA_i, B, sbk, sbj, loadB_k, work,
                                  (long long)s, 1, (long long)p * s);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  long long total = (long long)p * s;
  int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 32);
  k_split_reduce<<<blocks, 256, 0, st>>>(p, s, nsplit, work, C, sci, scj);
  return cudaGetLastError();
}

__global__ void k_gather_rows(const double2* __restrict__ U, long long m, int q, const int* __restrict__ rows,
                              int nrows, double2* __restrict__ out) {
  long long total = (long long)nrows * q;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    int i = (int)(idx % nrows), t = (int)(idx / nrows);
    out[i + (long long)t * nrows] = U[rows[i] + (long long)t * m];
  }
}

cudaError_t launch_gather_rows(const double2* U, long long m, int q, const int* rows, int nrows, double2* out,
                               cudaStream_t s) {
  long long total = (long long)nrows * q;
  if (total == 0) return cudaSuccess;
  int blocks = (int)std::min<long long>((total + 255) / 256, 4096);
  k_gather_rows<<<blocks, 256, 0, s>>>(U, m, q, rows, nrows, out);
  return cudaGetLastError();
}

template <typename T2>
__global__ void k_fold_alpha(OperatorDev op, WedgeDev w, const double2* __restrict__ U, int q,
                             const int* __restrict__ slot_x, long long nslots, T2* __restrict__ alpha) {
  const int N = op.N;
  const long long NN = (long long)N * N;
  for (long long sl = blockIdx.x * (long long)blockDim.x + threadIdx.x; sl < nslots;
       sl += (long long)gridDim.x * blockDim.x) {
    const int x = slot_x[sl];
    if (x < 0) {
      for (int t = 0; t < q; ++t) alpha[t * nslots + sl] = to_t2<T2>(make_double2(0.0, 0.0));
      continue;
    }
    double y1, y2;
    warped_point(op, x / N, x % N, w, y1, y2);
    double ph = y1 * (double)w.xc1 + y2 * (double)w.xc2;
    ph -= floor(ph);
    double s, c;
    sincospi(2.0 * ph, &s, &c);
    double2 e = make_double2(c / N, s / N);
    for (int t = 0; t < q; ++t) alpha[t * nslots + sl] = to_t2<T2>(cmul(U[x + t * NN], e));
  }
}

cudaError_t launch_fold_alpha(const OperatorDev& op, const WedgeDev& w, const double2* U, int q, const int* slot_x,
                              long long nslots, void* alpha, bool c64, cudaStream_t s) {
  int blocks = (int)std::min<long long>((nslots + 255) / 256, 148LL * 16);
  if (c64)
    k_fold_alpha<float2><<<blocks, 256, 0, s>>>(op, w, U, q, slot_x, nslots, (float2*)alpha);
  else
    k_fold_alpha<double2><<<blocks, 256, 0, s>>>(op, w, U, q, slot_x, nslots, (double2*)alpha);
  return cudaGetLastError();
}

// Skeleton storage (eq. probnewfac): U = A_[C] V S^{-1} is regenerated from
// the kernel entries A(x, C_c) -- never stored -- folded with the center phase and 1/N.
// Thread per slot; terms in chunks of 16 accumulators (entries recomputed per chunk).
template <typename T2, int QMAX>
__global__ void __launch_bounds__(128) k_rebuild_alpha(OperatorDev op, WedgeDev w, SkelWedge sk, int q,
                                                       const int* __restrict__ slot_x, long long nslots,
                                                       T2* __restrict__ alpha) {
  // Y = V S^{-1} (rc x q) and the skeleton columns C staged once per CTA in shared memory
  extern __shared__ __align__(16) unsigned char rb_smem[];
  double2* Ys = reinterpret_cast<double2*>(rb_smem);
  int* Cs = reinterpret_cast<int*>(Ys + (size_t)sk.rc * q);
  for (int i = threadIdx.x; i < sk.rc * q; i += blockDim.x) Ys[i] = sk.Y[i];
  for (int i = threadIdx.x; i < sk.rc; i += blockDim.x) Cs[i] = sk.C[i];
  __syncthreads();
  const int N = op.N;
  for (long long sl = blockIdx.x * (long long)blockDim.x + threadIdx.x; sl < nslots;
       sl += (long long)gridDim.x * blockDim.x) {
    const int x = slot_x[sl];
    if (x < 0) {
      for (int t = 0; t < q; ++t) alpha[t * nslots + sl] = to_t2<T2>(make_double2(0.0, 0.0));
      continue;
    }
    double y1, y2;
    warped_point(op, x / N, x % N, w, y1, y2);
    double ph = y1 * (double)w.xc1 + y2 * (double)w.xc2;
    ph -= floor(ph);
    double sn, cs;
    sincospi(2.0 * ph, &sn, &cs);
    const double2 e = make_double2(cs / N, sn / N);
    const double c1 = op.c1[x], c2 = op.c2[x];
    double g1, g2;
    grad_rho(c1, c2, w.u1, w.u2, g1, g2);
    double2 acc[QMAX];
#pragma unroll
    for (int k = 0; k < QMAX; ++k) acc[k] = make_double2(0.0, 0.0);
    for (int c = 0; c < sk.rc; ++c) {
      const double2 a = kernel_entry_x(op, x, c1, c2, g1, g2, Cs[c]);
      const double2* yc = Ys + c;
#pragma unroll
      for (int k = 0; k < QMAX; ++k)
        if (k < q) {
          const double2 yv = yc[(long long)k * sk.rc];
          acc[k].x = fma(a.x, yv.x, fma(-a.y, yv.y, acc[k].x));
          acc[k].y = fma(a.x, yv.y, fma(a.y, yv.x, acc[k].y));
        }
    }
#pragma unroll
    for (int k = 0; k < QMAX; ++k)
      if (k < q) alpha[k * nslots + sl] = to_t2<T2>(cmul(acc[k], e));
  }
}

template <typename T2, int QMAX>
static cudaError_t launch_rebuild_q(const OperatorDev& op, const WedgeDev& w, const SkelWedge& sk, int q,
                                    const int* slot_x, long long nslots, T2* alpha, cudaStream_t s) {
  const size_t smem = rebuild_smem_bytes(sk.rc, q);  // attribute set at plan time (configure_rebuild)
  int blocks = (int)std::min<long long>((nslots + 127) / 128, 148LL * 8);
  k_rebuild_alpha<T2, QMAX><<<blocks, 128, smem, s>>>(op, w, sk, q, slot_x, nslots, alpha);
  return cudaGetLastError();
}

size_t rebuild_smem_bytes(int rc, int q) { return sizeof(double2) * (size_t)rc * q + sizeof(int) * (size_t)rc; }

// Opt the rebuild kernels of this dtype into `smem` bytes of dynamic shared memory on the current
// device (cudaFuncSetAttribute is per device: called by every plan for its own device).
cudaError_t configure_rebuild(bool c64, size_t smem) {
  if (smem <= 48 * 1024) return cudaSuccess;
  cudaError_t e;
#define FIO_RBA(QM)                                                                                             \
  e = c64 ? raise_smem_attr((const void*)k_rebuild_alpha<float2, QM>, smem)                                   \
          : raise_smem_attr((const void*)k_rebuild_alpha<double2, QM>, smem);                                   \
  if (e != cudaSuccess) return e;
  FIO_RBA(16)
  FIO_RBA(32)
  FIO_RBA(64)
#undef FIO_RBA
  return cudaSuccess;
}

cudaError_t launch_rebuild_alpha(const OperatorDev& op, const WedgeDev& w, const SkelWedge& sk, int q,
                                 const int* slot_x, long long nslots, void* alpha, bool c64, cudaStream_t s) {
  if (nslots == 0 || q == 0) return cudaSuccess;
  if (q > 64) return cudaErrorInvalidValue;  // plan caps the separation rank far below (r_max / 4 * 3)
#define FIO_RB(QM)                                                                                        \
  return c64 ? launch_rebuild_q<float2, QM>(op, w, sk, q, slot_x, nslots, (float2*)alpha, s)              \
             : launch_rebuild_q<double2, QM>(op, w, sk, q, slot_x, nslots, (double2*)alpha, s);
  if (q <= 16) { FIO_RB(16) }
  if (q <= 32) { FIO_RB(32) }
  FIO_RB(64)
#undef FIO_RB
}

// Fine-grid coordinates u = frac(y_l(x)) (n1f, n2f) of every output point (plan time, FP64).
__global__ void k_fine_coords(OperatorDev op, WedgeDev w, double2* __restrict__ u) {
  const int N = op.N;
  const long long NN = (long long)N * N;
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < NN; x += (long long)gridDim.x * blockDim.x) {
    double y1, y2;
    warped_point(op, (int)(x / N), (int)(x % N), w, y1, y2);
    y1 -= floor(y1);
    y2 -= floor(y2);
    u[x] = make_double2(y1 * w.n1f, y2 * w.n2f);
  }
}

cudaError_t launch_fine_coords(const OperatorDev& op, const WedgeDev& w, double2* u, cudaStream_t s) {
  long long NN = (long long)op.N * op.N;
  int blocks = (int)std::min<long long>((NN + 255) / 256, 148LL * 16);
  k_fine_coords<<<blocks, 256, 0, s>>>(op, w, u);
  return cudaGetLastError();
}

template <typename T2>
__global__ void k_fold_beta(int N, WedgeDev w, const int* __restrict__ members, int n,
                            const double2* __restrict__ beta, int q, const double* __restrict__ d1,
                            const double* __restrict__ d2, const double* __restrict__ chi, T2* __restrict__ betap) {
  long long total = (long long)n * q;
  const long long box = (long long)w.n1 * w.n2;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    int t = (int)(idx % q), j = (int)(idx / q);
    int kf = members[j];
    int k1 = kf / N, k2 = kf - k1 * N;
    int xi1 = k1 >= N / 2 ? k1 - N : k1, xi2 = k2 >= N / 2 ? k2 - N : k2;
    int i1 = w.M[0] * xi1 + w.M[1] * xi2 - w.xc1 + w.n1 / 2;
    int i2 = w.M[2] * xi1 + w.M[3] * xi2 - w.xc2 + w.n2 / 2;
    double2 b = beta[t + (long long)j * q];
    double d = d1[i1] * d2[i2];
    if (chi) d *= chi[j];  // smooth partition weight chi_l(xi) (reading R2)
    betap[t * box + (long long)i1 * w.n2 + i2] = to_t2<T2>(make_double2(b.x * d, b.y * d));
  }
}

cudaError_t launch_fold_beta(int N, const WedgeDev& w, const int* members, int n, const double2* beta, int q,
                             const double* d1, const double* d2, const double* chi, void* betap, bool c64,
                             cudaStream_t s) {
  long long total = (long long)n * q;
  if (total == 0) return cudaSuccess;
  int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
  if (c64)
    k_fold_beta<float2><<<blocks, 256, 0, s>>>(N, w, members, n, beta, q, d1, d2, chi, (float2*)betap);
  else
    k_fold_beta<double2><<<blocks, 256, 0, s>>>(N, w, members, n, beta, q, d1, d2, chi, (double2*)betap);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ shared-memory FFT
// Mixed-radix (4, 2, 3, 5) Stockham autosort FFT on `nseq` sequences of length
// fl.L held in shared memory; element e of sequence b at buf[b*sb + e*si].
// sign = +1: G_j = sum_k c_k e^{+2 pi i jk/L} (the NUFFT's fine grid); -1: DFT.
template <typename T2>
__device__ __forceinline__ T2 mul_i(T2 v, int sign) {  // (sign i) * v
  return sign > 0 ? mk<T2>(-v.y, v.x) : mk<T2>(v.y, -v.x);
}

template <typename T2, int R>
__device__ __forceinline__ void dft_small(T2 (&v)[R], int sign) {
  using Rt = typename Real<T2>::type;
  if constexpr (R == 2) {
    T2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if constexpr (R == 4) {
    T2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
    T2 s13 = cadd(v[1], v[3]), d13 = mul_i(csub(v[1], v[3]), sign);
    v[0] = cadd(s02, s13);
    v[2] = csub(s02, s13);
    v[1] = cadd(d02, d13);
    v[3] = csub(d02, d13);
  } else if constexpr (R == 3) {
    const Rt h = (Rt)0.86602540378443864676;
    T2 t1 = cadd(v[1], v[2]), t2 = csub(v[1], v[2]);
    T2 m = mk<T2>(v[0].x - (Rt)0.5 * t1.x, v[0].y - (Rt)0.5 * t1.y);
    T2 r = mul_i(mk<T2>(h * t2.x, h * t2.y), sign);
    v[0] = cadd(v[0], t1);
    v[1] = cadd(m, r);
    v[2] = csub(m, r);
  } else if constexpr (R == 5) {
    const Rt c1 = (Rt)0.30901699437494742410, c2 = (Rt)-0.80901699437494742410;
    const Rt s1 = (Rt)0.95105651629515357212, s2 = (Rt)0.58778525229247312917;
    T2 a1 = cadd(v[1], v[4]), b1 = csub(v[1], v[4]);
    T2 a2 = cadd(v[2], v[3]), b2 = csub(v[2], v[3]);
    T2 m1 = mk<T2>(v[0].x + c1 * a1.x + c2 * a2.x, v[0].y + c1 * a1.y + c2 * a2.y);
    T2 m2 = mk<T2>(v[0].x + c2 * a1.x + c1 * a2.x, v[0].y + c2 * a1.y + c1 * a2.y);
    T2 r1 = mul_i(mk<T2>(s1 * b1.x + s2 * b2.x, s1 * b1.y + s2 * b2.y), sign);
    T2 r2 = mul_i(mk<T2>(s2 * b1.x - s1 * b2.x, s2 * b1.y - s1 * b2.y), sign);
    v[0] = mk<T2>(v[0].x + a1.x + a2.x, v[0].y + a1.y + a2.y);
    v[1] = cadd(m1, r1);
    v[4] = csub(m1, r1);
    v[2] = cadd(m2, r2);
    v[3] = csub(m2, r2);
  }
}

__device__ __forceinline__ int fdiv(int n, const FastDiv& f) {
  return (int)((__umulhi(f.m, (unsigned)n) + (unsigned)n) >> f.l);
}
__device__ __forceinline__ FastDiv make_fastdiv_dev(unsigned d) {
  unsigned l = 0;
  while ((1ull << l) < d) ++l;
  unsigned long long m = ((((1ull << l) - d) << 32) / d) + 1;
  return FastDiv{(unsigned)m, l, d};
}

// cp.async helpers (K2 input staging, K3 rings)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

#ifndef FIO_K1_THREADS
#define FIO_K1_THREADS 256
#endif
// K1's smem row stride of the last FFT stage (odd: conflict-free transposed read-out; the plan sizes
// K1's shared memory for L + 1 per row, k1_row_bytes)
#ifndef FIO_K1_LD
#define FIO_K1_LD(L) ((L) | 1)
#endif
#ifndef FIO_K2_THREADS
#define FIO_K2_THREADS 256
#endif

// One radix-R Stockham stage over nseq sequences (element e of sequence q at q sb + e si).
// Twiddles w_r = w_1^r: one table (complex128) or SFU (complex64, |error| ~ 1e-6, far below its
// budget) twiddle per butterfly, the others by complex products (c128 K1+K2 2.68 -> 2.37 ms).
template <typename T2, int R>
__device__ __forceinline__ void stockham_stage(const T2* __restrict__ a, T2* __restrict__ b, int L, int Ns,
                                               const FastDiv& dnb, const FastDiv& dns, const T2* __restrict__ tw,
                                               int nseq, int si, int sb, int sign) {
  const int nb = L / R;
  const int span = L / (Ns * R);
  const int total = nseq * nb;
  const float wscale = 6.283185307179586f / (float)L;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    int sq = fdiv(idx, dnb);
    int j = idx - sq * nb;
    int jq = fdiv(j, dns);
    int k = j - jq * Ns;
    const T2* in = a + sq * sb;
    T2* out = b + sq * sb;
    T2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = in[(j + r * nb) * si];
    T2 w1;
    if constexpr (sizeof(T2) == 8) {
      float sn, cs;
      __sincosf(wscale * (float)(k * span), &sn, &cs);
      w1 = mk<T2>(cs, sn);
    } else {
      w1 = tw[k * span];
    }
    if (sign < 0) w1.y = -w1.y;
    T2 wr = w1;
#pragma unroll
    for (int r = 1; r < R; ++r) {
      v[r] = cmul(v[r], wr);
      if (r + 1 < R) wr = cmul(wr, w1);
    }
    dft_small<T2, R>(v, sign);
    int base = jq * Ns * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) out[(base + r * Ns) * si] = v[r];
  }
}

// Returns the buffer holding the result (a or b).  Ends with __syncthreads().
template <typename T2>
__device__ T2* smem_fft(T2* a, T2* b, const FftLen& fl, const T2* tw, int nseq, int si, int sb, int sign) {
  int Ns = 1;
  for (int st = 0; st < fl.nst; ++st) {
    const int R = fl.radix[st];
    const FastDiv& dnb = fl.div_nb[st];
    const FastDiv& dns = fl.div_ns[st];
    switch (R) {
      case 4: stockham_stage<T2, 4>(a, b, fl.L, Ns, dnb, dns, tw, nseq, si, sb, sign); break;
      case 2: stockham_stage<T2, 2>(a, b, fl.L, Ns, dnb, dns, tw, nseq, si, sb, sign); break;
      case 3: stockham_stage<T2, 3>(a, b, fl.L, Ns, dnb, dns, tw, nseq, si, sb, sign); break;
      default: stockham_stage<T2, 5>(a, b, fl.L, Ns, dnb, dns, tw, nseq, si, sb, sign); break;
    }
    __syncthreads();
    T2* t = a;
    a = b;
    b = t;
    Ns *= R;
  }
  return a;
}

// Stockham FFT whose first stage reads its inputs through `load(seq, e)` (e.g. straight from
// global memory, skipping the zero padding) and whose last stage writes through
// `store(seq, e, v)` (e.g. straight to the fine grid); the stages in between ping-pong in shared
// memory (a, b: nseq sequences of length L, stride L).  Same arithmetic as smem_fft.
template <typename T2, int R, class Load, class Store>
__device__ __forceinline__ void stockham_stage_io(int L, int Ns, const FastDiv& dnb, const FastDiv& dns,
                                                  const T2* __restrict__ tw, int nseq, int sign, Load load,
                                                  Store store) {
  const int nb = L / R;
  const int span = fdiv(nb, dns);  // L / (Ns R), exact
  const int total = nseq * nb;
  const float wscale = 6.283185307179586f / (float)L;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int sq = fdiv(idx, dnb);
    const int j = idx - sq * nb;
    const int jq = fdiv(j, dns);
    const int k = j - jq * Ns;
    T2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = load(sq, j + r * nb);
    if (Ns > 1) {  // twiddles w_r = w_1^r (as in stockham_stage)
      T2 w1;
      if constexpr (sizeof(T2) == 8) {
        float sn, cs;
        __sincosf(wscale * (float)(k * span), &sn, &cs);
        w1 = mk<T2>(cs, sn);
      } else {
        w1 = tw[k * span];
      }
      if (sign < 0) w1.y = -w1.y;
      T2 wr = w1;
#pragma unroll
      for (int r = 1; r < R; ++r) {
        v[r] = cmul(v[r], wr);
        if (r + 1 < R) wr = cmul(wr, w1);
      }
    }
    dft_small<T2, R>(v, sign);
    const int base = jq * Ns * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) store(sq, base + r * Ns, v[r]);
  }
}

template <typename T2, class Load, class Store>
__device__ __forceinline__ void stage_dispatch(int R, int L, int Ns, const FastDiv& dnb, const FastDiv& dns,
                                               const T2* tw, int nseq, int sign, Load load, Store store) {
  switch (R) {
    case 4: stockham_stage_io<T2, 4>(L, Ns, dnb, dns, tw, nseq, sign, load, store); break;
    case 2: stockham_stage_io<T2, 2>(L, Ns, dnb, dns, tw, nseq, sign, load, store); break;
    case 3: stockham_stage_io<T2, 3>(L, Ns, dnb, dns, tw, nseq, sign, load, store); break;
    default: stockham_stage_io<T2, 5>(L, Ns, dnb, dns, tw, nseq, sign, load, store); break;
  }
}

// Returns the shared buffer holding the result when the last stage writes to shared memory
// (store_last_to_smem; sequence stride last_ld >= L there, 0 = L), else nullptr.  Ends with
// __syncthreads().
template <typename T2, class LoadFirst, class StoreLast>
__device__ T2* smem_fft_io(T2* a, T2* b, const FftLen& fl, const T2* tw, int nseq, int sign, LoadFirst load_first,
                           StoreLast store_last, bool store_last_to_smem, int last_ld = 0) {
  const int L = fl.L;
  const int ldl = last_ld > 0 ? last_ld : L;
  int Ns = 1;
  T2* in = a;   // unused by stage 0 (reads through load_first)
  T2* out = b;
  for (int st = 0; st < fl.nst; ++st) {
    const int R = fl.radix[st];
    const bool first = st == 0, last = st == fl.nst - 1;
    auto sload = [&](int sq, int e) { return in[sq * L + e]; };
    auto sstore = [&](int sq, int e, T2 v) { out[sq * L + e] = v; };
    auto sstore_ld = [&](int sq, int e, T2 v) { out[sq * ldl + e] = v; };  // the last stage, in smem
    if (first && last && !store_last_to_smem)
      stage_dispatch<T2>(R, L, Ns, fl.div_nb[st], fl.div_ns[st], tw, nseq, sign, load_first, store_last);
    else if (first && last)
      stage_dispatch<T2>(R, L, Ns, fl.div_nb[st], fl.div_ns[st], tw, nseq, sign, load_first, sstore_ld);
    else if (first)
      stage_dispatch<T2>(R, L, Ns, fl.div_nb[st], fl.div_ns[st], tw, nseq, sign, load_first, sstore);
    else if (last && !store_last_to_smem)
      stage_dispatch<T2>(R, L, Ns, fl.div_nb[st], fl.div_ns[st], tw, nseq, sign, sload, store_last);
    else if (last)
      stage_dispatch<T2>(R, L, Ns, fl.div_nb[st], fl.div_ns[st], tw, nseq, sign, sload, sstore_ld);
    else
      stage_dispatch<T2>(R, L, Ns, fl.div_nb[st], fl.div_ns[st], tw, nseq, sign, sload, sstore);
    __syncthreads();
    in = out;
    out = (out == b) ? a : b;
    Ns *= R;
  }
  return store_last_to_smem ? in : nullptr;
}

// ------------------------------------------------------------------ K0: input spectrum
// Rows of length L (row-major, row stride L): out = FFT_sign(in) * scale.
template <typename T2>
__global__ void __launch_bounds__(256) k_fft_rows(const T2* __restrict__ in, T2* __restrict__ out, int nrows,
                                                  int rows_per_cta, const FftLen* __restrict__ ffts, int fidx,
                                                  const T2* __restrict__ tw, int sign, double scale) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const FftLen& fl = ffts[fidx];
  const int L = fl.L;
  const int r0 = blockIdx.x * rows_per_cta;
  const int nr = min(rows_per_cta, nrows - r0);
  if (nr <= 0) return;
  T2* a = reinterpret_cast<T2*>(smem_raw);
  T2* b = a + rows_per_cta * L;
  for (int idx = threadIdx.x; idx < nr * L; idx += blockDim.x) a[idx] = in[(long long)r0 * L + idx];
  __syncthreads();
  T2* res = smem_fft<T2>(a, b, fl, tw + fl.tw_off, nr, 1, L, sign);
  using Rt = typename Real<T2>::type;
  const Rt sc = (Rt)scale;
  for (int idx = threadIdx.x; idx < nr * L; idx += blockDim.x) {
    T2 v = res[idx];
    out[(long long)r0 * L + idx] = mk<T2>(v.x * sc, v.y * sc);
  }
}

// Columns [c0, c0 + C) of an L x ncols row-major array, FFT along the rows index.
template <typename T2>
__global__ void __launch_bounds__(256) k_fft_cols(const T2* __restrict__ in, T2* __restrict__ out, int ncols,
                                                  int cols_per_cta, const FftLen* __restrict__ ffts, int fidx,
                                                  const T2* __restrict__ tw, int sign, double scale) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const FftLen& fl = ffts[fidx];
  const int L = fl.L;
  const int c0 = blockIdx.x * cols_per_cta;
  const int C = min(cols_per_cta, ncols - c0);
  if (C <= 0) return;
  T2* a = reinterpret_cast<T2*>(smem_raw);
  T2* b = a + cols_per_cta * L;
  for (int idx = threadIdx.x; idx < L * C; idx += blockDim.x) {
    int i = idx / C, c = idx - i * C;
    a[i * C + c] = in[(long long)i * ncols + c0 + c];
  }
  __syncthreads();
  T2* res = smem_fft<T2>(a, b, fl, tw + fl.tw_off, C, C, 1, sign);
  using Rt = typename Real<T2>::type;
  const Rt sc = (Rt)scale;
  for (int idx = threadIdx.x; idx < L * C; idx += blockDim.x) {
    int i = idx / C, c = idx - i * C;
    T2 v = res[i * C + c];
    out[(long long)i * ncols + c0 + c] = mk<T2>(v.x * sc, v.y * sc);
  }
}

__device__ __forceinline__ int imod(int a, int n) {
  int r = a % n;
  return r < 0 ? r + n : r;
}

// ------------------------------------------------------------------ K1: window x beta + row FFT
// Job (w, t, start, count): box rows i1 in [start, start + count) of wedge w, term t.
// h(i1, i2) = beta'_lt(i1, i2) fhat(M^{-1}(k' + xi_c)), k' = (i1 - n1/2, i2 - n2/2),
// placed at fine index k'_2 mod n2f, then H = FFT_{+}(h) along axis 2.  The result is
// written TRANSPOSED, p1[t][j2][i1] (row length n1), so that K2 reads contiguous columns.
template <typename T2>
__global__ void __launch_bounds__(FIO_K1_THREADS) k_rowpass(int N, const WedgeDev* __restrict__ wedges,
                                                 const FftJob* __restrict__ jobs, const FftLen* __restrict__ ffts,
                                                 const T2* __restrict__ tw, const T2* const* __restrict__ betas,
                                                 const T2* __restrict__ fhat, T2* __restrict__ p1) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const FftJob job = jobs[blockIdx.x];
  const WedgeDev& w = wedges[job.w];
  const FftLen& fl = ffts[job.fft];
  const int L = fl.L, n1 = w.n1, n2 = w.n2, cnt = job.count;
  // the last stage writes its rows with an odd stride: the transposed read-out below (consecutive
  // threads: consecutive rows, same column) is then free of shared-memory bank conflicts
  const int ld = FIO_K1_LD(L);
  T2* a = reinterpret_cast<T2*>(smem_raw);
  T2* b = a + cnt * ld;
  const T2* bet = betas[job.w] + ((long long)job.t * n1 + job.start) * n2;
  {  // the job's beta' rows are one contiguous block of cnt n2 elements: stage it in the first buffer
    const int nel = cnt * n2;
    if constexpr (sizeof(T2) == 16) {
      for (int e = threadIdx.x; e < nel; e += blockDim.x) cp_async16(a + e, bet + e);
    } else {
      for (int e = threadIdx.x; e < nel; e += blockDim.x) cp_async8(a + e, bet + e);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    bet = a;
  }
  const int hi = n2 - n2 / 2;  // fine index pos = k'_2 mod L holds box column i2 = k'_2 + n2/2
  // The first Stockham stage reads h straight from beta' and fhat (no zero fill / placement pass).
  const int h2 = n2 / 2, lo2 = L - h2;
  const int m0 = w.Mi[0], m1 = w.Mi[1], m2 = w.Mi[2], m3 = w.Mi[3];
  const int zb1 = job.start - n1 / 2 + w.xc1, zb2 = w.xc2 - h2;
  const bool pow2 = (N & (N - 1)) == 0;
  auto fidx = [&](int r, int i2) {
    const int z1 = zb1 + r, z2 = zb2 + i2;
    const int xi1 = m0 * z1 + m1 * z2, xi2 = m2 * z1 + m3 * z2;
    const int r1 = pow2 ? (xi1 & (N - 1)) : imod(xi1, N), r2 = pow2 ? (xi2 & (N - 1)) : imod(xi2, N);
    return r1 * N + r2;
  };
  auto load_h = [&](int r, int pos) -> T2 {
    const int i2 = pos < hi ? pos + h2 : pos - lo2;  // box column (valid iff pos < hi or pos >= L - n2/2)
    T2 out = mk<T2>(0, 0);
    if (pos < hi || pos >= lo2) {
      const T2 bv = bet[r * n2 + i2];
      if (bv.x != 0 || bv.y != 0) out = cmul(bv, fhat[fidx(r, i2)]);
    }
    return out;
  };
  auto no_store = [](int, int, T2) {};
  T2* res = smem_fft_io<T2>(a, b, fl, tw + fl.tw_off, cnt, +1, load_h, no_store, true, ld);
  T2* dst = p1 + w.p1_off + (long long)job.t * L * n1 + job.start;
  const FastDiv dc = make_fastdiv_dev((unsigned)cnt);
  for (int idx = threadIdx.x; idx < cnt * L; idx += blockDim.x) {  // consecutive threads: consecutive i1
    const int j2 = fdiv(idx, dc), r = idx - j2 * cnt;
    dst[(long long)j2 * n1 + r] = res[r * ld + j2];
  }
}

// ------------------------------------------------------------------ K2: column FFT -> fine grid
// Job (w, t, c0, C): fine columns j2 in [c0, c0 + C).  Column j2 of the row-pass output
// (contiguous in p1) is placed at fine index (i1 - n1/2) mod n1f and transformed
// (FFT_{+}, length n1f).  The fine grid is stored TRANSPOSED with a periodic halo on
// its contiguous axis: G_lt[j2][kHalo + j1] (row length n1f + 2 kHalo), the layout K3
// reads (K3's rows are j2, its columns j1).
template <typename T2>
__global__ void __launch_bounds__(FIO_K2_THREADS) k_colpass(const WedgeDev* __restrict__ wedges, const FftJob* __restrict__ jobs,
                                                 const FftLen* __restrict__ ffts, const T2* __restrict__ tw,
                                                 const T2* __restrict__ p1, T2* __restrict__ g) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const FftJob job = jobs[blockIdx.x];
  const WedgeDev& w = wedges[job.w];
  const FftLen& fl = ffts[job.fft];
  const int L = fl.L, n1 = w.n1, C = job.count, c0 = job.start;
  T2* a = reinterpret_cast<T2*>(smem_raw);
  T2* b = a + C * L;
  const T2* src = p1 + w.p1_off + ((long long)job.t * w.n2f + c0) * n1;
  const int hi = n1 - n1 / 2;  // fine index pos = (i1 - n1/2) mod L
  // the job's input is one contiguous block of C n1 elements: copy it into the (not yet used) first
  // ping-pong buffer with cp.async -- every thread keeps several copies in flight -- and let the
  // first Stockham stage read it from shared memory
  {
    const int nel = C * n1;
    if constexpr (sizeof(T2) == 16) {
      for (int e = threadIdx.x; e < nel; e += blockDim.x) cp_async16(a + e, src + e);
    } else {
      for (int e = threadIdx.x; e < nel; e += blockDim.x) cp_async8(a + e, src + e);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
  }
  const T2* srcs = a;
  // First stage reads the row-pass output; last stage writes the haloed fine-grid row.
  const int h1 = n1 / 2, lo1 = L - h1;
  auto load_p = [&](int c, int pos) -> T2 {
    const int i1 = pos < hi ? pos + h1 : pos - lo1;  // valid iff pos < hi or pos >= L - n1/2
    T2 out = mk<T2>(0, 0);
    if (pos < hi || pos >= lo1) out = srcs[c * n1 + i1];
    return out;
  };
  const int rowp = L + 2 * kHalo;
  T2* dst = g + w.g_off + ((long long)job.t * w.n2f + c0) * rowp + kHalo;
  auto store_g = [&](int c, int j1, T2 v) {
    T2* rp = dst + (long long)c * rowp;
    rp[j1] = v;
    if (j1 < kHalo) rp[L + j1] = v;
    if (j1 >= L - kHalo) rp[j1 - L] = v;
  };
  smem_fft_io<T2>(a, b, fl, tw + fl.tw_off, C, +1, load_p, store_g, false);
}

// ------------------------------------------------------------------ K3: interpolation + alpha epilogue
// c + a * (b.x, b.y) as one packed FFMA2 (sm_100 fma.rn.f32x2)
__device__ __forceinline__ float2 ffma2(float a, float2 b, float2 c) {
  float2 r;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %2};\n\tmov.b64 rb, {%3, %4};\n\tmov.b64 rc, {%5, %6};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}
__device__ __forceinline__ float2 cfma_real(float a, float2 b, float2 c) { return ffma2(a, b, c); }
// a * (x, x) + c as one packed FFMA2
__device__ __forceinline__ float2 ffma2_v(float2 a, float x, float2 c) { return ffma2(x, a, c); }
__device__ __forceinline__ double2 cfma_real(double a, double2 b, double2 c) {
  return make_double2(fma(a, b.x, c.x), fma(a, b.y, c.y));
}

// Interpolation weights of P points along one axis: w[k][i] for the window
// positions i < NW of the point at offset o_k = u_k - anchor.  The point's first tap sits at window
// position d_k = [o_k > TAPS/2] (always 0 when NW == TAPS: the axis has no run), tap j at distance
// s_k - j, s_k = o_k - d_k, with phi(s_k - j) = sum_{m <= DEG} c[j][m] x_k^m,
// x_k = 2 (s_k - TAPS/2) + 1 (the plan's piecewise polynomial of the ES kernel, EsPoly, fitted at
// exactly degree DEG = k3_poly_deg(TAPS)).  Coefficient-outer Horner: each coefficient is read once
// per call (uniform) and applied to all P points.  FP32 (two taps per packed FFMA2) for complex64,
// FP64 for complex128; the adjoint calls the same functions, so it stays the exact transpose.
template <int TAPS, int NW, int P>
__device__ __forceinline__ void axis_weights(const float (&o)[P], const EsPoly& poly, float (&w)[P][NW]) {
  constexpr int NP = (TAPS + 1) / 2;  // tap pairs
  constexpr int DEG = k3_poly_deg(TAPS);
  float x[P];
  bool d[P];
#pragma unroll
  for (int k = 0; k < P; ++k) {
    d[k] = NW > TAPS && o[k] > 0.5f * TAPS;
    x[k] = 2.f * (o[k] - (d[k] ? 1.f : 0.f) - 0.5f * TAPS) + 1.f;
  }
  float2 qv[P][NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const float2 c = make_float2(poly.cf[DEG][2 * p], poly.cf[DEG][2 * p + 1]);
#pragma unroll
    for (int k = 0; k < P; ++k) qv[k][p] = c;
  }
#pragma unroll
  for (int m = DEG - 1; m >= 0; --m) {
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const float2 c = make_float2(poly.cf[m][2 * p], poly.cf[m][2 * p + 1]);
#pragma unroll
      for (int k = 0; k < P; ++k) qv[k][p] = ffma2_v(qv[k][p], x[k], c);
    }
  }
#pragma unroll
  for (int k = 0; k < P; ++k) {
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      const float a = i < TAPS ? (i % 2 ? qv[k][(i < TAPS ? i : 0) / 2].y : qv[k][(i < TAPS ? i : 0) / 2].x) : 0.f;
      const int im = i >= 1 ? i - 1 : 0;
      const float b = (i >= 1 && i - 1 < TAPS) ? (im % 2 ? qv[k][(i - 1 < TAPS ? im : 0) / 2].y
                                                         : qv[k][(i - 1 < TAPS ? im : 0) / 2].x)
                                               : 0.f;
      w[k][i] = d[k] ? b : a;
    }
  }
}

template <int TAPS, int NW, int P>
__device__ __forceinline__ void axis_weights(const double (&o)[P], const EsPoly& poly, double (&w)[P][NW]) {
  constexpr int DEG = k3_poly_deg(TAPS);
  double x[P];
  bool d[P];
#pragma unroll
  for (int k = 0; k < P; ++k) {
    d[k] = NW > TAPS && o[k] > 0.5 * TAPS;
    x[k] = 2.0 * (o[k] - (d[k] ? 1.0 : 0.0) - 0.5 * TAPS) + 1.0;
  }
  double qv[P][TAPS];
#pragma unroll
  for (int j = 0; j < TAPS; ++j) {
    const double c = poly.c[j][DEG];
#pragma unroll
    for (int k = 0; k < P; ++k) qv[k][j] = c;
  }
#pragma unroll
  for (int m = DEG - 1; m >= 0; --m) {
#pragma unroll
    for (int j = 0; j < TAPS; ++j) {
      const double c = poly.c[j][m];
#pragma unroll
      for (int k = 0; k < P; ++k) qv[k][j] = fma(qv[k][j], x[k], c);
    }
  }
#pragma unroll
  for (int k = 0; k < P; ++k) {
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      const double a = i < TAPS ? qv[k][i < TAPS ? i : 0] : 0.0;
      const double b = (i >= 1 && i - 1 < TAPS) ? qv[k][(i >= 1 && i - 1 < TAPS) ? i - 1 : 0] : 0.0;
      w[k][i] = d[k] ? b : a;
    }
  }
}

template <typename T2> struct OffT;
template <> struct OffT<float2> { using type = float2; };
template <> struct OffT<double2> { using type = double2; };

template <typename T2, int TAPS> struct GroupP { static constexpr int value = group_p(sizeof(T2) == 8, TAPS); };

// K3 launch shape: threads per CTA (= groups per chunk) and the CTAs per SM the registers allow
template <typename T2> struct K3Cfg;
template <> struct K3Cfg<float2> {
#ifndef FIO_K3_MINB64
#define FIO_K3_MINB64 10
#endif
#ifndef FIO_K3_TT64
#define FIO_K3_TT64 1
#endif
  // TT terms per step of the term loop (interleaved: more independent FMA chains per row); the ring
  // holds two steps (the one computed and the one in flight)
  // 10 CTAs per SM (102 registers) measured 5 % faster than 8 at N = 1024 for w <= 8 (the c64 range
  // the eps floor allows); wider windows take 8 or 6, which they need to stay free of spills
#ifndef FIO_K3_ST64
#define FIO_K3_ST64 (2 * FIO_K3_TT64)
#endif
#ifndef FIO_K3_RP64
#define FIO_K3_RP64 2
#endif
  static constexpr int BLOCK = kK3BlockC64, TT = FIO_K3_TT64, STAGES = FIO_K3_ST64, RP = FIO_K3_RP64;
  static constexpr int minb(int taps) { return taps <= 8 ? FIO_K3_MINB64 : (taps <= 10 ? 8 : 6); }
  static_assert(kK3TileCapC64 % (2 * BLOCK) == 0, "tile cap: a whole number of 16-byte units per thread");
};
template <> struct K3Cfg<double2> {
#ifndef FIO_K3_MINB128
#define FIO_K3_MINB128 4
#endif
#ifndef FIO_K3_TT128
#define FIO_K3_TT128 1
#endif
#ifndef FIO_K3_ST128
#define FIO_K3_ST128 (2 * FIO_K3_TT128)
#endif
#ifndef FIO_K3_RP128
#define FIO_K3_RP128 2
#endif
  static constexpr int BLOCK = kK3BlockC128, TT = FIO_K3_TT128, STAGES = FIO_K3_ST128, RP = FIO_K3_RP128;
  static constexpr int minb(int) { return FIO_K3_MINB128; }
  static_assert(kK3TileCapC128 % BLOCK == 0, "tile cap: a whole number of 16-byte units per thread");
};

// Shared memory of K3 (16-aligned sections).  Per-point arrays are element-major with the thread
// index innermost -- [k][thread] -- the same order the plan stores them in global memory inside each
// chunk (k3_slot): the CTA copies a chunk's block with coalesced 16-byte cp.async units and a warp's
// loads of element k hit 32 consecutive words (no bank conflicts):
//   alpha' ring   [S][P][BLOCK] T2          the chunk's alpha'(t) for the S terms in flight
//   row weights   [WINR][P/RPV][BLOCK]x16B  phi1 of every point (FP32 c64, FP64 c128), thread-written
//   running sums  [P][BLOCK] T2             Lf(x_k) before this wedge (cp.async gathers)
//   slots         [2][P][BLOCK] int         output index of every point (current, next chunk)
//   offsets       [P][BLOCK] O2             fine-grid offsets from the anchor (next chunk)
//   anchors       [BLOCK] int2              (next chunk)
//   boxes         [2][kBoxInts] int         footprint box of the current and the next chunk
//   tile ring     [S][cap] T2               the chunk's footprint tile of G_lt per term in flight
// FIO_K3_P1REG: the row weights stay in registers for the chunk (no shared-memory reloads per term;
// c64 K3 2.08 -> 1.93 ms, c128 10.04 -> 9.87 ms at N = 1024) wherever they fit without spills
// (ptxas -v, all instantiations): otherwise they stay in shared memory
#ifndef FIO_K3_P1REG
#define FIO_K3_P1REG 1
#endif
constexpr bool k3_p1reg(bool c64, int taps, int nr) {
  return FIO_K3_P1REG && (c64 ? (nr == 1 ? (taps <= 5 || (taps >= 9 && taps <= 11)) : (taps <= 7 || taps >= 9))
                              : (nr == 1 ? taps <= 9 : taps <= 7));
}
template <typename T2, int TAPS, int P, int NR = 1>
struct K3Layout {  // NR right-hand sides: NR running-sum buffers, NR tiles per ring stage
  using Rt = typename Real<T2>::type;
  static constexpr int BLOCK = K3Cfg<T2>::BLOCK;
  static constexpr int WINR = k3_window_rows(TAPS, sizeof(T2) == 8);
  static constexpr size_t al(size_t b) { return (b + 15) / 16 * 16; }
  static constexpr size_t kRing = 0;
  static constexpr size_t kP1 = kRing + al(sizeof(T2) * K3Cfg<T2>::STAGES * BLOCK * P);
  static constexpr bool PREG = k3_p1reg(sizeof(T2) == 8, TAPS, NR);  // row weights in registers
  static constexpr size_t kLf = kP1 + (PREG ? 0 : al(sizeof(Rt) * WINR * BLOCK * P));
  static constexpr size_t kSlot = kLf + al(sizeof(T2) * BLOCK * P * NR);
  static constexpr size_t kOff = kSlot + al(sizeof(int) * 2 * BLOCK * P);
  static constexpr size_t kAnchor = kOff + al(sizeof(typename OffT<T2>::type) * BLOCK * P);
  static constexpr size_t kBox = kAnchor + al(sizeof(int2) * BLOCK);
  static constexpr size_t kBar = kBox + al(sizeof(int) * 2 * kBoxInts);
  // the tile ring: 128-byte aligned (TMA destination); the plan rounds the slot size (tile_cap) to
  // a multiple of 128 bytes
  static constexpr size_t kFixed = (kBar + al(8 * (K3Cfg<T2>::STAGES + 2)) + 127) / 128 * 128;
  static size_t bytes(long long cap) { return kFixed + sizeof(T2) * K3Cfg<T2>::STAGES * NR * (size_t)cap; }
};

// ---- the TMA engine (cp.async.bulk) for K3's contiguous alpha' blocks, completing on mbarriers
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared, `bytes` (multiple of 16, both addresses 16-byte aligned), completing on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// FIO_K3_L2HINT: L2 eviction priorities for K3's streams -- alpha' blocks and chunk tables are read
// exactly once (evict_first), the fine-grid tiles are re-read by neighbouring chunks (evict_last), so the
// 14 GB alpha' stream does not push a wedge's ~31 MB of G out of the 126 MB L2
#ifndef FIO_K3_L2HINT
#define FIO_K3_L2HINT 1
#endif
__device__ __forceinline__ unsigned long long l2_policy_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long l2_policy_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
// bulk_g2s with an L2 cache policy
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                              unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void cp_async16_hint(void* smem, const void* gmem, unsigned long long pol) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "l"(pol) : "memory");
}
// TMA tensor copy: the box at (x, y, z) of a 3-D tensor map into shared memory, completing on `bar`
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* map, int x, int y, int z,
                                                 unsigned long long* bar, unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3, %4}], [%5], %6;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// `bytes` (a multiple of 16) from global to shared memory by the whole CTA, 16-byte cp.async units
template <int BLOCK>
__device__ __forceinline__ void cta_copy16(void* dst, const void* src, int bytes) {
  char* d = static_cast<char*>(dst);
  const char* s = static_cast<const char*>(src);
  for (int u = threadIdx.x; u < bytes / 16; u += BLOCK) cp_async16(d + 16 * u, s + 16 * u);
}

// The right-hand sides one K3 launch serves (NEXT-2: one alpha' pass for NR inputs): per RHS its fine
// grids, its spectrum (DC term) and its output / running sum.
constexpr int kK3MaxRhs = 2;
template <typename T2>
struct K3Rhs {
  const T2* g[kK3MaxRhs];
  const T2* fhat[kK3MaxRhs];
  T2* Lf[kK3MaxRhs];
};

// K3: one CTA processes chunks of BLOCK consecutive groups (one group of up to P points per thread;
// chunks are padded to BLOCK groups at plan time, so chunk c's groups are [c BLOCK, (c+1) BLOCK)).
// Per chunk every thread evaluates the interpolation weights of its points once -- column weights
// phi2 in registers, row weights phi1 in shared memory -- and starts the copy of its points' running
// sums Lf(x_k); then, for every term t, the CTA stages with cp.async the chunk's footprint tile of
// G_lt (rows wrapped mod the fine grid, columns from the haloed row layout; every thread copies a
// fixed set of 16-byte units whose addresses it computes once per chunk) and the chunk's alpha'(t)
// block into a K3Cfg::STAGES-deep ring, so global latency overlaps the arithmetic of earlier terms.
// Per group, term and window row i the thread loads the row once and applies it to all P points:
//   F_k += phi1_k[i] sum_j phi2_k[j] G_lt[a1 + i][a2 + j]
//   acc_k += alpha'_lt(x_k) F_k
// The next chunk's tables (anchors, box, slots, offsets) are prefetched during the current one.
// Lf[x_k] is written (first wedge of the stream, + the DC term of rank 0) or read-modify-written:
// each point occurs in exactly one group per wedge, so one launch per wedge is race-free and the
// summation order over wedges is fixed (deterministic).  With NR > 1 right-hand sides (fio_apply_batch)
// the weights, tables and alpha'(t) blocks of a chunk serve all of them: per term the CTA stages NR
// tiles and every RHS runs the same arithmetic as a single apply (bit-identical results).
template <typename T2, int TAPS, int P, int NR>
__global__ void __launch_bounds__(K3Cfg<T2>::BLOCK, NR == 1 ? K3Cfg<T2>::minb(TAPS)
                                                          : K3Cfg<T2>::minb(TAPS) - (sizeof(T2) == 8 ? 2 : 1))
    k_interp_groups(InterpWedge iw, K3Rhs<T2> rhs, const double2* __restrict__ a0, int first, int add_dc,
                    EsPoly poly, const __grid_constant__ CUtensorMap tmap) {
  static_assert(NR >= 1 && NR <= kK3MaxRhs, "K3 right-hand sides");
  using Rt = typename Real<T2>::type;
  using O2 = typename OffT<T2>::type;
  using L = K3Layout<T2, TAPS, P, NR>;
  constexpr bool C64 = sizeof(T2) == 8;
  constexpr int WIN = k3_window_cols(TAPS, C64);
  constexpr int WINR = k3_window_rows(TAPS, C64);
  constexpr int BLOCK = K3Cfg<T2>::BLOCK;
  constexpr int S = K3Cfg<T2>::STAGES;
  constexpr int TT = K3Cfg<T2>::TT;
  constexpr int RP = K3Cfg<T2>::RP;
  constexpr int LA = S - TT;  // terms staged ahead of the step being computed
  static_assert(LA >= TT, "K3 ring: at least one step in flight");
  constexpr int EPC = 16 / (int)sizeof(T2);  // complex elements per 16-byte unit
  constexpr int RPV = 16 / (int)sizeof(Rt);  // row weights per 16-byte unit
  constexpr int MAXC = C64 ? kK3TileCapC64 / 2 / BLOCK : kK3TileCapC128 / BLOCK;  // tile units per thread
  static_assert(P % RPV == 0, "K3 group size");
  extern __shared__ __align__(128) unsigned char k3_smem[];
  T2* aring = reinterpret_cast<T2*>(k3_smem + L::kRing);
  unsigned char* p1s = k3_smem + L::kP1;
  T2* lfb = reinterpret_cast<T2*>(k3_smem + L::kLf);
  int* m_slot = reinterpret_cast<int*>(k3_smem + L::kSlot);
  O2* m_off = reinterpret_cast<O2*>(k3_smem + L::kOff);
  int2* m_anchor = reinterpret_cast<int2*>(k3_smem + L::kAnchor);
  int* sbox = reinterpret_cast<int*>(k3_smem + L::kBox);
  unsigned long long* bar_a = reinterpret_cast<unsigned long long*>(k3_smem + L::kBar);  // [S] alpha' blocks
  T2* tring = reinterpret_cast<T2*>(k3_smem + L::kFixed);
  const int tid = threadIdx.x;
  const int cap = iw.tile_cap;
  const int nrow = iw.nrow, n2p = iw.ncolp, q = iw.q;  // K3 rows / haloed row length of G_lt
  const long long gstride = (long long)nrow * n2p;
  const long long nslots = (long long)iw.ngroups * P;
  const T2* G[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) G[r] = rhs.g[r] + iw.g_off + kHalo;
  const T2* __restrict__ alpha = reinterpret_cast<const T2*>(iw.alpha);
  const O2* __restrict__ offs = reinterpret_cast<const O2*>(iw.slot_off);
  constexpr int kA = sizeof(int2) * BLOCK, kB = sizeof(int) * kBoxInts, kS = sizeof(int) * BLOCK * P,
                kO = sizeof(O2) * BLOCK * P, kAl = sizeof(T2) * BLOCK * P;
  unsigned long long* bar_m = bar_a + S;  // [2] chunk tables
  // the chunk's tables are four contiguous blocks: four bulk copies (TMA engine) by thread 0
  auto prefetch_meta = [&](int chn, int buf) {
    if (chn < iw.nchunks && tid == 0) {
      const long long c0 = (long long)chn * BLOCK * P;  // first physical slot of the chunk
      mbar_expect_tx(bar_m + buf, (unsigned)(kA + kB + kS + kO));
      if (FIO_K3_L2HINT) {
        const unsigned long long pf = l2_policy_first();
        bulk_g2s_hint(m_anchor, iw.anchor + 2 * (long long)chn * BLOCK, kA, bar_m + buf, pf);
        bulk_g2s_hint(sbox + kBoxInts * buf, iw.box + (long long)kBoxInts * chn, kB, bar_m + buf, pf);
        bulk_g2s_hint(m_slot + buf * BLOCK * P, iw.slot_x + c0, kS, bar_m + buf, pf);
        bulk_g2s_hint(m_off, offs + c0, kO, bar_m + buf, pf);
      } else {
      bulk_g2s(m_anchor, iw.anchor + 2 * (long long)chn * BLOCK, kA, bar_m + buf);
      bulk_g2s(sbox + kBoxInts * buf, iw.box + (long long)kBoxInts * chn, kB, bar_m + buf);
      bulk_g2s(m_slot + buf * BLOCK * P, iw.slot_x + c0, kS, bar_m + buf);
      bulk_g2s(m_off, offs + c0, kO, bar_m + buf);
      }
    }
  };
  if (tid == 0) {
    for (int st = 0; st < S + 2; ++st) mbar_init(bar_a + st, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  unsigned gterm = 0;  // terms this CTA has staged before the current chunk (ring slot / mbarrier phase)
  prefetch_meta(blockIdx.x, 0);
  int it = 0;
  for (int ch = blockIdx.x; ch < iw.nchunks; ch += gridDim.x, ++it) {
    const int buf = it & 1;
    mbar_wait(bar_m + buf, (unsigned)(it >> 1) & 1u);
    __syncthreads();  // this chunk's tables are visible; every thread is done with the previous chunk
    const int* cb = sbox + kBoxInts * buf;  // first group, row origin, column origin, rows, columns, groups
    const int br = cb[1], bc = cb[2], bnr = cb[3], bnc = cb[4];
    const int sst = cb[6];      // row stride of the tile in shared memory (>= bnc, chosen at plan time)
    const bool tma = NR == 1 && iw.tma && cb[7];  // the tile by one TMA request per term (plan-time choice)
    const int cpr = bnc / EPC;  // 16-byte units per tile row
    const int tchunks = bnr * cpr;
    const T2* __restrict__ al = alpha + (long long)ch * BLOCK * P;
    // this thread's share of every tile copy, fixed for the chunk: source offsets within G_lt (row
    // wrapped mod the fine grid) and destination offsets within the tile
    int csrc[MAXC], cdst[MAXC];
    int ncp = 0;
#pragma unroll
    for (int u = 0; u < MAXC; ++u) {
      const int idx = tid + u * BLOCK;
      csrc[u] = 0;
      cdst[u] = 0;
      if (!tma && idx < tchunks) {  // (TMA chunks copy their tile without per-thread addresses)
        const int rr = idx / cpr, cc = idx - rr * cpr;
        int r = br + rr;
        r = r < 0 ? r + nrow : (r >= nrow ? r - nrow : r);
        csrc[u] = r * n2p + bc + cc * EPC;
        cdst[u] = rr * sst + cc * EPC;
        ncp = u + 1;
      }
    }
    // the running sums Lf(x_k) of this thread's points, gathered while the term loop runs
    if (!first) {
#pragma unroll
      for (int k = 0; k < P; ++k) {
        const int x = m_slot[(buf * P + k) * BLOCK + tid];
        if (x >= 0) {
#pragma unroll
          for (int r = 0; r < NR; ++r) {
            if constexpr (C64)
              cp_async8(lfb + (r * P + k) * BLOCK + tid, rhs.Lf[r] + x);
            else
              cp_async16(lfb + (r * P + k) * BLOCK + tid, rhs.Lf[r] + x);
          }
        }
      }
    }
    // stage term t into ring slot t % S: the chunk's alpha'(t) block and the tile
    // the chunk's alpha'(t) block is contiguous: one bulk copy (TMA engine) on the stage's mbarrier;
    // the tile (short scattered rows) by cp.async from every thread
    auto issue = [&](int t, bool next_meta) {
      if (t < q) {
        const int st = (int)((gterm + t) % S);
        if (tma) {  // alpha'(t) and the tile (the fixed TMA box at the chunk's origin) on one mbarrier
          if (tid == 0) {
            constexpr int kTile = (C64 ? kK3BoxRows64 * kK3BoxCols64 : kK3BoxRows128 * kK3BoxCols128) * sizeof(T2);
            mbar_expect_tx(bar_a + st, (unsigned)(kAl + kTile));
            if (FIO_K3_L2HINT) {
              bulk_g2s_hint(aring + st * BLOCK * P, al + t * nslots, (unsigned)kAl, bar_a + st, l2_policy_first());
              tma_load_3d_hint(tring + st * NR * cap, &tmap, (bc + kHalo) * (int)(sizeof(T2) / 8), br, t, bar_a + st,
                               l2_policy_last());
            } else {
            bulk_g2s(aring + st * BLOCK * P, al + t * nslots, (unsigned)kAl, bar_a + st);
            tma_load_3d(tring + st * NR * cap, &tmap, (bc + kHalo) * (int)(sizeof(T2) / 8), br, t, bar_a + st);
            }
          }
        } else {
        if (tid == 0) {
          mbar_expect_tx(bar_a + st, (unsigned)kAl);
          if (FIO_K3_L2HINT)
            bulk_g2s_hint(aring + st * BLOCK * P, al + t * nslots, (unsigned)kAl, bar_a + st, l2_policy_first());
          else
            bulk_g2s(aring + st * BLOCK * P, al + t * nslots, (unsigned)kAl, bar_a + st);
        }
        const unsigned long long pl = FIO_K3_L2HINT ? l2_policy_last() : 0ull;
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          const T2* __restrict__ gt = G[r] + t * gstride;
          T2* tile = tring + (st * NR + r) * cap;
#pragma unroll
          for (int u = 0; u < MAXC; ++u)
            if (u < ncp) {
              if (FIO_K3_L2HINT)
                cp_async16_hint(tile + cdst[u], gt + csrc[u], pl);
              else
                cp_async16(tile + cdst[u], gt + csrc[u]);
            }
        }
        }
      }
      // the next chunk's tables, issued once every thread has consumed the current offsets/anchors
      if (next_meta) prefetch_meta(ch + gridDim.x, buf ^ 1);
      cp_async_commit();
    };
#pragma unroll
    for (int u = 0; u < LA; ++u) issue(u, false);
    // weights of this thread's points: phi2 (columns) in registers, phi1 (rows) in shared memory
    const int2 an = m_anchor[tid];
    const int woff = (an.x - br) * sst + (an.y - bc);
    Rt p2[P][WIN];
    constexpr bool PREG = L::PREG;
    Rt p1r[P][PREG ? WINR : 1];  // row weights kept in registers (k3_p1reg)
    {
      Rt o1[P], o2[P];
#pragma unroll
      for (int k = 0; k < P; ++k) {
        const O2 o = m_off[k * BLOCK + tid];
        o1[k] = o.x;
        o2[k] = o.y;
      }
      {
        Rt w1[P][WINR];
        axis_weights<TAPS, WINR, P>(o1, poly, w1);
        if constexpr (PREG) {
#pragma unroll
          for (int k = 0; k < P; ++k)
#pragma unroll
            for (int i = 0; i < WINR; ++i) p1r[k][i] = w1[k][i];
        } else
#pragma unroll
        for (int i = 0; i < WINR; ++i)
#pragma unroll
          for (int cc = 0; cc < P / RPV; ++cc) {
            if constexpr (sizeof(Rt) == 4)
              *reinterpret_cast<float4*>(p1s + ((i * (P / RPV) + cc) * BLOCK + tid) * 16) =
                  make_float4(w1[4 * cc][i], w1[4 * cc + 1][i], w1[4 * cc + 2][i], w1[4 * cc + 3][i]);
            else
              *reinterpret_cast<double2*>(p1s + ((i * (P / RPV) + cc) * BLOCK + tid) * 16) =
                  make_double2(w1[2 * cc][i], w1[2 * cc + 1][i]);
          }
      }
      axis_weights<TAPS, WIN, P>(o2, poly, p2);
    }
    if (q == 0) {  // no term loop: fetch the next chunk's tables here
      __syncthreads();
      prefetch_meta(ch + gridDim.x, buf ^ 1);
    }
    T2 acc[NR][P];
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
      for (int k = 0; k < P; ++k) acc[r][k] = mk<T2>(0, 0);
    for (int t0 = 0; t0 < q; t0 += TT) {
      // step: terms t0 .. t0 + TT - 1 (those < q); their tiles are the only copies in flight
      cp_async_wait<LA - TT>();  // this step's tiles (the newer LA - TT terms may stay in flight)
#pragma unroll
      for (int u = 0; u < TT; ++u)
        if (t0 + u < q) mbar_wait(bar_a + (gterm + t0 + u) % S, (unsigned)((gterm + t0 + u) / S) & 1u);
      __syncthreads();  // this step staged by every thread; every thread is done with the previous step
#pragma unroll
      for (int u = 0; u < TT; ++u) issue(t0 + LA + u, t0 == 0 && u == 0);
#pragma unroll
      for (int rh = 0; rh < NR; ++rh) {  // right-hand side rh: its tiles, the shared weights and alpha'
      const T2* __restrict__ win[TT];
#pragma unroll
      for (int u = 0; u < TT; ++u) win[u] = tring + ((int)((gterm + t0 + u) % S) * NR + rh) * cap + woff;
      T2 F[TT][P];
#pragma unroll
      for (int u = 0; u < TT; ++u)
#pragma unroll
        for (int k = 0; k < P; ++k) F[u][k] = mk<T2>(0, 0);
      // RP window rows per iteration: RP independent column sums per point in flight (latency hiding;
      // the same operations in the same order, so the results do not depend on RP)
#pragma unroll
      for (int i0 = 0; i0 < WINR; i0 += RP) {
        Rt w1[RP][P];
#pragma unroll
        for (int r = 0; r < RP; ++r) {
          if (i0 + r >= WINR) continue;
          const int i = i0 + r;
          if constexpr (PREG) {
#pragma unroll
            for (int k = 0; k < P; ++k) w1[r][k] = p1r[k][i];
          } else {
#pragma unroll
            for (int cc = 0; cc < P / RPV; ++cc) {
              if constexpr (sizeof(Rt) == 4) {
                const float4 a = *reinterpret_cast<const float4*>(p1s + ((i * (P / RPV) + cc) * BLOCK + tid) * 16);
                w1[r][4 * cc] = a.x; w1[r][4 * cc + 1] = a.y; w1[r][4 * cc + 2] = a.z; w1[r][4 * cc + 3] = a.w;
              } else {
                const double2 a = *reinterpret_cast<const double2*>(p1s + ((i * (P / RPV) + cc) * BLOCK + tid) * 16);
                w1[r][2 * cc] = a.x; w1[r][2 * cc + 1] = a.y;
              }
            }
          }
        }
#pragma unroll
        for (int u = 0; u < TT; ++u) {
          if (TT > 1 && t0 + u >= q) continue;  // uniform: the last step may be partial
          T2 v[RP][WIN];
#pragma unroll
          for (int r = 0; r < RP; ++r) {
            if (i0 + r >= WINR) continue;
            const int i = i0 + r;
            if constexpr (C64 && WIN % 2 == 0) {  // complex64: even anchors -> 16-byte aligned pairs
              const float4* wp = reinterpret_cast<const float4*>(win[u] + i * sst);
#pragma unroll
              for (int jj = 0; jj < WIN / 2; ++jj) {
                const float4 a = wp[jj];
                v[r][2 * jj] = mk<T2>(a.x, a.y);
                v[r][2 * jj + 1] = mk<T2>(a.z, a.w);
              }
            } else {
#pragma unroll
              for (int jj = 0; jj < WIN; ++jj) v[r][jj] = win[u][i * sst + jj];
            }
          }
#pragma unroll
          for (int k = 0; k < P; ++k) {
            T2 rr[RP];
#pragma unroll
            for (int r = 0; r < RP; ++r) rr[r] = mk<T2>(0, 0);
#pragma unroll
            for (int jj = 0; jj < WIN; ++jj)
#pragma unroll
              for (int r = 0; r < RP; ++r)
                if (i0 + r < WINR) rr[r] = cfma_real(p2[k][jj], v[r][jj], rr[r]);
#pragma unroll
            for (int r = 0; r < RP; ++r)
              if (i0 + r < WINR) F[u][k] = cfma_real(w1[r][k], rr[r], F[u][k]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < TT; ++u) {
        if (TT > 1 && t0 + u >= q) continue;
        const T2* ring = aring + (int)((gterm + t0 + u) % S) * BLOCK * P + tid;
#pragma unroll
        for (int k = 0; k < P; ++k) {
          const T2 av = ring[k * BLOCK];
          acc[rh][k].x = fma(av.x, F[u][k].x, fma(-av.y, F[u][k].y, acc[rh][k].x));
          acc[rh][k].y = fma(av.x, F[u][k].y, fma(av.y, F[u][k].x, acc[rh][k].y));
        }
      }
      }  // right-hand sides
    }
    gterm += q;
    cp_async_wait<0>();  // the running sums (in the first copy group) have landed
#pragma unroll
    for (int rh = 0; rh < NR; ++rh) {
      T2 f0 = mk<T2>(0, 0);
      if (first && add_dc) f0 = rhs.fhat[rh][0];
#pragma unroll
      for (int k = 0; k < P; ++k) {
        const int x = m_slot[(buf * P + k) * BLOCK + tid];
        if (x < 0) continue;
        T2 b0 = mk<T2>(0, 0);
        if (!first) {
          b0 = lfb[(rh * P + k) * BLOCK + tid];
        } else if (add_dc) {
          const double2 d = a0[x];
          b0 = mk<T2>((Rt)(d.x * (double)f0.x - d.y * (double)f0.y), (Rt)(d.x * (double)f0.y + d.y * (double)f0.x));
        }
        rhs.Lf[rh][x] = mk<T2>(b0.x + acc[rh][k].x, b0.y + acc[rh][k].y);
      }
    }
  }
}

// Lf = a(x,0) fhat(0) / N (rank 0) or 0: used only when this rank owns no wedge.
template <typename T2>
__global__ void k_dc_only(int N, const double2* __restrict__ a0, const T2* __restrict__ fhat, int add_dc,
                          T2* __restrict__ Lf) {
  using Rt = typename Real<T2>::type;
  const long long NN = (long long)N * N;
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < NN; x += (long long)gridDim.x * blockDim.x) {
    T2 v = mk<T2>(0, 0);
    if (add_dc) {
      double2 d = a0[x];
      T2 f0 = fhat[0];
      v = mk<T2>((Rt)(d.x * (double)f0.x - d.y * (double)f0.y), (Rt)(d.x * (double)f0.y + d.y * (double)f0.x));
    }
    Lf[x] = v;
  }
}

// Lf += acc[0] + ... + acc[n-1] (the other streams' partial sums of K3, fixed order)
template <typename T2>
__global__ void k_accum(T2* __restrict__ Lf, const T2* __restrict__ a0, const T2* __restrict__ a1,
                        const T2* __restrict__ a2, int n, long long NN) {
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < NN; x += (long long)gridDim.x * blockDim.x) {
    T2 u = Lf[x];
    const T2 v = a0[x];
    u.x += v.x;
    u.y += v.y;
    if (n > 1) {
      const T2 w = a1[x];
      u.x += w.x;
      u.y += w.y;
    }
    if (n > 2) {
      const T2 w = a2[x];
      u.x += w.x;
      u.y += w.y;
    }
    Lf[x] = u;
  }
}

template <typename T2, int TAPS, int P, int NR>
static cudaError_t launch_groups_tpr(const ApplyArgs& a, const InterpWedge& iw, const K3Rhs<T2>& rhs, int first,
                                     int add_dc, const CUtensorMap& tmap, cudaStream_t s) {
  constexpr int BLOCK = K3Cfg<T2>::BLOCK;
  // the plan opted this instance into its largest footprint's smem on its device (configure_interp)
  const size_t smem = K3Layout<T2, TAPS, P, NR>::bytes(iw.tile_cap);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_interp_groups<T2, TAPS, P, NR>, BLOCK, smem);
  per_sm = std::max(per_sm, 1);
  const int blocks = std::max(1, std::min(iw.nchunks, per_sm * a.sms));
  k_interp_groups<T2, TAPS, P, NR><<<blocks, BLOCK, smem, s>>>(iw, rhs, a.a0, first, add_dc, *a.poly, tmap);
  return cudaGetLastError();
}

template <typename T2, int TAPS, int P>
static cudaError_t launch_groups_tp(const ApplyArgs& a, const InterpWedge& iw, const K3Rhs<T2>& rhs, int nr,
                                    int first, int add_dc, const CUtensorMap& tmap, cudaStream_t s) {
  return nr == 2 ? launch_groups_tpr<T2, TAPS, P, 2>(a, iw, rhs, first, add_dc, tmap, s)
                 : launch_groups_tpr<T2, TAPS, P, 1>(a, iw, rhs, first, add_dc, tmap, s);
}

template <typename T2, int TAPS>
static cudaError_t configure_interp_tp(long long tile_cap) {
  constexpr int P = GroupP<T2, TAPS>::value;
  cudaError_t e = raise_smem_attr((const void*)k_interp_groups<T2, TAPS, P, 1>, K3Layout<T2, TAPS, P, 1>::bytes(tile_cap));
  if (e != cudaSuccess) return e;
  return raise_smem_attr((const void*)k_interp_groups<T2, TAPS, P, 2>, K3Layout<T2, TAPS, P, 2>::bytes(tile_cap));
}

cudaError_t configure_interp(int taps, bool c64, long long max_tile_cap) {
#define FIO_CFG_CASE(TP) \
  case TP:               \
    return c64 ? configure_interp_tp<float2, TP>(max_tile_cap) : configure_interp_tp<double2, TP>(max_tile_cap);
  switch (taps) {
    FIO_CFG_CASE(3)
    FIO_CFG_CASE(4)
    FIO_CFG_CASE(5)
    FIO_CFG_CASE(6)
    FIO_CFG_CASE(7)
    FIO_CFG_CASE(8)
    FIO_CFG_CASE(9)
    FIO_CFG_CASE(10)
    FIO_CFG_CASE(11)
    FIO_CFG_CASE(12)
    default: return cudaErrorInvalidValue;
  }
#undef FIO_CFG_CASE
}

template <typename T2>
static cudaError_t launch_groups(const ApplyArgs& a, const InterpWedge& iw, const K3Rhs<T2>& rhs, int nr, int first,
                                 int add_dc, const CUtensorMap& tmap, cudaStream_t s) {
#define FIO_GROUPS_CASE(TP) \
  case TP:                  \
    return launch_groups_tp<T2, TP, GroupP<T2, TP>::value>(a, iw, rhs, nr, first, add_dc, tmap, s);
  switch (a.taps) {
    FIO_GROUPS_CASE(3)
    FIO_GROUPS_CASE(4)
    FIO_GROUPS_CASE(5)
    FIO_GROUPS_CASE(6)
    FIO_GROUPS_CASE(7)
    FIO_GROUPS_CASE(8)
    FIO_GROUPS_CASE(9)
    FIO_GROUPS_CASE(10)
    FIO_GROUPS_CASE(11)
    FIO_GROUPS_CASE(12)
    default: return cudaErrorInvalidValue;
  }
#undef FIO_GROUPS_CASE
}

// K3 of the whole apply: one launch per owned wedge, alternating between the caller's stream (into Lf)
// and the plan's side stream (into the second accumulator), so one wedge's tail and the next one's
// start overlap; the two partial sums are added in a fixed order (deterministic).  Skeleton storage:
// alpha' is first regenerated into the stream's scratch.  One alpha' serves every right-hand side.
template <typename T2>
static cudaError_t launch_interp(const ApplyArgs* args, int nrhs, T2* Lf0, cudaStream_t s, int* n) {
  const ApplyArgs& a = args[0];
  const long long NN = (long long)a.N * a.N;
  cudaError_t e;
  if (a.nw == 0) {
    int blocks = (int)std::min<long long>((NN + 255) / 256, 148LL * 8);
    for (int b = 0; b < nrhs; ++b) {
      k_dc_only<T2><<<blocks, 256, 0, s>>>(a.N, a.a0, reinterpret_cast<const T2*>(args[b].fhat), a.add_dc,
                                            Lf0 + b * NN);
      ++*n;
    }
    return cudaGetLastError();
  }
  const int ns = a.nw > 1 && a.side[0] ? 2 : 1;
  if (ns > 1) {
    if ((e = cudaEventRecord(a.fork, s)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(a.side[0], a.fork, 0)) != cudaSuccess) return e;
  }
  for (int wi = 0; wi < a.nw; ++wi) {
    const int sj = wi % ns;
    cudaStream_t sw = sj ? a.side[0] : s;
    const InterpWedge& iw = a.iw[wi];
    if (a.skel) {
      e = launch_rebuild_alpha(a.op, a.wd_host[wi], a.skel[wi], iw.q, iw.slot_x,
                               (long long)iw.ngroups * group_p(sizeof(T2) == 8, a.taps), const_cast<void*>(iw.alpha),
                               sizeof(T2) == sizeof(float2), sw);
      if (e != cudaSuccess) return e;
      ++*n;
    }
    // up to k3_rhs right-hand sides per launch: one pass over the wedge's alpha' serves them all
    for (int b = 0; b < nrhs;) {
      // (w > 7 would spill with two right-hand sides' accumulators: one at a time there)
      const int nr = a.taps > 7 ? 1 : std::max(1, std::min({a.k3_rhs, kK3MaxRhs, nrhs - b}));
      K3Rhs<T2> rhs{};
      for (int r = 0; r < nr; ++r) {
        rhs.g[r] = reinterpret_cast<const T2*>(args[b + r].g);
        rhs.fhat[r] = reinterpret_cast<const T2*>(args[b + r].fhat);
        rhs.Lf[r] = sj ? reinterpret_cast<T2*>(args[b + r].acc[0]) : Lf0 + (b + r) * NN;
      }
      // TMA tiles read the plan's own fine grids: the first right-hand side of a single apply only
      InterpWedge iwl = iw;
      iwl.tma = (a.tmaps && nr == 1 && rhs.g[0] == reinterpret_cast<const T2*>(a.g)) ? iw.tma : 0;
      const CUtensorMap tm = iwl.tma ? a.tmaps[wi] : CUtensorMap{};
      if ((e = launch_groups<T2>(a, iwl, rhs, nr, wi < ns, (wi == 0 && a.add_dc) ? 1 : 0, tm, sw)) != cudaSuccess)
        return e;
      ++*n;
      b += nr;
    }
  }
  if (ns > 1) {
    if ((e = cudaEventRecord(a.join[0], a.side[0])) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(s, a.join[0], 0)) != cudaSuccess) return e;
    const int accb = (int)std::min<long long>((NN + 255) / 256, 148LL * 8);
    for (int b = 0; b < nrhs; ++b) {
      const T2* acc1 = reinterpret_cast<const T2*>(args[b].acc[0]);
      k_accum<T2><<<accb, 256, 0, s>>>(Lf0 + b * NN, acc1, acc1, acc1, 1, NN);
      ++*n;
    }
  }
  return cudaGetLastError();
}

// ================================================================== adjoint
// The exact conjugate transpose of the discrete fast forward operator above:
//   K3*  spread: G*_lt[cell] += sum_points phi(x, cell) conj(alpha'_lt(x)) g(x)   (NUFFT type 1)
//   K2*  per fine row j2: fold halos, FFT_{-} (length n1f), keep box indices -> P1*[t][j2][i1]
//   K1*  per box row i1: FFT_{-} (length n2f) of P1*[t][.][i1], keep box indices,
//        fhat*(xi) = sum_t conj(beta'_lt) h*_t  (each xi belongs to one wedge and one box cell)
//   DC   fhat*(0) = sum_x conj(a(x,0)/N) g(x)
//   K0*  L* g = (1/N) sum_xi e^{+2 pi i x.xi} fhat*(xi)
// K3* accumulates with global RED atomics (native on sm_100a; the shared-memory float atomic
// is a CAS loop), so its summation order -- and the last bits of the adjoint -- can vary
// from run to run.
// one vector RED (REDG.E.ADD.F32x2) for complex64; two FP64 REDs for complex128
__device__ __forceinline__ void red_add(float2* p, float2 v) { atomicAdd(p, v); }
__device__ __forceinline__ void red_add(double2* p, double2 v) {
  atomicAdd(&p->x, v.x);
  atomicAdd(&p->y, v.y);
}

template <typename T2>
__device__ __forceinline__ T2 shfl_down_t2(T2 v, int d) {
  T2 r;
  r.x = __shfl_down_sync(0xffffffffu, v.x, d);
  r.y = __shfl_down_sync(0xffffffffu, v.y, d);
  return r;
}

// K3*: one thread per half group of PH = min(P, 4) points (persistent grid-stride loop, whole warps
// iterate together; PH keeps both weight sets in registers).  Lanes whose windows share an anchor
// (the two halves of a group, and neighbouring groups with the same anchor, consecutive in the
// group order) are summed with a segmented shuffle reduction first, so only the segment head issues
// the RED atomics for each window cell.
template <typename T2, int TAPS, int P>
__global__ void __launch_bounds__(128) k_spread_groups(InterpWedge iw, T2* __restrict__ gstar,
                                                       const T2* __restrict__ g, EsPoly poly) {
  using Rt = typename Real<T2>::type;
  using O2 = typename OffT<T2>::type;
  constexpr int PH = P < 4 ? P : 4;
  constexpr int SPLIT = P / PH;
  static_assert(P % PH == 0, "group size");
  constexpr int WIN = k3_window_cols(TAPS, sizeof(T2) == 8);
  constexpr int WINR = k3_window_rows(TAPS, sizeof(T2) == 8);
  const int n1f = iw.nrow, n2p = iw.ncolp, q = iw.q;
  const long long gstride = (long long)n1f * n2p;
  const long long nslots = (long long)iw.ngroups * P;
  T2* __restrict__ G = gstar + iw.g_off + kHalo;
  const T2* __restrict__ alpha = reinterpret_cast<const T2*>(iw.alpha);
  const O2* __restrict__ offs = reinterpret_cast<const O2*>(iw.slot_off);
  const int lane = threadIdx.x & 31;
  const int stride = gridDim.x * blockDim.x;
  const int nvg = iw.ngroups * SPLIT;
  // whole warps step through the half groups so that the shuffles below see converged warps
  for (int base = (blockIdx.x * blockDim.x + threadIdx.x) - lane; base < nvg; base += stride) {
    const int vg = base + lane;
    const bool valid = vg < nvg;
    const int grp = valid ? vg / SPLIT : 0;
    const int k0 = (vg - grp * SPLIT) * PH;  // this thread's points: k0 .. k0 + PH - 1 of the group
    constexpr int BLK = K3Cfg<T2>::BLOCK;    // slots in K3's physical layout (k3_slot)
    int a1 = 0, a2 = 0;
    if (valid) {
      a1 = iw.anchor[2 * grp];
      a2 = iw.anchor[2 * grp + 1];
    }
    // segment = run of consecutive lanes with the same anchor; run_len = lanes from me to the run end
    const unsigned long long key = valid ? (((unsigned long long)(unsigned)a1 << 32) | (unsigned)a2) : ~0ull;
    const unsigned same = __match_any_sync(0xffffffffu, key);
    const unsigned above = same >> lane;                   // bit 0 = me
    // contiguous lanes from me with my key (all 32: ~above == 0, where __ffs would give 0)
    const int run = above == 0xffffffffu ? 32 : __ffs(~above) - 1;
    const bool head = lane == 0 || !((same >> (lane - 1)) & 1u);
    int maxrun = run;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) maxrun = max(maxrun, __shfl_xor_sync(0xffffffffu, maxrun, d));
    const int r0 = a1 < 0 ? a1 + n1f : a1;
    Rt p1[PH][WINR], p2[PH][WIN], o1[PH], o2[PH];
    T2 gx[PH];
#pragma unroll
    for (int k = 0; k < PH; ++k) {
      int x = -1;
      O2 o;
      o.x = (Rt)(0.5 * TAPS);
      o.y = (Rt)(0.5 * TAPS);
      if (valid) {
        const long long sl = k3_slot(grp, k0 + k, P, BLK);
        x = iw.slot_x[sl];
        o = offs[sl];
      }
      gx[k] = x >= 0 ? g[x] : mk<T2>(0, 0);
      o1[k] = o.x;
      o2[k] = o.y;
    }
    // the same weights (same function, same precision) as K3: the adjoint stays the exact
    // conjugate transpose of the forward operator
    axis_weights<TAPS, WINR, PH>(o1, poly, p1);
    axis_weights<TAPS, WIN, PH>(o2, poly, p2);
    T2 anext[sizeof(T2) == 8 ? PH : 1];  // c64: alpha'(t+1), loaded one term ahead
    if constexpr (sizeof(T2) == 8) {
#pragma unroll
      for (int k = 0; k < PH; ++k) anext[k] = (valid && q > 0) ? alpha[k3_slot(grp, k0 + k, P, BLK)] : mk<T2>(0, 0);
    }
    for (int t = 0; t < q; ++t) {
      T2 c[PH];
#pragma unroll
      for (int k = 0; k < PH; ++k) {
        // conj(alpha') g; alpha' one term ahead for c64, at use for c128 (ahead: 52.7 vs 48.3 ms)
        T2 av;
        if constexpr (sizeof(T2) == 8)
          av = anext[k];
        else
          av = valid ? alpha[t * nslots + k3_slot(grp, k0 + k, P, BLK)] : mk<T2>(0, 0);
        c[k] = mk<T2>(av.x * gx[k].x + av.y * gx[k].y, av.x * gx[k].y - av.y * gx[k].x);
      }
      if constexpr (sizeof(T2) == 8) {
        if (t + 1 < q && valid) {
#pragma unroll
          for (int k = 0; k < PH; ++k) anext[k] = alpha[(t + 1) * nslots + k3_slot(grp, k0 + k, P, BLK)];
        }
      }
      T2* __restrict__ rp = G + t * gstride + (long long)r0 * n2p + a2;
      int r = r0;
#pragma unroll 1
      for (int i = 0; i < WINR; ++i) {
        T2 e[PH];
#pragma unroll
        for (int k = 0; k < PH; ++k) e[k] = mk<T2>(p1[k][i] * c[k].x, p1[k][i] * c[k].y);
        T2 v[WIN];
#pragma unroll
        for (int j = 0; j < WIN; ++j) {
          v[j] = mk<T2>(0, 0);
#pragma unroll
          for (int k = 0; k < PH; ++k) v[j] = cfma_real(p2[k][j], e[k], v[j]);
        }
        // segmented sum toward the run head over the whole window row at once (WIN independent
        // shuffle chains per step): after the steps d < maxrun the head holds the run total
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          if (d >= maxrun) break;  // warp-uniform
#pragma unroll
          for (int j = 0; j < WIN; ++j) {
            const T2 u = shfl_down_t2(v[j], d);
            if (d < run) v[j] = cadd(v[j], u);
          }
        }
        if (head && valid) {
#pragma unroll
          for (int j = 0; j < WIN; ++j) red_add(rp + j, v[j]);
        }
        rp += (r + 1 == n1f) ? -(long long)(n1f - 1) * n2p : (long long)n2p;
        r = (r + 1 == n1f) ? 0 : r + 1;
      }
    }
  }
}

// K2*: job (w, t, c0, C) over fine rows j2 in [c0, c0 + C) of G*_lt.
template <typename T2>
__global__ void __launch_bounds__(256) k_colpass_adj(const WedgeDev* __restrict__ wedges,
                                                     const FftJob* __restrict__ jobs, const FftLen* __restrict__ ffts,
                                                     const T2* __restrict__ tw, const T2* __restrict__ g,
                                                     T2* __restrict__ p1) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const FftJob job = jobs[blockIdx.x];
  const WedgeDev& w = wedges[job.w];
  const FftLen& fl = ffts[job.fft];
  const int L = fl.L, n1 = w.n1, C = job.count, c0 = job.start;
  const int Lp = L;
  T2* a = reinterpret_cast<T2*>(smem_raw);
  T2* b = a + C * Lp;
  const int rowp = L + 2 * kHalo;
  const T2* src = g + w.g_off + ((long long)job.t * w.n2f + c0) * rowp + kHalo;
  for (int c = 0; c < C; ++c) {
    const T2* rp = src + (long long)c * rowp;
    for (int j1 = threadIdx.x; j1 < L; j1 += blockDim.x) {
      T2 v = rp[j1];
      if (j1 < kHalo) v = cadd(v, rp[L + j1]);        // right halo holds columns 0..kHalo-1
      if (j1 >= L - kHalo) v = cadd(v, rp[j1 - L]);   // left halo holds columns L-kHalo..L-1
      a[c * Lp + j1] = v;
    }
  }
  __syncthreads();
  T2* res = smem_fft<T2>(a, b, fl, tw + fl.tw_off, C, 1, Lp, -1);
  T2* dst = p1 + w.p1_off + ((long long)job.t * w.n2f + c0) * n1;
  for (int c = 0; c < C; ++c)
    for (int i1 = threadIdx.x; i1 < n1; i1 += blockDim.x) {
      int pos = i1 - n1 / 2;
      pos = pos < 0 ? pos + L : pos;
      dst[(long long)c * n1 + i1] = res[c * Lp + pos];
    }
}

// K1*: job (w, -, start, count) over box rows i1, all terms t in-CTA (deterministic sum over t).
template <typename T2>
__global__ void __launch_bounds__(256) k_rowpass_adj(int N, const WedgeDev* __restrict__ wedges,
                                                     const FftJob* __restrict__ jobs, const FftLen* __restrict__ ffts,
                                                     const T2* __restrict__ tw, const T2* const* __restrict__ betas,
                                                     const unsigned char* const* __restrict__ masks,
                                                     const T2* __restrict__ p1, T2* __restrict__ fhat,
                                                     int accumulate) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const FftJob job = jobs[blockIdx.x];
  const WedgeDev& w = wedges[job.w];
  const FftLen& fl = ffts[job.fft];
  const int L = fl.L, n1 = w.n1, n2 = w.n2, cnt = job.count;
  const int Lp = L;
  T2* a = reinterpret_cast<T2*>(smem_raw);
  T2* b = a + cnt * Lp;
  T2* acc = b + cnt * Lp;
  for (int idx = threadIdx.x; idx < cnt * n2; idx += blockDim.x) acc[idx] = mk<T2>(0, 0);
  const FastDiv dc = make_fastdiv_dev((unsigned)cnt);
  for (int t = 0; t < w.q; ++t) {
    const T2* src = p1 + w.p1_off + (long long)t * L * n1 + job.start;
    __syncthreads();
    for (int idx = threadIdx.x; idx < cnt * L; idx += blockDim.x) {
      const int j2 = fdiv(idx, dc), r = idx - j2 * cnt;
      a[r * Lp + j2] = src[(long long)j2 * n1 + r];
    }
    __syncthreads();
    T2* res = smem_fft<T2>(a, b, fl, tw + fl.tw_off, cnt, 1, Lp, -1);
    const T2* bet = betas[job.w] + ((long long)t * n1 + job.start) * n2;
    for (int r = 0; r < cnt; ++r)
      for (int i2 = threadIdx.x; i2 < n2; i2 += blockDim.x) {
        const T2 bv = bet[r * n2 + i2];
        int pos = i2 - n2 / 2;
        pos = pos < 0 ? pos + L : pos;
        const T2 h = res[r * Lp + pos];
        T2 v = acc[r * n2 + i2];
        v.x += bv.x * h.x + bv.y * h.y;  // conj(beta') h
        v.y += bv.x * h.y - bv.y * h.x;
        acc[r * n2 + i2] = v;
      }
  }
  __syncthreads();
  const unsigned char* mk_ = masks[job.w] + (long long)job.start * n2;
  for (int r = 0; r < cnt; ++r)
    for (int i2 = threadIdx.x; i2 < n2; i2 += blockDim.x) {
      if (!mk_[r * n2 + i2]) continue;
      const int kp1 = job.start + r - n1 / 2, kp2 = i2 - n2 / 2;
      const int z1 = kp1 + w.xc1, z2 = kp2 + w.xc2;
      const int xi1 = w.Mi[0] * z1 + w.Mi[1] * z2, xi2 = w.Mi[2] * z1 + w.Mi[3] * z2;
      T2* dst = fhat + (long long)imod(xi1, N) * N + imod(xi2, N);
      if (accumulate)  // smooth partition: up to two wedges carry this xi (fhat* zeroed first)
        red_add(dst, acc[r * n2 + i2]);
      else
        *dst = acc[r * n2 + i2];  // indicator wedges: each xi belongs to exactly one wedge
    }
}

// fhat*(0) = sum_x conj(a0(x)) g(x): one CTA, fixed-order tree reduction in FP64.
template <typename T2>
__global__ void __launch_bounds__(1024) k_dc_adj(long long NN, const double2* __restrict__ a0,
                                                 const T2* __restrict__ g, T2* __restrict__ fhat) {
  __shared__ double sr[1024], si[1024];
  double r = 0, im = 0;
  for (long long x = threadIdx.x; x < NN; x += blockDim.x) {
    const double2 d = a0[x];
    const double gr = (double)g[x].x, gi = (double)g[x].y;
    r += d.x * gr + d.y * gi;
    im += d.x * gi - d.y * gr;
  }
  sr[threadIdx.x] = r;
  si[threadIdx.x] = im;
  __syncthreads();
  for (int h = blockDim.x / 2; h > 0; h >>= 1) {
    if (threadIdx.x < h) {
      sr[threadIdx.x] += sr[threadIdx.x + h];
      si[threadIdx.x] += si[threadIdx.x + h];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) fhat[0] = mk<T2>((typename Real<T2>::type)sr[0], (typename Real<T2>::type)si[0]);
}

template <typename T2, int TAPS, int P>
static cudaError_t launch_spread_tp(const ApplyArgs& a, int wi, const T2* g, cudaStream_t s) {
  const InterpWedge& iw = a.iw[wi];
  const int nvg = iw.ngroups * (P / (P < 4 ? P : 4));
  int blocks = std::max(1, std::min((nvg + 127) / 128, a.sms * 8));
  k_spread_groups<T2, TAPS, P><<<blocks, 128, 0, s>>>(iw, reinterpret_cast<T2*>(a.g), g, *a.poly);
  return cudaGetLastError();
}

template <typename T2>
static cudaError_t enqueue_adjoint_t(const ApplyArgs& a, const T2* g, T2* out, cudaStream_t s, int* launches) {
  cudaError_t e;
  int n = 0;
  const bool c64 = sizeof(T2) == sizeof(float2);
  const T2* tw = reinterpret_cast<const T2*>(a.tw);
  T2* fhat = reinterpret_cast<T2*>(a.fhat);
  T2* tmp = reinterpret_cast<T2*>(a.tmp);
  const long long NN = (long long)a.N * a.N;
  if ((e = cudaMemsetAsync(fhat, 0, sizeof(T2) * NN, s)) != cudaSuccess) return e;
  if (a.nw > 0) {
    if ((e = cudaMemsetAsync(a.g, 0, sizeof(T2) * a.fine_elems, s)) != cudaSuccess) return e;
    // the wedges' spreads write disjoint G*_l: they alternate between the caller's stream and the
    // plan's side stream (not in skeleton mode, whose alpha' scratch is shared)
    const bool two = a.side[0] != nullptr && a.nw >= 2;  // skeleton: 2 scratches
    if (two) {
      if ((e = cudaEventRecord(a.fork, s)) != cudaSuccess) return e;
      if ((e = cudaStreamWaitEvent(a.side[0], a.fork, 0)) != cudaSuccess) return e;
    }
    for (int wi = 0; wi < a.nw; ++wi) {
      cudaStream_t sw = (two && (wi & 1)) ? a.side[0] : s;
      if (a.skel) {
        const InterpWedge& iw = a.iw[wi];
        e = launch_rebuild_alpha(a.op, a.wd_host[wi], a.skel[wi], iw.q, iw.slot_x,
                                 (long long)iw.ngroups * group_p(sizeof(T2) == 8, a.taps), const_cast<void*>(iw.alpha), c64, sw);
        if (e != cudaSuccess) return e;
        ++n;
      }
#define FIO_SPREAD_CASE(TP)                                   \
  case TP:                                                    \
    e = launch_spread_tp<T2, TP, GroupP<T2, TP>::value>(a, wi, g, sw); \
    break;
      switch (a.taps) {
        FIO_SPREAD_CASE(3)
        FIO_SPREAD_CASE(4)
        FIO_SPREAD_CASE(5)
        FIO_SPREAD_CASE(6)
        FIO_SPREAD_CASE(7)
        FIO_SPREAD_CASE(8)
        FIO_SPREAD_CASE(9)
        FIO_SPREAD_CASE(10)
        FIO_SPREAD_CASE(11)
        FIO_SPREAD_CASE(12)
        default: return cudaErrorInvalidValue;
      }
#undef FIO_SPREAD_CASE
      if (e != cudaSuccess) return e;
      ++n;
    }
    if (two) {
      if ((e = cudaEventRecord(a.join[0], a.side[0])) != cudaSuccess) return e;
      if ((e = cudaStreamWaitEvent(s, a.join[0], 0)) != cudaSuccess) return e;
    }
    k_colpass_adj<T2><<<a.njobs_col, 256, a.smem_col, s>>>(a.wedges, a.jobs_col, a.ffts, tw,
                                                           reinterpret_cast<const T2*>(a.g),
                                                           reinterpret_cast<T2*>(a.p1));
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ++n;
    const T2* const* betas = reinterpret_cast<const T2* const*>(a.beta);
    k_rowpass_adj<T2><<<a.njobs_rowadj, 256, a.smem_rowadj, s>>>(a.N, a.wedges, a.jobs_rowadj, a.ffts, tw, betas,
                                                                a.masks, reinterpret_cast<const T2*>(a.p1), fhat,
                                                                a.overlap);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ++n;
  }
  if (a.add_dc) {
    k_dc_adj<T2><<<1, 1024, 0, s>>>(NN, a.a0, g, fhat);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ++n;
  }
  // K0*: out = (1/N) sum_xi e^{+2 pi i x.xi} fhat*(xi)
  const size_t seq = fft_seq_bytes(a.N, c64);
  int rpc = a.rows_per_cta_N;
  k_fft_rows<T2><<<(a.N + rpc - 1) / rpc, 256, rpc * seq, s>>>(fhat, tmp, a.N, rpc, a.ffts, a.fft_N, tw, +1, 1.0);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  int cpc = a.cols_per_cta_N;
  k_fft_cols<T2><<<(a.N + cpc - 1) / cpc, 256, cpc * seq, s>>>(tmp, out, a.N, cpc, a.ffts, a.fft_N, tw, +1,
                                                               1.0 / a.N);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  n += 2;
  if (launches) *launches = n;
  return cudaSuccess;
}

cudaError_t enqueue_adjoint(const ApplyArgs& a, bool c64, const void* g, void* out, cudaStream_t s, int* launches) {
  if (c64) return enqueue_adjoint_t<float2>(a, (const float2*)g, (float2*)out, s, launches);
  return enqueue_adjoint_t<double2>(a, (const double2*)g, (double2*)out, s, launches);
}

size_t k1_row_bytes(int L, bool c64) { return fft_seq_bytes(L + 1, c64); }

size_t fft_seq_bytes(int L, bool c64) {
  return c64 ? 2 * (size_t)L * sizeof(float2)
             : 2 * (size_t)L * sizeof(double2);
}

cudaError_t configure_kernels(size_t smem_bytes) {
  cudaError_t e;
#define FIO_SMEM(K)                                                                          \
  e = raise_smem_attr((const void*)K, smem_bytes);                                           \
  if (e != cudaSuccess) return e;
  FIO_SMEM(k_fft_rows<double2>)
  FIO_SMEM(k_fft_rows<float2>)
  FIO_SMEM(k_fft_cols<double2>)
  FIO_SMEM(k_fft_cols<float2>)
  FIO_SMEM(k_rowpass<double2>)
  FIO_SMEM(k_rowpass<float2>)
  FIO_SMEM(k_colpass<double2>)
  FIO_SMEM(k_colpass<float2>)
  FIO_SMEM(k_rowpass_adj<double2>)
  FIO_SMEM(k_rowpass_adj<float2>)
  FIO_SMEM(k_colpass_adj<double2>)
  FIO_SMEM(k_colpass_adj<float2>)
#undef FIO_SMEM
  return cudaSuccess;
}

template <typename T2>
static cudaError_t enqueue_apply_t(const ApplyArgs* args, int nrhs, const T2* f0, T2* Lf, cudaStream_t s,
                                   int* launches, cudaEvent_t* ev) {
  cudaError_t e;
  int n = 0;
  int stage = 0;
  auto mark = [&]() {
    if (ev && nrhs == 1) cudaEventRecord(ev[stage], s);
    ++stage;
  };
  mark();
  const ApplyArgs& a0 = args[0];
  const T2* tw = reinterpret_cast<const T2*>(a0.tw);
  const size_t seq = fft_seq_bytes(a0.N, sizeof(T2) == sizeof(float2));
  const long long NN = (long long)a0.N * a0.N;
  for (int b = 0; b < nrhs; ++b) {
    const ApplyArgs& a = args[b];
    const T2* f = f0 + b * NN;
    T2* fhat = reinterpret_cast<T2*>(a.fhat);
    T2* tmp = reinterpret_cast<T2*>(a.tmp);
    // K0: fhat = FFT2(f) / N  (forward sign, eq. dft)
    int rpc = a.rows_per_cta_N;
    k_fft_rows<T2><<<(a.N + rpc - 1) / rpc, 256, rpc * seq, s>>>(f, tmp, a.N, rpc, a.ffts, a.fft_N, tw, -1, 1.0);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ++n;
    mark();
    int cpc = a.cols_per_cta_N;
    k_fft_cols<T2><<<(a.N + cpc - 1) / cpc, 256, cpc * seq, s>>>(tmp, fhat, a.N, cpc, a.ffts, a.fft_N, tw, -1,
                                                                 1.0 / a.N);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ++n;
    mark();
    if (a.nw > 0) {
      const T2* const* betas = reinterpret_cast<const T2* const*>(a.beta);
      k_rowpass<T2><<<a.njobs_row, FIO_K1_THREADS, a.smem_row, s>>>(a.N, a.wedges, a.jobs_row, a.ffts, tw, betas, fhat,
                                                         reinterpret_cast<T2*>(a.p1));
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
      ++n;
      mark();
      k_colpass<T2><<<a.njobs_col, FIO_K2_THREADS, a.smem_col, s>>>(a.wedges, a.jobs_col, a.ffts, tw,
                                                         reinterpret_cast<const T2*>(a.p1), reinterpret_cast<T2*>(a.g));
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
      ++n;
      mark();
    } else {
      mark();
      mark();
    }
  }
  if ((e = launch_interp<T2>(args, nrhs, Lf, s, &n)) != cudaSuccess) return e;
  mark();
  if (launches) *launches = n;
  return cudaSuccess;
}

cudaError_t enqueue_apply(const ApplyArgs& a, bool c64, const void* f, void* Lf, cudaStream_t s, int* launches,
                          cudaEvent_t* ev) {
  if (c64) return enqueue_apply_t<float2>(&a, 1, (const float2*)f, (float2*)Lf, s, launches, ev);
  return enqueue_apply_t<double2>(&a, 1, (const double2*)f, (double2*)Lf, s, launches, ev);
}

cudaError_t enqueue_apply_batch(const ApplyArgs* args, int nrhs, bool c64, const void* f, void* Lf, cudaStream_t s,
                                int* launches) {
  if (c64) return enqueue_apply_t<float2>(args, nrhs, (const float2*)f, (float2*)Lf, s, launches, nullptr);
  return enqueue_apply_t<double2>(args, nrhs, (const double2*)f, (double2*)Lf, s, launches, nullptr);
}

}  // namespace fio
