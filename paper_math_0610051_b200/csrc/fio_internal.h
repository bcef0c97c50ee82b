// fio_internal.h -- structures shared by the host plan code and the CUDA kernels
// of the product library (never by the oracle).  See include/fio.h and DESIGN.md.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/fio.h"

#ifdef __CUDACC__
#define FIO_HD_EARLY __host__ __device__
#else
#define FIO_HD_EARLY
#endif

namespace fio {

constexpr int kMaxRadixStages = 24;
constexpr int kMaxTaps = 12;  // up to eps ~ 1e-11 (reading R10)
// K3 (interpolation + alpha epilogue).  One thread owns a group of up to P
// points whose w x w tap windows all lie inside one window of the fine grid, loads each window value
// once per term from shared memory and applies it to all P points (register reuse P: the shared ->
// register path, 128 B/clk/SM, is K3's binding on-chip resource).
#ifndef FIO_K3_P64
#define FIO_K3_P64 4
#endif
#ifndef FIO_K3_P128
#define FIO_K3_P128 4
#endif
#ifndef FIO_K3_BIGTAPS
#define FIO_K3_BIGTAPS 8  // above this many taps the column weights of P points no longer fit: P = 4
#endif
constexpr int kGroupPC64 = FIO_K3_P64;    // points per K3 group, complex64
constexpr int kGroupPC128 = FIO_K3_P128;  // complex128
FIO_HD_EARLY constexpr int group_p(bool c64, int taps) {
  return taps > FIO_K3_BIGTAPS ? 4 : (c64 ? kGroupPC64 : kGroupPC128);
}
#ifndef FIO_K3_BLOCK64
#define FIO_K3_BLOCK64 64
#endif
#ifndef FIO_K3_BLOCK128
#define FIO_K3_BLOCK128 64
#endif
constexpr int kK3BlockC64 = FIO_K3_BLOCK64;    // K3 threads per CTA (= groups per chunk), complex64
constexpr int kK3BlockC128 = FIO_K3_BLOCK128;  // complex128
#ifndef FIO_K3_CAP64
#define FIO_K3_CAP64 384
#endif
#ifndef FIO_K3_CAP128
#define FIO_K3_CAP128 384
#endif
// K3 pipeline: the term loop advances TT terms per step and stages the next step while computing
// (a ring of 2 TT terms; fio_kernels.cu K3Cfg).  Measured at N = 1024 (K3 ms, TT = 1): complex64 ring
// of 2 / 3 / 4 terms 2.59 / 2.62 / 2.72, complex128 11.16 / 12.47 / 12.52 -- shallow rings leave room
// for more CTAs per SM, which hide latency better than a deeper ring.
// Separation (reading R8): rows sampled for the column pivoting = min(8 r, 512) (at least r).  Measured over
// the seeded random operators of tests/test_gpu_parity.py (profiles/r02_sep_rows.txt): r rows leave a worst
// pointwise error of 136 eps (a point class the small sample misses), 8 r rows 22 eps; sum_q, plan time and
// the apply at N = 1024 are unchanged.
constexpr int kSepRowOversample = 8, kSepRowCap = 512;
constexpr int kK3TileCapC64 = FIO_K3_CAP64;     // max cells of a K3 chunk footprint, complex64
constexpr int kK3TileCapC128 = FIO_K3_CAP128;   // complex128
constexpr int kHalo = 8;  // periodic column halo on each side of a fine-grid row (K2 writes, K3 reads)
// Window shape: a group's points share the base row and lie within two base columns (complex64:
// w rows x (w+1) columns), or share the base column and lie within two base rows (complex128:
// (w+1) rows x w columns).  Row weights are kept per point in shared memory, column weights in
// registers, so the register cost per point is the column count.
constexpr int kSuperRowsC64 = 1, kSuperColsC64 = 2;
constexpr int kSuperRowsC128 = 2, kSuperColsC128 = 1;
#ifdef __CUDACC__
#define FIO_HD __host__ __device__
#else
#define FIO_HD
#endif
FIO_HD constexpr int super_rows(bool c64) { return c64 ? kSuperRowsC64 : kSuperRowsC128; }
FIO_HD constexpr int super_cols(bool c64) { return c64 ? kSuperColsC64 : kSuperColsC128; }
FIO_HD constexpr int k3_window_rows(int taps, bool c64) { return taps + super_rows(c64) - 1; }
FIO_HD constexpr int k3_window_cols(int taps, bool c64) { return taps + super_cols(c64) - 1; }

// Division by a runtime constant d via multiply-high (Granlund-Montgomery), exact for
// numerators n < 2^31: q = (umulhi(m, n) + n) >> l.
struct FastDiv {
  uint32_t m, l, d;
};
inline FastDiv make_fastdiv(uint32_t d) {
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  uint64_t m = ((((1ull << l) - d) << 32) / d) + 1;
  return FastDiv{(uint32_t)m, l, d};
}

// One FFT length L (5-smooth), its Stockham radix sequence, per-stage divisors (butterflies
// per sequence nb = L/R and span Ns) and the offset of its twiddle table e^{+2 pi i m / L}.
struct FftLen {
  int L;
  int nst;
  int tw_off;
  int pad;
  int8_t radix[kMaxRadixStages];
  FastDiv div_nb[kMaxRadixStages];
  FastDiv div_ns[kMaxRadixStages];
};

// Per owned wedge l:
//   box frequencies  k' = M xi - xi_c  in [-n1/2, n1/2) x [-n2/2, n2/2)
//   fine grid        n1f x n2f (oversampled, 5-smooth), index k' mod nf
//   warped points    y(x) = M^{-T} g_l(x), g_l(x) = x + b(x) + grad_xi rho(x, xihat_l)
struct WedgeDev {
  int l, q;
  int n1, n2, n1f, n2f;
  int M[4];     // row-major integer matrix in SL(2,Z)
  int Mi[4];    // its inverse (integer)
  int xc1, xc2; // xi_c
  int fft1, fft2;  // FftLen index for n1f (column pass) and n2f (row pass)
  double u1, u2;   // xihat_l = (cos 2 pi l / W, sin 2 pi l / W)
  long long p1_off;     // element offset of the row-pass buffer, [t][j2][i1] (q * n2f * n1)
  long long g_off;      // element offset of the fine grids, [t][j2][kHalo + j1] (q * n2f * (n1f + 2 kHalo))
};

// K3 (interpolation + alpha epilogue) data of one owned wedge.  Points are
// grouped at plan time: the P points of a group have their base fine cells
// b = ceil(u - w/2) in the same 2 x 2 "supercell", so one (w+1) x (w+1) window
// of the fine grid anchored at `anchor` covers all their taps.
// The fine grid is stored [j2][kHalo + j1]: K3's "rows" are j2 (nrow = n2f, wrapped) and
// its "columns" are j1 (ncol = n1f, haloed row stride ncolp = n1f + 2 kHalo).
constexpr int kBoxInts = 8;  // one 32-byte box record per K3 chunk (a bulk-copy unit)
// Physical position of slot k of group g: element-major inside each chunk of `block` groups,
// [chunk][k][g mod block] -- the shared-memory image K3 reads conflict-free (lane = group).
FIO_HD_EARLY inline long long k3_slot(long long g, int k, int P, int block) {
  return (g / block) * block * P + (long long)k * block + g % block;
}

struct InterpWedge {
  int q, nrow, ncol, ngroups;
  int ncolp;
  long long g_off;          // element offset of this wedge's fine grids
  const int* anchor;        // 2 ints per group (a1, a2), may be negative (wrapped in K3)
  const int* slot_x;        // per slot (k3_slot layout): flat output index, -1 = padding
  const void* slot_off;     // per slot: (u1 - a1, u2 - a2) as float2 (c64) / double2 (c128)
  const void* alpha;        // alpha'[t][slot] (k3_slot layout), plan dtype
  int nchunks;              // chunks of K3 BLOCK consecutive groups
  int tile_cap;             // max rows*cols of a chunk's window footprint (elements)
  const int* box;           // kBoxInts per chunk: first group, row origin, column origin, rows, columns, groups,
                            // shared-memory row stride of the tile (>= columns), 1 = tile by TMA (tensor map)
  int tma;                  // this launch may stage tiles by TMA (the plan's tensor map of this wedge's G)
};

// K3 tiles by TMA (cp.async.bulk.tensor.3d, one request per chunk and term): the fixed box (rows x
// columns of the fine grid) a chunk's footprint must fit, unwrapped, to use it; other chunks keep the
// per-thread cp.async copies.  Box widths are an odd number of 16-byte units (bank-conflict-free rows).
#ifndef FIO_K3_TMA
#define FIO_K3_TMA 1
#endif
#ifndef FIO_K3_BOXR64
#define FIO_K3_BOXR64 12
#endif
#ifndef FIO_K3_BOXR128
#define FIO_K3_BOXR128 12
#endif
constexpr int kK3BoxRows64 = FIO_K3_BOXR64, kK3BoxCols64 = 22;
constexpr int kK3BoxRows128 = FIO_K3_BOXR128, kK3BoxCols128 = 23;

// Work item of the batched FFT passes: one CTA processes `count` sequences of
// the (wedge, t) pair starting at row/column `start`.
struct alignas(32) FftJob {
  int w;      // index into the owned-wedge table
  int t;
  int start;
  int count;
  int fft;    // FftLen index of this pass (so the kernel's wedge and FFT-plan loads are independent)
  int pad[3];
};

// Host-side geometry of one wedge.
struct WedgeGeom {
  int l;
  std::vector<int> members;  // flat FFT-order frequency indices k1*N+k2
  std::vector<double> chi;   // smooth partition: chi_l of every member (empty: the indicator, chi = 1)
  int M[4], Mi[4];
  int xc1, xc2;
  int n1, n2, n1f, n2f;
  double u1, u2;
};

// Piecewise-polynomial form of the NUFFT kernel for K3 (c128): tap j of a point whose base
// cell is b and fractional offset s = u - b in (w/2 - 1, w/2] has weight
// phi(s - j) = sum_m c[j][m] x^m, x = 2 (s - w/2) + 1 in (-1, 1].
constexpr int kPolyMaxDeg = 20;
// Degree of the K3 kernel polynomial for w taps (fixed at compile time: one unrolled Horner per
// axis).  With the default beta = 2.3 w it meets the fit tolerance 2 e^{-beta}: w <= 5: 6, 6-7: 7,
// 8-9: 8, 10: 9, 11: 10, 12: 11 (measured by es_poly_fit).
FIO_HD_EARLY constexpr int k3_poly_deg(int taps) {
  return taps <= 5 ? 6 : taps <= 7 ? 7 : taps <= 9 ? 8 : taps == 10 ? 9 : taps == 11 ? 10 : 11;
}
struct EsPoly {
  int deg;
  double c[kMaxTaps][kPolyMaxDeg + 1];
  // the same coefficients in FP32, coefficient-major with taps padded to an even count, so
  // that taps (2i, 2i+1) are one float2 (packed FFMA2 Horner; c64 weights and the FP32 row weights)
  float cf[kPolyMaxDeg + 1][kMaxTaps + 2];
};

// Host helpers (fio_host.cpp).
int default_wedges(int N);
bool is_smooth5(int n);
int next_fine_size(int extent);
int wedge_of(int W, int xi1, int xi2);
void build_geometry(int N, int W, std::vector<WedgeGeom>& wedges, double overlap = 0.0);
double wedge_weight(int W, double overlap, int l, int xi1, int xi2);  // chi_l(xi), reading R2
std::vector<int8_t> radix_plan(int L);
double es_kernel(double z, int w, double beta);
double es_fourier(double s, int w, double beta);  // psi(s) = int phi(v) cos(2 pi s v) dv
int taps_for_eps(double eps);
// Fit EsPoly for (w, beta) at degree k3_poly_deg(w) (Chebyshev interpolation); returns the max error.
double es_poly_fit(int w, double beta, EsPoly& out);
void lpt_assign(int W, const double* cost, int nranks, int* owner);

// Group the output points of one wedge for K3 (see InterpWedge).  u: 2*NN doubles
// (K3 row / column fine coordinates in [0, n1f) x [0, n2f)).  Outputs: anchor (2 per group),
// slot_x (P per group, -1 padding), off (2 per slot: u - anchor).
void group_points(const double* u, long long NN, int taps, int P, int n1f, int n2f, int super_rows, int super_cols,
                  std::vector<int>& anchor, std::vector<int>& slot_x, std::vector<double>& off);
long long chunk_boxes(const std::vector<int>& anchor, int block, int win_rows, int win_cols, long long cap,
                      std::vector<int>& box, int elem_bytes);

// Complex helpers on interleaved doubles.
struct cplx {
  double re, im;
};

// One-sided (Hestenes) Jacobi SVD of a complex m x n column-major matrix A
// (m >= n): on return A holds U*Sigma (columns), V (n x n column-major) and
// sigma (n), sorted descending.
void jacobi_svd(int m, int n, std::vector<cplx>& A, std::vector<cplx>& V, std::vector<double>& sigma);

// Small dense helpers of the high-accuracy separation (shifted CholeskyQR3, fio_api.cu):
// G = R^H R (false if not positive definite; G overwritten by R), X = R^{-1}, C = A B.
bool cholesky_upper(int n, std::vector<cplx>& G);
void upper_inverse(int n, const std::vector<cplx>& R, std::vector<cplx>& X);
void small_matmul(int n, const std::vector<cplx>& A, const std::vector<cplx>& B, std::vector<cplx>& C);

// Column-pivoted modified Gram-Schmidt on the m x n column-major matrix B (destroyed);
// returns up to k pivot column indices in order.
std::vector<int> pivoted_columns(int m, int n, std::vector<cplx>& B, int k);

// Counter-based generator (splitmix64) and sampling without replacement.
struct Rng {
  uint64_t s;
  explicit Rng(uint64_t seed) : s(seed) {}
  uint64_t next();
  uint64_t below(uint64_t n);
};
std::vector<int> sample_distinct(Rng& rng, int n, int k);

void set_error(const std::string& msg);

}  // namespace fio
