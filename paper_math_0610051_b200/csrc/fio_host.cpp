// fio_host.cpp -- host-side plan logic of the product library: the wedge
// partition and lattice boxes, FFT radix plans, the NUFFT kernel and its
// Fourier transform, small dense linear algebra (Jacobi SVD, column-pivoted
// Gram-Schmidt), the counter-based RNG and the wedge->rank assignment.
// Shares no code with oracle/.  Citations are PAPER.md line numbers.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <unordered_set>

#include "fio_internal.h"

namespace fio {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
const char* last_error_cstr() { return g_err.c_str(); }

// Reading R1: W = 8 round(2 sqrt(N) / 8), at least 8.  The paper fixes W ~ sqrt(N)
// only up to a constant (the aperture 2 alpha / sqrt(N), alpha free); 2 is the measured optimum of
// the B200 apply at the headline size (N = 1024: W = 48/56/64/72 give 14.29/14.14/13.88/13.77 ms
// c128 and 3.27/3.32/3.27/3.39 ms c64; N = 2048: W = 80/88 give 69.3/70.6 ms).  A multiple of 8
// makes every boundary ray (2l+1) pi / W irrational-sloped, so no lattice point is ever on a
// wedge boundary.
int default_wedges(int N) {
  int w = 8 * (int)std::lround(2.0 * std::sqrt((double)N) / 8.0);
  return std::max(8, w);
}

bool is_smooth5(int n) {
  if (n <= 0) return false;
  for (int p : {2, 3, 5})
    while (n % p == 0) n /= p;
  return n == 1;
}

// Smallest even 5-smooth nf >= 2 * extent: oversampling sigma >= 2 (PAPER.md:1305-1325,
// reading R10), sizes the hand-written mixed-radix FFT supports.
int next_fine_size(int extent) {
  int nf = std::max(2 * extent, 8);
  while (!(is_smooth5(nf) && nf % 2 == 0)) ++nf;
  return nf;
}

// Wedge W_l = {xi : (2l-1) pi/W <= arg xi < (2l+1) pi/W}, arg
// measured from (1,0) and wrapped to [-pi/W, 2 pi - pi/W) (readings R4, R14);
// xi = 0 belongs to no wedge (reading R3).
int wedge_of(int W, int xi1, int xi2) {
  if (xi1 == 0 && xi2 == 0) return -1;
  const double pi = 3.14159265358979323846;
  double th = std::atan2((double)xi2, (double)xi1);
  double lo = -pi / W;
  if (th < lo) th += 2.0 * pi;
  int l = (int)std::floor((th - lo) / (2.0 * pi / W));
  return std::min(std::max(l, 0), W - 1);
}

// Smooth partition of unity over the angle (reading R2; BASELINE north_star "smooth
// polar-wedge partition"): with D = 2 pi / W, the paper's boundary rays b_l = (l - 1/2) D
// and a taper half-width h = overlap D / 2,
//   chi_l(xi) = S((theta - b_l) / h) (1 - S((theta - b_{l+1}) / h)),
// angles differences taken in (-pi, pi], where S is the C-infinity step S(tau) = g(u) / (g(u) + g(1-u)),
// u = (1 + tau) / 2, g(u) = e^{-1/u} (u > 0), S = 0 for tau <= -1 and 1 for tau >= 1.  S(tau) +
// S(-tau) = 1, so at every angle the two wedges sharing a boundary carry 1 - S and S (sum 1),
// chi_l = 1/2 on the paper's boundary rays and chi_l is the indicator outside the tapers.
// overlap <= 0: the paper's indicator wedges (wedge_of).
static double smooth_step(double tau) {
  if (tau <= -1.0) return 0.0;
  if (tau >= 1.0) return 1.0;
  const double u = 0.5 * (1.0 + tau), v = 1.0 - u;
  const double gu = std::exp(-1.0 / u), gv = std::exp(-1.0 / v);
  return gu / (gu + gv);
}

static double angle_diff(double a) {  // a wrapped to (-pi, pi]
  const double pi = 3.14159265358979323846, twopi = 2.0 * pi;
  a = std::fmod(a, twopi);
  if (a <= -pi) a += twopi;
  if (a > pi) a -= twopi;
  return a;
}

double wedge_weight(int W, double overlap, int l, int xi1, int xi2) {
  if (xi1 == 0 && xi2 == 0) return 0.0;
  if (!(overlap > 0.0)) return wedge_of(W, xi1, xi2) == l ? 1.0 : 0.0;
  const double pi = 3.14159265358979323846;
  const double D = 2.0 * pi / W, h = 0.5 * overlap * D;
  const double th = std::atan2((double)xi2, (double)xi1);
  const double lo = angle_diff(th - (l - 0.5) * D), hi = angle_diff(th - (l + 0.5) * D);
  return smooth_step(lo / h) * (1.0 - smooth_step(hi / h));
}

static void all_sl2z(std::vector<std::array<int, 4>>& out) {
  out.clear();
  // identity first so that ties keep the plain relabeling of PAPER.md:1331-1336
  out.push_back({1, 0, 0, 1});
  for (int a = -3; a <= 3; ++a)
    for (int b = -3; b <= 3; ++b)
      for (int c = -3; c <= 3; ++c)
        for (int d = -3; d <= 3; ++d)
          if (a * d - b * c == 1 && !(a == 1 && b == 0 && c == 0 && d == 1)) out.push_back({a, b, c, d});
}

// Partition Omega \ {0} into W wedges and pick, per wedge, the lattice map
// M in SL(2,Z) (entries in [-3,3]) whose relabelled box has the smallest
// oversampled volume (PAPER.md:1327-1347 uses the identity or a 45-degree
// shear; reading R5 generalizes to any small unimodular M -- still an exact
// relabeling).  xi_c places the box's k' range at [-floor(n/2), n - floor(n/2)).
void build_geometry(int N, int W, std::vector<WedgeGeom>& wedges, double overlap) {
  wedges.assign(W, WedgeGeom());
  const double pi = 3.14159265358979323846;
  for (int l = 0; l < W; ++l) {
    wedges[l].l = l;
    wedges[l].u1 = std::cos(2.0 * pi * l / W);
    wedges[l].u2 = std::sin(2.0 * pi * l / W);
  }
  for (int k1 = 0; k1 < N; ++k1) {
    int x1 = k1 >= N / 2 ? k1 - N : k1;
    for (int k2 = 0; k2 < N; ++k2) {
      int x2 = k2 >= N / 2 ? k2 - N : k2;
      if (!(overlap > 0.0)) {
        int l = wedge_of(W, x1, x2);
        if (l >= 0) wedges[l].members.push_back(k1 * N + k2);
        continue;
      }
      // smooth partition: the (at most two) wedges with chi_l(xi) > 0 around the indicator's wedge
      const int l0 = wedge_of(W, x1, x2);
      if (l0 < 0) continue;
      for (int dl = -1; dl <= 1; ++dl) {
        const int l = (l0 + dl + W) % W;
        const double c = wedge_weight(W, overlap, l, x1, x2);
        if (c > 0.0) {
          wedges[l].members.push_back(k1 * N + k2);
          wedges[l].chi.push_back(c);
        }
      }
    }
  }
  std::vector<std::array<int, 4>> mats;
  all_sl2z(mats);
#pragma omp parallel for schedule(dynamic, 1)
  for (int l = 0; l < W; ++l) {
    WedgeGeom& g = wedges[l];
    long long best = -1;
    for (const auto& M : mats) {
      int lo1 = 1 << 30, hi1 = -(1 << 30), lo2 = 1 << 30, hi2 = -(1 << 30);
      for (int k : g.members) {
        int k1 = k / N, k2 = k % N;
        int x1 = k1 >= N / 2 ? k1 - N : k1;
        int x2 = k2 >= N / 2 ? k2 - N : k2;
        int z1 = M[0] * x1 + M[1] * x2, z2 = M[2] * x1 + M[3] * x2;
        lo1 = std::min(lo1, z1); hi1 = std::max(hi1, z1);
        lo2 = std::min(lo2, z2); hi2 = std::max(hi2, z2);
      }
      if (g.members.empty()) { lo1 = hi1 = lo2 = hi2 = 0; }
      int n1f = next_fine_size(hi1 - lo1 + 1), n2f = next_fine_size(hi2 - lo2 + 1);
      long long cost = (long long)n1f * n2f;
      if (best < 0 || cost < best) {
        best = cost;
        std::memcpy(g.M, M.data(), sizeof(g.M));
        g.n1f = n1f; g.n2f = n2f;
        g.n1 = n1f / 2; g.n2 = n2f / 2;
        g.xc1 = lo1 + g.n1 / 2;
        g.xc2 = lo2 + g.n2 / 2;
      }
    }
    // inverse of a unimodular matrix [[a,b],[c,d]] is [[d,-b],[-c,a]]
    g.Mi[0] = g.M[3]; g.Mi[1] = -g.M[1]; g.Mi[2] = -g.M[2]; g.Mi[3] = g.M[0];
  }
}

// Stockham radix sequence: 4s, then 2, 3s, 5s (all sizes 5-smooth).  (Radix-8/16 stages were
// measured slower on B200 for these lengths -- fewer butterflies per stage than threads, more
// registers -- and removed.)
std::vector<int8_t> radix_plan(int L) {
  std::vector<int8_t> r;
  while (L % 4 == 0) { r.push_back(4); L /= 4; }
  while (L % 2 == 0) { r.push_back(2); L /= 2; }
  while (L % 3 == 0) { r.push_back(3); L /= 3; }
  while (L % 5 == 0) { r.push_back(5); L /= 5; }
  if (L != 1) r.clear();
  return r;
}

// "Exponential of semicircle" kernel phi(z) = exp(beta (sqrt(1 - (2z/w)^2) - 1)),
// |z| < w/2, in fine-grid units (reading R10: the paper's Dutt-Rokhlin
// parameters are not reproducible from the text; any kernel with a known
// Fourier transform works -- the deconvolution is folded into beta').
double es_kernel(double z, int w, double beta) {
  double t = 2.0 * z / w;
  if (std::fabs(t) >= 1.0) return 0.0;
  return std::exp(beta * (std::sqrt(1.0 - t * t) - 1.0));
}

// Gauss-Legendre nodes/weights on [-1,1] (Newton on P_n), cached for n = 256.
static void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& wt) {
  x.resize(n); wt.resize(n);
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < n; ++i) {
    double z = std::cos(pi * (i + 0.75) / (n + 0.5)), pp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p1 = 1.0, p2 = 0.0;
      for (int j = 1; j <= n; ++j) {
        double p3 = p2; p2 = p1;
        p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
      }
      pp = n * (z * p1 - p2) / (z * z - 1.0);
      double z1 = z;
      z = z1 - p1 / pp;
      if (std::fabs(z - z1) < 1e-16) break;
    }
    x[i] = z;
    wt[i] = 2.0 / ((1.0 - z * z) * pp * pp);
  }
}

// psi(s) = int_{-w/2}^{w/2} phi(v) cos(2 pi s v) dv: the factor by which
// interpolating with phi multiplies frequency k when s = k / nf, so beta'
// carries 1/(psi(k1/n1f) psi(k2/n2f)) (deconvolution step of the NUFFT).
struct GaussLegendre {
  std::vector<double> x, w;
  GaussLegendre() { gauss_legendre(256, x, w); }
};

double es_fourier(double s, int w, double beta) {
  static const GaussLegendre gl;  // thread-safe static init (C++11)
  const std::vector<double>& gx = gl.x;
  const std::vector<double>& gw = gl.w;
  const double pi = 3.14159265358979323846;
  double acc = 0.0, h = 0.5 * w;
  for (size_t i = 0; i < gx.size(); ++i) {
    double v = gx[i] * h;
    acc += gw[i] * h * es_kernel(v, w, beta) * std::cos(2.0 * pi * s * v);
  }
  return acc;
}

// Chebyshev interpolation of phi(s - j) on s in (w/2 - 1, w/2] at deg+1 nodes, converted to
// monomial coefficients in x = 2 (s - w/2) + 1, at the kernels' fixed degree k3_poly_deg(w); returns
// the error measured on a fine grid (about 1.5 e^{-beta} at the default beta, the kernel's own edge
// value: the polynomial is as accurate as the kernel it stands for).
double es_poly_fit(int w, double beta, EsPoly& out) {
  const double pi = 3.14159265358979323846;
  double err = 1.0;
  for (int deg = k3_poly_deg(w); deg <= k3_poly_deg(w); ++deg) {
    std::memset(&out, 0, sizeof(out));
    out.deg = deg;
    const int n = deg + 1;
    err = 0.0;
    for (int j = 0; j < w; ++j) {
      std::vector<double> f(n), a(n, 0.0);
      for (int k = 0; k < n; ++k) {
        double x = std::cos(pi * (k + 0.5) / n);
        double sv = 0.5 * w + 0.5 * (x - 1.0);
        f[k] = es_kernel(sv - j, w, beta);
      }
      for (int m = 0; m < n; ++m) {
        double acc = 0;
        for (int k = 0; k < n; ++k) acc += f[k] * std::cos(pi * m * (k + 0.5) / n);
        a[m] = acc * (m == 0 ? 1.0 : 2.0) / n;
      }
      // sum_m a_m T_m(x) -> monomials
      std::vector<double> tprev(n, 0.0), tcur(n, 0.0), coef(n, 0.0);
      tprev[0] = 1.0;                 // T_0
      if (n > 1) tcur[1] = 1.0;       // T_1
      for (int i = 0; i < n; ++i) coef[i] += a[0] * tprev[i];
      if (n > 1)
        for (int i = 0; i < n; ++i) coef[i] += a[1] * tcur[i];
      for (int m = 2; m < n; ++m) {
        std::vector<double> tnext(n, 0.0);
        for (int i = 0; i < n; ++i) {
          if (i > 0) tnext[i] += 2.0 * tcur[i - 1];
          tnext[i] -= tprev[i];
        }
        for (int i = 0; i < n; ++i) coef[i] += a[m] * tnext[i];
        tprev.swap(tcur);
        tcur.swap(tnext);
      }
      for (int m = 0; m < n; ++m) out.c[j][m] = coef[m];
      for (int k = 0; k <= 400; ++k) {
        double x = -1.0 + 2.0 * k / 400.0;
        if (k == 0) x += 1e-12;
        double sv = 0.5 * w + 0.5 * (x - 1.0);
        double p = 0;
        for (int m = n - 1; m >= 0; --m) p = p * x + coef[m];
        err = std::max(err, std::fabs(p - es_kernel(sv - j, w, beta)));
      }
    }
  }
  for (int m = 0; m <= out.deg; ++m)
    for (int j = 0; j < w; ++j) out.cf[m][j] = (float)out.c[j][m];
  return err;
}

// Reading R10: taps per dimension so that the NUFFT error (measured: ~1e-(w-1)
// relative l2 at sigma = 2, beta = 2.3 w) stays below ~2 eps.
int taps_for_eps(double eps) {
  int w = (int)std::ceil(-std::log10(2.0 * eps)) + 1;
  return std::min(std::max(w, 4), kMaxTaps);  // w = 3 is ~1e-2 accurate: never chosen
}

// Longest-processing-time greedy: wedges by decreasing cost, each to the least
// loaded rank (ties -> lowest rank).  Deterministic.
void lpt_assign(int W, const double* cost, int nranks, int* owner) {
  std::vector<int> idx(W);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return cost[a] > cost[b]; });
  std::vector<double> load(nranks, 0.0);
  for (int l : idx) {
    int r = (int)(std::min_element(load.begin(), load.end()) - load.begin());
    owner[l] = r;
    load[r] += cost[l];
  }
}

// K3 grouping: base cell b = ceil(u - w/2) per axis (the first of the point's w
// taps).  The window of a group spans kSuperRows x kSuperCols base cells -- (w + kSuperRows - 1) x
// (w + kSuperCols - 1) fine cells -- so a group may hold points whose base cells differ by at most
// one along the "run" axis (columns when kSuperCols == 2, rows when kSuperRows == 2).  Points are
// counting-sorted by (fixed axis, run axis, x) and cut greedily: a group takes the next points while
// they share the fixed-axis base and lie within two run-axis bases of the group's first point (its
// anchor), up to P points.  complex128 slides the anchor (only a run's last group can be partly
// empty); complex64 keeps a fixed lattice of two-column supercells, whose even anchors make every
// window row a run of 16-byte aligned pairs (vector loads).  Groups are then ordered in serpentine
// 16 x 16-cell blocks of their anchors, so a K3 chunk (consecutive groups) has a compact footprint.
static inline long long floor_div2(long long b) { return b >= 0 ? b / 2 : -((-b + 1) / 2); }

void group_points(const double* u, long long NN, int taps, int P, int n1f, int n2f, int kSuperRows, int kSuperCols,
                  std::vector<int>& anchor, std::vector<int>& slot_x, std::vector<double>& off) {
  const bool run_cols = kSuperCols == 2;  // c64: runs along columns within a base row
  const long long lo = -(taps / 2) - 2;    // smallest base index per axis (u >= 0)
  const long long nb1 = n1f + taps + 4, nb2 = n2f + taps + 4;
  std::vector<int> b1v(NN), b2v(NN);
  std::vector<int> key(NN);
  const long long nmaj = run_cols ? nb1 : nb2, nmin = run_cols ? nb2 : nb1;
#pragma omp parallel for schedule(static)
  for (long long x = 0; x < NN; ++x) {
    const long long b1 = (long long)std::ceil(u[2 * x] - 0.5 * taps);
    const long long b2 = (long long)std::ceil(u[2 * x + 1] - 0.5 * taps);
    b1v[x] = (int)b1;
    b2v[x] = (int)b2;
    const long long maj = (run_cols ? b1 : b2) - lo, mn = (run_cols ? b2 : b1) - lo;
    key[x] = (int)(maj * nmin + mn);
  }
  const long long nkeys = nmaj * nmin;
  std::vector<long long> cnt(nkeys + 1, 0);
  for (long long x = 0; x < NN; ++x) cnt[key[x] + 1]++;
  for (long long k = 0; k < nkeys; ++k) cnt[k + 1] += cnt[k];
  std::vector<int> order(NN);
  {
    std::vector<long long> pos(cnt.begin(), cnt.end() - 1);
    for (long long x = 0; x < NN; ++x) order[pos[key[x]]++] = (int)x;  // stable: by x within a cell
  }
  // greedy runs -> groups (first point index into `order`, count)
  std::vector<long long> gstart;
  std::vector<int> gcount;
  gstart.reserve(NN / P + 16);
  gcount.reserve(NN / P + 16);
  for (long long p = 0; p < NN;) {
    const int x0 = order[p];
    const int maj0 = run_cols ? b1v[x0] : b2v[x0], mn0 = run_cols ? b2v[x0] : b1v[x0];
    long long e = p + 1;
    while (e < NN && e - p < P) {
      const int x = order[e];
      const int maj = run_cols ? b1v[x] : b2v[x], mn = run_cols ? b2v[x] : b1v[x];
      // complex64 (runs along columns): fixed two-column supercells, so every anchor column is even
      // (16-byte aligned window rows); complex128: sliding pairs of base rows
      if (maj != maj0 || (run_cols ? (floor_div2(mn) != floor_div2(mn0)) : (mn > mn0 + 1))) break;
      ++e;
    }
    gstart.push_back(p);
    gcount.push_back((int)(e - p));
    p = e;
  }
  const long long G = (long long)gstart.size();
  // serpentine 16 x 16-cell blocks of anchors
  const long long BS = 16;
  std::vector<std::pair<long long, long long>> gk(G);
  const long long nbc = (std::max(nb1, nb2) + BS - 1) / BS + 2;
#pragma omp parallel for schedule(static)
  for (long long g = 0; g < G; ++g) {
    const int x0 = order[gstart[g]];
    const long long a1 = b1v[x0] - lo, a2 = b2v[x0] - lo;
    const long long br = a1 / BS, bcr = a2 / BS;
    const long long bc = (br % 2 == 0) ? bcr : nbc - 1 - bcr;
    // row-major inside a block for both window shapes: consecutive groups (a warp's lanes) sit at
    // consecutive anchor columns, so their window loads hit consecutive shared-memory words
    const long long inner = (a1 % BS) * BS + (a2 % BS);
    gk[g] = {(br * nbc + bc) * BS * BS + inner, g};
  }
  std::sort(gk.begin(), gk.end());
  anchor.assign(2 * G, 0);
  slot_x.assign((size_t)P * G, -1);
  off.assign((size_t)2 * P * G, 0.5 * taps);
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < G; ++i) {
    const long long g = gk[i].second;
    const long long p = gstart[g];
    const int x0 = order[p];
    const int a1 = b1v[x0], a2 = b2v[x0];
    // anchor = the window's first fine cell: the smallest base on each axis among the members
    // (complex64: the supercell's even column)
    int m1 = a1, m2 = a2;
    for (int j = 0; j < gcount[g]; ++j) {
      const int x = order[p + j];
      m1 = std::min(m1, b1v[x]);
      m2 = std::min(m2, b2v[x]);
    }
    if (run_cols) m2 = (int)(2 * floor_div2(a2));
    anchor[2 * i] = m1;
    anchor[2 * i + 1] = m2;
    for (int j = 0; j < gcount[g]; ++j) {
      const int x = order[p + j];
      const long long sl = i * P + j;
      slot_x[sl] = x;
      off[2 * sl] = u[2 * x] - m1;
      off[2 * sl + 1] = u[2 * x + 1] - m2;
    }
  }
}

// K3 chunks: runs of at most `block` consecutive groups whose windows' bounding box
// has at most `cap` cells.  Per chunk: {first group, row origin, column origin, rows,
// columns, groups}; returns the largest rows*cols.
// Tile rows are an odd number of 16-byte units long (complex128: odd columns; complex64: columns
// = 2 mod 4): lanes whose windows start on consecutive tile rows then hit distinct shared-memory
// banks.
static inline int pad_tile_cols(int nc, int elem_bytes) {
  if (elem_bytes == 16) return nc | 1;
  nc = (nc + 1) & ~1;                // even: 16-byte copy units
  return (nc % 4 == 0) ? nc + 2 : nc;
}

// complex64 tile rows are copied in 16-byte units: the column origin is rounded down to even
static inline int tile_col0(int clo, int elem_bytes) { return elem_bytes == 8 ? (clo & ~1) : clo; }

long long chunk_boxes(const std::vector<int>& anchor, int block, int win_rows, int win_cols, long long cap,
                      std::vector<int>& box, int elem_bytes) {
  const long long ng = (long long)anchor.size() / 2;
  box.clear();
  long long maxcap = 0;
  long long c0 = 0;
  while (c0 < ng) {
    int rlo = anchor[2 * c0], rhi = rlo, clo = anchor[2 * c0 + 1], chi = clo;
    long long c1 = c0 + 1;
    while (c1 < ng && c1 - c0 < block) {
      const int r = anchor[2 * c1], c = anchor[2 * c1 + 1];
      const int nrlo = std::min(rlo, r), nrhi = std::max(rhi, r), nclo = std::min(clo, c), nchi = std::max(chi, c);
      const long long nr = nrhi - nrlo + win_rows;
      const long long nc = pad_tile_cols(nchi - tile_col0(nclo, elem_bytes) + win_cols, elem_bytes);
      if (nr * nc > cap) break;
      rlo = nrlo; rhi = nrhi; clo = nclo; chi = nchi;
      ++c1;
    }
    clo = tile_col0(clo, elem_bytes);
    const int nr = rhi - rlo + win_rows;
    const int nc = pad_tile_cols(chi - clo + win_cols, elem_bytes);
    box.push_back((int)c0);
    box.push_back(rlo);
    box.push_back(clo);
    box.push_back(nr);
    box.push_back(nc);
    box.push_back((int)(c1 - c0));
    maxcap = std::max(maxcap, (long long)nr * nc);
    c0 = c1;
  }
  return maxcap;
}

uint64_t Rng::next() {
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
uint64_t Rng::below(uint64_t n) { return n ? next() % n : 0; }

// k distinct indices of [0, n), sorted (Floyd's algorithm); all of them if k >= n.
std::vector<int> sample_distinct(Rng& rng, int n, int k) {
  std::vector<int> out;
  if (k >= n) {
    out.resize(n);
    std::iota(out.begin(), out.end(), 0);
    return out;
  }
  std::unordered_set<int> s;
  s.reserve(2 * k);
  for (int j = n - k; j < n; ++j) {
    int t = (int)rng.below((uint64_t)j + 1);
    if (!s.insert(t).second) s.insert(j);
  }
  out.assign(s.begin(), s.end());
  std::sort(out.begin(), out.end());
  return out;
}

// ---------------------------------------------------------------- dense linear algebra
static inline cplx cmul(cplx a, cplx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
static inline cplx cconjmul(cplx a, cplx b) { return {a.re * b.re + a.im * b.im, a.re * b.im - a.im * b.re}; }

void jacobi_svd(int m, int n, std::vector<cplx>& A, std::vector<cplx>& V, std::vector<double>& sigma) {
  V.assign((size_t)n * n, cplx{0, 0});
  for (int i = 0; i < n; ++i) V[(size_t)i * n + i] = {1, 0};
  const double tol = 1e-15;
  for (int sweep = 0; sweep < 80; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n - 1; ++p) {
      for (int q = p + 1; q < n; ++q) {
        cplx* ap = &A[(size_t)p * m];
        cplx* aq = &A[(size_t)q * m];
        double alpha = 0, beta = 0;
        cplx gamma{0, 0};
        for (int i = 0; i < m; ++i) {
          alpha += ap[i].re * ap[i].re + ap[i].im * ap[i].im;
          beta += aq[i].re * aq[i].re + aq[i].im * aq[i].im;
          cplx c = cconjmul(ap[i], aq[i]);
          gamma.re += c.re; gamma.im += c.im;
        }
        double g = std::hypot(gamma.re, gamma.im);
        if (g == 0.0 || g <= tol * std::sqrt(alpha * beta)) continue;
        off = std::max(off, g / std::sqrt(alpha * beta));
        cplx ph{gamma.re / g, -gamma.im / g};  // e^{-i theta}
        double zeta = (beta - alpha) / (2.0 * g);
        double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        for (int i = 0; i < m; ++i) {
          cplx x = ap[i], y = cmul(ph, aq[i]);
          ap[i] = {c * x.re - s * y.re, c * x.im - s * y.im};
          aq[i] = {s * x.re + c * y.re, s * x.im + c * y.im};
        }
        cplx* vp = &V[(size_t)p * n];
        cplx* vq = &V[(size_t)q * n];
        for (int i = 0; i < n; ++i) {
          cplx x = vp[i], y = cmul(ph, vq[i]);
          vp[i] = {c * x.re - s * y.re, c * x.im - s * y.im};
          vq[i] = {s * x.re + c * y.re, s * x.im + c * y.im};
        }
      }
    }
    if (off <= tol) break;
  }
  sigma.resize(n);
  for (int k = 0; k < n; ++k) {
    double s2 = 0;
    for (int i = 0; i < m; ++i) s2 += A[(size_t)k * m + i].re * A[(size_t)k * m + i].re + A[(size_t)k * m + i].im * A[(size_t)k * m + i].im;
    sigma[k] = std::sqrt(s2);
  }
  // sort descending (permute columns of A and V)
  std::vector<int> ord(n);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return sigma[a] > sigma[b]; });
  std::vector<cplx> A2((size_t)m * n), V2((size_t)n * n);
  std::vector<double> s2(n);
  for (int k = 0; k < n; ++k) {
    std::memcpy(&A2[(size_t)k * m], &A[(size_t)ord[k] * m], sizeof(cplx) * m);
    std::memcpy(&V2[(size_t)k * n], &V[(size_t)ord[k] * n], sizeof(cplx) * n);
    s2[k] = sigma[ord[k]];
  }
  A.swap(A2); V.swap(V2); sigma.swap(s2);
}

// Upper Cholesky factor of a Hermitian positive definite n x n column-major matrix: G = R^H R.
// G is overwritten by R (lower part zeroed).  Returns false on a non-positive pivot.
bool cholesky_upper(int n, std::vector<cplx>& G) {
  for (int j = 0; j < n; ++j) {
    double d = G[j + (size_t)j * n].re;
    for (int k = 0; k < j; ++k) {
      const cplx r = G[k + (size_t)j * n];
      d -= r.re * r.re + r.im * r.im;
    }
    if (!(d > 0.0)) return false;
    d = std::sqrt(d);
    G[j + (size_t)j * n] = {d, 0.0};
    for (int i = j + 1; i < n; ++i) {
      cplx acc = G[j + (size_t)i * n];  // G(j, i)
      for (int k = 0; k < j; ++k) {    // - sum_k conj(R(k, j)) R(k, i)
        const cplx a = G[k + (size_t)j * n], b = G[k + (size_t)i * n];
        acc.re -= a.re * b.re + a.im * b.im;
        acc.im -= a.re * b.im - a.im * b.re;
      }
      G[j + (size_t)i * n] = {acc.re / d, acc.im / d};
    }
    for (int i = j + 1; i < n; ++i) G[i + (size_t)j * n] = {0.0, 0.0};
  }
  return true;
}

// X = R^{-1} for an upper triangular n x n column-major R (back substitution, column by column).
void upper_inverse(int n, const std::vector<cplx>& R, std::vector<cplx>& X) {
  X.assign((size_t)n * n, cplx{0, 0});
  for (int c = 0; c < n; ++c) {
    for (int i = c; i >= 0; --i) {
      cplx acc = {i == c ? 1.0 : 0.0, 0.0};
      for (int k = i + 1; k <= c; ++k) acc = {acc.re - cmul(R[i + (size_t)k * n], X[k + (size_t)c * n]).re,
                                              acc.im - cmul(R[i + (size_t)k * n], X[k + (size_t)c * n]).im};
      const cplx d = R[i + (size_t)i * n];
      const double den = d.re * d.re + d.im * d.im;
      X[i + (size_t)c * n] = {(acc.re * d.re + acc.im * d.im) / den, (acc.im * d.re - acc.re * d.im) / den};
    }
  }
}

// C = A B for n x n column-major matrices (small, host).
void small_matmul(int n, const std::vector<cplx>& A, const std::vector<cplx>& B, std::vector<cplx>& C) {
  C.assign((size_t)n * n, cplx{0, 0});
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k) {
      const cplx b = B[k + (size_t)j * n];
      if (b.re == 0.0 && b.im == 0.0) continue;
      for (int i = 0; i < n; ++i) {
        const cplx t = cmul(A[i + (size_t)k * n], b);
        C[i + (size_t)j * n].re += t.re;
        C[i + (size_t)j * n].im += t.im;
      }
    }
}

std::vector<int> pivoted_columns(int m, int n, std::vector<cplx>& B, int k) {
  std::vector<int> piv;
  std::vector<double> nrm(n);
  std::vector<char> used(n, 0);
  for (int j = 0; j < n; ++j) {
    double s = 0;
    for (int i = 0; i < m; ++i) s += B[(size_t)j * m + i].re * B[(size_t)j * m + i].re + B[(size_t)j * m + i].im * B[(size_t)j * m + i].im;
    nrm[j] = s;
  }
  double n0 = *std::max_element(nrm.begin(), nrm.end());
  std::vector<cplx> qv(m);
  for (int s = 0; s < k && s < n; ++s) {
    int p = -1;
    double best = -1;
    for (int j = 0; j < n; ++j)
      if (!used[j] && nrm[j] > best) { best = nrm[j]; p = j; }
    if (p < 0 || best <= 1e-28 * n0) break;
    used[p] = 1;
    piv.push_back(p);
    double inv = 1.0 / std::sqrt(best);
    for (int i = 0; i < m; ++i) qv[i] = {B[(size_t)p * m + i].re * inv, B[(size_t)p * m + i].im * inv};
#pragma omp parallel for schedule(static)
    for (int j = 0; j < n; ++j) {
      if (used[j]) continue;
      cplx* b = &B[(size_t)j * m];
      cplx c{0, 0};
      for (int i = 0; i < m; ++i) { cplx t = cconjmul(qv[i], b[i]); c.re += t.re; c.im += t.im; }
      double s2 = 0;
      for (int i = 0; i < m; ++i) {
        cplx t = cmul(c, qv[i]);
        b[i].re -= t.re; b[i].im -= t.im;
        s2 += b[i].re * b[i].re + b[i].im * b[i].im;
      }
      nrm[j] = s2;
    }
  }
  return piv;
}

}  // namespace fio
