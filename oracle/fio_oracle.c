/*
 * fio_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct FP64 CPU reference for the discrete Fourier
 * integral operator of arXiv math/0610051 (Candes, Demanet, Ying).  Only
 * tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and the
 * `--impl reference` arm) may load this library.  It shares no code, header,
 * table or constant generator with the CUDA product under
 * paper_math_0610051_b200/ and it never reads anything that path produced.
 *
 * Every function restates a definition of the paper:
 *
 *   oracle_dft2        eq. (dft)
 *                      fhat(xi) = (1/N) sum_{x in X} e^{-2 pi i x.xi} f(x)
 *   oracle_fio_points  eq. (dfio)
 *                      (Lf)(x) = (1/N) sum_{xi in Omega} a(x,xi) e^{2 pi i Phi(x,xi)} fhat(xi)
 *                      optionally restricted to a set of wedges W_l
 *                      (L_l of PAPER.md:236-241), which is how the per-wedge
 *                      partial sums of the wedge-sharded path are checked.
 *   oracle_wedge_of    the angular wedges W_l, with
 *                      sqrt(N) replaced by the wedge count W (DESIGN.md
 *                      reading R1) and arg(xi) = atan2(xi2, xi1) (reading R14).
 *   oracle_nudft2      the nonuniform Fourier series of step 3 of the
 *                      evaluation, summed directly.
 *   oracle_fio_adjoint_freq  the discrete adjoint of PAPER.md:1393-1396,
 *                      widehat(L* g)(xi) = (1/N) sum_y conj(a(y,xi)) e^{-2 pi i Phi(y,xi)} g(y).
 *
 * The operator family (the phase and amplitude are DATA, given on the grids):
 *     Phi(x,xi) = x.xi + b(x).xi + s rho(x,xi),  rho = sqrt(c1(x)^2 xi1^2 + c2(x)^2 xi2^2),
 *                 s = +1 or -1 (Phi_+- of PAPER.md:1600-1603)
 *     a(x,xi)   = sum_k px_k(x) pxi_k(xi)      (amp_kind 0; K = 0  ->  a == 1, the Egorov
 *                                                operator of PAPER.md:972-977)
 *     a(x,xi)   = (1/4pi) (J0(2 pi rho_e) + s i Y0(2 pi rho_e)) e^{-s 2 pi i rho_e}
 *                 (amp_kind 1: eq. ellipses_amp, the Appendix
 *                  split 2 J0 = (J0 + iY0) + (J0 - iY0)), with the
 *                  regularisation rho_e = max(rho, 1/2) (reading R22)
 * This covers every phase used by the paper's experiments with elliptic radii
 * (eq. nrphase; the wave phase x.xi +- c|xi|t,
 * PAPER.md:94-97) and all five BASELINE.json configurations.
 *
 * Layouts: complex arrays are interleaved (re, im) doubles.  Spatial arrays
 * are row-major over (n1, n2) with x = (n1/N, n2/N).  Frequency
 * arrays (fhat, pxi_k) are in FFT-natural order: index k in [0,N) stands for
 * xi = k - N [k >= N/2] (-N/2 <= xi_i < N/2).
 *
 * Argument reduction: x.xi = (n1 xi1 + n2 xi2)/N is reduced exactly in
 * integer arithmetic; the remaining real part of the phase is reduced to its
 * fractional part before the multiplication by 2 pi.  Sums are plain FP64 in
 * a fixed order (xi1 outer, xi2 inner) per output point.
 */
#define _DEFAULT_SOURCE 1
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static const double TWO_PI = 6.283185307179586476925286766559;

/* amplitude of eq. ellipses_amp at radius rho, phase sign s */
static void bessel_amp(double rho, int s, double* ar, double* ai) {
    const double PI = 3.14159265358979323846264338327950288;
    double re = rho < 0.5 ? 0.5 : rho;
    double J = j0(TWO_PI * re), Y = y0(TWO_PI * re);
    double fr = re - floor(re);
    double c = cos(TWO_PI * fr), sn = -(double)s * sin(TWO_PI * fr); /* e^{-s 2 pi i re} */
    /* (J + s i Y)(c + i sn) / (4 pi) */
    *ar = (J * c - (double)s * Y * sn) / (4.0 * PI);
    *ai = (J * sn + (double)s * Y * c) / (4.0 * PI);
}

static inline int freq_of_index(int k, int N) { return k >= N / 2 ? k - N : k; }

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* eq. (dft).  Separable direct DFT, O(N^3): first over n2
 * for every n1, then over n1.  The kernel e^{-2 pi i m/N} is taken from an
 * exact table indexed by m = (n k) mod N. */
void oracle_dft2(int N, const double* f, double* fhat) {
    double* tc = (double*)malloc(sizeof(double) * N);
    double* ts = (double*)malloc(sizeof(double) * N);
    double* tmp = (double*)malloc(sizeof(double) * 2 * (size_t)N * N);
    for (int m = 0; m < N; ++m) {
        tc[m] = cos(TWO_PI * (double)m / (double)N);
        ts[m] = -sin(TWO_PI * (double)m / (double)N);
    }
    /* tmp[n1][k2] = sum_{n2} f[n1][n2] e^{-2 pi i n2 k2 / N} */
#pragma omp parallel for schedule(static)
    for (int n1 = 0; n1 < N; ++n1) {
        for (int k2 = 0; k2 < N; ++k2) {
            double sr = 0.0, si = 0.0;
            for (int n2 = 0; n2 < N; ++n2) {
                int m = (int)(((int64_t)n2 * k2) % N);
                double fr = f[2 * ((size_t)n1 * N + n2)], fi = f[2 * ((size_t)n1 * N + n2) + 1];
                sr += fr * tc[m] - fi * ts[m];
                si += fr * ts[m] + fi * tc[m];
            }
            tmp[2 * ((size_t)n1 * N + k2)] = sr;
            tmp[2 * ((size_t)n1 * N + k2) + 1] = si;
        }
    }
    /* fhat[k1][k2] = (1/N) sum_{n1} tmp[n1][k2] e^{-2 pi i n1 k1 / N} */
#pragma omp parallel for schedule(static)
    for (int k1 = 0; k1 < N; ++k1) {
        for (int k2 = 0; k2 < N; ++k2) {
            double sr = 0.0, si = 0.0;
            for (int n1 = 0; n1 < N; ++n1) {
                int m = (int)(((int64_t)n1 * k1) % N);
                double fr = tmp[2 * ((size_t)n1 * N + k2)], fi = tmp[2 * ((size_t)n1 * N + k2) + 1];
                sr += fr * tc[m] - fi * ts[m];
                si += fr * ts[m] + fi * tc[m];
            }
            fhat[2 * ((size_t)k1 * N + k2)] = sr / (double)N;
            fhat[2 * ((size_t)k1 * N + k2) + 1] = si / (double)N;
        }
    }
    free(tc);
    free(ts);
    free(tmp);
}

/* Wedges W_l = { xi : (2l-1) pi / W <= arg xi < (2l+1) pi / W },
 * PAPER.md:214-217, arg measured from (1,0), wrapped to
 * [-pi/W, 2 pi - pi/W).  xi = 0 has no angle and belongs to no wedge (-1). */
int oracle_wedge_of(int W, int xi1, int xi2) {
    if (xi1 == 0 && xi2 == 0) return -1;
    const double PI = 3.14159265358979323846264338327950288;
    double th = atan2((double)xi2, (double)xi1); /* (-pi, pi] */
    double lo = -PI / (double)W;
    if (th < lo) th += 2.0 * PI;
    int l = (int)floor((th - lo) / (2.0 * PI / (double)W));
    if (l < 0) l = 0;
    if (l >= W) l = W - 1;
    return l;
}

/* eq. (dfio), at the flat output indices pts[p] = n1*N+n2.
 * wedge_sel: NULL -> every xi in Omega (the full operator); otherwise only
 * xi != 0 with wedge_sel[oracle_wedge_of(W, xi)] != 0, plus xi = 0 iff
 * include_dc (the partial operators L_l of PAPER.md:239-241).
 * b1, b2 may be NULL (b == 0).  K == 0 -> a == 1. */
void oracle_fio_points(int N, const double* c1, const double* c2, const double* b1,
                       const double* b2, int K, const double* px, const double* pxi,
                       const double* fhat, int64_t npts, const int64_t* pts, int W,
                       const int* wedge_sel, int include_dc, int rho_sign, int amp_kind,
                       double* out) {
    int* wsel = NULL;
    if (wedge_sel) {
        /* per-frequency selection mask, FFT-natural order */
        wsel = (int*)malloc(sizeof(int) * (size_t)N * N);
        for (int k1 = 0; k1 < N; ++k1)
            for (int k2 = 0; k2 < N; ++k2) {
                int x1 = freq_of_index(k1, N), x2 = freq_of_index(k2, N);
                int l = oracle_wedge_of(W, x1, x2);
                wsel[(size_t)k1 * N + k2] = (l < 0) ? (include_dc != 0) : (wedge_sel[l] != 0);
            }
    }
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t p = 0; p < npts; ++p) {
        int64_t idx = pts[p];
        int n1 = (int)(idx / N), n2 = (int)(idx % N);
        double C1 = c1[idx], C2 = c2[idx];
        double B1 = b1 ? b1[idx] : 0.0, B2 = b2 ? b2[idx] : 0.0;
        double sr = 0.0, si = 0.0;
        for (int k1 = 0; k1 < N; ++k1) {
            int x1 = freq_of_index(k1, N);
            for (int k2 = 0; k2 < N; ++k2) {
                size_t fi = (size_t)k1 * N + k2;
                if (wsel && !wsel[fi]) continue;
                int x2 = freq_of_index(k2, N);
                /* x.xi mod 1 exactly: ((n1 xi1 + n2 xi2) mod N) / N */
                int64_t m = ((int64_t)n1 * x1 + (int64_t)n2 * x2) % N;
                if (m < 0) m += N;
                /* b(x).xi + rho(x,xi), reduced to its fractional part */
                double rho = sqrt(C1 * C1 * (double)x1 * (double)x1 + C2 * C2 * (double)x2 * (double)x2);
                double s = B1 * (double)x1 + B2 * (double)x2 + (double)rho_sign * rho;
                s -= floor(s);
                double ph = (double)m / (double)N + s;
                ph -= floor(ph);
                double cr = cos(TWO_PI * ph), ci = sin(TWO_PI * ph);
                /* amplitude a(x,xi) = sum_k px_k(x) pxi_k(xi) */
                double ar = 1.0, ai = 0.0;
                if (amp_kind == 1) {
                    bessel_amp(rho, rho_sign, &ar, &ai);
                } else if (K > 0) {
                    ar = 0.0;
                    for (int k = 0; k < K; ++k) {
                        const double* pxk = px + 2 * (size_t)k * N * N;
                        const double* pik = pxi + 2 * (size_t)k * N * N;
                        double ur = pxk[2 * idx], ui = pxk[2 * idx + 1];
                        double vr = pik[2 * fi], vi = pik[2 * fi + 1];
                        ar += ur * vr - ui * vi;
                        ai += ur * vi + ui * vr;
                    }
                }
                /* kernel = a e^{2 pi i Phi} */
                double kr = ar * cr - ai * ci, ki = ar * ci + ai * cr;
                double hr = fhat[2 * fi], hi = fhat[2 * fi + 1];
                sr += kr * hr - ki * hi;
                si += kr * hi + ki * hr;
            }
        }
        out[2 * p] = sr / (double)N;
        out[2 * p + 1] = si / (double)N;
    }
    free(wsel);
}

/* Direct type-2 nonuniform Fourier series on an n1 x n2 box of integer
 * frequencies k_a in [-n_a/2, n_a/2) (coeffs row-major over (k1 + n1/2,
 * k2 + n2/2)):  F(y) = sum_k c_k e^{2 pi i (y1 k1 + y2 k2)}, the sum of step 3
 * of the evaluation, at arbitrary real points y. */
void oracle_nudft2(int n1, int n2, const double* coeffs, int64_t npts, const double* y,
                   double* out) {
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < npts; ++p) {
        double y1 = y[2 * p], y2 = y[2 * p + 1];
        double sr = 0.0, si = 0.0;
        for (int i1 = 0; i1 < n1; ++i1) {
            int k1 = i1 - n1 / 2;
            for (int i2 = 0; i2 < n2; ++i2) {
                int k2 = i2 - n2 / 2;
                double ph = y1 * (double)k1 + y2 * (double)k2;
                ph -= floor(ph);
                double cr = cos(TWO_PI * ph), ci = sin(TWO_PI * ph);
                size_t j = (size_t)i1 * n2 + i2;
                double hr = coeffs[2 * j], hi = coeffs[2 * j + 1];
                sr += cr * hr - ci * hi;
                si += cr * hi + ci * hr;
            }
        }
        out[2 * p] = sr;
        out[2 * p + 1] = si;
    }
}

/* Discrete adjoint, PAPER.md:1393-1396:
 *   widehat(L* g)(xi) = (1/N) sum_{y in X} conj(a(y,xi)) e^{-2 pi i Phi(y,xi)} g(y)
 * at the FFT-natural frequency indices fidx[p] = k1*N+k2. */
void oracle_fio_adjoint_freq(int N, const double* c1, const double* c2, const double* b1,
                             const double* b2, int K, const double* px, const double* pxi,
                             const double* g, int64_t nfreq, const int64_t* fidx, int rho_sign,
                             int amp_kind, double* out) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t p = 0; p < nfreq; ++p) {
        int64_t fi = fidx[p];
        int x1 = freq_of_index((int)(fi / N), N), x2 = freq_of_index((int)(fi % N), N);
        double sr = 0.0, si = 0.0;
        for (int n1 = 0; n1 < N; ++n1) {
            for (int n2 = 0; n2 < N; ++n2) {
                size_t idx = (size_t)n1 * N + n2;
                int64_t m = ((int64_t)n1 * x1 + (int64_t)n2 * x2) % N;
                if (m < 0) m += N;
                double C1 = c1[idx], C2 = c2[idx];
                double B1 = b1 ? b1[idx] : 0.0, B2 = b2 ? b2[idx] : 0.0;
                double rho = sqrt(C1 * C1 * (double)x1 * (double)x1 + C2 * C2 * (double)x2 * (double)x2);
                double s = B1 * (double)x1 + B2 * (double)x2 + (double)rho_sign * rho;
                s -= floor(s);
                double ph = (double)m / (double)N + s;
                ph -= floor(ph);
                double cr = cos(TWO_PI * ph), ci = -sin(TWO_PI * ph); /* e^{-2 pi i Phi} */
                double ar = 1.0, ai = 0.0;
                if (amp_kind == 1) {
                    bessel_amp(rho, rho_sign, &ar, &ai);
                } else if (K > 0) {
                    ar = 0.0;
                    for (int k = 0; k < K; ++k) {
                        const double* pxk = px + 2 * (size_t)k * N * N;
                        const double* pik = pxi + 2 * (size_t)k * N * N;
                        double ur = pxk[2 * idx], ui = pxk[2 * idx + 1];
                        double vr = pik[2 * fi], vi = pik[2 * fi + 1];
                        ar += ur * vr - ui * vi;
                        ai += ur * vi + ui * vr;
                    }
                }
                ai = -ai; /* conj(a) */
                double kr = ar * cr - ai * ci, ki = ar * ci + ai * cr;
                double hr = g[2 * idx], hi = g[2 * idx + 1];
                sr += kr * hr - ki * hi;
                si += kr * hi + ki * hr;
            }
        }
        out[2 * p] = sr / (double)N;
        out[2 * p + 1] = si / (double)N;
    }
}
