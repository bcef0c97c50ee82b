/*
 * fio.h -- C ABI of the B200-native fast Fourier integral operator apply
 * (Candes, Demanet, Ying, "Fast computation of Fourier integral operators",
 * arXiv math/0610051; the paper text is cited as PAPER.md:<line>).
 *
 * The library evaluates the discrete FIO of eq. (dfio), PAPER.md:165-168,
 *
 *     (Lf)(x) = (1/N) sum_{xi in Omega} a(x,xi) e^{2 pi i Phi(x,xi)} fhat(xi),
 *     fhat(xi) = (1/N) sum_{x in X} e^{-2 pi i x.xi} f(x)      (eq. dft)
 *
 * on the grid X = {(n1/N, n2/N)}, Omega = [-N/2, N/2)^2
 * (PAPER.md:172-174), with the wedge-decomposed algorithm of PAPER.md:332-378:
 * W angular wedges, per wedge a residual kernel separated
 * to rank q_l by a randomized skeleton, and per (l,t) a
 * type-2 NUFFT at the warped points (M_l^{-T} grad_xi Phi(x, xihat_l))
 * whose result is multiplied by alpha_lt(x) and summed
 * (PAPER.md:1296-1302).
 *
 * Preprocessing (fio_plan) is done once per (Phi, a, eps) and reused for many
 * f.  Evaluation (fio_apply) runs entirely in this
 * library's sm_100a CUDA kernels; there is no CPU fallback.
 *
 * Conventions used by every entry point
 *  - complex arrays are interleaved (re, im); C64 = 2 x float, C128 = 2 x double.
 *  - spatial arrays are row-major N x N over (n1, n2), x = (n1/N, n2/N); axis 0
 *    is x1 <-> xi1 (reading R14).
 *  - frequency arrays are N x N in FFT-natural order: index k stands for
 *    xi = k - N [k >= N/2].
 *  - every call returns fio_status: 0 ok, < 0 error (nothing was done, the
 *    message is in fio_last_error()), > 0 warning (the call did its work).
 *  - the library never frees caller memory; handles own their device memory
 *    and release it in fio_destroy.
 */
#ifndef FIO_B200_H
#define FIO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fio_plan_s* fio_handle; /* opaque, owned by the library */

typedef enum { FIO_C64 = 1, FIO_C128 = 2 } fio_dtype;

typedef enum {
  FIO_OK = 0,
  FIO_WNOTCERT = 1,   /* plan built, but a wedge's sampled separation error
                          exceeded 10 eps; it still evaluates */
  FIO_EINVAL = -1,    /* bad argument (message says which) */
  FIO_ENOMEM = -2,    /* device or host allocation failed */
  FIO_ECUDA = -3,     /* CUDA runtime error (launch or sync) */
  FIO_ENCCL = -4,     /* NCCL failure (libnccl.so.2 missing, communicator setup or reduce-scatter) */
  FIO_ENOTHOMOG = -5, /* reserved, never returned: the phase interface (fio_phase: the elliptic family
                         x.xi + b(x).xi +- sqrt(c1^2 xi1^2 + c2^2 xi2^2) given by its coefficient grids) is
                         homogeneous of degree 1 in xi by construction, so there is nothing to check */
  FIO_EINTERNAL = -6  /* internal invariant violated (a bug) */
} fio_status;

/* The phase, PAPER.md:54-61 (homogeneous of degree 1 in xi), given as data on X:
 *     Phi(x,xi) = x.xi + b(x).xi + s rho(x,xi),  rho = sqrt(c1(x)^2 xi1^2 + c2(x)^2 xi2^2),
 * s = rho_sign in {+1, -1} (0 means +1): Phi_+- of PAPER.md:1600-1603.
 * This family contains the identity (c = b = 0), the wave
 * propagator x.xi +- c|xi|t (c1 = c2 = c t), the paper's
 * ellipse phases (eq. nrphase) and every BASELINE config.
 * c1, c2: host arrays of N*N doubles (required).  b1, b2: N*N doubles or NULL (0).
 * The library copies them during fio_plan. */
typedef struct {
  const double* c1;
  const double* c2;
  const double* b1;
  const double* b2;
  int rho_sign;
} fio_phase;

typedef enum { FIO_AMP_SEPARABLE = 0, FIO_AMP_BESSEL_GRT = 1 } fio_amp_kind;

/* The amplitude (order-0 symbol).
 * kind FIO_AMP_SEPARABLE: rank-K separable on the grids, a(x,xi) = sum_{k<K} px_k(x) pxi_k(xi).
 * kind FIO_AMP_BESSEL_GRT (K = 0): the ellipse-GRT amplitude of eq. ellipses_amp
 *     a(x,xi) = (1/4 pi)(J0(2 pi rho_e) + s i Y0(2 pi rho_e)) e^{-s 2 pi i rho_e},
 *     rho_e = max(rho(x,xi), 1/2) (reading R22), rho and s from the phase
 *     (with r1 = r2 = r of eq. circlerad it is the paper's Table tbl:result_b).
 * K = 0 (px = pxi = NULL) is a == 1, the Egorov operator of PAPER.md:972-977.
 * px: K*N*N interleaved complex doubles over X; pxi: K*N*N over Omega in FFT
 * order.  Copied during fio_plan.  The amplitude is folded into the separated
 * kernel (reading R9). */
typedef struct {
  int K;
  const double* px;
  const double* pxi;
  int kind;
} fio_amplitude;

/* Options; fio_default_opts() fills the defaults shown. */
typedef struct {
  fio_dtype dtype;    /* FIO_C128 */
  int n_wedges;       /* 0 -> W = 8 round(2 sqrt(N)/8), >= 8 (reading R1) */
  int nufft_w;        /* 0 -> taps per dimension chosen from eps (reading R10); 3..12 */
  double nufft_beta;  /* 0 -> 2.30 w (exponential-of-semicircle kernel) */
  uint64_t seed;      /* 0x5EED: seed of the randomized separation */
  int device;         /* CUDA device ordinal; -1 -> current device */
  int rank, nranks;   /* 0, 1: this process owns the wedges assigned to `rank`
                         among `nranks` (BASELINE north_star (3)) */
  int r_init;         /* 32: initial skeleton size r of PAPER.md:1211-1221 */
  int r_max;          /* 512: cap of the doubling */
  int certify;        /* 1: compute the sampled error of PAPER.md:1464-1477 */
  int skeleton;       /* 0: store alpha' (fast).  1: skeleton storage of PAPER.md:1223-1241 --
                         keep only the skeleton columns C and V S^{-1} per wedge and rebuild
                         alpha' = A_[C] V S^{-1} (with the center phase) before each wedge's
                         interpolation; O(r q) storage per wedge, extra compute per apply */
  const void* nccl_id; /* NULL.  Else FIO_NCCL_ID_BYTES bytes of an NCCL unique id
                         (fio_nccl_unique_id on one rank, broadcast by the caller); fio_plan then
                         creates this rank's communicator (a collective call: every rank must call
                         fio_plan with the same id) and fio_apply ends with the cross-GPU sum.
                         NULL with nranks > 1: fio_apply returns this rank's N x N partial sum. */
  double wedge_overlap; /* 0: the paper's indicator wedges chi_l.  In (0, 1]: the
                         smooth polar-wedge partition of DESIGN.md reading R2 -- a C-infinity angular
                         taper of half-width wedge_overlap pi / W around every boundary ray, sum_l
                         chi_l = 1 exactly, so L is unchanged; each wedge's support,
                         box and rank grow with the overlap. */
  int paper_accept;   /* 0: skeleton columns by column pivoting on a random row sample, accepted when
                         q <= 3r/4 (reading R8; backed by the certification).  1: the paper's
                         column step -- r columns drawn uniformly, r doubled until
                         q <= r/3; rows as in the default.  Same operator; more
                         plan time. */
  int allgather;      /* 0: with a communicator every rank receives its (N/R) x N row slab.  1: every rank
                         receives the full N x N result -- the reduce-scatter into the rank's rows of
                         Lf_dev is followed by an in-place NCCL all-gather on the same stream (SURVEY.md
                         8(b) ownership).  Requires nccl_id (FIO_EINVAL without it). */
} fio_opts;

#define FIO_NCCL_ID_BYTES 128

/* Write a fresh NCCL unique id (FIO_NCCL_ID_BYTES bytes) to id_out (host).  Host-only; loads
 * libnccl.so.2 at run time (FIO_ENCCL if it cannot). */
fio_status fio_nccl_unique_id(void* id_out);

void fio_default_opts(fio_opts* opts);

/* Build a plan for the N x N operator (N even, 5-smooth, 8 <= N <= 4096) at
 * separation accuracy eps in (0, 1) (the relative singular
 * value cutoff, reading R6), eps >= 1e-6 for FIO_C64 and >= 1e-11 for FIO_C128
 * (FIO_EINVAL below: the arithmetic could not deliver it, reading R24).  opts may be NULL (defaults).  Runs on the device
 * (kernel-entry evaluation, Gram products, factor expansion) and the host
 * (partition, pivoting, small Jacobi SVDs).  Synchronous.
 * Returns FIO_OK, FIO_WNOTCERT, or an error (*out is then NULL). */
fio_status fio_plan(fio_handle* out, int N, const fio_phase* phase, const fio_amplitude* amp,
                    double eps, const fio_opts* opts);

/* Evaluate L f.  f_dev: device N x N complex of the plan dtype (caller-owned,
 * read-only).  Lf_dev: device complex of the plan dtype (caller-owned, fully
 * overwritten; must not overlap f_dev):
 *  - nranks == 1: the N x N result;
 *  - nranks > 1 with a communicator (opts.nccl_id): every rank passes the full
 *    f and receives its row slab of L f, rows [rank N/R, (rank+1) N/R) -- an
 *    (N/R) x N array -- after the wedge partials of all ranks are summed by an
 *    NCCL reduce-scatter on `stream` (L = sum_l L_l; the
 *    collective: every rank must call fio_apply);
 *  - the same with opts.allgather = 1: the full N x N L f on every rank (the
 *    reduce-scatter writes this rank's rows, an in-place all-gather the rest);
 *  - nranks > 1 without a communicator: this rank's N x N partial sum over its
 *    own wedges (the DC term on rank 0 only), for the caller to sum.
 * stream: a cudaStream_t (NULL = legacy default stream).  Asynchronous on
 * `stream`; one apply in flight per handle (the workspace is per handle).
 * Errors: FIO_EINVAL (arguments), FIO_ECUDA (launch), FIO_ENCCL (collective). */
fio_status fio_apply(fio_handle h, const void* f_dev, void* Lf_dev, void* stream);

/* The adjoint: out = L~* g, the exact conjugate transpose of the fast
 * operator fio_apply evaluates (so <L~f, g> = <f, L~* g> to rounding), approximating
 * (L* g)(x) = (1/N) sum_xi e^{2 pi i x.xi} (1/N) sum_y conj(a(y,xi)) e^{-2 pi i Phi(y,xi)} g(y).
 * g_dev, out_dev: device N x N complex of the plan dtype (no overlap).  With nranks > 1 the
 * result is this rank's row slab (with a communicator) or its partial over its wedges (without;
 * the DC term on rank 0), exactly as for fio_apply.  Asynchronous on stream;
 * shares the handle's workspace with fio_apply (one call in flight per handle).  The type-1
 * spreading step accumulates with atomics: the last bits may vary between runs. */
fio_status fio_apply_adjoint(fio_handle h, const void* g_dev, void* out_dev, void* stream);

/* Multi-RHS apply (NEXT-2): Lf_b = L f_b for b < nrhs; f_dev holds nrhs contiguous N x N complex
 * arrays of the plan dtype, Lf_dev nrhs contiguous outputs of fio_apply's shape (device, no
 * overlap).  The FFT stages run per input;
 * per wedge the interpolation then serves every input from one alpha' (in skeleton storage mode
 * alpha' is rebuilt once per wedge for the whole batch).  The first call with a larger nrhs
 * allocates (nrhs - 1) extra spectra and fine-grid workspaces (synchronizing `stream`). */
fio_status fio_apply_batch(fio_handle h, int nrhs, const void* f_dev, void* Lf_dev, void* stream);

/* End-to-end variant: f_host / Lf_host are HOST buffers (pinned for overlap);
 * the host->device copy, the apply and the device->host copy are enqueued on
 * `stream`, which is synchronized before return.  Lf_host has the shape
 * fio_apply gives Lf_dev (the row slab with a communicator). */
fio_status fio_apply_host(fio_handle h, const void* f_host, void* Lf_host, void* stream);

/* Streaming end-to-end variant (serving loop): Lf_i = L f_i for i < count, f_host holding `count`
 * contiguous N x N HOST inputs and Lf_host `count` contiguous HOST outputs of fio_apply's shape
 * (both pinned for overlap; no overlap between them).  Every input is copied to the device and
 * every result back inside the call, pipelined: the copy of input i+1 and the read-back of result
 * i-1 run on two plan-owned copy streams while apply i runs on `stream` (double-buffered device
 * staging, allocated on first use).  The results equal fio_apply's bit for bit (a communicator
 * plan: every rank calls it with the same count).  `stream` is synchronized before return.
 * Errors: FIO_EINVAL (arguments, count < 0), FIO_ECUDA, FIO_ENCCL. */
fio_status fio_apply_host_stream(fio_handle h, int count, const void* f_host, void* Lf_host, void* stream);

fio_status fio_destroy(fio_handle h);

typedef struct {
  int N, W, nufft_w, dtype, rank, nranks;
  int n_owned;            /* wedges owned by this rank */
  int sum_q;              /* sum of q_l over owned wedges */
  int certified;          /* 1 if every owned wedge passed the sampled check */
  double nufft_beta;
  double max_sep_err;     /* max sampled relative Frobenius error */
  double plan_seconds;
  size_t alpha_bytes, beta_bytes, workspace_bytes, fine_elems, p1_elems;
  int launches_per_apply; /* kernels one fio_apply enqueues */
  size_t meta_bytes;      /* K3 point-group tables (anchors, slot indices, offsets) */
  long long slots;        /* sum over owned wedges of the padded K3 group slots */
  long long max_tile_cap; /* largest K3 chunk footprint (fine-grid elements) */
  long long k3_thread_slots; /* K3 chunks x threads per CTA (slots / P / this = thread fill) */
  double rank_balance;    /* predicted max/mean per-rank cost of the wedge assignment (1 if nranks = 1) */
  long long slot_terms;   /* sum over owned wedges of K3 slots x q_l (K3 work units per apply) */
  int group_p;            /* points per K3 group */
  int k3_window_rows;     /* rows of the K3 interpolation window (w or w+1 rounded up to even) */
  size_t skeleton_bytes;  /* skeleton storage: C and V S^{-1} of every owned wedge (0 otherwise);
                             alpha_bytes is then the size of the shared rebuild scratch */
  int k3_window_cols;     /* columns of the K3 interpolation window (w or w+1) */
  int k3_streams;         /* concurrent K3 streams of an apply (wedge l on stream l mod k3_streams) */
  int has_comm;           /* 1 if the plan owns an NCCL communicator (fio_apply returns the row slab) */
  int out_rows;           /* rows of the array fio_apply writes: N / nranks with a communicator, else N */
  double wedge_overlap;   /* 0: indicator wedges; > 0: smooth partition (opts.wedge_overlap) */
  long long members;      /* sum over owned wedges of |supp chi_l| (frequencies carried) */
} fio_info;

fio_status fio_plan_info(fio_handle h, fio_info* info);

/* Per owned wedge: l, q_l, n1, n2, n1f, n2f, M (4 ints, row-major), xi_c (2 ints),
 * r (final skeleton size) and the sampled error; arrays of length >= n_owned
 * (any pointer may be NULL). */
fio_status fio_plan_wedges(fio_handle h, int* l, int* q, int* box /* 4 per wedge */,
                           int* M /* 4 per wedge */, int* xc /* 2 per wedge */, int* r,
                           double* sep_err);

/* Host-only geometry of the partition (no GPU needed; used by the CPU tests):
 * wedge_of[k1*N+k2] = wedge of xi(k) in [0,W) or -1 for xi = 0 (PAPER.md:214-217,
 * readings R3/R4); for each wedge: M (4 ints), xi_c (2), box n1,n2 and fine n1f,n2f
 * (4) as chosen by the plan (reading R5). */
fio_status fio_geometry(int N, int W, int* wedge_of, int* M, int* xc, int* box);

/* Partition weights chi_l(xi) of every wedge l < W at the frequency (xi1, xi2) (host only):
 * the indicator for overlap 0, the smooth taper of reading R2 for overlap in (0, 1]. */
fio_status fio_partition_weights(int W, double overlap, int xi1, int xi2, double* chi /* W */);

/* Wedge -> rank assignment used for nranks > 1 (owner[l] in [0, nranks)), from
 * per-wedge costs (longest-processing-time greedy, deterministic). Host-only. */
fio_status fio_assign_wedges(int W, const double* cost, int nranks, int* owner);

/* Live per-stage timing for bench.py: after fio_profile_begin(h, S), each of the
 * next S applies records CUDA events between its kernels on its stream;
 * fio_profile_end synchronizes and writes, per stage (K0 rows, K0 cols, K1, K2,
 * K3 -- 5 entries), the SUM of the stage durations in milliseconds over the
 * recorded applies, and the number of applies recorded. */
fio_status fio_profile_begin(fio_handle h, int max_applies);
fio_status fio_profile_end(fio_handle h, double* stage_ms /* 5 */, int* n_applies);

/* Plan save / load.  fio_plan_save writes the separation of every owned
 * wedge in compact form -- skeleton columns C and Y = V S^{-1} (U = A(:, C) Y),
 * skeleton rows R and Z = U_R^+ (beta = T = Z A(R, members)), the chosen r and
 * the sampled error -- plus a header (N, W, dtype, taps, eps, beta, seed, rank, nranks and an FNV-1a
 * hash of the phase / amplitude arrays).  fio_plan_load takes the same arguments as fio_plan plus
 * the path; it validates the header against them (FIO_EINVAL on any mismatch or a malformed file)
 * and rebuilds the plan with U and beta recomputed from the factors by the same kernels, skipping
 * the randomized search: the loaded plan applies bit-identically to the saved one.  The file is
 * host-endian binary; the caller owns path. */
fio_status fio_plan_save(fio_handle h, const char* path);
fio_status fio_plan_load(fio_handle* out, const char* path, int N, const fio_phase* phase,
                         const fio_amplitude* amp, double eps, const fio_opts* opts);

const char* fio_last_error(void); /* thread-local message of the last error */
const char* fio_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FIO_B200_H */
