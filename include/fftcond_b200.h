/* fftcond_b200.h -- C ABI of the B200 FFT field-iteration library.
 *
 * Drop-in boundary for the reference solver loops of `fftcond`
 * (arXiv 2001.08289 companion package).  The reference has no FFI of its
 * own: its replaceable seam is the private pair
 *
 *     _solve_h(pmap, cfg, accelerated)   reference pkg/src/fftcond/solvers.py:280-331
 *     _solve_aug(pmap, cfg, accelerated) reference pkg/src/fftcond/solvers.py:366-443
 *
 * reached through _DISPATCH / solve() (solvers.py:481-491).  fftc_solve()
 * replaces both loops for d = 2 (the reference's dimension) and d = 3.
 * Everything above the seam -- SolverConfig validation (solvers.py:110-120),
 * the reference-medium choice _reference_h / _reference_aug (:221-240,
 * :334-352), map_t / solve_p (transform.py:99-110, :152-168) -- stays on the
 * host and only its scalar outputs cross this boundary (fftc_params).
 *
 * Plain C types only: no torch, no CUDA types in the signatures (streams are
 * passed as void*, a cudaStream_t or NULL for the legacy default stream).
 *
 * Error convention (mirrors the reference split between exceptions and
 * numerical outcomes, solvers.py:243-277): parameter errors are raised by the
 * host layer before the call; a nonzero return code means a CUDA /
 * allocation / unsupported-shape failure and fftc_last_error() describes it.
 * Converged / MaxIters / Diverged / degenerate-flux are RESULTS, returned in
 * fftc_result, never errors.
 */
#ifndef FFTCOND_B200_H
#define FFTCOND_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* schemes: same order as reference transform.py:23-39 (SchemeKind) */
enum { FFTC_BASIC = 0, FFTC_EM = 1, FFTC_BASIC_SUB = 2, FFTC_EM_SUB = 3 };
/* termination: reference solvers.py:54-57 (TerminationStatus) */
enum { FFTC_CONVERGED = 0, FFTC_MAX_ITERS = 1, FFTC_DIVERGED = 2 };

typedef struct fftc_problem {
  int32_t d;          /* 2 or 3 */
  int32_t reserved;
  int64_t n[3];       /* n[0] = nx (fastest), n[1] = ny, n[2] = nz (1 for d = 2) */
  const uint8_t* chi; /* DEVICE pointer, nz*ny*nx bytes, 1 = phase 1 (PhaseMap.chi, geometry.py:20-39) */
} fftc_problem;

typedef struct fftc_params {
  int32_t scheme;       /* FFTC_* */
  int32_t reserved;
  double sigma1[2];     /* inclusion conductivity (re, im)            SolverConfig.sigma1 */
  double sigma0[2];     /* reference medium from _reference_h/_aug    solvers.py:221,334 */
  double t[2];          /* map_t(sigma1) (substituted schemes)        transform.py:99 */
  double p1[2], p2[2], p3[2]; /* solve_p(interval)                    transform.py:152 */
  double e0[3][2];      /* applied field, d complex components        SolverConfig.e0 */
  double tol;           /* SolverConfig.tol */
  int64_t max_iters;    /* SolverConfig.max_iters */
  double gamma1_scale;  /* test hook, reference spectral_ops.py:29-30 (1.0) */
} fftc_params;

typedef struct fftc_result {
  int32_t status;          /* FFTC_CONVERGED / FFTC_MAX_ITERS / FFTC_DIVERGED */
  int32_t degenerate_flux; /* SolveResult.degenerate_flux */
  int64_t iterations;      /* len(history) */
  double sigma_star[2];    /* last recorded sigma* (or last evaluated if none, solvers.py:323) */
  double mean_E[3][2];     /* compensated-style mean of the returned E field */
  double mean_J[3][2];     /* mean of the returned J field */
  int64_t kernel_launches; /* number of library kernels launched by this call */
  double device_ms;        /* device time of the solve (CUDA events) */
} fftc_result;

/* Run one solve on the device.
 *   history : HOST buffer of history_cap records x 3 doubles
 *             (sigma*_re, sigma*_im, residual); record k-1 is iteration k.
 *   E, J    : nullable DEVICE buffers of d*N complex128 (component-major,
 *             layout (c, z, y, x) like VectorField.data, spectral_ops.py:58-70)
 *   aug     : nullable DEVICE buffer of 3*d*N complex128, (Q, S, T) of the
 *             substituted schemes (SolveResult.aug_field)
 *   stream  : cudaStream_t or NULL.
 * Returns 0 on success. */
int fftc_solve(const fftc_problem* problem, const fftc_params* params, double* history,
               int64_t history_cap, void* E, void* J, void* aug, fftc_result* out, void* stream);

/* BASELINE config 5: n_points independent solves on one grid (e.g. a sweep
 * of sigma1), histories laid out [n_points][history_cap][3], one result per
 * point.  Fields are not returned (only the per-point averages).  Replaces
 * sequential calls of solve() such as cli.cmd_compare (cli.py:352-408) and
 * analysis.misestimation_report (analysis.py:166-201). */
int fftc_solve_batch(const fftc_problem* problem, const fftc_params* params, int32_t n_points,
                     double* histories, int64_t history_cap, fftc_result* out, void* stream);

/* z-slab decomposition of a 3-D solve over `world` ranks (BASELINE config 4,
 * north star: "slab-decomposed across the 8 GPUs ... NCCL all-to-all FFT
 * transposes").  Rank r owns z-planes [z0, z0+nzl) of the state and of the
 * work fields A_z/B_z (layout (c, z_l, y, x)); the z pass runs on a y-slab
 * copy A_y/B_y (layout (c, y_l, z, x), y-planes [y0, y0+nyl)) that the caller
 * produces with an all-to-all transpose after FFTC_SLAB_ROWS_FWD and
 * transposes back (A only) after FFTC_SLAB_MID.  Every phase returns
 * rank-local partial sums the caller all-reduces:
 *   INIT     -> out[6]  e0 - (local sum of the initial iterate)/N   (per component re, im)
 *   ROWS_FWD -> out[7]  local <j> contribution (6) and sum |Js|^2 chi (1)
 *   MID      -> out[1]  local sum_x |Gamma j|^2
 *   ROWS_INV -> out[6]  as INIT for the new iterate
 * The caller forms the global delta = sum_r out_r - (world-1) e0 and installs
 * it with fftc_slab_set_delta; fftc_slab_monitor runs the reference stopping
 * rule (solvers.py:243-277) on the global totals {<j> (6), js2, parseval} and
 * returns {stopped, status, degenerate, nrec, sigma*_re, sigma*_im, residual}. */
enum { FFTC_SLAB_INIT = 0, FFTC_SLAB_ROWS_FWD = 1, FFTC_SLAB_MID = 2, FFTC_SLAB_ROWS_INV = 3 };
typedef struct fftc_slab_desc {
  int32_t d;          /* 3 */
  int32_t reserved;
  int64_t n[3];       /* GLOBAL nx, ny, nz */
  int64_t z0, nzl;    /* this rank's z-slab */
  int64_t y0, nyl;    /* this rank's y-slab after the transpose */
  const uint8_t* chi; /* DEVICE, local z-slab of the indicator (nzl*ny*nx bytes) */
} fftc_slab_desc;
typedef struct fftc_slab fftc_slab;
int fftc_slab_create(const fftc_slab_desc* desc, const fftc_params* params, void* A_z, void* B_z, void* A_y,
                     void* B_y, fftc_slab** out, void* stream);
int fftc_slab_phase(fftc_slab* slab, int32_t phase, double* out, void* stream);
int fftc_slab_set_delta(fftc_slab* slab, const double* delta6, void* stream);
int fftc_slab_monitor(fftc_slab* slab, const double* totals8, double* record7, void* stream);
int fftc_slab_finalize(fftc_slab* slab, void* E, void* J, void* aug, double* means12, void* stream);
void fftc_slab_destroy(fftc_slab* slab);
/* Fused transposes (NVLink peer memory): after this call the y forward pass
 * of FFTC_SLAB_ROWS_FWD writes its output rows directly into the y-slab
 * buffers of their owning ranks, and FFTC_SLAB_MID writes its result back
 * into the owning ranks' z-slab buffers, so the caller skips both
 * all-to-alls and only orders the phases (a barrier after ROWS_FWD; the
 * all-reduce after MID).  Ay, Az (and By for em / em_sub): `world` device
 * pointers, rank order, peer-accessible from this rank.  Returns 3 when the
 * grid cannot use the fused passes (y and z lines of 256..1024).  In this
 * mode the work buffers are library-private in layout: A_z/B_z and A_y/B_y
 * switch to the z-blocked layout (2^zs z-planes of a row adjacent, zs chosen
 * per slab as for the monolithic solve; FFTC_ZBLOCK=0 keeps the plain
 * layouts), so callers must not read them as (c, z_l, y, x) / (c, y_l, z, x)
 * after fftc_slab_set_peers. */
int fftc_slab_set_peers(fftc_slab* slab, int32_t world, void* const* Ay, void* const* By, void* const* Az,
                        void* stream);

/* Device buffers shared between rank processes (CUDA IPC), for the fused
 * transposes when ranks live in different processes: allocate the slab work
 * buffers here, export their handles (64 bytes each), open the peers'
 * handles (mapped over NVLink between GPUs, or aliased on one GPU), and pass
 * the resulting pointers to fftc_slab_set_peers. */
int fftc_ipc_alloc(int64_t bytes, void** ptr);
int fftc_ipc_free(void* ptr);
int fftc_ipc_handle(void* ptr, void* handle64);
int fftc_ipc_open(const void* handle64, void** ptr);
int fftc_ipc_close(void* ptr);

/* Same contract, host-resident chi and outputs (the library copies in and
 * out; E/J/aug host buffers are nullable).  For FFI users without a device
 * allocator. */
int fftc_solve_host(const fftc_problem* problem_with_host_chi, const fftc_params* params,
                    double* history, int64_t history_cap, void* E_host, void* J_host,
                    void* aug_host, fftc_result* out);

/* Operator API on DEVICE fields of d*N complex128 (layout as above).
 *
 * fftc_fft: in-place unnormalised DFT of every component along each axis in
 * axes_mask (bit 0 = x, 1 = y, 2 = z); inverse != 0 uses exp(+i...).
 * Building block of numpy.fft.fftn/ifftn as called by the reference
 * (spectral_ops.py:123,128).
 *
 * fftc_gamma1: out = Gamma_1(in), the curl-free zero-mean projection with
 * multiplier k k^T/|k|^2 * scale (k = 0 dropped, Nyquist kept), replacing
 * _gamma1_arr (spectral_ops.py:120-128); scale mirrors the _gamma1_scale
 * test hook (:29-30).  in may equal out. */
int fftc_fft(const fftc_problem* problem, void* data, int32_t inverse, int32_t axes_mask, void* stream);
int fftc_gamma1(const fftc_problem* problem, const void* in, void* out, double scale, void* stream);

/* Pointwise augmented-space operators on DEVICE (Q, S, T) fields, each
 * d*N complex128 (AugmentedField, spectral_ops.py:141-173), chi from the
 * problem.  coef = {p1, p2, p3, t, sigma0} as (re, im) pairs (10 doubles).
 *   FFTC_AUG_CHI         apply_chi_aug     (spectral_ops.py:227-237): (p1 u, p2 u, p3 u),
 *                        u = chi (p1 Q + p2 S + p3 T)
 *   FFTC_AUG_LOCAL_A     apply_local_A     (spectral_ops.py:240-250): A = (t-1) chi'' + I
 *   FFTC_AUG_INV_SHIFTED invert_shifted_A  (spectral_ops.py:253-278): (A + sigma0 I)^-1
 * S and T outputs are zero off chi.  Outputs may alias inputs.  The
 * singular-shift checks (sigma0 = -1, sigma0 = -t) are the host layer's. */
enum { FFTC_AUG_CHI = 0, FFTC_AUG_LOCAL_A = 1, FFTC_AUG_INV_SHIFTED = 2 };
int fftc_aug_apply(const fftc_problem* problem, int32_t op, const double* coef, const void* Q, const void* S,
                   const void* T, void* Q_out, void* S_out, void* T_out, void* stream);

/* j = sigma e on DEVICE fields, sigma = sigma1 on chi and 1 elsewhere
 * (extract_sigma_star, solvers.py:147-155; the loop's j, :286, :311). */
int fftc_apply_sigma(const fftc_problem* problem, const double* sigma1, const void* e, void* j, void* stream);

/* Deterministic reductions of DEVICE fields (fixed-order trees; the
 * reference's compensated sums, spectral_ops.py:33-55, :96-106, :182-200).
 * Results go to the HOST array out; the call synchronises the stream.
 *   FFTC_RED_SUM          out[2d]: per-component sums of a (re, im)
 *   FFTC_RED_DOT          out[2]:  sum over components and voxels of conj(a) b
 *   FFTC_RED_NORM2        out[1]:  sum |a|^2
 *   FFTC_RED_OFF_SUPPORT  out[1]:  number of phase-2 voxels where a (or b,
 *                                  nullable) is nonzero (_check_support, :176-179)
 * mask = FFTC_MASK_CHI restricts SUM/DOT/NORM2 to phase-1 voxels. */
enum { FFTC_RED_SUM = 0, FFTC_RED_DOT = 1, FFTC_RED_NORM2 = 2, FFTC_RED_OFF_SUPPORT = 3 };
enum { FFTC_MASK_NONE = 0, FFTC_MASK_CHI = 1 };
int fftc_reduce(const fftc_problem* problem, int32_t op, int32_t mask, const void* a, const void* b, double* out,
                void* stream);

/* Per-kernel timing.  fftc_profile(1) resets the counters and brackets every
 * subsequent library launch with CUDA events on its stream (device time,
 * harvested at the solver's existing synchronisation points);
 * fftc_kernel_stats() returns up to max_entries {kind, launches, total_ms}. */
typedef struct fftc_kstat {
  char name[32];
  int64_t launches;
  double total_ms;
} fftc_kstat;
void fftc_profile(int32_t enable);
int fftc_kernel_stats(fftc_kstat* out, int32_t max_entries);

/* 1 if fftc_solve accepts an axis of length n: even and >= 2, the
 * reference's PhaseMap rule (geometry.py:37). */
int fftc_supported_length(int64_t n);

/* 1 if an axis of length n runs the fused sweeps (powers of two 2..4096).
 * Grids with any other even axis run the general path (pointwise kernels
 * around cuFFT) in fftc_solve, fftc_fft and fftc_gamma1. */
int fftc_fused_length(int64_t n);

/* Description of the last error on this thread ("" if none). */
const char* fftc_last_error(void);

/* ABI version (major*100 + minor). */
int fftc_version(void);

/* Total kernels launched by this library in this process. */
int64_t fftc_launch_count(void);

/* Work-field layout of this thread's last fftc_solve: the z-block shift
 * (2^shift consecutive z-planes of a y-row adjacent; 0 = the reference
 * (c, z, y, x) layout).  Diagnostics only; results do not depend on it. */
int32_t fftc_last_layout(void);

#ifdef __cplusplus
}
#endif
#endif /* FFTCOND_B200_H */
