// sweeps.cuh -- the fused per-iteration sweeps of the FFT field iteration.
//
// One reference iteration (solvers.py:300-321 for basic/em, :395-432 for
// basic_sub/em_sub) becomes, on a 2-D grid, three kernels:
//
//   sweep 1 (rows, x-FFT):   prologue = the pointwise update that produces
//                            the fields to transform (j = sigma e, or the
//                            augmented flux Jq and the EM residual field R),
//                            reductions <j> (and sum |Js|^2 chi), x-FFT.
//   sweep 2 (columns):       y-FFT, Gamma_1 projection k k^T/|k|^2 in
//                            registers (spectral_ops.py:120-128), residual by
//                            Parseval, y-iFFT of the field the update needs;
//                            the last CTA runs the stopping monitor
//                            (solvers.py:243-277) on device.
//   sweep 3 (rows, x-iFFT):  epilogue = the state update for iteration k+1
//                            and the reduction <Q_raw> / <e_raw> that gives
//                            the next mean-field pin delta (solvers.py:309,416).
//
// On a 3-D grid the y pass and y^-1 pass are separate column sweeps and the
// Gamma projection moves to the z pass.  All reductions are deterministic:
// fixed per-thread order, shuffle trees, per-CTA partials and a last-CTA
// fixed-order combine (no floating-point atomics).
#pragma once
#include "fft_engine.cuh"

namespace fftc {

enum SchemeId { BASIC = 0, EM = 1, BASIC_SUB = 2, EM_SUB = 3 };
enum StatusId { ST_CONVERGED = 0, ST_MAXITERS = 1, ST_DIVERGED = 2 };

constexpr double DIVERGENCE_FACTOR = 1e6;  // solvers.py:50
constexpr double TINY = 1e-300;            // solvers.py:51
constexpr int NQMAX = 8;                   // reduction slots per CTA

struct DevState {
  int stopped;
  int status;
  int degenerate;
  int nrec;          // records written so far (== iterations)
  long long k;       // index of the iteration being executed (1-based)
  int has_prev;
  int pad0;
  double res0;
  double2 prev_sstar;
  double2 last_sstar;  // sigma* of the last evaluated iteration (recorded or not)
  double2 delta[3];    // mean-field pin of the current iterate
  double2 jmean[3];    // <j> / <Jq> of the current iterate
  double js2;          // sum |Js|^2 chi
  double parseval;     // sum_k |Gamma j^|^2
  double2 meanE[3];
  double2 meanJ[3];
  unsigned int counter;  // last-CTA detection
  unsigned int pad1;
};

// Bulk L2 prefetch of a contiguous range (one instruction, no registers):
// issued for the NEXT line while the current line's FFT runs, so its loads
// hit L2 instead of paying the HBM round trip on the critical path.
__device__ __forceinline__ void l2_prefetch(const void* p, unsigned bytes) {
  if (bytes >= 16) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes & ~15u) : "memory");
}

struct Args {
  int d, nx, ny, nz;
  long long N;
  const uint8_t* chi;
  const int2* row_ext;  // per row (z,y): [first, last+1) x-extent of phase 1 (empty: x0 >= x1)
  // chi rows permuted for the TMA row sweeps (16 elements per thread): row
  // byte t*16 + i holds chi[t + i*nx/16], so a thread's 16 phase flags are one
  // 16-byte shared-memory load (k_chi_perm16)
  const uint8_t* chiT;
  int row_e;  // elements per thread of that order: row_e(nx, scheme), 16 or 8
  // Compact S/T slots (the memory-lean em_sub schedule, abi.cu): when rowoff
  // is set, X[1] and X[2] hold only the phase-1 voxels -- row r's, in x
  // order, at [rowoff[r], rowoff[r+1]) of each component's block of M --
  // and chiR holds, in chiT's thread-blocked order, 0 for phase 2 and
  // 1 + the voxel's rank among its row's phase-1 voxels.
  const long long* rowoff;  // rows + 1 entries, or null (full-grid slots)
  long long M;              // phase-1 voxel count (component stride of the compact slots)
  const uint16_t* chiR;
  double2* X[3];  // state slots: e_raw | Q_raw, S_raw, T_raw
  double2* A;     // work field 0 (d*N)
  double2* B;     // work field 1 (d*N)
  double2* outE;  // finalize targets (nullable)
  double2* outJ;
  double2* outAug;  // (3, d, grid)
  double* partials;
  double* history;  // [hist_cap][3]
  int hist_cap;
  int op_mode;  // 1: operator API call -- no stop flag, no monitor
  DevState* st;
  unsigned long long* dbg;  // debug phase counters (FFTC_PHASE_TIMING builds), else null
  int dist;                 // slab-decomposed solve: sweeps leave rank-local partials, the host combines
  // z-blocked layout of the work fields A/B (3-D): row (z, y) of component c
  // starts at c*N + (((z >> zbs)*ny + y) << zbs | (z & (2^zbs - 1)))*nx, i.e.
  // 2^zbs consecutive z-planes of one y-row are adjacent, so a z-line touches
  // nz / 2^zbs 2 MB pages instead of nz.  zbs = 0 is the reference layout.
  int zbs;
  const double2* tw[3];  // twiddles for n_x, n_y, n_z
  // scalars (host-prepared, see abi.cu)
  double2 sigma1, s0, e0[3];
  double e0sq, tol, inv_n, gscale;
  long long max_iters;
  double2 inv_s0;                  // 1/s0
  double2 inv_sum1, inv_sum2;      // 1/(sigma1+s0), 1/(1+s0)
  double2 sum1, sum2;              // sigma1+s0, 1+s0
  double2 sm1, sm2;                // sigma1-s0, 1-s0
  double2 two_s0_e0[3];            // (2 s0) e0_c
  double2 p1, p2, p3;
  double2 tm1p1, tm1p2, tm1p3;     // (t-1) p_i
  double2 cq, cs;                  // p1*((t-1)p1), p2*((t-1)p1)
  double2 sinv;                    // 1/(1+s0)
  double2 cinv_p1, cinv_p2, cinv_p3;  // ((t-1)/(t+s0)) p_i
};

// Elements per thread of the TMA row sweeps on rows of length L, scheme S
// (rows_tma.cuh): 16 (radix-16 stages), except rows of 512 = 8 x 8 x 8 of the
// substituted schemes, where 8 per thread costs the same two exchanges as
// 16 x 2 x 16 and twice the warps fit an SM.  Measured at 512^3 (8 vs 16, ms):
// em_sub sweep 1 5.31 / 5.39, sweep 3 3.25 / 3.70; basic_sub 2.94 / 2.75 and
// 3.12 / 3.40; basic sweep 1 2.50 / 2.30 and em 4.87 / 4.58 (already near the
// HBM rate with 16), so basic and em keep 16.  FFTC_ROW_E512 = 16 switches it off.
#ifndef FFTC_ROW_E512
#define FFTC_ROW_E512 8
#endif
__host__ __device__ constexpr int row_e(int L, int S) {
  return (L == 512 && (S == 2 || S == 3)) ? FFTC_ROW_E512 : 16;  // (S: BASIC_SUB = 2, EM_SUB = 3)
}

// index of voxel (row, x) in the thread-blocked row order of chiT / chiR
// (E = Args::row_e elements per thread: x = t + i*nx/E sits at E t + i)
__device__ __forceinline__ long long tblock_index(long long row, int x, int nx, int E) {
  const int T = nx / E;
  return row * nx + E * (x % T) + x / T;
}

// compact S/T slot of voxel p = row*nx + x, component c (lean layout), or -1
// on phase 2
__device__ __forceinline__ long long compact_slot(const Args& a, int c, long long p) {
  const long long row = p / a.nx;
  const int x = (int)(p - row * a.nx);
  const int code = a.chiR[tblock_index(row, x, a.nx, a.row_e)];
  return code ? (long long)c * a.M + a.rowoff[row] + (code - 1) : -1;
}

// element offset of row `row` = z*ny + y of component c of a work field (A/B)
__device__ __forceinline__ size_t work_off(const Args& a, int c, long long row) {
  const int z = (int)(row / a.ny), y = (int)(row - (long long)z * a.ny);
  const int s = a.zbs;
  const long long r = ((long long)((z >> s) * a.ny + y) << s) | (z & ((1 << s) - 1));
  return (size_t)c * a.N + (size_t)r * a.nx;
}

// ----------------------------------------------------------------------------
// deterministic block reduction + last-CTA combine
// ----------------------------------------------------------------------------
template <int NQ>
__device__ __forceinline__ void warp_sum(double (&acc)[NQ]) {
#pragma unroll
  for (int q = 0; q < NQ; ++q)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_down_sync(0xffffffffu, acc[q], o);
}

// Reduce acc over the CTA, write the CTA partial, and return true in the
// last CTA to finish, with `tot` holding the grid total (fixed order).
template <int NQ>
__device__ bool grid_reduce(double (&acc)[NQ], double (&tot)[NQ], const Args& a) {
  __shared__ double red[32][NQ];
  __shared__ int am_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  warp_sum<NQ>(acc);
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NQ; ++q) red[warp][q] = acc[q];
  __syncthreads();
  if (threadIdx.x == 0) {
    double s[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) s[q] = 0.0;
    for (int w = 0; w < nw; ++w)
#pragma unroll
      for (int q = 0; q < NQ; ++q) s[q] += red[w][q];
#pragma unroll
    for (int q = 0; q < NQ; ++q) a.partials[(size_t)blockIdx.x * NQ + q] = s[q];
    __threadfence();
    unsigned prev = atomicAdd(&a.st->counter, 1u);
    am_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return false;
  __threadfence();
  double s[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) s[q] = 0.0;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x)
#pragma unroll
    for (int q = 0; q < NQ; ++q) s[q] += __ldcg(&a.partials[(size_t)b * NQ + q]);
  warp_sum<NQ>(s);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NQ; ++q) red[warp][q] = s[q];
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NQ; ++q) tot[q] = 0.0;
  for (int w = 0; w < nw; ++w)
#pragma unroll
    for (int q = 0; q < NQ; ++q) tot[q] += red[w][q];
  if (threadIdx.x == 0) a.st->counter = 0;
  return true;
}

// accumulate complex v into slot pair (2c, 2c+1) with a runtime component c
template <int NQ>
__device__ __forceinline__ void acc_c(double (&acc)[NQ], int c, double2 v) {
#pragma unroll
  for (int cc = 0; cc < 3; ++cc)
    if (2 * cc + 1 < NQ && c == cc) {
      acc[2 * cc] += v.x;
      acc[2 * cc + 1] += v.y;
    }
}

// ----------------------------------------------------------------------------
// pointwise algebra shared by the sweeps (reference formulas)
// ----------------------------------------------------------------------------
__device__ __forceinline__ double2 sigma_at(const Args& a, bool in1) {
  return in1 ? a.sigma1 : make_double2(1.0, 0.0);
}

// augmented local operator A (solvers.py:355-363) on one pixel/component
struct AugFlux {
  double2 jq, js, jt;
};
__device__ __forceinline__ AugFlux apply_A(const Args& a, bool in1, double2 q, double2 s, double2 t) {
  AugFlux f;
  if (in1) {
    double2 u = cadd(cadd(cmul(a.p1, q), cmul(a.p2, s)), cmul(a.p3, t));
    f.jq = cadd(cmul(a.tm1p1, u), q);
    f.js = cadd(cmul(a.tm1p2, u), s);
    f.jt = cadd(cmul(a.tm1p3, u), t);
  } else {
    f.jq = q;  // u = 0: (t-1) p1 * 0 + q
    f.js = czero();
    f.jt = czero();
  }
  return f;
}

// (A + s0 I)^{-1} W update of em_sub (solvers.py:408-411)
__device__ __forceinline__ void em_sub_update(const Args& a, bool in1, double2 wq, double2 ws, double2 wt,
                                              double2& q, double2& s, double2& t) {
  if (in1) {
    double2 u = cadd(cadd(cmul(a.p1, wq), cmul(a.p2, ws)), cmul(a.p3, wt));
    q = cmul(a.sinv, csub(wq, cmul(a.cinv_p1, u)));
    s = cmul(a.sinv, csub(ws, cmul(a.cinv_p2, u)));
    t = cmul(a.sinv, csub(wt, cmul(a.cinv_p3, u)));
  } else {
    q = cmul(a.sinv, wq);
    s = czero();
    t = czero();
  }
}

// Jq, Js of the pinned iterate (solvers.py:419-420)
__device__ __forceinline__ void pinned_flux(const Args& a, bool in1, double2 jq_raw, double2 js_raw, double2 dl,
                                            double2& jq, double2& js) {
  if (in1) {
    jq = cadd(cadd(jq_raw, cmul(a.cq, dl)), dl);
    js = cadd(js_raw, cmul(a.cs, dl));
  } else {
    jq = cadd(jq_raw, dl);
    js = js_raw;
  }
}

// ----------------------------------------------------------------------------
// stopping monitor (solvers.py:243-277), one thread
// ----------------------------------------------------------------------------
static __device__ __forceinline__ void monitor_step(const Args& a, double total_sq) {
  DevState* st = a.st;
  double2 jm[3];
  double den2 = 0.0;
  double2 s = czero();
  for (int c = 0; c < a.d; ++c) {
    jm[c] = st->jmean[c];
    den2 += cabs2(jm[c]);
    // np.vdot(e0, jmean): conj(e0) . jmean
    double2 e = a.e0[c];
    s = cadd(s, make_double2(e.x * jm[c].x + e.y * jm[c].y, e.x * jm[c].y - e.y * jm[c].x));
  }
  const double den = sqrt(den2);
  const double2 sstar = make_double2(s.x / a.e0sq, s.y / a.e0sq);
  st->last_sstar = sstar;
  if (den < TINY && isfinite(den)) {  // solvers.py:315-317 / :424-426
    st->degenerate = 1;
    st->status = ST_DIVERGED;
    st->stopped = 1;
    return;
  }
  const double res = sqrt(total_sq * a.inv_n) / den;
  if (!(isfinite(res) && isfinite(sstar.x) && isfinite(sstar.y))) {  // :256-260
    st->status = ST_DIVERGED;
    st->stopped = 1;
    return;
  }
  const int slot = st->nrec % a.hist_cap;
  a.history[3 * slot + 0] = sstar.x;
  a.history[3 * slot + 1] = sstar.y;
  a.history[3 * slot + 2] = res;
  st->nrec += 1;
  if (st->nrec == 1) st->res0 = res;
  bool settled = true;
  if (st->has_prev) {
    double2 dlt = csub(sstar, st->prev_sstar);
    settled = hypot(dlt.x, dlt.y) <= a.tol * hypot(sstar.x, sstar.y);
  }
  if (res <= a.tol && settled) {
    st->status = ST_CONVERGED;
    st->stopped = 1;
    return;
  }
  if (st->res0 > 0.0 && res > DIVERGENCE_FACTOR * st->res0) {
    st->status = ST_DIVERGED;
    st->stopped = 1;
    return;
  }
  st->prev_sstar = sstar;
  st->has_prev = 1;
  if (st->k >= a.max_iters) {  // loop exhausted: status stays MaxIters
    st->stopped = 1;
    return;
  }
  st->k += 1;
}

// ----------------------------------------------------------------------------
// shared memory buffer accessor for fft_line
// ----------------------------------------------------------------------------
struct SmemBuf {
  double2* base;
  int stride;  // distance between channel buffers (double2 units)
  __device__ __forceinline__ double2* operator()(int c) const { return base + c * stride; }
};
struct SyncAll {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
// named barrier over n threads (a multiple of 32) -- a group of warps
struct HalfSync {
  int id;
  int n;
  __device__ __forceinline__ void operator()() const { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
};

// L2 prefetch of everything a row sweep reads for line `ln` = (c, row).
// S/T slots are fetched only over the row's phase-1 extent.
template <int S, int L, bool SWEEP3>
__device__ __forceinline__ void prefetch_row_inputs(const Args& a, long long ln, long long lines, long long rows) {
  if (ln >= lines) return;
  const int c = (int)(ln / rows);
  const long long row = ln - (long long)c * rows;
  const size_t off = (size_t)c * a.N + (size_t)row * L;
  constexpr unsigned RB = (unsigned)(L * sizeof(double2));
  l2_prefetch(a.chi + (size_t)row * L, L);
  if (SWEEP3) l2_prefetch(a.A + work_off(a, c, row), RB);
  if (!SWEEP3 || S == BASIC || S == BASIC_SUB) l2_prefetch(a.X[0] + off, RB);
  if (S == BASIC_SUB || S == EM_SUB) {
    const int2 ext = a.row_ext[row];
    if (ext.x < ext.y) {
      const int x0 = ext.x & ~1;  // 32-B aligned start
      const unsigned nb = (unsigned)((ext.y - x0) * sizeof(double2) + 15) & ~15u;
      if (SWEEP3 && S == EM_SUB) l2_prefetch(a.X[0] + off + x0, nb);
      l2_prefetch(a.X[1] + off + x0, nb);
      if (S == EM_SUB) l2_prefetch(a.X[2] + off + x0, nb);
    }
  }
}

// ============================================================================
// sweep 1: rows (x-pass), forward.  Line = (component c, row r); a CTA runs
// G lines at a time (one per thread group of T = L/E threads).
// ============================================================================
template <int S>
struct Sweep1Traits;
template <>
struct Sweep1Traits<BASIC> { static constexpr int C = 1; static constexpr int NQ = 6; };
template <>
struct Sweep1Traits<EM> { static constexpr int C = 2; static constexpr int NQ = 6; };
template <>
struct Sweep1Traits<BASIC_SUB> { static constexpr int C = 1; static constexpr int NQ = 7; };
template <>
struct Sweep1Traits<EM_SUB> { static constexpr int C = 2; static constexpr int NQ = 7; };

template <int S, int L, int E, int G>
__global__ void __launch_bounds__(G * Sweep1Traits<S>::C * (L / E), 2) k_sweep1(Args a) {
  // The C output channels of a line (EM residual field R and flux J) are
  // split across C thread groups that share the line's inputs (the second
  // group's loads hit L1/L2), so each thread carries one channel.
  using P = Plan<L, E>;
  constexpr int CH = Sweep1Traits<S>::C;
  constexpr int NQ = Sweep1Traits<S>::NQ;
  constexpr int T = P::T;
  extern __shared__ double2 smem[];
  if (a.st->stopped) return;
  const int t = threadIdx.x % T, ch = (threadIdx.x / T) % CH, g = threadIdx.x / (T * CH);
  const bool jchan = (ch == CH - 1);  // the channel carrying the flux j / Jq
  const long long rows = (long long)a.ny * a.nz;
  const long long lines = rows * a.d;
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  SmemBuf buf{smem + (g * CH + ch) * P::LP, 0};
  double2* OUT = (CH == 2 && ch == 1) ? a.B : a.A;
  for (long long line0 = (long long)blockIdx.x * G; line0 < lines; line0 += (long long)gridDim.x * G) {
    const long long line = line0 + g;
    const bool live = line < lines;
    const int c = live ? (int)(line / rows) : 0;
    const long long row = live ? line - (long long)c * rows : 0;
    const size_t off = (size_t)c * a.N + (size_t)row * L;
    const uint8_t* chi = a.chi + (size_t)row * L;
    const double2 dl = a.st->delta[c];
    const size_t woff = work_off(a, c, row);  // work field A/B row
    if (t == 0 && ch == 0) prefetch_row_inputs<S, L, false>(a, line + (long long)gridDim.x * G, lines, rows);
    // gather first: every load of the line is issued before any is used
    // (written as one loop, the per-element branches kept each chi/X pair
    // waiting on the previous one -- 16 serial round trips per line)
    bool in1v[E];
    double2 xq[E], xs[E], xt[E];
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int x = pos_first<L, E>(false, t, i);
      in1v[i] = live && chi[x] != 0;
      xq[i] = live ? a.X[0][off + x] : czero();
    }
    if constexpr (S == BASIC_SUB || S == EM_SUB) {
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int x = pos_first<L, E>(false, t, i);
        xs[i] = in1v[i] ? a.X[1][off + x] : czero();
        xt[i] = (S == EM_SUB && in1v[i]) ? a.X[2][off + x] : czero();
      }
    }
    double2 v[1][E];
#pragma unroll
    for (int i = 0; i < E; ++i) {
      if (!live) {
        v[0][i] = czero();
        continue;
      }
      const bool in1 = in1v[i];
      if constexpr (S == BASIC) {
        double2 j = cmul(sigma_at(a, in1), cadd(xq[i], dl));  // j = sigma e  (solvers.py:310-311)
        v[0][i] = j;
        acc_c<NQ>(acc, c, j);
      } else if constexpr (S == EM) {
        const double2 er = xq[i];
        if (jchan) {
          const double2 j = cmul(sigma_at(a, in1), cadd(er, dl));  // j = sigma (e_raw + delta)
          v[0][i] = j;
          acc_c<NQ>(acc, c, j);
        } else {
          v[0][i] = cmul(in1 ? a.sm1 : a.sm2, er);  // r = (sigma - s0) e_raw  (:303)
        }
      } else {
        const double2 q = xq[i];
        const AugFlux f = apply_A(a, in1, q, xs[i], xt[i]);  // (:412)
        if (jchan) {
          double2 jq, js;
          pinned_flux(a, in1, f.jq, f.js, dl, jq, js);
          v[0][i] = jq;
          acc_c<NQ>(acc, c, jq);
          if (in1) acc[6] += cabs2(js);  // sum |Js|^2 chi  (:429)
        } else {
          v[0][i] = csub(f.jq, cmul(a.s0, q));  // Rq = Jq_raw - s0 Q_raw  (:398)
        }
      }
    }
    fft_line<L, E, 1, false>(v, t, a.tw[0], buf, SyncAll{});
    if (live) {
#pragma unroll
      for (int i = 0; i < E; ++i) OUT[woff + pos_last<L, E>(false, t, i)] = v[0][i];
    }
  }
  double tot[NQ];
  if (grid_reduce<NQ>(acc, tot, a) && threadIdx.x == 0) {
    for (int c = 0; c < a.d; ++c) a.st->jmean[c] = make_double2(tot[2 * c] * a.inv_n, tot[2 * c + 1] * a.inv_n);
    if constexpr (NQ > 6) a.st->js2 = tot[NQ - 1];
    else a.st->js2 = 0.0;
  }
}

// ============================================================================
// sweep 3: rows (x-pass), inverse + state update.  Line = (c, row).
// ============================================================================
template <int S, int L, int E, int G>
__global__ void __launch_bounds__(G*(L / E), 2) k_sweep3(Args a) {
  using P = Plan<L, E>;
  constexpr int NQ = 6;
  constexpr int T = P::T;
  extern __shared__ double2 smem[];
  if (a.st->stopped) return;
  const int t = threadIdx.x % T, g = threadIdx.x / T;
  const long long rows = (long long)a.ny * a.nz;
  const long long lines = rows * a.d;
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  SmemBuf buf{smem + g * P::LP, P::LP};
  for (long long line0 = (long long)blockIdx.x * G; line0 < lines; line0 += (long long)gridDim.x * G) {
    const long long line = line0 + g;
    const bool live = line < lines;
    const int c = live ? (int)(line / rows) : 0;
    const long long row = live ? line - (long long)c * rows : 0;
    const size_t off = (size_t)c * a.N + (size_t)row * L;
    const uint8_t* chi = a.chi + (size_t)row * L;
    const double2 dl = a.st->delta[c];
    const size_t woff = work_off(a, c, row);  // work field A/B row
    if (t == 0) prefetch_row_inputs<S, L, true>(a, line + (long long)gridDim.x * G, lines, rows);
    double2 v[1][E];
#pragma unroll
    for (int i = 0; i < E; ++i) v[0][i] = live ? a.A[woff + pos_first<L, E>(true, t, i)] : czero();
    // the update's inputs are loaded before the transform so their latency
    // hides behind it (after it, the state stores kept them serial)
    bool in1v[E];
    double2 xq[E], xs[E], xt[E];
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int x = pos_last<L, E>(true, t, i);
      in1v[i] = live && chi[x] != 0;
      xq[i] = (live && (S == BASIC || S == BASIC_SUB)) ? a.X[0][off + x] : czero();
    }
    fft_line<L, E, 1, true>(v, t, a.tw[0], buf, SyncAll{});
    if (!live) continue;
    // S/T (phase 1 only) after the transform: across it they would spill;
    // em_sub gathers and updates half a line at a time for the same reason
    constexpr int CHK = (S == EM_SUB && E > 1) ? E / 2 : E;
#pragma unroll
    for (int i0 = 0; i0 < E; i0 += CHK) {
    if constexpr (S == BASIC_SUB || S == EM_SUB) {
#pragma unroll
      for (int i = i0; i < i0 + CHK; ++i) {
        const int x = pos_last<L, E>(true, t, i);
        if (S == EM_SUB) xq[i] = in1v[i] ? a.X[0][off + x] : czero();  // read on phase 1 only
        xs[i] = in1v[i] ? a.X[1][off + x] : czero();
        xt[i] = (S == EM_SUB && in1v[i]) ? a.X[2][off + x] : czero();
      }
    }
#pragma unroll
    for (int i = i0; i < i0 + CHK; ++i) {
      const int x = pos_last<L, E>(true, t, i);
      const bool in1 = in1v[i];
      const double2 gq = cscale(v[0][i], a.inv_n);  // ifft normalisation 1/N
      double2 qn;
      if constexpr (S == BASIC) {
        // e_raw <- (e_raw + delta) - g / s0      (solvers.py:306)
        qn = csub(cadd(xq[i], dl), cmul(gq, a.inv_s0));
        a.X[0][off + x] = qn;
      } else if constexpr (S == EM) {
        // w = 2 s0 e0 + (I - 2 Gamma) r;  e_raw = w / (sigma + s0)   (:303-308)
        double2 w = cadd(a.two_s0_e0[c], gq);
        qn = cmul(w, in1 ? a.inv_sum1 : a.inv_sum2);
        a.X[0][off + x] = qn;
      } else if constexpr (S == BASIC_SUB) {
        // Q_raw <- Q - g/s0 ; S_raw <- chi (S - Js/s0)   (:405-406)
        double2 q = xq[i];
        qn = csub(cadd(q, dl), cmul(gq, a.inv_s0));
        a.X[0][off + x] = qn;
        if (in1) {
          double2 s = xs[i];
          AugFlux f = apply_A(a, true, q, s, czero());
          double2 jq, js;
          pinned_flux(a, true, f.jq, f.js, dl, jq, js);
          a.X[1][off + x] = csub(s, cmul(js, a.inv_s0));
        }
      } else {
        // em_sub: W from the raw iterate, then (A + s0)^-1 W   (:398-411)
        double2 wq = cadd(a.two_s0_e0[c], gq);
        double2 ws = czero(), wt = czero();
        if (in1) {
          double2 q = xq[i], s = xs[i], tt = xt[i];
          AugFlux f = apply_A(a, true, q, s, tt);
          const double2 rs = csub(f.js, cmul(a.s0, s));  // Rs = Js_raw - s0 S_raw
          ws = make_double2(-rs.x, -rs.y);
          wt = csub(f.jt, cmul(a.s0, tt));               // Rt = Jt_raw - s0 T_raw
        }
        double2 sn, tn;
        em_sub_update(a, in1, wq, ws, wt, qn, sn, tn);
        a.X[0][off + x] = qn;
        if (in1) {
          a.X[1][off + x] = sn;
          a.X[2][off + x] = tn;
        }
      }
      acc_c<NQ>(acc, c, qn);
    }
    }
  }
  double tot[NQ];
  if (grid_reduce<NQ>(acc, tot, a) && threadIdx.x == 0) {
    for (int c = 0; c < a.d; ++c) {
      double2 m = make_double2(tot[2 * c] * a.inv_n, tot[2 * c + 1] * a.inv_n);
      a.st->delta[c] = csub(a.e0[c], m);  // delta = e0 - <raw>  (:309, :416)
    }
  }
}

// ============================================================================
// plain row transform (operator API / tests): line = (c, row) of field A,
// in place, optional scale on output.
// ============================================================================
template <bool INV, int L, int E, int G>
__global__ void __launch_bounds__(G*(L / E)) k_row_plain(Args a, double scale) {
  using P = Plan<L, E>;
  constexpr int T = P::T;
  extern __shared__ double2 smem[];
  const int t = threadIdx.x % T, g = threadIdx.x / T;
  const long long lines = (long long)a.ny * a.nz * a.d;
  SmemBuf buf{smem + g * P::LP, P::LP};
  for (long long line0 = (long long)blockIdx.x * G; line0 < lines; line0 += (long long)gridDim.x * G) {
    const long long line = line0 + g;
    const bool live = line < lines;
    const size_t off = (size_t)(live ? line : 0) * L;
    double2 v[1][E];
#pragma unroll
    for (int i = 0; i < E; ++i) v[0][i] = live ? a.A[off + pos_first<L, E>(INV, t, i)] : czero();
    fft_line<L, E, 1, INV>(v, t, a.tw[0], buf, SyncAll{});
    if (live)
#pragma unroll
      for (int i = 0; i < E; ++i) a.A[off + pos_last<L, E>(INV, t, i)] = cscale(v[0][i], scale);
  }
}

// ============================================================================
// column sweeps.  A "line" is a strip of W adjacent x-columns of one field
// along an axis with element stride `stride`; the line origin is
// outer*ostride + strip*W.  A CTA runs G lines at a time.  MODE:
//   MID_BASIC : fwd, g = Gamma F (Parseval), inv, write back      (basic, basic_sub)
//   MID_EM    : field 0: fwd, (I - 2 Gamma) F, inv, write back;
//               field 1: fwd, Parseval of Gamma F only            (em, em_sub)
//   COL_FWD / COL_INV : plain transform of one component          (3-D y passes)
// ============================================================================
enum ColMode { MID_BASIC = 0, MID_EM = 1, COL_FWD = 2, COL_INV = 3 };

struct ColGeom {
  int axis;           // twiddle table / wave-number axis of the line (1 = y, 2 = z)
  int nouter;         // outer lines per strip row
  long long stride;   // element stride along the line
  long long ostride;  // stride of the outer index
  int nstrips;        // nx / W
  int o0;             // global index of outer = 0 (y offset of a y-slab, 3-D z pass)
  int on;             // global extent of the outer axis (ny)
  int pad;
};

// geometry of a TMA 3-D column pass (cols3_lg.cuh)
struct Line3 {
  int nouter;   // outer lines per field (z for the y passes, y for the z pass)
  int o0, on;   // global index of outer 0 and the outer axis extent (wave numbers)
  int nfields;  // 1, or 2 (fields A and B: EM-type schemes)
  int axis;     // twiddle table of the line axis (1 = y, 2 = z)
  // tensor-map coordinates of outer line o: {.., (o >> obs) * om, o & (2^obs - 1), ..}
  // when om > 0 (y passes over the z-blocked layout), else {.., 0, o, ..}
  int obs, om;
  int f0;          // field of the first tile (1: a Parseval-only pass over field B's map)
  int no_monitor;  // projection pass whose residual belongs to another launch
};

// Destinations of a column pass whose outputs go straight to the rank that
// owns them (fused z-slab <-> y-slab transposes of the decomposed 3-D solve,
// peer memory over NVLink): element (c, line position pos, x) of the tile at
// outer index o lands in rank q = pos / rows_per_rank at
//   dst[field][q] + c*comp_stride + (outer0 + o)*outer_stride
//                 + (pos - q*rows_per_rank)*line_stride + x.
// With zs > 0 the destination is z-blocked (2^zs planes of a row adjacent,
// like Args::zbs): row ((b >> zs)*bn + u) << zs | (b & (2^zs - 1)) of length
// row_len, where (b, u) = (line position, outer) when blk_line, else
// (outer, line position); address = c*comp_stride + row*row_len + x.
struct PeerOut {
  double2* dst[2][8];
  int world, rows_per_rank;
  long long line_stride, outer_stride, outer0, comp_stride;
  int zs, blk_line;
  long long bn, row_len;
};

template <int MODE, int L, int E, int W, int C, int G>
__global__ void __launch_bounds__(G*W*(L / E)) k_col(Args a, ColGeom gm) {
  using P = Plan<L, E>;
  constexpr int T = P::T;
  constexpr int NQ = 1;
  constexpr int SKEW = (W > 1) ? 8 / W : 0;
  constexpr int CHS = W * (P::LP + SKEW);  // channel stride in shared memory
  extern __shared__ double2 smem[];
  if (!a.op_mode && a.st->stopped) return;
  const int col = threadIdx.x % W, t = (threadIdx.x / W) % T, g = threadIdx.x / (W * T);
  SmemBuf buf{smem + (size_t)g * C * CHS + col * (P::LP + SKEW), CHS};
  const int nfields = (MODE == MID_EM) ? 2 : 1;
  const int ncomp_lines = (C == 1) ? a.d : 1;  // plain passes: one component per line
  const long long per_field = (long long)gm.nouter * gm.nstrips * ncomp_lines;
  const long long lines = per_field * nfields;
  const double2* tw = a.tw[gm.axis];
  double acc[NQ] = {0.0};
  for (long long line0 = (long long)blockIdx.x * G; line0 < lines; line0 += (long long)gridDim.x * G) {
    const long long line = line0 + g;
    const bool live = line < lines;
    const int f = live ? (int)(line / per_field) : 0;
    long long rem = live ? line - (long long)f * per_field : 0;
    const int cl = (int)(rem / ((long long)gm.nouter * gm.nstrips));
    rem -= (long long)cl * gm.nouter * gm.nstrips;
    const int outer = (int)(rem / gm.nstrips);
    const int strip = (int)(rem - (long long)outer * gm.nstrips);
    const int x = strip * W + col;
    double2* F = (f == 0) ? a.A : a.B;
    const size_t base = (size_t)outer * gm.ostride + x;
    double2 v[C][E];
    if constexpr (MODE == COL_INV) {
#pragma unroll
      for (int i = 0; i < E; ++i)
        v[0][i] = live ? F[(size_t)cl * a.N + base + (size_t)pos_first<L, E>(true, t, i) * gm.stride] : czero();
      fft_line<L, E, 1, true>(v, t, tw, buf, SyncAll{});
      if (live)
#pragma unroll
        for (int i = 0; i < E; ++i)
          F[(size_t)cl * a.N + base + (size_t)pos_last<L, E>(true, t, i) * gm.stride] = v[0][i];
    } else {
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const size_t p = base + (size_t)pos_first<L, E>(false, t, i) * gm.stride;
#pragma unroll
        for (int c = 0; c < C; ++c) v[c][i] = live ? F[(size_t)(C == 1 ? cl : c) * a.N + p] : czero();
      }
      fft_line<L, E, C, false>(v, t, tw, buf, SyncAll{});
      if constexpr (MODE == COL_FWD) {
        if (live)
#pragma unroll
          for (int i = 0; i < E; ++i)
            F[(size_t)cl * a.N + base + (size_t)pos_last<L, E>(false, t, i) * gm.stride] = v[0][i];
      } else {
        // Gamma projection in registers (spectral_ops.py:124-127).  Wave
        // numbers: x from the column, the line axis from the position, the
        // remaining axis (3-D) from the outer index.
        const double kx = (double)wavenum(x, a.nx);
        double kyo = 0.0;
        if constexpr (C == 3) kyo = (double)wavenum(gm.o0 + outer, gm.on);
        const bool parseval_only = (MODE == MID_EM) && f == 1;
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int pos = pos_last<L, E>(false, t, i);
          double k[3];
          k[0] = kx;
          if constexpr (C == 2) {
            k[1] = (double)wavenum(pos, a.ny);
            k[2] = 0.0;
          } else {
            k[1] = kyo;
            k[2] = (double)wavenum(pos, a.nz);
          }
          double k2 = k[0] * k[0];
#pragma unroll
          for (int c = 1; c < C; ++c) k2 += k[c] * k[c];
          const double ik2 = (k2 != 0.0) ? inv_k2(k2) * a.gscale : 0.0;
          double2 dot = cscale(v[0][i], k[0]);
#pragma unroll
          for (int c = 1; c < C; ++c) dot = cadd(dot, cscale(v[c][i], k[c]));
          dot = cscale(dot, ik2);
          if (MODE == MID_BASIC || parseval_only) {
#pragma unroll
            for (int c = 0; c < C; ++c) {
              const double2 gc = cscale(dot, k[c]);
              // Parseval: sum_x |g|^2 = N sum_k |g^/N|^2; square the 1/N-scaled
              // mode so the sum overflows no earlier than the reference's
              if (live) acc[0] += cabs2(cscale(gc, a.inv_n));
              v[c][i] = gc;
            }
          } else {
#pragma unroll
            for (int c = 0; c < C; ++c) v[c][i] = csub(v[c][i], cscale(dot, 2.0 * k[c]));
          }
        }
        // Parseval-only lines need no inverse; skip it when the whole CTA agrees
        if (MODE == MID_EM && __syncthreads_and(parseval_only || !live)) continue;
        fft_line<L, E, C, true>(v, t, tw, buf, SyncAll{});
        if (live && !parseval_only) {
#pragma unroll
          for (int i = 0; i < E; ++i) {
            const size_t p = base + (size_t)pos_last<L, E>(true, t, i) * gm.stride;
#pragma unroll
            for (int c = 0; c < C; ++c) F[(size_t)c * a.N + p] = v[c][i];
          }
        }
      }
    }
  }
  if constexpr (MODE == MID_BASIC || MODE == MID_EM) {
    double tot[NQ];
    if (grid_reduce<NQ>(acc, tot, a) && threadIdx.x == 0 && !a.op_mode) {
      if (a.dist) a.st->parseval = tot[0] / a.inv_n;  // rank-local sum_x |g|^2
      else monitor_step(a, tot[0] / a.inv_n + a.st->js2);
    }
  }
}

// per-row x-extent of phase 1 (used to bound S/T prefetches); one warp per row
static __global__ void __launch_bounds__(256) k_row_extent(const uint8_t* __restrict__ chi, int nx, long long rows,
                                                     int2* __restrict__ ext) {
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r = warp; r < rows; r += nw) {
    int lo = nx, hi = -1;
    for (int x = lane; x < nx; x += 32)
      if (chi[(size_t)r * nx + x]) {
        lo = min(lo, x);
        hi = max(hi, x);
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) ext[r] = make_int2(lo, hi + 1);
  }
}

// chi rows -> the thread-blocked order of the row sweeps (Args::chiT): one
// thread per E-byte output chunk (row r, thread slot t) gathers the E bytes
// chi[r][t + i*T], i = 0..E-1, T = nx/E (consecutive t read consecutive bytes)
static __global__ void __launch_bounds__(256) k_chi_perm16(const uint8_t* __restrict__ chi, int nx, long long rows,
                                                          uint8_t* __restrict__ out, int E) {
  const int T = nx / E;  // (E = 16 or 8: Args::row_e)
  const long long n = rows * T;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long r = idx / T;
    const int t = (int)(idx - r * T);
    const uint8_t* src = chi + (size_t)r * nx + t;
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (4 * k < E)
        w[k] = (uint32_t)(src[(4 * k) * T] != 0) | ((uint32_t)(src[(4 * k + 1) * T] != 0) << 8) |
               ((uint32_t)(src[(4 * k + 2) * T] != 0) << 16) | ((uint32_t)(src[(4 * k + 3) * T] != 0) << 24);
    uint8_t* dst = out + (size_t)r * nx + (size_t)E * t;
    if (E == 16) *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
    else *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
  }
}

// phase-1 voxels per row (compact S/T layout): one warp per row
static __global__ void __launch_bounds__(256) k_row_counts(const uint8_t* __restrict__ chi, int nx, long long rows,
                                                         long long* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r = warp; r < rows; r += nw) {
    int n = 0;
    for (int x = lane; x < nx; x += 32) n += chi[(size_t)r * nx + x] != 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    if (lane == 0) cnt[r] = n;
  }
}

// rank codes of the compact layout (Args::chiR): one warp per row, lane l
// scans x in [l*nx/32, (l+1)*nx/32) in order after a warp prefix sum of the
// lanes' counts; codes land in the thread-blocked order of chiT
static __global__ void __launch_bounds__(256) k_chi_rank16(const uint8_t* __restrict__ chi, int nx, long long rows,
                                                         uint16_t* __restrict__ out, int E) {
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int span = nx >= 32 ? nx / 32 : 1;
  for (long long r = warp; r < rows; r += nw) {
    const uint8_t* row = chi + (size_t)r * nx;
    const int x0 = lane * span, x1 = min(nx, x0 + span);
    int n = 0;
    for (int x = x0; x < x1; ++x) n += row[x] != 0;
    int incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    int rank = incl - n;
    for (int x = x0; x < x1; ++x) {
      const bool in1 = row[x] != 0;
      out[tblock_index(r, x, nx, E)] = in1 ? (uint16_t)(rank + 1) : (uint16_t)0;
      rank += in1;
    }
  }
}

// ============================================================================
// 2-D projection sweep, component-split variant (the hot 2-D sweep 2).
// One thread carries ONE component of one column (E = 16 per thread, radix-16
// stages: two shared-memory exchanges per direction).  Lane layout inside a
// warp: bit 0 = column of the 2-wide strip, bit 1 = component, bits 2..4 =
// low bits of t; so the partner holding the other component of the same
// (column, t) is lane ^ 2 and the Gamma projection needs one complex shuffle
// per element (the partial dot product k_c F_c).  A warp touches 8 rows x 2
// components x 32 B: every 32-B sector it reads or writes is fully used.
// ============================================================================
template <int MODE, int L, int E>
__global__ void __launch_bounds__(4 * (L / E)) k_mid2(Args a, ColGeom gm) {
  using P = Plan<L, E>;
  constexpr int T = P::T;
  constexpr int NQ = 1;
  constexpr int SKEW = 2;                    // 4 channel buffers at bank offsets 0,2,4,6
  extern __shared__ double2 smem[];
  if (!a.op_mode && a.st->stopped) return;
  const int col = threadIdx.x & 1, comp = (threadIdx.x >> 1) & 1, t = threadIdx.x >> 2;
  double2* mybuf = smem + (comp * 2 + col) * (P::LP + SKEW);
  const SmemBuf buf{mybuf, 0};
  const int nfields = (MODE == MID_EM) ? 2 : 1;
  const long long lines = (long long)gm.nstrips * nfields;
  double acc[NQ] = {0.0};
  for (long long line = blockIdx.x; line < lines; line += gridDim.x) {
    const int f = (int)(line / gm.nstrips);
    const int strip = (int)(line - (long long)f * gm.nstrips);
    const int x = strip * 2 + col;
    double2* F = ((f == 0) ? a.A : a.B) + (size_t)comp * a.N + x;
    double2 v[1][E];
#pragma unroll
    for (int i = 0; i < E; ++i) v[0][i] = F[(size_t)pos_first<L, E>(false, t, i) * a.nx];
    fft_line<L, E, 1, false>(v, t, a.tw[1], buf, SyncAll{});
    const double kx = (double)wavenum(x, a.nx);
    const bool parseval_only = (MODE == MID_EM) && f == 1;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const double ky = (double)wavenum(pos_last<L, E>(false, t, i), a.ny);
      const double kc = comp ? ky : kx;
      const double k2 = kx * kx + ky * ky;
      const double ik2 = (k2 != 0.0) ? inv_k2(k2) * a.gscale : 0.0;
      const double2 mine = cscale(v[0][i], kc);
      double2 other;
      other.x = __shfl_xor_sync(0xffffffffu, mine.x, 2);
      other.y = __shfl_xor_sync(0xffffffffu, mine.y, 2);
      // same operand order in both lanes: kx F_x + ky F_y (spectral_ops.py:124)
      double2 dot = comp ? cadd(other, mine) : cadd(mine, other);
      dot = cscale(dot, ik2);
      if (MODE == MID_BASIC || parseval_only) {
        const double2 g = cscale(dot, kc);
        acc[0] += cabs2(cscale(g, a.inv_n));
        v[0][i] = g;
      } else {
        v[0][i] = csub(v[0][i], cscale(dot, 2.0 * kc));
      }
    }
    if (parseval_only) continue;  // uniform per CTA (one line per trip)
    fft_line<L, E, 1, true>(v, t, a.tw[1], buf, SyncAll{});
#pragma unroll
    for (int i = 0; i < E; ++i) F[(size_t)pos_last<L, E>(true, t, i) * a.nx] = v[0][i];
  }
  double tot[NQ];
  if (grid_reduce<NQ>(acc, tot, a) && threadIdx.x == 0 && !a.op_mode) {
    if (a.dist) a.st->parseval = tot[0] / a.inv_n;
    else monitor_step(a, tot[0] / a.inv_n + a.st->js2);
  }
}

// ============================================================================
// init and finalize (elementwise over component-major d*N)
// ============================================================================
template <int S>
__global__ void __launch_bounds__(256) k_init(Args a) {
  constexpr int NQ = 6;
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  const long long total = (long long)a.d * a.N;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i / a.N);
    const long long p = i - (long long)c * a.N;
    const bool in1 = a.chi[p] != 0;
    const double2 e0 = a.e0[c];
    double2 q;
    if constexpr (S == BASIC) {
      q = e0;
    } else if constexpr (S == EM) {
      double2 w = cmul(in1 ? a.sum1 : a.sum2, e0);  // w = (sigma + s0) e0   (:294)
      q = cmul(w, in1 ? a.inv_sum1 : a.inv_sum2);   // e_raw = w/(sigma+s0) (:308)
    } else if constexpr (S == BASIC_SUB) {
      q = e0;
      a.X[1][i] = czero();
    } else {
      // W = A F + s0 F with F = (e0, 0, 0)   (:386-387), then (A+s0)^-1 W
      AugFlux f = apply_A(a, in1, e0, czero(), czero());
      double2 wq = cadd(f.jq, cmul(a.s0, e0));
      double2 ws = f.js, wt = f.jt;
      double2 sn, tn;
      em_sub_update(a, in1, wq, ws, wt, q, sn, tn);
      if (a.rowoff) {  // compact slots: phase-1 voxels only
        if (in1) {
          const long long ci = compact_slot(a, c, p);
          a.X[1][ci] = sn;
          a.X[2][ci] = tn;
        }
      } else {
        a.X[1][i] = sn;
        a.X[2][i] = tn;
      }
    }
    a.X[0][i] = q;
    acc_c<NQ>(acc, c, q);
  }
  double tot[NQ];
  if (grid_reduce<NQ>(acc, tot, a) && threadIdx.x == 0) {
    DevState* st = a.st;
    for (int c = 0; c < a.d; ++c) {
      double2 m = make_double2(tot[2 * c] * a.inv_n, tot[2 * c + 1] * a.inv_n);
      st->delta[c] = csub(a.e0[c], m);
    }
    st->stopped = 0;
    st->status = ST_MAXITERS;
    st->degenerate = 0;
    st->nrec = 0;
    st->k = 1;
    st->has_prev = 0;
    st->res0 = 0.0;
    st->last_sstar = czero();
  }
}

template <int S>
__global__ void __launch_bounds__(256) k_finalize(Args a) {
  constexpr int NQ = 12;  // meanE (6) + meanJ (6)
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  const long long total = (long long)a.d * a.N;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i / a.N);
    const long long p = i - (long long)c * a.N;
    const bool in1 = a.chi[p] != 0;
    const double2 dl = a.st->delta[c];
    double2 E, J;
    if constexpr (S == BASIC || S == EM) {
      E = cadd(a.X[0][i], dl);
      J = cmul(sigma_at(a, in1), E);
    } else {
      double2 q = a.X[0][i];
      const long long si = (a.rowoff && in1) ? compact_slot(a, c, p) : i;
      double2 s = in1 ? a.X[1][si] : czero();
      double2 tt = (S == EM_SUB && in1) ? a.X[2][si] : czero();
      AugFlux f = apply_A(a, in1, q, s, tt);
      double2 js;
      pinned_flux(a, in1, f.jq, f.js, dl, J, js);
      E = cadd(q, dl);
      if (a.outAug) {
        a.outAug[i] = E;
        a.outAug[total + i] = s;
        a.outAug[2 * total + i] = tt;
      }
    }
    if (a.outE) a.outE[i] = E;
    if (a.outJ) a.outJ[i] = J;
#pragma unroll
    for (int cc = 0; cc < 3; ++cc)
      if (c == cc) {
        acc[2 * cc] += E.x;
        acc[2 * cc + 1] += E.y;
        acc[6 + 2 * cc] += J.x;
        acc[6 + 2 * cc + 1] += J.y;
      }
  }
  double tot[NQ];
  if (grid_reduce<NQ>(acc, tot, a) && threadIdx.x == 0) {
    for (int c = 0; c < a.d; ++c) {
      a.st->meanE[c] = make_double2(tot[2 * c] * a.inv_n, tot[2 * c + 1] * a.inv_n);
      a.st->meanJ[c] = make_double2(tot[6 + 2 * c] * a.inv_n, tot[6 + 2 * c + 1] * a.inv_n);
    }
  }
}

}  // namespace fftc
